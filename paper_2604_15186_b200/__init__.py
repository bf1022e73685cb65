"""Python binding of the B200-native exhaustive ALP allocation search (Scepsy, arXiv 2604.15186).

Thin ctypes layer over the in-tree C-ABI library ``lib/libscepsy_alp.so`` (include/alp.h): it
marshals arguments only — every step of the search (option terms, candidate evaluation,
argmin/count, winner decode and FP64 prediction) runs in the sm_100a kernels.  There is no CPU
fallback: importing this package on a machine without the built library raises.

    from paper_2604_15186_b200 import Alp
    alp = Alp.from_instance(json_dict)          # alp_build
    r = alp.search(target, budget_units)        # alp_search -> Result
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field
from typing import Any, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("ALP_LIB") or os.path.join(HERE, "lib", "libscepsy_alp.so")  # ALP_LIB: tuning builds
MAX_M = 16
PCT = {"mean": 0, "p50": 1, "p90": 2, "p99": 3}

ALP_OK, ALP_EINVAL, ALP_EINFEASIBLE, ALP_EINTERNAL, ALP_ECUDA, ALP_ENCCL = range(6)


class AlpError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"alp status {status}: {msg}")
        self.status = status


class _Desc(ctypes.Structure):
    _fields_ = [("M", ctypes.c_int32), ("F", ctypes.c_int32), ("n", ctypes.c_void_p), ("p", ctypes.c_void_p),
                ("nS", ctypes.c_int32), ("nT", ctypes.c_int32), ("nR", ctypes.c_int32),
                ("share_units", ctypes.c_void_p), ("tp", ctypes.c_void_p), ("replicas", ctypes.c_void_p),
                ("prof_off", ctypes.c_void_p), ("rate", ctypes.c_void_p), ("lat", ctypes.c_void_p * 4),
                ("tmax", ctypes.c_void_p), ("min_units", ctypes.c_void_p), ("pct", ctypes.c_int32),
                ("meas_off", ctypes.c_void_p), ("meas_rate", ctypes.c_void_p), ("meas_lat", ctypes.c_void_p * 4),
                ("meas_tmax", ctypes.c_void_p)]


class _Result(ctypes.Structure):
    _fields_ = [("found", ctypes.c_int32), ("M", ctypes.c_int32), ("index", ctypes.c_uint64),
                ("latency_key", ctypes.c_float), ("latency", ctypes.c_double), ("throughput", ctypes.c_double),
                ("units", ctypes.c_int64), ("feasible_count", ctypes.c_uint64), ("candidates", ctypes.c_uint64),
                ("share_units", ctypes.c_int32 * MAX_M), ("tp", ctypes.c_int32 * MAX_M),
                ("replicas", ctypes.c_int32 * MAX_M), ("fallback", ctypes.c_int32)]


EXPORTS = ["alp_build", "alp_build_from_terms", "alp_destroy", "alp_num_candidates", "alp_h2d_bytes", "alp_decode",
           "alp_option_table", "alp_predict", "alp_search", "alp_search_batch", "alp_num_items", "alp_shard_range",
           "alp_search_shard", "alp_finalize", "alp_finalize_gathered", "alp_last_kernel_ms", "alp_last_launches",
           "alp_last_step_ms", "alp_last_path", "alp_last_error", "alp_plan_cache_clear", "alp_search_queries",
           "alp_schedule_egalitarian", "alp_workflow_stats", "alp_place", "alp_workspace_bytes",
           "alp_peer_bytes", "alp_peer_alloc", "alp_peer_free", "alp_peer_ipc_handle", "alp_peer_open",
           "alp_peer_close", "alp_search_peer"]

_lib = None


def lib():
    """Load the C-ABI library (fails loudly if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built: run `python -m paper_2604_15186_b200.build` "
                              "(there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        vp, i32, i64, u64, d = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_double
        sig = {
            "alp_build": (i32, [vp, vp]), "alp_build_from_terms": (i32, [i32, i32, vp, vp, vp]),
            "alp_destroy": (None, [vp]), "alp_num_candidates": (u64, [vp]), "alp_h2d_bytes": (u64, [vp]),
            "alp_decode": (i32, [vp, u64, vp, vp, vp]), "alp_option_table": (i32, [vp, d, vp, vp, vp, vp]),
            "alp_predict": (i32, [vp, vp, i32, d, i64, vp, vp, vp, vp]),
            "alp_search": (i32, [vp, d, i64, vp]), "alp_search_batch": (i32, [vp, vp, i32, i64, vp]),
            "alp_num_items": (u64, [vp, i64]), "alp_shard_range": (i32, [vp, i64, i32, i32, vp, vp]),
            "alp_search_shard": (i32, [vp, vp, i32, i64, u64, u64, vp, vp, vp, vp]),
            "alp_finalize": (i32, [vp, vp, i32, i64, vp, vp, vp, vp, vp]),
            "alp_finalize_gathered": (i32, [vp, vp, i32, i64, vp, i32, vp, vp, vp]),
            "alp_workspace_bytes": (ctypes.c_size_t, [vp, i32]),
            "alp_last_kernel_ms": (ctypes.c_float, [vp]), "alp_last_launches": (i32, [vp]),
            "alp_last_step_ms": (ctypes.c_float, [vp]), "alp_last_path": (i32, [vp]),
            "alp_last_error": (ctypes.c_char_p, []), "alp_plan_cache_clear": (None, []),
            "alp_search_queries": (i32, [vp, vp, vp, i32, vp]),
            "alp_schedule_egalitarian": (i32, [vp, vp, i32, i32, i32, vp, vp, vp, vp]),
            "alp_workflow_stats": (i32, [i32, i32, i64, vp, vp, vp, vp, vp, vp]),
            "alp_place": (i32, [i32, i32, vp, vp, i32, vp, vp, vp, vp]),
            "alp_peer_bytes": (ctypes.c_size_t, [i32, i32]), "alp_peer_alloc": (i32, [ctypes.c_size_t, vp]),
            "alp_peer_free": (i32, [vp]), "alp_peer_ipc_handle": (i32, [vp, vp]), "alp_peer_open": (i32, [vp, vp]),
            "alp_peer_close": (i32, [vp]),
            "alp_search_peer": (i32, [vp, vp, i32, i64, u64, u64, i32, i32, vp, vp, vp, vp]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _stream(stream_ptr: int | None):
    """cudaStream_t for the C ABI: None -> NULL (the handle's own stream); a torch stream handle of
    0 (the legacy default stream) -> cudaStreamLegacy, so the call is ordered with torch's default
    stream instead of silently running on the handle's stream."""
    if stream_ptr is None:
        return None
    return stream_ptr or 1  # 0x1 = cudaStreamLegacy


def plan_cache_clear() -> None:
    """alp_plan_cache_clear: drop the process-wide cache of static search plans."""
    lib().alp_plan_cache_clear()


def schedule_egalitarian(alps: Sequence["Alp"], targets: Sequence[float], gpus: int, units_per_gpu: int):
    """alp_schedule_egalitarian: split `gpus` whole GPUs across workflows (max-min utility).
    Returns (gpus per workflow, per-workflow Result, min utility, sum utility)."""
    W = len(alps)
    hs = (ctypes.c_void_p * W)(*[a._h.value for a in alps])
    t = _arr(targets, np.float64)
    g = np.zeros(W, np.int32)
    out = (_Result * W)()
    mn = ctypes.c_double()
    sm = ctypes.c_double()
    _check(lib().alp_schedule_egalitarian(hs, t.ctypes.data, W, gpus, units_per_gpu, g.ctypes.data, out,
                                          ctypes.byref(mn), ctypes.byref(sm)), (ALP_OK, ALP_EINFEASIBLE))
    return g.tolist(), [Result._from(x) for x in out], mn.value, sm.value


def workflow_stats(n_req: int, M: int, req, llm, start, end):
    """alp_workflow_stats: (n_m, p_m) per LLM from invocation records."""
    r = _arr(req, np.int32)
    l = _arr(llm, np.int32)
    s = _arr(start, np.float64)
    e = _arr(end, np.float64)
    n = np.zeros(M, np.float64)
    p = np.zeros(M, np.float64)
    _check(lib().alp_workflow_stats(n_req, M, len(r), r.ctypes.data, l.ctypes.data, s.ctypes.data, e.ctypes.data,
                                    n.ctypes.data, p.ctypes.data))
    return n, p


def place(gpu_node, gpu_domain, F: int, share_units, tp, replicas):
    """alp_place: GPU index of every shard, ordered (LLM, replica, shard)."""
    gn = _arr(gpu_node, np.int32)
    gd = _arr(gpu_domain, np.int32)
    s = _arr(share_units, np.int32)
    t = _arr(tp, np.int32)
    r = _arr(replicas, np.int32)
    out = np.zeros(int((t * r).sum()), np.int32)
    _check(lib().alp_place(len(gn), F, gn.ctypes.data, gd.ctypes.data, len(s), s.ctypes.data, t.ctypes.data,
                           r.ctypes.data, out.ctypes.data))
    return out.tolist()


class PeerBuffer:
    """An exchange buffer of the fused peer exchange (alp_peer_alloc on the current device), or a
    mapping of another process's buffer (from_ipc).  Frees / unmaps on close."""

    def __init__(self, ptr: int, owned: bool):
        self.ptr, self._owned = ptr, owned

    @staticmethod
    def nbytes(n_targets: int, world: int) -> int:
        return int(lib().alp_peer_bytes(n_targets, world))

    @classmethod
    def alloc(cls, n_targets: int, world: int) -> "PeerBuffer":
        p = ctypes.c_void_p()
        _check(lib().alp_peer_alloc(cls.nbytes(n_targets, world), ctypes.byref(p)))
        return cls(p.value, True)

    def ipc_handle(self) -> bytes:
        h = ctypes.create_string_buffer(64)
        _check(lib().alp_peer_ipc_handle(ctypes.c_void_p(self.ptr), h))
        return h.raw

    @classmethod
    def from_ipc(cls, handle: bytes) -> "PeerBuffer":
        p = ctypes.c_void_p()
        _check(lib().alp_peer_open(ctypes.create_string_buffer(handle, 64), ctypes.byref(p)))
        return cls(p.value, False)

    def close(self):
        if self.ptr:
            (lib().alp_peer_free if self._owned else lib().alp_peer_close)(ctypes.c_void_p(self.ptr))
        self.ptr = 0


def _check(st: int, ok=(ALP_OK,)) -> int:
    if st not in ok:
        raise AlpError(st, lib().alp_last_error().decode())
    return st


@dataclass
class Result:
    found: bool
    index: int
    latency_key: float          # canonical binary32 objective
    latency: float              # FP64 Eq. 1
    throughput: float           # FP64 Eq. 2
    units: int
    feasible_count: int
    candidates: int
    share_units: list = field(default_factory=list)
    tp: list = field(default_factory=list)
    replicas: list = field(default_factory=list)
    # found = False but fallback = True: index / share_units / tp / replicas / units / throughput are
    # the candidate with the maximal Eq. 2 T_w within the budget ("INFEASIBLE-rate")
    fallback: bool = False

    @staticmethod
    def _from(r: _Result) -> "Result":
        M = r.M
        shown = r.found or r.fallback
        return Result(bool(r.found), int(r.index) if shown else -1, float(np.float32(r.latency_key)), r.latency,
                      r.throughput, int(r.units), int(r.feasible_count), int(r.candidates),
                      list(r.share_units[:M]), list(r.tp[:M]), list(r.replicas[:M]), bool(r.fallback))


def _arr(x, dt):
    return np.ascontiguousarray(np.asarray(x, dtype=dt))


class Desc:
    """Host-side alp_desc: the profile tables and workflow statistics of an instance dict
    (workloads/instances/*.json layout) as contiguous arrays, kept alive with the struct."""

    def __init__(self, d: dict, percentile: str | None = None):
        M, T = d["M"], d["tp"]
        off, rate, lat, tmax = [0], [], {k: [] for k in PCT}, []
        for m in range(M):
            for ti in range(len(T)):
                c = d["profiles"][m][ti]
                rate += c["rate"]
                for k in PCT:
                    lat[k] += c["lat"][k] if k in c["lat"] else [float("nan")] * len(c["rate"])
                tmax.append(c["tmax"] if c.get("tmax") is not None else c["rate"][-1])
                off.append(len(rate))
        keep = dict(n=_arr(d["n"], np.float64), p=_arr(d["p"], np.float64), S=_arr(d["share_units"], np.int32),
                    T=_arr(T, np.int32), R=_arr(d["replicas"], np.int32), off=_arr(off, np.int32),
                    rate=_arr(rate, np.float64), tmax=_arr(tmax, np.float64),
                    **{f"lat_{k}": _arr(v, np.float64) for k, v in lat.items()})
        mu = d.get("min_units")
        if mu is not None:
            keep["minu"] = _arr(mu, np.int32).reshape(-1)
        meas = d.get("measured") or []
        if meas:  # profiles measured at (LLM, tp index, share index): CSR over (m, t, s) curves
            nS = len(d["share_units"])
            by = {(c["llm"], c["tp_index"], c["share_index"]): c for c in meas}
            moff, mrate, mlat, mtmax = [0], [], {k: [] for k in PCT}, []
            for m in range(M):
                for ti in range(len(T)):
                    for si in range(nS):
                        c = by.get((m, ti, si))
                        if c is not None:
                            mrate += c["rate"]
                            for k in PCT:
                                mlat[k] += c["lat"][k] if k in c["lat"] else [float("nan")] * len(c["rate"])
                        mtmax.append((c["tmax"] if c.get("tmax") is not None else c["rate"][-1]) if c else 0.0)
                        moff.append(len(mrate))
            keep.update(moff=_arr(moff, np.int32), mrate=_arr(mrate, np.float64), mtmax=_arr(mtmax, np.float64),
                        **{f"mlat_{k}": _arr(v, np.float64) for k, v in mlat.items()})
        c = _Desc()
        c.M, c.F = M, d["F"]
        c.n, c.p = keep["n"].ctypes.data, keep["p"].ctypes.data
        c.nS, c.nT, c.nR = len(keep["S"]), len(keep["T"]), len(keep["R"])
        c.share_units, c.tp, c.replicas = keep["S"].ctypes.data, keep["T"].ctypes.data, keep["R"].ctypes.data
        c.prof_off, c.rate = keep["off"].ctypes.data, keep["rate"].ctypes.data
        for k, i in PCT.items():
            c.lat[i] = keep[f"lat_{k}"].ctypes.data
        c.tmax = keep["tmax"].ctypes.data
        c.min_units = keep["minu"].ctypes.data if "minu" in keep else None
        if "moff" in keep:
            c.meas_off, c.meas_rate, c.meas_tmax = (keep["moff"].ctypes.data, keep["mrate"].ctypes.data,
                                                    keep["mtmax"].ctypes.data)
            for k, i in PCT.items():
                c.meas_lat[i] = keep[f"mlat_{k}"].ctypes.data
        c.pct = PCT[percentile or d.get("percentile", "mean")]
        self.c, self.M, self._keep = c, M, keep

    @property
    def nbytes(self) -> int:
        """Bytes of the arrays alp_build reads (the selected latency column only)."""
        sel = {p + k for k, i in PCT.items() if i == self.c.pct for p in ("lat_", "mlat_")}
        return int(sum(v.nbytes for k, v in self._keep.items() if not k.startswith(("lat_", "mlat_")) or k in sel))


class Alp:
    """Handle to an immutable ALP (alp_t).  Not thread-safe; one handle per host thread."""

    def __init__(self, handle: int, M: int, keep: Any = None):
        self._h = ctypes.c_void_p(handle)
        self.M = M
        self._keep = keep

    # ------------------------------------------------------------------ construction
    @classmethod
    def from_instance(cls, d: dict, percentile: str | None = None) -> "Alp":
        """alp_build from an instance dict (workloads/instances/*.json layout)."""
        return cls.build(Desc(d, percentile))

    @classmethod
    def build(cls, desc: "Desc") -> "Alp":
        """alp_build from prepared host arrays (Desc)."""
        h = ctypes.c_void_p()
        _check(lib().alp_build(ctypes.byref(desc.c), ctypes.byref(h)))
        return cls(h.value, desc.M)

    @classmethod
    def from_terms(cls, tau: np.ndarray, u: np.ndarray) -> "Alp":
        """Test-only: alp_build_from_terms over given binary32 option terms and units [M, K]."""
        t = _arr(tau, np.float32)
        uu = _arr(u, np.int32)
        M, K = t.shape
        h = ctypes.c_void_p()
        _check(lib().alp_build_from_terms(M, K, t.ctypes.data, uu.ctypes.data, ctypes.byref(h)))
        return cls(h.value, M)

    def close(self):
        if self._h is not None and self._h.value:
            lib().alp_destroy(self._h)
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # ------------------------------------------------------------------ queries
    @property
    def num_candidates(self) -> int:
        return int(lib().alp_num_candidates(self._h))

    @property
    def h2d_bytes(self) -> int:
        return int(lib().alp_h2d_bytes(self._h))

    def decode(self, index: int):
        s = np.zeros(self.M, np.int32)
        t = np.zeros(self.M, np.int32)
        r = np.zeros(self.M, np.int32)
        _check(lib().alp_decode(self._h, index, s.ctypes.data, t.ctypes.data, r.ctypes.data))
        return list(zip(s.tolist(), t.tolist(), r.tolist()))

    def option_table(self, lam: float, K: int):
        tau = np.empty((self.M, K), np.float32)
        term = np.empty((self.M, K), np.float64)
        b = np.empty((self.M, K), np.float64)
        u = np.empty((self.M, K), np.int32)
        _check(lib().alp_option_table(self._h, lam, tau.ctypes.data, term.ctypes.data, b.ctypes.data, u.ctypes.data))
        return {"tau": tau, "term": term, "b": b, "u": u}

    def predict(self, opts: Sequence[Sequence[int]], lam: float, budget: int):
        o = _arr(opts, np.int32).reshape(-1, self.M)
        n = o.shape[0]
        lat = np.empty(n, np.float64)
        thr = np.empty(n, np.float64)
        units = np.empty(n, np.int64)
        feas = np.empty(n, np.int32)
        _check(lib().alp_predict(self._h, o.ctypes.data, n, lam, budget, lat.ctypes.data, thr.ctypes.data,
                                 units.ctypes.data, feas.ctypes.data))
        return {"latency": lat, "throughput": thr, "units": units, "feasible": feas.astype(bool)}

    # ------------------------------------------------------------------ search
    def search(self, target: float, budget: int) -> Result:
        r = _Result()
        _check(lib().alp_search(self._h, target, budget, ctypes.byref(r)), (ALP_OK, ALP_EINFEASIBLE))
        return Result._from(r)

    def search_batch(self, targets: Sequence[float], budget: int) -> list[Result]:
        t = _arr(targets, np.float64)
        out = (_Result * len(t))()
        _check(lib().alp_search_batch(self._h, t.ctypes.data, len(t), budget, out), (ALP_OK, ALP_EINFEASIBLE))
        return [Result._from(x) for x in out]

    def search_queries(self, targets: Sequence[float], budgets: Sequence[int]) -> list[Result]:
        """alp_search_queries: independent (target, budget) pairs in one pass."""
        t = _arr(targets, np.float64)
        bu = _arr(budgets, np.int64)
        if len(t) != len(bu):
            raise ValueError("targets and budgets differ in length")
        out = (_Result * len(t))()
        _check(lib().alp_search_queries(self._h, t.ctypes.data, bu.ctypes.data, len(t), out), (ALP_OK, ALP_EINFEASIBLE))
        return [Result._from(x) for x in out]

    def num_items(self, budget: int) -> int:
        return int(lib().alp_num_items(self._h, budget))

    def shard_range(self, budget: int, rank: int, world: int) -> tuple[int, int]:
        lo = ctypes.c_uint64()
        hi = ctypes.c_uint64()
        _check(lib().alp_shard_range(self._h, budget, rank, world, ctypes.byref(lo), ctypes.byref(hi)))
        return lo.value, hi.value

    def workspace_bytes(self, n_targets: int) -> int:
        """alp_workspace_bytes: size of a caller workspace for n_targets (allocate zero-filled, e.g.
        torch.zeros(bytes, dtype=torch.uint8, device="cuda"))."""
        return int(lib().alp_workspace_bytes(self._h, n_targets))

    def search_shard(self, targets: Sequence[float], budget: int, lo: int, hi: int, keys_ptr: int, counts_ptr: int,
                     stream_ptr: int | None = None, workspace_ptr: int | None = None) -> None:
        """Async: evaluate items [lo, hi) for every target into device int64 keys/counts (on a caller
        workspace when workspace_ptr is given: not ordered against other calls)."""
        t = _arr(targets, np.float64)
        _check(lib().alp_search_shard(self._h, t.ctypes.data, len(t), budget, lo, hi, workspace_ptr,
                                      _stream(stream_ptr), keys_ptr, counts_ptr))

    def finalize(self, targets: Sequence[float], budget: int, keys_ptr: int, counts_ptr: int,
                 stream_ptr: int | None = None, workspace_ptr: int | None = None) -> list[Result]:
        t = _arr(targets, np.float64)
        out = (_Result * len(t))()
        _check(lib().alp_finalize(self._h, t.ctypes.data, len(t), budget, keys_ptr, counts_ptr, workspace_ptr,
                                  _stream(stream_ptr), out),
               (ALP_OK, ALP_EINFEASIBLE))
        return [Result._from(x) for x in out]

    def finalize_gathered(self, targets: Sequence[float], budget: int, gathered_ptr: int, world: int,
                          stream_ptr: int | None = None, workspace_ptr: int | None = None) -> list[Result]:
        """alp_finalize_gathered: finalize from all-gathered per-rank int64[world][2][n] pairs."""
        t = _arr(targets, np.float64)
        out = (_Result * len(t))()
        _check(lib().alp_finalize_gathered(self._h, t.ctypes.data, len(t), budget, gathered_ptr, world,
                                           workspace_ptr, _stream(stream_ptr), out), (ALP_OK, ALP_EINFEASIBLE))
        return [Result._from(x) for x in out]

    def search_peer(self, targets: Sequence[float], budget: int, lo: int, hi: int, rank: int, bufs: Sequence[int],
                    stream_ptr: int | None = None, workspace_ptr: int | None = None) -> list[Result]:
        """alp_search_peer: search items [lo, hi) and reduce across the len(bufs) ranks inside the
        kernel over peer memory (bufs = every rank's exchange buffer pointer in this process)."""
        t = _arr(targets, np.float64)
        b = (ctypes.c_void_p * len(bufs))(*bufs)
        out = (_Result * len(t))()
        _check(lib().alp_search_peer(self._h, t.ctypes.data, len(t), budget, lo, hi, rank, len(bufs), b,
                                     workspace_ptr, _stream(stream_ptr), out), (ALP_OK, ALP_EINFEASIBLE))
        return [Result._from(x) for x in out]

    @property
    def last_kernel_ms(self) -> float:
        return float(lib().alp_last_kernel_ms(self._h))

    @property
    def last_step_ms(self) -> float:
        """Device time of the last complete search step (alp_last_step_ms)."""
        return float(lib().alp_last_step_ms(self._h))

    @property
    def last_path(self) -> str:
        """Search kernel of the last search: "k_search" or "k_search_u" (alp_last_path)."""
        return "k_search_u" if lib().alp_last_path(self._h) == 1 else "k_search"

    @property
    def last_launches(self) -> int:
        return int(lib().alp_last_launches(self._h))
