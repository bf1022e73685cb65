"""ORACLE — test infrastructure only (not the product path).

Plain CPU reference for the Scepsy ALP allocation search (arXiv 2604.15186).
Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / ``--impl reference`` legs may
import this package.  It never imports paper_2604_15186_b200 and shares no code with it.

* O1  ``liboracle.so`` (alp_oracle.c): literal option terms + brute-force enumeration.
* O2  ``oracle.dp``: multiple-choice-knapsack DP + lowest-index DFS + counting DP (independent
      algorithm, used as a cross-check and for full-size C3-C5 answers).

Function-level citations are in alp_oracle.c's header; the readings of the paper are listed in
DESIGN.md §3.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass
from typing import Any

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(HERE, "alp_oracle.c")
_LIB = os.path.join(HERE, "liboracle.so")
PCT_KEYS = ("mean", "p50", "p90", "p99")


def build_lib(force: bool = False) -> str:
    """Compile the C oracle (plain gcc, no FMA contraction, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fPIC",
                               "-shared", "-pthread", _SRC, "-o", tmp, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


class _Inst(ctypes.Structure):
    _fields_ = [("M", ctypes.c_int), ("F", ctypes.c_int), ("nS", ctypes.c_int), ("nT", ctypes.c_int),
                ("nR", ctypes.c_int), ("n", ctypes.c_void_p), ("p", ctypes.c_void_p), ("S", ctypes.c_void_p),
                ("T", ctypes.c_void_p), ("R", ctypes.c_void_p), ("prof_off", ctypes.c_void_p),
                ("rate", ctypes.c_void_p), ("lat", ctypes.c_void_p), ("tmax", ctypes.c_void_p),
                ("min_units", ctypes.c_void_p), ("meas_off", ctypes.c_void_p), ("mrate", ctypes.c_void_p),
                ("mlat", ctypes.c_void_p), ("mtmax", ctypes.c_void_p)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(build_lib())
        P = ctypes.POINTER(_Inst)
        L.orc_lookup.restype = ctypes.c_double
        L.orc_lookup.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_double]
        L.orc_option.restype = ctypes.c_int
        L.orc_option.argtypes = [P, ctypes.c_double, ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                                 ctypes.c_void_p, ctypes.c_void_p]
        L.orc_option_table.restype = None
        L.orc_option_table.argtypes = [P, ctypes.c_double] + [ctypes.c_void_p] * 5
        L.orc_predict.restype = ctypes.c_int
        L.orc_predict.argtypes = [P, ctypes.c_double, ctypes.c_int64, ctypes.c_void_p] + [ctypes.c_void_p] * 4
        L.orc_search.restype = ctypes.c_int
        L.orc_search.argtypes = [P, ctypes.c_double, ctypes.c_int64, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int,
                                 ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
        L.orc_candidate.restype = ctypes.c_int
        L.orc_candidate.argtypes = [P, ctypes.c_double, ctypes.c_int64, ctypes.c_uint64, ctypes.c_void_p,
                                    ctypes.c_void_p]
        _lib = L
    return _lib


@dataclass
class Instance:
    """An ALP instance in the oracle's own flattened layout (kept alive with its numpy buffers)."""
    M: int
    F: int
    S: np.ndarray
    T: np.ndarray
    R: np.ndarray
    n: np.ndarray
    p: np.ndarray
    prof_off: np.ndarray
    rate: np.ndarray
    lat: np.ndarray
    tmax: np.ndarray
    min_units: np.ndarray | None
    budget: int
    raw: dict
    meas_off: np.ndarray | None = None   # measured per-share curves (R2), CSR over (m, t_i, s_i)
    mrate: np.ndarray | None = None
    mlat: np.ndarray | None = None
    mtmax: np.ndarray | None = None

    @property
    def K(self) -> int:
        return len(self.S) * len(self.T) * len(self.R)

    @property
    def N(self) -> int:
        return self.K ** self.M

    def cstruct(self) -> _Inst:
        return _Inst(self.M, self.F, len(self.S), len(self.T), len(self.R), self.n.ctypes.data, self.p.ctypes.data,
                     self.S.ctypes.data, self.T.ctypes.data, self.R.ctypes.data, self.prof_off.ctypes.data,
                     self.rate.ctypes.data, self.lat.ctypes.data, self.tmax.ctypes.data,
                     self.min_units.ctypes.data if self.min_units is not None else None,
                     *((self.meas_off.ctypes.data, self.mrate.ctypes.data, self.mlat.ctypes.data,
                        self.mtmax.ctypes.data) if self.meas_off is not None else (None, None, None, None)))


def from_json(d: dict[str, Any], percentile: str | None = None) -> Instance:
    pct = percentile or d.get("percentile", "mean")
    M, T = d["M"], d["tp"]
    off, rate, lat, tmax = [0], [], [], []
    for m in range(M):
        for ti in range(len(T)):
            c = d["profiles"][m][ti]
            rate += c["rate"]
            lat += c["lat"][pct]
            tmax.append(c["tmax"] if c.get("tmax") is not None else c["rate"][-1])
            off.append(len(rate))
    mu = d.get("min_units")
    I = Instance(M=M, F=d["F"], S=np.asarray(d["share_units"], np.int32), T=np.asarray(T, np.int32),
                 R=np.asarray(d["replicas"], np.int32), n=np.asarray(d["n"], np.float64),
                 p=np.asarray(d["p"], np.float64), prof_off=np.asarray(off, np.int32),
                 rate=np.asarray(rate, np.float64), lat=np.asarray(lat, np.float64),
                 tmax=np.asarray(tmax, np.float64),
                 min_units=None if mu is None else np.asarray(mu, np.int32).reshape(-1),
                 budget=int(d["budget_units"]), raw=d)
    meas = d.get("measured") or []
    if meas:  # R2: curves measured at (LLM, tp index, share index) -- SPEC.md:204
        nT, nS = len(T), len(d["share_units"])
        by = {(c["llm"], c["tp_index"], c["share_index"]): c for c in meas}
        moff, mrate, mlat, mtmax = [0], [], [], []
        for m in range(M):
            for ti in range(nT):
                for si in range(nS):
                    c = by.get((m, ti, si))
                    if c is not None:
                        mrate += c["rate"]
                        mlat += c["lat"][pct]
                    mtmax.append((c["tmax"] if c.get("tmax") is not None else c["rate"][-1]) if c else 0.0)
                    moff.append(len(mrate))
        I.meas_off = np.asarray(moff, np.int32)
        I.mrate = np.asarray(mrate, np.float64)
        I.mlat = np.asarray(mlat, np.float64)
        I.mtmax = np.asarray(mtmax, np.float64)
    return I


def lookup(rates, lats, x: float) -> float:
    r = np.ascontiguousarray(rates, np.float64)
    l = np.ascontiguousarray(lats, np.float64)
    return lib().orc_lookup(r.ctypes.data, l.ctypes.data, len(r), float(x))


def option(I: Instance, lam: float, m: int, k: int):
    tau = ctypes.c_float()
    term = ctypes.c_double()
    b = ctypes.c_double()
    u = ctypes.c_int()
    s = I.cstruct()
    ok = lib().orc_option(ctypes.byref(s), lam, m, k, ctypes.byref(tau), ctypes.byref(term), ctypes.byref(b),
                          ctypes.byref(u))
    return {"ok": bool(ok), "tau": np.float32(tau.value), "term": term.value, "b": b.value, "u": u.value}


def option_table(I: Instance, lam: float) -> dict[str, np.ndarray]:
    K = I.K
    tau = np.empty((I.M, K), np.float32)
    term = np.empty((I.M, K), np.float64)
    b = np.empty((I.M, K), np.float64)
    u = np.empty((I.M, K), np.int32)
    ok = np.empty((I.M, K), np.uint8)
    s = I.cstruct()
    lib().orc_option_table(ctypes.byref(s), lam, tau.ctypes.data, term.ctypes.data, b.ctypes.data, u.ctypes.data,
                           ok.ctypes.data)
    return {"tau": tau, "term": term, "b": b, "u": u, "ok": ok.astype(bool)}


@dataclass
class SearchResult:
    found: bool
    latency_key: float      # canonical FP32 objective (np.float32 value)
    index: int              # canonical mixed-radix index (lowest among ties)
    count: int              # feasible candidates


def search(I: Instance, lam: float, budget: int | None = None, lo: int = 0, hi: int | None = None,
           threads: int = 1) -> SearchResult:
    """O1 brute force over canonical indices [lo, hi)."""
    B = I.budget if budget is None else budget
    hi = I.N if hi is None else hi
    best = ctypes.c_float()
    idx = ctypes.c_uint64()
    cnt = ctypes.c_uint64()
    s = I.cstruct()
    found = lib().orc_search(ctypes.byref(s), lam, B, lo, hi, threads, ctypes.byref(best), ctypes.byref(idx),
                             ctypes.byref(cnt))
    return SearchResult(bool(found), float(np.float32(best.value)), int(idx.value) if found else -1, int(cnt.value))


def decode(I: Instance, idx: int) -> list[int]:
    """Canonical index -> per-LLM option index k_m (LLM 0 most significant)."""
    K = I.K
    out = []
    for _ in range(I.M):
        out.append(idx % K)
        idx //= K
    return out[::-1]


def option_grid(I: Instance, k: int) -> tuple[int, int, int]:
    """Option index k -> (share units, tp, replicas); k = (s_i*nT + t_i)*nR + r_i."""
    nT, nR = len(I.T), len(I.R)
    return int(I.S[k // (nT * nR)]), int(I.T[(k // nR) % nT]), int(I.R[k % nR])


def predict(I: Instance, lam: float, opts: list[int], budget: int | None = None):
    """FP64 Eq. 1 latency, Eq. 2 throughput, units, FP32 key, feasibility for one allocation."""
    B = I.budget if budget is None else budget
    o = np.asarray(opts, np.int32)
    L = ctypes.c_double()
    Tw = ctypes.c_double()
    U = ctypes.c_int64()
    l32 = ctypes.c_float()
    s = I.cstruct()
    ok = lib().orc_predict(ctypes.byref(s), lam, B, o.ctypes.data, ctypes.byref(L), ctypes.byref(Tw),
                           ctypes.byref(U), ctypes.byref(l32))
    return {"feasible": bool(ok), "latency": L.value, "throughput": Tw.value, "units": U.value,
            "latency_key": float(np.float32(l32.value))}


def candidate(I: Instance, lam: float, idx: int, budget: int | None = None):
    """One candidate recomputed from the profiles (no hoisting)."""
    B = I.budget if budget is None else budget
    l32 = ctypes.c_float()
    U = ctypes.c_int64()
    s = I.cstruct()
    ok = lib().orc_candidate(ctypes.byref(s), lam, B, idx, ctypes.byref(l32), ctypes.byref(U))
    return bool(ok), float(np.float32(l32.value)), U.value


def lambda_star(I: Instance, budget: int | None = None) -> float:
    """Budget-aware maximum workflow throughput: the largest v among all Eq. 2 terms
    b_m[k] such that some candidate is feasible at target lambda = v, i.e.
    sum_m min{u_m[k] : option k of LLM m is feasible at lambda = v} <= B.  Feasibility is the full R4
    test (x <= T and b >= lambda, both in FP64, plus the memory floor), so lambda* itself is feasible."""
    B = I.budget if budget is None else budget
    b = option_table(I, 1.0)["b"]  # Eq. 2 terms do not depend on lambda
    for v in np.unique(b)[::-1]:
        tab = option_table(I, float(v))
        tot = 0
        for m in range(I.M):
            sel = tab["u"][m][tab["ok"][m]]
            if sel.size == 0:
                tot = None
                break
            tot += int(sel.min())
        if tot is not None and tot <= B:
            return float(v)
    return 0.0


def floor_ok(I: Instance, m: int, k: int) -> bool:
    """Memory floor of option k of LLM m: share units >= min_units[m][tp index]."""
    if I.min_units is None:
        return True
    nT, nR = len(I.T), len(I.R)
    return int(I.S[k // (nT * nR)]) >= int(np.asarray(I.min_units).reshape(I.M, nT)[m][(k // nR) % nT])


def max_throughput(I: Instance, budget: int | None = None):
    """SPEC.md:374 "no feasible candidate -> returns the candidate with maximal T_w": by its plain
    definition, a brute force over every candidate within the budget whose options clear their
    memory floors, T_w = min_m b_m (Eq. 2, FP64; the Eq. 2 terms do not depend on the target),
    the lowest canonical index among equal T_w.  Small instances only (pure-Python loop).
    Returns None when no candidate fits the budget, else dict(index, throughput, units)."""
    import itertools
    B = I.budget if budget is None else budget
    tab = option_table(I, 1.0)
    ok = [[floor_ok(I, m, k) for k in range(I.K)] for m in range(I.M)]
    best = None
    for idx, ks in enumerate(itertools.product(range(I.K), repeat=I.M)):  # canonical order, LLM 0 first
        if not all(ok[m][k] for m, k in enumerate(ks)):
            continue
        units = sum(int(tab["u"][m][k]) for m, k in enumerate(ks))
        if units > B:
            continue
        tw = min(float(tab["b"][m][k]) for m, k in enumerate(ks))
        if best is None or tw > best["throughput"]:
            best = {"index": idx, "throughput": tw, "units": units}
    return best
