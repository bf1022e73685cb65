"""Benchmark: exhaustive ALP allocation search (Scepsy, arXiv 2604.15186) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload C4] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...        (one rank per GPU, NCCL)

A step = one full search of the workload: at N=1 one fused kernel (option terms, exhaustive
evaluation of all N candidates, finalize; result stored zero-copy); at N>1 the sharded search
kernel on every rank, ONE NCCL all-gather of the 16-byte (key, count) pairs, device finalize.  value = candidates evaluated per second for the whole job (max over
ranks of the device time); inputs (profile tables) are resident in HBM before the timed region.
e2e = the same metric through the C ABI from HOST buffers: alp_build (H2D of the profiles and the
plan) + search + D2H of the result + alp_destroy, per step.

Rank 0 prints ONE JSON line.  See DESIGN.md §6 for the roofline definition.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "ALP candidates evaluated/sec and time-to-optimum at 1/2/4/8 B200 vs CPU oracle"
UNIT = "candidates/s"
ISSUE_LANES_PER_SM_PER_CLK = 128   # 4 SMSPs x 1 warp-instruction/clk x 32 lanes
INSTR_PER_CANDIDATE_MIN = 1.0      # 1/2 FADD2 + 1/2 FMNMX3


def _env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


def load_workload(name):
    from workloads import generate
    return generate.load(name)


# --------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.12)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
            except ValueError:
                continue
            for nm, v in zip(names, f[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


# --------------------------------------------------------------------------- CPU oracle leg
def oracle_rate(d, seconds=12.0, threads=None):
    """O1 brute force (the oracle as it stands) on a bounded contiguous sample of the workload,
    all host cores; returns (cand/s, cores, sample description, elapsed s)."""
    import oracle
    I = oracle.from_json(d)
    lam = d["targets"][0]
    threads = threads or os.cpu_count() or 1
    n = min(I.N, 4_000_000 * threads)
    t0 = time.perf_counter()
    oracle.search(I, lam, I.budget, lo=0, hi=n, threads=threads)
    dt = time.perf_counter() - t0
    n2 = int(min(I.N, max(n, n * seconds / max(dt, 1e-3))))
    t0 = time.perf_counter()
    o = oracle.search(I, lam, I.budget, lo=0, hi=n2, threads=threads)
    dt = time.perf_counter() - t0
    full = o if n2 == I.N else None  # the whole space: the oracle's answer for a parity check
    return n2 / dt, threads, f"canonical indices [0, {n2}) of {d['name']} (N={I.N}), {threads} threads", dt, full


def run_reference(args):
    rank = _env_int("RANK", 0)
    if rank != 0:
        return
    d = load_workload(args.workload)
    import oracle
    I = oracle.from_json(d)
    threads = os.cpu_count() or 1
    lam = d["targets"][0]
    n = min(I.N, 30_000_000 * threads // 8)
    for _ in range(args.warmup):
        oracle.search(I, lam, I.budget, lo=0, hi=min(n, 1_000_000), threads=threads)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        oracle.search(I, lam, I.budget, lo=0, hi=n, threads=threads)
        times.append(time.perf_counter() - t0)
    tot = sum(times)
    v = n * len(times) / tot
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * tot / len(times), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": _config(d, I.N, args.gpus),
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": "oracle",
                             "sample": f"canonical indices [0, {n}) of {d['name']} per step (O1 brute force)"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def _config(d, N, world, exchange=None):
    if world == 1:
        par = "one GPU: the whole index space"
    elif exchange == "peer":
        par = f"index-space shard x{world} + fused peer exchange in the search kernel (NVLink stores, no collective)"
    else:
        par = f"index-space shard x{world} + NCCL all-gather of (key, count) pairs" + (
            f" [{exchange}]" if exchange and exchange != "nccl" else "")
    return {"workload": f"{d['name']}: {d['description']}", "candidates": N * len(d["targets"]), "M": d["M"],
            "options_per_llm": len(d["share_units"]) * len(d["tp"]) * len(d["replicas"]),
            "budget_units": d["budget_units"], "F": d["F"], "target_req_s": d["targets"][0],
            "n_targets": len(d["targets"]), "parallelism": par,
            "l2": "flushed between timed steps (256 MiB write)"}


# --------------------------------------------------------------------------- our path
def run_ours(args):
    import torch
    import torch.distributed as dist

    rank = _env_int("RANK", 0)
    world = _env_int("WORLD_SIZE", 1)
    local = _env_int("LOCAL_RANK", 0)
    # one rank per GPU; ALP_DIST_BACKEND=gloo lets several ranks share one GPU (test only: NCCL
    # rejects duplicate devices), the product path is NCCL over NVLink.
    backend = os.environ.get("ALP_DIST_BACKEND", "nccl")
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    from paper_2604_15186_b200 import build as pbuild
    if rank == 0 or world == 1:
        pbuild.build()
    if world > 1:
        dist.barrier()
    import paper_2604_15186_b200 as P
    from paper_2604_15186_b200.dist import PeerExchange, gather_pairs

    d = load_workload(args.workload)
    B = int(d["budget_units"])
    targets = list(d["targets"])  # C1-C4: one target; C5: the 256-target Pareto sweep in one pass
    nt = len(targets)
    alp = P.Alp.from_instance(d)
    N = alp.num_candidates
    lo, hi = alp.shard_range(B, rank, world)
    stream = torch.cuda.Stream(device=dev)
    pairs = torch.empty(2 * nt, dtype=torch.int64, device=dev)             # this rank's (keys, counts)
    gathered = torch.empty(world * 2 * nt, dtype=torch.int64, device=dev)  # every rank's pairs
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    exchange = args.exchange if world > 1 else "none"
    px, probe = None, None
    if exchange in ("peer", "auto"):
        try:
            px = PeerExchange(nt)  # IPC handles of every rank's exchange buffer over the group
        except Exception as e:  # no peer access between these GPUs: the NCCL exchange instead
            probe = {"peer_unavailable": str(e)[:160]}
        ok = torch.tensor([1 if px is not None else 0], dtype=torch.int64, device=dev)
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        if not int(ok.item()):
            px = None
    ws = torch.zeros(alp.workspace_bytes(nt), dtype=torch.uint8, device=dev) if px is not None else None
    use_peer = px is not None and exchange == "peer"

    def run_step(a, lo_, hi_, peer=None):
        """One search step through the public API: at N=1 the single-GPU call (option terms +
        exhaustive search + finalize); at N>1 shard search, then the exchange: the fused peer
        exchange inside the search kernel, or ONE NCCL all-gather of the (key, count) pairs + the
        device finalize."""
        if world == 1:
            return a.search_batch(targets, B)[-1]
        if use_peer if peer is None else peer:
            w2 = ws if a is alp else torch.zeros(a.workspace_bytes(nt), dtype=torch.uint8, device=dev)
            return a.search_peer(targets, B, lo_, hi_, rank, px.ptrs, stream.cuda_stream, w2.data_ptr())[-1]
        with torch.cuda.stream(stream):
            a.search_shard(targets, B, lo_, hi_, pairs.data_ptr(), pairs.data_ptr() + 8 * nt, stream.cuda_stream)
            w = gather_pairs(pairs, gathered)  # ONE all-gather of the 16-byte (key, count) pairs
            return a.finalize_gathered(targets, B, gathered.data_ptr(), w, stream.cuda_stream)[-1]

    if exchange == "auto" and px is not None:
        # measured choice: both exchanges on this box (device step, max over ranks, median of 10 after
        # 3 warm-ups, L2 flushed); they must return the same result; the faster one is timed below
        probe = {}
        got = {}
        for mode in ("nccl", "peer"):
            ms, good = [], 1
            try:
                for i in range(13):
                    with torch.cuda.stream(stream):
                        flush.zero_()
                    torch.cuda.synchronize()
                    dist.barrier()
                    r = run_step(alp, lo, hi, mode == "peer")
                    if i >= 3:
                        ms.append(alp.last_step_ms)
                got[mode] = (r.found, r.index, r.feasible_count)
            except Exception as e:  # e.g. a peer-exchange timeout: the NCCL exchange is timed
                good = 0
                probe[f"{mode}_error"] = str(e)[:160]
            t = torch.tensor([sorted(ms)[len(ms) // 2] if ms else 1e9, good], dtype=torch.float64, device=dev)
            dist.all_reduce(t[:1], op=dist.ReduceOp.MAX)
            dist.all_reduce(t[1:], op=dist.ReduceOp.MIN)
            probe[f"{mode}_step_ms"] = float(t[0]) if int(t[1]) else None
        agree = torch.tensor([1 if got.get("peer") is not None and got.get("peer") == got.get("nccl") else 0],
                             dtype=torch.int64, device=dev)
        dist.all_reduce(agree, op=dist.ReduceOp.MIN)
        probe["results_agree"] = bool(agree.item())
        use_peer = bool(agree.item()) and probe["peer_step_ms"] is not None and \
            probe["peer_step_ms"] < (probe["nccl_step_ms"] or 1e9)
    exchange = "peer" if use_peer else ("nccl" if world > 1 else "none")

    def step():
        return run_step(alp, lo, hi)

    for _ in range(max(3, args.warmup)):
        res = step()
    # Step time = CUDA events on the search stream, recorded by the library from the start of the
    # search call to the completion of the result D2H (alp_last_step_ms).  host_ms = host wall time
    # of the call until the result is on the host (time to optimum, incl. launch + wake-up).
    step_ms, kern_ms, host_ms = [], [], []
    launches = 0
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            with torch.cuda.stream(stream):
                flush.zero_()
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            h0 = time.perf_counter()
            res = step()  # returns with the result on the host
            host_ms.append(1e3 * (time.perf_counter() - h0))
            step_ms.append(alp.last_step_ms)
            kern_ms.append(alp.last_kernel_ms)
            launches += alp.last_launches
    tot_ms = sum(step_ms)
    kern_tot = sum(kern_ms)
    t = torch.tensor([tot_ms, kern_tot, sum(host_ms)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    tot_ms, kern_max, host_tot = t.tolist()

    # ---- end to end through the C ABI from host buffers: alp_build (validation, H2D of the profile
    # tables from pinned staging; the static plan comes from the process-wide plan cache) + search
    # (K1, K2, all-reduce, K3) + D2H of the result + alp_destroy, per step.  One extra "cold" step
    # first clears the plan cache so it also pays host planning + the plan upload.
    desc = P.Desc(d)  # host arrays of the step's inputs, prepared outside the timed region

    def e2e_step():
        t0 = time.perf_counter()
        a2 = P.Alp.build(desc)
        lo2, hi2 = a2.shard_range(B, rank, world)
        r2 = run_step(a2, lo2, hi2)
        h2d = a2.h2d_bytes + 8 * len(targets)
        a2.close()
        assert r2.index == res.index
        return (time.perf_counter() - t0) * 1e3, h2d
    if world > 1:
        dist.barrier()
    P.plan_cache_clear()
    cold_ms, cold_h2d = e2e_step()
    e2e_ms = []
    h2d = 0
    for i in range(args.e2e_steps):
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        ms, h2d = e2e_step()
        e2e_ms.append(ms)
    te = torch.tensor([sum(e2e_ms), cold_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_tot, cold_ms = te.tolist()

    if rank == 0:
        cs = clk.summary()
        sm_count = torch.cuda.get_device_properties(dev).multi_processor_count
        f_max = (cs["sm_max_mhz"] or 1965.0) * 1e6
        cand_rank = N * nt * (hi - lo) / max(1, alp.num_items(B))
        achieved = cand_rank / (kern_max / len(kern_ms) * 1e-3)  # per GPU, dominant kernel
        peak = sm_count * ISSUE_LANES_PER_SM_PER_CLK * f_max / INSTR_PER_CANDIDATE_MIN
        # DRAM traffic and pipe utilisation of the search kernel cannot be measured inside a timed run
        # (ncu replays kernels): they come from this round's committed `ncu --set full` capture of the
        # same kernel on the same workload (profiles/ncu_summary.json, tools/collect_profiles.sh)
        traffic, pipes = None, None
        tp = os.path.join(ROOT, "profiles", "ncu_summary.json")
        if os.path.exists(tp):
            try:
                ent = json.load(open(tp)).get(args.workload)
                if ent:
                    traffic = ent.get("dram_bytes")
                    pipes = {k: ent[k] for k in ("fma_pipe_frac", "alu_pipe_frac", "issue_active_frac",
                                                 "sass_instr_per_candidate", "kernel_us", "source") if k in ent}
            except Exception:
                traffic, pipes = None, None
        line = {
            "metric": METRIC, "value": N * nt * args.steps / (tot_ms * 1e-3), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": tot_ms / args.steps,
            "time_to_optimum_ms": host_tot / args.steps, "host_ms_per_step": host_tot / args.steps,
            "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded profile tables, workloads/instances)",
            "config": {**_config(d, N, world, exchange if world > 1 else None),
                       **({"exchange_probe": probe} if probe else {})},
            "result": {"index": res.index, "latency_key": res.latency_key, "latency_s": res.latency,
                       "throughput_req_s": res.throughput, "units": res.units,
                       "feasible_count": res.feasible_count},
            "roofline": {"bound": "alu", "achieved": achieved / 1e9, "peak": peak / 1e9, "unit": "Gcandidates/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "kernel": {"k_search_u": "k_search_u (uniform-register search; after k_uprep: option "
                                                  "terms + constant-bank tables)",
                                    "k_search": "k_search (fused option terms + search)"}[alp.last_path],
                         "kernel_ms": kern_max / len(kern_ms), "pipes_ncu": pipes,
                         "peak_def": f"{sm_count} SMs x 128 issue lanes/clk x {f_max / 1e6:.0f} MHz / 1 instr per candidate"},
            "e2e": {"value": N * nt * len(e2e_ms) / (e2e_tot * 1e-3), "unit": UNIT,
                    "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(P.ctypes.sizeof(P._Result)),
                    "ms_per_step": e2e_tot / len(e2e_ms),
                    "cold_ms": cold_ms, "cold_h2d_bytes": int(cold_h2d),
                    "includes": "alp_build from host arrays (pinned H2D) + search + D2H result + alp_destroy; "
                                "cold = first build after alp_plan_cache_clear (adds host planning + plan upload)"},
            "gpu_launches": launches,
            "clocks": cs,
            "env": {"device": torch.cuda.get_device_name(dev), "sm_count": sm_count,
                    "cuda": torch.version.cuda, "torch": torch.__version__, "host_cores": os.cpu_count(),
                    "search_kernel": alp.last_path},
        }
        if world == 1 and not args.no_cpu_baseline:
            v, cores, sample, _dt, full = oracle_rate(d, seconds=args.cpu_seconds)
            line["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample}
            if full is not None and nt == 1:
                # the sample was the whole space: the timed GPU result vs the oracle's, bit for bit
                line["cpu_baseline"]["parity"] = bool(
                    full.found == res.found and full.count == res.feasible_count
                    and (not full.found or (full.index == res.index and full.latency_key == res.latency_key)))
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", default="C4")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--exchange", choices=["auto", "nccl", "peer"], default="auto",
                    help="N>1 cross-GPU reduction: NCCL all-gather + finalize kernel, the fused peer exchange, or "
                         "auto = both probed on this box (same result required), the faster one timed")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
