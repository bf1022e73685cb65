"""Where does the C4 step time go?  Host enqueue cost of each library call vs device time.

  host_shard_us   wall time of alp.search_shard (H2D of the targets + K1 + K2 enqueue, no sync)
  host_fin_us     wall time of alp.finalize (K3 + D2H enqueue + stream sync)
  step_us         device time e0 -> e1 around the whole step (as bench.py times it)
  gpu_only_us     the same step with the GPU kept busy by a spin kernel while the host enqueues,
                  timed from the end of the spin kernel: the step's pure device time
  k2_us           alp.last_kernel_ms (K2 launch, CUDA events inside the library)

Usage: python tools/step_breakdown.py [--workload C4] [--reps 50]
"""
import argparse
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import paper_2604_15186_b200 as P
    from workloads import generate

    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="C4")
    ap.add_argument("--reps", type=int, default=50)
    args = ap.parse_args()
    d = generate.load(args.workload)
    B = int(d["budget_units"])
    targets = list(d["targets"])
    alp = P.Alp.from_instance(d)
    lo, hi = alp.shard_range(B, 0, 1)
    st = torch.cuda.Stream()
    keys = torch.empty(len(targets), dtype=torch.int64, device="cuda")
    counts = torch.empty(len(targets), dtype=torch.int64, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    rec = {k: [] for k in ("host_shard_us", "host_fin_us", "step_us", "gpu_only_us", "k2_us")}
    for rep in range(args.reps + 3):
        for spin in (False, True):
            with torch.cuda.stream(st):
                flush.zero_()
            torch.cuda.synchronize()
            with torch.cuda.stream(st):
                ev[0].record(st)
                if spin:
                    torch.cuda._sleep(2_000_000)  # ~1 ms at 1.9 GHz: the host enqueues meanwhile
                ev[1].record(st)
                t0 = time.perf_counter()
                alp.search_shard(targets, B, lo, hi, keys.data_ptr(), counts.data_ptr(), st.cuda_stream)
                t1 = time.perf_counter()
                alp.finalize(targets, B, keys.data_ptr(), counts.data_ptr(), st.cuda_stream)
                t2 = time.perf_counter()
                ev[2].record(st)
            torch.cuda.synchronize()
            if rep < 3:
                continue
            if spin:
                rec["gpu_only_us"].append(1e3 * ev[1].elapsed_time(ev[2]))
            else:
                rec["step_us"].append(1e3 * ev[0].elapsed_time(ev[2]))
                rec["host_shard_us"].append(1e6 * (t1 - t0))
                rec["host_fin_us"].append(1e6 * (t2 - t1))
                rec["k2_us"].append(1e3 * alp.last_kernel_ms)
    out = {k: round(statistics.median(v), 2) for k, v in rec.items()}
    out["workload"] = args.workload
    print(json.dumps(out))


if __name__ == "__main__":
    main()
