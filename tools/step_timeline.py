"""Device timeline of one search step (CUPTI via torch.profiler): every kernel / memcpy of the step
with its start offset and duration, so gaps between launches are visible.

    python tools/step_timeline.py [--workload C4] [--mode shard|search|peer]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from torch.profiler import profile, ProfilerActivity
    import paper_2604_15186_b200 as P
    from workloads import generate

    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="C4")
    ap.add_argument("--mode", default="shard")
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
    buf = P.PeerBuffer.alloc(len(targets), 1) if args.mode == "peer" else None

    def step():
        with torch.cuda.stream(st):
            if args.mode == "search":
                return alp.search_batch(targets, B)
            if args.mode == "peer":  # search + in-kernel exchange (one rank, the whole range)
                return alp.search_peer(targets, B, lo, hi, 0, [buf.ptr], st.cuda_stream)
            alp.search_shard(targets, B, lo, hi, keys.data_ptr(), counts.data_ptr(), st.cuda_stream)
            return alp.finalize(targets, B, keys.data_ptr(), counts.data_ptr(), st.cuda_stream)

    for _ in range(5):
        step()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        for _ in range(3):
            with torch.cuda.stream(st):
                flush.zero_()
            torch.cuda.synchronize()
            step()
            torch.cuda.synchronize()
    ev = [e for e in prof.events() if e.device_type.name == "CUDA"]
    ev.sort(key=lambda e: e.time_range.start)
    # last step: everything after the last flush kernel
    idx = max(i for i, e in enumerate(ev) if "fill" in e.name.lower() or "elementwise" in e.name.lower())
    step_ev = ev[idx + 1:]
    t0 = step_ev[0].time_range.start
    prev_end = t0
    for e in step_ev:
        s, en = e.time_range.start, e.time_range.end
        print(f"{s - t0:9.1f} us  +{s - prev_end:7.1f} gap  {en - s:8.1f} us  {e.name[:90]}")
        prev_end = en
    print(f"step span {step_ev[-1].time_range.end - t0:.1f} us")
    # host side of the same step: runtime API calls (CUPTI), same clock as the device events
    api = [e for e in prof.events() if e.device_type.name == "CPU" and e.name.startswith("cuda")
           and e.time_range.start >= step_ev[0].time_range.start - 200]
    api.sort(key=lambda e: e.time_range.start)
    for e in api[:40]:
        s, en = e.time_range.start, e.time_range.end
        print(f"  host {s - t0:9.1f} us  {en - s:7.1f} us  {e.name[:60]}")


if __name__ == "__main__":
    main()
