import os, sys, threading
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2604_15186_b200 as P
from workloads import generate
d = generate.load("hand")
alps = [P.Alp.from_instance(d) for _ in range(2)]
bufs = [P.PeerBuffer.alloc(1, 2) for _ in range(2)]
wss = [torch.zeros(a.workspace_bytes(1), dtype=torch.uint8, device="cuda") for a in alps]
sts = [torch.cuda.Stream() for _ in range(2)]
out = [None, None]
for r in range(2):
    print("rank", r, "range", alps[r].shard_range(d["budget_units"], r, 2))
def run(r, delay):
    import time
    time.sleep(delay)
    torch.cuda.set_device(0)
    lo, hi = alps[r].shard_range(d["budget_units"], r, 2)
    try:
        x = alps[r].search_peer(d["targets"][:1], d["budget_units"], lo, hi, r, [b.ptr for b in bufs], sts[r].cuda_stream, wss[r].data_ptr())[0]
        out[r] = (x.found, x.index, x.feasible_count, x.fallback)
    except Exception as e:
        out[r] = str(e)
order = [float(x) for x in sys.argv[1:3]] if len(sys.argv) > 2 else [0, 0]
th = [threading.Thread(target=run, args=(r, order[r])) for r in range(2)]
for t in th: t.start()
for t in th: t.join()
print(out)
