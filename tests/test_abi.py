"""Host-side checks that need no GPU: the C-ABI library loads and exports every symbol that
include/alp.h declares; the oracle library is independent of it; host logic (shard ranges,
cross-rank key reduction over gloo) is correct."""
from __future__ import annotations

import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "alp.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(alp_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_2604_15186_b200 import build
    lib = build.build()
    out = subprocess.check_output(["nm", "-D", "--defined-only", lib], text=True)
    exported = set(re.findall(r" T (alp_\w+)", out))
    missing = [s for s in _declared() if s not in exported]
    assert not missing, missing
    import paper_2604_15186_b200 as P
    L = P.lib()  # ctypes load succeeds without a GPU
    for s in _declared():
        assert hasattr(L, s)
    assert set(P.EXPORTS) == set(_declared())


def test_library_is_sm100a():
    from paper_2604_15186_b200 import build
    lib = build.build()
    out = subprocess.check_output(["/usr/local/cuda/bin/cuobjdump", "-lelf", lib], text=True)
    assert "sm_100a" in out
    sass = subprocess.check_output(["/usr/local/cuda/bin/cuobjdump", "-sass", lib], text=True)
    assert "FADD2" in sass and "FMNMX3" in sass  # the packed add / 3-input min inner loop


def test_no_shared_code_between_oracle_and_product():
    for root, _dirs, files in os.walk(os.path.join(ROOT, "paper_2604_15186_b200")):
        for f in files:
            if f.endswith((".py", ".cu", ".h", ".cpp")):
                txt = open(os.path.join(root, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt and "alp_oracle" not in txt, f
    for f in os.listdir(os.path.join(ROOT, "oracle")):
        if f.endswith((".py", ".c")):
            txt = open(os.path.join(ROOT, "oracle", f)).read()
            assert not re.search(r"^\s*(import|from)\s+paper_2604_15186_b200", txt, re.M), f
            assert "libscepsy_alp" not in txt, f


def test_cuda_missing_fails_loudly():
    import paper_2604_15186_b200 as P
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("GPU present")
    except Exception:
        pass
    from workloads import generate
    with pytest.raises(P.AlpError):
        P.Alp.from_instance(generate.load("hand"))


def _gloo_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2604_15186_b200.dist import reduce_keys
    # per-rank partial (key, count) pairs for 3 targets; key = bits(value) << 32 | segment
    import numpy as np
    vals = [np.float32(1.5 + rank), np.float32(2.0), np.float32(np.inf)]
    segs = [10 + rank, 100 - rank, 0]
    keys = []
    for v, s in zip(vals, segs):
        keys.append(0x7FFFFFFFFFFFFFFF if not np.isfinite(v) else (int(v.view(np.uint32)) << 32) | s)
    k = torch.tensor(keys, dtype=torch.int64)
    c = torch.tensor([rank + 1, 5, 0], dtype=torch.int64)
    pairs = torch.cat([k, c])
    reduce_keys(k, c)
    from paper_2604_15186_b200.dist import gather_pairs
    gathered = torch.empty(world * pairs.numel(), dtype=torch.int64)
    w = gather_pairs(pairs, gathered)
    q.put((rank, k.tolist(), c.tolist(), w, gathered.tolist(), pairs.tolist()))
    dist.destroy_process_group()


def test_gloo_two_rank_key_reduction():
    import multiprocessing as mp
    import numpy as np
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 1000
    ps = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    out = [q.get(timeout=120) for _ in ps]
    for p in ps:
        p.join(timeout=60)
    exp0 = (int(np.float32(1.5).view(np.uint32)) << 32) | 10       # lower value wins
    exp1 = (int(np.float32(2.0).view(np.uint32)) << 32) | 99       # equal values: lower segment wins
    for _rank, k, c, _w, _g, _p in out:
        assert k == [exp0, exp1, 0x7FFFFFFFFFFFFFFF]
        assert c == [3, 10, 0]
    # one all-gather: rank r's (keys, counts) land in row r; MIN / SUM over rows = the all-reduces
    own = {r: p for r, _k, _c, _w, _g, p in out}
    for _rank, k, c, w, g, _p in out:
        assert w == 2 and g == own[0] + own[1]
        rows = [g[0:6], g[6:12]]
        assert [min(rows[0][i], rows[1][i]) for i in range(3)] == k
        assert [rows[0][3 + i] + rows[1][3 + i] for i in range(3)] == c


def test_search_u_keeps_uniform_datapath():
    """ptxas keeps k_search_u's b operands in uniform registers only while nothing perturbs its
    analysis (a __syncwarp before the epilogue, an inlined exchange, a register cap each dropped it
    silently: DESIGN.md §5).  Guard on the built object: every variant for b rows of >= 12 options
    (NB4 >= 3: C4's 18, the 64-column chunks of C3) has FADD2 with a uniform-register operand and
    <= 88 registers (>= 23 one-warp blocks/SM; the full-row loop holds its b pairs in uniform
    registers and took C4's variant from 76 to 84); no variant spills.  The variants for rows of 2-10
    options (NB4 <= 2, e.g. the 8-option hand case) may lose it: their rows are short anyway."""
    import re
    import shutil
    import subprocess

    from paper_2604_15186_b200 import build
    build.build()
    obj = os.path.join(os.path.dirname(build.LIB), "alp_search_u.o")
    if not shutil.which("cuobjdump") or not os.path.exists(obj):
        pytest.skip("cuobjdump or the object file is missing")
    out = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
    funcs = {f.split("\n", 1)[0].strip(): f for f in re.split(r"\n\s*Function : ", out)[1:]}
    names = [n for n in funcs if "k_search_u" in n]
    assert len(names) >= 18
    for n in names:
        ins = [ln.split("*/", 1)[1] for ln in funcs[n].split("\n") if re.match(r"\s*/\*[0-9a-f]{4,}\*/", ln)]
        fadd2 = [i for i in ins if "FADD2" in i]
        nb4 = int(re.search(r"k_search_uILi(\d+)E", n).group(1))
        if fadd2 and nb4 >= 3:
            assert any(re.search(r"\bUR\d", i) for i in fadd2), n
        assert not any("STL" in i for i in ins), n
    ptx = open(obj + ".ptxas.txt").read()
    for m in re.finditer(r"Function properties for (\S*k_search_u\S*)\n.*\n.*Used (\d+) registers", ptx):
        if int(re.search(r"k_search_uILi(\d+)E", m.group(1)).group(1)) >= 3:
            assert int(m.group(2)) <= 88, m.group(1)


def test_collective_failure_maps_to_alp_enccl(monkeypatch):
    """A failing collective surfaces as AlpError(ALP_ENCCL) from the exchange helpers (§8(b) status
    5), not as a bare backend exception (one-rank gloo group on 127.0.0.1; the collective is made to
    fail)."""
    import socket

    import torch
    import torch.distributed as dist

    import paper_2604_15186_b200 as P
    from paper_2604_15186_b200 import dist as pdist
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    try:
        def boom(*a, **k):
            raise RuntimeError("simulated transport failure")
        monkeypatch.setattr(dist, "all_gather", boom)
        monkeypatch.setattr(dist, "get_world_size", lambda group=None: 2)
        monkeypatch.setattr(dist, "all_reduce", boom)
        pairs = torch.zeros(2, dtype=torch.int64)
        with pytest.raises(P.AlpError) as e:
            pdist.gather_pairs(pairs, torch.empty(4, dtype=torch.int64))
        assert e.value.status == P.ALP_ENCCL
        with pytest.raises(P.AlpError) as e:
            pdist.reduce_keys(torch.zeros(1, dtype=torch.int64), torch.zeros(1, dtype=torch.int64))
        assert e.value.status == P.ALP_ENCCL
    finally:
        monkeypatch.undo()
        dist.destroy_process_group()
