"""The fused peer exchange (alp_search_peer, SURVEY.md §8(a) A6 inside the search kernel): every
rank's last block finalizes its shard, stores (key, count, result) rows into every rank's exchange
buffer and reduces them after acquiring all ranks' flags.  Checked against the oracle (O2 on C4,
brute force on the small cases): several logical ranks sharing one GPU inside one process (one
host thread per rank), and two processes sharing buffers by CUDA IPC handles over gloo."""
from __future__ import annotations

import json
import os
import socket
import subprocess
import sys
import threading

import numpy as np
import pytest

import oracle
from oracle import dp
from workloads import generate

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _expect(I, lam, B, name):
    if name == "C4":
        tab = oracle.option_table(I, lam)
        f, v, i, c = dp.search(tab["tau"], tab["u"], B)
        return f, v, i, c
    o = oracle.search(I, lam, B)
    return o.found, o.latency_key, o.index, o.count


def _check(r, exp, I, lam, B):
    f, v, i, c = exp
    assert r.found == f and r.feasible_count == c
    if f:
        assert r.index == i
        assert np.float32(r.latency_key).view(np.uint32) == np.float32(v).view(np.uint32)
        p = oracle.predict(I, lam, oracle.decode(I, r.index), B)
        assert r.latency == pytest.approx(p["latency"], rel=1e-6)
        assert r.throughput == pytest.approx(p["throughput"], rel=1e-6)


def test_peer_bytes_layout():
    """Host-side sizes of the exchange buffer (no device needed): 512-byte header + two slots of
    world x n rows of (key, count, alp_result)."""
    import ctypes

    import paper_2604_15186_b200 as P
    row = 16 + ctypes.sizeof(P._Result)
    assert P.PeerBuffer.nbytes(1, 1) == 512 + 2 * row
    assert P.PeerBuffer.nbytes(8, 16) == 512 + 2 * 16 * 8 * row
    assert P.PeerBuffer.nbytes(0, 4) == 0 and P.PeerBuffer.nbytes(3, 0) == 0


@pytest.mark.gpu
@pytest.mark.parametrize("name,world", [("hand", 1), ("hand", 3), ("C1", 2), ("C4", 1), ("C4", 2), ("C4", 8)])
def test_peer_exchange_logical_ranks(name, world):
    """`world` ranks on one GPU in one process (a thread per rank, own handle, workspace, stream and
    exchange buffer; one of them takes the uniform-register kernel, the others the fused k_search):
    three exchanges in a row (both row slots) with 1 and 3 targets, every rank's result equal to
    the oracle's."""
    import torch

    import paper_2604_15186_b200 as P
    d = generate.load(name)
    I = oracle.from_json(d)
    B = d["budget_units"]
    lam = d["targets"][0]
    sets = [[lam], [lam, 2.0 * lam, 40.0 * lam], [0.5 * lam]]
    alps = [P.Alp.from_instance(d) for _ in range(world)]
    bufs = [P.PeerBuffer.alloc(3, world) for _ in range(world)]
    ptrs = [b.ptr for b in bufs]
    ws = [torch.zeros(a.workspace_bytes(3), dtype=torch.uint8, device="cuda") for a in alps]
    streams = [torch.cuda.Stream() for _ in range(world)]
    try:
        for targets in sets:
            out, err = [None] * world, []

            def run(r):
                try:
                    torch.cuda.set_device(0)
                    lo, hi = alps[r].shard_range(B, r, world)
                    out[r] = alps[r].search_peer(targets, B, lo, hi, r, ptrs, streams[r].cuda_stream,
                                                 ws[r].data_ptr())
                except Exception as e:  # pragma: no cover - reported below
                    err.append(e)
            th = [threading.Thread(target=run, args=(r,)) for r in range(world)]
            for t in th:
                t.start()
            for t in th:
                t.join(timeout=120)
            assert not err, err
            for lam_t, *rs in zip(targets, *out):
                exp = _expect(I, lam_t, B, name)
                for r in rs:
                    _check(r, exp, I, lam_t, B)
    finally:
        for b in bufs:
            b.close()


@pytest.mark.gpu
def test_peer_exchange_partial_range_matches_shard():
    """A one-rank exchange over a partial item range equals alp_search_shard + alp_finalize over the
    same range (the local finalize inside the kernel is K3's)."""
    import torch

    import paper_2604_15186_b200 as P
    d = generate.load("C4")
    alp = P.Alp.from_instance(d)
    B = d["budget_units"]
    lam = [d["targets"][0], 3.0 * d["targets"][0]]
    buf = P.PeerBuffer.alloc(2, 1)
    keys = torch.empty(2, dtype=torch.int64, device="cuda")
    cnts = torch.empty(2, dtype=torch.int64, device="cuda")
    try:
        for r in range(8):
            lo, hi = alp.shard_range(B, r, 8)
            a = alp.search_peer(lam, B, lo, hi, 0, [buf.ptr])
            alp.search_shard(lam, B, lo, hi, keys.data_ptr(), cnts.data_ptr())
            b = alp.finalize(lam, B, keys.data_ptr(), cnts.data_ptr())
            assert [(x.found, x.index, x.feasible_count, x.latency) for x in a] == \
                   [(x.found, x.index, x.feasible_count, x.latency) for x in b]
    finally:
        buf.close()


def _torchrun(script, nproc, args, env=None, timeout=300):
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr=127.0.0.1", f"--master-port={port}", script, *args]
    return subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, cwd=ROOT,
                          env={**os.environ, **(env or {})})


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["C4", "hand"])
def test_peer_exchange_two_processes_ipc(name):
    """Two processes (both on GPU 0 of a one-GPU box, their kernels time-sliced) share exchange
    buffers by CUDA IPC handles sent over a gloo group and run three peer exchanges; both ranks
    return the oracle's result."""
    p = _torchrun("tests/peer_worker.py", 2, [name])
    assert p.returncode == 0, p.stderr[-3000:]
    out = json.loads([x for x in p.stdout.splitlines() if x.startswith("{")][-1])
    assert out["world"] == 2
    d = generate.load(name)
    I = oracle.from_json(d)
    B = d["budget_units"]
    for targets, res in zip(out["targets"], out["results"]):
        for lam, (found, idx, cnt, key, lat, thr) in zip(targets, res):
            f, v, i, c = _expect(I, lam, B, name)
            assert (found, cnt) == (f, c)
            if f:
                assert idx == i and np.float32(key) == np.float32(v)
                p_ = oracle.predict(I, lam, oracle.decode(I, idx), B)
                assert lat == pytest.approx(p_["latency"], rel=1e-6)
                assert thr == pytest.approx(p_["throughput"], rel=1e-6)


@pytest.mark.gpu
def test_peer_exchange_timeout_reports_error():
    """A rank whose peers never arrive gives up after ALP_PEER_TIMEOUT_MS with ALP_EINTERNAL."""
    code = ("import paper_2604_15186_b200 as P\n"
            "from workloads import generate\n"
            "d = generate.load('hand')\n"
            "a = P.Alp.from_instance(d)\n"
            "bufs = [P.PeerBuffer.alloc(1, 2) for _ in range(2)]\n"
            "lo, hi = a.shard_range(d['budget_units'], 0, 2)\n"
            "try:\n"
            "    a.search_peer(d['targets'][:1], d['budget_units'], lo, hi, 0, [b.ptr for b in bufs])\n"
            "    print('NO ERROR')\n"
            "except P.AlpError as e:\n"
            "    print('STATUS', e.status, e)\n")
    p = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=120, cwd=ROOT,
                       env={**os.environ, "ALP_PEER_TIMEOUT_MS": "300", "PYTHONPATH": ROOT})
    assert "STATUS 3" in p.stdout and "timed out" in p.stdout, p.stdout + p.stderr[-2000:]
