"""Parity of the CUDA path (through the C ABI) with the CPU oracle.  Needs a B200 (-m gpu).

Bar (BASELINE.json north star): chosen index and feasible count bit-exact; latency_key (the
canonical binary32 objective) bit-exact; FP64 latency / throughput within 1e-6 relative (they are
expected to be bit-identical: same IEEE operations in the same order).
"""
from __future__ import annotations

import itertools
import json

import numpy as np
import pytest

import oracle
from oracle import dp
from workloads import generate

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import paper_2604_15186_b200 as P
    return P


def _same(g, o_found, o_key, o_idx, o_cnt, tag=""):
    assert g.found == o_found, tag
    assert g.feasible_count == o_cnt, tag
    if o_found:
        assert g.index == o_idx, tag
        assert np.float32(g.latency_key).view(np.uint32) == np.float32(o_key).view(np.uint32), tag


def _check_winner(P, alp, I, lam, B, g):
    """FP64 Eq. 1 / Eq. 2 of the winner vs the oracle's prediction (rel 1e-6; expected exact)."""
    if not g.found:
        return
    ks = oracle.decode(I, g.index)
    p = oracle.predict(I, lam, ks, B)
    assert p["feasible"] and p["units"] == g.units
    assert g.latency == pytest.approx(p["latency"], rel=1e-6)
    assert g.throughput == pytest.approx(p["throughput"], rel=1e-6)
    assert p["latency_key"] == g.latency_key
    grid = [oracle.option_grid(I, k) for k in ks]
    assert [x[0] for x in grid] == g.share_units and [x[1] for x in grid] == g.tp and [x[2] for x in grid] == g.replicas


# ----------------------------------------------------------------------------- option table
@pytest.mark.parametrize("name", ["hand", "C1", "C2", "C3", "C4"])
def test_option_table_bitexact(P, name):
    d = generate.load(name)
    I = oracle.from_json(d)
    alp = P.Alp.from_instance(d)
    for lam in d["targets"] + [d["targets"][0] * 3.7, d["targets"][0] * 0.01]:
        g = alp.option_table(lam, I.K)
        o = oracle.option_table(I, lam)
        assert np.array_equal(g["tau"].view(np.uint32), o["tau"].view(np.uint32))
        assert np.array_equal(g["b"].view(np.uint64), o["b"].view(np.uint64))
        assert np.array_equal(g["u"], o["u"])
        fin = o["ok"]
        assert np.array_equal(g["term"][fin].view(np.uint64), o["term"][fin].view(np.uint64))


def test_option_table_edge_cases(P):
    # x exactly at r_0, at an interior r_i and at T; x below r_0; b exactly lambda; f = 1/F; d = 3.
    d = {"M": 2, "F": 4, "share_units": [1, 2, 4], "tp": [1, 2], "replicas": [1, 2, 3], "n": [2.0, 3.0],
         "p": [1.0, 1.5], "min_units": None, "budget_units": 40, "percentile": "mean",
         "profiles": [[{"rate": [0.5, 1.0, 2.0, 4.0], "lat": {k: [0.1, 0.2, 0.5, 1.1] for k in oracle.PCT_KEYS},
                        "tmax": 4.0},
                       {"rate": [0.25, 3.0], "lat": {k: [0.05, 0.3] for k in oracle.PCT_KEYS}, "tmax": 5.0}]] * 2}
    I = oracle.from_json(d)
    alp = P.Alp.from_instance(d)
    for lam in [0.0625, 0.125, 0.25, 0.5, 1.0 / 3.0, 0.7, 1.5, 2.0]:
        g = alp.option_table(lam, I.K)
        o = oracle.option_table(I, lam)
        assert np.array_equal(g["tau"].view(np.uint32), o["tau"].view(np.uint32)), lam
        assert np.array_equal(g["b"].view(np.uint64), o["b"].view(np.uint64)), lam


# ----------------------------------------------------------------------------- hand case
def test_hand_case_all_rows(P):
    with open("tests/golden/hand_case.json") as f:
        g = json.load(f)["searches"]
    from fractions import Fraction
    d = generate.load("hand")
    I = oracle.from_json(d)
    alp = P.Alp.from_instance(d)
    for lam_s, B, found, idx, _kg, _kv, Lw, Tw, units, feas in g["rows"]:
        lam = float(Fraction(lam_s))
        r = alp.search(lam, B)
        assert r.found == found and r.feasible_count == feas
        if found:
            assert r.index == idx and r.units == units
            assert r.latency == pytest.approx(float(Fraction(Lw)), rel=1e-12)
            assert r.throughput == float(Fraction(Tw))
            _check_winner(P, alp, I, lam, B, r)


# ----------------------------------------------------------------------------- percentile P
def test_percentile_hand_case(P):
    # PAPER.md:356 "the percentile P": each row of the golden percentile table (App. A terms x the
    # column's factors, exact-rational winners) through the C ABI with that column selected
    with open("tests/golden/hand_case.json") as f:
        g = json.load(f)["percentile_searches"]
    from fractions import Fraction
    d = generate.load("hand")
    for pct, lam_s, B, idx, _kg, _kv, Lw, Tw, units, feas in g["rows"]:
        I = oracle.from_json(d, pct)
        alp = P.Alp.from_instance(d, pct)
        lam = float(Fraction(lam_s))
        r = alp.search(lam, B)
        assert (r.found, r.index, r.feasible_count, r.units) == (True, idx, feas, units), (pct, B)
        assert r.latency == pytest.approx(float(Fraction(Lw)), rel=1e-12)
        assert r.throughput == float(Fraction(Tw))
        _check_winner(P, alp, I, lam, B, r)
        alp.close()


@pytest.mark.parametrize("pct", ["p50", "p90", "p99"])
def test_percentile_option_tables_bitexact(P, pct):
    # the stock C4 columns (mean x {0.8, 1.9, 3.5}) and a per-(LLM, tp) skewed column
    for d in (generate.load("C4"), generate.skew_percentile(generate.load("C4"), pct, seed=11)):
        I = oracle.from_json(d, pct)
        alp = P.Alp.from_instance(d, pct)
        for lam in (d["targets"][0], d["lambda_star"]):
            g = alp.option_table(lam, I.K)
            o = oracle.option_table(I, lam)
            assert np.array_equal(g["tau"].view(np.uint32), o["tau"].view(np.uint32)), (pct, lam)
            assert np.array_equal(g["term"][o["ok"]].view(np.uint64), o["term"][o["ok"]].view(np.uint64))
        alp.close()


@pytest.mark.slow
@pytest.mark.parametrize("pct", ["p90", "p99"])
def test_percentile_c4_vs_bruteforce(P, pct):
    # C4 with a skewed tail column: the optimum moves away from the mean's; GPU (the column selected
    # in alp_desc.pct) == full O1 brute force on every host core == O2
    import os
    d = generate.skew_percentile(generate.load("C4"), pct, seed=5)
    I = oracle.from_json(d, pct)
    lam = d["targets"][0]
    alp = P.Alp.from_instance(d, pct)
    r = alp.search(lam, I.budget)
    o = oracle.search(I, lam, I.budget, threads=os.cpu_count() or 8)
    _same(r, o.found, o.latency_key, o.index, o.count, pct)
    tab = oracle.option_table(I, lam)
    f, v, idx, cnt = dp.search(tab["tau"], tab["u"], I.budget)
    _same(r, f, v, idx, cnt, pct)
    _check_winner(P, alp, I, lam, I.budget, r)
    mean = P.Alp.from_instance(d, "mean").search(lam, I.budget)
    assert mean.index != r.index  # the selected column decides the optimum


# ----------------------------------------------------------------------------- measured profiles (R2)
def test_measured_profiles_hand_case_gpu(P):
    # SPEC.md:204 "measured profiles always win": the golden hand rows with two measured curves
    with open("tests/golden/hand_case.json") as f:
        g = json.load(f)["measured_profiles"]
    from fractions import Fraction
    d = generate.with_measured(generate.load("hand"), g["curves"])
    I = oracle.from_json(d)
    alp = P.Alp.from_instance(d)
    tab = alp.option_table(1.0, I.K)
    for m, k, term, b, u in g["terms_lambda_1"]["rows"]:
        assert tab["term"][m, k] == pytest.approx(float(Fraction(term)), rel=4e-16) and tab["u"][m, k] == u
        assert tab["b"][m, k] == float(Fraction(b))
    for lam_s, B, idx, _kg, _kv, Lw, Tw, units, feas in g["searches"]["rows"]:
        r = alp.search(float(Fraction(lam_s)), B)
        assert (r.found, r.index, r.feasible_count, r.units) == (True, idx, feas, units), B
        assert r.latency == pytest.approx(float(Fraction(Lw)), rel=1e-12) and r.throughput == float(Fraction(Tw))
        _check_winner(P, alp, I, 1.0, B, r)


@pytest.mark.parametrize("name,seed", [("C2", 1), ("C3", 2), ("C4", 3)])
def test_measured_profiles_option_tables_and_search(P, name, seed):
    # a seeded subset of (LLM, tp, share) measured (perturbed scaled curves): option tables bit-exact
    # against the oracle on every launch path's kernel, and the search against O2
    d = generate.random_measured(generate.load(name), seed)
    assert d["measured"]
    I = oracle.from_json(d)
    alp = P.Alp.from_instance(d)
    for lam in (d["targets"][0], d["targets"][0] * 2.5):
        g = alp.option_table(lam, I.K)
        o = oracle.option_table(I, lam)
        assert np.array_equal(g["tau"].view(np.uint32), o["tau"].view(np.uint32)), lam
        assert np.array_equal(g["b"].view(np.uint64), o["b"].view(np.uint64)), lam
        assert np.array_equal(g["term"][o["ok"]].view(np.uint64), o["term"][o["ok"]].view(np.uint64))
        r = alp.search(lam, I.budget)
        f, v, idx, cnt = dp.search(o["tau"], o["u"], I.budget)
        _same(r, f, v, idx, cnt, (name, lam))
        _check_winner(P, alp, I, lam, I.budget, r)
    # a measured curve equal to the scaled one changes nothing (powers-of-two shares)
    F = d["F"]
    which = [(m, ti, si) for m in range(d["M"]) for ti in range(len(d["tp"]))
             for si, s in enumerate(d["share_units"]) if (F // s) * s == F and (F // s) & (F // s - 1) == 0]
    base = generate.load(name)
    a0 = P.Alp.from_instance(base).search(base["targets"][0], I.budget)
    a1 = P.Alp.from_instance(generate.scaled_measured(base, which)).search(base["targets"][0], I.budget)
    assert (a0.index, a0.feasible_count, a0.latency_key, a0.latency) == (a1.index, a1.feasible_count, a1.latency_key,
                                                                        a1.latency)


@pytest.mark.slow
def test_measured_profiles_c4_vs_bruteforce(P):
    import os
    d = generate.random_measured(generate.load("C4"), 7)
    I = oracle.from_json(d)
    lam = d["targets"][0]
    r = P.Alp.from_instance(d).search(lam, I.budget)
    o = oracle.search(I, lam, I.budget, threads=os.cpu_count() or 8)
    _same(r, o.found, o.latency_key, o.index, o.count)


# ----------------------------------------------------------------------------- configs
@pytest.mark.parametrize("name", ["C1", "C2"])
def test_full_bruteforce_small(P, name):
    d = generate.load(name)
    I = oracle.from_json(d)
    alp = P.Alp.from_instance(d)
    for lam in (d["targets"][0], d["targets"][0] * 2, d["lambda_star"]):
        for B in (I.budget, I.budget // 2, I.budget * 4):
            r = alp.search(lam, B)
            o = oracle.search(I, lam, B)
            _same(r, o.found, o.latency_key, o.index, o.count, (name, lam, B))
            _check_winner(P, alp, I, lam, B, r)


@pytest.mark.parametrize("name", ["C3", "C4"])
def test_full_size_vs_dp(P, name):
    d = generate.load(name)
    I = oracle.from_json(d)
    alp = P.Alp.from_instance(d)
    lam = d["targets"][0]
    for B in (I.budget, I.budget // 2 + 3):
        r = alp.search(lam, B)
        tab = oracle.option_table(I, lam)
        f, v, idx, cnt = dp.search(tab["tau"], tab["u"], B)
        _same(r, f, v, idx, cnt, (name, B))
        assert r.candidates == I.N
        _check_winner(P, alp, I, lam, B, r)
        # the winner, recomputed one by one from the profiles
        ok, l32, _ = oracle.candidate(I, lam, r.index, B)
        assert ok and l32 == r.latency_key


@pytest.mark.slow
@pytest.mark.parametrize("name", ["C3", "C4"])
def test_full_size_vs_bruteforce(P, name):
    # SURVEY.md §8(c) parity contract: full C3 / C4 against O1 (literal brute force over every
    # canonical index) on all host cores (C3: 6.9e10 candidates, ~17 s on 16 cores)
    import os
    d = generate.load(name)
    I = oracle.from_json(d)
    lam = d["targets"][0]
    alp = P.Alp.from_instance(d)
    r = alp.search(lam, I.budget)
    o = oracle.search(I, lam, I.budget, threads=os.cpu_count() or 8)
    _same(r, o.found, o.latency_key, o.index, o.count, name)
    assert r.candidates == I.N
    _check_winner(P, alp, I, lam, I.budget, r)


def test_uniform_register_graph_replay_interleaved(P):
    """The uniform-register prep/copy/search sequence is replayed as a cached CUDA graph whose
    kernel arguments are rewritten when they change: two handles of the same shape (one graph)
    interleaved, target and budget changing on every call, each result against the DP oracle."""
    d = generate.load("C4")
    I = oracle.from_json(d)
    A, B = P.Alp.from_instance(d), P.Alp.from_instance(d)
    lam0 = d["targets"][0]
    tabs = {}
    for i, (h, lam, bud) in enumerate([(A, lam0, I.budget), (B, lam0 * 0.5, I.budget), (A, lam0 * 0.5, I.budget - 7),
                                        (B, lam0, I.budget - 7), (A, lam0, I.budget), (A, lam0 * 1.7, I.budget),
                                        (B, lam0 * 1.7, I.budget - 7)]):
        r = h.search(lam, bud)
        assert h.last_path == "k_search_u" and h.last_kernel_ms > 0
        if lam not in tabs:
            tabs[lam] = oracle.option_table(I, lam)
        f, v, idx, cnt = dp.search(tabs[lam]["tau"], tabs[lam]["u"], bud)
        _same(r, f, v, idx, cnt, (i, lam, bud))


def test_uniform_register_without_graph_matches(P):
    """ALP_U_NOGRAPH=1 (read once per process, so in a child process) launches the prep, the
    constant-bank copy and the search as separate stream calls: same results as the graph replay."""
    import os
    import subprocess
    import sys
    code = ("import json, paper_2604_15186_b200 as P\n"
            "from workloads import generate\n"
            "out = []\n"
            "for name in ('hand', 'C4'):\n"
            "    d = generate.load(name); a = P.Alp.from_instance(d)\n"
            "    for f in (1.0, 0.4):\n"
            "        r = a.search(d['targets'][0] * f, d['budget_units'])\n"
            "        out.append([a.last_path, r.index, r.feasible_count, r.latency_key])\n"
            "print(json.dumps(out))\n")
    env = dict(os.environ, ALP_U_NOGRAPH="1")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = subprocess.run([sys.executable, "-c", code], env=env, cwd=root, capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stderr[-2000:]
    child = json.loads(res.stdout.strip().splitlines()[-1])
    mine = []
    for name in ("hand", "C4"):
        d = generate.load(name)
        a = P.Alp.from_instance(d)
        for f in (1.0, 0.4):
            r = a.search(d["targets"][0] * f, d["budget_units"])
            mine.append([a.last_path, r.index, r.feasible_count, r.latency_key])
    assert all(x[0] == "k_search_u" for x in mine)
    assert child == mine


def test_c4_window_bruteforce(P):
    # exhaustive O1 around the optimum: no candidate in a 2e7-wide canonical window beats it
    d = generate.load("C4")
    I = oracle.from_json(d)
    alp = P.Alp.from_instance(d)
    lam = d["targets"][0]
    r = alp.search(lam, I.budget)
    lo = max(0, r.index - 10_000_000)
    o = oracle.search(I, lam, I.budget, lo=lo, hi=min(I.N, r.index + 10_000_000), threads=8)
    assert o.found and o.index == r.index and o.latency_key == r.latency_key


def test_c5_target_batch(P):
    d = generate.load("C5")
    I = oracle.from_json(d)
    alp = P.Alp.from_instance(d)
    targets = d["targets"]
    res = alp.search_batch(targets, I.budget)
    assert len(res) == 256
    prev_cnt = None
    for j in range(256):  # every target against O2
        tab = oracle.option_table(I, targets[j])
        f, v, idx, cnt = dp.search(tab["tau"], tab["u"], I.budget)
        _same(res[j], f, v, idx, cnt, j)
    for j in (0, 128, 255):
        _check_winner(P, alp, I, targets[j], I.budget, res[j])
    for j in range(256):  # Pareto invariants over the sweep (exact count monotonicity)
        if prev_cnt is not None:
            assert res[j].feasible_count <= prev_cnt
        prev_cnt = res[j].feasible_count
    assert res[255].found and res[255].feasible_count >= 1


# ----------------------------------------------------------------------------- fuzzing
@pytest.mark.parametrize("seed", range(24))
def test_random_instances_vs_bruteforce(P, seed):
    rng = np.random.default_rng(7000 + seed)
    M = int(rng.integers(1, 6))
    S = sorted(set(int(x) for x in rng.integers(1, 5, size=int(rng.integers(1, 4)))))
    T = [1, 2, 4, 8][: int(rng.integers(1, 5))]
    R = list(range(1, int(rng.integers(2, 6))))
    K = len(S) * len(T) * len(R)
    while K ** M > 3_000_000:
        M -= 1
    budget = int(rng.integers(0, 40))
    d = generate.random_instance(seed, M=M, F=4, S=S, T=T, R=R, budget=budget, min_units=bool(seed % 4 == 1))
    I = oracle.from_json(d)
    alp = P.Alp.from_instance(d)
    for lam in (0.02, 0.2, 1.1):
        r = alp.search(lam, budget)
        o = oracle.search(I, lam, budget, threads=4)
        _same(r, o.found, o.latency_key, o.index, o.count, (seed, lam))
        _check_winner(P, alp, I, lam, budget, r)


@pytest.mark.parametrize("seed", range(8))
def test_injected_terms_ties_and_exact_sums(P, seed):
    # dyadic terms (multiples of 2^-10, sums < 2^14): every binary32 sum is exact; heavy ties.
    rng = np.random.default_rng(seed)
    M = int(rng.integers(2, 5))
    K = int(rng.integers(2, 12))
    tau = (rng.integers(1, 9, size=(M, K)) * 128 / 1024.0).astype(np.float32)
    tau[rng.random((M, K)) < 0.15] = np.inf
    u = rng.integers(0, 6, size=(M, K)).astype(np.int32)
    B = int(rng.integers(0, 6 * M))
    alp = P.Alp.from_terms(tau, u)
    r = alp.search(1.0, B)
    best, bidx, cnt = None, None, 0
    for i, ks in enumerate(itertools.product(range(K), repeat=M)):
        if sum(u[m, k] for m, k in enumerate(ks)) > B or not all(np.isfinite(tau[m, k]) for m, k in enumerate(ks)):
            continue
        cnt += 1
        v = sum(int(tau[m, k] * 1024) for m, k in enumerate(ks))
        if best is None or v < best:
            best, bidx = v, i
    assert r.feasible_count == cnt
    assert r.found == (cnt > 0)
    if cnt:
        assert r.index == bidx and r.latency_key == best / 1024.0


def test_subulp_terms_match_dp(P):
    rng = np.random.default_rng(3)
    M, K = 4, 20
    tau = (np.float32(1.0) + rng.integers(0, 4, size=(M, K)).astype(np.float32) * np.float32(2.0 ** -23))
    tau = tau.astype(np.float32)
    u = rng.integers(1, 5, size=(M, K)).astype(np.int32)
    for B in (4, 7, 11, 16, 80):
        alp = P.Alp.from_terms(tau, u)
        r = alp.search(1.0, B)
        f, v, idx, cnt = dp.search(tau, u, B)
        _same(r, f, v, idx, cnt, B)


# ----------------------------------------------------------------------------- sharding / edges
def test_partition_independence(P):
    import torch
    d = generate.load("C4")
    I = oracle.from_json(d)
    alp = P.Alp.from_instance(d)
    lam = [d["targets"][0]]
    ref = alp.search(lam[0], I.budget)
    tab = oracle.option_table(I, lam[0])
    o2 = dp.search(tab["tau"], tab["u"], I.budget)
    for world in (2, 3, 5, 8):
        keys = torch.empty((world, 1), dtype=torch.int64, device="cuda")
        counts = torch.empty((world, 1), dtype=torch.int64, device="cuda")
        for rank in range(world):
            lo, hi = alp.shard_range(I.budget, rank, world)
            alp.search_shard(lam, I.budget, lo, hi, keys[rank].data_ptr(), counts[rank].data_ptr())
            torch.cuda.synchronize()
        k = keys.min(dim=0).values.contiguous()
        c = counts.sum(dim=0).contiguous()
        r = alp.finalize(lam, I.budget, k.data_ptr(), c.data_ptr())[0]
        assert (r.index, r.feasible_count, r.latency_key) == (ref.index, ref.feasible_count, ref.latency_key)
        _same(r, *o2, world)  # the reduced shards against the oracle directly
        _check_winner(P, alp, I, lam[0], I.budget, r)


def test_finalize_gathered_matches_allreduce(P):
    """The one-all-gather exchange: per-rank int64[2n] (keys, counts) rows, reduced inside K3."""
    import torch
    d = generate.load("C4")
    I = oracle.from_json(d)
    alp = P.Alp.from_instance(d)
    lam = [d["targets"][0], d["targets"][0] * 2.0, d["targets"][0] * 40.0]  # incl. an infeasible target
    ref = alp.search_batch(lam, I.budget)
    n = len(lam)
    for world in (1, 3, 8):
        gathered = torch.empty(world * 2 * n, dtype=torch.int64, device="cuda")
        for rank in range(world):
            lo, hi = alp.shard_range(I.budget, rank, world)
            row = gathered[rank * 2 * n:(rank + 1) * 2 * n]
            alp.search_shard(lam, I.budget, lo, hi, row.data_ptr(), row.data_ptr() + 8 * n)
            torch.cuda.synchronize()
        res = alp.finalize_gathered(lam, I.budget, gathered.data_ptr(), world)
        for r, e, l in zip(res, ref, lam):
            assert (r.found, r.index, r.feasible_count, r.latency_key, r.units) == (e.found, e.index, e.feasible_count,
                                                                                   e.latency_key, e.units)
            tab = oracle.option_table(I, l)
            _same(r, *dp.search(tab["tau"], tab["u"], I.budget), (world, l))  # against the oracle directly
            _check_winner(P, alp, I, l, I.budget, r)


def test_infeasible_and_zero_budget(P):
    d = generate.load("C1")
    I = oracle.from_json(d)
    alp = P.Alp.from_instance(d)
    r = alp.search(1e6, 16)  # no candidate meets the target: the max-T_w fallback
    fb = oracle.max_throughput(I, 16)
    assert not r.found and r.feasible_count == 0 and r.fallback and r.index == fb["index"]
    assert r.throughput == fb["throughput"] and r.units == fb["units"] and r.latency == float("inf")
    r = alp.search(d["targets"][0], 0)  # nothing fits a zero budget: no fallback either
    assert not r.found and r.feasible_count == 0 and not r.fallback and r.index == -1


def _fallback_closed_form(I, B):
    """Separable construction of the max-T_w candidate (pinned against the brute-force definition in
    tests/test_oracle.py::test_max_throughput_separable_closed_form), for spaces too large to enumerate."""
    tab = oracle.option_table(I, 1.0)
    ok = [[oracle.floor_ok(I, m, k) for k in range(I.K)] for m in range(I.M)]

    def minu(m, v):
        c = [int(tab["u"][m][k]) for k in range(I.K) if ok[m][k] and tab["b"][m][k] >= v]
        return min(c) if c else None
    best = None
    for v in sorted(set(tab["b"].ravel().tolist())):
        mus = [minu(m, v) for m in range(I.M)]
        if all(x is not None for x in mus) and sum(mus) <= B:
            best = v
    if best is None:
        return None
    idx, used = 0, 0
    for m in range(I.M):
        rest = sum(minu(j, best) for j in range(m + 1, I.M))
        k = next(k for k in range(I.K) if ok[m][k] and tab["b"][m][k] >= best and used + int(tab["u"][m][k]) + rest <= B)
        used += int(tab["u"][m][k])
        idx = idx * I.K + k
    return {"index": idx, "throughput": best, "units": used}


def test_infeasible_fallback_hand_case(P):
    """The App. A hand case at lambda = 5 (infeasible for every budget): B = 8 -> index 45, T_w 4,
    8 units; B = 7 -> 9 (T_w 2, 4 units); B = 3 -> 0; B = 1 -> no candidate fits (no fallback)."""
    d = generate.load("hand")
    alp = P.Alp.from_instance(d)
    for B, (idx, tw, units) in {8: (45, 4.0, 8), 7: (9, 2.0, 4), 3: (0, 1.0, 2)}.items():
        r = alp.search(5.0, B)
        assert not r.found and r.fallback and (r.index, r.throughput, r.units) == (idx, tw, units), B
        assert r.feasible_count == 0 and r.latency == float("inf")
    r = alp.search(5.0, 1)
    assert not r.found and not r.fallback and r.index == -1
    # through the batch and the budget-sweep paths too
    res = alp.search_batch([5.0, 1.0], 8)
    assert res[0].fallback and res[0].index == 45 and res[1].found and not res[1].fallback
    res = alp.search_queries([5.0] * 4, [8, 7, 3, 1])
    assert [(x.fallback, x.index) for x in res] == [(True, 45), (True, 9), (True, 0), (False, -1)]


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4"])
def test_infeasible_fallback_vs_oracle(P, name):
    d = generate.load(name)
    I = oracle.from_json(d)
    alp = P.Alp.from_instance(d)
    lam = 50.0 * d["lambda_star"]
    for B in (d["budget_units"], d["budget_units"] // 3, 5):
        r = alp.search(lam, B)
        fb = oracle.max_throughput(I, B) if I.N <= 70000 else _fallback_closed_form(I, B)
        assert not r.found and r.feasible_count == 0
        if fb is None:
            assert not r.fallback
            continue
        assert r.fallback and (r.index, r.throughput, r.units) == (fb["index"], fb["throughput"], fb["units"]), B
        grid = [oracle.option_grid(I, k) for k in oracle.decode(I, r.index)]
        assert [g[0] for g in grid] == r.share_units and [g[1] for g in grid] == r.tp and [g[2] for g in grid] == r.replicas
    # the sharded path (shard search + finalize) reports the same fallback
    import torch
    keys = torch.empty(1, dtype=torch.int64, device="cuda")
    cnts = torch.empty(1, dtype=torch.int64, device="cuda")
    B = d["budget_units"]
    lo, hi = alp.shard_range(B, 1, 3)
    alp.search_shard([lam], B, lo, hi, keys.data_ptr(), cnts.data_ptr())
    r = alp.finalize([lam], B, keys.data_ptr(), cnts.data_ptr())[0]
    assert r.fallback and r.index == alp.search(lam, B).index


def test_validation_errors(P):
    d = generate.load("C1")
    bad = json.loads(json.dumps(d))
    bad["n"][1] = -1.0
    with pytest.raises(P.AlpError, match="n\\[1\\]"):
        P.Alp.from_instance(bad)
    bad = json.loads(json.dumps(d))
    bad["profiles"][0][1]["rate"][3] = bad["profiles"][0][1]["rate"][2]
    with pytest.raises(P.AlpError, match="strictly increasing"):
        P.Alp.from_instance(bad)
    alp = P.Alp.from_instance(d)
    with pytest.raises(P.AlpError, match="targets"):
        alp.search(-1.0, 16)


def test_predict_matches_oracle(P):
    d = generate.load("C3")
    I = oracle.from_json(d)
    alp = P.Alp.from_instance(d)
    rng = np.random.default_rng(0)
    opts = rng.integers(0, I.K, size=(500, I.M))
    lam = d["targets"][0]
    g = alp.predict(opts, lam, I.budget)
    for i in range(len(opts)):
        o = oracle.predict(I, lam, list(opts[i]), I.budget)
        assert g["feasible"][i] == o["feasible"] and g["units"][i] == o["units"]
        assert g["throughput"][i] == o["throughput"]
        if np.isfinite(o["latency"]):
            assert g["latency"][i] == o["latency"]


def test_decode_roundtrip(P):
    d = generate.load("C4")
    I = oracle.from_json(d)
    alp = P.Alp.from_instance(d)
    for idx in [0, 1, I.N - 1, 123456789, 9725594165]:
        assert alp.decode(idx) == [oracle.option_grid(I, k) for k in oracle.decode(I, idx)]


def test_plan_cache_shared_and_cleared(P):
    d = generate.load("C4")
    lam = d["targets"][0]
    a1 = P.Alp.from_instance(d)
    r1 = a1.search(lam, d["budget_units"])
    a2 = P.Alp.from_instance(d)  # plan cache hit: only the profile tables are uploaded
    assert a2.h2d_bytes < a1.h2d_bytes or a1.h2d_bytes < 200_000
    P.plan_cache_clear()
    a3 = P.Alp.from_instance(d)  # rebuilt plan
    for a in (a2, a3):
        r = a.search(lam, d["budget_units"])
        assert (r.index, r.feasible_count, r.latency_key) == (r1.index, r1.feasible_count, r1.latency_key)
    a1.close()
    r = a2.search(lam, d["budget_units"])  # a2 keeps its (now uncached) plan alive
    assert r.index == r1.index


# ----------------------------------------------------------------------------- budget queries / NEXT-1
def test_search_queries_budget_sweep(P):
    d = generate.load("C4")
    I = oracle.from_json(d)
    alp = P.Alp.from_instance(d)
    lam = d["targets"][0]
    budgets = [0, 7, 16, 33, 64, 96, 128, 200, 10**6]
    res = alp.search_queries([lam] * len(budgets), budgets)
    tab = oracle.option_table(I, lam)
    for B, r in zip(budgets, res):
        f, v, idx, cnt = dp.search(tab["tau"], tab["u"], min(B, 10**4))
        _same(r, f, v, idx, cnt, B)
    # mixed targets and budgets in one pass
    qs = [(lam, 128), (lam * 2, 64), (lam * 0.5, 100), (d["lambda_star"], 128)]
    res = alp.search_queries([q[0] for q in qs], [q[1] for q in qs])
    for (l, B), r in zip(qs, res):
        t2 = oracle.option_table(I, l)
        f, v, idx, cnt = dp.search(t2["tau"], t2["u"], B)
        _same(r, f, v, idx, cnt, (l, B))


@pytest.mark.parametrize("names,gpus,F", [(("C1", "C1"), 8, 4), (("hand", "C4"), 16, 2), (("C2", "C3"), 16, 8)])
def test_egalitarian_vs_oracle(P, names, gpus, F):
    from oracle import multi
    ds = [generate.load(n) for n in names]
    alps = [P.Alp.from_instance(d) for d in ds]
    targets = [d["targets"][0] for d in ds]
    split, res, mn, sm = P.schedule_egalitarian(alps, targets, gpus, F)
    lat = [multi.best_latencies(oracle.from_json(d), t, gpus, F) for d, t in zip(ds, targets)]
    osplit, omn, osm = multi.egalitarian(lat, gpus)
    assert split == osplit and mn == omn and sm == osm
    for d, t, g, r in zip(ds, targets, split, res):
        I = oracle.from_json(d)
        tab = oracle.option_table(I, t)
        f, v, idx, cnt = dp.search(tab["tau"], tab["u"], g * F)
        _same(r, f, v, idx, cnt, (d["name"], g))


# ----------------------------------------------------------------------------- fused vs classic launch paths
@pytest.mark.parametrize("name", ["hand", "C1", "C2", "C4"])
def test_fused_and_classic_paths_agree(P, name, monkeypatch):
    """<= 8 targets run as one fused kernel (terms + search + finalize); ALP_NO_FUSED forces the
    K1 + K2 + K3 path.  Both must give the same, oracle-identical results."""
    d = generate.load(name)
    I = oracle.from_json(d)
    lam0 = d["targets"][0]
    lams = [lam0 * f for f in (0.5, 1.0, 1.7, 3.0, 40.0)]  # includes an infeasible target
    alp = P.Alp.from_instance(d)
    fused = alp.search_batch(lams, I.budget)
    assert alp.last_launches == (2 if alp.last_path == "k_search_u" else 1)  # fused or uniform-register pair
    monkeypatch.setenv("ALP_NO_FUSED", "1")
    classic = alp.search_batch(lams, I.budget)
    assert alp.last_launches == 3
    monkeypatch.delenv("ALP_NO_FUSED")
    for lam, a, b in zip(lams, fused, classic):
        assert (a.found, a.index, a.feasible_count, a.units) == (b.found, b.index, b.feasible_count, b.units)
        assert np.float32(a.latency_key).view(np.uint32) == np.float32(b.latency_key).view(np.uint32)
        assert (a.latency == b.latency) or (not a.found)
        assert a.throughput == b.throughput or not a.found
        assert (a.share_units, a.tp, a.replicas) == (b.share_units, b.tp, b.replicas)
        if name != "C4":
            o = oracle.search(I, lam, I.budget, threads=4)
            _same(a, o.found, o.latency_key, o.index, o.count, (name, lam))
    # fused scratch returns to its rest state: repeating the search gives the same answer
    again = alp.search_batch(lams, I.budget)
    assert [(x.index, x.feasible_count) for x in again] == [(x.index, x.feasible_count) for x in fused]


def test_fused_empty_shard_and_uneven_world(P):
    """A rank with an empty item range still writes (KeyNone, 0) and the option terms its finalize
    needs; more ranks than items is legal."""
    import torch
    d = generate.load("C1")
    I = oracle.from_json(d)
    alp = P.Alp.from_instance(d)
    lam = [d["targets"][0]]
    ref = alp.search(lam[0], I.budget)
    items = alp.num_items(I.budget)
    world = items + 3
    keys = torch.empty((world, 1), dtype=torch.int64, device="cuda")
    counts = torch.empty((world, 1), dtype=torch.int64, device="cuda")
    for rank in range(world):
        lo, hi = alp.shard_range(I.budget, rank, world)
        alp.search_shard(lam, I.budget, lo, hi, keys[rank].data_ptr(), counts[rank].data_ptr())
        torch.cuda.synchronize()
        if hi == lo:
            assert int(keys[rank, 0]) == 0x7FFFFFFFFFFFFFFF and int(counts[rank, 0]) == 0
    k = keys.min(dim=0).values.contiguous()
    c = counts.sum(dim=0).contiguous()
    r = alp.finalize(lam, I.budget, k.data_ptr(), c.data_ptr())[0]
    assert (r.index, r.feasible_count, r.latency_key) == (ref.index, ref.feasible_count, ref.latency_key)


def test_cross_stream_calls_are_ordered(P):
    """An async shard search on a caller stream followed at once by a search on the handle's own
    stream: the second call waits for the first (they share the handle's scratch)."""
    import torch
    d = generate.load("C4")
    B = d["budget_units"]
    lam = d["targets"][0]
    alp = P.Alp.from_instance(d)
    lo, hi = alp.shard_range(B, 0, 1)
    keys = torch.empty(1, dtype=torch.int64, device="cuda")
    counts = torch.empty(1, dtype=torch.int64, device="cuda")
    st = torch.cuda.Stream()
    alp.search_shard([lam], B, lo, hi, keys.data_ptr(), counts.data_ptr(), st.cuda_stream)
    st.synchronize()
    ref_key, ref_cnt = int(keys[0]), int(counts[0])
    ref_half = alp.search(lam * 0.5, B)
    for _ in range(3):
        keys.fill_(0)
        counts.fill_(0)
        torch.cuda.synchronize()
        alp.search_shard([lam], B, lo, hi, keys.data_ptr(), counts.data_ptr(), st.cuda_stream)  # async
        r = alp.search(lam * 0.5, B)  # handle stream, issued while the shard search may still run
        st.synchronize()
        assert (int(keys[0]), int(counts[0])) == (ref_key, ref_cnt)
        assert (r.index, r.feasible_count, r.latency_key) == (ref_half.index, ref_half.feasible_count,
                                                              ref_half.latency_key)


@pytest.mark.parametrize("rows", [8, 16])
@pytest.mark.parametrize("name", ["hand", "C1", "C2"])
def test_rows_per_lane_variants_agree(P, name, rows, monkeypatch):
    """The tuning variants (8 / 16 rows per lane; the default is 12) give identical results."""
    d = generate.load(name)
    I = oracle.from_json(d)
    lam = d["targets"][0]
    ref = P.Alp.from_instance(d).search(lam, I.budget)
    monkeypatch.setenv("ALP_ROWS_PER_LANE", str(rows))
    r = P.Alp.from_instance(d).search(lam, I.budget)
    assert (r.found, r.index, r.feasible_count, r.latency_key) == (ref.found, ref.index, ref.feasible_count,
                                                                    ref.latency_key)


@pytest.mark.parametrize("M,S,T,R,budget", [(10, [1, 2], [1], [1, 2], 14), (12, [1], [1, 2], [1, 2], 20),
                                             (16, [1, 2], [1], [1], 22), (9, [1, 2, 4], [1], [1, 2], 17),
                                             (16, [1], [1], [1, 2, 3], 30)])
def test_many_llms_vs_bruteforce(P, M, S, T, R, budget):
    """Many LLMs (up to ALP_MAX_M = 16): several prefix LLMs above the sort group, the prefix-chunk
    table and multi-digit chunk decode, against the brute-force oracle over the whole space."""
    d = generate.random_instance(900 + M, M=M, F=4, S=S, T=T, R=R, budget=budget)
    I = oracle.from_json(d)
    alp = P.Alp.from_instance(d)
    for lam in (0.05, 0.3):
        r = alp.search(lam, budget)
        o = oracle.search(I, lam, budget, threads=8)
        _same(r, o.found, o.latency_key, o.index, o.count, (M, lam))
        _check_winner(P, alp, I, lam, budget, r)


def test_max_options_per_llm_vs_bruteforce(P):
    """K = 1024 options per LLM (ALP_MAX_K): a one-LLM sort group, b rows split into chunks."""
    S = [1, 2, 3, 4]
    T = [1, 2, 4, 8]
    R = list(range(1, 65))
    d = generate.random_instance(4242, M=3, F=4, S=S, T=T, R=R, budget=600)
    I = oracle.from_json(d)
    assert I.K == 1024
    alp = P.Alp.from_instance(d)
    for lam in (0.05, 0.5):
        r = alp.search(lam, 600)
        o = oracle.search(I, lam, 600, threads=16)
        _same(r, o.found, o.latency_key, o.index, o.count, lam)
        _check_winner(P, alp, I, lam, 600, r)


def test_search_distributed_single_process(P):
    """dist.search_distributed without a process group (world 1) on torch's default stream: the
    gather-based exchange and the finalize must be ordered with the search."""
    from paper_2604_15186_b200.dist import search_distributed
    d = generate.load("C4")
    alp = P.Alp.from_instance(d)
    lam = [d["targets"][0], d["targets"][0] * 3.0]
    ref = alp.search_batch(lam, d["budget_units"])
    for _ in range(3):
        res = search_distributed(alp, lam, d["budget_units"])
        assert [(r.index, r.feasible_count) for r in res] == [(e.index, e.feasible_count) for e in ref]


@pytest.mark.parametrize("world", [1, 2])
def test_nccl_search_distributed(P, world):
    """Row A6 end to end over a real NCCL process group (torch.distributed.run, 127.0.0.1): sharded
    search, ONE NCCL all-gather of the (key, count) pairs, the finalize kernel's MIN/SUM -- checked
    against O2 on C4.  world 2 puts both ranks on one GPU when only one is visible; NCCL may refuse
    that (duplicate GPU), which skips the case."""
    import os
    import socket
    import subprocess
    import sys
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr=127.0.0.1", f"--master-port={port}", "tests/nccl_worker.py", "C4"]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=300)
    if p.returncode != 0 and world > 1 and ("uplicate GPU" in p.stderr + p.stdout or "ncclInvalidUsage" in p.stderr + p.stdout):
        pytest.skip("NCCL refuses two ranks on one GPU")
    assert p.returncode == 0, p.stderr[-3000:]
    line = [x for x in p.stdout.splitlines() if x.startswith("{")][-1]
    out = json.loads(line)
    assert out["world"] == world and out["backend"] == "nccl"
    d = generate.load("C4")
    I = oracle.from_json(d)
    targets = [d["targets"][0], 2.0 * d["targets"][0], 40.0 * d["targets"][0]]
    for (found, idx, cnt, key, lat), lam in zip(out["results"], targets):
        tab = oracle.option_table(I, lam)
        f, v, oi, oc = dp.search(tab["tau"], tab["u"], I.budget)
        assert (found, cnt) == (f, oc)
        if f:
            assert idx == oi and np.float32(key) == np.float32(v)
            assert lat == pytest.approx(oracle.predict(I, lam, oracle.decode(I, idx))["latency"], rel=1e-6)


def test_fused_many_b_chunks_eight_targets(P):
    """One LLM with K = 1024 options (b columns split in several chunks) and 8 targets: the fused
    launch's work counters cover targets x chunks phases."""
    S = [1, 2, 3, 4]
    T = [1, 2, 4, 8]
    R = list(range(1, 65))
    d = generate.random_instance(77, M=1, F=4, S=S, T=T, R=R, budget=300)
    I = oracle.from_json(d)
    alp = P.Alp.from_instance(d)
    lams = [0.02 * (i + 1) for i in range(8)]
    res = alp.search_batch(lams, 300)
    assert alp.last_launches == 1
    for lam, r in zip(lams, res):
        o = oracle.search(I, lam, 300)
        _same(r, o.found, o.latency_key, o.index, o.count, lam)


@pytest.mark.parametrize("name", ["hand", "C4"])
def test_uniform_register_path_matches_fused(P, name, monkeypatch):
    """Single-target searches with short b rows run the uniform-register pair (k_uprep: option
    terms + constant-bank tables; k_search_u: one warp per block, warp-uniform masked rows from the
    constant bank, mixed groups from shared memory); ALP_NO_UR forces the fused kernel."""
    d = generate.load(name)
    I = oracle.from_json(d)
    alp = P.Alp.from_instance(d)
    for lam in (d["targets"][0], d["targets"][0] * 0.3, d["targets"][0] * 2.5):
        u = alp.search(lam, I.budget)
        assert alp.last_launches == 2
        monkeypatch.setenv("ALP_NO_UR", "1")
        f = alp.search(lam, I.budget)
        assert alp.last_launches == 1
        monkeypatch.delenv("ALP_NO_UR")
        assert (u.found, u.index, u.feasible_count, u.units) == (f.found, f.index, f.feasible_count, f.units)
        assert u.latency_key == f.latency_key and (u.latency == f.latency or not u.found)
        if name == "hand":
            o = oracle.search(I, lam, I.budget)
            _same(u, o.found, o.latency_key, o.index, o.count, lam)


@pytest.mark.parametrize("seed", range(10))
def test_uniform_register_path_random_vs_bruteforce(P, seed):
    """Random instances whose b rows fit the uniform-register path (<= 34 options per LLM)."""
    rng = np.random.default_rng(5000 + seed)
    M = int(rng.integers(2, 6))
    S = sorted(set(int(x) for x in rng.integers(1, 5, size=int(rng.integers(1, 3)))))
    T = [1, 2, 4][: int(rng.integers(1, 4))]
    R = list(range(1, int(rng.integers(2, 4))))
    K = len(S) * len(T) * len(R)
    while K ** M > 2_000_000:
        M -= 1
    budget = int(rng.integers(2, 40))
    d = generate.random_instance(5000 + seed, M=M, F=4, S=S, T=T, R=R, budget=budget, min_units=bool(seed % 3 == 1))
    I = oracle.from_json(d)
    alp = P.Alp.from_instance(d)
    for lam in (0.02, 0.3, 1.5):
        r = alp.search(lam, budget)
        o = oracle.search(I, lam, budget, threads=4)
        _same(r, o.found, o.latency_key, o.index, o.count, (seed, lam))
        _check_winner(P, alp, I, lam, budget, r)


@pytest.mark.parametrize("seed", range(12))
def test_uniform_register_long_rows_vs_bruteforce(P, seed, monkeypatch):
    """Long b rows (K > 34 options per LLM) on the uniform-register path: 64-column b chunks with
    per-chunk luts and de-duplicated masked rows, a ragged last chunk, unit sums clamped at R + 1,
    budgets from 0 to above the total -- against brute force (O1) and the k_search path."""
    rng = np.random.default_rng(9100 + seed)
    M = int(rng.integers(1, 4))
    S = sorted(set(int(x) for x in rng.integers(1, 9, size=int(rng.integers(2, 6)))))
    T = [1, 2, 4, 8][: int(rng.integers(1, 5))]
    R = list(range(1, int(rng.integers(4, 17))))
    K = len(S) * len(T) * len(R)
    while K <= 34:
        R.append(R[-1] + 1)
        K = len(S) * len(T) * len(R)
    while K ** M > 4_000_000:
        M -= 1
    budgets = [0, int(rng.integers(1, 20)), int(rng.integers(20, 200)), 10_000]
    d = generate.random_instance(9100 + seed, M=M, F=8, S=S, T=T, R=R, budget=budgets[1],
                                 min_units=bool(seed % 3 == 2))
    I = oracle.from_json(d)
    alp = P.Alp.from_instance(d)
    for lam in (0.05, 0.6):
        for B in budgets:
            r = alp.search(lam, B)
            assert alp.last_path == "k_search_u", (K, M)
            o = oracle.search(I, lam, B, threads=8)
            _same(r, o.found, o.latency_key, o.index, o.count, (seed, K, M, lam, B))
            _check_winner(P, alp, I, lam, B, r)
            monkeypatch.setenv("ALP_NO_UR", "1")
            f = alp.search(lam, B)
            monkeypatch.delenv("ALP_NO_UR")
            assert (f.index, f.feasible_count, f.latency_key) == (r.index, r.feasible_count, r.latency_key)


def test_uniform_register_path_concurrent_streams(P):
    """Two handles with different problems search on two streams at once through the shared
    constant-bank tables: the ordering event keeps them from overwriting each other's tables."""
    import torch
    dA, dB = generate.load("C4"), generate.load("hand")
    A, B = P.Alp.from_instance(dA), P.Alp.from_instance(dB)
    la, lb = [dA["targets"][0]], [dB["targets"][0]]
    refA, refB = A.search(la[0], dA["budget_units"]), B.search(lb[0], dB["budget_units"])
    sA, sB = torch.cuda.Stream(), torch.cuda.Stream()
    kA = torch.empty(2, dtype=torch.int64, device="cuda")
    kB = torch.empty(2, dtype=torch.int64, device="cuda")
    for _ in range(3):
        loA, hiA = A.shard_range(dA["budget_units"], 0, 1)
        loB, hiB = B.shard_range(dB["budget_units"], 0, 1)
        A.search_shard(la, dA["budget_units"], loA, hiA, kA.data_ptr(), kA.data_ptr() + 8, sA.cuda_stream)
        B.search_shard(lb, dB["budget_units"], loB, hiB, kB.data_ptr(), kB.data_ptr() + 8, sB.cuda_stream)
        assert A.last_path == "k_search_u" and B.last_path == "k_search_u"
        rA = A.finalize(la, dA["budget_units"], kA.data_ptr(), kA.data_ptr() + 8, sA.cuda_stream)[0]
        rB = B.finalize(lb, dB["budget_units"], kB.data_ptr(), kB.data_ptr() + 8, sB.cuda_stream)[0]
        assert (rA.index, rA.feasible_count, rA.latency_key) == (refA.index, refA.feasible_count, refA.latency_key)
        assert (rB.index, rB.feasible_count, rB.latency_key) == (refB.index, refB.feasible_count, refB.latency_key)


def _wait_event(ev, timeout_s):
    """Poll a CUDA event from the host; True if it completed within timeout_s."""
    import time
    t0 = time.monotonic()
    while not ev.query():
        if time.monotonic() - t0 > timeout_s:
            return False
        time.sleep(0.0005)
    return True


def test_workspace_searches_overlap_across_streams(P):
    """SURVEY.md §8(b) / SPEC.md:303 ("predictions are pure and may run concurrently"): two searches
    on ONE handle with distinct caller workspaces on two streams are not ordered against each other.
    Stream A is held by a ~1 s spin kernel before its search; search B on stream B completes while A
    is still held (it would wait the whole second if the library serialised it behind A), then both
    results match the oracle (O2).  Control: with the handle's own scratch, B does wait for A."""
    import torch
    d = generate.load("C4")
    I = oracle.from_json(d)
    alp = P.Alp.from_instance(d)
    B_ = I.budget
    la, lb = [d["targets"][0]], [2.0 * d["targets"][0]]
    nbytes = alp.workspace_bytes(1)
    assert nbytes > 0
    wA = torch.zeros(nbytes, dtype=torch.uint8, device="cuda")
    wB = torch.zeros(nbytes, dtype=torch.uint8, device="cuda")
    sA, sB = torch.cuda.Stream(), torch.cuda.Stream()
    kA = torch.empty(2, dtype=torch.int64, device="cuda")
    kB = torch.empty(2, dtype=torch.int64, device="cuda")
    lo, hi = alp.shard_range(B_, 0, 1)
    rate = torch.cuda.get_device_properties(0).clock_rate * 1000  # kHz -> Hz
    for use_ws in (True, False):
        torch.cuda.synchronize()
        endA, endB = torch.cuda.Event(), torch.cuda.Event()
        with torch.cuda.stream(sA):
            torch.cuda._sleep(int(1.0 * rate))  # hold stream A for ~1 s
        alp.search_shard(la, B_, lo, hi, kA.data_ptr(), kA.data_ptr() + 8, sA.cuda_stream,
                         wA.data_ptr() if use_ws else None)
        endA.record(sA)
        alp.search_shard(lb, B_, lo, hi, kB.data_ptr(), kB.data_ptr() + 8, sB.cuda_stream,
                         wB.data_ptr() if use_ws else None)
        endB.record(sB)
        b_first = _wait_event(endB, 0.5)
        a_pending = not endA.query()
        torch.cuda.synchronize()
        if use_ws:
            assert b_first and a_pending, "search B was serialised behind search A"
            for lam, k, w in ((la, kA, wA), (lb, kB, wB)):
                r = alp.finalize(lam, B_, k.data_ptr(), k.data_ptr() + 8, None, w.data_ptr())[0]
                tab = oracle.option_table(I, lam[0])
                _same(r, *dp.search(tab["tau"], tab["u"], B_), lam)
                _check_winner(P, alp, I, lam[0], B_, r)
        else:
            assert not b_first, "control: the handle's own scratch orders B after A"
    # a workspace is reusable without clearing (its control section is zero after every call), for
    # any target count up to its size
    w8 = torch.zeros(alp.workspace_bytes(8), dtype=torch.uint8, device="cuda")
    k8 = torch.empty(16, dtype=torch.int64, device="cuda")
    for n in (1, 3, 8, 2):
        lams = [d["targets"][0] * (1 + 0.5 * j) for j in range(n)]
        alp.search_shard(lams, B_, lo, hi, k8.data_ptr(), k8.data_ptr() + 8 * n, None, w8.data_ptr())
        res = alp.finalize(lams, B_, k8.data_ptr(), k8.data_ptr() + 8 * n, None, w8.data_ptr())
        for r, lam in zip(res, lams):
            tab = oracle.option_table(I, lam)
            _same(r, *dp.search(tab["tau"], tab["u"], B_), (n, lam))
    assert bool((w8[:64] == 0).all())


def test_uniform_register_batch_groups_vs_oracle(P):
    """A 12-target batch runs as uniform-register groups of 8 + 4 (results zero-copy, one sync);
    every target against the brute-force oracle, including infeasible ones."""
    d = generate.load("hand")
    I = oracle.from_json(d)
    alp = P.Alp.from_instance(d)
    lams = [0.125 * (i + 1) for i in range(10)] + [4.0, 5.0]
    res = alp.search_batch(lams, I.budget)
    assert alp.last_path == "k_search_u" and alp.last_launches == 4
    for lam, r in zip(lams, res):
        o = oracle.search(I, lam, I.budget)
        _same(r, o.found, o.latency_key, o.index, o.count, lam)
        _check_winner(P, alp, I, lam, I.budget, r)


@pytest.mark.parametrize("B", [0, 1, 9, 64, 255, 256, 10_000])
def test_c4_budgets_vs_dp(P, B):
    """The headline instance on the uniform-register path across budgets: empty (0), tiny, binding,
    at and above the total of the per-LLM maxima (the cap), against the DP oracle (O2)."""
    d = generate.load("C4")
    I = oracle.from_json(d)
    alp = P.Alp.from_instance(d)
    for lam in (d["targets"][0], d["targets"][0] * 3.9):
        r = alp.search(lam, B)
        assert alp.last_path == "k_search_u"
        tab = oracle.option_table(I, lam)
        f, v, idx, cnt = dp.search(tab["tau"], tab["u"], min(B, int(tab["u"].max(axis=1).sum())))
        _same(r, f, v, idx, cnt, (B, lam))
        if r.found:
            _check_winner(P, alp, I, lam, B, r)
