"""The one-pass budget-indexed search (alp_levels.cu):
one target, many budgets, every candidate evaluated once.  Each budget's winner and count against
the oracle (O2 on C4/C3, brute force on the small cases), and against the per-budget passes
(ALP_NO_LEVELS) in a child process."""
from __future__ import annotations

import json
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle
from oracle import dp
from workloads import generate

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _check(I, lam, budgets, res, brute=False):
    tab = oracle.option_table(I, lam)
    for B, r in zip(budgets, res):
        if brute:
            o = oracle.search(I, lam, B)
            f, v, i, c = o.found, o.latency_key, o.index, o.count
        else:
            f, v, i, c = dp.search(tab["tau"], tab["u"], min(B, 10**5))
        assert (r.found, r.feasible_count) == (f, c), B
        if f:
            assert r.index == i, B
            assert np.float32(r.latency_key).view(np.uint32) == np.float32(v).view(np.uint32), B
            p = oracle.predict(I, lam, oracle.decode(I, r.index), B)
            assert r.latency == pytest.approx(p["latency"], rel=1e-6)
            assert r.throughput == pytest.approx(p["throughput"], rel=1e-6)


@pytest.fixture(scope="module")
def P():
    import paper_2604_15186_b200 as P
    return P


def test_c4_every_gpu_count(P):
    """C4 on 0..64 whole GPUs (F = 2): 65 budgets in one pass, every winner and count vs O2."""
    d = generate.load("C4")
    I = oracle.from_json(d)
    alp = P.Alp.from_instance(d)
    lam = d["targets"][0]
    budgets = [2 * g for g in range(65)]
    res = alp.search_queries([lam] * len(budgets), budgets)
    assert alp.last_launches == 4  # K1, the one-pass search, the per-budget finish, K3
    _check(I, lam, budgets, res)


@pytest.mark.parametrize("name", ["hand", "C1", "C2"])
def test_small_vs_bruteforce(P, name):
    d = generate.load(name)
    I = oracle.from_json(d)
    alp = P.Alp.from_instance(d)
    B = d["budget_units"]
    budgets = sorted({0, 1, 2, 3, B // 3, B // 2, B - 1, B, B + 5, 3 * B})
    for lam in (d["targets"][0], 3.0 * d["targets"][0]):
        res = alp.search_queries([lam] * len(budgets), budgets[::-1])  # any order, duplicates allowed
        _check(I, lam, budgets[::-1], res, brute=True)


def test_c3_budgets_vs_dp(P):
    d = generate.load("C3")
    I = oracle.from_json(d)
    alp = P.Alp.from_instance(d)
    lam = d["targets"][0]
    budgets = [0, 8, 16, 40, 64, 100, 127, 128, 128, 500]
    _check(I, lam, budgets, alp.search_queries([lam] * len(budgets), budgets))


@pytest.mark.parametrize("seed", range(10))
def test_random_instances_vs_bruteforce(P, seed):
    rng = np.random.default_rng(seed)
    M = int(rng.integers(2, 5))
    d = generate.random_instance(900 + seed, M=M, F=4, S=[1, 2, 4], T=[1, 2], R=[1, 2, 3], budget=24,
                                 min_units=bool(seed % 2))
    I = oracle.from_json(d)
    alp = P.Alp.from_instance(d)
    budgets = list(range(0, 41, 3))
    for lam in (0.05, 0.3, 1.0):
        _check(I, lam, budgets, alp.search_queries([lam] * len(budgets), budgets), brute=True)


def test_matches_per_budget_passes(P):
    """The same sweep through the per-budget passes (ALP_NO_LEVELS=1, child process) gives the same
    results bit for bit."""
    d = generate.load("C4")
    lam = d["targets"][0]
    budgets = [2 * g for g in range(0, 65, 4)]
    alp = P.Alp.from_instance(d)
    res = alp.search_queries([lam] * len(budgets), budgets)
    code = ("import json, paper_2604_15186_b200 as P\nfrom workloads import generate\n"
            "d = generate.load('C4')\na = P.Alp.from_instance(d)\n"
            f"r = a.search_queries([{lam!r}] * {len(budgets)}, {budgets!r})\n"
            "print(json.dumps([[x.found, x.index, x.feasible_count, x.latency, x.throughput, x.units] for x in r]))\n")
    p = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300, cwd=ROOT,
                       env={**os.environ, "ALP_NO_LEVELS": "1", "PYTHONPATH": ROOT})
    assert p.returncode == 0, p.stderr[-2000:]
    ref = json.loads(p.stdout.strip().splitlines()[-1])
    assert [[x.found, x.index, x.feasible_count, x.latency, x.throughput, x.units] for x in res] == ref
