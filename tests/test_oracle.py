"""Pins for the CPU oracle (oracle/), run with -m "not gpu".

Every check here compares the oracle with something other than itself: values the paper / SPEC
print (tests/golden/spec_examples.json), the hand-derived exact two-LLM case (tests/golden/
hand_case.json), closed forms, invariants, an independent DP algorithm (O2) and
exact-integer brute force on tiny dyadic inputs.
"""
from __future__ import annotations

import itertools
import json
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle
from oracle import dp
from workloads import generate

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def _curve(rates, lats, tmax=None):
    return {"rate": list(rates), "lat": {k: list(lats) for k in ("mean", "p50", "p90", "p99")},
            "tmax": rates[-1] if tmax is None else tmax}


def _inst(llms, F=1, S=(1,), T=(1,), R=(1,), budget=10**6, min_units=None):
    """llms: list of dicts with n, p, curves (one per tp)."""
    return oracle.from_json({"M": len(llms), "F": F, "share_units": list(S), "tp": list(T), "replicas": list(R),
                             "n": [l["n"] for l in llms], "p": [l["p"] for l in llms],
                             "profiles": [l["curves"] for l in llms], "min_units": min_units,
                             "budget_units": budget, "percentile": "mean"})


# ----------------------------------------------------------------------------- SPEC examples
def test_lookup_spec_examples():
    g = _gold("spec_examples.json")
    for ex in g["lookup"]:
        assert oracle.lookup(ex["rates"], ex["lats"], ex["x"]) == ex["L"], ex["cite"]


def test_interior_bracket_hits_point_exactly():
    # R3: i = max{i : r_i <= x}, so x = r_{i+1} returns L_{i+1} exactly, and the last point holds.
    assert oracle.lookup([1.0, 3.0, 7.0], [0.1, 0.7, 2.9], 3.0) == 0.7
    assert oracle.lookup([1.0, 3.0, 7.0], [0.1, 0.7, 2.9], 7.0) == 2.9
    assert oracle.lookup([1.0, 3.0, 7.0], [0.1, 0.7, 2.9], 9.0) == 2.9  # (r_last, T] held flat
    # interpolation weight is (x - r_i) / (r_{i+1} - r_i) of the bracketing pair, not of the curve ends
    assert oracle.lookup([1.0, 3.0, 7.0], [1.0, 2.0, 10.0], 5.0) == 6.0


def test_infeasible_above_T():
    g = _gold("spec_examples.json")["infeasible_above_T"]
    I = _inst([{"n": 1.0, "p": 1.0, "curves": [_curve([1.0, g["T"]], [1.0, 2.0])]}])
    assert not oracle.option(I, g["T"] * g["factor"], 0, 0)["ok"]
    assert oracle.option(I, g["T"], 0, 0)["ok"]  # R4: rate = T is feasible


def test_fraction_scaling_spec():
    g = _gold("spec_examples.json")["fraction_scaling"]
    # F=2, S={1} -> f = 0.5; base profile L(4) = 1, T = 10; n = p = d = 1
    I = _inst([{"n": 1.0, "p": 1.0, "curves": [_curve([g["base_rate"], 8.0], [g["base_L"], 2.0], tmax=g["T"])]}],
              F=2, S=(1,))
    o = oracle.option(I, g["scaled_rate"], 0, 0)
    assert o["ok"]
    assert o["b"] == g["T_scaled"]            # T' = f T
    assert o["term"] == g["scaled_L"]         # L'(2) = L(2/f)/f = 2


def test_eq1_sum_spec():
    g = _gold("spec_examples.json")["eq1_sum"]
    A, B = g["A"], g["B"]
    I = _inst([{"n": A["n"], "p": A["p"], "curves": [_curve([10.0, 20.0], [A["L"], 5.0])]},
               {"n": B["n"], "p": B["p"], "curves": [_curve([10.0, 20.0], [B["L"], 5.0])]}])
    r = oracle.predict(I, 1.0, [0, 0])
    assert r["feasible"] and r["latency"] == g["total"]


def test_eq1_identity_and_eq2_identity():
    I = _inst([{"n": 1.0, "p": 1.0, "curves": [_curve([1.0, 5.0, 9.0], [0.25, 0.5, 4.0], tmax=9.0)]}])
    for lam in (0.5, 1.0, 3.0, 5.0, 7.0, 9.0):
        r = oracle.predict(I, lam, [0])
        assert r["latency"] == oracle.lookup([1.0, 5.0, 9.0], [0.25, 0.5, 4.0], lam)
        assert r["throughput"] == 9.0


def test_eq2_min_and_doubling_spec():
    g = _gold("spec_examples.json")["eq2_min"]
    I = _inst([{"n": g["A"]["n"], "p": 1.0, "curves": [_curve([1.0, g["A"]["T"]], [1.0, 2.0])]},
               {"n": g["B"]["n"], "p": 1.0, "curves": [_curve([1.0, g["B"]["T"]], [1.0, 2.0])]}], R=(1, 2))
    assert oracle.predict(I, 0.5, [0, 0])["throughput"] == g["Tw"]
    # doubling d of the unique bottleneck (B, term 4 < 5) doubles its term
    assert oracle.option(I, 0.5, 1, 1)["b"] == 2 * oracle.option(I, 0.5, 1, 0)["b"]
    assert oracle.predict(I, 0.5, [0, 1])["throughput"] == 5.0  # A becomes the bottleneck


def test_memory_floor_filters_option():
    # an option below the per-(LLM, tp) unit floor is infeasible.
    I = _inst([{"n": 1.0, "p": 1.0, "curves": [_curve([1.0, 8.0], [1.0, 2.0])]}], F=4, S=(1, 2, 4),
              min_units=[[2]])
    oks = [oracle.option(I, 0.1, 0, k)["ok"] for k in range(3)]
    assert oks == [False, True, True]


# ----------------------------------------------------------------------------- hand case (App. A)
def _F(s):
    return Fraction(s)


def test_hand_case_option_terms():
    g = _gold("hand_case.json")["option_terms_lambda_1"]
    I = oracle.from_json(generate.load("hand"))
    for row in g["rows"]:
        k, s, t, d = row[:4]
        assert oracle.option_grid(I, k) == (s, t, d)
        for m, (x, term, b, u) in enumerate([row[4:8], row[8:12]]):
            o = oracle.option(I, 1.0, m, k)
            assert o["ok"]
            assert o["u"] == u
            assert o["b"] == float(_F(b))
            assert o["term"] == pytest.approx(float(_F(term)), rel=4e-16, abs=0)


def test_hand_case_searches():
    g = _gold("hand_case.json")["searches"]
    I = oracle.from_json(generate.load("hand"))
    for lam_s, B, found, idx, kg, kv, Lw, Tw, units, feas in g["rows"]:
        lam = float(_F(lam_s))
        r = oracle.search(I, lam, B)
        assert r.found == found and r.count == feas, (lam_s, B)
        if not found:
            continue
        assert r.index == idx and oracle.decode(I, idx) == [kg, kv]
        p = oracle.predict(I, lam, [kg, kv], B)
        assert p["feasible"] and p["units"] == units
        assert p["throughput"] == float(_F(Tw))
        assert p["latency"] == pytest.approx(float(_F(Lw)), rel=1e-15)


def test_hand_case_fp_goldens():
    g = _gold("hand_case.json")["fp_goldens"]
    I = oracle.from_json(generate.load("hand"))
    for lam_s, B, key, lat in g["rows"]:
        lam = float(_F(lam_s))
        r = oracle.search(I, lam, B)
        assert np.float32(r.latency_key) == np.float32(key)
        assert oracle.predict(I, lam, oracle.decode(I, r.index), B)["latency"] == float(lat)


def _hand_pct_enumeration(pct):
    """Exact-rational winners of the hand case at a percentile column: App. A terms (golden) times the
    column's per-tp factor, brute force over the 64 candidates (lowest index on exact ties)."""
    from workloads.generate import HAND_PCT_FACTOR
    rows = _gold("hand_case.json")["option_terms_lambda_1"]["rows"]
    c = [Fraction(x).limit_denominator() for x in HAND_PCT_FACTOR[pct]]
    fac = [c[0] if r[2] == 1 else c[1] for r in rows]  # tp 1 -> tp index 0, tp 2 -> tp index 1
    G = [fac[k] * _F(r[5]) for k, r in enumerate(rows)]
    V = [fac[k] * _F(r[9]) for k, r in enumerate(rows)]
    out = {}
    for B in (8, 16, 3):
        best, cnt = None, 0
        for kg, kv in itertools.product(range(8), range(8)):
            if rows[kg][7] + rows[kv][11] <= B:
                cnt += 1
                L = G[kg] + V[kv]
                if best is None or L < best[0]:
                    best = (L, 8 * kg + kv)
        out[B] = (best[1], best[0], cnt)
    return G, V, out


@pytest.mark.parametrize("pct", ["mean", "p50", "p90", "p99"])
def test_hand_case_percentile_columns(pct):
    # the prediction takes "the percentile P at which latency should be evaluated".
    # The hand instance's percentile columns are the mean column times per-tp factors; the Eq. 1
    # term is linear in the latency column, so every option term is factor x the App. A term.
    I = oracle.from_json(generate.load("hand"), pct)
    G, V, _ = _hand_pct_enumeration(pct)
    for k in range(8):
        for m, want in ((0, G[k]), (1, V[k])):
            o = oracle.option(I, 1.0, m, k)
            assert o["ok"] and o["term"] == pytest.approx(float(want), rel=4e-16, abs=0), (pct, m, k)


def test_hand_case_percentile_searches():
    g = _gold("hand_case.json")["percentile_searches"]
    d = generate.load("hand")
    for pct, lam_s, B, idx, kg, kv, Lw, Tw, units, feas in g["rows"]:
        _, _, enum = _hand_pct_enumeration(pct)
        assert enum[B] == (idx, _F(Lw), feas), (pct, B)   # the fixture is the enumeration
        I = oracle.from_json(d, pct)
        lam = float(_F(lam_s))
        r = oracle.search(I, lam, B)
        assert r.found and r.index == idx and r.count == feas, (pct, B)
        p = oracle.predict(I, lam, [kg, kv], B)
        assert p["units"] == units and p["throughput"] == float(_F(Tw))
        assert p["latency"] == pytest.approx(float(_F(Lw)), rel=1e-15)
    # the selected column matters: p90 moves the B = 8 winner from TP (54) to replicas (45)
    I_mean, I_p90 = oracle.from_json(d, "mean"), oracle.from_json(d, "p90")
    assert oracle.search(I_mean, 1.0, 8).index == 54 and oracle.search(I_p90, 1.0, 8).index == 45


# ----------------------------------------------------------------------------- measured profiles (R2)
def test_measured_profiles_hand_case():
    # a profile measured at the share is used verbatim (no capacity scaling); the
    # hand-derived terms and the exact-rational winners (tests/golden/hand_case.json)
    g = _gold("hand_case.json")["measured_profiles"]
    d = generate.with_measured(generate.load("hand"), g["curves"])
    I = oracle.from_json(d)
    base = oracle.from_json(generate.load("hand"))
    changed = {(m, k) for m, k, *_ in g["terms_lambda_1"]["rows"]}
    for m, k, term, b, u in g["terms_lambda_1"]["rows"]:
        o = oracle.option(I, 1.0, m, k)
        assert o["ok"] and o["u"] == u and o["b"] == float(_F(b))
        assert o["term"] == pytest.approx(float(_F(term)), rel=4e-16, abs=0)
    for m in range(2):  # every other option keeps its scaled (App. A) term
        for k in range(8):
            if (m, k) not in changed:
                assert oracle.option(I, 1.0, m, k) == oracle.option(base, 1.0, m, k)
    rows = _gold("hand_case.json")["option_terms_lambda_1"]["rows"]
    G = [_F(r[5]) for r in rows]
    V = [_F(r[9]) for r in rows]
    for m, k, term, *_ in g["terms_lambda_1"]["rows"]:
        (G if m == 0 else V)[k] = _F(term)
    for lam_s, B, idx, kg, kv, Lw, Tw, units, feas in g["searches"]["rows"]:
        cands = sorted((G[a] + V[b], 8 * a + b) for a, b in itertools.product(range(8), range(8))
                       if rows[a][7] + rows[b][11] <= B)
        assert (cands[0][1], cands[0][0], len(cands)) == (idx, _F(Lw), feas)   # fixture = enumeration
        r = oracle.search(I, float(_F(lam_s)), B)
        assert r.found and r.index == idx and r.count == feas, B
        p = oracle.predict(I, 1.0, [kg, kv], B)
        assert p["units"] == units and p["throughput"] == float(_F(Tw))
        assert p["latency"] == pytest.approx(float(_F(Lw)), rel=1e-15)


@pytest.mark.parametrize("name", ["hand", "C1", "C2"])
def test_measured_equal_to_scaled_profile_is_exact(name):
    # Invariant of R2: a measured curve equal to the capacity-scaled base curve (rates x f,
    # latencies / f, T x f) reproduces the scaled option terms bit for bit when f is a power of two
    # (every step of the lookup scales exactly).  All (LLM, tp, share) measured this way.
    d = generate.load(name)
    F = d["F"]
    shares = [si for si, s in enumerate(d["share_units"]) if (F // s) * s == F and (F // s) & (F // s - 1) == 0]
    which = [(m, ti, si) for m in range(d["M"]) for ti in range(len(d["tp"])) for si in shares]
    dm = generate.scaled_measured(d, which)
    I, Im = oracle.from_json(d), oracle.from_json(dm)
    assert Im.meas_off is not None and int(Im.meas_off[-1]) > 0
    for lam in (d["targets"][0], d["targets"][0] * 3.0, d.get("lambda_star", d["targets"][0] * 4.0)):
        a, b = oracle.option_table(I, lam), oracle.option_table(Im, lam)
        for k in ("tau", "b", "u", "ok"):
            assert np.array_equal(a[k], b[k]), (name, lam, k)
        fin = a["ok"]
        assert np.array_equal(a["term"][fin], b["term"][fin])


def test_measured_profile_capacity_and_boundary():
    # measured T_f bounds the per-replica rate directly (x = T_f feasible, above it infeasible) and
    # gives the Eq. 2 term d*T_f/n (SPEC.md:190 boundary rule on the measured curve)
    llm = {"n": 2.0, "p": 1.0, "curves": [_curve([1.0, 4.0], [1.0, 3.0])]}
    d = {"M": 1, "F": 2, "share_units": [1, 2], "tp": [1], "replicas": [1, 2], "n": [2.0], "p": [1.0],
         "profiles": [llm["curves"]], "min_units": None, "budget_units": 10, "percentile": "mean"}
    d = generate.with_measured(d, [{"llm": 0, "tp_index": 0, "share_index": 0, "rate": [1.0, 3.0],
                                     "lat": [2.0, 6.0], "tmax": 3.0}])
    I = oracle.from_json(d)
    o = oracle.option(I, 1.5, 0, 0)       # s=1 (f=1/2), d=1: x = 1.5*2/1 = 3 = T_f -> feasible
    assert o["ok"] and o["term"] == 6.0 * 2.0 and o["b"] == 1.0 * 3.0 / 2.0
    assert not oracle.option(I, 1.5000001, 0, 0)["ok"]
    o = oracle.option(I, 1.0, 0, 1)       # d=2: x = 1 -> L = 2, term 4, b = 2*3/2 = 3
    assert o["ok"] and o["term"] == 4.0 and o["b"] == 3.0
    o = oracle.option(I, 1.0, 0, 2)       # s=2 (f=1) not measured: base curve, x = 2 -> L = 5/3
    assert o["ok"] and o["term"] == pytest.approx((1.0 + 2.0 * (1.0 / 3.0)) * 2.0, rel=1e-15)


# ----------------------------------------------------------------------------- lambda*
@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4"])
def test_lambda_star_is_maximal(name):
    # lambda* = the largest Eq. 2 value v = b_m[k] at which some candidate is
    # feasible with target lambda = v (i.e. the largest T_w of an allocation that is feasible at its
    # own T_w).  Pinned with the counting DP (O2, an independent algorithm): >= 1 feasible candidate
    # at lambda*, none at the next distinct Eq. 2 value above it, nor at 2 lambda*.  Option
    # feasibility is monotone non-increasing in lambda (x = ((lambda n)/d)/f is RNE-monotone and
    # "x <= T", "b >= lambda" both tighten), so no larger Eq. 2 value is feasible either.  (Targets
    # strictly between lambda* and the next Eq. 2 value can still be feasible: there the bound
    # x <= T, evaluated in FP64, decides at the option whose b is that next value; such a target is
    # not an Eq. 2 value of any allocation feasible at it.)
    d = generate.load(name)
    I = oracle.from_json(d)
    ls = d["lambda_star"]
    assert ls == oracle.lambda_star(I)
    b = np.unique(oracle.option_table(I, 1.0)["b"])
    nxt = b[b > ls]
    tab = oracle.option_table(I, ls)
    assert dp.count(tab["tau"], tab["u"], I.budget) >= 1
    above = [2.0 * ls] + ([float(nxt[0])] if nxt.size else [])
    for lam in above:
        tab = oracle.option_table(I, lam)
        assert dp.count(tab["tau"], tab["u"], I.budget) == 0, (name, lam)
    # monotonicity spot-check on a few more Eq. 2 values above lambda*
    for lam in nxt[1:4]:
        tab = oracle.option_table(I, float(lam))
        assert dp.count(tab["tau"], tab["u"], I.budget) == 0, (name, lam)
    if I.N <= 100_000:  # brute force agrees (C1, C2)
        assert oracle.search(I, ls).count >= 1
        assert all(oracle.search(I, lam).count == 0 for lam in above)


# ----------------------------------------------------------------------------- closed forms
def test_canonical_sum_order():
    # tau = [1, 2^-24, 2^-24]: ((1 + 2^-24) + 2^-24) rounds to 1 twice (ties-to-even), whereas
    # 1 + (2^-24 + 2^-24) = 1 + 2^-23.  The canonical left-to-right binary32 sum (R7) gives 1.0;
    # the FP64 Eq. 1 sum is exactly 1 + 2^-23.
    e = 2.0 ** -24
    I = _inst([{"n": 1.0, "p": 1.0, "curves": [_curve([1.0, 2.0], [L, 2 * L])]} for L in (1.0, e, e)])
    r = oracle.search(I, 0.5)
    assert r.found and r.index == 0 and r.latency_key == 1.0
    assert oracle.predict(I, 0.5, [0, 0, 0])["latency"] == 1.0 + 2.0 ** -23


@pytest.mark.parametrize("seed", range(6))
def test_separable_closed_form(seed):
    # B >= sum of max units: optimum = canonical FP32 sum of per-LLM minima; count = prod #finite.
    d = generate.random_instance(seed, M=3, F=2, S=[1, 2], T=[1, 2], R=[1, 2, 3], budget=10**6)
    I = oracle.from_json(d)
    lam = 0.4
    tab = oracle.option_table(I, lam)
    r = oracle.search(I, lam)
    nfin = tab["ok"].sum(axis=1)
    assert r.count == int(np.prod(nfin))
    if r.count:
        mins = [tab["tau"][m][tab["ok"][m]].min() for m in range(I.M)]
        v = np.float32(mins[0])
        for x in mins[1:]:
            v = np.float32(v + np.float32(x))
        assert np.float32(r.latency_key) == v
        # lowest index: per-LLM lowest option attaining the minimum (separable + monotone sum)
        exp = [int(np.flatnonzero(tab["ok"][m] & (tab["tau"][m] == mins[m]))[0]) for m in range(I.M)]
        assert oracle.decode(I, r.index) == exp


def test_single_llm_linear_scan():
    d = generate.random_instance(7, M=1, F=4, S=[1, 2, 4], T=[1, 2], R=[1, 2], budget=6)
    I = oracle.from_json(d)
    lam = 0.3
    best = None
    cnt = 0
    for k in range(I.K):
        s, t, dd = oracle.option_grid(I, k)
        o = oracle.option(I, lam, 0, k)
        if o["ok"] and s * t * dd <= 6:
            cnt += 1
            if best is None or o["tau"] < best[0]:
                best = (o["tau"], k)
    r = oracle.search(I, lam, 6)
    assert r.count == cnt and r.index == best[1] and np.float32(r.latency_key) == best[0]


def test_dyadic_exact_bruteforce():
    # Exactly-representable terms: f = 1, n = p = 1, x at or below the first point -> tau = L_0 exactly;
    # L_0 are multiples of 2^-10 with sums < 2^14, so every binary32 sum is exact and the optimum is
    # the exact integer-arithmetic optimum (enumerated here with Python ints).
    rng = np.random.default_rng(11)
    M, K = 3, 4
    L0 = rng.integers(1, 4096, size=(M, K))
    L0[0, 1] = L0[0, 2]  # force ties
    L0[2, 0] = L0[2, 3]
    llms = []
    for m in range(M):
        curves = [_curve([1.0, 2.0], [float(L0[m, k]) / 1024.0, float(L0[m, k]) / 512.0]) for k in range(K)]
        llms.append({"n": 1.0, "p": 1.0, "curves": curves})
    I = _inst(llms, T=(1, 2, 4, 8), budget=40)  # option k <-> tp index k; units = tp
    r = oracle.search(I, 0.5, 40)
    best, bidx, cnt = None, None, 0
    for idx, ks in enumerate(itertools.product(range(K), repeat=M)):
        units = sum([1, 2, 4, 8][k] for k in ks)
        if units > 40:
            continue
        cnt += 1
        v = sum(int(L0[m, k]) for m, k in enumerate(ks))
        if best is None or v < best:
            best, bidx = v, idx
    assert r.count == cnt and r.index == bidx and r.latency_key == best / 1024.0


# ----------------------------------------------------------------------------- O1 vs O2
@pytest.mark.parametrize("seed", range(40))
def test_bruteforce_matches_dp(seed):
    rng = np.random.default_rng(1000 + seed)
    M = int(rng.integers(1, 4))
    S = [1, 2, 4][: int(rng.integers(1, 4))]
    T = [1, 2, 4][: int(rng.integers(1, 4))]
    R = list(range(1, int(rng.integers(2, 4))))
    budget = int(rng.integers(2, 30))
    d = generate.random_instance(seed, M=M, F=4, S=S, T=T, R=R, budget=budget, min_units=bool(seed % 3 == 0))
    I = oracle.from_json(d)
    for lam in (0.05, 0.3, 1.0):
        tab = oracle.option_table(I, lam)
        r = oracle.search(I, lam)
        f, v, idx, cnt = dp.search(tab["tau"], tab["u"], budget)
        assert (r.found, r.count) == (f, cnt)
        if f:
            assert (r.latency_key, r.index) == (v, idx)


def test_dp_on_subulp_ties():
    # near-tie terms within one binary32 ulp: DP, brute force and the tie-break must agree.
    rng = np.random.default_rng(5)
    M, K = 3, 6
    base = np.float32(1.0)
    tau = (base + rng.integers(0, 3, size=(M, K)).astype(np.float32) * np.float32(2.0 ** -23)).astype(np.float32)
    u = rng.integers(1, 4, size=(M, K))
    B = 8
    f, v, idx, cnt = dp.search(tau, u, B)
    best, bidx, c = None, None, 0
    for i, ks in enumerate(itertools.product(range(K), repeat=M)):
        if sum(u[m, k] for m, k in enumerate(ks)) > B:
            continue
        c += 1
        s = tau[0, ks[0]]
        for m in range(1, M):
            s = np.float32(s + tau[m, ks[m]])
        if best is None or s < best:
            best, bidx = s, i
    assert (cnt, idx, np.float32(v)) == (c, bidx, best)


# ----------------------------------------------------------------------------- invariants
def _c(name):
    d = generate.load(name)
    return d, oracle.from_json(d)


def test_throughput_monotone_in_replicas_and_latency_nonincreasing():
    d, I = _c("C2")
    lam = d["targets"][0]
    nR = len(I.R)
    for m in range(I.M):
        for base in range(0, I.K, nR):
            b = [oracle.option(I, lam, m, base + r)["b"] for r in range(nR)]
            assert all(x <= y for x, y in zip(b, b[1:]))        # PAPER.md:334 exact
            terms = [oracle.option(I, lam, m, base + r) for r in range(nR)]
            fin = [t["term"] for t in terms if t["ok"]]
            assert all(y <= x * (1 + 1e-15) for x, y in zip(fin, fin[1:]))


def test_infeasible_when_over_budget():
    d, I = _c("C1")
    lam = d["targets"][0]
    for idx in range(0, I.N, 7):
        ks = oracle.decode(I, idx)
        p = oracle.predict(I, lam, ks)
        if p["units"] > I.budget:
            assert not p["feasible"]


def test_budget_and_target_monotonicity():
    d, I = _c("C1")
    lam = d["targets"][0]
    prev = None
    for B in range(0, 40, 3):
        r = oracle.search(I, lam, B)
        if prev is not None:
            assert r.count >= prev.count
            if prev.found:
                assert r.found and r.latency_key <= prev.latency_key
        prev = r
    prev = None
    for lam in np.linspace(0.01, 0.25, 9):
        r = oracle.search(I, float(lam))
        if prev is not None:
            assert r.count <= prev.count
            if r.found:
                assert r.latency_key >= prev.latency_key * (1 - 1e-6)
        prev = r


def test_eq2_independent_of_p():
    d, I = _c("C1")
    d2 = json.loads(json.dumps(d))
    d2["p"] = [x * 1.7 for x in d2["p"]]
    I2 = oracle.from_json(d2)
    t1 = oracle.option_table(I, 0.05)
    t2 = oracle.option_table(I2, 0.05)
    assert np.array_equal(t1["b"].view(np.uint64), t2["b"].view(np.uint64))
    assert np.array_equal(t1["ok"], t2["ok"])


def test_permutation_of_llms():
    d = generate.random_instance(3, M=3, F=2, S=[1, 2], T=[1, 2], R=[1, 2], budget=12)
    I = oracle.from_json(d)
    perm = [2, 0, 1]
    d2 = json.loads(json.dumps(d))
    for key in ("n", "p", "profiles"):
        d2[key] = [d[key][i] for i in perm]
    I2 = oracle.from_json(d2)
    r1 = oracle.search(I, 0.2)
    r2 = oracle.search(I2, 0.2)
    assert r1.count == r2.count
    if r1.found:
        assert r2.latency_key == pytest.approx(r1.latency_key, rel=3 * 2.0 ** -24)
        # the permuted optimum evaluates (FP64) to within re-association of the original optimum
        k1 = oracle.decode(I, r1.index)
        k2 = oracle.decode(I2, r2.index)
        p1 = oracle.predict(I, 0.2, k1)["latency"]
        p2 = oracle.predict(I2, 0.2, k2)["latency"]
        assert p2 == pytest.approx(p1, rel=1e-6)


def test_workload_acceptance():
    # SURVEY.md §8(d) instance acceptance: budget binds at the optimum, the target makes >= 1 option
    # infeasible, feasible_count > 0 (checked with O2 at full size).
    for name in ("C1", "C2", "C3", "C4"):
        d, I = _c(name)
        lam = d["targets"][0]
        tab = oracle.option_table(I, lam)
        f, v, idx, cnt = dp.search(tab["tau"], tab["u"], I.budget)
        assert f and cnt > 0
        assert not tab["ok"].all()
        ks = oracle.decode(I, idx)
        units = sum(int(tab["u"][m, k]) for m, k in enumerate(ks))
        sep = sum(int(tab["u"][m][tab["ok"][m] & (tab["tau"][m] == tab["tau"][m][tab["ok"][m]].min())].min())
                  for m in range(I.M))
        assert sep > I.budget
        assert units >= I.budget - int(tab["u"].max())


def test_c1_full_bruteforce_vs_literal_candidates():
    # O1's hoisted table equals per-candidate recomputation from the profiles (no hoisting), on all of C1.
    d, I = _c("C1")
    lam = d["targets"][0]
    r = oracle.search(I, lam)
    best = None
    cnt = 0
    for idx in range(I.N):
        ok, l32, _u = oracle.candidate(I, lam, idx)
        if ok:
            cnt += 1
            if best is None or l32 < best[0]:
                best = (l32, idx)
    assert (r.count, r.latency_key, r.index) == (cnt, best[0], best[1])


# ----------------------------------------------------------------------------- multi-workflow (NEXT-1)
def test_egalitarian_single_workflow_degenerates_to_search():
    # search_multi with one workflow degenerates exactly to search (all GPUs, u = 1)
    from oracle import multi
    d = generate.load("C1")
    I = oracle.from_json(d)
    lat = multi.best_latencies(I, d["targets"][0], 4, 4)
    split, mn, sm = multi.egalitarian([lat], 4)
    assert split == [4] and mn == 1.0 and sm == 1.0
    r = oracle.search(I, d["targets"][0], 16)
    assert lat[4] == oracle.predict(I, d["targets"][0], oracle.decode(I, r.index), 16)["latency"]


def test_egalitarian_identical_workflows_split_evenly():
    # two identical workflows with identical rates on an even cluster -> symmetric
    # split, equal utilities
    from oracle import multi
    d = generate.load("C1")
    I = oracle.from_json(d)
    lat = multi.best_latencies(I, d["targets"][0], 8, 4)
    split, mn, sm = multi.egalitarian([lat, lat], 8)
    assert split == [4, 4]
    u = lat[8] / lat[4]
    assert mn == u and sm == u + u
    assert all(a >= b for a, b in zip(lat, lat[1:]))  # more GPUs never hurt (budget monotone)


# ----------------------------------------------------------------------------- max-throughput fallback
def test_max_throughput_hand_case():
    """SPEC.md:374 fallback on the App. A hand case, derived by hand: Eq. 2 terms d*f*T/n are
    {1, 2, 1.75, 3.5, 2, 4, 3.5, 7} for both LLMs (options k = (s*2 + tp)*2 + d), units
    {1, 2, 2, 4, 2, 4, 4, 8}.  B = 8: T_w = 4 needs option 5 (4 units) for both LLMs (7 would need
    16 units) -> index 5*8 + 5 = 45, the App. A row lambda = 4 (lambda = 5 infeasible).  B = 7:
    T_w = 3.5 needs 8 units, T_w = 2 needs 2 + 2 -> index 1*8 + 1 = 9.  B = 3: only T_w = 1
    (1 + 1 units) -> index 0.  B = 1: two LLMs need 2 units -> none."""
    I = oracle.from_json(generate.load("hand"))
    assert oracle.max_throughput(I, 8) == {"index": 45, "throughput": 4.0, "units": 8}
    assert oracle.max_throughput(I, 7) == {"index": 9, "throughput": 2.0, "units": 4}
    assert oracle.max_throughput(I, 3) == {"index": 0, "throughput": 1.0, "units": 2}
    assert oracle.max_throughput(I, 1) is None


@pytest.mark.parametrize("name", ["hand", "C1", "C2"])
def test_max_throughput_equals_lambda_star(name):
    """The largest T_w within the budget bounds lambda*, the largest target at which some candidate
    is feasible (oracle.lambda_star, the full R4 test of the C oracle at lambda = v), from above: a
    candidate feasible at lambda has every b_m >= lambda.  At the configs' budgets they are equal;
    at B = 3 on C1/C2 the max-T_w candidate has b = lambda exactly but x = ((lambda*n)/d)/f lands one
    ulp above T, so R4 rejects it at lambda = T_w (reading R17: the fallback maximises Eq. 2 alone)."""
    d = generate.load(name)
    I = oracle.from_json(d)
    for B in (d["budget_units"], d["budget_units"] // 2, 3):
        r = oracle.max_throughput(I, B)
        ls = oracle.lambda_star(I, B)
        assert (r is None and ls == 0.0) or ls <= r["throughput"], (name, B)
        if B != 3:
            assert r["throughput"] == ls, (name, B)


def test_max_throughput_separable_closed_form():
    """Against the separable construction (max-min over independent per-LLM choices): theta* = max
    over Eq. 2 values v with sum_m min{u : b >= v, floor ok} <= B; lowest index by digits, each the
    smallest option whose completion still fits — on random instances with memory floors."""
    for seed in range(12):
        d = generate.random_instance(500 + seed, M=3, F=4, S=[1, 2, 4], T=[1, 2], R=[1, 2], budget=14,
                                     min_units=bool(seed % 2))
        I = oracle.from_json(d)
        tab = oracle.option_table(I, 1.0)
        ok = [[oracle.floor_ok(I, m, k) for k in range(I.K)] for m in range(I.M)]
        for B in (2, 5, 9, 14, 40):
            def minu(m, v):
                c = [int(tab["u"][m][k]) for k in range(I.K) if ok[m][k] and tab["b"][m][k] >= v]
                return min(c) if c else None
            best = None
            for v in sorted(set(tab["b"].ravel().tolist())):
                mus = [minu(m, v) for m in range(I.M)]
                if all(x is not None for x in mus) and sum(mus) <= B:
                    best = v
            r = oracle.max_throughput(I, B)
            if best is None:
                assert r is None
                continue
            idx, used = 0, 0
            for m in range(I.M):
                rest = sum(minu(j, best) for j in range(m + 1, I.M))
                k = next(k for k in range(I.K) if ok[m][k] and tab["b"][m][k] >= best
                         and used + int(tab["u"][m][k]) + rest <= B)
                used += int(tab["u"][m][k])
                idx = idx * I.K + k
            assert r == {"index": idx, "throughput": best, "units": used}, (seed, B)
