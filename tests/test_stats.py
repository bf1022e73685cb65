"""NEXT-4: workflow statistics n_m, p_m from traces.  Host-side library code
(alp_workflow_stats) vs the exact-rational oracle (oracle/stats.py), and oracle pins."""
from __future__ import annotations

from fractions import Fraction

import numpy as np
import pytest

from oracle import stats as ostats


def _beam_trace(n_req=3, rounds=4):
    """Beam search shaped like PAPER.md Fig. 1 / :323: every round three beams call GEN
    concurrently, then VER is called on two of them concurrently (one beam repeated the same
    value).  Expected p_GEN = 3, p_VER = 2 exactly; n_GEN = 3*rounds, n_VER = 2*rounds."""
    inv = []
    for r in range(n_req):
        t = Fraction(r * 1000)
        for _ in range(rounds):
            for _b in range(3):
                inv.append((r, 0, t, t + 2))
            t += 2
            for _b in range(2):
                inv.append((r, 1, t, t + Fraction(1, 2)))
            t += 1
    return inv


def test_spec_example_overlap():
    # one request, invocations [0,2],[0,2],[1,3] -> counts 2,3,1 -> p = 2.0; n = 3
    n, p = ostats.stats(1, 1, [(0, 0, 0, 2), (0, 0, 0, 2), (0, 0, 1, 3)])
    assert n == [3] and p == [2]


def test_sequential_chain_is_one():
    # strictly sequential chain -> p_m = 1 for every LLM
    inv = [(0, m % 2, t, t + 1) for m, t in enumerate(range(0, 10, 2))]
    n, p = ostats.stats(1, 2, inv)
    assert p == [1, 1] and n == [3, 2]


def test_beam_search_matches_paper_values():
    # "p_GEN ~ 3 and p_VER ~ 2"
    n, p = ostats.stats(3, 2, _beam_trace())
    assert p == [3, 2] and n == [12, 8]


def test_translation_and_scaling_invariance():
    rng = np.random.default_rng(1)
    inv = [(int(rng.integers(0, 3)), int(rng.integers(0, 2)), Fraction(int(a)), Fraction(int(a) + int(b)))
           for a, b in zip(rng.integers(0, 50, 40), rng.integers(1, 9, 40))]
    n, p = ostats.stats(3, 2, inv)
    n2, p2 = ostats.stats(3, 2, [(r, m, 7 * s + 11, 7 * e + 11) for r, m, s, e in inv])
    assert n == n2 and p == p2


def test_library_matches_oracle():
    import paper_2604_15186_b200 as P
    cases = [(1, 1, [(0, 0, 0, 2), (0, 0, 0, 2), (0, 0, 1, 3)]), (3, 2, _beam_trace())]
    rng = np.random.default_rng(7)
    for _ in range(20):
        n_req, M = int(rng.integers(1, 5)), int(rng.integers(1, 4))
        k = int(rng.integers(0, 60))
        st = rng.uniform(0, 20, k)
        cases.append((n_req, M, [(int(rng.integers(0, n_req)), int(rng.integers(0, M)), float(s),
                                  float(s + rng.exponential(2.0))) for s in st]))
    for n_req, M, inv in cases:
        n, p = ostats.stats(n_req, M, inv)
        r = [x[0] for x in inv]
        m = [x[1] for x in inv]
        s = [float(x[2]) for x in inv]
        e = [float(x[3]) for x in inv]
        ln, lp = P.workflow_stats(n_req, M, r, m, s, e)
        assert np.allclose(ln, [float(x) for x in n], rtol=0, atol=0)
        assert np.allclose(lp, [float(x) for x in p], rtol=1e-12)


def test_library_validation():
    import paper_2604_15186_b200 as P
    with pytest.raises(P.AlpError, match="start <= end"):
        P.workflow_stats(1, 1, [0], [0], [2.0], [1.0])
    with pytest.raises(P.AlpError, match="n_req"):
        P.workflow_stats(0, 1, [], [], [], [])
