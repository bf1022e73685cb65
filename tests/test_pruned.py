"""NEXT-2: the paper's pruned scheduler as a comparator (comparators/pruned_search.py)."""
from __future__ import annotations

import pytest

from comparators import pruned_search as ps


def test_unpruned_count_matches_paper():
    # 5 LLMs, 16 GPUs, 10 fractions per GPU -> C(16*10+5-1, 5-1) "~ 29 million"
    # (= 29,051,001; SPEC.md:340's 29,772,765 is C(165,4), an off-by-one, SURVEY finding 1)
    assert ps.count_unpruned(16, 10, 5) == 29_051_001
    assert ps.count_unpruned(1, 1, 1) == 1 and ps.count_unpruned(2, 2, 2) == 5


def test_enumeration_ordering_example():
    # ratios 0.9/0.1, mins 1/1, 4 units -> {(3,1), (2,2)}; (1,3) excluded by ordering
    assert sorted(ps.fraction_assignments(4, [1, 1])) == [(2, 2), (3, 1)]
    assert list(ps.fraction_assignments(4, [3, 3])) == []          # mins exceed the budget
    assert list(ps.fraction_assignments(7, [1])) == [(7,)]           # single LLM: all units


def test_ordering_relaxation_for_memory_minimums():
    # SPEC.md:349 / :401: a lower-ratio LLM whose memory minimum exceeds the higher-ratio LLM's part
    # waives the ordering for that pair: mins [1, 3] with 4 units -> (1, 3), which ordering alone forbids
    assert list(ps.fraction_assignments(4, [1, 3])) == [(1, 3)]
    # 6 units: (3, 3) is ordered; after parts 2 and 1 the minimum 3 forces the waiver -> (2, 4), (1, 5)
    assert sorted(ps.fraction_assignments(6, [1, 3])) == [(1, 5), (2, 4), (3, 3)]
    # mins [1, 1] never waive: the SPEC.md:347 example is unchanged
    assert sorted(ps.fraction_assignments(4, [1, 1])) == [(2, 2), (3, 1)]
    # the waiver is pairwise: the third LLM is still ordered against the second
    got = list(ps.fraction_assignments(6, [1, 3, 1]))
    assert sorted(got) == [(1, 3, 2), (1, 4, 1), (2, 3, 1)] and all(c[2] <= c[1] for c in got)


def test_packing_example():
    # PAPER.md:392 / SPEC.md:356: 1.66 GPUs with F = 10 -> 10 units on GPU 1 and 6 on GPU 2
    (pieces, whole), = ps.pack((16,), 10)
    assert pieces == [10, 6] and not whole
    lay = ps.pack((5, 5), 10)                                        # co-located on GPU 1
    assert lay == [([5], False), ([5], False)]
    assert ps.pack((30,), 10) == [([10, 10, 10], True)]              # exact fit


def test_parallelism_examples():
    # span of 4 whole GPUs, NVLink domain 2 -> {(tp 1, d 4), (tp 2, d 2)}
    opts = ps.parallelism([10, 10, 10, 10], True, 10, [1, 2, 4, 8], list(range(1, 9)), [10], nvlink=2)
    assert opts == [(10, 1, 4), (10, 2, 2)]
    # 6 units of F = 10 with a 3-unit minimum -> tp 1, d in {1, 2}
    opts = ps.parallelism([6], False, 10, [1], list(range(1, 9)), list(range(1, 11)), nvlink=8, minu=3)
    assert opts == [(3, 1, 2), (6, 1, 1)]


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["C1", "C2", "C3"])
def test_pruned_never_beats_exhaustive(name):
    import oracle
    import paper_2604_15186_b200 as P
    from workloads import generate
    d = generate.load(name)
    alp = P.Alp.from_instance(d)
    lam, B = d["targets"][0], d["budget_units"]
    ex = alp.search(lam, B)
    pr = ps.pruned_search(alp, d, lam, B // d["F"])
    assert pr.candidates > 0
    if pr.found:
        assert pr.latency >= ex.latency
        I = oracle.from_json(d)
        ks = [(I.S.tolist().index(s) * len(I.T) + I.T.tolist().index(t)) * len(I.R) + I.R.tolist().index(r)
              for s, t, r in pr.allocation]
        o = oracle.predict(I, lam, ks, B)
        assert o["feasible"] and o["latency"] == pr.latency and o["units"] == pr.units
