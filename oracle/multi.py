"""ORACLE — test infrastructure only.  Multi-workflow allocation with egalitarian welfare
("constructs a multi-workflow resource allocation ... how many GPUs to allocate to
each workflow ... searches for the per-workflow allocation independently ... egalitarian welfare
policy"; the utility, which the paper does not define, is SPEC.md:383's
u_w = L_w^solo-best / L_w^achieved in (0, 1], 0 when infeasible; DESIGN.md §3 reading R14).

Per workflow and GPU count g the best allocation comes from the DP oracle (O2) at budget g*F and
its FP64 latency from oracle.predict; the split search is a plain enumeration.
"""
from __future__ import annotations

import itertools

import numpy as np

import oracle
from oracle import dp


def best_latencies(I: oracle.Instance, lam: float, gpus: int, units_per_gpu: int) -> list[float]:
    """L_w(g) for g = 0..gpus: FP64 latency of the canonical optimum at budget g*F (inf if none)."""
    tab = oracle.option_table(I, lam)
    out = []
    for g in range(gpus + 1):
        f, _v, idx, _cnt = dp.search(tab["tau"], tab["u"], g * units_per_gpu)
        out.append(oracle.predict(I, lam, oracle.decode(I, idx), g * units_per_gpu)["latency"] if f else float("inf"))
    return out


def egalitarian(lat: list[list[float]], gpus: int):
    """Split `gpus` whole GPUs: maximise min_w u_w, then sum_w u_w, then the lowest split
    (g_0 most significant; the last workflow takes the remainder).  Returns (split, min u, sum u)."""
    W = len(lat)
    best = None
    for head in itertools.product(range(gpus + 1), repeat=W - 1):
        if sum(head) > gpus:
            continue
        split = list(head) + [gpus - sum(head)]
        us = []
        for w, g in enumerate(split):
            solo, l = lat[w][gpus], lat[w][g]
            us.append(solo / l if np.isfinite(l) and np.isfinite(solo) else 0.0)
        mn = min(us)
        sm = 0.0
        for u in us:
            sm = sm + u
        key = (mn, sm)
        if best is None or key > best[0]:  # strict: keeps the lowest split on exact ties
            best = (key, split)
    return best[1], best[0][0], best[0][1]
