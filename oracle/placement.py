"""ORACLE — test infrastructure only.  Placement checks:
validate() lists violations of the placement invariants; exact_place() decides by exhaustive
backtracking whether ANY valid placement exists (small instances only: the paper calls the optimum
NP-hard)."""
from __future__ import annotations


def shards(share_units, tp, replicas):
    """(llm, replica, shard, units) in the library's output order."""
    out = []
    for m, (s, t, d) in enumerate(zip(share_units, tp, replicas)):
        for r in range(d):
            for k in range(t):
                out.append((m, r, k, s))
    return out


def validate(gpu_node, gpu_domain, F, share_units, tp, replicas, shard_gpu):
    sh = shards(share_units, tp, replicas)
    errs = []
    if len(shard_gpu) != len(sh):
        return ["shard count mismatch"]
    load = [0] * len(gpu_node)
    groups = {}
    for (m, r, _k, s), g in zip(sh, shard_gpu):
        if not 0 <= g < len(gpu_node):
            errs.append(f"shard of LLM {m} on invalid GPU {g}")
            continue
        load[g] += s
        groups.setdefault((m, r), []).append(g)
    errs += [f"GPU {g} over capacity ({u}/{F})" for g, u in enumerate(load) if u > F]
    for (m, r), gs in groups.items():
        if len(set(gs)) != len(gs):
            errs.append(f"tensor group ({m},{r}) reuses a GPU")
        if len({gpu_domain[g] for g in gs}) > 1:
            errs.append(f"tensor group ({m},{r}) spans NVLink domains")
    return errs


def exact_place(gpu_node, gpu_domain, F, share_units, tp, replicas, limit=24):
    """True iff some valid placement exists (backtracking over tensor groups, largest first)."""
    groups = [(s, t) for s, t, d in zip(share_units, tp, replicas) for _ in range(d)]
    if sum(t for _s, t in groups) > limit or len(gpu_node) > 8:
        raise ValueError("instance over the exact-placement guard rails")
    if sum(s * t for s, t in groups) > F * len(gpu_node):
        return False
    groups.sort(key=lambda x: -x[0] * x[1])
    doms = {}
    for g, dm in enumerate(gpu_domain):
        doms.setdefault(dm, []).append(g)
    free = [F] * len(gpu_node)

    def rec(i):
        if i == len(groups):
            return True
        s, t = groups[i]
        tried = set()
        for gs in doms.values():
            cand = [g for g in gs if free[g] >= s]
            if len(cand) < t:
                continue
            from itertools import combinations
            for combo in combinations(cand, t):
                sig = tuple(sorted(free[g] for g in combo)) + (id(gs),)
                if sig in tried:
                    continue  # symmetric GPU choices
                tried.add(sig)
                for g in combo:
                    free[g] -= s
                ok = rec(i + 1)
                for g in combo:
                    free[g] += s
                if ok:
                    return True
        return False

    return rec(0)
