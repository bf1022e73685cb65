"""ORACLE — test infrastructure only.  Workflow statistics from execution traces, written out
literally ("the average number of invocations per workflow request, n_m, and its
average request-level parallelism, p_m ... determined by overlapping timestamps"; SPEC.md:113-115
for the time-average / busy-time weighting, DESIGN.md §3 reading R15), in exact rational arithmetic.

For each request and LLM the busy timeline is cut at every start/end point; on each elementary
segment the number of running invocations c is counted; p_r = (sum over segments with c >= 1 of
c * length) / (sum of those lengths); p_m = busy-time-weighted mean of p_r over requests.
"""
from __future__ import annotations

from fractions import Fraction


def stats(n_req: int, M: int, invocations):
    """invocations: iterable of (request, llm, start, end).  Returns (n[M], p[M]) as Fractions."""
    inv = [(int(r), int(m), Fraction(s), Fraction(e)) for r, m, s, e in invocations]
    n = [Fraction(sum(1 for x in inv if x[1] == m), n_req) for m in range(M)]
    p = []
    for m in range(M):
        num = Fraction(0)
        den = Fraction(0)
        for r in range(n_req):
            iv = [(s, e) for rr, mm, s, e in inv if rr == r and mm == m]
            if not iv:
                continue
            pts = sorted({t for s, e in iv for t in (s, e)})
            busy = Fraction(0)
            area = Fraction(0)
            for a, b in zip(pts, pts[1:]):
                c = sum(1 for s, e in iv if s <= a and e >= b)  # running on the whole segment [a, b]
                if c >= 1:
                    busy += b - a
                    area += c * (b - a)
            if busy > 0:
                p_r = area / busy
                num += p_r * busy  # weight = request busy time
                den += busy
        p.append(num / den if den > 0 else Fraction(1))
    return n, p
