"""Seeded synthetic ALP instances (profile tables + grids) shared by the oracle and the CUDA path.

This module holds NO arithmetic of the method (no Eq. 1 / Eq. 2, no interpolation, no
fraction scaling, no search).  It only draws per-LLM workload parameters and writes
synthetic throughput-latency profile tables whose *shape* follows SURVEY.md App. C:

* rates   r_i = mu*sigma(t) * 0.01 * 95**(i/11), i = 0..11, T_m = r_11
* latency L_i = (ell/sigma(t)) / (1 - r_i/(mu*sigma(t)))        (M/M/1-PS shape)
* p50/p90/p99 = mean * {0.8, 1.9, 3.5}                           (monotone)
* sigma(t) = {1: 1.0, 2: 1.7, 4: 2.8, 8: 4.5}                     (SPEC.md:547 + 8 invented)

Per-LLM parameters (ell, mu, n, p) are drawn with numpy.random.default_rng(seed) in the order
ell, mu, n (log-uniform), then p (uniform), per LLM.  Seeds are 20260417 + config id.

Targets (lambda) are NOT produced here: they need the method's Eq. 2 terms, so
`oracle/make_targets.py` (oracle-only script) computes lambda* and writes them into the JSON.

Workloads (BASELINE.json "configs"):
  C1  beam search GEN+VER, 4 GPUs,  F=4, S={1,2,4}/4, T={1,2,4},   R=1..4,  B=16
  C2  beam search GEN+VER, 8 GPUs,  F=8, S=1..8/8,   T={1,2,4,8}, R=1..8,  B=64
  C3  4-LLM agent, 16 GPUs,         F=8, S=1..8/8,   T={1,2,4,8}, R=1..16, B=128
  C4  8-LLM workflow, 64 GPUs,      F=2, S={1,2}/2,  T={1,2,4},   R={1,2,4}, B=128
  C5  C4 with 256 throughput targets (Pareto sweep)
  hand  SURVEY.md App. A two-LLM hand case (exact rationals)
"""
from __future__ import annotations

import json
import math
import os
from typing import Any

import numpy as np

SIGMA = {1: 1.0, 2: 1.7, 4: 2.8, 8: 4.5}
PCT_SCALE = {"mean": 1.0, "p50": 0.8, "p90": 1.9, "p99": 3.5}
N_POINTS = 12
SEED_BASE = 20260417

HERE = os.path.dirname(os.path.abspath(__file__))
INSTANCE_DIR = os.path.join(HERE, "instances")


def _profile(ell: float, mu: float, t: int) -> dict[str, Any]:
    """One synthetic per-(LLM, TP) profile curve (App. C shape, not the method)."""
    sig = SIGMA[t]
    cap = mu * sig
    rates = [cap * 0.01 * 95.0 ** (i / 11.0) for i in range(N_POINTS)]
    mean = [(ell / sig) / (1.0 - r / cap) for r in rates]
    lat = {k: [m * s for m in mean] for k, s in PCT_SCALE.items()}
    return {"rate": rates, "lat": lat, "tmax": rates[-1]}


def _loguniform(rng: np.random.Generator, lo: float, hi: float) -> float:
    return float(math.exp(rng.uniform(math.log(lo), math.log(hi))))


def _instance(name: str, cid: int, llms: list[dict[str, float]], F: int, S: list[int], T: list[int],
              R: list[int], budget: int, description: str) -> dict[str, Any]:
    return {
        "name": name,
        "config_id": cid,
        "seed": SEED_BASE + cid,
        "description": description,
        "M": len(llms),
        "F": F,
        "share_units": S,
        "tp": T,
        "replicas": R,
        "n": [l["n"] for l in llms],
        "p": [l["p"] for l in llms],
        "llm_params": llms,
        "profiles": [[_profile(l["ell"], l["mu"], t) for t in T] for l in llms],
        "min_units": None,
        "budget_units": budget,
        "percentile": "mean",
    }


BEAM = [  # GEN ~ Llama-3.2-1B, VER ~ Llama-3.1-8B-PRM; n inside 24-844,
    {"name": "GEN", "ell": 0.08, "mu": 40.0, "n": 160.0, "p": 3.0},  # p_GEN ~ 3
    {"name": "VER", "ell": 0.25, "mu": 12.0, "n": 160.0, "p": 2.0},  # p_VER ~ 2
]


def _drawn(cid: int, M: int, ell: tuple[float, float], mu: tuple[float, float], n: tuple[float, float],
           p: tuple[float, float]) -> list[dict[str, float]]:
    rng = np.random.default_rng(SEED_BASE + cid)
    out = []
    for m in range(M):
        e = _loguniform(rng, *ell)
        u = _loguniform(rng, *mu)
        nn = _loguniform(rng, *n)
        pp = float(rng.uniform(*p))
        out.append({"name": f"LLM{m}", "ell": e, "mu": u, "n": nn, "p": pp})
    return out


def make_c1() -> dict[str, Any]:
    return _instance("C1", 1, [dict(x) for x in BEAM], 4, [1, 2, 4], [1, 2, 4], [1, 2, 3, 4], 16,
                     "beam search GEN+VER (2 LLMs), 4 GPUs, shares {1/4,1/2,1}, TP {1,2,4}, replicas 1-4")


def make_c2() -> dict[str, Any]:
    return _instance("C2", 2, [dict(x) for x in BEAM], 8, list(range(1, 9)), [1, 2, 4, 8], list(range(1, 9)), 64,
                     "beam search GEN+VER on one 8-GPU node, shares in 1/8 steps, TP {1,2,4,8}, replicas 1-8")


def make_c3() -> dict[str, Any]:
    llms = _drawn(3, 4, (0.05, 2.0), (2.0, 60.0), (2.0, 12.0), (1.0, 3.0))
    for l, nm in zip(llms, ["planner", "coder", "critic", "verifier"]):
        l["name"] = nm
    return _instance("C3", 3, llms, 8, list(range(1, 9)), [1, 2, 4, 8], list(range(1, 17)), 128,
                     "4-LLM agentic workflow (planner/coder/critic/verifier) on 16 GPUs, full share/TP/replica grid")


def make_c4() -> dict[str, Any]:
    llms = _drawn(4, 8, (0.02, 2.0), (2.0, 200.0), (1.0, 50.0), (1.0, 4.0))
    return _instance("C4", 4, llms, 2, [1, 2], [1, 2, 4], [1, 2, 4], 128,
                     "8-LLM workflow on a 64-GPU cluster: 18^8 ~ 1.1e10 candidates")


def make_c5() -> dict[str, Any]:
    inst = make_c4()
    inst["name"] = "C5"
    inst["config_id"] = 5
    inst["description"] = "throughput-target sweep: 256 targets batched over the 8-LLM (C4) space"
    return inst


# Hand-case percentile columns: the mean column times a per-tp factor (tp index 0, tp index 1), so
# every percentile's option terms are exact multiples of App. A's (tests/golden/hand_case.json
# "percentile_searches"); p90/p99 penalise tensor parallelism, which moves the winner.
HAND_PCT_FACTOR = {"mean": (1.0, 1.0), "p50": (0.5, 0.5), "p90": (1.0, 3.0), "p99": (2.0, 5.0)}


def make_hand() -> dict[str, Any]:
    """F=2, S={1,2}, T={1,2}, R={1,2}; exact-rational profiles."""
    def prof(rates, lats, ti):
        return {"rate": rates, "lat": {k: [c[ti] * x for x in lats] for k, c in HAND_PCT_FACTOR.items()},
                "tmax": rates[-1]}
    return {
        "name": "hand", "config_id": 0, "seed": 0,
        "description": "SURVEY.md App. A two-LLM hand case (GEN n=4 p=2, VER n=2 p=1)",
        "M": 2, "F": 2, "share_units": [1, 2], "tp": [1, 2], "replicas": [1, 2],
        "n": [4.0, 2.0], "p": [2.0, 1.0],
        "llm_params": [{"name": "GEN"}, {"name": "VER"}],
        "profiles": [
            [prof([1.0, 8.0], [0.5, 1.5], 0), prof([1.0, 14.0], [0.25, 1.0], 1)],
            [prof([1.0, 4.0], [1.0, 3.0], 0), prof([1.0, 7.0], [0.5, 2.0], 1)],
        ],
        "min_units": None, "budget_units": 8, "percentile": "mean",
    }


MAKERS = {"hand": make_hand, "C1": make_c1, "C2": make_c2, "C3": make_c3, "C4": make_c4, "C5": make_c5}


def instance_path(name: str) -> str:
    return os.path.join(INSTANCE_DIR, f"{name}.json")


def load(name: str) -> dict[str, Any]:
    """Load a committed instance (profiles + oracle-written targets)."""
    with open(instance_path(name)) as f:
        return json.load(f)


def write_profiles(names=None) -> None:
    """(Re)write the profile part of the instance JSONs; keeps any targets already present."""
    os.makedirs(INSTANCE_DIR, exist_ok=True)
    for name in names or MAKERS:
        inst = MAKERS[name]()
        path = instance_path(name)
        if os.path.exists(path):
            with open(path) as f:
                old = json.load(f)
            for k in ("targets", "lambda_star", "targets_note"):
                if k in old:
                    inst[k] = old[k]
        with open(path, "w") as f:
            json.dump(inst, f, indent=1)
            f.write("\n")


def skew_percentile(d: dict[str, Any], pct: str, seed: int, lo: float = 1.0, hi: float = 4.0) -> dict[str, Any]:
    """Copy of instance d whose `pct` latency column is the mean column times a seeded per-(LLM, tp)
    factor in [lo, hi) (tests: a tail percentile whose shape differs from the mean's, so the optimum
    moves when the percentile is selected)."""
    rng = np.random.default_rng(seed)
    out = json.loads(json.dumps(d))
    for per_t in out["profiles"]:
        for c in per_t:
            f = float(rng.uniform(lo, hi))
            c["lat"][pct] = [f * x for x in c["lat"]["mean"]]
    return out


def with_measured(d: dict[str, Any], curves: list[dict[str, Any]]) -> dict[str, Any]:
    """Copy of instance d with profiles measured at given (llm, tp_index, share_index); each curve's
    latency list is used for every percentile column unless it is already a per-percentile dict."""
    out = json.loads(json.dumps(d))
    meas = []
    for c in curves:
        c = dict(c)
        if not isinstance(c["lat"], dict):
            c["lat"] = {k: list(c["lat"]) for k in PCT_SCALE}
        meas.append(c)
    out["measured"] = meas
    return out


def scaled_measured(d: dict[str, Any], which) -> dict[str, Any]:
    """Copy of d where every (llm, tp_index, share_index) in `which` gets a measured curve equal to the
    capacity-scaled base curve (rates x f, latencies / f, tmax x f with f = share/F): the reading R2
    makes such a curve reproduce the scaled profile exactly when f is a power of two."""
    curves = []
    for m, ti, si in which:
        base = d["profiles"][m][ti]
        f = d["share_units"][si] / d["F"]
        curves.append({"llm": m, "tp_index": ti, "share_index": si, "rate": [r * f for r in base["rate"]],
                       "lat": {k: [x / f for x in v] for k, v in base["lat"].items()},
                       "tmax": (base["tmax"] if base.get("tmax") is not None else base["rate"][-1]) * f})
    return with_measured(d, curves)


def random_measured(d: dict[str, Any], seed: int, frac: float = 0.3) -> dict[str, Any]:
    """Copy of d with seeded measured curves on a random subset of (llm, tp, share): the scaled base
    curve perturbed (latencies x U[0.7, 1.3], capacity x U[0.8, 1.2]), monotone by construction."""
    rng = np.random.default_rng(seed)
    curves = []
    for m in range(d["M"]):
        for ti in range(len(d["tp"])):
            for si in range(len(d["share_units"])):
                if rng.random() >= frac:
                    continue
                base = d["profiles"][m][ti]
                f = d["share_units"][si] / d["F"]
                lf, cf = float(rng.uniform(0.7, 1.3)), float(rng.uniform(0.8, 1.2))
                curves.append({"llm": m, "tp_index": ti, "share_index": si,
                               "rate": [r * f * cf for r in base["rate"]],
                               "lat": {k: [x / f * lf for x in v] for k, v in base["lat"].items()},
                               "tmax": (base["tmax"] if base.get("tmax") is not None else base["rate"][-1]) * f * cf})
    return with_measured(d, curves)


# ---------------------------------------------------------------- random small instances (tests)
def random_instance(seed: int, M: int, F: int, S: list[int], T: list[int], R: list[int], budget: int,
                    points: int = 4, min_units: bool = False) -> dict[str, Any]:
    """Small seeded instance with arbitrary piecewise-linear monotone profiles (test fuzzing)."""
    rng = np.random.default_rng(seed)
    profiles = []
    for _m in range(M):
        per_t = []
        for _t in T:
            r0 = float(rng.uniform(0.05, 1.0))
            steps = rng.uniform(0.2, 3.0, size=points - 1)
            rates = [r0]
            for s in steps:
                rates.append(rates[-1] + float(s))
            l0 = float(rng.uniform(0.05, 2.0))
            lsteps = rng.uniform(0.0, 2.0, size=points - 1)
            lats = [l0]
            for s in lsteps:
                lats.append(lats[-1] + float(s))
            tmax = rates[-1] * (1.0 + float(rng.uniform(0.0, 0.3)) * float(rng.integers(0, 2)))
            per_t.append({"rate": rates, "lat": {"mean": lats, "p50": lats, "p90": [2 * x for x in lats],
                                                  "p99": [3 * x for x in lats]}, "tmax": tmax})
        profiles.append(per_t)
    n = [float(rng.uniform(0.5, 8.0)) for _ in range(M)]
    p = [float(rng.uniform(1.0, 3.0)) for _ in range(M)]
    mu = None
    if min_units:
        mu = [[int(rng.integers(1, max(S) + 1)) for _ in T] for _ in range(M)]
    return {"name": f"rand{seed}", "config_id": -1, "seed": seed, "description": "random test instance",
            "M": M, "F": F, "share_units": S, "tp": T, "replicas": R, "n": n, "p": p,
            "profiles": profiles, "min_units": mu, "budget_units": budget, "percentile": "mean"}


if __name__ == "__main__":
    write_profiles()
    print("wrote", ", ".join(MAKERS))
