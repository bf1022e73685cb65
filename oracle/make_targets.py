"""ORACLE script (test infrastructure): writes the throughput targets into workloads/instances/*.json.

The targets need the method's Eq. 2 terms, so they are computed here from the oracle only (never
from the CUDA path) and stored in the committed JSON, which both sides then read:

  lambda* = budget-aware maximum throughput, computed by oracle.lambda_star;
  single-target configs: lambda = 0.25 * lambda*  (exact in binary);
  C5: lambda_j = lambda* * (j + 1) / 256, j = 0..255  (top target is lambda* itself, so count >= 1).
  hand: the App. A rows use their own exact targets (tests/golden/hand_case.json).

Run:  python -m oracle.make_targets
"""
from __future__ import annotations

import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import oracle  # noqa: E402
from workloads import generate  # noqa: E402


def main() -> None:
    generate.write_profiles()
    for name in ["C1", "C2", "C3", "C4", "C5"]:
        d = generate.load(name)
        I = oracle.from_json(d)
        ls = oracle.lambda_star(I)
        d["lambda_star"] = ls
        if name == "C5":
            d["targets"] = [ls * (j + 1) / 256.0 for j in range(256)]
            d["targets_note"] = "lambda_j = lambda* (j+1)/256 (oracle.make_targets)"
        else:
            d["targets"] = [0.25 * ls]
            d["targets_note"] = "lambda = 0.25 lambda* (oracle.make_targets)"
        with open(generate.instance_path(name), "w") as f:
            json.dump(d, f, indent=1)
            f.write("\n")
        print(f"{name}: lambda*={ls!r} N={I.N}")
    d = generate.load("hand")
    d["targets"] = [1.0]
    d["targets_note"] = "SURVEY.md App. A row lambda=1, B=8"
    with open(generate.instance_path("hand"), "w") as f:
        json.dump(d, f, indent=1)
        f.write("\n")


if __name__ == "__main__":
    main()
