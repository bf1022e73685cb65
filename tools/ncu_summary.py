"""profiles/ncu_summary.json from `ncu --set full` raw-page exports of the search kernel (one launch
per workload), read by bench.py for the roofline line's DRAM traffic and pipe utilisation (neither
can be measured inside a timed run: ncu replays the kernel).

    python tools/ncu_summary.py C4=profiles/r02_C4_k_search_ncu_raw.csv C3=profiles/r02_C3_k_search_ncu_raw.csv
"""
import csv
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from workloads import generate  # noqa: E402

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "inst": 1, "us": 1, "ms": 1e3, "ns": 1e-3, "%": 1}


def main():
    out = {"_note": "search kernel, one launch, ncu --set full --clock-control none (tools/ncu_summary.py); "
                    "dram_bytes = dram__bytes_read.sum + dram__bytes_write.sum; pipe / issue fractions "
                    "= sm__pipe_{fma,alu}_cycles_active / sm__inst_issued .avg.pct_of_peak_sustained_active; "
                    "sass_instr_per_candidate = 32 x smsp__inst_executed.sum / candidates"}
    for arg in sys.argv[1:]:
        w, path = arg.split("=", 1)
        rows = list(csv.reader(open(path)))
        h, u, v = rows[0], rows[1], rows[2]

        def get(k):
            i = h.index(k)
            return float(v[i].replace(",", "")) * UNIT.get(u[i], 1)
        d = generate.load(w)
        cand = d.get("num_candidates") or 1
        if cand == 1:
            K = len(d["share_units"]) * len(d["tp"]) * len(d["replicas"])
            cand = K ** d["M"] * len(d["targets"])
        out[w] = {
            "kernel": v[h.index("Kernel Name")] if "Kernel Name" in h else None,
            "kernel_us": get("gpu__time_duration.sum"),
            "dram_bytes": int(round(get("dram__bytes_read.sum") + get("dram__bytes_write.sum"))),
            "fma_pipe_frac": get("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active") / 100,
            "alu_pipe_frac": get("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active") / 100,
            "issue_active_frac": get("sm__inst_issued.avg.pct_of_peak_sustained_active") / 100,
            "sass_instr_per_candidate": 32 * get("smsp__inst_executed.sum") / cand,
            "source": os.path.basename(path),
        }
    json.dump(out, open("profiles/ncu_summary.json", "w"), indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
