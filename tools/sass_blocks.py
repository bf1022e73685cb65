"""Straight-line SASS blocks of a kernel by executed warp-instructions (from an ncu source page).

    ncu -i rep.ncu-rep --page source --csv --print-source sass > sass.csv
    python tools/sass_blocks.py sass.csv [--candidates N] [--top 30]

A block = consecutive instructions with the same 'Instructions Executed' count.  Prints each
block's start offset, executions, length, share of all warp-instructions and opcode histogram,
plus thread-instructions per candidate when --candidates is given.
"""
import argparse
import collections
import csv


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--candidates", type=float, default=0)
    ap.add_argument("--top", type=int, default=30)
    args = ap.parse_args()
    rows = list(csv.reader(open(args.csv)))
    hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    hdr = rows[hdr_i]
    ci = hdr.index("Instructions Executed")
    si = hdr.index("Source")
    ins = []
    for r in rows[hdr_i + 1:]:
        if len(r) <= ci or not r[0].startswith("0x"):
            continue
        try:
            n = int(r[ci])
        except ValueError:
            continue
        op = [o for o in r[si].strip().split() if not o.startswith("@")]
        ins.append((int(r[0], 16), n, op[0].split(".")[0] if op else "?"))
    blocks = []
    for addr, n, op in ins:
        if blocks and blocks[-1]["n"] == n and n > 0:
            blocks[-1]["len"] += 1
            blocks[-1]["ops"][op] += 1
        else:
            blocks.append({"addr": addr, "n": n, "len": 1, "ops": collections.Counter({op: 1})})
    total = sum(b["n"] * b["len"] for b in blocks)
    base = ins[0][0] if ins else 0
    line = f"total warp-instructions {total}"
    if args.candidates:
        line += f" = {32 * total / args.candidates:.3f} thread-instructions per candidate"
    print(line)
    for b in sorted(blocks, key=lambda b: -b["n"] * b["len"])[:args.top]:
        share = b["n"] * b["len"] / max(1, total)
        print(f"+{b['addr'] - base:05x} execs {b['n']:9d} len {b['len']:4d} share {100 * share:5.1f}%  "
              f"{dict(b['ops'].most_common(8))}")


if __name__ == "__main__":
    main()
