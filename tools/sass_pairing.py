"""Static schedule check of the hottest FADD2/FMNMX3 loop of k_search_u: how often an FADD2 follows an
FADD2 (both need the FMA pipe for 2 cycles: back-to-back pairs from one warp stall at dispatch) and
how often an FMNMX3 follows an FMNMX3.  python tools/sass_pairing.py obj [name-filter]"""
import re
import subprocess
import sys

obj = sys.argv[1]
flt = sys.argv[2] if len(sys.argv) > 2 else "k_search_uILi4ELb1"
out = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
for f in re.split(r"\n\s*Function : ", out)[1:]:
    if flt not in f.split("\n", 1)[0]:
        continue
    ins = []
    for ln in f.split("\n"):
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s*(.*?);", ln)
        if m:
            ins.append((int(m.group(1), 16), m.group(2).strip()))
    addr = {a: i for i, (a, _) in enumerate(ins)}
    for i, (a, t) in enumerate(ins):
        m = re.search(r"BRA(?:\.U)?\s.*?0x([0-9a-f]+)\s*$", t)
        if not m or int(m.group(1), 16) >= a or int(m.group(1), 16) not in addr:
            continue
        body = [x for _, x in ins[addr[int(m.group(1), 16)]:i + 1]]
        if len(body) > 600 or sum("FMNMX3" in x for x in body) < 100:
            continue
        ops = ["A" if x.startswith("FADD2") else "M" if x.startswith("FMNMX3") else "o" for x in body]
        aa = sum(1 for p, q in zip(ops, ops[1:]) if p == q == "A")
        mm = sum(1 for p, q in zip(ops, ops[1:]) if p == q == "M")
        print(f"loop {int(m.group(1), 16):#07x} len {len(body)}: FADD2->FADD2 {aa}, FMNMX3->FMNMX3 {mm}")
