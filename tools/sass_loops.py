"""List the loops (backward branches) of a kernel's SASS with their size and FADD2 operand kinds:
    python tools/sass_loops.py obj [name-filter]
Loop = [branch target, branch]; FADD2.UR = FADD2 with a uniform-register operand."""
import re
import subprocess
import sys

obj = sys.argv[1]
flt = sys.argv[2] if len(sys.argv) > 2 else "k_search_uILi4ELb1"
out = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
for f in re.split(r"\n\s*Function : ", out)[1:]:
    name = f.split("\n", 1)[0].strip()
    if flt not in name:
        continue
    ins = []
    for ln in f.split("\n"):
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s*(.*?);", ln)
        if m:
            ins.append((int(m.group(1), 16), m.group(2)))
    addr = {a: i for i, (a, _) in enumerate(ins)}
    print(name[:80], "instructions", len(ins))
    for i, (a, t) in enumerate(ins):
        m = re.search(r"BRA(?:\.U)?\s.*?0x([0-9a-f]+)\s*$", t)
        if not m:
            continue
        tgt = int(m.group(1), 16)
        if tgt >= a or tgt not in addr:
            continue
        body = [x for _, x in ins[addr[tgt]:i + 1]]
        fa = [x for x in body if "FADD2" in x]
        ur = sum(1 for x in fa if re.search(r"\bUR\d", x))
        print(f"  loop {tgt:#07x}-{a:#07x}: {len(body):5d} instr ({len(body) * 16 / 1024:5.1f} KB)  FADD2 {len(fa):4d} (UR {ur:4d})  "
              f"FMNMX3 {sum(1 for x in body if 'FMNMX3' in x):4d}  LDCU {sum(1 for x in body if 'LDCU' in x):3d}  LDC {sum(1 for x in body if re.match(r'LDC[ .]', x.split(' ', 1)[-1]) or x.startswith('LDC ') or x.startswith('LDC.')):3d}")
