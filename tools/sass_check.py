"""SASS sanity check of the search kernels (run here, no GPU): per kernel the registers, the
instruction count, FADD2 total and FADD2 with a uniform-register operand (the uniform datapath
ptxas may silently drop), LDCU, spills.

    python tools/sass_check.py [object or .so] [name-filter]
"""
import re
import subprocess
import sys

obj = sys.argv[1] if len(sys.argv) > 1 else "paper_2604_15186_b200/lib/alp_search_u.o"
flt = sys.argv[2] if len(sys.argv) > 2 else "k_search_u"
out = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s*Function : ", out)
for f in funcs[1:]:
    name = f.split("\n", 1)[0].strip()
    if flt not in name:
        continue
    body = [ln for ln in f.split("\n") if re.match(r"\s*/\*[0-9a-f]{4,}\*/", ln)]
    ins = [ln.split("*/", 1)[1].strip() for ln in body]
    fadd2 = [i for i in ins if "FADD2" in i]
    print(f"{name[:70]:70s} instr {len(ins):5d} FADD2 {len(fadd2):4d} FADD2.UR {sum(1 for i in fadd2 if re.search(r'\bUR\d', i)):4d} "
          f"LDCU {sum(1 for i in ins if i.startswith('LDCU') or ' LDCU' in i):4d} "
          f"STL {sum(1 for i in ins if 'STL' in i):3d}")
