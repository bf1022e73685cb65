#!/bin/bash
# Compile alp_search_u.cu alone (same flags as build.py) and print k_search_u's registers and uniform FADD2 count.
set -e
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -ftz=false -prec-div=true -prec-sqrt=true -Xptxas -v ${EXTRA:-} -c paper_2604_15186_b200/csrc/alp_search_u.cu -o /tmp/qs.o 2> /tmp/qs.ptxas
grep -A3 "k_search_uILi4ELb1" /tmp/qs.ptxas | grep Used
python tools/sass_check.py /tmp/qs.o | grep -E "ILi4ELb1|ILi16ELb0"
