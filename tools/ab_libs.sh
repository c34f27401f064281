#!/bin/bash
# A/B of library variants on the advance sweep (graph us/call), twice each.
for rep in 1 2; do
for v in "$@"; do echo "== $v"; NGPULM_LIB=$PWD/paper_2505_22857_b200/lib/libngpulm$v.so SWEEP_QUICK=1 SWEEP_KERNELS=0 python tools/adv_sweep.py 2>&1 | grep -v "^lib\|^B,"; done
done
