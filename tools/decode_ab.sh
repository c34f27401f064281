#!/bin/bash
# Persistent CTC decode: per-chain phase cycles (timing build) and A/B of library variants
# (decode ms at configs[2]); libraries prebuilt in-tree. Usage: bash tools/decode_ab.sh _ring2 _ring3 ...
mkdir -p gpurun_out
[ -z "$NO_TIMING" ] && NGPULM_LIB=$PWD/paper_2505_22857_b200/lib/libngpulm_timing.so timeout 300 python tools/seg_timing.py 2>&1 | grep -v Warn
for rep in 1 2; do
for v in "" "$@"; do echo "== lib$v"; NGPULM_LIB=$PWD/paper_2505_22857_b200/lib/libngpulm$v.so timeout 300 python tools/decode_sweep.py 2>&1 | tail -1; done
done
