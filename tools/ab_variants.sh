for rep in 1 2; do
for v in "" _st0 _st1184; do echo "== $v"; NGPULM_LIB=$PWD/paper_2505_22857_b200/lib/libngpulm$v.so SWEEP_QUICK=1 SWEEP_KERNELS=0 python tools/adv_sweep.py 2>&1 | grep -v "^lib\|^B,"; done
done
