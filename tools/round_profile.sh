#!/bin/bash
# One GPU call: GPU tests, the bench line, the bench's launch list, and full
# ncu captures of the advance and fused-step kernels. Outputs under gpurun_out/.
set -x
TAG=${TAG:-r01}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1
tail -2 gpurun_out/smoke_$TAG.log
if [ -z "$NO_TESTS" ]; then
  timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$TAG.log 2>&1
  tail -3 gpurun_out/pytest_gpu_$TAG.log
fi
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
tail -2 gpurun_out/bench_$TAG.err; cat gpurun_out/bench_$TAG.json
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 300 --csv \
    --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 50 --warmup 5 --no-cpu --no-fused > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:advance_warp -s 10 -c 1 \
    -o gpurun_out/adv_$TAG -f python tools/prof_advance.py --batch 1024 > gpurun_out/ncu_full_$TAG.log 2>&1
tail -3 gpurun_out/ncu_full_$TAG.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fused_warp -s 10 -c 1 \
    -o gpurun_out/fused_ctc_$TAG -f python tools/prof_advance.py --batch 256 --mode ctc > gpurun_out/ncu_fused_$TAG.log 2>&1
tail -3 gpurun_out/ncu_fused_$TAG.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ctc_decode -s 2 -c 1 \
    -o gpurun_out/decode_$TAG -f python tools/prof_advance.py --batch 256 --mode decode --iters 4 > gpurun_out/ncu_decode_$TAG.log 2>&1
tail -3 gpurun_out/ncu_decode_$TAG.log
