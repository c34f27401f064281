#!/bin/bash
# One GPU call: bench line, the bench's launch list, and a full ncu capture of
# the advance kernel. Outputs under gpurun_out/.
set -x
TAG=${TAG:-r01}
python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
tail -2 gpurun_out/bench_$TAG.err
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 300 --csv \
    --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 50 --warmup 5 --no-cpu --no-fused > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:advance_warp -s 10 -c 1 \
    -o gpurun_out/adv_$TAG -f python tools/prof_advance.py --batch 1024 > gpurun_out/ncu_full_$TAG.log 2>&1
tail -3 gpurun_out/ncu_full_$TAG.log
