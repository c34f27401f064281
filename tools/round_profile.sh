#!/bin/bash
# One GPU call: smoke, GPU tests, the bench line, the bench's launch list, a
# graph-level ncu capture of the timed advance regime (256 calls in one CUDA
# graph, outputs rotating over 512 MiB), full ncu captures of the advance,
# fused-step and decode kernels, and the fused-step phase / loop-floor
# microbenchmarks. Outputs under gpurun_out/.
set -x
TAG=${TAG:-r02}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1
tail -2 gpurun_out/smoke_$TAG.log
if [ -z "$NO_TESTS" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$TAG.log 2>&1
  tail -3 gpurun_out/pytest_gpu_$TAG.log
fi
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
tail -2 gpurun_out/bench_$TAG.err; cat gpurun_out/bench_$TAG.json
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 300 --csv \
    --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 50 --warmup 5 --no-cpu --no-fused --no-large > /dev/null 2>&1
timeout 600 ncu --graph-profiling graph --clock-control none \
    --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_sector_hit_rate.pct \
    --csv --log-file gpurun_out/graph_$TAG.csv python tools/prof_advance.py --batch 1024 --graph 256 --iters 3 > /dev/null 2>&1
timeout 600 ncu --graph-profiling graph --clock-control none \
    --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_sector_hit_rate.pct \
    --csv --log-file gpurun_out/graph_indep_$TAG.csv python tools/prof_advance.py --batch 1024 --graph 256 --iters 3 --independent > /dev/null 2>&1
cat gpurun_out/graph_$TAG.csv | tail -4; cat gpurun_out/graph_indep_$TAG.csv | tail -4
timeout 600 ncu --set full --clock-control none --import-source on -k regex:advance_warp -s 10 -c 1 \
    -o gpurun_out/adv_$TAG -f python tools/prof_advance.py --batch 1024 > gpurun_out/ncu_full_$TAG.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fused_warp -s 10 -c 1 \
    -o gpurun_out/fused_ctc_$TAG -f python tools/prof_advance.py --batch 256 --mode ctc > gpurun_out/ncu_fused_$TAG.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:ctc_ --csv \
    --log-file gpurun_out/decode_launches_$TAG.csv python tools/prof_advance.py --batch 256 --mode decode --iters 4 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ctc_seg -s 4 -c 2 \
    -o gpurun_out/decode_$TAG -f python tools/prof_advance.py --batch 256 --mode decode --iters 4 > gpurun_out/ncu_decode_$TAG.log 2>&1
python -c "from paper_2505_22857_b200 import _build; _build.build_phase_timing()" > /dev/null 2>&1
( python tools/fused_phases.py; NET=1 python tools/fused_phases.py ) > gpurun_out/fused_phases_$TAG.txt 2>&1
python tools/loop_floor.py > gpurun_out/loop_floor_$TAG.txt 2>&1
cat gpurun_out/fused_phases_$TAG.txt gpurun_out/loop_floor_$TAG.txt
