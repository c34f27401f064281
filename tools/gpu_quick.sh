#!/bin/bash
# Scratch GPU check: build, selected tests (outputs under gpurun_out/).
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build2.log 2>&1
tail -3 gpurun_out/build2.log
timeout 900 python -m pytest tests/test_gpu_transducer.py -x -q > gpurun_out/pytest_tr.log 2>&1
tail -30 gpurun_out/pytest_tr.log
timeout 900 python -m pytest tests -m gpu -x -q --deselect tests/test_gpu_large.py > gpurun_out/pytest_all.log 2>&1
tail -5 gpurun_out/pytest_all.log
timeout 600 python bench.py --steps 200 --warmup 10 --no-cpu > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err
tail -3 gpurun_out/bench_q.err
python -c "import json; d=json.load(open('gpurun_out/bench_q.json')); print(d['fused_step_us'])"
