#!/bin/bash
# Scratch GPU check: build, selected tests, phase timing, a short bench (outputs under gpurun_out/).
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build2.log 2>&1
timeout 900 python -m pytest tests/test_gpu_ctc_decode.py -x -q > gpurun_out/pytest_decode.log 2>&1
tail -3 gpurun_out/pytest_decode.log
python tools/decode_timing.py
timeout 1500 python -m pytest tests/test_gpu_large.py -x -q --durations=10 > gpurun_out/pytest_large.log 2>&1
tail -20 gpurun_out/pytest_large.log
