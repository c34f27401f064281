#!/bin/bash
# Scratch GPU check: build, selected tests (outputs under gpurun_out/).
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build2.log 2>&1
timeout 900 python -m pytest tests/test_gpu_fusion_ext.py -x -q > gpurun_out/pytest_ext.log 2>&1
tail -30 gpurun_out/pytest_ext.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ctc_decode.py -x -q > gpurun_out/pytest_par.log 2>&1
tail -5 gpurun_out/pytest_par.log
