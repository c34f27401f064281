#!/bin/bash
# Round-end style check on a fresh box: build, smoke, all GPU tests, the default bench line.
set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/final_smoke.log 2>&1
tail -1 gpurun_out/final_smoke.log
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/final_pytest.log 2>&1
tail -1 gpurun_out/final_pytest.log
timeout 900 python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err
cat gpurun_out/final_bench.json | cut -c1-600
