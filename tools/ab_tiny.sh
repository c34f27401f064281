#!/bin/bash
for rep in 1 2; do for v in "$@"; do echo "== $v"; NGPULM_LIB=$PWD/paper_2505_22857_b200/lib/libngpulm$v.so python tools/tiny_sweep.py 2>&1 | tail -1; done; done
