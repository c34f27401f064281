"""configs[3] / configs[4] advance launches for ncu (cold and warm trie): the bench's LMs
(8-gram ~4.9M n-grams, 10-gram ~20M n-grams), trajectory states, `--iters` advance calls.

    ncu [--cache-control all|none] -k regex:advance -s S -c 1 python tools/prof_large.py --cfg 4
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2505_22857_b200 as ng  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--cfg", type=int, default=4, choices=[3, 4])
p.add_argument("--iters", type=int, default=6)
p.add_argument("--dependent", action="store_true")
a = p.parse_args()
key, B = ("cfg4", 4096) if a.cfg == 4 else ("cfg3", 512)
files, nglm = bench.lm_files("/tmp/ngpulm_bench", key, 0, 1, lambda: None)
m = ng.load_binary(nglm, device=0)
st = torch.from_numpy(bench.trajectory(m, files, B * a.iters, seed=31).reshape(a.iters, B)).cuda()
sc = torch.empty((B, m.V), dtype=torch.float32, device="cuda")
nx = torch.empty((B, m.V), dtype=torch.int32, device="cuda")
fi = torch.empty(B, dtype=torch.float32, device="cuda")
for i in range(a.iters):
    m.advance(st[i], sc, nx, fi, independent=not a.dependent)
torch.cuda.synchronize()
print(f"cfg{a.cfg} B={B}: {a.iters} advance calls, check {m.check()}", flush=True)
