"""configs[4] advance (10-gram ~20M n-grams, B=4096, one GPU) us/call, independent and dependent
calls, for the library NGPULM_LIB selects (A/B of advance build variants on the DRAM-resident LM)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2505_22857_b200 as ng  # noqa: E402

t0 = time.perf_counter()
files, nglm = bench.lm_files("/tmp/ngpulm_bench", "cfg4", 0, 1, lambda: None)
m = ng.load_binary(nglm, device=0)
B, V, R = 4096, 1024, 4
allst = bench.trajectory(m, files, B * R, seed=31).reshape(R, B)
st = torch.from_numpy(allst).cuda()
sc = torch.empty((R, B, V), dtype=torch.float32, device="cuda")
nx = torch.empty((R, B, V), dtype=torch.int32, device="cuda")
fi = torch.empty((R, B), dtype=torch.float32, device="cuda")
stream = torch.cuda.Stream()
for ind in (True, False):
    us = bench.window_ms(lambda k: m.advance(st[k % R], sc[k % R], nx[k % R], fi[k % R], stream=stream,
                                             independent=ind), 128, stream, reps=7) * 1e3 / 128
    print(f"{os.path.basename(os.environ.get('NGPULM_LIB', 'libngpulm.so'))} {'indep' if ind else 'dep'}: "
          f"{us:.2f} us/call = {8 * B * V / (us * 1e-6) / 1e9:.0f} GB/s (setup {time.perf_counter() - t0:.0f} s)",
          flush=True)
torch.cuda.synchronize()
s1, n1, f1 = m.advance(st[0])
torch.cuda.synchronize()
print("digest", int(s1.view(torch.int32).sum()), int(n1.sum()), flush=True)
