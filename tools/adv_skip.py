"""What limits the advance call? Per-call time (CUDA graph, rotating buffers) of
the debug build with phases switched off (g_skip bits: 2 no bulk stores, 4 no arc
gathers/writes, 8 no root fill), for B = 128, 1024, 4096. Timing only: the
skipped variants compute wrong rows."""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["NGPULM_LIB"] = os.path.join(ROOT, "paper_2505_22857_b200", "lib", "libngpulm_timing.so")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2505_22857_b200 as ng  # noqa: E402
import synth  # noqa: E402

L = ng.lib()
L.ngpulm_debug_skip.argtypes = [C.c_int]
f = synth.make_lm("/tmp/ngpulm_prof", 1024, 6, tokens=430000, seed=1, heldout=4000, tag="bench_6gram")
m = ng.load_arpa(f.arpa, vocab_size=1024, device=0)
ctx = synth.sample_contexts(synth.read_sentences(f.heldout), 6, 4096 * 16, seed=2)
allst = np.array([m.state_of(b, t) for b, t in ctx], dtype=np.int32)
stream = torch.cuda.Stream()
for B in (128, 1024, 4096):
    R = 16
    st = torch.from_numpy(allst[: R * B].reshape(R, B)).cuda()
    sc = torch.empty((R, B, 1024), dtype=torch.float32, device="cuda")
    nx = torch.empty((R, B, 1024), dtype=torch.int32, device="cuda")
    out = []
    for skip in (0, 2, 4, 8, 12, 14):
        L.ngpulm_debug_skip(skip)
        g = torch.cuda.CUDAGraph()
        n = 64
        with torch.cuda.stream(stream):
            for k in range(3):
                m.advance(st[k % R], sc[k % R], nx[k % R], want_final=False, stream=stream)
            stream.synchronize()
            with torch.cuda.graph(g, stream=stream):
                for k in range(n):
                    m.advance(st[k % R], sc[k % R], nx[k % R], want_final=False, stream=stream)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ts = []
        for rep in range(3):
            with torch.cuda.stream(stream):
                e0.record(stream); g.replay(); e1.record(stream)
            stream.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3 / n)
        out.append(f"skip{skip}={min(ts):.2f}")
    L.ngpulm_debug_skip(0)
    print(f"B={B}: us/call " + " ".join(out), flush=True)
