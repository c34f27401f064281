"""What the advance kernel costs with steps switched off (debug build): per-call
us in a CUDA graph (B=1024, rotating outputs) and single-launch phase medians."""
import ctypes as C
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["NGPULM_LIB"] = os.path.join(ROOT, "paper_2505_22857_b200", "lib", "libngpulm_timing.so")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2505_22857_b200 as ng  # noqa: E402
import synth  # noqa: E402

L = ng.lib()
L.ngpulm_debug_phases.argtypes = [C.c_void_p, C.c_int]
pass
pass
f = synth.make_lm("/tmp/ngpulm_prof", 1024, 6, tokens=430000, seed=1, heldout=4000, tag="bench_6gram")
m = ng.load_arpa(f.arpa, vocab_size=1024, device=0)
ctx = synth.sample_contexts(synth.read_sentences(f.heldout), 6, 1024 * 16, seed=2)
allst = np.array([m.state_of(b, t) for b, t in ctx], dtype=np.int32)
stream = torch.cuda.Stream()
B, R, n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024, 16, 200
st = torch.from_numpy(allst[: R * B].reshape(R, B)).cuda()
sc = torch.empty((R, B, 1024), dtype=torch.float32, device="cuda")
nx = torch.empty((R, B, 1024), dtype=torch.int32, device="cuda")
for skip in (0, 1, 2, 3):
    L.ngpulm_debug_skip(skip)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(stream):
        for k in range(3):
            m.advance(st[k], sc[k], nx[k], want_final=False, stream=stream)
        stream.synchronize()
        with torch.cuda.graph(g, stream=stream):
            for k in range(n):
                m.advance(st[k % R], sc[k % R], nx[k % R], want_final=False, stream=stream)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(3):
        with torch.cuda.stream(stream):
            e0.record(stream); g.replay(); e1.record(stream)
        stream.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3 / n)
    m.advance(st[0], sc[0], nx[0], want_final=False)
    torch.cuda.synchronize()
    buf = np.zeros(B * 8, dtype=np.uint64)
    L.ngpulm_debug_phases(buf.ctypes.data, B * 8)
    ph = buf.reshape(B, 8).astype(np.int64)
    d = lambda a, b: int(np.median(ph[:, b] - ph[:, a]))
    mx = lambda a, b: int(np.max(ph[:, b] - ph[:, a]))
    end = ph[:, 7] - ph[:, 0].min()
    ex = np.zeros(B * 4, dtype=np.uint64)
    L.ngpulm_debug_extra(ex.ctypes.data, B * 4)
    ex = ex.reshape(B, 4).astype(np.int64)
    print(f"   states load {int(np.median(ex[:,1]-ex[:,0]))} (max {int(np.max(ex[:,1]-ex[:,0]))}), "
          f"record+levels {int(np.median(ex[:,2]-ex[:,1]))} (max {int(np.max(ex[:,2]-ex[:,1]))}), "
          f"barrier {int(np.median(ex[:,3]-ex[:,2]))} cycles")
    print(f"skip={skip}: graph {statistics.median(ts):6.2f} us/call | single: prologue+wait {d(1,2)} levels {d(2,5)} "
          f"(max {mx(2,5)}) scatter {d(5,4)} (max {mx(5,4)}) output {d(4,6)} (max {mx(4,6)}) cycles; "
          f"end med {np.median(end):.0f} max {end.max()} ns", flush=True)
