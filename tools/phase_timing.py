"""Per-row phase timing of the advance kernel (debug build lib/libngpulm_timing.so).

Stamps (thread 0 of each row's CTA, kept in shared memory during the row):
0 entry ns, 1 entry clk, 2 after griddepcontrol.wait, 3 levels published,
4 arcs staged, 5 root fix-up barrier, 6 levels written, 7 TMA stores issued,
8 end ns, 9 SM id. Prints medians / p90 / max of each phase in SM cycles.
"""
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
f = synth.make_lm("/tmp/ngpulm_prof", 1024, 6, tokens=430000, seed=1, heldout=4000, tag="bench_6gram")
m = ng.load_arpa(f.arpa, vocab_size=1024, device=0)
m.set_advance_kernel(int(os.environ.get("ADVANCE_KERNEL", "0")))
ctx = synth.sample_contexts(synth.read_sentences(f.heldout), 6, 4096 * 16, seed=2)
allst = np.array([m.state_of(b, t) for b, t in ctx], dtype=np.int32)
stream = torch.cuda.Stream()
h = m.host_arrays()
off, bt = h["arc_offsets"], h["boff_to_states"]


def total_arcs(s):
    T, x = 0, int(s)
    while x != 0:
        T += int(off[x + 1] - off[x])
        x = int(bt[x])
    return T


def phases(B):
    buf = np.zeros(B * 16, dtype=np.uint64)
    assert L.ngpulm_debug_phases(buf.ctypes.data, B * 16) == 0
    return buf.reshape(B, 16).astype(np.int64)


def q(a):
    return f"{int(np.median(a)):6d}/{int(np.percentile(a, 90)):6d}/{int(a.max()):6d}"


def report(tag, ph, Ts=None):
    keep = ph[:, 8] > 0  # rows that carry stamps (warp kernel: warp 0's rows only)
    ph = ph[keep]
    if Ts is not None:
        Ts = Ts[keep]
    names = [("wait", 1, 2), ("st", 2, 10), ("rec", 10, 11), ("bar", 11, 3), ("stage", 3, 4), ("fixup", 4, 5), ("write", 5, 6), ("store", 6, 7)]
    if (ph[:, 12] > 0).all():  # warp kernel: stage = root fill + window loads issued
        names[4:5] = [("fill", 3, 12), ("issue", 12, 4)]
    parts = " ".join(f"{n} {q(ph[:, b] - ph[:, a])}" for n, a, b in names)
    g0 = ph[:, 0].min()
    print(f"{tag}: med/p90/max cycles: {parts} | entry ns {q(ph[:, 0] - g0)} end ns {q(ph[:, 8] - g0)} "
          f"| SMs {len(set(ph[:, 9].tolist()))}", flush=True)
    if Ts is not None:
        end = ph[:, 8] - g0
        slow = np.argsort(-end)[:5]
        print("   slowest rows (T, end ns, stage, write):",
              [(int(Ts[i]), int(end[i]), int(ph[i, 4] - ph[i, 3]), int(ph[i, 6] - ph[i, 5])) for i in slow])


for B in (1, 128, 1024, 4096):
    R = 16
    st = torch.from_numpy(allst[: R * B].reshape(R, B)).cuda()
    sc = torch.empty((R, B, 1024), dtype=torch.float32, device="cuda")
    nx = torch.empty((R, B, 1024), dtype=torch.int32, device="cuda")
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
    with torch.cuda.stream(stream):
        g.replay()
        e0.record(stream); g.replay(); e1.record(stream)
    stream.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / n
    report(f"B={B:5d} graph {us:6.2f}us/call", phases(B))
    with torch.cuda.stream(stream):
        m.advance(st[0], sc[0], nx[0], want_final=False, stream=stream)
    stream.synchronize()
    Ts = np.array([total_arcs(x) for x in allst[:B]]) if B <= 1024 else None
    report(f"B={B:5d} single          ", phases(B), Ts)
    with torch.cuda.stream(stream):
        m.advance(st[0], sc[0], nx[0], want_final=False, stream=stream)
    stream.synchronize()
    report(f"B={B:5d} single, repeat  ", phases(B))

# probe: the same two dependent loads on the model's own data, in isolation
L.ngpulm_debug_probe_model.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_void_p]
for B in (128, 1024):
    st = torch.from_numpy(allst[:B].copy()).cuda()
    o = torch.zeros(B * 3, dtype=torch.int64, device="cuda")
    for _ in range(2):
        L.ngpulm_debug_probe_model(m._h, st.data_ptr(), B, o.data_ptr())
    r = o.view(B, 3).cpu().numpy()
    print(f"probe B={B}: states load {q(r[:, 0])}  record load {q(r[:, 1])}")

# bisect: the same single launch without the TMA prologue
L.ngpulm_debug_skip.argtypes = [C.c_int]
L.ngpulm_debug_skip(1)
for B in (128, 1024):
    st = torch.from_numpy(allst[:B].copy()).cuda()
    sc = torch.empty((B, 1024), dtype=torch.float32, device="cuda")
    nx = torch.empty((B, 1024), dtype=torch.int32, device="cuda")
    for _ in range(2):
        m.advance(st, sc, nx, want_final=False)
        torch.cuda.synchronize()
    report(f"B={B:5d} single, no TMA prologue", phases(B))
L.ngpulm_debug_skip(0)
