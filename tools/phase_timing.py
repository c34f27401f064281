"""Per-CTA phase timing of the advance kernel (debug build lib/libngpulm_timing.so).
Phases (clock64 cycles since CTA entry): 2 after griddepcontrol.wait, 5 levels
loaded, 3 pass-1 scatter done, 4 pass-2 done, 6 stores issued; globaltimer at
entry (0) and end (7) for the cross-CTA picture."""
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
ctx = synth.sample_contexts(synth.read_sentences(f.heldout), 6, 4096 * 16, seed=2)
allst = np.array([m.state_of(b, t) for b, t in ctx], dtype=np.int32)
stream = torch.cuda.Stream()


def phases(B):
    buf = np.zeros(B * 8, dtype=np.uint64)
    assert L.ngpulm_debug_phases(buf.ctypes.data, B * 8) == 0
    return buf.reshape(B, 8).astype(np.int64)


def report(tag, ph):
    cyc = {k: ph[:, k] - ph[:, 1] for k in (2, 5, 4, 6)}
    ent = ph[:, 0] - ph[:, 0].min()
    end = ph[:, 7] - ph[:, 0].min()
    q = lambda a: f"{int(np.median(a)):6d}/{int(np.percentile(a, 90)):6d}/{int(a.max()):6d}"
    print(f"{tag}: cycles since entry (med/p90/max) wait {q(cyc[2])} levels {q(cyc[5])} "
          f"gather {q(cyc[4])} stores {q(cyc[6])} | entry spread ns {q(ent)} end ns {q(end)} "
          f"| SMs used {len(set(ph[:, 3].tolist()))}", flush=True)


for mode, name in ((ng.CHAIN_TABLE, "table"), (ng.CHAIN_WALK, "walk")):
    m.set_chain_mode(mode)
    for B in (1, 16, 128, 1024, 4096):
        R = 16
        st = torch.from_numpy(allst[: R * B].reshape(R, B)).cuda()
        sc = torch.empty((R, B, 1024), dtype=torch.float32, device="cuda")
        nx = torch.empty((R, B, 1024), dtype=torch.int32, device="cuda")
        fi = torch.empty((R, B), dtype=torch.float32, device="cuda")
        g = torch.cuda.CUDAGraph()
        n = 64
        with torch.cuda.stream(stream):
            for k in range(3):
                m.advance(st[k % R], sc[k % R], nx[k % R], fi[k % R], stream=stream)
            stream.synchronize()
            with torch.cuda.graph(g, stream=stream):
                for k in range(n):
                    m.advance(st[k % R], sc[k % R], nx[k % R], fi[k % R], stream=stream)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            g.replay()
            e0.record(stream); g.replay(); e1.record(stream)
        stream.synchronize()
        report(f"{name} B={B:5d} graph {e0.elapsed_time(e1)*1e3/n:6.2f}us/call", phases(B))
        with torch.cuda.stream(stream):
            m.advance(st[0], sc[0], nx[0], fi[0], stream=stream)
        stream.synchronize()
        report(f"{name} B={B:5d} single           ", phases(B))

# torch floor: graph of tiny fills
for nbytes in (8 << 10, 8 << 20):
    x = torch.empty(nbytes // 4, dtype=torch.float32, device="cuda")
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(stream):
        x.fill_(1.0); stream.synchronize()
        with torch.cuda.graph(g, stream=stream):
            for k in range(64):
                x.fill_(float(k))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        g.replay(); e0.record(stream); g.replay(); e1.record(stream)
    stream.synchronize()
    print(f"torch fill_ {nbytes} B graph: {e0.elapsed_time(e1)*1e3/64:.2f} us/node")


# ---- tail analysis: which rows are slow in a single launch (B=1024, table)?
h = m.host_arrays()
off, bt = h["arc_offsets"], h["boff_to_states"]


def chain_stats(s):
    T, nl, x = 0, 0, int(s)
    while x != 0:
        c = int(off[x + 1] - off[x])
        T += c
        nl += c > 0
        x = int(bt[x])
    return T, nl


m.set_chain_mode(ng.CHAIN_TABLE)
B = 1024
st = torch.from_numpy(allst[:B].copy()).cuda()
sc = torch.empty((B, 1024), dtype=torch.float32, device="cuda")
nx = torch.empty((B, 1024), dtype=torch.int32, device="cuda")
for rep in range(3):
    m.advance(st, sc, nx)
    torch.cuda.synchronize()
    ph = phases(B)
    g0 = ph[:, 0].min()
    end = ph[:, 7] - g0
    gat = ph[:, 4] - ph[:, 5]
    lev = ph[:, 5] - ph[:, 2]
    order = np.argsort(-end)[:12]
    print(f"rep {rep}: end med {np.median(end):.0f} ns max {end.max()} ns")
    for i in order:
        T, nl = chain_stats(allst[i])
        print(f"  row {i:4d} state {allst[i]:7d} T {T:5d} nlev {nl} sm {ph[i,3]:3d} entry {ph[i,0]-g0:5d}ns "
              f"levels {lev[i]:6d} gather {gat[i]:6d} store {ph[i,6]-ph[i,4]:6d} end {end[i]}ns")
    Ts = np.array([chain_stats(x)[0] for x in allst[:B]])
    print("  corr(T, gather cycles) = %.3f; gather med for T<500: %.0f, T>1000: %.0f" % (
        np.corrcoef(Ts, gat)[0, 1], np.median(gat[Ts < 500]), np.median(gat[Ts > 1000]) if (Ts > 1000).any() else -1))
