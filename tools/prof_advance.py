"""Profiling driver: the bench's advance launch (6-gram, V=1024, B trajectory rows).
Run under ncu on the GPU box, e.g.
  ncu --set full --clock-control none --import-source on -k regex:advance -s 10 -c 3 \
      -o gpurun_out/prof_adv python tools/prof_advance.py
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2505_22857_b200 as ng  # noqa: E402
import synth  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--batch", type=int, default=1024)
p.add_argument("--iters", type=int, default=20)
p.add_argument("--mode", default="advance", choices=["advance", "ctc", "rnnt", "aed", "decode"])
p.add_argument("--graph", type=int, default=0,
               help="advance: capture this many calls in one CUDA graph (outputs rotating over 64 sets = "
                    "512 MiB at B=1024, as bench.py) and replay it --iters times; for ncu --graph-profiling graph")
p.add_argument("--independent", action="store_true", help="advance calls with NGPULM_ADVANCE_INDEPENDENT")
a = p.parse_args()
f = synth.make_lm("/tmp/ngpulm_prof", 1024, 6, tokens=430000, seed=1, heldout=4000, tag="bench_6gram")
m = ng.load_arpa(f.arpa, vocab_size=1024, device=0)
ctx = synth.sample_contexts(synth.read_sentences(f.heldout), 6, a.batch * 4, seed=2)
st_np = np.array([m.state_of(b, t) for b, t in ctx], dtype=np.int32).reshape(4, a.batch)
st = torch.from_numpy(st_np).cuda()
if a.mode == "advance" and a.graph:
    R = 64
    ctx = synth.sample_contexts(synth.read_sentences(f.heldout), 6, a.batch * R, seed=2)
    st = torch.from_numpy(np.array([m.state_of(b, t) for b, t in ctx], dtype=np.int32).reshape(R, a.batch)).cuda()
    sc = torch.empty((R, a.batch, 1024), dtype=torch.float32, device="cuda")
    nx = torch.empty((R, a.batch, 1024), dtype=torch.int32, device="cuda")
    fi = torch.empty((R, a.batch), dtype=torch.float32, device="cuda")
    s_ = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s_):
        for i in range(3):
            m.advance(st[i % R], sc[i % R], nx[i % R], fi[i % R], stream=s_, independent=a.independent)
        s_.synchronize()
        with torch.cuda.graph(g, stream=s_):
            for i in range(a.graph):
                m.advance(st[i % R], sc[i % R], nx[i % R], fi[i % R], stream=s_, independent=a.independent)
        for _ in range(a.iters):
            g.replay()
    s_.synchronize()
elif a.mode == "advance":
    sc = torch.empty((4, a.batch, 1024), dtype=torch.float32, device="cuda")
    nx = torch.empty((4, a.batch, 1024), dtype=torch.int32, device="cuda")
    fi = torch.empty((4, a.batch), dtype=torch.float32, device="cuda")
    for i in range(a.iters):
        m.advance(st[i % 4], sc[i % 4], nx[i % 4], fi[i % 4], independent=a.independent)
elif a.mode == "decode":  # persistent CTC decode, BASELINE configs[2] shape
    T = 500
    x = torch.from_numpy(synth.ctc_logits(synth.read_sentences(f.heldout), a.batch, T, 1024, seed=4)).cuda()
    for i in range(a.iters):
        s = torch.zeros(a.batch, dtype=torch.int32, device="cuda")
        pv = torch.full((a.batch,), -1, dtype=torch.int32, device="cuda")
        m.ctc_greedy_decode(x, s, pv, lam=0.3)
else:
    mode = {"ctc": ng.CTC, "rnnt": ng.RNNT, "aed": ng.AED}[a.mode]
    x = torch.from_numpy(synth.rnnt_logits(a.batch, 4, 1024, seed=4)).cuda()
    pv = torch.full((a.batch,), -1, dtype=torch.int32, device="cuda")
    for i in range(a.iters):
        s = st[i % 4].clone()
        m.fused_greedy_step(mode, x[i % 4], s, prev=pv, lam=0.3)
torch.cuda.synchronize()
print("done")
