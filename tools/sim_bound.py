"""CPU estimate (oracle rows) of how often the bound-based CTC frame decision
(decode v2) decides a frame without the candidates' LM values
(level 0), with the top-2 candidates' exact values (level 1), or needs the
full row (level 2), on the bench's configs[2] CTC logits."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
from oracle import Oracle
import paper_2505_22857_b200 as ng

f = synth.make_lm("/tmp/ngpulm_prof", 1024, 6, tokens=430000, seed=1, heldout=4000, tag="bench_6gram")
V, T, B, lam = 1024, 500, int(os.environ.get("B", 16)), 0.3
o = Oracle(f.arpa, vocab_size=V)
h = ng.load_arpa(f.arpa, vocab_size=V, device=-1).host_arrays()
off, bt, bw, w = (np.asarray(h[k]) for k in ("arc_offsets", "boff_to_states", "boff_weights", "arc_weights"))
S = len(off) - 1
maxw = np.full(S, -np.inf, np.float32)
nz = np.diff(off) > 0
maxw[nz] = np.maximum.reduceat(w, off[:-1][nz])
ub = np.full(S, -np.inf, np.float32); acc = np.zeros(S, np.float32); cur = np.arange(S)
for _ in range(12):
    m = cur != 0
    ub[m] = np.maximum(ub[m], (acc[m] + maxw[cur[m]]).astype(np.float32))
    acc[m] = (acc[m] + bw[cur[m]]).astype(np.float32)
    cur = np.where(m, bt[cur], 0)
ub = np.maximum(ub, (acc + maxw[0]).astype(np.float32))
x = synth.ctc_logits(synth.read_sentences(f.heldout), B, T, V, seed=4)
sp = V
cnt = np.zeros(3, np.int64); emis = 0
for b in range(B):
    st, pc = 0, -1
    for t in range(T):
        row, _, nxt, _ = o.rows(np.array([st], np.int32), want64=False) if False else (None, None, None, None)
        s32, _, n_o, _ = o.rows(np.array([st], np.int32), want64=False)
        lm = np.append(s32[0], np.float32(0))  # column sp = V: blank, lm 0
        xr = x[b, t]
        val = np.where(np.arange(V + 1) == pc, xr, (np.float32(lam) * lm + xr).astype(np.float32))
        d = int(np.argmax(val))
        tok = np.where(np.arange(V + 1) == sp, -np.inf, xr)
        order = np.argsort(-tok, kind="stable")
        c1, c2, c3 = order[:3]
        lmub = ub[st]
        cands = [(xr[sp], sp)] + ([(xr[pc], pc)] if pc >= 0 else [])
        r1ex = tok[c2] if c1 == pc else tok[c1]
        best = max(cands, key=lambda z: (z[0], -z[1]))
        if best[0] > np.float32(lam) * lmub + r1ex:
            lvl = 0
        else:
            for c in (c1, c2):
                if c != pc: cands.append((val[c], c))
            best = max(cands, key=lambda z: (z[0], -z[1]))
            lvl = 1 if best[0] > np.float32(lam) * lmub + tok[c3] else 2
        if lvl < 2: assert best[1] == d, (b, t, best, d)
        cnt[lvl] += 1
        if d == sp: pc = -1
        elif d != pc:
            emis += 1; st = int(n_o[0][d]); pc = d
print(f"B={B} frames {cnt.sum()}: level0 {cnt[0]} level1 {cnt[1]} level2 {cnt[2]} ({cnt[2]/cnt.sum():.3%}); emissions {emis}")
