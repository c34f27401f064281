"""Fused greedy step us per step (CUDA graph of 256 steps, state carried) for the
bench shapes: CTC B=256, RNN-T / AED B=512, on the bench 6-gram LM. NGPULM_LIB picks the variant."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2505_22857_b200 as ng  # noqa: E402
import synth  # noqa: E402

f = synth.make_lm("/tmp/ngpulm_prof", 1024, 6, tokens=430000, seed=1, heldout=4000, tag="bench_6gram")
m = ng.load_arpa(f.arpa, vocab_size=1024, device=0)
V, s = 1024, torch.cuda.Stream()
out = []
for name, mode, B, gen in (("ctc", ng.CTC, 256, synth.rnnt_logits), ("rnnt", ng.RNNT, 512, synth.rnnt_logits),
                           ("aed", ng.AED, 512, synth.aed_logits)):
    NB, n = 16, 256
    xs = torch.from_numpy(gen(B, NB, V, seed=4)).cuda()
    st0 = torch.from_numpy(synth.uniform_states(m.num_states, B, seed=3)).cuda()
    st, pv = st0.clone(), torch.full((B,), -1, dtype=torch.int32, device="cuda")
    tok = torch.empty(B, dtype=torch.int32, device="cuda")
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        m.fused_greedy_step(mode, xs[0], st, prev=pv, lam=0.3, tokens_out=tok, stream=s)
        s.synchronize()
        with torch.cuda.graph(g, stream=s):
            for k in range(n):
                m.fused_greedy_step(mode, xs[k % NB], st, prev=pv, lam=0.3, tokens_out=tok, stream=s)
    ts = []
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(5):
        with torch.cuda.stream(s):
            st.copy_(st0)
            e0.record(s); g.replay(); e1.record(s)
        s.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3 / n)
    out.append(f"{name}_b{B} {statistics.median(ts):.2f}")
# CTC frame steps reading [B, T, V+1] logits from HBM (the bench's configs[2] leg)
B, T = 256, 500
x = torch.from_numpy(synth.ctc_logits(synth.read_sentences(f.heldout), B, T, V, seed=4)).cuda()
st = torch.zeros(B, dtype=torch.int32, device="cuda")
pv = torch.full((B,), -1, dtype=torch.int32, device="cuda")
fr = torch.empty((T, B), dtype=torch.int32, device="cuda")
g = torch.cuda.CUDAGraph()
with torch.cuda.stream(s):
    for t in range(2):
        m.fused_greedy_step(ng.CTC, x[:, t], st, prev=pv, lam=0.3, tokens_out=fr[t], stream=s)
    s.synchronize()
    with torch.cuda.graph(g, stream=s):
        for t in range(T):
            m.fused_greedy_step(ng.CTC, x[:, t], st, prev=pv, lam=0.3, tokens_out=fr[t], stream=s)
ts = []
for _ in range(3):
    with torch.cuda.stream(s):
        st.zero_(); pv.fill_(-1)
        e0.record(s); g.replay(); e1.record(s)
    s.synchronize()
    ts.append(e0.elapsed_time(e1) * 1e3 / T)
out.append(f"ctc_hbm_b256 {statistics.median(ts):.2f}")
print("fused us/step:", " ".join(out), flush=True)
