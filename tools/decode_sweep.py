"""Persistent CTC decode ms per utterance batch (B=256, T=500, 6-gram, lambda=0.3), NGPULM_LIB selects the variant."""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2505_22857_b200 as ng, synth
f = synth.make_lm("/tmp/ngpulm_prof", 1024, 6, tokens=430000, seed=1, heldout=4000, tag="bench_6gram")
m = ng.load_arpa(f.arpa, vocab_size=1024, device=0)
B, T = 256, 500
x = torch.from_numpy(synth.ctc_logits(synth.read_sentences(f.heldout), B, T, 1024, seed=4)).cuda()
st = torch.zeros(B, dtype=torch.int32, device="cuda"); pv = torch.full((B,), -1, dtype=torch.int32, device="cuda")
ts = []
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for _ in range(5):
    st.zero_(); pv.fill_(-1)
    e0.record(); fr, em, el = m.ctc_greedy_decode(x, st, pv, lam=0.3); e1.record(); torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
# outputs digest (variants must agree bit for bit)
import hashlib
h = hashlib.sha1()
for t in (fr, el, st, pv):
    h.update(t.cpu().numpy().tobytes())
for b in range(B):
    h.update(em[b, :int(el[b])].cpu().numpy().tobytes())
print(f"decode ms: {statistics.median(ts[1:]):.4f} digest {h.hexdigest()[:12]}", flush=True)
