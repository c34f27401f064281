"""One persistent CTC decode per variant at configs[2] (B=256, T=500, 6-gram), for ncu:
plain (no LM) and lambda=0.3."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2505_22857_b200 as ng, synth
f = synth.make_lm("/tmp/ngpulm_prof", 1024, 6, tokens=430000, seed=1, heldout=4000, tag="bench_6gram")
m = ng.load_arpa(f.arpa, vocab_size=1024, device=0)
B = int(os.environ.get("B", 256))
x = torch.from_numpy(synth.ctc_logits(synth.read_sentences(f.heldout), B, 500, 1024, seed=4)).cuda()
for plain in (True, False):
    st = torch.zeros(B, dtype=torch.int32, device="cuda"); pv = torch.full((B,), -1, dtype=torch.int32, device="cuda")
    m.ctc_greedy_decode(x, None if plain else st, pv, lam=0.0 if plain else 0.3)
torch.cuda.synchronize()
