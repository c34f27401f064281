"""Persistent CTC decode ms per utterance batch vs B (T=500, 6-gram), plain (no LM) and lambda=0.3:
is the per-frame time a per-row latency (flat in B) or a throughput limit (grows with B)?"""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2505_22857_b200 as ng, synth
f = synth.make_lm("/tmp/ngpulm_prof", 1024, 6, tokens=430000, seed=1, heldout=4000, tag="bench_6gram")
m = ng.load_arpa(f.arpa, vocab_size=1024, device=0)
T = 500
xa = torch.from_numpy(synth.ctc_logits(synth.read_sentences(f.heldout), 256, T, 1024, seed=4)).cuda()
for B in (1, 16, 64, 148, 256):
    x = xa[:B]
    res = {}
    for lam, plain in ((0.3, False), (0.0, True)):
        st = torch.zeros(B, dtype=torch.int32, device="cuda"); pv = torch.full((B,), -1, dtype=torch.int32, device="cuda")
        ts = []
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for _ in range(5):
            st.zero_(); pv.fill_(-1)
            e0.record(); m.ctc_greedy_decode(x, None if plain else st, pv, lam=lam); e1.record(); torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        res["plain" if plain else "fused"] = statistics.median(ts[1:])
    print(f"B={B}: fused {res['fused']:.4f} ms, plain {res['plain']:.4f} ms, "
          f"logits {x.numel()*4/res['fused']/1e6:.0f} GB/s", flush=True)
