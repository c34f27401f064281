"""advance us/call on the bench's tiny keyword-biasing-sized LM (model in shared memory), B = 128, 1024, 4096."""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2505_22857_b200 as ng, synth
f = synth.make_lm("/tmp/ngpulm_tiny", 1024, 3, tokens=600, seed=11, heldout=200, tag="tiny_bias")
m = ng.load_arpa(f.arpa, vocab_size=1024, device=0)
m.set_advance_kernel(int(os.environ.get("KIND", "0")))
s = torch.cuda.Stream()
out = []
for B in (128, 1024, 4096):
    R = max(2, min(64, 600 * 2**20 // (B * 8192)))
    st = torch.from_numpy(synth.uniform_states(m.num_states, B * R, seed=12).reshape(R, B)).cuda()
    sc = torch.empty((R, B, 1024), dtype=torch.float32, device="cuda")
    nx = torch.empty((R, B, 1024), dtype=torch.int32, device="cuda")
    g = torch.cuda.CUDAGraph()
    n = 256
    with torch.cuda.stream(s):
        m.advance(st[0], sc[0], nx[0], want_final=False, stream=s); s.synchronize()
        with torch.cuda.graph(g, stream=s):
            for k in range(n):
                m.advance(st[k % R], sc[k % R], nx[k % R], want_final=False, stream=s)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(3):
        with torch.cuda.stream(s):
            e0.record(s); g.replay(); e1.record(s)
        s.synchronize(); ts.append(e0.elapsed_time(e1) * 1e3 / n)
    out.append(f"B{B} {statistics.median(ts):.2f}")
print("tiny us/call:", " ".join(out), "resident", m.info.tiny_resident, flush=True)
