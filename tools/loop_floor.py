"""Per-iteration cost of decoder-loop shapes (CUDA graph of 256 iterations, B=512, 6-gram):
network kernel alone, + a tiny torch kernel, + plain / fused RNN-T step, + the overlap mode
(advance on a side stream while the network runs, then the fused step from the LM rows)."""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2505_22857_b200 as ng, synth

f = synth.make_lm("/tmp/ngpulm_prof", 1024, 6, tokens=430000, seed=1, heldout=4000, tag="bench_6gram")
m = ng.load_arpa(f.arpa, vocab_size=1024, device=0)
B, V, NB, N = int(os.environ.get("B", 512)), 1024, 16, 256
dev = torch.device("cuda", 0)
xs = torch.from_numpy(synth.rnnt_logits(B, NB, V, seed=4)).to(dev)
buf = torch.empty_like(xs[0])
st0 = torch.from_numpy(synth.uniform_states(m.num_states, B, seed=3)).to(dev)
st = st0.clone()
tok = torch.empty(B, dtype=torch.int32, device=dev)
tiny = torch.zeros(1, device=dev)
sc = torch.empty((B, V), device=dev); nx = torch.empty((B, V), dtype=torch.int32, device=dev)
fi = torch.empty(B, device=dev)
main, side = torch.cuda.Stream(), torch.cuda.Stream()


def net(k):
    torch.mul(xs[k % NB], 1.0, out=buf)


def graph_us(body):
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(main):
        st.copy_(st0); body(); torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=main):
            body()
    ts = []
    for _ in range(7):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(main):
            st.copy_(st0)
            e0.record(main); g.replay(); e1.record(main)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3 / N)
    return statistics.median(ts[1:])


def overlap_body():
    ev_done = torch.cuda.Event()
    for k in range(N):
        ev_done.record(main)
        side.wait_event(ev_done)
        m.advance(st, sc, nx, fi, stream=side)   # LM rows of the current states
        net(k)                                    # the network on the main stream meanwhile
        ev_adv = torch.cuda.Event()
        ev_adv.record(side)
        main.wait_event(ev_adv)
        m.fused_greedy_step_rows(ng.RNNT, buf, sc, nx, fi, st, lam=0.3, tokens_out=tok, stream=main)


res = {
    "net": graph_us(lambda: [net(k) for k in range(N)]),
    "net+tiny": graph_us(lambda: [(net(k), tiny.add_(1.0)) for k in range(N)]),
    "net+plain": graph_us(lambda: [(net(k), m.fused_greedy_step(ng.RNNT, buf, None, lam=0.0, tokens_out=tok, stream=main)) for k in range(N)]),
    "net+fused": graph_us(lambda: [(net(k), m.fused_greedy_step(ng.RNNT, buf, st, lam=0.3, tokens_out=tok, stream=main)) for k in range(N)]),
    "plain b2b": graph_us(lambda: [m.fused_greedy_step(ng.RNNT, xs[k % NB], None, lam=0.0, tokens_out=tok, stream=main) for k in range(N)]),
    "fused b2b": graph_us(lambda: [m.fused_greedy_step(ng.RNNT, xs[k % NB], st, lam=0.3, tokens_out=tok, stream=main) for k in range(N)]),
    "advance b2b": graph_us(lambda: [m.advance(st, sc, nx, fi, stream=main) for k in range(N)]),
    "net+overlap": graph_us(overlap_body),
}
print({k: round(v, 3) for k, v in res.items()}, flush=True)
