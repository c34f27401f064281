"""Latency/throughput sweep of ngpulm_advance on the bench LM (GPU box).
Prints per-call us for: back-to-back graph replays (rotating outputs), and
single launches (event-timed with a sync), for several B and both chain modes."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2505_22857_b200 as ng  # noqa: E402
import synth  # noqa: E402

f = synth.make_lm("/tmp/ngpulm_prof", 1024, 6, tokens=430000, seed=1, heldout=4000, tag="bench_6gram")
m = ng.load_arpa(f.arpa, vocab_size=1024, device=0)
ctx = synth.sample_contexts(synth.read_sentences(f.heldout), 6, 4096 * 64, seed=2)
allst = np.array([m.state_of(b, t) for b, t in ctx], dtype=np.int32)
stream = torch.cuda.Stream()
R_BYTES = 600 * 2**20
INDEP = bool(int(os.environ.get("SWEEP_INDEP", "0")))  # NGPULM_ADVANCE_INDEPENDENT calls


def run(B, mode, n=400):
    m.set_chain_mode(mode)
    R = max(2, min(64, R_BYTES // (B * 1024 * 8)))
    st = torch.from_numpy(allst[: R * B].reshape(R, B)).cuda()
    sc = torch.empty((R, B, 1024), dtype=torch.float32, device="cuda")
    nx = torch.empty((R, B, 1024), dtype=torch.int32, device="cuda")
    fi = torch.empty((R, B), dtype=torch.float32, device="cuda")
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(stream):
        for k in range(3):
            m.advance(st[k % R], sc[k % R], nx[k % R], fi[k % R], stream=stream, independent=INDEP)
        stream.synchronize()
        with torch.cuda.graph(g, stream=stream):
            for k in range(n):
                m.advance(st[k % R], sc[k % R], nx[k % R], fi[k % R], stream=stream, independent=INDEP)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(5):
        with torch.cuda.stream(stream):
            e0.record(stream); g.replay(); e1.record(stream)
        stream.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3 / n)
    graph_us = statistics.median(ts)
    single = []
    for k in range(50):
        with torch.cuda.stream(stream):
            e0.record(stream)
            m.advance(st[k % R], sc[k % R], nx[k % R], fi[k % R], stream=stream)
            e1.record(stream)
        stream.synchronize()
        single.append(e0.elapsed_time(e1) * 1e3)
    return graph_us, statistics.median(single[5:])


MODES = ((ng.CHAIN_TABLE, "table"), (ng.CHAIN_WALK, "walk"))
BS = tuple(int(x) for x in os.environ.get("SWEEP_BS", "1,16,128,512,1024,2048,4096").split(","))
if os.environ.get("SWEEP_QUICK"):
    MODES = MODES[:1]
    if not os.environ.get("SWEEP_BS"):
        BS = (1, 128, 1024, 4096)
print("lib", os.path.basename(ng.LIB_PATH))
print("B, kernel, mode, graph_us_per_call, single_launch_us, GB/s(graph)")
KINDS = [int(x) for x in os.environ.get("SWEEP_KERNELS", "0,1,2").split(",")]
if os.environ.get("SWEEP_SKIP"):  # debug build only: parts of the warp kernel switched off (timing only)
    ng.lib().ngpulm_debug_skip(int(os.environ["SWEEP_SKIP"]))
    print("skip bits", os.environ["SWEEP_SKIP"])
for kind in KINDS:
    m.set_advance_kernel(kind)
    for mode, name in MODES:
        for B in BS:
            gus, sus = run(B, mode)
            print(f"{B:5d} {['auto', 'warp', 'cta'][kind]:4s} {name:5s} {gus:8.2f} {sus:8.2f} "
                  f"{B*1024*8/gus/1e3:8.1f}", flush=True)
m.set_advance_kernel(ng.ADVANCE_AUTO)
