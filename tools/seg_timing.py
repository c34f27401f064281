"""Per-chain phase cycles of the segment-parallel CTC decode's pass 1 (debug build lib/libngpulm_timing.so):
per frame: ring wait, loads + refill issue, decision, record writes; per rebuild: chain record, arc gathers +
writes, final sync, register reload; medians over chains."""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("NGPULM_LIB", os.path.join(ROOT, "paper_2505_22857_b200", "lib", "libngpulm_timing.so"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2505_22857_b200 as ng  # noqa: E402
import synth  # noqa: E402

L = ng.lib()
L.ngpulm_debug_phases.argtypes = [C.c_void_p, C.c_int]
f = synth.make_lm("/tmp/ngpulm_prof", 1024, 6, tokens=430000, seed=1, heldout=4000, tag="bench_6gram")
m = ng.load_arpa(f.arpa, vocab_size=1024, device=0)
T = 500
xa = torch.from_numpy(synth.ctc_logits(synth.read_sentences(f.heldout), 256, T, 1024, seed=4)).cuda()
for B in (1, 148, 256):
    x = xa[:B]
    for rep in range(2):
        st = torch.zeros(B, dtype=torch.int32, device="cuda")
        pv = torch.full((B,), -1, dtype=torch.int32, device="cuda")
        scratch = np.zeros(16 * 4096, np.uint64)
        L.ngpulm_debug_phases(scratch.ctypes.data, 16 * 4096)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        m.ctc_greedy_decode(x, st, pv, lam=0.3)
        e1.record()
        torch.cuda.synchronize()
    buf = np.zeros((8192 + 4096) * 16, dtype=np.uint64)
    L.ngpulm_debug_phases(buf.ctypes.data, (8192 + 4096) * 16)
    allp = buf.reshape(8192 + 4096, 16).astype(np.int64)
    ph = allp[:4096]
    ph = ph[ph[:, 5] > 0]
    names = ["reload", "wait", "load+issue", "decide", "records", "frames", "rebuilds", "record", "arcs+writes",
             "sync"]
    med = {n: int(np.median(ph[:, i])) for i, n in enumerate(names)}
    per = {n: round(med[n] / max(1, med["frames"])) for n in ["wait", "load+issue", "decide", "records"]}
    per_rb = {n: round(med[n] / max(1, med["rebuilds"])) for n in ["record", "arcs+writes", "sync", "reload"]}
    tot = ph[:, [0, 1, 2, 3, 4, 7, 8, 9]].sum(1)
    fix = allp[8192:8192 + B, 1:8]
    print(f"B={B}: {e0.elapsed_time(e1) * 1e3:.0f} us, {len(ph)} chains; medians {med}; per frame {per}; "
          f"per rebuild {per_rb}; chain cycles median {int(np.median(tot))} "
          f"p90 {int(np.percentile(tot, 90))} max {int(tot.max())}; pass-2 frames per row: mean "
          f"{fix.sum(1).mean():.1f} max {fix.sum(1).max()} (per segment max {fix.max(0).tolist()})", flush=True)
