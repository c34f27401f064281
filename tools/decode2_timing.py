"""Per-row decider phases of the bound-pruned CTC decode (debug build lib/libngpulm_timing.so):
cycles in summary waits, level 0, lookups, staging waits, level-2 builds / argmax, state loads,
outputs, and the level counts (medians over rows)."""
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
for B in (1, 256):
    T = 500
    x = torch.from_numpy(synth.ctc_logits(synth.read_sentences(f.heldout), B, T, 1024, seed=4)).cuda()
    for rep in range(2):
        st = torch.zeros(B, dtype=torch.int32, device="cuda")
        pv = torch.full((B,), -1, dtype=torch.int32, device="cuda")
        scratch = np.zeros(16 * B, np.uint64)
        L.ngpulm_debug_phases(scratch.ctypes.data, 16 * B)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        m.ctc_greedy_decode(x, st, pv, lam=0.3)
        e1.record()
        torch.cuda.synchronize()
    buf = np.zeros(B * 16, dtype=np.uint64)
    L.ngpulm_debug_phases(buf.ctypes.data, B * 16)
    ph = buf.reshape(B, 16).astype(np.int64)
    names = ["sumwait", "level0", "lookup", "stagewait", "l2build", "l2argmax", "stateload", "output",
             "n_l0", "n_l1", "n_l2", "n_build", "n_state"]
    med = {n: int(np.median(ph[:, i])) for i, n in enumerate(names)}
    print(f"B={B}: {e0.elapsed_time(e1) * 1e3:.0f} us; medians {med}; total cycles {int(np.median(ph[:, :8].sum(1)))}",
          flush=True)
