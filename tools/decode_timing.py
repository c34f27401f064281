"""Per-row phase cycles of the persistent CTC decode (debug build lib/libngpulm_timing.so).

Accumulated per row (clock64): first LM-row build, ring refills issued, logits
waits, frame decisions, rebuilds (count), frames. Prints medians over rows,
then the same with rebuilds skipped (g_skip bit 4: decisions on a stale LM
row, timing only).
"""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["NGPULM_LIB"] = os.path.join(ROOT, "paper_2505_22857_b200", "lib", "libngpulm_timing.so")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2505_22857_b200 as ng  # noqa: E402
import synth  # noqa: E402

L = ng.lib()
L.ngpulm_debug_phases.argtypes = [C.c_void_p, C.c_int]
L.ngpulm_debug_skip.argtypes = [C.c_int]
f = synth.make_lm("/tmp/ngpulm_prof", 1024, 6, tokens=430000, seed=1, heldout=4000, tag="bench_6gram")
m = ng.load_arpa(f.arpa, vocab_size=1024, device=0)
B, T = int(os.environ.get("B", 256)), 500
x = torch.from_numpy(synth.ctc_logits(synth.read_sentences(f.heldout), B, T, 1024, seed=4)).cuda()
for skip in (0, 16):
    L.ngpulm_debug_skip(skip)
    for rep in range(3):
        st = torch.zeros(B, dtype=torch.int32, device="cuda")
        pv = torch.full((B,), -1, dtype=torch.int32, device="cuda")
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        scratch = np.zeros(16 * B, np.uint64)  # (kept alive across the call)
        L.ngpulm_debug_phases(scratch.ctypes.data, 16 * B)  # clear
        e0.record()
        m.ctc_greedy_decode(x, st, pv, lam=0.3)
        e1.record()
        torch.cuda.synchronize()
    buf = np.zeros(B * 16, dtype=np.uint64)
    L.ngpulm_debug_phases(buf.ctypes.data, B * 16)
    ph = buf.reshape(B, 16).astype(np.int64)
    names = ["first", "record", "wait", "decide", "reload", "n_rebuild", "frames", "gather", "write"]
    med = {n: int(np.median(ph[:, i])) for i, n in enumerate(names)}
    tot = ph[:, [0, 1, 2, 3, 4, 7, 8]].sum(axis=1)
    med["rebuild"] = med["record"] + med["gather"] + med["write"] + med["reload"]
    print(f"skip={skip} launch {e0.elapsed_time(e1) * 1e3:.0f} us; per-row medians:", med,
          f"total cycles med {int(np.median(tot))} max {int(tot.max())}",
          f"per rebuild {med['rebuild'] / max(1, med['n_rebuild']):.0f} cyc, per frame decide "
          f"{med['decide'] / max(1, med['frames']):.0f} wait {med['wait'] / max(1, med['frames']):.0f}; "
          f"per rebuild: record {med['record'] / max(1, med['n_rebuild']):.0f} gather+root "
          f"{med['gather'] / max(1, med['n_rebuild']):.0f} write {med['write'] / max(1, med['n_rebuild']):.0f} "
          f"reload {med['reload'] / max(1, med['n_rebuild']):.0f}")
