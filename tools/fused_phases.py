"""Per-row phase stamps of the fused warp kernel (debug build lib/libngpulm_timing.so):
0 entry ns, 2 after griddepcontrol.wait, 11 record, 3 gathers issued, 4 root fill,
5 root targets landed, 6 levels written, 12 logits landed, 7 argmax done, 8 end."""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("NGPULM_LIB", os.path.join(ROOT, "paper_2505_22857_b200", "lib", "libngpulm_timing.so"))
NET = int(os.environ.get("NET", 0))  # 1: a (non-PDL) network kernel writes each step's logits first
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2505_22857_b200 as ng  # noqa: E402
import synth  # noqa: E402

L = ng.lib()
L.ngpulm_debug_phases.argtypes = [C.c_void_p, C.c_int]
f = synth.make_lm("/tmp/ngpulm_prof", 1024, 6, tokens=430000, seed=1, heldout=4000, tag="bench_6gram")
m = ng.load_arpa(f.arpa, vocab_size=1024, device=0)
V = 1024


def phases(B):
    buf = np.zeros(B * 16, dtype=np.uint64)
    assert L.ngpulm_debug_phases(buf.ctypes.data, B * 16) == 0
    ph = buf.reshape(B, 16).astype(np.int64)
    return ph[ph[:, 8] > 0]


def q(a):
    return f"{int(np.median(a)):6d}/{int(np.percentile(a, 90)):6d}/{int(a.max()):6d}"


def report(tag, ph):
    if len(ph) == 0:
        print(f"{tag}: no stamps (this kernel path carries no phase stamps)", flush=True)
        return
    names = [("wait", 1, 2), ("st+rec", 2, 11), ("issue", 11, 3), ("fill", 3, 4), ("rootto", 4, 5),
             ("write", 5, 6), ("logits", 6, 12), ("argmax", 12, 7), ("out", 7, 8)]
    parts = " ".join(f"{n} {q(ph[:, b] - ph[:, a])}" for n, a, b in names)
    print(f"{tag}: {parts}", flush=True)


stream = torch.cuda.Stream()
for name, mode, gen in (("rnnt", ng.RNNT, synth.rnnt_logits), ("aed", ng.AED, synth.aed_logits),
                        ("ctc", ng.CTC, synth.rnnt_logits)):
    B, NB = 512, 16
    xs = torch.from_numpy(gen(B, NB, V, seed=4)).cuda()
    st = torch.from_numpy(synth.uniform_states(m.num_states, B, seed=3)).cuda()
    pv = torch.full((B,), -1, dtype=torch.int32, device="cuda")
    tok = torch.empty(B, dtype=torch.int32, device="cuda")
    buf = torch.empty_like(xs[0])
    with torch.cuda.stream(stream):
        for k in range(64):
            x = xs[k % NB]
            if NET:
                torch.mul(x, 1.0, out=buf)
                x = buf
            m.fused_greedy_step(mode, x, st, prev=pv if mode == ng.CTC else None, lam=0.3, tokens_out=tok,
                                stream=stream)
    stream.synchronize()
    report(f"{name} B={B} (64th step{', after a network kernel' if NET else ''})", phases(B))
