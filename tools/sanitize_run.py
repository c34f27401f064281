"""Every hot-path kernel once on small inputs, each result checked against the
oracle — the workload of the compute-sanitizer runs (memcheck, racecheck,
synccheck, initcheck; tools/sanitize.sh). Sizes are small (the sanitizers
slow kernels down 10-1000x) but reach every kernel path: warp / tiny / CTA
advance (table and walk), vocabulary tiles, final, the CTC/AED warp step, the
transducer warp pair and single-warp steps, ILM, top-k, label looping
(RNN-T and TDT), the persistent CTC decode (LM and plain), the rows mode."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2505_22857_b200 as ng  # noqa: E402
import synth  # noqa: E402
from oracle import Oracle  # noqa: E402
from paper_2505_22857_b200.decode import transducer_greedy_decode  # noqa: E402

D = "/tmp/ngpulm_sanitize"
ONLY = set(filter(None, os.environ.get("SAN_ONLY", "").split(",")))  # sections to run (default: all)
want = lambda sec: not ONLY or sec in ONLY  # noqa: E731
dev = torch.device("cuda", 0)
T_ = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
ok = []


def same(a, b):
    return np.array_equal(np.asarray(a).view(np.int32), np.asarray(b).view(np.int32))


def check(name, cond):
    ok.append((name, bool(cond)))
    print(f"{'ok  ' if cond else 'FAIL'} {name}", flush=True)


lms = {"tri64": (64, 3, 2000), "ten24": (24, 10, 1500), "six1024": (1024, 6, 30000)}
if os.environ.get("SAN_LMS"):
    lms = {k: v for k, v in lms.items() if k in os.environ["SAN_LMS"].split(",")}
models = {}
for name, (V, N, toks) in lms.items():
    f = synth.make_lm(D, V, N, tokens=toks, seed=1, lexicon=200, heldout=50, tag=name)
    models[name] = (ng.load_arpa(f.arpa, vocab_size=V, device=0), Oracle(f.arpa, vocab_size=V), f)
rng = np.random.default_rng(7)

for name, (m, o, f) in models.items():
    V = m.V
    for B in (3, 70, 200):
        if not (want("adv") or want("fused") or want("topk") or want("rows")):
            break
        st = synth.uniform_states(o.num_states, B, seed=B)
        s32, _, n_o, _ = o.rows(st)
        f32, _ = o.finals(st)
        for kind in ((ng.ADVANCE_AUTO, ng.ADVANCE_WARP, ng.ADVANCE_CTA) if want("adv") else ()):
            for chain in (ng.CHAIN_TABLE, ng.CHAIN_WALK):
                m.set_advance_kernel(kind); m.set_chain_mode(chain)
                s, n, fi = m.advance(T_(st))
                torch.cuda.synchronize()
                check(f"advance {name} B={B} kind={kind} chain={chain}",
                      same(s.cpu(), s32) and np.array_equal(n.cpu().numpy(), n_o) and same(fi.cpu(), f32))
        m.set_advance_kernel(ng.ADVANCE_AUTO); m.set_chain_mode(ng.CHAIN_TABLE)
        fi2 = m.final(T_(st))
        torch.cuda.synchronize()
        check(f"final {name} B={B}", same(fi2.cpu(), f32))
        for Bf in ((B, 600 if name != "six1024" else B) if want("fused") else ()):
            stf = synth.uniform_states(o.num_states, Bf, seed=Bf + 1)
            x = rng.standard_normal((Bf, V + 1)).astype(np.float32)
            for mode in (ng.CTC, ng.RNNT, ng.AED):
                pv = np.where(rng.random(Bf) < 0.5, -1, rng.integers(0, V, Bf)).astype(np.int32)
                sd, pd = T_(stf), T_(pv)
                tok = m.fused_greedy_step(mode, T_(x), sd, prev=pd, lam=0.7)
                torch.cuda.synchronize()
                to, so, po = o.fused_step(mode, x, stf, prev=pv, lam=0.7)
                check(f"fused {name} mode={mode} B={Bf}", np.array_equal(tok.cpu().numpy(), to)
                      and np.array_equal(sd.cpu().numpy(), so))
                tok0 = m.fused_greedy_step(mode, T_(x), None, prev=T_(pv), lam=0.0)
                torch.cuda.synchronize()
                to0, _, _ = o.fused_step(mode, x, stf, prev=pv, lam=0.0)
                check(f"plain {name} mode={mode} B={Bf}", np.array_equal(tok0.cpu().numpy(), to0))
            ilm = (rng.standard_normal((Bf, V)) - 3).astype(np.float32)
            sd = T_(stf)
            tok = m.fused_greedy_step_ilm(ng.RNNT, T_(x), sd, T_(ilm), 0.2, lam=0.7)
            torch.cuda.synchronize()
            to, so, _ = o.fused_step_ilm(ng.RNNT, x, stf, ilm, 0.2, lam=0.7)
            check(f"ilm {name} B={Bf}", np.array_equal(tok.cpu().numpy(), to))
        x = rng.standard_normal((B, V + 1)).astype(np.float32)
        if not (want("topk") or want("rows")):
            continue
        sc, cols, nxt = m.fused_topk(T_(x[:B]), T_(st), 4, lam=0.7)
        torch.cuda.synchronize()
        ts, tc, tn = o.topk(x[:B], st, 4, lam=0.7)
        check(f"topk {name} B={B}", np.array_equal(cols.cpu().numpy(), tc) and same(sc.cpu(), ts))
        # rows mode
        s, n, fi = m.advance(T_(st))
        sd = T_(st)
        tok = m.fused_greedy_step_rows(ng.AED, T_(x[:B]), s, n, fi, sd, lam=0.7)
        torch.cuda.synchronize()
        to, so, _ = o.fused_step(ng.AED, x[:B], st, lam=0.7)
        check(f"rows {name} B={B}", np.array_equal(tok.cpu().numpy(), to))
    # persistent CTC decode (LM and plain)
    Bc, Tc = 6, 40
    if not want("decode"):
        Bc = 0
    xc = rng.standard_normal((Bc, Tc, V + 1)).astype(np.float32)
    xc[:, :, V] += 1.5
    lengths = np.array([0, 1, 17, 40, 33, 40], np.int32)
    for chain in ((ng.CHAIN_TABLE, ng.CHAIN_WALK) if Bc else ()):
        m.set_chain_mode(chain)
        st0 = np.zeros(Bc, np.int32); pv0 = np.full(Bc, -1, np.int32)
        sd, pd = T_(st0), T_(pv0)
        em0 = torch.full((Bc, Tc), -1, dtype=torch.int32, device=dev)  # entries past emit_len are never written
        fr, em, el = m.ctc_greedy_decode(T_(xc), sd, pd, lam=0.7, lengths=T_(lengths), emit_out=em0)
        torch.cuda.synchronize()
        ref = o.ctc_decode(xc, st0, prev=pv0, lam=0.7, lengths=lengths)
        check(f"ctc decode {name} chain={chain}", np.array_equal(fr.cpu().numpy(), ref[0])
              and np.array_equal(el.cpu().numpy(), ref[2]))
    m.set_chain_mode(ng.CHAIN_TABLE)
    if Bc:  # segment-parallel decode (T >= 128: K = 3 segments), ragged lengths
        Bs, Ts = 3, 200
        xs = rng.standard_normal((Bs, Ts, V + 1)).astype(np.float32)
        xs[:, :, V] += 1.0
        ls = np.array([200, 130, 70], np.int32)
        st0 = np.zeros(Bs, np.int32); pv0 = np.full(Bs, -1, np.int32)
        sd, pd = T_(st0), T_(pv0)
        em0 = torch.full((Bs, Ts), -1, dtype=torch.int32, device=dev)
        fr, em, el = m.ctc_greedy_decode(T_(xs), sd, pd, lam=0.7, lengths=T_(ls), emit_out=em0)
        torch.cuda.synchronize()
        ref = o.ctc_decode(xs, st0, prev=pv0, lam=0.7, lengths=ls)
        check(f"ctc segment decode {name}", np.array_equal(fr.cpu().numpy(), ref[0])
              and np.array_equal(el.cpu().numpy(), ref[2]) and np.array_equal(sd.cpu().numpy(), ref[3]))
    if Bc:
        pd = T_(np.full(Bc, -1, np.int32))
        em0 = torch.full((Bc, Tc), -1, dtype=torch.int32, device=dev)
        fr, em, el = m.ctc_greedy_decode(T_(xc), None, pd, lam=0.0, lengths=T_(lengths), emit_out=em0)
        torch.cuda.synchronize()
        ref = o.ctc_decode(xc, np.zeros(Bc, np.int32), prev=np.full(Bc, -1, np.int32), lam=0.0, lengths=lengths)
        check(f"ctc decode plain {name}", np.array_equal(fr.cpu().numpy(), ref[0]))
    # label looping: RNN-T and TDT
    Bl = 8
    ll = np.array([0, 1, 5, 9, 12, 3, 7, 11], np.int32)

    def joint(frame, u, last, out):
        synth.joint_gpu(5151, frame, u, last, out, temperature=2.0, blank=V, blank_bias=0.75)
    for durs in ((None, [0, 1, 2, 4]) if want("loop") else ()):
        res = transducer_greedy_decode(m, joint, T_(ll), lam=0.5, max_symbols=3, durations=durs, graph_steps=4)
        torch.cuda.synchronize()
        if durs is None:
            em, el, sto = o.transducer_decode(5151, ll, np.zeros(Bl, np.int32), lam=0.5, max_symbols=3,
                                              temperature=2.0, max_len=res.emitted.shape[1], blank_bias=0.75)[:3]
        else:
            em, el, sto, _ = o.tdt_decode(5151, ll, np.zeros(Bl, np.int32), durs, lam=0.5, max_symbols=3,
                                          temperature=2.0, max_len=res.emitted.shape[1], blank_bias=0.75)
        check(f"label loop {name} tdt={durs is not None}", np.array_equal(res.emit_len.cpu().numpy(), el))

# vocabulary tiles (rows beyond shared memory)
if want("tiled"):
    f = synth.make_lm(D, 40000, 2, tokens=60000, seed=9, heldout=50, tag="bigv")
    m, o = ng.load_arpa(f.arpa, vocab_size=40000, device=0), Oracle(f.arpa, vocab_size=40000)
    st = synth.uniform_states(o.num_states, 5, seed=3)
    s, n, fi = m.advance(T_(st))
    torch.cuda.synchronize()
    s32, _, n_o, _ = o.rows(st)
    check("advance tiled V=40000", same(s.cpu(), s32) and np.array_equal(n.cpu().numpy(), n_o))
bad = [n for n, c in ok if not c]
print(f"sanitize_run: {len(ok)} checks, {len(bad)} failed", flush=True)
sys.exit(1 if bad else 0)
