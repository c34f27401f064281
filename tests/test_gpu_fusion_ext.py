"""GPU parity of the SURVEY.md §8(f) f3 extensions against the oracle:
ngpulm_fused_greedy_step_ilm (internal-LM subtraction, R21) and ngpulm_fused_topk
(the k best AED expansions for beam search with NGPU-LM fusion). Bar: tokens,
states, columns and next states bit-exact; top-k scores bit-exact (same float
operations in the same order as the oracle)."""
import numpy as np
import pytest

import synth
from oracle import AED, CTC, RNNT

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2505_22857_b200 as ng  # noqa: E402

from test_gpu_parity import dev, same_bits, trajectory_states, using  # noqa: E402


def T(a, dt=None):
    return torch.from_numpy(np.ascontiguousarray(a if dt is None else a.astype(dt))).to(dev())


@pytest.mark.parametrize("kernel", [ng.ADVANCE_AUTO, ng.ADVANCE_WARP, ng.ADVANCE_CTA])
@pytest.mark.parametrize("lam_ilm", [0.0, 0.6])
@pytest.mark.parametrize("mode", [CTC, RNNT, AED])
@pytest.mark.parametrize("name", ["tri64", "ten24"])
def test_fused_step_ilm_matches_oracle(pairs, name, mode, lam_ilm, kernel):
    m, o, _ = pairs[name]
    B = 257
    rng = np.random.default_rng(41)
    x = synth.rnnt_logits(B, 1, o.V, seed=42)[0]
    st = synth.uniform_states(o.num_states, B, seed=43)
    ilm = rng.normal(-4, 2, size=(B, o.V)).astype(np.float32)
    prev = rng.integers(-1, o.V, size=B).astype(np.int32) if mode == CTC else None
    active = (rng.random(B) > 0.1).astype(np.uint8)
    st_d = T(st)
    pv_d = T(prev) if prev is not None else None
    with using(m, kernel=kernel):
        tok = m.fused_greedy_step_ilm(mode, T(x), st_d, T(ilm), lam_ilm, prev=pv_d, active=T(active), lam=1.1)
    torch.cuda.synchronize()
    to, so, po = o.fused_step_ilm(mode, x, st, ilm, lam_ilm, prev=prev, active=active, lam=1.1)
    assert np.array_equal(tok.cpu().numpy(), to) and np.array_equal(st_d.cpu().numpy(), so)
    if mode == CTC:
        assert np.array_equal(pv_d.cpu().numpy(), po)


@pytest.mark.parametrize("chain", [ng.CHAIN_TABLE, ng.CHAIN_WALK])
@pytest.mark.parametrize("kernel", [ng.ADVANCE_AUTO, ng.ADVANCE_WARP])
@pytest.mark.parametrize("k", [1, 4, 33])
@pytest.mark.parametrize("lam", [0.0, 0.3, 3.0])
@pytest.mark.parametrize("name", ["tiny3", "five48", "ten24"])
def test_topk_matches_oracle(pairs, name, lam, k, kernel, chain):
    m, o, _ = pairs[name]
    B = 150
    x = synth.rnnt_logits(B, 1, o.V, seed=44)[0]
    x[::7, 5] = x[::7, 2]                         # exact ties
    st = synth.uniform_states(o.num_states, B, seed=45)
    with using(m, chain, kernel):
        sc, cols, nx = m.fused_topk(T(x), T(st), k, lam=lam)
    torch.cuda.synchronize()
    so, co, no = o.topk(x, st, k, lam=lam)
    assert np.array_equal(cols.cpu().numpy(), co)
    assert same_bits(sc.cpu().numpy(), so)
    assert np.array_equal(nx.cpu().numpy(), no)


@pytest.mark.parametrize("eos", [0, 11])
def test_topk_with_ilm_and_eos_inside(pairs, eos):
    m, o, _ = pairs["tri64"]
    B, k = 100, 8
    x = synth.rnnt_logits(B, 1, o.V, seed=46, blank=eos)[0]
    st = synth.uniform_states(o.num_states, B, seed=47)
    ilm = np.random.default_rng(48).normal(-4, 2, size=(B, o.V)).astype(np.float32)
    sc, cols, nx = m.fused_topk(T(x), T(st), k, lam=0.9, eos_id=eos, ilm=T(ilm), lam_ilm=0.4)
    torch.cuda.synchronize()
    so, co, no = o.topk(x, st, k, lam=0.9, eos_id=eos, ilm=ilm, lam_ilm=0.4)
    assert np.array_equal(cols.cpu().numpy(), co) and same_bits(sc.cpu().numpy(), so)
    assert np.array_equal(nx.cpu().numpy(), no)


def test_topk_beam_shape_6gram(lm6):
    """AED beam-search shape on the configs[1] LM: beam 4 x 128 utterances = 512
    hypothesis rows, k = 4 (beam = 4), trajectory states."""
    m, o, f = lm6
    B, k = 512, 4
    st, _ = trajectory_states(m, f, B, seed=49)
    x = synth.aed_logits(B, 1, m.V, seed=50)[0]
    sc, cols, nx = m.fused_topk(T(x), T(st), k, lam=0.3)
    torch.cuda.synchronize()
    rows = np.arange(B)
    so, co, no = o.topk(x[rows], st[rows], k, lam=0.3)
    assert np.array_equal(cols.cpu().numpy()[rows], co) and same_bits(sc.cpu().numpy()[rows], so)
    assert np.array_equal(nx.cpu().numpy()[rows], no)


def test_topk_invalid_state_and_bad_k(pairs):
    m, o, _ = pairs["tri64"]
    x = synth.rnnt_logits(3, 1, o.V, seed=1)[0]
    st = np.array([1, o.num_states + 5, 2], np.int32)
    sc, cols, nx = m.fused_topk(T(x), T(st), 3, lam=0.5)
    torch.cuda.synchronize()
    assert (cols.cpu().numpy()[1] == -1).all() and np.isnan(sc.cpu().numpy()[1]).all()
    assert m.check() == 1
    with pytest.raises(ng.NgpulmError):
        m.fused_topk(T(x), T(st), 0)
    with pytest.raises(ng.NgpulmError):
        m.fused_topk(T(x), T(st), ng.MAX_TOPK + 1)


@pytest.mark.parametrize("kernel", [ng.ADVANCE_AUTO, ng.ADVANCE_WARP])
@pytest.mark.parametrize("B", [100, 592, 593, 1500])
@pytest.mark.parametrize("mode", [CTC, RNNT, AED])
def test_fused_step_kernel_paths_by_batch(pairs, mode, B, kernel):
    """Both transducer paths (the warp pair up to 4 rows per SM, one warp per row
    beyond) and the CTC/AED warp kernel across batch sizes, vs the oracle; AUTO
    takes the tiny-LM path (model in shared memory), WARP the global-memory kernels."""
    m, o, _ = pairs["five48"]
    x = synth.rnnt_logits(B, 1, o.V, seed=B)[0]
    st = synth.uniform_states(o.num_states, B, seed=B + 1)
    prev = np.random.default_rng(B).integers(-1, o.V, size=B).astype(np.int32) if mode == CTC else None
    st_d, pv_d = T(st), (T(prev) if prev is not None else None)
    m.set_advance_kernel(kernel)
    try:
        tok = m.fused_greedy_step(mode, T(x), st_d, prev=pv_d, lam=0.8)
        torch.cuda.synchronize()
    finally:
        m.set_advance_kernel(ng.ADVANCE_AUTO)
    to, so, po = o.fused_step(mode, x, st, prev=prev, lam=0.8)
    assert np.array_equal(tok.cpu().numpy(), to) and np.array_equal(st_d.cpu().numpy(), so)
    if mode == CTC:
        assert np.array_equal(pv_d.cpu().numpy(), po)


def test_every_hot_call_is_graph_capturable(pairs):
    """advance, final, fused step (3 modes), ILM step, top-k, CTC decode and the
    loop step captured in one CUDA graph: replaying it gives the eager results
    (emission buffers start at -1: entries past the emission counts are not written)."""
    m, o, f = pairs["five48"]
    B, V = 64, o.V
    rng = np.random.default_rng(5)
    st0 = synth.uniform_states(o.num_states, B, seed=6)
    x = T(synth.rnnt_logits(B, 1, V, seed=7)[0])
    xc = T(synth.ctc_logits(synth.read_sentences(f.heldout), B, 9, V, seed=8))
    ilm = T(rng.normal(-4, 2, size=(B, V)).astype(np.float32))
    lengths = T(rng.integers(0, 6, size=B).astype(np.int32))
    s = torch.cuda.Stream()

    def run(bufs):
        st, sc, nx, fi, fo, toks, tk, dec, loop = bufs
        m.advance(st[0], sc, nx, fi, stream=s)
        m.final(st[0], fo, stream=s)
        for i, mode in enumerate((CTC, RNNT, AED)):
            m.fused_greedy_step(mode, x, st[1 + i], prev=st[4], lam=0.7, tokens_out=toks[i], stream=s)
        m.fused_greedy_step_ilm(RNNT, x, st[5], ilm, 0.3, lam=0.7, tokens_out=toks[3], stream=s)
        r = m.fused_topk(x, st[0], 3, lam=0.7, stream=s)
        tk[0].copy_(r[1])
        m.ctc_greedy_decode(xc, st[6], st[7], lam=0.7, frames_out=dec[0], emit_out=dec[1], emit_len=dec[2][0],
                            stream=s)
        m.transducer_loop_step(x, st[8], loop[0], loop[1], lengths, loop[2], loop[3], lam=0.7, max_symbols=2,
                               tokens_out=toks[4], stream=s)

    def fresh():
        st = torch.from_numpy(np.stack([st0] * 9)).to(dev())
        st[4].fill_(-1)
        st[7].fill_(-1)
        return (st, torch.empty((B, V), device=dev()), torch.empty((B, V), dtype=torch.int32, device=dev()),
                torch.empty(B, device=dev()), torch.empty(B, device=dev()),
                torch.empty((5, B), dtype=torch.int32, device=dev()), torch.empty((1, B, 3), dtype=torch.int32,
                                                                                  device=dev()),
                (torch.empty((B, 9), dtype=torch.int32, device=dev()), torch.full((B, 9), -1, dtype=torch.int32,
                                                                                  device=dev()),
                 torch.empty((1, B), dtype=torch.int32, device=dev())),
                (torch.zeros(B, dtype=torch.int32, device=dev()), torch.zeros(B, dtype=torch.int32, device=dev()),
                 torch.full((B, 4), -1, dtype=torch.int32, device=dev()), torch.zeros(B, dtype=torch.int32,
                                                                                    device=dev())))
    eager = fresh()
    with torch.cuda.stream(s):
        run(eager)
    s.synchronize()
    graphed = fresh()
    with torch.cuda.stream(s):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            run(graphed)
        g.replay()
    s.synchronize()

    def flat(b):
        out = []
        for t in b:
            out.extend(flat(t) if isinstance(t, tuple) else [t])
        return out
    for a, b in zip(flat(eager), flat(graphed)):
        if a.dtype == torch.float32:
            assert same_bits(a.cpu().numpy(), b.cpu().numpy())
        else:
            assert torch.equal(a.cpu(), b.cpu())


@pytest.mark.parametrize("plain", [False, True])
@pytest.mark.parametrize("lm", ["five48", "lm6"])
def test_logits_ready_ctc_frame_loop(pairs, lm6, lm, plain):
    """NGPULM_STEP_LOGITS_READY (logits copied before the PDL wait): a CTC frame
    loop over precomputed logits, every step flagged, equals the
    oracle's decode; with the LM (tiny and global paths) and plain greedy."""
    m, o, f = pairs[lm] if lm != "lm6" else lm6
    B, Tn = 300, 60
    x = synth.ctc_logits(synth.read_sentences(f.heldout), B, Tn, o.V, seed=17)
    xd = T(x)
    lam = 0.0 if plain else 0.5
    st, pv = T(np.zeros(B, np.int32)), T(np.full(B, -1, np.int32))
    frames = torch.empty((Tn, B), dtype=torch.int32, device=dev())
    for t in range(Tn):
        m.fused_greedy_step(CTC, xd[:, t], None if plain else st, prev=pv, lam=lam, tokens_out=frames[t],
                            logits_ready=True)
    torch.cuda.synchronize()
    ref = o.ctc_decode(x, np.zeros(B, np.int32), prev=np.full(B, -1, np.int32), lam=lam)
    assert np.array_equal(frames.cpu().numpy().T, ref[0])
    assert np.array_equal(pv.cpu().numpy(), ref[4])
    if not plain:
        assert np.array_equal(st.cpu().numpy(), ref[3])


@pytest.mark.parametrize("mode,B", [(AED, 200), (RNNT, 700)])
def test_logits_ready_other_modes(lm6, mode, B):
    m, o, f = lm6
    x = synth.rnnt_logits(B, 1, o.V, seed=B)[0]
    st = synth.uniform_states(o.num_states, B, seed=B + 3)
    st_d = T(st)
    tok = m.fused_greedy_step(mode, T(x), st_d, lam=0.4, logits_ready=True)
    torch.cuda.synchronize()
    to, so, _ = o.fused_step(mode, x, st, lam=0.4)
    assert np.array_equal(tok.cpu().numpy(), to) and np.array_equal(st_d.cpu().numpy(), so)


@pytest.mark.parametrize("B", [1, 148, 512, 700])
@pytest.mark.parametrize("mode", [CTC, RNNT, AED])
def test_fused_step_inputs_ready_after_plain_kernel(lm6, mode, B):
    """NGPULM_STEP_INPUTS_READY (one warp per row for every mode, the state read
    once, logits copied at the kernel's start) after a plain (non-PDL) torch kernel
    that writes the step's logits, as in a transducer / AED loop: every row vs the
    oracle, and the same tokens / states / prev as flags == 0 (6-gram, packed arcs)."""
    m, o, f = lm6
    x = synth.rnnt_logits(B, 1, o.V, seed=B + 3)[0]
    st, _ = trajectory_states(m, f, B, seed=B)
    prev = np.random.default_rng(B).integers(-1, o.V, size=B).astype(np.int32) if mode == CTC else None
    src = T(x)
    res = []
    for ready in (False, True):
        buf = torch.empty_like(src)
        st_d, pv_d = T(st), (T(prev) if prev is not None else None)
        torch.mul(src, 1.0, out=buf)  # the "network" kernel: a plain launch writing the logits
        tok = m.fused_greedy_step(mode, buf, st_d, prev=pv_d, lam=0.3, inputs_ready=ready)
        torch.cuda.synchronize()
        res.append((tok.cpu().numpy(), st_d.cpu().numpy(), pv_d.cpu().numpy() if pv_d is not None else None))
    to, so, po = o.fused_step(mode, x, st, prev=prev, lam=0.3)
    for tok, sd, pd in res:
        assert np.array_equal(tok, to) and np.array_equal(sd, so)
        if mode == CTC:
            assert np.array_equal(pd, po)
