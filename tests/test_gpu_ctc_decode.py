"""GPU parity of the persistent whole-utterance CTC decode (ngpulm_ctc_greedy_decode,
SURVEY.md §8(f) f1) against the oracle's decode (oracle_ctc_decode: the frame loop
of SPEC.md:307-316 over the oracle's fused CTC step) and against T launches of the
per-frame fused step. Bar: frames, emissions, states and prev bit-exact."""
import numpy as np
import pytest

import synth
from oracle import CTC, Oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2505_22857_b200 as ng  # noqa: E402

from test_gpu_parity import dev, using  # noqa: E402


def gpu_decode(m, x, start, prev0, lam, lengths=None, blank=None, view=None):
    xd = torch.from_numpy(x).to(dev()) if view is None else view
    st = torch.from_numpy(np.ascontiguousarray(start, np.int32)).to(dev())
    pv = torch.from_numpy(np.ascontiguousarray(prev0, np.int32)).to(dev())
    ln = None if lengths is None else torch.from_numpy(np.ascontiguousarray(lengths, np.int32)).to(dev())
    fr, em, el = m.ctc_greedy_decode(xd, st, pv, lam=lam, blank_id=blank, lengths=ln)
    torch.cuda.synchronize()
    return fr.cpu().numpy(), em.cpu().numpy(), el.cpu().numpy(), st.cpu().numpy(), pv.cpu().numpy()


def assert_same(g, o):
    fr, em, el, st, pv = g
    fo, eo, elo, so, po = o
    assert np.array_equal(fr, fo), "frame selections differ"
    assert np.array_equal(el, elo), "emission counts differ"
    for b in range(fr.shape[0]):
        assert np.array_equal(em[b, : el[b]], eo[b, : elo[b]]), f"row {b}: emissions differ"
    assert np.array_equal(st, so) and np.array_equal(pv, po), "final states / prev differ"


@pytest.mark.parametrize("kernel", [ng.ADVANCE_AUTO, ng.ADVANCE_WARP])
@pytest.mark.parametrize("chain", [ng.CHAIN_TABLE, ng.CHAIN_WALK])
@pytest.mark.parametrize("lam", [0.0, 0.3, 3.0])
@pytest.mark.parametrize("name", ["tiny3", "tri64", "five48", "ten24"])
def test_decode_matches_oracle(pairs, name, lam, chain, kernel):
    m, o, f = pairs[name]
    sents = synth.read_sentences(f.heldout)
    B, T = 37, 41
    x = synth.ctc_logits(sents, B, T, o.V, seed=11)
    rng = np.random.default_rng(3)
    lengths = rng.integers(0, T + 1, size=B).astype(np.int32)
    lengths[:3] = [0, T, 1]
    start = synth.uniform_states(o.num_states, B, seed=6)
    start[::5] = o.bos_state
    prev0 = rng.integers(-1, o.V, size=B).astype(np.int32)
    with using(m, chain, kernel):
        g = gpu_decode(m, x, start, prev0, lam, lengths)
    assert_same(g, o.ctc_decode(x, start, prev=prev0, lam=lam, lengths=lengths))


@pytest.mark.parametrize("blank", [0, 17])
def test_decode_blank_column_inside(pairs, blank):
    """blank_id != V: tokens v >= blank sit in column v+1 (R19)."""
    m, o, f = pairs["tri64"]
    sents = synth.read_sentences(f.heldout)
    B, T = 20, 30
    x = synth.ctc_logits(sents, B, T, o.V, seed=12, blank=blank)
    start = np.zeros(B, np.int32)
    prev0 = np.full(B, -1, np.int32)
    g = gpu_decode(m, x, start, prev0, 1.0, blank=blank)
    assert_same(g, o.ctc_decode(x, start, prev=prev0, lam=1.0, blank_id=blank))


def test_decode_equals_per_frame_steps_config2(lm6):
    """BASELINE configs[2]: B=256, T=500, V=1024+blank, 6-gram, lambda=0.3 — one
    persistent launch == 500 launches of the fused step (all rows, bit-exact), and
    == the oracle on every row (ragged lengths), and the bench's launch (every row
    at full length, no lengths array) == the oracle on every row."""
    m, o, f = lm6
    B, T = 256, 500
    sents = synth.read_sentences(f.heldout)
    x = synth.ctc_logits(sents, B, T, m.V, seed=4)
    lengths = np.random.default_rng(5).integers(T // 2, T + 1, size=B).astype(np.int32)
    lengths[0] = T
    xd = torch.from_numpy(x).to(dev())
    start = np.zeros(B, np.int32)
    prev0 = np.full(B, -1, np.int32)
    g = gpu_decode(m, x, start, prev0, 0.3, lengths, view=xd)
    # per-frame fused steps with active = t < len
    st = torch.zeros(B, dtype=torch.int32, device=dev())
    pv = torch.full((B,), -1, dtype=torch.int32, device=dev())
    ln = torch.from_numpy(lengths).to(dev())
    frames = torch.empty((T, B), dtype=torch.int32, device=dev())
    for t in range(T):
        act = (ln > t).to(torch.uint8)
        m.fused_greedy_step(CTC, xd[:, t], st, prev=pv, active=act, lam=0.3, tokens_out=frames[t])
    torch.cuda.synchronize()
    assert np.array_equal(g[0], frames.cpu().numpy().T)
    assert np.array_equal(g[3], st.cpu().numpy()) and np.array_equal(g[4], pv.cpu().numpy())
    assert_same(g, o.ctc_decode(x, start, prev=prev0, lam=0.3, lengths=lengths))
    gb = gpu_decode(m, x, start, prev0, 0.3, None, view=xd)  # the bench's call
    assert_same(gb, o.ctc_decode(x, start, prev=prev0, lam=0.3))
    # the LM changed decisions relative to lambda = 0 (the test means something)
    g0 = gpu_decode(m, x, start, prev0, 0.0, lengths, view=xd)
    assert (g0[0] != g[0]).any()


def test_decode_strided_views_and_edge_cases(pairs):
    m, o, f = pairs["five48"]
    sents = synth.read_sentences(f.heldout)
    B, T = 9, 25
    big = synth.ctc_logits(sents, B, T + 3, o.V, seed=13)
    view = torch.from_numpy(big).to(dev())[:, 2:2 + T]   # frame rows start at odd offsets
    x = np.ascontiguousarray(big[:, 2:2 + T])
    start = synth.uniform_states(o.num_states, B, seed=2)
    prev0 = np.full(B, -1, np.int32)
    g = gpu_decode(m, x, start, prev0, 0.7, view=view)
    assert_same(g, o.ctc_decode(x, start, prev=prev0, lam=0.7))
    # time-major [T, B, V+1] storage, decoded through a transposed view
    tm = torch.from_numpy(np.ascontiguousarray(x.transpose(1, 0, 2))).to(dev())
    g2 = gpu_decode(m, x, start, prev0, 0.7, view=tm.transpose(0, 1))
    assert_same(g2, o.ctc_decode(x, start, prev=prev0, lam=0.7))
    # an invalid start state decides nothing; the others are unaffected
    bad = start.copy()
    bad[4] = o.num_states + 3
    g3 = gpu_decode(m, x, bad, prev0, 0.7)
    assert (g3[0][4] == -1).all() and g3[2][4] == 0 and g3[3][4] == bad[4]
    keep = np.arange(B) != 4
    assert np.array_equal(g3[0][keep], g[0][keep])
    assert m.check() == 4
    # B = 0 and T = 0 are no-ops
    e = torch.empty((0, T, o.V + 1), dtype=torch.float32, device=dev())
    z = torch.empty(0, dtype=torch.int32, device=dev())
    m.ctc_greedy_decode(e, z, z.clone(), lam=0.3)
    g4 = gpu_decode(m, x[:, :0], start, prev0, 0.7, view=view[:, :0])
    assert g4[2].sum() == 0 and np.array_equal(g4[3], start)


def test_decode_refuses_v_not_multiple_of_4(pairs):
    m, o, _ = pairs["fig1"]   # V = 6
    x = torch.zeros((2, 3, o.V + 1), dtype=torch.float32, device=dev())
    st = torch.zeros(2, dtype=torch.int32, device=dev())
    with pytest.raises(ng.NgpulmError):
        m.ctc_greedy_decode(x, st, st.clone() - 1)


@pytest.mark.parametrize("lam", [0.0, 0.3, 3.0])
@pytest.mark.parametrize("B,T", [(1, 700), (7, 300), (64, 256), (300, 200)])
def test_segmented_decode_matches_oracle_and_sequential(lm6, B, T, lam):
    """The segment-parallel decode (frames_out and emit_out given, T >= 128): every
    row vs the oracle's decode and vs the single-chain kernel (frames_out = NULL),
    with ragged lengths around the segment boundaries (0, 1, 63, 64, 65, T)."""
    m, o, f = lm6
    rng = np.random.default_rng(B * 7 + T)
    x = synth.ctc_logits(synth.read_sentences(f.heldout), B, T, m.V, seed=B + T)
    lengths = rng.integers(0, T + 1, size=B).astype(np.int32)
    special = [0, 1, 63, 64, 65, T, T // 2, T - 1]
    lengths[: min(B, len(special))] = special[: min(B, len(special))]
    start = np.where(rng.random(B) < 0.5, 0, m.bos_state).astype(np.int32)
    prev0 = np.where(rng.random(B) < 0.7, -1, rng.integers(0, m.V, B)).astype(np.int32)
    g = gpu_decode(m, x, start, prev0, lam, lengths)
    assert_same(g, o.ctc_decode(x, start, prev=prev0, lam=lam, lengths=lengths))
    # the single-chain kernel (no frame records): same emissions, states, prev
    xd = torch.from_numpy(x).cuda()
    st, pv = torch.from_numpy(start.copy()).cuda(), torch.from_numpy(prev0.copy()).cuda()
    _, em, el = m.ctc_greedy_decode(xd, st, pv, lam=lam, lengths=torch.from_numpy(lengths).cuda(),
                                    want_frames=False)
    torch.cuda.synchronize()
    el = el.cpu().numpy()
    assert np.array_equal(el, g[2]) and np.array_equal(st.cpu().numpy(), g[3]) and np.array_equal(pv.cpu().numpy(), g[4])
    emn = em.cpu().numpy()
    for r in range(B):
        assert np.array_equal(emn[r, : el[r]], g[1][r, : el[r]])


def T_(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(dev())


@pytest.mark.parametrize("kernel", [ng.ADVANCE_AUTO, ng.ADVANCE_WARP])
def test_segmented_decode_edge_cases(pairs, kernel):
    """Segments on a small LM (tiny path with AUTO, unpacked global path with WARP):
    an invalid start state, all-NaN frames (no column selected), ties, blank column 0."""
    m, o, f = pairs["five48"]
    B, T = 40, 260
    rng = np.random.default_rng(9)
    x = rng.standard_normal((B, T, o.V + 1)).astype(np.float32)
    x[:, :, 0] += 1.0
    x[3, 70:75] = np.nan          # frames selecting nothing, inside a segment
    x[4, 64] = np.nan             # on a segment boundary
    x[5, ::7] = np.round(x[5, ::7] * 2) / 2  # ties
    start = synth.uniform_states(o.num_states, B, seed=10)
    start[6] = o.num_states + 5   # invalid
    prev0 = np.full(B, -1, np.int32)
    lengths = np.full(B, T, np.int32)
    m.set_advance_kernel(kernel)
    try:
        g = gpu_decode(m, x, start, prev0, 0.8, lengths, blank=0)
        assert m.check() == 6
    finally:
        m.set_advance_kernel(ng.ADVANCE_AUTO)
    ok = np.ones(B, bool)
    ok[[3, 4, 6]] = False  # NaN frames are unspecified (R15): rows 3, 4 are checked against the single chain
    ref = o.ctc_decode(x[ok], start[ok], prev=prev0[ok], lam=0.8, lengths=lengths[ok], blank_id=0)
    assert np.array_equal(g[0][ok], ref[0]) and np.array_equal(g[2][ok], ref[2])
    assert np.array_equal(g[3][ok], ref[3]) and np.array_equal(g[4][ok], ref[4])
    assert (g[0][6] == -1).all() and g[2][6] == 0 and g[3][6] == start[6]
    # every row, NaN frames included: the segments agree with the single-chain kernel
    m.set_advance_kernel(kernel)
    try:
        st, pv = T_(start), T_(prev0)
        _, em, el = m.ctc_greedy_decode(T_(x), st, pv, lam=0.8, blank_id=0, lengths=T_(lengths), want_frames=False)
        torch.cuda.synchronize()
    finally:
        m.set_advance_kernel(ng.ADVANCE_AUTO)
    el = el.cpu().numpy()
    assert np.array_equal(el, g[2]) and np.array_equal(st.cpu().numpy(), g[3]) and np.array_equal(pv.cpu().numpy(), g[4])
    emn = em.cpu().numpy()
    for r in range(B):
        assert np.array_equal(emn[r, : el[r]], g[1][r, : el[r]])
    assert (g[0][3, 70:75] == -1).all() and g[0][4, 64] == -1  # a NaN frame selects nothing
    assert m.check() == 6  # (the single-chain run set the sticky word again; read and clear it)


@pytest.mark.parametrize("kernel", [ng.ADVANCE_AUTO, ng.ADVANCE_WARP])
def test_segmented_decode_long_chains(pairs, kernel):
    """Two segments per row (B in (395, 592]) of ~450 frames with an emission on most
    frames: a chain rebuilds its row more than 255 times, so the 8-bit rebuild
    generations of the row entries wrap inside one chain; every row vs the oracle."""
    m, o, f = pairs["tri64"]
    B, T = 420, 900
    rng = np.random.default_rng(21)
    x = rng.standard_normal((B, T, o.V + 1)).astype(np.float32)
    x[:, :, o.V] -= 1.0  # blank rarely wins: an emission on most frames
    start = synth.uniform_states(o.num_states, B, seed=22)
    prev0 = np.full(B, -1, np.int32)
    lengths = np.full(B, T, np.int32)
    lengths[:4] = [T - 1, 451, 450, 449]
    m.set_advance_kernel(kernel)
    try:
        g = gpu_decode(m, x, start, prev0, 0.1, lengths)
    finally:
        m.set_advance_kernel(ng.ADVANCE_AUTO)
    assert (g[2] > 600).sum() > B // 2  # most rows emit on most frames: > 255 rebuilds per segment
    assert_same(g, o.ctc_decode(x, start, prev=prev0, lam=0.1, lengths=lengths))
