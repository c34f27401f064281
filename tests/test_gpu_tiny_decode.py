"""Tiny-LM path of the decode kernels (the paper's keyword-
biasing LM used in greedy decoding): a keyword-biasing-sized LM
(chain table + packed arcs <= 96 KiB, info.tiny_resident) is copied into every
CTA's shared memory by the fused greedy step, the label-looping step and the
persistent CTC decode. Each is compared bit-exact with the global-memory path
(ADVANCE_WARP: same model read from HBM/L2) and with the oracle.
"""
import numpy as np
import pytest

import synth
from oracle import AED, CTC, RNNT, Oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2505_22857_b200 as ng  # noqa: E402
from paper_2505_22857_b200.decode import transducer_greedy_decode  # noqa: E402


def dev():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return torch.device("cuda:0")


def T(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(dev())


@pytest.fixture(scope="module")
def bias_lm(lm_dir):
    """V = 1024 3-gram from 600 corpus tokens (~800 states): the bench's keyword-biasing LM."""
    f = synth.make_lm(lm_dir, 1024, 3, tokens=600, seed=11, heldout=200, tag="tiny_bias")
    m = ng.load_arpa(f.arpa, vocab_size=1024, device=0)
    assert m.info.tiny_resident == 1
    return m, Oracle(f.arpa, vocab_size=1024), f


def both_paths(m, fn):
    """fn() on the tiny (AUTO) path and on the global-memory path (ADVANCE_WARP)."""
    a = fn()
    m.set_advance_kernel(ng.ADVANCE_WARP)
    try:
        b = fn()
    finally:
        m.set_advance_kernel(ng.ADVANCE_AUTO)
    return a, b


@pytest.mark.parametrize("B", [5, 148, 700, 2000])
@pytest.mark.parametrize("mode", [CTC, RNNT, AED])
def test_fused_step_tiny_vs_global_vs_oracle(bias_lm, mode, B):
    m, o, _ = bias_lm
    rng = np.random.default_rng(B + mode)
    states = synth.uniform_states(o.num_states, B, seed=B)
    x = rng.standard_normal((B, m.V + 1)).astype(np.float32)
    prev = np.where(rng.random(B) < 0.5, -1, rng.integers(0, m.V, B)).astype(np.int32)
    active = (rng.random(B) < 0.9).astype(np.uint8)

    def run():
        st, pv = T(states), T(prev)
        tok = m.fused_greedy_step(mode, T(x), st, prev=pv, active=T(active), lam=1.5)
        torch.cuda.synchronize()
        return tok.cpu().numpy(), st.cpu().numpy(), pv.cpu().numpy()
    a, b = both_paths(m, run)
    to, so, po = o.fused_step(mode, x, states, prev=prev, active=active, lam=1.5)
    for u, v in zip(a, b):
        assert np.array_equal(u, v)
    assert np.array_equal(a[0], to) and np.array_equal(a[1], so)
    if mode == CTC:
        assert np.array_equal(a[2], po)


def test_fused_step_ilm_tiny(bias_lm):
    m, o, _ = bias_lm
    B = 300
    rng = np.random.default_rng(3)
    states = synth.uniform_states(o.num_states, B, seed=4)
    x = rng.standard_normal((B, m.V + 1)).astype(np.float32)
    ilm = (rng.standard_normal((B, m.V)) - 3).astype(np.float32)

    def run():
        st = T(states)
        tok = m.fused_greedy_step_ilm(RNNT, T(x), st, T(ilm), 0.4, lam=1.0)
        torch.cuda.synchronize()
        return tok.cpu().numpy(), st.cpu().numpy()
    a, b = both_paths(m, run)
    to, so, _ = o.fused_step_ilm(RNNT, x, states, ilm, 0.4, lam=1.0)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[0], to) and np.array_equal(a[1], so)


@pytest.mark.parametrize("B", [3, 256])
def test_ctc_decode_tiny(bias_lm, B):
    m, o, f = bias_lm
    Tn = 120
    x = synth.ctc_logits(synth.read_sentences(f.heldout), B, Tn, m.V, seed=9)
    lengths = np.random.default_rng(5).integers(0, Tn + 1, size=B).astype(np.int32)
    start = np.zeros(B, np.int32)

    def run():
        st, pv = T(start), T(np.full(B, -1, np.int32))
        fr, em, el = m.ctc_greedy_decode(T(x), st, pv, lam=1.0, lengths=T(lengths))
        torch.cuda.synchronize()
        return fr.cpu().numpy(), el.cpu().numpy(), st.cpu().numpy(), em.cpu().numpy()
    a, b = both_paths(m, run)
    for u, v in zip(a, b):
        assert np.array_equal(u, v)
    ref = o.ctc_decode(x, start, prev=np.full(B, -1, np.int32), lam=1.0, lengths=lengths)
    assert np.array_equal(a[0], ref[0]) and np.array_equal(a[1], ref[2])
    # the LM changed decisions (the test means something)
    ref0 = o.ctc_decode(x, start, prev=np.full(B, -1, np.int32), lam=0.0, lengths=lengths)
    assert not np.array_equal(ref[0], ref0[0])


@pytest.mark.parametrize("durs", [None, [0, 1, 2, 4]])
@pytest.mark.parametrize("B", [8, 700])
def test_label_loop_tiny(bias_lm, durs, B):
    m, o, _ = bias_lm
    lengths = np.random.default_rng(6).integers(0, 25, size=B).astype(np.int32)
    seed, temp = 4242, 2.0

    def joint(frame, u, last, out):
        synth.joint_gpu(seed, frame, u, last, out, temperature=temp, blank=m.V, blank_bias=0.75)

    def run():
        res = transducer_greedy_decode(m, joint, T(lengths), lam=1.0, max_symbols=3, durations=durs,
                                       graph_steps=8)
        torch.cuda.synchronize()
        return res.emitted.cpu().numpy(), res.emit_len.cpu().numpy(), res.states.cpu().numpy()
    a, b = both_paths(m, run)
    for u, v in zip(a, b):
        assert np.array_equal(u, v)
    ml = a[0].shape[1]
    if durs is None:
        em, el, st = o.transducer_decode(seed, lengths, np.zeros(B, np.int32), lam=1.0, max_symbols=3,
                                         temperature=temp, max_len=ml, blank_bias=0.75)
    else:
        em, el, st, _ = o.tdt_decode(seed, lengths, np.zeros(B, np.int32), durs, lam=1.0, max_symbols=3,
                                     temperature=temp, max_len=ml, blank_bias=0.75)
    assert np.array_equal(a[1], el) and np.array_equal(a[2], st)
    for r in range(B):
        assert np.array_equal(a[0][r, : min(el[r], ml)], em[r, : min(el[r], ml)])
