"""GPU parity of the round-2 hot-path calls against the oracle:

* TDT label looping (ngpulm_tdt_loop_step through the CUDA-graph driver;
  PAPER.md:135, R25) vs the oracle's frame loop (oracle.tdt_decode),
  in both kernel paths (warp pair: B <= 592, one warp per row beyond);
* plain greedy decoding without an LM (states = NULL, lambda = 0) in the fused
  step, the persistent CTC decode and the label loop vs the oracle at lambda = 0;
* the fused step from precomputed LM rows (ngpulm_fused_greedy_step_rows, the
  overlap mode) vs the oracle's fused step, every mode and weight.

Bar: tokens, emitted sequences, counts and LM states bit-exact."""
import numpy as np
import pytest

import synth
from oracle import AED, CTC, RNNT

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2505_22857_b200 as ng  # noqa: E402
from paper_2505_22857_b200.decode import transducer_greedy_decode  # noqa: E402

from test_gpu_parity import SMALL, dev, trajectory_states, using  # noqa: E402
from test_gpu_transducer import BIAS, T, check, synth_joint  # noqa: E402

DURS = [0, 1, 2, 3, 4]


def tie_logits(rng, B, ncols):
    x = rng.standard_normal((B, ncols)).astype(np.float32)
    q = rng.random(B) < 0.2  # exact ties in some rows
    x[q] = np.round(x[q] * 4) / 4
    return x


# ---------------------------------------------------------------- TDT
@pytest.mark.parametrize("B", [40, 700])
@pytest.mark.parametrize("durs", [DURS, [1, 2], [2, 4, 8], [0]])
@pytest.mark.parametrize("lam", [0.0, 0.5])
@pytest.mark.parametrize("name", ["tri64", "ten24"])
def test_tdt_driver_matches_oracle(pairs, name, lam, durs, B):
    m, o, f = pairs[name]
    rng = np.random.default_rng(61)
    lengths = rng.integers(0, 30, size=B).astype(np.int32)
    lengths[:2] = [0, 1]
    start = np.where(rng.random(B) < 0.5, 0, o.bos_state).astype(np.int32)
    seed, temp, max_sym = 5151, 2.0, 3
    res = transducer_greedy_decode(m, synth_joint(seed, temp, o.V), T(lengths), states=T(start), lam=lam,
                                   max_symbols=max_sym, durations=durs, graph_steps=8)
    torch.cuda.synchronize()
    em, el, st, _ = o.tdt_decode(seed, lengths, start, durs, lam=lam, max_symbols=max_sym, temperature=temp,
                                 max_len=res.emitted.shape[1], blank_bias=BIAS)
    check(res, (em, el, st))


@pytest.mark.parametrize("chain", [ng.CHAIN_TABLE, ng.CHAIN_WALK])
def test_tdt_driver_config3_shape(lm6, chain):
    """TDT label looping at B=512 on the 6-gram (lambda=0.3): every row vs the oracle."""
    m, o, f = lm6
    B = 512
    lengths = np.random.default_rng(62).integers(20, 60, size=B).astype(np.int32)
    seed, temp = 1618, 8.0
    with using(m, chain):
        res = transducer_greedy_decode(m, synth_joint(seed, temp, m.V), T(lengths), lam=0.3, max_symbols=10,
                                       durations=DURS)
    torch.cuda.synchronize()
    em, el, st, steps = o.tdt_decode(seed, lengths, np.zeros(B, np.int32), DURS, lam=0.3, max_symbols=10,
                                     temperature=temp, max_len=res.emitted.shape[1], blank_bias=BIAS)
    check(res, (em, el, st))
    assert el.sum() > 0 and steps.sum() < lengths.sum() + el.sum()  # durations skip frames


# ---------------------------------------------------------------- plain greedy (no LM)
@pytest.mark.parametrize("B", [5, 300, 700])
@pytest.mark.parametrize("mode", [CTC, RNNT, AED])
def test_plain_greedy_step(pairs, mode, B):
    m, o, f = pairs["tri64"]
    rng = np.random.default_rng(63 + B)
    x = tie_logits(rng, B, o.V + 1)
    prev = rng.integers(-1, o.V + 1, size=B).astype(np.int32)
    pv = T(prev)
    for kernel in (ng.ADVANCE_AUTO, ng.ADVANCE_CTA):
        pv = T(prev)
        with using(m, kernel=kernel):
            tok = m.fused_greedy_step(mode, T(x), None, prev=pv, lam=0.0)
        torch.cuda.synchronize()
        to, _, po = o.fused_step(mode, x, np.zeros(B, np.int32), prev=prev.copy(), lam=0.0)
        assert np.array_equal(tok.cpu().numpy(), to)
        if mode == CTC:
            assert np.array_equal(pv.cpu().numpy(), po)
    with pytest.raises(ng.NgpulmError):
        m.fused_greedy_step(mode, T(x), None, prev=pv, lam=0.3)


def test_plain_ctc_decode_and_label_loop(pairs):
    m, o, f = pairs["tri64"]
    B, Tn = 37, 41
    xc = synth.ctc_logits(synth.read_sentences(f.heldout), B, Tn, o.V, seed=64)
    lengths = np.random.default_rng(65).integers(0, Tn + 1, size=B).astype(np.int32)
    pv = torch.full((B,), -1, dtype=torch.int32, device=dev())
    fr, em, el = m.ctc_greedy_decode(T(xc), None, pv, lam=0.0, lengths=T(lengths))
    torch.cuda.synchronize()
    fo, eo, elo, _, po = o.ctc_decode(xc, np.zeros(B, np.int32), lam=0.0, lengths=lengths)
    assert np.array_equal(fr.cpu().numpy(), fo) and np.array_equal(el.cpu().numpy(), elo)
    assert np.array_equal(pv.cpu().numpy(), po)
    lengths = np.random.default_rng(66).integers(0, 25, size=B).astype(np.int32)
    seed, temp = 909, 2.0
    res = transducer_greedy_decode(m, synth_joint(seed, temp, o.V), T(lengths), lam=0.0, max_symbols=3,
                                   use_lm=False)
    torch.cuda.synchronize()
    em, el, _ = o.transducer_decode(seed, lengths, np.zeros(B, np.int32), lam=0.0, max_symbols=3, temperature=temp,
                                    max_len=res.emitted.shape[1], blank_bias=BIAS)
    assert np.array_equal(res.emit_len.cpu().numpy(), el)
    got = res.emitted.cpu().numpy()
    for b in range(B):
        assert np.array_equal(got[b, : el[b]], em[b, : el[b]])
    assert (res.states.cpu().numpy() == 0).all()  # no LM state kept


# ---------------------------------------------------------------- fused step from precomputed rows
@pytest.mark.parametrize("lam", [0.0, 0.3, 3.0])
@pytest.mark.parametrize("mode", [CTC, RNNT, AED])
@pytest.mark.parametrize("name", SMALL + ["fig1"])
def test_fused_step_rows_matches_oracle(pairs, name, mode, lam):
    m, o, f = pairs[name]
    B = 2 * o.num_states + 5
    rng = np.random.default_rng(67)
    states = rng.integers(0, o.num_states, size=B).astype(np.int32)
    x = tie_logits(rng, B, o.V + 1)
    prev = rng.integers(-1, o.V + 1, size=B).astype(np.int32)
    active = (rng.random(B) < 0.9).astype(np.uint8)
    st = T(states)
    sc, nx, fi = m.advance(st)
    pv = T(prev)
    tok = m.fused_greedy_step_rows(mode, T(x), sc, nx, fi, st, prev=pv, active=T(active), lam=lam)
    torch.cuda.synchronize()
    to, so, po = o.fused_step(mode, x, states.copy(), prev=prev.copy(), active=active, lam=lam)
    assert np.array_equal(tok.cpu().numpy(), to)
    assert np.array_equal(st.cpu().numpy(), so)
    if mode == CTC:
        assert np.array_equal(pv.cpu().numpy(), po)


def test_fused_step_rows_invalid_state(pairs):
    m, o, f = pairs["tri64"]
    states = np.array([1, o.num_states + 7, 2], np.int32)
    x = tie_logits(np.random.default_rng(68), 3, o.V + 1)
    st = T(states)
    sc, nx, fi = m.advance(st)
    tok = m.fused_greedy_step_rows(RNNT, T(x), sc, nx, fi, st, lam=0.5)
    torch.cuda.synchronize()
    assert tok.cpu().numpy()[1] == -1 and st.cpu().numpy()[1] == states[1]
    assert m.check() == 1


@pytest.mark.parametrize("mode", [CTC, RNNT, AED])
def test_fused_step_rows_b512_overlapped_streams(lm6, mode):
    """The overlap mode as a decoder runs it: each step's advance on a side stream
    (ordered after the previous step), the logits on the main stream, the rows
    step after both; 12 carried steps at B=512, every row vs the oracle."""
    m, o, f = lm6
    B, steps = 512, 12
    states, _ = trajectory_states(m, f, B, seed=69)
    gen = {CTC: synth.rnnt_logits, RNNT: synth.rnnt_logits, AED: synth.aed_logits}[mode]
    xs = gen(B, steps, m.V, seed=70)
    st = T(states)
    pv = torch.full((B,), -1, dtype=torch.int32, device=dev())
    side, main = torch.cuda.Stream(), torch.cuda.current_stream()
    sc = torch.empty((B, m.V), dtype=torch.float32, device=dev())
    nx = torch.empty((B, m.V), dtype=torch.int32, device=dev())
    fi = torch.empty(B, dtype=torch.float32, device=dev())
    so, po = states.copy(), np.full(B, -1, np.int32)
    xd = T(xs)
    for k in range(steps):
        side.wait_stream(main)
        m.advance(st, sc, nx, fi, stream=side)
        main.wait_stream(side)
        tok = m.fused_greedy_step_rows(mode, xd[k], sc, nx, fi, st, prev=pv, lam=0.3)
        to, so, po = o.fused_step(mode, xs[k], so, prev=po, lam=0.3)
        assert np.array_equal(tok.cpu().numpy(), to), f"step {k}"
    assert np.array_equal(st.cpu().numpy(), so)
