"""GPU parity of the label-looping transducer driver:
paper_2505_22857_b200.decode.transducer_greedy_decode (CUDA-graph captured loop
of synthetic joint + ngpulm_transducer_loop_step) against the oracle's
frame-by-frame greedy transducer loop over its own copy of the
same counter-based synthetic joint. Bar: emitted label sequences, counts and
final LM states bit-exact."""
import numpy as np
import pytest

import synth
from oracle import RNNT

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2505_22857_b200 as ng  # noqa: E402
from paper_2505_22857_b200.decode import transducer_greedy_decode  # noqa: E402

from test_gpu_parity import dev, trajectory_states, using  # noqa: E402


BIAS = 0.75  # blank bias of the synthetic joint: blank wins most rows (as in real transducers)


def synth_joint(seed, temp, blank, bias=BIAS):
    def joint(frame, u, last, out):
        synth.joint_gpu(seed, frame, u, last, out, temperature=temp, blank=blank, blank_bias=bias)
    return joint


def T(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(dev())


def check(res, ref):
    em, el, st = res.emitted.cpu().numpy(), res.emit_len.cpu().numpy(), res.states.cpu().numpy()
    eo, elo, so = ref
    assert np.array_equal(el, elo), "emission counts differ"
    for b in range(el.size):
        n = min(el[b], em.shape[1])
        assert np.array_equal(em[b, :n], eo[b, :n]), f"row {b}: labels differ"
    assert np.array_equal(st, so), "final LM states differ"


def test_joint_twins_identical():
    """synth/joint.cu and its numpy twin produce the same bits."""
    fr = np.array([0, 3, 17, 250], np.int32)
    u = np.array([0, 1, 9, 40], np.int32)
    last = np.array([-1, 4, 0, 1023], np.int32)
    out = torch.empty((4, 1025), dtype=torch.float32, device=dev())
    synth.joint_gpu(99, T(fr), T(u), T(last), out, temperature=8.0, blank=1024, blank_bias=0.7)
    torch.cuda.synchronize()
    ref = np.stack([synth.synthetic_joint_raw(99, int(a), int(b), int(c), 1025, 8.0, 1024, 0.7)
                    for a, b, c in zip(fr, u, last)])
    assert np.array_equal(out.cpu().numpy().view(np.int32), ref.view(np.int32))


@pytest.mark.parametrize("graph_steps,use_graph", [(1, False), (7, True), (32, True)])
@pytest.mark.parametrize("max_sym", [1, 3, 10])
@pytest.mark.parametrize("lam", [0.0, 0.5, 3.0])
@pytest.mark.parametrize("name", ["tri64", "ten24"])
def test_driver_matches_oracle(pairs, name, lam, max_sym, graph_steps, use_graph):
    m, o, f = pairs[name]
    B = 40
    rng = np.random.default_rng(51)
    lengths = rng.integers(0, 30, size=B).astype(np.int32)
    lengths[:2] = [0, 1]
    start = np.where(rng.random(B) < 0.5, 0, o.bos_state).astype(np.int32)
    seed, temp = 4242, 2.0
    res = transducer_greedy_decode(m, synth_joint(seed, temp, o.V), T(lengths), states=T(start), lam=lam,
                                   max_symbols=max_sym, graph_steps=graph_steps, use_graph=use_graph)
    torch.cuda.synchronize()
    ref = o.transducer_decode(seed, lengths, start, lam=lam, max_symbols=max_sym, temperature=temp,
                              max_len=res.emitted.shape[1], blank_bias=BIAS)
    check(res, ref)


@pytest.mark.parametrize("kernel", [ng.ADVANCE_AUTO, ng.ADVANCE_WARP])
@pytest.mark.parametrize("chain", [ng.CHAIN_TABLE, ng.CHAIN_WALK])
def test_driver_with_ilm_and_truncation(pairs, chain, kernel):
    """HAT decoding (-ILM+LM) through the loop, and a max_len that truncates."""
    m, o, f = pairs["five48"]
    B = 30
    lengths = np.random.default_rng(52).integers(5, 25, size=B).astype(np.int32)
    ilm = np.random.default_rng(53).normal(-4, 2, size=(B, o.V)).astype(np.float32)
    seed, temp = 31337, 2.0
    with using(m, chain, kernel):
        res = transducer_greedy_decode(m, synth_joint(seed, temp, o.V, 0.5), T(lengths), lam=1.0, max_symbols=4,
                                       max_len=6, ilm=T(ilm), lam_ilm=0.5)
    torch.cuda.synchronize()
    ref = o.transducer_decode(seed, lengths, np.zeros(B, np.int32), lam=1.0, max_symbols=4, max_len=6,
                              temperature=temp, ilm=ilm, lam_ilm=0.5, blank_bias=0.5)
    check(res, ref)
    assert (res.emit_len.cpu().numpy() > 6).any()  # some rows were truncated


def test_driver_config3_shape(lm6):
    """RNN-T label looping at BASELINE configs[3]'s batch (B=512) on the 6-gram LM:
    every row bit-exact against the oracle's loop, lambda=0.3."""
    m, o, f = lm6
    B = 512
    lengths = np.random.default_rng(54).integers(20, 60, size=B).astype(np.int32)
    seed, temp = 2718, 8.0
    res = transducer_greedy_decode(m, synth_joint(seed, temp, m.V), T(lengths), lam=0.3, max_symbols=10)
    torch.cuda.synchronize()
    rows = np.arange(B)
    ref = o.transducer_decode(seed, lengths[rows], np.zeros(rows.size, np.int32), lam=0.3, max_symbols=10,
                              temperature=temp, max_len=res.emitted.shape[1], blank_bias=BIAS)
    em, el, st = res.emitted.cpu().numpy()[rows], res.emit_len.cpu().numpy()[rows], res.states.cpu().numpy()[rows]
    assert np.array_equal(el, ref[1]) and np.array_equal(st, ref[2])
    for i in range(rows.size):
        assert np.array_equal(em[i, : el[i]], ref[0][i, : el[i]])
    assert el.sum() > 0


def test_driver_large_batch_single_warp_path(pairs):
    """B > 592 rows: the loop step runs one warp per row (not the pair kernel)."""
    m, o, f = pairs["tri64"]
    B = 700
    lengths = np.random.default_rng(55).integers(0, 12, size=B).astype(np.int32)
    seed, temp = 777, 2.0
    res = transducer_greedy_decode(m, synth_joint(seed, temp, o.V), T(lengths), lam=0.7, max_symbols=3)
    torch.cuda.synchronize()
    check(res, o.transducer_decode(seed, lengths, np.zeros(B, np.int32), lam=0.7, max_symbols=3, temperature=temp,
                                   max_len=res.emitted.shape[1], blank_bias=BIAS))


@pytest.mark.parametrize("durations", [None, (0, 1, 2)])
@pytest.mark.parametrize("B", [64, 512, 700])
def test_driver_inputs_ready(lm6, B, durations):
    """The label-looping driver with NGPULM_STEP_INPUTS_READY (the synthetic joint is a
    plain launch): one warp per row, the state read once and the logits copied at the
    step's start; identical to the flags == 0 driver and, on every row, to the oracle
    (RNN-T and TDT, 6-gram, lambda = 0.3)."""
    m, o, f = lm6
    lengths = np.random.default_rng(B + 1).integers(10, 40, size=B).astype(np.int32)
    seed, temp = 4242, 8.0
    ncols = m.V + 1 + (len(durations) if durations else 0)

    def joint(frame, u, last, out):
        synth.joint_gpu(seed, frame, u, last, out, temperature=temp, blank=m.V, blank_bias=BIAS)

    res = [transducer_greedy_decode(m, joint, T(lengths), lam=0.3, max_symbols=4, durations=durations,
                                    joint_plain_launch=ready) for ready in (False, True)]
    torch.cuda.synchronize()
    a, b = res
    assert np.array_equal(a.emit_len.cpu().numpy(), b.emit_len.cpu().numpy())
    assert np.array_equal(a.emitted.cpu().numpy(), b.emitted.cpu().numpy())
    assert np.array_equal(a.states.cpu().numpy(), b.states.cpu().numpy())
    if durations is None:
        rows = np.arange(B)
        ref = o.transducer_decode(seed, lengths[rows], np.zeros(rows.size, np.int32), lam=0.3, max_symbols=4,
                                  temperature=temp, max_len=b.emitted.shape[1], blank_bias=BIAS)
        el, st = b.emit_len.cpu().numpy()[rows], b.states.cpu().numpy()[rows]
        assert np.array_equal(el, ref[1]) and np.array_equal(st, ref[2])
    assert ncols > m.V
