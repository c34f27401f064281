"""GPU parity at BASELINE.json's full LM sizes (configs[3] and configs[4]), in the
launch configurations the bench and the decoders use, against the oracle on
every row of the launch plus properties that hold for every row:

* configs[3]: token 8-gram LM (~4.9M n-grams, V=1024), RNN-T fused greedy steps
  over B=512 rows (label-looping shape: per-step logits, state carried), and
  advance at B=512;
* configs[4]: token 10-gram LM (~20M n-grams, V=1024, ~1.9 GB resident with the
  chain table), advance at B=4096, the B=4096 batch sharded 4 ways (the per-GPU
  share at 4 GPUs) == unsharded, and a replica == the original.

Bar: next-state ids and argmax tokens bit-exact, scores bit-exact against the
oracle's Algorithm-1-order float32 value; per-row normalization
sum_v exp(score) + exp(final) = 1 (Witten-Bell LMs are normalized).
"""
import numpy as np
import pytest

import synth
from oracle import RNNT, Oracle

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu, pytest.mark.slow]

import paper_2505_22857_b200 as ng  # noqa: E402

from test_gpu_parity import dev, gpu_advance, same_bits, trajectory_states, using  # noqa: E402


@pytest.fixture(scope="module")
def lm8(lm_dir):
    f = synth.make_lm(lm_dir, 1024, 8, tokens=1_600_000, seed=5, heldout=2000, tag="cfg3_8gram")
    return ng.load_arpa(f.arpa, vocab_size=1024, device=0), Oracle(f.arpa, vocab_size=1024), f


@pytest.fixture(scope="module")
def lm10(lm_dir):
    f = synth.make_lm(lm_dir, 1024, 10, tokens=5_200_000, seed=7, heldout=2000, tag="cfg4_10gram")
    return ng.load_arpa(f.arpa, vocab_size=1024, device=0), Oracle(f.arpa, vocab_size=1024), f


def normalized(s, fin, tol=1e-4):
    tot = np.exp(s.astype(np.float64)).sum(1) + np.exp(fin.astype(np.float64))
    return np.max(np.abs(tot - 1)) < tol


def test_config3_sizes(lm8):
    m, o, f = lm8
    n = sum(int(line.split("=")[1]) for line in open(f.arpa).read().split("\n\n")[0].splitlines()[1:])
    assert 4_500_000 < n < 6_000_000 and m.order == 8


@pytest.mark.parametrize("kernel", [ng.ADVANCE_AUTO, ng.ADVANCE_WARP, ng.ADVANCE_CTA])
def test_config3_rnnt_fused_steps_b512(lm8, kernel):
    """16 label-looping-shaped steps (B=512, per-step logits, state carried from
    step to step, ~50 % blank rows), every row and step bit-exact vs the oracle."""
    m, o, f = lm8
    B, steps = 512, 16
    states, _ = trajectory_states(m, f, B, seed=21)
    xs = synth.rnnt_logits(B, steps, m.V, seed=22)
    st_d = torch.from_numpy(states.copy()).to(dev())
    so = states.copy()
    with using(m, kernel=kernel):
        for k in range(steps):
            tok = m.fused_greedy_step(RNNT, torch.from_numpy(xs[k]).to(dev()), st_d, lam=0.3)
            to, so, _ = o.fused_step(RNNT, xs[k], so, lam=0.3)
            assert np.array_equal(tok.cpu().numpy(), to), f"step {k}: tokens differ"
    assert np.array_equal(st_d.cpu().numpy(), so)


def test_config3_advance_b512(lm8):
    m, o, f = lm8
    states, _ = trajectory_states(m, f, 512, seed=23)
    s, n, fin = gpu_advance(m, states)
    s32, s64, n_o, _ = o.rows(states)  # every row
    f32, _ = o.finals(states)
    assert np.array_equal(n, n_o) and same_bits(s, s32) and same_bits(fin, f32)
    assert np.max(np.abs(s - s64)) < 1e-5
    assert normalized(s, fin)


def test_config4_sizes(lm10):
    m, o, f = lm10
    n = sum(int(line.split("=")[1]) for line in open(f.arpa).read().split("\n\n")[0].splitlines()[1:])
    assert 18_000_000 < n < 23_000_000 and m.order == 10


def test_config4_advance_b4096_sharded_and_replica(lm10):
    """configs[4]: B=4096 over a replicated 10-gram trie. One launch at B=4096, the
    same rows as 4 shards of 1024 (each GPU's share at 4 GPUs) and on a replica:
    bit-identical; every row vs the oracle; normalization on every row."""
    m, o, f = lm10
    B = 4096
    states, _ = trajectory_states(m, f, B, seed=31)
    s, n, fin = gpu_advance(m, states)
    s32, s64, n_o, _ = o.rows(states)  # every row of the launch
    f32, _ = o.finals(states)
    assert np.array_equal(n, n_o) and same_bits(s, s32) and same_bits(fin, f32)
    assert np.max(np.abs(s - s64)) < 2e-5   # f32 bound at 10 levels
    assert normalized(s, fin)
    parts = [gpu_advance(m, states[i:i + 1024]) for i in range(0, B, 1024)]
    assert same_bits(np.concatenate([p[0] for p in parts]), s)
    assert np.array_equal(np.concatenate([p[1] for p in parts]), n)
    r = m.replicate(0)
    s2, n2, f2 = gpu_advance(r, states)
    assert same_bits(s2, s) and np.array_equal(n2, n) and same_bits(f2, fin)
    assert m.check() == -1


def test_config3_label_looping_decode_b512(lm8):
    """configs[3] end to end: label-looping greedy transducer decoding with fusion
    (B=512 utterances, 8-gram ~4.9M n-grams, lambda=0.3) through the CUDA-graph
    driver, against the oracle's frame-by-frame loop on every utterance."""
    from paper_2505_22857_b200.decode import transducer_greedy_decode
    m, o, f = lm8
    B = 512
    lengths = np.random.default_rng(41).integers(20, 60, size=B).astype(np.int32)
    seed, temp, bias = 8080, 8.0, 0.75

    def joint(frame, u, last, out):
        synth.joint_gpu(seed, frame, u, last, out, temperature=temp, blank=m.V, blank_bias=bias)
    res = transducer_greedy_decode(m, joint, torch.from_numpy(lengths).to(dev()), lam=0.3, max_symbols=10)
    torch.cuda.synchronize()
    rows = np.arange(B)
    eo, elo, so = o.transducer_decode(seed, lengths[rows], np.zeros(rows.size, np.int32), lam=0.3, max_symbols=10,
                                      temperature=temp, max_len=res.emitted.shape[1], blank_bias=bias)
    em, el, st = res.emitted.cpu().numpy()[rows], res.emit_len.cpu().numpy()[rows], res.states.cpu().numpy()[rows]
    assert np.array_equal(el, elo) and np.array_equal(st, so)
    for i in range(rows.size):
        assert np.array_equal(em[i, : el[i]], eo[i, : el[i]])
    assert el.sum() > 0


def test_config4_binary_reload(lm10, tmp_path):
    """f4: the 20M-n-gram model saved as NGLM and reloaded without the ARPA parse
    answers bit-identically (and loads several times faster than the ARPA)."""
    import time
    m, o, f = lm10
    p = str(tmp_path / "lm10.nglm")
    m.save(p)
    t0 = time.perf_counter()
    r = ng.load_binary(p, device=0)
    t_bin = time.perf_counter() - t0
    t0 = time.perf_counter()
    ng.load_arpa(f.arpa, vocab_size=1024, device=-1)
    t_arpa = time.perf_counter() - t0
    states, _ = trajectory_states(m, f, 1024, seed=33)
    a, b = gpu_advance(m, states), gpu_advance(r, states)
    assert same_bits(a[0], b[0]) and np.array_equal(a[1], b[1]) and same_bits(a[2], b[2])
    print(f"NGLM reload {t_bin:.1f} s (incl. upload) vs ARPA parse+build {t_arpa:.1f} s (host only)")
    assert t_bin < t_arpa
