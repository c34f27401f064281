"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle, element by element.

Bar (BASELINE.json north_star): next-state ids and argmax tokens bit-exact;
scores within 1e-5 (f32). Against the oracle's Algorithm-1-order float32 value
(score32) the kernels are required to be BIT-EXACT, and
within 1e-5 of the f64 definition where the f32 bound allows it.
"""
import numpy as np
import pytest

import synth
from oracle import AED, CTC, RNNT, Oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2505_22857_b200 as ng  # noqa: E402

SMALL = ["uni16", "bi16", "tiny3", "tri64", "five48", "ten24"]


def dev():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return torch.device("cuda:0")


def same_bits(a, b):
    return np.array_equal(np.asarray(a, np.float32).view(np.int32), np.asarray(b, np.float32).view(np.int32))


KERNELS = [ng.ADVANCE_AUTO, ng.ADVANCE_WARP, ng.ADVANCE_CTA]


class using:
    """Temporarily select the chain mode / advance kernel of a model."""

    def __init__(self, m, chain=ng.CHAIN_TABLE, kernel=ng.ADVANCE_AUTO):
        self.m, self.chain, self.kernel = m, chain, kernel

    def __enter__(self):
        self.m.set_chain_mode(self.chain)
        self.m.set_advance_kernel(self.kernel)

    def __exit__(self, *exc):
        self.m.set_chain_mode(ng.CHAIN_TABLE)
        self.m.set_advance_kernel(ng.ADVANCE_AUTO)


def gpu_advance(m, states_np):
    st = torch.from_numpy(np.ascontiguousarray(states_np, np.int32)).to(dev())
    s, n, f = m.advance(st)
    torch.cuda.synchronize()
    return s.cpu().numpy(), n.cpu().numpy(), f.cpu().numpy()


@pytest.mark.parametrize("kernel", KERNELS)
@pytest.mark.parametrize("chain", [ng.CHAIN_TABLE, ng.CHAIN_WALK])
@pytest.mark.parametrize("name", SMALL + ["fig1"])
def test_advance_exhaustive_small(pairs, name, chain, kernel):
    """All states x all tokens of every small LM (config 0 = tiny3), both ways of
    obtaining the back-off levels (load-time chain table / Algorithm 1 walk),
    every advance kernel."""
    m, o, _ = pairs[name]
    states = np.arange(o.num_states, dtype=np.int32)
    with using(m, chain, kernel):
        s, n, f = gpu_advance(m, states)
    s32, s64, n_o, _ = o.rows(states)
    f32, f64 = o.finals(states)
    assert np.array_equal(n, n_o)
    assert same_bits(s, s32)
    assert same_bits(f, f32)
    assert np.max(np.abs(s - s64)) < 1e-5
    assert m.check() == -1


def test_config0_batches_of_4(pairs):
    """BASELINE configs[0]: tiny 3-gram V=32, batch 4 states."""
    m, o, _ = pairs["tiny3"]
    rng = np.random.default_rng(11)
    for _ in range(10):
        states = rng.integers(0, o.num_states, size=4).astype(np.int32)
        s, n, f = gpu_advance(m, states)
        s32, _, n_o, _ = o.rows(states, want64=False)
        assert np.array_equal(n, n_o) and same_bits(s, s32)


def test_unaligned_outputs_scalar_path(pairs):
    m, o, _ = pairs["tri64"]
    B, V = 37, m.V
    states = torch.arange(B, dtype=torch.int32, device=dev()) * 3 % o.num_states
    sc = torch.empty(B * V + 1, dtype=torch.float32, device=dev())[1:]
    nx = torch.empty(B * V + 1, dtype=torch.int32, device=dev())[1:]
    m.advance(states, scores=sc, next=nx, want_final=False)
    torch.cuda.synchronize()
    s32, _, n_o, _ = o.rows(states.cpu().numpy(), want64=False)
    assert same_bits(sc.cpu().numpy().reshape(B, V), s32)
    assert np.array_equal(nx.cpu().numpy().reshape(B, V), n_o)


def test_invalid_state_and_empty_batch(pairs):
    m, o, _ = pairs["tri64"]
    states = np.array([0, 5, o.num_states + 3, 2, -1], dtype=np.int32)
    s, n, f = gpu_advance(m, states)
    assert np.isnan(s[2]).all() and (n[2] == -1).all() and np.isnan(f[2])
    assert m.check() == 2
    assert m.check() == -1                     # sticky word cleared by the read
    s32, _, n_o, _ = o.rows(states[[0, 1, 3]], want64=False)
    assert same_bits(s[[0, 1, 3]], s32) and np.array_equal(n[[0, 1, 3]], n_o)
    e = torch.empty(0, dtype=torch.int32, device=dev())
    m.advance(e)                                # B = 0: no-op
    fin = m.final(torch.tensor([1, -7], dtype=torch.int32, device=dev()))
    torch.cuda.synchronize()
    assert np.isnan(fin[1].item()) and m.check() == 1


def trajectory_states(m, f, n, seed):
    ctx = synth.sample_contexts(synth.read_sentences(f.heldout), f.order, n, seed)
    return np.array([m.state_of(b, t) for b, t in ctx], dtype=np.int32), ctx


@pytest.mark.parametrize("kernel", KERNELS)
@pytest.mark.parametrize("chain", [ng.CHAIN_TABLE, ng.CHAIN_WALK])
def test_config1_b128_full_rows(lm6, chain, kernel):
    m, o, f = lm6
    assert m.info.num_arcs > 500_000 and 800_000 < sum(1 for _ in open(f.arpa)) < 1_300_000
    assert m.info.packed_arcs == 1
    st_traj, ctx = trajectory_states(m, f, 96, seed=2)
    # the library's and the oracle's context -> state maps agree (R6, R7)
    assert [o.state_of(b, t) for b, t in ctx] == st_traj.tolist()
    states = np.concatenate([st_traj, synth.uniform_states(m.num_states, 32, seed=3)])
    with using(m, chain, kernel):
        s, n, fin = gpu_advance(m, states)
    s32, s64, n_o, lv = o.rows(states)
    f32, _ = o.finals(states)
    assert np.array_equal(n, n_o) and same_bits(s, s32) and same_bits(fin, f32)
    assert np.max(np.abs(s - s64)) < 1e-5
    assert lv.max() <= 6


@pytest.mark.parametrize("kernel", KERNELS)
def test_headline_b1024_every_row(lm6, kernel):
    """The bench launch (B=1024 trajectory rows, the same states bench.py times):
    EVERY row against the oracle (score32 bit-exact, next ids, finals), plus
    the f64 definition within 1e-5 and normalization of every row."""
    m, o, f = lm6
    states, _ = trajectory_states(m, f, 1024, seed=2)
    with using(m, kernel=kernel):
        s, n, fin = gpu_advance(m, states)
    s32, s64, n_o, _ = o.rows(states)
    f32, _ = o.finals(states)
    assert np.array_equal(n, n_o) and same_bits(s, s32) and same_bits(fin, f32)
    assert np.max(np.abs(s - s64)) < 1e-5
    tot = np.exp(s.astype(np.float64)).sum(1) + np.exp(fin.astype(np.float64))
    assert np.max(np.abs(tot - 1)) < 1e-4
    # sharded == unsharded, bit for bit (rows are independent)
    with using(m, kernel=kernel):
        parts = [gpu_advance(m, states[i:i + 256]) for i in range(0, 1024, 256)]
    assert same_bits(np.concatenate([p[0] for p in parts]), s)
    assert np.array_equal(np.concatenate([p[1] for p in parts]), n)


@pytest.mark.parametrize("kernel", KERNELS)
def test_large_batch_b4096_every_row(lm6, kernel):
    """More rows than 8 per SM (the warp kernel's 8-slot windows), every row vs the oracle."""
    m, o, f = lm6
    states, _ = trajectory_states(m, f, 4096, seed=4)
    with using(m, kernel=kernel):
        s, n, fin = gpu_advance(m, states)
    s32, _, n_o, _ = o.rows(states, want64=False)
    f32, _ = o.finals(states)
    assert np.array_equal(n, n_o) and same_bits(s, s32) and same_bits(fin, f32)


@pytest.mark.parametrize("name", SMALL + ["fig1"])
def test_final_every_state(pairs, name):
    """ngpulm_final on its own: every state of each small LM,
    bit-exact vs the oracle's final32 (R9), B in one launch and in a ragged tail."""
    m, o, _ = pairs[name]
    states = np.arange(o.num_states, dtype=np.int32)
    f32, f64 = o.finals(states)
    got = m.final(torch.from_numpy(states).to(dev())).cpu().numpy()
    assert same_bits(got, f32)
    assert np.max(np.abs(got - f64)) < 1e-5
    perm = np.random.default_rng(1).permutation(states)[: max(1, o.num_states - 3)]
    got2 = m.final(torch.from_numpy(perm).to(dev())).cpu().numpy()
    assert same_bits(got2, f32[perm])
    assert m.check() == -1


def test_final_b1024_trajectory(lm6):
    """ngpulm_final at the bench batch (1024 trajectory states of the 6-gram) and
    across more than one 256-thread block, bit-exact vs the oracle."""
    m, o, f = lm6
    states, _ = trajectory_states(m, f, 1024, seed=2)
    states = np.concatenate([states, synth.uniform_states(m.num_states, 301, seed=9)])
    f32, _ = o.finals(states)
    got = m.final(torch.from_numpy(states).to(dev())).cpu().numpy()
    assert same_bits(got, f32)


def test_advance_host_and_replica_and_streams(lm6):
    m, o, f = lm6
    states, _ = trajectory_states(m, f, 200, seed=7)
    s, n, fin = gpu_advance(m, states)
    sh = torch.empty((200, m.V), dtype=torch.float32).pin_memory()
    nh = torch.empty((200, m.V), dtype=torch.int32).pin_memory()
    fh = torch.empty(200, dtype=torch.float32).pin_memory()
    m.advance_host(torch.from_numpy(states).pin_memory(), sh, nh, fh)
    assert same_bits(sh.numpy(), s) and np.array_equal(nh.numpy(), n) and same_bits(fh.numpy(), fin)
    r = m.replicate(0)
    s2, n2, _ = gpu_advance(r, states)
    assert same_bits(s2, s) and np.array_equal(n2, n)
    st = torch.from_numpy(states).to(dev())
    outs = []
    for _ in range(2):
        with torch.cuda.stream(torch.cuda.Stream()):
            outs.append(m.advance(st))
    torch.cuda.synchronize()
    for a, b, _ in outs:
        assert same_bits(a.cpu().numpy(), s) and np.array_equal(b.cpu().numpy(), n)


# ---------------------------------------------------------------- fused greedy step
def gpu_step(m, mode, logits_np, states, prev=None, active=None, lam=0.3, blank=None):
    x = torch.from_numpy(np.ascontiguousarray(logits_np, np.float32)).to(dev())
    st = torch.from_numpy(np.array(states, np.int32)).to(dev())
    pv = torch.from_numpy(np.array(prev, np.int32)).to(dev()) if prev is not None else None
    ac = torch.from_numpy(np.array(active, np.uint8)).to(dev()) if active is not None else None
    tok = m.fused_greedy_step(mode, x, st, prev=pv, active=ac, lam=lam, blank_id=blank)
    torch.cuda.synchronize()
    return tok.cpu().numpy(), st.cpu().numpy(), (pv.cpu().numpy() if pv is not None else None)


@pytest.mark.parametrize("kernel", KERNELS)
@pytest.mark.parametrize("chain", [ng.CHAIN_TABLE, ng.CHAIN_WALK])
@pytest.mark.parametrize("mode", [CTC, RNNT, AED])
@pytest.mark.parametrize("lam", [0.0, 0.3, 3.0])
@pytest.mark.parametrize("name", ["tiny3", "five48", "ten24"])
def test_fused_step_matches_oracle(pairs, mode, lam, name, chain, kernel):
    m, o, _ = pairs[name]
    m.set_chain_mode(chain)
    m.set_advance_kernel(kernel)
    rng = np.random.default_rng(17)
    B = 300
    x = synth.rnnt_logits(B, 1, o.V, seed=9)[0]
    x[::11, 2] = x[::11].max(axis=1)              # exact ties at the top
    states = rng.integers(0, o.num_states, size=B).astype(np.int32)
    prev = rng.integers(-1, o.V + 1, size=B).astype(np.int32)
    prev[prev == o.V] = -1
    active = (rng.random(B) > 0.1).astype(np.uint8)
    try:
        tg, sg, pg = gpu_step(m, mode, x, states, prev if mode == CTC else None, active, lam)
    finally:
        m.set_chain_mode(ng.CHAIN_TABLE)
        m.set_advance_kernel(ng.ADVANCE_AUTO)
    to, so, po = o.fused_step(mode, x, states, prev=prev if mode == CTC else None, active=active, lam=lam)
    assert np.array_equal(tg, to) and np.array_equal(sg, so)
    if mode == CTC:
        assert np.array_equal(pg, po)


@pytest.mark.parametrize("mode", [CTC, RNNT, AED])
def test_fused_step_blank_first_column(pairs, mode):
    """blank_id = 0 (special column first): tokens v sit in column v+1 (R19)."""
    m, o, _ = pairs["tri64"]
    B = 200
    x = synth.rnnt_logits(B, 1, o.V, seed=3, blank=0)[0]
    states = synth.uniform_states(o.num_states, B, seed=4)
    prev = np.full(B, -1, np.int32)
    tg, sg, pg = gpu_step(m, mode, x, states, prev if mode == CTC else None, None, 1.0, blank=0)
    to, so, po = o.fused_step(mode, x, states, prev=prev if mode == CTC else None, lam=1.0, blank_id=0)
    assert np.array_equal(tg, to) and np.array_equal(sg, so)


def test_ctc_decode_loop_config2_shape(lm6):
    """BASELINE configs[2] layout: logits [B, T, V+1] (row stride T*(V+1)), lambda=0.3,
    frame loop on the GPU vs the oracle on every utterance."""
    m, o, f = lm6
    B, T = 256, 64
    sents = synth.read_sentences(f.heldout)
    x = synth.ctc_logits(sents, B, T, m.V, seed=4)
    xd = torch.from_numpy(x).to(dev())
    st = torch.zeros(B, dtype=torch.int32, device=dev())
    pv = torch.full((B,), -1, dtype=torch.int32, device=dev())
    frames = torch.empty((T, B), dtype=torch.int32, device=dev())
    for t in range(T):
        m.fused_greedy_step(CTC, xd[:, t], st, prev=pv, lam=0.3, tokens_out=frames[t])
    torch.cuda.synchronize()
    rows = np.arange(B)
    so, po = np.zeros(rows.size, np.int32), np.full(rows.size, -1, np.int32)
    fo = []
    for t in range(T):
        tok, so, po = o.fused_step(CTC, x[rows, t], so, prev=po, lam=0.3)
        fo.append(tok)
    assert np.array_equal(frames.cpu().numpy()[:, rows], np.stack(fo))
    assert np.array_equal(st.cpu().numpy()[rows], so) and np.array_equal(pv.cpu().numpy()[rows], po)
    # the LM changed some decisions relative to plain greedy (the test means something)
    assert (np.stack(fo) != np.argmax(x[rows], axis=2).T).any()


def test_fused_invalid_state(pairs):
    m, o, _ = pairs["tri64"]
    x = synth.rnnt_logits(3, 1, o.V, seed=1)[0]
    tg, sg, pg = gpu_step(m, CTC, x, [1, o.num_states, 2], [-1, -1, -1], None, 0.5)
    assert tg[1] == -1 and sg[1] == o.num_states and m.check() == 1


def test_binary_model_same_results(lm6, tmp_path):
    """A model reloaded from its NGLM file answers bit-identically."""
    m, o, f = lm6
    p = str(tmp_path / "lm6.nglm")
    m.save(p)
    r = ng.load_binary(p, device=0)
    states, _ = trajectory_states(m, f, 1024, seed=61)
    a, b = gpu_advance(m, states), gpu_advance(r, states)
    assert same_bits(a[0], b[0]) and np.array_equal(a[1], b[1]) and same_bits(a[2], b[2])
    x = synth.rnnt_logits(256, 1, m.V, seed=62)[0]
    for mode in (CTC, RNNT, AED):
        g = [gpu_step(mm, mode, x, states[:256], np.full(256, -1, np.int32) if mode == CTC else None, None, 0.4)
             for mm in (m, r)]
        assert all(np.array_equal(g[0][i], g[1][i]) for i in range(2))


@pytest.mark.parametrize("B", [149, 600, 1036])
@pytest.mark.parametrize("name", ["uni16", "bi16", "tiny3", "tri64", "five48", "ten24"])
def test_mid_size_batches_full_rows(pairs, name, B):
    """Batches between one row per SM and 7 per SM (the 16-slot warp kernel with the
    CTA-shared root level) against the oracle: full rows of every batch row."""
    m, o, _ = pairs[name]
    assert m.info.num_states > 0
    states = synth.uniform_states(o.num_states, B, seed=B)
    s, n, f = gpu_advance(m, states)
    uniq, inv = np.unique(states, return_inverse=True)
    s32, _, n_o, _ = o.rows(uniq, want64=False)
    f32, _ = o.finals(uniq)
    assert np.array_equal(n, n_o[inv]) and same_bits(s, s32[inv]) and same_bits(f, f32[inv])


@pytest.fixture(scope="module")
def lm_bigv(lm_dir):
    """V = 40000 (beyond one shared-memory row): a word-level-sized vocabulary, 3-gram."""
    f = synth.make_lm(lm_dir, 40000, 3, tokens=300000, seed=9, heldout=300, tag="bigv_3gram")
    return ng.load_arpa(f.arpa, vocab_size=40000, device=0), Oracle(f.arpa, vocab_size=40000), f


@pytest.mark.parametrize("chain", [ng.CHAIN_TABLE, ng.CHAIN_WALK])
def test_vocab_tiled_advance(lm_bigv, chain):
    """rows larger than shared memory are answered tile by tile
    (one CTA per (row, vocabulary tile)); full rows bit-exact vs the oracle."""
    m, o, f = lm_bigv
    assert m.V > m.info.max_fused_vocab and m.info.max_vocab >= m.V
    states, _ = trajectory_states(m, f, 24, seed=71)
    states[:3] = [0, m.bos_state, o.num_states - 1]
    with using(m, chain):
        s, n, fin = gpu_advance(m, states)
    s32, s64, n_o, _ = o.rows(states)
    f32, _ = o.finals(states)
    assert np.array_equal(n, n_o) and same_bits(s, s32) and same_bits(fin, f32)
    # the fused step refuses a row that does not fit
    x = torch.zeros((2, m.V + 1), dtype=torch.float32, device=dev())
    with pytest.raises(ng.NgpulmError):
        m.fused_greedy_step(RNNT, x, torch.zeros(2, dtype=torch.int32, device=dev()))


def test_vocab_tiled_unaligned_v(lm_dir):
    """V % 4 != 0 beyond one row: the scalar (no-TMA) path, tiled."""
    f = synth.make_lm(lm_dir, 30001, 2, tokens=100000, seed=10, heldout=100, tag="bigv_odd")
    m, o = ng.load_arpa(f.arpa, vocab_size=30001, device=0), Oracle(f.arpa, vocab_size=30001)
    states = synth.uniform_states(o.num_states, 16, seed=72)
    s, n, fin = gpu_advance(m, states)
    s32, _, n_o, _ = o.rows(states, want64=False)
    assert np.array_equal(n, n_o) and same_bits(s, s32)


@pytest.mark.parametrize("B", [7, 100, 148, 600, 3000])
def test_tiny_lm_resident_kernel(pairs, B):
    """SURVEY.md §8(f) f4 tiny-LM path: a keyword-biasing-sized LM is answered from
    a copy in every CTA's shared memory (AUTO) — bit-identical to the global-memory
    warp kernel and to the oracle."""
    m, o, _ = pairs["tri64"]
    assert m.info.tiny_resident == 1
    states = synth.uniform_states(o.num_states, B, seed=B + 1)
    s, n, f = gpu_advance(m, states)
    with using(m, kernel=ng.ADVANCE_WARP):
        s2, n2, f2 = gpu_advance(m, states)
    assert same_bits(s, s2) and np.array_equal(n, n2) and same_bits(f, f2)
    uniq, inv = np.unique(states, return_inverse=True)
    s32, _, n_o, _ = o.rows(uniq, want64=False)
    assert np.array_equal(n, n_o[inv]) and same_bits(s, s32[inv])


@pytest.fixture(scope="module")
def pruned_pairs(pruned_lms):
    return {n: (ng.load_arpa(f.arpa, vocab_size=f.vocab_size, device=0), Oracle(f.arpa, vocab_size=f.vocab_size), f)
            for n, f in pruned_lms.items()}


@pytest.mark.parametrize("kernel", KERNELS)
@pytest.mark.parametrize("chain", [ng.CHAIN_TABLE, ng.CHAIN_WALK])
@pytest.mark.parametrize("name", ["pr3", "pr4", "pr6"])
def test_pruned_lms_exhaustive(pruned_pairs, name, chain, kernel):
    """Count-pruned LMs with missing suffix contexts (R7/R8, the paper's pruned SPGI
    LM): every state x every token bit-exact vs the oracle, and the fused steps."""
    m, o, f = pruned_pairs[name]
    states = np.arange(o.num_states, dtype=np.int32)
    with using(m, chain, kernel):
        s, n, fin = gpu_advance(m, states)
        x = synth.rnnt_logits(o.num_states, 1, o.V, seed=81)[0]
        steps = [gpu_step(m, mode, x, states, np.full(o.num_states, -1, np.int32) if mode == CTC else None, None, 1.3)
                 for mode in (CTC, RNNT, AED)]
    s32, _, n_o, _ = o.rows(states, want64=False)
    f32, _ = o.finals(states)
    assert np.array_equal(n, n_o) and same_bits(s, s32) and same_bits(fin, f32)
    for mode, (tg, sg, _) in zip((CTC, RNNT, AED), steps):
        to, so, _ = o.fused_step(mode, x, states, prev=np.full(o.num_states, -1) if mode == CTC else None, lam=1.3)
        assert np.array_equal(tg, to) and np.array_equal(sg, so), mode


@pytest.mark.parametrize("graph", [False, True])
def test_speculative_build_states_written_by_previous_kernel(lm6, graph):
    """The advance kernel builds each row from the state read before
    griddepcontrol.wait and re-reads it after the wait. Here the
    previous kernel (a fused RNN-T step, launched with PDL) rewrites the states in
    place right before every advance, so the early read can be stale: the rows
    must still be those of the new states."""
    m, o, f = lm6
    B, K = 512, 6
    st0, _ = trajectory_states(m, f, B, seed=91)
    xs = torch.from_numpy(synth.rnnt_logits(B, K, m.V, seed=92)).to(dev())
    st = torch.from_numpy(st0.copy()).to(dev())
    sc = torch.empty((K, B, m.V), dtype=torch.float32, device=dev())
    nx = torch.empty((K, B, m.V), dtype=torch.int32, device=dev())
    snap = torch.empty((K, B), dtype=torch.int32, device=dev())
    s = torch.cuda.Stream()

    def seq():
        for k in range(K):
            m.fused_greedy_step(RNNT, xs[k], st, lam=0.3, stream=s)
            m.advance(st, sc[k], nx[k], want_final=False, stream=s)
            snap[k].copy_(st)
    with torch.cuda.stream(s):
        if graph:
            g = torch.cuda.CUDAGraph()
            seq()  # warm-up, then replay from the same start
            s.synchronize()
            st.copy_(torch.from_numpy(st0))
            with torch.cuda.graph(g, stream=s):
                seq()
            st.copy_(torch.from_numpy(st0))
            g.replay()
        else:
            seq()
    s.synchronize()
    snap_np, sc_np, nx_np = snap.cpu().numpy(), sc.cpu().numpy(), nx.cpu().numpy()
    assert (snap_np[0] != st0).any()  # the steps did change states
    for k in range(K):
        rows = np.arange(k, B, 37)
        s32, _, n_o, _ = o.rows(snap_np[k, rows], want64=False)
        assert np.array_equal(nx_np[k, rows], n_o) and same_bits(sc_np[k, rows], s32), k


def test_advance_rejects_outputs_overlapping_states(pairs):
    m, o, _ = pairs["tri64"]
    buf = torch.zeros(8 * m.V + 8, dtype=torch.int32, device=dev())
    st = buf[:8]
    sc = torch.empty((8, m.V), dtype=torch.float32, device=dev())
    with pytest.raises(ng.NgpulmError):
        m.advance(st, sc, buf[4:4 + 8 * m.V].view(8, m.V))


from hypothesis import HealthCheck, given, settings  # noqa: E402
from hypothesis import strategies as hst  # noqa: E402


@settings(max_examples=10, deadline=None, suppress_health_check=[HealthCheck.function_scoped_fixture])
@given(V=hst.sampled_from([8, 20, 32, 64]), order=hst.integers(1, 6), tokens=hst.integers(60, 2000),
       seed=hst.integers(1, 10_000), prune=hst.lists(hst.integers(0, 3), min_size=6, max_size=6),
       lam=hst.sampled_from([0.0, 0.4, 2.5]))
def test_random_lms_exhaustive(tmp_path_factory, V, order, tokens, seed, prune, lam):
    """Random small LMs (order, vocabulary, corpus, count pruning): every state x
    token of advance, and the three fused steps, bit-exact vs the oracle."""
    d = str(tmp_path_factory.mktemp("rndg"))
    pr = ",".join(["0"] + [str(x) for x in prune[: order - 1]]) if order >= 2 else None
    f = synth.make_lm(d, V, order, tokens=tokens, seed=seed, lexicon=max(20, V * 3), heldout=5, tag="r", prune=pr)
    m, o = ng.load_arpa(f.arpa, vocab_size=V, device=0), Oracle(f.arpa, vocab_size=V)
    states = np.arange(o.num_states, dtype=np.int32)
    s, n, fin = gpu_advance(m, states)
    s32, _, n_o, _ = o.rows(states, want64=False)
    f32, _ = o.finals(states)
    assert np.array_equal(n, n_o) and same_bits(s, s32) and same_bits(fin, f32)
    x = synth.rnnt_logits(o.num_states, 1, V, seed=seed)[0]
    for mode in (CTC, RNNT, AED):
        pv = np.full(o.num_states, -1, np.int32) if mode == CTC else None
        tg, sg, _ = gpu_step(m, mode, x, states, pv, None, lam)
        to, so, _ = o.fused_step(mode, x, states, prev=pv, lam=lam)
        assert np.array_equal(tg, to) and np.array_equal(sg, so), mode


@pytest.mark.parametrize("kernel", [ng.ADVANCE_AUTO, ng.ADVANCE_WARP])
@pytest.mark.parametrize("B", [1024, 4096, 100])
def test_advance_independent_calls(lm6, B, kernel):
    """NGPULM_ADVANCE_INDEPENDENT (rows built and stored before the PDL wait, the wait
    at the end): K back-to-back calls over independent batches into distinct buffers,
    captured in one CUDA graph and replayed — every row of every call bit-exact vs the
    oracle; a consumer kernel right after the last call sees all calls complete
    (stream completion order kept)."""
    m, o, f = lm6
    K = 6
    st_np = np.stack([trajectory_states(m, f, B, seed=40 + k)[0] for k in range(K)])
    st = torch.from_numpy(st_np).to(dev())
    sc = torch.empty((K, B, m.V), dtype=torch.float32, device=dev())
    nx = torch.empty((K, B, m.V), dtype=torch.int32, device=dev())
    fi = torch.empty((K, B), dtype=torch.float32, device=dev())
    stream = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with using(m, kernel=kernel), torch.cuda.stream(stream):
        for k in range(K):  # warm-up
            m.advance(st[k], sc[k], nx[k], fi[k], stream=stream, independent=True)
        stream.synchronize()
        sc.zero_(); nx.fill_(-7)
        with torch.cuda.graph(g, stream=stream):
            for k in range(K):
                m.advance(st[k], sc[k], nx[k], fi[k], stream=stream, independent=True)
            total = nx.sum(dtype=torch.int64)  # a consumer of every call's outputs
        g.replay()
        stream.synchronize()
    tot_host = 0
    for k in range(K):
        uniq, inv = np.unique(st_np[k], return_inverse=True)
        s32, _, n_o, _ = o.rows(uniq, want64=False)
        f32, _ = o.finals(uniq)
        assert same_bits(sc[k].cpu().numpy(), s32[inv]) and np.array_equal(nx[k].cpu().numpy(), n_o[inv])
        assert same_bits(fi[k].cpu().numpy(), f32[inv])
        tot_host += int(n_o[inv].astype(np.int64).sum())
    assert int(total.item()) == tot_host
