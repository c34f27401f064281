"""Oracle pins for the fused greedy decisions (§2.3), CPU only.

Special cases that reduce to library routines (lambda = 0 -> numpy argmax /
plain greedy CTC collapse), invariants (blank retention, repeat rule) and
hand-computed constructed cases on the Fig. 1 LM whose LM values are exact
fractions (tests/golden/fig1_rows.txt).
"""
import itertools
import math

import numpy as np
import pytest

import synth
from oracle import AED, CTC, RNNT, Oracle


@pytest.fixture(scope="module")
def tri(small_lms):
    f = small_lms["tri64"]
    return Oracle(f.arpa, vocab_size=f.vocab_size), f


@pytest.fixture(scope="module")
def fig1(fig1_paths):
    return Oracle(*fig1_paths)


def test_lambda0_is_plain_argmax(tri):
    o, f = tri
    sents = synth.read_sentences(f.heldout)
    x = synth.rnnt_logits(B=64, steps=4, V=o.V, seed=4).reshape(-1, o.V + 1)
    # force several exact ties at the max
    x[::7, 3] = x[::7].max(axis=1)
    states = synth.uniform_states(o.num_states, x.shape[0], seed=3)
    for mode in (RNNT, AED):
        tok, st, _ = o.fused_step(mode, x, states, lam=0.0)
        assert (tok == np.argmax(x, axis=1)).all()          # numpy: first max wins
    tok, st, pv = o.fused_step(CTC, x, states, prev=np.full(x.shape[0], -1), lam=0.0)
    assert (tok == np.argmax(x, axis=1)).all()


def ctc_decode(o, logits, lam, start):
    """Frame loop over the oracle's fused step; returns emitted tokens per row."""
    B, T, _ = logits.shape
    st = np.full(B, start, dtype=np.int32)
    pv = np.full(B, -1, dtype=np.int32)
    out = [[] for _ in range(B)]
    adv = np.zeros(B, dtype=np.int64)
    frames = []
    for t in range(T):
        old_pv, old_st = pv.copy(), st.copy()
        tok, st, pv = o.fused_step(CTC, logits[:, t], st, prev=pv, lam=lam)
        frames.append(tok)
        for b in range(B):
            if tok[b] != o.V and tok[b] != old_pv[b]:
                out[b].append(int(tok[b]))
            adv[b] += int(st[b] != old_st[b] or (tok[b] != o.V and tok[b] != old_pv[b]))
    return out, np.stack(frames, 1), adv


def test_ctc_lambda0_is_greedy_collapse(tri):
    o, f = tri
    sents = synth.read_sentences(f.heldout)
    x = synth.ctc_logits(sents, B=6, T=40, V=o.V, seed=4)
    out, frames, adv = ctc_decode(o, x, 0.0, 0)
    for b in range(6):
        path = np.argmax(x[b], axis=1)
        collapsed = [int(k) for k, _ in itertools.groupby(path) if k != o.V]
        assert out[b] == collapsed
        assert adv[b] == len(collapsed)       # one LM advance per emission


def test_ctc_fused_changes_decisions_and_counts_advances(tri):
    o, f = tri
    sents = synth.read_sentences(f.heldout)
    x = synth.ctc_logits(sents, B=6, T=40, V=o.V, seed=5)
    out0, fr0, _ = ctc_decode(o, x, 0.0, 0)
    out1, fr1, adv = ctc_decode(o, x, 3.0, 0)
    assert (fr0 != fr1).any()                 # the LM matters at this weight
    for b in range(6):
        assert adv[b] == len(out1[b])


def test_rnnt_blank_retention(tri):
    o, f = tri
    x = synth.rnnt_logits(B=128, steps=2, V=o.V, seed=7).reshape(-1, o.V + 1)
    states = synth.uniform_states(o.num_states, x.shape[0], seed=3)
    raw = np.argmax(x, axis=1)
    for lam in (0.0, 1.0, 10.0):
        tok, st, _ = o.fused_step(RNNT, x, states, lam=lam)
        blank = raw == o.V
        assert (tok[blank] == o.V).all() and (st[blank] == states[blank]).all()
        assert (tok[~blank] != o.V).all()


def test_constructed_fig1_cases(fig1):
    """State 11 ("on the"): lm(sat) = ln 1/32, lm(mat) = ln 21/32, final = ln 1/32.
    asr: sat = -1.0, mat = -1.5, eos/blank column 6 = -1.2, others -10.
    lambda = 1: sat -> -1 + ln(1/32) = -4.466, mat -> -1.5 + ln(21/32) = -1.921."""
    o = fig1
    row = np.full((1, 7), -10.0, dtype=np.float32)
    row[0, 2], row[0, 4], row[0, 6] = -1.0, -1.5, -1.2
    s = np.array([11], dtype=np.int32)
    # RNN-T: stage 1 raw argmax = sat (non-blank) -> stage 2 picks mat -> "the mat" = 8
    tok, st, _ = o.fused_step(RNNT, row, s, lam=1.0)
    assert tok[0] == 4 and st[0] == 8
    # lambda = 0: stays with the raw argmax
    tok, st, _ = o.fused_step(RNNT, row, s, lam=0.0)
    assert tok[0] == 2 and st[0] == 3            # "on the" + sat -> "sat" (3)
    # CTC: the blank column is never rescored: raw -1.2 beats fused mat (-1.921)
    tok, st, pv = o.fused_step(CTC, row, s, prev=np.array([-1]), lam=1.0)
    assert tok[0] == 6 and st[0] == 11 and pv[0] == -1
    # CTC with blank at -3.0, prev = none: mat wins as for the transducer
    rowc = row.copy(); rowc[0, 6] = -3.0
    tok, st, pv = o.fused_step(CTC, rowc, s, prev=np.array([-1]), lam=1.0)
    assert tok[0] == 4 and st[0] == 8 and pv[0] == 4
    # CTC, prev = sat: the repeated token keeps its raw -1.0 and beats mat's -1.921:
    # selected but collapsed -> no LM advance, prev stays sat
    tok, st, pv = o.fused_step(CTC, rowc, s, prev=np.array([2]), lam=1.0)
    assert tok[0] == 2 and st[0] == 11 and pv[0] == 2
    # CTC: blank column raw -1.2 vs fused mat -1.921 -> blank when it is the best raw
    row2 = row.copy(); row2[0, 6] = -0.5
    tok, st, pv = o.fused_step(CTC, row2, s, prev=np.array([4]), lam=1.0)
    assert tok[0] == 6 and st[0] == 11 and pv[0] == -1
    # AED: eos column = -1.2 + ln(1/32) = -4.666 loses to mat; with asr[eos] = 2.0
    # eos = 2 - 3.466 = -1.466 beats mat (-1.921): stop, state unchanged
    tok, st, _ = o.fused_step(AED, row, s, lam=1.0)
    assert tok[0] == 4 and st[0] == 8
    row3 = row.copy(); row3[0, 6] = 2.0
    tok, st, _ = o.fused_step(AED, row3, s, lam=1.0)
    assert tok[0] == 6 and st[0] == 11
    assert math.isclose(2.0 + math.log(1 / 32), -1.4657359, abs_tol=1e-6)


def test_inactive_rows_untouched(fig1):
    row = np.zeros((2, 7), dtype=np.float32)
    row[:, 1] = 1.0
    tok, st, pv = fig1.fused_step(CTC, row, np.array([11, 11]), prev=np.array([-1, -1]),
                                  active=np.array([0, 1]), lam=0.0)
    assert tok[0] == -1 and st[0] == 11 and pv[0] == -1
    assert tok[1] == 1 and st[1] == 7


def test_fusion_weight_tie_break_lowest_column(fig1):
    # two columns with identical fused values: lowest column wins (torch.argmax rule)
    row = np.full((1, 7), -10.0, dtype=np.float32)
    # state 0: lm(cat) = lm(sat) = ln 1/8; equal asr -> equal fused values
    row[0, 1] = row[0, 2] = -0.25
    for mode in (RNNT, AED, CTC):
        tok, st, _ = fig1.fused_step(mode, row, np.array([0]), prev=np.array([-1]), lam=0.7)
        assert tok[0] == 1 and st[0] == 2


def test_oracle_ctc_decode_lambda0_is_greedy_collapse_ragged(tri):
    """Whole-utterance oracle decode at lambda = 0 with ragged lengths = numpy's
    per-frame argmax collapsed (itertools.groupby, blanks dropped) on each row's prefix."""
    o, f = tri
    sents = synth.read_sentences(f.heldout)
    B, T = 7, 37
    x = synth.ctc_logits(sents, B=B, T=T, V=o.V, seed=8)
    lengths = np.array([0, 1, 5, 37, 20, 36, 2], np.int32)
    frames, emitted, elen, st, pv = o.ctc_decode(x, np.zeros(B, np.int32), lam=0.0, lengths=lengths)
    for b in range(B):
        path = np.argmax(x[b, : lengths[b]], axis=1)
        collapsed = [int(k) for k, _ in itertools.groupby(path) if k != o.V]
        assert list(emitted[b, : elen[b]]) == collapsed
        assert (frames[b, : lengths[b]] == path).all() and (frames[b, lengths[b]:] == -1).all()
        assert pv[b] == (-1 if lengths[b] == 0 or path[-1] == o.V else path[-1])


def test_oracle_ctc_decode_is_the_frame_loop(tri):
    """The whole-utterance decode equals T single fused steps with active = t < len."""
    o, f = tri
    sents = synth.read_sentences(f.heldout)
    B, T = 6, 30
    x = synth.ctc_logits(sents, B=B, T=T, V=o.V, seed=9)
    lengths = np.array([30, 0, 7, 29, 15, 30], np.int32)
    start = synth.uniform_states(o.num_states, B, seed=5)
    prev0 = np.array([-1, 3, -1, 5, -1, -1], np.int32)
    frames, emitted, elen, st, pv = o.ctc_decode(x, start, prev=prev0, lam=2.0, lengths=lengths)
    s, p = start.copy(), prev0.copy()
    for t in range(T):
        act = (t < lengths).astype(np.uint8)
        p_old = p.copy()
        tok, s, p = o.fused_step(CTC, x[:, t], s, prev=p, active=act, lam=2.0)
        assert (frames[:, t] == tok).all()
    assert (st == s).all() and (pv == p).all()
    # emissions: selections that are neither blank nor the previous selection
    for b in range(B):
        sel = list(frames[b, : lengths[b]])
        em, last = [], prev0[b]
        for c in sel:
            if c != o.V and c != last:
                em.append(c)
            last = -1 if c == o.V else c
        assert list(emitted[b, : elen[b]]) == em


# ---------------------------------------------------------------- ILM subtraction (R21) and top-k (f3)
def _margin_ok(vals, tol=1e-3):
    """rows whose best value beats the runner-up by more than tol (decision not rounding-sensitive)"""
    s = np.sort(vals, axis=1)
    return (s[:, -1] - s[:, -2]) > tol


@pytest.mark.parametrize("mode", [CTC, RNNT, AED])
def test_ilm_zero_weight_is_plain_fusion(tri, mode):
    o, f = tri
    B = 64
    x = synth.rnnt_logits(B, 1, o.V, seed=31)[0]
    st = synth.uniform_states(o.num_states, B, seed=32)
    ilm = np.random.default_rng(33).normal(-5, 2, size=(B, o.V)).astype(np.float32)
    pv = np.full(B, -1, np.int32) if mode == CTC else None
    a = o.fused_step(mode, x, st, prev=pv, lam=0.8)
    b = o.fused_step_ilm(mode, x, st, ilm, 0.0, prev=pv, lam=0.8)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


def test_ilm_term_against_float64_definition(tri):
    """AED decisions = argmax of asr + lam*lm - lam_ilm*ilm computed in float64 from
    the textbook score64 rows and final64, wherever the margin is clear."""
    o, f = tri
    B = 400
    x = synth.rnnt_logits(B, 1, o.V, seed=34)[0]
    st = synth.uniform_states(o.num_states, B, seed=35)
    ilm = np.random.default_rng(36).normal(-4, 2, size=(B, o.V)).astype(np.float32)
    lam, lam_ilm = 1.5, 0.7
    _, s64, _, _ = o.rows(st)
    _, f64 = o.finals(st)
    ref = np.empty((B, o.V + 1))
    ref[:, : o.V] = x[:, : o.V].astype(np.float64) + lam * s64 - lam_ilm * ilm.astype(np.float64)
    ref[:, o.V] = x[:, o.V] + lam * f64
    tok, _, _ = o.fused_step_ilm(AED, x, st, ilm, lam_ilm, lam=lam)
    ok = _margin_ok(ref)
    assert ok.sum() > 0.9 * B
    assert np.array_equal(tok[ok], np.argmax(ref, axis=1)[ok])
    # the ILM term changes decisions at this weight (the pin means something)
    tok0, _, _ = o.fused_step(AED, x, st, lam=lam)
    assert (tok0 != tok).any()


def test_ilm_cancels_lm(tri):
    """ilm = the LM row and lam_ilm = lam: the terms cancel, so the
    decisions are the raw argmax wherever the margin is clear."""
    o, f = tri
    B = 300
    x = synth.rnnt_logits(B, 1, o.V, seed=37)[0]
    st = synth.uniform_states(o.num_states, B, seed=38)
    s32, _, _, _ = o.rows(st, want64=False)
    tok, _, _ = o.fused_step_ilm(RNNT, x, st, s32, 2.0, lam=2.0)
    raw = x.astype(np.float64)
    ok = _margin_ok(raw[:, : o.V], 1e-4) & (np.argmax(raw, axis=1) != o.V)
    assert np.array_equal(tok[ok], np.argmax(raw[:, : o.V], axis=1)[ok])


def test_topk_special_cases(tri):
    o, f = tri
    B, k = 50, 9
    x = synth.rnnt_logits(B, 1, o.V, seed=39)[0]
    x[::5, 7] = x[::5, 3]                    # exact ties: the lower column first
    st = synth.uniform_states(o.num_states, B, seed=40)
    # lambda = 0: numpy's stable descending sort of the logits
    sc, cols, nx = o.topk(x, st, k, lam=0.0)
    order = np.argsort(-x, axis=1, kind="stable")[:, :k]
    assert np.array_equal(cols, order)
    assert np.array_equal(sc, np.take_along_axis(x, order, 1))
    # candidates' next states: the LM row's next ids (eos keeps the state)
    _, _, n_o, _ = o.rows(st, want64=False)
    for b in range(B):
        for c, s in zip(cols[b], nx[b]):
            assert s == (st[b] if c == o.V else n_o[b, c])
    # k = 1 is the AED fused greedy decision
    sc1, cols1, _ = o.topk(x, st, 1, lam=1.3)
    tok, _, _ = o.fused_step(AED, x, st, lam=1.3)
    assert np.array_equal(cols1[:, 0], tok)
    # values: the float64 definition within the f32 bound; descending order
    sc, cols, _ = o.topk(x, st, k, lam=1.3)
    _, s64, _, _ = o.rows(st)
    _, f64 = o.finals(st)
    full = np.concatenate([s64, f64[:, None]], 1)
    ref = np.take_along_axis(x.astype(np.float64), cols, 1) + 1.3 * np.take_along_axis(full, cols, 1)
    assert np.max(np.abs(sc - ref)) < 1e-4
    assert (np.diff(sc, axis=1) <= 0).all()
    # more candidates than columns: the tail is empty
    sc, cols, nx = o.topk(x[:2], st[:2], o.V + 4, lam=0.5)
    assert (cols[:, o.V + 1:] == -1).all() and np.isneginf(sc[:, o.V + 1:]).all()


# ---------------------------------------------------------------- greedy transducer loop (f2)
def _plain_transducer(seed, T, V, max_sym, temp=8.0, bias=0.0):
    """Plain greedy transducer over the synthetic joint (numpy twin), no LM:
    frame loop, <= max_sym labels per frame, raw argmax (first max) per row."""
    out, u, last = [], 0, -1
    for t in range(T):
        for _ in range(max_sym):
            row = synth.synthetic_joint_raw(seed, t, u, last, V + 1, temp, V, bias)
            c = int(np.argmax(row))
            if c == V:
                break
            out.append(c)
            u += 1
            last = c
    return out


def test_transducer_decode_lambda0_is_plain_greedy(tri):
    """lambda = 0 -> the plain greedy transducer loop (here a numpy
    simulator over the CPU twin of the synthetic joint)."""
    o, f = tri
    lengths = np.array([0, 1, 5, 12, 7], np.int32)
    for max_sym, bias in ((1, 0.0), (3, 0.5), (10, 0.75)):
        em, el, st = o.transducer_decode(1234, lengths, np.zeros(5, np.int32), lam=0.0, max_symbols=max_sym,
                                         temperature=2.0, blank_bias=bias)
        for b, T in enumerate(lengths):
            ref = _plain_transducer(1234, int(T), o.V, max_sym, temp=2.0, bias=bias)
            assert list(em[b, : el[b]]) == ref
            # LM state = the emitted tokens replayed from the root (SPEC.md: LM-state consistency)
            assert st[b] == o.state_of(False, [int(x) for x in ref])


def test_transducer_decode_fused_float64_simulator(tri):
    """lambda = 2: the decoded labels follow a float64 two-stage simulator (score64
    rows, SPEC.md:325 'brute-force two-stage simulator run in 64-bit') for as long
    as every stage-2 decision has a clear margin."""
    o, f = tri
    seed, T, lam, max_sym, temp = 77, 20, 2.0, 4, 2.0
    em, el, st = o.transducer_decode(seed, np.array([T], np.int32), np.zeros(1, np.int32), lam=lam,
                                     max_symbols=max_sym, temperature=temp, blank_bias=0.25)
    got = list(em[0, : el[0]])
    ref, u, last, s, checked = [], 0, -1, 0, 0
    for t in range(T):
        for _ in range(max_sym):
            row = synth.synthetic_joint_raw(seed, t, u, last, o.V + 1, temp, o.V, 0.25).astype(np.float64)
            if int(np.argmax(row)) == o.V:
                break
            _, s64, nx, _ = o.rows(np.array([s], np.int32))
            fused = row[: o.V] + lam * s64[0]
            srt = np.sort(fused)
            if srt[-1] - srt[-2] < 1e-3:
                break
            c = int(np.argmax(fused))
            ref.append(c)
            checked += 1
            s, u, last = int(nx[0, c]), u + 1, c
        else:
            continue
        if checked and (srt[-1] - srt[-2] < 1e-3):
            break
    assert checked > 5 and got[: len(ref)] == ref
    # the LM matters at this weight
    assert got != _plain_transducer(seed, T, o.V, max_sym, temp, 0.25)


# ---------------------------------------------------------------- greedy TDT loop (f2, R25)
TDT_DURATIONS = np.array([0, 1, 2, 3, 4], np.int32)


def _plain_tdt(seed, T, V, durations, max_sym, temp=8.0, bias=0.0):
    """Plain greedy TDT over the synthetic joint (numpy twin), no LM, written from
    the TDT decoding rule (Xu et al. 2023): token = first argmax of
    the V+1 token columns, duration = durations[first argmax of the D duration
    columns]; blank advances max(d, 1) frames, a label d frames (d = 0: same
    frame, at most max_sym labels there)."""
    out, t, u, last, sym, steps = [], 0, 0, -1, 0, 0
    D = len(durations)
    while t < T:
        row = synth.synthetic_joint_raw(seed, t, u, last, V + 1 + D, temp, V, bias)
        c = int(np.argmax(row[: V + 1]))
        d = int(durations[int(np.argmax(row[V + 1:]))])
        steps += 1
        if c == V:
            t += max(d, 1)
            sym = 0
            continue
        out.append(c)
        u, last = u + 1, c
        if d > 0:
            t, sym = t + d, 0
        else:
            sym += 1
            if sym >= max_sym:
                t, sym = t + 1, 0
    return out, steps


def test_tdt_decode_lambda0_is_plain_greedy_tdt(tri):
    o, f = tri
    lengths = np.array([0, 1, 5, 17, 9], np.int32)
    for max_sym, bias in ((1, 0.0), (3, 0.5), (10, 0.75)):
        em, el, st, steps = o.tdt_decode(4321, lengths, np.zeros(5, np.int32), TDT_DURATIONS, lam=0.0,
                                         max_symbols=max_sym, temperature=2.0, blank_bias=bias)
        for b, T in enumerate(lengths):
            ref, nsteps = _plain_tdt(4321, int(T), o.V, TDT_DURATIONS, max_sym, temp=2.0, bias=bias)
            assert list(em[b, : el[b]]) == ref and steps[b] == nsteps
            assert st[b] == o.state_of(False, [int(x) for x in ref])
    # durations > 1 really skip frames: fewer joint evaluations than frames + labels
    _, el, _, steps = o.tdt_decode(4321, np.array([40], np.int32), np.zeros(1, np.int32), TDT_DURATIONS, lam=0.0,
                                   max_symbols=3, temperature=2.0, blank_bias=0.5)
    assert steps[0] < 40 + el[0]


@pytest.mark.parametrize("lam", [0.0, 0.5, 2.0])
def test_tdt_reduces_to_rnnt(tri, lam):
    """Special cases that reduce to the (separately pinned) RNN-T loop, at any LM
    weight: the token columns of the joint do not depend on the number of
    duration columns, so durations = {1} is the RNN-T loop with max_symbols = 1,
    and durations = {0} is the RNN-T loop with max_symbols labels per frame."""
    o, f = tri
    lengths = np.array([3, 11, 0, 8], np.int32)
    z = np.zeros(4, np.int32)
    for durs, max_sym in (([1], 1), ([0], 4), ([0], 1)):
        em, el, st, _ = o.tdt_decode(99, lengths, z, np.array(durs, np.int32), lam=lam, max_symbols=max_sym,
                                     temperature=4.0, blank_bias=0.5)
        er, elr, sr = o.transducer_decode(99, lengths, z, lam=lam, max_symbols=max_sym, temperature=4.0,
                                          blank_bias=0.5, max_len=em.shape[1])
        assert np.array_equal(el, elr) and np.array_equal(st, sr)
        for b in range(4):
            assert list(em[b, : el[b]]) == list(er[b, : elr[b]])


def test_tdt_decode_fused_float64_simulator(tri):
    """lambda = 2 with durations {0..4}: the labels follow a float64 simulator
    (score64 rows, two-stage token rule, raw duration argmax) while every stage-2
    decision has a clear margin; the LM changes the result."""
    o, f = tri
    seed, T, lam, max_sym, temp, bias = 55, 30, 2.0, 3, 2.0, 0.25
    D = len(TDT_DURATIONS)
    em, el, st, _ = o.tdt_decode(seed, np.array([T], np.int32), np.zeros(1, np.int32), TDT_DURATIONS, lam=lam,
                                 max_symbols=max_sym, temperature=temp, blank_bias=bias)
    got = list(em[0, : el[0]])
    ref, t, u, last, s, sym, checked = [], 0, 0, -1, 0, 0, 0
    while t < T:
        row = synth.synthetic_joint_raw(seed, t, u, last, o.V + 1 + D, temp, o.V, bias).astype(np.float64)
        d = int(TDT_DURATIONS[int(np.argmax(row[o.V + 1:]))])
        if int(np.argmax(row[: o.V + 1])) == o.V:
            t, sym = t + max(d, 1), 0
            continue
        _, s64, nx, _ = o.rows(np.array([s], np.int32))
        fused = row[: o.V] + lam * s64[0]
        srt = np.sort(fused)
        if srt[-1] - srt[-2] < 1e-3:
            break
        c = int(np.argmax(fused))
        ref.append(c)
        checked += 1
        s, u, last = int(nx[0, c]), u + 1, c
        if d > 0:
            t, sym = t + d, 0
        else:
            sym += 1
            if sym >= max_sym:
                t, sym = t + 1, 0
    assert checked > 5 and got[: len(ref)] == ref
    assert got != _plain_tdt(seed, T, o.V, TDT_DURATIONS, max_sym, temp, bias)[0]
