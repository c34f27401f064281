"""Oracle pin: the paper's Fig. 1 worked example (§2.1) with exact
hand-derived values (tests/golden/fig1_rows.txt). CPU only."""
import math
import os
from fractions import Fraction

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import Oracle

WORDS = ["the", "cat", "sat", "on", "mat", "dog"]


def read_golden():
    rows = []
    with open(os.path.join(GOLDEN, "fig1_rows.txt")) as f:
        for line in f:
            if not line.strip() or line.startswith("#"):
                continue
            sid, ctx, cells, fin = [x.strip() for x in line.split("|")]
            ctx = [] if ctx == "-" else ctx.split()
            p, nx = [], []
            for cell in cells.split():
                a, b = cell.split(":")
                p.append(Fraction(a)); nx.append(int(b))
            rows.append((int(sid), ctx, p, nx, Fraction(fin)))
    return rows


@pytest.fixture(scope="module")
def fig1(fig1_paths):
    arpa, vocab = fig1_paths
    return Oracle(arpa, vocab)


def ctx_words(o, s):
    return ["<s>" if t == o.V else WORDS[t] for t in o.context(s)]


def test_structure_13_states(fig1):
    # 6 unigram contexts (5 words + <s>) + 6 bigram contexts + root
    assert fig1.V == 6 and fig1.order == 3
    assert fig1.num_states == 13
    assert fig1.num_unk_filled == 1           # "dog" has no unigram
    assert ctx_words(fig1, fig1.bos_state) == ["<s>"]
    for sid, ctx, *_ in read_golden():
        assert ctx_words(fig1, sid) == ctx


def test_rows_exact(fig1):
    g = read_golden()
    states = np.array([r[0] for r in g], dtype=np.int32)
    s32, s64, nx, lv = fig1.rows(states)
    for i, (sid, ctx, p, nxt, fin) in enumerate(g):
        exp = np.array([math.log(float(x)) for x in p])
        np.testing.assert_allclose(s64[i], exp, rtol=0, atol=1e-12)
        # Algorithm-1-order float32 value: within the f32 rounding of <= N+1 steps
        assert np.all(np.abs(s32[i].astype(np.float64) - exp) <= 4 * np.spacing(np.float32(3.5)))
        assert nx[i].tolist() == nxt, (sid, ctx)
        # Algorithm 1 iterations never exceed the order
        assert 1 <= lv[i] <= 3
        assert sum(p) + fin == 1                # the golden rows themselves are normalized


def test_finals_exact(fig1):
    g = read_golden()
    states = np.array([r[0] for r in g], dtype=np.int32)
    f32, f64 = fig1.finals(states)
    for i, r in enumerate(g):
        assert abs(f64[i] - math.log(float(r[4]))) < 1e-12
        assert abs(float(f32[i]) - math.log(float(r[4]))) < 1e-6
    # explicit finals (Fig. 1 double circles) are exactly the </s> n-gram weights
    assert abs(f64[0] - math.log(1 / 8)) < 1e-12        # root: </s> unigram
    assert abs(f64[5] - math.log(9 / 16)) < 1e-12       # "mat </s>"
    assert abs(f64[8] - math.log(25 / 32)) < 1e-12      # "the mat </s>"


def test_root_single_iteration_and_third_order_targets(fig1):
    _, _, nx, lv = fig1.rows(np.array([0, 7, 9, 10, 11, 12], dtype=np.int32))
    assert lv[0] == 1                                    # root row: one iteration
    # 3-gram arcs point to 2-gram states: the cat +sat -> cat sat
    assert nx[1][2] == 9 and nx[2][3] == 10 and nx[3][0] == 11 and nx[4][4] == 8


def test_state_of_histories(fig1):
    ids = {w: i for i, w in enumerate(WORDS)}
    hist = [ids[w] for w in "the cat sat on the".split()]
    assert fig1.state_of(True, hist) == 11               # "on the"
    assert fig1.state_of(True, []) == fig1.bos_state
    assert fig1.state_of(False, [ids["dog"]]) == 0       # unk-filled -> root
    assert fig1.state_of(True, [ids["the"]]) == 12       # "<s> the"


def test_sentence_score(fig1):
    """score_sentence: "the cat sat on the mat" = product of the
    Witten-Bell fractions along the sentence, then the final weight."""
    ids = {w: i for i, w in enumerate(WORDS)}
    s, total = fig1.bos_state, 0.0
    for w in "the cat sat on the mat".split():
        s32, s64, nx, _ = fig1.rows(np.array([s], dtype=np.int32))
        total += s64[0][ids[w]]
        s = int(nx[0][ids[w]])
    total += fig1.finals(np.array([s], dtype=np.int32))[1][0]
    exp = Fraction(5, 8) * Fraction(21, 32) * Fraction(25, 32) * Fraction(25, 32) \
        * Fraction(13, 16) * Fraction(21, 32) * Fraction(25, 32)
    assert abs(total - math.log(float(exp))) < 1e-12
