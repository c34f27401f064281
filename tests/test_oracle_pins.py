"""Oracle pins against things other than the oracle itself (CPU only):

* the Witten-Bell interpolation recomputed from raw corpus counts (wb_counts.py)
  equals the oracle's back-off value score64 for every state and
  token, and its final weight;
* per-state normalization  sum_v exp(score) + exp(final) = 1;
* sentence replay through next states reproduces the interpolated probability
  of the full N-1-token history at every step (pins next);
* Algorithm-1-order float32 value within the f32 error bound of the f64 value;
* depth bound, root row = unigram row, N = 1.
"""
import math

import numpy as np
import pytest

import synth
from oracle import Oracle
from wb_counts import BOS, EOS, WittenBell

NAMES = ["uni16", "bi16", "tiny3", "tri64", "five48", "ten24"]


@pytest.fixture(scope="module")
def models(small_lms):
    out = {}
    for name in NAMES:
        f = small_lms[name]
        o = Oracle(f.arpa, vocab_size=f.vocab_size)
        wb = WittenBell(synth.read_sentences(f.corpus), f.order, f.vocab_size)
        out[name] = (f, o, wb)
    return out


def ctx_of(o, s):
    return tuple(BOS if t == o.V else t for t in o.context(s))


@pytest.mark.parametrize("name", NAMES)
def test_backoff_equals_interpolation_from_counts(models, name):
    f, o, wb = models[name]
    states = np.arange(o.num_states, dtype=np.int32)
    if states.size > 400:
        states = np.sort(np.random.default_rng(0).choice(states, 400, replace=False))
    s32, s64, nx, lv = o.rows(states)
    f32, f64 = o.finals(states)
    for i, s in enumerate(states):
        ctx = ctx_of(o, s)
        exp = np.array([wb.lnP(v, ctx) for v in range(o.V)])
        # ARPA values carry 10 significant digits: |error| ~ 1e-10 per term
        np.testing.assert_allclose(s64[i], exp, rtol=0, atol=2e-8, err_msg=f"state {s} {ctx}")
        assert abs(f64[i] - wb.lnP(EOS, ctx)) < 2e-8


@pytest.mark.parametrize("name", NAMES)
def test_normalization(models, name):
    f, o, wb = models[name]
    assert o.num_unk_filled == wb.M and wb.M >= 1
    states = np.arange(o.num_states, dtype=np.int32)
    s32, s64, nx, lv = o.rows(states)
    f32, f64 = o.finals(states)
    tot = np.exp(s64).sum(axis=1) + np.exp(f64)
    np.testing.assert_allclose(tot, 1.0, rtol=0, atol=1e-7)
    tot32 = np.exp(s32.astype(np.float64)).sum(axis=1) + np.exp(f32.astype(np.float64))
    np.testing.assert_allclose(tot32, 1.0, rtol=0, atol=1e-4)


@pytest.mark.parametrize("name", NAMES)
def test_f32_algorithm1_within_bound_of_definition(models, name):
    f, o, wb = models[name]
    states = np.arange(o.num_states, dtype=np.int32)
    s32, s64, nx, lv = o.rows(states)
    # <= N back-off conversions + adds and one weight conversion, each <= 1/2 ulp
    # of a magnitude <= |score| (all WB weights and back-offs are <= 0)
    bound = (o.order + 1) * np.spacing(np.abs(s64).astype(np.float32)).astype(np.float64)
    assert np.all(np.abs(s32 - s64) <= bound)
    assert np.max(np.abs(s32 - s64)) < 1e-5


@pytest.mark.parametrize("name", NAMES)
def test_depth_bound_and_root(models, name):
    f, o, wb = models[name]
    states = np.arange(o.num_states, dtype=np.int32)
    s32, s64, nx, lv = o.rows(states)
    assert lv.max() <= max(1, o.order)
    assert lv[0] == 1
    # the root row is the unigram row (unk-normalized for absent tokens)
    exp = np.array([wb.lnP(v, ()) for v in range(o.V)])
    np.testing.assert_allclose(s64[0], exp, atol=2e-8)
    for v in range(o.V):
        if (v,) not in wb.count or o.order == 1:
            assert nx[0][v] == 0                # unk-filled (or N = 1): root
        else:
            assert o.context(nx[0][v]) == [v]   # the unigram state of v
    # every next id is a state whose context is a suffix of ctx(s)+v
    for i in range(0, len(states), max(1, len(states) // 50)):
        c = list(o.context(int(states[i])))
        for v in range(0, o.V, 3):
            nc = o.context(int(nx[i][v]))
            full = c + [v]
            assert full[len(full) - len(nc):] == nc if nc else True


def test_unigram_only_model(models):
    f, o, wb = models["uni16"]
    assert o.order == 1 and o.num_states == 1 and o.bos_state == 0


@pytest.mark.parametrize("name", NAMES)
def test_sentence_replay_pins_next(models, name):
    """Walking next states from <s> must keep the full history: the score at every
    step equals the interpolated P(v | last N-1 tokens), computed from counts."""
    f, o, wb = models[name]
    sents = synth.read_sentences(f.heldout)[:20] + synth.read_sentences(f.corpus)[:5]
    for sent in sents:
        s, hist = o.bos_state, [BOS]
        for v in sent:
            s32, s64, nx, _ = o.rows(np.array([s], dtype=np.int32))
            assert abs(s64[0][v] - wb.lnP(v, tuple(hist))) < 2e-8
            s = int(nx[0][v])
            hist.append(v)
        f32, f64 = o.finals(np.array([s], dtype=np.int32))
        assert abs(f64[0] - wb.lnP(EOS, tuple(hist))) < 2e-8


def test_state_of_matches_replay(models):
    f, o, wb = models["five48"]
    for sent in synth.read_sentences(f.heldout)[:10]:
        s = o.bos_state
        for i, v in enumerate(sent):
            _, _, nx, _ = o.rows(np.array([s], dtype=np.int32), want64=False)
            s = int(nx[0][v])
            assert o.state_of(True, sent[: i + 1]) == s


def test_bad_arpa_rejected(tmp_path, fig1_paths):
    arpa, vocab = fig1_paths
    txt = open(arpa).read()
    cases = {
        "noend": txt.replace("\\end\\", ""),
        "count": txt.replace("ngram 2=7", "ngram 2=8"),
        "oov": txt.replace("\tcat sat\t", "\tcat zzz\t"),
        "noeos": txt.replace("-0.90308998699194354\t</s>\n", ""),
        "dup": txt.replace("\\3-grams:\n", "\\3-grams:\n-0.1\tthe cat sat\n").replace("ngram 3=6", "ngram 3=7"),
    }
    for name, t in cases.items():
        p = tmp_path / f"{name}.arpa"
        p.write_text(t)
        with pytest.raises(ValueError):
            Oracle(str(p), vocab)


# ---------------------------------------------------------------- pruned LMs: missing contexts (R7, R8)
def _arpa_entries(path):
    ents, sec = set(), 0
    for line in open(path):
        line = line.strip()
        if line.startswith("\\") and line.endswith("-grams:"):
            sec = int(line[1:].split("-")[0])
        elif sec and line and not line.startswith("\\"):
            ents.add(tuple(line.split("\t")[1].split()))
    return ents


@pytest.mark.parametrize("name", ["pr3", "pr4", "pr6"])
def test_pruned_lms_have_missing_suffixes_and_stay_normalized(pruned_lms, name):
    """lmgen renormalizes the back-off weights of a pruned LM (its own derivation);
    the oracle's back-off definition must then still sum to one for every state —
    with kept n-grams whose suffix context is missing, this pins the oracle's
    reading of missing contexts (they add log 1 = 0 and the walk goes on to the
    next shorter suffix, R8) and its arc targets (longest suffix that is a state,
    R7: replay below)."""
    f = pruned_lms[name]
    ents = _arpa_entries(f.arpa)
    missing = sum(1 for e in ents if len(e) >= 3 and e[1:] not in ents)
    assert missing > 10, "the thresholds must leave missing suffixes"
    o = Oracle(f.arpa, vocab_size=f.vocab_size)
    st = np.arange(o.num_states, dtype=np.int32)
    s32, s64, nx, lv = o.rows(st)
    _, f64 = o.finals(st)
    tot = np.exp(s64).sum(1) + np.exp(f64)
    assert np.max(np.abs(tot - 1)) < 1e-7
    assert (lv <= f.order).all()                       # depth bound
    # next ids = the state of the longest suffix of context + v (replayed histories)
    sents = synth.read_sentences(f.heldout)
    for snt in sents[:20]:
        s = o.state_of(True, [])
        for i, v in enumerate(snt):
            _, _, n1, _ = o.rows(np.array([s], np.int32), want64=False)
            s = int(n1[0, v])
            assert s == o.state_of(True, snt[: i + 1])
