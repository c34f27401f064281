"""libngpulm.so on CPU: it loads, exports every symbol of include/ngpulm.h, and its
host-side builder (ARPA -> flat trie) is structurally right. No kernel runs here.
Structure pins: Fig. 1 and the
invariants of SPEC.md:106-110; state numbering agrees with the oracle's."""
import os
import re

import numpy as np
import pytest

import paper_2505_22857_b200 as ng
from conftest import ROOT


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "ngpulm.h")).read()
    return sorted(set(re.findall(r"\b(ngpulm_[a-z_]+)\s*\(", txt)))


def test_library_exports_every_header_symbol():
    L = ng.lib()
    syms = header_symbols()
    assert len(syms) >= 13
    for s in syms:
        assert hasattr(L, s), s
    assert set(syms) == set(ng.SIGNATURES), "binding and header disagree"


@pytest.fixture(scope="module")
def fig1(fig1_paths):
    arpa, vocab = fig1_paths
    return ng.load_arpa(arpa, vocab, device=-1)


def test_fig1_structure(fig1):
    i = fig1.info
    assert (i.order, i.vocab_size, i.num_states, i.bos_state, i.num_unk_filled) == (3, 6, 13, 6, 1)
    h = fig1.host_arrays()
    off, tok, to = h["arc_offsets"], h["arc_tokens"], h["arc_to_states"]
    assert i.num_arcs == 17
    arcs = {s: [(int(tok[a]), int(to[a])) for a in range(off[s], off[s + 1])] for s in range(13)}
    # root -> every token; the absent "dog" (5) is unk-filled and targets the root
    assert arcs[0] == [(0, 1), (1, 2), (2, 3), (3, 4), (4, 5), (5, 0)]
    assert arcs[1] == [(1, 7), (4, 8)] and arcs[2] == [(2, 9)] and arcs[3] == [(3, 10)]
    assert arcs[4] == [(0, 11)] and arcs[6] == [(0, 12)]
    # 3-gram arcs point to 2-gram states (Fig. 1 green arcs)
    assert arcs[7] == [(2, 9)] and arcs[9] == [(3, 10)] and arcs[10] == [(0, 11)]
    assert arcs[11] == [(4, 8)] and arcs[12] == [(1, 7)]
    assert arcs[5] == [] and arcs[8] == []                # only </s> finals
    assert h["boff_to_states"].tolist() == [0, 0, 0, 0, 0, 0, 0, 2, 5, 3, 4, 1, 1]
    bo = h["boff_weights"]
    assert bo[0] == 0 and np.allclose(bo[1:], np.log(0.5))
    fw = h["final_weights"].astype(np.float64)
    np.testing.assert_allclose(fw[[0, 5, 8]], np.log([1 / 8, 9 / 16, 25 / 32]), atol=1e-6)
    np.testing.assert_allclose(fw[7], np.log(1 / 32), atol=1e-6)  # via back-offs
    np.testing.assert_allclose(h["arc_weights"][5], np.log(1 / 8), atol=1e-7)  # unk-normalized


@pytest.mark.parametrize("name", ["uni16", "bi16", "tiny3", "tri64", "five48", "ten24"])
def test_builder_invariants_and_numbering(small_lms, name):
    from oracle import Oracle
    f = small_lms[name]
    m = ng.load_arpa(f.arpa, vocab_size=f.vocab_size, device=-1)
    o = Oracle(f.arpa, vocab_size=f.vocab_size)
    assert m.num_states == o.num_states and m.order == o.order and m.bos_state == o.bos_state
    h = m.host_arrays()
    off, tok = h["arc_offsets"], h["arc_tokens"]
    V, S = m.V, m.num_states
    assert off[0] == 0 and off[1] == V and (tok[:V] == np.arange(V)).all()
    for s in range(S):
        seg = tok[off[s]:off[s + 1]]
        assert (np.diff(seg) > 0).all()
    bt = h["boff_to_states"]
    assert bt[0] == 0 and h["boff_weights"][0] == 0
    for s in range(S):
        x, hops = s, 0
        while x != 0:
            x, hops = bt[x], hops + 1
        assert hops <= max(0, m.order - 1)
    assert (h["arc_to_states"] >= 0).all() and (h["arc_to_states"] < S).all()
    # the builder's ids equal the oracle's pinned numbering (R6)
    for s in range(S):
        ctx = o.context(s)
        bos = bool(ctx) and ctx[0] == o.V
        toks = ctx[1:] if bos else ctx
        assert m.state_of(bos, toks) == s


def test_bad_arpa_rejected(tmp_path, fig1_paths):
    arpa, vocab = fig1_paths
    txt = open(arpa).read()
    cases = {
        "noend": txt.replace("\\end\\", ""),
        "count": txt.replace("ngram 2=7", "ngram 2=8"),
        "oov": txt.replace("\tcat sat\t", "\tcat zzz\t"),
        "noeos": txt.replace("-0.90308998699194354\t</s>\n", "").replace("ngram 1=8", "ngram 1=7"),
        "dup": txt.replace("\\3-grams:\n", "\\3-grams:\n-0.1\tthe cat sat\n").replace("ngram 3=6", "ngram 3=7"),
        "prefix": txt.replace("\\3-grams:\n", "\\3-grams:\n-0.1\tmat the cat\n").replace("ngram 3=6", "ngram 3=7"),
        "predict_bos": txt.replace("\\2-grams:\n", "\\2-grams:\n-0.1\tthe <s>\n").replace("ngram 2=7", "ngram 2=8"),
        "nounk": txt.replace("-0.90308998699194354\t<unk>\n", "").replace("ngram 1=8", "ngram 1=7"),
        # a line in a section declared empty (order above N)
        "empty4": txt.replace("ngram 3=6\n", "ngram 3=6\nngram 4=0\n")
                     .replace("\\end\\", "\\4-grams:\n-0.1\tthe cat sat on\n\n\\end\\"),
    }
    # sections up to 200 declared empty, then a 200-token line —
    # more tokens than NGPULM_MAX_ORDER; must be EDOMAIN, never a buffer overrun
    decl = "".join(f"ngram {k}=0\n" for k in range(4, 201))
    hdrs = "".join(f"\\{k}-grams:\n" for k in range(4, 200))
    cases["order200"] = (txt.replace("ngram 3=6\n", "ngram 3=6\n" + decl)
                         .replace("\\end\\", hdrs + "\\200-grams:\n-0.1\t" + " ".join(["the"] * 200) + "\n\n\\end\\"))
    for name, t in cases.items():
        p = tmp_path / f"{name}.arpa"
        p.write_text(t)
        with pytest.raises(ng.NgpulmError) as e:
            ng.load_arpa(str(p), vocab, device=-1)
        assert e.value.code == ng.NGPULM_EDOMAIN, name
    with pytest.raises(ng.NgpulmError) as e:
        ng.load_arpa(str(tmp_path / "missing.arpa"), vocab, device=-1)
    assert e.value.code == ng.NGPULM_EIO


def test_unk_ngrams_dropped(tmp_path, fig1_paths):
    arpa, vocab = fig1_paths
    t = open(arpa).read().replace("\\2-grams:\n", "\\2-grams:\n-0.5\tthe <unk>\n").replace("ngram 2=7", "ngram 2=8")
    p = tmp_path / "unk.arpa"
    p.write_text(t)
    m = ng.load_arpa(str(p), vocab, device=-1)
    assert m.info.num_dropped == 1 and m.num_states == 13


def test_hot_calls_refuse_host_only_model(fig1):
    import ctypes as C
    L = ng.lib()
    r = L.ngpulm_advance(fig1._h, C.c_void_p(16), 1, C.c_void_p(16), C.c_void_p(16), None, None)
    assert r == ng.NGPULM_EUSAGE
    r = L.ngpulm_fused_greedy_step(fig1._h, 0, C.c_void_p(16), 7, 1, C.c_void_p(16), C.c_void_p(16),
                                   None, 0.5, 6, C.c_void_p(16), None)
    assert r == ng.NGPULM_EUSAGE


def test_step_flags_validated(fig1):
    """Unknown flag bits are refused (EUSAGE) by every *_ex step call, before any device work."""
    import ctypes as C
    L = ng.lib()
    p = C.c_void_p(16)
    for bad in (4, 8, 1 << 31):
        r = L.ngpulm_fused_greedy_step_ex(fig1._h, 0, p, 7, 1, p, p, None, 0.5, 6, p, bad, None)
        assert r == ng.NGPULM_EUSAGE
        r = L.ngpulm_transducer_loop_step_ex(fig1._h, p, 7, 1, p, p, p, p, 3, 0.5, 6, None, 0, 0.0, p, p, p, p, 8,
                                             bad, None)
        assert r == ng.NGPULM_EUSAGE
        d = (C.c_int32 * 1)(1)
        r = L.ngpulm_tdt_loop_step_ex(fig1._h, p, 7, p, 1, C.cast(d, C.c_void_p), 1, 1, p, p, p, p, 3, 0.5, 6, None,
                                      0, 0.0, p, p, p, p, 8, bad, None)
        assert r == ng.NGPULM_EUSAGE
    assert ng.STEP_LOGITS_READY == 1 and ng.STEP_INPUTS_READY == 2


def test_touched_bytes(fig1):
    # states 7 (the cat) -> 2 (cat) -> root: 2 state records + 1 + 1 arcs + root arcs + finals
    b = fig1.touched_bytes(np.array([7, 7], dtype=np.int32))
    assert b == 6 * 12 + 2 * 4 + 2 * 16 + 2 * 12


@pytest.mark.parametrize("name", ["pr3", "pr4", "pr6"])
def test_builder_on_pruned_lms(pruned_lms, name):
    """Pruned ARPAs with missing suffix contexts (R7/R8): the library's arc targets
    equal the oracle's next ids, its back-off targets are the longest proper suffix
    that is a state, and state numbering / state_of agree with the oracle."""
    from oracle import Oracle
    f = pruned_lms[name]
    m = ng.load_arpa(f.arpa, vocab_size=f.vocab_size, device=-1)
    o = Oracle(f.arpa, vocab_size=f.vocab_size)
    assert m.num_states == o.num_states
    h = m.host_arrays()
    off, tok, to, bt = h["arc_offsets"], h["arc_tokens"], h["arc_to_states"], h["boff_to_states"]
    st = np.arange(o.num_states, dtype=np.int32)
    _, _, nx, _ = o.rows(st, want64=False)
    for s in range(o.num_states):
        for a in range(off[s], off[s + 1]):
            assert to[a] == nx[s, tok[a]], (s, tok[a])
        if s == 0:
            continue
        ctx = o.context(s)[1:]
        bos = len(ctx) > 0 and ctx[0] == o.V
        assert bt[s] == o.state_of(bos, ctx[1:] if bos else ctx), s
