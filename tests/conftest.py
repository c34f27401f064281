"""Shared fixtures. GPU tests are marked @pytest.mark.gpu; everything else runs on CPU."""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")

# (name, V, order, corpus tokens, lexicon) — config 0 of BASELINE.json is "tiny3"
SMALL_LMS = [
    ("uni16", 16, 1, 300, 20),
    ("bi16", 16, 2, 400, 20),
    ("tiny3", 32, 3, 100, 40),
    ("tri64", 64, 3, 2000, 200),
    ("five48", 48, 5, 3000, 300),
    ("ten24", 24, 10, 1500, 100),
]


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: large synthetic LMs (seconds to minutes)")


@pytest.fixture(scope="session")
def lm_dir(tmp_path_factory):
    return str(tmp_path_factory.mktemp("lms"))


@pytest.fixture(scope="session")
def small_lms(lm_dir):
    import synth
    out = {}
    for name, V, N, T, L in SMALL_LMS:
        out[name] = synth.make_lm(lm_dir, V, N, tokens=T, seed=1, lexicon=L,
                                  keep_corpus=True, heldout=50, tag=name)
    return out


# count-pruned LMs (lmgen --prune, thresholds per order): non-monotone thresholds
# drop lower-order n-grams whose extensions survive, so kept n-grams have missing
# suffix contexts (the SPGI LM of PAPER.md:155 is pruned; readings R7/R8)
PRUNED_LMS = [
    ("pr3", 40, 3, 3000, 200, "0,4,0"),
    ("pr4", 48, 4, 4000, 300, "0,3,0,0"),
    ("pr6", 32, 6, 3000, 150, "0,2,5,0,1,0"),
]


@pytest.fixture(scope="session")
def pruned_lms(lm_dir):
    import synth
    return {name: synth.make_lm(lm_dir, V, N, tokens=T, seed=3, lexicon=L, heldout=50, tag=name, prune=pr)
            for name, V, N, T, L, pr in PRUNED_LMS}


@pytest.fixture(scope="session")
def fig1_paths():
    return os.path.join(GOLDEN, "fig1.arpa"), os.path.join(GOLDEN, "fig1.vocab")


# ---------------------------------------------------------------- GPU fixtures (session: built once)
GPU_SMALL = ["uni16", "bi16", "tiny3", "tri64", "five48", "ten24"]


@pytest.fixture(scope="session")
def pairs(small_lms, fig1_paths):
    """(library model on cuda:0, oracle, files) for every small LM and Fig. 1."""
    import paper_2505_22857_b200 as ng
    from oracle import Oracle
    out = {}
    for n in GPU_SMALL:
        f = small_lms[n]
        out[n] = (ng.load_arpa(f.arpa, vocab_size=f.vocab_size, device=0), Oracle(f.arpa, vocab_size=f.vocab_size), f)
    arpa, vocab = fig1_paths
    out["fig1"] = (ng.load_arpa(arpa, vocab, device=0), Oracle(arpa, vocab), None)
    return out


@pytest.fixture(scope="session")
def lm6(lm_dir):
    """BASELINE configs[1]: token 6-gram, V=1024 BPE-like, ~1M n-grams."""
    import paper_2505_22857_b200 as ng
    import synth
    from oracle import Oracle
    f = synth.make_lm(lm_dir, 1024, 6, tokens=430000, seed=1, heldout=2000, tag="cfg1_6gram")
    return ng.load_arpa(f.arpa, vocab_size=1024, device=0), Oracle(f.arpa, vocab_size=1024), f
