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


@pytest.fixture(scope="session")
def fig1_paths():
    return os.path.join(GOLDEN, "fig1.arpa"), os.path.join(GOLDEN, "fig1.vocab")
