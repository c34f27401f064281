"""Property tests over random small LMs (hypothesis): corpora of random size,
vocabulary, order and count pruning (missing suffix contexts included). For
each generated ARPA, on CPU:
* the oracle's back-off values stay normalized per state (the generator
  renormalizes back-offs by its own derivation);
* the library's host builder agrees with the oracle: same state count, every
  arc target = the oracle's next id, every back-off target = the longest proper
  suffix that is a state, and state_of agrees on random histories.
The GPU side of the same LMs is exercised by tests/test_gpu_parity.py."""
import numpy as np
import pytest
from hypothesis import HealthCheck, given, settings
from hypothesis import strategies as st

import paper_2505_22857_b200 as ng
import synth
from oracle import Oracle


@settings(max_examples=40, deadline=None, suppress_health_check=[HealthCheck.function_scoped_fixture])
@given(V=st.sampled_from([8, 12, 20, 32]), order=st.integers(1, 5), tokens=st.integers(60, 1500),
       seed=st.integers(1, 10_000), prune=st.lists(st.integers(0, 4), min_size=5, max_size=5))
def test_random_lm_builder_and_oracle_agree(tmp_path_factory, V, order, tokens, seed, prune):
    d = str(tmp_path_factory.mktemp("rnd"))
    pr = ",".join(["0"] + [str(x) for x in prune[: order - 1]]) if order >= 2 else None
    f = synth.make_lm(d, V, order, tokens=tokens, seed=seed, lexicon=max(20, V * 3), heldout=5, tag="r", prune=pr)
    o = Oracle(f.arpa, vocab_size=V)
    m = ng.load_arpa(f.arpa, vocab_size=V, device=-1)
    assert m.num_states == o.num_states
    states = np.arange(o.num_states, dtype=np.int32)
    _, s64, nx, lv = o.rows(states)
    _, f64 = o.finals(states)
    tot = np.exp(s64).sum(1) + np.exp(f64)
    assert np.max(np.abs(tot - 1)) < 1e-6
    assert (lv <= max(1, m.order)).all()
    h = m.host_arrays()
    off, tok, to, bt = h["arc_offsets"], h["arc_tokens"], h["arc_to_states"], h["boff_to_states"]
    assert (off[1] == V) and (tok[:V] == np.arange(V)).all()   # the root owns the V root arcs
    for s in range(o.num_states):
        a, b = off[s], off[s + 1]
        assert (np.diff(tok[a:b]) > 0).all()                   # sorted by token
        assert (to[a:b] == nx[s, tok[a:b]]).all()
        if s:
            ctx = o.context(s)[1:]
            bos = len(ctx) > 0 and ctx[0] == o.V
            assert bt[s] == o.state_of(bos, ctx[1:] if bos else ctx)
    rng = np.random.default_rng(seed)
    for _ in range(50):
        toks = rng.integers(0, V, size=int(rng.integers(0, order + 3))).tolist()
        b = bool(rng.integers(2))
        assert m.state_of(b, toks) == o.state_of(b, toks)
