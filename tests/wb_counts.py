"""Interpolated Witten-Bell probabilities recomputed straight from corpus counts.

Used as an independent pin for the oracle: the oracle only ever sees the ARPA
file and evaluates the back-off recursion of PAPER.md:98; this module never
reads the ARPA and evaluates the *interpolation* formula of the estimator
 from raw n-gram counts. For an interpolated Witten-Bell LM
with back-off alpha(c) = T(c)/(C(c)+T(c)) the two are the same function, so any
dropped term, wrong sign, wrong suffix or transposed index in the oracle's
back-off walk shows up as a mismatch.
"""
from __future__ import annotations

import math
from collections import Counter, defaultdict
from functools import lru_cache

BOS, EOS = "<s>", "</s>"


class WittenBell:
    def __init__(self, sentences, order: int, V: int, u: float = 1.0):
        self.N, self.V, self.u = order, V, u
        self.count = Counter()            # n-gram tuple -> count
        for s in sentences:
            pad = [BOS] + list(s) + [EOS]
            for i in range(len(pad)):
                for k in range(1, order + 1):
                    if i + k > len(pad):
                        break
                    self.count[tuple(pad[i:i + k])] += 1
        self.ctx_total = Counter()        # C(c) = sum of successor counts
        self.ctx_types = Counter()        # T(c) = number of distinct successors
        for g, c in self.count.items():
            if len(g) >= 2:
                self.ctx_total[g[:-1]] += c
                self.ctx_types[g[:-1]] += 1
        self.ntok = sum(c for g, c in self.count.items() if len(g) == 1 and g[0] != BOS)
        self.M = sum(1 for v in range(V) if (v,) not in self.count)
        self.P = lru_cache(maxsize=None)(self._P)

    def _P(self, v, ctx: tuple) -> float:
        """P(v | ctx), v a token id or EOS; ctx a tuple of ids (and BOS)."""
        ctx = ctx[-(self.N - 1):] if self.N > 1 else ()
        if not ctx:
            c = self.count.get((v,), 0)
            if c:
                return c / (self.ntok + self.u)
            return (self.u / (self.ntok + self.u)) / self.M  # normalized <unk>
        C, T = self.ctx_total.get(ctx, 0), self.ctx_types.get(ctx, 0)
        lower = self.P(v, ctx[1:])
        if C == 0:
            return lower
        return (self.count.get(ctx + (v,), 0) + T * lower) / (C + T)

    def lnP(self, v, ctx) -> float:
        return math.log(self.P(v, tuple(ctx)))
