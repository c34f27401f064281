"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

INPUT GENERATION ONLY: nothing here computes NGPU-LM's method (no back-off
walk, no Algorithm 1, no fusion, no argmax). Both sides of every parity test
receive the same bytes from this module and compute on them independently.

* ``make_lm``      — runs ``lmgen`` (C++, interpolated Witten-Bell, see
                     lmgen.cpp) to write an ARPA file shaped like the paper's
                     token-level BPE-1024 LMs.
* ``read_sentences`` / ``sample_contexts`` — held-out token histories used to
                     pick "trajectory" LM states.
* ``ctc_logits`` / ``rnnt_logits`` / ``aed_logits`` — the logits recipe of
                     SURVEY.md §8(d) (seed 4): peaked log-softmax rows with
                     confusions and exact ties.
* ``splitmix64`` / ``synthetic_scorer_row`` — SPEC.md:280-283,348.

Recipes are stated in DESIGN.md §"Inputs".
"""
from __future__ import annotations

import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LMGEN_SRC = os.path.join(HERE, "lmgen.cpp")
LMGEN_BIN = os.path.join(HERE, "lmgen")
JOINT_SRC = os.path.join(HERE, "joint.cu")
JOINT_LIB = os.path.join(HERE, "libsynthjoint.so")


def build_lmgen(force: bool = False) -> str:
    if force or not os.path.exists(LMGEN_BIN) or (
        os.path.getmtime(LMGEN_BIN) < os.path.getmtime(LMGEN_SRC)
    ):
        subprocess.check_call(
            ["g++", "-O2", "-std=c++17", "-o", LMGEN_BIN, LMGEN_SRC]
        )
    return LMGEN_BIN


@dataclass
class LMFiles:
    arpa: str
    vocab_size: int
    order: int
    corpus: str | None = None
    heldout: str | None = None


def make_lm(
    out_dir: str,
    V: int,
    order: int,
    tokens: int = 0,
    seed: int = 1,
    absent: int = 1,
    lexicon: int = 20000,
    heldout: int = 0,
    keep_corpus: bool = False,
    corpus_in: str | None = None,
    minlen: int = 5,
    maxlen: int = 25,
    tag: str | None = None,
    prune: str | None = None,
) -> LMFiles:
    """Generate (deterministically from the arguments) an ARPA LM in out_dir."""
    build_lmgen()
    os.makedirs(out_dir, exist_ok=True)
    tag = tag or f"V{V}_N{order}_T{tokens}_s{seed}_a{absent}_L{lexicon}"
    arpa = os.path.join(out_dir, tag + ".arpa")
    cmd = [LMGEN_BIN, "--arpa", arpa, "--V", str(V), "--order", str(order),
           "--seed", str(seed), "--absent", str(absent), "--lexicon", str(lexicon),
           "--minlen", str(minlen), "--maxlen", str(maxlen)]
    corpus = held = None
    if prune:
        cmd += ["--prune", prune]
    if corpus_in is not None:
        cmd += ["--corpus-in", corpus_in]
        corpus = corpus_in
    else:
        cmd += ["--tokens", str(tokens)]
        if keep_corpus:
            corpus = os.path.join(out_dir, tag + ".corpus")
            cmd += ["--corpus-out", corpus]
    if heldout:
        held = os.path.join(out_dir, tag + ".heldout")
        cmd += ["--heldout", str(heldout), "--heldout-out", held]
    subprocess.run(cmd, check=True, stderr=subprocess.DEVNULL)
    return LMFiles(arpa=arpa, vocab_size=V, order=order, corpus=corpus, heldout=held)


def read_sentences(path: str) -> list[list[int]]:
    with open(path) as f:
        return [[int(t) for t in line.split()] for line in f if line.strip()]


def sample_contexts(sentences, order: int, n: int, seed: int):
    """Histories "<s> w1 .. wi" cut at random positions of held-out sentences.

    Returns a list of (with_bos, tokens) with at most order-1 trailing tokens:
    the LM context a decoder would hold after emitting w1..wi
    ("starts with the start-of-sequence token as a context").
    """
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(n):
        s = sentences[int(rng.integers(len(sentences)))]
        i = int(rng.integers(len(s) + 1))  # history length 0..len
        hist = s[:i]
        keep = order - 1
        if keep <= 0:
            out.append((False, []))
        elif len(hist) >= keep:
            out.append((False, hist[len(hist) - keep:]))
        else:
            out.append((True, hist))
    return out


def uniform_states(num_states: int, B: int, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    return rng.integers(0, num_states, size=B, dtype=np.int64).astype(np.int32)


# ----------------------------------------------------------------- logits recipe
def _log_softmax64(x: np.ndarray) -> np.ndarray:
    m = x.max(axis=-1, keepdims=True)
    z = x - m
    return z - np.log(np.exp(z).sum(axis=-1, keepdims=True))


def _peaked_rows(rng, targets: np.ndarray, ncols: int, blank_col: int,
                 confuse_p: float = 0.15, tie_frac: float = 0.01) -> np.ndarray:
    """targets[i] = column that should win row i. Returns f32 log-softmax rows."""
    n = targets.shape[0]
    x = rng.standard_normal((n, ncols))
    delta = rng.uniform(3.0, 7.0, size=n)
    x[np.arange(n), targets] += delta
    # confusions on token rows: another token column gets + (delta - eps)
    tok_rows = np.nonzero((targets != blank_col) & (rng.random(n) < confuse_p))[0]
    if tok_rows.size:
        other = rng.integers(0, ncols - 1, size=tok_rows.size)
        other = np.where(other >= blank_col, other + 1, other)  # never the blank column
        eps = rng.exponential(1.0 / 0.5, size=tok_rows.size)
        x[tok_rows, other] += delta[tok_rows] - eps
    # exact ties: some rows are quantized to multiples of 1/64 and get a second
    # column equal to their maximum, so the raw argmax has a tie to break
    tie_rows = np.nonzero(rng.random(n) < tie_frac)[0]
    if tie_rows.size:
        x[tie_rows] = np.round(x[tie_rows] * 64.0) / 64.0
        dup = rng.integers(0, ncols, size=tie_rows.size)
        x[tie_rows, dup] = x[tie_rows].max(axis=1)
    return _log_softmax64(x).astype(np.float32)


def _ctc_alignment(rng, ref: list[int], T: int, blank: int) -> np.ndarray:
    """Frame targets: each token holds 1/2/3 frames (p=.5/.3/.2); blanks fill the rest."""
    durs = rng.choice([1, 2, 3], size=len(ref), p=[0.5, 0.3, 0.2])
    # keep as many tokens as fit with one mandatory blank between repeats
    toks, frames, used = [], [], 0
    for t, d in zip(ref, durs):
        need = d + (1 if toks and toks[-1] == t else 0)
        if used + need > T:
            break
        toks.append(t); frames.append(int(d)); used += need
    spare = T - used
    gaps = np.zeros(len(toks) + 1, dtype=np.int64)
    if spare > 0:
        gaps += np.bincount(rng.integers(0, len(toks) + 1, size=spare), minlength=len(toks) + 1)
    out = []
    for i, (t, d) in enumerate(zip(toks, frames)):
        g = int(gaps[i]) + (1 if i and toks[i - 1] == t else 0)
        out += [blank] * g + [t] * d
    out += [blank] * int(gaps[-1])
    out = out[:T] + [blank] * max(0, T - len(out))
    return np.asarray(out, dtype=np.int64)


def ctc_logits(sentences, B: int, T: int, V: int, seed: int = 4,
               blank: int | None = None) -> np.ndarray:
    """[B, T, V+1] f32 log-softmax CTC posteriors (SURVEY.md §8(d) logits recipe)."""
    blank = V if blank is None else blank
    rng = np.random.default_rng(seed)
    out = np.empty((B, T, V + 1), dtype=np.float32)
    for b in range(B):
        ref = []
        while len(ref) < T:  # concatenate held-out sentences as the reference
            ref += sentences[int(rng.integers(len(sentences)))]
        tgt = _ctc_alignment(rng, ref[: T], T, V)  # token ids; V marks blank
        cols = np.where(tgt == V, blank, np.where(tgt >= blank, tgt + 1, tgt))
        out[b] = _peaked_rows(rng, cols, V + 1, blank)
    return out


def rnnt_logits(B: int, steps: int, V: int, seed: int = 4, blank_p: float = 0.5,
                blank: int | None = None) -> np.ndarray:
    """[steps, B, V+1]: per step the blank column wins with probability blank_p."""
    blank = V if blank is None else blank
    rng = np.random.default_rng(seed)
    out = np.empty((steps, B, V + 1), dtype=np.float32)
    for s in range(steps):
        is_blank = rng.random(B) < blank_p
        tok = rng.integers(0, V, size=B)
        cols = np.where(is_blank, blank, np.where(tok >= blank, tok + 1, tok))
        out[s] = _peaked_rows(rng, cols, V + 1, blank)
    return out


def aed_logits(B: int, steps: int, V: int, seed: int = 4,
               ref_len: tuple[int, int] = (5, 40), eos: int | None = None) -> np.ndarray:
    """[steps, B, V+1]: the eos column wins once a row reaches its reference length."""
    eos = V if eos is None else eos
    rng = np.random.default_rng(seed)
    L = rng.integers(ref_len[0], ref_len[1], size=B)
    out = np.empty((steps, B, V + 1), dtype=np.float32)
    for s in range(steps):
        tok = rng.integers(0, V, size=B)
        cols = np.where(s >= L, eos, np.where(tok >= eos, tok + 1, tok))
        out[s] = _peaked_rows(rng, cols, V + 1, eos)
    return out


# ----------------------------------------------------------------- SPEC scorer
_M64 = (1 << 64) - 1


def splitmix64(x: int) -> int:
    """z=(x+0x9E37..); z=(z^(z>>30))*0xBF58..; z=(z^(z>>27))*0x94D0..; z^(z>>31)."""
    z = (x + 0x9E3779B97F4A7C15) & _M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return z ^ (z >> 31)


def synthetic_scorer_row(seed: int, t: int, u: int, last: int, ncols: int,
                         temperature: float = 8.0) -> np.ndarray:
    """element v from splitmix64 of (seed, t, u, last+1, v) folded
    sequentially, mapped to [0,1), scaled by temperature, then log-softmax (f64 -> f32)."""
    h = seed
    for x in (t, u, last + 1):
        h = splitmix64(h ^ (x & _M64))
    vals = np.empty(ncols, dtype=np.float64)
    for v in range(ncols):
        vals[v] = (splitmix64(h ^ v) >> 11) * (1.0 / 9007199254740992.0)
    return _log_softmax64(vals * temperature).astype(np.float32)


# ---------------------------------------------------------------- synthetic transducer joint (f2 driver input)
def synthetic_joint_raw(seed: int, t: int, u: int, last: int, ncols: int, temperature: float = 8.0,
                        blank: int = -1, blank_bias: float = 0.0) -> np.ndarray:
    """CPU twin of synth/joint.cu: h = fold of (t, u, last+1) by splitmix64;
    x[v] = float32((splitmix64(h ^ v) >> 40) * 2^-24), x[blank] += blank_bias (float32),
    out = x * temperature; unnormalized scores."""
    h = seed & _M64
    for x in (t, u, last + 1):
        h = splitmix64(h ^ (x & _M64))
    r = np.array([splitmix64(h ^ v) >> 40 for v in range(ncols)], dtype=np.float64)
    x = r.astype(np.float32) * np.float32(5.9604644775390625e-08)
    if 0 <= blank < ncols:
        x[blank] = np.float32(x[blank] + np.float32(blank_bias))
    return x * np.float32(temperature)


def build_joint(force: bool = False) -> str:
    if force or not os.path.exists(JOINT_LIB) or os.path.getmtime(JOINT_LIB) < os.path.getmtime(JOINT_SRC):
        subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3",
                               "-shared", "-Xcompiler", "-fPIC", "-o", JOINT_LIB, JOINT_SRC])
    return JOINT_LIB


_joint = None


def joint_gpu(seed: int, frame, u, last, out, temperature: float = 8.0, blank: int = -1, blank_bias: float = 0.0,
              stream=None):
    """Fill out [B, ncols] (CUDA f32, contiguous rows) with the synthetic joint rows for
    (frame[b], u[b], last[b]) (CUDA int32 [B]); graph-capturable."""
    import ctypes as C
    import torch
    global _joint
    if _joint is None:
        L = C.CDLL(build_joint())
        L.synth_joint.restype = C.c_int
        L.synth_joint.argtypes = [C.c_uint64, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_int32,
                                  C.c_float, C.c_float, C.c_void_p, C.c_int64, C.c_void_p]
        _joint = L
    st = (stream or torch.cuda.current_stream()).cuda_stream
    rc = _joint.synth_joint(seed & _M64, out.shape[0], frame.data_ptr(), u.data_ptr(), last.data_ptr(),
                            out.shape[1], int(blank), float(blank_bias), float(temperature), out.data_ptr(),
                            out.stride(0), st)
    if rc != 0:
        raise RuntimeError(f"synth_joint: CUDA error {rc}")
