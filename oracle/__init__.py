"""NGPU-LM oracle — TEST INFRASTRUCTURE ONLY (ctypes over oracle.cpp).

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline and the
``--impl reference`` arm) may import this module. The product path
(paper_2505_22857_b200) never imports it; the two share no code. See
oracle.cpp's header for what each function computes and the paper passage it
follows, and DESIGN.md §Oracle for the pins.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "oracle.cpp")
LIB = os.path.join(HERE, "liboracle.so")
CTC, RNNT, AED = 0, 1, 2

_lib = None


def build(force: bool = False) -> str:
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        # -ffp-contract=off: every float add/fma is exactly the one written (R10, R13)
        subprocess.check_call(["g++", "-O2", "-std=c++17", "-fPIC", "-shared", "-pthread",
                               "-ffp-contract=off", "-o", LIB, SRC])
    return LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(LIB)
        P = C.c_void_p
        i32p, f32p, f64p = (np.ctypeslib.ndpointer(dtype=t, flags="C_CONTIGUOUS")
                            for t in (np.int32, np.float32, np.float64))
        L.oracle_last_error.restype = C.c_char_p
        L.oracle_load.restype = P
        L.oracle_load.argtypes = [C.c_char_p, C.c_char_p, C.c_int32]
        L.oracle_free.argtypes = [P]
        for n in ("oracle_vocab_size", "oracle_order", "oracle_num_states", "oracle_bos_state"):
            getattr(L, n).restype = C.c_int32
            getattr(L, n).argtypes = [P]
        L.oracle_num_unk_filled.restype = C.c_int64
        L.oracle_num_unk_filled.argtypes = [P]
        L.oracle_state_context.restype = C.c_int32
        L.oracle_state_context.argtypes = [P, C.c_int32, i32p, C.c_int32]
        L.oracle_state_of.restype = C.c_int32
        L.oracle_state_of.argtypes = [P, C.c_int32, i32p, C.c_int32]
        L.oracle_rows.argtypes = [P, i32p, C.c_int64, f32p, P, i32p, P, C.c_int]
        L.oracle_finals.argtypes = [P, i32p, C.c_int64, f32p, P]
        L.oracle_fused_step.argtypes = [P, C.c_int, f32p, C.c_int64, C.c_int64, i32p, P, P,
                                        C.c_float, C.c_int32, i32p, C.c_int]
        L.oracle_fused_step_ilm.argtypes = [P, C.c_int, f32p, C.c_int64, C.c_int64, i32p, P, P, C.c_float,
                                            C.c_int32, f32p, C.c_int64, C.c_float, i32p, C.c_int]
        L.oracle_topk.argtypes = [P, f32p, C.c_int64, C.c_int64, i32p, P, C.c_int64, C.c_float, C.c_float,
                                  C.c_int32, C.c_int32, f32p, i32p, i32p, C.c_int]
        L.oracle_transducer_decode.argtypes = [P, C.c_uint64, C.c_float, C.c_float, i32p, C.c_int64, i32p, C.c_float,
                                               C.c_int32, C.c_int32, C.c_int32, P, C.c_float, i32p, i32p, C.c_int]
        L.oracle_tdt_decode.argtypes = [P, C.c_uint64, C.c_float, C.c_float, i32p, C.c_int64, i32p, C.c_float,
                                        C.c_int32, i32p, C.c_int32, C.c_int32, C.c_int32, i32p, i32p, i32p, C.c_int]
        L.oracle_ctc_decode.argtypes = [P, f32p, C.c_int64, C.c_int64, C.c_int64, C.c_int32, P, i32p, i32p,
                                        C.c_float, C.c_int32, i32p, i32p, i32p, C.c_int]
        _lib = L
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


class Oracle:
    """Hash-map ARPA back-off model."""

    def __init__(self, arpa: str, vocab: str | None = None, vocab_size: int = 0):
        L = lib()
        h = L.oracle_load(arpa.encode(), vocab.encode() if vocab else None, vocab_size)
        if not h:
            raise ValueError("oracle: " + L.oracle_last_error().decode())
        self.h = h
        self.V = L.oracle_vocab_size(h)
        self.order = L.oracle_order(h)
        self.num_states = L.oracle_num_states(h)
        self.bos_state = L.oracle_bos_state(h)
        self.num_unk_filled = L.oracle_num_unk_filled(h)

    def __del__(self):
        if getattr(self, "h", None):
            lib().oracle_free(self.h)
            self.h = None

    def context(self, s: int) -> list[int]:
        buf = np.zeros(max(1, self.order), dtype=np.int32)
        n = lib().oracle_state_context(self.h, int(s), buf, buf.size)
        return buf[:n].tolist()

    def state_of(self, with_bos: bool, tokens) -> int:
        t = np.ascontiguousarray(tokens, dtype=np.int32)
        if t.size == 0:
            t = np.zeros(1, dtype=np.int32)
            return lib().oracle_state_of(self.h, int(with_bos), t, 0)
        return lib().oracle_state_of(self.h, int(with_bos), t, t.size)

    def rows(self, states, want64: bool = True, nthreads: int = 0):
        """-> (score32 [n,V] f32, score64 [n,V] f64 or None, next [n,V] i32, levels [n])"""
        st = np.ascontiguousarray(states, dtype=np.int32)
        n = st.size
        s32 = np.empty((n, self.V), dtype=np.float32)
        nx = np.empty((n, self.V), dtype=np.int32)
        lv = np.empty(n, dtype=np.int32)
        s64 = np.empty((n, self.V), dtype=np.float64) if want64 else None
        lib().oracle_rows(self.h, st, n, s32, _ptr(s64), nx, _ptr(lv), nthreads)
        return s32, s64, nx, lv

    def finals(self, states):
        st = np.ascontiguousarray(states, dtype=np.int32)
        f32 = np.empty(st.size, dtype=np.float32)
        f64 = np.empty(st.size, dtype=np.float64)
        lib().oracle_finals(self.h, st, st.size, f32, _ptr(f64))
        return f32, f64

    def fused_step(self, mode: int, logits, states, prev=None, active=None,
                   lam: float = 0.3, blank_id: int | None = None, nthreads: int = 0):
        """One greedy shallow-fusion step. logits [n, V+1] (or strided rows of a
        [n, T, V+1] array already sliced to frame t and made contiguous).
        Returns (tokens, new_states, new_prev)."""
        x = np.ascontiguousarray(logits, dtype=np.float32)
        n = x.shape[0]
        st = np.array(states, dtype=np.int32, copy=True)
        pv = None if prev is None else np.array(prev, dtype=np.int32, copy=True)
        act = None if active is None else np.ascontiguousarray(active, dtype=np.uint8)
        tok = np.empty(n, dtype=np.int32)
        blank = self.V if blank_id is None else blank_id
        lib().oracle_fused_step(self.h, mode, x, x.shape[1], n, st, _ptr(pv), _ptr(act),
                                float(lam), int(blank), tok, nthreads)
        return tok, st, pv

    def ctc_decode(self, logits, states, prev=None, lam: float = 0.3, blank_id: int | None = None,
                   lengths=None, nthreads: int = 0):
        """Whole-utterance greedy CTC with fusion over logits [n, T, V+1].
        Returns (frames [n,T], emitted [n,T], emit_len [n], states, prev)."""
        x = np.ascontiguousarray(logits, dtype=np.float32)
        n, T = x.shape[0], x.shape[1]
        st = np.array(states, dtype=np.int32, copy=True).reshape(n)
        pv = (np.full(n, -1, dtype=np.int32) if prev is None
              else np.array(prev, dtype=np.int32, copy=True).reshape(n))
        ln = None if lengths is None else np.ascontiguousarray(lengths, dtype=np.int32)
        frames = np.empty((n, T), dtype=np.int32)
        emitted = np.full((n, T), -1, dtype=np.int32)
        elen = np.empty(n, dtype=np.int32)
        blank = self.V if blank_id is None else blank_id
        lib().oracle_ctc_decode(self.h, x, T * x.shape[2], x.shape[2], n, T, _ptr(ln), st, pv,
                                float(lam), int(blank), frames, emitted, elen, nthreads)
        return frames, emitted, elen, st, pv

    def fused_step_ilm(self, mode: int, logits, states, ilm, lam_ilm: float, prev=None, active=None,
                       lam: float = 0.3, blank_id: int | None = None, nthreads: int = 0):
        """fused_step with the ILM term (R21). ilm [n, V]. Returns (tokens, states, prev)."""
        x = np.ascontiguousarray(logits, dtype=np.float32)
        a = np.ascontiguousarray(ilm, dtype=np.float32)
        n = x.shape[0]
        st = np.array(states, dtype=np.int32, copy=True)
        pv = None if prev is None else np.array(prev, dtype=np.int32, copy=True)
        act = None if active is None else np.ascontiguousarray(active, dtype=np.uint8)
        tok = np.empty(n, dtype=np.int32)
        blank = self.V if blank_id is None else blank_id
        lib().oracle_fused_step_ilm(self.h, mode, x, x.shape[1], n, st, _ptr(pv), _ptr(act), float(lam),
                                    int(blank), a, a.shape[1], float(lam_ilm), tok, nthreads)
        return tok, st, pv

    def topk(self, logits, states, k: int, lam: float = 0.3, eos_id: int | None = None, ilm=None,
             lam_ilm: float = 0.0, nthreads: int = 0):
        """k best AED expansions per row -> (scores [n,k], cols [n,k], next [n,k])."""
        x = np.ascontiguousarray(logits, dtype=np.float32)
        n = x.shape[0]
        st = np.ascontiguousarray(states, dtype=np.int32)
        a = None if ilm is None else np.ascontiguousarray(ilm, dtype=np.float32)
        sc = np.empty((n, k), dtype=np.float32)
        cols = np.empty((n, k), dtype=np.int32)
        nx = np.empty((n, k), dtype=np.int32)
        eos = self.V if eos_id is None else eos_id
        lib().oracle_topk(self.h, x, x.shape[1], n, st, _ptr(a), 0 if a is None else a.shape[1], float(lam),
                          float(lam_ilm), int(eos), int(k), sc, cols, nx, nthreads)
        return sc, cols, nx

    def transducer_decode(self, seed: int, lengths, states, lam: float = 0.3, blank_id: int | None = None,
                          max_symbols: int = 10, max_len: int = 0, temperature: float = 8.0, ilm=None,
                          lam_ilm: float = 0.0, blank_bias: float = 0.0, nthreads: int = 0):
        """SPEC.md:317-325 greedy transducer loop over the synthetic joint (synth/joint.cu twin).
        ilm: optional [n, V] per-utterance ILM row (constant over steps). Returns (emitted [n, max_len],
        emit_len [n], states)."""
        ln = np.ascontiguousarray(lengths, dtype=np.int32)
        n = ln.size
        st = np.array(states, dtype=np.int32, copy=True).reshape(n)
        max_len = max_len or int(ln.max(initial=0)) * max_symbols
        em = np.full((n, max(1, max_len)), -1, dtype=np.int32)
        el = np.empty(n, dtype=np.int32)
        a = None if ilm is None else np.ascontiguousarray(ilm, dtype=np.float32)
        blank = self.V if blank_id is None else blank_id
        lib().oracle_transducer_decode(self.h, seed & ((1 << 64) - 1), float(temperature), float(blank_bias), ln, n,
                                       st, float(lam),
                                       int(blank), int(max_symbols), int(max_len), _ptr(a), float(lam_ilm),
                                       em, el, nthreads)
        return em[:, :max_len], el, st

    def tdt_decode(self, seed: int, lengths, states, durations, lam: float = 0.3, blank_id: int | None = None,
                   max_symbols: int = 10, max_len: int = 0, temperature: float = 8.0, blank_bias: float = 0.0,
                   nthreads: int = 0):
        """Greedy TDT loop (R25) over the synthetic joint with
        V+1+D columns (token columns, then one per entry of `durations`).
        Returns (emitted [n, max_len], emit_len [n], states, steps [n])."""
        ln = np.ascontiguousarray(lengths, dtype=np.int32)
        n = ln.size
        st = np.array(states, dtype=np.int32, copy=True).reshape(n)
        du = np.ascontiguousarray(durations, dtype=np.int32)
        max_len = max_len or int(ln.max(initial=0)) * max_symbols
        em = np.full((n, max(1, max_len)), -1, dtype=np.int32)
        el = np.empty(n, dtype=np.int32)
        steps = np.empty(n, dtype=np.int32)
        blank = self.V if blank_id is None else blank_id
        lib().oracle_tdt_decode(self.h, seed & ((1 << 64) - 1), float(temperature), float(blank_bias), ln, n, st,
                                float(lam), int(blank), du, int(du.size), int(max_symbols), int(max_len), em, el,
                                steps, nthreads)
        return em[:, :max_len], el, st, steps
