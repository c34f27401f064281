"""paper_2505_22857_b200 — B200-native NGPU-LM hot path (arXiv 2505.22857).

Thin ctypes binding over lib/libngpulm.so (C ABI: include/ngpulm.h). Every step
of the hot path runs in the library's CUDA kernels; this module only marshals
arguments (torch tensors -> device pointers, the current CUDA stream). There
is no CPU or PyTorch fallback: if the library is missing or a call fails, it
raises.

    lm = load_arpa("lm.arpa", vocab_size=1024, device=0)
    scores, nxt, fin = lm.advance(states)             # [B,V] f32, [B,V] i32, [B] f32
    tokens = lm.fused_greedy_step(CTC, logits_t, states, prev=prev, lam=0.3)
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("NGPULM_LIB") or os.path.join(HERE, "lib", "libngpulm.so")

NGPULM_OK, NGPULM_EDOMAIN, NGPULM_EUSAGE, NGPULM_ECUDA, NGPULM_EIO = 0, 1, 2, 3, 4
CTC, RNNT, AED = 0, 1, 2
CHAIN_TABLE, CHAIN_WALK = 0, 1
ADVANCE_AUTO, ADVANCE_WARP, ADVANCE_CTA = 0, 1, 2
STEP_LOGITS_READY = 1  # ngpulm_fused_greedy_step_ex flags
STEP_INPUTS_READY = 2
ADVANCE_INDEPENDENT = 1  # ngpulm_advance_ex flag
MAX_ORDER = 32
MAX_TOPK = 256


class NgpulmError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"ngpulm error {code}: {msg}")
        self.code = code


class Info(C.Structure):
    _fields_ = [("order", C.c_int32), ("vocab_size", C.c_int32), ("num_states", C.c_int32),
                ("root_state", C.c_int32), ("bos_state", C.c_int32), ("device", C.c_int32),
                ("num_arcs", C.c_int64), ("num_unk_filled", C.c_int64), ("num_dropped", C.c_int64),
                ("device_bytes", C.c_int64), ("max_vocab", C.c_int32), ("chain_mode", C.c_int32),
                ("advance_kernel", C.c_int32), ("packed_arcs", C.c_int32), ("max_fused_vocab", C.c_int32),
                ("tiny_resident", C.c_int32)]


class HostView(C.Structure):
    _fields_ = [("arc_tokens", C.c_void_p), ("arc_weights", C.c_void_p),
                ("arc_to_states", C.c_void_p), ("arc_offsets", C.c_void_p),
                ("boff_to_states", C.c_void_p), ("boff_weights", C.c_void_p),
                ("final_weights", C.c_void_p)]


# (name, restype, argtypes) — every symbol of include/ngpulm.h
_P, _I32, _I64, _F = C.c_void_p, C.c_int32, C.c_int64, C.c_float
SIGNATURES = {
    "ngpulm_load_arpa": (C.c_int, [C.c_char_p, C.c_char_p, _I32, _I32, C.POINTER(_P)]),
    "ngpulm_replicate": (C.c_int, [_P, _I32, C.POINTER(_P)]),
    "ngpulm_save": (C.c_int, [_P, C.c_char_p]),
    "ngpulm_load_binary": (C.c_int, [C.c_char_p, _I32, C.POINTER(_P)]),
    "ngpulm_free": (None, [_P]),
    "ngpulm_set_chain_mode": (C.c_int, [_P, _I32]),
    "ngpulm_set_advance_kernel": (C.c_int, [_P, _I32]),
    "ngpulm_get_info": (C.c_int, [_P, C.POINTER(Info)]),
    "ngpulm_host_view_get": (C.c_int, [_P, C.POINTER(HostView)]),
    "ngpulm_last_error": (C.c_char_p, []),
    "ngpulm_state_of": (C.c_int, [_P, _I32, _P, _I32, C.POINTER(_I32)]),
    "ngpulm_advance": (C.c_int, [_P, _P, _I32, _P, _P, _P, _P]),
    "ngpulm_advance_ex": (C.c_int, [_P, _P, _I32, _P, _P, _P, C.c_uint32, _P]),
    "ngpulm_final": (C.c_int, [_P, _P, _I32, _P, _P]),
    "ngpulm_fused_greedy_step": (C.c_int, [_P, _I32, _P, _I64, _I32, _P, _P, _P, _F, _I32, _P, _P]),
    "ngpulm_fused_greedy_step_ex": (C.c_int, [_P, _I32, _P, _I64, _I32, _P, _P, _P, _F, _I32, _P, C.c_uint32,
                                               _P]),
    "ngpulm_fused_greedy_step_ilm": (C.c_int, [_P, _I32, _P, _I64, _I32, _P, _P, _P, _F, _I32, _P, _I64, _F, _P,
                                                _P]),
    "ngpulm_transducer_loop_step": (C.c_int, [_P, _P, _I64, _I32, _P, _P, _P, _P, _I32, _F, _I32, _P, _I64, _F,
                                               _P, _P, _P, _P, _I32, _P]),
    "ngpulm_tdt_loop_step": (C.c_int, [_P, _P, _I64, _P, _I64, _P, _I32, _I32, _P, _P, _P, _P, _I32, _F, _I32,
                                        _P, _I64, _F, _P, _P, _P, _P, _I32, _P]),
    "ngpulm_transducer_loop_step_ex": (C.c_int, [_P, _P, _I64, _I32, _P, _P, _P, _P, _I32, _F, _I32, _P, _I64, _F,
                                                  _P, _P, _P, _P, _I32, C.c_uint32, _P]),
    "ngpulm_tdt_loop_step_ex": (C.c_int, [_P, _P, _I64, _P, _I64, _P, _I32, _I32, _P, _P, _P, _P, _I32, _F, _I32,
                                           _P, _I64, _F, _P, _P, _P, _P, _I32, C.c_uint32, _P]),
    "ngpulm_fused_greedy_step_rows": (C.c_int, [_P, _I32, _P, _I64, _I32, _P, _P, _P, _I64, _P, _P, _P, _F, _I32,
                                                 _P, _P]),
    "ngpulm_fused_topk": (C.c_int, [_P, _P, _I64, _I32, _P, _P, _I64, _F, _F, _I32, _I32, _P, _P, _P, _P]),
    "ngpulm_ctc_greedy_decode": (C.c_int, [_P, _P, _I64, _I64, _I32, _I32, _P, _P, _P, _F, _I32, _P, _P, _P,
                                            _P]),
    "ngpulm_check": (C.c_int, [_P, _P, C.POINTER(_I64)]),
    "ngpulm_advance_host": (C.c_int, [_P, _P, _I32, _P, _P, _P, _P]),
    "ngpulm_touched_bytes": (C.c_int, [_P, _P, _I32, C.POINTER(_I64)]),
}

_lib = None


def lib():
    """Load libngpulm.so (in-tree). Raises if it has not been built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            if os.environ.get("NGPULM_LIB") and not hasattr(L, name):
                continue  # an older variant library (tools/ A/B runs) may lack newer calls
            fn = getattr(L, name)
            fn.restype, fn.argtypes = res, args
        _lib = L
    return _lib


def _check(code: int):
    if code != NGPULM_OK:
        raise NgpulmError(code, lib().ngpulm_last_error().decode(errors="replace"))


def _stream(stream):
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream  # torch.cuda.Stream


def _dev_ptr(t, dtype, name, numel=None):
    import torch
    if t is None:
        return None
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{name}: expected a CUDA tensor")
    if t.dtype != dtype:
        raise TypeError(f"{name}: expected {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name}: must be contiguous")
    if numel is not None and t.numel() < numel:
        raise ValueError(f"{name}: needs {numel} elements, has {t.numel()}")
    return t.data_ptr()


def _rows_ptr(t, B, ncols, name, row_stride=None):
    """Pointer to B rows of `ncols` contiguous float32 columns, row b at b*row_stride
    elements (default: the tensor's leading stride). Checks the column count and that
    every row the kernels read lies inside the tensor's storage."""
    import torch
    if not isinstance(t, torch.Tensor) or not t.is_cuda or t.dtype != torch.float32:
        raise TypeError(f"{name}: expected a CUDA float32 tensor")
    if t.dim() == 0 or t.shape[-1] != ncols or (t.dim() >= 2 and t.stride(-1) != 1):
        raise ValueError(f"{name}: needs {ncols} contiguous columns, got shape {tuple(t.shape)}")
    if t.dim() == 1 and B > 1:
        raise ValueError(f"{name}: a 1-D tensor holds one row, B = {B}")
    if t.dim() >= 2 and t.shape[0] < B:
        raise ValueError(f"{name}: needs {B} rows, has {t.shape[0]}")
    if row_stride is None:
        row_stride = t.stride(0) if t.dim() >= 2 else ncols
    if B > 1 and row_stride < ncols:
        raise ValueError(f"{name}: row stride {row_stride} < {ncols} columns")
    if B > 0:
        last = t.storage_offset() + (B - 1) * row_stride + ncols
        if last * 4 > t.untyped_storage().nbytes():
            raise ValueError(f"{name}: rows reach past the tensor's storage")
    return t.data_ptr(), row_stride


class NgpuLM:
    """A resident NGPU-LM model (one replica per device)."""

    def __init__(self, handle: int):
        self._h = C.c_void_p(handle)
        self.info = Info()
        _check(lib().ngpulm_get_info(self._h, C.byref(self.info)))
        self.V = self.info.vocab_size
        self.order = self.info.order
        self.num_states = self.info.num_states
        self.bos_state = self.info.bos_state
        self.device = self.info.device

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _lib is not None:
            _lib.ngpulm_free(h)
            self._h = None

    # ---------------------------------------------------------------- host helpers
    def set_chain_mode(self, mode: int) -> None:
        """CHAIN_TABLE (load-time chain records, default) or CHAIN_WALK (Algorithm 1 walk)."""
        _check(lib().ngpulm_set_chain_mode(self._h, mode))
        self.info.chain_mode = mode

    def set_advance_kernel(self, kind: int) -> None:
        """ADVANCE_AUTO (default: one warp per row, packed arcs when they fit),
        ADVANCE_WARP (one warp per row, three arc arrays) or ADVANCE_CTA (one CTA per row)."""
        _check(lib().ngpulm_set_advance_kernel(self._h, kind))
        self.info.advance_kernel = kind

    def save(self, path: str) -> None:
        """ngpulm_save: NGLM binary file (SPEC.md:209 format)."""
        _check(lib().ngpulm_save(self._h, path.encode()))

    def replicate(self, device: int) -> "NgpuLM":
        out = C.c_void_p()
        _check(lib().ngpulm_replicate(self._h, device, C.byref(out)))
        return NgpuLM(out.value)

    def state_of(self, with_bos: bool, tokens) -> int:
        arr = (C.c_int32 * max(1, len(tokens)))(*tokens)
        out = C.c_int32()
        _check(lib().ngpulm_state_of(self._h, int(with_bos), C.cast(arr, C.c_void_p), len(tokens),
                                     C.byref(out)))
        return out.value

    def host_arrays(self):
        """numpy views of the host copy of the flat trie (see ngpulm_host_view)."""
        import numpy as np
        hv = HostView()
        _check(lib().ngpulm_host_view_get(self._h, C.byref(hv)))
        A, S = self.info.num_arcs, self.num_states

        def arr(p, n, ct, dt):
            return np.ctypeslib.as_array(C.cast(p, C.POINTER(ct)), shape=(n,)).view(dt).copy()
        return {
            "arc_tokens": arr(hv.arc_tokens, A, C.c_int32, np.int32),
            "arc_weights": arr(hv.arc_weights, A, C.c_float, np.float32),
            "arc_to_states": arr(hv.arc_to_states, A, C.c_int32, np.int32),
            "arc_offsets": arr(hv.arc_offsets, S + 1, C.c_int32, np.int32),
            "boff_to_states": arr(hv.boff_to_states, S, C.c_int32, np.int32),
            "boff_weights": arr(hv.boff_weights, S, C.c_float, np.float32),
            "final_weights": arr(hv.final_weights, S, C.c_float, np.float32),
        }

    def touched_bytes(self, states_np) -> int:
        import numpy as np
        st = np.ascontiguousarray(states_np, dtype=np.int32)
        out = C.c_int64()
        _check(lib().ngpulm_touched_bytes(self._h, st.ctypes.data, st.size, C.byref(out)))
        return out.value

    # ---------------------------------------------------------------- hot path
    def advance(self, states, scores=None, next=None, final_out=None, want_final=True, stream=None,
                independent: bool = False):
        """ngpulm_advance: states [B] int32 (CUDA) -> scores [B,V] f32, next [B,V] i32, final [B].
        independent=True: ngpulm_advance_ex with NGPULM_ADVANCE_INDEPENDENT (no running kernel
        writes the states or touches the outputs: consecutive calls' stores overlap)."""
        import torch
        B = states.numel()
        if scores is None:
            scores = torch.empty((B, self.V), dtype=torch.float32, device=states.device)
        if next is None:
            next = torch.empty((B, self.V), dtype=torch.int32, device=states.device)
        if final_out is None and want_final:
            final_out = torch.empty(B, dtype=torch.float32, device=states.device)
        _check(lib().ngpulm_advance_ex(
            self._h, _dev_ptr(states, torch.int32, "states", B), B,
            _dev_ptr(scores, torch.float32, "scores", B * self.V),
            _dev_ptr(next, torch.int32, "next", B * self.V),
            _dev_ptr(final_out, torch.float32, "final_out", B), ADVANCE_INDEPENDENT if independent else 0,
            _stream(stream)))
        return scores, next, final_out

    def final(self, states, out=None, stream=None):
        import torch
        B = states.numel()
        if out is None:
            out = torch.empty(B, dtype=torch.float32, device=states.device)
        _check(lib().ngpulm_final(self._h, _dev_ptr(states, torch.int32, "states", B), B,
                                  _dev_ptr(out, torch.float32, "out", B), _stream(stream)))
        return out

    def fused_greedy_step(self, mode: int, logits, states, prev=None, active=None, lam: float = 0.3,
                          blank_id: int | None = None, tokens_out=None, row_stride: int | None = None,
                          B: int | None = None, stream=None, logits_ready: bool = False,
                          inputs_ready: bool = False):
        """ngpulm_fused_greedy_step (ngpulm_fused_greedy_step_ex with logits_ready:
        NGPULM_STEP_LOGITS_READY, inputs_ready: NGPULM_STEP_INPUTS_READY). logits: CUDA f32 tensor whose row b starts at
        b*row_stride (default: a [B, V+1] contiguous tensor, or a strided 2-D view
        such as logits3d[:, t] of a [B, T, V+1] tensor). states/prev updated in place.
        states=None with lam=0: plain greedy decoding (no LM)."""
        import torch
        if B is None:
            B = states.numel() if states is not None else logits.shape[0]
        lp, row_stride = _rows_ptr(logits, B, self.V + 1, "logits", row_stride)
        if tokens_out is None:
            tokens_out = torch.empty(B, dtype=torch.int32, device=logits.device)
        blank = self.V if blank_id is None else blank_id
        _check(lib().ngpulm_fused_greedy_step_ex(
            self._h, mode, lp, row_stride, B,
            _dev_ptr(states, torch.int32, "states", B) if states is not None else None,
            _dev_ptr(prev, torch.int32, "prev", B) if prev is not None else None,
            _dev_ptr(active, torch.uint8, "active", B) if active is not None else None,
            float(lam), blank, _dev_ptr(tokens_out, torch.int32, "tokens_out", B),
            (STEP_LOGITS_READY if logits_ready else 0) | (STEP_INPUTS_READY if inputs_ready else 0),
            _stream(stream)))
        return tokens_out

    def fused_greedy_step_ilm(self, mode: int, logits, states, ilm, lam_ilm: float, prev=None, active=None,
                              lam: float = 0.3, blank_id: int | None = None, tokens_out=None, stream=None):
        """ngpulm_fused_greedy_step_ilm: the fused step minus lam_ilm * ilm[b, v] on the
        LM-rescored columns. ilm: [B, V] CUDA f32 (rows contiguous)."""
        import torch
        B = states.numel()
        lp, ls = _rows_ptr(logits, B, self.V + 1, "logits")
        ip, istr = _rows_ptr(ilm, B, self.V, "ilm")
        if tokens_out is None:
            tokens_out = torch.empty(B, dtype=torch.int32, device=states.device)
        blank = self.V if blank_id is None else blank_id
        _check(lib().ngpulm_fused_greedy_step_ilm(
            self._h, mode, lp, ls, B,
            _dev_ptr(states, torch.int32, "states", B),
            _dev_ptr(prev, torch.int32, "prev", B) if prev is not None else None,
            _dev_ptr(active, torch.uint8, "active", B) if active is not None else None,
            float(lam), blank, ip, istr, float(lam_ilm),
            _dev_ptr(tokens_out, torch.int32, "tokens_out", B), _stream(stream)))
        return tokens_out

    def transducer_loop_step(self, logits, states, frame_idx, sym_count, lengths, emit_out, emit_len,
                             last_token=None, lam: float = 0.3, blank_id: int | None = None,
                             max_symbols: int = 10, ilm=None, lam_ilm: float = 0.0, tokens_out=None,
                             durations=None, dur_logits=None, stream=None, inputs_ready: bool = False):
        """One label-looping iteration over B rows (all int32 [B] CUDA tensors updated in
        place; emit_out [B, max_len]): ngpulm_transducer_loop_step(_ex), or with `durations`
        (a sequence of ints) ngpulm_tdt_loop_step(_ex) — dur_logits [B, D] (default: the
        logits tensor's columns V+1 .. V+D). states=None with lam=0: no LM. inputs_ready:
        NGPULM_STEP_INPUTS_READY (the joint kernel before the step is a plain launch)."""
        import torch
        B = frame_idx.numel()
        lp, ls = _rows_ptr(logits[:, : self.V + 1], B, self.V + 1, "logits")
        ip, istr = _rows_ptr(ilm, B, self.V, "ilm") if ilm is not None else (None, 0)
        if tokens_out is None:
            tokens_out = torch.empty(B, dtype=torch.int32, device=frame_idx.device)
        max_len = emit_out.shape[1] if emit_out.dim() == 2 else 0
        blank = self.V if blank_id is None else blank_id
        common = (_dev_ptr(states, torch.int32, "states", B) if states is not None else None,
                  _dev_ptr(frame_idx, torch.int32, "frame_idx", B), _dev_ptr(sym_count, torch.int32, "sym_count", B),
                  _dev_ptr(lengths, torch.int32, "lengths", B), int(max_symbols), float(lam), blank,
                  ip, istr, float(lam_ilm), _dev_ptr(tokens_out, torch.int32, "tokens_out", B),
                  _dev_ptr(emit_out, torch.int32, "emit_out", B * max_len) if max_len else None,
                  _dev_ptr(emit_len, torch.int32, "emit_len", B),
                  _dev_ptr(last_token, torch.int32, "last_token", B) if last_token is not None else None,
                  max_len, STEP_INPUTS_READY if inputs_ready else 0, _stream(stream))
        if durations is None:
            _check(lib().ngpulm_transducer_loop_step_ex(self._h, lp, ls, B, *common))
        else:
            D = len(durations)
            if dur_logits is None:
                dur_logits = logits[:, self.V + 1: self.V + 1 + D]
            dp, dstr = _rows_ptr(dur_logits, B, D, "dur_logits")
            arr = (C.c_int32 * max(1, D))(*[int(x) for x in durations])
            _check(lib().ngpulm_tdt_loop_step_ex(self._h, lp, ls, dp, dstr, C.cast(arr, C.c_void_p), D, B, *common))
        return tokens_out

    def fused_greedy_step_rows(self, mode: int, logits, lm_scores, lm_next, lm_final, states, prev=None,
                               active=None, lam: float = 0.3, blank_id: int | None = None, tokens_out=None,
                               stream=None):
        """ngpulm_fused_greedy_step_rows: the fused step from rows an earlier
        advance(states) produced (lm_scores/lm_next [B, V], lm_final [B], AED only)."""
        import torch
        B = states.numel()
        lp, ls = _rows_ptr(logits, B, self.V + 1, "logits")
        sp_, sstr = _rows_ptr(lm_scores, B, self.V, "lm_scores")
        if lm_next.dtype != torch.int32 or not lm_next.is_cuda or lm_next.dim() != 2 or lm_next.shape[1] != self.V \
                or lm_next.stride(0) != sstr or lm_next.stride(1) != 1 or lm_next.shape[0] < B:
            raise ValueError("lm_next: expected int32 CUDA [B, V] rows with the scores' row stride")
        if tokens_out is None:
            tokens_out = torch.empty(B, dtype=torch.int32, device=states.device)
        blank = self.V if blank_id is None else blank_id
        _check(lib().ngpulm_fused_greedy_step_rows(
            self._h, mode, lp, ls, B, sp_, lm_next.data_ptr(),
            _dev_ptr(lm_final, torch.float32, "lm_final", B) if lm_final is not None else None, sstr,
            _dev_ptr(states, torch.int32, "states", B),
            _dev_ptr(prev, torch.int32, "prev", B) if prev is not None else None,
            _dev_ptr(active, torch.uint8, "active", B) if active is not None else None,
            float(lam), blank, _dev_ptr(tokens_out, torch.int32, "tokens_out", B), _stream(stream)))
        return tokens_out

    def fused_topk(self, logits, states, k: int, lam: float = 0.3, eos_id: int | None = None, ilm=None,
                   lam_ilm: float = 0.0, want_next: bool = True, stream=None):
        """ngpulm_fused_topk -> (scores [B,k] f32, cols [B,k] i32, next [B,k] i32 or None)."""
        import torch
        B = states.numel()
        lp, ls = _rows_ptr(logits, B, self.V + 1, "logits")
        ip, istr = _rows_ptr(ilm, B, self.V, "ilm") if ilm is not None else (None, 0)
        dev = logits.device
        sc = torch.empty((B, k), dtype=torch.float32, device=dev)
        cols = torch.empty((B, k), dtype=torch.int32, device=dev)
        nx = torch.empty((B, k), dtype=torch.int32, device=dev) if want_next else None
        eos = self.V if eos_id is None else eos_id
        _check(lib().ngpulm_fused_topk(
            self._h, lp, ls, B, _dev_ptr(states, torch.int32, "states", B), ip, istr,
            float(lam), float(lam_ilm), eos, k, sc.data_ptr(), cols.data_ptr(),
            nx.data_ptr() if nx is not None else None, _stream(stream)))
        return sc, cols, nx

    def ctc_greedy_decode(self, logits, states, prev, lam: float = 0.3, blank_id: int | None = None,
                          lengths=None, frames_out=None, emit_out=None, emit_len=None, want_frames=True,
                          stream=None):
        """ngpulm_ctc_greedy_decode over a [B, T, V+1] CUDA f32 tensor (any strides
        with contiguous columns). states/prev [B] int32 are updated in place.
        Returns (frames [B,T] or None, emitted [B,T], emit_len [B])."""
        import torch
        if logits.dtype != torch.float32 or not logits.is_cuda or logits.dim() != 3:
            raise TypeError("logits: expected a [B, T, V+1] CUDA float32 tensor")
        if logits.stride(2) != 1 or logits.shape[2] != self.V + 1:
            raise ValueError("logits: need V+1 contiguous columns")
        B, T = logits.shape[0], logits.shape[1]
        dev = logits.device
        if frames_out is None and want_frames:
            frames_out = torch.empty((B, T), dtype=torch.int32, device=dev)
        if emit_out is None:
            emit_out = torch.empty((B, T), dtype=torch.int32, device=dev)
        if emit_len is None:
            emit_len = torch.empty(B, dtype=torch.int32, device=dev)
        blank = self.V if blank_id is None else blank_id
        _check(lib().ngpulm_ctc_greedy_decode(
            self._h, logits.data_ptr(), logits.stride(0), logits.stride(1), B, T,
            _dev_ptr(lengths, torch.int32, "lengths", B) if lengths is not None else None,
            _dev_ptr(states, torch.int32, "states", B) if states is not None else None,
            _dev_ptr(prev, torch.int32, "prev", B), float(lam), blank,
            _dev_ptr(frames_out, torch.int32, "frames_out", B * T) if frames_out is not None else None,
            _dev_ptr(emit_out, torch.int32, "emit_out", B * T),
            _dev_ptr(emit_len, torch.int32, "emit_len", B), _stream(stream)))
        return frames_out, emit_out, emit_len

    def check(self, stream=None) -> int:
        out = C.c_int64()
        _check(lib().ngpulm_check(self._h, _stream(stream), C.byref(out)))
        return out.value

    def advance_host(self, states_h, scores_h, next_h, final_h=None, stream=None):
        """ngpulm_advance_host over host (ideally pinned) CPU tensors."""
        import torch
        B = states_h.numel()
        for t, dt in ((states_h, torch.int32), (scores_h, torch.float32), (next_h, torch.int32)):
            assert not t.is_cuda and t.dtype == dt and t.is_contiguous()
        _check(lib().ngpulm_advance_host(
            self._h, states_h.data_ptr(), B, scores_h.data_ptr(), next_h.data_ptr(),
            final_h.data_ptr() if final_h is not None else None, _stream(stream)))


def load_arpa(arpa_path: str, vocab_path: str | None = None, vocab_size: int = 0,
              device: int | None = None) -> NgpuLM:
    """ngpulm_load_arpa. device=None -> torch's current device; -1 -> host-only model."""
    if device is None:
        import torch
        device = torch.cuda.current_device()
    out = C.c_void_p()
    _check(lib().ngpulm_load_arpa(arpa_path.encode(), vocab_path.encode() if vocab_path else None,
                                  vocab_size, device, C.byref(out)))
    return NgpuLM(out.value)


def load_binary(path: str, device: int | None = None) -> NgpuLM:
    """ngpulm_load_binary. device=None -> torch's current device; -1 -> host-only model."""
    if device is None:
        import torch
        device = torch.cuda.current_device()
    out = C.c_void_p()
    _check(lib().ngpulm_load_binary(path.encode(), device, C.byref(out)))
    return NgpuLM(out.value)


# C-ABI names, for callers that mirror include/ngpulm.h
ngpulm_load_arpa = load_arpa
ngpulm_advance = NgpuLM.advance
ngpulm_advance_ex = NgpuLM.advance
ngpulm_final = NgpuLM.final
ngpulm_fused_greedy_step = NgpuLM.fused_greedy_step
ngpulm_fused_greedy_step_ex = NgpuLM.fused_greedy_step
ngpulm_check = NgpuLM.check
ngpulm_ctc_greedy_decode = NgpuLM.ctc_greedy_decode
ngpulm_fused_greedy_step_ilm = NgpuLM.fused_greedy_step_ilm
ngpulm_fused_topk = NgpuLM.fused_topk
ngpulm_save = NgpuLM.save
ngpulm_transducer_loop_step = NgpuLM.transducer_loop_step
ngpulm_tdt_loop_step = NgpuLM.transducer_loop_step
ngpulm_fused_greedy_step_rows = NgpuLM.fused_greedy_step_rows
ngpulm_load_binary = load_binary
ngpulm_replicate = NgpuLM.replicate
ngpulm_set_chain_mode = NgpuLM.set_chain_mode
ngpulm_set_advance_kernel = NgpuLM.set_advance_kernel
ngpulm_state_of = NgpuLM.state_of
ngpulm_advance_host = NgpuLM.advance_host
ngpulm_touched_bytes = NgpuLM.touched_bytes
