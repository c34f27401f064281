"""Label-looping greedy transducer decoding with NGPU-LM shallow fusion
(the greedy loops run under CUDA
graphs, the LM query fused into the two-stage selection).

Every iteration of the loop is two launches on the decoder's stream — the
caller's joint network for each row's (frame, u, last label), then
ngpulm_transducer_loop_step (fused LM row + two-stage argmax + loop
bookkeeping, all on the GPU). `graph_steps` iterations are captured once in
one CUDA graph; the host reads the "any row still active" flag once per graph
replay, so the loop costs one host synchronisation per `graph_steps`
iterations and never a per-step one. Everything here is plumbing: the
arithmetic runs in libngpulm's kernels and the caller's joint.
"""
from __future__ import annotations

from dataclasses import dataclass


@dataclass
class TransducerResult:
    emitted: "object"   # [B, max_len] int32 CUDA: emitted columns (row b: emitted[b, :emit_len[b]])
    emit_len: "object"  # [B] int32 CUDA (> max_len: truncated)
    states: "object"    # [B] int32 CUDA: final LM states
    iterations: int     # loop iterations run (graph replays x graph_steps)


class TransducerGreedyDecoder:
    """Batched greedy transducer decoding with fusion, for batches of up to B rows.

    joint(frame_idx, u, last, out): fills out [B, V+1] (CUDA f32) with the joint
        network's logits for each row's current frame, label count u and last LM
        token (-1 = none), on the current stream; must be CUDA-graph capturable
        (fixed buffers, no host synchronisation). It is called for all B rows;
        rows that are done are ignored by the loop step.
    ilm: optional [B, V] f32 CUDA internal-LM rows (HAT), subtracted with lam_ilm.
    The graph is captured on first use and replayed for every later batch.
    """

    def __init__(self, model, joint, B: int, max_frames: int, lam: float = 0.3, max_symbols: int = 10,
                 max_len: int | None = None, blank_id: int | None = None, ilm=None, lam_ilm: float = 0.0,
                 graph_steps: int = 32, use_graph: bool = True, device=None, durations=None, use_lm: bool = True,
                 joint_plain_launch: bool = False):
        import torch
        self.m, self.joint, self.B = model, joint, B
        self.lam, self.max_symbols, self.blank_id = lam, max_symbols, blank_id
        self.ilm, self.lam_ilm = ilm, lam_ilm
        # TDT: the joint writes V+1 token and len(durations) duration logits per row
        self.durations = None if durations is None else [int(d) for d in durations]
        self.use_lm = use_lm  # False: plain greedy (no LM state), the overhead baseline
        # True: the joint launches its kernels without programmatic dependent launch (every cuBLAS /
        # PyTorch kernel), so each loop step runs with NGPULM_STEP_INPUTS_READY
        self.inputs_ready = joint_plain_launch
        self.graph_steps, self.use_graph = graph_steps, use_graph
        self.max_frames = max_frames
        self.max_len = max_len if max_len is not None else max_frames * max_symbols
        dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        z = lambda: torch.zeros(B, dtype=torch.int32, device=dev)  # noqa: E731
        self.lengths, self.st, self.frame, self.sym, self.elen = z(), z(), z(), z(), z()
        self.last = torch.full((B,), -1, dtype=torch.int32, device=dev)
        self.emit = torch.full((B, max(1, self.max_len)), -1, dtype=torch.int32, device=dev)[:, : self.max_len]
        ncols = model.V + 1 + (len(self.durations) if self.durations else 0)
        self.logits = torch.empty((B, ncols), dtype=torch.float32, device=dev)
        self.tok = torch.empty(B, dtype=torch.int32, device=dev)
        self.active = torch.zeros((), dtype=torch.bool, device=dev)
        self.stream = torch.cuda.Stream(device=dev)  # captures need a non-default stream
        self.graph = None

    def _iteration(self):
        self.joint(self.frame, self.elen, self.last, self.logits)
        self.m.transducer_loop_step(self.logits, self.st if self.use_lm else None, self.frame, self.sym,
                                    self.lengths, self.emit, self.elen, last_token=self.last,
                                    lam=self.lam if self.use_lm else 0.0, blank_id=self.blank_id,
                                    max_symbols=self.max_symbols, ilm=self.ilm, lam_ilm=self.lam_ilm,
                                    tokens_out=self.tok, durations=self.durations, stream=self.stream,
                                    inputs_ready=self.inputs_ready)

    def _body(self):
        import torch
        for _ in range(self.graph_steps):
            self._iteration()
        torch.any(self.frame < self.lengths, out=self.active)

    def _reset(self, lengths, states):
        self.lengths.copy_(lengths)
        if states is None:
            self.st.zero_()
        else:
            self.st.copy_(states)
        for t in (self.frame, self.sym, self.elen):
            t.zero_()
        self.last.fill_(-1)

    def __call__(self, lengths, states=None) -> TransducerResult:
        """Decode one batch: lengths [B] int32 CUDA (<= max_frames), states [B] int32
        CUDA start LM states (default: the root, SPEC.md's choice for transducers)."""
        import torch
        s = self.stream
        s.wait_stream(torch.cuda.current_stream(s.device))
        with torch.cuda.stream(s):
            self._reset(lengths, states)
            if self.use_graph and self.graph is None:
                self._body()  # one eager pass (joint warm-up), then capture from a clean state
                self._reset(lengths, states)
                s.synchronize()
                self.graph = torch.cuda.CUDAGraph()
                with torch.cuda.graph(self.graph, stream=s):
                    self._body()
            run = self.graph.replay if self.use_graph else self._body
            bound = self.max_frames * (self.max_symbols + 1) + 1  # each iteration advances a frame or emits
            bound = (bound + self.graph_steps - 1) // self.graph_steps * self.graph_steps
            iters = 0
            while iters < bound:
                run()
                iters += self.graph_steps
                if not bool(self.active.item()):
                    break
        torch.cuda.current_stream(s.device).wait_stream(s)
        return TransducerResult(self.emit, self.elen, self.st, iters)


def transducer_greedy_decode(model, joint, lengths, states=None, lam: float = 0.3, max_symbols: int = 10,
                             max_len: int | None = None, blank_id: int | None = None, ilm=None,
                             lam_ilm: float = 0.0, graph_steps: int = 32, use_graph: bool = True,
                             durations=None, use_lm: bool = True,
                             joint_plain_launch: bool = False) -> TransducerResult:
    """One-shot TransducerGreedyDecoder over lengths [B] int32 CUDA (see the class);
    durations=[...] decodes a TDT model (the joint writes V+1+len(durations) columns)."""
    B = lengths.numel()
    max_frames = int(lengths.max().item()) if B else 0
    dec = TransducerGreedyDecoder(model, joint, B, max_frames, lam=lam, max_symbols=max_symbols, max_len=max_len,
                                  blank_id=blank_id, ilm=ilm, lam_ilm=lam_ilm, graph_steps=graph_steps,
                                  use_graph=use_graph, device=lengths.device, durations=durations, use_lm=use_lm,
                                  joint_plain_launch=joint_plain_launch)
    if B == 0:
        return TransducerResult(dec.emit, dec.elen, dec.st, 0)
    return dec(lengths, states)
