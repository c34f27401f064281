#!/usr/bin/env python
"""NGPU-LM hot-path benchmark (driver contract: one JSON line from rank 0).

Metric (BASELINE.json): LM queries/s (B x V scores + next states) and % of the
B200 HBM roofline; fused greedy step us.

Workload at N=1 (the north_star headline): token 6-gram LM, V = 1024, ~0.94M
n-grams (synthetic interpolated Witten-Bell, synth/lmgen.cpp), one step = one
ngpulm_advance call with the fused final-weight gather (rows a0..a6 of
SURVEY.md §8(a)) over B = 1024 trajectory states per GPU. Multi-GPU: rows shard
across ranks with the trie replicated, no data-path collective (weak scaling).
Fused greedy steps (rows a7..a9) are timed in the same run and reported under
"fused_step_us".

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

V = 1024
ORDER = 6
CORPUS_TOKENS = 430_000
B_HEADLINE = 1024


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=2000)
    p.add_argument("--warmup", type=int, default=50)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--batch", type=int, default=B_HEADLINE)
    p.add_argument("--no-fused", action="store_true", help="skip the fused-step sub-benchmarks")
    p.add_argument("--no-cpu", action="store_true", help="skip the oracle cpu_baseline")
    p.add_argument("--cpu-seconds", type=float, default=10.0)
    p.add_argument("--workdir", default="/tmp/ngpulm_bench")
    return p.parse_args()


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)),
            int(os.environ.get("WORLD_SIZE", 1)))


def make_inputs(workdir, rank, B, nbatches, m=None):
    """LM + held-out histories (deterministic) and `nbatches` trajectory batches."""
    import numpy as np
    import synth
    f = synth.make_lm(workdir, V, ORDER, tokens=CORPUS_TOKENS, seed=1, heldout=4000, tag="bench_6gram")
    sents = synth.read_sentences(f.heldout)
    ctx = synth.sample_contexts(sents, ORDER, B * nbatches, seed=2 + 1000 * rank)
    return f, ctx


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """NVML SM-clock / throttle-reason sampler running during the measured window."""

    def __init__(self, index, pci=None, period=0.005):
        self.index, self.period, self.samples, self.ok = index, period, [], False
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = None
            if pci and pci[1] is not None:
                try:
                    bus = "%08x:%02x:%02x.0" % (pci[0], pci[1], pci[2])
                    self.h = pynvml.nvmlDeviceGetHandleByPciBusId(bus)
                except Exception:  # noqa: BLE001
                    self.h = None
            if self.h is None:
                self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # noqa: BLE001
            self.err = str(e)

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                mhz = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.samples.append((mhz, rs))
            except Exception:  # noqa: BLE001
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.ok:
            self.t.join()

    def summary(self):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"]}
        nv = self.nv
        names = {
            "gpu_idle": getattr(nv, "nvmlClocksEventReasonGpuIdle", 0x1),
            "sw_power_cap": getattr(nv, "nvmlClocksEventReasonSwPowerCap", 0x4),
            "hw_slowdown": getattr(nv, "nvmlClocksEventReasonHwSlowdown", 0x8),
            "sw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonSwThermalSlowdown", 0x20),
            "hw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonHwThermalSlowdown", 0x40),
            "hw_power_brake_slowdown": getattr(nv, "nvmlClocksEventReasonHwPowerBrakeSlowdown", 0x80),
        }
        reasons = set()
        for _, rs in self.samples:
            for n, bit in names.items():
                if rs & bit and n != "gpu_idle":
                    reasons.add(n)
        mhz = [s[0] for s in self.samples]
        return {"sm_mhz": statistics.median(mhz) if mhz else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(reasons), "samples": len(mhz)}


# ----------------------------------------------------------------------------- reference arm
def run_reference(args):
    """The oracle (CPU, as it stands) on a bounded sample of the same workload."""
    import numpy as np
    from oracle import Oracle
    rank, _, world = dist_env()
    if rank != 0:
        return
    f, ctx = make_inputs(args.workdir + "_ref", 0, args.batch, 1)
    o = Oracle(f.arpa, vocab_size=V)
    states = np.array([o.state_of(b, t) for b, t in ctx], dtype=np.int32)
    cores = len(os.sched_getaffinity(0))
    # size one step so the whole --steps/--warmup run stays within ~2 minutes
    t0 = time.perf_counter()
    o.rows(states[:cores], want64=False, nthreads=cores)
    rows_per_s = cores / max(time.perf_counter() - t0, 1e-6)
    budget = 120.0 / max(1, args.steps + args.warmup)
    rows = int(max(1, min(args.batch, rows_per_s * budget)))
    sample = states[:rows]
    for _ in range(args.warmup):
        o.rows(sample, want64=False, nthreads=cores)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        o.rows(sample, want64=False, nthreads=cores)
    el = time.perf_counter() - t0
    value = rows * V * args.steps / el
    line = {
        "impl": "reference", "metric": "LM token-queries/s (advance, B x V scores + next states)",
        "value": value, "unit": "queries/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": el / args.steps * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": workload_config(args.batch, world),
        "cpu_baseline": {"value": value, "unit": "queries/s", "cores": cores, "kind": "oracle",
                         "sample": f"{rows} of the {args.batch} trajectory rows per step (full V={V} rows)"},
        "e2e": {"value": value, "unit": "queries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def workload_config(B, world):
    return {"workload": f"advance+final: token {ORDER}-gram LM, V={V}, ~0.94M n-grams (synthetic "
                        f"Witten-Bell), B={B} trajectory states per GPU",
            "model": f"ngpulm-{ORDER}gram-V{V}", "global_batch": B * world, "B_per_gpu": B, "V": V,
            "order": ORDER, "parallelism": f"dp{world} (rows sharded, trie replicated)"}


# ----------------------------------------------------------------------------- our arm
def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2505_22857_b200 as ng
    from paper_2505_22857_b200.dist import max_over_ranks

    rank, local, world = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    B = args.batch
    props = torch.cuda.get_device_properties(dev)
    l2 = getattr(props, "L2_cache_size", 126 * 2**20) or 126 * 2**20
    out_bytes = B * V * 8
    R = max(2, math.ceil(4 * l2 / out_bytes))          # rotating sets: > 4x L2 of outputs
    f, ctx = make_inputs(f"{args.workdir}_r{rank}", rank, B, R)
    m = ng.load_arpa(f.arpa, vocab_size=V, device=local)
    states_np = np.array([m.state_of(b, t) for b, t in ctx], dtype=np.int32).reshape(R, B)
    states = torch.from_numpy(states_np).to(dev)
    scores = torch.empty((R, B, V), dtype=torch.float32, device=dev)
    nxt = torch.empty((R, B, V), dtype=torch.int32, device=dev)
    fin = torch.empty((R, B), dtype=torch.float32, device=dev)
    touched = statistics.mean(m.touched_bytes(states_np[r]) for r in range(min(R, 16)))
    stream = torch.cuda.Stream(device=dev)

    def step(k, s):
        r = k % R
        m.advance(states[r], scores[r], nxt[r], fin[r], stream=s)

    def graph_of(n):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(stream):
            for k in range(3):  # warm the capture stream
                step(k, stream)
            stream.synchronize()
            with torch.cuda.graph(g, stream=stream):
                for k in range(n):
                    step(k, stream)
        return g

    K, W = args.steps, args.warmup
    chunk = min(K, R * max(1, 512 // R))
    chunk = max(1, (chunk // R) * R) if chunk >= R else chunk
    g_main = graph_of(chunk)
    rem = K % chunk
    g_rem = graph_of(rem) if rem else None
    with torch.cuda.stream(stream):
        for k in range(max(3, W)):
            step(k, stream)
    stream.synchronize()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    sampler = ClockSampler(local, pci=(getattr(props, "pci_domain_id", 0), getattr(props, "pci_bus_id", None),
                                      getattr(props, "pci_device_id", 0)))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with sampler:
        # soak (untimed) so the clock record reflects the loaded GPU
        soak_end = time.perf_counter() + 0.5
        while time.perf_counter() < soak_end:
            with torch.cuda.stream(stream):
                g_main.replay()
            stream.synchronize()
        barrier()
        with torch.cuda.stream(stream):
            e0.record(stream)
            for _ in range(K // chunk):
                g_main.replay()
            if g_rem is not None:
                g_rem.replay()
            e1.record(stream)
        stream.synchronize()
        barrier()
    ms = max_over_ranks(e0.elapsed_time(e1), dev)  # the job's time: the slowest rank
    ms_per_step = ms / K
    value = world * B * V * K / (ms / 1e3)
    bytes_step = 8 * B * V + 4 * B + 4 * B + touched
    peak_gbs, peak_src = peaks()
    achieved = bytes_step / (ms_per_step * 1e-3) / 1e9

    # ---- e2e: the same metric through the C ABI with HOST buffers (H2D + D2H per step)
    Ke = min(K, 200)
    sh = torch.empty((B, V), dtype=torch.float32).pin_memory()
    nh = torch.empty((B, V), dtype=torch.int32).pin_memory()
    fh = torch.empty(B, dtype=torch.float32).pin_memory()
    st_h = [torch.from_numpy(states_np[r].copy()).pin_memory() for r in range(min(R, 8))]
    for r in range(3):
        m.advance_host(st_h[r % len(st_h)], sh, nh, fh, stream=stream)
    barrier()
    with torch.cuda.stream(stream):
        e0.record(stream)
        for k in range(Ke):
            m.advance_host(st_h[k % len(st_h)], sh, nh, fh, stream=stream)
        e1.record(stream)
    stream.synchronize()
    barrier()
    ms_e = max_over_ranks(e0.elapsed_time(e1), dev)
    e2e = {"value": world * B * V * Ke / (ms_e / 1e3), "unit": "queries/s",
           "h2d_bytes_per_step": 4 * B, "d2h_bytes_per_step": 8 * B * V + 4 * B, "steps": Ke}

    # per-rank results to every rank (BASELINE north_star: "NCCL is used only to gather
    # per-rank results"): outside the timed region, never part of the metric
    gather = None
    if world > 1:
        from paper_2505_22857_b200.dist import gather_rows
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        dist.barrier()
        torch.cuda.synchronize(dev)
        g0.record()
        allfin = gather_rows(fin[(K - 1) % R].contiguous(), device=dev)
        g1.record()
        torch.cuda.synchronize(dev)
        gather = {"what": "final weights of each rank's last step ([B] f32 per rank), all_gather over NCCL",
                  "rows": int(allfin.shape[0]), "us": max_over_ranks(g0.elapsed_time(g1), dev) * 1e3,
                  "timing": "CUDA events on the current stream, max over ranks"}
    variants = advance_variants(m, states, scores, nxt, fin, R, stream)
    variants.update(tiny_lm_variant(f"{args.workdir}_r{rank}", dev, stream))
    fused = {}
    if not args.no_fused:
        fused = bench_fused(m, f, dev, stream, rank)
    if world > 1:
        dist.barrier()
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    cpu = None
    if not args.no_cpu:
        cpu = cpu_baseline(f, states_np, args.cpu_seconds)

    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_advance_traffic.json")
    if os.path.exists(prof):
        with open(prof) as fh2:
            d = json.load(fh2)
        if d.get("B") == B:
            traffic = d.get("dram_bytes_per_launch")
    line = {
        "metric": "LM token-queries/s (advance, B x V scores + next states)",
        "value": value, "unit": "queries/s", "n_gpus": world, "steps": K, "warmup": W,
        "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f32", "data": "synthetic (seeded Witten-Bell token LM + held-out trajectory states)",
        "config": {**workload_config(B, world),
                   "l2": f"outputs rotate over {R} buffer sets = {R * out_bytes / 2**20:.0f} MiB > 4x L2 "
                         f"({l2 / 2**20:.0f} MiB)", "timing": "CUDA graph replays, CUDA events, max over ranks"},
        "rows_per_s": world * B * K / (ms / 1e3),
        "us_per_call": ms_per_step * 1e3,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak_gbs, "unit": "GB/s",
                     "frac": achieved / peak_gbs, "traffic": traffic, "peak_source": peak_src,
                     "algorithmic_bytes_per_launch": bytes_step,
                     "bytes_formula": "8*B*V outputs + 4*B states + 4*B finals + unique trie bytes touched"},
        "gpu_launches": K,
        "e2e": e2e,
        "clocks": sampler.summary(),
        "advance_us_per_call": variants,
        "results_gather": gather,
        "fused_step_us": fused,
        "cpu_baseline": cpu,
        "paper_context": ("PAPER.md:7,279: greedy decoding + NGPU-LM costs < 7 % over greedy decoding end to end "
                          "(RTFx, one RTX A6000, batch 32, Triton kernel); no kernel-level time is published "
                          "(BASELINE.md §1)"),
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def cpu_baseline(f, states_all, seconds):
    """The oracle as it stands, on all host cores, over a bounded sample of the
    workload's rows (the first rows of the step batches, about `seconds` s)."""
    from oracle import Oracle
    o = Oracle(f.arpa, vocab_size=V)
    cores = len(os.sched_getaffinity(0))
    flat = states_all.reshape(-1)
    o.rows(flat[:cores], want64=False, nthreads=cores)  # warm-up
    t0 = time.perf_counter()
    o.rows(flat[: 16 * cores], want64=False, nthreads=cores)
    rate = 16 * cores / max(time.perf_counter() - t0, 1e-6)
    rows = int(min(flat.size, max(cores, rate * seconds)))
    t0 = time.perf_counter()
    o.rows(flat[:rows], want64=False, nthreads=cores)
    el = time.perf_counter() - t0
    return {"value": rows * V / el, "unit": "queries/s", "cores": cores, "kind": "oracle",
            "sample": f"{rows} trajectory rows of the workload ({rows / B_HEADLINE:.1f} steps of B={B_HEADLINE}, "
                      f"full V={V} rows, score32 + next), {el:.1f} s on {cores} threads"}


def advance_variants(m, states, scores, nxt, fin, R, stream):
    """us per advance call (CUDA graph, rotating buffers) for the other shapes:
    BASELINE configs[1] (B=128) and Algorithm 1's literal chain walk."""
    import paper_2505_22857_b200 as ng
    out = {}
    for name, B, mode in (("b128_table", 128, ng.CHAIN_TABLE), ("b1024_table", states.shape[1], ng.CHAIN_TABLE),
                          ("b1024_walk", states.shape[1], ng.CHAIN_WALK)):
        m.set_chain_mode(mode)
        n = 4 * R

        def calls():
            for k in range(n):
                r = k % R
                m.advance(states[r, :B], scores[r, :B], nxt[r, :B], fin[r, :B], stream=stream)

        out[name] = _graph_time(calls, stream, None, reps=3, reset=lambda: None) * 1e3 / n
    m.set_chain_mode(ng.CHAIN_TABLE)
    return out


def tiny_lm_variant(workdir, dev, stream):
    """A keyword-biasing-sized LM (a 200-keyword LM; here a 3-gram from
    600 corpus tokens, V=1024, ~800 states): advance at B=128 with the model resident
    in shared memory (AUTO selects it up to one row per SM) vs read from global memory
    (WARP), and at B=1024 (AUTO: the global one-row-per-CTA kernel)."""
    import torch
    import paper_2505_22857_b200 as ng
    import synth
    f = synth.make_lm(workdir + "_tiny", V, 3, tokens=600, seed=11, heldout=200, tag="tiny_bias")
    m = ng.load_arpa(f.arpa, vocab_size=V, device=dev.index)
    R = 32
    out = {"tiny_lm_states": m.num_states, "tiny_resident": int(m.info.tiny_resident)}
    for name, B, kind in (("tiny_lm_b128_smem_us", 128, ng.ADVANCE_AUTO), ("tiny_lm_b128_global_us", 128, ng.ADVANCE_WARP),
                          ("tiny_lm_b1024_auto_us", 1024, ng.ADVANCE_AUTO)):
        st = torch.from_numpy(synth.uniform_states(m.num_states, B * R, seed=12).reshape(R, B)).to(dev)
        sc = torch.empty((R, B, V), dtype=torch.float32, device=dev)
        nx = torch.empty((R, B, V), dtype=torch.int32, device=dev)
        m.set_advance_kernel(kind)

        def calls():
            for k in range(4 * R):
                m.advance(st[k % R], sc[k % R], nx[k % R], want_final=False, stream=stream)
        out[name] = _graph_time(calls, stream, None, reps=3, reset=lambda: None) * 1e3 / (4 * R)
    m.set_advance_kernel(ng.ADVANCE_AUTO)
    return out


def bench_fused(m, f, dev, stream, rank):
    """Fused greedy step us (rows a7-a9): CTC config 2 shape, RNN-T and AED on the same LM."""
    import torch
    import paper_2505_22857_b200 as ng
    import synth
    out = {}
    sents = synth.read_sentences(f.heldout)
    # --- CTC: B=256, T=500, V+1 columns, lambda=0.3: one graph of 500 per-frame steps
    Bc, T = 256, 500
    x = torch.from_numpy(synth.ctc_logits(sents, Bc, T, V, seed=4 + rank)).to(dev)
    st = torch.zeros(Bc, dtype=torch.int32, device=dev)
    pv = torch.full((Bc,), -1, dtype=torch.int32, device=dev)
    frames = torch.empty((T, Bc), dtype=torch.int32, device=dev)

    def ctc_all():
        for t in range(T):
            m.fused_greedy_step(ng.CTC, x[:, t], st, prev=pv, lam=0.3, tokens_out=frames[t], stream=stream)
    ms = _graph_time(ctc_all, stream, dev, reps=5, reset=lambda: (st.zero_(), pv.fill_(-1)))
    out["ctc_b256_t500_us_per_frame"] = ms * 1e3 / T
    out["ctc_b256_t500_ms_per_utterance_batch"] = ms

    # the same utterance batch in ONE persistent launch
    fr2 = torch.empty((Bc, T), dtype=torch.int32, device=dev)
    em2 = torch.empty((Bc, T), dtype=torch.int32, device=dev)
    el2 = torch.empty(Bc, dtype=torch.int32, device=dev)

    def ctc_persistent():
        m.ctc_greedy_decode(x, st, pv, lam=0.3, frames_out=fr2, emit_out=em2, emit_len=el2, stream=stream)
    ms_p = _graph_time(ctc_persistent, stream, dev, reps=5, reset=lambda: (st.zero_(), pv.fill_(-1)))
    out["ctc_b256_t500_persistent_us_per_frame"] = ms_p * 1e3 / T
    out["ctc_b256_t500_persistent_ms_per_utterance_batch"] = ms_p
    out["ctc_b256_t500_logits_gbs_persistent"] = x.numel() * 4 / (ms_p * 1e-3) / 1e9

    def plain_all():  # plain greedy CTC frame step (argmax only, no LM): torch library op
        for t in range(T):
            frames[t].copy_(torch.argmax(x[:, t], dim=1))

    ms0 = _graph_time(plain_all, stream, dev, reps=3, reset=lambda: None)
    out["ctc_plain_argmax_torch_us_per_frame"] = ms0 * 1e3 / T
    del x
    # --- RNN-T / AED: B=512 rows, per-step logits rotating over 16 buffers
    for name, mode, gen in (("rnnt", ng.RNNT, synth.rnnt_logits), ("aed", ng.AED, synth.aed_logits)):
        Bt, NB = 512, 16
        xs = torch.from_numpy(gen(Bt, NB, V, seed=4 + rank)).to(dev)
        st = torch.from_numpy(synth.uniform_states(m.num_states, Bt, seed=3 + rank)).to(dev)
        st0 = st.clone()
        tok = torch.empty(Bt, dtype=torch.int32, device=dev)
        nsteps = 256

        def loop():
            for k in range(nsteps):
                m.fused_greedy_step(mode, xs[k % NB], st, lam=0.3, tokens_out=tok, stream=stream)

        ms = _graph_time(loop, stream, dev, reps=5, reset=lambda: st.copy_(st0))
        out[f"{name}_b{Bt}_us_per_step"] = ms * 1e3 / nsteps
        if mode == ng.RNNT:  # the same steps with the HAT internal-LM term (f3)
            ilm = torch.randn((NB, Bt, V), device=dev) - 4.0

            def loop_ilm():
                for k in range(nsteps):
                    m.fused_greedy_step_ilm(mode, xs[k % NB], st, ilm[k % NB], 0.2, lam=0.3, tokens_out=tok,
                                            stream=stream)
            ms = _graph_time(loop_ilm, stream, dev, reps=5, reset=lambda: st.copy_(st0))
            out[f"{name}_ilm_b{Bt}_us_per_step"] = ms * 1e3 / nsteps
        if mode == ng.AED:  # beam-search expansion: top-4 fused candidates per hypothesis row (f3)
            def loop_topk():
                for k in range(nsteps):
                    m.fused_topk(xs[k % NB], st, 4, lam=0.3, stream=stream)
            ms = _graph_time(loop_topk, stream, dev, reps=5, reset=lambda: None)
            out[f"aed_topk4_b{Bt}_us_per_call"] = ms * 1e3 / nsteps
    # --- label-looping transducer decode (f2): B=512 utterances of 100 frames, synthetic joint
    from paper_2505_22857_b200.decode import TransducerGreedyDecoder
    Bl = 512
    lengths = torch.full((Bl,), 100, dtype=torch.int32, device=dev)
    dec = None

    def joint(frame, u, last, outl):
        synth.joint_gpu(5 + rank, frame, u, last, outl, temperature=8.0, blank=V, blank_bias=0.75, stream=dec.stream)
    dec = TransducerGreedyDecoder(m, joint, Bl, 100, lam=0.3)
    dec(lengths)  # capture + warm-up
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    res = dec(lengths)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    out["rnnt_label_loop_b512_t100_ms"] = ms
    out["rnnt_label_loop_iterations"] = res.iterations
    out["rnnt_label_loop_us_per_iteration"] = ms * 1e3 / max(1, res.iterations)
    out["rnnt_label_loop_labels"] = int(res.emit_len.sum().item())
    return out


def _graph_time(fn, stream, dev, reps, reset):
    import torch
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(stream):
        reset()
        fn()
        stream.synchronize()
        reset()
        with torch.cuda.graph(g, stream=stream):
            fn()
    times = []
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(reps):
        with torch.cuda.stream(stream):
            reset()
            e0.record(stream)
            g.replay()
            e1.record(stream)
        stream.synchronize()
        times.append(e0.elapsed_time(e1))
    return statistics.median(times)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
