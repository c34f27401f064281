#!/usr/bin/env python
"""NGPU-LM hot-path benchmark (driver contract: one JSON line from rank 0).

Metric (BASELINE.json): LM queries/s (B x V scores + next states) and % of the
B200 HBM roofline; fused greedy step us.

Headline workload (every N, weak scaling): token 6-gram LM, V = 1024, ~0.94M
n-grams (synthetic interpolated Witten-Bell, synth/lmgen.cpp); one step = one
ngpulm_advance call with the fused final-weight gather (rows a0..a6 of
SURVEY.md §8(a)) over B = 1024 trajectory states per GPU. The K timed calls
sit inside a CUDA graph between untimed lead-in and lead-out calls, timed by
external event nodes on a side branch, so every timed call runs in the
pipelined steady state whatever K is. Rows shard across ranks with the trie
replicated and no data-path collective.

Also in the same line:
  config3  — 8-gram ~4.9M n-grams: advance B=512, RNN-T fused step B=512 (with a
             network kernel between steps), label-looping decode, overhead vs
             plain greedy;
  config4  — 10-gram ~20M n-grams, B=4096 split over the N ranks (strong
             scaling), NCCL gather of the per-rank rows checked bit-identical to
             the same batch on one GPU;
  fused    — configs[2] CTC B=256 T=500 (per-frame steps and the persistent
             decode, each vs plain greedy), RNN-T/AED steps, ILM, top-k.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""
from __future__ import annotations

import argparse
import json
import math
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

V = 1024
ORDER = 6
CORPUS_TOKENS = 430_000
B_HEADLINE = 1024
LMS = {  # BASELINE.json configs (synthetic Witten-Bell token LMs)
    "cfg1": dict(order=6, tokens=430_000, seed=1, heldout=4000, tag="bench_6gram"),
    "cfg3": dict(order=8, tokens=1_600_000, seed=5, heldout=2000, tag="cfg3_8gram"),
    "cfg4": dict(order=10, tokens=5_200_000, seed=7, heldout=2000, tag="cfg4_10gram"),
}
B_CFG3, B_CFG4 = 512, 4096


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=1000)
    p.add_argument("--warmup", type=int, default=20)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--batch", type=int, default=B_HEADLINE)
    p.add_argument("--no-fused", action="store_true", help="skip the fused-step sub-benchmarks")
    p.add_argument("--no-large", action="store_true", help="skip the configs[3]/[4] LMs")
    p.add_argument("--no-cpu", action="store_true", help="skip the oracle cpu_baseline")
    p.add_argument("--cpu-seconds", type=float, default=10.0)
    p.add_argument("--dependent", action="store_true",
                   help="headline calls without NGPULM_ADVANCE_INDEPENDENT (each waits for its predecessor)")
    p.add_argument("--workdir", default="/tmp/ngpulm_bench")
    p.add_argument("--launcher-selftest", action="store_true",
                   help="multi-rank plumbing only (gloo, no GPU): launch, shared files, shard, gather, check")
    return p.parse_args()


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)),
            int(os.environ.get("WORLD_SIZE", 1)))


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def relaunch(args) -> int:
    """`bench.py --gpus N` without a torchrun environment: run N ranks of this
    script under torch.distributed.run on this node (one process per GPU)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()), os.path.abspath(__file__),
           *sys.argv[1:]]
    return subprocess.call(cmd)


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def workload_config(B, world):
    """The headline workload; identical in both arms."""
    return {"workload": f"advance+final: token {ORDER}-gram LM, V={V}, ~0.94M n-grams (synthetic "
                        f"Witten-Bell), B={B} trajectory states per GPU",
            "model": f"ngpulm-{ORDER}gram-V{V}", "global_batch": B * world, "B_per_gpu": B, "V": V,
            "order": ORDER, "parallelism": f"dp{world} (rows sharded, trie replicated)",
            "l2": "inputs/outputs rotate over buffer sets > 4x L2 (126 MiB)",
            "timing": "K calls inside a CUDA graph between untimed lead-in/lead-out calls, external event "
                      "nodes, median over replays, max over ranks",
            "steps": "independent batches (each step its own states and output buffers)"}


# ----------------------------------------------------------------------------- shared inputs
def lm_files(workdir, key, rank, world, barrier, nglm=True):
    """The LM of LMS[key]: rank 0 generates the ARPA (cached in workdir, keyed by
    its generator arguments) and, for our arm, its NGLM binary; the other ranks
    wait, then load the binary (no re-parse)."""
    import synth
    spec = LMS[key]
    os.makedirs(workdir, exist_ok=True)
    stamp = os.path.join(workdir, spec["tag"] + ".done")
    want = json.dumps({"V": V, **spec})
    files = synth.LMFiles(arpa=os.path.join(workdir, spec["tag"] + ".arpa"), vocab_size=V, order=spec["order"],
                          heldout=os.path.join(workdir, spec["tag"] + ".heldout"))
    path = os.path.join(workdir, spec["tag"] + ".nglm")
    if rank == 0:
        if not (os.path.exists(stamp) and open(stamp).read() == want):
            files = synth.make_lm(workdir, V, spec["order"], tokens=spec["tokens"], seed=spec["seed"],
                                  heldout=spec["heldout"], tag=spec["tag"])
            if os.path.exists(path):
                os.remove(path)
            with open(stamp, "w") as fh:
                fh.write(want)
        if nglm and not os.path.exists(path):
            import paper_2505_22857_b200 as ng  # host-only parse + build, then the binary file
            ng.load_arpa(files.arpa, vocab_size=V, device=-1).save(path + ".tmp")
            os.replace(path + ".tmp", path)
    barrier()
    return files, path


def trajectory(m, files, n, seed):
    import numpy as np
    import synth
    ctx = synth.sample_contexts(synth.read_sentences(files.heldout), files.order, n, seed)
    return np.array([m.state_of(b, t) for b, t in ctx], dtype=np.int32)


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


# ----------------------------------------------------------------------------- timing helpers
class Window:
    """A CUDA graph of `lead` untimed calls, K timed calls and `tail` untimed calls,
    the K-call window bracketed by external event record nodes on a side branch
    (each recorded when the call before it completes), so the timed calls run in
    the same pipelined steady state as any long run of calls."""

    def __init__(self, call, K, stream, lead=64, tail=8):
        import torch
        self.K, self.stream = K, stream
        side = torch.cuda.Stream(device=stream.device)
        self.e0 = torch.cuda.Event(enable_timing=True, external=True)
        self.e1 = torch.cuda.Event(enable_timing=True, external=True)
        self.g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(stream):
            for k in range(3):  # warm the capture stream
                call(k)
            stream.synchronize()
            with torch.cuda.graph(self.g, stream=stream):
                for k in range(lead):
                    call(k)
                side.wait_stream(stream)
                self.e0.record(side)
                for k in range(lead, lead + K):
                    call(k)
                side.wait_stream(stream)
                self.e1.record(side)
                for k in range(lead + K, lead + K + tail):
                    call(k)
                stream.wait_stream(side)

    def replay(self) -> float:
        """One replay; ms of the K-call window."""
        import torch
        with torch.cuda.stream(self.stream):
            self.g.replay()
        self.stream.synchronize()
        return self.e0.elapsed_time(self.e1)


def window_ms(call, K, stream, reps=7, barrier=None):
    """Median over replays of the K-call window (max over ranks per replay)."""
    from paper_2505_22857_b200.dist import max_over_ranks
    w = Window(call, K, stream)
    w.replay()
    out = []
    for _ in range(reps):
        if barrier:
            barrier()
        ms = w.replay()
        out.append(max_over_ranks(ms, stream.device) if barrier else ms)
    return statistics.median(out)


def graph_ms(fn, stream, reps, reset):
    """Median ms of one replay of a graph of fn() (reset() runs before each replay, outside)."""
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


def single_call_us(call, stream, reps=15):
    """Latency of one call alone on an idle GPU: a graph of [event, call, event]
    (no predecessor to overlap with, no host launch time inside), median."""
    w = Window(call, 1, stream, lead=0, tail=0)
    w.replay()
    return statistics.median(w.replay() for _ in range(reps)) * 1e3


# ----------------------------------------------------------------------------- reference arm
def run_reference(args):
    """The oracle (CPU, as it stands) on a bounded sample of the same workload."""
    from oracle import Oracle
    rank, _, world = dist_env()
    if rank != 0:
        return
    files, _ = lm_files(args.workdir, "cfg1", 0, 1, lambda: None, nglm=False)
    o = Oracle(files.arpa, vocab_size=V)
    states = trajectory(o, files, args.batch, seed=2)
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

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    B = args.batch
    props = torch.cuda.get_device_properties(dev)
    l2 = getattr(props, "L2_cache_size", 126 * 2**20) or 126 * 2**20
    out_bytes = B * V * 8
    R = max(2, math.ceil(4 * l2 / out_bytes))          # rotating sets: > 4x L2 of outputs
    files, nglm = lm_files(args.workdir, "cfg1", rank, world, barrier)
    m = ng.load_binary(nglm, device=local)
    states_np = trajectory(m, files, B * R, seed=2 + 1000 * rank).reshape(R, B)
    states = torch.from_numpy(states_np).to(dev)
    scores = torch.empty((R, B, V), dtype=torch.float32, device=dev)
    nxt = torch.empty((R, B, V), dtype=torch.int32, device=dev)
    fin = torch.empty((R, B), dtype=torch.float32, device=dev)
    touched = statistics.mean(m.touched_bytes(states_np[r]) for r in range(min(R, 16)))
    stream = torch.cuda.Stream(device=dev)

    # one step = one ngpulm_advance call over its own batch into its own buffer set: the
    # steps are independent (NGPULM_ADVANCE_INDEPENDENT), unless --dependent
    indep = not args.dependent

    def step(k):
        r = k % R
        m.advance(states[r], scores[r], nxt[r], fin[r], stream=stream, independent=indep)

    K, W = args.steps, args.warmup
    with torch.cuda.stream(stream):
        for k in range(max(3, W)):  # W untimed warm-up steps
            step(k)
    stream.synchronize()
    win = Window(step, K, stream)
    win.replay()
    sampler = ClockSampler(local, pci=(getattr(props, "pci_domain_id", 0), getattr(props, "pci_bus_id", None),
                                      getattr(props, "pci_device_id", 0)))
    times = []
    with sampler:
        t_end = time.perf_counter() + 0.5  # >= 0.5 s of timed replays: the clock record sees the loaded GPU
        while time.perf_counter() < t_end or len(times) < 7:
            barrier()
            times.append(max_over_ranks(win.replay(), dev))
            barrier()
    ms = statistics.median(times)
    ms_per_step = ms / K
    value = world * B * V * K / (ms / 1e3)
    compulsory = 8 * B * V + 4 * B + 4 * B  # outputs + states + finals (HBM-compulsory)
    peak_gbs, peak_src = peaks()
    achieved = compulsory / (ms_per_step * 1e-3) / 1e9
    lat = {"b1024_us": single_call_us(step, stream)}

    e2e = e2e_pipelined(m, states_np, B, dev, world)
    variants = advance_variants(m, states, scores, nxt, fin, R, stream)
    variants.update(tiny_lm_variant(f"{args.workdir}_r{rank}", dev, stream))
    variants["single_call_latency_us"] = lat
    large = {}
    if not args.no_large:
        large["config4"] = bench_config4(args, rank, local, world, dev, stream, barrier)
        large["config3"] = bench_config3(args, rank, world, dev, stream, barrier, args.no_fused)
    fused = {}
    if not args.no_fused:
        fused = bench_fused(m, files, dev, stream, rank)
    barrier()
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    cpu = None if args.no_cpu else cpu_baseline(files, states_np, args.cpu_seconds)
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
        "config": workload_config(B, world),
        "rows_per_s": world * B * K / (ms / 1e3),
        "us_per_call": ms_per_step * 1e3,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak_gbs, "unit": "GB/s",
                     "frac": achieved / peak_gbs, "traffic": traffic, "peak_source": peak_src,
                     "algorithmic_bytes_per_launch": compulsory,
                     "bytes_formula": "8*B*V outputs + 4*B states + 4*B finals (HBM-compulsory; the trie is "
                                      "L2-resident, its unique bytes are reported apart)",
                     "trie_unique_bytes_per_launch": touched,
                     "call_mode": "independent (NGPULM_ADVANCE_INDEPENDENT)" if indep else "dependent"},
        "roofline_dependent_calls": {
            "us_per_call": variants.get("b1024_table_dependent"),
            "frac": (compulsory / (variants["b1024_table_dependent"] * 1e-6) / 1e9 / peak_gbs
                     if variants.get("b1024_table_dependent") else None),
            "what": "the same step through plain ngpulm_advance: each call waits for its predecessor to "
                    "complete before storing (the regime of a decode loop whose next states come from the "
                    "previous step)"},
        "gpu_launches": K,
        "e2e": e2e,
        "clocks": sampler.summary(),
        "timed_replays": len(times),
        "advance_us_per_call": variants,
        "fused_step_us": fused,
        **large,
        "cpu_baseline": cpu,
        "paper_context": ("PAPER.md:7,279: greedy decoding + NGPU-LM costs < 7 % over greedy decoding end to end "
                          "(RTFx, one RTX A6000, batch 32, Triton kernel); no kernel-level time is published "
                          "(BASELINE.md §1)"),
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def e2e_pipelined(m, states_np, B, dev, world, steps=64):
    """The same metric end to end through the public API with HOST buffers: every
    step copies its states in from pinned memory, runs ngpulm_advance and copies
    the full [B,V] scores + next rows and finals back to pinned memory; two
    streams alternate so one step's copies overlap the other's (PCIe-bound)."""
    import torch
    from paper_2505_22857_b200.dist import max_over_ranks
    R = states_np.shape[0]
    nslot = 2
    st_h = [torch.from_numpy(states_np[r].copy()).pin_memory() for r in range(min(R, 8))]
    sh = [torch.empty((B, V), dtype=torch.float32).pin_memory() for _ in range(nslot)]
    nh = [torch.empty((B, V), dtype=torch.int32).pin_memory() for _ in range(nslot)]
    fh = [torch.empty(B, dtype=torch.float32).pin_memory() for _ in range(nslot)]
    sd = [torch.empty(B, dtype=torch.int32, device=dev) for _ in range(nslot)]
    scd = [torch.empty((B, V), dtype=torch.float32, device=dev) for _ in range(nslot)]
    nxd = [torch.empty((B, V), dtype=torch.int32, device=dev) for _ in range(nslot)]
    fd = [torch.empty(B, dtype=torch.float32, device=dev) for _ in range(nslot)]
    streams = [torch.cuda.Stream(device=dev) for _ in range(nslot)]

    def one(k):
        i = k % nslot
        s = streams[i]
        with torch.cuda.stream(s):
            sd[i].copy_(st_h[k % len(st_h)], non_blocking=True)
            m.advance(sd[i], scd[i], nxd[i], fd[i], stream=s)
            sh[i].copy_(scd[i], non_blocking=True)
            nh[i].copy_(nxd[i], non_blocking=True)
            fh[i].copy_(fd[i], non_blocking=True)

    for k in range(4):
        one(k)
    torch.cuda.synchronize(dev)
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    cur = torch.cuda.current_stream(dev)
    t0.record(cur)
    for s in streams:
        s.wait_stream(cur)
    for k in range(steps):
        one(k)
    for s in streams:
        cur.wait_stream(s)
    t1.record(cur)
    torch.cuda.synchronize(dev)
    ms = max_over_ranks(t0.elapsed_time(t1), dev)
    return {"value": world * B * V * steps / (ms / 1e3), "unit": "queries/s",
            "h2d_bytes_per_step": 4 * B, "d2h_bytes_per_step": 8 * B * V + 4 * B, "steps": steps,
            "how": "pinned host buffers, H2D states + ngpulm_advance + D2H scores/next/finals every step, "
                   "2 streams alternating (PCIe-bound: 8 MiB of results per step)"}


def cpu_baseline(files, states_all, seconds):
    """The oracle as it stands, on all host cores, over a bounded sample of the
    workload's rows (the first rows of the step batches, about `seconds` s)."""
    from oracle import Oracle
    o = Oracle(files.arpa, vocab_size=V)
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
    """us per advance call in the steady state (Window) for the other shapes:
    BASELINE configs[1] (B=128), B=4096 and Algorithm 1's literal chain walk; each
    in both call modes — independent (NGPULM_ADVANCE_INDEPENDENT: the calls' batches
    and buffers are independent, rows stored before the PDL wait) and dependent
    (plain ngpulm_advance: every call waits for its predecessor before storing)."""
    import paper_2505_22857_b200 as ng
    out = {}
    Bh = states.shape[1]
    for name, Bv, mode, ind in (("b128_table", 128, ng.CHAIN_TABLE, True), ("b1024_table", Bh, ng.CHAIN_TABLE, True),
                                ("b1024_walk", Bh, ng.CHAIN_WALK, True),
                                ("b128_table_dependent", 128, ng.CHAIN_TABLE, False),
                                ("b1024_table_dependent", Bh, ng.CHAIN_TABLE, False)):
        m.set_chain_mode(mode)

        def call(k):
            r = k % R
            m.advance(states[r, :Bv], scores[r, :Bv], nxt[r, :Bv], fin[r, :Bv], stream=stream, independent=ind)
        out[name] = window_ms(call, 256, stream) * 1e3 / 256
    m.set_chain_mode(ng.CHAIN_TABLE)
    # B = 4096: four of the rotating batches side by side
    import torch
    R4 = R // 4
    st4 = states[: 4 * R4].reshape(R4, 4 * Bh)
    sc4 = scores[: 4 * R4].reshape(R4, 4 * Bh, -1)
    nx4 = nxt[: 4 * R4].reshape(R4, 4 * Bh, -1)
    fi4 = fin[: 4 * R4].reshape(R4, 4 * Bh)

    for ind, name in ((True, "b4096_table"), (False, "b4096_table_dependent")):
        def call4(k):
            r = k % R4
            m.advance(st4[r], sc4[r], nx4[r], fi4[r], stream=stream, independent=ind)
        out[name] = window_ms(call4, 128, stream) * 1e3 / 128
    del torch
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

        def call(k):
            m.advance(st[k % R], sc[k % R], nx[k % R], want_final=False, stream=stream)
        out[name] = window_ms(call, 128, stream) * 1e3 / 128
    m.set_advance_kernel(ng.ADVANCE_AUTO)
    # the decode kernels with the biasing LM (f4 tiny path vs the same model read from global memory):
    # configs[2]-shaped CTC (B=256, T=500): per-frame fused steps and the persistent decode
    Bc, T = 256, 500
    x = torch.from_numpy(synth.ctc_logits(synth.read_sentences(f.heldout), Bc, T, V, seed=4)).to(dev)
    stc = torch.zeros(Bc, dtype=torch.int32, device=dev)
    pv = torch.full((Bc,), -1, dtype=torch.int32, device=dev)
    frames = torch.empty((T, Bc), dtype=torch.int32, device=dev)
    reset = lambda: (stc.zero_(), pv.fill_(-1))  # noqa: E731
    for kind, tag in ((ng.ADVANCE_AUTO, "smem"), (ng.ADVANCE_WARP, "global")):
        m.set_advance_kernel(kind)

        def ctc_all():
            for t in range(T):
                m.fused_greedy_step(ng.CTC, x[:, t], stc, prev=pv, lam=0.3, tokens_out=frames[t], stream=stream)
        out[f"tiny_lm_ctc_b256_fused_us_per_frame_{tag}"] = graph_ms(ctc_all, stream, 5, reset) * 1e3 / T

        def ctc_persistent():
            m.ctc_greedy_decode(x, stc, pv, lam=0.3, stream=stream)
        out[f"tiny_lm_ctc_b256_t500_persistent_ms_{tag}"] = graph_ms(ctc_persistent, stream, 5, reset)
    m.set_advance_kernel(ng.ADVANCE_AUTO)
    return out


# ----------------------------------------------------------------------------- configs[3] and [4]
def bench_config4(args, rank, local, world, dev, stream, barrier):
    """configs[4]: 10-gram ~20M n-grams, B=4096 split over the N ranks (strong
    scaling: 4096/N rows per GPU), trie replicated (NGLM reload on every rank);
    after the timed region the per-rank rows are all-gathered over NCCL and
    checked bit-identical to the whole batch answered on one GPU."""
    import numpy as np
    import torch
    import paper_2505_22857_b200 as ng
    from paper_2505_22857_b200.dist import gather_rows, max_over_ranks, shard_range
    t0 = time.perf_counter()
    files, nglm = lm_files(args.workdir, "cfg4", rank, world, barrier)
    m = ng.load_binary(nglm, device=local)
    load_s = time.perf_counter() - t0
    Bg = B_CFG4
    lo, hi = shard_range(Bg, rank, world)
    Bl = hi - lo
    R = max(2, math.ceil(4 * 126 * 2**20 / (Bl * V * 8)))
    allst = trajectory(m, files, Bg * R, seed=31).reshape(R, Bg)  # same on every rank
    st = torch.from_numpy(np.ascontiguousarray(allst[:, lo:hi])).to(dev)
    sc = torch.empty((R, Bl, V), dtype=torch.float32, device=dev)
    nx = torch.empty((R, Bl, V), dtype=torch.int32, device=dev)
    fi = torch.empty((R, Bl), dtype=torch.float32, device=dev)

    def call(k, ind=True):  # independent batches (NGPULM_ADVANCE_INDEPENDENT), as the headline
        r = k % R
        m.advance(st[r], sc[r], nx[r], fi[r], stream=stream, independent=ind)
    K = 128
    ms = window_ms(call, K, stream, reps=7, barrier=barrier)
    us = ms * 1e3 / K
    us_dep = window_ms(lambda k: call(k, False), K, stream, reps=7, barrier=barrier) * 1e3 / K
    peak_gbs, _ = peaks()
    comp = 8 * Bl * V + 8 * Bl
    touched = statistics.mean(m.touched_bytes(allst[r, lo:hi]) for r in range(min(R, 4)))
    out = {"workload": f"advance+final: token 10-gram LM, V={V}, {m.info.num_arcs} arcs / {m.num_states} states "
                       f"(~20M n-grams), B={Bg} global = {Bl} rows on each of {world} GPU(s)",
           "us_per_call": us, "queries_per_s": Bg * V / (us * 1e-6), "rows_per_gpu": Bl,
           "roofline": {"bound": "hbm", "achieved": comp / (us * 1e-6) / 1e9, "peak": peak_gbs, "unit": "GB/s",
                        "frac": comp / (us * 1e-6) / 1e9 / peak_gbs,
                        "algorithmic_bytes_per_launch": comp,
                        "trie_unique_bytes_per_launch": touched,
                        "frac_incl_trie": (comp + touched) / (us * 1e-6) / 1e9 / peak_gbs},
           "us_per_call_dependent": us_dep,
           "frac_dependent": comp / (us_dep * 1e-6) / 1e9 / peak_gbs,
           "model_bytes_per_gpu": m.info.device_bytes, "load_s_rank0": load_s,
           "single_call_latency_us": single_call_us(call, stream)}
    # the NCCL gather of per-rank results (outside the timed region) and the check
    call(0)
    torch.cuda.synchronize(dev)
    barrier()
    g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    g0.record()
    gs = gather_rows(sc[0], device=dev)
    gn = gather_rows(nx[0], device=dev)
    gf = gather_rows(fi[0], device=dev)
    g1.record()
    torch.cuda.synchronize(dev)
    out["gather"] = {"what": f"scores+next+finals of batch 0 from every rank ({Bg} rows, "
                             f"{(8 * V + 4) * Bg / 2**20:.1f} MiB) all-gathered over NCCL",
                     "us": max_over_ranks(g0.elapsed_time(g1), dev) * 1e3}
    if rank == 0:  # the same batch answered on one GPU, bit for bit
        one = torch.from_numpy(allst[0].copy()).to(dev)
        s1, n1, f1 = m.advance(one)
        torch.cuda.synchronize(dev)
        same = (torch.equal(s1.view(torch.int32), gs.view(torch.int32)) and torch.equal(n1, gn)
                and torch.equal(f1.view(torch.int32), gf.view(torch.int32)))
        out["gather"]["bit_identical_to_one_gpu"] = bool(same)
        out["check"] = int(m.check())
    barrier()
    return out


def network_kernel(src, dst):
    """Stand-in for the network step between two decoder steps (the joint /
    decoder producing the next logits): one elementwise kernel, launched
    without programmatic dependent launch, as a framework's kernel would be."""
    import torch
    torch.mul(src, 1.0, out=dst)


def bench_config3(args, rank, world, dev, stream, barrier, no_fused):
    """configs[3]: 8-gram ~4.9M n-grams; advance B=512 and the RNN-T fused step
    B=512, back to back and with a network kernel between steps; the plain
    greedy step (lambda = 0) for the paper's overhead figure; label-looping decode."""
    import torch
    import paper_2505_22857_b200 as ng
    import synth
    files, nglm = lm_files(args.workdir, "cfg3", rank, world, barrier)
    m = ng.load_binary(nglm, device=dev.index)
    B = B_CFG3
    R = 64
    stn = trajectory(m, files, B * R, seed=21 + rank).reshape(R, B)
    st = torch.from_numpy(stn).to(dev)
    sc = torch.empty((R, B, V), dtype=torch.float32, device=dev)
    nx = torch.empty((R, B, V), dtype=torch.int32, device=dev)
    fi = torch.empty((R, B), dtype=torch.float32, device=dev)

    def adv(k, ind=True):  # independent batches (NGPULM_ADVANCE_INDEPENDENT), as the headline
        r = k % R
        m.advance(st[r], sc[r], nx[r], fi[r], stream=stream, independent=ind)
    us = window_ms(adv, 256, stream) * 1e3 / 256
    us_dep = window_ms(lambda k: adv(k, False), 256, stream) * 1e3 / 256
    peak_gbs, _ = peaks()
    comp = 8 * B * V + 8 * B
    touched = statistics.mean(m.touched_bytes(stn[r]) for r in range(4))
    out = {"workload": f"token 8-gram LM, V={V}, {m.info.num_arcs} arcs / {m.num_states} states (~4.9M n-grams), "
                       f"B={B}",
           "advance_us_per_call": us,
           "advance_us_per_call_dependent": us_dep,
           "advance_roofline": {"bound": "hbm", "achieved": comp / (us * 1e-6) / 1e9, "peak": peak_gbs,
                                "unit": "GB/s", "frac": comp / (us * 1e-6) / 1e9 / peak_gbs,
                                "algorithmic_bytes_per_launch": comp, "trie_unique_bytes_per_launch": touched},
           "advance_single_call_latency_us": single_call_us(adv, stream)}
    if no_fused:
        return out
    out.update(transducer_steps(m, stn[0], dev, stream, rank, "rnnt"))
    out.update(label_loop(m, dev, stream, rank))
    return out


def transducer_steps(m, states0, dev, stream, rank, tag, nsteps=256):
    """RNN-T fused steps at B rows: back to back, and each after a network kernel
    that writes the step's logits (per-step time = loop - network-only loop);
    the same for the plain greedy step (lambda = 0: no LM row)."""
    import torch
    import paper_2505_22857_b200 as ng
    import synth
    B, NB = states0.size, 16
    xs = torch.from_numpy(synth.rnnt_logits(B, NB, V, seed=4 + rank)).to(dev)
    buf = torch.empty_like(xs[0])
    st0 = torch.from_numpy(states0.copy()).to(dev)
    st = st0.clone()
    tok = torch.empty(B, dtype=torch.int32, device=dev)
    out = {}
    for lam, name in ((0.3, "fused"), (0.0, "plain")):
        sv = st if name == "fused" else None  # plain greedy: no LM state (the C ABI's states == NULL path)

        def b2b():
            for k in range(nsteps):
                m.fused_greedy_step(ng.RNNT, xs[k % NB], sv, lam=lam, tokens_out=tok, stream=stream)

        def with_net(ready=False):
            for k in range(nsteps):
                network_kernel(xs[k % NB], buf)
                m.fused_greedy_step(ng.RNNT, buf, sv, lam=lam, tokens_out=tok, stream=stream, inputs_ready=ready)
        reset = lambda: st.copy_(st0)  # noqa: E731
        out[f"{tag}_b{B}_{name}_us_per_step_back_to_back"] = graph_ms(b2b, stream, 5, reset) * 1e3 / nsteps
        out[f"{tag}_b{B}_{name}_us_per_step_after_network"] = graph_ms(with_net, stream, 5, reset) * 1e3 / nsteps
        # NGPULM_STEP_INPUTS_READY: the network kernel is a plain launch, so the step's inputs are final
        out[f"{tag}_b{B}_{name}_us_per_step_after_network_inputs_ready"] = graph_ms(
            lambda: with_net(True), stream, 5, reset) * 1e3 / nsteps
    def net_only():
        for k in range(nsteps):
            network_kernel(xs[k % NB], buf)
    net = graph_ms(net_only, stream, 5, lambda: None) * 1e3 / nsteps
    out[f"{tag}_b{B}_network_kernel_us"] = net
    f_ = out[f"{tag}_b{B}_fused_us_per_step_after_network"]
    p_ = out[f"{tag}_b{B}_plain_us_per_step_after_network"]
    out[f"{tag}_b{B}_fused_step_us_in_loop"] = f_ - net
    out[f"{tag}_b{B}_plain_step_us_in_loop"] = p_ - net
    out[f"{tag}_b{B}_lm_overhead_vs_plain_loop"] = f_ / p_ - 1.0
    fr_ = out[f"{tag}_b{B}_fused_us_per_step_after_network_inputs_ready"]
    pr_ = out[f"{tag}_b{B}_plain_us_per_step_after_network_inputs_ready"]
    out[f"{tag}_b{B}_fused_step_us_in_loop_inputs_ready"] = fr_ - net
    out[f"{tag}_b{B}_plain_step_us_in_loop_inputs_ready"] = pr_ - net
    out[f"{tag}_b{B}_lm_overhead_vs_plain_loop_inputs_ready"] = fr_ / pr_ - 1.0
    return out


def label_loop(m, dev, stream, rank):
    """Label-looping transducer decode (f2), B=512 utterances of 100 frames with the
    synthetic joint: with the LM (lambda=0.3) and plain greedy (lambda=0)."""
    import torch
    import synth
    from paper_2505_22857_b200.decode import TransducerGreedyDecoder
    Bl = 512
    lengths = torch.full((Bl,), 100, dtype=torch.int32, device=dev)
    out = {}
    for lam, name in ((0.3, "fused"), (0.0, "plain")):
        dec = None

        def joint(frame, u, last, outl):
            synth.joint_gpu(5 + rank, frame, u, last, outl, temperature=8.0, blank=V, blank_bias=0.75,
                            stream=dec.stream)
        # the synthetic joint is a plain launch: NGPULM_STEP_INPUTS_READY holds
        dec = TransducerGreedyDecoder(m, joint, Bl, 100, lam=lam, use_lm=name == "fused", joint_plain_launch=True)
        dec(lengths)  # capture + warm-up
        ts = []
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            res = dec(lengths)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        out[f"rnnt_label_loop_b512_t100_{name}_ms"] = statistics.median(ts)
        out[f"rnnt_label_loop_{name}_iterations"] = res.iterations
        out[f"rnnt_label_loop_{name}_labels"] = int(res.emit_len.sum().item())
    out["rnnt_label_loop_lm_overhead"] = (out["rnnt_label_loop_b512_t100_fused_ms"]
                                          / out["rnnt_label_loop_b512_t100_plain_ms"] - 1.0)
    return out


def bench_fused(m, files, dev, stream, rank):
    """Fused greedy step us (rows a7-a9): configs[2] CTC (per-frame and persistent,
    each vs plain greedy), RNN-T / AED steps on the 6-gram, ILM, top-k."""
    import torch
    import paper_2505_22857_b200 as ng
    import synth
    out = {}
    sents = synth.read_sentences(files.heldout)
    # --- CTC: B=256, T=500, V+1 columns, lambda=0.3: one graph of 500 per-frame steps
    Bc, T = 256, 500
    x = torch.from_numpy(synth.ctc_logits(sents, Bc, T, V, seed=4 + rank)).to(dev)
    st = torch.zeros(Bc, dtype=torch.int32, device=dev)
    pv = torch.full((Bc,), -1, dtype=torch.int32, device=dev)
    frames = torch.empty((T, Bc), dtype=torch.int32, device=dev)
    reset = lambda: (st.zero_(), pv.fill_(-1))  # noqa: E731
    for lam, name in ((0.3, "fused"), (0.0, "plain")):
        sv = st if name == "fused" else None  # plain greedy: no LM state

        for ready in (False, True):  # logits_ready: NGPULM_STEP_LOGITS_READY (the encoder output precedes the loop)
            def ctc_all():
                for t in range(T):
                    m.fused_greedy_step(ng.CTC, x[:, t], sv, prev=pv, lam=lam, tokens_out=frames[t], stream=stream,
                                        logits_ready=ready)
            ms = graph_ms(ctc_all, stream, 5, reset)
            out[f"ctc_b256_t500_{name}{'_logits_ready' if ready else ''}_us_per_frame"] = ms * 1e3 / T
    out["ctc_per_frame_lm_overhead"] = out["ctc_b256_t500_fused_us_per_frame"] / out["ctc_b256_t500_plain_us_per_frame"] - 1
    out["ctc_per_frame_lm_overhead_logits_ready"] = (out["ctc_b256_t500_fused_logits_ready_us_per_frame"]
                                                     / out["ctc_b256_t500_plain_logits_ready_us_per_frame"] - 1)

    # the same utterance batch in ONE persistent launch
    fr2 = torch.empty((Bc, T), dtype=torch.int32, device=dev)
    em2 = torch.empty((Bc, T), dtype=torch.int32, device=dev)
    el2 = torch.empty(Bc, dtype=torch.int32, device=dev)
    for lam, name in ((0.3, "fused"), (0.0, "plain")):
        sv = st if name == "fused" else None  # plain greedy: no LM state

        def ctc_persistent():
            m.ctc_greedy_decode(x, sv, pv, lam=lam, frames_out=fr2, emit_out=em2, emit_len=el2, stream=stream)
        ms_p = graph_ms(ctc_persistent, stream, 5, reset)
        out[f"ctc_b256_t500_persistent_{name}_ms"] = ms_p
        out[f"ctc_b256_t500_persistent_{name}_us_per_frame"] = ms_p * 1e3 / T  # per frame of the whole batch
        out[f"ctc_b256_t500_persistent_{name}_logits_gbs"] = x.numel() * 4 / (ms_p * 1e-3) / 1e9
    peak_gbs, _ = peaks()
    out["ctc_persistent_roofline"] = {
        "bound": "hbm", "achieved": out["ctc_b256_t500_persistent_fused_logits_gbs"], "peak": peak_gbs,
        "unit": "GB/s", "frac": out["ctc_b256_t500_persistent_fused_logits_gbs"] / peak_gbs,
        "algorithmic_bytes_per_launch": x.numel() * 4, "bytes_formula": "4*B*T*(V+1) logits (read once)"}
    out["ctc_persistent_lm_overhead"] = (out["ctc_b256_t500_persistent_fused_ms"]
                                         / out["ctc_b256_t500_persistent_plain_ms"] - 1)
    del x
    # --- RNN-T / AED on the 6-gram, B=512, per-step logits rotating over 16 buffers
    stu = synth.uniform_states(m.num_states, 512, seed=3 + rank)
    out.update(transducer_steps(m, stu, dev, stream, rank, "rnnt6"))
    Bt, NB, nsteps = 512, 16, 256
    xs = torch.from_numpy(synth.aed_logits(Bt, NB, V, seed=4 + rank)).to(dev)
    st = torch.from_numpy(stu).to(dev)
    st0 = st.clone()
    tok = torch.empty(Bt, dtype=torch.int32, device=dev)

    def aed():
        for k in range(nsteps):
            m.fused_greedy_step(ng.AED, xs[k % NB], st, lam=0.3, tokens_out=tok, stream=stream)
    out[f"aed_b{Bt}_us_per_step"] = graph_ms(aed, stream, 5, lambda: st.copy_(st0)) * 1e3 / nsteps
    xr = torch.from_numpy(synth.rnnt_logits(Bt, NB, V, seed=4 + rank)).to(dev)
    ilm = torch.randn((NB, Bt, V), device=dev) - 4.0

    def rnnt_ilm():
        for k in range(nsteps):
            m.fused_greedy_step_ilm(ng.RNNT, xr[k % NB], st, ilm[k % NB], 0.2, lam=0.3, tokens_out=tok,
                                    stream=stream)
    out[f"rnnt_ilm_b{Bt}_us_per_step"] = graph_ms(rnnt_ilm, stream, 5, lambda: st.copy_(st0)) * 1e3 / nsteps

    def topk():  # beam-search expansion: top-4 fused candidates per hypothesis row (f3)
        for k in range(nsteps):
            m.fused_topk(xs[k % NB], st, 4, lam=0.3, stream=stream)
    out[f"aed_topk4_b{Bt}_us_per_call"] = graph_ms(topk, stream, 5, lambda: None) * 1e3 / nsteps
    return out


# ----------------------------------------------------------------------------- launcher self-test
def launcher_selftest(args):
    """Multi-rank plumbing without a GPU (gloo): the rank/world environment,
    rank 0 writing shared files while the others wait, the row partition, the
    gather in rank order and the bit-identity check; rank 0 prints one line."""
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_2505_22857_b200.dist import gather_rows, max_over_ranks, shard_range
    rank, _, world = dist_env()
    if world > 1:
        dist.init_process_group("gloo")
    os.makedirs(args.workdir, exist_ok=True)
    path = os.path.join(args.workdir, "selftest_rows.npy")
    rows = np.random.default_rng(7).integers(0, 1 << 30, size=(37, 5)).astype(np.int32)
    if rank == 0:
        np.save(path, rows)
    if world > 1:
        dist.barrier()
    allr = np.load(path)
    lo, hi = shard_range(len(allr), rank, world)
    got = gather_rows(torch.from_numpy(allr[lo:hi].copy()))
    t = max_over_ranks(float(rank + 1))
    if rank == 0:
        print(json.dumps({"selftest": "launcher", "world": world, "gpus": args.gpus,
                          "bit_identical": bool(np.array_equal(got.numpy(), rows)), "max_over_ranks": t}),
              flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(relaunch(args))
    _, _, world = dist_env()
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.launcher_selftest:
        launcher_selftest(args)
    elif args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
