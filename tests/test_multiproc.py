"""World-size-2 gloo test of the multi-GPU host logic, on CPU:
rows are sharded contiguously over ranks, each rank answers its own rows
(here with the oracle: no GPU in this container), the verification gather
reassembles them in rank order, and the job time is the max over ranks."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2505_22857_b200.dist import gather_rows, max_over_ranks, shard_range


def test_shard_range_partitions():
    for n in (0, 1, 7, 1024, 4099):
        for world in (1, 2, 3, 8):
            spans = [shard_range(n, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [hi - lo for lo, hi in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_range(4, 2, 2)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, arpa, V, states, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import Oracle
        o = Oracle(arpa, vocab_size=V)
        lo, hi = shard_range(len(states), rank, world)
        s32, _, nx, _ = o.rows(states[lo:hi], want64=False, nthreads=1)
        rows_s = gather_rows(torch.from_numpy(s32))
        rows_n = gather_rows(torch.from_numpy(nx))
        t = max_over_ranks(float(rank + 1))
        if rank == 0:
            np.save(os.path.join(out_dir, "s.npy"), rows_s.numpy())
            np.save(os.path.join(out_dir, "n.npy"), rows_n.numpy())
            np.save(os.path.join(out_dir, "t.npy"), np.array([t]))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_sharded_equals_unsharded(small_lms, tmp_path):
    from oracle import Oracle
    f = small_lms["tri64"]
    o = Oracle(f.arpa, vocab_size=f.vocab_size)
    states = np.random.default_rng(3).integers(0, o.num_states, size=37).astype(np.int32)
    mp.spawn(_worker, args=(2, _free_port(), f.arpa, f.vocab_size, states, str(tmp_path)), nprocs=2, join=True)
    s32, _, nx, _ = o.rows(states, want64=False)
    assert np.array_equal(np.load(tmp_path / "s.npy").view(np.int32), s32.view(np.int32))
    assert np.array_equal(np.load(tmp_path / "n.npy"), nx)
    assert np.load(tmp_path / "t.npy")[0] == 2.0  # the slowest rank's time


def test_bench_launcher_world2(tmp_path):
    """`bench.py --gpus 2` without a torchrun environment launches two ranks itself
    (torch.distributed.run, 127.0.0.1); the plumbing bench.py uses at N > 1 — rank 0
    writing shared inputs while the others wait, the row partition, the rank-order
    gather and the bit-identity check, rank 0 alone printing — runs over gloo."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "LOCAL_RANK", "WORLD_SIZE")}
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--launcher-selftest",
                        "--workdir", str(tmp_path)], capture_output=True, text=True, timeout=300, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1  # rank 0 only
    d = lines[0]
    assert d["world"] == 2 and d["gpus"] == 2 and d["bit_identical"] and d["max_over_ranks"] == 2.0
