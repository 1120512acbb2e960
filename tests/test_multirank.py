"""CPU, world_size 2 over gloo: the multi-rank plumbing bench.py uses for
N GPUs (one process per GPU, output-row slabs, no data exchange, max-over-ranks
timing) and the slab partition rule of the C ABI."""
from __future__ import annotations

import os
import socket

import pytest
import torch.multiprocessing as mp

from conftest import ROOT


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank: int, world: int, port: int, n: int, q) -> None:
    import sys
    sys.path.insert(0, str(ROOT))
    os.environ.update({"RANK": str(rank), "LOCAL_RANK": str(rank), "WORLD_SIZE": str(world),
                       "MASTER_ADDR": "127.0.0.1", "MASTER_PORT": str(port)})
    import torch
    import torch.distributed as dist
    import bench
    d = bench.Dist()  # gloo: no CUDA in this container
    assert d.pg is not None and dist.get_backend() == "gloo"
    lo, hi = bench.shard_rows(n, d.rank, d.world, 256)
    spans = [None] * world
    dist.all_gather_object(spans, (lo, hi))
    t = d.max(float(rank + 1) * 1.5)  # max-over-ranks of a per-rank time
    d.barrier()
    if rank == 0:
        q.put((spans, t))
    d.close()


@pytest.mark.parametrize("world,n", [(2, 131072), (2, 1000), (2, 256)])
def test_ranks_partition_rows_and_reduce_time(world, n):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    mp.start_processes(_worker, args=(world, port, n, q), nprocs=world, join=True, start_method="spawn")
    spans, t = q.get(timeout=60)
    assert t == 1.5 * world
    covered = []
    for lo, hi in spans:
        assert lo % 256 == 0 and lo <= hi
        covered.extend(range(lo, hi))
    assert covered == list(range(n))  # disjoint, contiguous, complete: no exchange needed


def test_slab_rule_matches_for_every_part_count():
    import paper_1909_01554_b200 as bmm
    for m in (0, 1, 63, 64, 65, 1000, 131072, 1 << 20):
        for parts in (1, 2, 3, 4, 7, 8):
            prev = 0
            for i in range(parts):
                lo, hi = bmm.slab_rows(m, parts, i, 64)
                assert lo == prev and (lo % 64 == 0 or lo == m)
                prev = hi
            assert prev == m
    with pytest.raises(ValueError):
        bmm.slab_rows(10, 2, 2, 64)


@pytest.mark.gpu
def test_bench_two_ranks_share_one_gpu():
    """bench.py under torchrun with two ranks (gloo for the rank plumbing, so both may
    share the box's one GPU): each rank multiplies its output-row slab, rank 0 prints
    one line with the aggregate over both slabs and the max-over-ranks time."""
    import json
    import os
    import subprocess
    import sys
    env = dict(os.environ, BMM_DIST_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29531", "bench.py", "--gpus", "2", "--workload",
           "c1-gf2-cubic-8192", "--steps", "3", "--warmup", "3", "--no-cpu-baseline"]
    r = subprocess.run(cmd, cwd=str(ROOT), env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["rows_per_rank"] == 4096 and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 4096 * 128 * 8 + 8192 * 128 * 8


@pytest.mark.gpu
def test_alt_tile_partition_two_ranks():
    """The multi-GPU fast product (4 x 4 output tiles, each the XOR of 4 alt-basis block
    products, round robin over ranks): two ranks sharing one GPU, every tile of rank 0
    checked against the tensor-core cubic product."""
    import json
    import os
    import subprocess
    import sys
    env = dict(os.environ, BMM_DIST_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29533", "bench.py", "--gpus", "2", "--workload",
           "c4s-gf2-altsi-16384", "--leaf-log2", "9", "--steps", "3", "--warmup", "3", "--check"]
    r = subprocess.run(cmd, cwd=str(ROOT), env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    d = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][0])
    assert d["n_gpus"] == 2 and d["config"]["tiles_per_rank0"] == 8 and d["tiles_checked_rank0"] == 8
    assert d["value"] > 0 and d["gpu_launches"] > 0
