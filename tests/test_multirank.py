"""CPU, world_size 2 over gloo: the multi-rank plumbing bench.py uses for
N GPUs (one process per GPU, output-row slabs, max-over-ranks timing), the slab
partition rule of the C ABI, and the fast product's one exchange step (all-to-all
of row slabs + XOR fold of the partial products)."""
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


def _exchange_worker(rank: int, world: int, port: int, q) -> None:
    import sys
    sys.path.insert(0, str(ROOT))
    os.environ.update({"RANK": str(rank), "LOCAL_RANK": str(rank), "WORLD_SIZE": str(world),
                       "MASTER_ADDR": "127.0.0.1", "MASTER_PORT": str(port)})
    import torch
    import bench
    d = bench.Dist()
    n, w = 1280, 3
    slabs = [bench.shard_rows(n, r, world, 256) for r in range(world)]
    g = torch.Generator().manual_seed(100 + rank)
    P = torch.randint(-2**62, 2**62, (n, w), dtype=torch.int64, generator=g)  # this rank's partial product
    r0, r1 = slabs[rank]
    R = torch.empty((world * (r1 - r0), w), dtype=torch.int64)

    def fold(k):
        R[: r1 - r0] ^= R[k * (r1 - r0):(k + 1) * (r1 - r0)]
    bench.slab_exchange_xor(P, R, slabs, rank, world, True, fold)
    q.put((rank, r0, r1, R[: r1 - r0].clone()))
    d.close()


@pytest.mark.parametrize("world", [2, 3])
def test_partial_products_exchange_and_fold(world):
    """The multi-rank fast product's exchange step on CPU over gloo: after the all-to-all of
    row slabs and the XOR fold, rank r holds slab r of the XOR of every rank's partial."""
    import torch
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_exchange_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    n, w = 1280, 3
    total = torch.zeros((n, w), dtype=torch.int64)
    for r in range(world):
        g = torch.Generator().manual_seed(100 + r)
        total ^= torch.randint(-2**62, 2**62, (n, w), dtype=torch.int64, generator=g)
    covered = 0
    for rank, r0, r1, slab in got:
        assert torch.equal(slab, total[r0:r1]), rank
        covered += r1 - r0
    assert covered == n


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
def test_alt_subinstance_deal_two_ranks():
    """The multi-GPU fast product (host-layer sub-instances dealt round robin over ranks,
    partial products XOR-folded after one all-to-all of output-row slabs): two ranks
    sharing one GPU, every rank's slab checked against the tensor-core cubic product and
    by Freivalds."""
    import json
    import os
    import subprocess
    import sys
    env = dict(os.environ, BMM_DIST_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29533", "bench.py", "--gpus", "2", "--workload",
           "c4s-gf2-altsi-16384", "--leaf-log2", "9", "--steps", "3", "--warmup", "3"]
    r = subprocess.run(cmd, cwd=str(ROOT), env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    d = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][0])
    assert d["n_gpus"] == 2 and d["config"]["host_levels"] == 1 and d["config"]["subinstances_rank0"] == 4
    assert d["parity"]["ok"] is True and d["parity"]["slab_equals_cubic_product"] is True
    assert d["value"] > 0 and d["gpu_launches"] > 0


@pytest.mark.gpu
def test_out_of_core_two_ranks_share_host_b():
    """Out-of-core driver under two ranks: B lives once in /dev/shm (generated by rank 0,
    mapped and page-locked by both), each rank streams its row slab through a small
    device budget; rows and a column of C are checked on the CPU."""
    import json
    import os
    import subprocess
    import sys
    env = dict(os.environ, BMM_DIST_BACKEND="gloo")
    before = {f for f in os.listdir("/dev/shm") if f.startswith("bmm_B_32768")}
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29535", "bench.py", "--gpus", "2", "--workload",
           "c5s-gf2-ooc-32768", "--steps", "1", "--warmup", "1", "--device-budget", str(48 << 20), "--check"]
    r = subprocess.run(cmd, cwd=str(ROOT), env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    d = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][0])
    assert d["n_gpus"] == 2 and d["spot_check"] is True and d["config"]["rows_per_rank"] == 16384
    assert {f for f in os.listdir("/dev/shm") if f.startswith("bmm_B_32768")} <= before  # nothing left behind


@pytest.mark.gpu
def test_out_of_core_alt_tiles_two_ranks():
    """Out-of-core fast product under two ranks: each rank runs its run of output row
    panels (bmmgpu_multiply_panels, alt-si block products in 4096-bit tiles) with B in
    shared host memory; every slab is checked by Freivalds and numpy rows / a column."""
    import json
    import os
    import subprocess
    import sys
    env = dict(os.environ, BMM_DIST_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29537", "bench.py", "--gpus", "2", "--workload",
           "c5s-gf2-altooc-32768", "--steps", "1", "--warmup", "1", "--alt-tile-log2", "12", "--leaf-log2", "10",
           "--check"]
    r = subprocess.run(cmd, cwd=str(ROOT), env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    d = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][0])
    assert d["n_gpus"] == 2 and d["spot_check"] is True and d["config"]["rows_per_rank"] == 16384
    assert d["parity"]["freivalds_64_columns"] is True and d["config"]["algo"] == "alt-si"
