#!/usr/bin/env python
"""Benchmark: effective Pbop/s of the Boolean / GF(2) bit-matrix product on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload NAME] [--kernel auto|lop3|umma]
    python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N ...   (one rank per GPU)
    python bench.py --impl reference ...   (the reference's own CPU implementation, oracle/_ref)

Default workload (BASELINE.json configs[2], the one quoted at 1/2/4/8 GPUs):
Boolean product of A = BitMatrix::random(131072, 131072, 1) and
B = random(131072, 131072, 2), cubic kernel.  The output rows are split into
N contiguous slabs, one per rank, with no exchange (strong scaling: total
work fixed).  One step = Bt = transpose(B) + the slab product, inputs resident
in HBM; `e2e` repeats the step through the public C ABI (bmmgpu_cubic) from
pinned host buffers, H2D/D2H inside the timed region.  Inputs (2 GiB per
operand) are far larger than the 126 MB L2, so no explicit flush is needed.

Metric convention (reference bmm_cli.cpp:134-141):
effective bop/s = (2 m k n - m n) / T, reported in Pbop/s.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "effective Pbop/s (n^3 bops/s), Boolean & GF(2) products, 1/2/4/8 B200"
UNIT = "Pbop/s"
GF2, BOOL = 1, 0

WORKLOADS = {
    # name: (n, ring, algo, description)
    "c3-bool-cubic-131072": (131072, BOOL, 0, "Boolean product n=131072 cubic (BASELINE configs[2])"),
    "c3-gf2-cubic-131072": (131072, GF2, 0, "GF(2) product n=131072 cubic"),
    "c1-gf2-cubic-8192": (8192, GF2, 0, "GF(2) product n=8192 cubic (BASELINE configs[0])"),
    "c1-bool-cubic-8192": (8192, BOOL, 0, "Boolean product n=8192 cubic (BASELINE configs[0])"),
    "c2-gf2-altsi-65536": (65536, GF2, 2, "GF(2) product n=65536 alternative-basis Strassen (BASELINE configs[1])"),
    "c4-gf2-cubic-262144": (262144, GF2, 0, "GF(2) product n=262144, output row slabs (BASELINE configs[3])"),
    "c4-gf2-altsi-262144": (262144, GF2, 2, "GF(2) product n=262144 alternative-basis Strassen"),
    # a small instance of the same multi-GPU tile partition (tests)
    "c4s-gf2-altsi-16384": (16384, GF2, 2, "GF(2) product n=16384 alternative-basis Strassen (multi-rank test size)"),
    # configs[4] (n = 2^20 on 8 GPUs needs 384 GiB of host memory for A, B, C; one box has
    # 196 GB), scaled to one GPU: n = 2^19 from pinned host memory through the out-of-core
    # driver with a device budget below the operands (A row panels resident, B streamed in
    # K-chunks, partial products XOR/OR-folded on device, C tiles back to host).
    "c5-bool-ooc-524288": (524288, BOOL, 0, "Boolean n=2^19 out-of-core from host (configs[4] scaled to 1 GPU)"),
    "c5-gf2-ooc-524288": (524288, GF2, 0, "GF(2) n=2^19 out-of-core from host (configs[4] scaled to 1 GPU)"),
    # the same GF(2) product with alternative-basis block products inside the output tiles
    # (csrc/alt_tiles.cu): C[I, J] = XOR_K A[I, K] . B[K, J], each block product the
    # device-resident alt-si recursion, tiles streamed from host memory
    "c5-gf2-altooc-524288": (524288, GF2, 2, "GF(2) n=2^19 out-of-core, alt-si block products in output tiles "
                                             "(configs[4] scaled to 1 GPU)"),
    # a small instance of the same out-of-core path (tests; run with a small --device-budget)
    "c5s-gf2-ooc-32768": (32768, GF2, 0, "GF(2) n=2^15 out-of-core from host (test size)"),
    "c5s-gf2-altooc-32768": (32768, GF2, 2, "GF(2) n=2^15 out-of-core alt-si tiles (test size)"),
}
OOC_BUDGET = 40 << 30  # device bytes the out-of-core workloads may use (operands are 3 x 32 GiB)
DEFAULT_WORKLOAD = "c3-bool-cubic-131072"
# Paper V100 numbers for the same metric/config at 1 GPU, Pbop/s.
PUBLISHED_1GPU = {"c3-bool-cubic-131072": 0.15127, "c3-gf2-cubic-131072": 0.17014, "c1-gf2-cubic-8192": 0.13283,
                  "c1-bool-cubic-8192": 0.14000, "c2-gf2-altsi-65536": 0.30177}
KERNEL_IDS = {"auto": 0, "lop3": 1, "umma": 2}


def eff_bops(m: int, k: int, n: int) -> float:
    return 2.0 * m * k * n - float(m) * n


def n3_rate(value: float, n: int) -> dict:
    """BASELINE.json names the metric "n^3 bops/s"; the headline `value` follows the reference's
    numerator 2n^3 - n^2 (bmm_cli.cpp:134-141).  Both are reported: this is
    the same measurement with n^3 as the numerator."""
    return {"value": value * float(n) ** 3 / eff_bops(n, n, n), "unit": UNIT,
            "note": "n^3 / T (about half the headline (2n^3 - n^2) / T)"}


# ------------------------------------------------------------------ distributed plumbing
class Dist:
    """One process per GPU (torchrun env).  NCCL for the barrier and the max-over-ranks
    reduction; BMM_DIST_BACKEND=gloo runs the same rank logic over gloo, which also
    lets several ranks share one GPU (the multi-rank path tested on a 1-GPU box)."""

    def __init__(self) -> None:
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local_rank = int(os.environ.get("LOCAL_RANK", "0"))
        self.device = self.local_rank
        self.pg = None
        self.backend = None
        if self.world > 1:
            import torch
            import torch.distributed as dist
            cuda = torch.cuda.is_available()
            if cuda:
                self.device = self.local_rank % torch.cuda.device_count()
            self.backend = os.environ.get("BMM_DIST_BACKEND") or ("nccl" if cuda else "gloo")
            if self.backend == "nccl":
                torch.cuda.set_device(self.device)
            dist.init_process_group(backend=self.backend)
            self.pg = dist

    def barrier(self) -> None:
        if self.pg is not None:
            if self.backend == "nccl":
                self.pg.barrier(device_ids=[self.device])
            else:
                self.pg.barrier()

    def max(self, x: float) -> float:
        if self.pg is None:
            return x
        import torch
        dev = f"cuda:{self.device}" if self.backend == "nccl" else "cpu"
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        self.pg.all_reduce(t, op=self.pg.ReduceOp.MAX)
        return float(t.item())

    def close(self) -> None:
        if self.pg is not None:
            self.pg.destroy_process_group()


def bind_to_gpu_cpus(dev: int) -> list[int] | None:
    """Pin this process to the host cores NVML reports as local to GPU `dev` (its NUMA
    node), before any page-locked buffer is allocated: the pinned operand buffers then
    sit in the GPU's local memory and the end-to-end copies do not cross the socket
    interconnect (measured run-to-run e2e spread without it: 60-79 ms at n=65536)."""
    try:
        import pynvml
        pynvml.nvmlInit()
        visible = [v for v in os.environ.get("CUDA_VISIBLE_DEVICES", "").split(",") if v.strip().isdigit()]
        idx = int(visible[dev]) if dev < len(visible) else dev
        h = pynvml.nvmlDeviceGetHandleByIndex(idx)
        n_cpu = os.cpu_count() or 1
        words = pynvml.nvmlDeviceGetCpuAffinity(h, (n_cpu + 63) // 64)
        cpus = [w * 64 + b for w, m in enumerate(words) for b in range(64) if (m >> b) & 1 and w * 64 + b < n_cpu]
        if cpus:
            os.sched_setaffinity(0, cpus)
            return cpus
    except Exception:
        pass
    return None


def shard_rows(n: int, rank: int, world: int, gran: int = 64) -> tuple[int, int]:
    """Contiguous output-row slab of `rank`, aligned to `gran` rows (no exchange
    between slabs): the C ABI's bmmgpu_slab_rows, the same rule bmmgpu_cubic
    applies across devices."""
    import paper_1909_01554_b200 as bmm
    return bmm.slab_rows(n, world, rank, gran)


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi sampled every 200 ms while the timed region runs."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int) -> None:
        self.gpu = gpu_index
        self.proc = None
        self.lines: list[str] = []
        self.thread = None

    def start(self) -> None:
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self) -> None:
        assert self.proc is not None and self.proc.stdout is not None
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict | None:
        if self.proc is None:
            return None
        # a timed region shorter than the poller's start-up and period (the n = 8192 lines) has no
        # sample inside it: take the poller's next one, right after the region
        t_end = time.time() + 1.0
        while not self.lines and time.time() < t_end:
            time.sleep(0.01)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        sm, smax, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                smax = max(smax, float(parts[1]))
            except ValueError:
                continue
            for name, val in zip(names, parts[4:8]):
                if val.lower() == "active":
                    reasons.add(name)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------------ reference CPU arm
def cpu_model() -> str | None:
    try:
        for ln in Path("/proc/cpuinfo").read_text().splitlines():
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def cpu_sample_shape(n: int) -> tuple[int, int]:
    """C[0:rows, 0:cols] (full K = n) timed for the CPU reference: the whole product up
    to n = 8192, else a slab sized for ~5 s per repetition on 16 host threads (the
    reference cubic runs at ~2 Tbop/s there), ~10-30 s over the repetitions."""
    if n <= 8192:
        return n, n
    return min(n, 1024), min(n, 32768)


ALT_SAMPLE_N = 8192  # reference alt-si sub-instance (full product, 1 worker: ~2-3 s)


def alt_auto_plan(n: int) -> tuple[int, int]:
    """(d_serial, d_parallel) of the reference's auto_plan (engine.cpp:13-22)."""
    k = n.bit_length() - 1 - 6
    return k - min(3, k), min(3, k)


def reference_sample(n: int, ring: int, rows: int, cols: int, hB: np.ndarray | None):
    """A bounded sample of the workload for the reference CPU implementation:
    C[0:rows, 0:cols] = A[0:rows, :] . B[:, 0:cols] with the full K = n, through
    the unmodified reference multiply_cubic (oracle/_ref) on all host cores."""
    from oracle import Reference
    ref = Reference()
    # rows [0, rows) of BitMatrix::random(n, n, 1) are random(rows, n, 1): one mt19937_64 draw
    # per word in row-major order (reference bitmatrix.cpp:64-77)
    a = ref.random(rows, n, 1)
    if hB is None:
        hB = ref.random(n, n, 2)
    b = np.ascontiguousarray(hB.reshape(n, n // 64)[:, : cols // 64]).ravel()
    workers = os.cpu_count() or 1

    def step() -> float:
        t0 = time.perf_counter()
        ref.multiply_cubic(a, b, rows, n, cols, ring, workers)
        return time.perf_counter() - t0

    return step, eff_bops(rows, n, cols), workers


def run_reference(args, dist: Dist) -> None:
    n, ring, algo, desc = WORKLOADS[args.workload]
    if dist.rank != 0:
        return
    rows, cols = cpu_sample_shape(n)
    if algo != 0:
        # the reference alt-si path on a bounded sub-instance: an n_s = ALT_SAMPLE_N full product, workers=1
        # (more workers make the reference alt path slower)
        from oracle import Reference
        ref = Reference()
        ns = ALT_SAMPLE_N
        a = ref.random(ns, ns, 1)
        b = ref.random(ns, ns, 2)

        def step() -> float:
            t0 = time.perf_counter()
            ref.multiply(a, b, ns, 2, 0, *alt_auto_plan(ns), 1, GF2)
            return time.perf_counter() - t0
        bops, workers, sample = eff_bops(ns, ns, ns), 1, f"alt-si full product n={ns}, auto plan, 1 worker"
    else:
        step, bops, workers = reference_sample(n, ring, rows, cols, None)
        sample = f"C[0:{rows}, 0:{cols}] of the n={n} product (full K={n}), multiply_cubic, {workers} threads"
    for _ in range(args.warmup):
        step()
    times = [step() for _ in range(args.steps)]
    t = statistics.median(times)
    value = bops / t / 1e15
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "u64", "n3_rate": n3_rate(value, n), "data": "synthetic (BitMatrix::random seeds 1, 2)",
            "config": {"workload": args.workload, "desc": desc, "n": n, "ring": "gf2" if ring else "boolean",
                       "sample": sample},
            "impl": "reference",
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": workers, "kind": "reference", "sample": sample,
                             "cpu_model": cpu_model(), "host_threads": os.cpu_count(),
                             "code": "unmodified reference bmm_core (oracle/_ref/libbmmref.so, built from "
                                     "/root/reference/proj/src); inputs from its own BitMatrix::random"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ our arm
def spot_check(hA: np.ndarray, hB: np.ndarray, hC: np.ndarray, n: int, ring: int, rows: list[int],
               col: int, m: int | None = None) -> bool:
    """Independent CPU check of full rows and one full column of C (numpy, no GPU,
    no oracle): row i = fold over k with A[i,k] = 1 of B row k; column j = per-row
    parity / OR of A[i,:] & B[:, j]."""
    w = n // 64
    m = n if m is None else m  # rows of this rank's slab of A and C
    A = hA[: m * w].reshape(m, w)
    B = hB.reshape(n, w)
    C = hC[: m * w].reshape(m, w)
    for i in rows:
        bits = np.unpackbits(A[i].view(np.uint8), bitorder="little")[:n]
        ks = np.flatnonzero(bits)
        acc = np.zeros(w, dtype=np.uint64)
        for c0 in range(0, ks.size, 4096):
            blk = B[ks[c0:c0 + 4096]]
            if ring == GF2:
                acc ^= np.bitwise_xor.reduce(blk, axis=0)
            else:
                acc |= np.bitwise_or.reduce(blk, axis=0)
        if not np.array_equal(acc, C[i]):
            return False
    bcol = ((B[:, col // 64] >> np.uint64(col % 64)) & np.uint64(1)).astype(np.uint8)
    bw = np.packbits(bcol, bitorder="little").view(np.uint64)
    got = ((C[:, col // 64] >> np.uint64(col % 64)) & np.uint64(1)).astype(np.uint8)
    for r0 in range(0, m, 8192):
        x = A[r0:r0 + 8192] & bw
        if ring == GF2:
            v = np.bitwise_xor.reduce(x, axis=1)
            v ^= v >> np.uint64(32)
            v ^= v >> np.uint64(16)
            v ^= v >> np.uint64(8)
            v ^= v >> np.uint64(4)
            v ^= v >> np.uint64(2)
            v ^= v >> np.uint64(1)
            want = (v & np.uint64(1)).astype(np.uint8)
        else:
            want = (np.bitwise_or.reduce(x, axis=1) != 0).astype(np.uint8)
        if not np.array_equal(want, got[r0:r0 + 8192]):
            return False
    return True


# ------------------------------------------------------------------ parity at the benchmarked size
# Independent checks of the timed product's output, run after the timed region.  They use
# stock PyTorch ops (gather / XOR) and numpy only -- never the library's kernels.
FREIVALDS_SEED = 12345


def gf2_matvec64(M, cols: int, X, row_block: int = 1024):
    """Y = M . X over GF(2) for a packed bit matrix M (rows x ceil(cols/64) words, torch
    int64, host or device; only the first `cols` bits of a row are used) and X = 64 packed
    bit-columns (`cols` words on the device).  Four Russians with byte tables: table c holds
    the XOR of the X rows selected by each 8-bit value of byte c, so row i of Y is the XOR
    over c of table_c[byte c of row i].  Stock torch ops (gather, bitwise XOR); host row
    blocks are streamed to the device."""
    import torch
    dev = X.device
    nbytes = -(-cols // 8)
    xpad = torch.zeros(nbytes * 8, dtype=torch.int64, device=dev)
    xpad[:cols] = X[:cols]
    xb = xpad.view(nbytes, 8)
    v = torch.arange(256, device=dev)
    T = torch.zeros((nbytes, 256), dtype=torch.int64, device=dev)
    for b in range(8):
        sel = ((v >> b) & 1).bool()
        T ^= torch.where(sel[None, :], xb[:, b:b + 1], torch.zeros((), dtype=torch.int64, device=dev))
    Tf = T.view(-1)
    p2 = 1 << (nbytes - 1).bit_length()
    offs = (torch.arange(nbytes, device=dev) * 256)[None, :]
    rows = M.shape[0]
    out = torch.empty(rows, dtype=torch.int64, device=dev)
    for r0 in range(0, rows, row_block):
        blk = M[r0:r0 + row_block].to(dev, non_blocking=False).contiguous()
        by = blk.view(torch.uint8)[:, :nbytes].long()
        if cols % 8:
            by[:, -1] &= (1 << (cols % 8)) - 1
        g = Tf[by + offs]
        if p2 != nbytes:
            g = torch.nn.functional.pad(g, (0, p2 - nbytes))
        h = p2
        while h > 1:
            h //= 2
            g = g[:, :h] ^ g[:, h:2 * h]
        out[r0:r0 + blk.shape[0]] = g[:, 0]
    return out


def freivalds_gf2(A, B, C, m: int, k: int, n: int, reps: int = 1) -> bool:
    """C == A . B over GF(2) with probability of a false pass <= 2^-64 per rep:
    C X == A (B X) for 64 random bit-columns X.  A: m x >=k bits,
    B: k x >= n bits, C: m x >= n bits (torch int64 word matrices, host or device)."""
    import torch
    dev = "cuda" if torch.cuda.is_available() else "cpu"
    g = torch.Generator(device=dev).manual_seed(FREIVALDS_SEED)
    for _ in range(reps):
        X = torch.randint(-2**63, 2**63 - 1, (n,), dtype=torch.int64, device=dev, generator=g)
        lhs = gf2_matvec64(C[:m], n, X)
        rhs = gf2_matvec64(A[:m], k, gf2_matvec64(B[:k], n, X))
        if not torch.equal(lhs, rhs):
            return False
    return True


def sparse_boolean_inputs(m: int, n: int, r0: int, k_and: int = 9):
    """Seeded sparse operands for a non-vacuous Boolean check at size: each bit is the AND of
    k_and uniform bits (density 2^-k_and; at n = 131072 and k_and = 9 about 39 % of C is
    one).  Returns device tensors A (rows r0 .. r0+m of an n x n matrix) and B (n x n)."""
    import torch
    w = n // 64
    gen = torch.Generator(device="cuda").manual_seed(2024)

    def rnd():
        out = torch.full((n, w), -1, dtype=torch.int64, device="cuda")
        for _ in range(k_and):
            out &= torch.randint(-2**63, 2**63 - 1, (n, w), dtype=torch.int64, device="cuda", generator=gen)
        return out
    B = rnd()
    A = rnd()[r0:r0 + m].contiguous()
    return A, B


def parity_in_core(args, dist, n: int, m: int, r0: int, ring: int, algo: int, kernel: int, dA, dB, dBt, dC,
                   hA_np: np.ndarray, hB_np: np.ndarray, hC_e2e, run_step) -> dict:
    """Parity of the benchmarked product at its full size (after the timed region).
    GF(2): Freivalds with 64 random bit-columns on the timed output + full rows and a full
    column recomputed in numpy.  Boolean: the dense product must be all ones (every bit),
    then a sparse seeded product (AND-of-9 inputs, ~39 % ones in C at n = 131072) goes
    through the same device path (transpose + the same kernel, same shape, so the same
    long-K wave-aligned mode) and full rows / columns are recomputed in numpy.  The e2e
    leg's host output must equal the device-resident result bit for bit."""
    import torch
    t0 = time.perf_counter()
    w = n // 64
    res: dict = {}
    C = dC[:m, :w]
    if hC_e2e is not None:
        res["e2e_output_equals_device_output"] = bool(np.array_equal(
            hC_e2e[: m * w], C.contiguous().cpu().numpy().view(np.uint64).ravel()))
    rows = sorted({0, m // 3, m // 2 + 1, m - 1})
    if ring == GF2:
        res["freivalds_64_columns"] = freivalds_gf2(dA[:m, :w], dB.view(n, w), C, m, n, n)
        hC = C.contiguous().cpu().numpy().view(np.uint64).ravel()
        res["numpy_rows_and_column"] = spot_check(hA_np, hB_np, hC, n, GF2, rows[:2], (7 * n) // 11, m)
        res["method"] = "GF(2): Freivalds C.X == A.(B.X), 64 random bit-columns (torch gather/XOR, error <= 2^-64); " \
                        f"rows {rows[:2]} and column {(7 * n) // 11} recomputed in numpy"
    else:
        res["dense_all_ones"] = bool(int((C != -1).sum().item()) == 0)
        sA, sB = sparse_boolean_inputs(m, n, r0)
        dA[:m, :w].copy_(sA)
        dB.view(n, w).copy_(sB)
        del sA, sB
        run_step()
        torch.cuda.synchronize()
        hAs = dA[:m, :w].contiguous().cpu().numpy().view(np.uint64).ravel()
        hBs = dB.view(n, w).cpu().numpy().view(np.uint64).ravel()
        Cs = dC[:m, :w].contiguous().cpu().numpy().view(np.uint64).ravel()
        dens = float(np.unpackbits(Cs[: min(Cs.size, 1 << 22)].view(np.uint8)).mean())
        srows = sorted({int(x) for x in np.linspace(0, m - 1, 24)})
        res["sparse_rows_and_columns"] = bool(all(spot_check(hAs, hBs, Cs, n, BOOL, srows if i == 0 else [], j, m)
                                                  for i, j in enumerate([n // 5, (7 * n) // 11])))
        res["sparse_density_of_C"] = round(dens, 4)
        res["method"] = ("Boolean: dense product all ones (every word checked on device); sparse AND-of-9 seeded "
                         f"inputs through the same transpose + kernel at the same shape, {len(srows)} full rows and "
                         "2 full columns recomputed in numpy")
    ok = all(v for v in res.values() if isinstance(v, bool))
    res["ok"] = bool(dist.max(0.0 if ok else 1.0) == 0.0)
    res["seconds"] = round(time.perf_counter() - t0, 2)
    return res


class SharedHostWords:
    """A host word array shared by the ranks of one node: a /dev/shm file created by rank
    0 (its name broadcast to the others), mapped by every rank and page-locked with
    cudaHostRegister so the copies run at link speed.  Rank 0 unlinks the file as soon as
    every rank has mapped it."""

    def __init__(self, tag: str, words: int, dist: Dist) -> None:
        import torch
        import torch.distributed as tdist
        name = [f"/dev/shm/{tag}"] if dist.rank == 0 else [None]
        if dist.rank == 0:
            with open(name[0], "wb") as f:
                f.truncate(words * 8)
        tdist.broadcast_object_list(name, src=0)
        self.path, self.rank = name[0], dist.rank
        self.tensor = torch.from_file(self.path, shared=True, size=words, dtype=torch.int64)
        dist.barrier()
        if dist.rank == 0:
            os.unlink(self.path)  # the mappings keep the pages; nothing is left behind on a crash
        rc = torch.cuda.cudart().cudaHostRegister(self.tensor.data_ptr(), words * 8, 0)
        self.registered = int(rc) == 0 if not isinstance(rc, tuple) else int(rc[0]) == 0

    def close(self) -> None:
        import torch
        if self.registered:
            torch.cuda.cudart().cudaHostUnregister(self.tensor.data_ptr())


def run_ooc(args, dist: Dist) -> None:
    """Out-of-core workloads: the inputs live in (pinned) host memory by definition, so
    the measured number is the end-to-end one through bmmgpu_cubic; value = e2e."""
    import torch
    import paper_1909_01554_b200 as bmm

    n, ring, algo, desc = WORKLOADS[args.workload]
    lib = bmm.lib()
    dev = dist.device
    torch.cuda.set_device(dev)
    w = n // 64
    if algo == 0:
        r0, r1 = shard_rows(n, dist.rank, dist.world, 256)
        tile_log2, p0, p1 = 0, 0, 0
    else:
        # output row panels of b x b tiles, a contiguous run of panels per rank
        b = min(131072, n // max(2, dist.world)) if not args.alt_tile_log2 else 1 << args.alt_tile_log2
        T = n // b
        if T % dist.world:
            raise SystemExit(f"{T} tile panels do not split over {dist.world} ranks")
        tile_log2 = b.bit_length() - 1
        p0, p1 = dist.rank * T // dist.world, (dist.rank + 1) * T // dist.world
        r0, r1 = p0 * b, p1 * b
    m = r1 - r0
    t_gen = time.perf_counter()
    hA = torch.empty(max(m, 1) * w, dtype=torch.int64, pin_memory=True)
    hC = torch.empty(max(m, 1) * w, dtype=torch.int64, pin_memory=True)
    shared_b = None
    if dist.world > 1:
        # one copy of B in host memory for all ranks of the node (the paper's shared-memory
        # host; at n = 2^20 a per-rank copy would be 128 GiB each): rank 0 generates it
        # into /dev/shm, every rank maps it and page-locks its mapping
        shared_b = SharedHostWords(f"bmm_B_{n}_{os.getpid() if dist.rank == 0 else 0}", n * w, dist)
        hB = shared_b.tensor
        if dist.rank == 0:
            bmm.random_rows_into(hB.numpy().view(np.uint64), n, 2, 0, n)
        dist.barrier()
    else:
        hB = torch.empty(n * w, dtype=torch.int64, pin_memory=True)
        bmm.random_rows_into(hB.numpy().view(np.uint64), n, 2, 0, n)
    hA_np, hB_np, hC_np = (t.numpy().view(np.uint64) for t in (hA, hB, hC))
    bmm.random_rows_into(hA_np, n, 1, r0, r1)
    t_gen = time.perf_counter() - t_gen
    budget = args.device_budget or OOC_BUDGET
    opts = bmm._opts(0 if args.kernel == "auto" else KERNEL_IDS[args.kernel], device_mask=1 << dev,
                     device_budget=budget, force_streaming=1)
    # fast GF(2) on one rank: the sub-instance driver (BMMGPU_ALT_OOC=tiles or several ranks: output tiles)
    subinst = algo != 0 and dist.world == 1 and os.environ.get("BMMGPU_ALT_OOC") != "tiles"
    plan_c = bmm._Plan(0, (n // 64).bit_length() - 1, 0, 1, 1)
    dh_sub = 0
    if subinst:
        depth = (n // 64).bit_length() - 1
        e_all = max(0, min(depth, depth + 6 - (args.leaf_log2 or 12)))
        # the library's choice (alt.cu subinst_levels): the two generated children and ~11 sub-instance arrays
        dh_sub = next((d for d in range(1, 5) if d < e_all and (n >> d) >= 8192
                       and 2 * (n // 2) ** 2 / 8 + 11 * (n >> d) ** 2 / 8 <= budget), min(max(1, e_all - 1), 4))

    def check(rc: int) -> None:
        if rc != 0:
            raise RuntimeError(lib.bmmgpu_last_error().decode())

    def step() -> float:
        dist.barrier()
        s0 = time.perf_counter()
        if algo == 0:
            check(lib.bmmgpu_cubic(hA.data_ptr(), hB.data_ptr(), hC.data_ptr(), m, n, n, ring, ctypes.byref(opts)))
        elif subinst:
            # one rank: bmmgpu_multiply's out-of-core driver runs the recursion's own top-level
            # sub-instances (7^dh of n >> dh, generated on the device from streamed sub-blocks)
            check(lib.bmmgpu_multiply(hA.data_ptr(), hB.data_ptr(), hC.data_ptr(), n, algo, ctypes.byref(plan_c),
                                      GF2, ctypes.byref(opts)))
        else:
            # the library addresses A and C as whole n x n matrices and touches only this
            # rank's panel rows: hand it base pointers r0 rows before the slab buffers
            check(lib.bmmgpu_multiply_panels(hA.data_ptr() - r0 * w * 8, hB.data_ptr(), hC.data_ptr() - r0 * w * 8,
                                             n, algo, tile_log2, p0, p1, ctypes.byref(opts)))
        return time.perf_counter() - s0

    for _ in range(args.warmup):
        step()
    visible = [v for v in os.environ.get("CUDA_VISIBLE_DEVICES", "").split(",") if v.strip().isdigit()]
    sampler = ClockSampler(int(visible[dev]) if dev < len(visible) else dev)
    sampler.start()
    check(lib.bmmgpu_block_timer(1))
    times = [step() for _ in range(args.steps)]
    clocks = sampler.stop()
    k2clk = read_k2_clock(lib)
    blk_ms, blk_launches = ctypes.c_double(0.0), ctypes.c_uint64(0)
    check(lib.bmmgpu_block_timer_read(ctypes.byref(blk_ms), ctypes.byref(blk_launches)))
    check(lib.bmmgpu_block_timer(0))
    launches = lib.bmmgpu_last_launch_count()
    h2d, d2h = ctypes.c_uint64(0), ctypes.c_uint64(0)
    check(lib.bmmgpu_last_copy_bytes(ctypes.byref(h2d), ctypes.byref(d2h)))
    t = dist.max(statistics.median(times))
    total_bops = eff_bops(n, n, n)
    value = total_bops / t / 1e15
    ok = None
    parity = None
    if args.check:
        # every rank checks its own slab: rows and a column in numpy; GF(2) also Freivalds with
        # 64 random bit-columns, the operands streamed from host memory in row blocks
        pt0 = time.perf_counter()
        ok = spot_check(hA_np, hB_np, hC_np, n, ring, [0, m // 2 + 1, m - 1], n // 3, m)
        parity = {"numpy_rows_and_column": bool(ok)}
        if ring == GF2:
            parity["freivalds_64_columns"] = freivalds_gf2(hA.view(-1, w), hB.view(n, w), hC.view(-1, w), m, n, n)
        good = all(v for v in parity.values() if isinstance(v, bool))
        parity["method"] = ("rows 0, m/2+1, m-1 and column n/3 of this rank's slab recomputed in numpy" +
                            ("; Freivalds C.X == A.(B.X) with 64 random bit-columns (torch gather/XOR)"
                             if ring == GF2 else ""))
        parity["ok"] = bool(dist.max(0.0 if good else 1.0) == 0.0)
        parity["seconds"] = round(time.perf_counter() - pt0, 2)
        ok = parity["ok"]
    peaks = json.loads((ROOT / "profiles" / "peaks.json").read_text())
    kms = blk_ms.value / args.steps
    if algo == 0:
        launch_bops, kname = eff_bops(m, n, n), "cubic_umma2_kernel (K-chunk products of the tile driver)"
    elif subinst:
        # leaf layers of the 7^dh sub-instances: 7^e products of L = n >> e in all
        depth = (n // 64).bit_length() - 1
        e_levels = max(0, min(depth, depth + 6 - (args.leaf_log2 or 12)))
        leaf = n >> e_levels
        launch_bops = 7**e_levels * eff_bops(leaf, leaf, leaf)
        kname = (f"cubic_umma2_kernel (leaf layers of the 7^{dh_sub} sub-instances of {n >> dh_sub}: "
                 f"7^{e_levels} products of {leaf}^3 in all)")
    else:
        # leaf layers of the (n/b)^2 (m/b) block products: 7^e products of L = b >> e each
        bt = 1 << tile_log2
        depth = (bt // 64).bit_length() - 1
        e_levels = max(0, min(depth, depth + 6 - (args.leaf_log2 or 12)))
        leaf = bt >> e_levels
        launch_bops = (m // bt) * (n // bt) ** 2 * 7**e_levels * eff_bops(leaf, leaf, leaf)
        kname = (f"cubic_umma2_kernel (leaf layers of {(m // bt) * (n // bt) ** 2} alt-si block products of {bt}: "
                 f"7^{e_levels} products of {leaf}^3 each)")
    achieved = launch_bops / (kms * 1e-3)
    if dist.rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": dist.world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "n3_rate": n3_rate(value, n), "dtype": "e2m1",
                "data": "synthetic (BitMatrix::random seeds 1, 2, mt19937_64), pinned host memory",
                "config": {"workload": args.workload, "desc": desc, "n": n, "ring": "gf2" if ring else "boolean",
                           "algo": ["cubic", "sw", "alt-si", "alt-chain"][algo], "rows_per_rank": m,
                           "device_budget_bytes": budget if algo == 0 else None,
                           "driver": ("out-of-core tiles (force_streaming=1)" if algo == 0 else
                                      f"out-of-core sub-instances (bmmgpu_multiply: 7^{dh_sub} = {7 ** dh_sub} of "
                                      f"{n >> dh_sub}, generated on the device from streamed sub-blocks, "
                                      f"Q folded into C by host threads)" if subinst else
                                      f"out-of-core alt tiles (bmmgpu_multiply_panels, b = 2^{tile_log2}, "
                                      f"panels [{p0}, {p1}) on rank 0)"),
                           "device_budget_bytes_alt": budget if subinst else None,
                           "value_is": "end to end from pinned host buffers (the operands exceed the budget)",
                           "input_generation_s": t_gen,
                           "parallelism": f"output row slabs x{dist.world}, no exchange"},
                "roofline": {"bound": "tensor", "achieved": achieved / 1e12,
                             "peak": peaks["umma_mxf4_bops_sustained"] / 1e12, "unit": "Tbop/s",
                             "frac": achieved / peaks["umma_mxf4_bops_sustained"], "traffic": None,
                             "kernel": kname,
                             "kernel_ms": kms, "kernel_launches_per_step": blk_launches.value / args.steps,
                             "kernel_share_of_step": kms / (t * 1e3)},
                "cpu_baseline": None,
                "e2e": {"value": value, "unit": UNIT, "ms_per_step": t * 1e3,
                        "h2d_bytes_per_step": int(h2d.value), "d2h_bytes_per_step": int(d2h.value),
                        "h2d_note": ("counted by the library (bmmgpu_last_copy_bytes): each source sub-block once per "
                                     "sub-instance that selects it" if subinst else
                                     "counted by the library (bmmgpu_last_copy_bytes): A once, B once per "
                                     "resident row panel of the plan"),
                        "path": ("bmmgpu_cubic" if algo == 0 else "bmmgpu_multiply" if subinst else
                                 "bmmgpu_multiply_panels") +
                                " (include/bmmgpu.h) from pinned host buffers, per rank"},
                "spot_check": ok, "parity": parity, "clocks": clocks, "gpu_launches": int(launches * args.steps)}
        print(json.dumps(line), flush=True)
    if shared_b is not None:
        shared_b.close()


def read_k2_clock(lib) -> tuple[int, int]:
    """(cycles, ns) of CTA pair 0's MMA loop in the last K2 launch (bmmgpu_debug_k2_clock):
    read right after the timed steps, before any other product runs."""
    cyc, ns = ctypes.c_uint64(0), ctypes.c_uint64(0)
    if lib.bmmgpu_debug_k2_clock(ctypes.byref(cyc), ctypes.byref(ns)) != 0:
        return 0, 0
    return cyc.value, ns.value


def k2_clock(clk: tuple[int, int], launch_macs: float, kms: float) -> dict:
    """Effective SM clock of the last timed K2 launch (clock64 / globaltimer of CTA pair 0's MMA
    loop) and the MACs per SM clock it implies: nvidia-smi's clocks.sm does not show the power
    cap's clock slowdown, this does."""
    import torch
    cyc, ns = clk
    if not ns:
        return {}
    mhz = cyc / ns * 1e3
    sms = torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count
    per_clk = launch_macs / (kms * 1e-3) / sms / (mhz * 1e6)
    return {"sm_clock_effective_mhz": round(mhz, 1), "mac_per_sm_clock": round(per_clk, 1),
            "frac_per_clock": round(per_clk / 16384.0, 4),
            "per_clock_note": "achieved MACs per SM per effective clock against the tensor pipe's 16,384 "
                              "(kind::mxf4 M256 N256 K64 pair); the rest of the gap to the peak is the SM "
                              "clock under the power cap"}


def slab_exchange_xor(P, R, slabs: list[tuple[int, int]], me: int, G: int, stage_on_host: bool, fold) -> None:
    """The multi-rank fast product's one exchange step: rank d receives row slab d of every
    rank's partial product P (n x w words) into R (G pieces of its slab, rank order) by one
    all-to-all, then XOR-folds pieces 1 .. G-1 into piece 0 (`fold(d)`, the library's fold
    kernel on the GPU).  With gloo the tensors are staged through host memory."""
    import torch
    import torch.distributed as tdist
    r0, r1 = slabs[me]
    w = P.shape[1]
    if G > 1:
        splits_in = [(r1 - r0) * w] * G
        splits_out = [(b - a) * w for a, b in slabs]
        if stage_on_host:
            recv = torch.empty(R.numel(), dtype=torch.int64)
            tdist.all_to_all_single(recv, P.reshape(-1).cpu(), splits_in, splits_out)
            R.view(-1).copy_(recv)
        else:
            tdist.all_to_all_single(R.view(-1), P.reshape(-1), splits_in, splits_out)
    else:
        R.copy_(P[r0:r1])
    for d in range(1, G):
        fold(d)


def run_alt_deal(args, dist: Dist) -> None:
    """Fast GF(2) product on several GPUs (SURVEY section 8e, configs[3]): the top dh
    levels of the recursion are 7^dh independent sub-instances (the reference host layer,
    pipeline.cpp:198-369), dealt round robin to the ranks; each rank computes the partial
    product of its share on its GPU from resident A and Bt (bmmgpu_dev_multiply_partial),
    then the one exchange step: an all-to-all of output-row slabs (NCCL over NVLink), each
    rank XOR-folding the partials of the slab it owns.  dh is the library's most even deal
    (bmmgpu_host_levels: 343 sub-instances of n/8 over 8 ranks)."""
    import torch
    import torch.distributed as tdist
    import paper_1909_01554_b200 as bmm

    n, ring, algo, desc = WORKLOADS[args.workload]
    lib = bmm.lib()
    dev = dist.device
    torch.cuda.set_device(dev)
    G, me = dist.world, dist.rank
    w = n // 64
    dh = lib.bmmgpu_host_levels(n, G, args.leaf_log2)
    subs = 7 ** dh
    mine = len(range(me, subs, G))
    slabs = [bmm.slab_rows(n, G, d, 256) for d in range(G)]
    r0, r1 = slabs[me]
    hA = torch.empty(n * w, dtype=torch.int64, pin_memory=True)
    hB = torch.empty(n * w, dtype=torch.int64, pin_memory=True)
    bmm.random_rows_into(hA.numpy().view(np.uint64), n, 1, 0, n)
    bmm.random_rows_into(hB.numpy().view(np.uint64), n, 2, 0, n)
    dA = hA.view(n, w).to(f"cuda:{dev}")
    dB = hB.view(n, w).to(f"cuda:{dev}")
    dBt = torch.empty((n, w), dtype=torch.int64, device=f"cuda:{dev}")
    dP = torch.empty((n, w), dtype=torch.int64, device=f"cuda:{dev}")       # this rank's partial product
    dR = torch.empty((G * (r1 - r0), w), dtype=torch.int64, device=f"cuda:{dev}")  # received pieces of my slab
    stream = torch.cuda.current_stream()
    sp = ctypes.c_void_p(stream.cuda_stream)
    on_cpu = dist.backend == "gloo"
    torch.cuda.synchronize()

    def check(rc: int) -> None:
        if rc != 0:
            raise RuntimeError(lib.bmmgpu_last_error().decode())

    def step() -> None:
        check(lib.bmmgpu_dev_transpose(dB.data_ptr(), w, n, n, dBt.data_ptr(), n, w, sp))
        check(lib.bmmgpu_dev_multiply_partial(dA.data_ptr(), w, dBt.data_ptr(), w, dP.data_ptr(), w, n, algo, dh,
                                              me, G, args.leaf_log2, 0, sp))
        slab_exchange_xor(dP, dR, slabs, me, G, on_cpu,
                          lambda d: check(lib.bmmgpu_dev_fold(dR.data_ptr(), w, dR.data_ptr() + 8 * d * (r1 - r0) * w,
                                                              w, r1 - r0, w, ring, sp)))

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    visible = [v for v in os.environ.get("CUDA_VISIBLE_DEVICES", "").split(",") if v.strip().isdigit()]
    sampler = ClockSampler(int(visible[dev]) if dev < len(visible) else dev)
    sampler.start()
    check(lib.bmmgpu_block_timer(1))
    dist.barrier()
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = lib.bmmgpu_last_launch_count()
    t0.record(stream)
    for _ in range(args.steps):
        step()
    t1.record(stream)
    torch.cuda.synchronize()
    launches = lib.bmmgpu_last_launch_count() - launches0
    dist.barrier()
    clocks = sampler.stop()
    blk_ms, blk_n = ctypes.c_double(0.0), ctypes.c_uint64(0)
    check(lib.bmmgpu_block_timer_read(ctypes.byref(blk_ms), ctypes.byref(blk_n)))
    check(lib.bmmgpu_block_timer(0))
    ms = dist.max(t0.elapsed_time(t1) / args.steps)
    parity = None
    if args.check:
        # this rank's slab against the tensor-core cubic product of A[slab, :] . B (a different
        # algorithm) and, independently of the library, Freivalds with 64 random bit-columns
        pt0 = time.perf_counter()
        ref = torch.empty((r1 - r0, w), dtype=torch.int64, device=f"cuda:{dev}")
        check(lib.bmmgpu_dev_cubic(dA.data_ptr() + 8 * r0 * w, w, dBt.data_ptr(), w, ref.data_ptr(), w, r1 - r0, n, w,
                                   ring, 0, 0, sp))
        torch.cuda.synchronize()
        mine_slab = dR[: r1 - r0]
        ok_cubic = bool(torch.equal(ref, mine_slab))
        ok_frei = freivalds_gf2(dA[r0:r1], dB, mine_slab, r1 - r0, n, n)
        good = ok_cubic and ok_frei
        parity = {"slab_equals_cubic_product": ok_cubic, "freivalds_64_columns": ok_frei,
                  "ok": bool(dist.max(0.0 if good else 1.0) == 0.0), "seconds": round(time.perf_counter() - pt0, 2),
                  "method": "every rank's output slab equal to the tensor-core cubic product A[slab,:].B and passing "
                            "Freivalds (64 random bit-columns, torch gather/XOR)"}
    e = max(0, min((n // 64).bit_length() - 1, (n // 64).bit_length() - 1 + 6 - (args.leaf_log2 or 12)))
    e_sub = e - dh
    leaf = n >> e
    kms = blk_ms.value / args.steps
    launch_bops = mine * 7 ** e_sub * eff_bops(leaf, leaf, leaf)
    peaks = json.loads((ROOT / "profiles" / "peaks.json").read_text())
    achieved = launch_bops / (kms * 1e-3)
    value = eff_bops(n, n, n) / (ms * 1e-3) / 1e15
    if dist.rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": dist.world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "n3_rate": n3_rate(value, n), "dtype": "e2m1",
                "data": "synthetic (BitMatrix::random seeds 1, 2, mt19937_64)",
                "config": {"workload": args.workload, "desc": desc, "n": n, "ring": "gf2",
                           "algo": ["cubic", "sw", "alt-si", "alt-chain"][algo],
                           "parallelism": f"7^{dh} host-layer sub-instances of n/{2 ** dh} round robin over "
                                          f"{dist.world} ranks, partial products XOR-folded after one all-to-all "
                                          "of output-row slabs",
                           "host_levels": dh, "subinstances_rank0": mine},
                "roofline": {"bound": "tensor", "achieved": achieved / 1e12, "peak": peaks["umma_mxf4_bops_sustained"] / 1e12,
                             "unit": "Tbop/s", "frac": achieved / peaks["umma_mxf4_bops_sustained"], "traffic": None,
                             "kernel": f"cubic_umma2_kernel (leaf layer: 7^{e_sub} products of {leaf}^3 per "
                                       "sub-instance)",
                             "kernel_ms": kms, "kernel_share_of_step": kms / ms},
                "cpu_baseline": None, "e2e": None, "parity": parity, "clocks": clocks,
                "gpu_launches": int(launches)}
        print(json.dumps(line), flush=True)


def cpu_baseline_incore(args, n: int, ring: int, algo: int, hB_np) -> dict:
    """The reference CPU implementation on a bounded sample of the in-core workload, all host cores
    (rank 0 at N = 1): the `cpu_baseline` object of the bench line."""
    import paper_1909_01554_b200 as bmm
    os.sched_setaffinity(0, range(os.cpu_count() or 1))  # every host core, not just the GPU's node
    if algo == 0:
        rows, cols = cpu_sample_shape(n)
        stepf, sb, workers = reference_sample(n, ring, rows, cols, hB_np)
        sample = f"C[0:{rows}, 0:{cols}] of the n={n} product (full K={n}), reference multiply_cubic"
    else:
        from oracle import Reference
        ref = Reference()
        ns = ALT_SAMPLE_N
        a4 = np.zeros(ns * ns // 64, dtype=np.uint64)
        b4 = np.zeros_like(a4)
        bmm.random_rows_into(a4, ns, 1, 0, ns)
        bmm.random_rows_into(b4, ns, 2, 0, ns)

        def stepf() -> float:
            s0 = time.perf_counter()
            ref.multiply(a4, b4, ns, 2, 0, *alt_auto_plan(ns), 1, GF2)
            return time.perf_counter() - s0
        sb, workers, sample = eff_bops(ns, ns, ns), 1, f"reference alt-si n={ns}, auto plan, 1 worker"
    ts = [stepf() for _ in range(args.cpu_reps)]
    cpu = {"value": sb / statistics.median(ts) / 1e15, "unit": UNIT, "cores": workers, "kind": "reference",
           "sample": sample, "seconds": sum(ts), "cpu_model": cpu_model()}
    return cpu


def run_ours(args, dist: Dist) -> None:
    import torch
    import paper_1909_01554_b200 as bmm

    n, ring, algo, desc = WORKLOADS[args.workload]
    args.cpus = bind_to_gpu_cpus(dist.device)
    if args.workload.startswith(("c5-", "c5s-")):
        return run_ooc(args, dist)
    kernel = KERNEL_IDS[args.kernel]
    lib = bmm.lib()
    dev = dist.device
    torch.cuda.set_device(dev)
    gm, gn, gk = bmm.granularity(kernel)
    w = n // 64
    if algo == 0:
        r0, r1 = shard_rows(n, dist.rank, dist.world, gm)
    else:
        if dist.world > 1:
            return run_alt_deal(args, dist)
        r0, r1 = 0, n
    m = r1 - r0
    # pinned host inputs (the e2e leg copies from these every step)
    hA = torch.empty(max(m, 1) * w, dtype=torch.int64, pin_memory=True)
    hB = torch.empty(n * w, dtype=torch.int64, pin_memory=True)
    hC = torch.empty(max(m, 1) * w, dtype=torch.int64, pin_memory=True)
    hA_np, hB_np = hA.numpy().view(np.uint64), hB.numpy().view(np.uint64)
    bmm.random_rows_into(hA_np, n, 1, r0, r1)
    bmm.random_rows_into(hB_np, n, 2, 0, n)

    stream = torch.cuda.current_stream()
    sp = ctypes.c_void_p(stream.cuda_stream)
    m_pad = -(-m // gm) * gm
    n_pad = -(-n // 256) * 256
    kw = -(-w // (gk // 64)) * (gk // 64)
    dA = torch.zeros((m_pad, kw), dtype=torch.int64, device="cuda")
    dA[:m, :w].copy_(hA[: m * w].view(m, w), non_blocking=True)
    dB = hB.to("cuda", non_blocking=True)
    dBt = torch.empty((n_pad, kw), dtype=torch.int64, device="cuda")
    dC = torch.empty((m_pad, n_pad // 64), dtype=torch.int64, device="cuda")
    torch.cuda.synchronize()

    def check(rc: int) -> None:
        if rc != 0:
            raise RuntimeError(lib.bmmgpu_last_error().decode())

    launches_per_step = 0

    def step(i: int) -> None:
        nonlocal launches_per_step
        before = lib.bmmgpu_last_launch_count()
        check(lib.bmmgpu_dev_transpose(dB.data_ptr(), w, n, n, dBt.data_ptr(), n_pad, kw, sp))
        if algo == 0:
            check(lib.bmmgpu_dev_cubic(dA.data_ptr(), kw, dBt.data_ptr(), kw, dC.data_ptr(), n_pad // 64, m_pad,
                                       n_pad, kw, ring, kernel, 0, sp))
        else:
            check(lib.bmmgpu_dev_multiply(dA.data_ptr(), kw, dBt.data_ptr(), kw, dC.data_ptr(), n_pad // 64, n,
                                          algo, args.leaf_log2, kernel, sp))
        launches_per_step = lib.bmmgpu_last_launch_count() - before

    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize()
    # bracket every block-product launch of the timed steps with events (the dominant
    # kernel's device time, also inside the fast pipeline)
    check(lib.bmmgpu_block_timer(1))
    visible = [v for v in os.environ.get("CUDA_VISIBLE_DEVICES", "").split(",") if v.strip().isdigit()]
    sampler = ClockSampler(int(visible[dev]) if dev < len(visible) else dev)
    sampler.start()
    dist.barrier()
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for i in range(args.steps):
        step(args.warmup + i)
    t1.record(stream)
    torch.cuda.synchronize()
    dist.barrier()
    clocks = sampler.stop()
    k2clk = read_k2_clock(lib)
    blk_ms, blk_launches = ctypes.c_double(0.0), ctypes.c_uint64(0)
    check(lib.bmmgpu_block_timer_read(ctypes.byref(blk_ms), ctypes.byref(blk_launches)))
    check(lib.bmmgpu_block_timer(0))
    local_ms = t0.elapsed_time(t1) / args.steps
    ms = dist.max(local_ms)
    total_bops = eff_bops(n, n, n)
    value = total_bops / (ms * 1e-3) / 1e15

    # ---- end to end through the public C ABI, host buffers, copies inside the timed region
    e2e = None
    if not args.no_e2e and algo == 0:
        opts = bmm._opts(kernel, device_mask=1 << dev, device_budget=args.device_budget,
                         force_streaming=args.stream)

        def e2e_step() -> None:
            check(lib.bmmgpu_cubic(hA.data_ptr(), hB.data_ptr(), hC.data_ptr(), m, n, n, ring, ctypes.byref(opts)))

        e2e_step()
        e2e_step()
        dist.barrier()
        te = []
        # small products finish in about a millisecond: take more samples of them
        reps = max(1, min(args.steps, args.e2e_steps)) if n >= 65536 else max(args.e2e_steps, 20)
        for _ in range(reps):
            dist.barrier()
            s0 = time.perf_counter()
            e2e_step()
            te.append(time.perf_counter() - s0)
        e2e_t = dist.max(statistics.median(te))
        e2e = {"value": total_bops / e2e_t / 1e15, "unit": UNIT, "ms_per_step": e2e_t * 1e3,
               "h2d_bytes_per_step": int(m * w * 8 + n * w * 8), "d2h_bytes_per_step": int(m * w * 8),
               "path": "bmmgpu_cubic (include/bmmgpu.h) from pinned host buffers, per rank"}
    elif not args.no_e2e:
        import paper_1909_01554_b200 as bmm2
        a = bmm2.BitMatrix(n, n, hA_np[: n * w])
        b = bmm2.BitMatrix(n, n, hB_np)
        out = bmm2.BitMatrix(n, n, hC.numpy().view(np.uint64)[: n * w])
        plan = bmm2.LayerPlan.auto_plan(n, 1)
        for _ in range(2):  # warm: the first calls grow the memory pool and search the streaming order
            bmm2.multiply(a, b, bmm2.Algo(algo), plan, bmm2.Semiring(ring), kernel=kernel,
                          leaf_log2=args.leaf_log2, out=out)
        te = []
        # products of ~50 ms: take more samples of them
        reps = max(1, min(args.steps, args.e2e_steps)) if n > 65536 else max(args.e2e_steps, 10)
        for _ in range(reps):
            s0 = time.perf_counter()
            bmm2.multiply(a, b, bmm2.Algo(algo), plan, bmm2.Semiring(ring), kernel=kernel,
                          leaf_log2=args.leaf_log2, out=out)
            te.append(time.perf_counter() - s0)
        e2e_t = statistics.median(te)
        e2e = {"value": total_bops / e2e_t / 1e15, "unit": UNIT, "ms_per_step": e2e_t * 1e3,
               "h2d_bytes_per_step": int(2 * n * w * 8), "d2h_bytes_per_step": int(n * w * 8),
               "path": "bmmgpu_multiply (include/bmmgpu.h) from pinned host buffers",
               "samples_ms": [round(x * 1e3, 2) for x in te]}

    # ---- parity of the benchmarked output at full size (after the timed regions)
    parity = None
    if args.check:
        hC_e2e = hC.numpy().view(np.uint64) if e2e is not None else None
        parity = parity_in_core(args, dist, n, m, r0, ring, algo, kernel, dA, dB, dBt, dC, hA_np, hB_np, hC_e2e,
                                lambda: step(0))

    # ---- roofline of the dominant kernel
    peaks = json.loads((ROOT / "profiles" / "peaks.json").read_text())
    resolved = kernel if kernel else 2  # AUTO = the tcgen05 CTA-pair kernel (csrc/capi.cu resolve_kernel)
    peak = peaks["lop3_bops"] if resolved == 1 else peaks["umma_mxf4_bops_sustained"]
    kname = {1: "cubic_lop3_kernel", 2: "cubic_umma2_kernel"}[resolved]
    if algo == 0:
        # algorithmic work of the one product launch: the slab's 2 m n k - m n
        launch_bops = eff_bops(m, n, n)
        e_levels = 0
    else:
        # the leaf layer: 7^e products of L = n >> e (the recursion's exact block products)
        depth = (n // 64).bit_length() - 1
        e_levels = max(0, min(depth, depth + 6 - (args.leaf_log2 or 12)))
        leaf = n >> e_levels
        launch_bops = 7**e_levels * eff_bops(leaf, leaf, leaf)
        kname = f"{kname} (leaf layer: 7^{e_levels} products of {leaf}^3)"
    kms = blk_ms.value / args.steps  # block-product device time per step
    achieved = launch_bops / (kms * 1e-3)
    traffic = None
    tf = ROOT / "profiles" / "traffic.json"
    if tf.exists():
        traffic = json.loads(tf.read_text()).get(f"{args.workload}:{resolved}")
    roofline = {"bound": "alu" if resolved == 1 else "tensor", "achieved": achieved / 1e12,
                "peak": peak / 1e12, "unit": "Tbop/s", "frac": achieved / peak, "traffic": traffic,
                "kernel": kname, "kernel_ms": kms, "kernel_launches_per_step": blk_launches.value / args.steps,
                "kernel_share_of_step": kms / ms,
                "peak_source": ("profiles/peaks.json lop3_bops (measured LOP3 issue rate, microbench/ubench.cu)"
                                if resolved == 1 else
                                "profiles/peaks.json umma_mxf4_bops_sustained: the K2 MMA instruction back to "
                                "back for seconds on K2-like operands under the power cap (microbench/"
                                "ubench_sustained.cu, 16,375 MAC/SM-clock at an effective 1845 MHz); "
                                "MEASURED_PEAKS.json has no integer-ALU or fp4 figure")}
    if resolved != 1:
        roofline.update(k2_clock(k2clk, launch_bops / 2.0, kms))
    mp = ROOT / "MEASURED_PEAKS.json"
    if mp.exists() and resolved != 1:
        # cross-check against the driver's bf16 GEMM figure: kind::mxf4 issues 4 MACs per
        # bf16 MAC slot, so a bf16-derived bit-product peak would be 4 x 2 x bf16 FLOP/s / 2
        bf16 = json.loads(mp.read_text()).get("bf16_tflops")
        if bf16:
            roofline["bf16_derived_peak"] = {"value": 4.0 * bf16, "unit": "Tbop/s",
                                             "frac": achieved / (4.0 * bf16 * 1e12),
                                             "note": "MEASURED_PEAKS.json bf16_tflops x 4 (cuBLAS bf16 reaches "
                                                     "~74 % of its nominal rate, so this understates the tensor "
                                                     "pipe; the frac above uses the directly measured mxf4 rate)"}

    # ---- CPU baseline: the reference on this box's host cores, rank 0 at N=1
    cpu = None
    if dist.world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_baseline_incore(args, n, ring, algo, hB_np)
        except Exception as e:  # the reference library missing on this box must not cost the bench line
            cpu = {"unavailable": f"{type(e).__name__}: {e}"}

    if dist.rank == 0:
        published = PUBLISHED_1GPU.get(args.workload) if dist.world == 1 else None
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": dist.world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": (value / published) if published else None, "n3_rate": n3_rate(value, n),
                "dtype": "u32" if resolved == 1 else "e2m1",
                "data": "synthetic (BitMatrix::random seeds 1, 2, mt19937_64)",
                "config": {"workload": args.workload, "desc": desc, "n": n, "ring": "gf2" if ring else "boolean",
                           "algo": ["cubic", "sw", "alt-si", "alt-chain"][algo], "kernel": args.kernel,
                           "rows_per_rank": m, "l2": "inputs (n^2/8 B per operand) far exceed the 126 MB L2",
                           "host_cpus_bound": len(args.cpus) if args.cpus else None,
                           "parallelism": f"output row slabs x{dist.world}, no exchange"},
                "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "parity": parity, "clocks": clocks,
                "gpu_launches": int(launches_per_step * args.steps)}
        print(json.dumps(line), flush=True)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default=DEFAULT_WORKLOAD)
    ap.add_argument("--kernel", choices=sorted(KERNEL_IDS), default="auto")
    ap.add_argument("--leaf-log2", dest="leaf_log2", type=int, default=0)
    ap.add_argument("--alt-tile-log2", dest="alt_tile_log2", type=int, default=0,
                    help="out-of-core alt workloads: log2 of the output tile side (0: min(2^17, n / ranks))")
    ap.add_argument("--e2e-steps", dest="e2e_steps", type=int, default=3)
    ap.add_argument("--cpu-reps", dest="cpu_reps", type=int, default=3)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--stream", type=int, default=0, choices=[0, 1, 2],
                    help="e2e driver: 0 auto, 1 out-of-core tiles (A panels resident, B streamed in K-chunks), "
                         "2 K-outer pipeline (C resident, A/B K-chunks uploaded behind the product)")
    ap.add_argument("--device-budget", dest="device_budget", type=int, default=0,
                    help="HBM bytes the e2e call may use (0 = free memory; the c5 workloads default to 40 GiB)")
    ap.add_argument("--check", action=argparse.BooleanOptionalAction, default=True,
                    help="verify the benchmarked output at full size after the timed region (default on): GF(2) "
                         "Freivalds + numpy rows/columns, Boolean all-ones + a sparse product's rows/columns in "
                         "numpy, out-of-core rows/columns in numpy, multi-rank alt tiles against the cubic product")
    args = ap.parse_args()
    dist = Dist()
    try:
        if args.impl == "reference":
            try:
                run_reference(args, dist)
            except Exception as e:  # e.g. oracle/_ref not built on this box: say so, exit 0
                if dist.rank == 0:
                    print(json.dumps({"impl": "reference", "unavailable": f"{type(e).__name__}: {e}"}), flush=True)
        else:
            run_ours(args, dist)
    finally:
        dist.close()


if __name__ == "__main__":
    main()
