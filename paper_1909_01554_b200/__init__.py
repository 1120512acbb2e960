"""B200-native Boolean / GF(2) bit-matrix multiplication engine.

Python mirror of the reference's `bmm::` operator API for the product path
(reference proj/include/bmm/engine.hpp, bitmatrix.hpp): the same names,
argument meaning and exception types, all computed through the C ABI in
include/bmmgpu.h (libbmmgpu.so, sm_100a kernels).  There is no CPU fallback:
if the native library or a CUDA device is missing, calls raise.

The C++ drop-in of the same API is include/bmm/*.hpp + libbmm_b200.so.
"""
from __future__ import annotations

import ctypes
import enum
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
LIB_PATH = _HERE / "libbmmgpu.so"
HOST_LIB_PATH = _HERE / "libbmm_b200.so"

__all__ = [
    "Semiring", "Algo", "Kernel", "LayerPlan", "BitMatrix", "ShapeError", "FormatError", "EngineError",
    "multiply_cubic", "multiply", "lib", "device_count", "granularity", "read_bmm1", "write_bmm1", "PinnedWords",
]


class ShapeError(RuntimeError):
    """Dimensions do not fit the operation (bmm::ShapeError)."""


class FormatError(RuntimeError):
    """Invalid BMM1 contents (bmm::FormatError)."""


class EngineError(RuntimeError):
    """CUDA / device failure inside the engine (no CPU fallback exists)."""


class Semiring(enum.IntEnum):
    BooleanOrAnd = 0
    Gf2XorAnd = 1


class Algo(enum.IntEnum):
    Cubic = 0
    StrassenWinograd = 1
    AltSelfInverse = 2
    AltChaining = 3


class Kernel(enum.IntEnum):
    AUTO = 0
    LOP3 = 1
    UMMA_F4 = 2


class _Opts(ctypes.Structure):
    _fields_ = [("device_mask", ctypes.c_uint32), ("kernel", ctypes.c_int32), ("accumulate", ctypes.c_int32),
                ("leaf_log2", ctypes.c_int32), ("timing_ms", ctypes.POINTER(ctypes.c_double)),
                ("device_budget", ctypes.c_uint64), ("force_streaming", ctypes.c_int32),
                ("reserved", ctypes.c_int32)]


class _Plan(ctypes.Structure):
    _fields_ = [("d_host", ctypes.c_int32), ("d_serial", ctypes.c_int32), ("d_parallel", ctypes.c_int32),
                ("d_inner", ctypes.c_int32), ("workers", ctypes.c_int32)]


_u64p = ctypes.POINTER(ctypes.c_uint64)
_lib: ctypes.CDLL | None = None


def lib() -> ctypes.CDLL:
    """The loaded libbmmgpu.so (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise EngineError(f"{LIB_PATH} is missing: run `python __graft_entry__.py` / build() first; "
                              "the engine has no CPU fallback")
        L = ctypes.CDLL(str(LIB_PATH))
        u64, i32, vp = ctypes.c_uint64, ctypes.c_int32, ctypes.c_void_p
        L.bmmgpu_cubic.argtypes = [vp, vp, vp, u64, u64, u64, i32, ctypes.POINTER(_Opts)]
        L.bmmgpu_multiply.argtypes = [vp, vp, vp, u64, i32, ctypes.POINTER(_Plan), i32, ctypes.POINTER(_Opts)]
        L.bmmgpu_basis_change.argtypes = [vp, u64, i32, i32, i32, i32]
        L.bmmgpu_dev_granularity.argtypes = [i32, _u64p, _u64p, _u64p]
        L.bmmgpu_dev_transpose.argtypes = [vp, u64, u64, u64, vp, u64, u64, vp]
        L.bmmgpu_dev_cubic.argtypes = [vp, u64, vp, u64, vp, u64, u64, u64, u64, i32, i32, i32, vp]
        L.bmmgpu_dev_multiply.argtypes = [vp, u64, vp, u64, vp, u64, u64, i32, i32, i32, vp]
        L.bmmgpu_dev_cubic_batched.argtypes = [vp, u64, u64, vp, u64, u64, vp, u64, u64, u64, u64, u64, u64, i32,
                                               i32, i32, vp]
        L.bmmgpu_slab_rows.argtypes = [u64, ctypes.c_uint32, ctypes.c_uint32, u64, _u64p, _u64p]
        L.bmmgpu_slab_rows.restype = ctypes.c_int
        L.bmmgpu_dev_fold.argtypes = [vp, u64, vp, u64, u64, u64, i32, vp]
        L.bmmgpu_dev_fold.restype = ctypes.c_int
        L.bmmgpu_multiply_alt.argtypes = [vp, vp, vp, i32, i32, ctypes.POINTER(_Opts)]
        L.bmmgpu_multiply_alt.restype = ctypes.c_int
        L.bmmgpu_last_copy_bytes.argtypes = [_u64p, _u64p]
        L.bmmgpu_last_copy_bytes.restype = ctypes.c_int
        L.bmmgpu_block_timer.argtypes = [i32]
        L.bmmgpu_block_timer.restype = ctypes.c_int
        L.bmmgpu_block_timer_read.argtypes = [ctypes.POINTER(ctypes.c_double), _u64p]
        L.bmmgpu_block_timer_read.restype = ctypes.c_int
        L.bmmgpu_last_launch_count.restype = u64
        L.bmmgpu_dev_multiply_partial.argtypes = [vp, u64, vp, u64, vp, u64, u64, i32, i32, ctypes.c_uint32,
                                                  ctypes.c_uint32, i32, i32, vp]
        L.bmmgpu_dev_multiply_partial.restype = ctypes.c_int
        L.bmmgpu_host_levels.argtypes = [u64, ctypes.c_uint32, i32]
        L.bmmgpu_host_levels.restype = ctypes.c_int
        L.bmmgpu_bmm1_info.argtypes = [ctypes.c_char_p, _u64p, _u64p]
        L.bmmgpu_bmm1_info.restype = ctypes.c_int
        L.bmmgpu_bmm1_read.argtypes = [ctypes.c_char_p, vp, u64, i32]
        L.bmmgpu_bmm1_read.restype = ctypes.c_int
        L.bmmgpu_bmm1_write.argtypes = [ctypes.c_char_p, u64, u64, vp, i32]
        L.bmmgpu_bmm1_write.restype = ctypes.c_int
        L.bmmgpu_host_alloc.argtypes = [u64, ctypes.POINTER(ctypes.c_void_p)]
        L.bmmgpu_host_alloc.restype = ctypes.c_int
        L.bmmgpu_host_free.argtypes = [vp]
        L.bmmgpu_host_free.restype = ctypes.c_int
        L.bmmgpu_mem_info.argtypes = [i32, _u64p, _u64p]
        L.bmmgpu_mem_info.restype = ctypes.c_int
        L.bmmgpu_init.argtypes = [ctypes.c_uint32, u64]
        L.bmmgpu_init.restype = ctypes.c_int
        L.bmmgpu_multiply_panels.argtypes = [vp, vp, vp, u64, i32, i32, u64, u64, ctypes.POINTER(_Opts)]
        L.bmmgpu_multiply_panels.restype = ctypes.c_int
        L.bmmgpu_layout.argtypes = [vp, vp, u64, u64, i32, ctypes.POINTER(_Opts)]
        L.bmmgpu_layout.restype = ctypes.c_int
        L.bmmgpu_dev_layout.argtypes = [vp, vp, u64, u64, i32, vp]
        L.bmmgpu_dev_layout.restype = ctypes.c_int
        L.bmmgpu_debug_k2_clock.argtypes = [_u64p, _u64p]
        L.bmmgpu_debug_k2_clock.restype = ctypes.c_int
        L.bmmgpu_debug_ts_launches.argtypes = [_u64p]
        L.bmmgpu_debug_ts_launches.restype = ctypes.c_int
        L.bmmgpu_kernel64.argtypes = [vp, vp, vp, i32]
        L.bmmgpu_kernel64.restype = ctypes.c_int
        L.bmmgpu_debug_wave_stats.argtypes = [_u64p, _u64p]
        L.bmmgpu_debug_wave_stats.restype = ctypes.c_int
        L.bmmgpu_device_count.restype = ctypes.c_int
        L.bmmgpu_last_error.restype = ctypes.c_char_p
        L.bmmgpu_version.restype = ctypes.c_char_p
        for name in ("bmmgpu_cubic", "bmmgpu_multiply", "bmmgpu_basis_change", "bmmgpu_dev_granularity",
                     "bmmgpu_dev_transpose", "bmmgpu_dev_cubic", "bmmgpu_dev_multiply", "bmmgpu_dev_cubic_batched"):
            getattr(L, name).restype = ctypes.c_int
        _lib = L
    return _lib


def _check(status: int) -> None:
    if status == 0:
        return
    msg = lib().bmmgpu_last_error().decode(errors="replace")
    if status == 3:
        raise ShapeError(msg)
    if status == 4:
        raise FormatError(msg)
    if status == 1:
        raise ValueError(msg)  # std::invalid_argument
    raise EngineError(msg)


def init(device_mask: int = 0, reserve_bytes: int = 0) -> None:
    """bmmgpu_init: load every kernel and warm the stream / memory pools of the devices in
    `device_mask` (0: device 0), optionally reserving `reserve_bytes` of HBM in the pool."""
    _check(lib().bmmgpu_init(device_mask, reserve_bytes))


def device_count() -> int:
    return int(lib().bmmgpu_device_count())


def slab_rows(m: int, parts: int, index: int, gran: int = 64) -> tuple[int, int]:
    """Output-row slab of part `index` of `parts` (bmmgpu_slab_rows): the one
    partition rule shared by the multi-device driver and the multi-rank bench."""
    lo, hi = ctypes.c_uint64(), ctypes.c_uint64()
    _check(lib().bmmgpu_slab_rows(m, parts, index, gran, ctypes.byref(lo), ctypes.byref(hi)))
    return lo.value, hi.value


def granularity(kernel: int = Kernel.AUTO) -> tuple[int, int, int]:
    """(row granule of A, row granule of Bt, K granule in bits) of a panel-product kernel."""
    gm, gn, gk = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint64()
    _check(lib().bmmgpu_dev_granularity(int(kernel), ctypes.byref(gm), ctypes.byref(gn), ctypes.byref(gk)))
    return gm.value, gn.value, gk.value


@dataclass
class LayerPlan:
    """bmm::LayerPlan (reference plan.hpp:26-44)."""
    d_host: int = 0
    d_serial: int = 0
    d_parallel: int = 0
    d_inner: int = 1
    workers: int = 1

    def depth(self) -> int:
        return self.d_host + self.d_serial + self.d_parallel

    def matrix_dim(self) -> int:
        return 64 << self.depth()

    @staticmethod
    def auto_plan(n: int, workers: int) -> "LayerPlan":
        """Up to three parallel levels, the rest serial (reference engine.cpp:13-22)."""
        if n < 64 or n & (n - 1):
            raise ShapeError("matrix dimension must be 64 * 2^k")
        k = n.bit_length() - 1 - 6
        dp = min(3, k)
        return LayerPlan(0, k - dp, dp, 1, max(1, workers))


@dataclass(eq=False)
class BitMatrix:
    """bmm::BitMatrix (reference bitmatrix.hpp:31-52): row-major packed bits."""
    rows: int
    cols: int
    words: np.ndarray = field(repr=False)

    def words_per_row(self) -> int:
        return (self.cols + 63) // 64

    @staticmethod
    def zeros(rows: int, cols: int) -> "BitMatrix":
        return BitMatrix(rows, cols, np.zeros(rows * ((cols + 63) // 64), dtype=np.uint64))

    @staticmethod
    def random(rows: int, cols: int, seed: int) -> "BitMatrix":
        """std::mt19937_64(seed), one draw per word, row-major, tail masked
        (reference bitmatrix.cpp:64-77) -- via the drop-in C++ library."""
        m = BitMatrix.zeros(rows, cols)
        if m.words.size:
            _host().bmmh_random(rows, cols, ctypes.c_uint64(seed), m.words.ctypes.data)
        return m

    def row(self, i: int) -> np.ndarray:
        w = self.words_per_row()
        return self.words[i * w:(i + 1) * w]

    def get(self, i: int, j: int) -> bool:
        if i >= self.rows or j >= self.cols or i < 0 or j < 0:
            raise ShapeError("bit index out of range")
        return bool((int(self.words[i * self.words_per_row() + j // 64]) >> (j % 64)) & 1)

    def set(self, i: int, j: int, value: bool) -> None:
        if i >= self.rows or j >= self.cols or i < 0 or j < 0:
            raise ShapeError("bit index out of range")
        k = i * self.words_per_row() + j // 64
        bit = np.uint64(1 << (j % 64))
        self.words[k] = (self.words[k] | bit) if value else (self.words[k] & ~bit)

    def __eq__(self, other: object) -> bool:
        return (isinstance(other, BitMatrix) and self.rows == other.rows and self.cols == other.cols
                and np.array_equal(self.words, other.words))


def read_bmm1(path: str, out: np.ndarray | None = None, threads: int = 0) -> BitMatrix:
    """bmm::read_bmm1 (reference bitmatrix.cpp:187-233): the same checks and messages
    (FormatError), read with parallel positioned I/O straight into `out` when given (e.g.
    page-locked memory from `pinned_words`, so the words go to the GPU without a copy)."""
    rows, cols = ctypes.c_uint64(), ctypes.c_uint64()
    L = lib()
    if L.bmmgpu_bmm1_info(str(path).encode(), ctypes.byref(rows), ctypes.byref(cols)) != 0:
        raise FormatError(L.bmmgpu_last_error().decode())
    n = rows.value * ((cols.value + 63) // 64)
    words = np.zeros(n, dtype=np.uint64) if out is None else out[:n]
    if words.size != n or not words.flags["C_CONTIGUOUS"]:
        raise ValueError(f"destination needs {n} contiguous words")
    _check(L.bmmgpu_bmm1_read(str(path).encode(), words.ctypes.data, n, threads))
    return BitMatrix(rows.value, cols.value, words)


def write_bmm1(m: BitMatrix, path: str, threads: int = 0) -> None:
    """bmm::write_bmm1 (reference bitmatrix.cpp:218-233), parallel positioned writes."""
    L = lib()
    _check(L.bmmgpu_bmm1_write(str(path).encode(), m.rows, m.cols, m.words.ctypes.data, threads))


class Operand(enum.IntEnum):
    """bmm::Operand (reference bitmatrix.hpp): right operands store their blocks transposed."""
    Left = 0
    Right = 1
    Result = 2


LAYOUT_TRANSPOSE_BLOCKS64, LAYOUT_TO_INTERLEAVED, LAYOUT_TO_INTERLEAVED_RIGHT = 0, 1, 2
LAYOUT_FROM_INTERLEAVED, LAYOUT_FROM_INTERLEAVED_RIGHT = 3, 4


def layout(src: np.ndarray, dst: np.ndarray, rows: int, cols: int, op: int, device_mask: int = 0) -> None:
    """bmmgpu_layout: one of the layout conversions on host buffers (pinned or pageable),
    streamed through the GPU (csrc/layout.cu)."""
    if src.dtype != np.uint64 or dst.dtype != np.uint64 or not (src.flags["C_CONTIGUOUS"] and dst.flags["C_CONTIGUOUS"]):
        raise ValueError("layout needs C-contiguous uint64 buffers")
    need = rows * ((cols + 63) // 64)
    if src.size < need or dst.size < need:
        raise ValueError(f"layout needs {need} words in each buffer")
    o = _opts(0, device_mask=device_mask)
    _check(lib().bmmgpu_layout(src.ctypes.data, dst.ctypes.data, rows, cols, int(op), ctypes.byref(o)))


def transpose_blocks64(m: BitMatrix) -> None:
    """bmm::transpose_blocks64 (reference bitmatrix.cpp:97-110), in place, on the GPU."""
    if m.rows % 64 or m.cols % 64:
        raise ShapeError("block transpose needs dimensions divisible by 64")
    if m.words.size:
        layout(m.words, m.words, m.rows, m.cols, LAYOUT_TRANSPOSE_BLOCKS64)


def to_interleaved(m: BitMatrix, plan: LayerPlan, which: Operand, out: np.ndarray | None = None) -> np.ndarray:
    """bmm::to_interleaved (reference bitmatrix.cpp:112-148): the words of the
    BitVectorTensor with modes [4]*depth + [4096], on the GPU."""
    n = plan.matrix_dim()
    if m.rows != n or m.cols != n:
        raise ShapeError("matrix does not match plan dimension")
    t = np.empty(n * n // 64, dtype=np.uint64) if out is None else out
    layout(_contig(m), t, n, n, LAYOUT_TO_INTERLEAVED_RIGHT if which == Operand.Right else LAYOUT_TO_INTERLEAVED)
    return t


def from_interleaved(t: np.ndarray, plan: LayerPlan, which: Operand, out: np.ndarray | None = None) -> BitMatrix:
    """bmm::from_interleaved (reference bitmatrix.cpp:150-173), on the GPU."""
    n = plan.matrix_dim()
    if t.size != n * n // 64:
        raise ShapeError("tensor does not match plan shape")
    w = np.empty(n * n // 64, dtype=np.uint64) if out is None else out
    layout(np.ascontiguousarray(t, dtype=np.uint64), w, n, n,
           LAYOUT_FROM_INTERLEAVED_RIGHT if which == Operand.Right else LAYOUT_FROM_INTERLEAVED)
    return BitMatrix(n, n, w)


class PinnedWords:
    """Page-locked host words (bmmgpu_host_alloc): `.words` is a numpy view; free() or
    garbage collection releases them."""

    def __init__(self, n: int) -> None:
        self._p = ctypes.c_void_p()
        _check(lib().bmmgpu_host_alloc(max(8, 8 * n), ctypes.byref(self._p)))
        self.words = np.ctypeslib.as_array((ctypes.c_uint64 * max(1, n)).from_address(self._p.value))[:n]

    def free(self) -> None:
        if self._p.value:
            self.words = None
            lib().bmmgpu_host_free(self._p)
            self._p = ctypes.c_void_p()

    def __del__(self) -> None:
        try:
            self.free()
        except Exception:
            pass


_host_lib: ctypes.CDLL | None = None


def _host() -> ctypes.CDLL:
    global _host_lib
    if _host_lib is None:
        if not HOST_LIB_PATH.exists():
            raise EngineError(f"{HOST_LIB_PATH} is missing: run build() first")
        L = ctypes.CDLL(str(HOST_LIB_PATH))
        L.bmmh_random.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_void_p]
        L.bmmh_random.restype = None
        L.bmmh_random_rows.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64,
                                       ctypes.c_void_p]
        L.bmmh_random_rows.restype = None
        _host_lib = L
    return _host_lib


def random_rows_into(out: np.ndarray, cols: int, seed: int, row_begin: int, row_end: int) -> None:
    """Rows [row_begin, row_end) of BitMatrix.random(*, cols, seed) into `out`
    (any C-contiguous 8-byte buffer, e.g. pinned host memory)."""
    if row_end > row_begin:
        _host().bmmh_random_rows(cols, seed, row_begin, row_end, out.ctypes.data)


def _opts(kernel: int, leaf_log2: int = 0, timing: ctypes.c_double | None = None, device_mask: int = 0,
          accumulate: bool = False, device_budget: int = 0, force_streaming: bool = False) -> _Opts:
    o = _Opts()
    o.device_mask = device_mask
    o.kernel = int(kernel)
    o.accumulate = int(accumulate)
    o.leaf_log2 = int(leaf_log2)
    o.timing_ms = ctypes.pointer(timing) if timing is not None else ctypes.POINTER(ctypes.c_double)()
    o.device_budget = int(device_budget)
    o.force_streaming = int(force_streaming)
    return o


def _contig(m: BitMatrix) -> np.ndarray:
    w = np.ascontiguousarray(m.words, dtype=np.uint64)
    if w.size != m.rows * m.words_per_row():
        raise ShapeError("word storage does not match the shape")
    return w


def kernel64(a: np.ndarray, b_transposed: np.ndarray, ring: Semiring) -> np.ndarray:
    """One 64 x 64 block product in the reference's operand form (engine.cpp:34-56):
    out[i] bit k = dot(row i of a, column k of B), B given column-major (word k = column k)."""
    aw = np.ascontiguousarray(a, dtype=np.uint64)
    bw = np.ascontiguousarray(b_transposed, dtype=np.uint64)
    if aw.size != 64 or bw.size != 64:
        raise ValueError("kernel64 takes 64 words per operand")
    out = np.zeros(64, dtype=np.uint64)
    _check(lib().bmmgpu_kernel64(aw.ctypes.data, bw.ctypes.data, out.ctypes.data, int(ring)))
    return out


def multiply_cubic(a: BitMatrix, b: BitMatrix, ring: Semiring, workers: int = 1, *, kernel: int = Kernel.AUTO,
                   device_mask: int = 0, out: BitMatrix | None = None, accumulate: bool = False,
                   timing: ctypes.c_double | None = None, device_budget: int = 0,
                   force_streaming: bool = False) -> BitMatrix:
    """bmm::multiply_cubic (reference engine.cpp:132-144) on the GPU.

    With `accumulate`, `out` is XOR/OR-folded with A.B (K-split integration).
    `device_budget` (bytes per device) / `force_streaming` select the
    out-of-core driver (csrc/stream.cu) for products larger than HBM."""
    if a.cols != b.rows:
        raise ShapeError("inner dimensions differ")
    c = out if out is not None else BitMatrix.zeros(a.rows, b.cols)
    if (c.rows, c.cols) != (a.rows, b.cols):
        raise ShapeError("output shape mismatch")
    aw, bw = _contig(a), _contig(b)
    _check(lib().bmmgpu_cubic(aw.ctypes.data, bw.ctypes.data, c.words.ctypes.data, a.rows, a.cols, b.cols,
                              int(ring), ctypes.byref(_opts(kernel, 0, timing, device_mask, accumulate,
                                                            device_budget, force_streaming))))
    return c


def multiply(a: BitMatrix, b: BitMatrix, algo: Algo, plan: LayerPlan, ring: Semiring, *,
             kernel: int = Kernel.AUTO, leaf_log2: int = 0, timing: ctypes.c_double | None = None,
             out: BitMatrix | None = None, device_mask: int = 0, device_budget: int = 0,
             force_streaming: bool = False) -> BitMatrix:
    """bmm::multiply (reference engine.cpp:351-382) on the GPU.  `out` may supply
    the result storage (e.g. pinned host memory).  Operands beyond `device_budget` (0: the
    free HBM) or `force_streaming` run out of core: output tiles of alternative-basis
    block products streamed from host memory (csrc/alt_tiles.cu)."""
    if algo == Algo.Cubic:
        return multiply_cubic(a, b, ring, plan.workers, kernel=kernel, timing=timing)
    if ring == Semiring.BooleanOrAnd:
        raise ValueError("the Boolean semiring has no subtraction, so cancellation-based fast algorithms are "
                         "unsound over it; use the cubic algorithm")
    if a.rows != a.cols or b.rows != b.cols or a.rows != b.rows:
        raise ShapeError("fast algorithms need equal square operands")
    n = a.rows
    if n < 64 or n & (n - 1):
        raise ShapeError("fast algorithms need n = 64 * 2^k")
    if (plan.matrix_dim() != n or plan.d_host < 0 or plan.d_serial < 0 or plan.d_parallel < 0
            or plan.d_inner != 1 or plan.workers < 1):
        raise ValueError("layer plan does not match the operands")
    c = out if out is not None else BitMatrix.zeros(n, n)
    if (c.rows, c.cols) != (n, n) or c.words.size != n * (n // 64):
        raise ShapeError("output shape mismatch")
    p = _Plan(plan.d_host, plan.d_serial, plan.d_parallel, plan.d_inner, plan.workers)
    _check(lib().bmmgpu_multiply(_contig(a).ctypes.data, _contig(b).ctypes.data, c.words.ctypes.data, n, int(algo),
                                 ctypes.byref(p), int(ring),
                                 ctypes.byref(_opts(kernel, leaf_log2, timing, device_mask=device_mask,
                                                    device_budget=device_budget, force_streaming=force_streaming))))
    return c
