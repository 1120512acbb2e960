"""Parity oracle -- TEST INFRASTRUCTURE ONLY.

`Oracle` wraps oracle/liboracle.so, the plain-C restatement of the reference
product path (oracle/bmm_oracle.c, each function citing the reference
file:line it restates).  `Reference` wraps oracle/_ref/libbmmref.so, the
UNMODIFIED reference bmm_core compiled from /root/reference/proj/src by
oracle/Makefile.  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import this package; the product
(paper_1909_01554_b200) never does.
"""
from __future__ import annotations

import ctypes
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ORACLE_SO = HERE / "liboracle.so"
REF_SO = HERE / "_ref" / "libbmmref.so"
REF_SRC = Path("/root/reference/proj")

_u64 = ctypes.c_uint64
_vp = ctypes.c_void_p
_i32 = ctypes.c_int


def build(ref: bool = True) -> None:
    """Compile the C restatement and, when the reference sources are present, oracle/_ref."""
    targets = [str(ORACLE_SO)]
    if ref and REF_SRC.exists():
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", str(HERE), *targets], check=True)


def _p(a: np.ndarray) -> int:
    assert a.dtype == np.uint64 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data


class Oracle:
    """The C restatement (bmm_oracle.c)."""

    def __init__(self) -> None:
        if not ORACLE_SO.exists():
            build(ref=False)
        L = ctypes.CDLL(str(ORACLE_SO))
        L.bmmo_random.argtypes = [_u64, _u64, _u64, _vp]
        L.bmmo_random.restype = None
        L.bmmo_transpose_blocks64.argtypes = [_u64, _u64, _vp]
        L.bmmo_multiply_cubic.argtypes = [_vp, _vp, _vp, _u64, _u64, _u64, _i32]
        L.bmmo_kernel64.argtypes = [_vp, _vp, _vp, _i32]
        L.bmmo_kernel64.restype = None
        L.bmmo_to_interleaved.argtypes = [_i32, _i32, _vp, _vp]
        L.bmmo_to_interleaved.restype = None
        L.bmmo_from_interleaved.argtypes = [_i32, _i32, _vp, _vp]
        L.bmmo_from_interleaved.restype = None
        L.bmmo_interleaved_bit_index.argtypes = [_i32, _i32, _u64, _u64]
        L.bmmo_interleaved_bit_index.restype = _u64
        L.bmmo_basis_change.argtypes = [_vp, _u64, _i32, _i32]
        L.bmmo_basis_change.restype = None
        L.bmmo_multiply_alt.argtypes = [_vp, _vp, _vp, _i32]
        L.bmmo_multiply_alt.restype = None
        L.bmmo_multiply_alt_si.argtypes = [_vp, _vp, _vp, _i32]
        L.bmmo_multiply_alt_si.restype = None
        L.bmmo_fnv1a64.argtypes = [_vp, _u64]
        L.bmmo_fnv1a64.restype = _u64
        L.bmmo_popcount.argtypes = [_vp, _u64]
        L.bmmo_popcount.restype = _u64
        L.bmmo_mt64_state_size.restype = _u64
        L.bmmo_mt64_seed.argtypes = [_vp, _u64]
        L.bmmo_mt64_seed.restype = None
        L.bmmo_mt64_next.argtypes = [_vp]
        L.bmmo_mt64_next.restype = _u64
        self.L = L

    def random(self, rows: int, cols: int, seed: int) -> np.ndarray:
        w = np.zeros(rows * ((cols + 63) // 64), dtype=np.uint64)
        if w.size:
            self.L.bmmo_random(rows, cols, seed, _p(w))
        return w

    def mt64(self, seed: int, count: int) -> list[int]:
        st = ctypes.create_string_buffer(int(self.L.bmmo_mt64_state_size()))
        self.L.bmmo_mt64_seed(st, seed)
        return [int(self.L.bmmo_mt64_next(st)) for _ in range(count)]

    def multiply_cubic(self, a: np.ndarray, b: np.ndarray, m: int, k: int, n: int, ring: int) -> np.ndarray:
        c = np.zeros(m * ((n + 63) // 64), dtype=np.uint64)
        rc = self.L.bmmo_multiply_cubic(_p(a), _p(b), _p(c), m, k, n, ring)
        assert rc == 0
        return c

    def kernel64(self, a: np.ndarray, bt: np.ndarray, ring: int) -> np.ndarray:
        out = np.zeros(64, dtype=np.uint64)
        self.L.bmmo_kernel64(_p(a), _p(bt), _p(out), ring)
        return out

    def transpose_blocks64(self, rows: int, cols: int, w: np.ndarray) -> np.ndarray:
        w = w.copy()
        assert self.L.bmmo_transpose_blocks64(rows, cols, _p(w)) == 0
        return w

    def to_interleaved(self, depth: int, which: int, m: np.ndarray) -> np.ndarray:
        t = np.zeros_like(m)
        self.L.bmmo_to_interleaved(depth, which, _p(m), _p(t))
        return t

    def from_interleaved(self, depth: int, which: int, t: np.ndarray) -> np.ndarray:
        m = np.zeros_like(t)
        self.L.bmmo_from_interleaved(depth, which, _p(t), _p(m))
        return m

    def interleaved_bit_index(self, depth: int, which: int, i: int, j: int) -> int:
        return int(self.L.bmmo_interleaved_bit_index(depth, which, i, j))

    def basis_change(self, v: np.ndarray, levels: int, which: int) -> np.ndarray:
        v = v.copy()
        self.L.bmmo_basis_change(_p(v), v.size, levels, which)
        return v

    def multiply_alt(self, a_hat: np.ndarray, b_hat: np.ndarray, depth: int) -> np.ndarray:
        c = np.zeros_like(a_hat)
        self.L.bmmo_multiply_alt(_p(a_hat), _p(b_hat), _p(c), depth)
        return c

    def multiply_alt_si(self, a: np.ndarray, b: np.ndarray, depth: int) -> np.ndarray:
        c = np.zeros_like(a)
        self.L.bmmo_multiply_alt_si(_p(a), _p(b), _p(c), depth)
        return c

    def fnv1a64(self, w: np.ndarray) -> int:
        w = np.ascontiguousarray(w, dtype=np.uint64)
        return int(self.L.bmmo_fnv1a64(_p(w), w.size))

    def popcount(self, w: np.ndarray) -> int:
        w = np.ascontiguousarray(w, dtype=np.uint64)
        return int(self.L.bmmo_popcount(_p(w), w.size))


class Reference:
    """The unmodified reference bmm_core (oracle/_ref/libbmmref.so)."""

    def __init__(self) -> None:
        if not REF_SO.exists():
            if REF_SRC.exists():
                build(ref=True)
            else:
                raise FileNotFoundError(f"{REF_SO} not built and {REF_SRC} absent")
        L = ctypes.CDLL(str(REF_SO))
        L.bmmref_random.argtypes = [_u64, _u64, _u64, _vp]
        L.bmmref_random.restype = None
        L.bmmref_multiply_cubic.argtypes = [_vp, _vp, _vp, _u64, _u64, _u64, _i32, _i32, _vp]
        L.bmmref_multiply.argtypes = [_vp, _vp, _vp, _u64, _i32, _i32, _i32, _i32, _i32, _i32, _vp]
        L.bmmref_auto_plan.argtypes = [_u64, _i32, _vp]
        L.bmmref_transpose_blocks64.argtypes = [_u64, _u64, _vp]
        L.bmmref_to_interleaved.argtypes = [_i32, _i32, _vp, _vp]
        L.bmmref_from_interleaved.argtypes = [_i32, _i32, _vp, _vp]
        L.bmmref_basis_change.argtypes = [_vp, _i32, _i32, _i32]
        L.bmmref_multiply_alt.argtypes = [_vp, _vp, _vp, _i32, _i32, _i32, _i32]
        L.bmmref_read_bmm1.argtypes = [ctypes.c_char_p, _vp, _vp, _vp]
        L.bmmref_write_bmm1.argtypes = [ctypes.c_char_p, _u64, _u64, _vp]
        L.bmmref_coordinate.argtypes = [_vp, _vp, _vp, _i32, _i32, _i32, _i32, _i32, _vp]
        L.bmmref_kernel64.argtypes = [_vp, _vp, _vp, _i32]
        L.bmmref_kernel64.restype = None
        L.bmmref_predicted_additions.argtypes = [_i32, _i32, _i32]
        L.bmmref_predicted_additions.restype = _u64
        L.bmmref_last_error.restype = ctypes.c_char_p
        self.L = L

    def _ok(self, rc: int) -> None:
        if rc != 0:
            raise RuntimeError(f"reference rc={rc}: {self.L.bmmref_last_error().decode()}")

    def random(self, rows: int, cols: int, seed: int) -> np.ndarray:
        w = np.zeros(rows * ((cols + 63) // 64), dtype=np.uint64)
        if w.size:
            self.L.bmmref_random(rows, cols, seed, _p(w))
        return w

    def multiply_cubic(self, a, b, m, k, n, ring, workers=1, counts=False):
        c = np.zeros(m * ((n + 63) // 64), dtype=np.uint64)
        cnt = np.zeros(4, dtype=np.uint64)
        self._ok(self.L.bmmref_multiply_cubic(_p(a), _p(b), _p(c), m, k, n, ring, workers,
                                              _p(cnt) if counts else None))
        return (c, cnt) if counts else c

    def multiply(self, a, b, n, algo, d_host, d_serial, d_parallel, workers=1, ring=1, counts=False):
        c = np.zeros(n * (n // 64), dtype=np.uint64)
        cnt = np.zeros(4, dtype=np.uint64)
        self._ok(self.L.bmmref_multiply(_p(a), _p(b), _p(c), n, algo, d_host, d_serial, d_parallel, workers, ring,
                                        _p(cnt) if counts else None))
        return (c, cnt) if counts else c

    def read_bmm1(self, path: str):
        rows, cols = ctypes.c_uint64(), ctypes.c_uint64()
        self._ok(self.L.bmmref_read_bmm1(path.encode(), ctypes.byref(rows), ctypes.byref(cols), None))
        w = np.zeros(rows.value * ((cols.value + 63) // 64), dtype=np.uint64)
        self._ok(self.L.bmmref_read_bmm1(path.encode(), ctypes.byref(rows), ctypes.byref(cols), _p(w)))
        return rows.value, cols.value, w

    def write_bmm1(self, path: str, rows: int, cols: int, words: np.ndarray) -> None:
        self._ok(self.L.bmmref_write_bmm1(path.encode(), rows, cols, _p(words)))

    def coordinate(self, a_hat, b_hat, d_host, d_serial, d_parallel, workers=1, scheme=1, counts=False):
        c = np.zeros_like(a_hat)
        cnt = np.zeros(4, dtype=np.uint64)
        self._ok(self.L.bmmref_coordinate(_p(a_hat), _p(b_hat), _p(c), d_host, d_serial, d_parallel, workers, scheme,
                                          _p(cnt) if counts else None))
        return (c, cnt) if counts else c

    def kernel64(self, a, bt, ring):
        out = np.zeros(64, dtype=np.uint64)
        self.L.bmmref_kernel64(_p(a), _p(bt), _p(out), ring)
        return out

    def transpose_blocks64(self, rows, cols, w):
        w = w.copy()
        self._ok(self.L.bmmref_transpose_blocks64(rows, cols, _p(w)))
        return w

    def to_interleaved(self, depth, which, m):
        t = np.zeros_like(m)
        self._ok(self.L.bmmref_to_interleaved(depth, which, _p(m), _p(t)))
        return t

    def from_interleaved(self, depth, which, t):
        m = np.zeros_like(t)
        self._ok(self.L.bmmref_from_interleaved(depth, which, _p(t), _p(m)))
        return m

    def basis_change(self, v, depth, which, scheme=1):
        v = v.copy()
        self._ok(self.L.bmmref_basis_change(_p(v), depth, which, scheme))
        return v

    def multiply_alt(self, a_hat, b_hat, d_serial, d_parallel, workers=1, scheme=1):
        c = np.zeros_like(a_hat)
        self._ok(self.L.bmmref_multiply_alt(_p(a_hat), _p(b_hat), _p(c), d_serial, d_parallel, workers, scheme))
        return c

    def predicted_additions(self, scheme, depth, part):
        return int(self.L.bmmref_predicted_additions(scheme, depth, part))


def fnv1a64_np(w: np.ndarray) -> int:
    """FNV-1a 64 over the little-endian bytes of a word array (numpy, for huge arrays use Oracle.fnv1a64)."""
    h = 0xcbf29ce484222325
    for byte in np.ascontiguousarray(w, dtype="<u8").view(np.uint8).tolist():
        h ^= byte
        h = (h * 0x100000001b3) & 0xFFFFFFFFFFFFFFFF
    return h
