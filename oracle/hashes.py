"""ctypes loader for the C hash oracle (TEST INFRASTRUCTURE)."""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "hash_oracle.c")
OUT = os.path.join(HERE, "_build", "liboracle.so")


def build() -> str:
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    if not os.path.exists(OUT) or os.path.getmtime(OUT) < os.path.getmtime(SRC):
        subprocess.run(["gcc", "-O2", "-shared", "-fPIC", "-o", OUT, SRC], check=True)
    return OUT


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        _lib.oracle_prefix_hashes.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p,
                                              C.c_void_p]
        _lib.oracle_pixel_digest.argtypes = [C.c_void_p, C.c_int64, C.c_void_p]
        _lib.oracle_xxh64.argtypes = [C.c_void_p, C.c_int64, C.c_uint64]
        _lib.oracle_xxh64.restype = C.c_uint64
        _lib.oracle_kv_checksum.argtypes = [C.c_void_p, C.c_int64, C.c_void_p, C.c_int64,
                                            C.c_int64, C.c_int64]
        _lib.oracle_kv_checksum.restype = C.c_uint64
    return _lib


def xxh64(data: bytes, seed: int = 0) -> int:
    buf = np.frombuffer(bytes(data), np.uint8) if len(data) else np.zeros(1, np.uint8)
    return int(lib().oracle_xxh64(buf.ctypes.data, len(data), seed & (2 ** 64 - 1)))


def kv_checksum(planes: np.ndarray, rows, n_rows: int) -> int:
    """planes: [L, 2, slots, row] array (any dtype, C-contiguous); rows: int32
    slot of logical row i, or None (identity).  Same definition as
    emm_kv_checksum (include/emm.h)."""
    planes = np.ascontiguousarray(planes)
    L = planes.shape[0]
    stride = planes.strides[1]
    row_bytes = planes.shape[3] * planes.itemsize
    r = None if rows is None else np.ascontiguousarray(rows, dtype=np.int32)
    return int(lib().oracle_kv_checksum(planes.ctypes.data, stride,
                                        None if r is None else r.ctypes.data, int(n_rows),
                                        row_bytes, L))


def prefix_hashes(keys, weights):
    keys = np.ascontiguousarray(keys, dtype=np.uint64)
    w = np.ascontiguousarray(weights, dtype=np.int64)
    h0 = np.empty(len(keys), np.uint64)
    h1 = np.empty(len(keys), np.uint64)
    lib().oracle_prefix_hashes(keys.ctypes.data, w.ctypes.data, len(keys), h0.ctypes.data,
                               h1.ctypes.data)
    return h0, h1


def pixel_digest(data) -> tuple[int, int]:
    b = np.ascontiguousarray(np.frombuffer(bytes(data), dtype=np.uint8)
                             if not isinstance(data, np.ndarray) else data.reshape(-1),
                             dtype=np.uint8)
    out = np.empty(2, np.uint64)
    lib().oracle_pixel_digest(b.ctypes.data, b.size, out.ctypes.data)
    return int(out[0]), int(out[1])
