"""CPU oracle for the COMET W4Ax path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The
product path (``paper_2410_12168_b200``) never imports it and shares no code
with it; see ``comet_oracle.c`` for the definitions and their citations into
PAPER.md (arXiv 2410.12168).

This module is argument marshalling around ``comet_oracle.c`` (numpy arrays
in, numpy arrays out) plus an on-demand gcc build of ``liboracle.so``.

Parity status: every function here is pinned by ``tests/test_oracle.py``
(hand-worked blocks, library routines, brute force, invariants).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "comet_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

OK, ERR_INPUT, ERR_SHAPE = 0, 1, 2


class OracleError(RuntimeError):
    pass


def build(force: bool = False) -> str:
    """Compile comet_oracle.c with gcc (-O2, OpenMP, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(
            ["gcc", "-O2", "-std=c11", "-fopenmp", "-fPIC", "-shared", "-fno-fast-math",
             "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = ctypes.CDLL(_LIB)
            P = ctypes.c_void_p
            i32, i64 = ctypes.c_int32, ctypes.c_int64
            L.oracle_half_to_float.argtypes = [ctypes.c_uint16]
            L.oracle_half_to_float.restype = ctypes.c_float
            L.oracle_double_to_half.argtypes = [ctypes.c_double]
            L.oracle_double_to_half.restype = ctypes.c_uint16
            L.oracle_quantize_block.argtypes = [P, i32, i32, P, P]
            L.oracle_quantize_block.restype = None
            L.oracle_pack_int4.argtypes = [P, i32, P]
            L.oracle_pack_int4.restype = None
            L.oracle_unpack_int4.argtypes = [P, i32, P]
            L.oracle_unpack_int4.restype = None
            L.oracle_quantize_act.argtypes = [P, i64, i32, i32, i32, P, P, P, i64, P, i64, P, i64]
            L.oracle_quantize_act.restype = i32
            L.oracle_pack_weight.argtypes = [P, i64, i32, i32, P, i32, P, P]
            L.oracle_pack_weight.restype = i32
            L.oracle_w4ax_gemm.argtypes = [P, i64, P, i64, P, i64, P, i32, i32, i32,
                                           P, P, i32, i32, P, i32, P, P, P]
            L.oracle_w4ax_gemm.restype = i32
            L.oracle_num_threads.argtypes = []
            L.oracle_num_threads.restype = i32
            _lib = L
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _check(rc):
    if rc != OK:
        raise OracleError({ERR_INPUT: "input error", ERR_SHAPE: "shape error"}.get(rc, rc))


def num_threads() -> int:
    return int(lib().oracle_num_threads())


# ---------------------------------------------------------------- fp16 ----
def half_to_float(h: int) -> float:
    return float(lib().oracle_half_to_float(int(h)))


def double_to_half_bits(d: float) -> int:
    return int(lib().oracle_double_to_half(float(d)))


# -------------------------------------------------------- quantization ----
def quantize_block(x: np.ndarray, qmax: int):
    """O3 on one block: returns (q int8[n], s float32)."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    q = np.zeros(x.size, np.int8)
    s = np.zeros(1, np.float32)
    lib().oracle_quantize_block(_ptr(x), x.size, int(qmax), _ptr(q), _ptr(s))
    return q, s[0]


def pack_int4(q: np.ndarray) -> np.ndarray:
    q = np.ascontiguousarray(q, dtype=np.int8).reshape(-1)
    out = np.zeros(q.size // 2, np.uint8)
    lib().oracle_pack_int4(_ptr(q), q.size, _ptr(out))
    return out


def unpack_int4(p: np.ndarray, n: int) -> np.ndarray:
    p = np.ascontiguousarray(p, dtype=np.uint8).reshape(-1)
    out = np.zeros(n, np.int8)
    lib().oracle_unpack_int4(_ptr(p), n, _ptr(out))
    return out


def plane_widths(bits, k: int = 128):
    bits = np.asarray(bits)
    n8 = int((bits == 8).sum())
    n4 = int((bits == 4).sum())
    return k * n8, k * n4  # K8, K4 (elements)


def ldsx_for(M: int) -> int:
    return (M + 3) // 4 * 4


def quantize_act(X: np.ndarray, bits, perm=None, k: int = 128):
    """FMPQ quantization of fp16 activations X [M x K].

    Returns (Xq8 int8 [M x K8], Xq4 uint8 [M x K4/2], Sx float32 [nb x ldsx])."""
    X = np.ascontiguousarray(X, dtype=np.float16)
    M, K = X.shape
    bits = np.ascontiguousarray(bits, dtype=np.uint8)
    K8, K4 = plane_widths(bits, k)
    ldsx = ldsx_for(M)
    Xq8 = np.zeros((M, K8), np.int8)
    Xq4 = np.zeros((M, K4 // 2), np.uint8)
    Sx = np.zeros((K // k, ldsx), np.float32)
    perm_a = None if perm is None else np.ascontiguousarray(perm, dtype=np.int32)
    rc = lib().oracle_quantize_act(_ptr(X.view(np.uint16)), K, M, K, k, _ptr(perm_a), _ptr(bits),
                                   _ptr(Xq8), max(K8, 1), _ptr(Xq4), max(K4 // 2, 1), _ptr(Sx), ldsx)
    _check(rc)
    return Xq8, Xq4, Sx


def pack_weight(W: np.ndarray, group: int = 128, perm=None):
    """INT4 weight packing of fp16 W [N x K]: returns (Wq uint8 [N x K/2], Sw float32 [K/group x N])."""
    W = np.ascontiguousarray(W, dtype=np.float16)
    N, K = W.shape
    Wq = np.zeros((N, K // 2), np.uint8)
    Sw = np.zeros((K // group, N), np.float32)
    perm_a = None if perm is None else np.ascontiguousarray(perm, dtype=np.int32)
    rc = lib().oracle_pack_weight(_ptr(W.view(np.uint16)), K, N, K, _ptr(perm_a), group, _ptr(Wq), _ptr(Sw))
    _check(rc)
    return Wq, Sw


def w4ax_gemm(Xq8, Xq4, Sx, bits, Wq, Sw, group: int = 128, k: int = 128, rows=None,
              want_y64: bool = False, want_acc: bool = False):
    """Y = dequant(Xq . Wq^T).  Returns dict with 'y' (float16 [R x N]) and
    optionally 'y64' (float64) and 'acc' (int32 [nb x R x N], logical units)."""
    Xq8 = np.ascontiguousarray(Xq8, dtype=np.int8)
    Xq4 = np.ascontiguousarray(Xq4, dtype=np.uint8)
    Sx = np.ascontiguousarray(Sx, dtype=np.float32)
    Wq = np.ascontiguousarray(Wq, dtype=np.uint8)
    Sw = np.ascontiguousarray(Sw, dtype=np.float32)
    bits = np.ascontiguousarray(bits, dtype=np.uint8)
    N = Wq.shape[0]
    K = Wq.shape[1] * 2
    M = max(Xq8.shape[0], Xq4.shape[0])  # both planes are [M x .] (width may be 0)
    nb = K // k
    rows_a = None if rows is None else np.ascontiguousarray(rows, dtype=np.int32)
    R = M if rows is None else rows_a.size
    y = np.zeros((R, N), np.uint16)
    y64 = np.zeros((R, N), np.float64) if want_y64 else None
    acc = np.zeros((nb, R, N), np.int32) if want_acc else None
    ld8 = max(Xq8.shape[1], 1)
    ld4 = max(Xq4.shape[1], 1)
    rc = lib().oracle_w4ax_gemm(_ptr(Xq8), ld8, _ptr(Xq4), ld4, _ptr(Sx), Sx.shape[1], _ptr(bits), M, K, k,
                                _ptr(Wq), _ptr(Sw), N, group, _ptr(rows_a), R, _ptr(y), _ptr(y64), _ptr(acc))
    _check(rc)
    out = {"y": y.view(np.float16)}
    if want_y64:
        out["y64"] = y64
    if want_acc:
        out["acc"] = acc
    return out
