"""Python binding of libcomet.so (include/comet.h) -- argument marshalling only.

Every function here has the name of the C entry point it wraps and does no
arithmetic of the method: it checks dtypes/devices, allocates outputs with
torch (device memory is PyTorch's job), passes raw pointers and the current
CUDA stream, and raises on a non-OK status.  There is no CPU fallback: if
libcomet.so is missing or the device is not sm_100, calls raise.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional, Sequence

import numpy as np
import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libcomet.so")
BLOCK = 128

STATUS = {0: "COMET_OK", 1: "COMET_ERR_INVALID_ARG", 2: "COMET_ERR_SHAPE", 3: "COMET_ERR_ALIGNMENT",
          4: "COMET_ERR_WORKSPACE", 5: "COMET_ERR_UNSUPPORTED", 6: "COMET_ERR_CUDA"}
EXPORTS = ["comet_act_plane8_bytes", "comet_act_plane4_bytes", "comet_act_ldsx", "comet_w4ax_gemm_workspace_bytes",
           "comet_w4ax_linear_scratch_bytes", "comet_pack_weight", "comet_quantize_act", "comet_w4ax_gemm",
           "comet_w4ax_gemm_acc_i32", "comet_w4ax_linear", "comet_calib_absmax", "comet_fmpq_map",
           "comet_quantize_kv", "comet_dequantize_kv", "comet_static_act_scales", "comet_quantize_act_static",
           "comet_quantize_act_bf16", "comet_gather_shards", "comet_w4ax_gemm_allgather",
           "comet_w4ax_linear_allgather", "comet_attention_kv4",
           "comet_pack_weight_f16s", "comet_w4ax_gemm_f16s", "comet_w4ax_gemm_f16s_workspace_bytes",
           "comet_pack_weight_bf16s", "comet_w4ax_gemm_bf16s",
           "comet_attention_kv4_workspace_bytes",
           "comet_status_str", "comet_last_cuda_error",
           "comet_launch_count"]


class CometError(RuntimeError):
    def __init__(self, fn, status):
        msg = f"{fn} -> {STATUS.get(status, status)}"
        if status == 6:
            msg += f" ({lib().comet_last_cuda_error().decode()})"
        super().__init__(msg)
        self.status = status


_lib = None


def lib():
    """Load libcomet.so (building it first if the sources are newer)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            from . import build as _build
            _build.build()
        L = ctypes.CDLL(LIB_PATH)
        P, i32, i64, sz = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_size_t
        L.comet_act_plane8_bytes.argtypes = [i32, i32, P]
        L.comet_act_plane8_bytes.restype = i64
        L.comet_act_plane4_bytes.argtypes = [i32, i32, P]
        L.comet_act_plane4_bytes.restype = i64
        L.comet_act_ldsx.argtypes = [i32]
        L.comet_act_ldsx.restype = i64
        L.comet_w4ax_gemm_workspace_bytes.argtypes = [i32, i32, i32]
        L.comet_w4ax_gemm_workspace_bytes.restype = i64
        L.comet_w4ax_linear_scratch_bytes.argtypes = [i32, i32, i32, P]
        L.comet_w4ax_linear_scratch_bytes.restype = i64
        L.comet_pack_weight.argtypes = [P, i64, i32, i32, P, i32, P, P, P]
        L.comet_pack_weight.restype = ctypes.c_int
        L.comet_quantize_act.argtypes = [P, i64, i32, i32, P, P, P, P, P, i64, P]
        L.comet_quantize_act.restype = ctypes.c_int
        L.comet_w4ax_gemm.argtypes = [P, P, P, i64, P, i32, i32, P, P, i32, i32, P, i64, P, sz, P]
        L.comet_w4ax_gemm.restype = ctypes.c_int
        L.comet_w4ax_gemm_acc_i32.argtypes = [P, P, P, i64, P, i32, i32, P, P, i32, i32, P, P, sz, P]
        L.comet_w4ax_gemm_acc_i32.restype = ctypes.c_int
        L.comet_w4ax_linear.argtypes = [P, i64, i32, i32, P, P, P, P, i32, i32, P, i64, P, sz, P]
        L.comet_w4ax_linear.restype = ctypes.c_int
        L.comet_calib_absmax.argtypes = [P, i64, i32, i32, P, P]
        L.comet_calib_absmax.restype = ctypes.c_int
        L.comet_fmpq_map.argtypes = [P, i32, ctypes.c_float, P, P, P]
        L.comet_fmpq_map.restype = ctypes.c_int
        L.comet_quantize_kv.argtypes = [P, i64, i32, i32, i32, P, P, P, P]
        L.comet_quantize_kv.restype = ctypes.c_int
        L.comet_dequantize_kv.argtypes = [P, P, P, i32, i32, i32, P, i64, P]
        L.comet_dequantize_kv.restype = ctypes.c_int
        L.comet_pack_weight_f16s.argtypes = [P, i64, i32, i32, P, i32, P, P, P]
        L.comet_pack_weight_f16s.restype = ctypes.c_int
        L.comet_w4ax_gemm_f16s_workspace_bytes.argtypes = [i32, i32, i32, i32]
        L.comet_w4ax_gemm_f16s_workspace_bytes.restype = i64
        L.comet_w4ax_gemm_f16s.argtypes = [P, P, P, i64, P, i32, i32, P, P, i32, i32, P, i64, P, sz, P]
        L.comet_w4ax_gemm_f16s.restype = ctypes.c_int
        L.comet_pack_weight_bf16s.argtypes = [P, i64, i32, i32, P, i32, P, P, P]
        L.comet_pack_weight_bf16s.restype = ctypes.c_int
        L.comet_w4ax_gemm_bf16s.argtypes = [P, P, P, i64, P, i32, i32, P, P, i32, i32, P, i64, P, sz, P]
        L.comet_w4ax_gemm_bf16s.restype = ctypes.c_int
        L.comet_attention_kv4_workspace_bytes.argtypes = [i32, i32]
        L.comet_attention_kv4_workspace_bytes.restype = i64
        L.comet_attention_kv4.argtypes = [P, P, P, P, P, P, P, i32, i32, i32, i32, ctypes.c_float, P, P, sz, P]
        L.comet_attention_kv4.restype = ctypes.c_int
        L.comet_gather_shards.argtypes = [P, i32, i32, i32, i32, P, i64, P]
        L.comet_gather_shards.restype = ctypes.c_int
        L.comet_w4ax_gemm_allgather.argtypes = [P, P, P, i64, P, i32, i32, P, P, i32, i32, P, i32, i64, i64, P,
                                                sz, P]
        L.comet_w4ax_gemm_allgather.restype = ctypes.c_int
        L.comet_w4ax_linear_allgather.argtypes = [P, i64, i32, i32, P, P, P, P, i32, i32, P, i32, i64, i64, P, sz, P]
        L.comet_w4ax_linear_allgather.restype = ctypes.c_int
        L.comet_quantize_act_bf16.argtypes = [P, i64, i32, i32, P, P, P, P, P, i64, P]
        L.comet_quantize_act_bf16.restype = ctypes.c_int
        L.comet_static_act_scales.argtypes = [P, i32, P, P, P, P]
        L.comet_static_act_scales.restype = ctypes.c_int
        L.comet_quantize_act_static.argtypes = [P, i64, i32, i32, P, P, P, P, P, P, i64, P]
        L.comet_quantize_act_static.restype = ctypes.c_int
        L.comet_status_str.argtypes = [ctypes.c_int]
        L.comet_status_str.restype = ctypes.c_char_p
        L.comet_last_cuda_error.argtypes = []
        L.comet_last_cuda_error.restype = ctypes.c_char_p
        L.comet_launch_count.argtypes = []
        L.comet_launch_count.restype = i64
        _lib = L
    return _lib


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def _check(fn, st):
    if st != 0:
        raise CometError(fn, st)


class BlockBits:
    """Host copy of a layer's static precision mask (K/128 entries of 4/8)."""

    def __init__(self, bits: Sequence[int]):
        self.array = np.ascontiguousarray(np.asarray(bits, dtype=np.uint8))
        self.ptr = self.array.ctypes.data_as(ctypes.c_void_p)
        self.n8 = int((self.array == 8).sum())
        self.n4 = int((self.array == 4).sum())

    def __len__(self):
        return self.array.size


def as_bits(bits) -> BlockBits:
    return bits if isinstance(bits, BlockBits) else BlockBits(bits)


def launch_count() -> int:
    return int(lib().comet_launch_count())


# ---------------------------------------------------------------- layout ----
def wq_tiled_to_rowmajor(wq_tiled: np.ndarray, N: int, K: int) -> np.ndarray:
    """Tiled packed weights (include/comet.h) -> row-major [N x K/2] bytes.

    Pure data movement (no arithmetic of the method): slab (n//128, k-block b)
    of 128 rows x 64 B is contiguous; 16-B chunk c of row r sits at chunk
    c ^ ((r >> 1) & 3)."""
    nb = K // BLOCK
    t = np.asarray(wq_tiled, dtype=np.uint8).reshape(N // 128, nb, 128, 4, 16)
    r = np.arange(128)[:, None]
    c = np.arange(4)[None, :]
    t = t[:, :, r, c ^ ((r >> 1) & 3), :]             # undo the chunk swizzle
    return np.ascontiguousarray(t.transpose(0, 2, 1, 3, 4).reshape(N, K // 2))


# ----------------------------------------------------------------- sizes ----
def comet_act_ldsx(M: int) -> int:
    return int(lib().comet_act_ldsx(M))


def comet_w4ax_gemm_workspace_bytes(M: int, N: int, K: int) -> int:
    return int(lib().comet_w4ax_gemm_workspace_bytes(M, N, K))


def comet_w4ax_linear_scratch_bytes(M: int, N: int, K: int, bits) -> int:
    return int(lib().comet_w4ax_linear_scratch_bytes(M, N, K, as_bits(bits).ptr))


def new_workspace(nbytes: int, device) -> Optional[torch.Tensor]:
    """Device workspace; the first 64 KiB (tile counters) must start zeroed."""
    if nbytes <= 0:
        return None
    return torch.zeros(nbytes, dtype=torch.uint8, device=device)


# -------------------------------------------------------------- entries ----
def comet_pack_weight(W: torch.Tensor, perm: Optional[torch.Tensor] = None, group: int = BLOCK, stream=None):
    """a0: W fp16 [N x K] -> (Wq uint8 [N x K/2] bytes in the TILED layout,
    Sw fp32 [K/group x N]); see wq_tiled_to_rowmajor."""
    assert W.is_cuda and W.dtype == torch.float16 and W.dim() == 2 and W.stride(1) == 1
    N, K = W.shape
    Wq = torch.empty((N, K // 2), dtype=torch.uint8, device=W.device)
    Sw = torch.empty((K // group, N), dtype=torch.float32, device=W.device)
    st = lib().comet_pack_weight(_ptr(W), W.stride(0), N, K, _ptr(perm), group, _ptr(Wq), _ptr(Sw), _stream(stream))
    _check("comet_pack_weight", st)
    return Wq, Sw


def alloc_act_planes(M: int, K: int, bits, device):
    b = as_bits(bits)
    ldsx = comet_act_ldsx(M)
    Xq8 = torch.empty((M, BLOCK * b.n8), dtype=torch.int8, device=device)
    Xq4 = torch.empty((M, BLOCK * b.n4 // 2), dtype=torch.uint8, device=device)
    Sx = torch.empty((K // BLOCK, ldsx), dtype=torch.float32, device=device)
    return Xq8, Xq4, Sx


def comet_quantize_act(X: torch.Tensor, bits, perm: Optional[torch.Tensor] = None, out=None, stream=None):
    """a1+a2: X fp16 [M x K] -> (Xq8, Xq4, Sx)."""
    assert X.is_cuda and X.dtype == torch.float16 and X.dim() == 2 and X.stride(1) == 1
    b = as_bits(bits)
    M, K = X.shape
    Xq8, Xq4, Sx = out if out is not None else alloc_act_planes(M, K, b, X.device)
    st = lib().comet_quantize_act(_ptr(X), X.stride(0), M, K, _ptr(perm), b.ptr, _ptr(Xq8) if b.n8 else None,
                                  _ptr(Xq4) if b.n4 else None, _ptr(Sx), Sx.shape[1], _stream(stream))
    _check("comet_quantize_act", st)
    return Xq8, Xq4, Sx


def comet_static_act_scales(maxabs: torch.Tensor, bits, perm: Optional[torch.Tensor] = None, stream=None):
    """f4: static per-block activation scales (DEVICE fp32[K/128]) from the
    calibration maxabs (DEVICE fp32[K]) -- see comet.h."""
    assert maxabs.is_cuda and maxabs.dtype == torch.float32 and maxabs.dim() == 1
    b = as_bits(bits)
    K = maxabs.shape[0]
    scales = torch.empty(K // BLOCK, dtype=torch.float32, device=maxabs.device)
    st = lib().comet_static_act_scales(_ptr(maxabs), K, _ptr(perm), b.ptr, _ptr(scales), _stream(stream))
    _check("comet_static_act_scales", st)
    return scales


def comet_quantize_act_static(X: torch.Tensor, bits, scales: torch.Tensor, perm: Optional[torch.Tensor] = None,
                              out=None, stream=None):
    """f4: X fp16 [M x K] -> (Xq8, Xq4, Sx) with the static per-block scales."""
    assert X.is_cuda and X.dtype == torch.float16 and X.dim() == 2 and X.stride(1) == 1
    assert scales.is_cuda and scales.dtype == torch.float32
    b = as_bits(bits)
    M, K = X.shape
    Xq8, Xq4, Sx = out if out is not None else alloc_act_planes(M, K, b, X.device)
    st = lib().comet_quantize_act_static(_ptr(X), X.stride(0), M, K, _ptr(perm), b.ptr, _ptr(scales),
                                         _ptr(Xq8) if b.n8 else None, _ptr(Xq4) if b.n4 else None, _ptr(Sx),
                                         Sx.shape[1], _stream(stream))
    _check("comet_quantize_act_static", st)
    return Xq8, Xq4, Sx


def comet_quantize_act_bf16(X: torch.Tensor, bits, perm: Optional[torch.Tensor] = None, out=None, stream=None):
    """f4: comet_quantize_act for bf16 activations X [M x K]."""
    assert X.is_cuda and X.dtype == torch.bfloat16 and X.dim() == 2 and X.stride(1) == 1
    b = as_bits(bits)
    M, K = X.shape
    Xq8, Xq4, Sx = out if out is not None else alloc_act_planes(M, K, b, X.device)
    st = lib().comet_quantize_act_bf16(_ptr(X), X.stride(0), M, K, _ptr(perm), b.ptr, _ptr(Xq8) if b.n8 else None,
                                       _ptr(Xq4) if b.n4 else None, _ptr(Sx), Sx.shape[1], _stream(stream))
    _check("comet_quantize_act_bf16", st)
    return Xq8, Xq4, Sx


def comet_calib_absmax(X: torch.Tensor, maxabs: Optional[torch.Tensor] = None, stream=None):
    """f2: per-channel max |X| over the rows of X fp16 [M x K], accumulated
    into maxabs (DEVICE fp32[K], zero-initialised when None)."""
    assert X.is_cuda and X.dtype == torch.float16 and X.dim() == 2 and X.stride(1) == 1
    M, K = X.shape
    if maxabs is None:
        maxabs = torch.zeros(K, dtype=torch.float32, device=X.device)
    st = lib().comet_calib_absmax(_ptr(X), X.stride(0), M, K, _ptr(maxabs), _stream(stream))
    _check("comet_calib_absmax", st)
    return maxabs


def comet_fmpq_map(score, theta: float = 8.0):
    """f2 (host): per-channel scores -> (perm int32[K], block_bits uint8[K/128],
    number of outliers), the SPEC S:L139-165 rule (see comet.h)."""
    import numpy as np
    sc = np.ascontiguousarray(np.asarray(score.cpu() if hasattr(score, "cpu") else score, dtype=np.float32))
    K = sc.shape[0]
    perm = np.empty(K, dtype=np.int32)
    bits = np.empty(K // BLOCK, dtype=np.uint8)
    n = ctypes.c_int32(0)
    st = lib().comet_fmpq_map(sc.ctypes.data, K, float(theta), perm.ctypes.data, bits.ctypes.data, ctypes.byref(n))
    _check("comet_fmpq_map", st)
    return perm, bits, int(n.value)


def comet_quantize_kv(KV: torch.Tensor, group: int, stream=None):
    """f3: KV fp16 [T x C] -> (Q uint8 [T x C/2] packed, scale fp32 [G x C],
    zp uint8 [G x C]), G = ceil(T / group)."""
    assert KV.is_cuda and KV.dtype == torch.float16 and KV.dim() == 2 and KV.stride(1) == 1
    T, C = KV.shape
    ng = (T + group - 1) // group
    Q = torch.empty((T, C // 2), dtype=torch.uint8, device=KV.device)
    scale = torch.empty((ng, C), dtype=torch.float32, device=KV.device)
    zp = torch.empty((ng, C), dtype=torch.uint8, device=KV.device)
    st = lib().comet_quantize_kv(_ptr(KV), KV.stride(0), T, C, group, _ptr(Q), _ptr(scale), _ptr(zp), _stream(stream))
    _check("comet_quantize_kv", st)
    return Q, scale, zp


def comet_dequantize_kv(Q: torch.Tensor, scale: torch.Tensor, zp: torch.Tensor, group: int, stream=None):
    """f3: packed KV4 -> fp16 [T x C]."""
    T, C = Q.shape[0], Q.shape[1] * 2
    out = torch.empty((T, C), dtype=torch.float16, device=Q.device)
    st = lib().comet_dequantize_kv(_ptr(Q), _ptr(scale), _ptr(zp), T, C, group, _ptr(out), out.stride(0),
                                   _stream(stream))
    _check("comet_dequantize_kv", st)
    return out


def comet_w4ax_gemm(Xq8, Xq4, Sx, bits, Wq, Sw, group: int = BLOCK, out: Optional[torch.Tensor] = None,
                    workspace: Optional[torch.Tensor] = None, stream=None):
    """a3..a8: Y fp16 [M x N] = dequant(Xq . Wq^T)."""
    b = as_bits(bits)
    M = Xq8.shape[0] if b.n8 else Xq4.shape[0]
    N, K = Wq.shape[0], Wq.shape[1] * 2
    Y = out if out is not None else torch.empty((M, N), dtype=torch.float16, device=Wq.device)
    need = comet_w4ax_gemm_workspace_bytes(M, N, K)
    if need > 0 and (workspace is None or workspace.numel() < need):
        raise CometError("comet_w4ax_gemm", 4)
    st = lib().comet_w4ax_gemm(_ptr(Xq8) if b.n8 else None, _ptr(Xq4) if b.n4 else None, _ptr(Sx), Sx.shape[1], b.ptr,
                               M, K, _ptr(Wq), _ptr(Sw), N, group, _ptr(Y), Y.stride(0),
                               _ptr(workspace), 0 if workspace is None else workspace.numel(), _stream(stream))
    _check("comet_w4ax_gemm", st)
    return Y


def comet_pack_weight_f16s(W: torch.Tensor, perm: Optional[torch.Tensor] = None, group: int = BLOCK, stream=None,
                           bf16: bool = False):
    """f4: as comet_pack_weight, with fp16 (bf16=True: bf16) scales Sw16 [K/group x N] (the quantization scale)."""
    assert W.is_cuda and W.dtype == torch.float16 and W.dim() == 2 and W.stride(1) == 1
    N, K = W.shape
    Wq = torch.empty((N, K // 2), dtype=torch.uint8, device=W.device)
    Sw = torch.empty((K // group, N), dtype=torch.bfloat16 if bf16 else torch.float16, device=W.device)
    fn = "comet_pack_weight_bf16s" if bf16 else "comet_pack_weight_f16s"
    st = getattr(lib(), fn)(_ptr(W), W.stride(0), N, K, _ptr(perm), group, _ptr(Wq), _ptr(Sw), _stream(stream))
    _check(fn, st)
    return Wq, Sw


def comet_pack_weight_bf16s(W: torch.Tensor, perm: Optional[torch.Tensor] = None, group: int = BLOCK, stream=None):
    """f4: as comet_pack_weight, with bf16 scales Sw16 [K/group x N] (the quantization scale)."""
    return comet_pack_weight_f16s(W, perm, group, stream, bf16=True)


def comet_w4ax_gemm_bf16s(Xq8, Xq4, Sx, bits, Wq, Sw16, group: int = BLOCK, out=None, workspace=None, stream=None):
    """f4: comet_w4ax_gemm with bf16 weight scales."""
    return comet_w4ax_gemm_f16s(Xq8, Xq4, Sx, bits, Wq, Sw16, group, out, workspace, stream)


def comet_w4ax_gemm_f16s(Xq8, Xq4, Sx, bits, Wq, Sw16, group: int = BLOCK, out=None, workspace=None, stream=None):
    """f4: comet_w4ax_gemm with fp16 (or, for a bf16 Sw16, bf16) weight scales."""
    b = as_bits(bits)
    M = Xq8.shape[0] if b.n8 else Xq4.shape[0]
    N, K = Wq.shape[0], Wq.shape[1] * 2
    Y = out if out is not None else torch.empty((M, N), dtype=torch.float16, device=Wq.device)
    need = int(lib().comet_w4ax_gemm_f16s_workspace_bytes(M, N, K, group))
    if workspace is None or workspace.numel() < need:
        workspace = new_workspace(need, Wq.device)
    fn = "comet_w4ax_gemm_bf16s" if Sw16.dtype == torch.bfloat16 else "comet_w4ax_gemm_f16s"
    st = getattr(lib(), fn)(_ptr(Xq8) if b.n8 else None, _ptr(Xq4) if b.n4 else None, _ptr(Sx), Sx.shape[1],
                            b.ptr, M, K, _ptr(Wq), _ptr(Sw16), N, group, _ptr(Y), Y.stride(0),
                            _ptr(workspace), workspace.numel(), _stream(stream))
    _check(fn, st)
    return Y


def comet_attention_kv4(q: torch.Tensor, K, V, group: int, softmax_scale: float, workspace=None, stream=None):
    """f3: decode attention over KV4 caches (K, V: (Q packed [T x C/2], scale [G x C], zp [G x C]) from
    comet_quantize_kv); q fp16 [H x 128] -> out fp16 [H x 128]."""
    H, D = q.shape
    Kq, Ks, Kz = K
    Vq, Vs, Vz = V
    T = Kq.shape[0]
    need = int(lib().comet_attention_kv4_workspace_bytes(T, H))
    if workspace is None or workspace.numel() < need:
        workspace = torch.empty(max(need, 16), dtype=torch.uint8, device=q.device)
    out = torch.empty((H, D), dtype=torch.float16, device=q.device)
    st = lib().comet_attention_kv4(_ptr(q), _ptr(Kq), _ptr(Ks), _ptr(Kz), _ptr(Vq), _ptr(Vs), _ptr(Vz), T, H, D, group,
                                   float(softmax_scale), _ptr(out), _ptr(workspace), workspace.numel(), _stream(stream))
    _check("comet_attention_kv4", st)
    return out


def comet_gather_shards(Yall: torch.Tensor, N: int, out: Optional[torch.Tensor] = None, stream=None):
    """(e): rank-major gathered shards [P x M x per] -> Y [M x N] (padding dropped)."""
    P, M, per = Yall.shape
    Y = out if out is not None else torch.empty((M, N), dtype=Yall.dtype, device=Yall.device)
    st = lib().comet_gather_shards(_ptr(Yall), P, M, per, N, _ptr(Y), Y.stride(0), _stream(stream))
    _check("comet_gather_shards", st)
    return Y


def comet_w4ax_gemm_acc_i32(Xq8, Xq4, Sx, bits, Wq, Sw, group: int = BLOCK, workspace: Optional[torch.Tensor] = None,
                            stream=None):
    """Debug: per-block INT32 accumulators [K/128 x M x N] (logical units)."""
    b = as_bits(bits)
    M = Xq8.shape[0] if b.n8 else Xq4.shape[0]
    N, K = Wq.shape[0], Wq.shape[1] * 2
    Acc = torch.empty((K // BLOCK, M, N), dtype=torch.int32, device=Wq.device)
    need = comet_w4ax_gemm_workspace_bytes(M, N, K)
    if need > 0 and (workspace is None or workspace.numel() < need):
        workspace = new_workspace(need, Wq.device)
    st = lib().comet_w4ax_gemm_acc_i32(_ptr(Xq8) if b.n8 else None, _ptr(Xq4) if b.n4 else None, _ptr(Sx), Sx.shape[1],
                                       b.ptr, M, K, _ptr(Wq), _ptr(Sw), N, group, _ptr(Acc), _ptr(workspace),
                                       0 if workspace is None else workspace.numel(), _stream(stream))
    _check("comet_w4ax_gemm_acc_i32", st)
    return Acc


def comet_w4ax_linear(X: torch.Tensor, bits, Wq, Sw, perm=None, group: int = BLOCK, out: Optional[torch.Tensor] = None,
                      scratch: Optional[torch.Tensor] = None, stream=None, sync: bool = True):
    """Whole linear layer through the C ABI; X / out may be host (pinned) tensors.
    The C call only enqueues the work; with a host `out` and sync=True this
    synchronizes the stream so `out` is complete on return (sync=False: the
    caller synchronizes, and consecutive host-buffer calls overlap their
    copies)."""
    b = as_bits(bits)
    M, K = X.shape
    N = Wq.shape[0]
    Y = out if out is not None else torch.empty((M, N), dtype=torch.float16, device=Wq.device)
    need = comet_w4ax_linear_scratch_bytes(M, N, K, b)
    if scratch is None or scratch.numel() < need:
        raise CometError("comet_w4ax_linear", 4)
    st = lib().comet_w4ax_linear(_ptr(X), X.stride(0), M, K, _ptr(perm), b.ptr, _ptr(Wq), _ptr(Sw), N, group,
                                 _ptr(Y), Y.stride(0), _ptr(scratch), scratch.numel(), _stream(stream))
    _check("comet_w4ax_linear", st)
    if sync and not Y.is_cuda:
        (stream if stream is not None else torch.cuda.current_stream()).synchronize()
    return Y


def _dest_array(dests):
    """f1 destinations: tensors (this process's buffers) or raw device
    addresses (peers' buffers mapped into this process) -> void*[]"""
    ptrs = [d.data_ptr() if isinstance(d, torch.Tensor) else int(d) for d in dests]
    return (ctypes.c_void_p * len(ptrs))(*ptrs), len(ptrs)


def comet_w4ax_gemm_allgather(Xq8, Xq4, Sx, bits, Wq, Sw, dests, ldy: int, col0: int, group: int = BLOCK,
                              workspace: Optional[torch.Tensor] = None, stream=None):
    """f1: the GEMM's epilogue writes its [M x N] result into columns
    [col0, col0 + N) of every destination [M x ldy] fp16 (dests[0] local,
    the rest peers' copies); the caller's cross-rank barrier follows."""
    b = as_bits(bits)
    M = Xq8.shape[0] if b.n8 else Xq4.shape[0]
    N, K = Wq.shape[0], Wq.shape[1] * 2
    need = comet_w4ax_gemm_workspace_bytes(M, N, K)
    if need > 0 and (workspace is None or workspace.numel() < need):
        raise CometError("comet_w4ax_gemm_allgather", 4)
    arr, n = _dest_array(dests)
    st = lib().comet_w4ax_gemm_allgather(_ptr(Xq8) if b.n8 else None, _ptr(Xq4) if b.n4 else None, _ptr(Sx),
                                         Sx.shape[1], b.ptr, M, K, _ptr(Wq), _ptr(Sw), N, group, arr, n, ldy, col0,
                                         _ptr(workspace), 0 if workspace is None else workspace.numel(),
                                         _stream(stream))
    _check("comet_w4ax_gemm_allgather", st)


def comet_w4ax_linear_allgather(X: torch.Tensor, bits, Wq, Sw, dests, ldy: int, col0: int, perm=None,
                                group: int = BLOCK, scratch: Optional[torch.Tensor] = None, stream=None):
    """f1: the whole layer with the all-gather fused into the GEMM epilogue
    (device buffers only); see comet_w4ax_gemm_allgather."""
    b = as_bits(bits)
    M, K = X.shape
    N = Wq.shape[0]
    need = comet_w4ax_linear_scratch_bytes(M, N, K, b)
    if scratch is None or scratch.numel() < need:
        raise CometError("comet_w4ax_linear_allgather", 4)
    arr, n = _dest_array(dests)
    st = lib().comet_w4ax_linear_allgather(_ptr(X), X.stride(0), M, K, _ptr(perm), b.ptr, _ptr(Wq), _ptr(Sw), N,
                                           group, arr, n, ldy, col0, _ptr(scratch), scratch.numel(), _stream(stream))
    _check("comet_w4ax_linear_allgather", st)


class W4AxLinear:
    """A packed W4Ax linear layer: weights packed once (a0), forward = a1..a8."""

    def __init__(self, W: torch.Tensor, bits, perm: Optional[torch.Tensor] = None, group: int = BLOCK):
        self.bits = as_bits(bits)
        self.perm = perm
        self.group = group
        self.N, self.K = W.shape
        self.Wq, self.Sw = comet_pack_weight(W, perm, group)
        self._ws = {}

    def workspace(self, M: int):
        need = comet_w4ax_gemm_workspace_bytes(M, self.N, self.K)
        ws = self._ws.get(need)
        if ws is None and need > 0:
            ws = self._ws[need] = new_workspace(need, self.Wq.device)
        return ws

    def __call__(self, X: torch.Tensor, out: Optional[torch.Tensor] = None, planes=None):
        Xq8, Xq4, Sx = comet_quantize_act(X, self.bits, self.perm, out=planes)
        return comet_w4ax_gemm(Xq8, Xq4, Sx, self.bits, self.Wq, self.Sw, self.group, out=out,
                               workspace=self.workspace(X.shape[0]))
