"""torch-tensor front end of the device entry points in libemm.so.

PyTorch provides device memory and streams only; every op here launches one
of our sm_100a kernels through the C ABI.  There is no fallback: calling an
op on a non-CUDA tensor raises.
"""
from __future__ import annotations

import ctypes as C

import torch

from . import _lib
from ._lib import check, lib

vp, i64, i32, u64 = C.c_void_p, C.c_int64, C.c_int32, C.c_uint64

_lib.declare_more({
    "emm_launch_count": (C.c_uint64, []),
    "emm_device_sm_count": (C.c_int, [C.c_int, C.POINTER(C.c_int)]),
    "emm_gemm_bf16": (C.c_int, [vp, i64, vp, i64, vp, i64, i64, i64, i64, vp, vp, i64, C.c_int,
                                vp]),
})

EPI_NONE, EPI_GELU_TANH, EPI_QUICK_GELU, EPI_GELU_ERF, EPI_GLU_SILU = 0, 1, 2, 3, 4


def _stream(t: torch.Tensor | None = None):
    return torch.cuda.current_stream().cuda_stream


def _req_cuda(*ts):
    for t in ts:
        if t is not None and not t.is_cuda:
            raise RuntimeError("emm ops need CUDA tensors (no CPU fallback)")


def _ptr(t):
    return None if t is None else t.data_ptr()


def launch_count() -> int:
    return int(lib.emm_launch_count())


def gemm(a: torch.Tensor, b: torch.Tensor, out: torch.Tensor | None = None,
         bias: torch.Tensor | None = None, residual: torch.Tensor | None = None,
         epi: int = EPI_NONE) -> torch.Tensor:
    """out[M,N] = epi(a[M,K] @ b[N,K]^T + bias) (+ residual) on tcgen05.

    For EPI_GLU_SILU, b holds gate/up rows interleaved in blocks of 128
    (see interleave_glu) and out is [M, N/2]."""
    _req_cuda(a, b, bias, residual)
    assert a.dtype == torch.bfloat16 and b.dtype == torch.bfloat16
    assert a.dim() == 2 and b.dim() == 2 and a.shape[1] == b.shape[1]
    assert a.stride(1) == 1 and b.stride(1) == 1
    M, K = a.shape
    N = b.shape[0]
    n_out = N // 2 if epi == EPI_GLU_SILU else N
    if out is None:
        out = torch.empty(M, n_out, device=a.device, dtype=torch.bfloat16)
    assert out.shape == (M, n_out) and out.stride(1) == 1
    if residual is not None:
        assert residual.shape == (M, n_out) and residual.stride(1) == 1
    check(lib.emm_gemm_bf16(a.data_ptr(), a.stride(0), b.data_ptr(), b.stride(0),
                            out.data_ptr(), out.stride(0), M, N, K, _ptr(bias), _ptr(residual),
                            residual.stride(0) if residual is not None else 0, epi,
                            _stream()))
    return out


def interleave_glu(w_gate: torch.Tensor, w_up: torch.Tensor, block: int = 128) -> torch.Tensor:
    """[I,K] gate and up -> [2I,K] with rows [g0..g127, u0..u127, g128..] so the
    GLU epilogue finds gate and up of the same feature in one 256-wide tile."""
    inter, k = w_gate.shape
    assert inter % block == 0, "intermediate size must be a multiple of 128"
    g = w_gate.reshape(inter // block, block, k)
    u = w_up.reshape(inter // block, block, k)
    return torch.stack([g, u], dim=1).reshape(2 * inter, k).contiguous()


def interleave_glu_bias(b_gate: torch.Tensor, b_up: torch.Tensor, block: int = 128):
    inter = b_gate.shape[0]
    return torch.stack([b_gate.reshape(-1, block), b_up.reshape(-1, block)], 1).reshape(2 * inter)
