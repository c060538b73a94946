"""Projector GEMM with a boundary epilogue.

``projector_gemm`` runs the encoder's last layer, Y = X . W^T (tinymodel.hpp:62,
the ``enc_w2`` projector), on the sm_100a tensor cores through
``hb_projector_gemm`` (``csrc/kernels/projector_gemm.cu``: TMA-fed tcgen05.mma,
TMEM accumulators, warp-specialised). Its epilogue stores each output row to a
table of destination rows, which is how the boundary writes the projector
output straight into every consumer's destination shard (local or a peer GPU's
over NVSwitch) instead of writing the source shard and resharding it.
"""
from __future__ import annotations

import ctypes

from ._lib import HetBridgeError, check, lib


def projector_gemm_rows(x, w, row_dst, fan: int, stream=None):
    """Y = x @ w.T with row m stored to every non-zero ``row_dst[m, f]`` (int64
    device addresses of N-element bf16 rows). x: [M, K] bf16, w: [N, K] bf16."""
    import torch

    if x.dtype != torch.bfloat16 or w.dtype != torch.bfloat16:
        raise HetBridgeError(24, "projector_gemm takes bf16 operands")
    if x.dim() != 2 or w.dim() != 2 or x.shape[1] != w.shape[1]:
        raise HetBridgeError(13, f"shapes {tuple(x.shape)} x {tuple(w.shape)}^T do not chain")
    if x.stride(1) != 1 or w.stride(1) != 1:
        raise HetBridgeError(24, "projector operands must be row-major (unit inner stride)")
    M, K = x.shape
    N = w.shape[0]
    if row_dst.dtype != torch.int64 or row_dst.numel() != M * fan or not row_dst.is_cuda:
        raise HetBridgeError(13, "row_dst must be an int64 CUDA tensor of M * fan addresses")
    s = stream if stream is not None else torch.cuda.current_stream()
    check(lib().hb_projector_gemm(ctypes.c_void_p(x.data_ptr()), x.stride(0), ctypes.c_void_p(w.data_ptr()),
                                  w.stride(0), ctypes.c_void_p(row_dst.data_ptr()), fan, M, N, K,
                                  ctypes.c_void_p(s.cuda_stream)))


def projector_gemm(x, w, out=None, stream=None):
    """Plain Y = x @ w.T (bf16) into ``out`` [M, N] (allocated if None)."""
    import torch

    M, N = x.shape[0], w.shape[0]
    if out is None:
        out = torch.empty(M, N, dtype=torch.bfloat16, device=x.device)
    rows = out.data_ptr() + torch.arange(M, device=x.device, dtype=torch.int64) * (out.stride(0) * 2)
    projector_gemm_rows(x, w, rows, 1, stream)
    return out
