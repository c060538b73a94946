"""PyTorch autograd binding of the boundary communicator, and the colocated
three-phase packed boundary tensor.

The reference declares the boundary as a pair of role calls per rank
(``BridgeRuntime::forward_*`` / ``backward_*``, bridge.hpp:146-173); the
paper's Megatron implementation wraps it as an autograd op (P:63-67,
P:1095-1101) and, for colocated modules, runs a three-phase schedule
(S:371-374):

1. encoder forward once over the microbatch window, then the colocated
   forward transform into a *packed boundary tensor* in the LLM PP0 layout;
2. the packed tensor is detached as a leaf and the LLM's 1F1B consumes
   per-microbatch views of it (no encoder collectives inside this phase);
3. after the LLM drains, the gradients accumulated on the packed tensor are
   handed to the colocated backward transform, which returns them to the
   source owners, and encoder backward runs.

Here every tensor the LLM sees is a view of the runtime's device region:
phase-1 outputs are the DST_ACT buffers of the microbatch's buffer set, the
leaves' ``.grad`` are pre-bound to the DST_GRAD buffers (autograd accumulates
into an existing ``.grad`` in place, so LLM gradients land where the backward
kernel reads them), and phase 3 hands the SRC_GRAD buffers to the encoder's
autograd graph. Nothing is copied on the boundary except by the sm_100a
kernels. Every call is collective across the processes of a multi-GPU exec
group, in the same order.
"""
from __future__ import annotations

import torch

from ._lib import HetBridgeError
from .bridge import SLOT_DST_ACT, SLOT_DST_GRAD, SLOT_SRC_ACT, SLOT_SRC_GRAD, BridgeRuntime


def _shape(rt: BridgeRuntime, rank: int, slot: int) -> tuple[int, int]:
    """Row-major 2-D shape of a buffer: samples x W, or token rows x d_h for a
    splice destination."""
    n = rt.buffer_numel(rank, slot)
    w = rt.splice.d_h if (rt.splice is not None and slot in (SLOT_DST_ACT, SLOT_DST_GRAD)) \
        else rt.plan.edge.feature_width
    return (n // w, w)


def _view(rt: BridgeRuntime, rank: int, slot: int, mb: int):
    return rt.buffer(rank, slot, mb % rt.mb_slots).reshape(_shape(rt, rank, slot))


def _attach(rt: BridgeRuntime, rank: int, slot: int, mb: int, t, zero_copy: bool):
    """Make ``t`` the (rank, slot) buffer of microbatch mb's set: bound in place
    (zero_copy; a no-op when already bound) or copied into the runtime's own
    buffer (the runtime keeps its previous binding otherwise)."""
    buf_shape = _shape(rt, rank, slot)
    if t.numel() != buf_shape[0] * buf_shape[1]:
        raise HetBridgeError(13, f"rank {rank} slot {slot}: {t.numel()} elements, plan needs "
                                 f"{buf_shape[0] * buf_shape[1]}")
    if zero_copy:
        t2 = t.detach()
        if t2.dtype != rt._dtype_of(slot):
            raise HetBridgeError(13, f"rank {rank} slot {slot}: dtype {t2.dtype}, runtime carries "
                                     f"{rt._dtype_of(slot)} (zero_copy needs the runtime's dtype)")
        if not (t2.dim() == 2 and t2.shape == buf_shape and t2.stride(1) == 1) and not t2.is_contiguous():
            t2 = t2.contiguous()
        if t2.dim() != 2:
            t2 = t2.reshape(buf_shape)
        rt.bind(rank, slot, t2, mb % rt.mb_slots)
        return
    buf = _view(rt, rank, slot, mb)
    if t.data_ptr() != buf.data_ptr():  # the producer may already have written into the buffer
        buf.copy_(t.reshape(buf.shape))


class _Boundary(torch.autograd.Function):
    """One boundary op pair: forward reshard (+splice) / gradient return."""

    @staticmethod
    def forward(ctx, rt: BridgeRuntime, mb: int, zero_copy: bool, *src):
        src_ranks, dst_ranks = rt.local_ranks(SLOT_SRC_ACT), rt.local_ranks(SLOT_DST_ACT)
        if len(src) != len(src_ranks):
            raise HetBridgeError(24, f"expected {len(src_ranks)} source shards (ranks {src_ranks}), got {len(src)}")
        stream = torch.cuda.current_stream()
        for r, t in zip(src_ranks, src):
            _attach(rt, r, SLOT_SRC_ACT, mb, t, zero_copy)
        rt.sync_bindings()  # collective at N > 1 when a binding changed on any GPU
        rt.forward(mb, stream)
        ctx.rt, ctx.mb, ctx.zero_copy = rt, mb, zero_copy
        ctx.src_meta = [(t.dtype, t.shape) for t in src]
        outs = tuple(_view(rt, r, SLOT_DST_ACT, mb) for r in dst_ranks)
        # outputs alias the runtime's buffers of this microbatch's set: they
        # stay valid until the set is reused (mb + mb_slots)
        return outs if len(outs) != 1 else outs[0]

    @staticmethod
    def backward(ctx, *grads):
        rt, mb, zc = ctx.rt, ctx.mb, ctx.zero_copy
        dst_ranks, src_ranks = rt.local_ranks(SLOT_DST_ACT), rt.local_ranks(SLOT_SRC_ACT)
        for r, g in zip(dst_ranks, grads):
            if g is None:
                g = torch.zeros(_shape(rt, r, SLOT_DST_GRAD), dtype=rt._dtype_of(SLOT_DST_GRAD),
                                device=rt.device)
            _attach(rt, r, SLOT_DST_GRAD, mb, g.to(rt._dtype_of(SLOT_DST_GRAD)) if zc else g, zc)
        # zero_copy: the kernel writes each returned gradient straight into a
        # fresh tensor (bound as the SRC_GRAD buffer, beta=0) when the runtime
        # already carries the source dtype; otherwise fp32 buffer + cast copy
        direct = zc and all(dt == rt._dtype_of(SLOT_SRC_GRAD) for dt, _ in ctx.src_meta)
        fresh = []
        if direct:
            for r in src_ranks:
                o = torch.empty(_shape(rt, r, SLOT_SRC_GRAD), dtype=rt._dtype_of(SLOT_SRC_GRAD), device=rt.device)
                rt.bind(r, SLOT_SRC_GRAD, o, mb % rt.mb_slots)
                fresh.append(o)
        rt.sync_bindings()
        rt.backward(mb, 0.0, torch.cuda.current_stream())
        if direct:
            out = [o.view(shape) for o, (dt, shape) in zip(fresh, ctx.src_meta)]
        else:
            # always a fresh tensor: an alias of SRC_GRAD could be kept as a leaf's
            # .grad by AccumulateGrad and then overwritten when the set is reused
            out = [_view(rt, r, SLOT_SRC_GRAD, mb).to(dt, copy=True).view(shape)
                   for r, (dt, shape) in zip(src_ranks, ctx.src_meta)]
        return (None, None, None, *out)


def boundary(rt: BridgeRuntime, mb: int, *src_shards, zero_copy: bool = True):
    """Differentiable boundary op for microbatch ``mb``.

    ``src_shards``: this process's source-rank shards in ascending rank order
    (``rt.local_ranks(SLOT_SRC_ACT)``). Returns the destination shards of the
    local destination ranks (ascending), as views of the runtime's buffers.
    Backward returns the gradient to each source shard (the reference's
    ``backward_*`` role calls), fp32-accumulated and cast to the shard dtype.

    zero_copy (default): the caller's shards and the incoming gradients are
    bound as the runtime's buffers (hb_exec_bind; across GPUs the peers map
    them through CUDA IPC, one binding exchange when a pointer changed) and the
    returned gradients are written by the kernel into fresh tensors, so no
    staging copy touches HBM. A changed pointer rebuilds the device tables at
    the next op (host cost), so a steady-state caller keeps its tensors or
    writes into ``rt.buffer`` views; zero_copy=False copies into the runtime's
    buffers instead."""
    return _Boundary.apply(rt, mb, zero_copy, *src_shards)


class PackedBoundary:
    """Colocated three-phase schedule over one boundary edge.

    ``rt`` needs ``mb_slots >= n_microbatches``: microbatch k lives in buffer
    set k, so the packed boundary tensor is the runtime's DST_ACT buffers of
    sets 0..n-1 and no phase overwrites another microbatch's data.
    """

    def __init__(self, rt: BridgeRuntime, n_microbatches: int):
        if n_microbatches < 1:
            raise HetBridgeError(24, "n_microbatches must be >= 1")
        if rt.mb_slots < n_microbatches:
            raise HetBridgeError(24, f"runtime has {rt.mb_slots} buffer sets; the packed tensor needs "
                                     f"{n_microbatches} (one per microbatch)")
        self.rt, self.n = rt, n_microbatches
        self.src_ranks = rt.local_ranks(SLOT_SRC_ACT)
        self.dst_ranks = rt.local_ranks(SLOT_DST_ACT)
        self._enc_out = None
        self._leaves = None
        self.phase = 0

    # -- phase 1
    def source_view(self, mb: int, rank: int):
        """Where the encoder's projector may write microbatch ``mb`` of source
        rank ``rank`` directly (``torch.matmul(..., out=view)``): no copy."""
        return _view(self.rt, rank, SLOT_SRC_ACT, mb)

    def forward(self, encoder_outputs):
        """Phase 1. ``encoder_outputs[mb][i]``: the encoder output of microbatch
        ``mb`` for local source rank ``self.src_ranks[i]`` (part of the
        encoder's autograd graph). Runs the colocated forward transform for
        every microbatch and returns the packed tensor's leaves
        ``leaves[mb][j]`` for local destination rank ``self.dst_ranks[j]``."""
        if self.phase != 0:
            raise HetBridgeError(24, "phase 1 already ran; call backward() first")
        if len(encoder_outputs) != self.n:
            raise HetBridgeError(24, f"expected {self.n} microbatches, got {len(encoder_outputs)}")
        stream = torch.cuda.current_stream()
        for mb, outs in enumerate(encoder_outputs):
            if len(outs) != len(self.src_ranks):
                raise HetBridgeError(24, f"microbatch {mb}: expected {len(self.src_ranks)} source shards")
            for r, t in zip(self.src_ranks, outs):
                buf = self.source_view(mb, r)
                if t.data_ptr() != buf.data_ptr():
                    buf.copy_(t.detach().reshape(buf.shape))
            self.rt.forward(mb, stream)
        self._enc_out = encoder_outputs
        leaves = []
        for mb in range(self.n):
            row = []
            for r in self.dst_ranks:
                leaf = _view(self.rt, r, SLOT_DST_ACT, mb).detach().requires_grad_(True)
                g = _view(self.rt, r, SLOT_DST_GRAD, mb)
                g.zero_()
                if g.dtype == leaf.dtype:
                    leaf.grad = g  # AccumulateGrad adds LLM gradients into the DST_GRAD buffer in place
                row.append(leaf)
            leaves.append(row)
        self._leaves = leaves
        self.phase = 1
        return leaves

    # -- phase 2
    def view(self, mb: int, rank: int):
        """Phase 2: the detached leaf the LLM's PP0 consumes for microbatch ``mb``."""
        if self.phase != 1:
            raise HetBridgeError(24, "no packed boundary tensor: run phase 1 first")
        return self._leaves[mb][self.dst_ranks.index(rank)]

    # -- phase 3
    def backward(self, run_encoder_backward: bool = True):
        """Phase 3: hand the gradients accumulated on the packed tensor to the
        colocated backward transform (one launch per microbatch, gradients
        returned to the source owners), then run encoder backward through the
        saved encoder outputs. Returns ``grads[mb][i]`` (fp32, source layout)."""
        if self.phase != 1:
            raise HetBridgeError(24, "phase 3 needs phase 1")
        stream = torch.cuda.current_stream()
        for mb in range(self.n):
            for leaf, r in zip(self._leaves[mb], self.dst_ranks):
                buf = _view(self.rt, r, SLOT_DST_GRAD, mb)
                if leaf.grad is None:
                    buf.zero_()
                elif leaf.grad.data_ptr() != buf.data_ptr():  # autograd replaced .grad (e.g. set_to_none)
                    buf.copy_(leaf.grad.reshape(buf.shape))
            self.rt.backward(mb, 0.0, stream)
        grads = [[_view(self.rt, r, SLOT_SRC_GRAD, mb) for r in self.src_ranks] for mb in range(self.n)]
        if run_encoder_backward:
            outs, gs = [], []
            for mb in range(self.n):
                for t, g in zip(self._enc_out[mb], grads[mb]):
                    if t.requires_grad:
                        outs.append(t)
                        gs.append(g.to(t.dtype, copy=True).view(t.shape))  # never an alias of SRC_GRAD
            if outs:
                torch.autograd.backward(outs, gs)
        for row in self._leaves:
            for leaf in row:
                leaf.grad = None
        self._leaves = None
        self._enc_out = None
        self.phase = 0
        return grads
