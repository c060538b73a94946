"""Boundary communicator — Python face of ``hetsim::bridge`` (bridge.hpp:15-185).

``plan_bridge`` / ``export_plan`` / ``classify_dp_relation`` keep the
reference's names. ``BridgeRuntime`` replaces the reference's per-rank
runtime: one instance per process drives one GPU and executes, per boundary
op, the work of every logical rank resident on that GPU with one sm_100a
kernel launch (``csrc/kernels/boundary_kernels.cu``). ``bridge_forward`` /
``bridge_backward`` are the whole-edge test entry points (bridge.hpp:175-185)
with all logical ranks resident on one GPU.

There is no CPU fallback: every data-moving call goes through
``libhetbridge.so`` on a CUDA device and raises if it is unavailable.
"""
from __future__ import annotations

import ctypes
import enum
from dataclasses import dataclass

from . import _lib
from ._lib import HetBridgeError, check, lib
from .grid import BatchInterval, BoundaryEdge, ModuleLayout, Placement, partition_batch

SLOT_SRC_ACT, SLOT_DST_ACT, SLOT_DST_GRAD, SLOT_SRC_GRAD, SLOT_TEXT = range(5)
TEXT_FULL, TEXT_SLICE, TEXT_INPLACE = 0, 1, 2
HB_BF16, HB_FP16, HB_FP32, HB_FP64 = range(4)


class DpKind(enum.IntEnum):
    Equal = 0
    FanIn = 1
    FanOut = 2


@dataclass(frozen=True)
class DpRelation:
    kind: DpKind = DpKind.Equal
    factor: int = 1


def dp_kind_name(k: DpKind) -> str:
    return DpKind(k).name


def classify_dp_relation(edge: BoundaryEdge) -> DpRelation:
    k, f = ctypes.c_int(), ctypes.c_int()
    check(lib().hb_classify_dp_relation(ctypes.byref(edge._c()), ctypes.byref(k), ctypes.byref(f)))
    return DpRelation(DpKind(k.value), f.value)


class BridgePlan:
    """Compiled routing for one edge (bridge.hpp:122-135); owns an ``hb_plan*``."""

    def __init__(self, edge: BoundaryEdge):
        self.edge = edge
        h = ctypes.c_void_p()
        check(lib().hb_plan_create(ctypes.byref(edge._c()), ctypes.byref(h)))
        self._h = h
        pl, kind, fac, xm, world = (ctypes.c_int() for _ in range(5))
        check(lib().hb_plan_info(h, *(ctypes.byref(x) for x in (pl, kind, fac, xm, world))))
        self.placement = Placement(pl.value)
        self.relation = DpRelation(DpKind(kind.value), fac.value)
        self._xmsgs = xm.value
        self.world = world.value
        self.label = f"{edge.source.name}->{edge.dest.name}"
        self.src_intervals = partition_batch(edge.global_batch, edge.source.dp)
        self.dest_intervals = partition_batch(edge.global_batch, edge.dest.dp)

    def cross_boundary_messages(self) -> int:
        return self._xmsgs

    def __del__(self):
        try:
            h = getattr(self, "_h", None)
            if h and _lib._lib is not None:
                _lib._lib.hb_plan_destroy(h)
                self._h = None
        except Exception:  # interpreter shutdown
            pass


def hbb_fingerprint(plan: BridgePlan) -> str:
    return export_plan(plan, 8)


def plan_bridge(edge: BoundaryEdge) -> BridgePlan:
    return BridgePlan(edge)


def export_plan(plan: BridgePlan, elem_bytes: int = 8) -> str:
    n = ctypes.c_size_t()
    check(lib().hb_plan_export(plan._h, elem_bytes, None, 0, ctypes.byref(n)))
    buf = ctypes.create_string_buffer(n.value + 1)
    check(lib().hb_plan_export(plan._h, elem_bytes, buf, len(buf), ctypes.byref(n)))
    return buf.value.decode()


def cp_token_slice(seq_len: int, cp: int, cp_idx: int) -> BatchInterval:
    a, b = ctypes.c_int(), ctypes.c_int()
    check(lib().hb_cp_token_slice(seq_len, cp, cp_idx, ctypes.byref(a), ctypes.byref(b)))
    return BatchInterval(a.value, b.value)


class SpliceSpec:
    """Placeholder table for the embedding splice (generalises tinymodel.hpp:94-112).

    ``codes[q*S+p] >= 0``: vision token row ``j*S_v + t`` of the destination
    shard (local sample j, token t); ``< 0``: text row ``-1-code``.
    """

    def __init__(self, Q: int, S: int, d_h: int, S_v: int, codes, text_mode: int = TEXT_FULL):
        import numpy as np

        self.Q, self.S, self.d_h, self.S_v, self.text_mode = Q, S, d_h, S_v, text_mode
        self.codes = np.ascontiguousarray(np.asarray(codes, dtype=np.int32).reshape(-1))
        h = ctypes.c_void_p()
        check(lib().hb_splice_create(Q, S, d_h, S_v, text_mode,
                                     self.codes.ctypes.data_as(ctypes.POINTER(ctypes.c_int)),
                                     ctypes.byref(h)))
        self._h = h

    @staticmethod
    def reference_layout(n: int, S: int, S_v: int, d_h: int) -> "SpliceSpec":
        """tinymodel.hpp:24-26: vision tokens at [0,S_v) of each sample's sequence."""
        import numpy as np

        q = np.arange(n)[:, None]
        p = np.arange(S)[None, :]
        codes = np.where(p < S_v, q * S_v + p, -1 - (q * (S - S_v) + (p - S_v)))
        return SpliceSpec(n, S, d_h, S_v, codes, TEXT_FULL)

    def __del__(self):
        try:
            h = getattr(self, "_h", None)
            if h and _lib._lib is not None:
                _lib._lib.hb_splice_destroy(h)
                self._h = None
        except Exception:  # interpreter shutdown
            pass


def index_forward(plan: BridgePlan, splice: SpliceSpec | None = None):
    """Forward ownership map: list of (src_rank, src_slot, src_off, dst_rank, dst_slot, dst_off, n)."""
    n = ctypes.c_size_t()
    sh = splice._h if splice else None
    check(lib().hb_index_forward(plan._h, sh, None, 0, ctypes.byref(n)))
    arr = (_lib.CopySeg * max(n.value, 1))()
    check(lib().hb_index_forward(plan._h, sh, arr, n.value, ctypes.byref(n)))
    return [(s.src_rank, s.src_slot, s.src_off, s.dst_rank, s.dst_slot, s.dst_off, s.n)
            for s in arr[: n.value]]


def index_backward(plan: BridgePlan, splice: SpliceSpec | None = None, balanced: bool = False):
    """Backward map: list of (dst_rank, dst_slot, dst_off, n, [(rank, slot, off), ...]).

    balanced=False is the reference data path (tp=0 copies); True is the map the
    device runtime executes by default (terms read from the holder's tp replicas)."""
    n, tn = ctypes.c_size_t(), ctypes.c_size_t()
    sh = splice._h if splice else None
    fn = lib().hb_index_backward_balanced if balanced else lib().hb_index_backward
    check(fn(plan._h, sh, None, 0, ctypes.byref(n), None, 0, ctypes.byref(tn)))
    arr = (_lib.ReduceSeg * max(n.value, 1))()
    terms = (_lib.Ref * max(tn.value, 1))()
    check(fn(plan._h, sh, arr, n.value, ctypes.byref(n), terms, tn.value, ctypes.byref(tn)))
    out = []
    for s in arr[: n.value]:
        ts = [(t.rank, t.slot, t.off) for t in terms[s.term0: s.term0 + s.nterms]]
        out.append((s.dst_rank, s.dst_slot, s.dst_off, s.n, ts))
    return out


def buffer_elems(plan: BridgePlan, rank: int, slot: int, splice: SpliceSpec | None = None) -> int:
    v = ctypes.c_longlong()
    check(lib().hb_index_buffer_elems(plan._h, splice._h if splice else None, rank, slot,
                                      ctypes.byref(v)))
    return v.value


# ---------------------------------------------------------------------------- device


def _torch_dtype_code(dt) -> int:
    import torch

    table = {torch.bfloat16: HB_BF16, torch.float16: HB_FP16, torch.float32: HB_FP32,
             torch.float64: HB_FP64}
    if dt not in table:
        raise HetBridgeError(24, f"unsupported dtype {dt}")
    return table[dt]


class _CAI:
    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {"data": (ptr, False), "shape": (nbytes,), "typestr": "|u1",
                                         "version": 3, "strides": None}


class BridgeRuntime:
    """Per-process device runtime for one edge (replaces bridge.hpp:146-173).

    ``rank_to_gpu`` maps every logical rank of the edge to a GPU index in
    ``[0, n_gpus)``; this process drives ``my_gpu`` (the current CUDA device).
    ``forward(mb)`` / ``backward(mb, beta)`` launch one kernel each for all
    resident ranks. With ``n_gpus > 1`` construction is collective and
    :meth:`exchange_handles` must be called on every process before the first op.
    """

    def __init__(self, plan: BridgePlan, splice: SpliceSpec | None = None, *, n_gpus: int = 1,
                 my_gpu: int = 0, rank_to_gpu=None, act_dtype=None, grad_in_dtype=None,
                 grad_out_dtype=None, mb_slots: int = 1, internal_alloc: bool = True,
                 blocks_per_sm: int = 0, threads: int = 0, timeout_s: float = 0.0,
                 fwd_mode: int = 0, partition: int = 0, strict_provenance: bool = False,
                 text_embedding: bool = False, max_ctas: int = 0, max_ctas_bwd: int = 0,
                 tma_chunk_kib: int = 0):
        import torch

        self.plan, self.splice = plan, splice
        self.n_gpus, self.my_gpu = n_gpus, my_gpu
        self.rank_to_gpu = list(rank_to_gpu) if rank_to_gpu is not None else [0] * plan.world
        self.act_dtype = act_dtype or torch.bfloat16
        self.grad_in_dtype = grad_in_dtype or torch.bfloat16
        self.grad_out_dtype = grad_out_dtype or torch.float32
        self.mb_slots = mb_slots
        cfg = _lib.ExecConfig()
        lib().hb_exec_config_default(ctypes.byref(cfg))
        cfg.act_dtype = _torch_dtype_code(self.act_dtype)
        cfg.grad_in_dtype = _torch_dtype_code(self.grad_in_dtype)
        cfg.grad_out_dtype = _torch_dtype_code(self.grad_out_dtype)
        cfg.mb_slots = mb_slots
        cfg.internal_alloc = 1 if internal_alloc else 0
        cfg.blocks_per_sm = blocks_per_sm
        cfg.threads = threads
        cfg.timeout_s = timeout_s
        cfg.fwd_mode = fwd_mode  # 0 auto, 1 pull, 2 push
        cfg.partition = partition
        cfg.strict_provenance = 1 if strict_provenance else 0
        cfg.text_embedding = 1 if text_embedding else 0
        cfg.max_ctas = max_ctas
        cfg.max_ctas_bwd = max_ctas_bwd
        cfg.tma_chunk_kib = tma_chunk_kib
        self.text_embedding = bool(text_embedding)
        if not torch.cuda.is_available():
            raise HetBridgeError(25, "BridgeRuntime needs a CUDA device (no CPU fallback)")
        self.device = torch.device("cuda", torch.cuda.current_device())  # the exec's GPU
        m = (ctypes.c_int * len(self.rank_to_gpu))(*self.rank_to_gpu)
        h = ctypes.c_void_p()
        check(lib().hb_exec_create(plan._h, splice._h if splice else None, n_gpus, my_gpu, m,
                                   len(self.rank_to_gpu), ctypes.byref(cfg), ctypes.byref(h)))
        self._h = h
        self._keep = {}
        self._bind_dirty = False
        self._local_group = None  # set by LocalGroup (bindings shared in-process)

    # -- multi-GPU
    def ipc_handle(self) -> bytes:
        buf = ctypes.create_string_buffer(64)
        check(lib().hb_exec_ipc_handle(self._h, buf))
        return buf.raw

    def open_peers(self, handles: bytes):
        check(lib().hb_exec_open_peers(self._h, handles, len(handles)))

    def open_peers_local(self, runtimes):
        """Single-process group setup (hb_exec_open_peers_local): ``runtimes[g]``
        is this process's runtime of GPU g of the group."""
        arr = (ctypes.c_void_p * len(runtimes))(*[rt._h.value if rt is not None else None for rt in runtimes])
        check(lib().hb_exec_open_peers_local(self._h, arr, len(runtimes)))

    def exchange_handles(self, group=None):
        """All-gather the 64-byte IPC handles over torch.distributed and open peers."""
        import torch
        import torch.distributed as dist

        # every process must build the same buffer layout (same plan, map, dtypes, mb slots)
        import hashlib

        sp_fp = hashlib.sha256(self.splice.codes.tobytes()).hexdigest() if self.splice is not None else ""
        fp = hashlib.sha256(repr((hbb_fingerprint(self.plan), sp_fp, self.rank_to_gpu, str(self.act_dtype),
                                  str(self.grad_in_dtype), str(self.grad_out_dtype), self.mb_slots,
                                  self.n_gpus, self.text_embedding)).encode()).digest()
        fps = [None] * dist.get_world_size(group)
        dist.all_gather_object(fps, fp, group=group)
        if any(f != fp for f in fps):
            raise HetBridgeError(24, "BridgeRuntime configuration differs across processes")
        mine = torch.frombuffer(bytearray(self.ipc_handle()), dtype=torch.uint8)
        dev = torch.device("cuda", torch.cuda.current_device())
        backend = dist.get_backend(group)
        t = mine.to(dev) if backend == "nccl" else mine
        out = [torch.empty_like(t) for _ in range(dist.get_world_size(group))]
        dist.all_gather(out, t, group=group)
        self.open_peers(b"".join(bytes(o.cpu().numpy().tobytes()) for o in out))

    # -- buffers
    def _dtype_of(self, slot):
        import torch

        if slot == SLOT_TEXT and self.text_embedding:
            return torch.int32  # token ids, one per text row
        return {SLOT_DST_GRAD: self.grad_in_dtype, SLOT_SRC_GRAD: self.grad_out_dtype}.get(slot, self.act_dtype)

    def set_text_embedding(self, table):
        """Embedding table [vocab, d_h] (activation dtype, this GPU) that the
        splice gathers its text rows from (``text_embedding=True``)."""
        if not table.is_cuda or not table.is_contiguous() or table.dtype != self.act_dtype:
            raise HetBridgeError(24, "embedding table must be a contiguous CUDA tensor of the activation dtype")
        check(lib().hb_exec_set_text_embedding(self._h, ctypes.c_void_p(table.data_ptr()), table.shape[0]))
        self._keep["embedding"] = table

    def set_text_embedding_shard(self, rank: int, shard, vocab_begin: int, vocab: int):
        """Vocab-parallel table: resident ``rank`` holds rows [vocab_begin,
        vocab_begin + shard.shape[0]) of the [vocab, d_h] embedding table
        (Megatron's VocabParallelEmbedding; shards of a TP group equal-sized, in
        tp order). The splice gathers each text row from the rank owning its id,
        locally or from a peer GPU. In a multi-process group call
        :meth:`exchange_bindings` on every process afterwards (collective)."""
        if not shard.is_cuda or not shard.is_contiguous() or shard.dtype != self.act_dtype or shard.dim() != 2:
            raise HetBridgeError(24, "embedding shard must be a contiguous 2-D CUDA tensor of the activation dtype")
        check(lib().hb_exec_set_text_embedding_shard(self._h, rank, ctypes.c_void_p(shard.data_ptr()), vocab_begin,
                                                     shard.shape[0], vocab))
        self._keep[("embedding_shard", rank)] = shard
        self._bind_dirty = True

    def buffer(self, rank: int, slot: int, mb_slot: int = 0):
        """Device tensor view (1-D, element dtype of the slot) of a resident rank's buffer."""
        import torch

        if (rank, slot, mb_slot) in self._keep:  # a caller-bound tensor (possibly row-strided)
            return self._keep[(rank, slot, mb_slot)]
        p, n = ctypes.c_void_p(), ctypes.c_size_t()
        check(lib().hb_exec_buffer(self._h, rank, slot, mb_slot, ctypes.byref(p), ctypes.byref(n)))
        if not p.value or n.value == 0:
            return None
        raw = torch.as_tensor(_CAI(p.value, n.value), device=self.device)
        return raw.view(self._dtype_of(slot))

    def bind(self, rank: int, slot: int, tensor, mb_slot: int = 0, row_stride: int | None = None):
        """Use a caller-owned CUDA tensor as a resident rank's buffer (no copy).

        ``tensor``: 1-D contiguous, or 2-D [rows, row width] with a unit inner
        stride (its row stride is taken from ``tensor.stride(0)`` unless
        ``row_stride`` is given). ``None`` reverts to the runtime's region. In a
        multi-GPU group call :meth:`exchange_bindings` on every process
        afterwards (collective)."""
        if tensor is None:
            check(lib().hb_exec_bind(self._h, rank, slot, mb_slot, None, 0))
            self._bind_dirty |= self._keep.pop((rank, slot, mb_slot), None) is not None
            return
        if not tensor.is_cuda:
            raise HetBridgeError(24, "bind needs a CUDA tensor")
        if tensor.dtype != self._dtype_of(slot):
            raise HetBridgeError(13, f"slot {slot} expects {self._dtype_of(slot)}, got {tensor.dtype}")
        if tensor.dim() == 2 and tensor.stride(1) == 1:
            stride = tensor.stride(0) if row_stride is None else row_stride
            nbytes = ((tensor.shape[0] - 1) * tensor.stride(0) + tensor.shape[1]) * tensor.element_size()
        elif tensor.is_contiguous():
            stride = row_stride or 0
            nbytes = tensor.numel() * tensor.element_size()
        else:
            raise HetBridgeError(24, "bind needs a contiguous tensor or rows with a unit inner stride")
        old = self._keep.get((rank, slot, mb_slot))
        if old is not None and old.data_ptr() == tensor.data_ptr() and old.stride() == tensor.stride() and \
                old.shape == tensor.shape:
            self._keep[(rank, slot, mb_slot)] = tensor
            return  # already bound here: tables and graphs stay valid
        check(lib().hb_exec_bind_strided(self._h, rank, slot, mb_slot, ctypes.c_void_p(tensor.data_ptr()),
                                         nbytes, stride))
        self._keep[(rank, slot, mb_slot)] = tensor
        self._bind_dirty = True

    def sync_bindings(self, group=None):
        """Collective at N > 1: exchange bindings if any process rebound a
        buffer since the last exchange (one tiny all-reduce otherwise)."""
        if self.n_gpus == 1 or self._local_group is not None:
            self._bind_dirty = False
            return
        import torch
        import torch.distributed as dist

        dev = self.device if dist.get_backend(group) == "nccl" else "cpu"
        flag = torch.tensor([1 if self._bind_dirty else 0], device=dev)
        dist.all_reduce(flag, op=dist.ReduceOp.MAX, group=group)
        if flag.item():
            self.exchange_bindings(group)

    def exchange_bindings(self, group=None):
        """Collective: all-gather every process's binding blob (CUDA IPC handles
        of its caller-bound buffers) and import the peers' ones."""
        import torch.distributed as dist

        n = ctypes.c_size_t()
        check(lib().hb_exec_export_bindings(self._h, None, 0, ctypes.byref(n)))
        buf = ctypes.create_string_buffer(n.value)
        check(lib().hb_exec_export_bindings(self._h, buf, n.value, ctypes.byref(n)))
        blobs = [None] * dist.get_world_size(group)
        dist.all_gather_object(blobs, (self.my_gpu, buf.raw[: n.value]), group=group)
        for g, blob in blobs:
            if g != self.my_gpu:
                check(lib().hb_exec_import_bindings(self._h, g, blob, len(blob)))
        self._bind_dirty = False

    def buffer_numel(self, rank: int, slot: int) -> int:
        """Elements of a logical rank's buffer (0: the rank has none in this slot)."""
        return buffer_elems(self.plan, rank, slot, self.splice)

    def local_ranks(self, slot: int) -> list[int]:
        """Logical ranks resident on this GPU that own a buffer in ``slot``, ascending."""
        return [r for r in range(self.plan.world)
                if self.rank_to_gpu[r] == self.my_gpu and self.buffer_numel(r, slot) > 0]

    # -- ops
    @staticmethod
    def _stream(stream):
        import torch

        s = stream if stream is not None else torch.cuda.current_stream()
        return ctypes.c_void_p(s.cuda_stream)

    def forward(self, mb: int = 0, stream=None):
        check(lib().hb_exec_forward(self._h, mb, self._stream(stream)))

    def forward_projected(self, mb: int, x, w, stream=None):
        """Forward with the encoder projector fused in (hb_exec_forward_projected):
        x [rows, K] bf16 = pre-projection token rows of the local source ranks
        stacked in ascending rank order (``rows`` = those ranks' token rows; x
        may be None when this GPU hosts no source rank); w [d_h, K] bf16. Each
        projected row goes straight to every destination row; SRC_ACT is not
        written."""
        import torch

        if w.dtype != torch.bfloat16 or w.dim() != 2 or w.stride(1) != 1:
            raise HetBridgeError(24, "forward_projected takes a row-major bf16 weight [d_h, K]")
        d_h, K = w.shape
        rows = sum(self.buffer_numel(r, SLOT_SRC_ACT) for r in self.local_ranks(SLOT_SRC_ACT)) // d_h
        if x is None:
            if rows:
                raise HetBridgeError(13, f"forward_projected needs x [{rows}, {K}] for the local source ranks")
            xp, ldx = None, K
        else:
            if x.dtype != torch.bfloat16 or x.dim() != 2 or x.stride(1) != 1 or not x.is_cuda:
                raise HetBridgeError(24, "forward_projected takes a row-major bf16 CUDA x [rows, K]")
            if tuple(x.shape) != (rows, K):
                raise HetBridgeError(13, f"x is {tuple(x.shape)}, the local source ranks need ({rows}, {K})")
            xp, ldx = ctypes.c_void_p(x.data_ptr()), x.stride(0)
        check(lib().hb_exec_forward_projected(self._h, mb, xp, rows, ldx, ctypes.c_void_p(w.data_ptr()),
                                              w.stride(0), d_h, K, self._stream(stream)))

    def backward(self, mb: int = 0, beta: float = 0.0, stream=None):
        check(lib().hb_exec_backward(self._h, mb, ctypes.c_float(beta), self._stream(stream)))

    def paired(self, fwd_mb: int, bwd_mb: int, beta: float = 0.0, stream=None) -> bool:
        """forward(fwd_mb) and backward(bwd_mb, beta) in one fused launch (a
        1F1B schedule call). Peers may issue the two ops separately. Returns
        True if the fused kernel ran (False: two launches)."""
        fused = ctypes.c_int(0)
        check(lib().hb_exec_paired(self._h, fwd_mb, bwd_mb, ctypes.c_float(beta), self._stream(stream),
                                   ctypes.byref(fused)))
        return bool(fused.value)

    GRAPH_FWD, GRAPH_STEP, GRAPH_BWD, GRAPH_CYCLE, GRAPH_PAIRED, GRAPH_PAIRED_FUSED = 0, 1, 2, 3, 4, 5

    def capture_step(self, mb_slot: int = 0, beta: float = 1.0, with_backward: bool = True, stream=None,
                     what: int | None = None):
        """Capture one buffer set's ops into a CUDA graph (what: 0 fwd, 1 fwd+bwd, 2 bwd;
        3 = fwd+bwd of every buffer set in order, one graph per cycle of mb_slots steps;
        4 = the 1F1B-paired cycle: step k = fwd of set k concurrently with bwd of set k-1)."""
        what = (1 if with_backward else 0) if what is None else what
        check(lib().hb_exec_graph_capture(self._h, mb_slot, what, ctypes.c_float(beta), self._stream(stream)))

    def replay_step(self, mb_slot: int = 0, stream=None, what: int = 1):
        check(lib().hb_exec_graph_launch(self._h, mb_slot, what, self._stream(stream)))

    def seed_forward_record(self, mb: int):
        check(lib().hb_exec_seed_forward_record(self._h, mb))

    def status(self) -> int:
        e = ctypes.c_uint()
        check(lib().hb_exec_status(self._h, ctypes.byref(e)))
        return e.value

    def reset_protocol(self, group=None):
        """Recover the exec group after a Timeout / GroupMismatch (collective:
        every process calls it; barriers on both sides of the reset)."""
        import torch

        torch.cuda.synchronize(self.device)
        multi = self.n_gpus > 1 and self._local_group is None
        if multi:
            import torch.distributed as dist

            dist.barrier(group)
        check(lib().hb_exec_reset_protocol(self._h))
        if multi:
            dist.barrier(group)

    def stats(self) -> dict:
        v = [ctypes.c_longlong() for _ in range(5)]
        check(lib().hb_exec_stats(self._h, *(ctypes.byref(x) for x in v)))
        keys = ["fwd_segments", "bwd_segments", "fwd_bytes", "bwd_elems", "launches"]
        return dict(zip(keys, (x.value for x in v)))

    def validate(self) -> int:
        """Static race and bounds check of this exec's device tables
        (hb_exec_validate); raises HetBridgeError("ValidationError") on the
        first violation, else returns the number of items checked."""
        n = ctypes.c_longlong()
        check(lib().hb_exec_validate(self._h, ctypes.byref(n)))
        return n.value

    def trace(self, kind: int):
        """HB_TRACE=1 diagnostics: per-CTA stamps of the last launch of `kind`
        (0 fwd, 1 bwd) as a [ctas x 8] uint64 numpy array (empty when off)."""
        import numpy as np

        grid, n = ctypes.c_int(), ctypes.c_int()
        check(lib().hb_exec_trace(self._h, kind, None, 0, ctypes.byref(n), ctypes.byref(grid)))
        out = np.zeros((max(grid.value, 1), 8), dtype=np.uint64)
        check(lib().hb_exec_trace(self._h, kind, out.ctypes.data, grid.value, ctypes.byref(n), ctypes.byref(grid)))
        return out[:n.value]

    def close(self):
        h = getattr(self, "_h", None)
        if h and _lib._lib is not None:
            _lib._lib.hb_exec_destroy(h)
        self._h = None
        self._keep = {}

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class LocalGroup:
    """One process driving a whole exec group: one :class:`BridgeRuntime` per
    (virtual) GPU g on ``devices[g]``, peers opened with
    hb_exec_open_peers_local, each op launched on every GPU's stream from this
    thread (the kernels of one op run concurrently and meet in the in-kernel
    barrier). ``devices`` may repeat a device: several execs then share it and
    ``max_ctas`` (default: an equal share of two CTAs per SM) keeps their grids
    co-resident, so the cross-GPU protocol runs on a single physical GPU."""

    def __init__(self, plan: BridgePlan, splice: SpliceSpec | None = None, *, devices, rank_to_gpu=None,
                 max_ctas: int | None = None, **kw):
        import torch

        self.devices = [torch.device("cuda", d) if isinstance(d, int) else torch.device(d) for d in devices]
        n = len(self.devices)
        shared = len({d.index for d in self.devices}) < n
        if max_ctas is None:
            per_dev = {}
            for d in self.devices:
                per_dev[d.index] = per_dev.get(d.index, 0) + 1
            sms = torch.cuda.get_device_properties(self.devices[0]).multi_processor_count
            max_ctas = (2 * sms) // max(per_dev.values()) if shared else 0
        from .configs import rank_to_gpu as _r2g

        r2g = list(rank_to_gpu) if rank_to_gpu is not None else _r2g(plan.world, n)
        self.rts, self.streams = [], []
        for g, d in enumerate(self.devices):
            with torch.cuda.device(d):
                self.rts.append(BridgeRuntime(plan, splice, n_gpus=n, my_gpu=g, rank_to_gpu=r2g,
                                              max_ctas=max_ctas, **kw))
                self.streams.append(torch.cuda.Stream(device=d))
        for rt in self.rts:
            rt.open_peers_local(self.rts)
            rt._local_group = self
        self.plan, self.splice, self.rank_to_gpu, self.max_ctas = plan, splice, r2g, max_ctas

    def runtime_of(self, rank: int) -> "BridgeRuntime":
        return self.rts[self.rank_to_gpu[rank]]

    def buffer(self, rank: int, slot: int, mb_slot: int = 0):
        return self.runtime_of(rank).buffer(rank, slot, mb_slot)

    def bind(self, rank: int, slot: int, tensor, mb_slot: int = 0, row_stride: int | None = None):
        """Caller-owned buffer for ``rank`` (on its GPU); every exec re-reads its
        peers' bindings (hb_exec_open_peers_local)."""
        self.runtime_of(rank).bind(rank, slot, tensor, mb_slot, row_stride)
        for rt in self.rts:
            rt.open_peers_local(self.rts)

    def set_text_embedding_shard(self, rank: int, shard, vocab_begin: int, vocab: int):
        self.runtime_of(rank).set_text_embedding_shard(rank, shard, vocab_begin, vocab)

    def reset_protocol(self):
        """Recover every exec of the group after a Timeout / GroupMismatch."""
        self.synchronize()
        for rt in self.rts:
            rt.reset_protocol()

    def forward(self, mb: int = 0):
        for rt, st in zip(self.rts, self.streams):
            rt.forward(mb, st)

    def backward(self, mb: int = 0, beta: float = 0.0):
        for rt, st in zip(self.rts, self.streams):
            rt.backward(mb, beta, st)

    def paired(self, fwd_mb: int, bwd_mb: int, beta: float = 0.0, fuse=None):
        """fuse[g] False: GPU g issues the two ops as separate launches (the
        peers' fused launches must interoperate with it). Returns, per GPU,
        whether one fused launch ran."""
        out = []
        for g, (rt, st) in enumerate(zip(self.rts, self.streams)):
            if fuse is None or fuse[g]:
                out.append(rt.paired(fwd_mb, bwd_mb, beta, st))
            else:
                rt.forward(fwd_mb, st)
                rt.backward(bwd_mb, beta, st)
                out.append(False)
        return out

    def synchronize(self):
        for st in self.streams:
            st.synchronize()

    def status(self) -> int:
        return max(rt.status() for rt in self.rts)

    def close(self):
        self.synchronize()
        for rt in self.rts:
            rt.close()
        self.rts = []


def _stage_ranks(layout: ModuleLayout, stage: int):
    from .grid import ranks_of_stage

    return ranks_of_stage(layout, stage)


def bridge_forward(plan: BridgePlan, shards: dict, mb: int = 0, splice: SpliceSpec | None = None,
                   text: dict | None = None):
    """Whole edge on one GPU (bridge.hpp:178-181): {src rank: tensor} -> {dest rank: tensor}.

    Outputs are (rows, feature_width) for a plain edge, or (Q*L, d_h) token
    slices when ``splice`` is given. Tensors must share one CUDA device and dtype.
    """
    import torch

    any_t = next(iter(shards.values()))
    rt = BridgeRuntime(plan, splice, act_dtype=any_t.dtype, internal_alloc=False)
    for r, t in shards.items():
        rt.bind(r, SLOT_SRC_ACT, t.contiguous().view(-1))
    for r, t in (text or {}).items():
        rt.bind(r, SLOT_TEXT, t.contiguous().view(-1))
    outs = {}
    for r in _stage_ranks(plan.edge.dest, 0):
        n = buffer_elems(plan, r, SLOT_DST_ACT, splice)
        o = torch.empty(n, dtype=any_t.dtype, device=any_t.device)
        rt.bind(r, SLOT_DST_ACT, o)
        width = splice.d_h if splice else plan.edge.feature_width
        outs[r] = o.view(-1, width)
    rt.forward(mb)
    torch.cuda.current_stream().synchronize()
    rt.close()
    return outs


def bridge_backward(plan: BridgePlan, grads: dict, mb: int = 0, splice: SpliceSpec | None = None,
                    out_dtype=None, accumulate_into: dict | None = None, beta: float = 0.0):
    """Whole edge on one GPU (bridge.hpp:182-185): {dest rank: grad} -> {src rank: grad}.

    ``accumulate_into`` supplies existing source-gradient tensors that receive
    ``beta*old + returned`` (fp32 accumulation).
    """
    import torch

    import torch as _t

    any_t = next(iter(grads.values()))
    out_dtype = out_dtype or (next(iter(accumulate_into.values())).dtype if accumulate_into else _t.float32)
    rt = BridgeRuntime(plan, splice, grad_in_dtype=any_t.dtype, grad_out_dtype=out_dtype,
                       internal_alloc=False)
    rt.seed_forward_record(mb)
    for r, t in grads.items():
        rt.bind(r, SLOT_DST_GRAD, t.contiguous().view(-1))
    outs = {}
    for r in _stage_ranks(plan.edge.source, plan.edge.source.pp - 1):
        if accumulate_into and r in accumulate_into:
            o = accumulate_into[r].view(-1)
        else:
            o = torch.empty(buffer_elems(plan, r, SLOT_SRC_GRAD, splice), dtype=out_dtype,
                            device=any_t.device)
        rt.bind(r, SLOT_SRC_GRAD, o)
        outs[r] = o.view(-1, plan.edge.feature_width)
    rt.backward(mb, beta)
    torch.cuda.current_stream().synchronize()
    rt.close()
    return outs
