"""ctypes binding of the hetbridge C-ABI (``include/hetbridge.h``).

The product path is ``libhetbridge.so`` built in-tree for sm_100a. There is no
CPU fallback: if the library is missing, importing the device entry points
fails loudly.
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# HB_LIB_PATH: an alternative in-tree build (A/B experiments only)
LIB_PATH = os.environ.get("HB_LIB_PATH") or os.path.join(HERE, "libhetbridge.so")

ERROR_NAMES = [
    "RankOutOfModule", "CoordOutOfBounds", "IndivisibleBatch", "PartialOverlap", "NonIntegerFan",
    "PlanInfeasible", "ShardIntervalMismatch", "MissingSourceShard", "GradIntervalMismatch",
    "UnknownMicrobatch", "Deadlock", "GroupMismatch", "ShapeMismatch", "ChannelMismatch",
    "SnapshotWhileActive", "DivisibilityViolation", "CyclicGraph", "DanglingEdge",
    "InfeasibleSchedule", "NotColocated", "StructureMismatch", "ParseError", "ValidationError",
    "InvalidArgument", "CudaError", "Timeout",
]

# Exported symbols declared in include/hetbridge.h (checked by tests).
EXPORTS = [
    "hb_last_error", "hb_error_name", "hb_abi_version",
    "hb_coord_of_rank", "hb_rank_of_coord", "hb_partition_batch", "hb_leader_rank",
    "hb_placement_of_edge", "hb_ranks_of_stage", "hb_replica_group", "hb_module_group",
    "hb_classify_dp_relation", "hb_plan_create", "hb_plan_destroy", "hb_plan_export", "hb_plan_info",
    "hb_cp_token_slice", "hb_splice_create", "hb_splice_destroy",
    "hb_index_forward", "hb_index_backward", "hb_index_backward_balanced", "hb_index_buffer_elems",
    "hb_exec_config_default", "hb_exec_create", "hb_exec_destroy", "hb_exec_ipc_handle",
    "hb_exec_open_peers", "hb_exec_open_peers_local", "hb_exec_buffer", "hb_exec_bind", "hb_exec_bind_strided",
    "hb_exec_export_bindings", "hb_exec_import_bindings", "hb_exec_forward", "hb_exec_backward", "hb_exec_paired",
    "hb_exec_seed_forward_record", "hb_exec_status", "hb_exec_reset_protocol", "hb_exec_stats", "hb_exec_graph_capture", "hb_projector_gemm",
    "hb_exec_forward_projected", "hb_exec_set_text_embedding", "hb_exec_set_text_embedding_shard",
    "hb_exec_graph_launch", "hb_exec_trace", "hb_exec_validate",
    "hb_stage_graph_create", "hb_stage_graph_destroy", "hb_stage_graph_nodes", "hb_stage_graph_edges",
    "hb_dispatch_generate", "hb_dispatch_validate", "hb_dispatch_render", "hb_dispatch_nc_order",
    "hb_nccl_unique_id", "hb_runtime_config_default", "hb_runtime_create", "hb_runtime_destroy", "hb_runtime_info",
    "hb_runtime_group", "hb_runtime_edge_exec", "hb_runtime_stage_buffer", "hb_runtime_stream", "hb_runtime_step",
    "hb_runtime_last_step_ms", "hb_runtime_paired_ops",
    "hb_config_parse", "hb_config_destroy", "hb_config_num_modules", "hb_config_module", "hb_config_run",
    "hb_config_edge", "hb_config_render",
]


class HetBridgeError(RuntimeError):
    """A non-zero C-ABI status; ``code`` is the reference ErrorCode name."""

    def __init__(self, status: int, message: str):
        self.status = status
        self.code = ERROR_NAMES[status - 1] if 1 <= status <= len(ERROR_NAMES) else f"status{status}"
        super().__init__(message)


class Layout(ctypes.Structure):
    _fields_ = [("name", ctypes.c_char_p), ("tp", ctypes.c_int), ("cp", ctypes.c_int),
                ("pp", ctypes.c_int), ("dp", ctypes.c_int), ("rank_offset", ctypes.c_int)]


class Edge(ctypes.Structure):
    _fields_ = [("source", Layout), ("dest", Layout), ("global_batch", ctypes.c_int),
                ("feature_width", ctypes.c_int)]


class CopySeg(ctypes.Structure):
    _fields_ = [("src_rank", ctypes.c_int), ("src_slot", ctypes.c_int), ("src_off", ctypes.c_longlong),
                ("dst_rank", ctypes.c_int), ("dst_slot", ctypes.c_int), ("dst_off", ctypes.c_longlong),
                ("n", ctypes.c_longlong)]


class Ref(ctypes.Structure):
    _fields_ = [("rank", ctypes.c_int), ("slot", ctypes.c_int), ("off", ctypes.c_longlong)]


class ReduceSeg(ctypes.Structure):
    _fields_ = [("dst_rank", ctypes.c_int), ("dst_slot", ctypes.c_int), ("dst_off", ctypes.c_longlong),
                ("n", ctypes.c_longlong), ("nterms", ctypes.c_int), ("term0", ctypes.c_int)]


class Cell(ctypes.Structure):
    _fields_ = [("row", ctypes.c_int), ("node", ctypes.c_int), ("op", ctypes.c_int), ("edge", ctypes.c_int),
                ("kind", ctypes.c_int), ("mb", ctypes.c_int), ("bwd", ctypes.c_int)]


class ExecConfig(ctypes.Structure):
    _fields_ = [("act_dtype", ctypes.c_int), ("grad_in_dtype", ctypes.c_int),
                ("grad_out_dtype", ctypes.c_int), ("mb_slots", ctypes.c_int),
                ("internal_alloc", ctypes.c_int), ("blocks_per_sm", ctypes.c_int),
                ("threads", ctypes.c_int), ("timeout_s", ctypes.c_double), ("fwd_mode", ctypes.c_int),
                ("partition", ctypes.c_int), ("strict_provenance", ctypes.c_int),
                ("text_embedding", ctypes.c_int), ("max_ctas", ctypes.c_int), ("max_ctas_bwd", ctypes.c_int),
                ("tma_chunk_kib", ctypes.c_int)]


_lib = None


def _declare(L):
    I, U, Sz, V, C = ctypes.c_int, ctypes.c_uint, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_char_p
    P = ctypes.POINTER
    LL = ctypes.c_longlong
    sig = {
        "hb_last_error": (Sz, [C, Sz]),
        "hb_error_name": (C, [I]),
        "hb_abi_version": (I, []),
        "hb_coord_of_rank": (I, [P(Layout), I, P(I)]),
        "hb_rank_of_coord": (I, [P(Layout), P(I), P(I)]),
        "hb_partition_batch": (I, [I, I, P(I), I]),
        "hb_leader_rank": (I, [P(Layout), I, I, P(I)]),
        "hb_placement_of_edge": (I, [P(Edge), P(I)]),
        "hb_ranks_of_stage": (I, [P(Layout), I, P(I), I, P(I)]),
        "hb_replica_group": (I, [P(Layout), I, I, P(I), I, P(I)]),
        "hb_module_group": (I, [P(Layout), I, I, P(I), I, P(I)]),
        "hb_classify_dp_relation": (I, [P(Edge), P(I), P(I)]),
        "hb_plan_create": (I, [P(Edge), P(V)]),
        "hb_plan_destroy": (None, [V]),
        "hb_plan_export": (I, [V, I, C, Sz, P(Sz)]),
        "hb_plan_info": (I, [V, P(I), P(I), P(I), P(I), P(I)]),
        "hb_cp_token_slice": (I, [I, I, I, P(I), P(I)]),
        "hb_splice_create": (I, [I, I, I, I, I, P(I), P(V)]),
        "hb_splice_destroy": (None, [V]),
        "hb_index_forward": (I, [V, V, P(CopySeg), Sz, P(Sz)]),
        "hb_index_backward": (I, [V, V, P(ReduceSeg), Sz, P(Sz), P(Ref), Sz, P(Sz)]),
        "hb_index_backward_balanced": (I, [V, V, P(ReduceSeg), Sz, P(Sz), P(Ref), Sz, P(Sz)]),
        "hb_index_buffer_elems": (I, [V, V, I, I, P(LL)]),
        "hb_exec_config_default": (None, [P(ExecConfig)]),
        "hb_exec_create": (I, [V, V, I, I, P(I), I, P(ExecConfig), P(V)]),
        "hb_exec_destroy": (None, [V]),
        "hb_exec_ipc_handle": (I, [V, V]),
        "hb_exec_open_peers": (I, [V, V, Sz]),
        "hb_exec_open_peers_local": (I, [V, P(V), I]),
        "hb_exec_buffer": (I, [V, I, I, I, P(V), P(Sz)]),
        "hb_exec_bind": (I, [V, I, I, I, V, Sz]),
        "hb_exec_bind_strided": (I, [V, I, I, I, V, Sz, LL]),
        "hb_exec_export_bindings": (I, [V, V, Sz, P(Sz)]),
        "hb_exec_import_bindings": (I, [V, I, V, Sz]),
        "hb_exec_forward": (I, [V, I, V]),
        "hb_exec_backward": (I, [V, I, ctypes.c_float, V]),
        "hb_exec_paired": (I, [V, I, I, ctypes.c_float, V, ctypes.POINTER(ctypes.c_int)]),
        "hb_exec_seed_forward_record": (I, [V, I]),
        "hb_exec_graph_capture": (I, [V, I, I, ctypes.c_float, V]),
        "hb_exec_graph_launch": (I, [V, I, I, V]),
        "hb_exec_status": (I, [V, P(U)]),
        "hb_exec_reset_protocol": (I, [V]),
        "hb_exec_stats": (I, [V, P(LL), P(LL), P(LL), P(LL), P(LL)]),
        "hb_projector_gemm": (I, [V, LL, V, LL, V, I, I, I, I, V]),
        "hb_exec_forward_projected": (I, [V, I, V, LL, LL, V, LL, I, I, V]),
        "hb_exec_set_text_embedding": (I, [V, V, LL]),
        "hb_exec_set_text_embedding_shard": (I, [V, I, V, LL, LL, LL]),
        "hb_exec_trace": (I, [V, I, V, I, P(I), P(I)]),
        "hb_exec_validate": (I, [V, P(LL)]),
        "hb_stage_graph_create": (I, [P(Layout), I, P(I), P(I), I, P(V)]),
        "hb_stage_graph_destroy": (None, [V]),
        "hb_stage_graph_nodes": (I, [V, P(I), I, P(I)]),
        "hb_stage_graph_edges": (I, [V, P(I), I, P(I)]),
        "hb_dispatch_generate": (I, [V, I, P(Cell), Sz, P(Sz), P(I)]),
        "hb_dispatch_validate": (I, [V, P(Cell), Sz, I, C, Sz, P(Sz), P(I)]),
        "hb_dispatch_render": (I, [V, I, C, Sz, P(Sz)]),
        "hb_dispatch_nc_order": (I, [V, I, I, P(Cell), Sz, P(Sz)]),
        "hb_config_parse": (I, [C, P(V)]),
        "hb_config_destroy": (None, [V]),
        "hb_config_num_modules": (I, [V, P(I)]),
        "hb_config_module": (I, [V, I, P(Layout), P(I)]),
        "hb_config_run": (I, [V, P(I), P(I), P(I), P(LL), P(ctypes.c_double)]),
        "hb_config_edge": (I, [V, C, I, P(Edge)]),
        "hb_config_render": (I, [V, C, Sz, P(Sz)]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name, None)
        if f is None and os.environ.get("HB_LIB_PATH"):  # older A/B build: skip newer entry points
            continue
        if f is None:
            raise ImportError(f"{LIB_PATH} does not export {name}")
        f.restype = res
        f.argtypes = args


def lib():
    """Load libhetbridge.so; raises if it was not built (no fallback path)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"hetbridge native library not built: {LIB_PATH} is missing "
                "(run __graft_entry__.build() or `make -C paper_2605_27678_b200/csrc`)")
        _lib = ctypes.CDLL(LIB_PATH)
        _declare(_lib)
    return _lib


def last_error() -> str:
    buf = ctypes.create_string_buffer(4096)
    lib().hb_last_error(buf, len(buf))
    return buf.value.decode(errors="replace")


def check(status: int):
    if status != 0:
        raise HetBridgeError(status, last_error())
