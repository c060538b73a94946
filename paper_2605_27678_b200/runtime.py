"""Host-owned per-module runtime — Python face of ``hb_runtime_*``
(the C++ is csrc/hb/runtime_host.cpp).

One :class:`HostRuntime` per process (one GPU) for modules with disjoint rank
ranges. The C++ host owns this rank's per-module groups, an NCCL world
communicator and each module's PP communicator (``ncclCommSplit``), one
boundary exec per module edge, a highest-priority boundary stream, a PP stream
and a compute stream; :meth:`step` enqueues this rank's column of the
graph-aware 1F1B dispatch table (``sched.generate_1f1b_dispatch``): P2P cells
as grouped NCCL send/recv, NC cells as the edge exec's forward/backward,
compute cells through a callback, ordered by CUDA events. Python only
broadcasts the NCCL unique id (torch.distributed) and hands over callbacks.
"""
from __future__ import annotations

import ctypes

from . import _lib
from ._lib import check, lib
from .bridge import BridgeRuntime, plan_bridge
from .grid import BoundaryEdge

COMPUTE_FN = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p)

SKIP_NC, SKIP_P2P, SKIP_COMPUTE = 1, 2, 4
ACT_IN, ACT_OUT, GRAD_IN, GRAD_OUT = range(4)


class RuntimeConfig(ctypes.Structure):
    _fields_ = [("nmb", ctypes.c_int), ("max_ctas", ctypes.c_int), ("pp_bytes", ctypes.c_longlong),
                ("act_dtype", ctypes.c_int), ("grad_in_dtype", ctypes.c_int), ("grad_out_dtype", ctypes.c_int),
                ("timeout_s", ctypes.c_double), ("skip", ctypes.c_int)]


def _declare():
    L = lib()
    if getattr(L, "_hb_rt_declared", False):
        return L
    I, V, Sz, LL = ctypes.c_int, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_longlong
    P = ctypes.POINTER
    sig = {
        "hb_nccl_unique_id": (I, [V]),
        "hb_runtime_config_default": (None, [P(RuntimeConfig)]),
        "hb_runtime_create": (I, [P(_lib.Layout), I, P(I), P(I), I, I, I, I, I, V, P(RuntimeConfig), P(V)]),
        "hb_runtime_destroy": (None, [V]),
        "hb_runtime_info": (I, [V, P(I), P(I), P(I), P(I)]),
        "hb_runtime_group": (I, [V, I, P(I), I, P(I)]),
        "hb_runtime_edge_exec": (I, [V, I, P(V)]),
        "hb_runtime_stage_buffer": (I, [V, I, I, P(V), P(Sz)]),
        "hb_runtime_stream": (I, [V, I, P(V)]),
        "hb_runtime_step": (I, [V, COMPUTE_FN, V]),
        "hb_runtime_last_step_ms": (I, [V, P(ctypes.c_float)]),
        "hb_runtime_paired_ops": (I, [V, P(ctypes.c_longlong)]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype, f.argtypes = res, args
    L._hb_rt_declared = True
    return L


def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    check(_declare().hb_nccl_unique_id(buf))
    return buf.raw


class HostRuntime:
    """modules: ModuleLayouts with disjoint rank ranges; edges: (source module,
    dest module) index pairs; every process of the torch.distributed world
    constructs it (collective)."""

    def __init__(self, modules, edges, global_batch: int, feature_width: int, *, nmb: int = 4,
                 max_ctas: int = 0, pp_bytes: int = 0, act_dtype=None, grad_in_dtype=None, grad_out_dtype=None,
                 timeout_s: float = 20.0, skip: int = 0, group=None):
        import torch
        import torch.distributed as dist

        from .bridge import _torch_dtype_code

        L = _declare()
        self.modules, self.edges = list(modules), [tuple(e) for e in edges]
        self.global_batch, self.feature_width, self.nmb = global_batch, feature_width, nmb
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        obj = [nccl_unique_id() if self.rank == 0 else None]
        dist.broadcast_object_list(obj, src=0, group=group)
        cfg = RuntimeConfig()
        L.hb_runtime_config_default(ctypes.byref(cfg))
        cfg.nmb, cfg.max_ctas, cfg.pp_bytes, cfg.timeout_s, cfg.skip = nmb, max_ctas, pp_bytes, timeout_s, skip
        self.act_dtype = act_dtype or torch.bfloat16
        self.grad_in_dtype = grad_in_dtype or torch.bfloat16
        self.grad_out_dtype = grad_out_dtype or torch.float32
        cfg.act_dtype = _torch_dtype_code(self.act_dtype)
        cfg.grad_in_dtype = _torch_dtype_code(self.grad_in_dtype)
        cfg.grad_out_dtype = _torch_dtype_code(self.grad_out_dtype)
        arr = (_lib.Layout * len(self.modules))(*[m._c() for m in self.modules])
        ne = max(1, len(self.edges))
        src = (ctypes.c_int * ne)(*[e[0] for e in self.edges])
        dst = (ctypes.c_int * ne)(*[e[1] for e in self.edges])
        h = ctypes.c_void_p()
        check(L.hb_runtime_create(arr, len(self.modules), src, dst, len(self.edges), global_batch, feature_width,
                                  self.world, self.rank, obj[0], ctypes.byref(cfg), ctypes.byref(h)))
        self._h = h
        self.device = torch.device("cuda", torch.cuda.current_device())
        n, m, nn, rows = (ctypes.c_int() for _ in range(4))
        check(L.hb_runtime_info(h, *(ctypes.byref(x) for x in (n, m, nn, rows))))
        self.node, self.module, self.n_nodes, self.rows = n.value, m.value, nn.value, rows.value
        self._edge_rts = {}
        self._cb = None

    # -- groups / buffers / streams
    def group(self, kind: int) -> list[int]:
        out, n = (ctypes.c_int * 64)(), ctypes.c_int()
        check(_declare().hb_runtime_group(self._h, kind, out, 64, ctypes.byref(n)))
        return list(out[: n.value])

    def edge_runtime(self, k: int) -> BridgeRuntime:
        """The module edge's exec as a BridgeRuntime view (owned by this runtime)."""
        if k not in self._edge_rts:
            p = ctypes.c_void_p()
            check(_declare().hb_runtime_edge_exec(self._h, k, ctypes.byref(p)))
            s, d = self.edges[k]
            rt = BridgeRuntime.__new__(BridgeRuntime)
            rt.plan = plan_bridge(BoundaryEdge(self.modules[s], self.modules[d], self.global_batch,
                                               self.feature_width))
            rt.splice, rt.n_gpus, rt.my_gpu = None, self.world, self.rank
            rt.rank_to_gpu = list(range(self.world))
            rt.act_dtype, rt.grad_in_dtype, rt.grad_out_dtype = self.act_dtype, self.grad_in_dtype, self.grad_out_dtype
            rt.mb_slots, rt.text_embedding, rt.device = self.nmb, False, self.device
            rt._h, rt._keep, rt._bind_dirty, rt._local_group = p, {}, False, None
            self._edge_rts[k] = rt
        return self._edge_rts[k]

    def stage_buffer(self, which: int, mb: int):
        import torch

        p, n = ctypes.c_void_p(), ctypes.c_size_t()
        check(_declare().hb_runtime_stage_buffer(self._h, which, mb, ctypes.byref(p), ctypes.byref(n)))
        if not p.value or not n.value:
            return None
        from .bridge import _CAI

        return torch.as_tensor(_CAI(p.value, n.value), device=self.device)

    def stream(self, which: int):
        import torch

        p = ctypes.c_void_p()
        check(_declare().hb_runtime_stream(self._h, which, ctypes.byref(p)))
        return torch.cuda.ExternalStream(p.value, device=self.device)

    # -- execution
    def step(self, compute=None):
        """Enqueue one step; ``compute(node, mb, bwd, stream_ptr)`` runs at each
        compute cell (None: event-only compute)."""
        if compute is None:
            cb = ctypes.cast(None, COMPUTE_FN)
        else:
            cb = COMPUTE_FN(lambda user, node, mb, bwd, st: compute(node, mb, bwd, st))
        self._cb = cb  # keep alive while the step's host calls run
        check(_declare().hb_runtime_step(self._h, cb, None))

    def last_step_ms(self) -> float:
        ms = ctypes.c_float()
        check(_declare().hb_runtime_last_step_ms(self._h, ctypes.byref(ms)))
        return ms.value

    def paired_ops(self) -> int:
        """Boundary forward/backward pairs issued as one fused call so far."""
        n = ctypes.c_longlong()
        check(_declare().hb_runtime_paired_ops(self._h, ctypes.byref(n)))
        return n.value

    def close(self):
        h = getattr(self, "_h", None)
        if h and _lib._lib is not None:
            for rt in self._edge_rts.values():
                rt._h = None
            _declare().hb_runtime_destroy(h)
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
