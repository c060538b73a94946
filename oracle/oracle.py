"""ORACLE — test infrastructure only.

ctypes/numpy wrapper over ``oracle/_ref/libhb_oracle.so`` (the C++ restatement
of the reference's bridge/splice over the reference's own ``simnet``/``grid``,
see ``oracle/src/bridge_oracle.cpp``). Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline legs may import
this module; the product package never does.

Parity status: pinned by the SPEC.md prose known-answer tests made executable
in ``tests/test_oracle_kats.py`` and by the reference's grid tests; the bridge
itself has no executable reference test.
"""
from __future__ import annotations

import ctypes
import os
import re
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_ref", "libhb_oracle.so")
REF_CORE = "/root/reference/proj/core"

_lib = None


def build(force: bool = False) -> str:
    """Compile the oracle (needs /root/reference); returns the .so path."""
    if os.path.isdir(REF_CORE):
        subprocess.run(["make", "-s", "-C", HERE] + (["-B"] if force else []), check=True)
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"oracle library missing at {LIB_PATH} and /root/reference is absent")
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        _lib = ctypes.CDLL(LIB_PATH)
        _declare(_lib)
    return _lib


def _declare(L):
    I, Lg, D, Ch = ctypes.c_int, ctypes.c_long, ctypes.c_double, ctypes.c_char_p
    IP, LP, DP = ctypes.POINTER(I), ctypes.POINTER(Lg), ctypes.POINTER(D)
    DPP = ctypes.POINTER(DP)
    sig = {
        "oracle_last_error": (Ch, []),
        "oracle_plan_export": (I, [IP, Ch, IP, Ch, I, I, Ch, Lg, LP]),
        "oracle_classify": (I, [IP, IP, IP, IP]),
        "oracle_cross_boundary_messages": (I, [IP, IP, I, I, IP]),
        "oracle_bridge_forward": (I, [IP, Ch, IP, Ch, I, I, I, I, DPP, DPP, Ch, Lg, LP, DP]),
        "oracle_bridge_backward": (I, [IP, Ch, IP, Ch, I, I, I, I, DPP, DPP, Ch, Lg, LP, DP]),
        "oracle_splice_forward": (I, [IP, I, I, I, I, I, DP, Lg, DP, Lg, Lg, DP]),
        "oracle_splice_backward": (I, [IP, I, I, I, I, I, DP, Lg, DP]),
        "oracle_cp_token_slice": (I, [I, I, I, IP, IP]),
        "oracle_assemble_tokens": (I, [I, I, I, I, DP, DP, I, I, DP]),
        "oracle_split_vision_grad": (I, [I, I, I, I, DP, I, I, DP]),
        "oracle_interval_oracle": (I, [I, I, I, IP, I, IP]),
        "oracle_coord_of_rank": (I, [IP, I, IP]),
        "oracle_placement_of_edge": (I, [IP, IP, IP]),
        "oracle_gaussian_fill": (I, [ctypes.c_ulonglong, Ch, DP, Lg, D]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"oracle status {code}: {msg}")
        self.code = code
        self.msg = msg


def _check(rc: int):
    if rc != 0:
        raise OracleError(rc, lib().oracle_last_error().decode())


@dataclass(frozen=True)
class Layout:
    """Mirror of hetsim::grid::ModuleLayout (grid.hpp:16-31)."""

    name: str
    tp: int = 1
    cp: int = 1
    pp: int = 1
    dp: int = 1
    rank_offset: int = 0

    @property
    def world_size(self):
        return self.tp * self.cp * self.pp * self.dp

    @property
    def rank_end(self):
        return self.rank_offset + self.world_size

    def arr(self):
        return (ctypes.c_int * 5)(self.tp, self.cp, self.pp, self.dp, self.rank_offset)

    # grid.cpp:21-53 restated for test-side bookkeeping
    def coord(self, r):
        lin = r - self.rank_offset
        t = lin % self.tp
        lin //= self.tp
        c = lin % self.cp
        lin //= self.cp
        d = lin % self.dp
        lin //= self.dp
        return (t, c, lin, d)

    def rank(self, t, c, p, d):
        return self.rank_offset + ((p * self.dp + d) * self.cp + c) * self.tp + t

    def stage_ranks(self, p):
        return sorted(self.rank(t, c, p, d) for d in range(self.dp) for c in range(self.cp)
                      for t in range(self.tp))


def intervals(B, dp):
    n = B // dp
    return [(i * n, n) for i in range(dp)]


def export_plan(src: Layout, dst: Layout, B: int, W: int) -> str:
    buf = ctypes.create_string_buffer(1 << 20)
    n = ctypes.c_long()
    _check(lib().oracle_plan_export(src.arr(), src.name.encode(), dst.arr(), dst.name.encode(),
                                    B, W, buf, len(buf), ctypes.byref(n)))
    return buf.value.decode()


def classify(src: Layout, dst: Layout):
    k, f = ctypes.c_int(), ctypes.c_int()
    _check(lib().oracle_classify(src.arr(), dst.arr(), ctypes.byref(k), ctypes.byref(f)))
    return ["Equal", "FanIn", "FanOut"][k.value], f.value


def cross_boundary_messages(src, dst, B, W=1):
    n = ctypes.c_int()
    _check(lib().oracle_cross_boundary_messages(src.arr(), dst.arr(), B, W, ctypes.byref(n)))
    return n.value


def _ptrs(world, arrays):
    P = ctypes.POINTER(ctypes.c_double)
    out = (P * world)()
    for r in range(world):
        a = arrays.get(r)
        out[r] = a.ctypes.data_as(P) if a is not None else P()
    return out


def parse_ledger(text: str):
    led = {}
    for line in text.strip().splitlines():
        label, direction, msgs, nbytes = line.rsplit(" ", 3)
        led[(label, direction)] = (int(msgs), int(nbytes))
    return led


def bridge_forward(src: Layout, dst: Layout, B: int, W: int, shards: dict, mb: int = 0):
    """shards: {global rank: (rows x W) float64 array}. Returns ({rank: out}, ledger, seconds)."""
    world = max(src.rank_end, dst.rank_end)
    shards = {r: np.ascontiguousarray(a, dtype=np.float64) for r, a in shards.items()}
    DI = intervals(B, dst.dp)
    outs = {r: np.empty((DI[dst.coord(r)[3]][1], W)) for r in dst.stage_ranks(0)}
    buf = ctypes.create_string_buffer(1 << 16)
    n = ctypes.c_long()
    sec = ctypes.c_double()
    _check(lib().oracle_bridge_forward(src.arr(), src.name.encode(), dst.arr(), dst.name.encode(),
                                       B, W, mb, world, _ptrs(world, shards), _ptrs(world, outs),
                                       buf, len(buf), ctypes.byref(n), ctypes.byref(sec)))
    return outs, parse_ledger(buf.value.decode()), sec.value


def bridge_backward(src: Layout, dst: Layout, B: int, W: int, grads: dict, mb: int = 0):
    """grads: {global dest rank: (rows x W) float64}. Returns ({src rank: grad}, ledger, seconds)."""
    world = max(src.rank_end, dst.rank_end)
    grads = {r: np.ascontiguousarray(a, dtype=np.float64) for r, a in grads.items()}
    SI = intervals(B, src.dp)
    outs = {r: np.empty((SI[src.coord(r)[3]][1], W)) for r in src.stage_ranks(src.pp - 1)}
    buf = ctypes.create_string_buffer(1 << 16)
    n = ctypes.c_long()
    sec = ctypes.c_double()
    _check(lib().oracle_bridge_backward(src.arr(), src.name.encode(), dst.arr(), dst.name.encode(),
                                        B, W, mb, world, _ptrs(world, grads), _ptrs(world, outs),
                                        buf, len(buf), ctypes.byref(n), ctypes.byref(sec)))
    return outs, parse_ledger(buf.value.decode()), sec.value


def _dp(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _ip(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_int))


def splice_forward(codes, Q, S, d_h, slice_start, slice_len, vision, text, text_offset=0):
    codes = np.ascontiguousarray(codes, dtype=np.int32)
    vision = np.ascontiguousarray(vision, dtype=np.float64).reshape(-1, d_h)
    text = np.ascontiguousarray(text, dtype=np.float64).reshape(-1, d_h)
    out = np.empty((Q * slice_len, d_h))
    _check(lib().oracle_splice_forward(_ip(codes), Q, S, d_h, slice_start, slice_len, _dp(vision),
                                       ctypes.c_long(vision.shape[0]), _dp(text),
                                       ctypes.c_long(text.shape[0]), ctypes.c_long(text_offset),
                                       _dp(out)))
    return out


def splice_backward(codes, Q, S, d_h, slice_start, slice_len, token_grad, vision_rows):
    codes = np.ascontiguousarray(codes, dtype=np.int32)
    token_grad = np.ascontiguousarray(token_grad, dtype=np.float64)
    out = np.empty((vision_rows, d_h))
    _check(lib().oracle_splice_backward(_ip(codes), Q, S, d_h, slice_start, slice_len,
                                        _dp(token_grad), ctypes.c_long(vision_rows), _dp(out)))
    return out


def cp_token_slice(S, cp, c):
    a, b = ctypes.c_int(), ctypes.c_int()
    _check(lib().oracle_cp_token_slice(S, cp, c, ctypes.byref(a), ctypes.byref(b)))
    return a.value, b.value


def assemble_tokens(S, S_v, d_h, vision, text, slice_start, slice_len):
    vision = np.ascontiguousarray(vision, dtype=np.float64)
    text = np.ascontiguousarray(text, dtype=np.float64)
    n = vision.shape[0]
    out = np.empty((n * slice_len, d_h))
    _check(lib().oracle_assemble_tokens(S, S_v, d_h, n, _dp(vision), _dp(text), slice_start,
                                        slice_len, _dp(out)))
    return out


def split_vision_grad(S, S_v, d_h, n, token_grad, slice_start, slice_len):
    token_grad = np.ascontiguousarray(token_grad, dtype=np.float64)
    out = np.empty((n, S_v * d_h))
    _check(lib().oracle_split_vision_grad(S, S_v, d_h, n, _dp(token_grad), slice_start, slice_len,
                                          _dp(out)))
    return out


def interval_oracle(B, dp_src, dp_dst):
    cap = 4 * (B + 1)
    buf = (ctypes.c_int * cap)()
    n = ctypes.c_int()
    _check(lib().oracle_interval_oracle(B, dp_src, dp_dst, buf, cap, ctypes.byref(n)))
    out = [[] for _ in range(dp_dst)]
    for i in range(n.value):
        d, s, st, ln = buf[4 * i:4 * i + 4]
        out[d].append((s, (st, ln)))
    return out


def coord_of_rank(layout: Layout, rank: int):
    c = (ctypes.c_int * 4)()
    _check(lib().oracle_coord_of_rank(layout.arr(), rank, c))
    return tuple(c)


def placement_of_edge(src: Layout, dst: Layout) -> str:
    p = ctypes.c_int()
    _check(lib().oracle_placement_of_edge(src.arr(), dst.arr(), ctypes.byref(p)))
    return ["Colocated", "NonColocated"][p.value]


def gaussian(seed: int, tag: str, n: int, scale: float = 1.0) -> np.ndarray:
    out = np.empty(n)
    _check(lib().oracle_gaussian_fill(ctypes.c_ulonglong(seed), tag.encode(), _dp(out),
                                      ctypes.c_long(n), ctypes.c_double(scale)))
    return out


ERROR_NAMES = [
    "RankOutOfModule", "CoordOutOfBounds", "IndivisibleBatch", "PartialOverlap", "NonIntegerFan",
    "PlanInfeasible", "ShardIntervalMismatch", "MissingSourceShard", "GradIntervalMismatch",
    "UnknownMicrobatch", "Deadlock", "GroupMismatch", "ShapeMismatch", "ChannelMismatch",
    "SnapshotWhileActive", "DivisibilityViolation", "CyclicGraph", "DanglingEdge",
    "InfeasibleSchedule", "NotColocated", "StructureMismatch", "ParseError", "ValidationError",
    "InvalidArgument",
]


def error_name(status: int) -> str:
    return ERROR_NAMES[status - 1] if 1 <= status <= len(ERROR_NAMES) else f"status{status}"


def export_lines(text: str):
    return [ln for ln in text.strip().splitlines()]


_IV = re.compile(r"\[(\d+),(\d+)\)")
