"""Layout algebra — Python face of ``hetsim::grid`` (grid.hpp:13-94).

Thin wrappers over the C-ABI (the logic lives in ``csrc/hb/grid.cpp``); names,
fields and error categories match the reference so a test written against
the reference reads the same here.
"""
from __future__ import annotations

import ctypes
import enum
from dataclasses import dataclass

from . import _lib
from ._lib import check, lib


@dataclass(frozen=True)
class ModuleLayout:
    name: str = ""
    tp: int = 1
    cp: int = 1
    pp: int = 1
    dp: int = 1
    rank_offset: int = 0

    def world_size(self) -> int:
        return self.tp * self.cp * self.pp * self.dp

    def rank_begin(self) -> int:
        return self.rank_offset

    def rank_end(self) -> int:
        return self.rank_offset + self.world_size()

    def contains(self, rank: int) -> bool:
        return self.rank_begin() <= rank < self.rank_end()

    def _c(self) -> _lib.Layout:
        return _lib.Layout(self.name.encode(), self.tp, self.cp, self.pp, self.dp, self.rank_offset)


@dataclass(frozen=True)
class GridCoord:
    tp_idx: int = 0
    cp_idx: int = 0
    pp_idx: int = 0
    dp_idx: int = 0


@dataclass(frozen=True)
class BatchInterval:
    start: int = 0
    length: int = 0

    def end(self) -> int:
        return self.start + self.length


@dataclass(frozen=True)
class BoundaryEdge:
    source: ModuleLayout
    dest: ModuleLayout
    global_batch: int = 0
    feature_width: int = 0

    def _c(self) -> _lib.Edge:
        return _lib.Edge(self.source._c(), self.dest._c(), self.global_batch, self.feature_width)


class Placement(enum.IntEnum):
    Colocated = 0
    NonColocated = 1


def coord_of_rank(layout: ModuleLayout, rank: int) -> GridCoord:
    c = (ctypes.c_int * 4)()
    check(lib().hb_coord_of_rank(ctypes.byref(layout._c()), rank, c))
    return GridCoord(*c)


def rank_of_coord(layout: ModuleLayout, coord: GridCoord) -> int:
    c = (ctypes.c_int * 4)(coord.tp_idx, coord.cp_idx, coord.pp_idx, coord.dp_idx)
    r = ctypes.c_int()
    check(lib().hb_rank_of_coord(ctypes.byref(layout._c()), c, ctypes.byref(r)))
    return r.value


def partition_batch(batch: int, dp: int) -> list[BatchInterval]:
    n = max(dp, 0)
    buf = (ctypes.c_int * (2 * max(n, 1)))()
    check(lib().hb_partition_batch(batch, dp, buf, n))
    return [BatchInterval(buf[2 * i], buf[2 * i + 1]) for i in range(n)]


def leader_rank(layout: ModuleLayout, pp_idx: int, dp_idx: int) -> int:
    r = ctypes.c_int()
    check(lib().hb_leader_rank(ctypes.byref(layout._c()), pp_idx, dp_idx, ctypes.byref(r)))
    return r.value


def placement_of_edge(edge: BoundaryEdge) -> Placement:
    p = ctypes.c_int()
    check(lib().hb_placement_of_edge(ctypes.byref(edge._c()), ctypes.byref(p)))
    return Placement(p.value)


def _list(fn, *args) -> list[int]:
    n = ctypes.c_int()
    buf = (ctypes.c_int * 4096)()
    check(fn(*args, buf, len(buf), ctypes.byref(n)))
    return list(buf[: n.value])


def ranks_of_stage(layout: ModuleLayout, pp_idx: int) -> list[int]:
    return _list(lib().hb_ranks_of_stage, ctypes.byref(layout._c()), pp_idx)


def replica_group(layout: ModuleLayout, pp_idx: int, dp_idx: int) -> list[int]:
    return _list(lib().hb_replica_group, ctypes.byref(layout._c()), pp_idx, dp_idx)


GROUP_KINDS = {"tp": 0, "cp": 1, "pp": 2, "dp": 3}


def module_group(layout: ModuleLayout, rank: int, kind: str) -> list[int]:
    """Ranks of `rank`'s TP / CP / PP / DP group inside its module (ascending)."""
    return _list(lib().hb_module_group, ctypes.byref(layout._c()), rank, GROUP_KINDS[kind])


def module_groups(layout: ModuleLayout) -> dict:
    """Every distinct TP/CP/PP/DP group of a module: {kind: [sorted rank lists]}."""
    out = {}
    for kind in GROUP_KINDS:
        seen = []
        for r in range(layout.rank_begin(), layout.rank_end()):
            g = module_group(layout, r, kind)
            if g not in seen:
                seen.append(g)
        out[kind] = seen
    return out


def replica_position(layout: ModuleLayout, c: GridCoord) -> int:
    return c.cp_idx * layout.tp + c.tp_idx


def to_string(iv: BatchInterval) -> str:
    return f"[{iv.start},{iv.end()})"
