"""Graph-aware pipeline dispatch — Python face of the C++ ``hb::sched``
(SPEC.md:358-437 `sched`; PAPER.md:374-395 and the
Appendix D dispatch figure). The reference ships only an empty
``sched.cpp``; names follow the SPEC module: ``build_stage_graph``,
``generate_1f1b_dispatch``, ``validate_dispatch``.

Nodes are (module, pp stage); P2P edges chain a module's stages, NC edges
join a source module's last stage to a destination module's first stage (one
per declared module edge, carrying that edge's BridgePlan identity). The 1F1B
table warms node n up with min(distance-to-sink(n), NMB) forwards; every
send and its receive share one schedule call.
"""
from __future__ import annotations

import ctypes
import enum
from dataclasses import dataclass

from . import _lib
from ._lib import check, lib
from .grid import ModuleLayout


class Op(enum.IntEnum):
    Compute = 0
    SendFwd = 1
    RecvFwd = 2
    SendBwd = 3
    RecvBwd = 4


class EdgeKind(enum.IntEnum):
    P2P = 0
    NC = 1


@dataclass(frozen=True)
class StageNode:
    module: int
    pp: int
    distance: int
    name: str


@dataclass(frozen=True)
class StageEdge:
    src: int
    dst: int
    kind: EdgeKind
    boundary: int  # index of the declared module edge (NC), -1 for P2P


@dataclass(frozen=True)
class Cell:
    row: int
    node: int
    op: Op
    edge: int
    kind: EdgeKind
    mb: int
    bwd: bool = False


class StageGraph:
    """SPEC `StageGraph` (owns an ``hb_stage_graph*``)."""

    def __init__(self, modules, edges):
        self.modules = list(modules)
        self.module_edges = [tuple(e) for e in edges]
        arr = (_lib.Layout * len(self.modules))(*[m._c() for m in self.modules])
        src = (ctypes.c_int * max(1, len(self.module_edges)))(*[e[0] for e in self.module_edges])
        dst = (ctypes.c_int * max(1, len(self.module_edges)))(*[e[1] for e in self.module_edges])
        h = ctypes.c_void_p()
        check(lib().hb_stage_graph_create(arr, len(self.modules), src, dst, len(self.module_edges), ctypes.byref(h)))
        self._h = h
        n = ctypes.c_int()
        check(lib().hb_stage_graph_nodes(h, None, 0, ctypes.byref(n)))
        buf = (ctypes.c_int * (3 * n.value))()
        check(lib().hb_stage_graph_nodes(h, buf, n.value, ctypes.byref(n)))
        self.nodes = [StageNode(buf[3 * i], buf[3 * i + 1], buf[3 * i + 2],
                                f"{self.modules[buf[3 * i]].name}P{buf[3 * i + 1]}") for i in range(n.value)]
        check(lib().hb_stage_graph_edges(h, None, 0, ctypes.byref(n)))
        buf = (ctypes.c_int * (4 * n.value))()
        check(lib().hb_stage_graph_edges(h, buf, n.value, ctypes.byref(n)))
        self.edges = [StageEdge(buf[4 * i], buf[4 * i + 1], EdgeKind(buf[4 * i + 2]), buf[4 * i + 3])
                      for i in range(n.value)]

    def node(self, name: str) -> int:
        return [n.name for n in self.nodes].index(name)

    def distances(self) -> dict:
        return {n.name: n.distance for n in self.nodes}

    def __del__(self):
        try:
            h = getattr(self, "_h", None)
            if h and _lib._lib is not None:
                _lib._lib.hb_stage_graph_destroy(h)
                self._h = None
        except Exception:
            pass


@dataclass
class DispatchTable:
    rows: int
    nmb: int
    cells: list

    def of_node(self, node: int) -> list:
        return [c for c in self.cells if c.node == node]


def build_stage_graph(modules, edges) -> StageGraph:
    """modules: list of ModuleLayout (rank ranges); edges: (source module index,
    dest module index) pairs."""
    return StageGraph(modules, edges)


def _to_c(cells):
    arr = (_lib.Cell * max(1, len(cells)))()
    for i, c in enumerate(cells):
        arr[i] = _lib.Cell(c.row, c.node, int(c.op), c.edge, int(c.kind), c.mb, int(c.bwd))
    return arr


def generate_1f1b_dispatch(graph: StageGraph, nmb: int) -> DispatchTable:
    n, rows = ctypes.c_size_t(), ctypes.c_int()
    check(lib().hb_dispatch_generate(graph._h, nmb, None, 0, ctypes.byref(n), ctypes.byref(rows)))
    arr = (_lib.Cell * max(1, n.value))()
    check(lib().hb_dispatch_generate(graph._h, nmb, arr, n.value, ctypes.byref(n), ctypes.byref(rows)))
    cells = [Cell(c.row, c.node, Op(c.op), c.edge, EdgeKind(c.kind), c.mb, bool(c.bwd)) for c in arr[: n.value]]
    return DispatchTable(rows.value, nmb, cells)


def validate_dispatch(graph: StageGraph, table: DispatchTable | list, nmb: int | None = None) -> list:
    """Violation list (empty = valid); never raises on a bad table."""
    cells = table.cells if isinstance(table, DispatchTable) else list(table)
    nmb = table.nmb if nmb is None else nmb
    arr = _to_c(cells)
    ln, nv = ctypes.c_size_t(), ctypes.c_int()
    check(lib().hb_dispatch_validate(graph._h, arr, len(cells), nmb, None, 0, ctypes.byref(ln), ctypes.byref(nv)))
    buf = ctypes.create_string_buffer(ln.value + 1)
    check(lib().hb_dispatch_validate(graph._h, arr, len(cells), nmb, buf, len(buf), ctypes.byref(ln),
                                     ctypes.byref(nv)))
    return [x for x in buf.value.decode().split("\n") if x]


def nc_issue_order(graph: StageGraph, nmb: int, node: int) -> list:
    """The NC cells of ``node`` in the order the host runtime issues them on its
    boundary stream (row, module edge, forward before backward)."""
    n = ctypes.c_size_t()
    check(lib().hb_dispatch_nc_order(graph._h, nmb, node, None, 0, ctypes.byref(n)))
    arr = (_lib.Cell * max(1, n.value))()
    check(lib().hb_dispatch_nc_order(graph._h, nmb, node, arr, n.value, ctypes.byref(n)))
    return [Cell(c.row, c.node, Op(c.op), c.edge, EdgeKind(c.kind), c.mb, bool(c.bwd)) for c in arr[: n.value]]


def render(graph: StageGraph, nmb: int) -> str:
    ln = ctypes.c_size_t()
    check(lib().hb_dispatch_render(graph._h, nmb, None, 0, ctypes.byref(ln)))
    buf = ctypes.create_string_buffer(ln.value + 1)
    check(lib().hb_dispatch_render(graph._h, nmb, buf, len(buf), ctypes.byref(ln)))
    return buf.value.decode()


def fig4a_modules():
    """PAPER Fig. 4(a) / Appendix D: Encoder 1 with two PP stages, Encoder 2 with
    one, the LLM with three; disjoint rank sets (tp = dp = 1)."""
    return ([ModuleLayout("E1", pp=2, rank_offset=0), ModuleLayout("E2", pp=1, rank_offset=2),
             ModuleLayout("LLM", pp=3, rank_offset=3)], [(0, 2), (1, 2)])
