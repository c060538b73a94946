"""Graph-aware dispatch (SPEC.md:358-437 `sched`; acceptance criterion 6,
SPEC.md:554; Appendix D figure). CPU tests of the C++ hb::sched
through the C-ABI."""
import dataclasses

import pytest

from paper_2605_27678_b200 import sched as S
from paper_2605_27678_b200._lib import HetBridgeError
from paper_2605_27678_b200.grid import ModuleLayout


def fig4a():
    mods, edges = S.fig4a_modules()
    return S.build_stage_graph(mods, edges)


def test_single_module_chain():
    g = S.build_stage_graph([ModuleLayout("LLM", pp=3)], [])
    assert [n.name for n in g.nodes] == ["LLMP0", "LLMP1", "LLMP2"]
    assert [(e.src, e.dst, e.kind) for e in g.edges] == [(0, 1, S.EdgeKind.P2P), (1, 2, S.EdgeKind.P2P)]
    assert g.distances() == {"LLMP0": 2, "LLMP1": 1, "LLMP2": 0}


def test_fig4a_stage_graph():
    """6 nodes; E1P1->LLM0 and E2P0->LLM0 are NC edges; distances
    LLM2=0, LLM1=1, LLM0=2, E1P1=3, E1P0=4, E2P0=3."""
    g = fig4a()
    assert len(g.nodes) == 6
    nc = {(g.nodes[e.src].name, g.nodes[e.dst].name) for e in g.edges if e.kind == S.EdgeKind.NC}
    assert nc == {("E1P1", "LLMP0"), ("E2P0", "LLMP0")}
    p2p = {(g.nodes[e.src].name, g.nodes[e.dst].name) for e in g.edges if e.kind == S.EdgeKind.P2P}
    assert p2p == {("E1P0", "E1P1"), ("LLMP0", "LLMP1"), ("LLMP1", "LLMP2")}
    assert g.distances() == {"LLMP2": 0, "LLMP1": 1, "LLMP0": 2, "E1P1": 3, "E1P0": 4, "E2P0": 3}


def test_graph_errors():
    a, b = ModuleLayout("A", rank_offset=0), ModuleLayout("B", rank_offset=1)
    with pytest.raises(HetBridgeError) as ei:
        S.build_stage_graph([a, b], [(0, 1), (1, 0)])
    assert ei.value.code == "CyclicGraph"
    with pytest.raises(HetBridgeError) as ei:
        S.build_stage_graph([a, b], [(0, 2)])
    assert ei.value.code == "DanglingEdge"
    with pytest.raises(HetBridgeError) as ei:
        S.build_stage_graph([a, b], [])  # two sinks
    assert ei.value.code == "InfeasibleSchedule"
    with pytest.raises(HetBridgeError) as ei:
        S.generate_1f1b_dispatch(S.build_stage_graph([a], []), 0)
    assert ei.value.code == "InfeasibleSchedule"


def test_single_stage_alternates_compute_no_comm():
    g = S.build_stage_graph([ModuleLayout("LLM")], [])
    t = S.generate_1f1b_dispatch(g, 2)
    assert all(c.op == S.Op.Compute for c in t.cells)
    assert [(c.mb, c.bwd) for c in t.cells] == [(0, False), (0, True), (1, False), (1, True)]
    assert S.validate_dispatch(g, t) == []


@pytest.mark.parametrize("nmb", [1, 2, 4, 8])
def test_fig4a_dispatch_structure(nmb):
    """Acceptance 6: the generated table validates with zero
    violations; E1P0->E1P1 cells are p2p, E1P1->LLM0 and E2P0->LLM0 are NC;
    LLM0's Compute(mb) follows both NC RecvFwd(mb); each boundary gradient goes
    back over its forward edge; every (edge, mb) moves once each way."""
    g = fig4a()
    t = S.generate_1f1b_dispatch(g, nmb)
    assert S.validate_dispatch(g, t) == []
    name = {i: n.name for i, n in enumerate(g.nodes)}
    for c in t.cells:
        if c.op == S.Op.Compute:
            continue
        e = g.edges[c.edge]
        pair = (name[e.src], name[e.dst])
        assert c.kind == (S.EdgeKind.NC if pair[1] == "LLMP0" and pair[0] != "LLMP0" else S.EdgeKind.P2P)
        if pair == ("E1P0", "E1P1"):
            assert c.kind == S.EdgeKind.P2P
    llm0 = g.node("LLMP0")
    for mb in range(nmb):
        comp = [c.row for c in t.cells if c.node == llm0 and c.op == S.Op.Compute and c.mb == mb and not c.bwd]
        recvs = [c for c in t.cells if c.node == llm0 and c.op == S.Op.RecvFwd and c.mb == mb]
        assert len(recvs) == 2 and all(r.kind == S.EdgeKind.NC for r in recvs)
        assert all(r.row < comp[0] for r in recvs)
        # gradients leave LLM0 over the same two NC edges the activations came in on
        sends = [c for c in t.cells if c.node == llm0 and c.op == S.Op.SendBwd and c.mb == mb]
        assert sorted(c.edge for c in sends) == sorted(c.edge for c in recvs)
    for e in range(len(g.edges)):
        for mb in range(nmb):
            for op in (S.Op.SendFwd, S.Op.RecvFwd, S.Op.SendBwd, S.Op.RecvBwd):
                assert sum(1 for c in t.cells if c.edge == e and c.mb == mb and c.op == op) == 1


def test_fig4a_warmup_first_sends():
    """S:406 (Appendix D): E1P0's first send is p2p to E1P1; E1P1's next forward
    send is NC; E2P0's first forward send is already NC."""
    g = fig4a()
    t = S.generate_1f1b_dispatch(g, 4)

    def first_send(node):
        return next(c for c in t.cells if c.node == g.node(node) and c.op == S.Op.SendFwd)

    assert first_send("E1P0").kind == S.EdgeKind.P2P and g.nodes[g.edges[first_send("E1P0").edge].dst].name == "E1P1"
    assert first_send("E1P1").kind == S.EdgeKind.NC
    assert first_send("E2P0").kind == S.EdgeKind.NC


def test_linear_chain_reduces_to_1f1b():
    """Longest-path warmup on a chain is standard 1F1B: stage s warms up with
    PP-1-s forwards (S:430 design decision)."""
    g = S.build_stage_graph([ModuleLayout("LLM", pp=4)], [])
    t = S.generate_1f1b_dispatch(g, 8)
    assert S.validate_dispatch(g, t) == []
    for s in range(4):
        comp = [c for c in t.of_node(s) if c.op == S.Op.Compute]
        first_b = next(i for i, c in enumerate(comp) if c.bwd)
        assert first_b == 3 - s + 1  # warmup forwards, then the first steady-state forward
        # steady state alternates F/B
        seq = [c.bwd for c in comp[first_b - 1: len(comp) - (3 - s)]]
        assert seq == [False, True] * (len(seq) // 2)


def test_validate_flags_join_readiness():
    """A table with LLM0's Compute before one encoder RecvFwd names the edge and mb."""
    g = fig4a()
    t = S.generate_1f1b_dispatch(g, 4)
    llm0 = g.node("LLMP0")
    cells = list(t.cells)
    i = next(k for k, c in enumerate(cells) if c.node == llm0 and c.op == S.Op.RecvFwd and c.mb == 2
             and g.nodes[g.edges[c.edge].src].name == "E2P0")
    comp_row = next(c.row for c in cells if c.node == llm0 and c.op == S.Op.Compute and c.mb == 2 and not c.bwd)
    # delay the receive (and its paired send) past the compute
    send = next(k for k, c in enumerate(cells) if c.edge == cells[i].edge and c.op == S.Op.SendFwd and c.mb == 2)
    cells[i] = dataclasses.replace(cells[i], row=comp_row + 1)
    cells[send] = dataclasses.replace(cells[send], row=comp_row + 1)
    v = S.validate_dispatch(g, cells, 4)
    assert any("join readiness" in x and "LLMP0 mb 2" in x and "E2P0->LLMP0" in x for x in v), v


def test_validate_flags_wrong_gradient_edge():
    """Routing a boundary gradient over the other encoder's edge is an
    edge-identity violation."""
    g = fig4a()
    t = S.generate_1f1b_dispatch(g, 4)
    llm0 = g.node("LLMP0")
    e1 = next(i for i, e in enumerate(g.edges) if g.nodes[e.src].name == "E1P1")
    e2 = next(i for i, e in enumerate(g.edges) if g.nodes[e.src].name == "E2P0")
    cells = list(t.cells)
    k = next(k for k, c in enumerate(cells) if c.node == llm0 and c.op == S.Op.SendBwd and c.mb == 1 and c.edge == e1)
    cells[k] = dataclasses.replace(cells[k], edge=e2)
    v = S.validate_dispatch(g, cells, 4)
    assert any("edge identity" in x and "E1P1->LLMP0" in x for x in v), v


def test_validate_flags_double_consumption():
    g = fig4a()
    t = S.generate_1f1b_dispatch(g, 2)
    cells = list(t.cells) + [t.cells[1]]
    assert any("double consumption" in x or "appears" in x for x in S.validate_dispatch(g, cells, 2))


def test_render_grid():
    g = fig4a()
    txt = S.render(g, 4)
    head = txt.splitlines()[0]
    for n in ("E1P0", "E1P1", "E2P0", "LLMP0", "LLMP1", "LLMP2"):
        assert n in head
    assert "sf0:p2p" in txt and "sf0:NC" in txt and "rf0:NC" in txt and "sb0:NC" in txt


def test_host_runtime_rejects_colocated_modules_before_nccl():
    """The host runtime drives non-colocated modules; shared ranks fail at
    validation, before any communicator or CUDA call."""
    import ctypes

    from paper_2605_27678_b200 import _lib
    from paper_2605_27678_b200 import runtime as R

    L = R._declare()
    mods = (_lib.Layout * 2)(_lib.Layout(b"vit", 1, 1, 1, 2, 0), _lib.Layout(b"llm", 2, 1, 1, 1, 0))
    src, dst = (ctypes.c_int * 1)(0), (ctypes.c_int * 1)(1)
    out = ctypes.c_void_p()
    st = L.hb_runtime_create(mods, 2, src, dst, 1, 4, 8, 2, 0, b"\0" * 128, None, ctypes.byref(out))
    assert st == 24 and "share ranks" in _lib.last_error() and not out.value
    cfg = R.RuntimeConfig()
    L.hb_runtime_config_default(ctypes.byref(cfg))
    cfg.nmb = 0
    mods2 = (_lib.Layout * 2)(_lib.Layout(b"vit", 1, 1, 1, 1, 0), _lib.Layout(b"llm", 1, 1, 1, 1, 1))
    st = L.hb_runtime_create(mods2, 2, src, dst, 1, 4, 8, 2, 0, b"\0" * 128, ctypes.byref(cfg), ctypes.byref(out))
    assert st == 19  # InfeasibleSchedule


def _rendezvous(graph, seqs):
    """Serial boundary streams, one per node: an NC op (module edge, direction,
    mb) runs when it is at the head of BOTH endpoints' streams (the in-kernel
    "started" barrier). Returns the ops left when no stream can advance."""
    ep = {}
    for e in graph.edges:
        if e.kind == S.EdgeKind.NC:
            ep[e.boundary] = (e.src, e.dst)

    def key(c):
        return (graph.edges[c.edge].boundary, c.op in (S.Op.SendBwd, S.Op.RecvBwd), c.mb)

    q = {n: [key(c) for c in v] for n, v in seqs.items()}
    moved = True
    while moved:
        moved = False
        for n, v in q.items():
            if not v:
                continue
            a, b = ep[v[0][0]]
            other = b if n == a else a
            if q[other] and q[other][0] == v[0]:
                q[n].pop(0)
                q[other].pop(0)
                moved = True
    return {n: v for n, v in q.items() if v}


def _topologies():
    mods, edges = S.fig4a_modules()
    yield "fig4a", mods, edges
    yield "join4", [ModuleLayout("E1", pp=2, rank_offset=0), ModuleLayout("E2", rank_offset=2),
                    ModuleLayout("LLM", rank_offset=3)], [(0, 2), (1, 2)]
    yield "c5", [ModuleLayout("vit", dp=2), ModuleLayout("llm", tp=2, pp=3, rank_offset=2)], [(0, 1)]
    yield "three-encoders", [ModuleLayout("A", pp=3), ModuleLayout("B", pp=2, rank_offset=3),
                             ModuleLayout("C", rank_offset=5), ModuleLayout("LLM", pp=2, rank_offset=6)], \
        [(0, 3), (1, 3), (2, 3)]


@pytest.mark.parametrize("nmb", [1, 2, 4, 8])
def test_nc_issue_order_meets_every_rendezvous(nmb):
    """The host runtime's boundary-stream order (hb_dispatch_nc_order) drains on
    every topology: each NC op is issued by its two endpoints in the same
    relative order (row, module edge, forward before backward)."""
    for name, mods, edges in _topologies():
        g = S.build_stage_graph(mods, edges)
        seqs = {n: S.nc_issue_order(g, nmb, n) for n in range(len(g.nodes))}
        assert all(a.row <= b.row for v in seqs.values() for a, b in zip(v, v[1:]))
        assert _rendezvous(g, seqs) == {}, name


def test_table_order_would_deadlock_at_a_join():
    """Regression (round-2 N=4 hang): issuing a row's NC cells in the table's own
    order makes E1P1 run F2 before B1 while LLMP0 runs B1 before F2 at the join."""
    _, mods, edges = next(t for t in _topologies() if t[0] == "join4")
    g = S.build_stage_graph(mods, edges)
    t = S.generate_1f1b_dispatch(g, 4)
    raw = {n: [c for c in t.cells if c.node == n and c.op != S.Op.Compute and c.kind == S.EdgeKind.NC]
           for n in range(len(g.nodes))}
    assert _rendezvous(g, raw) != {}
