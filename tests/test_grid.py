"""Layout algebra: the reference's own known-answer tests
(/root/reference/proj/tests/test_grid.cpp:29-219) restated against the product
grid, plus an exhaustive cross-check against the reference grid library that
the oracle compiles from /root/reference sources."""
import itertools

import pytest

from helpers import O
from paper_2605_27678_b200 import HetBridgeError
from paper_2605_27678_b200 import grid as G
from paper_2605_27678_b200.grid import BatchInterval, GridCoord, ModuleLayout


def enumerate_coords(l):  # test_grid.cpp:18-25
    return [GridCoord(t, c, p, d) for p in range(l.pp) for d in range(l.dp) for c in range(l.cp)
            for t in range(l.tp)]


def code_of(fn, *a):
    with pytest.raises(HetBridgeError) as ei:
        fn(*a)
    return ei.value.code


def test_coord_singleton():
    assert G.coord_of_rank(ModuleLayout("m", 1, 1, 1, 1, 0), 0) == GridCoord(0, 0, 0, 0)


def test_coord_matches_enumeration():
    l = ModuleLayout("m", 2, 1, 2, 2, 0)
    coords = enumerate_coords(l)
    assert len(coords) == 8
    for r in range(8):
        assert G.coord_of_rank(l, r) == coords[r]


def test_coord_rejects_outside_module():
    l = ModuleLayout("enc", 4, 1, 1, 2, 8)
    with pytest.raises(HetBridgeError) as ei:
        G.coord_of_rank(l, 7)
    assert ei.value.code == "RankOutOfModule" and "outside module" in str(ei.value)
    G.coord_of_rank(l, 8)
    G.coord_of_rank(l, 15)
    assert code_of(G.coord_of_rank, l, 16) == "RankOutOfModule"


def test_rank_bijection():
    l = ModuleLayout("m", 2, 1, 1, 4, 0)
    seen = {G.rank_of_coord(l, c) for c in enumerate_coords(l)}
    assert seen == set(range(8))


def test_rank_singleton_offset():
    assert G.rank_of_coord(ModuleLayout("m", 1, 1, 1, 1, 13), GridCoord()) == 13


def test_rank_rejects_oob():
    assert code_of(G.rank_of_coord, ModuleLayout("m", 2, 1, 1, 1, 0), GridCoord(2, 0, 0, 0)) == "CoordOutOfBounds"


LAYOUTS = [ModuleLayout("a", 1, 1, 1, 1, 0), ModuleLayout("b", 2, 2, 2, 2, 0), ModuleLayout("c", 4, 1, 2, 8, 0),
           ModuleLayout("d", 2, 4, 1, 4, 16), ModuleLayout("e", 8, 1, 1, 8, 3), ModuleLayout("f", 1, 2, 4, 2, 5),
           ModuleLayout("g", 4, 2, 2, 4, 0), ModuleLayout("h", 1, 1, 8, 8, 0)]


@pytest.mark.parametrize("l", LAYOUTS, ids=lambda l: l.name)
def test_mutual_inverse_up_to_world_64(l):
    assert l.world_size() <= 64
    for r in range(l.rank_begin(), l.rank_end()):
        assert G.rank_of_coord(l, G.coord_of_rank(l, r)) == r
    for c in enumerate_coords(l):
        assert G.coord_of_rank(l, G.rank_of_coord(l, c)) == c


def test_partition_batch_kats():
    assert G.partition_batch(8, 1) == [BatchInterval(0, 8)]
    assert G.partition_batch(8, 4) == [BatchInterval(0, 2), BatchInterval(2, 2), BatchInterval(4, 2),
                                       BatchInterval(6, 2)]


def test_partition_batch_floor_rule():
    for B in (8, 12, 24, 64):
        for dp in (1, 2, 4, 8):
            if B % dp:
                continue
            parts = G.partition_batch(B, dp)
            for j in range(B):
                s = j * dp // B
                assert parts[s].start <= j < parts[s].end()
            assert sum(p.length for p in parts) == B
            assert all(parts[i].start == parts[i - 1].end() for i in range(1, len(parts)))


def test_partition_batch_indivisible():
    assert code_of(G.partition_batch, 10, 4) == "IndivisibleBatch"


def test_leader_canonical_unique():
    l = ModuleLayout("m", 2, 2, 1, 2, 0)
    coords = enumerate_coords(l)
    leaders = set()
    for d in range(l.dp):
        lead = G.leader_rank(l, 0, d)
        c = G.coord_of_rank(l, lead)
        assert (c.tp_idx, c.cp_idx, c.dp_idx) == (0, 0, d)
        first = next(i for i, x in enumerate(coords) if x == GridCoord(0, 0, 0, d))
        assert lead == first
        leaders.add(lead)
    assert len(leaders) == l.dp


def test_leader_every_cell_when_tp_cp_one():
    l = ModuleLayout("m", 1, 1, 2, 3, 0)
    for p in range(2):
        for d in range(3):
            assert G.leader_rank(l, p, d) == G.rank_of_coord(l, GridCoord(0, 0, p, d))


def test_leader_offset_translation():
    base = ModuleLayout("m", 2, 2, 1, 2, 0)
    moved = ModuleLayout("m", 2, 2, 1, 2, 8)
    for d in range(2):
        assert G.leader_rank(moved, 0, d) == G.leader_rank(base, 0, d) + 8


def test_placement_classification():
    llm = ModuleLayout("language", 2, 1, 2, 2, 0)
    enc = ModuleLayout("images", 1, 1, 1, 8, 0)
    assert G.placement_of_edge(G.BoundaryEdge(enc, llm, 8, 3)) == G.Placement.Colocated
    llm4 = ModuleLayout("language", 2, 1, 2, 1, 0)
    enc4 = ModuleLayout("images", 1, 1, 1, 4, 4)
    assert G.placement_of_edge(G.BoundaryEdge(enc4, llm4, 8, 3)) == G.Placement.NonColocated
    a, b = ModuleLayout("a", 1, 1, 1, 6, 0), ModuleLayout("b", 1, 1, 1, 4, 4)
    assert code_of(G.placement_of_edge, G.BoundaryEdge(a, b, 8, 3)) == "PartialOverlap"


def test_placement_symmetric():
    a, b, c = ModuleLayout("a", 2, 1, 1, 2, 0), ModuleLayout("b", 1, 1, 1, 4, 4), ModuleLayout("c", 4, 1, 1, 1, 0)
    assert G.placement_of_edge(G.BoundaryEdge(a, b, 8, 1)) == G.placement_of_edge(G.BoundaryEdge(b, a, 8, 1))
    assert G.placement_of_edge(G.BoundaryEdge(a, c, 8, 1)) == G.placement_of_edge(G.BoundaryEdge(c, a, 8, 1))


def test_stage_and_replica_groups():
    l = ModuleLayout("m", 2, 2, 2, 2, 4)
    stage0 = G.ranks_of_stage(l, 0)
    assert len(stage0) == 8 and stage0 == sorted(stage0)
    assert all(G.coord_of_rank(l, r).pp_idx == 0 for r in stage0)
    grp = G.replica_group(l, 1, 1)
    assert len(grp) == 4 and grp[0] == G.leader_rank(l, 1, 1)
    assert all(G.coord_of_rank(l, r).pp_idx == 1 and G.coord_of_rank(l, r).dp_idx == 1 for r in grp)


def test_invalid_layout():
    assert code_of(G.coord_of_rank, ModuleLayout("z", 0, 1, 1, 1, 0), 0) == "InvalidArgument"
    assert code_of(G.coord_of_rank, ModuleLayout("z", 1, 1, 1, 1, -1), 0) == "InvalidArgument"


def test_cross_check_reference_grid_library():
    """Product grid == the reference's grid.cpp (compiled into the oracle) on every rank
    of every layout with tp,cp,pp,dp in {1,2,4} and a few offsets."""
    for tp, cp, pp, dp in itertools.product((1, 2, 4), repeat=4):
        for off in (0, 3):
            l = ModuleLayout("m", tp, cp, pp, dp, off)
            ol = O.Layout("m", tp, cp, pp, dp, off)
            for r in range(l.rank_begin(), l.rank_end()):
                c = G.coord_of_rank(l, r)
                assert (c.tp_idx, c.cp_idx, c.pp_idx, c.dp_idx) == O.coord_of_rank(ol, r)


def test_cross_check_reference_placement():
    for a_off, a_n, b_off, b_n in itertools.product((0, 2, 4), (2, 4), (0, 2, 4, 6), (2, 4)):
        a, b = ModuleLayout("a", dp=a_n, rank_offset=a_off), ModuleLayout("b", dp=b_n, rank_offset=b_off)
        oa, ob = O.Layout("a", dp=a_n, rank_offset=a_off), O.Layout("b", dp=b_n, rank_offset=b_off)
        try:
            ref = O.placement_of_edge(oa, ob)
        except O.OracleError as e:
            ref = O.error_name(e.code)
        try:
            got = G.placement_of_edge(G.BoundaryEdge(a, b, 8, 1)).name
        except HetBridgeError as e:
            got = e.code
        assert got == ref


def test_module_groups_partition_the_module():
    l = ModuleLayout("llm", 2, 2, 3, 2, 5)
    for kind, size in (("tp", 2), ("cp", 2), ("pp", 3), ("dp", 2)):
        groups = G.module_groups(l)[kind]
        flat = sorted(r for g in groups for r in g)
        assert flat == list(range(l.rank_begin(), l.rank_end()))
        assert all(len(g) == size for g in groups)
        for g in groups:  # members differ from each other only in that axis
            cs = [G.coord_of_rank(l, r) for r in g]
            for attr in ("tp_idx", "cp_idx", "pp_idx", "dp_idx"):
                if not attr.startswith(kind):
                    assert len({getattr(c, attr) for c in cs}) == 1
    # the replica group of a (pp, dp) cell is the union of tp x cp around its leader
    assert sorted(set(G.module_group(l, 5, "tp")) | set(G.module_group(l, 5, "cp")) |
                  set(G.module_group(l, 8, "tp"))) == G.replica_group(l, 0, 0)
    # C5: LLM stage-to-stage partners of rank 2 are its PP group
    assert G.module_group(ModuleLayout("llm", tp=2, pp=3, rank_offset=2), 2, "pp") == [2, 4, 6]
