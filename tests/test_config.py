"""module_parallelisms configuration ingestion (SPEC cli module S:495-545;
paper Appendix B). CPU only: parsing, validation, edges, round trip."""
import pytest

from paper_2605_27678_b200 import bridge as hbb
from paper_2605_27678_b200 import configs
from paper_2605_27678_b200._lib import HetBridgeError
from paper_2605_27678_b200.config import parse_config
from paper_2605_27678_b200.grid import Placement, placement_of_edge

# Appendix B, left panel: disjoint GPU sets
APPENDIX_B_LEFT = """
# Megatron MIMO parallelism, non-colocated
[module.language]
tensor_model_parallel_size = 2
pipeline_model_parallel_size = 2
data_parallel_size = 1
rank_offset = 0          # ranks [0, 4)

[module.images]
tensor_model_parallel_size = 1
pipeline_model_parallel_size = 1
data_parallel_size = 4
rank_offset = 4          # ranks [4, 8)

[run]
global_batch = 8
"""

# Appendix B, right panel: one shared GPU set
APPENDIX_B_RIGHT = """
[module.language]
tensor_model_parallel_size = 4
pipeline_model_parallel_size = 1
data_parallel_size = 2
rank_offset = 0
[module.images]
data_parallel_size = 8
[run]
global_batch = 64
num_microbatches = 1
tolerance = 1e-10
seed = 7
"""


def test_appendix_b_left_is_noncolocated():
    c = parse_config(APPENDIX_B_LEFT)
    assert list(c.modules) == ["language", "images"]
    assert (c.language.tp, c.language.pp, c.language.dp, c.language.rank_offset) == (2, 2, 1, 0)
    e = c.edge("images", 16)
    assert placement_of_edge(e) == Placement.NonColocated
    assert (e.source.rank_begin(), e.source.rank_end()) == (4, 8)
    assert (e.dest.rank_begin(), e.dest.rank_end()) == (0, 4)


def test_appendix_b_right_is_colocated_and_matches_c2():
    c = parse_config(APPENDIX_B_RIGHT)
    assert c.seed == 7 and c.tolerance == pytest.approx(1e-10) and c.global_batch == 64
    c2 = configs.get("c2")
    e = c.edge("images", c2.width)
    assert placement_of_edge(e) == Placement.Colocated
    # the same plan as the hand-built C2 edge (names aside)
    ref = hbb.export_plan(hbb.plan_bridge(c2.edge()))
    got = hbb.export_plan(hbb.plan_bridge(e))
    assert got.replace("images", "vit").replace("language", "llm") == ref


def test_microbatch_edge():
    c = parse_config(APPENDIX_B_RIGHT.replace("num_microbatches = 1", "num_microbatches = 4"))
    assert c.edge("images", 8).global_batch == 16


def test_indivisible_batch_is_a_validation_error():
    text = APPENDIX_B_RIGHT.replace("data_parallel_size = 8", "data_parallel_size = 3").replace(
        "global_batch = 64", "global_batch = 8")
    with pytest.raises(HetBridgeError) as ei:
        parse_config(text)
    assert ei.value.code == "ValidationError" and "IndivisibleBatch" in str(ei.value)


def test_partial_overlap_is_a_validation_error():
    text = APPENDIX_B_LEFT.replace("rank_offset = 4", "rank_offset = 2")
    with pytest.raises(HetBridgeError) as ei:
        parse_config(text)
    assert ei.value.code == "ValidationError" and "PartialOverlap" in str(ei.value)


@pytest.mark.parametrize("text,line,what", [
    ("[module.language]\ntensor_model_parallel_size = two\n", 2, "integer or decimal"),
    ("[module.language]\nwidth = 3\n", 2, "unknown module key"),
    ("[modules]\n", 1, "unknown section"),
    ("[module.language\n", 1, "unterminated"),
    ("tensor_model_parallel_size = 2\n", 1, "outside any section"),
    ("[module.language]\n\n# c\ndata_parallel_size = 2\ndata_parallel_size = 4\n", 5, "repeated"),
    ("[module.language]\n[module.language]\n", 2, "defined twice"),
    ("[module.language]\ndata_parallel_size = 0\n", 2, "out of range"),
    ("[module.language]\njust words\n", 2, "expected 'key = value'"),
])
def test_parse_errors_carry_the_line(text, line, what):
    with pytest.raises(HetBridgeError) as ei:
        parse_config(text)
    assert ei.value.code == "ParseError"
    assert f"line {line}:" in str(ei.value) and what in str(ei.value)


@pytest.mark.parametrize("text,what", [
    ("[module.images]\ndata_parallel_size = 2\n", "exactly one [module.language]"),
    ("[module.language]\ndata_parallel_size = 2\n", "at least one encoder"),
])
def test_module_set_invariants(text, what):
    with pytest.raises(HetBridgeError) as ei:
        parse_config(text)
    assert ei.value.code == "ValidationError" and what in str(ei.value)


@pytest.mark.parametrize("text", [APPENDIX_B_LEFT, APPENDIX_B_RIGHT])
def test_render_round_trip_is_stable(text):
    c = parse_config(text)
    r1 = c.render()
    c2 = parse_config(r1)
    assert c2.render() == r1
    assert c2.modules == c.modules
    assert (c2.global_batch, c2.num_microbatches, c2.seed) == (c.global_batch, c.num_microbatches, c.seed)


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4", "c5"])
def test_baseline_configs_expressible(name):
    """Every BASELINE config's layouts round-trip through the grammar into the same edge."""
    cfg = configs.get(name, scale=64)
    keys = ("tensor_model_parallel_size", "context_parallel_size", "pipeline_model_parallel_size",
            "data_parallel_size", "rank_offset")
    lines = []
    for mod, lay in (("language", cfg.dst), ("enc", cfg.src)):
        lines.append(f"[module.{mod}]")
        lines += [f"{k} = {v}" for k, v in zip(keys, (lay.tp, lay.cp, lay.pp, lay.dp, lay.rank_offset))]
    lines += ["[run]", f"global_batch = {cfg.batch}"]
    e = parse_config("\n".join(lines) + "\n").edge("enc", cfg.width)
    want = cfg.edge()
    for a, b in ((e.source, want.source), (e.dest, want.dest)):
        assert (a.tp, a.cp, a.pp, a.dp, a.rank_offset) == (b.tp, b.cp, b.pp, b.dp, b.rank_offset)
    assert (e.global_batch, e.feature_width) == (want.global_batch, want.feature_width)
