"""module_parallelisms configuration ingestion — Python face of ``parse_config``.

The reference specifies the schema in SPEC.md's cli module (S:495-545:
``ExperimentConfig``, ``parse_config``, the ``[module.<name>]`` grammar),
mirroring the paper's Appendix B ``module_parallelisms={"language": ...,
"images": ...}``. Parsing and validation run in the product
library (``csrc/hb/config.cpp``); errors keep the reference categories
(``ParseError`` with the line number, ``ValidationError`` naming the invariant).

    cfg = parse_config(open("exp.cfg").read())
    edge = cfg.edge("images", feature_width=576 * 4096)   # -> bridge.plan_bridge(edge)
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

from . import _lib
from ._lib import check, lib
from .grid import BoundaryEdge, ModuleLayout


def _layout(c: _lib.Layout) -> ModuleLayout:
    return ModuleLayout(c.name.decode(), c.tp, c.cp, c.pp, c.dp, c.rank_offset)


@dataclass
class ExperimentConfig:
    modules: dict = field(default_factory=dict)  # name -> ModuleLayout, file order
    global_batch: int = 0
    num_microbatches: int = 1
    steps: int = 1
    seed: int = 0
    tolerance: float = 0.0
    _h: object = None

    @property
    def language(self) -> ModuleLayout:
        return self.modules["language"]

    @property
    def encoders(self) -> list:
        return [m for n, m in self.modules.items() if n != "language"]

    def edge(self, encoder: str, feature_width: int) -> BoundaryEdge:
        """Encoder -> language edge of one microbatch (global_batch / num_microbatches samples)."""
        e = _lib.Edge()
        check(lib().hb_config_edge(self._h, encoder.encode(), feature_width, ctypes.byref(e)))
        return BoundaryEdge(_layout(e.source), _layout(e.dest), e.global_batch, e.feature_width)

    def render(self) -> str:
        n = ctypes.c_size_t()
        check(lib().hb_config_render(self._h, None, 0, ctypes.byref(n)))
        buf = ctypes.create_string_buffer(n.value + 1)
        check(lib().hb_config_render(self._h, buf, n.value + 1, ctypes.byref(n)))
        return buf.value.decode()

    def __del__(self):
        h, self._h = self._h, None
        if h and _lib._lib is not None:
            _lib._lib.hb_config_destroy(h)


def parse_config(text: str) -> ExperimentConfig:
    h = ctypes.c_void_p()
    check(lib().hb_config_parse(text.encode(), ctypes.byref(h)))
    cfg = ExperimentConfig(_h=h)
    n = ctypes.c_int()
    check(lib().hb_config_num_modules(h, ctypes.byref(n)))
    for i in range(n.value):
        lay, is_lang = _lib.Layout(), ctypes.c_int()
        check(lib().hb_config_module(h, i, ctypes.byref(lay), ctypes.byref(is_lang)))
        m = _layout(lay)
        cfg.modules[m.name] = m
    gb, nmb, steps, seed, tol = ctypes.c_int(), ctypes.c_int(), ctypes.c_int(), ctypes.c_longlong(), ctypes.c_double()
    check(lib().hb_config_run(h, ctypes.byref(gb), ctypes.byref(nmb), ctypes.byref(steps), ctypes.byref(seed),
                              ctypes.byref(tol)))
    cfg.global_batch, cfg.num_microbatches, cfg.steps = gb.value, nmb.value, steps.value
    cfg.seed, cfg.tolerance = seed.value, tol.value
    return cfg
