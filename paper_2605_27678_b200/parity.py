"""Parity metric and the device-side restatement of the ownership maps.

``ParityReport`` / ``parity_compare`` follow the reference's
``hetsim::oracle::ParityReport`` / ``parity_compare``
(R:core/include/hetsim/oracle.hpp:53-75): the worst
``|a - b| / max(1, |b|)`` per named tensor, items sorted worst-first, judged
against one tolerance; names or shapes that disagree raise StructureMismatch.

``expected_forward`` / ``expected_backward`` restate, with plain torch slicing
on whatever device holds the inputs, what the boundary kernels must produce
from the index maps the plan compiles to (``hb_index_forward`` /
``hb_index_backward_balanced``): one source element per destination element
(forward, bit-exact) and ordered fp32 sums from +0.0 accumulated with
``beta`` (backward). ``bench.py`` checks the buffers it just timed against
them at full width on every rank. The maps themselves are pinned against the
oracle by the CPU tests (tests/test_index_map.py, tests/test_golden.py).
"""
from __future__ import annotations

from dataclasses import dataclass, field

from ._lib import HetBridgeError

STRUCTURE_MISMATCH = 21  # ErrorCode::StructureMismatch ordinal + 1 (error.hpp)


@dataclass
class ParityItem:
    tensor: str
    max_rel: float = 0.0


@dataclass
class ParityReport:
    items: list = field(default_factory=list)  # sorted worst-first
    loss_rel: float = 0.0
    tolerance: float = 0.0
    passed: bool = False

    @property
    def pass_(self) -> bool:  # the reference's field name is `pass`
        return self.passed

    def worst(self) -> float:
        return max([self.loss_rel] + [i.max_rel for i in self.items])

    def render(self) -> str:
        lines = [f"parity {'PASS' if self.passed else 'FAIL'} tol={self.tolerance:g} loss_rel={self.loss_rel:.3g}"]
        lines += [f"  {i.tensor}: max_rel={i.max_rel:.3g}" for i in self.items]
        return "\n".join(lines)

    def render_machine(self) -> str:
        """One ``parity tensor=<name> max_rel=<v> pass=<0|1>`` line per tensor."""
        return "\n".join(f"parity tensor={i.tensor} max_rel={i.max_rel:.17g} pass={int(i.max_rel <= self.tolerance)}"
                         for i in self.items)


def _max_rel(a, b) -> float:
    import numpy as np

    try:
        import torch

        if isinstance(a, torch.Tensor) or isinstance(b, torch.Tensor):
            a = torch.as_tensor(a).double()
            b = torch.as_tensor(b, device=a.device).double()
            if a.numel() == 0:
                return 0.0
            return float(((a - b).abs() / b.abs().clamp(min=1.0)).max())
    except ImportError:  # numpy-only callers
        pass
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    if a.size == 0:
        return 0.0
    return float(np.max(np.abs(a - b) / np.maximum(1.0, np.abs(b))))


def parity_compare(distributed: dict, reference: dict, distributed_loss: float = 0.0,
                   reference_loss: float = 0.0, tolerance: float = 1e-10) -> ParityReport:
    """oracle.hpp:71-75: elementwise |a-b|/max(1,|b|) per named tensor."""
    if set(distributed) != set(reference):
        raise HetBridgeError(STRUCTURE_MISMATCH, f"tensor names differ: {sorted(set(distributed) ^ set(reference))}")
    items = []
    for name in sorted(distributed):
        a, b = distributed[name], reference[name]
        if tuple(getattr(a, "shape", ())) != tuple(getattr(b, "shape", ())):
            raise HetBridgeError(STRUCTURE_MISMATCH, f"{name}: shape {tuple(a.shape)} vs {tuple(b.shape)}")
        items.append(ParityItem(name, _max_rel(a, b)))
    items.sort(key=lambda i: -i.max_rel)
    loss_rel = abs(distributed_loss - reference_loss) / max(1.0, abs(reference_loss))
    rep = ParityReport(items, loss_rel, tolerance)
    rep.passed = all(i.max_rel <= tolerance for i in items) and loss_rel <= tolerance
    return rep


# ---------------------------------------------------------------------------- restatement


def expected_forward(fwd_map, rank: int, numel: int, src_of, base=None):
    """Destination buffer of ``rank`` the forward must produce.

    fwd_map: ``bridge.index_forward`` tuples; src_of(rank, slot) -> 1-D tensor of
    that source buffer (any device). base: the buffer before the op, for maps
    that write only part of it (an in-place splice leaves the text rows the
    caller wrote); elements outside the map must keep it. Returns (expected,
    covered elements)."""
    import torch

    out = None if base is None else base.clone()
    covered = 0
    for (sr, ss, so, dr, ds, do, n) in fwd_map:
        if dr != rank:
            continue
        s = src_of(sr, ss)
        if out is None:
            out = torch.zeros(numel, dtype=s.dtype, device=s.device)
        out[do:do + n] = s[so:so + n]
        covered += n
    return out, covered


def expected_backward(bwd_map, rank: int, prev, beta: float, term_of):
    """Source-gradient buffer of ``rank`` after one backward: for each run,
    beta*prev + (0.0 + t0 + t1 + ...) in fp32 in term order — the kernel's
    operation sequence (fmaf(beta, prev, sum) == prev + sum for beta = 1), so a
    correct kernel matches bit for bit. prev: fp32 1-D tensor (the buffer before
    the op); term_of(rank, slot) -> 1-D tensor of a destination gradient."""
    import torch

    out = prev.clone() if beta != 0.0 else torch.zeros_like(prev)
    for (dr, ds, do, n, terms) in bwd_map:
        if dr != rank:
            continue
        acc = None
        for (tr, ts, to) in terms:
            t = term_of(tr, ts)[to:to + n].to(device=prev.device, dtype=torch.float32)
            acc = (0.0 + t) if acc is None else acc + t
        if acc is None:
            acc = torch.zeros(n, dtype=torch.float32, device=prev.device)
        if beta == 0.0:
            out[do:do + n] = acc
        elif beta == 1.0:
            out[do:do + n] = prev[do:do + n] + acc
        else:
            out[do:do + n] = torch.addcmul(acc, prev[do:do + n], torch.full_like(acc, beta))
    return out
