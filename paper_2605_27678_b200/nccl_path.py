"""NCCL comparison path: the reference's boundary plan executed literally with NCCL.

This is the *comparison* leg the north star asks for ("NCCL send/recv over
NVLink only as the comparison path"), not the product. It replays the plan the
way the reference's runtime would move bytes over simnet
(``R:core/include/hetsim/bridge.hpp:17-36``; steps as ``export_plan`` lists
them):

* non-colocated: leader send/recv of each piece, then the destination TP/CP
  broadcast; backward: cp all-reduce, leader send/recv back, source broadcast;
* colocated: k-member all-gathers, deliver broadcasts, local selects; backward:
  cp all-reduce, sibling all-gathers, delivers, selects;
* CP splice: the reference composition, i.e. the full bridge forward followed
  by a local ``assemble_tokens`` per CP slice (and ``split_vision_grad`` + bridge
  backward), which is what the fused hetbridge kernels avoid.

One process per logical rank (``WORLD_SIZE == plan.world``), NCCL via
torch.distributed. Gradients are reduced in fp32.
"""
from __future__ import annotations

import re

import torch
import torch.distributed as dist

from . import bridge as hbb

_IV = re.compile(r"\[(\d+),(\d+)\)")
_GRP = re.compile(r"group=\[([\d,]+)\]")


def _parse(text: str):
    steps = []
    for ln in text.strip().splitlines()[1:]:
        parts = ln.split()
        direction, op = parts[0], parts[1]
        ivs = [(int(a), int(b)) for a, b in _IV.findall(ln)]
        st = {"dir": direction, "op": op, "iv": ivs[-1]}
        m = _GRP.search(ln)
        if m:
            st["group"] = [int(x) for x in m.group(1).split(",")]
        if op == "send":
            st["src"], st["dst"] = int(parts[2][1:]), int(parts[4][1:])
        if "root=" in ln:
            st["root"] = int(ln.split("root=r")[1].split()[0])
        if op == "select":
            st["rank"] = int(parts[2][1:])
            st["parent"] = ivs[0]
        if op == "all_gather":
            st["parts"] = ivs[:-1]
        steps.append(st)
    return steps


class NcclPlanExecutor:
    def __init__(self, plan: hbb.BridgePlan, splice: hbb.SpliceSpec | None = None, device=None,
                 act_dtype=torch.bfloat16, grad_dtype=torch.bfloat16):
        self.plan, self.splice = plan, splice
        self.rank = dist.get_rank()
        if dist.get_world_size() != plan.world:
            raise ValueError("the NCCL comparison path needs one process per logical rank")
        self.dev = device or torch.device("cuda", torch.cuda.current_device())
        e = plan.edge
        self.W = e.feature_width
        self.steps = _parse(hbb.export_plan(plan, 8))
        self.SI, self.DI = plan.src_intervals, plan.dest_intervals
        from .grid import coord_of_rank, ranks_of_stage

        self.src_stage = ranks_of_stage(e.source, e.source.pp - 1)
        self.dst_stage = ranks_of_stage(e.dest, 0)
        r = self.rank
        self.s_iv = self.SI[coord_of_rank(e.source, r).dp_idx] if r in self.src_stage else None
        self.d_iv = self.DI[coord_of_rank(e.dest, r).dp_idx] if r in self.dst_stage else None
        self.cp_idx = coord_of_rank(e.dest, r).cp_idx if r in self.dst_stage else 0
        # every process creates every subgroup in the same order (torch requirement)
        self.groups = {}
        for st in self.steps:
            if "group" in st:
                key = tuple(sorted(st["group"]))
                if key not in self.groups:
                    self.groups[key] = dist.new_group(list(key))
        W = self.W
        z = lambda iv, dt: torch.zeros(iv.length, W, dtype=dt, device=self.dev) if iv else None  # noqa: E731
        self.src = z(self.s_iv, act_dtype)
        self.dst = z(self.d_iv, act_dtype)
        self.dst_grad = z(self.d_iv, torch.float32)
        self.src_grad = z(self.s_iv, torch.float32)
        self.gathered = {}
        if splice is not None:
            cp = e.dest.cp
            self.L = splice.S // cp
            codes = torch.from_numpy(splice.codes).to(self.dev).long().view(splice.Q, splice.S)
            self.codes = codes[:, self.cp_idx * self.L:(self.cp_idx + 1) * self.L].reshape(-1)
            self.tokens = torch.zeros(splice.Q * self.L, splice.d_h, dtype=act_dtype, device=self.dev)
            ntext = int((self.codes < 0).sum())
            self.text = torch.zeros(max(ntext, 1), splice.d_h, dtype=act_dtype, device=self.dev)
            self.token_grad = torch.zeros(splice.Q * self.L, splice.d_h, dtype=grad_dtype, device=self.dev)

    # --- helpers
    def _rows(self, buf, have, iv):
        a, b = iv
        return buf[a - have.start:b - have.start]

    def _run(self, direction):
        me = self.rank
        held = self.dst_grad if direction == "bwd" else None
        p2p = []
        for st in [s for s in self.steps if s["dir"] == direction]:
            op = st["op"]
            if op == "send":
                if me == st["src"]:
                    buf = self.src if direction == "fwd" else held
                    have = self.s_iv if direction == "fwd" else self.d_iv
                    p2p.append(dist.P2POp(dist.isend, self._rows(buf, have, st["iv"]).contiguous(), st["dst"]))
                elif me == st["dst"]:
                    out = self.dst if direction == "fwd" else self.src_grad
                    have = self.d_iv if direction == "fwd" else self.s_iv
                    view = self._rows(out, have, st["iv"])
                    p2p.append(dist.P2POp(dist.irecv, view, st["src"]))
                continue
            if p2p:  # flush batched point-to-point before the next collective
                for req in dist.batch_isend_irecv(p2p):
                    req.wait()
                p2p = []
            if me not in st.get("group", [st.get("rank", -1)]):
                continue
            grp = self.groups.get(tuple(sorted(st.get("group", []))))
            if op == "broadcast":
                buf = self.dst if direction == "fwd" else self.src_grad
                dist.broadcast(buf, src=st["root"], group=grp)
            elif op == "all_reduce":
                dist.all_reduce(held, group=grp)
            elif op == "all_gather":
                a, b = st["iv"]
                if direction == "fwd":
                    own = self.d_iv is not None and (self.d_iv.start, self.d_iv.end()) == (a, b)
                    out = self.dst if own else torch.empty(b - a, self.W, dtype=self.src.dtype, device=self.dev)
                    dist.all_gather_into_tensor(out, self.src, group=grp)
                else:
                    own = self.s_iv is not None and (self.s_iv.start, self.s_iv.end()) == (a, b)
                    out = self.src_grad if own else torch.empty(b - a, self.W, dtype=torch.float32, device=self.dev)
                    dist.all_gather_into_tensor(out, held, group=grp)
                self.gathered[(a, b)] = out
            elif op == "deliver":
                root = st["root"]
                a, b = st["iv"]
                if direction == "fwd":
                    if me == root:
                        if (a, b) in self.gathered:
                            tmp = self.gathered[(a, b)].contiguous()
                        else:
                            tmp = self._rows(self.src, self.s_iv, st["iv"]).contiguous()
                    else:
                        tmp = torch.empty(b - a, self.W, dtype=self.dst.dtype, device=self.dev)
                    dist.broadcast(tmp, src=root, group=grp)
                    if me != root:
                        self.dst.copy_(tmp)
                else:
                    if me == root:
                        if (a, b) in self.gathered:
                            tmp = self.gathered[(a, b)].contiguous()
                        else:
                            tmp = self._rows(held, self.d_iv, st["iv"]).contiguous()
                    else:
                        tmp = torch.empty(b - a, self.W, dtype=torch.float32, device=self.dev)
                    dist.broadcast(tmp, src=root, group=grp)
                    if me != root:
                        self.src_grad.copy_(tmp)
            elif op == "select" and me == st["rank"]:
                if direction == "fwd":
                    self.dst.copy_(self._rows(self.src, self.s_iv, st["iv"]))
                else:
                    self.src_grad.copy_(self._rows(held, self.d_iv, st["iv"]))
        if p2p:
            for req in dist.batch_isend_irecv(p2p):
                req.wait()

    # --- public
    def forward(self):
        self.gathered = {}
        self._run("fwd")
        if self.splice is not None and self.d_iv is not None:
            d_h = self.splice.d_h
            vis = self.dst.view(-1, d_h)
            c = self.codes
            txt_rows = torch.cumsum((c < 0).long(), 0) - 1
            self.tokens.copy_(torch.where((c >= 0)[:, None], vis[c.clamp(min=0)], self.text[txt_rows.clamp(min=0)]))

    def backward(self):
        self.gathered = {}
        if self.splice is not None and self.d_iv is not None:
            d_h = self.splice.d_h
            g = torch.zeros(self.dst_grad.numel() // d_h, d_h, dtype=torch.float32, device=self.dev)
            c = self.codes
            sel = c >= 0
            g.index_add_(0, c[sel], self.token_grad[sel].float())
            self.dst_grad.view(-1, d_h).copy_(g)
        self._run("bwd")
