// ORACLE — test infrastructure only. Never linked into or called by the
// product path (paper_2605_27678_b200/). Only tests/, __graft_entry__.smoke()
// and bench.py's cpu_baseline / --impl reference leg may load it.
//
// CPU restatement of the reference's boundary communicator. The reference
// declares the API in /root/reference/proj/core/include/hetsim/bridge.hpp:1-187
// but ships no body (proj/core/src/bridge.cpp is a 2-line stub), so this file
// implements exactly those declarations, following:
//   * bridge.hpp:17-36   (contract: leader routing, colocated reinterpretation,
//                          replica-gradient rule: tp replicas identical, cp summed)
//   * SPEC.md:109-189    (plan_bridge / bridge_forward / bridge_backward contract)
//   * SURVEY.md App. A   (reference-silent choices, marked with "◆")
// and executes every transfer over the reference's own deterministic fabric
// (proj/core/src/simnet.cpp) and layout algebra (proj/core/src/grid.cpp),
// which are compiled from their sources by oracle/Makefile.
//
// Parity status: the bridge has no executable reference test; this oracle is
// pinned by the SPEC prose known-answer tests made executable in
// tests/test_oracle_kats.py and by the reference's own grid tests.

#include <algorithm>
#include <sstream>
#include <stdexcept>

#include "hetsim/bridge.hpp"

namespace hetsim::bridge {

using grid::BatchInterval;
using grid::GridCoord;
using grid::ModuleLayout;
using simnet::Direction;
using simnet::Payload;

const char* dp_kind_name(DpKind k) {
  switch (k) {
    case DpKind::Equal: return "Equal";
    case DpKind::FanIn: return "FanIn";
    case DpKind::FanOut: return "FanOut";
  }
  return "Unknown";
}

void ShardedTensor::validate() const {
  if (interval.length < 0 || feature_width < 0)
    raise(ErrorCode::InvalidArgument, "negative shard shape");
  if (payload.size() != static_cast<size_t>(interval.length) * feature_width)
    raise(ErrorCode::ShapeMismatch,
          "shard payload has " + std::to_string(payload.size()) + " elements, expected " +
              std::to_string(static_cast<long>(interval.length) * feature_width));
}

ShardedTensor make_shard(const BatchInterval& iv, int width, double fill) {
  ShardedTensor t;
  t.interval = iv;
  t.feature_width = width;
  t.payload.assign(static_cast<size_t>(iv.length) * width, fill);
  return t;
}

namespace {

bool intersect(const BatchInterval& a, const BatchInterval& b, BatchInterval* out) {
  const int s = std::max(a.start, b.start), e = std::min(a.end(), b.end());
  if (e <= s) return false;
  *out = {s, e - s};
  return true;
}

bool covers(const BatchInterval& outer, const BatchInterval& inner) {
  return inner.start >= outer.start && inner.end() <= outer.end();
}

// Rows `want` of a payload that holds rows `have`, row width W.
Payload rows_of(const Payload& p, const BatchInterval& have, const BatchInterval& want,
                int width) {
  if (!covers(have, want))
    raise(ErrorCode::PlanInfeasible, "interval " + grid::to_string(want) +
                                         " not inside held " + grid::to_string(have));
  const size_t off = static_cast<size_t>(want.start - have.start) * width;
  const size_t n = static_cast<size_t>(want.length) * width;
  return Payload(p.begin() + off, p.begin() + off + n);
}

bool contains(const std::vector<int>& v, int x) {
  return std::find(v.begin(), v.end(), x) != v.end();
}

std::string grp(const std::vector<int>& g) {
  std::string s = "[";
  for (size_t i = 0; i < g.size(); ++i) s += (i ? "," : "") + std::to_string(g[i]);
  return s + "]";
}

// Collective / channel labels. Per-step labels keep simnet's group-mismatch
// detector (simnet.cpp:229-251) from conflating distinct steps.
std::string L(const BridgePlan& p, const char* dir, const char* kind, int idx = -1) {
  std::string s = p.label + "/" + dir + "/" + kind;
  if (idx >= 0) s += "/" + std::to_string(idx);
  return s;
}

// Destination stage-0 holders of DI[d] in backward, in position order (◆):
// tp=0 ranks of every cp slice when cp>1 (after the cp all_reduce), else every
// tp replica (each holds its own, contractually identical, gradient).
std::vector<int> bwd_holders(const ModuleLayout& dst, int d) {
  std::vector<int> h;
  if (dst.cp > 1) {
    for (int c = 0; c < dst.cp; ++c) h.push_back(grid::rank_of_coord(dst, GridCoord{0, c, 0, d}));
  } else {
    for (int t = 0; t < dst.tp; ++t) h.push_back(grid::rank_of_coord(dst, GridCoord{t, 0, 0, d}));
  }
  return h;
}

}  // namespace

// --- classification & planning ----------------------------------------------

// SPEC.md:131-139; NonIntegerFan when neither DP divides the other.
DpRelation classify_dp_relation(const grid::BoundaryEdge& edge) {
  edge.source.validate();
  edge.dest.validate();
  const int u = edge.source.dp, v = edge.dest.dp;
  if (u == v) return {DpKind::Equal, 1};
  if (u > v && u % v == 0) return {DpKind::FanIn, u / v};
  if (v > u && v % u == 0) return {DpKind::FanOut, v / u};
  raise(ErrorCode::NonIntegerFan, "dp " + std::to_string(u) + " -> " + std::to_string(v) +
                                      " is not an integer fan");
}

int BridgePlan::cross_boundary_messages() const {
  if (placement != grid::Placement::NonColocated) return 0;
  int n = 0;
  for (const auto& r : nc.routes) n += static_cast<int>(r.pieces.size());
  return n;
}

BridgePlan plan_bridge(const grid::BoundaryEdge& edge) {
  BridgePlan p;
  p.edge = edge;
  p.placement = grid::placement_of_edge(edge);  // PartialOverlap (grid.cpp:80)
  p.relation = classify_dp_relation(edge);
  if (edge.feature_width < 1)
    raise(ErrorCode::InvalidArgument, "feature_width must be >= 1");
  p.src_intervals = grid::partition_batch(edge.global_batch, edge.source.dp);
  p.dest_intervals = grid::partition_batch(edge.global_batch, edge.dest.dp);
  p.label = edge.source.name + "->" + edge.dest.name;

  const ModuleLayout& src = edge.source;
  const ModuleLayout& dst = edge.dest;
  const int ps = src.pp - 1;  // boundary source stage
  const auto& SI = p.src_intervals;
  const auto& DI = p.dest_intervals;
  const int k = p.relation.factor;
  const DpKind kind = p.relation.kind;

  if (p.placement == grid::Placement::NonColocated) {
    for (int d = 0; d < dst.dp; ++d) {
      NcRoute r;
      r.dest_shard = d;
      r.dest_leader = grid::leader_rank(dst, 0, d);
      for (int s = 0; s < src.dp; ++s) {
        BatchInterval iv;
        if (intersect(SI[s], DI[d], &iv)) r.pieces.push_back({grid::leader_rank(src, ps, s), iv});
      }
      r.bcast_group = grid::replica_group(dst, 0, d);
      p.nc.routes.push_back(r);
    }
    for (int s = 0; s < src.dp; ++s) {
      p.nc.src_shards.push_back(
          {s, grid::leader_rank(src, ps, s), SI[s], grid::replica_group(src, ps, s)});
    }
    if (dst.cp > 1) {
      for (int d = 0; d < dst.dp; ++d) {
        ReduceStep rs;
        rs.dest_shard = d;
        for (int c = 0; c < dst.cp; ++c) rs.group.push_back(grid::rank_of_coord(dst, {0, c, 0, d}));
        std::sort(rs.group.begin(), rs.group.end());
        p.nc.reduces.push_back(rs);
      }
    }
    return p;
  }

  // Colocated (bridge.hpp:26-31).
  ColoPlan& cp = p.colo;
  const auto Rs = grid::ranks_of_stage(src, ps);
  const auto Rd = grid::ranks_of_stage(dst, 0);
  auto src_shard_of = [&](int r) { return grid::coord_of_rank(src, r).dp_idx; };
  auto dst_shard_of = [&](int r) { return grid::coord_of_rank(dst, r).dp_idx; };

  // ---- forward
  std::vector<std::vector<int>> cover_fwd(dst.dp);  // ranks holding data covering DI[d]
  if (kind == DpKind::FanIn) {
    for (int d = 0; d < dst.dp; ++d) {
      for (int j = 0; j < src.tp * src.cp; ++j) {
        GatherStep g;
        g.shard = d;
        for (int s = k * d; s < k * d + k; ++s) {
          g.members.push_back(grid::rank_of_coord(src, {j % src.tp, j / src.tp, ps, s}));
          g.member_intervals.push_back(SI[s]);
        }
        for (int m : g.members) cover_fwd[d].push_back(m);
        cp.fwd_gathers.push_back(g);
      }
    }
  } else {
    for (int r : Rs) {
      const int s = src_shard_of(r);
      for (int d = 0; d < dst.dp; ++d)
        if (covers(SI[s], DI[d])) cover_fwd[d].push_back(r);
    }
  }
  std::vector<std::vector<int>> need_fwd(dst.dp);
  for (int r : Rd) {
    const int d = dst_shard_of(r);
    bool done = false;
    if (kind == DpKind::FanIn) {
      for (size_t i = 0; i < cp.fwd_gathers.size() && !done; ++i) {
        const auto& g = cp.fwd_gathers[i];
        if (g.shard == d && contains(g.members, r)) {
          cp.fwd_actions[r] = {ColoSource::Gather, static_cast<int>(i), DI[d], DI[d]};
          done = true;
        }
      }
    } else if (contains(Rs, r) && covers(SI[src_shard_of(r)], DI[d])) {
      cp.fwd_actions[r] = {ColoSource::OwnShard, -1, SI[src_shard_of(r)], DI[d]};
      done = true;
    }
    if (!done) need_fwd[d].push_back(r);
  }
  for (int d = 0; d < dst.dp; ++d) {
    if (need_fwd[d].empty()) continue;
    DeliverStep st;  // ◆ root = lowest covering rank; group = root + receivers ascending
    st.root = *std::min_element(cover_fwd[d].begin(), cover_fwd[d].end());
    st.group.push_back(st.root);
    for (int r : need_fwd[d]) st.group.push_back(r);
    st.shard = d;
    st.interval = DI[d];
    const int idx = static_cast<int>(cp.fwd_delivers.size());
    cp.fwd_delivers.push_back(st);
    for (int r : need_fwd[d]) cp.fwd_actions[r] = {ColoSource::Deliver, idx, DI[d], DI[d]};
  }

  // ---- backward
  if (dst.cp > 1) {
    for (int d = 0; d < dst.dp; ++d) {
      ReduceStep rs;
      rs.dest_shard = d;
      for (int c = 0; c < dst.cp; ++c) rs.group.push_back(grid::rank_of_coord(dst, {0, c, 0, d}));
      std::sort(rs.group.begin(), rs.group.end());
      cp.bwd_reduces.push_back(rs);
    }
  }
  std::vector<std::vector<int>> cover_bwd(src.dp);
  if (kind == DpKind::FanOut) {
    const int H = static_cast<int>(bwd_holders(dst, 0).size());
    for (int s = 0; s < src.dp; ++s) {
      for (int h = 0; h < H; ++h) {
        GatherStep g;
        g.shard = s;
        for (int d = k * s; d < k * s + k; ++d) {
          g.members.push_back(bwd_holders(dst, d)[h]);
          g.member_intervals.push_back(DI[d]);
        }
        for (int m : g.members) cover_bwd[s].push_back(m);
        cp.bwd_gathers.push_back(g);
      }
    }
  } else {
    for (int s = 0; s < src.dp; ++s) {
      const int d = (kind == DpKind::FanIn) ? s / k : s;
      for (int h : bwd_holders(dst, d)) cover_bwd[s].push_back(h);
    }
  }
  std::vector<std::vector<int>> need_bwd(src.dp);
  for (int r : Rs) {
    const int s = src_shard_of(r);
    bool done = false;
    if (kind == DpKind::FanOut) {
      for (size_t i = 0; i < cp.bwd_gathers.size() && !done; ++i) {
        const auto& g = cp.bwd_gathers[i];
        if (g.shard == s && contains(g.members, r)) {
          cp.bwd_actions[r] = {ColoSource::Gather, static_cast<int>(i), SI[s], SI[s]};
          done = true;
        }
      }
    } else {
      const int d = (kind == DpKind::FanIn) ? s / k : s;
      if (contains(bwd_holders(dst, d), r)) {
        cp.bwd_actions[r] = {ColoSource::OwnGrad, -1, DI[d], SI[s]};
        done = true;
      }
    }
    if (!done) need_bwd[s].push_back(r);
  }
  for (int s = 0; s < src.dp; ++s) {
    if (need_bwd[s].empty()) continue;
    DeliverStep st;  // ◆ root = lowest holder covering SI[s]
    st.root = *std::min_element(cover_bwd[s].begin(), cover_bwd[s].end());
    st.group.push_back(st.root);
    for (int r : need_bwd[s]) st.group.push_back(r);
    st.shard = s;
    st.interval = SI[s];
    const int idx = static_cast<int>(cp.bwd_delivers.size());
    cp.bwd_delivers.push_back(st);
    for (int r : need_bwd[s]) cp.bwd_actions[r] = {ColoSource::Deliver, idx, SI[s], SI[s]};
  }
  return p;
}

// Structured-text export: one line per transfer/collective,
// byte counts follow simnet's ledger accounting (simnet.cpp:281-313,460-462)
// with 8-byte elements (simnet.hpp:27-29).
std::string export_plan(const BridgePlan& p) {
  std::ostringstream os;
  const long W = p.edge.feature_width;
  const long E = 8;
  auto bytes = [&](const BatchInterval& iv) { return static_cast<long>(iv.length) * W * E; };
  os << "edge " << p.label << " placement="
     << (p.placement == grid::Placement::Colocated ? "Colocated" : "NonColocated")
     << " relation=" << dp_kind_name(p.relation.kind) << " k=" << p.relation.factor
     << " batch=" << p.edge.global_batch << " width=" << W << " elem_bytes=" << E << "\n";
  if (p.placement == grid::Placement::NonColocated) {
    for (const auto& r : p.nc.routes) {
      for (const auto& [ldr, iv] : r.pieces)
        os << "fwd send r" << ldr << " -> r" << r.dest_leader << " " << grid::to_string(iv)
           << " bytes=" << bytes(iv) << "\n";
      if (r.bcast_group.size() > 1)
        os << "fwd broadcast root=r" << r.dest_leader << " group=" << grp(r.bcast_group) << " "
           << grid::to_string(p.dest_intervals[r.dest_shard])
           << " bytes=" << bytes(p.dest_intervals[r.dest_shard]) * (long)(r.bcast_group.size() - 1)
           << "\n";
    }
    for (const auto& rs : p.nc.reduces) {
      const long n = static_cast<long>(rs.group.size());
      os << "bwd all_reduce group=" << grp(rs.group) << " "
         << grid::to_string(p.dest_intervals[rs.dest_shard])
         << " bytes=" << bytes(p.dest_intervals[rs.dest_shard]) * n * (n - 1) << "\n";
    }
    for (const auto& r : p.nc.routes)
      for (const auto& [ldr, iv] : r.pieces)
        os << "bwd send r" << r.dest_leader << " -> r" << ldr << " " << grid::to_string(iv)
           << " bytes=" << bytes(iv) << "\n";
    for (const auto& s : p.nc.src_shards)
      if (s.bcast_group.size() > 1)
        os << "bwd broadcast root=r" << s.src_leader << " group=" << grp(s.bcast_group) << " "
           << grid::to_string(s.interval)
           << " bytes=" << bytes(s.interval) * (long)(s.bcast_group.size() - 1) << "\n";
    return os.str();
  }
  const ColoPlan& c = p.colo;
  auto gather_line = [&](const char* dir, const GatherStep& g, const BatchInterval& whole) {
    const long n = static_cast<long>(g.members.size());
    os << dir << " all_gather group=" << grp(g.members) << " parts=";
    for (size_t i = 0; i < g.member_intervals.size(); ++i)
      os << (i ? "+" : "") << grid::to_string(g.member_intervals[i]);
    os << " " << grid::to_string(whole) << " bytes=" << bytes(whole) * (n - 1) << "\n";
  };
  auto deliver_line = [&](const char* dir, const DeliverStep& s) {
    os << dir << " deliver root=r" << s.root << " group=" << grp(s.group) << " "
       << grid::to_string(s.interval)
       << " bytes=" << bytes(s.interval) * (long)(s.group.size() - 1) << "\n";
  };
  auto select_lines = [&](const char* dir, const std::map<int, ColoAction>& acts) {
    for (const auto& [r, a] : acts)
      if (a.from == ColoSource::OwnShard || a.from == ColoSource::OwnGrad)
        os << dir << " select r" << r << " " << grid::to_string(a.parent) << " -> "
           << grid::to_string(a.out) << " bytes=0\n";
  };
  for (const auto& g : c.fwd_gathers) gather_line("fwd", g, p.dest_intervals[g.shard]);
  for (const auto& s : c.fwd_delivers) deliver_line("fwd", s);
  select_lines("fwd", c.fwd_actions);
  for (const auto& rs : c.bwd_reduces) {
    const long n = static_cast<long>(rs.group.size());
    os << "bwd all_reduce group=" << grp(rs.group) << " "
       << grid::to_string(p.dest_intervals[rs.dest_shard])
       << " bytes=" << bytes(p.dest_intervals[rs.dest_shard]) * n * (n - 1) << "\n";
  }
  for (const auto& g : c.bwd_gathers) gather_line("bwd", g, p.src_intervals[g.shard]);
  for (const auto& s : c.bwd_delivers) deliver_line("bwd", s);
  select_lines("bwd", c.bwd_actions);
  return os.str();
}

// --- runtime -----------------------------------------------------------------

// a forward record is consumed exactly once by backward.
void BridgeRuntime::record_forward(int mb) {
  if (forward_done_.count(mb))
    raise(ErrorCode::InvalidArgument, "microbatch " + std::to_string(mb) +
                                          " forwarded twice without backward");
  forward_done_.insert(mb);
  backward_done_.erase(mb);
}

void BridgeRuntime::consume_forward(int mb) {
  if (!forward_done_.count(mb))
    raise(ErrorCode::UnknownMicrobatch,
          "no forward record for microbatch " + std::to_string(mb) +
              (backward_done_.count(mb) ? " (already consumed)" : ""));
  forward_done_.erase(mb);
  backward_done_.insert(mb);
}

namespace {
int src_shard_checked(const BridgePlan& p, int r) {
  const auto c = grid::coord_of_rank(p.edge.source, r);
  if (c.pp_idx != p.edge.source.pp - 1)
    raise(ErrorCode::RankOutOfModule, "rank " + std::to_string(r) + " not on the source boundary stage");
  return c.dp_idx;
}
int dst_shard_checked(const BridgePlan& p, int r) {
  const auto c = grid::coord_of_rank(p.edge.dest, r);
  if (c.pp_idx != 0)
    raise(ErrorCode::RankOutOfModule, "rank " + std::to_string(r) + " not on the destination stage 0");
  return c.dp_idx;
}
void check_shard(const BridgePlan& p, const ShardedTensor& t, const BatchInterval& want,
                 ErrorCode code) {
  if (t.feature_width != p.edge.feature_width || !(t.interval == want))
    raise(code, "shard " + grid::to_string(t.interval) + " x " + std::to_string(t.feature_width) +
                    " does not match planned " + grid::to_string(want) + " x " +
                    std::to_string(p.edge.feature_width));
  t.validate();
}
}  // namespace

void BridgeRuntime::forward_source(simnet::Rank& ctx, int mb, const ShardedTensor& shard) {
  const BridgePlan& p = *plan_;
  if (p.placement != grid::Placement::NonColocated)
    raise(ErrorCode::NotColocated, "forward_source on a colocated plan");
  const int me = ctx.id();
  const int s = src_shard_checked(p, me);
  check_shard(p, shard, p.src_intervals[s], ErrorCode::ShardIntervalMismatch);
  record_forward(mb);
  if (p.nc.src_shards[s].src_leader != me) return;  // non-leaders send nothing
  for (const auto& r : p.nc.routes)
    for (const auto& [ldr, iv] : r.pieces)
      if (ldr == me)
        ctx.send(r.dest_leader, L(p, "fwd", "send"), mb, Direction::Forward,
                 rows_of(shard.payload, shard.interval, iv, shard.feature_width));
}

ShardedTensor BridgeRuntime::forward_dest(simnet::Rank& ctx, int mb) {
  const BridgePlan& p = *plan_;
  if (p.placement != grid::Placement::NonColocated)
    raise(ErrorCode::NotColocated, "forward_dest on a colocated plan");
  const int me = ctx.id();
  const int d = dst_shard_checked(p, me);
  record_forward(mb);
  const NcRoute& r = p.nc.routes[d];
  Payload out;
  if (r.dest_leader == me) {
    for (const auto& [ldr, iv] : r.pieces) {
      Payload part = ctx.recv(ldr, L(p, "fwd", "send"), mb, Direction::Forward);
      out.insert(out.end(), part.begin(), part.end());  // batch order
    }
  }
  if (r.bcast_group.size() > 1)
    out = ctx.broadcast(r.bcast_group, r.dest_leader, L(p, "fwd", "broadcast", d), mb,
                        Direction::Forward, std::move(out));
  ShardedTensor t{p.dest_intervals[d], p.edge.feature_width, std::move(out)};
  t.validate();
  return t;
}

void BridgeRuntime::backward_dest(simnet::Rank& ctx, int mb, const ShardedTensor& grad) {
  const BridgePlan& p = *plan_;
  if (p.placement != grid::Placement::NonColocated)
    raise(ErrorCode::NotColocated, "backward_dest on a colocated plan");
  const int me = ctx.id();
  const int d = dst_shard_checked(p, me);
  check_shard(p, grad, p.dest_intervals[d], ErrorCode::GradIntervalMismatch);
  consume_forward(mb);
  const auto c = grid::coord_of_rank(p.edge.dest, me);
  Payload g = grad.payload;
  if (p.edge.dest.cp > 1) {
    if (c.tp_idx != 0) return;  // tp replicas contribute nothing (bridge.hpp:33-35)
    g = ctx.all_reduce(p.nc.reduces[d].group, L(p, "bwd", "all_reduce", d), mb,
                       Direction::Backward, std::move(g));
  }
  const NcRoute& r = p.nc.routes[d];
  if (r.dest_leader != me) return;
  for (const auto& [ldr, iv] : r.pieces)
    ctx.send(ldr, L(p, "bwd", "send"), mb, Direction::Backward,
             rows_of(g, p.dest_intervals[d], iv, p.edge.feature_width));
}

ShardedTensor BridgeRuntime::backward_source(simnet::Rank& ctx, int mb) {
  const BridgePlan& p = *plan_;
  if (p.placement != grid::Placement::NonColocated)
    raise(ErrorCode::NotColocated, "backward_source on a colocated plan");
  const int me = ctx.id();
  const int s = src_shard_checked(p, me);
  consume_forward(mb);
  const NcSrcShard& sh = p.nc.src_shards[s];
  Payload out;
  if (sh.src_leader == me) {
    for (const auto& r : p.nc.routes)
      for (const auto& [ldr, iv] : r.pieces)
        if (ldr == me) {
          Payload part = ctx.recv(r.dest_leader, L(p, "bwd", "send"), mb, Direction::Backward);
          out.insert(out.end(), part.begin(), part.end());
        }
  }
  if (sh.bcast_group.size() > 1)
    out = ctx.broadcast(sh.bcast_group, sh.src_leader, L(p, "bwd", "broadcast", s), mb,
                        Direction::Backward, std::move(out));
  ShardedTensor t{sh.interval, p.edge.feature_width, std::move(out)};
  t.validate();
  return t;
}

std::optional<ShardedTensor> BridgeRuntime::forward_colocated(
    simnet::Rank& ctx, int mb, const std::optional<ShardedTensor>& src) {
  const BridgePlan& p = *plan_;
  if (p.placement != grid::Placement::Colocated)
    raise(ErrorCode::NotColocated, "forward_colocated on a non-colocated plan");
  const ColoPlan& c = p.colo;
  const int me = ctx.id();
  const auto Rs = grid::ranks_of_stage(p.edge.source, p.edge.source.pp - 1);
  const auto Rd = grid::ranks_of_stage(p.edge.dest, 0);
  const bool in_src = contains(Rs, me), in_dst = contains(Rd, me);
  if (src) {
    if (!in_src) raise(ErrorCode::ShardIntervalMismatch, "rank holds no source shard slot");
    check_shard(p, *src, p.src_intervals[src_shard_checked(p, me)], ErrorCode::ShardIntervalMismatch);
  }
  record_forward(mb);
  auto need_src = [&]() -> const ShardedTensor& {
    if (!src) raise(ErrorCode::MissingSourceShard, "rank " + std::to_string(me) + " needs its source shard");
    return *src;
  };
  Payload gathered;
  BatchInterval gathered_iv;
  for (size_t i = 0; i < c.fwd_gathers.size(); ++i) {
    const auto& g = c.fwd_gathers[i];
    if (!contains(g.members, me)) continue;
    gathered = ctx.all_gather(g.members, L(p, "fwd", "all_gather", (int)i), mb,
                              Direction::Forward, need_src().payload);
    gathered_iv = p.dest_intervals[g.shard];
  }
  Payload delivered;
  for (size_t i = 0; i < c.fwd_delivers.size(); ++i) {
    const auto& st = c.fwd_delivers[i];
    if (!contains(st.group, me)) continue;
    Payload mine;
    if (st.root == me) {
      if (p.relation.kind == DpKind::FanIn)
        mine = rows_of(gathered, gathered_iv, st.interval, p.edge.feature_width);
      else
        mine = rows_of(need_src().payload, src->interval, st.interval, p.edge.feature_width);
    }
    Payload res = ctx.broadcast(st.group, st.root, L(p, "fwd", "deliver", (int)i), mb,
                                Direction::Forward, std::move(mine));
    if (in_dst) {
      auto it = c.fwd_actions.find(me);
      if (it != c.fwd_actions.end() && it->second.from == ColoSource::Deliver &&
          it->second.step == (int)i)
        delivered = std::move(res);
    }
  }
  if (!in_dst) return std::nullopt;
  const ColoAction& a = c.fwd_actions.at(me);
  ShardedTensor out{a.out, p.edge.feature_width, {}};
  switch (a.from) {
    case ColoSource::OwnShard:
      out.payload = rows_of(need_src().payload, src->interval, a.out, p.edge.feature_width);
      break;
    case ColoSource::Gather: out.payload = std::move(gathered); break;
    case ColoSource::Deliver: out.payload = std::move(delivered); break;
    default: raise(ErrorCode::PlanInfeasible, "bad forward action");
  }
  out.validate();
  return out;
}

std::optional<ShardedTensor> BridgeRuntime::backward_colocated(
    simnet::Rank& ctx, int mb, const std::optional<ShardedTensor>& grad) {
  const BridgePlan& p = *plan_;
  if (p.placement != grid::Placement::Colocated)
    raise(ErrorCode::NotColocated, "backward_colocated on a non-colocated plan");
  const ColoPlan& c = p.colo;
  const int me = ctx.id();
  const auto Rs = grid::ranks_of_stage(p.edge.source, p.edge.source.pp - 1);
  const auto Rd = grid::ranks_of_stage(p.edge.dest, 0);
  const bool in_src = contains(Rs, me), in_dst = contains(Rd, me);
  BatchInterval held_iv{};
  if (grad) {
    if (!in_dst) raise(ErrorCode::GradIntervalMismatch, "rank holds no destination shard slot");
    held_iv = p.dest_intervals[dst_shard_checked(p, me)];
    check_shard(p, *grad, held_iv, ErrorCode::GradIntervalMismatch);
  }
  consume_forward(mb);
  Payload held;
  if (grad) held = grad->payload;
  auto need_grad = [&]() {
    if (!grad) raise(ErrorCode::GradIntervalMismatch, "rank " + std::to_string(me) + " needs its gradient");
  };
  for (size_t i = 0; i < c.bwd_reduces.size(); ++i) {
    const auto& rs = c.bwd_reduces[i];
    if (!contains(rs.group, me)) continue;
    need_grad();
    held = ctx.all_reduce(rs.group, L(p, "bwd", "all_reduce", (int)i), mb, Direction::Backward,
                          std::move(held));
  }
  Payload gathered;
  BatchInterval gathered_iv{};
  for (size_t i = 0; i < c.bwd_gathers.size(); ++i) {
    const auto& g = c.bwd_gathers[i];
    if (!contains(g.members, me)) continue;
    need_grad();
    gathered = ctx.all_gather(g.members, L(p, "bwd", "all_gather", (int)i), mb,
                              Direction::Backward, held);
    gathered_iv = p.src_intervals[g.shard];
  }
  Payload delivered;
  for (size_t i = 0; i < c.bwd_delivers.size(); ++i) {
    const auto& st = c.bwd_delivers[i];
    if (!contains(st.group, me)) continue;
    Payload mine;
    if (st.root == me) {
      if (p.relation.kind == DpKind::FanOut)
        mine = rows_of(gathered, gathered_iv, st.interval, p.edge.feature_width);
      else {
        need_grad();
        mine = rows_of(held, held_iv, st.interval, p.edge.feature_width);
      }
    }
    Payload res = ctx.broadcast(st.group, st.root, L(p, "bwd", "deliver", (int)i), mb,
                                Direction::Backward, std::move(mine));
    if (in_src) {
      auto it = c.bwd_actions.find(me);
      if (it != c.bwd_actions.end() && it->second.from == ColoSource::Deliver &&
          it->second.step == (int)i)
        delivered = std::move(res);
    }
  }
  if (!in_src) return std::nullopt;
  const ColoAction& a = c.bwd_actions.at(me);
  ShardedTensor out{a.out, p.edge.feature_width, {}};
  switch (a.from) {
    case ColoSource::OwnGrad:
      need_grad();
      out.payload = rows_of(held, held_iv, a.out, p.edge.feature_width);
      break;
    case ColoSource::Gather: out.payload = std::move(gathered); break;
    case ColoSource::Deliver: out.payload = std::move(delivered); break;
    default: raise(ErrorCode::PlanInfeasible, "bad backward action");
  }
  out.validate();
  return out;
}

// --- whole-edge entry points (bridge.hpp:175-185) ------------------------------

namespace {
int world_for(const BridgePlan& p) {
  return std::max(p.edge.source.rank_end(), p.edge.dest.rank_end());
}
}  // namespace

std::map<int, ShardedTensor> bridge_forward(const BridgePlan& plan,
                                            const std::map<int, ShardedTensor>& shards,
                                            int mb, simnet::TrafficLedger* ledger_out) {
  const auto Rs = grid::ranks_of_stage(plan.edge.source, plan.edge.source.pp - 1);
  const auto Rd = grid::ranks_of_stage(plan.edge.dest, 0);
  for (const auto& [r, t] : shards)
    if (!contains(Rs, r))
      raise(ErrorCode::ShardIntervalMismatch, "shard given for non-source rank " + std::to_string(r));
  simnet::World w(world_for(plan));
  std::map<int, ShardedTensor> out;
  std::vector<BridgeRuntime> rt(w.size(), BridgeRuntime(plan));
  if (plan.placement == grid::Placement::NonColocated) {
    for (const auto& s : plan.nc.src_shards)
      if (!shards.count(s.src_leader))
        raise(ErrorCode::MissingSourceShard, "source leader r" + std::to_string(s.src_leader) +
                                                 " has no shard");
    for (int r : Rs) {
      auto it = shards.find(r);
      if (it == shards.end()) continue;
      w.set_script(r, [&, r](simnet::Rank& ctx) { rt[r].forward_source(ctx, mb, shards.at(r)); });
    }
    for (int r : Rd)
      w.set_script(r, [&, r](simnet::Rank& ctx) { out[r] = rt[r].forward_dest(ctx, mb); });
  } else {
    std::vector<int> all = Rs;
    for (int r : Rd)
      if (!contains(all, r)) all.push_back(r);
    for (int r : all) {
      w.set_script(r, [&, r](simnet::Rank& ctx) {
        std::optional<ShardedTensor> in;
        auto it = shards.find(r);
        if (it != shards.end()) in = it->second;
        auto res = rt[r].forward_colocated(ctx, mb, in);
        if (res) out[r] = std::move(*res);
      });
    }
  }
  w.run();
  if (ledger_out) *ledger_out = w.ledger();
  return out;
}

std::map<int, ShardedTensor> bridge_backward(const BridgePlan& plan,
                                             const std::map<int, ShardedTensor>& grads,
                                             int mb, simnet::TrafficLedger* ledger_out) {
  const auto Rs = grid::ranks_of_stage(plan.edge.source, plan.edge.source.pp - 1);
  const auto Rd = grid::ranks_of_stage(plan.edge.dest, 0);
  for (const auto& [r, t] : grads)
    if (!contains(Rd, r))
      raise(ErrorCode::GradIntervalMismatch, "gradient given for non-destination rank " + std::to_string(r));
  simnet::World w(world_for(plan));
  std::map<int, ShardedTensor> out;
  std::vector<BridgeRuntime> rt(w.size(), BridgeRuntime(plan));
  for (auto& r : rt) r.seed_forward_record(mb);
  if (plan.placement == grid::Placement::NonColocated) {
    for (int r : Rd) {
      if (!grads.count(r))
        raise(ErrorCode::GradIntervalMismatch, "missing gradient for destination rank " + std::to_string(r));
      w.set_script(r, [&, r](simnet::Rank& ctx) { rt[r].backward_dest(ctx, mb, grads.at(r)); });
    }
    for (int r : Rs)
      w.set_script(r, [&, r](simnet::Rank& ctx) { out[r] = rt[r].backward_source(ctx, mb); });
  } else {
    std::vector<int> all = Rs;
    for (int r : Rd)
      if (!contains(all, r)) all.push_back(r);
    for (int r : all) {
      w.set_script(r, [&, r](simnet::Rank& ctx) {
        std::optional<ShardedTensor> in;
        auto it = grads.find(r);
        if (it != grads.end()) in = it->second;
        auto res = rt[r].backward_colocated(ctx, mb, in);
        if (res) out[r] = std::move(*res);
      });
    }
  }
  w.run();
  if (ledger_out) *ledger_out = w.ledger();
  return out;
}

}  // namespace hetsim::bridge
