// hetbridge — plan compilation (bridge.hpp:137-142 of the reference; contract
// SPEC.md:140-148, non-colocated routing P:276-301, colocated reinterpretation
// P:323-332, reference-silent choices fixed in SURVEY App. A).
//
// Pure host integer code: deterministic and identical on every rank that
// computes it, so each process compiles its own copy.
#include <algorithm>
#include <sstream>

#include "hb/bridge.hpp"

namespace hb::bridge {

using grid::BatchInterval;
using grid::GridCoord;
using grid::ModuleLayout;

const char* dp_kind_name(DpKind k) {
  return k == DpKind::Equal ? "Equal" : k == DpKind::FanIn ? "FanIn" : "FanOut";
}

DpRelation classify_dp_relation(const grid::BoundaryEdge& e) {
  e.source.validate();
  e.dest.validate();
  const int u = e.source.dp, v = e.dest.dp;
  const int hi = std::max(u, v), lo = std::min(u, v);
  if (hi % lo)
    raise(ErrorCode::NonIntegerFan,
          "dp " + std::to_string(u) + " -> " + std::to_string(v) + " is not an integer fan");
  if (u == v) return {DpKind::Equal, 1};
  return {u > v ? DpKind::FanIn : DpKind::FanOut, hi / lo};
}

int BridgePlan::cross_boundary_messages() const {
  int n = 0;
  if (placement == grid::Placement::NonColocated)
    for (const auto& r : nc.routes) n += static_cast<int>(r.pieces.size());
  return n;
}

std::vector<int> BridgePlan::source_stage_ranks() const {
  return grid::ranks_of_stage(edge.source, edge.source.pp - 1);
}
std::vector<int> BridgePlan::dest_stage_ranks() const { return grid::ranks_of_stage(edge.dest, 0); }

int BridgePlan::source_shard_of(int r) const {
  if (!edge.source.contains(r)) return -1;
  const auto c = grid::coord_of_rank(edge.source, r);
  return c.pp_idx == edge.source.pp - 1 ? c.dp_idx : -1;
}
int BridgePlan::dest_shard_of(int r) const {
  if (!edge.dest.contains(r)) return -1;
  const auto c = grid::coord_of_rank(edge.dest, r);
  return c.pp_idx == 0 ? c.dp_idx : -1;
}

namespace {

// Ranks holding DI[d] after the backward cp reduction, in holder-position
// order: the tp=0 rank of each cp slice if cp>1, otherwise each tp replica.
std::vector<int> grad_holders(const ModuleLayout& dst, int d) {
  std::vector<int> h;
  const bool by_cp = dst.cp > 1;
  const int n = by_cp ? dst.cp : dst.tp;
  for (int i = 0; i < n; ++i)
    h.push_back(grid::rank_of_coord(dst, by_cp ? GridCoord{0, i, 0, d} : GridCoord{i, 0, 0, d}));
  return h;
}

std::vector<ReduceStep> cp_reduce_steps(const ModuleLayout& dst) {
  std::vector<ReduceStep> v;
  if (dst.cp <= 1) return v;
  for (int d = 0; d < dst.dp; ++d) {
    ReduceStep s{grad_holders(dst, d), d};
    std::sort(s.group.begin(), s.group.end());
    v.push_back(std::move(s));
  }
  return v;
}

bool has(const std::vector<int>& v, int x) { return std::find(v.begin(), v.end(), x) != v.end(); }

int gather_step_of(const std::vector<GatherStep>& steps, int shard, int rank) {
  for (size_t i = 0; i < steps.size(); ++i)
    if (steps[i].shard == shard && has(steps[i].members, rank)) return static_cast<int>(i);
  return -1;
}

// Builds one direction of a colocated plan. `out_shards` are the intervals the
// receiving side materialises; `cover[x]` the ranks whose data covers
// out_shards[x] after gathers; `own(r, x)` says whether rank r covers x from
// data it already holds (OwnShard / OwnGrad).
template <class OwnFn>
void finish_colocated(const std::vector<int>& receivers, const std::vector<int>& shard_of,
                      const std::vector<BatchInterval>& out_iv,
                      const std::vector<std::vector<int>>& cover,
                      const std::vector<GatherStep>& gathers, ColoSource own_kind,
                      OwnFn own_parent, std::vector<DeliverStep>* delivers,
                      std::map<int, ColoAction>* actions) {
  std::vector<std::vector<int>> wanting(out_iv.size());
  for (size_t i = 0; i < receivers.size(); ++i) {
    const int r = receivers[i], x = shard_of[i];
    const int g = gather_step_of(gathers, x, r);
    BatchInterval parent;
    if (g >= 0) {
      (*actions)[r] = {ColoSource::Gather, g, out_iv[x], out_iv[x]};
    } else if (own_parent(r, x, &parent)) {
      (*actions)[r] = {own_kind, -1, parent, out_iv[x]};
    } else {
      wanting[x].push_back(r);
    }
  }
  for (size_t x = 0; x < out_iv.size(); ++x) {
    if (wanting[x].empty()) continue;
    DeliverStep st;
    st.root = *std::min_element(cover[x].begin(), cover[x].end());
    st.group = {st.root};
    st.group.insert(st.group.end(), wanting[x].begin(), wanting[x].end());
    st.shard = static_cast<int>(x);
    st.interval = out_iv[x];
    for (int r : wanting[x])
      (*actions)[r] = {ColoSource::Deliver, static_cast<int>(delivers->size()), out_iv[x], out_iv[x]};
    delivers->push_back(std::move(st));
  }
}

}  // namespace

BridgePlan plan_bridge(const grid::BoundaryEdge& edge) {
  BridgePlan p;
  p.edge = edge;
  p.placement = grid::placement_of_edge(edge);
  p.relation = classify_dp_relation(edge);
  if (edge.feature_width < 1) raise(ErrorCode::InvalidArgument, "feature_width must be >= 1");
  p.src_intervals = grid::partition_batch(edge.global_batch, edge.source.dp);
  p.dest_intervals = grid::partition_batch(edge.global_batch, edge.dest.dp);
  p.label = edge.source.name + "->" + edge.dest.name;

  const ModuleLayout& S = edge.source;
  const ModuleLayout& D = edge.dest;
  const int last = S.pp - 1;
  const auto& SI = p.src_intervals;
  const auto& DI = p.dest_intervals;
  const DpKind kind = p.relation.kind;
  const int k = p.relation.factor;

  if (p.placement == grid::Placement::NonColocated) {
    // Leaders carry every cross-boundary transfer; ceil-free because both dp
    // divide B, so SI[s] ∩ DI[d] is empty or one whole interval.
    for (int d = 0; d < D.dp; ++d) {
      NcRoute r{d, grid::leader_rank(D, 0, d), {}, grid::replica_group(D, 0, d)};
      for (int s = 0; s < S.dp; ++s) {
        const int b = std::max(SI[s].start, DI[d].start), e = std::min(SI[s].end(), DI[d].end());
        if (b < e) r.pieces.emplace_back(grid::leader_rank(S, last, s), BatchInterval{b, e - b});
      }
      p.nc.routes.push_back(std::move(r));
    }
    for (int s = 0; s < S.dp; ++s)
      p.nc.src_shards.push_back({s, grid::leader_rank(S, last, s), SI[s], grid::replica_group(S, last, s)});
    p.nc.reduces = cp_reduce_steps(D);
    return p;
  }

  ColoPlan& c = p.colo;
  const auto Rs = p.source_stage_ranks();
  const auto Rd = p.dest_stage_ranks();
  std::vector<int> rs_shard, rd_shard;
  for (int r : Rs) rs_shard.push_back(p.source_shard_of(r));
  for (int r : Rd) rd_shard.push_back(p.dest_shard_of(r));

  // Forward: fan-in all-gathers k consecutive source shards per replica position.
  std::vector<std::vector<int>> fcover(D.dp);
  if (kind == DpKind::FanIn) {
    for (int d = 0; d < D.dp; ++d)
      for (int j = 0; j < S.tp * S.cp; ++j) {
        GatherStep g;
        g.shard = d;
        for (int s = k * d; s < k * (d + 1); ++s) {
          g.members.push_back(grid::rank_of_coord(S, {j % S.tp, j / S.tp, last, s}));
          g.member_intervals.push_back(SI[s]);
        }
        fcover[d].insert(fcover[d].end(), g.members.begin(), g.members.end());
        c.fwd_gathers.push_back(std::move(g));
      }
  } else {
    for (size_t i = 0; i < Rs.size(); ++i)
      for (int d = 0; d < D.dp; ++d)
        if (SI[rs_shard[i]].contains(DI[d])) fcover[d].push_back(Rs[i]);
  }
  finish_colocated(
      Rd, rd_shard, DI, fcover, c.fwd_gathers, ColoSource::OwnShard,
      [&](int r, int d, BatchInterval* parent) {
        if (kind == DpKind::FanIn || !has(Rs, r)) return false;
        const auto& iv = SI[p.source_shard_of(r)];
        if (!iv.contains(DI[d])) return false;
        *parent = iv;
        return true;
      },
      &c.fwd_delivers, &c.fwd_actions);

  // Backward: cp reduction first, then fan-out all-gathers sibling gradients.
  c.bwd_reduces = cp_reduce_steps(D);
  std::vector<std::vector<int>> bcover(S.dp);
  auto dshard_for = [&](int s) { return kind == DpKind::FanIn ? s / k : s; };
  if (kind == DpKind::FanOut) {
    const int H = static_cast<int>(grad_holders(D, 0).size());
    for (int s = 0; s < S.dp; ++s)
      for (int h = 0; h < H; ++h) {
        GatherStep g;
        g.shard = s;
        for (int d = k * s; d < k * (s + 1); ++d) {
          g.members.push_back(grad_holders(D, d)[h]);
          g.member_intervals.push_back(DI[d]);
        }
        bcover[s].insert(bcover[s].end(), g.members.begin(), g.members.end());
        c.bwd_gathers.push_back(std::move(g));
      }
  } else {
    for (int s = 0; s < S.dp; ++s) bcover[s] = grad_holders(D, dshard_for(s));
  }
  finish_colocated(
      Rs, rs_shard, SI, bcover, c.bwd_gathers, ColoSource::OwnGrad,
      [&](int r, int s, BatchInterval* parent) {
        if (kind == DpKind::FanOut) return false;
        const int d = dshard_for(s);
        if (!has(grad_holders(D, d), r)) return false;
        *parent = DI[d];
        return true;
      },
      &c.bwd_delivers, &c.bwd_actions);
  return p;
}

std::string export_plan(const BridgePlan& p, int elem_bytes) {
  std::ostringstream os;
  const long W = p.edge.feature_width, E = elem_bytes;
  auto B = [&](const BatchInterval& iv) { return static_cast<long>(iv.length) * W * E; };
  auto G = [](const std::vector<int>& g) {
    std::string s;
    for (size_t i = 0; i < g.size(); ++i) s += (i ? "," : "") + std::to_string(g[i]);
    return "[" + s + "]";
  };
  auto iv = [](const BatchInterval& x) { return grid::to_string(x); };
  const bool colo = p.placement == grid::Placement::Colocated;
  os << "edge " << p.label << " placement=" << (colo ? "Colocated" : "NonColocated")
     << " relation=" << dp_kind_name(p.relation.kind) << " k=" << p.relation.factor
     << " batch=" << p.edge.global_batch << " width=" << W << " elem_bytes=" << E << "\n";
  auto reduce_lines = [&](const std::vector<ReduceStep>& v) {
    for (const auto& r : v) {
      const long n = static_cast<long>(r.group.size());
      os << "bwd all_reduce group=" << G(r.group) << " " << iv(p.dest_intervals[r.dest_shard])
         << " bytes=" << B(p.dest_intervals[r.dest_shard]) * n * (n - 1) << "\n";
    }
  };
  if (!colo) {
    for (const auto& r : p.nc.routes) {
      for (const auto& [l, x] : r.pieces)
        os << "fwd send r" << l << " -> r" << r.dest_leader << " " << iv(x) << " bytes=" << B(x) << "\n";
      if (r.bcast_group.size() > 1)
        os << "fwd broadcast root=r" << r.dest_leader << " group=" << G(r.bcast_group) << " "
           << iv(p.dest_intervals[r.dest_shard]) << " bytes="
           << B(p.dest_intervals[r.dest_shard]) * static_cast<long>(r.bcast_group.size() - 1) << "\n";
    }
    reduce_lines(p.nc.reduces);
    for (const auto& r : p.nc.routes)
      for (const auto& [l, x] : r.pieces)
        os << "bwd send r" << r.dest_leader << " -> r" << l << " " << iv(x) << " bytes=" << B(x) << "\n";
    for (const auto& s : p.nc.src_shards)
      if (s.bcast_group.size() > 1)
        os << "bwd broadcast root=r" << s.src_leader << " group=" << G(s.bcast_group) << " "
           << iv(s.interval) << " bytes=" << B(s.interval) * static_cast<long>(s.bcast_group.size() - 1)
           << "\n";
    return os.str();
  }
  const ColoPlan& c = p.colo;
  auto gathers = [&](const char* dir, const std::vector<GatherStep>& v,
                     const std::vector<BatchInterval>& whole) {
    for (const auto& g : v) {
      os << dir << " all_gather group=" << G(g.members) << " parts=";
      for (size_t i = 0; i < g.member_intervals.size(); ++i)
        os << (i ? "+" : "") << iv(g.member_intervals[i]);
      os << " " << iv(whole[g.shard])
         << " bytes=" << B(whole[g.shard]) * static_cast<long>(g.members.size() - 1) << "\n";
    }
  };
  auto delivers = [&](const char* dir, const std::vector<DeliverStep>& v) {
    for (const auto& s : v)
      os << dir << " deliver root=r" << s.root << " group=" << G(s.group) << " " << iv(s.interval)
         << " bytes=" << B(s.interval) * static_cast<long>(s.group.size() - 1) << "\n";
  };
  auto selects = [&](const char* dir, const std::map<int, ColoAction>& acts) {
    for (const auto& [r, a] : acts)
      if (a.from == ColoSource::OwnShard || a.from == ColoSource::OwnGrad)
        os << dir << " select r" << r << " " << iv(a.parent) << " -> " << iv(a.out) << " bytes=0\n";
  };
  gathers("fwd", c.fwd_gathers, p.dest_intervals);
  delivers("fwd", c.fwd_delivers);
  selects("fwd", c.fwd_actions);
  reduce_lines(c.bwd_reduces);
  gathers("bwd", c.bwd_gathers, p.src_intervals);
  delivers("bwd", c.bwd_delivers);
  selects("bwd", c.bwd_actions);
  return os.str();
}

}  // namespace hb::bridge
