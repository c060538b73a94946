// hetbridge — ownership index builder (see index_map.hpp).
#include "hb/index_map.hpp"

#include <algorithm>

namespace hb::index {

using bridge::BridgePlan;
using bridge::ColoSource;
using bridge::DpKind;
using grid::BatchInterval;

namespace {

bool colocated(const BridgePlan& p) { return p.placement == grid::Placement::Colocated; }

// Member of a gather step whose interval holds sample j.
RowRef gather_member(const bridge::GatherStep& g, int j) {
  for (size_t i = 0; i < g.members.size(); ++i) {
    const auto& iv = g.member_intervals[i];
    if (j >= iv.start && j < iv.end()) return {g.members[i], j - iv.start};
  }
  raise(ErrorCode::PlanInfeasible, "sample " + std::to_string(j) + " not in gather step");
}

int step_holding(const std::vector<bridge::GatherStep>& steps, int shard, int rank) {
  for (size_t i = 0; i < steps.size(); ++i)
    if (steps[i].shard == shard &&
        std::find(steps[i].members.begin(), steps[i].members.end(), rank) != steps[i].members.end())
      return static_cast<int>(i);
  return -1;
}

// Destination gradient held by `h` for sample j after the backward cp
// reduction (all_reduce over the tp=0 group in ascending group order).
std::vector<RowRef> held_grad(const BridgePlan& p, int h, int j) {
  const int d = p.dest_shard_of(h);
  const BatchInterval& DI = p.dest_intervals[d];
  if (p.edge.dest.cp > 1) {
    const auto& steps = colocated(p) ? p.colo.bwd_reduces : p.nc.reduces;
    for (const auto& s : steps)
      if (s.dest_shard == d) {
        std::vector<RowRef> v;
        for (int g : s.group) v.push_back({g, j - DI.start});
        return v;
      }
    raise(ErrorCode::PlanInfeasible, "missing cp reduce step");
  }
  return {{h, j - DI.start}};
}

}  // namespace

RowRef forward_origin(const BridgePlan& p, int r, int j) {
  const int n_s = p.src_intervals[0].length;
  if (!colocated(p)) {
    const int s = j / n_s;
    return {p.nc.src_shards[s].src_leader, j - p.src_intervals[s].start};
  }
  const auto& a = p.colo.fwd_actions.at(r);
  auto own = [&](int rank) {
    const int s = p.source_shard_of(rank);
    return RowRef{rank, j - p.src_intervals[s].start};
  };
  switch (a.from) {
    case ColoSource::OwnShard: return own(r);
    case ColoSource::Gather: return gather_member(p.colo.fwd_gathers[a.step], j);
    case ColoSource::Deliver: {
      const auto& st = p.colo.fwd_delivers[a.step];
      if (p.relation.kind == DpKind::FanIn)
        return gather_member(p.colo.fwd_gathers[step_holding(p.colo.fwd_gathers, st.shard, st.root)], j);
      return own(st.root);
    }
    default: break;
  }
  raise(ErrorCode::PlanInfeasible, "bad forward action");
}

std::vector<RowRef> backward_origin(const BridgePlan& p, int r, int j) {
  const int n_d = p.dest_intervals[0].length;
  if (!colocated(p)) return held_grad(p, p.nc.routes[j / n_d].dest_leader, j);
  const auto& a = p.colo.bwd_actions.at(r);
  auto via_gather = [&](const bridge::GatherStep& g) {
    const RowRef m = gather_member(g, j);
    return held_grad(p, m.rank, j);
  };
  switch (a.from) {
    case ColoSource::OwnGrad: return held_grad(p, r, j);
    case ColoSource::Gather: return via_gather(p.colo.bwd_gathers[a.step]);
    case ColoSource::Deliver: {
      const auto& st = p.colo.bwd_delivers[a.step];
      if (p.relation.kind == DpKind::FanOut)
        return via_gather(p.colo.bwd_gathers[step_holding(p.colo.bwd_gathers, st.shard, st.root)]);
      return held_grad(p, st.root, j);
    }
    default: break;
  }
  raise(ErrorCode::PlanInfeasible, "bad backward action");
}

void SpliceSpec::validate(const BridgePlan& plan) const {
  if (Q < 1 || S < 1 || d_h < 1 || S_v < 1)
    raise(ErrorCode::InvalidArgument, "splice dimensions must be >= 1");
  if (static_cast<int64_t>(S_v) * d_h != plan.edge.feature_width)
    raise(ErrorCode::ShapeMismatch, "feature_width must equal S_v * d_h for a splice edge");
  if (S % plan.edge.dest.cp)
    raise(ErrorCode::DivisibilityViolation, "sequence length not divisible by destination cp");
  if (static_cast<int64_t>(codes.size()) != static_cast<int64_t>(Q) * S)
    raise(ErrorCode::ShapeMismatch, "placeholder table must have Q*S entries");
  const int64_t vis_rows = static_cast<int64_t>(plan.dest_intervals[0].length) * S_v;
  std::vector<char> seen(vis_rows, 0);
  for (int32_t c : codes) {
    if (c < 0) continue;
    if (c >= vis_rows) raise(ErrorCode::ShapeMismatch, "vision code beyond the destination shard");
    if (seen[c]++) raise(ErrorCode::InvalidArgument, "vision row placed at two positions");
  }
}

namespace {

// Append with coalescing: extend the previous segment when both sides continue.
void push_copy(std::vector<CopySeg>& v, const CopySeg& s) {
  if (!v.empty()) {
    CopySeg& b = v.back();
    if (b.dst.rank == s.dst.rank && b.dst.slot == s.dst.slot && b.dst.off + b.n == s.dst.off &&
        b.src.rank == s.src.rank && b.src.slot == s.src.slot && b.src.off + b.n == s.src.off) {
      b.n += s.n;
      return;
    }
  }
  v.push_back(s);
}

void push_reduce(std::vector<ReduceSeg>& v, ReduceSeg&& s) {
  if (!v.empty()) {
    ReduceSeg& b = v.back();
    bool ok = b.dst.rank == s.dst.rank && b.dst.slot == s.dst.slot && b.dst.off + b.n == s.dst.off &&
              b.terms.size() == s.terms.size();
    for (size_t i = 0; ok && i < s.terms.size(); ++i)
      ok = b.terms[i].rank == s.terms[i].rank && b.terms[i].slot == s.terms[i].slot &&
           b.terms[i].off + b.n == s.terms[i].off;
    if (ok) {
      b.n += s.n;
      return;
    }
  }
  v.push_back(std::move(s));
}

}  // namespace

namespace {

// Chooses which tensor-parallel replica of a gradient holder serves a term:
// the source rank itself when it is one of the replicas (no transfer), else
// the replica that has served the fewest elements so far (ties: lowest tp).
// Decided per (source sample, holder) so a sample's rows stay one run.
struct ReplicaChooser {
  const BridgePlan& p;
  std::vector<int64_t> load;
  int operator()(int h, int r, int64_t weight) {
    const auto& L = p.edge.dest;
    if (L.tp == 1) return h;
    grid::GridCoord c = grid::coord_of_rank(L, h);
    int best = -1;
    for (int k = 0; k < L.tp; ++k) {
      c.tp_idx = k;
      const int cand = grid::rank_of_coord(L, c);
      if (cand == r) {
        best = cand;
        break;
      }
      if (best < 0 || load[cand] < load[best]) best = cand;
    }
    load[best] += weight;
    return best;
  }
};

}  // namespace

IndexMap build_index_map(const BridgePlan& p, const SpliceSpec* sp, bool balance_replicas) {
  if (sp) sp->validate(p);
  IndexMap m;
  m.world = std::max(p.edge.source.rank_end(), p.edge.dest.rank_end());
  m.elems.assign(m.world, std::vector<int64_t>(kNumSlots, 0));
  const int64_t W = p.edge.feature_width;
  const auto Rs = p.source_stage_ranks();
  const auto Rd = p.dest_stage_ranks();
  for (int r : Rs) {
    const int64_t n = p.src_intervals[p.source_shard_of(r)].length * W;
    m.elems[r][kSrcAct] = n;
    m.elems[r][kSrcGrad] = n;
  }

  ReplicaChooser choose{p, std::vector<int64_t>(m.world, 0)};
  if (!sp) {
    for (int r : Rd) {
      const auto& DI = p.dest_intervals[p.dest_shard_of(r)];
      m.elems[r][kDstAct] = m.elems[r][kDstGrad] = DI.length * W;
      for (int j = DI.start; j < DI.end(); ++j) {
        const RowRef o = forward_origin(p, r, j);
        push_copy(m.fwd, {{o.rank, kSrcAct, o.row * W}, {r, kDstAct, (j - DI.start) * W}, W});
      }
    }
    for (int r : Rs) {
      const auto& SI = p.src_intervals[p.source_shard_of(r)];
      for (int j = SI.start; j < SI.end(); ++j) {
        ReduceSeg s{{r, kSrcGrad, (j - SI.start) * W}, W, {}};
        for (const RowRef& t : backward_origin(p, r, j))
          s.terms.push_back({balance_replicas ? choose(t.rank, r, W) : t.rank, kDstGrad, t.row * W});
        m.max_terms = std::max<int>(m.max_terms, s.terms.size());
        push_reduce(m.bwd, std::move(s));
      }
    }
    return m;
  }

  // ---- splice composition
  const int64_t dh = sp->d_h;
  const int cp = p.edge.dest.cp;
  const int L = sp->S / cp;
  const int n_d = p.dest_intervals[0].length;
  // Inverse placeholder table: vision row -> (q, p), -1 if not placed.
  std::vector<int64_t> pos_of(static_cast<int64_t>(n_d) * sp->S_v, -1);
  for (int64_t i = 0; i < static_cast<int64_t>(sp->codes.size()); ++i)
    if (sp->codes[i] >= 0) pos_of[sp->codes[i]] = i;

  for (int r : Rd) {
    const int d = p.dest_shard_of(r);
    const int c = grid::coord_of_rank(p.edge.dest, r).cp_idx;
    const int64_t base = static_cast<int64_t>(c) * L;
    m.elems[r][kDstAct] = m.elems[r][kDstGrad] = static_cast<int64_t>(sp->Q) * L * dh;
    int64_t text_k = 0, text_max = -1;
    for (int q = 0; q < sp->Q; ++q)
      for (int pos = 0; pos < L; ++pos) {
        const int32_t code = sp->codes[static_cast<int64_t>(q) * sp->S + base + pos];
        const Ref dst{r, kDstAct, (static_cast<int64_t>(q) * L + pos) * dh};
        if (code >= 0) {
          const int jl = code / sp->S_v, t = code % sp->S_v;
          const RowRef o = forward_origin(p, r, p.dest_intervals[d].start + jl);
          push_copy(m.fwd, {{o.rank, kSrcAct, o.row * W + t * dh}, dst, dh});
        } else if (sp->text_mode != TextMode::InPlace) {
          const int64_t row = sp->text_mode == TextMode::Slice ? text_k++ : (-1 - int64_t{code});
          text_max = std::max(text_max, row);
          push_copy(m.fwd, {{r, kText, row * dh}, dst, dh});
        }
      }
    m.elems[r][kText] = (text_max + 1) * dh;
  }
  for (int r : Rs) {
    const auto& SI = p.src_intervals[p.source_shard_of(r)];
    for (int j = SI.start; j < SI.end(); ++j) {
      auto origin = backward_origin(p, r, j);
      if (balance_replicas)
        for (RowRef& o : origin) {
          // weight: the rows of sample j that lie inside the holder's slice
          const int c = grid::coord_of_rank(p.edge.dest, o.rank).cp_idx;
          int64_t rows = 0;
          for (int t = 0; t < sp->S_v; ++t) {
            const int64_t at = pos_of[static_cast<int64_t>(o.row) * sp->S_v + t];
            const int pos = at < 0 ? -1 : static_cast<int>(at % sp->S);
            rows += pos >= c * L && pos < (c + 1) * L;
          }
          if (rows) o.rank = choose(o.rank, r, rows * dh);
        }
      for (int t = 0; t < sp->S_v; ++t) {
        ReduceSeg s{{r, kSrcGrad, (j - SI.start) * W + t * dh}, dh, {}};
        for (const RowRef& o : origin) {
          const int64_t at = pos_of[static_cast<int64_t>(o.row) * sp->S_v + t];
          if (at < 0) continue;  // never placed: zero gradient
          const int q = static_cast<int>(at / sp->S), pos = static_cast<int>(at % sp->S);
          const int c = grid::coord_of_rank(p.edge.dest, o.rank).cp_idx;
          if (pos < c * L || pos >= (c + 1) * L) continue;  // outside this rank's slice: zero
          s.terms.push_back({o.rank, kDstGrad, (static_cast<int64_t>(q) * L + pos - c * L) * dh});
        }
        m.max_terms = std::max<int>(m.max_terms, s.terms.size());
        push_reduce(m.bwd, std::move(s));
      }
    }
  }
  return m;
}

}  // namespace hb::index
