// hetbridge — layout algebra. Behaviour follows the reference contract
// (grid.hpp:13-94 / SPEC.md:60-108); checked against the reference library by
// tests/test_grid.py and against the reference's own test_grid.cpp KATs.
#include "hb/grid.hpp"

#include <algorithm>

namespace hb {

const char* error_code_name(ErrorCode code) {
  static const char* const kNames[] = {
      "RankOutOfModule",    "CoordOutOfBounds",      "IndivisibleBatch",      "PartialOverlap",
      "NonIntegerFan",      "PlanInfeasible",        "ShardIntervalMismatch", "MissingSourceShard",
      "GradIntervalMismatch", "UnknownMicrobatch",   "Deadlock",              "GroupMismatch",
      "ShapeMismatch",      "ChannelMismatch",       "SnapshotWhileActive",   "DivisibilityViolation",
      "CyclicGraph",        "DanglingEdge",          "InfeasibleSchedule",    "NotColocated",
      "StructureMismatch",  "ParseError",            "ValidationError",       "InvalidArgument",
      "CudaError",          "Timeout"};
  const int i = static_cast<int>(code);
  return (i >= 0 && i < static_cast<int>(sizeof(kNames) / sizeof(kNames[0]))) ? kNames[i]
                                                                              : "UnknownError";
}

namespace grid {

namespace {
std::string range_str(int b, int e) {
  return "[" + std::to_string(b) + ", " + std::to_string(e) + ")";
}
}  // namespace

void ModuleLayout::validate() const {
  if (std::min({tp, cp, pp, dp}) < 1)
    raise(ErrorCode::InvalidArgument, "module '" + name + "' has a parallel size < 1");
  if (rank_offset < 0)
    raise(ErrorCode::InvalidArgument, "module '" + name + "' has negative rank_offset");
}

GridCoord coord_of_rank(const ModuleLayout& l, int rank) {
  l.validate();
  if (!l.contains(rank))
    raise(ErrorCode::RankOutOfModule, "rank " + std::to_string(rank) + " outside module '" +
                                          l.name + "' ranks " +
                                          range_str(l.rank_begin(), l.rank_end()));
  // Mixed-radix digits of the module-local index, least significant first.
  const int lin = rank - l.rank_offset;
  const int tc = l.tp * l.cp, tcd = tc * l.dp;
  return GridCoord{lin % l.tp, (lin / l.tp) % l.cp, lin / tcd, (lin / tc) % l.dp};
}

int rank_of_coord(const ModuleLayout& l, const GridCoord& c) {
  l.validate();
  const bool ok = c.tp_idx >= 0 && c.tp_idx < l.tp && c.cp_idx >= 0 && c.cp_idx < l.cp &&
                  c.pp_idx >= 0 && c.pp_idx < l.pp && c.dp_idx >= 0 && c.dp_idx < l.dp;
  if (!ok) raise(ErrorCode::CoordOutOfBounds, "coordinate outside module '" + l.name + "' grid");
  return l.rank_offset + c.tp_idx + l.tp * (c.cp_idx + l.cp * (c.dp_idx + l.dp * c.pp_idx));
}

std::vector<BatchInterval> partition_batch(int batch, int dp) {
  if (dp < 1) raise(ErrorCode::InvalidArgument, "dp must be >= 1");
  if (batch <= 0 || batch % dp)
    raise(ErrorCode::IndivisibleBatch,
          "batch " + std::to_string(batch) + " not divisible by dp " + std::to_string(dp));
  std::vector<BatchInterval> v(dp);
  const int n = batch / dp;
  for (int i = 0; i < dp; ++i) v[i] = {i * n, n};
  return v;
}

int leader_rank(const ModuleLayout& l, int pp_idx, int dp_idx) {
  return rank_of_coord(l, GridCoord{0, 0, pp_idx, dp_idx});
}

Placement placement_of_edge(const BoundaryEdge& e) {
  e.source.validate();
  e.dest.validate();
  const int sb = e.source.rank_begin(), se = e.source.rank_end();
  const int db = e.dest.rank_begin(), de = e.dest.rank_end();
  if (sb == db && se == de) return Placement::Colocated;
  if (se <= db || de <= sb) return Placement::NonColocated;
  raise(ErrorCode::PartialOverlap, "modules '" + e.source.name + "' " + range_str(sb, se) +
                                       " and '" + e.dest.name + "' " + range_str(db, de) +
                                       " overlap without being identical");
}

std::vector<int> ranks_of_stage(const ModuleLayout& l, int pp_idx) {
  // Stage pp occupies one contiguous block of tp*cp*dp ranks under the fixed order.
  const int n = l.tp * l.cp * l.dp;
  const int first = rank_of_coord(l, GridCoord{0, 0, pp_idx, 0});
  std::vector<int> v(n);
  for (int i = 0; i < n; ++i) v[i] = first + i;
  return v;
}

std::vector<int> replica_group(const ModuleLayout& l, int pp_idx, int dp_idx) {
  const int n = l.tp * l.cp;
  const int first = leader_rank(l, pp_idx, dp_idx);
  std::vector<int> v(n);
  for (int i = 0; i < n; ++i) v[i] = first + i;
  return v;
}

std::vector<int> module_group(const ModuleLayout& l, int rank, GroupKind kind) {
  const GridCoord c = coord_of_rank(l, rank);
  const int n = kind == GroupKind::TP ? l.tp : kind == GroupKind::CP ? l.cp : kind == GroupKind::PP ? l.pp : l.dp;
  std::vector<int> v;
  v.reserve(n);
  for (int i = 0; i < n; ++i) {
    GridCoord x = c;
    (kind == GroupKind::TP ? x.tp_idx : kind == GroupKind::CP ? x.cp_idx : kind == GroupKind::PP ? x.pp_idx : x.dp_idx) = i;
    v.push_back(rank_of_coord(l, x));
  }
  std::sort(v.begin(), v.end());
  return v;
}

std::string to_string(const BatchInterval& iv) {
  return "[" + std::to_string(iv.start) + "," + std::to_string(iv.end()) + ")";
}

}  // namespace grid
}  // namespace hb
