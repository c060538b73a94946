// hetbridge — boundary plan (drop-in for the plan half of hetsim::bridge,
// /root/reference/proj/core/include/hetsim/bridge.hpp:38-142).
//
// The plan structures keep the reference's names and fields so the routing a
// reference caller inspects (leaders, pieces, gather groups, deliver roots,
// per-rank actions) is the same object. Execution does not replay those steps
// hop by hop: index_map.hpp collapses every route to "which source element
// feeds which destination element" and the sm_100a kernels pull those bytes
// directly over NVSwitch (same bytes per consumer, no second
// hop). The ledger/export stay leader-based for parity with the reference.
#pragma once

#include <map>
#include <string>
#include <vector>

#include "hb/grid.hpp"

namespace hb::bridge {

enum class DpKind { Equal, FanIn, FanOut };

struct DpRelation {
  DpKind kind = DpKind::Equal;
  int factor = 1;
};

const char* dp_kind_name(DpKind k);

struct NcRoute {
  int dest_shard = 0;
  int dest_leader = 0;
  std::vector<std::pair<int, grid::BatchInterval>> pieces;  // (source leader, interval), batch order
  std::vector<int> bcast_group;
};

struct NcSrcShard {
  int src_shard = 0;
  int src_leader = 0;
  grid::BatchInterval interval;
  std::vector<int> bcast_group;
};

struct ReduceStep {
  std::vector<int> group;  // cp replicas at tp=0 of one destination shard
  int dest_shard = 0;
};

struct NcPlan {
  std::vector<NcRoute> routes;
  std::vector<NcSrcShard> src_shards;
  std::vector<ReduceStep> reduces;
};

struct GatherStep {
  std::vector<int> members;
  std::vector<grid::BatchInterval> member_intervals;
  int shard = 0;
};

struct DeliverStep {
  int root = 0;
  std::vector<int> group;
  int shard = 0;
  grid::BatchInterval interval;
};

enum class ColoSource { OwnShard, OwnGrad, Gather, Deliver };

struct ColoAction {
  ColoSource from = ColoSource::OwnShard;
  int step = -1;
  grid::BatchInterval parent;
  grid::BatchInterval out;
};

struct ColoPlan {
  std::vector<GatherStep> fwd_gathers;
  std::vector<DeliverStep> fwd_delivers;
  std::map<int, ColoAction> fwd_actions;
  std::vector<ReduceStep> bwd_reduces;
  std::vector<GatherStep> bwd_gathers;
  std::vector<DeliverStep> bwd_delivers;
  std::map<int, ColoAction> bwd_actions;
};

struct BridgePlan {
  grid::BoundaryEdge edge;
  grid::Placement placement = grid::Placement::NonColocated;
  DpRelation relation;
  std::string label;
  std::vector<grid::BatchInterval> src_intervals, dest_intervals;
  NcPlan nc;
  ColoPlan colo;

  int cross_boundary_messages() const;

  // Convenience views used by the index builder and runtime.
  std::vector<int> source_stage_ranks() const;  // ranks_of_stage(src, pp_s-1)
  std::vector<int> dest_stage_ranks() const;    // ranks_of_stage(dst, 0)
  int source_shard_of(int rank) const;          // -1 if not on the source boundary stage
  int dest_shard_of(int rank) const;            // -1 if not on destination stage 0
};

DpRelation classify_dp_relation(const grid::BoundaryEdge& edge);
BridgePlan plan_bridge(const grid::BoundaryEdge& edge);

/// One text line per transfer/collective. `elem_bytes`
/// scales byte counts; 8 reproduces the reference's 8-byte-real accounting
/// (simnet.hpp:27-29) and is text-identical to the oracle's export.
std::string export_plan(const BridgePlan& plan, int elem_bytes = 8);

}  // namespace hb::bridge
