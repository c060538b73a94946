// hetbridge — graph-aware pipeline dispatch over the PP-stage graph
// (SPEC.md:358-437 `sched`: build_stage_graph,
// generate_1f1b_dispatch, validate_dispatch; PAPER.md:374-395 and the
// Appendix D dispatch figure). The reference's sched.cpp is an
// empty stub; the types and operations follow the SPEC module.
//
// The table drives the device runtime (runtime_host.hpp): P2P cells are the
// LLM's / encoders' own pipeline sends (NCCL), NC cells are boundary
// forward/backward ops of the edge's Exec on the boundary stream.
#pragma once

#include <string>
#include <vector>

#include "hb/grid.hpp"

namespace hb::sched {

enum class EdgeKind { P2P = 0, NC = 1 };

struct StageNode {
  int module = 0;    // index into the module list
  int pp = 0;        // pipeline stage of that module
  int distance = 0;  // longest path (in edges) to the sink
  std::string name;  // "<module>P<pp>"
};

struct StageEdge {
  int src = 0, dst = 0;  // node indices
  EdgeKind kind = EdgeKind::P2P;
  int boundary = -1;     // NC: index into the declared module edges (the BridgePlan identity)
};

// SPEC `StageGraph`: nodes (module, pp_idx); intra-module chain edges; one
// boundary edge from each source module's last stage to each destination
// module's first stage. Acyclic, single sink.
struct StageGraph {
  std::vector<grid::ModuleLayout> modules;
  std::vector<std::pair<int, int>> module_edges;  // (source module, dest module) as declared
  std::vector<StageNode> nodes;
  std::vector<StageEdge> edges;
  int sink = -1;
  std::vector<int> in_edges(int node) const;   // ascending edge index (declared order)
  std::vector<int> out_edges(int node) const;
  int node_of(int module, int pp) const;
};

// build_stage_graph(modules, edges): CyclicGraph when the module graph has a
// cycle, DanglingEdge when an edge names an undeclared module (or a self
// edge), InfeasibleSchedule when the graph has several sinks.
StageGraph build_stage_graph(const std::vector<grid::ModuleLayout>& modules,
                             const std::vector<std::pair<int, int>>& module_edges);

enum class Op { Compute = 0, SendFwd = 1, RecvFwd = 2, SendBwd = 3, RecvBwd = 4 };

// One dispatch-table cell entry: at schedule call `row`, node `node` runs `op`
// for microbatch `mb` (Compute: forward when !bwd); communication entries name
// the stage edge and its kind (P2P intra-module, NC across a boundary).
struct Cell {
  int row = 0;
  int node = 0;
  Op op = Op::Compute;
  int edge = -1;
  EdgeKind kind = EdgeKind::P2P;
  int mb = 0;
  bool bwd = false;
};

struct DispatchTable {
  int rows = 0;
  int nmb = 0;
  std::vector<Cell> cells;  // ordered by row, then node, then op order within the call
};

// generate_1f1b_dispatch: node n warms up with min(distance(n), nmb)
// forwards, then pairs one forward with one backward per call, then drains.
// A call computes at most one microbatch per node; the sends it produces and
// the matching receives sit in the same row (a schedule call is one exchange
// step), so executing the rows in order never waits on a later row.
// InfeasibleSchedule if nmb < 1.
DispatchTable generate_1f1b_dispatch(const StageGraph& g, int nmb);

// validate_dispatch: (a) join readiness — Compute F(mb) of a node is preceded
// by RecvFwd(mb) on every incoming edge (and B(mb) by RecvBwd(mb) on every
// outgoing edge); (b) edge identity — SendBwd(e, mb) reverses a forward edge
// e that delivered mb to that node, RecvBwd(e, mb) reverses one it sent mb on;
// (c) no double consumption and completeness — each (edge, mb) moves exactly
// once forward and once backward, sends and receives paired in one row, cell
// kinds matching the graph. Returns the violations (never throws).
std::vector<std::string> validate_dispatch(const StageGraph& g, const std::vector<Cell>& cells, int nmb);

// nc_issue_order: the NC cells of `node` in the order its boundary stream
// executes them — by row, then by module edge (the BridgePlan identity), then
// forward before backward. A boundary op is a rendezvous of its endpoints'
// kernels (the in-kernel "started" barrier), and both endpoints see it in the
// same row, so with this order every GPU's boundary stream is a linear
// extension of one global order (row, edge, direction) and every rendezvous
// is met. The table's own within-row order is not enough: at a join the
// source may list F2 before B1 while the destination lists B1 before F2, and
// two serial streams waiting on each other deadlock.
std::vector<Cell> nc_issue_order(const StageGraph& g, const DispatchTable& t, int node);
bool nc_before(const StageGraph& g, const Cell& a, const Cell& b);

// Text grid (rows = schedule calls, columns = nodes): compute "F3"/"B3",
// communication "sf3:p2p", "rf3:NC", "sb3:NC", "rb3:p2p".
std::string render(const StageGraph& g, const DispatchTable& t);

const char* op_name(Op op);

}  // namespace hb::sched
