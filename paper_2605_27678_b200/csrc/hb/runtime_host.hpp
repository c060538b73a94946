// hetbridge — host-owned per-module runtime.
//
// One HostRuntime per process (one GPU each) owns, for a set of modules with
// disjoint rank ranges (the non-colocated topology of PAPER.md Fig. 4(a)):
//   * the per-module rank groups of this rank (TP / CP / PP / DP, from the
//     reference's fixed rank order, grid.cpp:41-53, 87-106);
//   * one NCCL communicator over the world and, per module, a PP communicator
//     split from it (ncclCommSplit; color = the rank's (tp, cp, dp) cell) that
//     carries the module's own pipeline P2P;
//   * one boundary Exec per module edge (the NC communicator, set up
//     collectively: CUDA IPC handles all-gathered over NCCL);
//   * three streams: the boundary stream at the highest priority, a PP stream
//     and a compute stream, with boundary kernels capped at max_ctas CTAs so
//     pipeline P2P and compute keep SMs;
//   * the graph-aware 1F1B dispatch table of the stage graph (sched.hpp).
// step() executes this rank's column of the table: P2P cells as grouped NCCL
// send/recv on the PP stream, NC cells as the edge Exec's forward/backward on
// the boundary stream, compute cells through the caller's callback on the
// compute stream, ordered by CUDA events (RecvFwd(mb) -> F(mb) -> SendFwd(mb),
// RecvBwd(mb) -> B(mb) -> SendBwd(mb)). Nothing waits on the host.
#pragma once

#include <cuda_runtime.h>

#include <memory>
#include <vector>

#include "hb/runtime.hpp"
#include "hb/sched.hpp"

namespace hb::rt {

struct HostConfig {
  int nmb = 4;             // microbatches per step (the dispatch table's NMB)
  int max_ctas = 0;        // CTA cap of the boundary kernels (0: fill the GPU)
  int64_t pp_bytes = 0;    // bytes of one microbatch's stage activation / gradient per rank (P2P buffers)
  int act_dtype = dev::kBF16, grad_in_dtype = dev::kBF16, grad_out_dtype = dev::kFP32;
  double timeout_s = 20.0;
  // bit 0: skip NC cells, bit 1: skip P2P cells, bit 2: event-only compute
  // (no callback) — isolates one traffic class for overlap measurements
  int skip = 0;
};

// compute callback: node of the stage graph, microbatch, 1 = backward, the
// compute stream (cudaStream_t)
using ComputeFn = void (*)(void* user, int node, int mb, int bwd, void* stream);

class HostRuntime {
 public:
  HostRuntime(std::vector<grid::ModuleLayout> modules, std::vector<std::pair<int, int>> module_edges,
              int global_batch, int feature_width, int world, int my_rank, const void* nccl_id128,
              const HostConfig& cfg);
  ~HostRuntime();
  HostRuntime(const HostRuntime&) = delete;
  HostRuntime& operator=(const HostRuntime&) = delete;

  const sched::StageGraph& graph() const { return graph_; }
  const sched::DispatchTable& table() const { return table_; }
  int my_node() const { return node_; }  // -1: this rank holds no stage
  int my_module() const { return module_; }
  std::vector<int> group(int kind) const;  // grid::GroupKind of this rank's module
  Exec* edge_exec(int module_edge) const;
  // P2P stage buffers of this rank: 0 act_in (RecvFwd), 1 act_out (SendFwd),
  // 2 grad_in (RecvBwd), 3 grad_out (SendBwd); one per microbatch
  void* stage_buffer(int which, int mb, size_t* bytes) const;
  cudaStream_t stream(int which) const;  // 0 boundary, 1 PP, 2 compute

  // Enqueue one step (this rank's column of the table); returns at once.
  void step(ComputeFn fn, void* user);
  // Device time of the last step on this rank (compute-stream events around
  // it, joined with the other streams); synchronises.
  float last_step_ms();
  int64_t steps() const { return steps_; }
  // forward/backward boundary-op pairs issued as one paired call (all steps)
  int64_t paired_ops() const { return paired_ops_; }

 private:
  struct Nccl;
  std::unique_ptr<Nccl> nccl_;
  std::vector<grid::ModuleLayout> modules_;
  std::vector<std::pair<int, int>> module_edges_;
  sched::StageGraph graph_;
  sched::DispatchTable table_;
  HostConfig cfg_;
  int world_, rank_, node_ = -1, module_ = -1, device_ = 0;
  std::vector<std::unique_ptr<bridge::BridgePlan>> plans_;
  std::vector<std::unique_ptr<Exec>> execs_;
  cudaStream_t st_[3] = {nullptr, nullptr, nullptr};
  unsigned char* stage_mem_ = nullptr;
  size_t stage_bytes_ = 0;
  int prev_pp_ = -1, next_pp_ = -1;  // PP-comm ranks of this rank's neighbours (-1: none)
  std::vector<cudaEvent_t> ev_;        // per microbatch: fwd in, fwd done, bwd in, bwd done
  cudaEvent_t t0_ = nullptr, t1_ = nullptr;
  int64_t steps_ = 0;
  int64_t paired_ops_ = 0;
  cudaEvent_t& ev(int kind, int mb) { return ev_[kind * cfg_.nmb + mb]; }
};

// 128-byte NCCL unique id for hb_runtime_create (rank 0 makes it, the caller
// broadcasts it).
void nccl_unique_id(void* out128);

}  // namespace hb::rt
