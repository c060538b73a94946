// hetsim_bridge_hb.cpp — the reference-side binding a hetsim maintainer would
// add: hetsim::grid / hetsim::bridge call sites kept, the
// work done by hetbridge through its C-ABI (include/hetbridge.h). Built by
// oracle/Makefile (target `shimcheck`) against the reference's own headers.
#include "hetsim_bridge_hb.hpp"

#include <string>
#include <vector>

#include "hetbridge.h"

namespace hetsim_hb {
namespace {
void check(int st) {
  if (st) {
    char msg[512];
    hb_last_error(msg, sizeof msg);
    throw hetsim::SimError(static_cast<hetsim::ErrorCode>(st - 1), msg);
  }
}
hb_layout lay(const hetsim::grid::ModuleLayout& m) { return {m.name.c_str(), m.tp, m.cp, m.pp, m.dp, m.rank_offset}; }
hb_edge edge(const hetsim::grid::BoundaryEdge& e) { return {lay(e.source), lay(e.dest), e.global_batch, e.feature_width}; }
}  // namespace

// hetsim::bridge::export_plan(plan_bridge(e)), byte for byte
std::string export_plan(const hetsim::grid::BoundaryEdge& e) {
  hb_edge he = edge(e);
  hb_plan* p = nullptr;
  check(hb_plan_create(&he, &p));
  size_t n = 0;
  check(hb_plan_export(p, 8, nullptr, 0, &n));
  std::string s(n + 1, '\0');
  check(hb_plan_export(p, 8, s.data(), s.size(), &n));
  hb_plan_destroy(p);
  s.resize(n);
  return s;
}

// hetsim::bridge::classify_dp_relation(e)
hetsim::bridge::DpRelation classify_dp_relation(const hetsim::grid::BoundaryEdge& e) {
  hb_edge he = edge(e);
  int kind = 0, factor = 0;
  check(hb_classify_dp_relation(&he, &kind, &factor));
  return {static_cast<hetsim::bridge::DpKind>(kind), factor};
}

// hetsim::grid::placement_of_edge(e)
hetsim::grid::Placement placement_of_edge(const hetsim::grid::BoundaryEdge& e) {
  hb_edge he = edge(e);
  int pl = 0;
  check(hb_placement_of_edge(&he, &pl));
  return static_cast<hetsim::grid::Placement>(pl);
}

// hetsim::grid::coord_of_rank(l, rank)
hetsim::grid::GridCoord coord_of_rank(const hetsim::grid::ModuleLayout& l, int rank) {
  hb_layout hl = lay(l);
  int c[4];
  check(hb_coord_of_rank(&hl, rank, c));
  return {c[0], c[1], c[2], c[3]};
}

// Device runtime, one per process/GPU. rank_to_gpu maps
// every logical rank; with n_gpus > 1 all-gather hb_exec_ipc_handle() over the
// caller's launcher, then call open_peers(). Compiled and linked by shim_check;
// it needs a GPU to run, so the CPU check does not construct it.
DeviceBridge::DeviceBridge(const hetsim::grid::BoundaryEdge& e, int n_gpus, int my_gpu,
                           const std::vector<int>& rank_to_gpu) {
  hb_edge he = edge(e);
  check(hb_plan_create(&he, &plan_));
  hb_exec_config c;
  hb_exec_config_default(&c);  // bf16 activations/gradients, fp32 accumulators
  check(hb_exec_create(plan_, nullptr, n_gpus, my_gpu, rank_to_gpu.data(), static_cast<int>(rank_to_gpu.size()),
                       &c, &x_));
}
DeviceBridge::~DeviceBridge() {
  hb_exec_destroy(x_);
  hb_plan_destroy(plan_);
}
std::vector<unsigned char> DeviceBridge::ipc_handle() const {
  std::vector<unsigned char> h(64);
  check(hb_exec_ipc_handle(x_, h.data()));
  return h;
}
void DeviceBridge::open_peers(const std::vector<unsigned char>& all_handles) {
  check(hb_exec_open_peers(x_, all_handles.data(), all_handles.size()));
}
void* DeviceBridge::buffer(int rank, int slot, int mb_slot, size_t* bytes) const {
  void* p = nullptr;
  check(hb_exec_buffer(x_, rank, slot, mb_slot, &p, bytes));
  return p;
}
// forward_colocated / forward_source+forward_dest of every resident rank (bridge.hpp:150-160)
void DeviceBridge::forward(int mb, void* stream) { check(hb_exec_forward(x_, mb, stream)); }
// backward_* of every resident rank; source gradients accumulate as beta*old + returned
void DeviceBridge::backward(int mb, float beta, void* stream) { check(hb_exec_backward(x_, mb, beta, stream)); }
void DeviceBridge::seed_forward_record(int mb) { check(hb_exec_seed_forward_record(x_, mb)); }

}  // namespace hetsim_hb
