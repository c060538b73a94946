// Reference-side binding of hetbridge (see hetsim_bridge_hb.cpp).
#pragma once

#include <cstddef>
#include <string>
#include <vector>

#include "hetbridge.h"
#include "hetsim/bridge.hpp"
#include "hetsim/error.hpp"
#include "hetsim/grid.hpp"

namespace hetsim_hb {
std::string export_plan(const hetsim::grid::BoundaryEdge& e);
hetsim::bridge::DpRelation classify_dp_relation(const hetsim::grid::BoundaryEdge& e);
hetsim::grid::Placement placement_of_edge(const hetsim::grid::BoundaryEdge& e);
hetsim::grid::GridCoord coord_of_rank(const hetsim::grid::ModuleLayout& l, int rank);

// hetsim::bridge::BridgeRuntime's role calls for every logical rank resident on
// this process's GPU, one launch per op (streams are cudaStream_t passed as void*).
class DeviceBridge {
 public:
  DeviceBridge(const hetsim::grid::BoundaryEdge& e, int n_gpus, int my_gpu, const std::vector<int>& rank_to_gpu);
  ~DeviceBridge();
  DeviceBridge(const DeviceBridge&) = delete;
  DeviceBridge& operator=(const DeviceBridge&) = delete;
  std::vector<unsigned char> ipc_handle() const;
  void open_peers(const std::vector<unsigned char>& all_handles);
  void* buffer(int rank, int slot, int mb_slot, size_t* bytes) const;
  void forward(int mb, void* stream);
  void backward(int mb, float beta, void* stream);
  void seed_forward_record(int mb);

 private:
  hb_plan* plan_ = nullptr;
  hb_exec* x_ = nullptr;
};
}  // namespace hetsim_hb
