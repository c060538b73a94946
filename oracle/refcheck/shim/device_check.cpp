// device_check — executes the reference-side DeviceBridge (hetsim_bridge_hb.cpp:
// hetsim::grid::BoundaryEdge in, hetsim's role calls collapsed onto one GPU's
// launches through the hetbridge C-ABI) on cuda:0 and compares what it moves
// with the oracle's hetsim::bridge::bridge_forward / bridge_backward
// (R:core/include/hetsim/bridge.hpp:178-185) over the same inputs.
//
// Test infrastructure (run by tests/test_reference_tests.py on a GPU box).
// Values are multiples of 1/8 below 8 in magnitude, so bf16 activations and
// gradients and their fp32 sums are exact: forward placement and the backward
// return must match bit for bit. Exit 0 iff every layout agrees.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "hetsim_bridge_hb.hpp"

using hetsim::grid::BoundaryEdge;
using hetsim::grid::ModuleLayout;
namespace br = hetsim::bridge;

namespace {

int g_fail = 0, g_checks = 0;

void cuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    std::fprintf(stderr, "%s: %s\n", what, cudaGetErrorString(e));
    std::exit(2);
  }
}

uint16_t to_bf16(double v) {  // exact for the values used here
  const float f = static_cast<float>(v);
  uint32_t u;
  std::memcpy(&u, &f, 4);
  return static_cast<uint16_t>(u >> 16);
}
double from_bf16(uint16_t h) {
  const uint32_t u = static_cast<uint32_t>(h) << 16;
  float f;
  std::memcpy(&f, &u, 4);
  return f;
}

// value of global row `row`, column `c` of activation (kind 0) or gradient (kind 1)
double val(int kind, int row, int c) {
  const int k = ((row * 131 + c * 31 + kind * 17) % 127) - 63;  // -63..63
  return k / 8.0;
}

ModuleLayout lay(const char* name, int tp, int cp, int pp, int dp, int off = 0) {
  ModuleLayout m;
  m.name = name;
  m.tp = tp, m.cp = cp, m.pp = pp, m.dp = dp, m.rank_offset = off;
  return m;
}

void run(const char* label, const BoundaryEdge& e) {
  const int W = e.feature_width;
  const auto plan = br::plan_bridge(e);
  const int world = std::max(e.source.rank_offset + e.source.world_size(), e.dest.rank_offset + e.dest.world_size());
  std::vector<int> r2g(world, 0);
  hetsim_hb::DeviceBridge dbr(e, 1, 0, r2g);

  // ---- forward: every source rank with a device shard gets its interval's rows
  std::map<int, br::ShardedTensor> shards;
  for (int r = 0; r < world; ++r) {
    size_t bytes = 0;
    void* p = dbr.buffer(r, HB_SLOT_SRC_ACT, 0, &bytes);
    if (!p || !bytes) continue;
    const auto c = hetsim::grid::coord_of_rank(e.source, r);
    const auto iv = plan.src_intervals[c.dp_idx];
    br::ShardedTensor t{iv, W, std::vector<double>(static_cast<size_t>(iv.length) * W)};
    std::vector<uint16_t> h(t.payload.size());
    for (int i = 0; i < iv.length; ++i)
      for (int j = 0; j < W; ++j) {
        t.payload[static_cast<size_t>(i) * W + j] = val(0, iv.start + i, j);
        h[static_cast<size_t>(i) * W + j] = to_bf16(val(0, iv.start + i, j));
      }
    if (bytes != h.size() * 2) {
      std::printf("FAIL %s: source rank %d buffer %zu B, interval needs %zu B\n", label, r, bytes, h.size() * 2);
      ++g_fail;
      return;
    }
    cuda(cudaMemcpy(p, h.data(), bytes, cudaMemcpyHostToDevice), "H2D src");
    shards[r] = std::move(t);
  }
  const auto ref = br::bridge_forward(plan, shards, 0);
  dbr.forward(0, nullptr);
  cuda(cudaDeviceSynchronize(), "forward");
  for (const auto& [r, t] : ref) {
    size_t bytes = 0;
    void* p = dbr.buffer(r, HB_SLOT_DST_ACT, 0, &bytes);
    ++g_checks;
    if (!p || bytes != t.payload.size() * 2) {
      std::printf("FAIL %s: dest rank %d has no matching device buffer\n", label, r);
      ++g_fail;
      continue;
    }
    std::vector<uint16_t> h(t.payload.size());
    cuda(cudaMemcpy(h.data(), p, bytes, cudaMemcpyDeviceToHost), "D2H dst");
    for (size_t i = 0; i < h.size(); ++i)
      if (from_bf16(h[i]) != t.payload[i]) {
        std::printf("FAIL %s: forward rank %d element %zu: device %g oracle %g\n", label, r, i, from_bf16(h[i]),
                    t.payload[i]);
        ++g_fail;
        break;
      }
  }

  // ---- backward (beta = 0): destination gradients identical across replicas (the contract)
  std::map<int, br::ShardedTensor> grads;
  for (const auto& [r, t] : ref) {
    size_t bytes = 0;
    void* p = dbr.buffer(r, HB_SLOT_DST_GRAD, 0, &bytes);
    if (!p || !bytes) continue;
    br::ShardedTensor g{t.interval, W, std::vector<double>(t.payload.size())};
    std::vector<uint16_t> h(g.payload.size());
    for (int i = 0; i < t.interval.length; ++i)
      for (int j = 0; j < W; ++j) {
        g.payload[static_cast<size_t>(i) * W + j] = val(1, t.interval.start + i, j);
        h[static_cast<size_t>(i) * W + j] = to_bf16(val(1, t.interval.start + i, j));
      }
    cuda(cudaMemcpy(p, h.data(), bytes, cudaMemcpyHostToDevice), "H2D grad");
    grads[r] = std::move(g);
  }
  const auto refb = br::bridge_backward(plan, grads, 0);
  dbr.backward(0, 0.0f, nullptr);
  cuda(cudaDeviceSynchronize(), "backward");
  for (const auto& [r, t] : refb) {
    size_t bytes = 0;
    void* p = dbr.buffer(r, HB_SLOT_SRC_GRAD, 0, &bytes);
    ++g_checks;
    if (!p || bytes != t.payload.size() * 4) {
      std::printf("FAIL %s: source rank %d has no matching gradient buffer\n", label, r);
      ++g_fail;
      continue;
    }
    std::vector<float> h(t.payload.size());
    cuda(cudaMemcpy(h.data(), p, bytes, cudaMemcpyDeviceToHost), "D2H grad");
    for (size_t i = 0; i < h.size(); ++i)
      if (static_cast<double>(h[i]) != t.payload[i]) {
        std::printf("FAIL %s: backward rank %d element %zu: device %g oracle %g\n", label, r, i, h[i],
                    t.payload[i]);
        ++g_fail;
        break;
      }
  }
  std::printf("%-58s fwd ranks %zu, bwd ranks %zu\n", label, ref.size(), refb.size());
}

}  // namespace

int main() {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
    std::printf("device_check: no CUDA device\n");
    return 2;
  }
  const int W = 512;
  struct Case {
    const char* label;
    ModuleLayout s, d;
    int B;
  };
  const std::vector<Case> cases = {
      {"C1 equal-DP enc{dp2} -> llm{dp2}", lay("enc", 1, 1, 1, 2), lay("llm", 1, 1, 1, 2), 8},
      {"C2 fan-in vit{dp8} -> llm{tp4,dp2}", lay("vit", 1, 1, 1, 8), lay("llm", 4, 1, 1, 2), 64},
      {"C3 fan-out enc{tp4,dp2} -> llm{dp8}", lay("enc", 4, 1, 1, 2), lay("llm", 1, 1, 1, 8), 64},
      {"C3' deliver enc{pp4,dp2} -> llm{dp8}", lay("enc", 1, 1, 4, 2), lay("llm", 1, 1, 1, 8), 64},
      {"C5 non-colocated vit{dp2}@0 -> llm{tp2,pp3}@2", lay("vit", 1, 1, 1, 2), lay("llm", 2, 1, 3, 1, 2), 16},
      {"App-C vision{tp4,dp2} -> language{tp2,pp2,dp2}", lay("vision", 4, 1, 1, 2), lay("language", 2, 1, 2, 2), 16},
      {"cp reduce vit{dp8} -> llm{tp2,cp4}", lay("vit", 1, 1, 1, 8), lay("llm", 2, 4, 1, 1), 16},
  };
  for (const auto& c : cases) {
    try {
      run(c.label, BoundaryEdge{c.s, c.d, c.B, W});
    } catch (const std::exception& e) {
      std::printf("FAIL %s: %s\n", c.label, e.what());
      ++g_fail;
    }
  }
  std::printf("device_check: %d checks, %d mismatches\n", g_checks, g_fail);
  return g_fail ? 1 : 0;
}
