// hetbridge — projector GEMM with a boundary epilogue (see projector_gemm.cu).
#pragma once

#include <cstdint>

#include "kernels/boundary_kernels.cuh"

namespace hb::dev {

// Y[M x N] = X[M x K] . W[N x K]^T, bf16 in, fp32 accumulate (TMEM), bf16 out.
// Output row m is stored to row_dst[m*fan + f] for every non-null f < fan
// (each a pointer to N contiguous bf16 elements, 16-B aligned; local or peer).
constexpr int kMaxProjFan = 8;  // destinations per output row

struct ProjectorArgs {
  int M, N, K;
  unsigned char* const* row_dst;  // device array [M * fan]
  int fan;
  SyncArgs sync;  // launch protocol (push: peers' destinations); empty masks on one GPU
};

// 0 OK; 1 shape (N % 256, K % 64), 3 alignment, 4 tensor map, 5 launch.
int projector_check_shape(int M, int N, int K);
int launch_projector(const void* x, int64_t ldx, const void* w, int64_t ldw, const ProjectorArgs& args,
                     int sm_count, void* stream);

}  // namespace hb::dev
