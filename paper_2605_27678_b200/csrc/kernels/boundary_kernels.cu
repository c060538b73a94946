// hetbridge — sm_100a boundary kernels.
//
// K1/K2  copy_segments  : forward reshard and fused reshard+splice. Every
//        destination element has exactly one source element (index_map.hpp),
//        so forward is a persistent gather over (src, dst, bytes) runs whose
//        sources are local HBM or a peer GPU's HBM mapped over NVSwitch.
//        128-bit coalesced loads/stores, 4 independent 16 B loads in flight
//        per thread before any store.
// K3/K4  reduce_segments: backward gradient return with fp32 sum-accumulate
//        (dst = beta*dst + sum of terms in fixed order from +0.0f). Terms are
//        the cp-replica contributions (or the single owner) pulled from peers.
//
// Both kernels open with an epoch barrier on peer-mapped flag words (release
// stores / acquire loads at system scope) so a GPU reads a peer's buffers only
// after that peer's preceding stream work is done; with one GPU the barrier is
// compiled in but has empty masks.
//
// Roofline (pure data movement; tensor cores not applicable): time >=
// max(HBM bytes / HBM BW, NVLink ingress / NVLink BW); see DESIGN.md.
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdio>

#include "kernels/boundary_kernels.cuh"

namespace hb::dev {

namespace {

__device__ __forceinline__ uint4 ld_stream(const void* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}

__device__ __forceinline__ void st_vec(void* p, const uint4& v) {
  asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
}

__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Returns false if the barrier timed out (error flag set; caller skips work).
__device__ bool epoch_barrier(const SyncArgs& s, uint32_t* target_out) {
  __shared__ uint32_t target;
  __shared__ int ok;
  if (threadIdx.x == 0) {
    target = *reinterpret_cast<volatile uint32_t*>(s.ctr) + 1;
    ok = 1;
  }
  __syncthreads();
  const uint32_t e = target;
  *target_out = e;
  if (s.wait_mask | s.post_mask) {
    const int g = threadIdx.x;
    if (blockIdx.x == 0 && g < kMaxGpus && ((s.post_mask >> g) & 1u)) {
      __threadfence_system();
      st_release_sys(s.peer_pad[g] + s.my_gpu, e);
    }
    if (g < kMaxGpus && ((s.wait_mask >> g) & 1u)) {
      const long long t0 = clock64();
      while (static_cast<int32_t>(ld_acquire_sys(s.pad + g) - e) < 0) {
        __nanosleep(64);
        if (static_cast<uint64_t>(clock64() - t0) > s.timeout_cycles) {
          atomicExch(s.ctr + 2, 1u);
          ok = 0;
          break;
        }
      }
    }
    __syncthreads();
  }
  return ok != 0;
}

__device__ void epoch_finish(const SyncArgs& s, uint32_t e) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const uint32_t done = atomicAdd(s.ctr + 1, 1u);
    if (done == gridDim.x - 1) {
      s.ctr[1] = 0;
      __threadfence();
      atomicExch(s.ctr, e);
    }
  }
}

template <class S>
__device__ __forceinline__ int find_seg(const S* segs, int nseg, uint64_t chunk) {
  int lo = 0, hi = nseg - 1;
  while (lo < hi) {  // last seg with chunk0 <= chunk
    const int mid = (lo + hi + 1) >> 1;
    if (segs[mid].chunk0 <= chunk) lo = mid; else hi = mid - 1;
  }
  return lo;
}

template <class T>
__device__ __forceinline__ void copy_scalar(const unsigned char* src, unsigned char* dst, uint64_t lo,
                                            uint64_t hi) {
  const T* s = reinterpret_cast<const T*>(src);
  T* d = reinterpret_cast<T*>(dst);
  for (uint64_t i = lo / sizeof(T) + threadIdx.x; i < hi / sizeof(T); i += blockDim.x) d[i] = s[i];
}

constexpr int kUnroll = 4;

__global__ void __launch_bounds__(512) copy_segments_kernel(const CopySeg* __restrict__ segs, int nseg,
                                                            uint64_t total_chunks, SyncArgs sync) {
  uint32_t epoch;
  const bool ok = epoch_barrier(sync, &epoch);
  if (ok && nseg > 0) {
    for (uint64_t chunk = blockIdx.x; chunk < total_chunks; chunk += gridDim.x) {
      const CopySeg sg = segs[find_seg(segs, nseg, chunk)];
      const uint64_t lo = (chunk - sg.chunk0) * kCopyChunk;
      const uint64_t hi = min(lo + kCopyChunk, sg.nbytes);
      const uint64_t align = reinterpret_cast<uint64_t>(sg.src) | reinterpret_cast<uint64_t>(sg.dst) | sg.nbytes;
      if ((align & 15) == 0) {
        const unsigned char* s = sg.src;
        unsigned char* d = sg.dst;
        const uint64_t step = static_cast<uint64_t>(blockDim.x) * 16;
        uint64_t i = lo + threadIdx.x * 16;
        for (; i + (kUnroll - 1) * step < hi; i += kUnroll * step) {
          uint4 v[kUnroll];
#pragma unroll
          for (int u = 0; u < kUnroll; ++u) v[u] = ld_stream(s + i + u * step);
#pragma unroll
          for (int u = 0; u < kUnroll; ++u) st_vec(d + i + u * step, v[u]);
        }
        for (; i < hi; i += step) st_vec(d + i, ld_stream(s + i));
      } else if ((align & 3) == 0) {
        copy_scalar<uint32_t>(sg.src, sg.dst, lo, hi);
      } else if ((align & 1) == 0) {
        copy_scalar<uint16_t>(sg.src, sg.dst, lo, hi);
      } else {
        copy_scalar<unsigned char>(sg.src, sg.dst, lo, hi);
      }
    }
  }
  epoch_finish(sync, epoch);
}

// ---- reduction ---------------------------------------------------------------

template <class T> struct Cvt;
template <> struct Cvt<float> {
  __device__ static float to(float x) { return x; }
  __device__ static float from(float x) { return x; }
};
template <> struct Cvt<__nv_bfloat16> {
  __device__ static float to(__nv_bfloat16 x) { return __bfloat162float(x); }
  __device__ static __nv_bfloat16 from(float x) { return __float2bfloat16_rn(x); }
};
template <> struct Cvt<__half> {
  __device__ static float to(__half x) { return __half2float(x); }
  __device__ static __half from(float x) { return __float2half_rn(x); }
};

// 8 elements of T through 16 B vector accesses (1 x uint4 for 2-byte T, 2 for fp32).
template <class T>
__device__ __forceinline__ void load8(const T* p, float (&f)[8]) {
  constexpr int NV = sizeof(T) * 8 / 16;
  uint4 v[NV];
#pragma unroll
  for (int i = 0; i < NV; ++i) v[i] = ld_stream(reinterpret_cast<const uint4*>(p) + i);
  const T* e = reinterpret_cast<const T*>(v);
#pragma unroll
  for (int i = 0; i < 8; ++i) f[i] = Cvt<T>::to(e[i]);
}

template <class T>
__device__ __forceinline__ void load8_coherent(const T* p, float (&f)[8]) {
  constexpr int NV = sizeof(T) * 8 / 16;
  uint4 v[NV];
#pragma unroll
  for (int i = 0; i < NV; ++i) v[i] = *(reinterpret_cast<const uint4*>(p) + i);
  const T* e = reinterpret_cast<const T*>(v);
#pragma unroll
  for (int i = 0; i < 8; ++i) f[i] = Cvt<T>::to(e[i]);
}

template <class T>
__device__ __forceinline__ void store8(T* p, const float (&f)[8]) {
  constexpr int NV = sizeof(T) * 8 / 16;
  uint4 v[NV];
  T* e = reinterpret_cast<T*>(v);
#pragma unroll
  for (int i = 0; i < 8; ++i) e[i] = Cvt<T>::from(f[i]);
#pragma unroll
  for (int i = 0; i < NV; ++i) st_vec(reinterpret_cast<uint4*>(p) + i, v[i]);
}

template <class TIn, class TOut>
__global__ void __launch_bounds__(512) reduce_segments_kernel(const ReduceSeg* __restrict__ segs, int nseg,
                                                              const void* const* __restrict__ terms,
                                                              uint64_t total_chunks, float beta,
                                                              SyncArgs sync) {
  uint32_t epoch;
  const bool ok = epoch_barrier(sync, &epoch);
  if (ok && nseg > 0) {
    for (uint64_t chunk = blockIdx.x; chunk < total_chunks; chunk += gridDim.x) {
      const ReduceSeg sg = segs[find_seg(segs, nseg, chunk)];
      const uint64_t lo = (chunk - sg.chunk0) * kReduceChunk;
      const uint64_t hi = min(lo + kReduceChunk, sg.nelem);
      TOut* dst = static_cast<TOut*>(sg.dst);
      const TIn* const* tp = reinterpret_cast<const TIn* const*>(terms + sg.term0);
      uint64_t align = reinterpret_cast<uint64_t>(dst + lo);
      for (int t = 0; t < sg.nterms; ++t) align |= reinterpret_cast<uint64_t>(tp[t] + lo);
      uint64_t i = lo;
      if ((align & 15) == 0) {
        const uint64_t vec_hi = lo + ((hi - lo) & ~uint64_t(7));
        for (i = lo + threadIdx.x * 8; i < vec_hi; i += static_cast<uint64_t>(blockDim.x) * 8) {
          float acc[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) acc[k] = 0.0f;
          for (int t = 0; t < sg.nterms; ++t) {
            float v[8];
            load8(tp[t] + i, v);
#pragma unroll
            for (int k = 0; k < 8; ++k) acc[k] += v[k];
          }
          if (beta != 0.0f) {
            float o[8];
            load8_coherent(dst + i, o);
#pragma unroll
            for (int k = 0; k < 8; ++k) acc[k] = fmaf(beta, o[k], acc[k]);
          }
          store8(dst + i, acc);
        }
        i = vec_hi;
      }
      // scalar tail / unaligned path
      for (uint64_t e = i + threadIdx.x; e < hi; e += blockDim.x) {
        float acc = 0.0f;
        for (int t = 0; t < sg.nterms; ++t) acc += Cvt<TIn>::to(tp[t][e]);
        if (beta != 0.0f) acc = fmaf(beta, Cvt<TOut>::to(dst[e]), acc);
        dst[e] = Cvt<TOut>::from(acc);
      }
    }
  }
  epoch_finish(sync, epoch);
}

}  // namespace

int device_sm_count() {
  int dev = 0, n = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n;
}

void launch_copy(const CopySeg* segs, int nseg, uint64_t total_chunks, const SyncArgs& sync,
                 LaunchCfg cfg, void* stream) {
  const int grid = static_cast<int>(std::max<uint64_t>(1, std::min<uint64_t>(cfg.grid, total_chunks)));
  copy_segments_kernel<<<grid, cfg.block, 0, static_cast<cudaStream_t>(stream)>>>(segs, nseg, total_chunks,
                                                                                  sync);
}

template <class TIn, class TOut>
static void launch_reduce_t(const ReduceSeg* segs, int nseg, const void* const* terms, uint64_t total_chunks,
                            float beta, const SyncArgs& sync, int grid, int block, cudaStream_t st) {
  reduce_segments_kernel<TIn, TOut><<<grid, block, 0, st>>>(segs, nseg, terms, total_chunks, beta, sync);
}

void launch_reduce(const ReduceSeg* segs, int nseg, const void* const* terms, uint64_t total_chunks,
                   int in_dtype, int out_dtype, float beta, const SyncArgs& sync, LaunchCfg cfg,
                   void* stream) {
  const int grid = static_cast<int>(std::max<uint64_t>(1, std::min<uint64_t>(cfg.grid, total_chunks)));
  auto st = static_cast<cudaStream_t>(stream);
#define HB_RED(TI, TO) launch_reduce_t<TI, TO>(segs, nseg, terms, total_chunks, beta, sync, grid, cfg.block, st)
  switch (in_dtype * 4 + out_dtype) {
    case kBF16 * 4 + kBF16: HB_RED(__nv_bfloat16, __nv_bfloat16); break;
    case kBF16 * 4 + kFP16: HB_RED(__nv_bfloat16, __half); break;
    case kBF16 * 4 + kFP32: HB_RED(__nv_bfloat16, float); break;
    case kFP16 * 4 + kBF16: HB_RED(__half, __nv_bfloat16); break;
    case kFP16 * 4 + kFP16: HB_RED(__half, __half); break;
    case kFP16 * 4 + kFP32: HB_RED(__half, float); break;
    case kFP32 * 4 + kBF16: HB_RED(float, __nv_bfloat16); break;
    case kFP32 * 4 + kFP16: HB_RED(float, __half); break;
    case kFP32 * 4 + kFP32: HB_RED(float, float); break;
    default: break;  // validated on the host
  }
#undef HB_RED
}

}  // namespace hb::dev
