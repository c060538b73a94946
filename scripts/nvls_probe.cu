// NVLS multicast vs NVLink pulls for an all-gather-shaped step (C2's forward,
// C3's gradient gather): one process drives N GPUs. Every GPU owns a shard of
// `shard_mb` MB; afterwards every GPU must hold all N shards.
//   pull : each GPU's kernel reads the N-1 peer shards (LDG.128 over NVLink,
//          peer access) and writes them locally — the boundary kernels' pattern
//   mcast: each GPU's kernel stores its own shard once through a multicast
//          address (multimem.st); the NVSwitch replicates it into every GPU
// Prints per-GPU ingress GB/s for both, all GPUs running concurrently.
// Measurement tool only (not on the product path).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o nvls_probe nvls_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                               \
  do {                                                                                      \
    CUresult r_ = (x);                                                                      \
    if (r_ != CUDA_SUCCESS) {                                                               \
      const char* s_ = nullptr;                                                             \
      cuGetErrorString(r_, &s_);                                                            \
      std::fprintf(stderr, "%s:%d %s -> %s\n", __FILE__, __LINE__, #x, s_ ? s_ : "?");       \
      std::exit(2);                                                                         \
    }                                                                                       \
  } while (0)
#define CR(x)                                                                               \
  do {                                                                                      \
    cudaError_t e_ = (x);                                                                   \
    if (e_ != cudaSuccess) {                                                                \
      std::fprintf(stderr, "%s:%d %s -> %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
      std::exit(2);                                                                         \
    }                                                                                       \
  } while (0)

__global__ void mcast_store(const uint4* __restrict__ src, unsigned long long mc_dst, size_t n16) {
  constexpr int U = 4;  // loads of U vectors in flight before their multicast stores
  const size_t step = (size_t)gridDim.x * blockDim.x;
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  for (; i + (U - 1) * step < n16; i += U * step) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = src[i + u * step];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const unsigned long long p = mc_dst + (i + u * step) * 16;
      asm volatile("multimem.st.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v[u].x), "r"(v[u].y),
                   "r"(v[u].z), "r"(v[u].w)
                   : "memory");
    }
  }
  for (; i < n16; i += step) {
    const uint4 v = src[i];
    asm volatile("multimem.st.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(mc_dst + i * 16), "r"(v.x), "r"(v.y),
                 "r"(v.z), "r"(v.w)
                 : "memory");
  }
}

// pull: n_src peer shards, each n16 x 16 B, into dst (shard k at dst + k*n16)
__global__ void pull_copy(const uint4* const* __restrict__ srcs, int n_src, uint4* __restrict__ dst, size_t n16) {
  constexpr int U = 8;  // independent 16-B peer loads in flight per thread (the LDG engine's depth)
  const size_t step = (size_t)gridDim.x * blockDim.x;
  for (int k = 0; k < n_src; ++k) {
    const uint4* s = srcs[k];
    uint4* d = dst + k * n16;
    size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    for (; i + (U - 1) * step < n16; i += U * step) {
      uint4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] = s[i + u * step];
#pragma unroll
      for (int u = 0; u < U; ++u) d[i + u * step] = v[u];
    }
    for (; i < n16; i += step) d[i] = s[i];
  }
}

int main(int argc, char** argv) {
  const size_t shard = (argc > 1 ? std::atoll(argv[1]) : 32) << 20;
  int N = 0;
  CR(cudaGetDeviceCount(&N));
  if (argc > 2) N = std::atoi(argv[2]);
  CK(cuInit(0));
  std::vector<CUdevice> dev(N);
  std::vector<CUcontext> ctx(N);
  for (int d = 0; d < N; ++d) {
    CK(cuDeviceGet(&dev[d], d));
    CR(cudaSetDevice(d));
    CR(cudaFree(nullptr));
    CK(cuCtxGetCurrent(&ctx[d]));
    int mc = 0;
    CK(cuDeviceGetAttribute(&mc, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev[d]));
    if (!mc) {
      std::printf("{\"multicast_supported\": false}\n");
      return 0;
    }
  }
  const size_t total = shard * N;
  // multicast object over N devices, `total` bytes
  CUmulticastObjectProp mp{};
  mp.numDevices = N;
  mp.size = total;
  mp.handleTypes = CU_MEM_HANDLE_TYPE_NONE;
  size_t gran = 0;
  CK(cuMulticastGetGranularity(&gran, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED));
  const size_t size = (total + gran - 1) / gran * gran;
  mp.size = size;
  CUmemGenericAllocationHandle mch;
  CK(cuMulticastCreate(&mch, &mp));
  for (int d = 0; d < N; ++d) CK(cuMulticastAddDevice(mch, dev[d]));
  std::vector<CUmemGenericAllocationHandle> phys(N);
  std::vector<CUdeviceptr> uc(N), mcva(N);
  for (int d = 0; d < N; ++d) {
    CK(cuCtxSetCurrent(ctx[d]));
    CUmemAllocationProp ap{};
    ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ap.location.id = d;
    size_t ag = 0;
    CK(cuMemGetAllocationGranularity(&ag, &ap, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
    CK(cuMemCreate(&phys[d], size, &ap, 0));
    CK(cuMulticastBindMem(mch, 0, phys[d], 0, size, 0));
    // unicast view of this GPU's copy, accessible by every GPU (pull baseline)
    CK(cuMemAddressReserve(&uc[d], size, 0, 0, 0));
    CK(cuMemMap(uc[d], size, 0, phys[d], 0));
    std::vector<CUmemAccessDesc> acc(N);
    for (int p = 0; p < N; ++p) {
      acc[p].location.type = CU_MEM_LOCATION_TYPE_DEVICE;
      acc[p].location.id = p;
      acc[p].flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    }
    CK(cuMemSetAccess(uc[d], size, acc.data(), N));
    // multicast view for this GPU
    CK(cuMemAddressReserve(&mcva[d], size, 0, 0, 0));
    CK(cuMemMap(mcva[d], size, 0, mch, 0));
    CUmemAccessDesc a1{};
    a1.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    a1.location.id = d;
    a1.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    CK(cuMemSetAccess(mcva[d], size, &a1, 1));
  }
  // per-GPU source shard (plain allocation) and the pull destination
  std::vector<uint4*> src(N), dstp(N);
  std::vector<const uint4**> srcs_dev(N);
  std::vector<cudaStream_t> st(N);
  const size_t n16 = shard / 16;
  for (int d = 0; d < N; ++d) {
    CR(cudaSetDevice(d));
    CR(cudaMalloc(&src[d], shard));
    CR(cudaMemset(src[d], d + 1, shard));
    CR(cudaMalloc(&dstp[d], shard * (N - 1)));
    CR(cudaStreamCreateWithFlags(&st[d], cudaStreamNonBlocking));
    std::vector<const uint4*> s;
    for (int p = 0; p < N; ++p)
      if (p != d) s.push_back(reinterpret_cast<const uint4*>(uc[p] + p * shard));  // peer's own shard slot
    CR(cudaMalloc(&srcs_dev[d], s.size() * sizeof(void*)));
    CR(cudaMemcpy(srcs_dev[d], s.data(), s.size() * sizeof(void*), cudaMemcpyHostToDevice));
    // put each GPU's shard into its own slot of its unicast copy (the pull sources)
    CR(cudaMemcpy(reinterpret_cast<void*>(uc[d] + d * shard), src[d], shard, cudaMemcpyDeviceToDevice));
  }
  int sms = 0;
  CR(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  auto run = [&](bool mcast, int reps) {
    std::vector<cudaEvent_t> e0(N), e1(N);
    for (int d = 0; d < N; ++d) {
      CR(cudaSetDevice(d));
      CR(cudaEventCreate(&e0[d]));
      CR(cudaEventCreate(&e1[d]));
    }
    for (int d = 0; d < N; ++d) {
      CR(cudaSetDevice(d));
      CR(cudaDeviceSynchronize());
    }
    for (int d = 0; d < N; ++d) {
      CR(cudaSetDevice(d));
      CR(cudaEventRecord(e0[d], st[d]));
      for (int r = 0; r < reps; ++r) {
        if (mcast)
          mcast_store<<<2 * sms, 512, 0, st[d]>>>(src[d], mcva[d] + d * shard, n16);
        else
          pull_copy<<<2 * sms, 512, 0, st[d]>>>(srcs_dev[d], N - 1, dstp[d], n16);
      }
      CR(cudaEventRecord(e1[d], st[d]));
    }
    float worst = 0;
    for (int d = 0; d < N; ++d) {
      CR(cudaSetDevice(d));
      CR(cudaEventSynchronize(e1[d]));
      float ms = 0;
      CR(cudaEventElapsedTime(&ms, e0[d], e1[d]));
      worst = ms > worst ? ms : worst;
    }
    CR(cudaGetLastError());
    return worst / reps;
  };
  run(false, 2);
  run(true, 2);
  const float t_pull = run(false, 10), t_mc = run(true, 10);
  // check: every GPU's multicast copy holds every shard
  bool ok = true;
  for (int d = 0; d < N && ok; ++d)
    for (int p = 0; p < N && ok; ++p) {
      unsigned char b = 0;
      CR(cudaMemcpy(&b, reinterpret_cast<void*>(uc[d] + p * shard + shard / 2), 1, cudaMemcpyDeviceToHost));
      ok = b == static_cast<unsigned char>(p + 1);
    }
  const double ingress = static_cast<double>(shard) * (N - 1);
  std::printf(
      "{\"n_gpus\": %d, \"shard_mb\": %zu, \"pull_ms\": %.4f, \"pull_ingress_gbs\": %.1f, \"mcast_ms\": %.4f, "
      "\"mcast_ingress_gbs\": %.1f, \"mcast_egress_gbs\": %.1f, \"mcast_copies_ok\": %s}\n",
      N, shard >> 20, t_pull, ingress / (t_pull * 1e-3) / 1e9, t_mc, ingress / (t_mc * 1e-3) / 1e9,
      static_cast<double>(shard) / (t_mc * 1e-3) / 1e9, ok ? "true" : "false");
  return 0;
}
