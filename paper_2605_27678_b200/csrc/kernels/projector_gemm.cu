// hetbridge — sm_100a projector GEMM with a boundary epilogue.
//
// The encoder's last layer (the projector, tinymodel.hpp:62 enc_w2) computes
// Y[M x N] = X[M x K] . W[N x K]^T for one source rank's M token rows. This
// kernel computes it on the 5th-generation tensor cores and writes every output
// row straight to each destination row the boundary plan maps it to (the tp
// replicas of the destination shard, local or on a peer GPU over NVSwitch),
// instead of writing the source shard and running the forward reshard over it.
//
// Structure (one CTA per SM, persistent over 128 x 256 output tiles):
//   warp 0      TMA producer: cp.async.bulk.tensor 2-D loads of X and W tiles
//               (128B-swizzled, 64-element K blocks) into a 3-stage smem ring
//   warp 1      MMA issuer: one lane issues tcgen05.mma.cta_group::1.kind::f16
//               (M=128, N=256, K=16) into a TMEM accumulator; tcgen05.commit
//               frees smem stages and publishes a finished accumulator
//   warps 2..5  epilogue: tcgen05.ld 32x32b.x32 (warp w reads TMEM lanes
//               32*(w%4)..+31 = its tile rows), fp32 -> bf16 into a per-lane
//               512-B smem row, then one TMA bulk store of the row per
//               destination (local HBM or a peer over NVSwitch). TMEM is
//               released as soon as the tile sits in smem; the accumulator is
//               double buffered (2 x 256 columns) so the next tile's MMAs run
//               under this tile's stores.
// Three variants (HB_PROJ_CLUSTER): single CTAs (1), CTA pairs sharing the W
// tile by TMA multicast (2), and the default, CTA pairs running one 256 x 256
// tile with tcgen05.mma.cta_group::2 (3): each CTA stages its 128 rows of X
// and its 128 rows of W (32 KiB per k-block instead of 48), the leader CTA
// issues M=256 MMAs that read both CTAs' shared memory and write each CTA's
// 128 accumulator rows into its own TMEM. That halves the per-SM shared-memory
// read traffic of the B operand, which (with the TMA writes) is what bounds the
// single-CTA M=128 x N=256 MMA.
// Roofline: tensor (2*M*N*K flop) for K large; for the projector shapes the
// output stores (M*N*2 B per destination) usually bind.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdint>
#include <cstdlib>

#include "kernels/launch_protocol.cuh"
#include "kernels/projector_gemm.cuh"

namespace hb::dev {

namespace {

constexpr int kBM = 128, kBN = 256, kBK = 64;  // tile; kBK = one 128-B swizzle row of bf16
constexpr int kStages = 3;    // single / multicast pair: 48 KiB stages
// 2-SM pair: 32 KiB stages; 4 for short K (the projector's 1024-1280), 5 for
// long K (kDeep), where a half-row epilogue staging makes room for the 5th
constexpr int kStages2Sm = 4, kStages2SmDeep = 5;
constexpr uint32_t kABytes = kBM * kBK * 2, kBBytes = kBN * kBK * 2;  // 16 KiB, 32 KiB
constexpr uint32_t kStageBytes = kABytes + kBBytes;
constexpr uint32_t kStageBytes2Sm = kABytes + kBBytes / 2;  // own X rows + own half of the W tile
constexpr int kEpiWarps = 4;
constexpr int kThreads = 32 * (2 + kEpiWarps);
constexpr uint32_t kTmemCols = 2 * kBN;  // two accumulators
// epilogue staging: per epilogue warp 32 tile rows of 512 B (256 bf16), rows
// padded to 528 B so the lanes' 16-B writes of one chunk spread over all banks
constexpr int kEpiRowPitch = kBN * 2 + 16;
constexpr uint32_t kEpiBytes = kEpiWarps * 32 * kEpiRowPitch;
constexpr size_t kSmemBytes = kStages * kStageBytes + kEpiBytes + 1024;  // + alignment slack
// 2-SM variant: the epilogue stages a tile row in two halves of 128 columns
// (one bulk store per half and destination), which frees smem for a 5th stage
constexpr int kEpiRowPitchHalf = kBN / 2 * 2 + 16;
static_assert(kStages2Sm * kStageBytes2Sm + kEpiBytes + 1024 <= kSmemBytes, "2-SM ring fits the dynamic smem");
static_assert(kStages2SmDeep * kStageBytes2Sm + kEpiWarps * 32 * kEpiRowPitchHalf + 1024 <= kSmemBytes,
              "deep 2-SM ring + half-row staging fit the dynamic smem");
constexpr int kDeepK = 2048;  // K from which the 2-SM variant takes the deep ring

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra W;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* smem, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
      "[%4];" ::"r"(smem_u32(smem)),
      "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
// multicast variant: the W half this CTA loads lands in both CTAs of the pair
__device__ __forceinline__ void tma_load_2d_mc(void* smem, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                               uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.multicast::cluster [%0], "
      "[%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(smem)),
      "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "h"(mask)
      : "memory");
}
__device__ __forceinline__ void tc_commit_mc(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(mask)
      : "memory");
}
// 2-SM pair load: the bytes land in this CTA's smem and complete on the
// LEADER's barrier (the peer bit of the barrier's shared::cluster address cleared)
__device__ __forceinline__ void tma_load_2d_2sm(void* smem, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
      "[%4];" ::"r"(smem_u32(smem)),
      "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar) & 0xFEFFFFFFu)
      : "memory");
}
__device__ __forceinline__ void tc_commit_2sm(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(mask)
      : "memory");
}
// arrive on the barrier at the same smem offset in CTA `rank` of the cluster
__device__ __forceinline__ void mbar_arrive_cluster(uint64_t* bar, uint32_t rank) {
  asm volatile(
      "{\n .reg .b32 ra;\n mapa.shared::cluster.u32 ra, %0, %1;\n"
      " mbarrier.arrive.release.cluster.shared::cluster.b64 _, [ra];\n}\n" ::"r"(smem_u32(bar)),
      "r"(rank)
      : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

// Work items: single tiles (kCM = 1) or, for a CTA pair (kCM = 2), pairs of
// M-adjacent tiles that share their W tile: CTA r of the pair takes m-tile
// 2*i + r, and each CTA loads half of W and multicasts it to both.
template <int kCM>
struct TileMap {
  int tiles_m, tiles_n, tiles_mp, rank;
  __device__ TileMap(int M, int N, int r)
      : tiles_m((M + kBM - 1) / kBM), tiles_n(N / kBN), tiles_mp((tiles_m + kCM - 1) / kCM), rank(r) {}
  __device__ int items() const { return tiles_mp * tiles_n; }
  __device__ int first() const { return static_cast<int>(blockIdx.x) / kCM; }
  __device__ int step() const { return static_cast<int>(gridDim.x) / kCM; }
  // Grouped rasterisation: items walk every n tile of a group of kGroupM
  // m-tiles (pairs) before the next group, so the tiles in flight at once
  // (about one per SM pair) share a few X row blocks and W column blocks that
  // stay in L2. Walking all of M per n column re-read X from DRAM once per n
  // column when X exceeds L2 (16384x4096x4096: 1.88 GB of DRAM reads, 49% L2
  // hits, against 0.31 GB for cuBLAS).
  static constexpr int kGroupM = 8;
  __device__ void coords(int item, int& m0, int& n0) const {
    const int per_group = kGroupM * tiles_n;
    const int g = item / per_group;
    const int first = g * kGroupM;
    const int rows = tiles_mp - first < kGroupM ? tiles_mp - first : kGroupM;
    const int local = item - g * per_group;
    m0 = ((first + local % rows) * kCM + rank) * kBM;  // may lie beyond M in the last pair: rows are skipped
    n0 = (local / rows) * kBN;
  }
};

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
// K-major, 128B-swizzled operand tile: 8-row atoms of 1024 B (SBO), version 1 (sm100)
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr) {
  return static_cast<uint64_t>((saddr >> 4) & 0x3FFF) | (static_cast<uint64_t>(1) << 16) |
         (static_cast<uint64_t>(1024 >> 4) << 32) | (static_cast<uint64_t>(1) << 46) |
         (static_cast<uint64_t>(2) << 61);
}
// kind::f16 instruction descriptor: D fp32, A/B bf16, both K-major, N=256, M=128 (M=256 for the pair)
constexpr uint32_t idesc_f16(int m) {
  return (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(kBN >> 3) << 17) |
         (static_cast<uint32_t>(m >> 4) << 24);
}
constexpr uint32_t kIdesc = idesc_f16(kBM);
constexpr uint32_t kIdesc2Sm = idesc_f16(2 * kBM);
__device__ __forceinline__ void umma_bf16(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(kIdesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void umma_bf16_2sm(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(kIdesc2Sm), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ uint32_t pack_bf16(uint32_t lo, uint32_t hi) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(__uint_as_float(hi)), "f"(__uint_as_float(lo)));
  return r;
}
#define HB_TMEM_LD32(addr, v)                                                                                   \
  asm volatile(                                                                                                  \
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,"  \
      "%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"                                      \
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),         \
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),   \
        "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]),             \
        "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]),             \
        "=r"(v[30]), "=r"(v[31])                                                                               \
      : "r"(addr))

__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {  // sees remote release arrivals
  asm volatile(
      "{\n .reg .pred p;\n"
      "W: mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra W;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// kCM: CTAs per cluster (1 or 2); k2Sm: the pair runs tcgen05.mma.cta_group::2
template <int kCM, bool k2Sm, bool kDeep = false>
__global__ void __launch_bounds__(kThreads, 1)
    projector_gemm_kernel(const __grid_constant__ CUtensorMap map_x, const __grid_constant__ CUtensorMap map_w,
                          ProjectorArgs args) {
  static_assert(!k2Sm || kCM == 2, "the 2-SM MMA runs on a CTA pair");
  static_assert(!kDeep || k2Sm, "the deep ring is a 2-SM variant");
  constexpr int S = k2Sm ? (kDeep ? kStages2SmDeep : kStages2Sm) : kStages;
  constexpr uint32_t SB = k2Sm ? kStageBytes2Sm : kStageBytes;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t full[S], empty[S], tfull[2], tempty[2];
  __shared__ uint32_t tmem_base_sh;
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int num_k = args.K / kBK;
  const uint32_t crank = kCM > 1 ? cluster_rank() : 0;
  const TileMap<kCM> tm(args.M, args.N, static_cast<int>(crank));

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(&map_x) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&map_w) : "memory");
    for (int i = 0; i < S; ++i) {
      mbar_init(&full[i], 1);
      // multicast pair: both CTAs' MMAs read a stage the pair filled; 2-SM: the
      // leader's one commit frees the stage in both CTAs
      mbar_init(&empty[i], k2Sm ? 1 : kCM);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      // 2-SM: one arrival per epilogue warp of both CTAs, on the leader's barrier
      mbar_init(&tempty[i], k2Sm ? 2 * kEpiWarps : kEpiWarps * 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // launch protocol: count in (epoch), CTA 0 posts "started" to the peers
  // whose destinations this launch writes
  __shared__ CtaSync cs;
  if (blockIdx.x == 0 && warp == 0) post_peers_warp(args.sync, 0);
  if (threadIdx.x == 0) cta_arrive_finish(args.sync, cs, cta_arrive_issue(args.sync));
  if (warp == 1) {  // one warp allocates (and later frees) the two accumulators
    if constexpr (k2Sm) {  // the same warp of both CTAs, the same smem slot: one pair allocation
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_u32(&tmem_base_sh)),
                   "r"(kTmemCols)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_u32(&tmem_base_sh)),
                   "r"(kTmemCols)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (kCM > 1) cluster_sync_all();  // the peer's barriers exist before anything multicasts into them
  tc_fence_after();
  const uint32_t tmem_base = tmem_base_sh;

  if (warp == 0) {
    if (lane == 0) {  // ---- TMA producer
      int stage = 0;
      uint32_t phase = 0;
      for (int item = tm.first(); item < tm.items(); item += tm.step()) {
        int m0, n0;
        tm.coords(item, m0, n0);
        for (int kb = 0; kb < num_k; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          unsigned char* a = smem + stage * SB;
          if constexpr (k2Sm) {
            // each CTA stages its own X rows and its own half of the W tile; all
            // of the pair's bytes complete on the leader's full barrier
            if (crank == 0) mbar_expect_tx(&full[stage], 2 * SB);
            tma_load_2d_2sm(a, &map_x, &full[stage], kb * kBK, m0);
            tma_load_2d_2sm(a + kABytes, &map_w, &full[stage], kb * kBK, n0 + static_cast<int>(crank) * (kBN / 2));
            if (++stage == S) {
              stage = 0;
              phase ^= 1;
            }
            continue;
          }
          mbar_expect_tx(&full[stage], kStageBytes);  // own X tile + both W halves
          tma_load_2d(a, &map_x, &full[stage], kb * kBK, m0);
          if constexpr (kCM == 1) {
            tma_load_2d(a + kABytes, &map_w, &full[stage], kb * kBK, n0);
          } else {
            constexpr int kHalf = kBN / kCM;
            tma_load_2d_mc(a + kABytes + crank * (kBBytes / kCM), &map_w, &full[stage], kb * kBK,
                           n0 + static_cast<int>(crank) * kHalf, static_cast<uint16_t>((1u << kCM) - 1));
          }
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && (!k2Sm || crank == 0)) {  // ---- MMA issuer (2-SM: the leader CTA only)
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int item = tm.first(); item < tm.items(); item += tm.step(), ++it) {
        const int acc = it & 1;
        const uint32_t aphase = (it >> 1) & 1;
        // the epilogue drained this accumulator (2-SM: in both CTAs)
        if constexpr (k2Sm) mbar_wait_cluster(&tempty[acc], aphase ^ 1);
        else mbar_wait(&tempty[acc], aphase ^ 1);
        tc_fence_after();
        const uint32_t d = tmem_base + acc * kBN;
        if constexpr (k2Sm) {
          for (int kb = 0; kb < num_k; ++kb) {
            mbar_wait(&full[stage], phase);
            tc_fence_after();
            // the same smem offsets in both CTAs: A = the CTA's 128 X rows, B = its 128 W rows
            const uint32_t a = smem_u32(smem + stage * SB), b = a + kABytes;
#pragma unroll
            for (int k = 0; k < kBK / 16; ++k)
              umma_bf16_2sm(d, umma_desc_sw128(a + k * 32), umma_desc_sw128(b + k * 32), (kb | k) != 0);
            tc_commit_2sm(&empty[stage], 0x3);  // frees the stage in both CTAs
            if (++stage == S) {
              stage = 0;
              phase ^= 1;
            }
          }
          tc_commit_2sm(&tfull[acc], 0x3);  // each CTA's 128 accumulator rows are complete
          continue;
        }
        for (int kb = 0; kb < num_k; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t a = smem_u32(smem + stage * kStageBytes), b = a + kABytes;
#pragma unroll
          for (int k = 0; k < kBK / 16; ++k)  // K=16 per MMA: 32 B along the swizzled row
            umma_bf16(d, umma_desc_sw128(a + k * 32), umma_desc_sw128(b + k * 32), (kb | k) != 0);
          // frees the stage once these MMAs have read it (in both CTAs of a pair:
          // each one's producer multicast into the other's stage)
          if constexpr (kCM == 1) tc_commit(&empty[stage]);
          else tc_commit_mc(&empty[stage], static_cast<uint16_t>((1u << kCM) - 1));
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
        tc_commit(&tfull[acc]);  // accumulator complete
      }
    }
  } else {  // ---- epilogue warps: TMEM -> registers -> bf16 -> smem rows -> TMA bulk stores per destination
    const int q = warp % 4;  // TMEM lane quarter this warp may access
    constexpr int H = kDeep ? 2 : 1;                    // staging passes per tile row
    constexpr int RP = kDeep ? kEpiRowPitchHalf : kEpiRowPitch;
    constexpr int CPH = kBN / 32 / H;                  // 32-column TMEM chunks per pass
    unsigned char* stage_w = smem + S * SB + (warp - 2) * (32 * RP);
    unsigned char* my_row = stage_w + lane * RP;
    // before the first store: every peer has started this op, so its
    // destination buffers of this set are no longer read
    bool ok = true;
    if (lane == 0)
      for (int g = 0; g < kMaxGpus; ++g)
        if (((args.sync.wait_mask >> g) & 1u) && !spin_until(args.sync, args.sync.pad + g, cs.e)) ok = false;
    ok = __shfl_sync(0xffffffffu, ok, 0);
    int it = 0;
    for (int item = tm.first(); item < tm.items(); item += tm.step(), ++it) {
      const int acc = it & 1;
      const uint32_t aphase = (it >> 1) & 1;
      int m0, n0;
      tm.coords(item, m0, n0);
      const int row = m0 + q * 32 + lane;
      mbar_wait(&tfull[acc], aphase);
      tc_fence_after();
#pragma unroll 1
      for (int h = 0; h < H; ++h) {
        // this lane's staging row is free once its previous bulk stores have read it
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
#pragma unroll 1
        for (int cc = 0; cc < CPH; ++cc) {
          const int c = h * CPH + cc;
          uint32_t v[32];
          HB_TMEM_LD32(tmem_base + acc * kBN + c * 32 + (static_cast<uint32_t>(q * 32) << 16), v);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          uint4* dst = reinterpret_cast<uint4*>(my_row + cc * 64);
#pragma unroll
          for (int i = 0; i < 4; ++i)
            dst[i] = make_uint4(pack_bf16(v[8 * i], v[8 * i + 1]), pack_bf16(v[8 * i + 2], v[8 * i + 3]),
                                pack_bf16(v[8 * i + 4], v[8 * i + 5]), pack_bf16(v[8 * i + 6], v[8 * i + 7]));
        }
        if (h == H - 1) {
          // the whole accumulator has been read: hand TMEM back to the MMA warp
          tc_fence_before();
          if constexpr (k2Sm) {  // one arrival per warp, on the leader's barrier
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(&tempty[acc], 0);
          } else {
            mbar_arrive(&tempty[acc]);
          }
        }
        // each lane stores its row piece (512 / H contiguous bytes) to every destination
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        if (row < args.M && ok) {
          unsigned char* const* d = args.row_dst + static_cast<size_t>(row) * args.fan;
          for (int f = 0; f < args.fan; ++f) {
            unsigned char* p = d[f];
            if (!p) break;
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(
                             p + (static_cast<size_t>(n0) + static_cast<size_t>(h) * (kBN / H)) * 2),
                         "r"(smem_u32(my_row)), "r"(static_cast<uint32_t>(kBN / H * 2))
                         : "memory");
          }
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
      }
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // every store complete before the end protocol
  }
  __syncthreads();
  if constexpr (kCM > 1) cluster_sync_all();  // no CTA leaves while its peer may still arrive on its barriers
  if (warp == 1) {
    tc_fence_after();
    if constexpr (k2Sm)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(kTmemCols)
                   : "memory");
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(kTmemCols)
                   : "memory");
  }
  // end: "writes done" to every peer written, wait for every writer into this GPU
  if (threadIdx.x == 0) launch_end_lane(args.sync, cs);
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }();
  return fn;
}

// 2-D bf16 tensor map over a row-major [rows x cols] matrix, box [box_rows x 64], 128B swizzle
bool make_map(CUtensorMap* m, const void* base, uint64_t rows, uint64_t cols, uint64_t ld_elems,
              uint32_t box_rows) {
  auto fn = encode_fn();
  if (!fn) return false;
  const cuuint64_t dims[2] = {cols, rows};
  const cuuint64_t strides[1] = {ld_elems * 2};
  const cuuint32_t box[2] = {static_cast<cuuint32_t>(kBK), box_rows};
  const cuuint32_t estr[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

int projector_check_shape(int M, int N, int K) {
  if (M < 0 || N < kBN || K < kBK) return 1;
  if (N % kBN || K % kBK) return 2;
  return 0;
}

int launch_projector(const void* x, int64_t ldx, const void* w, int64_t ldw, const ProjectorArgs& args,
                     int sm_count, void* stream) {
  if (projector_check_shape(args.M, args.N, args.K) || args.fan < 1 || args.fan > kMaxProjFan) return 1;
  if ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(w)) & 15) return 3;
  if ((ldx * 2) % 16 || (ldw * 2) % 16) return 3;
  // 3 (default): CTA pairs with the 2-SM MMA; 2: CTA pairs sharing W tiles
  // through TMA multicast; 1: single CTAs (HB_PROJ_CLUSTER, A/B knob)
  static const int mode = [] {
    const char* v = std::getenv("HB_PROJ_CLUSTER");
    return (v && (v[0] == '1' || v[0] == '2')) ? v[0] - '0' : 3;
  }();
  const int cm = mode == 1 ? 1 : 2;
  CUtensorMap mx{}, mw{};
  // M == 0: this GPU projects no rows but still takes part in the launch protocol
  if (args.M > 0 && (!make_map(&mx, x, args.M, args.K, ldx, kBM) || !make_map(&mw, w, args.N, args.K, ldw, kBN / cm)))
    return 4;
  static PerDeviceOnce once;  // function attributes are per device
  int dev = 0;
  cudaGetDevice(&dev);
  once(dev, [] {
    cudaFuncSetAttribute(projector_gemm_kernel<1, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(kSmemBytes));
    cudaFuncSetAttribute(projector_gemm_kernel<2, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(kSmemBytes));
    cudaFuncSetAttribute(projector_gemm_kernel<2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(kSmemBytes));
    cudaFuncSetAttribute(projector_gemm_kernel<2, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(kSmemBytes));
  });
  const int items = ((args.M + kBM - 1) / kBM + cm - 1) / cm * (args.N / kBN);
  int grid = items * cm < sm_count ? items * cm : sm_count - sm_count % cm;
  if (grid < cm) grid = cm;
  auto st = static_cast<cudaStream_t>(stream);
  if (cm == 1) {
    projector_gemm_kernel<1, false><<<grid, kThreads, kSmemBytes, st>>>(mx, mw, args);
  } else {
    cudaLaunchConfig_t lc{};
    lc.gridDim = dim3(grid);
    lc.blockDim = dim3(kThreads);
    lc.dynamicSmemBytes = kSmemBytes;
    lc.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
    const cudaError_t e =
        mode != 3         ? cudaLaunchKernelEx(&lc, projector_gemm_kernel<2, false>, mx, mw, args)
        : args.K >= kDeepK ? cudaLaunchKernelEx(&lc, projector_gemm_kernel<2, true, true>, mx, mw, args)
                           : cudaLaunchKernelEx(&lc, projector_gemm_kernel<2, true>, mx, mw, args);
    if (e != cudaSuccess) return 5;
  }
  return cudaGetLastError() == cudaSuccess ? 0 : 5;
}

}  // namespace hb::dev
