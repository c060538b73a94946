// hetbridge — sm_100a boundary kernels.
//
// K1/K2  copy_segments  : forward reshard and fused reshard+splice. Every
//        destination element has exactly one source element (index_map.hpp),
//        so forward is a persistent gather over (src, dst, bytes) runs whose
//        sources are local HBM or a peer GPU's HBM mapped over NVSwitch.
//        Two engines: (a) LDG/STG.128 with 8 independent 16 B loads in flight
//        per thread, (b) TMA bulk copies (cp.async.bulk global->smem->global,
//        mbarrier-tracked, one issuing lane per CTA, 3-stage smem ring).
// K3/K4  reduce_segments: backward gradient return with fp32 sum-accumulate
//        (dst = beta*dst + sum of terms in fixed order from +0.0f). Terms are
//        the cp-replica contributions (or the single owner) pulled from peers.
//
// Work split over CTAs (Partition::mode): contiguous ranges with a host-built
// first-segment table, interleaved equal shares of every segment, or dynamic
// chunks handed out by an atomic counter (monotone per-CTA segment cursor).
//
// Both kernels open with an epoch barrier on peer-mapped flag words (release
// stores / acquire loads at system scope) so a GPU reads a peer's buffers only
// after that peer's preceding stream work is done; with one GPU the barrier is
// compiled in but has empty masks. In push mode the last CTA also publishes
// "writes done" and waits for every writer into this GPU before the kernel ends.
//
// Roofline (pure data movement; tensor cores not applicable): time >=
// max(HBM bytes / HBM BW, NVLink ingress / NVLink BW); see DESIGN.md.
#include <cstdlib>
#include <tuple>

#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "kernels/boundary_kernels.cuh"
#include "kernels/launch_protocol.cuh"


namespace hb::dev {

namespace {

// Plain (coherent) global load that skips L1 allocation. Deliberately not
// `.nc`: ptxas may sink non-coherent loads below the stores that follow them,
// which collapses the 8-deep load batch to ~4 in flight (seen in SASS).
__device__ __forceinline__ uint4 ld_stream(const void* p) {
  uint4 v;
  asm volatile("ld.global.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}

__device__ __forceinline__ void st_vec(void* p, const uint4& v) {
  asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
}

constexpr uint32_t kNoChunk = 0xffffffffu;

// Work queues (dynamic / TMA partitions). One thread per CTA drives them.
// A claim is issued (atomic in flight) before the current chunk is processed
// and resolved after it, so the claim round trip overlaps the copy. Once the
// current queue is within one grid of its end, the first claim of the other
// queue is started too, so the switch costs no extra round trip (every CTA
// still claims each non-empty queue until exactly one claim fails there).
struct Claimer {
  int q;           // current queue: 1 remote, 0 local
  int passes;      // queues finished
  uint32_t first;  // static first chunk of the home queue (kNoChunk: none)
  unsigned long long pre[2];  // raw value of the claim in flight per queue (valid if has[q])
  bool has[2];

  __device__ static uint32_t total_of(const Partition& p, int qq) { return qq ? p.rtotal_chunks : p.total_chunks; }
  __device__ void init(const Partition& p) {
    const int b = static_cast<int>(blockIdx.x);
    q = b < p.remote_ctas ? 1 : 0;
    passes = 0;
    has[0] = has[1] = false;
    if (blockIdx.x >= p.claimers) {  // outside this kind's partition (fused launch with a larger grid)
      passes = 2;
      first = kNoChunk;
      return;
    }
    const uint32_t idx = q ? static_cast<uint32_t>(b) : static_cast<uint32_t>(b - p.remote_ctas);
    first = idx < (q ? p.rstatic : p.lstatic) ? idx : kNoChunk;
    if (total_of(p, q) == 0) advance_queue(p);
  }
  __device__ void advance_queue(const Partition& p) {  // next non-empty queue, or done
    while (++passes < 2) {
      q ^= 1;
      if (total_of(p, q) != 0) return;
    }
  }
  __device__ bool done() const { return passes >= 2; }
  __device__ void claim(const SyncArgs& s, int qq) {
    pre[qq] = atomicAdd(s.queue + qq * (kCtrLine / 2), 1ull);
    has[qq] = true;
  }
  // Start the claim after chunk `c` of the current queue (kNoChunk: none held)
  // and, near the queue's end, the other queue's first claim.
  __device__ void issue(const Partition& p, const SyncArgs& s, uint32_t c) {
    claim(s, q);
    const int o = q ^ 1;
    if (p.prefetch_other && passes == 0 && !has[o] && total_of(p, o) != 0 &&
        (c == kNoChunk || static_cast<unsigned long long>(c) + p.claimers >= total_of(p, q)))
      claim(s, o);
  }
  __device__ uint32_t resolve(const Partition& p, uint32_t e, unsigned long long raw, int qq) const {
    const uint32_t total = total_of(p, qq);
    const uint32_t stat = qq ? p.rstatic : p.lstatic;
    const unsigned long long adv = static_cast<unsigned long long>(total - stat) + p.claimers;
    const unsigned long long idx = raw - static_cast<unsigned long long>(e - 1) * adv + stat;
    return idx < total ? static_cast<uint32_t>(idx) : kNoChunk;
  }
  // Next chunk (kNoChunk: this CTA is done); *remote = its queue. Consumes the
  // claims in flight (claiming synchronously only if none is), and starts the
  // following claim.
  __device__ uint32_t next(const Partition& p, const SyncArgs& s, uint32_t e, int* remote) {
    while (!done()) {
      if (!has[q]) claim(s, q);
      has[q] = false;
      const uint32_t c = resolve(p, e, pre[q], q);
      if (c != kNoChunk) {
        *remote = q;
        issue(p, s, c);
        return c;
      }
      advance_queue(p);
    }
    *remote = q;
    return kNoChunk;
  }
};

// Interleaved partition: CTA b takes quanta [q*b/G, q*(b+1)/G) of a segment.
__device__ __forceinline__ bool cta_share(uint64_t n, uint64_t* a, uint64_t* b) {
  const uint64_t q = (n + kQuantum - 1) / kQuantum;
  *a = (q * blockIdx.x / gridDim.x) * kQuantum;
  const uint64_t e = (q * (blockIdx.x + 1) / gridDim.x) * kQuantum;
  *b = e < n ? e : n;
  return *a < *b;
}

// Drives `body(seg, a, b)` over this CTA's work under the partition's mode,
// between the launch's arrival and end protocol. Dynamic mode keeps two
// queues: chunks whose data stays on this GPU (no peer dependency: started
// immediately, hiding the barrier latency) and chunks that touch a peer
// (handed out only after this CTA confirmed the peers' arrival). The first
// `remote_ctas` CTAs drain the remote queue first, the rest the local one;
// both then help with the other queue. A CTA's first chunk is static; the
// arrival round trip overlaps it.
template <int MODE, class S, class Len, class Body>
__device__ __forceinline__ void run_shares(const S* __restrict__ segs, int nseg, const Partition& part,
                                           const SyncArgs& sync, Len len, Body body) {
  __shared__ CtaSync cs;
  __shared__ uint32_t cur;  // chunk being processed (kNoChunk: none)
  __shared__ int cur_remote;
  unsigned long long arr = 0;
  griddep_wait();
  if (blockIdx.x == 0 && threadIdx.x < 32) {
    post_peers_warp(sync, 0);
    __syncwarp();
  }
  if (threadIdx.x == 0) {
    trace_at(sync, kTrEntry);
    arr = cta_arrive_issue(sync);
  }
  if constexpr (MODE == kPartDynamic) {
    // Claim state lives in shared memory: only thread 0 touches it, between
    // chunks, and keeping it out of registers across the body avoids spills
    // in the 64-register reduce loop.
    __shared__ Claimer cl;
    __shared__ uint32_t nch, nrem;  // trace counters
    if (threadIdx.x == 0) {
      nch = nrem = 0;
      cl.init(part);
      cur = cl.done() ? kNoChunk : cl.first;
      cur_remote = cl.q;
      if (!cl.done()) cl.issue(part, sync, cl.first);  // the claim after the static chunk, in flight
      // a remote first chunk needs the peers first (all of them: a per-peer
      // wait here would put two dependent table loads on thread 0's path
      // between chunks; measured slower for the gradient return)
      if (cur != kNoChunk && cl.q == 1) {
        cta_arrive_finish(sync, cs, arr);
        arr = ~0ull;
        sync_wait_lane(sync, cs);
      }
    }
    __syncthreads();
    bool first = true;
    while (true) {
      const uint32_t c = cur;
      // a remote chunk after a timed-out wait is claimed but not executed
      if (c != kNoChunk && (!cur_remote || cs.ok)) {
        const uint2 t = (cur_remote ? part.rchunks : part.chunks)[c];
        const S sg = segs[t.x];
        const uint64_t cu = cur_remote ? part.rchunk : part.chunk;
        const uint64_t a = static_cast<uint64_t>(t.y & 0xffffffu) * cu, e = a + ((t.y >> 24) + 1) * cu, n = len(sg);
        body(sg, a, e < n ? e : n, cur_remote != 0);
        if (threadIdx.x == 0 && sync.trace) {
          ++nch;
          nrem += cur_remote != 0;
        }
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        if (first) trace_at(sync, kTrFirst);
        if (first && arr != ~0ull) cta_arrive_finish(sync, cs, arr);
        first = false;
        int rq = 0;
        cur = cl.next(part, sync, cs.e, &rq);
        cur_remote = rq;
        if (cur != kNoChunk && rq) sync_wait_lane(sync, cs);
      }
      __syncthreads();
      if (cur == kNoChunk) break;
    }
    griddep_launch_dependents();  // this CTA's work is done: the next op may take its slot
    if (threadIdx.x == 0) {
      trace_at(sync, kTrDone);
      launch_end_lane(sync, cs);
      trace_at(sync, kTrExit);
      trace_val(sync, kTrChunks, nch);
      trace_val(sync, kTrRemote, nrem);
    }
  } else {
    if (threadIdx.x == 0) {
      cta_arrive_finish(sync, cs, arr);
      sync_wait_lane(sync, cs);
    }
    __syncthreads();
    if (cs.ok && nseg > 0) {
      if constexpr (MODE == kPartInterleaved) {
        for (int s = 0; s < nseg; ++s) {
          const S sg = segs[s];
          uint64_t a, b;
          if (cta_share(len(sg), &a, &b)) body(sg, a, b, false);
        }
      } else {
        const uint64_t lo = blockIdx.x * part.per_cta, hi = lo + part.per_cta;
        for (int s = part.first_seg[blockIdx.x]; s < nseg; ++s) {
          const S sg = segs[s];
          if (sg.w0 >= hi) break;
          const uint64_t a = (lo > sg.w0 ? lo : sg.w0) - sg.w0;
          const uint64_t e = sg.w0 + len(sg);
          const uint64_t b = (hi < e ? hi : e) - sg.w0;
          if (a < b) body(sg, a, b, false);
        }
      }
    }
    __syncthreads();
    griddep_launch_dependents();
    if (threadIdx.x == 0) launch_end_lane(sync, cs);
  }
}

template <class T>
__device__ __forceinline__ void copy_scalar(const unsigned char* src, unsigned char* const* dst, int ndst,
                                            uint64_t lo, uint64_t hi) {
  const T* s = reinterpret_cast<const T*>(src);
  for (uint64_t i = lo / sizeof(T) + threadIdx.x; i < hi / sizeof(T); i += blockDim.x) {
    const T v = s[i];
    for (int d = 0; d < ndst; ++d) reinterpret_cast<T*>(dst[d])[i] = v;
  }
}

constexpr int kUnroll = 8;

__device__ __forceinline__ void copy_range_from(const CopySeg& sg, const unsigned char* __restrict__ src, uint64_t a,
                                                uint64_t b);

// Source address of byte `off` of a gather run (nullptr: bad id, error set).
__device__ __forceinline__ const unsigned char* gather_src(const CopySeg& sg, uint64_t off, uint32_t* err) {
  const int64_t id = sg.ids[off / sg.row_bytes];
  if (id < 0 || id >= sg.vocab) {
    atomicExch(err, kErrBadId);
    return nullptr;
  }
  if (sg.shards) {  // vocab-parallel: the owner shard of the TP group (local or a peer's)
    const uint64_t s = static_cast<uint64_t>(id) / sg.shard_rows;
    return sg.shards[s] + (static_cast<uint64_t>(id) - s * sg.shard_rows) * sg.row_bytes + off % sg.row_bytes;
  }
  return sg.src + static_cast<uint64_t>(id) * sg.row_bytes + off % sg.row_bytes;
}

// Copies bytes [a, b) of one segment to each of its destinations with the
// whole CTA: every 16 B of the source is loaded once and stored ndst times.
// Gather runs are copied row piece by row piece.
__device__ __forceinline__ void copy_range(const CopySeg& sg, uint64_t a, uint64_t b, uint32_t* err) {
  if (!sg.ids) {
    copy_range_from(sg, sg.src, a, b);
    return;
  }
  for (uint64_t off = a; off < b;) {
    const uint64_t end = min(b, (off / sg.row_bytes + 1) * sg.row_bytes);
    const unsigned char* p = gather_src(sg, off, err);
    // copy_range_from indexes its source by the run offset: rebase the row piece
    if (p) copy_range_from(sg, p - off, off, end);
    off = end;
  }
}

__device__ __forceinline__ void copy_range_from(const CopySeg& sg, const unsigned char* __restrict__ src, uint64_t a,
                                                uint64_t b) {
  const int nd = sg.ndst;
  uint64_t align = reinterpret_cast<uint64_t>(src) | a;
  for (int d = 0; d < nd; ++d) align |= reinterpret_cast<uint64_t>(sg.dst[d]);
  if ((align & 15) == 0) {
    const uint64_t vend = a + ((b - a) & ~uint64_t(15));
    const uint64_t step = static_cast<uint64_t>(blockDim.x) * 16;
    uint64_t i = a + threadIdx.x * 16;
    for (; i + (kUnroll - 1) * step < vend; i += kUnroll * step) {
      uint4 v[kUnroll];
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) v[u] = ld_stream(src + i + u * step);
      for (int d = 0; d < nd; ++d) {
        unsigned char* dst = sg.dst[d];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) st_vec(dst + i + u * step, v[u]);
      }
    }
    for (; i < vend; i += step) {
      const uint4 v = ld_stream(src + i);
      for (int d = 0; d < nd; ++d) st_vec(sg.dst[d] + i, v);
    }
    for (uint64_t j = vend + threadIdx.x; j < b; j += blockDim.x)
      for (int d = 0; d < nd; ++d) sg.dst[d][j] = src[j];
  } else {
    const uint64_t al = align | b;
    if ((al & 3) == 0) copy_scalar<uint32_t>(src, sg.dst, nd, a, b);
    else if ((al & 1) == 0) copy_scalar<uint16_t>(src, sg.dst, nd, a, b);
    else copy_scalar<unsigned char>(src, sg.dst, nd, a, b);
  }
}

struct CopyLen {
  __device__ uint64_t operator()(const CopySeg& s) const { return s.nbytes; }
};

template <int MODE>
__global__ void __launch_bounds__(512, 2) copy_segments_kernel(const CopySeg* __restrict__ segs, int nseg,
                                                            Partition part, SyncArgs sync) {
  run_shares<MODE>(segs, nseg, part, sync, CopyLen{},
                   [&](const CopySeg& sg, uint64_t a, uint64_t b, bool) { copy_range(sg, a, b, sync.err); });
}

// ---- TMA bulk-copy engine ------------------------------------------------------

// Stage ring variants (chunk = one stage); selected by Partition::chunk.
// 3 x 32 KiB (default), 6 x 16 KiB, 8 x 8 KiB: 96 / 96 / 64 KiB of smem.

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_expect(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra W;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void bulk_g2s(void* smem, const void* gmem, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(smem)),
      "l"(gmem), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void bulk_store(void* gmem, const void* smem, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gmem), "r"(smem_u32(smem)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }

template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// One warp per CTA; lane 0 issues TMA bulk copies through a kTmaStages ring of
// shared-memory stages: loads for the next stages are in flight while the
// current stage is stored (once per destination of the run). Chunks (= one
// stage) come from the work queues; unaligned runs are copied by lane 0.
// The issuing lane of a TMA copy: arrival, the stage ring over the claimed
// chunks, and the end-of-launch protocol (called by exactly one thread of the
// CTA; `full` and `cs` are that CTA's shared memory).
template <int kTmaStages, uint32_t kTmaStageBytes>
__device__ __forceinline__ void tma_copy_lane(const CopySeg* __restrict__ segs, const Partition& part,
                                              const SyncArgs& sync, unsigned char* stage_mem, uint64_t* full,
                                              CtaSync& cs) {
  trace_at(sync, kTrEntry);
  const unsigned long long arr = cta_arrive_issue(sync);
  for (int i = 0; i < kTmaStages; ++i) mbar_init(&full[i]);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  // chunk k lives in stage k % kTmaStages; its barrier phase is (k / kTmaStages) & 1
  uint32_t pend_seg[kTmaStages];
  uint32_t pend_bytes[kTmaStages];
  uint64_t pend_off[kTmaStages];
  bool pend_bad[kTmaStages];  // gather chunk with an out-of-range id: its rows are not stored
  uint32_t issued = 0, nremote = 0;
  bool more = true, arrived = false;
  Claimer cl;
  cl.init(part);
  bool use_first = !cl.done();
  if (!cl.done()) cl.issue(part, sync, cl.first);  // the claim after the static chunk, in flight
  auto arrive = [&]() {
    if (!arrived) {
      cta_arrive_finish(sync, cs, arr);
      arrived = true;
    }
  };
  auto issue = [&]() {  // next chunk: start its global->smem load
    while (more) {
      uint32_t c;
      int rq;
      if (use_first) {
        use_first = false;
        c = cl.first;
        rq = cl.q;
      } else {
        arrive();
        c = cl.next(part, sync, cs.e, &rq);
        if (c == kNoChunk) {
          more = false;
          return;
        }
      }
      if (c == kNoChunk) continue;
      const uint2 t = (rq ? part.rchunks : part.chunks)[c];
      const CopySeg& sg = segs[t.x];
      if (rq == 1) {
        arrive();
        if (!sync_wait_peers(sync, cs, sg.peers)) continue;  // timed out: claimed, not executed
      }
      const uint64_t a = static_cast<uint64_t>(t.y & 0xffffffu) * part.chunk;  // (copy chunks are one unit)
      const uint64_t e = a + part.chunk < sg.nbytes ? a + part.chunk : sg.nbytes;
      const uint32_t bytes = static_cast<uint32_t>(e - a);
      const int nd = sg.ndst;
      uint64_t al = reinterpret_cast<uint64_t>(sg.src + a) | bytes | (sg.ids ? sg.row_bytes : 0u);
      for (int d = 0; d < nd; ++d) al |= reinterpret_cast<uint64_t>(sg.dst[d] + a);
      if (al & 15) {  // rare unaligned run: plain byte copy by this lane
        for (uint64_t i = a; i < e; ++i) {
          const unsigned char* p = sg.ids ? gather_src(sg, i, sync.err) : sg.src + i;
          if (p)
            for (int d = 0; d < nd; ++d) sg.dst[d][i] = *p;
        }
        continue;
      }
      const int st = issued % kTmaStages;
      bool bad = false;
      mbar_expect(&full[st], bytes);
      if (!sg.ids) {
        bulk_g2s(stage_mem + st * kTmaStageBytes, sg.src + a, bytes, &full[st]);
      } else {  // gather run: one bulk load per row piece (a bad id loads row 0, its stores are skipped below)
        for (uint64_t off = a; off < e;) {
          const uint64_t end = min(e, (off / sg.row_bytes + 1) * sg.row_bytes);
          const unsigned char* p = gather_src(sg, off, sync.err);
          bad |= p == nullptr;
          bulk_g2s(stage_mem + st * kTmaStageBytes + (off - a), p ? p : sg.src + off % sg.row_bytes,
                   static_cast<uint32_t>(end - off), &full[st]);
          off = end;
        }
      }
      pend_bad[st] = bad;
      pend_seg[st] = t.x;
      pend_off[st] = a;
      pend_bytes[st] = bytes;
      ++issued;
      nremote += rq;
      return;
    }
  };
  for (int i = 0; i < kTmaStages; ++i) issue();
  for (uint32_t k = 0; k < issued; ++k) {
    const int st = k % kTmaStages;
    mbar_wait(&full[st], (k / kTmaStages) & 1u);
    if (k == 0) trace_at(sync, kTrFirst);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    // one bulk group per chunk: a store to every destination of the run
    const CopySeg& sg = segs[pend_seg[st]];
    const int nd = sg.ndst;
    if (!pend_bad[st]) {
      for (int d = 0; d < nd; ++d)
        bulk_store(sg.dst[d] + pend_off[st], stage_mem + st * kTmaStageBytes, pend_bytes[st]);
    } else {  // error path: store the good row pieces only (bad rows stay untouched, as in copy_range)
      const uint64_t a = pend_off[st], e = a + pend_bytes[st];
      for (uint64_t off = a; off < e;) {
        const uint64_t end = min(e, (off / sg.row_bytes + 1) * sg.row_bytes);
        const int64_t id = sg.ids[off / sg.row_bytes];
        if (id >= 0 && id < sg.vocab)
          for (int d = 0; d < nd; ++d)
            bulk_store(sg.dst[d] + off, stage_mem + st * kTmaStageBytes + (off - a), static_cast<uint32_t>(end - off));
        off = end;
      }
    }
    bulk_commit();
    if (k >= 1 && more) {
      bulk_wait_read<1>();  // store k-1 has finished reading its stage
      issue();              // chunk k-1+kTmaStages reuses stage (k-1) % kTmaStages
    }
  }
  // Push mode publishes "writes done" to peers: the stores must be complete.
  // Otherwise only the stage reads must be (the grid's completion makes the
  // stores visible to the stream's next kernel, as a TMA-store epilogue does).
  if (sync.end_sync) bulk_wait_all();
  else bulk_wait_read<0>();
  griddep_launch_dependents();  // this CTA's work is issued and its stages read: the next op may take its slot
  arrive();
  trace_at(sync, kTrDone);
  launch_end_lane(sync, cs);
  trace_at(sync, kTrExit);
  trace_val(sync, kTrChunks, issued);
  trace_val(sync, kTrRemote, nremote);
}

template <int kTmaStages, uint32_t kTmaStageBytes>
__global__ void __launch_bounds__(32) copy_segments_tma_kernel(const CopySeg* __restrict__ segs, int nseg,
                                                               Partition part, SyncArgs sync) {
  extern __shared__ __align__(128) unsigned char stage_mem[];
  __shared__ __align__(8) uint64_t full[kTmaStages];
  __shared__ CtaSync cs;
  griddep_wait();
  if (blockIdx.x == 0) {
    post_peers_warp(sync, 0);
    __syncwarp();
  }
  if (threadIdx.x != 0) return;  // one issuing lane; the rest of the warp has nothing to do
  tma_copy_lane<kTmaStages, kTmaStageBytes>(segs, part, sync, stage_mem, full, cs);
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

// 8 elements of T <-> 8 floats through 16 B vector accesses (1 x uint4 for
// 2-byte T, 2 for fp32). Conversions work on the 32-bit words with bit ops
// and packed cvt instructions, so nothing is type-punned through memory (a
// punned uint4 array ends up in local memory under the 64-register cap).
template <class T> struct Pack8;
template <> struct Pack8<float> {
  static constexpr int NV = 2;
  __device__ static void unpack(const uint4 (&v)[NV], float (&f)[8]) {
    f[0] = __uint_as_float(v[0].x); f[1] = __uint_as_float(v[0].y);
    f[2] = __uint_as_float(v[0].z); f[3] = __uint_as_float(v[0].w);
    f[4] = __uint_as_float(v[1].x); f[5] = __uint_as_float(v[1].y);
    f[6] = __uint_as_float(v[1].z); f[7] = __uint_as_float(v[1].w);
  }
  __device__ static void pack(const float (&f)[8], uint4 (&v)[NV]) {
    v[0] = make_uint4(__float_as_uint(f[0]), __float_as_uint(f[1]), __float_as_uint(f[2]), __float_as_uint(f[3]));
    v[1] = make_uint4(__float_as_uint(f[4]), __float_as_uint(f[5]), __float_as_uint(f[6]), __float_as_uint(f[7]));
  }
};
__device__ __forceinline__ uint32_t cvt_bf16x2(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}
__device__ __forceinline__ uint32_t cvt_f16x2(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}
__device__ __forceinline__ float f16_lo(uint32_t w) { return __half2float(__ushort_as_half(static_cast<unsigned short>(w & 0xffffu))); }
__device__ __forceinline__ float f16_hi(uint32_t w) { return __half2float(__ushort_as_half(static_cast<unsigned short>(w >> 16))); }
template <> struct Pack8<__nv_bfloat16> {
  static constexpr int NV = 1;
  __device__ static void unpack(const uint4 (&v)[NV], float (&f)[8]) {
    const uint32_t w[4] = {v[0].x, v[0].y, v[0].z, v[0].w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      f[2 * i] = __uint_as_float(w[i] << 16);
      f[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
    }
  }
  __device__ static void pack(const float (&f)[8], uint4 (&v)[NV]) {
    v[0] = make_uint4(cvt_bf16x2(f[0], f[1]), cvt_bf16x2(f[2], f[3]), cvt_bf16x2(f[4], f[5]), cvt_bf16x2(f[6], f[7]));
  }
};
template <> struct Pack8<__half> {
  static constexpr int NV = 1;
  __device__ static void unpack(const uint4 (&v)[NV], float (&f)[8]) {
    const uint32_t w[4] = {v[0].x, v[0].y, v[0].z, v[0].w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      f[2 * i] = f16_lo(w[i]);
      f[2 * i + 1] = f16_hi(w[i]);
    }
  }
  __device__ static void pack(const float (&f)[8], uint4 (&v)[NV]) {
    v[0] = make_uint4(cvt_f16x2(f[0], f[1]), cvt_f16x2(f[2], f[3]), cvt_f16x2(f[4], f[5]), cvt_f16x2(f[6], f[7]));
  }
};

#if HB_PUN_CONVERT  // A/B: element-wise conversion through a punned uint4 array
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
#else
template <class T>
__device__ __forceinline__ void load8(const T* p, float (&f)[8]) {
  uint4 v[Pack8<T>::NV];
#pragma unroll
  for (int i = 0; i < Pack8<T>::NV; ++i) v[i] = ld_stream(reinterpret_cast<const uint4*>(p) + i);
  Pack8<T>::unpack(v, f);
}

template <class T>
__device__ __forceinline__ void load8_coherent(const T* p, float (&f)[8]) {
  uint4 v[Pack8<T>::NV];
#pragma unroll
  for (int i = 0; i < Pack8<T>::NV; ++i) v[i] = *(reinterpret_cast<const uint4*>(p) + i);
  Pack8<T>::unpack(v, f);
}

template <class T>
__device__ __forceinline__ void store8(T* p, const float (&f)[8]) {
  uint4 v[Pack8<T>::NV];
  Pack8<T>::pack(f, v);
#pragma unroll
  for (int i = 0; i < Pack8<T>::NV; ++i) st_vec(reinterpret_cast<uint4*>(p) + i, v[i]);
}
#endif

// acc[] (+)= the n terms' 8 elements at offset i (acc starts at +0.0f: terms
// are summed in order from +0.0, as simnet's all_reduce does).
template <class TIn>
__device__ __forceinline__ void sum_terms8(const TIn* const* __restrict__ tp, int nterms, uint64_t i,
                                           float (&acc)[8]) {
  load8(tp[0] + i, acc);
#pragma unroll
  for (int k = 0; k < 8; ++k) acc[k] = 0.0f + acc[k];
  for (int t = 1; t < nterms; ++t) {
    float v[8];
    load8(tp[t] + i, v);
#pragma unroll
    for (int k = 0; k < 8; ++k) acc[k] += v[k];
  }
}

// Two groups (offsets i and i + step) with every load of a term issued before
// any of them is consumed (the loop over terms is data-dependent, so separate
// per-group calls would serialise the groups' load latencies).
template <class TIn>
__device__ __forceinline__ void sum_terms8x2(const TIn* const* __restrict__ tp, int nterms, uint64_t i,
                                             uint64_t step, float (&acc0)[8], float (&acc1)[8]) {
  load8(tp[0] + i, acc0);
  load8(tp[0] + i + step, acc1);
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    acc0[k] = 0.0f + acc0[k];
    acc1[k] = 0.0f + acc1[k];
  }
  for (int t = 1; t < nterms; ++t) {
    float v0[8], v1[8];
    load8(tp[t] + i, v0);
    load8(tp[t] + i + step, v1);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      acc0[k] += v0[k];
      acc1[k] += v1[k];
    }
  }
}

template <class TOut>
__device__ __forceinline__ void finish8(TOut* __restrict__ dst, uint64_t i, float beta, float (&acc)[8]) {
  if (beta != 0.0f) {
    float o[8];
    load8_coherent(dst + i, o);
#pragma unroll
    for (int k = 0; k < 8; ++k) acc[k] = fmaf(beta, o[k], acc[k]);
  }
  store8(dst + i, acc);
}

// dst[a, b) = beta*dst + sum of the terms, whole CTA, two 8-element groups per
// thread per iteration (their loads are issued together).
template <class TIn, class TOut>
__device__ __forceinline__ void reduce_range(TOut* __restrict__ dst, const TIn* const* __restrict__ tp, int nterms,
                                             uint64_t a, uint64_t b, float beta, uint32_t tid, uint32_t nthr) {
  uint64_t align = reinterpret_cast<uint64_t>(dst + a);
  for (int t = 0; t < nterms; ++t) align |= reinterpret_cast<uint64_t>(tp[t] + a);
  uint64_t i = a;
  if ((align & 15) == 0 && nterms > 0) {
    const uint64_t vend = a + ((b - a) & ~uint64_t(7));
    const uint64_t step = static_cast<uint64_t>(nthr) * 8;
    for (i = a + tid * 8; i + step < vend; i += 2 * step) {
      float acc0[8], acc1[8];
      sum_terms8x2(tp, nterms, i, step, acc0, acc1);
      if (beta != 0.0f) {  // both accumulator loads in flight before either store
        float o0[8], o1[8];
        load8_coherent(dst + i, o0);
        load8_coherent(dst + i + step, o1);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          acc0[k] = fmaf(beta, o0[k], acc0[k]);
          acc1[k] = fmaf(beta, o1[k], acc1[k]);
        }
      }
      store8(dst + i, acc0);
      store8(dst + i + step, acc1);
    }
    if (i < vend) {
      float acc[8];
      sum_terms8(tp, nterms, i, acc);
      finish8(dst, i, beta, acc);
    }
    i = vend;
  }
  for (uint64_t e = i + tid; e < b; e += nthr) {  // tail / unaligned
    float acc = 0.0f;
    for (int t = 0; t < nterms; ++t) acc += Cvt<TIn>::to(tp[t][e]);
    if (beta != 0.0f) acc = fmaf(beta, Cvt<TOut>::to(dst[e]), acc);
    dst[e] = Cvt<TOut>::from(acc);
  }
}
template <class TIn, class TOut>
__device__ __forceinline__ void reduce_range(TOut* __restrict__ dst, const TIn* const* __restrict__ tp, int nterms,
                                             uint64_t a, uint64_t b, float beta) {
  reduce_range<TIn, TOut>(dst, tp, nterms, a, b, beta, threadIdx.x, blockDim.x);
}

// reduce_range for a fan-out segment: the terms' sum is formed once per
// 8-element group and read-modify-written into each of the nd accumulators.
template <class TIn, class TOut>
__device__ __forceinline__ void reduce_range_fan(TOut* const* __restrict__ dl, int nd, const TIn* const* __restrict__ tp,
                                              int nterms, uint64_t a, uint64_t b, float beta, uint32_t tid,
                                              uint32_t nthr) {
  uint64_t align = 0;
  for (int d = 0; d < nd; ++d) align |= reinterpret_cast<uint64_t>(dl[d] + a);
  for (int t = 0; t < nterms; ++t) align |= reinterpret_cast<uint64_t>(tp[t] + a);
  uint64_t i = a;
  if ((align & 15) == 0 && nterms > 0) {
    const uint64_t vend = a + ((b - a) & ~uint64_t(7));
    const uint64_t step = static_cast<uint64_t>(nthr) * 8;
    for (i = a + tid * 8; i + step < vend; i += 2 * step) {
      float acc0[8], acc1[8];
      sum_terms8x2(tp, nterms, i, step, acc0, acc1);
      for (int d = 0; d < nd; ++d) {
        TOut* dst = dl[d];
        float o0[8], o1[8];
        if (beta != 0.0f) {
          load8_coherent(dst + i, o0);
          load8_coherent(dst + i + step, o1);
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            o0[k] = fmaf(beta, o0[k], acc0[k]);
            o1[k] = fmaf(beta, o1[k], acc1[k]);
          }
        } else {
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            o0[k] = acc0[k];
            o1[k] = acc1[k];
          }
        }
        store8(dst + i, o0);
        store8(dst + i + step, o1);
      }
    }
    if (i < vend) {
      float acc[8];
      sum_terms8(tp, nterms, i, acc);
      for (int d = 0; d < nd; ++d) {
        float o[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) o[k] = acc[k];
        finish8(dl[d], i, beta, o);
      }
    }
    i = vend;
  }
  for (uint64_t e = i + tid; e < b; e += nthr) {  // tail / unaligned
    float acc = 0.0f;
    for (int t = 0; t < nterms; ++t) acc += Cvt<TIn>::to(tp[t][e]);
    for (int d = 0; d < nd; ++d) {
      const float v = beta != 0.0f ? fmaf(beta, Cvt<TOut>::to(dl[d][e]), acc) : acc;
      dl[d][e] = Cvt<TOut>::from(v);
    }
  }
}
template <class TIn, class TOut>
__device__ __forceinline__ void reduce_range_fan(TOut* const* __restrict__ dl, int nd, const TIn* const* __restrict__ tp,
                                              int nterms, uint64_t a, uint64_t b, float beta) {
  reduce_range_fan<TIn, TOut>(dl, nd, tp, nterms, a, b, beta, threadIdx.x, blockDim.x);
}

struct ReduceLen {
  __device__ uint64_t operator()(const ReduceSeg& s) const { return s.nelem; }
};

// Remote single-term chunks (the gradient-return pulls of the dynamic
// partition) stream their term through a ring of shared-memory stages filled by
// TMA bulk loads from the peer (one issuing thread, kRedRingBytes in flight per
// CTA), so NVLink latency is hidden by the ring rather than by per-thread loads;
// every thread reads its 8-element groups from smem and does the fp32
// read-modify-write of the local accumulator (its dst loads are issued before
// it waits for the stage). Everything else uses reduce_range.
constexpr uint32_t kRedSub = 4096;                 // elements per stage
constexpr uint32_t kRedRingBytes = 64 * 1024;      // per CTA
template <class TIn>
__host__ __device__ constexpr int red_stages() { return static_cast<int>(kRedRingBytes / (kRedSub * sizeof(TIn))); }

template <class TIn, class TOut>
struct RedRing {
  uint64_t* full;            // [stages] mbarriers (shared)
  unsigned char* mem;        // stages x kRedSub x sizeof(TIn) (dynamic shared)
  uint32_t used;             // stages consumed so far (uniform across the CTA)

  __device__ void issue(const TIn* src, uint32_t k, uint32_t nelem) {  // sub-load k of the ring's lifetime
    constexpr int S = red_stages<TIn>();
    const int st = k % S;
    const uint32_t bytes = nelem * sizeof(TIn);
    mbar_expect(&full[st], bytes);
    bulk_g2s(mem + st * (kRedSub * sizeof(TIn)), src, bytes, &full[st]);
  }

  // dl[d][off, off + n) = beta*dl[d] + term[0, n) for each of the nd accumulators
  // (a fan-out segment): the staged term is read from smem once per accumulator.
  __device__ __forceinline__ void run_fan(TOut* const* dl, int nd, uint64_t off, const TIn* __restrict__ term, uint64_t n,
                                       float beta) {
    constexpr int S = red_stages<TIn>();
    const uint32_t nsub = static_cast<uint32_t>((n + kRedSub - 1) / kRedSub);
    auto sub_len = [&](uint32_t i) {
      const uint64_t r = n - static_cast<uint64_t>(i) * kRedSub;
      return static_cast<uint32_t>(r < kRedSub ? r : kRedSub);
    };
    if (threadIdx.x == 0)
      for (uint32_t i = 0; i < nsub && i < static_cast<uint32_t>(S); ++i)
        issue(term + static_cast<uint64_t>(i) * kRedSub, used + i, sub_len(i));
    for (uint32_t i = 0; i < nsub; ++i) {
      const uint32_t k = used + i, len = sub_len(i);
      const int st = k % S;
      const uint64_t base = off + static_cast<uint64_t>(i) * kRedSub;
      const TIn* T = reinterpret_cast<const TIn*>(mem + st * (kRedSub * sizeof(TIn)));
      mbar_wait(&full[st], (k / S) & 1u);
      for (uint32_t j = threadIdx.x * 8; j < len; j += blockDim.x * 8) {
        float acc[8];
        load8_coherent(T + j, acc);
        for (int d = 0; d < nd; ++d) {
          TOut* p = dl[d] + base + j;
          float o[8];
          if (beta != 0.0f) {
            load8_coherent(p, o);
#pragma unroll
            for (int q = 0; q < 8; ++q) o[q] = fmaf(beta, o[q], 0.0f + acc[q]);
          } else {
#pragma unroll
            for (int q = 0; q < 8; ++q) o[q] = 0.0f + acc[q];
          }
          store8(p, o);
        }
      }
      __syncthreads();  // stage st fully read
      if (threadIdx.x == 0 && i + S < nsub) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        issue(term + static_cast<uint64_t>(i + S) * kRedSub, k + S, sub_len(i + S));
      }
    }
    used += nsub;
  }

  // dst[0, n) = beta*dst + term[0, n); n a multiple of 8, 16-B aligned pointers
  __device__ void run(TOut* __restrict__ dst, const TIn* __restrict__ term, uint64_t n, float beta) {
    constexpr int S = red_stages<TIn>();
    const uint32_t nsub = static_cast<uint32_t>((n + kRedSub - 1) / kRedSub);
    auto sub_len = [&](uint32_t i) {
      const uint64_t r = n - static_cast<uint64_t>(i) * kRedSub;
      return static_cast<uint32_t>(r < kRedSub ? r : kRedSub);
    };
    if (threadIdx.x == 0)
      for (uint32_t i = 0; i < nsub && i < static_cast<uint32_t>(S); ++i)
        issue(term + static_cast<uint64_t>(i) * kRedSub, used + i, sub_len(i));
    for (uint32_t i = 0; i < nsub; ++i) {
      const uint32_t k = used + i, len = sub_len(i);
      const int st = k % S;
      TOut* d = dst + static_cast<uint64_t>(i) * kRedSub;
      const TIn* T = reinterpret_cast<const TIn*>(mem + st * (kRedSub * sizeof(TIn)));
      // the first group's accumulator load goes out before the stage wait
      const uint32_t j0 = threadIdx.x * 8;
      float o[8];
      if (beta != 0.0f && j0 < len) load8_coherent(d + j0, o);
      mbar_wait(&full[st], (k / S) & 1u);
      for (uint32_t j = j0; j < len; j += blockDim.x * 8) {
        if (j != j0 && beta != 0.0f) load8_coherent(d + j, o);
        float acc[8];
        load8_coherent(T + j, acc);
#pragma unroll
        for (int q = 0; q < 8; ++q) acc[q] = beta != 0.0f ? fmaf(beta, o[q], 0.0f + acc[q]) : 0.0f + acc[q];
        store8(d + j, acc);
      }
      __syncthreads();  // stage st fully read
      if (threadIdx.x == 0 && i + S < nsub) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        issue(term + static_cast<uint64_t>(i + S) * kRedSub, k + S, sub_len(i + S));
      }
    }
    used += nsub;
  }
};

// FAN: the launch has fan-out segments (ndst > 1); every segment then takes the
// fan-out code path (a separate instantiation keeps the single-accumulator
// kernel's register allocation untouched).
template <class TIn, class TOut, int MODE, bool FAN>
__global__ void __launch_bounds__(512, 2) reduce_segments_kernel(const ReduceSeg* __restrict__ segs, int nseg,
                                                              const void* const* __restrict__ terms,
                                                              Partition part, float beta, SyncArgs sync) {
  constexpr int S = red_stages<TIn>();
  extern __shared__ __align__(128) unsigned char red_mem[];
  __shared__ __align__(8) uint64_t full[S];
  RedRing<TIn, TOut> ring{full, red_mem, 0};
  if constexpr (MODE == kPartDynamic) {
    if (threadIdx.x == 0) {
      for (int i = 0; i < S; ++i) mbar_init(&full[i]);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    // (run_shares syncs the CTA before the first body)
  }
  run_shares<MODE>(segs, nseg, part, sync, ReduceLen{},
                   [&](const ReduceSeg& sg, uint64_t a, uint64_t b, bool remote) {
    const TIn* const* tp = reinterpret_cast<const TIn* const*>(terms + sg.term0);
    TOut* dst = static_cast<TOut*>(sg.dst);
    if constexpr (FAN) {  // fan-out: one term read, several accumulators
      // the side array holds the accumulator pointers too (written as const void*)
      TOut* const* dl = reinterpret_cast<TOut* const*>(const_cast<void* const*>(terms + sg.dst0));
      if constexpr (MODE == kPartDynamic) {
        if (remote && sg.nterms == 1 && part.ring) {
          const uint64_t n8 = (b - a) & ~uint64_t(7);
          uint64_t al = reinterpret_cast<uint64_t>(tp[0] + a);
          for (int d = 0; d < sg.ndst; ++d) al |= reinterpret_cast<uint64_t>(dl[d] + a);
          if ((al & 15) == 0 && n8 > 0) {
            ring.run_fan(dl, sg.ndst, a, tp[0] + a, n8, beta);
            if (a + n8 < b) reduce_range_fan<TIn, TOut>(dl, sg.ndst, tp, 1, a + n8, b, beta);
            return;
          }
        }
      }
      reduce_range_fan<TIn, TOut>(dl, sg.ndst, tp, sg.nterms, a, b, beta);
      return;
    }
    if constexpr (MODE == kPartDynamic) {
      if (remote && sg.nterms == 1 && part.ring) {  // (remote chunks exist => the ring smem was allocated)
        const uint64_t n8 = (b - a) & ~uint64_t(7);
        const uint64_t al = reinterpret_cast<uint64_t>(dst + a) | reinterpret_cast<uint64_t>(tp[0] + a);
        if ((al & 15) == 0 && n8 > 0) {
          ring.run(dst + a, tp[0] + a, n8, beta);
          if (a + n8 < b) reduce_range<TIn, TOut>(dst, tp, 1, a + n8, b, beta);
          return;
        }
      }
    }
    reduce_range<TIn, TOut>(dst, tp, sg.nterms, a, b, beta);
  });
}

// Streaming gradient return (dynamic partition, the default): one continuous
// stage ring per CTA across chunk boundaries. Thread 0 is the producer: it
// claims chunks (the same two queues, static first chunks and claim prefetch
// as run_shares) and turns them into a sequence of work items, one per ring
// slot:
//   staged : <= kRedSub elements of a remote single-term chunk, TMA-loaded from
//            the peer into the slot's stage (the slot's mbarrier completes on
//            the bytes);
//   direct : a whole local (or multi-term / unaligned) chunk, reduced straight
//            from global memory by reduce_range (the slot's mbarrier completes
//            on a plain arrive);
//   end    : no more work.
// Every thread consumes the items in order; after item k the producer refills
// its slot with item k + S. So while the CTA reduces one item, the next S-1
// items' loads are in flight whatever chunk they belong to: the NVLink round
// trip is paid once per CTA, not once per chunk (the per-chunk ring of
// RedRing drained at each chunk boundary). Item metadata is written by thread
// 0 at least one __syncthreads before it is read (S >= 2).
enum : uint32_t { kItStaged = 0, kItDirect = 1, kItEnd = 2 };
struct RedItem {
  uint32_t seg, kind;
  uint64_t a, b;  // elements [a, b) of segment seg
};
struct RedProducer {  // thread 0's state (shared memory keeps it out of the consumers' registers)
  Claimer cl;
  unsigned long long arr;
  uint32_t seg;
  uint64_t pa, pmid, pb;  // staged [pa, pmid), then a direct tail [pmid, pb)
  int more, arrived, use_first;
  uint32_t nch, nrem;
};

template <class TIn, class TOut, bool FAN>
__global__ void __launch_bounds__(512, 2) reduce_segments_stream_kernel(const ReduceSeg* __restrict__ segs, int nseg,
                                                            const void* const* __restrict__ terms, Partition part,
                                                            float beta, SyncArgs sync) {
  constexpr int S = red_stages<TIn>();
  static_assert(S >= 2, "items are published one __syncthreads ahead");
  extern __shared__ __align__(128) unsigned char red_mem[];
  __shared__ __align__(8) uint64_t full[S];
  __shared__ RedItem item[S];
  __shared__ CtaSync cs;
  __shared__ RedProducer pr;
  griddep_wait();
  if (blockIdx.x == 0 && threadIdx.x < 32) {
    post_peers_warp(sync, 0);
    __syncwarp();
  }
  auto arrive = [&]() {
    if (!pr.arrived) {
      cta_arrive_finish(sync, cs, pr.arr);
      pr.arrived = 1;
    }
  };
  // thread 0: write item k into its slot (claiming chunks as needed)
  auto produce = [&](uint32_t k) {
    const int st = k % S;
    RedItem& it = item[st];
    while (true) {
      if (pr.pa < pr.pmid) {  // next stage of the current remote chunk
        const ReduceSeg& sg = segs[pr.seg];
        const TIn* tp = reinterpret_cast<const TIn*>(terms[sg.term0]);
        const uint64_t n = min(static_cast<uint64_t>(kRedSub), pr.pmid - pr.pa);
        it = RedItem{pr.seg, kItStaged, pr.pa, pr.pa + n};
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // the slot's generic reads are done
        mbar_expect(&full[st], static_cast<uint32_t>(n * sizeof(TIn)));
        bulk_g2s(red_mem + st * (kRedSub * sizeof(TIn)), tp + pr.pa, static_cast<uint32_t>(n * sizeof(TIn)),
                 &full[st]);
        pr.pa += n;
        return;
      }
      if (pr.pmid < pr.pb) {  // direct remainder of the current chunk
        it = RedItem{pr.seg, kItDirect, pr.pmid, pr.pb};
        pr.pa = pr.pmid = pr.pb;  // the chunk is done (pa too: [pa, pmid) must stay empty)
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&full[st])) : "memory");
        return;
      }
      if (!pr.more) {
        it.kind = kItEnd;
        return;
      }
      uint32_t c;
      int rq;
      if (pr.use_first) {
        pr.use_first = 0;
        c = pr.cl.first;
        rq = pr.cl.q;
      } else {
        arrive();
        c = pr.cl.next(part, sync, cs.e, &rq);
        if (c == kNoChunk) {
          pr.more = 0;
          continue;
        }
      }
      if (c == kNoChunk) continue;
      const uint2 t = (rq ? part.rchunks : part.chunks)[c];
      const ReduceSeg& sg = segs[t.x];
      const uint64_t cu = rq ? part.rchunk : part.chunk;
      const uint64_t a = static_cast<uint64_t>(t.y & 0xffffffu) * cu;
      const uint64_t b = min(a + ((t.y >> 24) + 1) * cu, sg.nelem);
      if (rq) {
        arrive();
        if (!sync_wait_lane(sync, cs)) continue;  // timed out: claimed, not executed
        ++pr.nrem;
      }
      ++pr.nch;
      pr.seg = t.x;
      pr.pa = pr.pmid = a;
      pr.pb = b;
      if ((rq || part.stage_local) && sg.nterms == 1 && part.ring) {
        uint64_t al = reinterpret_cast<uint64_t>(static_cast<const TIn*>(terms[sg.term0]) + a);
        if constexpr (FAN) {
          for (int d = 0; d < sg.ndst; ++d) al |= reinterpret_cast<uint64_t>(static_cast<const TOut*>(terms[sg.dst0 + d]) + a);
        } else {
          al |= reinterpret_cast<uint64_t>(static_cast<const TOut*>(sg.dst) + a);
        }
        if ((al & 15) == 0) pr.pmid = a + ((b - a) & ~uint64_t(7));
      }
    }
  };
  if (threadIdx.x == 0) {
    trace_at(sync, kTrEntry);
    pr.arr = cta_arrive_issue(sync);
    pr.arrived = 0;
    pr.nch = pr.nrem = 0;
    for (int i = 0; i < S; ++i) mbar_init(&full[i]);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    pr.cl.init(part);
    pr.more = !pr.cl.done();
    pr.use_first = pr.more;
    pr.pa = pr.pmid = pr.pb = 0;
    if (pr.more) pr.cl.issue(part, sync, pr.cl.first);  // the claim after the static chunk, in flight
    for (uint32_t k = 0; k < static_cast<uint32_t>(S); ++k) produce(k);
  }
  __syncthreads();
  for (uint32_t k = 0;; ++k) {
    const int st = k % S;
    const RedItem it = item[st];
    if (it.kind == kItEnd) break;
    const ReduceSeg sg = segs[it.seg];
    const TIn* const* tp = reinterpret_cast<const TIn* const*>(terms + sg.term0);
    if (it.kind == kItStaged) {
      const TIn* T = reinterpret_cast<const TIn*>(red_mem + st * (kRedSub * sizeof(TIn)));
      const uint32_t len = static_cast<uint32_t>(it.b - it.a);
      if constexpr (FAN) {
        TOut* const* dl = reinterpret_cast<TOut* const*>(const_cast<void* const*>(terms + sg.dst0));
        mbar_wait(&full[st], (k / S) & 1u);
        for (uint32_t j = threadIdx.x * 8; j < len; j += blockDim.x * 8) {
          float acc[8];
          load8_coherent(T + j, acc);
          for (int d = 0; d < sg.ndst; ++d) {
            TOut* p = dl[d] + it.a + j;
            float o[8];
            if (beta != 0.0f) {
              load8_coherent(p, o);
#pragma unroll
              for (int q = 0; q < 8; ++q) o[q] = fmaf(beta, o[q], 0.0f + acc[q]);
            } else {
#pragma unroll
              for (int q = 0; q < 8; ++q) o[q] = 0.0f + acc[q];
            }
            store8(p, o);
          }
        }
      } else {
        TOut* d = static_cast<TOut*>(sg.dst) + it.a;
        // the first group's accumulator load goes out before the stage wait
        const uint32_t j0 = threadIdx.x * 8;
        float o[8];
        if (beta != 0.0f && j0 < len) load8_coherent(d + j0, o);
        mbar_wait(&full[st], (k / S) & 1u);
        for (uint32_t j = j0; j < len; j += blockDim.x * 8) {
          if (j != j0 && beta != 0.0f) load8_coherent(d + j, o);
          float acc[8];
          load8_coherent(T + j, acc);
#pragma unroll
          for (int q = 0; q < 8; ++q) acc[q] = beta != 0.0f ? fmaf(beta, o[q], 0.0f + acc[q]) : 0.0f + acc[q];
          store8(d + j, acc);
        }
      }
    } else {
      mbar_wait(&full[st], (k / S) & 1u);  // (a plain arrive: keeps the slot's phases in step)
      if constexpr (FAN) {
        TOut* const* dl = reinterpret_cast<TOut* const*>(const_cast<void* const*>(terms + sg.dst0));
        reduce_range_fan<TIn, TOut>(dl, sg.ndst, tp, sg.nterms, it.a, it.b, beta);
      } else {
        reduce_range<TIn, TOut>(static_cast<TOut*>(sg.dst), tp, sg.nterms, it.a, it.b, beta);
      }
    }
    __syncthreads();  // slot st fully read
    if (threadIdx.x == 0) {
      if (k == 0) trace_at(sync, kTrFirst);
      produce(k + S);
    }
  }
  griddep_launch_dependents();  // this CTA's work is done: the next op may take its slot
  if (threadIdx.x == 0) {
    arrive();
    trace_at(sync, kTrDone);
    launch_end_lane(sync, cs);
    trace_at(sync, kTrExit);
    trace_val(sync, kTrChunks, pr.nch);
    trace_val(sync, kTrRemote, pr.nrem);
  }
}

// ---- fused 1F1B-paired step ----------------------------------------------------
// One launch runs a forward and a gradient return at once (the pair a pipeline
// schedule call issues: microbatch k+1's activations in, microbatch k's
// gradient back), warp-specialised inside each CTA: lane 0 of warp 0 drives the
// TMA copy ring of the forward (tma_copy_lane), warps 1-15 run the gradient
// return with LDG.128 loads (remote terms too), synchronised among themselves
// by a named barrier. Each side keeps its own claim queues, arrival counter,
// pads and end-of-launch protocol (op kinds 0 and 1), so the pair is exactly
// one forward op and one backward op for the peers. Unlike two concurrent
// kernels, nothing depends on both grids being co-resident: both halves of
// every CTA are resident together by construction.
constexpr uint32_t kPairedThreads = 512, kPairedRedThreads = kPairedThreads - 32;

__device__ __forceinline__ void group_sync(uint32_t nthr) {
  asm volatile("bar.sync 1, %0;" ::"r"(nthr) : "memory");
}

template <class TIn, class TOut, bool FAN>
__device__ __forceinline__ void reduce_group_loop(const ReduceSeg* __restrict__ segs, const void* const* __restrict__ terms,
                                                  const Partition& part, float beta, const SyncArgs& sync, CtaSync& cs,
                                                  uint32_t tid, uint32_t nthr) {
  __shared__ Claimer cl;
  __shared__ uint32_t cur;
  __shared__ int cur_remote;
  __shared__ uint32_t nch, nrem;  // trace counters (HB_TRACE)
  unsigned long long arr = 0;
  if (tid == 0) {
    trace_at(sync, kTrEntry);
    arr = cta_arrive_issue(sync);
    nch = nrem = 0;
    cl.init(part);
    cur = cl.done() ? kNoChunk : cl.first;
    cur_remote = cl.q;
    if (!cl.done()) cl.issue(part, sync, cl.first);
    if (cur != kNoChunk && cl.q == 1) {
      cta_arrive_finish(sync, cs, arr);
      arr = ~0ull;
      sync_wait_lane(sync, cs);
    }
  }
  group_sync(nthr);
  bool first = true;
  while (true) {
    const uint32_t c = cur;
    if (c != kNoChunk && (!cur_remote || cs.ok)) {
      const uint2 t = (cur_remote ? part.rchunks : part.chunks)[c];
      const ReduceSeg sg = segs[t.x];
      const uint64_t cu = cur_remote ? part.rchunk : part.chunk;
      const uint64_t a = static_cast<uint64_t>(t.y & 0xffffffu) * cu, e = a + ((t.y >> 24) + 1) * cu;
      const uint64_t b = e < sg.nelem ? e : sg.nelem;
      const TIn* const* tp = reinterpret_cast<const TIn* const*>(terms + sg.term0);
      if constexpr (FAN) {
        TOut* const* dl = reinterpret_cast<TOut* const*>(const_cast<void* const*>(terms + sg.dst0));
        reduce_range_fan<TIn, TOut>(dl, sg.ndst, tp, sg.nterms, a, b, beta, tid, nthr);
      } else {
        reduce_range<TIn, TOut>(static_cast<TOut*>(sg.dst), tp, sg.nterms, a, b, beta, tid, nthr);
      }
      if (tid == 0 && sync.trace) {
        ++nch;
        nrem += cur_remote != 0;
      }
    }
    group_sync(nthr);
    if (tid == 0) {
      if (first) trace_at(sync, kTrFirst);
      if (first && arr != ~0ull) cta_arrive_finish(sync, cs, arr);
      first = false;
      int rq = 0;
      cur = cl.next(part, sync, cs.e, &rq);
      cur_remote = rq;
      if (cur != kNoChunk && rq) sync_wait_lane(sync, cs);
    }
    group_sync(nthr);
    if (cur == kNoChunk) break;
  }
  if (tid == 0) {
    trace_at(sync, kTrDone);
    launch_end_lane(sync, cs);
    trace_at(sync, kTrExit);
    trace_val(sync, kTrChunks, nch);
    trace_val(sync, kTrRemote, nrem);
  }
}

template <class TIn, class TOut, bool FAN>
__global__ void __launch_bounds__(kPairedThreads, 2)
    paired_step_kernel(const CopySeg* __restrict__ csegs, Partition cpart, SyncArgs csync,
                       const ReduceSeg* __restrict__ rsegs, const void* const* __restrict__ terms, Partition rpart,
                       float beta, SyncArgs rsync) {
  extern __shared__ __align__(128) unsigned char stage_mem[];
  __shared__ __align__(8) uint64_t full[3];
  __shared__ CtaSync ccs, rcs;
  griddep_wait();
  if (blockIdx.x == 0 && threadIdx.x < 32) {  // "started" of both ops to every peer
    post_peers_warp(csync, 0);
    post_peers_warp(rsync, 0);
    __syncwarp();
  }
  if (threadIdx.x < 32) {
    if (threadIdx.x == 0) tma_copy_lane<3, 32 * 1024>(csegs, cpart, csync, stage_mem, full, ccs);
  } else {
    reduce_group_loop<TIn, TOut, FAN>(rsegs, terms, rpart, beta, rsync, rcs, threadIdx.x - 32, kPairedRedThreads);
  }
}

}  // namespace

int device_sm_count() {
  int dev = 0, n = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n;
}

int copy_blocks_per_sm(int threads) {
  int n = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, copy_segments_kernel<kPartContiguous>, threads, 0);
  return n > 0 ? n : 1;
}

template <int ST, uint32_t SB>
static int tma_occupancy() {
  static PerDeviceOnce once;
  static int n = 1;
  int dev = 0;
  cudaGetDevice(&dev);
  once(dev, [] {
    const int smem = ST * SB;
    cudaFuncSetAttribute(copy_segments_tma_kernel<ST, SB>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(copy_segments_tma_kernel<ST, SB>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    int k = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&k, copy_segments_tma_kernel<ST, SB>, 32, smem);
    n = k < 1 ? 1 : k;  // identical devices: one value serves them all
  });
  return n;
}

int tma_blocks_per_sm(uint64_t chunk) {
  if (chunk == 16 * 1024) return tma_occupancy<6, 16 * 1024>();
  if (chunk == 8 * 1024) return tma_occupancy<8, 8 * 1024>();
  return tma_occupancy<3, 32 * 1024>();
}

uint64_t tma_chunk_bytes(int kib) { return (kib == 16 || kib == 8) ? kib * 1024ull : 32 * 1024ull; }

// Every boundary kernel goes out with programmatic stream serialisation (PDL,
// launch_protocol.cuh); HB_PDL=0 launches them plainly (A/B knob).
template <class... KArgs, class... Args>
static void launch_pdl(void (*k)(KArgs...), int grid, int block, size_t smem, cudaStream_t st, Args... args) {
  static const bool env_pdl = [] {
    const char* v = std::getenv("HB_PDL");
    return !(v && v[0] == '0');
  }();
  // SyncArgs (the last argument) says whether this exec may overlap launches
  const bool pdl = env_pdl && std::get<sizeof...(Args) - 1>(std::make_tuple(args...)).pdl;
  cudaLaunchConfig_t lc{};
  lc.gridDim = dim3(grid);
  lc.blockDim = dim3(block);
  lc.dynamicSmemBytes = smem;
  lc.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  lc.attrs = at;
  lc.numAttrs = pdl ? 1 : 0;
  cudaLaunchKernelEx(&lc, k, args...);
}

template <class TIn, class TOut, bool FAN>
static int launch_paired_t(const CopySeg* csegs, const Partition& cpart, const SyncArgs& csync,
                           const ReduceSeg* rsegs, const void* const* terms, const Partition& rpart, float beta,
                           const SyncArgs& rsync, int grid, cudaStream_t st) {
  static PerDeviceOnce once;
  int dev = 0;
  cudaGetDevice(&dev);
  once(dev, [] {
    cudaFuncSetAttribute(paired_step_kernel<TIn, TOut, FAN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         3 * 32 * 1024);
    cudaFuncSetAttribute(paired_step_kernel<TIn, TOut, FAN>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  });
  // (PDL: the next step's CTAs may be scheduled once every CTA's copy lane is done)
  launch_pdl(paired_step_kernel<TIn, TOut, FAN>, grid, static_cast<int>(kPairedThreads), 3 * 32 * 1024, st, csegs,
             cpart, csync, rsegs, terms, rpart, beta, rsync);
  return cudaGetLastError() == cudaSuccess ? 0 : 5;
}

int launch_paired(const CopySeg* csegs, Partition cpart, const SyncArgs& csync, const ReduceSeg* rsegs,
                  const void* const* terms, Partition rpart, int in_dtype, int out_dtype, float beta,
                  const SyncArgs& rsync, int grid, void* stream) {
  // A fan-out gradient return (some run writes several TP replicas) needs the
  // full 1024 threads per SM of its own launch: fused it measured 10% slower
  // than forward-then-backward at N=1 and 8% at N=4 (C3), so it is not fused.
  if (cpart.mode != kPartTma || cpart.chunk != 32 * 1024 || rpart.mode != kPartDynamic || rpart.fan) return 1;
  auto st = static_cast<cudaStream_t>(stream);
  int rc = 2;
#define HB_PAIRED(TI, TO) rc = launch_paired_t<TI, TO, false>(csegs, cpart, csync, rsegs, terms, rpart, beta, rsync, grid, st)
  switch (in_dtype * 4 + out_dtype) {
    case kBF16 * 4 + kFP32: HB_PAIRED(__nv_bfloat16, float); break;
    case kBF16 * 4 + kBF16: HB_PAIRED(__nv_bfloat16, __nv_bfloat16); break;
    case kFP32 * 4 + kFP32: HB_PAIRED(float, float); break;
    default: break;
  }
#undef HB_PAIRED
  return rc;
}

void launch_copy(const CopySeg* segs, int nseg, Partition part, const SyncArgs& sync, LaunchCfg cfg,
                 void* stream) {
  auto st = static_cast<cudaStream_t>(stream);
  if (part.mode == kPartTma) {
    tma_blocks_per_sm(part.chunk);
    if (part.chunk == 16 * 1024)
      launch_pdl(copy_segments_tma_kernel<6, 16 * 1024>, cfg.grid, 32, 6 * 16 * 1024, st, segs, nseg, part, sync);
    else if (part.chunk == 8 * 1024)
      launch_pdl(copy_segments_tma_kernel<8, 8 * 1024>, cfg.grid, 32, 8 * 8 * 1024, st, segs, nseg, part, sync);
    else
      launch_pdl(copy_segments_tma_kernel<3, 32 * 1024>, cfg.grid, 32, 3 * 32 * 1024, st, segs, nseg, part, sync);
  } else if (part.mode == kPartInterleaved) {
    launch_pdl(copy_segments_kernel<kPartInterleaved>, cfg.grid, cfg.block, 0, st, segs, nseg, part, sync);
  } else if (part.mode == kPartDynamic) {
    launch_pdl(copy_segments_kernel<kPartDynamic>, cfg.grid, cfg.block, 0, st, segs, nseg, part, sync);
  } else {
    launch_pdl(copy_segments_kernel<kPartContiguous>, cfg.grid, cfg.block, 0, st, segs, nseg, part, sync);
  }
}

template <class TIn, class TOut, bool FAN>
static int red_ring_smem() {
  static PerDeviceOnce once;
  int dev = 0;
  cudaGetDevice(&dev);
  once(dev, [] {
    cudaFuncSetAttribute(reduce_segments_kernel<TIn, TOut, kPartDynamic, FAN>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, kRedRingBytes);
  });
  return static_cast<int>(kRedRingBytes);
}

// HB_RED_STREAM=0 selects the per-chunk ring kernel (reduce_segments_kernel)
// for the dynamic partition instead of the streaming one (A/B knob).
static bool red_stream() {
  static const bool on = [] {
    const char* v = std::getenv("HB_RED_STREAM");
    return !(v && v[0] == '0');
  }();
  return on;
}

template <class TIn, class TOut, bool FAN>
static int red_stream_smem() {
  static PerDeviceOnce once;
  int dev = 0;
  cudaGetDevice(&dev);
  once(dev, [] {
    cudaFuncSetAttribute(reduce_segments_stream_kernel<TIn, TOut, FAN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         kRedRingBytes);
  });
  return static_cast<int>(kRedRingBytes);
}

// HB_RED_CARVEOUT (A/B knob, percent of the unified L1/smem given to shared
// memory for the reduce kernels; 0 = driver default). Setting it to the TMA
// copy kernel's 100 avoids an L1/smem reconfiguration between a forward and a
// backward launch.
template <class TIn, class TOut, bool FAN>
static void red_carveout() {
  static PerDeviceOnce once;
  int dev = 0;
  cudaGetDevice(&dev);
  once(dev, [] {
    const char* v = std::getenv("HB_RED_CARVEOUT");
    const int pct = v && *v ? std::atoi(v) : 0;
    if (pct > 0) {
      cudaFuncSetAttribute(reduce_segments_kernel<TIn, TOut, kPartDynamic, FAN>,
                           cudaFuncAttributePreferredSharedMemoryCarveout, pct);
      cudaFuncSetAttribute(reduce_segments_kernel<TIn, TOut, kPartContiguous, FAN>,
                           cudaFuncAttributePreferredSharedMemoryCarveout, pct);
      cudaFuncSetAttribute(reduce_segments_kernel<TIn, TOut, kPartInterleaved, FAN>,
                           cudaFuncAttributePreferredSharedMemoryCarveout, pct);
    }
  });
}

template <class TIn, class TOut, bool FAN>
static void launch_reduce_f(const ReduceSeg* segs, int nseg, const void* const* terms, Partition part,
                            float beta, const SyncArgs& sync, int grid, int block, cudaStream_t st) {
  red_carveout<TIn, TOut, FAN>();
  if (part.mode == kPartInterleaved)
    launch_pdl(reduce_segments_kernel<TIn, TOut, kPartInterleaved, FAN>, grid, block, 0, st, segs, nseg, terms, part,
               beta, sync);
  else if (part.mode == kPartDynamic && red_stream() && part.ring && (part.rtotal_chunks || part.stage_local))
    // remote chunks to stage: the streaming ring (a launch with local chunks only
    // measured 3-7% faster in the per-chunk kernel at N=1, which skips the
    // per-item slot bookkeeping)
    launch_pdl(reduce_segments_stream_kernel<TIn, TOut, FAN>, grid, block, red_stream_smem<TIn, TOut, FAN>(), st, segs, nseg,
               terms, part, beta, sync);
  else if (part.mode == kPartDynamic)
    launch_pdl(reduce_segments_kernel<TIn, TOut, kPartDynamic, FAN>, grid, block,
               part.ring && part.rtotal_chunks ? red_ring_smem<TIn, TOut, FAN>() : 0, st, segs, nseg, terms, part,
               beta, sync);
  else
    launch_pdl(reduce_segments_kernel<TIn, TOut, kPartContiguous, FAN>, grid, block, 0, st, segs, nseg, terms, part,
               beta, sync);
}

template <class TIn, class TOut>
static void launch_reduce_t(const ReduceSeg* segs, int nseg, const void* const* terms, Partition part,
                            float beta, const SyncArgs& sync, int grid, int block, cudaStream_t st) {
  if (part.fan) launch_reduce_f<TIn, TOut, true>(segs, nseg, terms, part, beta, sync, grid, block, st);
  else launch_reduce_f<TIn, TOut, false>(segs, nseg, terms, part, beta, sync, grid, block, st);
}

template <class TIn, class TOut>
static int occ_t(int threads) {
  int n = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, reduce_segments_kernel<TIn, TOut, kPartContiguous, false>, threads, 0);
  return n > 0 ? n : 1;
}

#define HB_DISPATCH(IN, OUT, MACRO)                                   \
  switch ((IN) * 4 + (OUT)) {                                         \
    case kBF16 * 4 + kBF16: MACRO(__nv_bfloat16, __nv_bfloat16); break; \
    case kBF16 * 4 + kFP16: MACRO(__nv_bfloat16, __half); break;        \
    case kBF16 * 4 + kFP32: MACRO(__nv_bfloat16, float); break;         \
    case kFP16 * 4 + kBF16: MACRO(__half, __nv_bfloat16); break;        \
    case kFP16 * 4 + kFP16: MACRO(__half, __half); break;               \
    case kFP16 * 4 + kFP32: MACRO(__half, float); break;                \
    case kFP32 * 4 + kBF16: MACRO(float, __nv_bfloat16); break;         \
    case kFP32 * 4 + kFP16: MACRO(float, __half); break;                \
    case kFP32 * 4 + kFP32: MACRO(float, float); break;                 \
    default: break;                                                   \
  }

uint64_t red_ring_elems(int in_dtype) { return kRedRingBytes / dtype_size(in_dtype); }

int reduce_blocks_per_sm(int threads, int in_dtype, int out_dtype) {
  int n = 1;
#define HB_OCC(TI, TO) n = occ_t<TI, TO>(threads)
  HB_DISPATCH(in_dtype, out_dtype, HB_OCC)
#undef HB_OCC
  return n;
}

void launch_reduce(const ReduceSeg* segs, int nseg, const void* const* terms, Partition part, int in_dtype,
                   int out_dtype, float beta, const SyncArgs& sync, LaunchCfg cfg, void* stream) {
  auto st = static_cast<cudaStream_t>(stream);
#define HB_RED(TI, TO) launch_reduce_t<TI, TO>(segs, nseg, terms, part, beta, sync, cfg.grid, cfg.block, st)
  HB_DISPATCH(in_dtype, out_dtype, HB_RED)
#undef HB_RED
}

}  // namespace hb::dev
