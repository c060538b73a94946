// hetbridge — the in-kernel launch protocol shared by every boundary kernel
// (copy, reduce, fused projector): per-CTA arrival with the launch epoch,
// "started" posts to peers, lazy peer waits, and the end-of-launch contract.
// See boundary_kernels.cuh (SyncArgs) and DESIGN.md §4.
#pragma once

#include <cuda_runtime.h>

#include "kernels/boundary_kernels.cuh"

namespace hb::dev {
namespace {

__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// "+1" to this GPU's slot in every peer's pad (`word` = 0: started, kMaxGpus:
// finished pushing). Called by every thread of a warp: lane g posts to peer g,
// so the posts to several peers go out in parallel.
__device__ __forceinline__ void post_peers_warp(const SyncArgs& s, int word) {
  const int g = threadIdx.x & 31;
  if ((s.post_mask >> g) & 1u) {
    asm volatile("red.release.sys.global.add.u32 [%0], %1;" ::"l"(s.peer_pad[g] + word + s.my_gpu), "r"(1u)
                 : "memory");
  }
}

// Programmatic dependent launch (PDL). Boundary kernels are launched with
// programmatic stream serialisation: the next kernel of the stream may be
// scheduled as soon as every CTA of this one has called launch_dependents (we
// call it on entry, so each SM slot this grid frees takes a CTA of the next
// op at once), and griddepcontrol.wait blocks until this stream's previous
// grid has completed and its memory is visible. Every boundary kernel waits
// before its first global access (the "started" post, counters, buffers), so
// the launch protocol's meaning is unchanged: only launch latency and CTA
// scheduling overlap the previous kernel's tail. Without a programmatic
// dependency (first kernel, a producer launched without PDL) wait returns at once.
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void griddep_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// Trace stamp k of this CTA (no-op unless HB_TRACE set SyncArgs::trace).
__device__ __forceinline__ void trace_at(const SyncArgs& s, int k) {
  if (s.trace && blockIdx.x < kTraceMaxCtas) s.trace[blockIdx.x * kTraceWords + k] = global_ns();
}
__device__ __forceinline__ void trace_val(const SyncArgs& s, int k, unsigned long long v) {
  if (s.trace && blockIdx.x < kTraceMaxCtas) s.trace[blockIdx.x * kTraceWords + k] = v;
}
enum TraceSlot : int { kTrEntry = 0, kTrArrived = 1, kTrPeers = 2, kTrFirst = 3, kTrDone = 4, kTrExit = 5,
                       kTrChunks = 6, kTrRemote = 7 };

// Per-CTA view of the launch (shared memory).
struct CtaSync {
  uint32_t e;     // this launch's epoch (valid after cta_arrive_finish)
  uint32_t have;  // GPUs whose arrival at e this CTA has confirmed
  int ok;         // no timeout
};

// Bounded spin until *flag >= e; false on timeout (error word set). A peer
// may be at most one op ahead (it can finish op e only after every peer
// started e, so it cannot start e+2 before we start e+1): a count of e+2 or
// more is a protocol violation and is reported, not waited past.
__device__ __forceinline__ bool spin_until(const SyncArgs& s, const uint32_t* flag, uint32_t e) {
  const long long t0 = clock64();
  uint32_t v;
  while (static_cast<int32_t>((v = ld_acquire_sys(flag)) - e) < 0) {
    __nanosleep(64);
    if (static_cast<uint64_t>(clock64() - t0) > s.timeout_cycles) {
      atomicExch(s.err, kErrTimeout);
      return false;
    }
  }
  if (static_cast<int32_t>(v - e) > 1) {
    atomicExch(s.err, kErrOutOfTurn);
    return false;
  }
  return true;
}

// Start of a launch, one thread per CTA: count this CTA in (CTA 0's first
// warp posts "started" to every peer with post_peers_warp). Returns the raw arrival word; its latency overlaps
// the CTA's first (static, local) chunk and is consumed by cta_arrive_finish.
__device__ __forceinline__ unsigned long long cta_arrive_issue(const SyncArgs& s) {
  return atomicAdd(s.arrive, 1ull);
}

__device__ __forceinline__ void cta_arrive_finish(const SyncArgs& s, CtaSync& cs, unsigned long long old) {
  trace_at(s, kTrArrived);
  cs.e = static_cast<uint32_t>(old >> 32) + 1;
  cs.have = 0;
  cs.ok = 1;
  // last CTA in: advance the epoch, zero the arrivals (every CTA of this
  // launch has read the word; the next launch starts after this one ends)
  if ((old & 0xffffffffull) == gridDim.x - 1) atomicAdd(s.arrive, (1ull << 32) - gridDim.x);
}

// Wait (one thread per CTA) until every GPU in `peers` started op e: after
// that those peers' buffers of this op may be read (pull) or written (push).
// Each peer is confirmed once per CTA, so a CTA whose chunk reads only early
// peers proceeds while a late peer is still launching.
__device__ bool sync_wait_peers(const SyncArgs& s, CtaSync& cs, uint32_t peers) {
  uint32_t need = peers & s.wait_mask & ~cs.have;
  if (need) {
    while (need) {
      const int g = __ffs(need) - 1;
      need &= need - 1;
      if (!spin_until(s, s.pad + g, cs.e)) cs.ok = 0;
    }
    cs.have |= peers & s.wait_mask;
    if (cs.have == s.wait_mask) trace_at(s, kTrPeers);
  }
  return cs.ok != 0;
}
__device__ __forceinline__ bool sync_wait_lane(const SyncArgs& s, CtaSync& cs) {
  return sync_wait_peers(s, cs, s.wait_mask);
}

// End of a launch, one thread per CTA. CTA 0 confirms every peer started op e,
// so completion of op e implies every peer completed op e-1 (the buffer-reuse
// contract), whatever work this GPU had. Push mode: the last CTA done writing
// publishes "my writes into your buffers are done" and waits for every writer
// into this GPU.
__device__ void launch_end_lane(const SyncArgs& s, CtaSync& cs) {
  if (blockIdx.x == 0) sync_wait_lane(s, cs);
  if (!s.end_sync) return;
  __threadfence_system();  // this CTA's remote stores before "done"
  if (atomicAdd(s.fin, 1u) != gridDim.x - 1) return;
  *s.fin = 0;
  __threadfence_system();
  for (int g = 0; g < kMaxGpus; ++g)
    if ((s.post_mask >> g) & 1u) atomicAdd_system(s.peer_pad[g] + kMaxGpus + s.my_gpu, 1u);
  for (int g = 0; g < kMaxGpus; ++g)
    if ((s.wait_mask >> g) & 1u) spin_until(s, s.pad + kMaxGpus + g, cs.e);
}

}  // namespace
}  // namespace hb::dev
