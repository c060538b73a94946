// hetbridge — device-side descriptors shared by the runtime and the kernels.
#pragma once

#include <atomic>
#include <cstdint>

#include <vector_types.h>

namespace hb::dev {

enum Dtype : int { kBF16 = 0, kFP16 = 1, kFP32 = 2, kFP64 = 3, kI32 = 4 };

inline int dtype_size(int dt) { return (dt == kFP32 || dt == kI32) ? 4 : dt == kFP64 ? 8 : 2; }

// Work space: every segment occupies [w0, w0 + n) of a padded linear work
// space (bytes for copies, elements for reductions); w0 is rounded up to
// kQuantum so every CTA boundary is 16-B aligned inside each segment. CTA b
// owns the contiguous range [b*per_cta, (b+1)*per_cta) and starts at segment
// first_seg[b] (precomputed on the host): no per-chunk searches.
constexpr uint64_t kQuantum = 4096;

// One source run copied to up to kMaxFan destinations: the run is read once
// (HBM or NVLink) and stored to every destination (the TP/CP replicas that
// hold the same rows on this GPU in pull mode; every consumer of a local run
// in push mode).
constexpr int kMaxFan = 8;
//
// Gather runs (text-embedding lookup fused into the splice): when `ids` is set,
// the run is nbytes/row_bytes rows and row i comes from src + ids[i]*row_bytes
// (src = the embedding table, `vocab` rows); an id outside [0, vocab) sets the
// error word to kErrBadId and that row of the destination is left unwritten.
// Vocab-parallel tables (`shards` set): the table is split over the
// destination rank's TP group in `shard_rows`-row pieces, piece s at shards[s]
// (this GPU's or a peer's memory): row id comes from
// shards[id / shard_rows] + (id % shard_rows) * row_bytes.
struct CopySeg {
  const unsigned char* src;
  unsigned char* dst[kMaxFan];
  uint64_t nbytes;
  uint64_t w0;
  int32_t ndst;
  uint32_t row_bytes;  // gather runs only
  const int32_t* ids;  // nullptr: contiguous run
  int64_t vocab;
  uint32_t peers;      // GPUs this run reads (pull) or writes (push) besides this one
  uint32_t shard_rows;                   // vocab-parallel gather: rows per shard
  const unsigned char* const* shards;    // vocab-parallel gather: shard bases (nullptr: one table at src)
};
// kErrOutOfTurn: a peer's "started" count ran 2+ ops ahead of this launch's
// epoch, which the end-of-launch contract makes impossible unless the GPUs'
// op sequences diverged (the device analogue of simnet's out-of-turn check,
// R:core/src/simnet.cpp:202-207).
constexpr uint32_t kErrTimeout = 1, kErrBadId = 2, kErrOutOfTurn = 3;

// dst[i] = beta*dst[i] + sum_t term_t[i], fp32 accumulation, terms summed in
// order starting from +0.0f; term pointers live in a side array. A segment
// with ndst > 1 applies the same sum to several accumulators (the TP replicas
// of a source shard resident on this GPU): the terms are read once and each
// accumulator gets its own read-modify-write; the ndst accumulator pointers
// sit in the side array at dst0 (dst = the first of them).
struct ReduceSeg {
  void* dst;
  uint64_t nelem;
  uint64_t w0;
  int32_t nterms;
  int32_t term0;
  uint32_t peers;  // GPUs holding this segment's terms besides this one
  int32_t ndst;
  int32_t dst0;
  int32_t pad_;
};

// How a launch's work space is split over CTAs.
enum PartMode : int {
  kPartContiguous = 0,   // CTA b owns [b*per_cta, (b+1)*per_cta); first_seg[b] precomputed
  kPartInterleaved = 1,  // every CTA takes an equal quantum-aligned share of every segment
  kPartDynamic = 2,      // `chunk`-sized pieces handed out by an atomic counter (ctr[3]) in the
                         // order of a host-built table that advances every segment at the
                         // same fractional pace (local HBM and remote NVLink runs overlap)
  kPartTma = 3,          // dynamic chunks moved by TMA bulk copies through shared memory (copy kernel)
};

struct Partition {
  const int32_t* first_seg;  // [grid] (contiguous mode)
  uint64_t per_cta;          // work units per CTA (contiguous mode; multiple of kQuantum)
  int mode;
  uint32_t total_chunks;     // dynamic / TMA: chunks with no peer dependency
  uint64_t chunk;            // dynamic / TMA chunk size
  const uint2* chunks;       // [total_chunks] (segment, first unit | (units - 1) << 24), in hand-out order
  uint32_t rtotal_chunks;    // dynamic / TMA: chunks that read (pull) or write (push) a peer
  const uint2* rchunks;      // [rtotal_chunks]
  uint64_t rchunk;           // dynamic: remote chunk size (copy / TMA: = chunk)
  int remote_ctas;           // CTAs that start on the remote queue
  // Static first chunks: CTA b < remote_ctas starts on remote chunk b, CTA
  // b >= remote_ctas on local chunk b - remote_ctas (no claim round trip);
  // the rest is claimed from the queue counters.
  uint32_t lstatic;          // = min(grid - remote_ctas, total_chunks)
  uint32_t rstatic;          // = min(remote_ctas, rtotal_chunks)
  int ring;                  // reduce: stage remote single-term chunks through the TMA ring
  int prefetch_other;        // start the other queue's first claim near the current queue's end
  int fan;                   // reduce: some segment has ndst > 1 (fan-out kernel variant)
  int stage_local;           // reduce (streaming kernel): stage local single-term chunks through the ring too
  uint32_t claimers;         // dynamic / TMA: CTAs that take part in the queues (the partition's grid). A
                             // launch with a larger grid (the fused paired kernel) leaves the extra CTAs out,
                             // so the queue counters advance by the same amount in every launch of the kind.
};

// Cross-GPU epoch barrier over peer-mapped flag words. Every GPU of an exec
// group launches exactly one kernel per boundary op, so the per-exec op
// counts stay in lockstep: at its op e each GPU adds 1 to its slot in every
// peer's pad (so pad[g] = ops GPU g has started) and, before touching a
// peer's buffers, waits until pad[g] >= e for every peer g.
//
// Device counters (one 128-B line each, no false sharing between them):
//   arrive : (epoch << 32) | CTAs arrived in this launch. Each CTA adds 1 once
//            at start and learns e = epoch + 1; the last to arrive advances the
//            epoch and zeroes the arrivals (no CTA of this launch reads it after).
//   queue[2]: monotone 64-bit claim counters of the local / remote work queue.
//            Every claiming CTA claims until one claim fails in each non-empty queue, so
//            a launch advances queue q by exactly (total_q - static_q) + claimers and
//            launch e's chunk index is raw - (e-1)*advance + static_q: no reset,
//            no end-of-launch counter, no fence.
//   fin    : push mode only — CTAs done writing (last CTA posts "writes done").
//   err    : error word (1 = a flag wait timed out; the exec is unusable after).
constexpr int kMaxGpus = 32;
constexpr int kCtrLine = 32;  // u32 words per 128-B line
struct SyncArgs {
  uint32_t* pad;                  // local pad: pad[g] = ops GPU g started, pad[32+g] = ops it finished pushing
  uint32_t* peer_pad[kMaxGpus];   // peers' pads (nullptr for self / non-members)
  unsigned long long* arrive;
  unsigned long long* queue;      // [0] local, [kCtrLine/2] remote
  uint32_t* fin;
  uint32_t* err;
  uint32_t wait_mask;             // GPUs to wait for
  uint32_t post_mask;             // GPUs to post to
  int end_sync;                   // push mode: also post/wait "writes done" (pad[32+g]) before exit
  int my_gpu;
  uint64_t timeout_cycles;
  // Diagnostics (HB_TRACE=1; nullptr otherwise): per CTA kTraceWords u64 of
  // %globaltimer stamps written by the CTA's driving thread — entry, arrival
  // resolved, peers confirmed, first chunk landed, work done, exit — and the
  // CTA's chunk counts (total, remote).
  unsigned long long* trace;
  // host-side: launch with programmatic dependent launch (off when execs of
  // one group share a device: early-scheduled CTAs of one exec could hold the
  // slots a co-resident peer exec needs to start)
  int pdl;
};
constexpr int kTraceWords = 8;
constexpr int kTraceMaxCtas = 4096;
constexpr int kCtrBytes = 4 * 128;  // arrive | queues | fin | err lines

struct LaunchCfg {
  int grid;
  int block;
};

// Kernel attributes (dynamic shared memory size, carveout, clusters) are per
// device: one process may drive several GPUs (hb_exec_open_peers_local), so
// set them once per device, not once per process.
struct PerDeviceOnce {
  std::atomic<uint64_t> done{0};
  template <class F>
  void operator()(int device, F&& f) {
    const uint64_t bit = 1ull << (device & 63);
    if (done.load(std::memory_order_acquire) & bit) return;
    f();  // idempotent: two racing threads both setting an attribute is harmless
    done.fetch_or(bit, std::memory_order_acq_rel);
  }
};

// Host-side launchers (defined in boundary_kernels.cu).
void launch_copy(const CopySeg* segs, int nseg, Partition part, const SyncArgs& sync, LaunchCfg cfg,
                 void* stream);
void launch_reduce(const ReduceSeg* segs, int nseg, const void* const* terms, Partition part,
                   int in_dtype, int out_dtype, float beta, const SyncArgs& sync, LaunchCfg cfg,
                   void* stream);
// Fused 1F1B-paired step (one forward + one gradient return in one launch,
// warp-specialised). Needs the TMA copy partition with 32 KiB stages and the
// dynamic reduce partition; 0 on launch, 1 unsupported partition, 2 unsupported
// dtype pair (bf16->fp32, bf16->bf16, fp32->fp32), 5 launch error.
int launch_paired(const CopySeg* csegs, Partition cpart, const SyncArgs& csync, const ReduceSeg* rsegs,
                  const void* const* terms, Partition rpart, int in_dtype, int out_dtype, float beta,
                  const SyncArgs& rsync, int grid, void* stream);
int device_sm_count();
int copy_blocks_per_sm(int threads);
int tma_blocks_per_sm(uint64_t chunk);
uint64_t tma_chunk_bytes(int kib);  // 32 (default), 16 or 8 KiB stages
int reduce_blocks_per_sm(int threads, int in_dtype, int out_dtype);
uint64_t red_ring_elems(int in_dtype);  // elements of the reduce kernel's remote TMA ring

}  // namespace hb::dev
