// hetbridge — per-edge device runtime (the B200 replacement for
// hetsim::bridge::BridgeRuntime, bridge.hpp:146-173, and for simnet as the
// transport, simnet.hpp:86-148).
//
// One Exec per (edge, process). A process drives one GPU and executes, in one
// kernel launch per boundary op, the work of every logical rank that the
// rank->GPU map places on it: with 1 GPU all logical ranks are resident (HBM
// only); with N GPUs each process pulls the rows its ranks need straight from
// the owners' HBM over NVSwitch through CUDA-IPC-mapped peer buffers.
//
// Buffer layout: each GPU owns one device region (cudaMalloc, IPC-exported)
// holding a 4 KiB signal pad followed by the buffers of its resident ranks in
// a layout every process can compute from the plan alone, so a peer buffer's
// address is peer_base + offset with no table exchange (a symmetric-heap
// discipline, as NVSHMEM uses, without the library).
#pragma once

#include <cstdint>
#include <map>
#include <memory>
#include <set>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "hb/bridge.hpp"
#include "hb/index_map.hpp"
#include "kernels/boundary_kernels.cuh"

namespace hb::rt {

struct NvtxRange {  // profiler range for a host call (runtime.cpp)
  NvtxRange(const char* what, int mb);
  ~NvtxRange();
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

struct ExecConfig {
  int act_dtype = dev::kBF16;       // source / destination activations (copy width)
  int grad_in_dtype = dev::kBF16;   // destination gradients
  int grad_out_dtype = dev::kFP32;  // source gradients (accumulator)
  int mb_slots = 1;                 // buffer sets for microbatches in flight
  int internal_alloc = 1;           // allocate the device region (else bind() every buffer)
  int blocks_per_sm = 0;  // 0: as many as fit (occupancy)
  int threads = 512;
  double timeout_s = 20.0;          // flag-wait timeout
  int fwd_mode = 0;                 // forward: 0 auto, 1 consumers pull from owners, 2 owners push
  int partition = 0;                // 0 auto, 1 contiguous, 2 interleaved, 3 dynamic, 4 TMA bulk (copy)
  int strict_provenance = 0;        // 1: backward reads tp=0 copies only (index_map.hpp balance_replicas)
  int text_embedding = 0;           // splice: TEXT holds int32 token ids, rows gathered from an embedding table
  int max_ctas = 0;                 // cap on every boundary kernel's grid (0: fill the GPU); leaves SMs to
                                    // concurrent work (PP P2P, compute) and lets several execs share one GPU
  int max_ctas_bwd = 0;             // cap on the backward grid alone (0: max_ctas)
  int tma_chunk_kib = 0;            // TMA copy stage KiB (0: HB_TMA_CHUNK_KB or 32)
  int pdl = 1;                      // launch with programmatic dependent launch (off: execs sharing a device,
                                    // the host runtime whose NCCL kernels need SMs next to boundary kernels)
};

class Exec {
 public:
  Exec(const bridge::BridgePlan& plan, const index::SpliceSpec* splice, int n_gpus, int my_gpu,
       std::vector<int> rank_to_gpu, const ExecConfig& cfg);
  ~Exec();
  Exec(const Exec&) = delete;
  Exec& operator=(const Exec&) = delete;

  // Multi-GPU setup (collective across the exec group's processes).
  void ipc_handle(void* out64) const;
  void open_peers(const void* handles);  // n_gpus * 64 bytes, ordered by GPU index
  // Single-process form: execs[g] is the exec of GPU g of the same group in
  // this process (one host thread drives every GPU); peer regions are used
  // directly (peer access enabled between distinct devices, none needed when
  // several execs share one device).
  void open_peers_local(Exec* const* execs, int n);

  // Buffers of logical rank `rank` (must be resident here unless peer-mapped read-only use).
  void* buffer(int rank, int slot, int mb_slot, size_t* bytes) const;
  // Caller-owned buffer of a resident rank (ptr null: back to the library's
  // region). row_stride: elements between consecutive rows (0 or the row
  // width: packed); rows are samples (W) or, for splice slots, tokens (d_h).
  void bind(int rank, int slot, int mb_slot, void* ptr, size_t bytes, int64_t row_stride = 0);
  // Multi-process groups: this GPU's bindings as a blob (CUDA IPC handle of
  // each bound buffer's allocation + offset + stride; returns the size) and
  // the import of a peer GPU's blob (collective: every process exports,
  // all-gathers, imports every peer's blob before its next op).
  size_t export_bindings(void* out, size_t cap) const;
  void import_bindings(int gpu, const void* blob, size_t len);
  uint64_t bind_version() const { return bind_version_; }
  size_t buffer_bytes(int rank, int slot) const;

  void forward(int mb, void* stream);
  // Forward with the encoder projector fused in: computes
  // X . W^T for every local source rank (X: their token rows stacked in
  // ascending rank order, [rows x K]; W: [d_h x K]) on the tensor cores and
  // stores each output row straight into every destination row the plan maps
  // it to, local or on a peer GPU (push over NVSwitch); the source shards are
  // never materialised. Any GPU count, non-splice edges.
  // x_rows: rows of x (must equal the local source ranks' token rows).
  void forward_projected(int mb, const void* x, int64_t ldx, const void* w, int64_t ldw, int d_h, int K,
                         int64_t x_rows, void* stream);
  void backward(int mb, float beta, void* stream);
  // 1F1B pair in one launch: forward of fwd_mb and backward of bwd_mb (its
  // forward recorded), both ops of every peer's epoch sequence, run together by
  // the fused paired step kernel (two launches when the partitions cannot fuse).
  // Returns true if the fused kernel ran.
  bool paired(int fwd_mb, int bwd_mb, float beta, void* stream);
  void seed_forward_record(int mb);
  // Embedding table [vocab x d_h] (act dtype, on this GPU) the splice gathers
  // text rows from when cfg.text_embedding.
  void set_text_embedding(const void* table, int64_t vocab);
  // Vocab-parallel table (Megatron's VocabParallelEmbedding): resident rank
  // `rank` holds rows [begin, begin + rows) of the [vocab x d_h] table at
  // `shard`. Shards of one TP group are equal-sized and ordered by tp index
  // (begin = tp_idx * rows); the splice gathers each text row from the shard
  // that owns its id, on this GPU or a peer's (exported with the bindings).
  void set_text_embedding_shard(int rank, const void* shard, int64_t begin, int64_t rows, int64_t vocab);

  // CUDA-graph capture of one buffer set's forward (+ backward with `beta`):
  // the step is replayed with one graph launch (no per-kernel host overhead).
  // Replays bypass the microbatch records (a replay is a complete fwd+bwd).
  // what: 0 forward only, 1 forward + backward, 2 backward only, 3 forward +
  // backward of every buffer set in turn, 4 the 1F1B-paired cycle (step k =
  // forward of set k concurrently with the backward of set k-1), 5 the same
  // cycle with each pair in one warp-specialised launch.
  void graph_capture(int mb_slot, int what, float beta, void* stream);
  void graph_launch(int mb_slot, int what, void* stream);
  uint32_t device_error() const;  // synchronises
  // Recovery after a timeout or GroupMismatch: zero this exec's launch
  // counters, claim queues, error word and signal pad, and drop the
  // microbatch records. Collective: every exec of the group calls it with its
  // device idle, between two group-wide barriers; the group then starts again
  // from epoch 0 with its tables and captured graphs intact.
  void reset_protocol();
  // HB_TRACE=1 diagnostics: copies the last launch of `kind`'s per-CTA stamps
  // (dev::kTraceWords u64 each) into out; returns CTAs copied (0: tracing off).
  int read_trace(int kind, unsigned long long* out, int max_ctas, int* grid) const;

  // Static race and bounds check of every buffer set's device tables as the
  // kernels will read them (runtime_validate.cpp): "" when clean, else the
  // first violation; *checks = items checked.
  std::string validate(uint64_t* checks);

  const index::IndexMap& map() const { return map_; }
  int local_fwd_segments() const { return static_cast<int>(fwd_local_.size()); }
  int local_bwd_segments() const { return static_cast<int>(bwd_local_.size()); }
  uint64_t local_fwd_bytes() const;
  uint64_t local_bwd_elems() const;
  int launches() const { return launches_; }
  const bridge::BridgePlan& plan() const { return plan_; }

 private:
  int gpu_of(int rank) const { return rank_to_gpu_.at(rank); }
  int slot_dtype(int slot) const;
  uint64_t slot_bytes(int rank, int slot) const;
  int64_t text_row_elems() const;  // d_h of the splice (elements per text row)
  int64_t splice_d_h_ = 0;
  const unsigned char* embed_table_ = nullptr;
  int64_t embed_vocab_ = 0;
  struct EmbedShard {
    const unsigned char* ptr = nullptr;
    int64_t begin = 0, rows = 0;
  };
  std::vector<EmbedShard> shard_;        // [rank]: vocab-parallel shards (resident: set; peers: imported)
  EmbedShard shard_of(int rank) const;   // a peer exec's own entry in single-process groups
  bool sharded() const;                  // some rank has a shard: gathers use the TP group's shards
  const unsigned char** shard_dev_ = nullptr;  // [world * tp]: each dest rank's TP-group shard bases
  uint64_t offset_of(int gpu, int rank, int slot, int mb_slot) const;
  void prepare_fwd();  // resolve pointers, upload descriptors (after bind/open)
  void prepare_bwd();
  static constexpr int kFwdKind = 0, kBwdKind = 1, kProjKind = 2, kNumKinds = 3;
  dev::SyncArgs make_sync_args(int kind, bool push) const;

  bridge::BridgePlan plan_;
  index::IndexMap map_;
  int n_gpus_, my_gpu_, device_;
  std::vector<int> rank_to_gpu_;
  ExecConfig cfg_;
  uint32_t group_mask_ = 0;
  bool fwd_push_ = false;  // resolved forward mode

  // layout: offsets_[gpu][rank*kNumSlots+slot] (for mb slot 0), stride per mb slot
  std::vector<std::vector<uint64_t>> offsets_;
  std::vector<uint64_t> mb_stride_;  // per gpu
  uint64_t region_bytes_ = 0;
  unsigned char* local_base_ = nullptr;
  std::vector<unsigned char*> peer_base_;
  std::vector<char> peer_ipc_;  // peer_base_[g] was opened with cudaIpcOpenMemHandle (closed at exit)
  int grid_cap(int grid) const { return cfg_.max_ctas > 0 && cfg_.max_ctas < grid ? cfg_.max_ctas : grid; }
  int grid_cap_bwd(int grid) const {
    const int c = cfg_.max_ctas_bwd > 0 ? cfg_.max_ctas_bwd : cfg_.max_ctas;
    return c > 0 && c < grid ? c : grid;
  }
  int tma_kib() const;
  struct Binding {
    void* ptr = nullptr;
    int64_t stride = 0;  // elements between rows (0: packed)
  };
  std::vector<std::vector<Binding>> bound_;       // [rank*kNumSlots+slot][mb]: caller buffers of resident ranks
  std::vector<std::vector<Binding>> peer_bound_;  // same for peers' ranks (imported, or read from a local peer exec)
  std::vector<Exec*> peer_exec_;                  // single-process groups
  std::map<std::string, unsigned char*> ipc_open_;  // opened binding handles (by handle bytes)
  uint64_t bind_version_ = 0;
  bool work_dirty_ = true;
  void build_work();
  int64_t row_width(int slot) const;
  const Binding* binding_of(int rank, int slot, int mb) const;
  bool strided(int rank, int slot) const;
  unsigned char* addr(int rank, int slot, int mb, int64_t off, int es) const;

  // Forward work of this GPU: source runs with every destination that needs
  // them (pull: destinations resident here; push: sources resident here), so a
  // run crosses NVLink / leaves HBM once however many replicas consume it.
  struct FanSeg {
    index::Ref src;
    std::vector<index::Ref> dsts;
    int64_t n = 0;
    bool remote = false;  // reads (pull) or writes (push) a peer's buffer
  };
  std::vector<FanSeg> fwd_local_;
  std::vector<index::ReduceSeg> bwd_local_;

  struct DevTables {
    dev::CopySeg* copy = nullptr;
    dev::ReduceSeg* reduce = nullptr;
    const void** terms = nullptr;
  };
  std::vector<DevTables> tables_;  // per mb slot
  struct ProjTable {
    int d_h = 0;
    int fan = 0;
    int rows = 0;
    int staged = -1;                     // the table is for the staged path (rows -> own source shard)
    unsigned char** rows_dev = nullptr;  // [rows * fan]
  };
  // The fused projector pushes each row to every destination, so a GPU hosting
  // several consumers of a row receives it once per consumer over NVLink. When
  // that happens anywhere in the group (decided from the plan: every GPU takes
  // the same path), forward_projected stages instead: the projector writes the
  // source shards and the pulled forward fans each row out on its GPU.
  bool proj_staged() const;
  std::vector<ProjTable> proj_;  // per mb slot
  // Static contiguous partition of each direction's work space over the grid.
  struct DevPartition {
    int32_t* first_seg = nullptr;
    uint64_t per_cta = 0;
    int grid = 1;
    int mode = 0;
    uint32_t total_chunks = 0;
    uint64_t chunk = 0;
    uint2* chunks = nullptr;
    uint32_t rtotal_chunks = 0;
    uint2* rchunks = nullptr;
    uint64_t rchunk = 0;
    int remote_ctas = 0;
    uint32_t lstatic = 0, rstatic = 0;
    int ring = 1;
    int prefetch_other = 1;
    int fan = 0;
    int stage_local = 0;
    dev::Partition dev() const {
      return {first_seg, per_cta, mode, total_chunks, chunk, chunks, rtotal_chunks, rchunks, rchunk, remote_ctas,
              lstatic, rstatic, ring, prefetch_other, fan, stage_local, static_cast<uint32_t>(grid)};
    }
  };
  DevPartition fwd_part_, bwd_part_;
  void upload_copies(int mb, uint64_t unit, std::vector<uint64_t>* w0s, std::vector<uint64_t>* ns);
  int copy_mode() const;
  int reduce_mode() const;
  uint64_t pad_unit(int mode, bool copy) const;
  int copy_grid() const;
  // remote[s]: segment s reads (pull) or writes (push) a peer's buffer; cost_local/remote in bytes
  void build_partition(const std::vector<uint64_t>& w0, const std::vector<uint64_t>& n,
                       const std::vector<char>& remote, double local_bytes, double remote_bytes, int grid,
                       int mode, uint64_t unit, DevPartition* out, uint64_t runit = 0, bool taper = false);
  bool dirty_fwd_ = true, dirty_bwd_ = true;
  bool graphs_invalidated_ = false;
  bool shared_device_ = false;  // a peer exec of the group runs on this device (no PDL)
  void mark_dirty();  // tables rebuilt at the next op; captured graphs dropped
  void check_forward_mb(int mb) const;
  int bwd_groups_ = 0;  // device reduce segments (fan-out groups of bwd_local_)
  uint32_t* ctr_ = nullptr;  // device counters
  unsigned long long* trace_ = nullptr;  // HB_TRACE diagnostics
  dev::SyncArgs sync_fwd_{}, sync_bwd_{}, sync_proj_{};
  int clock_khz_ = 2000000;
  int sm_count_ = 0;
  int launches_ = 0;
  std::set<int> fwd_done_;
  std::map<std::pair<int, int>, std::pair<void*, int>> graphs_;  // (slot, what) -> (cudaGraphExec_t, kernels)
  cudaStream_t side_ = nullptr;  // the 1F1B-paired graph's backward stream (what = 4)
  cudaEvent_t fork_ = nullptr, join_ = nullptr;
  void launch_forward(int mb_slot, void* stream);
  bool launch_paired(int fslot, int bslot, float beta, void* stream);
  void launch_backward(int mb_slot, float beta, void* stream);
};

}  // namespace hb::rt
