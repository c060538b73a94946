// hetbridge — per-edge device runtime (see runtime.hpp).
#include "hb/runtime.hpp"

#include "kernels/projector_gemm.cuh"

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <tuple>

namespace hb::rt {

// NVTX range for the scope (header-only NVTX3: free unless a tool such as
// ncu --nvtx or nsys is attached): every boundary op shows up by name and
// microbatch on the profiler's timeline.
NvtxRange::NvtxRange(const char* what, int mb) {
  char b[64];
  std::snprintf(b, sizeof b, "hetbridge %s mb %d", what, mb);
  nvtxRangePushA(b);
}
NvtxRange::~NvtxRange() { nvtxRangePop(); }

namespace {
void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    raise(ErrorCode::CudaError, std::string(what) + ": " + cudaGetErrorString(e));
}
constexpr uint64_t kPadBytes = 4096;
// Makes the exec's device current for the scope (one host thread may drive
// several GPUs' execs; kernels must go to the device their stream belongs to).
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) == cudaSuccess && prev != dev) cudaSetDevice(dev);
    else prev = -1;
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
  DeviceGuard(const DeviceGuard&) = delete;
  DeviceGuard& operator=(const DeviceGuard&) = delete;
};
constexpr uint64_t kAlign = 256;
uint64_t align_up(uint64_t x) { return (x + kAlign - 1) / kAlign * kAlign; }
}  // namespace

Exec::Exec(const bridge::BridgePlan& plan, const index::SpliceSpec* splice, int n_gpus, int my_gpu,
           std::vector<int> rank_to_gpu, const ExecConfig& cfg)
    : plan_(plan), n_gpus_(n_gpus), my_gpu_(my_gpu), rank_to_gpu_(std::move(rank_to_gpu)), cfg_(cfg) {
  if (n_gpus < 1 || n_gpus > dev::kMaxGpus || my_gpu < 0 || my_gpu >= n_gpus)
    raise(ErrorCode::InvalidArgument, "bad GPU count / index");
  if (cfg.mb_slots < 1) raise(ErrorCode::InvalidArgument, "mb_slots must be >= 1");
  for (int dt : {cfg.act_dtype, cfg.grad_in_dtype, cfg.grad_out_dtype})
    if (dt < dev::kBF16 || dt > dev::kFP64) raise(ErrorCode::InvalidArgument, "unknown dtype");
  if (cfg.grad_in_dtype == dev::kFP64 || cfg.grad_out_dtype == dev::kFP64)
    raise(ErrorCode::InvalidArgument, "fp64 gradients are not supported on the device path");
  map_ = index::build_index_map(plan_, splice, cfg.strict_provenance == 0);
  splice_d_h_ = splice ? splice->d_h : 0;
  if (cfg.text_embedding && !splice)
    raise(ErrorCode::InvalidArgument, "text_embedding needs a splice edge (text rows to gather)");
  if (cfg.text_embedding && splice->text_mode == index::TextMode::InPlace)
    raise(ErrorCode::InvalidArgument, "text_embedding gathers text rows; an in-place splice has none to gather");
  if (static_cast<int>(rank_to_gpu_.size()) < map_.world)
    raise(ErrorCode::InvalidArgument, "rank_to_gpu must cover every logical rank of the edge");
  for (int r = 0; r < map_.world; ++r)
    if (rank_to_gpu_[r] < 0 || rank_to_gpu_[r] >= n_gpus)
      raise(ErrorCode::InvalidArgument, "rank_to_gpu entry out of range");

  // Exec group: GPUs hosting any rank with a buffer.
  for (int r = 0; r < map_.world; ++r)
    for (int s = 0; s < index::kNumSlots; ++s)
      if (map_.elems[r][s]) group_mask_ |= 1u << gpu_of(r);

  // Deterministic per-GPU layouts.
  offsets_.assign(n_gpus, std::vector<uint64_t>(map_.world * index::kNumSlots, 0));
  mb_stride_.assign(n_gpus, 0);
  for (int g = 0; g < n_gpus; ++g) {
    uint64_t off = 0;
    for (int r = 0; r < map_.world; ++r) {
      if (gpu_of(r) != g) continue;
      for (int s = 0; s < index::kNumSlots; ++s) {
        offsets_[g][r * index::kNumSlots + s] = off;
        off += align_up(slot_bytes(r, s));
      }
    }
    mb_stride_[g] = off;
    region_bytes_ = std::max(region_bytes_, kPadBytes + off * cfg.mb_slots);
  }
  bound_.assign(map_.world * index::kNumSlots, std::vector<Binding>(cfg.mb_slots));
  shard_.assign(map_.world, EmbedShard{});
  peer_bound_.assign(map_.world * index::kNumSlots, std::vector<Binding>(cfg.mb_slots));
  peer_exec_.assign(n_gpus_, nullptr);

  // Forward mode. Pull (consumers read the owners' HBM) needs one barrier;
  // push (owners write the consumers' HBM) needs a second "writes done"
  // barrier. Measured with the host out of the loop (scripts/sweep_probe.py,
  // N=4, profiles/r01_n4_sweep.log) pull is faster for every config, one-way
  // and bidirectional (c2w4 68 vs 72 us, c4w4 68 vs 81 us, c2 150 vs 168 us),
  // so auto means pull; push stays selectable.
  fwd_push_ = cfg_.fwd_mode == 2 && n_gpus_ > 1;
  build_work();

  ck(cudaGetDevice(&device_), "cudaGetDevice");
  sm_count_ = dev::device_sm_count();
  if (cfg_.internal_alloc || n_gpus_ > 1) {
    ck(cudaMalloc(&local_base_, region_bytes_), "cudaMalloc(region)");
    ck(cudaMemset(local_base_, 0, kPadBytes), "cudaMemset(pad)");
    static_assert(2 * kNumKinds * dev::kMaxGpus * sizeof(uint32_t) <= kPadBytes, "pad holds start and done flags of every kind");
  }
  ck(cudaMalloc(&ctr_, kNumKinds * dev::kCtrBytes), "cudaMalloc(ctr)");
  ck(cudaMemset(ctr_, 0, kNumKinds * dev::kCtrBytes), "cudaMemset(ctr)");
  if (const char* tr = std::getenv("HB_TRACE"); tr && tr[0] == '1') {  // diagnostics: per-CTA timestamps of the last launch of each kind
    const size_t tb = kNumKinds * static_cast<size_t>(dev::kTraceMaxCtas) * dev::kTraceWords * 8;
    ck(cudaMalloc(&trace_, tb), "cudaMalloc(trace)");
    ck(cudaMemset(trace_, 0, tb), "cudaMemset(trace)");
  }
  peer_base_.assign(n_gpus_, nullptr);
  peer_ipc_.assign(n_gpus_, 0);
  peer_base_[my_gpu_] = local_base_;
  tables_.resize(cfg.mb_slots);
  proj_.resize(cfg.mb_slots);
  int khz = 0;
  cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, device_);
  clock_khz_ = khz > 0 ? khz : 2000000;
  sync_fwd_ = make_sync_args(kFwdKind, fwd_push_);
  sync_bwd_ = make_sync_args(kBwdKind, false);
  sync_proj_ = make_sync_args(kProjKind, true);
}

Exec::~Exec() {
  if (side_) {
    cudaStreamSynchronize(side_);
    cudaStreamDestroy(side_);
    cudaEventDestroy(fork_);
    cudaEventDestroy(join_);
  }
  DeviceGuard dg(device_);
  for (auto& kv : graphs_) cudaGraphExecDestroy(static_cast<cudaGraphExec_t>(kv.second.first));
  for (auto& t : proj_) cudaFree(t.rows_dev);
  for (auto& t : tables_) {
    cudaFree(t.copy);
    cudaFree(t.reduce);
    cudaFree(t.terms);
  }
  cudaFree(fwd_part_.first_seg);
  for (auto* p : {&fwd_part_, &bwd_part_}) {
    cudaFree(p->chunks);
    cudaFree(p->rchunks);
  }
  cudaFree(bwd_part_.first_seg);
  for (int g = 0; g < n_gpus_; ++g)
    if (g != my_gpu_ && peer_base_[g] && peer_ipc_[g]) cudaIpcCloseMemHandle(peer_base_[g]);
  for (auto& kv : ipc_open_) cudaIpcCloseMemHandle(kv.second);
  cudaFree(local_base_);
  cudaFree(ctr_);
  cudaFree(trace_);
  cudaFree(shard_dev_);
}

// Elements per row of a slot's buffer: a sample (W) for activations and
// gradients, a token (d_h) for splice token slices and text rows. A bound
// buffer with a row stride places row i at element i*stride.
int64_t Exec::row_width(int slot) const {
  if (splice_d_h_ && (slot == index::kDstAct || slot == index::kDstGrad || slot == index::kText)) return splice_d_h_;
  return plan_.edge.feature_width;
}

const Exec::Binding* Exec::binding_of(int rank, int slot, int mb) const {
  const auto& b = bound_[rank * index::kNumSlots + slot][mb];
  if (b.ptr) return &b;
  const auto& p = peer_bound_[rank * index::kNumSlots + slot][mb];
  return p.ptr ? &p : nullptr;
}

// Rows of (rank, slot) are not packed in some buffer set: runs over it are
// split at row boundaries so every piece is contiguous in memory.
bool Exec::strided(int rank, int slot) const {
  for (int mb = 0; mb < cfg_.mb_slots; ++mb) {
    const Binding* b = binding_of(rank, slot, mb);
    if (b && b->stride) return true;
  }
  return false;
}

unsigned char* Exec::addr(int rank, int slot, int mb, int64_t off, int es) const {
  const Binding* b = binding_of(rank, slot, mb);
  if (b) {
    if (b->stride) {
      const int64_t w = row_width(slot);
      off = off / w * b->stride + off % w;
    }
    return static_cast<unsigned char*>(b->ptr) + off * es;
  }
  const int g = gpu_of(rank);
  if (!peer_base_[g])
    raise(ErrorCode::InvalidArgument, "buffer of rank " + std::to_string(rank) +
                                          " unavailable (peer not opened or not bound)");
  return peer_base_[g] + offset_of(g, rank, slot, mb) + off * es;
}

// This GPU's forward and backward work from the index map: runs split at the
// row boundaries of strided bound buffers, forward runs grouped by source run
// (fan-out: one read, up to kMaxFan destinations).
void Exec::build_work() {
  auto next_cut = [&](const index::Ref& r, int64_t pos) -> int64_t {  // elements left in r's current row
    if (!strided(r.rank, r.slot)) return INT64_MAX;
    const int64_t w = row_width(r.slot);
    return w - (r.off + pos) % w;
  };
  std::vector<index::CopySeg> fwd;
  for (const auto& s : map_.fwd) {
    if (gpu_of(fwd_push_ ? s.src.rank : s.dst.rank) != my_gpu_) continue;
    for (int64_t pos = 0; pos < s.n;) {
      const int64_t len = std::min({s.n - pos, next_cut(s.src, pos), next_cut(s.dst, pos)});
      index::CopySeg c = s;
      c.src.off += pos;
      c.dst.off += pos;
      c.n = len;
      fwd.push_back(c);
      pos += len;
    }
  }
  // Fan-out grouping: every destination of one source run that this GPU
  // executes shares a single read of the run (decided per GPU; the symmetric
  // layout means no process needs another's grouping).
  fwd_local_.clear();
  std::map<std::tuple<int, int, int64_t, int64_t>, std::vector<size_t>> groups;
  std::vector<std::tuple<int, int, int64_t, int64_t>> order;
  for (size_t i = 0; i < fwd.size(); ++i) {
    const auto& s = fwd[i];
    const auto key = std::make_tuple(s.src.rank, s.src.slot, s.src.off, s.n);
    auto& g = groups[key];
    if (g.empty()) order.push_back(key);
    g.push_back(i);
  }
  for (const auto& key : order) {
    const auto& idx = groups[key];
    for (size_t k = 0; k < idx.size(); k += dev::kMaxFan) {
      FanSeg f;
      const auto& first = fwd[idx[k]];
      f.src = first.src;
      f.n = first.n;
      f.remote = !fwd_push_ && gpu_of(first.src.rank) != my_gpu_;
      // a vocab-parallel gather reads the shards of the destination's TP group:
      // behind the peer wait when any of them sits on another GPU
      if (first.src.slot == index::kText && cfg_.text_embedding && sharded())
        for (int m : grid::module_group(plan_.edge.dest, first.src.rank, grid::GroupKind::TP))
          if (gpu_of(m) != my_gpu_) f.remote = true;
      for (size_t j = k; j < std::min(idx.size(), k + dev::kMaxFan); ++j) {
        const auto& d = fwd[idx[j]].dst;
        f.dsts.push_back(d);
        if (fwd_push_ && gpu_of(d.rank) != my_gpu_) f.remote = true;
      }
      fwd_local_.push_back(std::move(f));
    }
  }
  bwd_local_.clear();
  for (const auto& s : map_.bwd) {
    if (gpu_of(s.dst.rank) != my_gpu_) continue;
    for (int64_t pos = 0; pos < s.n;) {
      int64_t len = std::min(s.n - pos, next_cut(s.dst, pos));
      for (const auto& t : s.terms) len = std::min(len, next_cut(t, pos));
      index::ReduceSeg r = s;
      r.dst.off += pos;
      for (auto& t : r.terms) t.off += pos;
      r.n = len;
      bwd_local_.push_back(std::move(r));
      pos += len;
    }
  }
  work_dirty_ = false;
}

int Exec::slot_dtype(int slot) const {
  switch (slot) {
    case index::kDstGrad: return cfg_.grad_in_dtype;
    case index::kSrcGrad: return cfg_.grad_out_dtype;
    case index::kText: return cfg_.text_embedding ? dev::kI32 : cfg_.act_dtype;
    default: return cfg_.act_dtype;
  }
}

int64_t Exec::text_row_elems() const { return splice_d_h_; }

// Bytes of a rank's buffer: elements x dtype, except token ids (one per text row).
uint64_t Exec::slot_bytes(int rank, int slot) const {
  int64_t n = map_.elems[rank][slot];
  if (slot == index::kText && cfg_.text_embedding) n /= splice_d_h_;
  return static_cast<uint64_t>(n) * dev::dtype_size(slot_dtype(slot));
}

uint64_t Exec::offset_of(int gpu, int rank, int slot, int mb_slot) const {
  return kPadBytes + mb_stride_[gpu] * mb_slot + offsets_[gpu][rank * index::kNumSlots + slot];
}

size_t Exec::buffer_bytes(int rank, int slot) const {
  if (rank < 0 || rank >= map_.world || slot < 0 || slot >= index::kNumSlots)
    raise(ErrorCode::InvalidArgument, "buffer index out of range");
  return static_cast<size_t>(slot_bytes(rank, slot));
}

void Exec::ipc_handle(void* out64) const {
  if (!local_base_) raise(ErrorCode::InvalidArgument, "no device region to export");
  cudaIpcMemHandle_t h;
  ck(cudaIpcGetMemHandle(&h, local_base_), "cudaIpcGetMemHandle");
  static_assert(sizeof(h) == 64, "IPC handle size");
  std::memcpy(out64, &h, 64);
}

void Exec::open_peers(const void* handles) {
  DeviceGuard dg(device_);
  for (int g = 0; g < n_gpus_; ++g) {
    if (g == my_gpu_ || !((group_mask_ >> g) & 1u) || peer_base_[g]) continue;
    cudaIpcMemHandle_t h;
    std::memcpy(&h, static_cast<const unsigned char*>(handles) + 64 * g, 64);
    void* p = nullptr;
    ck(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
    peer_base_[g] = static_cast<unsigned char*>(p);
    peer_ipc_[g] = 1;
  }
  sync_fwd_ = make_sync_args(kFwdKind, fwd_push_);
  sync_bwd_ = make_sync_args(kBwdKind, false);
  sync_proj_ = make_sync_args(kProjKind, true);
  mark_dirty();
}

void Exec::open_peers_local(Exec* const* execs, int n) {
  DeviceGuard dg(device_);
  if (n != n_gpus_) raise(ErrorCode::InvalidArgument, "open_peers_local needs one exec per GPU of the group");
  for (int g = 0; g < n_gpus_; ++g) {
    if (g == my_gpu_ || !((group_mask_ >> g) & 1u) || peer_base_[g]) continue;
    const Exec* p = execs[g];
    if (!p || p == this) raise(ErrorCode::InvalidArgument, "open_peers_local: missing exec of GPU " + std::to_string(g));
    // the symmetric layout: every exec of the group derived the same offsets from the same plan
    if (p->my_gpu_ != g || p->n_gpus_ != n_gpus_ || p->rank_to_gpu_ != rank_to_gpu_ || p->offsets_ != offsets_ ||
        p->mb_stride_ != mb_stride_ || p->cfg_.mb_slots != cfg_.mb_slots || !p->local_base_)
      raise(ErrorCode::InvalidArgument, "open_peers_local: exec of GPU " + std::to_string(g) +
                                            " has a different configuration or no device region");
    if (p->device_ == device_) shared_device_ = true;
    if (p->device_ != device_) {
      int can = 0;
      ck(cudaDeviceCanAccessPeer(&can, device_, p->device_), "cudaDeviceCanAccessPeer");
      if (!can) raise(ErrorCode::CudaError, "no peer access from device " + std::to_string(device_) + " to " +
                                                std::to_string(p->device_));
      const cudaError_t e = cudaDeviceEnablePeerAccess(p->device_, 0);
      if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
      else ck(e, "cudaDeviceEnablePeerAccess");
    }
    peer_base_[g] = p->local_base_;
  }
  // the peers' caller-bound buffers (same address space): re-read on every call
  for (int g = 0; g < n_gpus_; ++g) {
    if (g == my_gpu_ || !execs[g]) continue;
    peer_exec_[g] = execs[g];
    for (int r = 0; r < map_.world; ++r)
      if (gpu_of(r) == g)
        for (int sl = 0; sl < index::kNumSlots; ++sl)
          peer_bound_[r * index::kNumSlots + sl] = execs[g]->bound_[r * index::kNumSlots + sl];
  }
  work_dirty_ = true;
  sync_fwd_ = make_sync_args(kFwdKind, fwd_push_);
  sync_bwd_ = make_sync_args(kBwdKind, false);
  sync_proj_ = make_sync_args(kProjKind, true);
  mark_dirty();
}

// Every change of a buffer pointer, the peer mapping or the embedding table
// rebuilds the device tables at the next op, and captured graphs hold the old
// tables' addresses as kernel arguments: drop them (an in-flight replay
// finishes first, cudaGraphExecDestroy defers) so a stale replay cannot
// touch freed tables; graph_launch then asks for a recapture.
void Exec::mark_dirty() {
  dirty_fwd_ = dirty_bwd_ = true;
  for (auto& kv : graphs_) cudaGraphExecDestroy(static_cast<cudaGraphExec_t>(kv.second.first));
  if (!graphs_.empty()) graphs_invalidated_ = true;
  graphs_.clear();
}

void* Exec::buffer(int rank, int slot, int mb_slot, size_t* bytes) const {
  const size_t n = buffer_bytes(rank, slot);
  if (bytes) *bytes = n;
  if (mb_slot < 0 || mb_slot >= cfg_.mb_slots) raise(ErrorCode::InvalidArgument, "mb slot out of range");
  if (void* b = bound_[rank * index::kNumSlots + slot][mb_slot].ptr) return b;
  if (gpu_of(rank) != my_gpu_) raise(ErrorCode::InvalidArgument, "rank is not resident on this GPU");
  if (!local_base_ || n == 0) return nullptr;
  return local_base_ + offset_of(my_gpu_, rank, slot, mb_slot);
}

void Exec::bind(int rank, int slot, int mb_slot, void* ptr, size_t bytes, int64_t row_stride) {
  const size_t n = buffer_bytes(rank, slot);
  if (mb_slot < 0 || mb_slot >= cfg_.mb_slots) raise(ErrorCode::InvalidArgument, "mb slot out of range");
  if (gpu_of(rank) != my_gpu_) raise(ErrorCode::InvalidArgument, "can only bind resident ranks");
  if (row_stride < 0) raise(ErrorCode::InvalidArgument, "row stride must be >= 0");
  const int64_t w = row_width(slot);
  if (row_stride == w) row_stride = 0;  // packed
  if (row_stride && row_stride < w) raise(ErrorCode::ShapeMismatch, "row stride smaller than the row width");
  if (row_stride && slot == index::kText && cfg_.text_embedding)
    raise(ErrorCode::InvalidArgument, "token-id buffers are packed (no row stride)");
  const int es = dev::dtype_size(slot_dtype(slot));
  const int64_t elems = map_.elems[rank][slot];
  const size_t need = row_stride && elems ? static_cast<size_t>(((elems / w - 1) * row_stride + w) * es) : n;
  if (ptr && bytes < need) raise(ErrorCode::ShapeMismatch, "bound buffer smaller than the planned shard");
  Binding& b = bound_[rank * index::kNumSlots + slot][mb_slot];
  if (b.ptr == ptr && b.stride == row_stride) return;  // unchanged: keep tables and graphs
  const bool was_strided = strided(rank, slot);
  b = {ptr, ptr ? row_stride : 0};
  if (strided(rank, slot) != was_strided) work_dirty_ = true;
  ++bind_version_;
  mark_dirty();
}

namespace {
// cuMemGetAddressRange through the runtime's driver entry point (no -lcuda).
void* allocation_base(void* p, size_t* size) {
  using Fn = int (*)(unsigned long long*, size_t*, unsigned long long);
  static Fn fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      f = nullptr;
    return reinterpret_cast<Fn>(f);
  }();
  if (!fn) raise(ErrorCode::CudaError, "cuMemGetAddressRange unavailable");
  unsigned long long base = 0;
  if (fn(&base, size, reinterpret_cast<unsigned long long>(p)) != 0)
    raise(ErrorCode::CudaError, "cuMemGetAddressRange failed (not a device allocation?)");
  return reinterpret_cast<void*>(base);
}

struct BindRecord {  // one exported binding (fixed 96-byte record)
  int32_t rank, slot, mb_slot, pad;
  int64_t offset;  // bytes from the allocation base
  int64_t stride;  // elements (0: packed)
  unsigned char handle[64];
};
static_assert(sizeof(BindRecord) == 96, "record layout");
// a vocab-parallel embedding shard travels as a record with this slot:
// mb_slot = 0, pad = first vocab row, stride = rows
constexpr int32_t kShardSlot = 1000;
}  // namespace

size_t Exec::export_bindings(void* out, size_t cap) const {
  DeviceGuard dg(device_);
  std::vector<BindRecord> recs;
  for (int r = 0; r < map_.world; ++r) {
    if (gpu_of(r) != my_gpu_) continue;
    for (int s = 0; s < index::kNumSlots; ++s)
      for (int mb = 0; mb < cfg_.mb_slots; ++mb) {
        const Binding& b = bound_[r * index::kNumSlots + s][mb];
        if (!b.ptr) continue;
        BindRecord rec{};
        rec.rank = r;
        rec.slot = s;
        rec.mb_slot = mb;
        size_t sz = 0;
        void* base = allocation_base(b.ptr, &sz);
        rec.offset = static_cast<unsigned char*>(b.ptr) - static_cast<unsigned char*>(base);
        rec.stride = b.stride;
        cudaIpcMemHandle_t h;
        ck(cudaIpcGetMemHandle(&h, base), "cudaIpcGetMemHandle(bound buffer)");
        std::memcpy(rec.handle, &h, 64);
        recs.push_back(rec);
      }
  }
  for (int r = 0; r < map_.world; ++r) {
    if (gpu_of(r) != my_gpu_ || !shard_[r].ptr) continue;
    if (shard_[r].begin > 0x7fffffffll) raise(ErrorCode::InvalidArgument, "vocab-parallel shard begins beyond 2^31");
    BindRecord rec{};
    rec.rank = r;
    rec.slot = kShardSlot;
    rec.pad = static_cast<int32_t>(shard_[r].begin);
    size_t sz = 0;
    void* base = allocation_base(const_cast<unsigned char*>(shard_[r].ptr), &sz);
    rec.offset = shard_[r].ptr - static_cast<unsigned char*>(base);
    rec.stride = shard_[r].rows;
    cudaIpcMemHandle_t h;
    ck(cudaIpcGetMemHandle(&h, base), "cudaIpcGetMemHandle(embedding shard)");
    std::memcpy(rec.handle, &h, 64);
    recs.push_back(rec);
  }
  const size_t need = 8 + recs.size() * sizeof(BindRecord);
  if (out && cap >= need) {
    const uint64_t n = recs.size();
    std::memcpy(out, &n, 8);
    if (!recs.empty()) std::memcpy(static_cast<unsigned char*>(out) + 8, recs.data(), recs.size() * sizeof(BindRecord));
  }
  return need;
}

void Exec::import_bindings(int gpu, const void* blob, size_t len) {
  DeviceGuard dg(device_);
  if (gpu < 0 || gpu >= n_gpus_) raise(ErrorCode::InvalidArgument, "bad GPU index");
  if (gpu == my_gpu_) return;
  if (len < 8) raise(ErrorCode::InvalidArgument, "binding blob too short");
  uint64_t n = 0;
  std::memcpy(&n, blob, 8);
  if (len < 8 + n * sizeof(BindRecord)) raise(ErrorCode::InvalidArgument, "binding blob truncated");
  // bindings of `gpu`'s ranks not in the blob revert to the peer region
  for (int r = 0; r < map_.world; ++r)
    if (gpu_of(r) == gpu) {
      for (int s = 0; s < index::kNumSlots; ++s)
        for (auto& b : peer_bound_[r * index::kNumSlots + s]) b = {};
      shard_[r] = {};
    }
  for (uint64_t i = 0; i < n; ++i) {
    BindRecord rec;
    std::memcpy(&rec, static_cast<const unsigned char*>(blob) + 8 + i * sizeof(BindRecord), sizeof(rec));
    if (rec.slot == kShardSlot) {  // a peer rank's vocab-parallel embedding shard
      if (rec.rank < 0 || rec.rank >= map_.world || gpu_of(rec.rank) != gpu || rec.stride < 1)
        raise(ErrorCode::InvalidArgument, "embedding shard record does not match this group's layout");
      const std::string key(reinterpret_cast<const char*>(rec.handle), 64);
      auto it = ipc_open_.find(key);
      if (it == ipc_open_.end()) {
        cudaIpcMemHandle_t h;
        std::memcpy(&h, rec.handle, 64);
        void* p = nullptr;
        ck(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle(embedding shard)");
        it = ipc_open_.emplace(key, static_cast<unsigned char*>(p)).first;
      }
      shard_[rec.rank] = {it->second + rec.offset, rec.pad, rec.stride};
      continue;
    }
    if (rec.rank < 0 || rec.rank >= map_.world || gpu_of(rec.rank) != gpu || rec.slot < 0 ||
        rec.slot >= index::kNumSlots || rec.mb_slot < 0 || rec.mb_slot >= cfg_.mb_slots)
      raise(ErrorCode::InvalidArgument, "binding record does not match this group's layout");
    const std::string key(reinterpret_cast<const char*>(rec.handle), 64);
    auto it = ipc_open_.find(key);
    if (it == ipc_open_.end()) {
      cudaIpcMemHandle_t h;
      std::memcpy(&h, rec.handle, 64);
      void* p = nullptr;
      ck(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle(bound buffer)");
      it = ipc_open_.emplace(key, static_cast<unsigned char*>(p)).first;
    }
    peer_bound_[rec.rank * index::kNumSlots + rec.slot][rec.mb_slot] = {it->second + rec.offset, rec.stride};
  }
  work_dirty_ = true;
  mark_dirty();
}

namespace {
constexpr uint64_t kDynCopyChunk = 128 * 1024;   // bytes per dynamic copy chunk
uint64_t env_u64(const char* name, uint64_t dflt) {
  const char* v = std::getenv(name);
  return v && *v ? std::strtoull(v, nullptr, 10) : dflt;
}
// elements per dynamic reduce chunk; TMA stage size (tuning knobs, HB_RED_CHUNK / HB_TMA_CHUNK_KB)
const uint64_t kDynReduceChunk = env_u64("HB_RED_CHUNK", 0);  // 0: sized per launch (prepare_bwd)
const int kTmaChunkKiB = static_cast<int>(env_u64("HB_TMA_CHUNK_KB", 32));
// A remote copy chunk waits for every peer's arrival by default; HB_WAIT_ALL_PEERS=0 waits
// only for the GPUs the chunk touches. Measured at N=4 (one box, A/B): per-peer waits save
// ~1 us on c4w4 but cost 6 us on c2x4's all-gather (early peers' links fill first, the
// late peer's share becomes the tail).
const bool kWaitAllPeers = env_u64("HB_WAIT_ALL_PEERS", 1) != 0;
uint64_t pad_to(uint64_t x, uint64_t q) { return (x + q - 1) / q * q; }
}  // namespace

int Exec::copy_mode() const {
  switch (cfg_.partition) {
    case 2: return dev::kPartInterleaved;
    case 3: return dev::kPartDynamic;
    case 1: return dev::kPartContiguous;
    default: return dev::kPartTma;  // 0 auto: TMA bulk copies (measured 97% of the HBM copy peak, C2 N=1)
  }
}

int Exec::reduce_mode() const {
  // The backward reduce runs the LDG/STG engine over dynamic chunks under the
  // TMA copy partition (measured at N=1, C2-C5: 0.87-0.97 of HBM; a one-warp
  // TMA-staged reduce reached only 0.29-0.34, its in-smem fp32 pass being
  // issue-bound, and was dropped).
  const int m = copy_mode();
  return m == dev::kPartTma ? dev::kPartDynamic : m;
}

uint64_t Exec::pad_unit(int mode, bool copy) const {
  if (mode == dev::kPartTma) return dev::tma_chunk_bytes(tma_kib());
  if (mode == dev::kPartDynamic) return copy ? kDynCopyChunk : kDynReduceChunk;
  return dev::kQuantum;
}

void Exec::build_partition(const std::vector<uint64_t>& w0, const std::vector<uint64_t>& n,
                           const std::vector<char>& remote, double local_bytes, double remote_bytes, int grid,
                           int mode, uint64_t unit, DevPartition* out, uint64_t runit, bool taper) {
  const uint64_t total = w0.empty() ? 0 : w0.back() + n.back();
  if (runit == 0) runit = unit;
  // Tapered hand-out (the gradient return): chunks are described in quarter
  // units; the tail of every segment (the last ~2 grids' worth of work of the
  // queue, at most half of it) goes out in single quarter units, so the
  // launch's last claims are short and the CTAs finish together. A table
  // entry is (segment, start | (units - 1) << 24), in units of the quarter.
  const uint64_t div = taper ? 4 : 1;
  cudaFree(out->first_seg);
  cudaFree(out->chunks);
  cudaFree(out->rchunks);
  out->first_seg = nullptr;
  out->chunks = out->rchunks = nullptr;
  out->grid = grid;
  out->mode = mode;
  out->chunk = unit / div;
  out->rchunk = runit / div;
  out->total_chunks = out->rtotal_chunks = 0;
  out->remote_ctas = 0;
  out->lstatic = out->rstatic = 0;
  out->per_cta = 0;
  if (mode == dev::kPartDynamic || mode == dev::kPartTma) {
    // Two queues (local / remote). Hand-out order within a queue: chunk j of
    // segment s gets key (j + 0.5) / chunks(s), so every segment advances at
    // the same fractional pace; ties keep segment order.
    for (int q = 0; q < 2; ++q) {
      std::vector<std::pair<double, uint2>> order;
      const uint64_t u = q ? runit : unit, su = u / div;
      uint64_t qtotal = 0;
      for (size_t s = 0; s < n.size(); ++s)
        if ((remote[s] != 0) == (q == 1)) qtotal += n[s];
      const double tail = taper && qtotal ? std::min(0.5, 2.0 * grid * static_cast<double>(u) / qtotal) : 0.0;
      for (size_t s = 0; s < n.size(); ++s) {
        if ((remote[s] != 0) != (q == 1)) continue;
        const uint64_t k = (n[s] + su - 1) / su;  // quarter units of this segment
        if (k >= (1u << 24)) raise(ErrorCode::InvalidArgument, "segment too long for the chunk table");
        const uint64_t small = taper ? std::min<uint64_t>(k, static_cast<uint64_t>(std::ceil(tail * k))) : 0;
        for (uint64_t j = 0; j < k;) {
          const uint64_t len = j < k - small ? std::min<uint64_t>(div, k - small - j) : 1;
          order.push_back({(j + 0.5 * len) / static_cast<double>(k),
                           make_uint2(static_cast<unsigned>(s), static_cast<unsigned>(j | (len - 1) << 24))});
          j += len;
        }
      }
      std::stable_sort(order.begin(), order.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
      std::vector<uint2> table(order.size());
      for (size_t i = 0; i < order.size(); ++i) table[i] = order[i].second;
      uint2** dst = q ? &out->rchunks : &out->chunks;
      (q ? out->rtotal_chunks : out->total_chunks) = static_cast<uint32_t>(table.size());
      if (!table.empty()) {
        ck(cudaMalloc(dst, table.size() * sizeof(uint2)), "cudaMalloc(chunk table)");
        ck(cudaMemcpy(*dst, table.data(), table.size() * sizeof(uint2), cudaMemcpyHostToDevice), "upload");
      }
    }
    // Grid sized to the op: no more CTAs than chunks (a CTA without a chunk
    // only adds arrival and claim traffic); a GPU with no work for this kind
    // keeps one CTA, which posts "started" and waits for its peers.
    {
      const uint32_t chunks = out->total_chunks + out->rtotal_chunks;
      int g = static_cast<int>(std::min<uint64_t>(static_cast<uint64_t>(grid), std::max<uint32_t>(chunks, 1)));
      if (out->total_chunks && out->rtotal_chunks) g = std::max(g, std::min(grid, 2));
      grid = g;
      out->grid = g;
    }
    // CTAs that start on the remote queue ~ the remote share of the time
    // (NVLink ~770 GB/s vs HBM copy ~6.5 TB/s counted read+write).
    if (out->rtotal_chunks == 0) {
      out->remote_ctas = 0;
    } else if (out->total_chunks == 0) {
      out->remote_ctas = grid;
    } else {
      // remote_bytes: NVLink bytes; local_bytes: HBM bytes counted as a copy's (read + write) / 2
      const double tr = remote_bytes / 770e9, tl = 2.0 * local_bytes / 6.5e12;
      // HB_REMOTE_PCT overrides the remote share of the grid (tuning knob)
      static const double frac = static_cast<double>(env_u64("HB_REMOTE_PCT", 0)) / 100.0;
      const double f = frac > 0 ? frac : tr / (tr + tl);
      out->remote_ctas = grid < 2 ? 0 : std::clamp(static_cast<int>(grid * f + 0.5), 1, grid - 1);
    }
    static const int prefetch = static_cast<int>(env_u64("HB_CLAIM_PREFETCH", 1));  // A/B knob
    out->prefetch_other = prefetch;
    out->rstatic = std::min<uint32_t>(out->remote_ctas, out->rtotal_chunks);
    out->lstatic = std::min<uint32_t>(grid - out->remote_ctas, out->total_chunks);
    return;
  }
  if (mode != dev::kPartContiguous) return;
  const uint64_t per = std::max<uint64_t>(dev::kQuantum, pad_to((total + grid - 1) / grid, dev::kQuantum));
  std::vector<int32_t> first(grid, static_cast<int32_t>(w0.size()));
  size_t s = 0;
  for (int b = 0; b < grid; ++b) {
    const uint64_t lo = static_cast<uint64_t>(b) * per;
    while (s < w0.size() && w0[s] + n[s] <= lo) ++s;  // first segment ending after lo
    first[b] = static_cast<int32_t>(s);
  }
  ck(cudaMalloc(&out->first_seg, grid * sizeof(int32_t)), "cudaMalloc(partition)");
  ck(cudaMemcpy(out->first_seg, first.data(), grid * sizeof(int32_t), cudaMemcpyHostToDevice), "upload");
  out->per_cta = per;
}

void Exec::upload_copies(int mb, uint64_t unit, std::vector<uint64_t>* w0s, std::vector<uint64_t>* ns) {
  std::vector<dev::CopySeg> cs;
  uint64_t w = 0;
  w0s->clear();
  ns->clear();
  // vocab-parallel gathers: each destination rank's TP-group shard bases, [world x tp]
  const size_t tp_ = static_cast<size_t>(plan_.edge.dest.tp);
  std::vector<const unsigned char*> shard_host;
  if (cfg_.text_embedding && sharded()) {
    shard_host.assign(static_cast<size_t>(map_.world) * tp_, nullptr);
    if (mb == 0) {  // a fresh array per table rebuild (cudaFree waits for launches still reading the old one)
      cudaFree(shard_dev_);
      shard_dev_ = nullptr;
      ck(cudaMalloc(reinterpret_cast<void**>(&shard_dev_), shard_host.size() * sizeof(void*)), "cudaMalloc(shards)");
    }
  }
  for (const auto& f : fwd_local_) {
    const bool gather = f.src.slot == index::kText && cfg_.text_embedding;
    const int es = dev::dtype_size(gather ? cfg_.act_dtype : slot_dtype(f.src.slot));
    const uint64_t nbytes = static_cast<uint64_t>(f.n) * es;
    dev::CopySeg c{};
    if (gather && sharded()) {  // rows of the destination's TP-group shards
      const int r = f.src.rank;  // the TEXT ids belong to the destination rank
      const auto grp = grid::module_group(plan_.edge.dest, r, grid::GroupKind::TP);
      const int64_t rows = shard_of(grp[0]).rows;
      for (size_t i = 0; i < grp.size(); ++i) {
        const EmbedShard e = shard_of(grp[i]);
        if (!e.ptr) raise(ErrorCode::InvalidArgument, "vocab-parallel embedding: no shard set for rank " +
                                                          std::to_string(grp[i]) + " (peers: exchange bindings)");
        if (e.rows != rows || e.begin != static_cast<int64_t>(i) * rows)
          raise(ErrorCode::ShapeMismatch, "vocab-parallel embedding: shards of a TP group must be equal-sized and "
                                          "ordered by tp index (begin = tp_idx * rows)");
        shard_host[static_cast<size_t>(r) * tp_ + i] = e.ptr;
        if (gpu_of(grp[i]) != my_gpu_) c.peers |= 1u << gpu_of(grp[i]);
      }
      if (rows * static_cast<int64_t>(grp.size()) < embed_vocab_)
        raise(ErrorCode::ShapeMismatch, "vocab-parallel embedding: the TP group's shards do not cover the vocabulary");
      c.src = shard_of(grp[0]).ptr;
      c.shards = shard_dev_ + static_cast<size_t>(r) * tp_;
      c.shard_rows = static_cast<uint32_t>(rows);
      c.ids = reinterpret_cast<const int32_t*>(addr(f.src.rank, f.src.slot, mb, f.src.off / splice_d_h_, 4));
      c.row_bytes = static_cast<uint32_t>(splice_d_h_ * es);
      c.vocab = embed_vocab_;
    } else if (gather) {  // rows table[ids[k]] for the run's text rows k
      if (!embed_table_) raise(ErrorCode::InvalidArgument, "text_embedding: call set_text_embedding first");
      c.src = embed_table_;
      c.ids = reinterpret_cast<const int32_t*>(addr(f.src.rank, f.src.slot, mb, f.src.off / splice_d_h_, 4));
      c.row_bytes = static_cast<uint32_t>(splice_d_h_ * es);
      c.vocab = embed_vocab_;
    } else {
      c.src = addr(f.src.rank, f.src.slot, mb, f.src.off, es);
    }
    c.ndst = static_cast<int32_t>(f.dsts.size());
    for (size_t d = 0; d < f.dsts.size(); ++d)
      c.dst[d] = addr(f.dsts[d].rank, f.dsts[d].slot, mb, f.dsts[d].off, es);
    c.nbytes = nbytes;
    c.w0 = w;
    // the peers whose arrival this run waits for: a remote source (pull), remote destinations (push)
    if (!gather && gpu_of(f.src.rank) != my_gpu_) c.peers |= 1u << gpu_of(f.src.rank);
    for (const auto& d : f.dsts)
      if (gpu_of(d.rank) != my_gpu_) c.peers |= 1u << gpu_of(d.rank);
    if (c.peers && kWaitAllPeers) c.peers = ~0u;
    cs.push_back(c);
    w0s->push_back(w);
    ns->push_back(nbytes);
    w = pad_to(w + nbytes, unit);
  }
  if (!shard_host.empty())
    ck(cudaMemcpy(shard_dev_, shard_host.data(), shard_host.size() * sizeof(void*), cudaMemcpyHostToDevice),
       "upload(shards)");
  dev::CopySeg*& out = tables_[mb].copy;
  cudaFree(out);
  out = nullptr;
  if (!cs.empty()) {
    ck(cudaMalloc(&out, cs.size() * sizeof(dev::CopySeg)), "cudaMalloc(copy table)");
    ck(cudaMemcpy(out, cs.data(), cs.size() * sizeof(dev::CopySeg), cudaMemcpyHostToDevice), "upload");
  }
}

int Exec::tma_kib() const { return cfg_.tma_chunk_kib > 0 ? cfg_.tma_chunk_kib : kTmaChunkKiB; }

int Exec::copy_grid() const {
  if (copy_mode() == dev::kPartTma) {
    const int occ = dev::tma_blocks_per_sm(dev::tma_chunk_bytes(tma_kib()));
    return grid_cap(sm_count_ * (cfg_.blocks_per_sm > 0 ? std::min(cfg_.blocks_per_sm, occ) : occ));
  }
  const int occ = dev::copy_blocks_per_sm(cfg_.threads);
  return grid_cap(sm_count_ * (cfg_.blocks_per_sm > 0 ? std::min(cfg_.blocks_per_sm, occ) : occ));
}

void Exec::prepare_fwd() {
  if (!dirty_fwd_) return;
  if (work_dirty_) build_work();
  const int mode = copy_mode();
  const uint64_t unit = pad_unit(mode, true);
  std::vector<uint64_t> w0s, ns;
  for (int mb = 0; mb < cfg_.mb_slots; ++mb) upload_copies(mb, unit, &w0s, &ns);
  std::vector<char> rem;
  double lb = 0, rb = 0;
  for (size_t i = 0; i < fwd_local_.size(); ++i) {
    const auto& f = fwd_local_[i];
    rem.push_back(f.remote);
    // time weights: NVLink bytes of a remote run (one read in pull, one write
    // per peer destination in push); HBM read + writes of a local run
    int peer_dsts = 0;
    for (const auto& d : f.dsts) peer_dsts += gpu_of(d.rank) != my_gpu_;
    if (f.remote) rb += static_cast<double>(ns[i]) * (fwd_push_ ? peer_dsts : 1);
    else lb += static_cast<double>(ns[i]) * 0.5 * (1.0 + f.dsts.size());
  }
  build_partition(w0s, ns, rem, lb, rb, copy_grid(), mode, unit, &fwd_part_);
  dirty_fwd_ = false;
}

void Exec::prepare_bwd() {
  if (!dirty_bwd_) return;
  if (work_dirty_) build_work();
  const int mode = reduce_mode();
  uint64_t unit = pad_unit(mode, false);
  if (mode == dev::kPartDynamic && unit == 0) {
    // at least ~2 chunks per CTA, 8K..32K elements: large returns keep long
    // streaming chunks, small ones spread over the whole grid (measured: c2x4
    // at 1/8 width 12.5 -> 9.0 us with 8K chunks; C2 N=1 best at 32K)
    uint64_t total = 0;
    for (const auto& s : bwd_local_) total += static_cast<uint64_t>(s.n);
    const uint64_t grid = static_cast<uint64_t>(
        grid_cap_bwd(sm_count_ * dev::reduce_blocks_per_sm(cfg_.threads, cfg_.grad_in_dtype, cfg_.grad_out_dtype)));
    unit = 8192;
    while (unit < 32768 && total / (2 * unit) >= 2 * grid) unit *= 2;
  }
  const int es_in = dev::dtype_size(cfg_.grad_in_dtype), es_out = dev::dtype_size(cfg_.grad_out_dtype);
  // Fan-out groups: segments with the same length and the same ordered terms
  // (the TP replicas of one source shard on this GPU) become one device segment
  // that reads the terms once and accumulates into each replica (<= kMaxFan).
  // HB_RED_FAN=0 keeps one segment per accumulator (A/B knob).
  std::vector<std::vector<size_t>> groups;
  {
    static const bool fan = env_u64("HB_RED_FAN", 1) != 0;
    std::map<std::vector<int64_t>, size_t> open;  // key -> index of its group
    for (size_t i = 0; i < bwd_local_.size(); ++i) {
      const auto& sg = bwd_local_[i];
      std::vector<int64_t> key{static_cast<int64_t>(sg.n)};
      for (const auto& t : sg.terms) {
        key.push_back(t.rank);
        key.push_back(t.slot);
        key.push_back(static_cast<int64_t>(t.off));
      }
      auto it = fan ? open.find(key) : open.end();
      if (it != open.end() && groups[it->second].size() < static_cast<size_t>(dev::kMaxFan)) {
        groups[it->second].push_back(i);
      } else {
        if (fan) open[key] = groups.size();
        groups.push_back({i});
      }
    }
  }
  std::vector<uint64_t> w0s, ns;
  for (int mb = 0; mb < cfg_.mb_slots; ++mb) {
    DevTables& T = tables_[mb];
    std::vector<dev::ReduceSeg> rs;
    std::vector<const void*> terms;
    uint64_t w = 0;
    w0s.clear();
    ns.clear();
    for (const auto& grp : groups) {
      const auto& s = bwd_local_[grp[0]];
      auto acc_ptr = [&](size_t k) {
        const auto& g = bwd_local_[k];
        return addr(g.dst.rank, g.dst.slot, mb, g.dst.off, es_out);
      };
      dev::ReduceSeg d{};
      d.dst = acc_ptr(grp[0]);
      d.nelem = s.n;
      d.w0 = w;
      d.nterms = static_cast<int32_t>(s.terms.size());
      d.term0 = static_cast<int32_t>(terms.size());
      for (const auto& t : s.terms) {
        terms.push_back(addr(t.rank, t.slot, mb, t.off, es_in));
        if (gpu_of(t.rank) != my_gpu_) d.peers |= 1u << gpu_of(t.rank);
      }
      d.ndst = static_cast<int32_t>(grp.size());
      d.dst0 = static_cast<int32_t>(terms.size());
      for (size_t k : grp) terms.push_back(acc_ptr(k));
      rs.push_back(d);
      w0s.push_back(w);
      ns.push_back(s.n);
      w = pad_to(w + s.n, unit);
    }
    cudaFree(T.reduce);
    cudaFree(T.terms);
    T.reduce = nullptr;
    T.terms = nullptr;
    if (!rs.empty()) {
      ck(cudaMalloc(&T.reduce, rs.size() * sizeof(dev::ReduceSeg)), "cudaMalloc(reduce table)");
      ck(cudaMemcpy(T.reduce, rs.data(), rs.size() * sizeof(dev::ReduceSeg), cudaMemcpyHostToDevice), "upload");
    }
    if (!terms.empty()) {
      ck(cudaMalloc(&T.terms, terms.size() * sizeof(void*)), "cudaMalloc(terms)");
      ck(cudaMemcpy(T.terms, terms.data(), terms.size() * sizeof(void*), cudaMemcpyHostToDevice), "upload");
    }
  }
  const int occ = dev::reduce_blocks_per_sm(cfg_.threads, cfg_.grad_in_dtype, cfg_.grad_out_dtype);
  const int bps = cfg_.blocks_per_sm > 0 ? std::min(cfg_.blocks_per_sm, occ) : occ;
  std::vector<char> rem;
  double lb = 0, rb = 0;
  uint64_t rtotal = 0;
  for (size_t i = 0; i < groups.size(); ++i) {
    int rterms = 0;
    for (const auto& t : bwd_local_[groups[i][0]].terms) rterms += gpu_of(t.rank) != my_gpu_;
    rem.push_back(rterms > 0);
    // time weights: a remote group costs its NVLink ingress (each remote term
    // once; its HBM read-modify-write runs under the link time), a local one
    // its HBM reads + accumulator read-modify-writes
    if (rterms) {
      rb += static_cast<double>(ns[i]) * es_in * rterms;
      rtotal += ns[i];
    } else {
      lb += 0.5 * static_cast<double>(ns[i]) * (es_in * bwd_local_[groups[i][0]].terms.size() +
                                                 2 * es_out * groups[i].size());
    }
  }
  bwd_groups_ = static_cast<int>(groups.size());
  int fan = 0;
  for (const auto& g : groups) fan |= g.size() > 1;
  const int bgrid = grid_cap_bwd(sm_count_ * bps);
  // Remote chunks: longer than local ones when the return is large (every
  // stage of a chunk is in flight at once), up to half the TMA ring and while
  // every CTA still gets >= 4 remote chunks. Measured at N=4 (one box, A/B):
  // c3x4 bwd 239.6 -> 232.3 us with 16K-element remote chunks; c4 (9.4M
  // remote elements per GPU) is 2-4% slower with 16K or 32K than with 8K.
  // HB_RED_RCHUNK sets it (elements; A/B knob).
  uint64_t runit = unit;
  if (mode == dev::kPartDynamic) {
    static const uint64_t env_r = env_u64("HB_RED_RCHUNK", 0);
    const uint64_t ring_elems = dev::red_ring_elems(cfg_.grad_in_dtype);
    if (env_r) {
      runit = pad_to(env_r, 8);
    } else {
      runit = 8192;
      while (runit * 2 <= ring_elems / 2 && rtotal / (runit * 2) >= 4 * static_cast<uint64_t>(bgrid)) runit *= 2;
    }
  }
  static const bool taper = env_u64("HB_RED_TAPER", 0) != 0;  // A/B knob (off: measured slower)
  build_partition(w0s, ns, rem, lb, rb, bgrid, mode, unit, &bwd_part_, runit, taper && mode == dev::kPartDynamic);
  bwd_part_.ring = static_cast<int>(env_u64("HB_RED_RING", 1));  // A/B knob: 0 = LDG for remote chunks too
  bwd_part_.fan = fan;
  // HB_RED_STAGE_LOCAL=1: the streaming kernel stages local single-term chunks
  // through its TMA ring as well (A/B knob; off: local chunks are reduced by LDG)
  bwd_part_.stage_local = static_cast<int>(env_u64("HB_RED_STAGE_LOCAL", 0));
  dirty_bwd_ = false;
}

// Forward and backward launches keep separate counters and pad slots: each
// kind's launch count stays in lockstep across the group's GPUs (every GPU
// issues the same op sequence), and a kind's queue counters advance by a fixed
// amount per launch of that kind (boundary_kernels.cuh).
dev::SyncArgs Exec::make_sync_args(int kind, bool push) const {
  dev::SyncArgs s{};
  const uint64_t pad_off = static_cast<uint64_t>(kind) * 2 * dev::kMaxGpus;  // u32 words
  uint32_t* c = ctr_ + kind * (dev::kCtrBytes / 4);
  s.pad = reinterpret_cast<uint32_t*>(local_base_) + (local_base_ ? pad_off : 0);
  s.arrive = reinterpret_cast<unsigned long long*>(c);
  s.queue = reinterpret_cast<unsigned long long*>(c + dev::kCtrLine);
  s.fin = c + 3 * dev::kCtrLine;
  s.err = ctr_ + 3 * dev::kCtrLine + 1;  // one error word per exec
  s.my_gpu = my_gpu_;
  s.end_sync = push && n_gpus_ > 1;
  // HB_DEBUG_NO_SYNC=1 drops the cross-GPU barrier (UNSAFE; overhead experiments only).
  static const bool no_sync = [] {
    const char* v = std::getenv("HB_DEBUG_NO_SYNC");
    return v && v[0] == '1';
  }();
  if (n_gpus_ > 1 && !no_sync && ((group_mask_ >> my_gpu_) & 1u)) {
    const uint32_t peers = group_mask_ & ~(1u << my_gpu_);
    s.wait_mask = peers;
    s.post_mask = peers;
    for (int g = 0; g < n_gpus_; ++g)
      if ((peers >> g) & 1u) s.peer_pad[g] = reinterpret_cast<uint32_t*>(peer_base_[g]) + pad_off;
  }
  s.timeout_cycles = static_cast<uint64_t>(cfg_.timeout_s * clock_khz_ * 1e3);
  if (trace_) s.trace = trace_ + static_cast<size_t>(kind) * dev::kTraceMaxCtas * dev::kTraceWords;
  s.pdl = cfg_.pdl && !shared_device_ ? 1 : 0;
  return s;
}

void Exec::launch_forward(int mb_slot, void* stream) {
  const DevTables& T = tables_[mb_slot];
  dev::launch_copy(T.copy, static_cast<int>(fwd_local_.size()), fwd_part_.dev(),
                   sync_fwd_, {fwd_part_.grid, cfg_.threads}, stream);
  ck(cudaGetLastError(), "copy_segments launch");
  ++launches_;
}

void Exec::launch_backward(int mb_slot, float beta, void* stream) {
  const DevTables& T = tables_[mb_slot];
  dev::launch_reduce(T.reduce, bwd_groups_, T.terms, bwd_part_.dev(), cfg_.grad_in_dtype,
                     cfg_.grad_out_dtype, beta, sync_bwd_, {bwd_part_.grid, cfg_.threads}, stream);
  ck(cudaGetLastError(), "reduce_segments launch");
  ++launches_;
}

// The forward of set f and the gradient return of set b in one warp-specialised
// launch (dev::launch_paired); two launches when the partitions do not allow it.
bool Exec::launch_paired(int fslot, int bslot, float beta, void* stream) {
  const DevTables& F = tables_[fslot];
  const DevTables& R = tables_[bslot];
  const int grid = std::max(fwd_part_.grid, bwd_part_.grid);
  const int rc = dev::launch_paired(F.copy, fwd_part_.dev(), sync_fwd_, R.reduce, R.terms, bwd_part_.dev(),
                                    cfg_.grad_in_dtype, cfg_.grad_out_dtype, beta, sync_bwd_, grid, stream);
  if (rc == 5) ck(cudaGetLastError(), "paired_step launch");
  if (rc == 0) {
    ++launches_;
    return true;
  }
  launch_forward(fslot, stream);
  launch_backward(bslot, beta, stream);
  return false;
}

bool Exec::paired(int fwd_mb, int bwd_mb, float beta, void* stream) {
  NvtxRange nv("paired", fwd_mb);
  DeviceGuard dg(device_);
  if (!fwd_done_.count(bwd_mb))
    raise(ErrorCode::UnknownMicrobatch, "no forward record for microbatch " + std::to_string(bwd_mb));
  // bwd_mb's set is released by this call: its backward reads only the
  // gradient slots, the forward writes only the activation slots
  fwd_done_.erase(bwd_mb);
  try {
    check_forward_mb(fwd_mb);
  } catch (...) {
    fwd_done_.insert(bwd_mb);
    throw;
  }
  prepare_fwd();
  prepare_bwd();
  const bool fused = launch_paired(fwd_mb % cfg_.mb_slots, bwd_mb % cfg_.mb_slots, beta, stream);
  fwd_done_.insert(fwd_mb);
  return fused;
}

// A forward writes buffer set mb % mb_slots; a microbatch still awaiting its
// backward on the same set would have its activations (and, later, its
// gradients) overwritten, so in-flight microbatches must map to distinct sets
// (mb_slots >= microbatches in flight).
void Exec::check_forward_mb(int mb) const {
  if (mb < 0) raise(ErrorCode::InvalidArgument, "microbatch index must be >= 0");
  if (fwd_done_.count(mb))
    raise(ErrorCode::InvalidArgument, "microbatch " + std::to_string(mb) + " forwarded twice without backward");
  for (int m : fwd_done_)
    if (m % cfg_.mb_slots == mb % cfg_.mb_slots)
      raise(ErrorCode::InvalidArgument, "microbatch " + std::to_string(mb) + " shares buffer set " +
                                            std::to_string(mb % cfg_.mb_slots) + " with in-flight microbatch " +
                                            std::to_string(m) + " (raise mb_slots)");
}

void Exec::forward(int mb, void* stream) {
  NvtxRange nv("forward", mb);
  DeviceGuard dg(device_);
  check_forward_mb(mb);
  prepare_fwd();
  launch_forward(mb % cfg_.mb_slots, stream);
  fwd_done_.insert(mb);
}

void Exec::forward_projected(int mb, const void* x, int64_t ldx, const void* w, int64_t ldw, int d_h, int K,
                             int64_t x_rows, void* stream) {
  NvtxRange nv("forward_projected", mb);
  DeviceGuard dg(device_);
  check_forward_mb(mb);
  if (cfg_.act_dtype != dev::kBF16) raise(ErrorCode::InvalidArgument, "the fused projector writes bf16 activations");
  for (int r = 0; r < map_.world; ++r)
    if (map_.elems[r][index::kText])
      raise(ErrorCode::InvalidArgument, "fused projector forward on a splice edge: use forward()");
  if (d_h <= 0 || plan_.edge.feature_width % d_h)
    raise(ErrorCode::ShapeMismatch, "d_h must divide the feature width");
  if (dev::projector_check_shape(1, d_h, K))
    raise(ErrorCode::ShapeMismatch, "projector GEMM needs d_h % 256 == 0 and K % 64 == 0");
  const int slot = mb % cfg_.mb_slots;
  ProjTable& P = proj_[slot];
  const bool staged = proj_staged();
  if (P.d_h != d_h || !P.rows_dev || dirty_fwd_ || P.staged != static_cast<int>(staged)) {
    prepare_fwd();
    // token row -> destination rows, from the forward map (every destination,
    // in map order); rows are numbered over the local source ranks ascending
    std::map<int, int64_t> row_base;  // source rank -> first stacked row
    int64_t rows = 0;
    for (int r = 0; r < map_.world; ++r)
      if (map_.elems[r][index::kSrcAct] && gpu_of(r) == my_gpu_) {
        row_base[r] = rows;
        rows += map_.elems[r][index::kSrcAct] / d_h;
      }
    std::vector<std::vector<unsigned char*>> dst(rows);
    const int es = dev::dtype_size(cfg_.act_dtype);
    if (staged) {  // every row to its own source shard; the pulled forward does the rest
      for (const auto& [r, base] : row_base)
        for (int64_t i = 0; i < map_.elems[r][index::kSrcAct] / d_h; ++i)
          dst[base + i].push_back(addr(r, index::kSrcAct, slot, i * d_h, es));
    }
    for (const auto& sg : map_.fwd) {
      if (staged) break;
      // rows this GPU projects: its own source ranks' (pushed to local and peer destinations)
      if (sg.src.slot != index::kSrcAct || gpu_of(sg.src.rank) != my_gpu_) continue;
      if (sg.src.off % d_h || sg.dst.off % d_h || sg.n % d_h)
        raise(ErrorCode::ShapeMismatch, "forward runs are not whole d_h rows");
      for (int64_t i = 0; i < sg.n / d_h; ++i)
        dst[row_base.at(sg.src.rank) + sg.src.off / d_h + i].push_back(
            addr(sg.dst.rank, sg.dst.slot, slot, sg.dst.off + i * d_h, es));
    }
    int fan = 1;
    for (const auto& v : dst) fan = std::max<int>(fan, static_cast<int>(v.size()));
    std::vector<unsigned char*> flat(static_cast<size_t>(rows) * fan, nullptr);
    for (int64_t m = 0; m < rows; ++m)
      for (size_t f = 0; f < dst[m].size(); ++f) flat[m * fan + f] = dst[m][f];
    cudaFree(P.rows_dev);
    P.rows_dev = nullptr;
    ck(cudaMalloc(&P.rows_dev, flat.size() * sizeof(unsigned char*)), "cudaMalloc(projector rows)");
    ck(cudaMemcpy(P.rows_dev, flat.data(), flat.size() * sizeof(unsigned char*), cudaMemcpyHostToDevice), "upload");
    P.d_h = d_h;
    P.fan = fan;
    P.rows = static_cast<int>(rows);
    P.staged = staged;
  }
  if (P.rows > 0 && !x) raise(ErrorCode::InvalidArgument, "null projector input for the local source rows");
  // the TMA map spans P.rows x K of x: a shorter or narrower operand would be read out of bounds
  if (x_rows != P.rows)
    raise(ErrorCode::ShapeMismatch, "projector input has " + std::to_string(x_rows) + " rows, the local source ranks need " +
                                        std::to_string(P.rows));
  if (P.rows > 0 && ldx < K) raise(ErrorCode::ShapeMismatch, "projector input leading dimension < K");
  if (ldw < K) raise(ErrorCode::ShapeMismatch, "projector weight leading dimension < K");
  dev::SyncArgs ps = sync_proj_;
  if (staged) ps.wait_mask = ps.post_mask = 0, ps.end_sync = 0;  // local stores only: no cross-GPU protocol
  const dev::ProjectorArgs a{P.rows, d_h, K, P.rows_dev, P.fan, ps};
  // persistent GEMM: one CTA per SM in CTA pairs, so the cap is rounded down to even
  const int proj_ctas = cfg_.max_ctas > 0 ? std::max(2, std::min(sm_count_, cfg_.max_ctas) & ~1) : sm_count_;
  const int st = dev::launch_projector(x, ldx, w, ldw, a, proj_ctas, stream);
  if (st) raise(st == 3 ? ErrorCode::InvalidArgument : ErrorCode::CudaError,
                "projector GEMM launch failed (" + std::to_string(st) + ")");
  ++launches_;
  if (staged) launch_forward(slot, stream);  // the pulled reshard of the freshly projected shards
  fwd_done_.insert(mb);
}

bool Exec::proj_staged() const {
  static const int env = [] {  // HB_PROJ_FUSE: 1 always push, 0 always stage, unset/other: auto
    const char* v = std::getenv("HB_PROJ_FUSE");
    return v && (v[0] == '0' || v[0] == '1') ? v[0] - '0' : -1;
  }();
  if (env >= 0) return env == 0;
  // auto: stage when some row would reach one GPU more than once over NVLink
  std::map<std::tuple<int, int64_t, int>, int> arrivals;  // (source rank, element, destination GPU)
  for (const auto& sg : map_.fwd) {
    if (sg.src.slot != index::kSrcAct) continue;
    const int gs = gpu_of(sg.src.rank), gd = gpu_of(sg.dst.rank);
    if (gs == gd) continue;
    if (++arrivals[{sg.src.rank, sg.src.off, gd}] > 1) return true;
  }
  return false;
}

void Exec::backward(int mb, float beta, void* stream) {
  NvtxRange nv("backward", mb);
  DeviceGuard dg(device_);
  if (!fwd_done_.count(mb))
    raise(ErrorCode::UnknownMicrobatch, "no forward record for microbatch " + std::to_string(mb));
  prepare_bwd();
  launch_backward(mb % cfg_.mb_slots, beta, stream);
  fwd_done_.erase(mb);
}

void Exec::graph_capture(int mb_slot, int what, float beta, void* stream) {
  DeviceGuard dg(device_);
  if (mb_slot < 0 || mb_slot >= cfg_.mb_slots) raise(ErrorCode::InvalidArgument, "mb slot out of range");
  if (what < 0 || what > 5)
    raise(ErrorCode::InvalidArgument, "graph 'what' must be 0 (fwd), 1 (fwd+bwd), 2 (bwd), 3 (a step per buffer "
                                      "set), 4 (a 1F1B-paired cycle), 5 (the same cycle with fused paired steps)");
  if (what >= 4 && cfg_.mb_slots < 2) raise(ErrorCode::InvalidArgument, "a paired cycle needs mb_slots >= 2");
  if (what >= 3) mb_slot = 0;  // cycle graphs are keyed on slot 0
  if (!stream) raise(ErrorCode::InvalidArgument, "graph capture needs a non-default stream");
  if (what != 2) prepare_fwd();
  if (what != 0) prepare_bwd();
  const auto key = std::make_pair(mb_slot, what);
  auto it = graphs_.find(key);
  if (it != graphs_.end()) {
    cudaGraphExecDestroy(static_cast<cudaGraphExec_t>(it->second.first));
    graphs_.erase(it);
  }
  auto st = static_cast<cudaStream_t>(stream);
  const int before = launches_;
  ck(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal), "cudaStreamBeginCapture");
  if (what == 3) {  // fwd + bwd of buffer set 0, then 1, ... : one launch replays a full cycle
    for (int k = 0; k < cfg_.mb_slots; ++k) {
      launch_forward(k, stream);
      launch_backward(k, beta, stream);
    }
  } else if (what == 5) {  // 1F1B pairing, each pair in one fused launch
    for (int k = 0; k < cfg_.mb_slots; ++k) launch_paired(k, (k + cfg_.mb_slots - 1) % cfg_.mb_slots, beta, stream);
  } else if (what == 4) {
    // 1F1B pairing, as a pipeline's schedule call issues it (the LLM's first
    // stage receives mb k+1 and returns mb k's gradient in the same call):
    // step k = forward of set k on `stream` concurrently with the backward of
    // set k-1 on a side stream, joined before step k+1. The two ops touch
    // disjoint buffers (SRC_ACT/DST_ACT of k, DST_GRAD/SRC_GRAD of k-1) and use
    // separate per-kind counters and pads, so the only requirement is that
    // both grids fit on the GPU together (the exec's max_ctas).
    if (!side_) {
      int least = 0, greatest = 0;
      ck(cudaDeviceGetStreamPriorityRange(&least, &greatest), "priority range");
      ck(cudaStreamCreateWithPriority(&side_, cudaStreamNonBlocking, greatest), "side stream");
      ck(cudaEventCreateWithFlags(&fork_, cudaEventDisableTiming), "event");
      ck(cudaEventCreateWithFlags(&join_, cudaEventDisableTiming), "event");
    }
    for (int k = 0; k < cfg_.mb_slots; ++k) {
      ck(cudaEventRecord(fork_, st), "fork");
      ck(cudaStreamWaitEvent(side_, fork_, 0), "fork");
      launch_forward(k, stream);
      launch_backward((k + cfg_.mb_slots - 1) % cfg_.mb_slots, beta, side_);
      ck(cudaEventRecord(join_, side_), "join");
      ck(cudaStreamWaitEvent(st, join_, 0), "join");
    }
  } else {
    if (what != 2) launch_forward(mb_slot, stream);
    if (what != 0) launch_backward(mb_slot, beta, stream);
  }
  cudaGraph_t g = nullptr;
  ck(cudaStreamEndCapture(st, &g), "cudaStreamEndCapture");
  cudaGraphExec_t ge = nullptr;
  ck(cudaGraphInstantiate(&ge, g, 0), "cudaGraphInstantiate");
  cudaGraphDestroy(g);
  graphs_[key] = {ge, launches_ - before};
  launches_ = before;  // captured launches are counted when replayed
}

void Exec::graph_launch(int mb_slot, int what, void* stream) {
  NvtxRange nv(what == 0 ? "graph fwd" : what == 1 ? "graph step" : what == 2 ? "graph bwd"
               : what == 3 ? "graph cycle" : "graph paired cycle", mb_slot);
  DeviceGuard dg(device_);
  auto it = graphs_.find(std::make_pair(what >= 3 ? 0 : mb_slot, what));
  if (it == graphs_.end())
    raise(ErrorCode::InvalidArgument,
          graphs_invalidated_ ? "graph invalidated by bind / open_peers / set_text_embedding: recapture it"
                              : "no graph captured for this (mb slot, what)");
  ck(cudaGraphLaunch(static_cast<cudaGraphExec_t>(it->second.first), static_cast<cudaStream_t>(stream)),
     "cudaGraphLaunch");
  launches_ += it->second.second;
}

void Exec::seed_forward_record(int mb) {
  if (mb < 0) raise(ErrorCode::InvalidArgument, "microbatch index must be >= 0");
  fwd_done_.insert(mb);
}

void Exec::set_text_embedding(const void* table, int64_t vocab) {
  if (!cfg_.text_embedding) raise(ErrorCode::InvalidArgument, "exec was created without text_embedding");
  if (!table || vocab < 1) raise(ErrorCode::InvalidArgument, "embedding table must be non-null with vocab >= 1");
  embed_table_ = static_cast<const unsigned char*>(table);
  embed_vocab_ = vocab;
  mark_dirty();
}

void Exec::set_text_embedding_shard(int rank, const void* shard, int64_t begin, int64_t rows, int64_t vocab) {
  if (!cfg_.text_embedding) raise(ErrorCode::InvalidArgument, "exec was created without text_embedding");
  if (rank < 0 || rank >= map_.world || gpu_of(rank) != my_gpu_)
    raise(ErrorCode::InvalidArgument, "a vocab-parallel shard belongs to a rank resident on this GPU");
  if (!shard || rows < 1 || begin < 0 || vocab < 1 || rows > 0xffffffffll)
    raise(ErrorCode::InvalidArgument, "vocab-parallel shard: non-null, 1 <= rows < 2^32, begin >= 0, vocab >= 1");
  shard_[rank] = {static_cast<const unsigned char*>(shard), begin, rows};
  embed_vocab_ = vocab;
  work_dirty_ = true;  // gather runs may turn remote
  mark_dirty();
  for (Exec* p : peer_exec_)  // single-process groups read this shard directly
    if (p && p != this) {
      p->embed_vocab_ = vocab;
      p->work_dirty_ = true;
      p->mark_dirty();
    }
}

Exec::EmbedShard Exec::shard_of(int rank) const {
  const int g = gpu_of(rank);
  if (g != my_gpu_ && peer_exec_[g]) return peer_exec_[g]->shard_[rank];
  return shard_[rank];
}

bool Exec::sharded() const {
  for (int r = 0; r < map_.world; ++r)
    if (shard_of(r).ptr) return true;
  return false;
}

int Exec::read_trace(int kind, unsigned long long* out, int max_ctas, int* grid) const {
  DeviceGuard dg(device_);
  if (kind < 0 || kind >= kNumKinds) raise(ErrorCode::InvalidArgument, "trace kind out of range");
  const int g = kind == kFwdKind ? fwd_part_.grid : kind == kBwdKind ? bwd_part_.grid : 0;
  if (grid) *grid = g;
  if (!trace_ || !out) return 0;
  const int n = std::min({g, max_ctas, dev::kTraceMaxCtas});
  ck(cudaMemcpy(out, trace_ + static_cast<size_t>(kind) * dev::kTraceMaxCtas * dev::kTraceWords,
                static_cast<size_t>(n) * dev::kTraceWords * 8, cudaMemcpyDeviceToHost), "read trace");
  return n;
}

void Exec::reset_protocol() {
  DeviceGuard dg(device_);
  ck(cudaDeviceSynchronize(), "reset: synchronize");
  ck(cudaMemset(ctr_, 0, kNumKinds * dev::kCtrBytes), "reset: counters");
  if (local_base_) ck(cudaMemset(local_base_, 0, kPadBytes), "reset: signal pad");
  ck(cudaDeviceSynchronize(), "reset: synchronize");
  fwd_done_.clear();
}

uint32_t Exec::device_error() const {
  DeviceGuard dg(device_);
  uint32_t v = 0;
  ck(cudaMemcpy(&v, ctr_ + 3 * dev::kCtrLine + 1, sizeof(v), cudaMemcpyDeviceToHost), "read status");
  return v;
}

uint64_t Exec::local_fwd_bytes() const {
  uint64_t b = 0;
  for (const auto& f : fwd_local_) b += static_cast<uint64_t>(f.n) * f.dsts.size() * dev::dtype_size(cfg_.act_dtype);
  return b;
}

uint64_t Exec::local_bwd_elems() const {
  uint64_t b = 0;
  for (const auto& s : bwd_local_) b += s.n;
  return b;
}

}  // namespace hb::rt
