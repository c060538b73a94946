// hetbridge — host-owned per-module runtime (see runtime_host.hpp).
#include "hb/runtime_host.hpp"

#include <dlfcn.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <string>

#include <nccl.h>

namespace hb::rt {

namespace {
void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) raise(ErrorCode::CudaError, std::string(what) + ": " + cudaGetErrorString(e));
}

// NCCL is resolved at run time from the library the process already uses
// (torch's libnccl.so.2) so libhetbridge.so loads without it.
struct NcclApi {
  decltype(&ncclGetUniqueId) get_id = nullptr;
  decltype(&ncclCommInitRank) init = nullptr;
  decltype(&ncclCommSplit) split = nullptr;
  decltype(&ncclCommDestroy) destroy = nullptr;
  decltype(&ncclSend) send = nullptr;
  decltype(&ncclRecv) recv = nullptr;
  decltype(&ncclGroupStart) group_start = nullptr;
  decltype(&ncclGroupEnd) group_end = nullptr;
  decltype(&ncclAllGather) all_gather = nullptr;
  decltype(&ncclGetErrorString) err = nullptr;

  static const NcclApi& get() {
    static NcclApi api = [] {
      NcclApi a;
      void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
      if (!h) {
        if (const char* p = std::getenv("HB_NCCL_LIB")) h = dlopen(p, RTLD_NOW | RTLD_GLOBAL);
      }
      if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
      if (!h) raise(ErrorCode::CudaError, "libnccl.so.2 not found (import torch first or set HB_NCCL_LIB)");
      auto sym = [&](const char* n) {
        void* f = dlsym(h, n);
        if (!f) raise(ErrorCode::CudaError, std::string("NCCL symbol missing: ") + n);
        return f;
      };
      a.get_id = reinterpret_cast<decltype(a.get_id)>(sym("ncclGetUniqueId"));
      a.init = reinterpret_cast<decltype(a.init)>(sym("ncclCommInitRank"));
      a.split = reinterpret_cast<decltype(a.split)>(sym("ncclCommSplit"));
      a.destroy = reinterpret_cast<decltype(a.destroy)>(sym("ncclCommDestroy"));
      a.send = reinterpret_cast<decltype(a.send)>(sym("ncclSend"));
      a.recv = reinterpret_cast<decltype(a.recv)>(sym("ncclRecv"));
      a.group_start = reinterpret_cast<decltype(a.group_start)>(sym("ncclGroupStart"));
      a.group_end = reinterpret_cast<decltype(a.group_end)>(sym("ncclGroupEnd"));
      a.all_gather = reinterpret_cast<decltype(a.all_gather)>(sym("ncclAllGather"));
      a.err = reinterpret_cast<decltype(a.err)>(sym("ncclGetErrorString"));
      return a;
    }();
    return api;
  }
  void ok(ncclResult_t r, const char* what) const {
    if (r != ncclSuccess) raise(ErrorCode::CudaError, std::string(what) + ": " + err(r));
  }
};
}  // namespace

void nccl_unique_id(void* out128) {
  static_assert(sizeof(ncclUniqueId) == 128, "NCCL unique id size");
  const auto& n = NcclApi::get();
  ncclUniqueId id;
  n.ok(n.get_id(&id), "ncclGetUniqueId");
  std::memcpy(out128, &id, 128);
}

struct HostRuntime::Nccl {
  ncclComm_t world = nullptr;
  ncclComm_t pp = nullptr;
};

HostRuntime::HostRuntime(std::vector<grid::ModuleLayout> modules, std::vector<std::pair<int, int>> module_edges,
                         int global_batch, int feature_width, int world, int my_rank, const void* nccl_id128,
                         const HostConfig& cfg)
    : nccl_(std::make_unique<Nccl>()), modules_(std::move(modules)), module_edges_(std::move(module_edges)),
      cfg_(cfg), world_(world), rank_(my_rank) {
  if (world < 1 || my_rank < 0 || my_rank >= world) raise(ErrorCode::InvalidArgument, "bad world / rank");
  if (!nccl_id128) raise(ErrorCode::InvalidArgument, "null NCCL unique id");
  if (cfg_.nmb < 1) raise(ErrorCode::InfeasibleSchedule, "NMB must be >= 1");
  for (size_t a = 0; a < modules_.size(); ++a) {
    if (modules_[a].rank_end() > world) raise(ErrorCode::RankOutOfModule, "module '" + modules_[a].name +
                                                                            "' extends past the world");
    for (size_t b = a + 1; b < modules_.size(); ++b)
      if (modules_[a].rank_begin() < modules_[b].rank_end() && modules_[b].rank_begin() < modules_[a].rank_end())
        raise(ErrorCode::InvalidArgument, "modules '" + modules_[a].name + "' and '" + modules_[b].name +
                                              "' share ranks: the host runtime drives non-colocated modules "
                                              "(colocated edges use the three-phase PackedBoundary)");
  }
  graph_ = sched::build_stage_graph(modules_, module_edges_);
  table_ = sched::generate_1f1b_dispatch(graph_, cfg_.nmb);
  // the table the runtime executes must pass the checker
  if (const auto bad = sched::validate_dispatch(graph_, table_.cells, cfg_.nmb); !bad.empty())
    raise(ErrorCode::InfeasibleSchedule, "dispatch table fails validate_dispatch: " + bad.front());
  for (size_t m = 0; m < modules_.size(); ++m)
    if (modules_[m].contains(rank_)) {
      module_ = static_cast<int>(m);
      node_ = graph_.node_of(module_, grid::coord_of_rank(modules_[m], rank_).pp_idx);
    }
  ck(cudaGetDevice(&device_), "cudaGetDevice");

  // communicators: the world, and each module's PP groups split from it
  const auto& N = NcclApi::get();
  ncclUniqueId id;
  std::memcpy(&id, nccl_id128, 128);
  N.ok(N.init(&nccl_->world, world_, id, rank_), "ncclCommInitRank");
  int color = NCCL_SPLIT_NOCOLOR, key = 0;
  if (module_ >= 0) {
    const auto& L = modules_[module_];
    const auto c = grid::coord_of_rank(L, rank_);
    color = module_ * 65536 + (c.dp_idx * L.cp + c.cp_idx) * L.tp + c.tp_idx;
    key = c.pp_idx;
    prev_pp_ = c.pp_idx > 0 ? c.pp_idx - 1 : -1;
    next_pp_ = c.pp_idx + 1 < L.pp ? c.pp_idx + 1 : -1;
  }
  N.ok(N.split(nccl_->world, color, key, &nccl_->pp, nullptr), "ncclCommSplit");

  int least = 0, greatest = 0;
  ck(cudaDeviceGetStreamPriorityRange(&least, &greatest), "cudaDeviceGetStreamPriorityRange");
  ck(cudaStreamCreateWithPriority(&st_[0], cudaStreamNonBlocking, greatest), "boundary stream");
  ck(cudaStreamCreateWithPriority(&st_[1], cudaStreamNonBlocking, least), "PP stream");
  ck(cudaStreamCreateWithPriority(&st_[2], cudaStreamNonBlocking, least), "compute stream");

  // one boundary Exec per module edge, created on every process (collective)
  std::vector<int> ident(world_);
  for (int r = 0; r < world_; ++r) ident[r] = r;
  void* dh = nullptr;
  ck(cudaMalloc(&dh, 64 * (world_ + 1)), "cudaMalloc(handles)");
  std::vector<unsigned char> all(64 * world_);
  for (const auto& [s, d] : module_edges_) {
    grid::BoundaryEdge e{modules_[s], modules_[d], global_batch, feature_width};
    plans_.push_back(std::make_unique<bridge::BridgePlan>(bridge::plan_bridge(e)));
    ExecConfig ec;
    ec.act_dtype = cfg_.act_dtype;
    ec.grad_in_dtype = cfg_.grad_in_dtype;
    ec.grad_out_dtype = cfg_.grad_out_dtype;
    ec.mb_slots = cfg_.nmb;
    ec.max_ctas = cfg_.max_ctas;
    ec.timeout_s = cfg_.timeout_s;
    // no early-scheduled boundary CTAs holding SMs the PP stream's NCCL kernels need
    ec.pdl = 0;
    auto x = std::make_unique<Exec>(*plans_.back(), nullptr, world_, rank_, ident, ec);
    unsigned char h[64] = {0};
    x->ipc_handle(h);
    ck(cudaMemcpy(static_cast<unsigned char*>(dh) + 64 * world_, h, 64, cudaMemcpyHostToDevice), "upload handle");
    N.ok(N.all_gather(static_cast<unsigned char*>(dh) + 64 * world_, dh, 64, ncclUint8, nccl_->world, st_[2]),
         "ncclAllGather(IPC handles)");
    ck(cudaStreamSynchronize(st_[2]), "handle exchange");
    ck(cudaMemcpy(all.data(), dh, all.size(), cudaMemcpyDeviceToHost), "download handles");
    x->open_peers(all.data());
    execs_.push_back(std::move(x));
  }
  cudaFree(dh);

  // P2P stage buffers: act_in, act_out, grad_in, grad_out per microbatch
  stage_bytes_ = static_cast<size_t>((cfg_.pp_bytes + 255) / 256 * 256);
  if (stage_bytes_ && node_ >= 0) {
    ck(cudaMalloc(&stage_mem_, 4 * stage_bytes_ * cfg_.nmb), "cudaMalloc(stage buffers)");
    ck(cudaMemset(stage_mem_, 0, 4 * stage_bytes_ * cfg_.nmb), "cudaMemset(stage buffers)");
  }
  ev_.resize(4 * cfg_.nmb);
  for (auto& e : ev_) ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
  ck(cudaEventCreate(&t0_), "cudaEventCreate");
  ck(cudaEventCreate(&t1_), "cudaEventCreate");
}

HostRuntime::~HostRuntime() {
  int prev = -1;
  cudaGetDevice(&prev);
  cudaSetDevice(device_);
  for (auto* s : st_)
    if (s) cudaStreamSynchronize(s);
  execs_.clear();
  for (auto& e : ev_) cudaEventDestroy(e);
  cudaEventDestroy(t0_);
  cudaEventDestroy(t1_);
  cudaFree(stage_mem_);
  const auto& N = NcclApi::get();
  if (nccl_->pp) N.destroy(nccl_->pp);
  if (nccl_->world) N.destroy(nccl_->world);
  for (auto* s : st_)
    if (s) cudaStreamDestroy(s);
  if (prev >= 0) cudaSetDevice(prev);
}

std::vector<int> HostRuntime::group(int kind) const {
  if (module_ < 0) return {};
  if (kind < 0 || kind > 3) raise(ErrorCode::InvalidArgument, "group kind must be 0..3 (TP, CP, PP, DP)");
  return grid::module_group(modules_[module_], rank_, static_cast<grid::GroupKind>(kind));
}

Exec* HostRuntime::edge_exec(int k) const {
  if (k < 0 || k >= static_cast<int>(execs_.size())) raise(ErrorCode::InvalidArgument, "module edge out of range");
  return execs_[k].get();
}

void* HostRuntime::stage_buffer(int which, int mb, size_t* bytes) const {
  if (which < 0 || which > 3 || mb < 0 || mb >= cfg_.nmb) raise(ErrorCode::InvalidArgument, "stage buffer index");
  if (bytes) *bytes = static_cast<size_t>(cfg_.pp_bytes);
  return stage_mem_ ? stage_mem_ + (static_cast<size_t>(which) * cfg_.nmb + mb) * stage_bytes_ : nullptr;
}

cudaStream_t HostRuntime::stream(int which) const {
  if (which < 0 || which > 2) raise(ErrorCode::InvalidArgument, "stream index");
  return st_[which];
}

void HostRuntime::step(ComputeFn fn, void* user) {
  NvtxRange nv("runtime step", static_cast<int>(steps_));
  int prev = -1;
  cudaGetDevice(&prev);
  if (prev != device_) cudaSetDevice(device_);
  const auto& N = NcclApi::get();
  cudaStream_t sb = st_[0], sp = st_[1], sc = st_[2];
  ck(cudaEventRecord(t0_, sc), "record");
  ck(cudaStreamWaitEvent(sb, t0_, 0), "wait");
  ck(cudaStreamWaitEvent(sp, t0_, 0), "wait");
  const int64_t base = steps_ * cfg_.nmb;  // microbatch ids seen by the edge Execs
  const bool has_in = node_ >= 0 && !graph_.in_edges(node_).empty();
  const bool has_out = node_ >= 0 && !graph_.out_edges(node_).empty();
  size_t i = 0;
  const auto& cells = table_.cells;
  while (i < cells.size()) {
    const int row = cells[i].row;
    std::vector<const sched::Cell*> mine;
    for (; i < cells.size() && cells[i].row == row; ++i)
      if (cells[i].node == node_) mine.push_back(&cells[i]);
    if (mine.empty()) continue;
    // compute (at most one per call), then this call's sends and receives
    for (const auto* c : mine) {
      if (c->op != sched::Op::Compute) continue;
      const int mb = c->mb;
      if (!c->bwd) {
        if (has_in) ck(cudaStreamWaitEvent(sc, ev(0, mb), 0), "wait fwd in");
      } else if (has_out) {
        ck(cudaStreamWaitEvent(sc, ev(2, mb), 0), "wait bwd in");
      }
      if (fn && !(cfg_.skip & 4)) fn(user, node_, mb, c->bwd ? 1 : 0, sc);
      ck(cudaEventRecord(ev(c->bwd ? 3 : 1, mb), sc), "record compute");
    }
    std::vector<const sched::Cell*> p2p, nc;
    for (const auto* c : mine)
      if (c->op != sched::Op::Compute) (c->kind == sched::EdgeKind::P2P ? p2p : nc).push_back(c);
    if (!p2p.empty()) {
      for (const auto* c : p2p)
        if (c->op == sched::Op::SendFwd || c->op == sched::Op::SendBwd)
          ck(cudaStreamWaitEvent(sp, ev(c->op == sched::Op::SendFwd ? 1 : 3, c->mb), 0), "wait send");
      if (!(cfg_.skip & 2) && cfg_.pp_bytes > 0) {
        N.ok(N.group_start(), "ncclGroupStart");
        for (const auto* c : p2p) {
          const int which = c->op == sched::Op::RecvFwd ? 0 : c->op == sched::Op::SendFwd ? 1
                          : c->op == sched::Op::RecvBwd ? 2 : 3;
          void* buf = stage_buffer(which, c->mb, nullptr);
          const int peer = (c->op == sched::Op::SendFwd || c->op == sched::Op::RecvBwd) ? next_pp_ : prev_pp_;
          if (peer < 0) raise(ErrorCode::InvalidArgument, "P2P cell without a pipeline neighbour");
          if (c->op == sched::Op::SendFwd || c->op == sched::Op::SendBwd)
            N.ok(N.send(buf, cfg_.pp_bytes, ncclUint8, peer, nccl_->pp, sp), "ncclSend");
          else
            N.ok(N.recv(buf, cfg_.pp_bytes, ncclUint8, peer, nccl_->pp, sp), "ncclRecv");
        }
        N.ok(N.group_end(), "ncclGroupEnd");
      }
      for (const auto* c : p2p)
        if (c->op == sched::Op::RecvFwd || c->op == sched::Op::RecvBwd)
          ck(cudaEventRecord(ev(c->op == sched::Op::RecvFwd ? 0 : 2, c->mb), sp), "record recv");
    }
    // one global order of boundary ops across the GPUs (sched::nc_issue_order)
    std::stable_sort(nc.begin(), nc.end(),
                     [&](const sched::Cell* a, const sched::Cell* b) { return sched::nc_before(graph_, *a, *b); });
    // A call that hands one microbatch's gradient back and takes the next
    // microbatch's activation (Megatron's send_backward_recv_forward /
    // send_forward_recv_backward) issues both boundary ops of the same edge
    // as one fused paired launch (HB_RT_PAIRED=1, read per step; default off):
    // the two ops overlap on every SM. Peers that issue the ops separately
    // interoperate (each op is still one op of its kind's epoch sequence).
    // Measured at N=4 with event-only compute (profiles/r02/host_runtime_paired_n4.json):
    // boundary-only steps 24-32% shorter, but a paired Recv also waits for its
    // partner Send's compute event, so on a P2P-bound table (c5w4) the
    // forward can no longer run ahead and the full step is 9% longer; on join4
    // it is 16% shorter. Pairing only Send->Recv (where the Recv was queued
    // behind that wait anyway) measured no gain either way.
    const char* pe = std::getenv("HB_RT_PAIRED");
    const bool pair_ops = pe && pe[0] == '1';
    auto is_fwd = [](sched::Op o) { return o == sched::Op::SendFwd || o == sched::Op::RecvFwd; };
    for (size_t j = 0; j < nc.size(); ++j) {
      const auto* c = nc[j];
      Exec* x = execs_.at(graph_.edges[c->edge].boundary).get();
      const int64_t id = base + c->mb;
      if (pair_ops && !(cfg_.skip & 1) && j + 1 < nc.size() &&
          graph_.edges[nc[j + 1]->edge].boundary == graph_.edges[c->edge].boundary &&
          is_fwd(c->op) != is_fwd(nc[j + 1]->op) &&
          c->mb != nc[j + 1]->mb) {
        const auto* f = is_fwd(c->op) ? c : nc[j + 1];
        const auto* b = is_fwd(c->op) ? nc[j + 1] : c;
        if (f->op == sched::Op::SendFwd) ck(cudaStreamWaitEvent(sb, ev(1, f->mb), 0), "wait");
        if (b->op == sched::Op::SendBwd) ck(cudaStreamWaitEvent(sb, ev(3, b->mb), 0), "wait");
        x->paired(static_cast<int>(base + f->mb), static_cast<int>(base + b->mb), 0.0f, sb);
        ++paired_ops_;
        if (f->op == sched::Op::RecvFwd) ck(cudaEventRecord(ev(0, f->mb), sb), "record");
        if (b->op == sched::Op::RecvBwd) ck(cudaEventRecord(ev(2, b->mb), sb), "record");
        ++j;
        continue;
      }
      switch (c->op) {
        case sched::Op::SendFwd:  // encoder last stage: its activation is ready
          ck(cudaStreamWaitEvent(sb, ev(1, c->mb), 0), "wait");
          if (!(cfg_.skip & 1)) x->forward(static_cast<int>(id), sb);
          break;
        case sched::Op::RecvFwd:  // LLM first stage pulls the rows it needs
          if (!(cfg_.skip & 1)) x->forward(static_cast<int>(id), sb);
          ck(cudaEventRecord(ev(0, c->mb), sb), "record");
          break;
        case sched::Op::SendBwd:  // LLM first stage: its input gradient is ready
          ck(cudaStreamWaitEvent(sb, ev(3, c->mb), 0), "wait");
          if (!(cfg_.skip & 1)) x->backward(static_cast<int>(id), 0.0f, sb);
          break;
        case sched::Op::RecvBwd:  // encoder last stage pulls its gradients back
          if (!(cfg_.skip & 1)) x->backward(static_cast<int>(id), 0.0f, sb);
          ck(cudaEventRecord(ev(2, c->mb), sb), "record");
          break;
        default: break;
      }
    }
  }
  // join the step's streams into the compute stream
  cudaEvent_t jb = ev(0, 0), jp = ev(2, 0);
  ck(cudaEventRecord(jb, sb), "record");
  ck(cudaEventRecord(jp, sp), "record");
  ck(cudaStreamWaitEvent(sc, jb, 0), "join");
  ck(cudaStreamWaitEvent(sc, jp, 0), "join");
  ck(cudaEventRecord(t1_, sc), "record");
  ++steps_;
  if (prev >= 0 && prev != device_) cudaSetDevice(prev);
}

float HostRuntime::last_step_ms() {
  float ms = 0;
  ck(cudaEventSynchronize(t1_), "sync");
  ck(cudaEventElapsedTime(&ms, t0_, t1_), "elapsed");
  for (const auto& x : execs_)
    if (x->device_error()) raise(ErrorCode::Timeout, "boundary flag wait timed out on the device");
  return ms;
}

}  // namespace hb::rt
