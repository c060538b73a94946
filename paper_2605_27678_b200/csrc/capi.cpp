// hetbridge — C-ABI implementation (include/hetbridge.h). Every entry point
// catches hb::Error and maps it to `ErrorCode ordinal + 1`; nothing throws
// across the boundary.
#include "hetbridge.h"

#include <cstring>
#include <map>
#include <mutex>

#include <cuda_runtime.h>
#include <memory>
#include <string>

#include "hb/bridge.hpp"
#include "hb/config.hpp"
#include "hb/index_map.hpp"
#include "hb/runtime.hpp"
#include "hb/runtime_host.hpp"
#include "hb/sched.hpp"
#include "kernels/projector_gemm.cuh"

struct hb_plan {
  hb::bridge::BridgePlan plan;
};
struct hb_splice {
  hb::index::SpliceSpec spec;
};
struct hb_exec {
  std::unique_ptr<hb::rt::Exec> own;
  hb::rt::Exec* x = nullptr;
  bool borrowed = false;  // an edge Exec of an hb_runtime (owned by it)
};
struct hb_runtime {
  std::unique_ptr<hb::rt::HostRuntime> r;
  std::vector<std::unique_ptr<hb_exec>> edge_execs;
};
struct hb_config {
  hb::config::ExperimentConfig c;
};
struct hb_stage_graph {
  hb::sched::StageGraph g;
};

namespace {
thread_local std::string g_err;

template <class F>
int guard(F&& f) {
  try {
    f();
    return HB_OK;
  } catch (const hb::Error& e) {
    g_err = e.what();
    return static_cast<int>(e.code()) + 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return static_cast<int>(hb::ErrorCode::InvalidArgument) + 1;
  }
}

void need(const void* p, const char* what) {
  if (!p) hb::raise(hb::ErrorCode::InvalidArgument, std::string("null ") + what);
}

hb::grid::ModuleLayout layout(const hb_layout* l) {
  need(l, "layout");
  hb::grid::ModuleLayout m;
  m.name = l->name ? l->name : "";
  m.tp = l->tp;
  m.cp = l->cp;
  m.pp = l->pp;
  m.dp = l->dp;
  m.rank_offset = l->rank_offset;
  return m;
}

hb::grid::BoundaryEdge edge(const hb_edge* e) {
  need(e, "edge");
  return {layout(&e->source), layout(&e->dest), e->global_batch, e->feature_width};
}

void fill(const std::vector<int>& v, int* out, int cap, int* n) {
  need(n, "count");
  *n = static_cast<int>(v.size());
  for (int i = 0; i < cap && i < *n; ++i) out[i] = v[i];
}

const hb::index::SpliceSpec* spec(const hb_splice* s) { return s ? &s->spec : nullptr; }
}  // namespace

extern "C" {

size_t hb_last_error(char* buf, size_t cap) {
  if (buf && cap) {
    const size_t n = std::min(cap - 1, g_err.size());
    std::memcpy(buf, g_err.data(), n);
    buf[n] = 0;
  }
  return g_err.size();
}

const char* hb_error_name(int status) {
  if (status == HB_OK) return "OK";
  return hb::error_code_name(static_cast<hb::ErrorCode>(status - 1));
}

int hb_abi_version(void) { return 7; }

int hb_coord_of_rank(const hb_layout* l, int rank, int coord4[4]) {
  return guard([&] {
    need(coord4, "coord");
    const auto c = hb::grid::coord_of_rank(layout(l), rank);
    coord4[0] = c.tp_idx;
    coord4[1] = c.cp_idx;
    coord4[2] = c.pp_idx;
    coord4[3] = c.dp_idx;
  });
}

int hb_rank_of_coord(const hb_layout* l, const int coord4[4], int* rank) {
  return guard([&] {
    need(coord4, "coord");
    need(rank, "rank");
    *rank = hb::grid::rank_of_coord(layout(l), {coord4[0], coord4[1], coord4[2], coord4[3]});
  });
}

int hb_partition_batch(int batch, int dp, int* start_len, int cap_pairs) {
  return guard([&] {
    const auto v = hb::grid::partition_batch(batch, dp);
    for (int i = 0; i < cap_pairs && i < static_cast<int>(v.size()); ++i) {
      start_len[2 * i] = v[i].start;
      start_len[2 * i + 1] = v[i].length;
    }
  });
}

int hb_leader_rank(const hb_layout* l, int pp, int dp, int* rank) {
  return guard([&] {
    need(rank, "rank");
    *rank = hb::grid::leader_rank(layout(l), pp, dp);
  });
}

int hb_placement_of_edge(const hb_edge* e, int* placement) {
  return guard([&] {
    need(placement, "placement");
    *placement = static_cast<int>(hb::grid::placement_of_edge(edge(e)));
  });
}

int hb_ranks_of_stage(const hb_layout* l, int pp, int* out, int cap, int* n) {
  return guard([&] { fill(hb::grid::ranks_of_stage(layout(l), pp), out, cap, n); });
}

int hb_replica_group(const hb_layout* l, int pp, int dp, int* out, int cap, int* n) {
  return guard([&] { fill(hb::grid::replica_group(layout(l), pp, dp), out, cap, n); });
}

int hb_module_group(const hb_layout* l, int rank, int kind, int* out, int cap, int* n) {
  return guard([&] {
    if (kind < 0 || kind > 3) hb::raise(hb::ErrorCode::InvalidArgument, "group kind must be 0..3");
    fill(hb::grid::module_group(layout(l), rank, static_cast<hb::grid::GroupKind>(kind)), out, cap, n);
  });
}

int hb_classify_dp_relation(const hb_edge* e, int* kind, int* factor) {
  return guard([&] {
    need(kind, "kind");
    need(factor, "factor");
    const auto r = hb::bridge::classify_dp_relation(edge(e));
    *kind = static_cast<int>(r.kind);
    *factor = r.factor;
  });
}

int hb_plan_create(const hb_edge* e, hb_plan** out) {
  return guard([&] {
    need(out, "out");
    *out = nullptr;
    auto p = std::make_unique<hb_plan>();
    p->plan = hb::bridge::plan_bridge(edge(e));
    *out = p.release();
  });
}

void hb_plan_destroy(hb_plan* p) { delete p; }

int hb_plan_export(const hb_plan* p, int elem_bytes, char* buf, size_t cap, size_t* len) {
  return guard([&] {
    need(p, "plan");
    if (elem_bytes < 1) hb::raise(hb::ErrorCode::InvalidArgument, "elem_bytes must be >= 1");
    const std::string s = hb::bridge::export_plan(p->plan, elem_bytes);
    if (len) *len = s.size();
    if (buf && cap) {
      const size_t n = std::min(cap - 1, s.size());
      std::memcpy(buf, s.data(), n);
      buf[n] = 0;
    }
  });
}

int hb_config_parse(const char* text, hb_config** out) {
  return guard([&] {
    need(text, "text");
    need(out, "out");
    *out = nullptr;
    auto c = std::make_unique<hb_config>();
    c->c = hb::config::parse_config(text);
    *out = c.release();
  });
}

void hb_config_destroy(hb_config* c) { delete c; }

int hb_config_num_modules(const hb_config* c, int* n) {
  return guard([&] {
    need(c, "config");
    need(n, "n");
    *n = static_cast<int>(c->c.modules.size());
  });
}

int hb_config_module(const hb_config* c, int i, hb_layout* out, int* is_language) {
  return guard([&] {
    need(c, "config");
    need(out, "out");
    if (i < 0 || i >= static_cast<int>(c->c.modules.size()))
      hb::raise(hb::ErrorCode::InvalidArgument, "module index out of range");
    const auto& l = c->c.modules[i].layout;
    *out = {l.name.c_str(), l.tp, l.cp, l.pp, l.dp, l.rank_offset};
    if (is_language) *is_language = l.name == "language";
  });
}

int hb_config_run(const hb_config* c, int* global_batch, int* num_microbatches, int* steps, long long* seed,
                  double* tolerance) {
  return guard([&] {
    need(c, "config");
    if (global_batch) *global_batch = c->c.global_batch;
    if (num_microbatches) *num_microbatches = c->c.num_microbatches;
    if (steps) *steps = c->c.steps;
    if (seed) *seed = c->c.seed;
    if (tolerance) *tolerance = c->c.tolerance;
  });
}

int hb_config_edge(const hb_config* c, const char* encoder, int feature_width, hb_edge* out) {
  return guard([&] {
    need(c, "config");
    need(encoder, "encoder");
    need(out, "out");
    const auto e = c->c.edge(encoder, feature_width);
    const auto& s = c->c.module(e.source.name).layout;
    const auto& d = c->c.language().layout;
    *out = {{s.name.c_str(), s.tp, s.cp, s.pp, s.dp, s.rank_offset},
            {d.name.c_str(), d.tp, d.cp, d.pp, d.dp, d.rank_offset},
            e.global_batch,
            e.feature_width};
  });
}

int hb_config_render(const hb_config* c, char* buf, size_t cap, size_t* len) {
  return guard([&] {
    need(c, "config");
    const std::string s = hb::config::render_config(c->c);
    if (len) *len = s.size();
    if (buf && cap) {
      const size_t n = std::min(cap - 1, s.size());
      std::memcpy(buf, s.data(), n);
      buf[n] = 0;
    }
  });
}

int hb_plan_info(const hb_plan* p, int* placement, int* kind, int* factor, int* xmsgs, int* world) {
  return guard([&] {
    need(p, "plan");
    const auto& b = p->plan;
    if (placement) *placement = static_cast<int>(b.placement);
    if (kind) *kind = static_cast<int>(b.relation.kind);
    if (factor) *factor = b.relation.factor;
    if (xmsgs) *xmsgs = b.cross_boundary_messages();
    if (world) *world = std::max(b.edge.source.rank_end(), b.edge.dest.rank_end());
  });
}

int hb_cp_token_slice(int seq_len, int cp, int cp_idx, int* start, int* length) {
  return guard([&] {
    need(start, "start");
    need(length, "length");
    if (cp < 1 || cp_idx < 0 || cp_idx >= cp) hb::raise(hb::ErrorCode::InvalidArgument, "cp index out of range");
    if (seq_len % cp)
      hb::raise(hb::ErrorCode::DivisibilityViolation, "seq_len not divisible by cp");
    *length = seq_len / cp;
    *start = cp_idx * *length;
  });
}

int hb_splice_create(int Q, int S, int d_h, int S_v, int text_mode, const int* codes, hb_splice** out) {
  return guard([&] {
    need(out, "out");
    need(codes, "codes");
    if (Q < 1 || S < 1) hb::raise(hb::ErrorCode::InvalidArgument, "Q and S must be >= 1");
    if (text_mode != HB_TEXT_FULL && text_mode != HB_TEXT_SLICE && text_mode != HB_TEXT_INPLACE)
      hb::raise(hb::ErrorCode::InvalidArgument, "unknown text mode");
    auto s = std::make_unique<hb_splice>();
    s->spec.Q = Q;
    s->spec.S = S;
    s->spec.d_h = d_h;
    s->spec.S_v = S_v;
    s->spec.text_mode = static_cast<hb::index::TextMode>(text_mode);
    s->spec.codes.assign(codes, codes + static_cast<size_t>(Q) * S);
    *out = s.release();
  });
}

void hb_splice_destroy(hb_splice* s) { delete s; }

int hb_index_forward(const hb_plan* p, const hb_splice* s, hb_copy_seg* out, size_t cap, size_t* n) {
  return guard([&] {
    need(p, "plan");
    need(n, "count");
    const auto m = hb::index::build_index_map(p->plan, spec(s));
    *n = m.fwd.size();
    for (size_t i = 0; out && i < cap && i < m.fwd.size(); ++i) {
      const auto& c = m.fwd[i];
      out[i] = {c.src.rank, c.src.slot, c.src.off, c.dst.rank, c.dst.slot, c.dst.off, c.n};
    }
  });
}

namespace {
int index_backward(const hb_plan* p, const hb_splice* s, bool balanced, hb_reduce_seg* out, size_t cap, size_t* n,
                   hb_ref* terms, size_t tcap, size_t* tn) {
  return guard([&] {
    need(p, "plan");
    need(n, "count");
    const auto m = hb::index::build_index_map(p->plan, spec(s), balanced);
    *n = m.bwd.size();
    size_t t = 0;
    for (size_t i = 0; i < m.bwd.size(); ++i) {
      const auto& r = m.bwd[i];
      if (out && i < cap)
        out[i] = {r.dst.rank, r.dst.slot, r.dst.off, r.n, static_cast<int>(r.terms.size()), static_cast<int>(t)};
      for (const auto& x : r.terms) {
        if (terms && t < tcap) terms[t] = {x.rank, x.slot, x.off};
        ++t;
      }
    }
    if (tn) *tn = t;
  });
}
}  // namespace

int hb_index_backward(const hb_plan* p, const hb_splice* s, hb_reduce_seg* out, size_t cap, size_t* n,
                      hb_ref* terms, size_t tcap, size_t* tn) {
  return index_backward(p, s, false, out, cap, n, terms, tcap, tn);
}

int hb_index_backward_balanced(const hb_plan* p, const hb_splice* s, hb_reduce_seg* out, size_t cap, size_t* n,
                               hb_ref* terms, size_t tcap, size_t* tn) {
  return index_backward(p, s, true, out, cap, n, terms, tcap, tn);
}

int hb_index_buffer_elems(const hb_plan* p, const hb_splice* s, int rank, int slot, long long* elems) {
  return guard([&] {
    need(p, "plan");
    need(elems, "elems");
    const auto m = hb::index::build_index_map(p->plan, spec(s));
    if (rank < 0 || rank >= m.world || slot < 0 || slot >= hb::index::kNumSlots)
      hb::raise(hb::ErrorCode::InvalidArgument, "rank/slot out of range");
    *elems = m.elems[rank][slot];
  });
}

void hb_exec_config_default(hb_exec_config* c) {
  if (!c) return;
  hb::rt::ExecConfig d;
  c->act_dtype = d.act_dtype;
  c->grad_in_dtype = d.grad_in_dtype;
  c->grad_out_dtype = d.grad_out_dtype;
  c->mb_slots = d.mb_slots;
  c->internal_alloc = d.internal_alloc;
  c->blocks_per_sm = d.blocks_per_sm;
  c->threads = d.threads;
  c->timeout_s = d.timeout_s;
  c->fwd_mode = d.fwd_mode;
  c->partition = d.partition;
  c->strict_provenance = d.strict_provenance;
  c->text_embedding = d.text_embedding;
  c->max_ctas = d.max_ctas;
  c->max_ctas_bwd = d.max_ctas_bwd;
  c->tma_chunk_kib = d.tma_chunk_kib;
}

int hb_exec_create(const hb_plan* p, const hb_splice* s, int n_gpus, int my_gpu, const int* rank_to_gpu,
                   int n_ranks, const hb_exec_config* cfg, hb_exec** out) {
  return guard([&] {
    need(p, "plan");
    need(out, "out");
    *out = nullptr;
    hb::rt::ExecConfig c;
    if (cfg) {
      c.act_dtype = cfg->act_dtype;
      c.grad_in_dtype = cfg->grad_in_dtype;
      c.grad_out_dtype = cfg->grad_out_dtype;
      c.mb_slots = cfg->mb_slots;
      c.internal_alloc = cfg->internal_alloc;
      c.blocks_per_sm = cfg->blocks_per_sm > 0 ? cfg->blocks_per_sm : c.blocks_per_sm;
      c.threads = cfg->threads > 0 ? cfg->threads : c.threads;
      c.timeout_s = cfg->timeout_s > 0 ? cfg->timeout_s : c.timeout_s;
      c.fwd_mode = cfg->fwd_mode;
      c.partition = cfg->partition;
      c.strict_provenance = cfg->strict_provenance;
      c.text_embedding = cfg->text_embedding;
      c.max_ctas = cfg->max_ctas > 0 ? cfg->max_ctas : 0;
      c.max_ctas_bwd = cfg->max_ctas_bwd > 0 ? cfg->max_ctas_bwd : 0;
      c.tma_chunk_kib = cfg->tma_chunk_kib;
      if (c.tma_chunk_kib && c.tma_chunk_kib != 8 && c.tma_chunk_kib != 16 && c.tma_chunk_kib != 32)
        hb::raise(hb::ErrorCode::InvalidArgument, "tma_chunk_kib must be 0, 8, 16 or 32");
    }
    std::vector<int> map;
    if (rank_to_gpu) map.assign(rank_to_gpu, rank_to_gpu + n_ranks);
    else map.assign(n_ranks, 0);
    auto x = std::make_unique<hb_exec>();
    x->own = std::make_unique<hb::rt::Exec>(p->plan, spec(s), n_gpus, my_gpu, std::move(map), c);
    x->x = x->own.get();
    *out = x.release();
  });
}

void hb_exec_destroy(hb_exec* x) {
  if (x && !x->borrowed) delete x;
}

int hb_exec_ipc_handle(hb_exec* x, void* out64) {
  return guard([&] {
    need(x, "exec");
    need(out64, "out");
    x->x->ipc_handle(out64);
  });
}

int hb_exec_open_peers(hb_exec* x, const void* handles, size_t nbytes) {
  return guard([&] {
    need(x, "exec");
    need(handles, "handles");
    (void)nbytes;
    x->x->open_peers(handles);
  });
}

int hb_exec_open_peers_local(hb_exec* x, hb_exec* const* execs, int n) {
  return guard([&] {
    need(x, "exec");
    need(execs, "execs");
    if (n < 1 || n > hb::dev::kMaxGpus) hb::raise(hb::ErrorCode::InvalidArgument, "bad exec count");
    std::vector<hb::rt::Exec*> v(n, nullptr);
    for (int g = 0; g < n; ++g) v[g] = execs[g] ? execs[g]->x : nullptr;
    x->x->open_peers_local(v.data(), n);
  });
}

int hb_exec_buffer(hb_exec* x, int rank, int slot, int mb_slot, void** ptr, size_t* bytes) {
  return guard([&] {
    need(x, "exec");
    need(ptr, "ptr");
    *ptr = x->x->buffer(rank, slot, mb_slot, bytes);
  });
}

int hb_exec_bind(hb_exec* x, int rank, int slot, int mb_slot, void* ptr, size_t bytes) {
  return guard([&] {
    need(x, "exec");
    x->x->bind(rank, slot, mb_slot, ptr, bytes);
  });
}

int hb_exec_bind_strided(hb_exec* x, int rank, int slot, int mb_slot, void* ptr, size_t bytes, long long row_stride) {
  return guard([&] {
    need(x, "exec");
    x->x->bind(rank, slot, mb_slot, ptr, bytes, row_stride);
  });
}

int hb_exec_export_bindings(hb_exec* x, void* buf, size_t cap, size_t* len) {
  return guard([&] {
    need(x, "exec");
    need(len, "len");
    *len = x->x->export_bindings(buf, cap);
    if (buf && cap < *len) hb::raise(hb::ErrorCode::InvalidArgument, "binding buffer too small");
  });
}

int hb_exec_import_bindings(hb_exec* x, int gpu, const void* blob, size_t len) {
  return guard([&] {
    need(x, "exec");
    need(blob, "blob");
    x->x->import_bindings(gpu, blob, len);
  });
}

int hb_exec_forward(hb_exec* x, int mb, void* stream) {
  return guard([&] {
    need(x, "exec");
    x->x->forward(mb, stream);
  });
}

int hb_exec_backward(hb_exec* x, int mb, float beta, void* stream) {
  return guard([&] {
    need(x, "exec");
    x->x->backward(mb, beta, stream);
  });
}

int hb_exec_paired(hb_exec* x, int fwd_mb, int bwd_mb, float beta, void* stream, int* fused) {
  return guard([&] {
    need(x, "exec");
    const bool f = x->x->paired(fwd_mb, bwd_mb, beta, stream);
    if (fused) *fused = f ? 1 : 0;
  });
}

int hb_exec_graph_capture(hb_exec* x, int mb_slot, int what, float beta, void* stream) {
  return guard([&] {
    need(x, "exec");
    x->x->graph_capture(mb_slot, what, beta, stream);
  });
}

int hb_exec_graph_launch(hb_exec* x, int mb_slot, int what, void* stream) {
  return guard([&] {
    need(x, "exec");
    x->x->graph_launch(mb_slot, what, stream);
  });
}

int hb_exec_seed_forward_record(hb_exec* x, int mb) {
  return guard([&] {
    need(x, "exec");
    x->x->seed_forward_record(mb);
  });
}

int hb_exec_reset_protocol(hb_exec* x) {
  return guard([&] {
    need(x, "exec");
    x->x->reset_protocol();
  });
}

int hb_exec_status(hb_exec* x, unsigned* device_error) {
  return guard([&] {
    need(x, "exec");
    const unsigned e = x->x->device_error();
    if (device_error) *device_error = e;
    if (e == hb::dev::kErrBadId) hb::raise(hb::ErrorCode::InvalidArgument, "text token id outside [0, vocab)");
    if (e == hb::dev::kErrOutOfTurn)
      hb::raise(hb::ErrorCode::GroupMismatch,
                "a peer GPU started a boundary op two or more ahead of this one: the group's op sequences diverged");
    if (e) hb::raise(hb::ErrorCode::Timeout, "cross-GPU flag wait timed out on the device");
  });
}

int hb_exec_stats(hb_exec* x, long long* fs, long long* bs, long long* fb, long long* be, long long* nl) {
  return guard([&] {
    need(x, "exec");
    if (fs) *fs = x->x->local_fwd_segments();
    if (bs) *bs = x->x->local_bwd_segments();
    if (fb) *fb = static_cast<long long>(x->x->local_fwd_bytes());
    if (be) *be = static_cast<long long>(x->x->local_bwd_elems());
    if (nl) *nl = x->x->launches();
  });
}

int hb_exec_trace(hb_exec* x, int kind, unsigned long long* out, int max_ctas, int* n_ctas, int* grid) {
  return guard([&] {
    need(x, "exec");
    const int n = x->x->read_trace(kind, out, max_ctas, grid);
    if (n_ctas) *n_ctas = n;
  });
}

int hb_exec_validate(hb_exec* x, long long* checks) {
  return guard([&] {
    need(x, "exec");
    uint64_t n = 0;
    const std::string why = x->x->validate(&n);
    if (checks) *checks = static_cast<long long>(n);
    if (!why.empty()) hb::raise(hb::ErrorCode::ValidationError, "device tables: " + why);
  });
}

int hb_exec_set_text_embedding_shard(hb_exec* x, int rank, const void* shard, long long vocab_begin, long long rows,
                                     long long vocab) {
  return guard([&] {
    need(x, "exec");
    x->x->set_text_embedding_shard(rank, shard, vocab_begin, rows, vocab);
  });
}

int hb_exec_set_text_embedding(hb_exec* x, const void* table, long long vocab) {
  return guard([&] {
    need(x, "exec");
    x->x->set_text_embedding(table, vocab);
  });
}

int hb_exec_forward_projected(hb_exec* x, int mb, const void* act, long long x_rows, long long ldx, const void* w,
                              long long ldw, int d_h, int K, void* cuda_stream) {
  return guard([&] {
    need(x, "exec");
    need(w, "w");  // act may be null when this GPU hosts no source rank
    x->x->forward_projected(mb, act, ldx, w, ldw, d_h, K, x_rows, cuda_stream);
  });
}

int hb_projector_gemm(const void* x, long long ldx, const void* w, long long ldw, void* const* row_dst, int fan,
                      int M, int N, int K, void* cuda_stream) {
  return guard([&] {
    need(x, "x");
    need(w, "w");
    need(row_dst, "row_dst");
    if (fan < 1) hb::raise(hb::ErrorCode::InvalidArgument, "fan must be >= 1");
    if (hb::dev::projector_check_shape(M, N, K))
      hb::raise(hb::ErrorCode::ShapeMismatch, "projector GEMM needs N % 256 == 0 and K % 64 == 0");
    // standalone GEMM: no peers, no launch protocol (counters must still be valid)
    static std::mutex mu;
    static std::map<int, unsigned long long*> per_device;
    int dev = 0;
    cudaGetDevice(&dev);
    unsigned long long* scratch = nullptr;
    {
      std::lock_guard<std::mutex> lk(mu);
      auto& p = per_device[dev];
      if (!p) {
        void* q = nullptr;
        if (cudaMalloc(&q, hb::dev::kCtrBytes) != cudaSuccess || cudaMemset(q, 0, hb::dev::kCtrBytes) != cudaSuccess)
          hb::raise(hb::ErrorCode::CudaError, "projector scratch counters");
        p = static_cast<unsigned long long*>(q);
      }
      scratch = p;
    }
    hb::dev::SyncArgs none{};
    none.arrive = scratch;
    none.queue = scratch + hb::dev::kCtrLine / 2;
    none.fin = reinterpret_cast<uint32_t*>(scratch) + 3 * hb::dev::kCtrLine;
    none.err = none.fin + 1;
    hb::dev::ProjectorArgs a{M, N, K, reinterpret_cast<unsigned char* const*>(row_dst), fan, none};
    const int st = hb::dev::launch_projector(x, ldx, w, ldw, a, hb::dev::device_sm_count(), cuda_stream);
    if (st == 3) hb::raise(hb::ErrorCode::InvalidArgument, "projector operands must be 16-B aligned");
    if (st) hb::raise(hb::ErrorCode::CudaError, "projector GEMM launch failed (" + std::to_string(st) + ")");
  });
}

/* ---- graph-aware dispatch (SPEC.md:358-437 sched) ---------------------------- */

int hb_stage_graph_create(const hb_layout* modules, int n_modules, const int* edge_src, const int* edge_dst,
                          int n_edges, hb_stage_graph** out) {
  return guard([&] {
    need(modules, "modules");
    need(out, "out");
    *out = nullptr;
    std::vector<hb::grid::ModuleLayout> ms;
    for (int i = 0; i < n_modules; ++i) ms.push_back(layout(&modules[i]));
    std::vector<std::pair<int, int>> es;
    for (int i = 0; i < n_edges; ++i) es.emplace_back(edge_src[i], edge_dst[i]);
    auto g = std::make_unique<hb_stage_graph>();
    g->g = hb::sched::build_stage_graph(ms, es);
    *out = g.release();
  });
}

void hb_stage_graph_destroy(hb_stage_graph* g) { delete g; }

int hb_stage_graph_nodes(const hb_stage_graph* g, int* out, int cap, int* n) {
  return guard([&] {
    need(g, "graph");
    need(n, "n");
    *n = static_cast<int>(g->g.nodes.size());
    for (int i = 0; out && i < *n && i < cap; ++i) {
      out[3 * i] = g->g.nodes[i].module;
      out[3 * i + 1] = g->g.nodes[i].pp;
      out[3 * i + 2] = g->g.nodes[i].distance;
    }
  });
}

int hb_stage_graph_edges(const hb_stage_graph* g, int* out, int cap, int* n) {
  return guard([&] {
    need(g, "graph");
    need(n, "n");
    *n = static_cast<int>(g->g.edges.size());
    for (int i = 0; out && i < *n && i < cap; ++i) {
      const auto& e = g->g.edges[i];
      out[4 * i] = e.src;
      out[4 * i + 1] = e.dst;
      out[4 * i + 2] = static_cast<int>(e.kind);
      out[4 * i + 3] = e.boundary;
    }
  });
}

namespace {
hb_cell to_c(const hb::sched::Cell& c) {
  return {c.row, c.node, static_cast<int>(c.op), c.edge, static_cast<int>(c.kind), c.mb, c.bwd ? 1 : 0};
}
hb::sched::Cell from_c(const hb_cell& c) {
  return {c.row, c.node, static_cast<hb::sched::Op>(c.op), c.edge, static_cast<hb::sched::EdgeKind>(c.kind), c.mb,
          c.bwd != 0};
}
void put_text(const std::string& s, char* buf, size_t cap, size_t* len) {
  need(len, "len");
  *len = s.size();
  if (buf && cap) {
    const size_t n = std::min(cap - 1, s.size());
    std::memcpy(buf, s.data(), n);
    buf[n] = 0;
  }
}
}  // namespace

int hb_dispatch_generate(const hb_stage_graph* g, int nmb, hb_cell* cells, size_t cap, size_t* n, int* rows) {
  return guard([&] {
    need(g, "graph");
    need(n, "n");
    const auto t = hb::sched::generate_1f1b_dispatch(g->g, nmb);
    *n = t.cells.size();
    if (rows) *rows = t.rows;
    for (size_t i = 0; cells && i < t.cells.size() && i < cap; ++i) cells[i] = to_c(t.cells[i]);
  });
}

int hb_dispatch_validate(const hb_stage_graph* g, const hb_cell* cells, size_t n, int nmb, char* report, size_t cap,
                         size_t* len, int* n_violations) {
  return guard([&] {
    need(g, "graph");
    need(n_violations, "n_violations");
    std::vector<hb::sched::Cell> v;
    for (size_t i = 0; i < n; ++i) v.push_back(from_c(cells[i]));
    const auto out = hb::sched::validate_dispatch(g->g, v, nmb);
    *n_violations = static_cast<int>(out.size());
    std::string text;
    for (const auto& s : out) text += s + "\n";
    put_text(text, report, cap, len);
  });
}

int hb_dispatch_nc_order(const hb_stage_graph* g, int nmb, int node, hb_cell* cells, size_t cap, size_t* n) {
  return guard([&] {
    need(g, "graph");
    need(n, "n");
    const auto v = hb::sched::nc_issue_order(g->g, hb::sched::generate_1f1b_dispatch(g->g, nmb), node);
    *n = v.size();
    for (size_t i = 0; cells && i < v.size() && i < cap; ++i) cells[i] = to_c(v[i]);
  });
}

int hb_dispatch_render(const hb_stage_graph* g, int nmb, char* buf, size_t cap, size_t* len) {
  return guard([&] {
    need(g, "graph");
    put_text(hb::sched::render(g->g, hb::sched::generate_1f1b_dispatch(g->g, nmb)), buf, cap, len);
  });
}

/* ---- host-owned per-module runtime (a24 + the f2 dispatch executor) --------- */

int hb_nccl_unique_id(void* out128) {
  return guard([&] {
    need(out128, "out");
    hb::rt::nccl_unique_id(out128);
  });
}

void hb_runtime_config_default(hb_runtime_config* c) {
  if (!c) return;
  hb::rt::HostConfig d;
  c->nmb = d.nmb;
  c->max_ctas = d.max_ctas;
  c->pp_bytes = d.pp_bytes;
  c->act_dtype = d.act_dtype;
  c->grad_in_dtype = d.grad_in_dtype;
  c->grad_out_dtype = d.grad_out_dtype;
  c->timeout_s = d.timeout_s;
  c->skip = d.skip;
}

int hb_runtime_create(const hb_layout* modules, int n_modules, const int* edge_src, const int* edge_dst, int n_edges,
                      int global_batch, int feature_width, int world, int my_rank, const void* nccl_id128,
                      const hb_runtime_config* cfg, hb_runtime** out) {
  return guard([&] {
    need(modules, "modules");
    need(out, "out");
    *out = nullptr;
    std::vector<hb::grid::ModuleLayout> ms;
    for (int i = 0; i < n_modules; ++i) ms.push_back(layout(&modules[i]));
    std::vector<std::pair<int, int>> es;
    for (int i = 0; i < n_edges; ++i) es.emplace_back(edge_src[i], edge_dst[i]);
    hb::rt::HostConfig c;
    if (cfg) {
      c.nmb = cfg->nmb;
      c.max_ctas = cfg->max_ctas;
      c.pp_bytes = cfg->pp_bytes;
      c.act_dtype = cfg->act_dtype;
      c.grad_in_dtype = cfg->grad_in_dtype;
      c.grad_out_dtype = cfg->grad_out_dtype;
      c.timeout_s = cfg->timeout_s > 0 ? cfg->timeout_s : c.timeout_s;
      c.skip = cfg->skip;
    }
    auto r = std::make_unique<hb_runtime>();
    r->r = std::make_unique<hb::rt::HostRuntime>(ms, es, global_batch, feature_width, world, my_rank, nccl_id128, c);
    for (int k = 0; k < n_edges; ++k) {
      auto x = std::make_unique<hb_exec>();
      x->x = r->r->edge_exec(k);
      x->borrowed = true;
      r->edge_execs.push_back(std::move(x));
    }
    *out = r.release();
  });
}

void hb_runtime_destroy(hb_runtime* r) { delete r; }

int hb_runtime_info(const hb_runtime* r, int* node, int* module, int* n_nodes, int* rows) {
  return guard([&] {
    need(r, "runtime");
    if (node) *node = r->r->my_node();
    if (module) *module = r->r->my_module();
    if (n_nodes) *n_nodes = static_cast<int>(r->r->graph().nodes.size());
    if (rows) *rows = r->r->table().rows;
  });
}

int hb_runtime_group(const hb_runtime* r, int kind, int* out, int cap, int* n) {
  return guard([&] {
    need(r, "runtime");
    fill(r->r->group(kind), out, cap, n);
  });
}

int hb_runtime_edge_exec(hb_runtime* r, int module_edge, hb_exec** out) {
  return guard([&] {
    need(r, "runtime");
    need(out, "out");
    if (module_edge < 0 || module_edge >= static_cast<int>(r->edge_execs.size()))
      hb::raise(hb::ErrorCode::InvalidArgument, "module edge out of range");
    *out = r->edge_execs[module_edge].get();
  });
}

int hb_runtime_stage_buffer(hb_runtime* r, int which, int mb, void** ptr, size_t* bytes) {
  return guard([&] {
    need(r, "runtime");
    need(ptr, "ptr");
    *ptr = r->r->stage_buffer(which, mb, bytes);
  });
}

int hb_runtime_stream(hb_runtime* r, int which, void** stream) {
  return guard([&] {
    need(r, "runtime");
    need(stream, "stream");
    *stream = r->r->stream(which);
  });
}

int hb_runtime_step(hb_runtime* r, hb_compute_fn fn, void* user) {
  return guard([&] {
    need(r, "runtime");
    r->r->step(reinterpret_cast<hb::rt::ComputeFn>(fn), user);
  });
}

int hb_runtime_last_step_ms(hb_runtime* r, float* ms) {
  return guard([&] {
    need(r, "runtime");
    need(ms, "ms");
    *ms = r->r->last_step_ms();
  });
}

int hb_runtime_paired_ops(const hb_runtime* r, long long* n) {
  return guard([&] {
    need(r, "runtime");
    need(n, "n");
    *n = r->r->paired_ops();
  });
}

}  // extern "C"
