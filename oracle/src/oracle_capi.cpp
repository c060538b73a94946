// ORACLE — test infrastructure only (see bridge_oracle.cpp header).
//
// Flat C entry points over the oracle so the Python tests and bench.py's CPU
// baseline leg can drive it through ctypes. Status convention mirrors the
// product C-ABI: 0 = OK, ErrorCode ordinal + 1 on SimError, -1 otherwise.
// Layouts are int[5] = {tp, cp, pp, dp, rank_offset}.

#include <chrono>
#include <cstring>
#include <string>

#include "hetsim/bridge.hpp"
#include "hetsim/oracle.hpp"
#include "hetsim/tinymodel.hpp"
#include "splice_oracle.hpp"

using namespace hetsim;

namespace {
thread_local std::string g_err;

template <class F>
int guard(F&& f) {
  try {
    f();
    g_err.clear();
    return 0;
  } catch (const SimError& e) {
    g_err = e.what();
    return static_cast<int>(e.code()) + 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

grid::ModuleLayout lay(const int* v, const char* name) {
  grid::ModuleLayout l;
  l.name = name ? name : "";
  l.tp = v[0];
  l.cp = v[1];
  l.pp = v[2];
  l.dp = v[3];
  l.rank_offset = v[4];
  return l;
}

grid::BoundaryEdge edge(const int* src, const char* sname, const int* dst, const char* dname,
                        int B, int W) {
  return grid::BoundaryEdge{lay(src, sname), lay(dst, dname), B, W};
}

int copy_out(const std::string& s, char* buf, long cap, long* len) {
  if (len) *len = static_cast<long>(s.size());
  if (buf && cap > 0) {
    const long n = std::min<long>(cap - 1, static_cast<long>(s.size()));
    std::memcpy(buf, s.data(), n);
    buf[n] = 0;
  }
  return 0;
}
}  // namespace

extern "C" {

const char* oracle_last_error() { return g_err.c_str(); }

int oracle_plan_export(const int* src, const char* sname, const int* dst, const char* dname,
                       int B, int W, char* buf, long cap, long* len) {
  return guard([&] {
    auto p = bridge::plan_bridge(edge(src, sname, dst, dname, B, W));
    copy_out(bridge::export_plan(p), buf, cap, len);
  });
}

/// kind: 0 Equal, 1 FanIn, 2 FanOut.
int oracle_classify(const int* src, const int* dst, int* kind, int* factor) {
  return guard([&] {
    auto r = bridge::classify_dp_relation(edge(src, "src", dst, "dst", 1, 1));
    *kind = static_cast<int>(r.kind);
    *factor = r.factor;
  });
}

int oracle_cross_boundary_messages(const int* src, const int* dst, int B, int W, int* n) {
  return guard([&] { *n = bridge::plan_bridge(edge(src, "src", dst, "dst", B, W)).cross_boundary_messages(); });
}

/// Whole-edge forward over the reference simnet. in_by_rank[r] is rank r's
/// source shard (rows x W doubles) or NULL; out_by_rank[r] receives the
/// destination shard for every destination stage-0 rank (caller-sized).
/// The ledger render is copied to ledger_buf. seconds_out gets the wall time
/// of the fabric run (for the CPU baseline leg).
int oracle_bridge_forward(const int* src, const char* sname, const int* dst, const char* dname,
                          int B, int W, int mb, int world, const double* const* in_by_rank,
                          double* const* out_by_rank, char* ledger_buf, long cap, long* len,
                          double* seconds_out) {
  return guard([&] {
    auto p = bridge::plan_bridge(edge(src, sname, dst, dname, B, W));
    const auto SI = p.src_intervals;
    std::map<int, bridge::ShardedTensor> shards;
    for (int r = 0; r < world; ++r) {
      if (!in_by_rank[r]) continue;
      const auto c = grid::coord_of_rank(p.edge.source, r);
      const auto iv = SI[c.dp_idx];
      bridge::ShardedTensor t{iv, W, {}};
      t.payload.assign(in_by_rank[r], in_by_rank[r] + static_cast<size_t>(iv.length) * W);
      shards[r] = std::move(t);
    }
    simnet::TrafficLedger ledger;
    const auto t0 = std::chrono::steady_clock::now();
    auto out = bridge::bridge_forward(p, shards, mb, &ledger);
    const auto t1 = std::chrono::steady_clock::now();
    if (seconds_out) *seconds_out = std::chrono::duration<double>(t1 - t0).count();
    for (auto& [r, t] : out) {
      if (r >= world || !out_by_rank[r]) raise(ErrorCode::InvalidArgument, "missing output buffer");
      std::memcpy(out_by_rank[r], t.payload.data(), t.payload.size() * sizeof(double));
    }
    copy_out(ledger.render(), ledger_buf, cap, len);
  });
}

int oracle_bridge_backward(const int* src, const char* sname, const int* dst, const char* dname,
                           int B, int W, int mb, int world, const double* const* grad_by_rank,
                           double* const* out_by_rank, char* ledger_buf, long cap, long* len,
                           double* seconds_out) {
  return guard([&] {
    auto p = bridge::plan_bridge(edge(src, sname, dst, dname, B, W));
    const auto DI = p.dest_intervals;
    std::map<int, bridge::ShardedTensor> grads;
    for (int r = 0; r < world; ++r) {
      if (!grad_by_rank[r]) continue;
      const auto c = grid::coord_of_rank(p.edge.dest, r);
      const auto iv = DI[c.dp_idx];
      bridge::ShardedTensor t{iv, W, {}};
      t.payload.assign(grad_by_rank[r], grad_by_rank[r] + static_cast<size_t>(iv.length) * W);
      grads[r] = std::move(t);
    }
    simnet::TrafficLedger ledger;
    const auto t0 = std::chrono::steady_clock::now();
    auto out = bridge::bridge_backward(p, grads, mb, &ledger);
    const auto t1 = std::chrono::steady_clock::now();
    if (seconds_out) *seconds_out = std::chrono::duration<double>(t1 - t0).count();
    for (auto& [r, t] : out) {
      if (r >= world || !out_by_rank[r]) raise(ErrorCode::InvalidArgument, "missing output buffer");
      std::memcpy(out_by_rank[r], t.payload.data(), t.payload.size() * sizeof(double));
    }
    copy_out(ledger.render(), ledger_buf, cap, len);
  });
}

int oracle_splice_forward(const int* codes, int Q, int S, int d_h, int slice_start,
                          int slice_len, const double* vision, long vision_rows,
                          const double* text, long text_rows, long text_offset, double* out) {
  return guard([&] {
    std::vector<int> c(codes, codes + static_cast<size_t>(Q) * S);
    hb_oracle::splice_forward(c, Q, S, d_h, {slice_start, slice_len}, vision, vision_rows, text,
                              text_rows, text_offset, out);
  });
}

int oracle_splice_backward(const int* codes, int Q, int S, int d_h, int slice_start,
                           int slice_len, const double* token_grad, long vision_rows,
                           double* out) {
  return guard([&] {
    std::vector<int> c(codes, codes + static_cast<size_t>(Q) * S);
    hb_oracle::splice_backward(c, Q, S, d_h, {slice_start, slice_len}, token_grad, vision_rows,
                               out);
  });
}

int oracle_cp_token_slice(int S, int cp, int c, int* start, int* length) {
  return guard([&] {
    auto iv = tinymodel::cp_token_slice(S, cp, c);
    *start = iv.start;
    *length = iv.length;
  });
}

/// Reference-signature assemble_tokens (tinymodel.hpp:97-101) for the
/// reference layout; out is (n*slice_len) x d_h.
int oracle_assemble_tokens(int S, int S_v, int d_h, int n, const double* vision,
                           const double* text, int slice_start, int slice_len, double* out) {
  return guard([&] {
    tinymodel::TinyModelSpec spec;
    spec.seq_len = S;
    spec.vision_tokens = S_v;
    spec.d_h = d_h;
    Matrix v(n, S_v * d_h), t(n, (S - S_v) * d_h);
    std::memcpy(v.a.data(), vision, v.a.size() * sizeof(double));
    std::memcpy(t.a.data(), text, t.a.size() * sizeof(double));
    auto m = tinymodel::assemble_tokens(spec, v, t, {slice_start, slice_len});
    std::memcpy(out, m.a.data(), m.a.size() * sizeof(double));
  });
}

int oracle_split_vision_grad(int S, int S_v, int d_h, int n, const double* token_grad,
                             int slice_start, int slice_len, double* out) {
  return guard([&] {
    tinymodel::TinyModelSpec spec;
    spec.seq_len = S;
    spec.vision_tokens = S_v;
    spec.d_h = d_h;
    Matrix g(n * slice_len, d_h);
    std::memcpy(g.a.data(), token_grad, g.a.size() * sizeof(double));
    auto m = tinymodel::split_vision_grad(spec, g, {slice_start, slice_len}, n);
    std::memcpy(out, m.a.data(), m.a.size() * sizeof(double));
  });
}

/// interval_oracle flattened: out holds (dst, src, start, length) quadruples.
int oracle_interval_oracle(int B, int dp_src, int dp_dst, int* out, int cap, int* n) {
  return guard([&] {
    auto v = oracle::interval_oracle(B, dp_src, dp_dst);
    int k = 0;
    for (int d = 0; d < static_cast<int>(v.size()); ++d)
      for (auto& [s, iv] : v[d]) {
        if (k + 4 <= cap) {
          out[k] = d;
          out[k + 1] = s;
          out[k + 2] = iv.start;
          out[k + 3] = iv.length;
        }
        k += 4;
      }
    *n = k / 4;
  });
}

/// The reference's own grid functions, exposed so tests can cross-check the
/// product's host grid against them (grid.cpp:21-106).
int oracle_coord_of_rank(const int* l, int rank, int* coord4) {
  return guard([&] {
    auto c = grid::coord_of_rank(lay(l, "m"), rank);
    coord4[0] = c.tp_idx;
    coord4[1] = c.cp_idx;
    coord4[2] = c.pp_idx;
    coord4[3] = c.dp_idx;
  });
}

int oracle_placement_of_edge(const int* src, const int* dst, int* placement) {
  return guard([&] {
    *placement = static_cast<int>(grid::placement_of_edge(edge(src, "a", dst, "b", 1, 1)));
  });
}

/// Reference GaussianStream (matrix.cpp:136-180) for seeded synthetic inputs.
int oracle_gaussian_fill(unsigned long long seed, const char* tag, double* out, long n,
                         double scale) {
  return guard([&] {
    GaussianStream g(seed, tag);
    for (long i = 0; i < n; ++i) out[i] = g.next() * scale;
  });
}
}
