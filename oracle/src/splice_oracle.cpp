// ORACLE — test infrastructure only (see bridge_oracle.cpp header).
//
// CPU restatement of the reference's embedding-splice helpers, declared in
// /root/reference/proj/core/include/hetsim/tinymodel.hpp:94-112 with no body
// (proj/core/src/tinymodel.cpp is a stub), plus the brute-force interval oracle
// declared in oracle.hpp:17-22. Semantics follow tinymodel.hpp:24-26 (vision
// tokens at [0,S_v), text at the rest), SPEC.md:343-345,355 (every CP rank keeps
// the positions inside its contiguous slice; vision gradients are full-width
// with zeros outside the slice) and SURVEY App. A "Splice".
//
// Token-matrix layout (◆, reference-silent): the stage-0 token matrix has one
// row per (sample, position) in sample-major order and d_h columns, which is
// what the token-wise LLM layers of tinymodel.hpp:148-184 multiply.
//
// The generalised form takes a placeholder table code[q*S+p]: code >= 0 is a
// vision token row (local sample j, token t) -> j*S_v+t of the bridge payload
// viewed as token rows; code < 0 is text row -1-code. The reference layout is
// the special case built by reference_codes().

#include <map>
#include <vector>

#include "hetsim/oracle.hpp"
#include "hetsim/tinymodel.hpp"
#include "splice_oracle.hpp"

namespace hetsim::tinymodel {

// tinymodel.hpp:93-95: contiguous CP slices [c*S/cp, (c+1)*S/cp).
grid::BatchInterval cp_token_slice(int seq_len, int cp, int cp_idx) {
  if (cp < 1 || cp_idx < 0 || cp_idx >= cp)
    raise(ErrorCode::InvalidArgument, "cp index out of range");
  if (seq_len % cp != 0)
    raise(ErrorCode::DivisibilityViolation,
          "seq_len " + std::to_string(seq_len) + " not divisible by cp " + std::to_string(cp));
  const int L = seq_len / cp;
  return {cp_idx * L, L};
}

Matrix assemble_tokens(const TinyModelSpec& spec, const Matrix& vision_rows,
                       const Matrix& text_rows, const grid::BatchInterval& slice) {
  const int n = vision_rows.rows;
  if (vision_rows.cols != spec.vision_tokens * spec.d_h || text_rows.rows != n ||
      text_rows.cols != spec.text_tokens() * spec.d_h)
    raise(ErrorCode::ShapeMismatch, "assemble_tokens operand shapes");
  const auto codes = hb_oracle::reference_codes(n, spec.seq_len, spec.vision_tokens);
  Matrix out(n * slice.length, spec.d_h);
  hb_oracle::splice_forward(codes, n, spec.seq_len, spec.d_h, slice, vision_rows.a.data(),
                            static_cast<long>(n) * spec.vision_tokens, text_rows.a.data(),
                            static_cast<long>(n) * spec.text_tokens(), 0, out.a.data());
  return out;
}

Matrix split_vision_grad(const TinyModelSpec& spec, const Matrix& token_grad,
                         const grid::BatchInterval& slice, int n_samples) {
  if (token_grad.rows != n_samples * slice.length || token_grad.cols != spec.d_h)
    raise(ErrorCode::ShapeMismatch, "split_vision_grad operand shape");
  const auto codes = hb_oracle::reference_codes(n_samples, spec.seq_len, spec.vision_tokens);
  Matrix out(n_samples, spec.vision_tokens * spec.d_h);
  hb_oracle::splice_backward(codes, n_samples, spec.seq_len, spec.d_h, slice,
                             token_grad.a.data(),
                             static_cast<long>(n_samples) * spec.vision_tokens, out.a.data());
  return out;
}

}  // namespace hetsim::tinymodel

namespace hetsim::oracle {

// oracle.hpp:17-22 / SPEC.md:468-476: sample j -> src floor(j*dp_src/B),
// dst floor(j*dp_dst/B), grouped into ordered runs per destination shard.
std::vector<std::vector<std::pair<int, grid::BatchInterval>>> interval_oracle(
    int batch, int dp_src, int dp_dst) {
  if (dp_src < 1 || dp_dst < 1) raise(ErrorCode::InvalidArgument, "dp must be >= 1");
  if (batch <= 0 || batch % dp_src || batch % dp_dst)
    raise(ErrorCode::IndivisibleBatch, "batch not divisible");
  std::vector<std::vector<std::pair<int, grid::BatchInterval>>> out(dp_dst);
  for (int j = 0; j < batch; ++j) {
    const int s = static_cast<int>(static_cast<long>(j) * dp_src / batch);
    const int d = static_cast<int>(static_cast<long>(j) * dp_dst / batch);
    auto& v = out[d];
    if (!v.empty() && v.back().first == s && v.back().second.end() == j)
      v.back().second.length++;
    else
      v.push_back({s, grid::BatchInterval{j, 1}});
  }
  return out;
}

}  // namespace hetsim::oracle

namespace hb_oracle {

std::vector<int> reference_codes(int n, int S, int S_v) {
  std::vector<int> codes(static_cast<size_t>(n) * S);
  for (int q = 0; q < n; ++q)
    for (int p = 0; p < S; ++p)
      codes[static_cast<size_t>(q) * S + p] =
          p < S_v ? q * S_v + p : -1 - (q * (S - S_v) + (p - S_v));
  return codes;
}

void splice_forward(const std::vector<int>& codes, int Q, int S, int d_h,
                    const hetsim::grid::BatchInterval& slice, const double* vision,
                    long vision_rows, const double* text, long text_rows, long text_offset,
                    double* out) {
  using hetsim::ErrorCode;
  if (static_cast<long>(codes.size()) != static_cast<long>(Q) * S)
    hetsim::raise(ErrorCode::ShapeMismatch, "placeholder table size");
  if (slice.start < 0 || slice.end() > S)
    hetsim::raise(ErrorCode::InvalidArgument, "slice outside sequence");
  for (int q = 0; q < Q; ++q) {
    for (int p = slice.start; p < slice.end(); ++p) {
      const int code = codes[static_cast<size_t>(q) * S + p];
      const double* row;
      if (code >= 0) {
        if (code >= vision_rows) hetsim::raise(ErrorCode::ShapeMismatch, "vision row out of range");
        row = vision + static_cast<long>(code) * d_h;
      } else {
        const long t = -1L - code - text_offset;
        if (t < 0 || t >= text_rows) hetsim::raise(ErrorCode::ShapeMismatch, "text row out of range");
        row = text + t * d_h;
      }
      double* o = out + (static_cast<long>(q) * slice.length + (p - slice.start)) * d_h;
      for (int h = 0; h < d_h; ++h) o[h] = row[h];
    }
  }
}

void splice_backward(const std::vector<int>& codes, int Q, int S, int d_h,
                     const hetsim::grid::BatchInterval& slice, const double* token_grad,
                     long vision_rows, double* out) {
  using hetsim::ErrorCode;
  if (static_cast<long>(codes.size()) != static_cast<long>(Q) * S)
    hetsim::raise(ErrorCode::ShapeMismatch, "placeholder table size");
  for (long i = 0; i < vision_rows * d_h; ++i) out[i] = 0.0;  // zeros outside the slice
  for (int q = 0; q < Q; ++q) {
    for (int p = slice.start; p < slice.end(); ++p) {
      const int code = codes[static_cast<size_t>(q) * S + p];
      if (code < 0) continue;  // text positions carry no gradient (tinymodel.hpp:103-107)
      if (code >= vision_rows) hetsim::raise(ErrorCode::ShapeMismatch, "vision row out of range");
      const double* g = token_grad + (static_cast<long>(q) * slice.length + (p - slice.start)) * d_h;
      double* o = out + static_cast<long>(code) * d_h;
      for (int h = 0; h < d_h; ++h) o[h] += g[h];  // adjoint of placement, from +0.0
    }
  }
}

}  // namespace hb_oracle
