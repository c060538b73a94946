// ORACLE — test infrastructure only (see bridge_oracle.cpp header).
#pragma once

#include <vector>

#include "hetsim/grid.hpp"

namespace hb_oracle {

/// Placeholder table of the reference layout (tinymodel.hpp:24-26): sequence q
/// is sample q, vision tokens at positions [0,S_v), text at [S_v,S).
std::vector<int> reference_codes(int n, int S, int S_v);

/// Generalised assemble_tokens: materialise positions `slice` of Q sequences.
void splice_forward(const std::vector<int>& codes, int Q, int S, int d_h,
                    const hetsim::grid::BatchInterval& slice, const double* vision,
                    long vision_rows, const double* text, long text_rows, long text_offset,
                    double* out);

/// Generalised split_vision_grad: full-width vision-row gradient, zeros outside
/// the slice.
void splice_backward(const std::vector<int>& codes, int Q, int S, int d_h,
                     const hetsim::grid::BatchInterval& slice, const double* token_grad,
                     long vision_rows, double* out);

}  // namespace hb_oracle
