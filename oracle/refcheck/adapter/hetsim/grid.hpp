// Adapter (test infrastructure only): compiles the reference's own
// /root/reference/proj/tests/test_grid.cpp against the PRODUCT's layout algebra
// (paper_2605_27678_b200/csrc/hb/grid.hpp). Same struct layouts and function
// names, so the reference's known-answer tests run unmodified.
#pragma once
#include "hb/grid.hpp"

namespace hetsim {
using ErrorCode = hb::ErrorCode;
using SimError = hb::Error;
namespace grid = hb::grid;
}  // namespace hetsim
