// hetsim_bridge_hb.cpp — the reference-side binding a hetsim maintainer would
// add: hetsim::grid / hetsim::bridge call sites kept, the
// work done by hetbridge through its C-ABI (include/hetbridge.h). Built by
// oracle/Makefile (target `shimcheck`) against the reference's own headers.
#include "hetsim_bridge_hb.hpp"

#include <string>
#include <vector>

#include "hetbridge.h"

namespace hetsim_hb {
namespace {
void check(int st) {
  if (st) {
    char msg[512];
    hb_last_error(msg, sizeof msg);
    throw hetsim::SimError(static_cast<hetsim::ErrorCode>(st - 1), msg);
  }
}
hb_layout lay(const hetsim::grid::ModuleLayout& m) { return {m.name.c_str(), m.tp, m.cp, m.pp, m.dp, m.rank_offset}; }
hb_edge edge(const hetsim::grid::BoundaryEdge& e) { return {lay(e.source), lay(e.dest), e.global_batch, e.feature_width}; }
}  // namespace

// hetsim::bridge::export_plan(plan_bridge(e)), byte for byte
std::string export_plan(const hetsim::grid::BoundaryEdge& e) {
  hb_edge he = edge(e);
  hb_plan* p = nullptr;
  check(hb_plan_create(&he, &p));
  size_t n = 0;
  check(hb_plan_export(p, 8, nullptr, 0, &n));
  std::string s(n + 1, '\0');
  check(hb_plan_export(p, 8, s.data(), s.size(), &n));
  hb_plan_destroy(p);
  s.resize(n);
  return s;
}

// hetsim::bridge::classify_dp_relation(e)
hetsim::bridge::DpRelation classify_dp_relation(const hetsim::grid::BoundaryEdge& e) {
  hb_edge he = edge(e);
  int kind = 0, factor = 0;
  check(hb_classify_dp_relation(&he, &kind, &factor));
  return {static_cast<hetsim::bridge::DpKind>(kind), factor};
}

// hetsim::grid::placement_of_edge(e)
hetsim::grid::Placement placement_of_edge(const hetsim::grid::BoundaryEdge& e) {
  hb_edge he = edge(e);
  int pl = 0;
  check(hb_placement_of_edge(&he, &pl));
  return static_cast<hetsim::grid::Placement>(pl);
}

// hetsim::grid::coord_of_rank(l, rank)
hetsim::grid::GridCoord coord_of_rank(const hetsim::grid::ModuleLayout& l, int rank) {
  hb_layout hl = lay(l);
  int c[4];
  check(hb_coord_of_rank(&hl, rank, c));
  return {c[0], c[1], c[2], c[3]};
}

}  // namespace hetsim_hb
