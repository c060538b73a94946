// shim_check — drives the reference-side binding (hetsim_bridge_hb.cpp, i.e.
// hetsim types -> hetbridge C-ABI -> product library) and compares every answer
// with the same call on the reference side: the reference's own grid (compiled
// from /root/reference) and the oracle's restatement of hetsim::bridge. Sweeps
// every layout pair of <= 8 ranks (tp, cp, pp, dp in {1, 2, 4}, offsets 0 and
// disjoint). Errors must map to the same hetsim::ErrorCode. Exit 0 iff all agree.
#include <cstdio>
#include <functional>
#include <string>
#include <vector>

#include "hetsim_bridge_hb.hpp"

using hetsim::grid::BoundaryEdge;
using hetsim::grid::ModuleLayout;

namespace {
int g_checks = 0, g_fail = 0;

template <class A, class B, class Eq>
void same(const char* what, const std::string& label, A ref, B hb, Eq eq) {
  ++g_checks;
  std::string re, he;
  bool rok = true, hok = true;
  decltype(ref()) rv{};
  decltype(hb()) hv{};
  hetsim::ErrorCode rc{}, hc{};
  try {
    rv = ref();
  } catch (const hetsim::SimError& e) {
    rok = false;
    rc = e.code();
  }
  try {
    hv = hb();
  } catch (const hetsim::SimError& e) {
    hok = false;
    hc = e.code();
  }
  const bool ok = rok == hok && (rok ? eq(rv, hv) : rc == hc);
  if (!ok) {
    ++g_fail;
    if (g_fail <= 10)
      std::printf("MISMATCH %s %s: ref %s / hetbridge %s\n", what, label.c_str(), rok ? "ok" : "error",
                  hok ? "ok" : "error");
  }
}

std::vector<ModuleLayout> layouts(const char* name, int offset) {
  std::vector<ModuleLayout> v;
  for (int tp : {1, 2, 4})
    for (int cp : {1, 2})
      for (int pp : {1, 2})
        for (int dp : {1, 2, 4, 8}) {
          if (tp * cp * pp * dp > 8) continue;
          ModuleLayout m;
          m.name = name;
          m.tp = tp, m.cp = cp, m.pp = pp, m.dp = dp, m.rank_offset = offset;
          v.push_back(m);
        }
  return v;
}

std::string label(const BoundaryEdge& e) {
  char b[160];
  std::snprintf(b, sizeof b, "enc{tp%d cp%d pp%d dp%d @%d} -> llm{tp%d cp%d pp%d dp%d @%d} B=%d W=%d", e.source.tp,
                e.source.cp, e.source.pp, e.source.dp, e.source.rank_offset, e.dest.tp, e.dest.cp, e.dest.pp,
                e.dest.dp, e.dest.rank_offset, e.global_batch, e.feature_width);
  return b;
}
}  // namespace

int main() {
  namespace g = hetsim::grid;
  namespace br = hetsim::bridge;
  auto src = layouts("enc", 0), dst0 = layouts("llm", 0);
  for (const auto& s : src) {
    for (int r = 0; r < s.world_size(); ++r)
      same("coord_of_rank", s.name + std::to_string(r), [&] { return g::coord_of_rank(s, r); },
           [&] { return hetsim_hb::coord_of_rank(s, r); }, [](auto a, auto b) { return a == b; });
    for (const auto& d0 : dst0)
      for (int disjoint : {0, 1})
        for (int B : {8, 16, 6}) {
          ModuleLayout d = d0;
          if (disjoint) d.rank_offset = s.world_size();
          BoundaryEdge e{s, d, B, 3};
          const std::string l = label(e);
          same("placement_of_edge", l, [&] { return g::placement_of_edge(e); },
               [&] { return hetsim_hb::placement_of_edge(e); }, [](auto a, auto b) { return a == b; });
          same("classify_dp_relation", l, [&] { return br::classify_dp_relation(e); },
               [&] { return hetsim_hb::classify_dp_relation(e); },
               [](auto a, auto b) { return a.kind == b.kind && a.factor == b.factor; });
          same("export_plan", l, [&] { return br::export_plan(br::plan_bridge(e)); },
               [&] { return hetsim_hb::export_plan(e); }, [](const auto& a, const auto& b) { return a == b; });
        }
  }
  // a partial overlap must raise the same category on both sides
  ModuleLayout a, b;
  a.name = "enc", a.dp = 4;
  b.name = "llm", b.dp = 4, b.rank_offset = 2;
  BoundaryEdge po{a, b, 8, 3};
  same("placement_of_edge", "partial overlap", [&] { return g::placement_of_edge(po); },
       [&] { return hetsim_hb::placement_of_edge(po); }, [](auto x, auto y) { return x == y; });
  std::printf("shim_check: %d checks, %d mismatches\n", g_checks, g_fail);
  return g_fail ? 1 : 0;
}
