// hetbridge — graph-aware pipeline dispatch (see sched.hpp).
#include "hb/sched.hpp"

#include <algorithm>
#include <functional>
#include <map>
#include <set>
#include <sstream>
#include <tuple>

namespace hb::sched {

const char* op_name(Op op) {
  switch (op) {
    case Op::Compute: return "Compute";
    case Op::SendFwd: return "SendFwd";
    case Op::RecvFwd: return "RecvFwd";
    case Op::SendBwd: return "SendBwd";
    case Op::RecvBwd: return "RecvBwd";
  }
  return "?";
}

std::vector<int> StageGraph::in_edges(int node) const {
  std::vector<int> v;
  for (size_t e = 0; e < edges.size(); ++e)
    if (edges[e].dst == node) v.push_back(static_cast<int>(e));
  return v;
}

std::vector<int> StageGraph::out_edges(int node) const {
  std::vector<int> v;
  for (size_t e = 0; e < edges.size(); ++e)
    if (edges[e].src == node) v.push_back(static_cast<int>(e));
  return v;
}

int StageGraph::node_of(int module, int pp) const {
  for (size_t i = 0; i < nodes.size(); ++i)
    if (nodes[i].module == module && nodes[i].pp == pp) return static_cast<int>(i);
  return -1;
}

StageGraph build_stage_graph(const std::vector<grid::ModuleLayout>& modules,
                             const std::vector<std::pair<int, int>>& module_edges) {
  StageGraph g;
  g.modules = modules;
  g.module_edges = module_edges;
  const int M = static_cast<int>(modules.size());
  if (M == 0) raise(ErrorCode::InvalidArgument, "no modules");
  for (const auto& m : modules) m.validate();
  for (const auto& [s, d] : module_edges) {
    if (s < 0 || s >= M || d < 0 || d >= M)
      raise(ErrorCode::DanglingEdge, "edge references an undeclared module (" + std::to_string(s) + " -> " +
                                         std::to_string(d) + ")");
    if (s == d) raise(ErrorCode::DanglingEdge, "edge from module '" + modules[s].name + "' to itself");
  }
  // module-level cycle check (Kahn)
  {
    std::vector<int> indeg(M, 0);
    for (const auto& e : module_edges) ++indeg[e.second];
    std::vector<int> q;
    for (int m = 0; m < M; ++m)
      if (!indeg[m]) q.push_back(m);
    int seen = 0;
    while (!q.empty()) {
      const int m = q.back();
      q.pop_back();
      ++seen;
      for (const auto& e : module_edges)
        if (e.first == m && --indeg[e.second] == 0) q.push_back(e.second);
    }
    if (seen != M) raise(ErrorCode::CyclicGraph, "module graph has a cycle");
  }
  for (int m = 0; m < M; ++m)
    for (int p = 0; p < modules[m].pp; ++p)
      g.nodes.push_back({m, p, 0, modules[m].name + "P" + std::to_string(p)});
  // chain edges first (module order), then boundary edges in declared order
  for (int m = 0; m < M; ++m)
    for (int p = 0; p + 1 < modules[m].pp; ++p) g.edges.push_back({g.node_of(m, p), g.node_of(m, p + 1), EdgeKind::P2P, -1});
  for (size_t k = 0; k < module_edges.size(); ++k) {
    const auto [s, d] = module_edges[k];
    g.edges.push_back({g.node_of(s, modules[s].pp - 1), g.node_of(d, 0), EdgeKind::NC, static_cast<int>(k)});
  }
  std::vector<int> sinks;
  for (size_t n = 0; n < g.nodes.size(); ++n)
    if (g.out_edges(static_cast<int>(n)).empty()) sinks.push_back(static_cast<int>(n));
  if (sinks.size() != 1)
    raise(ErrorCode::InfeasibleSchedule, "the stage graph needs exactly one sink (the loss-bearing stage), found " +
                                             std::to_string(sinks.size()));
  g.sink = sinks[0];
  // longest path to the sink (the node DAG is acyclic because the module DAG is)
  const int Nn = static_cast<int>(g.nodes.size());
  std::vector<int> dist(Nn, -1);
  std::function<int(int)> dfs = [&](int n) -> int {
    if (dist[n] >= 0) return dist[n];
    int best = 0;
    for (int e : g.out_edges(n)) best = std::max(best, 1 + dfs(g.edges[e].dst));
    return dist[n] = best;
  };
  for (int n = 0; n < Nn; ++n) g.nodes[n].distance = dfs(n);
  return g;
}

DispatchTable generate_1f1b_dispatch(const StageGraph& g, int nmb) {
  if (nmb < 1) raise(ErrorCode::InfeasibleSchedule, "NMB must be >= 1");
  const int Nn = static_cast<int>(g.nodes.size());
  struct Act {
    int mb;
    bool bwd;
  };
  std::vector<std::vector<Act>> prog(Nn);
  for (int n = 0; n < Nn; ++n) {
    const int w = std::min(g.nodes[n].distance, nmb);
    for (int m = 0; m < w; ++m) prog[n].push_back({m, false});
    for (int k = 0; k + w < nmb; ++k) {
      prog[n].push_back({w + k, false});
      prog[n].push_back({k, true});
    }
    for (int m = nmb - w; m < nmb; ++m) prog[n].push_back({m, true});
  }
  std::vector<std::vector<int>> in(Nn), out(Nn);
  for (int n = 0; n < Nn; ++n) {
    in[n] = g.in_edges(n);
    out[n] = g.out_edges(n);
  }
  // deliveries visible from the next row on
  std::vector<std::vector<int>> fwd_in(Nn, std::vector<int>(nmb, 0)), bwd_in(Nn, std::vector<int>(nmb, 0));
  std::vector<std::vector<char>> f_done(Nn, std::vector<char>(nmb, 0));
  std::vector<size_t> pc(Nn, 0);
  DispatchTable t;
  t.nmb = nmb;
  size_t remaining = 0;
  for (const auto& p : prog) remaining += p.size();
  int row = 0;
  while (remaining) {
    std::vector<std::tuple<int, int, bool>> deliver;  // (node, mb, bwd)
    std::vector<Cell> comm;
    bool progressed = false;
    for (int n = 0; n < Nn; ++n) {
      if (pc[n] >= prog[n].size()) continue;
      const Act a = prog[n][pc[n]];
      const bool ready = a.bwd ? (f_done[n][a.mb] && bwd_in[n][a.mb] == static_cast<int>(out[n].size()))
                               : fwd_in[n][a.mb] == static_cast<int>(in[n].size());
      if (!ready) continue;
      progressed = true;
      ++pc[n];
      --remaining;
      t.cells.push_back({row, n, Op::Compute, -1, EdgeKind::P2P, a.mb, a.bwd});
      if (!a.bwd) {
        f_done[n][a.mb] = 1;
        for (int e : out[n]) {
          const auto& E = g.edges[e];
          t.cells.push_back({row, n, Op::SendFwd, e, E.kind, a.mb, false});
          comm.push_back({row, E.dst, Op::RecvFwd, e, E.kind, a.mb, false});
          deliver.emplace_back(E.dst, a.mb, false);
        }
      } else {
        for (int e : in[n]) {
          const auto& E = g.edges[e];
          t.cells.push_back({row, n, Op::SendBwd, e, E.kind, a.mb, true});
          comm.push_back({row, E.src, Op::RecvBwd, e, E.kind, a.mb, true});
          deliver.emplace_back(E.src, a.mb, true);
        }
      }
    }
    if (!progressed) raise(ErrorCode::InfeasibleSchedule, "1F1B dispatch deadlocked at call " + std::to_string(row));
    t.cells.insert(t.cells.end(), comm.begin(), comm.end());
    for (const auto& [n, mb, b] : deliver) ++(b ? bwd_in : fwd_in)[n][mb];
    ++row;
  }
  t.rows = row;
  std::stable_sort(t.cells.begin(), t.cells.end(), [](const Cell& a, const Cell& b) {
    return std::tie(a.row, a.node) < std::tie(b.row, b.node);
  });
  return t;
}

std::vector<std::string> validate_dispatch(const StageGraph& g, const std::vector<Cell>& cells, int nmb) {
  std::vector<std::string> v;
  const int Nn = static_cast<int>(g.nodes.size()), Ne = static_cast<int>(g.edges.size());
  auto ename = [&](int e) {
    const auto& E = g.edges[e];
    return g.nodes[E.src].name + "->" + g.nodes[E.dst].name + (E.kind == EdgeKind::NC ? "[NC]" : "[p2p]");
  };
  // row of each (op, edge, mb) and (node, mb, bwd) compute; duplicates flagged
  std::map<std::tuple<int, int, int>, std::vector<int>> comm_rows;  // (op, edge, mb) -> rows
  std::map<std::tuple<int, int, int>, std::vector<int>> comp_rows;  // (node, mb, bwd) -> rows
  for (const auto& c : cells) {
    if (c.node < 0 || c.node >= Nn || c.mb < 0 || c.mb >= nmb) {
      v.push_back("cell at call " + std::to_string(c.row) + ": node or microbatch out of range");
      continue;
    }
    if (c.op == Op::Compute) {
      comp_rows[{c.node, c.mb, c.bwd ? 1 : 0}].push_back(c.row);
      continue;
    }
    if (c.edge < 0 || c.edge >= Ne) {
      v.push_back("call " + std::to_string(c.row) + " " + g.nodes[c.node].name + ": " + op_name(c.op) +
                  " on an unknown edge");
      continue;
    }
    const auto& E = g.edges[c.edge];
    const int expect_node = (c.op == Op::SendFwd || c.op == Op::RecvBwd) ? E.src : E.dst;
    if (c.node != expect_node)
      v.push_back("edge identity: " + std::string(op_name(c.op)) + "(mb " + std::to_string(c.mb) + ") at " +
                  g.nodes[c.node].name + " uses " + ename(c.edge) + ", which does not end there");
    if (c.kind != E.kind)
      v.push_back("call " + std::to_string(c.row) + ": " + ename(c.edge) + " dispatched as " +
                  (c.kind == EdgeKind::NC ? "NC" : "p2p"));
    comm_rows[{static_cast<int>(c.op), c.edge, c.mb}].push_back(c.row);
  }
  auto one = [&](const std::map<std::tuple<int, int, int>, std::vector<int>>& m, std::tuple<int, int, int> k,
                 const std::string& what) -> int {
    auto it = m.find(k);
    if (it == m.end() || it->second.empty()) {
      v.push_back("missing: " + what);
      return -1;
    }
    if (it->second.size() > 1) v.push_back("double consumption: " + what + " appears " +
                                           std::to_string(it->second.size()) + " times");
    return it->second.front();
  };
  for (int e = 0; e < Ne; ++e) {
    const auto& E = g.edges[e];
    for (int mb = 0; mb < nmb; ++mb) {
      const std::string sfx = " of mb " + std::to_string(mb) + " on " + ename(e);
      const int sf = one(comm_rows, {static_cast<int>(Op::SendFwd), e, mb}, "forward send" + sfx);
      const int rf = one(comm_rows, {static_cast<int>(Op::RecvFwd), e, mb}, "forward receive" + sfx);
      const int sb = one(comm_rows, {static_cast<int>(Op::SendBwd), e, mb}, "gradient send" + sfx);
      const int rb = one(comm_rows, {static_cast<int>(Op::RecvBwd), e, mb}, "gradient receive" + sfx);
      if (sf >= 0 && rf >= 0 && sf != rf) v.push_back("forward send and receive" + sfx + " in different calls");
      if (sb >= 0 && rb >= 0 && sb != rb) v.push_back("gradient send and receive" + sfx + " in different calls");
      if (sb >= 0 && rf >= 0 && sb <= rf)
        v.push_back("edge identity: gradient" + sfx + " returned before the activation arrived");
      auto cf = comp_rows.find({E.src, mb, 0});
      if (sf >= 0 && cf != comp_rows.end() && !cf->second.empty() && cf->second.front() > sf)
        v.push_back("forward send" + sfx + " before " + g.nodes[E.src].name + " computed it");
      auto cb = comp_rows.find({E.dst, mb, 1});
      if (sb >= 0 && cb != comp_rows.end() && !cb->second.empty() && cb->second.front() > sb)
        v.push_back("gradient send" + sfx + " before " + g.nodes[E.dst].name + " computed it");
    }
  }
  // a join's gradients must go back over the edge each activation came in on
  auto count = [&](Op op, int e, int mb) {
    auto it = comm_rows.find({static_cast<int>(op), e, mb});
    return it == comm_rows.end() ? 0 : static_cast<int>(it->second.size());
  };
  for (int n = 0; n < Nn; ++n)
    for (int mb = 0; mb < nmb; ++mb) {
      const auto ins = g.in_edges(n);
      for (int e : ins)
        if (count(Op::RecvFwd, e, mb) == 1 && count(Op::SendBwd, e, mb) == 0)
          for (int o : ins)
            if (o != e && count(Op::SendBwd, o, mb) > 1)
              v.push_back("edge identity: the gradient of mb " + std::to_string(mb) + " that entered " +
                          g.nodes[n].name + " over " + ename(e) + " is returned over " + ename(o));
    }
  for (int n = 0; n < Nn; ++n)
    for (int mb = 0; mb < nmb; ++mb) {
      const std::string who = g.nodes[n].name + " mb " + std::to_string(mb);
      const int f = one(comp_rows, {n, mb, 0}, "forward compute of " + who);
      const int b = one(comp_rows, {n, mb, 1}, "backward compute of " + who);
      if (f >= 0 && b >= 0 && b <= f) v.push_back("backward of " + who + " before its forward");
      if (f >= 0)
        for (int e : g.in_edges(n)) {  // join readiness
          auto it = comm_rows.find({static_cast<int>(Op::RecvFwd), e, mb});
          if (it != comm_rows.end() && !it->second.empty() && it->second.front() >= f)
            v.push_back("join readiness: " + who + " computed before its input arrived on " + ename(e));
        }
      if (b >= 0)
        for (int e : g.out_edges(n)) {
          auto it = comm_rows.find({static_cast<int>(Op::RecvBwd), e, mb});
          if (it != comm_rows.end() && !it->second.empty() && it->second.front() >= b)
            v.push_back("backward of " + who + " before its gradient arrived on " + ename(e));
        }
    }
  return v;
}

bool nc_before(const StageGraph& g, const Cell& a, const Cell& b) {
  auto key = [&](const Cell& c) {
    const bool bwd = c.op == Op::SendBwd || c.op == Op::RecvBwd;
    return std::make_tuple(c.row, g.edges.at(c.edge).boundary, bwd ? 1 : 0, c.mb);
  };
  return key(a) < key(b);
}

std::vector<Cell> nc_issue_order(const StageGraph& g, const DispatchTable& t, int node) {
  std::vector<Cell> v;
  for (const auto& c : t.cells)
    if (c.node == node && c.op != Op::Compute && c.kind == EdgeKind::NC) v.push_back(c);
  std::stable_sort(v.begin(), v.end(), [&](const Cell& a, const Cell& b) { return nc_before(g, a, b); });
  return v;
}

std::string render(const StageGraph& g, const DispatchTable& t) {
  const int Nn = static_cast<int>(g.nodes.size());
  std::vector<std::vector<std::string>> grid(t.rows, std::vector<std::string>(Nn));
  for (const auto& c : t.cells) {
    std::string tok;
    const std::string k = c.kind == EdgeKind::NC ? "NC" : "p2p";
    switch (c.op) {
      case Op::Compute: tok = (c.bwd ? "B" : "F") + std::to_string(c.mb); break;
      case Op::SendFwd: tok = "sf" + std::to_string(c.mb) + ":" + k; break;
      case Op::RecvFwd: tok = "rf" + std::to_string(c.mb) + ":" + k; break;
      case Op::SendBwd: tok = "sb" + std::to_string(c.mb) + ":" + k; break;
      case Op::RecvBwd: tok = "rb" + std::to_string(c.mb) + ":" + k; break;
    }
    auto& s = grid[c.row][c.node];
    s += (s.empty() ? "" : " ") + tok;
  }
  std::vector<size_t> w(Nn);
  for (int n = 0; n < Nn; ++n) {
    w[n] = g.nodes[n].name.size();
    for (int r = 0; r < t.rows; ++r) w[n] = std::max(w[n], grid[r][n].size());
  }
  std::ostringstream os;
  auto pad = [](const std::string& s, size_t n) { return s + std::string(n - s.size(), ' '); };
  os << "call ";
  for (int n = 0; n < Nn; ++n) os << " | " << pad(g.nodes[n].name, w[n]);
  os << "\n";
  for (int r = 0; r < t.rows; ++r) {
    std::string idx = std::to_string(r);
    os << pad(idx, 5);
    for (int n = 0; n < Nn; ++n) os << " | " << pad(grid[r][n], w[n]);
    os << "\n";
  }
  return os.str();
}

}  // namespace hb::sched
