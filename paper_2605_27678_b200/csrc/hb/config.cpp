// hetbridge — module_parallelisms configuration ingestion (see config.hpp).
// Reference: SPEC.md cli module, paper Appendix B.
#include "hb/config.hpp"

#include <cctype>
#include <cerrno>
#include <cstdlib>
#include <sstream>

namespace hb::config {
namespace {

struct LayoutKey {
  const char* key;
  int grid::ModuleLayout::*field;
};
// Appendix B's ModuleParallelismConfig field names, plus the
// context-parallel size of the SPEC's schema.
constexpr LayoutKey kLayoutKeys[] = {
    {"tensor_model_parallel_size", &grid::ModuleLayout::tp},
    {"context_parallel_size", &grid::ModuleLayout::cp},
    {"pipeline_model_parallel_size", &grid::ModuleLayout::pp},
    {"data_parallel_size", &grid::ModuleLayout::dp},
    {"rank_offset", &grid::ModuleLayout::rank_offset},
};

[[noreturn]] void parse_error(int line, const std::string& what) {
  raise(ErrorCode::ParseError, "line " + std::to_string(line) + ": " + what);
}

[[noreturn]] void invalid(const std::string& what) { raise(ErrorCode::ValidationError, what); }

std::string trim(const std::string& s) {
  size_t a = 0, b = s.size();
  while (a < b && std::isspace(static_cast<unsigned char>(s[a]))) ++a;
  while (b > a && std::isspace(static_cast<unsigned char>(s[b - 1]))) --b;
  return s.substr(a, b - a);
}

bool is_ident(const std::string& s) {
  if (s.empty()) return false;
  for (char c : s)
    if (!(std::isalnum(static_cast<unsigned char>(c)) || c == '_' || c == '-' || c == '.')) return false;
  return true;
}

// integers and decimals only: [+-]digits[.digits][e[+-]digits]
bool is_number(const std::string& v) {
  if (v.empty()) return false;
  const char* p = v.c_str();
  char* end = nullptr;
  errno = 0;
  std::strtod(p, &end);
  return errno == 0 && end && *end == '\0' && !std::isalpha(static_cast<unsigned char>(v[0])) &&
         v.find_first_of("xXnN") == std::string::npos;  // no hex / inf / nan
}

long long to_int(int line, const std::string& key, const std::string& v) {
  char* end = nullptr;
  errno = 0;
  const long long x = std::strtoll(v.c_str(), &end, 10);
  if (errno != 0 || !end || *end != '\0') parse_error(line, "'" + key + "' needs an integer, got '" + v + "'");
  return x;
}

}  // namespace

const ModuleEntry& ExperimentConfig::language() const { return module("language"); }

const ModuleEntry& ExperimentConfig::module(const std::string& name) const {
  for (const auto& m : modules)
    if (m.layout.name == name) return m;
  raise(ErrorCode::InvalidArgument, "no module named '" + name + "'");
}

grid::BoundaryEdge ExperimentConfig::edge(const std::string& encoder, int feature_width) const {
  if (encoder == "language") raise(ErrorCode::InvalidArgument, "the edge's source must be an encoder module");
  if (feature_width < 1) raise(ErrorCode::InvalidArgument, "feature_width must be >= 1");
  if (global_batch < 1) raise(ErrorCode::InvalidArgument, "[run] global_batch is required for an edge");
  grid::BoundaryEdge e;
  e.source = module(encoder).layout;
  e.dest = language().layout;
  e.global_batch = global_batch / num_microbatches;
  e.feature_width = feature_width;
  grid::placement_of_edge(e);  // PartialOverlap for ranges that neither match nor separate
  return e;
}

ExperimentConfig parse_config(const std::string& text) {
  ExperimentConfig c;
  std::istringstream in(text);
  std::string raw;
  int line = 0;
  enum { kNone, kModule, kModel, kRun } section = kNone;
  std::map<std::string, int> seen;  // "section/key" -> line (duplicate keys)
  std::string sec_name;
  while (std::getline(in, raw)) {
    ++line;
    const size_t hash = raw.find('#');
    const std::string s = trim(hash == std::string::npos ? raw : raw.substr(0, hash));
    if (s.empty()) continue;
    if (s.front() == '[') {
      if (s.back() != ']') parse_error(line, "unterminated section header '" + s + "'");
      const std::string name = trim(s.substr(1, s.size() - 2));
      if (name.rfind("module.", 0) == 0) {
        const std::string mod = name.substr(7);
        if (!is_ident(mod) || mod.find('.') != std::string::npos)
          parse_error(line, "bad module name '" + mod + "'");
        for (const auto& m : c.modules)
          if (m.layout.name == mod) parse_error(line, "module '" + mod + "' defined twice (first at line " +
                                                          std::to_string(m.line) + ")");
        ModuleEntry e;
        e.layout.name = mod;
        e.line = line;
        c.modules.push_back(e);
        section = kModule;
      } else if (name == "model") {
        section = kModel;
      } else if (name == "run") {
        section = kRun;
      } else {
        parse_error(line, "unknown section '[" + name + "]' (expected [module.<name>], [model] or [run])");
      }
      sec_name = name;
      continue;
    }
    const size_t eq = s.find('=');
    if (eq == std::string::npos) parse_error(line, "expected 'key = value', got '" + s + "'");
    const std::string key = trim(s.substr(0, eq)), val = trim(s.substr(eq + 1));
    if (!is_ident(key)) parse_error(line, "bad key '" + key + "'");
    if (!is_number(val)) parse_error(line, "'" + key + "' needs an integer or decimal value, got '" + val + "'");
    if (section == kNone) parse_error(line, "key '" + key + "' outside any section");
    const std::string sk = sec_name + "/" + key;
    if (auto it = seen.find(sk); it != seen.end())
      parse_error(line, "key '" + key + "' repeated (first at line " + std::to_string(it->second) + ")");
    seen[sk] = line;
    if (section == kModule) {
      bool known = false;
      for (const auto& k : kLayoutKeys) {
        if (key != k.key) continue;
        const long long x = to_int(line, key, val);
        if (x < (k.field == &grid::ModuleLayout::rank_offset ? 0 : 1) || x > (1 << 20))
          parse_error(line, "'" + key + "' out of range: " + val);
        c.modules.back().layout.*(k.field) = static_cast<int>(x);
        known = true;
      }
      if (!known) parse_error(line, "unknown module key '" + key + "'");
    } else if (section == kModel) {
      c.model[key] = val;
    } else {
      c.run[key] = val;
      if (key == "global_batch") c.global_batch = static_cast<int>(to_int(line, key, val));
      else if (key == "num_microbatches") c.num_microbatches = static_cast<int>(to_int(line, key, val));
      else if (key == "steps") c.steps = static_cast<int>(to_int(line, key, val));
      else if (key == "seed") c.seed = to_int(line, key, val);
      else if (key == "tolerance") c.tolerance = std::strtod(val.c_str(), nullptr);
    }
  }

  // ---- validation (ExperimentConfig invariants)
  int n_lang = 0;
  for (const auto& m : c.modules) n_lang += m.layout.name == "language";
  if (n_lang != 1) invalid("exactly one [module.language] is required");
  if (c.modules.size() < 2) invalid("at least one encoder module is required besides [module.language]");
  if (c.num_microbatches < 1) invalid("num_microbatches must be >= 1");
  if (c.steps < 0) invalid("steps must be >= 0");
  if (c.global_batch < 0) invalid("global_batch must be >= 0");
  if (c.global_batch > 0 && c.global_batch % c.num_microbatches != 0)
    invalid("IndivisibleBatch: global_batch " + std::to_string(c.global_batch) + " not divisible by num_microbatches " +
            std::to_string(c.num_microbatches));
  for (const auto& m : c.modules) {
    try {
      m.layout.validate();
    } catch (const Error& e) {
      invalid(std::string("module '") + m.layout.name + "': " + e.what());
    }
    const int mb = c.global_batch > 0 ? c.global_batch / c.num_microbatches : 0;
    if (mb > 0 && mb % m.layout.dp != 0)
      invalid("IndivisibleBatch: microbatch of " + std::to_string(mb) + " samples not divisible by module '" +
              m.layout.name + "' data_parallel_size " + std::to_string(m.layout.dp));
  }
  const auto& lang = c.language().layout;
  for (const auto& m : c.modules) {
    if (m.layout.name == "language") continue;
    grid::BoundaryEdge e{m.layout, lang, 0, 0};
    try {
      grid::placement_of_edge(e);
    } catch (const Error& err) {
      invalid(std::string("PartialOverlap: ") + err.what());
    }
  }
  return c;
}

std::string render_config(const ExperimentConfig& c) {
  std::ostringstream o;
  for (const auto& m : c.modules) {
    o << "[module." << m.layout.name << "]\n";
    for (const auto& k : kLayoutKeys) o << k.key << " = " << m.layout.*(k.field) << "\n";
    o << "\n";
  }
  if (!c.model.empty()) {
    o << "[model]\n";
    for (const auto& [k, v] : c.model) o << k << " = " << v << "\n";
    o << "\n";
  }
  if (!c.run.empty()) {
    o << "[run]\n";
    for (const auto& [k, v] : c.run) o << k << " = " << v << "\n";
  }
  return o.str();
}

}  // namespace hb::config
