// hetbridge — module_parallelisms configuration ingestion.
//
// The reference declares the schema in SPEC.md's cli module (S:495-545:
// ExperimentConfig, parse_config, the `[module.<name>]` grammar) mirroring the
// paper's Appendix B (`module_parallelisms={"language": ...,
// "images": ...}`); its config.cpp is a stub. This is the parser and
// validator, producing the grid::ModuleLayout of every module and the
// encoder -> language BoundaryEdge the boundary plan is built from.
#pragma once

#include <map>
#include <string>
#include <vector>

#include "hb/grid.hpp"

namespace hb::config {

struct ModuleEntry {
  grid::ModuleLayout layout;  // layout.name = the module name
  int line = 0;               // line of its section header
};

struct ExperimentConfig {
  std::vector<ModuleEntry> modules;  // in file order
  std::map<std::string, std::string> model;  // [model] key -> numeric text
  std::map<std::string, std::string> run;    // [run] key -> numeric text
  int global_batch = 0;       // [run] global_batch (0: absent)
  int num_microbatches = 1;   // [run] num_microbatches
  int steps = 1;              // [run] steps
  long long seed = 0;         // [run] seed
  double tolerance = 0.0;     // [run] tolerance

  const ModuleEntry& language() const;  // the single "language" module
  const ModuleEntry& module(const std::string& name) const;
  // encoder -> language edge of one microbatch (global_batch / num_microbatches samples)
  grid::BoundaryEdge edge(const std::string& encoder, int feature_width) const;
};

// Grammar: `#` comments to end of line; blank lines; section headers
// `[module.<name>]`, `[model]`, `[run]`; `key = value` lines with an integer
// or decimal value. Module keys: tensor_model_parallel_size,
// context_parallel_size, pipeline_model_parallel_size, data_parallel_size,
// rank_offset (defaults 1, 1, 1, 1, 0). Errors: ParseError "line N: ..." for
// malformed text, ValidationError naming the violated invariant (exactly one
// "language" module and >= 1 encoder; valid layouts; global_batch divisible by
// every data_parallel_size and by num_microbatches; every encoder's rank range
// equal to or disjoint from the language module's).
ExperimentConfig parse_config(const std::string& text);

// Canonical text: parse(render(c)) == c and render is byte-stable.
std::string render_config(const ExperimentConfig& c);

}  // namespace hb::config
