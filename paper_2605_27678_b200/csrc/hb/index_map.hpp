// hetbridge — ownership index builder.
//
// Collapses a BridgePlan's multi-hop routes (leader send + broadcast,
// all-gather, deliver, cp all-reduce) into direct element maps:
//   forward : every destination element has exactly one source element
//             (pure placement; bit-exact copy),
//   backward: every source-gradient element is an ordered sum of destination
//             gradient elements (the cp all-reduce order of simnet.cpp:299-313,
//             i.e. ascending group order starting from +0.0).
// Provenance follows the exact data path the reference roles take
// (bridge.hpp:150-162), including which tp replica's copy a
// rank reads, so results equal the oracle even for inputs that violate the
// "tp replicas are identical" contract.
//
// With a SpliceSpec the maps are composed with the embedding splice
// (tinymodel.hpp:94-112): forward writes each CP rank's token slice straight
// from the encoder owners' rows, backward returns each vision token's
// gradient from the single CP slice that holds its position. Positions that
// lie outside a slice are structural zeros and are dropped from the sums.
#pragma once

#include <cstdint>
#include <vector>

#include "hb/bridge.hpp"

namespace hb::index {

// Per-logical-rank buffer slots.
enum Slot : int {
  kSrcAct = 0,   // source shard (forward input)
  kDstAct = 1,   // destination shard or token slice (forward output)
  kDstGrad = 2,  // destination gradient or token-slice gradient (backward input)
  kSrcGrad = 3,  // source gradient (backward output, accumulate target)
  kText = 4,     // text embedding rows (splice forward input)
  kNumSlots = 5,
};

struct Ref {
  int rank = -1;
  int slot = 0;
  int64_t off = 0;  // element offset
};

struct CopySeg {
  Ref src, dst;
  int64_t n = 0;  // elements
};

struct ReduceSeg {
  Ref dst;
  int64_t n = 0;
  std::vector<Ref> terms;  // each covers n contiguous elements from term.off; summed in order
};

// Text rows of a CP slice: Full / Slice — the boundary copies them from the
// TEXT buffer (indexed by global text row / by position within the slice);
// InPlace — the caller's embedding layer already wrote them into the
// destination slice (DST_ACT bound to the LLM's input-embedding tensor), and
// the boundary writes only the vision rows at the placeholder positions (the
// masked scatter `inputs_embeds[image_mask] = image_features` of VLM
// implementations): no TEXT buffer, no text bytes through the boundary.
enum class TextMode { Full = 0, Slice = 1, InPlace = 2 };

struct SpliceSpec {
  int Q = 0;        // sequences per destination shard
  int S = 0;        // positions per sequence
  int d_h = 0;      // hidden width (elements per token row)
  int S_v = 0;      // vision tokens per sample; feature_width == S_v * d_h
  TextMode text_mode = TextMode::Full;
  std::vector<int32_t> codes;  // Q*S: >=0 vision row j*S_v+t of the shard, <0 text row -1-code

  void validate(const bridge::BridgePlan& plan) const;
};

struct IndexMap {
  int world = 0;                            // logical ranks [0, world)
  std::vector<CopySeg> fwd;                 // grouped by destination rank, ascending offsets
  std::vector<ReduceSeg> bwd;               // grouped by destination rank, ascending offsets
  std::vector<std::vector<int64_t>> elems;  // [rank][slot] buffer size in elements (0 = unused)
  int max_terms = 0;
};

/// balance_replicas: the backward reads each destination-gradient term from
/// one of the holder's tensor-parallel replicas instead of always the tp=0
/// copy (bridge.hpp:33-36: tp replicas hand back identical gradients), chosen
/// as the source rank itself when it is one of them, else replica j % tp for
/// global sample j. The sums are unchanged for inputs that honour the
/// contract, and the NVLink egress of a gradient return is spread over the tp
/// replicas instead of concentrating on the tp=0 rank. false reproduces the
/// reference data path replica for replica (strict provenance).
IndexMap build_index_map(const bridge::BridgePlan& plan, const SpliceSpec* splice, bool balance_replicas = false);

/// Row-level provenance, exposed for tests: source rank/row that feeds
/// destination rank `r`'s global sample j in forward, and the ordered
/// destination (rank,row) terms that sum into source rank `r`'s sample j.
struct RowRef {
  int rank;
  int row;
};
RowRef forward_origin(const bridge::BridgePlan& plan, int r, int j);
std::vector<RowRef> backward_origin(const bridge::BridgePlan& plan, int r, int j);

}  // namespace hb::index
