// FSDP layout planner (host only).  SURVEY.md §8(a) A0 / §8(e).
//
// Canonical order (layer-major), independent restatement:
//   MLP  : fc1.w [H x Din], fc1.b [H], fc2.w [C x H], fc2.b [C]
//   GPT  : wte [V x D], wpe [T x D];
//          per block: ln1.g, ln1.b [D], qkv.w [3D x D], qkv.b [3D], proj.w [D x D], proj.b [D],
//                     ln2.g, ln2.b [D], fc.w [F x D], fc.b [F], mproj.w [D x F], mproj.b [D];
//          lnf.g, lnf.b [D], head.w [V x D] (absent when tied)
//   Llama: tok [V x D]; per block: attn_norm [D], wq [Hq*hd x D], wk [Hkv*hd x D],
//          wv [Hkv*hd x D], wo [D x Hq*hd], mlp_norm [D], wg [F x D], wu [F x D], wd [D x F];
//          norm [D], head.w [V x D] (absent when tied)
// Units: MLP = {all}; GPT/Llama = {embedding}, {block l} x L, {final norm (+ head)}.
#pragma once

#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/slq.h"

namespace slq {

struct TensorSlot {
  std::string name;
  int64_t offset;  // within its unit
  int64_t rows, cols;  // cols == 1 for vectors
  int64_t numel() const { return rows * cols; }
};

struct UnitPlan {
  std::vector<TensorSlot> tensors;
  int64_t global_offset = 0;  // canonical offset of the unit's first parameter
  int64_t numel = 0;          // real parameters
  int64_t padded = 0;         // roundup(numel, 16 * world)
  int64_t chunk = 0;          // padded / world
  int64_t local_offset = 0;   // offset of this unit's chunk in the local shard
  const TensorSlot& t(const std::string& n) const;
};

struct LayoutPlan {
  std::vector<UnitPlan> units;
  int64_t P = 0;      // real parameters
  int64_t P_loc = 0;  // local shard length (padded)
  int world = 1;
};

void validate_desc(const slq_model_desc& d);
LayoutPlan plan_layout(const slq_model_desc& d, int world);

}  // namespace slq
