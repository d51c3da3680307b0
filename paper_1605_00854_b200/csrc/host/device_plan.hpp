// Host-side encoder: pbn_plan_view (the reference's flat prepared_simulation
// arrays) -> device blob (dev_plan.h). Pure host code, testable without a GPU.
#pragma once

#include <cstdint>
#include <vector>

#include "../../../include/pbn_b200.h"
#include "../device/dev_plan.h"

namespace pbn_b200 {

struct encoded_plan {
  dev_plan_header h{};
  std::vector<std::uint8_t> blob;  // stageable prefix (h.blob_bytes) + exact section
  std::uint32_t total_bytes = 0;   // blob.size()
};

encoded_plan encode_plan(const pbn_plan_view& v);

// Exact combined-function rule of engine.hpp:285-290 for one 53-bit draw, and
// the per-cell cut points of its integer form (dev_plan.h a53).
std::uint32_t alias53_cell(std::uint64_t r53, std::uint32_t n);
double alias53_frac(std::uint64_t r53, std::uint32_t n);
std::vector<std::uint64_t> alias53_cut_points(const double* cut, std::uint32_t n);
// a53 records {alias[c], hi32 of cut point c} of one group, and the kernel's
// integer choice from the draw's high word (rare: boundary draw, FP64 path).
std::vector<std::uint32_t> alias53_records(const double* cut, const std::uint32_t* alias,
                                           std::uint32_t n);
std::uint32_t alias53_pick_int(const std::uint32_t* rec, std::uint32_t n, std::uint32_t hi,
                               bool& rare);

// Predicate terms (engine bit, value) -> per-word masks (engine.hpp:328-332).
dev_predicate compile_dev_predicate(const std::uint32_t* bits, const std::uint8_t* vals,
                                    std::uint32_t n, std::uint32_t n_kept);

// Philox round keys of a 64-bit seed (key bump 0x9E3779B9 / 0xBB67AE85).
void philox_round_keys(std::uint64_t seed, std::uint32_t rk0[10], std::uint32_t rk1[10]);

}  // namespace pbn_b200
