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
  std::vector<std::uint8_t> blob;  // core sections then tables
};

encoded_plan encode_plan(const pbn_plan_view& v);

// Predicate terms (engine bit, value) -> per-word masks (engine.hpp:328-332).
dev_predicate compile_dev_predicate(const std::uint32_t* bits, const std::uint8_t* vals,
                                    std::uint32_t n, std::uint32_t n_kept);

// Philox round keys of a 64-bit seed (key bump 0x9E3779B9 / 0xBB67AE85).
void philox_round_keys(std::uint64_t seed, std::uint32_t rk0[10], std::uint32_t rk1[10]);

}  // namespace pbn_b200
