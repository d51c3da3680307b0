// BASELINE-shaped synthetic network generator; see generator.cpp.
#pragma once

#include <cstdint>
#include <vector>

#include "model.hpp"

namespace pbn_b200 {

struct gen_params {
  std::uint32_t n = 100;
  std::uint32_t f_min = 1, f_max = 3;
  std::uint32_t p_min = 1, p_max = 3;
  double leaf_frac = 0.0;
  double p = 0.01;
  std::uint32_t n_targets = 2;
  bool targets_fixed = false;
  std::uint64_t seed = 1605;
};

struct generated_network {
  network net;
  std::vector<std::uint32_t> pred_nodes;  // original indices
  std::vector<std::uint8_t> pred_vals;
};

generated_network generate_network(const gen_params& gp);

}  // namespace pbn_b200
