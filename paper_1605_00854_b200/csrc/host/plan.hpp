// Structural preprocessing ("Preparation", Alg. 5 of the paper): leaf
// reduction, grouped perturbation plan, node grouping and the flattening into
// the arrays the per-step kernel reads.
//
// The output is byte-identical to the reference's pbn::prepare
// (engine.hpp:85-164) for the same (model, theta, k_max, max_group_parents):
// tests/test_plan_parity.py compares every array bitwise against the
// unmodified reference built in oracle/_ref.
#pragma once

#include <cstdint>
#include <vector>

#include "model.hpp"

namespace pbn_b200 {

// Walker alias table, two-worklist construction (alias.hpp:18-56).
struct walker_table {
  std::vector<double> cut;
  std::vector<std::uint32_t> alias;
  std::uint32_t size() const { return static_cast<std::uint32_t>(cut.size()); }
};
walker_table build_walker(const double* probs, std::size_t n);

// Smallest m with m * (prod w)^(1/m) <= theta (grouping.hpp:50-57, Ineq. 2).
std::uint32_t partition_lower_bound(const std::vector<std::uint32_t>& w, std::uint64_t theta);
// Greedy multiplicative partition (grouping.hpp:63-82, Alg. 3), O(n log m).
std::vector<std::vector<std::uint32_t>> greedy_product_partition(
    const std::vector<std::uint32_t>& w, std::uint32_t m);

inline constexpr std::uint64_t kGroupEntryCap = 1ull << 22;  // grouping.hpp:42
inline constexpr std::uint64_t kTotalEntryCap = 1ull << 24;  // grouping.hpp:46
inline constexpr std::uint32_t kPertMaxWidth = 24;           // perturbation.hpp:23
inline constexpr std::uint32_t kGatherPad = 8;               // engine.hpp:52

struct prepared_plan {
  // reduction (reduction.hpp:14-22)
  std::uint32_t original_n = 0;
  std::vector<std::uint32_t> removed;
  std::vector<std::int32_t> index_map;
  double t = 1.0;
  network kept;
  // perturbation plan (perturbation.hpp:16-44)
  std::uint32_t g = 0, k = 0, k_prime = 0;
  std::uint64_t mask = 0;
  walker_table pert;
  // grouping (grouping.hpp:30-39)
  std::vector<std::vector<std::uint32_t>> members;  // reduced indices, engine order
  std::vector<std::uint32_t> cum;
  // engine arrays (engine.hpp:22-79)
  std::vector<std::uint32_t> engine_pos, engine_nodes;
  std::vector<std::uint32_t> grp_offset, grp_fn_begin, grp_alias_begin, grp_alias_size;
  std::vector<double> alias_cut;
  std::vector<std::uint32_t> alias_idx;
  std::vector<std::uint64_t> fn_gather_begin, fn_table_begin;
  std::vector<std::uint32_t> fn_gather_count;
  std::vector<std::uint32_t> fn_gather;
  std::vector<std::uint64_t> fn_tables;
  // stepper kind (see pbn_plan_view): grouped by default
  std::uint32_t pert_mode = 0, has_leaf = 1;
  double pert_p = 0.0;
  std::vector<std::uint32_t> grp_members;  // node-wise plans only

  std::uint32_t n_kept() const { return kept.size(); }
};

prepared_plan prepare_plan(const network& m, std::uint64_t theta, std::uint32_t k_max,
                           std::uint32_t max_group_parents);

// Node-wise plan for the node-by-node steppers (engine.hpp:168-242): one group
// per node of the full (reduced = false) or leaf-reduced model, per-node alias
// selectors over the node's functions (alias.hpp:18-56), each function's own
// parent order as its gather list and its truth table as the table.
prepared_plan prepare_nodewise_plan(const network& m, bool reduced);

}  // namespace pbn_b200
