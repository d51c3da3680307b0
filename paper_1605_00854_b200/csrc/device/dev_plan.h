// Device encoding of a prepared plan: one contiguous, 16-byte-aligned blob the
// kernel stages into shared memory with a 1-D bulk copy (cp.async.bulk), plus
// a small header passed by value as a kernel parameter.
//
// Layout (all offsets in bytes from the blob start, each section 16-aligned;
// order core sections | tables | pert32 | pert53, so every placement level is
// a prefix: 0 nothing staged, 1 core, 2 core + tables, 3 + perturbation cells
// of the launch's stream):
//   pert53[2^k]   u64  perturbation cells for the U53 stream:
//                      bits [0, 53-k) threshold T, bits [53-k, 53) cell result
//                      on a miss. A draw r53 picks cell c = r53 >> (53-k) and
//                      returns (r53 & (2^(53-k)-1)) < T ? c : alias — exactly
//                      alias_table::next (alias.hpp:70-76) for N = 2^k, where
//                      T = ceil(cut * 2^(53-k)); cells whose cut rounds to the
//                      whole range store (T=0, alias=c).
//   pert32[2^k]   u32  the same for the U32 stream with 32-k threshold bits.
//   groups[G]     uint4 {offset, fn_begin, alias_begin, alias_size | (members-1)<<24};
//                      the A alias groups come first (grouping.hpp: multi-function
//                      groups precede single-function ones), so the function phase
//                      runs an alias region [0, A) and a plain region [A, G).
//   fns[F]        uint4 {table byte offset — or, when the whole table fits in 32
//                        bits (members * 2^gather_count <= 32), the table itself,
//                        gather count | entry log2 << 5 | inline << 7 | extra-record quad << 8,
//                        records 0,1 (u16 each), records 2,3}
//   grec[...]     u16  gather records 4.. of functions with more than 4 parents,
//                      4-aligned per function. A record is
//                      (word32 << 5) | ((bit32 - slot) & 31): a funnel rotate by the
//                      low 5 bits lands the parent bit at `slot`. Unused slots hold
//                      the always-zero bit n' (engine.hpp:149-150).
//   acut[A]       f64  group alias cut-offs (U53 path, FP64 like engine.hpp:285-290)
//   aidx[A]       u32  group alias targets
//   a32[A]        uint2 {ceil(cut * 2^32) or 0, alias or self}: U32 integer path
//   arec[A1]      u32  compact record of the leading single-node alias groups:
//                      base | alias_size << 24 (their fn_begin == alias_begin == base)
//   tables        packed member outputs, entry width 1/2/4/8 bytes by member count
#pragma once

#include <cstdint>

namespace pbn_b200 {

inline constexpr std::uint32_t kMaxPredWords = 16;

struct dev_plan_header {
  std::uint32_t n_kept;
  std::uint32_t sw32;       // u32 state words per trajectory (= 2 * (n_kept/64 + 1))
  std::uint32_t g;          // perturbation groups
  std::uint32_t k;          // perturbation width
  std::uint32_t last_mask;  // 2^k' - 1 (k' <= 24)
  std::uint32_t n_groups;
  std::uint32_t max_alias;  // largest group alias table
  std::uint64_t leaf_thr53; // floor(t * 2^53): leaf perturbation iff r53 > thr
  std::uint32_t leaf_thr32; // floor(t * 2^32) (saturated)
  std::uint32_t leaf_never; // t == 1: the leaf draw can never fire
  std::uint32_t off_pert53, off_pert32, off_groups, off_fns, off_grec;
  std::uint32_t off_acut, off_aidx, off_a32, off_arec, off_tables;
  std::uint32_t core_bytes;   // bytes [0, off_tables)
  std::uint32_t table_bytes;  // bytes [off_tables, off_pert32)
  std::uint32_t blob_bytes;   // whole blob: core | tables | pert32 | pert53
  std::uint32_t u32_ok;       // every group alias size <= 2^21 (U32 path exact)
  std::uint32_t n_alias_groups;  // A: groups [0, A) draw a combined function
  std::uint32_t n_single_alias;  // A1 <= A: groups [0, A1) are single nodes at offset = index,
                                 // every function's table inline (1 bit x <= 32 entries)
  std::uint32_t rg_ok;           // sw32 <= 32: one state word per lane fits a warp (SHFL gather)
  std::uint32_t single_gc5;      // some function of groups [0, A1) has 5 parents
  std::uint32_t pert_mode;       // 0 grouped patterns, 1 per-node Bernoulli(p) (Method_old)
  std::uint32_t has_leaf;        // phase A ends with the leaf draw
  std::uint64_t pthr53;          // Bernoulli: flip iff r53 < ceil(p * 2^53)
  std::uint64_t pthr32;          //            flip iff r32 < ceil(p * 2^32)
};

// Compiled predicate: the state satisfies it iff for every i,
// (word[w[i]] & mask[i]) == want[i].
struct dev_predicate {
  std::uint32_t n;
  std::uint32_t w[kMaxPredWords];
  std::uint32_t mask[kMaxPredWords];
  std::uint32_t want[kMaxPredWords];
};

struct dev_run_params {
  std::uint32_t rk0[10], rk1[10];  // Philox round keys of the seed
  std::uint64_t traj_begin;
  std::uint32_t n_traj;
  std::uint32_t pad0;
  std::uint64_t step_begin;
  std::uint64_t n_steps;
  dev_predicate pred;
  // predicate-process statistics (estimator.hpp:76-102): transitions between
  // samples taken every `kappa`-th step; first previous sample = the input
  // state's predicate with phase 0 (thin_mode 0), carried over from
  // tprev[traj] = prev | phase << 2 (1; prev 2 = none), or none (2)
  std::uint32_t kappa;
  std::uint32_t thin_mode;
  std::uint8_t* tprev;          // per trajectory, in/out, may be null
  // optional series of predicate bits: step i -> bit series_bit0 + i of the
  // trajectory's row; series_init: the input state's bit at series_bit0 - 1
  std::uint32_t* series;
  std::uint64_t series_stride;  // u32 words per trajectory row
  std::uint64_t series_bit0;
  std::uint32_t series_init;
  std::uint32_t pad1;
  // optional per-node one-counts (engine.hpp:378-379): n_traj x n_kept u64,
  // accumulated (+=) over the call's steps
  std::uint64_t* node_counts;
};

}  // namespace pbn_b200
