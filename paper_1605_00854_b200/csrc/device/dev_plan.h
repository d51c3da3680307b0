// Device encoding of a prepared plan: one contiguous, 16-byte-aligned blob the
// kernel stages into shared memory with a 1-D bulk copy (cp.async.bulk), plus
// a small header passed by value as a kernel parameter.
//
// Layout (all offsets in bytes from the blob start, each section 16-aligned;
// order core sections | tables | pert32 | pert53 | exact, so every placement
// level is a prefix: 0 nothing staged, 1 core, 2 core + tables, 3 +
// perturbation cells of the launch's stream; `exact` is never staged):
//
// U53 draws are compared in raw-word form: the two Philox words of a draw,
// R = x[2e+1] << 32 | x[2e], satisfy r53 = R >> 11, so r53 < T  <=>  R < T << 11.
//
//   pert53[2^k]   u64  perturbation cells for the U53 stream, raw-word form:
//                      bits [11, 64-k) threshold T, bits [64-k, 64) cell result
//                      on a miss. A draw picks cell c = R >> (64-k) and returns
//                      (R mod 2^(64-k)) < (cell mod 2^(64-k)) ? c : alias —
//                      exactly alias_table::next (alias.hpp:70-76) for N = 2^k,
//                      where T = ceil(cut * 2^(53-k)); cells whose cut rounds to
//                      the whole range store (T=0, alias=c).
//   pert32[2^k]   u32  the same for the U32 stream with 32-k threshold bits.
//   pert53h[2^k]  u32  the high words of pert53 (cell result + the threshold's top
//                      32-k bits), never staged: launches that read the cells
//                      through L1/L2 decide on these (half the cache footprint of
//                      the 8-byte cells: 256 KiB at k = 16) and touch pert53
//                      itself only on a tie.
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
//   acell[A]      uint4 group alias cells {U53: alias[c], hi32 of C[c]; U32: threshold,
//                      alias}. U32: {ceil(cut * 2^32) or 0, alias or self}; a draw x
//                      with P = x * N picks c = P >> 32 iff (P mod 2^32) < threshold.
//                      U53: integer form of engine.hpp:285-290 for groups of N <= 2048
//                      functions, C[c] = the first r53 of cell c whose fraction
//                      reaches cut[c] (alias53_cut_points; capped at 2^53-1). From the
//                      draw's high word hi: P = hi * N, e = P >> 32. Unless (P mod
//                      2^32) > ~N (hi is the last high word of bucket e, where the
//                      double rounding can cross into cell e+1; N < 2^21 keeps it
//                      within one step) or hi == hi32(C[e]), the choice is
//                      hi < hi32(C[e]) ? e : alias[e]; the rare rest (about N+1 draws
//                      in 2^32) takes the exact FP64 path.
//   arec[A1]      u32  compact record of the leading single-node alias groups:
//                      base | alias_size << 24 (their fn_begin == alias_begin == base)
//   scol          (single_compact) bank-column records of the single-node groups:
//                      rows of kScolSlots 8-byte slots (128 bytes); group j owns slot
//                      j % kScolSlots, so a half-warp's 16 lanes of one round read 16
//                      distinct bank pairs. Per group, consecutive rows of its slot
//                      hold N U53 cells {alias, hi32(C)}, N U32 cells {threshold,
//                      alias} and N function records {rec0 | rec1 << 10 | rec2 << 20,
//                      rec3 | table << 16} (10-bit gather records word << 5 | rotation)
//   arec4[A1]     uint4 (single_compact) {byte offset of the group's first U53 cell,
//                      of its first function record, N, ~N}; row stride 128 bytes
//   tables        packed member outputs, entry width 1/2/4/8 bytes by member count
//   acut[A] f64, aidx[A] u32 (exact section): the group cut-offs and targets
//                      for the FP64 path (boundary draws, groups with N > 2048)
//   sgrp[A1]      uint4 (single_compact_l, n' > 2047) per single-node alias group
//                      j (N <= 4 functions): U53 cell c in word c = hi32(C[c]) with
//                      bits [0, 4) replaced by alias[c] << 2 | (c == 0 ? N-1 : 0);
//                      a draw's high word hi picks e = (hi * N) >> 32 and then
//                      e if hi >> 4 < word_e >> 4, alias if greater — equal, or
//                      (hi * N mod 2^32) > ~N, is rare (exact redo). First
//                      section, staged by every GM 4 launch.
//   sfn[4 A1]     uint4 (single_compact_l) function c of group j at 4j + c:
//                      {1-bit table of <= 32 entries, records 0 | 1 << 16,
//                      records 2 | 3 << 16, record 4 | gather count << 16}
//   fns_s, acell_s     (single_compact) the single-node groups' fns and acell
//                      entries, moved out of the staged core: the compact kernels
//                      read scol instead; fallback kernels (other LPT) read these
#pragma once

#include <cstdint>

namespace pbn_b200 {

inline constexpr std::uint32_t kMaxPredWords = 16;
#ifndef PBN_CHUNK_BLOCKS
#define PBN_CHUNK_BLOCKS 1
#endif
// Phase-B Philox blocks each lane computes per draw-buffer chunk (a chunk is
// LPT * kChunkBlocks blocks); the per-trajectory draw buffer holds one chunk.
inline constexpr std::uint32_t kChunkBlocks = PBN_CHUNK_BLOCKS;
#ifndef PBN_PHILOX_PIPELINE
#define PBN_PHILOX_PIPELINE 0
#endif
// 1: the next chunk's Philox blocks are computed while the current chunk's
// rounds run (software pipelining; ALU work overlaps the rounds' load latency)
inline constexpr bool kPhiloxPipeline = PBN_PHILOX_PIPELINE != 0;
#ifndef PBN_COMPACT_SINGLE
#define PBN_COMPACT_SINGLE 1
#endif
#ifndef PBN_QUAD_ROUNDS
#define PBN_QUAD_ROUNDS 1
#endif
// four compact single-node rounds interleaved when a chunk holds four rounds
// (U32: 4 draws per block; U53 would need two blocks per lane, which costs more)
inline constexpr bool kQuadRounds = PBN_QUAD_ROUNDS != 0;
inline constexpr bool kUseCompactSingle = PBN_COMPACT_SINGLE != 0;  // GM = 2 when the plan allows
inline constexpr std::uint32_t kA53MaxCells = 2048;
inline constexpr std::uint32_t kScolSlots = 16;          // 8-byte slots per 128-byte row           // alias fits the low 11 bits
inline constexpr std::uint32_t kGroupExactAlias = 1u << 23;   // groups[].w flag: FP64 path only

struct dev_plan_header {
  std::uint32_t n_kept;
  std::uint32_t sw32;       // u32 state words per trajectory (= 2 * (n_kept/64 + 1))
  std::uint32_t g;          // perturbation groups
  std::uint32_t k;          // perturbation width
  std::uint32_t last_mask;  // 2^k' - 1 (k' <= 24)
  std::uint32_t n_groups;
  std::uint32_t max_alias;  // largest group alias table
  std::uint64_t leaf_thr53; // raw word: leaf perturbation iff R > floor(t * 2^53) << 11 | 0x7FF
  std::uint32_t leaf_thr32; // floor(t * 2^32) (saturated)
  std::uint32_t leaf_never; // t == 1: the leaf draw can never fire
  std::uint32_t off_pert53, off_pert32, off_groups, off_fns, off_grec;
  std::uint32_t off_acut, off_aidx, off_acell, off_arec, off_scol, off_arec4, off_tables;
  std::uint32_t off_fns_s, off_acell_s;  // single-node groups' fns / acell entries (absolute
                                         // indices): the unstaged tail when fn_base or
                                         // cell_base != 0, else = off_fns / off_acell
  std::uint32_t fn_base, cell_base;      // groups[].y / .z are relative to these
  std::uint32_t core_bytes;   // bytes [0, off_tables)
  std::uint32_t table_bytes;  // bytes [off_tables, off_pert32)
  std::uint32_t blob_bytes;   // stageable prefix: core | tables | pert32 | pert53
  std::uint32_t u32_ok;       // every group alias size <= 2^21 (U32 path exact)
  std::uint32_t n_alias_groups;  // A: groups [0, A) draw a combined function
  std::uint32_t n_single_alias;  // A1 <= A: groups [0, A1) are single nodes at offset = index,
                                 // every function's table inline (1 bit x <= 32 entries)
  std::uint32_t rg_ok;           // sw32 <= 32: one state word per lane fits a warp (SHFL gather)
  std::uint32_t single_gc5;      // some function of groups [0, A1) has 5 parents
  std::uint32_t single_compact;  // rg_ok, A1 >= 32, no 5-parent function: sfn/arec4 present
  std::uint32_t single_compact_l;  // !rg_ok, A1 >= 32, every single group N <= 4: sgrp/sfn present
  std::uint32_t off_sgrp, off_sfn;  // sgrp at 0: the GM 4 kernels stage [0, off_sfn)
  std::uint32_t pert_mode;       // 0 grouped patterns, 1 per-node Bernoulli(p) (Method_old)
  std::uint32_t has_leaf;        // phase A ends with the leaf draw
  std::uint64_t pthr53;          // Bernoulli: flip iff R < ceil(p * 2^53) << 11 (raw word)
  std::uint64_t pthr32;          //            flip iff r32 < ceil(p * 2^32)
  std::uint32_t off_pert53h;     // high words of pert53 (unstaged tail)
  std::uint32_t reserved1;
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
  std::uint32_t exact_alias;  // 1: every U53 combined-function choice takes the FP64 path
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
  std::uint32_t reserved0;
  // optional per-node one-counts (engine.hpp:378-379): n_traj x n_kept u64,
  // accumulated (+=) over the call's steps
  std::uint64_t* node_counts;
  // scripted replay (pbn_gpu_run_scripted): the draws' raw words in the
  // stream's slot layout — trajectory t, step i, block b at
  // [(t * n_steps + i) * script_bps + b]: high words in script_hi, low words in
  // script_lo (draw e of block b = word e; r53 = (hi << 32 | lo) >> 11)
  const void* script_hi;  // 16-byte blocks
  const void* script_lo;
  std::uint64_t script_bps;
  std::uint64_t reserved2;  // keeps the parameters that follow 16-byte aligned
};

}  // namespace pbn_b200
