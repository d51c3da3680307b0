// Ensemble trajectory kernel: many independent PBN trajectories, each advanced
// `n_steps` steps of the structure-based stepper (Alg. 5 of the paper; the
// reference's grouped_simulator::step, engine.hpp:255-312, driven by
// simulate(), engine.hpp:371-384), bit-exact on the injected Philox stream.
//
// Work decomposition: one trajectory per sub-warp of LPT lanes (LPT = 32:
// one per warp; LPT = 1: one per thread). Per step, lane r of a sub-warp
//   * phase A: draws Philox blocks r, r+LPT, ... holding the step's first g+1
//     draws (the g grouped-perturbation draws and the leaf draw), looks each
//     pattern up in the perturbation cells and XORs any flip into the state
//     (engine.hpp:257-266); a sub-warp ballot is the short-circuit — any kept
//     flip ends the step (engine.hpp:267), otherwise the leaf draw decides
//     (engine.hpp:268);
//   * function phase, in lockstep rounds: in round t lane r evaluates group
//     t*LPT + r — one combined-function draw (engine.hpp:284-291), a gather
//     of that function's parent bits from the shared state (engine.hpp:
//     292-302), one table lookup (engine.hpp:303) — and the round's outputs
//     are ORed into the next state (engine.hpp:304-309): one ballot word when
//     every group of the round is a single node, shared-memory atomics
//     otherwise. Phase-B draws are produced LPT blocks at a time (lane r
//     computes one block into a per-trajectory draw buffer), because the
//     stream starts phase B on a fresh Philox block.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <type_traits>

#include "kernel_common.cuh"

namespace pbn_b200 {

#ifndef PBN_GENERAL_PAIRS
#define PBN_GENERAL_PAIRS 1
#endif
constexpr bool kGeneralPairs = PBN_GENERAL_PAIRS != 0;
#ifndef PBN_RG2
#define PBN_RG2 1
#endif
constexpr bool kUseRg2 = PBN_RG2 != 0;
#ifndef PBN_PLAIN_SHFL
#define PBN_PLAIN_SHFL 1
#endif
constexpr bool kPlainShfl = PBN_PLAIN_SHFL != 0;

// Block b of the current step's stream (high words) and its low block. The
// scripted-replay translation unit (ensemble_script.cu includes this file
// with PBN_SCRIPT_TU) reads caller-supplied draws laid out in the stream's own
// (step, block) slots instead of computing Philox — the reference's
// forced-draw traces (tests/oracles.hpp:235-254) replayed by the same kernel.
#ifdef PBN_SCRIPT_TU
#define pbn_ensemble_kernel pbn_ensemble_script_kernel
#define PBN_BLK(b) __ldg(static_cast<const uint4*>(rp.script_hi) + script_row + (b))
#define PBN_BLK_LO(b) __ldg(static_cast<const uint4*>(rp.script_lo) + script_row + (b))
#define PBN_BLK_LO_INLINE(b) __ldg(static_cast<const uint4*>(rp.script_lo) + script_row + (b))
#else
#define PBN_BLK(b) philox_block(sp, (b), rp.rk0, rp.rk1)
#define PBN_BLK_LO(b) philox_lo_block(sp, (b), rp.rk0, rp.rk1)
#define PBN_BLK_LO_INLINE(b) philox_block(sp, (b) | kLoBlock, rp.rk0, rp.rk1)
#endif
// Phase-A prefetch (the PF kernels: perturbation-dominated launches of k = 16
// plans with at most one phase-A block per lane): the class of a step is a
// function of the stream alone, so the next step's phase-A Philox block and its
// four perturbation-cell words are fetched into registers while the current
// step finishes (1: issued before the step's ballots; 2: after the function
// phase). Measured on every kernel (A/B on one box): c5 p >= 0.01 +6 %, but
// c2 -10 % and c5 p <= 1e-3 -3..5 % (the hot function-phase loops lose
// registers), so only launches that almost never reach the function phase
// take it (capi.cpp kPertDominated).
#ifndef PBN_PA_PREFETCH
#define PBN_PA_PREFETCH 1
#endif
constexpr int kPaPrefetch = PBN_PA_PREFETCH;
#ifndef PBN_CARVEOUT
#define PBN_CARVEOUT 1
#endif
#ifndef PBN_GATHER_UNROLL
#define PBN_GATHER_UNROLL 1
#endif
#ifndef PBN_PA2
#define PBN_PA2 1
#endif
constexpr bool kPa2 = PBN_PA2 != 0;
#ifndef PBN_PF_WARPS
#define PBN_PF_WARPS 28
#endif
constexpr int kMaxWarpsPf = PBN_PF_WARPS;  // PF kernels: warps per CTA (32 -> 64 registers: spills in the step loop)

// PA2 (two steps per phase-A pass, see the kernel): words of the per-lane
// pattern stash in a trajectory's shared-memory slot, 0 when the plan's phase A
// is not the k = 16 word path filling at most half a warp. Host and device
// size the slot with it.
__host__ __device__ inline std::uint32_t pa2_words(const dev_plan_header& h, std::uint32_t lpt) {
  const std::uint32_t nb0 = (h.g + h.has_leaf + 3) / 4;
  return kPa2 && lpt == 32 && h.pert_mode == 0 && h.k == 16 && 2 * nb0 <= lpt ? 2 * lpt : 0u;
}

// One trajectory per warp runs <= 28 warps per CTA (4096 trajectories fill
// the 148 SMs in one wave), which leaves 72 registers per thread.
constexpr int kMaxWarpsLpt32 = 28;

// GM: parent gather mode — 0 shared-memory state words, 1 one state word per
// lane with shuffles (RG), 2 RG with the compact single-node records (SC), 3
// two state words per lane (RG2, n' <= 2047) for the single-node groups
// (general groups gather from shared memory: they run under divergence).
template <int LPT, int STREAM, int PLACE, int GM, bool PF = false, bool PA2 = false>
__global__ void __launch_bounds__(LPT == 32 ? (PF ? kMaxWarpsPf : kMaxWarpsLpt32) * 32 : 1024, 1)
    pbn_ensemble_kernel(const __grid_constant__ dev_plan_header h, const std::uint8_t* __restrict__ gblob,
                        const __grid_constant__ dev_run_params rp, std::uint64_t* __restrict__ states,
                        std::uint64_t* __restrict__ counts) {
  extern __shared__ __align__(16) std::uint8_t smem[];
  __shared__ std::uint64_t stage_bar;
  constexpr bool GC = placement<PLACE>::global_core;    // core sections read from global
  constexpr bool GT = placement<PLACE>::global_tables;  // tables read from global
  constexpr bool GP = placement<PLACE>::global_pert;    // perturbation cells read from global
  constexpr std::uint32_t DPB = draws<STREAM>::kPerBlock;
  constexpr bool RG = GM >= 1 && GM <= 3;
  constexpr bool RG2 = GM == 3;
  constexpr bool SC = GM == 2;
  constexpr bool SCL = GM == 4;  // compact single-node records, shared-memory gathers (n' > 2047)

  // GM 4 stages at least the sgrp section (blob bytes [0, off_sfn))
  const std::uint32_t staged =
      SCL && staged_prefix<STREAM>(h, PLACE) < h.off_sfn
          ? (stage_plan(smem, gblob, h.off_sfn, &stage_bar), h.off_sfn)
          : stage_placement<STREAM, PLACE>(smem, gblob, h, &stage_bar);

  const std::uint8_t* core = GC ? gblob : smem;
  const std::uint8_t* tab = GT ? gblob + h.off_tables : smem + h.off_tables;
  const std::uint8_t* pcells = pert_cells<STREAM, PLACE>(smem, gblob, h);
  const std::uint8_t* pfast = pert_fast_base<STREAM, GP>(pcells, gblob, h);
  const uint4* groups = reinterpret_cast<const uint4*>(core + h.off_groups);
  const uint4* fns = reinterpret_cast<const uint4*>(core + h.off_fns);
  const uint2* grec = reinterpret_cast<const uint2*>(core + h.off_grec);
  // FP64 cut-offs of the exact path: never staged (dev_plan.h)
  const double* acut = reinterpret_cast<const double*>(gblob + h.off_acut);
  const std::uint32_t* aidx = reinterpret_cast<const std::uint32_t*>(gblob + h.off_aidx);
  const uint4* acell = reinterpret_cast<const uint4*>(core + h.off_acell);
  // single-node groups' fns / acell entries for the non-compact single path
  // (generic loads: staged or the unstaged tail, dev_plan.h)
  const std::uint8_t* sbase = (h.fn_base || h.cell_base) ? gblob : core;
  const uint4* fns_s = reinterpret_cast<const uint4*>(sbase + h.off_fns_s);
  const uint4* acell_s = reinterpret_cast<const uint4*>(sbase + h.off_acell_s);
  const std::uint32_t* arec = reinterpret_cast<const std::uint32_t*>(core + h.off_arec);
  const uint4* arec4 = reinterpret_cast<const uint4*>(core + h.off_arec4);
  const uint4* sgrp = reinterpret_cast<const uint4*>(smem + h.off_sgrp);  // GM 4: always staged
  const uint4* sfn = reinterpret_cast<const uint4*>(core + h.off_sfn);

  const std::uint32_t lane = threadIdx.x & 31;
  const std::uint32_t r = lane % LPT;
  const std::uint32_t sub = lane / LPT;
  const std::uint32_t smask =
      LPT == 32 ? 0xFFFFFFFFu : (((1u << (LPT & 31)) - 1u) << ((sub * LPT) & 31));
  const std::uint32_t slots = blockDim.x / LPT;
  const std::uint32_t slot = threadIdx.x / LPT;
  const std::uint64_t tloc = static_cast<std::uint64_t>(blockIdx.x) * slots + slot;
  if (tloc >= rp.n_traj) return;

  // per-trajectory shared memory: two state buffers + the phase-B draw buffer
  const std::uint32_t sw32 = h.sw32;
  constexpr std::uint32_t CB = kChunkBlocks;
  constexpr std::uint32_t kBuf = LPT * 4 * CB;  // one chunk of Philox blocks (4 words)
  const std::uint32_t nc_words = rp.node_counts ? 8 * sw32 : 0u;  // counter bit-planes
  // PA2 pattern stash, 8 bytes per lane (the host sizes the slots of a PA2-capable plan with it;
  // kernels other than PA2 leave it unused)
  constexpr std::uint32_t pa2w = PA2 ? 2u * LPT : 0u;
  const std::uint32_t stride = (2 * sw32 + kBuf + pa2w + nc_words + 3) & ~3u;
  std::uint32_t* S0 = reinterpret_cast<std::uint32_t*>(smem + staged) +
                      static_cast<std::size_t>(slot) * stride;
  std::uint32_t* S1 = S0 + sw32;
  std::uint32_t* dbuf = S0 + 2 * sw32;  // 16-B aligned: 2*sw32 is a multiple of 4
  std::uint32_t* pa2buf = dbuf + kBuf;   // PA2: lane r's deferred patterns at [2r], [2r+1]
  std::uint32_t* planes = pa2buf + pa2w;  // node counts: plane i of word w at [8*w + i]
  {
    const std::uint32_t* src = reinterpret_cast<const std::uint32_t*>(states + tloc * (sw32 / 2));
    for (std::uint32_t w = r; w < sw32; w += LPT) S0[w] = src[w] & state_word_mask(h.n_kept, w);
    if (rp.node_counts)
      for (std::uint32_t w = r; w < sw32; w += LPT)
#pragma unroll
        for (int i = 0; i < 8; ++i) planes[8 * w + i] = 0;
  }
  __syncwarp(smask);

  // Per-node one-counts: each lane adds its state words to 8-plane bit-sliced
  // counters (carry-save, 3 ops per plane) and flushes them to the global u64
  // counts every 255 steps and at the end.
  std::uint32_t nc_pending = 0;
  auto nc_flush = [&]() {
    std::uint64_t* dst = rp.node_counts + tloc * h.n_kept;
    for (std::uint32_t w = r; w < sw32; w += LPT) {
      std::uint32_t pl[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        pl[i] = planes[8 * w + i];
        planes[8 * w + i] = 0;
      }
      for (std::uint32_t b = 0; b < 32; ++b) {
        const std::uint32_t node = 32 * w + b;
        if (node >= h.n_kept) break;
        std::uint32_t c = 0;
#pragma unroll
        for (int i = 0; i < 8; ++i) c |= ((pl[i] >> b) & 1u) << i;
        if (c) dst[node] += c;
      }
    }
    nc_pending = 0;
  };

  const std::uint32_t k = h.k, g = h.g;
  const bool exact_all = rp.exact_alias != 0;
  const std::uint32_t nb0 = (g + h.has_leaf + DPB - 1) / DPB;  // blocks of phase A
  const std::uint32_t A = h.n_alias_groups, NG = h.n_groups, A1 = h.n_single_alias;
  const std::uint32_t traj = static_cast<std::uint32_t>(rp.traj_begin + tloc);
  std::uint32_t thi0, tlo0;
  mulhilo(kPhiloxM0, traj, thi0, tlo0);
  // opaque to the compiler: kept in registers rather than rematerialised from
  // the block/thread ids (S2R + multiply) in every step
  asm volatile("" : "+r"(thi0), "+r"(tlo0));

  // Predicate (engine.hpp:328-332): lane r checks terms r, r+LPT, ...; the
  // sub-warp vote combines them. Called by every lane of the sub-warp.
  auto pred_eval = [&](const std::uint32_t* S) -> std::uint32_t {
    bool ok = true;
    if constexpr (LPT >= kMaxPredWords) {
      if (r < rp.pred.n) ok = (S[rp.pred.w[r]] & rp.pred.mask[r]) == rp.pred.want[r];
    } else {
      for (std::uint32_t i = r; i < rp.pred.n; i += LPT)
        ok = ok && (S[rp.pred.w[i]] & rp.pred.mask[i]) == rp.pred.want[i];
    }
    return rp.pred.n != 0 && __all_sync(smask, ok) ? 1u : 0u;
  };

  // the step's Philox constants (the redo path recomputes draws from them)
  step_philox sp{};
#ifdef PBN_SCRIPT_TU
  std::uint64_t script_row = 0;  // first block of the current step's draws
#endif
  // U53: a combined-function choice made on the draw's high word alone is
  // exact unless the draw sits on a cell boundary or ties the cut point
  // (about N+1 draws in 2^32, dev_plan.h acell) or the group/launch takes the
  // FP64 path. The hot loops only OR such events into `rare_acc`; a function
  // phase in which any lane saw one is recomputed exactly (redo_fn_phase).
  bool rare_acc = false;

  // Combined-function choice of alias group (engine.hpp:284-291) from draw jj
  // of the draw buffer (the draws' high words), fast form: U53 integer cells
  // (dev_plan.h a53), U32 integer cells (exact, never rare). Branch-free, so
  // the two groups of a round pair keep independent dependency chains.
  auto alias_fast = [&](const uint4* cells, std::uint32_t asz, std::uint32_t ab,
                        std::uint32_t jj, bool& rare) -> std::uint32_t {
    if constexpr (STREAM == STREAM_U53) {
      const std::uint32_t hi = dbuf[jj];  // the draw's high word: bits [21, 53) of r53
      const std::uint64_t P = static_cast<std::uint64_t>(hi) * asz;
      const std::uint32_t e = static_cast<std::uint32_t>(P >> 32);
      const uint2 V = ldp<GC>(reinterpret_cast<const uint2*>(cells + ab + e));  // {alias, hi32(C)}
      rare = rare || static_cast<std::uint32_t>(P) > ~asz || hi == V.y;
      return hi < V.y ? e : V.x;
    } else {
      // x*N < 2^53 is exact, so floor and fraction are the product's halves
      const std::uint64_t P = static_cast<std::uint64_t>(dbuf[jj]) * asz;
      const std::uint32_t c = static_cast<std::uint32_t>(P >> 32);
      const uint2 cell = ldp<GC>(reinterpret_cast<const uint2*>(cells + ab + c) + 1);  // {thr, alias}
      return static_cast<std::uint32_t>(P) < cell.x ? c : cell.y;
    }
  };
  auto alias_pick = [&](std::uint32_t asz, std::uint32_t ab, std::uint32_t jj,
                        bool exact) -> std::uint32_t {
    bool rare = exact;
    const std::uint32_t c = alias_fast(acell, asz, ab, jj, rare);  // ab relative to cell_base
    if constexpr (STREAM == STREAM_U53) rare_acc = rare_acc || rare;
    return c;
  };

  // Gathered parent valuation of combined function record F (engine.hpp:292-302).
  auto gather_fn = [&](const std::uint32_t* Sc, const uint4& F) -> std::uint32_t {
    const std::uint32_t gc = F.y & 31u;
    std::uint32_t v = gather4(Sc, F.z, F.w, 0);
    if (gc > 4) {
      const std::uint32_t xq = F.y >> 8;
#if PBN_GATHER_UNROLL
      // inputs 4..7 without the per-lane loop (up to 8 inputs: every
      // max_group_parents <= 8 plan); the loop only for wider functions
      const uint2 r4 = ldp<GC>(grec + xq);
      v |= gather4(Sc, r4.x, r4.y, 4);
      if (__builtin_expect(gc > 8, 0))
        for (std::uint32_t q = 8; q < gc; q += 4) {
          const uint2 rr = ldp<GC>(grec + xq + ((q - 4) >> 2));
          v |= gather4(Sc, rr.x, rr.y, q);
        }
#else
      for (std::uint32_t q = 4; q < gc; q += 4) {
        const uint2 rr = ldp<GC>(grec + xq + ((q - 4) >> 2));
        v |= gather4(Sc, rr.x, rr.y, q);
      }
#endif
    }
    return v;
  };

  // One group of the function phase (engine.hpp:281-310): combined-function
  // choice, gather of its own parents, table lookup. Returns the packed member
  // outputs; `off`/`members` describe where they go.
  // UNI (RG kernels): every lane of the warp evaluates a group (the plain
  // region's rounds, inactive lanes on a clamped index), so the parents can
  // come by shuffles; the extra-record loop runs to the warp's widest gather.
  std::uint32_t wreg_s = 0;  // RG: state word `lane` of the current state (set per function phase)
  std::uint32_t wreg1 = 0;   // RG2: state word `lane + 32`
  auto gather_fn_shfl = [&](const uint4& F) -> std::uint32_t {
    const std::uint32_t gc = F.y & 31u;
    std::uint32_t v = RG2 ? gather4_shfl2(wreg_s, wreg1, F.z, F.w, 0) : gather4_shfl(wreg_s, F.z, F.w, 0);
    const std::uint32_t gmax = __reduce_max_sync(smask, gc);
    const std::uint32_t xq = F.y >> 8;
    for (std::uint32_t q = 4; q < gmax; q += 4) {
      const bool has = q < gc;
      const uint2 rr = has ? ldp<GC>(grec + xq + ((q - 4) >> 2)) : make_uint2(F.z, F.w);
      const std::uint32_t t =
          RG2 ? gather4_shfl2(wreg_s, wreg1, rr.x, rr.y, q) : gather4_shfl(wreg_s, rr.x, rr.y, q);
      if (has) v |= t;
    }
    return v;
  };
  // Packed member outputs of combined function F at parent valuation v
  // (engine.hpp:303): inline table or an entry of 1/2/4/8 bytes.
  auto table_out = [&](const uint4& F, std::uint32_t v, std::uint32_t members, std::uint32_t& olo,
                       std::uint32_t& ohi) {
    ohi = 0;
    if (F.y & 0x80u) {  // inline table
      const std::uint32_t m = members >= 32 ? 0xFFFFFFFFu : ((1u << members) - 1u);
      olo = (F.x >> (v * members)) & m;
      return;
    }
    const std::uint32_t el2 = (F.y >> 5) & 3u;
    if (el2 == 0) {
      olo = ldp<GT>(tab + F.x + v);
    } else if (el2 == 1) {
      olo = ldp<GT>(reinterpret_cast<const std::uint16_t*>(tab + F.x) + v);
    } else if (el2 == 2) {
      olo = ldp<GT>(reinterpret_cast<const std::uint32_t*>(tab + F.x) + v);
    } else {
      const uint2 o = ldp<GT>(reinterpret_cast<const uint2*>(tab + F.x) + v);
      olo = o.x;
      ohi = o.y;
    }
  };
  // OR a group's packed outputs into the next state at bit `off` with shared
  // atomics (engine.hpp:304-309; up to 64 members span three words)
  auto emit_atomic = [&](std::uint32_t* Sn, std::uint32_t olo, std::uint32_t ohi, std::uint32_t off) {
    const std::uint32_t w = off >> 5, sh = off & 31;
    const std::uint32_t a0 = olo << sh;
    const std::uint32_t a1 = sh ? (olo >> (32 - sh)) | (ohi << sh) : ohi;
    const std::uint32_t a2 = sh ? (ohi >> (32 - sh)) : 0u;
    if (a0) atomicOr(Sn + w, a0);
    if (a1) atomicOr(Sn + w + 1, a1);
    if (a2) atomicOr(Sn + w + 2, a2);
  };
  auto eval_group = [&](const std::uint32_t* Sc, std::uint32_t gi, std::uint32_t jj,
                        std::uint32_t& olo, std::uint32_t& ohi, std::uint32_t& off,
                        std::uint32_t& members, auto uni_c) {
    constexpr bool UNI = decltype(uni_c)::value && RG && !RG2 && LPT == 32;
    const uint4 G = ldp<GC>(groups + gi);
    const std::uint32_t asz = G.w & 0x7FFFFFu;
    members = (G.w >> 24) + 1;
    off = G.x;
    const std::uint32_t idx =
        asz != 0 ? alias_pick(asz, G.z, jj, exact_all || (G.w & kGroupExactAlias)) : 0u;
    const uint4 F = ldp<GC>(fns + G.y + idx);
    std::uint32_t v;
    if constexpr (UNI)
      v = gather_fn_shfl(F);
    else
      v = gather_fn(Sc, F);
    table_out(F, v, members, olo, ohi);
  };

  // OR one round's outputs into the next state (engine.hpp:304-309). A round
  // of single-node groups covers consecutive bits: one ballot builds the word.
  auto emit_round = [&](std::uint32_t* Sn, bool act, std::uint32_t olo, std::uint32_t ohi,
                        std::uint32_t off, std::uint32_t members) {
    // lane r's group must sit at bit off0 + r (true for grouped plans; node-wise
    // plans put multi-function nodes first, so their offsets can jump)
    const std::uint32_t off0 = __shfl_sync(smask, off, (sub * LPT) & 31);
    const bool single = __all_sync(smask, !act || (members == 1 && off == off0 + r));
    if (single) {
      std::uint32_t bits = __ballot_sync(smask, act && (olo & 1u));
      if constexpr (LPT < 32) bits = (bits >> (sub * LPT)) & ((1u << (LPT & 31)) - 1u);
      if (r == 0 && bits) {
        const std::uint32_t w = off >> 5, sh = off & 31;
        atomicOr(Sn + w, bits << sh);
        if (sh && (bits >> (32 - sh))) atomicOr(Sn + w + 1, bits >> (32 - sh));
      }
    } else if (act) {
      emit_atomic(Sn, olo, ohi, off);
    }
  };

  // gather records of slots 4..7 pointing at the always-zero bit n'
  auto zrec = [&](std::uint32_t b) -> std::uint32_t {
    return ((h.n_kept >> 5) << 5) | (((h.n_kept & 31) - b) & 31);
  };
  const std::uint32_t zrec01 = zrec(4) | (zrec(5) << 16), zrec23 = zrec(6) | (zrec(7) << 16);

  // Single-node alias group j (offset j, inline 1-bit table): a handle of the
  // chosen function (rare: see alias_fast) — its index, or with the compact
  // records (SC) the byte offset of its scol function record — then its output bit;
  // loads and shuffles only, so two groups can be interleaved by the scheduler.
  auto single_fn = [&](std::uint32_t j, std::uint32_t jj, bool& rare) -> std::uint32_t {
    rare = false;
    if constexpr (SCL) {
      // sgrp cells (dev_plan.h): the choice on the high word's top 28 bits
      const uint4 R = lds128(sgrp + j);  // always staged (GM 4)
      const std::uint32_t hi = dbuf[jj];
      const std::uint32_t N = (R.x & 3u) + 1u;
      const std::uint64_t P = static_cast<std::uint64_t>(hi) * N;
      const std::uint32_t e = static_cast<std::uint32_t>(P >> 32);
      const std::uint32_t cell = e == 0 ? R.x : e == 1 ? R.y : e == 2 ? R.z : R.w;
      const std::uint32_t hT = hi >> 4, cT = cell >> 4;
      rare = static_cast<std::uint32_t>(P) > ~N || hT == cT;
      return 4 * j + (hT < cT ? e : (cell >> 2) & 3u);
    } else if constexpr (SC) {
      const uint4 ar = ldp<GC>(arec4 + j);  // {U53 cell offset, function offset, N, ~N}
      std::uint32_t pick;
      if constexpr (STREAM == STREAM_U53) {
        const std::uint32_t hi = dbuf[jj];
        const std::uint64_t P = static_cast<std::uint64_t>(hi) * ar.z;
        const std::uint32_t e = static_cast<std::uint32_t>(P >> 32);
        const uint2 V = ldp<GC>(reinterpret_cast<const uint2*>(core + ar.x + 8 * kScolSlots * e));
        rare = rare || static_cast<std::uint32_t>(P) > ar.w || hi == V.y;
        pick = hi < V.y ? e : V.x;
      } else {
        const std::uint64_t P = static_cast<std::uint64_t>(dbuf[jj]) * ar.z;
        const std::uint32_t c = static_cast<std::uint32_t>(P >> 32);
        const uint2 cell =
            ldp<GC>(reinterpret_cast<const uint2*>(core + ar.x + 8 * kScolSlots * (ar.z + c)));
        pick = static_cast<std::uint32_t>(P) < cell.x ? c : cell.y;
      }
      return ar.y + 8 * kScolSlots * pick;
    } else {
      const std::uint32_t ar = ldp<GC>(arec + j);
      const std::uint32_t base = ar & 0xFFFFFFu;
      // acell_s == acell unless the plan has the unstaged tail (then it is in
      // global memory and ldp<false> is a generic load): branch-free, so the
      // two groups of a round pair keep independent dependency chains
      return base + alias_fast(acell_s, ar >> 24, base, jj, rare);
    }
  };
  auto single_out = [&](const std::uint32_t* Sc, std::uint32_t wreg, std::uint32_t f) -> bool {
    if constexpr (SCL) {
      // five 16-bit records from the shared state (unused slots read bit n')
      const uint4 F = ldp<GC>(sfn + f);
      const std::uint32_t w4 = Sc[(F.w & 0xFFFFu) >> 5];
      const std::uint32_t v = gather4(Sc, F.y, F.z, 0) | (__funnelshift_r(w4, w4, F.w) & 16u);
      return (F.x >> v) & 1u;
    } else if constexpr (SC) {
      // compact record: 10-bit records (word << 5 | rotation), table at bits 16..31
      const uint2 F = ldp<GC>(reinterpret_cast<const uint2*>(core + f));
      const std::uint32_t w0 = __shfl_sync(0xFFFFFFFFu, wreg, F.x >> 5);
      const std::uint32_t w1 = __shfl_sync(0xFFFFFFFFu, wreg, F.x >> 15);
      const std::uint32_t w2 = __shfl_sync(0xFFFFFFFFu, wreg, F.x >> 25);
      const std::uint32_t w3 = __shfl_sync(0xFFFFFFFFu, wreg, F.y >> 5);
      const std::uint32_t v = 16u | (__funnelshift_r(w0, w0, F.x) & 1u) |
                              (__funnelshift_r(w1, w1, F.x >> 10) & 2u) |
                              (__funnelshift_r(w2, w2, F.x >> 20) & 4u) |
                              (__funnelshift_r(w3, w3, F.y) & 8u);
      return (F.y >> v) & 1u;
    } else {
      const uint4 F = ldp<GC>(fns_s + f);  // == fns + f unless the plan has the unstaged tail
      std::uint32_t v;
      if constexpr (RG2) {
        v = gather4_shfl2(wreg, wreg1, F.z, F.w, 0);
        if (h.single_gc5) {  // plan-uniform
          uint2 rr = make_uint2(zrec01, zrec23);
          if ((F.y & 31u) > 4) rr = ldp<GC>(grec + (F.y >> 8));
          v |= gather4_shfl2(wreg, wreg1, rr.x, rr.y, 4);
        }
      } else if constexpr (RG) {
        v = gather4_shfl(wreg, F.z, F.w, 0);
        if (h.single_gc5) {  // plan-uniform: every lane takes the same branch
          uint2 rr = make_uint2(zrec01, zrec23);
          if ((F.y & 31u) > 4) rr = ldp<GC>(grec + (F.y >> 8));
          v |= gather4_shfl(wreg, rr.x, rr.y, 4);
        }
      } else {
        v = gather_fn(Sc, F);
      }
      return (F.x >> v) & 1u;
    }
  };
  auto single_bit = [&](const std::uint32_t* Sc, std::uint32_t wreg, std::uint32_t j,
                        std::uint32_t jj) -> bool {
    bool rare;
    const std::uint32_t f = single_fn(j, jj, rare);
    if constexpr (STREAM == STREAM_U53) rare_acc = rare_acc || rare;
    return single_out(Sc, wreg, f);
  };
  // A single-node round's ballot word lands at bit jr of the next state.
  // full: all LPT groups of the round exist (a partial last round shares its
  // word with the next region and must OR atomically).
  auto store_bits = [&](std::uint32_t* Sn, std::uint32_t jr, std::uint32_t bits, bool full) {
    if constexpr (LPT < 32) bits = (bits >> (sub * LPT)) & ((1u << (LPT & 31)) - 1u);
    if (LPT == 32 && full) {
      if (r == 0) Sn[jr >> 5] = bits;  // jr is a multiple of 32: the word is this round's alone
    } else if (r == 0 && bits) {
      const std::uint32_t w = jr >> 5, sh = jr & 31;
      atomicOr(Sn + w, bits << sh);
      if (sh && (bits >> (32 - sh))) atomicOr(Sn + w + 1, bits >> (32 - sh));
    }
  };

  // Two single-node rounds (groups jr0 + r and jr0 + LPT + r, draws t*LPT + r
  // and (t+1)*LPT + r of the chunk): both rounds' loads are issued before
  // either ballot/store, so the two dependency chains overlap.
  auto single_pair = [&](const std::uint32_t* Sc, std::uint32_t* Sn, std::uint32_t wreg,
                         std::uint32_t jr0, std::uint32_t t) {
    const std::uint32_t jr1 = jr0 + LPT;
    bool rare0, rare1;
    const std::uint32_t f0 = single_fn(jr0 + r, t * LPT + r, rare0);
    const std::uint32_t f1 = single_fn(jr1 + r, (t + 1) * LPT + r, rare1);
    if constexpr (STREAM == STREAM_U53) rare_acc = rare_acc || rare0 || rare1;
    const bool b0 = single_out(Sc, wreg, f0);
    const bool b1 = single_out(Sc, wreg, f1);
    store_bits(Sn, jr0, __ballot_sync(smask, b0), true);
    store_bits(Sn, jr1, __ballot_sync(smask, b1), true);
  };

  // Four single-node rounds at once (U32 compact: a chunk of 4-draw blocks):
  // four independent chains.
  auto single_quad = [&](const std::uint32_t* Sc, std::uint32_t* Sn, std::uint32_t wreg,
                         std::uint32_t jr0, std::uint32_t t) {
    bool rr[4];
    std::uint32_t f[4];
#pragma unroll
    for (std::uint32_t u = 0; u < 4; ++u) f[u] = single_fn(jr0 + u * LPT + r, (t + u) * LPT + r, rr[u]);
    if constexpr (STREAM == STREAM_U53) rare_acc = rare_acc || rr[0] || rr[1] || rr[2] || rr[3];
    bool b[4];
#pragma unroll
    for (std::uint32_t u = 0; u < 4; ++u) b[u] = single_out(Sc, wreg, f[u]);
#pragma unroll
    for (std::uint32_t u = 0; u < 4; ++u) store_bits(Sn, jr0 + u * LPT, __ballot_sync(smask, b[u]), true);
  };

  // The exact choice of engine.hpp:285-290 in IEEE double without
  // contraction, from the full 53-bit draw r53 (U53).
  auto alias_fp64 = [&](std::uint32_t asz, std::uint32_t ab, std::uint64_t r53) -> std::uint32_t {
    const double u = __ull2double_rn(r53) * 0x1.0p-53;
    const double xx = __dmul_rn(u, __uint2double_rn(asz));
    std::uint32_t c = __double2uint_rz(xx);
    if (c >= asz) c = asz - 1;
    const double fr = __dsub_rn(xx, __uint2double_rn(c));
    return fr < __ldg(acut + ab + c) ? c : __ldg(aidx + ab + c);
  };
  // Exact recomputation of a function phase (engine.hpp:270-311) whose fast
  // pass saw a rare U53 choice (rare_acc; ~1e-6 of function phases on c2):
  // every combined-function draw rebuilt as its full 53 bits (high word from
  // block b, low word from block b | kLoBlock) and chosen in FP64; parents from
  // the shared-memory state; outputs ORed into the re-zeroed next state.
  auto redo_fn_phase = [&](const std::uint32_t* Scur, std::uint32_t* Snext) {
    for (std::uint32_t w = r; w < sw32; w += LPT) Snext[w] = 0;
    __syncwarp(smask);
    for (std::uint32_t gi = r; gi < NG; gi += LPT) {
      std::uint64_t r53 = 0;
      if (gi < A) {  // draw gi of phase B (alias groups come first)
        const std::uint32_t b = nb0 + gi / DPB, e = gi % DPB;
        const uint4 x = PBN_BLK(b);
        const uint4 y = PBN_BLK_LO_INLINE(b);
        r53 = ((static_cast<std::uint64_t>(pick32(x, e)) << 32) | pick32(y, e)) >> 11;
      }
      uint4 F;
      std::uint32_t off, members;
      if (gi < A1) {  // single node at offset gi (dev_plan.h arec; fns_s: absolute indices)
        const std::uint32_t ar = ldp<GC>(arec + gi);
        const std::uint32_t base = ar & 0xFFFFFFu;
        F = fns_s[base + alias_fp64(ar >> 24, base, r53)];
        off = gi;
        members = 1;
      } else {
        const uint4 G = ldp<GC>(groups + gi);
        const std::uint32_t asz = G.w & 0x7FFFFFu;
        members = (G.w >> 24) + 1;
        off = G.x;
        F = ldp<GC>(fns + G.y + (asz ? alias_fp64(asz, G.z + h.cell_base, r53) : 0u));
      }
      std::uint32_t olo, ohi;
      table_out(F, gather_fn(Scur, F), members, olo, ohi);
      emit_atomic(Snext, olo, ohi, off);
    }
    __syncwarp(smask);
  };

  // Phase-A masks of a block's draws (engine.hpp:257-268): full patterns for
  // groups before the last, the k'-bit mask for the last group (:261),
  // nothing for the leaf draw and past it; lane r's own first block's masks
  // are step-invariant and kept in registers.
  auto pa_mask = [&](std::uint32_t b, std::uint32_t e) -> std::uint32_t {
    const int q = static_cast<int>(g) - 1 - static_cast<int>(b * DPB + e);
    return q > 0 ? 0xFFFFFFFFu : (q == 0 ? h.last_mask : 0u);
  };
  auto lf_elem = [&](std::uint32_t b) -> std::uint32_t {  // the leaf draw's element (>= DPB: none)
    const int e = static_cast<int>(g) - static_cast<int>(b * DPB);
    return h.has_leaf && e >= 0 && e < static_cast<int>(DPB) ? static_cast<std::uint32_t>(e) : DPB;
  };
  static_assert(DPB == 4, "phase A masks are kept as a uint4");
  // Two steps per phase-A pass (PA2): the class of a step depends on the
  // stream alone, so when a step's phase A fills at most half the lanes
  // (k = 16, 2 * nb0 <= LPT; c2: 16 blocks) lanes 0..15 compute step s and
  // lanes 16..31 step s + 1 in one pass on even steps; each step then applies
  // its own half's patterns. Halves the phase-A Philox work per step.
  // (PA2 kernels — a template parameter, so that they carry no other phase-A
  // code: the hot path must stay inside the instruction cache — are the RG
  // instantiations the host launches when pa2_words() != 0.)
  static_assert(!PA2 || (LPT == 32 && !PF), "PA2 kernels: one trajectory per warp");
  constexpr bool pa2 = PA2;
  const std::uint32_t pa2_half = r / (LPT / 2 > 0 ? LPT / 2 : 1);
  const std::uint32_t rb = pa2 ? r % (LPT / 2 > 0 ? LPT / 2 : 1) : r;  // the lane's phase-A block
  const uint4 pam0 = make_uint4(pa_mask(rb, 0), pa_mask(rb, 1), pa_mask(rb, 2), pa_mask(rb, 3));
  const std::uint32_t lfe0 = lf_elem(rb);

  // Phase-A prefetch (kPaPrefetch): lane r < nb0 fetches step s's block r and
  // the high words (U32: the words) of its four perturbation cells.
  const bool pa_pf = PF && kPaPrefetch != 0 && h.pert_mode == 0 && k == 16 && nb0 <= LPT;
  uint4 pfx = make_uint4(0, 0, 0, 0), pfe = make_uint4(0, 0, 0, 0);
  auto pa_fetch = [&](std::uint64_t s) {
    const step_philox spn = make_step_philox(thi0, tlo0, s, rp.rk0, rp.rk1);
    pfx = philox_block(spn, r, rp.rk0, rp.rk1);
    auto cell = [&](std::uint32_t hw) -> std::uint32_t {
      if constexpr (STREAM == STREAM_U53)
        return pert53_hi_word<GP, false>(pfast, hw >> 16);
      else
        return ldp<GP>(reinterpret_cast<const std::uint32_t*>(pfast) + (hw >> 16));
    };
    pfe = make_uint4(cell(pfx.x), cell(pfx.y), cell(pfx.z), cell(pfx.w));
  };
  if constexpr (PF)
    if (pa_pf && r < nb0) pa_fetch(rp.step_begin);

  // PF kernels keep the state in registers between function phases: lane r
  // owns words 2r, 2r+1 — exactly its phase-A block's patterns at k = 16 — so
  // a perturbed step touches no shared memory; the rare function phase writes
  // them to S0, runs as usual into S1 and reads them back.
  uint2 sreg = make_uint2(0, 0);
  if constexpr (PF)
    if (2 * r < sw32) sreg = reinterpret_cast<const uint2*>(S0)[r];
  // predicate on the register state: the terms on a lane's two words merged
  // into one (mask, want) pair per word, fixed for the launch
  uint2 pmask = make_uint2(0, 0), pwant = make_uint2(0, 0);
  if constexpr (PF) {
    for (std::uint32_t i = 0; i < rp.pred.n; ++i) {
      const std::uint32_t w = rp.pred.w[i];
      if ((w >> 1) != r) continue;
      if (w & 1u) {
        pmask.y |= rp.pred.mask[i];
        pwant.y |= rp.pred.want[i];
      } else {
        pmask.x |= rp.pred.mask[i];
        pwant.x |= rp.pred.want[i];
      }
    }
  }
  auto pred_eval_reg = [&]() -> std::uint32_t {
    const bool ok = (((sreg.x & pmask.x) ^ pwant.x) | ((sreg.y & pmask.y) ^ pwant.y)) == 0;
    return rp.pred.n != 0 && __all_sync(smask, ok) ? 1u : 0u;
  };

  std::uint32_t pa2_cls = 0;  // PA2: the classes of the pass's two steps
  step_philox spa{};          // PA2: the lane's own step's stream constants in phase A
  std::uint32_t cur = 0;
  const std::uint32_t z0 = pred_eval(S0);
  std::uint32_t prev = 2u, kphase = 0;  // previous sample (2 = none), steps since it
  if (rp.thin_mode == 0) prev = z0;
  if (rp.thin_mode == 1 && rp.tprev) {
    const std::uint32_t tp = rp.tprev[tloc];
    prev = tp & 3u;
    kphase = tp >> 2;
  }
  // sampled transitions as four sums over samples with a previous sample:
  // nv samples, np1 with prev = 1, nh1 with hit = 1, n11 with both
  // (n10 = np1 - n11, n01 = nh1 - n11, n00 = nv - np1 - nh1 + n11)
  // The counters are warp-uniform: with LPT >= 8 lane r of the sub-warp
  // keeps counter r (0 hits, 1 nv, 2 np1, 3 nh1, 4 n11, 5 function-phase
  // steps, 6 perturbed steps) in one register `cnt`; each step ORs its events
  // into a bit word and every lane adds its own bit (registers the hot loops
  // need instead of seven loop-carried counters).
  constexpr bool LANE_COUNTERS = LPT >= 8;
  std::uint32_t cnt = 0;
  std::uint32_t nv = 0, np1 = 0, nh1 = 0, n11 = 0, nhit = 0, nfn = 0, npert = 0;
  // (the series row is recomputed where used: a pointer kept live across the
  // step loop costs registers the hot loops need)
  std::uint32_t sword = 0;   // series bits of the current word (lane r == 0)
  if (rp.series != nullptr && r == 0 && rp.series_init && rp.series_bit0 > 0 && z0) {
    std::uint32_t* ser = rp.series + tloc * rp.series_stride;
    const std::uint64_t p0 = rp.series_bit0 - 1;
    ser[p0 >> 5] |= 1u << (p0 & 31);
  }
  const std::uint64_t s_end = rp.step_begin + rp.n_steps;

  for (std::uint64_t s = rp.step_begin; s < s_end; ++s) {
    std::uint32_t* Sc = cur ? S1 : S0;
#ifdef PBN_SCRIPT_TU
    script_row = (tloc * rp.n_steps + (s - rp.step_begin)) * rp.script_bps;
#else
    sp = make_step_philox(thi0, tlo0, s, rp.rk0, rp.rk1);
#endif

    // ---- phase A: grouped perturbation + leaf draw (draws 0..g). Every draw
    // of a block is looked up; a per-draw mask keeps full patterns for draws
    // before the last group, the k'-bit mask for the last group (engine.hpp:
    // 261) and nothing for the leaf draw and the block's unused tail.
    bool flip = false, leaf = false;
    // One Philox block of phase A: draws b*DPB .. b*DPB+DPB-1, each looked up
    // and masked (pam: full patterns before the last group, the k'-bit mask
    // for the last group (engine.hpp:261), nothing for the leaf draw and the
    // block's unused tail); `lfe` is the leaf draw's element (>= DPB: none).
    // U53: decided on the draws' high words; a tie recomputes the block's
    // decisions with the low words (one more Philox block, ~2^-14 of blocks
    // at k = 16). WPB (k * DPB = 32 or 64: k = 8 or 16) — the block's patterns
    // fill exactly state words b*WPB.., which no other lane touches: they are
    // XOR-ed in with plain read-modify-writes; otherwise per-draw atomics.
    auto phase_a_block = [&](std::uint32_t b, const uint4 pam, std::uint32_t lfe,
                             auto bern_c, auto wpb_c, auto defer_c) {
      constexpr bool BERN = decltype(bern_c)::value;  // Method_old / Method_reduction plans
      constexpr std::uint32_t WPB = decltype(wpb_c)::value;
      constexpr bool DEFER = decltype(defer_c)::value;  // PA2: keep the patterns, apply per step
#ifdef PBN_SCRIPT_TU
      const uint4 x = PBN_BLK(b);
#else
      // PA2: the lane's own step's stream (spa: s or s + 1), else the step's
      uint4 x;
      if constexpr (DEFER)
        x = philox_block(spa, b, rp.rk0, rp.rk1);
      else
        x = PBN_BLK(b);
#endif
      std::uint32_t c[DPB];
      bool rare = false, lf = false;
#pragma unroll
      for (std::uint32_t e = 0; e < DPB; ++e)
        c[e] = pa_draw<STREAM, GP, BERN>(h, gblob, pfast, k, pick32(x, e), false, 0u, rare);
      if (lfe < DPB) lf = pa_leaf<STREAM>(h, pick32(x, lfe), false, 0u, rare);
      if constexpr (STREAM == STREAM_U53) {
        if (__builtin_expect(rare, 0)) {
#ifdef PBN_SCRIPT_TU
          const uint4 y = PBN_BLK_LO(b);
#else
          uint4 y;
          if constexpr (DEFER)
            y = philox_lo_block(spa, b, rp.rk0, rp.rk1);
          else
            y = PBN_BLK_LO(b);
#endif
          bool unused = false;
#pragma unroll
          for (std::uint32_t e = 0; e < DPB; ++e)
            c[e] = pa_draw<STREAM, GP, BERN>(h, gblob, pfast, k, pick32(x, e), true, pick32(y, e), unused);
          if (lfe < DPB) lf = pa_leaf<STREAM>(h, pick32(x, lfe), true, pick32(y, lfe), unused);
        }
      }
      if constexpr (DEFER) {
        static_assert(WPB == 2, "PA2 is the k = 16 word path");
        const std::uint32_t w0 = (c[0] & pam.x) | ((c[1] & pam.y) << 16);
        const std::uint32_t w1 = (c[2] & pam.z) | ((c[3] & pam.w) << 16);
        reinterpret_cast<uint2*>(pa2buf)[r] = make_uint2(w0, w1);  // read back by this lane only
        flip = (w0 | w1) != 0;
        leaf = lf;
        return;
      }
      leaf = leaf || lf;
      if constexpr (WPB == 2) {  // k = 16: elements 0,1 -> word 2b, elements 2,3 -> word 2b+1
        const std::uint32_t w0 = (c[0] & pam.x) | ((c[1] & pam.y) << 16);
        const std::uint32_t w1 = (c[2] & pam.z) | ((c[3] & pam.w) << 16);
        if (__builtin_expect((w0 | w1) != 0, 0)) {  // xor_chunk (bitstate.hpp:50-58)
          flip = true;
          // one 8-byte read-modify-write (words 2b, 2b+1: consecutive lanes
          // hit consecutive bank pairs; two 4-byte accesses would conflict)
          uint2* w = reinterpret_cast<uint2*>(Sc) + b;
          uint2 v = *w;
          v.x ^= w0;
          v.y ^= w1;
          *w = v;
        }
      } else if constexpr (WPB == 1) {  // k = 8: the block's four patterns are word b
        const std::uint32_t w0 = (c[0] & pam.x) | ((c[1] & pam.y) << 8) |
                                 ((c[2] & pam.z) << 16) | ((c[3] & pam.w) << 24);
        if (__builtin_expect(w0 != 0, 0)) {
          flip = true;
          Sc[b] ^= w0;
        }
      } else {
#pragma unroll
        for (std::uint32_t e = 0; e < DPB; ++e) {
          const std::uint32_t ce = c[e] & pick32(pam, e);
          if (__builtin_expect(ce != 0, 0)) {  // xor_chunk (bitstate.hpp:50-58)
            flip = true;
            const std::uint32_t o = (b * DPB + e) * k, w = o >> 5, sh = o & 31;
            atomicXor(Sc + w, ce << sh);
            if (sh != 0 && (ce >> (32 - sh)) != 0) atomicXor(Sc + w + 1, ce >> (32 - sh));
          }
        }
      }
    };
    // The same block from the prefetched words (k = 16, block r): pattern
    // c = draw's top 16 bits unless its next 16 bits reach the cell's
    // threshold bits (then the cell's alias), kernel_common.cuh pert_draw53_hi
    // / pert_draw32; a U53 tie on those bits redoes the block exactly.
    auto phase_a_prefetched = [&]() {
      const uint4 x = pfx, ce = pfe;
      std::uint32_t c[DPB];
      bool rare = false, lf = false;
#pragma unroll
      for (std::uint32_t e = 0; e < DPB; ++e) {
        const std::uint32_t hw = pick32(x, e), cw = pick32(ce, e);
        const std::uint32_t a = hw & 0xFFFFu, b = cw & 0xFFFFu;
        if constexpr (STREAM == STREAM_U53) rare = rare || a == b;
        c[e] = a < b ? (hw >> 16) : (cw >> 16);
      }
      if (lfe0 < DPB) lf = pa_leaf<STREAM>(h, pick32(x, lfe0), false, 0u, rare);
      if constexpr (STREAM == STREAM_U53) {
        if (__builtin_expect(rare, 0)) {
          const uint4 y = PBN_BLK_LO(r);
          bool unused = false;
#pragma unroll
          for (std::uint32_t e = 0; e < DPB; ++e)
            c[e] = pa_draw<STREAM, GP, false>(h, gblob, pfast, k, pick32(x, e), true, pick32(y, e), unused);
          if (lfe0 < DPB) lf = pa_leaf<STREAM>(h, pick32(x, lfe0), true, pick32(y, lfe0), unused);
        }
      }
      leaf = leaf || lf;
      const std::uint32_t w0 = (c[0] & pam0.x) | ((c[1] & pam0.y) << 16);
      const std::uint32_t w1 = (c[2] & pam0.z) | ((c[3] & pam0.w) << 16);
      flip = (w0 | w1) != 0;  // xor_chunk (bitstate.hpp:50-58) on the register state
      sreg.x ^= w0;
      sreg.y ^= w1;
    };
    auto phase_a = [&](auto bern_c, auto wpb_c) {
      if (nb0 <= LPT) {  // launch-uniform: at most one block per lane (masks precomputed)
        if (r < nb0) phase_a_block(r, pam0, lfe0, bern_c, wpb_c, std::false_type{});
      } else {
        for (std::uint32_t b = r; b < nb0; b += LPT)
          phase_a_block(b, make_uint4(pa_mask(b, 0), pa_mask(b, 1), pa_mask(b, 2), pa_mask(b, 3)),
                        lf_elem(b), bern_c, wpb_c, std::false_type{});
      }
    };
    bool any_flip, any_leaf;
    if constexpr (PA2) {
      const std::uint32_t j = static_cast<std::uint32_t>(s - rp.step_begin) & 1u;
      if (j == 0) {  // both steps' blocks: lanes 0..15 step s, lanes 16..31 step s + 1
        spa = make_step_philox(thi0, tlo0, s + pa2_half, rp.rk0, rp.rk1);
        if (rb < nb0)
          phase_a_block(rb, pam0, lfe0, std::false_type{}, std::integral_constant<std::uint32_t, 2>{},
                        std::true_type{});
        // the two steps' classes: bit j = step s + j has a kept flip, bit 2 + j = its leaf fired
        const std::uint32_t fm = __ballot_sync(smask, flip), lm = __ballot_sync(smask, leaf);
        pa2_cls = ((fm & 0xFFFFu) ? 1u : 0u) | ((fm >> 16) ? 2u : 0u) | ((lm & 0xFFFFu) ? 4u : 0u) |
                  ((lm >> 16) ? 8u : 0u);
      }
      any_flip = ((pa2_cls >> j) & 1u) != 0;
      any_leaf = ((pa2_cls >> (2 + j)) & 1u) != 0;
      if (any_flip && pa2_half == j && rb < nb0) {
        const uint2 pw = reinterpret_cast<const uint2*>(pa2buf)[r];
        if ((pw.x | pw.y) != 0) {  // xor_chunk (bitstate.hpp:50-58)
          uint2* w = reinterpret_cast<uint2*>(Sc) + rb;
          uint2 v = *w;
          v.x ^= pw.x;
          v.y ^= pw.y;
          *w = v;
        }
      }
    } else {
      if (PF && pa_pf) {  // launch-uniform
        if (r < nb0) {
          phase_a_prefetched();
          if constexpr (kPaPrefetch == 1) pa_fetch(s + 1);
        }
      } else if (h.pert_mode != 0)  // plan-uniform
        phase_a(std::true_type{}, std::integral_constant<std::uint32_t, 0>{});
      else if (k == 16)
        phase_a(std::false_type{}, std::integral_constant<std::uint32_t, 2>{});
      else if (k == 8)
        phase_a(std::false_type{}, std::integral_constant<std::uint32_t, 1>{});
      else
        phase_a(std::false_type{}, std::integral_constant<std::uint32_t, 0>{});
      any_flip = __ballot_sync(smask, flip) != 0;
      any_leaf = __ballot_sync(smask, leaf) != 0;
    }

    std::uint32_t ev = 0;  // this step's events (LANE_COUNTERS bit layout)
    if (any_flip) {
      if constexpr (!PF) __syncwarp(smask);
      if constexpr (LANE_COUNTERS)
        ev = 1u << 6;
      else
        ++npert;
    } else if (!any_leaf) {
      if constexpr (PF) {
        // ---- function phase of a perturbation-dominated launch (fewer than
        // kPertDominated of the steps): the generic exact evaluation — every
        // draw rebuilt as 53 bits, FP64 choices, parents from shared memory —
        // between a store and a reload of the register state
        if (2 * r < sw32) reinterpret_cast<uint2*>(S0)[r] = sreg;
        redo_fn_phase(S0, S1);  // zeroes S1 and synchronises before and after
        if (2 * r < sw32) sreg = reinterpret_cast<const uint2*>(S1)[r];
        __syncwarp(smask);
      } else {
      // ---- function phase, in lockstep rounds of LPT groups
      std::uint32_t* Sn = cur ? S0 : S1;
      for (std::uint32_t w = r; w < sw32; w += LPT) Sn[w] = 0;
      // the zeroing must be visible to the other lanes' ORs (shuffles and
      // votes do not order shared memory; a plan without alias groups goes
      // straight to the plain region's atomics)
      __syncwarp(smask);
      rare_acc = exact_all;
      std::uint32_t wreg = 0;  // RG: state word `lane` of the current state
      if constexpr (RG) wreg = lane < sw32 ? Sc[lane] : 0u;
      wreg_s = wreg;
      if constexpr (RG2) wreg1 = lane + 32 < sw32 ? Sc[lane + 32] : 0u;
      // alias region: chunks of LPT*DPB draws; lane r first computes phase-B
      // block nb0 + j0/DPB + r into the draw buffer
      // lane r computes blocks q*LPT + r of each chunk (independent chains)
      uint4 xb[CB];
      if constexpr (kPhiloxPipeline) {
#pragma unroll
        for (std::uint32_t q = 0; q < CB; ++q)
          xb[q] = PBN_BLK(nb0 + q * LPT + r);
      }
      std::uint32_t jstart = 0;
      if constexpr (SC && DPB * CB == 2 && !kPhiloxPipeline) {
        // chunks made of one single-node round pair (U53 compact): no round
        // bookkeeping; the general loop below takes the remaining chunks
        const std::uint32_t jfull = A1 & ~(2u * LPT - 1u);
        for (std::uint32_t j0 = 0; j0 < jfull; j0 += 2 * LPT) {
          const uint4 x = PBN_BLK(nb0 + j0 / DPB + r);
          *reinterpret_cast<uint4*>(dbuf + 4 * r) = x;
          __syncwarp(smask);
          single_pair(Sc, Sn, wreg, j0, 0);
          __syncwarp(smask);
        }
        jstart = jfull;
      } else if constexpr ((SC || SCL) && DPB * CB == 4 && kQuadRounds && !kPhiloxPipeline) {
        // U32 compact: chunks of one single-node quad
        const std::uint32_t jfull = A1 & ~(4u * LPT - 1u);
        for (std::uint32_t j0 = 0; j0 < jfull; j0 += 4 * LPT) {
          *reinterpret_cast<uint4*>(dbuf + 4 * r) = PBN_BLK(nb0 + j0 / DPB + r);
          __syncwarp(smask);
          single_quad(Sc, Sn, wreg, j0, 0);
          __syncwarp(smask);
        }
        jstart = jfull;
      }
      for (std::uint32_t j0 = jstart; j0 < A; j0 += LPT * DPB * CB) {
        if constexpr (!kPhiloxPipeline) {
#pragma unroll
          for (std::uint32_t q = 0; q < CB; ++q)
            xb[q] = PBN_BLK(nb0 + j0 / DPB + q * LPT + r);
        }
#pragma unroll
        for (std::uint32_t q = 0; q < CB; ++q)
          // (blocks past the region's last draw are stored too: never read)
          *reinterpret_cast<uint4*>(dbuf + 4 * (q * LPT + r)) = xb[q];
        __syncwarp(smask);
        if constexpr (kPhiloxPipeline) {  // next chunk's blocks (unused after the last)
#pragma unroll
          for (std::uint32_t q = 0; q < CB; ++q)
            xb[q] = PBN_BLK(nb0 + (j0 / DPB) + (CB + q) * LPT + r);
        }
        // rounds are taken in pairs: both rounds' loads are issued before
        // either ballot/store, so the two dependency chains overlap
#pragma unroll
        for (std::uint32_t t = 0; t < DPB * CB; t += 2) {
          const std::uint32_t jr0 = j0 + t * LPT, jr1 = jr0 + LPT;
          if (jr0 >= A) break;
          if constexpr (kQuadRounds && (SC || SCL) && DPB * CB >= 4) {
            // four single-node rounds at once: four independent chains
            if ((t & 3) == 0 && jr0 + 4 * LPT <= A1) {
              single_quad(Sc, Sn, wreg, jr0, t);
              t += 2;  // with the loop's += 2: next quad
              continue;
            }
          }
          if (jr1 + LPT <= A1) {
            single_pair(Sc, Sn, wreg, jr0, t);
            continue;
          }
          // two general rounds: both groups' loads before either emit (not in
          // the compact-record variant, whose register budget it would raise)
          if (kGeneralPairs && !SC && jr0 >= A1) {
            const std::uint32_t j0 = jr0 + r, j1 = jr1 + r;
            const bool a0 = j0 < A, a1 = j1 < A;
            std::uint32_t lo0 = 0, hi0 = 0, off0 = 0, m0 = 1, lo1 = 0, hi1 = 0, off1 = 0, m1 = 1;
            if constexpr (RG && !RG2 && LPT == 32 && kPlainShfl) {  // uniform, shuffle gathers
              eval_group(Sc, a0 ? j0 : A - 1, t * LPT + r, lo0, hi0, off0, m0, std::true_type{});
              eval_group(Sc, a1 ? j1 : A - 1, (t + 1) * LPT + r, lo1, hi1, off1, m1, std::true_type{});
            } else {
              if (a0) eval_group(Sc, j0, t * LPT + r, lo0, hi0, off0, m0, std::false_type{});
              if (a1) eval_group(Sc, j1, (t + 1) * LPT + r, lo1, hi1, off1, m1, std::false_type{});
            }
            emit_round(Sn, a0, lo0, hi0, off0, m0);
            if (jr1 < A) emit_round(Sn, a1, lo1, hi1, off1, m1);
            continue;
          }
#pragma unroll
          for (std::uint32_t u = 0; u < 2; ++u) {
            const std::uint32_t jr = jr0 + u * LPT;
            if (jr >= A) break;
            const std::uint32_t j = jr + r;
            if (jr + LPT <= A1) {
              store_bits(Sn, jr, __ballot_sync(smask, single_bit(Sc, wreg, j, (t + u) * LPT + r)),
                         true);
            } else if (A1 == A) {
              // partial last round of an all-single-node alias region: lanes
              // past the region evaluate a valid group and drop the bit
              const bool b = single_bit(Sc, wreg, j < A ? j : A - 1, (t + u) * LPT + r);
              store_bits(Sn, jr, __ballot_sync(smask, j < A && b), false);
            } else {
              const bool act = j < A;
              std::uint32_t olo = 0, ohi = 0, off = 0, members = 1;
              if constexpr (RG && !RG2 && LPT == 32 && kPlainShfl)
                eval_group(Sc, act ? j : A - 1, (t + u) * LPT + r, olo, ohi, off, members, std::true_type{});
              else if (act)
                eval_group(Sc, j, (t + u) * LPT + r, olo, ohi, off, members, std::false_type{});
              emit_round(Sn, act, olo, ohi, off, members);
            }
          }
        }
        __syncwarp(smask);
      }
      // plain region (one combined function per group, no draw), rounds in
      // pairs: both rounds' loads before either round's atomics
      for (std::uint32_t gr = A; gr < NG; gr += 2 * LPT) {
        const std::uint32_t g0 = gr + r, g1 = gr + LPT + r;
        const bool a0 = g0 < NG, a1 = g1 < NG;
        std::uint32_t lo0 = 0, hi0 = 0, off0 = 0, m0 = 1, lo1 = 0, hi1 = 0, off1 = 0, m1 = 1;
        if constexpr (RG && !RG2 && LPT == 32 && kPlainShfl) {  // every lane evaluates (clamped), shuffles
          eval_group(Sc, a0 ? g0 : NG - 1, 0, lo0, hi0, off0, m0, std::true_type{});
          eval_group(Sc, a1 ? g1 : NG - 1, 0, lo1, hi1, off1, m1, std::true_type{});
        } else {
          if (a0) eval_group(Sc, g0, 0, lo0, hi0, off0, m0, std::false_type{});
          if (a1) eval_group(Sc, g1, 0, lo1, hi1, off1, m1, std::false_type{});
        }
        emit_round(Sn, a0, lo0, hi0, off0, m0);
        if (gr + LPT < NG) emit_round(Sn, a1, lo1, hi1, off1, m1);
      }
      __syncwarp(smask);
      if constexpr (STREAM == STREAM_U53)
        if (__builtin_expect(__any_sync(smask, rare_acc), 0)) redo_fn_phase(Sc, Sn);
      cur ^= 1;
      }  // !PF
      if constexpr (LANE_COUNTERS)
        ev = 1u << 5;
      else
        ++nfn;
    }

    if constexpr (PF && kPaPrefetch == 2)
      if (pa_pf && r < nb0) pa_fetch(s + 1);

    // ---- statistics (engine.hpp:375-381) + sampled predicate transitions
    const std::uint32_t hit = PF && pa_pf ? pred_eval_reg() : pred_eval(cur ? S1 : S0);
    if constexpr (LANE_COUNTERS) {
      ev |= hit;
      if (++kphase == rp.kappa) {
        kphase = 0;
        const std::uint32_t valid = (prev >> 1) ^ 1u;  // prev 2 = none
        ev |= (valid << 1) | ((prev & 1u) << 2) | ((hit & valid) << 3) | ((prev & hit) << 4);
        prev = hit;
      }
      cnt += (ev >> r) & 1u;
    } else {
      nhit += hit;
      if (++kphase == rp.kappa) {
        kphase = 0;
        const std::uint32_t valid = (prev >> 1) ^ 1u;  // prev 2 = none
        nv += valid;
        np1 += prev & 1u;
        nh1 += hit & valid;
        n11 += prev & hit;
        prev = hit;
      }
    }
    if (rp.node_counts) {  // launch-uniform branch
      const std::uint32_t* Sf = cur ? S1 : S0;
      for (std::uint32_t w = r; w < sw32; w += LPT) {
        std::uint32_t x = Sf[w];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const std::uint32_t p = planes[8 * w + i];
          planes[8 * w + i] = p ^ x;
          x &= p;
        }
      }
      if (++nc_pending == 255) nc_flush();
    }
    if (rp.series != nullptr && r == 0) {  // launch-uniform test, then lane 0
      std::uint32_t* ser = rp.series + tloc * rp.series_stride;
      const std::uint64_t pos = rp.series_bit0 + (s - rp.step_begin);
      sword |= hit << (pos & 31);
      if ((pos & 31) == 31 || s + 1 == s_end) {
        if (sword) ser[pos >> 5] |= sword;
        sword = 0;
      }
    }
    __syncwarp(smask);
  }
  if (rp.tprev && r == 0) rp.tprev[tloc] = static_cast<std::uint8_t>(prev | (kphase << 2));
  if (rp.node_counts && nc_pending) nc_flush();

  {
    const std::uint32_t* Sf = cur ? S1 : S0;
    std::uint32_t* dst = reinterpret_cast<std::uint32_t*>(states + tloc * (sw32 / 2));
    if (PF && pa_pf) {
      if (2 * r < sw32) reinterpret_cast<uint2*>(dst)[r] = sreg;
    } else {
      for (std::uint32_t w = r; w < sw32; w += LPT) dst[w] = Sf[w];
    }
  }
  if constexpr (LANE_COUNTERS) {
    const std::uint32_t l0 = (sub * LPT) & 31;
    nhit = __shfl_sync(smask, cnt, l0 + 0);
    nv = __shfl_sync(smask, cnt, l0 + 1);
    np1 = __shfl_sync(smask, cnt, l0 + 2);
    nh1 = __shfl_sync(smask, cnt, l0 + 3);
    n11 = __shfl_sync(smask, cnt, l0 + 4);
    nfn = __shfl_sync(smask, cnt, l0 + 5);
    npert = __shfl_sync(smask, cnt, l0 + 6);
  }
  if (r == 0) {
    std::uint64_t* c = counts + tloc * 8;
    const bool pr = rp.pred.n != 0;
    c[0] = rp.n_steps;
    c[1] = pr ? nhit : 0;
    c[2] = pr ? nv - np1 - nh1 + n11 : 0;
    c[3] = pr ? nh1 - n11 : 0;
    c[4] = pr ? np1 - n11 : 0;
    c[5] = pr ? n11 : 0;
    c[6] = nfn;
    c[7] = npert;
  }
}

#ifndef PBN_SCRIPT_TU
// Pooled statistics of stored predicate series (estimator pilot): per
// trajectory row, triple counts n_ijk at period kappa (t = 2k, 3k, ...), thinned
// pair counts (t = k, 2k, ...) and ones in [1, len); summed over trajectories.
__global__ void pbn_series_stats_kernel(const std::uint32_t* __restrict__ series,
                                        std::uint32_t n_traj, std::uint64_t stride,
                                        std::uint64_t len, std::uint32_t kappa,
                                        unsigned long long* __restrict__ out) {
  const std::uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long c[13];
#pragma unroll
  for (int i = 0; i < 13; ++i) c[i] = 0;
  if (t < n_traj) {
    const std::uint32_t* row = series + t * stride;
    auto z = [&](std::uint64_t i) -> std::uint32_t { return (__ldg(row + (i >> 5)) >> (i & 31)) & 1u; };
    for (std::uint64_t i = 2ull * kappa; i < len; i += kappa) {
      const std::uint32_t idx = (z(i - 2 * kappa) << 2) | (z(i - kappa) << 1) | z(i);
#pragma unroll
      for (std::uint32_t q = 0; q < 8; ++q) c[q] += idx == q;
    }
    for (std::uint64_t i = kappa; i < len; i += kappa) {
      const std::uint32_t idx = (z(i - kappa) << 1) | z(i);
#pragma unroll
      for (std::uint32_t q = 0; q < 4; ++q) c[8 + q] += idx == q;
    }
    for (std::uint64_t w = 0; w * 32 < len; ++w) {
      std::uint32_t word = __ldg(row + w);
      if (w == 0) word &= ~1u;  // position 0 is the initial state
      const std::uint64_t end = len - w * 32;
      if (end < 32) word &= (1u << end) - 1u;
      c[12] += __popc(word);
    }
  }
#pragma unroll
  for (int i = 0; i < 13; ++i) {
    unsigned long long v = c[i];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xFFFFFFFFu, v, o);
    if ((threadIdx.x & 31) == 0 && v) atomicAdd(out + i, v);
  }
}

// Sum of per-trajectory count records (n x 8) into out[8].
__global__ void pbn_sum_counts_kernel(const std::uint64_t* __restrict__ counts, std::uint32_t n,
                                      unsigned long long* __restrict__ out) {
  const std::uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
#pragma unroll
  for (int f = 0; f < 8; ++f) {
    unsigned long long v = t < n ? counts[static_cast<std::uint64_t>(t) * 8 + f] : 0ull;
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xFFFFFFFFu, v, o);
    if ((threadIdx.x & 31) == 0 && v) atomicAdd(out + f, v);
  }
}

cudaError_t launch_series_stats(const std::uint32_t* d_series, std::uint32_t n_traj,
                                std::uint64_t stride, std::uint64_t len, std::uint32_t kappa,
                                unsigned long long* d_out13, cudaStream_t stream) {
  cudaError_t e = cudaMemsetAsync(d_out13, 0, 13 * sizeof(unsigned long long), stream);
  if (e != cudaSuccess) return e;
  pbn_series_stats_kernel<<<(n_traj + 255) / 256, 256, 0, stream>>>(d_series, n_traj, stride, len,
                                                                    kappa, d_out13);
  return cudaGetLastError();
}

cudaError_t launch_sum_counts(const std::uint64_t* d_counts, std::uint32_t n,
                              unsigned long long* d_out8, cudaStream_t stream) {
  cudaError_t e = cudaMemsetAsync(d_out8, 0, 8 * sizeof(unsigned long long), stream);
  if (e != cudaSuccess) return e;
  pbn_sum_counts_kernel<<<(n + 255) / 256, 256, 0, stream>>>(d_counts, n, d_out8);
  return cudaGetLastError();
}

// Known-answer kernel for the stream: out[i] = Philox4x32-10(ctr[i], key).
__global__ void pbn_philox_kat_kernel(const uint4* ctr, std::uint32_t k0, std::uint32_t k1,
                                      uint4* out, std::uint32_t n) {
  const std::uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = philox4x32_10(ctr[i], k0, k1);
}

// ----------------------------------------------------------------------------
// Host-side launch helpers (called from capi.cpp).

using kernel_fn = void (*)(const dev_plan_header, const std::uint8_t*, const dev_run_params,
                           std::uint64_t*, std::uint64_t*);

template <int LPT, int STREAM, int GM, bool PA2 = false>
kernel_fn pick_place(int place) {
  switch (place) {
    case PLACE_ALL:
      return pbn_ensemble_kernel<LPT, STREAM, PLACE_ALL, GM, false, PA2>;
    case PLACE_CORE_PERT:
      return pbn_ensemble_kernel<LPT, STREAM, PLACE_CORE_PERT, GM, false, PA2>;
    case PLACE_TABLES:
      return pbn_ensemble_kernel<LPT, STREAM, PLACE_TABLES, GM, false, PA2>;
    case PLACE_CORE:
      return pbn_ensemble_kernel<LPT, STREAM, PLACE_CORE, GM, false, PA2>;
    default:
      return pbn_ensemble_kernel<LPT, STREAM, PLACE_GLOBAL, GM, false, PA2>;
  }
}

template <int STREAM>
kernel_fn pick_lpt(std::uint32_t lpt, int place, int gm, bool pa2) {
  switch (lpt) {
    case 1:
      return pick_place<1, STREAM, 0>(place);
    case 2:
      return pick_place<2, STREAM, 0>(place);
    case 4:
      return pick_place<4, STREAM, 0>(place);
    case 8:
      return pick_place<8, STREAM, 0>(place);
    case 16:
      return pick_place<16, STREAM, 0>(place);
    default:
      if constexpr (STREAM == STREAM_U53)
        if (gm == 4) return pick_place<32, STREAM, 4>(place);
      if (pa2 && gm == 2) return pick_place<32, STREAM, 2, true>(place);
      if (pa2 && gm == 1) return pick_place<32, STREAM, 1, true>(place);
      return gm == 3   ? pick_place<32, STREAM, 3>(place)
             : gm == 2 ? pick_place<32, STREAM, 2>(place)
             : gm == 1 ? pick_place<32, STREAM, 1>(place)
                       : pick_place<32, STREAM, 0>(place);
  }
}

kernel_fn select_kernel(std::uint32_t lpt, int stream, int place, int gm, bool pert_dom, bool pa2) {
#ifdef PBN_FAST_BUILD  // register-allocation experiments: the headline instantiations only
  if (pert_dom) return pbn_ensemble_kernel<32, STREAM_U53, PLACE_GLOBAL, 0, true>;
  if (gm == 4) return pbn_ensemble_kernel<32, STREAM_U53, PLACE_GLOBAL, 4>;
  if (gm == 0) return pbn_ensemble_kernel<32, STREAM_U53, PLACE_CORE, 0>;
  if (pa2) return pbn_ensemble_kernel<32, STREAM_U53, PLACE_TABLES, 2, false, true>;
  return pbn_ensemble_kernel<32, STREAM_U53, PLACE_TABLES, 2>;
#else
  if (pert_dom)  // perturbation-dominated launch: plan through L1/L2, phase-A prefetch
    return stream == STREAM_U53 ? pbn_ensemble_kernel<32, STREAM_U53, PLACE_GLOBAL, 0, true>
                                : pbn_ensemble_kernel<32, STREAM_U32, PLACE_GLOBAL, 0, true>;
  return stream == STREAM_U53 ? pick_lpt<STREAM_U53>(lpt, place, gm, pa2)
                              : pick_lpt<STREAM_U32>(lpt, place, gm, pa2);
#endif
}

std::uint32_t pf_max_warps() { return kMaxWarpsPf; }

std::size_t slot_words(const dev_plan_header& h, std::uint32_t lpt, bool node_counts) {
  return (2 * h.sw32 + lpt * 4 * kChunkBlocks + pa2_words(h, lpt) + (node_counts ? 8 * h.sw32 : 0) + 3) & ~3u;
}

// Parent gather mode of the sub-warp kernel for a plan (GM template
// parameter): register gathers — one state word per lane (RG) whenever it
// fits: the single-node rounds and the uniform general / plain rounds use
// shuffles; with the compact single-node records (SC) when the plan has them;
// two words per lane (RG2) only for the single-node rounds (general rounds
// keep the shared-memory gather: two shuffles per parent lose to it).
// GM 4 (U53, n' > 2047): the compact sgrp/sfn single-node records with
// shared-memory gathers.
int ensemble_gather_mode(const dev_plan_header& h, std::uint32_t lpt, int stream) {
  const bool rg = lpt == 32 && h.rg_ok;
  const bool rg2 = lpt == 32 && !h.rg_ok && h.sw32 <= 64 && h.n_single_alias >= 32 && kUseRg2;
  if (!rg && !rg2 && lpt == 32 && h.single_compact_l && stream == STREAM_U53 && kUseCompactSingle)
    return 4;
  return rg2 ? 3 : !rg ? 0 : (h.single_compact && kUseCompactSingle) ? 2 : 1;
}

// Two-steps-per-pass phase A (PA2 kernels): the register-gather kernels on a
// plan whose phase A is the k = 16 word path over at most half a warp.
bool ensemble_pa2(const dev_plan_header& h, std::uint32_t lpt, int gm, bool pert_dom) {
  return !pert_dom && (gm == 1 || gm == 2) && pa2_words(h, lpt) != 0;
}

cudaError_t launch_ensemble(const dev_plan_header& h, const std::uint8_t* d_blob, int place,
                            int stream_kind, std::uint32_t lpt, std::uint32_t warps_per_cta,
                            const dev_run_params& rp, std::uint64_t* d_states,
                            std::uint64_t* d_counts, cudaStream_t stream,
                            std::uint32_t* launches, bool pert_dom) {
  const int gm = pert_dom ? 0 : ensemble_gather_mode(h, lpt, stream_kind);
  const kernel_fn fn = select_kernel(lpt, stream_kind, place, gm, pert_dom, ensemble_pa2(h, lpt, gm, pert_dom));
  const std::uint32_t threads = warps_per_cta * 32;
  const std::uint32_t slots = threads / lpt;
  const std::uint32_t grid = (rp.n_traj + slots - 1) / slots;
  std::size_t staged = stream_kind == STREAM_U53 ? staged_prefix<STREAM_U53>(h, place)
                                                : staged_prefix<STREAM_U32>(h, place);
  if (gm == 4) staged = std::max<std::size_t>(staged, h.off_sfn);
  const std::size_t smem =
      staged + static_cast<std::size_t>(slots) * slot_words(h, lpt, rp.node_counts != nullptr) * 4 + 16;
  cudaError_t err = cudaFuncSetAttribute(reinterpret_cast<const void*>(fn),
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
  if (err != cudaSuccess) return err;
#if PBN_CARVEOUT
  // one CTA per SM: carve out only what it takes (+1 KiB the system reserves
  // per CTA), so that the rest of the 256 KiB stays L1 for the plan sections
  // read through it (the perturbation cells; tables and records when unstaged)
  err = cudaFuncSetAttribute(reinterpret_cast<const void*>(fn),
                             cudaFuncAttributePreferredSharedMemoryCarveout,
                             static_cast<int>(std::min<std::size_t>(100, (smem + 1024) * 100 / (228 * 1024) + 1)));
  if (err != cudaSuccess) return err;
#endif
  if (grid == 0) return cudaSuccess;
  fn<<<grid, threads, smem, stream>>>(h, d_blob, rp, d_states, d_counts);
  if (launches) ++*launches;
  return cudaGetLastError();
}

cudaError_t launch_philox_kat(const uint4* d_ctr, std::uint32_t k0, std::uint32_t k1, uint4* d_out,
                              std::uint32_t n, cudaStream_t stream) {
  pbn_philox_kat_kernel<<<(n + 127) / 128, 128, 0, stream>>>(d_ctr, k0, k1, d_out, n);
  return cudaGetLastError();
}

#else  // PBN_SCRIPT_TU: the scripted-replay launcher (capi.cpp pbn_gpu_run_scripted)

// One instantiation: one trajectory per warp, U53 decisions, the whole plan
// read through L1/L2, shared-memory gathers.
cudaError_t launch_ensemble_script(const dev_plan_header& h, const std::uint8_t* d_blob,
                                   std::uint32_t warps_per_cta, const dev_run_params& rp,
                                   std::uint64_t* d_states, std::uint64_t* d_counts,
                                   cudaStream_t stream) {
  auto fn = pbn_ensemble_kernel<32, STREAM_U53, PLACE_GLOBAL, 0>;
  const std::uint32_t threads = warps_per_cta * 32;
  const std::uint32_t grid = (rp.n_traj + warps_per_cta - 1) / warps_per_cta;
  const std::size_t slot = (2 * h.sw32 + 32 * 4 * kChunkBlocks + (rp.node_counts ? 8 * h.sw32 : 0) + 3) & ~3u;
  const std::size_t smem = static_cast<std::size_t>(warps_per_cta) * slot * 4 + 16;
  cudaError_t err = cudaFuncSetAttribute(reinterpret_cast<const void*>(fn),
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
  if (err != cudaSuccess) return err;
  if (grid == 0) return cudaSuccess;
  fn<<<grid, threads, smem, stream>>>(h, d_blob, rp, d_states, d_counts);
  return cudaGetLastError();
}
#endif  // PBN_SCRIPT_TU

}  // namespace pbn_b200
