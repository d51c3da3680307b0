// Lane-per-trajectory ensemble kernel for small networks: the same step as
// ensemble.cu (the reference's grouped_simulator::step, engine.hpp:255-312,
// driven by simulate(), engine.hpp:371-384), bit-exact on the same injected
// stream, with one whole trajectory per lane.
//
// Why: a small network (c1: n' = 77, c3: n' = 65) has a handful of phase-A
// Philox blocks and ~30 groups, so a sub-warp per trajectory leaves most lanes
// idle or pays sub-warp ballots/atomics per round. Here every lane runs the
// reference's sequential group loop for its own trajectory:
//
//   * the group loop is warp-uniform (same plan, same group order), so the
//     group record, its entry width and its output offset are broadcast
//     reads; only the chosen combined function and the parent values differ
//     per lane;
//   * states live in shared memory in a [word][32 lanes] layout: the parent
//     gathers and the output ORs of 32 lanes touch 32 distinct banks;
//   * phase-B draws come straight from the lane's own Philox block in
//     registers (one block per DPB alias groups, at warp-uniform points).
//
// The function phase runs under divergence (lanes whose step short-circuits
// sit it out), so this layout pays when the ensemble is large (>= ~16 warps
// per SM) and the network small; the host picks it as lanes_per_traj = 1.
#include <cuda_runtime.h>

#include <cstdint>
#include <type_traits>

#include "kernel_common.cuh"

namespace pbn_b200 {

// The exact FP64 choice of engine.hpp:285-290 (boundary draws, forced FP64
// runs, groups beyond the integer cells). Out of line so the compiler cannot
// hoist it into the fast path.
__device__ __noinline__ std::uint32_t alias_exact_fp64(const double* __restrict__ acut,
                                                       const std::uint32_t* __restrict__ aidx,
                                                       std::uint32_t asz, std::uint32_t ab,
                                                       std::uint64_t r53) {
  const double u = __ull2double_rn(r53) * 0x1.0p-53;
  const double xx = __dmul_rn(u, __uint2double_rn(asz));
  std::uint32_t c = __double2uint_rz(xx);
  if (c >= asz) c = asz - 1;
  const double fr = __dsub_rn(xx, __uint2double_rn(c));
  return fr < __ldg(acut + ab + c) ? c : __ldg(aidx + ab + c);
}

constexpr int kLaneMaxWarps = 28;  // 896 threads: 72 registers per thread
#ifndef PBN_SCAN_FN_LANES
#define PBN_SCAN_FN_LANES 28
#endif
// SCAN: pending function phases a warp collects before running them
constexpr int kScanFnLanes = PBN_SCAN_FN_LANES;

// SCAN: lanes scan their own steps through phase A up to the next function
// phase (pays when the function phase is rare, c1); otherwise all lanes take
// step s together and the function phase runs under divergence (c3, where
// ~90% of steps reach it).
// MODE 0 lockstep, 1 scan-ahead (SCAN), 2 CTA-compacted function phases,
// 3 scan-ahead with a per-lane queue of precomputed phase-A steps (QUEUE).
#ifndef PBN_LANE_QUEUE
#define PBN_LANE_QUEUE 4
#endif
constexpr std::uint32_t kQueueDepth = PBN_LANE_QUEUE;
template <int STREAM, int PLACE, int MODE>
__global__ void __launch_bounds__(kLaneMaxWarps * 32, 1)
    pbn_lane_kernel(const __grid_constant__ dev_plan_header h, const std::uint8_t* __restrict__ gblob,
                    const __grid_constant__ dev_run_params rp, std::uint64_t* __restrict__ states,
                    std::uint64_t* __restrict__ counts) {
  extern __shared__ __align__(16) std::uint8_t smem[];
  __shared__ std::uint64_t stage_bar;
  constexpr bool GC = placement<PLACE>::global_core;    // core sections read from global
  constexpr bool GT = placement<PLACE>::global_tables;  // tables read from global
  constexpr bool GP = placement<PLACE>::global_pert;    // perturbation cells read from global
  constexpr std::uint32_t DPB = draws<STREAM>::kPerBlock;

  const std::uint32_t staged = stage_placement<STREAM, PLACE>(smem, gblob, h, &stage_bar);

  const std::uint8_t* core = GC ? gblob : smem;
  const std::uint8_t* tab = GT ? gblob + h.off_tables : smem + h.off_tables;
  const std::uint8_t* pcells = pert_cells<STREAM, PLACE>(smem, gblob, h);
  const std::uint8_t* pfast = pert_fast_base<STREAM, GP>(pcells, gblob, h);
  const uint4* groups = reinterpret_cast<const uint4*>(core + h.off_groups);
  const uint4* fns = reinterpret_cast<const uint4*>(core + h.off_fns);
  const uint2* grec = reinterpret_cast<const uint2*>(core + h.off_grec);
  const double* acut = reinterpret_cast<const double*>(gblob + h.off_acut);
  const std::uint32_t* aidx = reinterpret_cast<const std::uint32_t*>(gblob + h.off_aidx);
  const uint4* acell = reinterpret_cast<const uint4*>(core + h.off_acell);
  const std::uint8_t* sbase = (h.fn_base || h.cell_base) ? gblob : core;
  const uint4* fns_s = reinterpret_cast<const uint4*>(sbase + h.off_fns_s);
  const uint4* acell_s = reinterpret_cast<const uint4*>(sbase + h.off_acell_s);
  const std::uint32_t* arec = reinterpret_cast<const std::uint32_t*>(core + h.off_arec);

  const std::uint32_t lane = threadIdx.x & 31;
  const std::uint32_t warp = threadIdx.x >> 5;
  const std::uint64_t tloc = static_cast<std::uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  constexpr bool SCAN = MODE == 1;
  const bool alive = tloc < rp.n_traj;  // MODE 2 keeps the rest for the CTA barriers
  const std::uint32_t lmask = __ballot_sync(0xFFFFFFFFu, alive);  // live lanes
  if (MODE != 2 && !alive) return;

  // per-warp shared memory: two state buffers of sw32 words x 32 lanes, then
  // (node counts) 8 counter planes per word; lane columns
  const std::uint32_t sw32 = h.sw32;
  const std::uint32_t warp_words =
      (2 + (rp.node_counts ? 8u : 0u) + (MODE == 3 ? kQueueDepth : 0u)) * sw32 * 32;
  std::uint32_t* wbuf = reinterpret_cast<std::uint32_t*>(smem + staged) +
                        static_cast<std::size_t>(warp) * warp_words + lane;
  std::uint32_t* planes = wbuf + 2 * sw32 * 32;  // plane i of word w at [(8w + i) * 32]
  std::uint32_t cur = 0;                          // current state buffer (per lane)
  {
    const std::uint32_t* src = reinterpret_cast<const std::uint32_t*>(states + tloc * (sw32 / 2));
    for (std::uint32_t w = 0; w < sw32; ++w)
      wbuf[32 * w] = alive ? src[w] & state_word_mask(h.n_kept, w) : 0u;
    if (rp.node_counts)
      for (std::uint32_t i = 0; i < 8 * sw32; ++i) planes[32 * i] = 0;
  }

  const std::uint32_t k = h.k, g = h.g;
  const bool exact_all = rp.exact_alias != 0;
  const std::uint32_t nb0 = (g + h.has_leaf + DPB - 1) / DPB;  // blocks of phase A
  const std::uint32_t nplain = g ? (g - 1) / DPB : 0;         // blocks of full-width draws only
  const std::uint32_t A = h.n_alias_groups, NG = h.n_groups, A1 = h.n_single_alias;
  const std::uint32_t traj = static_cast<std::uint32_t>(rp.traj_begin + tloc);
  std::uint32_t thi0, tlo0;
  mulhilo(kPhiloxM0, traj, thi0, tlo0);

  auto pred_eval = [&](const std::uint32_t* S) -> std::uint32_t {
    bool ok = rp.pred.n != 0;
    for (std::uint32_t i = 0; i < rp.pred.n; ++i)
      ok = ok && (S[32 * rp.pred.w[i]] & rp.pred.mask[i]) == rp.pred.want[i];
    return ok ? 1u : 0u;
  };

  // Combined-function choice (engine.hpp:284-291) from raw draw x: U53 integer
  // cells with the rare FP64 path, U32 integer cells (dev_plan.h acell).
  auto alias_fast = [&](const uint4* cells, std::uint32_t asz, std::uint32_t ab, const raw53& r,
                        std::uint32_t r32, bool& rare) -> std::uint32_t {
    if constexpr (STREAM == STREAM_U53) {
      const std::uint64_t P = static_cast<std::uint64_t>(r.hi) * asz;
      const std::uint32_t e = static_cast<std::uint32_t>(P >> 32);
      const uint2 V = ldp<GC>(reinterpret_cast<const uint2*>(cells + ab + e));
      rare = rare || static_cast<std::uint32_t>(P) > ~asz || r.hi == V.y;
      return r.hi < V.y ? e : V.x;
    } else {
      const std::uint64_t P = static_cast<std::uint64_t>(r32) * asz;
      const std::uint32_t c = static_cast<std::uint32_t>(P >> 32);
      const uint2 cell = ldp<GC>(reinterpret_cast<const uint2*>(cells + ab + c) + 1);
      return static_cast<std::uint32_t>(P) < cell.x ? c : cell.y;
    }
  };
  auto gather_fn = [&](const std::uint32_t* S, const uint4& F) -> std::uint32_t {
    const std::uint32_t gc = F.y & 31u;
    std::uint32_t v = gather4_col(S, F.z, F.w, 0);
    if constexpr (MODE == 0) {
      // lockstep (c3: most chosen functions have more than four inputs): the loop form
      if (gc > 4) {
        const std::uint32_t xq = F.y >> 8;
        for (std::uint32_t q = 4; q < gc; q += 4) {
          const uint2 rr = ldp<GC>(grec + xq + ((q - 4) >> 2));
          v |= gather4_col(S, rr.x, rr.y, q);
        }
      }
    } else if (gc > 4) {
      // scan-ahead variants (c1: few do): inputs 4..7 without a loop; measured
      // per instantiation — c1 9.49e9 -> 1.04e10, while c3 loses 3.7 % with this form
      const std::uint32_t xq = F.y >> 8;
      const uint2 r4 = ldp<GC>(grec + xq);
      v |= gather4_col(S, r4.x, r4.y, 4);
      if (__builtin_expect(gc > 8, 0)) {
        for (std::uint32_t q = 8; q < gc; q += 4) {
          const uint2 rr = ldp<GC>(grec + xq + ((q - 4) >> 2));
          v |= gather4_col(S, rr.x, rr.y, q);
        }
      }
    }
    return v;
  };

  std::uint32_t nc_pending = 0;
  auto nc_flush = [&]() {
    std::uint64_t* dst = rp.node_counts + tloc * h.n_kept;
    for (std::uint32_t w = 0; w < sw32; ++w) {
      std::uint32_t pl[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        pl[i] = planes[32 * (8 * w + i)];
        planes[32 * (8 * w + i)] = 0;
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

  const std::uint32_t z0 = pred_eval(wbuf);
  std::uint32_t prev = 2u, kphase = 0;
  if (rp.thin_mode == 0) prev = z0;
  if (rp.thin_mode == 1 && rp.tprev) {
    const std::uint32_t tp = rp.tprev[tloc];
    prev = tp & 3u;
    kphase = tp >> 2;
  }
  std::uint32_t nv = 0, np1 = 0, nh1 = 0, n11 = 0, nhit = 0, nfn = 0, npert = 0;
  std::uint32_t* ser = rp.series ? rp.series + tloc * rp.series_stride : nullptr;
  std::uint32_t sword = 0;
  if (ser && rp.series_init && rp.series_bit0 > 0 && z0) {
    const std::uint64_t p0 = rp.series_bit0 - 1;
    ser[p0 >> 5] |= 1u << (p0 & 31);
  }
  const std::uint64_t s_end = rp.step_begin + rp.n_steps;

  // Statistics of step s on the state after it (engine.hpp:375-381) +
  // sampled predicate transitions, series bits and node counts.
  auto step_stats = [&](const std::uint32_t* Sc, std::uint64_t s) {
    const std::uint32_t hit = pred_eval(Sc);
    nhit += hit;
    if (++kphase == rp.kappa) {
      kphase = 0;
      const std::uint32_t valid = (prev >> 1) ^ 1u;
      nv += valid;
      np1 += prev & 1u;
      nh1 += hit & valid;
      n11 += prev & hit;
      prev = hit;
    }
    if (rp.node_counts) {  // launch-uniform branch
      for (std::uint32_t w = 0; w < sw32; ++w) {
        std::uint32_t x = Sc[32 * w];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const std::uint32_t p = planes[32 * (8 * w + i)];
          planes[32 * (8 * w + i)] = p ^ x;
          x &= p;
        }
      }
      if (++nc_pending == 255) nc_flush();
    }
    if (ser != nullptr) {
      const std::uint64_t pos = rp.series_bit0 + (s - rp.step_begin);
      sword |= hit << (pos & 31);
      if ((pos & 31) == 31 || s + 1 == s_end) {
        if (sword) ser[pos >> 5] |= sword;
        sword = 0;
      }
    }
  };

  // Phase-A masks (engine.hpp:257-268): full patterns for groups before the
  // last, the k'-bit mask for the last group (:261), nothing for the leaf
  // draw and past it; lf_elem: the leaf draw's element of block b (>= DPB: none).
  auto pa_mask = [&](std::uint32_t b, std::uint32_t e) -> std::uint32_t {
    const int q = static_cast<int>(g) - 1 - static_cast<int>(b * DPB + e);
    return q > 0 ? 0xFFFFFFFFu : (q == 0 ? h.last_mask : 0u);
  };
  auto lf_elem = [&](std::uint32_t b) -> std::uint32_t {
    const int e = static_cast<int>(g) - static_cast<int>(b * DPB);
    return h.has_leaf && e >= 0 && e < static_cast<int>(DPB) ? static_cast<std::uint32_t>(e) : DPB;
  };

  // Phase A of step `sp` on state Sc (engine.hpp:257-268): flips XORed in.
  auto phase_a_step = [&](std::uint32_t* Sc, const step_philox& sp, bool& flip, bool& leaf) {
    flip = false;
    leaf = false;
    // One Philox block: decisions of its DPB draws on the high words (U53:
    // a tie recomputes them with the low block), masks, XOR into the lane's
    // state column. Blocks [0, nplain) hold full-width pattern draws only; the
    // tail blocks hold the last group (k'-bit mask, engine.hpp:261) and the
    // leaf draw (warp-uniform masks). WPB (k = 16: 2, k = 8: 1): a block's
    // patterns fill exactly state words b*WPB.. — XOR each word once.
    auto block = [&](std::uint32_t b, bool tail, auto bern_c, auto wpb_c) {
      constexpr bool BERN = decltype(bern_c)::value;  // node-wise plans (Method_old / reduction)
      constexpr std::uint32_t WPB = decltype(wpb_c)::value;
      const uint4 x = philox_block(sp, b, rp.rk0, rp.rk1);
      const std::uint32_t lfe = tail ? lf_elem(b) : DPB;
      std::uint32_t c[DPB];
      bool rare = false, lf = false;
#pragma unroll
      for (std::uint32_t e = 0; e < DPB; ++e)
        c[e] = pa_draw<STREAM, GP, BERN>(h, gblob, pfast, k, pick32(x, e), false, 0u, rare);
      if (lfe < DPB) lf = pa_leaf<STREAM>(h, pick32(x, lfe), false, 0u, rare);
      if constexpr (STREAM == STREAM_U53) {
        if (__builtin_expect(rare, 0)) {
          const uint4 y = philox_lo_block(sp, b, rp.rk0, rp.rk1);
          bool unused = false;
#pragma unroll
          for (std::uint32_t e = 0; e < DPB; ++e)
            c[e] = pa_draw<STREAM, GP, BERN>(h, gblob, pfast, k, pick32(x, e), true, pick32(y, e), unused);
          if (lfe < DPB) lf = pa_leaf<STREAM>(h, pick32(x, lfe), true, pick32(y, lfe), unused);
        }
      }
      leaf = leaf || lf;
      if (tail) {
#pragma unroll
        for (std::uint32_t e = 0; e < DPB; ++e) c[e] &= pa_mask(b, e);
      }
      if constexpr (WPB == 2) {
        const std::uint32_t w0 = c[0] | (c[1] << 16), w1 = c[2] | (c[3] << 16);
        if (__builtin_expect((w0 | w1) != 0, 0)) {  // xor_chunk (bitstate.hpp:50-58)
          flip = true;
          Sc[32 * (2 * b)] ^= w0;
          Sc[32 * (2 * b + 1)] ^= w1;
        }
      } else if constexpr (WPB == 1) {
        const std::uint32_t w0 = c[0] | (c[1] << 8) | (c[2] << 16) | (c[3] << 24);
        if (__builtin_expect(w0 != 0, 0)) {
          flip = true;
          Sc[32 * b] ^= w0;
        }
      } else {
#pragma unroll
        for (std::uint32_t e = 0; e < DPB; ++e) {
          const std::uint32_t ce = c[e];
          if (__builtin_expect(ce != 0, 0)) {  // xor_chunk (bitstate.hpp:50-58)
            flip = true;
            const std::uint32_t o = (b * DPB + e) * k, w = o >> 5, sh = o & 31;
            Sc[32 * w] ^= ce << sh;
            if (sh != 0 && (ce >> (32 - sh)) != 0) Sc[32 * (w + 1)] ^= ce >> (32 - sh);
          }
        }
      }
    };
    auto phase_a = [&](auto bern_c, auto wpb_c) {
      for (std::uint32_t b = 0; b < nplain; ++b) block(b, false, bern_c, wpb_c);
      for (std::uint32_t b = nplain; b < nb0; ++b) block(b, true, bern_c, wpb_c);
    };
    if (h.pert_mode != 0)
      phase_a(std::true_type{}, std::integral_constant<std::uint32_t, 0>{});
    else if (k == 16)
      phase_a(std::false_type{}, std::integral_constant<std::uint32_t, 2>{});
    else if (k == 8)
      phase_a(std::false_type{}, std::integral_constant<std::uint32_t, 1>{});
    else
      phase_a(std::false_type{}, std::integral_constant<std::uint32_t, 0>{});
  };

  // Function phase of step `sp` (engine.hpp:270-311): the reference's group
  // loop from state Sc into Sn.
  auto fn_phase = [&](const std::uint32_t* Sc, std::uint32_t* Sn, const step_philox& sp) {
    for (std::uint32_t w = 0; w < sw32; ++w) Sn[32 * w] = 0;
    uint4 xb = make_uint4(0, 0, 0, 0);  // the phase-B block holding draw j
    // r53 of draw j = gi for the rare FP64 path: high word + the low block's word
    auto r53_of = [&](std::uint32_t gi, const raw53& r) -> std::uint64_t {
      return raw53{r.hi, lo_word<STREAM>(sp, nb0 + gi / DPB, gi % DPB, rp.rk0, rp.rk1)}.value();
    };
    for (std::uint32_t gi = 0; gi < NG; ++gi) {
      raw53 r{0, 0};
      std::uint32_t r32 = 0;
      if (gi < A) {  // draw j = gi (alias groups come first)
        const std::uint32_t e = gi % DPB;
        if (e == 0) xb = philox_block(sp, nb0 + gi / DPB, rp.rk0, rp.rk1);
        r.hi = pick32(xb, e);
        r32 = r.hi;
      }
      std::uint32_t olo, ohi = 0, off, members;
      if (gi < A1) {  // single node at offset gi, inline 1-bit tables (dev_plan.h arec)
        const std::uint32_t ar = ldp<GC>(arec + gi);
        const std::uint32_t base = ar & 0xFFFFFFu, asz = ar >> 24;
        bool rare = exact_all;
        // acell_s / fns_s == acell / fns unless the plan has the unstaged
        // tail of compact plans (global memory; ldp<false> is then generic)
        std::uint32_t f = base + alias_fast(acell_s, asz, base, r, r32, rare);
        if constexpr (STREAM == STREAM_U53)
          if (__builtin_expect(rare, 0)) f = base + alias_exact_fp64(acut, aidx, asz, base, r53_of(gi, r));
        const uint4 F = ldp<GC>(fns_s + f);
        olo = (F.x >> gather_fn(Sc, F)) & 1u;
        off = gi;
        members = 1;
      } else {
        const uint4 G = ldp<GC>(groups + gi);
        const std::uint32_t asz = G.w & 0x7FFFFFu;
        members = (G.w >> 24) + 1;
        off = G.x;
        std::uint32_t idx = 0;
        if (asz != 0) {
          bool rare = exact_all || (G.w & kGroupExactAlias);
          idx = alias_fast(acell, asz, G.z, r, r32, rare);
          if constexpr (STREAM == STREAM_U53)
            if (__builtin_expect(rare, 0)) idx = alias_exact_fp64(acut, aidx, asz, G.z + h.cell_base, r53_of(gi, r));
        }
        const uint4 F = ldp<GC>(fns + G.y + idx);
        const std::uint32_t v = gather_fn(Sc, F);
        if (F.y & 0x80u) {  // inline table
          const std::uint32_t m = members >= 32 ? 0xFFFFFFFFu : ((1u << members) - 1u);
          olo = (F.x >> (v * members)) & m;
        } else {
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
        }
      }
      // next |= out << offset (engine.hpp:304-309); offset and width are
      // the group's, so the branches are warp-uniform
      const std::uint32_t w = off >> 5, sh = off & 31;
      Sn[32 * w] |= olo << sh;
      if (sh + members > 32) {
        Sn[32 * (w + 1)] |= sh ? (olo >> (32 - sh)) | (ohi << sh) : ohi;
        if (sh + members > 64) Sn[32 * (w + 2)] |= ohi >> (32 - sh);
      }
    }
  };

  if constexpr (MODE == 2) {
    // CTA-compacted function phases: every trajectory of the CTA advances
    // one step per iteration; phase A and the statistics run with all lanes,
    // and the function phases the step needs are packed into a task list
    // (warp ballots + a prefix over the warps) that the first
    // ceil(tasks / 32) warps run with full lanes — a thread may run another
    // lane's trajectory: its state column, its buffer parity and its stream
    // (seed, trajectory, step) travel with the task.
    std::uint32_t* cta = reinterpret_cast<std::uint32_t*>(smem + staged) +
                         static_cast<std::size_t>(blockDim.x >> 5) * warp_words;
    std::uint32_t* wcnt = cta;                                          // [32]
    std::uint16_t* task = reinterpret_cast<std::uint16_t*>(cta + 32);  // [blockDim]
    std::uint32_t* states0 = reinterpret_cast<std::uint32_t*>(smem + staged);
    const std::uint32_t nwarps = blockDim.x >> 5;
    const std::uint32_t lt_mask = (1u << lane) - 1u;
    for (std::uint64_t s = rp.step_begin; s < s_end; ++s) {
      std::uint32_t* Sc = wbuf + cur * (sw32 * 32);
      bool need = false;
      if (alive) {
        const step_philox sp = make_step_philox(thi0, tlo0, s, rp.rk0, rp.rk1);
        bool flip, leaf;
        phase_a_step(Sc, sp, flip, leaf);
        need = !flip && !leaf;
        if (!need) {
          npert += flip ? 1u : 0u;
          step_stats(Sc, s);
        }
      }
      const std::uint32_t bal = __ballot_sync(0xFFFFFFFFu, need);
      if (lane == 0) wcnt[warp] = __popc(bal);
      __syncthreads();
      // exclusive prefix of the warp counts (every warp computes it)
      std::uint32_t v = lane < nwarps ? wcnt[lane] : 0u;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const std::uint32_t t = __shfl_up_sync(0xFFFFFFFFu, v, o);
        if (lane >= static_cast<std::uint32_t>(o)) v += t;
      }
      const std::uint32_t total = __shfl_sync(0xFFFFFFFFu, v, 31);
      const std::uint32_t before = __shfl_sync(0xFFFFFFFFu, v, warp) - __popc(bal);
      if (need) task[before + __popc(bal & lt_mask)] =
          static_cast<std::uint16_t>(threadIdx.x | (cur << 15));
      __syncthreads();
      if (threadIdx.x < total) {
        const std::uint32_t e = task[threadIdx.x];
        const std::uint32_t q = e & 0x7FFFu, qc = e >> 15;
        std::uint32_t* col = states0 + static_cast<std::size_t>(q >> 5) * warp_words + (q & 31u);
        const std::uint32_t tq = static_cast<std::uint32_t>(rp.traj_begin + blockIdx.x * blockDim.x + q);
        std::uint32_t qh, ql;
        mulhilo(kPhiloxM0, tq, qh, ql);
        const step_philox spq = make_step_philox(qh, ql, s, rp.rk0, rp.rk1);
        fn_phase(col + qc * (sw32 * 32), col + (qc ^ 1u) * (sw32 * 32), spq);
      }
      __syncthreads();
      if (need) {
        cur ^= 1;
        ++nfn;
        step_stats(wbuf + cur * (sw32 * 32), s);
      }
    }
  } else if constexpr (MODE == 3) {
    // QUEUE: the class of a step AND its flip patterns depend on the stream
    // only, so a lane whose next step needs the function phase keeps
    // producing: phase A of its following steps goes into a queue of up to
    // kQueueDepth (XOR mask, class) entries in shared memory ([slot][word]
    // [lane] columns) instead of waiting for the warp. Three kinds of rounds:
    // consume — every lane applies its queued perturbed / leaf steps up to its
    // next function-phase step (a few XORs + the statistics); function — run
    // by the warp once >= kScanFnLanes lanes have one at the head of their
    // queue (or nothing can be produced); produce — every lane with room
    // computes phase A of its next unqueued step. The expensive rounds
    // (produce: Philox + cell probes; function: the group loop) both run with
    // nearly full warps.
    std::uint32_t* qbuf = wbuf + (2 + (rp.node_counts ? 8u : 0u)) * sw32 * 32;
    std::uint64_t s = rp.step_begin;  // the lane's next step to take (head of the queue)
    std::uint32_t qn = 0;             // queued steps s .. s + qn - 1
    std::uint32_t qcls = 0;           // their classes, 2 bits each, head in bits 0-1: 0 flip, 1 leaf, 2 function
    std::uint32_t qhead = 0;          // slot of the head
    for (;;) {
      while (qn != 0 && (qcls & 3u) != 2u) {  // consume
        std::uint32_t* Sc = wbuf + cur * (sw32 * 32);
        if ((qcls & 3u) == 0u) {
          const std::uint32_t* q = qbuf + qhead * (sw32 * 32);
          for (std::uint32_t w = 0; w < sw32; ++w) Sc[32 * w] ^= q[32 * w];
          ++npert;
        }
        step_stats(Sc, s);
        ++s;
        qcls >>= 2;
        --qn;
        qhead = qhead + 1 == kQueueDepth ? 0u : qhead + 1;
      }
      const bool fn_head = qn != 0;  // its class is 2 after the consume loop
      const bool can_produce = qn < kQueueDepth && s + qn < s_end;
      const std::uint32_t pend = __ballot_sync(lmask, fn_head);
      const std::uint32_t prod = __ballot_sync(lmask, can_produce);
      if (pend == 0 && prod == 0) break;
      if (prod == 0 || __popc(pend) >= kScanFnLanes) {
        if (fn_head) {
          const step_philox sp = make_step_philox(thi0, tlo0, s, rp.rk0, rp.rk1);
          std::uint32_t* Sn = wbuf + (cur ^ 1) * (sw32 * 32);
          fn_phase(wbuf + cur * (sw32 * 32), Sn, sp);
          cur ^= 1;
          ++nfn;
          step_stats(Sn, s);
          ++s;
          qcls >>= 2;
          --qn;
          qhead = qhead + 1 == kQueueDepth ? 0u : qhead + 1;
        }
      } else if (can_produce) {
        std::uint32_t slot = qhead + qn;
        if (slot >= kQueueDepth) slot -= kQueueDepth;
        std::uint32_t* q = qbuf + slot * (sw32 * 32);
        for (std::uint32_t w = 0; w < sw32; ++w) q[32 * w] = 0;
        const step_philox sp = make_step_philox(thi0, tlo0, s + qn, rp.rk0, rp.rk1);
        bool flip, leaf;
        phase_a_step(q, sp, flip, leaf);
        qcls |= (flip ? 0u : leaf ? 1u : 2u) << (2 * qn);
        ++qn;
      }
    }
  } else if constexpr (SCAN) {
    // The class of a step (perturbed / leaf no-op / function phase) depends
    // on the stream only, never on the state: each lane scans its own steps
    // through phase A until one needs the function phase, so the warp runs
    // the (expensive, per-lane) function phase with every lane that still has
    // steps, instead of with the ~(1-p)^n' share whose current step needs it.
    // One phase-A round at a time: lanes without a pending function phase
    // advance one step; the warp runs the function phase once at least
    // kScanFnLanes lanes have one pending (or no lane can scan further), so
    // neither the scan rounds nor the function phases run with few lanes.
    std::uint64_t s = rp.step_begin;
    bool need = false;
    step_philox sp{};
    for (;;) {
      if (!need && s < s_end) {
        sp = make_step_philox(thi0, tlo0, s, rp.rk0, rp.rk1);
        bool flip, leaf;
        std::uint32_t* Sc = wbuf + cur * (sw32 * 32);
        phase_a_step(Sc, sp, flip, leaf);
        if (!flip && !leaf) {
          need = true;
        } else {
          npert += flip ? 1u : 0u;
          step_stats(Sc, s);
          ++s;
        }
      }
      const std::uint32_t pend = __ballot_sync(lmask, need);
      const std::uint32_t scanning = __ballot_sync(lmask, !need && s < s_end);
      if (pend == 0 && scanning == 0) break;
      if (scanning == 0 || __popc(pend) >= kScanFnLanes) {
        if (need) {
          std::uint32_t* Sn = wbuf + (cur ^ 1) * (sw32 * 32);
          fn_phase(wbuf + cur * (sw32 * 32), Sn, sp);
          cur ^= 1;
          ++nfn;
          step_stats(Sn, s);
          ++s;
          need = false;
        }
      }
    }
  } else {
    for (std::uint64_t s = rp.step_begin; s < s_end; ++s) {
      std::uint32_t* Sc = wbuf + cur * (sw32 * 32);
      const step_philox sp = make_step_philox(thi0, tlo0, s, rp.rk0, rp.rk1);
      bool flip, leaf;
      phase_a_step(Sc, sp, flip, leaf);
      if (flip) {
        ++npert;
      } else if (!leaf) {
        std::uint32_t* Sn = wbuf + (cur ^ 1) * (sw32 * 32);
        fn_phase(Sc, Sn, sp);
        cur ^= 1;
        Sc = Sn;
        ++nfn;
      }
      step_stats(Sc, s);
    }
  }
  if (!alive) return;
  if (rp.node_counts && nc_pending) nc_flush();
  if (rp.tprev) rp.tprev[tloc] = static_cast<std::uint8_t>(prev | (kphase << 2));
  {
    const std::uint32_t* Sf = wbuf + cur * (sw32 * 32);
    std::uint32_t* dst = reinterpret_cast<std::uint32_t*>(states + tloc * (sw32 / 2));
    for (std::uint32_t w = 0; w < sw32; ++w) dst[w] = Sf[32 * w];
  }
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

using lane_kernel_fn = void (*)(const dev_plan_header, const std::uint8_t*, const dev_run_params,
                                std::uint64_t*, std::uint64_t*);

template <int STREAM, int MODE>
lane_kernel_fn pick_lane_place(int place) {
  switch (place) {
    case PLACE_ALL:
      return pbn_lane_kernel<STREAM, PLACE_ALL, MODE>;
    case PLACE_CORE_PERT:
      return pbn_lane_kernel<STREAM, PLACE_CORE_PERT, MODE>;
    case PLACE_TABLES:
      return pbn_lane_kernel<STREAM, PLACE_TABLES, MODE>;
    case PLACE_CORE:
      return pbn_lane_kernel<STREAM, PLACE_CORE, MODE>;
    default:
      return pbn_lane_kernel<STREAM, PLACE_GLOBAL, MODE>;
  }
}

// The variant for steps that rarely reach the function phase (the host's
// `scan` choice): per-warp scan-ahead (1), or CTA compaction (2) — bit-exact,
// but on c1 6.4e9 vs 9.56e9 trajectory-steps/s: while the packed function
// phases run, most warps of the CTA wait at the barrier and the few working
// ones cannot hide the phase's load latency.
#ifndef PBN_LANE_COMPACT
#define PBN_LANE_COMPACT 0
#endif
// QUEUE (3) is bit-exact and cuts the produce rounds from 2.09 to 1.39 per
// step on c1, but its consume rounds and stash traffic cost more than that
// saves: 9.24e9 vs 9.49e9 trajectory-steps/s for SCAN.
#ifndef PBN_LANE_RARE_MODE
#define PBN_LANE_RARE_MODE 1
#endif
constexpr int kRareFnMode = PBN_LANE_COMPACT ? 2 : PBN_LANE_RARE_MODE;
const char* lane_rare_fn_name() {
  return kRareFnMode == 2 ? "compact" : kRareFnMode == 3 ? "queue" : "scan";
}
// Shared memory of the CTA-compaction variant: warp counts + the task list.
std::size_t lane_cta_bytes() { return kRareFnMode == 2 ? 4 * 32 + 2 * 32 * kLaneMaxWarps + 16 : 0; }

// The lane kernel serves lanes_per_traj = 1 for networks up to 255 kept nodes
// (8 state words; larger ones use ensemble.cu's one-lane sub-warps).
bool lane_kernel_fits(const dev_plan_header& h) { return h.sw32 <= 8; }
std::uint32_t lane_max_warps() { return kLaneMaxWarps; }

// Shared-memory words per warp of the lane kernel: two state buffers and the
// optional counter planes, sw32 words per lane each.
std::size_t lane_warp_words(const dev_plan_header& h, bool node_counts, bool scan) {
  return static_cast<std::size_t>(2 + (node_counts ? 8 : 0) +
                                  (scan && kRareFnMode == 3 ? kQueueDepth : 0)) * h.sw32 * 32;
}

cudaError_t launch_lane_ensemble(const dev_plan_header& h, const std::uint8_t* d_blob, int place,
                                 int stream_kind, bool scan, std::uint32_t warps_per_cta,
                                 const dev_run_params& rp, std::uint64_t* d_states,
                                 std::uint64_t* d_counts, cudaStream_t stream,
                                 std::uint32_t* launches) {
  const lane_kernel_fn fn =
      stream_kind == STREAM_U53
          ? (scan ? pick_lane_place<STREAM_U53, kRareFnMode>(place) : pick_lane_place<STREAM_U53, 0>(place))
          : (scan ? pick_lane_place<STREAM_U32, kRareFnMode>(place) : pick_lane_place<STREAM_U32, 0>(place));
  const std::uint32_t threads = warps_per_cta * 32;
  const std::uint32_t grid = (rp.n_traj + threads - 1) / threads;
  const std::size_t staged = stream_kind == STREAM_U53 ? staged_prefix<STREAM_U53>(h, place)
                                                      : staged_prefix<STREAM_U32>(h, place);
  const std::size_t smem = staged +
                           static_cast<std::size_t>(warps_per_cta) *
                               lane_warp_words(h, rp.node_counts != nullptr, scan) * 4 +
                           (scan ? lane_cta_bytes() : 0) + 16;
  cudaError_t err = cudaFuncSetAttribute(reinterpret_cast<const void*>(fn),
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
  if (err != cudaSuccess) return err;
  if (grid == 0) return cudaSuccess;
  fn<<<grid, threads, smem, stream>>>(h, d_blob, rp, d_states, d_counts);
  if (launches) ++*launches;
  return cudaGetLastError();
}

}  // namespace pbn_b200
