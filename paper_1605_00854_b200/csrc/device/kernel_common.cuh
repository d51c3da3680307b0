// Device helpers shared by the trajectory kernels (ensemble.cu: sub-warp per
// trajectory; lane_ensemble.cu: lane per trajectory with a warp-cooperative
// function phase): plan staging, the stream's draw layout, perturbation-cell
// lookups and parent-bit gathers.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "dev_plan.h"
#include "philox.cuh"

namespace pbn_b200 {

enum { STREAM_U53 = 0, STREAM_U32 = 1 };
// Plan placement = the staged prefix of the blob (dev_plan.h): 0 nothing (all
// reads through the read-only L1/L2 path), 1 core, 2 core + tables, 3 also the
// perturbation cells of the launch's stream.
// PLACE_CORE_PERT (4) stages the core and the launch stream's perturbation
// cells (two bulk copies; the cells land right after the core) and reads the
// tables through L1/L2: for plans whose tables are too large but whose cells
// fit (perturbation-dominated runs, c5 at high p).
enum { PLACE_GLOBAL = 0, PLACE_CORE = 1, PLACE_TABLES = 2, PLACE_ALL = 3, PLACE_CORE_PERT = 4 };

template <int STREAM>
__host__ __device__ inline std::uint32_t pert_off(const dev_plan_header& h) {
  return STREAM == 0 ? h.off_pert53 : h.off_pert32;
}
template <int STREAM>
__host__ __device__ inline std::uint32_t pert_bytes(const dev_plan_header& h) {
  return STREAM == 0 ? h.blob_bytes - h.off_pert53 : h.off_pert53 - h.off_pert32;
}

// Shared-memory bytes a launch stages for placement `place`.
template <int STREAM>
__host__ __device__ inline std::uint32_t staged_prefix(const dev_plan_header& h, int place) {
  if (place == PLACE_ALL) return STREAM == 0 ? h.blob_bytes : h.off_pert53;
  if (place == PLACE_TABLES) return h.off_pert32;
  if (place == PLACE_CORE) return h.core_bytes;
  if (place == PLACE_CORE_PERT) return h.core_bytes + pert_bytes<STREAM>(h);
  return 0;
}

// Which sections a placement reads through L1/L2 instead of shared memory.
template <int PLACE>
struct placement {
  static constexpr bool global_core = PLACE == PLACE_GLOBAL;
  static constexpr bool global_tables = PLACE != PLACE_TABLES && PLACE != PLACE_ALL;
  static constexpr bool global_pert = PLACE != PLACE_ALL && PLACE != PLACE_CORE_PERT;
};

template <bool G, class T>
__device__ __forceinline__ T ldp(const T* p) {
  if constexpr (G)
    return __ldg(p);
  else
    return *p;
}

__device__ __forceinline__ std::uint32_t smem_u32(const void* p) {
  return static_cast<std::uint32_t>(__cvta_generic_to_shared(p));
}

// One 16-byte shared-memory load that stays one LDS.128 (4 wavefronts per
// warp for consecutive records). Left to the compiler, a uint4 record whose
// components are consumed one by one under selects is split into 4-byte
// loads at a 16-byte lane stride — 4-way bank conflicts on each.
__device__ __forceinline__ uint4 lds128(const uint4* p) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(smem_u32(p)));
  return v;
}

// Stage bytes [0, n0) of the blob, then (n1 > 0) n1 bytes from src1 right
// after them, with bulk copies (multiples of 16 bytes) completing on one
// mbarrier; every thread of the CTA waits.
__device__ __forceinline__ void stage_plan(std::uint8_t* dst, const std::uint8_t* src,
                                           std::uint32_t n0, std::uint64_t* bar,
                                           const std::uint8_t* src1 = nullptr,
                                           std::uint32_t n1 = 0) {
  const std::uint32_t b = smem_u32(bar);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(n0 + n1)
                 : "memory");
    auto copy = [&](std::uint8_t* d, const std::uint8_t* sp, std::uint32_t bytes) {
      for (std::uint32_t off = 0; off < bytes; off += 32768u) {
        const std::uint32_t n = bytes - off < 32768u ? bytes - off : 32768u;
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
                "r"(smem_u32(d + off)),
            "l"(sp + off), "r"(n), "r"(b)
            : "memory");
      }
    };
    copy(dst, src, n0);
    if (n1) copy(dst + n0, src1, n1);
  }
  __syncthreads();
  std::uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(b)
        : "memory");
  }
}

// Stage what placement PLACE keeps in shared memory; returns the bytes used.
template <int STREAM, int PLACE>
__device__ __forceinline__ std::uint32_t stage_placement(std::uint8_t* smem, const std::uint8_t* gblob,
                                                         const dev_plan_header& h,
                                                         std::uint64_t* bar) {
  const std::uint32_t staged = staged_prefix<STREAM>(h, PLACE);
  if constexpr (PLACE == PLACE_CORE_PERT)
    stage_plan(smem, gblob, h.core_bytes, bar, gblob + pert_off<STREAM>(h), pert_bytes<STREAM>(h));
  else if (staged)
    stage_plan(smem, gblob, staged, bar);
  return staged;
}

// This stream's perturbation cells for placement PLACE.
template <int STREAM, int PLACE>
__device__ __forceinline__ const std::uint8_t* pert_cells(const std::uint8_t* smem,
                                                          const std::uint8_t* gblob,
                                                          const dev_plan_header& h) {
  if constexpr (PLACE == PLACE_CORE_PERT) return smem + h.core_bytes;
  if constexpr (PLACE == PLACE_ALL) return smem + pert_off<STREAM>(h);
  return gblob + pert_off<STREAM>(h);
}

// Valid bits of 32-bit state word w of an n-bit state: bits at and above n
// (the slack bit n' that padded gather slots read, and the rest of the last
// word) must be zero, so a caller's stray high bits are cleared on load.
__device__ __forceinline__ std::uint32_t state_word_mask(std::uint32_t n, std::uint32_t w) {
  const std::uint32_t lo = 32 * w;
  return lo + 32 <= n ? 0xFFFFFFFFu : lo >= n ? 0u : (1u << (n - lo)) - 1u;
}

// Both streams take 4 draws per Philox block: word e of block b is the high
// word of draw 4b + e (U32: the whole draw; U53: its low word is word e of
// block b | kLoBlock, philox.cuh).
template <int STREAM>
struct draws {
  static constexpr std::uint32_t kPerBlock = 4;
};

// The low block of block position b (U53 rare paths). Out of line: the hot
// paths keep the registers a second inlined Philox block would take.
static __device__ __noinline__ uint4 philox_lo_block(step_philox sp, std::uint32_t b,
                                              const std::uint32_t* rk0, const std::uint32_t* rk1) {
  return philox_block(sp, b | kLoBlock, rk0, rk1);
}

// Low word of draw e of block b (U53; U32 draws have none): the rare paths.
template <int STREAM>
__device__ __forceinline__ std::uint32_t lo_word(const step_philox& sp, std::uint32_t b,
                                                 std::uint32_t e, const std::uint32_t* rk0,
                                                 const std::uint32_t* rk1) {
  if constexpr (STREAM == STREAM_U53) {
    const uint4 y = philox_lo_block(sp, b, rk0, rk1);
    return e == 0 ? y.x : e == 1 ? y.y : e == 2 ? y.z : y.w;
  } else {
    return 0u;
  }
}

// Raw draw: r53 as (hi32, lo21) pieces (U32: lo = 0, r53 = r32 << 21, the
// same double r32 * 2^-32).
struct raw53 {
  std::uint32_t hi;  // bits [21, 53) of r53  (= x[2e+1])
  std::uint32_t lo;  // x[2e]; bits [0, 21) of r53 are lo >> 11
  __device__ __forceinline__ std::uint64_t value() const {
    return (static_cast<std::uint64_t>(hi) << 21) | (lo >> 11);
  }
  // raw word R = hi << 32 | lo; r53 = R >> 11 (dev_plan.h: raw-word thresholds)
  __device__ __forceinline__ std::uint64_t raw() const {
    return (static_cast<std::uint64_t>(hi) << 32) | lo;
  }
};

// Word e (0..3) of a block: two levels of selects, no branches.
__device__ __forceinline__ std::uint32_t pick32(const uint4& x, std::uint32_t e) {
  const std::uint32_t lo = (e & 1u) ? x.y : x.x, hi = (e & 1u) ? x.w : x.z;
  return (e & 2u) ? hi : lo;
}

#ifndef PBN_PERT53H
#define PBN_PERT53H 1
#endif
constexpr bool kPert53h = PBN_PERT53H != 0;  // 0: A/B switch, always the 8-byte cells

// The launch's perturbation cells as the fast paths read them: U53 launches
// that read the cells through L1/L2 (G) use the dense high-word array
// pert53h; otherwise the stream's (staged or global) cells.
template <int STREAM, bool G>
__device__ __forceinline__ const std::uint8_t* pert_fast_base(const std::uint8_t* pcells,
                                                              const std::uint8_t* gblob,
                                                              const dev_plan_header& h) {
  if constexpr (G && STREAM == 0 && kPert53h)
    return gblob + h.off_pert53h;
  else
    return pcells;
}
#ifndef PBN_PERT_NOALLOC
#define PBN_PERT_NOALLOC 1
#endif
// The high word of U53 cell c.
// NA (no L1 allocation): the random 4-byte probes of the 256 KiB table go
// through L2 without taking L1 lines from the plan sections that do get
// reused (+0.4-0.5 % on c2/c4/c5 p <= 1e-3); the PF kernels, where these
// probes are all there is, keep them in L1 (34 % hits; without: -40 %).
template <bool G, bool NA = true>
__device__ __forceinline__ std::uint32_t pert53_hi_word(const std::uint8_t* pfast, std::uint32_t c) {
  if constexpr (G && kPert53h) {
    if constexpr (NA && PBN_PERT_NOALLOC != 0) {
      std::uint32_t v;
      asm("ld.global.nc.L1::no_allocate.u32 %0, [%1];"
          : "=r"(v)
          : "l"(reinterpret_cast<const std::uint32_t*>(pfast) + c));
      return v;
    } else {
      return __ldg(reinterpret_cast<const std::uint32_t*>(pfast) + c);
    }
  } else {
    return ldp<G>(reinterpret_cast<const std::uint32_t*>(pfast) + 2 * c + 1);
  }
}
// The full 8-byte U53 cells (the exact paths): not kept in a register by G
// launches (the header and the blob pointer are kernel parameters).
template <bool G>
__device__ __forceinline__ const std::uint64_t* pert53_cells(const std::uint8_t* pfast,
                                                             const std::uint8_t* gblob,
                                                             const dev_plan_header& h) {
  if constexpr (G && kPert53h)
    return reinterpret_cast<const std::uint64_t*>(gblob + h.off_pert53);
  else
    return reinterpret_cast<const std::uint64_t*>(pfast);
}
// Perturbation cell lookup (alias.hpp:70-76 with N = 2^k), integer form on
// the raw draw word R = hi << 32 | lo: the cell index is the top k bits, the
// threshold compare runs on the remaining 64-k bits (dev_plan.h pert53).
// Fast form on the high word alone: decided unless its 32-k compare bits tie
// with the cell's (`rare`; pert_draw53_exact then needs the low word).
template <bool G>
__device__ __forceinline__ std::uint32_t pert_draw53_hi(const std::uint8_t* pfast, std::uint32_t hi,
                                                        std::uint32_t k, bool& rare) {
  const std::uint32_t c = hi >> (32 - k);
  const std::uint32_t hmask = 0xFFFFFFFFu >> k;
  const std::uint32_t ehi = pert53_hi_word<G>(pfast, c);
  const std::uint32_t a = hi & hmask, b = ehi & hmask;
  rare = rare || a == b;
  return a < b ? c : (ehi >> (32 - k));
}
__device__ __forceinline__ std::uint32_t pert_draw53_exact(const std::uint64_t* cells, raw53 r,
                                                           std::uint32_t k) {
  const std::uint32_t c = r.hi >> (32 - k);
  const std::uint32_t hmask = 0xFFFFFFFFu >> k;
  const std::uint64_t e = cells[c];  // generic load: smem or global
  const std::uint32_t ehi = static_cast<std::uint32_t>(e >> 32);
  const std::uint64_t rl = (static_cast<std::uint64_t>(r.hi & hmask) << 32) | r.lo;
  const std::uint64_t el = (static_cast<std::uint64_t>(ehi & hmask) << 32) | static_cast<std::uint32_t>(e);
  return rl < el ? c : (ehi >> (32 - k));
}

// One phase-A draw (engine.hpp:257-266) from its high word hw: the
// perturbation pattern, or (BERN, node-wise plans) 1 iff u < p (engine.hpp:198).
// U53 fast form (exact = false) sets `rare` when the high word ties with the
// threshold; the exact form then decides with the low word lo. U32: lo = 0,
// never rare.
template <int STREAM, bool G, bool BERN>
__device__ __forceinline__ std::uint32_t pa_draw(const dev_plan_header& h,
                                                 const std::uint8_t* gblob,
                                                 const std::uint8_t* pfast, std::uint32_t k,
                                                 std::uint32_t hw, bool exact, std::uint32_t lo,
                                                 bool& rare);
// The leaf draw (engine.hpp:268, reduction.hpp:98): u > t.
template <int STREAM>
__device__ __forceinline__ bool pa_leaf(const dev_plan_header& h, std::uint32_t hw, bool exact,
                                        std::uint32_t lo, bool& rare) {
  if constexpr (STREAM == STREAM_U53) {
    if (exact) return ((static_cast<std::uint64_t>(hw) << 32) | lo) > h.leaf_thr53;
    const std::uint32_t th = static_cast<std::uint32_t>(h.leaf_thr53 >> 32);
    rare = rare || hw == th;
    return hw > th;
  } else {
    return !h.leaf_never && hw > h.leaf_thr32;
  }
}

template <bool G>
__device__ __forceinline__ std::uint32_t pert_draw32(const std::uint32_t* cells, std::uint32_t r,
                                                     std::uint32_t k) {
  const std::uint32_t c = r >> (32 - k);
  const std::uint32_t lmask = (1u << (32 - k)) - 1;
  const std::uint32_t e = ldp<G>(cells + c);
  return (r & lmask) < (e & lmask) ? c : (e >> (32 - k));
}

template <int STREAM, bool G, bool BERN>
__device__ __forceinline__ std::uint32_t pa_draw(const dev_plan_header& h,
                                                 const std::uint8_t* gblob,
                                                 const std::uint8_t* pfast, std::uint32_t k,
                                                 std::uint32_t hw, bool exact, std::uint32_t lo,
                                                 bool& rare) {
  if constexpr (BERN) {
    if constexpr (STREAM == STREAM_U53) {
      if (exact) return ((static_cast<std::uint64_t>(hw) << 32) | lo) < h.pthr53 ? 1u : 0u;
      const std::uint32_t ph = static_cast<std::uint32_t>(h.pthr53 >> 32);
      rare = rare || hw == ph;
      return hw < ph ? 1u : 0u;
    } else {
      return hw < h.pthr32 ? 1u : 0u;
    }
  } else if constexpr (STREAM == STREAM_U53) {
    if (exact) return pert_draw53_exact(pert53_cells<G>(pfast, gblob, h), raw53{hw, lo}, k);
    return pert_draw53_hi<G>(pfast, hw, k, rare);
  } else {
    return pert_draw32<G>(reinterpret_cast<const std::uint32_t*>(pfast), hw, k);
  }
}

// Gather 4 parent bits (records r0..r3 packed in two words) into slots b0..b0+3.
__device__ __forceinline__ std::uint32_t gather4(const std::uint32_t* S, std::uint32_t p01,
                                                 std::uint32_t p23, std::uint32_t b0) {
  const std::uint32_t r0 = p01 & 0xFFFFu, r1 = p01 >> 16, r2 = p23 & 0xFFFFu, r3 = p23 >> 16;
  const std::uint32_t w0 = S[r0 >> 5], w1 = S[r1 >> 5], w2 = S[r2 >> 5], w3 = S[r3 >> 5];
  return (__funnelshift_r(w0, w0, r0) & (1u << b0)) | (__funnelshift_r(w1, w1, r1) & (2u << b0)) |
         (__funnelshift_r(w2, w2, r2) & (4u << b0)) | (__funnelshift_r(w3, w3, r3) & (8u << b0));
}

// Same, with two state words per lane (1023 < n' <= 2047: word w lives in
// lane w & 31, register w >> 5): both registers are shuffled and bit 10 of
// the record (bit 5 of the word index) picks one.
__device__ __forceinline__ std::uint32_t gather4_shfl2(std::uint32_t wr0, std::uint32_t wr1,
                                                       std::uint32_t p01, std::uint32_t p23,
                                                       std::uint32_t b0) {
  auto get = [&](std::uint32_t rec) {
    const std::uint32_t a = __shfl_sync(0xFFFFFFFFu, wr0, rec >> 5);
    const std::uint32_t b = __shfl_sync(0xFFFFFFFFu, wr1, rec >> 5);
    return (rec & 0x400u) ? b : a;
  };
  const std::uint32_t w0 = get(p01), w1 = get(p01 >> 16), w2 = get(p23), w3 = get(p23 >> 16);
  return (__funnelshift_r(w0, w0, p01) & (1u << b0)) |
         (__funnelshift_r(w1, w1, p01 >> 16) & (2u << b0)) |
         (__funnelshift_r(w2, w2, p23) & (4u << b0)) |
         (__funnelshift_r(w3, w3, p23 >> 16) & (8u << b0));
}

// Same, with the state held in a lane's column of a [word][32 lanes] array
// (lane_ensemble.cu): word w of the lane's trajectory at col[32 * w], so
// record r's word is col[r & ~31] and 32 lanes hit 32 distinct banks.
__device__ __forceinline__ std::uint32_t gather4_col(const std::uint32_t* col, std::uint32_t p01,
                                                     std::uint32_t p23, std::uint32_t b0) {
  // byte offset of record r's word: (r & ~31) * 4; the funnel shifts use the
  // low 5 bits of the packed records directly
  const std::uint8_t* cb = reinterpret_cast<const std::uint8_t*>(col);
  auto at = [&](std::uint32_t off) { return *reinterpret_cast<const std::uint32_t*>(cb + off); };
  const std::uint32_t w0 = at((p01 << 2) & 0x3FF80u), w1 = at((p01 >> 14) & 0x3FF80u),
                      w2 = at((p23 << 2) & 0x3FF80u), w3 = at((p23 >> 14) & 0x3FF80u);
  return (__funnelshift_r(w0, w0, p01) & (1u << b0)) |
         (__funnelshift_r(w1, w1, p01 >> 16) & (2u << b0)) |
         (__funnelshift_r(w2, w2, p23) & (4u << b0)) |
         (__funnelshift_r(w3, w3, p23 >> 16) & (8u << b0));
}

// Same, with the state held one word per lane (n' <= 1023, LPT = 32): the
// parent word comes from a shuffle (the source lane index is taken mod 32, so
// the packed record needs no masking) instead of a shared-memory load.
__device__ __forceinline__ std::uint32_t gather4_shfl(std::uint32_t wreg, std::uint32_t p01,
                                                      std::uint32_t p23, std::uint32_t b0) {
  const std::uint32_t w0 = __shfl_sync(0xFFFFFFFFu, wreg, p01 >> 5);
  const std::uint32_t w1 = __shfl_sync(0xFFFFFFFFu, wreg, p01 >> 21);
  const std::uint32_t w2 = __shfl_sync(0xFFFFFFFFu, wreg, p23 >> 5);
  const std::uint32_t w3 = __shfl_sync(0xFFFFFFFFu, wreg, p23 >> 21);
  return (__funnelshift_r(w0, w0, p01) & (1u << b0)) |
         (__funnelshift_r(w1, w1, p01 >> 16) & (2u << b0)) |
         (__funnelshift_r(w2, w2, p23) & (4u << b0)) |
         (__funnelshift_r(w3, w3, p23 >> 16) & (8u << b0));
}

}  // namespace pbn_b200
