// Philox4x32-10 for the trajectory kernels (Salmon et al., SC'11).
//
// Counter layout: c = (trajectory, draw block,
// step lo32, step hi32), key = seed; U53 low words come from the blocks
// b | kLoBlock. Within one step only the draw block
// changes, so the first round is two XORs and the second round one 32x32
// multiply: `step_philox` carries the block-independent parts, computed once
// per step, and `block()` runs the remaining ~8.5 rounds.
#pragma once

#include <cstdint>

namespace pbn_b200 {

constexpr std::uint32_t kPhiloxM0 = 0xD2511F53u;
constexpr std::uint32_t kPhiloxM1 = 0xCD9E8D57u;
// U53 draws are split over two blocks: draw e of block b takes
// its high word from block b and its low word from block b | kLoBlock. Every
// decision of the kernels is made by the high word alone except on a tie
// (about 2^-16 of perturbation draws at k = 16, ~N * 2^-32 of selections), so
// the low blocks are computed only in those rare paths.
constexpr std::uint32_t kLoBlock = 0x80000000u;

struct step_philox {
  std::uint32_t a;   // hi(M1*step_lo) ^ k0[0]        -> round-1 c0 = a ^ block
  std::uint32_t b2;  // lo(M0*traj) ^ k1[1]           -> round-2 c2 = hi(M0*c0) ^ b2
  std::uint32_t c0;  // round-2 output c0 (block-independent)
  std::uint32_t c1;  // round-2 output c1 (block-independent)
};

__device__ __forceinline__ void mulhilo(std::uint32_t m, std::uint32_t x, std::uint32_t& hi,
                                        std::uint32_t& lo) {
  const std::uint64_t p = static_cast<std::uint64_t>(m) * x;
  hi = static_cast<std::uint32_t>(p >> 32);
  lo = static_cast<std::uint32_t>(p);
}

// traj_hi0/traj_lo0 = M0 * traj, computed once per trajectory.
__device__ __forceinline__ step_philox make_step_philox(std::uint32_t traj_hi0,
                                                        std::uint32_t traj_lo0,
                                                        std::uint64_t step,
                                                        const std::uint32_t* rk0,
                                                        const std::uint32_t* rk1) {
  step_philox sp;
  std::uint32_t hi1, lo1;
  mulhilo(kPhiloxM1, static_cast<std::uint32_t>(step), hi1, lo1);
  // round 1: c0' = hi1 ^ block ^ k0, c1' = lo1, c2' = hi0 ^ step_hi ^ k1, c3' = lo0
  sp.a = hi1 ^ rk0[0];
  const std::uint32_t c2r1 = traj_hi0 ^ static_cast<std::uint32_t>(step >> 32) ^ rk1[0];
  // round 2: products M0*c0' (block-dependent) and M1*c2' (block-independent)
  std::uint32_t hi1b, lo1b;
  mulhilo(kPhiloxM1, c2r1, hi1b, lo1b);
  sp.c0 = hi1b ^ lo1 ^ rk0[1];
  sp.c1 = lo1b;
  sp.b2 = traj_lo0 ^ rk1[1];
  return sp;
}

__device__ __forceinline__ uint4 philox_block(const step_philox& sp, std::uint32_t block,
                                              const std::uint32_t* rk0,
                                              const std::uint32_t* rk1) {
  std::uint32_t hi0, lo0;
  mulhilo(kPhiloxM0, sp.a ^ block, hi0, lo0);
  std::uint32_t c0 = sp.c0, c1 = sp.c1, c2 = hi0 ^ sp.b2, c3 = lo0;
#pragma unroll
  for (int r = 2; r < 10; ++r) {
    std::uint32_t h0, l0, h1, l1;
    mulhilo(kPhiloxM0, c0, h0, l0);
    mulhilo(kPhiloxM1, c2, h1, l1);
    c0 = h1 ^ c1 ^ rk0[r];
    c1 = l1;
    c2 = h0 ^ c3 ^ rk1[r];
    c3 = l0;
  }
  return make_uint4(c0, c1, c2, c3);
}

// Plain reference form (all ten rounds), for the known-answer test kernel.
__device__ __forceinline__ uint4 philox4x32_10(uint4 c, std::uint32_t k0, std::uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    std::uint32_t h0, l0, h1, l1;
    mulhilo(kPhiloxM0, c.x, h0, l0);
    mulhilo(kPhiloxM1, c.z, h1, l1);
    c = make_uint4(h1 ^ c.y ^ k0, l1, h0 ^ c.w ^ k1, l0);
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return c;
}

}  // namespace pbn_b200
