/*
 * oracle/philox_stream.h — TEST INFRASTRUCTURE ONLY (the checker, never the product).
 *
 * The injected random stream both the reference stepper (through the adapter in
 * oracle/ref_driver.cpp) and the oracle restatement (oracle/pbn_oracle.c) consume.
 * The product (paper_1605_00854_b200/csrc/device/philox.cuh) has its own,
 * independent implementation; tests compare the two.
 *
 * Philox4x32-10 (Salmon et al., SC'11; constants as in curand_philox4x32_x.h):
 *   round: (hi0,lo0)=M0*c0, (hi1,lo1)=M1*c2, c = {hi1^c1^k0, lo1, hi0^c3^k1, lo0}
 *   key bump between rounds: k0 += 0x9E3779B9, k1 += 0xBB67AE85
 *
 * Stream layout:
 *   key     = (seed lo32, seed hi32)
 *   counter = (trajectory tau, draw block b, step lo32, step hi32)
 *   4 draws per block position b, draw e in {0..3}:
 *   U53: ((H[e] << 32 | L[e]) >> 11) * 2^-53 with H = block b, L = block
 *        b | 0x80000000 ("low block") — the same 53-bit conversion as
 *        xoshiro256::next_double (rng.hpp:35) of the 64-bit word H:L
 *   U32: H[e] * 2^-32
 *   Within a step the draws come in two phases (engine.hpp:255-312):
 *     phase A = the perturbation draws and the leaf draw (g + 1 draws for the
 *               grouped stepper; n for Method_old, n' + 1 for Method_reduction):
 *               draw d lives in block d / DPB at position d % DPB;
 *     phase B = the function-selection draws, j = d - g1 (g1 = phase-A draws):
 *               block NB0 + j / DPB, position j % DPB, NB0 = ceil(g1 / DPB),
 *     i.e. phase B starts on a fresh block, so the device can prefetch its
 *     draws in whole blocks. g is the plan's perturbation group count.
 */
#ifndef PBN_ORACLE_PHILOX_STREAM_H
#define PBN_ORACLE_PHILOX_STREAM_H

#include <stdint.h>

static inline void orc_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2],
                                     uint32_t out[4]) {
  uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
  uint32_t k0 = key_in[0], k1 = key_in[1];
  for (int r = 0; r < 10; ++r) {
    const uint64_t p0 = (uint64_t)0xD2511F53u * c0;
    const uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
    const uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    const uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    c0 = hi1 ^ c1 ^ k0;
    c1 = lo1;
    c2 = hi0 ^ c3 ^ k1;
    c3 = lo0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  out[0] = c0;
  out[1] = c1;
  out[2] = c2;
  out[3] = c3;
}

/* Stream position of one trajectory: (seed, tau, step, d). */
typedef struct orc_stream {
  uint64_t seed;
  uint32_t traj;
  uint64_t step;
  uint64_t d;        /* draws consumed in the current step */
  int kind;          /* 0 = U53, 1 = U32 */
  uint64_t g1;       /* phase-A draws per step: g + 1 */
  uint64_t nb0;      /* first phase-B block: ceil(g1 / DPB) */
  uint64_t cached_block;
  int have_block;
  uint32_t x[4];  /* high block */
  uint32_t y[4];  /* low block (U53) */
} orc_stream;

/* g1 = number of phase-A draws per step: g + 1 for the grouped stepper (g
 * pattern draws + leaf draw), n for Method_old, n' + 1 for Method_reduction. */
static inline void orc_stream_init(orc_stream* s, uint64_t seed, uint32_t traj, int kind,
                                   uint32_t g1) {
  const uint64_t dpb = 4;
  (void)kind;
  s->g1 = g1;
  s->nb0 = (s->g1 + dpb - 1) / dpb;
  s->seed = seed;
  s->traj = traj;
  s->step = 0;
  s->d = 0;
  s->kind = kind;
  s->have_block = 0;
  s->cached_block = 0;
}

static inline void orc_stream_begin_step(orc_stream* s, uint64_t step) {
  s->step = step;
  s->d = 0;
  s->have_block = 0;
}

/* Raw draw d of the current step as an integer: r53 (U53) or r32 (U32). */
static inline uint64_t orc_stream_raw(orc_stream* s, uint64_t d) {
  const uint64_t dpb = 4;
  const uint64_t b = d < s->g1 ? d / dpb : s->nb0 + (d - s->g1) / dpb;
  const unsigned e = (unsigned)(d < s->g1 ? d % dpb : (d - s->g1) % dpb);
  if (!s->have_block || s->cached_block != b) {
    const uint32_t key[2] = {(uint32_t)s->seed, (uint32_t)(s->seed >> 32)};
    const uint32_t ctr[4] = {s->traj, (uint32_t)b, (uint32_t)s->step, (uint32_t)(s->step >> 32)};
    orc_philox4x32_10(ctr, key, s->x);
    if (s->kind == 0) {
      const uint32_t ctr_lo[4] = {s->traj, (uint32_t)b | 0x80000000u, (uint32_t)s->step,
                                  (uint32_t)(s->step >> 32)};
      orc_philox4x32_10(ctr_lo, key, s->y);
    }
    s->cached_block = b;
    s->have_block = 1;
  }
  if (s->kind == 0) return (((uint64_t)s->x[e] << 32) | s->y[e]) >> 11;
  return s->x[e];
}

/* next_double(): the Rng concept the reference steppers consume. */
static inline double orc_stream_next_double(orc_stream* s) {
  const uint64_t r = orc_stream_raw(s, s->d++);
  if (s->kind == 0) return (double)r * 0x1.0p-53;
  return (double)r * 0x1.0p-32;
}

#endif
