/*
 * oracle/pbn_oracle.c — TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference's structure-based stepper and its
 * trajectory loop, used by tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg as the CHECKER of the CUDA path. Nothing in the product
 * (paper_1605_00854_b200/) links or calls this file.
 *
 * Parity pin: tests/test_oracle_pins.py checks this restatement bit-for-bit
 * against the unmodified reference (oracle/_ref/libpbnref.so, compiled from
 * /root/reference/proj/include by oracle/Makefile) on the same injected stream.
 *
 * Compile with -ffp-contract=off: the alias draw's u*N - c must not contract
 * into an FMA (alias.hpp:72-75, engine.hpp:285-290).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "../include/pbn_b200.h"
#include "philox_stream.h"

/* xor_chunk / or_chunk of a <=64-bit chunk at a bit offset (bitstate.hpp:50-69). */
static void orc_xor_chunk(uint64_t* w, uint64_t c, uint32_t offset) {
  const uint32_t wi = offset >> 6, b = offset & 63;
  w[wi] ^= c << b;
  if (b != 0) {
    const uint64_t hi = c >> (64 - b);
    if (hi != 0) w[wi + 1] ^= hi;
  }
}

static void orc_or_chunk(uint64_t* w, uint64_t c, uint32_t offset) {
  const uint32_t wi = offset >> 6, b = offset & 63;
  w[wi] |= c << b;
  if (b != 0) {
    const uint64_t hi = c >> (64 - b);
    if (hi != 0) w[wi + 1] |= hi;
  }
}

static int orc_test(const uint64_t* w, uint32_t i) { return (int)((w[i >> 6] >> (i & 63)) & 1); }

/* Walker single-uniform draw (alias.hpp:70-76; engine.hpp:284-291). */
static uint32_t orc_alias_draw(double u01, uint32_t n, const double* cut, const uint32_t* alias) {
  const double u = u01 * (double)n;
  uint32_t c = (uint32_t)u;
  if (c >= n) c = n - 1;
  return (u - (double)c) < cut[c] ? c : alias[c];
}

/* Step outcome classes, for statistics. */
enum { ORC_PERTURBED = 1, ORC_LEAF = 2, ORC_FN = 3 };

/* One step of grouped_simulator::step (engine.hpp:255-312) on engine-order words. */
static int orc_grouped_step(const pbn_plan_view* v, uint64_t* s, uint64_t* next, uint32_t words,
                            orc_stream* rng) {
  int perturbed = 0;
  if (v->pert_mode == 1) { /* per-node Bernoulli flips (engine.hpp:190-202) */
    for (uint32_t i = 0; i < v->pert_groups; ++i)
      if (orc_stream_next_double(rng) < v->pert_p) {
        orc_xor_chunk(s, 1, i);
        perturbed = 1;
      }
  } else {
    for (uint32_t i = 0; i < v->pert_groups; ++i) { /* engine.hpp:257-266 */
      uint64_t c = orc_alias_draw(orc_stream_next_double(rng), v->pert_size, v->pert_cut,
                                  v->pert_alias);
      if (i + 1 == v->pert_groups) c &= v->pert_mask;
      if (c != 0) {
        orc_xor_chunk(s, c, i * v->pert_k);
        perturbed = 1;
      }
    }
  }
  if (perturbed) return ORC_PERTURBED;                            /* engine.hpp:267 */
  if (v->has_leaf && orc_stream_next_double(rng) > v->t)          /* engine.hpp:268, :237 */
    return ORC_LEAF;

  memset(next, 0, sizeof(uint64_t) * words);                      /* engine.hpp:270 */
  for (uint32_t gi = 0; gi < v->n_groups; ++gi) {
    uint32_t idx = 0;
    const uint32_t asz = v->grp_alias_size[gi];
    if (asz != 0) {                                               /* engine.hpp:283-291 */
      const uint32_t ab = v->grp_alias_begin[gi];
      idx = orc_alias_draw(orc_stream_next_double(rng), asz, v->alias_cut + ab, v->alias_idx + ab);
    }
    const uint32_t f = v->grp_fn_begin[gi] + idx;
    const uint32_t* gb = v->fn_gather + v->fn_gather_begin[f];
    const uint32_t cnt = v->fn_gather_count[f];
    uint64_t val = 0;                                             /* engine.hpp:292-302 */
    const uint32_t slots = cnt <= 8 ? 8 : cnt;
    for (uint32_t b = 0; b < slots; ++b) val |= (uint64_t)orc_test(s, gb[b]) << b;
    const uint64_t out = v->fn_tables[v->fn_table_begin[f] + val]; /* engine.hpp:303 */
    orc_or_chunk(next, out, v->grp_offset[gi]);                   /* engine.hpp:304-309 */
  }
  memcpy(s, next, sizeof(uint64_t) * words);                      /* engine.hpp:311 */
  return ORC_FN;
}

static int orc_pred(const uint64_t* s, const uint32_t* bits, const uint8_t* vals, uint32_t n) {
  for (uint32_t i = 0; i < n; ++i) /* eval_predicate, engine.hpp:328-332 */
    if (orc_test(s, bits[i]) != (vals[i] != 0)) return 0;
  return 1;
}

/*
 * simulate() (engine.hpp:371-384) for a block of trajectories, with the
 * trajectory-keyed stream and the extra statistics the ensemble reports:
 *   - hits: steps whose post-step state satisfies the predicate (engine.hpp:380);
 *   - transitions of the predicate process sampled every `kappa`-th step of
 *     the call (steps i with (i+1) % kappa == 0), between consecutive samples —
 *     the estimator's thinned_counts (estimator.hpp:76-102). thin_mode 0: the
 *     first "previous" sample is the input state's predicate (kappa = 1 gives
 *     the raw chain of estimator.hpp:155-170) and the sampling phase starts at
 *     0; 1: both continue from tprev[t] = prev | phase << 2 (prev 2 = none) of
 *     the previous call; 2: no previous sample, phase 0. tprev[t] is updated
 *     when non-NULL;
 *   - step classes (function phase ran / kept flip).
 * series (optional, stride words per trajectory): predicate bit of step i at
 * bit series_bit0 + i; if series_init, the input state's bit at series_bit0 - 1.
 * states_inout: n_traj * (n_kept/64+1) words. counts_out: n_traj * 8.
 * node_counts_out (optional): n_traj * n_kept.
 */
int orc_simulate_ex(const pbn_plan_view* v, uint64_t seed, uint64_t traj_begin, uint32_t n_traj,
                    int stream_kind, uint64_t step_begin, uint64_t n_steps,
                    const uint32_t* pred_bits, const uint8_t* pred_vals, uint32_t n_pred,
                    uint64_t* states_inout, uint64_t* counts_out, uint64_t* node_counts_out,
                    uint32_t kappa, int thin_mode, uint8_t* tprev, uint32_t* series,
                    uint64_t series_stride, uint64_t series_bit0, int series_init) {
  const uint32_t words = v->n_kept / 64 + 1;
  uint64_t* next = (uint64_t*)malloc(sizeof(uint64_t) * words);
  if (!next) return 3;
  if (kappa == 0) kappa = 1;
  if (kappa > 63) return 1; /* phase is carried in 6 bits */
  for (uint32_t t = 0; t < n_traj; ++t) {
    uint64_t* s = states_inout + (uint64_t)t * words;
    uint64_t* cnt = counts_out + (uint64_t)t * PBN_COUNT_FIELDS;
    uint64_t* nc = node_counts_out ? node_counts_out + (uint64_t)t * v->n_kept : 0;
    uint32_t* ser = series ? series + (uint64_t)t * series_stride : 0;
    memset(cnt, 0, sizeof(uint64_t) * PBN_COUNT_FIELDS);
    if (nc) memset(nc, 0, sizeof(uint64_t) * v->n_kept);
    orc_stream rng;
    orc_stream_init(&rng, seed, (uint32_t)(traj_begin + t), stream_kind,
                    v->pert_groups + (v->has_leaf ? 1 : 0));
    const int z0 = n_pred ? orc_pred(s, pred_bits, pred_vals, n_pred) : 0;
    int prev = 2;
    uint32_t phase = 0; /* steps since the last sample */
    if (thin_mode == 0) prev = z0;
    if (thin_mode == 1 && tprev) {
      prev = tprev[t] & 3;
      phase = tprev[t] >> 2;
    }
    if (ser && series_init && series_bit0 > 0 && z0)
      ser[(series_bit0 - 1) >> 5] |= 1u << ((series_bit0 - 1) & 31);
    for (uint64_t k = 0; k < n_steps; ++k) {
      orc_stream_begin_step(&rng, step_begin + k);
      const int cls = orc_grouped_step(v, s, next, words, &rng);
      if (cls == ORC_PERTURBED) cnt[PBN_C_PERTSTEPS]++;
      if (cls == ORC_FN) cnt[PBN_C_FNSTEPS]++;
      if (nc)
        for (uint32_t i = 0; i < v->n_kept; ++i) nc[i] += (uint64_t)orc_test(s, i);
      if (n_pred) {
        const int cur = orc_pred(s, pred_bits, pred_vals, n_pred);
        cnt[PBN_C_HITS] += (uint64_t)cur;
        if (ser && cur) ser[(series_bit0 + k) >> 5] |= 1u << ((series_bit0 + k) & 31);
        if (++phase == kappa) {
          phase = 0;
          if (prev != 2) cnt[PBN_C_T00 + 2 * prev + cur]++;
          prev = cur;
        }
      }
    }
    if (tprev) tprev[t] = (uint8_t)(prev | (phase << 2));
    cnt[PBN_C_STEPS] = n_steps;
  }
  free(next);
  return 0;
}

int orc_simulate(const pbn_plan_view* v, uint64_t seed, uint64_t traj_begin, uint32_t n_traj,
                 int stream_kind, uint64_t step_begin, uint64_t n_steps,
                 const uint32_t* pred_bits, const uint8_t* pred_vals, uint32_t n_pred,
                 uint64_t* states_inout, uint64_t* counts_out, uint64_t* node_counts_out) {
  return orc_simulate_ex(v, seed, traj_begin, n_traj, stream_kind, step_begin, n_steps, pred_bits,
                         pred_vals, n_pred, states_inout, counts_out, node_counts_out, 1, 0, 0, 0,
                         0, 0, 0);
}

/* Single forced step with an explicit list of uniforms (the scripted_rng
 * precedent, oracles.hpp:235-254): returns the number of draws consumed. */
int orc_step_scripted(const pbn_plan_view* v, uint64_t* s, const double* uniforms, uint32_t n_u,
                      uint32_t* consumed) {
  const uint32_t words = v->n_kept / 64 + 1;
  uint64_t* next = (uint64_t*)malloc(sizeof(uint64_t) * words);
  if (!next) return 3;
  uint32_t pos = 0;
  /* Same control flow as orc_grouped_step, fed from the script. */
  int perturbed = 0;
  for (uint32_t i = 0; i < v->pert_groups; ++i) {
    uint64_t c = orc_alias_draw(uniforms[pos++ % n_u], v->pert_size, v->pert_cut, v->pert_alias);
    if (i + 1 == v->pert_groups) c &= v->pert_mask;
    if (c != 0) {
      orc_xor_chunk(s, c, i * v->pert_k);
      perturbed = 1;
    }
  }
  if (!perturbed && !(uniforms[pos++ % n_u] > v->t)) {
    memset(next, 0, sizeof(uint64_t) * words);
    for (uint32_t gi = 0; gi < v->n_groups; ++gi) {
      uint32_t idx = 0;
      const uint32_t asz = v->grp_alias_size[gi];
      if (asz != 0) {
        const uint32_t ab = v->grp_alias_begin[gi];
        idx = orc_alias_draw(uniforms[pos++ % n_u], asz, v->alias_cut + ab, v->alias_idx + ab);
      }
      const uint32_t f = v->grp_fn_begin[gi] + idx;
      const uint32_t* gb = v->fn_gather + v->fn_gather_begin[f];
      const uint32_t cnt = v->fn_gather_count[f];
      uint64_t val = 0;
      const uint32_t slots = cnt <= 8 ? 8 : cnt;
      for (uint32_t b = 0; b < slots; ++b) val |= (uint64_t)orc_test(s, gb[b]) << b;
      orc_or_chunk(next, v->fn_tables[v->fn_table_begin[f] + val], v->grp_offset[gi]);
    }
    memcpy(s, next, sizeof(uint64_t) * words);
  }
  *consumed = pos;
  free(next);
  return 0;
}

/* Raw Philox block, exported for the known-answer tests. */
void orc_philox_block(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
  orc_philox4x32_10(ctr, key, out);
}

/* Draw d of (seed, traj, step) as a double for a plan with g perturbation
 * groups, exported for stream tests. */
double orc_draw(uint64_t seed, uint32_t traj, uint64_t step, uint64_t d, int kind, uint32_t g) {
  orc_stream s;
  orc_stream_init(&s, seed, traj, kind, g + 1);
  orc_stream_begin_step(&s, step);
  const uint64_t r = orc_stream_raw(&s, d);
  return kind == 0 ? (double)r * 0x1.0p-53 : (double)r * 0x1.0p-32;
}
