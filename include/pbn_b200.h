/*
 * pbn_b200.h — C-ABI of the B200-native PBN trajectory engine.
 *
 * This is the drop-in boundary for the reference's hot path
 * (arxiv 1605.00854 artifact, /root/reference/proj):
 *
 *   reference interface (header-level C++ templates)          replaced by
 *   ----------------------------------------------------------  ---------------------------
 *   pbn::parse_model            io.hpp:74-197                   pbn_model_parse
 *   pbn::serialize_model        io.hpp:205-226                  pbn_model_serialize
 *   pbn::validate               model.hpp:81-117                (inside pbn_model_parse)
 *   pbn::reduce / find_leaves   reduction.hpp:28-94             pbn_prepare (+ pbn_plan_reduced)
 *   pbn::perturbation_plan::build perturbation.hpp:25-43        pbn_prepare
 *   pbn::partition / combine    grouping.hpp:102-308            pbn_prepare
 *   pbn::prepare                engine.hpp:85-164               pbn_prepare + pbn_plan_get_view
 *   pbn::compile_predicate      engine.hpp:357-362              pbn_compile_predicate
 *   pbn::grouped_simulator::step engine.hpp:255-312  ┐
 *   pbn::simulate               engine.hpp:371-384  ┘           pbn_gpu_run / pbn_gpu_run_device
 *   pbn::estimate_steady_state  estimator.hpp:137-244           pbn_estimate (pooled ensemble)
 *
 * Conventions (mirroring the reference):
 *   - No C++ exception crosses this boundary. Every call returns a status code;
 *     the reference's exception classes map to the CLI's exit codes
 *     (errors.hpp:10-32, pbn_main.cpp:302-311):
 *       PBN_OK=0, PBN_EUSAGE=1, PBN_EMODEL=2 (model_error/parse_error),
 *       PBN_ERESOURCE=3 (resource_error), PBN_ECUDA=4 (device failure).
 *     pbn_last_error() returns the message of the last failure on this thread.
 *   - The plan is immutable after pbn_prepare and may be shared by threads
 *     (SPEC.md:411). A device handle (pbn_gpu) is used by one host thread.
 *   - States are bit-packed in ENGINE bit order, exactly the reference's
 *     `pbn::state` words (bitstate.hpp:12-99): bit i lives in 64-bit word i/64,
 *     each trajectory owns pbn_state_words(n_kept) = n_kept/64 + 1 words (the
 *     last one carries the always-zero slack bit).
 *   - Randomness is the injected counter-based stream described in DESIGN.md:
 *     Philox4x32-10, key = seed, counter = (trajectory, draw block, step).
 *     Draw d of step s of trajectory tau is a function of (seed, tau, s, d)
 *     only, so results are identical for any device count / launch split.
 */
#ifndef PBN_B200_H
#define PBN_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PBN_OK 0
#define PBN_EUSAGE 1
#define PBN_EMODEL 2
#define PBN_ERESOURCE 3
#define PBN_ECUDA 4

/* Random stream kinds (how a Philox block is cut into next_double() values). */
#define PBN_STREAM_U53 0 /* 4 draws per block position b: ((H[e]<<32|L[e]) >> 11) * 2^-53 (rng.hpp:35),
                            H = Philox block b, L = Philox block b | 2^31          */
#define PBN_STREAM_U32 1 /* 4 draws per Philox block: x[e] * 2^-32 (fast stream)                      */

/* Per-trajectory statistics record, PBN_COUNT_FIELDS uint64 each. */
#define PBN_COUNT_FIELDS 8
#define PBN_C_STEPS 0      /* steps simulated in this call                                   */
#define PBN_C_HITS 1       /* steps whose post-step state satisfies the predicate (engine.hpp:380) */
#define PBN_C_T00 2        /* predicate-process transitions prev->cur: 0->0                 */
#define PBN_C_T01 3        /*                                          0->1                 */
#define PBN_C_T10 4        /*                                          1->0                 */
#define PBN_C_T11 5        /*                                          1->1                 */
#define PBN_C_FNSTEPS 6    /* steps that ran the function phase (no kept flip, leaf check passed) */
#define PBN_C_PERTSTEPS 7  /* steps with at least one kept-node flip (engine.hpp:267)        */

/* Run flags. */
#define PBN_RUN_NODE_COUNTS 1u /* also accumulate per-bit one-counts (engine.hpp:378-379) */
#define PBN_RUN_EXACT_ALIAS 2u /* U53: every combined-function choice in FP64 (no integer fast
                                  path); same results, for cross-checking the fast path */

/* Opaque handles. */
typedef struct pbn_model pbn_model; /* parsed + validated model           (model.hpp:57-69)  */
typedef struct pbn_plan pbn_plan;   /* prepared simulation (flat plan)    (engine.hpp:22-79) */
typedef struct pbn_gpu pbn_gpu;     /* device-resident encoded plan                           */

/*
 * Flat view of a prepared simulation: the hot-loop arrays of the reference's
 * prepared_simulation (engine.hpp:22-79), one plain array per field.
 * Any producer may fill it — pbn_plan_get_view() for plans built by this
 * library, or a reference-side shim over pbn::prepared_simulation
 * — and pbn_gpu_create() accepts either.
 */
typedef struct pbn_plan_view {
  uint32_t n_kept;          /* reduced node count n'                       (engine.hpp:75)   */
  double t;                 /* leaf no-perturb probability (1-p)^l         (reduction.hpp:91) */
  /* perturbation plan (perturbation.hpp:16-44) */
  uint32_t pert_groups;     /* g                                                            */
  uint32_t pert_k;          /* k                                                            */
  uint32_t pert_k_prime;    /* k'                                                           */
  uint32_t pert_size;       /* 2^k alias cells                                              */
  uint64_t pert_mask;       /* 2^k' - 1                                                     */
  const double* pert_cut;   /* [pert_size] alias cut-offs                  (alias.hpp:95)    */
  const uint32_t* pert_alias; /* [pert_size] alias targets                 (alias.hpp:96)    */
  /* groups in engine order (engine.hpp:29-36) */
  uint32_t n_groups;
  const uint32_t* grp_offset;      /* [n_groups] cum[i]                                      */
  const uint32_t* grp_fn_begin;    /* [n_groups] first combined function in fns              */
  const uint32_t* grp_alias_begin; /* [n_groups] into alias_cut / alias_idx                  */
  const uint32_t* grp_alias_size;  /* [n_groups] 0 when the group has one combined function  */
  /* flattened group alias tables (engine.hpp:40-41) */
  uint64_t n_alias;
  const double* alias_cut;
  const uint32_t* alias_idx;
  /* combined functions (engine.hpp:52-63) */
  uint32_t n_fns;
  const uint64_t* fn_gather_begin; /* [n_fns] into fn_gather                                 */
  const uint64_t* fn_table_begin;  /* [n_fns] into fn_tables, 2^gather_count entries         */
  const uint32_t* fn_gather_count; /* [n_fns]                                                */
  uint64_t n_gather;
  const uint32_t* fn_gather;       /* engine bit positions, lists padded to >= 8 with n_kept */
  uint64_t n_table;
  const uint64_t* fn_tables;       /* packed member outputs (member 0 = bit 0)               */
  /* Stepper kind. Grouped plans (pbn_prepare): pert_mode 0 (g pattern draws
   * through the 2^k alias cells), has_leaf 1 — REQUIRED: the grouped stepper
   * always makes the leaf draw (engine.hpp:268), so pbn_gpu_create rejects
   * pert_mode 0 with has_leaf 0 (PBN_EUSAGE) — grp_members NULL (member counts
   * follow from the offsets). Node-wise plans (pbn_prepare_nodewise, the
   * reference's Method_old / Method_reduction steppers, engine.hpp:168-242):
   * pert_mode 1 (g = n per-node Bernoulli(pert_p) draws, flip iff u < p),
   * has_leaf 0 (Method_old) or 1 (Method_reduction), one group per node at
   * offset = node index (multi-function nodes first), grp_members all 1. */
  uint32_t pert_mode;
  uint32_t has_leaf;
  double pert_p;
  const uint32_t* grp_members;     /* [n_groups] or NULL                                     */
} pbn_plan_view;

/* BASELINE-shaped synthetic network. */
typedef struct pbn_gen_params {
  uint32_t n;              /* nodes                                                         */
  uint32_t f_min, f_max;   /* predictor functions per node ~ U{f_min..f_max}                */
  uint32_t p_min, p_max;   /* parents per function ~ U{p_min..p_max} (distinct, sorted)     */
  double leaf_frac;        /* designated leaves (never drawn as parents)                    */
  double perturbation;     /* p                                                             */
  uint32_t n_targets;      /* interest / predicate nodes (never designated leaves)          */
  uint32_t targets_fixed;  /* 1: targets are nodes 0..n_targets-1 with value 1 (config 1)   */
  uint64_t seed;
} pbn_gen_params;

/* Run arguments of one ensemble launch. */
typedef struct pbn_run_args {
  uint64_t seed;
  uint64_t traj_begin;   /* global id of the first trajectory (keys the stream)            */
  uint32_t n_traj;
  uint32_t stream;       /* PBN_STREAM_*                                                   */
  uint64_t step_begin;   /* global index of the first step (resumable runs)                */
  uint64_t n_steps;
  const uint32_t* pred_bits;  /* engine bits of the predicate terms (host)                 */
  const uint8_t* pred_vals;   /* wanted values                                              */
  uint32_t n_pred;            /* 0 = no predicate (hits/transitions stay 0)                */
  uint32_t flags;             /* PBN_RUN_*                                                  */
  /* Predicate-process transitions (estimator.hpp:76-102) are counted between
   * samples taken every `kappa`-th step of the call (0 or 1: every step). The
   * first "previous" sample is the input state's predicate with sampling
   * phase 0 (thin_mode 0), carried over with its phase from tprev[traj] =
   * prev | phase << 2 (1; prev 2 = none), or none (2). tprev (n_traj bytes) is
   * updated when non-NULL. kappa <= 63. */
  uint32_t kappa;
  uint32_t thin_mode;
  uint8_t* tprev;
  /* Optional predicate series: step i -> bit series_bit0 + i of the
   * trajectory's row of series_stride u32 words; series_init also records the
   * input state's bit at series_bit0 - 1. (pbn_gpu_run: host pointers, copied;
   * pbn_gpu_run_device: device pointers.) */
  uint32_t* series;
  uint64_t series_stride;
  uint64_t series_bit0;
  uint32_t series_init;
  uint32_t reserved;
} pbn_run_args;

/* ---- errors / library info ------------------------------------------------- */
const char* pbn_last_error(void);
const char* pbn_version(void);
uint32_t pbn_state_words(uint32_t n_kept); /* n_kept/64 + 1 (bitstate.hpp:19) */

/* ---- model (io.hpp / model.hpp / own generator) ---------------------------- */
int pbn_model_parse(const char* text, size_t len, pbn_model** out);
int pbn_model_serialize(const pbn_model* m, char* buf, size_t cap, size_t* len_out);
int pbn_model_generate(const pbn_gen_params* gp, pbn_model** out, uint32_t* pred_nodes,
                       uint8_t* pred_vals, uint32_t* n_pred_out);
int pbn_model_info(const pbn_model* m, uint32_t* n, double* p, uint32_t* n_interest,
                   double* density);
int pbn_model_node_index(const pbn_model* m, const char* name, uint32_t* index_out);
/* Node name i into buf (NUL-terminated, truncated to cap); *len_out = full length. */
int pbn_model_node_name(const pbn_model* m, uint32_t i, char* buf, size_t cap, size_t* len_out);
void pbn_model_free(pbn_model* m);

/* ---- preparation (reduction.hpp, perturbation.hpp, grouping.hpp, engine.hpp:85) ---- */
int pbn_prepare(const pbn_model* m, uint64_t theta, uint32_t k_max, uint32_t max_group_parents,
                pbn_plan** out);
/* Node-wise plan of the reference's node-by-node steppers: reduced = 0 ->
 * reference_simulator on the full model (engine.hpp:168-221); reduced = 1 ->
 * reduced_simulator on the leaf-reduced model (engine.hpp:225-242). */
int pbn_prepare_nodewise(const pbn_model* m, int reduced, pbn_plan** out);
int pbn_plan_get_view(const pbn_plan* plan, pbn_plan_view* view); /* valid while plan lives */
/* Reduction bookkeeping: original n, removed count, index_map[n] (-1 removed),
 * engine_pos[n_kept] (reduced index -> engine bit). Arrays may be NULL. */
int pbn_plan_reduced(const pbn_plan* plan, uint32_t* original_n, uint32_t* n_removed,
                     int32_t* index_map, uint32_t* engine_pos, uint32_t* removed);
/* Group membership in engine order: members[n_kept] (reduced indices), cum[n_groups+1]. */
int pbn_plan_groups(const pbn_plan* plan, uint32_t* members, uint32_t* cum);
/* Predicate over ORIGINAL node indices -> engine bits (engine.hpp:357-362). */
int pbn_compile_predicate(const pbn_plan* plan, const uint32_t* nodes, const uint8_t* vals,
                          uint32_t n, uint32_t* engine_bits_out);
void pbn_plan_free(pbn_plan* plan);

/* ---- device engine ---------------------------------------------------------- */
int pbn_device_count(int* count);
/* Encode + upload a plan. lanes_per_traj: 0 = choose automatically, else 1,2,4,8,16,32. */
int pbn_gpu_create(const pbn_plan_view* view, int device, uint32_t lanes_per_traj,
                   pbn_gpu** out);
/* Force where the plan lives: 0 auto, 1 global (L1/L2), 2 core in smem, 3 core +
 * truth tables in smem, 4 everything (incl. perturbation cells) in smem, 5 core +
 * the perturbation cells in smem (tables through L1/L2).
 * PBN_ERESOURCE if it does not fit. pbn_gpu_info reports the level as
 * (placement code - 1): 0 global, 1 core, 2 tables, 3 all, 4 core + cells —
 * after a run, the level that run's launch actually used (a run steps down
 * when the ensemble's per-trajectory state does not fit next to the plan). */
int pbn_gpu_set_placement(pbn_gpu* g, uint32_t placement);
int pbn_gpu_info(const pbn_gpu* g, uint32_t* lanes_per_traj, uint32_t* tables_in_smem,
                 uint64_t* smem_bytes, uint64_t* plan_bytes, uint32_t* warps_per_cta);
/* End-to-end: HOST buffers. states_inout: n_traj * pbn_state_words(n_kept) uint64,
 * counts_out: n_traj * PBN_COUNT_FIELDS uint64, node_counts_out (flag NODE_COUNTS):
 * n_traj * n_kept uint64 one-counts of the call (engine.hpp:378-379), or NULL.
 * Synchronous. (pbn_gpu_run_device ADDS into d_node_counts.) */
int pbn_gpu_run(pbn_gpu* g, const pbn_run_args* a, uint64_t* states_inout, uint64_t* counts_out,
                uint64_t* node_counts_out);
/* Device-resident: DEVICE pointers, asynchronous on `stream` (a cudaStream_t, 0 = legacy). */
int pbn_gpu_run_device(pbn_gpu* g, const pbn_run_args* a, uint64_t* d_states,
                       uint64_t* d_counts, uint64_t* d_node_counts, void* stream);
/* Forced-draw replay — the device counterpart of the reference tests'
 * scripted_rng (tests/oracles.hpp:235-254; test_engine.cpp:89-153): trajectory
 * t consumes draws[t * n_draws + (i mod n_draws)], i = 0, 1, ..., in exactly
 * the reference's call order (engine.hpp:259-290: g perturbation draws; if no
 * kept node flipped the leaf draw; if it did not fire one draw per
 * multi-function group), for a->n_steps steps of a->n_traj trajectories
 * (a->seed / stream ignored; step_begin 0, no flags, carried samples or
 * series). The library lays the script out in the stream's (step, block)
 * slots with the reference's own FP64 rules and the SAME sub-warp kernel
 * source replays it (built with the draw blocks read from the script instead
 * of Philox). Decisions run on r53 = floor(u * 2^53): a draw that is not a
 * multiple of 2^-53 is accepted only if its rounding provably leaves the
 * decision it feeds unchanged, else PBN_EUSAGE names it. consumed_out[t]
 * (may be NULL) = draws trajectory t consumed (scripted_rng::consumed()).
 * HOST buffers; counts_out may be NULL. Grouped plans (pert_mode 0) only. */
int pbn_gpu_run_scripted(pbn_gpu* g, const pbn_run_args* a, const double* draws,
                         uint64_t n_draws, uint64_t* states_inout, uint64_t* counts_out,
                         uint64_t* consumed_out);
/* Stream known-answer hook: n Philox4x32-10 blocks of (4 x u32 counters) under key
 * = seed, computed by the device's Philox (tests compare with the oracle's). */
int pbn_philox_kat(const uint32_t* ctr, uint32_t n, uint64_t seed, uint32_t* out);
/* Launch count of the last run call (kernels launched). */
uint32_t pbn_gpu_last_launches(const pbn_gpu* g);
/* The kernel the last run launched, e.g.
 * "subwarp<lpt=32,gather=shfl_compact,stream=u53,place=tables,warps=28>" or
 * "lane<scan,stream=u53,place=all,warps=28>" (NUL-terminated into buf[cap];
 * *len_out = full length). */
int pbn_gpu_last_kernel(const pbn_gpu* g, char* buf, size_t cap, size_t* len_out);
/* The kernel a run of n_traj trajectories with `flags` would launch (same
 * format), without running: lets a test pin that it exercised the very
 * instantiation a benchmark of another ensemble size runs. */
int pbn_gpu_plan_launch(const pbn_gpu* g, uint32_t n_traj, uint32_t stream, uint32_t flags,
                        char* buf, size_t cap, size_t* len_out);
void pbn_gpu_destroy(pbn_gpu* g);

/* ---- device group: one ensemble over several GPUs ----------
 * The job's trajectories (global ids a->traj_begin .. + a->n_traj) are split
 * into contiguous per-rank ranges, one rank per device (rank r gets
 * n/R + (r < n%R) ids starting at r*(n/R) + min(r, n%R)); the plan is
 * replicated; the only collective is ONE ncclAllReduce (sum) of the pooled
 * counts (+ the pooled per-node one-counts with PBN_RUN_NODE_COUNTS) over
 * NVLink. Draws are keyed by global trajectory id, so every result is
 * identical for any device count. NCCL is bound at run time (libnccl.so.2);
 * without it the create calls return PBN_ERESOURCE.
 * Replaces: a caller looping simulate() (engine.hpp:371-384) over independent
 * trajectories and summing the results (pbn_main.cpp:230-240 runs one). */
typedef struct pbn_group pbn_group;
/* One process drives every device: devices[n_devices] (NULL: 0..n-1), ncclCommInitAll. */
int pbn_group_create(const pbn_plan_view* view, const int* devices, uint32_t n_devices,
                     uint32_t lanes_per_traj, pbn_group** out);
/* One process per device: rank `rank` of `nranks`; nccl_id = 128 bytes from
 * pbn_nccl_unique_id() on one rank, shared by the caller (MPI, a file, ...). */
int pbn_nccl_unique_id(uint8_t* nccl_id_out);
int pbn_group_create_rank(const pbn_plan_view* view, int device, uint32_t nranks, uint32_t rank,
                          const uint8_t* nccl_id, uint32_t lanes_per_traj, pbn_group** out);
int pbn_group_info(const pbn_group* gr, uint32_t* n_members, uint32_t* nranks,
                   uint32_t* first_rank);
/* The id range of rank `rank` for a job of n_total trajectories. */
int pbn_group_shard(const pbn_group* gr, uint64_t n_total, uint32_t rank, uint64_t* begin,
                    uint64_t* count);
/* Member i's engine (owned by the group), e.g. for pbn_gpu_info / last_kernel. */
int pbn_group_member(const pbn_group* gr, uint32_t i, pbn_gpu** eng);
/* Runs the whole job (collective: every rank calls it with the same args).
 * states_inout / counts_out (NULL allowed) hold THIS process's rows only —
 * the trajectories of its ranks, in global id order, row 0 = its first rank's
 * first trajectory. totals_out[PBN_COUNT_FIELDS] = job-wide pooled counts;
 * node_totals_out[n_kept] (iff PBN_RUN_NODE_COUNTS) = job-wide pooled
 * one-counts. No series / tprev (PBN_EUSAGE). Synchronous. */
int pbn_group_run(pbn_group* gr, const pbn_run_args* a, uint64_t* states_inout,
                  uint64_t* counts_out, uint64_t* totals_out, uint64_t* node_totals_out);
void pbn_group_destroy(pbn_group* gr);

/* ---- pooled ensemble steady-state estimate (estimator.hpp:137-244) ---------- */
typedef struct pbn_estimate_request {
  double precision;          /* r       (estimator.hpp:60) */
  double confidence;         /* 0.95    (estimator.hpp:61) */
  uint64_t pilot;            /* per-trajectory pilot steps (estimator.hpp:62) */
  double burn_epsilon;       /* 0 -> precision (estimator.hpp:63) */
  uint32_t max_refinements;  /* (estimator.hpp:64) */
  double sample_inflation;   /* 1.3 (estimator.hpp:68) */
  uint64_t seed;
  uint64_t traj_begin;
  uint32_t n_traj;
  uint32_t stream;
} pbn_estimate_request;

typedef struct pbn_estimate_result {
  double estimate;
  uint64_t sample_size_used; /* pooled recorded samples over all trajectories */
  uint64_t burn_in_used;     /* per trajectory */
  uint64_t steps_per_traj;   /* total steps simulated per trajectory */
  uint32_t kappa;
  uint32_t degenerate;
  double alpha, beta;
  double wall_seconds;
} pbn_estimate_result;

/* Device ensemble: req->n_traj trajectories (global ids traj_begin..), states
 * in/out on the host (n_traj * pbn_state_words words, engine order). */
int pbn_estimate(pbn_gpu* g, const pbn_estimate_request* req, const uint32_t* pred_bits,
                 const uint8_t* pred_vals, uint32_t n_pred, uint64_t* states_inout,
                 pbn_estimate_result* out);

/* The same estimator over a caller-supplied stepping backend (e.g. a CPU
 * restatement in tests): the host logic is backend-agnostic, like the
 * reference's estimate_steady_state<Stepper, Rng>. */
typedef struct pbn_estimator_backend {
  void* user;
  uint32_t n_traj;
  uint32_t reserved;
  uint64_t series_capacity; /* stored pilot bits per trajectory */
  /* advance every trajectory n_steps from step_begin; pooled counts into
   * totals[PBN_COUNT_FIELDS]; series_bit0 == UINT64_MAX: no series. 0 = ok */
  int (*run)(void* user, uint64_t step_begin, uint64_t n_steps, uint32_t kappa,
             uint32_t thin_mode, uint64_t series_bit0, uint32_t series_init, uint64_t* totals);
  /* pooled series statistics over positions [0, len): n_ijk[8], thinned pairs[4], ones */
  int (*series_stats)(void* user, uint32_t kappa, uint64_t len, uint64_t* out13);
} pbn_estimator_backend;
int pbn_estimate_with_backend(const pbn_estimate_request* req, const pbn_estimator_backend* be,
                              pbn_estimate_result* out);
int pbn_series_stats_host(const uint32_t* series, uint32_t n_traj, uint64_t stride, uint64_t len,
                          uint32_t kappa, uint64_t* out13);
/* Same over a DEVICE series buffer (distributed backends all-reduce out13). */
int pbn_series_stats_device(int device, const uint32_t* d_series, uint32_t n_traj, uint64_t stride,
                            uint64_t len, uint32_t kappa, uint64_t* out13);
double pbn_inverse_normal_cdf(double p);

/* ---- test hooks over host internals (grouping.hpp:50-82, alias.hpp:18-56) ---- */
uint32_t pbn_internal_lower_bound(const uint32_t* w, uint32_t n, uint64_t theta);
int pbn_internal_greedy_partition(const uint32_t* w, uint32_t n, uint32_t m, uint32_t* part_of);
int pbn_internal_alias_build(const double* probs, uint32_t n, double* cut, uint32_t* alias);
/* Device encoding of a plan without a device (test / sizing hook): out[] =
 * section offsets pert53, pert32, groups, fns, grec, acut, aidx, acell, arec,
 * scol, arec4, tables, fns_s, acell_s, then core_bytes, table_bytes,
 * blob_bytes (stageable), total bytes, A, A1, groups, sw32, rg_ok,
 * single_compact (first n_out of them). */
int pbn_internal_plan_layout(const pbn_plan_view* view, uint64_t* out, uint32_t n_out);
/* Integer form of the U53 combined-function choice (dev_plan.h a53) evaluated on
 * the host exactly as the kernel does it, fast path and boundary fallback, for
 * raw draw words R[i] = x[2e+1] << 32 | x[2e]; n <= 2048. Test hook. */
int pbn_internal_alias53_pick(const double* cut, const uint32_t* alias, uint32_t n,
                              const uint64_t* raw, uint64_t m, uint32_t* pick,
                              uint8_t* took_fast);

#ifdef __cplusplus
}
#endif
#endif /* PBN_B200_H */
