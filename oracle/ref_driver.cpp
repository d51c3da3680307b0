// oracle/ref_driver.cpp — TEST INFRASTRUCTURE ONLY.
//
// A thin extern "C" driver over the UNMODIFIED reference library, compiled
// from the headers where they lie (/root/reference/proj/include, plus the
// reference's own test oracles in /root/reference/proj/tests/oracles.hpp) by
// oracle/Makefile into oracle/_ref/libpbnref.so. No reference source is
// copied into this repository.
//
// Uses:
//   * pins the oracle restatement and the product's host library
//     (plan byte-identity vs pbn::prepare, engine.hpp:85-164);
//   * runs pbn::grouped_simulator through the unchanged pbn::simulate
//     (engine.hpp:371-384) on the injected Philox stream;
//   * the CPU baseline: the reference stepper with its shipped xoshiro256
//     (rng.hpp) fanned out over host threads.
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "oracles.hpp"
#include "pbn/engine.hpp"
#include "pbn/estimator.hpp"
#include "pbn/exact.hpp"
#include "pbn/generate.hpp"
#include "pbn/io.hpp"
#include "pbn/rng.hpp"

#include "../include/pbn_b200.h"
#include "philox_stream.h"

namespace {

thread_local std::string g_err;
thread_local std::uint64_t g_last_estimate_steps = 0;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const pbn::resource_error& e) {
    g_err = e.what();
    return 3;
  } catch (const pbn::model_error& e) {
    g_err = e.what();
    return 2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

struct ref_plan {
  pbn::prepared_simulation ps;
  // split arrays for the flat view
  std::vector<std::uint32_t> off, fnb, ab, asz, gcount;
  std::vector<std::uint64_t> gbeg, tbeg;
};

// Rng adapter: next_double() = draw d of step s of trajectory tau (the Rng
// concept). begin_step() is called by the wrapper stepper.
struct philox_rng {
  orc_stream st;
  std::uint64_t next_step = 0;
  double next_double() { return orc_stream_next_double(&st); }
  std::uint64_t next_u64() { return orc_stream_raw(&st, st.d++); }
};

// Wrapper stepper: one begin_step per step, plus step-class and predicate
// transition bookkeeping around the reference's own step().
struct wrapped_stepper {
  pbn::grouped_simulator inner;
  const pbn::compiled_predicate* pred = nullptr;
  int prev = 0;
  std::uint64_t trans[2][2] = {{0, 0}, {0, 0}};
  std::uint64_t fn_steps = 0, pert_steps = 0;

  explicit wrapped_stepper(const pbn::prepared_simulation& ps) : inner(ps) {}
  std::uint32_t state_bits() const { return inner.state_bits(); }

  template <class Rng>
  void step(pbn::state& s, Rng& rng) {
    orc_stream_begin_step(&rng.st, rng.next_step++);
    inner.step(s, rng);
    const auto& ps = inner.prepared();
    const std::uint64_t used = rng.st.d;
    if (used == ps.pplan.groups) {
      ++pert_steps;
    } else {
      // the leaf draw was draw index g; the function phase ran iff !(u > t)
      const std::uint64_t r = orc_stream_raw(&rng.st, ps.pplan.groups);
      const double u = rng.st.kind == 0 ? (double)r * 0x1.0p-53 : (double)r * 0x1.0p-32;
      if (!(u > ps.t())) ++fn_steps;
    }
    if (pred) {
      const int cur = pbn::eval_predicate(*pred, s) ? 1 : 0;
      ++trans[prev][cur];
      prev = cur;
    }
  }
};

// Counts the steps an estimator drives through the reference stepper.
struct counting_stepper {
  pbn::grouped_simulator inner;
  std::uint64_t steps = 0;
  explicit counting_stepper(const pbn::prepared_simulation& ps) : inner(ps) {}
  std::uint32_t state_bits() const { return inner.state_bits(); }
  template <class Rng>
  void step(pbn::state& s, Rng& rng) {
    ++steps;
    inner.step(s, rng);
  }
};

// Node-by-node stepper with the per-step stream counter (Method_old / Method_reduction).
struct nodewise_stepper {
  pbn::reference_simulator* o;
  pbn::reduced_simulator* r;
  std::uint32_t bits;
  std::uint32_t state_bits() const { return bits; }
  template <class Rng>
  void step(pbn::state& st, Rng& rng) {
    orc_stream_begin_step(&rng.st, rng.next_step++);
    if (r)
      r->step(st, rng);
    else
      o->step(st, rng);
  }
};

void fill_view(ref_plan& rp, pbn_plan_view* v) {
  const auto& ps = rp.ps;
  std::memset(v, 0, sizeof *v);
  v->n_kept = ps.kept_count();
  v->t = ps.t();
  v->pert_groups = ps.pplan.groups;
  v->pert_k = ps.pplan.k;
  v->pert_k_prime = ps.pplan.k_prime;
  v->pert_mask = ps.pplan.mask;
  v->pert_size = ps.pplan.table.size();
  v->pert_cut = ps.pplan.table.cutoffs().data();
  v->pert_alias = ps.pplan.table.aliases().data();
  v->n_groups = static_cast<std::uint32_t>(ps.exec.size());
  v->grp_offset = rp.off.data();
  v->grp_fn_begin = rp.fnb.data();
  v->grp_alias_begin = rp.ab.data();
  v->grp_alias_size = rp.asz.data();
  v->n_alias = ps.alias_prob.size();
  v->alias_cut = ps.alias_prob.data();
  v->alias_idx = ps.alias_idx.data();
  v->n_fns = static_cast<std::uint32_t>(ps.fns.size());
  v->fn_gather_begin = rp.gbeg.data();
  v->fn_table_begin = rp.tbeg.data();
  v->fn_gather_count = rp.gcount.data();
  v->n_gather = ps.fn_gather.size();
  v->fn_gather = ps.fn_gather.data();
  v->n_table = ps.fn_tables.size();
  v->fn_tables = ps.fn_tables.data();
  v->pert_mode = 0;
  v->has_leaf = 1;
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

int ref_model_parse(const char* text, std::size_t len, void** out) {
  return guarded([&] { *out = new pbn::model(pbn::parse_model(std::string(text, len))); });
}

void ref_model_free(void* m) { delete static_cast<pbn::model*>(m); }

int ref_model_serialize(const void* m, char* buf, std::size_t cap, std::size_t* len) {
  return guarded([&] {
    const std::string s = pbn::serialize_model(*static_cast<const pbn::model*>(m));
    *len = s.size();
    if (buf && cap >= s.size()) std::memcpy(buf, s.data(), s.size());
  });
}

int ref_generate_random(std::uint32_t n, double density, double leaf_pct, std::uint32_t max_f,
                        std::uint32_t max_p, std::uint64_t seed, double p, void** out) {
  return guarded([&] {
    pbn::generator_params gp;
    gp.n = n;
    gp.target_density = density;
    gp.leaf_pct = leaf_pct;
    gp.max_functions = max_f;
    gp.max_parents = max_p;
    gp.seed = seed;
    gp.perturbation_rate = p;
    *out = new pbn::model(pbn::generate_random(gp));
  });
}

int ref_prepare(const void* m, std::uint64_t theta, std::uint32_t k, std::uint32_t mgp,
                void** out) {
  return guarded([&] {
    auto rp = std::make_unique<ref_plan>();
    rp->ps = pbn::prepare(*static_cast<const pbn::model*>(m), theta, k, mgp);
    for (const auto& ge : rp->ps.exec) {
      rp->off.push_back(ge.offset);
      rp->fnb.push_back(ge.fn_begin);
      rp->ab.push_back(ge.alias_begin);
      rp->asz.push_back(ge.alias_size);
    }
    for (const auto& fe : rp->ps.fns) {
      rp->gbeg.push_back(fe.gather_begin);
      rp->tbeg.push_back(fe.table_begin);
      rp->gcount.push_back(fe.gather_count);
    }
    *out = rp.release();
  });
}

void ref_plan_free(void* p) { delete static_cast<ref_plan*>(p); }

int ref_plan_view(void* p, pbn_plan_view* v) {
  return guarded([&] { fill_view(*static_cast<ref_plan*>(p), v); });
}

int ref_plan_reduced(const void* p, std::uint32_t* original_n, std::uint32_t* n_removed,
                     std::int32_t* index_map, std::uint32_t* engine_pos, std::uint32_t* removed) {
  return guarded([&] {
    const auto& ps = static_cast<const ref_plan*>(p)->ps;
    if (original_n) *original_n = ps.reduced.original_n;
    if (n_removed) *n_removed = static_cast<std::uint32_t>(ps.reduced.removed.size());
    if (index_map)
      std::memcpy(index_map, ps.reduced.index_map.data(), 4 * ps.reduced.index_map.size());
    if (engine_pos) std::memcpy(engine_pos, ps.engine_pos.data(), 4 * ps.engine_pos.size());
    if (removed)
      std::memcpy(removed, ps.reduced.removed.data(), 4 * ps.reduced.removed.size());
  });
}

int ref_plan_groups(const void* p, std::uint32_t* members, std::uint32_t* cum) {
  return guarded([&] {
    const auto& ps = static_cast<const ref_plan*>(p)->ps;
    std::size_t k = 0;
    for (const auto& g : ps.gplan.groups)
      for (auto v : g.members) members[k++] = v;
    for (std::size_t i = 0; i < ps.gplan.cum.size(); ++i) cum[i] = ps.gplan.cum[i];
  });
}

int ref_compile_predicate(const void* p, const std::uint32_t* nodes, const std::uint8_t* vals,
                          std::uint32_t n, std::uint32_t* bits) {
  return guarded([&] {
    const auto& ps = static_cast<const ref_plan*>(p)->ps;
    std::vector<pbn::predicate_term> pred;
    for (std::uint32_t i = 0; i < n; ++i) pred.push_back({nodes[i], vals[i] != 0});
    const auto cp = pbn::compile_predicate(pred, ps);
    for (std::uint32_t i = 0; i < n; ++i) bits[i] = cp[i].first;
  });
}

// pbn::simulate over the reference grouped stepper on the injected stream.
int ref_simulate_philox(void* p, std::uint64_t seed, std::uint64_t traj_begin,
                        std::uint32_t n_traj, int kind, std::uint64_t step_begin,
                        std::uint64_t n_steps, const std::uint32_t* pred_bits,
                        const std::uint8_t* pred_vals, std::uint32_t n_pred,
                        std::uint64_t* states, std::uint64_t* counts,
                        std::uint64_t* node_counts) {
  return guarded([&] {
    const auto& ps = static_cast<ref_plan*>(p)->ps;
    const std::uint32_t n = ps.kept_count();
    const std::uint32_t words = n / 64 + 1;
    pbn::compiled_predicate cp;
    for (std::uint32_t i = 0; i < n_pred; ++i) cp.emplace_back(pred_bits[i], pred_vals[i] != 0);
    for (std::uint32_t t = 0; t < n_traj; ++t) {
      pbn::state s(n);
      std::uint64_t* sw = states + static_cast<std::uint64_t>(t) * words;
      std::memcpy(s.data(), sw, 8 * words);
      wrapped_stepper ws(ps);
      if (n_pred) {
        ws.pred = &cp;
        ws.prev = pbn::eval_predicate(cp, s) ? 1 : 0;
      }
      philox_rng rng;
      orc_stream_init(&rng.st, seed, static_cast<std::uint32_t>(traj_begin + t), kind,
                      ps.pplan.groups + 1);
      rng.next_step = step_begin;
      pbn::sim_options opt;
      opt.count_nodes = node_counts != nullptr;
      opt.predicate = n_pred ? &cp : nullptr;
      const pbn::trajectory tr = pbn::simulate(ws, s, n_steps, rng, opt);
      std::memcpy(sw, s.data(), 8 * words);
      std::uint64_t* c = counts + static_cast<std::uint64_t>(t) * PBN_COUNT_FIELDS;
      c[PBN_C_STEPS] = tr.steps;
      c[PBN_C_HITS] = tr.predicate_hits;
      c[PBN_C_T00] = ws.trans[0][0];
      c[PBN_C_T01] = ws.trans[0][1];
      c[PBN_C_T10] = ws.trans[1][0];
      c[PBN_C_T11] = ws.trans[1][1];
      c[PBN_C_FNSTEPS] = ws.fn_steps;
      c[PBN_C_PERTSTEPS] = ws.pert_steps;
      if (node_counts)
        std::memcpy(node_counts + static_cast<std::uint64_t>(t) * n, tr.one_counts.data(), 8 * n);
    }
  });
}

// pbn::simulate over the node-by-node steppers on the injected stream:
// reduced = 0 -> reference_simulator on the full model (engine.hpp:168-221),
// reduced = 1 -> reduced_simulator on the leaf-reduced model (engine.hpp:225-242).
// Phase A of the stream = the n (resp. n' + 1 with the leaf draw) first draws.
int ref_simulate_nodewise(const void* mp, int reduced, std::uint64_t seed,
                          std::uint64_t traj_begin, std::uint32_t n_traj, int kind,
                          std::uint64_t step_begin, std::uint64_t n_steps,
                          const std::uint32_t* pred_bits, const std::uint8_t* pred_vals,
                          std::uint32_t n_pred, std::uint64_t* states, std::uint64_t* counts,
                          std::uint64_t* node_counts) {
  return guarded([&] {
    const pbn::model& m = *static_cast<const pbn::model*>(mp);
    const pbn::reduced_model rm = pbn::reduce(m);
    const std::uint32_t n = reduced ? rm.kept_count() : m.size();
    const std::uint32_t words = n / 64 + 1;
    pbn::compiled_predicate cp;
    for (std::uint32_t i = 0; i < n_pred; ++i) cp.emplace_back(pred_bits[i], pred_vals[i] != 0);
    pbn::reference_simulator old_sim(m);
    pbn::reduced_simulator red_sim(rm);
    for (std::uint32_t t = 0; t < n_traj; ++t) {
      pbn::state s(n);
      std::uint64_t* sw = states + static_cast<std::uint64_t>(t) * words;
      std::memcpy(s.data(), sw, 8 * words);
      nodewise_stepper w{&old_sim, reduced ? &red_sim : nullptr, n};
      philox_rng rng;
      orc_stream_init(&rng.st, seed, static_cast<std::uint32_t>(traj_begin + t), kind,
                      n + (reduced ? 1 : 0));
      rng.next_step = step_begin;
      pbn::sim_options opt;
      opt.count_nodes = node_counts != nullptr;
      opt.predicate = n_pred ? &cp : nullptr;
      const pbn::trajectory tr = pbn::simulate(w, s, n_steps, rng, opt);
      std::memcpy(sw, s.data(), 8 * words);
      std::uint64_t* c = counts + static_cast<std::uint64_t>(t) * PBN_COUNT_FIELDS;
      std::memset(c, 0, 8 * PBN_COUNT_FIELDS);
      c[PBN_C_STEPS] = tr.steps;
      c[PBN_C_HITS] = tr.predicate_hits;
      if (node_counts)
        std::memcpy(node_counts + static_cast<std::uint64_t>(t) * n, tr.one_counts.data(), 8 * n);
    }
  });
}

// One grouped_simulator::step on scripted uniforms (oracles.hpp:235-254).
int ref_step_scripted(void* p, std::uint64_t* state_words, const double* u, std::uint32_t n_u,
                      std::uint32_t* consumed) {
  return guarded([&] {
    const auto& ps = static_cast<ref_plan*>(p)->ps;
    pbn::grouped_simulator sim(ps);
    pbn::state s(ps.kept_count());
    const std::uint32_t words = ps.kept_count() / 64 + 1;
    std::memcpy(s.data(), state_words, 8 * words);
    oracles::scripted_rng rng(std::vector<double>(u, u + n_u));
    sim.step(s, rng);
    std::memcpy(state_words, s.data(), 8 * words);
    *consumed = static_cast<std::uint32_t>(rng.consumed());
  });
}

// CPU baseline: the reference grouped stepper with its shipped xoshiro256,
// one independent trajectory per std::thread, timing
// simulate() only. Returns wall seconds of the parallel region.
int ref_bench_xoshiro(void* p, std::uint64_t seed, std::uint32_t n_threads,
                      std::uint64_t steps_per_thread, const std::uint32_t* pred_bits,
                      const std::uint8_t* pred_vals, std::uint32_t n_pred, int method,
                      const void* model, double* seconds_out, std::uint64_t* hits_out) {
  return guarded([&] {
    const auto& ps = static_cast<ref_plan*>(p)->ps;
    pbn::compiled_predicate cp;
    for (std::uint32_t i = 0; i < n_pred; ++i) cp.emplace_back(pred_bits[i], pred_vals[i] != 0);
    std::atomic<std::uint32_t> ready{0};
    std::atomic<bool> go{false};
    std::vector<std::uint64_t> hits(n_threads, 0);
    std::vector<std::thread> th;
    for (std::uint32_t i = 0; i < n_threads; ++i) {
      th.emplace_back([&, i] {
        pbn::xoshiro256 rng(seed + i);
        pbn::sim_options opt;
        opt.count_nodes = false;  // bench.hpp:116-124
        opt.predicate = n_pred ? &cp : nullptr;
        if (method == 0) {
          pbn::grouped_simulator sim(ps);
          pbn::state s(sim.state_bits());
          ready.fetch_add(1);
          while (!go.load()) {
          }
          hits[i] = pbn::simulate(sim, s, steps_per_thread, rng, opt).predicate_hits;
        } else if (method == 1) {
          // Method_old on the full model (engine.hpp:168-221), no predicate mapping
          pbn::reference_simulator sim(*static_cast<const pbn::model*>(model));
          pbn::state s(sim.state_bits());
          opt.predicate = nullptr;
          ready.fetch_add(1);
          while (!go.load()) {
          }
          hits[i] = pbn::simulate(sim, s, steps_per_thread, rng, opt).steps;
        } else {
          // Method_reduction (engine.hpp:225-242) on the plan's reduced model
          pbn::reduced_simulator sim(ps.reduced);
          pbn::state s(sim.state_bits());
          opt.predicate = nullptr;
          ready.fetch_add(1);
          while (!go.load()) {
          }
          hits[i] = pbn::simulate(sim, s, steps_per_thread, rng, opt).steps;
        }
      });
    }
    while (ready.load() != n_threads) {
    }
    const auto t0 = std::chrono::steady_clock::now();
    go.store(true);
    for (auto& t : th) t.join();
    *seconds_out =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    std::uint64_t h = 0;
    for (auto x : hits) h += x;
    *hits_out = h;
  });
}

// The CPU reference on the GPU arm's ensemble shape: n_traj independent
// trajectories (all-zero initial states, pbn_main.cpp:232; xoshiro256 seeded
// seed + trajectory id), each advanced `steps` steps by the unmodified
// stepper, dealt round-robin to n_threads host threads (harness-level
// parallelism only; the plan is shared, const). method as ref_bench_xoshiro.
int ref_bench_ensemble(void* p, std::uint64_t seed, std::uint32_t n_threads,
                       std::uint32_t n_traj, std::uint64_t steps, const std::uint32_t* pred_bits,
                       const std::uint8_t* pred_vals, std::uint32_t n_pred, int method,
                       const void* model, double* seconds_out, std::uint64_t* hits_out) {
  return guarded([&] {
    const auto& ps = static_cast<ref_plan*>(p)->ps;
    pbn::compiled_predicate cp;
    for (std::uint32_t i = 0; i < n_pred; ++i) cp.emplace_back(pred_bits[i], pred_vals[i] != 0);
    std::atomic<std::uint32_t> ready{0};
    std::atomic<bool> go{false};
    std::vector<std::uint64_t> hits(n_threads, 0);
    std::vector<std::thread> th;
    for (std::uint32_t i = 0; i < n_threads; ++i) {
      th.emplace_back([&, i] {
        pbn::sim_options opt;
        opt.count_nodes = false;  // bench.hpp:116-124
        opt.predicate = (method == 0 && n_pred) ? &cp : nullptr;
        ready.fetch_add(1);
        while (!go.load()) {
        }
        std::uint64_t h = 0;
        for (std::uint32_t t = i; t < n_traj; t += n_threads) {
          pbn::xoshiro256 rng(seed + t);
          if (method == 0) {
            pbn::grouped_simulator sim(ps);
            pbn::state s(sim.state_bits());
            h += pbn::simulate(sim, s, steps, rng, opt).predicate_hits;
          } else if (method == 1) {
            pbn::reference_simulator sim(*static_cast<const pbn::model*>(model));
            pbn::state s(sim.state_bits());
            h += pbn::simulate(sim, s, steps, rng, opt).steps;
          } else {
            pbn::reduced_simulator sim(ps.reduced);
            pbn::state s(sim.state_bits());
            h += pbn::simulate(sim, s, steps, rng, opt).steps;
          }
        }
        hits[i] = h;
      });
    }
    while (ready.load() != n_threads) {
    }
    const auto t0 = std::chrono::steady_clock::now();
    go.store(true);
    for (auto& t : th) t.join();
    *seconds_out =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    std::uint64_t h = 0;
    for (auto x : hits) h += x;
    *hits_out = h;
  });
}

std::uint64_t ref_last_estimate_steps() { return g_last_estimate_steps; }

// Reference two-state estimator (estimator.hpp:137-244) on one trajectory.
// kind < 0: shipped xoshiro256(seed); else the Philox stream of trajectory traj.
int ref_estimate(void* p, const std::uint32_t* pred_nodes, const std::uint8_t* pred_vals,
                 std::uint32_t n_pred, double precision, double confidence, std::uint64_t pilot,
                 std::uint64_t seed, int kind, std::uint32_t traj, double* estimate,
                 std::uint64_t* sample_size, std::uint64_t* burn_in, int* degenerate) {
  return guarded([&] {
    const auto& ps = static_cast<ref_plan*>(p)->ps;
    std::vector<pbn::predicate_term> pred;
    for (std::uint32_t i = 0; i < n_pred; ++i) pred.push_back({pred_nodes[i], pred_vals[i] != 0});
    const auto cp = pbn::compile_predicate(pred, ps);
    pbn::estimation_request req;
    req.predicate = pred;
    req.precision = precision;
    req.confidence = confidence;
    req.pilot = pilot;
    pbn::state s(ps.kept_count());
    pbn::estimation_result r;
    if (kind < 0) {
      counting_stepper sim(ps);
      pbn::xoshiro256 rng(seed);
      r = pbn::estimate_steady_state(sim, s, cp, req, rng);
      g_last_estimate_steps = sim.steps;
    } else {
      wrapped_stepper ws(ps);
      philox_rng rng;
      orc_stream_init(&rng.st, seed, traj, kind, ps.pplan.groups + 1);
      r = pbn::estimate_steady_state(ws, s, cp, req, rng);
      g_last_estimate_steps = rng.next_step;
    }
    *estimate = r.estimate;
    *sample_size = r.sample_size_used;
    *burn_in = r.burn_in_used;
    *degenerate = r.degenerate ? 1 : 0;
  });
}

// Exact-chain helpers from the reference (exact.hpp) and its test oracles
// (oracles.hpp:71-155), for small-n distribution checks.
int ref_exact_matrix(const void* m, double t, double* out) {
  return guarded([&] {
    const auto mat = pbn::exact_transition_matrix(*static_cast<const pbn::model*>(m), t);
    std::memcpy(out, mat.data(), 8 * mat.size());
  });
}

int ref_grouped_row(void* p, std::uint64_t e, double* out) {
  return guarded([&] {
    const auto row = oracles::grouped_row(static_cast<ref_plan*>(p)->ps, e);
    std::memcpy(out, row.data(), 8 * row.size());
  });
}

int ref_marginal_exact(const void* m, const std::uint32_t* nodes, const std::uint8_t* vals,
                       std::uint32_t n, double* out) {
  return guarded([&] {
    std::vector<pbn::predicate_term> pred;
    for (std::uint32_t i = 0; i < n; ++i) pred.push_back({nodes[i], vals[i] != 0});
    *out = pbn::marginal_steady_state_exact(*static_cast<const pbn::model*>(m), pred);
  });
}

int ref_random_small_model(std::uint64_t seed, std::uint32_t n, double p, std::uint32_t max_f,
                           std::uint32_t max_p, void** out) {
  return guarded([&] {
    pbn::xoshiro256 rng(seed);
    *out = new pbn::model(oracles::random_small_model(rng, n, p, max_f, max_p));
  });
}

int ref_alias_build(const double* probs, std::uint32_t n, double* cut, std::uint32_t* alias) {
  return guarded([&] {
    const auto t = pbn::alias_table::build(std::span<const double>(probs, n));
    std::memcpy(cut, t.cutoffs().data(), 8 * n);
    std::memcpy(alias, t.aliases().data(), 4 * n);
  });
}

double ref_inverse_normal_cdf(double p) { return pbn::inverse_normal_cdf(p); }

}  // extern "C"
