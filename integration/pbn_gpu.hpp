// integration/pbn_gpu.hpp — the reference-side binding of the B200 engine.
//
// What a maintainer of the reference (/root/reference/proj) adds next to its
// CLI (e.g. as tools/pbn_gpu.hpp) to run the hot path on the device: no
// reference header changes. It turns the reference's own plan
// (pbn::prepared_simulation, engine.hpp:22-79, built by pbn::prepare,
// engine.hpp:85-164) into the C-ABI's flat view and wraps the handle in the
// reference's call shape (simulate(grouped_simulator, ...), engine.hpp:371-384,
// for an ensemble of trajectories) with its exception classes
// (errors.hpp:10-32). INTEGRATION.md shows it; tests/test_integration_shim.py
// compiles it against the unmodified reference headers and checks it on the
// device against pbn::simulate(grouped_simulator) on the same stream.
//
// Link: -I<repo>/include -L<repo>/paper_1605_00854_b200 -lpbn_b200
#pragma once

#include <cstdint>
#include <stdexcept>
#include <vector>

#include "pbn/engine.hpp"
#include "pbn/errors.hpp"
#include "pbn_b200.h"

namespace pbn {

// Flat view of a reference plan. The per-group and per-function records are
// arrays of structs in the reference; the view wants one array per field, so
// they are split here (the big arrays — cut-offs, gather lists, tables — are
// passed by pointer). The view is valid while `ps` and this object live.
struct gpu_plan_view {
  std::vector<std::uint32_t> off, fnb, ab, asz, gcount;
  std::vector<std::uint64_t> gbeg, tbeg;
  pbn_plan_view v{};

  explicit gpu_plan_view(const prepared_simulation& ps) {
    for (const auto& ge : ps.exec) {  // engine.hpp:29-36
      off.push_back(ge.offset);
      fnb.push_back(ge.fn_begin);
      ab.push_back(ge.alias_begin);
      asz.push_back(ge.alias_size);
    }
    for (const auto& fe : ps.fns) {  // engine.hpp:54-58
      gbeg.push_back(fe.gather_begin);
      tbeg.push_back(fe.table_begin);
      gcount.push_back(fe.gather_count);
    }
    v.n_kept = ps.kept_count();
    v.t = ps.t();
    v.pert_groups = ps.pplan.groups;  // perturbation.hpp:16-21
    v.pert_k = ps.pplan.k;
    v.pert_k_prime = ps.pplan.k_prime;
    v.pert_mask = ps.pplan.mask;
    v.pert_size = static_cast<std::uint32_t>(ps.pplan.table.size());
    v.pert_cut = ps.pplan.table.cutoffs().data();  // alias.hpp:91-92
    v.pert_alias = ps.pplan.table.aliases().data();
    v.n_groups = static_cast<std::uint32_t>(off.size());
    v.grp_offset = off.data();
    v.grp_fn_begin = fnb.data();
    v.grp_alias_begin = ab.data();
    v.grp_alias_size = asz.data();
    v.n_alias = ps.alias_prob.size();  // engine.hpp:40-41
    v.alias_cut = ps.alias_prob.data();
    v.alias_idx = ps.alias_idx.data();
    v.n_fns = static_cast<std::uint32_t>(gbeg.size());
    v.fn_gather_begin = gbeg.data();
    v.fn_table_begin = tbeg.data();
    v.fn_gather_count = gcount.data();
    v.n_gather = ps.fn_gather.size();
    v.fn_gather = ps.fn_gather.data();
    v.n_table = ps.fn_tables.size();
    v.fn_tables = ps.fn_tables.data();
    // the grouped stepper: g pattern draws, then the leaf draw (engine.hpp:257-268)
    v.pert_mode = 0;
    v.has_leaf = 1;
    v.pert_p = 0.0;
    v.grp_members = nullptr;
  }
};

[[noreturn]] inline void gpu_throw(int rc) {
  if (rc == PBN_EMODEL) throw model_error(pbn_last_error());
  if (rc == PBN_ERESOURCE) throw resource_error(pbn_last_error());
  throw std::runtime_error(pbn_last_error());
}

// Ensemble counterpart of simulate(grouped_simulator&, state&, steps, rng):
// n_traj trajectories (global ids traj_begin..) advanced `steps` steps from
// step_begin on the injected Philox stream of `seed`. States are the
// reference's state words (state::data(), engine bit order), n_traj x
// (kept_count()/64 + 1) uint64; counts: n_traj x PBN_COUNT_FIELDS
// (steps, predicate hits — trajectory::predicate_hits, engine.hpp:380 —,
// predicate transitions, function-phase and perturbed step counts).
class gpu_ensemble {
 public:
  explicit gpu_ensemble(const prepared_simulation& ps, int device = 0,
                        std::uint32_t lanes_per_traj = 0)
      : view_(ps) {
    if (int rc = pbn_gpu_create(&view_.v, device, lanes_per_traj, &h_)) gpu_throw(rc);
  }
  ~gpu_ensemble() { pbn_gpu_destroy(h_); }
  gpu_ensemble(const gpu_ensemble&) = delete;
  gpu_ensemble& operator=(const gpu_ensemble&) = delete;

  void simulate(std::uint64_t seed, std::uint64_t traj_begin, std::uint32_t n_traj,
                std::uint64_t step_begin, std::uint64_t steps, const compiled_predicate& pred,
                std::uint64_t* states, std::uint64_t* counts,
                std::uint32_t stream = PBN_STREAM_U53) {
    std::vector<std::uint32_t> bits;
    std::vector<std::uint8_t> vals;
    for (const auto& [b, val] : pred) {  // engine.hpp:326 (engine bit, value) terms
      bits.push_back(b);
      vals.push_back(val ? 1 : 0);
    }
    pbn_run_args a{};
    a.seed = seed;
    a.traj_begin = traj_begin;
    a.n_traj = n_traj;
    a.stream = stream;
    a.step_begin = step_begin;
    a.n_steps = steps;
    a.pred_bits = bits.data();
    a.pred_vals = vals.data();
    a.n_pred = static_cast<std::uint32_t>(bits.size());
    if (int rc = pbn_gpu_run(h_, &a, states, counts, nullptr)) gpu_throw(rc);
  }

  pbn_gpu* handle() const { return h_; }

 private:
  gpu_plan_view view_;
  pbn_gpu* h_ = nullptr;
};

}  // namespace pbn
