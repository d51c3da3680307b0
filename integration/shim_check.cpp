// integration/shim_check.cpp — TEST PROGRAM for the reference-side binding.
//
// Compiled (oracle/Makefile, target `shim`) against the UNMODIFIED reference
// headers and the C-ABI library, like a maintainer's build would compile
// integration/pbn_gpu.hpp; the binary lands in oracle/_ref/ (it needs
// /root/reference to build, and travels to the GPU box prebuilt).
//
//   shim_check MODEL THETA K MGP N_TRAJ STEPS SEED NODE=VAL[,NODE=VAL...] [--no-device]
//
// Reads a PBN text file with pbn::parse_model (io.hpp:74-197), plans it with
// pbn::prepare (engine.hpp:85-164), runs the ensemble on the device through
// pbn::gpu_ensemble, then runs every trajectory through the reference's own
// pbn::simulate(grouped_simulator, ...) (engine.hpp:371-384) with an Rng that
// serves the same injected Philox stream (oracle/philox_stream.h), and compares
// final states and predicate hits bit for bit. --no-device: only builds the
// view and checks that pbn_gpu_create accepts it (it fails with PBN_ECUDA for
// want of a GPU, after validating and encoding the plan).
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <sstream>
#include <string>
#include <vector>

#include "../integration/pbn_gpu.hpp"
#include "../oracle/philox_stream.h"
#include "pbn/io.hpp"

namespace {

// The Rng concept the reference steppers consume (next_double only).
struct philox_rng {
  orc_stream st;
  double next_double() { return orc_stream_next_double(&st); }
};

// One begin_step per step around the reference's own step() (the stream is
// keyed by the step index).
struct stepping {
  pbn::grouped_simulator inner;
  std::uint64_t next_step = 0;
  explicit stepping(const pbn::prepared_simulation& ps) : inner(ps) {}
  std::uint32_t state_bits() const { return inner.state_bits(); }
  void step(pbn::state& s, philox_rng& rng) {
    orc_stream_begin_step(&rng.st, next_step++);
    inner.step(s, rng);
  }
};

}  // namespace

int main(int argc, char** argv) {
  if (argc < 9) {
    std::fprintf(stderr, "usage: %s MODEL THETA K MGP N_TRAJ STEPS SEED NODE=VAL,... [--no-device]\n",
                 argv[0]);
    return 1;
  }
  const bool no_device = argc > 9 && std::strcmp(argv[9], "--no-device") == 0;
  std::ifstream f(argv[1]);
  std::stringstream ss;
  ss << f.rdbuf();
  const pbn::model m = pbn::parse_model(ss.str());
  const std::uint64_t theta = std::strtoull(argv[2], nullptr, 10);
  const std::uint32_t k = std::strtoul(argv[3], nullptr, 10), mgp = std::strtoul(argv[4], nullptr, 10);
  const std::uint32_t n_traj = std::strtoul(argv[5], nullptr, 10);
  const std::uint64_t steps = std::strtoull(argv[6], nullptr, 10);
  const std::uint64_t seed = std::strtoull(argv[7], nullptr, 10);
  std::vector<pbn::predicate_term> terms;
  {
    std::stringstream ps(argv[8]);
    std::string item;
    while (std::getline(ps, item, ',')) {
      const auto eq = item.find('=');
      pbn::predicate_term t{};
      t.node = static_cast<std::uint32_t>(std::stoul(item.substr(0, eq)));
      t.value = item.substr(eq + 1) == "1";
      terms.push_back(t);
    }
  }
  const pbn::prepared_simulation ps = pbn::prepare(m, theta, k, mgp);
  const pbn::compiled_predicate pred = pbn::compile_predicate(terms, ps);

  if (no_device) {
    pbn::gpu_plan_view pv(ps);
    pbn_gpu* h = nullptr;
    const int rc = pbn_gpu_create(&pv.v, 0, 0, &h);
    if (h) pbn_gpu_destroy(h);
    // a zero-initialised Method flag (has_leaf = 0) must be refused, not run
    pbn_plan_view bad = pv.v;
    bad.has_leaf = 0;
    pbn_gpu* h2 = nullptr;
    const int rc_bad = pbn_gpu_create(&bad, 0, 0, &h2);
    if (h2) pbn_gpu_destroy(h2);
    std::printf("{\"mode\": \"no-device\", \"create_rc\": %d, \"create_rc_without_leaf\": %d, "
                "\"n_kept\": %u, \"groups\": %zu, \"error\": \"%s\"}\n",
                rc, rc_bad, ps.kept_count(), ps.exec.size(), pbn_last_error());
    return 0;
  }

  const std::uint32_t words = ps.kept_count() / 64 + 1;
  std::vector<std::uint64_t> dev_states(static_cast<std::size_t>(n_traj) * words, 0);
  std::vector<std::uint64_t> counts(static_cast<std::size_t>(n_traj) * PBN_COUNT_FIELDS, 0);
  pbn::gpu_ensemble eng(ps);
  eng.simulate(seed, 0, n_traj, 0, steps, pred, dev_states.data(), counts.data());

  std::uint32_t bad_states = 0, bad_hits = 0;
  std::uint64_t hits_total = 0, fn_total = 0;
  for (std::uint32_t t = 0; t < n_traj; ++t) {
    pbn::state s(ps.kept_count());  // all zeros, as the CLI (pbn_main.cpp:232)
    stepping st(ps);
    philox_rng rng;
    orc_stream_init(&rng.st, seed, t, 0, ps.pplan.groups + 1);
    pbn::sim_options opt;
    opt.count_nodes = false;
    opt.predicate = &pred;
    const pbn::trajectory tr = pbn::simulate(st, s, steps, rng, opt);
    if (std::memcmp(s.data(), dev_states.data() + static_cast<std::size_t>(t) * words, 8 * words))
      ++bad_states;
    const std::uint64_t* c = counts.data() + static_cast<std::size_t>(t) * PBN_COUNT_FIELDS;
    if (c[PBN_C_HITS] != tr.predicate_hits || c[PBN_C_STEPS] != steps) ++bad_hits;
    hits_total += tr.predicate_hits;
    fn_total += c[PBN_C_FNSTEPS];
  }
  // the same job through the device group (pbn_group_*):
  // every device of this box, one ncclAllReduce of the pooled counts
  int ndev = 0;
  pbn_device_count(&ndev);
  pbn::gpu_plan_view pv(ps);
  pbn_group* grp = nullptr;
  int grc = pbn_group_create(&pv.v, nullptr, static_cast<std::uint32_t>(ndev), 0, &grp);
  std::uint32_t group_bad = 0;
  std::uint64_t group_hits = 0;
  if (grc == PBN_OK) {
    std::vector<std::uint64_t> gstates(dev_states.size(), 0), totals(PBN_COUNT_FIELDS, 0);
    pbn_run_args a{};
    a.seed = seed;
    a.n_traj = n_traj;
    a.stream = PBN_STREAM_U53;
    a.n_steps = steps;
    std::vector<std::uint32_t> bits;  // compiled_predicate: (engine bit, value) pairs
    std::vector<std::uint8_t> vals;
    for (const auto& [bit, val] : pred) {
      bits.push_back(bit);
      vals.push_back(val ? 1 : 0);
    }
    a.pred_bits = bits.data();
    a.pred_vals = vals.data();
    a.n_pred = static_cast<std::uint32_t>(bits.size());
    grc = pbn_group_run(grp, &a, gstates.data(), nullptr, totals.data(), nullptr);
    group_bad = gstates == dev_states ? 0u : 1u;
    group_hits = totals[PBN_C_HITS];
    pbn_group_destroy(grp);
  }
  std::printf("{\"mode\": \"device\", \"trajectories\": %u, \"steps\": %llu, \"n_kept\": %u, "
              "\"state_mismatches\": %u, \"hit_mismatches\": %u, \"hits\": %llu, "
              "\"fn_phase_steps\": %llu, \"group_devices\": %d, \"group_rc\": %d, "
              "\"group_state_mismatch\": %u, \"group_hits\": %llu}\n",
              n_traj, static_cast<unsigned long long>(steps), ps.kept_count(), bad_states, bad_hits,
              static_cast<unsigned long long>(hits_total), static_cast<unsigned long long>(fn_total),
              ndev, grc, group_bad, static_cast<unsigned long long>(group_hits));
  return bad_states || bad_hits || grc != PBN_OK || group_bad || group_hits != hits_total ? 2 : 0;
}
