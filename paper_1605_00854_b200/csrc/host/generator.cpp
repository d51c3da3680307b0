// BASELINE-shaped synthetic networks. The reference's own
// generator (generate.hpp:34-176) is density/leaf-percentage driven and does
// not produce BASELINE.json's distributions, so this one is new:
//   * node v has F ~ U{f_min..f_max} predictor functions;
//   * each function has phi ~ U{p_min..p_max} distinct parents, sorted, drawn
//     uniformly from the readable nodes (designated leaves are never read);
//   * truth tables are uniform random bits; selection probabilities are
//     U(0,1) draws normalised per node;
//   * interest = the target nodes (never designated leaves), so reduction
//     removes designated and natural leaves.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <numeric>
#include <vector>

#include "generator.hpp"

namespace pbn_b200 {

namespace {

struct splitmix {
  std::uint64_t x;
  std::uint64_t next() {
    std::uint64_t z = (x += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  }
  std::uint64_t below(std::uint64_t n) { return next() % n; }  // n small: bias negligible
  std::uint32_t between(std::uint32_t lo, std::uint32_t hi) {
    return lo + static_cast<std::uint32_t>(below(static_cast<std::uint64_t>(hi - lo) + 1));
  }
  double open01() { return (static_cast<double>(next() >> 11) + 0.5) * 0x1.0p-53; }
};

}  // namespace

generated_network generate_network(const gen_params& gp) {
  if (gp.n < 2) throw model_error("generator needs n >= 2");
  if (gp.f_min < 1 || gp.f_max < gp.f_min) throw model_error("bad function-count range");
  if (gp.p_min < 1 || gp.p_max < gp.p_min || gp.p_max > 30) throw model_error("bad parent-count range");
  if (!(gp.leaf_frac >= 0.0 && gp.leaf_frac < 1.0)) throw model_error("leaf fraction must be in [0,1)");
  if (!(gp.p > 0.0 && gp.p < 1.0)) throw model_error("perturbation rate must be in (0,1)");
  if (gp.n_targets < 1 || gp.n_targets > gp.n) throw model_error("bad target count");

  splitmix rng{gp.seed};
  const std::uint32_t n = gp.n;
  generated_network out;
  // targets
  std::vector<std::uint32_t> perm(n);
  std::iota(perm.begin(), perm.end(), 0u);
  std::vector<char> is_target(n, 0);
  if (gp.targets_fixed) {
    for (std::uint32_t i = 0; i < gp.n_targets; ++i) {
      out.pred_nodes.push_back(i);
      out.pred_vals.push_back(1);
      is_target[i] = 1;
    }
  } else {
    for (std::uint32_t i = 0; i < gp.n_targets; ++i) {
      std::swap(perm[i], perm[i + rng.below(n - i)]);
      out.pred_nodes.push_back(perm[i]);
      out.pred_vals.push_back(static_cast<std::uint8_t>(rng.next() & 1));
      is_target[perm[i]] = 1;
    }
  }
  // designated leaves among non-targets
  std::vector<std::uint32_t> pool;
  for (std::uint32_t v = 0; v < n; ++v)
    if (!is_target[v]) pool.push_back(v);
  std::uint32_t leaves = static_cast<std::uint32_t>(std::llround(gp.leaf_frac * n));
  leaves = std::min<std::uint32_t>(leaves, static_cast<std::uint32_t>(pool.size()));
  std::vector<char> is_leaf(n, 0);
  for (std::uint32_t i = 0; i < leaves; ++i) {
    std::swap(pool[i], pool[i + rng.below(pool.size() - i)]);
    is_leaf[pool[i]] = 1;
  }
  std::vector<std::uint32_t> readable;
  for (std::uint32_t v = 0; v < n; ++v)
    if (!is_leaf[v]) readable.push_back(v);

  network& m = out.net;
  m.p = gp.p;
  m.nodes.resize(n);
  std::vector<std::uint32_t> picked;
  for (std::uint32_t v = 0; v < n; ++v) {
    pbn_node& nd = m.nodes[v];
    nd.name = "x" + std::to_string(v);
    const std::uint32_t nf = rng.between(gp.f_min, gp.f_max);
    double total = 0.0;
    for (std::uint32_t j = 0; j < nf; ++j) {
      predictor f;
      const std::uint32_t phi =
          std::min<std::uint32_t>(rng.between(gp.p_min, gp.p_max),
                                  static_cast<std::uint32_t>(readable.size()));
      picked.clear();
      while (picked.size() < phi) {  // rejection sampling of distinct parents
        const std::uint32_t q = readable[rng.below(readable.size())];
        if (std::find(picked.begin(), picked.end(), q) == picked.end()) picked.push_back(q);
      }
      std::sort(picked.begin(), picked.end());
      f.parents = picked;
      f.bits = predictor::zero_table(phi);
      for (std::uint64_t x = 0; x < (1ull << phi); ++x) f.set_output(x, rng.next() & 1);
      nd.fns.push_back(std::move(f));
      const double w = rng.open01();
      nd.probs.push_back(w);
      total += w;
    }
    for (double& w : nd.probs) w /= total;
  }
  for (std::uint32_t v = 0; v < n; ++v)
    if (is_target[v]) m.interest.push_back(v);
  // canonical form: what the text format round-trips to (both this library
  // and the reference parse the same serialized text)
  out.net = parse_network(serialize_network(m));
  return out;
}

}  // namespace pbn_b200
