// Preparation pipeline; see plan.hpp. Every floating-point expression keeps
// the reference's evaluation order (compiled with -ffp-contract=off) so the
// plan is bitwise identical to pbn::prepare.
#include "plan.hpp"

#include <algorithm>
#include <bit>
#include <cmath>
#include <numeric>
#include <queue>
#include <string>

namespace pbn_b200 {

// ---------------------------------------------------------------------------
// Walker alias table (alias.hpp:18-56). Items with scaled mass < 1 ("poor")
// are paired, last-in first-out, with the most recent item of mass >= 1
// ("rich"), which donates the deficit; leftovers keep cut-off 1.
walker_table build_walker(const double* probs, std::size_t n) {
  if (n == 0) throw model_error("alias table needs a non-empty distribution");
  double total = 0.0;
  for (std::size_t i = 0; i < n; ++i) {
    if (!(probs[i] >= 0.0)) throw model_error("alias table needs non-negative probabilities");
    total += probs[i];
  }
  if (std::abs(total - 1.0) > 1e-9)
    throw model_error("alias table input probabilities must sum to 1");

  walker_table t;
  t.cut.assign(n, 1.0);
  t.alias.resize(n);
  std::iota(t.alias.begin(), t.alias.end(), 0u);
  std::vector<double> mass(n);
  const double nd = static_cast<double>(n);
  for (std::size_t i = 0; i < n; ++i) mass[i] = probs[i] * nd / total;

  std::vector<std::uint32_t> poor, rich;
  for (std::uint32_t i = 0; i < n; ++i) {
    if (mass[i] < 1.0)
      poor.push_back(i);
    else
      rich.push_back(i);
  }
  while (!poor.empty() && !rich.empty()) {
    const std::uint32_t s = poor.back();
    poor.pop_back();
    const std::uint32_t l = rich.back();
    t.cut[s] = mass[s];
    t.alias[s] = l;
    mass[l] -= 1.0 - mass[s];
    if (mass[l] < 1.0) {
      rich.pop_back();
      poor.push_back(l);
    }
  }
  for (auto i : poor) t.cut[i] = 1.0;
  for (auto i : rich) t.cut[i] = 1.0;
  return t;
}

// ---------------------------------------------------------------------------
// Leaf reduction (Definition 1; reduction.hpp:28-94). A worklist over the
// number of distinct readers of each node; self-reads count as a reader.
namespace {

std::vector<std::uint32_t> distinct_parents(const pbn_node& nd) {
  std::vector<std::uint32_t> ps;
  for (const auto& f : nd.fns) ps.insert(ps.end(), f.parents.begin(), f.parents.end());
  std::sort(ps.begin(), ps.end());
  ps.erase(std::unique(ps.begin(), ps.end()), ps.end());
  return ps;
}

void reduce_into(const network& m, prepared_plan& pp) {
  const std::uint32_t n = m.size();
  pp.original_n = n;
  std::vector<std::vector<std::uint32_t>> reads(n);
  std::vector<std::uint32_t> readers(n, 0);
  for (std::uint32_t v = 0; v < n; ++v) {
    reads[v] = distinct_parents(m.nodes[v]);
    for (auto u : reads[v]) ++readers[u];
  }
  std::vector<char> of_interest(n, 0), gone(n, 0);
  for (auto i : m.interest) of_interest[i] = 1;

  std::vector<std::uint32_t> queue;
  for (std::uint32_t v = 0; v < n; ++v)
    if (!of_interest[v] && readers[v] == 0) queue.push_back(v);
  for (std::size_t head = 0; head < queue.size(); ++head) {  // FIFO order
    const std::uint32_t v = queue[head];
    gone[v] = 1;
    pp.removed.push_back(v);
    for (auto u : reads[v])
      if (!gone[u] && --readers[u] == 0 && !of_interest[u]) queue.push_back(u);
  }

  pp.index_map.assign(n, -1);
  std::uint32_t next = 0;
  for (std::uint32_t v = 0; v < n; ++v)
    if (!gone[v]) pp.index_map[v] = static_cast<std::int32_t>(next++);

  pp.kept.p = m.p;
  pp.kept.nodes.reserve(next);
  for (std::uint32_t v = 0; v < n; ++v) {
    if (gone[v]) continue;
    pbn_node nd = m.nodes[v];
    for (auto& f : nd.fns)
      for (auto& q : f.parents) q = static_cast<std::uint32_t>(pp.index_map[q]);
    pp.kept.nodes.push_back(std::move(nd));
  }
  for (auto i : m.interest)
    if (pp.index_map[i] >= 0) pp.kept.interest.push_back(static_cast<std::uint32_t>(pp.index_map[i]));
  std::sort(pp.kept.interest.begin(), pp.kept.interest.end());
  pp.t = std::pow(1.0 - m.p, static_cast<double>(pp.removed.size()));
}

// Grouped perturbation plan (Alg. 2 lines 2-3; perturbation.hpp:25-43).
void perturbation_into(std::uint32_t n, std::uint32_t k_max, double p, prepared_plan& pp) {
  if (n < 1) throw model_error("perturbation plan needs at least one node");
  if (k_max < 1 || k_max > kPertMaxWidth)
    throw resource_error("perturbation group width must be in [1, 24]");
  pp.g = (n + k_max - 1) / k_max;
  pp.k = (n + pp.g - 1) / pp.g;
  pp.k_prime = n - pp.k * (pp.g - 1);
  pp.mask = (1ull << pp.k_prime) - 1;
  std::vector<double> pat(1ull << pp.k);
  for (std::uint64_t c = 0; c < pat.size(); ++c) {
    const int ones = std::popcount(c);
    pat[c] = std::pow(p, static_cast<double>(ones)) *
             std::pow(1.0 - p, static_cast<double>(static_cast<int>(pp.k) - ones));
  }
  pp.pert = build_walker(pat.data(), pat.size());
}

std::vector<std::uint32_t> union_of_parents(const network& m,
                                            const std::vector<std::uint32_t>& members) {
  std::vector<std::uint32_t> u;
  for (auto v : members)
    for (const auto& f : m.nodes[v].fns) u.insert(u.end(), f.parents.begin(), f.parents.end());
  std::sort(u.begin(), u.end());
  u.erase(std::unique(u.begin(), u.end()), u.end());
  return u;
}

// The budget checks combine() applies before materialising a group's
// combined tables (grouping.hpp:106-116). Tables themselves are produced
// directly in sliced form during flattening.
void check_group_budget(const network& m, const std::vector<std::uint32_t>& members) {
  if (members.empty() || members.size() > 64) throw model_error("group must have 1..64 members");
  const std::size_t uni = union_of_parents(m, members).size();
  std::uint64_t combos = 1;
  for (auto v : members) {
    combos *= m.nodes[v].nfn();
    if (combos > kGroupEntryCap) throw resource_error("too many combined functions in one group");
  }
  if (uni >= 40 || (combos << uni) > kGroupEntryCap)
    throw resource_error("combined function tables exceed the memory budget");
}

// Node grouping (Alg. 3/4 plus the single-function pass; grouping.hpp:177-308).
void partition_into(const network& m, std::uint64_t theta, std::uint32_t mgp, prepared_plan& pp) {
  const std::uint32_t n = m.size();
  if (n == 0) throw model_error("cannot partition an empty model");
  std::vector<std::uint32_t> multi, singles;
  for (std::uint32_t v = 0; v < n; ++v) (m.nodes[v].nfn() >= 2 ? multi : singles).push_back(v);

  auto& groups = pp.members;
  if (!multi.empty()) {
    std::vector<std::uint32_t> w;
    w.reserve(multi.size());
    for (auto v : multi) {
      const std::uint32_t f = m.nodes[v].nfn();
      if (f > theta)
        throw resource_error("node " + m.nodes[v].name +
                             " has more predictor functions than theta allows");
      w.push_back(f);
    }
    // Per-node parent lists, so each part's union is a merge of small lists.
    std::vector<std::vector<std::uint32_t>> node_uni(multi.size());
    for (std::size_t i = 0; i < multi.size(); ++i) node_uni[i] = distinct_parents(m.nodes[multi[i]]);

    const std::uint32_t mc = static_cast<std::uint32_t>(multi.size());
    std::uint32_t mm = std::min(partition_lower_bound(w, theta), mc);
    std::vector<std::uint32_t> scratch;
    for (;; ++mm) {
      const auto parts = greedy_product_partition(w, std::min(mm, mc));
      long double weight_sum = 0.0L, entry_total = 0.0L;
      bool fits = true;
      for (const auto& part : parts) {
        if (part.empty()) continue;
        long double product = 1.0L;
        scratch.clear();
        for (auto idx : part) {
          product *= w[idx];
          scratch.insert(scratch.end(), node_uni[idx].begin(), node_uni[idx].end());
        }
        weight_sum += product;
        std::sort(scratch.begin(), scratch.end());
        const std::size_t uni =
            static_cast<std::size_t>(std::unique(scratch.begin(), scratch.end()) - scratch.begin());
        const long double entries = product * std::exp2(static_cast<double>(uni));
        entry_total += entries;
        if (uni >= 40 || entries > static_cast<long double>(kGroupEntryCap) ||
            (mm < mc && entry_total > static_cast<long double>(kTotalEntryCap))) {
          fits = false;
          break;
        }
      }
      if (fits && weight_sum <= static_cast<long double>(theta)) {
        for (const auto& part : parts) {
          if (part.empty()) continue;
          std::vector<std::uint32_t> mem;
          for (auto idx : part) mem.push_back(multi[idx]);
          std::sort(mem.begin(), mem.end());
          check_group_budget(m, mem);
          groups.push_back(std::move(mem));
        }
        break;
      }
      if (mm >= mc) throw resource_error("theta too small: even one node per group exceeds the budget");
    }
  }

  // Single-function nodes: join the admissible group sharing the most parents
  // (first one on ties), else open a new group (grouping.hpp:243-297).
  struct sgroup {
    std::vector<std::uint32_t> mem, uni;
  };
  std::vector<sgroup> sg;
  long double table_total = 0.0L;
  std::vector<std::uint32_t> merged;
  for (auto v : singles) {
    std::vector<std::uint32_t> ps = m.nodes[v].fns[0].parents;
    std::sort(ps.begin(), ps.end());
    ps.erase(std::unique(ps.begin(), ps.end()), ps.end());
    if (ps.size() > mgp)
      throw resource_error("node " + m.nodes[v].name + " has more parents than max_group_parents");
    long best = -1;
    std::size_t best_shared = 0;
    for (std::size_t j = 0; j < sg.size(); ++j) {
      const sgroup& gr = sg[j];
      if (gr.mem.size() >= 64) continue;
      // |union| and |intersection| of two sorted lists in one pass
      std::size_t a = 0, b = 0, uni = 0, shared = 0;
      while (a < gr.uni.size() || b < ps.size()) {
        if (b == ps.size() || (a < gr.uni.size() && gr.uni[a] < ps[b])) {
          ++a;
        } else if (a == gr.uni.size() || ps[b] < gr.uni[a]) {
          ++b;
        } else {
          ++a;
          ++b;
          ++shared;
        }
        ++uni;
      }
      if (uni > mgp) continue;
      const long double grown = table_total - std::exp2(static_cast<long double>(gr.uni.size())) +
                                std::exp2(static_cast<long double>(uni));
      if (grown > static_cast<long double>(theta)) continue;
      if (best < 0 || shared > best_shared) {
        best = static_cast<long>(j);
        best_shared = shared;
      }
    }
    if (best >= 0) {
      sgroup& gr = sg[static_cast<std::size_t>(best)];
      table_total -= std::exp2(static_cast<long double>(gr.uni.size()));
      merged.clear();
      std::set_union(gr.uni.begin(), gr.uni.end(), ps.begin(), ps.end(), std::back_inserter(merged));
      gr.uni = merged;
      table_total += std::exp2(static_cast<long double>(gr.uni.size()));
      gr.mem.push_back(v);
    } else {
      table_total += std::exp2(static_cast<long double>(ps.size()));
      if (table_total > static_cast<long double>(theta))
        throw resource_error("single-function group tables exceed theta");
      sg.push_back({{v}, std::move(ps)});
    }
  }
  for (auto& gr : sg) {
    check_group_budget(m, gr.mem);
    groups.push_back(std::move(gr.mem));
  }
  pp.cum.assign(groups.size() + 1, 0);
  for (std::size_t i = 0; i < groups.size(); ++i)
    pp.cum[i + 1] = pp.cum[i] + static_cast<std::uint32_t>(groups[i].size());
}

// Flattening into the hot-loop arrays (engine.hpp:95-162): per group its
// offset, alias table over the combined functions (member 0's choice varies
// slowest), and per combined function a gather list of its own parents
// (padded to 8 with the always-zero bit n') and a table sliced to them.
void flatten_into(prepared_plan& pp) {
  const network& m = pp.kept;
  const std::uint32_t n = m.size();
  pp.engine_pos.assign(n, 0);
  pp.engine_nodes.clear();
  for (const auto& mem : pp.members)
    for (auto v : mem) {
      pp.engine_pos[v] = static_cast<std::uint32_t>(pp.engine_nodes.size());
      pp.engine_nodes.push_back(v);
    }

  std::vector<std::uint32_t> choice, own, where(n, 0);
  std::vector<double> sel;
  for (std::size_t gi = 0; gi < pp.members.size(); ++gi) {
    const auto& mem = pp.members[gi];
    std::uint64_t combos = 1;
    for (auto v : mem) combos *= m.nodes[v].nfn();
    pp.grp_offset.push_back(pp.cum[gi]);
    pp.grp_fn_begin.push_back(static_cast<std::uint32_t>(pp.fn_gather_begin.size()));
    pp.grp_alias_begin.push_back(static_cast<std::uint32_t>(pp.alias_cut.size()));

    choice.assign(mem.size(), 0);
    sel.clear();
    for (std::uint64_t c = 0; c < combos; ++c) {
      std::uint64_t rem = c;
      for (std::size_t j = mem.size(); j-- > 0;) {
        const std::uint32_t nf = m.nodes[mem[j]].nfn();
        choice[j] = static_cast<std::uint32_t>(rem % nf);
        rem /= nf;
      }
      double prob = 1.0;
      for (std::size_t j = 0; j < mem.size(); ++j) prob *= m.nodes[mem[j]].probs[choice[j]];
      sel.push_back(prob);

      own.clear();
      for (std::size_t j = 0; j < mem.size(); ++j) {
        const auto& ps = m.nodes[mem[j]].fns[choice[j]].parents;
        own.insert(own.end(), ps.begin(), ps.end());
      }
      std::sort(own.begin(), own.end());
      own.erase(std::unique(own.begin(), own.end()), own.end());
      for (std::uint32_t b = 0; b < own.size(); ++b) where[own[b]] = b;

      pp.fn_gather_begin.push_back(pp.fn_gather.size());
      pp.fn_table_begin.push_back(pp.fn_tables.size());
      pp.fn_gather_count.push_back(static_cast<std::uint32_t>(own.size()));
      for (auto q : own) pp.fn_gather.push_back(pp.engine_pos[q]);
      for (std::size_t b = own.size(); b < kGatherPad; ++b) pp.fn_gather.push_back(n);

      const std::uint64_t len = 1ull << own.size();
      for (std::uint64_t v = 0; v < len; ++v) {
        std::uint64_t packed = 0;
        for (std::size_t j = 0; j < mem.size(); ++j) {
          const predictor& f = m.nodes[mem[j]].fns[choice[j]];
          std::uint64_t fv = 0;
          for (std::size_t b = 0; b < f.parents.size(); ++b)
            fv |= ((v >> where[f.parents[b]]) & 1ull) << b;
          packed |= static_cast<std::uint64_t>(f.output(fv)) << j;
        }
        pp.fn_tables.push_back(packed);
      }
    }
    if (combos > 1) {
      const walker_table wt = build_walker(sel.data(), sel.size());
      pp.grp_alias_size.push_back(wt.size());
      pp.alias_cut.insert(pp.alias_cut.end(), wt.cut.begin(), wt.cut.end());
      pp.alias_idx.insert(pp.alias_idx.end(), wt.alias.begin(), wt.alias.end());
    } else {
      pp.grp_alias_size.push_back(0);
    }
  }
}

}  // namespace

// ---------------------------------------------------------------------------
std::uint32_t partition_lower_bound(const std::vector<std::uint32_t>& w, std::uint64_t theta) {
  double lp = 0.0;
  for (auto x : w) lp += std::log(static_cast<double>(x));
  const double lt = std::log(static_cast<double>(theta));
  for (std::uint32_t m = 1;; ++m)
    if (std::log(static_cast<double>(m)) + lp / m <= lt + 1e-12) return m;
}

std::vector<std::vector<std::uint32_t>> greedy_product_partition(
    const std::vector<std::uint32_t>& w, std::uint32_t m) {
  std::vector<std::uint32_t> order(w.size());
  std::iota(order.begin(), order.end(), 0u);
  std::sort(order.begin(), order.end(), [&](std::uint32_t a, std::uint32_t b) {
    return w[a] != w[b] ? w[a] > w[b] : a < b;
  });
  std::vector<std::vector<std::uint32_t>> parts(m);
  // Min-heap on (product, part index): the same argmin as a linear scan
  // that keeps the lowest index among equal products.
  using entry = std::pair<double, std::uint32_t>;
  std::priority_queue<entry, std::vector<entry>, std::greater<entry>> heap;
  for (std::uint32_t j = 0; j < m; ++j) heap.push({1.0, j});
  for (auto idx : order) {
    auto [prod, j] = heap.top();
    heap.pop();
    parts[j].push_back(idx);
    heap.push({prod * static_cast<double>(w[idx]), j});
  }
  return parts;
}

prepared_plan prepare_nodewise_plan(const network& m, bool reduced) {
  prepared_plan pp;
  if (reduced) {
    reduce_into(m, pp);
  } else {  // identity "reduction": the full model, t = 1
    pp.original_n = m.size();
    pp.kept = m;
    pp.index_map.resize(m.size());
    std::iota(pp.index_map.begin(), pp.index_map.end(), 0);
    pp.t = 1.0;
  }
  const network& k = pp.kept;
  const std::uint32_t n = k.size();
  if (n == 0) throw model_error("network reduction removed every node");
  pp.pert_mode = 1;
  pp.has_leaf = reduced ? 1u : 0u;
  pp.pert_p = m.p;
  pp.g = n;  // one Bernoulli draw per node (engine.hpp:194-201)
  pp.k = 1;
  pp.k_prime = 1;
  pp.mask = 1;
  pp.pert.cut = {1.0, 1.0};
  pp.pert.alias = {0, 1};
  // groups: multi-function nodes first (their draws come in node order), then
  // single-function nodes; every group is one node at its own bit
  std::vector<std::uint32_t> order;
  for (std::uint32_t v = 0; v < n; ++v)
    if (k.nodes[v].nfn() > 1) order.push_back(v);
  for (std::uint32_t v = 0; v < n; ++v)
    if (k.nodes[v].nfn() == 1) order.push_back(v);
  pp.engine_pos.resize(n);
  pp.engine_nodes.resize(n);
  for (std::uint32_t v = 0; v < n; ++v) pp.engine_pos[v] = pp.engine_nodes[v] = v;
  for (auto v : order) {
    const pbn_node& nd = k.nodes[v];
    pp.members.push_back({v});
    pp.grp_members.push_back(1);
    pp.grp_offset.push_back(v);
    pp.grp_fn_begin.push_back(static_cast<std::uint32_t>(pp.fn_gather_begin.size()));
    pp.grp_alias_begin.push_back(static_cast<std::uint32_t>(pp.alias_cut.size()));
    if (nd.nfn() > 1) {  // selectors_ (engine.hpp:172-177)
      const walker_table wt = build_walker(nd.probs.data(), nd.probs.size());
      pp.grp_alias_size.push_back(wt.size());
      pp.alias_cut.insert(pp.alias_cut.end(), wt.cut.begin(), wt.cut.end());
      pp.alias_idx.insert(pp.alias_idx.end(), wt.alias.begin(), wt.alias.end());
    } else {
      pp.grp_alias_size.push_back(0);
    }
    for (const predictor& f : nd.fns) {  // boolean_function::eval (model.hpp:38-43)
      pp.fn_gather_begin.push_back(pp.fn_gather.size());
      pp.fn_table_begin.push_back(pp.fn_tables.size());
      pp.fn_gather_count.push_back(f.arity());
      for (auto q : f.parents) pp.fn_gather.push_back(q);
      for (std::size_t b = f.arity(); b < kGatherPad; ++b) pp.fn_gather.push_back(n);
      for (std::uint64_t x = 0; x < (1ull << f.arity()); ++x)
        pp.fn_tables.push_back(f.output(x) ? 1ull : 0ull);
    }
  }
  pp.cum.assign(1, 0);
  return pp;
}

prepared_plan prepare_plan(const network& m, std::uint64_t theta, std::uint32_t k_max,
                           std::uint32_t max_group_parents) {
  prepared_plan pp;
  reduce_into(m, pp);
  const std::uint32_t n = pp.kept.size();
  if (n == 0) throw model_error("network reduction removed every node");
  perturbation_into(n, k_max, m.p, pp);
  partition_into(pp.kept, theta, max_group_parents, pp);
  flatten_into(pp);
  return pp;
}

}  // namespace pbn_b200
