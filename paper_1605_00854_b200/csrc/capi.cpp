// extern "C" boundary of the engine (include/pbn_b200.h). No exception
// crosses it: reference exception classes map to status codes
// (errors.hpp:10-32 -> pbn_main.cpp:302-311 exit codes).
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <limits>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "../../include/pbn_b200.h"
#include "device/dev_plan.h"
#include "host/device_plan.hpp"
#include "host/estimator.hpp"
#include "host/generator.hpp"
#include "host/model.hpp"
#include "host/plan.hpp"

namespace pbn_b200 {
cudaError_t launch_ensemble(const dev_plan_header& h, const std::uint8_t* d_blob, int place,
                            int stream_kind, std::uint32_t lpt, std::uint32_t warps_per_cta,
                            const dev_run_params& rp, std::uint64_t* d_states,
                            std::uint64_t* d_counts, cudaStream_t stream,
                            std::uint32_t* launches, bool pert_dom);
cudaError_t launch_lane_ensemble(const dev_plan_header& h, const std::uint8_t* d_blob, int place,
                                 int stream_kind, bool scan, std::uint32_t warps_per_cta,
                                 const dev_run_params& rp, std::uint64_t* d_states,
                                 std::uint64_t* d_counts, cudaStream_t stream,
                                 std::uint32_t* launches);
cudaError_t launch_ensemble_script(const dev_plan_header& h, const std::uint8_t* d_blob,
                                   std::uint32_t warps_per_cta, const dev_run_params& rp,
                                   std::uint64_t* d_states, std::uint64_t* d_counts,
                                   cudaStream_t stream);
bool lane_kernel_fits(const dev_plan_header& h);
std::uint32_t pf_max_warps();
std::size_t slot_words(const dev_plan_header& h, std::uint32_t lpt, bool node_counts);
bool ensemble_pa2(const dev_plan_header& h, std::uint32_t lpt, int gm, bool pert_dom);
int ensemble_gather_mode(const dev_plan_header& h, std::uint32_t lpt, int stream);
std::uint32_t lane_max_warps();
std::size_t lane_warp_words(const dev_plan_header& h, bool node_counts, bool scan);
const char* lane_rare_fn_name();
std::size_t lane_cta_bytes();
cudaError_t launch_philox_kat(const uint4* d_ctr, std::uint32_t k0, std::uint32_t k1, uint4* d_out,
                              std::uint32_t n, cudaStream_t stream);
cudaError_t launch_series_stats(const std::uint32_t* d_series, std::uint32_t n_traj,
                                std::uint64_t stride, std::uint64_t len, std::uint32_t kappa,
                                unsigned long long* d_out13, cudaStream_t stream);
cudaError_t launch_sum_counts(const std::uint64_t* d_counts, std::uint32_t n,
                              unsigned long long* d_out8, cudaStream_t stream);
}  // namespace pbn_b200

using namespace pbn_b200;

struct pbn_model {
  network net;
};

struct pbn_plan {
  prepared_plan pp;
};

struct cuda_failure : std::runtime_error {
  explicit cuda_failure(const std::string& w) : std::runtime_error(w) {}
};

struct pbn_gpu {
  int device = 0;
  encoded_plan ep;
  int place = 0;  // PLACE_* of ensemble.cu
  bool place_fixed = false;  // set by pbn_gpu_set_placement (not "auto")
  std::uint32_t smem_optin = 0, sms = 0;
  std::uint8_t* d_blob = nullptr;
  // scratch for the host-buffer entry point
  std::uint64_t* d_states = nullptr;
  std::uint64_t* d_counts = nullptr;
  std::size_t cap_traj = 0;
  std::uint32_t launches = 0;
  std::uint32_t last_warps = 0;
  std::uint32_t lpt_fixed = 0;  // 0: chosen per run
  std::uint32_t last_lpt = 0;
  int last_place = -1;  // placement the last launch actually ran (-1: none yet)
  std::string last_kernel;  // kernel_name() of the last launch
  // device workspace kept across calls: pbn_estimate's states, counts,
  // carried samples, two pilot-series buffers and reduction scratch (0-5);
  // pbn_gpu_run's carried samples, series and node counts (6-8)
  struct ws_buf {
    void* p = nullptr;
    std::size_t bytes = 0;
  };
  ws_buf ws[9];
  double p_fn = 1.0;  // probability that a step reaches the function phase
  double p_group_flip = 0.0;  // probability that a full perturbation group flips
  // host copy of the plan's decision tables (pbn_gpu_run_scripted lays a
  // sequential script out in the stream's slots with the reference's own rules)
  struct script_tables {
    double t = 1.0;
    std::uint32_t groups = 0, size = 0, has_leaf = 0, pert_mode = 0;
    std::uint64_t mask = 0;
    std::vector<double> pert_cut, alias_cut;
    std::vector<std::uint32_t> pert_alias, alias_idx, a_begin, a_size;  // a_*: the alias groups, in order
  } st;
};

namespace {

thread_local std::string g_error;

template <class F>
int guard(F&& f) {
  try {
    f();
    return PBN_OK;
  } catch (const resource_error& e) {
    g_error = e.what();
    return PBN_ERESOURCE;
  } catch (const model_error& e) {
    g_error = e.what();
    return PBN_EMODEL;
  } catch (const cuda_failure& e) {
    g_error = e.what();
    return PBN_ECUDA;
  } catch (const std::bad_alloc&) {
    g_error = "out of host memory";
    return PBN_ERESOURCE;
  } catch (const std::exception& e) {
    g_error = e.what();
    return PBN_EUSAGE;
  }
}

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw cuda_failure(std::string(what) + ": " + cudaGetErrorString(e));
}

void need(const void* p, const char* what) {
  if (!p) throw std::invalid_argument(std::string("null argument: ") + what);
}

constexpr std::uint32_t kStateReserve = 24 * 1024;  // smem kept for trajectory states
// Lane kernel: scan phase A ahead per lane when fewer steps than this reach
// the function phase (c1: 0.37 -> +22%; c3: 0.91 -> -17%).
constexpr double kScanBelow = 0.65;
// Sub-warp kernel, perturbation-dominated launches: when fewer steps than this
// reach the function phase (c5 at p >= 0.01: < 1e-8), the launch stages
// nothing (every shared-memory byte the plan does not take stays L1 for the
// 256 KiB perturbation-cell words), runs 32 warps per CTA and prefetches the
// next step's phase A (ensemble.cu PF): c5 p = 0.1 1.71e9 -> see DESIGN §7a.
constexpr double kPertDominated = 0.02;

// Probability that a step reaches the function phase: no kept node flips
// (every pattern draw returns 0, or every Bernoulli draw misses) and the leaf
// draw stays below t (engine.hpp:259-268). Exact for the plan's own cells.
// Probability that a full perturbation group draws a non-zero pattern.
double group_flip_probability(const pbn_plan_view& v) {
  if (v.pert_mode != 0 || v.pert_size == 0) return v.pert_mode != 0 ? v.pert_p : 0.0;
  double zero = 0;
  const double n = static_cast<double>(v.pert_size);
  for (std::uint32_t c = 0; c < v.pert_size; ++c)
    zero += (c == 0 ? v.pert_cut[c] / n : 0.0) + (v.pert_alias[c] == 0 ? (1.0 - v.pert_cut[c]) / n : 0.0);
  return 1.0 - zero;
}

double fn_phase_probability(const pbn_plan_view& v) {
  double p_none;
  if (v.pert_mode != 0) {
    p_none = std::pow(1.0 - v.pert_p, static_cast<double>(v.pert_groups));
  } else {
    double full = 0, last = 0;
    const double n = static_cast<double>(v.pert_size);
    for (std::uint32_t c = 0; c < v.pert_size; ++c) {
      const double mine = v.pert_cut[c] / n, other = (1.0 - v.pert_cut[c]) / n;
      full += (c == 0 ? mine : 0.0) + (v.pert_alias[c] == 0 ? other : 0.0);
      last += ((c & v.pert_mask) == 0 ? mine : 0.0) + ((v.pert_alias[c] & v.pert_mask) == 0 ? other : 0.0);
    }
    p_none = v.pert_groups ? std::pow(full, static_cast<double>(v.pert_groups - 1)) * last : 1.0;
  }
  return p_none * (v.has_leaf ? v.t : 1.0);
}

// Lanes per trajectory: by network size, then doubled until the ensemble
// gives ~24 resident warps per SM (latency hiding) or one warp per trajectory.
// Lane-per-trajectory kernel (lane_ensemble.cu) for networks up to 255 kept
// nodes once the ensemble gives >= 6 warps of 32 trajectories per SM
// (measured on c1/c3: +10-30 % over sub-warps at 32768 trajectories, 2-3x at
// 131072; behind them at 16384).
std::uint32_t auto_lpt(std::uint32_t n_kept, std::uint64_t n_traj, std::uint32_t sms) {
  if (n_kept <= 255 && n_traj >= static_cast<std::uint64_t>(sms) * 192) return 1;
  std::uint32_t lpt = n_kept <= 256 ? 8 : n_kept <= 512 ? 16 : 32;
  while (lpt < 32 && n_traj * lpt / 32 < static_cast<std::uint64_t>(sms) * 24) lpt *= 2;
  return lpt;
}

// Staged prefix of the blob for a placement level (dev_plan.h); level 3
// counts both perturbation tables (the launch stages its stream's only).
std::uint32_t staged_bytes_at(const dev_plan_header& h, int place) {
  if (place == 4)  // core + the larger stream's perturbation cells
    return h.core_bytes + std::max(h.blob_bytes - h.off_pert53, h.off_pert53 - h.off_pert32);
  if (place == 3) return h.blob_bytes;
  if (place == 2) return h.off_pert32;
  if (place == 1) return h.core_bytes;
  return 0;
}
std::uint32_t staged_bytes(const pbn_gpu& g) { return staged_bytes_at(g.ep.h, g.place); }

// Placement levels from most to least shared memory: all, tables, core +
// perturbation cells, core, global (run_device steps down this order when
// the ensemble's state does not fit next to the staged plan).
constexpr int kPlaceOrder[] = {3, 2, 4, 1, 0};
int next_lower_place(int place) {
  for (int i = 0; i + 1 < 5; ++i)
    if (kPlaceOrder[i] == place) return kPlaceOrder[i + 1];
  return 0;
}

// Warps per CTA: enough resident slots for the whole ensemble in one wave
// (grid ~ #SMs), bounded by 32 warps and by the shared memory left for states.
std::uint32_t pick_warps(const pbn_gpu& g, std::uint32_t n_traj, std::uint32_t lpt,
                         bool node_counts, std::uint32_t min_staged = 0,
                         std::uint32_t max_warps_lpt32 = 28) {
  if (lpt == 1 && lane_kernel_fits(g.ep.h)) {  // lane kernel: 32 trajectories per warp
    const std::uint64_t warps_needed = (static_cast<std::uint64_t>(n_traj) + 31) / 32;
    std::uint64_t w = (warps_needed + g.sms - 1) / g.sms;
    w = std::max<std::uint64_t>(1, std::min<std::uint64_t>(lane_max_warps(), w));
    const std::uint64_t per_warp = lane_warp_words(g.ep.h, node_counts, g.p_fn < kScanBelow) * 4;
    const std::uint64_t avail = g.smem_optin - staged_bytes(g) - lane_cta_bytes() - 64;
    while (w > 1 && w * per_warp > avail) --w;
    if (w * per_warp > avail) throw resource_error("trajectory state does not fit in shared memory");
    return static_cast<std::uint32_t>(w);
  }
  const std::uint64_t warps_needed = (static_cast<std::uint64_t>(n_traj) * lpt + 31) / 32;
  std::uint64_t w = (warps_needed + g.sms - 1) / g.sms;
  w = std::max<std::uint64_t>(1, std::min<std::uint64_t>(lpt == 32 ? max_warps_lpt32 : 32, w));
  const std::uint64_t stride = slot_words(g.ep.h, lpt, node_counts);  // the launcher's own size
  const std::uint64_t per_warp = static_cast<std::uint64_t>(32 / lpt) * stride * 4;
  const std::uint64_t avail = g.smem_optin - std::max(staged_bytes(g), min_staged) - 64;
  while (w > 1 && w * per_warp > avail) --w;
  if (w * per_warp > avail) throw resource_error("trajectory state does not fit in shared memory");
  return static_cast<std::uint32_t>(w);
}

// A workspace slot of the engine with room for n T's (grown, never shrunk).
template <class T>
T* ws_take(pbn_gpu& g, int slot, std::size_t n) {
  auto& b = g.ws[slot];
  const std::size_t bytes = sizeof(T) * (n ? n : 1);
  if (b.bytes < bytes) {
    if (b.p) cudaFree(b.p);
    b.p = nullptr;
    b.bytes = 0;
    ck(cudaMalloc(&b.p, bytes), "cudaMalloc workspace");
    b.bytes = bytes;
  }
  return static_cast<T*>(b.p);
}

dev_run_params make_params(const pbn_gpu& g, const pbn_run_args& a) {
  dev_run_params rp{};
  philox_round_keys(a.seed, rp.rk0, rp.rk1);
  rp.traj_begin = a.traj_begin;
  rp.n_traj = a.n_traj;
  rp.step_begin = a.step_begin;
  rp.n_steps = a.n_steps;
  if (a.flags & ~(PBN_RUN_NODE_COUNTS | PBN_RUN_EXACT_ALIAS))
    throw std::invalid_argument("unknown run flags");
  rp.exact_alias = (a.flags & PBN_RUN_EXACT_ALIAS) ? 1u : 0u;
  if (a.n_pred) {
    need(a.pred_bits, "pred_bits");
    need(a.pred_vals, "pred_vals");
  }
  rp.pred = compile_dev_predicate(a.pred_bits, a.pred_vals, a.n_pred, g.ep.h.n_kept);
  if (a.stream != PBN_STREAM_U53 && a.stream != PBN_STREAM_U32)
    throw std::invalid_argument("unknown stream kind");
  if (a.stream == PBN_STREAM_U32 && !g.ep.h.u32_ok)
    throw resource_error("U32 stream needs every group alias table <= 2^21 cells");
  if (a.n_steps > 0xFFFFFFFFull)
    throw std::invalid_argument("at most 2^32-1 steps per call (chain calls with step_begin)");
  if (a.thin_mode > 2) throw std::invalid_argument("thin_mode must be 0, 1 or 2");
  rp.kappa = a.kappa ? a.kappa : 1;
  if (rp.kappa > 63) throw std::invalid_argument("kappa must be <= 63");
  rp.thin_mode = a.thin_mode;
  rp.tprev = a.tprev;
  rp.series = a.series;
  rp.series_stride = a.series_stride;
  rp.series_bit0 = a.series_bit0;
  rp.series_init = a.series_init;
  if (a.series && (a.series_bit0 + a.n_steps + 31) / 32 > a.series_stride)
    throw std::invalid_argument("series row too short for this call");
  if (a.traj_begin + a.n_traj > (1ull << 32))
    throw std::invalid_argument("trajectory ids must fit in 32 bits");
  return rp;
}

// What a run of n_traj trajectories launches: kernel, lanes per trajectory,
// warps per CTA, plan placement (possibly stepped down from the configured
// one when the ensemble's per-trajectory state does not fit next to it).
struct launch_choice {
  std::uint32_t lpt = 0, warps = 0;
  int place = 0;
  bool lane = false, scan = false;
  int gm = 0;
  bool pert_dom = false;  // sub-warp PF kernel (kPertDominated)
  bool pa2 = false;       // sub-warp PA2 kernel (two steps per phase-A pass)
};

launch_choice choose_launch(const pbn_gpu& g0, std::uint32_t n_traj, bool nc, std::uint32_t stream) {
  pbn_gpu& g = const_cast<pbn_gpu&>(g0);  // pick_warps reads g.place; restored below
  launch_choice c;
  c.lpt = g.lpt_fixed ? g.lpt_fixed : auto_lpt(g.ep.h.n_kept, n_traj, g.sms);
  c.lane = c.lpt == 1 && lane_kernel_fits(g.ep.h);
  c.gm = c.lane ? -1 : ensemble_gather_mode(g.ep.h, c.lpt, static_cast<int>(stream));
  // GM 4 kernels stage the compact single-node group records at any placement
  const std::uint32_t min_staged = c.gm == 4 ? g.ep.h.off_sfn : 0u;
  const int place0 = g.place;
  // perturbation-dominated launch of a k = 16 plan with one phase-A block per
  // lane, placement left to the engine: global placement, PF kernel
  const std::uint32_t nb0 = (g.ep.h.g + g.ep.h.has_leaf + 3) / 4;
  c.pert_dom = !c.lane && !nc && c.lpt == 32 && !g.place_fixed && g.p_fn < kPertDominated &&
               g.ep.h.pert_mode == 0 && g.ep.h.k == 16 && nb0 <= 32;
  if (c.pert_dom) {
    g.place = 0;
    c.gm = 0;
  }
  for (;;) {
    try {
      c.warps = pick_warps(g, n_traj, c.lpt, nc, c.pert_dom ? 0u : min_staged, c.pert_dom ? pf_max_warps() : 28u);
      break;
    } catch (const resource_error&) {
      if (g.place == 0) {
        g.place = place0;
        throw;
      }
      g.place = next_lower_place(g.place);
    }
  }
  c.place = g.place;
  g.place = place0;
  c.scan = c.lane && g.p_fn < kScanBelow;
  c.pa2 = !c.lane && ensemble_pa2(g.ep.h, c.lpt, c.gm, c.pert_dom);
  return c;
}

std::string kernel_name(const launch_choice& c, std::uint32_t stream) {
  static const char* places[] = {"global", "core", "tables", "all", "core_pert"};
  static const char* gms[] = {"smem", "shfl", "shfl_compact", "shfl2", "smem_compact"};
  std::string s = c.lane ? std::string("lane<") + (c.scan ? lane_rare_fn_name() : "lockstep")
                         : "subwarp<lpt=" + std::to_string(c.lpt) + ",gather=" + gms[c.gm];
  s += std::string(",stream=") + (stream == PBN_STREAM_U53 ? "u53" : "u32");
  s += std::string(",place=") + places[c.place] + ",warps=" + std::to_string(c.warps);
  if (c.pert_dom) s += ",pa_prefetch";
  if (c.pa2) s += ",pa2";
  s += ">";
  return s;
}

void run_device(pbn_gpu& g, const pbn_run_args& a, std::uint64_t* d_states,
                std::uint64_t* d_counts, std::uint64_t* d_node_counts, cudaStream_t stream) {
  dev_run_params rp = make_params(g, a);
  if (a.n_traj == 0) return;
  const bool nc = (a.flags & PBN_RUN_NODE_COUNTS) != 0;
  if (nc && !d_node_counts) throw std::invalid_argument("PBN_RUN_NODE_COUNTS needs node_counts");
  rp.node_counts = nc ? d_node_counts : nullptr;
  ck(cudaSetDevice(g.device), "cudaSetDevice");
  const launch_choice c = choose_launch(g, a.n_traj, nc, a.stream);

  g.last_lpt = c.lpt;
  g.last_warps = c.warps;
  g.last_place = c.place;
  g.last_kernel = kernel_name(c, a.stream);
  g.launches = 0;
  const cudaError_t e =
      c.lane ? launch_lane_ensemble(g.ep.h, g.d_blob, c.place, static_cast<int>(a.stream), c.scan,
                                    c.warps, rp, d_states, d_counts, stream, &g.launches)
             : launch_ensemble(g.ep.h, g.d_blob, c.place, static_cast<int>(a.stream), c.lpt,
                               c.warps, rp, d_states, d_counts, stream, &g.launches, c.pert_dom);
  ck(e, "ensemble launch");
}

}  // namespace

namespace pbn_b200 {
void set_last_error(const std::string& msg) { g_error = msg; }
}  // namespace pbn_b200

extern "C" {

const char* pbn_last_error(void) { return g_error.c_str(); }
const char* pbn_version(void) { return "pbn_b200 0.1 (sm_100a)"; }
uint32_t pbn_state_words(uint32_t n_kept) { return n_kept / 64 + 1; }

int pbn_model_parse(const char* text, size_t len, pbn_model** out) {
  return guard([&] {
    need(text, "text");
    need(out, "out");
    auto m = std::make_unique<pbn_model>();
    m->net = parse_network(std::string(text, len));
    *out = m.release();
  });
}

int pbn_model_serialize(const pbn_model* m, char* buf, size_t cap, size_t* len_out) {
  return guard([&] {
    need(m, "model");
    const std::string s = serialize_network(m->net);
    if (len_out) *len_out = s.size();
    if (buf && cap >= s.size()) std::memcpy(buf, s.data(), s.size());
  });
}

int pbn_model_generate(const pbn_gen_params* gp, pbn_model** out, uint32_t* pred_nodes,
                       uint8_t* pred_vals, uint32_t* n_pred_out) {
  return guard([&] {
    need(gp, "params");
    need(out, "out");
    gen_params p;
    p.n = gp->n;
    p.f_min = gp->f_min;
    p.f_max = gp->f_max;
    p.p_min = gp->p_min;
    p.p_max = gp->p_max;
    p.leaf_frac = gp->leaf_frac;
    p.p = gp->perturbation;
    p.n_targets = gp->n_targets;
    p.targets_fixed = gp->targets_fixed != 0;
    p.seed = gp->seed;
    generated_network g = generate_network(p);
    if (pred_nodes)
      std::copy(g.pred_nodes.begin(), g.pred_nodes.end(), pred_nodes);
    if (pred_vals) std::copy(g.pred_vals.begin(), g.pred_vals.end(), pred_vals);
    if (n_pred_out) *n_pred_out = static_cast<uint32_t>(g.pred_nodes.size());
    auto m = std::make_unique<pbn_model>();
    m->net = std::move(g.net);
    *out = m.release();
  });
}

int pbn_model_info(const pbn_model* m, uint32_t* n, double* p, uint32_t* n_interest,
                   double* density) {
  return guard([&] {
    need(m, "model");
    if (n) *n = m->net.size();
    if (p) *p = m->net.p;
    if (n_interest) *n_interest = static_cast<uint32_t>(m->net.interest.size());
    if (density) *density = network_density(m->net);
  });
}

int pbn_model_node_index(const pbn_model* m, const char* name, uint32_t* index_out) {
  return guard([&] {
    need(m, "model");
    need(name, "name");
    for (uint32_t i = 0; i < m->net.size(); ++i)
      if (m->net.nodes[i].name == name) {
        *index_out = i;
        return;
      }
    throw model_error(std::string("unknown node '") + name + "'");
  });
}

int pbn_model_node_name(const pbn_model* m, uint32_t i, char* buf, size_t cap, size_t* len_out) {
  return guard([&] {
    need(m, "model");
    if (i >= m->net.size()) throw model_error("node index out of range");
    const std::string& nm = m->net.nodes[i].name;
    if (len_out) *len_out = nm.size();
    if (buf && cap) {
      const std::size_t k = std::min(cap - 1, nm.size());
      std::memcpy(buf, nm.data(), k);
      buf[k] = 0;
    }
  });
}

void pbn_model_free(pbn_model* m) { delete m; }

int pbn_prepare(const pbn_model* m, uint64_t theta, uint32_t k_max, uint32_t mgp,
                pbn_plan** out) {
  return guard([&] {
    need(m, "model");
    need(out, "out");
    auto p = std::make_unique<pbn_plan>();
    p->pp = prepare_plan(m->net, theta, k_max, mgp);
    *out = p.release();
  });
}

int pbn_prepare_nodewise(const pbn_model* m, int reduced, pbn_plan** out) {
  return guard([&] {
    need(m, "model");
    need(out, "out");
    auto p = std::make_unique<pbn_plan>();
    p->pp = prepare_nodewise_plan(m->net, reduced != 0);
    *out = p.release();
  });
}

int pbn_plan_get_view(const pbn_plan* plan, pbn_plan_view* v) {
  return guard([&] {
    need(plan, "plan");
    need(v, "view");
    const prepared_plan& pp = plan->pp;
    std::memset(v, 0, sizeof *v);
    v->n_kept = pp.n_kept();
    v->t = pp.t;
    v->pert_groups = pp.g;
    v->pert_k = pp.k;
    v->pert_k_prime = pp.k_prime;
    v->pert_size = pp.pert.size();
    v->pert_mask = pp.mask;
    v->pert_cut = pp.pert.cut.data();
    v->pert_alias = pp.pert.alias.data();
    v->n_groups = static_cast<uint32_t>(pp.grp_offset.size());
    v->grp_offset = pp.grp_offset.data();
    v->grp_fn_begin = pp.grp_fn_begin.data();
    v->grp_alias_begin = pp.grp_alias_begin.data();
    v->grp_alias_size = pp.grp_alias_size.data();
    v->n_alias = pp.alias_cut.size();
    v->alias_cut = pp.alias_cut.data();
    v->alias_idx = pp.alias_idx.data();
    v->n_fns = static_cast<uint32_t>(pp.fn_gather_begin.size());
    v->fn_gather_begin = pp.fn_gather_begin.data();
    v->fn_table_begin = pp.fn_table_begin.data();
    v->fn_gather_count = pp.fn_gather_count.data();
    v->n_gather = pp.fn_gather.size();
    v->fn_gather = pp.fn_gather.data();
    v->n_table = pp.fn_tables.size();
    v->fn_tables = pp.fn_tables.data();
    v->pert_mode = pp.pert_mode;
    v->has_leaf = pp.has_leaf;
    v->pert_p = pp.pert_p;
    v->grp_members = pp.grp_members.empty() ? nullptr : pp.grp_members.data();
  });
}

int pbn_plan_reduced(const pbn_plan* plan, uint32_t* original_n, uint32_t* n_removed,
                     int32_t* index_map, uint32_t* engine_pos, uint32_t* removed) {
  return guard([&] {
    need(plan, "plan");
    const prepared_plan& pp = plan->pp;
    if (original_n) *original_n = pp.original_n;
    if (n_removed) *n_removed = static_cast<uint32_t>(pp.removed.size());
    if (index_map) std::copy(pp.index_map.begin(), pp.index_map.end(), index_map);
    if (engine_pos) std::copy(pp.engine_pos.begin(), pp.engine_pos.end(), engine_pos);
    if (removed) std::copy(pp.removed.begin(), pp.removed.end(), removed);
  });
}

int pbn_plan_groups(const pbn_plan* plan, uint32_t* members, uint32_t* cum) {
  return guard([&] {
    need(plan, "plan");
    const prepared_plan& pp = plan->pp;
    std::size_t k = 0;
    if (members)
      for (const auto& g : pp.members)
        for (auto v : g) members[k++] = v;
    if (cum) std::copy(pp.cum.begin(), pp.cum.end(), cum);
  });
}

int pbn_compile_predicate(const pbn_plan* plan, const uint32_t* nodes, const uint8_t* vals,
                          uint32_t n, uint32_t* bits) {
  return guard([&] {
    need(plan, "plan");
    if (n) {
      need(nodes, "nodes");
      need(bits, "engine_bits_out");
    }
    const prepared_plan& pp = plan->pp;
    for (uint32_t i = 0; i < n; ++i) {  // engine.hpp:343-362
      if (nodes[i] >= pp.original_n) throw model_error("predicate references a nonexistent node");
      const int32_t r = pp.index_map[nodes[i]];
      if (r < 0) throw model_error("predicate references a removed leaf node");
      bits[i] = pp.engine_pos[static_cast<uint32_t>(r)];
    }
    (void)vals;
  });
}

void pbn_plan_free(pbn_plan* plan) { delete plan; }

int pbn_device_count(int* count) {
  return guard([&] {
    int c = 0;
    const cudaError_t e = cudaGetDeviceCount(&c);
    if (e != cudaSuccess) {
      cudaGetLastError();
      c = 0;
    }
    *count = c;
  });
}

// Every array a view promises must be present (a NULL with a non-zero count
// would otherwise be dereferenced by the encoder).
void check_view(const pbn_plan_view& v) {
  auto req = [](bool ok, const char* what) {
    if (!ok) throw std::invalid_argument(std::string("plan view: missing ") + what);
  };
  req(v.pert_cut && v.pert_alias, "perturbation cells");
  if (v.n_groups)
    req(v.grp_offset && v.grp_fn_begin && v.grp_alias_begin && v.grp_alias_size, "group arrays");
  if (v.n_alias) req(v.alias_cut && v.alias_idx, "alias cells");
  if (v.n_fns) req(v.fn_gather_begin && v.fn_table_begin && v.fn_gather_count, "function arrays");
  if (v.n_gather) req(v.fn_gather != nullptr, "gather lists");
  if (v.n_table) req(v.fn_tables != nullptr, "tables");
  if (v.n_groups == 0) throw model_error("plan has no groups");
}

int pbn_gpu_create(const pbn_plan_view* view, int device, uint32_t lpt, pbn_gpu** out) {
  return guard([&] {
    need(view, "view");
    need(out, "out");
    check_view(*view);
    auto g = std::make_unique<pbn_gpu>();
    g->device = device;
    if (lpt != 0 && (lpt > 32 || (lpt & (lpt - 1)) != 0))
      throw std::invalid_argument("lanes per trajectory must be 0 (auto) or a power of two <= 32");
    g->lpt_fixed = lpt;
    g->ep = encode_plan(*view);
    g->p_fn = fn_phase_probability(*view);
    g->p_group_flip = group_flip_probability(*view);
    {
      auto& st = g->st;
      const pbn_plan_view& v = *view;
      st.t = v.t;
      st.groups = v.pert_groups;
      st.size = v.pert_size;
      st.has_leaf = v.has_leaf;
      st.pert_mode = v.pert_mode;
      st.mask = v.pert_mask;
      if (v.pert_mode == 0 && v.pert_size) {
        st.pert_cut.assign(v.pert_cut, v.pert_cut + v.pert_size);
        st.pert_alias.assign(v.pert_alias, v.pert_alias + v.pert_size);
      }
      if (v.n_alias) {
        st.alias_cut.assign(v.alias_cut, v.alias_cut + v.n_alias);
        st.alias_idx.assign(v.alias_idx, v.alias_idx + v.n_alias);
      }
      for (std::uint32_t gi = 0; gi < v.n_groups; ++gi)
        if (v.grp_alias_size[gi]) {
          st.a_begin.push_back(v.grp_alias_begin[gi]);
          st.a_size.push_back(v.grp_alias_size[gi]);
        }
    }
    ck(cudaSetDevice(device), "cudaSetDevice");
    int optin = 0, sms = 0;
    ck(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device), "attr");
    ck(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device), "attr");
    g->smem_optin = static_cast<uint32_t>(optin);
    g->sms = static_cast<uint32_t>(sms);
    const dev_plan_header& h = g->ep.h;
    g->place = 0;
    for (int lvl : kPlaceOrder)
      if (lvl != 0 && staged_bytes_at(h, lvl) + kStateReserve <= g->smem_optin) {
        g->place = lvl;
        break;
      }
    ck(cudaMalloc(&g->d_blob, g->ep.blob.size()), "cudaMalloc plan");
    ck(cudaMemcpy(g->d_blob, g->ep.blob.data(), g->ep.blob.size(), cudaMemcpyHostToDevice),
       "upload plan");
    *out = g.release();
  });
}

int pbn_gpu_set_placement(pbn_gpu* g, uint32_t placement) {
  return guard([&] {
    need(g, "gpu");
    if (placement > 5) throw std::invalid_argument("placement must be 0..5");
    if (placement == 0) return;
    // 0 global, 1 core, 2 +tables, 3 all, 4 core + perturbation cells
    const int want = static_cast<int>(placement) - 1;
    const std::uint64_t need_bytes = staged_bytes_at(g->ep.h, want);
    if (need_bytes + 4096 > g->smem_optin)
      throw resource_error("requested placement does not fit in shared memory");
    g->place = want;
    g->place_fixed = true;
  });
}

int pbn_gpu_info(const pbn_gpu* g, uint32_t* lpt, uint32_t* tables_in_smem, uint64_t* smem_bytes,
                 uint64_t* plan_bytes, uint32_t* warps_per_cta) {
  return guard([&] {
    need(g, "gpu");
    if (lpt) *lpt = g->last_lpt ? g->last_lpt : g->lpt_fixed;
    // the placement the last launch ran (run_device may step down from the
    // configured one when the ensemble's state does not fit next to it)
    const int place = g->last_place >= 0 ? g->last_place : g->place;
    if (tables_in_smem) *tables_in_smem = static_cast<uint32_t>(place);
    if (smem_bytes) *smem_bytes = staged_bytes_at(g->ep.h, place);
    if (plan_bytes) *plan_bytes = g->ep.blob.size();
    if (warps_per_cta) *warps_per_cta = g->last_warps;
  });
}

int pbn_gpu_run(pbn_gpu* g, const pbn_run_args* a, uint64_t* states, uint64_t* counts,
                uint64_t* node_counts) {
  return guard([&] {
    need(g, "gpu");
    need(a, "args");
    need(states, "states");
    need(counts, "counts");
    ck(cudaSetDevice(g->device), "cudaSetDevice");
    const std::size_t words = pbn_state_words(g->ep.h.n_kept);
    if (a->n_traj > g->cap_traj) {
      if (g->d_states) cudaFree(g->d_states);
      if (g->d_counts) cudaFree(g->d_counts);
      g->d_states = g->d_counts = nullptr;
      g->cap_traj = 0;
      ck(cudaMalloc(&g->d_states, 8 * words * a->n_traj), "cudaMalloc states");
      ck(cudaMalloc(&g->d_counts, 8 * PBN_COUNT_FIELDS * static_cast<std::size_t>(a->n_traj)),
         "cudaMalloc counts");
      g->cap_traj = a->n_traj;
    }
    if (a->n_traj == 0) return;
    ck(cudaMemcpy(g->d_states, states, 8 * words * a->n_traj, cudaMemcpyHostToDevice), "H2D");
    // optional per-trajectory buffers: host -> device copies around the launch
    pbn_run_args da = *a;
    std::uint8_t* d_tprev = nullptr;
    std::uint32_t* d_series = nullptr;
    const std::size_t series_bytes = 4 * a->series_stride * a->n_traj;
    if (a->tprev) {
      d_tprev = ws_take<std::uint8_t>(*g, 6, a->n_traj);
      ck(cudaMemcpy(d_tprev, a->tprev, a->n_traj, cudaMemcpyHostToDevice), "H2D");
      da.tprev = d_tprev;
    }
    if (a->series) {
      d_series = ws_take<std::uint32_t>(*g, 7, series_bytes / 4);
      ck(cudaMemcpy(d_series, a->series, series_bytes, cudaMemcpyHostToDevice), "H2D");
      da.series = d_series;
    }
    std::uint64_t* d_nc = nullptr;
    const std::size_t nc_bytes = 8ull * g->ep.h.n_kept * a->n_traj;
    if (a->flags & PBN_RUN_NODE_COUNTS) {
      need(node_counts, "node_counts");
      d_nc = ws_take<std::uint64_t>(*g, 8, nc_bytes / 8);
      ck(cudaMemset(d_nc, 0, nc_bytes), "memset");
    }
    run_device(*g, da, g->d_states, g->d_counts, d_nc, nullptr);
    if (d_nc) ck(cudaMemcpy(node_counts, d_nc, nc_bytes, cudaMemcpyDeviceToHost), "D2H");
    ck(cudaMemcpy(states, g->d_states, 8 * words * a->n_traj, cudaMemcpyDeviceToHost), "D2H");
    if (a->tprev) ck(cudaMemcpy(a->tprev, d_tprev, a->n_traj, cudaMemcpyDeviceToHost), "D2H");
    if (a->series) ck(cudaMemcpy(a->series, d_series, series_bytes, cudaMemcpyDeviceToHost), "D2H");
    ck(cudaMemcpy(counts, g->d_counts, 8 * PBN_COUNT_FIELDS * static_cast<std::size_t>(a->n_traj),
                  cudaMemcpyDeviceToHost),
       "D2H");
  });
}

// alias_table::next(rng) on one uniform (alias.hpp:70-76; the group draw of
// engine.hpp:284-290 is the same rule on the group's slice).
static std::uint32_t alias_next(double u01, const double* cut, const std::uint32_t* alias,
                                std::uint32_t n) {
  const double u = u01 * static_cast<double>(n);
  std::uint32_t i = static_cast<std::uint32_t>(u);
  if (i >= n) i = n - 1;
  return (u - static_cast<double>(i)) < cut[i] ? i : alias[i];
}

int pbn_gpu_run_scripted(pbn_gpu* g, const pbn_run_args* a, const double* draws, uint64_t n_draws,
                         uint64_t* states, uint64_t* counts, uint64_t* consumed) {
  return guard([&] {
    need(g, "gpu");
    need(a, "args");
    need(draws, "draws");
    need(states, "states");
    const auto& st = g->st;
    const dev_plan_header& h = g->ep.h;
    if (st.pert_mode != 0) throw std::invalid_argument("scripted replay serves grouped plans (pert_mode 0)");
    if (n_draws == 0) throw std::invalid_argument("empty script");
    if (a->step_begin != 0 || a->flags != 0 || a->tprev || a->series || a->thin_mode != 0)
      throw std::invalid_argument("scripted replay: step_begin 0, no flags, no carried samples or series");
    if (a->n_traj == 0) return;
    const std::uint32_t A = static_cast<std::uint32_t>(st.a_size.size());
    const std::uint32_t nb0 = (st.groups + st.has_leaf + 3) / 4;
    const std::uint64_t bps = nb0 + (A + 3) / 4;
    const std::uint64_t blocks = static_cast<std::uint64_t>(a->n_traj) * a->n_steps * bps;
    if (blocks > (1ull << 26)) throw resource_error("script too long (2^26 draw blocks at most)");
    // slack: the kernel computes whole chunks of 32 blocks past a region's last draw
    std::vector<std::uint32_t> hi(4 * (blocks + 64), 0u), lo(4 * (blocks + 64), 0u);
    // Every decision is made on the device in integers on r53 = floor(u * 2^53);
    // a script value that is not a multiple of 2^-53 is accepted only if the
    // reference's FP64 rule decides the same for u and for r53 * 2^-53.
    auto put = [&](std::uint64_t slot, double u, std::uint64_t& r53) {
      if (!(u >= 0.0 && u < 1.0)) throw std::invalid_argument("script draws must lie in [0, 1)");
      r53 = static_cast<std::uint64_t>(u * 9007199254740992.0);  // exact: a power-of-two scale
      const std::uint64_t raw = r53 << 11;
      hi[slot] = static_cast<std::uint32_t>(raw >> 32);
      lo[slot] = static_cast<std::uint32_t>(raw);
    };
    auto inexact = [](std::uint64_t i) {
      return std::invalid_argument("script draw " + std::to_string(i) +
                                   " is not a multiple of 2^-53 and its rounding changes a decision");
    };
    for (std::uint32_t t = 0; t < a->n_traj; ++t) {
      const double* row = draws + static_cast<std::size_t>(t) * n_draws;
      std::uint64_t pos = 0;
      auto next = [&]() { return row[pos++ % n_draws]; };
      for (std::uint64_t s = 0; s < a->n_steps; ++s) {
        const std::uint64_t base = 4 * ((static_cast<std::uint64_t>(t) * a->n_steps + s) * bps);
        bool perturbed = false;
        for (std::uint32_t i = 0; i < st.groups; ++i) {  // engine.hpp:259-266
          const double u = next();
          std::uint64_t r53;
          put(base + i, u, r53);
          std::uint64_t c = alias_next(u, st.pert_cut.data(), st.pert_alias.data(), st.size);
          const double uq = static_cast<double>(r53) * 0x1p-53;
          if (uq != u && alias_next(uq, st.pert_cut.data(), st.pert_alias.data(), st.size) != c)
            throw inexact(pos - 1);
          if (i + 1 == st.groups) c &= st.mask;
          perturbed = perturbed || c != 0;
        }
        if (perturbed) continue;  // engine.hpp:267
        if (st.has_leaf) {        // engine.hpp:268, reduction.hpp:98
          const double u = next();
          std::uint64_t r53;
          put(base + st.groups, u, r53);
          const double uq = static_cast<double>(r53) * 0x1p-53;
          if ((uq > st.t) != (u > st.t)) throw inexact(pos - 1);
          if (u > st.t) continue;
        }
        for (std::uint32_t j = 0; j < A; ++j) {  // engine.hpp:284-290
          const double u = next();
          std::uint64_t r53;
          put(base + 4ull * nb0 + j, u, r53);
          const double* cut = st.alias_cut.data() + st.a_begin[j];
          const std::uint32_t* idx = st.alias_idx.data() + st.a_begin[j];
          const double uq = static_cast<double>(r53) * 0x1p-53;
          if (uq != u && alias_next(uq, cut, idx, st.a_size[j]) != alias_next(u, cut, idx, st.a_size[j]))
            throw inexact(pos - 1);
        }
      }
      if (consumed) consumed[t] = pos;
    }
    ck(cudaSetDevice(g->device), "cudaSetDevice");
    pbn_run_args ua = *a;
    ua.stream = PBN_STREAM_U53;
    dev_run_params rp = make_params(*g, ua);
    const std::size_t words = pbn_state_words(h.n_kept);
    const std::size_t blk_bytes = 16 * (blocks + 64);
    std::uint64_t* d_states = ws_take<std::uint64_t>(*g, 0, words * a->n_traj);
    std::uint64_t* d_counts = ws_take<std::uint64_t>(*g, 1, static_cast<std::size_t>(a->n_traj) * PBN_COUNT_FIELDS);
    uint4* d_hi = ws_take<uint4>(*g, 3, blocks + 64);
    uint4* d_lo = ws_take<uint4>(*g, 4, blocks + 64);
    ck(cudaMemcpy(d_states, states, 8 * words * a->n_traj, cudaMemcpyHostToDevice), "H2D");
    ck(cudaMemcpy(d_hi, hi.data(), blk_bytes, cudaMemcpyHostToDevice), "H2D");
    ck(cudaMemcpy(d_lo, lo.data(), blk_bytes, cudaMemcpyHostToDevice), "H2D");
    rp.script_hi = d_hi;
    rp.script_lo = d_lo;
    rp.script_bps = bps;
    // one trajectory per warp; warps per CTA by the shared memory the states take
    const std::size_t slot_bytes = 4 * ((2 * h.sw32 + 32 * 4 * kChunkBlocks + 3) & ~3u);
    std::uint32_t warps = static_cast<std::uint32_t>(std::min<std::size_t>(8, (g->smem_optin - 64) / slot_bytes));
    if (warps == 0) throw resource_error("trajectory state does not fit in shared memory");
    g->launches = 0;
    ck(launch_ensemble_script(h, g->d_blob, warps, rp, d_states, d_counts, nullptr), "scripted launch");
    g->launches = 1;
    g->last_lpt = 32;
    g->last_warps = warps;
    g->last_place = 0;
    g->last_kernel = "subwarp_script<lpt=32,gather=smem,stream=u53,place=global,warps=" + std::to_string(warps) + ">";
    ck(cudaMemcpy(states, d_states, 8 * words * a->n_traj, cudaMemcpyDeviceToHost), "D2H");
    if (counts)
      ck(cudaMemcpy(counts, d_counts, 8 * PBN_COUNT_FIELDS * static_cast<std::size_t>(a->n_traj),
                    cudaMemcpyDeviceToHost), "D2H");
  });
}

int pbn_gpu_run_device(pbn_gpu* g, const pbn_run_args* a, uint64_t* d_states, uint64_t* d_counts,
                       uint64_t* d_node_counts, void* stream) {
  return guard([&] {
    need(g, "gpu");
    need(a, "args");
    run_device(*g, *a, d_states, d_counts, d_node_counts, static_cast<cudaStream_t>(stream));
  });
}

uint32_t pbn_gpu_last_launches(const pbn_gpu* g) { return g ? g->launches : 0; }

static void copy_str(const std::string& s, char* buf, size_t cap, size_t* len_out) {
  if (len_out) *len_out = s.size();
  if (buf && cap) {
    const std::size_t k = std::min(cap - 1, s.size());
    std::memcpy(buf, s.data(), k);
    buf[k] = 0;
  }
}

int pbn_gpu_last_kernel(const pbn_gpu* g, char* buf, size_t cap, size_t* len_out) {
  return guard([&] {
    need(g, "gpu");
    copy_str(g->last_kernel, buf, cap, len_out);
  });
}

int pbn_gpu_plan_launch(const pbn_gpu* g, uint32_t n_traj, uint32_t stream, uint32_t flags,
                        char* buf, size_t cap, size_t* len_out) {
  return guard([&] {
    need(g, "gpu");
    const launch_choice c = choose_launch(*g, n_traj, (flags & PBN_RUN_NODE_COUNTS) != 0, stream);
    copy_str(kernel_name(c, stream), buf, cap, len_out);
  });
}

void pbn_gpu_destroy(pbn_gpu* g) {
  if (!g) return;
  cudaSetDevice(g->device);
  if (g->d_blob) cudaFree(g->d_blob);
  if (g->d_states) cudaFree(g->d_states);
  if (g->d_counts) cudaFree(g->d_counts);
  for (auto& b : g->ws)
    if (b.p) cudaFree(b.p);
  delete g;
}

// Known-answer hook for the stream (tests): n counters (4 u32 each) -> blocks.
int pbn_philox_kat(const uint32_t* ctr, uint32_t n, uint64_t seed, uint32_t* out) {
  return guard([&] {
    uint4 *d_in = nullptr, *d_out = nullptr;
    ck(cudaMalloc(&d_in, 16 * static_cast<std::size_t>(n)), "malloc");
    ck(cudaMalloc(&d_out, 16 * static_cast<std::size_t>(n)), "malloc");
    ck(cudaMemcpy(d_in, ctr, 16 * static_cast<std::size_t>(n), cudaMemcpyHostToDevice), "H2D");
    ck(launch_philox_kat(d_in, static_cast<uint32_t>(seed), static_cast<uint32_t>(seed >> 32),
                         d_out, n, nullptr),
       "kat");
    ck(cudaMemcpy(out, d_out, 16 * static_cast<std::size_t>(n), cudaMemcpyDeviceToHost), "D2H");
    cudaFree(d_in);
    cudaFree(d_out);
  });
}

// ---- test hooks over host internals -----------------------------------------
uint32_t pbn_internal_lower_bound(const uint32_t* w, uint32_t n, uint64_t theta) {
  return partition_lower_bound(std::vector<std::uint32_t>(w, w + n), theta);
}

int pbn_internal_greedy_partition(const uint32_t* w, uint32_t n, uint32_t m, uint32_t* part_of) {
  return guard([&] {
    const auto parts = greedy_product_partition(std::vector<std::uint32_t>(w, w + n), m);
    for (uint32_t j = 0; j < parts.size(); ++j)
      for (auto idx : parts[j]) part_of[idx] = j;
  });
}

int pbn_internal_alias_build(const double* probs, uint32_t n, double* cut, uint32_t* alias) {
  return guard([&] {
    const walker_table t = build_walker(probs, n);
    std::copy(t.cut.begin(), t.cut.end(), cut);
    std::copy(t.alias.begin(), t.alias.end(), alias);
  });
}

int pbn_internal_plan_layout(const pbn_plan_view* view, uint64_t* out, uint32_t n_out) {
  return guard([&] {
    need(view, "view");
    need(out, "out");
    check_view(*view);
    const encoded_plan ep = encode_plan(*view);
    const dev_plan_header& h = ep.h;
    const uint64_t v[] = {h.off_pert53, h.off_pert32, h.off_groups, h.off_fns, h.off_grec,
                          h.off_acut, h.off_aidx, h.off_acell, h.off_arec, h.off_scol,
                          h.off_arec4, h.off_tables, h.off_fns_s, h.off_acell_s, h.core_bytes,
                          h.table_bytes, h.blob_bytes, ep.blob.size(), h.n_alias_groups,
                          h.n_single_alias, h.n_groups, h.sw32, h.rg_ok, h.single_compact};
    for (uint32_t i = 0; i < n_out && i < sizeof(v) / sizeof(v[0]); ++i) out[i] = v[i];
  });
}

int pbn_internal_alias53_pick(const double* cut, const uint32_t* alias, uint32_t n,
                              const uint64_t* raw, uint64_t m, uint32_t* pick,
                              uint8_t* took_fast) {
  return guard([&] {
    need(cut, "cut");
    need(alias, "alias");
    need(raw, "raw");
    need(pick, "pick");
    if (n < 2 || n > kA53MaxCells) throw std::invalid_argument("n must be in [2, 2048]");
    const std::vector<std::uint32_t> rec = alias53_records(cut, alias, n);
    for (uint64_t i = 0; i < m; ++i) {
      const std::uint64_t R = raw[i];
      bool rare = false;
      pick[i] = alias53_pick_int(rec.data(), n, static_cast<std::uint32_t>(R >> 32), rare);
      const bool fast = !rare;
      if (rare) {
        const std::uint64_t r53 = R >> 11;
        const std::uint32_t c = alias53_cell(r53, n);
        pick[i] = alias53_frac(r53, n) < cut[c] ? c : alias[c];
      }
      if (took_fast) took_fast[i] = fast ? 1 : 0;
    }
  });
}

}  // extern "C"

// ---- estimator backends --------------------------------------------------------
namespace {

template <class T>
struct dev_buf {
  T* p = nullptr;
  explicit dev_buf(std::size_t n) { ck(cudaMalloc(&p, sizeof(T) * (n ? n : 1)), "cudaMalloc"); }
  ~dev_buf() {
    if (p) cudaFree(p);
  }
  dev_buf(const dev_buf&) = delete;
  dev_buf& operator=(const dev_buf&) = delete;
  void swap(dev_buf& o) { std::swap(p, o.p); }
};

// Device ensemble: states, carried thin samples, pilot series and count
// records stay in HBM; each round returns 8 pooled counters. The pilot series
// buffer starts at the requested pilot length and grows (row copy) only when
// the estimator widens the pilot; its capacity bound is 2^33 bits in total.
class device_backend : public estimator_backend {
 public:
  device_backend(pbn_gpu& g, const pbn_estimate_request& req, const std::uint32_t* bits,
                 const std::uint8_t* vals, std::uint32_t n_pred)
      : g_(g), req_(req), bits_(bits), vals_(vals), n_pred_(n_pred),
        words_(pbn_state_words(g.ep.h.n_kept)),
        cap_(std::min<std::uint64_t>(1ull << 22,
                                     std::max<std::uint64_t>(1024, (1ull << 33) / std::max(1u, req.n_traj)))),
        stride_(std::min<std::uint64_t>((cap_ + 31) / 32,
                                        (std::max<std::uint64_t>(req.pilot, 100) + 32) / 32)),
        states_{ws_take<std::uint64_t>(g, 0, static_cast<std::size_t>(req.n_traj) * words_)},
        counts_{ws_take<std::uint64_t>(g, 1, static_cast<std::size_t>(req.n_traj) * PBN_COUNT_FIELDS)},
        tprev_{ws_take<std::uint8_t>(g, 2, req.n_traj)},
        series_{ws_take<std::uint32_t>(g, 3, static_cast<std::size_t>(req.n_traj) * stride_)},
        red_{ws_take<unsigned long long>(g, 5, 16)} {
    ck(cudaMemset(series_.p, 0, sizeof(std::uint32_t) * req.n_traj * stride_), "memset");
  }
  std::uint32_t n_traj() const override { return req_.n_traj; }
  std::uint64_t series_capacity() const override { return cap_; }
  void upload(const std::uint64_t* host) {
    ck(cudaMemcpy(states_.p, host, 8 * words_ * req_.n_traj, cudaMemcpyHostToDevice), "H2D");
  }
  void download(std::uint64_t* host) {
    ck(cudaMemcpy(host, states_.p, 8 * words_ * req_.n_traj, cudaMemcpyDeviceToHost), "D2H");
  }
  // make every row hold series positions [0, bits)
  void reserve_series(std::uint64_t bits) {
    const std::uint64_t need = (bits + 31) / 32;
    if (need <= stride_) return;
    const std::uint64_t stride = std::min<std::uint64_t>((cap_ + 31) / 32, std::max(need, 2 * stride_));
    const int spare = series_slot_ == 3 ? 4 : 3;
    std::uint32_t* grown = ws_take<std::uint32_t>(g_, spare, static_cast<std::size_t>(req_.n_traj) * stride);
    ck(cudaMemset(grown, 0, sizeof(std::uint32_t) * req_.n_traj * stride), "memset");
    ck(cudaMemcpy2D(grown, 4 * stride, series_.p, 4 * stride_, 4 * stride_, req_.n_traj,
                    cudaMemcpyDeviceToDevice),
       "series grow");
    series_.p = grown;
    series_slot_ = spare;
    stride_ = stride;
  }
  void run(std::uint64_t step_begin, std::uint64_t n_steps, std::uint32_t kappa,
           std::uint32_t thin_mode, std::uint64_t series_bit0, bool series_init,
           std::uint64_t totals[PBN_COUNT_FIELDS]) override {
    for (int i = 0; i < PBN_COUNT_FIELDS; ++i) totals[i] = 0;
    if (series_bit0 != std::numeric_limits<std::uint64_t>::max())
      reserve_series(series_bit0 + n_steps);
    std::uint64_t done = 0;
    while (done < n_steps) {  // at most 2^31 steps per launch
      const std::uint64_t n = std::min<std::uint64_t>(n_steps - done, 1ull << 31);
      pbn_run_args a{};
      a.seed = req_.seed;
      a.traj_begin = req_.traj_begin;
      a.n_traj = req_.n_traj;
      a.stream = req_.stream;
      a.step_begin = step_begin + done;
      a.n_steps = n;
      a.pred_bits = bits_;
      a.pred_vals = vals_;
      a.n_pred = n_pred_;
      a.kappa = kappa;
      a.thin_mode = done == 0 ? thin_mode : 1u;
      a.tprev = tprev_.p;
      if (series_bit0 != std::numeric_limits<std::uint64_t>::max()) {
        a.series = series_.p;
        a.series_stride = stride_;
        a.series_bit0 = series_bit0 + done;
        a.series_init = done == 0 && series_init;
      }
      run_device(g_, a, states_.p, counts_.p, nullptr, nullptr);
      ck(launch_sum_counts(counts_.p, req_.n_traj, red_.p, nullptr), "sum counts");
      unsigned long long t[8];
      ck(cudaMemcpy(t, red_.p, sizeof t, cudaMemcpyDeviceToHost), "D2H");
      for (int i = 0; i < 8; ++i) totals[i] += t[i];
      done += n;
    }
  }
  void series_stats(std::uint32_t kappa, std::uint64_t len, std::uint64_t out[13]) override {
    ck(launch_series_stats(series_.p, req_.n_traj, stride_, len, kappa, red_.p, nullptr),
       "series stats");
    unsigned long long t[13];
    ck(cudaMemcpy(t, red_.p, sizeof t, cudaMemcpyDeviceToHost), "D2H");
    for (int i = 0; i < 13; ++i) out[i] = t[i];
  }

 private:
  pbn_gpu& g_;
  pbn_estimate_request req_;
  const std::uint32_t* bits_;
  const std::uint8_t* vals_;
  std::uint32_t n_pred_;
  std::uint64_t words_, cap_, stride_;
  // views of the engine's workspace slots (pbn_gpu::ws)
  template <class T>
  struct view {
    T* p;
  };
  view<std::uint64_t> states_, counts_;
  view<std::uint8_t> tprev_;
  view<std::uint32_t> series_;
  view<unsigned long long> red_;
  int series_slot_ = 3;
};

class callback_backend : public estimator_backend {
 public:
  explicit callback_backend(const pbn_estimator_backend& b) : b_(b) {}
  std::uint32_t n_traj() const override { return b_.n_traj; }
  std::uint64_t series_capacity() const override { return b_.series_capacity; }
  void run(std::uint64_t step_begin, std::uint64_t n_steps, std::uint32_t kappa,
           std::uint32_t thin_mode, std::uint64_t series_bit0, bool series_init,
           std::uint64_t totals[PBN_COUNT_FIELDS]) override {
    if (b_.run(b_.user, step_begin, n_steps, kappa, thin_mode, series_bit0, series_init ? 1 : 0,
               totals) != 0)
      throw std::runtime_error("estimator backend run failed");
  }
  void series_stats(std::uint32_t kappa, std::uint64_t len, std::uint64_t out[13]) override {
    if (b_.series_stats(b_.user, kappa, len, out) != 0)
      throw std::runtime_error("estimator backend series_stats failed");
  }

 private:
  pbn_estimator_backend b_;
};

}  // namespace

extern "C" {

int pbn_estimate(pbn_gpu* g, const pbn_estimate_request* req, const uint32_t* pred_bits,
                 const uint8_t* pred_vals, uint32_t n_pred, uint64_t* states_inout,
                 pbn_estimate_result* out) {
  return guard([&] {
    need(g, "gpu");
    need(req, "request");
    need(out, "result");
    need(states_inout, "states");
    if (n_pred == 0) throw model_error("empty predicate");
    ck(cudaSetDevice(g->device), "cudaSetDevice");
    device_backend be(*g, *req, pred_bits, pred_vals, n_pred);
    be.upload(states_inout);
    *out = estimate_pooled(*req, be);
    be.download(states_inout);
  });
}

int pbn_estimate_with_backend(const pbn_estimate_request* req, const pbn_estimator_backend* be,
                              pbn_estimate_result* out) {
  return guard([&] {
    need(req, "request");
    need(be, "backend");
    need(out, "result");
    callback_backend cb(*be);
    *out = estimate_pooled(*req, cb);
  });
}

int pbn_series_stats_host(const uint32_t* series, uint32_t n_traj, uint64_t stride, uint64_t len,
                          uint32_t kappa, uint64_t* out13) {
  return guard([&] {
    need(series, "series");
    need(out13, "out");
    series_stats_host(series, n_traj, stride, len, kappa, out13);
  });
}

int pbn_series_stats_device(int device, const uint32_t* d_series, uint32_t n_traj, uint64_t stride,
                            uint64_t len, uint32_t kappa, uint64_t* out13) {
  return guard([&] {
    need(d_series, "series");
    need(out13, "out");
    ck(cudaSetDevice(device), "cudaSetDevice");
    dev_buf<unsigned long long> red(13);
    ck(launch_series_stats(d_series, n_traj, stride, len, kappa, red.p, nullptr), "series stats");
    unsigned long long t[13];
    ck(cudaMemcpy(t, red.p, sizeof t, cudaMemcpyDeviceToHost), "D2H");
    for (int i = 0; i < 13; ++i) out13[i] = t[i];
  });
}

double pbn_inverse_normal_cdf(double p) {
  try {
    return inverse_normal_cdf(p);
  } catch (const std::exception& e) {
    g_error = e.what();
    return std::numeric_limits<double>::quiet_NaN();
  }
}

}  // extern "C"
