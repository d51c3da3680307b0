// Pooled two-state Markov chain steady-state estimator over an ensemble of
// independent trajectories — the ensemble form of the reference's
// estimate_steady_state (estimator.hpp:137-244), independent of where the
// trajectories are stepped (device backend, or a test backend over the oracle).
//
// Pooling rule: all M trajectories start from the caller's states and run the
// same schedule. Every statistic of the reference's single chain is replaced by
// its sum over the M chains: the raw pilot transition counts, the BIC triple
// counts n_ijk(kappa) and thinned pair counts of the stored pilot series, and
// the thinned transition counts of the sampling phase. The burn-in applies to
// each trajectory; the required sample size N is met by the pooled number of
// recorded steps (each trajectory records ceil((N - recorded) / M) more steps
// per refinement). The estimate is pooled ones / pooled recorded. For M = 1
// this is exactly the reference algorithm (tests/test_estimator.py checks the
// one-trajectory estimate bit-for-bit against the unmodified reference on the
// same stream).
#pragma once

#include <cstdint>

#include "../../../include/pbn_b200.h"

namespace pbn_b200 {

class estimator_backend {
 public:
  virtual ~estimator_backend() = default;
  virtual std::uint32_t n_traj() const = 0;
  virtual std::uint64_t series_capacity() const = 0;  // stored pilot bits per trajectory
  // Advance every trajectory by n_steps from global step step_begin; pooled
  // counts (PBN_COUNT_FIELDS) out. kappa/thin_mode as in pbn_run_args.
  // series_bit0 == UINT64_MAX: no series; else record step i at bit
  // series_bit0 + i (and the input state's bit at series_bit0 - 1 if init).
  virtual void run(std::uint64_t step_begin, std::uint64_t n_steps, std::uint32_t kappa,
                   std::uint32_t thin_mode, std::uint64_t series_bit0, bool series_init,
                   std::uint64_t totals[PBN_COUNT_FIELDS]) = 0;
  // Pooled statistics of the stored series over positions [0, len):
  // out[0..8) n_ijk (t = 2k, 3k, ...), out[8..12) thinned pairs (t = k, 2k, ...),
  // out[12] ones in positions [1, len).
  virtual void series_stats(std::uint32_t kappa, std::uint64_t len, std::uint64_t out[13]) = 0;
};

double inverse_normal_cdf(double p);  // estimator.hpp:26-57

// Pooled series statistics on host bit rows (test backends; device has a kernel).
void series_stats_host(const std::uint32_t* series, std::uint32_t n_traj, std::uint64_t stride,
                       std::uint64_t len, std::uint32_t kappa, std::uint64_t out[13]);

pbn_estimate_result estimate_pooled(const pbn_estimate_request& req, estimator_backend& be);

}  // namespace pbn_b200
