// survscan/simgen.hpp — synthetic designs of the same family as the
// reference's simulators (/root/reference/proj/include/survscan/simgen.hpp):
// binary covariates, sparse Gaussian effects, exponential (Cox) or
// subdistribution-mixture (Fine-Gray) times, optional administrative cutoff.
// Test/bench infrastructure; the random streams are this library's own.
#pragma once

#include <cstdint>
#include <optional>
#include <vector>

#include "survscan/dataset.hpp"

namespace survscan {

struct SimConfig {
  std::size_t n = 0;
  std::size_t p = 0;
  double density = 0.05;
  double beta_sparsity = 0.80;
  double p_mix = 0.5;
  std::uint64_t seed = 0;
  std::optional<double> censoring_quantile;
};

struct CoxSim {
  SurvivalDataset data;
  std::vector<double> true_beta;
};
struct FineGraySim {
  SurvivalDataset data;
  std::vector<double> true_beta1;
  std::vector<double> true_beta2;
};

CoxSim simulate_cox(const SimConfig& config);
FineGraySim simulate_finegray(const SimConfig& config);

}  // namespace survscan
