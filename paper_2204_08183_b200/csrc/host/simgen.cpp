// simgen.cpp — synthetic survival designs (same model family as the
// reference simulators; this library's own counter-seeded random streams).
#include "survscan/simgen.hpp"

#include <algorithm>
#include <cmath>
#include <random>
#include <unordered_set>

#include "survscan/crossval.hpp"
#include "survscan/errors.hpp"

namespace survscan {

namespace {

constexpr std::size_t kBlockRows = 1 << 16;

void check(const SimConfig& c) {
  if (!(c.density >= 0.0 && c.density <= 1.0)) throw DomainError("density must lie in [0, 1]");
  if (!(c.beta_sparsity >= 0.0 && c.beta_sparsity <= 1.0))
    throw DomainError("beta_sparsity must lie in [0, 1]");
  if (!(c.p_mix > 0.0 && c.p_mix < 1.0)) throw DomainError("p_mix must lie in (0, 1)");
  if (c.censoring_quantile && !(*c.censoring_quantile > 0.0 && *c.censoring_quantile < 1.0))
    throw DomainError("censoring_quantile must lie in (0, 1)");
}

std::vector<double> true_effects(const SimConfig& c) {
  std::mt19937_64 rng(derive_seed(c.seed, 0x5eed0001ULL));
  std::normal_distribution<double> z(0.0, 1.0);
  std::uniform_real_distribution<double> u(0.0, 1.0);
  std::vector<double> beta(c.p, 0.0);
  for (auto& b : beta) {
    const bool keep = u(rng) >= c.beta_sparsity;
    const double v = z(rng);
    if (keep) b = v;
  }
  return beta;
}

// rows -> (time, status) via `outcome(rng, xbeta)`; covariates are a uniform
// random k-subset of the columns with k ~ Binomial(p, density)
template <class Outcome>
SurvivalDataset generate(const SimConfig& c, const std::vector<double>& beta, Outcome outcome) {
  std::vector<double> t(c.n);
  std::vector<int> s(c.n);
  std::vector<std::int64_t> rows, cols;
  rows.reserve(static_cast<std::size_t>(double(c.n) * double(c.p) * c.density * 1.05) + 16);
  cols.reserve(rows.capacity());
  std::unordered_set<std::uint32_t> pick;
  for (std::size_t b0 = 0; b0 < c.n; b0 += kBlockRows) {
    std::mt19937_64 rng(derive_seed(c.seed, 0x5eed0002ULL, b0 / kBlockRows));
    std::binomial_distribution<long> k_of(static_cast<long>(c.p), c.density);
    for (std::size_t i = b0; i < std::min(c.n, b0 + kBlockRows); ++i) {
      const auto k = static_cast<std::size_t>(c.p ? k_of(rng) : 0);
      pick.clear();
      std::uniform_int_distribution<std::uint32_t> any(0, c.p ? static_cast<std::uint32_t>(c.p - 1) : 0);
      while (pick.size() < k) pick.insert(any(rng));
      std::vector<std::uint32_t> chosen(pick.begin(), pick.end());
      std::sort(chosen.begin(), chosen.end());
      double xb = 0.0;
      for (std::uint32_t j : chosen) {
        xb += beta[j];
        rows.push_back(static_cast<std::int64_t>(i));
        cols.push_back(j);
      }
      const auto [ti, si] = outcome(rng, xb);
      t[i] = ti;
      s[i] = si;
    }
  }
  if (c.censoring_quantile) {  // administrative cutoff at a type-7 quantile of the times
    std::vector<double> sorted = t;
    std::sort(sorted.begin(), sorted.end());
    const double h = *c.censoring_quantile * static_cast<double>(sorted.size() - 1);
    const auto lo = static_cast<std::size_t>(h);
    const double frac = h - static_cast<double>(lo);
    const double cut = (frac == 0.0 || lo + 1 == sorted.size())
                           ? sorted[lo]
                           : sorted[lo] + frac * (sorted[lo + 1] - sorted[lo]);
    for (std::size_t i = 0; i < c.n; ++i)
      if (t[i] > cut) {
        t[i] = cut;
        s[i] = 0;
      }
  }
  std::vector<double> ones(rows.size(), 1.0);
  return dataset_from_coo(t, s, rows, cols, ones, c.p);
}

}  // namespace

CoxSim simulate_cox(const SimConfig& c) {
  check(c);
  CoxSim out;
  out.true_beta = true_effects(c);
  out.data = generate(c, out.true_beta, [](std::mt19937_64& rng, double xb) {
    std::exponential_distribution<double> ev(std::exp(xb));
    return std::pair<double, int>(ev(rng), 1);
  });
  return out;
}

FineGraySim simulate_finegray(const SimConfig& c) {
  check(c);
  FineGraySim out;
  out.true_beta1 = true_effects(c);
  out.true_beta2.resize(c.p);
  for (std::size_t j = 0; j < c.p; ++j) out.true_beta2[j] = -out.true_beta1[j];
  const double log_q = std::log1p(-c.p_mix);
  out.data = generate(c, out.true_beta1, [&](std::mt19937_64& rng, double xb) {
    std::uniform_real_distribution<double> u(0.0, 1.0);
    const double r = std::exp(xb);
    const double p1 = -std::expm1(r * log_q);  // P(primary) = 1 - (1 - p_mix)^r
    if (u(rng) < p1) {
      // inverse of the primary subdistribution F1(t) = 1 - [1 - p_mix (1 - e^-t)]^r
      for (;;) {
        const double v = u(rng) * p1;
        const double w = -std::expm1(std::log1p(-v) / r) / c.p_mix;
        const double time = -std::log1p(-w);
        if (std::isfinite(time)) return std::pair<double, int>(time, 1);
      }
    }
    std::exponential_distribution<double> other(1.0 / r);  // competing: rate exp(-x'beta)
    return std::pair<double, int>(other(rng), 2);
  });
  return out;
}

}  // namespace survscan
