// survscan/crossval.hpp — model selection with the reference API
// (/root/reference/proj/include/survscan/crossval.hpp:13-76).  Folds are row
// masks on the device-resident dataset (no subset copies); (grid, replicate)
// tasks are spread over the visible GPUs by the same slot-per-task merge, so
// the device count never changes the result.
#pragma once

#include <cstdint>
#include <vector>

#include "survscan/ccd.hpp"

namespace survscan {

struct CVConfig {
  std::uint32_t folds = 10;
  std::uint32_t repetitions = 10;
  std::vector<double> grid;
  std::uint64_t seed = 0;
  std::uint32_t parallel_replicates = 1;  // worker threads per device
  void validate() const;
};

struct CVPoint {
  double strength = 0.0;
  double mean_loglik = 0.0;
  double spread = 0.0;
  std::uint32_t evaluations = 0;
};

struct CVResult {
  std::vector<CVPoint> points;
  double selected_value = 0.0;
  FitResult final_fit;
  std::uint32_t failed_replicates = 0;
};

std::uint64_t mix64(std::uint64_t x);
std::uint64_t derive_seed(std::uint64_t seed, std::uint64_t a, std::uint64_t b = 0);

std::vector<std::uint32_t> fold_assignment(std::size_t n, std::uint32_t folds,
                                           std::uint64_t seed, std::uint64_t grid_index,
                                           std::uint64_t replicate);
double held_out_loglik(const SurvivalDataset& ds, const std::vector<std::uint32_t>& fold_of,
                       std::uint32_t fold, Model model, const std::vector<double>& beta,
                       const ChunkPlan& plan = {});
double gamma_max(const SurvivalDataset& ds, Model model, const ChunkPlan& plan = {});
// the same on a given device (-1 = $SURVSCAN_DEVICE or 0)
double gamma_max(const SurvivalDataset& ds, Model model, int device);
std::vector<double> auto_grid(double top);
// Pieces of cross_validate for multi-process drivers (one process per GPU):
// the resolved grid, the event-free-fold precheck, the per-task fold scores
// (task = grid_index * repetitions + replicate; failed => empty), and the
// task-ordered merge + final refit.
struct TaskScores {
  std::vector<double> fold_loglik;
  bool failed = false;
};
std::vector<double> cv_grid(const SurvivalDataset& ds, Model model, const CVConfig& cv,
                            const FitConfig& fit_config);
void cv_check_folds(const SurvivalDataset& ds, const CVConfig& cv, std::size_t n_grid);
std::vector<TaskScores> cv_run_tasks(const SurvivalDataset& ds, Model model, PenaltyKind kind,
                                     const std::vector<double>& grid, const CVConfig& cv,
                                     const FitConfig& fit_config,
                                     const std::vector<std::size_t>& tasks,
                                     const std::vector<int>& devices = {});
CVResult cv_merge(const SurvivalDataset& ds, Model model, PenaltyKind kind,
                  const std::vector<double>& grid, const CVConfig& cv, const FitConfig& fit_config,
                  const std::vector<TaskScores>& all_tasks, bool refit = true);

// devices: GPUs to spread the tasks over (empty = all visible)
CVResult cross_validate(const SurvivalDataset& ds, Model model, PenaltyKind kind,
                        const CVConfig& cv, const FitConfig& fit_config = {},
                        const std::vector<int>& devices = {});

struct BootstrapDraw {
  double value = 0.0;  // fitted beta[coefficient_index] of the resample
  bool failed = false;
};
struct BootstrapInterval {
  double lower = 0.0;
  double upper = 0.0;
  std::uint32_t failed_resamples = 0;
};
// bootstrap_interval (src/crossval.cpp:218-257) with the resamples' fits
// batched on each device and dealt over devices (and, through the pieces
// below, over ranks): resample b draws from derive_seed(seed, 0, b) as the
// reference does, so the draws and the interval equal the reference's.
BootstrapInterval bootstrap_interval(const SurvivalDataset& ds, Model model,
                                     const PenaltySpec& penalty, const FitConfig& fit_config,
                                     std::size_t coefficient_index, std::uint32_t resamples = 200,
                                     std::uint64_t seed = 0, const std::vector<int>& devices = {});

// the sorted row positions of resample b (derive_seed(seed, 0, b) stream)
std::vector<std::uint32_t> bootstrap_indices(std::size_t n, std::uint64_t seed,
                                            std::uint32_t resample);
// pieces for multi-process drivers: draws of the listed resamples, then the
// resample-ordered merge (> 10% failures -> DomainError, type-7 quantiles)
std::vector<BootstrapDraw> bootstrap_run(const SurvivalDataset& ds, Model model,
                                         const PenaltySpec& penalty, const FitConfig& fit_config,
                                         std::size_t coefficient_index,
                                         const std::vector<std::uint32_t>& resample_ids,
                                         std::uint64_t seed, const std::vector<int>& devices = {});
BootstrapInterval bootstrap_merge(const std::vector<BootstrapDraw>& draws,
                                  std::uint32_t resamples);

}  // namespace survscan
