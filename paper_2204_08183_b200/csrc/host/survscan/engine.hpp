// survscan/engine.hpp — Engine with the reference surface
// (/root/reference/proj/include/survscan/engine.hpp:33-90), backed by the
// device engine of the C ABI (include/gss.h): state (beta, eta, exp(eta),
// IPCW) lives on the GPU; accessors copy it back.
#pragma once

#include <cstddef>
#include <cstdint>
#include <span>
#include <vector>

#include "survscan/censoring.hpp"
#include "survscan/dataset.hpp"
#include "survscan/errors.hpp"
#include "survscan/scan.hpp"

struct gss_engine;

namespace survscan {

enum class Model { cox, fine_gray };

struct GradHess {
  double gradient = 0.0;
  double hessian = 0.0;
  double fixed_term = 0.0;
};

// delta' X_j for every column (engine.hpp:27), computed on the device.
std::vector<double> precompute_fixed_terms(const SurvivalDataset& ds);

class Engine {
 public:
  explicit Engine(const SurvivalDataset& ds, Model model, ChunkPlan plan = {},
                  std::size_t recompute_interval = 100);
  // Engine over the rows with row_mask[i] != 0 only — identical to building it
  // on ds.subset_rows(those positions, true) (the CV fold representation).
  Engine(const SurvivalDataset& ds, Model model, const std::vector<std::uint8_t>& row_mask,
         std::size_t recompute_interval = 100, int device = -1);
  ~Engine();
  Engine(const Engine&) = delete;
  Engine& operator=(const Engine&) = delete;

  const SurvivalDataset& data() const { return *ds_; }
  Model model_kind() const { return model_; }
  const ChunkPlan& plan() const { return plan_; }
  int device() const { return device_; }

  void load_beta(std::span<const double> beta);
  void update_xbeta_sparse(std::size_t column, double delta);
  void refresh();
  GradHess grad_hessian(std::size_t column);
  // unfused three-pass path (engine.hpp:61), the fusion ablation
  GradHess grad_hessian_separated(std::size_t column);
  // all columns in one device launch (the batched sweep behind gamma_max)
  std::vector<GradHess> grad_hessian_all();
  double log_likelihood() const;

  // Views of host copies of the device state, refreshed by each call (valid
  // until the next call of the same accessor or the next mutation), as the
  // reference's spans are valid until the engine mutates (engine.hpp:65-71).
  std::span<const double> beta() const;
  std::span<const double> xbeta() const;
  std::span<const double> exp_xbeta() const;
  std::span<const double> fixed_terms() const;
  const IpcwWeights& ipcw() const;
  std::size_t accepted_updates() const;
  std::size_t refresh_count() const;

  gss_engine* handle() const { return h_; }

 private:
  const SurvivalDataset* ds_;
  Model model_;
  ChunkPlan plan_;
  int device_ = 0;
  gss_engine* h_ = nullptr;
  mutable std::vector<double> beta_, xbeta_, exp_xbeta_, fixed_;
  mutable IpcwWeights ipcw_;
  mutable bool ipcw_valid_ = false;
};

// device for new engines: $SURVSCAN_DEVICE or 0
int default_device();
int device_count();

}  // namespace survscan
