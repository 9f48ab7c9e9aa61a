// survscan/engine.hpp — Engine with the reference surface
// (/root/reference/proj/include/survscan/engine.hpp:33-90), backed by the
// device engine of the C ABI (include/gss.h): state (beta, eta, exp(eta),
// IPCW) lives on the GPU; accessors copy it back.
#pragma once

#include <cstddef>
#include <cstdint>
#include <vector>

#include "survscan/dataset.hpp"

struct gss_engine;

namespace survscan {

enum class Model { cox, fine_gray };

struct GradHess {
  double gradient = 0.0;
  double hessian = 0.0;
  double fixed_term = 0.0;
};

// The reference's CPU chunk plan; accepted for API compatibility, ignored by
// the device engine (its tiling is fixed by the dataset pack).
struct ChunkPlan {
  std::size_t chunk_size = 65536;
  unsigned worker_count = 0;
};

struct IpcwWeights {
  std::vector<double> u, g;
};

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
  int device() const { return device_; }

  void load_beta(const std::vector<double>& beta);
  void update_xbeta_sparse(std::size_t column, double delta);
  void refresh();
  GradHess grad_hessian(std::size_t column);
  // unfused three-pass path (engine.hpp:61), the fusion ablation
  GradHess grad_hessian_separated(std::size_t column);
  // all columns in one device launch (the batched sweep behind gamma_max)
  std::vector<GradHess> grad_hessian_all();
  double log_likelihood();

  std::vector<double> beta() const;
  std::vector<double> xbeta() const;
  std::vector<double> exp_xbeta() const;
  std::vector<double> fixed_terms() const;
  IpcwWeights ipcw() const;
  std::size_t accepted_updates() const;
  std::size_t refresh_count() const;

  gss_engine* handle() const { return h_; }

 private:
  const SurvivalDataset* ds_;
  Model model_;
  int device_ = 0;
  gss_engine* h_ = nullptr;
};

// device for new engines: $SURVSCAN_DEVICE or 0
int default_device();
int device_count();

}  // namespace survscan
