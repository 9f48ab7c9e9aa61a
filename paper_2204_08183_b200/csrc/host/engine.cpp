// engine.cpp — survscan::Engine over the C ABI (include/gss.h) + status mapping.
#include "survscan/engine.hpp"

#include <cstdlib>
#include <string>

#include "../../../include/gss.h"
#include "survscan/errors.hpp"

namespace survscan {

[[noreturn]] void throw_status(int code) {
  const std::string msg = gss_last_error();
  switch (code) {
    case GSS_ERR_PARSE: throw ParseError(msg);
    case GSS_ERR_SCHEMA: throw SchemaError(msg);
    case GSS_ERR_DOMAIN: throw DomainError(msg);
    case GSS_ERR_INDEX: throw IndexError(msg);
    case GSS_ERR_DUPLICATE: throw DuplicateEntryError(msg);
    case GSS_ERR_INVALID_COLUMN: throw InvalidColumnError(msg);
    case GSS_ERR_NONPOS_DEN: throw NonPositiveDenominatorError(msg);
    case GSS_ERR_OVERFLOW: throw OverflowError(msg);
    case GSS_ERR_DEGENERATE: throw DegenerateCurveError(msg);
    case GSS_ERR_EMPTY_FOLD: throw EmptyFoldError(msg);
    default: throw DeviceError(msg.empty() ? "device error " + std::to_string(code) : msg);
  }
}

int device_count() { return gss_device_count(); }

int default_device() {
  if (const char* d = std::getenv("SURVSCAN_DEVICE")) return std::atoi(d);
  return 0;
}

static int model_code(Model m) { return m == Model::cox ? GSS_COX : GSS_FINE_GRAY; }

Engine::Engine(const SurvivalDataset& ds, Model model, ChunkPlan plan,
               std::size_t recompute_interval)
    : ds_(&ds), model_(model), plan_(plan), device_(default_device()) {
  plan_.validate();
  check(gss_engine_create(ds.device(device_), model_code(model),
                          static_cast<int64_t>(recompute_interval), nullptr, &h_));
}

Engine::Engine(const SurvivalDataset& ds, Model model, const std::vector<std::uint8_t>& row_mask,
               std::size_t recompute_interval, int device)
    : ds_(&ds), model_(model), device_(device < 0 ? default_device() : device) {
  if (!row_mask.empty() && row_mask.size() != ds.n())
    throw DomainError("row mask length differs from the dataset");
  check(gss_engine_create(ds.device(device_), model_code(model),
                          static_cast<int64_t>(recompute_interval),
                          row_mask.empty() ? nullptr : row_mask.data(), &h_));
}

Engine::~Engine() {
  if (h_) gss_engine_destroy(h_);
}

void Engine::load_beta(std::span<const double> beta) {
  check(gss_engine_load_beta(h_, beta.data(), static_cast<int64_t>(beta.size())));
}

void Engine::update_xbeta_sparse(std::size_t column, double delta) {
  check(gss_engine_update(h_, static_cast<int64_t>(column), delta));
}

void Engine::refresh() { check(gss_engine_refresh(h_)); }

GradHess Engine::grad_hessian(std::size_t column) {
  GradHess gh;
  check(gss_engine_grad_hessian(h_, static_cast<int64_t>(column), &gh.gradient, &gh.hessian,
                                &gh.fixed_term));
  return gh;
}

GradHess Engine::grad_hessian_separated(std::size_t column) {
  GradHess gh;
  check(gss_engine_grad_hessian_separated(h_, static_cast<int64_t>(column), &gh.gradient,
                                          &gh.hessian, &gh.fixed_term));
  return gh;
}

std::vector<GradHess> Engine::grad_hessian_all() {
  const std::size_t p = ds_->p();
  std::vector<double> g(p), h(p), f(p);
  check(gss_engine_grad_hessian_all(h_, g.data(), h.data(), f.data()));
  std::vector<GradHess> out(p);
  for (std::size_t j = 0; j < p; ++j) out[j] = {g[j], h[j], f[j]};
  return out;
}

double Engine::log_likelihood() const {
  double ll = 0.0;
  check(gss_engine_log_likelihood(h_, &ll));
  return ll;
}

std::span<const double> Engine::beta() const {
  beta_.resize(ds_->p());
  check(gss_engine_get_beta(h_, beta_.data(), static_cast<int64_t>(beta_.size())));
  return beta_;
}

std::span<const double> Engine::xbeta() const {
  xbeta_.resize(ds_->n());
  check(gss_engine_get_xbeta(h_, xbeta_.data(), static_cast<int64_t>(xbeta_.size())));
  return xbeta_;
}

std::span<const double> Engine::exp_xbeta() const {
  exp_xbeta_.resize(ds_->n());
  check(gss_engine_get_exp_xbeta(h_, exp_xbeta_.data(), static_cast<int64_t>(exp_xbeta_.size())));
  return exp_xbeta_;
}

std::span<const double> Engine::fixed_terms() const {
  fixed_.resize(ds_->p());
  check(gss_engine_get_fixed_terms(h_, fixed_.data(), static_cast<int64_t>(fixed_.size())));
  return fixed_;
}

const IpcwWeights& Engine::ipcw() const {
  // fixed at construction (censoring.cpp:65-90 runs once per Engine)
  if (!ipcw_valid_ && model_ == Model::fine_gray) {
    ipcw_.u.resize(ds_->n());
    ipcw_.g.resize(ds_->n());
    check(gss_engine_get_ipcw(h_, ipcw_.u.data(), ipcw_.g.data(), static_cast<int64_t>(ds_->n())));
  }
  ipcw_valid_ = true;
  return ipcw_;
}

std::vector<double> precompute_fixed_terms(const SurvivalDataset& ds) {
  Engine eng(ds, ds.has_competing() ? Model::fine_gray : Model::cox);
  auto f = eng.fixed_terms();
  return {f.begin(), f.end()};
}

std::size_t Engine::accepted_updates() const {
  int64_t a = 0, r = 0;
  check(gss_engine_counters(h_, &a, &r));
  return static_cast<std::size_t>(a);
}

std::size_t Engine::refresh_count() const {
  int64_t a = 0, r = 0;
  check(gss_engine_counters(h_, &a, &r));
  return static_cast<std::size_t>(r);
}

}  // namespace survscan
