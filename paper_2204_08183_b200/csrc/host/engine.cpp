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

Engine::Engine(const SurvivalDataset& ds, Model model, ChunkPlan, std::size_t recompute_interval)
    : ds_(&ds), model_(model), device_(default_device()) {
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

void Engine::load_beta(const std::vector<double>& beta) {
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

double Engine::log_likelihood() {
  double ll = 0.0;
  check(gss_engine_log_likelihood(h_, &ll));
  return ll;
}

std::vector<double> Engine::beta() const {
  std::vector<double> b(ds_->p());
  check(gss_engine_get_beta(h_, b.data(), static_cast<int64_t>(b.size())));
  return b;
}

std::vector<double> Engine::xbeta() const {
  std::vector<double> v(ds_->n());
  check(gss_engine_get_xbeta(h_, v.data(), static_cast<int64_t>(v.size())));
  return v;
}

std::vector<double> Engine::exp_xbeta() const {
  std::vector<double> v(ds_->n());
  check(gss_engine_get_exp_xbeta(h_, v.data(), static_cast<int64_t>(v.size())));
  return v;
}

std::vector<double> Engine::fixed_terms() const {
  std::vector<double> v(ds_->p());
  check(gss_engine_get_fixed_terms(h_, v.data(), static_cast<int64_t>(v.size())));
  return v;
}

IpcwWeights Engine::ipcw() const {
  IpcwWeights w;
  if (model_ != Model::fine_gray) return w;
  w.u.resize(ds_->n());
  w.g.resize(ds_->n());
  check(gss_engine_get_ipcw(h_, w.u.data(), w.g.data(), static_cast<int64_t>(ds_->n())));
  return w;
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
