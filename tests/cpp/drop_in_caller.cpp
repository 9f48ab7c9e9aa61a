// A caller written against the REFERENCE's public Engine / CCD API
// (/root/reference/proj/include/survscan/engine.hpp:33-90, ccd.hpp:13-72),
// compiled unchanged against this repo's mirror headers and linked with
// libsurvscan_b200 (device engine over the C ABI).  Exercises the surface a
// drop-in must keep: span-taking load_beta, const log_likelihood, span
// accessors, plan(), ChunkPlan::validate, IPCW accessor, fit_with_engine.
#include <cmath>
#include <cstdio>
#include <span>
#include <vector>

#include "survscan/ccd.hpp"
#include "survscan/dataset.hpp"
#include "survscan/engine.hpp"
#include "survscan/errors.hpp"

using namespace survscan;

static double objective_of(const Engine& eng) { return eng.log_likelihood(); }  // const Engine&

int main() {
  // 6 rows, 2 columns through the reference's builder (dataset.hpp:56-61, 105)
  RawData raw;
  raw.n_cols = 2;
  const double t[] = {5, 4, 3, 2, 2, 1};
  const int s[] = {1, 0, 1, 1, 0, 1};
  for (int i = 0; i < 6; ++i) raw.obs.push_back({t[i], s[i], 5 - i});
  raw.entries = {{0, 0, 1.0}, {2, 0, 1.0}, {3, 0, 1.0}, {1, 1, 0.5}, {4, 1, 2.0}, {5, 1, 1.5}};
  SurvivalDataset ds = sort_and_block(std::move(raw));
  ChunkPlan plan = ChunkPlan::serial();
  plan.validate();
  Engine eng(ds, Model::cox, plan, 100);
  const std::vector<double> b = {0.2, -0.1};
  eng.load_beta(b);                               // std::vector -> std::span<const double>
  eng.load_beta(std::span<const double>(b));
  const GradHess gh = eng.grad_hessian(0);
  const double ll = objective_of(eng);
  std::span<const double> beta = eng.beta();
  std::span<const double> xb = eng.xbeta();
  std::span<const double> ex = eng.exp_xbeta();
  std::span<const double> fx = eng.fixed_terms();
  const IpcwWeights& w = eng.ipcw();               // empty for cox
  if (beta.size() != 2 || xb.size() != 6 || ex.size() != 6 || fx.size() != 2 || !w.u.empty())
    return 2;
  if (eng.plan().chunk_size != plan.chunk_size) return 3;
  eng.update_xbeta_sparse(1, 0.05);
  if (eng.accepted_updates() != 1 || eng.refresh_count() != 0) return 4;
  PenaltySpec pen;
  pen.kind = PenaltyKind::l1;
  pen.strength = 0.1;
  FitConfig cfg;
  const FitResult fr = fit_with_engine(eng, pen, cfg);
  const StepOutcome st = coordinate_step(0.0, gh, pen, true, 1.0);
  try {
    eng.grad_hessian(7);
    return 5;
  } catch (const InvalidColumnError&) {
  }
  std::printf("drop-in caller ok: g=%.12g h=%.12g ll=%.12g fit cycles=%zu obj=%.12g step=%.6g\n",
              gh.gradient, gh.hessian, ll, fr.cycles, fr.objective, st.applied);
  return std::isfinite(fr.objective) ? 0 : 6;
}
