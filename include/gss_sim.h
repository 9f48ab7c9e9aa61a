/*
 * gss_sim.h — device generator of benchmark-scale synthetic survival data
 * (same design family as the reference's simulate_cox,
 * /root/reference/proj/src/simgen.cpp:108-122, with counter-based RNG streams).
 * Outputs the reference's sorted layout in pinned host memory, ready for
 * gss_dataset_pack().  Test/bench infrastructure; not on the CCD hot path.
 */
#ifndef GSS_SIM_H
#define GSS_SIM_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

typedef struct gss_sim_config {
  int64_t n, p;
  double density;            /* Bernoulli covariate density (simgen.cpp:69-77)   */
  double beta_sparsity;      /* P(true beta_j = 0) (simgen.cpp:31-39)            */
  uint64_t seed;
  double censoring_quantile; /* administrative cutoff quantile, <= 0: none       */
  double time_quantum;       /* t <- ceil(t*q)/q (Breslow ties), <= 0: none      */
  double p_mix;              /* > 0: Fine-Gray competing-risk design with primary
                                mixture mass p_mix (simgen.hpp:33-37); 0: Cox   */
} gss_sim_config;

typedef struct gss_sim_out {
  int64_t n, p, nnz;
  double* times;      /* [n] sorted desc (ties by original id asc)            */
  int32_t* status;    /* [n] */
  int64_t* col_ptr;   /* [p+1] */
  int32_t* row_idx;   /* [nnz] ascending sorted positions per column          */
  double* beta_true;  /* [p] */
} gss_sim_out;

int gss_simulate_cox(const gss_sim_config* cfg, int device, gss_sim_out* out);
/* same, Fine-Gray design when cfg->p_mix > 0 (status 2 = competing event) */
int gss_simulate(const gss_sim_config* cfg, int device, gss_sim_out* out);
void gss_sim_free(gss_sim_out* out);
const char* gss_sim_last_error(void);

#ifdef __cplusplus
}
#endif
#endif
