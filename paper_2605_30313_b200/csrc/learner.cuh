// Learner-plan internals shared by heads.cu / learner.cu / sac.cu.
#pragma once
#include "internal.cuh"

namespace ul {

constexpr int kAdvStatBlocks = 256;

struct PpoHeadArgs {
  int64_t n_local;
  double n_global;
  int A;
  const float* mean;
  int64_t ld_mean;
  const float* log_std;
  const float* act;
  int64_t ld_act;
  const float* blogp;
  const float* adv;
  const float* ret;
  const float* oldv;
  const float* v;
  int64_t ld_v;
  const double* adv_stats;  // [mean, std]
  double clip, vcoef;
  int clipped_v;
  float* dmean;
  int64_t ld_dmean;
  float* dv;
  double* part;
  unsigned int* ticket;
  float* dlogstd_out;
  float* loss_out;  // [pol_sum, val_sum, kl_sum]
  double ent_coef_add;
};

int launch_ppo_head(const PpoHeadArgs& a, cudaStream_t s);
int ppo_head_partial_doubles(int64_t n_local, int A);
int launch_adv_stats(const float* adv, int64_t n, double* part, unsigned int* ticket, double* out,
                     cudaStream_t s);
int launch_ppo_loss_finalize(const float* loss, const float* log_std, int A, double n,
                             double vcoef, double ecoef, int last_in_epoch, ul_opt_ctl* ctl,
                             ul_ppo_stats* st, cudaStream_t s);

}  // namespace ul
