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

// Fused output stage (ppo_fused.cu): both skinny output layers' forward and
// backward around the loss head; h.mean / h.v / h.dmean / h.dv are unused.
struct PpoFusedArgs {
  PpoHeadArgs h;
  const void* ha;  // actor's last hidden activations [n_local, Ka] (dtype rows)
  int64_t ldha;
  int Ka;
  const float* Wa;  // actor output layer W [A, Ka], b [A]
  const float* ba;
  const void* wba;  // the same W as the Adam-refreshed bf16 staged rows (pitch ldwb)
  int64_t ldwb;
  const void* hc;  // critic's last hidden activations [n_local, Kc]
  int64_t ldhc;
  int Kc;
  const float* Wc;  // critic output layer w [1, Kc], b [1]
  const float* bc;
  void* dha;  // out: dZ of the actor's layer below (dtype rows)
  int64_t lddha;
  void* dhc;
  int64_t lddhc;
  float* parta;  // per-block [dW_a | db_a | colsum(dh_a)] partials
  int64_t plena;
  int csa;  // emit colsum(dh_a) (bias gradient of the layer below)
  float *gwa, *gba, *gcsa;  // reduction targets
  float* partc;
  int64_t plenc;
  int csc;
  float *gwc, *gbc, *gcsc;
  // optional (tensor-core variant): per-block loss / dlog_std partials as
  // floats [block][lossld] for the pass's reduction launch instead of the
  // last-CTA fold (block 0 carries the entropy-coefficient term)
  float* lossp;
  int64_t lossld;
};
bool ppo_fused_ok(int A, int Ka, int Kc);
// jobs: the partial reductions (2, or 3 with the loss partials), for the
// caller's next reduction launch; *njobs receives their count
int launch_ppo_fused(const PpoFusedArgs& f, int dtype, ReduceJob* jobs, int* njobs,
                     cudaStream_t s);
int ppo_head_partial_doubles(int64_t n_local, int A);
int launch_adv_stats(const float* adv, int64_t n, double* part, unsigned int* ticket, double* out,
                     cudaStream_t s);
int launch_adv_finalize(const double* sums, double* out, cudaStream_t s);
int launch_ppo_loss_finalize(const float* loss, const float* log_std, int A, double n,
                             double vcoef, double ecoef, int last_in_epoch, ul_opt_ctl* ctl,
                             ul_ppo_stats* st, cudaStream_t s);

}  // namespace ul
