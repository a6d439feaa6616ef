// Launch-argument structs and host launchers shared by the kernel files and
// the C ABI (bmc_api.cu).  Host-only declarations; device code sees the structs.
#pragma once

#include "bmc_internal.cuh"

namespace bmc {

struct SearchPlan {
  int ty[3];
  int pg;
  int nmax;
  int ref_words;
  int cur_words;
  int smem;
};
struct LevelArgs {
  const void* planes;
  bmc_fme_params prm;
  SearchPlan plan;
  const int32_t* cur_index;
  const int32_t* ref_index;
  int level, final_level, b, gw, gh;
  const int32_t* parent_mv;
  const double* parent_e;
  const uint8_t* parent_matched;
  int32_t* mv;
  double* energy;
  uint8_t* matched;
  unsigned long long* evals;
  const double* tab16;
};
struct StageArgs {
  const void* cur;
  const void* ref;
  bmc_fme_params prm;
  SearchPlan plan;
  int ox, oy, b, cx, cy, r, s;
  int32_t* mv;
  double* energy;
  int32_t* nvalid;
  const double* tab16;
};
struct RefineArgs {
  const int32_t* mv_in;
  const double* e_in;
  int n_pairs, gh, gw, b, thr;
  const void* planes;
  bmc_fme_params prm;
  const int32_t* cur_index;
  const int32_t* ref_index;
  int32_t* mv_out;
  double* e_out;
  int32_t* replaced;
  const double* tab16;
};
struct DecideArgs {
  const double* energy;
  long long efs, ess;
  int n_streams, t_begin, t_end;
  bmc_select_params sp;
  double* acc;
  int32_t* fsk;
  int32_t* last_key;
  int32_t* kind;
  int32_t* ref;
  double* trigger;
  long long dss;
  int32_t* ref_next;
  int frames_per_stream;
  long long nleaf;  // leaves of numpy's pairwise tree over the coarse grid (host-computed)
};
struct PredictArgs {
  uint8_t* labels;
  long long fs, ss;
  const uint8_t* key_labels;
  int t;
  const int32_t* kind;
  const int32_t* ref;
  int ref_fixed;
  long long kss;
  int H, W;
  const int32_t* mv;
  long long mvfs, mvss;
  int gh, gw, B, scale;
};

int plan_level(SearchPlan& pl, const bmc_fme_params& p, int b);
int launch_fme_level(const LevelArgs& a, int n_pairs, cudaStream_t st);
int launch_stage(const StageArgs& a, cudaStream_t st);
int launch_pack(const void* raw, int n_frames, int kind, const bmc_fme_params& p, void* planes, cudaStream_t st);
int launch_refine(const RefineArgs& a, cudaStream_t st);
int launch_decide(const DecideArgs& a, cudaStream_t st);
int launch_predict(const PredictArgs& a, int n_streams, cudaStream_t st);
int launch_predict_features(const float* src, float* dst, int C, int H, int W, const int32_t* mv, int gw, int B,
                            int scale, cudaStream_t st);
int launch_block_energy(const double* a, const double* b, long long n, double lam, double tol, double* out,
                        cudaStream_t st);


}  // namespace bmc
