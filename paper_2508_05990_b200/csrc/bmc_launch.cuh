// Launch-argument structs and host launchers shared by the kernel files and
// the C ABI (bmc_api.cu).  Host-only declarations; device code sees the structs.
#pragma once

#include "bmc_internal.cuh"

namespace bmc {

// Host-computed plan of one search-stage launch (shared-memory layout, TMA boxes).
struct StagePlan {
  int ty;         // candidate rows per thread (template parameter TY)
  int parts;      // (plane, chunk) slices per candidate column group; each owns a partial-sum array
  int threads;    // CTA size (multiple of 32, <= kMaxStageThreads)
  int shift;      // 1: sub-word candidate offsets funnel-shifted in the inner loop (template SHIFT)
  int copies;     // sub-word phases served from pre-shifted window copies built once per stage:
                  // 0 none, 1 one region per phase, 2 one region (the stage uses a single phase)
  int copy_words; // distance between phase copies (32-bit words; bank-skewed)
  int nmax;       // candidates (2r+1)^2
  int pg;         // planes staged per pass
  int bw;         // window box width (elements; 16-byte multiple, +1 word slack)
  int hwin;       // window rows (TMA box height)
  int wrows;      // allocated window rows per plane (hwin + slack)
  int cbw;        // current-block box width (elements)
  int use_tma;    // 1: TMA boxes, 0: plain-load staging (window too large for a box)
  int cur_bytes, win_bytes, tma_bytes;
  int off_sad, off_klist, off_cur, off_win;
  int smem;
  int debug;      // measurement switches (BMC_DEBUG_SKIP): 1 skip selection, 2 skip screening
  // host-precomputed fast-division magics (fastdiv_magic) of the CTA-uniform divisors
  unsigned long long mG, mncg, mrho, mcpr, ms, mparts, mgw, mcells, mper;
  int split;      // split the partial last warp's items into one-unit sub-items (single-pass plans)
  int per;        // units per part (single-pass plans), 0 = compute on device
  int sea;        // 1: successive-elimination screening first (dense screening only as fallback)
  int off_vc;     // byte offset of the SEA column-sum region ([P][G][bw] uint16 (u8) / uint32 (u16))
  int sea_cap;    // max survivors per CTA before falling back to dense screening
  int vcs;        // SEA column-sum row stride (elements; an odd number of 32-bit words: no bank conflicts)
};

#ifndef BMC_STAGE_THREADS
#define BMC_STAGE_THREADS 416
#endif
constexpr int kMaxStageThreads = BMC_STAGE_THREADS;  // max CTA size of the search kernel

struct StageLaunch {
  const void* planes;       // current-frame plane buffer
  const void* ref_planes;   // reference-frame plane buffer (== planes for clips)
  bmc_fme_params prm;
  StagePlan plan;
  const int32_t* cur_index;
  const int32_t* ref_index;
  int level, final_level, b, gw, gh, n_pairs;
  int kblk;                 // horizontally adjacent blocks per CTA (shared-centre stages), >= 1
  int first, last;          // first / last searched stage of the level
  int r, s;
  int extra_evals;          // range-0 stages folded into this launch's candidate count
  const int32_t* parent_mv;
  const double* parent_e;
  const uint8_t* parent_matched;
  int32_t* mv;
  double* energy;
  uint8_t* matched;
  unsigned long long* evals;
  const double* tab16;
  int single;               // search_stage API: one block at (ox, oy), centre (cx, cy)
  int ox, oy, cx, cy;
  int32_t* nvalid_out;
  uint32_t gwg, total;      // set by the launcher: work items per block row / per launch
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
  // CaBR weight-free fallback (ring vote) on the flagged blocks of predicted frames:
  // flagged = final-level `matched` == 0, same frame / stream indexing as mv (cells, not cells*2)
  const uint8_t* matched;   // NULL: no refinement
  uint8_t* scratch;         // (streams, H, W) unrefined prediction of the current frame
};

int plan_stage(StagePlan& pl, const bmc_fme_params& p, int b, int r, int s, bool allow_tma, int kblk = 1);
int launch_fme_stage(const StageLaunch& a, int n_cur_frames, int n_ref_frames, dim3 grid, cudaStream_t st);
bool small_level_ok(const bmc_fme_params& p, int b);
int launch_fme_small(const StageLaunch& a, cudaStream_t st);
int launch_pack(const void* raw, int n_frames, int kind, const bmc_fme_params& p, void* planes, cudaStream_t st);
int launch_refine(const RefineArgs& a, cudaStream_t st);
int launch_decide(const DecideArgs& a, cudaStream_t st);
int launch_predict(const PredictArgs& a, int n_streams, cudaStream_t st);
int launch_predict_chain(const PredictArgs& a, int n_streams, int t_begin, int t_end, unsigned* barrier_ctr,
                         cudaStream_t st);
int launch_predict_features(const float* src, float* dst, int C, int H, int W, const int32_t* mv, int gw, int B,
                            int scale, cudaStream_t st);
int launch_block_energy(const double* a, const double* b, long long n, double lam, double tol, double* out,
                        cudaStream_t st);


}  // namespace bmc
