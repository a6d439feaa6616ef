// Float64 plane-stack motion search: the reference's ndarray input form
// (fme.py:188-190 -- a (P,H,W) stack is used as-is, no normalisation) and the
// general fallback for geometries the integer SIMD kernels do not cover (block
// sizes outside 8..64, any search_stage block size).  Every candidate is
// evaluated exactly: d = |r - c| in float64, numpy's pairwise sum over the
// flattened (P,b,b) difference, C = #(d > tol), E = (1-lam)*S/n + lam*C/n
// (fme.py:236-268); first minimum in canonical (dy, dx) order wins.
//
// One CTA (8 warps) per block of a level: warps take candidates round-robin,
// each candidate's energy is one warp's exact replay (power-of-two n >= 64) or
// one lane's sequential pairwise tree (other n); the CTA then takes the first
// minimum.  Levels, inheritance and masks follow estimate_motion
// (fme.py:324-392) exactly as the integer path does.
#include <cfloat>
#include <cstdint>

#include "../../include/bmc_ext.h"
#include "bmc_internal.cuh"

namespace bmc {

template <>
__device__ __forceinline__ double norm_sample<double>(double v, const double*) {
  return v;
}

namespace {

constexpr int kF64Threads = 256;

struct F64Stage {
  int range[3], step[3], n;
};

struct F64Args {
  const double* pc;
  const double* pr;
  int P, H, W;            // padded plane geometry (rows H, cols W, contiguous planes)
  int real_h, real_w;
  int b, gh, gw;
  int final_level;
  F64Stage st;
  double lam, oml, tol, split, refine;
  // parent level (nullptr at level 0)
  const int32_t* pmv;
  const double* pen;
  const uint8_t* pmatched;
  int pgw;
  // outputs
  int32_t* mv;
  double* energy;
  uint8_t* matched;
  unsigned long long* evals;
  // single-block mode (search_stage): origin given, no re-centring, n_valid out
  int single, ox, oy, cx, cy;
  int32_t* n_valid;
};

__device__ bool is_pow2_dev(int v) { return v > 0 && (v & (v - 1)) == 0; }

// exact energy of the candidate whose reference window starts at (rx, ry)
__device__ double candidate_energy(const F64Args& a, int ox, int oy, int rx, int ry) {
  const long long plane = (long long)a.H * a.W;
  const double* cur = a.pc + (long long)oy * a.W + ox;
  const double* ref = a.pr + (long long)ry * a.W + rx;
  const long long n = (long long)a.P * a.b * a.b;
  if (is_pow2_dev(a.b) && is_pow2_dev(a.P) && n >= 64) {  // perfect pairwise tree
    return exact_energy_generic<double>(cur, a.W, plane, ref, a.W, plane, a.b, a.P, nullptr, a.tol, a.oml, a.lam)
        .energy;
  }
  // general n: lane 0 walks numpy's pairwise tree sequentially
  double e = 0.0;
  if ((threadIdx.x & 31) == 0) {
    const int bb = a.b * a.b;
    auto value = [&](long long i) {
      const int p = int(i / bb), r = int(i % bb);
      const int y = r / a.b, x = r % a.b;
      return fabs(__dsub_rn(ref[p * plane + (long long)y * a.W + x], cur[p * plane + (long long)y * a.W + x]));
    };
    long long cnt = 0;
    for (long long i = 0; i < n; ++i) cnt += value(i) > a.tol;
    const double s = __dadd_rn(0.0, pairwise_tree([&](long long lo, int len) { return pairwise_leaf(value, lo, len); },
                                                  0, n));
    const double nd = (double)n;
    e = __dadd_rn(__dmul_rn(a.oml, __ddiv_rn(s, nd)), __dmul_rn(a.lam, __ddiv_rn((double)cnt, nd)));
  }
  return __shfl_sync(0xffffffffu, e, 0);
}

// one stage around (cx, cy); returns the number of valid candidates (0: none),
// best (mv, energy) in *bx, *by, *be (CTA-uniform).
__device__ int run_stage(const F64Args& a, int ox, int oy, int cx, int cy, int rng, int step, int* bx, int* by,
                         double* be, double* s_e, int* s_i) {
  const int side = 2 * rng + 1;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // valid rectangle of candidate indices (fme.py:250-253)
  double best = DBL_MAX;
  int best_i = INT32_MAX;
  for (int k = warp; k < side * side; k += kF64Threads / 32) {
    const int j = k / side, i = k % side;
    const int dx = cx + (i - rng) * step, dy = cy + (j - rng) * step;
    const int rx = ox + dx, ry = oy + dy;
    if (rx < 0 || ry < 0 || rx > a.W - a.b || ry > a.H - a.b) continue;
    const double e = candidate_energy(a, ox, oy, rx, ry);
    if (e < best) {  // k increases per warp: the first minimum is kept
      best = e;
      best_i = k;
    }
  }
  if (lane == 0) {
    s_e[warp] = best;
    s_i[warp] = best_i;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double e = DBL_MAX;
    int idx = INT32_MAX;
    for (int w = 0; w < kF64Threads / 32; ++w)
      if (s_i[w] != INT32_MAX && (s_e[w] < e || (s_e[w] == e && s_i[w] < idx))) {
        e = s_e[w];
        idx = s_i[w];
      }
    // valid count: product of the valid ranges per axis
    int nx = 0, ny = 0;
    for (int t = 0; t < side; ++t) {
      const int rx = ox + cx + (t - rng) * step, ry = oy + cy + (t - rng) * step;
      nx += (rx >= 0 && rx <= a.W - a.b);
      ny += (ry >= 0 && ry <= a.H - a.b);
    }
    s_i[kF64Threads / 32] = nx * ny;
    if (idx != INT32_MAX) {
      *bx = cx + (idx % side - rng) * step;
      *by = cy + (idx / side - rng) * step;
      *be = e;
    }
  }
  __syncthreads();
  const int n = s_i[kF64Threads / 32];
  __syncthreads();
  return n;
}

__global__ void __launch_bounds__(kF64Threads) fme_f64_kernel(F64Args a) {
  __shared__ double s_e[kF64Threads / 32];
  __shared__ int s_i[kF64Threads / 32 + 1];
  __shared__ int s_mv[2];
  __shared__ double s_best;
  const int cell = blockIdx.x;
  const int gx = a.single ? 0 : cell % a.gw, gy = a.single ? 0 : cell / a.gw;
  const int ox = a.single ? a.ox : gx * a.b, oy = a.single ? a.oy : gy * a.b;
  int sx = a.single ? a.cx : 0, sy = a.single ? a.cy : 0;
  double se = 0.0;
  if (a.pmv) {
    const int p = (gy >> 1) * a.pgw + (gx >> 1);
    if (a.pmatched[p]) {  // inherited: copy the parent (fme.py:352-359), matched stays set
      if (threadIdx.x == 0) {
        a.mv[2 * cell] = a.pmv[2 * p];
        a.mv[2 * cell + 1] = a.pmv[2 * p + 1];
        a.energy[cell] = a.pen[p];
        a.matched[cell] = 1;
      }
      return;
    }
    sx = a.pmv[2 * p];
    sy = a.pmv[2 * p + 1];
    se = a.pen[p];
  }
  if (threadIdx.x == 0) {
    s_mv[0] = sx;
    s_mv[1] = sy;
    s_best = se;
  }
  __syncthreads();
  unsigned long long evals = 0;
  for (int s = 0; s < a.st.n; ++s) {
    int cx = s_mv[0], cy = s_mv[1];
    int n = run_stage(a, ox, oy, cx, cy, a.st.range[s], a.st.step[s], &s_mv[0], &s_mv[1], &s_best, s_e, s_i);
    if (n == 0 && !a.single)  // re-centre on zero displacement (fme.py:310-313)
      n = run_stage(a, ox, oy, 0, 0, a.st.range[s], a.st.step[s], &s_mv[0], &s_mv[1], &s_best, s_e, s_i);
    evals += n;
    __syncthreads();
  }
  if (threadIdx.x != 0) return;
  if (a.single) {
    a.mv[0] = s_mv[0];
    a.mv[1] = s_mv[1];
    a.energy[0] = s_best;
    *a.n_valid = int(evals);
    return;
  }
  a.mv[2 * cell] = s_mv[0];
  a.mv[2 * cell + 1] = s_mv[1];
  a.energy[cell] = s_best;
  if (a.final_level) {
    const bool in_real = oy < a.real_h && ox < a.real_w;
    a.matched[cell] = !(s_best > a.refine && in_real);
  } else {
    a.matched[cell] = s_best <= a.split;
  }
  atomicAdd(a.evals, evals);
}

}  // namespace
}  // namespace bmc

using namespace bmc;

extern "C" int bmc_estimate_motion_f64(const double* cur_planes, const double* ref_planes, int planes, int pad_h,
                                       int pad_w, int real_h, int real_w, int n_levels, const int32_t* block_sizes,
                                       const int32_t* stage_range, const int32_t* stage_step, double lam,
                                       double sparsity_tolerance, double split_threshold,
                                       double refine_block_threshold, bmc_level_out* levels, void* stream) {
  if (!cur_planes || !ref_planes || !levels || !block_sizes || !stage_range || !stage_step || planes < 1 ||
      n_levels < 1 || n_levels > BMC_MAX_LEVELS || pad_h < 1 || pad_w < 1 || real_h > pad_h || real_w > pad_w) {
    set_error("estimate_motion_f64: invalid arguments");
    return BMC_E_ARG;
  }
  for (int l = 0; l < n_levels; ++l) {
    const int b = block_sizes[l];
    if (b < 1 || pad_h % b || pad_w % b) {
      set_error("estimate_motion_f64: padded planes must tile by every block size");
      return BMC_E_ARG;
    }
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  F64Args a{};
  a.pc = cur_planes;
  a.pr = ref_planes;
  a.P = planes;
  a.H = pad_h;
  a.W = pad_w;
  a.real_h = real_h;
  a.real_w = real_w;
  a.st.n = 3;
  for (int s = 0; s < 3; ++s) {
    a.st.range[s] = stage_range[s];
    a.st.step[s] = stage_step[s];
  }
  a.lam = lam;
  a.oml = 1.0 - lam;
  a.tol = sparsity_tolerance;
  a.split = split_threshold;
  a.refine = refine_block_threshold;
  for (int l = 0; l < n_levels; ++l) {
    a.b = block_sizes[l];
    a.gh = pad_h / a.b;
    a.gw = pad_w / a.b;
    a.final_level = l == n_levels - 1;
    a.mv = levels[l].mv;
    a.energy = levels[l].energy;
    a.matched = levels[l].matched;
    a.evals = levels[l].evals;
    if (l > 0) {
      a.pmv = levels[l - 1].mv;
      a.pen = levels[l - 1].energy;
      a.pmatched = levels[l - 1].matched;
      a.pgw = pad_w / block_sizes[l - 1];
    }
    int rc = cuda_status(cudaMemsetAsync(a.evals, 0, sizeof(unsigned long long), st), "estimate_motion_f64");
    if (rc) return rc;
    fme_f64_kernel<<<a.gh * a.gw, kF64Threads, 0, st>>>(a);
    if ((rc = cuda_status(cudaGetLastError(), "fme_f64_kernel"))) return rc;
  }
  return BMC_OK;
}

extern "C" int bmc_search_stage_f64(const double* cur_planes, const double* ref_planes, int planes, int height,
                                    int width, int origin_x, int origin_y, int block_size, int center_x,
                                    int center_y, int search_range, int step, double lam, double sparsity_tolerance,
                                    int32_t* mv_out, double* energy_out, int32_t* n_valid_out, void* stream) {
  if (!cur_planes || !ref_planes || !mv_out || !energy_out || !n_valid_out || planes < 1 || block_size < 1 ||
      search_range < 0) {
    set_error("search_stage_f64: invalid arguments");
    return BMC_E_ARG;
  }
  if (origin_x < 0 || origin_y < 0 || origin_x + block_size > width || origin_y + block_size > height) {
    set_error("block at (%d, %d) size %d lies outside the frame", origin_x, origin_y, block_size);
    return BMC_E_ARG;
  }
  F64Args a{};
  a.pc = cur_planes;
  a.pr = ref_planes;
  a.P = planes;
  a.H = height;
  a.W = width;
  a.real_h = height;
  a.real_w = width;
  a.b = block_size;
  a.gh = a.gw = 1;
  a.st.n = 1;
  a.st.range[0] = search_range;
  a.st.step[0] = step;
  a.lam = lam;
  a.oml = 1.0 - lam;
  a.tol = sparsity_tolerance;
  a.single = 1;
  a.ox = origin_x;
  a.oy = origin_y;
  a.mv = mv_out;
  a.energy = energy_out;
  a.n_valid = n_valid_out;
  a.cx = center_x;
  a.cy = center_y;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  fme_f64_kernel<<<1, kF64Threads, 0, st>>>(a);
  return cuda_status(cudaGetLastError(), "fme_f64_kernel");
}
