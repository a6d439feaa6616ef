// Ingest, MV refinement, AEM frame selection and motion compensation kernels
// (sm_100a).  All integer work is bit-exact by construction; the float64 work
// (energy re-evaluation, AEM accumulation and statistics) follows the
// reference's operation order with explicitly rounded intrinsics.
#include <cstdio>

#include <algorithm>
#include <mutex>

#include "bmc_internal.cuh"
#include "bmc_launch.cuh"

namespace bmc {

// ---------------------------------------------------------------------------
// Ingest: raw (frames, H, W) -> padded packed planes (frame_io.py:173-184,
// fme.py:181-211).  One thread writes one 32-bit word of one plane row; padded
// rows/columns replicate the last real sample (np.pad mode="edge").  Columns in
// [pad_w, pitch) are filled the same way so staging may read whole words.
// ---------------------------------------------------------------------------
template <typename Elem>
__device__ __forceinline__ uint32_t pack_pick(const Elem* __restrict__ row, int x0, int step, int w, int real_w) {
  constexpr int EPW = 4 / sizeof(Elem);
  uint32_t word = 0;
#pragma unroll
  for (int e = 0; e < EPW; ++e) {
    const int xs = min(w * EPW + e, real_w - 1);
    word |= (uint32_t)__ldg(row + x0 + step * xs) << (8 * sizeof(Elem) * e);
  }
  return word;
}

// One thread turns one 16-byte chunk of a raw row into two 32-bit words of
// each of the two CFA planes that row feeds (even / odd columns, split with
// PRMT): 16-byte loads, 8-byte stores.  A CTA walks kPackRows consecutive
// (frame, plane row, raw-row parity) rows; words that touch the right padding
// (or rows whose layout is not 16-byte aligned) take the clamped per-sample path.
constexpr int kPackRows = 8;
template <typename Elem>
__device__ __forceinline__ void pack_split(uint32_t a, uint32_t b, uint32_t& ev, uint32_t& od) {
  if constexpr (sizeof(Elem) == 1) {
    ev = __byte_perm(a, b, 0x6420);
    od = __byte_perm(a, b, 0x7531);
  } else {
    ev = __byte_perm(a, b, 0x5410);
    od = __byte_perm(a, b, 0x7632);
  }
}

template <typename Elem>
__global__ void pack_kernel(const Elem* __restrict__ raw, int kind, int H, int W, const bmc_fme_params p,
                            Elem* __restrict__ planes, int n_rows) {
  constexpr int EPW = 4 / sizeof(Elem);
  const int wpr = p.pitch / EPW;
  const bool bayer = kind == BMC_KIND_BAYER;
  const bool vec = bayer && (W % (4 * EPW)) == 0 && (p.pitch % (2 * EPW)) == 0 && (p.plane_stride % (2 * EPW)) == 0 &&
                   (p.frame_stride % (2 * EPW)) == 0;
  for (int rr = 0; rr < kPackRows; ++rr) {
    const int rowsel = blockIdx.x * kPackRows + rr;  // (f * pad_h + y) * par + parity
    if (rowsel >= n_rows) return;
    const int parity = bayer ? (rowsel & 1) : 0;
    const int fy = bayer ? (rowsel >> 1) : rowsel;
    const int f = fy / p.pad_h, y = fy - f * p.pad_h;
    const int ys = min(y, p.real_h - 1);
    const Elem* frame = raw + (long long)f * H * W;
    Elem* out = planes + (long long)f * p.frame_stride + (long long)y * p.pitch;
    if (!bayer) {
      const Elem* row = frame + (long long)ys * W;
      for (int w = threadIdx.x; w < wpr; w += blockDim.x) {
        const uint32_t word = ((w + 1) * EPW <= p.real_w && (W % EPW) == 0)
                                  ? __ldg(reinterpret_cast<const uint32_t*>(row) + w)
                                  : pack_pick<Elem>(row, 0, 1, w, p.real_w);
        reinterpret_cast<uint32_t*>(out)[w] = word;
      }
      continue;
    }
    const Elem* row = frame + (long long)(2 * ys + parity) * W;
    uint32_t* oe = reinterpret_cast<uint32_t*>(out + (2 * parity) * p.plane_stride);
    uint32_t* oo = reinterpret_cast<uint32_t*>(out + (2 * parity + 1) * p.plane_stride);
    for (int w2 = threadIdx.x; w2 < (wpr + 1) / 2; w2 += blockDim.x) {  // output word pair (2*w2, 2*w2+1)
      const int w = 2 * w2;
      if (vec && (w + 2) * EPW <= p.real_w && w + 1 < wpr) {
        const uint4 v = __ldg(reinterpret_cast<const uint4*>(row) + w2);  // 4*EPW raw samples
        uint2 e2, o2;
        pack_split<Elem>(v.x, v.y, e2.x, o2.x);
        pack_split<Elem>(v.z, v.w, e2.y, o2.y);
        reinterpret_cast<uint2*>(oe)[w2] = e2;
        reinterpret_cast<uint2*>(oo)[w2] = o2;
        continue;
      }
      for (int ww = w; ww < min(w + 2, wpr); ++ww) {
        uint32_t ev, od;
        if ((ww + 1) * EPW <= p.real_w && (W % (2 * EPW)) == 0) {
          const uint2 v = __ldg(reinterpret_cast<const uint2*>(row) + ww);  // 2*EPW raw samples
          pack_split<Elem>(v.x, v.y, ev, od);
        } else {
          ev = pack_pick<Elem>(row, 0, 2, ww, p.real_w);
          od = pack_pick<Elem>(row, 1, 2, ww, p.real_w);
        }
        oe[ww] = ev;
        oo[ww] = od;
      }
    }
  }
}

int launch_pack(const void* raw, int n_frames, int kind, const bmc_fme_params& p, void* planes, cudaStream_t st) {
  const int epw = 4 / p.elem_bytes;
  const int wpr = p.pitch / epw;
  const int par = kind == BMC_KIND_BAYER ? 2 : 1;
  const int rows_per_frame = p.pad_h * par;
  const int H = p.planes == 4 ? p.real_h * 2 : p.real_h;
  const int W = p.planes == 4 ? p.real_w * 2 : p.real_w;
  const int need = kind == BMC_KIND_BAYER ? (wpr + 1) / 2 : wpr;  // threads per row
  const int tpb = need <= 128 ? 128 : (need <= 256 ? 256 : 512);
  const long long n_rows = (long long)n_frames * rows_per_frame;
  if (n_rows > 0x7fffffffLL) {
    set_error("clip too large for the pack kernel");
    return BMC_E_ARG;
  }
  const unsigned grid = (unsigned)((n_rows + kPackRows - 1) / kPackRows);
  if (grid == 0) return BMC_OK;
  if (p.elem_bytes == 1)
    pack_kernel<uint8_t><<<grid, tpb, 0, st>>>((const uint8_t*)raw, kind, H, W, p, (uint8_t*)planes, (int)n_rows);
  else
    pack_kernel<uint16_t><<<grid, tpb, 0, st>>>((const uint16_t*)raw, kind, H, W, p, (uint16_t*)planes, (int)n_rows);
  const int rc = cuda_status(cudaGetLastError(), "pack_kernel");
  if (rc) return rc;
  return BMC_OK;
}

// ---------------------------------------------------------------------------
// fl(v / 65535) table for the uint16 exact replay.
// ---------------------------------------------------------------------------

// One table per device, built once under a lock.  The values are computed on
// the host (IEEE division is correctly rounded there too, so fl(v/65535) is the
// same double) and copied synchronously: no kernel on the legacy stream and no
// device-wide sync, so a later call cannot disturb another stream's work.  The
// first call must not happen inside a graph capture (the engines warm up first).
const double* norm_table_u16(int device) {
  static std::mutex mu;
  static double* tabs[64] = {nullptr};
  if (device < 0 || device >= 64) return nullptr;
  std::lock_guard<std::mutex> g(mu);
  if (!tabs[device]) {
    static double host[65536];
    for (int v = 0; v < 65536; ++v) host[v] = (double)v / 65535.0;
    double* t = nullptr;
    if (cudaMalloc(&t, 65536 * sizeof(double)) != cudaSuccess) return nullptr;
    if (cudaMemcpy(t, host, sizeof host, cudaMemcpyHostToDevice) != cudaSuccess) {
      cudaFree(t);
      return nullptr;
    }
    tabs[device] = t;
  }
  return tabs[device];
}

// ---------------------------------------------------------------------------
// MV refinement (mv_refine.py:17-69).  One warp per block: lane 0 takes the
// clipped 3x3 window of the INPUT field, the lower-middle order statistic of
// each component, and the Chebyshev test; replaced blocks re-evaluate their
// energy with the warp-cooperative exact replay on the padded planes.
// ---------------------------------------------------------------------------
__device__ __forceinline__ int lower_median(int* v, int n) {
  for (int i = 1; i < n; ++i) {  // insertion sort (<= 9 entries)
    const int x = v[i];
    int j = i - 1;
    while (j >= 0 && v[j] > x) {
      v[j + 1] = v[j];
      --j;
    }
    v[j + 1] = x;
  }
  return v[(n - 1) / 2];
}

template <typename Elem>
__global__ void __launch_bounds__(kThreads) refine_kernel(const RefineArgs a) {
  // Phase 1: one thread per block (clipped 3x3 window of the INPUT field, lower-middle
  // medians, Chebyshev test).  Phase 2: the CTA's replaced blocks whose new window is
  // in frame re-evaluate their energy, one warp per block (exact float64 replay).
  __shared__ double tab8[256];
  __shared__ int todo[kThreads];
  __shared__ int ntodo;
  const bmc_fme_params& p = a.prm;
  const double* tab = a.tab16;
  const long long per_pair = (long long)a.gh * a.gw;
  const long long cells = (long long)a.n_pairs * per_pair;
  const long long o = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (threadIdx.x == 0) ntodo = 0;
  __syncthreads();
  if (o < cells) {
    const int pair = (int)(o / per_pair);
    const int cell = (int)(o - pair * per_pair);
    const int gy = cell / a.gw, gx = cell - (cell / a.gw) * a.gw;
    const int32_t* mv = a.mv_in + (long long)pair * per_pair * 2;
    int vx[9], vy[9], n = 0;
    for (int y = max(0, gy - 1); y < min(a.gh, gy + 2); ++y)
      for (int x = max(0, gx - 1); x < min(a.gw, gx + 2); ++x) {
        vx[n] = mv[2 * (y * a.gw + x)];
        vy[n] = mv[2 * (y * a.gw + x) + 1];
        ++n;
      }
    const int medx = lower_median(vx, n), medy = lower_median(vy, n);
    int mx = mv[2 * cell], my = mv[2 * cell + 1], rep = 0;
    if (max(abs(mx - medx), abs(my - medy)) > a.thr) {
      mx = medx;
      my = medy;
      rep = 1;
    }
    a.mv_out[2 * o] = mx;
    a.mv_out[2 * o + 1] = my;
    a.e_out[o] = a.e_in[o];
    if (a.replaced) a.replaced[o] = rep;
    if (rep && a.planes) {
      const int rx = gx * a.b + mx, ry = gy * a.b + my;
      if (rx >= 0 && rx <= p.pad_w - a.b && ry >= 0 && ry <= p.pad_h - a.b)  // mv_refine.py:60
        todo[atomicAdd(&ntodo, 1)] = (int)threadIdx.x;
    }
  }
  __syncthreads();
  const int nt = ntodo;
  if (nt == 0) return;
  if (sizeof(Elem) == 1) {
    for (int v = threadIdx.x; v < 256; v += blockDim.x) tab8[v] = __ddiv_rn((double)v, (double)p.max_value);
    tab = tab8;
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int e = warp; e < nt; e += blockDim.x >> 5) {
    const long long oo = blockIdx.x * (long long)blockDim.x + todo[e];
    const int pair = (int)(oo / per_pair);
    const int cell = (int)(oo - pair * per_pair);
    const int gy = cell / a.gw, gx = cell - (cell / a.gw) * a.gw;
    const int mx = a.mv_out[2 * oo], my = a.mv_out[2 * oo + 1];
    const int ox = gx * a.b, oy = gy * a.b;
    const Elem* base = reinterpret_cast<const Elem*>(a.planes);
    const Elem* cur = base + (long long)a.cur_index[pair] * p.frame_stride + (long long)oy * p.pitch + ox;
    const Elem* ref = base + (long long)a.ref_index[pair] * p.frame_stride + (long long)(oy + my) * p.pitch + ox + mx;
    const double en = exact_energy_warp<Elem>(cur, ref, p.pitch, p.plane_stride, a.b, p.planes, tab,
                                              p.sparsity_tolerance, p.one_minus_lam, p.lam)
                          .energy;
    if (lane == 0) a.e_out[oo] = en;
  }
}

int launch_refine(const RefineArgs& a, cudaStream_t st) {
  const long long cells = (long long)a.n_pairs * a.gh * a.gw;
  const long long blocks = (cells + kThreads - 1) / kThreads;
  if (a.prm.elem_bytes == 1)
    refine_kernel<uint8_t><<<(unsigned)blocks, kThreads, 0, st>>>(a);
  else
    refine_kernel<uint16_t><<<(unsigned)blocks, kThreads, 0, st>>>(a);
  return cuda_status(cudaGetLastError(), "refine_kernel");
}

// ---------------------------------------------------------------------------
// AEM frame selection (frame_select.py:74-136).  One CTA per stream scans its
// frames in order: pooled = max over factor x factor children
// (frame_select.py:96), acc += pooled, trigger = max (exact) or numpy pairwise
// mean, key iff trigger > thr or frames_since_key+1 >= max_gop.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads) decide_kernel(const DecideArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ double red[kWarps];
  __shared__ double result;
  const int stream = blockIdx.x;
  const bmc_select_params& sp = a.sp;
  const int ncoarse = sp.coarse_h * sp.coarse_w;
  double* acc = a.acc + (long long)stream * ncoarse;
  const long long nleaf = a.nleaf;
  long long* leaf_lo = reinterpret_cast<long long*>(smem_raw);
  double* leaf_val = reinterpret_cast<double*>(leaf_lo + nleaf);
  int* leaf_len = reinterpret_cast<int*>(leaf_val + nleaf) + 1;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int t = a.t_begin; t < a.t_end; ++t) {
    const double* e = a.energy + stream * a.ess + t * a.efs;
    double mx = -INFINITY;
    for (int c = threadIdx.x; c < ncoarse; c += blockDim.x) {
      const int cy = c / sp.coarse_w, cx = c % sp.coarse_w;
      double pooled;
      if (sp.factor == 1) {
        pooled = e[c];
      } else {
        pooled = -INFINITY;
        for (int dy = 0; dy < sp.factor; ++dy)
          for (int dx = 0; dx < sp.factor; ++dx)
            pooled = fmax(pooled, e[(cy * sp.factor + dy) * sp.grid_w + cx * sp.factor + dx]);
      }
      const double v = __dadd_rn(acc[c], pooled);
      acc[c] = v;
      mx = fmax(mx, v);
    }
    double trig;
    if (!sp.statistic_mean) {
      for (int m = 16; m; m >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, m));
      if (lane == 0) red[warp] = mx;
      __syncthreads();
      if (threadIdx.x == 0) {
        double r = red[0];
        for (int w = 1; w < kWarps; ++w) r = fmax(r, red[w]);
        result = r;
      }
      __syncthreads();
      trig = result;
    } else {
      const double s = block_pairwise([&](long long i) { return acc[i]; }, ncoarse, leaf_lo, leaf_len, leaf_val,
                                      &result);
      trig = __ddiv_rn(s, (double)ncoarse);
    }
    __syncthreads();
    __shared__ int is_key_s;
    if (threadIdx.x == 0) {
      const int fsk = a.fsk[stream] + 1;
      const bool key = trig > sp.aem_threshold || (sp.has_max_gop && fsk >= sp.max_gop);
      int kind, ref;
      if (key) {  // frame_select.py:119-125: key resets the accumulator
        kind = 0;
        ref = -1;
        a.fsk[stream] = 0;
        a.last_key[stream] = t;
      } else if (sp.policy_keyframe) {
        kind = 2;
        ref = a.last_key[stream];
        a.fsk[stream] = fsk;
      } else {
        kind = 1;
        ref = t - 1;
        a.fsk[stream] = fsk;
      }
      const long long o = (long long)stream * a.dss + t;
      a.kind[o] = kind;
      a.ref[o] = ref;
      a.trigger[o] = trig;
      // reference frame of the NEXT frame's motion search (pipeline.py:102-106)
      if (a.ref_next)
        a.ref_next[stream] = stream * a.frames_per_stream + (sp.policy_keyframe ? a.last_key[stream] : t);
      is_key_s = key;
    }
    __syncthreads();
    if (is_key_s)
      for (int c = threadIdx.x; c < ncoarse; c += blockDim.x) acc[c] = 0.0;
    __syncthreads();
  }
}

// Register-resident AEM scan for the "max" statistic (the common case): each
// thread owns up to kDecideCells coarse cells for the whole clip; the pooled
// energies of frame t+1 are loaded while frame t is reduced, so a frame costs
// one CTA max-reduction and two barriers instead of global round trips.
// Operation order per cell is the reference's: acc' = acc + pooled (float64),
// trigger = max over cells (exact), key resets acc to 0 (frame_select.py:99-136).
constexpr int kDecideThreads = 1024;
constexpr int kDecideCells = 4;

__device__ __forceinline__ double pooled_cell(const double* __restrict__ e, int c, const bmc_select_params& sp) {
  if (sp.factor == 1) return e[c];
  const int cy = c / sp.coarse_w, cx = c - cy * sp.coarse_w;
  double v = -INFINITY;
  for (int dy = 0; dy < sp.factor; ++dy)
    for (int dx = 0; dx < sp.factor; ++dx) v = fmax(v, e[(cy * sp.factor + dy) * sp.grid_w + cx * sp.factor + dx]);
  return v;
}

__global__ void __launch_bounds__(kDecideThreads) decide_max_kernel(const DecideArgs a) {
  __shared__ double red[kDecideThreads / 32];
  __shared__ int is_key_s;
  const int stream = blockIdx.x;
  const bmc_select_params& sp = a.sp;
  const int ncoarse = sp.coarse_h * sp.coarse_w;
  double* accg = a.acc + (long long)stream * ncoarse;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double acc[kDecideCells], nxt[kDecideCells];
#pragma unroll
  for (int k = 0; k < kDecideCells; ++k) {
    const int c = threadIdx.x + k * kDecideThreads;
    acc[k] = c < ncoarse ? accg[c] : 0.0;
    nxt[k] = 0.0;
  }
  auto load_frame = [&](int t, double (&dst)[kDecideCells]) {
    const double* e = a.energy + stream * a.ess + t * a.efs;
#pragma unroll
    for (int k = 0; k < kDecideCells; ++k) {
      const int c = threadIdx.x + k * kDecideThreads;
      dst[k] = c < ncoarse ? pooled_cell(e, c, sp) : 0.0;
    }
  };
  load_frame(a.t_begin, nxt);
  int fsk = a.fsk[stream], last_key = a.last_key[stream];
  for (int t = a.t_begin; t < a.t_end; ++t) {
    double cur[kDecideCells];
#pragma unroll
    for (int k = 0; k < kDecideCells; ++k) cur[k] = nxt[k];
    if (t + 1 < a.t_end) load_frame(t + 1, nxt);  // prefetch: independent of the scan state
    double mx = -INFINITY;
#pragma unroll
    for (int k = 0; k < kDecideCells; ++k) {
      const int c = threadIdx.x + k * kDecideThreads;
      if (c < ncoarse) {
        acc[k] = __dadd_rn(acc[k], cur[k]);
        mx = fmax(mx, acc[k]);
      }
    }
    for (int m = 16; m; m >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, m));
    if (lane == 0) red[warp] = mx;
    __syncthreads();
    if (warp == 0) {
      double r = lane < (int)(blockDim.x >> 5) ? red[lane] : -INFINITY;
      for (int m = 16; m; m >>= 1) r = fmax(r, __shfl_xor_sync(0xffffffffu, r, m));
      if (lane == 0) {
        const int f = fsk + 1;
        const bool key = r > sp.aem_threshold || (sp.has_max_gop && f >= sp.max_gop);
        int kind, ref;
        if (key) {
          kind = 0;
          ref = -1;
          fsk = 0;
          last_key = t;
        } else if (sp.policy_keyframe) {
          kind = 2;
          ref = last_key;
          fsk = f;
        } else {
          kind = 1;
          ref = t - 1;
          fsk = f;
        }
        const long long o = (long long)stream * a.dss + t;
        a.kind[o] = kind;
        a.ref[o] = ref;
        a.trigger[o] = r;
        if (a.ref_next)
          a.ref_next[stream] = stream * a.frames_per_stream + (sp.policy_keyframe ? last_key : t);
        is_key_s = key;
      }
    }
    __syncthreads();
    if (is_key_s) {
#pragma unroll
      for (int k = 0; k < kDecideCells; ++k) acc[k] = 0.0;
    }
    // red[] and is_key_s are rewritten only after the next frame's first barrier
  }
#pragma unroll
  for (int k = 0; k < kDecideCells; ++k) {
    const int c = threadIdx.x + k * kDecideThreads;
    if (c < ncoarse) accg[c] = acc[k];
  }
  if (threadIdx.x == 0) {
    a.fsk[stream] = fsk;
    a.last_key[stream] = last_key;
  }
}

// ---------------------------------------------------------------------------
// AEM scan for large accumulator grids ("max" statistic): the serial
// dependence of the scan is only through the per-frame maximum, and the
// accumulator of every cell after frame t is a function of the last reset
// point alone -- acc_t(r) = (((base + p_{r+1}) + p_{r+2}) + ... + p_t) with
// base = 0 after a key frame r, or the carried-in accumulator when no key
// happened in this call (the reference's own float64 order, frame_select.py:99).
// So the maxima M(r, t) of every possible reset point r are computed in
// parallel (aem_prefix_max_kernel: one CTA per (cell chunk, r, stream), a CTA
// max per frame, one atomicMax per CTA on the ordered bits of non-negative
// doubles), a single thread per stream then walks the frames with
// trigger_t = M(last reset, t) (aem_scan_kernel), and the final accumulator is
// rebuilt from the last reset point (aem_final_acc_kernel).  Identical
// decisions, triggers and state to the per-frame scan.
// ---------------------------------------------------------------------------
constexpr int kAemThreads = 1024;
constexpr int kAemCellsPerThread = 4;

__global__ void __launch_bounds__(kAemThreads) aem_prefix_max_kernel(const DecideArgs a, unsigned long long* M) {
  __shared__ double red[kAemThreads / 32];
  const int stream = blockIdx.z, ri = blockIdx.y;  // ri = 0: carried-in accumulator; ri >= 1: key at t_begin+ri-1
  const bmc_select_params& sp = a.sp;
  const int ncoarse = sp.coarse_h * sp.coarse_w;
  const int nt = a.t_end - a.t_begin;
  const int t0 = ri == 0 ? a.t_begin : a.t_begin + ri;  // first frame accumulated from this reset point
  const double* accg = a.acc + (long long)stream * ncoarse;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int cbase = blockIdx.x * kAemThreads * kAemCellsPerThread + threadIdx.x;
  double acc[kAemCellsPerThread];
#pragma unroll
  for (int k = 0; k < kAemCellsPerThread; ++k) {
    const int c = cbase + k * kAemThreads;
    acc[k] = (ri == 0 && c < ncoarse) ? accg[c] : 0.0;
  }
  unsigned long long* Mrow = M + ((long long)stream * nt + ri) * nt;
  for (int t = t0; t < a.t_end; ++t) {
    const double* e = a.energy + stream * a.ess + t * a.efs;
    double mx = 0.0;  // accumulators are sums of non-negative energies
#pragma unroll
    for (int k = 0; k < kAemCellsPerThread; ++k) {
      const int c = cbase + k * kAemThreads;
      if (c < ncoarse) {
        acc[k] = __dadd_rn(acc[k], pooled_cell(e, c, sp));
        mx = fmax(mx, acc[k]);
      }
    }
    for (int m = 16; m; m >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, m));
    if (lane == 0) red[warp] = mx;
    __syncthreads();
    if (warp == 0) {
      double r = lane < (int)(blockDim.x >> 5) ? red[lane] : 0.0;
      for (int m = 16; m; m >>= 1) r = fmax(r, __shfl_xor_sync(0xffffffffu, r, m));
      if (lane == 0) atomicMax(Mrow + (t - a.t_begin), (unsigned long long)__double_as_longlong(r));
    }
    __syncthreads();
  }
}

__global__ void aem_scan_kernel(const DecideArgs a, const unsigned long long* M, int32_t* reset_out) {
  const int stream = blockIdx.x * blockDim.x + threadIdx.x;
  if (stream >= a.n_streams) return;
  const bmc_select_params& sp = a.sp;
  const int nt = a.t_end - a.t_begin;
  const unsigned long long* Ms = M + (long long)stream * nt * nt;
  int fsk = a.fsk[stream], last_key = a.last_key[stream];
  int ri = 0;  // current reset point (row of M)
  for (int t = a.t_begin; t < a.t_end; ++t) {
    const double r = __longlong_as_double((long long)Ms[(long long)ri * nt + (t - a.t_begin)]);
    const int f = fsk + 1;
    const bool key = r > sp.aem_threshold || (sp.has_max_gop && f >= sp.max_gop);
    int kind, ref;
    if (key) {
      kind = 0;
      ref = -1;
      fsk = 0;
      last_key = t;
      ri = t - a.t_begin + 1;
    } else if (sp.policy_keyframe) {
      kind = 2;
      ref = last_key;
      fsk = f;
    } else {
      kind = 1;
      ref = t - 1;
      fsk = f;
    }
    const long long o = (long long)stream * a.dss + t;
    a.kind[o] = kind;
    a.ref[o] = ref;
    a.trigger[o] = r;
    if (a.ref_next) a.ref_next[stream] = stream * a.frames_per_stream + (sp.policy_keyframe ? last_key : t);
  }
  a.fsk[stream] = fsk;
  a.last_key[stream] = last_key;
  reset_out[stream] = ri;
}

__global__ void aem_final_acc_kernel(const DecideArgs a, const int32_t* reset) {
  const int stream = blockIdx.y;
  const bmc_select_params& sp = a.sp;
  const int ncoarse = sp.coarse_h * sp.coarse_w;
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= ncoarse) return;
  const int ri = reset[stream];
  double* accg = a.acc + (long long)stream * ncoarse;
  double v = ri == 0 ? accg[c] : 0.0;
  for (int t = ri == 0 ? a.t_begin : a.t_begin + ri; t < a.t_end; ++t)
    v = __dadd_rn(v, pooled_cell(a.energy + stream * a.ess + t * a.efs, c, sp));
  accg[c] = v;
}

int launch_decide(const DecideArgs& a, cudaStream_t st) {
  const int ncoarse = a.sp.coarse_h * a.sp.coarse_w;
  const int nt = a.t_end - a.t_begin;
  if (!a.sp.statistic_mean && ncoarse > kDecideThreads * kDecideCells && nt >= 1) {
    // stream-ordered scratch (capturable): M (streams, nt, nt) + the final reset point per stream.
    // The device's default pool keeps its memory mapped between uses (release
    // threshold raised once per device): otherwise every synchronize trims it and
    // the next allocation pays for mapping pages again.
    {
      static std::mutex mu;
      static bool done[64] = {false};
      int dev = 0;
      cudaGetDevice(&dev);
      std::lock_guard<std::mutex> g(mu);
      if (dev >= 0 && dev < 64 && !done[dev]) {
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
          unsigned long long thr = ~0ull;
          cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        }
        done[dev] = true;
      }
    }
    const size_t mbytes = (size_t)a.n_streams * nt * nt * sizeof(unsigned long long);
    void* ws = nullptr;
    int rc = cuda_status(cudaMallocAsync(&ws, mbytes + (size_t)a.n_streams * sizeof(int32_t), st), "AEM scratch");
    if (rc) return rc;
    unsigned long long* M = static_cast<unsigned long long*>(ws);
    int32_t* reset = reinterpret_cast<int32_t*>(static_cast<char*>(ws) + mbytes);
    if ((rc = cuda_status(cudaMemsetAsync(M, 0, mbytes, st), "AEM scratch"))) return rc;
    const int chunks = (ncoarse + kAemThreads * kAemCellsPerThread - 1) / (kAemThreads * kAemCellsPerThread);
    aem_prefix_max_kernel<<<dim3(chunks, nt, a.n_streams), kAemThreads, 0, st>>>(a, M);
    if ((rc = cuda_status(cudaGetLastError(), "aem_prefix_max_kernel"))) return rc;
    aem_scan_kernel<<<(a.n_streams + 63) / 64, 64, 0, st>>>(a, M, reset);
    if ((rc = cuda_status(cudaGetLastError(), "aem_scan_kernel"))) return rc;
    aem_final_acc_kernel<<<dim3((ncoarse + 255) / 256, a.n_streams), 256, 0, st>>>(a, reset);
    if ((rc = cuda_status(cudaGetLastError(), "aem_final_acc_kernel"))) return rc;
    return cuda_status(cudaFreeAsync(ws, st), "AEM scratch");
  }
  if (!a.sp.statistic_mean && ncoarse <= kDecideThreads * kDecideCells) {
    decide_max_kernel<<<a.n_streams, kDecideThreads, 0, st>>>(a);
    return cuda_status(cudaGetLastError(), "decide_max_kernel");
  }
  const long long nleaf = pairwise_leaf_count(ncoarse);
  const size_t smem = (size_t)nleaf * (8 + 8 + 4) + 16;
  if (smem > 200 * 1024) {
    set_error("AEM grid of %d cells is too large for the on-chip mean", ncoarse);
    return BMC_E_ARG;
  }
  cudaError_t e = cudaFuncSetAttribute(decide_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return cuda_status(e, "cudaFuncSetAttribute(decide)");
  DecideArgs a2 = a;
  a2.nleaf = nleaf;
  decide_kernel<<<a.n_streams, kThreads, smem, st>>>(a2);
  return cuda_status(cudaGetLastError(), "decide_kernel");
}

// ---------------------------------------------------------------------------
// Motion compensation (propagate.py:17-55):
//   out[y, x] = ref[clip(y + s*dy), clip(x + s*dx)] with (dx, dy) the MV of the
// final block containing (y, x).  Key frames copy the injected key labels.
// One thread produces 16 consecutive output bytes (one 16-byte store).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads) predict_kernel(const PredictArgs a) {
  const int stream = blockIdx.y;
  const long long o = (long long)stream * a.kss + a.t;
  const int kind = a.kind ? a.kind[o] : 1;
  uint8_t* out = a.labels + stream * a.ss + a.t * a.fs;
  const int groups_per_row = (a.W + 15) / 16;
  const long long total = (long long)a.H * groups_per_row;
  if (kind == 0) {
    const uint8_t* src = a.key_labels + stream * a.ss + a.t * a.fs;
    for (long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x; g < total;
         g += (long long)gridDim.x * blockDim.x) {
      const int y = (int)(g / groups_per_row), x0 = (int)(g % groups_per_row) * 16;
      for (int x = x0; x < min(x0 + 16, a.W); ++x) out[(long long)y * a.W + x] = src[(long long)y * a.W + x];
    }
    return;
  }
  const int r = a.ref ? a.ref[o] : a.ref_fixed;
  const uint8_t* src = a.labels + stream * a.ss + (long long)r * a.fs;
  const int32_t* mv = a.mv + stream * a.mvss + a.t * a.mvfs;
  for (long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x; g < total;
       g += (long long)gridDim.x * blockDim.x) {
    const int y = (int)(g / groups_per_row), x0 = (int)(g % groups_per_row) * 16;
    const int gy = y / a.B;
    uint32_t words[4] = {0, 0, 0, 0};
    int gxc = -1, dx = 0, sy = 0;
    const int n = min(16, a.W - x0);
    for (int e = 0; e < n; ++e) {
      const int x = x0 + e;
      const int gx = x / a.B;
      if (gx != gxc) {
        gxc = gx;
        const int c = gy * a.gw + gx;
        dx = __ldg(mv + 2 * c) * a.scale;
        const int dy = __ldg(mv + 2 * c + 1) * a.scale;
        sy = min(max(y + dy, 0), a.H - 1);
      }
      const int sx = min(max(x + dx, 0), a.W - 1);
      words[e >> 2] |= (uint32_t)src[(long long)sy * a.W + sx] << (8 * (e & 3));
    }
    uint8_t* dst = out + (long long)y * a.W + x0;
    if (n == 16 && ((reinterpret_cast<uintptr_t>(dst) & 15) == 0)) {
      *reinterpret_cast<uint4*>(dst) = make_uint4(words[0], words[1], words[2], words[3]);
    } else {
      for (int e = 0; e < n; ++e) dst[e] = (uint8_t)(words[e >> 2] >> (8 * (e & 3)));
    }
  }
}

int launch_predict(const PredictArgs& a, int n_streams, cudaStream_t st) {
  const long long total = (long long)a.H * ((a.W + 15) / 16);
  long long bx = (total + kThreads - 1) / kThreads;
  if (bx > 148 * 8) bx = 148 * 8;
  if (bx < 1) bx = 1;
  predict_kernel<<<dim3((unsigned)bx, n_streams), kThreads, 0, st>>>(a);
  return cuda_status(cudaGetLastError(), "predict_kernel");
}

// ---------------------------------------------------------------------------
// Whole-clip label chain in ONE cooperative launch: frames are processed in
// order (frame t's reference labels are frame t-1's or the last key's output,
// both earlier), separated by a grid-wide barrier; every CTA strides over the
// (stream, row, 16-byte group) tasks of the frame.  Key frames copy their
// injected labels with 16-byte loads/stores; other frames gather, with a
// 5-word funnel-shift fast path when the 16 pixels share one block and need no
// clamping (propagate.py:39-53 semantics either way).
// ---------------------------------------------------------------------------
__device__ __forceinline__ void grid_barrier(unsigned* ctr, unsigned target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(ctr, 1u);
    while (*((volatile unsigned*)ctr) < target) __nanosleep(20);  // back off: spinning steals issue slots
    __threadfence();
  }
  __syncthreads();
}

// Unrefined prediction of the 16 pixels (row py, columns x0..x0+15, all inside
// final block column gx) of frame t: ref[clip(py + s*dy), clip(x + s*dx)] with
// the MV of block (py / B, gx) (propagate.py:39-53).  Lanes past the frame are 0.
__device__ __forceinline__ uint4 predict16(const PredictArgs& a, const uint8_t* src, const int32_t* mv, int py,
                                           int x0, int gx, bool vec_ok) {
  const int c = (py / a.B) * a.gw + gx;
  const int dx = __ldg(mv + 2 * c) * a.scale, dy = __ldg(mv + 2 * c + 1) * a.scale;
  const int sy = min(max(py + dy, 0), a.H - 1);
  const int sx = x0 + dx;
  const uint8_t* row = src + (long long)sy * a.W;
  if (vec_ok && sx >= 0 && sx + 16 <= a.W && x0 + 16 <= a.W) {
    const uint32_t* r32 = reinterpret_cast<const uint32_t*>(row);
    const int w0 = sx >> 2, sh = (sx & 3) * 8;
    uint32_t v[5];
#pragma unroll
    for (int q = 0; q < 4; ++q) v[q] = __ldcg(r32 + w0 + q);
    v[4] = sh ? __ldcg(r32 + w0 + 4) : 0u;
    return make_uint4(__funnelshift_r(v[0], v[1], sh), __funnelshift_r(v[1], v[2], sh),
                      __funnelshift_r(v[2], v[3], sh), __funnelshift_r(v[3], v[4], sh));
  }
  uint32_t w[4] = {0, 0, 0, 0};
  const int n = min(16, a.W - x0);
  for (int e = 0; e < n; ++e) {
    const int x = min(max(x0 + e + dx, 0), a.W - 1);
    w[e >> 2] |= (uint32_t)__ldcg(row + x) << (8 * (e & 3));
  }
  return make_uint4(w[0], w[1], w[2], w[3]);
}

// Unrefined prediction of one pixel (py, px) of frame t.
__device__ __forceinline__ int predict1(const PredictArgs& a, const uint8_t* src, const int32_t* mv, int py, int px) {
  const int c = (py / a.B) * a.gw + px / a.B;
  const int dx = __ldg(mv + 2 * c) * a.scale, dy = __ldg(mv + 2 * c + 1) * a.scale;
  return __ldcg(src + (long long)min(max(py + dy, 0), a.H - 1) * a.W + min(max(px + dx, 0), a.W - 1));
}

__device__ __forceinline__ int byte_of(const uint4& v, int e) {
  const uint32_t w = e < 8 ? (e < 4 ? v.x : v.y) : (e < 12 ? v.z : v.w);
  return (w >> (8 * (e & 3))) & 0xff;
}

// CaBR's weight-free fallback (cabr.py:257-303 _ring_vote, applied by
// refine_blocks(weights=None), :306-345) for one 16-pixel group of a FLAGGED
// final block (matched == 0) of predicted frame t, fused with the prediction:
// the ring pixels straight across the four block borders are predicted on the
// fly from the reference frame with THEIR blocks' MVs (the reference votes on
// the unrefined prediction of the whole frame), so no scratch frame and no
// second grid barrier are needed.  Candidates inside any flagged block are
// dropped unless all four are; among kept candidates at minimal distance the
// class with most votes wins, ties to the smallest class id.  All integer.
// Requires B % 16 == 0 (CaBR blocks are >= 16 px), so a group lies in one block.
__device__ void chain_vote_group(const PredictArgs& a, const uint8_t* src, const int32_t* mv, const uint8_t* m,
                                 uint8_t* out_row, int y, int x0, bool vec_ok) {
  const int k = a.B;
  const int gy = y / k, gx = x0 / k, y0 = gy * k, xb = gx * k, ly = y - y0;
  const int ty = min(max(y0 - 1, 0), a.H - 1), by = min(max(y0 + k, 0), a.H - 1);
  const int lxp = min(max(xb - 1, 0), a.W - 1), rxp = min(max(xb + k, 0), a.W - 1);
  auto flagged = [&](int py, int px) { return m[(py / k) * a.gw + px / k] == 0; };
  const uint4 top = predict16(a, src, mv, ty, x0, gx, vec_ok);
  const uint4 bot = predict16(a, src, mv, by, x0, gx, vec_ok);
  const int left = predict1(a, src, mv, y, lxp), right = predict1(a, src, mv, y, rxp);
  const bool ft = flagged(ty, x0), fb = flagged(by, x0), fl = flagged(y, lxp), fr = flagged(y, rxp);
  const bool any_clean = !(ft && fb && fl && fr);
  const bool use[4] = {!(any_clean && ft), !(any_clean && fb), !(any_clean && fl), !(any_clean && fr)};
  uint32_t w[4] = {0, 0, 0, 0};
  const int n = min(16, a.W - x0);
  // the 16 pixels are independent: fully unrolled so their vote chains interleave
  const int dT = ly + 1, dB = k - ly;
#pragma unroll
  for (int e = 0; e < 16; ++e) {
    const int lx = x0 + e - xb;
    const int cls[4] = {byte_of(top, e), byte_of(bot, e), left, right};
    const int dist[4] = {dT, dB, lx + 1, k - lx};
    int dmin = 0x7fffffff;
#pragma unroll
    for (int c = 0; c < 4; ++c)
      if (use[c]) dmin = min(dmin, dist[c]);
    // key = (4 - votes) * 256 + class: the smallest key has the most votes, ties to the smallest class
    int best_key = 0x7fffffff;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const bool at = use[c] && dist[c] == dmin;
      int votes = 0;
#pragma unroll
      for (int c2 = 0; c2 < 4; ++c2) votes += (use[c2] && dist[c2] == dmin && cls[c2] == cls[c]) ? 1 : 0;
      const int key = (4 - votes) * 256 + cls[c];
      best_key = at ? min(best_key, key) : best_key;
    }
    w[e >> 2] |= (uint32_t)(best_key & 0xff) << (8 * (e & 3));
  }
  if (vec_ok && n == 16) {
    *reinterpret_cast<uint4*>(out_row + x0) = make_uint4(w[0], w[1], w[2], w[3]);
  } else {
    for (int e = 0; e < n; ++e) out_row[x0 + e] = (uint8_t)(w[e >> 2] >> (8 * (e & 3)));
  }
}

// The same vote for ONE pixel (y, x) of a flagged block: the chain spreads a
// frame's flagged pixels over the whole grid (one pixel per thread) instead of
// giving one thread 16 of them.
__device__ __forceinline__ void chain_vote_pixel(const PredictArgs& a, const uint8_t* src, const int32_t* mv,
                                                 const uint8_t* m, uint8_t* out, int y, int x, int lb) {
  const int k = a.B;  // a power of two here (k == 1 << lb)
  const int y0 = (y >> lb) << lb, xb = (x >> lb) << lb, ly = y - y0, lx = x - xb;
  const int ty = min(max(y0 - 1, 0), a.H - 1), by = min(max(y0 + k, 0), a.H - 1);
  const int lxp = min(max(xb - 1, 0), a.W - 1), rxp = min(max(xb + k, 0), a.W - 1);
  const int ry[4] = {ty, by, y, y}, rx[4] = {x, x, lxp, rxp};
  const int dist[4] = {ly + 1, k - ly, lx + 1, k - lx};
  int cls[4];
  bool fl[4];
#pragma unroll
  for (int c = 0; c < 4; ++c) {  // the four ring pixels' unrefined predictions: independent load chains
    const int cell = (ry[c] >> lb) * a.gw + (rx[c] >> lb);
    const int dx = __ldg(mv + 2 * cell) * a.scale, dy = __ldg(mv + 2 * cell + 1) * a.scale;
    cls[c] = __ldcg(src + (long long)min(max(ry[c] + dy, 0), a.H - 1) * a.W + min(max(rx[c] + dx, 0), a.W - 1));
    fl[c] = m[cell] == 0;
  }
  const bool any_clean = !(fl[0] && fl[1] && fl[2] && fl[3]);
  int dmin = 0x7fffffff;
#pragma unroll
  for (int c = 0; c < 4; ++c)
    if (!(any_clean && fl[c])) dmin = min(dmin, dist[c]);
  int best_key = 0x7fffffff;
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const bool at = !(any_clean && fl[c]) && dist[c] == dmin;
    int votes = 0;
#pragma unroll
    for (int c2 = 0; c2 < 4; ++c2) votes += (!(any_clean && fl[c2]) && dist[c2] == dmin && cls[c2] == cls[c]) ? 1 : 0;
    best_key = at ? min(best_key, (4 - votes) * 256 + cls[c]) : best_key;
  }
  out[(long long)y * a.W + x] = (uint8_t)(best_key & 0xff);
}

// Gather of one 16-pixel group of a non-key frame t of one stream
// (propagate.py:39-53): out[y, x] = ref[clip(y + s*dy), clip(x + s*dx)].
__device__ __forceinline__ void chain_gather_group(const PredictArgs& a, int stream, int t, long long o, int y, int x0,
                                                   bool vec_ok, bool skip_flagged = false) {
  uint8_t* out = a.labels + stream * a.ss + t * a.fs + (long long)y * a.W;
  const int n = min(16, a.W - x0);
  const int r = a.ref ? a.ref[o] : a.ref_fixed;
  const uint8_t* src = a.labels + stream * a.ss + (long long)r * a.fs;
  const int32_t* mv = a.mv + stream * a.mvss + t * a.mvfs;
  if (a.matched) {  // CaBR ring vote on flagged blocks (cells indexed like mv, one byte per cell)
    const uint8_t* m = a.matched + stream * (a.mvss / 2) + t * (a.mvfs / 2);
    if (m[(y / a.B) * a.gw + x0 / a.B] == 0) {
      if (!skip_flagged) chain_vote_group(a, src, mv, m, out, y, x0, vec_ok);
      return;
    }
  }
  const int gy = y / a.B;
  const int gx0 = x0 / a.B, gx1 = (x0 + n - 1) / a.B;
  if (vec_ok && n == 16 && gx0 == gx1) {
    const int c = gy * a.gw + gx0;
    const int dx = __ldg(mv + 2 * c) * a.scale, dy = __ldg(mv + 2 * c + 1) * a.scale;
    const int sy = min(max(y + dy, 0), a.H - 1);
    const int sx = x0 + dx;
    if (sx >= 0 && sx + 16 <= a.W) {
      const uint32_t* row = reinterpret_cast<const uint32_t*>(src + (long long)sy * a.W);
      const int w0 = sx >> 2, sh = (sx & 3) * 8;
      uint32_t v[5];
#pragma unroll
      for (int q = 0; q < 4; ++q) v[q] = __ldcg(row + w0 + q);
      v[4] = sh ? __ldcg(row + w0 + 4) : 0u;
      uint4 o4;
      o4.x = __funnelshift_r(v[0], v[1], sh);
      o4.y = __funnelshift_r(v[1], v[2], sh);
      o4.z = __funnelshift_r(v[2], v[3], sh);
      o4.w = __funnelshift_r(v[3], v[4], sh);
      *reinterpret_cast<uint4*>(out + x0) = o4;
      return;
    }
  }
  uint32_t words[4] = {0, 0, 0, 0};
  int gxc = -1, dx = 0, sy = 0;
  for (int e = 0; e < n; ++e) {
    const int x = x0 + e;
    const int gx = x / a.B;
    if (gx != gxc) {
      gxc = gx;
      const int c = gy * a.gw + gx;
      dx = __ldg(mv + 2 * c) * a.scale;
      const int dy = __ldg(mv + 2 * c + 1) * a.scale;
      sy = min(max(y + dy, 0), a.H - 1);
    }
    const int sx = min(max(x + dx, 0), a.W - 1);
    words[e >> 2] |= (uint32_t)__ldcg(src + (long long)sy * a.W + sx) << (8 * (e & 3));
  }
  if (vec_ok && n == 16) {
    *reinterpret_cast<uint4*>(out + x0) = make_uint4(words[0], words[1], words[2], words[3]);
  } else {
    for (int e = 0; e < n; ++e) out[x0 + e] = (uint8_t)(words[e >> 2] >> (8 * (e & 3)));
  }
}

// The label chain of frames [t_begin, t_end) (pipeline.py:123-132).  Phase 1
// copies every key frame's injected labels at once: the copies are
// independent, so the whole grid streams them with eight 16-byte loads in
// flight per thread.  Phase 2 walks the non-key frames in order with a grid
// barrier only where a frame reads one written earlier in this phase; each
// predicted frame is ONE pass: plain gathers, and on flagged blocks (ring vote
// enabled) the fused predict + vote of chain_vote_group.
constexpr int kChainKindsSmem = 2048;
constexpr int kChainScanCells = 8192;  // cells (all streams) a CTA scans per frame for the flagged list
constexpr int kChainFlagCap = 2048;    // flagged blocks per frame handled per pixel
__global__ void __launch_bounds__(kThreads) predict_chain_kernel(const PredictArgs a, int n_streams, int t_begin,
                                                                 int t_end, unsigned* barrier_ctr) {
  __shared__ int kind_s[kChainKindsSmem];
  __shared__ int flag_list[kChainFlagCap];
  __shared__ int flag_n;
  __shared__ int warp_tot[kThreads / 32];
  const int groups_per_row = (a.W + 15) / 16;
  const long long per_stream = (long long)a.H * groups_per_row;
  const long long total = per_stream * n_streams;
  const int nt = t_end - t_begin;
  const bool vec_ok = (a.W % 16 == 0) && (a.fs % 16 == 0) && (a.ss % 16 == 0) &&
                      ((reinterpret_cast<uintptr_t>(a.labels) & 15) == 0) &&
                      (!a.key_labels || (reinterpret_cast<uintptr_t>(a.key_labels) & 15) == 0);
  const bool ks = a.kind && (long long)n_streams * nt <= kChainKindsSmem;
  if (ks)
    for (int i = threadIdx.x; i < n_streams * nt; i += blockDim.x)
      kind_s[i] = a.kind[(long long)(i / nt) * a.kss + t_begin + i % nt];
  __syncthreads();
  auto kind_of = [&](int stream, int t) -> int {
    if (!a.kind) return 1;
    return ks ? kind_s[stream * nt + (t - t_begin)] : a.kind[(long long)stream * a.kss + t];
  };
  auto frame_has = [&](int t, bool key) {
    for (int st = 0; st < n_streams; ++st)
      if ((kind_of(st, t) == 0) == key) return true;
    return false;
  };
  const long long stride = (long long)gridDim.x * blockDim.x;
  const long long gtid = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  // ---- phase 1: key frames
  bool any_nonkey = false;
  if (a.kind) {
    for (int t = t_begin; t < t_end; ++t) any_nonkey |= frame_has(t, false);
    // one 16-pixel group per thread, its key frames eight at a time: the
    // group's coordinates are computed once and eight loads are in flight
    constexpr int U = 8;
    for (long long g = gtid; g < total; g += stride) {
      const int stream = (int)(g / per_stream);
      const long long gg = g - stream * per_stream;
      const int y = (int)(gg / groups_per_row), x0 = (int)(gg - (long long)y * groups_per_row) * 16;
      const long long base = stream * a.ss + (long long)y * a.W + x0;
      const int n = min(16, a.W - x0);
      for (int t0 = t_begin; t0 < t_end; t0 += U) {
        if (vec_ok) {
          uint4 v[U];
          bool k[U];
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const int t = t0 + u;
            k[u] = t < t_end && kind_of(stream, t) == 0;
            if (k[u]) v[u] = __ldcs(reinterpret_cast<const uint4*>(a.key_labels + base + t * a.fs));
          }
#pragma unroll
          for (int u = 0; u < U; ++u)
            if (k[u]) *reinterpret_cast<uint4*>(a.labels + base + (t0 + u) * a.fs) = v[u];
        } else {
          for (int t = t0; t < min(t0 + U, t_end); ++t)
            if (kind_of(stream, t) == 0)
              for (int e = 0; e < n; ++e) a.labels[base + t * a.fs + e] = a.key_labels[base + t * a.fs + e];
        }
      }
    }
    if (!any_nonkey) return;
  }
  unsigned epoch = 0;
  if (a.kind) grid_barrier(barrier_ctr, ++epoch * gridDim.x);  // key frames visible to the gathers
  // ---- phase 2: non-key frames in order.  A thread's (stream, row, group) tasks
  // are the same for every frame: decode them once (32-bit, no 64-bit divides in
  // the frame loop); threads with more than kTasks tasks decode the rest per frame.
  constexpr int kTasks = 4;
  int ts[kTasks], ty[kTasks], tx[kTasks];
  int ntask = 0;
  const uint32_t gpr = (uint32_t)groups_per_row, pss = (uint32_t)per_stream;
  for (long long g = gtid; g < total && ntask < kTasks; g += stride, ++ntask) {
    const uint32_t gg32 = (uint32_t)g;
    ts[ntask] = (int)(gg32 / pss);
    const uint32_t rem = gg32 - (uint32_t)ts[ntask] * pss;
    ty[ntask] = (int)(rem / gpr);
    tx[ntask] = (int)(rem - (uint32_t)ty[ntask] * gpr) * 16;
  }
  const long long g_rest = gtid + (long long)kTasks * stride;
  // Ring vote per pixel: every CTA lists the frame's flagged blocks (all
  // streams) in shared memory, then the grid takes one flagged pixel per thread
  // -- instead of one thread voting 16 pixels while its warp waits.  Only when
  // the cells of a frame fit the scan budget and the list fits (else per group).
  const int cells = a.gh * a.gw;
  const bool pix_vote = a.matched && (long long)n_streams * cells <= kChainScanCells &&
                        (a.B & (a.B - 1)) == 0 && (long long)kChainFlagCap * a.B * a.B < (1ll << 31);
  bool prev_wrote = false;
  for (int t = t_begin; t < t_end; ++t) {
    const bool work = !a.kind || frame_has(t, false);
    if (!work) continue;
    // frame t reads frames <= t-1: any phase-2 work since the last barrier needs one first
    if (prev_wrote) grid_barrier(barrier_ctr, ++epoch * gridDim.x);
    bool per_pixel = false;
    if (pix_vote) {
      // ordered compaction (identical list in every CTA): thread i owns cells
      // [i*chunk, (i+1)*chunk), exclusive scan of the per-thread counts
      const int ncell = n_streams * cells;
      const int chunk = (ncell + blockDim.x - 1) / blockDim.x;
      const int c0 = threadIdx.x * chunk, c1 = min(ncell, c0 + chunk);
      auto is_flagged = [&](int i) {
        const int st = i / cells, c = i - st * cells;
        return kind_of(st, t) != 0 && a.matched[st * (a.mvss / 2) + t * (a.mvfs / 2) + c] == 0;
      };
      int cnt = 0;
      for (int i = c0; i < c1; ++i) cnt += is_flagged(i);
      const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
      int incl = cnt;
      for (int d = 1; d < 32; d <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, d);
        if (lane >= d) incl += v;
      }
      if (lane == 31) warp_tot[wid] = incl;
      __syncthreads();
      int base = 0;
      for (int w = 0; w < wid; ++w) base += warp_tot[w];
      if (threadIdx.x == blockDim.x - 1) flag_n = base + incl;
      int slot = base + incl - cnt;
      for (int i = c0; i < c1; ++i)
        if (is_flagged(i)) {
          if (slot < kChainFlagCap) flag_list[slot] = i;
          ++slot;
        }
      __syncthreads();
      per_pixel = flag_n <= kChainFlagCap;  // the same in every CTA
    }
#pragma unroll
    for (int q = 0; q < kTasks; ++q) {
      if (q < ntask && kind_of(ts[q], t) != 0)
        chain_gather_group(a, ts[q], t, (long long)ts[q] * a.kss + t, ty[q], tx[q], vec_ok, per_pixel);
    }
    for (long long g = g_rest; g < total; g += stride) {
      const uint32_t gg32 = (uint32_t)g;
      const int stream = (int)(gg32 / pss);
      if (kind_of(stream, t) == 0) continue;
      const uint32_t rem = gg32 - (uint32_t)stream * pss;
      const int y = (int)(rem / gpr), x0 = (int)(rem - (uint32_t)y * gpr) * 16;
      chain_gather_group(a, stream, t, (long long)stream * a.kss + t, y, x0, vec_ok, per_pixel);
    }
    if (per_pixel) {
      const int lb = __ffs(a.B) - 1, lkk = 2 * lb;
      const int npix = flag_n << lkk;  // <= kChainFlagCap * B^2
      for (int q = (int)gtid; q < npix; q += (int)stride) {
        const int id = flag_list[q >> lkk], pix = q & ((1 << lkk) - 1);
        const int st = id / cells, c = id - st * cells;
        const int y = (c / a.gw) * a.B + (pix >> lb), x = (c % a.gw) * a.B + (pix & (a.B - 1));
        if (y >= a.H || x >= a.W) continue;
        const uint8_t* src = a.labels + st * a.ss + (long long)a.ref[(long long)st * a.kss + t] * a.fs;
        chain_vote_pixel(a, src, a.mv + st * a.mvss + t * a.mvfs, a.matched + st * (a.mvss / 2) + t * (a.mvfs / 2),
                         a.labels + st * a.ss + t * a.fs, y, x, lb);
      }
    }
    prev_wrote = true;
  }
}

int launch_predict_chain(const PredictArgs& a, int n_streams, int t_begin, int t_end, unsigned* barrier_ctr,
                         cudaStream_t st) {
  int per_sm = 0, sms = 0;
  {
    // one query per process (thread-safe); one process drives one GPU model
    static std::mutex mu;
    static int c_per_sm = 0, c_sms = 0;
    std::lock_guard<std::mutex> g(mu);
    if (!c_per_sm) {
      cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c_per_sm, predict_chain_kernel, kThreads, 0);
      if (e != cudaSuccess) return cuda_status(e, "cudaOccupancyMaxActiveBlocksPerMultiprocessor(predict)");
      int dev = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&c_sms, cudaDevAttrMultiProcessorCount, dev);
      if (c_per_sm < 1) c_per_sm = 1;
    }
    per_sm = c_per_sm;
    sms = c_sms;
  }
  const long long tasks = (long long)n_streams * a.H * ((a.W + 15) / 16);
  if (tasks >= (1ll << 31)) {
    set_error("label chain of %lld 16-pixel groups exceeds the kernel's 32-bit task index", tasks);
    return BMC_E_ARG;
  }
  long long grid = (tasks + kThreads - 1) / kThreads;
  int use_per_sm = per_sm;
  if (const char* v = knob_env("BMC_CHAIN_PER_SM")) use_per_sm = std::max(1, std::min(per_sm, atoi(v)));
  const long long cap = (long long)use_per_sm * sms;
  if (grid > cap) grid = cap;
  if (grid < 1) grid = 1;
  int rc = cuda_status(cudaMemsetAsync(barrier_ctr, 0, sizeof(unsigned), st), "memset predict barrier");
  if (rc) return rc;
  PredictArgs a2 = a;
  void* args[] = {(void*)&a2, (void*)&n_streams, (void*)&t_begin, (void*)&t_end, (void*)&barrier_ctr};
  cudaError_t e = cudaLaunchCooperativeKernel((const void*)predict_chain_kernel, dim3((unsigned)grid), dim3(kThreads),
                                              args, 0, st);
  return cuda_status(e, "predict_chain_kernel");
}

__global__ void predict_features_kernel(const float* __restrict__ src, float* __restrict__ dst, int C, int H, int W,
                                        const int32_t* __restrict__ mv, int gw, int B, int scale) {
  const long long total = (long long)C * H * W;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int x = (int)(i % W);
    const int y = (int)((i / W) % H);
    const long long c = i / ((long long)H * W);
    const int cell = (y / B) * gw + (x / B);
    const int sy = min(max(y + __ldg(mv + 2 * cell + 1) * scale, 0), H - 1);
    const int sx = min(max(x + __ldg(mv + 2 * cell) * scale, 0), W - 1);
    dst[i] = src[(c * H + sy) * W + sx];
  }
}

int launch_predict_features(const float* src, float* dst, int C, int H, int W, const int32_t* mv, int gw, int B,
                            int scale, cudaStream_t st) {
  const long long total = (long long)C * H * W;
  long long blocks = (total + kThreads - 1) / kThreads;
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (blocks < 1) blocks = 1;
  predict_features_kernel<<<(unsigned)blocks, kThreads, 0, st>>>(src, dst, C, H, W, mv, gw, B, scale);
  return cuda_status(cudaGetLastError(), "predict_features_kernel");
}

// ---------------------------------------------------------------------------
// block_energy on arbitrary float64 arrays (fme.py:218-233).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads) block_energy_kernel(const double* __restrict__ a,
                                                                const double* __restrict__ b, long long n,
                                                                long long nleaf, double lam, double tol,
                                                                double* out) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ double result;
  __shared__ int cnt_s;
  long long* leaf_lo = reinterpret_cast<long long*>(smem_raw);
  double* leaf_val = reinterpret_cast<double*>(leaf_lo + nleaf);
  int* leaf_len = reinterpret_cast<int*>(leaf_val + nleaf) + 1;
  if (threadIdx.x == 0) cnt_s = 0;
  auto diff = [&](long long i) { return fabs(__dsub_rn(a[i], b[i])); };
  const double s = block_pairwise(diff, n, leaf_lo, leaf_len, leaf_val, &result);
  int c = 0;
  for (long long i = threadIdx.x; i < n; i += blockDim.x) c += diff(i) > tol;
  atomicAdd(&cnt_s, c);
  __syncthreads();
  if (threadIdx.x == 0) {
    const double nd = (double)n;
    // (1.0 - lam) * sad_norm + lam * sparsity  (fme.py:231-233)
    *out = __dadd_rn(__dmul_rn(__dsub_rn(1.0, lam), __ddiv_rn(s, nd)), __dmul_rn(lam, __ddiv_rn((double)cnt_s, nd)));
  }
}

int launch_block_energy(const double* a, const double* b, long long n, double lam, double tol, double* out,
                        cudaStream_t st) {
  const long long nleaf = pairwise_leaf_count(n);
  const size_t smem = (size_t)nleaf * 20 + 16;
  if (smem > 200 * 1024) {
    set_error("block of %lld samples is too large for block_energy", n);
    return BMC_E_ARG;
  }
  cudaError_t e = cudaFuncSetAttribute(block_energy_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return cuda_status(e, "cudaFuncSetAttribute(block_energy)");
  block_energy_kernel<<<1, kThreads, smem, st>>>(a, b, n, nleaf, lam, tol, out);
  return cuda_status(cudaGetLastError(), "block_energy_kernel");
}

}  // namespace bmc
