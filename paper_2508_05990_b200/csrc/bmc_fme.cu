// Block-matching motion estimation on packed Bayer / luma planes (sm_100a).
//
// Replaces fme.estimate_motion / _search_block / _stage_candidates
// (fme.py:236-392) and search_stage (fme.py:271-291).
//
// One CTA searches one block of one frame pair through the three chained
// stages (fme.py:306-315).  Per stage:
//   A. integer screening: the reference window (candidate grid + block halo) is
//      staged into shared memory once per CTA as EPW/gcd(step,EPW) copies, each
//      pre-shifted by a sub-word element offset, so every candidate row reads
//      aligned 32-bit words (no SHF/PRMT on the hot loop; those share the ALU
//      pipe with VABSDIFF4 and would halve throughput).  A thread owns TY
//      vertically adjacent candidates of one column and slides a TY-row
//      register window down the block, so each loaded ref word feeds TY packed
//      SAD instructions (VABSDIFF4.U8.ACC for uint8, VIMNMX.U16x2+IDP.2A for
//      uint16); the current block row is a broadcast LDS.128.
//   B. exact selection: E >= (1-lam)*SAD/(s*n) because the sparsity term is
//      >= 0, so only candidates whose integer lower bound does not exceed the
//      exact energy of the min-SAD candidate (+1e-11 slack, far above the
//      ~1e-15 float error) can win.  Those are replayed in float64 in numpy's
//      pairwise order (bmc_internal.cuh) and the first minimum in canonical
//      dy-major order wins (np.argmin, fme.py:266).
#include <cstdio>

#include "bmc_internal.cuh"
#include "bmc_launch.cuh"

namespace bmc {

constexpr double kScreenEps = 1e-11;

struct SmemLayout {
  double* tab;
  unsigned long long* red64;
  double* best_e;
  int* best_k;
  int* misc;
  double* miscd;
  uint32_t* sad;
  int* klist;
  uint32_t* cur;
  uint32_t* ref;
};

__device__ __forceinline__ SmemLayout carve(unsigned char* base, const SearchPlan& pl) {
  SmemLayout L;
  L.tab = reinterpret_cast<double*>(base);
  unsigned char* p = base + 256 * sizeof(double);
  L.red64 = reinterpret_cast<unsigned long long*>(p);
  p += kWarps * 8;
  L.best_e = reinterpret_cast<double*>(p);
  p += kWarps * 8;
  L.best_k = reinterpret_cast<int*>(p);
  p += kWarps * 4;
  L.misc = reinterpret_cast<int*>(p);
  p += 16 * 4;
  L.miscd = reinterpret_cast<double*>(p);
  p += 4 * 8;
  p = base + ((p - base + 15) & ~15);
  L.sad = reinterpret_cast<uint32_t*>(p);
  p += ((pl.nmax * 4 + 15) & ~15);
  L.klist = reinterpret_cast<int*>(p);
  p += ((pl.nmax * 4 + 15) & ~15);
  L.cur = reinterpret_cast<uint32_t*>(p);
  p += pl.pg * pl.cur_words * 4;
  L.ref = reinterpret_cast<uint32_t*>(p);
  return L;
}

// Frame geometry + arithmetic constants for one (cur, ref) pair.
template <typename Elem>
struct PairCtx {
  const Elem* cur;  // plane 0 of the current frame
  const Elem* ref;  // plane 0 of the reference frame
  int pitch;
  long long plane_stride;
  int frame_h, frame_w;  // candidate validity bounds (padded plane dims)
  int P;
  int max_value;
  const double* tab;  // fl(v/s) lookup
  double tol, lam, oml;
};

struct StageGeom {
  int r, s, G, ty, ncg;
  int cx, cy;
  int wx0, wy0, wwin, hwin;
  int cstep, ncopies, row_words, cs;
};

template <int EPW>
__device__ __forceinline__ StageGeom make_geom(int ox, int oy, int b, int cx, int cy, int r, int s, int ty) {
  StageGeom g;
  g.r = r;
  g.s = s;
  g.G = 2 * r + 1;
  g.ty = ty;
  g.ncg = (g.G + ty - 1) / ty;
  g.cx = cx;
  g.cy = cy;
  g.wx0 = ox + cx - r * s;
  g.wy0 = oy + cy - r * s;
  g.wwin = 2 * r * s + b;
  g.hwin = g.wwin;
  int gs = s % EPW == 0 ? EPW : (s % 2 == 0 ? 2 : 1);
  if (gs > EPW) gs = EPW;
  g.cstep = gs;
  g.ncopies = (g.G == 1) ? 1 : EPW / gs;
  g.row_words = (g.wwin + EPW - 1) / EPW;
  int cs = g.hwin * g.row_words;
  cs += ((8 - (cs & 31)) + 32) & 31;  // copy blocks start 8 banks apart
  g.cs = cs;
  return g;
}

__device__ __forceinline__ int floor_div(int a, int b) { return (a >= 0) ? a / b : -((-a + b - 1) / b); }

// Stage `npl` planes of the ref window (all alignment copies) and of the
// current block into shared memory.  `cur0`/`ref0` point at the first staged
// plane.  Out-of-frame rows/words are clamped to in-bounds memory: they only
// ever feed candidates that are invalid.  (Plain scalar arguments on purpose:
// an earlier version that took a copied context struct was miscompiled at -O3,
// losing the high word of the 64-bit plane stride.)
template <typename Elem>
__device__ void stage_planes(const SmemLayout& L, const Elem* __restrict__ cur0, const Elem* __restrict__ ref0,
                             int pitch, long long plane_stride, int frame_h, const StageGeom& g, int ox, int oy,
                             int b, int npl, const SearchPlan& pl) {
  constexpr int EPW = 4 / sizeof(Elem);
  constexpr int SH = 8 * sizeof(Elem);
  const int row_max_w = pitch / EPW - 1;
  const int per_copy = g.hwin * g.row_words;
  const int total = npl * g.ncopies * per_copy;
  for (int idx = threadIdx.x; idx < total; idx += kThreads) {
    int t = idx;
    const int w = t % g.row_words;
    t /= g.row_words;
    const int row = t % g.hwin;
    t /= g.hwin;
    const int sl = t % g.ncopies;
    const int pp = t / g.ncopies;
    const int gy = min(max(g.wy0 + row, 0), frame_h - 1);
    const int gx = g.wx0 + w * EPW + sl * g.cstep;
    const int gw0 = floor_div(gx, EPW);
    const int sh = gx - gw0 * EPW;
    const uint32_t* row32 =
        reinterpret_cast<const uint32_t*>(ref0 + (long long)pp * plane_stride + (long long)gy * pitch);
    const int w0 = min(max(gw0, 0), row_max_w);
    const int w1 = min(max(gw0 + 1, 0), row_max_w);
    const uint32_t lo = __ldg(row32 + w0);
    const uint32_t v = sh ? __funnelshift_r(lo, __ldg(row32 + w1), sh * SH) : lo;
    L.ref[pp * pl.ref_words + sl * g.cs + row * g.row_words + w] = v;
  }
  const int cw = b / EPW;
  const int ctot = npl * b * cw;
  for (int idx = threadIdx.x; idx < ctot; idx += kThreads) {
    const int w = idx % cw;
    const int row = (idx / cw) % b;
    const int pp = idx / (cw * b);
    const uint32_t* row32 =
        reinterpret_cast<const uint32_t*>(cur0 + (long long)pp * plane_stride + (long long)(oy + row) * pitch);
    const int gx = ox + w * EPW;
    const int gw0 = gx / EPW;
    const int sh = gx - gw0 * EPW;
    const uint32_t lo = __ldg(row32 + gw0);
    const uint32_t v = sh ? __funnelshift_r(lo, __ldg(row32 + gw0 + 1), sh * SH) : lo;
    L.cur[pp * pl.cur_words + row * cw + w] = v;
  }
}

template <int CW>
__device__ __forceinline__ void load_words(uint32_t (&dst)[CW], const uint32_t* src) {
#pragma unroll
  for (int w = 0; w < CW; ++w) dst[w] = src[w];
}

template <int CW>
__device__ __forceinline__ void load_cur(uint32_t (&dst)[CW], const uint32_t* src) {
  if constexpr (CW == 4) {
    const uint4 v = *reinterpret_cast<const uint4*>(src);
    dst[0] = v.x; dst[1] = v.y; dst[2] = v.z; dst[3] = v.w;
  } else {
    const uint2 v = *reinterpret_cast<const uint2*>(src);
    dst[0] = v.x; dst[1] = v.y;
  }
}

// Phase A: integer SAD of every (candidate, staged plane) into L.sad (atomics
// merge plane groups and column chunks).
template <typename Elem, int CW, int TY>
__device__ void sad_items(const SmemLayout& L, const StageGeom& g, int b, int npl, const SearchPlan& pl) {
  constexpr int EPW = 4 / sizeof(Elem);
  const int curw = b / EPW;
  const int cpr = curw / CW;
  const int items = g.G * g.ncg * cpr * npl;
  const int s = g.s;
  const int nrho = s < b ? s : b;
  for (int it = threadIdx.x; it < items; it += kThreads) {
    int t = it;
    const int i = t % g.G;
    t /= g.G;
    const int gi = t % g.ncg;
    t /= g.ncg;
    const int c = t % cpr;
    const int pp = t / cpr;
    const int xo = i * s;
    const int a = xo % EPW;
    const uint32_t* R0 = L.ref + pp * pl.ref_words + (a / g.cstep) * g.cs + (xo / EPW) + c * CW;
    const uint32_t* C0 = L.cur + pp * pl.cur_words + c * CW;
    uint32_t acc[TY];
#pragma unroll
    for (int j = 0; j < TY; ++j) acc[j] = 0;
    const int hmax = g.hwin - 1;
    for (int rho = 0; rho < nrho; ++rho) {
      const int M = (b - 1 - rho) / s + 1;
      const int base = rho + gi * TY * s;
      uint32_t R[TY][CW];
#pragma unroll
      for (int k = 0; k < TY - 1; ++k) {
        const int row = min(base + k * s, hmax);
        load_words<CW>(R[k], R0 + row * g.row_words);
      }
      for (int m0 = 0; m0 < M; m0 += TY) {
#pragma unroll
        for (int k = 0; k < TY; ++k) {
          const int m = m0 + k;
          if (m < M) {
            const int row = min(base + (m + TY - 1) * s, hmax);
            load_words<CW>(R[(k + TY - 1) % TY], R0 + row * g.row_words);
            uint32_t C[CW];
            load_cur<CW>(C, C0 + (rho + m * s) * curw);
#pragma unroll
            for (int j = 0; j < TY; ++j) {
#pragma unroll
              for (int w = 0; w < CW; ++w) acc[j] = sad_word(C[w], R[(k + j) % TY][w], acc[j], Elem());
            }
          }
        }
      }
    }
#pragma unroll
    for (int j = 0; j < TY; ++j) {
      const int jj = gi * TY + j;
      if (jj < g.G) atomicAdd(&L.sad[jj * g.G + i], acc[j]);
    }
  }
}

template <typename Elem, int CW>
__device__ void sad_dispatch(const SmemLayout& L, const StageGeom& g, int b, int npl, const SearchPlan& pl) {
  switch (g.ty) {
    case 1: sad_items<Elem, CW, 1>(L, g, b, npl, pl); break;
    case 2: sad_items<Elem, CW, 2>(L, g, b, npl, pl); break;
    case 3: sad_items<Elem, CW, 3>(L, g, b, npl, pl); break;
    case 4: sad_items<Elem, CW, 4>(L, g, b, npl, pl); break;
    case 5: sad_items<Elem, CW, 5>(L, g, b, npl, pl); break;
    case 6: sad_items<Elem, CW, 6>(L, g, b, npl, pl); break;
    case 7: sad_items<Elem, CW, 7>(L, g, b, npl, pl); break;
    case 8: sad_items<Elem, CW, 8>(L, g, b, npl, pl); break;
    case 9: sad_items<Elem, CW, 9>(L, g, b, npl, pl); break;
    case 10: sad_items<Elem, CW, 10>(L, g, b, npl, pl); break;
    case 11: sad_items<Elem, CW, 11>(L, g, b, npl, pl); break;
    default: sad_items<Elem, CW, 12>(L, g, b, npl, pl); break;
  }
}

struct StageResult {
  int dx, dy;
  double energy;
  int nvalid;
};

__device__ __forceinline__ bool cand_valid(const StageGeom& g, int ox, int oy, int b, int fh, int fw, int k,
                                           int& dx, int& dy) {
  const int i = k % g.G, j = k / g.G;
  dx = g.cx + (i - g.r) * g.s;
  dy = g.cy + (j - g.r) * g.s;
  const int x = ox + dx, y = oy + dy;
  return x >= 0 && x <= fw - b && y >= 0 && y <= fh - b;
}

// One stage for one block; all threads of the CTA participate and receive the
// result.  nvalid == 0 means every candidate window left the frame.
template <typename Elem, int CW>
__device__ StageResult stage_search(const SmemLayout& L, const PairCtx<Elem>& pc, const SearchPlan& pl, int ox,
                                    int oy, int b, int cx, int cy, int r, int s, int ty) {
  constexpr int EPW = 4 / sizeof(Elem);
  const StageGeom g = make_geom<EPW>(ox, oy, b, cx, cy, r, s, ty);
  const int N = g.G * g.G;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int n = pc.P * b * b;

  __syncthreads();  // previous users of smem are done
  for (int k = tid; k < N; k += kThreads) L.sad[k] = 0;
  for (int p0 = 0; p0 < pc.P; p0 += pl.pg) {
    const int npl = min(pl.pg, pc.P - p0);
    if (p0) __syncthreads();
    stage_planes<Elem>(L, pc.cur + (long long)p0 * pc.plane_stride, pc.ref + (long long)p0 * pc.plane_stride,
                       pc.pitch, pc.plane_stride, pc.frame_h, g, ox, oy, b, npl, pl);
    __syncthreads();
    sad_dispatch<Elem, CW>(L, g, b, npl, pl);
  }
  __syncthreads();

  // first min SAD among valid candidates (key = sad<<32 | k) and valid count
  unsigned long long best = ~0ull;
  int nvalid = 0;
  for (int k = tid; k < N; k += kThreads) {
    int dx, dy;
    if (cand_valid(g, ox, oy, b, pc.frame_h, pc.frame_w, k, dx, dy)) {
      ++nvalid;
      const unsigned long long key = ((unsigned long long)L.sad[k] << 32) | (unsigned)k;
      best = key < best ? key : best;
    }
  }
  for (int m = 16; m; m >>= 1) {
    const unsigned long long o = __shfl_xor_sync(0xffffffffu, best, m);
    best = o < best ? o : best;
    nvalid += __shfl_xor_sync(0xffffffffu, nvalid, m);
  }
  if (lane == 0) {
    L.red64[warp] = best;
    L.best_k[warp] = nvalid;
  }
  __syncthreads();
  if (tid == 0) {
    unsigned long long b0 = L.red64[0];
    int nv = L.best_k[0];
    for (int w = 1; w < kWarps; ++w) {
      b0 = L.red64[w] < b0 ? L.red64[w] : b0;
      nv += L.best_k[w];
    }
    L.misc[0] = (int)(b0 & 0xffffffffu);
    L.misc[1] = nv;
    L.misc[2] = (int)(b0 >> 32);
    L.misc[3] = 0;  // klist size
  }
  __syncthreads();
  StageResult res;
  res.nvalid = L.misc[1];
  if (res.nvalid == 0) {
    res.dx = res.dy = 0;
    res.energy = 0.0;
    return res;
  }
  const int m0 = L.misc[0];
  const unsigned sad0 = (unsigned)L.misc[2];

  // exact energy of the min-SAD candidate (S = 0 => E = 0 exactly).
  if (warp == 0) {
    double e0 = 0.0;
    if (sad0 != 0) {
      int dx, dy;
      cand_valid(g, ox, oy, b, pc.frame_h, pc.frame_w, m0, dx, dy);
      const long long roff = (long long)(oy + dy) * pc.pitch + (ox + dx);
      const long long coff = (long long)oy * pc.pitch + ox;
      e0 = exact_energy_warp<Elem>(pc.cur + coff, pc.ref + roff, pc.pitch, pc.plane_stride, b, pc.P, pc.tab,
                                   pc.tol, pc.oml, pc.lam)
               .energy;
    }
    if (lane == 0) L.miscd[0] = e0;
  }
  __syncthreads();
  const double e0 = L.miscd[0];
  const double bound = e0 + kScreenEps;
  const double unit = (double)pc.max_value * (double)n;
  for (int k = tid; k < N; k += kThreads) {
    int dx, dy;
    if (k != m0 && cand_valid(g, ox, oy, b, pc.frame_h, pc.frame_w, k, dx, dy)) {
      const double lb = pc.oml * ((double)L.sad[k] / unit);
      if (lb <= bound) L.klist[atomicAdd(&L.misc[3], 1)] = k;
    }
  }
  __syncthreads();
  const int nk = L.misc[3];
  double be = (warp == 0) ? e0 : 1e300;
  int bk = (warp == 0) ? m0 : 0x7fffffff;
  for (int e = warp; e < nk; e += kWarps) {
    const int k = L.klist[e];
    int dx, dy;
    cand_valid(g, ox, oy, b, pc.frame_h, pc.frame_w, k, dx, dy);
    const long long roff = (long long)(oy + dy) * pc.pitch + (ox + dx);
    const long long coff = (long long)oy * pc.pitch + ox;
    const double ek = exact_energy_warp<Elem>(pc.cur + coff, pc.ref + roff, pc.pitch, pc.plane_stride, b, pc.P,
                                              pc.tab, pc.tol, pc.oml, pc.lam)
                          .energy;
    if (ek < be || (ek == be && k < bk)) {
      be = ek;
      bk = k;
    }
  }
  if (lane == 0) {
    L.best_e[warp] = be;
    L.best_k[warp] = bk;
  }
  __syncthreads();
  if (tid == 0) {
    double e = L.best_e[0];
    int k = L.best_k[0];
    for (int w = 1; w < kWarps; ++w) {
      if (L.best_e[w] < e || (L.best_e[w] == e && L.best_k[w] < k)) {
        e = L.best_e[w];
        k = L.best_k[w];
      }
    }
    L.misc[4] = k;
    L.miscd[1] = e;
  }
  __syncthreads();
  const int kw = L.misc[4];
  cand_valid(g, ox, oy, b, pc.frame_h, pc.frame_w, kw, res.dx, res.dy);
  res.energy = L.miscd[1];
  return res;
}

template <typename Elem>
__device__ void init_table(const SmemLayout& L, PairCtx<Elem>& pc, const double* gtab) {
  if (sizeof(Elem) == 1) {
    for (int v = threadIdx.x; v < 256; v += kThreads) L.tab[v] = __ddiv_rn((double)v, (double)pc.max_value);
    pc.tab = L.tab;
  } else {
    pc.tab = gtab;
  }
}

template <typename Elem, int CW>
__global__ void __launch_bounds__(kThreads, 2) fme_level_kernel(const LevelArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const SmemLayout L = carve(smem_raw, a.plan);
  const int blk = blockIdx.x;
  const int pair = blockIdx.y;
  const int gx = blk % a.gw, gy = blk / a.gw;
  const long long cell = (long long)pair * a.gw * a.gh + blk;
  const int b = a.b;
  int sx = 0, sy = 0;
  if (a.level > 0) {
    const int pgw = a.gw / 2, pgh = a.gh / 2;
    const long long pcell = (long long)pair * pgw * pgh + (gy / 2) * pgw + (gx / 2);
    sx = a.parent_mv[2 * pcell];
    sy = a.parent_mv[2 * pcell + 1];
    if (a.parent_matched[pcell]) {  // inherited (fme.py:357-362)
      if (threadIdx.x == 0) {
        a.mv[2 * cell] = sx;
        a.mv[2 * cell + 1] = sy;
        a.energy[cell] = a.parent_e[pcell];
        a.matched[cell] = 1;
      }
      return;
    }
  }
  const bmc_fme_params& p = a.prm;
  PairCtx<Elem> pc;
  pc.cur = reinterpret_cast<const Elem*>(a.planes) + (long long)a.cur_index[pair] * p.frame_stride;
  pc.ref = reinterpret_cast<const Elem*>(a.planes) + (long long)a.ref_index[pair] * p.frame_stride;
  pc.pitch = p.pitch;
  pc.plane_stride = p.plane_stride;
  pc.frame_h = p.pad_h;
  pc.frame_w = p.pad_w;
  pc.P = p.planes;
  pc.max_value = p.max_value;
  pc.tol = p.sparsity_tolerance;
  pc.lam = p.lam;
  pc.oml = p.one_minus_lam;
  init_table<Elem>(L, pc, a.tab16);
  const int ox = gx * b, oy = gy * b;
  int mx = sx, my = sy;
  double e = 0.0;
  bool have = false;
  unsigned long long evals = 0;
  for (int st = 0; st < 3; ++st) {
    const int r = p.stage_range[st], s = p.stage_step[st];
    if (r == 0 && have) {  // single candidate == previous winner: same window, same energy
      evals += 1;
      continue;
    }
    StageResult res = stage_search<Elem, CW>(L, pc, a.plan, ox, oy, b, mx, my, r, s, a.plan.ty[st]);
    if (res.nvalid == 0)  // fme.py:310-313
      res = stage_search<Elem, CW>(L, pc, a.plan, ox, oy, b, 0, 0, r, s, a.plan.ty[st]);
    mx = res.dx;
    my = res.dy;
    e = res.energy;
    evals += res.nvalid;
    have = true;
  }
  if (threadIdx.x == 0) {
    a.mv[2 * cell] = mx;
    a.mv[2 * cell + 1] = my;
    a.energy[cell] = e;
    bool m;
    if (a.final_level) {
      const bool in_real = oy < p.real_h && ox < p.real_w;  // fme.py:380-384
      m = !(e > p.refine_block_threshold && in_real);
    } else {
      m = e <= p.split_threshold;  // fme.py:386
    }
    a.matched[cell] = m ? 1 : 0;
    atomicAdd(a.evals + pair, evals);
  }
}

template <typename Elem, int CW>
__global__ void __launch_bounds__(kThreads, 2) stage_kernel(const StageArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const SmemLayout L = carve(smem_raw, a.plan);
  const bmc_fme_params& p = a.prm;
  PairCtx<Elem> pc;
  pc.cur = reinterpret_cast<const Elem*>(a.cur);
  pc.ref = reinterpret_cast<const Elem*>(a.ref);
  pc.pitch = p.pitch;
  pc.plane_stride = p.plane_stride;
  pc.frame_h = p.real_h;  // search_stage works on unpadded planes (fme.py:279-284)
  pc.frame_w = p.real_w;
  pc.P = p.planes;
  pc.max_value = p.max_value;
  pc.tol = p.sparsity_tolerance;
  pc.lam = p.lam;
  pc.oml = p.one_minus_lam;
  init_table<Elem>(L, pc, a.tab16);
  const StageResult res = stage_search<Elem, CW>(L, pc, a.plan, a.ox, a.oy, a.b, a.cx, a.cy, a.r, a.s, a.plan.ty[0]);
  if (threadIdx.x == 0) {
    a.mv[0] = res.dx;
    a.mv[1] = res.dy;
    a.energy[0] = res.energy;
    a.nvalid[0] = res.nvalid;
  }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------

static int pick_ty(int G) {
  const int groups = (G + 11) / 12;
  return (G + groups - 1) / groups;
}

static int geom_ref_words(int epw, int b, int r, int s) {
  const int G = 2 * r + 1;
  int gs = s % epw == 0 ? epw : (s % 2 == 0 ? 2 : 1);
  if (gs > epw) gs = epw;
  const int ncopies = G == 1 ? 1 : epw / gs;
  const int wwin = 2 * r * s + b;
  const int row_words = (wwin + epw - 1) / epw;
  int cs = wwin * row_words;
  cs += ((8 - (cs & 31)) + 32) & 31;
  return ncopies * cs;
}

static const int kSmemBudget = 220 * 1024;
static const int kSmemTarget = 110 * 1024;

// Plan staging for stages (r[i], s[i]) of block size b.
static int make_plan(SearchPlan& pl, const bmc_fme_params& p, int b, const int* rs, const int* ss, int nst) {
  const int epw = 4 / p.elem_bytes;
  pl.nmax = 1;
  int refw = 0;
  for (int i = 0; i < 3; ++i) pl.ty[i] = 1;
  for (int i = 0; i < nst; ++i) {
    const int G = 2 * rs[i] + 1;
    pl.nmax = G * G > pl.nmax ? G * G : pl.nmax;
    pl.ty[i] = pick_ty(G);
    const int w = geom_ref_words(epw, b, rs[i], ss[i]);
    refw = w > refw ? w : refw;
  }
  pl.ref_words = (refw + 3) & ~3;
  pl.cur_words = b * b / epw;
  const int fixed = 256 * 8 + kWarps * 20 + 16 * 4 + 4 * 8 + 16 + 2 * ((pl.nmax * 4 + 15) & ~15);
  pl.pg = 0;
  for (int pg = p.planes; pg >= 1; --pg) {
    const int total = fixed + pg * (pl.cur_words + pl.ref_words) * 4;
    if (total <= kSmemTarget || (pg == 1 && total <= kSmemBudget)) {
      pl.pg = pg;
      pl.smem = total;
      break;
    }
  }
  if (!pl.pg) {
    set_error("search window of block %d with range/step (%d,%d) exceeds the %d KB shared-memory budget", b,
              rs[0], ss[0], kSmemBudget / 1024);
    return BMC_E_SMEM;
  }
  return BMC_OK;
}

int launch_fme_level(const LevelArgs& a, int n_pairs, cudaStream_t st) {
  const int epw = 4 / a.prm.elem_bytes;
  const int cw = (a.b / epw) >= 4 ? 4 : 2;
  dim3 grid(a.gw * a.gh, n_pairs);
  cudaError_t e;
#define BMC_LAUNCH_LEVEL(E, C)                                                                      \
  do {                                                                                              \
    e = cudaFuncSetAttribute(fme_level_kernel<E, C>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                             a.plan.smem);                                                          \
    if (e != cudaSuccess) return cuda_status(e, "cudaFuncSetAttribute(fme_level)");                \
    fme_level_kernel<E, C><<<grid, kThreads, a.plan.smem, st>>>(a);                                 \
  } while (0)
  if (a.prm.elem_bytes == 1) {
    if (cw == 4) BMC_LAUNCH_LEVEL(uint8_t, 4); else BMC_LAUNCH_LEVEL(uint8_t, 2);
  } else {
    BMC_LAUNCH_LEVEL(uint16_t, 4);
  }
#undef BMC_LAUNCH_LEVEL
  return cuda_status(cudaGetLastError(), "fme_level_kernel");
}

int plan_level(SearchPlan& pl, const bmc_fme_params& p, int b) {
  return make_plan(pl, p, b, p.stage_range, p.stage_step, 3);
}

int launch_stage(const StageArgs& a0, cudaStream_t st) {
  StageArgs a = a0;
  const int rs[1] = {a.r}, ss[1] = {a.s};
  int rc = make_plan(a.plan, a.prm, a.b, rs, ss, 1);
  if (rc) return rc;
  const int epw = 4 / a.prm.elem_bytes;
  const int cw = (a.b / epw) >= 4 ? 4 : 2;
  cudaError_t e;
#define BMC_LAUNCH_STAGE(E, C)                                                                              \
  do {                                                                                                      \
    e = cudaFuncSetAttribute(stage_kernel<E, C>, cudaFuncAttributeMaxDynamicSharedMemorySize, a.plan.smem); \
    if (e != cudaSuccess) return cuda_status(e, "cudaFuncSetAttribute(stage)");                            \
    stage_kernel<E, C><<<1, kThreads, a.plan.smem, st>>>(a);                                                \
  } while (0)
  if (a.prm.elem_bytes == 1) {
    if (cw == 4) BMC_LAUNCH_STAGE(uint8_t, 4); else BMC_LAUNCH_STAGE(uint8_t, 2);
  } else {
    BMC_LAUNCH_STAGE(uint16_t, 4);
  }
#undef BMC_LAUNCH_STAGE
  return cuda_status(cudaGetLastError(), "stage_kernel");
}

}  // namespace bmc
