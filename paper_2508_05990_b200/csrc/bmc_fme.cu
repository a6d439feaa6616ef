// Block-matching motion estimation on packed Bayer / luma planes (sm_100a).
//
// Replaces fme.estimate_motion / _search_block / _stage_candidates
// (fme.py:236-392) and search_stage (fme.py:271-291).
//
// One launch per (level, search stage); one CTA per (frame pair, block).  The
// three chained stages of a block (fme.py:306-315) communicate through the
// level's mv/energy arrays; stages with range 0 after a searched stage select
// the same candidate again and are folded into the candidate count on the
// host (no launch).  Per stage:
//
//   staging  one TMA box (cp.async.bulk.tensor.3d) brings the reference window
//            (candidate grid + block halo, all staged planes) into shared
//            memory and a second box the current block; the tensor map's
//            out-of-bounds zero fill covers frame borders (those windows only
//            belong to invalid candidates).  No per-word address math.
//   A        integer screening.  A thread owns TY vertically adjacent
//            candidates of one column (+ one plane): it slides a TY-row
//            register window down the block so every loaded reference word
//            feeds TY packed SAD instructions (VABSDIFF4.U8.ACC for uint8;
//            VIMNMX.U16x2 x2 + IDP.2A for uint16).  Sub-word candidate offsets
//            cost one SHF per loaded word (amortised over TY uses); the current
//            block row is a broadcast LDS.128.  Partial SADs of the planes meet
//            in a shared-memory array.
//   B        exact selection.  E >= (1-lam)*SAD/(s*n) because the sparsity
//            term is >= 0, so only candidates whose integer lower bound does
//            not exceed the exact energy of the min-SAD candidate (+1e-11, far
//            above the ~1e-15 float error) can win.  They are replayed in
//            float64 in numpy's pairwise order (bmc_internal.cuh); the first
//            minimum in canonical dy-major order wins (np.argmin, fme.py:266).
//            A min SAD of 0 has E == 0 exactly and wins outright (lam < 1).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "bmc_internal.cuh"
#include "bmc_launch.cuh"

namespace bmc {

constexpr double kScreenEps = 1e-11;

#ifndef BMC_SEARCH_THREADS
#define BMC_SEARCH_THREADS 128
#endif
#ifndef BMC_SEARCH_MINB
#define BMC_SEARCH_MINB 4
#endif
constexpr int kST = BMC_SEARCH_THREADS;  // threads per search CTA
constexpr int kSW = kST / 32;            // warps per search CTA

// ---------------------------------------------------------------------------
// shared-memory carve-up
// ---------------------------------------------------------------------------
struct SmemLayout {
  double* tab;                 // fl(v/255) for uint8
  unsigned long long* red64;   // [kSW]
  double* best_e;              // [kSW]
  int* best_k;                 // [kSW]
  int* misc;                   // [16]
  double* miscd;               // [4]
  unsigned long long* bar;     // mbarrier
  uint32_t* sad;               // [nmax]
  int* klist;                  // [nmax]
  uint32_t* cur;               // [pg][b][cbw_words]
  uint32_t* win;               // [pg][hwin][bw_words]
};

__device__ __forceinline__ SmemLayout carve(unsigned char* base, const StagePlan& pl) {
  SmemLayout L;
  L.tab = reinterpret_cast<double*>(base);
  unsigned char* p = base + 256 * sizeof(double);
  L.red64 = reinterpret_cast<unsigned long long*>(p);
  p += kSW * 8;
  L.best_e = reinterpret_cast<double*>(p);
  p += kSW * 8;
  L.best_k = reinterpret_cast<int*>(p);
  p += kSW * 4;
  L.misc = reinterpret_cast<int*>(p);
  p += 16 * 4;
  L.miscd = reinterpret_cast<double*>(p);
  p += 4 * 8;
  L.bar = reinterpret_cast<unsigned long long*>(p);
  L.sad = reinterpret_cast<uint32_t*>(base + pl.off_sad);
  L.klist = reinterpret_cast<int*>(base + pl.off_klist);
  L.cur = reinterpret_cast<uint32_t*>(base + pl.off_cur);
  L.win = reinterpret_cast<uint32_t*>(base + pl.off_win);
  return L;
}

// ---------------------------------------------------------------------------
// TMA helpers (inline PTX)
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(unsigned long long* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(unsigned long long* bar, uint32_t phase) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int x, int y, int z,
                                            unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::
          "r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
      : "memory");
}

// ---------------------------------------------------------------------------
// per-CTA context
// ---------------------------------------------------------------------------
template <typename Elem>
struct PairCtx {
  const Elem* cur;  // plane 0 of the current frame (global)
  const Elem* ref;  // plane 0 of the reference frame (global)
  int cur_z, ref_z; // first plane index of each frame in the tensor map's z dimension
  int pitch;
  long long plane_stride;
  int frame_h, frame_w;  // candidate validity bounds
  int P;
  int max_value;
  const double* tab;
  double tol, lam, oml;
};

struct StageGeom {
  int r, s, G, ncg;
  int cx, cy;
  int wx0, wy0;  // window origin in plane coordinates
  int tx0;       // x of the staged box (wx0 rounded down to 16 bytes for TMA)
  int d;         // wx0 - tx0: element offset of the window inside each staged row
};

__device__ __forceinline__ int floor_div(int a, int b) { return (a >= 0) ? a / b : -((-a + b - 1) / b); }

// Fallback staging with plain loads (windows larger than a TMA box).
template <typename Elem>
__device__ void stage_ldg(const SmemLayout& L, const Elem* __restrict__ cur0, const Elem* __restrict__ ref0,
                          int pitch, long long plane_stride, int frame_h, const StageGeom& g, int ox, int oy, int b,
                          int npl, const StagePlan& pl) {
  constexpr int EPW = 4 / sizeof(Elem);
  constexpr int SH = 8 * sizeof(Elem);
  const int bww = pl.bw / EPW;
  const int row_max_w = pitch / EPW - 1;
  const int total = npl * pl.hwin * bww;
  for (int idx = threadIdx.x; idx < total; idx += kST) {
    const int w = idx % bww;
    const int row = (idx / bww) % pl.hwin;
    const int pp = idx / (bww * pl.hwin);
    const int gy = min(max(g.wy0 + row, 0), frame_h - 1);
    const int gx = g.wx0 + w * EPW;
    const int gw0 = floor_div(gx, EPW);
    const int sh = gx - gw0 * EPW;
    const uint32_t* row32 =
        reinterpret_cast<const uint32_t*>(ref0 + (long long)pp * plane_stride + (long long)gy * pitch);
    const uint32_t lo = __ldg(row32 + min(max(gw0, 0), row_max_w));
    const uint32_t v = sh ? __funnelshift_r(lo, __ldg(row32 + min(max(gw0 + 1, 0), row_max_w)), sh * SH) : lo;
    L.win[(pp * pl.wrows + row) * bww + w] = v;
  }
  const int cbw = pl.cbw / EPW, cw = b / EPW;
  const int ctot = npl * b * cw;
  for (int idx = threadIdx.x; idx < ctot; idx += kST) {
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
    L.cur[(pp * b + row) * cbw + w] = v;
  }
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

// One reference row of CW words starting `sh` bits into word src[0].
template <int CW, bool SHIFT>
__device__ __forceinline__ void load_row(uint32_t (&dst)[CW], const uint32_t* src, int sh) {
  if constexpr (SHIFT) {
    uint32_t w[CW + 1];
#pragma unroll
    for (int q = 0; q <= CW; ++q) w[q] = src[q];
#pragma unroll
    for (int q = 0; q < CW; ++q) dst[q] = __funnelshift_r(w[q], w[q + 1], sh);
  } else {
#pragma unroll
    for (int q = 0; q < CW; ++q) dst[q] = src[q];
  }
}

// Phase A: integer SAD of every (candidate column, TY-row group, chunk, staged
// plane) item; partial sums meet in L.sad via shared atomics.
// Phase A: integer SAD.  Work item = (candidate column i, TY-row group gi,
// part) where `part` is one of pl.parts contiguous slices of the (plane,
// chunk) units of the block.  With one part a thread owns its TY candidates
// completely and stores the sums; otherwise partial sums meet via shared
// atomics.  The host picks the part count that best fills the CTA.
template <typename Elem, int CW, int TY, bool SHIFT>
__device__ void sad_items(const SmemLayout& L, const StageGeom& g, int b, int npl, const StagePlan& pl,
                          int coff_w, bool accumulate) {
  constexpr int EPW = 4 / sizeof(Elem);
  const int bww = pl.bw / EPW;
  const int cbw = pl.cbw / EPW;
  const int cpr = (b / EPW) / CW;
  const int units = npl * cpr;
  const int parts = min(pl.parts, units);
  const int per = (units + parts - 1) / parts;
  const int cols = g.G * g.ncg;
  const int items = cols * parts;
  const int s = g.s;
  const int nrho = s < b ? s : b;
  const int rstep = s * bww, cstep = s * cbw;
  // incremental mixed-radix decode of it = (part * ncg + gi) * G + i
  int i = threadIdx.x % g.G, q = threadIdx.x / g.G;
  const int di = kST % g.G, dq = kST / g.G;
  for (int it = threadIdx.x; it < items; it += kST) {
    const int gi = q % g.ncg, part = q / g.ncg;
    const int xo = g.d + i * s;
    const int sh = (xo % EPW) * 8 * (int)sizeof(Elem);
    uint32_t acc[TY];
#pragma unroll
    for (int j = 0; j < TY; ++j) acc[j] = 0;
    const int u_end = min(units, (part + 1) * per);
    for (int u = part * per; u < u_end; ++u) {
      const int pp = u / cpr, c = u - pp * cpr;
      // window rows past hwin (next plane / slack rows) only feed the padding
      // candidates of the last row group, whose sums are discarded.
      const uint32_t* R0 = L.win + pp * pl.wrows * bww + (xo / EPW) + c * CW;
      const uint32_t* C0 = L.cur + pp * b * cbw + coff_w + c * CW;
      for (int rho = 0; rho < nrho; ++rho) {
        const int M = (b - 1 - rho) / s + 1;
        const uint32_t* rp = R0 + (rho + gi * TY * s) * bww;
        const uint32_t* cp = C0 + rho * cbw;
        uint32_t R[TY][CW];
#pragma unroll
        for (int k = 0; k < TY - 1; ++k) load_row<CW, SHIFT>(R[k], rp + k * rstep, sh);
        rp += (TY - 1) * rstep;
        for (int m0 = 0; m0 < M; m0 += TY) {
#pragma unroll
          for (int k = 0; k < TY; ++k) {
            if (m0 + k < M) {
              load_row<CW, SHIFT>(R[(k + TY - 1) % TY], rp, sh);
              rp += rstep;
              uint32_t C[CW];
              load_cur<CW>(C, cp);
              cp += cstep;
#pragma unroll
              for (int j = 0; j < TY; ++j) {
#pragma unroll
                for (int w = 0; w < CW; ++w) acc[j] = sad_word(C[w], R[(k + j) % TY][w], acc[j], Elem());
              }
            }
          }
        }
      }
    }
    if (!accumulate) {
#pragma unroll
      for (int j = 0; j < TY; ++j) {
        const int jj = gi * TY + j;
        if (jj < g.G) L.sad[jj * g.G + i] = acc[j];
      }
    } else {
#pragma unroll
      for (int j = 0; j < TY; ++j) {
        const int jj = gi * TY + j;
        if (jj < g.G) atomicAdd(&L.sad[jj * g.G + i], acc[j]);
      }
    }
    i += di;
    q += dq;
    if (i >= g.G) {
      i -= g.G;
      ++q;
    }
  }
}

struct StageResult {
  int dx, dy;
  double energy;
  int nvalid;
};

__device__ __forceinline__ bool cand_valid_ij(const StageGeom& g, int ox, int oy, int b, int fh, int fw, int i, int j,
                                              int& dx, int& dy) {
  dx = g.cx + (i - g.r) * g.s;
  dy = g.cy + (j - g.r) * g.s;
  const int x = ox + dx, y = oy + dy;
  return x >= 0 && x <= fw - b && y >= 0 && y <= fh - b;
}

// Exact energy of candidate (i, j).  When every plane is resident in shared
// memory (pg == P) the replay reads the staged tiles; otherwise global memory.
template <typename Elem>
__device__ __forceinline__ double exact_cand(const SmemLayout& L, const StagePlan& pl, const StageGeom& g,
                                             const PairCtx<Elem>& pc, int ox, int oy, int b, int coff, int i, int j,
                                             int dx, int dy) {
  if (pl.pg == pc.P) {
    const Elem* cur = reinterpret_cast<const Elem*>(L.cur) + coff;
    const Elem* ref = reinterpret_cast<const Elem*>(L.win) + (long long)(j * g.s) * pl.bw + g.d + i * g.s;
    return exact_energy_generic<Elem>(cur, pl.cbw, (long long)b * pl.cbw, ref, pl.bw, (long long)pl.wrows * pl.bw, b,
                                      pc.P, pc.tab, pc.tol, pc.oml, pc.lam)
        .energy;
  }
  const long long roff = (long long)(oy + dy) * pc.pitch + (ox + dx);
  const long long coffg = (long long)oy * pc.pitch + ox;
  return exact_energy_generic<Elem>(pc.cur + coffg, pc.pitch, pc.plane_stride, pc.ref + roff, pc.pitch,
                                    pc.plane_stride, b, pc.P, pc.tab, pc.tol, pc.oml, pc.lam)
      .energy;
}

// One stage for one block; all threads participate and receive the result.
template <typename Elem, int CW, int TY, bool SHIFT>
__device__ StageResult stage_search(const SmemLayout& L, const PairCtx<Elem>& pc, const StagePlan& pl,
                                    const CUtensorMap* tm_win, const CUtensorMap* tm_cur, uint32_t& phase, int ox,
                                    int oy, int b, int cx, int cy, int r, int s) {
  StageGeom g;
  g.r = r;
  g.s = s;
  g.G = 2 * r + 1;
  g.ncg = (g.G + TY - 1) / TY;
  g.cx = cx;
  g.cy = cy;
  g.wx0 = ox + cx - r * s;
  g.wy0 = oy + cy - r * s;
  // TMA tile loads need the box's inner start coordinate on a 16-byte boundary
  constexpr int A16 = 16 / (int)sizeof(Elem);
  g.tx0 = pl.use_tma ? g.wx0 - (((g.wx0 % A16) + A16) % A16) : g.wx0;
  g.d = g.wx0 - g.tx0;
  const int cx0 = pl.use_tma ? ox - (ox % A16) : ox;  // ox >= 0
  const int coff_w = (ox - cx0) / (4 / (int)sizeof(Elem));
  const int coff_e = ox - cx0;  // element offset of the block inside each staged cur row
  const int N = g.G * g.G;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int n = pc.P * b * b;

  __syncthreads();  // previous users of smem are done; mbarrier init visible
  const bool accumulate = pl.parts > 1 || pl.pg < pc.P;
  if (accumulate)
    for (int k = tid; k < N; k += kST) L.sad[k] = 0;
  for (int p0 = 0; p0 < pc.P; p0 += pl.pg) {
    const int npl = min(pl.pg, pc.P - p0);
    if (p0) __syncthreads();
    if (pl.use_tma) {
      if (tid == 0) {
        mbar_expect_tx(L.bar, (uint32_t)(pl.tma_bytes));  // full boxes, OOB included
        tma_load_3d(L.win, tm_win, g.tx0, g.wy0, pc.ref_z + p0, L.bar);
        tma_load_3d(L.cur, tm_cur, cx0, oy, pc.cur_z + p0, L.bar);
      }
      mbar_wait(L.bar, phase);
      phase ^= 1;
    } else {
      stage_ldg<Elem>(L, pc.cur + (long long)p0 * pc.plane_stride, pc.ref + (long long)p0 * pc.plane_stride, pc.pitch,
                      pc.plane_stride, pc.frame_h, g, ox, oy, b, npl, pl);
    }
    __syncthreads();
    sad_items<Elem, CW, TY, SHIFT>(L, g, b, npl, pl, coff_w, accumulate);
  }
  __syncthreads();

  // pass 1: first minimum SAD among valid candidates (key = sad<<32 | k), valid count
  unsigned long long best = ~0ull;
  int nvalid = 0;
  {
    int i = tid % g.G, j = tid / g.G;
    const int di = kST % g.G, dj = kST / g.G;
    for (int k = tid; k < N; k += kST) {
      int dx, dy;
      if (cand_valid_ij(g, ox, oy, b, pc.frame_h, pc.frame_w, i, j, dx, dy)) {
        ++nvalid;
        const unsigned long long key = ((unsigned long long)L.sad[k] << 32) | (unsigned)k;
        best = key < best ? key : best;
      }
      i += di;
      j += dj;
      if (i >= g.G) {
        i -= g.G;
        ++j;
      }
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
    for (int w = 1; w < kSW; ++w) {
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
  if (sad0 == 0 && pc.oml > 0.0) {
    // S == 0 gives E == 0.0 exactly; any earlier candidate has S > 0 and,
    // with (1-lam) > 0, E > 0.  The first zero-SAD candidate wins.
    cand_valid_ij(g, ox, oy, b, pc.frame_h, pc.frame_w, m0 % g.G, m0 / g.G, res.dx, res.dy);
    res.energy = 0.0;
    return res;
  }
  if (sizeof(Elem) == 1)  // fl(v/255) table for the exact replays (only blocks that reach here pay for it)
    for (int v = tid; v < 256; v += kST) L.tab[v] = __ddiv_rn((double)v, (double)pc.max_value);
  __syncthreads();
  if (warp == 0) {
    double e0 = 0.0;
    if (sad0 != 0) {
      int dx, dy;
      cand_valid_ij(g, ox, oy, b, pc.frame_h, pc.frame_w, m0 % g.G, m0 / g.G, dx, dy);
      e0 = exact_cand<Elem>(L, pl, g, pc, ox, oy, b, coff_e, m0 % g.G, m0 / g.G, dx, dy);
    }
    if (lane == 0) L.miscd[0] = e0;
  }
  __syncthreads();
  const double e0 = L.miscd[0];
  const double bound = e0 + kScreenEps;
  const double unit = (double)pc.max_value * (double)n;
  {
    int i = tid % g.G, j = tid / g.G;
    const int di = kST % g.G, dj = kST / g.G;
    for (int k = tid; k < N; k += kST) {
      int dx, dy;
      if (k != m0 && cand_valid_ij(g, ox, oy, b, pc.frame_h, pc.frame_w, i, j, dx, dy)) {
        const double lb = pc.oml * ((double)L.sad[k] / unit);
        if (lb <= bound) L.klist[atomicAdd(&L.misc[3], 1)] = k;
      }
      i += di;
      j += dj;
      if (i >= g.G) {
        i -= g.G;
        ++j;
      }
    }
  }
  __syncthreads();
  const int nk = L.misc[3];
  double be = (warp == 0) ? e0 : 1e300;
  int bk = (warp == 0) ? m0 : 0x7fffffff;
  for (int e = warp; e < nk; e += kSW) {
    const int k = L.klist[e];
    int dx, dy;
    cand_valid_ij(g, ox, oy, b, pc.frame_h, pc.frame_w, k % g.G, k / g.G, dx, dy);
    const double ek = exact_cand<Elem>(L, pl, g, pc, ox, oy, b, coff_e, k % g.G, k / g.G, dx, dy);
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
    for (int w = 1; w < kSW; ++w) {
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
  cand_valid_ij(g, ox, oy, b, pc.frame_h, pc.frame_w, kw % g.G, kw / g.G, res.dx, res.dy);
  res.energy = L.miscd[1];
  return res;
}

// ---------------------------------------------------------------------------
// the stage kernel
// ---------------------------------------------------------------------------
template <typename Elem, int CW, int TY, bool SHIFT>
__global__ void __launch_bounds__(kST, BMC_SEARCH_MINB)
    fme_stage_kernel(const __grid_constant__ CUtensorMap tm_win, const __grid_constant__ CUtensorMap tm_cur,
                     const StageLaunch a) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const SmemLayout L = carve(smem_raw, a.plan);
  const bmc_fme_params& p = a.prm;
  const int b = a.b;
  int pair = 0, gx = 0, gy = 0, ox, oy, sx = 0, sy = 0;
  long long cell = 0;
  if (a.single) {
    ox = a.ox;
    oy = a.oy;
    sx = a.cx;
    sy = a.cy;
  } else {
    const int blk = blockIdx.x;
    pair = blockIdx.y;
    gx = blk % a.gw;
    gy = blk / a.gw;
    cell = (long long)pair * a.gw * a.gh + blk;
    ox = gx * b;
    oy = gy * b;
    if (a.level > 0) {
      const int pgw = a.gw / 2, pgh = a.gh / 2;
      const long long pcell = (long long)pair * pgw * pgh + (gy / 2) * pgw + (gx / 2);
      if (a.parent_matched[pcell]) {  // inherited: copy the parent (fme.py:352-362)
        if (a.first && threadIdx.x == 0) {
          a.mv[2 * cell] = a.parent_mv[2 * pcell];
          a.mv[2 * cell + 1] = a.parent_mv[2 * pcell + 1];
          a.energy[cell] = a.parent_e[pcell];
          a.matched[cell] = 1;
        }
        return;
      }
      if (a.first) {
        sx = a.parent_mv[2 * pcell];
        sy = a.parent_mv[2 * pcell + 1];
      }
    }
    if (!a.first) {
      sx = a.mv[2 * cell];
      sy = a.mv[2 * cell + 1];
    }
  }
  PairCtx<Elem> pc;
  const int cur_f = a.single ? 0 : a.cur_index[pair];
  const int ref_f = a.single ? 0 : a.ref_index[pair];
  pc.cur = reinterpret_cast<const Elem*>(a.planes) + (long long)cur_f * p.frame_stride;
  pc.ref = reinterpret_cast<const Elem*>(a.ref_planes) + (long long)ref_f * p.frame_stride;
  pc.cur_z = cur_f * p.planes;
  pc.ref_z = ref_f * p.planes;
  pc.pitch = p.pitch;
  pc.plane_stride = p.plane_stride;
  pc.frame_h = a.single ? p.real_h : p.pad_h;  // search_stage works on unpadded planes (fme.py:279-284)
  pc.frame_w = a.single ? p.real_w : p.pad_w;
  pc.P = p.planes;
  pc.max_value = p.max_value;
  pc.tol = p.sparsity_tolerance;
  pc.lam = p.lam;
  pc.oml = p.one_minus_lam;
  pc.tab = sizeof(Elem) == 1 ? L.tab : a.tab16;  // the uint8 table is filled lazily (first exact replay)
  uint32_t phase = 0;
  if (a.plan.use_tma && threadIdx.x == 0) mbar_init(L.bar, 1);
  StageResult res = stage_search<Elem, CW, TY, SHIFT>(L, pc, a.plan, &tm_win, &tm_cur, phase, ox, oy, b, sx, sy, a.r,
                                                      a.s);
  if (res.nvalid == 0)  // fme.py:310-313
    res = stage_search<Elem, CW, TY, SHIFT>(L, pc, a.plan, &tm_win, &tm_cur, phase, ox, oy, b, 0, 0, a.r, a.s);
  if (threadIdx.x != 0) return;
  if (a.single) {
    a.mv[0] = res.dx;
    a.mv[1] = res.dy;
    a.energy[0] = res.energy;
    a.nvalid_out[0] = res.nvalid;
    return;
  }
  a.mv[2 * cell] = res.dx;
  a.mv[2 * cell + 1] = res.dy;
  a.energy[cell] = res.energy;
  if (a.last) {
    bool m;
    if (a.final_level) {
      const bool in_real = oy < p.real_h && ox < p.real_w;  // fme.py:377-384
      m = !(res.energy > p.refine_block_threshold && in_real);
    } else {
      m = res.energy <= p.split_threshold;  // fme.py:386
    }
    a.matched[cell] = m ? 1 : 0;
  }
  atomicAdd(a.evals + pair, (unsigned long long)(res.nvalid + a.extra_evals));
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------

static PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// 3-D view of a plane buffer: x = column, y = row, z = plane index over all frames.
static int encode_map(CUtensorMap* m, const void* base, const bmc_fme_params& p, int n_frames, int box_w, int box_h,
                      int box_z) {
  auto enc = tensor_map_encoder();
  if (!enc) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return BMC_E_CUDA;
  }
  const cuuint64_t dims[3] = {(cuuint64_t)p.pad_w, (cuuint64_t)p.pad_h, (cuuint64_t)p.planes * n_frames};
  const cuuint64_t strides[2] = {(cuuint64_t)p.pitch * p.elem_bytes, (cuuint64_t)p.plane_stride * p.elem_bytes};
  const cuuint32_t box[3] = {(cuuint32_t)box_w, (cuuint32_t)box_h, (cuuint32_t)box_z};
  const cuuint32_t es[3] = {1, 1, 1};
  CUresult r = enc(m, p.elem_bytes == 1 ? CU_TENSOR_MAP_DATA_TYPE_UINT8 : CU_TENSOR_MAP_DATA_TYPE_UINT16, 3,
                   const_cast<void*>(base), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (%d) for box %dx%dx%d", (int)r, box_w, box_h, box_z);
    return BMC_E_CUDA;
  }
  return BMC_OK;
}

static int pick_ty(int G) {
  static const int cap = [] {
    const char* e = getenv("BMC_TY_MAX");
    const int v = e ? atoi(e) : 12;
    return v >= 1 && v <= 12 ? v : 12;
  }();
  const int groups = (G + cap - 1) / cap;
  return (G + groups - 1) / groups;
}

static const int kSmemBudget = 220 * 1024;
static const int kSmemTarget = 110 * 1024;

int plan_stage(StagePlan& pl, const bmc_fme_params& p, int b, int r, int s, bool allow_tma) {
  std::memset(&pl, 0, sizeof pl);
  const int eb = p.elem_bytes, epw = 4 / eb;
  const int G = 2 * r + 1;
  pl.ty = pick_ty(G);
  pl.nmax = G * G;
  const int wwin = 2 * r * s + b;
  const int align = 16 / eb;  // TMA: inner box extent and start coordinate on 16-byte boundaries
  static const bool no_tma = [] {
    const char* e = getenv("BMC_NO_TMA");
    return e && *e && *e != '0';
  }();
  // TMA box: the window widened by up to align-1 leading elements (16-byte aligned start) + 1 word of slack
  const int bw_tma = (wwin + (align - 1) + epw + align - 1) / align * align;
  pl.use_tma = (allow_tma && !no_tma && bw_tma <= 256 && wwin <= 256) ? 1 : 0;
  pl.bw = pl.use_tma ? bw_tma : (wwin + epw + align - 1) / align * align;
  pl.hwin = wwin;
  {
    // parts per (column, row-group): fill the CTA without splitting when the grid is large
    const int cols = G * ((G + pl.ty - 1) / pl.ty);
    const int units_max = p.planes * ((b / epw) / ((b / epw) >= 4 ? 4 : 2));
    int best = 1;
    double best_u = 0.0;
    for (int parts = 1; parts <= units_max; ++parts) {
      const int items = cols * parts;
      const int rounds = (items + kST - 1) / kST;
      const double util = (double)items / (rounds * kST) - 0.02 * (parts > 1);  // atomics cost a little
      if (util > best_u + 1e-9) {
        best_u = util;
        best = parts;
      }
    }
    pl.parts = best;
  }
  // plane stride in smem = hwin rows (the 3-D TMA box is written densely); the
  // padding rows of the last row group run into the next plane (harmless: their
  // sums are discarded) and past the last plane into ty*s slack rows.
  pl.wrows = wwin;
  pl.cbw = pl.use_tma ? (b * eb >= 16 ? b : align) : b;
  pl.shift = pl.use_tma ? 1 : ((G > 1 && s % epw != 0) ? 1 : 0);
  const int head = 256 * 8 + kSW * 20 + 16 * 4 + 4 * 8 + 16;
  pl.off_sad = (head + 127) & ~127;
  pl.off_klist = pl.off_sad + ((pl.nmax * 4 + 127) & ~127);
  pl.off_cur = pl.off_klist + ((pl.nmax * 4 + 127) & ~127);
  pl.pg = 0;
  for (int pg = p.planes; pg >= 1; --pg) {
    const int cur_bytes = pg * b * pl.cbw * eb;
    const int win_bytes = (pg * pl.wrows + pl.ty * s) * pl.bw * eb;
    const int off_win = pl.off_cur + ((cur_bytes + 127) & ~127);
    const int total = off_win + win_bytes;
    if (total <= kSmemTarget || (pg == 1 && total <= kSmemBudget)) {
      pl.pg = pg;
      if (pg < p.planes && pl.parts < 2) pl.parts = 2;  // several staging passes accumulate -> atomics
      pl.cur_bytes = cur_bytes;
      pl.win_bytes = win_bytes;
      pl.off_win = off_win;
      pl.smem = total;
      pl.tma_bytes = cur_bytes + pg * pl.hwin * pl.bw * eb;
      break;
    }
  }
  if (!pl.pg) {
    set_error("search window of block %d with range %d step %d exceeds the %d KB shared-memory budget", b, r, s,
              kSmemBudget / 1024);
    return BMC_E_SMEM;
  }
  return BMC_OK;
}

template <typename K>
static int set_smem(K kern, int bytes) {
  // cudaFuncSetAttribute is cheap but not free (and best kept out of graph
  // capture): remember the largest value set per instantiation.
  static std::mutex mu;
  static const void* keys[512];
  static int vals[512];
  static int n = 0;
  std::lock_guard<std::mutex> g(mu);
  const void* key = reinterpret_cast<const void*>(kern);
  for (int i = 0; i < n; ++i)
    if (keys[i] == key) {
      if (vals[i] >= bytes) return BMC_OK;
      cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
      if (e != cudaSuccess) return cuda_status(e, "cudaFuncSetAttribute");
      vals[i] = bytes;
      return BMC_OK;
    }
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e != cudaSuccess) return cuda_status(e, "cudaFuncSetAttribute");
  if (n < 512) {
    keys[n] = key;
    vals[n] = bytes;
    ++n;
  }
  return BMC_OK;
}

static bool sync_debug() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("BMC_SYNC_DEBUG");
    v = (e && *e && *e != '0') ? 1 : 0;
  }
  return v == 1;
}

template <typename E, int CW, int TY, bool SH>
static int launch_one(const CUtensorMap& tw, const CUtensorMap& tc, const StageLaunch& a, dim3 grid, cudaStream_t st) {
  int rc = set_smem(fme_stage_kernel<E, CW, TY, SH>, a.plan.smem);
  if (rc) return rc;
  fme_stage_kernel<E, CW, TY, SH><<<grid, kST, a.plan.smem, st>>>(tw, tc, a);
  rc = cuda_status(cudaGetLastError(), "fme_stage_kernel");
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  if (!rc && sync_debug() && cudaStreamIsCapturing(st, &cap) == cudaSuccess && cap == cudaStreamCaptureStatusNone) {
    cudaError_t e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) {
      set_error("fme_stage_kernel<eb=%d,CW=%d,TY=%d,shift=%d> level %d b %d r %d s %d tma %d box %dx%dx%d cbw %d "
                "smem %d: %s", (int)sizeof(E), CW, TY, (int)SH, a.level, a.b, a.r, a.s, a.plan.use_tma, a.plan.bw,
                a.plan.hwin, a.plan.pg, a.plan.cbw, a.plan.smem, cudaGetErrorString(e));
      return BMC_E_CUDA;
    }
  }
  return rc;
}

template <typename E, int CW, bool SH>
static int dispatch_ty(const CUtensorMap& tw, const CUtensorMap& tc, const StageLaunch& a, dim3 grid,
                       cudaStream_t st) {
  switch (a.plan.ty) {
    case 1: return launch_one<E, CW, 1, SH>(tw, tc, a, grid, st);
    case 2: return launch_one<E, CW, 2, SH>(tw, tc, a, grid, st);
    case 3: return launch_one<E, CW, 3, SH>(tw, tc, a, grid, st);
    case 4: return launch_one<E, CW, 4, SH>(tw, tc, a, grid, st);
    case 5: return launch_one<E, CW, 5, SH>(tw, tc, a, grid, st);
    case 6: return launch_one<E, CW, 6, SH>(tw, tc, a, grid, st);
    case 7: return launch_one<E, CW, 7, SH>(tw, tc, a, grid, st);
    case 8: return launch_one<E, CW, 8, SH>(tw, tc, a, grid, st);
    case 9: return launch_one<E, CW, 9, SH>(tw, tc, a, grid, st);
    case 10: return launch_one<E, CW, 10, SH>(tw, tc, a, grid, st);
    case 11: return launch_one<E, CW, 11, SH>(tw, tc, a, grid, st);
    default: return launch_one<E, CW, 12, SH>(tw, tc, a, grid, st);
  }
}

// Launch one stage.  The TMA maps view a.ref_planes (n_ref_frames frames) for
// the window and a.planes (n_cur_frames) for the current block.
int launch_fme_stage(const StageLaunch& a, int n_cur_frames, int n_ref_frames, dim3 grid, cudaStream_t st) {
  CUtensorMap tw, tc;
  std::memset(&tw, 0, sizeof tw);
  std::memset(&tc, 0, sizeof tc);
  if (a.plan.use_tma) {
    int rc = encode_map(&tw, a.ref_planes, a.prm, n_ref_frames, a.plan.bw, a.plan.hwin, a.plan.pg);
    if (rc) return rc;
    rc = encode_map(&tc, a.planes, a.prm, n_cur_frames, a.plan.cbw, a.b, a.plan.pg);
    if (rc) return rc;
  }
  const int epw = 4 / a.prm.elem_bytes;
  const bool cw4 = (a.b / epw) >= 4;
  const bool sh = a.plan.shift != 0;
  if (a.prm.elem_bytes == 1) {
    if (cw4)
      return sh ? dispatch_ty<uint8_t, 4, true>(tw, tc, a, grid, st) : dispatch_ty<uint8_t, 4, false>(tw, tc, a, grid, st);
    return sh ? dispatch_ty<uint8_t, 2, true>(tw, tc, a, grid, st) : dispatch_ty<uint8_t, 2, false>(tw, tc, a, grid, st);
  }
  return sh ? dispatch_ty<uint16_t, 4, true>(tw, tc, a, grid, st) : dispatch_ty<uint16_t, 4, false>(tw, tc, a, grid, st);
}

}  // namespace bmc
