// Block-matching motion estimation on packed Bayer / luma planes (sm_100a):
// device code of the stage kernel (included by the bmc_fme_k_*.cu instantiation units).
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
//            belong to invalid candidates).  TMA boxes must start on a 16-byte
//            boundary, so candidates whose window starts inside a 32-bit word
//            read one of up to three pre-shifted copies of the window, built
//            once per stage (one funnel shift per staged word instead of one
//            per loaded word per candidate row).
//   A        integer screening.  A work item is (candidate column, TY-row
//            group, part) where a part is a slice of the (plane, chunk) units
//            of the block.  The item slides a TY-row register window down the
//            block so every loaded reference word feeds TY packed SAD
//            instructions (VABSDIFF4.U8.ACC for uint8; VIMNMX.U16x2 x2 +
//            IDP.2A for uint16).  The window advances over exactly the block's
//            rows (full TY-periods unrolled, then an unrolled tail with a
//            uniform early exit), so no SAD instruction is issued predicated
//            off.  Each part owns a partial-sum array (no atomics); the CTA size
//            is chosen on the host so the items fill whole warps.
//   B        exact selection.  E >= (1-lam)*SAD/(s*n) because the sparsity
//            term is >= 0, so only candidates whose integer lower bound does
//            not exceed the exact energy of the min-SAD candidate (+1e-11, far
//            above the ~1e-15 float error) can win.  They are replayed in
//            float64 in numpy's pairwise order (bmc_internal.cuh); the first
//            minimum in canonical dy-major order wins (np.argmin, fme.py:266).
//            A min SAD of 0 has E == 0 exactly and wins outright (lam < 1).
#pragma once
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <type_traits>

#include "bmc_internal.cuh"
#include "bmc_launch.cuh"

namespace bmc {

constexpr double kScreenEps = 1e-11;
#ifndef BMC_STAGE_MINB
#define BMC_STAGE_MINB 2  // resident CTAs per SM the register budget is sized for
#endif
constexpr int kMaxSW = ((kMaxStageThreads + 31) / 32 + 1) / 2 * 2;  // warps per search CTA (max, even: keeps the
                                                                 // 8-byte members of the smem head aligned)

// ---------------------------------------------------------------------------
// shared-memory carve-up
// ---------------------------------------------------------------------------
struct SmemLayout {
  double* tab;                 // fl(v/255) for uint8
  unsigned long long* red64;   // [2][kMaxSW] (alternating per block of a kblk set)
  double* best_e;              // [kMaxSW]
  int* best_k;                 // [kMaxSW]
  int* misc;                   // [16]
  double* miscd;               // [4]
  unsigned long long* bar;     // mbarrier
  uint32_t* sad;               // [parts][nmax] partial sums
  int* klist;                  // [nmax]
  int* klist2;                 // [nmax]
  uint32_t* cur;               // [pg][b][cbw_words]
  uint32_t* win;               // [pg][hwin][bw_words] (+ phase copies at copy_words strides)
  int* csum;                   // [32] SEA: current-block plane sums (kb * P + p)
  uint32_t* seaT;              // [8] SEA: smallest exact SAD of the round-1 candidates per block
  int* seaM;                   // [8] SEA: smallest bound per block (-1: no valid candidate)
  int* rect;                   // [32] SEA: valid candidate rectangle per block (ilo, ihi, jlo, jhi)
  int* seaK0;                  // [8] SEA: first candidate (canonical order) with SAD 0 per block
  void* vc;                    // SEA column sums
};

__device__ __forceinline__ SmemLayout carve(unsigned char* base, const StagePlan& pl) {
  SmemLayout L;
  L.tab = reinterpret_cast<double*>(base);
  unsigned char* p = base + 256 * sizeof(double);
  L.red64 = reinterpret_cast<unsigned long long*>(p);
  p += 2 * kMaxSW * 8;
  L.best_e = reinterpret_cast<double*>(p);
  p += kMaxSW * 8;
  L.best_k = reinterpret_cast<int*>(p);
  p += kMaxSW * 4;
  L.misc = reinterpret_cast<int*>(p);
  p += 16 * 4;
  L.miscd = reinterpret_cast<double*>(p);
  p += 4 * 8;
  L.bar = reinterpret_cast<unsigned long long*>(p);
  p += 16;
  L.csum = reinterpret_cast<int*>(p);
  p += 32 * 4;
  L.seaT = reinterpret_cast<uint32_t*>(p);
  p += 8 * 4;
  L.seaM = reinterpret_cast<int*>(p);
  p += 8 * 4;
  L.rect = reinterpret_cast<int*>(p);
  p += 32 * 4;
  L.seaK0 = reinterpret_cast<int*>(p);
  L.vc = base + pl.off_vc;
  L.sad = reinterpret_cast<uint32_t*>(base + pl.off_sad);
  L.klist = reinterpret_cast<int*>(base + pl.off_klist);
  L.klist2 = L.klist + pl.nmax;
  L.cur = reinterpret_cast<uint32_t*>(base + pl.off_cur);
  L.win = reinterpret_cast<uint32_t*>(base + pl.off_win);
  return L;
}

static inline int smem_head_bytes() {
  return 256 * 8 + kMaxSW * 28 + 16 * 4 + 4 * 8 + 16 + 32 * 4 + 8 * 4 + 8 * 4 + 32 * 4 + 8 * 4;
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

// Division by a CTA-uniform divisor without the ~20-instruction integer divide
// (Granlund-Montgomery, exact for every 32-bit numerator): with l = ceil(log2 d)
// and m = floor(2^32 (2^l - d) / d) + 1,  q = (t + ((n - t) >> 1)) >> (l - 1)
// where t = umulhi(n, m).  Magics of the uniform divisors are computed on the
// host (fastdiv_magic); the device constructor is for rare per-block divisors.
__host__ __device__ inline unsigned long long fastdiv_magic(uint32_t d) {
  if (d <= 1) return 0ull;
  uint32_t l = 0;
  while ((1ull << l) < d) ++l;
  const unsigned long long m = (((1ull << l) - d) << 32) / d + 1ull;
  return (m & 0xffffffffull) | ((unsigned long long)l << 32);
}

struct FastDiv {
  uint32_t d, m, l;
  __device__ __forceinline__ FastDiv(uint32_t d_, unsigned long long mg) : d(d_), m((uint32_t)mg),
                                                                             l((uint32_t)(mg >> 32)) {}
  __device__ __forceinline__ explicit FastDiv(uint32_t d_) : FastDiv(d_, fastdiv_magic(d_)) {}
  __device__ __forceinline__ uint32_t div(uint32_t n) const {
    if (d <= 1) return n;
    const uint32_t t = __umulhi(n, m);
    return (t + ((n - t) >> 1)) >> (l - 1);
  }
  __device__ __forceinline__ void divmod(uint32_t n, uint32_t& q, uint32_t& r) const {
    q = div(n);
    r = n - q * d;
  }
};

// Fallback staging with plain loads (windows larger than a TMA box, or the
// single-block search_stage API with arbitrary origins).  Rows are stored
// unshifted relative to the window start (d == 0).
template <typename Elem>
__device__ void stage_ldg(const SmemLayout& L, const Elem* __restrict__ cur0, const Elem* __restrict__ ref0,
                          int pitch, long long plane_stride, int frame_h, const StageGeom& g, int ox, int oy, int b,
                          int npl, const StagePlan& pl) {
  constexpr int EPW = 4 / sizeof(Elem);
  constexpr int SH = 8 * sizeof(Elem);
  const int nt = blockDim.x;
  const int bww = pl.bw / EPW;
  const int row_max_w = pitch / EPW - 1;
  const int total = npl * pl.hwin * bww;
  for (int idx = threadIdx.x; idx < total; idx += nt) {
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
  for (int idx = threadIdx.x; idx < ctot; idx += nt) {
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

// Pre-shifted copies: copy f (1 <= f < EPW) holds every staged row advanced by
// f elements, so a candidate whose window starts at element x reads copy
// x % EPW at word x / EPW with plain aligned loads.  A thread turns one 16-byte
// quad of a staged row (+ the next word) into the same quad of every needed
// copy: 2 loads, one funnel shift per output word, one 16-byte store per copy.
// The last word of a row takes its high bytes from the next row; that word is
// slack (bw carries one spare word) and is never read by a candidate.
template <typename Elem>
__device__ void build_phase_copies(const SmemLayout& L, const StagePlan& pl, int npl, unsigned phase_mask) {
  constexpr int EPW = 4 / sizeof(Elem);
  constexpr int SH = 8 * sizeof(Elem);
  const int quads = npl * pl.wrows * (pl.bw / EPW) / 4;
  const int nt = blockDim.x;
  const int region1 = pl.copies == 2;  // single-phase stages keep their one copy in region 1
  for (int qd = threadIdx.x; qd < quads; qd += nt) {
    const uint4 v = reinterpret_cast<const uint4*>(L.win)[qd];
    const uint32_t nx = L.win[4 * qd + 4];
#pragma unroll
    for (int f = 1; f < EPW; ++f) {
      if (!(phase_mask & (1u << f))) continue;
      uint4 o;
      o.x = __funnelshift_r(v.x, v.y, f * SH);
      o.y = __funnelshift_r(v.y, v.z, f * SH);
      o.z = __funnelshift_r(v.z, v.w, f * SH);
      o.w = __funnelshift_r(v.w, nx, f * SH);
      reinterpret_cast<uint4*>(L.win + (region1 ? 1 : f) * pl.copy_words)[qd] = o;
    }
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

// One reference row of CW words; with SHIFT the row starts `sh` bits into src[0].
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

// One step of the sliding window: block row m (ring slot of its new reference
// row is (k + TY - 1) % TY), candidate j of the group pairs cur row m with
// reference row m + j (slot (k + j) % TY).  K is the step's position in the
// TY-period, so every ring index is a compile-time constant.
template <typename Elem, int CW, int TY, bool SHIFT, int K>
__device__ __forceinline__ void sad_step(uint32_t (&R)[TY][CW], uint32_t (&acc)[TY], const uint32_t*& rp,
                                         const uint32_t*& cp, int rstep, int cstep, int sh) {
  load_row<CW, SHIFT>(R[(K + TY - 1) % TY], rp, sh);
  rp += rstep;
  uint32_t C[CW];
  load_cur<CW>(C, cp);
  cp += cstep;
#pragma unroll
  for (int j = 0; j < TY; ++j) {
#pragma unroll
    for (int w = 0; w < CW; ++w) acc[j] = sad_word(C[w], R[(K + j) % TY][w], acc[j], Elem());
  }
}

template <typename Elem, int CW, int TY, bool SHIFT, int K = 0>
__device__ __forceinline__ void sad_period(uint32_t (&R)[TY][CW], uint32_t (&acc)[TY], const uint32_t*& rp,
                                           const uint32_t*& cp, int rstep, int cstep, int sh) {
  sad_step<Elem, CW, TY, SHIFT, K>(R, acc, rp, cp, rstep, cstep, sh);
  if constexpr (K + 1 < TY) sad_period<Elem, CW, TY, SHIFT, K + 1>(R, acc, rp, cp, rstep, cstep, sh);
}

// Tail of fewer than TY steps: uniform early exit between steps (a branch, not
// predication, so skipped steps issue nothing).
template <typename Elem, int CW, int TY, bool SHIFT, int K = 0>
__device__ __forceinline__ void sad_tail(uint32_t (&R)[TY][CW], uint32_t (&acc)[TY], const uint32_t*& rp,
                                         const uint32_t*& cp, int rstep, int cstep, int sh, int rem) {
  if constexpr (K + 1 < TY) {
    if (K >= rem) return;
    sad_step<Elem, CW, TY, SHIFT, K>(R, acc, rp, cp, rstep, cstep, sh);
    sad_tail<Elem, CW, TY, SHIFT, K + 1>(R, acc, rp, cp, rstep, cstep, sh, rem);
  }
}

// SAD of the TY candidates (rows gi*TY .. gi*TY+TY-1 of one column) over one
// residue class of block rows (M rows, stride s).
template <typename Elem, int CW, int TY, bool SHIFT>
__device__ __forceinline__ void sad_run(const uint32_t* rp, const uint32_t* cp, int rstep, int cstep, int M, int sh,
                                        uint32_t (&acc)[TY]) {
  uint32_t R[TY][CW];
#pragma unroll
  for (int k = 0; k < TY - 1; ++k) load_row<CW, SHIFT>(R[k], rp + k * rstep, sh);
  rp += (TY - 1) * rstep;
  int m0 = 0;
  for (; m0 + TY <= M; m0 += TY) sad_period<Elem, CW, TY, SHIFT>(R, acc, rp, cp, rstep, cstep, sh);
  if (m0 < M) sad_tail<Elem, CW, TY, SHIFT>(R, acc, rp, cp, rstep, cstep, sh, M - m0);
}

// Phase A: integer SAD of every (candidate column i, TY-row group gi, part)
// item.  A part is a contiguous slice of the (plane, chunk, row residue) units; it owns the
// partial-sum array L.sad[part][*].  `add` accumulates onto an earlier staging
// pass (the item -> thread mapping is identical in every pass).
template <typename Elem, int CW, int TY, bool SHIFT>
__device__ void sad_items(const SmemLayout& L, const StageGeom& g, int b, int npl, const StagePlan& pl, int coff_w,
                          bool add, int nblk, int tid0 = -1, int nthr = 0) {
  constexpr int EPW = 4 / sizeof(Elem);
  const int nt = nthr > 0 ? nthr : (int)blockDim.x;  // the threads taking part (a warp group in the WS kernel)
  const int t0 = tid0 >= 0 ? tid0 : (int)threadIdx.x;
  const int bww = pl.bw / EPW;
  const int cbw = pl.cbw / EPW;
  const int cpr = (b / EPW) / CW;
  const int s = g.s;
  const int nrho = s < b ? s : b;  // residue classes of block rows (independent sliding windows)
  const int units = npl * cpr * nrho;
  const int parts = pl.parts;
  const int per = pl.per > 0 ? pl.per : (units + parts - 1) / parts;
  const int cols = g.G * g.ncg;
  const int items = cols * parts * nblk;  // nblk horizontally adjacent blocks share the staged window
  const int rstep = s * bww, cstep = s * cbw;
  const int N = g.G * g.G;
  // uniform divisors with host-precomputed magics (no integer divide per block)
  const FastDiv fG(g.G, pl.mG), fncg(g.ncg, pl.mncg), frho(nrho, pl.mrho), fcpr(cpr, pl.mcpr), fs(s, pl.ms),
      fparts(parts, pl.mparts);
  // Items that would only partly fill the last warp are split into one-unit
  // sub-items (partial sums combined with shared atomics into a pre-zeroed
  // array), so that warp issues a fraction of a full item's SAD instructions.
  const int full32 = (items / 32) * 32;
  // only when the sub-items still fit in the warps the plan launches for the items
  const bool split = pl.split && !add && full32 + (items - full32) * per <= (items + 31) / 32 * 32;
  const int n_full = split ? full32 : items;
  const int n_virt = n_full + (items - n_full) * per;
  const FastDiv fper(per, pl.mper);
  const bool unit_is_plane = (s == 1 && cpr == 1);  // full-search stages: one unit per plane, all b rows
  for (int vt = t0; vt < n_virt; vt += nt) {
    int it = vt, sub = -1;
    if (vt >= n_full) {
      uint32_t qq, rr;
      fper.divmod(vt - n_full, qq, rr);
      it = n_full + (int)qq;
      sub = (int)rr;
    }
    uint32_t q, i, gi, part, kb;
    fG.divmod(it, q, i);
    fncg.divmod(q, part, gi);
    fparts.divmod(part, kb, part);
    const int xo = g.d + kb * b + i * s;
    const int ph = xo % EPW;
    const uint32_t* win = (SHIFT || ph == 0) ? L.win : L.win + (pl.copies == 2 ? 1 : ph) * pl.copy_words;
    const int sh = ph * 8 * (int)sizeof(Elem);
    uint32_t acc[TY];
#pragma unroll
    for (int j = 0; j < TY; ++j) acc[j] = 0;
    int u_beg = part * per, u_end = min(units, (part + 1) * per);
    if (sub >= 0) {
      u_beg += sub;
      u_end = min(u_end, u_beg + 1);
    }
    for (int u = u_beg; u < u_end; ++u) {
      uint32_t rho = 0, pc, pp = (uint32_t)u, c = 0;
      if (!unit_is_plane) {
        frho.divmod(u, pc, rho);
        fcpr.divmod(pc, pp, c);
      }
      // window rows past hwin (next plane / slack rows) only feed the padding
      // candidates of the last row group, whose sums are discarded.
      const uint32_t* R0 = win + pp * pl.wrows * bww + (xo / EPW) + c * CW;
      const uint32_t* C0 = L.cur + pp * b * cbw + coff_w + kb * (b / EPW) + c * CW;
      const int M = unit_is_plane ? b : (int)fs.div(b - 1 - rho) + 1;
      sad_run<Elem, CW, TY, SHIFT>(R0 + (rho + gi * TY * s) * bww, C0 + rho * cbw, rstep, cstep, M, sh, acc);
    }
    uint32_t* dst = L.sad + (kb * parts + part) * N;
#pragma unroll
    for (int j = 0; j < TY; ++j) {
      const int jj = gi * TY + j;
      if (jj < g.G) {
        const int k = jj * g.G + i;
        if (sub >= 0) {
          if (u_beg < u_end) atomicAdd(dst + k, acc[j]);
        } else {
          dst[k] = add ? dst[k] + acc[j] : acc[j];
        }
      }
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

// Partial exact replay of candidate (i, j) over chain groups [q0, q1) (see
// exact_partial): lets the CTA split one large replay across warps.
template <typename Elem>
__device__ __forceinline__ void exact_cand_partial(const SmemLayout& L, const StagePlan& pl, const StageGeom& g,
                                                   const PairCtx<Elem>& pc, int ox, int oy, int b, int coff, int i,
                                                   int j, int dx, int dy, int q0, int q1, double& total, int& cnt) {
  if (pl.pg == pc.P) {
    const Elem* cur = reinterpret_cast<const Elem*>(L.cur) + coff;
    const Elem* ref = reinterpret_cast<const Elem*>(L.win) + (long long)(j * g.s) * pl.bw + g.d + i * g.s;
    exact_partial<Elem>(cur, pl.cbw, (long long)b * pl.cbw, ref, pl.bw, (long long)pl.wrows * pl.bw, b, pc.P, pc.tab,
                        pc.tol, q0, q1, total, cnt);
    return;
  }
  const long long roff = (long long)(oy + dy) * pc.pitch + (ox + dx);
  const long long coffg = (long long)oy * pc.pitch + ox;
  exact_partial<Elem>(pc.cur + coffg, pc.pitch, pc.plane_stride, pc.ref + roff, pc.pitch, pc.plane_stride, b, pc.P,
                      pc.tab, pc.tol, q0, q1, total, cnt);
}

// Integer lower bound of the sparsity count of candidate (i, j): #(|r-c| >= D),
// warp-cooperative over packed 32-bit words (staged tiles, or global planes
// when not every plane is staged).  uint8: one VABSDIFF4 (per-byte |r-c|) and
// two VABSDIFF4.ACC against D-1 and D, using [d >= D] = (|d-(D-1)| - |d-D| + 1)/2
// for integers.  uint16: per-lane |r-c| = max - min (VIMNMX.U16x2), then the
// lane's bit 15 is set iff d >= D (7-bit-carry-free add), counted with POPC.
template <typename Elem>
__device__ __forceinline__ uint32_t ldw_shifted(const uint32_t* base, int elem) {
  constexpr int EPW = 4 / sizeof(Elem);
  const int w = elem / EPW, sh = elem % EPW;  // elem >= 0
  const uint32_t lo = base[w];
  return sh ? __funnelshift_r(lo, base[w + 1], sh * 8 * (int)sizeof(Elem)) : lo;
}

template <typename Elem>
__device__ int count_lo(const SmemLayout& L, const StagePlan& pl, const StageGeom& g, const PairCtx<Elem>& pc,
                        int ox, int oy, int b, int coff, int i, int j, int D) {
  constexpr int EPW = 4 / sizeof(Elem);
  const int lane = threadIdx.x & 31;
  const int n = pc.P * b * b;
  if (D > pc.max_value) return 0;
  const int wpr = b / EPW;                     // words per block row (2..16)
  const int rows_per_iter = 32 / wpr;          // block rows covered by one warp step
  const int wc = lane % wpr, r0 = lane / wpr;  // fixed word column of this lane
  const bool staged = pl.pg == pc.P;
  const int dx = g.cx + (i - g.r) * g.s, dy = g.cy + (j - g.r) * g.s;
  uint32_t k1, k2;
  if constexpr (EPW == 4) {
    k1 = 0x01010101u * (uint32_t)(D - 1);
    k2 = 0x01010101u * (uint32_t)D;
  } else {
    k1 = D <= 32768 ? 0x00010001u * (uint32_t)(0x8000 - D) : 0x00010001u * (uint32_t)(0x10000 - D);
    k2 = 0;
  }
  uint32_t a1 = 0, a2 = 0;
  int cnt = 0;
  auto count_word = [&](uint32_t cw, uint32_t rw) {
    if constexpr (EPW == 4) {
      const uint32_t d4 = __vabsdiffu4(cw, rw);
      asm("vabsdiff4.u32.u32.u32.add %0, %1, %2, %0;" : "+r"(a1) : "r"(d4), "r"(k1));
      asm("vabsdiff4.u32.u32.u32.add %0, %1, %2, %0;" : "+r"(a2) : "r"(d4), "r"(k2));
    } else {
      uint32_t mx, mn;
      asm("max.u16x2 %0, %1, %2;" : "=r"(mx) : "r"(cw), "r"(rw));
      asm("min.u16x2 %0, %1, %2;" : "=r"(mn) : "r"(cw), "r"(rw));
      const uint32_t d2 = mx - mn;
      const uint32_t f = D <= 32768 ? (((d2 & 0x7fff7fffu) + k1) | d2) : (((d2 & 0x7fff7fffu) + k1) & d2);
      cnt += __popc(f & 0x80008000u);
    }
  };
  if (staged) {
    // the candidate's window starts at element (g.d + i*s) of each staged row: one shift for all its words
    const int xoff = g.d + i * g.s;
    const int sh = (xoff % EPW) * 8 * (int)sizeof(Elem);
    const int cbw = pl.cbw / EPW, bww = pl.bw / EPW;
    for (int p = 0; p < pc.P; ++p) {
      const uint32_t* crow = L.cur + (p * b + r0) * cbw + coff / EPW + wc;
      const uint32_t* rrow = L.win + (p * pl.wrows + j * g.s + r0) * bww + xoff / EPW + wc;
      for (int y = r0; y < b; y += rows_per_iter) {
        const uint32_t lo = rrow[0];
        count_word(crow[0], sh ? __funnelshift_r(lo, rrow[1], sh) : lo);
        crow += rows_per_iter * cbw;
        rrow += rows_per_iter * bww;
      }
    }
  } else {
    const int xr = ox + dx;  // >= 0 for a valid candidate
    const int sh = (xr % EPW) * 8 * (int)sizeof(Elem);
    for (int p = 0; p < pc.P; ++p) {
      for (int y = r0; y < b; y += rows_per_iter) {
        const uint32_t* crow = reinterpret_cast<const uint32_t*>(pc.cur + p * pc.plane_stride +
                                                                 (long long)(oy + y) * pc.pitch) + ox / EPW + wc;
        const uint32_t* rrow = reinterpret_cast<const uint32_t*>(pc.ref + p * pc.plane_stride +
                                                                 (long long)(oy + dy + y) * pc.pitch) + xr / EPW + wc;
        const uint32_t lo = rrow[0];
        count_word(crow[0], sh ? __funnelshift_r(lo, rrow[1], sh) : lo);
      }
    }
  }
  if constexpr (EPW == 4) cnt = (int)a1 - (int)a2;
  for (int m = 16; m; m >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, m);
  return EPW == 4 ? (cnt + n) / 2 : cnt;
}

// ---------------------------------------------------------------------------
// Successive elimination (SEA) screening.  The sum-difference bound
//   LB(c) = sum_p | sum(cur_p) - sum(ref_p(c)) |  <=  SAD(c)
// (triangle inequality per CFA plane) costs two box sums per candidate instead
// of P*b*b absolute differences.  T = exact SAD of the candidate with the
// smallest LB is >= the minimum SAD, so every candidate that can be the
// (first) minimum, or tie it, has LB <= T: those get their exact SAD, all others
// keep LB (> T) in the sum array.  select_block is unchanged and stays exact:
// its first minimum is over exact values only (the rest exceed T), and every
// later test (SAD threshold, free sparsity bound, count_lo) only needs a LOWER
// bound of S, which LB is.  When too many candidates survive (content with no
// close match) the stage falls back to the dense screening.
// ---------------------------------------------------------------------------
template <typename Elem>
__device__ __forceinline__ uint32_t word_sum(uint32_t v) {
  if constexpr (sizeof(Elem) == 1) return __dp4a(v, 0x01010101u, 0u);
  else return (v & 0xffffu) + (v >> 16);
}

// Exact SAD of the candidate whose window starts at element xo of staged row yo
// (all P planes staged), warp-cooperative; every lane returns the sum.
template <typename Elem>
__device__ uint32_t warp_sad(const SmemLayout& L, const StagePlan& pl, int P, int b, int cur_w0, int xo, int yo) {
  constexpr int EPW = 4 / sizeof(Elem);
  const int lane = threadIdx.x & 31;
  const int lwpr = __ffs(b / EPW) - 1, lb = __ffs(b) - 1;  // b and b/EPW are powers of two
  const int total = P << (lb + lwpr);
  const int bww = pl.bw / EPW, cbw = pl.cbw / EPW;
  const int sh = (xo % EPW) * 8 * (int)sizeof(Elem), w0 = xo / EPW;
  uint32_t acc = 0;
  for (int idx = lane; idx < total; idx += 32) {
    const int w = idx & ((1 << lwpr) - 1), py = idx >> lwpr;  // py = p * b + y
    const int p = py >> lb, y = py & (b - 1);
    const uint32_t* rr = L.win + (p * pl.wrows + yo + y) * bww + w0 + w;
    const uint32_t lo = rr[0];
    const uint32_t rw = sh ? __funnelshift_r(lo, rr[1], sh) : lo;
    acc = sad_word(L.cur[py * cbw + cur_w0 + w], rw, acc, Elem());
  }
  for (int m = 16; m; m >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, m);
  return acc;
}

// Returns false (uniformly) when the dense screening must run instead.  Unit-step
// stages only (the planner enables it for s == 1).
template <typename Elem, int P>
__device__ bool sea_screen(const SmemLayout& L, const StageGeom& g, int b, const StagePlan& pl, int coff_w,
                           int nblk, int ox0, int oy, int frame_w, int frame_h) {
  using VcT = typename std::conditional<sizeof(Elem) == 1, uint16_t, uint32_t>::type;
  constexpr int EPW = 4 / sizeof(Elem);
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
  const int G = g.G, r = g.r, N = G * G;
  const int bww = pl.bw / EPW, cbw = pl.cbw / EPW, wpr = b / EPW;
  const int parts = pl.parts;
  const FastDiv fG(G, pl.mG);
  VcT* vc = reinterpret_cast<VcT*>(L.vc);  // [P][G][vcs]
  // bounds go to the part-0 arrays; later parts must read 0 when select_block folds them
  for (int k = tid; k < nblk * (parts - 1) * N; k += nt) L.sad[(k / ((parts - 1) * N)) * parts * N + N + k % ((parts - 1) * N)] = 0;
  if (tid < nblk) {
    // valid candidates of block kb: i in [ilo, ihi] x j in [jlo, jhi] (fme.py:250-253, step 1)
    const int ox = ox0 + tid * b;
    int* rc = L.rect + 4 * tid;
    rc[0] = max(0, r - (ox + g.cx));
    rc[1] = min(G - 1, r + (frame_w - b - ox - g.cx));
    rc[2] = max(0, r - (oy + g.cy));
    rc[3] = min(G - 1, r + (frame_h - b - oy - g.cy));
  }
  // current-block plane sums
  for (int q = warp; q < nblk * P; q += nw) {
    const int kb = q / P, p = q - kb * P;
    uint32_t acc = 0;
    for (int idx = lane; idx < b * wpr; idx += 32) {
      const int y = idx / wpr, w = idx - y * wpr;
      acc += word_sum<Elem>(L.cur[(p * b + y) * cbw + coff_w + kb * wpr + w]);
    }
    for (int m = 16; m; m >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, m);
    if (lane == 0) L.csum[q] = (int)acc;
  }
  // column sums over the b rows of every candidate row offset j, per element column:
  // a sliding window down the staged rows, all elements of a word at once
  for (int q = tid; q < P * bww; q += nt) {
    const int p = q / bww, w = q - p * bww;
    const uint32_t* col = L.win + p * pl.wrows * bww + w;
    VcT* dst = vc + p * G * pl.vcs + w * EPW;
    uint32_t a0 = 0, a1 = 0;
    auto add = [&](uint32_t v, bool sub) {
      uint32_t lo, hi;
      if constexpr (sizeof(Elem) == 1) {
        lo = v & 0x00ff00ffu;  // bytes 0, 2 in 16-bit lanes (b * 255 < 65536)
        hi = (v >> 8) & 0x00ff00ffu;
      } else {
        lo = v & 0xffffu;
        hi = v >> 16;
      }
      a0 = sub ? a0 - lo : a0 + lo;
      a1 = sub ? a1 - hi : a1 + hi;
    };
    for (int y = 0; y < b - 1; ++y) add(col[y * bww], false);
    for (int j = 0; j < G; ++j) {
      add(col[(j + b - 1) * bww], false);
      if constexpr (sizeof(Elem) == 1) {
        dst[0] = (VcT)(a0 & 0xffffu);
        dst[1] = (VcT)(a1 & 0xffffu);
        dst[2] = (VcT)(a0 >> 16);
        dst[3] = (VcT)(a1 >> 16);
      } else {
        dst[0] = a0;
        dst[1] = a1;
      }
      dst += pl.vcs;
      add(col[j * bww], true);
    }
  }
  __syncthreads();
  // LB of every candidate: one thread per (block, candidate row, column chunk)
  // slides the P box sums along its columns, keeping the smallest bound over valid
  // columns of the row (chunks combine with atomicMin)
  uint32_t* rowmin = reinterpret_cast<uint32_t*>(L.klist2);  // [nblk * G]
  const int nrow = nblk * G;
  const int nch = max(1, min(4, min(G, nt / nrow)));
  const int chw = (G + nch - 1) / nch;
  for (int q = tid; q < nrow; q += nt) rowmin[q] = 0xffffffffu;
  __syncthreads();
  for (int t = tid; t < nrow * nch; t += nt) {
    const int q = t / nch, ch = t - q * nch;
    uint32_t kb, j;
    fG.divmod(q, kb, j);
    const int i0 = ch * chw, i1 = min(G, i0 + chw);
    if (i0 >= i1) continue;
    const int* rc = L.rect + 4 * kb;
    const bool row_ok = (int)j >= rc[2] && (int)j <= rc[3];
    int box[P], C[P];
    const VcT* row = vc + j * pl.vcs + g.d + kb * b + i0;  // plane p at + p * G * vcs
    const int pst = G * pl.vcs;
#pragma unroll
    for (int p = 0; p < P; ++p) {
      box[p] = 0;
      C[p] = L.csum[kb * P + p];
    }
#pragma unroll 4
    for (int x = 0; x < b; ++x)
#pragma unroll
      for (int p = 0; p < P; ++p) box[p] += (int)row[p * pst + x];
    uint32_t* dst = L.sad + kb * parts * N + j * G;
    uint32_t mn = 0xffffffffu;
    const int vlo = row_ok ? rc[0] : G, vhi = row_ok ? rc[1] : -1;
    for (int i = i0; i < i1; ++i) {
      if (i > i0) {
#pragma unroll
        for (int p = 0; p < P; ++p) box[p] += (int)row[p * pst + i - i0 - 1 + b] - (int)row[p * pst + i - i0 - 1];
      }
      uint32_t lb = 0;
#pragma unroll
      for (int p = 0; p < P; ++p) lb += (uint32_t)abs(box[p] - C[p]);
      dst[i] = lb;
      if (i >= vlo && i <= vhi) mn = min(mn, lb);
    }
    if (mn != 0xffffffffu) atomicMin(rowmin + q, mn);
  }
  __syncthreads();
  // smallest bound per block (L.seaM[kb] = -1: no valid candidate)
  for (int kb = warp; kb < nblk; kb += nw) {
    uint32_t mn = 0xffffffffu;
    for (int j = lane; j < G; j += 32) mn = min(mn, rowmin[kb * G + j]);
    for (int m = 16; m; m >>= 1) mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, m));
    if (lane == 0) {
      const int* rc = L.rect + 4 * kb;
      L.seaM[kb] = (rc[0] <= rc[1] && rc[2] <= rc[3]) ? (int)mn : -1;
      L.seaT[kb] = 0xffffffffu;
      L.seaK0[kb] = 0x7fffffff;
    }
  }
  if (tid == 0) L.misc[9] = 0;
  __syncthreads();
  // Two rounds of exact SADs: (1) every candidate at the smallest bound -- the
  // exact match, where the content has one, has bound 0 -- giving T = their
  // smallest SAD; (2) every remaining candidate with bound <= T.  Only rows
  // whose smallest bound is in range are scanned.
  for (int round = 0; round < 2; ++round) {
    for (int q = tid; q < nblk * G; q += nt) {
      uint32_t kb, j;
      fG.divmod(q, kb, j);
      if (L.seaM[kb] < 0) continue;
      const uint32_t lo = (uint32_t)L.seaM[kb], hi = round == 0 ? lo : L.seaT[kb];
      if (rowmin[q] > hi || (round == 1 && hi <= lo)) continue;
      const int* rc = L.rect + 4 * kb;
      const uint32_t* lbs = L.sad + kb * parts * N + j * G;
      for (int i = rc[0]; i <= rc[1]; ++i) {
        const uint32_t v = lbs[i];
        // round 1 wrote exact SADs (>= their bound == lo) into the array: skip values at lo
        if (round == 0 ? v != lo : (v <= lo || v > hi)) continue;
        const int slot = atomicAdd(&L.misc[9], 1);
        if (slot < pl.sea_cap) L.klist[slot] = (int)(q * G) + i;
      }
    }
    __syncthreads();
    const int n = L.misc[9];
    if (n > pl.sea_cap) return false;
    for (int e = warp; e < n; e += nw) {
      uint32_t qb, i, kb, j;
      fG.divmod(L.klist[e], qb, i);
      fG.divmod(qb, kb, j);
      const uint32_t sd = warp_sad<Elem>(L, pl, P, b, coff_w + kb * wpr, g.d + kb * b + i, j);
      if (lane == 0) {
        L.sad[kb * parts * N + j * G + i] = sd;
        if (round == 0) atomicMin(&L.seaT[kb], sd);
        if (sd == 0) atomicMin(&L.seaK0[kb], (int)(j * G + i));
      }
    }
    __syncthreads();
    if (round == 0) {
      // T > 0: no exact match.  Candidates with bounds in (T, sthr] would reach
      // select_block's contender tests with their bound instead of their SAD and
      // cost a count_lo each; the dense screening is cheaper for those blocks.
      bool exact = true;
      for (int kb = 0; kb < nblk; ++kb) exact &= L.seaM[kb] < 0 || L.seaT[kb] == 0;
      if (!exact) return false;
    }
    if (tid == 0) L.misc[9] = 0;
    __syncthreads();
  }
  return true;
}

// Result of a block the SEA screening settled: every block it accepts has an
// exact match (minimum SAD 0), so with lam < 1 the answer is the first
// zero-SAD candidate in canonical order with energy 0.0 (select_block's
// zero-SAD exit, fme.py:266) -- no pass over the candidate sums is needed.
__device__ __forceinline__ StageResult sea_result(const SmemLayout& L, const StageGeom& g, int kb) {
  StageResult res;
  const int* rc = L.rect + 4 * kb;
  const int k = L.seaK0[kb];
  if (L.seaM[kb] < 0) {  // no valid candidate
    res.nvalid = 0;
    res.dx = res.dy = 0;
    res.energy = 0.0;
    return res;
  }
  res.nvalid = (rc[1] - rc[0] + 1) * (rc[3] - rc[2] + 1);
  res.dx = g.cx + (k % g.G - g.r) * g.s;
  res.dy = g.cy + (k / g.G - g.r) * g.s;
  res.energy = 0.0;
  return res;
}

// Staging + integer SAD of one stage for nblk horizontally adjacent blocks
// sharing one search centre (nblk > 1 only for level 0's first searched stage,
// whose centre is (0, 0) for every block).  All threads participate.
template <typename Elem, int CW, int TY, bool SHIFT>
__device__ StageGeom stage_sad(const SmemLayout& L, const PairCtx<Elem>& pc, const StagePlan& pl,
                               const CUtensorMap* tm_win, const CUtensorMap* tm_cur, uint32_t& phase, int ox, int oy,
                               int b, int cx, int cy, int r, int s, int nblk, int& coff_e) {
  constexpr int EPW = 4 / sizeof(Elem);
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
  const int coff_w = (ox - cx0) / EPW;
  coff_e = ox - cx0;  // element offset of the block inside each staged cur row
  const int tid = threadIdx.x;
  // sub-word phases used by this CTA's candidate columns
  unsigned phase_mask = 0;
  if (!SHIFT && pl.copies)
    for (int i = 0; i < min(g.G, EPW); ++i) phase_mask |= 1u << ((g.d + i * s) % EPW);

  __syncthreads();  // previous users of smem are done; mbarrier init visible
  if (tid == 0) L.misc[10] = 0;  // set to 1 below when the SEA screening settles the stage
  if (pl.use_tma && pl.pg == pc.P && !(phase_mask & ~1u) && !pl.debug) {
    // common case, one TMA pass: clear the atomic-accumulated sums while the
    // boxes are in flight; each thread's mbarrier wait then makes the staged
    // tiles visible to it, so no CTA barrier is needed after the wait
    if (tid == 0) {
      mbar_expect_tx(L.bar, (uint32_t)(pl.tma_bytes));  // full boxes, OOB included
      tma_load_3d(L.win, tm_win, g.tx0, g.wy0, pc.ref_z, L.bar);
      tma_load_3d(L.cur, tm_cur, cx0, oy, pc.cur_z, L.bar);
    }
    if (pl.split && !pl.sea)
      for (int k = tid; k < nblk * pl.parts * g.G * g.G; k += blockDim.x) L.sad[k] = 0;
    __syncthreads();
    mbar_wait(L.bar, phase);
    phase ^= 1;
    if (pl.sea) {
      const bool done = pc.P == 4 ? sea_screen<Elem, 4>(L, g, b, pl, coff_w, nblk, ox, oy, pc.frame_w, pc.frame_h)
                                  : sea_screen<Elem, 1>(L, g, b, pl, coff_w, nblk, ox, oy, pc.frame_w, pc.frame_h);
      if (done) {
        if (tid == 0) L.misc[10] = 1;
        __syncthreads();
        return g;
      }
      if (pl.split) {  // dense fallback: its split tail items accumulate with atomics
        for (int k = tid; k < nblk * pl.parts * g.G * g.G; k += blockDim.x) L.sad[k] = 0;
        __syncthreads();
      }
    }
    sad_items<Elem, CW, TY, SHIFT>(L, g, b, pc.P, pl, coff_w, false, nblk);
    __syncthreads();
    return g;
  }
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
    if (pl.split && p0 == 0)  // split tail items accumulate with atomics
      for (int k = tid; k < nblk * pl.parts * g.G * g.G; k += blockDim.x) L.sad[k] = 0;
    if (phase_mask & ~1u) {
      __syncthreads();
      build_phase_copies<Elem>(L, pl, npl, phase_mask);
    }
    __syncthreads();
#ifdef BMC_EXPERIMENTS
    if (pl.debug & 2) {  // measurement only (BMC_DEBUG_SKIP=2): no screening, every SAD reads 0
      for (int k = tid; k < nblk * pl.parts * g.G * g.G; k += blockDim.x) L.sad[k] = 0;
      continue;
    }
#endif
    sad_items<Elem, CW, TY, SHIFT>(L, g, b, npl, pl, coff_w, p0 > 0, nblk);
  }
  __syncthreads();
  return g;
}

// Exact selection for one block of the staged set (block kb: its window starts
// kb*b elements further into the staged rows, its partial sums at sad).
// All threads participate and receive the result.
template <typename Elem, int CW, int TY, bool SHIFT>
__device__ StageResult select_block(const SmemLayout& L, const PairCtx<Elem>& pc, const StagePlan& pl,
                                    const StageGeom& g, uint32_t* sad, int ox, int oy, int b, int coff_e,
                                    int slot = 0) {
  const FastDiv fGG(g.G, pl.mG);  // candidate index -> (i, j) without an integer divide
  const int r = g.r, s = g.s, cx = g.cx, cy = g.cy;
  const int N = g.G * g.G;
  const int nt = blockDim.x, nw = nt >> 5;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int n = pc.P * b * b;
#ifdef BMC_EXPERIMENTS
  if (pl.debug & 1) {  // measurement only (BMC_DEBUG_SKIP=1): no selection, report the centre
    StageResult res;
    res.dx = cx;
    res.dy = cy;
    res.energy = 0.0;
    res.nvalid = 1;
    return res;
  }
#endif
  // valid candidates form a rectangle i in [ilo, ihi] x j in [jlo, jhi] (fme.py:250-253)
  const FastDiv fsd(s, pl.ms);
  auto fdiv = [&](int a) { return a >= 0 ? (int)fsd.div(a) : -(int)fsd.div(-a + s - 1); };  // floor(a / s)
  const int ilo = max(0, r - fdiv(ox + cx)), ihi = min(g.G - 1, r + fdiv(pc.frame_w - b - ox - cx));
  const int jlo = max(0, r - fdiv(oy + cy)), jhi = min(g.G - 1, r + fdiv(pc.frame_h - b - oy - cy));
  const int wi = ihi - ilo + 1, wj = jhi - jlo + 1;
  StageResult res;
  res.nvalid = (wi > 0 && wj > 0) ? wi * wj : 0;
  if (res.nvalid == 0) {
    res.dx = res.dy = 0;
    res.energy = 0.0;
    return res;
  }

  const FastDiv fwi = wi == g.G ? FastDiv(wi, pl.mG) : FastDiv(wi);  // interior blocks: the full grid width
  // pass 1: fold the parts; first minimum SAD among valid candidates (key = sad<<32 | k)
  unsigned long long best = ~0ull;
  {
    const int parts = pl.parts;
    for (int v = tid; v < res.nvalid; v += nt) {
      const int jv = fwi.div(v);
      const int k = (jlo + jv) * g.G + ilo + (v - jv * wi);
      uint32_t sk = sad[k];
      for (int q = 1; q < parts; ++q) sk += sad[q * N + k];
      if (parts > 1) sad[k] = sk;  // the contender passes read the folded sums
      const unsigned long long key = ((unsigned long long)sk << 32) | (unsigned)k;
      best = key < best ? key : best;
    }
  }
  for (int m = 16; m; m >>= 1) {
    const unsigned long long o = __shfl_xor_sync(0xffffffffu, best, m);
    best = o < best ? o : best;
  }
  // consecutive blocks of a kblk set alternate halves of red64: the zero-SAD
  // exit below has no trailing barrier, so a fast warp's next write must not
  // land in the half a slower warp may still be folding
  unsigned long long* red = L.red64 + (slot & 1) * kMaxSW;
  if (lane == 0) red[warp] = best;
  __syncthreads();
  // every thread folds the per-warp minima itself (no serial step, no second barrier)
  unsigned long long b0 = red[0];
  for (int w = 1; w < nw; ++w) b0 = red[w] < b0 ? red[w] : b0;
  if (tid == 0) {
    L.misc[3] = 0;  // klist size   (ordered before use by the barrier after the table fill)
    L.misc[5] = 0;  // replay list size
  }
  const int m0 = (int)(b0 & 0xffffffffu);
  const unsigned sad0 = (unsigned)(b0 >> 32);
  if (sad0 == 0 && pc.oml > 0.0) {
    // S == 0 gives E == 0.0 exactly; any earlier candidate has S > 0 and,
    // with (1-lam) > 0, E > 0.  The first zero-SAD candidate wins.
    cand_valid_ij(g, ox, oy, b, pc.frame_h, pc.frame_w, (int)((m0) - fGG.div(m0) * g.G), (int)fGG.div(m0), res.dx, res.dy);
    res.energy = 0.0;
    return res;
  }
  if (sizeof(Elem) == 1)  // fl(v/255) table for the exact replays (only blocks that reach here pay for it)
    for (int v = tid; v < 256; v += nt) L.tab[v] = __ddiv_rn((double)v, (double)pc.max_value);
  __syncthreads();
  const double unit = (double)pc.max_value * (double)n;
  // exact energy of the min-SAD candidate: numpy's pairwise tree over n samples
  // is perfect, so W warps (a power of two dividing the chain-group count) each
  // take an aligned subtree and warp 0 joins the W subtree sums in tree order
  const int nq = n > 512 ? n / 512 : 1;  // chain groups: (n / 128 leaves) * 8 chains / 32 lanes
  int W = 1;
  while (2 * W <= nw && 2 * W <= nq) W *= 2;
  if (W > 1) {
    if (warp < W) {
      int dx, dy;
      const int mi = (int)((m0) - fGG.div(m0) * g.G), mj = (int)fGG.div(m0);
      cand_valid_ij(g, ox, oy, b, pc.frame_h, pc.frame_w, mi, mj, dx, dy);
      double tsum;
      int tcnt;
      exact_cand_partial<Elem>(L, pl, g, pc, ox, oy, b, coff_e, mi, mj, dx, dy, warp * (nq / W), (warp + 1) * (nq / W),
                               tsum, tcnt);
      if (lane == 0) {
        L.best_e[warp] = tsum;
        L.best_k[warp] = tcnt;
      }
    }
    __syncthreads();
  }
  if (warp == 0) {
    double e0 = 0.0;
    if (sad0 != 0) {
      if (W > 1) {
        if (lane == 0) {
          double v[kMaxSW];
          int cnt = 0;
          for (int w = 0; w < W; ++w) {
            v[w] = L.best_e[w];
            cnt += L.best_k[w];
          }
          for (int st = 1; st < W; st *= 2)
            for (int w = 0; w + st < W; w += 2 * st) v[w] = __dadd_rn(v[w], v[w + st]);
          e0 = exact_finish(v[0], cnt, n, pc.oml, pc.lam).energy;
        }
      } else {
        int dx, dy;
        cand_valid_ij(g, ox, oy, b, pc.frame_h, pc.frame_w, (int)((m0) - fGG.div(m0) * g.G), (int)fGG.div(m0), dx, dy);
        e0 = exact_cand<Elem>(L, pl, g, pc, ox, oy, b, coff_e, (int)((m0) - fGG.div(m0) * g.G), (int)fGG.div(m0), dx,
                              dy);
      }
    }
    if (lane == 0) {
      L.miscd[0] = e0;
      // integer SAD threshold: the largest S whose bound (1-lam)*S/(s*n) can
      // still reach e0 + eps (the bound is monotone in S)
      const double lim = e0 + kScreenEps;
      unsigned thr = 0xffffffffu;
      if (pc.oml > 0.0) {
        double est = floor(lim / pc.oml * unit) + 2.0;
        long long t = est > 4294967295.0 ? 4294967295LL : (long long)est;
        while (t >= 0 && __dmul_rn(pc.oml, __ddiv_rn((double)t, unit)) > lim) --t;
        thr = t < 0 ? 0u : (unsigned)t;
      }
      L.misc[6] = (int)thr;
    }
  }
  __syncthreads();
  const double e0 = L.miscd[0];
  const unsigned sthr = (unsigned)L.misc[6];
  // pass 2: SAD contenders (candidates whose lower bound reaches e0).  A
  // sample that does not count contributes at most D-1 to S and one that counts
  // at most s, so C >= (S - (D-1) n) / (s - D + 1): a free sparsity bound that
  // prunes poor candidates before any count_lo / float64 work.
  {
    const int Dc = (int)floor(pc.tol * (double)pc.max_value + 1e-9) + 1;
    const long long slack = (long long)(Dc - 1) * n;
    const int span = pc.max_value - Dc + 1;
    const double lim2 = e0 + kScreenEps;
    for (int v = tid; v < res.nvalid; v += nt) {
      const int jv = fwi.div(v);
      const int k = (jlo + jv) * g.G + ilo + (v - jv * wi);
      if (k == m0 || sad[k] > sthr) continue;
      if (pc.lam > 0.0 && span > 0 && (long long)sad[k] > slack) {
        const long long cl = ((long long)sad[k] - slack + span - 1) / span;
        const double elb = __dadd_rn(__dmul_rn(pc.oml, __ddiv_rn((double)sad[k], unit)),
                                     __dmul_rn(pc.lam, __ddiv_rn((double)cl, (double)n)));
        if (elb - kScreenEps > lim2) continue;
      }
      L.klist[atomicAdd(&L.misc[3], 1)] = k;
    }
  }
  __syncthreads();
  int nk = L.misc[3];
  const int* rlist = L.klist;
  if (nk > nw && pc.lam > 0.0) {
    // Too many for one round of float64 replays: tighten the bound with the
    // sparsity term.  C_lo = #(|r-c| >= D) <= C because every integer
    // difference >= D passes the float64 test d > tol; then
    // E >= (1-lam)*S/(s*n) + lam*C_lo/n (up to float rounding << eps).
    const int D = (int)floor(pc.tol * (double)pc.max_value + 1e-9) + 1;
    const double lim = e0 + kScreenEps;
    for (int e = warp; e < nk; e += nw) {
      const int k = L.klist[e];
      const int clo = count_lo<Elem>(L, pl, g, pc, ox, oy, b, coff_e, (int)((k) - fGG.div(k) * g.G), (int)fGG.div(k), D);
      const double elb = __dadd_rn(__dmul_rn(pc.oml, __ddiv_rn((double)sad[k], unit)),
                                   __dmul_rn(pc.lam, __ddiv_rn((double)clo, (double)n)));
      if (lane == 0 && elb - kScreenEps <= lim) L.klist2[atomicAdd(&L.misc[5], 1)] = k;
    }
    __syncthreads();
    nk = L.misc[5];
    rlist = L.klist2;
  }
  if (W > 1 && nk < nw) {
    // fewer replays than warps (large blocks): every replay split across W warps
    // (aligned subtrees, joined in tree order by thread 0), one after another
    if (tid == 0) {
      L.miscd[1] = e0;
      L.misc[4] = m0;
    }
    for (int e = 0; e < nk; ++e) {
      const int k = rlist[e];
      if (warp < W) {
        int dx, dy;
        const int ki = (int)((k) - fGG.div(k) * g.G), kj = (int)fGG.div(k);
        cand_valid_ij(g, ox, oy, b, pc.frame_h, pc.frame_w, ki, kj, dx, dy);
        double tsum;
        int tcnt;
        exact_cand_partial<Elem>(L, pl, g, pc, ox, oy, b, coff_e, ki, kj, dx, dy, warp * (nq / W),
                                 (warp + 1) * (nq / W), tsum, tcnt);
        if (lane == 0) {
          L.best_e[warp] = tsum;
          L.best_k[warp] = tcnt;
        }
      }
      __syncthreads();
      if (tid == 0) {
        double v[kMaxSW];
        int cnt = 0;
        for (int w = 0; w < W; ++w) {
          v[w] = L.best_e[w];
          cnt += L.best_k[w];
        }
        for (int st = 1; st < W; st *= 2)
          for (int w = 0; w + st < W; w += 2 * st) v[w] = __dadd_rn(v[w], v[w + st]);
        const double ek = exact_finish(v[0], cnt, n, pc.oml, pc.lam).energy;
        if (ek < L.miscd[1] || (ek == L.miscd[1] && k < L.misc[4])) {
          L.miscd[1] = ek;
          L.misc[4] = k;
        }
      }
      __syncthreads();
    }
    if (nk == 0) __syncthreads();
    const int kw = L.misc[4];
    cand_valid_ij(g, ox, oy, b, pc.frame_h, pc.frame_w, (int)((kw) - fGG.div(kw) * g.G), (int)fGG.div(kw), res.dx,
                  res.dy);
    res.energy = L.miscd[1];
    return res;
  }
  double be = (warp == 0) ? e0 : 1e300;
  int bk = (warp == 0) ? m0 : 0x7fffffff;
  for (int e = warp; e < nk; e += nw) {
    const int k = rlist[e];
    int dx, dy;
    cand_valid_ij(g, ox, oy, b, pc.frame_h, pc.frame_w, (int)((k) - fGG.div(k) * g.G), (int)fGG.div(k), dx, dy);
    const double ek = exact_cand<Elem>(L, pl, g, pc, ox, oy, b, coff_e, (int)((k) - fGG.div(k) * g.G), (int)fGG.div(k), dx, dy);
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
    for (int w = 1; w < nw; ++w) {
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
  cand_valid_ij(g, ox, oy, b, pc.frame_h, pc.frame_w, (int)((kw) - fGG.div(kw) * g.G), (int)fGG.div(kw), res.dx, res.dy);
  res.energy = L.miscd[1];
  return res;
}


// One stage for one block (the single-block path).
template <typename Elem, int CW, int TY, bool SHIFT>
__device__ StageResult stage_search(const SmemLayout& L, const PairCtx<Elem>& pc, const StagePlan& pl,
                                    const CUtensorMap* tm_win, const CUtensorMap* tm_cur, uint32_t& phase, int ox,
                                    int oy, int b, int cx, int cy, int r, int s) {
  int coff_e;
  const StageGeom g = stage_sad<Elem, CW, TY, SHIFT>(L, pc, pl, tm_win, tm_cur, phase, ox, oy, b, cx, cy, r, s, 1,
                                                     coff_e);
  if (pl.sea && L.misc[10]) return sea_result(L, g, 0);
  return select_block<Elem, CW, TY, SHIFT>(L, pc, pl, g, L.sad, ox, oy, b, coff_e);
}

// ---------------------------------------------------------------------------
// the stage kernel
// ---------------------------------------------------------------------------
template <typename Elem, int CW, int TY, bool SHIFT>
__global__ void __launch_bounds__(kMaxStageThreads, BMC_STAGE_MINB)
    fme_stage_kernel(const __grid_constant__ CUtensorMap tm_win, const __grid_constant__ CUtensorMap tm_cur,
                     const StageLaunch a) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const SmemLayout L = carve(smem_raw, a.plan);
  const bmc_fme_params& p = a.prm;
  const int b = a.b;
  uint32_t phase = 0;
  if (a.plan.use_tma && threadIdx.x == 0) mbar_init(L.bar, 1);
  // Persistent CTAs: the grid is sized to the resident capacity and strides
  // over the (pair, block) work list, so the prologue and the per-stage
  // constants are paid once per CTA, not once per block.
  const uint32_t cells = (uint32_t)a.gw * a.gh;
  for (uint32_t work = blockIdx.x; work < a.total; work += gridDim.x) {
    int pair = 0, gx = 0, gy = 0, ox, oy, sx = 0, sy = 0;
    long long cell = 0;
    if (a.single) {
      ox = a.ox;
      oy = a.oy;
      sx = a.cx;
      sy = a.cy;
    } else if (a.kblk > 1) {
      // nblk horizontally adjacent blocks of level 0's first stage share one window (centre (0, 0))
      const uint32_t gwg = a.gwg;
      const uint32_t cg = gwg * a.gh;
      pair = (int)FastDiv(cg, a.plan.mcells).div(work);
      const int blk = (int)(work - (uint32_t)pair * cg);
      gy = (int)FastDiv(gwg, a.plan.mgw).div(blk);
      const int gx0 = (blk - gy * (int)gwg) * a.kblk;
      const int nb = min(a.kblk, a.gw - gx0);
      PairCtx<Elem> pc;
      const int cur_f = a.cur_index[pair], ref_f = a.ref_index[pair];
      pc.cur = reinterpret_cast<const Elem*>(a.planes) + (long long)cur_f * p.frame_stride;
      pc.ref = reinterpret_cast<const Elem*>(a.ref_planes) + (long long)ref_f * p.frame_stride;
      pc.cur_z = cur_f * p.planes;
      pc.ref_z = ref_f * p.planes;
      pc.pitch = p.pitch;
      pc.plane_stride = p.plane_stride;
      pc.frame_h = p.pad_h;
      pc.frame_w = p.pad_w;
      pc.P = p.planes;
      pc.max_value = p.max_value;
      pc.tol = p.sparsity_tolerance;
      pc.lam = p.lam;
      pc.oml = p.one_minus_lam;
      pc.tab = sizeof(Elem) == 1 ? L.tab : a.tab16;
      const int ox0 = gx0 * b;
      oy = gy * b;
      int coff_e;
      const StageGeom g = stage_sad<Elem, CW, TY, SHIFT>(L, pc, a.plan, &tm_win, &tm_cur, phase, ox0, oy, b, 0, 0,
                                                         a.r, a.s, a.kblk, coff_e);
      const int nsad = a.plan.parts * g.G * g.G;
      for (int kb = 0; kb < nb; ++kb) {
        StageGeom gk = g;
        gk.d += kb * b;
        const StageResult res = (a.plan.sea && L.misc[10])
                                    ? sea_result(L, g, kb)
                                    : select_block<Elem, CW, TY, SHIFT>(L, pc, a.plan, gk, L.sad + kb * nsad,
                                                                        ox0 + kb * b, oy, b, coff_e + kb * b, kb);
        if (threadIdx.x == 0) {
          const long long c = (long long)pair * cells + (long long)gy * a.gw + gx0 + kb;
          a.mv[2 * c] = res.dx;
          a.mv[2 * c + 1] = res.dy;
          a.energy[c] = res.energy;
          if (a.last) {
            bool m;
            if (a.final_level) {
              const bool in_real = oy < p.real_h && ox0 + kb * b < p.real_w;  // fme.py:377-384
              m = !(res.energy > p.refine_block_threshold && in_real);
            } else {
              m = res.energy <= p.split_threshold;  // fme.py:386
            }
            a.matched[c] = m ? 1 : 0;
          }
          atomicAdd(a.evals + pair, (unsigned long long)(res.nvalid + a.extra_evals));
        }
      }
      continue;
    } else {
      pair = (int)FastDiv(cells, a.plan.mcells).div(work);
      const int blk = (int)(work - (uint32_t)pair * cells);
      gy = (int)FastDiv(a.gw, a.plan.mgw).div(blk);
      gx = blk - gy * a.gw;
      cell = (long long)pair * cells + blk;
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
          continue;
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
    StageResult res;
    for (int attempt = 0;; ++attempt) {  // no valid candidate: re-centre on (0, 0) (fme.py:310-313)
      res = stage_search<Elem, CW, TY, SHIFT>(L, pc, a.plan, &tm_win, &tm_cur, phase, ox, oy, b, attempt ? 0 : sx,
                                              attempt ? 0 : sy, a.r, a.s);
      if (res.nvalid || attempt) break;
    }
    if (threadIdx.x != 0) continue;
    if (a.single) {
      a.mv[0] = res.dx;
      a.mv[1] = res.dy;
      a.energy[0] = res.energy;
      a.nvalid_out[0] = res.nvalid;
      continue;
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
}

template <typename K>
inline int set_smem(K kern, int bytes) {
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

inline bool sync_debug() {
  static int v = -1;
  if (v < 0) {
    const char* e = knob_env("BMC_SYNC_DEBUG");
    v = (e && *e && *e != '0') ? 1 : 0;
  }
  return v == 1;
}

template <typename E, int CW, int TY, bool SH>
inline int launch_one(const CUtensorMap& tw, const CUtensorMap& tc, const StageLaunch& a, dim3 grid, cudaStream_t st) {
  int rc = set_smem(fme_stage_kernel<E, CW, TY, SH>, a.plan.smem);
  if (rc) return rc;
  StageLaunch la = a;
  la.gwg = (uint32_t)((a.gw + a.kblk - 1) / a.kblk);
  la.total = a.single ? 1u : la.gwg * (uint32_t)a.gh * (uint32_t)a.n_pairs;
  static const bool plan_log = [] {
    const char* e = knob_env("BMC_PLAN_LOG");
    return e && *e && *e != '0';
  }();
  if (plan_log)
    fprintf(stderr, "[bmc] stage eb=%d CW=%d TY=%d shift=%d level %d b %d r %d s %d grid %ux%u threads %d parts %d "
            "pg %d tma %d box %dx%d copies %d smem %d\n", (int)sizeof(E), CW, TY, (int)SH, a.level, a.b, a.r, a.s,
            grid.x, grid.y, a.plan.threads, a.plan.parts, a.plan.pg, a.plan.use_tma, a.plan.bw, a.plan.hwin,
            a.plan.copies, a.plan.smem);
  // persistent grid: resident capacity (occupancy x SMs), capped by the work count
  static std::mutex omu;
  static const void* okeys[512];
  static int othreads[512], osmem[512], ovals[512];
  static int on = 0;
  int per_sm = 0;
  {
    std::lock_guard<std::mutex> g(omu);
    const void* key = reinterpret_cast<const void*>(fme_stage_kernel<E, CW, TY, SH>);
    for (int i = 0; i < on; ++i)
      if (okeys[i] == key && othreads[i] == a.plan.threads && osmem[i] == a.plan.smem) per_sm = ovals[i];
    if (!per_sm) {
      cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fme_stage_kernel<E, CW, TY, SH>,
                                                                    a.plan.threads, a.plan.smem);
      if (e != cudaSuccess) return cuda_status(e, "cudaOccupancyMaxActiveBlocksPerMultiprocessor");
      if (per_sm < 1) per_sm = 1;
      if (on < 512) {
        okeys[on] = key;
        othreads[on] = a.plan.threads;
        osmem[on] = a.plan.smem;
        ovals[on] = per_sm;
        ++on;
      }
    }
  }
  static const int sms = [] {  // thread-safe one-time init
    int dev = 0, n = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n < 1 ? 1 : n;
  }();
  const long long work = (long long)grid.x * grid.y;
  static const int persist_mult = [] {  // resident waves per launch; 0 = one CTA per block
    const char* e = knob_env("BMC_PERSIST");
    return e ? atoi(e) : 0;
  }();
  const long long capacity = persist_mult > 0 ? (long long)per_sm * sms * persist_mult : work;
  const unsigned nblk = (unsigned)(work < capacity ? work : capacity);
  fme_stage_kernel<E, CW, TY, SH><<<nblk, a.plan.threads, a.plan.smem, st>>>(tw, tc, la);
  rc = cuda_status(cudaGetLastError(), "fme_stage_kernel");
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  if (!rc && sync_debug() && cudaStreamIsCapturing(st, &cap) == cudaSuccess && cap == cudaStreamCaptureStatusNone) {
    cudaError_t e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) {
      set_error("fme_stage_kernel<eb=%d,CW=%d,TY=%d,shift=%d> level %d b %d r %d s %d tma %d box %dx%dx%d cbw %d "
                "smem %d threads %d parts %d copies %d: %s", (int)sizeof(E), CW, TY, (int)SH, a.level, a.b, a.r, a.s,
                a.plan.use_tma, a.plan.bw, a.plan.hwin, a.plan.pg, a.plan.cbw, a.plan.smem, a.plan.threads,
                a.plan.parts, a.plan.copies, cudaGetErrorString(e));
      return BMC_E_CUDA;
    }
  }
  return rc;
}

template <typename E, int CW, bool SH>
inline int dispatch_ty(const CUtensorMap& tw, const CUtensorMap& tc, const StageLaunch& a, dim3 grid,
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


// One translation unit per (element type, chunk width, shift) instantiates its
// twelve TY variants (bmc_fme_k_*.cu), so the build compiles them in parallel.
int launch_stage_u8c4(bool shift, const CUtensorMap& tw, const CUtensorMap& tc, const StageLaunch& a, dim3 grid,
                      cudaStream_t st);
int launch_stage_u8c2(bool shift, const CUtensorMap& tw, const CUtensorMap& tc, const StageLaunch& a, dim3 grid,
                      cudaStream_t st);
int launch_stage_u16(bool shift, const CUtensorMap& tw, const CUtensorMap& tc, const StageLaunch& a, dim3 grid,
                     cudaStream_t st);

}  // namespace bmc
