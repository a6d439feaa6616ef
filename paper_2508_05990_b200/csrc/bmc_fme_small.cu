// Small-block motion estimation (sm_100a): one warp per block, the level's
// three chained stages (fme.py:294-316) run back to back inside the warp.
//
// Used when a candidate has at most 256 samples (P * b * b <= 256: 8x8 Bayer
// blocks, or luma blocks up to 16x16).  For such blocks the staged-window CTA
// of bmc_fme_impl.cuh spends most of its time on per-CTA fixed costs (TMA
// round trip, barriers, selection passes) -- a 4K uint16 clip has 1.9M blocks
// per pair set.  Here a lane owns a candidate: it reads the candidate's rows
// straight from L1/L2 (the two frames of a pair stay L2-resident while their
// blocks are processed), the current block sits in shared memory (broadcast
// reads), and one pass yields both the integer SAD S and the integer sparsity
// lower bound C_lo = #(|r-c| >= D) (bmc_fme_impl.cuh, count_lo).  Selection is
// then exact and warp-local:
//   * min S == 0 (and lam < 1): E == 0 exactly, the first such candidate wins;
//   * otherwise E >= E_lb = (1-lam)*S/(s*n) + lam*C_lo/n (float error << 1e-11):
//     replay (float64, numpy pairwise order) the candidate with the smallest
//     bound, then every candidate whose bound reaches its exact energy; the
//     first minimum in canonical dy-major order wins (np.argmin, fme.py:266).
#include <cuda.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "bmc_internal.cuh"
#include "bmc_launch.cuh"

namespace bmc {

namespace {

constexpr int kSmallWarps = 8;               // blocks per CTA
constexpr int kSmallCurWords = 256 / 2 + 8;  // 256 uint16 samples (or 256 uint8 + slack) per block
constexpr double kEps = 1e-11;

template <typename Elem, bool HIGHD>
__device__ __forceinline__ void word_sc(uint32_t cw, uint32_t rw, uint32_t& S, uint32_t& C, uint32_t k1, uint32_t k2,
                                        uint32_t& a2) {
  if constexpr (sizeof(Elem) == 1) {
    const uint32_t d4 = __vabsdiffu4(cw, rw);
    S = __dp4a(d4, 0x01010101u, S);
    asm("vabsdiff4.u32.u32.u32.add %0, %1, %2, %0;" : "+r"(C) : "r"(d4), "r"(k1));
    asm("vabsdiff4.u32.u32.u32.add %0, %1, %2, %0;" : "+r"(a2) : "r"(d4), "r"(k2));
  } else {
    uint32_t mx, mn;
    asm("max.u16x2 %0, %1, %2;" : "=r"(mx) : "r"(cw), "r"(rw));
    asm("min.u16x2 %0, %1, %2;" : "=r"(mn) : "r"(cw), "r"(rw));
    const uint32_t d2 = mx - mn;
    S = __dp2a_lo(d2, 0x0101u, S);
    const uint32_t f = HIGHD ? (((d2 & 0x7fff7fffu) + k1) & d2) : (((d2 & 0x7fff7fffu) + k1) | d2);
    // lane bit 15 set iff d >= D: IDP.2A adds 0x8000 per counted lane (C holds 0x8000 * count)
    C = __dp2a_lo(f & 0x80008000u, 0x0101u, C);
  }
}

// (S, C_lo) of one candidate: P planes x b rows of WPR words, reference rows
// read through L1 with one funnel shift per word (shift 0 for aligned rows).
// ALIGNED: the row starts on an 8-byte boundary with no sub-word shift (the
// coarse s = 8 and s = 4 stages of 8x8 blocks, half of the unit-step ones):
// one 16-byte or two 8-byte loads per row, no shifts.  Plane strides and the
// row pitch are 16-byte multiples, so the alignment holds for every row.
template <typename Elem, int WPR, bool HIGHD, bool ALIGNED>
__device__ __forceinline__ void cand_sc(const uint32_t* __restrict__ rrow, long long rpitch_w, long long rplane_w,
                                        const uint32_t* crow, int P, int b, int sh, uint32_t k1, uint32_t k2,
                                        uint32_t& S, uint32_t& C, uint32_t& a2) {
  for (int pl = 0; pl < P; ++pl) {
    const uint32_t* rr = rrow + pl * rplane_w;
    for (int y = 0; y < b; ++y) {
      uint32_t w[WPR + 1];
      if constexpr (ALIGNED && WPR == 4) {
        if (((reinterpret_cast<uintptr_t>(rrow)) & 15) == 0) {
          const uint4 v = __ldg(reinterpret_cast<const uint4*>(rr));
          w[0] = v.x; w[1] = v.y; w[2] = v.z; w[3] = v.w;
        } else {  // 8-byte aligned row
          const uint2 v0 = __ldg(reinterpret_cast<const uint2*>(rr)), v1 = __ldg(reinterpret_cast<const uint2*>(rr) + 1);
          w[0] = v0.x; w[1] = v0.y; w[2] = v1.x; w[3] = v1.y;
        }
        w[4] = 0;
      } else if constexpr (ALIGNED) {
        const uint2 v = __ldg(reinterpret_cast<const uint2*>(rr));
        w[0] = v.x; w[1] = v.y; w[2] = 0;
      } else {
#pragma unroll
        for (int q = 0; q <= WPR; ++q) w[q] = __ldg(rr + q);
      }
      uint32_t c[WPR];
      if constexpr (WPR == 4) {
        const uint4 v = *reinterpret_cast<const uint4*>(crow);
        c[0] = v.x; c[1] = v.y; c[2] = v.z; c[3] = v.w;
      } else {
        const uint2 v = *reinterpret_cast<const uint2*>(crow);
        c[0] = v.x; c[1] = v.y;
      }
#pragma unroll
      for (int q = 0; q < WPR; ++q)
        word_sc<Elem, HIGHD>(c[q], ALIGNED ? w[q] : __funnelshift_r(w[q], w[q + 1], sh), S, C, k1, k2, a2);
      rr += rpitch_w;
      crow += WPR;
    }
  }
}

struct SmallStage {
  int dx, dy, nvalid;
  double energy;
};

// One search stage of one block by one warp.
template <typename Elem>
__device__ SmallStage small_stage(const Elem* __restrict__ cur_g, const Elem* __restrict__ ref, const uint32_t* cur_s,
                                  const StageLaunch& a, int ox, int oy, int cx, int cy, int r, int s,
                                  const double* tab) {
  constexpr int EPW = 4 / sizeof(Elem);
  const bmc_fme_params& p = a.prm;
  const int lane = threadIdx.x & 31;
  const int b = a.b, P = p.planes;
  const int n = P * b * b;
  const int wpr = b / EPW;
  const int G = 2 * r + 1;
  const int fw = p.pad_w, fh = p.pad_h;
  // valid rectangle (fme.py:250-253)
  auto fdiv = [](int x, int d) { return x >= 0 ? x / d : -((-x + d - 1) / d); };
  const int ilo = max(0, r - fdiv(ox + cx, s)), ihi = min(G - 1, r + fdiv(fw - b - ox - cx, s));
  const int jlo = max(0, r - fdiv(oy + cy, s)), jhi = min(G - 1, r + fdiv(fh - b - oy - cy, s));
  const int wi = ihi - ilo + 1, wj = jhi - jlo + 1;
  SmallStage res;
  res.nvalid = (wi > 0 && wj > 0) ? wi * wj : 0;
  res.dx = res.dy = 0;
  res.energy = 0.0;
  if (!res.nvalid) return res;
  const int D = (int)floor(p.sparsity_tolerance * (double)p.max_value + 1e-9) + 1;
  const bool count = p.lam > 0.0 && D <= p.max_value;
  uint32_t k1 = 0, k2 = 0;
  if constexpr (EPW == 4) {
    k1 = 0x01010101u * (uint32_t)(D - 1);
    k2 = 0x01010101u * (uint32_t)min(D, 255);
  } else {
    k1 = D <= 32768 ? 0x00010001u * (uint32_t)(0x8000 - D) : 0x00010001u * (uint32_t)(0x10000 - D);
  }
  const bool highd = EPW == 2 && D > 32768;
  const double unit = (double)p.max_value * (double)n;
  // lane-per-candidate screening: (S, E_lb) of every valid candidate
  uint32_t bestS = 0xffffffffu;
  int bestS_k = 0x7fffffff;
  double bestL = 1e300;
  int bestL_k = 0x7fffffff;
  // keep per-lane candidate results for the contender pass (<= 32 * kMaxRounds)
  constexpr int kMaxRounds = 10;  // G <= 17: 289 candidates
  double lbs[kMaxRounds];
  int ks[kMaxRounds];
  const int rounds = (res.nvalid + 31) / 32;
  for (int q = 0; q < kMaxRounds; ++q) {
    lbs[q] = 1e300;
    ks[q] = -1;
  }
  for (int q = 0; q < rounds && q < kMaxRounds; ++q) {
    const int v = q * 32 + lane;
    if (v >= res.nvalid) break;
    const int jv = v / wi;
    const int i = ilo + (v - jv * wi), j = jlo + jv;
    const int dx = cx + (i - r) * s, dy = cy + (j - r) * s;
    const int xr = ox + dx;
    const int sh = (xr % EPW) * 8 * (int)sizeof(Elem);
    uint32_t S = 0, Cacc = 0, a2 = 0;
    const uint32_t* rrow = reinterpret_cast<const uint32_t*>(ref + (long long)(oy + dy) * p.pitch) + xr / EPW;
    const long long rpw = p.pitch / EPW, rplw = p.plane_stride / EPW;
    // whole-row vector loads: 16-byte (or, for 4-word rows, 8-byte) aligned rows without a sub-word shift
    const bool al = sh == 0 && (reinterpret_cast<uintptr_t>(rrow) & 7) == 0;
    if (wpr == 4) {
      if (al) {
        if (highd) cand_sc<Elem, 4, true, true>(rrow, rpw, rplw, cur_s, P, b, sh, k1, k2, S, Cacc, a2);
        else cand_sc<Elem, 4, false, true>(rrow, rpw, rplw, cur_s, P, b, sh, k1, k2, S, Cacc, a2);
      } else {
        if (highd) cand_sc<Elem, 4, true, false>(rrow, rpw, rplw, cur_s, P, b, sh, k1, k2, S, Cacc, a2);
        else cand_sc<Elem, 4, false, false>(rrow, rpw, rplw, cur_s, P, b, sh, k1, k2, S, Cacc, a2);
      }
    } else {
      if (al) {
        if (highd) cand_sc<Elem, 2, true, true>(rrow, rpw, rplw, cur_s, P, b, sh, k1, k2, S, Cacc, a2);
        else cand_sc<Elem, 2, false, true>(rrow, rpw, rplw, cur_s, P, b, sh, k1, k2, S, Cacc, a2);
      } else {
        if (highd) cand_sc<Elem, 2, true, false>(rrow, rpw, rplw, cur_s, P, b, sh, k1, k2, S, Cacc, a2);
        else cand_sc<Elem, 2, false, false>(rrow, rpw, rplw, cur_s, P, b, sh, k1, k2, S, Cacc, a2);
      }
    }
    int C = EPW == 4 ? ((int)Cacc - (int)a2 + n) / 2 : (int)(Cacc >> 15);
    if (!count) C = 0;
    const int k = j * G + i;
    const double lb = __dadd_rn(__dmul_rn(p.one_minus_lam, __ddiv_rn((double)S, unit)),
                                __dmul_rn(p.lam, __ddiv_rn((double)C, (double)n)));
    lbs[q] = lb;
    ks[q] = k;
    if (S < bestS || (S == bestS && k < bestS_k)) {
      bestS = S;
      bestS_k = k;
    }
    if (lb < bestL || (lb == bestL && k < bestL_k)) {
      bestL = lb;
      bestL_k = k;
    }
  }
  for (int m = 16; m; m >>= 1) {
    const uint32_t oS = __shfl_xor_sync(0xffffffffu, bestS, m);
    const int oSk = __shfl_xor_sync(0xffffffffu, bestS_k, m);
    if (oS < bestS || (oS == bestS && oSk < bestS_k)) {
      bestS = oS;
      bestS_k = oSk;
    }
    const double oL = __shfl_xor_sync(0xffffffffu, bestL, m);
    const int oLk = __shfl_xor_sync(0xffffffffu, bestL_k, m);
    if (oL < bestL || (oL == bestL && oLk < bestL_k)) {
      bestL = oL;
      bestL_k = oLk;
    }
  }
  const long long coff = (long long)oy * p.pitch + ox;
  auto replay = [&](int k) {
    const int i = k % G, j = k / G;
    const int dx = cx + (i - r) * s, dy = cy + (j - r) * s;
    return exact_energy_generic<Elem>(cur_g + coff, p.pitch, p.plane_stride,
                                      ref + (long long)(oy + dy) * p.pitch + ox + dx, p.pitch, p.plane_stride, b, P,
                                      tab, p.sparsity_tolerance, p.one_minus_lam, p.lam)
        .energy;
  };
  int wk;
  double we;
  if (bestS == 0 && p.one_minus_lam > 0.0) {
    wk = bestS_k;  // S == 0 => E == 0.0 exactly; every earlier candidate has E > 0
    we = 0.0;
  } else {
    wk = bestL_k;
    we = replay(wk);
    // contenders: bound within eps of the best exact energy found so far
    for (int q = 0; q < rounds && q < kMaxRounds; ++q) {
      unsigned m = __ballot_sync(0xffffffffu, ks[q] >= 0 && ks[q] != wk && lbs[q] - kEps <= we + kEps);
      while (m) {
        const int src = __ffs(m) - 1;
        m &= m - 1;
        const int k = __shfl_sync(0xffffffffu, ks[q], src);
        const double e = replay(k);
        if (e < we || (e == we && k < wk)) {
          we = e;
          wk = k;
        }
      }
    }
  }
  res.dx = cx + (wk % G - r) * s;
  res.dy = cy + (wk / G - r) * s;
  res.energy = we;
  return res;
}

template <typename Elem>
__global__ void __launch_bounds__(kSmallWarps * 32) fme_small_kernel(const StageLaunch a) {
  __shared__ uint32_t cur_s[kSmallWarps][kSmallCurWords];
  __shared__ double tab8[256];
  constexpr int EPW = 4 / sizeof(Elem);
  const bmc_fme_params& p = a.prm;
  if (sizeof(Elem) == 1)
    for (int v = threadIdx.x; v < 256; v += blockDim.x) tab8[v] = __ddiv_rn((double)v, (double)p.max_value);
  __syncthreads();
  const double* tab = sizeof(Elem) == 1 ? tab8 : a.tab16;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long cells = (long long)a.gw * a.gh;
  const long long wid = (long long)blockIdx.x * kSmallWarps + warp;
  if (wid >= cells * a.n_pairs) return;
  const int pair = (int)(wid / cells);
  const int blk = (int)(wid - (long long)pair * cells);
  const int gx = blk % a.gw, gy = blk / a.gw;
  const long long cell = (long long)pair * cells + blk;
  const int b = a.b;
  const int ox = gx * b, oy = gy * b;
  int sx = 0, sy = 0;
  if (a.level > 0) {
    const int pgw = a.gw / 2, pgh = a.gh / 2;
    const long long pcell = (long long)pair * pgw * pgh + (gy / 2) * pgw + (gx / 2);
    if (a.parent_matched[pcell]) {  // inherited (fme.py:352-362)
      if (lane == 0) {
        a.mv[2 * cell] = a.parent_mv[2 * pcell];
        a.mv[2 * cell + 1] = a.parent_mv[2 * pcell + 1];
        a.energy[cell] = a.parent_e[pcell];
        a.matched[cell] = 1;
      }
      return;
    }
    sx = a.parent_mv[2 * pcell];
    sy = a.parent_mv[2 * pcell + 1];
  }
  const Elem* cur = reinterpret_cast<const Elem*>(a.planes) + (long long)a.cur_index[pair] * p.frame_stride;
  const Elem* ref = reinterpret_cast<const Elem*>(a.ref_planes) + (long long)a.ref_index[pair] * p.frame_stride;
  // current block -> shared memory (word rows; ox is a multiple of b >= 8, so rows are word aligned)
  const int wpr = b / EPW;
  for (int t = lane; t < p.planes * b * wpr; t += 32) {
    const int w = t % wpr, y = (t / wpr) % b, pl = t / (wpr * b);
    cur_s[warp][t] = __ldg(reinterpret_cast<const uint32_t*>(cur + (long long)pl * p.plane_stride +
                                                             (long long)(oy + y) * p.pitch + ox) + w);
  }
  __syncwarp();
  unsigned long long evals = 0;
  int mx = sx, my = sy;
  double e = 0.0;
  bool searched = false;
  for (int st = 0; st < 3; ++st) {
    const int r = p.stage_range[st], s = p.stage_step[st];
    if (r == 0 && searched) {  // same window, same energy (fme.py:306-315)
      evals += 1;
      continue;
    }
    SmallStage res = small_stage<Elem>(cur, ref, cur_s[warp], a, ox, oy, mx, my, r, s, tab);
    if (!res.nvalid) res = small_stage<Elem>(cur, ref, cur_s[warp], a, ox, oy, 0, 0, r, s, tab);  // fme.py:310-313
    evals += res.nvalid;
    mx = res.dx;
    my = res.dy;
    e = res.energy;
    searched = true;
  }
  if (lane == 0) {
    a.mv[2 * cell] = mx;
    a.mv[2 * cell + 1] = my;
    a.energy[cell] = e;
    bool m;
    if (a.final_level) {
      const bool in_real = oy < p.real_h && ox < p.real_w;  // fme.py:377-384
      m = !(e > p.refine_block_threshold && in_real);
    } else {
      m = e <= p.split_threshold;  // fme.py:386
    }
    a.matched[cell] = m ? 1 : 0;
    atomicAdd(a.evals + pair, evals);
  }
}

}  // namespace

bool small_level_ok(const bmc_fme_params& p, int b) {
  static const bool off = [] {
    const char* e = knob_env("BMC_NO_SMALL");
    return e && *e && *e != '0';
  }();
  if (off) return false;
  if (p.planes * b * b > 256 || b < 8) return false;
  const int wpr = b * p.elem_bytes / 4;  // words per block row: the kernel is instantiated for 2 and 4
  if (wpr != 2 && wpr != 4) return false;
  for (int k = 0; k < 3; ++k)
    if (2 * p.stage_range[k] + 1 > 17) return false;  // per-lane candidate slots (10 rounds of 32)
  return true;
}

int launch_fme_small(const StageLaunch& a, cudaStream_t st) {
  const long long blocks = (long long)a.gw * a.gh * a.n_pairs;
  const long long grid = (blocks + kSmallWarps - 1) / kSmallWarps;
  if (a.prm.elem_bytes == 1)
    fme_small_kernel<uint8_t><<<(unsigned)grid, kSmallWarps * 32, 0, st>>>(a);
  else
    fme_small_kernel<uint16_t><<<(unsigned)grid, kSmallWarps * 32, 0, st>>>(a);
  return cuda_status(cudaGetLastError(), "fme_small_kernel");
}

}  // namespace bmc
