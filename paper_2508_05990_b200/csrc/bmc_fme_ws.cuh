// Warp-specialized persistent search-stage kernel (sm_100a).
//
// The stage kernel of bmc_fme_impl.cuh runs staging -> screening -> selection
// as one CTA-wide sequence per block, so the TMA round trip and the (mostly
// serial) exact selection leave the ALU pipe idle unless other resident CTAs
// happen to be screening.  Here a persistent CTA splits the work by warp:
//
//   warps 0..NS-1  screening: wait `full[slot]`, run the integer SAD items of
//                  the block staged in that slot, arrive on `done[slot]`.
//   warp NS        control: takes (pair, block) work items from a global
//                  counter (dynamic load balance), issues the TMA loads of the
//                  next block into a free slot, and -- while the screening
//                  warps work on the other slot -- runs the exact selection of
//                  the finished block and writes its outputs.
//
// Two slots (window + current block + partial sums) form a double buffer, so
// staging, screening and selection of consecutive blocks overlap.  Selection
// follows select_block exactly (same bounds, same replays, same first-minimum
// rule), restated warp-locally without CTA barriers.
#pragma once

#include "bmc_fme_impl.cuh"

namespace bmc {

constexpr int kWsMaxThreads = 288;  // NS <= 7 screening warps + producer warp + selector warp
constexpr int kWsScreenMax = kWsMaxThreads - 64;

struct WsSlotInfo {
  int valid, pair, gx, gy, cx, cy;
  long long cell;
};

__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Wait with a suspend-time hint so a waiting warp yields its issue slots to
// the screening warps instead of spinning.
__device__ __forceinline__ void mbar_wait_sleep(unsigned long long* bar, uint32_t phase) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAITS_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
      "@!p bra WAITS_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(phase), "r"(1000000u)
      : "memory");
}

// Warp-local exact selection of one staged block (slot layout L, sums in L.sad).
template <typename Elem>
__device__ StageResult ws_select(const SmemLayout& L, const PairCtx<Elem>& pc, const StagePlan& pl,
                                 const StageGeom& g, int ox, int oy, int b, int coff_e, int* klist) {
  const int lane = threadIdx.x & 31;
  const int r = g.r, s = g.s, cx = g.cx, cy = g.cy;
  const int G = g.G, N = G * G;
  const int n = pc.P * b * b;
  const int ilo = max(0, r - floor_div(ox + cx, s)), ihi = min(G - 1, r + floor_div(pc.frame_w - b - ox - cx, s));
  const int jlo = max(0, r - floor_div(oy + cy, s)), jhi = min(G - 1, r + floor_div(pc.frame_h - b - oy - cy, s));
  const int wi = ihi - ilo + 1, wj = jhi - jlo + 1;
  StageResult res;
  res.nvalid = (wi > 0 && wj > 0) ? wi * wj : 0;
  res.dx = res.dy = 0;
  res.energy = 0.0;
  if (!res.nvalid) return res;
  const FastDiv fwi(wi);
  unsigned long long best = ~0ull;
  for (int v = lane; v < res.nvalid; v += 32) {
    const int jv = fwi.div(v);
    const int k = (jlo + jv) * G + ilo + (v - jv * wi);
    uint32_t sk = L.sad[k];
    for (int q = 1; q < pl.parts; ++q) sk += L.sad[q * N + k];
    if (pl.parts > 1) L.sad[k] = sk;
    const unsigned long long key = ((unsigned long long)sk << 32) | (unsigned)k;
    best = key < best ? key : best;
  }
  for (int m = 16; m; m >>= 1) {
    const unsigned long long o = __shfl_xor_sync(0xffffffffu, best, m);
    best = o < best ? o : best;
  }
  __syncwarp();
  const int m0 = (int)(best & 0xffffffffu);
  const unsigned sad0 = (unsigned)(best >> 32);
  int wk = m0;
  double we = 0.0;
  if (!(sad0 == 0 && pc.oml > 0.0)) {  // S == 0 => E == 0.0 exactly, first such candidate wins
    int dx, dy;
    cand_valid_ij(g, ox, oy, b, pc.frame_h, pc.frame_w, m0 % G, m0 / G, dx, dy);
    we = sad0 ? exact_cand<Elem>(L, pl, g, pc, ox, oy, b, coff_e, m0 % G, m0 / G, dx, dy) : 0.0;
    const double unit = (double)pc.max_value * (double)n;
    const double lim = we + kScreenEps;
    unsigned thr = 0xffffffffu;
    if (pc.oml > 0.0) {
      double est = floor(lim / pc.oml * unit) + 2.0;
      long long t = est > 4294967295.0 ? 4294967295LL : (long long)est;
      while (t >= 0 && __dmul_rn(pc.oml, __ddiv_rn((double)t, unit)) > lim) --t;
      thr = t < 0 ? 0u : (unsigned)t;
    }
    // SAD contenders, compacted with ballots into the control warp's list
    int nk = 0;
    for (int v0 = 0; v0 < res.nvalid; v0 += 32) {
      const int v = v0 + lane;
      int k = -1;
      if (v < res.nvalid) {
        const int jv = fwi.div(v);
        k = (jlo + jv) * G + ilo + (v - jv * wi);
        if (k == m0 || L.sad[k] > thr) k = -1;
      }
      const unsigned m = __ballot_sync(0xffffffffu, k >= 0);
      if (k >= 0) klist[nk + __popc(m & ((1u << lane) - 1))] = k;
      nk += __popc(m);
    }
    __syncwarp();
    const int D = (int)floor(pc.tol * (double)pc.max_value + 1e-9) + 1;
    const bool tighten = nk > 1 && pc.lam > 0.0;
    for (int e = 0; e < nk; ++e) {
      const int k = klist[e];
      if (tighten) {
        // sparsity-tightened bound E >= (1-lam)*S/(s*n) + lam*C_lo/n before paying for the float64 replay
        const int clo = count_lo<Elem>(L, pl, g, pc, ox, oy, b, coff_e, k % G, k / G, D);
        const double elb = __dadd_rn(__dmul_rn(pc.oml, __ddiv_rn((double)L.sad[k], unit)),
                                     __dmul_rn(pc.lam, __ddiv_rn((double)clo, (double)n)));
        if (elb - kScreenEps > we + kScreenEps) continue;
      }
      int dx, dy;
      cand_valid_ij(g, ox, oy, b, pc.frame_h, pc.frame_w, k % G, k / G, dx, dy);
      const double ek = exact_cand<Elem>(L, pl, g, pc, ox, oy, b, coff_e, k % G, k / G, dx, dy);
      if (ek < we || (ek == we && k < wk)) {
        we = ek;
        wk = k;
      }
    }
  }
  cand_valid_ij(g, ox, oy, b, pc.frame_h, pc.frame_w, wk % G, wk / G, res.dx, res.dy);
  res.energy = we;
  return res;
}

template <typename Elem, int CW, int TY, bool SHIFT>
__global__ void __launch_bounds__(kWsMaxThreads, 3)
    fme_ws_kernel(const __grid_constant__ CUtensorMap tm_win, const __grid_constant__ CUtensorMap tm_cur,
                  const StageLaunch a, unsigned* work_ctr) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const StagePlan& pl = a.plan;
  const bmc_fme_params& p = a.prm;
  const int b = a.b;
  const int ns = pl.threads / 32;  // screening warps
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  SmemLayout L[2];
  L[0] = carve(smem_raw, pl);
  L[1] = L[0];
  L[1].sad = reinterpret_cast<uint32_t*>(smem_raw + pl.off_sad + pl.slot_bytes);
  L[1].cur = reinterpret_cast<uint32_t*>(smem_raw + pl.off_cur + pl.slot_bytes);
  L[1].win = reinterpret_cast<uint32_t*>(smem_raw + pl.off_win + pl.slot_bytes);
  unsigned long long* full = L[0].bar + 1;  // [2] window staged (TMA tx) / end marker
  unsigned long long* done = full + 2;      // [2] screening finished (NS arrivals)
  unsigned long long* freed = done + 2;     // [2] selection finished, slot reusable
  WsSlotInfo* info = reinterpret_cast<WsSlotInfo*>(freed + 2);  // [2]
  const uint32_t cells = (uint32_t)a.gw * a.gh;
  const uint32_t total = cells * (uint32_t)a.n_pairs;
  if (threadIdx.x == 0) {
    for (int sl = 0; sl < 2; ++sl) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(full + sl)), "r"(1));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(done + sl)), "r"(ns));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(freed + sl)), "r"(1));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (sizeof(Elem) == 1)
    for (int v = threadIdx.x; v < 256; v += blockDim.x) L[0].tab[v] = __ddiv_rn((double)v, (double)p.max_value);
  __syncthreads();
  constexpr int A16 = 16 / (int)sizeof(Elem);
  auto geom = [&](const WsSlotInfo& in, int& ox, int& oy, int& cx0, int& coff_e) {
    StageGeom g;
    g.r = a.r;
    g.s = a.s;
    g.G = 2 * a.r + 1;
    g.ncg = (g.G + TY - 1) / TY;
    g.cx = in.cx;
    g.cy = in.cy;
    ox = in.gx * b;
    oy = in.gy * b;
    g.wx0 = ox + in.cx - a.r * a.s;
    g.wy0 = oy + in.cy - a.r * a.s;
    g.tx0 = g.wx0 - (((g.wx0 % A16) + A16) % A16);
    g.d = g.wx0 - g.tx0;
    cx0 = ox - (ox % A16);
    coff_e = ox - cx0;
    return g;
  };
  auto frame_ctx = [&](int pair) {
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
    pc.tab = sizeof(Elem) == 1 ? L[0].tab : a.tab16;
    return pc;
  };

  if (warp == ns) {
    // ------------------------------------------------------------ producer warp
    // Takes the next non-inherited work item and starts its TMA loads into the
    // slot the selector has released (the first two fills pass at parity 1).
    uint32_t free_phase[2] = {1, 1};
    for (int sl = 0;; sl ^= 1) {
      mbar_wait_sleep(freed + sl, free_phase[sl]);
      free_phase[sl] ^= 1;
      int valid = 0;
      if (lane == 0) {
        WsSlotInfo in;
        in.valid = 0;
        for (;;) {
          const uint32_t w = atomicAdd(work_ctr, 1u);
          if (w >= total) break;
          in.pair = (int)(w / cells);
          const int blk = (int)(w - (uint32_t)in.pair * cells);
          in.gx = blk % a.gw;
          in.gy = blk / a.gw;
          in.cell = (long long)in.pair * cells + blk;
          in.cx = in.cy = 0;
          if (a.level > 0) {
            const int pgw = a.gw / 2, pgh = a.gh / 2;
            const long long pcell = (long long)in.pair * pgw * pgh + (in.gy / 2) * pgw + (in.gx / 2);
            if (a.parent_matched[pcell]) {  // inherited: copy the parent (fme.py:352-362), no search
              if (a.first) {
                a.mv[2 * in.cell] = a.parent_mv[2 * pcell];
                a.mv[2 * in.cell + 1] = a.parent_mv[2 * pcell + 1];
                a.energy[in.cell] = a.parent_e[pcell];
                a.matched[in.cell] = 1;
              }
              continue;
            }
            if (a.first) {
              in.cx = a.parent_mv[2 * pcell];
              in.cy = a.parent_mv[2 * pcell + 1];
            }
          }
          if (!a.first) {
            in.cx = a.mv[2 * in.cell];
            in.cy = a.mv[2 * in.cell + 1];
          }
          in.valid = 1;
          break;
        }
        info[sl] = in;
        valid = in.valid;
        if (in.valid) {
          int ox, oy, cx0, coff_e;
          const StageGeom g = geom(in, ox, oy, cx0, coff_e);
          const int cur_f = a.cur_index[in.pair], ref_f = a.ref_index[in.pair];
          mbar_expect_tx(full + sl, (uint32_t)pl.tma_bytes);
          tma_load_3d(L[sl].win, &tm_win, g.tx0, g.wy0, ref_f * p.planes, full + sl);
          tma_load_3d(L[sl].cur, &tm_cur, cx0, oy, cur_f * p.planes, full + sl);
        } else {
          mbar_arrive(full + sl);
        }
      }
      valid = __shfl_sync(0xffffffffu, valid, 0);
      if (!valid) return;
    }
  }
  if (warp == ns + 1) {
    // ------------------------------------------------------------ selector warp
    uint32_t full_phase[2] = {0, 0}, done_phase[2] = {0, 0};
    for (int sl = 0;; sl ^= 1) {
      mbar_wait_sleep(full + sl, full_phase[sl]);
      full_phase[sl] ^= 1;
      const WsSlotInfo in = info[sl];
      if (!in.valid) return;
      mbar_wait_sleep(done + sl, done_phase[sl]);
      done_phase[sl] ^= 1;
      int ox, oy, cx0, coff_e;
      const StageGeom g = geom(in, ox, oy, cx0, coff_e);
      const PairCtx<Elem> pc = frame_ctx(in.pair);
      StageResult res = ws_select<Elem>(L[sl], pc, pl, g, ox, oy, b, coff_e, L[0].klist);
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(freed + sl);  // window and sums of this slot are no longer read
        a.mv[2 * in.cell] = res.dx;
        a.mv[2 * in.cell + 1] = res.dy;
        a.energy[in.cell] = res.energy;
        if (a.last) {
          bool m;
          if (a.final_level) {
            const bool in_real = oy < p.real_h && ox < p.real_w;  // fme.py:377-384
            m = !(res.energy > p.refine_block_threshold && in_real);
          } else {
            m = res.energy <= p.split_threshold;  // fme.py:386
          }
          a.matched[in.cell] = m ? 1 : 0;
        }
        atomicAdd(a.evals + in.pair, (unsigned long long)(res.nvalid + a.extra_evals));
      }
    }
  }
  // -------------------------------------------------------------- screening warps
  uint32_t full_phase[2] = {0, 0};
  for (int sl = 0;; sl ^= 1) {
    mbar_wait_sleep(full + sl, full_phase[sl]);
    full_phase[sl] ^= 1;
    const WsSlotInfo in = info[sl];
    if (!in.valid) break;
    int ox, oy, cx0, coff_e;
    const StageGeom g = geom(in, ox, oy, cx0, coff_e);
    sad_items<Elem, CW, TY, SHIFT>(L[sl], g, b, p.planes, pl, (ox - cx0) * (int)sizeof(Elem) / 4, false, 1,
                                   threadIdx.x, ns * 32);
    __syncwarp();
    if (lane == 0) mbar_arrive(done + sl);
  }
}

template <typename E, int CW, int TY, bool SH>
inline int launch_ws_one(const CUtensorMap& tw, const CUtensorMap& tc, const StageLaunch& a, cudaStream_t st) {
  int rc = set_smem(fme_ws_kernel<E, CW, TY, SH>, a.plan.smem);
  if (rc) return rc;
  static std::mutex mu;
  static const void* keys[64];
  static int smems[64], vals[64];
  static int nk = 0;
  int per_sm = 0;
  {
    std::lock_guard<std::mutex> g(mu);
    const void* key = reinterpret_cast<const void*>(fme_ws_kernel<E, CW, TY, SH>);
    for (int i = 0; i < nk; ++i)
      if (keys[i] == key && smems[i] == a.plan.smem) per_sm = vals[i];
    if (!per_sm) {
      cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fme_ws_kernel<E, CW, TY, SH>,
                                                                    a.plan.threads + 64, a.plan.smem);
      if (e != cudaSuccess) return cuda_status(e, "cudaOccupancyMaxActiveBlocksPerMultiprocessor(ws)");
      if (per_sm < 1) per_sm = 1;
      if (nk < 64) {
        keys[nk] = key;
        smems[nk] = a.plan.smem;
        vals[nk] = per_sm;
        ++nk;
      }
    }
  }
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms < 1) sms = 1;
  }
  unsigned* ctr = ws_work_counter(st);
  if (!ctr) return -1;  // no counter available (first use inside a capture): caller falls back
  const long long work = (long long)a.gw * a.gh * a.n_pairs;
  const long long cap = (long long)per_sm * sms;
  const unsigned nblk = (unsigned)(work < cap ? work : cap);
  fme_ws_kernel<E, CW, TY, SH><<<nblk, a.plan.threads + 64, a.plan.smem, st>>>(tw, tc, a, ctr);
  return cuda_status(cudaGetLastError(), "fme_ws_kernel");
}

template <typename E, int CW, bool SH>
inline int dispatch_ws(const CUtensorMap& tw, const CUtensorMap& tc, const StageLaunch& a, cudaStream_t st) {
  switch (a.plan.ty) {
    case 1: return launch_ws_one<E, CW, 1, SH>(tw, tc, a, st);
    case 2: return launch_ws_one<E, CW, 2, SH>(tw, tc, a, st);
    case 3: return launch_ws_one<E, CW, 3, SH>(tw, tc, a, st);
    case 4: return launch_ws_one<E, CW, 4, SH>(tw, tc, a, st);
    case 5: return launch_ws_one<E, CW, 5, SH>(tw, tc, a, st);
    case 6: return launch_ws_one<E, CW, 6, SH>(tw, tc, a, st);
    case 7: return launch_ws_one<E, CW, 7, SH>(tw, tc, a, st);
    case 8: return launch_ws_one<E, CW, 8, SH>(tw, tc, a, st);
    case 9: return launch_ws_one<E, CW, 9, SH>(tw, tc, a, st);
    case 10: return launch_ws_one<E, CW, 10, SH>(tw, tc, a, st);
    case 11: return launch_ws_one<E, CW, 11, SH>(tw, tc, a, st);
    default: return launch_ws_one<E, CW, 12, SH>(tw, tc, a, st);
  }
}

}  // namespace bmc
