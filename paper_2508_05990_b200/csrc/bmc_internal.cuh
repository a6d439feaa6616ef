// Internal device helpers shared by the B200 kernels (sm_100a only).
//
// The reference computes energies in float64 on intensities normalised by the
// dtype maximum and sums |a-b| with numpy's pairwise summation
// (fme.py:229-233, :258-265; numpy loops_utils.h.src).  The integer SIMD search
// screens candidates; these helpers replay the exact float64 arithmetic for the
// few that can still win, in the same association order, with explicitly
// rounded operations (no FMA contraction) so results are bit-identical.
#pragma once

#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

#include "../../include/bmc.h"

namespace bmc {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;

// ---------------------------------------------------------------------------
// measurement knobs: environment switches read ONLY by experiment builds
// (tools/build_variants.sh compiles with -DBMC_EXPERIMENTS); the product
// library ignores the environment, so no variable can change its results.
// ---------------------------------------------------------------------------
inline const char* knob_env(const char* name) {
#ifdef BMC_EXPERIMENTS
  return getenv(name);
#else
  (void)name;
  return nullptr;
#endif
}

// ---------------------------------------------------------------------------
// error plumbing
// ---------------------------------------------------------------------------
void set_error(const char* fmt, ...);
int cuda_status(cudaError_t e, const char* where);

// ---------------------------------------------------------------------------
// packed-integer SAD words
// ---------------------------------------------------------------------------

// uint8: one VABSDIFF4.U8.ACC = 4 samples.
__device__ __forceinline__ uint32_t sad_word(uint32_t a, uint32_t b, uint32_t acc, uint8_t) {
  uint32_t d;
  asm("vabsdiff4.u32.u32.u32.add %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(acc));
  return d;
}

// uint16: |a-b| per 16-bit lane = max - min (VIMNMX.U16x2 x2, no cross-lane
// borrow because max >= min per lane), then IDP.2A sums both lanes into acc.
__device__ __forceinline__ uint32_t sad_word(uint32_t a, uint32_t b, uint32_t acc, uint16_t) {
  uint32_t mx, mn;
  asm("max.u16x2 %0, %1, %2;" : "=r"(mx) : "r"(a), "r"(b));
  asm("min.u16x2 %0, %1, %2;" : "=r"(mn) : "r"(a), "r"(b));
  return __dp2a_lo(mx - mn, 0x0101u, acc);
}

// ---------------------------------------------------------------------------
// exact float64 replay
// ---------------------------------------------------------------------------

// Normalised sample fl(v / s): table lookup (u8: 256 entries in smem; u16:
// 65536 entries in global memory, built once by bmc_norm_table()).
const double* norm_table_u16(int device);

template <typename Elem>
__device__ __forceinline__ double norm_sample(Elem v, const double* tab) {
  return tab[v];
}

// numpy's combine of the eight leaf accumulators.
__device__ __forceinline__ double leaf_combine8(const double r[8]) {
  return __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                   __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
}

__device__ __forceinline__ double shfl_xor_d(double v, int m) {
  return __shfl_xor_sync(0xffffffffu, v, m);
}

struct ExactResult {
  double energy;
  double sad;
  int count;
};

// Warp-cooperative exact energy of one candidate for power-of-two sample counts
// n = P*b*b >= 64 (every block size FmeConfig admits).  numpy's pairwise sum is
// then a perfect binary tree of min(n,128)-element leaves; each leaf runs eight
// strided accumulators (chains) for leaf/8 rounds.  Lane l owns chains
// l, l+32, ...; chains of one leaf sit in eight consecutive lanes, so xor
// butterflies 1,2,4 reproduce ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) and 8,16 the
// first two tree levels above the leaves (IEEE addition is commutative, so
// a+b == b+a bit for bit).  Remaining levels combine per-lane partials with a
// binary-carry stack, which is the same perfect tree.
//
// cur/ref: element (0,0) of plane 0 of the block / candidate window, with their
// own row pitch and plane stride (global planes or staged shared-memory tiles).
// Partial form: the perfect subtree over chain groups q in [q0, q1) (32 chains,
// i.e. 4 leaves, per q; q1 - q0 a power of two, q0 a multiple of it), plus the
// sparsity count of those elements.  Every lane returns the sum (the count is
// warp-reduced).  q0 = 0, q1 = nq is the whole tree.
template <typename Elem>
__device__ void exact_partial(const Elem* cur, int cpitch, long long cplane, const Elem* ref, int rpitch,
                              long long rplane, int b, int P, const double* tab, double tol, int q0, int q1,
                              double& total_out, int& cnt_out) {
  const int lane = threadIdx.x & 31;
  const int lb = __ffs(b) - 1;
  const int n = P << (2 * lb);
  const int leaf = n < 128 ? n : 128;
  const int rounds = leaf >> 3;
  const int chains = (n / leaf) * 8;
  int cnt = 0;
  double stack[16];  // carry depth log2(n/4096): 16 covers any n < 2^28
  double total = 0.0;
  for (int q = q0; q < q1; ++q) {
    const int c = lane + 32 * q;
    double r = 0.0;
    if (c < chains) {
      const int base = (c >> 3) * leaf + (c & 7);
      for (int t = 0; t < rounds; ++t) {
        const int e = base + 8 * t;
        const int p = e >> (2 * lb);
        const int y = (e >> lb) & (b - 1);
        const int x = e & (b - 1);
        const double cv = norm_sample(cur[p * cplane + (long long)y * cpitch + x], tab);
        const double rv = norm_sample(ref[p * rplane + (long long)y * rpitch + x], tab);
        const double dv = fabs(__dsub_rn(rv, cv));
        cnt += dv > tol;
        r = (t == 0) ? dv : __dadd_rn(r, dv);
      }
    }
    // leaf combine, then up to two tree levels across leaves held by this warp.
    r = __dadd_rn(r, shfl_xor_d(r, 1));
    r = __dadd_rn(r, shfl_xor_d(r, 2));
    r = __dadd_rn(r, shfl_xor_d(r, 4));
    if (chains > 8) r = __dadd_rn(r, shfl_xor_d(r, 8));
    if (chains > 16) r = __dadd_rn(r, shfl_xor_d(r, 16));
    if (q1 - q0 == 1) {
      total = r;
    } else {
      int k = q - q0, lvl = 0;
      while (k & 1) {
        r = __dadd_rn(stack[lvl], r);
        k >>= 1;
        ++lvl;
      }
      stack[lvl] = r;
      if (q == q1 - 1) total = r;
    }
  }
  for (int m = 16; m; m >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, m);
  total_out = __shfl_sync(0xffffffffu, total, 0);  // lanes past `chains` hold partial garbage
  cnt_out = cnt;
}

__device__ __forceinline__ ExactResult exact_finish(double total, int cnt, int n, double oml, double lam) {
  const double s_f = __dadd_rn(0.0, total);
  const double nd = (double)n;
  ExactResult res;
  res.sad = s_f;
  res.count = cnt;
  res.energy = __dadd_rn(__dmul_rn(oml, __ddiv_rn(s_f, nd)), __dmul_rn(lam, __ddiv_rn((double)cnt, nd)));
  return res;
}

template <typename Elem>
__device__ ExactResult exact_energy_generic(const Elem* cur, int cpitch, long long cplane, const Elem* ref, int rpitch,
                                            long long rplane, int b, int P, const double* tab, double tol, double oml,
                                            double lam) {
  const int lb = __ffs(b) - 1;
  const int n = P << (2 * lb);
  const int leaf = n < 128 ? n : 128;
  const int chains = (n / leaf) * 8;
  const int nq = chains > 32 ? chains / 32 : 1;
  double total;
  int cnt;
  exact_partial<Elem>(cur, cpitch, cplane, ref, rpitch, rplane, b, P, tab, tol, 0, nq, total, cnt);
  return exact_finish(total, cnt, n, oml, lam);
}

// Global-memory form: both operands in the same plane layout.
template <typename Elem>
__device__ ExactResult exact_energy_warp(const Elem* __restrict__ cur, const Elem* __restrict__ ref, int pitch,
                                         long long plane_stride, int b, int P, const double* tab, double tol,
                                         double oml, double lam) {
  return exact_energy_generic<Elem>(cur, pitch, plane_stride, ref, pitch, plane_stride, b, P, tab, tol, oml, lam);
}

// ---------------------------------------------------------------------------
// generic numpy pairwise sum (any n).  numpy splits n > 128 into
// n2 = n/2 - (n/2)%8 and n - n2 recursively; leaves (n <= 128) use eight
// strided accumulators (n >= 8) or a plain sequential sum from 0.0 (n < 8).
// ---------------------------------------------------------------------------

// numpy leaf semantics for len <= 128.
template <typename F>
__device__ double pairwise_leaf(F value, long long lo, int len) {
  if (len < 8) {
    double res = 0.0;
    for (int i = 0; i < len; ++i) res = __dadd_rn(res, value(lo + i));
    return res;
  }
  double r[8];
  for (int j = 0; j < 8; ++j) r[j] = value(lo + j);
  int i = 8;
  const int stop = len - (len % 8);
  for (; i < stop; i += 8)
    for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], value(lo + i + j));
  double res = leaf_combine8(r);
  for (; i < len; ++i) res = __dadd_rn(res, value(lo + i));
  return res;
}

// Walk numpy's split tree over [lo, lo+n) left to right; `leaf(lo, len)` gives
// each leaf's value, internal nodes add left + right.  Iterative (explicit
// stack) so it is cheap on device.
template <typename Leaf>
__device__ double pairwise_tree(Leaf leaf, long long lo, long long n) {
  struct Node { long long lo, n; int state; double left; };
  Node st[64];
  int sp = 0;
  st[0] = {lo, n, 0, 0.0};
  double ret = 0.0;
  for (;;) {
    Node& f = st[sp];
    if (f.state == 0 && f.n <= 128) {
      ret = leaf(f.lo, (int)f.n);
    } else if (f.state == 0) {
      long long n2 = f.n / 2;
      n2 -= n2 % 8;
      f.state = 1;
      st[sp + 1] = {f.lo, n2, 0, 0.0};
      ++sp;
      continue;
    } else if (f.state == 1) {
      long long n2 = f.n / 2;
      n2 -= n2 % 8;
      f.left = ret;
      f.state = 2;
      st[sp + 1] = {f.lo + n2, f.n - n2, 0, 0.0};
      ++sp;
      continue;
    } else {
      ret = __dadd_rn(f.left, ret);
    }
    if (sp == 0) break;
    --sp;
  }
  return ret;
}

// Number of leaves numpy's tree has for n elements (host only: recursion on
// device would need an unbounded stack).
inline long long pairwise_leaf_count(long long n) {
  if (n <= 128) return 1;
  long long n2 = n / 2;
  n2 -= n2 % 8;
  return pairwise_leaf_count(n2) + pairwise_leaf_count(n - n2);
}

// CTA-cooperative pairwise sum (result identical to the sequential tree):
// leaves are summed in parallel, thread 0 combines them in tree order.
// All threads must call; scratch holds >= pairwise_leaf_count(n) entries.
template <typename F>
__device__ double block_pairwise(F value, long long n, long long* leaf_lo, int* leaf_len, double* leaf_val,
                                 double* result_slot) {
  __syncthreads();
  if (threadIdx.x == 0) {
    int cnt = 0;
    pairwise_tree([&](long long lo, int len) { leaf_lo[cnt] = lo; leaf_len[cnt] = len; ++cnt; return 0.0; },
                  0, n);
    leaf_len[-1] = cnt;  // slot just before the array holds the count
  }
  __syncthreads();
  const int cnt = leaf_len[-1];
  for (int l = threadIdx.x; l < cnt; l += blockDim.x) leaf_val[l] = pairwise_leaf(value, leaf_lo[l], leaf_len[l]);
  __syncthreads();
  if (threadIdx.x == 0) {
    int k = 0;
    const double r = pairwise_tree([&](long long, int) { return leaf_val[k++]; }, 0, n);
    *result_slot = __dadd_rn(0.0, r);
  }
  __syncthreads();
  return *result_slot;
}

}  // namespace bmc
