// CaBR-Net on device: the context-aware block refinement network of the
// reference (cabr.py:60-90 extract_patch, :206-250 _conv2d/_encode/cabr_forward,
// :306-345 refine_blocks with weights) for every flagged block, fused into one
// kernel per frame.
//
// Network (cabr.py:28-32, :97-119) for block size K, patch side S = 2K+1:
//   image  (1,S,S)  -> conv3x3 s2 16 -> conv3x3 s2 32 -> conv3x3 s1 32  (relu each)
//   context(C,S,S)  -> conv3x3 s2 16 -> conv3x3 s2 32 -> conv3x3 s1 32  (relu each)
//   concat (64, K/2+1, K/2+1) -> conv3x3 32 relu -> nearest x4 -> conv3x3 32 relu
//   -> conv1x1 C -> logits cropped to the central K x K.
//
// Only the cropped logits are needed, so every layer is evaluated on the
// receptive field of the output only (`regions` below): for K = 32 the
// decoder's 3x3 conv runs on 32x32 instead of 68x68 pixels and the encoders on
// about 70% of their maps.  A CTA owns one (flagged block, TS x TS output tile)
// item (TS = min(K, 32), so shared memory stays bounded for any K); all
// activations of the item stay in shared memory, each layer's weights are
// staged into shared memory by cp.async while the previous layer computes
// (double-buffered; warp-uniform float4 broadcasts in the inner loop), and the arithmetic is plain fp32 FFMA: the reference computes
// in float32 and its tolerance (1e-5 relative) rules out TF32 tensor cores.
//
// The context input is the one-hot map of the predicted labels with the central
// 16x16 zeroed (cabr.py:84-89); instead of materialising C channels the first
// context conv looks up W[class][tap][:] per tap (a sum of <= 9 weight rows).
// Explicit (image, context) patches (the cabr_forward(CabrPatch) API) take the
// general C-channel conv instead.
//
// Float results are not bit-identical to the reference's numpy einsum
// (different association order); tests hold logits to a stated fp32 tolerance
// and labels to exact equality away from near-ties.
#include <algorithm>
#include <cstdint>
#include <cstring>

#include "../../include/bmc_ext.h"
#include "bmc_internal.cuh"

namespace bmc {
namespace {

constexpr int kCtxMask = 16;  // CONTEXT_MASK (cabr.py:27)
constexpr int kNumLayers = 9;  // img0 img1 img2 ctx0 ctx1 ctx2 dec0 dec1 head
constexpr int kMaxTile = 32;

struct WOff {
  long long w[kNumLayers], b[kNumLayers];
  int cin[kNumLayers], cout[kNumLayers], taps[kNumLayers];
  long long total;
};

// weight_spec order (cabr.py:97-119); conv weights are stored transposed
// (cin, tap, cout) so a thread's output channels are contiguous, the head as
// given (C, 32), biases follow their weights.
__host__ __device__ inline WOff cabr_offsets(int C) {
  WOff o{};
  const int cin[kNumLayers] = {1, 16, 32, C, 16, 32, 64, 32, 32};
  const int cout[kNumLayers] = {16, 32, 32, 16, 32, 32, 32, 32, C};
  long long off = 0;
  for (int l = 0; l < kNumLayers; ++l) {
    o.cin[l] = cin[l];
    o.cout[l] = cout[l];
    o.taps[l] = l == 8 ? 1 : 9;
    o.w[l] = off;
    off += (long long)cin[l] * cout[l] * o.taps[l];
    o.b[l] = off;
    off += cout[l];
  }
  o.total = off;
  return o;
}

// dec.1 over the x4 nearest-upsampled map: output rows u with u % 4 in {1, 2}
// read the same dec.0 row for all three kernel rows, so their three row taps
// collapse into one (W[ky=0] + W[ky=1]) + W[ky=2] -- stored (c, kx, o) after
// the payload, 16-byte aligned.  Rows with u % 4 in {0, 3} straddle two dec.0
// rows and keep the 3x3 weights.
constexpr int kMergedFloats = 32 * 3 * 32;
__host__ __device__ inline long long cabr_merged_offset(const WOff& o) { return (o.total + 3) & ~3ll; }
__host__ __device__ inline long long cabr_packed_floats(const WOff& o) { return cabr_merged_offset(o) + kMergedFloats; }

__global__ void cabr_merge_rows_kernel(float* __restrict__ packed, WOff o) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;  // (c, kx, oc)
  if (i >= kMergedFloats) return;
  const int oc = i % 32, kx = (i / 32) % 3, c = i / 96;
  const float* w = packed + o.w[7];  // dec.1 weights, (cin, tap, cout)
  const float v = __fadd_rn(__fadd_rn(w[(c * 9 + kx) * 32 + oc], w[(c * 9 + 3 + kx) * 32 + oc]),
                            w[(c * 9 + 6 + kx) * 32 + oc]);
  packed[cabr_merged_offset(o) + i] = v;
}

__global__ void cabr_pack_kernel(const float* __restrict__ src, float* __restrict__ dst, WOff o) {
  const long long n = o.total;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    int l = 0;
    while (l + 1 < kNumLayers && i >= o.w[l + 1]) ++l;
    if (i >= o.b[l] || l == 8) {  // biases and the 1x1 head keep their layout
      dst[i] = src[i];
      continue;
    }
    const long long r = i - o.w[l];  // source index (cout, cin, tap)
    const int taps = o.taps[l], ci = o.cin[l], co = o.cout[l];
    const int tap = (int)(r % taps);
    const long long oi = r / taps;
    const int c = (int)(oi % ci), oc = (int)(oi / ci);
    dst[o.w[l] + ((long long)c * taps + tap) * co + oc] = src[i];
  }
}

struct Range {
  int lo, hi;  // [lo, hi)
  __host__ __device__ int n() const { return hi - lo; }
};

struct Regions {
  Range p, e0, e1, e2, d0;
  int l0;  // first logits row/col of the tile in the (2K+4) decoder grid
};

// Receptive field of output rows [t0, t0+ts) of the K x K block in every layer
// (same along columns).  Layer sizes: enc0 K+1, enc1/enc2/dec0 K/2+1, decoder
// 2K+4; the crop starts at K/2+2 (cabr.py:244-249).
__host__ __device__ inline Regions regions(int K, int t0, int ts) {
  Regions r;
  const int nd = K / 2 + 1;
  r.l0 = K / 2 + 2 + t0;
  const int l1 = r.l0 + ts;
  r.d0 = {(r.l0 - 1) >> 2, (l1 >> 2) + 1};  // upsampled rows [l0-1, l1] -> dec0 rows u/4
  r.e2 = {r.d0.lo - 1 > 0 ? r.d0.lo - 1 : 0, r.d0.hi + 1 < nd ? r.d0.hi + 1 : nd};
  r.e1 = {r.e2.lo - 1 > 0 ? r.e2.lo - 1 : 0, r.e2.hi + 1 < nd ? r.e2.hi + 1 : nd};
  const int e0lo = 2 * r.e1.lo - 1, e0hi = 2 * (r.e1.hi - 1) + 2;
  r.e0 = {e0lo > 0 ? e0lo : 0, e0hi < K + 1 ? e0hi : K + 1};
  const int plo = 2 * r.e0.lo - 1, phi = 2 * (r.e0.hi - 1) + 2;
  r.p = {plo > 0 ? plo : 0, phi < 2 * K + 1 ? phi : 2 * K + 1};
  return r;
}

struct CabrGeo {
  int K, ts, tiles, threads;
  int np, ne0, ne1, ne2, nd0;  // max region sides over the tile positions
  int off_p, off_e0, off_e1, off_e2, off_w, off_lab;  // float offsets (off_lab: byte offset)
  int wfloats, wfloats1;
  int smem;
};

struct CabrArgs {
  // pixels: 0 uint8, 1 uint16 (divided by the dtype max, cabr.py:72-73), 2 float32 as-is
  const void* pix;
  int pix_kind;
  long long pix_fs, pix_ss;  // frame / stream strides (elements)
  const uint8_t* labels;
  long long lab_fs, lab_ss;
  int H, W, C;
  const float* wts;  // packed weights (cabr_offsets layout)
  // explicit patches (cabr_forward on a CabrPatch): image (n,1,S,S), context (n,C,S,S)
  const float* img_patch;
  const float* ctx_patch;
  // block list: origins (n,2) of frame 0 / stream 0 ...
  const int32_t* origins;
  int n_blocks;
  // ... or the flagged blocks of frame t (chain mode): ids s*cells + cell, count on device
  const int32_t* flag_list;
  const int32_t* flag_count;
  int t, gw, cells, B;
  // outputs
  float* logits;    // (n, C, K, K) or NULL
  uint8_t* argmax;  // (n, K, K) or NULL
  uint8_t* scratch; // chain mode: (streams, H, W) refined labels at the block positions
  long long scr_ss;
  CabrGeo g;
};

// Asynchronous copy of a layer's weights into shared memory (LDGSTS), one commit
// group; consumed after cp_async_wait_all() + __syncthreads().
__device__ __forceinline__ void stage_weights_async(float* dst, const float* src, int n) {
  const int n4 = n >> 2;
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  for (int i = threadIdx.x; i < n4; i += blockDim.x)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d + 16 * i), "l"(src + 4 * i));
  for (int i = (n4 << 2) + threadIdx.x; i < n; i += blockDim.x)
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(d + 4 * i), "l"(src + i));
  asm volatile("cp.async.commit_group;\n" ::);
}

__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

// out[o][r][c] (region ro x co, plane-major) = relu(bias[o] + sum_{ci, ky, kx}
// w[ci][ky*3+kx][o] * in[ci][r*stride-1+ky][c*stride-1+kx]), `in` zero outside
// [0, n_in)^2 (cabr.py:206-216, pad 1) and stored over region ri x ci_ (plane-major).
// w: this pass's input channels [ci0, ci0+cin) (smem); with `partial` the
// accumulation continues from a previous pass's sums over the earlier channels
// (same order as one pass); `finish` adds the bias and applies relu.
template <int CO, int PX>
__device__ void conv3x3(const float* __restrict__ in, Range ri, Range rc, int n_in, int cin,
                        const float* __restrict__ w, const float* __restrict__ bias, int cout, int stride,
                        float* __restrict__ out, Range ro, Range co, bool partial, bool finish) {
  const int oh = ro.n(), ow = co.n(), npix = oh * ow;
  const int wI = rc.n(), plane = ri.n() * wI;
  const int ngrp = (npix + PX - 1) / PX, nog = cout / CO;
  for (int it = threadIdx.x; it < ngrp * nog; it += blockDim.x) {
    const int og = it / ngrp, pg = it - og * ngrp;  // a warp shares og: weight loads broadcast
    int off[PX];
    unsigned vm[PX];
    float acc[PX][CO];
#pragma unroll
    for (int p = 0; p < PX; ++p) {
      const int pix = pg * PX + p;
      off[p] = 0;
      vm[p] = 0;
      if (pix < npix) {
        const int r = ro.lo + pix / ow, c = co.lo + pix % ow;
        const int ir0 = r * stride - 1, ic0 = c * stride - 1;
        off[p] = (ir0 - ri.lo) * wI + (ic0 - rc.lo);
#pragma unroll
        for (int tap = 0; tap < 9; ++tap) {
          const int ir = ir0 + tap / 3, ic = ic0 + tap % 3;
          if (ir >= 0 && ir < n_in && ic >= 0 && ic < n_in) vm[p] |= 1u << tap;
        }
      }
#pragma unroll
      for (int o = 0; o < CO; ++o)
        acc[p][o] = (partial && pix < npix) ? out[(og * CO + o) * npix + pix] : 0.f;
    }
    for (int c = 0; c < cin; ++c) {
      const float* ip = in + c * plane;
      const float* wp = w + c * 9 * cout + og * CO;
#pragma unroll
      for (int tap = 0; tap < 9; ++tap) {
        float x[PX];
#pragma unroll
        for (int p = 0; p < PX; ++p) x[p] = (vm[p] >> tap) & 1u ? ip[off[p] + (tap / 3) * wI + tap % 3] : 0.f;
#pragma unroll
        for (int j = 0; j < CO / 4; ++j) {
          const float4 wv = *reinterpret_cast<const float4*>(wp + tap * cout + 4 * j);
#pragma unroll
          for (int p = 0; p < PX; ++p) {
            acc[p][4 * j + 0] = fmaf(x[p], wv.x, acc[p][4 * j + 0]);
            acc[p][4 * j + 1] = fmaf(x[p], wv.y, acc[p][4 * j + 1]);
            acc[p][4 * j + 2] = fmaf(x[p], wv.z, acc[p][4 * j + 2]);
            acc[p][4 * j + 3] = fmaf(x[p], wv.w, acc[p][4 * j + 3]);
          }
        }
      }
    }
#pragma unroll
    for (int p = 0; p < PX; ++p) {
      const int pix = pg * PX + p;
      if (pix >= npix) continue;
#pragma unroll
      for (int o = 0; o < CO; ++o) {
        float v = acc[p][o];
        if (finish) v = fmaxf(v + bias[og * CO + o], 0.f);
        out[(og * CO + o) * npix + pix] = v;
      }
    }
  }
}

// First context conv on the masked one-hot map (cabr.py:84-89 + :206-216):
// out[o] = relu(b[o] + sum over in-patch, unmasked taps of T[class][tap][o]).
// lab: class bytes over the patch region rp x cp (patch coordinates).
__device__ void ctx_conv0_onehot(const uint8_t* __restrict__ lab, Range rp, Range cp, int S, int K, int C,
                                 const float* __restrict__ table, const float* __restrict__ bias,
                                 float* __restrict__ out, Range ro, Range co) {
  const int oh = ro.n(), ow = co.n(), npix = oh * ow, wP = cp.n();
  const int mlo = K - kCtxMask / 2, mhi = mlo + kCtxMask;
  for (int pix = threadIdx.x; pix < npix; pix += blockDim.x) {
    const int r = ro.lo + pix / ow, c = co.lo + pix % ow;
    float acc[16];
#pragma unroll
    for (int o = 0; o < 16; ++o) acc[o] = 0.f;
#pragma unroll
    for (int tap = 0; tap < 9; ++tap) {
      const int pr = 2 * r - 1 + tap / 3, pc = 2 * c - 1 + tap % 3;
      if (pr < 0 || pr >= S || pc < 0 || pc >= S) continue;  // conv zero padding
      if (pr >= mlo && pr < mhi && pc >= mlo && pc < mhi) continue;  // zeroed centre
      const int cls = lab[(pr - rp.lo) * wP + (pc - cp.lo)];
      if (cls >= C) continue;  // one-hot of an out-of-range class is all zero
      const float4* t4 = reinterpret_cast<const float4*>(table + ((long long)cls * 9 + tap) * 16);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float4 v = __ldg(t4 + j);
        acc[4 * j + 0] += v.x;
        acc[4 * j + 1] += v.y;
        acc[4 * j + 2] += v.z;
        acc[4 * j + 3] += v.w;
      }
    }
#pragma unroll
    for (int o = 0; o < 16; ++o) out[o * npix + pix] = fmaxf(acc[o] + __ldg(bias + o), 0.f);
  }
}

// dec.1 (3x3 on the x4 nearest-upsampled dec.0 map) + relu, head (1x1) and
// argmax over classes, for the tile's ts x ts output pixels (cabr.py:240-249,
// refine_blocks' np.argmax: first maximum wins).  A lane pair shares PX pixels:
// each lane owns 16 of the 32 decoder channels (PX x 16 accumulators), the head
// sums its half of every logit and one xor shuffle adds the partner's half.
template <int PX>
__device__ void dec1_head(const float* __restrict__ d0, Range rd, Range cd, int l0r, int l0c, int ts,
                          const float* __restrict__ w1, const float* __restrict__ b1, const float* __restrict__ hw,
                          const float* __restrict__ hb, const float* __restrict__ wm, int C, const CabrArgs& a,
                          int item, int bx, int by, int ty0, int tx0, int stream) {
  const int K = a.g.K;
  const int wD = cd.n(), plane = rd.n() * wD;
  const int half = threadIdx.x & 1, warp = threadIdx.x >> 5;
  // Pixels are assigned by row class u % 4 (u = l0r + i, the row in the x4 grid)
  // so every warp takes one class: classes 1 and 2 read one dec.0 row (merged
  // weights, 3 taps), classes 0 and 3 two (3x3 weights).  A warp's 16 lane pairs
  // cover 16 groups of PX pixels of one row; ts/4 rows per class.
  const int gpr = ts / PX;                          // groups per row
  const int wpc = (int)(blockDim.x >> 5) / 4;       // warps per class
  const int cls = warp / wpc;
  const int g = (warp - cls * wpc) * 16 + (threadIdx.x & 31) / 2;
  const int i = ((cls - l0r) & 3) + 4 * (g / gpr), j0 = (g % gpr) * PX;
  const int u = l0r + i;
  const bool merged = cls == 1 || cls == 2;
  int roff[3], coff[PX][3];
#pragma unroll
  for (int k = 0; k < 3; ++k) roff[k] = (((u - 1 + k) >> 2) - rd.lo) * wD;
#pragma unroll
  for (int p = 0; p < PX; ++p)
#pragma unroll
    for (int k = 0; k < 3; ++k) coff[p][k] = ((l0c + j0 + p - 1 + k) >> 2) - cd.lo;
  float acc[PX][16];
#pragma unroll
  for (int p = 0; p < PX; ++p)
#pragma unroll
    for (int o = 0; o < 16; ++o) acc[p][o] = 0.f;
  auto step = [&](const float* ip, const float* wrow, int r) {
#pragma unroll
    for (int kx = 0; kx < 3; ++kx) {
      float x[PX];
#pragma unroll
      for (int p = 0; p < PX; ++p) x[p] = ip[r + coff[p][kx]];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float4 wv = *reinterpret_cast<const float4*>(wrow + kx * 32 + 4 * j);
#pragma unroll
        for (int p = 0; p < PX; ++p) {
          acc[p][4 * j + 0] = fmaf(x[p], wv.x, acc[p][4 * j + 0]);
          acc[p][4 * j + 1] = fmaf(x[p], wv.y, acc[p][4 * j + 1]);
          acc[p][4 * j + 2] = fmaf(x[p], wv.z, acc[p][4 * j + 2]);
          acc[p][4 * j + 3] = fmaf(x[p], wv.w, acc[p][4 * j + 3]);
        }
      }
    }
  };
  if (merged) {
    for (int c = 0; c < 32; ++c) step(d0 + c * plane, wm + c * 96 + 16 * half, roff[1]);
  } else {
    for (int c = 0; c < 32; ++c) {
      const float* ip = d0 + c * plane;
      const float* wp = w1 + c * 9 * 32 + 16 * half;
#pragma unroll
      for (int ky = 0; ky < 3; ++ky) step(ip, wp + ky * 96, roff[ky]);
    }
  }
#pragma unroll
  for (int p = 0; p < PX; ++p)
#pragma unroll
    for (int o = 0; o < 16; ++o) acc[p][o] = fmaxf(acc[p][o] + b1[16 * half + o], 0.f);
  float best[PX];
  int arg[PX];
  for (int o = 0; o < C; ++o) {
    const float* hr = hw + o * 32 + 16 * half;
    float l[PX];
#pragma unroll
    for (int p = 0; p < PX; ++p) {
      float v = 0.f;
#pragma unroll
      for (int c = 0; c < 16; ++c) v = fmaf(acc[p][c], hr[c], v);
      l[p] = v;
    }
#pragma unroll
    for (int p = 0; p < PX; ++p) {
      // (low half + high half) in the same order on both lanes
      const float other = __shfl_xor_sync(0xffffffffu, l[p], 1);
      const float lo = half ? other : l[p], hi = half ? l[p] : other;
      const float v = (lo + hi) + hb[o];
      if (o == 0 || v > best[p]) {
        best[p] = v;
        arg[p] = o;
      }
      if (a.logits && half == 0) a.logits[(((long long)item * C + o) * K + ty0 + i) * K + tx0 + j0 + p] = v;
    }
  }
  if (half) return;
#pragma unroll
  for (int p = 0; p < PX; ++p) {
    const int yb = ty0 + i, xb = tx0 + j0 + p;  // position inside the K x K block
    if (a.argmax) a.argmax[((long long)item * K + yb) * K + xb] = (uint8_t)arg[p];
    if (a.scratch) {
      const int fy = by + yb, fx = bx + xb;
      if (fy < a.H && fx < a.W) a.scratch[stream * a.scr_ss + (long long)fy * a.W + fx] = (uint8_t)arg[p];
    }
  }
}

template <int TS, int THREADS>
__global__ void __launch_bounds__(THREADS, 1) cabr_kernel(const CabrArgs a) {
  extern __shared__ __align__(16) float smem[];
  const CabrGeo& g = a.g;
  const int K = g.K, S = 2 * K + 1, C = a.C;
  const int per_block = g.tiles * g.tiles;
  const int n_items = (a.flag_count ? a.flag_count[0] : a.n_blocks) * per_block;
  const WOff wo = cabr_offsets(C);
  float* sP = smem + g.off_p;
  float* sE0 = smem + g.off_e0;
  float* sE1 = smem + g.off_e1;
  float* sE2 = smem + g.off_e2;
  float* sW[2] = {smem + g.off_w, smem + g.off_w + g.wfloats};  // buffer 1 holds wfloats1 (dec.1 + head + merged)
  uint8_t* sLab = reinterpret_cast<uint8_t*>(smem) + g.off_lab;
  constexpr int PXD = 2 * TS * TS / THREADS;  // decoder pixels per lane pair
  // The item's eight weight stages, double-buffered: stage j lands in sW[j & 1]
  // while the layer before it computes from the other buffer.
  const float* wsrc[8] = {a.wts + wo.w[0], a.wts + wo.w[1], a.wts + wo.w[2], a.wts + wo.w[4],
                          a.wts + wo.w[5], a.wts + wo.w[6], a.wts + wo.w[6] + 32 * 9 * 32, a.wts + wo.w[7]};
  const int moff = (int)(cabr_merged_offset(wo) - wo.w[7]);  // merged dec.1 rows, relative to stage 7
  const int wlen[8] = {9 * 16 + 16, 16 * 9 * 32 + 32, 32 * 9 * 32 + 32, 16 * 9 * 32 + 32, 32 * 9 * 32 + 32,
                       32 * 9 * 32, 32 * 9 * 32 + 32, moff + kMergedFloats};
  auto issue = [&](int j) { stage_weights_async(sW[j & 1], wsrc[j], wlen[j]); };
  auto ready = [&]() {
    cp_async_wait_all();
    __syncthreads();
  };
  if ((int)blockIdx.x < n_items) issue(0);
  for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
    const int e = item / per_block, tile = item - e * per_block;
    const int ty0 = (tile / g.tiles) * TS, tx0 = (tile % g.tiles) * TS;
    int bx, by, stream = 0;
    if (a.flag_list) {
      const int id = a.flag_list[e];
      stream = id / a.cells;
      const int cell = id - stream * a.cells;
      bx = (cell % a.gw) * a.B;
      by = (cell / a.gw) * a.B;
    } else {
      bx = a.origins ? a.origins[2 * e] : 0;
      by = a.origins ? a.origins[2 * e + 1] : 0;
    }
    const Regions rr = regions(K, ty0, TS), rc = regions(K, tx0, TS);
    // ---- patch: image in [0, 1] and class bytes, edge-replicated (cabr.py:74-83)
    const int px0 = bx - K / 2, py0 = by - K / 2;
    const int hP = rr.p.n(), wP = rc.p.n();
    const bool explicit_patch = a.img_patch != nullptr;
    for (int i = threadIdx.x; i < hP * wP; i += blockDim.x) {
      const int r = rr.p.lo + i / wP, c = rc.p.lo + i % wP;
      float v;
      if (explicit_patch) {
        v = a.img_patch[((long long)e * S + r) * S + c];
      } else {
        const int fy = min(max(py0 + r, 0), a.H - 1), fx = min(max(px0 + c, 0), a.W - 1);
        const long long o = stream * a.pix_ss + a.t * a.pix_fs + (long long)fy * a.W + fx;
        if (a.pix_kind == 0)
          v = __fdiv_rn((float)static_cast<const uint8_t*>(a.pix)[o], 255.f);
        else if (a.pix_kind == 1)
          v = __fdiv_rn((float)static_cast<const uint16_t*>(a.pix)[o], 65535.f);
        else
          v = static_cast<const float*>(a.pix)[o];
        sLab[i] = a.labels[stream * a.lab_ss + a.t * a.lab_fs + (long long)fy * a.W + fx];
      }
      sP[i] = v;
    }
    ready();
    issue(1);
    // ---- image encoder (cabr.py:228-232)
    conv3x3<16, 1>(sP, rr.p, rc.p, S, 1, sW[0], sW[0] + 144, 16, 2, sE0, rr.e0, rc.e0, false, true);
    ready();
    issue(2);
    conv3x3<16, 2>(sE0, rr.e0, rc.e0, K + 1, 16, sW[1], sW[1] + 16 * 9 * 32, 32, 2, sE1, rr.e1, rc.e1, false, true);
    ready();
    issue(3);
    conv3x3<16, 2>(sE1, rr.e1, rc.e1, K / 2 + 1, 32, sW[0], sW[0] + 32 * 9 * 32, 32, 1, sE2, rr.e2, rc.e2, false,
                  true);
    __syncthreads();
    // ---- context encoder
    if (explicit_patch) {
      // general C-channel conv straight from the global patch (weights from global too)
      const float* ctx = a.ctx_patch + (long long)e * C * S * S;
      const Range full = {0, S};
      conv3x3<16, 1>(ctx, full, full, S, C, a.wts + wo.w[3], a.wts + wo.b[3], 16, 2, sE0, rr.e0, rc.e0, false, true);
    } else {
      ctx_conv0_onehot(sLab, rr.p, rc.p, S, K, C, a.wts + wo.w[3], a.wts + wo.b[3], sE0, rr.e0, rc.e0);
    }
    ready();
    issue(4);
    conv3x3<16, 2>(sE0, rr.e0, rc.e0, K + 1, 16, sW[1], sW[1] + 16 * 9 * 32, 32, 2, sE1, rr.e1, rc.e1, false, true);
    ready();
    issue(5);
    const int ne2 = rr.e2.n() * rc.e2.n();
    conv3x3<16, 2>(sE1, rr.e1, rc.e1, K / 2 + 1, 32, sW[0], sW[0] + 32 * 9 * 32, 32, 1, sE2 + 32 * ne2, rr.e2, rc.e2,
                  false, true);
    ready();
    issue(6);
    // ---- decoder conv 0 over the 64 fused channels, in two staged halves
    // (image half then context half: one accumulation order, cabr.py:235-237)
    float* sD0 = sE0;  // enc0 maps are dead
    conv3x3<16, 2>(sE2, rr.e2, rc.e2, K / 2 + 1, 32, sW[1], nullptr, 32, 1, sD0, rr.d0, rc.d0, false, false);
    ready();
    issue(7);
    conv3x3<16, 2>(sE2 + 32 * ne2, rr.e2, rc.e2, K / 2 + 1, 32, sW[0], sW[0] + 32 * 9 * 32, 32, 1, sD0, rr.d0, rc.d0,
                  true, true);
    ready();
    if (item + (int)gridDim.x < n_items) issue(0);  // the next item's first layer
    // ---- decoder conv 1 + head + argmax
    float* w7 = sW[1];
    dec1_head<PXD>(sD0, rr.d0, rc.d0, rr.l0, rc.l0, TS, w7, w7 + 32 * 9 * 32, w7 + 32 * 9 * 32 + 32,
                   w7 + 32 * 9 * 32 + 32 + C * 32, w7 + moff, C, a, e, bx, by, ty0, tx0, stream);
    __syncthreads();
  }
}

int plan_cabr(CabrGeo& g, int K, int C) {
  if (K < kCtxMask || K % 16) {
    set_error("CaBR block size must be a multiple of 16 and at least %d, got %d", kCtxMask, K);
    return BMC_E_ARG;
  }
  if (C < 1 || C > 256) {
    set_error("num_classes must be in 1..256 (uint8 labels), got %d", C);
    return BMC_E_ARG;
  }
  g.K = K;
  g.ts = K >= kMaxTile ? kMaxTile : 16;
  g.tiles = K / g.ts;
  g.threads = g.ts == 32 ? 512 : 256;
  g.np = g.ne0 = g.ne1 = g.ne2 = g.nd0 = 0;
  for (int t0 = 0; t0 < K; t0 += g.ts) {
    const Regions r = regions(K, t0, g.ts);
    g.np = r.p.n() > g.np ? r.p.n() : g.np;
    g.ne0 = r.e0.n() > g.ne0 ? r.e0.n() : g.ne0;
    g.ne1 = r.e1.n() > g.ne1 ? r.e1.n() : g.ne1;
    g.ne2 = r.e2.n() > g.ne2 ? r.e2.n() : g.ne2;
    g.nd0 = r.d0.n() > g.nd0 ? r.d0.n() : g.nd0;
  }
  auto up4 = [](int v) { return (v + 3) & ~3; };
  const int fp = up4(g.np * g.np);
  const int fe0 = up4(std::max(16 * g.ne0 * g.ne0, 32 * g.nd0 * g.nd0));  // dec0 output reuses enc0
  const int fe1 = up4(32 * g.ne1 * g.ne1);
  const int fe2 = up4(64 * g.ne2 * g.ne2);
  const WOff wo = cabr_offsets(C);
  g.wfloats = up4(32 * 9 * 32 + 32);  // buffer 0: the even stages
  g.wfloats1 = up4((int)(cabr_packed_floats(wo) - wo.w[7]));  // buffer 1 also takes stage 7 (dec.1 + head + merged)
  g.off_p = 0;
  g.off_e0 = g.off_p + fp;
  g.off_e1 = g.off_e0 + fe0;
  g.off_e2 = g.off_e1 + fe1;
  g.off_w = g.off_e2 + fe2;  // two weight buffers (double-buffered stages)
  g.off_lab = 4 * (g.off_w + g.wfloats + g.wfloats1);
  g.smem = g.off_lab + ((g.np * g.np + 15) & ~15);
  if (g.smem > 227 * 1024) {
    set_error("CaBR tile needs %d bytes of shared memory", g.smem);
    return BMC_E_ARG;
  }
  return BMC_OK;
}

template <int TS, int THREADS>
int launch_cabr_t(const CabrArgs& a, long long max_items, cudaStream_t st) {
  auto kern = cabr_kernel<TS, THREADS>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, a.g.smem);
  if (e != cudaSuccess) return cuda_status(e, "cudaFuncSetAttribute(cabr)");
  int dev = 0, sms = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, THREADS, a.g.smem);
  if (e != cudaSuccess) return cuda_status(e, "cudaOccupancyMaxActiveBlocksPerMultiprocessor(cabr)");
  long long grid = (long long)std::max(per_sm, 1) * sms;
  if (grid > max_items) grid = max_items;
  if (grid < 1) return BMC_OK;
  kern<<<(unsigned)grid, THREADS, a.g.smem, st>>>(a);
  return cuda_status(cudaGetLastError(), "cabr_kernel");
}

int launch_cabr(const CabrArgs& a, long long max_items, cudaStream_t st) {
  if (a.g.ts == 32) return launch_cabr_t<32, 512>(a, max_items, st);
  return launch_cabr_t<16, 256>(a, max_items, st);
}

// Flagged blocks of frames [t_begin, t_end) (pipeline.py:127-130: refinement_blocks
// of predicted frames), in (stream, gy, gx) order: list[(t - t_begin) * cap + k].
__global__ void cabr_flag_kernel(const uint8_t* __restrict__ matched, long long m_fs, long long m_ss,
                                 const int32_t* __restrict__ kind, long long kss, int n_streams, int cells,
                                 int t_begin, int32_t* __restrict__ list, int32_t* __restrict__ count, int cap) {
  __shared__ int warp_tot[32];
  __shared__ int base_s;
  const int t = t_begin + blockIdx.x;
  int32_t* out = list + (long long)blockIdx.x * cap;
  if (threadIdx.x == 0) base_s = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int total = n_streams * cells;
  for (int c0 = 0; c0 < total; c0 += blockDim.x) {
    const int i = c0 + threadIdx.x;
    bool f = false;
    if (i < total) {
      const int s = i / cells, c = i - s * cells;
      f = kind[(long long)s * kss + t] != 0 && matched[s * m_ss + t * m_fs + c] == 0;
    }
    const unsigned bal = __ballot_sync(0xffffffffu, f);
    if (lane == 0) warp_tot[wid] = __popc(bal);
    __syncthreads();
    int before = base_s;
    for (int w = 0; w < wid; ++w) before += warp_tot[w];
    if (f) out[before + __popc(bal & ((1u << lane) - 1))] = i;
    __syncthreads();
    if (threadIdx.x == 0) {
      int s = 0;
      for (int w = 0; w < nw; ++w) s += warp_tot[w];
      base_s += s;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) count[blockIdx.x] = base_s;
}

// refine_blocks' write-back (cabr.py:337-344): the refined pixels of every
// flagged block of frame t, clipped to the frame, from scratch into the labels.
__global__ void cabr_scatter_kernel(const int32_t* __restrict__ list, const int32_t* __restrict__ count,
                                    const uint8_t* __restrict__ scratch, long long scr_ss, uint8_t* labels,
                                    long long lab_ss, long long lab_off, int H, int W, int gw, int cells, int B) {
  const int n = count[0];
  for (int e = blockIdx.x; e < n; e += gridDim.x) {
    const int id = list[e];
    const int s = id / cells, cell = id - s * cells;
    const int bx = (cell % gw) * B, by = (cell / gw) * B;
    for (int i = threadIdx.x; i < B * B; i += blockDim.x) {
      const int y = by + i / B, x = bx + i % B;
      if (y < H && x < W) labels[s * lab_ss + lab_off + (long long)y * W + x] = scratch[s * scr_ss + (long long)y * W + x];
    }
  }
}

// extract_patch (cabr.py:60-90) for n origins: image (n,1,S,S) in [0,1] and the
// masked one-hot context (n,C,S,S), edge-replicated.
__global__ void cabr_extract_kernel(const void* __restrict__ pix, int pix_kind, const uint8_t* __restrict__ labels,
                                    int H, int W, const int32_t* __restrict__ origins, int n, int K, int C,
                                    float* __restrict__ image, float* __restrict__ context) {
  const int S = 2 * K + 1;
  const long long per = (long long)S * S;
  const int mlo = K - kCtxMask / 2, mhi = mlo + kCtxMask;
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < n * per;
       q += (long long)gridDim.x * blockDim.x) {
    const int e = (int)(q / per), rc = (int)(q % per), r = rc / S, c = rc % S;
    const int fy = min(max(origins[2 * e + 1] - K / 2 + r, 0), H - 1);
    const int fx = min(max(origins[2 * e] - K / 2 + c, 0), W - 1);
    const long long o = (long long)fy * W + fx;
    float v;
    if (pix_kind == 0) v = __fdiv_rn((float)static_cast<const uint8_t*>(pix)[o], 255.f);
    else if (pix_kind == 1) v = __fdiv_rn((float)static_cast<const uint16_t*>(pix)[o], 65535.f);
    else v = static_cast<const float*>(pix)[o];
    image[q] = v;
    const int cls = labels[o];
    const bool masked = r >= mlo && r < mhi && c >= mlo && c < mhi;
    float* ctx = context + (long long)e * C * per + rc;
    for (int ch = 0; ch < C; ++ch) ctx[ch * per] = (!masked && cls == ch) ? 1.f : 0.f;
  }
}

// Weight-free refinement (cabr.py:257-303 _ring_vote) of block e's pixels:
// the four ring pixels straight across the block borders (clamped), ring
// pixels inside flagged blocks ignored when a clean one exists, majority class
// among the nearest, ties to the smallest class.  Result into staging (n,K,K).
__global__ void ring_vote_blocks_kernel(const uint8_t* __restrict__ cls, const uint8_t* __restrict__ flagged, int H,
                                        int W, const int32_t* __restrict__ origins, int n, int k,
                                        uint8_t* __restrict__ staging) {
  const long long per = (long long)k * k;
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < n * per;
       q += (long long)gridDim.x * blockDim.x) {
    const int e = (int)(q / per), lyx = (int)(q % per), ly = lyx / k, lx = lyx % k;
    const int x0 = origins[2 * e], y0 = origins[2 * e + 1];
    const int x = min(max(x0 + lx, 0), W - 1), y = min(max(y0 + ly, 0), H - 1);
    const int ty = min(max(y0 - 1, 0), H - 1), by = min(max(y0 + k, 0), H - 1);
    const int lxr = min(max(x0 - 1, 0), W - 1), rxr = min(max(x0 + k, 0), W - 1);
    const long long at[4] = {(long long)ty * W + x, (long long)by * W + x, (long long)y * W + lxr,
                             (long long)y * W + rxr};
    const int dist[4] = {ly + 1, k - ly, lx + 1, k - lx};
    int cand[4];
    bool fl[4];
    bool any_clean = false;
    for (int c = 0; c < 4; ++c) {
      cand[c] = cls[at[c]];
      fl[c] = flagged[at[c]] != 0;
      any_clean |= !fl[c];
    }
    int dmin = 1 << 30;
    for (int c = 0; c < 4; ++c)
      if (!(any_clean && fl[c])) dmin = min(dmin, dist[c]);
    int best = -1, res = 0;
    for (int c = 0; c < 4; ++c) {
      const bool usable = !(any_clean && fl[c]);
      if (!usable || dist[c] != dmin) continue;
      int votes = 0;
      for (int b = 0; b < 4; ++b) votes += (!(any_clean && fl[b]) && dist[b] == dmin && cand[b] == cand[c]);
      const int score = votes * 256 + (255 - cand[c]);
      if (score > best) {
        best = score;
        res = cand[c];
      }
    }
    staging[q] = (uint8_t)res;
  }
}

// flagged_map of refine_blocks (cabr.py:324-326): 1 inside every listed block (clipped).
__global__ void mark_blocks_kernel(uint8_t* __restrict__ flagged, int H, int W, const int32_t* __restrict__ origins,
                                   int n, int k) {
  const long long per = (long long)k * k;
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < n * per;
       q += (long long)gridDim.x * blockDim.x) {
    const int e = (int)(q / per), r = (int)(q % per);
    const int y = origins[2 * e + 1] + r / k, x = origins[2 * e] + r % k;
    if (y < H && x < W) flagged[(long long)y * W + x] = 1;
  }
}

// Write-back in list order (cabr.py:337-344: later blocks overwrite earlier
// ones): pass 0 records the last block covering each pixel, pass 1 writes it.
__global__ void ordered_writeback_kernel(int pass, int32_t* __restrict__ owner, const uint8_t* __restrict__ staging,
                                         uint8_t* __restrict__ out, int H, int W, const int32_t* __restrict__ origins,
                                         int n, int k) {
  const long long per = (long long)k * k;
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < n * per;
       q += (long long)gridDim.x * blockDim.x) {
    const int e = (int)(q / per), r = (int)(q % per);
    const int y = origins[2 * e + 1] + r / k, x = origins[2 * e] + r % k;
    if (y >= H || x >= W) continue;
    const long long o = (long long)y * W + x;
    if (pass == 0) atomicMax(owner + o, e);
    else if (owner[o] == e) out[o] = staging[q];
  }
}

}  // namespace
}  // namespace bmc

using namespace bmc;

extern "C" size_t bmc_cabr_weight_floats(int num_classes) {
  if (num_classes < 1) return 0;
  return (size_t)cabr_packed_floats(cabr_offsets(num_classes));
}

extern "C" int bmc_cabr_pack_weights(const float* payload, int num_classes, float* packed, void* stream) {
  if (!payload || !packed || num_classes < 1 || num_classes > 256) {
    set_error("cabr_pack_weights: invalid arguments");
    return BMC_E_ARG;
  }
  const WOff o = cabr_offsets(num_classes);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cabr_pack_kernel<<<64, 256, 0, st>>>(payload, packed, o);
  cabr_merge_rows_kernel<<<(kMergedFloats + 255) / 256, 256, 0, st>>>(packed, o);
  return cuda_status(cudaGetLastError(), "cabr_pack_kernel");
}

static int cabr_common(CabrArgs& a, int block_size, int num_classes) {
  int rc = plan_cabr(a.g, block_size, num_classes);
  if (rc) return rc;
  a.C = num_classes;
  return BMC_OK;
}

extern "C" int bmc_cabr_forward_blocks(const void* pixels, int pixel_kind, const uint8_t* labels, int height,
                                       int width, const int32_t* origins, int n_blocks, int block_size,
                                       int num_classes, const float* packed, float* logits_out, uint8_t* argmax_out,
                                       void* stream) {
  if (!pixels || !labels || !origins || !packed || n_blocks < 0 || height < 1 || width < 1 || pixel_kind < 0 ||
      pixel_kind > 2) {
    set_error("cabr_forward_blocks: invalid arguments");
    return BMC_E_ARG;
  }
  CabrArgs a;
  std::memset(&a, 0, sizeof a);
  int rc = cabr_common(a, block_size, num_classes);
  if (rc) return rc;
  if (n_blocks == 0) return BMC_OK;
  a.pix = pixels;
  a.pix_kind = pixel_kind;
  a.labels = labels;
  a.H = height;
  a.W = width;
  a.wts = packed;
  a.origins = origins;
  a.n_blocks = n_blocks;
  a.logits = logits_out;
  a.argmax = argmax_out;
  return launch_cabr(a, (long long)n_blocks * a.g.tiles * a.g.tiles, static_cast<cudaStream_t>(stream));
}

extern "C" int bmc_cabr_forward_patches(const float* image, const float* context, int n_patches, int block_size,
                                        int num_classes, const float* packed, float* logits_out,
                                        uint8_t* argmax_out, void* stream) {
  if (!image || !context || !packed || n_patches < 0) {
    set_error("cabr_forward_patches: invalid arguments");
    return BMC_E_ARG;
  }
  CabrArgs a;
  std::memset(&a, 0, sizeof a);
  int rc = cabr_common(a, block_size, num_classes);
  if (rc) return rc;
  if (n_patches == 0) return BMC_OK;
  a.img_patch = image;
  a.ctx_patch = context;
  a.H = a.W = 2 * block_size + 1;
  a.wts = packed;
  a.n_blocks = n_patches;
  a.logits = logits_out;
  a.argmax = argmax_out;
  return launch_cabr(a, (long long)n_patches * a.g.tiles * a.g.tiles, static_cast<cudaStream_t>(stream));
}

extern "C" size_t bmc_cabr_chain_workspace(int n_streams, int n_frames, int grid_h, int grid_w) {
  const long long cap = (long long)n_streams * grid_h * grid_w;
  return (size_t)(n_frames * (cap + 1)) * sizeof(int32_t);
}

extern "C" int bmc_cabr_chain(uint8_t* labels, int64_t frame_stride, int64_t stream_stride, const uint8_t* key_labels,
                              int n_streams, int t_begin, int t_end, const int32_t* kind, const int32_t* ref,
                              int64_t kind_stream_stride, int height, int width, const int32_t* mv,
                              int64_t mv_frame_stride, int64_t mv_stream_stride, int grid_h, int grid_w,
                              int block_size, int scale, const uint8_t* matched, const void* pixels, int pixel_kind,
                              int64_t pix_frame_stride, int64_t pix_stream_stride, int num_classes,
                              const float* packed, uint8_t* scratch, int32_t* workspace, void* stream) {
  if (!labels || !key_labels || !kind || !ref || !mv || !matched || !pixels || !packed || !scratch || !workspace ||
      n_streams < 0 || pixel_kind < 0 || pixel_kind > 1 || (scale != 1 && scale != 2)) {
    set_error("cabr_chain: invalid arguments");
    return BMC_E_ARG;
  }
  const int B = block_size * scale;
  if (grid_w * B < width || grid_h * B < height) {
    set_error("motion field covers %dx%d, labels are %dx%d", grid_w * B, grid_h * B, width, height);
    return BMC_E_ARG;
  }
  CabrArgs a;
  std::memset(&a, 0, sizeof a);
  int rc = cabr_common(a, B, num_classes);
  if (rc) return rc;
  if (n_streams == 0 || height == 0 || width == 0 || t_end <= t_begin) return BMC_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int cells = grid_h * grid_w, nt = t_end - t_begin;
  const int cap = n_streams * cells;
  int32_t* list = workspace;
  int32_t* count = workspace + (long long)nt * cap;
  // matched is indexed like mv in cells: frame t at matched + t*(mv_frame_stride/2)
  cabr_flag_kernel<<<nt, 256, 0, st>>>(matched, mv_frame_stride / 2, mv_stream_stride / 2, kind, kind_stream_stride,
                                       n_streams, cells, t_begin, list, count, cap);
  if ((rc = cuda_status(cudaGetLastError(), "cabr_flag_kernel"))) return rc;
  a.pix = pixels;
  a.pix_kind = pixel_kind;
  a.pix_fs = pix_frame_stride;
  a.pix_ss = pix_stream_stride;
  a.labels = labels;
  a.lab_fs = frame_stride;
  a.lab_ss = stream_stride;
  a.H = height;
  a.W = width;
  a.wts = packed;
  a.gw = grid_w;
  a.cells = cells;
  a.B = B;
  a.scratch = scratch;
  a.scr_ss = (long long)height * width;
  for (int t = t_begin; t < t_end; ++t) {
    // plain prediction of frame t (key frames copy their labels)
    rc = bmc_predict_labels(labels, frame_stride, stream_stride, key_labels, n_streams, t, kind, ref, 0,
                            kind_stream_stride, height, width, mv, mv_frame_stride, mv_stream_stride, grid_h, grid_w,
                            block_size, scale, stream);
    if (rc) return rc;
    a.t = t;
    a.flag_list = list + (long long)(t - t_begin) * cap;
    a.flag_count = count + (t - t_begin);
    if ((rc = launch_cabr(a, (long long)cap * a.g.tiles * a.g.tiles, st))) return rc;
    cabr_scatter_kernel<<<std::min(cap, 1024), 256, 0, st>>>(a.flag_list, a.flag_count, scratch, a.scr_ss, labels,
                                                             stream_stride, t * frame_stride, height, width, grid_w,
                                                             cells, B);
    if ((rc = cuda_status(cudaGetLastError(), "cabr_scatter_kernel"))) return rc;
  }
  return BMC_OK;
}

extern "C" int bmc_cabr_extract_patches(const void* pixels, int pixel_kind, const uint8_t* labels, int height,
                                        int width, const int32_t* origins, int n, int block_size, int num_classes,
                                        float* image_out, float* context_out, void* stream) {
  if (!pixels || !labels || !origins || !image_out || !context_out || n < 0 || height < 1 || width < 1 ||
      pixel_kind < 0 || pixel_kind > 2 || num_classes < 1) {
    set_error("cabr_extract_patches: invalid arguments");
    return BMC_E_ARG;
  }
  if (block_size < kCtxMask) {
    set_error("CaBR block size must be at least %d: the fixed %dx%d context mask would cover a %dx%d block entirely",
              kCtxMask, kCtxMask, kCtxMask, block_size, block_size);
    return BMC_E_ARG;
  }
  if (n == 0) return BMC_OK;
  cabr_extract_kernel<<<1024, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      pixels, pixel_kind, labels, height, width, origins, n, block_size, num_classes, image_out, context_out);
  return cuda_status(cudaGetLastError(), "cabr_extract_kernel");
}

extern "C" int bmc_refine_blocks(const void* pixels, int pixel_kind, const uint8_t* labels_in, uint8_t* labels_out,
                                 int height, int width, const int32_t* origins, int n, int block_size,
                                 int num_classes, const float* packed, uint8_t* staging, int32_t* owner,
                                 uint8_t* flagged, void* stream) {
  if (!labels_in || !labels_out || !origins || !staging || !owner || n < 0 || height < 1 || width < 1 ||
      (packed && !pixels) || (!packed && !flagged)) {
    set_error("refine_blocks: invalid arguments");
    return BMC_E_ARG;
  }
  if (block_size < kCtxMask) {
    set_error("CaBR block size must be at least %d: the fixed %dx%d context mask would cover a %dx%d block entirely",
              kCtxMask, kCtxMask, kCtxMask, block_size, block_size);
    return BMC_E_ARG;
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int rc = cuda_status(cudaMemcpyAsync(labels_out, labels_in, (size_t)height * width, cudaMemcpyDeviceToDevice, st),
                       "refine_blocks copy");
  if (rc || n == 0) return rc;
  if (packed) {
    rc = bmc_cabr_forward_blocks(pixels, pixel_kind, labels_in, height, width, origins, n, block_size, num_classes,
                                 packed, nullptr, staging, stream);
    if (rc) return rc;
  } else {
    if ((rc = cuda_status(cudaMemsetAsync(flagged, 0, (size_t)height * width, st), "refine_blocks memset")))
      return rc;
    mark_blocks_kernel<<<1024, 256, 0, st>>>(flagged, height, width, origins, n, block_size);
    ring_vote_blocks_kernel<<<1024, 256, 0, st>>>(labels_in, flagged, height, width, origins, n, block_size, staging);
    if ((rc = cuda_status(cudaGetLastError(), "ring_vote_blocks_kernel"))) return rc;
  }
  if ((rc = cuda_status(cudaMemsetAsync(owner, 0xFF, (size_t)height * width * sizeof(int32_t), st),
                        "refine_blocks memset")))
    return rc;
  ordered_writeback_kernel<<<1024, 256, 0, st>>>(0, owner, staging, labels_out, height, width, origins, n, block_size);
  ordered_writeback_kernel<<<1024, 256, 0, st>>>(1, owner, staging, labels_out, height, width, origins, n, block_size);
  return cuda_status(cudaGetLastError(), "ordered_writeback_kernel");
}
