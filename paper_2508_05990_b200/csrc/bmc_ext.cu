// Ingest (raw sensor payload decode) and reporting (confusion matrices for
// mIoU) kernels: the data formats either side of the hot path (SURVEY.md §8f
// ranks 2 and 4).  Both are HBM/PCIe-class byte work: coalesced loads, one
// pass over the payload, grids sized to the SM count.
#include <algorithm>
#include <cstdint>

#include "../../include/bmc_ext.h"
#include "bmc_internal.cuh"

namespace bmc {
namespace {

int sm_count() {
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms > 0 ? sms : 148;
}

// ---------------------------------------------------------------------------
// raw decode: one thread per 8-pixel group of a row (BE16: 16 payload bytes,
// RAW10: 10, RAW12: 12), one 16-byte store of eight uint16.
// ---------------------------------------------------------------------------
template <int FMT>
__device__ __forceinline__ uint32_t decode_px(const uint8_t* row, int x) {
  if (FMT == BMC_RAW_BE16) {
    return (uint32_t(row[2 * x]) << 8) | row[2 * x + 1];
  } else if (FMT == BMC_RAW_MIPI10) {
    const uint8_t* g = row + (x >> 2) * 5;
    int i = x & 3;
    return (uint32_t(g[i]) << 2) | ((g[4] >> (2 * i)) & 3u);
  } else {
    const uint8_t* g = row + (x >> 1) * 3;
    int i = x & 1;
    return (uint32_t(g[i]) << 4) | ((g[2] >> (4 * i)) & 15u);
  }
}

template <int FMT>
__global__ void __launch_bounds__(256) unpack_raw_kernel(const uint8_t* __restrict__ src, int64_t frame_bytes,
                                                         int64_t row_bytes, int height, int width, int shift,
                                                         int groups_per_row, int64_t groups_per_frame,
                                                         int64_t total_groups, uint16_t* __restrict__ dst) {
  for (int64_t g = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; g < total_groups;
       g += int64_t(gridDim.x) * blockDim.x) {
    int64_t f = g / groups_per_frame;
    int64_t r = g - f * groups_per_frame;
    int y = int(r / groups_per_row);
    int x0 = int(r - int64_t(y) * groups_per_row) * 8;
    const uint8_t* row = src + f * frame_bytes + int64_t(y) * row_bytes;
    uint16_t* out = dst + (f * height + y) * int64_t(width) + x0;
    if (x0 + 8 <= width && (reinterpret_cast<uintptr_t>(out) & 15) == 0) {
      uint32_t v[8];
      if (FMT == BMC_RAW_BE16 && (reinterpret_cast<uintptr_t>(row + 2 * x0) & 15) == 0) {
        uint4 w = *reinterpret_cast<const uint4*>(row + 2 * x0);
        uint32_t ww[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          uint32_t s = __byte_perm(ww[k], 0, 0x2301);  // swap bytes within each 16-bit half
          v[2 * k] = s & 0xffffu;
          v[2 * k + 1] = s >> 16;
        }
      } else {
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = decode_px<FMT>(row, x0 + k);
      }
      uint4 o;
      o.x = ((v[0] << shift) & 0xffffu) | (((v[1] << shift) & 0xffffu) << 16);
      o.y = ((v[2] << shift) & 0xffffu) | (((v[3] << shift) & 0xffffu) << 16);
      o.z = ((v[4] << shift) & 0xffffu) | (((v[5] << shift) & 0xffffu) << 16);
      o.w = ((v[6] << shift) & 0xffffu) | (((v[7] << shift) & 0xffffu) << 16);
      *reinterpret_cast<uint4*>(out) = o;
    } else {
      for (int x = x0; x < min(x0 + 8, width); ++x) out[x - x0] = uint16_t(decode_px<FMT>(row, x) << shift);
    }
  }
}

__global__ void __launch_bounds__(256) pack_be16_kernel(const uint16_t* __restrict__ src, int64_t n,
                                                        uint8_t* __restrict__ dst) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    uint16_t v = src[i];
    dst[2 * i] = uint8_t(v >> 8);
    dst[2 * i + 1] = uint8_t(v & 0xff);
  }
}

// ---------------------------------------------------------------------------
// confusion matrices: a CTA owns a slice of one map; bins live in shared memory
// (num_classes^2 <= kSmemBins) or go straight to global atomics.  16-byte loads
// of pred and truth when both slices are aligned.
// ---------------------------------------------------------------------------
constexpr int kSmemBins = 12288;  // 48 KB of uint32 counters

template <bool SMEM>
__device__ __forceinline__ void tally(uint32_t t, uint32_t p, int nc, int ignore, uint32_t* sh,
                                      unsigned long long* gl, int32_t* overflow) {
  if (int(t) == ignore) return;
  uint32_t idx = t * uint32_t(nc) + p;
  if (idx >= uint32_t(nc) * uint32_t(nc)) {
    if (overflow) *overflow = 1;
    return;
  }
  if (SMEM)
    atomicAdd(sh + idx, 1u);
  else
    atomicAdd(gl + idx, 1ull);
}

template <bool SMEM>
__global__ void __launch_bounds__(512) confusion_kernel(const uint8_t* __restrict__ pred,
                                                        const uint8_t* __restrict__ truth, int64_t n,
                                                        int64_t map_stride, int nc, int ignore,
                                                        unsigned long long* __restrict__ conf, int32_t* overflow) {
  extern __shared__ uint32_t sh[];
  const int map = blockIdx.y;
  const int bins = nc * nc;
  unsigned long long* gl = conf + int64_t(map) * bins;
  if (SMEM) {
    for (int i = threadIdx.x; i < bins; i += blockDim.x) sh[i] = 0;
    __syncthreads();
  }
  const uint8_t* pm = pred + map * map_stride;
  const uint8_t* tm = truth + map * map_stride;
  // slice [lo, hi) of this CTA, 16-byte aligned interior
  int64_t per = ((n + gridDim.x - 1) / gridDim.x + 15) & ~int64_t(15);
  int64_t lo = min(n, per * blockIdx.x), hi = min(n, lo + per);
  bool vec = ((reinterpret_cast<uintptr_t>(pm + lo) | reinterpret_cast<uintptr_t>(tm + lo)) & 15) == 0;
  int64_t vend = vec ? lo + ((hi - lo) & ~int64_t(15)) : lo;
  for (int64_t i = lo + 16 * int64_t(threadIdx.x); i < vend; i += 16 * int64_t(blockDim.x)) {
    uint4 pv = *reinterpret_cast<const uint4*>(pm + i);
    uint4 tv = *reinterpret_cast<const uint4*>(tm + i);
    uint32_t pw[4] = {pv.x, pv.y, pv.z, pv.w}, tw[4] = {tv.x, tv.y, tv.z, tv.w};
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
      for (int j = 0; j < 4; ++j)
        tally<SMEM>((tw[k] >> (8 * j)) & 0xff, (pw[k] >> (8 * j)) & 0xff, nc, ignore, sh, gl, overflow);
  }
  for (int64_t i = vend + threadIdx.x; i < hi; i += blockDim.x) tally<SMEM>(tm[i], pm[i], nc, ignore, sh, gl, overflow);
  if (SMEM) {
    __syncthreads();
    for (int i = threadIdx.x; i < bins; i += blockDim.x)
      if (sh[i]) atomicAdd(gl + i, (unsigned long long)sh[i]);
  }
}

}  // namespace
}  // namespace bmc

using namespace bmc;

extern "C" int bmc_unpack_raw(const uint8_t* src, int64_t src_frame_bytes, int64_t src_row_bytes, int n_frames,
                              int height, int width, int format, int shift, uint16_t* dst, void* stream) {
  if (!src || !dst || n_frames < 0 || height <= 0 || width <= 0 || shift < 0 || shift > 15) {
    set_error("unpack_raw: invalid buffers or geometry");
    return BMC_E_ARG;
  }
  int64_t need = format == BMC_RAW_BE16 ? 2 * int64_t(width)
                 : format == BMC_RAW_MIPI10 ? (int64_t(width) + 3) / 4 * 5
                 : format == BMC_RAW_MIPI12 ? (int64_t(width) + 1) / 2 * 3
                                            : -1;
  if (need < 0) {
    set_error("unpack_raw: unknown payload format %d", format);
    return BMC_E_ARG;
  }
  if (src_row_bytes < need || src_frame_bytes < src_row_bytes * height) {
    set_error("unpack_raw: row stride %lld / frame stride %lld too small for %dx%d", (long long)src_row_bytes,
              (long long)src_frame_bytes, width, height);
    return BMC_E_ARG;
  }
  if (n_frames == 0) return BMC_OK;
  int gpr = (width + 7) / 8;
  int64_t gpf = int64_t(gpr) * height, total = gpf * n_frames;
  int64_t blocks = std::min<int64_t>((total + 255) / 256, int64_t(sm_count()) * 8);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (format == BMC_RAW_BE16)
    unpack_raw_kernel<BMC_RAW_BE16><<<int(blocks), 256, 0, st>>>(src, src_frame_bytes, src_row_bytes, height, width,
                                                                 shift, gpr, gpf, total, dst);
  else if (format == BMC_RAW_MIPI10)
    unpack_raw_kernel<BMC_RAW_MIPI10><<<int(blocks), 256, 0, st>>>(src, src_frame_bytes, src_row_bytes, height,
                                                                   width, shift, gpr, gpf, total, dst);
  else
    unpack_raw_kernel<BMC_RAW_MIPI12><<<int(blocks), 256, 0, st>>>(src, src_frame_bytes, src_row_bytes, height,
                                                                   width, shift, gpr, gpf, total, dst);
  return cuda_status(cudaGetLastError(), "unpack_raw_kernel");
}

extern "C" int bmc_pack_be16(const uint16_t* src, int64_t n, uint8_t* dst, void* stream) {
  if (!src || !dst || n < 0) {
    set_error("pack_be16: invalid buffers");
    return BMC_E_ARG;
  }
  if (n == 0) return BMC_OK;
  int64_t blocks = std::min<int64_t>((n + 255) / 256, int64_t(sm_count()) * 8);
  pack_be16_kernel<<<int(blocks), 256, 0, static_cast<cudaStream_t>(stream)>>>(src, n, dst);
  return cuda_status(cudaGetLastError(), "pack_be16_kernel");
}

extern "C" int bmc_confusion(const uint8_t* pred, const uint8_t* truth, int64_t n, int n_maps, int64_t map_stride,
                             int num_classes, int ignore_class, unsigned long long* confusion, int32_t* overflow,
                             void* stream) {
  if (!pred || !truth || !confusion || n < 0 || n_maps < 0 || num_classes < 1 || num_classes > 1024 ||
      (n_maps > 1 && map_stride < n)) {
    set_error("confusion: invalid buffers, sizes or num_classes (1..1024)");
    return BMC_E_ARG;
  }
  if (n_maps > 65535) {
    set_error("confusion: at most 65535 maps per call");
    return BMC_E_ARG;
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int bins = num_classes * num_classes;
  int rc = cuda_status(cudaMemsetAsync(confusion, 0, sizeof(unsigned long long) * bins * size_t(n_maps), st),
                       "confusion memset");
  if (rc) return rc;
  if (overflow && (rc = cuda_status(cudaMemsetAsync(overflow, 0, sizeof(int32_t), st), "confusion memset")))
    return rc;
  if (n == 0 || n_maps == 0) return BMC_OK;
  // enough CTAs to cover the SMs ~4 deep across all maps, at least 64 KB per CTA
  int64_t per_map = std::max<int64_t>(1, std::min<int64_t>((n + 65535) / 65536, (int64_t(sm_count()) * 4 + n_maps - 1) / n_maps));
  dim3 grid((unsigned)per_map, (unsigned)n_maps);
  if (bins <= kSmemBins)
    confusion_kernel<true><<<grid, 512, bins * sizeof(uint32_t), st>>>(pred, truth, n, map_stride, num_classes,
                                                                       ignore_class, confusion, overflow);
  else
    confusion_kernel<false><<<grid, 512, 0, st>>>(pred, truth, n, map_stride, num_classes, ignore_class, confusion,
                                                  overflow);
  return cuda_status(cudaGetLastError(), "confusion_kernel");
}
