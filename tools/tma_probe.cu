// Probe: does a tiled TMA load accept inner start coordinates that are not
// 16-byte aligned (uint8 tensor, x = 0..7, also negative)?  Prints one line per
// offset: OK / MISMATCH / error.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__global__ void probe(const __grid_constant__ CUtensorMap tm, int x, int y, int z, unsigned char* out, int bytes) {
  __shared__ __align__(128) unsigned char buf[64 * 8 * 2];
  __shared__ __align__(8) unsigned long long bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)), "r"(bytes) : "memory");
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
            smem_u32(buf)),
        "l"(reinterpret_cast<uint64_t>(&tm)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(&bar))
        : "memory");
  }
  asm volatile(
      "{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}\n" ::"r"(smem_u32(&bar)),
      "r"(0)
      : "memory");
  for (int i = threadIdx.x; i < bytes; i += blockDim.x) out[i] = buf[i];
}

int main() {
  const int W = 256, H = 64, Z = 2;
  std::vector<unsigned char> h(W * H * Z);
  for (size_t i = 0; i < h.size(); ++i) h[i] = (unsigned char)(i * 131 + 7);
  unsigned char *d, *o;
  cudaMalloc(&d, h.size());
  cudaMalloc(&o, 4096);
  cudaMemcpy(d, h.data(), h.size(), cudaMemcpyHostToDevice);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  CUtensorMap tm;
  const int BW = 64, BH = 8, BZ = 2;
  cuuint64_t dims[3] = {W, H, Z};
  cuuint64_t strides[2] = {W, (cuuint64_t)W * H};
  cuuint32_t box[3] = {BW, BH, BZ};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, d, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d\n", (int)r);
  const int xs[] = {0, 1, 2, 3, 5, 7, 13, 17, -3, 250};
  for (int x : xs) {
    const int y = 5;
    probe<<<1, 128>>>(tm, x, y, 0, o, BW * BH * BZ);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("x=%d error %s\n", x, cudaGetErrorString(e));
      return 1;
    }
    std::vector<unsigned char> got(BW * BH * BZ);
    cudaMemcpy(got.data(), o, got.size(), cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int zz = 0; zz < BZ; ++zz)
      for (int yy = 0; yy < BH; ++yy)
        for (int xx = 0; xx < BW; ++xx) {
          const int gx = x + xx, gy = y + yy;
          const unsigned char want = (gx >= 0 && gx < W && gy < H) ? h[(size_t)zz * W * H + gy * W + gx] : 0;
          if (got[(zz * BH + yy) * BW + xx] != want) ++bad;
        }
    printf("x=%d %s (%d bad)\n", x, bad ? "MISMATCH" : "OK", bad);
  }
  return 0;
}
