// Microbenchmark: sustained issue rate of the integer SAD instructions on sm_100a.
// Measures the R_sad denominator of the roofline: VABSDIFF4.U8.ACC
// (4 uint8 samples per instruction) and VABSDIFF.U32 (1 uint16 sample), plus the
// companion instructions the search kernel mixes in (LDS, SHF/PRMT, IDP.4A, DADD).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o sad_peak sad_peak.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

__device__ __forceinline__ uint32_t vsad4(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm volatile("vabsdiff4.u32.u32.u32.add %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}
__device__ __forceinline__ uint32_t vsad1(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm volatile("vabsdiff.u32.u32.u32.add %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}

constexpr int ITERS = 4096;
constexpr int NACC = 8;

struct Stat { unsigned long long cyc, ns; };

__device__ __forceinline__ void record(Stat* st, long long c0, unsigned long long t0) {
  long long c1 = clock64();
  unsigned long long t1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  if (threadIdx.x == 0) {
    atomicMax(&st->cyc, (unsigned long long)(c1 - c0));
    atomicMax(&st->ns, t1 - t0);
  }
}

// mode 0: pure VABSDIFF4.ACC; 1: pure VABSDIFF.U32.ACC; 2: VABSDIFF4 + SHF 1:1;
// 3: VABSDIFF4 + PRMT 1:1; 4: IDP.4A; 5: VABSDIFF4 (non-acc) + LOP3 + IADD + LOP3 + IDP (count idiom);
// 6: the uint16 SAD word of the search kernels (bmc_internal.cuh sad_word<uint16_t>):
//    max.u16x2 + min.u16x2 + IADD + IDP.2A per 2 samples
template <int MODE>
__global__ void k_alu(uint32_t* out, Stat* st, uint32_t seed) {
  uint32_t acc[NACC], k[NACC];
#pragma unroll
  for (int j = 0; j < NACC; ++j) { acc[j] = seed * (j + 1) + threadIdx.x; k[j] = seed ^ (j * 0x01010101u); }
  __syncthreads();
  long long c0 = clock64();
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int j = 0; j < NACC; ++j) {
      if (MODE == 0) acc[j] = vsad4(acc[j], k[j], acc[j]);
      if (MODE == 1) acc[j] = vsad1(acc[j], k[j], acc[j]);
      if (MODE == 2) { uint32_t s = __funnelshift_r(acc[j], k[j], it & 31); acc[j] = vsad4(s, k[j], acc[j]); }
      if (MODE == 3) { uint32_t s = __byte_perm(acc[j], k[j], 0x5432); acc[j] = vsad4(s, k[j], acc[j]); }
      if (MODE == 4) acc[j] = __dp4a(acc[j], k[j], acc[j]);
      if (MODE == 6) {
        uint32_t mx, mn;
        asm volatile("max.u16x2 %0, %1, %2;" : "=r"(mx) : "r"(acc[j]), "r"(k[j]));
        asm volatile("min.u16x2 %0, %1, %2;" : "=r"(mn) : "r"(acc[j]), "r"(k[j]));
        acc[j] = __dp2a_lo(mx - mn, 0x0101u, acc[j]);
      }
      if (MODE == 5) {
        uint32_t d = __vabsdiffu4(acc[j], k[j]);
        uint32_t t = (d & 0x7f7f7f7fu) + k[(j + 1) & 7];
        uint32_t m = (t | d) & 0x80808080u;
        acc[j] = __dp4a(m, 0x01010101u, acc[j]);
      }
    }
  }
  record(st, c0, t0);
  uint32_t s = 0;
#pragma unroll
  for (int j = 0; j < NACC; ++j) s ^= acc[j];
  if (s == 0x12345678u) out[0] = s;
}

// VABSDIFF4 fed from shared memory: each LDS.128 feeds RATIO*4 VABSDIFF4.
template <int RATIO>
__global__ void k_lds(uint32_t* out, Stat* st, uint32_t seed) {
  __shared__ uint4 sm[2048];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) sm[i] = make_uint4(seed + i, seed * i, i, seed ^ i);
  __syncthreads();
  uint32_t acc[NACC];
#pragma unroll
  for (int j = 0; j < NACC; ++j) acc[j] = seed + j;
  uint32_t c[4] = {seed, seed + 1, seed + 2, seed + 3};
  long long c0 = clock64();
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  int idx = threadIdx.x;
  for (int it = 0; it < ITERS / 4; ++it) {
#pragma unroll
    for (int q = 0; q < 8 / RATIO; ++q) {
      uint4 r = sm[(idx + q * 37 + it) & 2047];
#pragma unroll
      for (int t = 0; t < RATIO; ++t) {
        int j = (q * RATIO + t) & 7;
        acc[j] = vsad4(r.x, c[t & 3], acc[j]);
        acc[j] = vsad4(r.y, c[(t + 1) & 3], acc[j]);
        acc[j] = vsad4(r.z, c[(t + 2) & 3], acc[j]);
        acc[j] = vsad4(r.w, c[(t + 3) & 3], acc[j]);
      }
    }
  }
  record(st, c0, t0);
  uint32_t s = 0;
#pragma unroll
  for (int j = 0; j < NACC; ++j) s ^= acc[j];
  if (s == 0x12345678u) out[0] = s;
}

__global__ void k_dadd(double* out, Stat* st, double seed) {
  double acc[NACC];
#pragma unroll
  for (int j = 0; j < NACC; ++j) acc[j] = seed * (j + 1) + threadIdx.x;
  long long c0 = clock64();
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int j = 0; j < NACC; ++j) acc[j] = __dadd_rn(acc[j], seed);
  }
  record(st, c0, t0);
  double s = 0;
#pragma unroll
  for (int j = 0; j < NACC; ++j) s += acc[j];
  if (s == 1.2345) out[0] = s;
}

// fp32 FFMA issue rate (the CaBR-Net kernel's roofline denominator)
__global__ void k_ffma(float* out, Stat* st, float seed) {
  float acc[NACC];
#pragma unroll
  for (int j = 0; j < NACC; ++j) acc[j] = seed * (j + 1) + threadIdx.x;
  long long c0 = clock64();
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int j = 0; j < NACC; ++j) acc[j] = fmaf(acc[j], 0.999999f, seed);
  }
  record(st, c0, t0);
  float s = 0;
#pragma unroll
  for (int j = 0; j < NACC; ++j) s += acc[j];
  if (s == 1.2345f) out[0] = s;
}

int main() {
  int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  printf("{\"sms\": %d}\n", sms);
  uint32_t* out; Stat* st;
  CK(cudaMalloc(&out, 16)); CK(cudaMalloc(&st, sizeof(Stat)));
  int grid = sms * 4, block = 512;  // 64 warps/SM
  uint32_t seed = 0x9e3779b9u;
  auto L = [&](const char* n, void (*k)(uint32_t*, Stat*, uint32_t), double opi, double spo) {
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int rep = 0; rep < 3; ++rep) {
      cudaMemset(st, 0, sizeof(Stat));
      cudaEventRecord(e0);
      k<<<grid, block>>>(out, st, seed);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      Stat h; cudaMemcpy(&h, st, sizeof(Stat), cudaMemcpyDeviceToHost);
      double ops = (double)grid * block * ITERS * opi;
      printf("{\"kernel\": \"%s\", \"rep\": %d, \"ms_event\": %.4f, \"cycles\": %llu, \"ns\": %llu, \"mhz\": %.1f, "
             "\"lane_ops_per_clk_per_sm\": %.2f, \"Gops_per_s\": %.1f, \"Gsamples_per_s\": %.1f}\n",
             n, rep, ms, h.cyc, h.ns, (double)h.cyc / h.ns * 1e3, ops / ((double)h.cyc * sms),
             ops / (h.ns * 1e-9) / 1e9, ops * spo / (h.ns * 1e-9) / 1e9);
    }
  };
  L("vabsdiff4_acc", k_alu<0>, NACC, 4.0);
  L("vabsdiff_u32_acc", k_alu<1>, NACC, 1.0);
  L("vabsdiff4+shf", k_alu<2>, NACC, 4.0);
  L("vabsdiff4+prmt", k_alu<3>, NACC, 4.0);
  L("idp4a", k_alu<4>, NACC, 0.0);
  L("count_idiom(5 instr)", k_alu<5>, NACC, 4.0);
  L("u16_sad_word(vimnmx x2 + iadd + idp2a)", k_alu<6>, NACC, 2.0);
  L("lds128_x1_per4vsad", k_lds<1>, 32.0 / 4, 4.0);
  L("lds128_x1_per8vsad", k_lds<2>, 32.0 / 4, 4.0);
  L("lds128_x1_per16vsad", k_lds<4>, 32.0 / 4, 4.0);
  L("lds128_x1_per32vsad", k_lds<8>, 32.0 / 4, 4.0);
  {
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    double* dout; cudaMalloc(&dout, 16);
    for (int rep = 0; rep < 3; ++rep) {
      cudaMemset(st, 0, sizeof(Stat));
      cudaEventRecord(e0);
      k_dadd<<<grid, block>>>(dout, st, 1.000001);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      Stat h; cudaMemcpy(&h, st, sizeof(Stat), cudaMemcpyDeviceToHost);
      double ops = (double)grid * block * ITERS * NACC;
      printf("{\"kernel\": \"dadd\", \"rep\": %d, \"mhz\": %.1f, \"lane_ops_per_clk_per_sm\": %.2f, \"Gops_per_s\": %.1f}\n",
             rep, (double)h.cyc / h.ns * 1e3, ops / ((double)h.cyc * sms), ops / (h.ns * 1e-9) / 1e9);
    }
  }
  {
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    float* fout; cudaMalloc(&fout, 16);
    for (int rep = 0; rep < 3; ++rep) {
      cudaMemset(st, 0, sizeof(Stat));
      cudaEventRecord(e0);
      k_ffma<<<grid, block>>>(fout, st, 1.0001f);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      Stat h; cudaMemcpy(&h, st, sizeof(Stat), cudaMemcpyDeviceToHost);
      double ops = (double)grid * block * ITERS * NACC;
      printf("{\"kernel\": \"ffma_f32\", \"rep\": %d, \"mhz\": %.1f, \"lane_ops_per_clk_per_sm\": %.2f, "
             "\"Gops_per_s\": %.1f, \"TFLOPs\": %.2f}\n",
             rep, (double)h.cyc / h.ns * 1e3, ops / ((double)h.cyc * sms), ops / (h.ns * 1e-9) / 1e9,
             2 * ops / (h.ns * 1e-9) / 1e12);
    }
  }
  CK(cudaGetLastError());
  return 0;
}
