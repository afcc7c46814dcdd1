// FP64 peak microbenchmarks for B200 (sm_100a): DMMA (mma.sync m8n8k4 f64) and DFMA.
// Measures the roofline denominator P64.  Not part of the product path.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

template <int NACC>
__global__ void dmma_loop(double* out, int iters, double seed) {
  double a = seed + threadIdx.x * 1e-3, b = seed * 0.5 - threadIdx.x * 1e-3;
  double c[NACC][2];
#pragma unroll
  for (int i = 0; i < NACC; ++i) { c[i][0] = 0.0; c[i][1] = 0.0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[threadIdx.x] = s;
}

template <int NACC>
__global__ void dfma_loop(double* out, int iters, double seed) {
  double a = seed + threadIdx.x * 1e-9, b = 1.0 - 1e-12;
  double c[NACC];
#pragma unroll
  for (int i = 0; i < NACC; ++i) c[i] = i * 1e-3;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) c[i] = fma(c[i], b, a);
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i];
  if (s == 12345.678) out[threadIdx.x] = s;
}

int main() {
  cudaDeviceProp p;
  CK(cudaGetDeviceProperties(&p, 0));
  int clk_khz = 0; cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  printf("{\"device\":\"%s\",\"sms\":%d,\"smem_per_sm\":%zu,\"smem_optin\":%zu,\"l2\":%d,\"regs_per_sm\":%d,\"clock_khz\":%d,\"cc\":\"%d.%d\"}\n",
         p.name, p.multiProcessorCount, p.sharedMemPerMultiprocessor, p.sharedMemPerBlockOptin,
         p.l2CacheSize, p.regsPerMultiprocessor, clk_khz, p.major, p.minor);
  double* out; CK(cudaMalloc(&out, 1 << 20));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int sms = p.multiProcessorCount;
  int warps_list[] = {4, 8, 16, 32};
  for (int w : warps_list) {
    for (int rep = 0; rep < 2; ++rep) {
      int iters = 20000;
      int blocks = sms * 2, threads = w * 32 / 2;  // 2 blocks/SM -> w warps per SM
      dmma_loop<8><<<blocks, threads>>>(out, 100, 1.0);
      CK(cudaDeviceSynchronize());
      cudaEventRecord(e0);
      dmma_loop<8><<<blocks, threads>>>(out, iters, 1.0);
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double flops = 2.0 * 8 * 8 * 4 * 8.0 * iters * (double)blocks * (threads / 32);
      if (rep) printf("{\"kind\":\"dmma_m8n8k4\",\"warps_per_sm\":%d,\"ms\":%.3f,\"tflops\":%.2f}\n", w, ms, flops / ms / 1e9);
    }
  }
  for (int w : warps_list) {
    for (int rep = 0; rep < 2; ++rep) {
      int iters = 20000;
      int blocks = sms * 2, threads = w * 32 / 2;
      dfma_loop<16><<<blocks, threads>>>(out, 100, 1.0);
      CK(cudaDeviceSynchronize());
      cudaEventRecord(e0);
      dfma_loop<16><<<blocks, threads>>>(out, iters, 1.0);
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double flops = 2.0 * 16.0 * iters * (double)blocks * threads;
      if (rep) printf("{\"kind\":\"dfma\",\"warps_per_sm\":%d,\"ms\":%.3f,\"tflops\":%.2f}\n", w, ms, flops / ms / 1e9);
    }
  }
  return 0;
}
