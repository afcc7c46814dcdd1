// Microbenchmarks isolating the DMMA GEMM inner loop on B200 (not part of the product path).
//   mode 0: 8 independent accumulators, constant operands (pipe peak)
//   mode 1: 32x32 warp tile, fragments re-loaded from shared memory (LDS.128) every k-pair
//   mode 2: mode 1 + __syncthreads every 16 k (one k-tile)
//   mode 3: 32x32 warp tile, fragments from registers (no LDS), 16 accumulators
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_micro dmma_micro.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c[0]), "+d"(c[1])
      : "d"(a), "d"(b));
}

template <int MODE>
__global__ void __launch_bounds__(256, 2) kern(double* out, int iters) {
  __shared__ __align__(16) double sA[16 * 24 * 8];   // 128 rows x 24 (K-contig, padded)
  __shared__ __align__(16) double sB[16 * 24 * 8];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < 16 * 24 * 8; i += blockDim.x) {
    sA[i] = 1.0 + i * 1e-9;
    sB[i] = 1.0 - i * 1e-9;
  }
  __syncthreads();
  const int g = lane >> 2, t = lane & 3;
  const int wm = warp >> 1, wn = warp & 1;   // 4 x 2 warps, 32x32 tiles (128 x 64 CTA tile)
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  double ra[2][4], rb[2][4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    ra[0][i] = 1.0 + i + lane * 1e-3;
    ra[1][i] = 2.0 + i;
    rb[0][i] = 1.0 - i * 1e-3;
    rb[1][i] = 0.5 + i;
  }
  for (int it = 0; it < iters; ++it) {
    if (MODE == 0) {
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) dmma(acc[i][j], ra[0][0], rb[0][0]);
    } else if (MODE == 3) {
#pragma unroll
      for (int kp = 0; kp < 2; ++kp)
#pragma unroll
        for (int s = 0; s < 2; ++s)
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) dmma(acc[i][j], ra[s][i], rb[s][j]);
    } else {
#pragma unroll
      for (int kp = 0; kp < 2; ++kp) {
        double af[2][4], bf[2][4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const double2 v = *reinterpret_cast<const double2*>(sA + (wm * 32 + i * 8 + g) * 24 + kp * 8 + 2 * t);
          af[0][i] = v.x;
          af[1][i] = v.y;
          const double2 w = *reinterpret_cast<const double2*>(sB + (wn * 32 + i * 8 + g) * 24 + kp * 8 + 2 * t);
          bf[0][i] = w.x;
          bf[1][i] = w.y;
        }
#pragma unroll
        for (int s = 0; s < 2; ++s)
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) dmma(acc[i][j], af[s][i], bf[s][j]);
      }
      if (MODE == 2) __syncthreads();
    }
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) s += acc[i][j][0] + acc[i][j][1];
  if (s == 12345.678) out[tid] = s;
}

template <int MODE>
void run(const char* name, int sms, double* out, int blocks_per_sm) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 4000;
  const int blocks = sms * blocks_per_sm;
  kern<MODE><<<blocks, 256>>>(out, 10);
  cudaDeviceSynchronize();
  cudaEventRecord(e0);
  kern<MODE><<<blocks, 256>>>(out, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double dmmas_per_iter = (MODE == 0) ? 32 : 64;   // per warp
  const double flops = 512.0 * dmmas_per_iter * iters * blocks * 8;
  printf("{\"mode\":\"%s\",\"warps_per_sm\":%d,\"ms\":%.3f,\"tflops\":%.2f}\n", name,
         8 * blocks_per_sm, ms, flops / ms / 1e9);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, 1 << 20);
  for (int bps = 1; bps <= 2; ++bps) {
    run<0>("const_operands", sms, out, bps);
    run<3>("reg_fragments_32x32", sms, out, bps);
    run<1>("lds128_fragments_32x32", sms, out, bps);
    run<2>("lds128_plus_syncthreads", sms, out, bps);
  }
  cudaError_t e = cudaGetLastError();
  printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
