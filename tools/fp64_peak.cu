// Microbenchmark: FP64 DFMA vs DMMA (mma.sync m8n8k4 f64) throughput on sm_100a,
// plus mixed issue, and shared-memory LDS.64 bandwidth. Used to decide the
// per-order DMMA-vs-DFMA choice.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_kernel(double* out, int iters) {
  double a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const double b = 1.0000001, c = 1e-9;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
      a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

__global__ void dmma_kernel(double* out, int iters) {
  double c[8][2];
#pragma unroll
  for (int t = 0; t < 8; ++t) { c[t][0] = 0; c[t][1] = 0; }
  double a = threadIdx.x * 1e-3, b = 1e-3;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
#pragma unroll
      for (int t = 0; t < 8; ++t) dmma(c[t][0], c[t][1], a, b);
    }
  }
  double s = 0;
#pragma unroll
  for (int t = 0; t < 8; ++t) s += c[t][0] + c[t][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// mixed: per iteration 8 DMMA + 8x8 DFMA (equal MAC count per warp: 8*256 vs 64*32)
__global__ void mixed_kernel(double* out, int iters) {
  double c[4][2];
#pragma unroll
  for (int t = 0; t < 4; ++t) { c[t][0] = 0; c[t][1] = 0; }
  double a = threadIdx.x * 1e-3, b = 1e-3;
  double a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3;
  const double bb = 1.0000001, cc = 1e-9;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
#pragma unroll
      for (int t = 0; t < 4; ++t) dmma(c[t][0], c[t][1], a, b);
      a0 = fma(a0, bb, cc); a1 = fma(a1, bb, cc); a2 = fma(a2, bb, cc); a3 = fma(a3, bb, cc);
      a0 = fma(a0, bb, cc); a1 = fma(a1, bb, cc); a2 = fma(a2, bb, cc); a3 = fma(a3, bb, cc);
      a0 = fma(a0, bb, cc); a1 = fma(a1, bb, cc); a2 = fma(a2, bb, cc); a3 = fma(a3, bb, cc);
      a0 = fma(a0, bb, cc); a1 = fma(a1, bb, cc); a2 = fma(a2, bb, cc); a3 = fma(a3, bb, cc);
    }
  }
  double s = a0 + a1 + a2 + a3;
#pragma unroll
  for (int t = 0; t < 4; ++t) s += c[t][0] + c[t][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void lds_kernel(double* out, int iters) {
  __shared__ double s[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) s[i] = i;
  __syncthreads();
  double acc = 0;
  int idx = threadIdx.x;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) acc += s[(idx + u * 64) & 4095];
    idx = (idx + 32) & 4095;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double* out; cudaMalloc(&out, sizeof(double) * sms * 8 * 1024);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 4096;
  for (int threads : {256, 512, 1024}) {
    int blocks = sms * (2048 / threads);
    float ms;
    dfma_kernel<<<blocks, threads>>>(out, 16);
    cudaEventRecord(e0); dfma_kernel<<<blocks, threads>>>(out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 64 * iters * (double)blocks * threads;
    printf("DFMA  threads=%4d  %.2f TFLOP/s\n", threads, fl / ms / 1e9);
    dmma_kernel<<<blocks, threads>>>(out, 16);
    cudaEventRecord(e0); dmma_kernel<<<blocks, threads>>>(out, iters / 4); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    fl = 2.0 * 256 * 64 * (iters / 4) * (double)blocks * threads / 32;
    printf("DMMA  threads=%4d  %.2f TFLOP/s\n", threads, fl / ms / 1e9);
    mixed_kernel<<<blocks, threads>>>(out, 16);
    cudaEventRecord(e0); mixed_kernel<<<blocks, threads>>>(out, iters / 4); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    fl = (2.0 * 256 * 32 * (iters / 4) * (double)blocks * threads / 32) + 2.0 * 128 * (iters / 4) * (double)blocks * threads;
    printf("MIXED threads=%4d  %.2f TFLOP/s (half DMMA, half DFMA MACs)\n", threads, fl / ms / 1e9);
    lds_kernel<<<blocks, threads>>>(out, 16);
    cudaEventRecord(e0); lds_kernel<<<blocks, threads>>>(out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    double by = 8.0 * 16 * iters * (double)blocks * threads;
    printf("LDS64 threads=%4d  %.2f TB/s smem (%.1f B/clk/SM at %d MHz)\n", threads, by / ms / 1e9, by / (ms * 1e-3) / sms / (clk * 1e3), clk / 1000);
  }
  cudaError_t err = cudaGetLastError();
  printf("sms=%d clk=%d MHz err=%s\n", sms, clk / 1000, cudaGetErrorString(err));
  return 0;
}
