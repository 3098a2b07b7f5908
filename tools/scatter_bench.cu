// Microbenchmark: cost of the E->L scatter on B200 with the real BP gather
// pattern (element-major, x-fastest local numbering, shared nodes):
//   red   : atomicAdd (RED.E.ADD.F64) per element node   (what the apply does)
//   store : plain 8-byte store per element node          (lower bound, wrong sums)
//   gather: 8-byte load x[gid] per element node           (the E-restriction read)
// Usage: scatter_bench p n   (mesh n^3, order p)
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

__global__ void build_ids(int* ids, int n, int p) {
  const int d = p + 1, d3 = d * d * d;
  const long long npx = (long long)n * p + 1;
  const long long total = (long long)n * n * n * d3;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total; t += (long long)gridDim.x * blockDim.x) {
    long long e = t / d3; int l = t % d3;
    int i = l % d, j = (l / d) % d, k = l / (d * d);
    long long ex = e % n, ey = (e / n) % n, ez = e / ((long long)n * n);
    ids[t] = (int)((ex * p + i) + npx * ((ey * p + j) + npx * (ez * p + k)));
  }
}
__global__ void k_red(double* y, const int* ids, long long m) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < m; t += (long long)gridDim.x * blockDim.x)
    atomicAdd(y + ids[t], 1.0);
}
__global__ void k_store(double* y, const int* ids, long long m) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < m; t += (long long)gridDim.x * blockDim.x)
    y[ids[t]] = 1.0;
}
__global__ void k_gather(const double* x, const int* ids, double* out, long long m) {
  double s = 0;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < m; t += (long long)gridDim.x * blockDim.x)
    s += __ldg(x + ids[t]);
  if (s == 12345.0) out[0] = s;
}

int main(int argc, char** argv) {
  int p = argc > 1 ? atoi(argv[1]) : 4, n = argc > 2 ? atoi(argv[2]) : 54;
  const int d3 = (p + 1) * (p + 1) * (p + 1);
  long long m = (long long)n * n * n * d3, ndof = ((long long)n * p + 1) * (n * p + 1) * (n * p + 1);
  int* ids; double *y, *x;
  cudaMalloc(&ids, m * 4); cudaMalloc(&y, ndof * 8); cudaMalloc(&x, ndof * 8);
  cudaMemset(x, 0, ndof * 8);
  build_ids<<<148 * 8, 256>>>(ids, n, p);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const char* names[3] = {"red", "store", "gather"};
  for (int v = 0; v < 3; ++v) {
    for (int rep = 0; rep < 4; ++rep) {
      cudaMemsetAsync(y, 0, ndof * 8);
      cudaEventRecord(a);
      if (v == 0) k_red<<<148 * 8, 256>>>(y, ids, m);
      if (v == 1) k_store<<<148 * 8, 256>>>(y, ids, m);
      if (v == 2) k_gather<<<148 * 8, 256>>>(x, ids, y, m);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      if (rep == 3) printf("p=%d n=%d %-6s %8.3f ms  %7.1f G ops/s  (%lld ops, %.1f MB ids)\n", p, n, names[v], ms, m / ms / 1e6, m, m * 4 / 1e6);
    }
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
