// Microbenchmark: cost of the E->L scatter on B200 with the real BP gather
// pattern (element-major, x-fastest local numbering, shared nodes):
//   red   : atomicAdd (RED.E.ADD.F64) per element node   (what the apply does)
//   store : plain 8-byte store per element node          (lower bound, wrong sums)
//   gather: 8-byte load x[gid] per element node           (the E-restriction read)
//   redln : atomicAdd with the fused kernel's stage-E lane pattern: one thread
//           per x-line (element, j, k), looping over i (each RED instruction
//           touches one row per lane)
//   bulkln: the same lines through the TMA engine: each thread stages its line
//           in a 16-byte-aligned zero-padded shared-memory window and issues
//           one cp.reduce.async.bulk .add.f64 (UBLKRED) per line
// Usage: scatter_bench p n   (mesh n^3, order p)
#include <cstdio>
#include <cstdlib>
#include <cmath>
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
__global__ void k_red_lines(double* y, const int* ids, long long nlines, int d) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < nlines; t += (long long)gridDim.x * blockDim.x) {
    const int* r = ids + t * d;  // ids of line t (x-fastest: the line's d nodes are consecutive)
    for (int i = 0; i < d; ++i) atomicAdd(y + r[i], 1.0);
  }
}
__global__ void k_bulk_lines(double* y, const int* ids, long long nlines, int d) {
  __shared__ __align__(16) double st[256 * 12];
  double* my = st + threadIdx.x * 12;
  const unsigned sa = (unsigned)__cvta_generic_to_shared(my);
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < nlines; t += (long long)gridDim.x * blockDim.x) {
    const int g0 = ids[t * d];
    const int lead = g0 & 1;  // y is 256-byte aligned: 16-byte phase of the line
    const int n = (lead + d + 1) & ~1;
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // slot free again
    for (int i = 0; i < n; ++i) my[i] = (i >= lead && i < lead + d) ? 1.0 : 0.0;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f64 [%0], [%1], %2;"
                 :: "l"(y + g0 - lead), "r"(sa), "r"(8 * n) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
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
  const char* names[5] = {"red", "store", "gather", "redln", "bulkln"};
  std::vector<double> ref(ndof), got(ndof);
  for (int v = 0; v < 5; ++v) {
    for (int rep = 0; rep < 4; ++rep) {
      cudaMemsetAsync(y, 0, ndof * 8);
      cudaEventRecord(a);
      if (v == 0) k_red<<<148 * 8, 256>>>(y, ids, m);
      if (v == 1) k_store<<<148 * 8, 256>>>(y, ids, m);
      if (v == 2) k_gather<<<148 * 8, 256>>>(x, ids, y, m);
      if (v == 3) k_red_lines<<<148 * 8, 256>>>(y, ids, m / (p + 1), p + 1);
      if (v == 4) k_bulk_lines<<<148 * 4, 256>>>(y, ids, m / (p + 1), p + 1);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      if (rep == 3 && v == 0) cudaMemcpy(ref.data(), y, ndof * 8, cudaMemcpyDeviceToHost);
      if (rep == 3 && v == 4) {
        cudaMemcpy(got.data(), y, ndof * 8, cudaMemcpyDeviceToHost);
        double md = 0;
        for (long long i = 0; i < ndof; ++i) md = md > fabs(got[i] - ref[i]) ? md : fabs(got[i] - ref[i]);
        printf("bulkln vs red: max |diff| %g\n", md);
      }
      if (rep == 3) printf("p=%d n=%d %-6s %8.3f ms  %7.1f G ops/s  (%lld ops, %.1f MB ids)\n", p, n, names[v], ms, m / ms / 1e6, m, m * 4 / 1e6);
    }
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
