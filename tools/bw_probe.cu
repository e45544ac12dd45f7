// Calibration microbenchmark (not product code): achievable HBM throughput
// for (a) a streaming copy and (b) a thread-per-column primal update over a
// CSC with uniform short columns (transportation shape: n=1M, 2 per column).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bw_probe tools/bw_probe.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

__global__ void copy_k(const double* __restrict__ a, double* __restrict__ b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) b[i] = a[i];
}

// x+ = clamp(x - s (c - K^T y)), xbar update; thread per column.
__global__ void primal_direct(int n, const int* __restrict__ cp, const int* __restrict__ ri, const double* __restrict__ cv,
                              const double* __restrict__ y, const double* __restrict__ x, const double* __restrict__ c,
                              const double* __restrict__ l, const double* __restrict__ u, double* __restrict__ xn,
                              double* __restrict__ xbar, double step, double w) {
  int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  int b = cp[j], e = cp[j + 1];
  double acc = 0.0;
  for (int k = b; k < e; ++k) acc += cv[k] * y[ri[k]];
  double xo = x[j];
  double v = xo - step * (c[j] - acc);
  v = v < l[j] ? l[j] : v;
  v = u[j] < v ? u[j] : v;
  xn[j] = v;
  xbar[j] = (w * xbar[j] + v) / (w + 1.0);
}

// Same, with the uniform-length loop unrolled (L = 2) and loads hoisted.
template <int L>
__global__ void primal_direct_fixed(int n, const int* __restrict__ ri, const double* __restrict__ cv,
                                    const double* __restrict__ y, const double* __restrict__ x, const double* __restrict__ c,
                                    const double* __restrict__ l, const double* __restrict__ u, double* __restrict__ xn,
                                    double* __restrict__ xbar, double step, double w) {
  int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  double acc = 0.0;
#pragma unroll
  for (int k = 0; k < L; ++k) acc += cv[(size_t)j * L + k] * y[ri[(size_t)j * L + k]];
  double xo = x[j];
  double v = xo - step * (c[j] - acc);
  v = v < l[j] ? l[j] : v;
  v = u[j] < v ? u[j] : v;
  xn[j] = v;
  xbar[j] = (w * xbar[j] + v) / (w + 1.0);
}

int main() {
  const int n = 1000000, m = 2000, L = 2;
  const size_t nnz = (size_t)n * L;
  int *cp, *ri;
  double *cv, *y, *x, *c, *l, *u, *xn, *xbar, *a, *b;
  cudaMalloc(&cp, (n + 1) * 4);
  cudaMalloc(&ri, nnz * 4);
  cudaMalloc(&cv, nnz * 8);
  cudaMalloc(&y, m * 8);
  for (double** p : {&x, &c, &l, &u, &xn, &xbar}) cudaMalloc(p, n * 8);
  std::vector<int> hcp(n + 1), hri(nnz);
  for (int j = 0; j <= n; ++j) hcp[j] = j * L;
  for (size_t k = 0; k < nnz; ++k) hri[k] = (k % 2) ? 1000 + (k / 2) / 1000 : (k / 2) % 1000;
  cudaMemcpy(cp, hcp.data(), (n + 1) * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(ri, hri.data(), nnz * 4, cudaMemcpyHostToDevice);
  cudaMemset(cv, 0, nnz * 8);
  cudaMemset(y, 0, m * 8);
  for (double* p : {x, c, l, u, xn, xbar}) cudaMemset(p, 0, n * 8);
  const size_t big = 84ull << 20;
  cudaMalloc(&a, big);
  cudaMalloc(&b, big);
  cudaMemset(a, 1, big);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms;
  auto timeit = [&](const char* name, double bytes, auto fn) {
    for (int i = 0; i < 5; ++i) fn();
    cudaEventRecord(e0);
    const int R = 50;
    for (int i = 0; i < R; ++i) fn();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("%-28s %8.2f us  %7.0f GB/s\n", name, ms * 1e3 / R, bytes / (ms * 1e-3 / R) / 1e9);
  };
  for (int blocks : {148 * 4, 148 * 8, 148 * 16, 148 * 32}) {
    char nm[64];
    snprintf(nm, 64, "copy 84MB grid=%d", blocks);
    timeit(nm, 2.0 * big, [&] { copy_k<<<blocks, 256>>>(a, b, big / 8 / 2 * 2 / 2); });
  }
  const double pb = 12.0 * nnz + 4.0 * (n + 1) + 8.0 * m + 56.0 * n;
  for (int bs : {128, 256, 512}) {
    char nm[64];
    snprintf(nm, 64, "primal direct bs=%d", bs);
    timeit(nm, pb, [&] { primal_direct<<<(n + bs - 1) / bs, bs>>>(n, cp, ri, cv, y, x, c, l, u, xn, xbar, 0.1, 3.0); });
  }
  timeit("primal fixed L=2", pb - 4.0 * (n + 1),
         [&] { primal_direct_fixed<2><<<(n + 255) / 256, 256>>>(n, ri, cv, y, x, c, l, u, xn, xbar, 0.1, 3.0); });
  return 0;
}
