// Library comparator: one PDHG iteration built from
// cuSPARSE SpMV (CSR, FP64) plus separate elementwise kernels, timed on the
// same matrices as the fused step kernels -- measurement tool only, never
// linked into the product.
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC \
//        -o tools/_build/libcusparse_cmp.so tools/cusparse_cmp.cu -lcusparse
//
// cmp_iteration() uploads K (CSR) and K^T (CSR of the transpose = K's CSC),
// then times, with CUDA events on one stream (mean per launch, warm = back to
// back; cold = an L2 sweep before every launch, sweep time subtracted):
//   [0] K^T y  cusparseSpMV CSR_ALG2 on K^T        (reference MultiplyTranspose)
//   [1] K x    cusparseSpMV CSR_ALG2 on K          (reference Multiply)
//   [2] K^T y  cusparseSpMV CSR_ALG1 on K^T
//   [3] K x    cusparseSpMV CSR_ALG1 on K
//   [4] K^T y  cusparseSpMV TRANSPOSE of K (ALG1, no CSC copy)
//   [5] primal elementwise: x+ = clamp(x - s (c - K^T y), l, u), x-bar update
//   [6] dual elementwise:   y+ = proj(y + s (q - (2 K x+ - K x))), y-bar update
//   [7] a whole unfused iteration: [0] + [5] + [1] + [6] back to back
// times[k] = warm ms, times[8 + k] = cold ms.
#include <cuda_runtime.h>
#include <cusparse.h>

#include <cstdint>
#include <cstdio>
#include <vector>

#define CK(x)                                                                    \
  do {                                                                           \
    cudaError_t e_ = (x);                                                        \
    if (e_ != cudaSuccess) {                                                     \
      std::fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e_));              \
      return 1;                                                                  \
    }                                                                            \
  } while (0)
#define CS(x)                                                                    \
  do {                                                                           \
    cusparseStatus_t s_ = (x);                                                   \
    if (s_ != CUSPARSE_STATUS_SUCCESS) {                                         \
      std::fprintf(stderr, "%s: %s\n", #x, cusparseGetErrorString(s_));         \
      return 2;                                                                  \
    }                                                                            \
  } while (0)

__global__ void k_primal(int64_t n, const double* x, const double* c, const double* kty, const double* l,
                         const double* u, double step, double w, double* xn, double* xbar) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    double v = x[j] - step * (c[j] - kty[j]);
    v = v < l[j] ? l[j] : v;
    v = u[j] < v ? u[j] : v;
    xn[j] = v;
    xbar[j] = (w * xbar[j] + v) / (w + 1.0);
  }
}

__global__ void k_dual(int64_t m, int64_t m1, const double* y, const double* q, const double* kx, const double* kxn,
                       double step, double w, double* yn, double* ybar) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
    double v = y[i] + step * (q[i] - (2.0 * kxn[i] - kx[i]));
    if (i >= m1) v = v < 0.0 ? 0.0 : v;
    yn[i] = v;
    ybar[i] = (w * ybar[i] + v) / (w + 1.0);
  }
}

__global__ void k_sweep(double* b, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    b[i] += 1.0;
}

extern "C" int cmp_iteration(int64_t m, int64_t m1, int64_t n, int64_t nnz, const int32_t* rp, const int32_t* ci,
                             const double* rv, const int32_t* cp, const int32_t* ri, const double* cv, int reps,
                             double* times) {
  cudaStream_t st;
  CK(cudaStreamCreate(&st));
  int32_t *d_rp, *d_ci, *d_cp, *d_ri;
  double *d_rv, *d_cv;
  CK(cudaMalloc(&d_rp, (m + 1) * 4));
  CK(cudaMalloc(&d_cp, (n + 1) * 4));
  CK(cudaMalloc(&d_ci, nnz * 4));
  CK(cudaMalloc(&d_ri, nnz * 4));
  CK(cudaMalloc(&d_rv, nnz * 8));
  CK(cudaMalloc(&d_cv, nnz * 8));
  CK(cudaMemcpy(d_rp, rp, (m + 1) * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_cp, cp, (n + 1) * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_ci, ci, nnz * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_ri, ri, nnz * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_rv, rv, nnz * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_cv, cv, nnz * 8, cudaMemcpyHostToDevice));
  // vectors: x, xn, xbar, c, l, u, kty (n); y, yn, ybar, q, kx, kxn (m)
  std::vector<double*> vn(7), vm(6);
  for (auto& p : vn) {
    CK(cudaMalloc(&p, (n > 0 ? n : 1) * 8));
    CK(cudaMemset(p, 0, (n > 0 ? n : 1) * 8));
  }
  for (auto& p : vm) {
    CK(cudaMalloc(&p, (m > 0 ? m : 1) * 8));
    CK(cudaMemset(p, 0, (m > 0 ? m : 1) * 8));
  }
  double *x = vn[0], *xn = vn[1], *xbar = vn[2], *c = vn[3], *l = vn[4], *u = vn[5], *kty = vn[6];
  double *y = vm[0], *yn = vm[1], *ybar = vm[2], *q = vm[3], *kx = vm[4], *kxn = vm[5];
  {  // u = +inf, x = 0.5
    std::vector<double> h(n, 1e300);
    CK(cudaMemcpy(u, h.data(), n * 8, cudaMemcpyHostToDevice));
    std::vector<double> hx(n, 0.5);
    CK(cudaMemcpy(x, hx.data(), n * 8, cudaMemcpyHostToDevice));
    std::vector<double> hy(m, 0.25);
    CK(cudaMemcpy(y, hy.data(), m * 8, cudaMemcpyHostToDevice));
  }
  const int64_t sweep_n = (256ll << 20) / 8;  // 256 MB > 2x L2
  double* sweep;
  CK(cudaMalloc(&sweep, sweep_n * 8));
  CK(cudaMemset(sweep, 0, sweep_n * 8));

  cusparseHandle_t h;
  CS(cusparseCreate(&h));
  CS(cusparseSetStream(h, st));
  cusparseSpMatDescr_t K, KT;
  CS(cusparseCreateCsr(&K, m, n, nnz, d_rp, d_ci, d_rv, CUSPARSE_INDEX_32I, CUSPARSE_INDEX_32I,
                       CUSPARSE_INDEX_BASE_ZERO, CUDA_R_64F));
  CS(cusparseCreateCsr(&KT, n, m, nnz, d_cp, d_ri, d_cv, CUSPARSE_INDEX_32I, CUSPARSE_INDEX_32I,
                       CUSPARSE_INDEX_BASE_ZERO, CUDA_R_64F));
  cusparseDnVecDescr_t vx, vxn, vy, vyn, vkty, vkx, vkxn;
  CS(cusparseCreateDnVec(&vx, n, x, CUDA_R_64F));
  CS(cusparseCreateDnVec(&vxn, n, xn, CUDA_R_64F));
  CS(cusparseCreateDnVec(&vkty, n, kty, CUDA_R_64F));
  CS(cusparseCreateDnVec(&vy, m, y, CUDA_R_64F));
  CS(cusparseCreateDnVec(&vyn, m, yn, CUDA_R_64F));
  CS(cusparseCreateDnVec(&vkx, m, kx, CUDA_R_64F));
  CS(cusparseCreateDnVec(&vkxn, m, kxn, CUDA_R_64F));
  const double one = 1.0, zero = 0.0;
  struct Op {
    cusparseOperation_t op;
    cusparseSpMatDescr_t A;
    cusparseDnVecDescr_t in, out;
    cusparseSpMVAlg_t alg;
    void* buf;
  };
  Op ops[5] = {{CUSPARSE_OPERATION_NON_TRANSPOSE, KT, vy, vkty, CUSPARSE_SPMV_CSR_ALG2, nullptr},
               {CUSPARSE_OPERATION_NON_TRANSPOSE, K, vxn, vkxn, CUSPARSE_SPMV_CSR_ALG2, nullptr},
               {CUSPARSE_OPERATION_NON_TRANSPOSE, KT, vy, vkty, CUSPARSE_SPMV_CSR_ALG1, nullptr},
               {CUSPARSE_OPERATION_NON_TRANSPOSE, K, vxn, vkxn, CUSPARSE_SPMV_CSR_ALG1, nullptr},
               {CUSPARSE_OPERATION_TRANSPOSE, K, vy, vkty, CUSPARSE_SPMV_CSR_ALG1, nullptr}};
  for (Op& o : ops) {
    size_t bytes = 0;
    CS(cusparseSpMV_bufferSize(h, o.op, &one, o.A, o.in, &zero, o.out, CUDA_R_64F, o.alg, &bytes));
    CK(cudaMalloc(&o.buf, bytes > 0 ? bytes : 16));
#if CUSPARSE_VERSION >= 12400
    CS(cusparseSpMV_preprocess(h, o.op, &one, o.A, o.in, &zero, o.out, CUDA_R_64F, o.alg, o.buf));
#endif
  }
  auto spmv = [&](int k) {
    Op& o = ops[k];
    return cusparseSpMV(h, o.op, &one, o.A, o.in, &zero, o.out, CUDA_R_64F, o.alg, o.buf);
  };
  const int ew = 148 * 8;
  auto primal = [&] { k_primal<<<ew, 256, 0, st>>>(n, x, c, kty, l, u, 1e-3, 3.0, xn, xbar); };
  auto dual = [&] { k_dual<<<ew, 256, 0, st>>>(m, m1, y, q, kx, kxn, 1e-3, 3.0, yn, ybar); };
  auto run = [&](int k) -> int {
    if (k < 5) CS(spmv(k));
    else if (k == 5) primal();
    else if (k == 6) dual();
    else {
      CS(spmv(0));
      primal();
      CS(spmv(1));
      dual();
    }
    return 0;
  };
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  auto sweep_only = [&] { k_sweep<<<148 * 8, 256, 0, st>>>(sweep, sweep_n); };
  // sweep cost
  float ms_sweep = 0;
  for (int w = 0; w < 2; ++w) sweep_only();
  CK(cudaEventRecord(e0, st));
  for (int r = 0; r < reps; ++r) sweep_only();
  CK(cudaEventRecord(e1, st));
  CK(cudaEventSynchronize(e1));
  CK(cudaEventElapsedTime(&ms_sweep, e0, e1));
  for (int k = 0; k < 8; ++k) {
    for (int w = 0; w < 3; ++w)
      if (int rc = run(k)) return rc;
    float ms = 0;
    CK(cudaEventRecord(e0, st));
    for (int r = 0; r < reps; ++r)
      if (int rc = run(k)) return rc;
    CK(cudaEventRecord(e1, st));
    CK(cudaEventSynchronize(e1));
    CK(cudaEventElapsedTime(&ms, e0, e1));
    times[k] = ms / reps;
    CK(cudaEventRecord(e0, st));
    for (int r = 0; r < reps; ++r) {
      sweep_only();
      if (int rc = run(k)) return rc;
    }
    CK(cudaEventRecord(e1, st));
    CK(cudaEventSynchronize(e1));
    CK(cudaEventElapsedTime(&ms, e0, e1));
    times[8 + k] = (ms - ms_sweep) / reps;
  }
  CK(cudaStreamSynchronize(st));
  for (Op& o : ops) cudaFree(o.buf);
  cusparseDestroySpMat(K);
  cusparseDestroySpMat(KT);
  for (auto v : {vx, vxn, vy, vyn, vkty, vkx, vkxn}) cusparseDestroyDnVec(v);
  cusparseDestroy(h);
  for (auto p : vn) cudaFree(p);
  for (auto p : vm) cudaFree(p);
  cudaFree(sweep);
  cudaFree(d_rp);
  cudaFree(d_cp);
  cudaFree(d_ci);
  cudaFree(d_ri);
  cudaFree(d_rv);
  cudaFree(d_cv);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaStreamDestroy(st);
  return 0;
}
