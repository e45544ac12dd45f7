// Calibration microbenchmark (not product code): what a random-gather sparse
// pass can reach on this B200, independent of the PDHG kernels.
//
// An 8-byte gather of a vector entry costs a 32-byte L2 sector, so a pass
// whose column indices are scattered is bounded by L2 sector throughput (and,
// when the gathered vector does not stay L2-resident, by the DRAM re-reads of
// its sectors), not by the stream bytes HBM moves. This probe measures:
//   seq     streaming read of the (idx, val) arrays only -- the HBM stream rate;
//   gather  a uniform-length (L entries per segment) sparse pass, thread per
//           segment, random column indices uniform over a vector of S doubles,
//           storage-order sum, one store per segment: the cost of the
//           SpMV alone with the same nnz / vector size as an instance;
//   l2cap   random 8-byte gathers from an L2-resident 8 MB vector with no
//           stream (indices from a hash): the L2 sector-throughput ceiling.
// Every timing: CUDA events, L2 flushed (256 MB write) before each launch,
// median of 7.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/_build/gather_probe tools/gather_probe.cu
//   tools/_build/gather_probe [nnz_millions]
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                               \
  do {                                                                                      \
    cudaError_t e = (x);                                                                    \
    if (e != cudaSuccess) {                                                                 \
      std::fprintf(stderr, "%s: %s (%s:%d)\n", #x, cudaGetErrorString(e), __FILE__, __LINE__); \
      std::exit(1);                                                                         \
    }                                                                                       \
  } while (0)

__host__ __device__ inline uint32_t mix(uint64_t k) {
  k ^= k >> 33;
  k *= 0xff51afd7ed558ccdull;
  k ^= k >> 33;
  k *= 0xc4ceb9fe1a85ec53ull;
  k ^= k >> 33;
  return static_cast<uint32_t>(k);
}

__global__ void k_fill_idx(int32_t* idx, int64_t nnz, uint32_t S, uint64_t seed) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nnz; i += (int64_t)gridDim.x * blockDim.x)
    idx[i] = static_cast<int32_t>(mix(i * 0x9E3779B97F4A7C15ull + seed) % S);
}
__global__ void k_fill(double* a, int64_t n, double v) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    a[i] = v + 1e-9 * static_cast<double>(i & 1023);
}

// Streaming read of idx + val (the matrix stream of a pass), 16-byte loads.
__global__ void k_seq(const int4* __restrict__ idx, const double2* __restrict__ val, int64_t n4, double* out) {
  double acc = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    const int4 j = __ldcs(idx + i);
    const double2 a = __ldcs(val + 2 * i), b = __ldcs(val + 2 * i + 1);
    acc += a.x + a.y + b.x + b.y + static_cast<double>(j.x ^ j.y ^ j.z ^ j.w);
  }
  if (acc == 123.456) out[0] = acc;
}

// Thread per segment of L entries (offsets implicit), storage-order sum.
template <int L>
__global__ void __launch_bounds__(256) k_gather(const int32_t* __restrict__ idx, const double* __restrict__ val,
                                                const double* __restrict__ x, int64_t nseg, double* __restrict__ y) {
  const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s >= nseg) return;
  int32_t j[L];
  double v[L];
#pragma unroll
  for (int u = 0; u < L; ++u) {
    j[u] = __ldcs(idx + s * L + u);
    v[u] = __ldcs(val + s * L + u);
  }
  double acc = 0.0;
#pragma unroll
  for (int u = 0; u < L; ++u) acc += v[u] * x[j[u]];
  __stcs(y + s, acc);
}

// Random gathers from x[0, S) with hashed indices, G per thread in flight.
template <int G>
__global__ void __launch_bounds__(256) k_l2cap(const double* __restrict__ x, uint32_t S, int64_t nthreads,
                                               double* out, uint64_t seed) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= nthreads) return;
  double acc = 0.0;
  double v[G];
#pragma unroll
  for (int g = 0; g < G; ++g) v[g] = x[mix(t * G + g + seed) % S];
#pragma unroll
  for (int g = 0; g < G; ++g) acc += v[g];
  if (acc == 123.456) out[0] = acc;
}

struct Timer {
  cudaEvent_t a, b;
  Timer() {
    cudaEventCreate(&a);
    cudaEventCreate(&b);
  }
};

int main(int argc, char** argv) {
  const int64_t nnz = static_cast<int64_t>((argc > 1 ? std::atof(argv[1]) : 80.0) * 1e6) / 8 * 8;
  const int64_t flush_n = (256ll << 20) / 8;
  double *flush, *val, *x, *y, *out;
  int32_t* idx;
  const uint32_t smax = 64u << 20;  // up to 512 MB vectors
  CK(cudaMalloc(&flush, flush_n * 8));
  CK(cudaMalloc(&val, nnz * 8));
  CK(cudaMalloc(&idx, nnz * 4));
  CK(cudaMalloc(&x, static_cast<size_t>(smax) * 8));
  CK(cudaMalloc(&y, nnz / 1 * 8 / 1));
  CK(cudaMalloc(&out, 8));
  k_fill<<<148 * 8, 256>>>(val, nnz, 0.5);
  k_fill<<<148 * 8, 256>>>(x, smax, 1.0);
  CK(cudaDeviceSynchronize());
  Timer tm;
  auto time = [&](auto&& launch) {
    std::vector<float> ms;
    for (int r = 0; r < 8; ++r) {
      k_fill<<<148 * 8, 256>>>(flush, flush_n, 2.0);  // evict L2
      cudaEventRecord(tm.a);
      launch();
      cudaEventRecord(tm.b);
      CK(cudaEventSynchronize(tm.b));
      float t;
      cudaEventElapsedTime(&t, tm.a, tm.b);
      if (r) ms.push_back(t);
    }
    std::sort(ms.begin(), ms.end());
    return ms[ms.size() / 2] * 1e-3;
  };
  int dev;
  cudaDeviceProp pr;
  CK(cudaGetDevice(&dev));
  CK(cudaGetDeviceProperties(&pr, dev));
  std::printf("{\"device\": \"%s\", \"sms\": %d, \"nnz\": %lld}\n", pr.name, pr.multiProcessorCount, (long long)nnz);
  {
    const double s = time([&] { k_seq<<<148 * 16, 256>>>((const int4*)idx, (const double2*)val, nnz / 4, out); });
    std::printf("{\"probe\": \"seq\", \"us\": %.1f, \"GBps\": %.0f}\n", s * 1e6, nnz * 12.0 / s / 1e9);
  }
  for (uint32_t S : {1u << 20, 4u << 20, 5u << 20, 6u << 20, 7u << 20, 8u << 20, 9u << 20, 10u << 20, 16u << 20, 64u << 20}) {
    k_fill_idx<<<148 * 8, 256>>>(idx, nnz, S, 12345);
    CK(cudaDeviceSynchronize());
    for (int L : {8}) {
      const int64_t nseg = nnz / L;
      const double s = time([&] {
        if (L == 8) k_gather<8><<<(nseg + 255) / 256, 256>>>(idx, val, x, nseg, y);
        else k_gather<20><<<(nseg + 255) / 256, 256>>>(idx, val, x, nseg, y);
      });
      const double bytes = nnz * 12.0 + nseg * 8.0 + std::min<double>(S, nnz) * 8.0;  // stream + out + x once
      std::printf(
          "{\"probe\": \"gather\", \"L\": %d, \"vec_MB\": %.0f, \"us\": %.1f, \"Ggather_per_s\": %.2f, "
          "\"alg_GBps\": %.0f, \"sector_GBps\": %.0f}\n",
          L, S * 8.0 / 1e6, s * 1e6, nnz / s / 1e9, bytes / s / 1e9, (nnz * 44.0 + nseg * 8.0) / s / 1e9);
    }
  }
  for (uint32_t S : {1u << 20, 8u << 20}) {
    const int64_t nt = 148ll * 2048 * 64;
    const double s = time([&] { k_l2cap<8><<<(nt + 255) / 256, 256>>>(x, S, nt, out, 7); });
    std::printf("{\"probe\": \"l2cap\", \"vec_MB\": %.0f, \"us\": %.1f, \"Ggather_per_s\": %.2f, \"sector_GBps\": %.0f}\n",
                S * 8.0 / 1e6, s * 1e6, nt * 8.0 / s / 1e9, nt * 8.0 * 32.0 / s / 1e9);
  }
  return 0;
}
