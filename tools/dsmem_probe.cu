// Calibration microbenchmark (not product code): random 8-byte gathers from a
// 1.6 MB window of a vector, served by
//   l2     the window in global memory (L2-resident: every CTA gathers from it);
//   dsmem  the window split over the shared memory of an 8-CTA cluster
//          (200 KB per CTA), read with ld.shared::cluster through mapa;
//   smem   the CTA's own 200 KB slice only (local shared memory).
// The question it answers: can a block-structured LP's row pass (rows whose
// columns fall in one 200k-entry window, like a staircase stage) gather from
// distributed shared memory faster than from L2, whose random-gather ceiling
// on this B200 is ~287 G gathers/s (tools/gather_probe.cu)?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/_build/dsmem_probe tools/dsmem_probe.cu
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <vector>

namespace cg = cooperative_groups;

#define CK(x)                                                                                   \
  do {                                                                                          \
    cudaError_t e = (x);                                                                        \
    if (e != cudaSuccess) {                                                                     \
      std::fprintf(stderr, "%s: %s (%s:%d)\n", #x, cudaGetErrorString(e), __FILE__, __LINE__); \
      return 1;                                                                                 \
    }                                                                                           \
  } while (0)

constexpr int kCl = 8;                   // CTAs per cluster
constexpr int kSlice = 25600;            // doubles per CTA (200 KB)
constexpr int kWin = kCl * kSlice;       // 204800 doubles = 1.6 MB
constexpr int kG = 8;                    // gathers in flight per thread per round

__device__ __forceinline__ uint32_t mix(uint32_t k) {
  k ^= k >> 16;
  k *= 0x7feb352dU;
  k ^= k >> 15;
  k *= 0x846ca68bU;
  k ^= k >> 16;
  return k;
}

template <int MODE>  // 0 l2, 1 dsmem, 2 smem
__global__ void __cluster_dims__(kCl, 1, 1) __launch_bounds__(1024, 1)
    k_gather(const double* __restrict__ win, int rounds, double* out) {
  extern __shared__ double sl[];
  cg::cluster_group cl = cg::this_cluster();
  const int rank = static_cast<int>(cl.block_rank());
  if (MODE != 0) {
    for (int i = threadIdx.x; i < kSlice; i += blockDim.x) sl[i] = win[rank * kSlice + i];
    cl.sync();
  }
  uint32_t h = (blockIdx.x * blockDim.x + threadIdx.x) * 2654435761u;
  double acc = 0.0;
  for (int r = 0; r < rounds; ++r) {
    double v[kG];
#pragma unroll
    for (int g = 0; g < kG; ++g) {
      h = mix(h + g + 1);
      if (MODE == 0) {
        v[g] = win[h % kWin];
      } else if (MODE == 1) {
        const uint32_t j = h % kWin;
        const double* p = cl.map_shared_rank(sl, j / kSlice);
        v[g] = p[j % kSlice];
      } else {
        v[g] = sl[h % kSlice];
      }
    }
#pragma unroll
    for (int g = 0; g < kG; ++g) acc += v[g];
  }
  if (MODE != 0) cl.sync();
  if (acc == 1.2345) out[0] = acc;
}

// Sequential L2-resident reads: a 32 MB buffer read `reps` times (grid-stride,
// 16-byte loads) -- the L2 read bandwidth a streaming pass sees when its
// working set stays in L2 (transport's 96 MB per iteration mostly does).
__global__ void __launch_bounds__(256) k_l2seq(const double2* __restrict__ a, int64_t n2, int reps, double* out) {
  double acc = 0.0;
  for (int r = 0; r < reps; ++r)
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n2; i += (int64_t)gridDim.x * blockDim.x) {
      const double2 v = a[i];
      acc += v.x + v.y;
    }
  if (acc == 1.2345) out[0] = acc;
}

int main() {
  double *win, *out;
  CK(cudaMalloc(&win, kWin * sizeof(double)));
  CK(cudaMalloc(&out, 8));
  std::vector<double> h(kWin, 1.0);
  CK(cudaMemcpy(win, h.data(), kWin * sizeof(double), cudaMemcpyHostToDevice));
  const int smem = kSlice * sizeof(double);
  CK(cudaFuncSetAttribute(k_gather<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  CK(cudaFuncSetAttribute(k_gather<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  CK(cudaFuncSetAttribute(k_gather<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int rounds = 512;
  for (int threads : {256, 1024}) {
    const int grid = (sms / kCl) * kCl * 2;  // two waves of clusters
    for (int mode = 0; mode < 3; ++mode) {
      auto launch = [&] {
        if (mode == 0) k_gather<0><<<grid, threads, smem>>>(win, rounds, out);
        if (mode == 1) k_gather<1><<<grid, threads, smem>>>(win, rounds, out);
        if (mode == 2) k_gather<2><<<grid, threads, smem>>>(win, rounds, out);
      };
      launch();
      CK(cudaGetLastError());
      CK(cudaDeviceSynchronize());
      std::vector<float> t;
      for (int r = 0; r < 5; ++r) {
        cudaEventRecord(a);
        launch();
        cudaEventRecord(b);
        CK(cudaEventSynchronize(b));
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        t.push_back(ms);
      }
      std::sort(t.begin(), t.end());
      const double g = static_cast<double>(grid) * threads * rounds * kG;
      std::printf("{\"mode\": \"%s\", \"threads\": %d, \"grid\": %d, \"ms\": %.3f, \"Ggather_per_s\": %.1f}\n",
                  mode == 0 ? "l2" : (mode == 1 ? "dsmem" : "smem"), threads, grid, t[2], g / (t[2] * 1e-3) / 1e9);
    }
  }
  {
    const int64_t n2 = (32ll << 20) / 16;
    double2* buf;
    CK(cudaMalloc(&buf, n2 * 16));
    CK(cudaMemset(buf, 0, n2 * 16));
    for (int reps : {1, 20}) {
      k_l2seq<<<sms * 8, 256>>>(buf, n2, reps, out);
      CK(cudaDeviceSynchronize());
      std::vector<float> t;
      for (int r = 0; r < 5; ++r) {
        cudaEventRecord(a);
        k_l2seq<<<sms * 8, 256>>>(buf, n2, reps, out);
        cudaEventRecord(b);
        CK(cudaEventSynchronize(b));
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        t.push_back(ms);
      }
      std::sort(t.begin(), t.end());
      std::printf("{\"mode\": \"l2seq\", \"MB\": 32, \"reps\": %d, \"ms\": %.4f, \"GBps\": %.0f}\n", reps, t[2],
                  n2 * 16.0 * reps / (t[2] * 1e-3) / 1e9);
    }
  }
  return 0;
}
