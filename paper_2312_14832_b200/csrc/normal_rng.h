// Bit-exact, multi-threaded replica of the power-iteration start vector
// (reference solver.cpp:88-97): n draws of std::normal_distribution<double>
// (0, 1) from std::mt19937_64(seed), as libstdc++ 13 computes them.
//
// libstdc++'s normal_distribution is the Marsaglia polar method: every
// attempt consumes exactly two uniforms u = double(raw) / 2^64
// (generate_canonical<double, 53> over a 64-bit engine), x = 2u1 - 1,
// y = 2u2 - 1, r2 = x^2 + y^2, rejected if r2 > 1 or r2 == 0; an accepted
// attempt yields y * mult, then (cached) x * mult, with
// mult = sqrt(-2 log(r2) / r2) (random.tcc, normal_distribution::operator()).
// Attempt i therefore always uses raw draws 2i and 2i+1, so after the
// (sequential, cheap) raw engine stream is materialised, acceptance, the
// output index (a prefix count of accepted attempts) and the log/sqrt
// transform are all parallel -- and, computed with the same glibc log/sqrt
// and no FMA contraction, bit-identical to the sequential draw.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <limits>
#include <random>
#include <thread>
#include <vector>

namespace pdhg {

inline double canonical53(uint64_t raw) {
  double r = static_cast<double>(raw) / 18446744073709551616.0;  // 2^64
  if (r >= 1.0) r = std::nextafter(1.0, 0.0);
  return r;
}

inline void NormalVectorSequential(uint64_t seed, int64_t n, double* out) {
  std::mt19937_64 rng(seed);
  std::normal_distribution<double> gauss(0.0, 1.0);
  for (int64_t i = 0; i < n; ++i) out[i] = gauss(rng);
}

inline void NormalVector(uint64_t seed, int64_t n, double* out, int threads) {
  if (threads <= 0) threads = static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
  if (threads == 1 || n < (int64_t(1) << 15)) {
    NormalVectorSequential(seed, n, out);
    return;
  }
  const int64_t need = (n + 1) / 2;  // accepted attempts
  std::mt19937_64 rng(seed);
  std::vector<uint64_t> raw;
  std::vector<uint8_t> ok;
  int64_t attempts = 0;
  auto parallel = [&](int64_t count, auto&& fn) {  // fn(chunk, begin, end)
    std::vector<std::thread> pool;
    const int64_t per = (count + threads - 1) / threads;
    for (int t = 0; t < threads; ++t) {
      const int64_t b = std::min(count, t * per), e = std::min(count, b + per);
      pool.emplace_back([&fn, t, b, e] { fn(t, b, e); });
    }
    for (auto& th : pool) th.join();
  };
  std::vector<int64_t> counts(threads);
  int64_t accepted = 0;
  while (true) {
    // Expected acceptance pi/4; a 3% + 4096 margin almost always suffices.
    const int64_t want = attempts + static_cast<int64_t>((need - accepted) / 0.75) + 4096;
    raw.resize(2 * want);
    for (int64_t k = 2 * attempts; k < 2 * want; ++k) raw[k] = rng();
    attempts = want;
    ok.assign(attempts, 0);
    parallel(attempts, [&](int t, int64_t b, int64_t e) {
      int64_t c = 0;
      for (int64_t i = b; i < e; ++i) {
        const double x = 2.0 * canonical53(raw[2 * i]) - 1.0;
        const double y = 2.0 * canonical53(raw[2 * i + 1]) - 1.0;
        const double r2 = x * x + y * y;
        ok[i] = !(r2 > 1.0 || r2 == 0.0);
        c += ok[i];
      }
      counts[t] = c;
    });
    accepted = 0;
    for (int64_t c : counts) accepted += c;
    if (accepted >= need) break;
  }
  std::vector<int64_t> base(threads, 0);
  for (int t = 1; t < threads; ++t) base[t] = base[t - 1] + counts[t - 1];
  parallel(attempts, [&](int t, int64_t b, int64_t e) {
    int64_t k = base[t];
    for (int64_t i = b; i < e && k < need; ++i) {
      if (!ok[i]) continue;
      const double x = 2.0 * canonical53(raw[2 * i]) - 1.0;
      const double y = 2.0 * canonical53(raw[2 * i + 1]) - 1.0;
      const double r2 = x * x + y * y;
      const double mult = std::sqrt(-2 * std::log(r2) / r2);
      out[2 * k] = y * mult * 1.0 + 0.0;  // __ret * stddev + mean
      if (2 * k + 1 < n) out[2 * k + 1] = x * mult * 1.0 + 0.0;
      ++k;
    }
  });
}

}  // namespace pdhg
