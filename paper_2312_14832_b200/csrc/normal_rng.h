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
#include <condition_variable>
#include <cstdint>
#include <deque>
#include <limits>
#include <mutex>
#include <random>
#include <thread>
#include <vector>

namespace pdhg {

// double(raw) rounded to nearest-even, without the data-dependent branch of
// the compiler's unsigned conversion (half of all draws have bit 63 set):
// above 2^63 the halved value with a sticky low bit rounds identically.
inline double u64_to_double(uint64_t raw) {
  const double lo = static_cast<double>(static_cast<int64_t>(raw));
  const double hi = static_cast<double>(static_cast<int64_t>((raw >> 1) | (raw & 1))) * 2.0;
  return static_cast<int64_t>(raw) >= 0 ? lo : hi;
}

inline double canonical53(uint64_t raw) {
  double r = u64_to_double(raw) / 18446744073709551616.0;  // 2^64
  if (r >= 1.0) r = std::nextafter(1.0, 0.0);
  return r;
}

// std::mt19937_64 (the C++ standard's parameters; libstdc++'s seeding,
// twist and tempering) producing whole blocks: the twist of all 312 words
// and the tempering are plain array loops the compiler vectorises, unlike
// the engine's one-value operator(). Same sequence as std::mt19937_64(seed)
// (tests/test_instances_and_shards.py checks it against the standard engine).
// Twist and tempering as free functions cloned for AVX2 (GCC function
// multiversioning: integer ops only, so every clone is bit-identical).
namespace mt64 {
constexpr int kN = 312, kM = 156;
constexpr uint64_t kA = 0xB5026F5AA96619E9ULL, kUp = ~uint64_t(0) << 31, kLo = ~kUp;

__attribute__((target_clones("avx2", "default"))) static void Temper(const uint64_t* in, uint64_t* out, int n) {
  for (int i = 0; i < n; ++i) {
    uint64_t y = in[i];
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= y >> 43;
    out[i] = y;
  }
}

__attribute__((target_clones("avx2", "default"))) static void Twist(uint64_t* mt) {
  for (int i = 0; i < kN - kM; ++i) {
    const uint64_t y = (mt[i] & kUp) | (mt[i + 1] & kLo);
    mt[i] = mt[i + kM] ^ (y >> 1) ^ ((0 - (y & 1)) & kA);
  }
  for (int i = kN - kM; i < kN - 1; ++i) {
    const uint64_t y = (mt[i] & kUp) | (mt[i + 1] & kLo);
    mt[i] = mt[i + kM - kN] ^ (y >> 1) ^ ((0 - (y & 1)) & kA);
  }
  const uint64_t y = (mt[kN - 1] & kUp) | (mt[0] & kLo);
  mt[kN - 1] = mt[kM - 1] ^ (y >> 1) ^ ((0 - (y & 1)) & kA);
}
}  // namespace mt64

class Mt64Block {
 public:
  explicit Mt64Block(uint64_t seed) {
    mt_[0] = seed;
    for (int i = 1; i < mt64::kN; ++i) mt_[i] = 6364136223846793005ULL * (mt_[i - 1] ^ (mt_[i - 1] >> 62)) + i;
    pos_ = mt64::kN;
  }
  // Next `count` outputs.
  void Fill(uint64_t* out, int64_t count) {
    while (count > 0) {
      if (pos_ == mt64::kN) {
        mt64::Twist(mt_);
        pos_ = 0;
      }
      const int take = static_cast<int>(std::min<int64_t>(count, mt64::kN - pos_));
      mt64::Temper(mt_ + pos_, out, take);
      pos_ += take;
      out += take;
      count -= take;
    }
  }

 private:
  uint64_t mt_[mt64::kN];
  int pos_;
};

inline void NormalVectorSequential(uint64_t seed, int64_t n, double* out) {
  std::mt19937_64 rng(seed);
  std::normal_distribution<double> gauss(0.0, 1.0);
  for (int64_t i = 0; i < n; ++i) out[i] = gauss(rng);
}

// One accepted-attempt transform (random.tcc): y * mult, then x * mult.
inline void PolarEmit(uint64_t r0, uint64_t r1, int64_t k, int64_t n, double* out) {
  const double x = 2.0 * canonical53(r0) - 1.0;
  const double y = 2.0 * canonical53(r1) - 1.0;
  const double r2 = x * x + y * y;
  const double mult = std::sqrt(-2 * std::log(r2) / r2);
  out[2 * k] = y * mult * 1.0 + 0.0;  // __ret * stddev + mean
  if (2 * k + 1 < n) out[2 * k + 1] = x * mult * 1.0 + 0.0;
}

inline bool PolarAccept(uint64_t r0, uint64_t r1) {
  const double x = 2.0 * canonical53(r0) - 1.0;
  const double y = 2.0 * canonical53(r1) - 1.0;
  const double r2 = x * x + y * y;
  return !(r2 > 1.0 || r2 == 0.0);
}

// Pipelined: the calling thread only runs the engine (the one inherently
// sequential part), filling chunks of raw draws in a small ring of
// cache-resident buffers. Workers test acceptance per chunk (publishing the
// chunk's count), wait for the prefix of earlier chunks' counts -- the
// chunk's output base -- and run the log / sqrt transforms. Counting never
// blocks and chunks are taken in order, so the earliest chunk in flight can
// always finish.
inline void NormalVector(uint64_t seed, int64_t n, double* out, int threads) {
  if (threads <= 0) threads = static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
  threads = std::min(threads, 32);
  if (threads == 1 || n < (int64_t(1) << 15)) {
    NormalVectorSequential(seed, n, out);
    return;
  }
  const int64_t need = (n + 1) / 2;  // accepted attempts
  constexpr int kAttempts = 8192;    // per chunk (128 KB of raw draws)
  const int workers = threads - 1;
  const int ring = 4 * workers;
  struct Chunk {
    std::vector<uint64_t> raw;
    std::vector<uint8_t> ok;
  };
  std::vector<Chunk> buf(ring);
  for (Chunk& c : buf) {
    c.raw.resize(2 * kAttempts);
    c.ok.resize(kAttempts);
  }
  std::mutex mu;
  std::condition_variable cv;
  std::deque<std::pair<int64_t, int>> ready;  // (chunk sequence number, ring slot)
  std::deque<int> avail;
  for (int r = 0; r < ring; ++r) avail.push_back(r);
  std::vector<int64_t> count, base{0};  // per chunk; base[c] valid for c < base.size()
  std::vector<char> counted;
  bool done = false;
  std::vector<std::thread> pool;
  for (int t = 0; t < workers; ++t)
    pool.emplace_back([&] {
      while (true) {
        int64_t seq;
        int r;
        {
          std::unique_lock<std::mutex> lk(mu);
          cv.wait(lk, [&] { return done || !ready.empty(); });
          if (ready.empty()) return;
          seq = ready.front().first;
          r = ready.front().second;
          ready.pop_front();
        }
        Chunk& c = buf[r];
        int64_t acc = 0;
        for (int i = 0; i < kAttempts; ++i) acc += c.ok[i] = PolarAccept(c.raw[2 * i], c.raw[2 * i + 1]);
        int64_t k;
        {
          std::unique_lock<std::mutex> lk(mu);
          count[seq] = acc;
          counted[seq] = 1;
          for (size_t q = base.size() - 1; q < counted.size() && counted[q]; ++q) base.push_back(base.back() + count[q]);
          cv.notify_all();
          cv.wait(lk, [&] { return static_cast<int64_t>(base.size()) > seq; });
          k = base[seq];
        }
        for (int i = 0; i < kAttempts && k < need; ++i)
          if (c.ok[i]) PolarEmit(c.raw[2 * i], c.raw[2 * i + 1], k++, n, out);
        {
          std::lock_guard<std::mutex> lk(mu);
          avail.push_back(r);
        }
        cv.notify_all();
      }
    });
  Mt64Block rng(seed);
  // Expected acceptance pi/4; 3% + one chunk of margin, more chunks if short.
  int64_t target = static_cast<int64_t>(need / 0.75) / kAttempts + 2;
  int64_t issued = 0;
  while (true) {
    for (; issued < target; ++issued) {
      int r;
      {
        std::unique_lock<std::mutex> lk(mu);
        cv.wait(lk, [&] { return !avail.empty(); });
        r = avail.front();
        avail.pop_front();
      }
      uint64_t* raw = buf[r].raw.data();
      rng.Fill(raw, 2 * kAttempts);
      {
        std::lock_guard<std::mutex> lk(mu);
        count.push_back(0);
        counted.push_back(0);
        ready.emplace_back(issued, r);
      }
      cv.notify_all();
    }
    std::unique_lock<std::mutex> lk(mu);
    cv.wait(lk, [&] { return static_cast<int64_t>(base.size()) > issued; });
    if (base[issued] >= need) break;
    target += (need - base[issued]) / kAttempts + 2;
  }
  {
    std::lock_guard<std::mutex> lk(mu);
    done = true;
  }
  cv.notify_all();
  for (auto& th : pool) th.join();
}

}  // namespace pdhg
