// Host-side instance builders (input construction, off the solve path).
//
// GenRandomLp and GenPagerank restate the reference generators
// (proj/core/src/instance_gen.cpp:27-64, 90-141, 143-188) draw for draw with
// the same libstdc++ engines, so instances are bit-identical per seed
// (pinned by tests/test_generators.py against the reference build and the
// committed golden checksums). Matrices go through a FromTriplets
// equivalent (sparse_matrix.cpp:25-69: sort by (row, col), sum duplicates,
// drop zeros). The transportation generator is new.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <limits>
#include <random>
#include <stdexcept>
#include <string>
#include <thread>
#include <tuple>
#include <vector>

#include "../../include/pdhg.h"
#include "instance.h"

namespace {

using I = int64_t;

struct Trip {
  I row, col;
  double v;
};

// FromTriplets (sparse_matrix.cpp:25-69) into CSR arrays; >= 2^20 triplets
// are assembled on the device when one is present (pdhg_csr_from_triplets;
// the generators' duplicates -- repeated PageRank edges -- carry equal
// values, so the stable device order sums them to the same bits). The host
// std::sort path runs without a GPU and for PDHG_ORDER_DEPENDENT inputs;
// other device failures are thrown.
void FromTriplets(I rows, std::vector<Trip> t, std::vector<I>* ptr, std::vector<I>* idx, std::vector<double>* val,
                  I cols) {
  static_assert(sizeof(Trip) == sizeof(pdhg_triplet), "Trip layout");
  const char* da = std::getenv("PDHG_DEVICE_ASSEMBLY");  // "0": host only (A/B, tests)
  if (t.size() >= (size_t(1) << 20) && !(da && da[0] == '0') && pdhg_device_count() > 0) {
    const char* dv = std::getenv("PDHG_DEVICE");
    ptr->assign(rows + 1, 0);
    idx->resize(t.size());
    val->resize(t.size());
    int64_t nnz = 0;
    char err[256] = {0};
    const int rc = pdhg_csr_from_triplets(rows, cols, static_cast<int64_t>(t.size()),
                                          reinterpret_cast<const pdhg_triplet*>(t.data()), dv ? std::atoi(dv) : 0,
                                          ptr->data(), idx->data(), val->data(), &nnz, err, sizeof(err));
    if (rc == PDHG_OK) {
      idx->resize(nnz);
      val->resize(nnz);
      return;
    }
    if (rc != PDHG_ORDER_DEPENDENT) throw std::runtime_error(std::string("device triplet assembly: ") + err);
  }
  std::sort(t.begin(), t.end(),
            [](const Trip& a, const Trip& b) { return std::tie(a.row, a.col) < std::tie(b.row, b.col); });
  ptr->assign(rows + 1, 0);
  idx->clear();
  val->clear();
  idx->reserve(t.size());
  val->reserve(t.size());
  size_t i = 0;
  while (i < t.size()) {
    const I r = t[i].row, c = t[i].col;
    double v = 0.0;
    while (i < t.size() && t[i].row == r && t[i].col == c) v += t[i++].v;
    if (v != 0.0) {
      idx->push_back(c);
      val->push_back(v);
      ++(*ptr)[r + 1];
    }
  }
  for (I r = 0; r < rows; ++r) (*ptr)[r + 1] += (*ptr)[r];
}

// Row-sequential host product, only for building right-hand sides.
void CsrMul(const std::vector<I>& p, const std::vector<I>& j, const std::vector<double>& v, const double* x, I rows,
            double* y) {
  for (I r = 0; r < rows; ++r) {
    double acc = 0.0;
    for (I k = p[r]; k < p[r + 1]; ++k) acc += v[k] * x[j[k]];
    y[r] = acc;
  }
}

pdhg_instance* RandomLp(I m, I n, double density, uint64_t seed) {
  if (m < 1 || n < 1) throw std::invalid_argument("m and n must be >= 1");
  if (!(density > 0.0 && density <= 1.0)) throw std::invalid_argument("density must lie in (0, 1]");
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> unit(0.0, 1.0);
  std::uniform_real_distribution<double> sym(-1.0, 1.0);
  auto* p = new pdhg_instance;
  p->n = n;
  p->witness.resize(n);
  for (double& v : p->witness) v = unit(rng);
  std::vector<Trip> t;
  for (I i = 0; i < m; ++i) {
    I row_nnz = 0;
    for (I j = 0; j < n; ++j) {
      if (unit(rng) < density) {
        t.push_back({i, j, sym(rng)});
        ++row_nnz;
      }
    }
    if (row_nnz == 0) {
      const I j = static_cast<I>(rng() % static_cast<uint64_t>(n));
      t.push_back({i, j, sym(rng)});
    }
  }
  p->g_rows = m;
  FromTriplets(m, std::move(t), &p->g_ptr, &p->g_idx, &p->g_val, n);
  std::vector<double> gx(m);
  CsrMul(p->g_ptr, p->g_idx, p->g_val, p->witness.data(), m, gx.data());
  p->h.resize(m);
  for (I i = 0; i < m; ++i) p->h[i] = gx[i] - std::abs(0.3 * sym(rng));
  p->c.resize(n);
  for (double& v : p->c) v = sym(rng);
  p->l.assign(n, 0.0);
  p->u.assign(n, 1.0);
  return p;
}

// GenPagerankGraph (instance_gen.cpp:27-64): preferential attachment over a
// pool where node j appears in_degree(j) + 1 times, seeded by a directed
// cycle over the first attachment + 1 nodes. Deterministic per seed.
std::vector<std::pair<I, I>> PagerankGraph(I n_nodes, double damping, I attachment, uint64_t seed) {
  if (n_nodes < attachment + 1) throw std::invalid_argument("n_nodes must be at least attachment + 1");
  if (!(damping > 0.0 && damping < 1.0)) throw std::invalid_argument("damping must lie in (0, 1)");
  std::mt19937_64 rng(seed);
  std::vector<std::pair<I, I>> edges;
  edges.reserve(static_cast<size_t>(n_nodes * attachment));
  const I core = attachment + 1;
  for (I i = 0; i < core; ++i) edges.push_back({i, (i + 1) % core});
  std::vector<I> pool;
  pool.reserve(2 * static_cast<size_t>(n_nodes * attachment));
  for (I i = 0; i < core; ++i) pool.push_back(i);
  for (auto& e : edges) pool.push_back(e.second);
  std::vector<I> targets;
  for (I i = core; i < n_nodes; ++i) {
    targets.clear();
    while (static_cast<I>(targets.size()) < attachment) {
      std::uniform_int_distribution<size_t> dist(0, pool.size() - 1);
      const I pick = pool[dist(rng)];
      if (std::find(targets.begin(), targets.end(), pick) == targets.end()) targets.push_back(pick);
    }
    for (I t : targets) {
      edges.push_back({i, t});
      pool.push_back(t);
    }
    pool.push_back(i);
  }
  return edges;
}

// BuildPagerankLp (instance_gen.cpp:90-137): x_i - damping * sum_j S_ij x_j
// >= (1 - damping) / n per node (G), sum(x) = 1 (A), x >= 0, c = 0; dangling
// nodes get a self-loop so S stays column-stochastic.
pdhg_instance* PagerankLp(const std::pair<I, I>* edges, size_t count, I n_nodes, double damping) {
  if (n_nodes < 1) throw std::invalid_argument("empty graph");
  std::vector<I> outdeg(n_nodes, 0);
  for (size_t k = 0; k < count; ++k) {
    const auto& e = edges[k];
    if (e.first < 0 || e.first >= n_nodes || e.second < 0 || e.second >= n_nodes)
      throw std::invalid_argument("edge endpoint out of range");
    ++outdeg[e.first];
  }
  std::vector<I> dangling;
  for (I j = 0; j < n_nodes; ++j)
    if (outdeg[j] == 0) {
      dangling.push_back(j);
      outdeg[j] = 1;
    }
  std::vector<Trip> t;
  t.reserve(count + 2 * static_cast<size_t>(n_nodes));
  for (I i = 0; i < n_nodes; ++i) t.push_back({i, i, 1.0});
  for (size_t k = 0; k < count; ++k) t.push_back({edges[k].second, edges[k].first, -damping / outdeg[edges[k].first]});
  for (I j : dangling) t.push_back({j, j, -damping});
  auto* p = new pdhg_instance;
  p->n = n_nodes;
  p->g_rows = n_nodes;
  FromTriplets(n_nodes, std::move(t), &p->g_ptr, &p->g_idx, &p->g_val, n_nodes);
  p->h.assign(n_nodes, (1.0 - damping) / static_cast<double>(n_nodes));
  p->a_rows = 1;
  p->a_ptr = {0, n_nodes};
  p->a_idx.resize(n_nodes);
  for (I j = 0; j < n_nodes; ++j) p->a_idx[j] = j;
  p->a_val.assign(n_nodes, 1.0);
  p->b = {1.0};
  p->c.assign(n_nodes, 0.0);
  p->l.assign(n_nodes, 0.0);
  p->u.assign(n_nodes, std::numeric_limits<double>::infinity());
  return p;
}

pdhg_instance* Pagerank(I n_nodes, double damping, I attachment, uint64_t seed) {
  std::vector<std::pair<I, I>> edges = PagerankGraph(n_nodes, damping, attachment, seed);
  return PagerankLp(edges.data(), edges.size(), n_nodes, damping);
}

// Transportation LP. Variables x_ij, index i*T + j.
// Draw order: demands d_j, supplies s_i, then costs c_ij row-major.
pdhg_instance* Transport(I S, I T, uint64_t seed) {
  if (S < 1 || T < 1) throw std::invalid_argument("sources and sinks must be >= 1");
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> unit(0.0, 1.0);
  std::vector<double> d(T), s(S);
  double sd = 0.0, ss = 0.0;
  for (double& v : d) {
    v = 1.0 + unit(rng);
    sd += v;
  }
  for (double& v : s) {
    v = 1.0 + unit(rng);
    ss += v;
  }
  const double f = 1.2 * sd / ss;
  for (double& v : s) v *= f;
  auto* p = new pdhg_instance;
  const I n = S * T;
  p->n = n;
  p->c.resize(n);
  for (double& v : p->c) v = unit(rng);
  // A: demand rows (= d_j), row j holds x_ij for every source i.
  p->a_rows = T;
  p->a_ptr.resize(T + 1);
  p->a_idx.resize(n);
  p->a_val.assign(n, 1.0);
  for (I j = 0; j <= T; ++j) p->a_ptr[j] = j * S;
  for (I j = 0; j < T; ++j)
    for (I i = 0; i < S; ++i) p->a_idx[j * S + i] = i * T + j;
  p->b = d;
  // G: supply rows -sum_j x_ij >= -s_i.
  p->g_rows = S;
  p->g_ptr.resize(S + 1);
  p->g_idx.resize(n);
  p->g_val.assign(n, -1.0);
  for (I i = 0; i <= S; ++i) p->g_ptr[i] = i * T;
  for (I k = 0; k < n; ++k) p->g_idx[k] = k;
  p->h.resize(S);
  for (I i = 0; i < S; ++i) p->h[i] = -s[i];
  p->l.assign(n, 0.0);
  p->u.assign(n, std::numeric_limits<double>::infinity());
  return p;
}

// Multicommodity network flow LP. A power-law digraph
// of V nodes and E arcs (tail and head drawn from Zipf-like node weights
// w_v = (v + 1)^-0.8, self-loops redrawn), K commodities, variables
// x_{a,k} at column a*K + k, x >= 0, costs U(0,1).
//   A: conservation row k*V + v:  sum_{a out of v} x_{a,k} - sum_{a into v} x_{a,k} = b
//   G: capacity row a:            -sum_k x_{a,k} >= -cap_a
// Feasible by construction: a random witness flow (each x_{a,k} nonzero with
// probability 0.2, value U(0,1)) gives b = A x_hat and
// cap_a = 1.1 * sum_k x_hat_{a,k} + 0.1 U(0,1). Conservation row lengths are
// node degrees (heavy-tailed), capacity rows hold K, every column exactly 3.
// Draw order: arcs (tail, head), witness row-major over (a, k), capacity
// slack per arc, costs row-major over (a, k).
pdhg_instance* Mcf(I V, I E, I K, uint64_t seed) {
  if (V < 2 || E < 1 || K < 1) throw std::invalid_argument("need V >= 2, E >= 1, K >= 1");
  if (E * K >= (I(1) << 31) || 3 * E * K >= (I(1) << 31) - 4096)
    throw std::invalid_argument("instance too large for int32 device indices");
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> unit(0.0, 1.0);
  std::vector<double> cdf(V);
  double acc = 0.0;
  for (I v = 0; v < V; ++v) {
    acc += std::pow(static_cast<double>(v + 1), -0.8);
    cdf[v] = acc;
  }
  auto draw = [&]() -> I {
    const double r = unit(rng) * acc;
    const I v = static_cast<I>(std::upper_bound(cdf.begin(), cdf.end(), r) - cdf.begin());
    return std::min(v, V - 1);
  };
  std::vector<I> tail(E), head(E);
  for (I a = 0; a < E; ++a) {
    tail[a] = draw();
    do head[a] = draw();
    while (head[a] == tail[a]);
  }
  const I n = E * K;
  auto* p = new pdhg_instance;
  p->n = n;
  p->witness.assign(n, 0.0);
  for (I k = 0; k < n; ++k)
    if (unit(rng) < 0.2) p->witness[k] = unit(rng);
  // Incidence lists per node, arcs ascending (so columns ascend in each row).
  std::vector<I> deg(V + 1, 0);
  for (I a = 0; a < E; ++a) {
    ++deg[tail[a] + 1];
    ++deg[head[a] + 1];
  }
  for (I v = 0; v < V; ++v) deg[v + 1] += deg[v];
  std::vector<I> inc(2 * E), fill(deg.begin(), deg.end() - 1);
  for (I a = 0; a < E; ++a) {  // ascending a -> each list sorted
    inc[fill[tail[a]]++] = a;
    inc[fill[head[a]]++] = a;
  }
  p->a_rows = V * K;
  p->a_ptr.resize(V * K + 1);
  p->a_idx.resize(2 * n);
  p->a_val.resize(2 * n);
  p->b.assign(V * K, 0.0);
  I w = 0;
  for (I k = 0; k < K; ++k) {
    for (I v = 0; v < V; ++v) {
      p->a_ptr[k * V + v] = w;
      double bv = 0.0;
      for (I e = deg[v]; e < deg[v + 1]; ++e) {
        const I a = inc[e];
        const double s = tail[a] == v ? 1.0 : -1.0;
        p->a_idx[w] = a * K + k;
        p->a_val[w] = s;
        bv += s * p->witness[a * K + k];
        ++w;
      }
      p->b[k * V + v] = bv;
    }
  }
  p->a_ptr[V * K] = w;
  p->g_rows = E;
  p->g_ptr.resize(E + 1);
  p->g_idx.resize(n);
  p->g_val.assign(n, -1.0);
  p->h.resize(E);
  for (I a = 0; a < E; ++a) {
    double flow = 0.0;
    for (I k = 0; k < K; ++k) {
      p->g_idx[a * K + k] = a * K + k;
      flow += p->witness[a * K + k];
    }
    p->g_ptr[a] = a * K;
    p->h[a] = -(1.1 * flow + 0.1 * unit(rng));
  }
  p->g_ptr[E] = n;
  p->c.resize(n);
  for (double& v : p->c) v = unit(rng);
  p->l.assign(n, 0.0);
  p->u.assign(n, std::numeric_limits<double>::infinity());
  return p;
}

// Block-angular staircase LP. T stages of R rows and C
// columns; every row holds exactly D nonzeros U(-1,1): D - Dl in its own
// stage's columns and Dl linking ones in stage t-1's (stage 0: all D own).
// The first Req rows of each stage are equalities (A, b = row . x_hat), the
// rest inequalities (G, h = row . x_hat - |0.3 U(-1,1)|); x_hat ~ U(0,1),
// 0 <= x <= 2, c ~ U(-1,1). Stages are generated in parallel, each from its
// own engine mt19937_64(seed ^ (0x9E3779B97F4A7C15 * (t + 1))) (witness and
// costs of stage t first, then its rows), so the instance is bit-identical
// per seed for any thread count. Row layouts are fixed-length, so every
// thread writes its slice of the final CSR arrays in place.
pdhg_instance* Staircase(I T, I R, I C, I D, I Dl, I Req, uint64_t seed, int threads) {
  if (T < 1 || R < 1 || C < 1 || D < 1) throw std::invalid_argument("T, R, C, D must be >= 1");
  if (Dl < 0 || Dl >= D || D - Dl > C || Dl > C) throw std::invalid_argument("need 0 <= Dl < D, D - Dl <= C, Dl <= C");
  if (Req < 0 || Req > R) throw std::invalid_argument("need 0 <= Req <= R");
  const I n = T * C, rows = T * R;
  if (rows * D >= (I(1) << 31) - 4096 || n >= (I(1) << 31) - 1)
    throw std::invalid_argument("instance too large for int32 device indices");
  auto* p = new pdhg_instance;
  p->n = n;
  p->a_rows = T * Req;
  p->g_rows = T * (R - Req);
  p->a_ptr.resize(p->a_rows + 1);
  p->g_ptr.resize(p->g_rows + 1);
  for (I r = 0; r <= p->a_rows; ++r) p->a_ptr[r] = r * D;
  for (I r = 0; r <= p->g_rows; ++r) p->g_ptr[r] = r * D;
  p->a_idx.resize(p->a_rows * D);
  p->a_val.resize(p->a_rows * D);
  p->g_idx.resize(p->g_rows * D);
  p->g_val.resize(p->g_rows * D);
  p->b.resize(p->a_rows);
  p->h.resize(p->g_rows);
  p->witness.resize(n);
  p->c.resize(n);
  p->l.assign(n, 0.0);
  p->u.assign(n, 2.0);
  auto engine = [&](I t) { return std::mt19937_64(seed ^ (0x9E3779B97F4A7C15ull * static_cast<uint64_t>(t + 1))); };
  // Pass 1: witness + costs per stage (rows of stage t read stage t-1's x_hat).
  std::vector<std::mt19937_64> eng;
  eng.reserve(T);
  for (I t = 0; t < T; ++t) eng.push_back(engine(t));
  auto stage_vec = [&](I t) {
    std::uniform_real_distribution<double> unit(0.0, 1.0), sym(-1.0, 1.0);
    for (I j = t * C; j < (t + 1) * C; ++j) p->witness[j] = unit(eng[t]);
    for (I j = t * C; j < (t + 1) * C; ++j) p->c[j] = sym(eng[t]);
  };
  auto stage_rows = [&](I t) {
    std::mt19937_64& g = eng[t];
    std::uniform_real_distribution<double> sym(-1.0, 1.0);
    std::vector<I> cols;
    for (I i = 0; i < R; ++i) {
      const I dl = t > 0 ? Dl : 0, dn = D - dl;
      cols.clear();
      auto pick = [&](I lo, I cnt, I span) {
        std::uniform_int_distribution<I> dist(lo, lo + span - 1);
        const size_t base = cols.size();
        while (static_cast<I>(cols.size() - base) < cnt) {
          const I j = dist(g);
          if (std::find(cols.begin() + base, cols.end(), j) == cols.end()) cols.push_back(j);
        }
      };
      pick((t - 1) * C, dl, C);  // linking columns (stage t-1) come first: ascending
      pick(t * C, dn, C);
      std::sort(cols.begin(), cols.begin() + dl);
      std::sort(cols.begin() + dl, cols.end());
      const bool eq = i < Req;
      const I row = eq ? t * Req + i : t * (R - Req) + (i - Req);
      int64_t* idx = (eq ? p->a_idx.data() : p->g_idx.data()) + row * D;
      double* val = (eq ? p->a_val.data() : p->g_val.data()) + row * D;
      double acc = 0.0;
      for (I k = 0; k < D; ++k) {
        double v;
        do v = sym(g);
        while (v == 0.0);
        idx[k] = cols[k];
        val[k] = v;
        acc += v * p->witness[cols[k]];
      }
      if (eq) p->b[row] = acc;
      else p->h[row] = acc - std::abs(0.3 * sym(g));
    }
  };
  const int nt = std::max(1, std::min<int>(threads > 0 ? threads : static_cast<int>(std::thread::hardware_concurrency()),
                                           static_cast<int>(T)));
  auto parallel = [&](auto&& fn) {
    std::vector<std::thread> pool;
    for (int w = 0; w < nt; ++w)
      pool.emplace_back([&, w] {
        for (I t = w; t < T; t += nt) fn(t);
      });
    for (auto& th : pool) th.join();
  };
  parallel(stage_vec);
  parallel(stage_rows);
  return p;
}

template <class F>
int Guard(char* err, size_t len, F&& f) {
  try {
    f();
    return PDHG_OK;
  } catch (const std::invalid_argument& e) {
    if (err && len) std::snprintf(err, len, "%s", e.what());
    return PDHG_INVALID_ARGUMENT;
  } catch (const std::exception& e) {
    if (err && len) std::snprintf(err, len, "%s", e.what());
    return PDHG_INVALID_ARGUMENT;
  }
}

}  // namespace

extern "C" {

int pdhg_gen_random_lp(int64_t m, int64_t n, double density, uint64_t seed, pdhg_instance** out, char* err,
                       size_t errlen) {
  return Guard(err, errlen, [&] { *out = RandomLp(m, n, density, seed); });
}

int pdhg_gen_pagerank(int64_t n_nodes, double damping, int64_t attachment, uint64_t seed, pdhg_instance** out,
                      char* err, size_t errlen) {
  return Guard(err, errlen, [&] { *out = Pagerank(n_nodes, damping, attachment, seed); });
}

int64_t pdhg_pagerank_graph_edges(int64_t n_nodes, int64_t attachment) {
  if (attachment < 0 || n_nodes < attachment + 1) return 0;
  return (attachment + 1) + (n_nodes - attachment - 1) * attachment;
}

int pdhg_gen_pagerank_graph(int64_t n_nodes, double damping, int64_t attachment, uint64_t seed, int64_t* edges,
                            int64_t capacity, int64_t* count, char* err, size_t errlen) {
  return Guard(err, errlen, [&] {
    std::vector<std::pair<I, I>> e = PagerankGraph(n_nodes, damping, attachment, seed);
    if (static_cast<int64_t>(e.size()) > capacity) throw std::invalid_argument("edge buffer too small");
    for (size_t k = 0; k < e.size(); ++k) {
      edges[2 * k] = e[k].first;
      edges[2 * k + 1] = e[k].second;
    }
    *count = static_cast<int64_t>(e.size());
  });
}

int pdhg_build_pagerank_lp(const int64_t* edges, int64_t count, int64_t n_nodes, double damping,
                           pdhg_instance** out, char* err, size_t errlen) {
  static_assert(sizeof(std::pair<I, I>) == 2 * sizeof(int64_t), "edge layout");
  return Guard(err, errlen, [&] {
    if (count < 0 || (count > 0 && !edges)) throw std::invalid_argument("bad edge list");
    *out = PagerankLp(reinterpret_cast<const std::pair<I, I>*>(edges), static_cast<size_t>(count), n_nodes, damping);
  });
}

int pdhg_gen_transport(int64_t sources, int64_t sinks, uint64_t seed, pdhg_instance** out, char* err,
                       size_t errlen) {
  return Guard(err, errlen, [&] { *out = Transport(sources, sinks, seed); });
}

int pdhg_gen_mcf(int64_t nodes, int64_t arcs, int64_t commodities, uint64_t seed, pdhg_instance** out, char* err,
                 size_t errlen) {
  return Guard(err, errlen, [&] { *out = Mcf(nodes, arcs, commodities, seed); });
}

int pdhg_gen_staircase(int64_t stages, int64_t rows_per_stage, int64_t cols_per_stage, int64_t nnz_per_row,
                       int64_t linking_per_row, int64_t eq_rows_per_stage, uint64_t seed, int threads,
                       pdhg_instance** out, char* err, size_t errlen) {
  return Guard(err, errlen, [&] {
    *out = Staircase(stages, rows_per_stage, cols_per_stage, nnz_per_row, linking_per_row, eq_rows_per_stage, seed,
                     threads);
  });
}

int pdhg_instance_make_equalities(pdhg_instance* p, int64_t m1, char* err, size_t errlen) {
  return Guard(err, errlen, [&] {
    if (p->witness.empty()) throw std::invalid_argument("instance has no witness");
    if (m1 < 0 || m1 > p->g_rows) throw std::invalid_argument("m1 out of range");
    if (p->a_rows != 0) throw std::invalid_argument("instance already has equality rows");
    const I cut = p->g_ptr[m1];
    p->a_rows = m1;
    p->a_ptr.assign(p->g_ptr.begin(), p->g_ptr.begin() + m1 + 1);
    p->a_idx.assign(p->g_idx.begin(), p->g_idx.begin() + cut);
    p->a_val.assign(p->g_val.begin(), p->g_val.begin() + cut);
    p->b.resize(m1);
    CsrMul(p->a_ptr, p->a_idx, p->a_val, p->witness.data(), m1, p->b.data());
    std::vector<I> gp(p->g_rows - m1 + 1);
    for (I r = 0; r <= p->g_rows - m1; ++r) gp[r] = p->g_ptr[m1 + r] - cut;
    p->g_ptr = std::move(gp);
    p->g_idx.erase(p->g_idx.begin(), p->g_idx.begin() + cut);
    p->g_val.erase(p->g_val.begin(), p->g_val.begin() + cut);
    p->h.erase(p->h.begin(), p->h.begin() + m1);
    p->g_rows -= m1;
  });
}

int pdhg_instance_view(const pdhg_instance* p, pdhg_lp* v) {
  if (!p || !v) return PDHG_INVALID_ARGUMENT;
  v->a = {p->a_rows, p->n, p->a_ptr.data(), p->a_idx.data(), p->a_val.data()};
  v->g = {p->g_rows, p->n, p->g_ptr.data(), p->g_idx.data(), p->g_val.data()};
  v->n = p->n;
  v->c = p->c.data();
  v->b = p->b.data();
  v->h = p->h.data();
  v->l = p->l.data();
  v->u = p->u.data();
  v->objective_offset = p->offset;
  v->negated_objective = p->negated;
  return PDHG_OK;
}

const double* pdhg_instance_witness(const pdhg_instance* p) {
  return (p && !p->witness.empty()) ? p->witness.data() : nullptr;
}

void pdhg_instance_free(pdhg_instance* p) { delete p; }

}  // extern "C"
