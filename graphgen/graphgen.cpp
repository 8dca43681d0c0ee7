// graphgen — seeded synthetic graph inputs shared by the oracle tests, the GPU parity tests
// and bench.py.  This module holds NONE of DAWN's arithmetic: it produces CSR/CSC arrays
// and source lists only (SPEC S:L22-143 graph-core).
//
//   * gg_kron   Graph500 Kronecker ("RMAT") generator, A,B,C = .57,.19,.19:
//               per edge and per bit level two Bernoulli draws (the Graph500 octave reference
//               recipe), then a seeded random vertex relabelling.
//   * gg_er     directed Erdos-Renyi G(n, m): the first m distinct ordered pairs u != v of a
//               counter-based stream (BASELINE.json configs[0]).
//   * gg_grid   W x H 4-neighbour lattice, id = r*W + c, symmetric (configs[2]).
//   * normalisation: self-loops dropped, duplicates removed, rows sorted ascending
//               (SURVEY Q12); optional symmetrisation.
//   * gg_transpose  CSR -> CSC.
//   * gg_wcc_largest  union-find over arcs; the component with the most nodes, ties to more
//               arcs then smaller minimum id.
//   * gg_sample_sources  k sources uniform over vertices with out-degree > 0.
//
// Every random draw is a pure function of (seed, stream, counter) -> splitmix64, so results
// are independent of the thread count.
#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <thread>
#include <unordered_set>
#include <vector>

namespace {

inline uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
// counter-based stream: draw number `i` of stream `s` under `seed`
inline uint64_t draw(uint64_t seed, uint64_t s, uint64_t i) {
  return mix64(mix64(seed * 0x632BE59BD9B4E019ull + s) ^ (i * 0xD1B54A32D192ED03ull));
}

int n_threads() {
  const char *e = getenv("GRAPHGEN_THREADS");
  if (e && atoi(e) > 0) return atoi(e);
  unsigned h = std::thread::hardware_concurrency();
  return h ? (int)std::min(h, 64u) : 4;
}

template <class F> void parallel_for(int64_t n, F f) {
  int T = n_threads();
  if (n < 4096 || T == 1) { f(0, n, 0); return; }
  std::vector<std::thread> th;
  for (int t = 0; t < T; ++t) {
    int64_t a = n * t / T, b = n * (t + 1) / T;
    th.emplace_back([=] { f(a, b, t); });
  }
  for (auto &x : th) x.join();
}

struct Csr {
  int64_t n = 0, m = 0;
  std::vector<int64_t> row_ptr;
  std::vector<int32_t> col;
};

// Build a normalised CSR from packed arcs (u << 32 | v).  Drops loops and duplicates; rows
// sorted.  `arcs` is consumed.  Bucketed by source so each bucket sorts in cache, in parallel.
Csr build_csr(int64_t n, std::vector<uint64_t> &arcs) {
  Csr g;
  g.n = n;
  const int64_t A = (int64_t)arcs.size();
  int shift = 0;
  while (((n - 1) >> shift) >= 4096) ++shift;  // <= 4096 buckets
  const int64_t B = n ? ((n - 1) >> shift) + 1 : 1;
  int T = n_threads();
  if (A < 65536) T = 1;
  std::vector<std::vector<int64_t>> cnt(T, std::vector<int64_t>(B + 1, 0));
  auto chunk = [&](int t) { return std::make_pair(A * t / T, A * (t + 1) / T); };
  {
    std::vector<std::thread> th;
    for (int t = 0; t < T; ++t)
      th.emplace_back([&, t] {
        auto [a, b] = chunk(t);
        for (int64_t i = a; i < b; ++i) cnt[t][(arcs[i] >> 32) >> shift]++;
      });
    for (auto &x : th) x.join();
  }
  std::vector<int64_t> bstart(B + 1, 0);
  {
    int64_t run = 0;
    for (int64_t b = 0; b < B; ++b) {
      bstart[b] = run;
      for (int t = 0; t < T; ++t) { int64_t c = cnt[t][b]; cnt[t][b] = run; run += c; }
    }
    bstart[B] = run;
  }
  std::vector<uint64_t> bucketed(A);
  {
    std::vector<std::thread> th;
    for (int t = 0; t < T; ++t)
      th.emplace_back([&, t] {
        auto [a, b] = chunk(t);
        auto &c = cnt[t];
        for (int64_t i = a; i < b; ++i) bucketed[c[(arcs[i] >> 32) >> shift]++] = arcs[i];
      });
    for (auto &x : th) x.join();
  }
  std::vector<uint64_t>().swap(arcs);
  // per bucket: sort, unique, drop loops (compacted in place); record kept counts
  std::vector<int64_t> kept(B, 0);
  std::vector<int64_t> deg(n, 0);
  {
    std::atomic<int64_t> next{0};
    std::vector<std::thread> th;
    for (int t = 0; t < T; ++t)
      th.emplace_back([&] {
        for (;;) {
          int64_t b = next.fetch_add(1);
          if (b >= B) break;
          uint64_t *p = bucketed.data() + bstart[b], *e = bucketed.data() + bstart[b + 1];
          std::sort(p, e);
          int64_t w = 0;
          uint64_t prev = ~0ull;
          for (uint64_t *q = p; q < e; ++q) {
            uint64_t x = *q;
            if (x == prev) continue;
            prev = x;
            if ((x >> 32) == (x & 0xffffffffull)) continue;  // self-loop
            p[w++] = x;
            deg[x >> 32]++;
          }
          kept[b] = w;
        }
      });
    for (auto &x : th) x.join();
  }
  g.row_ptr.assign(n + 1, 0);
  for (int64_t v = 0; v < n; ++v) g.row_ptr[v + 1] = g.row_ptr[v] + deg[v];
  g.m = g.row_ptr[n];
  g.col.resize(g.m);
  parallel_for(B, [&](int64_t a, int64_t b, int) {
    for (int64_t k = a; k < b; ++k) {
      if (!kept[k]) continue;
      const uint64_t *p = bucketed.data() + bstart[k];
      int64_t dst = g.row_ptr[p[0] >> 32];
      for (int64_t i = 0; i < kept[k]; ++i) g.col[dst + i] = (int32_t)(p[i] & 0xffffffffull);
    }
  });
  return g;
}

}  // namespace

extern "C" {

typedef struct gg_csr_s {
  Csr g;
} gg_csr;

int64_t gg_n(const gg_csr *h) { return h->g.n; }
int64_t gg_m(const gg_csr *h) { return h->g.m; }
void gg_copy(const gg_csr *h, int64_t *row_ptr, int32_t *col) {
  std::memcpy(row_ptr, h->g.row_ptr.data(), sizeof(int64_t) * (h->g.n + 1));
  if (h->g.m) std::memcpy(col, h->g.col.data(), sizeof(int32_t) * h->g.m);
}
void gg_free(gg_csr *h) { delete h; }

// Arbitrary edge list -> normalised CSR (used by hand fixtures and the property corpus).
gg_csr *gg_from_edges(int64_t n, int64_t k, const int32_t *src, const int32_t *dst,
                      int symmetrize) {
  for (int64_t i = 0; i < k; ++i)
    if (src[i] < 0 || dst[i] < 0 || src[i] >= n || dst[i] >= n) return nullptr;
  std::vector<uint64_t> arcs;
  arcs.reserve(symmetrize ? 2 * k : k);
  for (int64_t i = 0; i < k; ++i) {
    arcs.push_back(((uint64_t)src[i] << 32) | (uint32_t)dst[i]);
    if (symmetrize) arcs.push_back(((uint64_t)dst[i] << 32) | (uint32_t)src[i]);
  }
  auto *h = new gg_csr;
  h->g = build_csr(n, arcs);
  return h;
}

// Graph500 Kronecker generator (scale, edge factor), symmetrised.
gg_csr *gg_kron(int scale, int edge_factor, uint64_t seed, int symmetrize) {
  const int64_t n = int64_t(1) << scale;
  const int64_t M = (int64_t)edge_factor * n;
  const double A = 0.57, B = 0.19, C = 0.19;
  const double ab = A + B, c_norm = C / (1.0 - ab), a_norm = A / ab;
  const uint64_t t_ab = (uint64_t)(ab * 4294967296.0), t_c = (uint64_t)(c_norm * 4294967296.0),
                 t_a = (uint64_t)(a_norm * 4294967296.0);
  // random relabelling: Fisher-Yates driven by stream 1
  std::vector<int32_t> perm(n);
  std::iota(perm.begin(), perm.end(), 0);
  for (int64_t i = n - 1; i > 0; --i) {
    uint64_t r = draw(seed, 1, (uint64_t)i);
    int64_t j = (int64_t)((unsigned __int128)r * (uint64_t)(i + 1) >> 64);
    std::swap(perm[i], perm[j]);
  }
  std::vector<uint64_t> arcs(symmetrize ? 2 * M : M);
  parallel_for(M, [&](int64_t a, int64_t b, int) {
    for (int64_t e = a; e < b; ++e) {
      uint64_t i = 0, j = 0;
      for (int l = 0; l < scale; ++l) {
        uint64_t r = draw(seed, 2, (uint64_t)e * 64 + l);
        uint64_t ii = (r & 0xffffffffull) >= t_ab;                  // rand > ab
        uint64_t jj = (r >> 32) >= (ii ? t_c : t_a);                // rand > c_norm / a_norm
        i |= ii << l;
        j |= jj << l;
      }
      uint64_t u = (uint32_t)perm[i], v = (uint32_t)perm[j];
      if (symmetrize) {
        arcs[2 * e] = (u << 32) | v;
        arcs[2 * e + 1] = (v << 32) | u;
      } else {
        arcs[e] = (u << 32) | v;
      }
    }
  });
  auto *h = new gg_csr;
  h->g = build_csr(n, arcs);
  return h;
}

// Directed G(n, m): first m distinct ordered pairs (u != v) of a counter-based stream.
gg_csr *gg_er(int64_t n, int64_t m, uint64_t seed) {
  if (n < 2 || m > n * (n - 1)) return nullptr;
  std::unordered_set<uint64_t> seen;
  std::vector<uint64_t> arcs;
  arcs.reserve(m);
  for (uint64_t i = 0; (int64_t)arcs.size() < m; ++i) {
    uint64_t r = draw(seed, 3, i);
    uint64_t u = (uint64_t)((unsigned __int128)(r & 0xffffffffull) * n >> 32);
    uint64_t v = (uint64_t)((unsigned __int128)(r >> 32) * n >> 32);
    if (u == v) continue;
    uint64_t key = (u << 32) | v;
    if (seen.insert(key).second) arcs.push_back(key);
  }
  auto *h = new gg_csr;
  h->g = build_csr(n, arcs);
  return h;
}

// W x H 4-neighbour lattice, vertex id r*W + c, symmetric.
gg_csr *gg_grid(int64_t W, int64_t H) {
  const int64_t n = W * H;
  auto *h = new gg_csr;
  Csr &g = h->g;
  g.n = n;
  g.row_ptr.assign(n + 1, 0);
  for (int64_t v = 0; v < n; ++v) {
    int64_t r = v / W, c = v % W;
    g.row_ptr[v + 1] = g.row_ptr[v] + (r > 0) + (c > 0) + (c + 1 < W) + (r + 1 < H);
  }
  g.m = g.row_ptr[n];
  g.col.resize(g.m);
  parallel_for(n, [&](int64_t a, int64_t b, int) {
    for (int64_t v = a; v < b; ++v) {
      int64_t r = v / W, c = v % W, o = g.row_ptr[v];
      if (r > 0) g.col[o++] = (int32_t)(v - W);  // ascending order
      if (c > 0) g.col[o++] = (int32_t)(v - 1);
      if (c + 1 < W) g.col[o++] = (int32_t)(v + 1);
      if (r + 1 < H) g.col[o++] = (int32_t)(v + W);
    }
  });
  return h;
}

// CSR -> CSC (exact transpose; rows of the CSC sorted ascending).
void gg_transpose(int64_t n, int64_t m, const int64_t *row_ptr, const int32_t *col,
                  int64_t *out_ptr, int32_t *out_idx) {
  std::vector<int64_t> c(n + 1, 0);
  for (int64_t j = 0; j < m; ++j) c[col[j] + 1]++;
  for (int64_t v = 0; v < n; ++v) c[v + 1] += c[v];
  std::memcpy(out_ptr, c.data(), sizeof(int64_t) * (n + 1));
  for (int64_t u = 0; u < n; ++u)  // ascending u keeps each CSC row sorted
    for (int64_t j = row_ptr[u]; j < row_ptr[u + 1]; ++j) out_idx[c[col[j]]++] = (int32_t)u;
}

static int64_t uf_find(std::vector<int64_t> &p, int64_t x) {
  while (p[x] != x) { p[x] = p[p[x]]; x = p[x]; }
  return x;
}

// Largest WCC: writes its vertices ascending into `verts` (capacity n);
// returns S_wcc, stores E_wcc (arcs with both ends inside).
int64_t gg_wcc_largest(int64_t n, const int64_t *row_ptr, const int32_t *col, int32_t *verts,
                       int64_t *e_wcc) {
  std::vector<int64_t> p(n);
  std::iota(p.begin(), p.end(), 0);
  for (int64_t u = 0; u < n; ++u)
    for (int64_t j = row_ptr[u]; j < row_ptr[u + 1]; ++j) {
      int64_t a = uf_find(p, u), b = uf_find(p, col[j]);
      if (a != b) { if (a < b) std::swap(a, b); p[a] = b; }  // root = smaller id
    }
  std::vector<int64_t> sz(n, 0), ec(n, 0);
  for (int64_t u = 0; u < n; ++u) {
    int64_t r = uf_find(p, u);
    sz[r]++;
    ec[r] += row_ptr[u + 1] - row_ptr[u];
  }
  int64_t best = -1;
  for (int64_t r = 0; r < n; ++r) {  // roots are component minima, scanned ascending
    if (p[r] != r) continue;
    if (best < 0 || sz[r] > sz[best] || (sz[r] == sz[best] && ec[r] > ec[best])) best = r;
  }
  int64_t k = 0;
  for (int64_t u = 0; u < n; ++u)
    if (uf_find(p, u) == best) verts[k++] = (int32_t)u;
  if (e_wcc) *e_wcc = ec[best];
  return k;
}

// k sources uniform (with replacement) over vertices with out-degree > 0; seeded.
int64_t gg_sample_sources(int64_t n, const int64_t *row_ptr, int64_t k, uint64_t seed,
                          int32_t *out) {
  std::vector<int32_t> pool;
  for (int64_t v = 0; v < n; ++v)
    if (row_ptr[v + 1] > row_ptr[v]) pool.push_back((int32_t)v);
  if (pool.empty()) return 0;
  for (int64_t i = 0; i < k; ++i) {
    uint64_t r = draw(seed, 4, (uint64_t)i);
    out[i] = pool[(size_t)((unsigned __int128)r * pool.size() >> 64)];
  }
  return k;
}

// Arc weights for the weighted (min,+) extension: w = 1 + mix64(seed ^ key) % wmax, key = the
// arc (u << 32 | v), or the unordered pair (min << 32 | max) when `symmetric` so both arcs of an
// undirected edge carry the same weight (Graph500 SSSP: one weight per edge).  Counter-based:
// independent of the thread count.
void gg_weights(int64_t n, const int64_t *row_ptr, const int32_t *col, uint64_t seed,
                uint32_t wmax, int symmetric, uint32_t *w) {
  parallel_for(n, [&](int64_t lo, int64_t hi, int) {
    for (int64_t u = lo; u < hi; ++u)
      for (int64_t j = row_ptr[u]; j < row_ptr[u + 1]; ++j) {
        const uint64_t v = (uint64_t)col[j];
        const uint64_t a = symmetric ? std::min<uint64_t>(u, v) : (uint64_t)u;
        const uint64_t b = symmetric ? std::max<uint64_t>(u, v) : v;
        w[j] = 1u + (uint32_t)(mix64(seed ^ ((a << 32) | b)) % (uint64_t)(wmax ? wmax : 1));
      }
  });
}

}  // extern "C"
