/*
 * oracle.c — TEST INFRASTRUCTURE ONLY.  A plain, slow, obviously-correct CPU oracle for DAWN's
 * unweighted shortest paths (arXiv 2208.04514).  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.  It shares no code,
 * header, table or helper with the CUDA path (paper_2208_04514_b200/csrc); neither includes or
 * links the other.
 *
 * Definition followed: d(s,s) = 0; d(s,v) = length of the shortest directed
 * path s ~> v along out-edges; ORACLE_UNREACHED (0xFFFFFFFF) if none (reading Q4 replaces the
 * paper's 0-sentinel).
 *
 *   oracle_sovm        Algorithm 2 "SOVM" written literally on dense byte
 *                      vectors alpha/beta, with readings Q1 (per-edge filter), Q4, Q5, Q6, Q7, Q8.
 *   oracle_bovm        Algorithm 1 "BOVM" on CSC, cumulative alpha, merge
 *                      after the sweep (reading Q2), early exit on first hit (Eq. 4).
 *   oracle_bfs_fifo    Algorithm 3 "General BFS", FIFO queue.
 *   oracle_floyd_warshall  brute-force all pairs, n <= 512 (BASELINE.json north_star).
 *   oracle_first_hit   Theorem 1 / Lemma 1 (L152-155): smallest k with
 *                      (A^k)_ij != 0 by saturating integer matrix powers, n <= 32.
 *   oracle_record      per-source record {ecc, reached, sum_dist, hash} + edges_reach (E10,
 *                      PAPER.md L299-302; SURVEY §8(c) derived outputs).
 *   oracle_certify     the four-invariant certificate (SURVEY §8(c) pins; Fact 1 L162-164).
 *   oracle_records     oracle_sovm over many sources on a pthread pool (sources are the paper's
 *                      own scaling axis).
 *   oracle_largest_wcc the largest weakly connected component (Table 1:
 *                      S_wcc, E_wcc; the APSP source set of E11-E12 L303-308): plain FIFO
 *                      labelling over the undirected view (out-arcs plus reversed arcs), vertices
 *                      taken in ascending order; "largest" = most nodes, then most arcs, then the
 *                      smaller minimum id (reading Q15).
 *
 * Weighted (min,+) extension ("(min,+) operations ... to
 * expand the applicability of DAWN on weighted graphs"; reading Q26 in DESIGN.md):
 *   oracle_minplus     Algorithm 2's round structure over the (min,+) semiring with synchronous
 *                      rounds: alpha = vertices whose distance dropped in the previous round;
 *                      each round relaxes alpha's out-arcs from the round-start distances and
 *                      beta = {u : d(u) dropped}; stop when beta is empty (<= n-1 rounds).
 *   oracle_dijkstra    textbook Dijkstra with a binary heap (independent check).
 *   oracle_floyd_warshall_w  brute-force weighted all pairs, n <= 512.
 *   oracle_certify_w   d(s) = 0, d(v) <= d(u) + w(u,v) on every arc, every reached v != s has a
 *                      tight in-arc, UNREACHED exactly where no in-arc comes from a reached
 *                      vertex: with weights >= 1 this proves d = delta.
 *   Distances are uint64 (ORACLE_UNREACHED64 = UINT64_MAX), weights uint32 aligned with col.
 *
 * Every function is pinned by tests/test_oracle.py against closed forms, brute force, golden
 * records (tests/golden/) or each other; see DESIGN.md "Oracle pins".
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORACLE_UNREACHED 0xFFFFFFFFu

typedef struct {
  uint32_t source, ecc, reached, pad;
  uint64_t sum_dist, hash;
} oracle_rec; /* 32 bytes, same field order as the documented record */

typedef struct {
  uint32_t iterations;       /* rounds that found >= 1 new vertex (= eccentricity)          */
  uint32_t rounds;           /* rounds executed including the final empty one              */
  uint64_t edge_inspections; /* adjacency entries examined                                  */
  uint64_t node_inspections; /* outer-loop node visits                                      */
} oracle_stats;

/* SplitMix64 finaliser (Steele, Lea, Flood 2014), as defined in SURVEY §8(c). */
static uint64_t oracle_splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

uint64_t oracle_hash_term(uint32_t v, uint32_t d) {
  return oracle_splitmix64(((uint64_t)v << 32) | (uint64_t)d);
}

/*
 * Algorithm 2 (SOVM), literally:
 *   while step < n:                                  (line 1; Q8)
 *     step <- step + 1                               (line 2)
 *     for i in [0, n-1] with alpha[i] = true:        (line 3)
 *       for j in [row_ptr[i], row_ptr[i+1]):         (lines 4-6)
 *         if distance[col[j]] is unset:              (line 6 read as a per-edge filter, Q1)
 *           beta[col[j]] <- true; distance <- step; is_converged <- false   (lines 7-11)
 *     alpha.swap(beta); beta cleared                 (line 14; Q6: alpha <- beta)
 *     if is_converged: break                         (lines 15-17; reset each round, Q5)
 * Initial alpha = e_s, step = 0 (Q7); distance[s] = 0 and "unset" = ORACLE_UNREACHED (Q4).
 */
int oracle_sovm(int64_t n, const int64_t *row_ptr, const int32_t *col, int64_t s,
                uint32_t *distance, oracle_stats *st) {
  if (n < 1 || s < 0 || s >= n) return 2;
  unsigned char *alpha = (unsigned char *)calloc((size_t)n, 1);
  unsigned char *beta = (unsigned char *)calloc((size_t)n, 1);
  if (!alpha || !beta) { free(alpha); free(beta); return 3; }
  oracle_stats z = {0, 0, 0, 0};
  for (int64_t v = 0; v < n; ++v) distance[v] = ORACLE_UNREACHED;
  distance[s] = 0;
  alpha[s] = 1;
  int64_t step = 0;
  while (step < n) {
    step = step + 1;
    int is_converged = 1;
    z.rounds++;
    for (int64_t i = 0; i < n; ++i) {
      if (!alpha[i]) continue;
      z.node_inspections++;
      for (int64_t j = row_ptr[i]; j < row_ptr[i + 1]; ++j) {
        z.edge_inspections++;
        int32_t t = col[j];
        if (distance[t] == ORACLE_UNREACHED) {
          beta[t] = 1;
          distance[t] = (uint32_t)step;
          is_converged = 0;
        }
      }
    }
    unsigned char *tmp = alpha; alpha = beta; beta = tmp;  /* alpha.swap */
    memset(beta, 0, (size_t)n);
    if (is_converged) break;
    z.iterations++;
  }
  free(alpha);
  free(beta);
  if (st) *st = z;
  return 0;
}

/*
 * Algorithm 1 (BOVM), on CSC (in-edges):
 *   while step < n: step <- step + 1
 *     for i with alpha[i] = false:                          (line 3)
 *       scan CSC column i (in-neighbours) until the first   (lines 4-8; Eq. 4 early exit)
 *       in-neighbour with alpha = true: beta[i] <- true, distance[i] <- step, converged <- false
 *     alpha <- merge(alpha, beta); beta cleared             (lines 12-13 applied once per round, Q2)
 *     if is_converged: break
 * alpha is the cumulative reached set; initial alpha = e_s.
 */
int oracle_bovm(int64_t n, const int64_t *col_ptr, const int32_t *row, int64_t s,
                uint32_t *distance, oracle_stats *st) {
  if (n < 1 || s < 0 || s >= n) return 2;
  unsigned char *alpha = (unsigned char *)calloc((size_t)n, 1);
  unsigned char *beta = (unsigned char *)calloc((size_t)n, 1);
  if (!alpha || !beta) { free(alpha); free(beta); return 3; }
  oracle_stats z = {0, 0, 0, 0};
  for (int64_t v = 0; v < n; ++v) distance[v] = ORACLE_UNREACHED;
  distance[s] = 0;
  alpha[s] = 1;
  int64_t step = 0;
  while (step < n) {
    step = step + 1;
    int is_converged = 1;
    z.rounds++;
    for (int64_t i = 0; i < n; ++i) {
      if (alpha[i]) continue;
      z.node_inspections++;
      for (int64_t j = col_ptr[i]; j < col_ptr[i + 1]; ++j) {
        z.edge_inspections++;
        if (row[j] != i && alpha[row[j]]) {  /* Q3: the guard is a self-loop guard on j */
          beta[i] = 1;
          distance[i] = (uint32_t)step;
          is_converged = 0;
          break;
        }
      }
    }
    for (int64_t i = 0; i < n; ++i) { alpha[i] = alpha[i] | beta[i]; beta[i] = 0; }
    if (is_converged) break;
    z.iterations++;
  }
  free(alpha);
  free(beta);
  if (st) *st = z;
  return 0;
}

/* Algorithm 3 (General BFS), with a FIFO queue and the Q4 sentinel. */
int oracle_bfs_fifo(int64_t n, const int64_t *row_ptr, const int32_t *col, int64_t s,
                    uint32_t *distance, oracle_stats *st) {
  if (n < 1 || s < 0 || s >= n) return 2;
  int32_t *pq = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
  if (!pq) return 3;
  oracle_stats z = {0, 0, 0, 0};
  for (int64_t v = 0; v < n; ++v) distance[v] = ORACLE_UNREACHED;
  distance[s] = 0;
  int64_t head = 0, tail = 0;
  pq[tail++] = (int32_t)s;
  while (head < tail) {
    int32_t i = pq[head++];
    z.node_inspections++;
    for (int64_t j = row_ptr[i]; j < row_ptr[i + 1]; ++j) {
      z.edge_inspections++;
      int32_t index = col[j];
      if (distance[index] == ORACLE_UNREACHED) {
        distance[index] = distance[i] + 1;
        if (distance[index] > z.iterations) z.iterations = distance[index];
        pq[tail++] = index;
      }
    }
  }
  free(pq);
  if (st) *st = z;
  return 0;
}

/* Floyd-Warshall over the unweighted digraph; D is n*n row-major (D[i*n+j] = d(i,j)). */
int oracle_floyd_warshall(int64_t n, const int64_t *row_ptr, const int32_t *col, uint32_t *D) {
  if (n < 1 || n > 512) return 4;
  const uint64_t INF = (uint64_t)1 << 40;
  uint64_t *W = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)(n * n));
  if (!W) return 3;
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = 0; j < n; ++j) W[i * n + j] = (i == j) ? 0 : INF;
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = row_ptr[i]; j < row_ptr[i + 1]; ++j)
      if (col[j] != i) W[i * n + col[j]] = 1;
  for (int64_t k = 0; k < n; ++k)
    for (int64_t i = 0; i < n; ++i)
      for (int64_t j = 0; j < n; ++j)
        if (W[i * n + k] + W[k * n + j] < W[i * n + j]) W[i * n + j] = W[i * n + k] + W[k * n + j];
  for (int64_t i = 0; i < n * n; ++i) D[i] = W[i] >= INF ? ORACLE_UNREACHED : (uint32_t)W[i];
  free(W);
  return 0;
}

/* Saturating walk counts: C = A * B over uint64 with saturation at UINT64_MAX (Lemma 1). */
static void sat_matmul(int64_t n, const uint64_t *A, const uint64_t *B, uint64_t *C) {
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = 0; j < n; ++j) {
      uint64_t acc = 0;
      for (int64_t l = 0; l < n; ++l) {
        uint64_t a = A[i * n + l], b = B[l * n + j], p;
        if (a == 0 || b == 0) continue;
        if (__builtin_mul_overflow(a, b, &p)) p = UINT64_MAX;
        if (__builtin_add_overflow(acc, p, &acc)) acc = UINT64_MAX;
      }
      C[i * n + j] = acc;
    }
}

/*
 * Theorem 1: d(i,j) = k_min, the first k with a_ij^(k) != 0, for i != j;
 * a_ij^(k) = (A^k)_ij counts length-k walks (Lemma 1).  k ranges over [1, n-1]; no hit => the
 * pair is unreached.  D[i*n+i] = 0.  Optional `counts_k`: if non-NULL receives A^k for k = kq.
 */
int oracle_first_hit(int64_t n, const int64_t *row_ptr, const int32_t *col, uint32_t *D,
                     int64_t kq, uint64_t *counts_k) {
  if (n < 1 || n > 32) return 4;
  size_t sz = sizeof(uint64_t) * (size_t)(n * n);
  uint64_t *A = (uint64_t *)calloc(1, sz), *P = (uint64_t *)calloc(1, sz),
           *Q = (uint64_t *)calloc(1, sz);
  if (!A || !P || !Q) { free(A); free(P); free(Q); return 3; }
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = row_ptr[i]; j < row_ptr[i + 1]; ++j) A[i * n + col[j]] += 1;
  for (int64_t i = 0; i < n * n; ++i) D[i] = ORACLE_UNREACHED;
  for (int64_t i = 0; i < n; ++i) D[i * n + i] = 0;
  memcpy(P, A, sz); /* P = A^1 */
  int64_t kmax = n - 1 > kq ? n - 1 : kq;
  for (int64_t k = 1; k <= kmax; ++k) {
    if (counts_k && k == kq) memcpy(counts_k, P, sz);
    if (k <= n - 1)
      for (int64_t i = 0; i < n; ++i)
        for (int64_t j = 0; j < n; ++j)
          if (i != j && D[i * n + j] == ORACLE_UNREACHED && P[i * n + j] != 0)
            D[i * n + j] = (uint32_t)k;
    sat_matmul(n, P, A, Q); /* A^(k+1) */
    memcpy(P, Q, sz);
  }
  free(A); free(P); free(Q);
  return 0;
}

/*
 * Derived per-source outputs:
 *   ecc = max finite d (0 if nothing reached); reached = #{v != s : d finite};
 *   sum_dist = sum of finite d; hash = sum over finite v of splitmix64(v<<32 | d) mod 2^64;
 *   edges_reach = sum over finite v (including s) of out-degree (E10).
 */
void oracle_record(int64_t n, const int64_t *row_ptr, int64_t s, const uint32_t *distance,
                   oracle_rec *rec, uint64_t *edges_reach) {
  oracle_rec r;
  memset(&r, 0, sizeof r);
  r.source = (uint32_t)s;
  uint64_t er = 0;
  for (int64_t v = 0; v < n; ++v) {
    uint32_t d = distance[v];
    if (d == ORACLE_UNREACHED) continue;
    if (d > r.ecc) r.ecc = d;
    if (v != s) r.reached++;
    r.sum_dist += d;
    r.hash += oracle_hash_term((uint32_t)v, d);
    er += (uint64_t)(row_ptr[v + 1] - row_ptr[v]);
  }
  if (rec) *rec = r;
  if (edges_reach) *edges_reach = er;
}

/*
 * Certificate, O(n + m).  Returns 0 if `distance` is the exact BFS distance
 * vector of source s, else the number of the first violated invariant, with *bad = vertex:
 *   1: d(s) = 0, and d(v) >= 1 for reached v != s
 *   2: for every arc u->v with d(u) finite: d(v) <= d(u) + 1
 *   3: every reached v != s has an in-neighbour u with d(u) = d(v) - 1  (Fact 1, L162-164)
 *   4: UNREACHED exactly on vertices with no reached in-neighbour, never on s
 * Uses CSR (row_ptr, col) for 2 and the CSC (in_ptr, in_idx) for 3 and 4.
 */
int oracle_certify(int64_t n, const int64_t *row_ptr, const int32_t *col, const int64_t *in_ptr,
                   const int32_t *in_idx, int64_t s, const uint32_t *distance, int64_t *bad) {
  *bad = -1;
  if (distance[s] != 0) { *bad = s; return 1; }
  for (int64_t v = 0; v < n; ++v)
    if (v != s && distance[v] == 0) { *bad = v; return 1; }
  for (int64_t u = 0; u < n; ++u) {
    if (distance[u] == ORACLE_UNREACHED) continue;
    for (int64_t j = row_ptr[u]; j < row_ptr[u + 1]; ++j) {
      uint32_t dv = distance[col[j]];
      if (dv == ORACLE_UNREACHED || (uint64_t)dv > (uint64_t)distance[u] + 1) {
        *bad = col[j];
        return 2;
      }
    }
  }
  for (int64_t v = 0; v < n; ++v) {
    uint32_t d = distance[v];
    int has_reached_in = 0, has_pred = 0;
    for (int64_t j = in_ptr[v]; j < in_ptr[v + 1]; ++j) {
      uint32_t du = distance[in_idx[j]];
      if (du != ORACLE_UNREACHED) has_reached_in = 1;
      if (d != ORACLE_UNREACHED && d >= 1 && du == d - 1) has_pred = 1;
    }
    if (v != s && d != ORACLE_UNREACHED && !has_pred) { *bad = v; return 3; }
    if (v != s && (d == ORACLE_UNREACHED) == has_reached_in) { *bad = v; return 4; }
  }
  return 0;
}

/* ---- oracle_records: oracle_sovm + oracle_record over k sources on a pthread pool -------- */
typedef struct {
  int64_t n;
  const int64_t *row_ptr;
  const int32_t *col;
  const int32_t *sources;
  int64_t k;
  oracle_rec *out;
  int64_t next;
  pthread_mutex_t mu;
  int err;
} rec_job;

static void *rec_worker(void *arg) {
  rec_job *J = (rec_job *)arg;
  uint32_t *dist = (uint32_t *)malloc(sizeof(uint32_t) * (size_t)J->n);
  if (!dist) { J->err = 3; return NULL; }
  for (;;) {
    pthread_mutex_lock(&J->mu);
    int64_t i = J->next++;
    pthread_mutex_unlock(&J->mu);
    if (i >= J->k) break;
    if (oracle_sovm(J->n, J->row_ptr, J->col, J->sources[i], dist, NULL)) { J->err = 2; break; }
    oracle_record(J->n, J->row_ptr, J->sources[i], dist, &J->out[i], NULL);
  }
  free(dist);
  return NULL;
}

int oracle_records(int64_t n, const int64_t *row_ptr, const int32_t *col, int64_t k,
                   const int32_t *sources, int threads, oracle_rec *out) {
  for (int64_t i = 0; i < k; ++i)
    if (sources[i] < 0 || sources[i] >= n) return 2;
  if (threads < 1) threads = 1;
  rec_job J = {n, row_ptr, col, sources, k, out, 0, PTHREAD_MUTEX_INITIALIZER, 0};
  pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * (size_t)threads);
  if (!th) return 3;
  for (int t = 0; t < threads; ++t) pthread_create(&th[t], NULL, rec_worker, &J);
  for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
  free(th);
  return J.err;
}

/*
 * Largest weakly connected component (Table 1; reading Q15 for "largest").
 * Components of the undirected view: u ~ v iff an arc u->v or v->u exists.  Labelling: for
 * v = 0, 1, ..., n-1 not yet labelled, a FIFO search over out- and in-arcs labels v's whole
 * component (so each component is found at its minimum vertex id).  Then per component the node
 * count and the arc count (arcs whose source lies in it); the chosen component has the most
 * nodes, ties -> the most arcs, then the smaller minimum id (the earlier one found).
 * Writes its vertices ascending into out (capacity n) and returns their number; *arcs_out gets
 * E_wcc.  Returns -1 on allocation failure.
 */
int64_t oracle_largest_wcc(int64_t n, const int64_t *row_ptr, const int32_t *col, int64_t *out,
                           uint64_t *arcs_out) {
  const int64_t m = row_ptr[n];
  /* reversed arcs (in-adjacency) by a counting sort */
  int64_t *in_ptr = calloc((size_t)n + 1, sizeof(int64_t));
  int32_t *in_src = malloc(sizeof(int32_t) * (size_t)(m > 0 ? m : 1));
  int64_t *label = malloc(sizeof(int64_t) * (size_t)n);
  int64_t *queue = malloc(sizeof(int64_t) * (size_t)n);
  if (!in_ptr || !in_src || !label || !queue) {
    free(in_ptr); free(in_src); free(label); free(queue);
    return -1;
  }
  for (int64_t j = 0; j < m; ++j) in_ptr[col[j] + 1]++;
  for (int64_t v = 0; v < n; ++v) in_ptr[v + 1] += in_ptr[v];
  {
    int64_t *fill = malloc(sizeof(int64_t) * (size_t)n);
    if (!fill) { free(in_ptr); free(in_src); free(label); free(queue); return -1; }
    for (int64_t v = 0; v < n; ++v) fill[v] = in_ptr[v];
    for (int64_t u = 0; u < n; ++u)
      for (int64_t j = row_ptr[u]; j < row_ptr[u + 1]; ++j) in_src[fill[col[j]]++] = (int32_t)u;
    free(fill);
  }
  for (int64_t v = 0; v < n; ++v) label[v] = -1;
  int64_t best = -1, best_nodes = 0;
  uint64_t best_arcs = 0;
  for (int64_t s = 0; s < n; ++s) {
    if (label[s] >= 0) continue;
    int64_t head = 0, tail = 0, nodes = 0;
    uint64_t arcs = 0;
    label[s] = s;
    queue[tail++] = s;
    while (head < tail) {
      const int64_t v = queue[head++];
      nodes++;
      arcs += (uint64_t)(row_ptr[v + 1] - row_ptr[v]);
      for (int64_t j = row_ptr[v]; j < row_ptr[v + 1]; ++j)
        if (label[col[j]] < 0) { label[col[j]] = s; queue[tail++] = col[j]; }
      for (int64_t j = in_ptr[v]; j < in_ptr[v + 1]; ++j)
        if (label[in_src[j]] < 0) { label[in_src[j]] = s; queue[tail++] = in_src[j]; }
    }
    /* s is this component's minimum id; a later component wins only if strictly larger */
    if (nodes > best_nodes || (nodes == best_nodes && arcs > best_arcs)) {
      best = s;
      best_nodes = nodes;
      best_arcs = arcs;
    }
  }
  int64_t k = 0;
  for (int64_t v = 0; v < n; ++v)
    if (label[v] == best) out[k++] = v;
  if (arcs_out) *arcs_out = best_arcs;
  free(in_ptr); free(in_src); free(label); free(queue);
  return k;
}


/* ------------------------------------------------------------------ weighted (min,+) */
#define ORACLE_UNREACHED64 0xFFFFFFFFFFFFFFFFull

/*
 * (min,+) SOVM, synchronous rounds (reading Q26):
 *   d_0 = e_s (0 at s, infinity elsewhere); alpha_0 = {s}
 *   round k: for every v in alpha_k, every arc v -> u:  cand(u) <- min(cand(u), d_k(v) + w)
 *            d_{k+1}(u) = min(d_k(u), cand(u));  alpha_{k+1} = {u : d_{k+1}(u) < d_k(u)}
 *   stop when alpha_{k+1} is empty.  st->iterations = rounds that improved >= 1 vertex,
 *   st->edge_inspections = arcs relaxed.
 */
int oracle_minplus(int64_t n, const int64_t *row_ptr, const int32_t *col, const uint32_t *w,
                   int64_t s, uint64_t *dist, oracle_stats *st) {
  if (n < 1 || s < 0 || s >= n) return 2;
  unsigned char *alpha = (unsigned char *)calloc((size_t)n, 1);
  unsigned char *beta = (unsigned char *)calloc((size_t)n, 1);
  uint64_t *cand = (uint64_t *)malloc((size_t)n * sizeof(uint64_t));
  if (!alpha || !beta || !cand) { free(alpha); free(beta); free(cand); return 3; }
  for (int64_t i = 0; i < n; ++i) dist[i] = ORACLE_UNREACHED64;
  dist[s] = 0;
  alpha[s] = 1;
  oracle_stats S = {0, 0, 0, 0};
  for (int64_t round = 0; round < n; ++round) {
    S.rounds++;
    for (int64_t i = 0; i < n; ++i) cand[i] = ORACLE_UNREACHED64;
    for (int64_t v = 0; v < n; ++v) {
      S.node_inspections++;
      if (!alpha[v]) continue;
      for (int64_t j = row_ptr[v]; j < row_ptr[v + 1]; ++j) {
        S.edge_inspections++;
        const uint64_t c = dist[v] + (uint64_t)w[j];
        if (c < cand[col[j]]) cand[col[j]] = c;
      }
    }
    int improved = 0;
    for (int64_t u = 0; u < n; ++u) {
      beta[u] = 0;
      if (cand[u] < dist[u]) {
        dist[u] = cand[u];
        beta[u] = 1;
        improved = 1;
      }
    }
    unsigned char *t = alpha;
    alpha = beta;
    beta = t;
    if (!improved) break;
    S.iterations++;
  }
  if (st) *st = S;
  free(alpha);
  free(beta);
  free(cand);
  return 0;
}

/* Dijkstra with a binary heap of (distance, vertex); lazy deletion. */
int oracle_dijkstra(int64_t n, const int64_t *row_ptr, const int32_t *col, const uint32_t *w,
                    int64_t s, uint64_t *dist) {
  if (n < 1 || s < 0 || s >= n) return 2;
  const int64_t cap = row_ptr[n] + 1;
  uint64_t *hk = (uint64_t *)malloc((size_t)cap * sizeof(uint64_t));
  int64_t *hv = (int64_t *)malloc((size_t)cap * sizeof(int64_t));
  unsigned char *done = (unsigned char *)calloc((size_t)n, 1);
  if (!hk || !hv || !done) { free(hk); free(hv); free(done); return 3; }
  for (int64_t i = 0; i < n; ++i) dist[i] = ORACLE_UNREACHED64;
  dist[s] = 0;
  int64_t hn = 0;
  hk[0] = 0; hv[0] = s; hn = 1;
  while (hn > 0) {
    const uint64_t k = hk[0];
    const int64_t v = hv[0];
    hn--;  /* pop: move the last entry to the root and sift down */
    hk[0] = hk[hn]; hv[0] = hv[hn];
    for (int64_t i = 0;;) {
      int64_t l = 2 * i + 1, r = l + 1, m = i;
      if (l < hn && hk[l] < hk[m]) m = l;
      if (r < hn && hk[r] < hk[m]) m = r;
      if (m == i) break;
      uint64_t tk = hk[i]; hk[i] = hk[m]; hk[m] = tk;
      int64_t tv = hv[i]; hv[i] = hv[m]; hv[m] = tv;
      i = m;
    }
    if (done[v] || k != dist[v]) continue;
    done[v] = 1;
    for (int64_t j = row_ptr[v]; j < row_ptr[v + 1]; ++j) {
      const int64_t u = col[j];
      const uint64_t c = k + (uint64_t)w[j];
      if (c < dist[u]) {
        dist[u] = c;
        int64_t i = hn++;  /* push and sift up */
        hk[i] = c; hv[i] = u;
        while (i > 0) {
          int64_t p = (i - 1) / 2;
          if (hk[p] <= hk[i]) break;
          uint64_t tk = hk[i]; hk[i] = hk[p]; hk[p] = tk;
          int64_t tv = hv[i]; hv[i] = hv[p]; hv[p] = tv;
          i = p;
        }
      }
    }
  }
  free(hk);
  free(hv);
  free(done);
  return 0;
}

/* Weighted Floyd-Warshall, n <= 512: D[i*n + j]; parallel arcs take the lightest. */
int oracle_floyd_warshall_w(int64_t n, const int64_t *row_ptr, const int32_t *col,
                            const uint32_t *w, uint64_t *D) {
  if (n < 1 || n > 512) return 2;
  for (int64_t i = 0; i < n * n; ++i) D[i] = ORACLE_UNREACHED64;
  for (int64_t i = 0; i < n; ++i) {
    D[i * n + i] = 0;
    for (int64_t j = row_ptr[i]; j < row_ptr[i + 1]; ++j)
      if (col[j] != i && (uint64_t)w[j] < D[i * n + col[j]]) D[i * n + col[j]] = w[j];
  }
  for (int64_t k = 0; k < n; ++k)
    for (int64_t i = 0; i < n; ++i) {
      if (D[i * n + k] == ORACLE_UNREACHED64) continue;
      for (int64_t j = 0; j < n; ++j)
        if (D[k * n + j] != ORACLE_UNREACHED64 && D[i * n + k] + D[k * n + j] < D[i * n + j])
          D[i * n + j] = D[i * n + k] + D[k * n + j];
    }
  return 0;
}

/* Certificate of a weighted distance vector (weights >= 1).  Returns 0 if valid, else the
 * number of the first failing condition; *bad = the offending vertex. */
int oracle_certify_w(int64_t n, const int64_t *row_ptr, const int32_t *col, const uint32_t *w,
                     int64_t s, const uint64_t *dist, int64_t *bad) {
  *bad = -1;
  if (dist[s] != 0) { *bad = s; return 1; }
  unsigned char *tight = (unsigned char *)calloc((size_t)n, 1);
  unsigned char *fed = (unsigned char *)calloc((size_t)n, 1);
  if (!tight || !fed) { free(tight); free(fed); return 9; }
  int rc = 0;
  for (int64_t u = 0; u < n && !rc; ++u) {
    if (dist[u] == ORACLE_UNREACHED64) continue;
    for (int64_t j = row_ptr[u]; j < row_ptr[u + 1]; ++j) {
      const int64_t v = col[j];
      const uint64_t c = dist[u] + (uint64_t)w[j];
      fed[v] = 1;
      if (dist[v] > c) { *bad = v; rc = 2; break; }        /* (ii) relaxed arc violated */
      if (dist[v] == c && v != s) tight[v] = 1;
    }
  }
  for (int64_t v = 0; v < n && !rc; ++v) {
    if (v == s) continue;
    if (dist[v] != ORACLE_UNREACHED64 && !tight[v]) { *bad = v; rc = 3; }   /* (iii) */
    else if (dist[v] == ORACLE_UNREACHED64 && fed[v]) { *bad = v; rc = 4; } /* (iv) */
  }
  free(tight);
  free(fed);
  return rc;
}
