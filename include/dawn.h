/*
 * dawn.h — C ABI of libdawn.so, the B200 (sm_100a) hot path of DAWN (arXiv 2208.04514):
 * unweighted single-source / multi-source / all-pairs shortest paths by repeated
 * boolean vector x CSR products (SOVM, Algorithm 2, Eq. 9) and
 * their pull form (BOVM, Algorithm 1, Eq. 4).
 *
 * Conventions:
 *  - Every function returns dawn_status; no C++ exception crosses this boundary.  On a
 *    non-DAWN_OK return dawn_last_error() (thread-local) describes the failure.
 *  - Argument validation happens on the host BEFORE anything is enqueued; on error nothing
 *    has been enqueued and no output has been written.
 *  - The library never allocates device memory.  Graph arrays, workspace and outputs are
 *    caller-owned device buffers (PyTorch tensors in the Python binding) that must outlive
 *    the dawn_graph handle.  Only the small host-side handle is heap-allocated.
 *  - Compute calls are asynchronous on `stream` (a cudaStream_t passed as void*).  Device
 *    faults surface at the caller's next synchronisation (DAWN_ERR_CUDA from a later call).
 *  - One in-flight call per graph handle (the handle's workspace holds the frontier state).
 *    The graph arrays themselves are immutable and may be shared by several handles.
 *  - Distances are uint32: d(s) = 0, d(v) = hop count of a shortest directed path s ~> v
 *    along out-edges (Theorem 1), DAWN_UNREACHED if none (reading Q4 of
 *    the paper's 0 sentinel collides with d(s) = 0).
 */
#ifndef DAWN_H
#define DAWN_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DAWN_UNREACHED 0xFFFFFFFFu
/* Sources per pass of the bit-parallel multi-source kernel (4 x 64-bit words per vertex) and the
 * unit of the APSP shard rule. */
#ifndef DAWN_MS_BATCH
#define DAWN_MS_BATCH 256
#endif

typedef enum {
  DAWN_OK = 0,
  DAWN_ERR_INVALID_ARGUMENT = 1, /* null pointer, n < 1, m < 0, unknown flag / variant       */
  DAWN_ERR_BOUNDS = 2,           /* a source id outside [0, n)    */
  DAWN_ERR_CONFIG = 3,           /* PULL requested on a directed graph loaded without CSC     */
  DAWN_ERR_CAPACITY = 4,         /* output capacity too small; m >= 2^32; n >= 2^31           */
  DAWN_ERR_WORKSPACE = 5,        /* workspace smaller than dawn_workspace_bytes()             */
  DAWN_ERR_INVALID_GRAPH = 6,    /* CSR invariant violated (only with DAWN_GRAPH_VALIDATE)    */
  DAWN_ERR_CUDA = 7              /* a CUDA runtime error (launch failure, earlier fault)      */
} dawn_status;

/* Graph flags. */
enum {
  DAWN_GRAPH_SYMMETRIC = 1, /* arcs come in both directions: CSC == CSR, in_* may be NULL   */
  DAWN_GRAPH_VALIDATE = 2,  /* check row_ptr monotone, row_ptr[0]=0, row_ptr[n]=m, cols in
                               range; synchronises `stream` once                           */
  DAWN_GRAPH_TRACE = 4,     /* dawn_sssp records one dawn_trace_rec per level (device
                               %globaltimer), readable with dawn_graph_trace               */
  DAWN_GRAPH_LEAN = 8       /* memory-frugal residency (E13): no
                               bit-parallel words (dawn_msssp / dawn_apsp then return
                               DAWN_ERR_CONFIG), no degree-ordered in-row copy (pull probes
                               the caller's adjacency order), no augmented arc array.  The
                               same distances; C4 workspace 7.5 GB -> 1.1 GB                  */
};

/* Direction variants of one level step. */
enum {
  DAWN_AUTO = 0, /* direction-optimising: push while the frontier is small, pull while it is
                    wide (switch on measured frontier density, device-side)                 */
  DAWN_PUSH = 1, /* SOVM only (Algorithm 2): expand the frontier's out-rows (CSR)            */
  DAWN_PULL = 2  /* BOVM only (Algorithm 1): unreached vertices scan in-rows (CSC) until the
                    first frontier in-neighbour                                              */
};

/* Per-source statistics of dawn_sssp (device memory, 32 bytes). */
typedef struct {
  uint32_t levels;         /* eccentricity eps(s): rounds that found >= 1 vertex    */
  uint32_t reached;        /* #{v != s : d(v) finite}       */
  uint64_t edges_reach;    /* E10: sum of out-degrees over reached v incl. s
                              = the GTEPS numerator                                          */
  uint64_t edges_examined; /* adjacency entries actually read by the executed schedule       */
  uint32_t push_levels;    /* levels run as push (SOVM)                                      */
  uint32_t pull_levels;    /* levels run as pull (BOVM)                                      */
} dawn_sssp_stats;

/* Per-source record for msssp / apsp (32 bytes; SURVEY §8(c) "derived outputs").
 * ecc = max finite d (0 if nothing reached); reached = #{v != s : d finite};
 * sum_dist = sum of finite d; hash = sum over finite v of splitmix64((v << 32) | d(v))
 * mod 2^64 (order independent).                                                             */
typedef struct {
  uint32_t source, ecc, reached, pad;
  uint64_t sum_dist, hash;
} dawn_record;

/* Per-level trace of the last dawn_sssp call on a graph loaded with DAWN_GRAPH_TRACE. */
typedef struct {
  uint64_t t_ns;     /* device %globaltimer when level `level` started (after its barrier)   */
  uint32_t level;    /* L: the frontier holds the vertices at distance L                     */
  uint32_t dir;      /* 0 push, 1 pull, 2 = stop (frontier empty / all reachable found)      */
  uint32_t nf;       /* |frontier L|                                                          */
  uint32_t rep;      /* frontier representation before the level: 0 queue, 1 bitmap          */
  uint64_t mf;       /* sum of out-degrees of frontier L                                      */
  uint64_t t_first;  /* %globaltimer when the first CTA finished level L's work               */
  uint64_t t_last;   /* %globaltimer when the last CTA finished level L's work (pre-barrier)  */
  uint64_t cyc[4];   /* SM cycles summed over all warps: [0] push items / pull light rows,
                        [1] pull heavy-row pieces, [2] queue flush + counters, [3] conversions */
} dawn_trace_rec;

typedef struct dawn_graph_s *dawn_graph;

/* Bytes of device workspace a graph handle needs (graph-resident arrays + the frontier state
 * of one SSSP + one 64-source batch).  flags as for dawn_graph_load_csr. Returns 0 if the
 * sizes are unsupported (n < 1, n >= 2^31, m < 0, m >= 2^32).                               */
size_t dawn_workspace_bytes(int64_t n, int64_t m, uint32_t flags);

/*
 * Make a graph resident (untimed per SPEC S:L357).
 *   n, m         vertex and arc counts (directed arcs; a symmetric graph stores both).
 *   row_ptr      device int64[n+1], CSR offsets (PAPER Table 1 "CSR", L103; D1).
 *   col          device int32[m], CSR column ids, rows need not be sorted; no self-loops are
 *                required for correctness (they never change a distance).
 *   in_row_ptr, in_col   device CSC (in-edges), or NULL.  Ignored when
 *                DAWN_GRAPH_SYMMETRIC is set (CSC == CSR).  Without them a directed graph
 *                supports only DAWN_PUSH / DAWN_AUTO (which then never pulls).
 *   flags        DAWN_GRAPH_SYMMETRIC | DAWN_GRAPH_VALIDATE.
 *   workspace    device buffer of >= dawn_workspace_bytes(n, m, flags) bytes, 256-B aligned.
 *   stream       cudaStream_t; the one-time conversion kernels are enqueued on it.
 *   out          receives the handle.  Arrays are referenced, not copied (except a 32-bit
 *                offset copy held in the workspace).
 * Errors: INVALID_ARGUMENT, CAPACITY (m >= 2^32, n >= 2^31), WORKSPACE, INVALID_GRAPH, CUDA.
 */
dawn_status dawn_graph_load_csr(int64_t n, int64_t m, const int64_t *row_ptr, const int32_t *col,
                                const int64_t *in_row_ptr, const int32_t *in_col, uint32_t flags,
                                void *workspace, size_t ws_bytes, void *stream, dawn_graph *out);

/* Free the host-side handle only (device memory belongs to the caller). NULL is a no-op. */
dawn_status dawn_graph_destroy(dawn_graph g);

/* Tunables of a graph handle (dawn_graph_set_param).  Defaults were measured on B200 with the
 * Kronecker-20/24 configs; they change speed only, never results.
 *   DAWN_PARAM_ALPHA  push -> pull when alpha * m_f^2 > n_u * m_u and the frontier grows
 *                     (m_f: out-degree sum of the frontier; n_u / m_u: vertices / arcs not yet
 *                     reached).  A pull sweep costs ~ n_u early-exit scans of length ~ m_u/m_f.
 *                     The switch idea is Beamer's, cited by the paper at L123.  Default 2.
 *   DAWN_PARAM_BETA   pull -> push when beta * n_f < n and the frontier shrinks.  Default 96.
 *   DAWN_PARAM_MS_ALPHA  the multi-source kernel pulls when ms_alpha * m_active > m_unsettled.
 *                     Default 2.
 *   DAWN_PARAM_BITMAP_PUSH_EDGES  push levels whose frontier has >= this many arcs mark
 *                     candidates in a bitmap (fire-and-forget) and settle them in a second pass
 *                     instead of one returning atomic per arc.  Default 262144.
 *   DAWN_PARAM_SOLO_EDGES  push levels with <= this many arcs run on one CTA with block-level
 *                     barriers only.  Default 512.
 *   DAWN_PARAM_BITMAP_PUSH_GROW_EDGES  the bitmap push threshold for a push level whose frontier
 *                     grew (such a level usually turns to pull next, which wants the bitmap and
 *                     no queue).  Default 4096 (Kronecker-20: 362 -> 389 GTEPS).
 *   DAWN_PARAM_CLUSTER_START  1: every push/auto dawn_sssp on a graph with n <= 20,971,520
 *                     starts on ONE 16-CTA thread-block cluster with the visited bitmap and the
 *                     frontier queues in distributed shared memory (k_narrow), and hands over to
 *                     the grid-wide kernel when a queue overflows or the next frontier's rows
 *                     exceed DAWN_PARAM_CLUSTER_HANDOVER_EDGES arcs.  0: grid-wide kernel only.
 *                     Default (set at load): 1 when at least half of the sampled arcs join
 *                     vertices whose visited words live in the same CTA (meshes, road networks:
 *                     ids follow space), else 0.
 *   DAWN_PARAM_CLUSTER_HANDOVER_EDGES  see above.  Default: unlimited for the local graphs
 *                     above (the cluster keeps the whole search), else 1024.  Values >= 1.8e19
 *                     mean unlimited.                                                          */
typedef enum {
  DAWN_PARAM_ALPHA = 0,
  DAWN_PARAM_BETA = 1,
  DAWN_PARAM_MS_ALPHA = 2,
  DAWN_PARAM_BITMAP_PUSH_EDGES = 3,
  DAWN_PARAM_SOLO_EDGES = 4,
  DAWN_PARAM_CLUSTER_START = 5,
  DAWN_PARAM_CLUSTER_HANDOVER_EDGES = 6,
  DAWN_PARAM_BITMAP_PUSH_GROW_EDGES = 7,
  DAWN_PARAM_NARROW_QUEUE_CAP = 8, /* lowers k_narrow's per-CTA queue capacity (entries, >= 32;
                                      capped at the load-time capacity).  Only for tests that
                                      force queue-overflow hand-overs; speed only.            */
  DAWN_PARAM_BATCH_LANES = 9,      /* dawn_sssp_batch on the grid-wide kernel runs this many
                                      searches at once, each on 1/lanes of the SMs with its own
                                      per-search state and stream (the sources are
                                      independent).  Lanes run the 2-CTA/SM
                                      kernel.  1 .. 16 (n <= 2^22) or 1 .. 8 (larger n; 1 with
                                      DAWN_GRAPH_LEAN).  Default set at
                                      load from B200 measurements.              */
  DAWN_PARAM_WEIGHT_DELTA = 12,    /* dawn_wsssp near/far step: a round expands only frontier
                                      vertices with d < T (the others stay in the frontier); T
                                      moves to (minimum frontier distance) + delta when no
                                      frontier vertex lies below it.  0 = off (every frontier
                                      vertex each round).  Speed only, never results.         */
  DAWN_PARAM_MS_LANES = 11,        /* dawn_msssp / dawn_apsp / dawn_apsp_rows run this many
                                      256-source batches at once, each on 1/lanes of the SMs with
                                      its own bit-parallel state and stream (independent sources,
                                      PAPER L303-308).  1 .. 3 for n <= 2^22, else 1.  Default
                                      set at load from B200 measurements.      */
  DAWN_PARAM_BATCH_DYNAMIC = 13,   /* 1: the batch lanes of dawn_sssp_batch take the batch's
                                      sources one at a time from a shared counter (each lane
                                      claims its next index when its current search ends), so
                                      the lanes finish together whatever the
                                      per-source cost; 0: lane l runs the fixed contiguous share
                                      [k*l/lanes, k*(l+1)/lanes).  Default 1 (B200:
                                      Kronecker-24 +1.7%, Kronecker-20 +5%).  Which lane runs a
                                      source never changes its row or statistics.  Speed only. */
  DAWN_PARAM_DENSE_MAX_ENTRIES = 10 /* dense distance outputs (dawn_msssp dist, one piece of
                                      dawn_apsp_rows) are refused with DAWN_ERR_CAPACITY when
                                      rows * n >= this ("dense-matrix mode refused
                                      above a configurable threshold").  Default and maximum
                                      2^40 entries.  Changes admission only, never results.    */
} dawn_param;

/* Set one tunable (INVALID_ARGUMENT for an unknown key or a negative value). */
dawn_status dawn_graph_set_param(dawn_graph g, dawn_param key, double value);
/* Read one tunable's current value (the load-time default until set). */
dawn_status dawn_graph_get_param(dawn_graph g, dawn_param key, double *value);

/*
 * Single-source shortest paths (SSSP), one enqueue: initialisation, every level (push or
 * pull, chosen on the device) and the per-source statistics run in ONE persistent kernel;
 * the frontier-empty test is on the device (no host round trip per level; PAPER L174-179
 * conditions 1-2, Algorithm 2 lines 15-17).
 *   source   vertex id in [0, n)                               -> else DAWN_ERR_BOUNDS
 *   variant  DAWN_AUTO / DAWN_PUSH / DAWN_PULL                   -> else INVALID_ARGUMENT
 *   dist     device uint32[n] output (fully overwritten)
 *   stats    device dawn_sssp_stats* or NULL
 */
dawn_status dawn_sssp(dawn_graph g, int64_t source, uint32_t variant, uint32_t *dist,
                      dawn_sssp_stats *stats, void *stream);

/*
 * k single-source searches with the same results as k dawn_sssp calls (the
 * sources are independent), on one stream with no host work between them:
 *   - graphs small enough for the one-CTA kernel: ONE launch of min(k, #SMs) CTAs, each holding
 *     the CSR in its shared memory and running searches b, b + grid, ... (concurrently);
 *   - graphs dawn_sssp starts on the cluster kernel: per search, k_narrow then k_sssp, both
 *     reading the source id from the device array;
 *   - otherwise ONE launch of the grid-wide kernel running the k searches one after the other
 *     (a grid barrier between searches instead of a kernel boundary).
 *   sources  DEVICE uint32[k], each in [0, n).  The list is validated ON THE DEVICE before any
 *            search starts (every kernel of the call checks the whole list first): if an id is
 *            >= n, nothing is written (dist, stats untouched) and the handle's sticky error flag
 *            is set; since the array is not read on the host the call itself returns DAWN_OK and
 *            dawn_graph_check() reports DAWN_ERR_BOUNDS (validation before work).
 *   dist     device uint32[k][n] (row i for sources[i], fully overwritten)
 *   stats    device dawn_sssp_stats[k] or NULL
 * k == 0 is a no-op; k >= 2^32 -> CAPACITY.
 */
dawn_status dawn_sssp_batch(dawn_graph g, const uint32_t *sources, int64_t k, uint32_t variant,
                            uint32_t *dist, dawn_sssp_stats *stats, void *stream);

/*
 * Multi-source: k sources (HOST array; all validated before any work),
 * processed DAWN_MS_BATCH (256) at a time by the bit-parallel kernel: each vertex holds four
 * 64-bit words, bit j of the batch's word w = source DAWN_MS_BATCH*b + 64w + j, so one adjacency
 * pass serves 256 BFS trees (a 32-byte word = one L2 sector).
 *   dist   device uint32[k][n] (source-major) or NULL.  k*n must be below
 *          DAWN_PARAM_DENSE_MAX_ENTRIES (default 2^40) else CAPACITY: stream the rows with
 *          dawn_apsp_rows instead.
 *   rec    device dawn_record[k] or NULL (record i belongs to sources[i]).
 * Repeated sources give identical rows and records.
 */
dawn_status dawn_msssp(dawn_graph g, const int64_t *sources, int64_t k, uint32_t *dist,
                       dawn_record *rec, void *stream);

/*
 * The host-side shard rule of dawn_apsp: the sources are cut into DAWN_MS_BATCH-source batches
 * in the given order; batch b belongs to rank (b mod world).  Writes the indices (into sources[])
 * owned by `rank`, ascending, into idx (capacity cap) and their count into *count.  Pure host
 * function, no device work.
 */
dawn_status dawn_apsp_shard(int64_t k, int32_t rank, int32_t world, int64_t *idx, int64_t cap,
                            int64_t *count);

/*
 * APSP records for this rank's shard (PAPER E11-E12 L303-308: APSP = one SOVM per source; the
 * caller passes e.g. the vertices of the largest WCC).  Computes the records of the sources
 * dawn_apsp_shard() assigns to `rank`, in that order, into rec[0 .. *n_written).  The caller
 * gathers the shards across ranks (torch.distributed / NCCL all-gather).
 *   sources  HOST int64[k], all in [0, n)       rec  device dawn_record[cap]
 *   n_written HOST, receives the shard size (known before any work; CAPACITY if > cap).
 */
dawn_status dawn_apsp(dawn_graph g, const int64_t *sources, int64_t k, int32_t rank, int32_t world,
                      dawn_record *rec, int64_t cap, int64_t *n_written, void *stream);

/*
 * All-pairs distance ROWS streamed to host memory through a caller sink ("for
 * large n a streaming per-row sink must be supplied"; the dense k x n matrix of dawn_msssp is
 * refused above DAWN_PARAM_DENSE_MAX_ENTRIES).  Row i = the distances from sources[i] (the
 * bit-parallel kernel, 256 sources per pass), delivered in order in pieces of `chunk` rows:
 *   piece p is computed on `stream` into dev_stage[p % 2], copied on an internal stream into
 *   host_stage[p % 2], and handed to sink(user, first_row, rows, host_rows) on the CALLING
 *   thread while piece p + 1 computes.  host_rows (rows x n uint32, row-major) is valid only
 *   during the sink call.  The sink returns 0 to continue; a nonzero return stops the call
 *   (DAWN_ERR_INVALID_ARGUMENT, rows already delivered stay delivered).
 *   sources     HOST int64[k], all in [0, n) (validated before any work -> DAWN_ERR_BOUNDS)
 *   chunk       rows per piece, >= 1 (a multiple of DAWN_MS_BATCH avoids partial passes);
 *               chunk * n >= DAWN_PARAM_DENSE_MAX_ENTRIES -> DAWN_ERR_CAPACITY
 *   dev_stage   DEVICE uint32[2 * chunk * n], caller-owned scratch
 *   host_stage  HOST uint32[2 * chunk * n], caller-owned; pinned (page-locked) memory makes the
 *               copies asynchronous
 * Returns when every row was delivered (synchronous in the host sense).  CONFIG on a
 * DAWN_GRAPH_LEAN handle.  Not concurrent with other calls on g.
 */
typedef int (*dawn_row_sink)(void *user, int64_t first_row, int64_t rows, const uint32_t *host_rows);
dawn_status dawn_apsp_rows(dawn_graph g, const int64_t *sources, int64_t k, int64_t chunk,
                           uint32_t *dev_stage, uint32_t *host_stage, dawn_row_sink sink,
                           void *user, void *stream);

/* Copy the per-level trace of the last dawn_sssp call (graph loaded with DAWN_GRAPH_TRACE)
 * into host_out[0 .. min(cap, levels+1)); *count receives the number of records.  With
 * cap >= DAWN_TRACE_CAP, host_out[DAWN_TRACE_CAP - 1] also receives the grid-wide kernel's
 * timeline record (t_ns = kernel entry, t_first = initialisation done, t_last = last level
 * done).  Synchronises `stream`.  CONFIG if the graph was loaded without DAWN_GRAPH_TRACE.   */
#define DAWN_TRACE_CAP 65536
dawn_status dawn_graph_trace(dawn_graph g, dawn_trace_rec *host_out, int64_t cap, int64_t *count,
                             void *stream);

/* Synchronise `stream` and report deferred errors of this handle: DAWN_ERR_BOUNDS if a
 * dawn_sssp_batch enqueued since the last check met a device source id outside [0, n) (that
 * call wrote nothing; the flag is cleared by this call), DAWN_ERR_CUDA if the stream holds a
 * CUDA error, else DAWN_OK.                                                                   */
dawn_status dawn_graph_check(dawn_graph g, void *stream);

/*
 * The largest weakly connected component (Table 1: S_wcc / E_wcc; the APSP
 * source set of E11-E12, L303-308), computed on the device: lock-free union-find hooking over
 * every arc (a directed arc joins its endpoints' components), the larger root hooked onto the
 * smaller so a root is its component's minimum id; then node and arc counts per component.
 * "Largest" = most nodes, ties -> more arcs, then the smaller minimum vertex id (DESIGN.md
 * reading Q15).  Uses the handle's frontier scratch: not concurrent with other calls on g.
 *   sources_out  HOST int64[n] or NULL: the component's vertices, ascending
 *   k            HOST, receives the component's node count S_wcc
 *   arcs         HOST or NULL, receives E_wcc = the arcs whose source lies in the component
 * Synchronises `stream`.  Errors: INVALID_ARGUMENT, CUDA.
 */
dawn_status dawn_largest_wcc(dawn_graph g, int64_t *sources_out, int64_t *k, uint64_t *arcs,
                             void *stream);

/* Executed-schedule counters of the bit-parallel kernel (dawn_msssp / dawn_apsp), summed over
 * every launch on this handle since load or the previous read, then reset.  Synchronises
 * `stream`.  host_out[0] levels run (over all batches), [1] adjacency entries gathered (push
 * arcs of active rows + pull in-edge probes; each costs a 4-B index and a 32-B word gather),
 * [2] 64-bit word reductions issued (red.or), [3] 256-source batches.  Measurement only
 * (bench.py derives the executed bytes B_exec of SURVEY §8(d) from them).                   */
dawn_status dawn_graph_ms_counters(dawn_graph g, uint64_t *host_out, void *stream);

/*
 * Compact distance rows for transfer: out[i] = dist[i] when dist[i] < 255, else 255 (255 =
 * DAWN_UNREACHED, or a finite distance >= 255, which also sets bit 0 of *flags — the caller then
 * transfers that row as uint32).  Low-diameter graphs (every config here has eps <= 8190; the
 * Kronecker ones <= 8) thus move 1 byte per vertex to the host instead of 4.
 *   dist  DEVICE uint32[count], 16-byte aligned;  out  DEVICE uint8[count], 4-byte aligned
 *   flags DEVICE uint32, OR-ed (never cleared by the call).  Enqueue only.
 */
dawn_status dawn_dist_u8(const uint32_t *dist, int64_t count, uint8_t *out, uint32_t *flags,
                         void *stream);

/*
 * The same compaction at 4 bits per vertex (two distances per byte): nibble value
 * min(dist[i], 15), 15 = DAWN_UNREACHED or a finite distance >= 15 (which sets bit 0 of *flags:
 * the caller then transfers the rows with dawn_dist_u8 or as uint32).  Entry 2j goes to the low
 * nibble of out[j], entry 2j + 1 to the high nibble; for an odd count the last high nibble is 15.
 * Kronecker graphs (eps <= 8 on C2/C4) thus move half a byte per vertex to the host.
 *   dist  DEVICE uint32[count], 16-byte aligned;  out  DEVICE uint8[ceil(count / 2)], 4-byte
 *   aligned;  flags DEVICE uint32, OR-ed (never cleared by the call).  Enqueue only.
 * Errors: INVALID_ARGUMENT (NULL with count > 0, misaligned pointers), CUDA.
 */
dawn_status dawn_dist_u4(const uint32_t *dist, int64_t count, uint8_t *out, uint32_t *flags,
                         void *stream);

/*
 * Weighted single-source shortest paths: DAWN's SOVM round over the
 * (min,+) semiring, the extension PAPER.md L596 names as future work (reading Q26 of
 * DESIGN.md): the frontier holds the vertices whose distance dropped in the previous round;
 * a round relaxes their out-arcs, d(u) <- min(d(u), d(v) + w(v,u)); stop when a round improves
 * nothing (<= n-1 rounds).  One persistent kernel, frontier-empty test on the device.
 *   weights  DEVICE uint32[m] aligned with the CSR col array, >= 0 (non-negative weights:
 *            the fixpoint is the shortest-path distance; a zero-weight arc is allowed)
 *   dist     DEVICE uint32[n]: d(s) = 0, DAWN_UNREACHED if no path; path weights saturate at
 *            0xFFFFFFFE (exact while every shortest path weighs < 2^32 - 1)
 *   stats    DEVICE or NULL: levels = rounds that lowered >= 1 distance, reached, edges_reach
 *            (E10 over the reached set), edges_examined = arcs relaxed
 * Errors: INVALID_ARGUMENT, BOUNDS, CUDA.  Uses the handle's frontier state.
 */
dawn_status dawn_wsssp(dawn_graph g, int64_t source, const uint32_t *weights, uint32_t *dist,
                       dawn_sssp_stats *stats, void *stream);
/* k weighted searches from a DEVICE source list (validated on the device before any write, as
 * dawn_sssp_batch: a bad id writes nothing and dawn_graph_check reports DAWN_ERR_BOUNDS), back to
 * back in one persistent launch.
 *   dist DEVICE uint32[k][n], stats DEVICE dawn_sssp_stats[k] or NULL.  k >= 2^32 -> CAPACITY. */
dawn_status dawn_wsssp_batch(dawn_graph g, const uint32_t *sources, int64_t k,
                             const uint32_t *weights, uint32_t *dist, dawn_sssp_stats *stats,
                             void *stream);

/* ------------------------------------------------------------------------------------------
 * Partitioned single-source SSSP over W GPUs: the graph is cut by
 * vertex ranges so each GPU holds ~2m/W arcs — the paper's memory-frugality motivation
 * (E13; L554: graphs a GPU cannot hold).  Rank r owns the ids
 * [lo, hi) = [r*B, min(n, (r+1)*B)), B = ceil(n/W) rounded up to a multiple of 32, and keeps
 * the arcs whose TARGET it owns, grouped twice: by source (the "out-slice", for push = SOVM,
 * Algorithm 2) and by target (the in-rows, for pull = BOVM, Algorithm 1).
 * Every discovery is then local; one level needs only the global frontier F_L, exchanged as an
 * all-gather of per-rank bitmap slices between two dawn_part_step calls (the caller's NCCL
 * all_gather: recv <- concat over ranks of send).  Distances equal dawn_sssp's bit for bit.
 *
 *   dawn_part_begin(p, s, variant, dist_own)     level-0 slice into `send`
 *   loop: all_gather(recv <- send); dawn_part_step(p)   until dawn_part_done() reports 1
 *   dawn_part_finish(p, stats)                   dist_own[t] = d(s, lo + t); statistics
 * Extra steps after convergence are no-ops, so the caller may test dawn_part_done every few
 * levels.  Every rank must call begin/step/finish the same number of times.
 * ------------------------------------------------------------------------------------------ */
typedef struct dawn_part_s *dawn_part;

/* The owned range [lo, hi) of `rank` (empty when rank * B >= n).  Host only. */
dawn_status dawn_part_range(int64_t n, int32_t world, int32_t rank, int64_t *lo, int64_t *hi);

/* Host-side partition builder from the global CSR (host arrays).  With all outputs NULL it only
 * counts *m_r = arcs whose target lies in [lo, hi).  Otherwise (caller-allocated host arrays):
 *   out_rp  int64[n+1], out_col int32[m_r]: the out-slice (row v = v's arcs into the range, in
 *           input order, targets as local ids t = u - lo)
 *   in_rp   int64[hi-lo+1], in_col int32[m_r]: the same arcs by target (sources ascending)
 *   own_deg uint32[hi-lo]: global out-degree of lo + t (the E10 counts)
 * Errors: INVALID_ARGUMENT, INVALID_GRAPH (row_ptr not a CSR, col out of range),
 * CAPACITY (m_r >= 2^32). */
dawn_status dawn_part_build(int64_t n, int64_t m, const int64_t *row_ptr, const int32_t *col,
                            int32_t world, int32_t rank, int64_t *m_r, int64_t *out_rp,
                            int32_t *out_col, int64_t *in_rp, int32_t *in_col, uint32_t *own_deg);

/* Device workspace bytes of one rank's handle (0 if the sizes are unsupported). */
size_t dawn_part_workspace_bytes(int64_t n, int64_t m_r, int32_t world, int32_t rank);

/* Make rank `rank`'s partition resident: the dawn_part_build arrays as DEVICE copies
 * (caller-owned, must outlive the handle), m = arcs of the whole graph.  Synchronises `stream`.
 * Errors: INVALID_ARGUMENT, CAPACITY, WORKSPACE, CUDA. */
dawn_status dawn_part_load(int64_t n, int64_t m, int32_t world, int32_t rank, int64_t m_r,
                           const int64_t *out_rp, const int32_t *out_col, const int64_t *in_rp,
                           const int32_t *in_col, const uint32_t *own_deg, void *workspace,
                           size_t ws_bytes, void *stream, dawn_part *out);
dawn_status dawn_part_destroy(dawn_part p);

/* The exchange buffers inside the workspace: send = this rank's slice (slice_words uint32:
 * 4 header words + B/32 bitmap words), recv = world slices in rank order. */
dawn_status dawn_part_exchange(dawn_part p, uint32_t **send, uint32_t **recv, int64_t *slice_words);

/* Start a search from global `source` (BOUNDS if not in [0, n)); dist_own = DEVICE
 * uint32[hi-lo], fully written by dawn_part_finish. */
dawn_status dawn_part_begin(dawn_part p, int64_t source, uint32_t variant, uint32_t *dist_own,
                            void *stream);
/* One level (reads recv, writes send).  Enqueue only. */
dawn_status dawn_part_step(dawn_part p, void *stream);
/* *done = 1 once the search converged (the frontier is empty on every rank).  Synchronises. */
dawn_status dawn_part_done(dawn_part p, int32_t *done, void *stream);
/* Write dist_own and (DEVICE, or NULL) the search's statistics: levels, reached, edges_reach
 * are global (identical on every rank), edges_examined counts this rank's reads. */
dawn_status dawn_part_finish(dawn_part p, dawn_sssp_stats *stats, void *stream);

/*
 * Fused exchange (the whole partitioned search in ONE persistent kernel per rank): each level
 * the rank writes its slice of the next frontier straight into every rank's receive buffer —
 * plain stores into peer memory over NVLink / NVSwitch, or local memory when ranks share a
 * device — and then adds 1 to every rank's arrival counter (system-scope release); a rank starts
 * the next level once all W slices of it landed.  No NCCL call, host round trip or kernel
 * boundary per level.  All ranks must run dawn_part_fused_sssp concurrently (the kernels wait
 * for each other): on one device, give each rank a share of the SMs with `grid`.
 *   dawn_part_fused_peers  every rank's exchange buffer as mapped in this process (rank order,
 *                          this rank's own included; e.g. CUDA IPC mappings of the peers'
 *                          buffers): peer_recv[q] = DEVICE uint32[2 * world * slice_words]
 *                          (dawn_part_exchange's slice_words), zero-initialised;
 *                          peer_flag[q] = DEVICE uint64 arrival counter, zero-initialised.  The
 *                          buffers are bound to this handle for its lifetime (the counters are
 *                          monotonic across searches).
 *   dawn_part_fused_sssp   one search; dist_own / stats as dawn_part_finish.  grid = CTAs of the
 *                          cooperative launch (0 = the whole device).  Enqueue only.
 * Errors: INVALID_ARGUMENT, BOUNDS, CONFIG (peers not set), CUDA. */
dawn_status dawn_part_fused_peers(dawn_part p, int32_t world, void *const *peer_recv,
                                  void *const *peer_flag);
dawn_status dawn_part_fused_sssp(dawn_part p, int64_t source, uint32_t variant, uint32_t *dist_own,
                                 dawn_sssp_stats *stats, int32_t grid, void *stream);

/* Thread-local description of the last error of this thread ("" if none). */
const char *dawn_last_error(void);

/* Library version string, e.g. "dawn-b200 0.1 sm_100a". */
const char *dawn_version(void);

#ifdef __cplusplus
}
#endif
#endif /* DAWN_H */
