/*
 * hf.h -- C ABI of libhf.so: dependency-ordered propagation over a large DAG on
 * B200 (sm_100a).  The hot path under Heteroflow's million-task timing-analysis
 * workload (arXiv 2203.08395), as named by
 * BASELINE.json:5 (north_star).  Readings R1-R16 are listed in DESIGN.md §2.
 *
 * Conventions for every entry point
 *   - Plain pointers and sizes only.  Functions without a suffix take HOST
 *     pointers and are synchronous (pull/push semantics, PAPER.md:419-435,
 *     495-512).  Functions with the _d suffix take DEVICE pointers (e.g. a torch
 *     tensor's data_ptr()) on the graph's device, enqueue work on the graph's
 *     stream and return without waiting (non-blocking run),
 *     unless stated otherwise.
 *   - The caller owns every array it passes.  hf_graph_create* copies its
 *     inputs; no call keeps a caller pointer after it returns.
 *   - Every call returns an hf_status and never aborts or throws (SPEC.md:129,
 *     446).  hf_last_error() returns a thread-local message for the last
 *     failure on the calling thread.  Errors detected on the device by an
 *     asynchronous _d call (non-finite scenario delay) are latched in the graph
 *     and returned by the next hf_sync() or host-pointer call.  A dataflow wait
 *     that outlives its watchdog (HF_WATCHDOG_SPINS poll rounds; a schedule bug,
 *     never a legal input) is latched the same way and returned as HF_ERR_CUDA.
 *   - Every entry point is one NVTX range named after the call (tracing).
 *   - Indices are int32, values fp32 (IEEE binary32, round-to-nearest-even, no
 *     flush-to-zero).  n, m < 2^31.  -0.0 inputs are canonicalised to +0.0;
 *     NaN / +-inf inputs are rejected with HF_ERR_INVALID_ARG (reading R9).
 *   - A graph is single-owner: do not call into one graph from two threads at
 *     once.
 *
 * Edge ids: edge e is position e of the fan-in CSR (reading R11).
 */
#ifndef HF_H
#define HF_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HF_VERSION 101

/* Largest scenario count of one batch call (s_local); larger -> HF_ERR_INVALID_ARG.
 * (The per-CTA worst-slack table of the kernels holds 4 bytes per scenario.) */
#define HF_MAX_SCENARIOS 8192

typedef struct hf_graph_s *hf_graph; /* opaque; owns device copies of the graph */

typedef enum {
    HF_OK = 0,
    HF_ERR_INVALID_ARG = 1,   /* NULL where required, negative size, non-finite value   */
    HF_ERR_BAD_CSR = 2,       /* malformed CSR, or fan-out is not the fan-in's transpose */
    HF_ERR_CYCLE = 3,         /* graph has a cycle; hf_last_error gives the count of
                                 never-ready nodes      */
    HF_ERR_NOT_LEVELIZED = 4, /* propagate/batch before hf_levelize   */
    HF_ERR_OOM = 5,
    HF_ERR_CUDA = 6,
    HF_ERR_NCCL = 7
} hf_status;

/* Layout of batched scenario delays (reading R12). */
#define HF_LAYOUT_SM 0 /* delays[s*m + e]: one delay set after another              */
#define HF_LAYOUT_MS 1 /* delays[e*S + s]: scenario-minor; the kernels' native layout */

/* Thread-local message describing the last error on this thread ("" if none). */
const char *hf_last_error(void);
/* Static name of a status code. */
const char *hf_status_string(hf_status s);
int hf_version(void);

/*
 * hf_graph_create -- build a graph from CSR fan-in (required) and fan-out
 * (optional), plus per-edge fp32 delays.  SURVEY.md §8(a) a1; "a directed acyclic
 * graph ... nodes = tasks, edges = dependency constraints" PAPER.md:330-331;
 * BASELINE.json:5 "hf_graph_create from CSR fan-in/fan-out arrays plus per-edge
 * weights".
 *   n, m        node and edge counts (n >= 0, m >= 0).
 *   fanin_ptr   [n+1] row offsets by sink node: edges e in [ptr[v], ptr[v+1])
 *               end at v.  ptr[0] = 0, non-decreasing, ptr[n] = m.
 *   fanin_src   [m] source node of each edge, 0 <= src < n.  Multi-edges allowed.
 *   fanout_ptr, fanout_dst   [n+1], [m] fan-out CSR by source, or both NULL
 *               (derived).  If given it must be the fan-in's transpose as a
 *               multiset of (src, dst) pairs, else HF_ERR_BAD_CSR.
 *   delay       [m] delay of edge e (fan-in position), finite; NULL => +0.
 *   device      CUDA device ordinal the graph lives on.
 *   cuda_stream cudaStream_t the graph's work is enqueued on (NULL = legacy default).
 *   out         receives the graph handle.
 * Cycles are NOT detected here (deferred to hf_levelize).
 * hf_graph_create: host pointers.  hf_graph_create_d: device pointers; both
 * synchronise the stream once (validation result).
 */
hf_status hf_graph_create(int32_t n, int32_t m, const int32_t *fanin_ptr,
                          const int32_t *fanin_src, const int32_t *fanout_ptr,
                          const int32_t *fanout_dst, const float *delay, int device,
                          void *cuda_stream, hf_graph *out);
hf_status hf_graph_create_d(int32_t n, int32_t m, const int32_t *fanin_ptr_d,
                            const int32_t *fanin_src_d, const int32_t *fanout_ptr_d,
                            const int32_t *fanout_dst_d, const float *delay_d, int device,
                            void *cuda_stream, hf_graph *out);
hf_status hf_graph_destroy(hf_graph g);
/* Re-target the graph's work to another stream on the same device. */
hf_status hf_graph_set_stream(hf_graph g, void *cuda_stream);
/* Analysis mode of the propagation calls that follow (NEXT-2, SURVEY.md §8(f);
 * PAPER.md:972-974 "analysis mode"; reading R18).  HF_MODE_LATE (default,
 * setup analysis): at = max-plus over fan-in, rat = min-plus over fan-out, slack =
 * fl(rat - at).  HF_MODE_EARLY (hold analysis): at = min over fan-in of
 * fl(at[u] + d), rat = max over fan-out of fl(rat[v] - d) (T at sinks), slack =
 * fl(at - rat); wns is the minimum slack in both modes.  Affects
 * hf_propagate_forward/backward[_d] and hf_run_batch[_d]; hf_critical_path[_d] is
 * defined for late mode only (HF_ERR_INVALID_ARG in early mode).  mode other than
 * 0/1 -> HF_ERR_INVALID_ARG. */
#define HF_MODE_LATE 0
#define HF_MODE_EARLY 1
hf_status hf_graph_set_mode(hf_graph g, int mode);
/* n, m and (after hf_levelize) the number of levels L; any pointer may be NULL.
 * num_levels = -1 while not levelized. */
hf_status hf_graph_info(hf_graph g, int32_t *n, int32_t *m, int32_t *num_levels);
/* Wait for the graph's stream; return (and clear) any latched device-side error. */
hf_status hf_sync(hf_graph g);

/*
 * hf_levelize -- on-device Kahn topological levelization.  SURVEY.md §8(a) a2-a4.
 *   level(v) = 0 for sources, else 1 + max level(pred) (reading R5) -- the index of
 *   the Kahn frontier that releases v (join counters).
 *   order    = node ids stable-sorted by level: ascending id within a level (R6).
 *   level_ptr[k] = first position of level k in order; level_ptr[L] = n.
 * Outputs (each may be NULL): num_levels (host int32), level [n], level_ptr
 * [L+1] (capacity n+1 suffices), order [n].  Synchronous in both variants (L is
 * returned to the host).  On a cycle returns HF_ERR_CYCLE; hf_last_error gives
 * the number of nodes that never become ready; the graph stays un-levelized.
 * n = 0 gives L = 0 and level_ptr = {0}.
 */
hf_status hf_levelize(hf_graph g, int32_t *num_levels, int32_t *level, int32_t *level_ptr,
                      int32_t *order);
hf_status hf_levelize_d(hf_graph g, int32_t *num_levels, int32_t *level_d,
                        int32_t *level_ptr_d, int32_t *order_d);

/*
 * hf_propagate_forward -- max-plus arrival times with the graph's own delays.
 * SURVEY.md §8(a) a5; BASELINE.json:5 "at[v] = max over fan-in of at[u] + d(u,v)".
 *   at_src [n] arrival time of each in-degree-0 node (other entries ignored), or
 *          NULL => +0 (reading R2).
 *   at     [n] output.
 * Requires hf_levelize (else HF_ERR_NOT_LEVELIZED).
 */
hf_status hf_propagate_forward(hf_graph g, const float *at_src, float *at);
hf_status hf_propagate_forward_d(hf_graph g, const float *at_src_d, float *at_d);

/*
 * hf_propagate_backward -- min-plus required times, fused slack and worst slack.
 * SURVEY.md §8(a) a6; BASELINE.json:5 "min-plus required time", "worst slack".
 *   t_req  required time T applied at every out-degree-0 node (reading R3).
 *   at     [n] arrival times from hf_propagate_forward (input).
 *   rat    [n] output: rat[u] = min over fan-out of fl(rat[v] - d(u,v)).
 *   slack  [n] output fl(rat - at), or NULL.
 *   wns    [1] output min over all nodes of slack (+inf when n = 0), or NULL (R4).
 */
hf_status hf_propagate_backward(hf_graph g, float t_req, const float *at, float *rat,
                                float *slack, float *wns);
hf_status hf_propagate_backward_d(hf_graph g, float t_req, const float *at_d, float *rat_d,
                                  float *slack_d, float *wns_d);

/*
 * hf_run_batch -- S independent what-if delay sets over the same graph (timing
 * views; BASELINE.json:10), forward + backward + worst slack
 * per scenario, then (optionally) an NCCL all-gather of the per-rank worst
 * slacks (BASELINE.json:5 "NCCL over NVLink used only to gather worst slack").
 *   s_local    number of scenarios on this rank, 1 <= s_local <= HF_MAX_SCENARIOS;
 *              HF_ERR_INVALID_ARG also when the pass would exceed 2^31 - 1 warp
 *              tasks (odd s_local on a graph of tens of millions of nodes).
 *   delays     [m*s_local] scenario delays in `layout` (HF_LAYOUT_MS preferred).
 *   t_req      [s_local] required time per scenario.
 *   at_src     [n] source arrival times shared by all scenarios, or NULL => +0.
 *   wns_local  [s_local] output worst slack per scenario.
 *   at, rat    (_d only) [n*s_local] outputs, node-major / scenario-minor, or NULL.
 *   nccl_comm  ncclComm_t from hf_nccl_comm_init, or NULL (no gather).
 *   wns_all    [s_local*nranks] gathered worst slacks (rank r's block at r*s_local),
 *              or NULL; required when nccl_comm is given.
 * The delays of the graph itself are not used.  Requires hf_levelize.
 */
hf_status hf_run_batch(hf_graph g, int32_t s_local, const float *delays, int layout,
                       const float *t_req, const float *at_src, float *wns_local,
                       void *nccl_comm, float *wns_all);
hf_status hf_run_batch_d(hf_graph g, int32_t s_local, const float *delays_d, int layout,
                         const float *t_req_d, const float *at_src_d, float *wns_local_d,
                         float *at_d, float *rat_d, void *nccl_comm, float *wns_all_d);

/*
 * hf_analyze -- the whole hot path in one call from HOST buffers: graph create
 * (SURVEY.md §8(a) a1), levelize (a2-a4), forward + backward + worst slack for
 * s_local delay sets (a5-a7), as hf_graph_create + hf_levelize + hf_run_batch.
 * The scenario data (the bulk of the host->device bytes) is uploaded on a second
 * stream while the graph is built and levelized; with pinned host buffers the
 * upload overlaps that work.
 *   n, m, fanin_ptr, fanin_src, delay   as hf_graph_create (fan-out derived).
 *   s_local, delays [m*s_local] in HF_LAYOUT_MS, t_req [s_local], at_src [n] or
 *   NULL => +0     as hf_run_batch (no NCCL gather).
 *   wns_local  [s_local] output worst slack per scenario.
 *   num_levels output L, or NULL.
 *   device, cuda_stream   as hf_graph_create.
 *   out_graph  receives the levelized graph (reusable with hf_run_batch; destroy
 *              with hf_graph_destroy), or NULL to destroy it before returning.
 * Synchronous: returns after wns_local is written; the host buffers may be reused
 * on return.  Errors as the three calls it stands for (nothing is returned in
 * out_graph on error).
 */
hf_status hf_analyze(int32_t n, int32_t m, const int32_t *fanin_ptr, const int32_t *fanin_src,
                     const float *delay, int32_t s_local, const float *delays, const float *t_req,
                     const float *at_src, float *wns_local, int32_t *num_levels, int device,
                     void *cuda_stream, hf_graph *out_graph);

/* NEXT-1: critical-path trace-back (PAPER.md:1002-1003
 * "extract graph information (critical paths, ...)"; reading R17).
 * Per scenario s: the endpoint is the sink (out-degree 0) with the smallest slack
 * fl(T_s - at_s[sink]), ties by the smallest node id; from it the path steps to the
 * source of the fan-in edge e attaining the max, fl(at_s[src e] + d_s[e]) == at_s[v],
 * ties by the smallest fan-in edge id, until a source (in-degree 0).
 * path[s*max_len + i]: i-th node from the endpoint (endpoint first, source last).
 *
 * hf_critical_path_d: device pointers, stream-ordered.  delays [m][S] in fan-in
 *   edge order (NULL: the graph's own delays, S must be 1); at [n][S] must be the
 *   forward result of those delays (hf_propagate_forward_d / hf_run_batch_d with
 *   at output); t_req [S] or NULL (t_scalar for all); path [S][max_len];
 *   path_len [S] receives the length, or -1 when at is not a forward result of the
 *   delays or the path is longer than max_len (max_len >= number of levels is
 *   always enough).  The graph need not be levelized.
 * hf_critical_path: host pointers, one delay set (the graph's), synchronous;
 *   HF_ERR_INVALID_ARG when path_len would be -1. */
hf_status hf_critical_path_d(hf_graph g, int32_t S, const float *delays, const float *at,
                             const float *t_req, float t_scalar, int32_t max_len,
                             int32_t *path, int32_t *path_len);
hf_status hf_critical_path(hf_graph g, const float *at, float t_req, int32_t max_len,
                           int32_t *path, int32_t *path_len);
/* hf_critical_paths_d: top-K endpoints per scenario (SURVEY.md §8(f) NEXT-1
 *   "with optional top-k endpoints").  The K sinks with the smallest (slack, node
 *   id), in that order, each traced as above.  endpoints [S][K] (or NULL) receives
 *   the sink ids, -1 past the number of sinks; path [S][K][max_len]; path_len
 *   [S][K] as for hf_critical_path_d, 0 past the number of sinks.  K = 1 gives
 *   hf_critical_path_d.  Device pointers, stream-ordered.  2 <= K <= 32: one
 *   selection for all K ranks (per-block sorted lists merged per scenario: 2
 *   launches, one pass over the n x S slacks) + 1 trace launch; K > 32: one
 *   selection pass per rank (K + 1 launches). */
hf_status hf_critical_paths_d(hf_graph g, int32_t S, const float *delays, const float *at,
                              const float *t_req, float t_scalar, int32_t K, int32_t max_len,
                              int32_t *endpoints, int32_t *path, int32_t *path_len);


/* NEXT-4: greedy maximal independent set (PAPER.md:1141-1150
 * "a parallel maximal independent set finding step using Blelloch's Algorithm";
 * DESIGN.md reading R19).  The graph is the undirected graph of the DAG's edges;
 * the result is the lexicographically-first MIS for the vertex order (prio[v], v):
 * v is in the set iff none of its neighbours earlier in that order is.
 * prio [n] int32 keys (ties broken by node id); in_set [n] bytes, 1 = in the set.
 * hf_mis_d: device pointers, stream-ordered.  hf_mis: host pointers, synchronous.
 * The graph need not be levelized. */
hf_status hf_mis_d(hf_graph g, const int32_t *prio, uint8_t *in_set);
hf_status hf_mis(hf_graph g, const int32_t *prio, uint8_t *in_set);

/* NCCL bootstrap (libnccl.so.2 is loaded on first use).  Rank 0 calls
 * hf_nccl_unique_id and broadcasts the 128 bytes (e.g. over torch.distributed);
 * every rank then calls hf_nccl_comm_init with its rank on its device. */
hf_status hf_nccl_unique_id(void *id128);
hf_status hf_nccl_comm_init(const void *id128, int rank, int nranks, int device, void **comm);
hf_status hf_nccl_comm_destroy(void *comm);

/* Device timing (CUDA events on the graph's stream) and launch count.
 * hf_profile_enable(g, 1) starts recording; hf_profile_read synchronises and
 * returns the milliseconds of the most recent hf_levelize call (whole call) and
 * of the most recent forward / backward propagation KERNEL (one persistent
 * launch each, all scenarios of the batch), and the total number of kernels
 * libhf launched on this graph so far. */
hf_status hf_profile_enable(hf_graph g, int on);
hf_status hf_profile_read(hf_graph g, float *ms_levelize, float *ms_forward,
                          float *ms_backward, int64_t *kernel_launches);
/* Milliseconds of the propagation phase of the most recent hf_run_batch call: from
 * the first propagation kernel to the worst slacks (forward and backward kernels
 * run concurrently on two streams, then the slack/WNS pass; ms_forward/ms_backward
 * above are the two kernels' own, overlapping, durations). */
hf_status hf_profile_read_batch(hf_graph g, float *ms_batch_propagation);

#ifdef __cplusplus
}
#endif
#endif /* HF_H */
