/*
 * oracle.c -- plain, slow, obviously correct CPU oracle for the DAG-propagation
 * hot path.  TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load it.  It shares no
 * code, header, table or helper with the CUDA path (paper_2203_08395_b200/).
 *
 * Compiled with: gcc -std=c11 -O2 -fno-fast-math -ffp-contract=off -fPIC -shared
 * (single precision adds are IEEE binary32 round-to-nearest-even on x86-64 SSE;
 * no contraction, no reassociation).
 *
 * What it computes (passages it follows):
 *   - the task graph is a DAG whose edges u->v mean "u runs before v", and a
 *     graph is valid "as long as no cycles are formed"
 *   - a node becomes ready when all its predecessors finished (join counter)
 *                                                           PAPER.md:840-848
 *   - acyclicity checked with Kahn's algorithm at submission SPEC.md:145
 *   - level(v) = 0 for sources, else 1 + max level(pred)    DESIGN.md reading R5
 *   - canonical order = ascending node id within a level    DESIGN.md reading R6
 *   - at[v] = max over fan-in of fl(at[u] + d(u,v))          BASELINE.json:5 (north_star)
 *   - rat[u] = min over fan-out of fl(rat[v] - d(u,v)), T at sinks
 *                                                           BASELINE.json:5; reading R3
 *   - slack = fl(rat - at), wns = min slack                  BASELINE.json:5; reading R4
 *   - batched what-if scenarios = independent delay sets     PAPER.md:969-980; BASELINE.json:10
 *   - critical path of the worst endpoint (argmax trace-back) PAPER.md:1002-1003; reading R17
 *     (and of the top-K endpoints by (slack, id))
 *   - greedy MIS by priority (Blelloch's lexicographically-first MIS)
 *                                                           PAPER.md:1141-1150; reading R19
 *   - early (hold) mode: min-plus forward, max-plus backward, slack = at - rat
 *                                                           PAPER.md:972-974 ("analysis mode"); reading R18
 *
 * Every function is a direct transcription of SURVEY.md §8(c)'s pseudo-code:
 * FIFO Kahn, then one sequential sweep over the topological order.  Status
 * codes: 0 ok, 1 invalid argument (non-finite value), 2 bad CSR, 3 cycle.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OR_OK 0
#define OR_INVALID 1
#define OR_BAD_CSR 2
#define OR_CYCLE 3

/* -0.0f -> +0.0f; everything else unchanged (reading R9). */
static float canon(float x) { return x == 0.0f ? 0.0f : x; }

/* CSR fan-in well-formedness: in_ptr[0]=0, non-decreasing, in_ptr[n]=m, 0<=src<n. */
int oracle_check_csr(int32_t n, int32_t m, const int32_t *in_ptr, const int32_t *in_src) {
    if (n < 0 || m < 0) return OR_BAD_CSR;
    if (in_ptr[0] != 0 || in_ptr[n] != m) return OR_BAD_CSR;
    for (int32_t v = 0; v < n; ++v)
        if (in_ptr[v + 1] < in_ptr[v]) return OR_BAD_CSR;
    for (int32_t e = 0; e < m; ++e)
        if (in_src[e] < 0 || in_src[e] >= n) return OR_BAD_CSR;
    return OR_OK;
}

/* Fan-out CSR = transpose of the fan-in CSR: stable counting sort of the fan-in
 * edges by source.  out_eid[k] = fan-in edge id of fan-out position k. */
void oracle_fanout(int32_t n, int32_t m, const int32_t *in_ptr, const int32_t *in_src,
                   int32_t *out_ptr, int32_t *out_dst, int32_t *out_eid) {
    for (int32_t u = 0; u <= n; ++u) out_ptr[u] = 0;
    for (int32_t e = 0; e < m; ++e) out_ptr[in_src[e] + 1] += 1;
    for (int32_t u = 0; u < n; ++u) out_ptr[u + 1] += out_ptr[u];
    int32_t *cursor = (int32_t *)malloc(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
    for (int32_t u = 0; u < n; ++u) cursor[u] = out_ptr[u];
    for (int32_t v = 0; v < n; ++v)
        for (int32_t e = in_ptr[v]; e < in_ptr[v + 1]; ++e) {
            int32_t k = cursor[in_src[e]]++;
            out_dst[k] = v;
            out_eid[k] = e;
        }
    free(cursor);
}

static int cmp_i32(const void *a, const void *b) {
    int32_t x = *(const int32_t *)a, y = *(const int32_t *)b;
    return (x > y) - (x < y);
}

/* Caller-supplied fan-out must be the transpose of the fan-in as a multiset:
 * same out_ptr, and each row holds the same destinations (compared sorted). */
int oracle_check_fanout(int32_t n, int32_t m, const int32_t *in_ptr, const int32_t *in_src,
                        const int32_t *fo_ptr, const int32_t *fo_dst) {
    int32_t *op = (int32_t *)malloc(sizeof(int32_t) * (size_t)(n + 1));
    int32_t *od = (int32_t *)malloc(sizeof(int32_t) * (size_t)(m > 0 ? m : 1));
    int32_t *oe = (int32_t *)malloc(sizeof(int32_t) * (size_t)(m > 0 ? m : 1));
    int32_t *row = (int32_t *)malloc(sizeof(int32_t) * (size_t)(m > 0 ? m : 1));
    int rc = OR_OK;
    oracle_fanout(n, m, in_ptr, in_src, op, od, oe);
    for (int32_t u = 0; u <= n && rc == OR_OK; ++u)
        if (fo_ptr[u] != op[u]) rc = OR_BAD_CSR;
    for (int32_t u = 0; u < n && rc == OR_OK; ++u) {
        int32_t b = op[u], len = op[u + 1] - op[u];
        for (int32_t k = 0; k < len; ++k) {
            if (fo_dst[b + k] < 0 || fo_dst[b + k] >= n) { rc = OR_BAD_CSR; break; }
            row[k] = fo_dst[b + k];
        }
        if (rc != OR_OK) break;
        qsort(row, (size_t)len, sizeof(int32_t), cmp_i32);
        /* derived rows are already ascending (fan-in edge ids ascend with sink id) */
        for (int32_t k = 0; k < len; ++k)
            if (row[k] != od[b + k]) { rc = OR_BAD_CSR; break; }
    }
    free(op); free(od); free(oe); free(row);
    return rc;
}

/* FIFO Kahn levelization (SURVEY.md §8(c) pseudo-code, lines "indeg..L").
 * Outputs: topo[n] (FIFO order, first *n_topo entries valid), level[n],
 * level_ptr[L+1], order[n], *num_levels.  On a cycle: returns OR_CYCLE and
 * *n_unready = n - |topo| (nodes that never become ready). */
int oracle_levelize(int32_t n, int32_t m, const int32_t *in_ptr, const int32_t *in_src,
                    int32_t *topo, int32_t *n_topo, int32_t *level, int32_t *level_ptr,
                    int32_t *order, int32_t *num_levels, int32_t *n_unready) {
    int rc = oracle_check_csr(n, m, in_ptr, in_src);
    if (rc) return rc;
    int32_t *out_ptr = (int32_t *)malloc(sizeof(int32_t) * (size_t)(n + 1));
    int32_t *out_dst = (int32_t *)malloc(sizeof(int32_t) * (size_t)(m > 0 ? m : 1));
    int32_t *out_eid = (int32_t *)malloc(sizeof(int32_t) * (size_t)(m > 0 ? m : 1));
    int32_t *indeg = (int32_t *)malloc(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
    oracle_fanout(n, m, in_ptr, in_src, out_ptr, out_dst, out_eid);
    int32_t head = 0, tail = 0;
    for (int32_t v = 0; v < n; ++v) {
        indeg[v] = in_ptr[v + 1] - in_ptr[v];
        level[v] = 0;
        if (indeg[v] == 0) topo[tail++] = v;          /* Q = sources, ascending id */
    }
    while (head < tail) {
        int32_t u = topo[head++];
        for (int32_t k = out_ptr[u]; k < out_ptr[u + 1]; ++k) {
            int32_t v = out_dst[k];
            if (level[u] + 1 > level[v]) level[v] = level[u] + 1;
            if (--indeg[v] == 0) topo[tail++] = v;
        }
    }
    *n_topo = tail;
    *n_unready = n - tail;
    if (tail < n) {
        rc = OR_CYCLE;
    } else {
        int32_t L = 0;
        for (int32_t v = 0; v < n; ++v)
            if (level[v] + 1 > L) L = level[v] + 1;
        *num_levels = L;
        for (int32_t l = 0; l <= L; ++l) level_ptr[l] = 0;
        for (int32_t v = 0; v < n; ++v) level_ptr[level[v] + 1] += 1;
        for (int32_t l = 0; l < L; ++l) level_ptr[l + 1] += level_ptr[l];
        int32_t *cursor = (int32_t *)malloc(sizeof(int32_t) * (size_t)(L > 0 ? L : 1));
        for (int32_t l = 0; l < L; ++l) cursor[l] = level_ptr[l];
        for (int32_t v = 0; v < n; ++v) order[cursor[level[v]]++] = v;
        free(cursor);
    }
    free(out_ptr); free(out_dst); free(out_eid); free(indeg);
    return rc;
}

/* Forward max-plus (late mode) or min-plus (early mode, NEXT-2) over the
 * topological order.  at_src may be NULL (=> +0).  delay[m] indexed by fan-in
 * position; stride = distance between consecutive edges' delays (1 for a single
 * delay set, S for the [m][S] layout). */
static void forward_pass(int32_t n, const int32_t *in_ptr, const int32_t *in_src,
                         const float *delay, int64_t stride, const float *at_src,
                         const int32_t *topo, float *at, int early) {
    for (int32_t i = 0; i < n; ++i) {
        int32_t v = topo[i];
        if (in_ptr[v + 1] == in_ptr[v]) {
            at[v] = at_src ? canon(at_src[v]) : 0.0f;
            continue;
        }
        float best = 0.0f;
        for (int32_t e = in_ptr[v]; e < in_ptr[v + 1]; ++e) {
            float x = at[in_src[e]] + canon(delay[(int64_t)e * stride]);
            if (e == in_ptr[v] || (early ? x < best : x > best)) best = x;   /* keeps first */
        }
        at[v] = best;
    }
}

/* Backward min-plus (late) or max-plus (early) over the reversed topological
 * order, then slack (late: rat - at; early / hold: at - rat) and its minimum. */
static float backward_pass(int32_t n, const int32_t *out_ptr, const int32_t *out_dst,
                           const int32_t *out_eid, const float *delay, int64_t stride,
                           float t_req, const int32_t *topo, const float *at, float *rat,
                           float *slack, int early) {
    float T = canon(t_req);
    for (int32_t i = n - 1; i >= 0; --i) {
        int32_t u = topo[i];
        if (out_ptr[u + 1] == out_ptr[u]) {
            rat[u] = T;
            continue;
        }
        float best = 0.0f;
        for (int32_t k = out_ptr[u]; k < out_ptr[u + 1]; ++k) {
            float x = rat[out_dst[k]] - canon(delay[(int64_t)out_eid[k] * stride]);
            if (k == out_ptr[u] || (early ? x > best : x < best)) best = x;
        }
        rat[u] = best;
    }
    float wns = INFINITY;
    for (int32_t v = 0; v < n; ++v) {
        float s = early ? at[v] - rat[v] : rat[v] - at[v];
        if (slack) slack[v] = s;
        if (s < wns) wns = s;
    }
    return wns;
}

static int all_finite(const float *x, int64_t count) {
    for (int64_t i = 0; i < count; ++i)
        if (!isfinite(x[i])) return 0;
    return 1;
}

/* Single-graph forward: at[n] (early != 0: min-plus, the hold-analysis arrival). */
int oracle_forward_mode(int32_t n, int32_t m, const int32_t *in_ptr, const int32_t *in_src,
                        const float *delay, const float *at_src, const int32_t *topo, float *at,
                        int early) {
    if (delay && !all_finite(delay, m)) return OR_INVALID;
    if (at_src && !all_finite(at_src, n)) return OR_INVALID;
    static const float zero = 0.0f;
    if (!delay) {
        /* NULL delays => +0 on every edge */
        forward_pass(n, in_ptr, in_src, &zero, 0, at_src, topo, at, early);
        return OR_OK;
    }
    forward_pass(n, in_ptr, in_src, delay, 1, at_src, topo, at, early);
    return OR_OK;
}
int oracle_forward(int32_t n, int32_t m, const int32_t *in_ptr, const int32_t *in_src,
                   const float *delay, const float *at_src, const int32_t *topo, float *at) {
    return oracle_forward_mode(n, m, in_ptr, in_src, delay, at_src, topo, at, 0);
}

/* Single-graph backward: rat[n], slack[n] (nullable), *wns (early: hold mode). */
int oracle_backward_mode(int32_t n, int32_t m, const int32_t *in_ptr, const int32_t *in_src,
                         const float *delay, float t_req, const int32_t *topo, const float *at,
                         float *rat, float *slack, float *wns, int early) {
    if (delay && !all_finite(delay, m)) return OR_INVALID;
    if (!isfinite(t_req)) return OR_INVALID;
    int32_t *out_ptr = (int32_t *)malloc(sizeof(int32_t) * (size_t)(n + 1));
    int32_t *out_dst = (int32_t *)malloc(sizeof(int32_t) * (size_t)(m > 0 ? m : 1));
    int32_t *out_eid = (int32_t *)malloc(sizeof(int32_t) * (size_t)(m > 0 ? m : 1));
    oracle_fanout(n, m, in_ptr, in_src, out_ptr, out_dst, out_eid);
    static const float zero = 0.0f;
    float w = backward_pass(n, out_ptr, out_dst, out_eid, delay ? delay : &zero,
                            delay ? 1 : 0, t_req, topo, at, rat, slack, early);
    if (wns) *wns = w;
    free(out_ptr); free(out_dst); free(out_eid);
    return OR_OK;
}
int oracle_backward(int32_t n, int32_t m, const int32_t *in_ptr, const int32_t *in_src,
                    const float *delay, float t_req, const int32_t *topo, const float *at,
                    float *rat, float *slack, float *wns) {
    return oracle_backward_mode(n, m, in_ptr, in_src, delay, t_req, topo, at, rat, slack, wns, 0);
}

/* ---- batched scenarios: the same passes per delay set --------------------- */
typedef struct {
    int32_t n, m, S;
    const int32_t *in_ptr, *in_src, *out_ptr, *out_dst, *out_eid, *topo;
    const float *delays, *t_req, *at_src;
    int layout;              /* 0: [S][m]; 1: [m][S] */
    int early;               /* NEXT-2 hold mode */
    float *wns, *at_all, *rat_all;   /* at_all/rat_all: [n][S] or NULL */
    int32_t next;            /* next scenario (guarded by mu) */
    pthread_mutex_t mu;
} batch_job;

static void *batch_worker(void *arg) {
    batch_job *J = (batch_job *)arg;
    float *at = (float *)malloc(sizeof(float) * (size_t)(J->n > 0 ? J->n : 1));
    float *rat = (float *)malloc(sizeof(float) * (size_t)(J->n > 0 ? J->n : 1));
    for (;;) {
        pthread_mutex_lock(&J->mu);
        int32_t s = J->next++;
        pthread_mutex_unlock(&J->mu);
        if (s >= J->S) break;
        const float *d = J->layout == 0 ? J->delays + (int64_t)s * J->m : J->delays + s;
        int64_t stride = J->layout == 0 ? 1 : J->S;
        forward_pass(J->n, J->in_ptr, J->in_src, d, stride, J->at_src, J->topo, at, J->early);
        J->wns[s] = backward_pass(J->n, J->out_ptr, J->out_dst, J->out_eid, d, stride,
                                  J->t_req[s], J->topo, at, rat, NULL, J->early);
        if (J->at_all)
            for (int32_t v = 0; v < J->n; ++v) J->at_all[(int64_t)v * J->S + s] = at[v];
        if (J->rat_all)
            for (int32_t v = 0; v < J->n; ++v) J->rat_all[(int64_t)v * J->S + s] = rat[v];
    }
    free(at); free(rat);
    return NULL;
}

/* S scenarios over one graph: wns[S] (+ optional at_all/rat_all [n][S]).
 * threads > 1 only splits scenarios across pthreads (timing); results do not
 * depend on it. */
int oracle_batch_mode(int32_t n, int32_t m, const int32_t *in_ptr, const int32_t *in_src,
                      int32_t S, const float *delays, int layout, const float *t_req,
                      const float *at_src, float *wns, float *at_all, float *rat_all, int threads,
                      int early) {
    int rc = oracle_check_csr(n, m, in_ptr, in_src);
    if (rc) return rc;
    if (!all_finite(delays, (int64_t)m * S) || !all_finite(t_req, S)) return OR_INVALID;
    if (at_src && !all_finite(at_src, n)) return OR_INVALID;
    int32_t *topo = (int32_t *)malloc(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
    int32_t *level = (int32_t *)malloc(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
    int32_t *lptr = (int32_t *)malloc(sizeof(int32_t) * (size_t)(n + 1));
    int32_t *order = (int32_t *)malloc(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
    int32_t nt = 0, L = 0, unready = 0;
    rc = oracle_levelize(n, m, in_ptr, in_src, topo, &nt, level, lptr, order, &L, &unready);
    if (rc) { free(topo); free(level); free(lptr); free(order); return rc; }
    int32_t *out_ptr = (int32_t *)malloc(sizeof(int32_t) * (size_t)(n + 1));
    int32_t *out_dst = (int32_t *)malloc(sizeof(int32_t) * (size_t)(m > 0 ? m : 1));
    int32_t *out_eid = (int32_t *)malloc(sizeof(int32_t) * (size_t)(m > 0 ? m : 1));
    oracle_fanout(n, m, in_ptr, in_src, out_ptr, out_dst, out_eid);
    batch_job J;
    J.n = n; J.m = m; J.S = S; J.in_ptr = in_ptr; J.in_src = in_src;
    J.out_ptr = out_ptr; J.out_dst = out_dst; J.out_eid = out_eid; J.topo = topo;
    J.delays = delays; J.t_req = t_req; J.at_src = at_src; J.layout = layout;
    J.wns = wns; J.at_all = at_all; J.rat_all = rat_all; J.next = 0; J.early = early;
    pthread_mutex_init(&J.mu, NULL);
    if (threads < 1) threads = 1;
    if (threads > S) threads = S > 0 ? S : 1;
    pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * (size_t)threads);
    for (int t = 1; t < threads; ++t) pthread_create(&th[t], NULL, batch_worker, &J);
    batch_worker(&J);
    for (int t = 1; t < threads; ++t) pthread_join(th[t], NULL);
    pthread_mutex_destroy(&J.mu);
    free(th); free(topo); free(level); free(lptr); free(order);
    free(out_ptr); free(out_dst); free(out_eid);
    return OR_OK;
}
int oracle_batch(int32_t n, int32_t m, const int32_t *in_ptr, const int32_t *in_src,
                 int32_t S, const float *delays, int layout, const float *t_req,
                 const float *at_src, float *wns, float *at_all, float *rat_all, int threads) {
    return oracle_batch_mode(n, m, in_ptr, in_src, S, delays, layout, t_req, at_src, wns, at_all,
                             rat_all, threads, 0);
}

/* ---- NEXT-1: critical-path trace-back -------------------
 * PAPER.md:1002-1003 ("extract graph information (critical paths, ...)") names the
 * step; reading R17 fixes it:
 *   endpoint = the sink (out-degree 0) with the smallest slack fl(T - at[sink]),
 *              ties by the smallest node id;
 *   from v = endpoint, step to src(e) for the fan-in edge e of v with
 *              fl(at[src e] + d[e]) == at[v] (an edge that attains the max),
 *              ties by the smallest fan-in edge id, until a source (in-degree 0).
 * path[0] = endpoint ... path[len-1] = the source.  d is read with stride dstride
 * (1 for one delay set, S for the scenario-minor batch layout).  Returns
 * OR_INVALID if at is not a forward result of these delays (no attaining edge) or
 * the path is longer than max_len; n == 0 gives len = 0. */
int oracle_critical_path(int32_t n, int32_t m, const int32_t *in_ptr, const int32_t *in_src,
                         const float *d, int64_t dstride, const float *at, float T,
                         int32_t *path, int32_t max_len, int32_t *len) {
    *len = 0;
    if (n == 0) return OR_OK;
    int32_t *outdeg = (int32_t *)calloc((size_t)n, sizeof(int32_t));
    for (int32_t e = 0; e < m; ++e) outdeg[in_src[e]] += 1;
    T = canon(T);
    int32_t v = -1;
    float worst = 0.0f;
    for (int32_t u = 0; u < n; ++u) {
        if (outdeg[u] != 0) continue;
        float s = T - at[u];
        if (v < 0 || s < worst) { v = u; worst = s; }   /* ascending u: ties keep the smallest */
    }
    free(outdeg);
    if (v < 0) return OR_INVALID;   /* a DAG with n > 0 always has a sink */
    for (;;) {
        if (*len >= max_len) return OR_INVALID;
        path[(*len)++] = v;
        if (in_ptr[v + 1] == in_ptr[v]) return OR_OK;   /* source */
        int32_t best = -1;
        for (int32_t e = in_ptr[v]; e < in_ptr[v + 1] && best < 0; ++e) {
            float x = at[in_src[e]] + canon(d[(int64_t)e * dstride]);
            if (x == at[v]) best = e;
        }
        if (best < 0) return OR_INVALID;
        v = in_src[best];
    }
}

/* Top-K endpoints (SURVEY.md §8(f) NEXT-1 "with optional top-k endpoints"; reading
 * R17): the K sinks with the smallest (slack fl(T - at), node id), in that order,
 * and for each the same argmax trace-back as oracle_critical_path.  endpoints[K]
 * (-1 past the number of sinks), paths[K][max_len], lens[K] (0 past the number of
 * sinks). */
typedef struct {
    float slack;
    int32_t v;
} sink_key;
static int cmp_sink_key(const void *a, const void *b) {
    const sink_key *x = (const sink_key *)a, *y = (const sink_key *)b;
    if (x->slack < y->slack) return -1;
    if (x->slack > y->slack) return 1;
    return (x->v > y->v) - (x->v < y->v);
}
int oracle_critical_path_k(int32_t n, int32_t m, const int32_t *in_ptr, const int32_t *in_src,
                           const float *d, int64_t dstride, const float *at, float T, int32_t K,
                           int32_t *endpoints, int32_t *paths, int32_t max_len, int32_t *lens) {
    for (int32_t r = 0; r < K; ++r) {
        endpoints[r] = -1;
        lens[r] = 0;
    }
    if (n == 0) return OR_OK;
    int32_t *outdeg = (int32_t *)calloc((size_t)n, sizeof(int32_t));
    sink_key *keys = (sink_key *)malloc(sizeof(sink_key) * (size_t)n);
    for (int32_t e = 0; e < m; ++e) outdeg[in_src[e]] += 1;
    T = canon(T);
    int32_t ns = 0;
    for (int32_t u = 0; u < n; ++u)
        if (outdeg[u] == 0) {
            keys[ns].slack = T - at[u];
            keys[ns].v = u;
            ++ns;
        }
    free(outdeg);
    qsort(keys, (size_t)ns, sizeof(sink_key), cmp_sink_key);
    int rc = OR_OK;
    for (int32_t r = 0; r < K && r < ns && rc == OR_OK; ++r) {
        int32_t v = keys[r].v, len = 0;
        int32_t *path = paths + (int64_t)r * max_len;
        endpoints[r] = v;
        for (;;) {
            if (len >= max_len) { rc = OR_INVALID; break; }
            path[len++] = v;
            if (in_ptr[v + 1] == in_ptr[v]) break;   /* source */
            int32_t best = -1;
            for (int32_t e = in_ptr[v]; e < in_ptr[v + 1] && best < 0; ++e) {
                float x = at[in_src[e]] + canon(d[(int64_t)e * dstride]);
                if (x == at[v]) best = e;
            }
            if (best < 0) { rc = OR_INVALID; break; }
            v = in_src[best];
        }
        lens[r] = len;
    }
    free(keys);
    return rc;
}

/* S scenarios x top-K: endpoints [S][K], paths [S][K][max_len], lens [S][K]. */
int oracle_critical_paths_k(int32_t n, int32_t m, const int32_t *in_ptr, const int32_t *in_src,
                            int32_t S, const float *delays, const float *at_all,
                            const float *t_req, int32_t K, int32_t *endpoints, int32_t *paths,
                            int32_t max_len, int32_t *lens) {
    float *at = (float *)malloc(sizeof(float) * (size_t)(n > 0 ? n : 1));
    int rc = OR_OK;
    for (int32_t s = 0; s < S && rc == OR_OK; ++s) {
        for (int32_t v = 0; v < n; ++v) at[v] = at_all[(int64_t)v * S + s];
        rc = oracle_critical_path_k(n, m, in_ptr, in_src, delays + s, S, at, t_req[s], K,
                                    endpoints + (int64_t)s * K,
                                    paths + (int64_t)s * K * max_len, max_len,
                                    lens + (int64_t)s * K);
    }
    free(at);
    return rc;
}

/* S scenarios: delays [m][S] (scenario-minor), at_all [n][S], t_req[S];
 * paths [S][max_len], lens[S]. */
int oracle_critical_paths(int32_t n, int32_t m, const int32_t *in_ptr, const int32_t *in_src,
                          int32_t S, const float *delays, const float *at_all, const float *t_req,
                          int32_t *paths, int32_t max_len, int32_t *lens) {
    float *at = (float *)malloc(sizeof(float) * (size_t)(n > 0 ? n : 1));
    int rc = OR_OK;
    for (int32_t s = 0; s < S && rc == OR_OK; ++s) {
        for (int32_t v = 0; v < n; ++v) at[v] = at_all[(int64_t)v * S + s];
        rc = oracle_critical_path(n, m, in_ptr, in_src, delays + s, S, at, t_req[s],
                                  paths + (int64_t)s * max_len, max_len, lens + s);
    }
    free(at);
    return rc;
}

/* ---- NEXT-4: greedy maximal independent set -------------
 * the detailed-placement workload extracts "a maximal
 * independent set ... using Blelloch's Algorithm" (blelloch2012greedy), whose
 * result is the lexicographically-first MIS for a priority order.
 * reading R19: the graph is the undirected graph of the DAG's edges; vertices are
 * visited by increasing key (prio[v], v); v joins the set iff none of its
 * neighbours visited earlier joined.  in_set[v] = 1 / 0.  Sequential definition,
 * O(n log n + m). */
static const int32_t *g_prio;
static int cmp_prio(const void *a, const void *b) {
    int32_t x = *(const int32_t *)a, y = *(const int32_t *)b;
    if (g_prio[x] != g_prio[y]) return g_prio[x] < g_prio[y] ? -1 : 1;
    return (x > y) - (x < y);
}
int oracle_mis(int32_t n, int32_t m, const int32_t *in_ptr, const int32_t *in_src,
               const int32_t *prio, uint8_t *in_set) {
    int rc = oracle_check_csr(n, m, in_ptr, in_src);
    if (rc) return rc;
    int32_t *out_ptr = (int32_t *)malloc(sizeof(int32_t) * (size_t)(n + 1));
    int32_t *out_dst = (int32_t *)malloc(sizeof(int32_t) * (size_t)(m > 0 ? m : 1));
    int32_t *out_eid = (int32_t *)malloc(sizeof(int32_t) * (size_t)(m > 0 ? m : 1));
    oracle_fanout(n, m, in_ptr, in_src, out_ptr, out_dst, out_eid);
    int32_t *vis = (int32_t *)malloc(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
    for (int32_t v = 0; v < n; ++v) vis[v] = v;
    g_prio = prio;
    qsort(vis, (size_t)n, sizeof(int32_t), cmp_prio);
    for (int32_t v = 0; v < n; ++v) in_set[v] = 0;
    for (int32_t i = 0; i < n; ++i) {
        int32_t v = vis[i];
        int blocked = 0;
        for (int32_t e = in_ptr[v]; e < in_ptr[v + 1] && !blocked; ++e) blocked = in_set[in_src[e]];
        for (int32_t k = out_ptr[v]; k < out_ptr[v + 1] && !blocked; ++k) blocked = in_set[out_dst[k]];
        in_set[v] = (uint8_t)!blocked;   /* later neighbours are still 0 here */
    }
    free(vis); free(out_ptr); free(out_dst); free(out_eid);
    return OR_OK;
}
