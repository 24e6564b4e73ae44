// propagate.cu -- forward max-plus and backward min-plus (+ fused slack / worst
// slack) over the levelized DAG, for one delay set or S scenario sets.
// SURVEY.md §8(a) a5-a7; BASELINE.json:5 ("at[v] = max over fan-in of at[u] +
// d(u,v)", "min-plus required time").
//
// Data layout in HBM (scenario-minor): at[v*S + s], rat[v*S + s],
// delays[e*S + s].  Pull-based, no float atomics: every output is one fp32
// max/min over fl(x +/- d) terms, which is order-independent (0 ULP against
// the oracle, reading R10).
//
// Dataflow design.  One persistent cooperative launch per pass.
//   * The pass is a list of WARP TASKS in pass order (levels ascending forward,
//     descending backward; inside a level descriptor-major, scenario chunk of SC
//     columns minor; with one chunk, k_flow<..., ONE> maps task t to descriptor t).  A
//     normal task is a run of consecutive level-ordered rows (weight = edges +
//     rows <= tw + split); a row with more than `split` edges is cut into PART
//     tasks whose partial max/min go to part_buf.  Task t belongs to warp
//     t mod W; warps are all co-resident, walk their tasks in order, and a task
//     only depends on tasks of earlier levels, so the earliest unfinished task
//     can always proceed (no deadlock).
//   * READINESS IS THE DATA.  Before a pass the output rows (and part_buf) are
//     filled with a NaN sentinel.  Finite inputs never produce NaN at/rat values
//     (only +-inf on overflow), so a gathered value that is not NaN is the final
//     value: each 32-bit element is written exactly once and read with strong
//     (relaxed, gpu-scope) loads, so there is no flag, fence or barrier on the
//     dependency path -- a consumer re-polls only the elements still NaN.
//   * A warp stages the task's delay rows (and, backward, the at rows for the
//     slack) into its shared-memory scratch with cp.async while its gathers are
//     in flight; the task's index data (rows, neighbours, edge ids) were loaded
//     into registers during the previous task.
//   * Rows are reduced from shared memory by lane groups (LPN lanes x V floats
//     per SC-column chunk); backward fuses slack = rat - at and keeps per-lane
//     minima, folded per CTA into the worst slack (ordered-int atomicMin).
//   * Rows cut into parts are read by their consumers as the combine of their
//     partials (each sentinel-checked, PW in flight, waited on as a group in the
//     single-chunk kernels; the neighbour id is encoded as -(first part id + 1),
//     levelize.cu); their own rows are written after the pass by k_finalize_split.
//   * At S = 64 the passes are bound more by their instruction stream than by the
//     dependency chain (fake-gather diagnostic, ncu issue-active),
//     so the hot loops are written for instruction count: the poll rounds keep a
//     per-lane bitmask of missing slots (forward, single-chunk backward).
#include <algorithm>
#include <map>
#include <mutex>
#include <tuple>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "common.cuh"

namespace hf {

namespace {

constexpr int NWARP = 4;              // warps per CTA
#ifndef PW_BWD
#define PW_BWD 4                      // backward: partials of a long neighbour in flight
#endif
constexpr int FLOW_THREADS = NWARP * 32;
constexpr unsigned FULL = 0xffffffffu;

template <int V> struct Vec {
    float x[V];
};

template <int V> __device__ __forceinline__ Vec<V> ld_relaxed(const float *p) {
    Vec<V> r;
    if constexpr (V == 4) {
        asm volatile("ld.relaxed.gpu.global.v4.f32 {%0,%1,%2,%3}, [%4];"
                     : "=f"(r.x[0]), "=f"(r.x[1]), "=f"(r.x[2]), "=f"(r.x[3])
                     : "l"(p)
                     : "memory");
    } else if constexpr (V == 2) {
        asm volatile("ld.relaxed.gpu.global.v2.f32 {%0,%1}, [%2];"
                     : "=f"(r.x[0]), "=f"(r.x[1])
                     : "l"(p)
                     : "memory");
    } else {
        asm volatile("ld.relaxed.gpu.global.f32 %0, [%1];" : "=f"(r.x[0]) : "l"(p) : "memory");
    }
    return r;
}
template <int V> __device__ __forceinline__ void st_relaxed(float *p, const Vec<V> &v) {
    if constexpr (V == 4) {
        asm volatile("st.relaxed.gpu.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x[0]),
                     "f"(v.x[1]), "f"(v.x[2]), "f"(v.x[3])
                     : "memory");
    } else if constexpr (V == 2) {
        asm volatile("st.relaxed.gpu.global.v2.f32 [%0], {%1,%2};" ::"l"(p), "f"(v.x[0]), "f"(v.x[1])
                     : "memory");
    } else {
        asm volatile("st.relaxed.gpu.global.f32 [%0], %1;" ::"l"(p), "f"(v.x[0]) : "memory");
    }
}
template <int V> __device__ __forceinline__ Vec<V> nan_vec() {
    Vec<V> r;
#pragma unroll
    for (int j = 0; j < V; ++j) r.x[j] = __int_as_float(-1);   // the all-ones NaN sentinel
    return r;
}
template <int V> __device__ __forceinline__ void st_plain(float *p, const Vec<V> &v) {
    if constexpr (V == 4) {
        *reinterpret_cast<float4 *>(p) = make_float4(v.x[0], v.x[1], v.x[2], v.x[3]);
    } else if constexpr (V == 2) {
        *reinterpret_cast<float2 *>(p) = make_float2(v.x[0], v.x[1]);
    } else {
        *p = v.x[0];
    }
}
template <int V> __device__ __forceinline__ Vec<V> ld_s(const float *p) {
    Vec<V> r;
    if constexpr (V == 4) {
        const float4 t = *reinterpret_cast<const float4 *>(p);
        r.x[0] = t.x; r.x[1] = t.y; r.x[2] = t.z; r.x[3] = t.w;
    } else if constexpr (V == 2) {
        const float2 t = *reinterpret_cast<const float2 *>(p);
        r.x[0] = t.x; r.x[1] = t.y;
    } else {
        r.x[0] = *p;
    }
    return r;
}
template <int V> __device__ __forceinline__ void st_s(float *p, const Vec<V> &v) { st_plain<V>(p, v); }

template <int V> __device__ __forceinline__ bool has_nan(const Vec<V> &v) {
    bool b = false;
#pragma unroll
    for (int j = 0; j < V; ++j) b |= (v.x[j] != v.x[j]);
    return b;
}

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
// V floats global -> shared, asynchronous (LDGSTS); 16-byte copies bypass L1
template <int V> __device__ __forceinline__ void cp_async_v(float *dst, const float *src) {
    if constexpr (V == 4) {
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src)
                     : "memory");
    } else if constexpr (V == 2) {
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src)
                     : "memory");
    } else {
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst)), "l"(src)
                     : "memory");
    }
}
// delay rows are read once per pass: staged with an L2 evict-first policy so they do
// not push the recently written at / rat rows (the gathers' working set) out of L2
// (variant build -DHF_DELAY_EVICT_FIRST, A/B through HF_LIB)
template <int V> __device__ __forceinline__ void cp_async_v_ef(float *dst, const float *src,
                                                               unsigned long long pol) {
    if constexpr (V == 4) {
        asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)),
                     "l"(src), "l"(pol)
                     : "memory");
    } else if constexpr (V == 2) {
        asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], 8, %2;" ::"r"(smem_u32(dst)),
                     "l"(src), "l"(pol)
                     : "memory");
    } else {
        asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], 4, %2;" ::"r"(smem_u32(dst)),
                     "l"(src), "l"(pol)
                     : "memory");
    }
}
__device__ __forceinline__ unsigned long long policy_evict_first() {
    unsigned long long pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }
// all but the most recent group (HF_IDX_SMEM: the next task's index copies stay in
// flight); without HF_IDX_SMEM every group
__device__ __forceinline__ void cp_async_wait_keep1() {
#if HF_IDX_SMEM
    asm volatile("cp.async.wait_group 1;" ::: "memory");
#else
    asm volatile("cp.async.wait_group 0;" ::: "memory");
#endif
}

template <bool FWD> __device__ __forceinline__ float combine(float best, float x) {
    return FWD ? fmaxf(best, x) : fminf(best, x);
}
template <bool FWD> __device__ __forceinline__ float relax(float a, float d) {
    return FWD ? __fadd_rn(a, d) : __fsub_rn(a, d);
}
template <bool FWD> __device__ __forceinline__ float ident() {
    return __int_as_float(FWD ? 0xff800000 : 0x7f800000);   // -inf for max, +inf for min
}

__device__ __forceinline__ int atom_add_acq_rel_i(int *p, int v) {
    int old;
    asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
}
template <int V> __device__ __forceinline__ Vec<V> ld_ord_relaxed(const int32_t *p) {
    Vec<V> r;
    if constexpr (V == 4) {
        int a, b, c, d;
        asm volatile("ld.relaxed.gpu.global.v4.s32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(a), "=r"(b), "=r"(c), "=r"(d)
                     : "l"(p)
                     : "memory");
        r.x[0] = ord2f(a); r.x[1] = ord2f(b); r.x[2] = ord2f(c); r.x[3] = ord2f(d);
    } else if constexpr (V == 2) {
        int a, b;
        asm volatile("ld.relaxed.gpu.global.v2.s32 {%0,%1}, [%2];" : "=r"(a), "=r"(b) : "l"(p) : "memory");
        r.x[0] = ord2f(a); r.x[1] = ord2f(b);
    } else {
        int a;
        asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(a) : "l"(p) : "memory");
        r.x[0] = ord2f(a);
    }
    return r;
}

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

struct FlowParams {
    // level-ordered CSR of this direction: row i <-> node node_of[i]
    const int32_t *row_ptr;   // [n+1]
    const int32_t *nbr;       // [m] neighbour node id, long rows as -(first part id + 1)
    const int32_t *eid;       // [m] edge id (delay row)
    const int32_t *node_of;   // [n]
    const int4 *desc;         // task descriptors (TaskSched)
    const int32_t *nt;        // [L] tasks per chunk of pass-level q
    const int32_t *doff;      // [L+1]
    const int32_t *tb;        // [L+1] first global task of pass-level q
    int32_t L, S, nch;
    int32_t nch_shift;        // log2(nch) for a power of two, else -1
    int32_t ecap, ncap;       // per-warp scratch capacity (edges, rows)
    const int32_t *part_np;   // [parts] by first part id
    float *part_buf;          // [parts][S]   (HF_LASTPART = 0)
    int32_t *part_acc;        // [parts][S] ordered ints, by first part id (HF_LASTPART)
    int32_t *part_cnt;        // [parts][nch] finished parts per scenario chunk, by first part id
    const float *d;           // [m][S] by edge id
    const float *src_val;     // forward: at_src [n] (or null); backward: t_req [S] (or null)
    float t_scalar;           // backward: T when t_req is null
    const float *other;       // backward: at (for slack)
    float *out;               // forward: at; backward: rat
    float *prefill;           // forward, optional: the backward output (rat), NaN-filled
                              // row by row as the forward writes its own rows
    float *slack;             // backward, optional [n][S]
    int32_t *wns_ord;         // backward: [S] ordered-int minima
    uint32_t *err;
    int32_t sleep_max;        // ns, cap of the poll back-off
    int32_t watchdog_spins;   // poll rounds after which one wait gives up (ERR_WATCHDOG)
    int32_t poll_all;         // backward: 1 every lane re-polls its missing vectors; 0 one lane polls
    unsigned long long *trace;   // optional: per task {t, level, t_start, t_ready, t_done}
    int32_t trace_cap;
};

// per-warp shared-memory scratch (bytes), identical on host and device
#ifndef HF_IDX_SMEM
#define HF_IDX_SMEM 0
#endif
// HF_LASTPART (default): the part tasks of a long row fold their partial max / min into
// one ordered-int accumulator row (red.max / red.min) and count themselves on an
// acq_rel counter; the last one writes the row's final value (and, backward, its
// slack), so a long row is read by its consumers like any other row (plain neighbour
// ids) and no finalisation kernel runs after the pass.  0: partial rows in part_buf,
// every consumer combines them (PW at a time), k_finalize_split after the pass.
#ifndef HF_LASTPART
#define HF_LASTPART 0
#endif
struct WarpLayout {
    int d, a, at, nbr, eid, rp, node, ring, bytes;
    int ibytes;   // bytes of one index buffer (nbr, eid, rp, node); HF_IDX_SMEM keeps two
};
__host__ __device__ inline WarpLayout warp_layout(int ecap, int ncap, int SC, bool fwd, bool ga) {
    WarpLayout L;
    int o = 0;
    L.d = o;    o += ecap * SC * 4;
    L.a = o;    o += ga ? ecap * SC * 4 : 0;
    L.at = o;   o += fwd ? 0 : ncap * SC * 4;
    const int i0 = o;
    L.nbr = o;  o += ecap * 4;
    L.eid = o;  o += ecap * 4;
    L.rp = o;   o += (ncap + 1) * 4;
    L.node = o; o += ncap * 4;
    L.ibytes = o - i0;
    // HF_IDX_SMEM: a second index buffer (the next task's, filled by cp.async) and a
    // ring of three task descriptors {dsc, chunk}
    o += HF_IDX_SMEM ? L.ibytes : 0;
    o = (o + 15) & ~15;
    L.ring = o; o += HF_IDX_SMEM ? 3 * 32 : 0;
    L.bytes = (o + 15) & ~15;
    return L;
}
__host__ __device__ inline int wmin_bytes(int S) { return (S * 4 + 15) & ~15; }

// one task's index data, loaded into registers one task ahead (NSL slots per lane:
// a task has <= 32*NSL edges and <= 32*NSL - 1 rows)
template <int NSL> struct Idx {
    int4 dsc;
    int c;
    int nbr0, eid0, rp0, node0;   // slot 0: edge / row `lane`
    int nbr1, eid1, rp1, node1;   // slot 1: edge / row `lane + 32` (NSL == 2)
};
template <int LPN> constexpr int idx_slots() { return LPN <= 2 ? 2 : 1; }

// Launch bounds: the thread bound only.  An explicit minimum of 1 block lets ptxas
// spend 140-152 registers (3 CTAs per SM, +5% forward / +7% backward, measured);
// the backward experiment with 6 blocks is -DFLOW_MINB_BWD=6.
#ifndef FLOW_MINB_FWD
#define FLOW_MINB_FWD 0
#endif
#ifndef FLOW_MINB_BWD
#define FLOW_MINB_BWD 0
#endif
template <int V, bool FWD, bool ONE> constexpr int flow_minb() {
    return FWD ? FLOW_MINB_FWD : FLOW_MINB_BWD;
}
// ONE: the pass has one scenario chunk (S = SC): task t is descriptor t
template <int V, int LPN, bool FWD, bool GA, bool EARLY, bool ONE>
__global__ void __launch_bounds__(FLOW_THREADS, flow_minb<V, FWD, ONE>()) k_flow(FlowParams p) {
    // MX: the pass combines with max (late forward, early backward), else min
    constexpr bool MX = FWD != EARLY;
    constexpr int SC = V * LPN;   // columns per chunk
    constexpr int G = 32 / LPN;   // lane groups per warp
    constexpr int NSL = idx_slots<LPN>();
    // GA: gathers land in shared memory by cp.async (16-byte pieces, V == 4);
    // else in registers, RB per lane per batch
#ifndef RB4_FWD
#define RB4_FWD 4
#endif
#ifndef RB4_BWD
#define RB4_BWD 4
#endif
    constexpr int RB = V == 4 ? (FWD ? RB4_FWD : RB4_BWD) : 8;
    extern __shared__ __align__(16) unsigned char smem[];
    const int wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane / LPN, gl = lane % LPN;
    const int S = p.S;
    const WarpLayout WL = warp_layout(p.ecap, p.ncap, SC, FWD, GA);
    int32_t *s_wmin = reinterpret_cast<int32_t *>(smem);
    unsigned char *wb = smem + wmin_bytes(S) + wib * WL.bytes;
    float *s_d = reinterpret_cast<float *>(wb + WL.d);
    float *s_a = reinterpret_cast<float *>(wb + WL.a);
    float *s_at = reinterpret_cast<float *>(wb + WL.at);
#if HF_IDX_SMEM
    int32_t *s_nbr0 = reinterpret_cast<int32_t *>(wb + WL.nbr);
    int32_t *s_eid0 = reinterpret_cast<int32_t *>(wb + WL.eid);
    int32_t *s_rp0 = reinterpret_cast<int32_t *>(wb + WL.rp);
    int32_t *s_node0 = reinterpret_cast<int32_t *>(wb + WL.node);
    int32_t *s_nbr = s_nbr0, *s_eid = s_eid0, *s_rp = s_rp0, *s_node = s_node0;
#else
    int32_t *s_nbr = reinterpret_cast<int32_t *>(wb + WL.nbr);
    int32_t *s_eid = reinterpret_cast<int32_t *>(wb + WL.eid);
    int32_t *s_rp = reinterpret_cast<int32_t *>(wb + WL.rp);
    int32_t *s_node = reinterpret_cast<int32_t *>(wb + WL.node);
#endif

    // Rejected input already flagged (by the forward pass of this batch, or by the
    // pre-check of the concurrent batch): the results are void and the call reports
    // HF_ERR_INVALID_ARG, so the backward pass does nothing -- which is what lets it
    // use the delays unchecked (the forward pass checked the same delays; the graph's
    // own delays were checked by hf_graph_create).
    if (!FWD && (*reinterpret_cast<volatile uint32_t *>(p.err) & ERR_NONFINITE)) return;
    if (!FWD) {
        for (int s = threadIdx.x; s < S; s += blockDim.x) s_wmin[s] = 0x7f800000;
        __syncthreads();
    }
    const int W = gridDim.x * NWARP;
    const int w = wib * gridDim.x + blockIdx.x;   // consecutive tasks on different SMs
    const int T = __ldg(p.tb + p.L);
    const int L = p.L;

    // ---- task locator: pass-level q with tb[q] <= t < tb[q+1] (t increases) ----
    auto locate = [&](int t, int &q, int &c, int4 &dsc) {
        if constexpr (ONE) {
            // one scenario chunk: task bases are the descriptor offsets, task t is
            // descriptor t (no level search, no division)
            c = 0;
            dsc = __ldg(p.desc + t);
            return;
        }
        if (__ldg(p.tb + q + 1) <= t) {
            int lo = q + 1, step = 1;
            while (lo + step < L && __ldg(p.tb + lo + step) <= t) {
                lo += step;
                step <<= 1;
            }
            int hi = min(lo + step, L);
            while (hi - lo > 1) {
                const int mid = (lo + hi) >> 1;
                if (__ldg(p.tb + mid) <= t) lo = mid;
                else hi = mid;
            }
            q = lo;
        }
        // inside a pass-level the tasks are descriptor-major, chunk-minor
        // (t = tb[q] + j * nch + c): with a power-of-two chunk count a shift and a mask,
        // and a warp keeps one chunk when W is a multiple of nch
        const int rel = t - __ldg(p.tb + q);
        int j;
        if (p.nch_shift >= 0) {
            j = rel >> p.nch_shift;
            c = rel & (p.nch - 1);
        } else {
            j = rel / p.nch;
            c = rel - j * p.nch;
        }
        dsc = __ldg(p.desc + __ldg(p.doff + q) + j);
    };
    // index loads of one task (no use of the results here: they land during the
    // current task)
    auto load_idx = [&](const int4 &dsc, Idx<NSL> &x) {
        const bool part = dsc.y < 0;
        const int E = dsc.w - dsc.z;
        const int NR = part ? 1 : dsc.y - dsc.x;
        const int k0 = lane, k1 = lane + 32;
        x.nbr0 = k0 < E ? __ldg(p.nbr + dsc.z + k0) : 0;
        x.eid0 = k0 < E ? __ldg(p.eid + dsc.z + k0) : 0;
        x.rp0 = ((HF_LASTPART || !part) && k0 <= NR) ? __ldg(p.row_ptr + dsc.x + k0) : 0;
        x.node0 = k0 < NR ? __ldg(p.node_of + dsc.x + k0) : 0;
        if (NSL == 2) {
            x.nbr1 = k1 < E ? __ldg(p.nbr + dsc.z + k1) : 0;
            x.eid1 = k1 < E ? __ldg(p.eid + dsc.z + k1) : 0;
            x.rp1 = ((HF_LASTPART || !part) && k1 <= NR) ? __ldg(p.row_ptr + dsc.x + k1) : 0;
            x.node1 = k1 < NR ? __ldg(p.node_of + dsc.x + k1) : 0;
        }
    };

    bool bad = false;
    Vec<V> run;   // backward: running min of slack for column chunk run_c
    int run_c = -1;
#pragma unroll
    for (int j = 0; j < V; ++j) run.x[j] = ident<false>();
    auto flush_run = [&]() {
        if (!FWD && run_c >= 0) {
#pragma unroll
            for (int j = 0; j < V; ++j)
                if (run.x[j] != ident<false>())
                    atomicMin(s_wmin + run_c * SC + gl * V + j, f2ord(run.x[j]));
#pragma unroll
            for (int j = 0; j < V; ++j) run.x[j] = ident<false>();
        }
    };

    int qa = 0, qb = 0;          // locator cursors of the two look-ahead streams
    int t0 = w;
#if HF_IDX_SMEM
    // software pipeline in shared memory (no look-ahead registers): the index data of
    // the next task is copied by cp.async into the other index buffer while this task
    // runs; the descriptors of this, the next and the one after live in a 3-slot ring
    int4 *s_ring = reinterpret_cast<int4 *>(wb + WL.ring);   // [3] {dsc}, [3] {c} below
    int *s_ringc = reinterpret_cast<int *>(s_ring + 3);
    // index copies of one task into buffer b (4-byte cp.async, lanes over the arrays)
    auto copy_idx = [&](const int4 &dsc, int b) {
        const bool part = dsc.y < 0;
        const int E = dsc.w - dsc.z;
        const int NR = part ? 1 : dsc.y - dsc.x;
        int32_t *bn = reinterpret_cast<int32_t *>(reinterpret_cast<unsigned char *>(s_nbr) + b * WL.ibytes);
        int32_t *be = reinterpret_cast<int32_t *>(reinterpret_cast<unsigned char *>(s_eid) + b * WL.ibytes);
        int32_t *br = reinterpret_cast<int32_t *>(reinterpret_cast<unsigned char *>(s_rp) + b * WL.ibytes);
        int32_t *bo = reinterpret_cast<int32_t *>(reinterpret_cast<unsigned char *>(s_node) + b * WL.ibytes);
        for (int k = lane; k < E; k += 32) {
            cp_async_v<1>(reinterpret_cast<float *>(bn + k), reinterpret_cast<const float *>(p.nbr + dsc.z + k));
            cp_async_v<1>(reinterpret_cast<float *>(be + k), reinterpret_cast<const float *>(p.eid + dsc.z + k));
        }
        if (HF_LASTPART || !part)
            for (int k = lane; k <= NR; k += 32)
                cp_async_v<1>(reinterpret_cast<float *>(br + k), reinterpret_cast<const float *>(p.row_ptr + dsc.x + k));
        for (int k = lane; k < NR; k += 32)
            cp_async_v<1>(reinterpret_cast<float *>(bo + k), reinterpret_cast<const float *>(p.node_of + dsc.x + k));
    };
    int it = 0, rs = 0;   // task iteration; ring slot of this task (it % 3)
    if (t0 < T) {
        int4 dd;
        int cc;
        locate(t0, qa, cc, dd);
        if (lane == 0) {
            s_ring[0] = dd;
            s_ringc[0] = cc;
        }
        copy_idx(dd, 0);
        cp_async_commit();
        qb = qa;
        if (t0 + W < T) {
            locate(t0 + W, qb, cc, dd);
            if (lane == 0) {
                s_ring[1] = dd;
                s_ringc[1] = cc;
            }
        }
    }
#else
    // software pipeline: D1 = descriptor of the next task, X0 = index registers of
    // the current task, X1 of the next
    Idx<NSL> X0, X1;
    int4 D1 = make_int4(0, 0, 0, 0);
    int c1 = 0;
    if (t0 < T) {
        locate(t0, qa, X0.c, X0.dsc);
        load_idx(X0.dsc, X0);
        qb = qa;
        if (t0 + W < T) locate(t0 + W, qb, c1, D1);
    }
#endif
    for (int t = t0; t < T; t += W) {
        const unsigned long long tr0 = p.trace ? gtimer() : 0;
#ifdef HF_TRACE_EXT
        // extended trace fields (poll rounds, all-batches-ready time) cost registers
        // even when tracing is off: a separate build (HF_NVCC_FLAGS=-DHF_TRACE_EXT)
        int npoll = 0;
#define HF_NPOLL_INC() (++npoll)
#else
#define HF_NPOLL_INC() ((void)0)
#endif
        // ---- (1) this task's index data -> shared scratch; stage delays (+ at) ----
#if HF_IDX_SMEM
        cp_async_wait();   // this task's index copies (issued during the previous task)
        __syncwarp();
        const int4 dsc = s_ring[rs];
        const int c = s_ringc[rs];
        const int bsel = it & 1;
        int32_t *s_nbr = reinterpret_cast<int32_t *>(reinterpret_cast<unsigned char *>(s_nbr0) + bsel * WL.ibytes);
        int32_t *s_eid = reinterpret_cast<int32_t *>(reinterpret_cast<unsigned char *>(s_eid0) + bsel * WL.ibytes);
        int32_t *s_rp = reinterpret_cast<int32_t *>(reinterpret_cast<unsigned char *>(s_rp0) + bsel * WL.ibytes);
        int32_t *s_node = reinterpret_cast<int32_t *>(reinterpret_cast<unsigned char *>(s_node0) + bsel * WL.ibytes);
        const int rp_base = dsc.z;   // s_rp holds absolute row offsets here
#else
        const int4 dsc = X0.dsc;
        const int c = X0.c;
        const int rp_base = 0;
#endif
        const bool part = dsc.y < 0;
        const int E = dsc.w - dsc.z;
        const int NR = part ? 1 : dsc.y - dsc.x;
        const int col = c * SC + gl * V;
#if !HF_IDX_SMEM
        if (lane < E) {
            s_nbr[lane] = X0.nbr0;
            s_eid[lane] = X0.eid0;
        }
        if ((HF_LASTPART || !part) && lane <= NR) s_rp[lane] = X0.rp0 - dsc.z;
        if (lane < NR) s_node[lane] = X0.node0;
        if (NSL == 2) {
            const int k = lane + 32;
            if (k < E) {
                s_nbr[k] = X0.nbr1;
                s_eid[k] = X0.eid1;
            }
            if ((HF_LASTPART || !part) && k <= NR) s_rp[k] = X0.rp1 - dsc.z;
            if (k < NR) s_node[k] = X0.node1;
        }
        __syncwarp();
#endif
        for (int k = g; k < E; k += G)
#ifdef HF_DELAY_EVICT_FIRST
            cp_async_v_ef<V>(s_d + k * SC + gl * V, p.d + int64_t(s_eid[k]) * S + col,
                             policy_evict_first());
#elif defined(HF_DBG_FAKE_DELAY)
            // diagnostic build only (wrong results): every task reads delay row k of a
            // tiny L2-resident set -- how much of a pass is the delay rows' latency?
            cp_async_v<V>(s_d + k * SC + gl * V, p.d + int64_t(s_eid[k] & 8191) * S + col);
#else
            cp_async_v<V>(s_d + k * SC + gl * V, p.d + int64_t(s_eid[k]) * S + col);
#endif
        if (!FWD && !part && p.other)
            for (int i = g; i < NR; i += G)
                cp_async_v<V>(s_at + i * SC + gl * V, p.other + int64_t(s_node[i]) * S + col);
        cp_async_commit();
        // ---- (2) look-ahead: index loads of the next task, descriptor of the one after
#if HF_IDX_SMEM
        {
            const int rn = rs == 2 ? 0 : rs + 1, rnn = rn == 2 ? 0 : rn + 1;
            if (t + W < T) copy_idx(s_ring[rn], bsel ^ 1);
            cp_async_commit();   // (an empty group without a next task: wait_group 1 below)
            if (t + 2 * W < T) {
                int4 dd;
                int cc;
                locate(t + 2 * W, qb, cc, dd);
                if (lane == 0) {
                    s_ring[rnn] = dd;
                    s_ringc[rnn] = cc;
                }
            }
        }
#else
        if (t + W < T) {
            X1.dsc = D1;
            X1.c = c1;
            load_idx(D1, X1);
            if (t + 2 * W < T) locate(t + 2 * W, qb, c1, D1);
        }
#endif
        // ---- (3) edge-parallel gathers: x = fl(a[u] +/- d), sentinel-polled ----
        unsigned long long tr1 = 0;
        if constexpr (GA) {
            // every gathered row piece lands in s_a by cp.async (all edges in flight at
            // once); pieces still holding the sentinel are re-fetched after a back-off
            for (int k = g; k < E; k += G) {
                const int u = s_nbr[k];
                if (u >= 0) cp_async_v<V>(s_a + k * SC + gl * V, p.out + int64_t(u) * S + col);
            }
            cp_async_commit();
            for (int k = g; !HF_LASTPART && k < E; k += G) {   // neighbours cut into parts (rare)
                const int u = s_nbr[k];
                if (u < 0) {
                    const int q0 = -u - 1;
                    const int np = __ldg(p.part_np + q0);
                    Vec<V> acc;
#pragma unroll
                    for (int j = 0; j < V; ++j) acc.x[j] = ident<MX>();
                    for (int kk = 0; kk < np; ++kk) {
                        const float *src = p.part_buf + int64_t(q0 + kk) * S + col;
                        Vec<V> v = ld_relaxed<V>(src);
                        int ns = 32;
                        while (has_nan<V>(v)) {
                            __nanosleep(ns);
                            ns = min(ns * 2, p.sleep_max);
                            v = ld_relaxed<V>(src);
                        }
#pragma unroll
                        for (int j = 0; j < V; ++j) acc.x[j] = combine<MX>(acc.x[j], v.x[j]);
                    }
                    st_s<V>(s_a + k * SC + gl * V, acc);
                }
            }
            cp_async_wait();
            int ns = 32;
            for (;;) {
                bool miss = false;
                for (int k = g; k < E; k += G)
                    if (s_nbr[k] >= 0) miss |= has_nan<V>(ld_s<V>(s_a + k * SC + gl * V));
                if (!__ballot_sync(FULL, miss)) break;
                __nanosleep(ns);
                ns = min(ns * 2, p.sleep_max);
                for (int k = g; k < E; k += G) {
                    const int u = s_nbr[k];
                    if (u >= 0 && has_nan<V>(ld_s<V>(s_a + k * SC + gl * V)))
                        cp_async_v<V>(s_a + k * SC + gl * V, p.out + int64_t(u) * S + col);
                }
                cp_async_commit();
                cp_async_wait();
            }
            if (p.trace) tr1 = gtimer();
            for (int k = g; k < E; k += G) {
                float *dp = s_d + k * SC + gl * V;
                const Vec<V> dv = ld_s<V>(dp);
                const Vec<V> av = ld_s<V>(s_a + k * SC + gl * V);
                Vec<V> x;
#pragma unroll
                for (int j = 0; j < V; ++j) {
                    x.x[j] = relax<FWD>(av.x[j], FWD ? sane(dv.x[j], bad) : dv.x[j]);
                }
                st_s<V>(dp, x);
            }
        }
        for (int k0 = 0; !GA && k0 < E; k0 += G * RB) {
            Vec<V> a[RB];
            int uu[RB];
#pragma unroll
            for (int r = 0; r < RB; ++r) {
                const int k = k0 + r * G + g;
                uu[r] = k < E ? s_nbr[k] : INT32_MAX;
                if (uu[r] >= 0 && uu[r] != INT32_MAX)
#ifdef HF_DBG_FAKE_GATHER
                    // diagnostic build only (wrong results): gathers read always-final
                    // rows (delay rows of a 16 MB L2-resident set): the pass without its
                    // dependency waits -- what the instruction stream alone costs
                    a[r] = ld_relaxed<V>(p.d + int64_t(uu[r] & 0xffff) * S + col);
#else
                    a[r] = ld_relaxed<V>(p.out + int64_t(uu[r]) * S + col);
#endif
            }
            // neighbours cut into parts: combine of their partials (rare; HF_LASTPART:
            // never -- a long row's last part writes it like any other row)
#pragma unroll
            for (int r = 0; r < RB; ++r) {
                if (!HF_LASTPART && uu[r] < 0) {
                    const int q0 = -uu[r] - 1;
                    const int np = __ldg(p.part_np + q0);
#pragma unroll
                    for (int j = 0; j < V; ++j) a[r].x[j] = ident<MX>();
                    // PW partials in flight per step (a long row has up to
                    // ceil(degree / LO_PE) of them; backward rows are the long ones,
                    // the wide forward kernel keeps one to stay within its register budget)
                    constexpr int PW = (FWD && V == 4) ? 1 : PW_BWD;
                    for (int k = 0; k < np; k += PW) {
                        const float *src = p.part_buf + int64_t(q0 + k) * S + col;
                        Vec<V> v[PW];
#pragma unroll
                        for (int t = 0; t < PW; ++t) {
                            if (k + t < np) {
                                v[t] = ld_relaxed<V>(src + int64_t(t) * S);
                            } else {
#pragma unroll
                                for (int j = 0; j < V; ++j) v[t].x[j] = ident<MX>();
                            }
                        }
                        if constexpr (PW == 1 || !ONE) {
                            // one partial after the other (the four-column forward, PW 1,
                            // and the multi-chunk kernels: the group form below cost them
                            // 6% / 3..4% in codegen -- 128 registers at several chunks)
#pragma unroll
                            for (int t = 0; t < PW; ++t) {
                                int ns = 32;
                                while (has_nan<V>(v[t])) {
                                    __nanosleep(ns);
                                    ns = min(ns * 2, p.sleep_max);
                                    v[t] = ld_relaxed<V>(src + int64_t(t) * S);
                                }
                            }
                        } else {
                            // wait for the PW partials together: every round re-loads all
                            // the missing ones (one round trip for the group; waiting on one
                            // partial after the other paid a round trip per late partial)
                            int ns = 32, spins = 0;
                            for (;;) {
                                bool miss = false;
#pragma unroll
                                for (int t = 0; t < PW; ++t) miss |= has_nan<V>(v[t]);
                                if (!miss) break;
                                if (++spins > p.watchdog_spins) {
                                    atomicOr(p.err, ERR_WATCHDOG);
#pragma unroll
                                    for (int t = 0; t < PW; ++t)
#pragma unroll
                                        for (int j = 0; j < V; ++j) v[t].x[j] = 0.0f;
                                    break;
                                }
                                __nanosleep(ns);
                                ns = min(ns * 2, p.sleep_max);
#pragma unroll
                                for (int t = 0; t < PW; ++t)
                                    if (has_nan<V>(v[t])) v[t] = ld_relaxed<V>(src + int64_t(t) * S);
                            }
                        }
#pragma unroll
                        for (int t = 0; t < PW; ++t)
#pragma unroll
                            for (int j = 0; j < V; ++j) a[r].x[j] = combine<MX>(a[r].x[j], v[t].x[j]);
                    }
                }
            }
            // wait until every gathered element is final (not the NaN sentinel): every
            // lane re-loads its own missing vectors once per round (one round trip per
            // round, back-off between rounds): the lane's missing slots as a bitmask
            // (~40 instructions a round instead of ~120: forward -5%, single-chunk
            // backward -1%), or the per-slot re-check (multi-chunk backward)
            unsigned mm = 0;
#pragma unroll
            for (int r = 0; r < RB; ++r)
                if (uu[r] >= 0 && uu[r] != INT32_MAX && has_nan<V>(a[r])) mm |= 1u << r;
            unsigned bal = __ballot_sync(FULL, mm != 0);
            int ns = 32;
            if (p.trace && bal) HF_NPOLL_INC();
            int spins = 0;
            while (bal) {
                // watchdog: a wait of more than watchdog_spins poll rounds (each >= one
                // L2 round trip: seconds; a schedule bug, never a legal input) gives
                // up instead of hanging the GPU
                if (++spins > p.watchdog_spins) {
                    atomicOr(p.err, ERR_WATCHDOG);
#pragma unroll
                    for (int r = 0; r < RB; ++r)
#pragma unroll
                        for (int j = 0; j < V; ++j) a[r].x[j] = 0.0f;
                    break;
                }
                if (FWD || p.poll_all) {
                    __nanosleep(ns);
                    ns = min(ns * 2, p.sleep_max);
                } else if (lane == __ffs(bal) - 1) {
                    // (backward, HF_POLL_ALL=0, rejected: +20%) one lane polls one missing
                    // vector with back-off, then all re-load
                    const float *src = nullptr;
#pragma unroll
                    for (int r = RB - 1; r >= 0; --r)
                        if (uu[r] >= 0 && uu[r] != INT32_MAX && has_nan<V>(a[r]))
                            src = p.out + int64_t(uu[r]) * S + col;
                    Vec<V> v = ld_relaxed<V>(src);
                    while (has_nan<V>(v)) {
                        __nanosleep(ns);
                        ns = min(ns * 2, p.sleep_max);
                        v = ld_relaxed<V>(src);
                    }
                }
#ifndef HF_BWD_MASK
#define HF_BWD_MASK 1
#endif
                // the bitmask rounds in the forward kernels and in the single-chunk
                // four-column backward (-1..2%; at S = 1 +1.5%: not there); the
                // multi-chunk backward keeps the per-slot loop (the bitmask form cost
                // it +15% at S = 256)
                if constexpr (FWD || (HF_BWD_MASK && ONE && V == 4)) {
#pragma unroll
                    for (int r = 0; r < RB; ++r)
                        if (mm & (1u << r)) a[r] = ld_relaxed<V>(p.out + int64_t(uu[r]) * S + col);
                    unsigned m2 = 0;
#pragma unroll
                    for (int r = 0; r < RB; ++r)
                        if ((mm & (1u << r)) && has_nan<V>(a[r])) m2 |= 1u << r;
                    mm = m2;
                } else {
                    __syncwarp();
#pragma unroll
                    for (int r = 0; r < RB; ++r)
                        if (uu[r] >= 0 && uu[r] != INT32_MAX && has_nan<V>(a[r]))
                            a[r] = ld_relaxed<V>(p.out + int64_t(uu[r]) * S + col);
                    bool miss = false;
#pragma unroll
                    for (int r = 0; r < RB; ++r)
                        if (uu[r] >= 0 && uu[r] != INT32_MAX) miss |= has_nan<V>(a[r]);
                    mm = miss;
                }
                bal = __ballot_sync(FULL, mm != 0);
                if (p.trace) HF_NPOLL_INC();
            }
            if (p.trace && k0 == 0) tr1 = gtimer();
            cp_async_wait_keep1();   // this lane's own delay copies (it reads only those)
#pragma unroll
            for (int r = 0; r < RB; ++r) {
                const int k = k0 + r * G + g;
                if (k < E) {
                    float *dp = s_d + k * SC + gl * V;
                    const Vec<V> dv = ld_s<V>(dp);
                    Vec<V> x;
#pragma unroll
                    for (int j = 0; j < V; ++j) {
                        x.x[j] = relax<FWD>(a[r].x[j], FWD ? sane(dv.x[j], bad) : dv.x[j]);
                    }
                    st_s<V>(dp, x);
                }
            }
        }
        if (GA) cp_async_wait();
        else cp_async_wait_keep1();
        __syncwarp();
#ifdef HF_TRACE_EXT
        const unsigned long long tr2 = p.trace ? gtimer() : 0;
#endif
        // ---- (4) reduce rows / the part, store ----
        if (part) {
            Vec<V> acc;
#pragma unroll
            for (int j = 0; j < V; ++j) acc.x[j] = ident<MX>();
            for (int k = g; k < E; k += G) {   // the edges this group computed
                const Vec<V> x = ld_s<V>(s_d + k * SC + gl * V);
#pragma unroll
                for (int j = 0; j < V; ++j) acc.x[j] = combine<MX>(acc.x[j], x.x[j]);
            }
#pragma unroll
            for (int o = LPN; o < 32; o <<= 1)
#pragma unroll
                for (int j = 0; j < V; ++j)
                    acc.x[j] = combine<MX>(acc.x[j], __shfl_xor_sync(FULL, acc.x[j], o));
#if HF_LASTPART
            // this part's partial -> the row's accumulator; the last part writes the row
            const int rb_rel = s_rp[0] - rp_base, re_rel = s_rp[1] - rp_base;   // row - task edge base
            const int np = (re_rel - rb_rel + LO_PE - 1) / LO_PE;
            const int q0 = (-dsc.y - 1) - (-rb_rel) / LO_PE;   // first part id of the row
            int32_t *ap = p.part_acc + int64_t(q0) * S + col;
            if (g == 0) {
#pragma unroll
                for (int j = 0; j < V; ++j) {
                    if (MX) atomicMax(ap + j, f2ord(acc.x[j]));
                    else atomicMin(ap + j, f2ord(acc.x[j]));
                }
            }
            __syncwarp();   // every lane's red before lane 0's release
            int last = 0;
            // one counter per (row, scenario chunk): every chunk has its own np part tasks
            if (lane == 0) last = atom_add_acq_rel_i(p.part_cnt + int64_t(q0) * p.nch + c, 1) == np - 1;
            last = __shfl_sync(FULL, last, 0);
            if (last) {
                __syncwarp();   // lane 0's acquire before the accumulator loads
                if (!FWD && c != run_c) {
                    flush_run();
                    run_c = c;
                }
                if (g == 0) {
                    const Vec<V> best = ld_ord_relaxed<V>(ap);
                    const int node = s_node[0];
                    st_relaxed<V>(p.out + int64_t(node) * S + col, best);
                    if (FWD && p.prefill) st_plain<V>(p.prefill + int64_t(node) * S + col, nan_vec<V>());
                    if (!FWD && p.other) {
                        const Vec<V> av = ld_relaxed<V>(p.other + int64_t(node) * S + col);
                        Vec<V> sl;
#pragma unroll
                        for (int j = 0; j < V; ++j) {
                            sl.x[j] = EARLY ? __fsub_rn(av.x[j], best.x[j]) : __fsub_rn(best.x[j], av.x[j]);
                            run.x[j] = fminf(run.x[j], sl.x[j]);
                        }
                        if (p.slack) st_plain<V>(p.slack + int64_t(node) * S + col, sl);
                    }
                }
            }
#else
            if (g == 0) st_relaxed<V>(p.part_buf + int64_t(-dsc.y - 1) * S + col, acc);
#endif
        } else {
            if (!FWD && c != run_c) {
                flush_run();
                run_c = c;
            }
            for (int i = g; i < NR; i += G) {
                const int eb = s_rp[i] - rp_base, ee = s_rp[i + 1] - rp_base;
                const int node = s_node[i];
                Vec<V> best;
                if (ee == eb) {
                    if (FWD) {
                        const float a0 = p.src_val ? sane(__ldg(p.src_val + node), bad) : 0.0f;
#pragma unroll
                        for (int j = 0; j < V; ++j) best.x[j] = a0;
                    } else {
#pragma unroll
                        for (int j = 0; j < V; ++j)
                            best.x[j] = sane(p.src_val ? __ldg(p.src_val + col + j) : p.t_scalar, bad);
                    }
                } else {
                    best = ld_s<V>(s_d + eb * SC + gl * V);
                    for (int k = eb + 1; k < ee; ++k) {
                        const Vec<V> x = ld_s<V>(s_d + k * SC + gl * V);
#pragma unroll
                        for (int j = 0; j < V; ++j) best.x[j] = combine<MX>(best.x[j], x.x[j]);
                    }
                }
                st_relaxed<V>(p.out + int64_t(node) * S + col, best);
                if (FWD && p.prefill) st_plain<V>(p.prefill + int64_t(node) * S + col, nan_vec<V>());
                if (!FWD && p.other) {
                    const Vec<V> av = ld_s<V>(s_at + i * SC + gl * V);
                    Vec<V> sl;
#pragma unroll
                    for (int j = 0; j < V; ++j) {
                        // late slack rat - at; early (hold) slack at - rat
                        sl.x[j] = EARLY ? __fsub_rn(av.x[j], best.x[j])
                                        : __fsub_rn(best.x[j], av.x[j]);
                        run.x[j] = fminf(run.x[j], sl.x[j]);
                    }
                    if (p.slack) st_plain<V>(p.slack + int64_t(node) * S + col, sl);
                }
            }
        }
        __syncwarp();   // scratch is rewritten by the next task
        if (p.trace && lane == 0) {
            const int r = t;
            if (r < p.trace_cap) {
                // {warp, start, first gather batch final, all gathers + delays in,
                //  stores issued, poll rounds << 32 | edges << 16 | rows, 0, 0}
                unsigned long long *tr = p.trace + int64_t(r) * 8;
                tr[0] = (unsigned long long)w;
                tr[1] = tr0;
                tr[2] = tr1 ? tr1 : tr0;
#ifdef HF_TRACE_EXT
                tr[3] = tr2;
                tr[5] = (static_cast<unsigned long long>(npoll) << 32) |
                        (static_cast<unsigned long long>(E & 0xffff) << 16) | unsigned(NR & 0xffff);
#else
                tr[3] = tr[2];
                tr[5] = (static_cast<unsigned long long>(E & 0xffff) << 16) | unsigned(NR & 0xffff);
#endif
                tr[4] = gtimer();
                tr[6] = 0;
                tr[7] = 0;
            }
        }
#if HF_IDX_SMEM
        ++it;
        rs = rs == 2 ? 0 : rs + 1;
        __syncwarp();   // the index buffer / ring slot of this task is rewritten next
#else
        X0 = X1;
#endif
    }

    if (bad) atomicOr(p.err, ERR_NONFINITE);
    if (!FWD) {
        flush_run();
        __syncthreads();
        for (int s = threadIdx.x; s < S; s += blockDim.x)
            if (s_wmin[s] != 0x7f800000) atomicMin(p.wns_ord + s, s_wmin[s]);
    }
}

// After a pass: every long row gets its value (combine of its partials), its
// optional slack and its worst-slack contribution.  One thread per (first part id,
// V-wide column vector) up to the exact part count read on the device: all long
// rows and columns in parallel, the partials of a row loaded eight at a time; worst
// slack folded per block (ordered-int atomicMin).
template <bool FWD, bool EARLY, int V>
__global__ void k_finalize_split(const int32_t *__restrict__ np_arr, const int32_t *__restrict__ prow,
                                 const int32_t *__restrict__ nparts_dev,
                                 const int32_t *__restrict__ node_of, int32_t S,
                                 const float *__restrict__ part_buf, float *__restrict__ out,
                                 const float *__restrict__ other, float *__restrict__ slack,
                                 int32_t *__restrict__ wns_ord, float *__restrict__ prefill) {
    constexpr bool MX = FWD != EARLY;
    constexpr int FB = 8;   // partials in flight per thread
    extern __shared__ int32_t s_wmin[];
    const bool do_slack = !FWD && other;
    if (do_slack) {
        for (int s = threadIdx.x; s < S; s += blockDim.x) s_wmin[s] = 0x7f800000;
        __syncthreads();
    }
    const int64_t nparts = *nparts_dev;   // exact part count (the grid is sized by a bound)
    const int lpn = S / V;   // column vectors per row
    // long row p (first part id), column vector at col: combine the partials, store,
    // slack; the row minimum of the slack goes to mn
    auto row_vec = [&](int64_t p, int np, int64_t col, float *mn) {
        const int row = prow[p];
        const float *base = part_buf + p * S + col;
        Vec<V> acc;
        for (int k = 0; k < np; k += FB) {
            Vec<V> v[FB];
#pragma unroll
            for (int u = 0; u < FB; ++u)
                if (k + u < np) v[u] = ld_relaxed<V>(base + int64_t(k + u) * S);
            if (k == 0) acc = v[0];
#pragma unroll
            for (int u = 0; u < FB; ++u)
                if (k + u < np && k + u > 0)
#pragma unroll
                    for (int j = 0; j < V; ++j) acc.x[j] = combine<MX>(acc.x[j], v[u].x[j]);
        }
        const int64_t node = node_of[row];
        st_plain<V>(out + node * S + col, acc);
        if (FWD && prefill) st_plain<V>(prefill + node * S + col, nan_vec<V>());
        if (do_slack) {
            const Vec<V> a = ld_relaxed<V>(other + node * S + col);   // final: after the pass
            Vec<V> sl;
#pragma unroll
            for (int j = 0; j < V; ++j) {
                sl.x[j] = EARLY ? __fsub_rn(a.x[j], acc.x[j]) : __fsub_rn(acc.x[j], a.x[j]);
                mn[j] = fminf(mn[j], sl.x[j]);
            }
            if (slack) st_plain<V>(slack + node * S + col, sl);
        }
    };
    if (lpn <= int(blockDim.x)) {
        // a thread keeps one column vector (lane) for all its rows: minima in registers
        const int apb = blockDim.x / lpn * lpn;            // active threads per block
        const int64_t step = int64_t(gridDim.x) * apb;     // a multiple of lpn: lane fixed
        const int lane = int(threadIdx.x % lpn);
        const int64_t col = int64_t(lane) * V;
        float mn[V];
#pragma unroll
        for (int j = 0; j < V; ++j) mn[j] = __int_as_float(0x7f800000);
        if (int(threadIdx.x) < apb) {
            for (int64_t t = blockIdx.x * int64_t(apb) + threadIdx.x; t < nparts * lpn; t += step) {
                const int64_t p = t / lpn;
                const int np = np_arr[p];
                if (np == 0) continue;   // not the first part of a row
                row_vec(p, np, col, mn);
            }
            if (do_slack)
#pragma unroll
                for (int j = 0; j < V; ++j)
                    if (mn[j] != __int_as_float(0x7f800000))
                        atomicMin(s_wmin + col + j, f2ord(mn[j]));
        }
    } else {
        // rows wider than the block (S / V > blockDim): a block per row, the column
        // vectors strided over its threads, minima folded per row
        for (int64_t p = blockIdx.x; p < nparts; p += gridDim.x) {
            const int np = np_arr[p];
            if (np == 0) continue;
            for (int cv = threadIdx.x; cv < lpn; cv += blockDim.x) {
                float mn[V];
#pragma unroll
                for (int j = 0; j < V; ++j) mn[j] = __int_as_float(0x7f800000);
                row_vec(p, np, int64_t(cv) * V, mn);
                if (do_slack)
#pragma unroll
                    for (int j = 0; j < V; ++j)
                        if (mn[j] != __int_as_float(0x7f800000))
                            atomicMin(s_wmin + cv * V + j, f2ord(mn[j]));
            }
        }
    }
    if (do_slack) {
        __syncthreads();
        for (int s = threadIdx.x; s < S; s += blockDim.x)
            if (s_wmin[s] != 0x7f800000) atomicMin(wns_ord + s, s_wmin[s]);
    }
}

// plain neighbour ids (HF_LASTPART): a long neighbour's -(first part id + 1) -> its node
__global__ void k_plain_nbr(const int32_t *__restrict__ nbr, const int32_t *__restrict__ part_row,
                            const int32_t *__restrict__ node_of, int32_t m, int32_t *__restrict__ out) {
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < m;
         e += int64_t(gridDim.x) * blockDim.x) {
        const int u = nbr[e];
        out[e] = u >= 0 ? u : node_of[part_row[-u - 1]];
    }
}
// the long rows' accumulators at the combine's identity and their part counters at 0
__global__ void k_fill_acc(int32_t *acc, int32_t *cnt, const int32_t *count, int32_t S, int32_t nch,
                           int32_t ident) {
    const int64_t np = *count, total = np * S;   // nch <= S: the counters fit the same sweep
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total;
         i += int64_t(gridDim.x) * blockDim.x) {
        acc[i] = ident;
        if (i < np * nch) cnt[i] = 0;
    }
}

__global__ void k_fill_parts(uint32_t *buf, const int32_t *count, int32_t S) {
    const int64_t total = int64_t(*count) * S;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total;
         i += int64_t(gridDim.x) * blockDim.x)
        buf[i] = 0xffffffffu;
}

// flags a NaN / inf among count floats (the concurrent batch's pre-check)
__global__ void k_check_finite(const float *__restrict__ x, int64_t count, uint32_t *err) {
    bool bad = false;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < count;
         i += int64_t(gridDim.x) * blockDim.x)
        bad |= !(fabsf(__ldcs(x + i)) <= 3.40282346638528859812e+38f);
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(err, ERR_NONFINITE);
}

__global__ void k_fill_i32(int32_t *p, int32_t v, int64_t count) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < count;
         i += int64_t(gridDim.x) * blockDim.x)
        p[i] = v;
}

__global__ void k_ord_to_float(const int32_t *__restrict__ k, float *__restrict__ f,
                               int32_t count) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < count; i += gridDim.x * blockDim.x)
        f[i] = ord2f(k[i]);
}

// slack = fl(rat - at) for every node and scenario, the worst slack per scenario
// (ordered-int atomicMin), optional slack store: the epilogue of the concurrent
// batch, where the backward kernel runs next to the forward one and never sees at.
template <int V, bool EARLY>
__global__ void k_slack_wns(const float *__restrict__ at, const float *__restrict__ rat,
                            float *__restrict__ slack, int32_t n, int32_t S,
                            int32_t *__restrict__ wns_ord) {
    extern __shared__ int32_t s_wmin[];
    for (int s = threadIdx.x; s < S; s += blockDim.x) s_wmin[s] = 0x7f800000;
    __syncthreads();
    const int lpn = S / V;   // column vectors per row
    // one (row, column vector): slack, its optional store, the minimum into mn
    auto one = [&](int64_t row, int64_t col, float *mn) {
        const int64_t o = row * S + col;
        Vec<V> a, r, sl;
        if constexpr (V == 4) {
            const float4 x = __ldcs(reinterpret_cast<const float4 *>(at + o));
            const float4 y = __ldcs(reinterpret_cast<const float4 *>(rat + o));
            a.x[0] = x.x; a.x[1] = x.y; a.x[2] = x.z; a.x[3] = x.w;
            r.x[0] = y.x; r.x[1] = y.y; r.x[2] = y.z; r.x[3] = y.w;
        } else {
#pragma unroll
            for (int j = 0; j < V; ++j) {
                a.x[j] = __ldcs(at + o + j);
                r.x[j] = __ldcs(rat + o + j);
            }
        }
#pragma unroll
        for (int j = 0; j < V; ++j) {
            sl.x[j] = EARLY ? __fsub_rn(a.x[j], r.x[j]) : __fsub_rn(r.x[j], a.x[j]);
            mn[j] = fminf(mn[j], sl.x[j]);
        }
        if (slack) st_plain<V>(slack + o, sl);
    };
    if (lpn <= int(blockDim.x)) {
        const int apb = blockDim.x / lpn * lpn;             // active threads per block
        const int64_t step = int64_t(gridDim.x) * apb;      // a multiple of lpn: lane fixed
        const int lane = int(threadIdx.x % lpn);
        float mn[V];
#pragma unroll
        for (int j = 0; j < V; ++j) mn[j] = __int_as_float(0x7f800000);
        if (int(threadIdx.x) < apb) {
            for (int64_t t = blockIdx.x * int64_t(apb) + threadIdx.x; t < int64_t(n) * lpn; t += step)
                one(t / lpn, int64_t(lane) * V, mn);
#pragma unroll
            for (int j = 0; j < V; ++j)
                if (mn[j] != __int_as_float(0x7f800000)) atomicMin(s_wmin + lane * V + j, f2ord(mn[j]));
        }
    } else {
        // rows wider than the block: column vectors strided over the threads, minima
        // per thread and column vector over the block's rows
        for (int cv = threadIdx.x; cv < lpn; cv += blockDim.x) {
            float mn[V];
#pragma unroll
            for (int j = 0; j < V; ++j) mn[j] = __int_as_float(0x7f800000);
            for (int64_t row = blockIdx.x; row < n; row += gridDim.x) one(row, int64_t(cv) * V, mn);
#pragma unroll
            for (int j = 0; j < V; ++j)
                if (mn[j] != __int_as_float(0x7f800000)) atomicMin(s_wmin + cv * V + j, f2ord(mn[j]));
        }
    }
    __syncthreads();
    for (int s = threadIdx.x; s < S; s += blockDim.x)
        if (s_wmin[s] != 0x7f800000) atomicMin(wns_ord + s, s_wmin[s]);
}

// ---- task schedule (per direction; cached per tw) --------------------------------
// Inside a level the short rows (degree <= LO_SPLIT) come first, then the long ones
// (levelize.cu).  A short row weighs degree + 1; normal task j of a level holds the
// rows whose weight prefix from the level start lies in [j*tw, (j+1)*tw), so it has
// <= tw rows and <= tw + LO_SPLIT - rows edges; the prefix of row i is
// (row_ptr[i] - row_ptr[ls]) + (i - ls), no scan needed.  A level has
// floor(prefix of its last short row / tw) + 1 normal tasks (some may be empty when
// one row spans several multiples of tw).  Long row i becomes parts q[i]..q[i+1]-1
// of <= LO_PE edges.
// Per-level task counts and their prefix sums in one block (L is small): pass-level
// q = k (forward) or L-1-k (backward) has nt[q] = ntn + parts tasks per chunk,
// ntn = ceil-ish(weight of its short rows / tw); doff = exclusive scan of nt (the
// first descriptor of q), tb = exclusive scan of nt * nch (first global task of q).
__global__ void __launch_bounds__(1024) k_tb_sched(
    const int32_t *__restrict__ level_ptr, const int32_t *__restrict__ lstart,
    const int32_t *__restrict__ Q, const int32_t *__restrict__ row_ptr, int32_t L, int32_t tw,
    int32_t fwd, int32_t nch, int32_t *__restrict__ nt, int32_t *__restrict__ ntn,
    int32_t *__restrict__ doff, int32_t *__restrict__ tb) {
    __shared__ int warp_a[32], warp_b[32];
    __shared__ int carry_a, carry_b;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    if (threadIdx.x == 0) carry_a = carry_b = 0;
    __syncthreads();
    for (int q0 = 0; q0 < L; q0 += blockDim.x) {
        const int q = q0 + threadIdx.x;
        int a = 0;
        if (q < L) {
            const int k = fwd ? q : L - 1 - q;
            const int ls = level_ptr[k], le = level_ptr[k + 1], lo = lstart[k];
            const int c = lo > ls ? ((row_ptr[lo - 1] - row_ptr[ls]) + (lo - 1 - ls)) / tw + 1 : 0;
            ntn[k] = c;
            a = c + (Q[le] - Q[ls]);
            nt[q] = a;
        }
        int xa = a, xb = a * nch;
        const int va = xa, vb = xb;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int ya = __shfl_up_sync(0xffffffffu, xa, o);
            const int yb = __shfl_up_sync(0xffffffffu, xb, o);
            if (lane >= o) {
                xa += ya;
                xb += yb;
            }
        }
        if (lane == 31) {
            warp_a[wid] = xa;
            warp_b[wid] = xb;
        }
        __syncthreads();
        if (wid == 0) {
            int sa = lane < nw ? warp_a[lane] : 0, sb = lane < nw ? warp_b[lane] : 0;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int ya = __shfl_up_sync(0xffffffffu, sa, o);
                const int yb = __shfl_up_sync(0xffffffffu, sb, o);
                if (lane >= o) {
                    sa += ya;
                    sb += yb;
                }
            }
            if (lane < nw) {
                warp_a[lane] = sa;
                warp_b[lane] = sb;
            }
        }
        __syncthreads();
        const int ba = carry_a + (wid ? warp_a[wid - 1] : 0) + xa - va;
        const int bb = carry_b + (wid ? warp_b[wid - 1] : 0) + xb - vb;
        if (q < L) {
            doff[q] = ba;
            tb[q] = bb;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            carry_a += warp_a[nw - 1];
            carry_b += warp_b[nw - 1];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        nt[L] = 0;
        doff[L] = carry_a;
        tb[L] = carry_b;
    }
}
// task-base prefix only (a cached schedule used with another chunk count)
__global__ void __launch_bounds__(1024) k_tb_bases(const int32_t *__restrict__ nt, int32_t L,
                                                   int32_t nch, int32_t *__restrict__ tb) {
    __shared__ int warp_b[32];
    __shared__ int carry_b;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    if (threadIdx.x == 0) carry_b = 0;
    __syncthreads();
    for (int q0 = 0; q0 < L; q0 += blockDim.x) {
        const int q = q0 + threadIdx.x;
        const int vb = q < L ? nt[q] * nch : 0;
        int xb = vb;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int yb = __shfl_up_sync(0xffffffffu, xb, o);
            if (lane >= o) xb += yb;
        }
        if (lane == 31) warp_b[wid] = xb;
        __syncthreads();
        if (wid == 0) {
            int sb = lane < nw ? warp_b[lane] : 0;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int yb = __shfl_up_sync(0xffffffffu, sb, o);
                if (lane >= o) sb += yb;
            }
            if (lane < nw) warp_b[lane] = sb;
        }
        __syncthreads();
        if (q < L) tb[q] = carry_b + (wid ? warp_b[wid - 1] : 0) + xb - vb;
        __syncthreads();
        if (threadIdx.x == 0) carry_b += warp_b[nw - 1];
        __syncthreads();
    }
    if (threadIdx.x == 0) tb[L] = carry_b;
}
// Descriptors, one thread per row.  A short row i (> level start) starts every task
// j with P(i-1) < j*tw <= P(i) and ends task j - 1 (P = weight prefix of the
// level's short rows); a long row writes its part tasks after the level's ntn.
__global__ void k_tb_rows(const int32_t *__restrict__ level_ptr, const int32_t *__restrict__ row_ptr,
                          const int32_t *__restrict__ doff, const int32_t *__restrict__ ntn,
                          const int32_t *__restrict__ lstart, const int32_t *__restrict__ Q,
                          const int32_t *__restrict__ level, const int32_t *__restrict__ node_of,
                          int32_t n, int32_t L, int32_t tw, int32_t fwd, int4 *__restrict__ desc) {
    for (int64_t ii = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; ii < n;
         ii += int64_t(gridDim.x) * blockDim.x) {
        const int i = int(ii);
        const int k = level[node_of[i]];
        const int ls = level_ptr[k], lo = lstart[k];
        const int d0 = doff[fwd ? k : L - 1 - k];
        const int nn = ntn[k];
        if (i >= lo) {   // long row: its part tasks
            const int q0 = Q[i], np = Q[i + 1] - q0;
            const int rb = row_ptr[i], re = row_ptr[i + 1];
            const int base = d0 + nn + (q0 - Q[ls]);
            for (int t = 0; t < np; ++t)
                desc[base + t] = make_int4(i, -(q0 + t + 1), rb + t * LO_PE,
                                           min(re, rb + (t + 1) * LO_PE));
            continue;
        }
        int *d = reinterpret_cast<int *>(desc + d0);
        const int r0 = row_ptr[ls];
        const int rp = row_ptr[i];
        if (i == ls) {
            d[0] = i;
            d[2] = rp;
        } else {
            const int pprev = (row_ptr[i - 1] - r0) + (i - 1 - ls);
            const int pcur = (rp - r0) + (i - ls);
            const int jlo = pprev / tw + 1, jhi = pcur / tw;
            for (int j = jlo; j <= jhi; ++j) {
                d[4 * j] = i;
                d[4 * j + 2] = rp;
                d[4 * (j - 1) + 1] = i;
                d[4 * (j - 1) + 3] = rp;
            }
        }
        if (i == lo - 1) {
            d[4 * (nn - 1) + 1] = lo;
            d[4 * (nn - 1) + 3] = row_ptr[lo];
        }
    }
}

// no host round trip: descriptors are sized by the bound (n + m)/tw + L + parts.
// Two launches: the per-level counts and prefixes (one block), the descriptors.
template <bool FWD>
void build_tasks(Graph &g, const int32_t *row_ptr, const int32_t *node_of, const int32_t *Q,
                 int32_t nparts, int tw, int nch, TaskSched &ts) {
    cudaStream_t s = g.stream;
    const int32_t n = g.n, L = g.L, m = g.m;
    const int32_t *lst = FWD ? g.lo_in_lstart.as<int32_t>() : g.lo_out_lstart.as<int32_t>();
    DevBuf ntn;
    ntn.alloc(sizeof(int32_t) * (int64_t(L) + 1), s);
    ts.nt.alloc(sizeof(int32_t) * (int64_t(L) + 1), s);
    ts.doff.alloc(sizeof(int32_t) * (int64_t(L) + 1), s);
    ts.tb.alloc(sizeof(int32_t) * (int64_t(L) + 1), s);
    k_tb_sched<<<1, 1024, 0, s>>>(g.level_ptr.as<int32_t>(), lst, Q, row_ptr, L, tw, FWD ? 1 : 0,
                                  nch, ts.nt.as<int32_t>(), ntn.as<int32_t>(),
                                  ts.doff.as<int32_t>(), ts.tb.as<int32_t>());
    HF_CHECK_LAUNCH();
    const int64_t cap = (int64_t(n) + m) / tw + L + nparts + 1;
    ts.desc.alloc(sizeof(int4) * size_t(cap), s);
    k_tb_rows<<<grid_for(n, 256, g.sms), 256, 0, s>>>(
        g.level_ptr.as<int32_t>(), row_ptr, ts.doff.as<int32_t>(), ntn.as<int32_t>(), lst, Q,
        g.level.as<int32_t>(), node_of, n, L, tw, FWD ? 1 : 0, ts.desc.as<int4>());
    HF_CHECK_LAUNCH();
    g.launches += 2;
    ts.tb_nch = nch;
}

void task_bases(Graph &g, TaskSched &ts, int nch) {
    if (ts.tb_nch == nch) return;
    cudaStream_t s = g.stream;
    k_tb_bases<<<1, 1024, 0, s>>>(ts.nt.as<int32_t>(), g.L, nch, ts.tb.as<int32_t>());
    HF_CHECK_LAUNCH();
    g.launches += 1;
    ts.tb_nch = nch;
}

int pick_vec(int32_t S, std::initializer_list<const void *> ptrs) {
    auto aligned = [&](int bytes) {
        for (const void *q : ptrs)
            if (q && (reinterpret_cast<uintptr_t>(q) % bytes)) return false;
        return true;
    };
    if (S % 4 == 0 && aligned(16)) return 4;
    if (S % 2 == 0 && aligned(8)) return 2;
    return 1;
}

void prof_record(Graph &g, int idx, cudaStream_t st = nullptr) {
    if (g.prof) HF_CUDA(cudaEventRecord(g.ev[idx], st ? st : g.stream));
}

int env_int(const char *name, int dflt) {
    const char *e = getenv(name);
    return e ? atoi(e) : dflt;
}

template <int V, int LPN, bool FWD, bool GA, bool EARLY, bool ONE>
void launch_flow(Graph &g, FlowParams &p, cudaStream_t st, int cap_per_sm) {
    auto kern = k_flow<V, LPN, FWD, GA, EARLY, ONE>;
    constexpr int SC = V * LPN;
    const WarpLayout WL = warp_layout(p.ecap, p.ncap, SC, FWD, GA);
    const size_t smem = size_t(wmin_bytes(p.S)) + size_t(NWARP) * WL.bytes;
    // attribute + occupancy per (kernel, smem, device) once: no driver queries per call
    static std::map<std::tuple<const void *, size_t, int>, int> cache;
    static std::mutex mu;
    int per_sm = 0;
    const auto key = std::make_tuple((const void *)kern, smem, g.device);
    {
        std::lock_guard<std::mutex> lk(mu);
        auto it = cache.find(key);
        if (it != cache.end()) per_sm = it->second;
    }
    if (!per_sm) {
        ensure_dyn_smem((const void *)kern, g.device, smem);
        HF_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, FLOW_THREADS, smem));
        std::lock_guard<std::mutex> lk(mu);
        cache[key] = per_sm;
    }
    ensure_dyn_smem((const void *)kern, g.device, smem);   // (cached: a map lookup)
    if (per_sm < 1) fail(HF_ERR_CUDA, "propagation kernel does not fit on an SM");
    const int cap = env_int("HF_CTAS_PER_SM", 0);
    if (cap > 0) per_sm = std::min(per_sm, cap);
    if (cap_per_sm > 0) per_sm = std::min(per_sm, cap_per_sm);
    void *args[] = {&p};
    // all warps co-resident (cooperative launch): required by the dataflow wait.
    // With profiling on, events bracket exactly this launch (forward: ev 2/3,
    // backward 5/4).
    prof_record(g, FWD ? 2 : 5, st);
    HF_CUDA(cudaLaunchCooperativeKernel((const void *)kern, g.sms * per_sm, FLOW_THREADS, args,
                                        smem, st));
    prof_record(g, FWD ? 3 : 4, st);
    g.launches += 1;
}

// blocks per SM a kernel can keep resident alone (cached occupancy query)
template <int V, int LPN, bool FWD, bool GA, bool EARLY, bool ONE>
int occupancy_of(FlowParams &p) {
    auto kern = k_flow<V, LPN, FWD, GA, EARLY, ONE>;
    const WarpLayout WL = warp_layout(p.ecap, p.ncap, V * LPN, FWD, GA);
    const size_t smem = size_t(wmin_bytes(p.S)) + size_t(NWARP) * WL.bytes;
    static std::map<size_t, int> cache;
    static std::mutex mu;
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(smem);
    if (it != cache.end()) return it->second;
    int per_sm = 0;
    int dev = 0;
    HF_CUDA(cudaGetDevice(&dev));
    ensure_dyn_smem((const void *)kern, dev, smem);
    HF_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, FLOW_THREADS, smem));
    cache[smem] = per_sm;
    return per_sm;
}

// op = 0: launch, op = 1: return the solo occupancy (blocks per SM)
template <bool FWD, bool GA, bool EARLY>
int dispatch_ga(Graph &g, FlowParams &p, int LPN, cudaStream_t st, int cap, int op) {
    // one scenario chunk (S = V * LPN: S = 64 is the C4 headline, also S = 4..32):
    // the specialised kernel without the task locator
    const bool one = p.nch == 1 && env_int("HF_ONE", 1);
#define HF_CASE(L)                                                               \
    case L:                                                                      \
        if (one) {                                                               \
            if (op) return occupancy_of<4, L, FWD, GA, EARLY, true>(p);          \
            launch_flow<4, L, FWD, GA, EARLY, true>(g, p, st, cap);              \
            return 0;                                                            \
        }                                                                        \
        if (op) return occupancy_of<4, L, FWD, GA, EARLY, false>(p);             \
        launch_flow<4, L, FWD, GA, EARLY, false>(g, p, st, cap);                 \
        return 0;
    switch (LPN) {
        HF_CASE(16)
        HF_CASE(8)
        HF_CASE(4)
        HF_CASE(2)
    default:
        HF_CASE(1)
    }
#undef HF_CASE
}
template <bool FWD, bool EARLY>
int dispatch_mode(Graph &g, FlowParams &p, int V, int LPN, cudaStream_t st, int cap, int op) {
    if (V == 4) {
        // the cp.async-gather variant (HF_GA=1, measured slower) exists for late mode only
        if (!EARLY && env_int("HF_GA", 0))
            return dispatch_ga<FWD, true, false>(g, p, LPN, st, cap, op);
        return dispatch_ga<FWD, false, EARLY>(g, p, LPN, st, cap, op);
    } else if (V == 2) {
        // (S = 2: one chunk; odd multiples of 2 above: several)
        if (p.nch == 1 && env_int("HF_ONE", 1)) {
            if (op) return occupancy_of<2, 1, FWD, false, EARLY, true>(p);
            launch_flow<2, 1, FWD, false, EARLY, true>(g, p, st, cap);
        } else {
            if (op) return occupancy_of<2, 1, FWD, false, EARLY, false>(p);
            launch_flow<2, 1, FWD, false, EARLY, false>(g, p, st, cap);
        }
    } else {
        // (S = 1, the single-graph calls: one chunk)
        if (p.nch == 1 && env_int("HF_ONE", 1)) {
            if (op) return occupancy_of<1, 1, FWD, false, EARLY, true>(p);
            launch_flow<1, 1, FWD, false, EARLY, true>(g, p, st, cap);
        } else {
            if (op) return occupancy_of<1, 1, FWD, false, EARLY, false>(p);
            launch_flow<1, 1, FWD, false, EARLY, false>(g, p, st, cap);
        }
    }
    return 0;
}
template <bool FWD>
int dispatch(Graph &g, FlowParams &p, int V, int LPN, cudaStream_t st = nullptr, int cap = 0,
             int op = 0) {
    if (!st) st = g.stream;
    if (g.early) return dispatch_mode<FWD, true>(g, p, V, LPN, st, cap, op);
    return dispatch_mode<FWD, false>(g, p, V, LPN, st, cap, op);
}

// host-side state of a prepared pass
struct PassCtx {
    int LPN = 1;
    int32_t nparts = 0;
    const int32_t *Q = nullptr;
    DevBuf part_buf;
};

// all-ones (NaN sentinel) fill, 16-byte grid-stride stores: faster than
// cudaMemsetAsync of the same bytes
__global__ void k_fill_nan4(uint4 *__restrict__ p4, size_t n4, uint32_t *__restrict__ p,
                            size_t n) {
    const uint4 v = make_uint4(~0u, ~0u, ~0u, ~0u);
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n4;
         i += size_t(gridDim.x) * blockDim.x)
        p4[i] = v;
    for (size_t i = n4 * 4 + blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n;
         i += size_t(gridDim.x) * blockDim.x)
        p[i] = ~0u;
}

void fill_nan(Graph &g, float *buf, size_t cnt, cudaStream_t st) {
    const int ctas = env_int("HF_FILL_CTAS", 16 * g.sms);   // 0: cudaMemsetAsync (16 per SM: -1% phase vs 8)
    if (ctas > 0 && (reinterpret_cast<uintptr_t>(buf) & 15) == 0) {
        k_fill_nan4<<<ctas, 256, 0, st>>>(reinterpret_cast<uint4 *>(buf), cnt / 4,
                                          reinterpret_cast<uint32_t *>(buf), cnt);
        HF_CHECK_LAUNCH();
        g.launches += 1;
    } else {
        HF_CUDA(cudaMemsetAsync(buf, 0xff, sizeof(float) * cnt, st));
    }
}

void pnbr_prepare(Graph &g) {
    if (g.pnbr_ready) return;
    cudaStream_t s = g.stream;
    for (int dir = 0; dir < 2; ++dir) {
        const bool in = dir == 0;
        DevBuf &pn = in ? g.lo_in_pnbr : g.lo_out_pnbr;
        pn.alloc(sizeof(int32_t) * std::max<int64_t>(g.m, 1), s);
        if (!g.m) continue;
        const int32_t *npa = in ? g.lo_in_np.as<int32_t>() : g.lo_out_np.as<int32_t>();
        k_plain_nbr<<<grid_for(g.m, 256, g.sms), 256, 0, s>>>(
            in ? g.lo_in_nbr.as<int32_t>() : g.lo_out_nbr.as<int32_t>(),
            npa + (in ? g.np_cap_in : g.np_cap_out),
            in ? g.lo_in_node.as<int32_t>() : g.lo_out_node.as<int32_t>(), g.m, pn.as<int32_t>());
        HF_CHECK_LAUNCH();
        g.launches += 1;
    }
    g.pnbr_ready = true;
}

// task schedule, bases, partial buffer and the sentinel fill of the output (on the
// graph's stream)
template <bool FWD>
void prepare_pass(Graph &g, FlowParams &p, int V, PassCtx &cx, bool fill_out = true) {
    cudaStream_t s = g.stream;
    // scenario chunk: SC = V * LPN columns (largest power of two <= HF_SC dividing S)
    const int sc_max = std::max(1, env_int("HF_SC", 64));
    int LPN = 1;
    if (V == 4)
        while (LPN < 16 && p.S % (V * LPN * 2) == 0 && V * LPN * 2 <= sc_max) LPN *= 2;
    const int G = 32 / LPN;
    cx.LPN = LPN;
    p.nch = p.S / (V * LPN);
    p.nch_shift = (p.nch & (p.nch - 1)) == 0 ? __builtin_ctz(unsigned(p.nch)) : -1;
    // task shape: weight tw (rows + edges) per task; rows longer than LO_SPLIT edges
    // (at the end of their level, levelize.cu) are cut into parts of LO_PE edges;
    // scratch capacity ecap = tw + LO_SPLIT edges (>= LO_PE), ncap = tw rows
    const int slots = LPN <= 2 ? 2 : 1;   // idx_slots<LPN>()
    // measured per direction (tools/tune.py, C3 S=64): forward 12, backward 14
    // measured (C4, profiles/round2/c4_flow_variants.txt): one 64-column chunk per row
    // (S = 64) wants smaller tasks (forward 11, backward 10: -3%; with the single-chunk
    // kernel forward 10, -2%: profiles/round2/tw_retune_ab.txt); two chunks (S = 128)
    // 12 / 14; four and more (S = 256, 1024: the level already has >= 4x the tasks)
    // larger forward tasks (20: -4..-10% forward), backward 14
    const int tw_fb = p.nch == 1 ? (FWD ? 10 : 10) : (p.nch == 2 ? (FWD ? 12 : 14) : (FWD ? 20 : 14));
    const int tw_dflt = slots == 2 ? 32 : (G <= 2 ? tw_fb : 16);
    int tw = env_int(FWD ? "HF_TW_F" : "HF_TW_B", env_int("HF_TW", tw_dflt));
    tw = std::max(4, std::min(tw, 32 * slots - LO_SPLIT));
    p.ecap = std::max(tw + LO_SPLIT, LO_PE);   // a part task has up to LO_PE edges
    p.ncap = tw;
    p.sleep_max = std::max(32, env_int(FWD ? "HF_SLEEP_MAX" : "HF_SLEEP_MAX_B", env_int("HF_SLEEP_MAX", 64)));
    p.watchdog_spins = std::max(1, env_int("HF_WATCHDOG_SPINS", 1 << 22));
    p.poll_all = env_int("HF_POLL_ALL", 1);
    TaskSched &ts = FWD ? g.ts_f : g.ts_b;
    cx.nparts = FWD ? g.np_cap_in : g.np_cap_out;   // bound; exact count on the device
    const int32_t *nparts_dev = g.nparts_d + (FWD ? 0 : 1);
    cx.Q = FWD ? g.lo_in_q.as<int32_t>() : g.lo_out_q.as<int32_t>();
    // task ids and bases are int32: bound the pass's task count (the descriptor bound
    // of build_tasks times the chunk count)
    if (((int64_t(g.n) + g.m) / tw + g.L + cx.nparts + 1) * p.nch > INT32_MAX)
        fail(HF_ERR_INVALID_ARG, "too many warp tasks for one pass (scenario count x graph size)");
    if (ts.key != tw || !ts.desc.p) {
        build_tasks<FWD>(g, p.row_ptr, p.node_of, cx.Q, cx.nparts, tw, p.nch, ts);
        ts.key = tw;
    }
    task_bases(g, ts, p.nch);
    p.desc = ts.desc.as<int4>();
    p.nt = ts.nt.as<int32_t>();
    p.doff = ts.doff.as<int32_t>();
    p.tb = ts.tb.as<int32_t>();
    p.part_np = FWD ? g.lo_in_np.as<int32_t>() : g.lo_out_np.as<int32_t>();
    p.L = g.L;
    p.err = g.d_err();
#if HF_LASTPART
    pnbr_prepare(g);
    p.nbr = FWD ? g.lo_in_pnbr.as<int32_t>() : g.lo_out_pnbr.as<int32_t>();
    if (cx.nparts > 0) {
        cx.part_buf.alloc(sizeof(int32_t) * size_t(cx.nparts) * (size_t(p.S) + size_t(p.nch)), s);
        p.part_acc = cx.part_buf.as<int32_t>();
        p.part_cnt = p.part_acc + size_t(cx.nparts) * p.S;
        const bool mx = FWD != g.early;   // max for late forward / early backward
        k_fill_acc<<<grid_for(int64_t(cx.nparts) * p.S, 256, g.sms), 256, 0, s>>>(
            p.part_acc, p.part_cnt, nparts_dev, p.S, p.nch,
            mx ? int32_t(0x807fffff) : int32_t(0x7f800000));
        HF_CHECK_LAUNCH();
        g.launches += 1;
    }
    if (false) {
#else
    if (cx.nparts > 0) {
#endif
        cx.part_buf.alloc(sizeof(float) * size_t(cx.nparts) * p.S, s);
        p.part_buf = cx.part_buf.as<float>();
        // NaN sentinel over the partials actually used (count read on the device)
        k_fill_parts<<<grid_for(int64_t(cx.nparts) * p.S / 4 + 1, 256, g.sms), 256, 0, s>>>(
            reinterpret_cast<uint32_t *>(p.part_buf), nparts_dev, p.S);
        HF_CHECK_LAUNCH();
        g.launches += 1;
    }
    // the NaN sentinel (all-ones bit pattern): "not yet computed"
    if (fill_out) fill_nan(g, p.out, size_t(g.n) * p.S, s);
}

// the dataflow kernel and the long-row finalisation, on stream st
template <bool FWD>
void launch_pass(Graph &g, FlowParams &p, bool check_d, int V, PassCtx &cx, cudaStream_t st,
                 int cap) {
    dispatch<FWD>(g, p, V, cx.LPN, st, cap);
    if (!HF_LASTPART && cx.nparts > 0) {
        const int32_t *npa = FWD ? g.lo_in_np.as<int32_t>() : g.lo_out_np.as<int32_t>();
        const int32_t *prow = npa + (FWD ? g.np_cap_in : g.np_cap_out);
        const int32_t *nparts_dev = g.nparts_d + (FWD ? 0 : 1);
        const int lpn = p.S / V;
        const int grid = grid_for(int64_t(cx.nparts) * lpn, 256, g.sms);
        const size_t sm = sizeof(int32_t) * size_t(p.S);
#define HF_FIN(EE, VV)                                                                    \
    k_finalize_split<FWD, EE, VV><<<grid, 256, sm, st>>>(npa, prow, nparts_dev, p.node_of, p.S, \
                                                          p.part_buf, p.out, p.other, p.slack, \
                                                          p.wns_ord, p.prefill)
        if (g.early) {
            if (V == 4) HF_FIN(true, 4);
            else if (V == 2) HF_FIN(true, 2);
            else HF_FIN(true, 1);
        } else {
            if (V == 4) HF_FIN(false, 4);
            else if (V == 2) HF_FIN(false, 2);
            else HF_FIN(false, 1);
        }
#undef HF_FIN
        HF_CHECK_LAUNCH();
        g.launches += 1;
    }
}

// one pass: task schedule, sentinel fill, the dataflow kernel, split-row finalise
template <bool FWD> void run_pass(Graph &g, FlowParams &p, bool check_d, int V) {
    cudaStream_t s = g.stream;
    PassCtx cx;
    prepare_pass<FWD>(g, p, V, cx);
    const int SC = V * cx.LPN;
    // debugging timeline: HF_TRACE=<file prefix> dumps one record per task
    const char *trace_env = getenv("HF_TRACE");
    DevBuf tbuf;
    int32_t ntask = 0;
    if (trace_env) {
        HF_CUDA(cudaMemcpyAsync(&ntask, p.tb + g.L, 4, cudaMemcpyDeviceToHost, s));
        HF_CUDA(cudaStreamSynchronize(s));
        tbuf.alloc(sizeof(unsigned long long) * 8 * size_t(std::max(ntask, 1)), s);
        HF_CUDA(cudaMemsetAsync(tbuf.p, 0, tbuf.bytes, s));
        p.trace = tbuf.as<unsigned long long>();
        p.trace_cap = ntask;
    }
    launch_pass<FWD>(g, p, check_d, V, cx, s, 0);
    if (trace_env) {
        // per task: 8 words (k_flow's trace record) + the task bases per level
        std::vector<unsigned long long> h(size_t(ntask) * 8);
        std::vector<int32_t> tb(size_t(g.L) + 1);
        HF_CUDA(cudaMemcpyAsync(h.data(), p.trace, h.size() * 8, cudaMemcpyDeviceToHost, s));
        HF_CUDA(cudaMemcpyAsync(tb.data(), p.tb, tb.size() * 4, cudaMemcpyDeviceToHost, s));
        HF_CUDA(cudaStreamSynchronize(s));
        std::string fn = std::string(trace_env) + (FWD ? "_fwd_S" : "_bwd_S") + std::to_string(p.S) +
                         ".bin";
        if (FILE *f = fopen(fn.c_str(), "wb")) {
            const int32_t hdr[4] = {ntask, g.L, p.S, int32_t(SC)};
            fwrite(hdr, 4, 4, f);
            fwrite(tb.data(), 4, tb.size(), f);
            fwrite(h.data(), 8, h.size(), f);
            fclose(f);
        }
    }
}

}  // namespace

// level-synchronous passes for wide graphs (wide.cu)
bool wide_choice(const Graph &g, int32_t S);
void lo_delays_prepare(Graph &g);
template <bool FWD>
void wide_pass(Graph &g, const float *d, bool lo_delays, int32_t S, const float *src_val,
               float t_scalar, const float *other, float *out, float *slack, int32_t *wns_ord,
               cudaStream_t st);

// Forward over all levels (device pointers).  d: [m][S].
void forward_device(Graph &g, const float *d, int32_t S, bool check_d, const float *at_src,
                    float *at) {
    if (g.n == 0) return;
    if (wide_choice(g, S)) {
        // the graph's own delays: pre-permuted into level order (contiguous rows)
        const bool lo = S == 1 && d == g.delay.as<float>();
        if (lo) lo_delays_prepare(g);
        prof_record(g, 2);
        wide_pass<true>(g, lo ? g.lo_in_d.as<float>() : d, lo, S, at_src, 0.0f, nullptr, at,
                        nullptr, nullptr, g.stream);
        prof_record(g, 3);
        return;
    }
    FlowParams p{};
    const int V = pick_vec(S, {d, at});
    p.row_ptr = g.lo_in_ptr.as<int32_t>();
    p.nbr = g.lo_in_nbr.as<int32_t>();
    p.eid = g.lo_in_eid.as<int32_t>();
    p.node_of = g.lo_in_node.as<int32_t>();
    p.S = S;
    p.d = d;
    p.src_val = at_src;
    p.out = at;
    run_pass<true>(g, p, check_d, V);
}

// Backward over all levels + slack + wns (ordered ints, decoded into wns_f[S]).
void backward_device(Graph &g, const float *d, int32_t S, const float *t_arr, float t_scalar,
                     const float *at, float *rat, float *slack, float *wns_f) {
    cudaStream_t s = g.stream;
    g.ws_wns.alloc(sizeof(int32_t) * size_t(S), s);
    int32_t *ord = g.ws_wns.as<int32_t>();
    k_fill_i32<<<1, 256, 0, s>>>(ord, 0x7f800000, S);
    HF_CHECK_LAUNCH();
    g.launches += 1;
    if (g.n > 0 && wide_choice(g, S)) {
        const bool lo = S == 1 && d == g.delay.as<float>();
        if (lo) lo_delays_prepare(g);
        prof_record(g, 5);
        wide_pass<false>(g, lo ? g.lo_out_d.as<float>() : d, lo, S, t_arr, t_scalar, at, rat,
                         slack, ord, s);
        prof_record(g, 4);
    } else if (g.n > 0) {
        FlowParams p{};
        const int V = pick_vec(S, {d, at, rat, slack});
        p.row_ptr = g.lo_out_ptr.as<int32_t>();
        p.nbr = g.lo_out_nbr.as<int32_t>();
        p.eid = g.lo_out_eid.as<int32_t>();
        p.node_of = g.lo_out_node.as<int32_t>();
        p.S = S;
        p.d = d;
        p.src_val = t_arr;
        p.t_scalar = t_scalar;
        p.other = at;
        p.out = rat;
        p.slack = slack;
        p.wns_ord = ord;
        run_pass<false>(g, p, false, V);
    }
    if (wns_f) {
        k_ord_to_float<<<1, 256, 0, s>>>(ord, wns_f, S);
        HF_CHECK_LAUNCH();
        g.launches += 1;
    }
}

// Batch: forward then backward (default), or with HF_CONCURRENT=1 both passes at
// once.  The backward recurrence (rat of sinks = T, rat[u] = min fl(rat[v] - d))
// does not read at -- only the slack does -- so both dataflow kernels can be
// resident side by side (each capped at about half the blocks per SM it could hold
// alone) on two streams, the slack and worst slack following in one streaming pass.
// Measured on C4 (S = 64): slower (1.48 ms vs 1.32 ms for the phase), because each
// pass then has half the resident warps and the dataflow needs many warps to keep
// several levels in flight; kept for the record.
// (creating the side stream per graph cost ~70 us of host time per step)
Side &side_of(Graph &g) {
    thread_local Side sides[64];
    Side &x = sides[g.device & 63];
    if (!x.s2) {
        // lowest priority: its bandwidth-bound fills must not hold SM slots the
        // latency-bound set-up kernels on the graph's stream are waiting for
        int lo = 0, hi = 0;
        HF_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        HF_CUDA(cudaStreamCreateWithPriority(&x.s2, cudaStreamNonBlocking,
                                             env_int("HF_SIDE_PRIO", 1) ? lo : 0));
        HF_CUDA(cudaEventCreateWithFlags(&x.fork, cudaEventDisableTiming));
        HF_CUDA(cudaEventCreateWithFlags(&x.join, cudaEventDisableTiming));
    }
    return x;
}

void batch_device(Graph &g, const float *d, int32_t S, bool check_d, const float *at_src,
                  const float *t_arr, float *at, float *rat, float *slack, float *wns_f) {
    cudaStream_t s = g.stream;
    if (g.n == 0 || getenv("HF_TRACE") || env_int("HF_BATCH_PLAIN", 0) || wide_choice(g, S)) {
        // (wide graphs: two level-synchronous passes, no sentinel fills to overlap)
        prof_record(g, 6);
        forward_device(g, d, S, check_d, at_src, at);
        backward_device(g, d, S, t_arr, 0.0f, at, rat, slack, wns_f);
        prof_record(g, 7);
        return;
    }
    if (!env_int("HF_CONCURRENT", 0)) {
        // Forward then backward, with the set-up of both passes overlapped: the
        // sentinel fill of `at` runs on a second stream while this stream builds both
        // task schedules, and the forward kernel NaN-fills each rat row as it writes
        // the at row (so the backward needs no fill of its own).
        Side &sd = side_of(g);
        StageTimes pt("HF_PROP_TIMES", "batch");
        pt.mark("start", s);
        prof_record(g, 6);
        HF_CUDA(cudaEventRecord(sd.fork, s));
        HF_CUDA(cudaStreamWaitEvent(sd.s2, sd.fork, 0));
        const bool prefill = env_int("HF_PREFILL", 0) != 0;
        fill_nan(g, at, size_t(g.n) * S, sd.s2);
        if (!prefill) fill_nan(g, rat, size_t(g.n) * S, sd.s2);
        HF_CUDA(cudaEventRecord(sd.join, sd.s2));
        g.ws_wns.alloc(sizeof(int32_t) * size_t(S), s);
        int32_t *ord = g.ws_wns.as<int32_t>();
        k_fill_i32<<<1, 256, 0, s>>>(ord, 0x7f800000, S);
        HF_CHECK_LAUNCH();
        g.launches += 1;
        FlowParams pf{}, pb{};
        const int V = pick_vec(S, {d, at, rat, slack});
        pf.row_ptr = g.lo_in_ptr.as<int32_t>();
        pf.nbr = g.lo_in_nbr.as<int32_t>();
        pf.eid = g.lo_in_eid.as<int32_t>();
        pf.node_of = g.lo_in_node.as<int32_t>();
        pf.S = S;
        pf.d = d;
        pf.src_val = at_src;
        pf.out = at;
        pf.prefill = prefill ? rat : nullptr;
        pb.row_ptr = g.lo_out_ptr.as<int32_t>();
        pb.nbr = g.lo_out_nbr.as<int32_t>();
        pb.eid = g.lo_out_eid.as<int32_t>();
        pb.node_of = g.lo_out_node.as<int32_t>();
        pb.S = S;
        pb.d = d;
        pb.src_val = t_arr;
        pb.t_scalar = 0.0f;
        pb.other = at;
        pb.out = rat;
        pb.slack = slack;
        pb.wns_ord = ord;
        PassCtx cf, cb;
        prepare_pass<true>(g, pf, V, cf, false);
        prepare_pass<false>(g, pb, V, cb, false);
        pt.mark("build_tasks", s);
        HF_CUDA(cudaStreamWaitEvent(s, sd.join, 0));
        pt.mark("fills", s);
        launch_pass<true>(g, pf, check_d, V, cf, s, 0);
        pt.mark("forward+finalize", s);
        launch_pass<false>(g, pb, false, V, cb, s, 0);
        pt.mark("backward+finalize", s);
        prof_record(g, 7);
        if (wns_f) {
            k_ord_to_float<<<1, 256, 0, s>>>(ord, wns_f, S);
            HF_CHECK_LAUNCH();
            g.launches += 1;
        }
        return;
    }
    g.ws_wns.alloc(sizeof(int32_t) * size_t(S), s);
    int32_t *ord = g.ws_wns.as<int32_t>();
    k_fill_i32<<<1, 256, 0, s>>>(ord, 0x7f800000, S);
    HF_CHECK_LAUNCH();
    g.launches += 1;
    // the two passes run side by side: the backward one cannot rely on the forward's
    // check of the delays, so they are checked first (both kernels skip their work
    // when the check flags a non-finite value)
    k_check_finite<<<grid_for(int64_t(g.m) * S / 4 + 1, 256, g.sms), 256, 0, s>>>(
        d, int64_t(g.m) * S, g.d_err());
    HF_CHECK_LAUNCH();
    g.launches += 1;
    FlowParams pf{}, pb{};
    const int V = pick_vec(S, {d, at, rat, slack});
    pf.row_ptr = g.lo_in_ptr.as<int32_t>();
    pf.nbr = g.lo_in_nbr.as<int32_t>();
    pf.eid = g.lo_in_eid.as<int32_t>();
    pf.node_of = g.lo_in_node.as<int32_t>();
    pf.S = S;
    pf.d = d;
    pf.src_val = at_src;
    pf.out = at;
    pb.row_ptr = g.lo_out_ptr.as<int32_t>();
    pb.nbr = g.lo_out_nbr.as<int32_t>();
    pb.eid = g.lo_out_eid.as<int32_t>();
    pb.node_of = g.lo_out_node.as<int32_t>();
    pb.S = S;
    pb.d = d;
    pb.src_val = t_arr;
    pb.out = rat;
    pb.other = nullptr;   // no slack inside the pass
    PassCtx cf, cb;
    prepare_pass<true>(g, pf, V, cf);
    prepare_pass<false>(g, pb, V, cb);
    // blocks per SM for each kernel when both are resident
    const int of = dispatch<true>(g, pf, V, cf.LPN, s, 0, 1);
    const int ob = dispatch<false>(g, pb, V, cb.LPN, s, 0, 1);
    const int capf = std::max(1, env_int("HF_CAP_F", (of + 1) / 2));
    const int capb = std::max(1, env_int("HF_CAP_B", ob / 2));
    Side &sd = side_of(g);
    prof_record(g, 6);
    HF_CUDA(cudaEventRecord(sd.fork, s));
    HF_CUDA(cudaStreamWaitEvent(sd.s2, sd.fork, 0));
    launch_pass<false>(g, pb, false, V, cb, sd.s2, capb);
    launch_pass<true>(g, pf, check_d, V, cf, s, capf);
    HF_CUDA(cudaEventRecord(sd.join, sd.s2));
    HF_CUDA(cudaStreamWaitEvent(s, sd.join, 0));
    const int lpn = S / V;
    const int grid = grid_for(int64_t(g.n) * lpn, 512, g.sms);
    const size_t sm = sizeof(int32_t) * size_t(S);
    if (sm > 48 * 1024) fail(HF_ERR_INVALID_ARG, "too many scenarios");
#define HF_SLACK(VV)                                                                     \
    do {                                                                                 \
        if (g.early) k_slack_wns<VV, true><<<grid, 512, sm, s>>>(at, rat, slack, g.n, S, ord); \
        else k_slack_wns<VV, false><<<grid, 512, sm, s>>>(at, rat, slack, g.n, S, ord);  \
    } while (0)
    if (V == 4) HF_SLACK(4);
    else if (V == 2) HF_SLACK(2);
    else HF_SLACK(1);
#undef HF_SLACK
    HF_CHECK_LAUNCH();
    g.launches += 1;
    prof_record(g, 7);
    if (wns_f) {
        k_ord_to_float<<<1, 256, 0, s>>>(ord, wns_f, S);
        HF_CHECK_LAUNCH();
        g.launches += 1;
    }
    // cf / cb partial buffers are freed on s, after the join
}

void profile_mark(Graph &g, int idx) { prof_record(g, idx); }

}  // namespace hf
