// wide.cu -- level-synchronous propagation passes for WIDE graphs (many nodes per
// level: C5, 10M nodes in ~30 levels).  SURVEY.md §8(a) a5-a7 (same recurrences as
// propagate.cu: at[v] = max over fan-in of fl(at[u] + d), rat[u] = min over fan-out
// of fl(rat[v] - d), slack / worst slack fused; BASELINE.json:5).
//
// Why a second kernel.  The dataflow kernel (propagate.cu) walks warp tasks one at a
// time per warp: right for deep graphs, where the level-to-level hop is the critical
// path, but on a wide level (330k rows, 640k edges at C5) a warp's ~30 loads in
// flight per task leave the memory system idle (C5 ran at 5% of the HBM roofline).
// Here one persistent cooperative launch sweeps the levels with a grid barrier
// between them (~1.2 us, negligible against a wide level), and every thread owns
// whole units of work with all their loads in flight at once:
//   * a SHORT row (<= LO_SPLIT edges) of the level-ordered CSR x one column vector
//     (V scenarios): up to 8 neighbour gathers + 8 delay loads issued together,
//     combined in registers, stored once;
//   * a SLICE of WIDE_SL edges of a long row (fan-in up to 10^4 at C5): combined in
//     registers, then folded into the row's slot with an ordered-int atomicMax /
//     atomicMin (exact: max / min of floats is order-independent, reading R10).
//     Consumers of a long row read its slot (neighbour id -(first part id + 1),
//     levelize.cu); the slots become the row's value after the pass.
// No NaN sentinel, no task schedule, no fill of the outputs: readiness is the
// barrier.  Reads of values written during the pass bypass L1 (ld.global.cg); the
// barrier is release / acquire at gpu scope.
// Single delay set with the graph's own delays: the delays are pre-permuted into
// level order per direction (lo_*_d), so a row's delays are one contiguous run.
#include <algorithm>
#include <cstdlib>
#include <map>
#include <mutex>
#include <tuple>
#include <cstdio>
#include <string>
#include <vector>

#include "common.cuh"

namespace hf {

namespace {

constexpr int WIDE_THREADS = 512;
constexpr int32_t ORD_NEG_INF = int32_t(0x807fffff);   // f2ord(-inf)
constexpr int32_t ORD_POS_INF = int32_t(0x7f800000);   // f2ord(+inf)

template <int V> struct VecW {
    float x[V];
};

// read-only data: through the non-coherent path
template <int V> __device__ __forceinline__ VecW<V> ldg_v(const float *p) {
    VecW<V> r;
    if constexpr (V == 4) {
        const float4 t = __ldg(reinterpret_cast<const float4 *>(p));
        r.x[0] = t.x; r.x[1] = t.y; r.x[2] = t.z; r.x[3] = t.w;
    } else {
        r.x[0] = __ldg(p);
    }
    return r;
}
// values written earlier in this pass (other SMs): L2, never a stale L1 line
template <int V> __device__ __forceinline__ VecW<V> ldcg_v(const float *p) {
    VecW<V> r;
    if constexpr (V == 4) {
        const float4 t = __ldcg(reinterpret_cast<const float4 *>(p));
        r.x[0] = t.x; r.x[1] = t.y; r.x[2] = t.z; r.x[3] = t.w;
    } else {
        r.x[0] = __ldcg(p);
    }
    return r;
}
template <int V> __device__ __forceinline__ VecW<V> ldcg_ord(const int32_t *p) {
    VecW<V> r;
    if constexpr (V == 4) {
        const int4 t = __ldcg(reinterpret_cast<const int4 *>(p));
        r.x[0] = ord2f(t.x); r.x[1] = ord2f(t.y); r.x[2] = ord2f(t.z); r.x[3] = ord2f(t.w);
    } else {
        r.x[0] = ord2f(__ldcg(p));
    }
    return r;
}
template <int V> __device__ __forceinline__ void st_v(float *p, const VecW<V> &v) {
    if constexpr (V == 4) {
        *reinterpret_cast<float4 *>(p) = make_float4(v.x[0], v.x[1], v.x[2], v.x[3]);
    } else {
        *p = v.x[0];
    }
}

template <bool MX> __device__ __forceinline__ float comb(float a, float b) {
    return MX ? fmaxf(a, b) : fminf(a, b);
}

__device__ __forceinline__ unsigned ld_acq(const unsigned *p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
// grid barrier of a cooperative launch (monotonic counter, target grows per call)
__device__ __forceinline__ void grid_bar(unsigned *ctr, unsigned &target) {
    target += gridDim.x;
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
        while (ld_acq(ctr) < target) __nanosleep(32);
    }
    __syncthreads();
}

struct WideParams {
    const int32_t *level_ptr;   // [L+1]
    const int32_t *lstart;      // [L] first long row of each level
    const int32_t *row_ptr;     // [n+1] level-ordered CSR of this direction
    const int32_t *nbr;         // [m] neighbour id, or -(first part id + 1) if long
    const int32_t *eid;         // [m] delay row of each position, or null: d is level-ordered
    const int32_t *node_of;     // [n]
    const int32_t *q;           // [n+1] first part id of each row (slot index of long rows)
    const int32_t *sfirst;      // [n+1] first slice of each row
    const int2 *slice;          // {row, first edge}
    const int32_t *part_np;     // [np_cap] parts of the long row at its first part id
    const int32_t *part_row;    // [np_cap] that row
    const int32_t *nparts_d;    // exact part-id count
    int32_t L, S;
    const float *d;             // [m][S] by eid (or by position when eid is null)
    const float *src_val;       // forward: at_src [n] or null; backward: t_req [S] or null
    float t_scalar;             // backward: T when t_req is null
    const float *other;         // backward: at (slack), or null
    float *out;                 // at (forward) / rat (backward) [n][S]
    float *slack;               // [n][S] or null
    int32_t *slot;              // [parts][S] ordered ints
    int32_t *wns_ord;           // [S] (backward with other)
    uint32_t *err;
    unsigned *bar;              // zeroed grid-barrier counter
};

template <int V, bool FWD, bool EARLY>
__global__ void __launch_bounds__(WIDE_THREADS) k_wide(WideParams p) {
    constexpr bool MX = FWD != EARLY;   // combine with max (late forward / early backward)
    constexpr int EB = V == 1 ? 8 : 4;  // edges in flight per batch
    extern __shared__ int32_t s_wmin[];
    const int S = p.S;
    const bool do_slack = !FWD && p.other;
    if (do_slack) {
        for (int s = threadIdx.x; s < S; s += blockDim.x) s_wmin[s] = ORD_POS_INF;
    }
    const int T = gridDim.x * blockDim.x;
    const int tid = blockIdx.x * blockDim.x + threadIdx.x;
    unsigned target = 0;
    // slots of the long rows start at the combine's identity
    const int64_t nslot = int64_t(*p.nparts_d) * S;
    for (int64_t i = tid; i < nslot; i += T) p.slot[i] = MX ? ORD_NEG_INF : ORD_POS_INF;
    grid_bar(p.bar, target);

    const int lpn = S / V;               // column vectors per row
    const int upt = T / lpn;             // units per sweep of the grid
    const bool active = tid < upt * lpn;
    const int cv = tid % lpn, u0 = tid / lpn;
    const int64_t col = int64_t(cv) * V;
    bool bad = false;
    float mn[V];
#pragma unroll
    for (int j = 0; j < V; ++j) mn[j] = __int_as_float(ORD_POS_INF);
    const int L = p.L;
    for (int qq = 0; qq < L; ++qq) {
        const int k = FWD ? qq : L - 1 - qq;
        const int ls = __ldg(p.level_ptr + k), le = __ldg(p.level_ptr + k + 1);
        const int lo = __ldg(p.lstart + k);
        const int nshort = lo - ls;
        const int s0 = __ldg(p.sfirst + lo);
        const int nunits = nshort + (__ldg(p.sfirst + le) - s0);
        for (int u = u0; active && u < nunits; u += upt) {
            const bool lng = u >= nshort;
            int row, eb, ee;
            if (!lng) {
                row = ls + u;
                eb = __ldg(p.row_ptr + row);
                ee = __ldg(p.row_ptr + row + 1);
            } else {
                const int2 sd = __ldg(p.slice + s0 + (u - nshort));
                row = sd.x;
                eb = sd.y;
                ee = min(__ldg(p.row_ptr + row + 1), eb + WIDE_SL);
            }
            VecW<V> best;
#pragma unroll
            for (int j = 0; j < V; ++j) best.x[j] = __int_as_float(MX ? 0xff800000 : 0x7f800000);
            for (int e0 = eb; e0 < ee; e0 += EB) {
                int nb[EB];
                int64_t dr[EB];
#pragma unroll
                for (int j = 0; j < EB; ++j) {
                    const int e = e0 + j;
                    nb[j] = 0;
                    dr[j] = 0;
                    if (e < ee) {
                        nb[j] = __ldg(p.nbr + e);
                        dr[j] = p.eid ? __ldg(p.eid + e) : e;
                    }
                }
                VecW<V> a[EB], dv[EB];
#pragma unroll
                for (int j = 0; j < EB; ++j) {
                    if (e0 + j < ee) {
                        dv[j] = ldg_v<V>(p.d + dr[j] * S + col);
                        if (nb[j] >= 0) a[j] = ldcg_v<V>(p.out + int64_t(nb[j]) * S + col);
                        else a[j] = ldcg_ord<V>(p.slot + int64_t(-nb[j] - 1) * S + col);
                    }
                }
#pragma unroll
                for (int j = 0; j < EB; ++j) {
                    if (e0 + j < ee) {
#pragma unroll
                        for (int c = 0; c < V; ++c) {
                            const float dd = sane(dv[j].x[c], bad);
                            const float x = FWD ? __fadd_rn(a[j].x[c], dd) : __fsub_rn(a[j].x[c], dd);
                            best.x[c] = comb<MX>(best.x[c], x);
                        }
                    }
                }
            }
            if (!lng) {
                const int node = __ldg(p.node_of + row);
                if (ee == eb) {   // source (forward) / sink (backward)
#pragma unroll
                    for (int c = 0; c < V; ++c)
                        best.x[c] = FWD ? (p.src_val ? sane(__ldg(p.src_val + node), bad) : 0.0f)
                                        : sane(p.src_val ? __ldg(p.src_val + col + c) : p.t_scalar, bad);
                }
                st_v<V>(p.out + int64_t(node) * S + col, best);
                if (do_slack) {
                    const VecW<V> av = ldg_v<V>(p.other + int64_t(node) * S + col);
                    VecW<V> sl;
#pragma unroll
                    for (int c = 0; c < V; ++c) {
                        sl.x[c] = EARLY ? __fsub_rn(av.x[c], best.x[c]) : __fsub_rn(best.x[c], av.x[c]);
                        mn[c] = fminf(mn[c], sl.x[c]);
                    }
                    if (p.slack) st_v<V>(p.slack + int64_t(node) * S + col, sl);
                }
            } else {
                int32_t *sp = p.slot + int64_t(__ldg(p.q + row)) * S + col;
#pragma unroll
                for (int c = 0; c < V; ++c) {
                    if (MX) atomicMax(sp + c, f2ord(best.x[c]));
                    else atomicMin(sp + c, f2ord(best.x[c]));
                }
            }
        }
        grid_bar(p.bar, target);
    }
    // long rows: the slot is the row's value; slack and worst slack
    const int64_t nparts = *p.nparts_d;
    for (int64_t pp = u0; active && pp < nparts; pp += upt) {
        if (__ldg(p.part_np + pp) == 0) continue;   // not a first part id
        const int node = __ldg(p.node_of + __ldg(p.part_row + pp));
        const VecW<V> v = ldcg_ord<V>(p.slot + pp * S + col);
        st_v<V>(p.out + int64_t(node) * S + col, v);
        if (do_slack) {
            const VecW<V> av = ldg_v<V>(p.other + int64_t(node) * S + col);
            VecW<V> sl;
#pragma unroll
            for (int c = 0; c < V; ++c) {
                sl.x[c] = EARLY ? __fsub_rn(av.x[c], v.x[c]) : __fsub_rn(v.x[c], av.x[c]);
                mn[c] = fminf(mn[c], sl.x[c]);
            }
            if (p.slack) st_v<V>(p.slack + int64_t(node) * S + col, sl);
        }
    }
    if (bad) atomicOr(p.err, ERR_NONFINITE);
    if (do_slack) {
        if (active)
#pragma unroll
            for (int c = 0; c < V; ++c)
                if (mn[c] != __int_as_float(ORD_POS_INF)) atomicMin(s_wmin + col + c, f2ord(mn[c]));
        __syncthreads();
        for (int s = threadIdx.x; s < S; s += blockDim.x)
            if (s_wmin[s] != ORD_POS_INF) atomicMin(p.wns_ord + s, s_wmin[s]);
    }
}

// ---- S = 1: warp-cooperative level-synchronous pass (k_wide1) -------------------
// A warp unit is either 32 consecutive short rows of the level (their edges are one
// contiguous run of the level-ordered CSR) or a chunk of 32 consecutive edges of the
// level's long rows (one contiguous run as well: long rows sit at the end of their
// level).  Edges are processed 32 at a time, one per lane, all loads coalesced; a
// lane finds its row by a shuffle binary search over the row ends held by the
// lanes, and a segmented max / min scan over the lanes combines each row's edges.
// Short rows: the segment ends combine into a per-warp shared row buffer, then lane
// j stores row j.  Long rows: the segment ends fold into the row's slot (ordered-int
// atomic).  The barrier between levels is split: a block arrives as soon as its
// stores are issued, loads the structure of its first unit of the next level (row
// offsets, neighbours, delays: nothing written in the pass) and only then waits,
// so after the barrier a unit is one gather round trip from its result.
constexpr int W1_THREADS = 256;
#ifndef W1_NU_OVR
#define W1_NU_OVR 2
#endif
#ifndef W1_CH_OVR
#define W1_CH_OVR 2
#endif
constexpr int W1_NU = W1_NU_OVR;   // units of a warp per level whose structure is held in registers
constexpr int W1_CH = W1_CH_OVR;   // edge chunks (32 edges) of a unit held in registers

struct Wide1Params {
    const int32_t *level_ptr, *lstart, *row_ptr, *nbr, *eid, *node_of, *q;
    const int32_t *coff, *crow;
    const int32_t *part_np, *part_row, *nparts_d;
    int32_t L;
    const float *d;        // [m] by eid, or level-ordered when eid is null
    const float *src_val;  // forward: at_src [n] / null; backward: t_req [1] / null
    float t_scalar;
    const float *other;    // backward: at (slack) or null
    float *out, *slack;
    int32_t *slot, *wns_ord;
    uint32_t *err;
    unsigned *bar;
    unsigned long long *trace;   // optional (HF_TRACE): per level {barrier passed, stores issued}
};

struct LevelInfo {
    int ls, lo, le, lbase, lend, c0, us, nu;
};

__device__ __forceinline__ LevelInfo level_info(const Wide1Params &p, int k) {
    LevelInfo li;
    li.ls = __ldg(p.level_ptr + k);
    li.le = __ldg(p.level_ptr + k + 1);
    li.lo = __ldg(p.lstart + k);
    li.lbase = __ldg(p.row_ptr + li.lo);
    li.lend = __ldg(p.row_ptr + li.le);
    li.c0 = __ldg(p.coff + k);
    li.us = (li.lo - li.ls + 31) >> 5;
    li.nu = li.us + (__ldg(p.coff + k + 1) - li.c0);
    return li;
}

// The structure of W1_NU units (nothing written during the pass): row offsets and
// nodes (short units) or the chunk's first row, row ends and slot ids (long chunks),
// neighbours and delays / delay ids of the first W1_CH chunks.  Two dependent load
// rounds, every unit's loads of a round in flight together.
struct Units {
    int kind[W1_NU];   // 0: none, 1: short rows, 2: long-row chunk
    int r0[W1_NU], base[W1_NU], ne[W1_NU];
    int pj[W1_NU], qj[W1_NU], node[W1_NU];   // lane j: short: start / end / node of row r0+j;
                                             // long: slot / end of row r0+j
    int nb[W1_NU][W1_CH], dx[W1_CH][W1_NU];
};

__device__ __forceinline__ void load_units(const Wide1Params &p, const LevelInfo &li, int u0,
                                           int ustep, Units &U) {
    const int lane = threadIdx.x & 31;
    // round 1: row offsets / nodes of short units; chunk row + edges of long units
#pragma unroll
    for (int i = 0; i < W1_NU; ++i) {
        const int u = u0 + i * ustep;
        U.kind[i] = u >= li.nu ? 0 : (u < li.us ? 1 : 2);
        U.pj[i] = U.qj[i] = INT32_MAX;
        U.node[i] = 0;
        U.ne[i] = 0;
#pragma unroll
        for (int c = 0; c < W1_CH; ++c) U.nb[i][c] = U.dx[c][i] = 0;
        if (U.kind[i] == 1) {
            U.r0[i] = li.ls + (u << 5);
            const int r = U.r0[i] + lane;
            if (r < li.lo) {
                U.pj[i] = __ldg(p.row_ptr + r);
                U.qj[i] = __ldg(p.row_ptr + r + 1);
                U.node[i] = __ldg(p.node_of + r);
            }
        } else if (U.kind[i] == 2) {
            const int c = u - li.us;
            U.base[i] = li.lbase + (c << 5);
            U.ne[i] = min(32, li.lend - U.base[i]);
            U.r0[i] = __ldg(p.crow + li.c0 + c);
            if (lane < U.ne[i]) {
                const int e = U.base[i] + lane;
                U.nb[i][0] = __ldg(p.nbr + e);
                U.dx[0][i] = p.eid ? __ldg(p.eid + e) : __float_as_int(__ldg(p.d + e));
            }
        }
    }
    // round 2: edges of short units; row ends and slots of long chunks
#pragma unroll
    for (int i = 0; i < W1_NU; ++i) {
        if (U.kind[i] == 1) {
            const int nrows = min(32, li.lo - U.r0[i]);
            U.base[i] = __shfl_sync(0xffffffffu, U.pj[i], 0);
            U.ne[i] = __shfl_sync(0xffffffffu, U.qj[i], nrows - 1) - U.base[i];
#pragma unroll
            for (int c = 0; c < W1_CH; ++c) {
                if ((c << 5) + lane < U.ne[i]) {
                    const int e = U.base[i] + (c << 5) + lane;
                    U.nb[i][c] = __ldg(p.nbr + e);
                    U.dx[c][i] = p.eid ? __ldg(p.eid + e) : __float_as_int(__ldg(p.d + e));
                }
            }
        } else if (U.kind[i] == 2) {
            const int r = U.r0[i] + lane;
            if (r < li.le) {
                U.qj[i] = __ldg(p.row_ptr + r + 1);
                U.pj[i] = __ldg(p.q + r);
            }
        }
    }
}

// one chunk of 32 edges of a unit: x = fl(a[u] +/- d) per lane, rows by a shuffle
// binary search over the lanes' row ends, a segmented scan combines each row's
// edges; the segment ends go to the warp's row buffer (short) or the row's slot
template <bool FWD, bool EARLY>
__device__ __forceinline__ void chunk_combine(const Wide1Params &p, int kind, int e, bool valid,
                                              float x, int qj, int pj, float *s_val) {
    constexpr bool MX = FWD != EARLY;
    const int lane = threadIdx.x & 31;
    int r = 0;
#pragma unroll
    for (int step = 16; step >= 1; step >>= 1) {
        const int t = __shfl_sync(0xffffffffu, qj, r + step - 1);
        if (t <= e) r += step;
    }
    const int rr = valid ? r : 32 + lane;
    const int prv = __shfl_up_sync(0xffffffffu, rr, 1);
    const int nxt = __shfl_down_sync(0xffffffffu, rr, 1);
    const unsigned smask = __ballot_sync(0xffffffffu, lane == 0 || prv != rr);
    const int sstart = 31 - __clz(smask & ((2u << lane) - 1u));
    float v = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const float y = __shfl_up_sync(0xffffffffu, v, o);
        if (lane - o >= sstart) v = comb<MX>(v, y);
    }
    const bool seg_end = valid && (lane == 31 || nxt != rr);
    const int slot_id = __shfl_sync(0xffffffffu, pj, r & 31);
    if (seg_end) {
        if (kind == 1) {
            s_val[r] = comb<MX>(s_val[r], v);
        } else {
            if (MX) atomicMax(p.slot + slot_id, f2ord(v));
            else atomicMin(p.slot + slot_id, f2ord(v));
        }
    }
}

template <bool FWD>
__device__ __forceinline__ float relax1(float a, float d) {
    return FWD ? __fadd_rn(a, d) : __fsub_rn(a, d);
}

// gathers of every unit at once (one round trip), then per unit: combine, store
template <bool FWD, bool EARLY>
__device__ __forceinline__ void finish_units(const Wide1Params &p, const Units &U, float *s_val,
                                             bool &bad, float &mn) {
    constexpr bool MX = FWD != EARLY;
    const int lane = threadIdx.x & 31;
    const float ident = __int_as_float(MX ? 0xff800000 : 0x7f800000);
    const bool do_slack = !FWD && p.other;
    float a[W1_NU][W1_CH], dd[W1_NU][W1_CH], at_node[W1_NU];
#pragma unroll
    for (int i = 0; i < W1_NU; ++i) {
        at_node[i] = 0.0f;
        if (do_slack && U.kind[i] == 1 && U.qj[i] != INT32_MAX) at_node[i] = __ldg(p.other + U.node[i]);
#pragma unroll
        for (int c = 0; c < W1_CH; ++c) {
            a[i][c] = ident;
            dd[i][c] = 0.0f;
            if (U.kind[i] && (c << 5) + lane < U.ne[i]) {
                const int nb = U.nb[i][c];
                a[i][c] = nb >= 0 ? __ldcg(p.out + nb) : ord2f(__ldcg(p.slot + (-nb - 1)));
                dd[i][c] = p.eid ? __ldg(p.d + U.dx[c][i]) : __int_as_float(U.dx[c][i]);
            }
        }
    }
#pragma unroll
    for (int i = 0; i < W1_NU; ++i) {
        if (!U.kind[i]) continue;
        if (U.kind[i] == 1) s_val[lane] = ident;
        __syncwarp();
#pragma unroll
        for (int c = 0; c < W1_CH; ++c) {
            if ((c << 5) < U.ne[i]) {
                const int k = (c << 5) + lane;
                const bool valid = k < U.ne[i];
                const float x = valid ? relax1<FWD>(a[i][c], sane(dd[i][c], bad)) : ident;
                chunk_combine<FWD, EARLY>(p, U.kind[i], U.base[i] + k, valid, x, U.qj[i], U.pj[i],
                                          s_val);
                __syncwarp();
            }
        }
        // short units with more than W1_CH chunks (rows of up to 8 edges): the rest
        for (int c = W1_CH; (c << 5) < U.ne[i]; ++c) {
            const int k = (c << 5) + lane;
            const bool valid = k < U.ne[i];
            float x = ident;
            if (valid) {
                const int e = U.base[i] + k;
                const int nb = __ldg(p.nbr + e);
                const float av = nb >= 0 ? __ldcg(p.out + nb) : ord2f(__ldcg(p.slot + (-nb - 1)));
                const float dv = p.eid ? __ldg(p.d + __ldg(p.eid + e)) : __ldg(p.d + e);
                x = relax1<FWD>(av, sane(dv, bad));
            }
            chunk_combine<FWD, EARLY>(p, U.kind[i], U.base[i] + k, valid, x, U.qj[i], U.pj[i],
                                      s_val);
            __syncwarp();
        }
        if (U.kind[i] == 1 && U.qj[i] != INT32_MAX) {
            float best;
            if (U.qj[i] > U.pj[i]) {
                best = s_val[lane];
            } else {   // source (forward) / sink (backward)
                best = FWD ? (p.src_val ? sane(__ldg(p.src_val + U.node[i]), bad) : 0.0f)
                           : sane(p.src_val ? __ldg(p.src_val) : p.t_scalar, bad);
            }
            p.out[U.node[i]] = best;
            if (do_slack) {
                const float sl = EARLY ? __fsub_rn(at_node[i], best) : __fsub_rn(best, at_node[i]);
                mn = fminf(mn, sl);
                if (p.slack) p.slack[U.node[i]] = sl;
            }
        }
        __syncwarp();
    }
}

__device__ __forceinline__ unsigned long long wide_gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

template <bool FWD, bool EARLY>
__global__ void __launch_bounds__(W1_THREADS) k_wide1(Wide1Params p) {
    constexpr bool MX = FWD != EARLY;
    __shared__ float s_rows[W1_THREADS / 32][32];
    __shared__ int32_t s_wmin;
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    float *s_val = s_rows[wib];
    if (threadIdx.x == 0) s_wmin = ORD_POS_INF;
    const int tid = blockIdx.x * blockDim.x + threadIdx.x;
    const int T = gridDim.x * blockDim.x;
    const int W = T >> 5;
    const int w = wib * gridDim.x + blockIdx.x;   // consecutive units on different SMs
    unsigned target = 0;
    const int64_t nslot = *p.nparts_d;
    for (int64_t i = tid; i < nslot; i += T) p.slot[i] = MX ? ORD_NEG_INF : ORD_POS_INF;
    const int L = p.L;
    LevelInfo li = level_info(p, FWD ? 0 : L - 1);
    Units U;
    load_units(p, li, w, W, U);
    grid_bar(p.bar, target);
    bool bad = false;
    float mn = __int_as_float(ORD_POS_INF);
    for (int qq = 0; qq < L; ++qq) {
        // round 0 was loaded before the barrier; a warp with more than W1_NU units in
        // this level loads the further rounds here
        if (p.trace && threadIdx.x == 0) p.trace[(2 * qq) * gridDim.x + blockIdx.x] = wide_gtimer();
        for (int r0 = 0; w + r0 * W1_NU * W < li.nu; ++r0) {
            if (r0) load_units(p, li, w + r0 * W1_NU * W, W, U);
            finish_units<FWD, EARLY>(p, U, s_val, bad, mn);
        }
        if (p.trace) {
            __syncthreads();
            if (threadIdx.x == 0) p.trace[(2 * qq + 1) * gridDim.x + blockIdx.x] = wide_gtimer();
        }
        if (qq + 1 == L) break;
        // split barrier: arrive, load the next level's first round, wait
        target += gridDim.x;
        __syncthreads();
        if (threadIdx.x == 0)
            asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(p.bar) : "memory");
        li = level_info(p, FWD ? qq + 1 : L - 2 - qq);
        load_units(p, li, w, W, U);
        if (threadIdx.x == 0)
            while (ld_acq(p.bar) < target) __nanosleep(32);
        __syncthreads();
    }
    grid_bar(p.bar, target);
    // long rows: the slot is the row's value; slack and worst slack
    const bool do_slack = !FWD && p.other;
    const int64_t nparts = *p.nparts_d;
    for (int64_t pp = tid; pp < nparts; pp += T) {
        if (__ldg(p.part_np + pp) == 0) continue;   // not a first part id
        const int node = __ldg(p.node_of + __ldg(p.part_row + pp));
        const float v = ord2f(__ldcg(p.slot + pp));
        p.out[node] = v;
        if (do_slack) {
            const float a = __ldg(p.other + node);
            const float sl = EARLY ? __fsub_rn(a, v) : __fsub_rn(v, a);
            mn = fminf(mn, sl);
            if (p.slack) p.slack[node] = sl;
        }
    }
    if (bad) atomicOr(p.err, ERR_NONFINITE);
    if (do_slack) {
        // warp minimum, then one shared and one global atomic per block
#pragma unroll
        for (int o = 16; o; o >>= 1) mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
        __syncthreads();
        if (lane == 0 && mn != __int_as_float(ORD_POS_INF)) atomicMin(&s_wmin, f2ord(mn));
        __syncthreads();
        if (threadIdx.x == 0 && s_wmin != ORD_POS_INF) atomicMin(p.wns_ord, s_wmin);
    }
}

// chunk tables of the long rows (k_wide1): per level the number of 32-edge chunks
// of its long-row run, exclusive scan in one block (levels ascending)
__global__ void __launch_bounds__(1024) k_w1_coff(const int32_t *__restrict__ level_ptr,
                                                  const int32_t *__restrict__ lstart,
                                                  const int32_t *__restrict__ row_ptr, int32_t L,
                                                  int32_t *__restrict__ coff) {
    __shared__ int warp_s[32];
    __shared__ int carry;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int k0 = 0; k0 < L; k0 += blockDim.x) {
        const int k = k0 + threadIdx.x;
        int v = 0;
        if (k < L) v = (row_ptr[level_ptr[k + 1]] - row_ptr[lstart[k]] + 31) >> 5;
        int x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) warp_s[wid] = x;
        __syncthreads();
        if (wid == 0) {
            int sx = lane < nw ? warp_s[lane] : 0;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, sx, o);
                if (lane >= o) sx += y;
            }
            if (lane < nw) warp_s[lane] = sx;
        }
        __syncthreads();
        if (k < L) coff[k] = carry + (wid ? warp_s[wid - 1] : 0) + x - v;
        __syncthreads();
        if (threadIdx.x == 0) carry += warp_s[nw - 1];
        __syncthreads();
    }
    if (threadIdx.x == 0) coff[L] = carry;
}
// crow[coff[k] + c] = the long row of level k holding the level's long-run edge 32c
__global__ void k_w1_crow(const int32_t *__restrict__ row_ptr, const int32_t *__restrict__ node_of,
                          const int32_t *__restrict__ level, const int32_t *__restrict__ lstart,
                          const int32_t *__restrict__ coff, int32_t n, int32_t *__restrict__ crow) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x) {
        const int k = __ldg(level + __ldg(node_of + i));
        const int lo = __ldg(lstart + k);
        if (i < lo) continue;
        const int base = row_ptr[lo];
        const int b = row_ptr[i] - base, e = row_ptr[i + 1] - base;
        for (int c = (b + 31) >> 5; (c << 5) < e; ++c) crow[coff[k] + c] = int(i);
    }
}

// slices of the long rows: count per row, then {row, first edge} per slice
__global__ void k_wide_count(const int32_t *__restrict__ row_ptr, const int32_t *__restrict__ node_of,
                             const int32_t *__restrict__ level, const int32_t *__restrict__ lstart,
                             int32_t n, int32_t *__restrict__ cnt) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i <= n;
         i += int64_t(gridDim.x) * blockDim.x) {
        int c = 0;
        if (i < n && i >= __ldg(lstart + __ldg(level + __ldg(node_of + i))))
            c = (row_ptr[i + 1] - row_ptr[i] + WIDE_SL - 1) / WIDE_SL;
        cnt[i] = c;
    }
}
__global__ void k_wide_slices(const int32_t *__restrict__ row_ptr, const int32_t *__restrict__ sfirst,
                              int32_t n, int2 *__restrict__ slice) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x) {
        const int f = sfirst[i], c = sfirst[i + 1] - f;
        const int rb = row_ptr[i];
        for (int t = 0; t < c; ++t) slice[f + t] = make_int2(int(i), rb + t * WIDE_SL);
    }
}
// the graph's delays in level order of one direction
__global__ void k_gather_delay(const float *__restrict__ delay, const int32_t *__restrict__ eid,
                               int32_t m, float *__restrict__ out) {
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < m;
         e += int64_t(gridDim.x) * blockDim.x)
        out[e] = delay[eid[e]];
}

int env_int_w(const char *name, int dflt) {
    const char *e = getenv(name);
    return e ? atoi(e) : dflt;
}

template <int V, bool FWD, bool EARLY>
void launch_wide(Graph &g, WideParams &p, cudaStream_t st) {
    auto kern = k_wide<V, FWD, EARLY>;
    const size_t smem = sizeof(int32_t) * size_t(p.S);
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
        HF_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, WIDE_THREADS, smem));
        std::lock_guard<std::mutex> lk(mu);
        cache[key] = per_sm;
    }
    ensure_dyn_smem((const void *)kern, g.device, smem);
    if (per_sm < 1) fail(HF_ERR_CUDA, "wide propagation kernel does not fit on an SM");
    const int cap = env_int_w("HF_WIDE_CTAS_PER_SM", 0);
    if (cap > 0) per_sm = std::min(per_sm, cap);
    void *args[] = {&p};
    HF_CUDA(cudaLaunchCooperativeKernel((const void *)kern, g.sms * per_sm, WIDE_THREADS, args, smem,
                                        st));
    g.launches += 1;
}

template <bool FWD, bool EARLY>
int w1_occupancy(const Graph &g) {
    auto kern = k_wide1<FWD, EARLY>;
    static std::map<std::pair<const void *, int>, int> cache;
    static std::mutex mu;
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find({(const void *)kern, g.device});
    if (it != cache.end()) return it->second;
    int per_sm = 0;
    HF_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, W1_THREADS, 0));
    cache[{(const void *)kern, g.device}] = per_sm;
    return per_sm;
}
template <bool FWD, bool EARLY>
int w1_blocks(const Graph &g) {
    int per_sm = w1_occupancy<FWD, EARLY>(g);
    const int cap = env_int_w("HF_WIDE_CTAS_PER_SM", 0);
    if (cap > 0) per_sm = std::min(per_sm, cap);
    return g.sms * per_sm;
}

template <bool FWD, bool EARLY>
void launch_w1(Graph &g, Wide1Params &p, cudaStream_t st) {
    auto kern = k_wide1<FWD, EARLY>;
    const int nblk = w1_blocks<FWD, EARLY>(g);
    if (nblk < 1) fail(HF_ERR_CUDA, "wide propagation kernel does not fit on an SM");
    void *args[] = {&p};
    HF_CUDA(cudaLaunchCooperativeKernel((const void *)kern, nblk, W1_THREADS, args, 0, st));
    g.launches += 1;
}

// ---- S = 1: row ranges with shared-memory row accumulators (k_wide2) ------------
// Each level of the level-ordered CSR is cut into RANGES of consecutive rows of
// weight (rows + edges) <= W2_TW = W2_R * W2_THREADS, so a range holds <= W2_TW rows
// and one contiguous edge run (a hub row of any fan-in is one range).  A CTA (1024
// threads, one per SM) takes ranges j = blockIdx.x, += gridDim.x of the level, each
// in two dependent load rounds:
//   round 1: a range descriptor {first row, first edge} (prefetched one range ahead,
//            and across the grid barrier for the next level's first range), then per
//            thread its <= W2_R rows' nodes and <= W2_U edges' {neighbour, row} and
//            delays -- all coalesced, all in flight together;
//   round 2: the gathers a[neighbour] and, per row, at_src (sources) or at (slack).
// Then x = fl(a +/- d), a segmented max / min over the warp's 32 consecutive edges
// (rows are contiguous), segment ends fold into the row's shared accumulator with an
// ordered-int shared atomic (exact: max / min are order-independent, R10), and every
// thread stores its own rows (sources / sinks: at_src / T; backward the slack and
// the worst-slack minimum).  A thread initialises and reads only its own rows'
// accumulators, so two block barriers per range suffice.  Level-synchronous (grid
// barrier between levels): no sentinel, no fill, no task schedule; a row is never
// split between CTAs, so long rows need no parts or slots.
// MEASURED AND REJECTED as the default (C5, S = 1, one B200): forward 0.50 / backward
// 0.47 ms against k_wide1's 0.37 / 0.40 ms; 512- and 256-thread CTAs (2 and 4 per
// SM) and 16k / 8k / 4k-weight ranges were no better (profiles/round2_c5_wide.txt).
// Kept behind HF_WIDE2=1 and parity-tested (tests/test_gpu_wide.py).
#ifndef W2_THREADS_OVR
#define W2_THREADS_OVR 1024
#endif
constexpr int W2_THREADS = W2_THREADS_OVR;
constexpr int W2_R = 4;
constexpr int W2_U = 4;
constexpr int W2_TW = W2_R * W2_THREADS;

struct Wide2Params {
    const int32_t *node;      // [n] node of each row, ~node (negative) for a row with no edges
    const int2 *nbr_row;      // [m] {plain neighbour node id, row of the edge}
    const int32_t *eid;       // [m] delay index of each position, or null: d is level-ordered
    const int32_t *roff;      // [L+1] first descriptor of each level
    const int2 *rdesc;        // [roff[L]] {first row, first edge} per range + the level end
    int32_t L;
    const float *d;
    const float *src_val;     // forward: at_src [n] or null; backward: t_req [1] or null
    float t_scalar;
    const float *other;       // backward: at (slack) or null
    float *out, *slack;
    int32_t *wns_ord;
    uint32_t *err;
    unsigned *bar;
    unsigned long long *trace;   // optional: per level and block {start, ranges done}
};

template <bool FWD, bool EARLY>
__global__ void __launch_bounds__(W2_THREADS, 1024 / W2_THREADS) k_wide2(Wide2Params p) {
    constexpr bool MX = FWD != EARLY;
    constexpr int32_t IDENT_ORD = MX ? ORD_NEG_INF : ORD_POS_INF;
    constexpr int B = W2_THREADS;
    __shared__ int32_t s_acc[W2_TW];   // row accumulators (ordered ints)
    __shared__ int32_t s_wmin;
    const int tid = threadIdx.x, lane = tid & 31;
    const float ident = __int_as_float(MX ? 0xff800000 : 0x7f800000);
    const bool do_slack = !FWD && p.other;
    const float tb = FWD ? 0.0f : (p.src_val ? __ldg(p.src_val) : p.t_scalar);
    if (tid == 0) s_wmin = ORD_POS_INF;
    unsigned target = 0;
    bool bad = false;
    float mn = __int_as_float(ORD_POS_INF);
    // descriptors of this block's first range of the first level
    int k = FWD ? 0 : p.L - 1;
    int r0 = __ldg(p.roff + k), nr = __ldg(p.roff + k + 1) - r0 - 1;
    int2 lo = make_int2(0, 0), hi = make_int2(0, 0);
    if (int(blockIdx.x) < nr) {
        lo = __ldg(p.rdesc + r0 + blockIdx.x);
        hi = __ldg(p.rdesc + r0 + blockIdx.x + 1);
    }
    for (int qq = 0; qq < p.L; ++qq) {
        if (p.trace && tid == 0) p.trace[(2 * qq) * gridDim.x + blockIdx.x] = wide_gtimer();
        for (int j = blockIdx.x; j < nr; j += gridDim.x) {
            const int ra = lo.x, ea = lo.y, rb = hi.x, eb = hi.y;
            // next range's descriptor (same level), one range ahead
            if (j + int(gridDim.x) < nr) {
                lo = __ldg(p.rdesc + r0 + j + gridDim.x);
                hi = __ldg(p.rdesc + r0 + j + gridDim.x + 1);
            }
            if (ra == rb) continue;   // block-uniform
            // ---- round 1: rows' nodes, edges' {neighbour, row} and delays
            int nd[W2_R];
#pragma unroll
            for (int u = 0; u < W2_R; ++u) {
                const int r = ra + u * B + tid;
                nd[u] = r < rb ? __ldg(p.node + r) : INT32_MIN;
            }
            int2 nr_[W2_U];
            float dv[W2_U];
#pragma unroll
            for (int u = 0; u < W2_U; ++u) {
                const int e = ea + u * B + tid;
                nr_[u] = make_int2(0, -1 - lane);   // unique negative key: never stored
                dv[u] = 0.0f;
                if (e < eb) {
                    nr_[u] = __ldg(p.nbr_row + e);
                    dv[u] = p.eid ? __ldg(p.d + __ldg(p.eid + e)) : __ldg(p.d + e);
                }
            }
#pragma unroll
            for (int u = 0; u < W2_R; ++u) s_acc[u * B + tid] = IDENT_ORD;   // own rows
            __syncthreads();   // every accumulator initialised before any atomic
            // ---- round 2: gathers; at_src of sources (forward) / at for the slack
            float av[W2_U], aux[W2_R];
#pragma unroll
            for (int u = 0; u < W2_U; ++u) av[u] = nr_[u].y >= 0 ? __ldcg(p.out + nr_[u].x) : ident;
#pragma unroll
            for (int u = 0; u < W2_R; ++u) {
                const int node = nd[u] >= 0 ? nd[u] : ~nd[u];
                aux[u] = 0.0f;
                if (nd[u] != INT32_MIN) {
                    if (FWD && nd[u] < 0 && p.src_val) aux[u] = __ldg(p.src_val + node);
                    if (do_slack) aux[u] = __ldg(p.other + node);
                }
            }
            for (int e0 = ea;;) {
#pragma unroll
                for (int u = 0; u < W2_U; ++u) {
                    if (e0 + u * B >= eb) break;   // block-uniform
                    const int key = nr_[u].y;
                    const bool valid = key >= 0;
                    float v = valid ? relax1<FWD>(av[u], sane(dv[u], bad)) : ident;
                    // segmented combine over the warp's consecutive edges
                    const int prv = __shfl_up_sync(0xffffffffu, key, 1);
                    const int nxt = __shfl_down_sync(0xffffffffu, key, 1);
                    const unsigned smask = __ballot_sync(0xffffffffu, lane == 0 || prv != key);
                    const int sstart = 31 - __clz(smask & ((2u << lane) - 1u));
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const float y = __shfl_up_sync(0xffffffffu, v, o);
                        if (lane - o >= sstart) v = comb<MX>(v, y);
                    }
                    if (valid && (lane == 31 || nxt != key)) {
                        if (MX) atomicMax(s_acc + (key - ra), f2ord(v));
                        else atomicMin(s_acc + (key - ra), f2ord(v));
                    }
                }
                e0 += W2_U * B;
                if (e0 >= eb) break;   // block-uniform
                // a range with more edges than one sweep (one row of fan-in > W2_TW)
#pragma unroll
                for (int u = 0; u < W2_U; ++u) {
                    const int e = e0 + u * B + tid;
                    nr_[u] = make_int2(0, -1 - lane);
                    dv[u] = 0.0f;
                    if (e < eb) {
                        nr_[u] = __ldg(p.nbr_row + e);
                        dv[u] = p.eid ? __ldg(p.d + __ldg(p.eid + e)) : __ldg(p.d + e);
                    }
                }
#pragma unroll
                for (int u = 0; u < W2_U; ++u) av[u] = nr_[u].y >= 0 ? __ldcg(p.out + nr_[u].x) : ident;
            }
            __syncthreads();   // all atomics done
            // ---- this thread's rows
#pragma unroll
            for (int u = 0; u < W2_R; ++u) {
                if (nd[u] == INT32_MIN) continue;
                const bool empty = nd[u] < 0;
                const int node = empty ? ~nd[u] : nd[u];
                // source (forward) / sink (backward): at_src / T
                const float best = !empty ? ord2f(s_acc[u * B + tid]) : sane(FWD ? aux[u] : tb, bad);
                p.out[node] = best;
                if (do_slack) {
                    const float sl = EARLY ? __fsub_rn(aux[u], best) : __fsub_rn(best, aux[u]);
                    mn = fminf(mn, sl);
                    if (p.slack) p.slack[node] = sl;
                }
            }
        }
        if (p.trace) {
            __syncthreads();
            if (tid == 0) p.trace[(2 * qq + 1) * gridDim.x + blockIdx.x] = wide_gtimer();
        }
        if (qq + 1 == p.L) break;
        // split grid barrier: arrive, load the next level's first descriptor, wait
        target += gridDim.x;
        __syncthreads();
        if (tid == 0) asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(p.bar) : "memory");
        k = FWD ? qq + 1 : p.L - 2 - qq;
        r0 = __ldg(p.roff + k);
        nr = __ldg(p.roff + k + 1) - r0 - 1;
        if (int(blockIdx.x) < nr) {
            lo = __ldg(p.rdesc + r0 + blockIdx.x);
            hi = __ldg(p.rdesc + r0 + blockIdx.x + 1);
        }
        if (tid == 0)
            while (ld_acq(p.bar) < target) __nanosleep(32);
        __syncthreads();
    }
    if (bad) atomicOr(p.err, ERR_NONFINITE);
    if (do_slack) {
#pragma unroll
        for (int o = 16; o; o >>= 1) mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
        __syncthreads();
        if (lane == 0 && mn != __int_as_float(ORD_POS_INF)) atomicMin(&s_wmin, f2ord(mn));
        __syncthreads();
        if (tid == 0 && s_wmin != ORD_POS_INF) atomicMin(p.wns_ord, s_wmin);
    }
}

// {plain neighbour id, row} per level-ordered edge (a long neighbour's -(first part
// id + 1) decoded to its node), and per row its node, ~node for a row with no edges
__global__ void k_w2_edges(const int32_t *__restrict__ nbr, const int32_t *__restrict__ part_row,
                           const int32_t *__restrict__ node_of, const int32_t *__restrict__ erow,
                           int32_t m, int2 *__restrict__ out) {
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < m;
         e += int64_t(gridDim.x) * blockDim.x) {
        const int u = nbr[e];
        out[e] = make_int2(u >= 0 ? u : node_of[part_row[-u - 1]], erow[e]);
    }
}
__global__ void k_w2_nodes(const int32_t *__restrict__ row_ptr, const int32_t *__restrict__ node_of,
                           int32_t n, int32_t *__restrict__ out) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x)
        out[i] = row_ptr[i + 1] == row_ptr[i] ? ~node_of[i] : node_of[i];
}
// per level: ranges = floor(P(last row) / W2_TW) + 1 (P = weight before a row inside its
// level), entries = ranges + 1; roff = exclusive scan of the entries (one block)
__global__ void __launch_bounds__(1024) k_w2_roff(const int32_t *__restrict__ level_ptr,
                                                  const int32_t *__restrict__ row_ptr, int32_t L,
                                                  int32_t *__restrict__ roff) {
    __shared__ int warp_s[32];
    __shared__ int carry;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int k0 = 0; k0 < L; k0 += blockDim.x) {
        const int k = k0 + threadIdx.x;
        int v = 0;
        if (k < L) {
            const int ls = level_ptr[k], le = level_ptr[k + 1];
            const long long P = (long long)(row_ptr[le - 1] - row_ptr[ls]) + (le - 1 - ls);
            v = int(P / W2_TW) + 2;
        }
        int x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) warp_s[wid] = x;
        __syncthreads();
        if (wid == 0) {
            int sx = lane < nw ? warp_s[lane] : 0;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, sx, o);
                if (lane >= o) sx += y;
            }
            if (lane < nw) warp_s[lane] = sx;
        }
        __syncthreads();
        if (k < L) roff[k] = carry + (wid ? warp_s[wid - 1] : 0) + x - v;
        __syncthreads();
        if (threadIdx.x == 0) carry += warp_s[nw - 1];
        __syncthreads();
    }
    if (threadIdx.x == 0) roff[L] = carry;
}
// range descriptors {first row, first edge}: row i starts every range j with
// P(i-1) < j * W2_TW <= P(i) (range 0 at the level's first row); the level's last row
// also writes the end entry {level end, its edge offset}
__global__ void k_w2_rdesc(const int32_t *__restrict__ row_ptr, const int32_t *__restrict__ node_of,
                           const int32_t *__restrict__ level, const int32_t *__restrict__ level_ptr,
                           const int32_t *__restrict__ roff, int32_t n, int2 *__restrict__ rdesc) {
    for (int64_t ii = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; ii < n;
         ii += int64_t(gridDim.x) * blockDim.x) {
        const int i = int(ii);
        const int k = level[node_of[i]];
        const int ls = level_ptr[k], le = level_ptr[k + 1];
        const int base = roff[k];
        const long long P = (long long)(row_ptr[i] - row_ptr[ls]) + (i - ls);
        const int j = int(P / W2_TW);
        if (i == ls) {
            rdesc[base] = make_int2(ls, row_ptr[ls]);
        } else {
            const long long Pp = (long long)(row_ptr[i - 1] - row_ptr[ls]) + (i - 1 - ls);
            for (int jj = int(Pp / W2_TW) + 1; jj <= j; ++jj) rdesc[base + jj] = make_int2(i, row_ptr[i]);
        }
        if (i == le - 1) rdesc[base + j + 1] = make_int2(le, row_ptr[le]);
    }
}

template <bool FWD, bool EARLY>
int w2_blocks(const Graph &g) {
    auto kern = k_wide2<FWD, EARLY>;
    static std::map<std::pair<const void *, int>, int> cache;
    static std::mutex mu;
    int per_sm = 0;
    {
        std::lock_guard<std::mutex> lk(mu);
        auto it = cache.find({(const void *)kern, g.device});
        if (it != cache.end()) per_sm = it->second;
    }
    if (!per_sm) {
        HF_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, W2_THREADS, 0));
        std::lock_guard<std::mutex> lk(mu);
        cache[{(const void *)kern, g.device}] = per_sm;
    }
    const int cap = env_int_w("HF_WIDE_CTAS_PER_SM", 0);
    if (cap > 0) per_sm = std::min(per_sm, cap);
    return g.sms * per_sm;
}

// ---- S = 1: edge units, ordered-int row accumulation in place (k_wide3) ----------
// The output array holds ORDERED INTS during the pass (f2ord: order-preserving for
// every non-NaN float), initialised to the combine's identity, or to at_src / T for
// the rows without edges.  A level of the level-ordered CSR is one contiguous edge
// run [row_ptr[level start], row_ptr[level end]); warp units are 32 consecutive
// edges of it -- no row structure is needed, every address is arithmetic: per edge
// one {plain neighbour, destination node} int2 and the delay (coalesced), then the
// gather out[neighbour] (an ordered int: ord2f).  x = fl(a +/- d); a segmented max /
// min over the lanes (a row's edges are consecutive) leaves one value per row piece:
// a row wholly inside the unit is stored, a row that continues into a neighbouring
// unit is folded in with an ordered-int atomic max / min (exact: R10).  W3_U units
// per warp are in flight together.  Grid barrier between levels, split: a block
// arrives, loads its first units of the next level, then waits.  After the pass one
// streaming kernel turns the ordered ints back into floats in place (backward: the
// slack and the worst slack fused).
constexpr int W3_THREADS = 256;
#ifndef W3_U_OVR
#define W3_U_OVR 8
#endif
constexpr int W3_U = W3_U_OVR;

struct Wide3Params {
    const int32_t *level_ptr;   // [L+1]
    const int32_t *row_ptr;     // [n+1] level-ordered CSR of this direction
    const int2 *edge;           // [m] {plain neighbour node, destination node}
    const int32_t *eid;         // [m] delay index of each position, or null: d level-ordered
    const float *d;
    int32_t L;
    int32_t *out;               // [n] ordered ints during the pass
    uint32_t *err;
    unsigned *bar;
};

template <bool FWD, bool EARLY>
__global__ void __launch_bounds__(W3_THREADS) k_wide3(Wide3Params p) {
    constexpr bool MX = FWD != EARLY;
    const int lane = threadIdx.x & 31;
    const int W = (gridDim.x * blockDim.x) >> 5;
    const int w = (threadIdx.x >> 5) * gridDim.x + blockIdx.x;   // consecutive units on different SMs
    const float ident = __int_as_float(MX ? 0xff800000 : 0x7f800000);
    unsigned target = 0;
    bool bad = false;
    int k = FWD ? 0 : p.L - 1;
    int eb = __ldg(p.row_ptr + __ldg(p.level_ptr + k)), ee = __ldg(p.row_ptr + __ldg(p.level_ptr + k + 1));
    // round-1 loads of U units: {neighbour, destination}, delay, the keys next to the unit
    int2 ed[W3_U];
    float dv[W3_U];
    int kprev[W3_U], knext[W3_U];
    auto load_units = [&](int ubase) {
#pragma unroll
        for (int i = 0; i < W3_U; ++i) {
            const int e0 = eb + ((ubase + i * W) << 5);
            const int e = e0 + lane;
            ed[i] = make_int2(0, -1 - lane);   // unique negative key: never stored
            dv[i] = 0.0f;
            kprev[i] = knext[i] = -1;
            if (e < ee) {
                ed[i] = __ldg(p.edge + e);
                dv[i] = p.eid ? __ldg(p.d + __ldg(p.eid + e)) : __ldg(p.d + e);
            }
            if (e0 < ee) {
                if (lane == 0 && e0 > eb) kprev[i] = __ldg(p.edge + e0 - 1).y;
                if (lane == 31 && e0 + 32 < ee) knext[i] = __ldg(p.edge + e0 + 32).y;
            }
        }
    };
    load_units(w);
    for (int qq = 0; qq < p.L; ++qq) {
        const int nunits = (ee - eb + 31) >> 5;
        for (int ub = w; ub < nunits; ub += W3_U * W) {
            if (ub != w) load_units(ub);
            float av[W3_U];
#pragma unroll
            for (int i = 0; i < W3_U; ++i)
                av[i] = ed[i].y >= 0 ? ord2f(__ldcg(p.out + ed[i].x)) : ident;
#pragma unroll
            for (int i = 0; i < W3_U; ++i) {
                if (ub + i * W >= nunits) break;   // warp-uniform
                const int key = ed[i].y;
                const bool valid = key >= 0;
                float v = valid ? relax1<FWD>(av[i], sane(dv[i], bad)) : ident;
                const int prv = __shfl_up_sync(0xffffffffu, key, 1);
                const int nxt = __shfl_down_sync(0xffffffffu, key, 1);
                const unsigned smask = __ballot_sync(0xffffffffu, lane == 0 || prv != key);
                const int sstart = 31 - __clz(smask & ((2u << lane) - 1u));
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const float y = __shfl_up_sync(0xffffffffu, v, o);
                    if (lane - o >= sstart) v = comb<MX>(v, y);
                }
                const bool seg_end = valid && (lane == 31 || nxt != key);
                // the row continues into the previous / next unit?
                const int kp = __shfl_sync(0xffffffffu, kprev[i], 0);
                const int kn = __shfl_sync(0xffffffffu, knext[i], 31);
                const bool open = (sstart == 0 && kp == key) || (lane == 31 && kn == key);
                if (seg_end) {
                    if (open) {
                        if (MX) atomicMax(p.out + key, f2ord(v));
                        else atomicMin(p.out + key, f2ord(v));
                    } else {
                        p.out[key] = f2ord(v);
                    }
                }
            }
        }
        if (qq + 1 == p.L) break;
        // split grid barrier: arrive, load the first units of the next level, wait
        target += gridDim.x;
        __syncthreads();
        if (threadIdx.x == 0) asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(p.bar) : "memory");
        k = FWD ? qq + 1 : p.L - 2 - qq;
        eb = __ldg(p.row_ptr + __ldg(p.level_ptr + k));
        ee = __ldg(p.row_ptr + __ldg(p.level_ptr + k + 1));
        load_units(w);
        if (threadIdx.x == 0)
            while (ld_acq(p.bar) < target) __nanosleep(32);
        __syncthreads();
    }
    if (bad) atomicOr(p.err, ERR_NONFINITE);
}

// ---- S = 1: k_wide4 -- k_wide3's edge units with the structure staged in shared memory
// Each CTA (1024 threads, one per SM) owns one contiguous share of every level's edge
// run, processed in tiles of W4_TE edges.  A tile's {neighbour, destination} int2s and
// delays (or delay ids) are copied into shared memory by cp.async one tile AHEAD --
// the next tile of the level, or the next level's first tile (structure is never
// written by the pass, so it may be fetched before the grid barrier) -- so after the
// barrier a tile costs one gather round trip: every thread issues the gathers of its
// up to W4_K edges at once, then the segmented combine / store / ordered-int atomic
// of k_wide3 (a row that continues past the tile or the CTA's share is folded in
// atomically).  Two tile buffers (2 x 73 KB).
// MEASURED AND NOT TAKEN (C5): 0.367 + 0.349 ms against k_wide3's 0.313 + 0.302 -- one
// gather round trip per tile does not help because the level is bound by the random
// 32-byte sector traffic (one sector per 4-byte gather and per row store), not by the
// number of dependent round trips; kept behind HF_WIDE4=1 and parity-tested.
constexpr int W4_THREADS = 1024;
constexpr int W4_TE = 6144;
constexpr int W4_K = W4_TE / W4_THREADS;   // edges per thread per tile

struct Wide4Params {
    const int32_t *level_ptr, *row_ptr;   // level-ordered CSR of this direction
    const int2 *edge;                     // [m] {plain neighbour node, destination node}
    const int32_t *eid;                   // [m] delay index per position, or null: d level-ordered
    const float *d;
    int32_t L;
    int32_t *out;                         // [n] ordered ints during the pass
    uint32_t *err;
    unsigned *bar;
};

__device__ __forceinline__ void cp_async_8(void *dst, const void *src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
                 "l"(src)
                 : "memory");
}
__device__ __forceinline__ void cp_async_4(void *dst, const void *src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
                 "l"(src)
                 : "memory");
}

template <bool FWD, bool EARLY>
__global__ void __launch_bounds__(W4_THREADS, 1) k_wide4(Wide4Params p) {
    constexpr bool MX = FWD != EARLY;
    extern __shared__ __align__(16) unsigned char w4_smem[];
    int2 *s_e[2] = {reinterpret_cast<int2 *>(w4_smem), reinterpret_cast<int2 *>(w4_smem) + W4_TE};
    int32_t *s_d[2] = {reinterpret_cast<int32_t *>(s_e[1] + W4_TE),
                       reinterpret_cast<int32_t *>(s_e[1] + W4_TE) + W4_TE};
    __shared__ int s_keys[2][2];   // destination of the edge before / after the tile (-1: none)
    const int tid = threadIdx.x, lane = tid & 31;
    const int nC = gridDim.x, c = blockIdx.x;
    const float ident = __int_as_float(MX ? 0xff800000 : 0x7f800000);
    unsigned target = 0;
    bool bad = false;
    // a tile: [ta, tb) of level edge run [eb, ee)
    auto share = [&](int k, int &sa, int &sb, int &eb, int &ee) {
        eb = __ldg(p.row_ptr + __ldg(p.level_ptr + k));
        ee = __ldg(p.row_ptr + __ldg(p.level_ptr + k + 1));
        const int len = ee - eb, sz = (len + nC - 1) / nC;
        sa = min(ee, eb + c * sz);
        sb = min(ee, sa + sz);
    };
    auto issue = [&](int buf, int ta, int tb, int eb, int ee) {
        for (int j = tid; j < tb - ta; j += W4_THREADS) {
            cp_async_8(s_e[buf] + j, p.edge + ta + j);
            cp_async_4(s_d[buf] + j, p.eid ? reinterpret_cast<const void *>(p.eid + ta + j)
                                           : reinterpret_cast<const void *>(p.d + ta + j));
        }
        if (tid == 0) {
            if (ta > eb && ta < tb) cp_async_4(&s_keys[buf][0], &p.edge[ta - 1].y);
            else s_keys[buf][0] = -1;
            if (tb < ee && ta < tb) cp_async_4(&s_keys[buf][1], &p.edge[tb].y);
            else s_keys[buf][1] = -1;
        }
    };
    // first tile of the first level
    int qq = 0;
    int k = FWD ? 0 : p.L - 1;
    int sa, sb, eb, ee;
    share(k, sa, sb, eb, ee);
    int t = 0, cur = 0;
    issue(0, sa, min(sb, sa + W4_TE), eb, ee);
    asm volatile("cp.async.commit_group;" ::: "memory");
    for (;;) {
        const int ntiles = max(1, (sb - sa + W4_TE - 1) / W4_TE);
        const int ta = min(sb, sa + t * W4_TE), tb = min(sb, ta + W4_TE);
        // the next item: the next tile of this level, or the next level's first tile
        int nk = k, nsa = sa, nsb = sb, neb = eb, nee = ee, nt = t + 1;
        const bool more = t + 1 < ntiles || qq + 1 < p.L;
        if (t + 1 >= ntiles && qq + 1 < p.L) {
            nk = FWD ? qq + 1 : p.L - 2 - qq;
            share(nk, nsa, nsb, neb, nee);
            nt = 0;
        }
        if (more) {
            const int nta = min(nsb, nsa + nt * W4_TE);
            issue(cur ^ 1, nta, min(nsb, nta + W4_TE), neb, nee);
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
        asm volatile("cp.async.wait_group 1;" ::: "memory");   // this tile's copies
        __syncthreads();
        // ---- the tile: all gathers in flight, then the combine
        const int nt_e = tb - ta;
        const int2 *E = s_e[cur];
        const int32_t *Dd = s_d[cur];
        float av[W4_K], dv[W4_K];
#pragma unroll
        for (int i = 0; i < W4_K; ++i) {
            const int j = tid + i * W4_THREADS;
            av[i] = ident;
            dv[i] = 0.0f;
            if (j < nt_e) {
                av[i] = ord2f(__ldcg(p.out + E[j].x));
                dv[i] = p.eid ? __ldg(p.d + Dd[j]) : __int_as_float(Dd[j]);
            }
        }
        const int kb = s_keys[cur][0], ka = s_keys[cur][1];
#pragma unroll
        for (int i = 0; i < W4_K; ++i) {
            if (i * W4_THREADS >= nt_e) break;   // block-uniform
            const int j = tid + i * W4_THREADS;
            const bool valid = j < nt_e;
            const int key = valid ? E[j].y : -1 - lane;
            float v = valid ? relax1<FWD>(av[i], sane(dv[i], bad)) : ident;
            const int prv = __shfl_up_sync(0xffffffffu, key, 1);
            const int nxt = __shfl_down_sync(0xffffffffu, key, 1);
            const unsigned smask = __ballot_sync(0xffffffffu, lane == 0 || prv != key);
            const int sstart = 31 - __clz(smask & ((2u << lane) - 1u));
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const float y = __shfl_up_sync(0xffffffffu, v, o);
                if (lane - o >= sstart) v = comb<MX>(v, y);
            }
            if (valid && (lane == 31 || nxt != key)) {
                // the key of the edge before this segment / after it (tile boundary: the
                // neighbouring tile's or share's edge)
                const int j0 = j - (lane - sstart);
                const int kprev = j0 > 0 ? E[j0 - 1].y : kb;
                const int knext = j + 1 < nt_e ? E[j + 1].y : ka;
                if (kprev == key || knext == key) {
                    if (MX) atomicMax(p.out + key, f2ord(v));
                    else atomicMin(p.out + key, f2ord(v));
                } else {
                    p.out[key] = f2ord(v);
                }
            }
        }
        __syncthreads();   // buffer `cur` is refilled two items from now
        cur ^= 1;
        if (!more) break;
        if (t + 1 < ntiles) {
            ++t;
            continue;
        }
        // level done: grid barrier, then the next level (its first tile is in flight)
        target += gridDim.x;
        if (tid == 0) {
            asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(p.bar) : "memory");
            while (ld_acq(p.bar) < target) __nanosleep(32);
        }
        __syncthreads();
        ++qq;
        k = nk;
        sa = nsa;
        sb = nsb;
        eb = neb;
        ee = nee;
        t = 0;
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    if (bad) atomicOr(p.err, ERR_NONFINITE);
}

template <bool FWD, bool EARLY>
void launch_w4(Graph &g, Wide4Params &w, cudaStream_t st) {
    auto kern = k_wide4<FWD, EARLY>;
    const int smem = int(2 * W4_TE * (sizeof(int2) + sizeof(int32_t)));
    static std::map<std::pair<const void *, int>, int> cache;
    static std::mutex mu;
    int per_sm = 0;
    {
        std::lock_guard<std::mutex> lk(mu);
        auto it = cache.find({(const void *)kern, g.device});
        if (it != cache.end()) per_sm = it->second;
    }
    if (!per_sm) {
        ensure_dyn_smem((const void *)kern, g.device, size_t(smem));
        HF_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, W4_THREADS, smem));
        std::lock_guard<std::mutex> lk(mu);
        cache[{(const void *)kern, g.device}] = per_sm;
    }
    if (per_sm < 1) fail(HF_ERR_CUDA, "wide propagation kernel does not fit on an SM");
    void *args[] = {&w};
    HF_CUDA(cudaLaunchCooperativeKernel((const void *)kern, g.sms, W4_THREADS, args, smem, st));
    g.launches += 1;
}

// before a k_wide3 pass: every node's accumulator at the identity, nodes without edges
// in this direction at their value (forward: at_src or +0; backward: T) -- by node id,
// so every access is coalesced (ptr = the node-indexed CSR of this direction)
template <bool FWD, bool EARLY>
__global__ void k_w3_init(const int32_t *__restrict__ ptr, int32_t n,
                          const float *__restrict__ src_val, float t_scalar,
                          int32_t *__restrict__ out, uint32_t *err) {
    constexpr bool MX = FWD != EARLY;
    bool bad = false;
    const float tb = FWD ? 0.0f : (src_val ? src_val[0] : t_scalar);
    for (int64_t v = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; v < n;
         v += int64_t(gridDim.x) * blockDim.x) {
        int32_t o;
        if (ptr[v + 1] != ptr[v]) {
            o = MX ? ORD_NEG_INF : ORD_POS_INF;
        } else {
            const float x = FWD ? (src_val ? sane(src_val[v], bad) : 0.0f) : sane(tb, bad);
            o = f2ord(x);
        }
        out[v] = o;
    }
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(err, ERR_NONFINITE);
}

// after a k_wide3 pass: ordered ints back to floats in place; backward: slack and the
// worst slack (ordered-int atomicMin per block)
template <bool FWD, bool EARLY>
__global__ void k_w3_final(int32_t *__restrict__ out, int32_t n, const float *__restrict__ other,
                           float *__restrict__ slack, int32_t *__restrict__ wns_ord) {
    __shared__ int32_t s_wmin;
    const bool do_slack = !FWD && other;
    if (threadIdx.x == 0) s_wmin = ORD_POS_INF;
    __syncthreads();
    float mn = __int_as_float(ORD_POS_INF);
    for (int64_t v = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; v < n;
         v += int64_t(gridDim.x) * blockDim.x) {
        const float x = ord2f(out[v]);
        reinterpret_cast<float *>(out)[v] = x;
        if (do_slack) {
            const float a = other[v];
            const float sl = EARLY ? __fsub_rn(a, x) : __fsub_rn(x, a);
            mn = fminf(mn, sl);
            if (slack) slack[v] = sl;
        }
    }
    if (do_slack) {
#pragma unroll
        for (int o = 16; o; o >>= 1) mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
        if ((threadIdx.x & 31) == 0 && mn != __int_as_float(ORD_POS_INF)) atomicMin(&s_wmin, f2ord(mn));
        __syncthreads();
        if (threadIdx.x == 0 && s_wmin != ORD_POS_INF) atomicMin(wns_ord, s_wmin);
    }
}

// {plain neighbour, destination node} per level-ordered edge (k_wide3)
__global__ void k_w3_edges(const int32_t *__restrict__ nbr, const int32_t *__restrict__ part_row,
                           const int32_t *__restrict__ node_of, const int32_t *__restrict__ erow,
                           int32_t m, int2 *__restrict__ out) {
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < m;
         e += int64_t(gridDim.x) * blockDim.x) {
        const int u = nbr[e];
        out[e] = make_int2(u >= 0 ? u : node_of[part_row[-u - 1]], node_of[erow[e]]);
    }
}

template <bool FWD, bool EARLY>
int w3_blocks(const Graph &g) {
    auto kern = k_wide3<FWD, EARLY>;
    static std::map<std::pair<const void *, int>, int> cache;
    static std::mutex mu;
    int per_sm = 0;
    {
        std::lock_guard<std::mutex> lk(mu);
        auto it = cache.find({(const void *)kern, g.device});
        if (it != cache.end()) per_sm = it->second;
    }
    if (!per_sm) {
        HF_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, W3_THREADS, 0));
        std::lock_guard<std::mutex> lk(mu);
        cache[{(const void *)kern, g.device}] = per_sm;
    }
    const int cap = env_int_w("HF_WIDE_CTAS_PER_SM", 0);
    if (cap > 0) per_sm = std::min(per_sm, cap);
    return g.sms * per_sm;
}

}  // namespace

// Build (once per levelization) the slices of both directions.
void wide_prepare(Graph &g) {
    if (g.wide_ready) return;
    cudaStream_t s = g.stream;
    const int32_t n = g.n, m = g.m;
    const int64_t scap = int64_t(m) / WIDE_SL + int64_t(m) / (LO_SPLIT + 1) + 1;
    DevBuf cnt;
    cnt.alloc(sizeof(int32_t) * (int64_t(n) + 1), s);
    for (int dir = 0; dir < 2; ++dir) {
        const bool in = dir == 0;
        const int32_t *rp = in ? g.lo_in_ptr.as<int32_t>() : g.lo_out_ptr.as<int32_t>();
        const int32_t *no = in ? g.lo_in_node.as<int32_t>() : g.lo_out_node.as<int32_t>();
        const int32_t *ls = in ? g.lo_in_lstart.as<int32_t>() : g.lo_out_lstart.as<int32_t>();
        DevBuf &sf = in ? g.wide_in_sfirst : g.wide_out_sfirst;
        DevBuf &sl = in ? g.wide_in_slice : g.wide_out_slice;
        sf.alloc(sizeof(int32_t) * (int64_t(n) + 1), s);
        sl.alloc(sizeof(int2) * size_t(scap), s);
        k_wide_count<<<grid_for(int64_t(n) + 1, 256, g.sms), 256, 0, s>>>(
            rp, no, g.level.as<int32_t>(), ls, n, cnt.as<int32_t>());
        HF_CHECK_LAUNCH();
        scan_exclusive(cnt.as<int32_t>(), sf.as<int32_t>(), int64_t(n) + 1, nullptr, s, g);
        k_wide_slices<<<grid_for(n, 256, g.sms), 256, 0, s>>>(rp, sf.as<int32_t>(), n,
                                                             sl.as<int2>());
        HF_CHECK_LAUNCH();
        g.launches += 2;
        DevBuf &co = in ? g.wide_in_coff : g.wide_out_coff;
        DevBuf &cr = in ? g.wide_in_crow : g.wide_out_crow;
        co.alloc(sizeof(int32_t) * (int64_t(g.L) + 1), s);
        cr.alloc(sizeof(int32_t) * size_t(int64_t(m) / 32 + g.L + 1), s);
        k_w1_coff<<<1, 1024, 0, s>>>(g.level_ptr.as<int32_t>(), ls, rp, g.L, co.as<int32_t>());
        HF_CHECK_LAUNCH();
        k_w1_crow<<<grid_for(n, 256, g.sms), 256, 0, s>>>(rp, no, g.level.as<int32_t>(), ls,
                                                         co.as<int32_t>(), n, cr.as<int32_t>());
        HF_CHECK_LAUNCH();
        g.launches += 2;
    }
    g.wide_ready = true;
}

// k_wide2 tables of both directions (once per levelization): plain neighbour ids,
// the row of every edge, the row ranges of every level.
void wide2_prepare(Graph &g) {
    if (g.w2_ready) return;
    cudaStream_t s = g.stream;
    const int32_t n = g.n, m = g.m;
    DevBuf erow;
    erow.alloc(sizeof(int32_t) * std::max<int64_t>(m, 1), s);
    for (int dir = 0; dir < 2; ++dir) {
        const bool in = dir == 0;
        const int32_t *rp = in ? g.lo_in_ptr.as<int32_t>() : g.lo_out_ptr.as<int32_t>();
        const int32_t *no = in ? g.lo_in_node.as<int32_t>() : g.lo_out_node.as<int32_t>();
        const int32_t *nb = in ? g.lo_in_nbr.as<int32_t>() : g.lo_out_nbr.as<int32_t>();
        const int32_t *npa = in ? g.lo_in_np.as<int32_t>() : g.lo_out_np.as<int32_t>();
        const int32_t *prow = npa + (in ? g.np_cap_in : g.np_cap_out);
        DevBuf &pn = in ? g.w2_in_nbr : g.w2_out_nbr;     // int2 {neighbour, row}
        DevBuf &nd = in ? g.w2_in_erow : g.w2_out_erow;   // int32 encoded node per row
        DevBuf &ro = in ? g.w2_in_roff : g.w2_out_roff;
        DevBuf &rs = in ? g.w2_in_rstart : g.w2_out_rstart;   // int2 descriptors
        pn.alloc(sizeof(int2) * std::max<int64_t>(m, 1), s);
        nd.alloc(sizeof(int32_t) * std::max<int64_t>(n, 1), s);
        ro.alloc(sizeof(int32_t) * (int64_t(g.L) + 1), s);
        // entries: sum over levels of (ranges + 1) <= (n + m) / W2_TW + 2L
        rs.alloc(sizeof(int2) * size_t((int64_t(n) + m) / W2_TW + 2 * int64_t(g.L) + 1), s);
        if (m) {
            csr_row_ids(rp, n, erow.as<int32_t>(), s, g);
            k_w2_edges<<<grid_for(m, 256, g.sms), 256, 0, s>>>(nb, prow, no, erow.as<int32_t>(), m,
                                                               pn.as<int2>());
            HF_CHECK_LAUNCH();
        }
        k_w2_nodes<<<grid_for(n, 256, g.sms), 256, 0, s>>>(rp, no, n, nd.as<int32_t>());
        HF_CHECK_LAUNCH();
        k_w2_roff<<<1, 1024, 0, s>>>(g.level_ptr.as<int32_t>(), rp, g.L, ro.as<int32_t>());
        HF_CHECK_LAUNCH();
        k_w2_rdesc<<<grid_for(n, 256, g.sms), 256, 0, s>>>(rp, no, g.level.as<int32_t>(),
                                                          g.level_ptr.as<int32_t>(),
                                                          ro.as<int32_t>(), n, rs.as<int2>());
        HF_CHECK_LAUNCH();
        g.launches += 5;
    }
    g.w2_ready = true;
}

// k_wide3 edge table of both directions (once per levelization)
void wide3_prepare(Graph &g) {
    if (g.w3_ready) return;
    cudaStream_t s = g.stream;
    const int32_t n = g.n, m = g.m;
    DevBuf erow;
    erow.alloc(sizeof(int32_t) * std::max<int64_t>(m, 1), s);
    for (int dir = 0; dir < 2; ++dir) {
        const bool in = dir == 0;
        DevBuf &ed = in ? g.w3_in_edge : g.w3_out_edge;
        ed.alloc(sizeof(int2) * std::max<int64_t>(m, 1), s);
        if (!m) continue;
        const int32_t *rp = in ? g.lo_in_ptr.as<int32_t>() : g.lo_out_ptr.as<int32_t>();
        const int32_t *npa = in ? g.lo_in_np.as<int32_t>() : g.lo_out_np.as<int32_t>();
        csr_row_ids(rp, n, erow.as<int32_t>(), s, g);
        k_w3_edges<<<grid_for(m, 256, g.sms), 256, 0, s>>>(
            in ? g.lo_in_nbr.as<int32_t>() : g.lo_out_nbr.as<int32_t>(),
            npa + (in ? g.np_cap_in : g.np_cap_out),
            in ? g.lo_in_node.as<int32_t>() : g.lo_out_node.as<int32_t>(), erow.as<int32_t>(), m,
            ed.as<int2>());
        HF_CHECK_LAUNCH();
        g.launches += 2;
    }
    g.w3_ready = true;
}

// The graph's own delays in level order of both directions (single-set calls).
void lo_delays_prepare(Graph &g) {
    if (g.lo_d_ready) return;
    cudaStream_t s = g.stream;
    const int64_t mm = (g.m > 0 ? g.m : 1) + LO_PAD;
    g.lo_in_d.alloc(sizeof(float) * mm, s);
    g.lo_out_d.alloc(sizeof(float) * mm, s);
    if (g.m) {
        k_gather_delay<<<grid_for(g.m, 256, g.sms), 256, 0, s>>>(
            g.delay.as<float>(), g.lo_in_eid.as<int32_t>(), g.m, g.lo_in_d.as<float>());
        HF_CHECK_LAUNCH();
        k_gather_delay<<<grid_for(g.m, 256, g.sms), 256, 0, s>>>(
            g.delay.as<float>(), g.lo_out_eid.as<int32_t>(), g.m, g.lo_out_d.as<float>());
        HF_CHECK_LAUNCH();
        g.launches += 2;
    }
    g.lo_d_ready = true;
}

// Should the passes of this graph run level-synchronously?  HF_WIDE=1 / 0 forces
// the choice; by default for a single delay set (S = 1) when the mean level holds
// >= 32768 nodes (C5: ~333k; the deep C3/C4 graph: 7500, where the dataflow kernel's
// overlap of levels wins).  With S >= 4 columns per row the dataflow kernel's
// vectorised rows do as well or better on C5 (profiles/round2_*), so it keeps them.
bool wide_choice(const Graph &g, int32_t S) {
    const int f = env_int_w("HF_WIDE", -1);
    if (f >= 0) return f != 0;
    return S == 1 && g.L > 0 && int64_t(g.n) >= int64_t(g.L) * 32768;
}

// One level-synchronous pass.  d: [m][S] by edge id, or level-ordered [m] when
// lo_delays (S == 1, the graph's own delays).  wns_ord [S] must hold +inf ords.
template <bool FWD>
void wide_pass(Graph &g, const float *d, bool lo_delays, int32_t S, const float *src_val,
               float t_scalar, const float *other, float *out, float *slack, int32_t *wns_ord,
               cudaStream_t st) {
    wide_prepare(g);
    WideParams p{};
    const bool in = FWD;
    p.level_ptr = g.level_ptr.as<int32_t>();
    p.lstart = in ? g.lo_in_lstart.as<int32_t>() : g.lo_out_lstart.as<int32_t>();
    p.row_ptr = in ? g.lo_in_ptr.as<int32_t>() : g.lo_out_ptr.as<int32_t>();
    p.nbr = in ? g.lo_in_nbr.as<int32_t>() : g.lo_out_nbr.as<int32_t>();
    p.eid = lo_delays ? nullptr : (in ? g.lo_in_eid.as<int32_t>() : g.lo_out_eid.as<int32_t>());
    p.node_of = in ? g.lo_in_node.as<int32_t>() : g.lo_out_node.as<int32_t>();
    p.q = in ? g.lo_in_q.as<int32_t>() : g.lo_out_q.as<int32_t>();
    p.sfirst = in ? g.wide_in_sfirst.as<int32_t>() : g.wide_out_sfirst.as<int32_t>();
    p.slice = in ? g.wide_in_slice.as<int2>() : g.wide_out_slice.as<int2>();
    const int32_t npcap = in ? g.np_cap_in : g.np_cap_out;
    p.part_np = in ? g.lo_in_np.as<int32_t>() : g.lo_out_np.as<int32_t>();
    p.part_row = p.part_np + npcap;
    p.nparts_d = g.nparts_d + (in ? 0 : 1);
    p.L = g.L;
    p.S = S;
    p.d = d;
    p.src_val = src_val;
    p.t_scalar = t_scalar;
    p.other = other;
    p.out = out;
    p.slack = slack;
    p.wns_ord = wns_ord;
    p.err = g.d_err();
    if (S == 1 && env_int_w("HF_WIDE3", 1)) {
        wide3_prepare(g);
        const int32_t *rp = in ? g.lo_in_ptr.as<int32_t>() : g.lo_out_ptr.as<int32_t>();
        int32_t *acc = reinterpret_cast<int32_t *>(out);   // ordered ints during the pass
#define HF_W3(EE)                                                                                  \
    do {                                                                                           \
        k_w3_init<FWD, EE><<<grid_for(g.n, 256, g.sms), 256, 0, st>>>(                            \
            in ? g.in_ptr.as<int32_t>() : g.out_ptr.as<int32_t>(), g.n, src_val, t_scalar, acc,     \
            p.err);                                                                                \
        HF_CHECK_LAUNCH();                                                                         \
        Wide3Params w{};                                                                           \
        w.level_ptr = g.level_ptr.as<int32_t>();                                                   \
        w.row_ptr = rp;                                                                            \
        w.edge = in ? g.w3_in_edge.as<int2>() : g.w3_out_edge.as<int2>();                         \
        w.eid = p.eid;                                                                             \
        w.d = d;                                                                                   \
        w.L = g.L;                                                                                 \
        w.out = acc;                                                                               \
        w.err = p.err;                                                                             \
        DevBuf bar3;                                                                               \
        bar3.alloc(sizeof(unsigned) * 2, st);                                                      \
        HF_CUDA(cudaMemsetAsync(bar3.p, 0, sizeof(unsigned) * 2, st));                             \
        w.bar = bar3.as<unsigned>();                                                               \
        if (env_int_w("HF_WIDE4", 0)) {                                                           \
            Wide4Params w4{};                                                                      \
            w4.level_ptr = w.level_ptr;                                                            \
            w4.row_ptr = w.row_ptr;                                                                \
            w4.edge = w.edge;                                                                      \
            w4.eid = w.eid;                                                                        \
            w4.d = w.d;                                                                            \
            w4.L = w.L;                                                                            \
            w4.out = w.out;                                                                        \
            w4.err = w.err;                                                                        \
            w4.bar = w.bar;                                                                        \
            launch_w4<FWD, EE>(g, w4, st);                                                         \
        } else {                                                                                   \
            const int nblk = w3_blocks<FWD, EE>(g);                                                \
            if (nblk < 1) fail(HF_ERR_CUDA, "wide propagation kernel does not fit on an SM");     \
            void *args[] = {&w};                                                                   \
            HF_CUDA(cudaLaunchCooperativeKernel((const void *)k_wide3<FWD, EE>, nblk, W3_THREADS,  \
                                                args, 0, st));                                     \
        }                                                                                          \
        k_w3_final<FWD, EE><<<grid_for(g.n, 256, g.sms), 256, 0, st>>>(acc, g.n, other, slack,     \
                                                                       wns_ord);                   \
        HF_CHECK_LAUNCH();                                                                         \
        g.launches += 3;                                                                           \
    } while (0)
        if (g.early) HF_W3(true);
        else HF_W3(false);
#undef HF_W3
        return;
    }
    if (S == 1 && env_int_w("HF_WIDE2", 0)) {
        wide2_prepare(g);
        Wide2Params w{};
        w.node = in ? g.w2_in_erow.as<int32_t>() : g.w2_out_erow.as<int32_t>();
        w.nbr_row = in ? g.w2_in_nbr.as<int2>() : g.w2_out_nbr.as<int2>();
        w.eid = p.eid;
        w.roff = in ? g.w2_in_roff.as<int32_t>() : g.w2_out_roff.as<int32_t>();
        w.rdesc = in ? g.w2_in_rstart.as<int2>() : g.w2_out_rstart.as<int2>();
        w.L = g.L;
        w.d = d;
        w.src_val = src_val;
        w.t_scalar = t_scalar;
        w.other = other;
        w.out = out;
        w.slack = slack;
        w.wns_ord = wns_ord;
        w.err = p.err;
        DevBuf bar2;
        bar2.alloc(sizeof(unsigned) * 2, st);
        HF_CUDA(cudaMemsetAsync(bar2.p, 0, sizeof(unsigned) * 2, st));
        w.bar = bar2.as<unsigned>();
        const int nblk = g.early ? w2_blocks<FWD, true>(g) : w2_blocks<FWD, false>(g);
        if (nblk < 1) fail(HF_ERR_CUDA, "wide propagation kernel does not fit on an SM");
        const char *trace_env = getenv("HF_TRACE");
        DevBuf tb;
        if (trace_env) {
            tb.alloc(sizeof(unsigned long long) * 2 * size_t(g.L) * nblk, st);
            HF_CUDA(cudaMemsetAsync(tb.p, 0, tb.bytes, st));
            w.trace = tb.as<unsigned long long>();
        }
        void *args[] = {&w};
        const void *kern = g.early ? (const void *)k_wide2<FWD, true> : (const void *)k_wide2<FWD, false>;
        HF_CUDA(cudaLaunchCooperativeKernel(kern, nblk, W2_THREADS, args, 0, st));
        g.launches += 1;
        if (trace_env) {
            std::vector<unsigned long long> h(2 * size_t(g.L) * nblk);
            HF_CUDA(cudaMemcpyAsync(h.data(), tb.p, h.size() * 8, cudaMemcpyDeviceToHost, st));
            HF_CUDA(cudaStreamSynchronize(st));
            const std::string fn = std::string(trace_env) + (FWD ? "_w2_fwd.bin" : "_w2_bwd.bin");
            if (FILE *f = fopen(fn.c_str(), "wb")) {
                const int32_t hdr[2] = {g.L, nblk};
                fwrite(hdr, 4, 2, f);
                fwrite(h.data(), 8, h.size(), f);
                fclose(f);
            }
        }
        return;
    }
    if (S == 1 && env_int_w("HF_WIDE1", 1)) {
        Wide1Params w{};
        w.level_ptr = p.level_ptr;
        w.lstart = p.lstart;
        w.row_ptr = p.row_ptr;
        w.nbr = p.nbr;
        w.eid = p.eid;
        w.node_of = p.node_of;
        w.q = p.q;
        w.coff = in ? g.wide_in_coff.as<int32_t>() : g.wide_out_coff.as<int32_t>();
        w.crow = in ? g.wide_in_crow.as<int32_t>() : g.wide_out_crow.as<int32_t>();
        w.part_np = p.part_np;
        w.part_row = p.part_row;
        w.nparts_d = p.nparts_d;
        w.L = g.L;
        w.d = d;
        w.src_val = src_val;
        w.t_scalar = t_scalar;
        w.other = other;
        w.out = out;
        w.slack = slack;
        w.wns_ord = wns_ord;
        w.err = p.err;
        DevBuf slots1, bar1;
        slots1.alloc(sizeof(int32_t) * std::max<size_t>(size_t(npcap), 1), st);
        bar1.alloc(sizeof(unsigned) * 2, st);
        HF_CUDA(cudaMemsetAsync(bar1.p, 0, sizeof(unsigned) * 2, st));
        w.slot = slots1.as<int32_t>();
        w.bar = bar1.as<unsigned>();
        // HF_TRACE=<prefix>: per level and block {start, all its units done} -> <prefix>_w1_<dir>.bin
        const char *trace_env = getenv("HF_TRACE");
        DevBuf tb;
        const int nblk = g.early ? w1_blocks<FWD, true>(g) : w1_blocks<FWD, false>(g);
        if (trace_env) {
            tb.alloc(sizeof(unsigned long long) * 2 * size_t(g.L) * nblk, st);
            HF_CUDA(cudaMemsetAsync(tb.p, 0, tb.bytes, st));
            w.trace = tb.as<unsigned long long>();
        }
        if (g.early) launch_w1<FWD, true>(g, w, st);
        else launch_w1<FWD, false>(g, w, st);
        if (trace_env) {
            std::vector<unsigned long long> h(2 * size_t(g.L) * nblk);
            HF_CUDA(cudaMemcpyAsync(h.data(), tb.p, h.size() * 8, cudaMemcpyDeviceToHost, st));
            HF_CUDA(cudaStreamSynchronize(st));
            const std::string fn = std::string(trace_env) + (FWD ? "_w1_fwd.bin" : "_w1_bwd.bin");
            if (FILE *f = fopen(fn.c_str(), "wb")) {
                const int32_t hdr[2] = {g.L, nblk};
                fwrite(hdr, 4, 2, f);
                fwrite(h.data(), 8, h.size(), f);
                fclose(f);
            }
        }
        return;
    }
    DevBuf slots, bar;
    slots.alloc(sizeof(int32_t) * std::max<size_t>(size_t(npcap) * size_t(S), 1), st);
    bar.alloc(sizeof(unsigned) * 2, st);
    HF_CUDA(cudaMemsetAsync(bar.p, 0, sizeof(unsigned) * 2, st));
    p.slot = slots.as<int32_t>();
    p.bar = bar.as<unsigned>();
    const bool v4 = S % 4 == 0 && (reinterpret_cast<uintptr_t>(d) & 15) == 0 &&
                    (reinterpret_cast<uintptr_t>(out) & 15) == 0 &&
                    (!other || (reinterpret_cast<uintptr_t>(other) & 15) == 0) &&
                    (!slack || (reinterpret_cast<uintptr_t>(slack) & 15) == 0);
    if (g.early) {
        if (v4) launch_wide<4, FWD, true>(g, p, st);
        else launch_wide<1, FWD, true>(g, p, st);
    } else {
        if (v4) launch_wide<4, FWD, false>(g, p, st);
        else launch_wide<1, FWD, false>(g, p, st);
    }
}

template void wide_pass<true>(Graph &, const float *, bool, int32_t, const float *, float,
                              const float *, float *, float *, int32_t *, cudaStream_t);
template void wide_pass<false>(Graph &, const float *, bool, int32_t, const float *, float,
                               const float *, float *, float *, int32_t *, cudaStream_t);

}  // namespace hf
