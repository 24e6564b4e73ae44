// propagate.cu -- forward max-plus and backward min-plus (+ fused slack / worst
// slack) over the levelized DAG, for one delay set or S scenario sets.
// SURVEY.md §8(a) a5-a7; BASELINE.json:5.
//
// Data layout in HBM (scenario-minor): at[v*S + s], rat[v*S + s],
// delays[e*S + s].  A node's S values are contiguous, so each edge touches S*4
// contiguous bytes; a node row is owned by LPN = S/V lanes holding V-wide
// vectors (V = 4 -> LDG.128 / STG.128).  Pull-based, no float atomics: every
// output is one fp32 max/min over fl(x +/- d) terms, which is order-independent
// (0 ULP against the oracle, reading R10).
//
// One persistent launch per pass (cooperative launch, one CTA per SM; no
// per-level launches, no grid barrier):
//   * every level is cut into weight-balanced PIECES (weight = edges + nodes);
//     piece j of a level belongs to CTA j mod P, and a CTA walks its pieces in
//     pass order (levels ascending forward, descending backward);
//   * STAGING: a piece's level-ordered rows, neighbour ids, edge ids and delay
//     slices are copied into shared memory with cp.async by all threads -- rows
//     two pieces ahead, delays one piece ahead of the piece being computed
//     (3-slot ring).  None of this depends on earlier levels, so the HBM stream
//     of delays runs ahead of the dependency front;
//   * DEPENDENCY: before computing a piece of level k the CTA waits until level
//     k-1 (k+1 backward) has published all its pieces: one acquire-poll of a
//     per-level counter by one thread.  Level k complete => every earlier level
//     complete, by induction; a CTA only waits on earlier levels whose pieces
//     belong to co-resident CTAs, so the schedule cannot deadlock;
//   * COMPUTE: edge-parallel gathers of at[u] / rat[v] from L2 (all edge-lane
//     items issue their loads at once), x = fl(a +/- d) written in place over the
//     staged delay, then each node's owner lanes reduce their row from shared
//     memory; rows longer than HUB_DEG are reduced by the whole CTA (strided
//     partials, shared-memory combine).  Stores, gpu-scope fence, one atomicAdd
//     publishes the piece;
//   * backward fuses slack = rat - at and keeps a per-lane running min; one
//     shared-memory reduction and one global atomicMin per scenario per CTA give
//     the worst slack.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "common.cuh"

namespace hf {

namespace {

constexpr int NCW = 16;                 // consumer warps
constexpr int NC = NCW * 32;            // consumer threads
constexpr int NPW = 2;                  // producer warps
constexpr int BLOCK = NC + 32 * NPW;
constexpr int NBUF = 4;                 // staging ring slots
constexpr int HUB_DEG = 64;    // rows longer than this are reduced by the whole CTA
constexpr int MAX_HUBS = 256;  // long rows per piece (piece weight bounds this)

template <int V> struct Vec {
    float x[V];
};

template <int V> __device__ __forceinline__ Vec<V> ldv_g(const float *p) {   // read-only input
    Vec<V> r;
    if constexpr (V == 4) {
        float4 t = __ldg(reinterpret_cast<const float4 *>(p));
        r.x[0] = t.x; r.x[1] = t.y; r.x[2] = t.z; r.x[3] = t.w;
    } else if constexpr (V == 2) {
        float2 t = __ldg(reinterpret_cast<const float2 *>(p));
        r.x[0] = t.x; r.x[1] = t.y;
    } else {
        r.x[0] = __ldg(p);
    }
    return r;
}
// values produced inside this launch by other CTAs: L2-coherent loads (never L1)
template <int V> __device__ __forceinline__ Vec<V> ldv_cg(const float *p) {
    Vec<V> r;
    if constexpr (V == 4) {
        float4 t = __ldcg(reinterpret_cast<const float4 *>(p));
        r.x[0] = t.x; r.x[1] = t.y; r.x[2] = t.z; r.x[3] = t.w;
    } else if constexpr (V == 2) {
        float2 t = __ldcg(reinterpret_cast<const float2 *>(p));
        r.x[0] = t.x; r.x[1] = t.y;
    } else {
        r.x[0] = __ldcg(p);
    }
    return r;
}
template <int V> __device__ __forceinline__ Vec<V> ldv_s(const float *p) {
    Vec<V> r;
    if constexpr (V == 4) {
        float4 t = *reinterpret_cast<const float4 *>(p);
        r.x[0] = t.x; r.x[1] = t.y; r.x[2] = t.z; r.x[3] = t.w;
    } else if constexpr (V == 2) {
        float2 t = *reinterpret_cast<const float2 *>(p);
        r.x[0] = t.x; r.x[1] = t.y;
    } else {
        r.x[0] = *p;
    }
    return r;
}
template <int V> __device__ __forceinline__ void stv_s(float *p, const Vec<V> &v) {
    if constexpr (V == 4) {
        *reinterpret_cast<float4 *>(p) = make_float4(v.x[0], v.x[1], v.x[2], v.x[3]);
    } else if constexpr (V == 2) {
        *reinterpret_cast<float2 *>(p) = make_float2(v.x[0], v.x[1]);
    } else {
        *p = v.x[0];
    }
}
template <int V> __device__ __forceinline__ void stv_g(float *p, const Vec<V> &v) {
    if constexpr (V == 4) {
        __stcg(reinterpret_cast<float4 *>(p), make_float4(v.x[0], v.x[1], v.x[2], v.x[3]));
    } else if constexpr (V == 2) {
        __stcg(reinterpret_cast<float2 *>(p), make_float2(v.x[0], v.x[1]));
    } else {
        __stcg(p, v.x[0]);
    }
}

__device__ __forceinline__ int ld_acquire(const int *p) {
    int v;
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cp_async4(void *dst, const void *src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst)), "l"(src)
                 : "memory");
}
__device__ __forceinline__ void cp_async16(void *dst, const void *src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src)
                 : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void cp_wait_prev() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

struct PassParams {
    // level-ordered CSR of this direction: row i <-> node node_of[i]
    const int32_t *row_ptr;    // [n+1]
    const int32_t *nbr;        // [m] neighbour node id (fan-in src / fan-out dst)
    const int32_t *eid;        // [m] edge id (delay row)
    const int32_t *node_of;    // [n]
    const int4 *cta_pc;        // per-CTA piece sequence (pass order): {pos_begin, pos_end,
                               // edge_begin, edge_end}
    const int32_t *cta_lv;     // level of each entry of cta_pc
    const int32_t *cta_off;    // [P+1] first entry of every CTA
    const int32_t *piece_off;  // [L+1] first piece of every level (pieces per level)
    int32_t L;
    int32_t ncap, ecap;        // staged rows / edges per ring slot
    int32_t split;             // rows longer than this are cut into part pieces
    int32_t psize;             // edges per part piece
    const int32_t *q;          // [n+1] first part id of every row (split rows)
    const int32_t *part_np;    // [parts] number of parts of the row whose first part id it is
    float *part_buf;           // [parts][S] partial results of part pieces
    int32_t *part_cnt;         // [parts] parts finished, indexed by a row's first part id
    int32_t S;                 // scenarios (row stride of at / rat / delays)
    const float *d;            // [m][S]
    const float *src_val;      // forward: at_src [n] (or null); backward: t_req [S] (or null)
    float t_scalar;            // backward: T when t_req is null
    const float *other;        // backward: at (for slack)
    float *out;                // forward: at; backward: rat
    float *slack;              // backward, optional [n][S]
    int32_t *wns_ord;          // backward: [S] ordered-int mins
    int32_t *done;             // [L] pieces published per level
    uint32_t *err;
    // optional timeline (HF_TRACE=1): per piece {level<<8|slot, cta, t_top, t_ready,
    // t_computed, t_published, edges, rows} in globaltimer ns
    unsigned long long *trace;
    int32_t *trace_n;
    int32_t trace_cap;
};

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// ring-slot layout in shared memory (bytes); identical on host and device
struct SlotLayout {
    int meta, node, rp, nbr, medrow, medpre, d, bytes;
};
constexpr int MAXMED = 256;   // medium rows per piece (bounded by ecap / CH)
constexpr int CH = 8;         // chunk of a medium row pre-reduced by one item
__host__ __device__ inline SlotLayout slot_layout(int ncap, int ecap, int S) {
    SlotLayout L;
    int o = 0;
    L.meta = o;   o += 16 * 4;
    L.node = o;   o += ncap * 4;
    L.rp = o;     o += (ncap + 1) * 4;
    L.nbr = o;    o += ecap * 4;
    L.medrow = o; o += MAXMED * 4;
    L.medpre = o; o += (MAXMED + 1) * 4;
    o = (o + 127) & ~127;
    L.d = o;      o += ecap * S * 4;
    L.bytes = (o + 127) & ~127;
    return L;
}
enum { MT_LV = 0, MT_POS, MT_NN, MT_RB, MT_E, MT_EST, MT_NMED, MT_PART, MT_QB };

template <bool FWD> __device__ __forceinline__ float combine(float best, float x) {
    return FWD ? fmaxf(best, x) : fminf(best, x);
}
template <bool FWD> __device__ __forceinline__ float relax(float a, float d) {
    return FWD ? __fadd_rn(a, d) : __fsub_rn(a, d);
}
template <bool FWD> __device__ __forceinline__ float ident() {
    return __int_as_float(FWD ? 0xff800000 : 0x7f800000);   // -inf for max, +inf for min
}

// combine v into *addr with max (forward) / min (backward); exact, order-free
template <bool FWD> __device__ __forceinline__ void atomic_combine(float *addr, float v) {
    int *ai = reinterpret_cast<int *>(addr);
    int old = __ldcg(ai);
    for (;;) {
        const float nv = combine<FWD>(__int_as_float(old), v);
        if (__float_as_int(nv) == old) return;
        const int prev = atomicCAS(ai, old, __float_as_int(nv));
        if (prev == old) return;
        old = prev;
    }
}

// at[u] / rat[u] of a neighbour; a neighbour that is a split row is encoded as
// -(first part id + 1) and read as the combine of its part partials (the row's
// own value is finalised off the critical path)
template <int V, bool FWD>
__device__ __forceinline__ Vec<V> gather_val(const PassParams &p, int u, int64_t col) {
    if (u >= 0) return ldv_cg<V>(p.out + int64_t(u) * p.S + col);
    const int qb = -u - 1;
    const int np = __ldg(p.part_np + qb);
    Vec<V> a = ldv_cg<V>(p.part_buf + int64_t(qb) * p.S + col);
    for (int k = 1; k < np; ++k) {
        const Vec<V> b = ldv_cg<V>(p.part_buf + int64_t(qb + k) * p.S + col);
#pragma unroll
        for (int j = 0; j < V; ++j) a.x[j] = combine<FWD>(a.x[j], b.x[j]);
    }
    return a;
}

__device__ __forceinline__ int pieces_in(const PassParams &p, int k) {
    return __ldg(p.piece_off + k + 1) - __ldg(p.piece_off + k);
}

// ---- mbarrier / bulk-copy / named-barrier PTX ----------------------------------
__device__ __forceinline__ void mbar_init(uint64_t *bar, int count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(
                     smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    uint32_t ok = 0;
    while (!ok) {
        asm volatile(
            "{\n\t.reg .pred q;\n\t"
            "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 q, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, q;\n\t}"
            : "=r"(ok)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
    }
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes,
                                         uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void consumer_sync() {   // named barrier 1: consumer warps only
    asm volatile("bar.sync 1, %0;" ::"n"(NC) : "memory");
}

// One CTA per SM: warps NCW.. are producers (stage pieces into a NBUF-slot ring
// with TMA bulk copies, off the critical path); warps 0..NCW-1 compute.
template <int V, bool FWD, bool CHECK_D, bool BULK>
__global__ void __launch_bounds__(BLOCK, 1) k_propagate(PassParams p) {
    extern __shared__ __align__(128) unsigned char smem[];
    const SlotLayout SL = slot_layout(p.ncap, p.ecap, p.S);
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + NBUF * SL.bytes);
    uint64_t *empty = full + NBUF;
    float *s_part = reinterpret_cast<float *>(empty + NBUF);                  // [NC*V]
    int32_t *s_min = reinterpret_cast<int32_t *>(s_part + NC * V);           // [S]
    float *s_row = reinterpret_cast<float *>(s_min + p.S);                    // [S]
    __shared__ int s_nhub;
    __shared__ int s_hub[MAX_HUBS];

    const int tid = threadIdx.x;
    const int b = blockIdx.x;
    const int seq0 = __ldg(p.cta_off + b), nseq = __ldg(p.cta_off + b + 1) - seq0;
    if (tid == 0) {
        for (int s = 0; s < NBUF; ++s) {
            mbar_init(full + s, 32);
            mbar_init(empty + s, NCW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (!FWD)
        for (int s = tid; s < p.S; s += BLOCK) s_min[s] = 0x7f800000;
    __syncthreads();

    if (tid >= NC) {
        // ============================ producers (NPW warps) ============================
        // warp w stages pieces t = w, w + NPW, ...; every load of a piece depends only
        // on its (prefetched) descriptor, so rows, neighbour ids and edge ids are
        // fetched in one round of independent loads, then the delay rows follow as
        // TMA bulk copies completing on the slot's mbarrier.
        const int pw = (tid - NC) >> 5, lane = (tid - NC) & 31;
        int4 pcn = make_int4(0, 0, 0, 0);
        int lvn = 0;
        if (pw < nseq) {
            pcn = __ldg(p.cta_pc + seq0 + pw);
            lvn = __ldg(p.cta_lv + seq0 + pw);
        }
        for (int t = pw; t < nseq; t += NPW) {
            const int st = t % NBUF;
            const int4 pc = pcn;
            const int lvl = lvn;
            if (t + NPW < nseq) {   // prefetch the next descriptor
                pcn = __ldg(p.cta_pc + seq0 + t + NPW);
                lvn = __ldg(p.cta_lv + seq0 + t + NPW);
            }
            mbar_wait(empty + st, ((t / NBUF) & 1) ^ 1);
            unsigned char *sb = smem + st * SL.bytes;
            int32_t *meta = reinterpret_cast<int32_t *>(sb + SL.meta);
            int32_t *s_node = reinterpret_cast<int32_t *>(sb + SL.node);
            int32_t *s_rp = reinterpret_cast<int32_t *>(sb + SL.rp);
            int32_t *s_nbr = reinterpret_cast<int32_t *>(sb + SL.nbr);
            int32_t *s_mr = reinterpret_cast<int32_t *>(sb + SL.medrow);
            int32_t *s_mp = reinterpret_cast<int32_t *>(sb + SL.medpre);
            float *s_d = reinterpret_cast<float *>(sb + SL.d);
            const int pos0 = pc.x, nn = pc.y - pc.x, rb = pc.z, E = pc.w - pc.z;
            const int nst = min(nn, p.ncap), est = min(E, p.ecap);
            const int rounds = max((nst + 1 + 127) / 128, (est + 127) / 128);
            for (int r0 = 0; r0 < rounds; ++r0) {
                int nd[4], rpv[4], nb[4], ev[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {   // independent loads first
                    const int i = r0 * 128 + u * 32 + lane;
                    if (i < nst) nd[u] = __ldg(p.node_of + pos0 + i);
                    if (i <= nst) rpv[u] = __ldg(p.row_ptr + pos0 + i);
                    if (i < est) {
                        nb[u] = __ldg(p.nbr + rb + i);
                        ev[u] = __ldg(p.eid + rb + i);
                    }
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int i = r0 * 128 + u * 32 + lane;
                    if (i < nst) s_node[i] = nd[u];
                    if (i <= nst) s_rp[i] = rpv[u] - rb;
                    if (i < est) {
                        s_nbr[i] = nb[u];
                        const float *src = p.d + int64_t(ev[u]) * p.S;
                        if (BULK) {
                            bulk_g2s(s_d + int64_t(i) * p.S, src, uint32_t(p.S) * 4u, full + st);
                        } else {
                            for (int c = 0; c < p.S; ++c) s_d[int64_t(i) * p.S + c] = __ldg(src + c);
                        }
                    }
                }
            }
            __syncwarp();
            // part piece: one slice of a split row; else list the medium rows
            const bool part = nn == 1 && (s_rp[1] - s_rp[0]) > p.split;
            int nrow = 0, nchk = 0;
            if (!part) {
                for (int i0 = 0; i0 < nst; i0 += 32) {
                    const int i = i0 + lane;
                    int nch = 0;
                    if (i < nst) {
                        const int eb = s_rp[i], ee = s_rp[i + 1];
                        if (ee - eb > CH && ee - eb <= p.split && ee <= est)
                            nch = (ee - eb + CH - 1) / CH;
                    }
                    const unsigned mk = __ballot_sync(0xffffffffu, nch > 0);
                    if (mk == 0) continue;
                    int incl = nch;
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const int y = __shfl_up_sync(0xffffffffu, incl, o);
                        if (lane >= o) incl += y;
                    }
                    if (nch > 0) {
                        const int slot = nrow + __popc(mk & ((1u << lane) - 1u));
                        if (slot < MAXMED) {
                            s_mr[slot] = i;
                            s_mp[slot] = nchk + incl - nch;
                        }
                    }
                    nrow += __popc(mk);
                    nchk += __shfl_sync(0xffffffffu, incl, 31);
                }
                if (nrow > MAXMED) {   // cannot happen with ecap/CH <= MAXMED; stay correct
                    nrow = 0;
                    nchk = 0;
                }
            }
            if (lane == 0) {
                s_mp[nrow] = nchk;
                meta[MT_LV] = lvl;
                meta[MT_POS] = pos0;
                meta[MT_NN] = nn;
                meta[MT_RB] = rb;
                meta[MT_E] = E;
                meta[MT_EST] = est;
                meta[MT_NMED] = nrow;
                meta[MT_PART] = part;
                meta[MT_QB] = part ? __ldg(p.q + pos0) : 0;
            }
            __syncwarp();
            if (BULK && lane == 0)
                mbar_arrive_tx(full + st, uint32_t(est) * uint32_t(p.S) * 4u);
            else
                mbar_arrive(full + st);
        }
        return;
    }

    // ================================= consumers ==================================
    const int warp = tid >> 5, wl = tid & 31;
    const int lpn = p.S / V;                       // lanes per node row
    const int active = (NC / lpn) * lpn;           // threads with a fixed lane
    const int slots = active / lpn;                // rows handled side by side
    const int lane = tid % lpn;
    const int64_t col = int64_t(lane) * V;
    const bool pow2 = (lpn & (lpn - 1)) == 0;
    bool bad = false;
    Vec<V> run_min;
#pragma unroll
    for (int k = 0; k < V; ++k) run_min.x[k] = ident<false>();

    for (int t = 0; t < nseq; ++t) {
        const int st = t % NBUF;
        const unsigned long long t_top = p.trace ? gtimer() : 0;
        mbar_wait(full + st, (t / NBUF) & 1);
        unsigned char *sb = smem + st * SL.bytes;
        const int32_t *meta = reinterpret_cast<const int32_t *>(sb + SL.meta);
        const int32_t *s_node = reinterpret_cast<const int32_t *>(sb + SL.node);
        const int32_t *s_rp = reinterpret_cast<const int32_t *>(sb + SL.rp);
        const int32_t *s_nbr = reinterpret_cast<const int32_t *>(sb + SL.nbr);
        const int32_t *s_mr = reinterpret_cast<const int32_t *>(sb + SL.medrow);
        const int32_t *s_mp = reinterpret_cast<const int32_t *>(sb + SL.medpre);
        float *s_d = reinterpret_cast<float *>(sb + SL.d);
        const int kc = meta[MT_LV], pos0 = meta[MT_POS], nn = meta[MT_NN], rb = meta[MT_RB];
        const int E = meta[MT_E], est = meta[MT_EST], nmed = meta[MT_NMED];
        const bool part = meta[MT_PART] != 0;
        const int nst = min(nn, p.ncap);
        // split-row bookkeeping, read now: the slot is recycled once the piece publishes
        const int part_node = part ? s_node[0] : 0;
        const int part_qb = part ? meta[MT_QB] : 0;
        const int part_n = part ? (s_rp[1] - s_rp[0] + p.psize - 1) / p.psize : 0;

        // (a) backward: prefetch at[] of this thread's first four rows (for the slack)
        Vec<V> pre_at[4];
        if (!FWD && tid < active) {
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const int i = tid / lpn + r * slots;
                if (i < nst) pre_at[r] = ldv_cg<V>(p.other + int64_t(s_node[i]) * p.S + col);
            }
        }
        // (b) wait until the previous level (pass order) is fully published; a level
        // whose only piece was this CTA's needs no poll (named barriers order it)
        const int dep = FWD ? kc - 1 : kc + 1;
        if (tid == 0 && dep >= 0 && dep < p.L) {
            const int np = pieces_in(p, dep);
            if (!(np == 1 && b == 0)) {
                const int need = np;
                if (ld_acquire(p.done + dep) < need)
                    while (ld_acquire(p.done + dep) < need) __nanosleep(20);
            }
        }
        consumer_sync();
        const unsigned long long t_ready = p.trace ? gtimer() : 0;
        if (tid == 0) s_nhub = 0;

        // (c1) edge-parallel: x = fl(a[u] +/- d) in place over the staged delay; up to
        // four items per thread issue their gathers together (one L2 round trip)
        if (pow2) {
            const int estep = NC / lpn, e0 = tid / lpn;
            for (int eb = e0; eb < est; eb += 4 * estep) {
                Vec<V> a[4];
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    const int e = eb + r * estep;
                    if (e < est) a[r] = gather_val<V, FWD>(p, s_nbr[e], col);
                }
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    const int e = eb + r * estep;
                    if (e < est) {
                        float *dp = s_d + int64_t(e) * p.S + col;
                        const Vec<V> dd = ldv_s<V>(dp);
                        Vec<V> x;
#pragma unroll
                        for (int j = 0; j < V; ++j) {
                            float d1 = dd.x[j];
                            if (CHECK_D) {
                                bad |= !isfinite(d1);
                                d1 = canon0(d1);
                            }
                            x.x[j] = relax<FWD>(a[r].x[j], d1);
                        }
                        stv_s<V>(dp, x);
                    }
                }
            }
        } else {
            for (int q = tid; q < est * lpn; q += NC) {
                const int e = q / lpn, l = q - e * lpn;
                float *dp = s_d + int64_t(e) * p.S + l * V;
                const Vec<V> dd = ldv_s<V>(dp);
                const Vec<V> a = gather_val<V, FWD>(p, s_nbr[e], int64_t(l) * V);
                Vec<V> x;
#pragma unroll
                for (int j = 0; j < V; ++j) {
                    float d1 = dd.x[j];
                    if (CHECK_D) {
                        bad |= !isfinite(d1);
                        d1 = canon0(d1);
                    }
                    x.x[j] = relax<FWD>(a.x[j], d1);
                }
                stv_s<V>(dp, x);
            }
        }
        consumer_sync();

        auto node_at = [&](int i) { return i < nst ? s_node[i] : __ldg(p.node_of + pos0 + i); };
        auto rel = [&](int i) { return i <= nst ? s_rp[i] : __ldg(p.row_ptr + pos0 + i) - rb; };
        auto finish = [&](int node, const Vec<V> &best, int i) {
            stv_g<V>(p.out + int64_t(node) * p.S + col, best);
            if (!FWD) {
                const int rr = i >= 0 ? (i - tid / lpn) / slots : 4;
                const Vec<V> a = (rr < 4 && i < nst)
                                     ? (rr == 0   ? pre_at[0]
                                        : rr == 1 ? pre_at[1]
                                        : rr == 2 ? pre_at[2]
                                                  : pre_at[3])
                                     : ldv_cg<V>(p.other + int64_t(node) * p.S + col);
                Vec<V> sl;
#pragma unroll
                for (int j = 0; j < V; ++j) {
                    sl.x[j] = __fsub_rn(best.x[j], a.x[j]);
                    run_min.x[j] = fminf(run_min.x[j], sl.x[j]);
                }
                if (p.slack) stv_g<V>(p.slack + int64_t(node) * p.S + col, sl);
            }
        };
        // gather-reduce of unstaged edges [e, ee) with stride `step` (rare paths)
        auto tail = [&](int e, int ee, int step, Vec<V> &acc) {   // rare paths
            for (; e < ee; e += 2 * step) {
                Vec<V> a[2], dd[2];
#pragma unroll
                for (int r = 0; r < 2; ++r) {
                    const int er = e + r * step;
                    if (er < ee) {
                        const int ge = rb + er;
                        a[r] = gather_val<V, FWD>(p, __ldg(p.nbr + ge), col);
                        dd[r] = ldv_g<V>(p.d + int64_t(__ldg(p.eid + ge)) * p.S + col);
                    }
                }
#pragma unroll
                for (int r = 0; r < 2; ++r) {
                    if (e + r * step < ee) {
#pragma unroll
                        for (int j = 0; j < V; ++j) {
                            float d1 = dd[r].x[j];
                            if (CHECK_D) {
                                bad |= !isfinite(d1);
                                d1 = canon0(d1);
                            }
                            acc.x[j] = combine<FWD>(acc.x[j], relax<FWD>(a[r].x[j], d1));
                        }
                    }
                }
            }
        };

        if (part) {
            // (c1b) one slice of a split row: partial over the staged edges by all slots,
            // stored to the row's part buffer; the last slice to finish (atomic count)
            // combines all partials and writes the row -- exact, no float atomics
            const int node = s_node[0];
            const int slot = tid / lpn;
            const int deg = s_rp[1] - s_rp[0];
            const int nparts = (deg + p.psize - 1) / p.psize;
            const int pid = meta[MT_QB] + (-s_rp[0]) / p.psize;
            Vec<V> acc;
#pragma unroll
            for (int j = 0; j < V; ++j) acc.x[j] = ident<FWD>();
            if (tid < active)
                for (int e = slot; e < est; e += slots) {
                    const Vec<V> x = ldv_s<V>(s_d + int64_t(e) * p.S + col);
#pragma unroll
                    for (int j = 0; j < V; ++j) acc.x[j] = combine<FWD>(acc.x[j], x.x[j]);
                }
            stv_s<V>(s_part + int64_t(tid) * V, acc);
            consumer_sync();
            if (tid < lpn) {
                Vec<V> best = ldv_s<V>(s_part + int64_t(tid) * V);
                for (int s2 = 1; s2 < slots; ++s2) {
                    const Vec<V> q = ldv_s<V>(s_part + int64_t(s2 * lpn + tid) * V);
#pragma unroll
                    for (int j = 0; j < V; ++j) best.x[j] = combine<FWD>(best.x[j], q.x[j]);
                }
                if (nparts == 1) {   // the whole row: final value directly
                    stv_g<V>(p.out + int64_t(node) * p.S + col, best);
                    if (!FWD) {
                        const Vec<V> a = ldv_cg<V>(p.other + int64_t(node) * p.S + col);
                        Vec<V> sl;
#pragma unroll
                        for (int j = 0; j < V; ++j) {
                            sl.x[j] = __fsub_rn(best.x[j], a.x[j]);
                            run_min.x[j] = fminf(run_min.x[j], sl.x[j]);
                        }
                        if (p.slack) stv_g<V>(p.slack + int64_t(node) * p.S + col, sl);
                    }
                } else {   // readers combine the partials; finalised after the publish
                    stv_g<V>(p.part_buf + int64_t(pid) * p.S + col, best);
                }
            }
        } else {
            // (c1c) medium rows: every CH-edge chunk pre-reduced in place (partial over
            // the chunk's first edge) by all threads in parallel
            if (nmed > 0) {
                const int items = s_mp[nmed] * lpn;
                for (int q = tid; q < items; q += NC) {
                    const int c = q / lpn, l = q - c * lpn;
                    int lo = 0, hi = nmed - 1;   // last r with s_mp[r] <= c
                    while (lo < hi) {
                        const int mid = (lo + hi + 1) >> 1;
                        if (s_mp[mid] <= c) lo = mid;
                        else hi = mid - 1;
                    }
                    const int i = s_mr[lo];
                    const int eb = s_rp[i] + (c - s_mp[lo]) * CH;
                    const int ee = min(s_rp[i + 1], eb + CH);
                    float *dp = s_d + int64_t(eb) * p.S + l * V;
                    Vec<V> acc = ldv_s<V>(dp);
                    for (int e = eb + 1; e < ee; ++e) {
                        const Vec<V> x = ldv_s<V>(s_d + int64_t(e) * p.S + l * V);
#pragma unroll
                        for (int j = 0; j < V; ++j) acc.x[j] = combine<FWD>(acc.x[j], x.x[j]);
                    }
                    stv_s<V>(dp, acc);
                }
                consumer_sync();
            }
            // (c2) rows reduced by their owner lanes; unstaged long rows deferred
            if (tid < active) {
                for (int i = tid / lpn; i < nn; i += slots) {
                    const int eb = rel(i), ee = rel(i + 1);
                    const int deg = ee - eb;
                    if (deg > p.split) continue;   // split rows live in part pieces
                    const bool chunked = deg > CH && ee <= est && nmed > 0 && i < nst;
                    if (deg > HUB_DEG && ee > est) {
                        if (lane == 0) {
                            const int h = atomicAdd(&s_nhub, 1);
                            if (h < MAX_HUBS) s_hub[h] = i;
                            else atomicOr(p.err, 0x80000000u);
                        }
                        continue;
                    }
                    const int node = node_at(i);
                    Vec<V> best;
                    if (deg == 0) {
                        if (FWD) {
                            const float a0 = p.src_val ? canon0(__ldg(p.src_val + node)) : 0.0f;
#pragma unroll
                            for (int j = 0; j < V; ++j) best.x[j] = a0;
                        } else {
#pragma unroll
                            for (int j = 0; j < V; ++j)
                                best.x[j] =
                                    canon0(p.src_val ? __ldg(p.src_val + col + j) : p.t_scalar);
                        }
                    } else {
#pragma unroll
                        for (int j = 0; j < V; ++j) best.x[j] = ident<FWD>();
                        const int es = min(ee, est);
                        for (int e = eb; e < es; e += chunked ? CH : 1) {
                            const Vec<V> x = ldv_s<V>(s_d + int64_t(e) * p.S + col);
#pragma unroll
                            for (int j = 0; j < V; ++j) best.x[j] = combine<FWD>(best.x[j], x.x[j]);
                        }
                        if (ee > es) tail(max(eb, es), ee, 1, best);
                    }
                    finish(node, best, i);
                }
            }
            consumer_sync();
            // (c3) unstaged long rows: all slots, strided, shared-memory combine
            const int nhub = min(s_nhub, MAX_HUBS);
            for (int h = 0; h < nhub; ++h) {
                const int i = s_hub[h];
                const int eb = rel(i), ee = rel(i + 1);
                const int slot = tid / lpn;
                Vec<V> acc;
#pragma unroll
                for (int j = 0; j < V; ++j) acc.x[j] = ident<FWD>();
                if (tid < active) {
                    int e = eb + slot;
                    for (; e < ee && e < est; e += slots) {
                        const Vec<V> x = ldv_s<V>(s_d + int64_t(e) * p.S + col);
#pragma unroll
                        for (int j = 0; j < V; ++j) acc.x[j] = combine<FWD>(acc.x[j], x.x[j]);
                    }
                    tail(e, ee, slots, acc);
                }
                stv_s<V>(s_part + int64_t(tid) * V, acc);
                consumer_sync();
                if (tid < lpn) {
                    Vec<V> best = ldv_s<V>(s_part + int64_t(tid) * V);
                    for (int s2 = 1; s2 < slots; ++s2) {
                        const Vec<V> q = ldv_s<V>(s_part + int64_t(s2 * lpn + tid) * V);
#pragma unroll
                        for (int j = 0; j < V; ++j) best.x[j] = combine<FWD>(best.x[j], q.x[j]);
                    }
                    finish(node_at(i), best, -1);
                }
                consumer_sync();
            }
        }
        // (d) publish: every warp releases its stores at gpu scope, the slot goes back
        // to the producer, and one thread counts the piece after all warps fenced
        const unsigned long long t_comp = p.trace ? gtimer() : 0;
        __syncwarp();
        if (wl == 0) {
            asm volatile("fence.acq_rel.gpu;" ::: "memory");
            mbar_arrive(empty + st);
        }
        consumer_sync();
        if (tid == 0) atomicAdd(p.done + kc, 1);
        // split rows (>= 2 parts) are finalised by k_finalize_split after the pass;
        // readers inside the pass combine their partials
        if (p.trace && tid == 0) {
            const int r = atomicAdd(p.trace_n, 1);
            if (r < p.trace_cap) {
                unsigned long long *tr = p.trace + int64_t(r) * 8;
                tr[0] = (unsigned long long)kc;
                tr[1] = (unsigned long long)b;
                tr[2] = t_top;
                tr[3] = t_ready;
                tr[4] = t_comp;
                tr[5] = gtimer();
                tr[6] = (unsigned long long)E;
                tr[7] = (unsigned long long)nn;
            }
        }
    }

    if (CHECK_D && bad) atomicOr(p.err, ERR_NONFINITE);
    if (!FWD) {
        if (tid < active) {
#pragma unroll
            for (int j = 0; j < V; ++j)
                if (run_min.x[j] != ident<false>())
                    atomicMin(s_min + col + j, f2ord(run_min.x[j]));
        }
        consumer_sync();
        for (int s = tid; s < p.S; s += NC)
            if (s_min[s] != 0x7f800000) atomicMin(p.wns_ord + s, s_min[s]);
    }
}

// After a pass: every row cut into >= 2 part pieces gets its value (combine of the
// partials), its optional slack and its worst-slack contribution.  One warp per
// split row; the rows are the positions with degree > split and > psize.
template <bool FWD>
__global__ void k_finalize_split(const int32_t *__restrict__ rows, const int32_t *__restrict__ nrows,
                                 const int32_t *__restrict__ row_ptr,
                                 const int32_t *__restrict__ node_of, const int32_t *__restrict__ q,
                                 int32_t psize, int32_t S, const float *__restrict__ part_buf,
                                 float *__restrict__ out, const float *__restrict__ other,
                                 float *__restrict__ slack, int32_t *__restrict__ wns_ord) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
    const int cnt = *nrows;
    for (int64_t r = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5; r < cnt; r += nw) {
        const int i = rows[r];
        const int d = row_ptr[i + 1] - row_ptr[i];
        const int np = (d + psize - 1) / psize, qb = q[i];
        const int64_t node = node_of[i];
        for (int s = lane; s < S; s += 32) {
            float v = part_buf[int64_t(qb) * S + s];
            for (int k = 1; k < np; ++k) v = combine<FWD>(v, part_buf[int64_t(qb + k) * S + s]);
            out[node * S + s] = v;
            if (!FWD) {
                const float sl = __fsub_rn(v, other[node * S + s]);
                if (slack) slack[node * S + s] = sl;
                atomicMin(wns_ord + s, f2ord(sl));
            }
        }
    }
}

// positions of the rows cut into >= 2 parts (read through their partials)
__global__ void k_split_list(const int32_t *__restrict__ row_ptr, int32_t n, int32_t split,
                             int32_t psize, int32_t *__restrict__ rows, int32_t *__restrict__ cnt) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x) {
        const int d = row_ptr[i + 1] - row_ptr[i];
        if (d > split && d > psize) rows[atomicAdd(cnt, 1)] = int(i);
    }
}

// Backward sinks (out-degree 0) do not depend on any level: rat = T_s, their
// slack and worst-slack contribution, in one bandwidth-bound sweep before the pass.
template <int V>
__global__ void k_bwd_sinks(const int32_t *__restrict__ out_ptr, int32_t n, int32_t S,
                            const float *__restrict__ t_arr, float t_scalar,
                            const float *__restrict__ at, float *__restrict__ rat,
                            float *__restrict__ slack, int32_t *__restrict__ wns_ord) {
    extern __shared__ int32_t s_wmin[];
    for (int s = threadIdx.x; s < S; s += blockDim.x) s_wmin[s] = 0x7f800000;
    __syncthreads();
    const int lpn = S / V;
    const int apb = blockDim.x / lpn * lpn;                 // active threads per block
    const int64_t step = int64_t(gridDim.x) * apb;          // a multiple of lpn: lane fixed
    const int64_t t0 = blockIdx.x * int64_t(apb) + threadIdx.x;
    const int lane = int(threadIdx.x % lpn);
    float mn[V];
#pragma unroll
    for (int j = 0; j < V; ++j) mn[j] = __int_as_float(0x7f800000);
    if (int(threadIdx.x) < apb) {
        for (int64_t t = t0; t < int64_t(n) * lpn; t += step) {
            const int64_t v = t / lpn;
            if (out_ptr[v + 1] != out_ptr[v]) continue;
            const int64_t o = v * S + int64_t(lane) * V;
            Vec<V> r, a, sl;
#pragma unroll
            for (int j = 0; j < V; ++j)
                r.x[j] = canon0(t_arr ? __ldg(t_arr + lane * V + j) : t_scalar);
            stv_g<V>(rat + o, r);
            a = ldv_cg<V>(at + o);
#pragma unroll
            for (int j = 0; j < V; ++j) {
                sl.x[j] = __fsub_rn(r.x[j], a.x[j]);
                mn[j] = fminf(mn[j], sl.x[j]);
            }
            if (slack) stv_g<V>(slack + o, sl);
        }
#pragma unroll
        for (int j = 0; j < V; ++j)
            if (mn[j] != __int_as_float(0x7f800000)) atomicMin(s_wmin + lane * V + j, f2ord(mn[j]));
    }
    __syncthreads();
    for (int s = threadIdx.x; s < S; s += blockDim.x)
        if (s_wmin[s] != 0x7f800000) atomicMin(wns_ord + s, s_wmin[s]);
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

__global__ void k_check_t(const float *__restrict__ t, int32_t S, uint32_t *err) {
    for (int i = threadIdx.x; i < S; i += blockDim.x)
        if (!isfinite(t[i])) atomicOr(err, ERR_NONFINITE);
}

// ---- piece schedule (per direction; cached per (P, weights, split)) -----------
// Rows of a level are in ascending degree, so the split rows (degree > split) form
// the tail [le_normal, le) of every level.  Normal rows get weight degree + 1 and
// are cut into weight-balanced pieces; a split row becomes ceil(deg/split) part
// pieces of <= split edges each.
// weight of a row: 2 per edge (delay + gather) + rw for the row itself (forward:
// the at store; backward: rat store + at read for the slack)
__global__ void k_piece_rows(const int32_t *__restrict__ row_ptr, int32_t n, int32_t split,
                             int32_t psize, int32_t rw, int32_t *__restrict__ w,
                             int32_t *__restrict__ parts) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x) {
        const int d = row_ptr[i + 1] - row_ptr[i];
        w[i] = d > split ? 0 : 2 * d + rw;
        parts[i] = d > split ? (d + psize - 1) / psize : 0;
    }
}
__global__ void k_piece_count(const int32_t *__restrict__ level_ptr, const int32_t *__restrict__ W,
                              const int32_t *__restrict__ Q, const int32_t *__restrict__ row_ptr,
                              int32_t L, int32_t P, int32_t ecap, int32_t ncap, int32_t wt_min,
                              int32_t split, int32_t rw, int32_t skip0, int32_t *__restrict__ np,
                              int32_t *__restrict__ npn, int32_t *__restrict__ lsnorm,
                              int32_t *__restrict__ lenorm) {
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < L; k += gridDim.x * blockDim.x) {
        int ls = level_ptr[k];
        const int le = level_ptr[k + 1];
        if (skip0) {   // degree-0 rows (backward sinks) are done by k_bwd_sinks
            int a = ls, z = le;
            while (a < z) {
                const int mid = (a + z) >> 1;
                if (row_ptr[mid + 1] - row_ptr[mid] > 0) z = mid;
                else a = mid + 1;
            }
            ls = a;
        }
        int lo = ls, hi = le;   // first row with degree > split
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (row_ptr[mid + 1] - row_ptr[mid] > split) hi = mid;
            else lo = mid + 1;
        }
        const int64_t wk = int64_t(W[lo]) - W[ls];   // 2*edges + rw*rows, normal rows
        const int64_t nk = lo - ls;
        const int64_t ek = (wk - rw * nk) / 2;
        const int parts = Q[le] - Q[ls];
        int64_t c = 0;
        if (nk > 0) {
            // enough pieces to fit a ring slot (3/4 of its edge and row capacity), else
            // one per CTA left after the part pieces, so a level is a single round
            const int64_t need = std::max<int64_t>((ek * 4 + 3 * ecap - 1) / (3 * ecap),
                                                   (nk * 4 + 3 * ncap - 1) / (3 * ncap));
            c = std::max<int64_t>(need, std::min<int64_t>(std::max(1, P - parts),
                                                          (wk + wt_min - 1) / wt_min));
            c = std::max<int64_t>(1, std::min<int64_t>(nk, c));
        }
        if (c + parts == 0) c = 1;   // keep one (empty) piece: levels publish in order
        npn[k] = int(c);
        lsnorm[k] = ls;
        lenorm[k] = lo;
        np[k] = int(c) + parts;
    }
}
// normal piece j of level k starts at the first row whose weight prefix reaches j*W_k/np_k
__global__ void k_piece_fill(const int32_t *__restrict__ lsnorm, const int32_t *__restrict__ W,
                             const int32_t *__restrict__ row_ptr, const int32_t *__restrict__ off,
                             const int32_t *__restrict__ npn, const int32_t *__restrict__ lenorm,
                             int32_t L, int4 *__restrict__ pieces) {
    for (int k = blockIdx.x; k < L; k += gridDim.x) {
        const int ls = lsnorm[k], le = lenorm[k];
        const int np = npn[k];
        const int64_t w0 = W[ls], wk = int64_t(W[le]) - w0;
        auto start_of = [&](int jj) {
            if (jj >= np) return le;
            if (jj == 0) return ls;
            const int64_t target = w0 + wk * jj / np;
            int lo = ls, hi = le;   // first i in [ls, le] with W[i] >= target
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if (W[mid] >= target) hi = mid;
                else lo = mid + 1;
            }
            return lo;
        };
        for (int j = threadIdx.x; j < np; j += blockDim.x) {
            const int a = start_of(j), z = start_of(j + 1);
            pieces[off[k] + j] = make_int4(a, z, row_ptr[a], row_ptr[z]);
        }
    }
}
__global__ void k_piece_parts(const int32_t *__restrict__ row_ptr, const int32_t *__restrict__ node_of,
                              const int32_t *__restrict__ level, const int32_t *__restrict__ level_ptr,
                              const int32_t *__restrict__ Q, const int32_t *__restrict__ off,
                              const int32_t *__restrict__ npn, int32_t n, int32_t split,
                              int32_t psize, int4 *__restrict__ pieces) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x) {
        const int rb = row_ptr[i], re = row_ptr[i + 1];
        if (re - rb <= split) continue;
        const int k = level[node_of[i]];
        const int base = off[k] + npn[k] + (Q[i] - Q[level_ptr[k]]);
        for (int t = 0; rb + t * psize < re; ++t)
            pieces[base + t] = make_int4(int(i), int(i) + 1, rb + t * psize,
                                         min(re, rb + (t + 1) * psize));
    }
}
// neighbour ids with split rows encoded as -(first part id + 1), and parts per row
__global__ void k_pos_of(const int32_t *__restrict__ node_of, int32_t n, int32_t *__restrict__ pos) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x)
        pos[node_of[i]] = int(i);
}
__global__ void k_part_np(const int32_t *__restrict__ row_ptr, const int32_t *__restrict__ Q,
                          int32_t n, int32_t split, int32_t psize, int32_t *__restrict__ part_np) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x) {
        const int d = row_ptr[i + 1] - row_ptr[i];
        if (d > split) part_np[Q[i]] = (d + psize - 1) / psize;
    }
}
__global__ void k_nbr_enc(const int32_t *__restrict__ nbr, int32_t m, const int32_t *__restrict__ pos,
                          const int32_t *__restrict__ row_ptr, const int32_t *__restrict__ Q,
                          int32_t split, int32_t psize, int32_t *__restrict__ enc) {
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < m;
         e += int64_t(gridDim.x) * blockDim.x) {
        const int v = nbr[e];
        const int i = pos[v];
        const int d = row_ptr[i + 1] - row_ptr[i];
        // only rows cut into >= 2 parts are read through their partials
        enc[e] = (d > split && d > psize) ? -(Q[i] + 1) : v;
    }
}

void build_pieces(Graph &g, const int32_t *row_ptr, const int32_t *node_of, const int32_t *nbr,
                  int P, int ecap, int ncap, int wt_min, int split, int psize, int rw,
                  int skip0, PieceSched &ps) {
    cudaStream_t s = g.stream;
    const int32_t n = g.n, L = g.L;
    DevBuf w, W, q, np, npn, lsnorm, lenorm;
    DevBuf &Q = ps.q, &off = ps.off, &pieces = ps.pieces;
    w.alloc(sizeof(int32_t) * (int64_t(n) + 1), s);
    W.alloc(sizeof(int32_t) * (int64_t(n) + 1), s);
    q.alloc(sizeof(int32_t) * (int64_t(n) + 1), s);
    Q.alloc(sizeof(int32_t) * (int64_t(n) + 1), s);
    np.alloc(sizeof(int32_t) * (int64_t(L) + 1), s);
    npn.alloc(sizeof(int32_t) * (int64_t(L) + 1), s);
    lenorm.alloc(sizeof(int32_t) * (int64_t(L) + 1), s);
    lsnorm.alloc(sizeof(int32_t) * (int64_t(L) + 1), s);
    off.alloc(sizeof(int32_t) * (int64_t(L) + 1), s);
    HF_CUDA(cudaMemsetAsync(w.as<int32_t>() + n, 0, sizeof(int32_t), s));
    HF_CUDA(cudaMemsetAsync(q.as<int32_t>() + n, 0, sizeof(int32_t), s));
    HF_CUDA(cudaMemsetAsync(np.as<int32_t>() + L, 0, sizeof(int32_t), s));
    k_piece_rows<<<grid_for(n, 256, g.sms), 256, 0, s>>>(row_ptr, n, split, psize, rw,
                                                         w.as<int32_t>(), q.as<int32_t>());
    HF_CHECK_LAUNCH();
    scan_exclusive(w.as<int32_t>(), W.as<int32_t>(), int64_t(n) + 1, nullptr, s, g);
    scan_exclusive(q.as<int32_t>(), Q.as<int32_t>(), int64_t(n) + 1, nullptr, s, g);
    k_piece_count<<<grid_for(L, 256, g.sms), 256, 0, s>>>(
        g.level_ptr.as<int32_t>(), W.as<int32_t>(), Q.as<int32_t>(), row_ptr, L, P, ecap, ncap,
        wt_min, split, rw, skip0, np.as<int32_t>(), npn.as<int32_t>(), lsnorm.as<int32_t>(),
        lenorm.as<int32_t>());
    HF_CHECK_LAUNCH();
    scan_exclusive(np.as<int32_t>(), off.as<int32_t>(), int64_t(L) + 1, nullptr, s, g);
    int32_t total = 0;
    HF_CUDA(cudaMemcpyAsync(&total, off.as<int32_t>() + L, sizeof(int32_t), cudaMemcpyDeviceToHost,
                            s));
    HF_CUDA(cudaMemcpyAsync(&ps.nparts, Q.as<int32_t>() + n, sizeof(int32_t),
                            cudaMemcpyDeviceToHost, s));
    HF_CUDA(cudaStreamSynchronize(s));
    pieces.alloc(sizeof(int4) * size_t(std::max(total, 1)), s);
    k_piece_fill<<<int(std::min<int64_t>(L, 65535)), 128, 0, s>>>(
        lsnorm.as<int32_t>(), W.as<int32_t>(), row_ptr, off.as<int32_t>(),
        npn.as<int32_t>(), lenorm.as<int32_t>(), L, pieces.as<int4>());
    HF_CHECK_LAUNCH();
    k_piece_parts<<<grid_for(n, 256, g.sms), 256, 0, s>>>(
        row_ptr, node_of, g.level.as<int32_t>(), g.level_ptr.as<int32_t>(), Q.as<int32_t>(),
        off.as<int32_t>(), npn.as<int32_t>(), n, split, psize, pieces.as<int4>());
    HF_CHECK_LAUNCH();
    // neighbours that are split rows, and the part count of every split row
    const int32_t m = g.m;
    ps.nbr_enc.alloc(sizeof(int32_t) * size_t(m > 0 ? m : 1), s);
    ps.part_np.alloc(sizeof(int32_t) * size_t(std::max(ps.nparts, 1)), s);
    if (ps.nparts == 0) {
        if (m)
            HF_CUDA(cudaMemcpyAsync(ps.nbr_enc.p, nbr, sizeof(int32_t) * size_t(m),
                                    cudaMemcpyDeviceToDevice, s));
    } else {
        DevBuf pos;
        pos.alloc(sizeof(int32_t) * size_t(n), s);
        k_pos_of<<<grid_for(n, 256, g.sms), 256, 0, s>>>(node_of, n, pos.as<int32_t>());
        HF_CHECK_LAUNCH();
        k_part_np<<<grid_for(n, 256, g.sms), 256, 0, s>>>(row_ptr, Q.as<int32_t>(), n, split,
                                                          psize, ps.part_np.as<int32_t>());
        HF_CHECK_LAUNCH();
        ps.split_rows.alloc(sizeof(int32_t) * (size_t(ps.nparts) + 1), s);
        HF_CUDA(cudaMemsetAsync(ps.split_rows.p, 0, sizeof(int32_t), s));
        k_split_list<<<grid_for(n, 256, g.sms), 256, 0, s>>>(
            row_ptr, n, split, psize, ps.split_rows.as<int32_t>() + 1, ps.split_rows.as<int32_t>());
        HF_CHECK_LAUNCH();
        g.launches += 1;
        if (m) {
            k_nbr_enc<<<grid_for(m, 256, g.sms), 256, 0, s>>>(nbr, m, pos.as<int32_t>(), row_ptr,
                                                              Q.as<int32_t>(), split, psize,
                                                              ps.nbr_enc.as<int32_t>());
            HF_CHECK_LAUNCH();
        }
        g.launches += 3;
    }
    g.launches += 5;
}

__global__ void k_gather_pieces(const int4 *__restrict__ pieces, const int32_t *__restrict__ idx,
                                int32_t total, int4 *__restrict__ out) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total;
         i += int64_t(gridDim.x) * blockDim.x)
        out[i] = pieces[idx[i]];
}

// Deal piece j of every level to CTA j mod P and lay each CTA's pieces out
// contiguously in pass order, so a CTA walks its schedule with sequential loads.
template <bool FWD> void deal_pieces(Graph &g, PieceSched &ps) {
    cudaStream_t s = g.stream;
    const int L = g.L, P = g.sms;
    std::vector<int32_t> off(size_t(L) + 1);
    HF_CUDA(cudaMemcpyAsync(off.data(), ps.off.p, sizeof(int32_t) * off.size(),
                            cudaMemcpyDeviceToHost, s));
    HF_CUDA(cudaStreamSynchronize(s));
    const int32_t total = off[L];
    std::vector<int32_t> cnt(size_t(P) + 1, 0), idx(size_t(std::max(total, 1))),
        lv(size_t(std::max(total, 1)));
    for (int k = 0; k < L; ++k)
        for (int j = 0; j < off[k + 1] - off[k]; ++j) cnt[size_t(j % P) + 1]++;
    for (int c = 0; c < P; ++c) cnt[c + 1] += cnt[c];
    std::vector<int32_t> cur(cnt.begin(), cnt.end() - 1);
    for (int kk = 0; kk < L; ++kk) {
        const int k = FWD ? kk : L - 1 - kk;
        for (int j = 0; j < off[k + 1] - off[k]; ++j) {
            const int c = j % P;
            idx[cur[c]] = off[k] + j;
            lv[cur[c]] = k;
            ++cur[c];
        }
    }
    DevBuf d_idx;
    d_idx.alloc(sizeof(int32_t) * idx.size(), s);
    ps.cta_lv.alloc(sizeof(int32_t) * lv.size(), s);
    ps.cta_off.alloc(sizeof(int32_t) * cnt.size(), s);
    ps.cta_pc.alloc(sizeof(int4) * idx.size(), s);
    HF_CUDA(cudaMemcpyAsync(d_idx.p, idx.data(), sizeof(int32_t) * idx.size(),
                            cudaMemcpyHostToDevice, s));
    HF_CUDA(cudaMemcpyAsync(ps.cta_lv.p, lv.data(), sizeof(int32_t) * lv.size(),
                            cudaMemcpyHostToDevice, s));
    HF_CUDA(cudaMemcpyAsync(ps.cta_off.p, cnt.data(), sizeof(int32_t) * cnt.size(),
                            cudaMemcpyHostToDevice, s));
    if (total > 0) {
        k_gather_pieces<<<grid_for(total, 256, g.sms), 256, 0, s>>>(
            ps.pieces.as<int4>(), d_idx.as<int32_t>(), total, ps.cta_pc.as<int4>());
        HF_CHECK_LAUNCH();
        g.launches += 1;
    }
    HF_CUDA(cudaStreamSynchronize(s));   // host vectors go out of scope
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

void prof_record(Graph &g, int idx) {
    if (g.prof) HF_CUDA(cudaEventRecord(g.ev[idx], g.stream));
}

template <int V, bool FWD, bool CHECK_D, bool VEC16>
void launch(Graph &g, PassParams &p, size_t smem) {
    auto kern = k_propagate<V, FWD, CHECK_D, VEC16>;
    HF_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    int per_sm = 0;
    HF_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, BLOCK, smem));
    if (per_sm < 1) fail(HF_ERR_CUDA, "propagation kernel does not fit on an SM");
    void *args[] = {&p};
    // one CTA per SM; the piece schedule was built for exactly g.sms CTAs.  With
    // profiling on, events bracket exactly this launch (forward: ev 2/3, backward 5/4).
    prof_record(g, FWD ? 2 : 5);
    HF_CUDA(cudaLaunchCooperativeKernel((const void *)kern, g.sms, BLOCK, args, smem, g.stream));
    prof_record(g, FWD ? 3 : 4);
    g.launches += 1;
}

constexpr int SMEM_BUDGET = 200 * 1024;

inline float __int_as_float_host(uint32_t b) {
    float f;
    memcpy(&f, &b, 4);
    return f;
}

template <bool FWD> void run_pass(Graph &g, PassParams &p, bool check_d, int V) {
    if (p.S / V > NC) fail(HF_ERR_INVALID_ARG, "too many scenarios for one pass (S/V > 512)");
    // staging capacity per ring slot: ecap edges of S floats (+ id), ncap rows
    const int fixed = 2 * NBUF * 8 + NC * 4 * 4 + 2 * p.S * 4;
    const int per_slot = (SMEM_BUDGET - fixed) / NBUF - 2 * MAXMED * 4 - 256;
    if (per_slot < 2048) fail(HF_ERR_INVALID_ARG, "too many scenarios for one pass");
    int ecap = std::min(std::min(4096, CH * MAXMED),
                        std::max(8, (per_slot - 256 * 8) / (4 + 4 * p.S)));
    int ncap = std::min(2048, std::max(16, (per_slot - ecap * (4 + 4 * p.S)) / 8 - 2));
    p.ecap = ecap;
    p.ncap = ncap;
    const int wt_min = 32;
    const int split = std::max(32, ecap / 4);
    p.split = split;
    p.psize = ecap;
    PieceSched &ps = FWD ? g.ps_f : g.ps_b;
    const int32_t want = (ecap * 4096 + ncap) * 8 + (g.sms & 7);
    if (ps.key != want || !ps.pieces.p) {
        build_pieces(g, p.row_ptr, p.node_of, p.nbr, g.sms, ecap, ncap, wt_min, split, ecap,
                     FWD ? 1 : 2, FWD ? 0 : 1, ps);
        deal_pieces<FWD>(g, ps);
        ps.key = want;
    }
    p.cta_pc = ps.cta_pc.as<int4>();
    p.cta_lv = ps.cta_lv.as<int32_t>();
    p.cta_off = ps.cta_off.as<int32_t>();
    p.piece_off = ps.off.as<int32_t>();
    p.q = ps.q.as<int32_t>();
    p.nbr = ps.nbr_enc.as<int32_t>();   // split-row neighbours encoded
    p.part_np = ps.part_np.as<int32_t>();
    DevBuf part_buf;
    if (ps.nparts > 0) {
        part_buf.alloc(sizeof(float) * size_t(ps.nparts) * p.S, g.stream);
        p.part_buf = part_buf.as<float>();
    }
    p.L = g.L;
    const SlotLayout SL = slot_layout(ncap, ecap, p.S);
    const size_t smem = size_t(NBUF) * SL.bytes + size_t(fixed);
    g.ws_sync.alloc(sizeof(int32_t) * (size_t(g.L) + 1), g.stream);   // warps published per level
    HF_CUDA(cudaMemsetAsync(g.ws_sync.p, 0, sizeof(int32_t) * (size_t(g.L) + 1), g.stream));
    p.done = g.ws_sync.as<int32_t>();
    p.err = g.d_err();
    // TMA bulk copies need 16-byte rows and 16-byte aligned sources
    const bool vec16 = (p.S % 4 == 0) && (reinterpret_cast<uintptr_t>(p.d) % 16 == 0);
    // debugging timeline: HF_TRACE=<file prefix> dumps one record per piece
    const char *trace_env = getenv("HF_TRACE");
    DevBuf tbuf;
    const int tcap = 1 << 20;
    if (trace_env) {
        tbuf.alloc(sizeof(unsigned long long) * 8 * tcap + 16, g.stream);
        HF_CUDA(cudaMemsetAsync(tbuf.p, 0, 16, g.stream));
        p.trace_n = reinterpret_cast<int32_t *>(tbuf.as<unsigned char>());
        p.trace = reinterpret_cast<unsigned long long *>(tbuf.as<unsigned char>() + 16);
        p.trace_cap = tcap;
    }
#define HF_LAUNCH(VV)                                                            \
    do {                                                                         \
        if (check_d && vec16) launch<VV, FWD, true, true>(g, p, smem);           \
        else if (check_d) launch<VV, FWD, true, false>(g, p, smem);              \
        else if (vec16) launch<VV, FWD, false, true>(g, p, smem);                \
        else launch<VV, FWD, false, false>(g, p, smem);                          \
    } while (0)
    if (V == 4) HF_LAUNCH(4);
    else if (V == 2) HF_LAUNCH(2);
    else HF_LAUNCH(1);
#undef HF_LAUNCH
    if (ps.nparts > 0) {
        k_finalize_split<FWD><<<g.sms, 256, 0, g.stream>>>(
            ps.split_rows.as<int32_t>() + 1, ps.split_rows.as<int32_t>(), p.row_ptr, p.node_of,
            p.q, p.psize, p.S, p.part_buf, p.out, p.other, p.slack, p.wns_ord);
        HF_CHECK_LAUNCH();
        g.launches += 1;
    }
    if (trace_env) {
        int32_t cnt = 0;
        HF_CUDA(cudaMemcpyAsync(&cnt, p.trace_n, 4, cudaMemcpyDeviceToHost, g.stream));
        HF_CUDA(cudaStreamSynchronize(g.stream));
        cnt = std::min(cnt, tcap);
        std::vector<unsigned long long> h(size_t(cnt) * 8);
        HF_CUDA(cudaMemcpy(h.data(), p.trace, h.size() * 8, cudaMemcpyDeviceToHost));
        std::string fn = std::string(trace_env) + (FWD ? "_fwd_S" : "_bwd_S") + std::to_string(p.S) +
                         ".bin";
        if (FILE *f = fopen(fn.c_str(), "wb")) {
            fwrite(h.data(), 8, h.size(), f);
            fclose(f);
        }
    }
}

}  // namespace

// Forward over all levels (device pointers).  d: [m][S].
void forward_device(Graph &g, const float *d, int32_t S, bool check_d, const float *at_src,
                    float *at) {
    if (g.n == 0) return;
    PassParams p{};
    const int V = pick_vec(S, {d, at});
    p.row_ptr = g.lo_in_ptr.as<int32_t>();
    p.nbr = g.lo_in_src.as<int32_t>();
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
    if (t_arr) {
        k_check_t<<<1, 256, 0, s>>>(t_arr, S, g.d_err());
        HF_CHECK_LAUNCH();
        g.launches += 1;
    }
    if (g.n > 0) {
        PassParams p{};
        const int V = pick_vec(S, {d, at, rat, slack});
        p.row_ptr = g.lo_out_ptr.as<int32_t>();
        p.nbr = g.lo_out_dst.as<int32_t>();
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
        // sinks first (independent of every level); the pass skips them
        const int lpn = S / V;
        const int grid = grid_for(int64_t(g.n) * lpn, 512, g.sms);
        const size_t sm = sizeof(int32_t) * size_t(S);
        if (sm > 48 * 1024) fail(HF_ERR_INVALID_ARG, "too many scenarios");
        if (V == 4)
            k_bwd_sinks<4><<<grid, 512, sm, s>>>(g.out_ptr.as<int32_t>(), g.n, S, t_arr, t_scalar,
                                                 at, rat, slack, ord);
        else if (V == 2)
            k_bwd_sinks<2><<<grid, 512, sm, s>>>(g.out_ptr.as<int32_t>(), g.n, S, t_arr, t_scalar,
                                                 at, rat, slack, ord);
        else
            k_bwd_sinks<1><<<grid, 512, sm, s>>>(g.out_ptr.as<int32_t>(), g.n, S, t_arr, t_scalar,
                                                 at, rat, slack, ord);
        HF_CHECK_LAUNCH();
        g.launches += 1;
        run_pass<false>(g, p, false, V);
    }
    if (wns_f) {
        k_ord_to_float<<<1, 256, 0, s>>>(ord, wns_f, S);
        HF_CHECK_LAUNCH();
        g.launches += 1;
    }
}

void profile_mark(Graph &g, int idx) { prof_record(g, idx); }

}  // namespace hf
