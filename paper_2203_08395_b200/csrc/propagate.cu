// propagate.cu -- forward max-plus and backward min-plus (+ fused slack / worst
// slack) over the levelized DAG, for one delay set or S scenario sets.
// SURVEY.md §8(a) a5-a7; BASELINE.json:5.
//
// Data layout in HBM (scenario-minor): at[v*S + s], rat[v*S + s],
// delays[e*S + s].  A node's S values are contiguous, so each edge touches S*4
// contiguous bytes; a node-slice of Sg scenarios is owned by LPN = Sg/V lanes
// holding V-wide vectors (V = 4 -> LDG.128 / STG.128).  Pull-based, no float
// atomics: every output is one fp32 max/min over fl(x +/- d) terms, which is
// order-independent (0 ULP against the oracle, reading R10).
//
// One persistent, warp-specialised launch per pass (no per-level launches, no
// grid barrier):
//   * Work = chunks of consecutive nodes of one level (level order forward,
//     reverse level order backward), sized by "vslots" (a node of degree d needs
//     ceil(d/PF) vslots of <= PF edges) so chunks are edge-balanced; hub nodes
//     get a chunk of their own.  CTAs claim chunks with an atomic ticket; a chunk
//     only waits on chunks with smaller tickets, held by running CTAs, so the
//     schedule is deadlock-free at any grid size.
//   * Producer warp: claims tickets up to NB chunks ahead, loads the chunk's
//     level-ordered CSR rows, builds the vslot table and stages every edge's
//     neighbour id and delay slice in shared memory with cp.async.bulk (TMA bulk
//     copies, completion on an mbarrier).  None of this depends on earlier levels,
//     so the HBM stream of delays runs ahead of the dependency front.
//   * Consumer warps: wait for the stage (mbarrier), then for the previous level
//     (one acquire-poll of its per-level chunk counter), gather at[u] / rat[v]
//     from L2, reduce each vslot in registers, combine a node's vslots through
//     shared memory, store, fence, and publish (release) the chunk.  Level k
//     complete => all earlier levels complete, by induction.
//   * Backward fuses slack = rat - at and keeps a per-lane running min; one
//     shared-memory reduction and one global atomicMin per scenario per CTA give
//     the worst slack.
#include <algorithm>

#include "common.cuh"

namespace hf {

namespace {

constexpr int NCW = 8;                     // consumer warps
constexpr int NCT = NCW * 32;              // consumer threads
constexpr int BLOCK = NCT + 32;            // + 1 producer warp
constexpr int PF = 4;                      // edges per vslot
constexpr int NB = 4;                      // pipeline stages

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
template <int V> __device__ __forceinline__ Vec<V> ldv_s(const float *p) {   // shared
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

// ---- PTX helpers: acquire load, mbarrier, bulk copy, named barrier ----------
__device__ __forceinline__ int ld_acquire(const int *p) {
    int v;
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
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
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
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
    asm volatile("bar.sync 1, %0;" ::"n"(NCT) : "memory");
}

struct PassParams {
    // level-ordered CSR of this direction: row i <-> node node_of[i]
    const int32_t *row_ptr;    // [n+1]
    const int32_t *nbr;        // [m] neighbour node id (fan-in src / fan-out dst)
    const int32_t *eid;        // [m] edge id (delay row)
    const int32_t *node_of;    // [n]
    const int32_t *chunk_pos;  // [C+1] first position of every chunk (+ n)
    const int32_t *chunk_ptr;  // [L+1] first chunk of every level
    int32_t L, C, G;           // levels, chunks, scenario groups
    int32_t T;                 // vslots per chunk target (= consumer slots)
    int32_t ecap;              // staged edges per stage
    int32_t S, Sg;             // row stride (scenarios), scenarios per group
    const float *d;            // [m][S]
    const float *src_val;      // forward: at_src [n] (or null); backward: t_req [S] (or null)
    float t_scalar;            // backward: T when t_req is null
    const float *other;        // backward: at (for slack)
    float *out;                // forward: at; backward: rat
    float *slack;              // backward, optional [n][S]
    int32_t *wns_ord;          // backward: [S] ordered-int mins
    int32_t *done;             // [G*L] chunks published per (group, level)
    int32_t *ticket;           // [1]
    uint32_t *err;
};

// per-stage shared-memory layout (offsets in bytes, computed identically on host)
struct StageLayout {
    int desc, node, rp, vb, vnode, nbr, d, bytes;
};
__host__ __device__ inline StageLayout stage_layout(int T, int ecap, int Sg) {
    StageLayout L;
    int o = 0;
    L.desc = o;  o += 16 * 4;
    L.node = o;  o += T * 4;
    L.rp = o;    o += (T + 1) * 4;
    L.vb = o;    o += (T + 1) * 4;
    L.vnode = o; o += 2 * T * 4;
    L.nbr = o;   o += ecap * 4;
    o = (o + 15) & ~15;
    L.d = o;     o += ecap * Sg * 4;
    L.bytes = (o + 127) & ~127;
    return L;
}
enum { D_T = 0, D_LV, D_G, D_POS, D_NN, D_RB, D_E, D_EST, D_NVS, D_HUB };

template <bool FWD> __device__ __forceinline__ float combine(float best, float x) {
    return FWD ? fmaxf(best, x) : fminf(best, x);
}
template <bool FWD> __device__ __forceinline__ float relax(float a, float d) {
    return FWD ? __fadd_rn(a, d) : __fsub_rn(a, d);
}
template <bool FWD> __device__ __forceinline__ float ident() {
    return __int_as_float(FWD ? 0xff800000 : 0x7f800000);   // -inf for max, +inf for min
}

template <int V, bool FWD, bool CHECK_D, bool BULK>
__global__ void __launch_bounds__(BLOCK, 2) k_propagate(PassParams p) {
    extern __shared__ __align__(128) unsigned char smem[];
    const StageLayout SL = stage_layout(p.T, p.ecap, p.Sg);
    const int lpn = p.Sg / V;                 // lanes per node slice
    const int slots = NCT / lpn;              // vslots handled per round
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + NB * SL.bytes);
    uint64_t *empty = full + NB;
    float *s_part = reinterpret_cast<float *>(smem + NB * SL.bytes + 2 * NB * 8);   // [2T][Sg]
    int32_t *s_min = reinterpret_cast<int32_t *>(s_part + 2 * p.T * p.Sg);           // [S]
    const int tid = threadIdx.x;

    if (tid == 0) {
        for (int s = 0; s < NB; ++s) {
            mbar_init(full + s, 32);
            mbar_init(empty + s, 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (!FWD)
        for (int s = tid; s < p.S; s += BLOCK) s_min[s] = 0x7f800000;
    __syncthreads();

    if (tid >= NCT) {
        // ============================ producer warp ============================
        const int lane = tid - NCT;
        int lv = FWD ? 0 : p.L - 1;
        for (int i = 0;; ++i) {
            const int st = i % NB;
            mbar_wait(empty + st, ((i / NB) & 1) ^ 1);
            unsigned char *sb = smem + st * SL.bytes;
            int32_t *desc = reinterpret_cast<int32_t *>(sb + SL.desc);
            int t = 0;
            if (lane == 0) t = atomicAdd(p.ticket, 1);
            t = __shfl_sync(0xffffffffu, t, 0);
            if (t >= p.C * p.G) {
                if (lane == 0) desc[D_T] = -1;
                mbar_arrive(full + st);
                break;
            }
            const int g = t % p.G;
            const int rank = FWD ? t / p.G : p.C - 1 - t / p.G;
            if (FWD) {
                while (__ldg(p.chunk_ptr + lv + 1) <= rank) ++lv;
            } else {
                while (__ldg(p.chunk_ptr + lv) > rank) --lv;
            }
            const int pos = __ldg(p.chunk_pos + rank);
            const int nn = __ldg(p.chunk_pos + rank + 1) - pos;
            int32_t *s_node = reinterpret_cast<int32_t *>(sb + SL.node);
            int32_t *s_rp = reinterpret_cast<int32_t *>(sb + SL.rp);
            int32_t *s_vb = reinterpret_cast<int32_t *>(sb + SL.vb);
            int32_t *s_vnode = reinterpret_cast<int32_t *>(sb + SL.vnode);
            int32_t *s_nbr = reinterpret_cast<int32_t *>(sb + SL.nbr);
            float *s_d = reinterpret_cast<float *>(sb + SL.d);
            const int rb = __ldg(p.row_ptr + pos);
            const int E = __ldg(p.row_ptr + pos + nn) - rb;
            const bool hub = nn == 1 && (E + PF - 1) / PF > p.T;
            // rows + vslot prefix (nodes are <= T)
            int carry = 0;
            for (int j0 = 0; j0 < nn; j0 += 32) {
                const int j = j0 + lane;
                int nv = 0;
                if (j < nn) {
                    s_node[j] = __ldg(p.node_of + pos + j);
                    const int a = __ldg(p.row_ptr + pos + j) - rb;
                    const int b = __ldg(p.row_ptr + pos + j + 1) - rb;
                    s_rp[j] = a;
                    nv = hub ? 0 : max(1, (b - a + PF - 1) / PF);
                }
                int incl = nv;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    int y = __shfl_up_sync(0xffffffffu, incl, o);
                    if (lane >= o) incl += y;
                }
                if (j < nn) s_vb[j] = carry + incl - nv;
                carry += __shfl_sync(0xffffffffu, incl, 31);
            }
            const int nvs = hub ? 0 : carry;
            if (lane == 0) {
                s_rp[nn] = E;
                s_vb[nn] = nvs;
            }
            __syncwarp();
            if (!hub)
                for (int j = lane; j < nn; j += 32)
                    for (int v = s_vb[j]; v < s_vb[j + 1]; ++v) s_vnode[v] = j;
            // stage neighbours + delay slices of the first est edges
            const int est = min(E, p.ecap);
            const int64_t col0 = int64_t(g) * p.Sg;
            for (int e = lane; e < est; e += 32) {
                s_nbr[e] = __ldg(p.nbr + rb + e);
                const float *src = p.d + int64_t(__ldg(p.eid + rb + e)) * p.S + col0;
                if (BULK) {
                    bulk_g2s(s_d + int64_t(e) * p.Sg, src, uint32_t(p.Sg) * 4u, full + st);
                } else {
                    for (int c = 0; c < p.Sg; ++c) s_d[int64_t(e) * p.Sg + c] = __ldg(src + c);
                }
            }
            if (lane == 0) {
                desc[D_T] = t;
                desc[D_LV] = lv;
                desc[D_G] = g;
                desc[D_POS] = pos;
                desc[D_NN] = nn;
                desc[D_RB] = rb;
                desc[D_E] = E;
                desc[D_EST] = est;
                desc[D_NVS] = nvs;
                desc[D_HUB] = hub;
            }
            __syncwarp();
            if (BULK && lane == 0)
                mbar_arrive_tx(full + st, uint32_t(est) * uint32_t(p.Sg) * 4u);
            else
                mbar_arrive(full + st);
        }
        return;
    }

    // ============================== consumer warps ==============================
    const int slot = tid / lpn;
    const int lane = tid - slot * lpn;
    const bool has_slot = slot < slots;
    bool bad = false;
    Vec<V> run_min;
#pragma unroll
    for (int k = 0; k < V; ++k) run_min.x[k] = ident<false>();

    for (int i = 0;; ++i) {
        const int st = i % NB;
        mbar_wait(full + st, (i / NB) & 1);
        unsigned char *sb = smem + st * SL.bytes;
        const int32_t *desc = reinterpret_cast<const int32_t *>(sb + SL.desc);
        if (desc[D_T] < 0) break;
        const int lv = desc[D_LV], g = desc[D_G], nn = desc[D_NN], rb = desc[D_RB];
        const int E = desc[D_E], est = desc[D_EST], nvs = desc[D_NVS];
        const bool hub = desc[D_HUB] != 0;
        const int32_t *s_node = reinterpret_cast<const int32_t *>(sb + SL.node);
        const int32_t *s_rp = reinterpret_cast<const int32_t *>(sb + SL.rp);
        const int32_t *s_vb = reinterpret_cast<const int32_t *>(sb + SL.vb);
        const int32_t *s_vnode = reinterpret_cast<const int32_t *>(sb + SL.vnode);
        const int32_t *s_nbr = reinterpret_cast<const int32_t *>(sb + SL.nbr);
        const float *s_d = reinterpret_cast<const float *>(sb + SL.d);
        const int64_t col = int64_t(g) * p.Sg + int64_t(lane) * V;   // scenario of lane
        const int scol = lane * V;                                     // column in stage

        // ---- wait until the previous level (pass order) of this group is published
        const int dep = FWD ? lv - 1 : lv + 1;
        if (tid == 0 && dep >= 0 && dep < p.L) {
            const int need = __ldg(p.chunk_ptr + dep + 1) - __ldg(p.chunk_ptr + dep);
            const int *cnt = p.done + g * p.L + dep;
            if (ld_acquire(cnt) < need)
                while (ld_acquire(cnt) < need) __nanosleep(20);
        }
        consumer_sync();

        // ---- partial max/min of every vslot (<= PF edges) or hub strip ----------
        auto edge_val = [&](int e, Vec<V> &acc, bool first) {
            int u;
            Vec<V> dd;
            if (e < est) {
                u = s_nbr[e];
                dd = ldv_s<V>(s_d + int64_t(e) * p.Sg + scol);
            } else {
                u = __ldg(p.nbr + rb + e);
                dd = ldv_g<V>(p.d + int64_t(__ldg(p.eid + rb + e)) * p.S + col);
            }
            Vec<V> a = ldv_cg<V>(p.out + int64_t(u) * p.S + col);
#pragma unroll
            for (int j = 0; j < V; ++j) {
                float d1 = dd.x[j];
                if (CHECK_D) {
                    bad |= !isfinite(d1);
                    d1 = canon0(d1);
                }
                const float x = relax<FWD>(a.x[j], d1);
                acc.x[j] = first ? x : combine<FWD>(acc.x[j], x);
            }
        };
        if (!hub) {
            for (int vs = slot; has_slot && vs < nvs; vs += slots) {
                const int j = s_vnode[vs];
                const int eb = s_rp[j] + (vs - s_vb[j]) * PF;
                const int ee = min(s_rp[j + 1], eb + PF);
                Vec<V> acc;
#pragma unroll
                for (int k = 0; k < V; ++k) acc.x[k] = ident<FWD>();
                // independent gathers of up to PF edges (one L2 round trip)
                Vec<V> a[PF];
                Vec<V> dd[PF];
#pragma unroll
                for (int k = 0; k < PF; ++k) {
                    const int e = eb + k;
                    if (e < ee) {
                        int u;
                        if (e < est) {
                            u = s_nbr[e];
                            dd[k] = ldv_s<V>(s_d + int64_t(e) * p.Sg + scol);
                        } else {
                            u = __ldg(p.nbr + rb + e);
                            dd[k] = ldv_g<V>(p.d + int64_t(__ldg(p.eid + rb + e)) * p.S + col);
                        }
                        a[k] = ldv_cg<V>(p.out + int64_t(u) * p.S + col);
                    }
                }
#pragma unroll
                for (int k = 0; k < PF; ++k) {
                    if (eb + k < ee) {
#pragma unroll
                        for (int j2 = 0; j2 < V; ++j2) {
                            float d1 = dd[k].x[j2];
                            if (CHECK_D) {
                                bad |= !isfinite(d1);
                                d1 = canon0(d1);
                            }
                            acc.x[j2] = combine<FWD>(acc.x[j2], relax<FWD>(a[k].x[j2], d1));
                        }
                    }
                }
                stv_s<V>(s_part + int64_t(vs) * p.Sg + scol, acc);
            }
        } else if (has_slot) {
            Vec<V> acc;
#pragma unroll
            for (int k = 0; k < V; ++k) acc.x[k] = ident<FWD>();
            for (int e = slot; e < E; e += slots) edge_val(e, acc, false);
            stv_s<V>(s_part + int64_t(slot) * p.Sg + scol, acc);
        }
        consumer_sync();

        // ---- combine each node's vslots, store, fused slack (backward) ----------
        const int nodes_here = hub ? 1 : nn;
        for (int j = slot; has_slot && j < nodes_here; j += slots) {
            const int node = s_node[j];
            Vec<V> best;
            const bool leaf = s_rp[j + 1] == s_rp[j];
            if (leaf) {
                if (FWD) {
                    const float a0 = p.src_val ? canon0(__ldg(p.src_val + node)) : 0.0f;
#pragma unroll
                    for (int k = 0; k < V; ++k) best.x[k] = a0;
                } else {
#pragma unroll
                    for (int k = 0; k < V; ++k)
                        best.x[k] = canon0(p.src_val ? __ldg(p.src_val + col + k) : p.t_scalar);
                }
            } else {
                const int v0 = hub ? 0 : s_vb[j];
                const int v1 = hub ? min(slots, E) : s_vb[j + 1];
                best = ldv_s<V>(s_part + int64_t(v0) * p.Sg + scol);
                for (int v = v0 + 1; v < v1; ++v) {
                    Vec<V> q = ldv_s<V>(s_part + int64_t(v) * p.Sg + scol);
#pragma unroll
                    for (int k = 0; k < V; ++k) best.x[k] = combine<FWD>(best.x[k], q.x[k]);
                }
            }
            stv_g<V>(p.out + int64_t(node) * p.S + col, best);
            if (!FWD) {
                Vec<V> a = ldv_cg<V>(p.other + int64_t(node) * p.S + col);
                Vec<V> sl;
#pragma unroll
                for (int k = 0; k < V; ++k) {
                    sl.x[k] = __fsub_rn(best.x[k], a.x[k]);
                    run_min.x[k] = fminf(run_min.x[k], sl.x[k]);
                }
                if (p.slack) stv_g<V>(p.slack + int64_t(node) * p.S + col, sl);
            }
        }
        // ---- publish: stores visible at gpu scope, then bump the level counter --
        __threadfence();
        consumer_sync();
        if (tid == 0) {
            atomicAdd(p.done + g * p.L + lv, 1);
            mbar_arrive(empty + st);
        }
    }

    if (CHECK_D && bad) atomicOr(p.err, ERR_NONFINITE);
    if (!FWD) {
        // backward runs with one scenario group (G == 1), so lane owns scenarios
        // lane*V .. lane*V+V-1 in every chunk
        if (has_slot) {
#pragma unroll
            for (int k = 0; k < V; ++k)
                if (run_min.x[k] != ident<false>())
                    atomicMin(s_min + lane * V + k, f2ord(run_min.x[k]));
        }
        asm volatile("bar.sync 1, %0;" ::"n"(NCT) : "memory");
        for (int s = tid; s < p.S; s += NCT)
            if (s_min[s] != 0x7f800000) atomicMin(p.wns_ord + s, s_min[s]);
    }
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

// ---- chunk schedule (per direction and T), cached in the graph ---------------
__global__ void k_chunk_nv(const int32_t *__restrict__ row_ptr, int32_t n, int32_t *__restrict__ nv) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x) {
        const int d = row_ptr[i + 1] - row_ptr[i];
        nv[i] = max(1, (d + PF - 1) / PF);
    }
}

__global__ void k_chunk_flags(const int32_t *__restrict__ order, const int32_t *__restrict__ level,
                              const int32_t *__restrict__ level_ptr, const int32_t *__restrict__ nv,
                              const int32_t *__restrict__ P, int32_t n, int32_t T,
                              int32_t *__restrict__ flag) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x) {
        const int ls = level_ptr[level[order[i]]];
        int f = 1;
        if (i > ls) {
            const int c = (P[i] - P[ls]) / T, cp = (P[i - 1] - P[ls]) / T;
            f = (c != cp) || nv[i] > T || nv[i - 1] > T;
        }
        flag[i] = f;
    }
}

__global__ void k_chunk_scatter(const int32_t *__restrict__ flag, const int32_t *__restrict__ F,
                                int32_t n, int32_t *__restrict__ chunk_pos) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x)
        if (flag[i]) chunk_pos[F[i]] = int(i);
    if (blockIdx.x == 0 && threadIdx.x == 0) chunk_pos[F[n]] = n;
}

__global__ void k_chunk_levels(const int32_t *__restrict__ level_ptr, const int32_t *__restrict__ F,
                               int32_t L, int32_t *__restrict__ chunk_ptr) {
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k <= L; k += gridDim.x * blockDim.x)
        chunk_ptr[k] = F[level_ptr[k]];
}

void build_schedule(Graph &g, const int32_t *row_ptr, int T, DevBuf &pos_buf, DevBuf &ptr_buf,
                    int32_t &C) {
    cudaStream_t s = g.stream;
    const int32_t n = g.n;
    DevBuf nv, P, flag, F;
    nv.alloc(sizeof(int32_t) * (int64_t(n) + 1), s);
    P.alloc(sizeof(int32_t) * (int64_t(n) + 1), s);
    flag.alloc(sizeof(int32_t) * (int64_t(n) + 1), s);
    F.alloc(sizeof(int32_t) * (int64_t(n) + 1), s);
    HF_CUDA(cudaMemsetAsync(nv.as<int32_t>() + n, 0, sizeof(int32_t), s));
    HF_CUDA(cudaMemsetAsync(flag.as<int32_t>() + n, 0, sizeof(int32_t), s));
    k_chunk_nv<<<grid_for(n, 256, g.sms), 256, 0, s>>>(row_ptr, n, nv.as<int32_t>());
    HF_CHECK_LAUNCH();
    scan_exclusive(nv.as<int32_t>(), P.as<int32_t>(), int64_t(n) + 1, nullptr, s, g);
    k_chunk_flags<<<grid_for(n, 256, g.sms), 256, 0, s>>>(
        g.order.as<int32_t>(), g.level.as<int32_t>(), g.level_ptr.as<int32_t>(), nv.as<int32_t>(),
        P.as<int32_t>(), n, T, flag.as<int32_t>());
    HF_CHECK_LAUNCH();
    scan_exclusive(flag.as<int32_t>(), F.as<int32_t>(), int64_t(n) + 1, nullptr, s, g);
    int32_t h_C = 0;
    HF_CUDA(cudaMemcpyAsync(&h_C, F.as<int32_t>() + n, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    HF_CUDA(cudaStreamSynchronize(s));
    C = h_C;
    pos_buf.alloc(sizeof(int32_t) * (int64_t(C) + 1), s);
    ptr_buf.alloc(sizeof(int32_t) * (int64_t(g.L) + 1), s);
    k_chunk_scatter<<<grid_for(n, 256, g.sms), 256, 0, s>>>(flag.as<int32_t>(), F.as<int32_t>(),
                                                            n, pos_buf.as<int32_t>());
    HF_CHECK_LAUNCH();
    k_chunk_levels<<<grid_for(int64_t(g.L) + 1, 256, g.sms), 256, 0, s>>>(
        g.level_ptr.as<int32_t>(), F.as<int32_t>(), g.L, ptr_buf.as<int32_t>());
    HF_CHECK_LAUNCH();
    g.launches += 5;
}

int pick_vec(int32_t Sg, std::initializer_list<const void *> ptrs) {
    auto aligned = [&](int bytes) {
        for (const void *q : ptrs)
            if (q && (reinterpret_cast<uintptr_t>(q) % bytes)) return false;
        return true;
    };
    if (Sg % 4 == 0 && aligned(16)) return 4;
    if (Sg % 2 == 0 && aligned(8)) return 2;
    return 1;
}

void prof_record(Graph &g, int idx) {
    if (g.prof) HF_CUDA(cudaEventRecord(g.ev[idx], g.stream));
}

template <int V, bool FWD, bool CHECK_D, bool BULK>
void launch(Graph &g, PassParams &p, size_t smem) {
    auto kern = k_propagate<V, FWD, CHECK_D, BULK>;
    HF_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    int per_sm = 0;
    HF_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, BLOCK, smem));
    if (per_sm < 1) fail(HF_ERR_CUDA, "propagation kernel does not fit on an SM");
    const int grid = std::max(1, std::min(per_sm * g.sms, p.C * p.G));
    kern<<<grid, BLOCK, smem, g.stream>>>(p);
    HF_CHECK_LAUNCH();
    g.launches += 1;
}

template <bool FWD>
void run_pass(Graph &g, PassParams &p, bool check_d, int V, bool bulk) {
    const int lpn = p.Sg / V;
    const int T = NCT / lpn;
    p.T = T;
    // chunk schedule (cached per direction and T)
    DevBuf &pos = FWD ? g.sched_f_pos : g.sched_b_pos;
    DevBuf &ptr = FWD ? g.sched_f_ptr : g.sched_b_ptr;
    int32_t &C = FWD ? g.sched_f_C : g.sched_b_C;
    int32_t &Tc = FWD ? g.sched_f_T : g.sched_b_T;
    if (Tc != T || !pos.p) {
        build_schedule(g, p.row_ptr, T, pos, ptr, C);
        Tc = T;
    }
    p.chunk_pos = pos.as<int32_t>();
    p.chunk_ptr = ptr.as<int32_t>();
    p.C = C;
    p.L = g.L;
    p.ecap = std::min(2 * T * PF, std::max(64, 16384 / (4 * p.Sg)));
    const StageLayout SL = stage_layout(T, p.ecap, p.Sg);
    size_t smem = size_t(NB) * SL.bytes + 2 * NB * 8 + sizeof(float) * 2 * T * p.Sg +
                  (FWD ? 0 : sizeof(int32_t) * p.S);
    // per-pass counters: done[G*L] + ticket
    g.ws_sync.alloc(sizeof(int32_t) * (size_t(p.G) * g.L + 1), g.stream);
    HF_CUDA(cudaMemsetAsync(g.ws_sync.p, 0, sizeof(int32_t) * (size_t(p.G) * g.L + 1), g.stream));
    p.done = g.ws_sync.as<int32_t>();
    p.ticket = p.done + size_t(p.G) * g.L;
    p.err = g.d_err();
#define HF_LAUNCH(VV)                                                                       \
    do {                                                                                    \
        if (check_d && bulk) launch<VV, FWD, true, true>(g, p, smem);                       \
        else if (check_d) launch<VV, FWD, true, false>(g, p, smem);                         \
        else if (bulk) launch<VV, FWD, false, true>(g, p, smem);                            \
        else launch<VV, FWD, false, false>(g, p, smem);                                     \
    } while (0)
    if (V == 4) HF_LAUNCH(4);
    else if (V == 2) HF_LAUNCH(2);
    else HF_LAUNCH(1);
#undef HF_LAUNCH
}

// scenario groups: Sg = S / G with Sg / V <= NCT
void choose_groups(int32_t S, const std::initializer_list<const void *> &ptrs, int &G, int &Sg,
                   int &V) {
    G = 1;
    while (true) {
        if (S % G == 0) {
            Sg = S / G;
            V = pick_vec(Sg, ptrs);
            if (Sg / V <= NCT) break;
        }
        ++G;
        if (G > S) fail(HF_ERR_INVALID_ARG, "cannot split scenarios into groups");
    }
}

}  // namespace

// Forward over all levels (device pointers).  d: [m][S].
void forward_device(Graph &g, const float *d, int32_t S, bool check_d, const float *at_src,
                    float *at) {
    if (g.n == 0) return;
    PassParams p{};
    int G, Sg, V;
    choose_groups(S, {d, at}, G, Sg, V);
    p.row_ptr = g.lo_in_ptr.as<int32_t>();
    p.nbr = g.lo_in_src.as<int32_t>();
    p.eid = g.lo_in_eid.as<int32_t>();
    p.node_of = g.order.as<int32_t>();
    p.S = S;
    p.Sg = Sg;
    p.G = G;
    p.d = d;
    p.src_val = at_src;
    p.out = at;
    const bool bulk = (Sg % 4 == 0) && (reinterpret_cast<uintptr_t>(d) % 16 == 0) && S % 4 == 0;
    run_pass<true>(g, p, check_d, V, bulk);
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
        int G, Sg, V;
        choose_groups(S, {d, at, rat, slack}, G, Sg, V);
        if (G > 1) fail(HF_ERR_INVALID_ARG, "backward: more than 1024 scenarios per call");
        p.row_ptr = g.lo_out_ptr.as<int32_t>();
        p.nbr = g.lo_out_dst.as<int32_t>();
        p.eid = g.lo_out_eid.as<int32_t>();
        p.node_of = g.order.as<int32_t>();
        p.S = S;
        p.Sg = Sg;
        p.G = G;
        p.d = d;
        p.src_val = t_arr;
        p.t_scalar = t_scalar;
        p.other = at;
        p.out = rat;
        p.slack = slack;
        p.wns_ord = ord;
        const bool bulk = (Sg % 4 == 0) && (reinterpret_cast<uintptr_t>(d) % 16 == 0) && S % 4 == 0;
        run_pass<false>(g, p, false, V, bulk);
    }
    if (wns_f) {
        k_ord_to_float<<<1, 256, 0, s>>>(ord, wns_f, S);
        HF_CHECK_LAUNCH();
        g.launches += 1;
    }
}

void profile_mark(Graph &g, int idx) { prof_record(g, idx); }

}  // namespace hf
