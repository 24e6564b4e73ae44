// propagate.cu -- forward max-plus and backward min-plus (+ fused slack / worst
// slack) over the levelized DAG, for one delay set or S scenario sets.
// SURVEY.md §8(a) a5-a7; BASELINE.json:5.
//
// Data layout in HBM (scenario-minor): at[v*S + s], rat[v*S + s],
// delays[e*S + s].  A node's S values are contiguous, so each fan-in/fan-out
// edge touches S*4 contiguous bytes; a node is owned by LPN = S/V lanes, each
// holding a V-wide vector (V = 4 -> LDG.128 / STG.128).  Pull-based: no float
// atomics; every output is one fp32 max/min over fl(x +/- d) terms, which is
// order-independent (0 ULP against the oracle, reading R10).
//
// One persistent launch per pass (no per-level launches, no grid barrier):
//   * the work is cut into chunks of `slots` consecutive nodes of one level, in
//     level order (forward) or reverse level order (backward); CTAs claim chunks
//     with an atomic ticket, so a CTA only ever waits on chunks with smaller
//     tickets, which are held by running CTAs -> deadlock-free at any grid size;
//   * a chunk of level k first PREFETCHES everything that does not depend on
//     earlier levels (level-ordered CSR row, source ids, edge delays -- the bulk
//     of the HBM traffic), THEN waits until level k-1 (k+1 backward) has
//     published all its chunks (one acquire-poll of a per-level counter by one
//     thread), then gathers at[u] / rat[v] from L2, reduces, stores, fences and
//     bumps its level's counter (release).  Level k complete => all earlier
//     levels complete, by induction;
//   * a node whose degree exceeds the light-path limit is processed by the whole
//     CTA (edges split across slots, shared-memory max/min reduction), so fan-in
//     hubs (C5: 10k) and fan-out hubs (C3: ~700) do not serialise one lane;
//   * backward keeps a per-lane running min of slack; one shared-memory reduction
//     and one global atomicMin per scenario per CTA at the end give the WNS.
#include <algorithm>

#include "common.cuh"

namespace hf {

namespace {

constexpr int BLOCK = 256;
constexpr int PF = 4;   // edges per node prefetched into registers before the wait

template <int V> struct Vec {
    float x[V];
};

template <int V> __device__ __forceinline__ Vec<V> ldv_nc(const float *p) {   // read-only input
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
template <int V> __device__ __forceinline__ void stv(float *p, const Vec<V> &v) {
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

struct PassParams {
    // level-ordered CSR of this direction: row i <-> node node_of[i]
    const int32_t *row_ptr;    // [n+1]
    const int32_t *nbr;        // [m] neighbour node id (fan-in src / fan-out dst)
    const int32_t *eid;        // [m] edge id (delay row)
    const int32_t *node_of;    // [n]
    const int32_t *level_ptr;  // [L+1]
    const int32_t *chunk_ptr;  // [L+1] chunks before level k (level order)
    int32_t L;
    int32_t total_chunks;
    int32_t slots;             // nodes per chunk
    int32_t lpn;               // lanes per node = S/V
    int32_t S;                 // row stride of at/rat/delays (scenarios)
    const float *d;            // [m][S]
    const float *src_val;      // forward: at_src [n] (or null); backward: t_req [S] (or null)
    float t_scalar;            // backward: T when t_req is null
    const float *other;        // backward: at (for slack)
    float *out;                // forward: at; backward: rat
    float *slack;              // backward, optional [n][S]
    int32_t *wns_ord;          // backward: [S] ordered-int mins
    int32_t *done;             // [L] chunks published per level
    int32_t *ticket;           // [1]
    uint32_t *err;
};

template <bool FWD> __device__ __forceinline__ float combine(float best, float x) {
    return FWD ? fmaxf(best, x) : fminf(best, x);
}
template <bool FWD> __device__ __forceinline__ float relax(float a, float d) {
    return FWD ? __fadd_rn(a, d) : __fsub_rn(a, d);
}

template <int V, bool FWD, bool CHECK_D>
__global__ void __launch_bounds__(BLOCK, 4) k_propagate(PassParams p) {
    __shared__ int s_ticket;
    __shared__ int s_heavy[BLOCK];
    __shared__ int s_nheavy;
    __shared__ float s_red[BLOCK * V];
    extern __shared__ int32_t s_min[];   // backward: [S]

    const int tid = threadIdx.x;
    const int slot = tid / p.lpn;
    const int lane = tid - slot * p.lpn;
    const bool has_slot = slot < p.slots;
    const int64_t col = int64_t(lane) * V;   // first scenario of this lane
    const int light_max = 8 * PF;
    bool bad = false;
    Vec<V> run_min;
#pragma unroll
    for (int k = 0; k < V; ++k) run_min.x[k] = __int_as_float(0x7f800000);
    if (!FWD) {
        for (int s = tid; s < p.S; s += BLOCK) s_min[s] = 0x7f800000;
    }
    int lv = FWD ? 0 : p.L - 1;   // level cursor (monotone in ticket order)

    for (;;) {
        if (tid == 0) s_ticket = atomicAdd(p.ticket, 1);
        if (tid == 0) s_nheavy = 0;
        __syncthreads();
        const int t = s_ticket;
        if (t >= p.total_chunks) break;
        // ticket -> (level, chunk in level); forward walks levels up, backward down
        int rank;   // position of the chunk in level-order enumeration
        if (FWD) {
            rank = t;
            while (__ldg(p.chunk_ptr + lv + 1) <= rank) ++lv;
        } else {
            rank = p.total_chunks - 1 - t;
            while (__ldg(p.chunk_ptr + lv) > rank) --lv;
        }
        const int lbeg = __ldg(p.level_ptr + lv), lend = __ldg(p.level_ptr + lv + 1);
        const int pos = lbeg + (rank - __ldg(p.chunk_ptr + lv)) * p.slots + slot;
        const bool valid = has_slot && pos < lend;

        // ---- prefetch: independent of earlier levels ----------------------------
        int node = 0, rb = 0, deg = 0;
        int nb[PF];
        Vec<V> dv[PF];
        if (valid) {
            node = __ldg(p.node_of + pos);
            rb = __ldg(p.row_ptr + pos);
            deg = __ldg(p.row_ptr + pos + 1) - rb;
#pragma unroll
            for (int k = 0; k < PF; ++k) {
                if (k < deg && deg <= light_max) {
                    nb[k] = __ldg(p.nbr + rb + k);
                    dv[k] = ldv_nc<V>(p.d + int64_t(__ldg(p.eid + rb + k)) * p.S + col);
                }
            }
        }
        Vec<V> seed;   // value for degree-0 nodes
        if (valid && deg == 0) {
            if (FWD) {
                float a0 = p.src_val ? canon0(__ldg(p.src_val + node)) : 0.0f;
#pragma unroll
                for (int k = 0; k < V; ++k) seed.x[k] = a0;
            } else {
#pragma unroll
                for (int k = 0; k < V; ++k)
                    seed.x[k] = canon0(p.src_val ? __ldg(p.src_val + col + k) : p.t_scalar);
            }
        }

        // ---- wait for the previous level (in pass order) to be published --------
        const int dep = FWD ? lv - 1 : lv + 1;
        if (tid == 0 && dep >= 0 && dep < p.L) {
            const int need = __ldg(p.chunk_ptr + dep + 1) - __ldg(p.chunk_ptr + dep);
            if (ld_acquire(p.done + dep) < need) {
                while (ld_acquire(p.done + dep) < need) __nanosleep(20);
            }
        }
        __syncthreads();

        // ---- light nodes: this slot's lanes reduce the node's edges --------------
        if (valid && deg > light_max && lane == 0) s_heavy[atomicAdd(&s_nheavy, 1)] = pos;
        if (valid && deg <= light_max) {
            Vec<V> best = seed;
            if (deg > 0) {
#pragma unroll
                for (int k = 0; k < PF; ++k) {
                    if (k < deg) {
                        Vec<V> a = ldv_cg<V>(p.out + int64_t(nb[k]) * p.S + col);
#pragma unroll
                        for (int j = 0; j < V; ++j) {
                            float dd = dv[k].x[j];
                            if (CHECK_D) {
                                bad |= !isfinite(dd);
                                dd = canon0(dd);
                            }
                            float x = relax<FWD>(a.x[j], dd);
                            best.x[j] = k == 0 ? x : combine<FWD>(best.x[j], x);
                        }
                    }
                }
                for (int k = PF; k < deg; ++k) {
                    const int e = rb + k;
                    Vec<V> a = ldv_cg<V>(p.out + int64_t(__ldg(p.nbr + e)) * p.S + col);
                    Vec<V> dd = ldv_nc<V>(p.d + int64_t(__ldg(p.eid + e)) * p.S + col);
#pragma unroll
                    for (int j = 0; j < V; ++j) {
                        float d1 = dd.x[j];
                        if (CHECK_D) {
                            bad |= !isfinite(d1);
                            d1 = canon0(d1);
                        }
                        best.x[j] = combine<FWD>(best.x[j], relax<FWD>(a.x[j], d1));
                    }
                }
            }
            stv<V>(p.out + int64_t(node) * p.S + col, best);
            if (!FWD) {
                Vec<V> a = ldv_cg<V>(p.other + int64_t(node) * p.S + col);
                Vec<V> sl;
#pragma unroll
                for (int j = 0; j < V; ++j) {
                    sl.x[j] = __fsub_rn(best.x[j], a.x[j]);
                    run_min.x[j] = fminf(run_min.x[j], sl.x[j]);
                }
                if (p.slack) stv<V>(p.slack + int64_t(node) * p.S + col, sl);
            }
        }
        __syncthreads();

        // ---- heavy nodes (degree > light_max): the whole CTA splits the edges ----
        const int nheavy = s_nheavy;
        for (int h = 0; h < nheavy; ++h) {
            const int hp = s_heavy[h];
            const int hnode = __ldg(p.node_of + hp);
            const int hb = __ldg(p.row_ptr + hp), he = __ldg(p.row_ptr + hp + 1);
            Vec<V> part;
            bool any = false;
            if (has_slot) {
                for (int e = hb + slot; e < he; e += p.slots) {
                    Vec<V> a = ldv_cg<V>(p.out + int64_t(__ldg(p.nbr + e)) * p.S + col);
                    Vec<V> dd = ldv_nc<V>(p.d + int64_t(__ldg(p.eid + e)) * p.S + col);
#pragma unroll
                    for (int j = 0; j < V; ++j) {
                        float d1 = dd.x[j];
                        if (CHECK_D) {
                            bad |= !isfinite(d1);
                            d1 = canon0(d1);
                        }
                        float x = relax<FWD>(a.x[j], d1);
                        part.x[j] = any ? combine<FWD>(part.x[j], x) : x;
                    }
                    any = true;
                }
            }
            // slots with no edge contribute the identity
#pragma unroll
            for (int j = 0; j < V; ++j)
                s_red[tid * V + j] = any ? part.x[j]
                                         : __int_as_float(FWD ? 0xff800000 : 0x7f800000);
            __syncthreads();
            if (slot == 0 && has_slot) {
                Vec<V> best;
#pragma unroll
                for (int j = 0; j < V; ++j) best.x[j] = s_red[tid * V + j];
                for (int sl2 = 1; sl2 < p.slots; ++sl2)
#pragma unroll
                    for (int j = 0; j < V; ++j)
                        best.x[j] = combine<FWD>(best.x[j], s_red[(sl2 * p.lpn + lane) * V + j]);
                stv<V>(p.out + int64_t(hnode) * p.S + col, best);
                if (!FWD) {
                    Vec<V> a = ldv_cg<V>(p.other + int64_t(hnode) * p.S + col);
                    Vec<V> sl;
#pragma unroll
                    for (int j = 0; j < V; ++j) {
                        sl.x[j] = __fsub_rn(best.x[j], a.x[j]);
                        run_min.x[j] = fminf(run_min.x[j], sl.x[j]);
                    }
                    if (p.slack) stv<V>(p.slack + int64_t(hnode) * p.S + col, sl);
                }
            }
            __syncthreads();
        }

        // ---- publish this chunk ------------------------------------------------------
        __threadfence();
        __syncthreads();
        if (tid == 0) atomicAdd(p.done + lv, 1);
    }

    if (CHECK_D && __syncthreads_or(bad) && tid == 0) atomicOr(p.err, ERR_NONFINITE);
    if (!FWD) {
        if (has_slot) {
#pragma unroll
            for (int j = 0; j < V; ++j)
                if (col + j < p.S && run_min.x[j] != __int_as_float(0x7f800000))
                    atomicMin(s_min + col + j, f2ord(run_min.x[j]));
        }
        __syncthreads();
        for (int s = tid; s < p.S; s += BLOCK)
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

// chunk_ptr for `slots` nodes per chunk, cached in the graph
void ensure_chunks(Graph &g, int slots) {
    if (g.chunk_slots == slots && g.chunk_ptr.p) return;
    std::vector<int32_t> cp(size_t(g.L) + 1, 0);
    for (int32_t k = 0; k < g.L; ++k) {
        int32_t w = g.h_level_ptr[k + 1] - g.h_level_ptr[k];
        cp[k + 1] = cp[k] + (w + slots - 1) / slots;
    }
    g.chunk_ptr.alloc(sizeof(int32_t) * cp.size(), g.stream);
    HF_CUDA(cudaMemcpyAsync(g.chunk_ptr.p, cp.data(), sizeof(int32_t) * cp.size(),
                            cudaMemcpyHostToDevice, g.stream));
    HF_CUDA(cudaStreamSynchronize(g.stream));   // cp is a host temporary
    g.chunk_slots = slots;
    g.total_chunks = cp.back();
}

template <int V, bool FWD, bool CHECK_D> int grid_of(Graph &g, size_t smem) {
    int per_sm = 0;
    HF_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_propagate<V, FWD, CHECK_D>,
                                                          BLOCK, smem));
    if (per_sm < 1) per_sm = 1;
    return std::max(1, std::min(per_sm * g.sms, g.total_chunks));
}

template <int V, bool FWD, bool CHECK_D> void launch(Graph &g, PassParams &p) {
    size_t smem = FWD ? 0 : sizeof(int32_t) * size_t(p.S);
    if (smem > 48 * 1024)
        HF_CUDA(cudaFuncSetAttribute(k_propagate<V, FWD, CHECK_D>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    int grid = grid_of<V, FWD, CHECK_D>(g, smem);
    k_propagate<V, FWD, CHECK_D><<<grid, BLOCK, smem, g.stream>>>(p);
    HF_CHECK_LAUNCH();
    g.launches += 1;
}

template <int V, bool FWD> void run_pass(Graph &g, PassParams &p, bool check_d) {
    const int lpn = p.S / V;
    p.lpn = lpn;
    p.slots = BLOCK / lpn;
    ensure_chunks(g, p.slots);
    p.chunk_ptr = g.chunk_ptr.as<int32_t>();
    p.total_chunks = g.total_chunks;
    p.level_ptr = g.level_ptr.as<int32_t>();
    p.L = g.L;
    // per-pass counters: done[L] + ticket
    g.ws_sync.alloc(sizeof(int32_t) * (size_t(g.L) + 1), g.stream);
    HF_CUDA(cudaMemsetAsync(g.ws_sync.p, 0, sizeof(int32_t) * (size_t(g.L) + 1), g.stream));
    p.done = g.ws_sync.as<int32_t>();
    p.ticket = p.done + g.L;
    p.err = g.d_err();
    if (check_d) launch<V, FWD, true>(g, p);
    else launch<V, FWD, false>(g, p);
}

template <bool FWD> void dispatch(Graph &g, PassParams &p, bool check_d, int V) {
    if (V == 4) run_pass<4, FWD>(g, p, check_d);
    else if (V == 2) run_pass<2, FWD>(g, p, check_d);
    else run_pass<1, FWD>(g, p, check_d);
}

void prof_record(Graph &g, int idx) {
    if (g.prof) HF_CUDA(cudaEventRecord(g.ev[idx], g.stream));
}

void check_S(int32_t S, int V) {
    if (S / V > BLOCK)
        fail(HF_ERR_INVALID_ARG, "too many scenarios in one call (S/V must be <= 256: S <= 1024 "
                                 "with 16-byte aligned buffers)");
}

}  // namespace

// Forward over all levels (device pointers).  d: [m][S].
void forward_device(Graph &g, const float *d, int32_t S, bool check_d, const float *at_src,
                    float *at) {
    if (g.n == 0) return;
    int V = pick_vec(S, {d, at});
    check_S(S, V);
    PassParams p{};
    p.row_ptr = g.lo_in_ptr.as<int32_t>();
    p.nbr = g.lo_in_src.as<int32_t>();
    p.eid = g.lo_in_eid.as<int32_t>();
    p.node_of = g.order.as<int32_t>();
    p.S = S;
    p.d = d;
    p.src_val = at_src;
    p.out = at;
    dispatch<true>(g, p, check_d, V);
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
        int V = pick_vec(S, {d, at, rat, slack});
        check_S(S, V);
        PassParams p{};
        p.row_ptr = g.lo_out_ptr.as<int32_t>();
        p.nbr = g.lo_out_dst.as<int32_t>();
        p.eid = g.lo_out_eid.as<int32_t>();
        p.node_of = g.order.as<int32_t>();
        p.S = S;
        p.d = d;
        p.src_val = t_arr;
        p.t_scalar = t_scalar;
        p.other = at;
        p.out = rat;
        p.slack = slack;
        p.wns_ord = ord;
        dispatch<false>(g, p, false, V);
    }
    if (wns_f) {
        k_ord_to_float<<<1, 256, 0, s>>>(ord, wns_f, S);
        HF_CHECK_LAUNCH();
        g.launches += 1;
    }
}

void profile_mark(Graph &g, int idx) { prof_record(g, idx); }

}  // namespace hf
