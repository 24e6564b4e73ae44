// propagate.cu -- forward max-plus and backward min-plus (+ fused slack / worst
// slack) over the levelized DAG, for one delay set or S scenario sets.
// SURVEY.md §8(a) a5-a7; BASELINE.json:5.
//
// Data layout in HBM (scenario-minor): at[v*S + s], rat[v*S + s],
// delays[e*S + s].  A node's S values are contiguous, so each fan-in/fan-out
// edge touches S*4 contiguous bytes and a thread owns a V-wide vector of them
// (V = 4 -> 16-byte LDG.128 / STG.128).  Pull-based: no float atomics; every
// output is one fp32 max/min over fl(x +/- d) terms, which is order-independent
// (0 ULP against the oracle, reading R10).
//
// v1 (this file): one launch per level, host loop over the level_ptr the
// levelizer returned.
#include <algorithm>

#include "common.cuh"

namespace hf {

namespace {

template <int V> struct VecT;
template <> struct VecT<1> { using T = float; };
template <> struct VecT<2> { using T = float2; };
template <> struct VecT<4> { using T = float4; };

template <int V> struct Vec {
    float x[V];
};

template <int V> __device__ __forceinline__ Vec<V> ldv(const float *p) {
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
// L2-coherent load (values written by other CTAs of earlier launches are fine
// either way; .cg keeps the gather from polluting L1)
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
        *reinterpret_cast<float4 *>(p) = make_float4(v.x[0], v.x[1], v.x[2], v.x[3]);
    } else if constexpr (V == 2) {
        *reinterpret_cast<float2 *>(p) = make_float2(v.x[0], v.x[1]);
    } else {
        *p = v.x[0];
    }
}

// Forward, one level: at[v] = max_e fl(at[src_e] + d_e) ; sources: at_src or +0.
// check_d: scenario delays come from the caller -> canonicalise -0, flag NaN/inf.
template <int V, bool CHECK_D>
__global__ void __launch_bounds__(256) k_fwd_level(
    const int32_t *__restrict__ nodes, int32_t count, const int32_t *__restrict__ in_ptr,
    const int32_t *__restrict__ in_src, const float *__restrict__ d, int32_t S,
    const float *__restrict__ at_src, float *__restrict__ at, uint32_t *err) {
    const int chunks = S / V;
    const int64_t work = int64_t(count) * chunks;
    bool bad = false;
    for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < work;
         t += int64_t(gridDim.x) * blockDim.x) {
        const int i = int(t / chunks);
        const int c = int(t - int64_t(i) * chunks);
        const int v = nodes[i];
        const int b = in_ptr[v], e_end = in_ptr[v + 1];
        Vec<V> best;
        if (b == e_end) {
            float a0 = at_src ? canon0(at_src[v]) : 0.0f;
#pragma unroll
            for (int k = 0; k < V; ++k) best.x[k] = a0;
        } else {
            for (int e = b; e < e_end; ++e) {
                const int u = in_src[e];
                Vec<V> a = ldv_cg<V>(at + int64_t(u) * S + c * V);
                Vec<V> dd = ldv<V>(d + int64_t(e) * S + c * V);
#pragma unroll
                for (int k = 0; k < V; ++k) {
                    float dk = dd.x[k];
                    if (CHECK_D) {
                        bad |= !isfinite(dk);
                        dk = canon0(dk);
                    }
                    float x = __fadd_rn(a.x[k], dk);
                    best.x[k] = (e == b) ? x : fmaxf(best.x[k], x);
                }
            }
        }
        stv<V>(at + int64_t(v) * S + c * V, best);
    }
    if (CHECK_D && __syncthreads_or(bad) && threadIdx.x == 0) atomicOr(err, ERR_NONFINITE);
}

// Backward, one level: rat[u] = min_e fl(rat[dst_e] - d_eid(e)); sinks: T_s.
// Fused: slack = fl(rat - at) (optional store), per-scenario min -> wns_ord.
template <int V>
__global__ void __launch_bounds__(256) k_bwd_level(
    const int32_t *__restrict__ nodes, int32_t count, const int32_t *__restrict__ out_ptr,
    const int32_t *__restrict__ out_dst, const int32_t *__restrict__ out_eid,
    const float *__restrict__ d, int32_t S, const float *__restrict__ t_arr, float t_scalar,
    const float *__restrict__ at, float *__restrict__ rat, float *__restrict__ slack,
    int32_t *__restrict__ wns_ord) {
    extern __shared__ int32_t s_min[];   // [S] ordered-int mins for this CTA
    for (int s = threadIdx.x; s < S; s += blockDim.x) s_min[s] = 0x7f800000;   // +inf
    __syncthreads();
    const int chunks = S / V;
    const int64_t work = int64_t(count) * chunks;
    for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < work;
         t += int64_t(gridDim.x) * blockDim.x) {
        const int i = int(t / chunks);
        const int c = int(t - int64_t(i) * chunks);
        const int u = nodes[i];
        const int b = out_ptr[u], e_end = out_ptr[u + 1];
        Vec<V> best;
        if (b == e_end) {
#pragma unroll
            for (int k = 0; k < V; ++k)
                best.x[k] = canon0(t_arr ? t_arr[c * V + k] : t_scalar);
        } else {
            for (int e = b; e < e_end; ++e) {
                const int v = out_dst[e];
                const int eid = out_eid[e];
                Vec<V> r = ldv_cg<V>(rat + int64_t(v) * S + c * V);
                Vec<V> dd = ldv<V>(d + int64_t(eid) * S + c * V);
#pragma unroll
                for (int k = 0; k < V; ++k) {
                    float x = __fsub_rn(r.x[k], canon0(dd.x[k]));
                    best.x[k] = (e == b) ? x : fminf(best.x[k], x);
                }
            }
        }
        stv<V>(rat + int64_t(u) * S + c * V, best);
        Vec<V> a = ldv_cg<V>(at + int64_t(u) * S + c * V);
        Vec<V> sl;
#pragma unroll
        for (int k = 0; k < V; ++k) sl.x[k] = __fsub_rn(best.x[k], a.x[k]);
        if (slack) stv<V>(slack + int64_t(u) * S + c * V, sl);
        if (S == 1) {
            int32_t key = f2ord(sl.x[0]);
            key = __reduce_min_sync(__activemask(), key);
            if ((threadIdx.x & 31) == __ffs(__activemask()) - 1) atomicMin(s_min, key);
        } else {
#pragma unroll
            for (int k = 0; k < V; ++k) atomicMin(s_min + c * V + k, f2ord(sl.x[k]));
        }
    }
    __syncthreads();
    for (int s = threadIdx.x; s < S; s += blockDim.x)
        if (s_min[s] != 0x7f800000) atomicMin(wns_ord + s, s_min[s]);
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
        for (const void *p : ptrs)
            if (p && (reinterpret_cast<uintptr_t>(p) % bytes)) return false;
        return true;
    };
    if (S % 4 == 0 && aligned(16)) return 4;
    if (S % 2 == 0 && aligned(8)) return 2;
    return 1;
}

template <int V>
void fwd_levels(Graph &g, const float *d, int32_t S, bool check_d, const float *at_src,
                float *at) {
    cudaStream_t s = g.stream;
    const int32_t *order = g.order.as<int32_t>();
    for (int32_t k = 0; k < g.L; ++k) {
        int32_t b = g.h_level_ptr[k], cnt = g.h_level_ptr[k + 1] - b;
        int64_t work = int64_t(cnt) * (S / V);
        int grid = int(std::min<int64_t>((work + 255) / 256, int64_t(g.sms) * 16));
        if (check_d)
            k_fwd_level<V, true><<<grid, 256, 0, s>>>(order + b, cnt, g.in_ptr.as<int32_t>(),
                                                     g.in_src.as<int32_t>(), d, S, at_src, at,
                                                     g.d_err());
        else
            k_fwd_level<V, false><<<grid, 256, 0, s>>>(order + b, cnt, g.in_ptr.as<int32_t>(),
                                                      g.in_src.as<int32_t>(), d, S, at_src, at,
                                                      g.d_err());
        HF_CHECK_LAUNCH();
        g.launches += 1;
    }
}

template <int V>
void bwd_levels(Graph &g, const float *d, int32_t S, const float *t_arr, float t_scalar,
                const float *at, float *rat, float *slack, int32_t *wns_ord) {
    cudaStream_t s = g.stream;
    const int32_t *order = g.order.as<int32_t>();
    size_t smem = sizeof(int32_t) * size_t(S);
    for (int32_t k = g.L - 1; k >= 0; --k) {
        int32_t b = g.h_level_ptr[k], cnt = g.h_level_ptr[k + 1] - b;
        int64_t work = int64_t(cnt) * (S / V);
        int grid = int(std::min<int64_t>((work + 255) / 256, int64_t(g.sms) * 16));
        k_bwd_level<V><<<grid, 256, smem, s>>>(order + b, cnt, g.out_ptr.as<int32_t>(),
                                                g.out_dst.as<int32_t>(), g.out_eid.as<int32_t>(),
                                                d, S, t_arr, t_scalar, at, rat, slack, wns_ord);
        HF_CHECK_LAUNCH();
        g.launches += 1;
    }
}

void prof_record(Graph &g, int idx) {
    if (g.prof) HF_CUDA(cudaEventRecord(g.ev[idx], g.stream));
}

}  // namespace

// Forward over all levels (device pointers).  d: [m][S].
void forward_device(Graph &g, const float *d, int32_t S, bool check_d, const float *at_src,
                    float *at) {
    if (g.n == 0) return;
    int V = pick_vec(S, {d, at});
    if (V == 4) fwd_levels<4>(g, d, S, check_d, at_src, at);
    else if (V == 2) fwd_levels<2>(g, d, S, check_d, at_src, at);
    else fwd_levels<1>(g, d, S, check_d, at_src, at);
}

// Backward over all levels + slack + wns (ordered ints in wns_ord[S], then
// decoded into wns_f[S] if non-null).
void backward_device(Graph &g, const float *d, int32_t S, const float *t_arr, float t_scalar,
                     const float *at, float *rat, float *slack, float *wns_f) {
    cudaStream_t s = g.stream;
    DevBuf ord;
    ord.alloc(sizeof(int32_t) * size_t(S), s);
    k_fill_i32<<<1, 256, 0, s>>>(ord.as<int32_t>(), 0x7f800000, S);
    HF_CHECK_LAUNCH();
    g.launches += 1;
    if (t_arr) {
        k_check_t<<<1, 256, 0, s>>>(t_arr, S, g.d_err());
        HF_CHECK_LAUNCH();
        g.launches += 1;
    }
    if (g.n > 0) {
        int V = pick_vec(S, {d, at, rat, slack});
        if (V == 4) bwd_levels<4>(g, d, S, t_arr, t_scalar, at, rat, slack, ord.as<int32_t>());
        else if (V == 2) bwd_levels<2>(g, d, S, t_arr, t_scalar, at, rat, slack, ord.as<int32_t>());
        else bwd_levels<1>(g, d, S, t_arr, t_scalar, at, rat, slack, ord.as<int32_t>());
    }
    if (wns_f) {
        k_ord_to_float<<<1, 256, 0, s>>>(ord.as<int32_t>(), wns_f, S);
        HF_CHECK_LAUNCH();
        g.launches += 1;
    }
}

void profile_mark(Graph &g, int idx) { prof_record(g, idx); }

}  // namespace hf
