// critical.cu -- NEXT-1 critical-path trace-back (
// PAPER.md:1002-1003 "extract graph information (critical paths, ...)"),
// DESIGN.md reading R17:
//   endpoint(s) = the sink (out-degree 0) with the smallest slack fl(T_s - at_s),
//                 ties by the smallest node id;
//   from v = endpoint step to src(e) for the fan-in edge e of v attaining the max,
//   fl(at_s[src e] + d_s[e]) == at_s[v], ties by the smallest fan-in edge id, until a
//   source.  path[s][0] = endpoint ... path[s][len-1] = source.
//
// Top-K endpoints (SURVEY.md §8(f) NEXT-1 "optional top-k endpoints"): the K sinks
// with the smallest (slack, id), each traced the same way.
//
// Endpoint selection: one 64-bit key per (sink, scenario) = {ordered slack, node id}
// (keys are unique).  K = 1: k_cp_endpoint, atomicMin per scenario.  K > 1: one
// selection for all K ranks -- k_cp_topk_local (grid bps x S: every thread keeps a
// sorted list of its K smallest keys, the block merges the lists' heads in K
// block-min rounds) and k_cp_topk_merge (one block per scenario merges the bps
// block lists the same way), independent of K in launches and in passes over n*S.
// Then k_cp_trace (one warp per (scenario, rank); per step
// the lanes recompute fl(at[u] + d) for 32 fan-in edges at a time and the smallest
// attaining edge id wins by ballot).  The trace is a dependent walk of <= L steps:
// latency-bound, scenarios in parallel.
#include <algorithm>

#include "common.cuh"

namespace hf {

namespace {

// key = (slack as an unsigned-ordered 32-bit value) << 32 | node id; keys are
// unique (the id), so the r-th endpoint is the smallest key above the (r-1)-th
__global__ void k_cp_endpoint(const int32_t *__restrict__ out_ptr, int32_t n, int32_t S,
                              const float *__restrict__ at, const float *__restrict__ t_arr,
                              float t_scalar, const unsigned long long *__restrict__ prev,
                              unsigned long long *__restrict__ key) {
    const int64_t total = int64_t(n) * S;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total;
         i += int64_t(gridDim.x) * blockDim.x) {
        const int64_t v = i / S;
        const int s = int(i - v * S);
        if (out_ptr[v + 1] != out_ptr[v]) continue;
        const float T = canon0(t_arr ? t_arr[s] : t_scalar);
        const float sl = __fsub_rn(T, at[i]);
        const unsigned o = unsigned(f2ord(sl)) ^ 0x80000000u;
        const unsigned long long k = (static_cast<unsigned long long>(o) << 32) | unsigned(v);
        if (prev && (prev[s] == ~0ull || k <= prev[s])) continue;
        atomicMin(key + s, k);
    }
}

constexpr int TOPK_MAX = 32;          // K <= TOPK_MAX: single selection; else K passes
constexpr int TOPK_THREADS = 256;

// block-wide minimum of one 64-bit value per thread (all threads call it)
__device__ __forceinline__ unsigned long long block_min_u64(unsigned long long v,
                                                            unsigned long long *s_red) {
    for (int o = 16; o; o >>= 1) {
        const unsigned long long w = __shfl_xor_sync(0xffffffffu, v, o);
        v = w < v ? w : v;
    }
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    __syncthreads();                       // s_red reused round after round
    if (lane == 0) s_red[wid] = v;
    __syncthreads();
    v = ~0ull;
    for (int i = 0; i < int(blockDim.x >> 5); ++i) v = s_red[i] < v ? s_red[i] : v;
    return v;
}

// K rounds: the smallest remaining head over the block's sorted per-thread lists
// (top[0..cnt) ascending) goes to out[r * ostride]; its owner advances.  Keys are
// unique, so exactly one thread owns the minimum.
__device__ __forceinline__ void block_merge_heads(const unsigned long long *top, int cnt, int K,
                                                  unsigned long long *out, int64_t ostride,
                                                  unsigned long long *s_red) {
    int h = 0;
    for (int r = 0; r < K; ++r) {
        const unsigned long long mine = h < cnt ? top[h] : ~0ull;
        const unsigned long long mn = block_min_u64(mine, s_red);
        if (mine == mn && mn != ~0ull) ++h;
        if (threadIdx.x == 0) out[r * ostride] = mn;
    }
}

__device__ __forceinline__ void topk_insert(unsigned long long *top, int &cnt, int K,
                                            unsigned long long k) {
    if (cnt == K && k >= top[K - 1]) return;
    int i = cnt < K ? cnt++ : K - 1;
    while (i > 0 && top[i - 1] > k) {
        top[i] = top[i - 1];
        --i;
    }
    top[i] = k;
}

// grid (bps, S): block b of scenario s scans nodes b*blockDim + t, stride bps*blockDim;
// cand[(s * bps + b) * K + r] = the block's r-th smallest key (~0 past its sinks)
__global__ void __launch_bounds__(TOPK_THREADS) k_cp_topk_local(
    const int32_t *__restrict__ out_ptr, int32_t n, int32_t S, const float *__restrict__ at,
    const float *__restrict__ t_arr, float t_scalar, int32_t K,
    unsigned long long *__restrict__ cand) {
    __shared__ unsigned long long s_red[TOPK_THREADS / 32];
    unsigned long long top[TOPK_MAX];
    int cnt = 0;
    const int s = blockIdx.y;
    const float T = canon0(t_arr ? t_arr[s] : t_scalar);
    for (int64_t v = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; v < n;
         v += int64_t(gridDim.x) * blockDim.x) {
        if (out_ptr[v + 1] != out_ptr[v]) continue;
        const float sl = __fsub_rn(T, at[v * S + s]);
        const unsigned o = unsigned(f2ord(sl)) ^ 0x80000000u;
        topk_insert(top, cnt, K, (static_cast<unsigned long long>(o) << 32) | unsigned(v));
    }
    block_merge_heads(top, cnt, K, cand + (int64_t(s) * gridDim.x + blockIdx.x) * K, 1, s_red);
}

// one block per scenario: merge the bps sorted block lists into key[r * S + s]
__global__ void __launch_bounds__(TOPK_THREADS) k_cp_topk_merge(
    const unsigned long long *__restrict__ cand, int32_t bps, int32_t S, int32_t K,
    unsigned long long *__restrict__ key) {
    __shared__ unsigned long long s_red[TOPK_THREADS / 32];
    unsigned long long top[TOPK_MAX];
    int cnt = 0;
    const int s = blockIdx.x;
    for (int b = threadIdx.x; b < bps; b += blockDim.x) {
        const unsigned long long *c = cand + (int64_t(s) * bps + b) * K;
        for (int r = 0; r < K; ++r) topk_insert(top, cnt, K, c[r]);
    }
    block_merge_heads(top, cnt, K, key + s, S, s_red);
}

// one warp per (scenario s, rank r); keys [K][S]
__global__ void k_cp_trace(const int32_t *__restrict__ in_ptr, const int32_t *__restrict__ in_src,
                           const float *__restrict__ d, const float *__restrict__ at, int32_t S,
                           int32_t K, const unsigned long long *__restrict__ key, int32_t max_len,
                           int32_t *__restrict__ endpoints, int32_t *__restrict__ path,
                           int32_t *__restrict__ len) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
    for (int64_t idx = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5; idx < int64_t(S) * K;
         idx += nw) {
        const int s = int(idx / K), r = int(idx - int64_t(s) * K);
        const unsigned long long k = key[int64_t(r) * S + s];
        int v = k == ~0ull ? -1 : int(unsigned(k));
        if (endpoints && lane == 0) endpoints[idx] = v;
        if (v < 0) {   // fewer than r + 1 sinks
            if (lane == 0) len[idx] = r == 0 ? -1 : 0;
            continue;
        }
        int32_t *p = path + idx * max_len;
        int cnt = 0;
        bool ok = true;
        while (ok) {
            if (cnt >= max_len) {
                ok = false;
                break;
            }
            if (lane == 0) p[cnt] = v;
            ++cnt;
            const int eb = in_ptr[v], ee = in_ptr[v + 1];
            if (eb == ee) break;   // source
            const float target = at[int64_t(v) * S + s];
            int best = -1;
            for (int e0 = eb; e0 < ee && best < 0; e0 += 32) {
                const int e = e0 + lane;
                bool hit = false;
                int u = 0;
                if (e < ee) {
                    u = in_src[e];
                    const float x = __fadd_rn(at[int64_t(u) * S + s], canon0(d[int64_t(e) * S + s]));
                    hit = x == target;
                }
                const unsigned b = __ballot_sync(0xffffffffu, hit);
                if (b) best = __shfl_sync(0xffffffffu, u, __ffs(b) - 1);
            }
            if (best < 0) {
                ok = false;
                break;
            }
            v = best;
        }
        if (lane == 0) len[idx] = ok ? cnt : -1;
    }
}

}  // namespace

// Device pointers: d [m][S] (fan-in edge order), at [n][S], t_arr [S] (or null ->
// t_scalar); K endpoints per scenario: endpoints [S][K] (or null), path
// [S][K][max_len], len [S][K] (-1 if at is not a forward result of d or the path
// exceeds max_len; 0 with endpoint -1 past the number of sinks).  One endpoint pass
// over all (sink, scenario) pairs per rank r, then one warp per (s, r) traces.
// Stream-ordered.
void critical_path_device(Graph &g, int32_t S, const float *d, const float *at,
                          const float *t_arr, float t_scalar, int32_t K, int32_t max_len,
                          int32_t *endpoints, int32_t *path, int32_t *len) {
    cudaStream_t s = g.stream;
    if (g.n == 0) {
        HF_CUDA(cudaMemsetAsync(len, 0, sizeof(int32_t) * size_t(S) * K, s));
        if (endpoints) HF_CUDA(cudaMemsetAsync(endpoints, 0xff, sizeof(int32_t) * size_t(S) * K, s));
        return;
    }
    DevBuf key;
    key.alloc(sizeof(unsigned long long) * size_t(S) * K, s);
    unsigned long long *kp = key.as<unsigned long long>();
    HF_CUDA(cudaMemsetAsync(kp, 0xff, sizeof(unsigned long long) * size_t(S) * K, s));
    int sel_launches = 0;
    if (K > 1 && K <= TOPK_MAX) {
        // one selection for all ranks: per-block lists, then a per-scenario merge
        const int64_t want = std::max<int64_t>(1, 4LL * g.sms / S);
        const int bps = int(std::min<int64_t>(
            std::min<int64_t>(want, (int64_t(g.n) + TOPK_THREADS - 1) / TOPK_THREADS), TOPK_THREADS));
        DevBuf cand;
        cand.alloc(sizeof(unsigned long long) * size_t(S) * bps * K, s);
        k_cp_topk_local<<<dim3(bps, S), TOPK_THREADS, 0, s>>>(g.out_ptr.as<int32_t>(), g.n, S, at,
                                                              t_arr, t_scalar, K,
                                                              cand.as<unsigned long long>());
        HF_CHECK_LAUNCH();
        k_cp_topk_merge<<<S, TOPK_THREADS, 0, s>>>(cand.as<unsigned long long>(), bps, S, K, kp);
        HF_CHECK_LAUNCH();
        sel_launches = 2;
    } else {
        // K = 1 (one atomicMin pass), or K > TOPK_MAX: pass r keeps keys above rank r-1's
        for (int r = 0; r < K; ++r) {
            k_cp_endpoint<<<grid_for(int64_t(g.n) * S, 256, g.sms), 256, 0, s>>>(
                g.out_ptr.as<int32_t>(), g.n, S, at, t_arr, t_scalar,
                r ? kp + int64_t(r - 1) * S : nullptr, kp + int64_t(r) * S);
            HF_CHECK_LAUNCH();
        }
        sel_launches = K;
    }
    const int warps = 8;
    k_cp_trace<<<int((int64_t(S) * K + warps - 1) / warps), 32 * warps, 0, s>>>(
        g.in_ptr.as<int32_t>(), g.in_src.as<int32_t>(), d, at, S, K, kp, max_len, endpoints,
        path, len);
    HF_CHECK_LAUNCH();
    g.launches += sel_launches + 1;
}

}  // namespace hf
