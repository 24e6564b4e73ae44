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
// Two kernels: k_cp_endpoint (one 64-bit key per (sink, scenario) = {ordered slack,
// node id}, atomicMin per scenario; pass r keeps keys above rank r-1's) and
// k_cp_trace (one warp per (scenario, rank); per step
// the lanes recompute fl(at[u] + d) for 32 fan-in edges at a time and the smallest
// attaining edge id wins by ballot).  The trace is a dependent walk of <= L steps:
// latency-bound, scenarios in parallel.
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
    for (int r = 0; r < K; ++r) {
        k_cp_endpoint<<<grid_for(int64_t(g.n) * S, 256, g.sms), 256, 0, s>>>(
            g.out_ptr.as<int32_t>(), g.n, S, at, t_arr, t_scalar,
            r ? kp + int64_t(r - 1) * S : nullptr, kp + int64_t(r) * S);
        HF_CHECK_LAUNCH();
    }
    const int warps = 8;
    k_cp_trace<<<int((int64_t(S) * K + warps - 1) / warps), 32 * warps, 0, s>>>(
        g.in_ptr.as<int32_t>(), g.in_src.as<int32_t>(), d, at, S, K, kp, max_len, endpoints,
        path, len);
    HF_CHECK_LAUNCH();
    g.launches += K + 1;
}

}  // namespace hf
