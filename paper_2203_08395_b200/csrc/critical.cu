// critical.cu -- NEXT-1 critical-path trace-back (
// PAPER.md:1002-1003 "extract graph information (critical paths, ...)"),
// DESIGN.md reading R17:
//   endpoint(s) = the sink (out-degree 0) with the smallest slack fl(T_s - at_s),
//                 ties by the smallest node id;
//   from v = endpoint step to src(e) for the fan-in edge e of v attaining the max,
//   fl(at_s[src e] + d_s[e]) == at_s[v], ties by the smallest fan-in edge id, until a
//   source.  path[s][0] = endpoint ... path[s][len-1] = source.
//
// Two kernels: k_cp_endpoint (one 64-bit key per (sink, scenario) = {ordered slack,
// node id}, atomicMin per scenario) and k_cp_trace (one warp per scenario; per step
// the lanes recompute fl(at[u] + d) for 32 fan-in edges at a time and the smallest
// attaining edge id wins by ballot).  The trace is a dependent walk of <= L steps:
// latency-bound, scenarios in parallel.
#include "common.cuh"

namespace hf {

namespace {

__global__ void k_cp_init(unsigned long long *key, int32_t S) {
    for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < S; s += gridDim.x * blockDim.x)
        key[s] = ~0ull;
}

// key = (slack as an unsigned-ordered 32-bit value) << 32 | node id
__global__ void k_cp_endpoint(const int32_t *__restrict__ out_ptr, int32_t n, int32_t S,
                              const float *__restrict__ at, const float *__restrict__ t_arr,
                              float t_scalar, unsigned long long *__restrict__ key) {
    const int64_t total = int64_t(n) * S;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total;
         i += int64_t(gridDim.x) * blockDim.x) {
        const int64_t v = i / S;
        const int s = int(i - v * S);
        if (out_ptr[v + 1] != out_ptr[v]) continue;
        const float T = canon0(t_arr ? t_arr[s] : t_scalar);
        const float sl = __fsub_rn(T, at[i]);
        const unsigned o = unsigned(f2ord(sl)) ^ 0x80000000u;
        atomicMin(key + s, (static_cast<unsigned long long>(o) << 32) | unsigned(v));
    }
}

// one warp per scenario
__global__ void k_cp_trace(const int32_t *__restrict__ in_ptr, const int32_t *__restrict__ in_src,
                           const float *__restrict__ d, const float *__restrict__ at, int32_t S,
                           const unsigned long long *__restrict__ key, int32_t max_len,
                           int32_t *__restrict__ path, int32_t *__restrict__ len) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
    for (int64_t s = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5; s < S; s += nw) {
        const unsigned long long k = key[s];
        int v = k == ~0ull ? -1 : int(unsigned(k));
        int cnt = 0;
        bool ok = v >= 0;
        while (ok) {
            if (cnt >= max_len) {
                ok = false;
                break;
            }
            if (lane == 0) path[s * max_len + cnt] = v;
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
        if (lane == 0) len[s] = ok ? cnt : -1;
    }
}

}  // namespace

// Device pointers: d [m][S] (fan-in edge order), at [n][S], t_arr [S] (or null ->
// t_scalar); path [S][max_len], len [S] (-1 if at is not a forward result of d or
// the path exceeds max_len).  Stream-ordered.
void critical_path_device(Graph &g, int32_t S, const float *d, const float *at,
                          const float *t_arr, float t_scalar, int32_t max_len, int32_t *path,
                          int32_t *len) {
    cudaStream_t s = g.stream;
    if (g.n == 0) {
        HF_CUDA(cudaMemsetAsync(len, 0, sizeof(int32_t) * size_t(S), s));
        return;
    }
    DevBuf key;
    key.alloc(sizeof(unsigned long long) * size_t(S), s);
    k_cp_init<<<grid_for(S, 256, g.sms), 256, 0, s>>>(key.as<unsigned long long>(), S);
    HF_CHECK_LAUNCH();
    k_cp_endpoint<<<grid_for(int64_t(g.n) * S, 256, g.sms), 256, 0, s>>>(
        g.out_ptr.as<int32_t>(), g.n, S, at, t_arr, t_scalar, key.as<unsigned long long>());
    HF_CHECK_LAUNCH();
    const int warps = 8;
    k_cp_trace<<<int((S + warps - 1) / warps), 32 * warps, 0, s>>>(
        g.in_ptr.as<int32_t>(), g.in_src.as<int32_t>(), d, at, S,
        key.as<unsigned long long>(), max_len, path, len);
    HF_CHECK_LAUNCH();
    g.launches += 3;
}

}  // namespace hf
