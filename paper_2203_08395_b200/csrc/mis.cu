// mis.cu -- NEXT-4: greedy maximal independent set (
// PAPER.md:1141-1150, "a parallel maximal independent set finding step using
// Blelloch's Algorithm"), reading R19: the lexicographically-first MIS of
// the undirected graph of the DAG's edges for the vertex order (prio[v], v).
//
// Blelloch-Fineman-Shun rounds on the priority DAG (every edge oriented from the
// earlier to the later endpoint), one persistent cooperative launch:
//   round r: every undecided vertex v scans its neighbours (fan-in and fan-out);
//     an earlier neighbour IN  -> v is OUT;
//     all earlier neighbours OUT -> v is IN;
//     otherwise v stays undecided and is appended to the next frontier (warp-
//     aggregated compaction); a grid barrier ends the round.
// Decisions only read final states (an undecided neighbour blocks IN), so reading
// states written earlier in the same round is safe and only adds progress; the
// undecided vertex with the smallest key always decides, so every round progresses
// (O(log^2 n) rounds expected for random priorities).
#include <algorithm>

#include "common.cuh"

namespace hf {

namespace {

enum : int32_t { MIS_UNDECIDED = 0, MIS_IN = 1, MIS_OUT = 2 };

struct MisBar {
    unsigned count;
    unsigned pad;
};

__device__ __forceinline__ unsigned mis_ld_acquire(const unsigned *p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void mis_grid_sync(MisBar *b, unsigned &target) {
    target += gridDim.x;
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(&b->count) : "memory");
        while (mis_ld_acquire(&b->count) < target) __nanosleep(20);
    }
    __syncthreads();
}
__device__ __forceinline__ int32_t ld_state(const int32_t *p) {
    int32_t v;
    asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_state(int32_t *p, int32_t v) {
    asm volatile("st.relaxed.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ bool earlier(int32_t pu, int32_t u, int32_t pv, int32_t v) {
    return pu < pv || (pu == pv && u < v);
}

// sizes: sz[r % 3] = frontier size of round r (0: all n vertices in id order)
__global__ void k_mis(const int32_t *__restrict__ in_ptr, const int32_t *__restrict__ in_src,
                      const int32_t *__restrict__ out_ptr, const int32_t *__restrict__ out_dst,
                      const int32_t *__restrict__ prio, int32_t n, int32_t *__restrict__ state,
                      int32_t *__restrict__ fa, int32_t *__restrict__ fb, int32_t *sz, MisBar *bar,
                      int32_t max_rounds) {
    const int lane = threadIdx.x & 31;
    const int64_t nthreads = int64_t(gridDim.x) * blockDim.x;
    const int64_t tid = (int64_t(threadIdx.x >> 5) * gridDim.x + blockIdx.x) * 32 + lane;
    int32_t *lists[2] = {fa, fb};
    unsigned target = 0;
    for (int r = 0; r < max_rounds; ++r) {
        volatile int32_t *vsz = sz;
        const int size = r == 0 ? n : vsz[r % 3];
        if (size == 0) break;
        if (blockIdx.x == 0 && threadIdx.x == 0) vsz[(r + 2) % 3] = 0;
        const int32_t *in = lists[r & 1];
        int32_t *out = lists[(r + 1) & 1];
        const int64_t lim = (int64_t(size) + 31) / 32 * 32;
        for (int64_t i = tid; i < lim; i += nthreads) {
            bool keep = false;
            int v = 0;
            if (i < size) {
                v = r == 0 ? int(i) : in[i];
                const int32_t pv = prio[v];
                bool blocked = false, open = false;
                for (int e = in_ptr[v]; e < in_ptr[v + 1] && !blocked; ++e) {
                    const int u = in_src[e];
                    if (!earlier(prio[u], u, pv, v)) continue;
                    const int32_t su = ld_state(state + u);
                    blocked = su == MIS_IN;
                    open |= su == MIS_UNDECIDED;
                }
                for (int k = out_ptr[v]; k < out_ptr[v + 1] && !blocked; ++k) {
                    const int u = out_dst[k];
                    if (!earlier(prio[u], u, pv, v)) continue;
                    const int32_t su = ld_state(state + u);
                    blocked = su == MIS_IN;
                    open |= su == MIS_UNDECIDED;
                }
                if (blocked) st_state(state + v, MIS_OUT);
                else if (!open) st_state(state + v, MIS_IN);
                else keep = true;
            }
            // warp-aggregated append of the still undecided vertices
            const unsigned mk = __ballot_sync(0xffffffffu, keep);
            if (mk) {
                int base = 0;
                const int leader = __ffs(mk) - 1;
                if (lane == leader) base = atomicAdd(sz + (r + 1) % 3, __popc(mk));
                base = __shfl_sync(0xffffffffu, base, leader);
                if (keep) out[base + __popc(mk & ((1u << lane) - 1u))] = v;
            }
        }
        mis_grid_sync(bar, target);
    }
}

// every vertex is decided after at most n rounds (the earliest undecided vertex
// decides in every round), so no UNDECIDED state survives the loop
__global__ void k_mis_out(const int32_t *__restrict__ state, int32_t n,
                          uint8_t *__restrict__ in_set) {
    for (int64_t v = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; v < n;
         v += int64_t(gridDim.x) * blockDim.x)
        in_set[v] = state[v] == MIS_IN ? 1 : 0;
}

__global__ void k_mis_init(int32_t *state, int32_t n, int32_t *sz) {
    for (int64_t v = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; v < n;
         v += int64_t(gridDim.x) * blockDim.x)
        state[v] = MIS_UNDECIDED;
    if (blockIdx.x == 0 && threadIdx.x < 3) sz[threadIdx.x] = 0;
}

}  // namespace

// Device pointers, stream-ordered: prio [n] (any int32 keys, ties by id), in_set [n]
// (1 = in the set).  Uses the graph's fan-in and fan-out CSR; no levelization needed.
void mis_device(Graph &g, const int32_t *prio, uint8_t *in_set) {
    cudaStream_t s = g.stream;
    const int32_t n = g.n;
    if (n == 0) return;
    DevBuf state, fa, fb, sz, bar;
    state.alloc(sizeof(int32_t) * size_t(n), s);
    fa.alloc(sizeof(int32_t) * size_t(n), s);
    fb.alloc(sizeof(int32_t) * size_t(n), s);
    sz.alloc(sizeof(int32_t) * 4, s);
    bar.alloc(sizeof(MisBar), s);
    HF_CUDA(cudaMemsetAsync(bar.p, 0, sizeof(MisBar), s));
    k_mis_init<<<grid_for(n, 256, g.sms), 256, 0, s>>>(state.as<int32_t>(), n, sz.as<int32_t>());
    HF_CHECK_LAUNCH();
    static int per_sm = 0;
    const int block = 512;
    if (!per_sm) {
        HF_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, (const void *)k_mis, block, 0));
        per_sm = std::max(1, std::min(per_sm, 2));
    }
    const int32_t *ip = g.in_ptr.as<int32_t>(), *is = g.in_src.as<int32_t>();
    const int32_t *op = g.out_ptr.as<int32_t>(), *od = g.out_dst.as<int32_t>();
    int32_t *st = state.as<int32_t>(), *a = fa.as<int32_t>(), *b = fb.as<int32_t>();
    int32_t *szp = sz.as<int32_t>();
    MisBar *barp = bar.as<MisBar>();
    int32_t nn = n, max_rounds = n + 1;
    void *args[] = {&ip, &is, &op, &od, &prio, &nn, &st, &a, &b, &szp, &barp, &max_rounds};
    HF_CUDA(cudaLaunchCooperativeKernel((const void *)k_mis, g.sms * per_sm, block, args, 0, s));
    k_mis_out<<<grid_for(n, 256, g.sms), 256, 0, s>>>(st, n, in_set);
    HF_CHECK_LAUNCH();
    g.launches += 3;
}

}  // namespace hf
