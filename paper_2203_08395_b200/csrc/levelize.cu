// levelize.cu -- hf_levelize: on-device Kahn levelization with chain contraction.
// SURVEY.md §8(a) a2-a4; PAPER.md:689-690 ("no cycles"), 840-848 (join counters).
//
// level(v) = 0 for sources, else 1 + max level(pred) (reading R5).
// Integer longest path, so it may be computed in any association order (exact):
//  1. in-degree-1 nodes form in-trees hanging below "junctions" (in-degree != 1).
//     Pointer jumping (Wyllie) gives every such node its junction root r(v) and
//     its distance dist(v) in O(log depth) rounds -- this is what makes the 1M
//     node chain (C2) cost 21 rounds instead of 1M frontier steps.
//  2. Kahn over the junctions only, with atomic join counters cnt[j] = indeg(j)
//     and a warp-aggregated frontier compaction: a contracted edge r(p) -> j
//     carries weight dist(p)+1, and level(j) = max(level(r(p)) + dist(p) + 1)
//     via atomicMax before the counter release.  The frontier expansion is
//     edge-balanced inside each warp (shuffle prefix sum + binary search), so
//     high-fan-out hubs do not serialise on one lane.
//  3. level(v) = level(r(v)) + dist(v) for the in-degree-1 nodes.
//  4. order = ids stably radix-sorted by level (ascending id inside a level),
//     level_ptr from the run boundaries.
// Nodes never resolved (on or below a cycle) are counted -> HF_ERR_CYCLE.
// Both persistent loops run as cooperative kernels with a grid barrier.
#include <algorithm>
#include <map>
#include <mutex>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "common.cuh"

namespace hf {

namespace {

struct GridBar {
    unsigned count;   // monotonic: arrivals over the kernel's lifetime
    unsigned pad;
};

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned *p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// Grid barrier for a cooperative launch: one release-add per CTA, then spin until
// all CTAs of this generation arrived (target grows by gridDim.x per call).
__device__ __forceinline__ void grid_sync(GridBar *b, unsigned &target) {
    target += gridDim.x;
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(&b->count) : "memory");
        while (ld_acquire_u32(&b->count) < target) __nanosleep(20);
    }
    __syncthreads();
}

__device__ __forceinline__ long long ld_pd(const long long *p) {
    return *reinterpret_cast<const volatile long long *>(p);
}
__device__ __forceinline__ void st_pd(long long *p, long long v) {
    *reinterpret_cast<volatile long long *>(p) = v;
}
__device__ __forceinline__ long long mk_pd(int parent, int dist) {
    return (long long)(((unsigned long long)(unsigned)dist << 32) | (unsigned)parent);
}
__device__ __forceinline__ int pd_parent(long long x) { return int(unsigned(x)); }
__device__ __forceinline__ int pd_dist(long long x) { return int(x >> 32); }

// warp-aggregated append of `item` when `pred` (all 32 lanes must call)
__device__ __forceinline__ void warp_append(bool pred, int item, int *list, int *count) {
    const int lane = threadIdx.x & 31;
    unsigned mask = __ballot_sync(0xffffffffu, pred);
    if (!mask) return;
    int leader = __ffs(mask) - 1;
    int base = 0;
    if (lane == leader) base = atomicAdd(count, __popc(mask));
    base = __shfl_sync(0xffffffffu, base, leader);
    if (pred) list[base + __popc(mask & ((1u << lane) - 1u))] = item;
}

// scalars: [0..2] active counts (rotating), [3..5] frontier counts (rotating),
//          [6] unresolved count, [7] max level, [8] visited junctions
enum { SC_ACT = 0, SC_FR = 3, SC_UNRES = 6, SC_MAXLV = 7, SC_VIS = 8 };

__global__ void k_lev_init(const int32_t *__restrict__ in_ptr, const int32_t *__restrict__ in_src,
                           int32_t n, long long *__restrict__ pd, int32_t *__restrict__ cnt,
                           int32_t *__restrict__ lev, int32_t *__restrict__ active,
                           int32_t *__restrict__ frontier, int32_t *sc) {
    __shared__ int s_w[33];
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    // block-uniform trip count (block_append synchronises the block)
    for (int64_t base = int64_t(blockIdx.x) * blockDim.x; base < n; base += stride) {
        const int64_t v = base + threadIdx.x;
        bool in = v < n;
        int deg = 0;
        if (in) {
            int b = in_ptr[v];
            deg = in_ptr[v + 1] - b;
            pd[v] = deg == 1 ? mk_pd(in_src[b], 1) : mk_pd(int(v), 0);
            cnt[v] = deg;
            lev[v] = 0;
        }
        block_append(in && deg == 1, int(v), active, sc + SC_ACT + 0, s_w);
        block_append(in && deg == 0, int(v), frontier, sc + SC_FR + 1, s_w);
    }
}

// Pointer jumping over the active in-degree-1 nodes until each points at its
// junction root (dist of a root is 0).  At most max_rounds rounds; nodes still
// active afterwards lie on/below an in-degree-1 cycle.
__global__ void k_lev_jump(long long *__restrict__ pd, int32_t *__restrict__ act_a,
                           int32_t *__restrict__ act_b, int32_t *sc, int max_rounds,
                           GridBar *bar) {
    const int64_t nthreads = int64_t(gridDim.x) * blockDim.x;
    // warp-granular interleave across SMs (a warp stays contiguous for coalescing)
    const int64_t tid = (int64_t(threadIdx.x >> 5) * gridDim.x + blockIdx.x) * 32 + (threadIdx.x & 31);
    int32_t *lists[2] = {act_a, act_b};
    __shared__ int s_w[33];
    unsigned bar_target = 0;
    for (int r = 0; r < max_rounds; ++r) {
        volatile int32_t *vsc = sc;
        int size = vsc[SC_ACT + r % 3];
        if (size == 0) break;
        if (tid == 0) vsc[SC_ACT + (r + 2) % 3] = 0;
        const int32_t *in = lists[r & 1];
        int32_t *out = lists[(r + 1) & 1];
        // block-uniform trip count (block_append synchronises the block)
        const int64_t iters = (int64_t(size) + nthreads - 1) / nthreads;
        for (int64_t it = 0; it < iters; ++it) {
            const int64_t i = tid + it * nthreads;
            bool keep = false;
            int v = 0;
            if (i < size) {
                v = __ldcg(in + i);
                long long x = ld_pd(pd + v);
                long long y = ld_pd(pd + pd_parent(x));
                if (pd_dist(y) != 0) {   // parent is not a root yet: jump
                    st_pd(pd + v, mk_pd(pd_parent(y), pd_dist(x) + pd_dist(y)));
                    keep = true;
                }
            }
            block_append(keep, v, out, sc + SC_ACT + (r + 1) % 3, s_w);
        }
        grid_sync(bar, bar_target);
    }
}

// Kahn over the junctions, frontier-synchronous; lev[j] = max(lev[r] + w) over the
// contracted edges r -> j (cdst, cw), released by the atomic join counter cnt[j].
__device__ __forceinline__ unsigned long long lev_gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

constexpr int KCH = 1;    // contracted edges per frontier entry (one lane per edge)
#ifndef KAHN_COOP_APPEND
#define KAHN_COOP_APPEND 1
#endif

// warp-aggregated append of `cnt` entries {start + t*KCH, node} (t < cnt) per lane
__device__ __forceinline__ void warp_append_chunks(int cnt, int start, int node, int2 *list,
                                                   int *count) {
    const int lane = threadIdx.x & 31;
    int incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    const int total = __shfl_sync(0xffffffffu, incl, 31);
    if (total == 0) return;
    int base = 0;
    if (lane == 31) base = atomicAdd(count, total);
    base = __shfl_sync(0xffffffffu, base, 31) + incl - cnt;
    for (int t = 0; t < cnt; ++t) list[base + t] = make_int2(start + t * KCH, node);
}

// warp-aggregated append with a 64-bit {arrivals:32 | count:32} round word: the
// count lives in the low half, so the barrier's spin read also returns the size
__device__ __forceinline__ void warp_append_chunks64(int cnt, int start, int node, int2 *list,
                                                     unsigned long long *word) {
    const int lane = threadIdx.x & 31;
    int incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    const int total = __shfl_sync(0xffffffffu, incl, 31);
    if (total == 0) return;
    int base = 0;
    if (lane == 31) base = int(unsigned(atomicAdd(word, (unsigned long long)total)));
    base = __shfl_sync(0xffffffffu, base, 31);
#if KAHN_COOP_APPEND
    // the warp writes its `total` entries together, 32 at a time: entry i belongs to
    // the lane o with excl[o] <= i < incl[o] (binary search over the lanes' inclusive
    // prefixes), so a hub's out-edges do not serialise on one lane
    const int excl = incl - cnt;
    for (int i0 = 0; i0 < total; i0 += 32) {
        const int i = i0 + lane;
        int o = 0;
#pragma unroll
        for (int b = 16; b >= 1; b >>= 1) {
            const int v = __shfl_sync(0xffffffffu, incl, o + b - 1);
            if (v <= i) o += b;
        }
        const int st = __shfl_sync(0xffffffffu, start, o);
        const int ex = __shfl_sync(0xffffffffu, excl, o);
        const int nd = __shfl_sync(0xffffffffu, node, o);
        if (i < total) list[base + i] = make_int2(st + (i - ex) * KCH, nd);
    }
#else
    base += incl - cnt;
    for (int t = 0; t < cnt; ++t) list[base + t] = make_int2(start + t * KCH, node);
#endif
}

// Kahn over the junctions, frontier-synchronous; lev[j] = max(lev[r] + w) over the
// contracted edges r -> j (cdst, cw), released by the atomic join counter cnt[j].
// A frontier entry is one contracted edge {edge, source node}: every lane does
// exactly one relaxation per round, so hub fan-outs are spread over the whole GPU.
// Round r+1's frontier is counted in the low half of the 64-bit word W[(r+1) % 3]
// and the grid barrier ending round r adds its arrivals to the high half, so one
// acquire read gives both "everyone arrived" and the next frontier size; the
// out-edge range of the target is loaded before the join-counter decrement returns.
__global__ void k_lev_kahn(const int32_t *__restrict__ cptr, const int32_t *__restrict__ cdst,
                           const int32_t *__restrict__ cw, int32_t *__restrict__ cnt,
                           int32_t *__restrict__ lev, int2 *__restrict__ fr_a,
                           int2 *__restrict__ fr_b, int32_t *sc, unsigned long long *W,
                           unsigned long long *trace) {
    __shared__ int s_size;
    const int lane = threadIdx.x & 31;
    const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
    // consecutive warp slots land on different SMs, so a small frontier is spread
    // over the whole GPU instead of the first few CTAs
    const int64_t wid = int64_t(threadIdx.x >> 5) * gridDim.x + blockIdx.x;
    int2 *lists[2] = {fr_a, fr_b};
    int size = reinterpret_cast<volatile int32_t *>(sc)[SC_FR + 0];   // seeded frontier
    for (int r = 0;; ++r) {
        if (size == 0) break;
        if (blockIdx.x == 0 && threadIdx.x == 0) W[(r + 2) % 3] = 0ull;
        const int2 *in = lists[r & 1];
        int2 *out = lists[(r + 1) & 1];
        unsigned long long *wn = W + (r + 1) % 3;
        if (trace && blockIdx.x == 0 && threadIdx.x == 0 && r < 4096) {
            trace[3 * r] = lev_gtimer();
            trace[3 * r + 2] = (unsigned long long)size;
        }
        for (int64_t base = wid * 32; base < size; base += nwarps * 32) {
            const int64_t i = base + lane;
            int nch = 0, kstart = 0, k = 0;
            if (i < size) {
                const int2 en = __ldcg(in + i);   // one contracted edge per entry
                k = __ldg(cdst + en.x);
                const int w = __ldg(cw + en.x);
                const int lj = __ldcg(lev + en.y);
                const int ks = __ldg(cptr + k), ke = __ldg(cptr + k + 1);   // speculative
                atomicMax(lev + k, lj + w);
                if (atomicSub(cnt + k, 1) == 1) {   // k ready: queue its out-edges
                    kstart = ks;
                    nch = ke - ks;
                }
            }
            warp_append_chunks64(nch, kstart, k, out, wn);
        }
        if (trace && blockIdx.x == 0 && threadIdx.x == 0 && r < 4096) trace[3 * r + 1] = lev_gtimer();
        // grid barrier fused with the next frontier's size
        __syncthreads();
        if (threadIdx.x == 0) {
            asm volatile("red.release.gpu.global.add.u64 [%0], %1;" ::"l"(wn),
                         "l"(1ull << 32)
                         : "memory");
            unsigned long long v;
            for (;;) {
                asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(wn) : "memory");
                if ((v >> 32) >= gridDim.x) break;
                __nanosleep(20);
            }
            s_size = int(unsigned(v));
        }
        __syncthreads();
        size = s_size;
    }
}

// ---- barrier-free Kahn over the junctions (HF_KAHN_ASYNC) -----------------------
// One list of contracted-edge entries {edge, level of its source} (64-bit words,
// pre-filled with the all-ones sentinel), appended in readiness order: position i
// is claimed by an atomic counter A and written once.  Warp w owns positions
// w*32 + lane + k*(warps*32): it polls its 32 positions, processes every entry that
// has arrived (cdst / cw / the target's out-edge range, atomicMax of the level,
// acq_rel decrement of the join counter); the lane that readies a junction reads its
// now final level and appends the junction's out-edges (warp-aggregated claim).
// There are no rounds and no grid barrier: the chain of dependent hops is the
// junction depth, every hop ~4 L2 round trips.  Termination: P counts processed
// entries (flushed by a warp once it has idled >= 4 us, so P stays off the hot path),
// appends precede their entry's P increment, so P == A (read in that order) means no
// entry is in flight and none can appear.  Cycles leave counters > 0 and simply end
// the same way.  A watchdog (globaltimer, HF_KAHN_WATCHDOG_MS, default 2000) aborts
// instead of hanging; the host then reports HF_ERR_CUDA.
__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed_u64(unsigned long long *p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ int ld_relaxed_s32(const int *p) {
    int v;
    asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ int atom_add_acq_rel(int *p, int v) {
    int old;
    asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
}
__device__ __forceinline__ int ld_acquire_s32(const int *p) {
    int v;
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// ctr: [0] A (appended), [1] P (processed), [2] abort flag
__global__ void __launch_bounds__(256) k_lev_kahn_async(
    const int32_t *__restrict__ cptr, const int32_t *__restrict__ cdst,
    const int32_t *__restrict__ cw, int32_t *__restrict__ cnt, int32_t *__restrict__ lev,
    unsigned long long *__restrict__ list, int64_t cap, int32_t *ctr,
    unsigned long long watchdog_ns) {
    const int lane = threadIdx.x & 31;
    const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
    const int64_t wid = int64_t(threadIdx.x >> 5) * gridDim.x + blockIdx.x;
    int myp = 0;                    // processed entries not yet published to P
    unsigned long long idle_since = 0;
    const unsigned long long t_start = lev_gtimer();
    for (int64_t base = wid * 32; base < cap; base += nwarps * 32) {
        const int64_t i = base + lane;
        bool pending = i < cap;
        int ns = 32;
        int a_seen = 0;   // a recent value of A: positions below it are claimed
        for (;;) {
            // poll only claimed positions (a claimed entry is written right after its
            // claim); a batch wholly past A waits on the counter alone
            const unsigned long long ev =
                (pending && i < a_seen) ? ld_relaxed_u64(list + i) : ~0ull;
            const bool have = ev != ~0ull;
            const unsigned hm = __ballot_sync(0xffffffffu, have);
            if (hm) {
                int nch = 0, ks = 0, lk = 0;
                if (have) {
                    const int e = int(unsigned(ev));
                    const int lj = int(unsigned(ev >> 32));
                    const int k = __ldg(cdst + e);
                    const int w = __ldg(cw + e);
                    ks = __ldg(cptr + k);
                    const int ke = __ldg(cptr + k + 1);
                    atomicMax(lev + k, lj + w);
                    // release: this level contribution before the decrement; acquire:
                    // the last decrementer sees every contribution
                    if (atom_add_acq_rel(cnt + k, -1) == 1) {
                        nch = ke - ks;
                        lk = ld_relaxed_s32(lev + k);   // final (ordered after the acquire)
                    }
                    pending = false;
                }
                // warp-aggregated claim of the readied junctions' out-edges
                int incl = nch;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int y = __shfl_up_sync(0xffffffffu, incl, o);
                    if (lane >= o) incl += y;
                }
                const int total = __shfl_sync(0xffffffffu, incl, 31);
                if (total) {
                    int b0 = 0;
                    if (lane == 31) b0 = atomicAdd(ctr + 0, total);
                    b0 = __shfl_sync(0xffffffffu, b0, 31) + incl - nch;
                    const unsigned long long hi = (unsigned long long)unsigned(lk) << 32;
                    for (int t = 0; t < nch; ++t)
                        st_relaxed_u64(list + b0 + t, hi | unsigned(ks + t));
                }
                myp += __popc(hm);
                idle_since = 0;
                ns = 32;
            }
            if (!__any_sync(0xffffffffu, pending)) break;
            // waiting: publish the processed count after a while, test for the end
            const unsigned long long now = lev_gtimer();
            if (idle_since == 0) idle_since = now;
            if (lane == 0 && myp && now - idle_since > 4000) {
                __threadfence();   // this warp's appends before its processed count
                atomicAdd(ctr + 1, myp);
                myp = 0;
            }
            myp = __shfl_sync(0xffffffffu, myp, 0);
            int done = 0, a = 0;
            if (lane == 0) {
                // P before A: P == A then means no entry was in flight when P was read,
                // so none can ever be appended (every pending position is >= A)
                const int pr = ld_acquire_s32(ctr + 1);
                a = ld_acquire_s32(ctr + 0);
                done = pr == a ? 1 : 0;
                if (ld_relaxed_s32(ctr + 2)) done = 2;
                if (now - t_start > watchdog_ns) {
                    atomicExch(ctr + 2, 1);
                    done = 2;
                }
            }
            done = __shfl_sync(0xffffffffu, done, 0);
            a_seen = __shfl_sync(0xffffffffu, a, 0);
            if (done == 2) return;
            if (done == 1) {
                // only lanes past the end remain: positions >= a never arrive
                if (lane == 0 && myp) atomicAdd(ctr + 1, myp);
                return;
            }
            // claimed positions pending: poll soon; otherwise the batch waits for appends
            const bool claimed = __any_sync(0xffffffffu, pending && i < a_seen);
            __nanosleep(claimed ? 32 : ns);
            ns = min(ns * 2, 1024);
        }
    }
    if (lane == 0 && myp) atomicAdd(ctr + 1, myp);
}

// seeds of the barrier-free Kahn: the sources' contracted out-edges {edge, level 0}
__global__ void k_lev_seed_async(const int32_t *__restrict__ src_list, const int32_t *__restrict__ cptr,
                                 const int32_t *sc, unsigned long long *__restrict__ list,
                                 int32_t *ctr) {
    const int size = sc[SC_FR + 1];
    const int lane = threadIdx.x & 31;
    const int64_t lim = (int64_t(size) + 31) / 32 * 32;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < lim;
         i += int64_t(gridDim.x) * blockDim.x) {
        int nch = 0, st = 0;
        if (i < size) {
            const int v = src_list[i];
            st = cptr[v];
            nch = cptr[v + 1] - st;
        }
        int incl = nch;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        const int total = __shfl_sync(0xffffffffu, incl, 31);
        if (total == 0) continue;
        int b0 = 0;
        if (lane == 31) b0 = atomicAdd(ctr + 0, total);
        b0 = __shfl_sync(0xffffffffu, b0, 31) + incl - nch;
        for (int t = 0; t < nch; ++t) list[b0 + t] = (unsigned long long)unsigned(st + t);
    }
}

// initial frontier: the sources' contracted out-edges as chunk entries
__global__ void k_lev_seed(const int32_t *__restrict__ src_list, const int32_t *__restrict__ cptr,
                           int2 *__restrict__ out, int32_t *sc) {
    const int size = sc[SC_FR + 1];   // sources were counted in slot 1 by k_lev_init
    const int64_t lim = (int64_t(size) + 31) / 32 * 32;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < lim;
         i += int64_t(gridDim.x) * blockDim.x) {
        int nch = 0, st = 0, v = 0;
        if (i < size) {
            v = src_list[i];
            st = cptr[v];
            nch = cptr[v + 1] - st;
        }
        warp_append_chunks(nch, st, v, out, sc + SC_FR + 0);
    }
}

// Contracted edges: every fan-in edge e = (p -> j) with j a junction of in-degree
// >= 2 and p resolved becomes r(p) -> j with weight dist(p) + 1.  Counting sort by
// r(p) (atomic cursors; order inside a row is irrelevant, max is commutative).
__device__ __forceinline__ int contracted_root(const int32_t *in_ptr, const long long *pd,
                                               int j, int p, int &w) {
    if (in_ptr[j + 1] - in_ptr[j] < 2) return -1;
    long long x = pd[p];
    int r = pd_parent(x);
    if (pd_dist(x) != 0 && pd_dist(pd[r]) != 0) return -1;   // p on/below a cycle
    w = pd_dist(x) + 1;
    return r;
}

// count pass: every contracted edge takes its slot in its root's row (the atomic's
// old value) and remembers {root, slot} and its weight, so the scatter pass is a
// sequential read plus one store per edge
__global__ void k_lev_ccount(const int32_t *__restrict__ in_ptr, const int32_t *__restrict__ in_src,
                             const int32_t *__restrict__ in_dst, const long long *__restrict__ pd,
                             int32_t m, int32_t *__restrict__ ccnt, int2 *__restrict__ eslot,
                             int32_t *__restrict__ ew) {
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < m;
         e += int64_t(gridDim.x) * blockDim.x) {
        int w = 0;
        const int r = contracted_root(in_ptr, pd, in_dst[e], in_src[e], w);
        eslot[e] = make_int2(r, r >= 0 ? atomicAdd(ccnt + r, 1) : 0);
        ew[e] = w;
    }
}

__global__ void k_lev_cscatter(const int32_t *__restrict__ in_dst, const int2 *__restrict__ eslot,
                               const int32_t *__restrict__ ew, int32_t m,
                               const int32_t *__restrict__ cptr, int32_t *__restrict__ cdst,
                               int32_t *__restrict__ cw) {
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < m;
         e += int64_t(gridDim.x) * blockDim.x) {
        const int2 rs = eslot[e];
        if (rs.x >= 0) {
            const int k = cptr[rs.x] + rs.y;
            cdst[k] = in_dst[e];
            cw[k] = ew[e];
        }
    }
}

// Level-ordered CSR for the propagation passes: flag[i] = row order[i] is long
// (degree > LO_SPLIT); flag[n] = 0 so the exclusive scan's last entry is the count.
__global__ void k_lo_flags(const int32_t *__restrict__ order, const int32_t *__restrict__ ptr,
                           int32_t n, int32_t *__restrict__ flag) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i <= n;
         i += int64_t(gridDim.x) * blockDim.x) {
        int f = 0;
        if (i < n) {
            const int v = order[i];
            f = ptr[v + 1] - ptr[v] > LO_SPLIT;
        }
        flag[i] = f;
    }
}
// stable partition of every level run of `order`: short rows, then long rows;
// also the row position of every node and the part count of every row
__global__ void k_lo_place(const int32_t *__restrict__ order, const int32_t *__restrict__ level,
                           const int32_t *__restrict__ level_ptr, const int32_t *__restrict__ fs,
                           const int32_t *__restrict__ flag, const int32_t *__restrict__ ptr,
                           int32_t n, int32_t *__restrict__ lo_node, int32_t *__restrict__ deg,
                           int32_t *__restrict__ parts, int32_t *__restrict__ pos_of,
                           int32_t *__restrict__ lstart) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i <= n;
         i += int64_t(gridDim.x) * blockDim.x) {
        if (i == n) {
            deg[n] = 0;
            parts[n] = 0;
            continue;
        }
        const int v = order[i];
        const int k = level[v];
        const int ls = level_ptr[k], le = level_ptr[k + 1];
        const int sl = fs[i] - fs[ls];
        const int nlong = fs[le] - fs[ls];
        const bool lng = flag[i] != 0;
        if (int(i) == ls) lstart[k] = le - nlong;   // first long row of the level
        const int pos = lng ? le - nlong + sl : ls + (int(i) - ls) - sl;
        const int d = ptr[v + 1] - ptr[v];
        lo_node[pos] = v;
        deg[pos] = d;
        parts[pos] = lng ? (d + LO_PE - 1) / LO_PE : 0;
        pos_of[v] = pos;
    }
}
// Per row i: the part count of a long row at its first part id (0 at its other
// part ids, so no fill of the array is needed: ids past the exact part count are
// never read) and the row of that part; per node u: its neighbour encoding, its id
// or -(first part id + 1) when its own row (this direction) is long, so the relabel
// reads one value per edge.
__global__ void k_lo_np_enc(const int32_t *__restrict__ lo_q, const int32_t *__restrict__ ptr,
                            const int32_t *__restrict__ pos, int32_t n, int32_t *__restrict__ np,
                            int32_t *__restrict__ prow, int32_t *__restrict__ enc) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x) {
        const int q0 = lo_q[i], q1 = lo_q[i + 1];
        if (q1 != q0) {
            np[q0] = q1 - q0;
            prow[q0] = int32_t(i);
            for (int q = q0 + 1; q < q1; ++q) np[q] = 0;
        }
        enc[i] = ptr[i + 1] - ptr[i] > LO_SPLIT ? -(lo_q[pos[i]] + 1) : int32_t(i);
    }
}
// A warp copies the rows of 32 consecutive output positions as one flattened edge
// range: every output store is coalesced and every lane does one edge per step (a
// lane finds its row by a shuffle binary search over the warp's row offsets).
__global__ void k_relabel_rows(const int32_t *__restrict__ order, int32_t n,
                               const int32_t *__restrict__ ptr, const int32_t *__restrict__ a,
                               const int32_t *__restrict__ eid_map,
                               const int32_t *__restrict__ nptr, const int32_t *__restrict__ enc,
                               int32_t *__restrict__ na, int32_t *__restrict__ neid) {
    const int lane = threadIdx.x & 31;
    const int64_t nwarps_total = (int64_t(gridDim.x) * blockDim.x) >> 5;
    for (int64_t wbase = ((int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5) * 32;
         wbase < n; wbase += nwarps_total * 32) {
        const int64_t i = wbase + lane;
        int b = 0, len = 0;
        if (i < n) {
            const int v = order[i];
            b = ptr[v];
            len = ptr[v + 1] - b;
        }
        int incl = len;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        const int excl = incl - len;
        const int total = __shfl_sync(0xffffffffu, incl, 31);
        const int o0 = nptr[wbase];
        for (int base = 0; base < total; base += 32) {
            const int p = base + lane;
            // last row r with excl[r] <= p (empty rows share their successor's offset)
            int r = 0;
#pragma unroll
            for (int st = 16; st; st >>= 1) {
                const int c = r + st;
                if (__shfl_sync(0xffffffffu, excl, c) <= p) r = c;
            }
            const int er = __shfl_sync(0xffffffffu, excl, r);
            const int br = __shfl_sync(0xffffffffu, b, r);
            if (p < total) {
                const int k = br + (p - er);
                na[o0 + p] = enc[a[k]];
                neid[o0 + p] = eid_map ? eid_map[k] : k;
            }
        }
    }
}

__global__ void k_lev_final(const long long *__restrict__ pd, const int32_t *__restrict__ cnt,
                            const int32_t *__restrict__ lev, int32_t n,
                            int32_t *__restrict__ level, int32_t *sc) {
    int unres = 0, mx = -1;
    for (int64_t v = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; v < n;
         v += int64_t(gridDim.x) * blockDim.x) {
        long long x = pd[v];
        int lv = -1;
        if (pd_dist(x) == 0) {
            if (cnt[v] == 0) lv = lev[v];
        } else {
            int r = pd_parent(x);
            if (pd_dist(pd[r]) == 0 && cnt[r] == 0) lv = lev[r] + pd_dist(x);
        }
        level[v] = lv;
        if (lv < 0) ++unres;
        mx = max(mx, lv);
    }
    // one atomic per block (per-warp atomics on one address serialise)
    __shared__ int s_un, s_mx;
    if (threadIdx.x == 0) {
        s_un = 0;
        s_mx = -1;
    }
    __syncthreads();
    unres = __reduce_add_sync(0xffffffffu, unres);
    mx = __reduce_max_sync(0xffffffffu, mx);
    if ((threadIdx.x & 31) == 0) {
        if (unres) atomicAdd(&s_un, unres);
        atomicMax(&s_mx, mx);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        if (s_un) atomicAdd(sc + SC_UNRES, s_un);
        atomicMax(sc + SC_MAXLV, s_mx);
    }
}

__global__ void k_set_scalars(int32_t *sc) {
    if (threadIdx.x < 16) sc[threadIdx.x] = 0;
    if (threadIdx.x == 0) sc[SC_MAXLV] = -1;
}

int env_int_l(const char *name, int dflt) {
    const char *e = getenv(name);
    return e ? atoi(e) : dflt;
}

// Persistent cooperative grid: at most `cap` CTAs per SM (fewer CTAs = cheaper
// grid barrier; the per-round work of these loops is small).
int coop_grid(const void *func, int block, int sms, int cap = 2) {
    // occupancy queries are cached: driver calls inside the timed step are avoided
    static std::map<std::pair<const void *, int>, int> cache;
    static std::mutex mu;
    int per_sm = 0;
    {
        std::lock_guard<std::mutex> lk(mu);
        auto it = cache.find({func, block});
        if (it != cache.end()) per_sm = it->second;
    }
    if (!per_sm) {
        HF_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, func, block, 0));
        std::lock_guard<std::mutex> lk(mu);
        cache[{func, block}] = per_sm;
    }
    if (per_sm < 1) fail(HF_ERR_CUDA, "cooperative kernel cannot be resident");
    return std::min(per_sm, cap) * sms;
}

}  // namespace

// Returns the number of never-ready nodes (0 on success); fills g.level/order/level_ptr.
int64_t levelize_device(Graph &g) {
    StageTimes lt("HF_LEV_TIMES", "levelize");
    cudaStream_t s = g.stream;
    const int32_t n = g.n, m = g.m;
    g.levelized = false;
    g.L = -1;
    g.level.alloc(sizeof(int32_t) * int64_t(n > 0 ? n : 1), s);
    g.order.alloc(sizeof(int32_t) * int64_t(n > 0 ? n : 1), s);
    g.level_ptr.alloc(sizeof(int32_t) * (int64_t(n) + 1), s);
    if (n == 0) {
        HF_CUDA(cudaMemsetAsync(g.level_ptr.p, 0, sizeof(int32_t), s));
        g.L = 0;
        g.levelized = true;
        HF_CUDA(cudaStreamSynchronize(s));
        return 0;
    }
    DevBuf pd, cnt, lev, la, lb, bar, skeys, cptr;
    lt.mark("start", s);
    pd.alloc(sizeof(long long) * n, s);
    cnt.alloc(sizeof(int32_t) * n, s);
    lev.alloc(sizeof(int32_t) * n, s);
    la.alloc(sizeof(int32_t) * n, s);
    lb.alloc(sizeof(int32_t) * n, s);
    bar.alloc(sizeof(GridBar), s);
    HF_CUDA(cudaMemsetAsync(bar.p, 0, sizeof(GridBar), s));
    int32_t *sc = g.d_scalars();
    k_set_scalars<<<1, 32, 0, s>>>(sc);
    HF_CHECK_LAUNCH();
    // frontier list F0 goes to `lb` (separate from the active list in `la`)
    k_lev_init<<<grid_for(n, 256, g.sms), 256, 0, s>>>(
        g.in_ptr.as<int32_t>(), g.in_src.as<int32_t>(), n, pd.as<long long>(),
        cnt.as<int32_t>(), lev.as<int32_t>(), la.as<int32_t>(), lb.as<int32_t>(), sc);
    HF_CHECK_LAUNCH();
    g.launches += 2;
    lt.mark("init", s);
    {
        // pointer jumping: lists la (active) / keys buffer as ping-pong partner
        DevBuf act2;
        act2.alloc(sizeof(int32_t) * n, s);
        int max_rounds = bits_for(n) + 2;
        const int block = std::max(64, std::min(1024, getenv("HF_JUMP_BLOCK") ? atoi(getenv("HF_JUMP_BLOCK")) : 1024));
        int grid = coop_grid((const void *)k_lev_jump, block, g.sms, 1);
        long long *pdp = pd.as<long long>();
        int32_t *a = la.as<int32_t>(), *b = act2.as<int32_t>();
        GridBar *barp = bar.as<GridBar>();
        void *args[] = {&pdp, &a, &b, &sc, &max_rounds, &barp};
        HF_CUDA(cudaLaunchCooperativeKernel((const void *)k_lev_jump, grid, block, args, 0, s));
        g.launches += 1;
    }
    lt.mark("jump", s);
    // contracted fan-out of the junctions (counting sort by root)
    DevBuf ccur, cdst, cw;
    cptr.alloc(sizeof(int32_t) * (int64_t(n) + 1), s);
    ccur.alloc(sizeof(int32_t) * (int64_t(n) + 1), s);
    cdst.alloc(sizeof(int32_t) * int64_t(m > 0 ? m : 1), s);
    cw.alloc(sizeof(int32_t) * int64_t(m > 0 ? m : 1), s);
    HF_CUDA(cudaMemsetAsync(ccur.p, 0, sizeof(int32_t) * (int64_t(n) + 1), s));
    {
        DevBuf eslot, ew;
        eslot.alloc(sizeof(int2) * int64_t(m > 0 ? m : 1), s);
        ew.alloc(sizeof(int32_t) * int64_t(m > 0 ? m : 1), s);
        if (m) {
            k_lev_ccount<<<grid_for(m, 256, g.sms), 256, 0, s>>>(
                g.in_ptr.as<int32_t>(), g.in_src.as<int32_t>(), g.in_dst.as<int32_t>(),
                pd.as<long long>(), m, ccur.as<int32_t>(), eslot.as<int2>(), ew.as<int32_t>());
            HF_CHECK_LAUNCH();
            g.launches += 1;
        }
        scan_exclusive(ccur.as<int32_t>(), cptr.as<int32_t>(), int64_t(n) + 1, nullptr, s, g);
        if (m) {
            k_lev_cscatter<<<grid_for(m, 256, g.sms), 256, 0, s>>>(
                g.in_dst.as<int32_t>(), eslot.as<int2>(), ew.as<int32_t>(), m, cptr.as<int32_t>(),
                cdst.as<int32_t>(), cw.as<int32_t>());
            HF_CHECK_LAUNCH();
            g.launches += 1;
        }
    }
    if (env_int_l("HF_KAHN_ASYNC", 0)) {
        // barrier-free Kahn: one list of all contracted-edge entries (<= cptr[n] <= m)
        DevBuf lst, ctr;
        const int64_t cap = std::max<int64_t>(m, 1);
        lst.alloc(sizeof(unsigned long long) * size_t(cap), s);
        ctr.alloc(sizeof(int32_t) * 4, s);
        HF_CUDA(cudaMemsetAsync(lst.p, 0xff, sizeof(unsigned long long) * size_t(cap), s));
        HF_CUDA(cudaMemsetAsync(ctr.p, 0, sizeof(int32_t) * 4, s));
        k_lev_seed_async<<<grid_for(n, 256, g.sms), 256, 0, s>>>(lb.as<int32_t>(), cptr.as<int32_t>(),
                                                                sc, lst.as<unsigned long long>(),
                                                                ctr.as<int32_t>());
        HF_CHECK_LAUNCH();
        lt.mark("contract+seed", s);
        const int per_sm = std::max(1, env_int_l("HF_KAHN_ASYNC_CTAS", 4));
        int grid = coop_grid((const void *)k_lev_kahn_async, 256, g.sms, per_sm);
        const int32_t *cp = cptr.as<int32_t>(), *cd = cdst.as<int32_t>(), *cwp = cw.as<int32_t>();
        int32_t *cn = cnt.as<int32_t>(), *lv = lev.as<int32_t>();
        unsigned long long *lp = lst.as<unsigned long long>();
        int32_t *cp2 = ctr.as<int32_t>();
        int64_t capv = cap;
        unsigned long long wd = 1000000ull * (unsigned long long)env_int_l("HF_KAHN_WATCHDOG_MS", 2000);
        void *args[] = {&cp, &cd, &cwp, &cn, &lv, &lp, &capv, &cp2, &wd};
        // cooperative launch only for the co-residency guarantee (the wait is a poll)
        HF_CUDA(cudaLaunchCooperativeKernel((const void *)k_lev_kahn_async, grid, 256, args, 0, s));
        g.launches += 3;
        lt.mark("kahn", s);
        int32_t abort_flag = 0;
        HF_CUDA(cudaMemcpyAsync(&abort_flag, cp2 + 2, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
        HF_CUDA(cudaStreamSynchronize(s));
        if (abort_flag) fail(HF_ERR_CUDA, "levelizer watchdog expired (barrier-free Kahn)");
    } else {
        // frontier entries {first contracted edge, node}: at most n + m/KCH per round
        DevBuf ea, eb2;
        const size_t ecap = size_t(n) + size_t(m) / KCH + 1;
        ea.alloc(sizeof(int2) * ecap, s);
        eb2.alloc(sizeof(int2) * ecap, s);
        k_lev_seed<<<grid_for(n, 256, g.sms), 256, 0, s>>>(lb.as<int32_t>(), cptr.as<int32_t>(),
                                                          ea.as<int2>(), sc);
        HF_CHECK_LAUNCH();
        g.launches += 1;
        HF_CUDA(cudaMemsetAsync(sc + SC_FR + 1, 0, sizeof(int32_t), s));   // round 0 appends here
        lt.mark("contract+seed", s);
        const int block = std::max(64, std::min(1024, getenv("HF_KAHN_BLOCK") ? atoi(getenv("HF_KAHN_BLOCK")) : 1024));
        int grid = coop_grid((const void *)k_lev_kahn, block, g.sms, 1);
        DevBuf wbuf;   // three 64-bit round words {arrivals | frontier size}
        wbuf.alloc(sizeof(unsigned long long) * 3, s);
        HF_CUDA(cudaMemsetAsync(wbuf.p, 0, sizeof(unsigned long long) * 3, s));
        const int32_t *cp = cptr.as<int32_t>(), *cd = cdst.as<int32_t>(), *cwp = cw.as<int32_t>();
        int32_t *cn = cnt.as<int32_t>(), *lv = lev.as<int32_t>();
        int2 *fa = ea.as<int2>(), *fb = eb2.as<int2>();
        unsigned long long *wp = wbuf.as<unsigned long long>();
        const char *trace_env = getenv("HF_TRACE");
        DevBuf tb;
        unsigned long long *tr = nullptr;
        if (trace_env) {
            tb.alloc(sizeof(unsigned long long) * 3 * 4096, s);
            HF_CUDA(cudaMemsetAsync(tb.p, 0, sizeof(unsigned long long) * 3 * 4096, s));
            tr = tb.as<unsigned long long>();
        }
        void *args[] = {&cp, &cd, &cwp, &cn, &lv, &fa, &fb, &sc, &wp, &tr};
        HF_CUDA(cudaLaunchCooperativeKernel((const void *)k_lev_kahn, grid, block, args, 0, s));
        g.launches += 1;
        lt.mark("kahn", s);
        if (trace_env) {
            std::vector<unsigned long long> h(3 * 4096);
            HF_CUDA(cudaMemcpyAsync(h.data(), tr, h.size() * 8, cudaMemcpyDeviceToHost, s));
            HF_CUDA(cudaStreamSynchronize(s));
            std::string fn = std::string(trace_env) + "_kahn.bin";
            if (FILE *f = fopen(fn.c_str(), "wb")) {
                fwrite(h.data(), 8, h.size(), f);
                fclose(f);
            }
        }
    }
    k_lev_final<<<grid_for(n, 256, g.sms), 256, 0, s>>>(pd.as<long long>(), cnt.as<int32_t>(),
                                                        lev.as<int32_t>(), n,
                                                        g.level.as<int32_t>(), sc);
    HF_CHECK_LAUNCH();
    g.launches += 1;
    int32_t h_sc[16];
    HF_CUDA(cudaMemcpyAsync(h_sc, sc, sizeof(h_sc), cudaMemcpyDeviceToHost, s));
    lt.mark("final", s);
    HF_CUDA(cudaStreamSynchronize(s));
    int64_t unresolved = h_sc[SC_UNRES];
    if (unresolved) return unresolved;
    const int32_t L = h_sc[SC_MAXLV] + 1;
    // canonical order: ids stably sorted by level
    skeys.alloc(sizeof(int32_t) * n, s);
    radix_sort_pairs(g.level.as<int32_t>(), nullptr, skeys.as<int32_t>(), g.order.as<int32_t>(),
                     n, bits_for(int64_t(L) - 1), s, g);
    keys_to_ptr(skeys.as<int32_t>(), n, L, g.level_ptr.as<int32_t>(), s, g);
    lt.mark("sync+sort", s);
    // relabel (a4): level-ordered CSR for the propagation passes.
    // Inside a level the rows with degree <= LO_SPLIT come first, then the longer
    // rows (cut into part tasks by the passes); both runs keep canonical order.
    {
        const int64_t mm = m > 0 ? m : 1;
        // +LO_PAD elements: the level-synchronous passes stage 16-byte-aligned runs of
        // these arrays with bulk copies that may read up to 3 elements past the end
        g.lo_in_node.alloc(sizeof(int32_t) * (int64_t(n) + LO_PAD), s);
        g.lo_out_node.alloc(sizeof(int32_t) * (int64_t(n) + LO_PAD), s);
        g.lo_in_ptr.alloc(sizeof(int32_t) * (int64_t(n) + 1 + LO_PAD), s);
        g.lo_out_ptr.alloc(sizeof(int32_t) * (int64_t(n) + 1 + LO_PAD), s);
        g.lo_in_q.alloc(sizeof(int32_t) * (int64_t(n) + 1 + LO_PAD), s);
        g.lo_out_q.alloc(sizeof(int32_t) * (int64_t(n) + 1 + LO_PAD), s);
        g.lo_in_nbr.alloc(sizeof(int32_t) * (mm + LO_PAD), s);
        g.lo_in_eid.alloc(sizeof(int32_t) * (mm + LO_PAD), s);
        g.lo_out_nbr.alloc(sizeof(int32_t) * (mm + LO_PAD), s);
        g.lo_out_eid.alloc(sizeof(int32_t) * (mm + LO_PAD), s);
        // the two directions are independent: fan-out on the side stream, fan-in here
        DevBuf flag[2], fs[2], deg[2], parts[2], pos[2], enc[2];
        const size_t npcap = size_t(m / (LO_SPLIT + 1) + m / LO_PE + 1);
        for (int dir = 0; dir < 2; ++dir) {
            flag[dir].alloc(sizeof(int32_t) * (int64_t(n) + 1), s);
            fs[dir].alloc(sizeof(int32_t) * (int64_t(n) + 1), s);
            deg[dir].alloc(sizeof(int32_t) * (int64_t(n) + 1), s);
            parts[dir].alloc(sizeof(int32_t) * (int64_t(n) + 1), s);
            pos[dir].alloc(sizeof(int32_t) * n, s);
            enc[dir].alloc(sizeof(int32_t) * n, s);
            // parts of every long row, indexed by its first part id (<= m/9 + m/LO_PE ids)
            (dir == 0 ? g.lo_in_np : g.lo_out_np).alloc(sizeof(int32_t) * npcap * 2, s);
            (dir == 0 ? g.lo_in_lstart : g.lo_out_lstart).alloc(sizeof(int32_t) * (int64_t(L) + 1), s);
        }
        g.np_cap_in = g.np_cap_out = int32_t(npcap);
        Side &sd = side_of(g);
        HF_CUDA(cudaEventRecord(sd.fork, s));
        HF_CUDA(cudaStreamWaitEvent(sd.s2, sd.fork, 0));
        for (int dir = 1; dir >= 0; --dir) {
            const bool in = dir == 0;
            cudaStream_t ds = in ? s : sd.s2;
            const int32_t *ptr = in ? g.in_ptr.as<int32_t>() : g.out_ptr.as<int32_t>();
            int32_t *lo_node = in ? g.lo_in_node.as<int32_t>() : g.lo_out_node.as<int32_t>();
            int32_t *lo_ptr = in ? g.lo_in_ptr.as<int32_t>() : g.lo_out_ptr.as<int32_t>();
            int32_t *lo_q = in ? g.lo_in_q.as<int32_t>() : g.lo_out_q.as<int32_t>();
            DevBuf &np = in ? g.lo_in_np : g.lo_out_np;
            k_lo_flags<<<grid_for(int64_t(n) + 1, 256, g.sms), 256, 0, ds>>>(
                g.order.as<int32_t>(), ptr, n, flag[dir].as<int32_t>());
            HF_CHECK_LAUNCH();
            scan_exclusive(flag[dir].as<int32_t>(), fs[dir].as<int32_t>(), int64_t(n) + 1, nullptr,
                           ds, g, dir);
            DevBuf &lst = in ? g.lo_in_lstart : g.lo_out_lstart;
            k_lo_place<<<grid_for(int64_t(n) + 1, 256, g.sms), 256, 0, ds>>>(
                g.order.as<int32_t>(), g.level.as<int32_t>(), g.level_ptr.as<int32_t>(),
                fs[dir].as<int32_t>(), flag[dir].as<int32_t>(), ptr, n, lo_node,
                deg[dir].as<int32_t>(), parts[dir].as<int32_t>(), pos[dir].as<int32_t>(),
                lst.as<int32_t>());
            HF_CHECK_LAUNCH();
            scan_exclusive(deg[dir].as<int32_t>(), lo_ptr, int64_t(n) + 1, nullptr, ds, g, dir);
            scan_exclusive(parts[dir].as<int32_t>(), lo_q, int64_t(n) + 1, sc + 12 + dir, ds, g,
                           dir);
            k_lo_np_enc<<<grid_for(n, 256, g.sms), 256, 0, ds>>>(
                lo_q, ptr, pos[dir].as<int32_t>(), n, np.as<int32_t>(), np.as<int32_t>() + npcap,
                enc[dir].as<int32_t>());
            HF_CHECK_LAUNCH();
            if (in)
                k_relabel_rows<<<grid_for(n, 256, g.sms), 256, 0, ds>>>(
                    lo_node, n, ptr, g.in_src.as<int32_t>(), nullptr, lo_ptr,
                    enc[dir].as<int32_t>(), g.lo_in_nbr.as<int32_t>(), g.lo_in_eid.as<int32_t>());
            else
                k_relabel_rows<<<grid_for(n, 256, g.sms), 256, 0, ds>>>(
                    lo_node, n, ptr, g.out_dst.as<int32_t>(), g.out_eid.as<int32_t>(), lo_ptr,
                    enc[dir].as<int32_t>(), g.lo_out_nbr.as<int32_t>(), g.lo_out_eid.as<int32_t>());
            HF_CHECK_LAUNCH();
            g.launches += 4;   // flags, place, np_enc, relabel (scans count themselves)
        }
        HF_CUDA(cudaEventRecord(sd.join, sd.s2));
        HF_CUDA(cudaStreamWaitEvent(s, sd.join, 0));   // before the scratch is freed on s
        lt.mark("relabel", s);
    }
    // no second host round trip: the passes size the part buffers by the bound
    // np_cap and read the exact part counts (sc[12], sc[13]) on the device
    g.nparts_d = sc + 12;
    g.ts_f.key = g.ts_b.key = -1;   // task schedules depend on the levels
    g.wide_ready = g.lo_d_ready = g.w2_ready = g.pnbr_ready = g.w3_ready = false;
    g.L = L;
    g.levelized = true;
    return 0;
}

}  // namespace hf
