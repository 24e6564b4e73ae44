// primitives.cu -- device building blocks for graph ingest and levelization:
// single-pass (decoupled look-back) exclusive scan, stable LSD radix sort (8-bit digits, warp-match
// ranking), sorted-keys -> CSR offsets, CSR row ids.  All hand-written sm_100a.
#include <algorithm>

#include "common.cuh"

namespace hf {

namespace {

// Block-wide exclusive sum of one value per thread; returns prefix, writes total.
__device__ __forceinline__ int block_exclusive_sum(int v, int *total) {
    __shared__ int warp_sums[32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) warp_sums[wid] = x;
    __syncthreads();
    const int nw = blockDim.x >> 5;
    if (wid == 0) {
        int s = lane < nw ? warp_sums[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int y = __shfl_up_sync(0xffffffffu, s, o);
            if (lane >= o) s += y;
        }
        if (lane < nw) warp_sums[lane] = s;
    }
    __syncthreads();
    int before = wid ? warp_sums[wid - 1] : 0;
    if (total) *total = warp_sums[nw - 1];
    int r = before + x - v;
    __syncthreads();
    return r;
}

// ---- single-pass scan (decoupled look-back) --------------------------------
// Tiles take ids in launch order from a monotonic counter (ids of this call start
// at `base`), so every predecessor tile is already running: no deadlock.  Each
// tile publishes its aggregate, then its inclusive prefix, as one 64-bit word
// {tag:32 | value:32} with tag = epoch*4 + kind (1 = aggregate, 2 = inclusive);
// words of older calls carry an older epoch and read as "not yet published".
constexpr int LB_BLOCK = 256;
constexpr int LB_ITEMS = 16;
constexpr int LB_TILE = LB_BLOCK * LB_ITEMS;

__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed_u64(unsigned long long *p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__global__ void __launch_bounds__(LB_BLOCK) k_scan_lookback(
    const int32_t *__restrict__ in, int32_t *__restrict__ out, int64_t count,
    unsigned long long *__restrict__ state, unsigned *__restrict__ ctr, unsigned base,
    unsigned epoch, int32_t *__restrict__ total) {
    __shared__ unsigned s_tile;
    __shared__ int s_excl;
    if (threadIdx.x == 0) s_tile = atomicAdd(ctr, 1u) - base;
    __syncthreads();
    const unsigned tile = s_tile;
    const int64_t i0 = int64_t(tile) * LB_TILE + int64_t(threadIdx.x) * LB_ITEMS;
    int v[LB_ITEMS];
    int sum = 0;
    if (i0 + LB_ITEMS <= count && (reinterpret_cast<uintptr_t>(in + i0) & 15) == 0) {
#pragma unroll
        for (int j = 0; j < LB_ITEMS; j += 4) {
            const int4 q = *reinterpret_cast<const int4 *>(in + i0 + j);
            v[j] = q.x; v[j + 1] = q.y; v[j + 2] = q.z; v[j + 3] = q.w;
        }
    } else {
#pragma unroll
        for (int j = 0; j < LB_ITEMS; ++j) v[j] = (i0 + j < count) ? in[i0 + j] : 0;
    }
#pragma unroll
    for (int j = 0; j < LB_ITEMS; ++j) sum += v[j];
    int agg;
    int pre = block_exclusive_sum(sum, &agg);
    const unsigned long long tagA = (unsigned long long)(epoch * 4u + 1u) << 32;
    const unsigned long long tagP = (unsigned long long)(epoch * 4u + 2u) << 32;
    if (threadIdx.x < 32) {
        int excl = 0;
        if (tile == 0) {
            if (threadIdx.x == 0) st_relaxed_u64(state, tagP | unsigned(agg));
        } else {
            if (threadIdx.x == 0) st_relaxed_u64(state + tile, tagA | unsigned(agg));
            // look back over windows of 32 predecessors
            int64_t look = int64_t(tile) - 1;
            const int lane = threadIdx.x;
            for (;;) {
                const int64_t j = look - lane;
                unsigned long long w = 0;
                unsigned kind = 0;
                if (j >= 0) {
                    do {
                        w = ld_relaxed_u64(state + j);
                        const unsigned tag = unsigned(w >> 32);
                        kind = (tag >> 2) == epoch ? (tag & 3u) : 0u;
                    } while (kind == 0);
                }
                // lanes past the first inclusive prefix (in look-back order) are ignored
                const unsigned pmask = __ballot_sync(0xffffffffu, j >= 0 && kind == 2);
                const int stop = pmask ? __ffs(pmask) - 1 : 31;
                int val = (j >= 0 && lane <= stop) ? int(unsigned(w)) : 0;
#pragma unroll
                for (int o = 16; o; o >>= 1) val += __shfl_xor_sync(0xffffffffu, val, o);
                excl += val;
                if (pmask || look - 32 < 0) break;
                look -= 32;
            }
            if (lane == 0) st_relaxed_u64(state + tile, tagP | unsigned(excl + agg));
        }
        if (threadIdx.x == 0) {
            s_excl = excl;
            const int64_t last = (count - 1) / LB_TILE;
            if (total && int64_t(tile) == last) *total = excl + agg;
        }
    }
    __syncthreads();
    pre += s_excl;
#pragma unroll
    for (int j = 0; j < LB_ITEMS; ++j) {
        if (i0 + j < count) out[i0 + j] = pre;
        pre += v[j];
    }
}

// ---- radix sort ----------------------------------------------------------
constexpr int RS_BLOCK = 256;
constexpr int RS_ROUNDS = 16;
constexpr int RS_TILE = RS_BLOCK * RS_ROUNDS;   // 4096 items per tile

__global__ void __launch_bounds__(RS_BLOCK) k_radix_upsweep(const int32_t *__restrict__ keys,
                                                            int64_t count, int shift,
                                                            int32_t *__restrict__ hist,
                                                            int nblocks) {
    __shared__ int h[256];
    h[threadIdx.x] = 0;
    __syncthreads();
    int64_t base = int64_t(blockIdx.x) * RS_TILE + threadIdx.x;
#pragma unroll 4
    for (int r = 0; r < RS_ROUNDS; ++r) {
        int64_t i = base + int64_t(r) * RS_BLOCK;
        if (i < count) atomicAdd(&h[(keys[i] >> shift) & 255], 1);
    }
    __syncthreads();
    hist[int64_t(threadIdx.x) * nblocks + blockIdx.x] = h[threadIdx.x];
}

__global__ void __launch_bounds__(RS_BLOCK) k_radix_downsweep(
    const int32_t *__restrict__ keys, const int32_t *__restrict__ vals,
    int32_t *__restrict__ keys_out, int32_t *__restrict__ vals_out, int64_t count, int shift,
    const int32_t *__restrict__ offsets, int nblocks) {
    __shared__ int run[256];
    __shared__ int base_off[256];
    __shared__ int wcnt[RS_BLOCK / 32][256];
    const int t = threadIdx.x, w = t >> 5, lane = t & 31;
    base_off[t] = offsets[int64_t(t) * nblocks + blockIdx.x];
    run[t] = 0;
#pragma unroll
    for (int w2 = 0; w2 < RS_BLOCK / 32; ++w2) wcnt[w2][t] = 0;
    __syncthreads();
    const unsigned lt_mask = (1u << lane) - 1u;
    const int64_t tile = int64_t(blockIdx.x) * RS_TILE;
    for (int r = 0; r < RS_ROUNDS; ++r) {
        int64_t i = tile + int64_t(r) * RS_BLOCK + t;
        bool valid = i < count;
        int key = valid ? keys[i] : 0;
        int val = valid ? (vals ? vals[i] : int(i)) : 0;
        int digit = valid ? ((key >> shift) & 255) : 256;
        unsigned peers = __match_any_sync(0xffffffffu, digit);
        int wrank = __popc(peers & lt_mask);
        if (valid && lane == __ffs(peers) - 1) wcnt[w][digit] = __popc(peers);
        __syncthreads();
        if (valid) {
            int pre = run[digit];
            for (int w2 = 0; w2 < w; ++w2) pre += wcnt[w2][digit];
            int pos = base_off[digit] + pre + wrank;
            keys_out[pos] = key;
            vals_out[pos] = val;
        }
        __syncthreads();
        int sum = 0;
#pragma unroll
        for (int w2 = 0; w2 < RS_BLOCK / 32; ++w2) {
            sum += wcnt[w2][t];
            wcnt[w2][t] = 0;
        }
        run[t] += sum;
        __syncthreads();
    }
}

__global__ void k_run_bounds(const int32_t *__restrict__ keys, int64_t count,
                             int32_t *__restrict__ acc) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < count;
         i += int64_t(gridDim.x) * blockDim.x) {
        int k = keys[i];
        if (i == 0 || keys[i - 1] != k) atomicSub(&acc[k], int(i));
        if (i == count - 1 || keys[i + 1] != k) atomicAdd(&acc[k], int(i + 1));
    }
}

// One lane per row; rows of >= 64 entries are written by the whole warp.
__global__ void k_row_ids(const int32_t *__restrict__ ptr, int32_t nrows,
                          int32_t *__restrict__ row_of) {
    const int lane = threadIdx.x & 31;
    const int64_t nwarps_total = (int64_t(gridDim.x) * blockDim.x) >> 5;
    for (int64_t wbase = ((int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5) * 32;
         wbase < nrows; wbase += nwarps_total * 32) {
        int64_t v = wbase + lane;
        int b = 0, e = 0;
        if (v < nrows) {
            b = ptr[v];
            e = ptr[v + 1];
        }
        bool longrow = (e - b) >= 64;
        if (!longrow)
            for (int k = b; k < e; ++k) row_of[k] = int(v);
        unsigned lm = __ballot_sync(0xffffffffu, longrow);
        while (lm) {
            int src = __ffs(lm) - 1;
            lm &= lm - 1;
            int bb = __shfl_sync(0xffffffffu, b, src);
            int ee = __shfl_sync(0xffffffffu, e, src);
            int vv = int(wbase + src);
            for (int k = bb + lane; k < ee; k += 32) row_of[k] = vv;
        }
    }
}

}  // namespace

void scan_exclusive(const int32_t *in, int32_t *out, int64_t count, int32_t *total_d,
                    cudaStream_t s, Graph &g, int slot) {
    if (count <= 0) {
        if (total_d) HF_CUDA(cudaMemsetAsync(total_d, 0, sizeof(int32_t), s));
        return;
    }
    const int64_t tiles = (count + LB_TILE - 1) / LB_TILE;
    // look-back state: one word per tile + the tile counter, zeroed once on growth
    const size_t need = sizeof(unsigned long long) * size_t(tiles + 1);
    Graph::ScanState &ss = g.scan[slot];
    if (ss.buf.bytes < need || ss.buf.s != s) {
        ss.buf.alloc(std::max(need, size_t(8) << 12), s);
        HF_CUDA(cudaMemsetAsync(ss.buf.p, 0, ss.buf.bytes, s));
        ss.base = 0;
        ss.epoch = 0;
    }
    if (++ss.epoch >= (1u << 29)) {   // tag overflow: start over from a clean state
        HF_CUDA(cudaMemsetAsync(ss.buf.p, 0, ss.buf.bytes, s));
        ss.base = 0;
        ss.epoch = 1;
    }
    unsigned long long *st = ss.buf.as<unsigned long long>();
    unsigned *ctr = reinterpret_cast<unsigned *>(st);   // word 0 is the tile counter
    k_scan_lookback<<<unsigned(tiles), LB_BLOCK, 0, s>>>(in, out, count, st + 1, ctr,
                                                         unsigned(ss.base), ss.epoch,
                                                         total_d);
    HF_CHECK_LAUNCH();
    ss.base += uint64_t(tiles);
    g.launches += 1;
}

void radix_sort_pairs(const int32_t *keys_in, const int32_t *vals_in, int32_t *keys_out,
                      int32_t *vals_out, int64_t count, int key_bits, cudaStream_t s,
                      Graph &g) {
    if (count <= 0) return;
    int passes = (key_bits + 7) / 8;
    if (passes == 0) passes = 1;   // still produce the (identity) permutation
    int nblocks = int((count + RS_TILE - 1) / RS_TILE);
    DevBuf hist, kt, vt;
    hist.alloc(sizeof(int32_t) * 256 * int64_t(nblocks), s);
    if (passes > 1) {
        kt.alloc(sizeof(int32_t) * count, s);
        vt.alloc(sizeof(int32_t) * count, s);
    }
    // ping-pong so that the last pass lands in keys_out / vals_out
    const int32_t *ksrc = keys_in;
    const int32_t *vsrc = vals_in;
    for (int p = 0; p < passes; ++p) {
        // pass p writes to out if (passes-1-p) is even, else to tmp
        bool to_out = ((passes - 1 - p) % 2) == 0;
        int32_t *kdst = to_out ? keys_out : kt.as<int32_t>();
        int32_t *vdst = to_out ? vals_out : vt.as<int32_t>();
        int shift = 8 * p;
        k_radix_upsweep<<<nblocks, RS_BLOCK, 0, s>>>(ksrc, count, shift, hist.as<int32_t>(),
                                                     nblocks);
        HF_CHECK_LAUNCH();
        scan_exclusive(hist.as<int32_t>(), hist.as<int32_t>(), 256 * int64_t(nblocks),
                       nullptr, s, g);
        k_radix_downsweep<<<nblocks, RS_BLOCK, 0, s>>>(ksrc, vsrc, kdst, vdst, count, shift,
                                                       hist.as<int32_t>(), nblocks);
        HF_CHECK_LAUNCH();
        g.launches += 2;
        ksrc = kdst;
        vsrc = vdst;
    }
}

void keys_to_ptr(const int32_t *sorted_keys, int64_t count, int32_t nkeys, int32_t *ptr,
                 cudaStream_t s, Graph &g) {
    HF_CUDA(cudaMemsetAsync(ptr, 0, sizeof(int32_t) * (int64_t(nkeys) + 1), s));
    if (count > 0) {
        k_run_bounds<<<grid_for(count, 256, g.sms), 256, 0, s>>>(sorted_keys, count, ptr);
        HF_CHECK_LAUNCH();
        g.launches += 1;
    }
    scan_exclusive(ptr, ptr, int64_t(nkeys) + 1, nullptr, s, g);
}

void csr_row_ids(const int32_t *ptr, int32_t nrows, int32_t *row_of, cudaStream_t s,
                 Graph &g) {
    if (nrows <= 0) return;
    k_row_ids<<<grid_for(nrows, 256, g.sms), 256, 0, s>>>(ptr, nrows, row_of);
    HF_CHECK_LAUNCH();
    g.launches += 1;
}

}  // namespace hf
