// primitives.cu -- device building blocks for graph ingest and levelization:
// 3-phase exclusive scan, stable LSD radix sort (8-bit digits, warp-match
// ranking), sorted-keys -> CSR offsets, CSR row ids.  All hand-written sm_100a.
#include "common.cuh"

namespace hf {

namespace {

constexpr int SCAN_BLOCK = 256;
constexpr int SCAN_ITEMS = 8;
constexpr int SCAN_TILE = SCAN_BLOCK * SCAN_ITEMS;

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

__global__ void k_scan_tiles(const int32_t *__restrict__ in, int64_t count,
                             int32_t *__restrict__ tile_sums) {
    int64_t base = int64_t(blockIdx.x) * SCAN_TILE + int64_t(threadIdx.x) * SCAN_ITEMS;
    int s = 0;
#pragma unroll
    for (int j = 0; j < SCAN_ITEMS; ++j)
        if (base + j < count) s += in[base + j];
    int tot;
    block_exclusive_sum(s, &tot);
    if (threadIdx.x == 0) tile_sums[blockIdx.x] = tot;
}

// single block: exclusive scan of tile sums in place (any length), total -> *total
__global__ void k_scan_partials(int32_t *__restrict__ p, int64_t count, int32_t *total) {
    int carry = 0;
    for (int64_t base = 0; base < count; base += SCAN_TILE) {
        int64_t i0 = base + int64_t(threadIdx.x) * SCAN_ITEMS;
        int v[SCAN_ITEMS];
        int s = 0;
#pragma unroll
        for (int j = 0; j < SCAN_ITEMS; ++j) {
            v[j] = (i0 + j < count) ? p[i0 + j] : 0;
            s += v[j];
        }
        int tot;
        int pre = block_exclusive_sum(s, &tot) + carry;
#pragma unroll
        for (int j = 0; j < SCAN_ITEMS; ++j) {
            if (i0 + j < count) p[i0 + j] = pre;
            pre += v[j];
        }
        carry += tot;
        __syncthreads();
    }
    if (threadIdx.x == 0 && total) *total = carry;
}

__global__ void k_scan_apply(const int32_t *__restrict__ in, int32_t *__restrict__ out,
                             int64_t count, const int32_t *__restrict__ tile_pre) {
    int64_t base = int64_t(blockIdx.x) * SCAN_TILE + int64_t(threadIdx.x) * SCAN_ITEMS;
    int v[SCAN_ITEMS];
    int s = 0;
#pragma unroll
    for (int j = 0; j < SCAN_ITEMS; ++j) {
        v[j] = (base + j < count) ? in[base + j] : 0;
        s += v[j];
    }
    int pre = block_exclusive_sum(s, nullptr) + tile_pre[blockIdx.x];
#pragma unroll
    for (int j = 0; j < SCAN_ITEMS; ++j) {
        if (base + j < count) out[base + j] = pre;
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
                    cudaStream_t s, Graph &g) {
    if (count <= 0) {
        if (total_d) HF_CUDA(cudaMemsetAsync(total_d, 0, sizeof(int32_t), s));
        return;
    }
    int64_t tiles = (count + SCAN_TILE - 1) / SCAN_TILE;
    DevBuf part;
    part.alloc(sizeof(int32_t) * tiles, s);
    k_scan_tiles<<<unsigned(tiles), SCAN_BLOCK, 0, s>>>(in, count, part.as<int32_t>());
    HF_CHECK_LAUNCH();
    k_scan_partials<<<1, SCAN_BLOCK, 0, s>>>(part.as<int32_t>(), tiles, total_d);
    HF_CHECK_LAUNCH();
    k_scan_apply<<<unsigned(tiles), SCAN_BLOCK, 0, s>>>(in, out, count, part.as<int32_t>());
    HF_CHECK_LAUNCH();
    g.launches += 3;
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
