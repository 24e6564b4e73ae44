// graph.cu -- hf_graph_create: validate CSR fan-in, canonicalise delays, derive
// (or verify) the fan-out CSR and out_eid on the device.  SURVEY.md §8(a) a1.
#include <algorithm>

#include "common.cuh"

namespace hf {

namespace {

// One pass over max(n, m): fan-in ptr monotone, src range, delay finiteness;
// copies delays with -0 -> +0.
__global__ void k_validate_fanin(const int32_t *__restrict__ ptr,
                                 const int32_t *__restrict__ src,
                                 const float *__restrict__ delay_in,
                                 float *__restrict__ delay_out, int32_t n, int32_t m,
                                 uint32_t *err) {
    uint32_t bits = 0;
    int64_t total = n > m ? n : m;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total;
         i += int64_t(gridDim.x) * blockDim.x) {
        if (i < n && ptr[i + 1] < ptr[i]) bits |= ERR_PTR;
        if (i < m) {
            int s = src[i];
            if (s < 0 || s >= n) bits |= ERR_SRC;
            float d = delay_in ? delay_in[i] : 0.0f;
            if (!isfinite(d)) bits |= ERR_NONFINITE;
            delay_out[i] = canon0(d);
        }
    }
    if (bits) atomicOr(err, bits);
}

__global__ void k_check_ends(const int32_t *__restrict__ ptr, int32_t n, int32_t m,
                             uint32_t *err, uint32_t bit) {
    if (ptr[0] != 0 || ptr[n] != m) atomicOr(err, bit);
}

__global__ void k_check_fanout(const int32_t *__restrict__ ptr, const int32_t *__restrict__ dst,
                               int32_t n, int32_t m, uint32_t *err) {
    uint32_t bits = 0;
    int64_t total = n > m ? n : m;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total;
         i += int64_t(gridDim.x) * blockDim.x) {
        if (i < n && ptr[i + 1] < ptr[i]) bits |= ERR_FO_PTR;
        if (i < m && (dst[i] < 0 || dst[i] >= n)) bits |= ERR_FO_DST;
    }
    if (bits) atomicOr(err, bits);
}

// count pass of the fan-out counting sort: every edge takes its slot in its
// source's row (the atomic's old value), so the scatter needs no second atomic
__global__ void k_count_slots(const int32_t *__restrict__ keys, int64_t count,
                              int32_t *__restrict__ cnt, int32_t *__restrict__ slot) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < count;
         i += int64_t(gridDim.x) * blockDim.x)
        slot[i] = atomicAdd(cnt + keys[i], 1);
}

__global__ void k_scatter_fanout(const int32_t *__restrict__ src, const int32_t *__restrict__ dst,
                                 int64_t m, const int32_t *__restrict__ out_ptr,
                                 const int32_t *__restrict__ slot, int32_t *__restrict__ out_dst,
                                 int32_t *__restrict__ out_eid) {
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < m;
         e += int64_t(gridDim.x) * blockDim.x) {
        const int k = out_ptr[src[e]] + slot[e];
        out_dst[k] = dst[e];
        out_eid[k] = int(e);
    }
}

__global__ void k_compare(const int32_t *__restrict__ a, const int32_t *__restrict__ b,
                          int64_t count, uint32_t *err, uint32_t bit) {
    bool bad = false;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < count;
         i += int64_t(gridDim.x) * blockDim.x)
        bad |= a[i] != b[i];
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(err, bit);
}

uint32_t read_err(Graph &g) {
    uint32_t e = 0;
    HF_CUDA(cudaMemcpyAsync(&e, g.d_err(), sizeof(e), cudaMemcpyDeviceToHost, g.stream));
    HF_CUDA(cudaStreamSynchronize(g.stream));
    return e;
}

}  // namespace

// Build the graph from DEVICE pointers (the host variant uploads first).
void graph_build(Graph &g, const int32_t *in_ptr, const int32_t *in_src,
                 const int32_t *fo_ptr, const int32_t *fo_dst, const float *delay) {
    cudaStream_t s = g.stream;
    const int32_t n = g.n, m = g.m;
    // keep freed device memory in the stream-ordered pool across synchronisations
    // (the default release threshold 0 hands it back to the driver at every sync,
    // and the next graph then pays for fresh mappings)
    {
        static bool done[64] = {};   // once per device
        if (g.device >= 0 && g.device < 64 && !done[g.device]) {
            cudaMemPool_t pool;
            HF_CUDA(cudaDeviceGetDefaultMemPool(&pool, g.device));
            uint64_t keep = UINT64_MAX;
            HF_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
            // map a working set into the pool once (1/8 of the device memory, at most
            // 24 GiB): later graphs carve their buffers from it instead of growing the
            // pool (a growth maps new memory: milliseconds on the host, mid-step)
            size_t free_b = 0, total_b = 0;
            HF_CUDA(cudaMemGetInfo(&free_b, &total_b));
            const size_t want = std::min<size_t>(total_b / 8, size_t(24) << 30);
            if (want < free_b / 2) {
                void *blk = nullptr;
                if (cudaMallocAsync(&blk, want, s) == cudaSuccess) {
                    cudaFreeAsync(blk, s);
                    HF_CUDA(cudaStreamSynchronize(s));
                }
                cudaGetLastError();
            }
            done[g.device] = true;
        }
    }
    g.d_small.alloc(64 * sizeof(int32_t), s);
    HF_CUDA(cudaMemsetAsync(g.d_small.p, 0, 64 * sizeof(int32_t), s));
    g.in_ptr.alloc(sizeof(int32_t) * (int64_t(n) + 1), s);
    g.in_src.alloc(sizeof(int32_t) * int64_t(m), s);
    g.in_dst.alloc(sizeof(int32_t) * int64_t(m), s);
    g.delay.alloc(sizeof(float) * int64_t(m), s);
    g.out_ptr.alloc(sizeof(int32_t) * (int64_t(n) + 1), s);
    g.out_dst.alloc(sizeof(int32_t) * int64_t(m), s);
    g.out_eid.alloc(sizeof(int32_t) * int64_t(m), s);
    HF_CUDA(cudaMemcpyAsync(g.in_ptr.p, in_ptr, sizeof(int32_t) * (int64_t(n) + 1),
                            cudaMemcpyDeviceToDevice, s));
    if (m)
        HF_CUDA(cudaMemcpyAsync(g.in_src.p, in_src, sizeof(int32_t) * int64_t(m),
                                cudaMemcpyDeviceToDevice, s));
    const int64_t total = n > m ? n : m;
    k_check_ends<<<1, 1, 0, s>>>(g.in_ptr.as<int32_t>(), n, m, g.d_err(), ERR_PTR);
    HF_CHECK_LAUNCH();
    k_validate_fanin<<<grid_for(total, 256, g.sms), 256, 0, s>>>(
        g.in_ptr.as<int32_t>(), g.in_src.as<int32_t>(), delay, g.delay.as<float>(), n, m,
        g.d_err());
    HF_CHECK_LAUNCH();
    g.launches += 2;
    uint32_t e = read_err(g);
    if (e & (ERR_PTR | ERR_SRC))
        fail(HF_ERR_BAD_CSR, (e & ERR_PTR) ? "fan-in ptr is not a valid CSR offset array"
                                           : "fan-in src out of range [0, n)");
    if (e & ERR_NONFINITE) fail(HF_ERR_INVALID_ARG, "delay contains NaN or inf");

    // fan-out: counting sort of the fan-in edges by source (atomic cursors; the
    // order inside a fan-out row is irrelevant: min is exact and commutative)
    csr_row_ids(g.in_ptr.as<int32_t>(), n, g.in_dst.as<int32_t>(), s, g);
    {
        DevBuf cur, slot;
        cur.alloc(sizeof(int32_t) * (int64_t(n) + 1), s);
        slot.alloc(sizeof(int32_t) * int64_t(m > 0 ? m : 1), s);
        HF_CUDA(cudaMemsetAsync(cur.p, 0, sizeof(int32_t) * (int64_t(n) + 1), s));
        if (m) {
            k_count_slots<<<grid_for(m, 256, g.sms), 256, 0, s>>>(g.in_src.as<int32_t>(), m,
                                                                cur.as<int32_t>(),
                                                                slot.as<int32_t>());
            HF_CHECK_LAUNCH();
            g.launches += 1;
        }
        scan_exclusive(cur.as<int32_t>(), g.out_ptr.as<int32_t>(), int64_t(n) + 1, nullptr, s, g);
        if (m) {
            k_scatter_fanout<<<grid_for(m, 256, g.sms), 256, 0, s>>>(
                g.in_src.as<int32_t>(), g.in_dst.as<int32_t>(), m, g.out_ptr.as<int32_t>(),
                slot.as<int32_t>(), g.out_dst.as<int32_t>(), g.out_eid.as<int32_t>());
            HF_CHECK_LAUNCH();
            g.launches += 1;
        }
    }
    if (fo_ptr || fo_dst) {
        if (!fo_ptr || !fo_dst)
            fail(HF_ERR_INVALID_ARG, "fanout_ptr and fanout_dst must both be given or both NULL");
        // caller's fan-out, canonicalised by (src, dst): sort by dst then (stably) by src
        DevBuf cptr, cdst, csrc, k1, v1, k2, v2;
        cptr.alloc(sizeof(int32_t) * (int64_t(n) + 1), s);
        cdst.alloc(sizeof(int32_t) * int64_t(m), s);
        csrc.alloc(sizeof(int32_t) * int64_t(m), s);
        HF_CUDA(cudaMemcpyAsync(cptr.p, fo_ptr, sizeof(int32_t) * (int64_t(n) + 1),
                                cudaMemcpyDeviceToDevice, s));
        if (m)
            HF_CUDA(cudaMemcpyAsync(cdst.p, fo_dst, sizeof(int32_t) * int64_t(m),
                                    cudaMemcpyDeviceToDevice, s));
        k_check_ends<<<1, 1, 0, s>>>(cptr.as<int32_t>(), n, m, g.d_err(), ERR_FO_PTR);
        HF_CHECK_LAUNCH();
        k_check_fanout<<<grid_for(total, 256, g.sms), 256, 0, s>>>(
            cptr.as<int32_t>(), cdst.as<int32_t>(), n, m, g.d_err());
        HF_CHECK_LAUNCH();
        g.launches += 2;
        e = read_err(g);
        if (e) fail(HF_ERR_BAD_CSR, "fan-out CSR malformed");
        k1.alloc(sizeof(int32_t) * int64_t(m), s);
        v1.alloc(sizeof(int32_t) * int64_t(m), s);
        k2.alloc(sizeof(int32_t) * int64_t(m), s);
        v2.alloc(sizeof(int32_t) * int64_t(m), s);
        csr_row_ids(cptr.as<int32_t>(), n, csrc.as<int32_t>(), s, g);
        int kb = bits_for(int64_t(n) - 1);
        radix_sort_pairs(cdst.as<int32_t>(), csrc.as<int32_t>(), k1.as<int32_t>(),
                         v1.as<int32_t>(), m, kb, s, g);   // by dst: (dst, src asc)
        radix_sort_pairs(v1.as<int32_t>(), k1.as<int32_t>(), k2.as<int32_t>(),
                         v2.as<int32_t>(), m, kb, s, g);   // by src: (src, dst asc)
        // canonical transpose of the fan-in: stable sort of edges (ascending id, so
        // ascending sink) by source -> rows ascending in dst
        DevBuf k3, v3, d3;
        k3.alloc(sizeof(int32_t) * int64_t(m), s);
        v3.alloc(sizeof(int32_t) * int64_t(m), s);
        d3.alloc(sizeof(int32_t) * int64_t(m), s);
        radix_sort_pairs(g.in_src.as<int32_t>(), g.in_dst.as<int32_t>(), k3.as<int32_t>(),
                         d3.as<int32_t>(), m, kb, s, g);
        int64_t cmp_n = int64_t(n) + 1;
        k_compare<<<grid_for(cmp_n, 256, g.sms), 256, 0, s>>>(
            cptr.as<int32_t>(), g.out_ptr.as<int32_t>(), cmp_n, g.d_err(), ERR_FO_PTR);
        HF_CHECK_LAUNCH();
        if (m) {
            k_compare<<<grid_for(m, 256, g.sms), 256, 0, s>>>(
                v2.as<int32_t>(), d3.as<int32_t>(), m, g.d_err(), ERR_FO_DST);
            HF_CHECK_LAUNCH();
        }
        g.launches += 2;
        e = read_err(g);
        if (e) fail(HF_ERR_BAD_CSR, "fan-out is not the transpose of the fan-in");
    }
    // no trailing synchronisation: the fan-out build is stream-ordered before every
    // later call, and the validation read above already completed the uploads
}

}  // namespace hf
