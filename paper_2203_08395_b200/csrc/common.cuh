// common.cuh -- shared internals of libhf.so (graph object, error plumbing,
// device helpers).  Nothing here is shared with oracle/.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/hf.h"

namespace hf {

// ---- error plumbing -------------------------------------------------------
void set_error(const std::string &msg);
const char *last_error();

struct Fail {
    hf_status st;
};

#define HF_CUDA(call)                                                                   \
    do {                                                                                \
        cudaError_t e_ = (call);                                                        \
        if (e_ != cudaSuccess) {                                                        \
            ::hf::set_error(std::string(#call) + ": " + cudaGetErrorString(e_));        \
            throw ::hf::Fail{e_ == cudaErrorMemoryAllocation ? HF_ERR_OOM : HF_ERR_CUDA}; \
        }                                                                               \
    } while (0)

#define HF_CHECK_LAUNCH() HF_CUDA(cudaGetLastError())

[[noreturn]] inline void fail(hf_status st, const std::string &msg) {
    set_error(msg);
    throw Fail{st};
}

// ---- device-side error bits (latched in hf_graph::d_err) ------------------
enum : uint32_t {
    ERR_PTR = 1u,        // fan-in ptr malformed
    ERR_SRC = 2u,        // src out of range
    ERR_NONFINITE = 4u,  // NaN / inf value
    ERR_FO_PTR = 8u,     // fan-out ptr malformed / mismatch
    ERR_FO_DST = 16u,    // fan-out dst out of range / not a transpose
    ERR_WATCHDOG = 32u,  // a dataflow pass waited past its deadline (must never happen)
};

// ---- stream-ordered scratch memory ----------------------------------------
struct DevBuf {
    void *p = nullptr;
    size_t bytes = 0;
    cudaStream_t s = nullptr;
    DevBuf() = default;
    DevBuf(const DevBuf &) = delete;
    DevBuf &operator=(const DevBuf &) = delete;
    ~DevBuf() { release(); }
    void alloc(size_t b, cudaStream_t st) {
        release();
        s = st;
        bytes = b;
        if (b) HF_CUDA(cudaMallocAsync(&p, b, st));
    }
    void release() {
        if (p) cudaFreeAsync(p, s);
        p = nullptr;
        bytes = 0;
    }
    template <class T> T *as() const { return static_cast<T *>(p); }
};

// ---- task schedule of one propagation direction (propagate.cu) -------------
// A pass is a list of warp tasks in pass order (levels ascending forward,
// descending backward; scenario chunks inside a level).  Descriptors are stored
// once per level; chunk c of level q reuses them.
struct TaskSched {
    DevBuf desc;        // int4: normal {row_begin, row_end, edge_begin, edge_end};
                        //       part   {row, -(part id + 1), edge_begin, edge_end}
    DevBuf nt;          // [L] tasks per chunk of pass-level q
    DevBuf doff;        // [L+1] first descriptor of pass-level q
    DevBuf tb;          // [L+1] first global task of pass-level q (for tb_nch chunks)
    int32_t tb_nch = -1;
    int64_t key = -1;   // tw the schedule was built for
};

// rows with more than LO_SPLIT edges sit at the end of their level in the
// level-ordered CSRs and are cut into part tasks by the propagation passes
#ifndef LO_SPLIT_OVR
#define LO_SPLIT_OVR 8
#endif
constexpr int LO_SPLIT = LO_SPLIT_OVR;
// a long row is cut into parts of LO_PE edges (part ids: exclusive scan over the
// level-ordered rows of ceil(degree / LO_PE) for long rows, 0 otherwise)
#ifndef LO_PE_OVR
#define LO_PE_OVR 20
#endif
constexpr int LO_PE = LO_PE_OVR;
// the level-synchronous passes cut a long row into slices of WIDE_SL edges (one
// thread each, all loads of a slice in flight at once)
constexpr int WIDE_SL = 8;
// padding (elements) after the level-ordered arrays (bulk-copy overrun, wide.cu)
constexpr int LO_PAD = 4;

// ---- the graph -------------------------------------------------------------
struct Graph {
    int device = 0;
    cudaStream_t stream = nullptr;
    int32_t n = 0, m = 0;
    int sms = 148;
    // CSR fan-in (edge id = fan-in position), fan-out, per-edge data
    DevBuf in_ptr, in_src, in_dst, delay;
    DevBuf out_ptr, out_dst, out_eid;
    // analysis mode (NEXT-2, reading R18): false = late (setup: max-plus forward,
    // min-plus backward, slack rat - at); true = early (hold: min-plus forward,
    // max-plus backward, slack at - rat)
    bool early = false;
    // levelization
    bool levelized = false;
    int32_t L = -1;
    DevBuf level, level_ptr, order;
    // level-ordered ("relabelled") CSR for the propagation passes: row i is node
    // order[i]; eid = original edge id (delay row).  Built by hf_levelize.
    // Within a level, rows of degree <= LO_SPLIT first, then the longer ones, each
    // run in canonical order (per direction): node ids lo_in_node / lo_out_node.
    DevBuf lo_in_node, lo_in_ptr, lo_in_nbr, lo_in_eid, lo_in_q, lo_in_np;
    DevBuf lo_out_node, lo_out_ptr, lo_out_nbr, lo_out_eid, lo_out_q, lo_out_np;
    // [L] first long row of every level (= level end when the level has none)
    DevBuf lo_in_lstart, lo_out_lstart;
    // lo_*_nbr: neighbour node id, or -(first part id + 1) when the neighbour's own
    // row (same direction) is long; lo_*_q: [n+1] first part id of every row;
    // lo_*_np: parts of the long row whose first part id is the index, then that row
    // part ids per direction: at most np_cap (host bound); the exact counts live on
    // the device (nparts_d[0] fan-in, nparts_d[1] fan-out).  lo_*_np holds [np_cap]
    // part counts (0 except at first part ids) then [np_cap] rows
    int32_t np_cap_in = 0, np_cap_out = 0;
    const int32_t *nparts_d = nullptr;
    // task schedules of the dataflow propagation kernels (per direction)
    TaskSched ts_f, ts_b;
    // level-synchronous ("wide") passes (wide.cu), built on first use after each
    // hf_levelize: per direction the long rows cut into slices of WIDE_SL edges --
    // wide_*_sfirst[n+1] first slice of every level-ordered row (0 slices for short
    // rows), wide_*_slice[] {row, first edge} -- and the graph's own delays
    // permuted into level order per direction (lo_*_d[m], single-delay-set calls)
    DevBuf wide_in_sfirst, wide_in_slice, wide_out_sfirst, wide_out_slice;
    // S = 1 (k_wide1): the long rows of a level as one edge range cut into chunks of
    // 32 edges; wide_*_coff[L+1] first chunk of each level, wide_*_crow[] the row
    // holding each chunk's first edge
    DevBuf wide_in_coff, wide_in_crow, wide_out_coff, wide_out_crow;
    DevBuf lo_in_d, lo_out_d;
    bool wide_ready = false, lo_d_ready = false;
    // S = 1 (k_wide2): per direction w2_*_nbr[m] int2 {plain neighbour id, row} of every
    // level-ordered edge, w2_*_erow[n] the node of every row (~node: no edges), and each
    // level cut into row ranges of weight (rows + edges) <= W2_TW: w2_*_roff[L+1] first
    // range-table entry of each level (a level of r ranges owns r + 1 entries),
    // w2_*_rstart[] first row of each range + the level end
    DevBuf w2_in_nbr, w2_in_erow, w2_in_roff, w2_in_rstart;
    DevBuf w2_out_nbr, w2_out_erow, w2_out_roff, w2_out_rstart;
    bool w2_ready = false;
    // dataflow passes (HF_LASTPART): plain neighbour ids of the level-ordered CSRs (a long
    // neighbour's -(first part id + 1) decoded to its node)
    DevBuf lo_in_pnbr, lo_out_pnbr;
    bool pnbr_ready = false;
    // S = 1 (k_wide3): {plain neighbour, destination node} per level-ordered edge
    DevBuf w3_in_edge, w3_out_edge;
    bool w3_ready = false;
    // batch workspace (at / rat when the caller does not want them), grows on demand
    DevBuf ws_at, ws_rat, ws_sync, ws_wns;
    // single-pass scan state (primitives.cu): per-tile words + tile counter; one per
    // stream that scans concurrently (slot 0: the graph's stream, 1: the side stream)
    struct ScanState {
        DevBuf buf;
        uint64_t base = 0;
        unsigned epoch = 0;
    } scan[2];
    // small device scalars: [0] error bits, [1..] scratch
    DevBuf d_small;
    uint32_t *d_err() const { return d_small.as<uint32_t>(); }
    int32_t *d_scalars() const { return d_small.as<int32_t>() + 8; }   // 56 int32 scratch
    // profiling
    bool prof = false;
    cudaEvent_t ev[8] = {};   // 0/1 levelize, 2/3 forward, 5/4 backward, 6/7 batch phase
    float ms_lev = 0, ms_fwd = 0, ms_bwd = 0, ms_prop = 0;
    bool lev_timed = false, prop_timed = false;
    int64_t launches = 0;
};

// second stream + fork/join events, one set per host thread and device, created
// once and kept for the process (propagate.cu)
struct Side {
    cudaStream_t s2 = nullptr;
    cudaEvent_t fork = nullptr, join = nullptr;
};
Side &side_of(Graph &g);

// Per-stage device times on stderr when the environment variable `env` is set
// (tools only: HF_LEV_TIMES in levelize, HF_PROP_TIMES in the batch).
struct StageTimes {
    const char *title;
    bool on;
    std::vector<std::pair<const char *, cudaEvent_t>> ev;
    StageTimes(const char *env, const char *t) : title(t), on(getenv(env) != nullptr) {}
    void mark(const char *name, cudaStream_t s) {
        if (!on) return;
        cudaEvent_t e;
        if (cudaEventCreate(&e) != cudaSuccess) return;
        cudaEventRecord(e, s);
        ev.emplace_back(name, e);
    }
    ~StageTimes() {
        if (!on || ev.empty()) return;
        cudaEventSynchronize(ev.back().second);
        std::string line = std::string(title) + " stages (us):";
        for (size_t i = 1; i < ev.size(); ++i) {
            float ms = 0;
            cudaEventElapsedTime(&ms, ev[i - 1].second, ev[i].second);
            line += std::string(" ") + ev[i].first + "=" + std::to_string(int(ms * 1000));
        }
        fprintf(stderr, "%s\n", line.c_str());
        for (auto &x : ev) cudaEventDestroy(x.second);
    }
};

// ---- primitives (primitives.cu) --------------------------------------------
// exclusive scan of int32 (out may alias in); writes the total to *total_d if non-null
void scan_exclusive(const int32_t *in, int32_t *out, int64_t count, int32_t *total_d,
                    cudaStream_t s, Graph &g, int slot = 0);
// stable LSD radix sort of (key, value) pairs, keys in [0, 2^key_bits); vals_in
// NULL => values are 0..count-1.  Results in keys_out / vals_out.
void radix_sort_pairs(const int32_t *keys_in, const int32_t *vals_in, int32_t *keys_out,
                      int32_t *vals_out, int64_t count, int key_bits, cudaStream_t s,
                      Graph &g);
// ptr[k] = first index i with sorted_keys[i] >= k, for k in [0, nkeys]; ptr[nkeys] = count
void keys_to_ptr(const int32_t *sorted_keys, int64_t count, int32_t nkeys, int32_t *ptr,
                 cudaStream_t s, Graph &g);
// row id of every CSR position: dst[e] = v for e in [ptr[v], ptr[v+1])
void csr_row_ids(const int32_t *ptr, int32_t nrows, int32_t *row_of, cudaStream_t s,
                 Graph &g);

inline int bits_for(int64_t max_key) {
    int b = 0;
    while (b < 31 && (int64_t(1) << b) <= max_key) ++b;
    return b;
}
// The dynamic shared-memory limit of a kernel is one attribute per (function,
// device): raise it to the largest size ever requested and never lower it, so that
// launches of one kernel with different scratch sizes (e.g. batches of S = 128, then
// 64, then 128 again) all stay within it.  Thread-safe; one driver call per new max.
inline void ensure_dyn_smem(const void *func, int device, size_t bytes) {
    static std::map<std::pair<const void *, int>, size_t> mx;
    static std::mutex mu;
    std::lock_guard<std::mutex> lk(mu);
    size_t &cur = mx[{func, device}];
    if (bytes <= cur) return;
    HF_CUDA(cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes)));
    cur = bytes;
}

inline int grid_for(int64_t work, int block, int sms, int per_sm = 8) {
    int64_t gsz = (work + block - 1) / block;
    int64_t cap = int64_t(sms) * per_sm;
    if (gsz > cap) gsz = cap;
    if (gsz < 1) gsz = 1;
    return int(gsz);
}

// ---- device helpers --------------------------------------------------------
// block-aggregated append of `item` when `pred`: one global atomic per block and
// call instead of one per warp (all threads of the block must call; s_w[33] shared)
__device__ __forceinline__ void block_append(bool pred, int item, int *list, int *count, int *s_w) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const unsigned mask = __ballot_sync(0xffffffffu, pred);
    if (lane == 0) s_w[wid] = __popc(mask);
    __syncthreads();
    if (threadIdx.x == 0) {
        int tot = 0;
        for (int w = 0; w < nw; ++w) {
            const int c = s_w[w];
            s_w[w] = tot;
            tot += c;
        }
        s_w[32] = tot ? atomicAdd(count, tot) : 0;
    }
    __syncthreads();
    if (pred) list[s_w[32] + s_w[wid] + __popc(mask & ((1u << lane) - 1u))] = item;
    __syncthreads();   // s_w is reused by the next call
}

// float <-> order-preserving int32 (reading R9): signed compare of the keys
// orders all non-NaN floats; the map is an involution.
__device__ __forceinline__ int32_t f2ord(float f) {
    int32_t b = __float_as_int(f);
    return b ^ ((b >> 31) & 0x7FFFFFFF);
}
__device__ __forceinline__ float ord2f(int32_t k) {
    return __int_as_float(k ^ ((k >> 31) & 0x7FFFFFFF));
}
__device__ __forceinline__ float canon0(float x) { return __fadd_rn(x, 0.0f); }  // -0 -> +0
// An input value (delay, source arrival, required time) as the propagation kernels
// use it: -0 -> +0; NaN / +-inf (rejected, reading R9) set `bad` (latched as
// HF_ERR_INVALID_ARG) and are replaced by +0, so no output row can become NaN -- the
// "not yet computed" sentinel of the dataflow kernels -- and every pass terminates.
__device__ __forceinline__ float sane(float x, bool &bad) {
    const bool ok = fabsf(x) <= 3.40282346638528859812e+38f;   // false for NaN and +-inf
    bad |= !ok;
    return ok ? canon0(x) : 0.0f;
}}  // namespace hf
