// abi.cu -- the extern "C" boundary of libhf.so (declared in include/hf.h).
// Argument checking, host<->device marshalling for the host-pointer variants,
// workspace management, NCCL bootstrap (libnccl.so.2 via dlopen), profiling.
#include <dlfcn.h>
#include <stdio.h>

#include <algorithm>
#include <cmath>
#include <string>

#include <nvtx3/nvToolsExt.h>

#include "common.cuh"

namespace hf {

static thread_local std::string t_err;
void set_error(const std::string &msg) { t_err = msg; }
const char *last_error() { return t_err.c_str(); }

void graph_build(Graph &g, const int32_t *in_ptr, const int32_t *in_src, const int32_t *fo_ptr,
                 const int32_t *fo_dst, const float *delay);
int64_t levelize_device(Graph &g);
void forward_device(Graph &g, const float *d, int32_t S, bool check_d, const float *at_src,
                    float *at);
void backward_device(Graph &g, const float *d, int32_t S, const float *t_arr, float t_scalar,
                     const float *at, float *rat, float *slack, float *wns_f);
void batch_device(Graph &g, const float *d, int32_t S, bool check_d, const float *at_src,
                  const float *t_arr, float *at, float *rat, float *slack, float *wns_f);
void profile_mark(Graph &g, int idx);
void mis_device(Graph &g, const int32_t *prio, uint8_t *in_set);
void critical_path_device(Graph &g, int32_t S, const float *d, const float *at,
                          const float *t_arr, float t_scalar, int32_t K, int32_t max_len,
                          int32_t *endpoints, int32_t *path, int32_t *len);

// ---- NCCL through dlopen (no link-time dependency) -------------------------
namespace nccl {
typedef struct {
    char internal[128];
} UniqueId;
typedef void *Comm;
typedef int (*GetUniqueId_t)(UniqueId *);
typedef int (*CommInitRank_t)(Comm *, int, UniqueId, int);
typedef int (*AllGather_t)(const void *, void *, size_t, int, Comm, cudaStream_t);
typedef int (*CommDestroy_t)(Comm);
typedef const char *(*GetErrorString_t)(int);
constexpr int kFloat32 = 7;   // ncclFloat32 (nccl.h)
struct Api {
    void *h = nullptr;
    GetUniqueId_t get_unique_id = nullptr;
    CommInitRank_t comm_init_rank = nullptr;
    AllGather_t all_gather = nullptr;
    CommDestroy_t comm_destroy = nullptr;
    GetErrorString_t err_str = nullptr;
};
static Api api;
static void load() {
    if (api.h) return;
    const char *env = getenv("HF_NCCL_LIBRARY");
    const char *names[] = {env, "libnccl.so.2", "libnccl.so"};
    for (const char *nm : names) {
        if (!nm) continue;
        api.h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
        if (!api.h) api.h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
        if (api.h) break;
    }
    if (!api.h)
        fail(HF_ERR_NCCL, "cannot load libnccl.so.2 (import torch first, or set HF_NCCL_LIBRARY)");
    api.get_unique_id = (GetUniqueId_t)dlsym(api.h, "ncclGetUniqueId");
    api.comm_init_rank = (CommInitRank_t)dlsym(api.h, "ncclCommInitRank");
    api.all_gather = (AllGather_t)dlsym(api.h, "ncclAllGather");
    api.comm_destroy = (CommDestroy_t)dlsym(api.h, "ncclCommDestroy");
    api.err_str = (GetErrorString_t)dlsym(api.h, "ncclGetErrorString");
    if (!api.get_unique_id || !api.comm_init_rank || !api.all_gather || !api.comm_destroy) {
        api.h = nullptr;
        fail(HF_ERR_NCCL, "libnccl is missing required symbols");
    }
}
static void check(int r, const char *what) {
    if (r != 0)
        fail(HF_ERR_NCCL, std::string(what) + ": " + (api.err_str ? api.err_str(r) : "error"));
}
}  // namespace nccl

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) HF_CUDA(cudaSetDevice(dev));
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

static void init_pool(int device) {
    static bool done[64] = {};
    if (device < 64 && done[device]) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
        uint64_t thr = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    if (device < 64) done[device] = true;
}

static hf_status latch(Graph &g) {
    uint32_t e = 0;
    HF_CUDA(cudaMemcpyAsync(&e, g.d_err(), sizeof(e), cudaMemcpyDeviceToHost, g.stream));
    HF_CUDA(cudaStreamSynchronize(g.stream));
    if (e) {
        HF_CUDA(cudaMemsetAsync(g.d_err(), 0, sizeof(uint32_t), g.stream));
        HF_CUDA(cudaStreamSynchronize(g.stream));
        if (e & ERR_WATCHDOG) {
            set_error("internal: a propagation pass waited past its watchdog deadline (results void)");
            return HF_ERR_CUDA;
        }
        set_error("device-side validation: NaN or inf in delays, source arrival times or required "
                  "times");
        return HF_ERR_INVALID_ARG;
    }
    return HF_OK;
}

// Every hf_* entry point is one NVTX range named after the call (SURVEY.md §5
// tracing; nvtx3 is header-only: without an attached tool a push / pop is one
// indirect call that returns at once), and a status instead of an exception.
struct NvtxRange {
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};

template <class F> static hf_status guarded_named(const char *name, F &&f) {
    NvtxRange r(name);
    try {
        return f();
    } catch (const Fail &x) {
        return x.st;
    } catch (const std::bad_alloc &) {
        set_error("host out of memory");
        return HF_ERR_OOM;
    } catch (...) {
        set_error("unexpected internal error");
        return HF_ERR_CUDA;
    }
}

#define guarded(...) guarded_named(__func__, __VA_ARGS__)

static Graph *G(hf_graph g) { return reinterpret_cast<Graph *>(g); }

static hf_status create_impl(bool device_ptrs, int32_t n, int32_t m, const int32_t *fanin_ptr,
                             const int32_t *fanin_src, const int32_t *fanout_ptr,
                             const int32_t *fanout_dst, const float *delay, int device,
                             void *stream, hf_graph *out) {
    return guarded([&]() -> hf_status {
        if (!out) fail(HF_ERR_INVALID_ARG, "out is NULL");
        *out = nullptr;
        if (n < 0 || m < 0) fail(HF_ERR_INVALID_ARG, "negative n or m");
        if (!fanin_ptr || (m > 0 && !fanin_src))
            fail(HF_ERR_INVALID_ARG, "fanin_ptr / fanin_src is NULL");
        int ndev = 0;
        HF_CUDA(cudaGetDeviceCount(&ndev));
        if (device < 0 || device >= ndev) fail(HF_ERR_INVALID_ARG, "bad device ordinal");
        DeviceGuard dg(device);
        init_pool(device);
        Graph *g = new Graph();
        g->device = device;
        g->stream = static_cast<cudaStream_t>(stream);
        g->n = n;
        g->m = m;
        HF_CUDA(cudaDeviceGetAttribute(&g->sms, cudaDevAttrMultiProcessorCount, device));
        try {
            if (device_ptrs) {
                graph_build(*g, fanin_ptr, fanin_src, fanout_ptr, fanout_dst, delay);
            } else {
                cudaStream_t s = g->stream;
                DevBuf ip, is, fp, fd, dl;
                ip.alloc(sizeof(int32_t) * (int64_t(n) + 1), s);
                is.alloc(sizeof(int32_t) * int64_t(m), s);
                HF_CUDA(cudaMemcpyAsync(ip.p, fanin_ptr, sizeof(int32_t) * (int64_t(n) + 1),
                                        cudaMemcpyHostToDevice, s));
                if (m)
                    HF_CUDA(cudaMemcpyAsync(is.p, fanin_src, sizeof(int32_t) * int64_t(m),
                                            cudaMemcpyHostToDevice, s));
                if (fanout_ptr) {
                    fp.alloc(sizeof(int32_t) * (int64_t(n) + 1), s);
                    HF_CUDA(cudaMemcpyAsync(fp.p, fanout_ptr, sizeof(int32_t) * (int64_t(n) + 1),
                                            cudaMemcpyHostToDevice, s));
                }
                if (fanout_dst) {
                    fd.alloc(sizeof(int32_t) * int64_t(m > 0 ? m : 1), s);
                    if (m)
                        HF_CUDA(cudaMemcpyAsync(fd.p, fanout_dst, sizeof(int32_t) * int64_t(m),
                                                cudaMemcpyHostToDevice, s));
                }
                if (delay) {
                    dl.alloc(sizeof(float) * int64_t(m), s);
                    if (m)
                        HF_CUDA(cudaMemcpyAsync(dl.p, delay, sizeof(float) * int64_t(m),
                                                cudaMemcpyHostToDevice, s));
                }
                graph_build(*g, ip.as<int32_t>(), is.as<int32_t>(), fp.as<int32_t>(),
                            fd.as<int32_t>(), dl.as<float>());
            }
        } catch (...) {
            cudaStreamSynchronize(g->stream);
            delete g;
            throw;
        }
        *out = reinterpret_cast<hf_graph>(g);
        return HF_OK;
    });
}

}  // namespace hf

using namespace hf;

extern "C" {

const char *hf_last_error(void) { return hf::last_error(); }

const char *hf_status_string(hf_status s) {
    switch (s) {
    case HF_OK: return "HF_OK";
    case HF_ERR_INVALID_ARG: return "HF_ERR_INVALID_ARG";
    case HF_ERR_BAD_CSR: return "HF_ERR_BAD_CSR";
    case HF_ERR_CYCLE: return "HF_ERR_CYCLE";
    case HF_ERR_NOT_LEVELIZED: return "HF_ERR_NOT_LEVELIZED";
    case HF_ERR_OOM: return "HF_ERR_OOM";
    case HF_ERR_CUDA: return "HF_ERR_CUDA";
    case HF_ERR_NCCL: return "HF_ERR_NCCL";
    }
    return "HF_ERR_UNKNOWN";
}

int hf_version(void) { return HF_VERSION; }

hf_status hf_graph_create(int32_t n, int32_t m, const int32_t *fanin_ptr,
                          const int32_t *fanin_src, const int32_t *fanout_ptr,
                          const int32_t *fanout_dst, const float *delay, int device,
                          void *cuda_stream, hf_graph *out) {
    return create_impl(false, n, m, fanin_ptr, fanin_src, fanout_ptr, fanout_dst, delay, device,
                       cuda_stream, out);
}

hf_status hf_graph_create_d(int32_t n, int32_t m, const int32_t *fanin_ptr_d,
                            const int32_t *fanin_src_d, const int32_t *fanout_ptr_d,
                            const int32_t *fanout_dst_d, const float *delay_d, int device,
                            void *cuda_stream, hf_graph *out) {
    return create_impl(true, n, m, fanin_ptr_d, fanin_src_d, fanout_ptr_d, fanout_dst_d, delay_d,
                       device, cuda_stream, out);
}

hf_status hf_graph_destroy(hf_graph h) {
    return guarded([&]() -> hf_status {
        if (!h) return HF_OK;
        Graph *g = G(h);
        DeviceGuard dg(g->device);
        cudaStreamSynchronize(g->stream);
        for (auto &e : g->ev)
            if (e) cudaEventDestroy(e);
        delete g;   // DevBufs free stream-ordered
        return HF_OK;
    });
}

hf_status hf_graph_set_stream(hf_graph h, void *stream) {
    return guarded([&]() -> hf_status {
        if (!h) fail(HF_ERR_INVALID_ARG, "graph is NULL");
        Graph *g = G(h);
        DeviceGuard dg(g->device);
        HF_CUDA(cudaStreamSynchronize(g->stream));
        g->stream = static_cast<cudaStream_t>(stream);
        return HF_OK;
    });
}

hf_status hf_graph_set_mode(hf_graph h, int mode) {
    return guarded([&]() -> hf_status {
        if (!h) fail(HF_ERR_INVALID_ARG, "graph is NULL");
        if (mode != HF_MODE_LATE && mode != HF_MODE_EARLY)
            fail(HF_ERR_INVALID_ARG, "mode must be HF_MODE_LATE or HF_MODE_EARLY");
        G(h)->early = mode == HF_MODE_EARLY;
        return HF_OK;
    });
}

hf_status hf_graph_info(hf_graph h, int32_t *n, int32_t *m, int32_t *num_levels) {
    return guarded([&]() -> hf_status {
        if (!h) fail(HF_ERR_INVALID_ARG, "graph is NULL");
        Graph *g = G(h);
        if (n) *n = g->n;
        if (m) *m = g->m;
        if (num_levels) *num_levels = g->levelized ? g->L : -1;
        return HF_OK;
    });
}

hf_status hf_sync(hf_graph h) {
    return guarded([&]() -> hf_status {
        if (!h) fail(HF_ERR_INVALID_ARG, "graph is NULL");
        Graph *g = G(h);
        DeviceGuard dg(g->device);
        return latch(*g);
    });
}

static hf_status levelize_impl(hf_graph h, int32_t *num_levels, int32_t *level, int32_t *lptr,
                               int32_t *order, bool device_out) {
    return guarded([&]() -> hf_status {
        if (!h) fail(HF_ERR_INVALID_ARG, "graph is NULL");
        Graph *g = G(h);
        DeviceGuard dg(g->device);
        if (g->prof) profile_mark(*g, 0);
        int64_t unready = levelize_device(*g);
        if (g->prof) profile_mark(*g, 1);   // read (synchronising) by hf_profile_read
        if (unready) {
            fail(HF_ERR_CYCLE, "cycle: " + std::to_string(unready) + " nodes never become ready");
        }
        if (num_levels) *num_levels = g->L;
        cudaMemcpyKind k = device_out ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
        if (level && g->n)
            HF_CUDA(cudaMemcpyAsync(level, g->level.p, sizeof(int32_t) * g->n, k, g->stream));
        if (order && g->n)
            HF_CUDA(cudaMemcpyAsync(order, g->order.p, sizeof(int32_t) * g->n, k, g->stream));
        if (lptr)
            HF_CUDA(cudaMemcpyAsync(lptr, g->level_ptr.p, sizeof(int32_t) * (g->L + 1), k,
                                    g->stream));
        HF_CUDA(cudaStreamSynchronize(g->stream));
        return HF_OK;
    });
}

hf_status hf_levelize(hf_graph g, int32_t *num_levels, int32_t *level, int32_t *level_ptr,
                      int32_t *order) {
    return levelize_impl(g, num_levels, level, level_ptr, order, false);
}

hf_status hf_levelize_d(hf_graph g, int32_t *num_levels, int32_t *level_d, int32_t *level_ptr_d,
                        int32_t *order_d) {
    return levelize_impl(g, num_levels, level_d, level_ptr_d, order_d, true);
}

static void need_levels(Graph *g) {
    if (!g->levelized) fail(HF_ERR_NOT_LEVELIZED, "call hf_levelize first");
}

static void prof_elapsed(Graph *g) {
    if (!g->prof) return;
    float ms = 0;
    if (cudaEventElapsedTime(&ms, g->ev[0], g->ev[1]) == cudaSuccess) g->ms_lev = ms;
    if (cudaEventElapsedTime(&ms, g->ev[2], g->ev[3]) == cudaSuccess) g->ms_fwd = ms;
    if (cudaEventElapsedTime(&ms, g->ev[5], g->ev[4]) == cudaSuccess) g->ms_bwd = ms;
    if (cudaEventElapsedTime(&ms, g->ev[6], g->ev[7]) == cudaSuccess) g->ms_prop = ms;
    cudaGetLastError();   // clear "not recorded" errors
}

hf_status hf_propagate_forward_d(hf_graph h, const float *at_src_d, float *at_d) {
    return guarded([&]() -> hf_status {
        if (!h || !at_d) fail(HF_ERR_INVALID_ARG, "graph or at is NULL");
        Graph *g = G(h);
        DeviceGuard dg(g->device);
        need_levels(g);
        forward_device(*g, g->delay.as<float>(), 1, false, at_src_d, at_d);
        return HF_OK;
    });
}

hf_status hf_propagate_forward(hf_graph h, const float *at_src, float *at) {
    return guarded([&]() -> hf_status {
        if (!h || !at) fail(HF_ERR_INVALID_ARG, "graph or at is NULL");
        Graph *g = G(h);
        DeviceGuard dg(g->device);
        need_levels(g);
        for (int32_t i = 0; at_src && i < g->n; ++i)
            if (!std::isfinite(at_src[i])) fail(HF_ERR_INVALID_ARG, "at_src has NaN or inf");
        DevBuf a, o;
        a.alloc(sizeof(float) * g->n, g->stream);
        o.alloc(sizeof(float) * g->n, g->stream);
        if (at_src && g->n)
            HF_CUDA(cudaMemcpyAsync(a.p, at_src, sizeof(float) * g->n, cudaMemcpyHostToDevice,
                                    g->stream));
        forward_device(*g, g->delay.as<float>(), 1, false, at_src ? a.as<float>() : nullptr,
                       o.as<float>());
        if (g->n)
            HF_CUDA(cudaMemcpyAsync(at, o.p, sizeof(float) * g->n, cudaMemcpyDeviceToHost,
                                    g->stream));
        return latch(*g);
    });
}

hf_status hf_propagate_backward_d(hf_graph h, float t_req, const float *at_d, float *rat_d,
                                  float *slack_d, float *wns_d) {
    return guarded([&]() -> hf_status {
        if (!h || !at_d || !rat_d) fail(HF_ERR_INVALID_ARG, "graph, at or rat is NULL");
        if (!std::isfinite(t_req)) fail(HF_ERR_INVALID_ARG, "t_req is NaN or inf");
        Graph *g = G(h);
        DeviceGuard dg(g->device);
        need_levels(g);
        backward_device(*g, g->delay.as<float>(), 1, nullptr, t_req, at_d, rat_d, slack_d, wns_d);
        return HF_OK;
    });
}

hf_status hf_propagate_backward(hf_graph h, float t_req, const float *at, float *rat,
                                float *slack, float *wns) {
    return guarded([&]() -> hf_status {
        if (!h || !at || !rat) fail(HF_ERR_INVALID_ARG, "graph, at or rat is NULL");
        if (!std::isfinite(t_req)) fail(HF_ERR_INVALID_ARG, "t_req is NaN or inf");
        Graph *g = G(h);
        DeviceGuard dg(g->device);
        need_levels(g);
        size_t nb = sizeof(float) * size_t(g->n);
        DevBuf a, r, sl, w;
        a.alloc(nb, g->stream);
        r.alloc(nb, g->stream);
        if (slack) sl.alloc(nb, g->stream);
        w.alloc(sizeof(float), g->stream);
        if (g->n) HF_CUDA(cudaMemcpyAsync(a.p, at, nb, cudaMemcpyHostToDevice, g->stream));
        backward_device(*g, g->delay.as<float>(), 1, nullptr, t_req, a.as<float>(), r.as<float>(),
                        slack ? sl.as<float>() : nullptr, w.as<float>());
        if (g->n) HF_CUDA(cudaMemcpyAsync(rat, r.p, nb, cudaMemcpyDeviceToHost, g->stream));
        if (slack && g->n)
            HF_CUDA(cudaMemcpyAsync(slack, sl.p, nb, cudaMemcpyDeviceToHost, g->stream));
        float wv = 0;
        HF_CUDA(cudaMemcpyAsync(&wv, w.p, sizeof(float), cudaMemcpyDeviceToHost, g->stream));
        const hf_status st = latch(*g);
        if (wns) *wns = wv;
        return st;
    });
}

// core of both batch variants (device pointers, layout already [m][S])
static void batch_core(Graph *g, int32_t S, const float *d_ms, const float *t_d,
                       const float *at_src_d, float *wns_d, float *at_d, float *rat_d,
                       void *comm, float *wns_all_d) {
    size_t nb = sizeof(float) * size_t(g->n) * size_t(S);
    if (!at_d) {   // workspace kept in the graph across calls (grows on demand)
        if (g->ws_at.bytes < nb || g->ws_at.s != g->stream) g->ws_at.alloc(nb, g->stream);
        at_d = g->ws_at.as<float>();
    }
    if (!rat_d) {
        if (g->ws_rat.bytes < nb || g->ws_rat.s != g->stream) g->ws_rat.alloc(nb, g->stream);
        rat_d = g->ws_rat.as<float>();
    }
    batch_device(*g, d_ms, S, true, at_src_d, t_d, at_d, rat_d, nullptr, wns_d);
    if (comm) {
        nccl::load();
        nccl::check(nccl::api.all_gather(wns_d, wns_all_d, size_t(S), nccl::kFloat32, comm,
                                         g->stream),
                    "ncclAllGather");
    }
}

__global__ void k_transpose_sm_to_ms(const float *__restrict__ in, float *__restrict__ out,
                                     int32_t S, int32_t m) {
    __shared__ float tile[32][33];
    for (int64_t eb = int64_t(blockIdx.x) * 32; eb < m; eb += int64_t(gridDim.x) * 32) {
        for (int sb = 0; sb < S; sb += 32) {
            int e = int(eb) + threadIdx.x;
            for (int j = threadIdx.y; j < 32; j += blockDim.y) {
                int s = sb + j;
                tile[j][threadIdx.x] = (e < m && s < S) ? in[int64_t(s) * m + e] : 0.0f;
            }
            __syncthreads();
            for (int j = threadIdx.y; j < 32; j += blockDim.y) {
                int ee = int(eb) + j;
                int s = sb + threadIdx.x;
                if (ee < m && s < S) out[int64_t(ee) * S + s] = tile[threadIdx.x][j];
            }
            __syncthreads();
        }
    }
}

hf_status hf_run_batch_d(hf_graph h, int32_t s_local, const float *delays_d, int layout,
                         const float *t_req_d, const float *at_src_d, float *wns_local_d,
                         float *at_d, float *rat_d, void *comm, float *wns_all_d) {
    return guarded([&]() -> hf_status {
        if (!h || !delays_d || !t_req_d || !wns_local_d)
            fail(HF_ERR_INVALID_ARG, "graph, delays, t_req or wns_local is NULL");
        if (s_local < 1 || s_local > HF_MAX_SCENARIOS)
            fail(HF_ERR_INVALID_ARG, "s_local outside [1, HF_MAX_SCENARIOS]");
        if (layout != HF_LAYOUT_SM && layout != HF_LAYOUT_MS) fail(HF_ERR_INVALID_ARG, "layout");
        if (comm && !wns_all_d) fail(HF_ERR_INVALID_ARG, "wns_all is NULL with a communicator");
        Graph *g = G(h);
        DeviceGuard dg(g->device);
        need_levels(g);
        const float *d = delays_d;
        DevBuf tr;
        if (layout == HF_LAYOUT_SM && s_local > 1 && g->m > 0) {
            tr.alloc(sizeof(float) * size_t(g->m) * s_local, g->stream);
            k_transpose_sm_to_ms<<<grid_for((g->m + 31) / 32, 1, g->sms, 8), dim3(32, 8), 0,
                                   g->stream>>>(delays_d, tr.as<float>(), s_local, g->m);
            HF_CHECK_LAUNCH();
            g->launches += 1;
            d = tr.as<float>();
        }
        batch_core(g, s_local, d, t_req_d, at_src_d, wns_local_d, at_d, rat_d, comm, wns_all_d);
        return HF_OK;
    });
}

hf_status hf_run_batch(hf_graph h, int32_t s_local, const float *delays, int layout,
                       const float *t_req, const float *at_src, float *wns_local, void *comm,
                       float *wns_all) {
    return guarded([&]() -> hf_status {
        if (!h || !delays || !t_req || !wns_local)
            fail(HF_ERR_INVALID_ARG, "graph, delays, t_req or wns_local is NULL");
        if (s_local < 1 || s_local > HF_MAX_SCENARIOS)
            fail(HF_ERR_INVALID_ARG, "s_local outside [1, HF_MAX_SCENARIOS]");
        if (layout != HF_LAYOUT_SM && layout != HF_LAYOUT_MS) fail(HF_ERR_INVALID_ARG, "layout");
        if (comm && !wns_all) fail(HF_ERR_INVALID_ARG, "wns_all is NULL with a communicator");
        Graph *g = G(h);
        DeviceGuard dg(g->device);
        need_levels(g);
        cudaStream_t s = g->stream;
        size_t db = sizeof(float) * size_t(g->m) * s_local;
        DevBuf d, t, a, w, wa;
        d.alloc(db, s);
        t.alloc(sizeof(float) * s_local, s);
        w.alloc(sizeof(float) * s_local, s);
        if (db) HF_CUDA(cudaMemcpyAsync(d.p, delays, db, cudaMemcpyHostToDevice, s));
        HF_CUDA(cudaMemcpyAsync(t.p, t_req, sizeof(float) * s_local, cudaMemcpyHostToDevice, s));
        if (at_src) {
            a.alloc(sizeof(float) * g->n, s);
            if (g->n)
                HF_CUDA(cudaMemcpyAsync(a.p, at_src, sizeof(float) * g->n,
                                        cudaMemcpyHostToDevice, s));
        }
        int nranks = 1;
        if (comm) {
            // size of the gather output = s_local * nranks; query via NCCL-free path:
            // the caller guarantees wns_all holds s_local*nranks floats; we learn nranks
            // from the communicator through ncclCommCount.
            nccl::load();
            typedef int (*CommCount_t)(void *, int *);
            auto cc = (CommCount_t)dlsym(nccl::api.h, "ncclCommCount");
            if (!cc) fail(HF_ERR_NCCL, "ncclCommCount missing");
            nccl::check(cc(comm, &nranks), "ncclCommCount");
            wa.alloc(sizeof(float) * s_local * nranks, s);
        }
        const float *dp = d.as<float>();
        DevBuf tr;
        if (layout == HF_LAYOUT_SM && s_local > 1 && g->m > 0) {
            tr.alloc(db, s);
            k_transpose_sm_to_ms<<<grid_for((g->m + 31) / 32, 1, g->sms, 8), dim3(32, 8), 0, s>>>(
                d.as<float>(), tr.as<float>(), s_local, g->m);
            HF_CHECK_LAUNCH();
            g->launches += 1;
            dp = tr.as<float>();
        }
        batch_core(g, s_local, dp, t.as<float>(), at_src ? a.as<float>() : nullptr, w.as<float>(),
                   nullptr, nullptr, comm, comm ? wa.as<float>() : nullptr);
        HF_CUDA(cudaMemcpyAsync(wns_local, w.p, sizeof(float) * s_local, cudaMemcpyDeviceToHost,
                                s));
        if (comm)
            HF_CUDA(cudaMemcpyAsync(wns_all, wa.p, sizeof(float) * s_local * nranks,
                                    cudaMemcpyDeviceToHost, s));
        return latch(*g);
    });
}

// upload stream + events for hf_analyze, one set per host thread and device (its
// own stream: the graph's side stream carries levelize work that must not queue
// behind a multi-millisecond upload)
struct Uploader {
    cudaStream_t s = nullptr;
    cudaEvent_t fork = nullptr, done = nullptr;
};
static Uploader &uploader_of(int device) {
    thread_local Uploader ups[64];
    Uploader &u = ups[device & 63];
    if (!u.s) {
        HF_CUDA(cudaStreamCreateWithFlags(&u.s, cudaStreamNonBlocking));
        HF_CUDA(cudaEventCreateWithFlags(&u.fork, cudaEventDisableTiming));
        HF_CUDA(cudaEventCreateWithFlags(&u.done, cudaEventDisableTiming));
    }
    return u;
}

hf_status hf_analyze(int32_t n, int32_t m, const int32_t *fanin_ptr, const int32_t *fanin_src,
                     const float *delay, int32_t s_local, const float *delays, const float *t_req,
                     const float *at_src, float *wns_local, int32_t *num_levels, int device,
                     void *cuda_stream, hf_graph *out_graph) {
    hf_graph h = nullptr;
    const hf_status st = guarded([&]() -> hf_status {
        if (out_graph) *out_graph = nullptr;
        if (s_local < 1 || s_local > HF_MAX_SCENARIOS)
            fail(HF_ERR_INVALID_ARG, "s_local outside [1, HF_MAX_SCENARIOS]");
        if (!delays || !t_req || !wns_local)
            fail(HF_ERR_INVALID_ARG, "delays, t_req or wns_local is NULL");
        if (n < 0 || m < 0) fail(HF_ERR_INVALID_ARG, "negative n or m");
        int ndev = 0;
        HF_CUDA(cudaGetDeviceCount(&ndev));
        if (device < 0 || device >= ndev) fail(HF_ERR_INVALID_ARG, "bad device ordinal");
        DeviceGuard dg(device);
        init_pool(device);
        Uploader &up = uploader_of(device);
        // the scenario data goes up on the upload stream while the graph is built
        HF_CUDA(cudaEventRecord(up.fork, static_cast<cudaStream_t>(cuda_stream)));
        HF_CUDA(cudaStreamWaitEvent(up.s, up.fork, 0));
        struct Drain {   // host buffers stay in use until the upload stream drains
            cudaStream_t s;
            ~Drain() { cudaStreamSynchronize(s); }
        } drain{up.s};
        const size_t db = sizeof(float) * size_t(m) * size_t(s_local);
        DevBuf d, t, a;
        d.alloc(db > 0 ? db : 4, up.s);
        t.alloc(sizeof(float) * size_t(s_local), up.s);
        if (db) HF_CUDA(cudaMemcpyAsync(d.p, delays, db, cudaMemcpyHostToDevice, up.s));
        HF_CUDA(cudaMemcpyAsync(t.p, t_req, sizeof(float) * size_t(s_local),
                                cudaMemcpyHostToDevice, up.s));
        if (at_src && n) {
            a.alloc(sizeof(float) * size_t(n), up.s);
            HF_CUDA(cudaMemcpyAsync(a.p, at_src, sizeof(float) * size_t(n),
                                    cudaMemcpyHostToDevice, up.s));
        }
        HF_CUDA(cudaEventRecord(up.done, up.s));
        hf_status cs = create_impl(false, n, m, fanin_ptr, fanin_src, nullptr, nullptr, delay,
                                   device, cuda_stream, &h);
        if (cs != HF_OK) return cs;
        cs = levelize_impl(h, num_levels, nullptr, nullptr, nullptr, false);
        if (cs != HF_OK) return cs;
        Graph *g = G(h);
        HF_CUDA(cudaStreamWaitEvent(g->stream, up.done, 0));
        DevBuf w;
        w.alloc(sizeof(float) * size_t(s_local), g->stream);
        batch_core(g, s_local, d.as<float>(), t.as<float>(), (at_src && n) ? a.as<float>() : nullptr,
                   w.as<float>(), nullptr, nullptr, nullptr, nullptr);
        HF_CUDA(cudaMemcpyAsync(wns_local, w.p, sizeof(float) * size_t(s_local),
                                cudaMemcpyDeviceToHost, g->stream));
        // latch synchronises the graph's stream: the batch is done before d/t/a are
        // freed (stream-ordered on the upload stream)
        return latch(*g);
    });
    if (st != HF_OK || !out_graph) {
        if (h) hf_graph_destroy(h);
        h = nullptr;
    }
    if (out_graph) *out_graph = h;
    return st;
}

hf_status hf_nccl_unique_id(void *id128) {
    return guarded([&]() -> hf_status {
        if (!id128) fail(HF_ERR_INVALID_ARG, "id is NULL");
        nccl::load();
        nccl::UniqueId id;
        nccl::check(nccl::api.get_unique_id(&id), "ncclGetUniqueId");
        memcpy(id128, &id, sizeof(id));
        return HF_OK;
    });
}

hf_status hf_nccl_comm_init(const void *id128, int rank, int nranks, int device, void **comm) {
    return guarded([&]() -> hf_status {
        if (!id128 || !comm) fail(HF_ERR_INVALID_ARG, "id or comm is NULL");
        if (nranks < 1 || rank < 0 || rank >= nranks) fail(HF_ERR_INVALID_ARG, "rank/nranks");
        nccl::load();
        DeviceGuard dg(device);
        nccl::UniqueId id;
        memcpy(&id, id128, sizeof(id));
        nccl::Comm c = nullptr;
        nccl::check(nccl::api.comm_init_rank(&c, nranks, id, rank), "ncclCommInitRank");
        *comm = c;
        return HF_OK;
    });
}

hf_status hf_nccl_comm_destroy(void *comm) {
    return guarded([&]() -> hf_status {
        if (!comm) return HF_OK;
        nccl::load();
        nccl::check(nccl::api.comm_destroy(comm), "ncclCommDestroy");
        return HF_OK;
    });
}

hf_status hf_profile_enable(hf_graph h, int on) {
    return guarded([&]() -> hf_status {
        if (!h) fail(HF_ERR_INVALID_ARG, "graph is NULL");
        Graph *g = G(h);
        DeviceGuard dg(g->device);
        if (on && !g->ev[0])
            for (auto &e : g->ev) HF_CUDA(cudaEventCreate(&e));
        g->prof = on != 0;
        return HF_OK;
    });
}

hf_status hf_profile_read(hf_graph h, float *ms_levelize, float *ms_forward, float *ms_backward,
                          int64_t *kernel_launches) {
    return guarded([&]() -> hf_status {
        if (!h) fail(HF_ERR_INVALID_ARG, "graph is NULL");
        Graph *g = G(h);
        DeviceGuard dg(g->device);
        if (g->prof) {
            HF_CUDA(cudaStreamSynchronize(g->stream));
            prof_elapsed(g);
        }
        if (ms_levelize) *ms_levelize = g->ms_lev;
        if (ms_forward) *ms_forward = g->ms_fwd;
        if (ms_backward) *ms_backward = g->ms_bwd;
        if (kernel_launches) *kernel_launches = g->launches;
        return HF_OK;
    });
}

hf_status hf_critical_path_d(hf_graph h, int32_t S, const float *delays_d, const float *at_d,
                             const float *t_req_d, float t_scalar, int32_t max_len,
                             int32_t *path_d, int32_t *path_len_d) {
    return guarded([&]() -> hf_status {
        if (!h || !at_d || !path_d || !path_len_d)
            fail(HF_ERR_INVALID_ARG, "graph, at, path or path_len is NULL");
        if (S < 1 || max_len < 1) fail(HF_ERR_INVALID_ARG, "S and max_len must be >= 1");
        Graph *g = G(h);
        DeviceGuard dg(g->device);
        if (g->early) fail(HF_ERR_INVALID_ARG, "the critical path is defined in late mode only");
        if (!delays_d && S != 1) fail(HF_ERR_INVALID_ARG, "graph delays need S == 1");
        critical_path_device(*g, S, delays_d ? delays_d : g->delay.as<float>(), at_d, t_req_d,
                             t_scalar, 1, max_len, nullptr, path_d, path_len_d);
        return HF_OK;
    });
}

hf_status hf_critical_paths_d(hf_graph h, int32_t S, const float *delays_d, const float *at_d,
                              const float *t_req_d, float t_scalar, int32_t K, int32_t max_len,
                              int32_t *endpoints_d, int32_t *path_d, int32_t *path_len_d) {
    return guarded([&]() -> hf_status {
        if (!h || !at_d || !path_d || !path_len_d)
            fail(HF_ERR_INVALID_ARG, "graph, at, path or path_len is NULL");
        if (S < 1 || K < 1 || max_len < 1)
            fail(HF_ERR_INVALID_ARG, "S, K and max_len must be >= 1");
        Graph *g = G(h);
        DeviceGuard dg(g->device);
        if (g->early) fail(HF_ERR_INVALID_ARG, "the critical path is defined in late mode only");
        if (!delays_d && S != 1) fail(HF_ERR_INVALID_ARG, "graph delays need S == 1");
        critical_path_device(*g, S, delays_d ? delays_d : g->delay.as<float>(), at_d, t_req_d,
                             t_scalar, K, max_len, endpoints_d, path_d, path_len_d);
        return HF_OK;
    });
}

hf_status hf_critical_path(hf_graph h, const float *at, float t_req, int32_t max_len,
                           int32_t *path, int32_t *path_len) {
    return guarded([&]() -> hf_status {
        if (!h || !at || !path || !path_len)
            fail(HF_ERR_INVALID_ARG, "graph, at, path or path_len is NULL");
        if (max_len < 1) fail(HF_ERR_INVALID_ARG, "max_len must be >= 1");
        if (!std::isfinite(t_req)) fail(HF_ERR_INVALID_ARG, "t_req is not finite");
        Graph *g = G(h);
        DeviceGuard dg(g->device);
        if (g->early) fail(HF_ERR_INVALID_ARG, "the critical path is defined in late mode only");
        cudaStream_t s = g->stream;
        DevBuf a, p, l;
        a.alloc(sizeof(float) * size_t(g->n > 0 ? g->n : 1), s);
        p.alloc(sizeof(int32_t) * size_t(max_len), s);
        l.alloc(sizeof(int32_t), s);
        if (g->n)
            HF_CUDA(cudaMemcpyAsync(a.p, at, sizeof(float) * g->n, cudaMemcpyHostToDevice, s));
        critical_path_device(*g, 1, g->delay.as<float>(), a.as<float>(), nullptr, t_req, 1,
                             max_len, nullptr, p.as<int32_t>(), l.as<int32_t>());
        int32_t ln = 0;
        HF_CUDA(cudaMemcpyAsync(&ln, l.p, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
        HF_CUDA(cudaStreamSynchronize(s));
        if (ln < 0) fail(HF_ERR_INVALID_ARG, "at is not a forward result of the graph's delays, "
                                             "or the critical path is longer than max_len");
        if (ln)
            HF_CUDA(cudaMemcpy(path, p.p, sizeof(int32_t) * size_t(ln), cudaMemcpyDeviceToHost));
        *path_len = ln;
        return HF_OK;
    });
}

hf_status hf_mis_d(hf_graph h, const int32_t *prio_d, uint8_t *in_set_d) {
    return guarded([&]() -> hf_status {
        if (!h || !in_set_d) fail(HF_ERR_INVALID_ARG, "graph or in_set is NULL");
        Graph *g = G(h);
        if (g->n && !prio_d) fail(HF_ERR_INVALID_ARG, "prio is NULL");
        DeviceGuard dg(g->device);
        mis_device(*g, prio_d, in_set_d);
        return HF_OK;
    });
}

hf_status hf_mis(hf_graph h, const int32_t *prio, uint8_t *in_set) {
    return guarded([&]() -> hf_status {
        if (!h || !in_set) fail(HF_ERR_INVALID_ARG, "graph or in_set is NULL");
        Graph *g = G(h);
        if (g->n && !prio) fail(HF_ERR_INVALID_ARG, "prio is NULL");
        DeviceGuard dg(g->device);
        cudaStream_t s = g->stream;
        if (g->n == 0) return HF_OK;
        DevBuf pr, out;
        pr.alloc(sizeof(int32_t) * size_t(g->n), s);
        out.alloc(size_t(g->n), s);
        HF_CUDA(cudaMemcpyAsync(pr.p, prio, sizeof(int32_t) * g->n, cudaMemcpyHostToDevice, s));
        mis_device(*g, pr.as<int32_t>(), out.as<uint8_t>());
        HF_CUDA(cudaMemcpyAsync(in_set, out.p, size_t(g->n), cudaMemcpyDeviceToHost, s));
        HF_CUDA(cudaStreamSynchronize(s));
        return latch(*g);
    });
}

hf_status hf_profile_read_batch(hf_graph h, float *ms_batch_propagation) {
    return guarded([&]() -> hf_status {
        if (!h) fail(HF_ERR_INVALID_ARG, "graph is NULL");
        Graph *g = G(h);
        DeviceGuard dg(g->device);
        if (g->prof) {
            HF_CUDA(cudaStreamSynchronize(g->stream));
            prof_elapsed(g);
        }
        if (ms_batch_propagation) *ms_batch_propagation = g->ms_prop;
        return HF_OK;
    });
}

// Test hook (not part of include/hf.h): exclusive scan of n int32 device values
// with the library's scan primitive, on the graph's stream.
hf_status hf_debug_scan(hf_graph h, const int32_t *in_d, int32_t *out_d, int64_t n,
                        int32_t *total_d) {
    return guarded([&]() -> hf_status {
        if (!h) fail(HF_ERR_INVALID_ARG, "graph is NULL");
        Graph *g = G(h);
        DeviceGuard dg(g->device);
        scan_exclusive(in_d, out_d, n, total_d, g->stream, *g);
        HF_CUDA(cudaStreamSynchronize(g->stream));
        return HF_OK;
    });
}

}  // extern "C"
