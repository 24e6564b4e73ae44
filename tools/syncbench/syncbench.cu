// syncbench.cu -- sync-floor microbenchmarks for the level-synchronous design
// (SURVEY.md §7 step 8): cost of one grid-wide barrier / dependency hop on B200.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o syncbench syncbench.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>

namespace cg = cooperative_groups;

__device__ __forceinline__ unsigned ld_acq(const unsigned *p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// monotonic-counter barrier: red.release + acquire spin by one thread per CTA
__global__ void k_bar_mono(unsigned *count, int iters) {
    unsigned target = 0;
    for (int i = 0; i < iters; ++i) {
        target += gridDim.x;
        __syncthreads();
        if (threadIdx.x == 0) {
            asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(count) : "memory");
            while (ld_acq(count) < target) __nanosleep(20);
        }
        __syncthreads();
    }
}
// same without nanosleep
__global__ void k_bar_mono_spin(unsigned *count, int iters) {
    unsigned target = 0;
    for (int i = 0; i < iters; ++i) {
        target += gridDim.x;
        __syncthreads();
        if (threadIdx.x == 0) {
            asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(count) : "memory");
            while (ld_acq(count) < target) {
            }
        }
        __syncthreads();
    }
}
// cooperative groups grid sync
__global__ void k_bar_cg(int iters) {
    cg::grid_group g = cg::this_grid();
    for (int i = 0; i < iters; ++i) g.sync();
}
// dependency hop: store + fence + flag, next CTA polls (ring of CTAs)
__global__ void k_hop(unsigned *flags, float *data, int iters) {
    // CTA b waits for CTA b-1's flag >= i, then writes data and its flag = i+1
    const int b = blockIdx.x, P = gridDim.x;
    for (int i = 0; i < iters; ++i) {
        if (threadIdx.x == 0) {
            if (!(b == 0 && i == 0)) {
                const int src = (b + P - 1) % P;
                const unsigned want = (b == 0) ? i : i + 1;
                while (ld_acq(flags + src * 32) < want) {
                }
            }
            data[b * 32] = float(i);
            asm volatile("fence.acq_rel.gpu;" ::: "memory");
            asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(flags + b * 32), "r"(i + 1)
                         : "memory");
        }
        __syncthreads();
    }
}
__global__ void k_empty() {}

int main() {
    int dev = 0, sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    unsigned *cnt;
    float *data;
    cudaMalloc(&cnt, 1 << 20);
    cudaMalloc(&data, 1 << 20);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int iters = 2000;
    float ms;
    for (int threads : {256, 1024}) {
        cudaMemset(cnt, 0, 4);
        void *args[] = {&cnt, (void *)&iters};
        int it = iters;
        args[1] = &it;
        cudaLaunchCooperativeKernel((void *)k_bar_mono, sms, threads, args, 0, 0);
        cudaMemset(cnt, 0, 4);
        cudaEventRecord(a);
        cudaLaunchCooperativeKernel((void *)k_bar_mono, sms, threads, args, 0, 0);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf("grid barrier (red.release + acquire spin, nanosleep) %d CTAs x %d: %.3f us\n", sms,
               threads, ms * 1e3 / iters);
        cudaMemset(cnt, 0, 4);
        cudaEventRecord(a);
        cudaLaunchCooperativeKernel((void *)k_bar_mono_spin, sms, threads, args, 0, 0);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf("grid barrier (busy spin)                         %d CTAs x %d: %.3f us\n", sms,
               threads, ms * 1e3 / iters);
        void *args2[] = {&it};
        cudaEventRecord(a);
        cudaLaunchCooperativeKernel((void *)k_bar_cg, sms, threads, args2, 0, 0);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf("cooperative_groups grid.sync                     %d CTAs x %d: %.3f us\n", sms,
               threads, ms * 1e3 / iters);
    }
    {
        cudaMemset(cnt, 0, 1 << 20);
        int it = iters;
        void *args[] = {&cnt, &data, &it};
        cudaEventRecord(a);
        cudaLaunchCooperativeKernel((void *)k_hop, sms, 128, args, 0, 0);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf("CTA->CTA dependency hop (store, fence, flag, poll): %.3f us per hop\n",
               ms * 1e3 / (iters * double(sms)));
    }
    {
        for (int i = 0; i < 100; ++i) k_empty<<<sms, 256>>>();
        cudaEventRecord(a);
        for (int i = 0; i < iters; ++i) k_empty<<<sms, 256>>>();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf("back-to-back empty kernel launches: %.3f us per launch\n", ms * 1e3 / iters);
        cudaStream_t st;
        cudaStreamCreate(&st);
        cudaGraph_t gr;
        cudaGraphExec_t ge;
        cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
        for (int i = 0; i < 200; ++i) k_empty<<<sms, 256, 0, st>>>();
        cudaStreamEndCapture(st, &gr);
        cudaGraphInstantiate(&ge, gr, 0);
        cudaGraphLaunch(ge, st);
        cudaStreamSynchronize(st);
        cudaEventRecord(a, st);
        for (int i = 0; i < 10; ++i) cudaGraphLaunch(ge, st);
        cudaEventRecord(b, st);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf("CUDA graph of empty kernels: %.3f us per kernel node\n", ms * 1e3 / 2000);
    }
    cudaError_t e = cudaDeviceSynchronize();
    printf("status: %s\n", cudaGetErrorString(e));
    return 0;
}
