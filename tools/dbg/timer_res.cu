// Resolution of %globaltimer against the SM clock on this GPU: one thread reads both
// back to back and records every globaltimer change (ns step, SM cycles since the
// previous change).  Tells whether the HF_TRACE per-task intervals (globaltimer) can
// resolve sub-microsecond phases.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/timer_res tools/dbg/timer_res.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k(unsigned long long *out, int n) {
    unsigned long long g0, g, c0, c;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
    c0 = clock64();
    int k = 0;
    while (k < n) {
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
        if (g != g0) {
            c = clock64();
            out[2 * k] = g - g0;
            out[2 * k + 1] = c - c0;
            g0 = g;
            c0 = c;
            ++k;
        }
    }
}

int main() {
    const int n = 2000;
    unsigned long long *d, h[2 * n];
    cudaMalloc(&d, sizeof(h));
    k<<<1, 1>>>(d, n);
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double sg = 0, sc = 0;
    unsigned long long mn = ~0ull, mx = 0;
    for (int i = 1; i < n; ++i) {
        sg += h[2 * i];
        sc += h[2 * i + 1];
        mn = h[2 * i] < mn ? h[2 * i] : mn;
        mx = h[2 * i] > mx ? h[2 * i] : mx;
    }
    printf("globaltimer steps: mean %.1f ns (min %llu, max %llu), %.1f SM cycles per step\n",
           sg / (n - 1), mn, mx, sc / (n - 1));
    for (int i = 1; i < 12; ++i) printf("  step %llu ns, %llu cycles\n", h[2 * i], h[2 * i + 1]);
    return 0;
}
