// bar_micro.cu -- latency of a software grid barrier across all SMs (one CTA per SM), the
// building block of the fused decode kernel.  Variants: release-red arrival + relaxed polling
// (A), atomicAdd arrival (B), and A with one polling warp per CTA using ld.acquire (C).
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ unsigned long long ld_relaxed(const unsigned long long* p) {
    unsigned long long v; asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory"); return v;
}
__device__ __forceinline__ unsigned long long ld_acq(const unsigned long long* p) {
    unsigned long long v; asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory"); return v;
}
__device__ __forceinline__ void red_rel(unsigned long long* p) {
    asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(p) : "memory");
}

template <int V>
__global__ void __launch_bounds__(288, 1) bar_k(unsigned long long* cnt, int iters, float* sink) {
    __shared__ float pad[40000];  // one CTA per SM
    const unsigned long long base = ld_relaxed(cnt) / gridDim.x * gridDim.x;
    for (int it = 0; it < iters; ++it) {
        __syncthreads();
        if (threadIdx.x == 0) {
            const unsigned long long target = base + (unsigned long long)(it + 1) * gridDim.x;
            if (V == 1) {
                __threadfence();
                atomicAdd(cnt, 1ull);
                while (ld_relaxed(cnt) < target) {}
                __threadfence();
            } else if (V == 2) {
                red_rel(cnt);
                while (ld_acq(cnt) < target) {}
            } else {
                red_rel(cnt);
                while (ld_relaxed(cnt) < target) {}
                asm volatile("fence.acq_rel.gpu;" ::: "memory");
            }
        }
        __syncthreads();
    }
    if (threadIdx.x == 0 && pad[threadIdx.x] == 123.f) *sink = pad[1];
}

int main() {
    int nsm;
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
    unsigned long long* cnt; float* sink;
    CK(cudaMalloc(&cnt, 1024)); CK(cudaMalloc(&sink, 4)); CK(cudaMemset(cnt, 0, 1024));
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    auto run = [&](const char* name, auto kern) {
        for (int iters : {1, 101}) {
            kern<<<nsm, 288>>>(cnt, iters, sink);
            cudaDeviceSynchronize();
            cudaEventRecord(e0);
            for (int r = 0; r < 10; ++r) kern<<<nsm, 288>>>(cnt, iters, sink);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            printf("%-40s iters %3d: %8.2f us per launch\n", name, iters, ms * 100.f);
        }
    };
    run("A red.release + relaxed poll + fence", bar_k<0>);
    run("B threadfence + atomicAdd + poll", bar_k<1>);
    run("C red.release + acquire poll", bar_k<2>);
    CK(cudaGetLastError());
    return 0;
}
