// Micro-benchmark: latency of every SM reading the SAME 16 KB activation vector (the fused
// kernels' x load) vs each SM reading its own copy (replicas) -- L2 hot-line contention.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/xbcast_micro tools/xbcast_micro.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

__global__ void k_read(const float* x, int d, int nrep, long long* out, float* sink) {
    const long long t0 = clock64();
    const float* src = x + (size_t)(blockIdx.x % nrep) * d;
    float acc = 0.f;
    for (int i = threadIdx.x * 8; i < d; i += blockDim.x * 8) {
        float v[8];
        asm volatile("ld.global.cg.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7])
                     : "l"(src + i));
        for (int k = 0; k < 8; ++k) acc += v[k];
    }
    const long long t1 = clock64();
    __syncthreads();
    const long long t2 = clock64();
    if ((threadIdx.x & 31) == 0) out[blockIdx.x * 32 + threadIdx.x / 32] = t1 - t0;
    if (threadIdx.x == 0) out[blockIdx.x * 32 + 31] = t2 - t0;
    if (acc == 12345.f) sink[0] = acc;
}

int main() {
    const int d = 4096, G = 148, T = 416;
    float* x; long long* out; float* sink;
    cudaMalloc(&x, (size_t)64 * d * 4); cudaMemset(x, 0, (size_t)64 * d * 4);
    cudaMalloc(&out, G * 32 * 8); cudaMalloc(&sink, 4);
    std::vector<long long> h(G * 32);
    for (int nrep : {1, 2, 4, 8, 16, 64}) {
        std::vector<double> warp_med, cta_all;
        for (int it = 0; it < 50; ++it) {
            k_read<<<G, T>>>(x, d, nrep, out, sink);
            cudaDeviceSynchronize();
            if (it < 5) continue;
            cudaMemcpy(h.data(), out, h.size() * 8, cudaMemcpyDeviceToHost);
            std::vector<long long> bar;
            for (int c = 0; c < G; ++c) bar.push_back(h[c * 32 + 31]);
            std::sort(bar.begin(), bar.end());
            cta_all.push_back((double)bar[G / 2]);
            warp_med.push_back((double)bar[G * 9 / 10]);
        }
        std::sort(cta_all.begin(), cta_all.end());
        std::sort(warp_med.begin(), warp_med.end());
        printf("replicas=%2d  CTA all-warps-landed cycles: median-over-CTAs %.0f  p90-over-CTAs %.0f\n", nrep,
               cta_all[cta_all.size() / 2], warp_med[warp_med.size() / 2]);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
