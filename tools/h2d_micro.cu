// h2d_micro.cu -- latency of getting 16 KB of host (pinned, mapped) data into device memory:
// a copy kernel (various shapes) vs cudaMemcpyAsync, each timed alone with events (median).
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>
__global__ void kcopy(uint4* dst, const uint4* src, int n16) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += gridDim.x * blockDim.x) dst[i] = __ldcv(src + i);
}
__global__ void kcopy_nc(uint4* dst, const uint4* src, int n16) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += gridDim.x * blockDim.x) dst[i] = src[i];
}
int main() {
    const int bytes = 16384, n16 = bytes / 16;
    uint4 *h, *d;
    cudaHostAlloc(&h, bytes, cudaHostAllocMapped);
    cudaMalloc(&d, bytes);
    cudaStream_t s; cudaStreamCreate(&s);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    auto run = [&](const char* name, auto fn) {
        std::vector<float> t;
        for (int r = 0; r < 200; ++r) {
            cudaEventRecord(e0, s); fn(); cudaEventRecord(e1, s); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1); t.push_back(ms * 1e3f);
        }
        std::sort(t.begin(), t.end());
        printf("%-40s median %6.2f us  p10 %6.2f\n", name, t[100], t[20]);
    };
    run("empty kernel", [&] { kcopy<<<1, 32, 0, s>>>(d, h, 0); });
    run("kcopy 4x256 ldcv", [&] { kcopy<<<4, 256, 0, s>>>(d, h, n16); });
    run("kcopy 1x1024 ldcv", [&] { kcopy<<<1, 1024, 0, s>>>(d, h, n16); });
    run("kcopy 8x128", [&] { kcopy_nc<<<8, 128, 0, s>>>(d, h, n16); });
    run("kcopy 16x64", [&] { kcopy_nc<<<16, 64, 0, s>>>(d, h, n16); });
    run("memcpyAsync H2D 16KB", [&] { cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, s); });
    run("kcopy D2H 4x256", [&] { kcopy<<<4, 256, 0, s>>>(h, d, n16); });
    run("memcpyAsync D2H 16KB", [&] { cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost, s); });
    return 0;
}
