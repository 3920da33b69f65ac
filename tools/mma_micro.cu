// mma_micro.cu -- cycles of the fused kernel's stage-2 inner loop (one 16-row tile, 32 k-steps
// of mma.sync m16n8k16 bf16 from shared memory) for 1..8 concurrent warps, and of a dependent
// mma chain, to size the predictor stage.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ void mma16816(float (&d)[4], const uint4& a, const uint2& b) {
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                 : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3]) : "r"(a.x), "r"(a.y), "r"(a.z), "r"(a.w), "r"(b.x), "r"(b.y));
}

__global__ void k(long long* out, float* sink, int nwarps_active, int kst, int chains) {
    __shared__ uint4 A[2 * 32 * 32];  // 4 tiles x 32 k-steps x 32 lanes x 16 B = 64 KB... keep 32 KB static limit: 2 tiles
    __shared__ uint2 B[32 * 32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < 2 * 32 * 32; i += blockDim.x) A[i] = make_uint4(i, i + 1, i + 2, i + 3);
    for (int i = threadIdx.x; i < 32 * 32; i += blockDim.x) B[i] = make_uint2(i, i * 3);
    __syncthreads();
    if (warp < nwarps_active) {
        float acc0[4] = {0, 0, 0, 0}, acc1[4] = {0, 0, 0, 0};
        const uint4* a = A + warp % 2 * kst * 32 + lane;
        const uint2* b = B + lane;
        const long long t0 = clock64();
        if (chains == 2) {
            int s = 0;
#pragma unroll 4
            for (; s + 1 < kst; s += 2) {
                mma16816(acc0, a[s * 32], b[s * 32]);
                mma16816(acc1, a[(s + 1) * 32], b[(s + 1) * 32]);
            }
        } else {
#pragma unroll 4
            for (int s = 0; s < kst; ++s) mma16816(acc0, a[s * 32], b[s * 32]);
        }
        const float z = acc0[0] + acc0[1] + acc1[0] + acc1[1] + acc0[2] + acc1[3];
        const long long t1 = clock64();
        if (lane == 0) out[blockIdx.x * 8 + warp] = t1 - t0;
        if (z == 1234.5f) *sink = z;
    }
}

int main() {
    long long* out; float* sink;
    CK(cudaMalloc(&out, 148 * 8 * 8)); CK(cudaMalloc(&sink, 4));
    CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 0));
    for (int chains : {1, 2})
        for (int nw : {1, 4, 8}) {
            k<<<1, 256>>>(out, sink, nw, 32, chains);
            CK(cudaDeviceSynchronize());
            k<<<1, 256>>>(out, sink, nw, 32, chains);
            CK(cudaDeviceSynchronize());
            long long h[8];
            CK(cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost));
            long long mx = 0;
            for (int w = 0; w < nw; ++w) mx = h[w] > mx ? h[w] : mx;
            printf("chains %d, %d warps: 32 k-steps in %lld cycles (max over warps)\n", chains, nw, mx);
        }
    return 0;
}
