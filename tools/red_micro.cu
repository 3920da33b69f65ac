// red_micro.cu -- cost of the cross-CTA y reduction of the fused decode kernel (one CTA per SM,
// 256 threads, each owning 16 of 4096 f32 columns) under different schemes.
//   A: red.global.add.v4 of every column from every CTA (what the kernel does)
//   B: as A, each CTA starting at a rotated column offset
//   C: 2-CTA clusters: halves exchanged through DSMEM, each CTA reds its half
//   D: as A into R copies (CTA c -> copy c % R), no final combine (lower bound for spreading)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o red_micro red_micro.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>

namespace cg = cooperative_groups;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ void red4(float* a, float x, float y, float z, float w) {
    asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(a), "f"(x), "f"(y), "f"(z), "f"(w) : "memory");
}

constexpr int D = 4096;

__global__ void __launch_bounds__(256) empty_k(float* y);

__device__ unsigned long long g_t[2][1024];
__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__global__ void __launch_bounds__(256) red_all(float* y, int rotate, int copies) {
    const int t = threadIdx.x;
    if (t == 0) g_t[0][blockIdx.x] = gtime();
    float* dst = y + (blockIdx.x % copies) * D;
    const int off = rotate ? (blockIdx.x * 128) % D : 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const int col = (off + (t + k * 256) * 4) % D;
        red4(dst + col, 1.f, 1.f, 1.f, 1.f);
    }
    __syncthreads();
    if (t == 0) {
        __threadfence();
        g_t[1][blockIdx.x] = gtime();
    }
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(256) red_cluster(float* y) {
    __shared__ float4 half_in[512];
    if (threadIdx.x == 0) g_t[0][blockIdx.x] = gtime();
    cg::cluster_group cl = cg::this_cluster();
    const unsigned rank = cl.block_rank();
    const int t = threadIdx.x;
    float4 mine[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) mine[k] = make_float4(1.f, 1.f, 1.f, 1.f);
    // columns [rank*2048, rank*2048+2048) are owned by this CTA; send the other half
    float4* peer = cl.map_shared_rank(half_in, rank ^ 1);
#pragma unroll
    for (int k = 0; k < 2; ++k) peer[t + k * 256] = mine[(rank ^ 1) * 2 + k];
    cl.sync();
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        const float4 o = half_in[t + k * 256];
        const float4 m = mine[rank * 2 + k];
        const int col = rank * 2048 + (t + k * 256) * 4;
        red4(y + col, m.x + o.x, m.y + o.y, m.z + o.z, m.w + o.w);
    }
    __syncthreads();
    if (t == 0) {
        __threadfence();
        g_t[1][blockIdx.x] = gtime();
    }
}

__device__ __forceinline__ unsigned smem_addr(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }

// E: each CTA stages its 16 KB partial in smem and issues ONE bulk reduction into y (the fused
// decode kernel's epilogue)
__global__ void __launch_bounds__(256) bulk_all(float* y) {
    __shared__ __align__(128) float ys[D];
    const int t = threadIdx.x;
    if (t == 0) g_t[0][blockIdx.x] = gtime();
    for (int i = t; i < D; i += 256) ys[i] = 1.f;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (t == 0) {
        asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], %2;" ::"l"(y),
                     "r"(smem_addr(ys)), "r"(D * 4) : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        g_t[1][blockIdx.x] = gtime();
    }
}

// F: 2-CTA clusters: rank 1 adds its partial into rank 0's smem over DSMEM, rank 0 bulk-reduces
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(256) bulk_cluster(float* y) {
    __shared__ __align__(128) float ys[D];
    cg::cluster_group cl = cg::this_cluster();
    const unsigned rank = cl.block_rank();
    const int t = threadIdx.x;
    if (t == 0) g_t[0][blockIdx.x] = gtime();
    for (int i = t; i < D; i += 256) ys[i] = 1.f;
    cl.sync();
    if (rank == 1) {
        float* peer = cl.map_shared_rank(ys, 0);
        for (int i = t * 4; i < D; i += 256 * 4) {
            const float4 v = *reinterpret_cast<const float4*>(ys + i);
            atomicAdd(peer + i, v.x);
            atomicAdd(peer + i + 1, v.y);
            atomicAdd(peer + i + 2, v.z);
            atomicAdd(peer + i + 3, v.w);
        }
    }
    cl.sync();
    if (rank == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        if (t == 0) {
            asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], %2;" ::"l"(y),
                         "r"(smem_addr(ys)), "r"(D * 4) : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        }
    }
    if (t == 0) g_t[1][blockIdx.x] = gtime();
}

__global__ void __launch_bounds__(256) empty_k(float* y) {
    if (threadIdx.x == 0) { g_t[0][blockIdx.x] = gtime(); __threadfence(); g_t[1][blockIdx.x] = gtime(); }
}

int main() {
    int nsm = 0;
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
    float* y;
    CK(cudaMalloc(&y, 16 * D * sizeof(float)));
    CK(cudaMemset(y, 0, 16 * D * sizeof(float)));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto time_it = [&](const char* name, auto fn) {
        for (int i = 0; i < 20; ++i) fn();
        cudaDeviceSynchronize();
        const int R = 200;
        cudaEventRecord(e0);
        for (int i = 0; i < R; ++i) fn();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        unsigned long long h[2][1024];
        cudaMemcpyFromSymbol(h, g_t, sizeof(h));
        unsigned long long t0 = ~0ull, t1 = 0;
        double mx = 0;
        for (int i = 0; i < nsm; ++i) {
            t0 = h[0][i] < t0 ? h[0][i] : t0;
            t1 = h[1][i] > t1 ? h[1][i] : t1;
            mx = (h[1][i] - h[0][i]) > mx ? (h[1][i] - h[0][i]) : mx;
        }
        printf("%-44s %7.2f us / launch   last launch: span %6.2f us, max per-CTA %6.2f us\n", name, ms * 1e3 / R,
               (t1 - t0) / 1e3, mx / 1e3);
    };
    time_it("empty launch (grid=SMs)", [&] { empty_k<<<nsm, 256>>>(y); });
    time_it("A red.v4 all CTAs -> one y", [&] { red_all<<<nsm, 256>>>(y, 0, 1); });
    time_it("B rotated start", [&] { red_all<<<nsm, 256>>>(y, 1, 1); });
    time_it("D 2 copies", [&] { red_all<<<nsm, 256>>>(y, 0, 2); });
    time_it("D 4 copies", [&] { red_all<<<nsm, 256>>>(y, 0, 4); });
    time_it("D 8 copies", [&] { red_all<<<nsm, 256>>>(y, 0, 8); });
    time_it("D 8 copies rotated", [&] { red_all<<<nsm, 256>>>(y, 1, 8); });
    time_it("C 2-CTA cluster DSMEM halves", [&] { red_cluster<<<nsm, 256>>>(y); });
    time_it("E bulk reduce 16 KB per CTA -> one y", [&] { bulk_all<<<nsm, 256>>>(y); });
    time_it("F 2-CTA cluster DSMEM add + bulk reduce", [&] { bulk_cluster<<<nsm, 256>>>(y); });
    CK(cudaGetLastError());
    return 0;
}
