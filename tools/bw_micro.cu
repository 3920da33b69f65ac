// bw_micro.cu -- HBM read-bandwidth microbenchmark for the B200 streaming design choices.
//   A: LDG.128 grid-stride (many CTAs, unrolled)      -- plain load path
//   B: 1-D TMA bulk ring, 1 CTA/SM, 1 issuing lane      -- what k_sparse does
//   C: TMA bulk ring with N CTAs per SM
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bw_micro bw_micro.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void ldg_stream(const uint4* __restrict__ p, size_t n16, unsigned long long* sink) {
    uint32_t acc = 0;
    size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (; i + 7 * stride < n16; i += 8 * stride) {
        uint4 v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = __ldcs(p + i + k * stride);
#pragma unroll
        for (int k = 0; k < 8; ++k) acc ^= v[k].x ^ v[k].y ^ v[k].z ^ v[k].w;
    }
    for (; i < n16; i += stride) { uint4 v = __ldcs(p + i); acc ^= v.x ^ v.w; }
    if (acc == 0x12345678) atomicAdd(sink, 1ull);
}

// chunk = bytes per bulk copy; copies_per_stage; each CTA streams a contiguous range.
__global__ void tma_stream(const uint8_t* __restrict__ p, size_t bytes, int chunk, int cps, int nstages,
                           unsigned long long* sink) {
    extern __shared__ __align__(1024) uint8_t smem[];
    const int stage_bytes = chunk * cps;
    uint64_t* full = (uint64_t*)(smem + (size_t)stage_bytes * nstages);
    uint64_t* empty = full + nstages;
    const int nwc = blockDim.x / 32 - 1;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const size_t per_cta = (bytes / gridDim.x) / stage_bytes * stage_bytes;
    const uint8_t* base = p + per_cta * blockIdx.x;
    const int nst = (int)(per_cta / stage_bytes);
    if (threadIdx.x == 0) {
        for (int s = 0; s < nstages; ++s) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&full[s])), "r"(1));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&empty[s])), "r"(nwc));
        }
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    if (warp == nwc) {
        if (lane == 0) {
            int st = 0; uint32_t ph = 0;
            for (int s = 0; s < nst; ++s) {
                uint32_t ok = 0;
                while (!ok) asm volatile("{.reg .pred q; mbarrier.try_wait.parity.shared::cta.b64 q, [%1], %2; selp.u32 %0,1,0,q;}" : "=r"(ok) : "r"(su32(&empty[st])), "r"(ph ^ 1));
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[st])), "r"(stage_bytes));
                for (int c = 0; c < cps; ++c)
                    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                                 ::"r"(su32(smem + (size_t)st * stage_bytes + (size_t)c * chunk)), "l"(base + (size_t)s * stage_bytes + (size_t)c * chunk),
                                 "r"(chunk), "r"(su32(&full[st])) : "memory");
                if (++st == nstages) { st = 0; ph ^= 1; }
            }
        }
    } else {
        uint32_t acc = 0;
        int st = 0; uint32_t ph = 0;
        for (int s = 0; s < nst; ++s) {
            uint32_t ok = 0;
            while (!ok) asm volatile("{.reg .pred q; mbarrier.try_wait.parity.shared::cta.b64 q, [%1], %2; selp.u32 %0,1,0,q;}" : "=r"(ok) : "r"(su32(&full[st])), "r"(ph));
            acc ^= *(const uint32_t*)(smem + (size_t)st * stage_bytes + threadIdx.x * 4);
            __syncwarp();
            if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&empty[st])));
            if (++st == nstages) { st = 0; ph ^= 1; }
        }
        if (acc == 0x12345678) atomicAdd(sink, 1ull);
    }
}

int main() {
    int nsm = 0;
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
    const size_t bytes = (size_t)1 << 30;  // 1 GiB >> L2
    uint8_t* buf;
    unsigned long long* sink;
    CK(cudaMalloc(&buf, bytes));
    CK(cudaMalloc(&sink, 8));
    CK(cudaMemset(buf, 1, bytes));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    auto time_it = [&](auto fn) {
        fn(); fn();
        cudaEventRecord(e0);
        for (int i = 0; i < 5; ++i) fn();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        return bytes * 5 / (ms * 1e-3) / 1e9;
    };
    for (int bpsm : {2, 4, 8}) {
        double gb = time_it([&] { ldg_stream<<<nsm * bpsm, 512>>>((const uint4*)buf, bytes / 16, sink); });
        printf("LDG.128 %3d CTA/SM x512 thr : %7.1f GB/s\n", bpsm, gb);
    }
    CK(cudaFuncSetAttribute(tma_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    struct Cfg { int chunk, cps, nst, ctas_per_sm, threads; };
    Cfg cfgs[] = {{8192, 1, 8, 1, 288}, {8192, 3, 8, 1, 288}, {8192, 1, 24, 1, 288}, {16384, 1, 12, 1, 288},
                  {32768, 1, 6, 1, 288}, {8192, 3, 4, 2, 288}, {8192, 1, 12, 2, 160}, {4096, 1, 24, 1, 288},
                  {2048, 1, 48, 1, 288}, {8192, 1, 4, 4, 96}, {16384, 1, 3, 4, 96}};
    for (const Cfg& c : cfgs) {
        const size_t smem = (size_t)c.chunk * c.cps * c.nst + 2 * c.nst * 8;
        if (smem * c.ctas_per_sm > 227 * 1024) { printf("skip\n"); continue; }
        double gb = time_it([&] { tma_stream<<<nsm * c.ctas_per_sm, c.threads, smem>>>(buf, bytes, c.chunk, c.cps, c.nst, sink); });
        CK(cudaGetLastError());
        printf("TMA chunk %6d x%d stages %2d  %d CTA/SM (%3zu KB smem, %5zu KB in flight/SM): %7.1f GB/s\n", c.chunk, c.cps,
               c.nst, c.ctas_per_sm, smem / 1024, smem * c.ctas_per_sm / 1024, gb);
    }
    return 0;
}
