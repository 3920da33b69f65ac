// rec_micro.cu -- how fast can 148 SMs stream a BURST of random 24 KB neuron records (the
// D-CountDown stage 3 pattern: ~1434 active records of one layer, ~10 per SM) with TMA bulk
// copies into an 8-deep smem ring?  Compares random vs sorted record order, one layer vs 8
// rotating layers (TLB reach), record sizes, ring depth.  No compute: consumers touch one word.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/rec_micro tools/rec_micro.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <random>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1); } } while (0)

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, int n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n));
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
    asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}" ::"r"(su32(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
                 ::"r"(su32(dst)), "l"(src), "r"(bytes), "r"(su32(bar)), "l"(pol) : "memory");
}
__device__ __forceinline__ uint64_t pol_first() {
    uint64_t p; asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p)); return p;
}

// idx: per launch, G contiguous lists (list c = idx[off[c] .. off[c+1]))
__global__ void __launch_bounds__(512, 1) burst(const uint8_t* __restrict__ base, int64_t rec_bytes, int copies,
                                                const int* __restrict__ idx, const int* __restrict__ off,
                                                int nstages, unsigned* sink, unsigned long long* tw) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + rec_bytes * nstages);
    uint64_t* empty = full + nstages;
    const int nwc = blockDim.x / 32 - 1, warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    if (threadIdx.x == 0) {
        for (int s = 0; s < nstages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], nwc); }
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    unsigned long long t0;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t0));
    if (threadIdx.x == 0) atomicMin(tw, t0);
    const int b0 = off[blockIdx.x], b1 = off[blockIdx.x + 1], n = b1 - b0;
    if (warp == nwc) {
        if (lane == 0) {
            const uint64_t pol = pol_first();
            const uint32_t part = (uint32_t)(rec_bytes / copies);
            for (int e = 0; e < n; ++e) {
                const int s = e % nstages;
                if (e >= nstages) mbar_wait(&empty[s], ((e / nstages) - 1) & 1);
                mbar_expect(&full[s], (uint32_t)rec_bytes);
                const uint8_t* src = base + (int64_t)idx[b0 + e] * rec_bytes;
                for (int q = 0; q < copies; ++q) bulk_g2s(smem + s * rec_bytes + q * part, src + q * part, part, &full[s], pol);
            }
        }
    } else {
        unsigned acc = 0;
        for (int e = 0; e < n; ++e) {
            const int s = e % nstages;
            mbar_wait(&full[s], (e / nstages) & 1);
            acc += reinterpret_cast<const unsigned*>(smem + s * rec_bytes)[threadIdx.x];
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
        }
        if (acc == 0x9e3779b9u) atomicAdd(sink, 1u);
    }
    __syncthreads();
    unsigned long long t1;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t1));
    if (threadIdx.x == 0) atomicMax(tw + 1, t1);
}

// LDG variant: thread t owns 16-byte column vector t of each part (512 threads x 16 B = 8 KB =
// one 4096-element bf16 row); DEPTH records in flight per thread (registers).
template <int DEPTH>
__global__ void __launch_bounds__(512, 1) burst_ldg(const uint8_t* __restrict__ base, int64_t rec_bytes,
                                                    const int* __restrict__ idx, const int* __restrict__ off,
                                                    unsigned* sink, unsigned long long* tw) {
    __syncthreads();
    unsigned long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    if (threadIdx.x == 0) atomicMin(tw, t0);
    const int b0 = off[blockIdx.x], b1 = off[blockIdx.x + 1], n = b1 - b0;
    const int64_t row = rec_bytes / 3;
    unsigned acc = 0;
    uint4 v[DEPTH][3];
    auto load = [&](int e, uint4 (&d)[3]) {
        const uint8_t* src = base + (int64_t)idx[b0 + e] * rec_bytes + threadIdx.x * 16;
#pragma unroll
        for (int q = 0; q < 3; ++q) d[q] = __ldcs(reinterpret_cast<const uint4*>(src + q * row));
    };
#pragma unroll
    for (int k = 0; k < DEPTH; ++k)
        if (k < n) load(k, v[k]);
    for (int e = 0; e < n; e += DEPTH) {
#pragma unroll
        for (int k = 0; k < DEPTH; ++k) {
            if (e + k < n) {
                acc += v[k][0].x ^ v[k][1].y ^ v[k][2].z;
                if (e + k + DEPTH < n) load(e + k + DEPTH, v[k]);
            }
        }
    }
    if (acc == 0x9e3779b9u) atomicAdd(sink, 1u);
    __syncthreads();
    unsigned long long t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    if (threadIdx.x == 0) atomicMax(tw + 1, t1);
}

// issue cost: lane 0 issues N bulk copies of `bytes` into distinct smem slots (clock64 around the
// issue loop), then waits for all
__global__ void issue_probe(const uint8_t* __restrict__ base, int n, uint32_t bytes, long long* out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 200 * 1024);
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;");
        const uint64_t pol = pol_first();
        mbar_expect(bar, n * bytes);
        const long long c0 = clock64();
        for (int i = 0; i < n; ++i)
            bulk_g2s(smem + (i * bytes) % (192 * 1024), base + (((int64_t)blockIdx.x * 977 + i * 131) % 14336) * 24576, bytes, bar, pol);
        const long long c1 = clock64();
        mbar_wait(bar, 0);
        const long long c2 = clock64();
        if (blockIdx.x == 0) { out[0] = c1 - c0; out[1] = c2 - c0; }
    }
}

int main() {
    const int G = 148, F = 14336, active = 1434, NLmax = 8;
    const int64_t rec = 3 * 4096 * 2;
    uint8_t* w;
    CK(cudaMalloc(&w, (size_t)NLmax * F * rec));
    CK(cudaMemset(w, 1, (size_t)NLmax * F * rec));
    unsigned* sink;
    CK(cudaMalloc(&sink, 4));
    unsigned long long* tw;
    const int NT = 8 * 64 + 64;
    CK(cudaMalloc(&tw, 16 * NT));
    std::vector<unsigned long long> th(2 * NT);
    auto reset = [&]() { for (int i = 0; i < NT; ++i) { th[2 * i] = ~0ull; th[2 * i + 1] = 0; }
                         CK(cudaMemcpy(tw, th.data(), 16 * NT, cudaMemcpyHostToDevice)); };
    auto inner = [&](int n) { CK(cudaMemcpy(th.data(), tw, 16 * NT, cudaMemcpyDeviceToHost));
                              std::vector<double> v; for (int i = 0; i < n; ++i) v.push_back((th[2*i+1] - th[2*i]) / 1e3);
                              std::sort(v.begin(), v.end()); return v[v.size() / 2]; };
    const int NI = 64;  // distinct launches (index sets)
    int *d_idx, *d_off;
    CK(cudaMalloc(&d_idx, sizeof(int) * active * NI));
    CK(cudaMalloc(&d_off, sizeof(int) * (G + 1) * NI));
    cudaStream_t st;
    CK(cudaStreamCreate(&st));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    std::mt19937 rng(7);
    {
        std::vector<int> z((G + 1) * NI, 0);
        CK(cudaMemcpy(d_off, z.data(), sizeof(int) * z.size(), cudaMemcpyHostToDevice));
        const size_t smem = rec * 8 + 1024;
        CK(cudaFuncSetAttribute(burst, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        for (int l = 0; l < NI; ++l) burst<<<G, 512, smem, st>>>(w, rec, 1, d_idx, d_off, 8, sink, tw);
        reset();
        CK(cudaEventRecord(e0, st));
        for (int l = 0; l < 8 * NI; ++l) burst<<<G, 512, smem, st>>>(w, rec, 1, d_idx, d_off, 8, sink, tw + 2 * l);
        CK(cudaEventRecord(e1, st));
        CK(cudaStreamSynchronize(st));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        printf("empty launch: %.2f us (inside: %.2f us)\n", 1e3 * ms / (8 * NI), inner(8 * NI));
    }
    {
        long long* d_out;
        CK(cudaMalloc(&d_out, 16));
        CK(cudaFuncSetAttribute(issue_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 201 * 1024));
        for (int n : {1, 8, 16})
            for (uint32_t by : {4096u, 8192u, 24576u}) {
                long long h[2] = {0, 0};
                for (int rep = 0; rep < 3; ++rep) issue_probe<<<G, 32, 201 * 1024, st>>>(w, n, by, d_out);
                CK(cudaMemcpy(h, d_out, 16, cudaMemcpyDeviceToHost));
                printf("issue probe: %2d copies x %5u B: issue %lld cycles (%.0f / copy), all landed after %lld cycles\n",
                       n, by, h[0], (double)h[0] / n, h[1]);
            }
    }
    for (int NL : {1, 8})
        for (int sorted : {0, 1})
            for (int nst : {4, 8})
                for (int copies : {1, 2}) {
                    std::vector<int> idx(active * NI), off((G + 1) * NI);
                    for (int l = 0; l < NI; ++l) {
                        std::vector<int> perm(F);
                        for (int i = 0; i < F; ++i) perm[i] = i;
                        std::shuffle(perm.begin(), perm.end(), rng);
                        std::vector<int> a(perm.begin(), perm.begin() + active);
                        if (sorted) std::sort(a.begin(), a.end());
                        const int layer = l % NL;
                        for (int i = 0; i < active; ++i) idx[l * active + i] = a[i] + layer * F;
                        for (int c = 0; c <= G; ++c) off[l * (G + 1) + c] = l * active + (int)((int64_t)c * active / G);
                    }
                    CK(cudaMemcpy(d_idx, idx.data(), sizeof(int) * idx.size(), cudaMemcpyHostToDevice));
                    CK(cudaMemcpy(d_off, off.data(), sizeof(int) * off.size(), cudaMemcpyHostToDevice));
                    const size_t smem = rec * nst + 1024;
                    CK(cudaFuncSetAttribute(burst, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
                    for (int l = 0; l < NI; ++l)
                        burst<<<G, 512, smem, st>>>(w, rec, copies, d_idx, d_off + l * (G + 1), nst, sink, tw);
                    CK(cudaStreamSynchronize(st));
                    reset();
                    const int reps = 8;
                    CK(cudaEventRecord(e0, st));
                    for (int r = 0; r < reps; ++r)
                        for (int l = 0; l < NI; ++l)
                            burst<<<G, 512, smem, st>>>(w, rec, copies, d_idx, d_off + l * (G + 1), nst, sink, tw + 2 * (r * NI + l));
                    CK(cudaEventRecord(e1, st));
                    CK(cudaStreamSynchronize(st));
                    float ms;
                    CK(cudaEventElapsedTime(&ms, e0, e1));
                    const double us = 1e3 * ms / (reps * NI);
                    const double in = inner(reps * NI);
                    printf("layers=%d sorted=%d stages=%d copies/rec=%d: %.2f us per launch, %.2f us inside (first CTA start to last CTA end) = %.0f GB/s\n",
                           NL, sorted, nst, copies, us, in, active * rec / in / 1e3);
                }
    for (int NL : {1, 8})
        for (int depth : {2, 4, 8}) {
            std::vector<int> idx(active * NI), off((G + 1) * NI);
            for (int l = 0; l < NI; ++l) {
                std::vector<int> perm(F);
                for (int i = 0; i < F; ++i) perm[i] = i;
                std::shuffle(perm.begin(), perm.end(), rng);
                const int layer = l % NL;
                for (int i = 0; i < active; ++i) idx[l * active + i] = perm[i] + layer * F;
                for (int c = 0; c <= G; ++c) off[l * (G + 1) + c] = l * active + (int)((int64_t)c * active / G);
            }
            CK(cudaMemcpy(d_idx, idx.data(), sizeof(int) * idx.size(), cudaMemcpyHostToDevice));
            CK(cudaMemcpy(d_off, off.data(), sizeof(int) * off.size(), cudaMemcpyHostToDevice));
            auto fn = depth == 2 ? burst_ldg<2> : depth == 4 ? burst_ldg<4> : burst_ldg<8>;
            for (int l = 0; l < NI; ++l) fn<<<G, 512, 0, st>>>(w, rec, d_idx, d_off + l * (G + 1), sink, tw);
            CK(cudaStreamSynchronize(st));
            reset();
            const int reps = 8;
            for (int r = 0; r < reps; ++r)
                for (int l = 0; l < NI; ++l) fn<<<G, 512, 0, st>>>(w, rec, d_idx, d_off + l * (G + 1), sink, tw + 2 * (r * NI + l));
            CK(cudaStreamSynchronize(st));
            const double in = inner(reps * NI);
            printf("LDG layers=%d depth=%d: %.2f us inside = %.0f GB/s\n", NL, depth, in, active * rec / in / 1e3);
        }
    return 0;
}
