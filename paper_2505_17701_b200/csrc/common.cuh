// common.cuh -- device helpers shared by the COUNTDOWN sm_100a kernels.
//
// PTX wrappers for the Blackwell async-copy path (mbarrier + cp.async.bulk, i.e. the
// 1-D TMA engine), programmatic dependent launch (griddepcontrol), vector reductions
// into global memory, bf16 unpacking, and the two gated-MLP activations in both the
// reference's exact form (double, one rounding: numerics.cpp:47-57) and the fast f32 form.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace cdk {

constexpr int kWarp = 32;
constexpr int kVec = 8;  // elements per vector unit: 16 B of bf16 / 32 B of f32 (== kVecElems)

enum Act : int { kSilu = 0, kGeluTanh = 1 };
enum DType : int { kF32 = 0, kBF16 = 1 };

__host__ __device__ __forceinline__ int64_t imin64(int64_t a, int64_t b) { return a < b ? a : b; }

// ---------------------------------------------------------------- activations
// Reference-exact: numerics.cpp:47-57 evaluates in double and rounds once.
__device__ __forceinline__ float act_exact(int act, float x) {
    const double xd = static_cast<double>(x);
    if (act == kSilu) return static_cast<float>(xd / (1.0 + exp(-xd)));
    const double inner = 0.7978845608028653558798921198687 * (xd + 0.044715 * xd * xd * xd);
    return static_cast<float>(0.5 * xd * (1.0 + tanh(inner)));
}

// Fast path: f32 with accurate expf/tanhf (well inside the 1e-4 output tolerance).
__device__ __forceinline__ float act_fast(int act, float x) {
    if (act == kSilu) return x / (1.0f + expf(-x));
    const float inner = 0.7978845608028654f * (x + 0.044715f * x * x * x);
    return 0.5f * x * (1.0f + tanhf(inner));
}

// Tensor-core epilogues (thousands of elements per thread block): SiLU with the hardware exp2 /
// reciprocal (relative error ~1e-7, far inside the 1e-4 output bound); GeLU-tanh as act_fast.
__device__ __forceinline__ float act_epi(int act, float x) {
    if (act == kSilu) return x * __frcp_rn(1.0f + __expf(-x));
    return act_fast(act, x);
}

// ---------------------------------------------------------------- vector loads
// 8 consecutive weights -> 8 floats.  bf16: one 16-byte load; f32: two.
template <typename W> struct Vec8;

template <> struct Vec8<__nv_bfloat16> {
    __device__ __forceinline__ static void load(const __nv_bfloat16* p, float (&v)[8]) {
        const uint4 raw = *reinterpret_cast<const uint4*>(p);
        const uint32_t w[4] = {raw.x, raw.y, raw.z, raw.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            v[2 * k] = __uint_as_float(w[k] << 16);
            v[2 * k + 1] = __uint_as_float(w[k] & 0xffff0000u);
        }
    }
};

template <> struct Vec8<float> {
    __device__ __forceinline__ static void load(const float* p, float (&v)[8]) {
        const float4 a = reinterpret_cast<const float4*>(p)[0];
        const float4 b = reinterpret_cast<const float4*>(p)[1];
        v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
        v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
    }
};

__device__ __forceinline__ float to_f32(float v) { return v; }
__device__ __forceinline__ float to_f32(__nv_bfloat16 v) { return __bfloat162float(v); }

// ---------------------------------------------------------------- warp reductions
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Transpose ("halving") reduction of V partial sums held by every lane (V a power of 2, <= 32):
// each step exchanges half the remaining values with the partner lane, so V sums cost
// (V-1) + log2(32/V) shuffles instead of 5V.  Returns the full warp sum of value
// index transpose_idx<V>(lane); the 32/V lanes of a group hold the same value.
template <int V>
__device__ __forceinline__ float warp_transpose_sum(float (&v)[V]) {
    static_assert(V >= 1 && V <= 32 && (V & (V - 1)) == 0, "V must be a power of two <= 32");
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int h = V / 2, o = 16; h >= 1; h /= 2, o /= 2) {
        const bool upper = (lane & o) != 0;
#pragma unroll
        for (int i = 0; i < h; ++i) {
            const float send = upper ? v[i] : v[i + h];
            const float keep = upper ? v[i + h] : v[i];
            v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
        }
    }
    float r = v[0];
#pragma unroll
    for (int o = 16 / V; o >= 1; o /= 2) r += __shfl_xor_sync(0xffffffffu, r, o);
    return r;
}

template <int V> __device__ __forceinline__ int transpose_idx(int lane) { return lane / (32 / V); }

// Blackwell packed FP32 FMA (FFMA2): (a0, a1) += (b0, b1) * (c0, c1), two lanes of work per
// instruction.
__device__ __forceinline__ void ffma2(float& a0, float& a1, float b0, float b1, float c0, float c1) {
    asm("{\n\t.reg .b64 ra, rb, rc;\n\t"
        "mov.b64 ra, {%0, %1};\n\t"
        "mov.b64 rb, {%2, %3};\n\t"
        "mov.b64 rc, {%4, %5};\n\t"
        "fma.rn.f32x2 ra, rb, rc, ra;\n\t"
        "mov.b64 {%0, %1}, ra;\n\t}"
        : "+f"(a0), "+f"(a1)
        : "f"(b0), "f"(b1), "f"(c0), "f"(c1));
}

// ---------------------------------------------------------------- global reductions
// red.global.add.v4.f32 (sm_90+): one vector reduction instead of four scalar atomics.
__device__ __forceinline__ void red_add_v4(float* addr, float a, float b, float c, float d) {
    asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(addr), "f"(a), "f"(b),
                 "f"(c), "f"(d)
                 : "memory");
}

__device__ __forceinline__ void red_add_f32(float* addr, float a) {
    asm volatile("red.global.add.f32 [%0], %1;" ::"l"(addr), "f"(a) : "memory");
}

__device__ __forceinline__ int ld_acquire_gpu(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// ---------------------------------------------------------------- PDL
// Programmatic dependent launch: wait for the upstream grid's memory, or let the
// downstream grid start its prologue early.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// ---------------------------------------------------------------- mbarrier + bulk copy (TMA)
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    while (!mbar_try_wait(bar, parity)) {
    }
}

// 1-D bulk async copy global -> shared (TMA engine), completing on an mbarrier.
// dst, src 16-byte aligned; bytes a multiple of 16.  evict-first L2 hint: weights are
// streamed exactly once per token.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                         uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
        "[%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}

// Bulk reduction shared -> global by the TMA engine: dst[i] += src[i] (f32), whole lines at L2.
// dst, src 16-byte aligned, bytes a multiple of 16.  Completion tracked by a bulk group.
__device__ __forceinline__ void bulk_reduce_add_f32(float* dst, const float* src, uint32_t bytes) {
    asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], %2;" ::"l"(dst),
                 "r"(smem_u32(src)), "r"(bytes)
                 : "memory");
}

// Commit this thread's bulk group and wait until its shared-memory SOURCES have been read (the
// global side completes asynchronously; kernel completion publishes it).
__device__ __forceinline__ void bulk_commit_and_wait_read() {
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}

// Order this thread's generic-proxy shared-memory writes before later async-proxy (TMA) reads.
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// Bulk prefetch global -> L2 (the TMA engine; no shared memory, no completion to wait for).
// Used to start DRAM traffic for rows whose consumer is decided later.
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}

__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}

__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}

// Named barrier among `nthreads` threads (ids 1..15; 0 is __syncthreads).
__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// ---------------------------------------------------------------- timeline probe
// Compiled in only with -DCD_TIMELINE (the _lib_tl/ development build): per-CTA
// %globaltimer stamps at kernel phases, read back with cd_debug_timeline().
constexpr int kTlKernels = 8, kTlCtas = 160, kTlPhases = 8;
#ifdef CD_TIMELINE
static __device__ unsigned long long g_timeline[kTlKernels][kTlCtas][kTlPhases];
__device__ __forceinline__ void tl_stamp(int kernel, int phase) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (blockIdx.x < kTlCtas) g_timeline[kernel][blockIdx.x][phase] = t;
}
#define TL(k, p) ::cdk::tl_stamp((k), (p))
#else
#define TL(k, p) ((void)0)
#endif

}  // namespace cdk
