// fused_common.cuh -- inter-CTA exchange helpers of the persistent fused decode kernels
// (kernels_fused.cu: D-CountDown, kernels_fused_mc.cu: M-CountDown).
//
// CTAs exchange data through EPOCH-TAGGED 64-bit words {payload, launch tag} written with one
// single-copy-atomic store; readers spin until the tag matches.  No fence sits on the critical
// path, so no CTA waits for its own in-flight bulk copies (a release fence does).  The launch
// tag lives in Scratch::ctl[kCtlEpoch]; the work-queue counters of a launch are the 4 words at
// ctl[kCtlQueue + (tag % 3) * 32].
#pragma once

#include <stdint.h>

namespace cdk {
namespace fused {

constexpr int kCtlEpoch = 0;    // ctl word: launch tag of the last completed launch
constexpr int kCtlQueue = 32;   // ctl words: 3 x 32 (launch tag % 3) work-queue counters
constexpr int kYZeroWord = 1023;  // t_count word: "y zeroed" flag of the launch


__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ unsigned ld_relaxed_u32(const unsigned* p) {
    unsigned v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void red_add_u32(unsigned* p, unsigned v) {
    asm volatile("red.relaxed.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ void st_relaxed_u64(unsigned long long* p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// A 16-byte streaming load the compiler may not sink towards its use (volatile asm keeps it
// ahead of griddepcontrol.wait, so its DRAM latency overlaps the previous grid's tail).
__device__ __forceinline__ uint4 ldg_early_v4(const void* p) {
    uint4 v;
    asm volatile("ld.global.cs.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p));
    return v;
}

// 8 consecutive f32 (an activation 8-vector) bypassing L1: one 256-bit load (LDG.256) when the
// vector is whole and 32-byte aligned -- a warp's request is then 1 KB of consecutive sectors
// instead of two half-efficient 16-byte passes -- else per-float4 loads of what lies below `avail`
__device__ __forceinline__ void ldcg_x8(const float* p, int64_t avail, float4& lo, float4& hi) {
    if (avail >= 8 && (reinterpret_cast<uintptr_t>(p) & 31u) == 0) {
        asm volatile("ld.global.cg.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                     : "=f"(lo.x), "=f"(lo.y), "=f"(lo.z), "=f"(lo.w), "=f"(hi.x), "=f"(hi.y), "=f"(hi.z), "=f"(hi.w)
                     : "l"(p));
        return;
    }
    const float4* src = reinterpret_cast<const float4*>(p);
    if (avail > 0) lo = __ldcg(src);
    if (avail > 4) hi = __ldcg(src + 1);
}

// Column sums of nw warp partials part[w * stride + v], v < V (V a power of two <= 32), by one
// whole warp: lane group g = lane / V adds warps g, g + 32/V, ..., then an xor butterfly over the
// groups -- every lane returns the total of column lane % V (a few shuffles instead of an
// nw-long chain of dependent shared loads)
template <int V>
__device__ __forceinline__ float sum_partials(const float* part, int stride, int nw, int lane) {
    static_assert(V >= 1 && V <= 32 && (V & (V - 1)) == 0, "V must be a power of two <= 32");
    constexpr int kG = 32 / V;
    const int v = lane % V;
    float s = 0.0f;
    for (int w = lane / V; w < nw; w += kG) s += part[w * stride + v];
#pragma unroll
    for (int o = V; o < 32; o <<= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    return s;
}

__device__ __forceinline__ unsigned long long tagged(uint32_t tag, uint32_t payload) {
    return (static_cast<unsigned long long>(tag) << 32) | payload;
}

// Spin until the word carries `tag`; return its payload.
__device__ __forceinline__ uint32_t await_relaxed(const unsigned long long* p, uint32_t tag) {
    unsigned long long w;
    do {
        w = ld_relaxed_u64(p);
    } while (static_cast<uint32_t>(w >> 32) != tag);
    return static_cast<uint32_t>(w);
}

__device__ __forceinline__ uint32_t await_acquire(const unsigned long long* p, uint32_t tag) {
    unsigned long long w;
    do {
        w = ld_acquire_u64(p);
    } while (static_cast<uint32_t>(w >> 32) != tag);
    return static_cast<uint32_t>(w);
}

__device__ __forceinline__ void named_bar_arrive(int id, int nthreads) {
    asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}


}  // namespace fused
}  // namespace cdk
