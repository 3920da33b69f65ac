// kernels_topm.cu -- exact top-m selection on the device (top_m_threshold, numerics.cpp:105-142).
//
// The reference orders lanes by magnitude, larger first, ties to the LOWER index, and returns
// tau = the (m+1)-th value in that order (+inf for m == 0, -inf for m == n) with the first m
// lanes alive.  Here one CTA per sample runs an MSB-first radix select over 32-bit order keys
// (4 passes of 8-bit digit histograms in shared memory) to find the (m+1)-th key T and its rank
// k among the lanes whose key equals T; a final pass marks every lane with key > T plus the
// first k - 1 lanes (by index) with key == T, using a block-wide ballot prefix count in index
// order.  The selected set and tau are exactly the reference's.
//
// Keys: magnitude order uses |v|'s bits (non-negative floats order as unsigned integers; -0 and
// +0 tie, as fabs makes them); signed order (the D-CountDown logit calibration, which thresholds
// s_hat itself) maps v to its order-preserving unsigned image.
#include <cuda_runtime.h>
#include <stdint.h>

#include <cmath>
#include <limits>

#include "common.cuh"
#include "kernels.h"
#include "launch.cuh"

namespace cdk {

namespace {

constexpr int kTopmThreads = 1024;

__device__ __forceinline__ uint32_t order_key(float v, bool signed_order) {
    const uint32_t b = __float_as_uint(v);
    if (!signed_order) return b & 0x7fffffffu;
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}

__global__ void __launch_bounds__(kTopmThreads) k_top_m(const float* __restrict__ v, int64_t n, int64_t ld, int64_t m,
                                                        int signed_order, float* __restrict__ tau_out,
                                                        uint8_t* __restrict__ mask_out, int64_t ld_mask) {
    __shared__ uint32_t hist[256];
    __shared__ uint32_t sel[2];  // [0] prefix T, [1] remaining rank k
    __shared__ uint32_t warp_cnt[kTopmThreads / 32];
    const float* vb = v + blockIdx.x * ld;
    uint8_t* mb = mask_out ? mask_out + blockIdx.x * ld_mask : nullptr;
    const bool sgn = signed_order != 0;
    pdl_wait();
    if (m <= 0 || m >= n) {
        if (threadIdx.x == 0 && tau_out)
            tau_out[blockIdx.x] = m <= 0 ? INFINITY : -INFINITY;
        if (mb)
            for (int64_t i = threadIdx.x; i < n; i += blockDim.x) mb[i] = m <= 0 ? 0 : 1;
        return;
    }
    if (threadIdx.x == 0) {
        sel[0] = 0u;
        sel[1] = static_cast<uint32_t>(m + 1);
    }
    for (int shift = 24; shift >= 0; shift -= 8) {
        for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0u;
        __syncthreads();
        const uint32_t prefix = sel[0];
        const uint32_t hi_mask = shift == 24 ? 0u : (0xffffffffu << (shift + 8));
        for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
            const uint32_t k = order_key(vb[i], sgn);
            if ((k & hi_mask) == (prefix & hi_mask)) atomicAdd(&hist[(k >> shift) & 0xffu], 1u);
        }
        __syncthreads();
        if (threadIdx.x < 32) {
            // walk the digits from the largest down: warp-parallel suffix sums over 8 digits each
            const int lane = threadIdx.x;
            uint32_t c[8], tot = 0;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                c[q] = hist[255 - (lane * 8 + q)];
                tot += c[q];
            }
            uint32_t incl = tot;  // inclusive prefix over lanes (lane 0 = largest digits)
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += t;
            }
            const uint32_t want = sel[1];
            const uint32_t excl = incl - tot;
            const bool mine = excl < want && incl >= want;
            const unsigned who = __ballot_sync(0xffffffffu, mine);
            if (mine) {
                uint32_t run = excl;
                int q = 0;
                for (; q < 8; ++q) {
                    if (run + c[q] >= want) break;
                    run += c[q];
                }
                const uint32_t digit = 255u - static_cast<uint32_t>(lane * 8 + q);
                sel[0] = prefix | (digit << shift);
                sel[1] = want - run;
            }
            (void)who;
        }
        __syncthreads();
    }
    const uint32_t T = sel[0];
    const uint32_t k_eq = sel[1];  // the (m+1)-th lane is the k_eq-th lane (by index) with key T
    if (threadIdx.x == 0 && tau_out) {
        // tau = the (m+1)-th value: |v| (magnitude order) or v (signed order) with key T
        const uint32_t b = sgn ? ((T & 0x80000000u) ? (T & 0x7fffffffu) : ~T) : T;
        tau_out[blockIdx.x] = __uint_as_float(b);
    }
    if (!mb) return;
    // lanes with key > T, plus the first k_eq - 1 lanes with key == T in index order
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int nw = blockDim.x / 32;
    uint32_t base = 0;
    for (int64_t c0 = 0; c0 < n; c0 += blockDim.x) {
        const int64_t i = c0 + threadIdx.x;
        uint32_t key = 0;
        bool eq = false;
        if (i < n) {
            key = order_key(vb[i], sgn);
            eq = key == T;
        }
        const unsigned bal = __ballot_sync(0xffffffffu, eq);
        if (lane == 0) warp_cnt[warp] = __popc(bal);
        __syncthreads();
        uint32_t before = base;
        for (int w = 0; w < warp; ++w) before += warp_cnt[w];
        before += __popc(bal & ((1u << lane) - 1u));
        uint32_t total = 0;
        for (int w = 0; w < nw; ++w) total += warp_cnt[w];
        if (i < n) mb[i] = (key > T || (eq && before < k_eq - 1)) ? 1 : 0;
        base += total;
        __syncthreads();
    }
}

}  // namespace

cudaError_t launch_top_m(const float* v, int batch, int64_t n, int64_t ld, int64_t m, bool signed_order,
                         float* tau_out, uint8_t* mask_out, int64_t ld_mask, const LaunchCfg& c) {
    if (batch <= 0 || n <= 0 || n >= (int64_t{1} << 31)) return cudaErrorInvalidValue;
    return launch_ex(k_top_m, dim3(batch), dim3(kTopmThreads), 0, c, false, v, n, ld, m, signed_order ? 1 : 0,
                     tau_out, mask_out, ld_mask);
}

}  // namespace cdk
