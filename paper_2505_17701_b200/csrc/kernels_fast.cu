// kernels_fast.cu -- the COUNTDOWN decode hot path for sm_100a (UnorderedAccumulate semantics).
//
// Kernel chain per token batch (PDL-chained, graph-capturable, no host round trips):
//   D-CountDown (Alg. 3; pipeline_dc blocked_exec.cpp:350-379):
//     k_latent_fast        latent = x theta_a                        (predictor.cpp:94-102)
//     k_indicator_dc       s_hat_i = latent . theta_bt[i]; s_hat > tau; compaction
//                                                                     (predictor.cpp:104-113,140-148)
//     k_sparse<DC>         s_i = (W_up[i].x) act(W_gate[i].x); y += s_i W_down[i]
//                                                                     (exec_dc blocked_exec.cpp:252-289)
//   M-CountDown (Alg. 2; pipeline_mc blocked_exec.cpp:316-328):
//     k_indicator_mc       u_i = W_up[i].x; |u| > tau; compaction    (blocked_exec.cpp:300-314)
//     k_sparse<MC>         s_i = act(W_gate[i].x) u_i; y += s_i W_down[i]
//                                                                     (exec_mc blocked_exec.cpp:174-212)
// All weight rows are streamed HBM -> shared memory by the TMA bulk-copy engine into an
// mbarrier ring (one producer warp, one elected lane), consumed by column-owning warps;
// y lives in registers and is reduced once per CTA with red.global.add.v4.f32.
#include "common.cuh"
#include "kernels.h"
#include "launch.cuh"

namespace cdk {

namespace {

constexpr int kStageBytesTarget = 32 * 1024;
constexpr int kMC_ = kMC, kDC_ = kDC, kCATS_ = kCATS;  // Method ids usable where kMC is shadowed
constexpr int kSmemBudget = 200 * 1024;

__device__ __forceinline__ int64_t ldcg_i64(const int64_t* p) { return __ldcg(p); }

// ============================================================================ zero
__global__ void k_zero(float* __restrict__ p, int64_t n) {
    pdl_launch_dependents();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        p[i] = 0.0f;
}

// ============================================================================ spin
// Keeps the stream busy for `ns` nanoseconds (stage timing: the host enqueues the timed work
// while this runs, so CUDA events measure device time, not host launch latency).
__global__ void k_spin(unsigned long long ns) {
    unsigned long long t0, t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    do {
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    } while (t - t0 < ns);
}

// ============================================================================ latent
// latent[b][q] += sum_{i in this CTA's rows} x[b][i] * theta_a[i][q]; reduced in smem then one
// vector reduction per column group per CTA.  theta_a rows are read once, coalesced.
template <typename W, int NB>
__global__ void __launch_bounds__(256) k_latent_fast(LayerDev L, const float* __restrict__ x,
                                                     float* __restrict__ latent,
                                                     int rows_per_cta) {
    if (threadIdx.x == 0) TL(0, 0);
    pdl_launch_dependents();
    __shared__ float red[NB * 2048];
    const int nvr = static_cast<int>(L.ldr / kVec);
    const int rpp = 256 / nvr;  // rows per pass
    const int t = threadIdx.x;
    const int cv = t % nvr, rg = t / nvr;
    const int64_t row0 = (int64_t)blockIdx.x * rows_per_cta;
    const int64_t row1 = imin64(L.d, row0 + rows_per_cta);
    const W* A = static_cast<const W*>(L.theta_a);

    float acc[NB][8];
#pragma unroll
    for (int b = 0; b < NB; ++b)
#pragma unroll
        for (int k = 0; k < 8; ++k) acc[b][k] = 0.0f;

    if (rg < rpp) {
#pragma unroll 4
        for (int64_t i = row0 + rg; i < row1; i += rpp) {
            float w[8];
            Vec8<W>::load(A + i * L.ldr + cv * kVec, w);
#pragma unroll
            for (int b = 0; b < NB; ++b) {
                const float xb = __ldg(x + b * L.d + i);
#pragma unroll
                for (int k = 0; k < 8; ++k) acc[b][k] = fmaf(xb, w[k], acc[b][k]);
            }
        }
#pragma unroll
        for (int b = 0; b < NB; ++b)
#pragma unroll
            for (int k = 0; k < 8; ++k) red[(b * rpp + rg) * (nvr * kVec) + cv * kVec + k] = acc[b][k];
    }
    __syncthreads();
    for (int c = t; c < nvr * 2; c += blockDim.x) {  // c indexes 4-float groups
        for (int b = 0; b < NB; ++b) {
            float s[4] = {0.f, 0.f, 0.f, 0.f};
            for (int g = 0; g < rpp; ++g)
#pragma unroll
                for (int k = 0; k < 4; ++k) s[k] += red[(b * rpp + g) * (nvr * kVec) + c * 4 + k];
            red_add_v4(latent + b * L.ldr + c * 4, s[0], s[1], s[2], s[3]);
        }
    }
    if (threadIdx.x == 0) TL(0, 1);
}

// ============================================================================ DC indicator
// One CTA per SM owns a contiguous chunk of neurons; its theta_bt rows (contiguous bytes)
// are streamed by the TMA engine while the latent is still being produced upstream (PDL).
template <typename W, int NB, int VPL>
__global__ void k_indicator_dc(LayerDev L, Scratch S, int nb, int rows_per_cta, int stage_rows,
                               int nstages, float tau, const uint8_t* __restrict__ ovr,
                               float* __restrict__ y, int64_t y_len, uint8_t* __restrict__ mask_out,
                               float* __restrict__ logits_out) {
    if (threadIdx.x == 0) TL(1, 0);
    pdl_launch_dependents();
    extern __shared__ __align__(1024) uint8_t smem[];
    const int nwc = blockDim.x / kWarp - 1;  // consumer warps
    const int warp = threadIdx.x / kWarp, lane = threadIdx.x % kWarp;
    const int64_t row_bytes = L.ldr * (int64_t)sizeof(W);
    const int64_t stage_bytes = row_bytes * stage_rows;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + stage_bytes * nstages);
    uint64_t* empty = full + nstages;
    int32_t* l_idx = reinterpret_cast<int32_t*>(empty + nstages);
    uint32_t* l_bits = reinterpret_cast<uint32_t*>(l_idx + rows_per_cta);
    int* n_local = reinterpret_cast<int*>(l_bits + rows_per_cta);
    int* alive_local = n_local + 1;
    float* wscratch = reinterpret_cast<float*>(alive_local + kMaxBatchFast);  // [nwc][kRB*NB]
    constexpr int kRB = 4;

    const int64_t c0 = (int64_t)blockIdx.x * rows_per_cta;
    const int64_t c1 = imin64(L.F, c0 + rows_per_cta);
    const int nrows = c1 > c0 ? static_cast<int>(c1 - c0) : 0;
    const int nst = (nrows + stage_rows - 1) / stage_rows;

    if (threadIdx.x == 0) {
        for (int s = 0; s < nstages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], nwc);
        }
        *n_local = 0;
        for (int b = 0; b < NB; ++b) alive_local[b] = 0;
        fence_mbar_init();
    }
    // y is accumulated by the downstream sparse kernel: zero it here.
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < y_len;
         i += (int64_t)gridDim.x * blockDim.x)
        y[i] = 0.0f;
    __syncthreads();

    const W* BT = static_cast<const W*>(L.theta_bt);
    if (warp == nwc) {
        // ---- producer: theta_bt does not depend on the latent, start streaming now.
        if (lane == 0) {
            const uint64_t pol = policy_evict_first();
            int st = 0;
            uint32_t ph = 0;
            for (int s = 0; s < nst; ++s) {
                const int64_t r0 = c0 + (int64_t)s * stage_rows;
                const int n = static_cast<int>(imin64(stage_rows, c1 - r0));
                mbar_wait(&empty[st], ph ^ 1);
                mbar_arrive_expect_tx(&full[st], static_cast<uint32_t>(n * row_bytes));
                bulk_g2s(smem + st * stage_bytes, BT + r0 * L.ldr, static_cast<uint32_t>(n * row_bytes),
                         &full[st], pol);
                if (++st == nstages) { st = 0; ph ^= 1; }
            }
        }
    } else {
        // ---- consumers: one warp per predictor row, latent held in registers.
        if (threadIdx.x == 0) TL(1, 1);
        pdl_wait();
        if (threadIdx.x == 0) TL(1, 2);
        const int nvr = static_cast<int>(L.ldr / kVec);
        float lat[NB][VPL][8];
#pragma unroll
        for (int v = 0; v < VPL; ++v) {
            const int vec = lane + v * kWarp;
#pragma unroll
            for (int b = 0; b < NB; ++b) {
                float4 lo = make_float4(0.f, 0.f, 0.f, 0.f), hi = lo;
                if (vec < nvr && b < nb) {
                    const float4* src = reinterpret_cast<const float4*>(S.latent + b * L.ldr + vec * kVec);
                    lo = __ldcg(src);
                    hi = __ldcg(src + 1);
                }
                lat[b][v][0] = lo.x; lat[b][v][1] = lo.y; lat[b][v][2] = lo.z; lat[b][v][3] = lo.w;
                lat[b][v][4] = hi.x; lat[b][v][5] = hi.y; lat[b][v][6] = hi.z; lat[b][v][7] = hi.w;
            }
        }
        if (threadIdx.x == 0) TL(1, 3);
        // Each warp takes kRB consecutive rows at a time: packed FFMA2 dot products, one
        // halving (transpose) shuffle reduction for all kRB x NB sums, then lanes 0..kRB-1
        // own one row each for thresholding and ballot compaction (one shared atomic per
        // kRB rows).
        int st = 0;
        uint32_t ph = 0;
        for (int s = 0; s < nst; ++s) {
            const int64_t r0 = c0 + (int64_t)s * stage_rows;
            const int n = static_cast<int>(imin64(stage_rows, c1 - r0));
            mbar_wait(&full[st], ph);
            if (threadIdx.x == 0 && s == 0) TL(1, 4);
            const W* base = reinterpret_cast<const W*>(smem + st * stage_bytes);
            for (int rr0 = warp * kRB; rr0 < n; rr0 += nwc * kRB) {
                constexpr int kV = kRB * NB;
                float v[kV];
#pragma unroll
                for (int j = 0; j < kRB; ++j) {
                    float w[VPL][8];
#pragma unroll
                    for (int q = 0; q < VPL; ++q) {
                        const int vec = lane + q * kWarp;
                        if (rr0 + j < n && vec < nvr) Vec8<W>::load(base + (rr0 + j) * L.ldr + vec * kVec, w[q]);
                        else
#pragma unroll
                            for (int k = 0; k < 8; ++k) w[q][k] = 0.0f;
                    }
#pragma unroll
                    for (int b = 0; b < NB; ++b) {
                        float a0 = 0.0f, a1 = 0.0f;
#pragma unroll
                        for (int q = 0; q < VPL; ++q)
#pragma unroll
                            for (int k = 0; k < 8; k += 2) ffma2(a0, a1, w[q][k], w[q][k + 1], lat[b][q][k], lat[b][q][k + 1]);
                        v[j * NB + b] = a0 + a1;
                    }
                }
                const float tot = warp_transpose_sum<kV>(v);
                // lanes g*(32/kV) hold value index g = row j * NB + sample b
                if ((lane % (32 / kV)) == 0) wscratch[warp * kV + lane / (32 / kV)] = tot;
                __syncwarp();
                const bool valid = lane < kRB && rr0 + lane < n;
                const int64_t gi = r0 + rr0 + lane;
                uint32_t bits = 0;
#pragma unroll
                for (int b = 0; b < NB; ++b) {
                    bool a = false;
                    if (valid && b < nb) {
                        const float z = wscratch[warp * kV + lane * NB + b];
                        a = ovr ? (ovr[b * L.F + gi] != 0) : (z > tau);
                        if (mask_out) mask_out[b * L.F + gi] = a ? 1 : 0;
                        if (logits_out) logits_out[b * L.F + gi] = z;
                    }
                    bits |= static_cast<uint32_t>(a) << b;
                    const unsigned bal = __ballot_sync(0xffffffffu, a);
                    if (lane == 0 && bal) atomicAdd(&alive_local[b], __popc(bal));
                }
                __syncwarp();
                const unsigned any = __ballot_sync(0xffffffffu, bits != 0);
                int e0 = 0;
                if (lane == 0 && any) e0 = atomicAdd(n_local, __popc(any));
                e0 = __shfl_sync(0xffffffffu, e0, 0);
                if (bits) {
                    const int e = e0 + __popc(any & ((1u << lane) - 1u));
                    l_idx[e] = static_cast<int32_t>(gi);
                    l_bits[e] = bits;
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[st]);
            if (++st == nstages) { st = 0; ph ^= 1; }
        }
    }
    if (threadIdx.x == 0) TL(1, 5);
    __syncthreads();
    __shared__ int base_s;
    if (threadIdx.x == 0) {
        base_s = atomicAdd(S.count, *n_local);
        for (int b = 0; b < NB; ++b)
            if (alive_local[b]) atomicAdd(S.alive + b, alive_local[b]);
    }
    __syncthreads();
    for (int e = threadIdx.x; e < *n_local; e += blockDim.x) {
        S.list[base_s + e] = l_idx[e];
        S.bits[base_s + e] = l_bits[e];
    }
    if (threadIdx.x == 0) TL(1, 6);
}

// ============================================================================ MC indicator
// Column ownership: consumer thread ct owns vectors ct + j*NC (j < VPT) of every row, with x
// in registers; a stage holds kSR consecutive W_up rows (one bulk copy).
constexpr int kSR = 4;

template <typename W, int NB, int VPT, bool kCats>
__global__ void __launch_bounds__(416, 1) k_indicator_mc(LayerDev L, Scratch S, int nb, const float* __restrict__ x,
                               int rows_per_cta, int nstages, float tau, float* __restrict__ y,
                               int64_t y_len, uint8_t* __restrict__ mask_out,
                               float* __restrict__ u_out) {
    if (threadIdx.x == 0) TL(4, 0);
    pdl_launch_dependents();
    extern __shared__ __align__(1024) uint8_t smem[];
    const int nwc = blockDim.x / kWarp - 1;
    const int nc = nwc * kWarp;
    const int warp = threadIdx.x / kWarp, lane = threadIdx.x % kWarp;
    const int nvec = static_cast<int>(L.ld / kVec);
    const int64_t row_bytes = L.ld * (int64_t)sizeof(W);
    const int64_t stage_bytes = row_bytes * kSR;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + stage_bytes * nstages);
    uint64_t* empty = full + nstages;
    float* red = reinterpret_cast<float*>(empty + nstages);  // [2][nwc][kSR*NB] partial sums
    int32_t* l_idx = reinterpret_cast<int32_t*>(red + 2 * nwc * kSR * NB);
    uint32_t* l_bits = reinterpret_cast<uint32_t*>(l_idx + rows_per_cta);
    float* l_val = reinterpret_cast<float*>(l_bits + rows_per_cta);  // [rows_per_cta][NB]
    int* n_local = reinterpret_cast<int*>(l_val + rows_per_cta * NB);
    int* alive_local = n_local + 1;

    const int64_t c0 = (int64_t)blockIdx.x * rows_per_cta;
    const int64_t c1 = imin64(L.F, c0 + rows_per_cta);
    const int nrows = c1 > c0 ? static_cast<int>(c1 - c0) : 0;
    const int nst = (nrows + kSR - 1) / kSR;

    if (threadIdx.x == 0) {
        for (int s = 0; s < nstages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], nwc);
        }
        *n_local = 0;
        for (int b = 0; b < NB; ++b) alive_local[b] = 0;
        fence_mbar_init();
    }
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < y_len;
         i += (int64_t)gridDim.x * blockDim.x)
        y[i] = 0.0f;
    __syncthreads();

    // M-CountDown thresholds u = W_up x; CATS (pipeline_cats blocked_exec.cpp:330-348)
    // thresholds h = act(W_gate x) and keeps h for the up-row phase.
    const W* U = static_cast<const W*>(kCats ? L.w_gate : L.w_up);
    if (warp == nwc) {
        if (lane == 0) {
            const uint64_t pol = policy_evict_first();
            int st = 0;
            uint32_t ph = 0;
            for (int s = 0; s < nst; ++s) {
                const int64_t r0 = c0 + (int64_t)s * kSR;
                const int n = static_cast<int>(imin64(kSR, c1 - r0));
                mbar_wait(&empty[st], ph ^ 1);
                mbar_arrive_expect_tx(&full[st], static_cast<uint32_t>(n * row_bytes));
                for (int q = 0; q < n; ++q)
                    bulk_g2s(smem + st * stage_bytes + q * row_bytes, U + (r0 + q) * L.rs,
                             static_cast<uint32_t>(row_bytes), &full[st], pol);
                if (++st == nstages) { st = 0; ph ^= 1; }
            }
        }
    } else {
        const int ct = threadIdx.x;
        float xr[NB][VPT][8];
#pragma unroll
        for (int j = 0; j < VPT; ++j) {
            const int vec = ct + j * nc;
#pragma unroll
            for (int b = 0; b < NB; ++b)
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const int64_t col = (int64_t)vec * kVec + k;
                    xr[b][j][k] = (vec < nvec && col < L.d && b < nb) ? __ldg(x + b * L.d + col) : 0.0f;
                }
        }
        int st = 0;
        uint32_t ph = 0;
        for (int s = 0; s < nst; ++s) {
            const int64_t r0 = c0 + (int64_t)s * kSR;
            const int n = static_cast<int>(imin64(kSR, c1 - r0));
            mbar_wait(&full[st], ph);
            const W* base = reinterpret_cast<const W*>(smem + st * stage_bytes);
            constexpr int kV = kSR * NB;
            float v[kV];
#pragma unroll
            for (int rr = 0; rr < kSR; ++rr) {
                float a0[NB], a1[NB];
#pragma unroll
                for (int b = 0; b < NB; ++b) a0[b] = a1[b] = 0.0f;
                if (rr < n) {
#pragma unroll
                    for (int j = 0; j < VPT; ++j) {
                        const int vec = ct + j * nc;
                        if (vec < nvec) {
                            float w[8];
                            Vec8<W>::load(base + rr * L.ld + vec * kVec, w);
#pragma unroll
                            for (int b = 0; b < NB; ++b)
#pragma unroll
                                for (int k = 0; k < 8; k += 2) ffma2(a0[b], a1[b], w[k], w[k + 1], xr[b][j][k], xr[b][j][k + 1]);
                        }
                    }
                }
#pragma unroll
                for (int b = 0; b < NB; ++b) v[rr * NB + b] = a0[b] + a1[b];
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[st]);  // stage data consumed
            const float tot = warp_transpose_sum<kV>(v);
            float* rb = red + (s & 1) * nwc * kV;
            if ((lane % (32 / kV)) == 0) rb[warp * kV + lane / (32 / kV)] = tot;
            named_bar_sync(1, nc);
            if (warp == 0) {
                const bool valid = lane < n;
                const int64_t gi = r0 + lane;
                uint32_t bits = 0;
                float uv[NB];
#pragma unroll
                for (int b = 0; b < NB; ++b) {
                    float u = 0.0f;
                    if (valid)
                        for (int w = 0; w < nwc; ++w) u += rb[w * kV + lane * NB + b];
                    if (kCats) u = act_fast(L.act, u);
                    uv[b] = u;
                    bool a = false;
                    if (valid && b < nb) {
                        a = fabsf(u) > tau;
                        if (mask_out) mask_out[b * L.F + gi] = a ? 1 : 0;
                        if (u_out) u_out[b * L.F + gi] = u;
                    }
                    bits |= static_cast<uint32_t>(a) << b;
                    const unsigned bal = __ballot_sync(0xffffffffu, a);
                    if (lane == 0 && bal) atomicAdd(&alive_local[b], __popc(bal));
                }
                const unsigned any = __ballot_sync(0xffffffffu, bits != 0);
                int e0 = 0;
                if (lane == 0 && any) e0 = atomicAdd(n_local, __popc(any));
                e0 = __shfl_sync(0xffffffffu, e0, 0);
                if (bits) {
                    const int e = e0 + __popc(any & ((1u << lane) - 1u));
                    l_idx[e] = static_cast<int32_t>(gi);
                    l_bits[e] = bits;
#pragma unroll
                    for (int b = 0; b < NB; ++b) l_val[e * NB + b] = ((bits >> b) & 1u) ? uv[b] : 0.0f;
                }
            }
            if (++st == nstages) { st = 0; ph ^= 1; }
        }
    }
    __syncthreads();
    __shared__ int base_s;
    if (threadIdx.x == 0) {
        base_s = atomicAdd(S.count, *n_local);
        for (int b = 0; b < NB; ++b)
            if (alive_local[b]) atomicAdd(S.alive + b, alive_local[b]);
    }
    __syncthreads();
    for (int e = threadIdx.x; e < *n_local; e += blockDim.x) {
        S.list[base_s + e] = l_idx[e];
        S.bits[base_s + e] = l_bits[e];
#pragma unroll
        for (int b = 0; b < NB; ++b) S.list_val[(int64_t)(base_s + e) * kMaxBatchFast + b] = l_val[e * NB + b];
    }
    if (threadIdx.x == 0) TL(4, 6);
}

// ============================================================================ sparse FFN
// Persistent CTAs take list slots blockIdx.x, blockIdx.x + G, ...  Per slot the producer
// warp bulk-copies the neuron's (up,) gate and down rows -- each one contiguous run -- into a
// ring stage; consumers (column owners) reduce the dot products across the CTA, apply the
// activation and accumulate s * W_down[i] into register-resident y.
constexpr int kGroup = 4;  // neurons per reduction round in k_sparse

struct SlotMeta {
    int32_t idx;
    uint32_t bits;
    float u[kMaxBatchFast];
};

// KIND: kDC  s = (W_up[i].x) act(W_gate[i].x)           copies [up|gate|down]
//       kMC  s = act(W_gate[i].x) u_i (u from the list)   copies [gate|down]
//       kCATS s = (W_up[i].x) h_i (h = act(gate) from the list) copies [up|gate|down] (the gate
//             row rides along unused: CATS is a comparison baseline, not the hot path)
template <typename W, int NB, int VPT, int KIND>
__global__ void __launch_bounds__(416, 1) k_sparse(LayerDev L, Scratch S, int nb, const float* __restrict__ x, int nstages,
                         bool dense, float* __restrict__ y, int* __restrict__ alive_out) {
    constexpr bool kMC = KIND == kMC_;
    constexpr bool kOneDot = KIND != kDC_;    // one dot product per neuron (MC, CATS)
    constexpr bool kListU = KIND != kDC_;     // per-sample factor comes from the list
    constexpr int kTl = kMC ? 3 : 2;
    if (threadIdx.x == 0) TL(kTl, 0);
    extern __shared__ __align__(1024) uint8_t smem[];
    constexpr int kRows = kMC ? 2 : 3;  // rows per neuron copied: (up,) gate, down
    constexpr int kDotRow = KIND == kDC_ ? 1 : 0;   // row of the (first) dot: DC gate, MC gate, CATS up
    constexpr int kDownRow = kMC ? 1 : 2;
    const int nwc = blockDim.x / kWarp - 1;
    const int nc = nwc * kWarp;
    const int warp = threadIdx.x / kWarp, lane = threadIdx.x % kWarp;
    const int nvec = static_cast<int>(L.ld / kVec);
    const int64_t row_bytes = L.ld * (int64_t)sizeof(W);
    const int64_t stage_bytes = row_bytes * kRows;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + stage_bytes * nstages);
    uint64_t* empty = full + nstages;
    SlotMeta* meta = reinterpret_cast<SlotMeta*>(empty + nstages);
    float* red = reinterpret_cast<float*>(meta + nstages);  // [nwc][kGroup * 2 * NB] warp sums
    float* sval = red + nwc * kGroup * 2 * NB;                // [kGroup * NB] activations s

    if (threadIdx.x == 0) {
        for (int s = 0; s < nstages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], nwc);
        }
        fence_mbar_init();
    }
    __syncthreads();

    pdl_wait();  // list / count / y-zeroing of the upstream kernel are now visible
    if (threadIdx.x == 0) TL(kTl, 1);
    const int n = dense ? static_cast<int>(L.F) : __ldcg(S.count);
    const int G = gridDim.x;
    if (!kMC && !dense && blockIdx.x == 0) {
        // The indicator kernel has consumed the latent: restore it to zero for the next chain.
        for (int64_t i = threadIdx.x; i < (int64_t)kMaxBatch * L.ldr; i += blockDim.x) S.latent[i] = 0.0f;
    }

    const W* WU = static_cast<const W*>(L.w_up);
    const W* WG = static_cast<const W*>(L.w_gate);
    const W* WD = static_cast<const W*>(L.w_down);
    const uint32_t all_bits = (1u << nb) - 1u;

    if (warp == nwc) {
        // ---- producer warp: prefetch 32 list entries at a time, lane 0 drives the TMA ring.
        const uint64_t pol = policy_evict_first();
        int st = 0;
        uint32_t ph = 0;
        for (int base = blockIdx.x; base < n; base += kWarp * G) {
            const int my = base + lane * G;
            int32_t my_i = 0;
            uint32_t my_bits = 0;
            float my_u[NB];
#pragma unroll
            for (int b = 0; b < NB; ++b) my_u[b] = 0.0f;
            if (my < n) {
                if (dense) {
                    my_i = my;
                    my_bits = all_bits;
                } else {
                    my_i = __ldcg(S.list + my);
                    my_bits = __ldcg(S.bits + my);
                    if (kListU) {
#pragma unroll
                        for (int b = 0; b < NB; ++b) my_u[b] = __ldcg(S.list_val + (int64_t)my * kMaxBatchFast + b);
                    }
                }
            }
            const int cnt = min(kWarp, (n - base + G - 1) / G);
            for (int k = 0; k < cnt; ++k) {
                const int32_t i = __shfl_sync(0xffffffffu, my_i, k);
                const uint32_t bits = __shfl_sync(0xffffffffu, my_bits, k);
                float u[NB];
#pragma unroll
                for (int b = 0; b < NB; ++b) u[b] = __shfl_sync(0xffffffffu, my_u[b], k);
                if (lane == 0) {
                    mbar_wait(&empty[st], ph ^ 1);
                    meta[st].idx = i;
                    meta[st].bits = bits;
#pragma unroll
                    for (int b = 0; b < NB; ++b) meta[st].u[b] = u[b];
                    uint8_t* dst = smem + st * stage_bytes;
                    mbar_arrive_expect_tx(&full[st], static_cast<uint32_t>(kRows * row_bytes));
                    // one bulk copy per neuron: its record part [(up,) gate, down] is contiguous
                    bulk_g2s(dst, (kMC ? WG : WU) + (int64_t)i * L.rs, (uint32_t)(kRows * row_bytes), &full[st], pol);
                }
                __syncwarp();
                if (++st == nstages) { st = 0; ph ^= 1; }
            }
        }
    } else {
        // ---- consumers: column owners.
        const int ct = threadIdx.x;
        float xr[NB][VPT][8];
        float yr[NB][VPT][8];
#pragma unroll
        for (int j = 0; j < VPT; ++j) {
            const int vec = ct + j * nc;
#pragma unroll
            for (int b = 0; b < NB; ++b)
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const int64_t col = (int64_t)vec * kVec + k;
                    xr[b][j][k] = (vec < nvec && col < L.d && b < nb) ? __ldcg(x + b * L.d + col) : 0.0f;
                    yr[b][j][k] = 0.0f;
                }
        }
        // Slots are consumed kGroup at a time: packed-FFMA2 partial dot products of up to
        // kGroup neurons, ONE halving shuffle reduction for all of them, one named barrier;
        // warp 0 alone finishes the cross-warp sums and the activation (no redundant work in
        // the other warps), a second barrier publishes s, then every column owner
        // accumulates s * W_down[i] into its register-resident y with FFMA2.
        constexpr int kM = kOneDot ? 1 : 2;        // dot products per neuron
        constexpr int kV = kGroup * kM * NB;       // partial sums per lane per group
        int st = 0;
        uint32_t ph = 0;
        int it = 0;
        for (int base = blockIdx.x; base < n; base += G * kGroup, ++it) {
            const int ns = min(kGroup, (n - base + G - 1) / G);
            int sts[kGroup];
            float v[kV];
#pragma unroll
            for (int q = 0; q < kGroup; ++q) {
                sts[q] = st;
                float g0[NB], g1[NB], u0[NB], u1[NB];
#pragma unroll
                for (int b = 0; b < NB; ++b) g0[b] = g1[b] = u0[b] = u1[b] = 0.0f;
                if (q < ns) {
                    mbar_wait(&full[st], ph);
                    if (threadIdx.x == 0 && it == 0 && q == 0) TL(kTl, 2);
                    const uint8_t* sbase = smem + st * stage_bytes;
                    const W* rup = reinterpret_cast<const W*>(sbase);
                    const W* rgate = reinterpret_cast<const W*>(sbase + kDotRow * row_bytes);
#pragma unroll
                    for (int j = 0; j < VPT; ++j) {
                        const int vec = ct + j * nc;
                        if (vec < nvec) {
                            float wg[8], wu[8];
                            Vec8<W>::load(rgate + vec * kVec, wg);
                            if (!kOneDot) Vec8<W>::load(rup + vec * kVec, wu);
#pragma unroll
                            for (int b = 0; b < NB; ++b)
#pragma unroll
                                for (int k = 0; k < 8; k += 2) {
                                    ffma2(g0[b], g1[b], wg[k], wg[k + 1], xr[b][j][k], xr[b][j][k + 1]);
                                    if (!kOneDot) ffma2(u0[b], u1[b], wu[k], wu[k + 1], xr[b][j][k], xr[b][j][k + 1]);
                                }
                        }
                    }
                    if (++st == nstages) { st = 0; ph ^= 1; }
                }
#pragma unroll
                for (int b = 0; b < NB; ++b) {
                    v[(q * kM) * NB + b] = g0[b] + g1[b];
                    if (!kOneDot) v[(q * kM + 1) * NB + b] = u0[b] + u1[b];
                }
            }
            const float tot = warp_transpose_sum<kV>(v);
            if ((lane % (32 / kV)) == 0) red[warp * kV + lane / (32 / kV)] = tot;
            named_bar_sync(1, nc);
            if (warp == 0 && lane < ns * NB) {
                const int q = lane / NB, b = lane % NB;
                float g = 0.0f, u = 0.0f;
                for (int w = 0; w < nwc; ++w) {
                    g += red[w * kV + (q * kM) * NB + b];
                    if (!kOneDot) u += red[w * kV + (q * kM + 1) * NB + b];
                }
                int sq = sts[0];
#pragma unroll
                for (int qq = 1; qq < kGroup; ++qq) sq = (q == qq) ? sts[qq] : sq;
                if (kListU) u = meta[sq].u[b];
                const bool alive = (meta[sq].bits >> b) & 1u;
                float sv = 0.0f;
                if (KIND == kDC_) sv = u * act_fast(L.act, g);
                else if (KIND == kMC_) sv = act_fast(L.act, g) * u;
                else sv = g * u;  // CATS: up dot times the list's act(gate)
                sval[lane] = alive ? sv : 0.0f;
            }
            named_bar_sync(1, nc);
#pragma unroll
            for (int q = 0; q < kGroup; ++q) {
                if (q < ns) {
                    const int sq = sts[q];
                    float sv[NB];
#pragma unroll
                    for (int b = 0; b < NB; ++b) sv[b] = sval[q * NB + b];
                    const W* rdown = reinterpret_cast<const W*>(smem + sq * stage_bytes + kDownRow * row_bytes);
#pragma unroll
                    for (int j = 0; j < VPT; ++j) {
                        const int vec = ct + j * nc;
                        if (vec < nvec) {
                            float wd[8];
                            Vec8<W>::load(rdown + vec * kVec, wd);
#pragma unroll
                            for (int b = 0; b < NB; ++b)
#pragma unroll
                                for (int k = 0; k < 8; k += 2)
                                    ffma2(yr[b][j][k], yr[b][j][k + 1], sv[b], sv[b], wd[k], wd[k + 1]);
                        }
                    }
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&empty[sq]);
                }
            }
        }
        // ---- one vector reduction per owned column group
        if (threadIdx.x == 0) TL(kTl, 3);
        if (n > blockIdx.x) {
#pragma unroll
            for (int j = 0; j < VPT; ++j) {
                const int vec = ct + j * nc;
                if (vec < nvec) {
#pragma unroll
                    for (int b = 0; b < NB; ++b)
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            if (b >= nb) continue;
                            const int64_t col = (int64_t)vec * kVec + h * 4;
                            float* dst = y + b * L.d + col;
                            if (col + 4 <= L.d && ((L.d & 3) == 0)) {
                                red_add_v4(dst, yr[b][j][h * 4], yr[b][j][h * 4 + 1], yr[b][j][h * 4 + 2],
                                           yr[b][j][h * 4 + 3]);
                            } else {
#pragma unroll
                                for (int k = 0; k < 4; ++k)
                                    if (col + k < L.d) red_add_f32(dst + k, yr[b][j][h * 4 + k]);
                            }
                        }
                }
            }
        }
    }
    // ---- last CTA restores the self-cleaning scratch (count, done, alive accumulators).
    __syncthreads();
    if (threadIdx.x == 0) {
        TL(kTl, 4);
        __threadfence();
        TL(kTl, 5);
        const int prev = atomicAdd(S.done, 1);
        if (prev == G - 1) {
            __threadfence();
            for (int b = 0; b < kMaxBatch; ++b) {
                const int a = atomicExch(S.alive + b, 0);
                if (alive_out && b < nb) alive_out[b] = dense ? static_cast<int>(L.F) : a;
            }
            atomicExch(S.count, 0);
            atomicExch(S.done, 0);
        }
        TL(kTl, 6);
    }
}

// ============================================================================ launch helpers
int choose_vpt(int64_t nvec) {
    // smallest vectors-per-thread with <= 384 consumer threads
    for (int v : {1, 2, 4, 8})
        if ((nvec + v - 1) / v <= 384) return v;
    return -1;
}

int consumer_warps(int64_t nvec, int vpt) {
    return static_cast<int>(((nvec + vpt - 1) / vpt + kWarp - 1) / kWarp);
}

}  // namespace

#ifdef CD_TIMELINE
cudaError_t read_timeline(unsigned long long* out, int64_t n) {
    const size_t cnt = (size_t)kTlKernels * kTlCtas * kTlPhases;
    if ((size_t)n < cnt) return cudaErrorInvalidValue;
    cudaError_t e = cudaMemcpyFromSymbol(out, g_timeline, cnt * sizeof(unsigned long long));
    static unsigned long long zeros[kTlKernels * kTlCtas * kTlPhases];
    if (e == cudaSuccess) e = cudaMemcpyToSymbol(g_timeline, zeros, sizeof(zeros));
    return e;
}
#else
cudaError_t read_timeline(unsigned long long*, int64_t) { return cudaErrorNotSupported; }
#endif

// Small host<->device staging copies as a kernel over mapped pinned memory: no copy-engine
// round trip (a 16 KB DMA costs ~10 us of latency in a synchronous call; this ~1-2 us).
__global__ void k_copy_bytes(uint8_t* __restrict__ dst, const uint8_t* __restrict__ src, size_t n) {
    // a PDL-launched successor (the step kernel) may start its weight prologue now; it waits on
    // griddepcontrol.wait for this copy before touching the input
    pdl_launch_dependents();
    const size_t i0 = (static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x) * 16;
    const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x * 16;
    const bool vec = ((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src)) & 15) == 0;
    for (size_t i = i0; i < n; i += stride) {
        if (vec && i + 16 <= n) {
            *reinterpret_cast<uint4*>(dst + i) = __ldcv(reinterpret_cast<const uint4*>(src + i));
        } else {
            for (size_t k = i; k < i + 16 && k < n; ++k) dst[k] = src[k];
        }
    }
}

// Upload check: counts f32 values that are not finite or overflow bf16 (|v| rounds to inf).
__global__ void k_count_nonfinite(const float* __restrict__ v, int64_t n, int* __restrict__ out) {
    int bad = 0;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        bad += !(fabsf(v[i]) < 3.3961e38f);  // NaN compares false
    bad = __reduce_add_sync(0xffffffffu, static_cast<unsigned>(bad));
    if ((threadIdx.x & 31) == 0 && bad) atomicAdd(out, bad);
}

// Input RMS norm of stacked layers: one CTA per sample, f32 sum of squares (tree order).
__global__ void k_rmsnorm(const float* __restrict__ x, int64_t d, float eps, float* __restrict__ xn) {
    __shared__ float part[32];
    const float* xb = x + blockIdx.x * d;
    float* ob = xn + blockIdx.x * d;
    pdl_wait();
    float ss = 0.0f;
    for (int64_t i = threadIdx.x; i < d; i += blockDim.x) ss = fmaf(xb[i], xb[i], ss);
    ss = warp_sum(ss);
    if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = ss;
    __syncthreads();
    if (threadIdx.x < 32) {
        float v = threadIdx.x < (blockDim.x >> 5) ? part[threadIdx.x] : 0.0f;
        v = warp_sum(v);
        if (threadIdx.x == 0) part[0] = rsqrtf(v / static_cast<float>(d) + eps);
    }
    __syncthreads();
    pdl_launch_dependents();
    const float inv = part[0];
    for (int64_t i = threadIdx.x; i < d; i += blockDim.x) ob[i] = xb[i] * inv;
}

// ---------------------------------------------------------------- public launchers
cudaError_t launch_rmsnorm(const float* x, int nb, int64_t d, float eps, float* xn, const LaunchCfg& c) {
    return launch_ex(k_rmsnorm, dim3(nb), dim3(512), 0, c, true, x, d, eps, xn);
}

cudaError_t launch_count_nonfinite(const float* v, int64_t n, int* out, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    const int64_t blocks = (n + 255) / 256;
    k_count_nonfinite<<<static_cast<unsigned>(blocks < 1184 ? blocks : 1184), 256, 0, s>>>(v, n, out);
    return cudaGetLastError();
}

cudaError_t launch_copy(void* dst, const void* src, size_t bytes, cudaStream_t s) {
    if (bytes == 0) return cudaSuccess;
    const size_t blocks = (bytes + 256 * 16 - 1) / (256 * 16);
    k_copy_bytes<<<static_cast<unsigned>(blocks < 64 ? blocks : 64), 256, 0, s>>>(
        static_cast<uint8_t*>(dst), static_cast<const uint8_t*>(src), bytes);
    return cudaGetLastError();
}

// The host-buffer call's outputs to mapped pinned memory in ONE kernel (y, then the alive
// counts), then a completion word the host polls instead of a stream synchronisation: one CTA,
// __threadfence_system() orders the payload before the word (incremented per call: a captured
// graph replays the same kernel).
__global__ void k_copy_out_signal(float* __restrict__ hy, const float* __restrict__ dy, int64_t ny,
                                  int* __restrict__ ha, const int* __restrict__ da, int na,
                                  unsigned long long* done) {
    pdl_wait();  // launched PDL behind the step kernel: resident early, waits for its y here
    if ((ny & 3) == 0 && ((reinterpret_cast<uintptr_t>(hy) | reinterpret_cast<uintptr_t>(dy)) & 15) == 0) {
        for (int64_t i = threadIdx.x; i < ny / 4; i += blockDim.x)
            reinterpret_cast<float4*>(hy)[i] = reinterpret_cast<const float4*>(dy)[i];
    } else {
        for (int64_t i = threadIdx.x; i < ny; i += blockDim.x) hy[i] = dy[i];
    }
    for (int i = threadIdx.x; i < na; i += blockDim.x) ha[i] = da[i];
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) {
        volatile unsigned long long* w = done;
        *w = *w + 1ull;
        __threadfence_system();
    }
}

cudaError_t launch_copy_out_signal(float* hy, const float* dy, int64_t ny, int* ha, const int* da, int na,
                                   unsigned long long* done, cudaStream_t s, bool pdl) {
    // 128 threads: small enough to be co-resident with the step kernel's CTA on an SM
    LaunchCfg c;
    c.stream = s;
    c.pdl = pdl;
    return launch_ex(k_copy_out_signal, dim3(1), dim3(128), 0, c, pdl, hy, dy, ny, ha, da, na, done);
}

cudaError_t launch_spin(unsigned long long ns, cudaStream_t s) {
    k_spin<<<1, 32, 0, s>>>(ns);
    return cudaGetLastError();
}

cudaError_t launch_latent_fast(const LayerDev& L, const Scratch& S, const float* x, int nb,
                               const LaunchCfg& c) {
    if (L.ldr / kVec > 256) return cudaErrorInvalidValue;
    const int G = c.num_sms;
    const int rpc = static_cast<int>((L.d + G - 1) / G);
    auto go = [&](auto kern) {
        return launch_ex(kern, dim3(G), dim3(256), 0, c, false, L, x, S.latent, rpc);
    };
    if (L.dtype == kBF16) {
        switch (nb) {
            case 1: return go(k_latent_fast<__nv_bfloat16, 1>);
            case 2: return go(k_latent_fast<__nv_bfloat16, 2>);
            default: return go(k_latent_fast<__nv_bfloat16, 4>);
        }
    }
    switch (nb) {
        case 1: return go(k_latent_fast<float, 1>);
        case 2: return go(k_latent_fast<float, 2>);
        default: return go(k_latent_fast<float, 4>);
    }
}

cudaError_t launch_indicator_dc_fast(const LayerDev& L, const Scratch& S, int nb, float tau,
                                     const uint8_t* mask_override, float* y, uint8_t* mask_out,
                                     float* logits_out, const LaunchCfg& c) {
    if (L.ldr / kVec > 256) return cudaErrorInvalidValue;
    const int G = c.num_sms;
    const int rpc = static_cast<int>((L.F + G - 1) / G);
    const int64_t esz = L.dtype == kBF16 ? 2 : 4;
    const int64_t row_bytes = L.ldr * esz;
    const int stage_rows = static_cast<int>(std::max<int64_t>(1, kStageBytesTarget / row_bytes));
    const int64_t tail = 16 * 16 + (int64_t)rpc * 8 + 64 + 8 * 16 * 4;
    int nstages = static_cast<int>(imin64(8, (kSmemBudget - tail) / (stage_rows * row_bytes)));
    nstages = std::max(nstages, 2);
    const size_t smem = stage_rows * row_bytes * nstages + 2 * nstages * 8 + (size_t)rpc * 8 + 64 + 8 * 16 * 4;
    const int threads = (8 + 1) * kWarp;
    const int64_t y_len = (int64_t)nb * L.d;
    auto go = [&](auto kern) {
        cudaError_t e = set_smem(kern, smem);
        if (e != cudaSuccess) return e;
        return launch_ex(kern, dim3(G), dim3(threads), smem, c, true, L, S, nb, rpc, stage_rows, nstages, tau,
                         mask_override, y, y_len, mask_out, logits_out);
    };
    const int nvr = static_cast<int>(L.ldr / kVec);
    const int vpl = nvr <= 32 ? 1 : nvr <= 64 ? 2 : nvr <= 128 ? 4 : 8;
    const int nbk = nb <= 1 ? 1 : (nb <= 2 ? 2 : 4);
    if (nbk * vpl > 16) return cudaErrorInvalidValue;
#define CD_DC_CASES(W)                                                                  \
    switch (nbk * 100 + vpl) {                                                          \
        case 101: return go(k_indicator_dc<W, 1, 1>);                                   \
        case 102: return go(k_indicator_dc<W, 1, 2>);                                   \
        case 104: return go(k_indicator_dc<W, 1, 4>);                                   \
        case 108: return go(k_indicator_dc<W, 1, 8>);                                   \
        case 201: return go(k_indicator_dc<W, 2, 1>);                                   \
        case 202: return go(k_indicator_dc<W, 2, 2>);                                   \
        case 204: return go(k_indicator_dc<W, 2, 4>);                                   \
        case 208: return go(k_indicator_dc<W, 2, 8>);                                   \
        case 401: return go(k_indicator_dc<W, 4, 1>);                                   \
        case 402: return go(k_indicator_dc<W, 4, 2>);                                   \
        case 404: return go(k_indicator_dc<W, 4, 4>);                                   \
    }                                                                                   \
    return cudaErrorInvalidValue;
    if (L.dtype == kBF16) { CD_DC_CASES(__nv_bfloat16) }
    CD_DC_CASES(float)
#undef CD_DC_CASES
}

template <typename W, int NB, bool kCats>
static cudaError_t dispatch_mc_vpt(int nb, int vpt, const LayerDev& L, const Scratch& S, const float* x,
                                   int rpc, int nstages, float tau, float* y, int64_t y_len,
                                   uint8_t* mask_out, float* u_out, size_t smem, int threads,
                                   const LaunchCfg& c) {
    auto go = [&](auto kern) {
        cudaError_t e = set_smem(kern, smem);
        if (e != cudaSuccess) return e;
        return launch_ex(kern, dim3(c.num_sms), dim3(threads), smem, c, false, L, S, nb, x, rpc, nstages, tau, y,
                         y_len, mask_out, u_out);
    };
    switch (vpt) {
        case 1: return go(k_indicator_mc<W, NB, 1, kCats>);
        case 2: return go(k_indicator_mc<W, NB, 2, kCats>);
        case 4: if constexpr (NB <= 2) return go(k_indicator_mc<W, NB, 4, kCats>); else return cudaErrorInvalidValue;
        case 8: if constexpr (NB == 1) return go(k_indicator_mc<W, NB, 8, kCats>); else return cudaErrorInvalidValue;
    }
    return cudaErrorInvalidValue;
}

template <typename W, bool kCats>
static cudaError_t dispatch_mc(int nb, int nbk, int vpt, const LayerDev& L, const Scratch& S, const float* x,
                               int rpc, int nstages, float tau, float* y, int64_t y_len, uint8_t* mask_out,
                               float* u_out, size_t smem, int threads, const LaunchCfg& c) {
    if (nbk == 1) return dispatch_mc_vpt<W, 1, kCats>(nb, vpt, L, S, x, rpc, nstages, tau, y, y_len, mask_out, u_out, smem, threads, c);
    if (nbk == 2) return dispatch_mc_vpt<W, 2, kCats>(nb, vpt, L, S, x, rpc, nstages, tau, y, y_len, mask_out, u_out, smem, threads, c);
    return dispatch_mc_vpt<W, 4, kCats>(nb, vpt, L, S, x, rpc, nstages, tau, y, y_len, mask_out, u_out, smem, threads, c);
}

cudaError_t launch_indicator_mc_fast(const LayerDev& L, const Scratch& S, const float* x, int nb,
                                     float tau, float* y, uint8_t* mask_out, float* u_out,
                                     const LaunchCfg& c, bool cats) {
    const int64_t nvec = L.ld / kVec;
    const int vpt = choose_vpt(nvec);
    if (vpt < 0) return cudaErrorInvalidValue;
    const int nwc = consumer_warps(nvec, vpt);
    const int threads = (nwc + 1) * kWarp;
    const int G = c.num_sms;
    const int rpc = static_cast<int>((L.F + G - 1) / G);
    const int64_t esz = L.dtype == kBF16 ? 2 : 4;
    const int64_t stage_bytes = L.ld * esz * kSR;
    const int nbk = nb <= 1 ? 1 : (nb <= 2 ? 2 : 4);
    const int64_t tail = 2 * 8 * 8 + (int64_t)2 * nwc * kSR * nbk * 4 + (int64_t)rpc * (8 + 4 * nbk) + 64;
    int nstages = static_cast<int>(imin64(8, (kSmemBudget - tail) / stage_bytes));
    nstages = std::max(nstages, 2);
    const size_t smem = stage_bytes * nstages + 2 * nstages * 8 + (size_t)2 * nwc * kSR * nbk * 4 +
                        (size_t)rpc * (8 + 4 * nbk) + 64;
    const int64_t y_len = (int64_t)nb * L.d;
    if (L.dtype == kBF16) {
        if (cats) return dispatch_mc<__nv_bfloat16, true>(nb, nbk, vpt, L, S, x, rpc, nstages, tau, y, y_len, mask_out, u_out, smem, threads, c);
        return dispatch_mc<__nv_bfloat16, false>(nb, nbk, vpt, L, S, x, rpc, nstages, tau, y, y_len, mask_out, u_out, smem, threads, c);
    }
    if (cats) return dispatch_mc<float, true>(nb, nbk, vpt, L, S, x, rpc, nstages, tau, y, y_len, mask_out, u_out, smem, threads, c);
    return dispatch_mc<float, false>(nb, nbk, vpt, L, S, x, rpc, nstages, tau, y, y_len, mask_out, u_out, smem, threads, c);
}

template <typename W, int NB, int KIND>
static cudaError_t dispatch_sparse_vpt(int nb, int vpt, const LayerDev& L, const Scratch& S, const float* x,
                                       int nstages, bool dense, float* y, int* alive_out, size_t smem,
                                       int threads, const LaunchCfg& c) {
    auto go = [&](auto kern) {
        cudaError_t e = set_smem(kern, smem);
        if (e != cudaSuccess) return e;
        return launch_ex(kern, dim3(c.num_sms), dim3(threads), smem, c, true, L, S, nb, x, nstages, dense, y,
                         alive_out);
    };
    switch (vpt) {
        case 1: return go(k_sparse<W, NB, 1, KIND>);
        case 2: return go(k_sparse<W, NB, 2, KIND>);
        case 4: if constexpr (NB <= 2) return go(k_sparse<W, NB, 4, KIND>); else return cudaErrorInvalidValue;
        case 8: if constexpr (NB == 1) return go(k_sparse<W, NB, 8, KIND>); else return cudaErrorInvalidValue;
    }
    return cudaErrorInvalidValue;
}

template <typename W, int KIND>
static cudaError_t dispatch_sparse_kind(int nb, int nbk, int vpt, const LayerDev& L, const Scratch& S,
                                        const float* x, int nstages, bool dense, float* y, int* alive_out,
                                        size_t smem, int threads, const LaunchCfg& c) {
    if (nbk == 1) return dispatch_sparse_vpt<W, 1, KIND>(nb, vpt, L, S, x, nstages, dense, y, alive_out, smem, threads, c);
    if (nbk == 2) return dispatch_sparse_vpt<W, 2, KIND>(nb, vpt, L, S, x, nstages, dense, y, alive_out, smem, threads, c);
    return dispatch_sparse_vpt<W, 4, KIND>(nb, vpt, L, S, x, nstages, dense, y, alive_out, smem, threads, c);
}

template <typename W>
static cudaError_t dispatch_sparse(int nb, int nbk, int method, int vpt, const LayerDev& L, const Scratch& S,
                                   const float* x, int nstages, bool dense, float* y, int* alive_out,
                                   size_t smem, int threads, const LaunchCfg& c) {
    if (method == kMC)
        return dispatch_sparse_kind<W, kMC>(nb, nbk, vpt, L, S, x, nstages, dense, y, alive_out, smem, threads, c);
    if (method == kCATS)
        return dispatch_sparse_kind<W, kCATS>(nb, nbk, vpt, L, S, x, nstages, dense, y, alive_out, smem, threads, c);
    return dispatch_sparse_kind<W, kDC>(nb, nbk, vpt, L, S, x, nstages, dense, y, alive_out, smem, threads, c);
}

cudaError_t launch_sparse_fast(const LayerDev& L, const Scratch& S, int method, bool dense,
                               const float* x, int nb, float* y, int* alive_out,
                               const LaunchCfg& c) {
    const int64_t nvec = L.ld / kVec;
    const int vpt = choose_vpt(nvec);
    if (vpt < 0) return cudaErrorInvalidValue;
    const int nbk = nb <= 1 ? 1 : (nb <= 2 ? 2 : 4);
    if (nbk * vpt > 8) return cudaErrorInvalidValue;
    const int nwc = consumer_warps(nvec, vpt);
    const int threads = (nwc + 1) * kWarp;
    const bool mc = method == kMC;
    const int64_t esz = L.dtype == kBF16 ? 2 : 4;
    const int64_t stage_bytes = L.ld * esz * (mc ? 2 : 3);
    const int64_t red_bytes = ((int64_t)nwc * kGroup * 2 * nbk + kGroup * nbk) * 4;
    const int64_t tail = 2 * 8 * 8 + 8 * (int64_t)sizeof(SlotMeta) + red_bytes + 64;
    int nstages = static_cast<int>(imin64(8, (kSmemBudget - tail) / stage_bytes));
    if (nstages < 2) return cudaErrorInvalidValue;
    const size_t smem = stage_bytes * nstages + 2 * nstages * 8 + nstages * sizeof(SlotMeta) + red_bytes + 64;
    if (dense) {
        // Dense comparator: no indicator kernel upstream, so zero y in a tiny PDL-primary kernel.
        cudaError_t e = launch_ex(k_zero, dim3(64), dim3(256), 0, c, false, y, (int64_t)nb * L.d);
        if (e != cudaSuccess) return e;
    }
    if (L.dtype == kBF16)
        return dispatch_sparse<__nv_bfloat16>(nb, nbk, method, vpt, L, S, x, nstages, dense, y, alive_out, smem, threads, c);
    return dispatch_sparse<float>(nb, nbk, method, vpt, L, S, x, nstages, dense, y, alive_out, smem, threads, c);
}

}  // namespace cdk
