// kernels_fused_mc.cu -- the M-CountDown decode step as ONE persistent sm_100a kernel.
//
// pipeline_mc (blocked_exec.cpp:316-328) / Alg. 2 with UnorderedAccumulate
// semantics, batch 1.  One CTA per SM owns a contiguous chunk of neurons:
//
//   stage 1   u_i = W_up[i] . x for the chunk (the dense indicator GEMV, blocked_exec.cpp:322),
//             W_up rows streamed by the TMA engine through the mbarrier ring -- the first ring's
//             worth is issued BEFORE griddepcontrol.wait (weights only), so it overlaps the
//             previous grid's tail; |u| > tau (threshold_mask, blocked_exec.cpp:300-314) with
//             ballot compaction as each group of rows completes.
//   stage 2   the stage-3 schedule of kernels_fused.cu: own active neurons up to the cap (the
//             previous launch's active count over the grid), the overflow published to the
//             launch's work queue as tagged words {neuron id} + {u}, stealing until empty.
//   stage 3   per active neuron ONE bulk copy of its [gate | down] rows (16 KB at d=4096 bf16);
//             s_i = act(W_gate[i] . x) u_i (exec_mc blocked_exec.cpp:188-205), y += s_i W_down[i]
//             in registers of the column-owning consumer threads; the partial y leaves the CTA
//             in one TMA bulk reduction (cp.reduce.async.bulk .add.f32).
//
// y zeroing, the launch tag and the per-CTA alive counts work as in kernels_fused.cu
// (fused_common.cuh).  Grid == number of SMs, one CTA per SM, all CTAs co-resident.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdlib>

#include "common.cuh"
#include "fused_common.cuh"
#include "kernels.h"
#include "launch.cuh"

namespace cdk {

namespace {

using namespace fused;

constexpr int kGroupM = 4;             // records per reduction round (stage 3)
constexpr int kSmemBudgetM = 220 * 1024;
constexpr int kMaxConsumersM = 512;

struct MetaM {
    int32_t idx;
    float u;
};

struct FusedMcParams {
    CUtensorMap wu_map;  // W_up as [rows (stride rs)][ld / inner][inner]: one box = 3 whole rows
    int use_map;
    LayerDev L;
    Scratch S;
    const float* x;
    float* y;
    uint8_t* mask_out;
    float* u_out;
    int* alive_out;
    float tau;
    int nstages, rows_per_cta, rows_per_stage;
    unsigned long long* tl;  // development (CD_MC_TL): per-CTA globaltimer stamps, 8 per CTA
};

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int c0, int c1, int c2, uint64_t* bar,
                                            uint64_t policy) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(smem_u32(dst)),
        "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}

__device__ __forceinline__ void mstamp(const FusedMcParams& P, int k) {
    if (P.tl) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        P.tl[blockIdx.x * 8 + k] = t;
    }
}

template <typename W, int VPT>
__global__ void __launch_bounds__(544, 1) k_mc_fused(const __grid_constant__ FusedMcParams P) {
    const LayerDev& L = P.L;
    const Scratch& S = P.S;
    const int nstages = P.nstages, rows_per_cta = P.rows_per_cta, rps = P.rows_per_stage;
    extern __shared__ __align__(1024) uint8_t smem[];
    constexpr int kBarC = 1;   // consumers only
    constexpr int kBarK = 3;   // consumers -> producer: own list, cap and launch tag in smem
    const int nwc = blockDim.x / kWarp - 1;
    const int nc = nwc * kWarp;
    const int warp = threadIdx.x / kWarp, lane = threadIdx.x % kWarp;
    const int G = gridDim.x;
    const int64_t row_bytes = L.ld * (int64_t)sizeof(W);
    const int64_t stage_bytes = 3 * row_bytes;   // one ring stage: 3 W_up rows or one record
    const int64_t rec_bytes = 2 * row_bytes;     // [gate | down]

    uint8_t* ring = smem;
    uint64_t* full = reinterpret_cast<uint64_t*>(ring + stage_bytes * nstages);
    uint64_t* empty = full + nstages;
    MetaM* meta = reinterpret_cast<MetaM*>(empty + nstages);
    int32_t* own_idx = reinterpret_cast<int32_t*>(meta + nstages);
    float* own_u = reinterpret_cast<float*>(own_idx + rows_per_cta);
    float* red = own_u + rows_per_cta;             // [2][nwc][4] stage-1 partials / [nwc][32] stage 3
    float* sval = red + nwc * 32;                  // [kGroupM]
    int* cnt = reinterpret_cast<int*>(sval + kGroupM);  // [0] n_own [1] tag [2] cap

    const int64_t c0 = (int64_t)blockIdx.x * rows_per_cta;
    const int64_t c1 = imin64(L.F, c0 + rows_per_cta);
    const int nrows = c1 > c0 ? static_cast<int>(c1 - c0) : 0;
    const int nst_u = (nrows + rps - 1) / rps;

    if (threadIdx.x == 0) {
        for (int s = 0; s < nstages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], nwc);
        }
        cnt[0] = 0;
        fence_mbar_init();
    }
    __syncthreads();
    pdl_launch_dependents();
    if (threadIdx.x == 0) mstamp(P, 0);

    const W* WU = static_cast<const W*>(L.w_up);
    const W* WG = static_cast<const W*>(L.w_gate);  // [gate | down] of neuron i at WG + i * rs

    if (warp == nwc) {
        // ================================================================ producer warp
        const uint64_t pol = policy_evict_first();
        int st = 0;
        uint32_t ph = 0;
        if (lane == 0) {
            // stage 1: the chunk's W_up rows (weights: the first ring's worth goes out before
            // griddepcontrol.wait, the rest as the consumers free slots)
            for (int s = 0; s < nst_u; ++s) {
                const int64_t r0 = c0 + (int64_t)s * rps;
                const int n = static_cast<int>(imin64(rps, c1 - r0));
                mbar_wait(&empty[st], ph ^ 1);
                if (P.use_map) {
                    // one tensor copy for the stage's rows (the box always carries rps rows; rows
                    // past the chunk are read but unused, past F zero-filled)
                    mbar_arrive_expect_tx(&full[st], static_cast<uint32_t>(rps * row_bytes));
                    tma_load_3d(ring + st * stage_bytes, &P.wu_map, 0, 0, static_cast<int>(r0), &full[st], pol);
                } else {
                    mbar_arrive_expect_tx(&full[st], static_cast<uint32_t>(n * row_bytes));
                    for (int q = 0; q < n; ++q)
                        bulk_g2s(ring + st * stage_bytes + q * row_bytes, WU + (r0 + q) * L.rs,
                                 static_cast<uint32_t>(row_bytes), &full[st], pol);
                }
                if (++st == nstages) { st = 0; ph ^= 1; }
            }
        }
        __syncwarp();
        st = __shfl_sync(0xffffffffu, st, 0);
        ph = __shfl_sync(0xffffffffu, ph, 0);
        auto issue = [&](int32_t i, float u) {
            mbar_wait(&empty[st], ph ^ 1);
            meta[st].idx = i;
            meta[st].u = u;
            mbar_arrive_expect_tx(&full[st], static_cast<uint32_t>(rec_bytes));
            bulk_g2s(ring + st * stage_bytes, WG + (int64_t)i * L.rs, static_cast<uint32_t>(rec_bytes), &full[st], pol);
            if (++st == nstages) { st = 0; ph ^= 1; }
        };
        // ---- stage 2: own actives up to the cap, overflow to the queue, then steal
        named_bar_sync(kBarK, nc + kWarp);
        const uint32_t tag = static_cast<uint32_t>(cnt[1]);
        const int n_own = cnt[0];
        const int kept = min(n_own, cnt[2]);
        const int ovf = n_own - kept;
        unsigned* qc = S.ctl + kCtlQueue + (tag % 3u) * 32u;  // [0] tail [1] head [2] pushed [3] actives
        int e = 0;
        if (lane == 0)
            for (; e < min(kept, nstages); ++e) issue(own_idx[e], own_u[e]);
        int base = 0;
        if (lane == 0) {
            red_add_u32(qc + 3, static_cast<unsigned>(n_own));
            if (ovf > 0) base = static_cast<int>(atomicAdd(qc + 0, static_cast<unsigned>(ovf)));
        }
        base = __shfl_sync(0xffffffffu, base, 0);
        for (int k = lane; k < ovf; k += kWarp) {
            st_relaxed_u64(S.t_list + base + k, tagged(tag, static_cast<uint32_t>(own_idx[kept + k])));
            st_relaxed_u64(S.t_aux + base + k, tagged(tag, __float_as_uint(own_u[kept + k])));
        }
        __syncwarp();
        if (lane == 0) {
            red_add_u32(qc + 2, 1u);
            for (; e < kept; ++e) issue(own_idx[e], own_u[e]);
            const unsigned G_u = static_cast<unsigned>(G);
            for (;;) {
                const unsigned slot = atomicAdd(qc + 1, 1u);
                bool got = false;
                uint32_t wi = 0, wu = 0;
                for (;;) {
                    if (slot < static_cast<unsigned>(L.F)) {
                        const unsigned long long w = ld_relaxed_u64(S.t_list + slot);
                        if (static_cast<uint32_t>(w >> 32) == tag) {
                            wi = static_cast<uint32_t>(w);
                            wu = await_relaxed(S.t_aux + slot, tag);
                            got = true;
                            break;
                        }
                    }
                    if (ld_relaxed_u32(qc + 2) == G_u && slot >= ld_relaxed_u32(qc + 0)) break;
                }
                if (!got) break;
                issue(static_cast<int32_t>(wi), __uint_as_float(wu));
            }
            mbar_wait(&empty[st], ph ^ 1);  // end-of-work sentinel
            meta[st].idx = -1;
            mbar_arrive(&full[st]);
        }
        __syncwarp();
    } else {
        // ================================================================ consumer warps
        const int ct = threadIdx.x;
        const int nvec = static_cast<int>(L.ld / kVec);
        pdl_wait();
        // x into registers first: in flight together with thread 0's launch-tag read
        float xr[VPT][8];
#pragma unroll
        for (int j = 0; j < VPT; ++j) {
            const int vec = ct + j * nc;
            float4 lo = make_float4(0.f, 0.f, 0.f, 0.f), hi = lo;
            const int64_t col = (int64_t)vec * kVec;
            if (vec < nvec) ldcg_x8(P.x + col, L.d - col, lo, hi);
            xr[j][0] = lo.x; xr[j][1] = lo.y; xr[j][2] = lo.z; xr[j][3] = lo.w;
            xr[j][4] = hi.x; xr[j][5] = hi.y; xr[j][6] = hi.z; xr[j][7] = hi.w;
        }
        unsigned prev_actives = 0;  // thread 0: consumed after stage 1 (one round trip here, not two)
        if (threadIdx.x == 0) {
            const uint32_t t = static_cast<uint32_t>(__ldcg(S.ctl + kCtlEpoch)) + 1u;
            cnt[1] = static_cast<int>(t);
            prev_actives = __ldcg(S.ctl + kCtlQueue + ((t + 2u) % 3u) * 32u + 3);
            if (blockIdx.x == 0) {
                unsigned* nq = S.ctl + kCtlQueue + ((t + 1u) % 3u) * 32u;
                nq[0] = 0u; nq[1] = 0u; nq[2] = 0u; nq[3] = 0u;
            }
        }
        if (blockIdx.x == G - 1) {
            for (int64_t i = ct; i < L.d; i += nc) P.y[i] = 0.0f;
            named_bar_sync(kBarC, nc);
            if (threadIdx.x == 0) {
                __threadfence();
                st_relaxed_u64(S.t_count + kYZeroWord, tagged(static_cast<uint32_t>(cnt[1]), 1u));
            }
        }
        named_bar_sync(kBarC, nc);
        const uint32_t tag = static_cast<uint32_t>(cnt[1]);

        // ---------------------------------------------------------- stage 1: u = W_up x, threshold
        // Stages are consumed (and handed back to the producer) one by one, but reduced across
        // warps in groups of kSG stages: one CTA barrier per 3 kSG rows instead of per 3.
        constexpr int kSG = 4;
        int st = 0;
        uint32_t ph = 0;
        for (int s0 = 0, grp = 0; s0 < nst_u; s0 += kSG, ++grp) {
            float v[4 * kSG];
#pragma unroll
            for (int g = 0; g < kSG; ++g) {
                const int s = s0 + g;
#pragma unroll
                for (int q = 0; q < 4; ++q) v[g * 4 + q] = 0.0f;
                if (s < nst_u) {
                    const int n = static_cast<int>(imin64(rps, c1 - (c0 + (int64_t)s * rps)));
                    mbar_wait(&full[st], ph);
                    if (s == 0 && threadIdx.x == 0) mstamp(P, 1);
                    const W* base = reinterpret_cast<const W*>(ring + st * stage_bytes);
#pragma unroll
                    for (int q = 0; q < 3; ++q) {
                        float a0 = 0.0f, a1 = 0.0f;
                        if (q < n) {
#pragma unroll
                            for (int j = 0; j < VPT; ++j) {
                                const int vec = ct + j * nc;
                                if (vec < nvec) {
                                    float w[8];
                                    Vec8<W>::load(base + q * L.ld + vec * kVec, w);
#pragma unroll
                                    for (int k = 0; k < 8; k += 2) ffma2(a0, a1, w[k], w[k + 1], xr[j][k], xr[j][k + 1]);
                                }
                            }
                        }
                        v[g * 4 + q] = a0 + a1;
                    }
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&empty[st]);  // stage data consumed: the producer refills it
                    if (++st == nstages) { st = 0; ph ^= 1; }
                }
            }
            const float tot = warp_transpose_sum<4 * kSG>(v);
            float* rb = red + (grp & 1) * nwc * 16;  // double-buffered: one barrier per group
            if ((lane & 1) == 0) rb[warp * 16 + (lane >> 1)] = tot;
            named_bar_sync(kBarC, nc);
            if (warp == 0) {
                // lane l: row q = l % 4 of stage s0 + l / 4
                const int s = s0 + (lane >> 2), q = lane & 3;
                const int64_t r0 = c0 + (int64_t)s * rps;
                const bool valid = lane < 4 * kSG && s < nst_u && q < 3 && r0 + q < c1;
                const float u = sum_partials<16>(rb, 16, nwc, lane);  // column lane (lane < 16)
                const int64_t gi = r0 + q;
                bool a = false;
                if (valid) {
                    a = fabsf(u) > P.tau;
                    if (P.mask_out) P.mask_out[gi] = a ? 1 : 0;
                    if (P.u_out) P.u_out[gi] = u;
                }
                const unsigned bal = __ballot_sync(0xffffffffu, a);
                int e0 = 0;
                if (lane == 0 && bal) e0 = atomicAdd(&cnt[0], __popc(bal));
                e0 = __shfl_sync(0xffffffffu, e0, 0);
                if (a) {
                    const int e = e0 + __popc(bal & ((1u << lane) - 1u));
                    own_idx[e] = static_cast<int32_t>(gi);
                    own_u[e] = u;
                }
            }
        }
        if (threadIdx.x == 0)  // own-work cap: the previous launch's active count over the grid
            cnt[2] = prev_actives > 0 ? static_cast<int>((prev_actives + G - 1) / G) : (1 << 30);
        named_bar_sync(kBarC, nc);
        if (threadIdx.x == 0) mstamp(P, 2);
        named_bar_arrive(kBarK, nc + kWarp);  // producer may schedule stage 3 now
        if (threadIdx.x == 0) {
            st_relaxed_u64(S.t_alive + blockIdx.x * kMaxBatchFast, tagged(tag, static_cast<uint32_t>(cnt[0])));
            (void)await_acquire(S.t_count + kYZeroWord, tag);
        }

        // ---------------------------------------------------------- stage 3: sparse gate / down
        float yr[VPT][8];
#pragma unroll
        for (int j = 0; j < VPT; ++j)
#pragma unroll
            for (int k = 0; k < 8; ++k) yr[j][k] = 0.0f;
        int n_rec = 0;
        for (bool done = false; !done;) {
            int ns = 0;
            int sts[kGroupM];
            float v[kGroupM];
#pragma unroll
            for (int q = 0; q < kGroupM; ++q) {
                sts[q] = st;
                float g0 = 0.0f, g1 = 0.0f;
                if (!done) {
                    mbar_wait(&full[st], ph);
                    if (meta[st].idx < 0) done = true;
                    if (n_rec == 0 && q == 0 && threadIdx.x == 0) mstamp(P, 3);
                }
                if (!done) {
                    ns = q + 1;
                    const W* rgate = reinterpret_cast<const W*>(ring + st * stage_bytes);
#pragma unroll
                    for (int j = 0; j < VPT; ++j) {
                        const int vec = ct + j * nc;
                        if (vec < nvec) {
                            float wg[8];
                            Vec8<W>::load(rgate + vec * kVec, wg);
#pragma unroll
                            for (int k = 0; k < 8; k += 2) ffma2(g0, g1, wg[k], wg[k + 1], xr[j][k], xr[j][k + 1]);
                        }
                    }
                    if (++st == nstages) { st = 0; ph ^= 1; }
                }
                v[q] = g0 + g1;
            }
            if (ns == 0) break;
            n_rec += ns;
            const float tot = warp_transpose_sum<kGroupM>(v);
            if ((lane & 7) == 0) red[warp * 32 + (lane >> 3)] = tot;
            named_bar_sync(kBarC, nc);
            if (warp == 0) {
                const float g = sum_partials<kGroupM>(red, 32, nwc, lane);
                if (lane < ns) {
                    int sq = sts[0];
#pragma unroll
                    for (int qq = 1; qq < kGroupM; ++qq) sq = (lane == qq) ? sts[qq] : sq;
                    sval[lane] = act_fast(L.act, g) * meta[sq].u;
                }
            }
            named_bar_sync(kBarC, nc);
#pragma unroll
            for (int q = 0; q < kGroupM; ++q) {
                if (q < ns) {
                    const int sq = sts[q];
                    const float sv = sval[q];
                    const W* rdown = reinterpret_cast<const W*>(ring + sq * stage_bytes + row_bytes);
#pragma unroll
                    for (int j = 0; j < VPT; ++j) {
                        const int vec = ct + j * nc;
                        if (vec < nvec) {
                            float wd[8];
                            Vec8<W>::load(rdown + vec * kVec, wd);
#pragma unroll
                            for (int k = 0; k < 8; k += 2) ffma2(yr[j][k], yr[j][k + 1], sv, sv, wd[k], wd[k + 1]);
                        }
                    }
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&empty[sq]);
                }
            }
        }
        if (threadIdx.x == 0) mstamp(P, 4);
        if (n_rec > 0) {
            named_bar_sync(kBarC, nc);  // every consumer is past its last ring read
            float* ys = reinterpret_cast<float*>(ring);
#pragma unroll
            for (int j = 0; j < VPT; ++j) {
                // d % 4 == 0 (launch requirement): whole float4s (scalar stores conflict 8-way)
                const int vec = ct + j * nc;
                const int64_t col = (int64_t)vec * kVec;
                if (vec >= nvec) continue;
                float4* dst = reinterpret_cast<float4*>(ys + col);
                if (col < L.d) dst[0] = make_float4(yr[j][0], yr[j][1], yr[j][2], yr[j][3]);
                if (col + 4 < L.d) dst[1] = make_float4(yr[j][4], yr[j][5], yr[j][6], yr[j][7]);
            }
            fence_proxy_async_smem();
            named_bar_sync(kBarC, nc);
            if (threadIdx.x == 0) {
                bulk_reduce_add_f32(P.y, ys, static_cast<uint32_t>(L.d * sizeof(float)));
                bulk_commit_and_wait_read();
            }
        }
        if (threadIdx.x == 0) mstamp(P, 5);
        if (blockIdx.x == 0 && warp == 0) {
            if (P.alive_out) {
                int a = 0;
                for (int i = lane; i < G; i += kWarp)
                    a += static_cast<int>(await_relaxed(S.t_alive + i * kMaxBatchFast, tag));
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
                if (lane == 0) P.alive_out[0] = a;
            }
            if (lane == 0) S.ctl[kCtlEpoch] = tag;
        }
    }
}

}  // namespace

cudaError_t launch_mc_fused(const LayerDev& L, const Scratch& S, const float* x, float tau, float* y,
                            uint8_t* mask_out, float* u_out, int* alive_out, const LaunchCfg& c) {
    if (!S.t_list || !S.t_aux || !S.t_count || !S.t_alive || !S.ctl) return cudaErrorInvalidValue;
    if (c.num_sms >= kYZeroWord || L.F >= (1 << 27)) return cudaErrorInvalidValue;
    if (L.d % 4 != 0 || (reinterpret_cast<uintptr_t>(y) & 15) != 0) return cudaErrorInvalidValue;
    const int64_t nvec = L.ld / kVec;
    int vpt = 0;
    for (int v : {1, 2, 4})
        if ((nvec + v - 1) / v <= kMaxConsumersM) { vpt = v; break; }
    if (vpt == 0) return cudaErrorInvalidValue;
    const int G = c.num_sms;
    const int rpc = static_cast<int>((L.F + G - 1) / G);
    const int64_t esz = L.dtype == kBF16 ? 2 : 4;
    const int64_t stage_bytes = 3 * L.ld * esz;
    const int nwc = static_cast<int>(std::max<int64_t>(8, ((nvec + vpt - 1) / vpt + kWarp - 1) / kWarp));
    const int threads = (nwc + 1) * kWarp;
    const int64_t fixed = (int64_t)rpc * 8 + (nwc * 32 + kGroupM) * 4 + 3 * 4 + 64;
    const int64_t per_stage = stage_bytes + 2 * 8 + (int64_t)sizeof(MetaM);
    const int nstages = static_cast<int>(imin64(12, (kSmemBudgetM - fixed) / per_stage));
    if (nstages < 2) return cudaErrorInvalidValue;
    const size_t smem = static_cast<size_t>(fixed + per_stage * nstages);
    auto go = [&](auto kern) {
        cudaError_t e = set_smem(kern, smem);
        if (e != cudaSuccess) return e;
        FusedMcParams p;
        p.L = L;
        p.S = S;
        p.x = x;
        p.y = y;
        p.mask_out = mask_out;
        p.u_out = u_out;
        p.alive_out = alive_out;
        p.tau = tau;
        p.nstages = nstages;
        p.rows_per_cta = rpc;
        p.rows_per_stage = 3;
        // W_up stage loads as one 3-D tensor copy: [rows][ld / inner][inner], no swizzle (the smem
        // image is the plain row-major 3 x ld block the consumers read)
        p.use_map = 0;
        static const bool map_env = dev_knob("CD_MC_TMAP", 1) != 0;
        int inner = 0;
        for (int cand : {256, 128, 64, 32, 16, 8})
            if (L.ld % cand == 0 && L.ld / cand <= 256) { inner = cand; break; }
        static PFN_cuTensorMapEncodeTiled_v12000 enc = [] {
            void* fp = nullptr;
            cudaDriverEntryPointQueryResult q;
            return (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q) == cudaSuccess &&
                    q == cudaDriverEntryPointSuccess)
                       ? reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fp)
                       : nullptr;
        }();
        if (map_env && inner > 0 && enc) {
            const cuuint64_t dims[3] = {static_cast<cuuint64_t>(inner), static_cast<cuuint64_t>(L.ld / inner),
                                        static_cast<cuuint64_t>(L.F)};
            const cuuint64_t strides[2] = {static_cast<cuuint64_t>(inner * esz), static_cast<cuuint64_t>(L.rs * esz)};
            const cuuint32_t box[3] = {static_cast<cuuint32_t>(inner), static_cast<cuuint32_t>(L.ld / inner), 3u};
            const cuuint32_t estr[3] = {1, 1, 1};
            if (enc(&p.wu_map, L.dtype == kBF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3,
                    const_cast<void*>(L.w_up), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS)
                p.use_map = 1;
        }
        static unsigned long long* tl_env = []() -> unsigned long long* {
#ifdef CD_TIMELINE  // development builds only: a device address taken from the environment
        const char* e = std::getenv("CD_MC_TL");
        return e ? reinterpret_cast<unsigned long long*>(std::strtoull(e, nullptr, 10)) : nullptr;
#else
        return nullptr;
#endif
    }();
        p.tl = tl_env;
        return launch_persistent(kern, dim3(G), dim3(threads), smem, c, true, p);
    };
    if (L.dtype == kBF16) {
        if (vpt == 1) return go(k_mc_fused<__nv_bfloat16, 1>);
        if (vpt == 2) return go(k_mc_fused<__nv_bfloat16, 2>);
        return go(k_mc_fused<__nv_bfloat16, 4>);
    }
    if (vpt == 1) return go(k_mc_fused<float, 1>);
    if (vpt == 2) return go(k_mc_fused<float, 2>);
    return go(k_mc_fused<float, 4>);
}

}  // namespace cdk
