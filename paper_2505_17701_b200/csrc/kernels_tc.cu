// kernels_tc.cu -- batched decode (B >= 8) and dense prefill on the 5th-generation tensor cores.
//
// SURVEY.md section 8f row 1.  At batch 64 the union of the per-sample masks covers ~every
// neuron (0.8^64 ~ 0), so the batched step streams ALL up/gate/down rows once and zeroes s per
// sample -- a masked row-union GEMM.  The reference semantics stay per sample
// (blocked_exec.cpp:252-298 for MC, :350-379 for DC; main.cpp:239-282 loops samples).
//
//   phase A (this file, k_tc_gateup): one CTA per 128-neuron tile x n-tile of samples.
//       TMA (128B-swizzled boxes) -> smem ring -> tcgen05.mma (one elected thread) ->
//       TMEM accumulators U = W_up X^T, G = W_gate X^T (+ Z = theta_b^T latent^T for D-CountDown)
//       -> epilogue warps: tcgen05.ld, per-sample mask (z > tau | |u| > tau | |act(g)| > tau |
//       override), s = u * act(g) or 0, written as bf16 (hi, lo) pairs; mask / indicator /
//       alive-count outputs.
//   phase B: y = S W_down, a plain GEMM (cuBLAS bf16 tensor-core GEMM, f32 out), then the
//       hi + lo fold.  The D-CountDown latent x theta_a is a plain GEMM as well.
//
// Precision.  Decode ("split" mode) carries every activation operand as a pair of bf16 values
// (hi = rn(v), lo = rn(v - hi)), so products with the bf16 weights are exact to ~2^-16 and the
// f32 accumulation dominates: the result matches the CUDA-core path to ~1e-5 relative, and the
// thresholds see the same logits.  Prefill (large token counts, dense) uses plain bf16
// activations (standard bf16 inference numerics, 1e-2 bound).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdlib>
#include <mutex>

#include "common.cuh"
#include "kernels.h"
#include "kernels_tc.h"
#include "launch.cuh"
#include "tc_common.cuh"

namespace cdk {
namespace tc {

namespace {

// ---------------------------------------------------------------- phase A kernel
//
// Work: tiles = (128-neuron m-tile, n-tile of samples), tile-major with the n-tiles of one
// m-tile adjacent (their weight boxes are shared through L2).  Each tile is nkb = kb_z + kb_x
// k-blocks (the D-CountDown predictor blocks theta_b^T x latent first, then up/gate blocks).
//
// Stream-K schedule: the grid is one CTA per SM and CTA c owns the contiguous k-block range
// [c U / G, (c+1) U / G) of all U = tiles x nkb k-blocks, so every SM streams the same number of
// weight bytes (a tile-per-CTA grid leaves 40 of 148 SMs idle at the Qwen shape).  A range splits
// into segments (one per tile it touches).  The segment holding a tile's k-block 0 (the LAST
// segment of its CTA) finishes the tile: it adds the partial accumulators that the following
// CTAs wrote for the rest of that tile -- their FIRST segments, so already available -- and runs
// the epilogue.  Partials travel through an L2-resident workspace with one release flag per
// CTA (the finisher resets it: self-cleaning across launches).  Needs all CTAs co-resident
// (grid <= SMs, one CTA per SM).
constexpr int kOvr = 4;  // epilogue kind: D-CountDown with a given mask (override / exec_dc)

// Prefill (a.dp): whole tiles instead -- wave w gives CTA c tile w G + c, tiles m-major, so the
// token tiles of one neuron tile run side by side on neighbouring CTAs and read its weight
// k-blocks through L2 once (stream-K ranges would re-stream each neuron tile from HBM per
// token tile: 8x the weight bytes at 2048 tokens).
// With a 2-CTA cluster (mc), the two CTAs of a cluster take the two token tiles of one
// (neuron tile, token-tile pair) and each multicasts one of the two weight boxes to both: the
// tile index is then m ntp + tt with ntp the token-tile count rounded up to even (a phantom
// odd tile reads zero-filled rows and stores nothing).
__device__ __forceinline__ bool gu_seg(int c, int si, int64_t U, int G, int nkb, bool dp, int tiles, Seg& sg,
                                       int mc = 0, int n_tiles = 1) {
    if (!dp) return seg_at(c, si, U, G, nkb, sg);
    if (mc) {
        const int half = (n_tiles + 1) / 2;  // token-tile pairs per neuron tile
        const int pairs = (tiles / n_tiles) * half;
        const int pi = (c >> 1) + si * (G >> 1);
        if (pi >= pairs) return false;
        sg = {(pi / half) * 2 * half + 2 * (pi % half) + (c & 1), 0, nkb};
        return true;
    }
    const int t = c + si * G;
    if (t >= tiles) return false;
    sg = {t, 0, nkb};
    return true;
}

template <int KIND, bool SPLIT, int ACT>
__global__ void __launch_bounds__(kThreads, 1)
k_tc_gateup(const __grid_constant__ CUtensorMap m_up, const __grid_constant__ CUtensorMap m_gate,
            const __grid_constant__ CUtensorMap m_x, const __grid_constant__ CUtensorMap m_tb,
            const __grid_constant__ CUtensorMap m_lat, const GateUpArgs a) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int N = a.N;
    const int stage_bytes = 2 * kABytes + N * kBK * 2;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + a.stages * stage_bytes);
    uint64_t* empty = full + a.stages;
    uint64_t* tfull = empty + a.stages;  // [2] accumulators of a segment complete (MMA -> epilogue)
    uint64_t* tempty = tfull + 2;        // [2] accumulators drained (epilogue -> MMA)
    uint64_t* pbar = tempty + 2;         // contributor partials landed in smem (finisher)
    // TMEM buffers: segment si accumulates into buffer si % nbuf (columns [b bstride, ...)), so
    // with two buffers the epilogue of one tile overlaps the MMAs of the next
    const int nbuf = a.nbuf > 1 ? 2 : 1;
    const uint32_t bstride = static_cast<uint32_t>(a.buf_cols);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(pbar + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nkb = a.kb_z + a.kb_x;
    const int G = gridDim.x, c = blockIdx.x;
    const int64_t U = static_cast<int64_t>(a.tiles) * nkb;

    if (warp == 0 && lane == 0) {
        for (int s = 0; s < a.stages; ++s) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, a.mc ? 2 : 1);  // mc: both CTAs' MMAs read the multicast boxes
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(tfull + b, 1);
            mbar_init(tempty + b, kEpiThreads);
        }
        mbar_init(pbar, 1);
        fence_mbar_init();
        prefetch_map(&m_up);
        prefetch_map(&m_gate);
        prefetch_map(&m_x);
        if (a.kb_z) {
            prefetch_map(&m_tb);
            prefetch_map(&m_lat);
        }
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(a.tmem_cols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    if (a.mc) cluster_sync();  // the peer's barriers are initialised before any multicast lands
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const int ntd = a.mc ? (a.n_tiles + 1) & ~1 : a.n_tiles;  // token tiles per neuron tile (decode)
    auto stamp = [&](int k) {
        if (a.tl) {
            unsigned long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            a.tl[c * 8 + k] = t;
        }
    };
    if (threadIdx.x == 0) stamp(0);

    if (warp == 0) {
        if (lane == 0) {
            // ---- TMA producer: the CTA's k-blocks in order, one continuous ring
            // weights: streamed once (decode) / shared by the token tiles of a wave (prefill);
            // activations: re-read by every neuron tile
            const uint64_t pw = a.dp ? policy_evict_last() : policy_evict_first();
            const uint64_t px = policy_evict_last();
            int it = 0;
            Seg sg;
            for (int si = 0; gu_seg(c, si, U, G, nkb, a.dp != 0, a.tiles, sg, a.mc, a.n_tiles); ++si) {
                const int m0 = (sg.tile / ntd) * kBM;
                const int row0 = (sg.tile % ntd) * N;
                for (int kb = sg.kb0; kb < sg.kb1; ++kb, ++it) {
                    const int s = it % a.stages;
                    if (it >= a.stages) mbar_wait(empty + s, ((it / a.stages) - 1) & 1);
                    uint8_t* st = smem + s * stage_bytes;
                    if (kb < a.kb_z) {
                        mbar_arrive_expect_tx(full + s, kABytes + N * kBK * 2);
                        tma_load_2d(st, &m_tb, kb * kBK, m0, full + s, pw);
                        tma_load_2d(st + 2 * kABytes, &m_lat, kb * kBK, row0, full + s, px);
                    } else {
                        const int k = (kb - a.kb_z) * kBK;
                        if (it == 0) stamp(1);
                        mbar_arrive_expect_tx(full + s, 2 * kABytes + N * kBK * 2);
                        if (!a.mc) {
                            tma_load_2d(st, &m_up, k, m0, full + s, pw);
                            tma_load_2d(st + kABytes, &m_gate, k, m0, full + s, pw);
                        } else if ((c & 1) == 0) {
                            tma_load_2d_mc(st, &m_up, k, m0, full + s, 0x3, pw);
                        } else {
                            tma_load_2d_mc(st + kABytes, &m_gate, k, m0, full + s, 0x3, pw);
                        }
                        tma_load_2d(st + 2 * kABytes, &m_x, k, row0, full + s, px);
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            // ---- MMA issuer: U at TMEM columns [0, N), G at [N, 2N), Z at [2N, 3N)
            const uint32_t idesc = idesc_bf16(kBM, N);
            int it = 0;
            Seg sg;
            for (int si = 0; gu_seg(c, si, U, G, nkb, a.dp != 0, a.tiles, sg, a.mc, a.n_tiles); ++si) {
                const int bf = si % nbuf;
                if (si >= nbuf) {
                    mbar_wait(tempty + bf, ((si / nbuf) - 1) & 1);  // the epilogue drained this buffer
                    tc_fence_after();
                }
                const uint32_t tU = tmem + bf * bstride, tG = tU + N, tZ = tU + 2 * N;
                const int first_ug = max(sg.kb0, a.kb_z);
                for (int kb = sg.kb0; kb < sg.kb1; ++kb, ++it) {
                    const int s = it % a.stages;
                    mbar_wait(full + s, (it / a.stages) & 1);
                    tc_fence_after();
                    const uint32_t base = smem_u32(smem + s * stage_bytes);
                    const uint64_t da0 = sw128_desc(base), da1 = sw128_desc(base + kABytes),
                                   db = sw128_desc(base + 2 * kABytes);
#pragma unroll
                    for (int k = 0; k < kBK / 16; ++k) {
                        // +32 bytes per 16-element K step inside the swizzle atom (descriptor units of 16 B)
                        const uint64_t o = static_cast<uint64_t>(2 * k);
                        if (kb < a.kb_z) {
                            umma_bf16(tZ, da0 + o, db + o, idesc, (kb > sg.kb0 || k > 0) ? 1u : 0u);
                        } else {
                            const uint32_t acc = (kb > first_ug || k > 0) ? 1u : 0u;
                            umma_bf16(tU, da0 + o, db + o, idesc, acc);
                            umma_bf16(tG, da1 + o, db + o, idesc, acc);
                        }
                    }
                    // frees the stage once these MMAs have read it (mc: in both CTAs)
                    if (a.mc) umma_commit_mc(empty + s, 0x3);
                    else umma_commit(empty + s);
                }
                umma_commit(tfull + bf);
            }
            stamp(2);
        }
    } else {
        // ---- epilogue: warp w reads TMEM lanes 32 (w % 4) .. +31 = the tile's neuron rows; the
        // two warps of a lane group split the samples (columns) in halves
        const int g = warp & 3;
        const int half = (warp - 2) >> 2;
        const int m = g * 32 + lane;
        const int et = threadIdx.x - 64;  // 0 .. kEpiThreads-1
        const uint32_t trow0 = tmem + (static_cast<uint32_t>(g * 32) << 16);
        constexpr bool kZ = KIND == kDC;
        constexpr int kParts = kZ ? 3 : 2;
        constexpr int kH = SPLIT ? 2 : 1;
        constexpr int kC = 8;  // samples per chunk
        Seg sg;
        for (int si = 0; gu_seg(c, si, U, G, nkb, a.dp != 0, a.tiles, sg, a.mc, a.n_tiles); ++si) {
            const int bf = si % nbuf;
            mbar_wait(tfull + bf, (si / nbuf) & 1);
            tc_fence_after();
            const uint32_t trow = trow0 + bf * bstride;
            if (et == 0) stamp(3 + (si > 2 ? 2 : si));
            const bool has_z = kZ && sg.kb0 < a.kb_z;
            const bool has_ug = sg.kb1 > a.kb_z;
            if (sg.kb0 > 0) {
                // contributor: park the partial accumulators (hi + lo summed) in this CTA's
                // workspace slot, laid out [part][sample][row]
                float* slot = a.ws + static_cast<int64_t>(c) * kParts * a.nbt * kBM;
                for (int q = 0; q < kParts; ++q) {
                    if (q == 2 ? !has_z : !has_ug) continue;
                    for (int c0 = half * 16; c0 < a.nbt; c0 += 32) {
                        float v[16];
                        tmem_ld16(trow + q * N + c0, v);
                        if constexpr (SPLIT) {
                            float w[16];
                            tmem_ld16(trow + q * N + a.nbt + c0, w);
                            tmem_wait_ld();
#pragma unroll
                            for (int j = 0; j < 16; ++j) v[j] += w[j];
                        } else {
                            tmem_wait_ld();
                        }
#pragma unroll
                        for (int j = 0; j < 16; ++j) slot[(q * a.nbt + c0 + j) * kBM + m] = v[j];
                    }
                }
                tc_fence_before();
                mbar_arrive(tempty + bf);
                __threadfence();
                named_bar_sync(1, kEpiThreads);
                if (et == 0) st_release_u32(a.flags + c, 1u);
                continue;
            }
            // finisher (holds k-block 0): gather the partials of the CTAs that follow
            const int tile = sg.tile;
            const int64_t tile_base = static_cast<int64_t>(tile) * nkb;
            int c_last = c;
            while (!a.dp && c_last + 1 < G && range_lo(c_last + 1, U, G) < tile_base + nkb) ++c_last;
            // the contributors' partials, pulled into the (now idle) ring with bulk copies when
            // they fit -- the finisher segment is its CTA's last, so no stage is in flight
            const int64_t slot_floats = static_cast<int64_t>(kParts) * a.nbt * kBM;
            const bool in_smem = (c_last - c) * slot_floats * 4 <= static_cast<int64_t>(a.stages) * stage_bytes;
            if (c_last > c) {
                if (et < c_last - c) {
                    unsigned* f = a.flags + c + 1 + et;
                    while (ld_acquire_u32(f) == 0u) {
                    }
                    *f = 0u;  // consumed: ready for the next launch
                }
                __threadfence();
                named_bar_sync(1, kEpiThreads);
                if (in_smem) {
                    if (et == 0) {
                        fence_proxy_async_smem();
                        const uint32_t bytes = static_cast<uint32_t>(slot_floats * 4);
                        mbar_arrive_expect_tx(pbar, bytes * (c_last - c));
                        for (int cc = c + 1; cc <= c_last; ++cc)
                            bulk_g2s(smem + (cc - c - 1) * bytes, a.ws + cc * slot_floats, bytes, pbar,
                                     policy_evict_first());
                    }
                    mbar_wait(pbar, 0);
                }
            }
            const int m0 = (tile / ntd) * kBM;
            const int ntile = tile % ntd;
            const int i = m0 + m;
            const bool valid = i < a.F;
            const int nbt = a.nbt;
            const int64_t F = a.F;
            const int64_t ld_s = a.ld_s;
            const int64_t gb0 = static_cast<int64_t>(ntile) * nbt;
            const int nlive = a.nb - gb0 < nbt ? static_cast<int>(a.nb - gb0) : nbt;
            const int hb = nbt / 2;  // samples per half
            const int sb0 = half * hb;
            // this row's s outputs: sample sb of the tile -> hi row (pair layout) / token row
            __nv_bfloat16* s_hi = a.s_out +
                                  (SPLIT ? static_cast<int64_t>(ntile) * N : static_cast<int64_t>(ntile) * nbt) * ld_s +
                                  static_cast<int64_t>(sb0) * ld_s + i;
            const int64_t lo_step = static_cast<int64_t>(nbt) * ld_s;
            for (int cb = sb0; cb < sb0 + hb; cb += kC, s_hi += kC * ld_s) {
                float acc[kParts][kH][kC];
#pragma unroll
                for (int q = 0; q < kParts; ++q) {
                    const bool own = q == 2 ? has_z : has_ug;
#pragma unroll
                    for (int h = 0; h < kH; ++h) {
                        if (own) {
                            tmem_ld8(trow + q * N + h * nbt + cb, acc[q][h]);
                        } else {
#pragma unroll
                            for (int j = 0; j < kC; ++j) acc[q][h][j] = 0.0f;
                        }
                    }
                }
                tmem_wait_ld();
                if (c_last > c) {
                    for (int cc = c + 1; cc <= c_last; ++cc) {
                        const int64_t q0 = range_lo(cc, U, G) - tile_base;
                        const int64_t q1 = range_lo(cc + 1, U, G) - tile_base;
#pragma unroll
                        for (int q = 0; q < kParts; ++q) {
                            if (q == 2 ? !(q0 < a.kb_z) : !(q1 > a.kb_z)) continue;
                            const int64_t off = (q * nbt + cb) * kBM + m;
                            if (in_smem) {
                                const float* sp = reinterpret_cast<const float*>(smem) + (cc - c - 1) * slot_floats + off;
#pragma unroll
                                for (int j = 0; j < kC; ++j) acc[q][0][j] += sp[j * kBM];
                            } else {
                                const float* gp = a.ws + cc * slot_floats + off;
#pragma unroll
                                for (int j = 0; j < kC; ++j) acc[q][0][j] += __ldcg(gp + j * kBM);
                            }
                        }
                    }
                }
                unsigned on_bits = 0;
                __nv_bfloat16* p = s_hi;
#pragma unroll
                for (int j = 0; j < kC; ++j, p += ld_s) {
                    float u = acc[0][0][j], gg = acc[1][0][j], z = kZ ? acc[kParts - 1][0][j] : 0.0f;
                    if constexpr (SPLIT) {
                        u += acc[0][kH - 1][j];
                        gg += acc[1][kH - 1][j];
                        if constexpr (kZ) z += acc[kParts - 1][kH - 1][j];
                    }
                    const bool live = valid && cb + j < nlive;
                    const float ag = act_epi(ACT, gg);
                    bool on;
                    if constexpr (KIND == kDC) {
                        on = z > a.tau;
                    } else if constexpr (KIND == kMC) {
                        on = fabsf(u) > a.tau;
                    } else if constexpr (KIND == kCATS) {
                        on = fabsf(ag) > a.tau;
                    } else if constexpr (KIND == kOvr) {
                        on = live && a.ovr[(gb0 + cb + j) * F + i] != 0;
                    } else {
                        on = true;
                    }
                    on = on && live;
                    on_bits |= on ? 1u << j : 0u;
                    const float sv = on ? u * ag : 0.0f;
                    if (live) {
                        const __nv_bfloat16 hv = __float2bfloat16_rn(sv);
                        *p = hv;
                        if constexpr (SPLIT) p[lo_step] = __float2bfloat16_rn(sv - __bfloat162float(hv));
                        if (a.ind_out) a.ind_out[(gb0 + cb + j) * F + i] = KIND == kDC ? z : KIND == kCATS ? ag : u;
                    }
                }
                if (valid && a.mask_out) {
                    for (int j = 0; j < kC && cb + j < nlive; ++j)
                        a.mask_out[(gb0 + cb + j) * F + i] = (on_bits >> j) & 1u;
                }
                if (a.alive_out) {
                    // per-sample counts: popc of the warp's ballot of each sample's bit
#pragma unroll
                    for (int j = 0; j < kC; ++j) {
                        const unsigned bal = __ballot_sync(0xffffffffu, (on_bits >> j) & 1u);
                        if (lane == j && bal) atomicAdd(a.alive_out + gb0 + cb + j, __popc(bal));
                    }
                }
            }
            tc_fence_before();
            mbar_arrive(tempty + bf);
        }
        tc_fence_before();
        if (et == 0) stamp(6);
    }
    __syncthreads();
    if (a.mc) cluster_sync();  // no multicast or remote commit still targets this CTA
    if (threadIdx.x == 0) stamp(7);
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(a.tmem_cols) : "memory");
    }
}

// ---------------------------------------------------------------- prefill down projection
//
// Y (nb x d, f32) = S W_down for dense prefill (weighted_sum / forward_dense, gated_mlp.cpp:28-59,
// over a token block): a plain compute-bound GEMM, M = tokens, N = d, K = F.
//   A = S rows (K-major, bf16, written by the gate/up kernel), TMA boxes 64 K x 128 tokens.
//   B = W_down as [F][d]: d contiguous in each neuron's down row, so B is MN-major; TMA boxes
//       64 d x 64 K, 128B-swizzled, four per 256-column tile (descriptor LBO = one box, 8 KB).
// CTA tile 256 tokens x 256 columns: two UMMA M=128 N=256 accumulators (the whole 512-column
// TMEM), each k-block loads 2 x 16 KB of A and 32 KB of B -- 64 KB per 2 x 4.2 MFLOP, the
// L2->SM feed that bounds a single-CTA tile.  Three 64 KB ring stages.
// Schedule: whole tiles first (tile t on CTA t mod G while a full wave remains: plain v4 stores),
// then the remaining tiles' k-blocks split evenly over all CTAs (stream-K, red.global.add.v4 into
// rows zeroed by k_tc_zero_tiles).  Epilogue: 8 warps, warp w drains TMEM lane quarter w % 4 of
// accumulator (w - 2) / 4, 16 columns per tcgen05.ld.
constexpr int kPfN = 256;                       // columns (d) per tile
constexpr int kPfM = 256;                       // tokens per tile (two M=128 accumulators)
constexpr int kPfStage = 2 * kABytes + 4 * kBK * kBK * 2;  // 64 KB

struct PfDownArgs {
    int nb = 0, d = 0;
    int nkb = 0;            // 64-neuron k-blocks
    int n_tt = 0, n_jt = 0; // token tiles, column tiles
    int n_full = 0;         // (pair-)tiles done whole (a multiple of the grid), the rest stream-K
    int stages = 0;
    int mc = 0;             // 2-CTA clusters: the pair takes two column tiles of one token tile and
                            // each CTA multicasts one of the two S boxes to both
    float* y = nullptr;
};

struct PfSeg {
    int tile, kb0, kb1;
    bool whole;
};

// Segment si of CTA c: its whole tiles c, c + G, ... < n_full, then its stream-K range over the
// remaining tiles' k-blocks.
__device__ __forceinline__ bool pf_seg(int c, int si, int G, const PfDownArgs& a, PfSeg& sg) {
    // units of the schedule: tiles, or (mc) column-tile pairs handled by the CTA pairs
    const int ju = a.mc ? (a.n_jt + 1) / 2 : a.n_jt;
    const int units = a.n_tt * ju;
    const int w = a.mc ? c >> 1 : c;
    const int W = a.mc ? G >> 1 : G;
    int u = -1, kb0 = 0, kb1 = a.nkb;
    bool whole = false;
    const int n_whole = a.n_full > w ? (a.n_full - w + W - 1) / W : 0;
    if (si < n_whole) {
        u = w + si * W;
        whole = true;
    } else {
        const int64_t U = static_cast<int64_t>(units - a.n_full) * a.nkb;
        Seg s2;
        if (U <= 0 || !seg_at(w, si - n_whole, U, W, a.nkb, s2)) return false;
        u = a.n_full + s2.tile;
        kb0 = s2.kb0;
        kb1 = s2.kb1;
    }
    const int tt = u / ju, jt = a.mc ? 2 * (u % ju) + (c & 1) : u % ju;
    sg = {tt * (a.mc ? 2 * ju : a.n_jt) + jt, kb0, kb1, whole};
    return true;
}

__global__ void __launch_bounds__(kThreads, 1)
k_tc_pf_down(const __grid_constant__ CUtensorMap m_s, const __grid_constant__ CUtensorMap m_w, const PfDownArgs a) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + a.stages * kPfStage);
    uint64_t* empty = full + a.stages;
    uint64_t* tfull = empty + a.stages;
    uint64_t* tempty = tfull + 1;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 1);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int G = gridDim.x, c = blockIdx.x;
    const int jw = a.mc ? 2 * ((a.n_jt + 1) / 2) : a.n_jt;  // tile index = tt jw + jt

    if (warp == 0 && lane == 0) {
        for (int s = 0; s < a.stages; ++s) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, a.mc ? 2 : 1);
        }
        mbar_init(tfull, 1);
        mbar_init(tempty, kEpiThreads);
        fence_mbar_init();
        prefetch_map(&m_s);
        prefetch_map(&m_w);
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(512)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    if (a.mc) cluster_sync();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    pdl_wait();  // S comes from the gate/up kernel

    if (warp == 0) {
        if (lane == 0) {
            const uint64_t ps = policy_evict_first();  // S: read once per column tile
            const uint64_t pw = policy_evict_last();   // W_down: re-read by every token tile
            int it = 0;
            PfSeg sg;
            for (int si = 0; pf_seg(c, si, G, a, sg); ++si) {
                const int tt = sg.tile / jw, jt = sg.tile % jw;
                for (int kb = sg.kb0; kb < sg.kb1; ++kb, ++it) {
                    const int s = it % a.stages;
                    if (it >= a.stages) mbar_wait(empty + s, ((it / a.stages) - 1) & 1);
                    uint8_t* st = smem + s * kPfStage;
                    mbar_arrive_expect_tx(full + s, kPfStage);
                    if (!a.mc) {
                        tma_load_2d(st, &m_s, kb * kBK, tt * kPfM, full + s, ps);
                        tma_load_2d(st + kABytes, &m_s, kb * kBK, tt * kPfM + kBM, full + s, ps);
                    } else {
                        const int h = c & 1;  // this CTA's half of the shared S boxes
                        tma_load_2d_mc(st + h * kABytes, &m_s, kb * kBK, tt * kPfM + h * kBM, full + s, 0x3, ps);
                    }
#pragma unroll
                    for (int q = 0; q < 4; ++q)
                        tma_load_2d(st + 2 * kABytes + q * (kBK * kBK * 2), &m_w, jt * kPfN + 64 * q, kb * kBK,
                                    full + s, pw);
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            // D[m][n] = sum_k S[m][k] W[k][n]: A K-major, B MN-major (bit 16), M = 128, N = 256
            const uint32_t idesc = idesc_bf16(kBM, kPfN) | (1u << 16);
            int it = 0;
            PfSeg sg;
            for (int si = 0; pf_seg(c, si, G, a, sg); ++si) {
                if (si >= 1) {
                    mbar_wait(tempty, (si - 1) & 1);  // the previous segment's accumulators drained
                    tc_fence_after();
                }
                for (int kb = sg.kb0; kb < sg.kb1; ++kb, ++it) {
                    const int s = it % a.stages;
                    mbar_wait(full + s, (it / a.stages) & 1);
                    tc_fence_after();
                    const uint32_t base = smem_u32(smem + s * kPfStage);
                    const uint64_t db = sw128_mn_desc(base + 2 * kABytes, kBK * kBK * 2);
#pragma unroll
                    for (int k = 0; k < kBK / 16; ++k) {
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            const uint64_t da = sw128_desc(base + h * kABytes);
                            // A: +32 B inside the swizzle atom per K=16; B: 16 K-rows of 128 B (+2 KB)
                            umma_bf16(tmem + h * kPfN, da + static_cast<uint64_t>(2 * k), db + static_cast<uint64_t>(128 * k),
                                      idesc, (kb > sg.kb0 || k > 0) ? 1u : 0u);
                        }
                    }
                    if (a.mc) umma_commit_mc(empty + s, 0x3);
                    else umma_commit(empty + s);
                }
                umma_commit(tfull);
            }
        }
    } else {
        // epilogue: warp w -> TMEM lanes 32 (w % 4) .. +31 (tokens) of accumulator h
        const int g = warp & 3;
        const int h = (warp - 2) >> 2;
        const uint32_t trow = tmem + (static_cast<uint32_t>(g * 32) << 16) + h * kPfN;
        PfSeg sg;
        for (int si = 0; pf_seg(c, si, G, a, sg); ++si) {
            mbar_wait(tfull, si & 1);
            tc_fence_after();
            const int tt = sg.tile / jw, jt = sg.tile % jw;
            const int64_t tok = static_cast<int64_t>(tt) * kPfM + h * kBM + g * 32 + lane;
            float* yrow = a.y + tok * a.d + jt * kPfN;
            const bool row_ok = tok < a.nb;
            const int ncols = min(kPfN, a.d - jt * kPfN);
            for (int cb = 0; cb < kPfN; cb += 16) {
                float v[16];
                tmem_ld16(trow + cb, v);
                tmem_wait_ld();
                if (row_ok && cb < ncols && (a.d & 3) != 0) {
#pragma unroll
                    for (int q = 0; q < 16; ++q) {
                        if (cb + q >= ncols) continue;
                        if (sg.whole) yrow[cb + q] = v[q];
                        else red_add_f32(yrow + cb + q, v[q]);
                    }
                } else if (row_ok && cb < ncols) {
                    if (sg.whole) {
#pragma unroll
                        for (int q = 0; q < 4; ++q)
                            if (cb + 4 * q < ncols)
                                *reinterpret_cast<float4*>(yrow + cb + 4 * q) = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
                    } else {
#pragma unroll
                        for (int q = 0; q < 4; ++q)
                            if (cb + 4 * q < ncols) red_add_v4(yrow + cb + 4 * q, v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
                    }
                }
            }
            tc_fence_before();
            mbar_arrive(tempty);
        }
    }
    __syncthreads();
    if (a.mc) cluster_sync();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512) : "memory");
    }
}

// Zero the blocks of y of the stream-K units >= first (tiles, or mc column-tile pairs):
// grid (units x 2, 8) x 256 threads.
__global__ void k_tc_zero_tiles(float* __restrict__ y, int nb, int d, int n_jt, int first, int mc) {
    const int ju = mc ? (n_jt + 1) / 2 : n_jt;
    const int u = first + blockIdx.x / 2;
    const int tt = u / ju;
    const int jt = mc ? 2 * (u % ju) + (blockIdx.x & 1) : u % ju;
    if ((!mc && (blockIdx.x & 1)) || jt >= n_jt) return;
    const int c0 = jt * kPfN, ncols = min(kPfN, d - c0);
    for (int r = blockIdx.y * 8 + threadIdx.x / 32; r < kPfM; r += gridDim.y * 8) {
        const int64_t tok = static_cast<int64_t>(tt) * kPfM + r;
        if (tok >= nb) break;
        for (int cc = threadIdx.x % 32; cc < ncols; cc += 32) y[tok * d + c0 + cc] = 0.0f;
    }
}

// ---------------------------------------------------------------- small element-wise kernels
__global__ void k_tc_fill_int(int* __restrict__ p, int64_t n, int v) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) p[i] = v;
}

__device__ __forceinline__ void split_store4(__nv_bfloat16* hi, __nv_bfloat16* lo, float4 v) {
    const __nv_bfloat162 h0 = __floats2bfloat162_rn(v.x, v.y), h1 = __floats2bfloat162_rn(v.z, v.w);
    const float2 f0 = __bfloat1622float2(h0), f1 = __bfloat1622float2(h1);
    const __nv_bfloat162 l0 = __floats2bfloat162_rn(v.x - f0.x, v.y - f0.y);
    const __nv_bfloat162 l1 = __floats2bfloat162_rn(v.z - f1.x, v.w - f1.y);
    uint2 hv, lv;
    hv.x = *reinterpret_cast<const uint32_t*>(&h0);
    hv.y = *reinterpret_cast<const uint32_t*>(&h1);
    lv.x = *reinterpret_cast<const uint32_t*>(&l0);
    lv.y = *reinterpret_cast<const uint32_t*>(&l1);
    *reinterpret_cast<uint2*>(hi) = hv;
    if (lo) *reinterpret_cast<uint2*>(lo) = lv;
}

// x (nb x d f32) -> xb (B-operand rows, ld elements, bf16).  split: sample b of n-tile t goes to
// rows t N + j (hi) and t N + nbt + j (lo), j = b % nbt.  Grid (ceil(d / 1024), nb), 256 threads,
// 4 columns per thread (d % 4 == 0; scalar otherwise).
__global__ void k_tc_pack_x(const float* __restrict__ x, int64_t d, int64_t ld, int split, int nbt,
                            __nv_bfloat16* __restrict__ xb) {
    const int64_t b = blockIdx.y;
    const int64_t r = split ? (b / nbt) * 2 * nbt + b % nbt : b;
    __nv_bfloat16* hi = xb + r * ld;
    __nv_bfloat16* lo = split ? xb + (r + nbt) * ld : nullptr;
    const float* xr = x + b * d;
    const int64_t c = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) * 4;
    if ((d & 3) == 0) {
        if (c < d) split_store4(hi + c, lo ? lo + c : nullptr, *reinterpret_cast<const float4*>(xr + c));
        return;
    }
    for (int64_t k = c; k < c + 4 && k < d; ++k) {
        const __nv_bfloat16 h = __float2bfloat16_rn(xr[k]);
        hi[k] = h;
        if (lo) lo[k] = __float2bfloat16_rn(xr[k] - __bfloat162float(h));
    }
}

}  // namespace

int64_t round_up64(int64_t v, int64_t m) { return (v + m - 1) / m * m; }

Plan plan_for(int64_t nb, int method) {
    Plan p;
    // Decode: pairs of bf16 (hi, lo) per activation, up to 64 samples per n-tile (UMMA N = 128).
    // Large dense batches (prefill): single bf16 activations, 256 tokens per n-tile (U and G fill
    // the 512 TMEM columns; N = 128 with double-buffered accumulators measured 1.27x slower,
    // 871 vs 685 us at 2048 tokens: the two MMAs per k-step then read 2 x 4 KB of B per 64
    // cycles, past the shared-memory port).
    p.split = !(method == kDense && nb > 256);
    if (p.split) {
        p.nbt = static_cast<int>(std::min<int64_t>(64, round_up64(nb, 16)));  // epilogue chunks of 16
        p.N = 2 * p.nbt;
    } else {
        p.nbt = 256;
        p.N = 256;
    }
    p.n_tiles = static_cast<int>((nb + p.nbt - 1) / p.nbt);
    p.rows = static_cast<int64_t>(p.n_tiles) * p.N;
    return p;
}

size_t workspace_bytes(const LayerDev& L, const Plan& p, int num_sms) {
    const int64_t ldr = L.ldr > 0 ? L.ldr : 8;
    size_t b = 0;
    b += round_up64(p.rows * L.ld * 2, 256);              // xb
    b += round_up64(p.rows * round_up64(L.F, 8) * 2, 256);  // s
    b += round_up64(p.rows * ldr * 2, 256);               // latent (pairs)
    b += round_up64(p.rows * ldr * 4, 256);               // latent f32 GEMM output
    b += round_up64(static_cast<int64_t>(num_sms) * 3 * p.N * kBM * 4, 256);  // stream-K partials
    return b;
}

cudaError_t launch_batched(const LayerDev& L, const Plan& p, void* ws, unsigned* flags, int method, int64_t nb,
                           const float* x, float tau, const uint8_t* ovr, float* y, uint8_t* mask_out,
                           float* ind_out, int* alive_out, const LaunchCfg& c) {
    if (L.dtype != 1 /* bf16 */ || !L.w_up) return cudaErrorInvalidValue;
    if (method == kDC && !ovr && !L.theta_bt) return cudaErrorInvalidValue;
    // decode (activations as bf16 pairs): one persistent kernel, kernels_tc_fused.cu
    if (p.split)
        return launch_batched_fused(L, p, ws, workspace_bytes(L, p, c.num_sms), flags, method, nb, x, tau, ovr, y,
                                    mask_out, ind_out, alive_out, c);
    // dense prefill: gate/up (k_tc_gateup, s as plain bf16 rows) then y = s W_down (k_tc_pf_down)
    if (method != kDense || ovr) return cudaErrorInvalidValue;
    const int64_t ld_s = round_up64(L.F, 8);
    uint8_t* w = static_cast<uint8_t*>(ws);
    auto take = [&](size_t bytes) {
        uint8_t* q = w;
        w += round_up64(static_cast<int64_t>(bytes), 256);
        return q;
    };
    auto* xb = reinterpret_cast<__nv_bfloat16*>(take(p.rows * L.ld * 2));
    auto* sb = reinterpret_cast<__nv_bfloat16*>(take(p.rows * ld_s * 2));
    const int64_t ldr = L.ldr > 0 ? L.ldr : 8;
    (void)take(p.rows * ldr * 2);
    (void)take(p.rows * ldr * 4);
    auto* ws_partial = reinterpret_cast<float*>(take(static_cast<size_t>(c.num_sms) * 3 * p.N * kBM * 4));

    cudaError_t e = cudaSuccess;
    k_tc_pack_x<<<dim3(static_cast<unsigned>((L.d + 1023) / 1024), static_cast<unsigned>(nb)), 256, 0, c.stream>>>(
        x, L.d, L.ld, 0, p.nbt, xb);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    // dense: every neuron is alive for every token -- the count is F, set here instead of the
    // epilogue's per-token ballots and atomics (7% of the gate/up kernel's stall samples)
    if (alive_out) {
        k_tc_fill_int<<<static_cast<unsigned>((nb + 255) / 256), 256, 0, c.stream>>>(alive_out, nb, static_cast<int>(L.F));
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
    }

    CUtensorMap m_up, m_gate, m_x;
    if (!make_map(&m_up, L.w_up, L.F, L.d, L.rs, kBM) || !make_map(&m_gate, L.w_gate, L.F, L.d, L.rs, kBM) ||
        !make_map(&m_x, xb, p.rows, L.d, L.ld, p.N))
        return cudaErrorInvalidValue;
    GateUpArgs a;
    a.F = static_cast<int>(L.F);
    a.nb = static_cast<int>(nb);
    a.nbt = p.nbt;
    a.N = p.N;
    a.kb_x = static_cast<int>((L.d + kBK - 1) / kBK);
    a.kb_z = 0;
    a.tau = tau;
    a.ovr = nullptr;
    a.s_out = sb;
    a.ld_s = ld_s;
    a.mask_out = mask_out;
    a.ind_out = ind_out;
    a.alive_out = nullptr;  // dense: filled above
    a.buf_cols = 2 * p.N;
    a.nbuf = 4 * p.N <= 512 ? 2 : 1;  // U and G double-buffered when they fit twice
    a.tmem_cols = a.nbuf * a.buf_cols <= 256 ? 256 : 512;
    if (a.nbuf * a.buf_cols > 512) return cudaErrorInvalidValue;
    a.n_tiles = p.n_tiles;
    a.tiles = static_cast<int>((L.F + kBM - 1) / kBM) * p.n_tiles;
    a.tl = nullptr;
    a.dp = 1;
    a.mc = 1;
    const int grid = std::min(c.num_sms, kMaxCtas) & ~1;  // pairs of CTAs (2-CTA clusters)
    a.ws = ws_partial;
    a.flags = flags;
    const int stage_bytes = 2 * kABytes + p.N * kBK * 2;
    const size_t fixed = 1024 + 256;
    a.stages = static_cast<int>(std::min<size_t>(8, (kMaxDynSmem - fixed) / stage_bytes));
    const size_t smem = fixed + static_cast<size_t>(a.stages) * stage_bytes;
    auto fn = L.act == 0 ? k_tc_gateup<kDense, false, 0> : k_tc_gateup<kDense, false, 1>;
    if ((e = set_smem(fn, smem)) != cudaSuccess) return e;
    CUtensorMap m_tb = m_up, m_lat = m_x;
    if ((e = launch_ex_cluster(fn, dim3(grid), dim3(kThreads), smem, c, false, 2u, m_up, m_gate, m_x, m_tb, m_lat,
                               a)) != cudaSuccess)
        return e;

    // y = s W_down (W_down rows are the third part of each neuron record, stride rs)
    PfDownArgs b;
    b.nb = static_cast<int>(nb);
    b.d = static_cast<int>(L.d);
    b.nkb = static_cast<int>((L.F + kBK - 1) / kBK);
    b.n_tt = static_cast<int>((nb + kPfM - 1) / kPfM);
    b.n_jt = static_cast<int>((L.d + kPfN - 1) / kPfN);
    const int dgrid = std::min(c.num_sms, kMaxCtas) & ~1;
    b.mc = 1;
    const int W = dgrid / 2;
    const int dunits = b.n_tt * ((b.n_jt + 1) / 2);
    b.n_full = dunits / W * W;
    b.y = y;
    b.stages = static_cast<int>(std::min<size_t>(4, (kMaxDynSmem - fixed) / kPfStage));
    const size_t dsmem = fixed + static_cast<size_t>(b.stages) * kPfStage;
    CUtensorMap m_s, m_w;
    if (!make_map(&m_s, sb, p.rows, L.F, ld_s, kBM) || !make_map(&m_w, L.w_down, L.F, L.d, L.rs, kBK))
        return cudaErrorInvalidValue;
    if (dunits > b.n_full) {
        k_tc_zero_tiles<<<dim3(static_cast<unsigned>(2 * (dunits - b.n_full)), 8), 256, 0, c.stream>>>(
            y, b.nb, b.d, b.n_jt, b.n_full, b.mc);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
    }
    if ((e = set_smem(k_tc_pf_down, dsmem)) != cudaSuccess) return e;
    return launch_ex_cluster(k_tc_pf_down, dim3(dgrid), dim3(kThreads), dsmem, c, true, 2u, m_s, m_w, b);
}

}  // namespace tc
}  // namespace cdk
