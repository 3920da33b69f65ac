// kernels_tc_fused.cu -- the batched decode step (B >= 8, bf16 hi/lo activation pairs) as ONE
// persistent tensor-core kernel: one CTA per SM, one continuous TMA -> smem -> tcgen05.mma ring.
//
//   phase 0 (D-CountDown only): latent = x theta_a, split-K over all CTAs (A = theta_a^T tiles,
//            B = x pairs), partials reduced with red.add into an f32 latent; the last CTA to
//            arrive re-splits it into bf16 (hi, lo) pairs and releases a flag.
//   phase A: U = W_up x^T, G = W_gate x^T (+ Z = theta_b^T latent^T, the predictor blocks placed
//            LAST in each tile so the latent is long ready), stream-K over all CTAs; the tile
//            finisher applies the per-sample mask and writes s as bf16 pairs (kernels_tc.cu
//            k_tc_gateup describes the schedule).
//   phase B: y += s W_down (A = W_down^T MN-major, hi and lo s rows into one accumulator),
//            stream-K, red.add into y.  Its W_down boxes do not depend on s, so the producer
//            streams them into the ring while the last phase-A epilogues finish; only the s boxes
//            wait for the grid-wide "s complete" count.
//
// Versus three launches (pack, gate/up, down): no launch gaps, the gate/up epilogue tail and the
// latent GEMM are hidden behind weight streaming.  Grid-wide waits need every CTA resident
// (grid = SMs, one CTA per SM, no other work on the device from this stream).
#include <cstdlib>

#include "kernels.h"
#include "kernels_tc.h"
#include "launch.cuh"
#include "tc_common.cuh"

namespace cdk {
namespace tc {
namespace {

constexpr int kDJF = 2;  // phase B: 128-column j sub-tiles per tile (sharing the s box)
constexpr int kOvrF = 4;

// control words (after the per-CTA partial flags)
constexpr int kWLatCount = kMaxCtas + 0;  // phase-0 arrivals
constexpr int kWLatReady = kMaxCtas + 1;  // latent pairs written
constexpr int kWSCount = kMaxCtas + 2;    // phase-A arrivals (s complete when == grid)
constexpr int kWEndCount = kMaxCtas + 3;  // phase-B arrivals (the last one resets the words)

struct FusedArgs {
    int F, d, r, nb, nbt, N, n_tiles;
    int mt0, mta, jt;    // m-tiles of phase 0 (latent rows), phase A (neurons), phase B j-tiles (256 wide)
    int kb_x, kb_z, kb_f;  // k-blocks over d, r (0 unless D-CountDown), F
    int stages, tmem_cols;
    int pb_pf;  // phase-B W_down k-blocks prefetched into L2 beyond the ring
    float tau;
    const uint8_t* ovr;
    __nv_bfloat16* s_out;
    int64_t ld_s;
    uint8_t* mask_out;
    float* ind_out;
    int* alive_out;
    float* ws;
    unsigned* flags;
    float* y;
    float* lat32;
    __nv_bfloat16* latb;
    int64_t ldr;
    unsigned long long* tl;  // development: per-CTA globaltimer stamps (8 per CTA) or null
};

__device__ __forceinline__ void fstamp(const FusedArgs& a, int k) {
    if (a.tl) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        a.tl[blockIdx.x * 8 + k] = t;
    }
}

__device__ __forceinline__ void fence_proxy_async_global() {
    asm volatile("fence.proxy.async.global;" ::: "memory");
}

__device__ __forceinline__ void spin_until_geq(const unsigned* p, unsigned v) {
    while (ld_acquire_u32(p) < v) {
    }
}

constexpr int kThreadsF = kThreads + 32;  // + one latent helper warp

template <int KIND, int ACT>
__global__ void __launch_bounds__(kThreadsF, 1)
k_tc_fused(const __grid_constant__ CUtensorMap m_up, const __grid_constant__ CUtensorMap m_gate,
           const __grid_constant__ CUtensorMap m_x, const __grid_constant__ CUtensorMap m_tb,
           const __grid_constant__ CUtensorMap m_lat, const __grid_constant__ CUtensorMap m_ta,
           const __grid_constant__ CUtensorMap m_w, const __grid_constant__ CUtensorMap m_s, const FusedArgs a) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    constexpr bool kZ = KIND == kDC;
    const int N = a.N, nbt = a.nbt;
    const int bbytes = N * kBK * 2;  // B box (x / latent / s pairs): N rows of 128 B
    const int stage_bytes = 2 * kABytes + bbytes;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + a.stages * stage_bytes);
    uint64_t* empty = full + a.stages;
    uint64_t* tfull = empty + a.stages;
    uint64_t* tempty = tfull + 1;
    uint64_t* pbar = tempty + 1;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(pbar + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int G = gridDim.x, c = blockIdx.x;
    // phases: units U_p = tiles_p x nkb_p, split evenly over the CTAs
    const int nkb0 = a.kb_x, nkbA = a.kb_x + a.kb_z, nkbB = a.kb_f;
    const int tiles0 = kZ ? a.mt0 * a.n_tiles : 0, tilesA = a.mta * a.n_tiles, tilesB = a.jt * a.n_tiles;
    const int64_t U0 = static_cast<int64_t>(tiles0) * nkb0, UA = static_cast<int64_t>(tilesA) * nkbA,
                  UB = static_cast<int64_t>(tilesB) * nkbB;

    if (warp == 0 && lane == 0) {
        for (int s = 0; s < a.stages; ++s) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, 1);
        }
        mbar_init(tfull, 1);
        mbar_init(tempty, kEpiThreads);
        mbar_init(pbar, 1);
        fence_mbar_init();
        prefetch_map(&m_up);
        prefetch_map(&m_gate);
        prefetch_map(&m_x);
        prefetch_map(&m_w);
        prefetch_map(&m_s);
        if (kZ) {
            prefetch_map(&m_tb);
            prefetch_map(&m_lat);
            prefetch_map(&m_ta);
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
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    if (threadIdx.x == 0) fstamp(a, 0);

    if (warp == 0) {
        if (lane == 0) {
            // ================= TMA producer
            const uint64_t pw = policy_evict_first();
            const uint64_t px = policy_evict_last();
            int it = 0;
            auto acquire_stage = [&]() -> uint8_t* {
                const int s = it % a.stages;
                if (it >= a.stages) mbar_wait(empty + s, ((it / a.stages) - 1) & 1);
                return smem + s * stage_bytes;
            };
            Seg sg;
            if (kZ) {
                for (int si = 0; seg_at(c, si, U0, G, nkb0, sg); ++si) {
                    const int m0 = (sg.tile / a.n_tiles) * kBM, row0 = (sg.tile % a.n_tiles) * N;
                    for (int kb = sg.kb0; kb < sg.kb1; ++kb, ++it) {
                        uint8_t* st = acquire_stage();
                        uint64_t* fb = full + it % a.stages;
                        mbar_arrive_expect_tx(fb, kABytes + bbytes);
                        tma_load_2d(st, &m_ta, kb * kBK, m0, fb, pw);
                        tma_load_2d(st + 2 * kABytes, &m_x, kb * kBK, row0, fb, px);
                    }
                }
            }
            bool lat_ready = !kZ;
            for (int si = 0; seg_at(c, si, UA, G, nkbA, sg); ++si) {
                const int m0 = (sg.tile / a.n_tiles) * kBM, row0 = (sg.tile % a.n_tiles) * N;
                for (int kb = sg.kb0; kb < sg.kb1; ++kb, ++it) {
                    uint8_t* st = acquire_stage();
                    uint64_t* fb = full + it % a.stages;
                    if (kb < a.kb_x) {
                        mbar_arrive_expect_tx(fb, 2 * kABytes + bbytes);
                        tma_load_2d(st, &m_up, kb * kBK, m0, fb, pw);
                        tma_load_2d(st + kABytes, &m_gate, kb * kBK, m0, fb, pw);
                        tma_load_2d(st + 2 * kABytes, &m_x, kb * kBK, row0, fb, px);
                    } else {
                        if (!lat_ready) {
                            spin_until_geq(a.flags + kWLatReady, static_cast<unsigned>(G));
                            fence_proxy_async_global();
                            lat_ready = true;
                        }
                        const int kz = (kb - a.kb_x) * kBK;
                        mbar_arrive_expect_tx(fb, kABytes + bbytes);
                        tma_load_2d(st, &m_tb, kz, m0, fb, pw);
                        tma_load_2d(st + 2 * kABytes, &m_lat, kz, row0, fb, px);
                    }
                }
            }
            // phase B: W_down boxes right away, the s boxes once every CTA has written its s
            bool s_ready = false;
            int pend_it[16], pend_kb[16], pend_row[16], npend = 0;
            auto flush = [&]() {
                fstamp(a, 2);
                spin_until_geq(a.flags + kWSCount, static_cast<unsigned>(G));
                fstamp(a, 3);
                fence_proxy_async_global();
                s_ready = true;
                for (int q = 0; q < npend; ++q) {
                    const int s = pend_it[q] % a.stages;
                    tma_load_2d(smem + s * stage_bytes + 2 * kABytes, &m_s, pend_kb[q] * kBK, pend_row[q], full + s, px);
                }
                npend = 0;
            };
            // L2 look-ahead: the W_down boxes of the k-blocks right after the ring's depth, so the HBM
            // keeps streaming while the phase-A epilogues finish
            {
                int q = 0;
                for (int si = 0; q < a.stages + a.pb_pf && seg_at(c, si, UB, G, nkbB, sg); ++si) {
                    const int j0 = (sg.tile / a.n_tiles) * kDJF * kBM;
                    for (int kb = sg.kb0; kb < sg.kb1 && q < a.stages + a.pb_pf; ++kb, ++q)
                        if (q >= a.stages)
                            for (int b4 = 0; b4 < 2 * kDJF; ++b4) tma_prefetch_l2_2d(&m_w, j0 + 64 * b4, kb * kBK);
                }
            }
            for (int si = 0; seg_at(c, si, UB, G, nkbB, sg); ++si) {
                const int j0 = (sg.tile / a.n_tiles) * kDJF * kBM, row0 = (sg.tile % a.n_tiles) * N;
                for (int kb = sg.kb0; kb < sg.kb1; ++kb, ++it) {
                    // (a stage still holding a pending s box is never re-acquired: the ring
                    // flushes when every stage is pending)
                    const int s = it % a.stages;
                    uint8_t* st = acquire_stage();
                    uint64_t* fb = full + s;
                    mbar_arrive_expect_tx(fb, 2 * kABytes + bbytes);
#pragma unroll
                    for (int q = 0; q < 2 * kDJF; ++q)
                        tma_load_2d(st + q * (kBK * kBK * 2), &m_w, j0 + 64 * q, kb * kBK, fb, pw);
                    if (s_ready) {
                        tma_load_2d(st + 2 * kABytes, &m_s, kb * kBK, row0, fb, px);
                    } else {
                        pend_it[npend] = it;
                        pend_kb[npend] = kb;
                        pend_row[npend] = row0;
                        if (++npend == a.stages || npend == 16) flush();
                    }
                }
            }
            if (!s_ready && npend) flush();
        }
    } else if (warp == 1) {
        if (lane == 0) {
            // ================= MMA issuer (one segment at a time in TMEM)
            int it = 0, gs = 0;
            Seg sg;
            auto begin_seg = [&]() {
                if (gs > 0) {
                    mbar_wait(tempty, (gs - 1) & 1);
                    tc_fence_after();
                }
            };
            auto stage_base = [&]() -> uint32_t {
                const int s = it % a.stages;
                mbar_wait(full + s, (it / a.stages) & 1);
                tc_fence_after();
                return smem_u32(smem + s * stage_bytes);
            };
            const uint32_t idA = idesc_bf16(kBM, N);
            if (kZ) {
                for (int si = 0; seg_at(c, si, U0, G, nkb0, sg); ++si, ++gs) {
                    begin_seg();
                    for (int kb = sg.kb0; kb < sg.kb1; ++kb, ++it) {
                        const uint32_t base = stage_base();
                        const uint64_t da = sw128_desc(base), db = sw128_desc(base + 2 * kABytes);
#pragma unroll
                        for (int k = 0; k < kBK / 16; ++k)
                            umma_bf16(tmem, da + 2 * k, db + 2 * k, idA, (kb > sg.kb0 || k > 0) ? 1u : 0u);
                        umma_commit(empty + it % a.stages);
                    }
                    umma_commit(tfull);
                }
            }
            for (int si = 0; seg_at(c, si, UA, G, nkbA, sg); ++si, ++gs) {
                begin_seg();
                const int first_z = max(sg.kb0, a.kb_x);
                for (int kb = sg.kb0; kb < sg.kb1; ++kb, ++it) {
                    const uint32_t base = stage_base();
                    const uint64_t da0 = sw128_desc(base), da1 = sw128_desc(base + kABytes),
                                   db = sw128_desc(base + 2 * kABytes);
#pragma unroll
                    for (int k = 0; k < kBK / 16; ++k) {
                        const uint64_t o = static_cast<uint64_t>(2 * k);
                        if (kb < a.kb_x) {
                            const uint32_t acc = (kb > sg.kb0 || k > 0) ? 1u : 0u;
                            umma_bf16(tmem, da0 + o, db + o, idA, acc);
                            umma_bf16(tmem + N, da1 + o, db + o, idA, acc);
                        } else {
                            umma_bf16(tmem + 2 * N, da0 + o, db + o, idA, (kb > first_z || k > 0) ? 1u : 0u);
                        }
                    }
                    umma_commit(empty + it % a.stages);
                }
                umma_commit(tfull);
            }
            fstamp(a, 1);
            const uint32_t idB = idesc_bf16(kBM, nbt) | (1u << 15);
            for (int si = 0; seg_at(c, si, UB, G, nkbB, sg); ++si, ++gs) {
                begin_seg();
                for (int kb = sg.kb0; kb < sg.kb1; ++kb, ++it) {
                    const uint32_t base = stage_base();
                    const uint64_t dbh = sw128_desc(base + 2 * kABytes);
                    const uint64_t dbl = sw128_desc(base + 2 * kABytes + nbt * kBK * 2);
#pragma unroll
                    for (int q = 0; q < kDJF; ++q) {
                        const uint64_t da = sw128_mn_desc(base + q * kABytes, kBK * kBK * 2);
#pragma unroll
                        for (int k = 0; k < kBK / 16; ++k) {
                            const uint64_t oa = static_cast<uint64_t>(128 * k), ob = static_cast<uint64_t>(2 * k);
                            umma_bf16(tmem + q * nbt, da + oa, dbh + ob, idB, (kb > sg.kb0 || k > 0) ? 1u : 0u);
                            umma_bf16(tmem + q * nbt, da + oa, dbl + ob, idB, 1u);
                        }
                    }
                    umma_commit(empty + it % a.stages);
                }
                umma_commit(tfull);
            }
        }
    } else if (warp < 2 + kEpiWarps) {
        // ================= epilogue warps
        const int g = warp & 3;
        const int half = (warp - 2) >> 2;
        const int m = g * 32 + lane;
        const int et = threadIdx.x - 64;
        const uint32_t trow = tmem + (static_cast<uint32_t>(g * 32) << 16);
        constexpr int kParts = kZ ? 3 : 2;
        constexpr int kC = 8;
        const int hb = nbt / 2;
        int gs = 0;
        Seg sg;
        auto wait_seg = [&]() {
            mbar_wait(tfull, gs & 1);
            tc_fence_after();
        };
        auto done_seg = [&]() {
            tc_fence_before();
            mbar_arrive(tempty);
            ++gs;
        };
        // ---- phase 0: latent partials -> red.add into lat32 [sample][ldr]
        if (kZ) {
            for (int si = 0; seg_at(c, si, U0, G, nkb0, sg); ++si) {
                wait_seg();
                const int jr = (sg.tile / a.n_tiles) * kBM + m;
                const int64_t gb0 = static_cast<int64_t>(sg.tile % a.n_tiles) * nbt;
                for (int cb = half * hb; cb < (half + 1) * hb; cb += kC) {
                    float v[kC], w[kC];
                    tmem_ld8(trow + cb, v);
                    tmem_ld8(trow + nbt + cb, w);
                    tmem_wait_ld();
                    if (jr < a.r) {
#pragma unroll
                        for (int j = 0; j < kC; ++j)
                            if (gb0 + cb + j < a.nb) red_add_f32(a.lat32 + (gb0 + cb + j) * a.ldr + jr, v[j] + w[j]);
                    }
                }
                done_seg();
            }
            // this CTA's latent partials are in: count it (the helper warp re-splits once every
            // CTA has counted -- the epilogue goes straight on to phase A and keeps TMEM moving)
            __threadfence();
            named_bar_sync(1, kEpiThreads);
            if (et == 0) atomicAdd(a.flags + kWLatCount, 1u);
        }
        // ---- phase A: gate/up tiles (contributors park partials, finishers apply the masks)
        for (int si = 0; seg_at(c, si, UA, G, nkbA, sg); ++si) {
            // Finisher of a split tile: its contributors parked their partials long ago (their
            // first segments), so pull them into free TMEM columns now, while this segment's MMAs
            // still run -- the epilogue then reads them from TMEM instead of walking a chain of
            // global round trips after the last k-block (the phase A -> B gap).
            int c_last = c;
            bool staged = false;
            uint32_t pb = 0;
            bool pz = false;  // the finisher holds Z: the contributors hold only Z (one column block)
            if (sg.kb0 == 0) {
                const int64_t tb = static_cast<int64_t>(sg.tile) * nkbA;
                while (c_last + 1 < G && range_lo(c_last + 1, UA, G) < tb + nkbA) ++c_last;
                if (c_last > c) {
                    if (et == 0) {
                        for (int cc = c + 1; cc <= c_last; ++cc) {
                            if (range_lo(cc, UA, G) == range_lo(cc + 1, UA, G)) continue;  // empty range
                            unsigned* f = a.flags + cc;
                            while (ld_acquire_u32(f) == 0u) {
                            }
                            *f = 0u;  // consumed: ready for the next launch
                        }
                    }
                    __threadfence();
                    named_bar_sync(1, kEpiThreads);
                    pz = kZ && sg.kb1 > a.kb_x;
                    pb = static_cast<uint32_t>((pz ? 3 : 2) * N);
                    staged = pb + static_cast<uint32_t>(kParts * nbt) <= static_cast<uint32_t>(a.tmem_cols);
                    if (staged) {
                        const int64_t slot_floats = static_cast<int64_t>(kParts) * nbt * kBM;
                        const int sb0 = half * hb;
#pragma unroll
                        for (int q = 0; q < kParts; ++q) {
                            if (pz && q != 2) continue;
                            // the whole half (<= 32 samples) of this row per contributor: all
                            // loads in flight at once (coalesced: [part][sample][row] slots)
                            float v[32];
#pragma unroll
                            for (int j = 0; j < 32; ++j) v[j] = 0.0f;
                            for (int cc = c + 1; cc <= c_last; ++cc) {
                                const int64_t q0 = range_lo(cc, UA, G) - tb, q1 = range_lo(cc + 1, UA, G) - tb;
                                if (q0 == q1 || (q == 2 ? !(q1 > a.kb_x) : !(q0 < a.kb_x))) continue;
                                const float* src = a.ws + cc * slot_floats + (static_cast<int64_t>(q) * nbt + sb0) * kBM + m;
#pragma unroll
                                for (int j = 0; j < 32; ++j)
                                    if (j < hb) v[j] += __ldcg(src + static_cast<int64_t>(j) * kBM);
                            }
#pragma unroll
                            for (int k = 0; k < 4; ++k) {
                                if (k * kC >= hb) break;
                                float v8[kC];
#pragma unroll
                                for (int j = 0; j < kC; ++j) v8[j] = v[k * kC + j];
                                tmem_st8(trow + pb + (pz ? 0u : static_cast<uint32_t>(q * nbt)) + sb0 + k * kC, v8);
                            }
                        }
                        tmem_wait_st();
                    }
                }
            }
            wait_seg();
            if (et == 0 && sg.kb0 == 0) fstamp(a, 7);
            const bool has_z = kZ && sg.kb1 > a.kb_x;
            const bool has_ug = sg.kb0 < a.kb_x;
            const int64_t slot_floats = static_cast<int64_t>(kParts) * nbt * kBM;
            if (sg.kb0 > 0) {
                float* slot = a.ws + static_cast<int64_t>(c) * slot_floats;
                for (int q = 0; q < kParts; ++q) {
                    if (q == 2 ? !has_z : !has_ug) continue;
                    for (int c0 = half * 16; c0 < nbt; c0 += 32) {
                        float v[16], w[16];
                        tmem_ld16(trow + q * N + c0, v);
                        tmem_ld16(trow + q * N + nbt + c0, w);
                        tmem_wait_ld();
                        // slot layout [part][sample][row]: a warp's stores are 128 consecutive bytes
                        float* dst = slot + (static_cast<int64_t>(q) * nbt + c0) * kBM + m;
#pragma unroll
                        for (int j = 0; j < 16; ++j) dst[static_cast<int64_t>(j) * kBM] = v[j] + w[j];
                    }
                }
                done_seg();
                __threadfence();
                named_bar_sync(1, kEpiThreads);
                if (et == 0) st_release_u32(a.flags + c, 1u);
                continue;
            }
            const int tile = sg.tile;
            const int64_t tile_base = static_cast<int64_t>(tile) * nkbA;
            // contributors (the following CTAs whose non-empty ranges start inside this tile):
            // their flags were consumed above, their partials staged in TMEM when they fit
            if (et == 0) fstamp(a, 6);
            const int i = (tile / a.n_tiles) * kBM + m;
            const bool valid = i < a.F;
            const int ntile = tile % a.n_tiles;
            const int64_t F = a.F, ld_s = a.ld_s;
            const int64_t gb0 = static_cast<int64_t>(ntile) * nbt;
            const int nlive = a.nb - gb0 < nbt ? static_cast<int>(a.nb - gb0) : nbt;
            const int sb0 = half * hb;
            __nv_bfloat16* s_hi = a.s_out + (static_cast<int64_t>(ntile) * N + sb0) * ld_s + i;
            const int64_t lo_step = static_cast<int64_t>(nbt) * ld_s;
            // contributor partials ([part][row][sample] slots), one chunk ahead of their use
            float4 pre[kParts][2];
            auto load_partials = [&](int cb, float4 (&d)[kParts][2]) {
#pragma unroll
                for (int q = 0; q < kParts; ++q) d[q][0] = d[q][1] = make_float4(0.f, 0.f, 0.f, 0.f);
                for (int cc = c + 1; cc <= c_last; ++cc) {
                    const int64_t q0 = range_lo(cc, UA, G) - tile_base;
                    const int64_t q1 = range_lo(cc + 1, UA, G) - tile_base;
                    if (q0 == q1) continue;  // empty range
                    const float* gp = a.ws + cc * slot_floats + static_cast<int64_t>(cb) * kBM + m;
#pragma unroll
                    for (int q = 0; q < kParts; ++q) {
                        if (q == 2 ? !(q1 > a.kb_x) : !(q0 < a.kb_x)) continue;
                        const float* p = gp + static_cast<int64_t>(q) * nbt * kBM;  // [part][sample][row]
                        d[q][0].x += __ldcg(p); d[q][0].y += __ldcg(p + kBM);
                        d[q][0].z += __ldcg(p + 2 * kBM); d[q][0].w += __ldcg(p + 3 * kBM);
                        d[q][1].x += __ldcg(p + 4 * kBM); d[q][1].y += __ldcg(p + 5 * kBM);
                        d[q][1].z += __ldcg(p + 6 * kBM); d[q][1].w += __ldcg(p + 7 * kBM);
                    }
                }
            };
            if (c_last > c && !staged) load_partials(sb0, pre);
            for (int cb = sb0; cb < sb0 + hb; cb += kC, s_hi += kC * ld_s) {
                float acc[kParts][2][kC];
#pragma unroll
                for (int q = 0; q < kParts; ++q) {
                    const bool own = q == 2 ? has_z : has_ug;
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        if (own) {
                            tmem_ld8(trow + q * N + h * nbt + cb, acc[q][h]);
                        } else {
#pragma unroll
                            for (int j = 0; j < kC; ++j) acc[q][h][j] = 0.0f;
                        }
                    }
                }
                if (staged) {
                    float pv[kParts][kC];
#pragma unroll
                    for (int q = 0; q < kParts; ++q) {
                        if (pz && q != 2) continue;
                        tmem_ld8(trow + pb + (pz ? 0u : static_cast<uint32_t>(q * nbt)) + cb, pv[q]);
                    }
                    tmem_wait_ld();
#pragma unroll
                    for (int q = 0; q < kParts; ++q) {
                        if (pz && q != 2) continue;
#pragma unroll
                        for (int j = 0; j < kC; ++j) acc[q][0][j] += pv[q][j];
                    }
                } else if (c_last > c) {
                    float4 cur[kParts][2];
#pragma unroll
                    for (int q = 0; q < kParts; ++q) cur[q][0] = pre[q][0], cur[q][1] = pre[q][1];
                    if (cb + kC < sb0 + hb) load_partials(cb + kC, pre);
                    tmem_wait_ld();
#pragma unroll
                    for (int q = 0; q < kParts; ++q) {
                        acc[q][0][0] += cur[q][0].x; acc[q][0][1] += cur[q][0].y;
                        acc[q][0][2] += cur[q][0].z; acc[q][0][3] += cur[q][0].w;
                        acc[q][0][4] += cur[q][1].x; acc[q][0][5] += cur[q][1].y;
                        acc[q][0][6] += cur[q][1].z; acc[q][0][7] += cur[q][1].w;
                    }
                } else {
                    tmem_wait_ld();
                }
                unsigned on_bits = 0;
                __nv_bfloat16* p = s_hi;
#pragma unroll
                for (int j = 0; j < kC; ++j, p += ld_s) {
                    const float u = acc[0][0][j] + acc[0][1][j];
                    const float gg = acc[1][0][j] + acc[1][1][j];
                    const float z = kZ ? acc[kParts - 1][0][j] + acc[kParts - 1][1][j] : 0.0f;
                    const bool live = valid && cb + j < nlive;
                    const float ag = act_epi(ACT, gg);
                    bool on;
                    if constexpr (KIND == kDC) {
                        on = z > a.tau;
                    } else if constexpr (KIND == kMC) {
                        on = fabsf(u) > a.tau;
                    } else if constexpr (KIND == kCATS) {
                        on = fabsf(ag) > a.tau;
                    } else if constexpr (KIND == kOvrF) {
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
                        p[lo_step] = __float2bfloat16_rn(sv - __bfloat162float(hv));
                        if (a.ind_out) a.ind_out[(gb0 + cb + j) * F + i] = KIND == kDC ? z : KIND == kCATS ? ag : u;
                    }
                }
                if (valid && a.mask_out) {
                    for (int j = 0; j < kC && cb + j < nlive; ++j)
                        a.mask_out[(gb0 + cb + j) * F + i] = (on_bits >> j) & 1u;
                }
                if (a.alive_out) {
#pragma unroll
                    for (int j = 0; j < kC; ++j) {
                        const unsigned bal = __ballot_sync(0xffffffffu, (on_bits >> j) & 1u);
                        if (lane == j && bal) atomicAdd(a.alive_out + gb0 + cb + j, __popc(bal));
                    }
                }
            }
            done_seg();
        }
        // s written by this CTA: make it visible to every CTA's TMA (async proxy) reads
        fence_proxy_async_global();
        __threadfence();
        named_bar_sync(1, kEpiThreads);
        if (et == 0) {
            __threadfence();
            atomicAdd(a.flags + kWSCount, 1u);
            fstamp(a, 4);
        }
        // ---- phase B: y += partial (red.add), sub-tile `half`
        for (int si = 0; seg_at(c, si, UB, G, nkbB, sg); ++si) {
            wait_seg();
            const int j = (sg.tile / a.n_tiles) * kDJF * kBM + half * kBM + m;
            const int64_t gb0 = static_cast<int64_t>(sg.tile % a.n_tiles) * nbt;
            for (int cb = 0; cb < nbt; cb += kC) {
                float v[kC];
                tmem_ld8(trow + half * nbt + cb, v);
                tmem_wait_ld();
                if (j < a.d) {
#pragma unroll
                    for (int t = 0; t < kC; ++t)
                        if (gb0 + cb + t < a.nb) red_add_f32(a.y + (gb0 + cb + t) * a.d + j, v[t]);
                }
            }
            done_seg();
        }
        named_bar_sync(1, kEpiThreads);
        if (et == 0) fstamp(a, 5);
        tc_fence_before();
    } else if (kZ) {
        // ================= latent helper warp: once every CTA's phase-0 partials are in, re-split
        // this CTA's slice of the f32 latent into the bf16 pairs the predictor blocks read
        if (lane == 0) spin_until_geq(a.flags + kWLatCount, static_cast<unsigned>(G));
        __syncwarp();
        __threadfence();
        const int64_t n = static_cast<int64_t>(a.nb) * a.r;
        for (int64_t e = c * n / G + lane; e < (c + 1) * n / G; e += 32) {
            const int64_t b = e / a.r, jr = e - b * a.r;
            const float v = __ldcg(a.lat32 + b * a.ldr + jr);
            const int64_t row = (b / nbt) * N + b % nbt;
            const __nv_bfloat16 h = __float2bfloat16_rn(v);
            a.latb[row * a.ldr + jr] = h;
            a.latb[(row + nbt) * a.ldr + jr] = __float2bfloat16_rn(v - __bfloat162float(h));
        }
        fence_proxy_async_global();
        __threadfence();
        __syncwarp();
        if (lane == 0) atomicAdd(a.flags + kWLatReady, 1u);
    }
    __syncthreads();
    if (threadIdx.x == 0 && atomicAdd(a.flags + kWEndCount, 1u) == static_cast<unsigned>(G - 1)) {
        // every warp of every CTA is past all its waits: reset the control words for the next launch
        a.flags[kWLatCount] = 0u;
        a.flags[kWLatReady] = 0u;
        a.flags[kWSCount] = 0u;
        a.flags[kWEndCount] = 0u;
    }
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(a.tmem_cols) : "memory");
    }
}

// x -> bf16 pairs; zero y, alive, the f32 latent.  Grid (ceil(max(d, ldr) / 1024), nb).
__global__ void k_tc_prep(const float* __restrict__ x, int64_t d, int64_t ld, int nbt, __nv_bfloat16* __restrict__ xb,
                          float* __restrict__ y, int* __restrict__ alive, float* __restrict__ lat32, int64_t ldr) {
    const int64_t b = blockIdx.y;
    const int64_t r = (b / nbt) * 2 * nbt + b % nbt;
    const int64_t c = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) * 4;
    if (c < d) {
        const float* xr = x + b * d;
        __nv_bfloat16* hi = xb + r * ld;
        __nv_bfloat16* lo = xb + (r + nbt) * ld;
        for (int64_t k = c; k < c + 4 && k < d; ++k) {
            const __nv_bfloat16 h = __float2bfloat16_rn(xr[k]);
            hi[k] = h;
            lo[k] = __float2bfloat16_rn(xr[k] - __bfloat162float(h));
            y[b * d + k] = 0.0f;
        }
    }
    if (lat32)
        for (int64_t k = c; k < c + 4 && k < ldr; ++k) lat32[b * ldr + k] = 0.0f;
    if (alive && blockIdx.x == 0 && threadIdx.x == 0) alive[b] = 0;
}

}  // namespace

cudaError_t launch_batched_fused(const LayerDev& L, const Plan& p, void* ws_base, size_t ws_bytes, unsigned* flags,
                                 int method, int64_t nb, const float* x, float tau, const uint8_t* ovr, float* y,
                                 uint8_t* mask_out, float* ind_out, int* alive_out, const LaunchCfg& c) {
    if (!p.split || L.dtype != 1 || !L.w_up) return cudaErrorInvalidValue;
    const bool dc_pred = method == kDC && !ovr;
    if (dc_pred && (!L.theta_bt || !L.theta_at)) return cudaErrorInvalidValue;
    const int64_t ldr = L.ldr > 0 ? L.ldr : 8;
    const int64_t ld_s = (L.F + 7) / 8 * 8;
    const int G = std::min(c.num_sms, kMaxCtas);
    uint8_t* w = static_cast<uint8_t*>(ws_base);
    size_t used = 0;
    auto take = [&](size_t bytes) {
        uint8_t* q = w + used;
        used += (bytes + 255) / 256 * 256;
        return q;
    };
    auto* xb = reinterpret_cast<__nv_bfloat16*>(take(p.rows * L.ld * 2));
    auto* sb = reinterpret_cast<__nv_bfloat16*>(take(p.rows * ld_s * 2));
    auto* latb = reinterpret_cast<__nv_bfloat16*>(take(p.rows * ldr * 2));
    auto* lat32 = reinterpret_cast<float*>(take(nb * ldr * 4));
    auto* part = reinterpret_cast<float*>(take(static_cast<size_t>(G) * 3 * p.nbt * kBM * 4));
    if (used > ws_bytes) return cudaErrorInvalidValue;

    cudaError_t e;
    const int64_t cols = std::max<int64_t>(L.d, dc_pred ? ldr : 0);
    k_tc_prep<<<dim3(static_cast<unsigned>((cols + 1023) / 1024), static_cast<unsigned>(nb)), 256, 0, c.stream>>>(
        x, L.d, L.ld, p.nbt, xb, y, alive_out, dc_pred ? lat32 : nullptr, ldr);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;

    CUtensorMap m_up, m_gate, m_x, m_tb, m_lat, m_ta, m_w, m_s;
    bool ok = make_map(&m_up, L.w_up, L.F, L.d, L.rs, kBM) && make_map(&m_gate, L.w_gate, L.F, L.d, L.rs, kBM) &&
              make_map(&m_x, xb, p.rows, L.d, L.ld, p.N) && make_map(&m_w, L.w_down, L.F, L.d, L.rs, kBK) &&
              make_map(&m_s, sb, p.rows, L.F, ld_s, p.N);
    if (dc_pred) {
        ok = ok && make_map(&m_tb, L.theta_bt, L.F, L.r, ldr, kBM) && make_map(&m_lat, latb, p.rows, L.r, ldr, p.N) &&
             make_map(&m_ta, L.theta_at, L.r, L.d, L.ld, kBM);
    } else {
        m_tb = m_lat = m_ta = m_up;
    }
    if (!ok) return cudaErrorInvalidValue;

    FusedArgs a{};
    a.F = static_cast<int>(L.F);
    a.d = static_cast<int>(L.d);
    a.r = static_cast<int>(L.r);
    a.nb = static_cast<int>(nb);
    a.nbt = p.nbt;
    a.N = p.N;
    a.n_tiles = p.n_tiles;
    a.mt0 = static_cast<int>((L.r + kBM - 1) / kBM);
    a.mta = static_cast<int>((L.F + kBM - 1) / kBM);
    a.jt = static_cast<int>((L.d + kDJF * kBM - 1) / (kDJF * kBM));
    a.kb_x = static_cast<int>((L.d + kBK - 1) / kBK);
    a.kb_z = dc_pred ? static_cast<int>((L.r + kBK - 1) / kBK) : 0;
    a.kb_f = static_cast<int>((L.F + kBK - 1) / kBK);
    a.tau = tau;
    a.ovr = ovr;
    a.s_out = sb;
    a.ld_s = ld_s;
    a.mask_out = mask_out;
    a.ind_out = ind_out;
    a.alive_out = alive_out;
    a.ws = part;
    a.flags = flags;
    a.y = y;
    a.lat32 = lat32;
    a.latb = latb;
    a.ldr = ldr;
    static unsigned long long* tl_env = []() -> unsigned long long* {
#ifdef CD_TIMELINE  // development builds only: a device address taken from the environment
        const char* e = std::getenv("CD_TC_TL");
        return e ? reinterpret_cast<unsigned long long*>(std::strtoull(e, nullptr, 10)) : nullptr;
#else
        return nullptr;
#endif
    }();
    a.tl = tl_env;
    static const int pf_env = dev_knob("CD_TC_PB_PF", 0);
    a.pb_pf = pf_env;
    // all 512 columns (one CTA per SM): the accumulators plus room to stage a tile's contributor
    // partials next to them
    a.tmem_cols = 512;
    const int stage_bytes = 2 * kABytes + p.N * kBK * 2;
    const size_t fixed = 1024 + 256;
    a.stages = static_cast<int>(std::min<size_t>(16, (kMaxDynSmem - fixed) / stage_bytes));
    const size_t smem = fixed + static_cast<size_t>(a.stages) * stage_bytes;
    using KFn = void (*)(CUtensorMap, CUtensorMap, CUtensorMap, CUtensorMap, CUtensorMap, CUtensorMap, CUtensorMap,
                         CUtensorMap, FusedArgs);
    const int kind = ovr ? kOvrF : method;
    KFn fn = nullptr;
#define CD_TCF_PICK(K) \
    if (kind == K) fn = L.act == 0 ? k_tc_fused<K, 0> : k_tc_fused<K, 1>;
    CD_TCF_PICK(kDense)
    CD_TCF_PICK(kMC)
    CD_TCF_PICK(kDC)
    CD_TCF_PICK(kCATS)
    CD_TCF_PICK(kOvrF)
#undef CD_TCF_PICK
    if (!fn) return cudaErrorInvalidValue;
    if ((e = set_smem(fn, smem)) != cudaSuccess) return e;
    LaunchCfg cc = c;
    cc.coop = true;  // not PDL-chained: the cooperative guarantee costs nothing here
    if ((e = launch_persistent(fn, dim3(G), dim3(kThreadsF), smem, cc, false, m_up, m_gate, m_x, m_tb, m_lat, m_ta,
                               m_w, m_s, a)) != cudaSuccess)
        return e;
    return cudaGetLastError();
}

}  // namespace tc
}  // namespace cdk
