// kernels_fused.cu -- the D-CountDown decode step as ONE persistent sm_100a kernel.
//
// pipeline_dc (blocked_exec.cpp:350-379) / Alg. 3 with UnorderedAccumulate
// semantics.  One CTA per SM.  Every weight byte is streamed by the TMA bulk-copy engine into
// shared memory; the step's three dependent stages exchange data between CTAs through
// EPOCH-TAGGED 64-bit words ({payload, launch tag} written with one single-copy-atomic store,
// readers spin until the tag matches) instead of grid barriers: there is no fence on the
// critical path, so no CTA ever waits for its own in-flight bulk copies to drain (a release
// fence does: measured 1.5-4.5 us per grid barrier with TMA traffic in flight).
//
//   prologue  (before griddepcontrol.wait -- overlaps the previous grid's tail)
//             producer lane streams this CTA's theta_at slice (its latent columns); consumers
//             load their chunk's theta_bt rows into registers (streaming 16-byte loads).
//   stage 1   latent[q] = theta_at[q] . x for q in this CTA's columns (predictor.cpp:94-102);
//             each value is published as a tagged word.
//   stage 2   all CTAs gather the latent (spinning on the tags), s_hat_i = latent . theta_bt[i]
//             for the chunk's neurons from registers (predictor.cpp:104-113), threshold
//             s_hat > tau_D or the mask override, ballot compaction into the own-work list.
//   stage 3   work stealing: each CTA streams its own actives up to the cap (the previous
//             launch's active count over the grid), publishes the overflow as tagged queue
//             entries, and pulls from the launch's queue until the sentinel.  A neuron's record
//             [up | gate | down] is ONE contiguous bulk copy; s_i = up act(gate) (exec_dc
//             blocked_exec.cpp:263-281) and y += s_i W_down[i] accumulate in registers of the
//             column-owning consumer threads; the partial y leaves the CTA in one TMA bulk
//             reduction.
//
// y is zeroed by CTA G-1 (no latent work at the Llama shape) and published by a fence before its
// count word, which every CTA acquires before its reductions.  The launch tag is read at start
// (after griddepcontrol.wait) and advanced by CTA 0 at its end: CTA 0 cannot finish before every
// CTA has published its count, i.e. read the tag.
//
// Requirements: grid == number of SMs, one CTA per SM (the dynamic shared memory forces it), all
// CTAs co-resident (the spins wait on other CTAs).
#include <cstdlib>
#include <type_traits>

#include "common.cuh"
#include "fused_common.cuh"
#include "kernels.h"
#include "launch.cuh"

namespace cdk {

namespace {

using namespace fused;

#ifndef CD_LAT_REP
#define CD_LAT_REP 8  // max latent copies (t_lat holds kMaxBatchFast x 2048 words)
#endif
#ifndef CD_PF_EARLY
#define CD_PF_EARLY 1  // next-layer predictor prefetch issued at the start of the chain (0: behind the records)
#endif
#ifndef CD_A_FIRST
#define CD_A_FIRST 1  // theta_b copy issued only after theta_a landed (theta_a gates stage 1)
#endif

constexpr int kRBf = 8;       // predictor rows per warp iteration (stage 2)
constexpr int kGroupF = 4;    // neurons per reduction round (stage 3)
constexpr int kSmemBudgetF = 220 * 1024;
// consumer threads per CTA (15 warps) + one producer warp: 16 warps = 512 threads keep the
// register cap at 128 per thread (17 warps are allocated as 20 and capped at 96 -> spills)
constexpr int kMaxConsumers = 480;
#ifdef CD_TIMELINE
// development build: stamps of the last 4 launches, slot = launch tag % 4 (stamps taken before
// the tag is known are held in registers)
static __device__ unsigned long long g_tlf[4][kTlKernels][kTlCtas][kTlPhases];
__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define TLF(k, p) do { if (blockIdx.x < kTlCtas) g_tlf[tl_tag & 3u][k][blockIdx.x][p] = gtime(); } while (0)
#define TLV(k, p, v) do { if (blockIdx.x < kTlCtas) g_tlf[tl_tag & 3u][k][blockIdx.x][p] = (v); } while (0)
#define TLC(p) do { if (blockIdx.x < kTlCtas) g_tlf[tl_tag & 3u][2][blockIdx.x][p] = clock64(); } while (0)
#else
#define TLC(p) ((void)0)
#define TLF(k, p) ((void)0)
#define TLV(k, p, v) ((void)0)
#endif

struct MetaF {
    int32_t idx;
    uint32_t bits;
    int32_t seq;  // position in the stage sequence (split stage 3: dot warps run n_dot records
                  // ahead, so a parity wait can alias the stage's previous use -- checked here)
    int32_t pad;
};

// Kernel arguments in one block (read through the constant bank as instruction operands).
struct FusedParams {
    LayerDev L;
    Scratch S;
    const float* x;
    const uint8_t* ovr;
    float* y;
    uint8_t* mask_out;
    float* logits_out;
    int* alive_out;
    float tau;
    float rms_eps;  // >= 0: the layer's input is RMSNorm(x) = x / sqrt(mean(x^2) + eps) per sample
    // the predictor of the layer that runs NEXT on this stream (same shape), or null: each CTA
    // prefetches its own slices of it into L2 once its records are issued, so the next step's
    // latent / logits stages read L2 instead of waiting on HBM (weights only: no dependence
    // on this step's output)
    const void* pf_at;
    const void* pf_bt;
    int nb, nstages, rows_per_cta, qrows;
    int b_smem;  // bf16: predictor rows staged by TMA in the ring, moved to registers after stage 1
    int n_dot;   // batch-1 bf16 stage 3: warps computing the records' up/gate dots (the rest: down)
    int lat_rep; // latent published in lat_rep copies; CTA c gathers copy c % lat_rep (spreads
                 // the all-CTA read of the same lines over lat_rep x more L2 lines)
};

template <typename W, int NB, int VPT, int VPL>
__global__ void __launch_bounds__(512, 1) k_dc_fused(const __grid_constant__ FusedParams P) {
    // bf16 layers keep the CTA's predictor rows in REGISTERS, loaded before griddepcontrol.wait
    // (the stage is then pure FFMA once the latent arrives); f32 layers stage them through smem
    constexpr bool kRegB = std::is_same<W, __nv_bfloat16>::value;
    constexpr int kRowsW = 8;  // predictor rows per consumer warp (register path)
    const LayerDev& L = P.L;
    const Scratch& S = P.S;
    const int nb = P.nb, nstages = P.nstages, rows_per_cta = P.rows_per_cta, qrows = P.qrows;
    const float tau = P.tau;
    const float* __restrict__ x = P.x;
    const uint8_t* __restrict__ ovr = P.ovr;
    float* __restrict__ y = P.y;
    uint8_t* __restrict__ mask_out = P.mask_out;
    float* __restrict__ logits_out = P.logits_out;
#ifdef CD_TIMELINE
    uint32_t tl_tag = 0;
    unsigned long long tl_h0 = gtime(), tl_h1 = 0, tl_h2 = 0;
#endif
    extern __shared__ __align__(1024) uint8_t smem[];
    constexpr int kBarC = 1;   // consumers only
    constexpr int kBarK = 3;   // consumers -> producer: own list, counts and launch tag in smem
    constexpr int kBarD = 2;   // stage-3 down warps (split stage 3)
    // batch-1 bf16: stage 3 splits each record between one "dot" warp (u, g over the whole row
    // from shared memory, s = u act(g)) and the "down" warps (column-owned y += s W_down[i]),
    // handing s over through a per-stage mbarrier -- no CTA-wide barrier per record group
    // (batch 2-4: when the columns fit one vector per consumer thread, VPT == 1 -- the down warps
    // then hold NB x 2 vectors of y; the dot warps compute only the samples a record is alive for)
    constexpr bool kSplit3 = kRegB && (NB == 1 || VPT == 1);
    constexpr int kVPD = NB == 1 ? 4 : 2;  // down-warp column vectors per thread (<= kVPD x 8 x nd columns)
    const int nwc = blockDim.x / kWarp - 1;
    const int nc = nwc * kWarp;
    const int warp = threadIdx.x / kWarp, lane = threadIdx.x % kWarp;
    const int G = gridDim.x;
    const int64_t rec_bytes = 3 * L.ld * (int64_t)sizeof(W);   // one neuron record
    const int64_t stage_bytes = rec_bytes;
    const int64_t brow_bytes = L.ldr * (int64_t)sizeof(W);     // one predictor row
    const int64_t arow_bytes = L.ld * (int64_t)sizeof(W);      // one theta_at row

    // ---- shared memory carve-up (all offsets multiples of 16).  The theta_at slice and x live
    // at the END of the ring (the predictor rows occupy its start): both are dead before the
    // first neuron record is streamed, so the whole ring serves stage 3.
    uint8_t* ring = smem;
    const int64_t aux_bytes = arow_bytes * qrows;
    W* abuf = reinterpret_cast<W*>(ring + stage_bytes * nstages - aux_bytes);  // [qrows][ld]
    float* latbuf = reinterpret_cast<float*>(ring + stage_bytes * nstages);    // [NB][ldr]
    uint64_t* full = reinterpret_cast<uint64_t*>(latbuf + NB * L.ldr);
    uint64_t* empty = full + nstages;
    uint64_t* bar_a = empty + nstages;
    uint64_t* bar_b = bar_a + 2;
    MetaF* meta = reinterpret_cast<MetaF*>(bar_a + 3);
    int32_t* own_idx = reinterpret_cast<int32_t*>(meta + nstages);
    uint32_t* own_bits = reinterpret_cast<uint32_t*>(own_idx + rows_per_cta);
    float* red = reinterpret_cast<float*>(own_bits + rows_per_cta);  // [nwc][32] warp partials
    float* sval = red + nwc * 32;                                      // [kGroupF * NB]
    int* cnt = reinterpret_cast<int*>(sval + kGroupF * NB);  // [0] n_own [1..NB] alive [NB+1] tag [NB+2] cap
    float* rms_red = reinterpret_cast<float*>(cnt + NB + 4);   // [nwc][NB] sum-of-squares partials
    // split stage 3: per-stage s hand-over barriers and values, x as f32 for the dot warps
    uint64_t* sready = reinterpret_cast<uint64_t*>((reinterpret_cast<uintptr_t>(rms_red + nwc * NB) + 15) & ~uintptr_t(15));
    float* svs = reinterpret_cast<float*>(sready + nstages);  // [nstages][NB]
    float* xs = reinterpret_cast<float*>((reinterpret_cast<uintptr_t>(svs + nstages * NB) + 15) & ~uintptr_t(15));
    const int n_dot = kSplit3 ? P.n_dot : 0;

    const int64_t c0 = (int64_t)blockIdx.x * rows_per_cta;
    const int64_t c1 = imin64(L.F, c0 + rows_per_cta);
    const int nrows = c1 > c0 ? static_cast<int>(c1 - c0) : 0;
    const int q0 = blockIdx.x * qrows;                      // this CTA's latent columns [q0, q1)
    const int q1 = min(static_cast<int>(L.r), q0 + qrows);
    const int nq = q1 > q0 ? q1 - q0 : 0;

    if (threadIdx.x == 0) {
        for (int s = 0; s < nstages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kSplit3 ? 1 + (nwc - n_dot) : nwc);
            if (kSplit3) mbar_init(&sready[s], 1);
        }
        mbar_init(bar_a, 1);
        mbar_init(bar_b, 1);
        for (int b = 0; b <= NB; ++b) cnt[b] = 0;
        fence_mbar_init();
    }
    __syncthreads();
    pdl_launch_dependents();

    const uint8_t* BT = static_cast<const uint8_t*>(L.theta_bt);
    const W* AT = static_cast<const W*>(L.theta_at);
    const W* REC = static_cast<const W*>(L.w_up);   // records [up | gate | down], stride L.rs

    if (warp == nwc) {
        // ================================================================ producer warp
        const uint64_t pol = policy_evict_first();
        int st = 0;
        uint32_t ph = 0;
        int pseq = 0;
        if (lane == 0) {
            // prologue: weights only (step-independent), overlaps the previous grid's tail
            if (nq > 0) {
                mbar_arrive_expect_tx(bar_a, static_cast<uint32_t>(nq * arow_bytes));
                bulk_g2s(abuf, AT + (int64_t)q0 * L.ld, static_cast<uint32_t>(nq * arow_bytes), bar_a, pol);
            }
            if ((!kRegB || P.b_smem) && nrows > 0) {
                // the chunk's predictor rows: one bulk copy into the (idle) ring head
#if CD_A_FIRST
                if (nq > 0) mbar_wait(bar_a, 0);  // theta_a gates stage 1: let it land first
#endif
                const int64_t bytes = nrows * brow_bytes;
                mbar_arrive_expect_tx(bar_b, static_cast<uint32_t>(bytes));
                bulk_g2s(ring, BT + c0 * brow_bytes, static_cast<uint32_t>(bytes), bar_b, pol);
            }
#if CD_PF_EARLY
            if (P.pf_bt) {
                // the next layer's theta slices of this CTA -> L2 while this step's dependent
                // chain (x -> latent -> logits -> mask) leaves HBM idle: the next step's prologue
                // then reads L2 instead of competing with this step's record stream for HBM.
                // After griddepcontrol.wait, so it does not compete with the previous step's.
                pdl_wait();
                if (nq > 0)
                    bulk_prefetch_l2(static_cast<const W*>(P.pf_at) + (int64_t)q0 * L.ld,
                                     static_cast<uint32_t>(nq * arow_bytes));
                for (int64_t off = 0; off < nrows * brow_bytes; off += 32768)
                    bulk_prefetch_l2(static_cast<const uint8_t*>(P.pf_bt) + c0 * brow_bytes + off,
                                     static_cast<uint32_t>(imin64(32768, nrows * brow_bytes - off)));
            }
#endif
        }
        __syncwarp();
        auto issue = [&](int32_t i, uint32_t bits) {
            mbar_wait(&empty[st], ph ^ 1);
            meta[st].idx = i;
            meta[st].bits = bits;
            meta[st].seq = pseq++;
            mbar_arrive_expect_tx(&full[st], static_cast<uint32_t>(rec_bytes));
            bulk_g2s(ring + st * stage_bytes, REC + (int64_t)i * L.rs, static_cast<uint32_t>(rec_bytes), &full[st],
                     pol);
            if (++st == nstages) { st = 0; ph ^= 1; }
        };
#ifdef CD_TIMELINE
        if (lane == 0) {  // arrival of the predictor slices (development build only)
            if (nq > 0) { mbar_wait(bar_a, 0); tl_h1 = gtime(); }
            if ((!kRegB || P.b_smem) && nrows > 0) { mbar_wait(bar_b, 0); tl_h2 = gtime(); }
        }
        __syncwarp();
#endif
        // ---- stage 3 schedule: this CTA's own active neurons up to the cap, its overflow
        // published to the launch's work queue, then stealing from that queue until empty.
        named_bar_sync(kBarK, nc + kWarp);
        const uint32_t tag = static_cast<uint32_t>(cnt[NB + 1]);
#ifdef CD_TIMELINE
        tl_tag = tag;
        if (lane == 0) {
            if (tl_h1) TLV(1, 4, tl_h1);
            if (tl_h2) TLV(1, 5, tl_h2);
        }
#endif
        const int n_own = cnt[0];
        const int kept = min(n_own, cnt[NB + 2]);
        const int ovf = n_own - kept;
        // [0..1] one 64-bit word {tail (low), pushed CTAs (high)}: a single load is a consistent
        // snapshot of both, so "all pushed" and the final tail arrive in one round trip.
        // [2] head (steal claims) [3] actives
        unsigned* qc = S.ctl + kCtlQueue + (tag % 3u) * 32u;
        unsigned long long* qtp = reinterpret_cast<unsigned long long*>(qc);
        int e = 0;
        if (lane == 0) {
            TLF(6, 5);
            for (; e < min(kept, nstages); ++e) issue(own_idx[e], own_bits[e]);  // fresh ring: no wait
            TLF(1, 0);
        }
        int base = 0;
        if (lane == 0) {
            red_add_u32(qc + 3, static_cast<unsigned>(n_own));
            if (ovf > 0) base = static_cast<int>(atomicAdd(qtp, static_cast<unsigned long long>(ovf)) & 0xFFFFFFFFull);
        }
        base = __shfl_sync(0xffffffffu, base, 0);
        for (int k = lane; k < ovf; k += kWarp) {
            const int32_t i = own_idx[kept + k];
            st_relaxed_u64(S.t_list + base + k, tagged(tag, static_cast<uint32_t>(i) | (own_bits[kept + k] << 27)));

        }
        __syncwarp();
        if (lane == 0) {
            atomicAdd(qtp, 1ull << 32);  // pushed (after this CTA's tail reservation returned)
            TLF(6, 6);
            for (; e < kept; ++e) issue(own_idx[e], own_bits[e]);
            TLF(1, 1);
            if (!CD_PF_EARLY && P.pf_bt) {
                // the next layer's theta slices of this CTA -> L2 (queued behind the records)
                if (nq > 0)
                    bulk_prefetch_l2(static_cast<const W*>(P.pf_at) + (int64_t)q0 * L.ld,
                                     static_cast<uint32_t>(nq * arow_bytes));
                for (int64_t off = 0; off < nrows * brow_bytes; off += 32768)
                    bulk_prefetch_l2(static_cast<const uint8_t*>(P.pf_bt) + c0 * brow_bytes + off,
                                     static_cast<uint32_t>(imin64(32768, nrows * brow_bytes - off)));
            }
            // steal: claim queue slots until the claim is past the final tail (known once every
            // CTA has pushed).  The next claim is requested before the current record waits for a
            // ring slot, so the last (empty) claim is usually back by the time the ring drains
            // and the sentinel follows the last record at once.
            const unsigned G_u = static_cast<unsigned>(G);
            unsigned tail_final = 0xFFFFFFFFu;
            int n_stolen = 0;
            unsigned next = atomicAdd(qc + 2, 1u);
            for (;;) {
                const unsigned slot = next;
                bool got = false;
                uint32_t wv = 0;
                while (slot < tail_final) {
                    // the entry and the {tail, pushed} snapshot in flight together
                    const bool in_list = slot < static_cast<unsigned>(L.F);
                    const unsigned long long w = in_list ? ld_relaxed_u64(S.t_list + slot) : 0ull;
                    const unsigned long long tp = ld_relaxed_u64(qtp);
                    if (in_list && static_cast<uint32_t>(w >> 32) == tag) {
                        wv = static_cast<uint32_t>(w);
                        got = true;
                        break;
                    }
                    // every CTA's tail reservation precedes its push in the word's order
                    if (static_cast<unsigned>(tp >> 32) == G_u) tail_final = static_cast<unsigned>(tp);
                }
                if (!got) break;
                next = atomicAdd(qc + 2, 1u);
                issue(static_cast<int32_t>(wv & ((1u << 27) - 1u)), wv >> 27);
                if (n_stolen++ == 0) TLF(1, 2);
                TLF(1, 3);
            }
#ifdef CD_TIMELINE
            TLV(1, 7, (unsigned long long)n_own | ((unsigned long long)kept << 16) |
                          ((unsigned long long)n_stolen << 32));
#endif
            // end-of-work sentinel for the consumers (completes the slot's phase, no bytes); split
            // stage 3: one per dot warp (dot warp w takes every n_dot-th stage in sequence)
            for (int k = 0; k < (kSplit3 ? n_dot : 1); ++k) {
                mbar_wait(&empty[st], ph ^ 1);
                meta[st].idx = -1;
                meta[st].seq = pseq++;
                mbar_arrive(&full[st]);
                if (++st == nstages) { st = 0; ph ^= 1; }
            }
            TLF(6, 4);
        }
        __syncwarp();
    } else {
        // ================================================================ consumer warps
        const int ct = threadIdx.x;
        const int nvec = static_cast<int>(L.ld / kVec);
        const int nvr = static_cast<int>(L.ldr / kVec);
        // register path: this warp's predictor rows (warp + i*nwc of the chunk), lane owns
        // vectors lane + v*32 of each row -- coalesced 16-byte loads, weights only
        uint4 rb[kRegB ? kRowsW : 1][VPL];
        if (kRegB && !P.b_smem) {
            // (b_smem: the rows arrive by TMA and are moved to registers after stage 1 instead --
            // 8 K register loads here would delay a late-starting CTA's griddepcontrol.wait,
            // and with it its latent columns that every CTA gathers)
            const W* BTw = static_cast<const W*>(L.theta_bt);
#pragma unroll
            for (int i = 0; i < kRowsW; ++i) {
                const int rl = warp + i * nwc;
#pragma unroll
                for (int v = 0; v < VPL; ++v) {
                    const int vec = lane + v * kWarp;
                    rb[i][v] = make_uint4(0u, 0u, 0u, 0u);
                    if (rl < nrows && vec < nvr) rb[i][v] = ldg_early_v4(BTw + (c0 + rl) * L.ldr + vec * kVec);
                }
            }
        }
        pdl_wait();  // y and the scratch words of the previous step are now safe to touch
        // x into registers right away (column ownership: vectors ct + j*nc), in flight together
        // with thread 0's launch-tag / queue-word reads below.  Plain vector loads, not the TMA
        // engine: a bulk copy of x would queue behind this CTA's predictor prefetch.
        float xr[NB][VPT][8];
        auto load_x = [&]() {
#pragma unroll
            for (int j = 0; j < VPT; ++j) {
                const int vec = ct + j * nc;
#pragma unroll
                for (int b = 0; b < NB; ++b) {
                    float4 lo = make_float4(0.f, 0.f, 0.f, 0.f), hi = lo;
                    const int64_t col = (int64_t)vec * kVec;
                    if (vec < nvec && b < nb) ldcg_x8(x + b * L.d + col, L.d - col, lo, hi);
                    xr[b][j][0] = lo.x; xr[b][j][1] = lo.y; xr[b][j][2] = lo.z; xr[b][j][3] = lo.w;
                    xr[b][j][4] = hi.x; xr[b][j][5] = hi.y; xr[b][j][6] = hi.z; xr[b][j][7] = hi.w;
                }
            }
        };
        load_x();
        float rms_inv[NB];  // the input RMS norm's per-sample scale (re-applied when x is reloaded)
#pragma unroll
        for (int b = 0; b < NB; ++b) rms_inv[b] = 1.0f;
        unsigned prev_actives = 0;  // thread 0: the previous launch's active count (in flight)
        if (threadIdx.x == 0) {
#ifdef CD_TIMELINE
            tl_h1 = gtime();
#endif
            const uint32_t t = static_cast<uint32_t>(__ldcg(S.ctl + kCtlEpoch)) + 1u;
#ifdef CD_TIMELINE
            tl_tag = t;
            TLV(5, 0, tl_h0);
            TLV(5, 1, tl_h1);
            TLC(0);
#endif
            cnt[NB + 1] = static_cast<int>(t);
            // own-work cap: the previous launch's active count spread over the grid (the first
            // launch keeps everything).  Only requested here -- it is consumed at the end of
            // stage 2, so stage 1 waits for one round trip (the tag), not two.  Queue counters of
            // the NEXT launch are reset here (the launch that used them last has completed).
            prev_actives = __ldcg(S.ctl + kCtlQueue + ((t + 2u) % 3u) * 32u + 3);
            if (blockIdx.x == 0) {
                unsigned* nq = S.ctl + kCtlQueue + ((t + 1u) % 3u) * 32u;
                nq[0] = 0u; nq[1] = 0u; nq[2] = 0u; nq[3] = 0u;
            }
        }
        if (P.rms_eps >= 0.0f) {
            // input RMS norm (stacked layers): every CTA holds all of x,
            // so each reduces the sum of squares itself -- one barrier, no exchange
#pragma unroll
            for (int b = 0; b < NB; ++b) {
                float ss = 0.0f;
#pragma unroll
                for (int j = 0; j < VPT; ++j)
#pragma unroll
                    for (int k = 0; k < 8; ++k) ss = fmaf(xr[b][j][k], xr[b][j][k], ss);
                ss = warp_sum(ss);
                if (lane == 0) rms_red[warp * NB + b] = ss;
            }
            named_bar_sync(kBarC, nc);
#pragma unroll
            for (int b = 0; b < NB; ++b) {
                const float ss = warp_sum(lane < nwc ? rms_red[lane * NB + b] : 0.0f);  // nwc <= 32
                const float inv = rsqrtf(ss / static_cast<float>(L.d) + P.rms_eps);
                rms_inv[b] = inv;
#pragma unroll
                for (int j = 0; j < VPT; ++j)
#pragma unroll
                    for (int k = 0; k < 8; ++k) xr[b][j][k] *= inv;
            }
        }
        if constexpr (kSplit3) {
            // x (normalised) as f32 in shared memory for the stage-3 dot warps
#pragma unroll
            for (int j = 0; j < VPT; ++j) {
                const int vec = ct + j * nc;
                if (vec < nvec) {
                    // two planes (elements 0-3 / 4-7 of every 8-vector): a dot warp's lanes then
                    // read consecutive 16-byte words (no 2-way bank conflict)
#pragma unroll
                    for (int b = 0; b < NB; ++b) {  // per sample: its two planes at b x ld floats
                        float4* lo = reinterpret_cast<float4*>(xs) + b * 2 * nvec;
                        lo[vec] = make_float4(xr[b][j][0], xr[b][j][1], xr[b][j][2], xr[b][j][3]);
                        lo[nvec + vec] = make_float4(xr[b][j][4], xr[b][j][5], xr[b][j][6], xr[b][j][7]);
                    }
                }
            }
        }
#ifdef CD_TIMELINE
        long long tl_xw = 0;
        if (lane == 0) {
            // per-warp x arrival (clock64): warps 0-7 in row 3, 8-15 in row 7
#pragma unroll
            for (int j = 0; j < VPT; ++j)
#pragma unroll
                for (int k = 0; k < 8; ++k) asm volatile("" ::"f"(xr[0][j][k]));
            tl_xw = clock64();  // written once the launch tag is known (below)
        }
        if (threadIdx.x == 0) {
            TLF(0, 0);
            TLC(1);
        }
#endif
        if (blockIdx.x == G - 1) {
            for (int64_t i = ct; i < (int64_t)nb * L.d; i += nc) y[i] = 0.0f;
            named_bar_sync(kBarC, nc);
            if (threadIdx.x == 0) {
                __threadfence();  // the zeroed y before the flag every CTA acquires before its reductions
                st_relaxed_u64(S.t_count + kYZeroWord, tagged(static_cast<uint32_t>(cnt[NB + 1]), 1u));
            }
        }
        // the launch tag (thread 0's read) reaches the other threads through stage 1's first
        // barrier -- none of its own, so every warp starts on its latent columns as soon as its x
        // and theta_a are in
        if (nq == 0) named_bar_sync(kBarC, nc);
        uint32_t tag = static_cast<uint32_t>(cnt[NB + 1]);  // nq > 0: re-read after that barrier
        if (threadIdx.x == 0) { TLF(6, 2); TLC(2); }

        // ---------------------------------------------------------- stage 1: latent columns
        if (nq > 0) {
            mbar_wait(bar_a, 0);
            if (threadIdx.x == 0) { TLF(6, 3); TLC(3); }
            constexpr int kQ = 4;
            for (int qb = 0; qb < nq; qb += kQ) {
                float v[kQ * NB];
                if constexpr (NB * VPT > 2 || VPL > 2) {
                    // (register-heavy variants: rows one at a time, no hoisting -- avoids spills)
#pragma unroll
                    for (int qq = 0; qq < kQ; ++qq) {
                        float a0[NB], a1[NB];
#pragma unroll
                        for (int b = 0; b < NB; ++b) a0[b] = a1[b] = 0.0f;
                        if (qb + qq < nq) {
#pragma unroll
                            for (int j = 0; j < VPT; ++j) {
                                const int vec = ct + j * nc;
                                if (vec < nvec) {
                                    float w[8];
                                    Vec8<W>::load(abuf + (int64_t)(qb + qq) * L.ld + vec * kVec, w);
#pragma unroll
                                    for (int b = 0; b < NB; ++b)
#pragma unroll
                                        for (int k = 0; k < 8; k += 2) ffma2(a0[b], a1[b], w[k], w[k + 1], xr[b][j][k], xr[b][j][k + 1]);
                                }
                            }
                        }
#pragma unroll
                        for (int b = 0; b < NB; ++b) v[qq * NB + b] = a0[b] + a1[b];
                    }
                } else {
                    // branch-free: every row / vector read is issued before the first FMA (clamped
                    // indices; x is zero past the end, and rows past nq are never published)
                    float w[kQ][VPT][8];
#pragma unroll
                    for (int qq = 0; qq < kQ; ++qq) {
                        const int row = min(qb + qq, nq - 1);
#pragma unroll
                        for (int j = 0; j < VPT; ++j)
                            Vec8<W>::load(abuf + (int64_t)row * L.ld + min(ct + j * nc, nvec - 1) * kVec, w[qq][j]);
                    }
#pragma unroll
                    for (int qq = 0; qq < kQ; ++qq) {
                        float a0[NB], a1[NB];
#pragma unroll
                        for (int b = 0; b < NB; ++b) a0[b] = a1[b] = 0.0f;
#pragma unroll
                        for (int j = 0; j < VPT; ++j)
#pragma unroll
                            for (int b = 0; b < NB; ++b)
#pragma unroll
                                for (int k = 0; k < 8; k += 2)
                                    ffma2(a0[b], a1[b], w[qq][j][k], w[qq][j][k + 1], xr[b][j][k], xr[b][j][k + 1]);
#pragma unroll
                        for (int b = 0; b < NB; ++b) v[qq * NB + b] = a0[b] + a1[b];
                    }
                }
                constexpr int kV = kQ * NB;
                if (threadIdx.x == 0 && qb == 0) { TLF(0, 1); TLC(4); }
                const float tot = warp_transpose_sum<kV>(v);
                if ((lane % (32 / kV)) == 0) red[warp * 32 + lane / (32 / kV)] = tot;
                named_bar_sync(kBarC, nc);
                tag = static_cast<uint32_t>(cnt[NB + 1]);
                if (threadIdx.x == 0 && qb == 0) { TLF(0, 2); TLC(5); }
                if (warp == 0) {
                    // every lane of column vv holds its total; lane group g publishes replicas
                    // g, g + 32/kV, ...
                    constexpr int kG = 32 / kV;
                    const int vv = lane % kV, g = lane / kV;
                    const float s = sum_partials<kV>(red, 32, nwc, lane);
                    const int qq = vv / NB, b = vv % NB;
                    if (qb + qq < nq && b < nb)
                        for (int rp = g; rp < P.lat_rep; rp += kG)
                            st_relaxed_u64(S.t_lat + (int64_t)rp * NB * L.ldr + b * L.ldr + q0 + qb + qq,
                                           tagged(tag, __float_as_uint(s)));
                }
                // (also keeps the other warps' latent polls off the L2 until this CTA's
                // columns are out: polling early measured slower)
                named_bar_sync(kBarC, nc);
                if (threadIdx.x == 0 && qb == 0) { TLF(0, 3); TLC(6); }
            }
        }
#ifdef CD_TIMELINE
        tl_tag = tag;
        if (lane == 0 && blockIdx.x < kTlCtas) g_tlf[tl_tag & 3u][warp < 8 ? 3 : 7][blockIdx.x][warp & 7] = tl_xw;
#endif
        if (threadIdx.x == 0) TLF(5, 2);
        if (kRegB && P.b_smem) {
            // predictor rows smem -> registers while the latent columns of the other CTAs arrive
            if (nrows > 0) mbar_wait(bar_b, 0);
            const int nvr_b = static_cast<int>(L.ldr / kVec);
#pragma unroll
            for (int i = 0; i < kRowsW; ++i) {
                const int rl = warp + i * nwc;
#pragma unroll
                for (int v = 0; v < VPL; ++v) {
                    const int vec = lane + v * kWarp;
                    rb[i][v] = make_uint4(0u, 0u, 0u, 0u);
                    if (rl < nrows && vec < nvr_b)
                        rb[i][v] = *reinterpret_cast<const uint4*>(ring + rl * brow_bytes + vec * 16);
                }
            }
        }

        // ---------------------------------------------------------- stage 2: predictor + compaction
        // gather the latent (every CTA published its columns as tagged words): all of a thread's
        // words are requested at once, stale ones re-polled
        const unsigned long long* t_lat = S.t_lat + (int64_t)(blockIdx.x % P.lat_rep) * NB * L.ldr;
        for (int e0 = ct; e0 < NB * (int)L.ldr; e0 += 4 * nc) {
            unsigned long long w[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int e = e0 + k * nc;
                int b = 0;
#pragma unroll
                for (int bb = 1; bb < NB; ++bb) b += e >= bb * (int)L.ldr;
                const int q = e - b * (int)L.ldr;
                w[k] = (e < NB * (int)L.ldr && b < nb && q < L.r) ? ld_relaxed_u64(t_lat + e) : tagged(tag, 0u);
            }
            // stale words re-polled together (one round trip per pass for all of a thread's words,
            // not one wait after another)
            for (;;) {
                bool stale = false;
#pragma unroll
                for (int k = 0; k < 4; ++k) stale |= static_cast<uint32_t>(w[k] >> 32) != tag;
                if (!stale) break;
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    if (static_cast<uint32_t>(w[k] >> 32) != tag) w[k] = ld_relaxed_u64(t_lat + e0 + k * nc);
            }
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int e = e0 + k * nc;
                if (e >= NB * (int)L.ldr) continue;
                // two planes per sample (elements 0-3 / 4-7 of every 8-vector): the stage-2 reads
                // of a warp are then consecutive 16-byte words (no 2-way bank conflict)
                int b = 0;
#pragma unroll
                for (int bb = 1; bb < NB; ++bb) b += e >= bb * (int)L.ldr;  // no runtime division
                const int q = e - b * (int)L.ldr;
                latbuf[b * L.ldr + ((q & 4) ? L.ldr / 2 : 0) + (q >> 3) * 4 + (q & 3)] =
                    __uint_as_float(static_cast<uint32_t>(w[k]));
            }
        }
        named_bar_sync(kBarC, nc);
        if (threadIdx.x == 0) { TLF(5, 3); TLC(7); }
        if constexpr (kRegB) {
            float lat[NB][VPL][8];
#pragma unroll
            for (int v = 0; v < VPL; ++v) {
                const int vec = lane + v * kWarp;
#pragma unroll
                for (int b = 0; b < NB; ++b) {
                    float4 lo = make_float4(0.f, 0.f, 0.f, 0.f), hi = lo;
                    if (vec < nvr) {
                        lo = reinterpret_cast<const float4*>(latbuf + b * L.ldr)[vec];
                        hi = reinterpret_cast<const float4*>(latbuf + b * L.ldr + L.ldr / 2)[vec];
                    }
                    lat[b][v][0] = lo.x; lat[b][v][1] = lo.y; lat[b][v][2] = lo.z; lat[b][v][3] = lo.w;
                    lat[b][v][4] = hi.x; lat[b][v][5] = hi.y; lat[b][v][6] = hi.z; lat[b][v][7] = hi.w;
                }
            }
            if (threadIdx.x == 0) TLF(6, 0);
            constexpr int kV = kRowsW * NB;
            float v[kV];
#pragma unroll
            for (int i = 0; i < kRowsW; ++i) {
                float a0[NB], a1[NB];
#pragma unroll
                for (int b = 0; b < NB; ++b) a0[b] = a1[b] = 0.0f;
#pragma unroll
                for (int q = 0; q < VPL; ++q) {
                    float w[8];
                    const uint32_t raw[4] = {rb[i][q].x, rb[i][q].y, rb[i][q].z, rb[i][q].w};
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        w[2 * k] = __uint_as_float(raw[k] << 16);
                        w[2 * k + 1] = __uint_as_float(raw[k] & 0xffff0000u);
                    }
#pragma unroll
                    for (int b = 0; b < NB; ++b)
#pragma unroll
                        for (int k = 0; k < 8; k += 2) ffma2(a0[b], a1[b], w[k], w[k + 1], lat[b][q][k], lat[b][q][k + 1]);
                }
#pragma unroll
                for (int b = 0; b < NB; ++b) v[i * NB + b] = a0[b] + a1[b];
            }
            const float tot = warp_transpose_sum<kV>(v);
            if ((lane % (32 / kV)) == 0) red[warp * 32 + lane / (32 / kV)] = tot;
            __syncwarp();
            // lanes 0..kRowsW-1: row warp + lane*nwc of the chunk
            const int rl = warp + lane * nwc;
            const bool valid = lane < kRowsW && rl < nrows;
            const int64_t gi = c0 + rl;
            uint32_t bits = 0;
#pragma unroll
            for (int b = 0; b < NB; ++b) {
                bool a = false;
                if (valid && b < nb) {
                    const float z = red[warp * 32 + lane * NB + b];
                    a = ovr ? (ovr[b * L.F + gi] != 0) : (z > tau);
                    if (mask_out) mask_out[b * L.F + gi] = a ? 1 : 0;
                    if (logits_out) logits_out[b * L.F + gi] = z;
                }
                bits |= static_cast<uint32_t>(a) << b;
                const unsigned bal = __ballot_sync(0xffffffffu, a);
                if (lane == 0 && bal) atomicAdd(&cnt[1 + b], __popc(bal));
            }
            const unsigned any = __ballot_sync(0xffffffffu, bits != 0);
            int e0 = 0;
            if (lane == 0 && any) e0 = atomicAdd(&cnt[0], __popc(any));
            e0 = __shfl_sync(0xffffffffu, e0, 0);
            if (bits) {
                const int e = e0 + __popc(any & ((1u << lane) - 1u));
                own_idx[e] = static_cast<int32_t>(gi);
                own_bits[e] = bits;
            }
        } else {
        float lat[NB][VPL][8];
#pragma unroll
        for (int v = 0; v < VPL; ++v) {
            const int vec = lane + v * kWarp;
#pragma unroll
            for (int b = 0; b < NB; ++b) {
                float4 lo = make_float4(0.f, 0.f, 0.f, 0.f), hi = lo;
                if (vec < nvr) {
                    lo = reinterpret_cast<const float4*>(latbuf + b * L.ldr)[vec];
                    hi = reinterpret_cast<const float4*>(latbuf + b * L.ldr + L.ldr / 2)[vec];
                }
                lat[b][v][0] = lo.x; lat[b][v][1] = lo.y; lat[b][v][2] = lo.z; lat[b][v][3] = lo.w;
                lat[b][v][4] = hi.x; lat[b][v][5] = hi.y; lat[b][v][6] = hi.z; lat[b][v][7] = hi.w;
            }
        }
        if (nrows > 0) mbar_wait(bar_b, 0);
        if (threadIdx.x == 0) TLF(6, 0);
        {
            const W* base = reinterpret_cast<const W*>(ring);
            for (int rr0 = warp * kRBf; rr0 < nrows; rr0 += nwc * kRBf) {
                constexpr int kV = kRBf * NB;
                float v[kV];
#pragma unroll
                for (int j = 0; j < kRBf; ++j) {
                    float w[VPL][8];
#pragma unroll
                    for (int q = 0; q < VPL; ++q) {
                        const int vec = lane + q * kWarp;
                        if (rr0 + j < nrows && vec < nvr) Vec8<W>::load(base + (rr0 + j) * L.ldr + vec * kVec, w[q]);
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
                if ((lane % (32 / kV)) == 0) red[warp * 32 + lane / (32 / kV)] = tot;
                __syncwarp();
                const bool valid = lane < kRBf && rr0 + lane < nrows;
                const int64_t gi = c0 + rr0 + lane;
                uint32_t bits = 0;
#pragma unroll
                for (int b = 0; b < NB; ++b) {
                    bool a = false;
                    if (valid && b < nb) {
                        const float z = red[warp * 32 + lane * NB + b];
                        a = ovr ? (ovr[b * L.F + gi] != 0) : (z > tau);
                        if (mask_out) mask_out[b * L.F + gi] = a ? 1 : 0;
                        if (logits_out) logits_out[b * L.F + gi] = z;
                    }
                    bits |= static_cast<uint32_t>(a) << b;
                    const unsigned bal = __ballot_sync(0xffffffffu, a);
                    if (lane == 0 && bal) atomicAdd(&cnt[1 + b], __popc(bal));
                }
                const unsigned any = __ballot_sync(0xffffffffu, bits != 0);
                int e0 = 0;
                if (lane == 0 && any) e0 = atomicAdd(&cnt[0], __popc(any));
                e0 = __shfl_sync(0xffffffffu, e0, 0);
                if (bits) {
                    const int e = e0 + __popc(any & ((1u << lane) - 1u));
                    own_idx[e] = static_cast<int32_t>(gi);
                    own_bits[e] = bits;
                }
                __syncwarp();
            }
        }
        }
        if (threadIdx.x == 0) {
            TLF(6, 1);
            cnt[NB + 2] = prev_actives > 0 ? static_cast<int>((prev_actives + G - 1) / G) : (1 << 30);
        }
        named_bar_sync(kBarC, nc);
        if (threadIdx.x == 0) TLF(5, 4);
        named_bar_arrive(kBarK, nc + kWarp);  // producer may schedule stage 3 now
        if (threadIdx.x == 0) {
            st_relaxed_u64(S.t_alive + blockIdx.x * kMaxBatchFast, tagged(tag, static_cast<uint32_t>(cnt[1])));
            for (int b = 1; b < NB; ++b)
                st_relaxed_u64(S.t_alive + blockIdx.x * kMaxBatchFast + b, tagged(tag, static_cast<uint32_t>(cnt[1 + b])));
            (void)await_acquire(S.t_count + kYZeroWord, tag);  // y zeroed (set long ago: one round trip)
            TLF(5, 5);
        }
        if constexpr (!kSplit3) {
        if constexpr (NB > 1) {
            // x again (L2 hits, in flight while the first records stream in): not holding it in
            // registers through stage 2 keeps the batch-2..4 variants from spilling there
            load_x();
            if (P.rms_eps >= 0.0f)
#pragma unroll
                for (int b = 0; b < NB; ++b)
#pragma unroll
                    for (int j = 0; j < VPT; ++j)
#pragma unroll
                        for (int k = 0; k < 8; ++k) xr[b][j][k] *= rms_inv[b];
        }
        int st = 0;
        uint32_t ph = 0;

        // ---------------------------------------------------------- stage 3: sparse FFN
        float yr[NB][VPT][8];
#pragma unroll
        for (int j = 0; j < VPT; ++j)
#pragma unroll
            for (int b = 0; b < NB; ++b)
#pragma unroll
                for (int k = 0; k < 8; ++k) yr[b][j][k] = 0.0f;
        const int64_t row_bytes = L.ld * (int64_t)sizeof(W);
        int n_rec = 0;  // records consumed (until the producer's sentinel)
        for (bool done = false; !done;) {
            int ns = 0;
            constexpr int kV = kGroupF * 2 * NB;
            int sts[kGroupF];
            float v[kV];
#pragma unroll
            for (int q = 0; q < kGroupF; ++q) {
                sts[q] = st;
                float g0v[NB], g1v[NB], u0[NB], u1[NB];
#pragma unroll
                for (int b = 0; b < NB; ++b) g0v[b] = g1v[b] = u0[b] = u1[b] = 0.0f;
                if (!done) {
                    mbar_wait(&full[st], ph);
                    if (meta[st].idx < 0) done = true;
                }
                if (!done) {
                    ns = q + 1;
#ifdef CD_TIMELINE
                    if (threadIdx.x == 0 && blockIdx.x < kTlCtas) {
                        const int rec = n_rec + q;
                        if (rec == 0) TLF(4, 0);
                        if (rec == 3) TLF(4, 1);
                        if (rec == 6) TLF(4, 2);
                        TLF(4, 3);
                        TLV(4, 7, rec + 1);
                    }
#endif
                    const uint8_t* sb = ring + st * stage_bytes;
                    const W* rup = reinterpret_cast<const W*>(sb);
                    const W* rgate = reinterpret_cast<const W*>(sb + row_bytes);
#pragma unroll
                    for (int j = 0; j < VPT; ++j) {
                        const int vec = ct + j * nc;
                        if (vec < nvec) {
                            float wg[8], wu[8];
                            Vec8<W>::load(rgate + vec * kVec, wg);
                            Vec8<W>::load(rup + vec * kVec, wu);
#pragma unroll
                            for (int b = 0; b < NB; ++b)
#pragma unroll
                                for (int k = 0; k < 8; k += 2) {
                                    ffma2(g0v[b], g1v[b], wg[k], wg[k + 1], xr[b][j][k], xr[b][j][k + 1]);
                                    ffma2(u0[b], u1[b], wu[k], wu[k + 1], xr[b][j][k], xr[b][j][k + 1]);
                                }
                        }
                    }
                    if (++st == nstages) { st = 0; ph ^= 1; }
                }
#pragma unroll
                for (int b = 0; b < NB; ++b) {
                    v[(q * 2) * NB + b] = g0v[b] + g1v[b];
                    v[(q * 2 + 1) * NB + b] = u0[b] + u1[b];
                }
            }
            if (ns == 0) break;
            n_rec += ns;
            const float tot = warp_transpose_sum<kV>(v);
            if ((lane % (32 / kV)) == 0) red[warp * 32 + lane / (32 / kV)] = tot;
            named_bar_sync(kBarC, nc);
            if (warp == 0) {
                const float col = sum_partials<kV>(red, 32, nwc, lane);  // column lane % kV
                const int q = lane / NB, b = lane % NB;
                const float g = __shfl_sync(0xffffffffu, col, ((q * 2) * NB + b) % kV);
                const float u = __shfl_sync(0xffffffffu, col, ((q * 2 + 1) * NB + b) % kV);
                if (lane < ns * NB) {
                    int sq = sts[0];
#pragma unroll
                    for (int qq = 1; qq < kGroupF; ++qq) sq = (q == qq) ? sts[qq] : sq;
                    const bool alive = (meta[sq].bits >> b) & 1u;
                    sval[lane] = alive ? u * act_fast(L.act, g) : 0.0f;
                }
            }
            named_bar_sync(kBarC, nc);
#pragma unroll
            for (int q = 0; q < kGroupF; ++q) {
                if (q < ns) {
                    const int sq = sts[q];
                    float sv[NB];
#pragma unroll
                    for (int b = 0; b < NB; ++b) sv[b] = sval[q * NB + b];
                    const W* rdown = reinterpret_cast<const W*>(ring + sq * stage_bytes + 2 * row_bytes);
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
        if (threadIdx.x == 0) TLF(5, 6);
        if (n_rec > 0) {
            // this CTA's partial y -> shared memory (the ring is idle now) -> ONE bulk reduction
            // into global y by the TMA engine (cp.reduce.async.bulk .add.f32): line-granular
            // adds at L2 instead of 1024 contended red.v4 per CTA, which the next step's
            // griddepcontrol.wait would otherwise have to drain
            named_bar_sync(kBarC, nc);  // every consumer is past its last ring read
            float* ys = reinterpret_cast<float*>(ring);
#pragma unroll
            for (int j = 0; j < VPT; ++j) {
                const int vec = ct + j * nc;
#pragma unroll
                for (int b = 0; b < NB; ++b) {
                    // d % 4 == 0 (launch requirement): whole float4s (scalar stores conflict 8-way)
                    const int64_t col = (int64_t)vec * kVec;
                    if (b >= nb || vec >= nvec) continue;
                    float4* dst = reinterpret_cast<float4*>(ys + b * L.d + col);
                    if (col < L.d) dst[0] = make_float4(yr[b][j][0], yr[b][j][1], yr[b][j][2], yr[b][j][3]);
                    if (col + 4 < L.d) dst[1] = make_float4(yr[b][j][4], yr[b][j][5], yr[b][j][6], yr[b][j][7]);
                }
            }
            fence_proxy_async_smem();
            named_bar_sync(kBarC, nc);
            if (threadIdx.x == 0) {
                bulk_reduce_add_f32(y, ys, static_cast<uint32_t>(nb * L.d * sizeof(float)));
                bulk_commit_and_wait_read();
            }
        }
        } else {
        // ---------------------------------------------------------- stage 3 (split): batch 1, bf16
        const int64_t row_bytes = L.ld * (int64_t)sizeof(W);
        if (warp < n_dot) {
            // dot warp: records warp, warp + n_dot, ... of the stage sequence
            int sq = warp;  // e % nstages and its use parity, advanced without a division
            uint32_t upar = 0;
            for (int e = warp;; e += n_dot) {
                if (e != warp) {
                    sq += n_dot;
                    if (sq >= nstages) { sq -= nstages; upar ^= 1u; }
                }
                // the stage's previous use (e - nstages) may still be loading: its incomplete
                // phase has the other parity, so the wait can return early -- retry until the
                // stage holds record e
                // (meta.seq == e implies the previous use completed, so the second wait is exact)
                for (;;) {
                    mbar_wait(&full[sq], upar);
                    if (*reinterpret_cast<volatile int32_t*>(&meta[sq].seq) == e) break;
                }
                mbar_wait(&full[sq], upar);
                if (meta[sq].idx < 0) {
                    // this warp's sentinel: forward it (the down warps stop at the first one)
                    if (lane == 0) mbar_arrive(&sready[sq]);
                    break;
                }
#ifdef CD_TIMELINE
                if (lane == 0 && blockIdx.x < kTlCtas) {
                    if (e == 0) TLF(4, 0);
                    if (e == 3) TLF(4, 1);
                    if (e == 6) TLF(4, 2);
                    TLF(4, 3);
                    TLV(4, 7, e + 1);
                }
#endif
                const W* rup = reinterpret_cast<const W*>(ring + sq * stage_bytes);
                const W* rgate = reinterpret_cast<const W*>(ring + sq * stage_bytes + row_bytes);
                const uint32_t bits = meta[sq].bits;
#pragma unroll
                for (int b = 0; b < NB; ++b) {
                    float sb = 0.0f;
                    if ((bits >> b) & 1u) {  // (a record of the union: only its live samples)
                        const float4* xp = reinterpret_cast<const float4*>(xs) + b * 2 * nvec;
                        float u0 = 0.f, u1 = 0.f, g0 = 0.f, g1 = 0.f;
#pragma unroll 4
                        for (int v = lane; v < nvec; v += kWarp) {
                            float wu[8], wg[8];
                            Vec8<W>::load(rup + v * kVec, wu);
                            Vec8<W>::load(rgate + v * kVec, wg);
                            const float4 xa = xp[v];
                            const float4 xb = xp[nvec + v];
                            const float xv[8] = {xa.x, xa.y, xa.z, xa.w, xb.x, xb.y, xb.z, xb.w};
#pragma unroll
                            for (int k = 0; k < 8; k += 2) {
                                ffma2(u0, u1, wu[k], wu[k + 1], xv[k], xv[k + 1]);
                                ffma2(g0, g1, wg[k], wg[k + 1], xv[k], xv[k + 1]);
                            }
                        }
                        float v2[2] = {u0 + u1, g0 + g1};
                        const float tot = warp_transpose_sum<2>(v2);  // lanes 0-15: u, 16-31: g
                        const float gsum = __shfl_sync(0xffffffffu, tot, 16);
                        sb = tot * act_fast(L.act, gsum);
                    }
                    if (lane == 0) svs[sq * NB + b] = sb;
                }
                __syncwarp();
                if (lane == 0) {
                    mbar_arrive(&sready[sq]);  // release-orders the s stores for the down warps
                    mbar_arrive(&empty[sq]);
                }
            }
        } else {
            // down warps: column vectors td + j nd of y, every record in sequence
            const int td = ct - n_dot * kWarp;
            const int nd = (nwc - n_dot) * kWarp;
            float yd[NB][kVPD][8];
#pragma unroll
            for (int b = 0; b < NB; ++b)
#pragma unroll
                for (int j = 0; j < kVPD; ++j)
#pragma unroll
                    for (int k = 0; k < 8; ++k) yd[b][j][k] = 0.0f;
            int n_rec = 0;
            int sq = -1;
            uint32_t upar = 0;
            for (;;) {
                if (++sq == nstages) { sq = 0; upar ^= 1u; }
                mbar_wait(&sready[sq], upar);
                if (meta[sq].idx < 0) break;
                float sv[NB];
#pragma unroll
                for (int b = 0; b < NB; ++b) sv[b] = svs[sq * NB + b];
                const W* rdown = reinterpret_cast<const W*>(ring + sq * stage_bytes + 2 * row_bytes);
#pragma unroll
                for (int j = 0; j < kVPD; ++j) {
                    const int vec = td + j * nd;
                    if (vec < nvec) {
                        float wd[8];
                        Vec8<W>::load(rdown + vec * kVec, wd);
#pragma unroll
                        for (int b = 0; b < NB; ++b)
#pragma unroll
                            for (int k = 0; k < 8; k += 2)
                                ffma2(yd[b][j][k], yd[b][j][k + 1], sv[b], sv[b], wd[k], wd[k + 1]);
                    }
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[sq]);
                ++n_rec;
            }
            if (td == 0) TLF(5, 6);
            if (n_rec > 0) {
                // partial y -> shared memory (stage 0 of the ring: no record is in flight past the
                // sentinel) -> one bulk reduction into global y
                named_bar_sync(kBarD, nd);
                float* ys = reinterpret_cast<float*>(ring);
#pragma unroll
                for (int j = 0; j < kVPD; ++j) {
                    const int vec = td + j * nd;
                    if (vec < nvec) {
                        // d % 4 == 0 (launch requirement): whole float4s, 8 lanes per 128 bytes
#pragma unroll
                        for (int b = 0; b < NB; ++b) {
                            if (b >= nb) continue;
                            float4* dst = reinterpret_cast<float4*>(ys + b * L.d + (int64_t)vec * kVec);
                            if ((int64_t)vec * kVec < L.d) dst[0] = make_float4(yd[b][j][0], yd[b][j][1], yd[b][j][2], yd[b][j][3]);
                            if ((int64_t)vec * kVec + 4 < L.d) dst[1] = make_float4(yd[b][j][4], yd[b][j][5], yd[b][j][6], yd[b][j][7]);
                        }
                    }
                }
                fence_proxy_async_smem();
                named_bar_sync(kBarD, nd);
                if (td == 0) {
                    (void)await_acquire(S.t_count + kYZeroWord, tag);  // y zeroed
                    bulk_reduce_add_f32(y, ys, static_cast<uint32_t>(nb * L.d * sizeof(float)));
                    bulk_commit_and_wait_read();
                }
            }
            if (td == 0) TLF(5, 7);
        }
        }
        if (blockIdx.x == 0 && warp == 0) {
            // per-sample alive counts (sum of the CTAs' tagged counts), then advance the tag:
            // every CTA read it before publishing the count CTA 0's producer waited for
            if (P.alive_out)
                for (int b = 0; b < nb; ++b) {
                    int a = 0;
                    for (int i = lane; i < G; i += kWarp)
                        a += static_cast<int>(await_relaxed(S.t_alive + i * kMaxBatchFast + b, tag));
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
                    if (lane == 0) P.alive_out[b] = a;
                }
            if (lane == 0) S.ctl[kCtlEpoch] = tag;
        }
    }
    if (!kSplit3 && threadIdx.x == 0) TLF(5, 7);
}

}  // namespace

#ifdef CD_TIMELINE
// The second most recent launch (its successor's prologue overlapped its tail: steady state).
cudaError_t read_timeline_fused(unsigned long long* out, int64_t n) {
    const size_t cnt = (size_t)kTlKernels * kTlCtas * kTlPhases;
    if ((size_t)n < cnt) return cudaErrorInvalidValue;
    static unsigned long long all[4 * kTlKernels * kTlCtas * kTlPhases];
    cudaError_t e = cudaMemcpyFromSymbol(all, g_tlf, sizeof(all));
    if (e != cudaSuccess) return e;
    unsigned long long last[4] = {0, 0, 0, 0};
    for (int sl = 0; sl < 4; ++sl)
        for (int c = 0; c < kTlCtas; ++c) {
            const unsigned long long v = all[((size_t)(sl * kTlKernels + 5) * kTlCtas + c) * kTlPhases + 1];
            if (v > last[sl]) last[sl] = v;
        }
    int best = 0, second = -1;
    for (int sl = 1; sl < 4; ++sl) if (last[sl] > last[best]) best = sl;
    for (int sl = 0; sl < 4; ++sl)
        if (sl != best && last[sl] > 0 && (second < 0 || last[sl] > last[second])) second = sl;
    const int pick = second >= 0 ? second : best;
    for (size_t i = 0; i < cnt; ++i) out[i] = all[pick * cnt + i];
    static unsigned long long zeros[4 * kTlKernels * kTlCtas * kTlPhases];
    return cudaMemcpyToSymbol(g_tlf, zeros, sizeof(zeros));
}
#else
cudaError_t read_timeline_fused(unsigned long long*, int64_t) { return cudaErrorNotSupported; }
#endif

cudaError_t launch_dc_fused(const LayerDev& L, const Scratch& S, const float* x, int nb, float tau,
                            const uint8_t* mask_override, float* y, uint8_t* mask_out, float* logits_out,
                            int* alive_out, const LaunchCfg& c, float rms_eps, const void* pf_at,
                            const void* pf_bt) {
    if (!L.theta_at || !S.t_lat || !S.t_list || !S.t_count || !S.t_alive || !S.ctl) return cudaErrorInvalidValue;
    if (c.num_sms >= kYZeroWord || L.F >= (1 << 27)) return cudaErrorInvalidValue;
    // x rows are staged by the TMA engine: 16-byte aligned rows of a multiple of 16 bytes
    if (L.d % 4 != 0 || (reinterpret_cast<uintptr_t>(x) & 15) != 0) return cudaErrorInvalidValue;
    const int64_t nvec = L.ld / kVec;
    // consumer threads own vpt 8-element column vectors each: up to 16 consumer warps
    int vpt = 0;
    for (int v : {1, 2, 4})
        if ((nvec + v - 1) / v <= kMaxConsumers) { vpt = v; break; }
    if (vpt == 0) return cudaErrorInvalidValue;
    const int nvr = static_cast<int>(L.ldr / kVec);
    const int vpl = nvr <= 32 ? 1 : nvr <= 64 ? 2 : nvr <= 128 ? 4 : 0;
    if (vpl == 0) return cudaErrorInvalidValue;
    const int nbk = nb <= 1 ? 1 : (nb <= 2 ? 2 : 4);
    if (nbk * kRBf > 32 || nbk * kGroupF * 2 > 32 || nbk * vpt > 8) return cudaErrorInvalidValue;
    const int G = c.num_sms;
    const bool regb = L.dtype == kBF16;
    const int rpc = static_cast<int>((L.F + G - 1) / G);
    const int qrows = static_cast<int>((L.r + G - 1) / G);
    const int64_t esz = L.dtype == kBF16 ? 2 : 4;
    const int64_t stage_bytes = 3 * L.ld * esz;
    const int64_t brow_bytes = L.ldr * esz;
    // consumer warps: enough for the columns at vpt vectors each and (bf16) for the chunk's
    // predictor rows at 8 per warp; at most 15 (+ the producer warp = 512 threads)
    int64_t nwc64 = std::max<int64_t>(8, ((nvec + vpt - 1) / vpt + kWarp - 1) / kWarp);
    if (regb) nwc64 = std::max<int64_t>(nwc64, (rpc + 7) / 8);
    // split stage 3 (batch 1, bf16): 8 down warps own the columns (<= 4 vectors each), the
    // other consumer warps (>= 2) compute the records' dots
    const bool split3 = regb && (nbk == 1 || vpt == 1);
    if (split3) nwc64 = std::max<int64_t>(nwc64, 10);
    const int nwc = static_cast<int>(nwc64);
    if (split3 && (nvec + 8 * kWarp - 1) / (8 * kWarp) > (nbk == 1 ? 4 : 2)) return cudaErrorInvalidValue;
    if (nwc * kWarp > kMaxConsumers) return cudaErrorInvalidValue;
    const int threads = (nwc + 1) * kWarp;
    // fixed carve-up beside the ring: latent, barriers, meta, lists, scratch, latent fragments
    // (the theta_at slice is overlaid on the ring's tail)
    const int64_t aux_bytes = (int64_t)qrows * L.ld * esz;
    const int64_t fixed = (int64_t)nbk * L.ldr * 4 + 3 * 8 + (int64_t)rpc * 8 + (nwc * 32 + kGroupF * nbk) * 4 +
                          (4 + nbk) * 4 + nwc * nbk * 4 + 64 +
                          (split3 ? 12 * (8 + 4 * nbk) + nbk * L.ld * 4 + 32 : 0);  // s hand-over, x f32
    const int64_t per_stage = stage_bytes + 2 * 8 + (int64_t)sizeof(MetaF);
    const int nstages = static_cast<int>(imin64(12, (kSmemBudgetF - fixed) / per_stage));
    if (nstages < 2) return cudaErrorInvalidValue;
    // dot warps run at most nstages - 1 records ahead of the stage sequence (their parity waits
    // are sequence-checked against one previous use of a stage)
    const int n_dot = split3 ? std::min(nwc - 8, nstages - 1) : 0;
    if (split3 && n_dot < 1) return cudaErrorInvalidValue;
    static const bool bsmem_env = dev_knob("CD_DC_BSMEM", 1) != 0;
    const int b_smem = regb && bsmem_env && (int64_t)rpc * brow_bytes + aux_bytes <= stage_bytes * nstages ? 1 : 0;
    if (regb ? rpc > nwc * 8 : (int64_t)rpc * brow_bytes + aux_bytes > stage_bytes * nstages)
        return cudaErrorInvalidValue;  // register path: <= 8 predictor rows per consumer warp
    if (aux_bytes > stage_bytes * nstages) return cudaErrorInvalidValue;
    const size_t smem = static_cast<size_t>(fixed + per_stage * nstages);
    auto go = [&](auto kern) {
        cudaError_t e = set_smem(kern, smem);
        if (e != cudaSuccess) return e;
        FusedParams p;
        p.L = L;
        p.S = S;
        p.x = x;
        p.ovr = mask_override;
        p.y = y;
        p.mask_out = mask_out;
        p.logits_out = logits_out;
        p.alive_out = alive_out;
        p.tau = tau;
        p.rms_eps = rms_eps;
        p.pf_at = pf_bt ? pf_at : nullptr;
        p.pf_bt = pf_at ? pf_bt : nullptr;
        p.nb = nb;
        p.nstages = nstages;
        p.rows_per_cta = rpc;
        p.qrows = qrows;
        p.b_smem = b_smem;
        p.n_dot = n_dot;
        p.lat_rep = 1;
        while (p.lat_rep < CD_LAT_REP && (int64_t)p.lat_rep * 2 * nbk * L.ldr <= kMaxBatchFast * 2048) p.lat_rep *= 2;
        return launch_persistent(kern, dim3(G), dim3(threads), smem, c, true, p);
    };
#define CD_FUSED_CASES(W)                                          \
    switch (nbk * 100 + vpt * 10 + vpl) {                          \
        case 121: return go(k_dc_fused<W, 1, 2, 1>);               \
        case 122: return go(k_dc_fused<W, 1, 2, 2>);               \
        case 124: return go(k_dc_fused<W, 1, 2, 4>);               \
        case 111: return go(k_dc_fused<W, 1, 1, 1>);               \
        case 112: return go(k_dc_fused<W, 1, 1, 2>);               \
        case 114: return go(k_dc_fused<W, 1, 1, 4>);               \
        case 141: return go(k_dc_fused<W, 1, 4, 1>);               \
        case 142: return go(k_dc_fused<W, 1, 4, 2>);               \
        case 221: return go(k_dc_fused<W, 2, 2, 1>);               \
        case 222: return go(k_dc_fused<W, 2, 2, 2>);               \
        case 211: return go(k_dc_fused<W, 2, 1, 1>);               \
        case 212: return go(k_dc_fused<W, 2, 1, 2>);               \
        case 241: return go(k_dc_fused<W, 2, 4, 1>);               \
        case 242: return go(k_dc_fused<W, 2, 4, 2>);               \
        case 421: return go(k_dc_fused<W, 4, 2, 1>);               \
        case 422: return go(k_dc_fused<W, 4, 2, 2>);               \
        case 411: return go(k_dc_fused<W, 4, 1, 1>);               \
        case 412: return go(k_dc_fused<W, 4, 1, 2>);               \
    }                                                              \
    return cudaErrorInvalidValue;
    if (L.dtype == kBF16) { CD_FUSED_CASES(__nv_bfloat16) }
    CD_FUSED_CASES(float)
#undef CD_FUSED_CASES
}

}  // namespace cdk
