// kernels.h -- host-side launch interface of the COUNTDOWN sm_100a kernels.
//
// Device data layout (one layer / one tensor-parallel shard), all in HBM:
//   neuron records       : F x [up | gate | down], each part ld = round_up(d, 8) elements
//                          (zero-padded to whole 16-byte vectors).  The reference stores the
//                          three matrices neuron-major (gated_mlp.hpp:16-19); here the three
//                          rows of one neuron are also adjacent, so an active neuron is ONE
//                          contiguous run of 3*ld elements = one TMA bulk copy (a bulk copy
//                          costs ~170 ns of per-SM issue time regardless of size, so three
//                          separate 8 KB row copies cap an SM at ~28 GB/s -- measured).
//                          w_up / w_gate / w_down point into the record (offsets 0, ld, 2ld)
//                          with row stride rs = 3*ld.
//   theta_a              : d x ldr (reference layout, predictor.hpp:17), ldr = round_up(r, 8).
//   theta_bt             : F x ldr, theta_b (r x F, predictor.hpp:18) transposed so one
//                          neuron's predictor row is contiguous.
// Weights are f32 (oracle mode) or bf16 (RNE-rounded, perf mode); x, y, and all
// accumulation are f32.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace cdk {

constexpr int kVecElems = 8;      // weights per 16-byte (bf16) vector unit; row stride multiple
constexpr int kMaxBatchFast = 4;   // samples per fused-kernel instance (union of masks)
constexpr int kMaxBatch = 32;      // samples per call (bitmask width)
constexpr int kMaxCtas = 1024;     // fused kernel grid bound (== SM count)

struct LayerDev {
    int64_t d = 0, F = 0, ld = 0;  // d_model, rows in this shard, padded row length
    int64_t rs = 0;                // stride between consecutive neurons' rows (= 3*ld)
    int act = 0, dtype = 0;
    const void* w_up = nullptr;
    const void* w_gate = nullptr;
    const void* w_down = nullptr;
    int64_t r = 0, ldr = 0;
    const void* theta_a = nullptr;   // d x ldr
    const void* theta_at = nullptr;  // r x ld  (theta_a transposed: one latent column per row)
    const void* theta_bt = nullptr;  // F x ldr
    int pred_kind = 0;               // 0: low-rank (theta_a, theta_bt); 1: ternary (Q^T in theta_bt)
    float gamma = 0.0f;              // ternary scale
};

// Per-handle device scratch.  latent/count/done are "self-cleaning": every kernel
// chain leaves them zero for the next one (initialised by cudaMemset at creation).
struct Scratch {
    float* latent = nullptr;       // kMaxBatch x ldr
    int32_t* list = nullptr;       // F : compacted neuron ids (union over samples)
    uint32_t* bits = nullptr;      // F : per-sample alive bits of each list entry
    float* list_val = nullptr;     // F x kMaxBatchFast : MC indicator u per entry & sample
    int* count = nullptr;          // union list length
    int* done = nullptr;           // last-CTA arrival counter
    int* alive = nullptr;          // kMaxBatch per-sample alive counts (accumulator)
    float* ind = nullptr;          // kMaxBatch x F : exact-mode indicator (u or logits)
    float* ex_s = nullptr;         // kMaxBatch x F : exact-mode s
    float* ex_lat = nullptr;       // kMaxBatch x ldr : exact-mode latent
    // fused kernel (kernels_fused.cu): epoch-tagged words {payload, launch tag}
    unsigned* ctl = nullptr;                  // [0] launch tag of the last completed launch
    unsigned long long* t_lat = nullptr;      // kMaxBatchFast x 2048 : latent values
    unsigned long long* t_list = nullptr;     // F : rest-list entries (neuron id | bits << 27)
    unsigned long long* t_aux = nullptr;      // F : per-entry payload (M-CountDown: u)
    unsigned long long* t_count = nullptr;    // kMaxCtas : rest-list length per CTA
    unsigned long long* t_alive = nullptr;    // kMaxCtas x kMaxBatchFast : alive counts per CTA
    unsigned* tc_flags = nullptr;             // kMaxCtas + 64 : tensor-core path flags / counters (zero at rest)
};

struct LaunchCfg {
    int num_sms = 148;
    cudaStream_t stream = nullptr;
    bool pdl = true;
    bool coop = true;  // persistent kernels: cooperative launch (false: PDL-chained, device owned)
};

// Indicator kinds
enum Method : int { kDense = 0, kMC = 1, kDC = 2, kCATS = 3 };

// ---------------------------------------------------------------- fast path (UnorderedAccumulate)
// DC: latent = x theta_a (split over d rows, vector reductions into the zeroed latent).
cudaError_t launch_latent_fast(const LayerDev& L, const Scratch& S, const float* x, int nb,
                               const LaunchCfg& c);
// DC indicator: s_hat = latent theta_bt^T per neuron, threshold s_hat > tau (or override mask),
// compaction into the union list.  Zeroes y.  Optional mask / logits outputs (B x F).
cudaError_t launch_indicator_dc_fast(const LayerDev& L, const Scratch& S, int nb, float tau,
                                     const uint8_t* mask_override, float* y, uint8_t* mask_out,
                                     float* logits_out, const LaunchCfg& c);
// MC indicator: u = W_up x per neuron, threshold |u| > tau, compaction (u kept per entry).
// cats=true: CATS indicator h = act(W_gate x), threshold |h| > tau, h kept per entry.
cudaError_t launch_indicator_mc_fast(const LayerDev& L, const Scratch& S, const float* x, int nb,
                                     float tau, float* y, uint8_t* mask_out, float* u_out,
                                     const LaunchCfg& c, bool cats = false);
// Fused sparse FFN over the compacted list: gathered up/gate rows (DC) or gate rows (MC,
// u from the list), act inline, row-sparse W_down accumulate; y += via red.v4.
// dense=true processes every row (count = F) without a list.
cudaError_t launch_sparse_fast(const LayerDev& L, const Scratch& S, int method, bool dense,
                               const float* x, int nb, float* y, int* alive_out,
                               const LaunchCfg& c);
// D-CountDown step as one persistent kernel (kernels_fused.cu): latent, predictor, threshold,
// (pf_at / pf_bt: theta_at / theta_bt of the next layer of identical shape, L2-prefetched),
// compaction and the sparse FFN (work-stealing schedule); zeroes and accumulates y, writes
// alive_out.  Returns cudaErrorInvalidValue for shapes it does not cover (the caller then
// uses the three-kernel chain).
cudaError_t launch_dc_fused(const LayerDev& L, const Scratch& S, const float* x, int nb, float tau,
                            const uint8_t* mask_override, float* y, uint8_t* mask_out, float* logits_out,
                            int* alive_out, const LaunchCfg& c, float rms_eps = -1.0f,
                            const void* pf_at = nullptr, const void* pf_bt = nullptr);
// M-CountDown step (batch 1) as one persistent kernel (kernels_fused_mc.cu): dense u = W_up x
// over each CTA's neuron chunk, |u| > tau, compaction, and the sparse gate / down stage with
// the work-stealing schedule.  Zeroes and accumulates y; optional mask / u / alive outputs.
// Returns cudaErrorInvalidValue for shapes it does not cover (the caller uses the chain).
cudaError_t launch_mc_fused(const LayerDev& L, const Scratch& S, const float* x, float tau, float* y,
                            uint8_t* mask_out, float* u_out, int* alive_out, const LaunchCfg& c);
// xn[b] = x[b] / sqrt(mean(x[b]^2) + eps) for b < nb (rows of d values, ld apart): the input
// RMS norm of stacked layers for the engines that do not fuse it.
cudaError_t launch_rmsnorm(const float* x, int nb, int64_t d, float eps, float* xn, const LaunchCfg& c);
// Host-supplied masks (exec_mc / exec_dc): ordered compaction + zero y (+ MC u gather).
cudaError_t launch_compact_masks(const LayerDev& L, const Scratch& S, const uint8_t* masks,
                                 const float* u_full, int nb, float* y, const LaunchCfg& c);

// ---------------------------------------------------------------- exact path (DeterministicOrdered)
// Bitwise-equal to the reference's serial folds (fresh f32 accumulator, ascending index,
// separate multiply/add roundings, activations in double).
cudaError_t launch_exact_latent(const LayerDev& L, const Scratch& S, const float* x, int nb,
                                const LaunchCfg& c);
// out[b][row] = fold_j W[row][j] * v[b][j] for every row of W (ncols = fold length).
cudaError_t launch_exact_rowdot_all(const void* W, int dtype, int64_t nrows, int64_t ld,
                                    int64_t ncols, const float* v, int64_t ldv, int nb,
                                    float* out, int64_t ldo, const LaunchCfg& c);
// Ordered union compaction from indicator values (mode 0: |v| > tau, 1: v > tau) or from
// given masks (mode 2).  Writes masks / per-sample alive counts / list / bits / count.
cudaError_t launch_exact_compact(const LayerDev& L, const Scratch& S, int mode,
                                 const float* ind, const uint8_t* masks_in, int nb, float tau,
                                 uint8_t* mask_out, int* alive_out, const LaunchCfg& c);
// Phase 1 over the list: DC/dense s = up * act(gate); MC s = act(gate) * u; CATS s = up * h.
cudaError_t launch_exact_phase1(const LayerDev& L, const Scratch& S, int method,
                                const float* x, const float* u_full, int nb,
                                const LaunchCfg& c);
// v[i] = act(v[i]) in place, double precision / one rounding (numerics.cpp:47-67).
cudaError_t launch_exact_act(int act, float* v, int64_t n, const LaunchCfg& c);
// out[i] = x[i] * g (one f32 rounding): the ternary predictor's scaled input.
cudaError_t launch_exact_scale(const float* x, int64_t n, float g, float* out, const LaunchCfg& c);
// y[b][j] = fold over list (ascending neuron) of s * W_down[i][j] for alive samples.
cudaError_t launch_exact_down(const LayerDev& L, const Scratch& S, int nb, float* y,
                              const LaunchCfg& c);

// Exact top-m per sample (top_m_threshold, numerics.cpp:105-142): rows of n values, ld apart;
// magnitude order (signed_order false) or signed order; ties to the lower index.  tau_out[b]
// (optional) = the (m+1)-th value (+inf for m <= 0, -inf for m >= n); mask_out (optional) rows
// ld_mask apart, the first m lanes in that order alive.
cudaError_t launch_top_m(const float* v, int batch, int64_t n, int64_t ld, int64_t m, bool signed_order,
                         float* tau_out, uint8_t* mask_out, int64_t ld_mask, const LaunchCfg& c);

// dst[0, bytes) = src[0, bytes) by a kernel (either side may be mapped pinned host memory).
cudaError_t launch_copy(void* dst, const void* src, size_t bytes, cudaStream_t s);

// *out += number of values of v[0, n) that are non-finite or overflow bf16 (upload check).
cudaError_t launch_count_nonfinite(const float* v, int64_t n, int* out, cudaStream_t s);

// One-thread kernel that occupies the stream for `ns` nanoseconds (timing helper).
cudaError_t launch_spin(unsigned long long ns, cudaStream_t s);
cudaError_t launch_copy_out_signal(float* hy, const float* dy, int64_t ny, int* ha, const int* da, int na,
                                   unsigned long long* done, cudaStream_t s, bool pdl);

// Development build only (-DCD_TIMELINE): copy the per-CTA phase stamps to the host.
cudaError_t read_timeline(unsigned long long* out, int64_t n);
cudaError_t read_timeline_fused(unsigned long long* out, int64_t n);

// ---------------------------------------------------------------- layout helpers
// dst row r = src row r (cols values, zero-padded to ld_pad), rows ld_dst apart.
cudaError_t launch_pack_rows(const float* src, int64_t rows, int64_t cols, int64_t ld_src,
                             void* dst, int dtype, int64_t ld_pad, int64_t ld_dst, cudaStream_t s);
// dst (cols_sel x ldr) = transpose of src[:, col_begin:col_begin+cols_sel] (src rows x ld_src).
cudaError_t launch_pack_transpose(const float* src, int64_t rows, int64_t ld_src,
                                  int64_t col_begin, int64_t cols_sel, void* dst, int dtype,
                                  int64_t ld_dst, cudaStream_t s);

}  // namespace cdk
