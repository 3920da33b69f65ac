/*
 * countdown_b200.h -- C-ABI of libcountdown_b200.so, the B200 (sm_100a) drop-in for the
 * COUNTDOWN sparse Gated-MLP decode path (arXiv 2505.17701).
 *
 * The reference exposes this path as the C++ operator API of
 * /root/reference/proj/include/countdown/{blocked_exec,sparsity,predictor}.hpp.  Every entry
 * point below names the reference interface it replaces (file:line).  Plain pointers and
 * sizes only: no C++ or torch types cross this boundary, so cgo / JNI / ctypes / a C++ shim
 * can bind it directly (the C++ shim that re-implements
 * blocked_exec.hpp over this ABI is paper_2505_17701_b200/shim/blocked_exec_gpu.cpp).
 *
 * Conventions
 *   - Matrices are row-major f32 on the host, laid out exactly as the reference stores them:
 *     w_up / w_gate / w_down are d_inter x d_model, neuron-major (gated_mlp.hpp:16-19);
 *     theta_a is d_model x d_rank, theta_b is d_rank x d_inter (predictor.hpp:17-18).
 *   - Batched inputs are `batch` consecutive rows: x is batch x d_model, y batch x d_model,
 *     masks batch x d_inter (uint8, 0/1), indicators batch x d_inter.  The reference is
 *     strictly per-sample (main.cpp:239-282); batch > 1 computes every sample with its own
 *     mask (rows of the per-sample union are streamed once).
 *   - Status codes follow the reference's error taxonomy (errors.hpp:1-17, exit-code mapping
 *     main.cpp:566-581): 0 ok, 2 DataError, 3 NumericError, 4 CUDA / device failure.
 *     cd_last_error() returns a thread-local message for the last failure on this thread.
 *   - Reduction modes mirror BlockConfig::reduction (blocked_exec.hpp:18-24):
 *       CD_REDUCTION_ORDERED   == Reduction::DeterministicOrdered: results are bit-identical
 *                                 to the reference's serial folds (exact kernels).
 *       CD_REDUCTION_UNORDERED == Reduction::UnorderedAccumulate: the fused B200 hot path;
 *                                 y within 1e-4 relative L2 of ORDERED in f32
 *                                 (test_blocked_exec.cpp:87-99).
 *     blk_m / blk_n have no GPU meaning; results are invariant to them (acceptance.cpp:336-342).
 *   - Thread safety: every entry point may be called from any thread.  Calls that enqueue
 *     work on a device's internal stream (host-buffer operators, create / load / destroy,
 *     set_predictor) are serialised by a per-device lock, then a per-handle lock.  No host
 *     threads are spawned.
 */
#ifndef COUNTDOWN_B200_H
#define COUNTDOWN_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CD_OK 0
#define CD_ERR_USAGE 1
#define CD_ERR_DATA 2
#define CD_ERR_NUMERIC 3
#define CD_ERR_CUDA 4

/* Activation (numerics.hpp:78) */
#define CD_ACT_SILU 0
#define CD_ACT_GELU_TANH 1

/* Weight storage type on the device (x, y and accumulation are always f32). */
#define CD_DTYPE_F32 0
#define CD_DTYPE_BF16 1

/* Reduction (blocked_exec.hpp:18) */
#define CD_REDUCTION_ORDERED 0
#define CD_REDUCTION_UNORDERED 1

/* Method selector for cd_forward_device (costmodel.hpp:52 CostMethod). */
#define CD_METHOD_DENSE 0
#define CD_METHOD_MC 1
#define CD_METHOD_DC 2
#define CD_METHOD_CATS 3

#if defined(__GNUC__)
#define CD_API __attribute__((visibility("default")))
#else
#define CD_API
#endif

typedef struct cd_layer cd_layer;

/* ---------------------------------------------------------------- library */
CD_API const char* cd_last_error(void);
CD_API int cd_version(void);
/* Number of SMs and compute capability of `device` (fails on a device that is not sm_100). */
CD_API int cd_device_info(int device, int* num_sms, int* cc_major, int* cc_minor);

/* ---------------------------------------------------------------- layer handles
 * Replaces the GatedMlpLayer value type (gated_mlp.hpp:12-23) crossing into the operators:
 * weights are uploaded once (re-laid out for the device) and referenced by handle.
 * GatedMlpLayer::validate() (gated_mlp.cpp:8-26) -> CD_ERR_DATA on bad dims. */
CD_API int cd_layer_create(int device, int64_t d_model, int64_t d_inter, int activation, int dtype,
                    const float* w_up, const float* w_gate, const float* w_down, cd_layer** out);

/* Tensor-parallel shard: keeps neurons [row_begin, row_end) of a d_inter_total-wide layer
 * (contiguous rows of the neuron-major matrices).  w_* are the FULL
 * d_inter_total x d_model host matrices. */
CD_API int cd_layer_create_shard(int device, int64_t d_model, int64_t d_inter_total, int64_t row_begin,
                          int64_t row_end, int activation, int dtype, const float* w_up,
                          const float* w_gate, const float* w_down, cd_layer** out);

/* Attach the low-rank predictor (LowRankPredictor, predictor.hpp:15-21).  theta_b is the full
 * d_rank x d_inter_total matrix; a shard keeps its columns.  Stored transposed (neuron-major). */
CD_API int cd_layer_set_predictor(cd_layer* h, int64_t d_rank, const float* theta_a,
                           const float* theta_b);

/* read_model (model_io.cpp:140-224) straight to the device: parses and validates a CDWN1 model
 * file exactly as the reference does (magic, header schema, byte counts, finite values ->
 * CD_ERR_DATA with the reference's messages), uploads the layer in `dtype` and attaches a
 * low-rank predictor.  dims_out[5] (optional) = {d_model, d_inter, d_rank, activation, seed}
 * (seed: the header's uint64 bit pattern, read exactly as get<uint64_t>, model_io.cpp:153);
 * d_rank is 0 without a predictor and -1 for a ternary predictor (not attached: the B200 path
 * runs the low-rank predictor only). */
CD_API int cd_layer_load_cdwn1(int device, const char* path, int dtype, cd_layer** out, int64_t* dims_out);

CD_API int cd_layer_destroy(cd_layer* h);

CD_API int cd_layer_shape(const cd_layer* h, int64_t* d_model, int64_t* d_inter, int64_t* d_rank,
                   int* dtype, int* activation);

/* Device bytes held by the handle (weights + scratch). */
CD_API int cd_layer_device_bytes(const cd_layer* h, int64_t* bytes);

/* Kernel launches issued by the most recent forward call on this handle. */
CD_API int cd_layer_last_launches(const cd_layer* h, int* launches);

/* Engine that ran the most recent forward call: CD_PATH_EXACT (ordered folds, CUDA cores),
 * CD_PATH_FAST (fused sparse kernels, CUDA cores, batch chunks of 4) or CD_PATH_TENSOR
 * (bf16 layer at batch >= 8, M-CountDown / CATS from batch 3: masked row-union GEMM on the tcgen05 tensor cores). */
#define CD_PATH_EXACT 0
#define CD_PATH_FAST 1
#define CD_PATH_TENSOR 2
CD_API int cd_layer_last_path(const cd_layer* h, int* path);

/* Engine selection (no reference equivalent: the reference has one CPU engine).  Default:
 * all on.  CD_ENGINE_FUSED: batch <= 4 D-/M-CountDown steps as one persistent kernel (off:
 * the multi-kernel chains).  CD_ENGINE_TENSOR: bf16 layers at batch >= 8 on the tcgen05
 * masked row-union GEMM (off: the CUDA-core kernels in chunks of 4).  CD_ENGINE_HOST_GRAPH:
 * host-buffer calls replay a captured CUDA graph of their whole sequence.  Results stay
 * within each reduction mode's contract whatever the selection; this is for A/B tests.
 * CD_ENGINE_PDL_CHAIN (off by default): the batch-1..4 persistent kernels (k_dc_fused,
 * k_mc_fused) are launched with programmatic dependent launch instead of as cooperative
 * grids, so a step's prologue overlaps the previous step's tail (1.4 us per Llama-shape step
 * measured).  The caller then guarantees that no other kernel shares the device while these
 * run (their CTAs wait on each other; a cooperative launch makes the driver guarantee it). */
#define CD_ENGINE_FUSED 1
#define CD_ENGINE_TENSOR 2
#define CD_ENGINE_HOST_GRAPH 4
#define CD_ENGINE_ALL 7
#define CD_ENGINE_PDL_CHAIN 8
CD_API int cd_layer_set_engines(cd_layer* h, int engines);

/* ---------------------------------------------------------------- host-buffer operators
 * Synchronous: inputs are read from host memory, outputs written to host memory before
 * return.  Optional outputs may be NULL. */

/* exec_dense (blocked_exec.hpp:34-35): dense three-projection forward, every lane alive. */
CD_API int cd_exec_dense(cd_layer* h, int64_t batch, const float* x, int reduction, float* y);

/* exec_mc (blocked_exec.hpp:39-40): masked gate GEMV fused with act(gate)*u, masked down.
 * u: batch x d_inter (only alive lanes are read); mask: batch x d_inter. */
CD_API int cd_exec_mc(cd_layer* h, int64_t batch, const float* x, const float* u, const uint8_t* mask,
               int reduction, float* y);

/* exec_dc (blocked_exec.hpp:47-48): fused masked up/gate GEMV, masked down. */
CD_API int cd_exec_dc(cd_layer* h, int64_t batch, const float* x, const uint8_t* mask, int reduction,
               float* y);

/* exec_cats (blocked_exec.hpp:43-44): masked up GEMV times the caller's act(gate)
 * (batch x d_inter, only alive lanes read), masked down.  CATS is the paper's comparison
 * baseline, not the COUNTDOWN hot path. */
CD_API int cd_exec_cats(cd_layer* h, int64_t batch, const float* x, const float* act_gate,
                        const uint8_t* mask, int reduction, float* y);

/* pipeline_cats (blocked_exec.hpp:63-64): h = act(W_gate x), mask = |h| > tau (strict),
 * exec_cats.  act_out: batch x d_inter (optional). */
CD_API int cd_pipeline_cats(cd_layer* h, int64_t batch, const float* x, float tau, int reduction,
                            float* y, uint8_t* mask_out, int64_t* alive_out, float* act_out);

/* pipeline_mc (blocked_exec.hpp:60-61) / forward_practical MC (sparsity.hpp:53-54):
 * u = W_up x (dense indicator), mask = |u| > tau (strict), sparse gate/down.
 * alive: per-sample alive counts (batch entries); u_out: batch x d_inter. */
CD_API int cd_pipeline_mc(cd_layer* h, int64_t batch, const float* x, float tau, int reduction,
                   float* y, uint8_t* mask_out, int64_t* alive_out, float* u_out);

/* pipeline_dc (blocked_exec.hpp:67-68) / forward_practical DC: logits = x theta_a theta_b,
 * mask = mask_override (if non-NULL; predictor cost kept, blocked_exec.cpp:366-367) else
 * logits > tau_d (predict_mask, predictor.cpp:140-148, uses tau_d = 0; Alg. 3
 * thresholds at a calibrated tau_D). */
CD_API int cd_pipeline_dc(cd_layer* h, int64_t batch, const float* x, float tau_d,
                   const uint8_t* mask_override, int reduction, float* y, uint8_t* mask_out,
                   int64_t* alive_out, float* logits_out);

/* predict_logits (predictor.hpp:157, low-rank variant): bitwise equal to the reference. */
CD_API int cd_predict_logits(cd_layer* h, int64_t batch, const float* x, float* logits);

/* ---------------------------------------------------------------- device-pointer hot path
 * Asynchronous on `stream` (a cudaStream_t; NULL = the handle's stream), no host
 * synchronisation and no allocation, so a sequence of calls can be captured in a CUDA graph.
 * d_x: batch x d_model f32 device buffer; d_y: batch x d_model (overwritten).
 * method CD_METHOD_DENSE ignores tau.  Optional outputs (NULL to skip):
 *   d_mask: batch x d_inter uint8, d_indicator: batch x d_inter f32 (u for MC, logits for
 *   DC), d_alive: batch int32 per-sample alive counts.
 * d_mask_override (DC only, NULL for the thresholded path): batch x d_inter uint8.
 * The step kernels are persistent (one CTA per SM, all resident at once): calls must not
 * execute concurrently with another handle's call on a different stream of the same device
 * (order them on one stream, or join the streams).  The host-buffer entry points use one
 * internal stream per device and are safe from any thread. */
CD_API int cd_forward_device(cd_layer* h, int method, int64_t batch, const float* d_x, float tau,
                      int reduction, const uint8_t* d_mask_override, float* d_y,
                      uint8_t* d_mask, float* d_indicator, int32_t* d_alive, void* stream);

/* cd_forward_device on RMSNorm(d_x): each sample's input is x / sqrt(mean(x^2) + rms_eps)
 * (no gain).  This is the chaining of configs[3]'s layer stack (layer l+1's
 * input is the RMS-normalised y_l; the reference has no residual), so a decode step of a
 * stack is one call per layer on the previous layer's (all-reduced) output with no separate
 * norm kernel: k_dc_fused normalises inside the step; the other engines run one norm kernel
 * first.  rms_eps must be finite and >= 0 (CD_ERR_DATA otherwise). */
CD_API int cd_forward_device_normed(cd_layer* h, int method, int64_t batch, const float* d_x,
                                    float rms_eps, float tau, int reduction,
                                    const uint8_t* d_mask_override, float* d_y, uint8_t* d_mask,
                                    float* d_indicator, int32_t* d_alive, void* stream);

/* Weight prefetch across a sequence of layers (a decode step through a stack, or layers
 * replayed in a fixed order): every fused D-CountDown step on `h` prefetches the predictor of
 * `next` (same shape, dtype and rank) into L2 once its own records are issued, so the step that
 * runs `next` reads its theta from L2 -- the HBM bytes move under this step's record stream,
 * off the next step's latent -> logits chain.  Weights only: correct whatever runs next.
 * NULL clears.  Re-issue after cd_layer_set_predictor(next, ...) (the theta buffers move). */
CD_API int cd_layer_set_prefetch(cd_layer* h, const cd_layer* next);

/* Block until all work queued on the handle's stream has finished. */
CD_API int cd_layer_sync(cd_layer* h);

/* ---------------------------------------------------------------- predictor-only handle
 * For predict_logits / predict_mask on a bare Predictor (predictor.hpp:157-160): a handle that
 * holds only theta (forward calls that need W_* fail with CD_ERR_DATA). */
CD_API int cd_predictor_create(int device, int64_t d_model, int64_t d_rank, int64_t d_inter,
                               int dtype, const float* theta_a, const float* theta_b,
                               cd_layer** out);

/* Ternary predictor handle (TernaryPredictor, predictor.hpp:23-34): q is the d_model x d_inter
 * quantized view (TernaryPredictor::quantized(), codes -1 / 0 / 1) and gamma its scale
 * (gamma()).  cd_predict_logits on it computes z = x @ (gamma * Q) with the reference's fold
 * (predictor.cpp:116-126), bit-identical.  Exact kernels only: the decode hot path is the
 * low-rank predictor. */
CD_API int cd_predictor_create_ternary(int device, int64_t d_model, int64_t d_inter, float gamma,
                                       const int8_t* q, cd_layer** out);

/* ---------------------------------------------------------------- selection / calibration
 * top_m_threshold (numerics.hpp:96-100, numerics.cpp:105-142) for `batch` vectors of n values
 * (host buffers): the m lanes of largest magnitude, ties to the lower index; tau_out[b] = the
 * (m+1)-th magnitude (+inf for m = 0, -inf for m = n); mask_out (batch x n, optional) = those
 * lanes.  signed_order != 0 orders by the value itself instead of |value| (the D-CountDown
 * tau_D calibration).  Errors as the reference: n = 0 or m outside [0, n] -> CD_ERR_DATA. */
CD_API int cd_top_m(int device, int64_t batch, int64_t n, const float* v, int64_t m, int signed_order,
                    float* tau_out, uint8_t* mask_out);
/* The same on device buffers (rows ld apart; mask rows n apart), asynchronous on `stream`. */
CD_API int cd_top_m_device(const float* d_v, int64_t batch, int64_t n, int64_t ld, int64_t m,
                           int signed_order, float* d_tau, uint8_t* d_mask, void* stream);

/* calibrate (calibration.hpp:20-21, calibration.cpp:11-37) on the device: for each of the
 * n_samples inputs xs (host, n_samples x d_model) the exact indicator -- u = W_up x for
 * CD_METHOD_MC, h = act(W_gate x) for CD_METHOD_CATS -- and its exact top-m threshold
 * (m = alive_count_for(k, d_inter)); *tau_hat = their mean in double, ascending sample order.
 * Bit-identical to the reference.  per_sample (optional): the n_samples thresholds.
 * CD_METHOD_DC (no reference equivalent: the reference rejects dc here) calibrates tau_D on the
 * signed predictor logits (Alg. 3) the same way. */
CD_API int cd_calibrate(cd_layer* h, int method, int64_t n_samples, const float* xs, double k,
                        double* tau_hat, float* per_sample);

/* ---------------------------------------------------------------- timing
 * bench() (blocked_exec.hpp:85-86) device analogue: upload x (batch x d_model, host) once, run
 * `warmup` untimed forwards, then `iters` forwards each bracketed by CUDA events on the
 * handle's stream; ns_out[i] receives iteration i's device time in nanoseconds. */
CD_API int cd_bench_device(cd_layer* h, int method, int64_t batch, const float* x, float tau,
                           int reduction, int64_t warmup, int64_t iters, int64_t* ns_out);

/* Per-kernel device time of the fused chain (UnorderedAccumulate, batch <= 4): the chain runs
 * `warmup + iters` times, rotating over the n_handles layers (so a layer's rows are evicted
 * from L2 between its uses when the handles together exceed L2), with programmatic dependent
 * launch OFF and a CUDA event after every kernel.  stage_ns_out[k] receives the SUM over the
 * timed iterations of stage k's time; *n_stages_out the number of stages (DC: 1, the fused
 * persistent kernel, or 3 -- latent, indicator, sparse FFN -- where the fused kernel does not
 * cover the shape; MC 2: indicator, sparse FFN; dense 1).  d_x: batch x d_model device
 * f32.  Used for the roofline of the dominant kernel; the bench's headline rate is timed
 * with the chain PDL-overlapped (cd_forward_device in a CUDA graph). */
CD_API int cd_bench_stages(cd_layer* const* hs, int n_handles, int method, int64_t batch,
                           const float* d_x, float tau, int64_t warmup, int64_t iters,
                           int64_t* stage_ns_out, int* n_stages_out);

/* ---------------------------------------------------------------- synthetic inputs
 * The reference bench()'s seeded workload (blocked_exec.cpp:396-415): make_random_layer
 * (gated_mlp.cpp:61-75) then x ~ N(0,1) then make_lowrank_predictor on rng.fork()
 * (predictor.cpp:52-69), bit-identical to the reference's Rng (numerics.cpp:11-24).
 * Any output may be NULL; d_rank <= 0 skips the predictor. */
CD_API int cd_synth_layer(uint64_t seed, int64_t d_model, int64_t d_inter, int64_t d_rank,
                          float* w_up, float* w_gate, float* w_down, float* x, float* theta_a,
                          float* theta_b);
/* n draws of Rng(seed).normal_f() (extra decode inputs, calibration samples). */
CD_API int cd_synth_normals(uint64_t seed, int64_t n, float* out);

#ifdef __cplusplus
}
#endif

#endif /* COUNTDOWN_B200_H */
