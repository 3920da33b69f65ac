// kernels_tc.h -- batched decode / prefill on the tensor cores (kernels_tc.cu).
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "kernels.h"

namespace cdk {
namespace tc {

// Arguments of the phase-A kernel (k_tc_gateup).
struct GateUpArgs {
    int F = 0, nb = 0;
    int nbt = 0;        // samples (tokens) per n-tile
    int N = 0;          // UMMA N: 2 nbt (split) or nbt
    int kb_x = 0;       // 64-wide k-blocks over d
    int kb_z = 0;       // 64-wide k-blocks over r (D-CountDown predictor fused), else 0
    int stages = 0;
    int tmem_cols = 0;
    int tiles = 0;      // m-tiles x n-tiles
    int n_tiles = 0;
    int dp = 0;                 // whole tiles in waves (prefill) instead of stream-K ranges
    int mc = 0;                 // dp with 2-CTA clusters multicasting the weight boxes
    int nbuf = 1, buf_cols = 0; // TMEM accumulator buffers and columns per buffer
    float* ws = nullptr;        // stream-K partial accumulators, one slot per CTA
    unsigned* flags = nullptr;  // one release flag per CTA (zero between launches)
    unsigned long long* tl = nullptr;  // development: per-CTA globaltimer stamps (8 per CTA) or null
    float tau = 0.0f;
    const uint8_t* ovr = nullptr;     // nb x F mask override (D-CountDown) or null
    __nv_bfloat16* s_out = nullptr;   // s rows (pair layout in split mode)
    int64_t ld_s = 0;
    uint8_t* mask_out = nullptr;      // nb x F
    float* ind_out = nullptr;         // nb x F: DC logits, MC u, CATS act(gate), dense u
    int* alive_out = nullptr;         // nb
};

// Tiling of a batch: `split` carries activations as bf16 (hi, lo) pairs (decode); nbt samples per
// n-tile; rows = B-operand rows of the whole batch (n_tiles x N).
struct Plan {
    int split = 1, nbt = 0, N = 0, n_tiles = 0;
    int64_t rows = 0;
};

Plan plan_for(int64_t nb, int method);
size_t workspace_bytes(const LayerDev& L, const Plan& p, int num_sms);

// One batched FFN step: y (nb x d f32) from x (nb x d f32), bf16 weights only.  DC uses the
// attached predictor (or `ovr`), MC |u| > tau, CATS |act(g)| > tau, dense all rows.
// `ws` holds workspace_bytes(L, p); `flags` kMaxCtas zero-initialised words (left zero);
// alive_out is zeroed and accumulated.  Returns
// cudaErrorInvalidValue for layers it does not cover (f32 weights, missing predictor).
cudaError_t launch_batched(const LayerDev& L, const Plan& p, void* ws, unsigned* flags, int method, int64_t nb,
                           const float* x, float tau, const uint8_t* ovr, float* y, uint8_t* mask_out,
                           float* ind_out, int* alive_out, const LaunchCfg& c);

// The same step (split mode only) as ONE persistent kernel (kernels_tc_fused.cu): latent,
// gate/up + masks, down.  `ws` of ws_bytes (workspace_bytes); flags: kMaxCtas + 4 zeroed words.
cudaError_t launch_batched_fused(const LayerDev& L, const Plan& p, void* ws, size_t ws_bytes, unsigned* flags,
                                 int method, int64_t nb, const float* x, float tau, const uint8_t* ovr, float* y,
                                 uint8_t* mask_out, float* ind_out, int* alive_out, const LaunchCfg& c);

}  // namespace tc
}  // namespace cdk
