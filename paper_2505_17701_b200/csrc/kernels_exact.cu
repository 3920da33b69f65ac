// kernels_exact.cu -- DeterministicOrdered path: bitwise equal to the reference CPU folds.
//
// The reference evaluates every dot product as a fresh f32 accumulator folded in ascending
// index order, multiply and add rounded separately (numerics.cpp:77-87, sparsity.cpp:44-71,
// predictor.cpp:94-113; its x86-64 build has no FMA), activations in double with one
// rounding (numerics.cpp:47-57), and y as the ascending-i fold of weighted_sum
// (gated_mlp.cpp:28-44).  These kernels restate exactly that with one thread per output
// element (__fmul_rn / __fadd_rn forbid FMA contraction), so masks, s and y match the
// reference bit-for-bit; they back Reduction::DeterministicOrdered and the oracle-mode
// parity tests.  Also here: the ordered union compaction shared with the fast path and the
// weight-layout packing kernels.
#include "common.cuh"
#include "kernels.h"
#include "launch.cuh"

namespace cdk {

namespace {

template <typename W> __device__ __forceinline__ float ldw(const W* p) { return to_f32(*p); }

// ============================================================================ compaction
// Single CTA, ascending-neuron union compaction.
//   mode 0: alive_b(i) = |ind[b][i]| > tau   (MC, blocked_exec.cpp:300-314)
//   mode 1: alive_b(i) =  ind[b][i]  > tau   (DC, predictor.cpp:140-148 with tau = tau_D)
//   mode 2: alive_b(i) = masks[b][i] != 0    (caller-supplied masks: exec_mc / exec_dc / override)
//   mode 3: every lane alive                 (dense)
// Writes list / bits / count, per-sample alive counts, optional masks, optional MC u per entry,
// and zeroes y when given (fast path accumulates into it).
__global__ void __launch_bounds__(1024) k_compact(LayerDev L, Scratch S, int mode,
                                                  const float* __restrict__ ind,
                                                  const uint8_t* __restrict__ masks,
                                                  const float* __restrict__ u_full, int nb,
                                                  float tau, uint8_t* __restrict__ mask_out,
                                                  int* __restrict__ alive_out, float* __restrict__ y) {
    __shared__ int warp_tot[32];
    __shared__ int alive_s[kMaxBatch];
    const int t = threadIdx.x, lane = t % kWarp, warp = t / kWarp;
    if (t < kMaxBatch) alive_s[t] = 0;
    if (y)
        for (int64_t i = t; i < (int64_t)nb * L.d; i += blockDim.x) y[i] = 0.0f;
    __syncthreads();
    auto alive_of = [&](int b, int64_t i) -> bool {
        switch (mode) {
            case 0: return fabsf(ind[b * L.F + i]) > tau;
            case 1: return ind[b * L.F + i] > tau;
            case 2: return masks[b * L.F + i] != 0;
            default: return true;
        }
    };
    const int64_t seg = (L.F + blockDim.x - 1) / blockDim.x;
    const int64_t i0 = imin64(L.F, t * seg), i1 = imin64(L.F, i0 + seg);
    int cnt = 0;
    for (int64_t i = i0; i < i1; ++i) {
        bool any = false;
        for (int b = 0; b < nb; ++b) any |= alive_of(b, i);
        cnt += any;
    }
    int incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
    }
    if (lane == 31) warp_tot[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        const int nw = blockDim.x / kWarp;
        int v = lane < nw ? warp_tot[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int u = __shfl_up_sync(0xffffffffu, v, o);
            if (lane >= o) v += u;
        }
        if (lane < nw) warp_tot[lane] = v;
    }
    __syncthreads();
    int pos = incl - cnt + (warp > 0 ? warp_tot[warp - 1] : 0);
    int my_alive[kMaxBatch];
    for (int b = 0; b < nb; ++b) my_alive[b] = 0;
    for (int64_t i = i0; i < i1; ++i) {
        uint32_t bits = 0;
        for (int b = 0; b < nb; ++b) {
            const bool a = alive_of(b, i);
            bits |= (a ? 1u : 0u) << b;
            my_alive[b] += a;
            if (mask_out) mask_out[b * L.F + i] = a ? 1 : 0;
        }
        if (bits) {
            S.list[pos] = static_cast<int32_t>(i);
            S.bits[pos] = bits;
            if (u_full)
                for (int b = 0; b < nb && b < kMaxBatchFast; ++b)
                    S.list_val[(int64_t)pos * kMaxBatchFast + b] =
                        ((bits >> b) & 1u) ? u_full[b * L.F + i] : 0.0f;
            ++pos;
        }
    }
    for (int b = 0; b < nb; ++b)
        if (my_alive[b]) atomicAdd(&alive_s[b], my_alive[b]);
    __syncthreads();
    if (t == blockDim.x - 1) *S.count = pos;  // the last segment ends at the total
    if (t < nb) {
        S.alive[t] = alive_s[t];
        if (alive_out) alive_out[t] = alive_s[t];
    }
}

// ============================================================================ exact latent
// lowrank_latent (predictor.cpp:94-102): latent[q] = fold_{i asc} x[i] * theta_a[i][q].
template <typename W>
__global__ void ke_latent(LayerDev L, const float* __restrict__ x, float* __restrict__ lat) {
    const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int b = blockIdx.y;
    if (q >= L.ldr) return;
    const W* A = static_cast<const W*>(L.theta_a);
    float acc = 0.0f;
    if (q < L.r)
        for (int64_t i = 0; i < L.d; ++i) acc = __fadd_rn(acc, __fmul_rn(x[b * L.d + i], ldw(A + i * L.ldr + q)));
    lat[b * L.ldr + q] = acc;
}

// ============================================================================ exact row dot
// out[b][row] = fold_{j asc < ncols} W[row][j] * v[b][j]  (gemv numerics.cpp:77-87,
// lowrank_logits predictor.cpp:104-113 over theta_bt).
template <typename W>
__global__ void ke_rowdot(const W* __restrict__ Wm, int64_t nrows, int64_t ld, int64_t ncols,
                          const float* __restrict__ v, int64_t ldv, float* __restrict__ out,
                          int64_t ldo) {
    const int64_t row = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int b = blockIdx.y;
    if (row >= nrows) return;
    const W* wr = Wm + row * ld;
    const float* vb = v + b * ldv;
    float acc = 0.0f;
    for (int64_t j = 0; j < ncols; ++j) acc = __fadd_rn(acc, __fmul_rn(ldw(wr + j), vb[j]));
    out[b * ldo + row] = acc;
}

// ============================================================================ exact phase 1
// DC / dense (exec_dc blocked_exec.cpp:263-281, forward_sparse sparsity.cpp:58-66):
//   s = up * act(gate), up/gate independent ascending folds.
// MC (exec_mc blocked_exec.cpp:188-205): s = act(gate) * u[i].
// Dead (sample, lane) pairs never read their row or their u.
template <typename W>
__global__ void ke_phase1(LayerDev L, Scratch S, int method, const float* __restrict__ x,
                          const float* __restrict__ u_full) {
    const int slot = blockIdx.x * blockDim.x + threadIdx.x;
    const int b = blockIdx.y;
    const int n = *S.count;
    if (slot >= n) return;
    const uint32_t bits = S.bits[slot];
    float s = 0.0f;
    if ((bits >> b) & 1u) {
        const int64_t i = S.list[slot];
        const W* wg = static_cast<const W*>(L.w_gate) + i * L.rs;
        const float* xb = x + b * L.d;
        if (method == kMC) {
            float g = 0.0f;
            for (int64_t j = 0; j < L.d; ++j) g = __fadd_rn(g, __fmul_rn(ldw(wg + j), xb[j]));
            s = __fmul_rn(act_exact(L.act, g), u_full[b * L.F + i]);
        } else if (method == kCATS) {
            // exec_cats (blocked_exec.cpp:227-243): s = (W_up[i] . x) * act_gate[i]
            const W* wu = static_cast<const W*>(L.w_up) + i * L.rs;
            float u = 0.0f;
            for (int64_t j = 0; j < L.d; ++j) u = __fadd_rn(u, __fmul_rn(ldw(wu + j), xb[j]));
            s = __fmul_rn(u, u_full[b * L.F + i]);
        } else {
            const W* wu = static_cast<const W*>(L.w_up) + i * L.rs;
            float u = 0.0f, g = 0.0f;
            for (int64_t j = 0; j < L.d; ++j) {
                u = __fadd_rn(u, __fmul_rn(ldw(wu + j), xb[j]));
                g = __fadd_rn(g, __fmul_rn(ldw(wg + j), xb[j]));
            }
            s = __fmul_rn(u, act_exact(L.act, g));
        }
    }
    S.ex_s[(int64_t)b * L.F + slot] = s;
}

// ============================================================================ exact activation
// pipeline_cats (blocked_exec.cpp:338-341): act[i] = apply_activation(gate[i]), in place.
__global__ void ke_act(int act, float* __restrict__ v, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        v[i] = act_exact(act, v[i]);
}

// ternary predictor input (predictor.cpp:116-126): out[i] = x[i] * gamma, one f32 rounding.
__global__ void ke_scale(const float* __restrict__ x, int64_t n, float g, float* __restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = __fmul_rn(x[i], g);
}

// ============================================================================ exact down projection
// down_projection Ordered (blocked_exec.cpp:85-97) == weighted_sum (gated_mlp.cpp:28-44):
// y[j] = fold over alive i ascending of s[i] * W_down[i][j]; one thread per column.
template <typename W>
__global__ void ke_down(LayerDev L, Scratch S, float* __restrict__ y) {
    const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int b = blockIdx.y;
    if (j >= L.d) return;
    const int n = *S.count;
    const W* WD = static_cast<const W*>(L.w_down);
    const float* sb = S.ex_s + (int64_t)b * L.F;
    float acc = 0.0f;
    for (int slot = 0; slot < n; ++slot) {
        if (!((S.bits[slot] >> b) & 1u)) continue;
        acc = __fadd_rn(acc, __fmul_rn(sb[slot], ldw(WD + (int64_t)S.list[slot] * L.rs + j)));
    }
    y[b * L.d + j] = acc;
}

// ============================================================================ layout packing
template <typename W> __device__ __forceinline__ W from_f32(float v);
template <> __device__ __forceinline__ float from_f32<float>(float v) { return v; }
template <> __device__ __forceinline__ __nv_bfloat16 from_f32<__nv_bfloat16>(float v) {
    return __float2bfloat16_rn(v);  // RNE, SURVEY.md section 8d
}

template <typename W>
__global__ void k_pack_rows(const float* __restrict__ src, int64_t rows, int64_t cols,
                            int64_t ld_src, W* __restrict__ dst, int64_t ld_pad, int64_t ld_dst) {
    const int64_t n = rows * ld_pad;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = e / ld_pad, c = e % ld_pad;
        dst[r * ld_dst + c] = from_f32<W>(c < cols ? src[r * ld_src + c] : 0.0f);
    }
}

// dst[c][r] = src[r][col_begin + c] for c < cols_sel, r < rows; zero for r in [rows, ld_dst).
template <typename W>
__global__ void k_pack_transpose(const float* __restrict__ src, int64_t rows, int64_t ld_src,
                                 int64_t col_begin, int64_t cols_sel, W* __restrict__ dst,
                                 int64_t ld_dst) {
    __shared__ float tile[32][33];
    const int64_t r0 = blockIdx.y * 32, c0 = blockIdx.x * 32;
    for (int k = threadIdx.y; k < 32; k += blockDim.y) {
        const int64_t r = r0 + k, c = c0 + threadIdx.x;
        tile[k][threadIdx.x] = (r < rows && c < cols_sel) ? src[r * ld_src + col_begin + c] : 0.0f;
    }
    __syncthreads();
    for (int k = threadIdx.y; k < 32; k += blockDim.y) {
        const int64_t c = c0 + k, r = r0 + threadIdx.x;
        if (c < cols_sel && r < ld_dst) dst[c * ld_dst + r] = from_f32<W>(tile[threadIdx.x][k]);
    }
}

}  // namespace

// ---------------------------------------------------------------- launchers
cudaError_t launch_compact_masks(const LayerDev& L, const Scratch& S, const uint8_t* masks,
                                 const float* u_full, int nb, float* y, const LaunchCfg& c) {
    return launch_ex(k_compact, dim3(1), dim3(1024), 0, c, false, L, S, masks ? 2 : 3,
                     (const float*)nullptr, masks, u_full, nb, 0.0f, (uint8_t*)nullptr,
                     (int*)nullptr, y);
}

cudaError_t launch_exact_compact(const LayerDev& L, const Scratch& S, int mode, const float* ind,
                                 const uint8_t* masks_in, int nb, float tau, uint8_t* mask_out,
                                 int* alive_out, const LaunchCfg& c) {
    return launch_ex(k_compact, dim3(1), dim3(1024), 0, c, false, L, S, mode, ind, masks_in,
                     (const float*)nullptr, nb, tau, mask_out, alive_out, (float*)nullptr);
}

cudaError_t launch_exact_latent(const LayerDev& L, const Scratch& S, const float* x, int nb,
                                const LaunchCfg& c) {
    dim3 grid(static_cast<unsigned>((L.ldr + 127) / 128), nb);
    if (L.dtype == kBF16) return launch_ex(ke_latent<__nv_bfloat16>, grid, dim3(128), 0, c, false, L, x, S.ex_lat);
    return launch_ex(ke_latent<float>, grid, dim3(128), 0, c, false, L, x, S.ex_lat);
}

cudaError_t launch_exact_rowdot_all(const void* W, int dtype, int64_t nrows, int64_t ld,
                                    int64_t ncols, const float* v, int64_t ldv, int nb,
                                    float* out, int64_t ldo, const LaunchCfg& c) {
    dim3 grid(static_cast<unsigned>((nrows + 127) / 128), nb);
    if (dtype == kBF16)
        return launch_ex(ke_rowdot<__nv_bfloat16>, grid, dim3(128), 0, c, false,
                         static_cast<const __nv_bfloat16*>(W), nrows, ld, ncols, v, ldv, out, ldo);
    return launch_ex(ke_rowdot<float>, grid, dim3(128), 0, c, false, static_cast<const float*>(W),
                     nrows, ld, ncols, v, ldv, out, ldo);
}

cudaError_t launch_exact_phase1(const LayerDev& L, const Scratch& S, int method,
                                const float* x, const float* u_full, int nb,
                                const LaunchCfg& c) {
    dim3 grid(static_cast<unsigned>((L.F + 127) / 128), nb);
    if (L.dtype == kBF16)
        return launch_ex(ke_phase1<__nv_bfloat16>, grid, dim3(128), 0, c, false, L, S, method, x, u_full);
    return launch_ex(ke_phase1<float>, grid, dim3(128), 0, c, false, L, S, method, x, u_full);
}

cudaError_t launch_exact_act(int act, float* v, int64_t n, const LaunchCfg& c) {
    const int blocks = static_cast<int>(imin64(1024, (n + 255) / 256));
    return launch_ex(ke_act, dim3(blocks), dim3(256), 0, c, false, act, v, n);
}

cudaError_t launch_exact_scale(const float* x, int64_t n, float g, float* out, const LaunchCfg& c) {
    const int blocks = static_cast<int>(imin64(1024, (n + 255) / 256));
    return launch_ex(ke_scale, dim3(blocks), dim3(256), 0, c, false, x, n, g, out);
}

cudaError_t launch_exact_down(const LayerDev& L, const Scratch& S, int nb, float* y,
                              const LaunchCfg& c) {
    dim3 grid(static_cast<unsigned>((L.d + 127) / 128), nb);
    if (L.dtype == kBF16) return launch_ex(ke_down<__nv_bfloat16>, grid, dim3(128), 0, c, false, L, S, y);
    return launch_ex(ke_down<float>, grid, dim3(128), 0, c, false, L, S, y);
}

cudaError_t launch_pack_rows(const float* src, int64_t rows, int64_t cols, int64_t ld_src,
                             void* dst, int dtype, int64_t ld_pad, int64_t ld_dst, cudaStream_t s) {
    const int blocks = static_cast<int>(imin64(4096, (rows * ld_pad + 255) / 256));
    if (dtype == kBF16)
        k_pack_rows<__nv_bfloat16><<<blocks, 256, 0, s>>>(src, rows, cols, ld_src,
                                                          static_cast<__nv_bfloat16*>(dst), ld_pad, ld_dst);
    else
        k_pack_rows<float><<<blocks, 256, 0, s>>>(src, rows, cols, ld_src, static_cast<float*>(dst), ld_pad,
                                                  ld_dst);
    return cudaGetLastError();
}

cudaError_t launch_pack_transpose(const float* src, int64_t rows, int64_t ld_src,
                                  int64_t col_begin, int64_t cols_sel, void* dst, int dtype,
                                  int64_t ld_dst, cudaStream_t s) {
    dim3 grid(static_cast<unsigned>((cols_sel + 31) / 32), static_cast<unsigned>((ld_dst + 31) / 32));
    dim3 block(32, 8);
    if (dtype == kBF16)
        k_pack_transpose<__nv_bfloat16><<<grid, block, 0, s>>>(src, rows, ld_src, col_begin, cols_sel,
                                                               static_cast<__nv_bfloat16*>(dst), ld_dst);
    else
        k_pack_transpose<float><<<grid, block, 0, s>>>(src, rows, ld_src, col_begin, cols_sel,
                                                       static_cast<float*>(dst), ld_dst);
    return cudaGetLastError();
}

}  // namespace cdk
