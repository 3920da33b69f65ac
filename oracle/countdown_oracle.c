/*
 * countdown_oracle.c -- CPU ORACLE (test infrastructure only; see countdown_oracle.h).
 *
 * A plain-C restatement of the reference's decode-path semantics.  Each function
 * cites the reference file:line it restates (paths relative to
 * /root/reference/proj/).  Build with -ffp-contract=off so that every
 * `acc += a * b` rounds the product and the sum separately, exactly as the
 * reference's baseline x86-64 build does (no FMA instructions in its objects).
 */
#include "countdown_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ---- Rng: numerics.hpp:33-61, numerics.cpp:11-24 ------------------------------ */

void cdo_rng_init(cdo_rng* r, uint64_t seed) {
    r->state = seed;
    r->has_spare = 0;
    r->spare = 0.0;
}

uint64_t cdo_rng_next_u64(cdo_rng* r) {
    r->state += 0x9E3779B97F4A7C15ull;
    uint64_t z = r->state;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

double cdo_rng_uniform(cdo_rng* r) {
    return (double)(cdo_rng_next_u64(r) >> 11) * 0x1.0p-53;
}

double cdo_rng_normal(cdo_rng* r) {
    if (r->has_spare) {
        r->has_spare = 0;
        return r->spare;
    }
    double u1 = 1.0 - cdo_rng_uniform(r);
    double u2 = cdo_rng_uniform(r);
    double rad = sqrt(-2.0 * log(u1));
    double a = 6.283185307179586476925286766559 * u2;
    r->spare = rad * sin(a);
    r->has_spare = 1;
    return rad * cos(a);
}

float cdo_rng_normal_f(cdo_rng* r, float mean, float stddev) {
    return mean + stddev * (float)cdo_rng_normal(r);
}

uint64_t cdo_rng_fork_seed(cdo_rng* r) { return cdo_rng_next_u64(r); }

void cdo_fill_normal(cdo_rng* r, float* out, int64_t n) {
    for (int64_t i = 0; i < n; ++i) out[i] = cdo_rng_normal_f(r, 0.0f, 1.0f);
}

/* ---- layer / predictor generation ------------------------------------------ */

/* gated_mlp.cpp:61-75: std = 1/sqrt(float(d)), fill W_up, W_gate, W_down row-major. */
void cdo_make_random_layer(cdo_rng* r, int64_t d_model, int64_t d_inter, float* w_up,
                           float* w_gate, float* w_down) {
    const float sd = 1.0f / sqrtf((float)d_model);
    const int64_t n = d_model * d_inter;
    float* mats[3] = {w_up, w_gate, w_down};
    for (int m = 0; m < 3; ++m)
        for (int64_t i = 0; i < n; ++i) mats[m][i] = cdo_rng_normal_f(r, 0.0f, sd);
}

/* predictor.cpp:52-55 */
static void fill_uniform(float* m, int64_t n, int64_t fan_in, cdo_rng* r) {
    const float bound = 1.0f / sqrtf((float)fan_in);
    for (int64_t i = 0; i < n; ++i) m[i] = bound * (float)(2.0 * cdo_rng_uniform(r) - 1.0);
}

/* predictor.cpp:57-69 */
void cdo_make_lowrank_predictor(cdo_rng* r, int64_t d_model, int64_t d_rank, int64_t d_inter,
                                float* theta_a, float* theta_b) {
    fill_uniform(theta_a, d_model * d_rank, d_model, r);
    fill_uniform(theta_b, d_rank * d_inter, d_rank, r);
}

/* ---- activations: numerics.cpp:47-61 ---------------------------------------- */

float cdo_silu(float x) {
    double xd = x;
    return (float)(xd / (1.0 + exp(-xd)));
}

float cdo_gelu_tanh(float x) {
    double xd = x;
    double inner = 0.7978845608028653558798921198687 * (xd + 0.044715 * xd * xd * xd);
    return (float)(0.5 * xd * (1.0 + tanh(inner)));
}

float cdo_act(int act, float x) { return act == CDO_ACT_SILU ? cdo_silu(x) : cdo_gelu_tanh(x); }

/* ---- gemv: numerics.cpp:77-87 ----------------------------------------------- */

void cdo_gemv(const float* w, int64_t rows, int64_t cols, const float* x, float* out) {
    for (int64_t i = 0; i < rows; ++i) {
        const float* wr = w + i * cols;
        float acc = 0.0f;
        for (int64_t j = 0; j < cols; ++j) acc += wr[j] * x[j];
        out[i] = acc;
    }
}

/* ---- sparsity.cpp:19-27 ------------------------------------------------------- */

int64_t cdo_alive_count_for(double k, int64_t d_inter) {
    if (!(k > 0.0 && k < 1.0)) return -1;
    if (d_inter <= 0) return -1;
    return (int64_t)floor((1.0 - k) * (double)d_inter);
}

/* ---- top_m_threshold: numerics.cpp:105-142 ------------------------------------ */

typedef struct {
    float mag;
    int32_t idx;
} mag_idx;

/* Total order of numerics.cpp:125-130: larger magnitude first, then lower index. */
static int before_cmp(const void* pa, const void* pb) {
    const mag_idx* a = (const mag_idx*)pa;
    const mag_idx* b = (const mag_idx*)pb;
    if (a->mag != b->mag) return a->mag > b->mag ? -1 : 1;
    return a->idx < b->idx ? -1 : (a->idx > b->idx ? 1 : 0);
}

int cdo_top_m_threshold(const float* v, int64_t n, int64_t m, float* tau_out,
                        uint8_t* mask_out) {
    if (n == 0) return CDO_DATA_ERROR;
    if (m < 0 || m > n) return CDO_DATA_ERROR;
    if (mask_out) memset(mask_out, 0, (size_t)n);
    if (m == 0) {
        *tau_out = INFINITY;
        return CDO_OK;
    }
    if (m == n) {
        *tau_out = -INFINITY;
        if (mask_out) memset(mask_out, 1, (size_t)n);
        return CDO_OK;
    }
    mag_idx* order = (mag_idx*)malloc(sizeof(mag_idx) * (size_t)n);
    for (int64_t i = 0; i < n; ++i) {
        order[i].mag = fabsf(v[i]);
        order[i].idx = (int32_t)i;
    }
    /* A full sort under the same strict total order selects exactly the set nth_element does. */
    qsort(order, (size_t)n, sizeof(mag_idx), before_cmp);
    *tau_out = order[m].mag;
    if (mask_out)
        for (int64_t i = 0; i < m; ++i) mask_out[order[i].idx] = 1;
    free(order);
    return CDO_OK;
}

/* ---- gated_mlp.cpp:28-59 ------------------------------------------------------ */

void cdo_weighted_sum(int64_t d, int64_t F, const float* w_down, const float* s,
                      const uint8_t* mask, float* y) {
    for (int64_t j = 0; j < d; ++j) y[j] = 0.0f;
    for (int64_t i = 0; i < F; ++i) {
        if (mask && !mask[i]) continue;
        const float si = s[i];
        const float* wr = w_down + i * d;
        for (int64_t j = 0; j < d; ++j) y[j] += si * wr[j];
    }
}

void cdo_forward_dense(int64_t d, int64_t F, int act, const float* w_up, const float* w_gate,
                       const float* w_down, const float* x, float* u, float* h, float* s,
                       float* y) {
    float* uu = (float*)malloc(sizeof(float) * (size_t)F);
    float* hh = (float*)malloc(sizeof(float) * (size_t)F);
    float* ss = (float*)malloc(sizeof(float) * (size_t)F);
    cdo_gemv(w_up, F, d, x, uu);
    cdo_gemv(w_gate, F, d, x, hh);
    for (int64_t i = 0; i < F; ++i) hh[i] = cdo_act(act, hh[i]);
    for (int64_t i = 0; i < F; ++i) ss[i] = uu[i] * hh[i];
    cdo_weighted_sum(d, F, w_down, ss, NULL, y);
    if (u) memcpy(u, uu, sizeof(float) * (size_t)F);
    if (h) memcpy(h, hh, sizeof(float) * (size_t)F);
    if (s) memcpy(s, ss, sizeof(float) * (size_t)F);
    free(uu);
    free(hh);
    free(ss);
}

/* ---- sparsity.cpp:44-71 ------------------------------------------------------- */

void cdo_forward_sparse(int64_t d, int64_t F, int act, const float* w_up, const float* w_gate,
                        const float* w_down, const float* x, const uint8_t* mask, float* y) {
    for (int64_t j = 0; j < d; ++j) y[j] = 0.0f;
    for (int64_t i = 0; i < F; ++i) {
        if (!mask[i]) continue;
        const float* up = w_up + i * d;
        const float* gate = w_gate + i * d;
        float u = 0.0f, g = 0.0f;
        for (int64_t j = 0; j < d; ++j) {
            u += up[j] * x[j];
            g += gate[j] * x[j];
        }
        const float s = u * cdo_act(act, g);
        const float* down = w_down + i * d;
        for (int64_t j = 0; j < d; ++j) y[j] += s * down[j];
    }
}

/* ---- predictor.cpp:94-113 ------------------------------------------------------- */

void cdo_lowrank_logits(int64_t d, int64_t r, int64_t F, const float* theta_a,
                        const float* theta_b, const float* x, float* latent_out, float* z_out) {
    float* latent = (float*)calloc((size_t)r, sizeof(float));
    for (int64_t i = 0; i < d; ++i) {
        const float xi = x[i];
        const float* ar = theta_a + i * r;
        for (int64_t q = 0; q < r; ++q) latent[q] += xi * ar[q];
    }
    for (int64_t j = 0; j < F; ++j) z_out[j] = 0.0f;
    for (int64_t q = 0; q < r; ++q) {
        const float lr = latent[q];
        const float* br = theta_b + q * F;
        for (int64_t j = 0; j < F; ++j) z_out[j] += lr * br[j];
    }
    if (latent_out) memcpy(latent_out, latent, sizeof(float) * (size_t)r);
    free(latent);
}

/* ---- masks: blocked_exec.cpp:300-314, predictor.cpp:140-148 ---------------------- */

int64_t cdo_threshold_abs(const float* v, int64_t n, float tau, uint8_t* mask_out) {
    int64_t alive = 0;
    for (int64_t i = 0; i < n; ++i) {
        const uint8_t a = fabsf(v[i]) > tau ? 1 : 0;
        mask_out[i] = a;
        alive += a;
    }
    return alive;
}

int64_t cdo_threshold_signed(const float* v, int64_t n, float tau, uint8_t* mask_out) {
    int64_t alive = 0;
    for (int64_t i = 0; i < n; ++i) {
        const uint8_t a = v[i] > tau ? 1 : 0;
        mask_out[i] = a;
        alive += a;
    }
    return alive;
}

/* ---- pipelines: blocked_exec.cpp:316-379 -------------------------------------- */

int64_t cdo_pipeline_mc(int64_t d, int64_t F, int act, const float* w_up, const float* w_gate,
                        const float* w_down, const float* x, float tau, float* y,
                        uint8_t* mask_out, float* u_out) {
    float* u = (float*)malloc(sizeof(float) * (size_t)F);
    uint8_t* mask = mask_out ? mask_out : (uint8_t*)malloc((size_t)F);
    cdo_gemv(w_up, F, d, x, u);
    const int64_t alive = cdo_threshold_abs(u, F, tau, mask);
    /* exec_mc phase 1 (blocked_exec.cpp:188-205): s = act(gate . x) * u for alive lanes. */
    float* s = (float*)calloc((size_t)F, sizeof(float));
    for (int64_t i = 0; i < F; ++i) {
        if (!mask[i]) continue;
        const float* wr = w_gate + i * d;
        float acc = 0.0f;
        for (int64_t j = 0; j < d; ++j) acc += wr[j] * x[j];
        s[i] = cdo_act(act, acc) * u[i];
    }
    /* down_projection Ordered (blocked_exec.cpp:85-97) == weighted_sum over alive lanes. */
    cdo_weighted_sum(d, F, w_down, s, mask, y);
    if (u_out) memcpy(u_out, u, sizeof(float) * (size_t)F);
    free(s);
    free(u);
    if (!mask_out) free(mask);
    return alive;
}

int64_t cdo_pipeline_dc(int64_t d, int64_t F, int64_t r, int act, const float* w_up,
                        const float* w_gate, const float* w_down, const float* theta_a,
                        const float* theta_b, const float* x, float tau_d,
                        const uint8_t* mask_override, float* y, uint8_t* mask_out,
                        float* logits_out) {
    float* z = (float*)malloc(sizeof(float) * (size_t)F);
    uint8_t* mask = mask_out ? mask_out : (uint8_t*)malloc((size_t)F);
    cdo_lowrank_logits(d, r, F, theta_a, theta_b, x, NULL, z);
    int64_t alive = 0;
    if (mask_override) {
        memcpy(mask, mask_override, (size_t)F);
        for (int64_t i = 0; i < F; ++i) alive += mask[i] != 0;
    } else {
        alive = cdo_threshold_signed(z, F, tau_d, mask);
    }
    /* exec_dc (blocked_exec.cpp:252-289) Ordered == forward_sparse bitwise. */
    cdo_forward_sparse(d, F, act, w_up, w_gate, w_down, x, mask, y);
    if (logits_out) memcpy(logits_out, z, sizeof(float) * (size_t)F);
    free(z);
    if (!mask_out) free(mask);
    return alive;
}

/* ---- costmodel.cpp:27-103 -------------------------------------------------------- */

int cdo_traffic_dense_split(int64_t d, int64_t F, int64_t out[3]) {
    if (d <= 0 || F <= 0) return CDO_DATA_ERROR;
    out[0] = 3 * d * F;
    out[1] = 2 * d + 4 * F;
    out[2] = 4 * F + d;
    return CDO_OK;
}

int cdo_traffic_mc_split(int64_t d, int64_t F, int64_t s, int64_t out[3]) {
    if (d <= 0 || F <= 0 || s < 0) return CDO_DATA_ERROR;
    out[0] = d * F + 2 * d * s;
    out[1] = 2 * d + 4 * F + s;
    out[2] = 4 * F + d;
    return CDO_OK;
}

int cdo_traffic_dc_split(int64_t d, int64_t F, int64_t r, int64_t s, int64_t out[3]) {
    if (d <= 0 || F <= 0 || r <= 0 || s < 0) return CDO_DATA_ERROR;
    out[0] = d * r + r * F + 3 * d * s;
    out[1] = 2 * d + r + 3 * F;
    out[2] = 3 * F + r + d;
    return CDO_OK;
}

int64_t cdo_traffic_dc_oracle(int64_t d, int64_t F, int64_t s) {
    return 3 * d * s + 2 * d + 3 * F + 3 * F + d;
}

int64_t cdo_flops_dense(int64_t d, int64_t F, int64_t c_act) {
    return 6 * d * F + c_act * F + F;
}

int64_t cdo_flops_mc(int64_t d, int64_t F, int64_t s, int64_t c_act) {
    return 2 * d * F + 2 * F + 4 * d * s + c_act * s + s;
}

int64_t cdo_flops_dc(int64_t d, int64_t F, int64_t r, int64_t s, int64_t c_act) {
    return 2 * d * r + 2 * r * F + F + 6 * d * s + c_act * s + s;
}

/* ---- calibration.cpp:11-37 (MC indicator) ----------------------------------------- */

int cdo_calibrate_mc(int64_t d, int64_t F, const float* w_up, const float* xs, int64_t T,
                     double k, double* tau_hat_out) {
    if (T <= 0) return CDO_DATA_ERROR;
    const int64_t m = cdo_alive_count_for(k, F);
    if (m < 0) return CDO_DATA_ERROR;
    float* u = (float*)malloc(sizeof(float) * (size_t)F);
    double sum = 0.0;
    for (int64_t t = 0; t < T; ++t) {
        float tau = 0.0f;
        cdo_gemv(w_up, F, d, xs + t * d, u);
        cdo_top_m_threshold(u, F, m, &tau, NULL);
        sum += (double)tau;
    }
    free(u);
    *tau_hat_out = sum / (double)T;
    return CDO_OK;
}
