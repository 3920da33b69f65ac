/*
 * countdown_oracle.h -- CPU ORACLE for the COUNTDOWN sparse Gated-MLP decode path.
 *
 * TEST INFRASTRUCTURE ONLY.  This is a plain-C restatement of the reference
 * algorithm (/root/reference/proj/src/*.cpp) used as the parity checker for the
 * CUDA path.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load it.  The product library (libcountdown_b200.so)
 * never links or calls anything here.
 *
 * Parity pinning: every function is checked bit-for-bit against the reference
 * library itself, compiled from /root/reference sources into oracle/_ref/ by
 * oracle/Makefile (tests/test_oracle_vs_ref.py), and against the committed golden
 * vectors in tests/golden/ (generated from oracle/_ref by tests/golden/make_golden.py)
 * plus the reference unit tests' frozen integers and hand examples.
 *
 * Arithmetic contract (matches the reference build: x86-64 SSE, no FMA
 * contraction -- compile with -ffp-contract=off):
 *   - every dot product is a fresh f32 accumulator folded in ascending index
 *     order with separate multiply and add roundings;
 *   - activations are evaluated in double and rounded once to f32.
 */
#ifndef COUNTDOWN_ORACLE_H
#define COUNTDOWN_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CDO_OK 0
#define CDO_DATA_ERROR 2

#define CDO_ACT_SILU 0
#define CDO_ACT_GELU_TANH 1

/* splitmix64 + Box-Muller with a cached spare (numerics.hpp:33-61, numerics.cpp:11-24). */
typedef struct {
    uint64_t state;
    int has_spare;
    double spare;
} cdo_rng;

void cdo_rng_init(cdo_rng* r, uint64_t seed);
uint64_t cdo_rng_next_u64(cdo_rng* r);
double cdo_rng_uniform(cdo_rng* r);
double cdo_rng_normal(cdo_rng* r);
float cdo_rng_normal_f(cdo_rng* r, float mean, float stddev);
/* Rng::fork(): a child seeded with next_u64() (numerics.hpp:56). Returns the child's seed. */
uint64_t cdo_rng_fork_seed(cdo_rng* r);
/* Fills n values with normal_f(0, 1), the bench/test input convention (blocked_exec.cpp:398-399). */
void cdo_fill_normal(cdo_rng* r, float* out, int64_t n);

/* make_random_layer (gated_mlp.cpp:61-75): N(0, 1/sqrt(d)) fill of W_up, W_gate, W_down,
 * each d_inter x d_model row-major, in that order. */
void cdo_make_random_layer(cdo_rng* r, int64_t d_model, int64_t d_inter, float* w_up,
                           float* w_gate, float* w_down);
/* make_lowrank_predictor (predictor.cpp:52-69): theta_a (d x r) then theta_b (r x F),
 * U(-1/sqrt(fan_in), +1/sqrt(fan_in)). */
void cdo_make_lowrank_predictor(cdo_rng* r, int64_t d_model, int64_t d_rank, int64_t d_inter,
                                float* theta_a, float* theta_b);

/* numerics.cpp:47-67 */
float cdo_silu(float x);
float cdo_gelu_tanh(float x);
float cdo_act(int act, float x);

/* gemv (numerics.cpp:77-87): out[i] = sum_j w[i][j] x[j], j ascending. */
void cdo_gemv(const float* w, int64_t rows, int64_t cols, const float* x, float* out);

/* alive_count_for (sparsity.cpp:19-27); returns -1 for k outside (0,1) or d_inter <= 0. */
int64_t cdo_alive_count_for(double k, int64_t d_inter);

/* top_m_threshold (numerics.cpp:105-142). mask_out may be NULL. Returns CDO_DATA_ERROR for
 * n == 0 or m outside [0, n]. */
int cdo_top_m_threshold(const float* v, int64_t n, int64_t m, float* tau_out, uint8_t* mask_out);

/* forward_dense (gated_mlp.cpp:46-59); u, h, s (d_inter) and y (d_model); any may be NULL
 * except y. */
void cdo_forward_dense(int64_t d, int64_t F, int act, const float* w_up, const float* w_gate,
                       const float* w_down, const float* x, float* u, float* h, float* s,
                       float* y);

/* weighted_sum (gated_mlp.cpp:28-44) */
void cdo_weighted_sum(int64_t d, int64_t F, const float* w_down, const float* s,
                      const uint8_t* mask, float* y);

/* forward_sparse (sparsity.cpp:44-71): per alive i ascending, u/g folds, s = u*act(g),
 * y[j] += s * w_down[i][j]. Dead rows are never read. */
void cdo_forward_sparse(int64_t d, int64_t F, int act, const float* w_up, const float* w_gate,
                        const float* w_down, const float* x, const uint8_t* mask, float* y);

/* lowrank_latent / lowrank_logits (predictor.cpp:94-113). latent_out may be NULL. */
void cdo_lowrank_logits(int64_t d, int64_t r, int64_t F, const float* theta_a,
                        const float* theta_b, const float* x, float* latent_out, float* z_out);

/* Practical masks: MC |u| > tau (sparsity.cpp:103-111, blocked_exec.cpp:300-314);
 * DC z > tau_d (predictor.cpp:140-148 with tau_d = 0; tau_d generalises Alg. 3).
 * Return the alive count. */
int64_t cdo_threshold_abs(const float* v, int64_t n, float tau, uint8_t* mask_out);
int64_t cdo_threshold_signed(const float* v, int64_t n, float tau, uint8_t* mask_out);

/* pipeline_mc (blocked_exec.cpp:316-328) semantics: u = gemv(W_up, x); mask = |u| > tau;
 * y = forward_sparse-equivalent (exec_mc, Ordered).  u_out may be NULL. Returns alive. */
int64_t cdo_pipeline_mc(int64_t d, int64_t F, int act, const float* w_up, const float* w_gate,
                        const float* w_down, const float* x, float tau, float* y,
                        uint8_t* mask_out, float* u_out);

/* pipeline_dc (blocked_exec.cpp:350-379): logits = x theta_a theta_b; mask = mask_override or
 * logits > tau_d; y = exec_dc (Ordered). logits_out may be NULL. Returns alive. */
int64_t cdo_pipeline_dc(int64_t d, int64_t F, int64_t r, int act, const float* w_up,
                        const float* w_gate, const float* w_down, const float* theta_a,
                        const float* theta_b, const float* x, float tau_d,
                        const uint8_t* mask_override, float* y, uint8_t* mask_out,
                        float* logits_out);

/* Closed-form element counts (costmodel.cpp:59-103), out[3] = {weight, vector, writes}.
 * Return CDO_DATA_ERROR on a bad shape (costmodel.cpp:15-23). */
int cdo_traffic_dense_split(int64_t d, int64_t F, int64_t out[3]);
int cdo_traffic_mc_split(int64_t d, int64_t F, int64_t s, int64_t out[3]);
int cdo_traffic_dc_split(int64_t d, int64_t F, int64_t r, int64_t s, int64_t out[3]);
int64_t cdo_traffic_dc_oracle(int64_t d, int64_t F, int64_t s);
int64_t cdo_flops_dense(int64_t d, int64_t F, int64_t c_act);
int64_t cdo_flops_mc(int64_t d, int64_t F, int64_t s, int64_t c_act);
int64_t cdo_flops_dc(int64_t d, int64_t F, int64_t r, int64_t s, int64_t c_act);

/* calibrate (calibration.cpp:11-37) for the MC indicator |u|: mean over T samples of each
 * sample's top-m threshold.  xs is T x d row-major.  Returns CDO_DATA_ERROR on bad input. */
int cdo_calibrate_mc(int64_t d, int64_t F, const float* w_up, const float* xs, int64_t T,
                     double k, double* tau_hat_out);

#ifdef __cplusplus
}
#endif

#endif
