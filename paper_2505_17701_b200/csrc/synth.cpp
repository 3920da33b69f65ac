// synth.cpp -- seeded synthetic inputs for benches and smoke runs (host only).
//
// The reference's bench() builds its workload from a seed (blocked_exec.cpp:396-415):
// make_random_layer (gated_mlp.cpp:61-75) draws W_up, W_gate, W_down ~ N(0, 1/sqrt(d)) from a
// splitmix64 stream with Box-Muller normals (numerics.hpp:33-61, numerics.cpp:11-24), then
// x ~ N(0, 1) from the same stream, then the low-rank predictor from rng.fork()
// (predictor.cpp:52-69).  The product needs the same inputs to measure the same workload, so
// this file implements that generator (with -ffp-contract=off, like the reference build) and
// exposes it through the C-ABI.  It produces data only; no FFN arithmetic lives here.
#include <cmath>
#include <cstdint>
#include <cstring>

#include "../../include/countdown_b200.h"

namespace {

struct SplitMix {
    uint64_t state;
    bool has_spare = false;
    double spare = 0.0;
    explicit SplitMix(uint64_t s) : state(s) {}
    uint64_t next() {
        state += 0x9E3779B97F4A7C15ull;
        uint64_t z = state;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        return z ^ (z >> 31);
    }
    double uniform() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
    double normal() {
        if (has_spare) {
            has_spare = false;
            return spare;
        }
        const double u1 = 1.0 - uniform();
        const double u2 = uniform();
        const double r = std::sqrt(-2.0 * std::log(u1));
        const double a = 6.283185307179586476925286766559 * u2;
        spare = r * std::sin(a);
        has_spare = true;
        return r * std::cos(a);
    }
    float normal_f(float mean, float sd) { return mean + sd * static_cast<float>(normal()); }
};

}  // namespace

extern "C" {

// bench() setup sequence; any output may be NULL (its draws are still consumed so the stream
// position matches the reference).  d_rank <= 0 skips the predictor.
int cd_synth_layer(uint64_t seed, int64_t d_model,
                                                          int64_t d_inter, int64_t d_rank,
                                                          float* w_up, float* w_gate,
                                                          float* w_down, float* x,
                                                          float* theta_a, float* theta_b) {
    if (d_model <= 0 || d_inter <= 0) return CD_ERR_DATA;
    SplitMix rng(seed);
    const float sd = 1.0f / std::sqrt(static_cast<float>(d_model));
    const int64_t n = d_model * d_inter;
    float* mats[3] = {w_up, w_gate, w_down};
    for (float* m : mats)
        for (int64_t i = 0; i < n; ++i) {
            const float v = rng.normal_f(0.0f, sd);
            if (m) m[i] = v;
        }
    for (int64_t i = 0; i < d_model; ++i) {
        const float v = rng.normal_f(0.0f, 1.0f);
        if (x) x[i] = v;
    }
    if (d_rank > 0) {
        SplitMix prng(rng.next());  // Rng::fork()
        const float ba = 1.0f / std::sqrt(static_cast<float>(d_model));
        for (int64_t i = 0; i < d_model * d_rank; ++i) {
            const float v = ba * static_cast<float>(2.0 * prng.uniform() - 1.0);
            if (theta_a) theta_a[i] = v;
        }
        const float bb = 1.0f / std::sqrt(static_cast<float>(d_rank));
        for (int64_t i = 0; i < d_rank * d_inter; ++i) {
            const float v = bb * static_cast<float>(2.0 * prng.uniform() - 1.0);
            if (theta_b) theta_b[i] = v;
        }
    }
    return CD_OK;
}

// n draws of normal_f(0, 1) from Rng(seed): extra decode inputs / calibration samples.
int cd_synth_normals(uint64_t seed, int64_t n, float* out) {
    if (n < 0 || (n > 0 && !out)) return CD_ERR_DATA;
    SplitMix rng(seed);
    for (int64_t i = 0; i < n; ++i) out[i] = rng.normal_f(0.0f, 1.0f);
    return CD_OK;
}

}  // extern "C"
