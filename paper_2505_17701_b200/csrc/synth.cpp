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

// splitmix64 is counter-based (numerics.hpp:33-45): the k-th output of Rng(seed) is
// mix(seed + k * golden), so any stretch of the stream can be generated independently.  The
// Box-Muller pairs of a fresh stream are (draws 2p+1, 2p+2) -> normals (2p, 2p+1) (cos, then
// the cached sin), which lets the layer fill run on all host threads, bit-identical to the
// sequential generator.
uint64_t splitmix_at(uint64_t seed, uint64_t k) {
    uint64_t z = seed + k * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

inline double uniform_of(uint64_t u) { return static_cast<double>(u >> 11) * 0x1.0p-53; }

}  // namespace

extern "C" {

// bench() setup sequence; any output may be NULL (its draws are still consumed so the stream
// position matches the reference).  d_rank <= 0 skips the predictor.
int cd_synth_layer(uint64_t seed, int64_t d_model, int64_t d_inter, int64_t d_rank, float* w_up,
                   float* w_gate, float* w_down, float* x, float* theta_a, float* theta_b) {
    if (d_model <= 0 || d_inter <= 0) return CD_ERR_DATA;
    const float sd = 1.0f / std::sqrt(static_cast<float>(d_model));
    const int64_t n = d_model * d_inter;
    // normals 0 .. 3n-1 fill W_up, W_gate, W_down (sd), then d_model normals of x (sd 1)
    const int64_t total = 3 * n + d_model;
    auto store = [&](int64_t k, double v) {
        if (k < 3 * n) {
            float* m = k < n ? w_up : (k < 2 * n ? w_gate : w_down);
            if (m) m[k % n] = 0.0f + sd * static_cast<float>(v);
        } else if (k < total && x) {
            x[k - 3 * n] = 0.0f + 1.0f * static_cast<float>(v);
        }
    };
    const int64_t pairs = (total + 1) / 2;
#pragma omp parallel for schedule(static)
    for (int64_t p = 0; p < pairs; ++p) {
        const double u1 = 1.0 - uniform_of(splitmix_at(seed, 2 * static_cast<uint64_t>(p) + 1));
        const double u2 = uniform_of(splitmix_at(seed, 2 * static_cast<uint64_t>(p) + 2));
        const double r = std::sqrt(-2.0 * std::log(u1));
        const double a = 6.283185307179586476925286766559 * u2;
        store(2 * p, r * std::cos(a));
        store(2 * p + 1, r * std::sin(a));
    }
    if (d_rank > 0) {
        // Rng::fork(): the next draw after the 2 * pairs Box-Muller draws seeds the child
        const uint64_t child = splitmix_at(seed, 2 * static_cast<uint64_t>(pairs) + 1);
        const float ba = 1.0f / std::sqrt(static_cast<float>(d_model));
        const float bb = 1.0f / std::sqrt(static_cast<float>(d_rank));
        const int64_t na = d_model * d_rank, nbm = d_rank * d_inter;
#pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < na + nbm; ++i) {
            const double u = uniform_of(splitmix_at(child, static_cast<uint64_t>(i) + 1));
            if (i < na) {
                if (theta_a) theta_a[i] = ba * static_cast<float>(2.0 * u - 1.0);
            } else if (theta_b) {
                theta_b[i - na] = bb * static_cast<float>(2.0 * u - 1.0);
            }
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
