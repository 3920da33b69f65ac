// practical_fast.cpp -- a C++ caller of the reference API (sparsity.hpp / predictor.hpp) linked
// against the B200 drop-in shims: forward_practical in both reduction modes.
//   * Ordered (the default): bit-identical to forward_sparse on predict_mask's mask.
//   * UnorderedAccumulate (countdown::gpu::set_reduction): the fused decode kernel runs
//     (engine "fast", one launch for the step), y within 1e-4 relative L2 of the Ordered y.
// Prints one JSON line; tests/test_gpu_parity.py runs it on the B200.  Test infrastructure.
#include <cmath>
#include <cstdio>
#include <cstring>

#include "countdown/gated_mlp.hpp"
#include "countdown/predictor.hpp"
#include "countdown/sparsity.hpp"
#include "countdown_b200.h"
#include "countdown_gpu.hpp"
#include "gpu_handles.hpp"

using namespace countdown;

int main() {
    const int64_t d = 1024, F = 4096, r = 128;
    Rng rng(2024);
    const GatedMlpLayer layer = make_random_layer(d, F, Activation::Silu, rng);
    Vec32 x(static_cast<size_t>(d));
    for (auto& v : x) v = rng.normal_f();
    Rng prng = rng.fork();
    const Predictor pred = make_lowrank_predictor(d, r, F, prng);
    SparsityConfig cfg{SparsityMethod::DCountdown, SparsityMode::Practical, 0.5};
    PracticalContext ctx;
    ctx.predictor = &pred;

    const PracticalResult ord = forward_practical(layer, x, cfg, ctx);
    int path_ord = -1;
    cd_layer_last_path(gpu_shim::cache().get(layer, &pred), &path_ord);
    const Vec32 ys = forward_sparse(layer, x, ord.mask);
    const bool bitwise = std::memcmp(ys.data(), ord.y.data(), ys.size() * 4) == 0;

    gpu::set_reduction(Reduction::UnorderedAccumulate);
    const PracticalResult fast = forward_practical(layer, x, cfg, ctx);
    int path_fast = -1, launches = -1;
    cd_layer* h = gpu_shim::cache().get(layer, &pred);
    cd_layer_last_path(h, &path_fast);
    cd_layer_last_launches(h, &launches);
    double num = 0, den = 0;
    int64_t flips = 0;
    for (size_t j = 0; j < ord.y.size(); ++j) {
        num += (double(fast.y[j]) - ord.y[j]) * (double(fast.y[j]) - ord.y[j]);
        den += double(ord.y[j]) * ord.y[j];
    }
    for (size_t i = 0; i < ord.mask.alive.size(); ++i) flips += ord.mask.alive[i] != fast.mask.alive[i];
    std::printf("{\"path_ordered\": %d, \"bitwise_forward_sparse\": %s, \"path_fast\": %d, \"host_call_launches\": %d, "
                "\"rel_l2\": %.3e, \"flips\": %lld, \"alive\": %lld}\n",
                path_ord, bitwise ? "true" : "false", path_fast, launches, std::sqrt(num / den),
                static_cast<long long>(flips), static_cast<long long>(ord.mask.alive_count));
    return 0;
}
