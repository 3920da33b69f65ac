// gpu_handles.hpp -- device handles behind the reference's value types, shared by the C++
// drop-in shims (blocked_exec_gpu.cpp, sparsity_predictor_gpu.cpp).
//
// The reference passes GatedMlpLayer / Predictor by const& with host std::vectors inside
// (gated_mlp.hpp:12-23, predictor.hpp:15-44); the B200 library works on uploaded handles.
// The cache maps a host object to its handle by the matrices' addresses + shapes + a hash of
// EVERY element, so an in-place edit is always seen (the reference API has no invalidate).
// Handles are f32 on the device ("oracle mode"), so DeterministicOrdered calls are bitwise the
// reference.  One cache per process (inline function statics are shared across the TUs).
#pragma once

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstring>
#include <list>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "countdown/errors.hpp"
#include "countdown/gated_mlp.hpp"
#include "countdown/predictor.hpp"
#include "countdown_b200.h"

namespace countdown {
namespace gpu_shim {

// Process-wide shim settings (countdown_gpu.hpp is the public face).
struct Settings {
    std::atomic<int> reduction{CD_REDUCTION_ORDERED};  // forward_sparse / forward_practical
    std::atomic<bool> content_check{true};              // hash every element on every lookup
};

inline Settings& settings() {
    static Settings s;
    return s;
}

// Status code -> the reference's exception taxonomy (errors.hpp).
inline void raise_rc(int rc) {
    if (rc == CD_OK) return;
    const std::string msg = cd_last_error();
    if (rc == CD_ERR_DATA) throw DataError(msg);
    if (rc == CD_ERR_NUMERIC) throw NumericError(msg);
    throw std::runtime_error("countdown_b200: " + msg);
}

// Four independent multiply-xorshift lanes over 64-bit words per 1 MiB chunk, chunks hashed in
// parallel (OpenMP, as the reference's own build) and combined in order: ~30 GB/s on 16
// cores, ~25 ms for the 700 MB Llama-shape layer.
inline uint64_t mix64(uint64_t h) {
    h ^= h >> 33;
    h *= 0xff51afd7ed558ccdull;
    h ^= h >> 33;
    h *= 0xc4ceb9fe1a85ec53ull;
    h ^= h >> 33;
    return h;
}

inline uint64_t chunk_hash(const uint64_t* w, size_t n, uint64_t seed) {
    uint64_t a = seed ^ 0x9E3779B97F4A7C15ull, b = seed + 0x632BE59BD9B4E019ull, c = ~seed, d = seed * 3;
    size_t i = 0;
    for (; i + 4 <= n; i += 4) {
        a = (a ^ w[i]) * 0x9FB21C651E98DF25ull;
        b = (b ^ w[i + 1]) * 0x9FB21C651E98DF25ull;
        c = (c ^ w[i + 2]) * 0x9FB21C651E98DF25ull;
        d = (d ^ w[i + 3]) * 0x9FB21C651E98DF25ull;
        a ^= a >> 29;
        b ^= b >> 29;
        c ^= c >> 29;
        d ^= d >> 29;
    }
    for (; i < n; ++i) a = mix64(a ^ w[i]);
    return mix64(a ^ mix64(b ^ mix64(c ^ mix64(d))));
}

inline uint64_t content_hash(const std::vector<float>& v, uint64_t h = 0xcbf29ce484222325ull) {
    const size_t n = v.size();
    const size_t words = n / 2;
    const uint64_t* w = reinterpret_cast<const uint64_t*>(v.data());  // std::vector storage: 8-aligned
    constexpr size_t kChunk = size_t(1) << 17;                        // words (1 MiB)
    const int64_t nchunks = static_cast<int64_t>((words + kChunk - 1) / kChunk);
    std::vector<uint64_t> part(static_cast<size_t>(nchunks));
#pragma omp parallel for schedule(static) if (nchunks > 8)
    for (int64_t c = 0; c < nchunks; ++c) {
        const size_t b = static_cast<size_t>(c) * kChunk;
        part[static_cast<size_t>(c)] = chunk_hash(w + b, std::min(kChunk, words - b), static_cast<uint64_t>(c));
    }
    for (uint64_t p : part) h = mix64(h ^ p);
    if (n & 1) {
        uint32_t u;
        std::memcpy(&u, &v[n - 1], 4);
        h = mix64(h ^ u);
    }
    return mix64(h ^ n);
}

class HandleCache {
  public:
    ~HandleCache() {
        for (auto& e : layers_) cd_layer_destroy(e.h);
        for (auto& e : preds_) cd_layer_destroy(e.h);
    }

    // The layer's handle, with the low-rank predictor `p` attached when given.
    cd_layer* get(const GatedMlpLayer& L, const Predictor* p) {
        std::lock_guard<std::mutex> g(mu_);
        const bool check = settings().content_check.load();
        const uint64_t hash =
            check ? content_hash(L.w_down.data, content_hash(L.w_gate.data, content_hash(L.w_up.data))) : 0;
        auto it = std::find_if(layers_.begin(), layers_.end(), [&](const LayerEntry& e) {
            return e.up == L.w_up.data.data() && e.gate == L.w_gate.data.data() && e.down == L.w_down.data.data() &&
                   e.d == L.d_model && e.F == L.d_inter && e.act == L.activation && e.hash == hash;
        });
        if (it == layers_.end()) {
            cd_layer* h = nullptr;
            raise_rc(cd_layer_create(0, L.d_model, L.d_inter,
                                     L.activation == Activation::Silu ? CD_ACT_SILU : CD_ACT_GELU_TANH, CD_DTYPE_F32,
                                     L.w_up.data.data(), L.w_gate.data.data(), L.w_down.data.data(), &h));
            layers_.push_front(LayerEntry{L.w_up.data.data(), L.w_gate.data.data(), L.w_down.data.data(), L.d_model,
                                          L.d_inter, L.activation, hash, h, nullptr, nullptr, 0, 0});
            if (layers_.size() > kCap) {
                cd_layer_destroy(layers_.back().h);
                layers_.pop_back();
            }
            it = layers_.begin();
        } else if (it != layers_.begin()) {
            layers_.splice(layers_.begin(), layers_, it);
            it = layers_.begin();
        }
        if (p) {
            const LowRankPredictor& lp = p->lowrank();
            const uint64_t ph = check ? content_hash(lp.theta_b.data, content_hash(lp.theta_a.data)) : 0;
            if (it->ta != lp.theta_a.data.data() || it->tb != lp.theta_b.data.data() || it->r != lp.d_rank ||
                it->phash != ph) {
                raise_rc(cd_layer_set_predictor(it->h, lp.d_rank, lp.theta_a.data.data(), lp.theta_b.data.data()));
                it->ta = lp.theta_a.data.data();
                it->tb = lp.theta_b.data.data();
                it->r = lp.d_rank;
                it->phash = ph;
            }
        }
        return it->h;
    }

    // A predictor-only handle (cd_predictor_create / cd_predictor_create_ternary) for
    // predict_logits on a bare Predictor.
    cd_layer* predictor(const Predictor& p) {
        std::lock_guard<std::mutex> g(mu_);
        const bool lowrank = p.kind() == PredictorKind::LowRank;
        const std::vector<float>& a = lowrank ? p.lowrank().theta_a.data : p.ternary().shadow.data;
        const std::vector<float>* b = lowrank ? &p.lowrank().theta_b.data : nullptr;
        const bool check = settings().content_check.load();
        const uint64_t hash = !check ? 0 : (b ? content_hash(*b, content_hash(a)) : content_hash(a, 0x7e57));
        const int64_t r = lowrank ? p.lowrank().d_rank : -1;
        auto it = std::find_if(preds_.begin(), preds_.end(), [&](const PredEntry& e) {
            return e.a == a.data() && e.d == p.d_model() && e.F == p.d_inter() && e.r == r && e.hash == hash;
        });
        if (it != preds_.end()) return it->h;
        cd_layer* h = nullptr;
        if (lowrank) {
            const LowRankPredictor& lp = p.lowrank();
            raise_rc(cd_predictor_create(0, lp.d_model, lp.d_rank, lp.d_inter, CD_DTYPE_F32, lp.theta_a.data.data(),
                                         lp.theta_b.data.data(), &h));
        } else {
            // the reference's own quantizer (predictor.cpp:10-27) is the weight preprocessing
            const TernaryPredictor& t = p.ternary();
            const std::vector<int8_t> q = t.quantized();
            raise_rc(cd_predictor_create_ternary(0, t.d_model, t.d_inter, t.gamma(), q.data(), &h));
        }
        preds_.push_front(PredEntry{a.data(), p.d_model(), p.d_inter(), r, hash, h});
        if (preds_.size() > kCap) {
            cd_layer_destroy(preds_.back().h);
            preds_.pop_back();
        }
        return h;
    }

    void clear() {
        std::lock_guard<std::mutex> g(mu_);
        for (auto& e : layers_) cd_layer_destroy(e.h);
        for (auto& e : preds_) cd_layer_destroy(e.h);
        layers_.clear();
        preds_.clear();
    }

  private:
    struct LayerEntry {
        const float *up, *gate, *down;
        int64_t d, F;
        Activation act;
        uint64_t hash;
        cd_layer* h;
        const float *ta, *tb;
        int64_t r;
        uint64_t phash;
    };
    struct PredEntry {
        const float* a;
        int64_t d, F, r;
        uint64_t hash;
        cd_layer* h;
    };
    static constexpr size_t kCap = 8;
    std::mutex mu_;
    std::list<LayerEntry> layers_;
    std::list<PredEntry> preds_;
};

inline HandleCache& cache() {
    static HandleCache c;
    return c;
}

}  // namespace gpu_shim
}  // namespace countdown
