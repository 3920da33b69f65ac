// blocked_exec_gpu.cpp -- drop-in replacement of the reference's blocked_exec.cpp that runs
// every operator on the B200 through libcountdown_b200.so (include/countdown_b200.h).
//
// Same header (countdown/blocked_exec.hpp), same signatures, same validation messages and
// exception types, same TrafficCounter accounting: link this file INSTEAD of
// proj/src/blocked_exec.cpp and the reference's callers (tests, CLI, acceptance gate) run on
// the GPU.  oracle/Makefile's `gpu-tests` target links the reference's own unit tests this
// way (oracle/_ref/ref_unit_tests_gpu).
//
// Mapping:
//   GatedMlpLayer (host f32)   -> a cached cd_layer handle (f32 on the device, "oracle mode"),
//                                 keyed by the matrices' addresses + shapes + content hash;
//   Predictor (low-rank)       -> cd_layer_set_predictor on that handle (re-attached when the
//                                 theta content changes);
//   BlockConfig::reduction     -> CD_REDUCTION_ORDERED (bitwise, the exact kernels) or
//                                 CD_REDUCTION_UNORDERED (the fused fast path, <= 1e-4 rel-L2);
//   blk_m / blk_n              -> no GPU meaning; results are invariant to them, exactly as the
//                                 reference promises (acceptance.cpp:336-342);
//   TrafficCounter             -> the reference's per-stream element counts at the realized
//                                 alive count (blocked_exec.cpp:63, 127-131, 145-169, 206-210,
//                                 245-249, 283-287, 304-310, 322-324, 336-341, 362-376).
// Status codes map back to the reference's exceptions: 2 -> DataError, 3 -> NumericError,
// anything else -> std::runtime_error.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <list>
#include <mutex>
#include <sstream>
#include <stdexcept>

#include "countdown/blocked_exec.hpp"
#include "countdown_b200.h"
#include "gpu_handles.hpp"

namespace countdown {

using gpu_shim::cache;
using gpu_shim::raise_rc;

namespace {

int red_of(const BlockConfig& cfg) {
    return cfg.reduction == Reduction::DeterministicOrdered ? CD_REDUCTION_ORDERED : CD_REDUCTION_UNORDERED;
}

// check_exec_inputs (blocked_exec.cpp:24-36): identical messages.
void check_inputs(const GatedMlpLayer& layer, const Vec32& x, const ActivationMask* mask, const char* who) {
    if (static_cast<int64_t>(x.size()) != layer.d_model) {
        std::ostringstream oss;
        oss << who << ": x has length " << x.size() << ", layer d_model " << layer.d_model;
        throw DataError(oss.str());
    }
    if (mask && mask->size() != layer.d_inter) {
        std::ostringstream oss;
        oss << who << ": mask has " << mask->size() << " lanes, layer d_inter " << layer.d_inter;
        throw DataError(oss.str());
    }
}

// Normalised 0/1 copy of a mask (the reference treats any non-zero byte as alive).
std::vector<uint8_t> mask_bytes(const ActivationMask& m) {
    std::vector<uint8_t> out(m.alive.size());
    for (size_t i = 0; i < out.size(); ++i) out[i] = m.alive[i] != 0;
    return out;
}

int64_t count_alive(const ActivationMask& m) {
    int64_t n = 0;
    for (uint8_t a : m.alive) n += a != 0;
    return n;
}

// Stream accounting of the phase-1 kernels + down_projection (blocked_exec.cpp:127-131).
void count_down(TrafficCounter* tc, int64_t d, int64_t F, int64_t alive) {
    if (!tc) return;
    tc->weight_reads += d * alive;
    tc->vector_reads += F;
    tc->writes += d;
}

}  // namespace

Vec32 exec_dense(const GatedMlpLayer& layer, const Vec32& x, const BlockConfig& cfg, TrafficCounter* tc) {
    layer.validate();
    check_inputs(layer, x, nullptr, "exec_dense");
    cd_layer* h = cache().get(layer, nullptr);
    Vec32 y(static_cast<size_t>(layer.d_model));
    raise_rc(cd_exec_dense(h, 1, x.data(), red_of(cfg), y.data()));
    if (tc) {  // blocked_exec.cpp:145-169
        const int64_t d = layer.d_model, F = layer.d_inter;
        tc->weight_reads += 2 * d * F;
        tc->vector_reads += d + d + F + 2 * F;
        tc->writes += F + F + F + F;
        count_down(tc, d, F, F);
    }
    return y;
}

Vec32 exec_mc(const GatedMlpLayer& layer, const Vec32& x, const Vec32& u, const ActivationMask& mask,
              const BlockConfig& cfg, TrafficCounter* tc) {
    layer.validate();
    check_inputs(layer, x, &mask, "exec_mc");
    if (static_cast<int64_t>(u.size()) != layer.d_inter) throw DataError("exec_mc: u length does not match d_inter");
    cd_layer* h = cache().get(layer, nullptr);
    const std::vector<uint8_t> m = mask_bytes(mask);
    Vec32 y(static_cast<size_t>(layer.d_model));
    raise_rc(cd_exec_mc(h, 1, x.data(), u.data(), m.data(), red_of(cfg), y.data()));
    if (tc) {  // blocked_exec.cpp:206-210
        const int64_t d = layer.d_model, F = layer.d_inter, a = count_alive(mask);
        tc->weight_reads += d * a;
        tc->vector_reads += d + F + a;
        tc->writes += F;
        count_down(tc, d, F, a);
    }
    return y;
}

Vec32 exec_cats(const GatedMlpLayer& layer, const Vec32& x, const Vec32& act_gate, const ActivationMask& mask,
                const BlockConfig& cfg, TrafficCounter* tc) {
    layer.validate();
    check_inputs(layer, x, &mask, "exec_cats");
    if (static_cast<int64_t>(act_gate.size()) != layer.d_inter)
        throw DataError("exec_cats: act_gate length does not match d_inter");
    cd_layer* h = cache().get(layer, nullptr);
    const std::vector<uint8_t> m = mask_bytes(mask);
    Vec32 y(static_cast<size_t>(layer.d_model));
    raise_rc(cd_exec_cats(h, 1, x.data(), act_gate.data(), m.data(), red_of(cfg), y.data()));
    if (tc) {  // blocked_exec.cpp:245-249
        const int64_t d = layer.d_model, F = layer.d_inter, a = count_alive(mask);
        tc->weight_reads += d * a;
        tc->vector_reads += d + F + a;
        tc->writes += F;
        count_down(tc, d, F, a);
    }
    return y;
}

Vec32 exec_dc(const GatedMlpLayer& layer, const Vec32& x, const ActivationMask& mask, const BlockConfig& cfg,
              TrafficCounter* tc) {
    layer.validate();
    check_inputs(layer, x, &mask, "exec_dc");
    cd_layer* h = cache().get(layer, nullptr);
    const std::vector<uint8_t> m = mask_bytes(mask);
    Vec32 y(static_cast<size_t>(layer.d_model));
    raise_rc(cd_exec_dc(h, 1, x.data(), m.data(), red_of(cfg), y.data()));
    if (tc) {  // blocked_exec.cpp:283-287
        const int64_t d = layer.d_model, F = layer.d_inter, a = count_alive(mask);
        tc->weight_reads += 2 * d * a;
        tc->vector_reads += d + F;
        tc->writes += F;
        count_down(tc, d, F, a);
    }
    return y;
}

PipelineResult pipeline_dense(const GatedMlpLayer& layer, const Vec32& x, const BlockConfig& cfg) {
    PipelineResult r;
    r.mask = ActivationMask::all_alive(layer.d_inter);
    r.y = exec_dense(layer, x, cfg, &r.traffic);
    return r;
}

namespace {

ActivationMask mask_from(const std::vector<uint8_t>& m, int64_t alive, float tau) {
    ActivationMask a;
    a.alive = m;
    a.alive_count = alive;
    a.tau = tau;
    return a;
}

// threshold_mask's stream accounting (blocked_exec.cpp:304-310).
void count_threshold(TrafficCounter& tc, int64_t F) {
    tc.vector_reads += 2 * F;
    tc.writes += 2 * F;
}

}  // namespace

PipelineResult pipeline_mc(const GatedMlpLayer& layer, const Vec32& x, float tau, const BlockConfig& cfg) {
    layer.validate();
    check_inputs(layer, x, nullptr, "pipeline_mc");
    cd_layer* h = cache().get(layer, nullptr);
    const int64_t d = layer.d_model, F = layer.d_inter;
    PipelineResult r;
    r.y.resize(static_cast<size_t>(d));
    std::vector<uint8_t> m(static_cast<size_t>(F));
    int64_t alive = 0;
    raise_rc(cd_pipeline_mc(h, 1, x.data(), tau, red_of(cfg), r.y.data(), m.data(), &alive, nullptr));
    r.mask = mask_from(m, alive, tau);
    r.traffic.weight_reads += d * F;  // dense up pass (blocked_exec.cpp:322-324)
    r.traffic.vector_reads += d;
    r.traffic.writes += F;
    count_threshold(r.traffic, F);
    r.traffic.weight_reads += d * alive;  // exec_mc
    r.traffic.vector_reads += d + F + alive;
    r.traffic.writes += F;
    count_down(&r.traffic, d, F, alive);
    return r;
}

PipelineResult pipeline_cats(const GatedMlpLayer& layer, const Vec32& x, float tau, const BlockConfig& cfg) {
    layer.validate();
    check_inputs(layer, x, nullptr, "pipeline_cats");
    cd_layer* h = cache().get(layer, nullptr);
    const int64_t d = layer.d_model, F = layer.d_inter;
    PipelineResult r;
    r.y.resize(static_cast<size_t>(d));
    std::vector<uint8_t> m(static_cast<size_t>(F));
    int64_t alive = 0;
    raise_rc(cd_pipeline_cats(h, 1, x.data(), tau, red_of(cfg), r.y.data(), m.data(), &alive, nullptr));
    r.mask = mask_from(m, alive, tau);
    r.traffic.weight_reads += d * F;  // dense gate pass (blocked_exec.cpp:336-337)
    r.traffic.vector_reads += d + F;  // + act pass (:338-342)
    r.traffic.writes += F + F;
    count_threshold(r.traffic, F);
    r.traffic.weight_reads += d * alive;  // exec_cats
    r.traffic.vector_reads += d + F + alive;
    r.traffic.writes += F;
    count_down(&r.traffic, d, F, alive);
    return r;
}

PipelineResult pipeline_dc(const GatedMlpLayer& layer, const Vec32& x, const Predictor& p, const BlockConfig& cfg,
                           const ActivationMask* mask_override) {
    layer.validate();
    check_inputs(layer, x, mask_override, "pipeline_dc");
    if (p.kind() != PredictorKind::LowRank)
        throw DataError("pipeline_dc: the blocked pipeline models the low-rank predictor");
    const LowRankPredictor& lp = p.lowrank();
    if (lp.d_model != layer.d_model || lp.d_inter != layer.d_inter)
        throw DataError("pipeline_dc: predictor shape does not match the layer");
    cd_layer* h = cache().get(layer, &p);
    const int64_t d = layer.d_model, F = layer.d_inter, rk = lp.d_rank;
    PipelineResult r;
    r.y.resize(static_cast<size_t>(d));
    std::vector<uint8_t> m(static_cast<size_t>(F));
    std::vector<uint8_t> ovr;
    if (mask_override) ovr = mask_bytes(*mask_override);
    int64_t alive = 0;
    raise_rc(cd_pipeline_dc(h, 1, x.data(), 0.0f, mask_override ? ovr.data() : nullptr, red_of(cfg), r.y.data(),
                            m.data(), &alive, nullptr));
    if (mask_override) {
        r.mask = *mask_override;  // the override itself, tau and count as given (blocked_exec.cpp:366-367)
    } else {
        r.mask = mask_from(m, alive, 0.0f);
    }
    r.traffic.weight_reads += d * rk + rk * F;  // predictor (blocked_exec.cpp:362-364)
    r.traffic.vector_reads += d + rk;
    r.traffic.writes += rk + F;
    r.traffic.vector_reads += F;  // read logits, write mask (:375-376)
    r.traffic.writes += F;
    r.traffic.weight_reads += 2 * d * alive;  // exec_dc
    r.traffic.vector_reads += d + F;
    r.traffic.writes += F;
    count_down(&r.traffic, d, F, alive);
    return r;
}

namespace {

int64_t percentile(const std::vector<int64_t>& sorted, double q) {
    const size_t n = sorted.size();
    return sorted[static_cast<size_t>(std::llround(q * static_cast<double>(n - 1)))];
}

}  // namespace

// bench (blocked_exec.hpp:85-86): the same seeded workload, per-input ideal thresholds and
// warmup as blocked_exec.cpp:391-455; each timed iteration is one synchronous GPU pipeline
// call (host copies included), timed with steady_clock like the reference.
BenchStats bench(CostMethod method, const ShapeSpec& shape, double k, int64_t iters, const BlockConfig& cfg,
                 uint64_t seed) {
    if (iters <= 0) throw DataError("bench: iters must be positive");
    using clock = std::chrono::steady_clock;
    Rng rng(seed);
    GatedMlpLayer layer = make_random_layer(shape.d_model, shape.d_inter, Activation::Silu, rng);
    Vec32 x(static_cast<size_t>(shape.d_model));
    for (auto& v : x) v = rng.normal_f();
    const ForwardTrace trace = forward_dense(layer, x);  // setup only (gated_mlp.cpp:46-59)
    float tau_u = 0.0f, tau_h = 0.0f;
    ActivationMask ideal_s;
    Predictor predictor;
    if (method != CostMethod::Dense) {
        const int64_t m = alive_count_for(k, shape.d_inter);
        tau_u = top_m_threshold(trace.u, m).tau;
        tau_h = top_m_threshold(trace.h, m).tau;
        ideal_s = top_m_threshold(trace.s, m).mask;
        if (method == CostMethod::DC) {
            Rng prng = rng.fork();
            predictor = make_lowrank_predictor(shape.d_model, shape.d_rank, shape.d_inter, prng);
        }
    }
    auto run_once = [&]() -> PipelineResult {
        switch (method) {
            case CostMethod::Dense: return pipeline_dense(layer, x, cfg);
            case CostMethod::Cats: return pipeline_cats(layer, x, tau_h, cfg);
            case CostMethod::MC: return pipeline_mc(layer, x, tau_u, cfg);
            default: return pipeline_dc(layer, x, predictor, cfg, &ideal_s);
        }
    };
    const int64_t warmup = std::max<int64_t>(10, iters / 10);
    for (int64_t i = 0; i < warmup; ++i) (void)run_once();
    std::vector<int64_t> ns(static_cast<size_t>(iters));
    TrafficCounter last;
    for (int64_t i = 0; i < iters; ++i) {
        const auto t0 = clock::now();
        PipelineResult r = run_once();
        const auto t1 = clock::now();
        ns[static_cast<size_t>(i)] = std::chrono::duration_cast<std::chrono::nanoseconds>(t1 - t0).count();
        last = r.traffic;
    }
    std::sort(ns.begin(), ns.end());
    const int64_t dense_total = traffic_dense(shape);
    BenchStats st;
    st.method = cost_method_name(method);
    st.k = method == CostMethod::Dense ? 0.0 : k;
    st.d_model = shape.d_model;
    st.d_inter = shape.d_inter;
    st.iters = iters;
    st.p50_ns = percentile(ns, 0.50);
    st.p95_ns = percentile(ns, 0.95);
    st.traffic_elements = last.total();
    st.element_read_ratio = static_cast<double>(last.total()) / static_cast<double>(dense_total);
    return st;
}

// bench_reference_dense (blocked_exec.hpp:88-89) is, by definition, the SERIAL CPU timing of
// forward_dense (gated_mlp.cpp:46-59) -- a host comparator, not an operator; it keeps its
// meaning (and its timings) under the drop-in.
BenchStats bench_reference_dense(const ShapeSpec& shape, int64_t iters, uint64_t seed) {
    if (iters <= 0) throw DataError("bench: iters must be positive");
    using clock = std::chrono::steady_clock;
    Rng rng(seed);
    GatedMlpLayer layer = make_random_layer(shape.d_model, shape.d_inter, Activation::Silu, rng);
    Vec32 x(static_cast<size_t>(shape.d_model));
    for (auto& v : x) v = rng.normal_f();
    const int64_t warmup = std::max<int64_t>(10, iters / 10);
    for (int64_t i = 0; i < warmup; ++i) (void)forward_dense(layer, x);
    std::vector<int64_t> ns(static_cast<size_t>(iters));
    for (int64_t i = 0; i < iters; ++i) {
        const auto t0 = clock::now();
        (void)forward_dense(layer, x);
        const auto t1 = clock::now();
        ns[static_cast<size_t>(i)] = std::chrono::duration_cast<std::chrono::nanoseconds>(t1 - t0).count();
    }
    std::sort(ns.begin(), ns.end());
    BenchStats st;
    st.method = "dense-ref";
    st.d_model = shape.d_model;
    st.d_inter = shape.d_inter;
    st.iters = iters;
    st.p50_ns = percentile(ns, 0.50);
    st.p95_ns = percentile(ns, 0.95);
    st.traffic_elements = traffic_dense(shape);
    st.element_read_ratio = 1.0;
    return st;
}

}  // namespace countdown
