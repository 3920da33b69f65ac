// ref_capi.cpp -- extern "C" bindings over the UNMODIFIED reference library.
//
// TEST / BASELINE INFRASTRUCTURE ONLY.  oracle/Makefile compiles this file together
// with the reference sources where they lie (/root/reference/proj/src/*.cpp, never
// copied) into oracle/_ref/libcountdown_ref.so.  It is used
//   * to pin the C oracle (oracle/countdown_oracle.c) bit-for-bit,
//   * to generate the golden fixtures in tests/golden/, and
//   * as the CPU baseline / `bench.py --impl reference` arm (the reference's own
//     OpenMP bench() and pipeline_* functions).
// Exceptions map to the reference CLI's exit-code convention (main.cpp:566-581):
// DataError -> 2, NumericError -> 3, anything else -> 1.
#include <cstring>
#include <string>

#include "countdown/blocked_exec.hpp"
#include "countdown/calibration.hpp"
#include "countdown/costmodel.hpp"
#include "countdown/errors.hpp"
#include "countdown/gated_mlp.hpp"
#include "countdown/model_io.hpp"
#include "countdown/predictor.hpp"
#include "countdown/sparsity.hpp"

#ifdef _OPENMP
#include <omp.h>
#endif

using namespace countdown;

namespace {

thread_local std::string g_err;

template <typename F> int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const DataError& e) {
        g_err = e.what();
        return 2;
    } catch (const NumericError& e) {
        g_err = e.what();
        return 3;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

Mat32 mat(int64_t rows, int64_t cols, const float* p) {
    Mat32 m(rows, cols);
    std::memcpy(m.data.data(), p, sizeof(float) * static_cast<size_t>(rows * cols));
    return m;
}

GatedMlpLayer layer_of(int64_t d, int64_t F, int act, const float* up, const float* gate,
                       const float* down) {
    GatedMlpLayer l;
    l.d_model = d;
    l.d_inter = F;
    l.activation = act == 0 ? Activation::Silu : Activation::GeluTanh;
    l.w_up = mat(F, d, up);
    l.w_gate = mat(F, d, gate);
    l.w_down = mat(F, d, down);
    return l;
}

Predictor predictor_of(int64_t d, int64_t r, int64_t F, const float* ta, const float* tb) {
    LowRankPredictor lp;
    lp.d_model = d;
    lp.d_rank = r;
    lp.d_inter = F;
    lp.theta_a = mat(d, r, ta);
    lp.theta_b = mat(r, F, tb);
    return Predictor{lp};
}

ActivationMask mask_of(int64_t F, const uint8_t* m) {
    ActivationMask am;
    am.alive.assign(m, m + F);
    am.recount();
    return am;
}

Vec32 vec(const float* p, int64_t n) { return Vec32(p, p + n); }

void put(const Vec32& v, float* out) {
    if (out) std::memcpy(out, v.data(), sizeof(float) * v.size());
}

void put_mask(const ActivationMask& m, uint8_t* out) {
    if (out) std::memcpy(out, m.alive.data(), m.alive.size());
}

BlockConfig cfg_of(int64_t blk_m, int64_t blk_n, int reduction) {
    BlockConfig c;
    c.blk_m = blk_m;
    c.blk_n = blk_n;
    c.reduction = reduction == 0 ? Reduction::DeterministicOrdered : Reduction::UnorderedAccumulate;
    return c;
}

void put_traffic(const TrafficCounter& t, int64_t* out) {
    if (!out) return;
    out[0] = t.weight_reads;
    out[1] = t.vector_reads;
    out[2] = t.writes;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_max_threads() {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

// bench() setup order (blocked_exec.cpp:396-415): layer, x, then predictor from rng.fork().
// Any output pointer may be NULL; d_rank <= 0 skips the predictor.
int ref_generate(uint64_t seed, int64_t d, int64_t F, int64_t r, int act, float* up,
                 float* gate, float* down, float* x, float* ta, float* tb) {
    return guarded([&] {
        Rng rng(seed);
        GatedMlpLayer l = make_random_layer(d, F, act == 0 ? Activation::Silu : Activation::GeluTanh, rng);
        Vec32 xv(static_cast<size_t>(d));
        for (auto& v : xv) v = rng.normal_f();
        if (up) std::memcpy(up, l.w_up.data.data(), sizeof(float) * static_cast<size_t>(d * F));
        if (gate) std::memcpy(gate, l.w_gate.data.data(), sizeof(float) * static_cast<size_t>(d * F));
        if (down) std::memcpy(down, l.w_down.data.data(), sizeof(float) * static_cast<size_t>(d * F));
        put(xv, x);
        if (r > 0) {
            Rng prng = rng.fork();
            Predictor p = make_lowrank_predictor(d, r, F, prng);
            const auto& lp = p.lowrank();
            if (ta) std::memcpy(ta, lp.theta_a.data.data(), sizeof(float) * static_cast<size_t>(d * r));
            if (tb) std::memcpy(tb, lp.theta_b.data.data(), sizeof(float) * static_cast<size_t>(r * F));
        }
    });
}

int ref_rng_normals(uint64_t seed, int64_t n, double* out) {
    return guarded([&] {
        Rng rng(seed);
        for (int64_t i = 0; i < n; ++i) out[i] = rng.normal();
    });
}

int ref_activation(int act, const float* x, int64_t n, float* out) {
    return guarded([&] {
        for (int64_t i = 0; i < n; ++i)
            out[i] = apply_activation(act == 0 ? Activation::Silu : Activation::GeluTanh, x[i]);
    });
}

int ref_alive_count_for(double k, int64_t F, int64_t* out) {
    return guarded([&] { *out = alive_count_for(k, F); });
}

int ref_top_m_threshold(const float* v, int64_t n, int64_t m, float* tau, uint8_t* mask) {
    return guarded([&] {
        TopM t = top_m_threshold(vec(v, n), m);
        *tau = t.tau;
        put_mask(t.mask, mask);
    });
}

int ref_forward_dense(int64_t d, int64_t F, int act, const float* up, const float* gate,
                      const float* down, const float* x, float* u, float* h, float* s, float* y) {
    return guarded([&] {
        const GatedMlpLayer l = layer_of(d, F, act, up, gate, down);
        ForwardTrace t = forward_dense(l, vec(x, d));
        put(t.u, u);
        put(t.h, h);
        put(t.s, s);
        put(t.y, y);
    });
}

int ref_forward_sparse(int64_t d, int64_t F, int act, const float* up, const float* gate,
                       const float* down, const float* x, const uint8_t* mask, float* y) {
    return guarded([&] {
        const GatedMlpLayer l = layer_of(d, F, act, up, gate, down);
        put(forward_sparse(l, vec(x, d), mask_of(F, mask)), y);
    });
}

int ref_predict_logits(int64_t d, int64_t r, int64_t F, const float* ta, const float* tb,
                       const float* x, float* z) {
    return guarded([&] { put(predict_logits(predictor_of(d, r, F, ta, tb), vec(x, d)), z); });
}

// method: 0 mc (tau_hat), 1 dc (predictor).  Returns mask + y.
int ref_forward_practical(int method, int64_t d, int64_t F, int64_t r, int act, const float* up,
                          const float* gate, const float* down, const float* ta, const float* tb,
                          const float* x, float tau_hat, float* y, uint8_t* mask, int64_t* alive) {
    return guarded([&] {
        const GatedMlpLayer l = layer_of(d, F, act, up, gate, down);
        SparsityConfig cfg;
        cfg.mode = SparsityMode::Practical;
        PracticalContext ctx;
        Predictor p;
        if (method == 0) {
            cfg.method = SparsityMethod::MCountdown;
            ctx.tau_hat = tau_hat;
        } else {
            cfg.method = SparsityMethod::DCountdown;
            p = predictor_of(d, r, F, ta, tb);
            ctx.predictor = &p;
        }
        PracticalResult res = forward_practical(l, vec(x, d), cfg, ctx);
        put(res.y, y);
        put_mask(res.mask, mask);
        if (alive) *alive = res.mask.alive_count;
    });
}

int ref_exec_dense(int64_t d, int64_t F, int act, const float* up, const float* gate,
                   const float* down, const float* x, int64_t blk_m, int64_t blk_n, int reduction,
                   float* y, int64_t* traffic) {
    return guarded([&] {
        const GatedMlpLayer l = layer_of(d, F, act, up, gate, down);
        TrafficCounter tc;
        put(exec_dense(l, vec(x, d), cfg_of(blk_m, blk_n, reduction), &tc), y);
        put_traffic(tc, traffic);
    });
}

int ref_exec_mc(int64_t d, int64_t F, int act, const float* up, const float* gate,
                const float* down, const float* x, const float* u, const uint8_t* mask,
                int64_t blk_m, int64_t blk_n, int reduction, float* y, int64_t* traffic) {
    return guarded([&] {
        const GatedMlpLayer l = layer_of(d, F, act, up, gate, down);
        TrafficCounter tc;
        put(exec_mc(l, vec(x, d), vec(u, F), mask_of(F, mask), cfg_of(blk_m, blk_n, reduction), &tc), y);
        put_traffic(tc, traffic);
    });
}

int ref_exec_dc(int64_t d, int64_t F, int act, const float* up, const float* gate,
                const float* down, const float* x, const uint8_t* mask, int64_t blk_m,
                int64_t blk_n, int reduction, float* y, int64_t* traffic) {
    return guarded([&] {
        const GatedMlpLayer l = layer_of(d, F, act, up, gate, down);
        TrafficCounter tc;
        put(exec_dc(l, vec(x, d), mask_of(F, mask), cfg_of(blk_m, blk_n, reduction), &tc), y);
        put_traffic(tc, traffic);
    });
}

int ref_pipeline_mc(int64_t d, int64_t F, int act, const float* up, const float* gate,
                    const float* down, const float* x, float tau, int64_t blk_m, int64_t blk_n,
                    int reduction, float* y, uint8_t* mask, int64_t* alive, int64_t* traffic) {
    return guarded([&] {
        const GatedMlpLayer l = layer_of(d, F, act, up, gate, down);
        PipelineResult r = pipeline_mc(l, vec(x, d), tau, cfg_of(blk_m, blk_n, reduction));
        put(r.y, y);
        put_mask(r.mask, mask);
        if (alive) *alive = r.mask.alive_count;
        put_traffic(r.traffic, traffic);
    });
}

int ref_pipeline_dc(int64_t d, int64_t F, int64_t rank, int act, const float* up,
                    const float* gate, const float* down, const float* ta, const float* tb,
                    const float* x, const uint8_t* mask_override, int64_t blk_m, int64_t blk_n,
                    int reduction, float* y, uint8_t* mask, int64_t* alive, int64_t* traffic) {
    return guarded([&] {
        const GatedMlpLayer l = layer_of(d, F, act, up, gate, down);
        const Predictor p = predictor_of(d, rank, F, ta, tb);
        ActivationMask ov;
        if (mask_override) ov = mask_of(F, mask_override);
        PipelineResult r = pipeline_dc(l, vec(x, d), p, cfg_of(blk_m, blk_n, reduction),
                                       mask_override ? &ov : nullptr);
        put(r.y, y);
        put_mask(r.mask, mask);
        if (alive) *alive = r.mask.alive_count;
        put_traffic(r.traffic, traffic);
    });
}

// A persistent reference layer + predictor (built once), so a timed loop measures pipeline_dc
// itself rather than the construction of a 700 MB GatedMlpLayer from raw arrays per call.
struct RefModel {
    GatedMlpLayer layer;
    Predictor pred;
};

int ref_model_new(int64_t d, int64_t F, int64_t rank, int act, const float* up, const float* gate,
                  const float* down, const float* ta, const float* tb, void** out) {
    return guarded([&] {
        *out = new RefModel{layer_of(d, F, act, up, gate, down), predictor_of(d, rank, F, ta, tb)};
    });
}

int ref_model_free(void* h) {
    delete static_cast<RefModel*>(h);
    return 0;
}

int ref_model_pipeline_dc(void* h, const float* x, const uint8_t* mask_override, int64_t blk_m, int64_t blk_n,
                          int reduction, float* y, int64_t* alive) {
    return guarded([&] {
        const RefModel& m = *static_cast<const RefModel*>(h);
        const int64_t d = m.layer.d_model, F = m.layer.d_inter;
        ActivationMask ov;
        if (mask_override) ov = mask_of(F, mask_override);
        PipelineResult r = pipeline_dc(m.layer, vec(x, d), m.pred, cfg_of(blk_m, blk_n, reduction),
                                       mask_override ? &ov : nullptr);
        put(r.y, y);
        if (alive) *alive = r.mask.alive_count;
    });
}

// method: 0 dense, 1 cats, 2 mc, 3 dc.  out: p50_ns, p95_ns, traffic_elements; ratio.
int ref_bench(int method, int64_t d, int64_t F, int64_t r, double k, int64_t iters,
              int64_t blk_m, int64_t blk_n, int reduction, uint64_t seed, int64_t* out3,
              double* ratio) {
    return guarded([&] {
        ShapeSpec s;
        s.d_model = d;
        s.d_inter = F;
        s.d_rank = r;
        const CostMethod m = method == 0   ? CostMethod::Dense
                             : method == 1 ? CostMethod::Cats
                             : method == 2 ? CostMethod::MC
                                           : CostMethod::DC;
        BenchStats st = bench(m, s, k, iters, cfg_of(blk_m, blk_n, reduction), seed);
        out3[0] = st.p50_ns;
        out3[1] = st.p95_ns;
        out3[2] = st.traffic_elements;
        *ratio = st.element_read_ratio;
    });
}

int ref_bench_reference_dense(int64_t d, int64_t F, int64_t iters, uint64_t seed, int64_t* out3) {
    return guarded([&] {
        ShapeSpec s;
        s.d_model = d;
        s.d_inter = F;
        BenchStats st = bench_reference_dense(s, iters, seed);
        out3[0] = st.p50_ns;
        out3[1] = st.p95_ns;
        out3[2] = st.traffic_elements;
    });
}

int ref_calibrate_mc(int64_t d, int64_t F, const float* up, const float* xs, int64_t T, double k,
                     double* tau_hat) {
    return guarded([&] {
        GatedMlpLayer l;
        l.d_model = d;
        l.d_inter = F;
        l.w_up = mat(F, d, up);
        // calibrate() runs forward_dense, which needs all three matrices; only u is used.
        l.w_gate = Mat32(F, d);
        l.w_down = Mat32(F, d);
        std::vector<Vec32> v;
        for (int64_t t = 0; t < T; ++t) v.push_back(vec(xs + t * d, d));
        *tau_hat = calibrate(l, v, k, SparsityMethod::MCountdown).tau_hat;
    });
}

int ref_traffic_split(int method, int64_t d, int64_t F, int64_t r, int64_t s_alive,
                      int64_t* out3) {
    return guarded([&] {
        ShapeSpec s;
        s.d_model = d;
        s.d_inter = F;
        s.d_rank = r;
        s.s_alive = s_alive;
        TrafficSplit t = method == 0   ? traffic_dense_split(s)
                         : method == 1 ? traffic_cats_split(s)
                         : method == 2 ? traffic_mc_split(s)
                                       : traffic_dc_split(s);
        out3[0] = t.weight_reads;
        out3[1] = t.vector_reads;
        out3[2] = t.writes;
    });
}

int ref_flops(int method, int64_t d, int64_t F, int64_t r, int64_t s_alive, int64_t* out) {
    return guarded([&] {
        ShapeSpec s;
        s.d_model = d;
        s.d_inter = F;
        s.d_rank = r;
        s.s_alive = s_alive;
        *out = method == 0 ? flops_dense(s) : method == 1 ? flops_cats(s) : method == 2 ? flops_mc(s) : flops_dc(s);
    });
}

// write_model (model_io.cpp:94-138) of the seeded bench() workload: the layer of Rng(seed),
// x discarded, a low-rank predictor of rank r from rng.fork() (r <= 0: no predictor).
int ref_write_model(const char* path, uint64_t seed, int64_t d, int64_t F, int64_t r, int act, double k) {
    return guarded([&] {
        Rng rng(seed);
        ModelFile mf;
        mf.layer = make_random_layer(d, F, act == 0 ? Activation::Silu : Activation::GeluTanh, rng);
        for (int64_t i = 0; i < d; ++i) (void)rng.normal_f();
        mf.seed = seed;
        if (r > 0) {
            Rng prng = rng.fork();
            mf.predictor = make_lowrank_predictor(d, r, F, prng);
            mf.predictor_k = k;
        }
        write_model(path, mf);
    });
}

// read_model (model_io.cpp:140-224): dims[5] = {d, F, r, act, seed}; any array may be NULL.
int ref_read_model(const char* path, int64_t* dims, float* up, float* gate, float* down, float* ta,
                   float* tb) {
    return guarded([&] {
        ModelFile mf = read_model(path);
        dims[0] = mf.layer.d_model;
        dims[1] = mf.layer.d_inter;
        dims[2] = mf.predictor && mf.predictor->kind() == PredictorKind::LowRank ? mf.predictor->lowrank().d_rank : 0;
        dims[3] = mf.layer.activation == Activation::Silu ? 0 : 1;
        dims[4] = static_cast<int64_t>(mf.seed);
        auto cp = [](const Mat32& m, float* out) {
            if (out) std::memcpy(out, m.data.data(), m.data.size() * sizeof(float));
        };
        cp(mf.layer.w_up, up);
        cp(mf.layer.w_gate, gate);
        cp(mf.layer.w_down, down);
        if (dims[2] > 0) {
            cp(mf.predictor->lowrank().theta_a, ta);
            cp(mf.predictor->lowrank().theta_b, tb);
        }
    });
}

}  // extern "C"
