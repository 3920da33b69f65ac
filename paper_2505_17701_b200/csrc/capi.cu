// capi.cu -- implementation of the C-ABI declared in include/countdown_b200.h.
//
// Owns the per-layer device state (re-laid-out weights, self-cleaning scratch, a stream,
// pinned staging for the host-buffer entry points) and sequences the kernel chains of
// kernels_fast.cu (UnorderedAccumulate) and kernels_exact.cu (DeterministicOrdered).
// No CPU compute path exists: every operator runs on the device or fails.
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: ranges cost nothing without a profiler

#include <algorithm>
#include <atomic>
#include <cerrno>
#include <cmath>
#include <fstream>
#include <map>
#include <sstream>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/countdown_b200.h"
#include "kernels.h"
#include "kernels_tc.h"

namespace {

thread_local std::string g_err;

struct Fail {
    int code;
};

[[noreturn]] void fail(int code, const std::string& msg) {
    g_err = msg;
    throw Fail{code};
}

void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) fail(CD_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

template <typename F> int guarded(F&& f) {
    try {
        f();
        return CD_OK;
    } catch (const Fail& e) {
        return e.code;
    } catch (const std::exception& e) {
        g_err = e.what();
        return CD_ERR_USAGE;
    }
}

int64_t round_up(int64_t v, int64_t m) { return (v + m - 1) / m * m; }

// A device (or pinned host) buffer that only grows; freed with its owner.
struct Grow {
    bool host = false;
    void* p = nullptr;
    size_t cap = 0;
    uint64_t* gen = nullptr;  // owner's generation: bumped when the buffer moves
    Grow() = default;
    explicit Grow(bool on_host) : host(on_host) {}
    Grow(const Grow&) = delete;
    Grow& operator=(const Grow&) = delete;
    template <typename T> T* get(size_t n) {
        const size_t bytes = std::max<size_t>(n, 1) * sizeof(T);
        if (bytes > cap) {
            release();
            const size_t want = std::max(bytes, cap * 2);
            ck(host ? cudaMallocHost(&p, want) : cudaMalloc(&p, want), host ? "cudaMallocHost" : "cudaMalloc");
            cap = want;
            if (gen) ++*gen;
        }
        return static_cast<T*>(p);
    }
    void release() {
        if (p) host ? cudaFreeHost(p) : cudaFree(p);
        p = nullptr;
        cap = 0;
    }
    ~Grow() { release(); }
};

}  // namespace

struct cd_layer {
    int device = 0;
    int num_sms = 148;
    cdk::LayerDev L;
    cdk::Scratch S;
    int64_t F_total = 0, row_begin = 0;
    cudaStream_t stream = nullptr;
    std::recursive_mutex* dev_mu = nullptr;  // the device's lock (see device_stream)
    std::mutex mu;
    // Device-state generation: bumped whenever a pointer a captured host graph could hold
    // changes (predictor re-attached, a workspace regrown).  Part of the host-graph key.
    uint64_t gen = 1;
    std::vector<std::pair<void*, size_t>> dev_allocs;
    std::vector<void*> host_allocs;
    int64_t bytes = 0;
    int last_launches = 0;
    int last_path = CD_PATH_FAST;
    // engines (cd_layer_set_engines): all on by default
    bool use_fused = true;  // batch <= 4 DC / MC as one persistent kernel (off: the kernel chains)
    bool pdl_chain = false; // CD_ENGINE_PDL_CHAIN: persistent kernels PDL-chained, not cooperative
    bool use_tc = true;     // batches >= kTcMinBatch of a bf16 layer on the tensor cores
    bool weights_finite = true;  // every uploaded weight finite: the row-union GEMM may read any row
    const void* pf_at = nullptr;  // cd_layer_set_prefetch: the next layer's predictor (L2 prefetch)
    const void* pf_bt = nullptr;
    Grow tc_ws;             // tensor-core path workspace
    Grow rms_ws;            // RMS-normalised inputs for the engines that do not fuse the norm
    // host-call CUDA graph: [H2D inputs, kernels, D2H outputs] replayed while the call signature
    // (method, batch, tau, options) repeats -- one launch instead of four API calls per step
    struct HostGraph {
        uint64_t key = 0;
        int seen = 0;  // consecutive calls with this key (capture on the second)
        cudaGraphExec_t exec = nullptr;
        int launches = 0, path = 0;
    } hg;
    bool use_host_graph = true;  // host-buffer calls replay a captured graph
    bool mapped_staging = true;  // fixed pinned staging is device-addressable (copy kernels)
    // large-batch staging (host-buffer calls on the tensor-core path)
    Grow g_dx, g_dy, g_dmask_in, g_dmask_out, g_du_in, g_dind, g_dalive;
    Grow g_hx{true}, g_hy{true}, g_hmask{true}, g_hind{true}, g_halive{true};
    // device staging for the host-buffer entry points
    float* d_x = nullptr;
    float* d_y = nullptr;
    uint8_t* d_mask_in = nullptr;
    uint8_t* d_mask_out = nullptr;
    float* d_u_in = nullptr;
    float* d_ind = nullptr;
    int* d_alive = nullptr;
    // pinned host staging
    float* h_x = nullptr;
    float* h_y = nullptr;
    uint8_t* h_mask = nullptr;
    float* h_ind = nullptr;
    int* h_alive = nullptr;
    // completion word of the host-buffer calls (mapped pinned): the last kernel increments it,
    // the host polls it instead of synchronising the stream (lower wake-up latency)
    unsigned long long* h_done = nullptr;
    unsigned long long done_seen = 0;

    template <typename T> T* dalloc(size_t n, bool zero = true) {
        void* p = nullptr;
        ck(cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T)), "cudaMalloc");
        dev_allocs.emplace_back(p, n * sizeof(T));
        bytes += static_cast<int64_t>(n * sizeof(T));
        if (zero) ck(cudaMemset(p, 0, std::max<size_t>(n, 1) * sizeof(T)), "cudaMemset");
        return static_cast<T*>(p);
    }
    // Free one dalloc'd buffer (a replaced predictor) once the stream no longer uses it.
    void dfree(const void* p) {
        for (auto it = dev_allocs.begin(); it != dev_allocs.end(); ++it)
            if (it->first == p) {
                bytes -= static_cast<int64_t>(it->second);
                cudaFree(it->first);
                dev_allocs.erase(it);
                return;
            }
    }
    template <typename T> T* halloc(size_t n) {
        void* p = nullptr;
        // mapped: the copy kernels of the host-buffer calls read / write it directly (UVA: the
        // device address is the host address; otherwise those calls use the DMA engine)
        ck(cudaHostAlloc(&p, std::max<size_t>(n, 1) * sizeof(T), cudaHostAllocMapped), "cudaHostAlloc");
        void* dp = nullptr;
        if (cudaHostGetDevicePointer(&dp, p, 0) != cudaSuccess || dp != p) {
            (void)cudaGetLastError();
            mapped_staging = false;
        }
        host_allocs.push_back(p);
        return static_cast<T*>(p);
    }
    ~cd_layer() {
        if (stream) {  // the device's shared stream: drained, not destroyed
            cudaSetDevice(device);
            cudaStreamSynchronize(stream);
        }
        if (hg.exec) cudaGraphExecDestroy(hg.exec);
        for (auto& a : dev_allocs) cudaFree(a.first);
        for (void* p : host_allocs) cudaFreeHost(p);
    }
};

namespace {

using cdk::kMaxBatch;
using cdk::kMaxBatchFast;

// One internal stream and one lock per device, shared by every handle on it.
//  - The persistent kernels (k_dc_fused, k_mc_fused, k_tc_fused) need all of their CTAs
//    resident at once; two of them running concurrently on different streams could each hold
//    part of the GPU and wait forever for the rest.  Sharing the stream serialises them.
//  - The lock is held across every call that enqueues on that stream (host-buffer operators,
//    uploads, predictor attach, destroy).  A host call captures its sequence into a CUDA graph
//    on the shared stream; without the lock, another thread's work enqueued meanwhile would
//    become part of that graph.
struct DeviceCtx {
    cudaStream_t stream = nullptr;
    std::recursive_mutex mu;
};

// Never destroyed: handles freed during static destruction (a C++ caller's cache, destroyed
// after this library's statics) must still find their device's lock.
DeviceCtx& device_ctx(int device) {
    static std::mutex* mu = new std::mutex;
    static auto* ctxs = new std::map<int, DeviceCtx*>;
    std::lock_guard<std::mutex> g(*mu);
    auto it = ctxs->find(device);
    if (it != ctxs->end()) return *it->second;
    auto* c = new DeviceCtx;
    if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess) {
        delete c;
        ck(cudaGetLastError(), "cudaStreamCreate");
        fail(CD_ERR_CUDA, "cudaStreamCreate failed");
    }
    ctxs->emplace(device, c);
    return *c;
}

// Device lock, then handle lock (always in this order).
struct CallLock {
    std::unique_lock<std::recursive_mutex> d;
    std::unique_lock<std::mutex> h;
    explicit CallLock(cd_layer* l) : d(*l->dev_mu), h(l->mu) {}
};


// Upload rows [row_begin, row_end) of a full host matrix (rows x cols f32) into a padded
// device matrix (dtype, row stride ld), via an f32 staging buffer and the pack kernel.
void upload_rows(cd_layer* h, const float* host, int64_t row_begin, int64_t nrows, int64_t cols,
                 void* dst, int64_t ld_pad, int64_t ld_dst, float* tmp, int* nonfinite = nullptr) {
    ck(cudaMemcpyAsync(tmp, host + row_begin * cols, sizeof(float) * nrows * cols,
                       cudaMemcpyHostToDevice, h->stream),
       "upload");
    if (nonfinite) ck(cdk::launch_count_nonfinite(tmp, nrows * cols, nonfinite, h->stream), "upload check");
    ck(cdk::launch_pack_rows(tmp, nrows, cols, cols, dst, h->L.dtype, ld_pad, ld_dst, h->stream), "pack_rows");
}

struct Req {
    int method = cdk::kDC;
    bool with_masks = false;  // exec_mc / exec_dc: caller-supplied masks
    int nb = 1;
    const float* x = nullptr;
    float tau = 0.0f;
    int reduction = CD_REDUCTION_UNORDERED;
    const uint8_t* ovr = nullptr;       // DC mask override
    const uint8_t* masks_in = nullptr;  // exec masks
    const float* u_in = nullptr;        // exec_mc u
    float* y = nullptr;
    uint8_t* mask_out = nullptr;
    float* ind_out = nullptr;
    int* alive_out = nullptr;
    float rms_eps = -1.0f;  // >= 0: the input is RMSNorm(x) (stacked layers)
    cudaStream_t stream = nullptr;
    // Stage timing (cd_bench_stages): PDL off, an event recorded after every launch.
    cudaEvent_t* marks = nullptr;
};

constexpr int kTcMinBatch = 8;  // batches from here on run on the tensor cores (bf16 layers)
// M-CountDown / CATS at batch 2-7: their CUDA-core path is two kernels (a dense W_up / W_gate
// GEMV, then the union records), register-bound at 2-4 samples (Gemma B=4: 116 us, 0.23 of
// HBM); the row-union GEMM streams all rows but at ~0.6 of HBM (72 us) -- it wins from batch 3
// (measured: B=2 59.7 vs 71.7 us, B=3 105.5 vs 71.6, B=4 122.1 vs 71.5)
constexpr int kTcMinBatchMC = 3;

// The tensor-core path (kernels_tc.cu) covers bf16 layers at batch >= 8 for the calls that
// threshold their own masks (pipelines, dense).  Caller-supplied masks -- exec_dc / exec_mc /
// exec_cats and pipeline_dc's mask_override -- stay on the CUDA-core kernels at every batch
// size: the reference guarantees a dead lane's rows and u entries are never read (its tests
// poison them with NaN, test_blocked_exec.cpp:101-116), while the row-union GEMM reads every
// row and 0 x NaN would reach y.
bool tc_eligible(const cd_layer* h, const Req& r) {
    const int min_nb = (r.method == cdk::kMC || r.method == cdk::kCATS) ? kTcMinBatchMC : kTcMinBatch;
    if (!h->use_tc || h->L.dtype != CD_DTYPE_BF16 || !h->L.w_up || r.nb < min_nb || r.marks) return false;
    if (!h->weights_finite) return false;
    if (r.reduction != CD_REDUCTION_UNORDERED) return false;
    if (r.with_masks || r.ovr) return false;
    return r.method != cdk::kDC || h->L.theta_bt;
}


// Enqueue one operator call (device pointers) on r.stream.  Returns the number of launches.
int run_chain(cd_layer* h, const Req& r) {
    const cdk::LayerDev& L = h->L;
    const cdk::Scratch& S = h->S;
    cdk::LaunchCfg c;
    c.num_sms = h->num_sms;
    c.stream = r.stream ? r.stream : h->stream;
    c.coop = !h->pdl_chain;
    const int64_t d = L.d, F = L.F;
    int launches = 0;
    if (r.marks) {
        c.pdl = false;
        if (r.nb > kMaxBatchFast || r.reduction != CD_REDUCTION_UNORDERED || r.with_masks)
            fail(CD_ERR_DATA, "stage timing covers the fused chain at batch <= 4 only");
    }
    // after each launch of the fused chain: stage-boundary event (timing runs only)
    auto mark = [&](int n_launched) {
        if (r.marks) ck(cudaEventRecord(r.marks[n_launched], c.stream), "event");
    };
    if (r.method == cdk::kDC && !r.with_masks && !L.theta_bt)
        fail(CD_ERR_DATA, "pipeline_dc: layer has no low-rank predictor attached");
    if (!L.w_up) fail(CD_ERR_DATA, "forward: handle holds only a predictor (no layer weights)");

    // input RMS norm: fused into k_dc_fused where that kernel runs, else one norm kernel first
    float* xn = r.rms_eps >= 0.0f ? h->rms_ws.get<float>(static_cast<size_t>(r.nb) * d) : nullptr;
    if (tc_eligible(h, r)) {
        if (xn) {
            ck(cdk::launch_rmsnorm(r.x, r.nb, d, r.rms_eps, xn, c), "rmsnorm");
            Req rn = r;
            rn.x = xn;
            rn.rms_eps = -1.0f;
            return 1 + run_chain(h, rn);
        }
        const cdk::tc::Plan p = cdk::tc::plan_for(r.nb, r.method);
        void* ws = h->tc_ws.get<uint8_t>(cdk::tc::workspace_bytes(L, p, c.num_sms));
        const uint8_t* ovr = r.with_masks ? r.masks_in : r.ovr;
        ck(cdk::tc::launch_batched(L, p, ws, S.tc_flags, r.method, r.nb, r.x, r.tau, ovr, r.y, r.mask_out,
                                   r.ind_out, r.alive_out, c),
           "batched (tensor cores)");
        h->last_path = CD_PATH_TENSOR;
        if (p.split) return 1;  // decode: one persistent kernel (k_tc_fused)
        // prefill: x pack, gate/up, [zero of the stream-K tiles], down
        const int64_t units = ((r.nb + 255) / 256) * ((d + 511) / 512);  // column-tile pairs
        const int64_t clusters = (std::min<int64_t>(c.num_sms, cdk::kMaxCtas) & ~1) / 2;
        return 3 + (units % clusters != 0 ? 1 : 0);
    }
    h->last_path = r.reduction == CD_REDUCTION_UNORDERED ? CD_PATH_FAST : CD_PATH_EXACT;
    if (r.reduction == CD_REDUCTION_UNORDERED) {
        for (int c0 = 0; c0 < r.nb; c0 += kMaxBatchFast) {
            const int n = std::min(kMaxBatchFast, r.nb - c0);
            const float* xc = r.x + c0 * d;
            auto norm_x = [&]() {
                if (xn && xc != xn + c0 * d) {
                    ck(cdk::launch_rmsnorm(r.x + c0 * d, n, d, r.rms_eps, xn + c0 * d, c), "rmsnorm");
                    xc = xn + c0 * d;
                    launches += 1;
                }
            };
            float* yc = r.y + c0 * d;
            uint8_t* mo = r.mask_out ? r.mask_out + c0 * F : nullptr;
            float* io = r.ind_out ? r.ind_out + c0 * F : nullptr;
            int* ao = r.alive_out ? r.alive_out + c0 : nullptr;
            if (r.with_masks) {
                norm_x();
                ck(cdk::launch_compact_masks(L, S, r.masks_in + c0 * F,
                                             r.method != cdk::kDC ? r.u_in + c0 * F : nullptr, n, yc, c),
                   "compact_masks");
                ck(cdk::launch_sparse_fast(L, S, r.method, false, xc, n, yc, ao, c), "sparse");
                launches += 2;
            } else if (r.method == cdk::kDense) {
                // two launches: the y-zeroing kernel, then the all-rows FFN kernel
                norm_x();
                ck(cdk::launch_sparse_fast(L, S, cdk::kDC, true, xc, n, yc, ao, c), "dense");
                launches += 2;
                mark(0);
            } else if (r.method == cdk::kMC && n == 1 && h->use_fused && (norm_x(), true) &&
                       cdk::launch_mc_fused(L, S, xc, r.tau, yc, mo, io, ao, c) == cudaSuccess) {
                launches += 1;
                mark(0);
            } else if (r.method == cdk::kMC || r.method == cdk::kCATS) {
                (void)cudaGetLastError();
                norm_x();
                const bool cats = r.method == cdk::kCATS;
                ck(cdk::launch_indicator_mc_fast(L, S, xc, n, r.tau, yc, mo, io, c, cats), "indicator_mc");
                mark(0);
                ck(cdk::launch_sparse_fast(L, S, r.method, false, xc, n, yc, ao, c), "sparse_mc");
                mark(1);
                launches += 2;
            } else if (h->use_fused &&
                       cdk::launch_dc_fused(L, S, xc, n, r.tau, r.ovr ? r.ovr + c0 * F : nullptr, yc, mo, io, ao,
                                            c, r.rms_eps, h->pf_at, h->pf_bt) == cudaSuccess) {
                launches += 1;
                mark(0);
            } else {
                (void)cudaGetLastError();  // an unsupported fused shape: use the chain
                norm_x();
                ck(cdk::launch_latent_fast(L, S, xc, n, c), "latent");
                mark(0);
                ck(cdk::launch_indicator_dc_fast(L, S, n, r.tau, r.ovr ? r.ovr + c0 * F : nullptr, yc, mo, io, c),
                   "indicator_dc");
                mark(1);
                ck(cdk::launch_sparse_fast(L, S, cdk::kDC, false, xc, n, yc, ao, c), "sparse_dc");
                mark(2);
                launches += 3;
            }
        }
        return launches;
    }

    // ---- DeterministicOrdered: bitwise reference folds.
    for (int c0 = 0; c0 < r.nb; c0 += kMaxBatch) {
        const int n = std::min(kMaxBatch, r.nb - c0);
        const float* xc = r.x + c0 * d;
        if (xn) {
            ck(cdk::launch_rmsnorm(xc, n, d, r.rms_eps, xn + c0 * d, c), "rmsnorm");
            xc = xn + c0 * d;
            launches += 1;
        }
        float* yc = r.y + c0 * d;
        uint8_t* mo = r.mask_out ? r.mask_out + c0 * F : nullptr;
        int* ao = r.alive_out ? r.alive_out + c0 : nullptr;
        float* ind = r.ind_out ? r.ind_out + c0 * F : S.ind;
        const float* u_full = nullptr;
        if (r.with_masks) {
            if (r.method == cdk::kMC || r.method == cdk::kCATS) u_full = r.u_in + c0 * F;
            ck(cdk::launch_exact_compact(L, S, 2, nullptr, r.masks_in + c0 * F, n, 0.0f, mo, ao, c), "compact");
            launches += 1;
        } else if (r.method == cdk::kDense) {
            ck(cdk::launch_exact_compact(L, S, 3, nullptr, nullptr, n, 0.0f, mo, ao, c), "compact");
            launches += 1;
        } else if (r.method == cdk::kMC) {
            ck(cdk::launch_exact_rowdot_all(L.w_up, L.dtype, F, L.rs, d, xc, d, n, ind, F, c), "rowdot_up");
            ck(cdk::launch_exact_compact(L, S, 0, ind, nullptr, n, r.tau, mo, ao, c), "compact");
            u_full = ind;
            launches += 2;
        } else if (r.method == cdk::kCATS) {
            // pipeline_cats (blocked_exec.cpp:330-348): gate pass, act, |act| > tau
            ck(cdk::launch_exact_rowdot_all(L.w_gate, L.dtype, F, L.rs, d, xc, d, n, ind, F, c), "rowdot_gate");
            ck(cdk::launch_exact_act(L.act, ind, (int64_t)n * F, c), "act");
            ck(cdk::launch_exact_compact(L, S, 0, ind, nullptr, n, r.tau, mo, ao, c), "compact");
            u_full = ind;
            launches += 3;
        } else {
            ck(cdk::launch_exact_latent(L, S, xc, n, c), "latent_exact");
            ck(cdk::launch_exact_rowdot_all(L.theta_bt, L.dtype, F, L.ldr, L.r, S.ex_lat, L.ldr, n, ind, F, c),
               "logits_exact");
            if (r.ovr)
                ck(cdk::launch_exact_compact(L, S, 2, nullptr, r.ovr + c0 * F, n, 0.0f, mo, ao, c), "compact");
            else
                ck(cdk::launch_exact_compact(L, S, 1, ind, nullptr, n, r.tau, mo, ao, c), "compact");
            launches += 3;
        }
        const int m = r.method == cdk::kDense ? cdk::kDC : r.method;
        ck(cdk::launch_exact_phase1(L, S, m, xc, u_full, n, c), "phase1");
        ck(cdk::launch_exact_down(L, S, n, yc, c), "down");
        launches += 2;
        // restore the self-cleaning scratch the fast chain relies on
        ck(cudaMemsetAsync(S.count, 0, sizeof(int), c.stream), "memset");
        ck(cudaMemsetAsync(S.alive, 0, sizeof(int) * kMaxBatch, c.stream), "memset");
    }
    return launches;
}

void check_layer(const cd_layer* h) {
    if (!h) fail(CD_ERR_DATA, "null layer handle");
}

void check_common(const cd_layer* h, int64_t batch, const float* x, const float* y) {
    check_layer(h);
    if (batch <= 0) fail(CD_ERR_DATA, "batch must be positive");
    if (!x) fail(CD_ERR_DATA, "x is null");
    if (!y) fail(CD_ERR_DATA, "y is null");
}

void check_reduction(int reduction) {
    if (reduction != CD_REDUCTION_ORDERED && reduction != CD_REDUCTION_UNORDERED)
        fail(CD_ERR_DATA, "unknown reduction mode");
}

// Host-buffer call: stage through pinned memory in chunks of kMaxBatch samples.
struct HostIO {
    const float* x = nullptr;
    const uint8_t* masks_in = nullptr;
    const uint8_t* ovr = nullptr;
    const float* u_in = nullptr;
    float* y = nullptr;
    uint8_t* mask_out = nullptr;
    float* ind_out = nullptr;
    int64_t* alive_out = nullptr;
};

// NVTX range for the length of a scope (host-side enqueue of one operator call)
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};

void host_call(cd_layer* h, Req base, int64_t batch, const HostIO& io) {
    NvtxRange nv("cd.host_call");
    CallLock lk(h);
    ck(cudaSetDevice(h->device), "cudaSetDevice");
    const int64_t d = h->L.d, F = h->L.F;
    cudaStream_t s = h->stream;
    int launches = 0;
    // the tensor-core path takes the whole batch at once (large-batch staging grows on demand)
    Req probe = base;
    probe.nb = static_cast<int>(std::min<int64_t>(batch, 1 << 30));
    const int64_t chunk = tc_eligible(h, probe) ? batch : kMaxBatch;
    const bool big = chunk > kMaxBatch;
    const size_t cf = static_cast<size_t>(chunk * F), cd = static_cast<size_t>(chunk * d);
    float* d_x = big ? h->g_dx.get<float>(cd) : h->d_x;
    float* d_y = big ? h->g_dy.get<float>(cd) : h->d_y;
    int* d_alive = big ? h->g_dalive.get<int>(chunk) : h->d_alive;
    float* h_x = big ? h->g_hx.get<float>(cd) : h->h_x;
    float* h_y = big ? h->g_hy.get<float>(cd) : h->h_y;
    int* h_alive = big ? h->g_halive.get<int>(chunk) : h->h_alive;
    const bool need_mask = io.masks_in || io.ovr || io.mask_out;
    uint8_t* d_mask_in = big ? ((io.masks_in || io.ovr) ? h->g_dmask_in.get<uint8_t>(cf) : nullptr) : h->d_mask_in;
    uint8_t* d_mask_out = big ? (io.mask_out ? h->g_dmask_out.get<uint8_t>(cf) : nullptr) : h->d_mask_out;
    uint8_t* h_mask = big ? (need_mask ? h->g_hmask.get<uint8_t>(cf) : nullptr) : h->h_mask;
    float* d_u_in = big ? (io.u_in ? h->g_du_in.get<float>(cf) : nullptr) : h->d_u_in;
    float* d_ind = big ? (io.ind_out ? h->g_dind.get<float>(cf) : nullptr) : h->d_ind;
    float* h_ind = big ? ((io.ind_out || io.u_in) ? h->g_hind.get<float>(cf) : nullptr) : h->h_ind;
    // single-chunk calls from the fixed staging replay a captured graph of the whole sequence
    const bool graphable = h->use_host_graph && !big && batch <= chunk;
    uint64_t key = 0;
    if (graphable) {
        uint32_t tau_bits;
        std::memcpy(&tau_bits, &base.tau, 4);
        key = (static_cast<uint64_t>(tau_bits) << 32) ^ (static_cast<uint64_t>(batch) << 20) ^
              (static_cast<uint64_t>(base.method) << 16) ^ (static_cast<uint64_t>(base.reduction) << 12) ^
              (base.with_masks ? 1u << 8 : 0u) ^ (io.ovr ? 1u << 9 : 0u) ^ (io.masks_in ? 1u << 10 : 0u) ^
              (io.u_in ? 1u << 11 : 0u) ^ (io.mask_out ? 1u << 5 : 0u) ^ (io.ind_out ? 1u << 6 : 0u) ^ 1u;
        key = key * 0x9E3779B97F4A7C15ull ^ h->gen;  // device state the graph's pointers come from
        if (h->hg.key != key) {
            if (h->hg.exec) cudaGraphExecDestroy(h->hg.exec);
            h->hg = {};
            h->hg.key = key;
        }
    }
    for (int64_t c0 = 0; c0 < batch; c0 += chunk) {
        const int n = static_cast<int>(std::min<int64_t>(chunk, batch - c0));
        std::memcpy(h_x, io.x + c0 * d, sizeof(float) * n * d);
        const uint8_t* masks = io.masks_in ? io.masks_in : io.ovr;
        if (masks) std::memcpy(h_mask, masks + c0 * F, static_cast<size_t>(n * F));
        if (io.u_in) std::memcpy(h_ind, io.u_in + c0 * F, sizeof(float) * n * F);
        const bool replay = graphable && h->hg.exec;
        // small single-chunk calls without mask / indicator outputs: copy-out + completion word
        const bool signal = !big && h->mapped_staging && h->h_done && batch <= chunk && !io.mask_out && !io.ind_out;
        const bool capture = graphable && !replay && ++h->hg.seen >= 2;
        const uint64_t gen_before = h->gen;
        if (replay) {
            ck(cudaGraphLaunch(h->hg.exec, s), "graph launch");
            launches += h->hg.launches;
            h->last_path = h->hg.path;
        } else {
        cudaGraph_t graph = nullptr;
        if (capture) ck(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal), "capture");
        // small transfers from the fixed (mapped) pinned staging: a copy kernel, not the DMA engine
        auto xfer = [&](void* dst, const void* src, size_t bytes, cudaMemcpyKind kind, const char* what) {
            if (!big && h->mapped_staging && bytes <= (size_t{1} << 20))
                ck(cdk::launch_copy(dst, src, bytes, s), what);
            else
                ck(cudaMemcpyAsync(dst, src, bytes, kind, s), what);
        };
        xfer(d_x, h_x, sizeof(float) * n * d, cudaMemcpyHostToDevice, "H2D x");
        if (masks) xfer(d_mask_in, h_mask, static_cast<size_t>(n * F), cudaMemcpyHostToDevice, "H2D mask");
        if (io.u_in) xfer(d_u_in, h_ind, sizeof(float) * n * F, cudaMemcpyHostToDevice, "H2D u");
        Req r = base;
        r.nb = n;
        r.x = d_x;
        r.y = d_y;
        r.masks_in = io.masks_in ? d_mask_in : nullptr;
        r.ovr = io.ovr ? d_mask_in : nullptr;
        r.u_in = io.u_in ? d_u_in : nullptr;
        r.mask_out = io.mask_out ? d_mask_out : nullptr;
        r.ind_out = io.ind_out ? d_ind : nullptr;
        r.alive_out = d_alive;
        r.stream = s;
        int nl = 0;
        try {
            nl = run_chain(h, r);
            if (signal) {
                ck(cdk::launch_copy_out_signal(h_y, d_y, n * d, h_alive, d_alive, n, h->h_done, s, h->pdl_chain),
                   "D2H y + signal");
            } else {
                xfer(h_y, d_y, sizeof(float) * n * d, cudaMemcpyDeviceToHost, "D2H y");
                xfer(h_alive, d_alive, sizeof(int) * n, cudaMemcpyDeviceToHost, "D2H alive");
            }
            // pinned staging is reused below: the stream sync orders the uploads before the reuse
            if (io.mask_out) xfer(h_mask, d_mask_out, static_cast<size_t>(n * F), cudaMemcpyDeviceToHost, "D2H mask");
            if (io.ind_out) xfer(h_ind, d_ind, sizeof(float) * n * F, cudaMemcpyDeviceToHost, "D2H ind");
        } catch (...) {
            if (capture) {
                cudaStreamEndCapture(s, &graph);
                if (graph) cudaGraphDestroy(graph);
                h->use_host_graph = false;
            }
            throw;
        }
        launches += nl;
        if (capture) {
            ck(cudaStreamEndCapture(s, &graph), "capture end");
            const cudaError_t ie = cudaGraphInstantiate(&h->hg.exec, graph, 0);
            cudaGraphDestroy(graph);
            if (ie != cudaSuccess) {
                h->hg.exec = nullptr;
                h->use_host_graph = false;
                ck(ie, "graph instantiate");
            }
            h->hg.launches = nl;
            h->hg.path = h->last_path;
            ck(cudaGraphLaunch(h->hg.exec, s), "graph launch");
            if (h->gen != gen_before) {  // a buffer moved while capturing: never replay this graph
                ck(cudaStreamSynchronize(s), "forward");
                cudaGraphExecDestroy(h->hg.exec);
                h->hg = {};
            }
        }
        }
        if (signal) {
            // the completion word: spin on it (wakes within ~1 us of the kernel's write, where a
            // stream synchronisation sleeps); after ~50 ms fall back to the synchronisation,
            // which also reports a failed launch
            const unsigned long long want = ++h->done_seen;
            const volatile unsigned long long* w = h->h_done;
            bool ok = false;
            for (long it = 0; it < (1L << 22); ++it)
                if (*w >= want) {
                    ok = true;
                    break;
                }
            if (!ok) {
                ck(cudaStreamSynchronize(s), "forward");
                if (*w < want) fail(CD_ERR_CUDA, "forward: completion word not written");
            }
            std::atomic_thread_fence(std::memory_order_acquire);
            const cudaError_t qe = cudaStreamQuery(s);  // a sticky device error surfaces here
            if (qe != cudaSuccess && qe != cudaErrorNotReady) ck(qe, "forward");
            if (qe == cudaErrorNotReady) (void)cudaGetLastError();
        } else {
            ck(cudaStreamSynchronize(s), "forward");
        }
        std::memcpy(io.y + c0 * d, h_y, sizeof(float) * n * d);
        if (io.mask_out) std::memcpy(io.mask_out + c0 * F, h_mask, static_cast<size_t>(n * F));
        if (io.ind_out) std::memcpy(io.ind_out + c0 * F, h_ind, sizeof(float) * n * F);
        if (io.alive_out)
            for (int b = 0; b < n; ++b) io.alive_out[c0 + b] = h_alive[b];
    }
    h->last_launches = launches;
}

// ---------------------------------------------------------------- CDWN1 model files
// The reference's on-disk model container (model_io.cpp:94-224): magic "CDWN1", u32 header
// length, JSON header, then little-endian f32 blobs W_up, W_gate, W_down and the optional
// predictor.  A small JSON reader covers the header schema (objects, strings, numbers, null).
struct JVal {
    enum Kind { kNull, kNum, kStr, kObj } kind = kNull;
    double num = 0.0;
    std::string tok;  // the number's literal (integers are read from it exactly)
    std::string str;
    std::map<std::string, JVal> obj;
};

struct JParser {
    const std::string& s;
    size_t i = 0;
    void ws() {
        while (i < s.size() && (s[i] == ' ' || s[i] == '\n' || s[i] == '\t' || s[i] == '\r')) ++i;
    }
    [[noreturn]] void bad() { throw std::runtime_error("bad header JSON"); }
    std::string str() {
        if (s[i] != '"') bad();
        std::string out;
        for (++i; i < s.size() && s[i] != '"'; ++i) {
            if (s[i] == '\\') {
                if (++i >= s.size()) bad();
            }
            out.push_back(s[i]);
        }
        if (i >= s.size()) bad();
        ++i;
        return out;
    }
    JVal value() {
        ws();
        if (i >= s.size()) bad();
        JVal v;
        if (s[i] == '{') {
            v.kind = JVal::kObj;
            ++i;
            ws();
            if (s[i] == '}') { ++i; return v; }
            for (;;) {
                ws();
                std::string k = str();
                ws();
                if (s[i++] != ':') bad();
                v.obj[k] = value();
                ws();
                if (s[i] == ',') { ++i; continue; }
                if (s[i] == '}') { ++i; return v; }
                bad();
            }
        }
        if (s[i] == '"') {
            v.kind = JVal::kStr;
            v.str = str();
            return v;
        }
        if (s.compare(i, 4, "null") == 0) {
            i += 4;
            return v;
        }
        size_t end = i;
        while (end < s.size() && std::strchr("+-.0123456789eE", s[end])) ++end;
        if (end == i) bad();
        v.kind = JVal::kNum;
        v.tok = s.substr(i, end - i);
        v.num = std::stod(v.tok);
        i = end;
        return v;
    }
};

// Field access with nlohmann's get<T> semantics (model_io.cpp:146-153, 165-170): a missing key
// or a value of the wrong JSON kind is a DataError "<path>: <what>: ..."; integers are read
// exactly from their literal (a fractional literal converts like get<int64_t> on a float).
const JVal& jfield(const JVal& o, const char* k, const std::string& path, const char* what = "bad header field") {
    auto it = o.obj.find(k);
    if (o.kind != JVal::kObj || it == o.obj.end())
        fail(CD_ERR_DATA, path + ": " + what + ": key '" + k + "' not found");
    return it->second;
}

const std::string& jstr(const JVal& o, const char* k, const std::string& path, const char* what = "bad header field") {
    const JVal& v = jfield(o, k, path, what);
    if (v.kind != JVal::kStr) fail(CD_ERR_DATA, path + ": " + what + ": '" + k + "' must be a string");
    return v.str;
}

double jnum(const JVal& o, const char* k, const std::string& path, const char* what = "bad header field") {
    const JVal& v = jfield(o, k, path, what);
    if (v.kind != JVal::kNum) fail(CD_ERR_DATA, path + ": " + what + ": '" + k + "' must be a number");
    return v.num;
}

template <typename T>
T jint(const JVal& o, const char* k, const std::string& path, const char* what = "bad header field") {
    const JVal& v = jfield(o, k, path, what);
    if (v.kind != JVal::kNum) fail(CD_ERR_DATA, path + ": " + what + ": '" + k + "' must be a number");
    if (v.tok.find_first_of(".eE") != std::string::npos) return static_cast<T>(static_cast<long double>(v.num));
    errno = 0;
    char* end = nullptr;
    T out;
    if (v.tok[0] == '-') {
        const long long t = std::strtoll(v.tok.c_str(), &end, 10);
        out = static_cast<T>(t);
    } else {
        const unsigned long long t = std::strtoull(v.tok.c_str(), &end, 10);
        out = static_cast<T>(t);
    }
    if (errno == ERANGE || !end || *end != '\0')
        fail(CD_ERR_DATA, path + ": " + what + ": '" + k + "' is out of range");
    return out;
}

void check_finite_blob(const float* p, size_t n, const std::string& path, const char* what) {
    for (size_t i = 0; i < n; ++i)
        if (!std::isfinite(p[i]))
            fail(CD_ERR_DATA, path + ": " + std::string(what) + " contains a non-finite value at index " +
                                  std::to_string(i));
}

// Sub-allocation of one block: a sizing pass (base null) then a carving pass.
struct Carve {
    size_t off = 0;
    uint8_t* base = nullptr;
    template <typename T> T* take(size_t n) {
        off = (off + 255) & ~size_t{255};
        T* p = base ? reinterpret_cast<T*>(base + off) : nullptr;
        off += std::max<size_t>(n, 1) * sizeof(T);
        return p;
    }
};

cd_layer* create_impl(int device, int64_t d, int64_t F_total, int64_t rb, int64_t re, int act,
                      int dtype, const float* w_up, const float* w_gate, const float* w_down,
                      bool predictor_only = false) {
    if (d <= 0 || F_total <= 0) {
        fail(CD_ERR_DATA, "layer: bad dims d_model=" + std::to_string(d) + " d_inter=" + std::to_string(F_total));
    }
    if (rb < 0 || re > F_total || re <= rb) fail(CD_ERR_DATA, "layer: bad shard row range");
    if (act != CD_ACT_SILU && act != CD_ACT_GELU_TANH) fail(CD_ERR_DATA, "layer: unknown activation");
    if (dtype != CD_DTYPE_F32 && dtype != CD_DTYPE_BF16) fail(CD_ERR_DATA, "layer: unknown dtype");
    if (!predictor_only && (!w_up || !w_gate || !w_down)) fail(CD_ERR_DATA, "layer: null weight pointer");
    int ndev = 0;
    ck(cudaGetDeviceCount(&ndev), "cudaGetDeviceCount");
    if (device < 0 || device >= ndev) fail(CD_ERR_CUDA, "no such CUDA device");
    ck(cudaSetDevice(device), "cudaSetDevice");
    cudaDeviceProp prop;
    ck(cudaGetDeviceProperties(&prop, device), "cudaGetDeviceProperties");
    if (prop.major != 10 || prop.minor != 0)
        fail(CD_ERR_CUDA, "libcountdown_b200 is built for sm_100a (B200); device is sm_" +
                              std::to_string(prop.major) + std::to_string(prop.minor));

    auto h = std::make_unique<cd_layer>();
    h->device = device;
    h->num_sms = prop.multiProcessorCount;
    DeviceCtx& ctx = device_ctx(device);
    std::lock_guard<std::recursive_mutex> dlock(ctx.mu);
    h->stream = ctx.stream;
    h->dev_mu = &ctx.mu;
    for (Grow* g : {&h->tc_ws, &h->rms_ws, &h->g_dx, &h->g_dy, &h->g_dmask_in, &h->g_dmask_out, &h->g_du_in,
                    &h->g_dind, &h->g_dalive, &h->g_hx, &h->g_hy, &h->g_hmask, &h->g_hind, &h->g_halive})
        g->gen = &h->gen;
    cdk::LayerDev& L = h->L;
    L.d = d;
    L.F = re - rb;
    L.ld = round_up(d, cdk::kVecElems);
    L.rs = 3 * L.ld;
    L.act = act;
    L.dtype = dtype;
    h->F_total = F_total;
    h->row_begin = rb;
    const size_t esz = dtype == CD_DTYPE_BF16 ? 2 : 4;
    const size_t nw = static_cast<size_t>(L.F * L.rs);
    if (!predictor_only) {
    // neuron records [up | gate | down]; the padding columns are zeroed by the pack kernel
    uint8_t* rec = h->dalloc<uint8_t>(nw * esz, false);
    void* wu = rec;
    void* wg = rec + L.ld * esz;
    void* wd = rec + 2 * L.ld * esz;
    float* tmp = nullptr;
    ck(cudaMalloc(&tmp, sizeof(float) * (L.F * d + 1)), "cudaMalloc tmp");
    int* nonfinite = reinterpret_cast<int*>(tmp + L.F * d);
    int bad = 0;
    try {
        ck(cudaMemsetAsync(nonfinite, 0, sizeof(int), h->stream), "memset");
        upload_rows(h.get(), w_up, rb, L.F, d, wu, L.ld, L.rs, tmp, nonfinite);
        upload_rows(h.get(), w_gate, rb, L.F, d, wg, L.ld, L.rs, tmp, nonfinite);
        upload_rows(h.get(), w_down, rb, L.F, d, wd, L.ld, L.rs, tmp, nonfinite);
        ck(cudaMemcpyAsync(&bad, nonfinite, sizeof(int), cudaMemcpyDeviceToHost, h->stream), "upload check");
        ck(cudaStreamSynchronize(h->stream), "upload");
    } catch (...) {
        cudaFree(tmp);
        throw;
    }
    cudaFree(tmp);
    // The reference accepts non-finite weights (GatedMlpLayer::validate checks shapes only) and
    // never reads a dead lane's gate / down rows.  The row-union GEMM reads every row, so a
    // layer holding a non-finite (or bf16-overflowing) weight stays on the CUDA-core kernels.
    h->weights_finite = bad == 0;
    L.w_up = wu;
    L.w_gate = wg;
    L.w_down = wd;
    }

    cdk::Scratch& S = h->S;
    // scratch and staging: ONE zeroed device block and ONE mapped pinned block, carved up
    // (a handle is created per cached layer by the C++ shims: ~20 separate allocations cost
    // more than the small layers' calls themselves)
    const size_t Fz = static_cast<size_t>(L.F), dz = static_cast<size_t>(d);
    auto carve_dev = [&](Carve& cv) {
        S.list = cv.take<int32_t>(Fz);
        S.bits = cv.take<uint32_t>(Fz);
        S.list_val = cv.take<float>(Fz * kMaxBatchFast);
        S.count = cv.take<int>(1);
        S.done = cv.take<int>(1);
        S.alive = cv.take<int>(kMaxBatch);
        S.ctl = cv.take<unsigned>(128);
        S.t_list = cv.take<unsigned long long>(Fz + cdk::kMaxCtas);  // per-CTA regions of ceil(F/G)
        S.t_aux = cv.take<unsigned long long>(Fz);
        S.t_count = cv.take<unsigned long long>(cdk::kMaxCtas);
        S.t_alive = cv.take<unsigned long long>(cdk::kMaxCtas * kMaxBatchFast);
        S.tc_flags = cv.take<unsigned>(cdk::kMaxCtas + 64);
        S.ind = cv.take<float>(kMaxBatch * Fz);
        S.ex_s = cv.take<float>(kMaxBatch * Fz);
        h->d_x = cv.take<float>(kMaxBatch * dz);
        h->d_y = cv.take<float>(kMaxBatch * dz);
        h->d_mask_in = cv.take<uint8_t>(kMaxBatch * Fz);
        h->d_mask_out = cv.take<uint8_t>(kMaxBatch * Fz);
        h->d_u_in = cv.take<float>(kMaxBatch * Fz);
        h->d_ind = cv.take<float>(kMaxBatch * Fz);
        h->d_alive = cv.take<int>(kMaxBatch);
    };
    Carve sizing;
    carve_dev(sizing);
    Carve dev_cv;
    dev_cv.base = h->dalloc<uint8_t>(sizing.off);  // zeroed
    carve_dev(dev_cv);
    auto carve_host = [&](Carve& cv) {
        h->h_x = cv.take<float>(kMaxBatch * dz);
        h->h_y = cv.take<float>(kMaxBatch * dz);
        h->h_mask = cv.take<uint8_t>(kMaxBatch * Fz);
        h->h_ind = cv.take<float>(kMaxBatch * Fz);
        h->h_alive = cv.take<int>(kMaxBatch);
        h->h_done = cv.take<unsigned long long>(1);
    };
    Carve hsize;
    carve_host(hsize);
    Carve host_cv;
    host_cv.base = h->halloc<uint8_t>(hsize.off);
    carve_host(host_cv);
    *h->h_done = 0;  // pinned allocations are not zeroed: the completion word counts from 0
    h->done_seen = 0;
    return h.release();
}

}  // namespace

extern "C" {

const char* cd_last_error(void) { return g_err.c_str(); }

int cd_version(void) { return 1; }

int cd_device_info(int device, int* num_sms, int* cc_major, int* cc_minor) {
    return guarded([&] {
        cudaDeviceProp prop;
        ck(cudaGetDeviceProperties(&prop, device), "cudaGetDeviceProperties");
        if (num_sms) *num_sms = prop.multiProcessorCount;
        if (cc_major) *cc_major = prop.major;
        if (cc_minor) *cc_minor = prop.minor;
    });
}

int cd_layer_create(int device, int64_t d_model, int64_t d_inter, int activation, int dtype,
                    const float* w_up, const float* w_gate, const float* w_down, cd_layer** out) {
    return guarded([&] {
        if (!out) fail(CD_ERR_DATA, "out is null");
        *out = create_impl(device, d_model, d_inter, 0, d_inter, activation, dtype, w_up, w_gate, w_down);
    });
}

int cd_layer_create_shard(int device, int64_t d_model, int64_t d_inter_total, int64_t row_begin,
                          int64_t row_end, int activation, int dtype, const float* w_up,
                          const float* w_gate, const float* w_down, cd_layer** out) {
    return guarded([&] {
        if (!out) fail(CD_ERR_DATA, "out is null");
        *out = create_impl(device, d_model, d_inter_total, row_begin, row_end, activation, dtype, w_up,
                           w_gate, w_down);
    });
}

int cd_layer_load_cdwn1(int device, const char* path, int dtype, cd_layer** out, int64_t* dims_out) {
    return guarded([&] {
        if (!out || !path) fail(CD_ERR_DATA, "load: null argument");
        const std::string p(path);
        std::ifstream in(p, std::ios::binary);
        if (!in) fail(CD_ERR_DATA, "cannot open '" + p + "' for reading");
        std::ostringstream oss;
        oss << in.rdbuf();
        const std::string buf = oss.str();
        if (buf.size() < 5 || buf.compare(0, 5, "CDWN1") != 0)
            fail(CD_ERR_DATA, p + ": not a model file (bad magic, expected CDWN1)");
        if (buf.size() < 9) fail(CD_ERR_DATA, p + ": truncated header length");
        uint32_t hlen = 0;
        std::memcpy(&hlen, buf.data() + 5, 4);
        if (buf.size() < 9 + static_cast<size_t>(hlen)) fail(CD_ERR_DATA, p + ": truncated header");
        const std::string hs = buf.substr(9, hlen);
        JVal h;
        try {
            JParser jp{hs};
            h = jp.value();
        } catch (const std::exception& e) {
            fail(CD_ERR_DATA, p + ": bad header JSON: " + e.what());
        }
        if (jstr(h, "schema", p) != "v1") fail(CD_ERR_DATA, p + ": unsupported schema");
        const int64_t d = jint<int64_t>(h, "d_model", p);
        const int64_t F = jint<int64_t>(h, "d_inter", p);
        const std::string act_name = jstr(h, "activation", p);
        int act = -1;
        if (act_name == "silu") act = CD_ACT_SILU;
        else if (act_name == "gelu") act = CD_ACT_GELU_TANH;
        else fail(CD_ERR_DATA, "unknown activation '" + act_name + "' (expected silu|gelu)");
        const uint64_t seed = jint<uint64_t>(h, "seed", p);
        if (d <= 0 || F <= 0) fail(CD_ERR_DATA, p + ": non-positive dimensions in header");
        const size_t mat = static_cast<size_t>(d) * static_cast<size_t>(F);
        size_t expected = 3 * mat * 4;
        int64_t r = 0;  // 0: no predictor, -1: ternary (not attached: no B200 path)
        auto pit = h.obj.find("predictor");
        if (pit != h.obj.end() && pit->second.kind == JVal::kObj) {
            const char* pd = "bad predictor descriptor";
            const std::string kind = jstr(pit->second, "kind", p, pd);
            (void)jnum(pit->second, "k", p, pd);
            if (kind == "lowrank") {
                r = jint<int64_t>(pit->second, "d_rank", p, pd);
                if (r <= 0) fail(CD_ERR_DATA, p + ": non-positive predictor rank");
                expected += (static_cast<size_t>(d) * r + static_cast<size_t>(r) * F) * 4;
            } else if (kind == "ternary") {
                r = -1;
                expected += 4 + mat * 4;
            } else {
                fail(CD_ERR_DATA, p + ": unknown predictor kind '" + kind + "'");
            }
        }
        const size_t payload = buf.size() - 9 - hlen;
        if (payload != expected)
            fail(CD_ERR_DATA, p + ": payload is " + std::to_string(payload) + " bytes, expected " +
                                  std::to_string(expected));
        const float* blob = reinterpret_cast<const float*>(buf.data() + 9 + hlen);
        if ((reinterpret_cast<uintptr_t>(blob) & 3) != 0) {
            // unaligned header length: copy the payload to an aligned buffer
            static thread_local std::vector<float> aligned;
            aligned.resize(payload / 4);
            std::memcpy(aligned.data(), blob, payload);
            blob = aligned.data();
        }
        check_finite_blob(blob, mat, p, "w_up");
        check_finite_blob(blob + mat, mat, p, "w_gate");
        check_finite_blob(blob + 2 * mat, mat, p, "w_down");
        std::unique_ptr<cd_layer> hl(create_impl(device, d, F, 0, F, act, dtype, blob, blob + mat, blob + 2 * mat));
        if (r > 0) {
            const float* ta = blob + 3 * mat;
            const float* tb = ta + d * r;
            check_finite_blob(ta, static_cast<size_t>(d * r), p, "theta_a");
            check_finite_blob(tb, static_cast<size_t>(r * F), p, "theta_b");
            const int rc = cd_layer_set_predictor(hl.get(), r, ta, tb);
            if (rc != CD_OK) throw Fail{rc};
        }
        if (dims_out) {
            dims_out[0] = d;
            dims_out[1] = F;
            dims_out[2] = r;
            dims_out[3] = act;
            dims_out[4] = static_cast<int64_t>(seed);
        }
        *out = hl.release();
    });
}

int cd_layer_set_predictor(cd_layer* h, int64_t d_rank, const float* theta_a, const float* theta_b) {
    return guarded([&] {
        check_layer(h);
        if (d_rank <= 0) fail(CD_ERR_DATA, "make_lowrank_predictor: dims must be positive");
        if (!theta_a || !theta_b) fail(CD_ERR_DATA, "predictor: null theta pointer");
        CallLock lk(h);
        ck(cudaSetDevice(h->device), "cudaSetDevice");
        cdk::LayerDev& L = h->L;
        const int64_t ldr = round_up(d_rank, cdk::kVecElems);
        if (ldr / cdk::kVecElems > 256) fail(CD_ERR_DATA, "predictor: d_rank > 2048 is not supported");
        const size_t esz = L.dtype == CD_DTYPE_BF16 ? 2 : 4;
        void* ta = h->dalloc<uint8_t>(static_cast<size_t>(L.d * ldr) * esz, false);
        void* tat = h->dalloc<uint8_t>(static_cast<size_t>(d_rank * L.ld) * esz, false);
        void* tbt = h->dalloc<uint8_t>(static_cast<size_t>(L.F * ldr) * esz, false);
        float* tmp = nullptr;
        const size_t tmp_n = static_cast<size_t>(std::max(L.d * d_rank, d_rank * h->F_total));
        ck(cudaMalloc(&tmp, sizeof(float) * tmp_n), "cudaMalloc tmp");
        cudaError_t e = cudaMemcpyAsync(tmp, theta_a, sizeof(float) * L.d * d_rank, cudaMemcpyHostToDevice, h->stream);
        if (e == cudaSuccess) e = cdk::launch_pack_rows(tmp, L.d, d_rank, d_rank, ta, L.dtype, ldr, ldr, h->stream);
        if (e == cudaSuccess)
            e = cdk::launch_pack_transpose(tmp, L.d, d_rank, 0, d_rank, tat, L.dtype, L.ld, h->stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
        if (e == cudaSuccess)
            e = cudaMemcpyAsync(tmp, theta_b, sizeof(float) * d_rank * h->F_total, cudaMemcpyHostToDevice, h->stream);
        if (e == cudaSuccess)
            e = cdk::launch_pack_transpose(tmp, d_rank, h->F_total, h->row_begin, L.F, tbt, L.dtype, ldr, h->stream);

        if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
        cudaFree(tmp);
        ck(e, "predictor upload");
        if (!h->S.latent) h->S.latent = h->dalloc<float>(kMaxBatch * 2048);
        if (!h->S.ex_lat) h->S.ex_lat = h->dalloc<float>(kMaxBatch * 2048);
        if (!h->S.t_lat) h->S.t_lat = h->dalloc<unsigned long long>(kMaxBatchFast * 2048);
        // the replaced predictor: its buffers are freed (cudaFree waits for the device) and the
        // saved host graph, which holds their addresses, is dropped
        h->dfree(L.theta_a);
        h->dfree(L.theta_at);
        h->dfree(L.theta_bt);
        if (h->hg.exec) cudaGraphExecDestroy(h->hg.exec);
        h->hg = {};
        ++h->gen;
        L.pred_kind = 0;
        L.r = d_rank;
        L.ldr = ldr;
        L.theta_a = ta;
        L.theta_at = tat;
        L.theta_bt = tbt;
    });
}

int cd_layer_destroy(cd_layer* h) {
    return guarded([&] {
        if (!h) return;
        std::lock_guard<std::recursive_mutex> d(*h->dev_mu);
        delete h;
    });
}

int cd_layer_shape(const cd_layer* h, int64_t* d_model, int64_t* d_inter, int64_t* d_rank, int* dtype,
                   int* activation) {
    return guarded([&] {
        check_layer(h);
        if (d_model) *d_model = h->L.d;
        if (d_inter) *d_inter = h->L.F;
        if (d_rank) *d_rank = h->L.r;
        if (dtype) *dtype = h->L.dtype;
        if (activation) *activation = h->L.act;
    });
}

int cd_layer_last_path(const cd_layer* h, int* path) {
    return guarded([&] {
        check_layer(h);
        if (!path) fail(CD_ERR_DATA, "path is null");
        *path = h->last_path;
    });
}

int cd_layer_device_bytes(const cd_layer* h, int64_t* bytes) {
    return guarded([&] {
        check_layer(h);
        *bytes = h->bytes;
    });
}

int cd_layer_last_launches(const cd_layer* h, int* launches) {
    return guarded([&] {
        check_layer(h);
        *launches = h->last_launches;
    });
}

int cd_exec_dense(cd_layer* h, int64_t batch, const float* x, int reduction, float* y) {
    return guarded([&] {
        check_common(h, batch, x, y);
        check_reduction(reduction);
        Req r;
        r.method = cdk::kDense;
        r.reduction = reduction;
        HostIO io;
        io.x = x;
        io.y = y;
        host_call(h, r, batch, io);
    });
}

int cd_exec_mc(cd_layer* h, int64_t batch, const float* x, const float* u, const uint8_t* mask,
               int reduction, float* y) {
    return guarded([&] {
        check_common(h, batch, x, y);
        check_reduction(reduction);
        if (!u || !mask) fail(CD_ERR_DATA, "exec_mc: u and mask are required");
        Req r;
        r.method = cdk::kMC;
        r.with_masks = true;
        r.reduction = reduction;
        HostIO io;
        io.x = x;
        io.y = y;
        io.u_in = u;
        io.masks_in = mask;
        host_call(h, r, batch, io);
    });
}

int cd_exec_dc(cd_layer* h, int64_t batch, const float* x, const uint8_t* mask, int reduction, float* y) {
    return guarded([&] {
        check_common(h, batch, x, y);
        check_reduction(reduction);
        if (!mask) fail(CD_ERR_DATA, "exec_dc: mask is required");
        Req r;
        r.method = cdk::kDC;
        r.with_masks = true;
        r.reduction = reduction;
        HostIO io;
        io.x = x;
        io.y = y;
        io.masks_in = mask;
        host_call(h, r, batch, io);
    });
}

int cd_pipeline_mc(cd_layer* h, int64_t batch, const float* x, float tau, int reduction, float* y,
                   uint8_t* mask_out, int64_t* alive_out, float* u_out) {
    return guarded([&] {
        check_common(h, batch, x, y);
        check_reduction(reduction);
        Req r;
        r.method = cdk::kMC;
        r.tau = tau;
        r.reduction = reduction;
        HostIO io;
        io.x = x;
        io.y = y;
        io.mask_out = mask_out;
        io.alive_out = alive_out;
        io.ind_out = u_out;
        host_call(h, r, batch, io);
    });
}

int cd_exec_cats(cd_layer* h, int64_t batch, const float* x, const float* act_gate, const uint8_t* mask,
                 int reduction, float* y) {
    return guarded([&] {
        check_common(h, batch, x, y);
        check_reduction(reduction);
        if (!act_gate || !mask) fail(CD_ERR_DATA, "exec_cats: act_gate and mask are required");
        Req r;
        r.method = cdk::kCATS;
        r.with_masks = true;
        r.reduction = reduction;
        HostIO io;
        io.x = x;
        io.y = y;
        io.u_in = act_gate;
        io.masks_in = mask;
        host_call(h, r, batch, io);
    });
}

int cd_pipeline_cats(cd_layer* h, int64_t batch, const float* x, float tau, int reduction, float* y,
                     uint8_t* mask_out, int64_t* alive_out, float* act_out) {
    return guarded([&] {
        check_common(h, batch, x, y);
        check_reduction(reduction);
        Req r;
        r.method = cdk::kCATS;
        r.tau = tau;
        r.reduction = reduction;
        HostIO io;
        io.x = x;
        io.y = y;
        io.mask_out = mask_out;
        io.alive_out = alive_out;
        io.ind_out = act_out;
        host_call(h, r, batch, io);
    });
}

int cd_pipeline_dc(cd_layer* h, int64_t batch, const float* x, float tau_d, const uint8_t* mask_override,
                   int reduction, float* y, uint8_t* mask_out, int64_t* alive_out, float* logits_out) {
    return guarded([&] {
        check_common(h, batch, x, y);
        check_reduction(reduction);
        if (!h->L.theta_bt) fail(CD_ERR_DATA, "pipeline_dc: layer has no low-rank predictor attached");
        Req r;
        r.method = cdk::kDC;
        r.tau = tau_d;
        r.reduction = reduction;
        HostIO io;
        io.x = x;
        io.y = y;
        io.ovr = mask_override;
        io.mask_out = mask_out;
        io.alive_out = alive_out;
        io.ind_out = logits_out;
        host_call(h, r, batch, io);
    });
}

int cd_predict_logits(cd_layer* h, int64_t batch, const float* x, float* logits) {
    return guarded([&] {
        check_layer(h);
        if (batch <= 0 || !x || !logits) fail(CD_ERR_DATA, "predict_logits: bad arguments");
        if (!h->L.theta_bt) fail(CD_ERR_DATA, "predict_logits: layer has no low-rank predictor attached");
        CallLock lk(h);
        ck(cudaSetDevice(h->device), "cudaSetDevice");
        const cdk::LayerDev& L = h->L;
        cdk::LaunchCfg c;
        c.num_sms = h->num_sms;
        c.stream = h->stream;
        for (int64_t c0 = 0; c0 < batch; c0 += kMaxBatch) {
            const int n = static_cast<int>(std::min<int64_t>(kMaxBatch, batch - c0));
            std::memcpy(h->h_x, x + c0 * L.d, sizeof(float) * n * L.d);
            ck(cudaMemcpyAsync(h->d_x, h->h_x, sizeof(float) * n * L.d, cudaMemcpyHostToDevice, h->stream), "H2D");
            if (L.pred_kind == 1) {
                // ternary: z[j] = fold_i (x[i] * gamma) * q[i][j] (predictor.cpp:116-126) -- the
                // same ascending fold as the low-rank second stage, with Q^T as theta_bt
                float* xs = h->S.ex_lat;
                for (int b = 0; b < n; ++b)
                    ck(cdk::launch_exact_scale(h->d_x + b * L.d, L.d, L.gamma, xs + b * L.ldr, c), "scale");
                ck(cdk::launch_exact_rowdot_all(L.theta_bt, L.dtype, L.F, L.ldr, L.d, xs, L.ldr, n, h->d_ind, L.F, c),
                   "ternary logits");
                ck(cudaMemcpyAsync(h->h_ind, h->d_ind, sizeof(float) * n * L.F, cudaMemcpyDeviceToHost, h->stream),
                   "D2H");
                ck(cudaStreamSynchronize(h->stream), "predict_logits");
                std::memcpy(logits + c0 * L.F, h->h_ind, sizeof(float) * n * L.F);
                continue;
            }
            ck(cdk::launch_exact_latent(L, h->S, h->d_x, n, c), "latent");
            ck(cdk::launch_exact_rowdot_all(L.theta_bt, L.dtype, L.F, L.ldr, L.r, h->S.ex_lat, L.ldr, n, h->d_ind,
                                            L.F, c),
               "logits");
            ck(cudaMemcpyAsync(h->h_ind, h->d_ind, sizeof(float) * n * L.F, cudaMemcpyDeviceToHost, h->stream), "D2H");
            ck(cudaStreamSynchronize(h->stream), "predict_logits");
            std::memcpy(logits + c0 * L.F, h->h_ind, sizeof(float) * n * L.F);
        }
        h->last_launches = 2;
    });
}

int cd_forward_device(cd_layer* h, int method, int64_t batch, const float* d_x, float tau, int reduction,
                      const uint8_t* d_mask_override, float* d_y, uint8_t* d_mask, float* d_indicator,
                      int32_t* d_alive, void* stream) {
    NvtxRange nv("cd.forward_device");
    return guarded([&] {
        check_common(h, batch, d_x, d_y);
        check_reduction(reduction);
        if (method != CD_METHOD_DENSE && method != CD_METHOD_MC && method != CD_METHOD_DC &&
            method != CD_METHOD_CATS)
            fail(CD_ERR_DATA, "unknown method");
        if (d_mask_override && method != CD_METHOD_DC) fail(CD_ERR_DATA, "mask override is DC-only");
        CallLock lk(h);
        ck(cudaSetDevice(h->device), "cudaSetDevice");
        Req r;
        r.method = method;
        r.nb = static_cast<int>(batch);
        r.x = d_x;
        r.tau = tau;
        r.reduction = reduction;
        r.ovr = d_mask_override;
        r.y = d_y;
        r.mask_out = d_mask;
        r.ind_out = d_indicator;
        r.alive_out = d_alive;
        r.stream = static_cast<cudaStream_t>(stream);
        h->last_launches = run_chain(h, r);
    });
}

int cd_forward_device_normed(cd_layer* h, int method, int64_t batch, const float* d_x, float rms_eps, float tau,
                             int reduction, const uint8_t* d_mask_override, float* d_y, uint8_t* d_mask,
                             float* d_indicator, int32_t* d_alive, void* stream) {
    NvtxRange nv("cd.forward_device_normed");
    return guarded([&] {
        check_common(h, batch, d_x, d_y);
        check_reduction(reduction);
        if (!(rms_eps >= 0.0f) || !std::isfinite(rms_eps)) fail(CD_ERR_DATA, "rms_eps must be finite and >= 0");
        if (method != CD_METHOD_DENSE && method != CD_METHOD_MC && method != CD_METHOD_DC &&
            method != CD_METHOD_CATS)
            fail(CD_ERR_DATA, "unknown method");
        if (d_mask_override && method != CD_METHOD_DC) fail(CD_ERR_DATA, "mask override is DC-only");
        CallLock lk(h);
        ck(cudaSetDevice(h->device), "cudaSetDevice");
        Req r;
        r.method = method;
        r.nb = static_cast<int>(batch);
        r.x = d_x;
        r.tau = tau;
        r.reduction = reduction;
        r.ovr = d_mask_override;
        r.y = d_y;
        r.mask_out = d_mask;
        r.ind_out = d_indicator;
        r.alive_out = d_alive;
        r.rms_eps = rms_eps;
        r.stream = static_cast<cudaStream_t>(stream);
        h->last_launches = run_chain(h, r);
    });
}

int cd_predictor_create(int device, int64_t d_model, int64_t d_rank, int64_t d_inter, int dtype,
                        const float* theta_a, const float* theta_b, cd_layer** out) {
    return guarded([&] {
        if (!out) fail(CD_ERR_DATA, "out is null");
        std::unique_ptr<cd_layer> h(create_impl(device, d_model, d_inter, 0, d_inter, CD_ACT_SILU, dtype,
                                                nullptr, nullptr, nullptr, true));
        const int rc = cd_layer_set_predictor(h.get(), d_rank, theta_a, theta_b);
        if (rc != CD_OK) throw Fail{rc};
        *out = h.release();
    });
}

int cd_predictor_create_ternary(int device, int64_t d_model, int64_t d_inter, float gamma, const int8_t* q,
                                cd_layer** out) {
    return guarded([&] {
        if (!out || !q) fail(CD_ERR_DATA, "predictor: null argument");
        if (d_model <= 0 || d_inter <= 0) fail(CD_ERR_DATA, "make_ternary_predictor: dims must be positive");
        if (!std::isfinite(gamma)) fail(CD_ERR_DATA, "ternary predictor: non-finite scale");
        std::unique_ptr<cd_layer> h(create_impl(device, d_model, d_inter, 0, d_inter, CD_ACT_SILU, CD_DTYPE_F32,
                                                nullptr, nullptr, nullptr, true));
        CallLock lk(h.get());
        cdk::LayerDev& L = h->L;
        const int64_t ldr = round_up(d_model, cdk::kVecElems);
        std::vector<float> qf(static_cast<size_t>(d_model * d_inter));
        for (size_t i = 0; i < qf.size(); ++i) {
            if (q[i] < -1 || q[i] > 1) fail(CD_ERR_DATA, "ternary predictor: codes must be -1, 0 or 1");
            qf[i] = static_cast<float>(q[i]);
        }
        void* tbt = h->dalloc<uint8_t>(static_cast<size_t>(d_inter * ldr) * sizeof(float), false);
        float* tmp = nullptr;
        ck(cudaMalloc(&tmp, sizeof(float) * qf.size()), "cudaMalloc tmp");
        cudaError_t e = cudaMemcpyAsync(tmp, qf.data(), sizeof(float) * qf.size(), cudaMemcpyHostToDevice, h->stream);
        if (e == cudaSuccess)
            e = cdk::launch_pack_transpose(tmp, d_model, d_inter, 0, d_inter, tbt, CD_DTYPE_F32, ldr, h->stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
        cudaFree(tmp);
        ck(e, "ternary predictor upload");
        h->S.ex_lat = h->dalloc<float>(static_cast<size_t>(kMaxBatch * ldr));
        L.pred_kind = 1;
        L.gamma = gamma;
        L.r = d_model;
        L.ldr = ldr;
        L.theta_bt = tbt;
        *out = h.release();
    });
}

// alive_count_for (sparsity.cpp:19-27), same messages.
int64_t alive_count(double k, int64_t F) {
    if (!(k > 0.0 && k < 1.0)) {
        std::ostringstream oss;
        oss << "alive_count_for: k = " << k << " outside (0, 1)";
        fail(CD_ERR_DATA, oss.str());
    }
    if (F <= 0) fail(CD_ERR_DATA, "alive_count_for: d_inter must be positive");
    return static_cast<int64_t>(std::floor((1.0 - k) * static_cast<double>(F)));
}

int cd_top_m(int device, int64_t batch, int64_t n, const float* v, int64_t m, int signed_order, float* tau_out,
             uint8_t* mask_out) {
    return guarded([&] {
        if (n <= 0) fail(CD_ERR_DATA, "top_m_threshold: empty vector");
        if (m < 0 || m > n) {
            std::ostringstream oss;
            oss << "top_m_threshold: m = " << m << " outside [0, " << n << "]";
            fail(CD_ERR_DATA, oss.str());
        }
        if (batch <= 0 || !v) fail(CD_ERR_DATA, "top_m: bad arguments");
        ck(cudaSetDevice(device), "cudaSetDevice");
        DeviceCtx& ctx = device_ctx(device);
        std::lock_guard<std::recursive_mutex> dl(ctx.mu);
        int sms = 148;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
        const size_t nv = static_cast<size_t>(batch * n);
        float* dv = nullptr;
        ck(cudaMalloc(&dv, nv * sizeof(float) + nv + static_cast<size_t>(batch) * sizeof(float) + 16), "cudaMalloc");
        uint8_t* dm = reinterpret_cast<uint8_t*>(dv + nv);
        float* dt = reinterpret_cast<float*>(reinterpret_cast<uintptr_t>(dm + nv + 15) & ~uintptr_t{15});
        cdk::LaunchCfg c;
        c.num_sms = sms;
        c.stream = ctx.stream;
        cudaError_t e = cudaMemcpyAsync(dv, v, nv * sizeof(float), cudaMemcpyHostToDevice, c.stream);
        if (e == cudaSuccess)
            e = cdk::launch_top_m(dv, static_cast<int>(batch), n, n, m, signed_order != 0, dt, mask_out ? dm : nullptr,
                                  n, c);
        if (e == cudaSuccess && tau_out)
            e = cudaMemcpyAsync(tau_out, dt, static_cast<size_t>(batch) * sizeof(float), cudaMemcpyDeviceToHost, c.stream);
        if (e == cudaSuccess && mask_out) e = cudaMemcpyAsync(mask_out, dm, nv, cudaMemcpyDeviceToHost, c.stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(c.stream);
        cudaFree(dv);
        ck(e, "top_m");
    });
}

int cd_top_m_device(const float* d_v, int64_t batch, int64_t n, int64_t ld, int64_t m, int signed_order,
                    float* d_tau, uint8_t* d_mask, void* stream) {
    return guarded([&] {
        if (n <= 0) fail(CD_ERR_DATA, "top_m_threshold: empty vector");
        if (m < 0 || m > n) {
            std::ostringstream oss;
            oss << "top_m_threshold: m = " << m << " outside [0, " << n << "]";
            fail(CD_ERR_DATA, oss.str());
        }
        if (batch <= 0 || !d_v || ld < n) fail(CD_ERR_DATA, "top_m: bad arguments");
        cdk::LaunchCfg c;
        c.stream = static_cast<cudaStream_t>(stream);
        ck(cdk::launch_top_m(d_v, static_cast<int>(batch), n, ld, m, signed_order != 0, d_tau, d_mask, n, c), "top_m");
    });
}

int cd_calibrate(cd_layer* h, int method, int64_t n_samples, const float* xs, double k, double* tau_hat,
                 float* per_sample) {
    return guarded([&] {
        check_layer(h);
        if (!xs || !tau_hat) fail(CD_ERR_DATA, "calibrate: null argument");
        if (n_samples <= 0) fail(CD_ERR_DATA, "calibrate: no calibration samples");
        if (method != CD_METHOD_MC && method != CD_METHOD_CATS && method != CD_METHOD_DC)
            fail(CD_ERR_DATA, "calibrate: unknown indicator");
        const cdk::LayerDev& L = h->L;
        if (method == CD_METHOD_DC ? !L.theta_bt : !L.w_up)
            fail(CD_ERR_DATA, method == CD_METHOD_DC ? "calibrate: dc needs a predictor attached"
                                                     : "calibrate: handle holds no layer weights");
        const int64_t m = alive_count(k, L.F);
        CallLock lk(h);
        ck(cudaSetDevice(h->device), "cudaSetDevice");
        cdk::LaunchCfg c;
        c.num_sms = h->num_sms;
        c.stream = h->stream;
        std::vector<float> taus(static_cast<size_t>(n_samples));
        float* d_tau = h->d_ind;  // scratch: kMaxBatch * F >= kMaxBatch
        for (int64_t c0 = 0; c0 < n_samples; c0 += kMaxBatch) {
            const int n = static_cast<int>(std::min<int64_t>(kMaxBatch, n_samples - c0));
            ck(cudaMemcpyAsync(h->d_x, xs + c0 * L.d, sizeof(float) * n * L.d, cudaMemcpyHostToDevice, c.stream), "H2D");
            // the indicator with the exact kernels (bitwise the reference's gemv / apply_activation /
            // predict_logits folds): u = W_up x (MC), h = act(W_gate x) (CATS), s_hat (DC)
            float* ind = h->S.ind;
            if (method == CD_METHOD_MC) {
                ck(cdk::launch_exact_rowdot_all(L.w_up, L.dtype, L.F, L.rs, L.d, h->d_x, L.d, n, ind, L.F, c), "u");
            } else if (method == CD_METHOD_CATS) {
                ck(cdk::launch_exact_rowdot_all(L.w_gate, L.dtype, L.F, L.rs, L.d, h->d_x, L.d, n, ind, L.F, c), "gate");
                ck(cdk::launch_exact_act(L.act, ind, static_cast<int64_t>(n) * L.F, c), "act");
            } else {
                ck(cdk::launch_exact_latent(L, h->S, h->d_x, n, c), "latent");
                ck(cdk::launch_exact_rowdot_all(L.theta_bt, L.dtype, L.F, L.ldr, L.r, h->S.ex_lat, L.ldr, n, ind, L.F, c),
                   "logits");
            }
            // MC / CATS: magnitude top-m (calibration.cpp:29-30); DC: the signed logits (Alg. 3's
            // tau_D thresholds s_hat itself)
            ck(cdk::launch_top_m(ind, n, L.F, L.F, m, method == CD_METHOD_DC, d_tau, nullptr, 0, c), "top_m");
            ck(cudaMemcpyAsync(taus.data() + c0, d_tau, sizeof(float) * n, cudaMemcpyDeviceToHost, c.stream), "D2H");
        }
        ck(cudaStreamSynchronize(c.stream), "calibrate");
        // fixed ascending-order mean in double (calibration.cpp:33-36)
        double sum = 0.0;
        for (float t : taus) sum += static_cast<double>(t);
        *tau_hat = sum / static_cast<double>(n_samples);
        if (per_sample) std::memcpy(per_sample, taus.data(), taus.size() * sizeof(float));
        h->last_launches = 0;
    });
}

int cd_bench_device(cd_layer* h, int method, int64_t batch, const float* x, float tau, int reduction,
                    int64_t warmup, int64_t iters, int64_t* ns_out) {
    return guarded([&] {
        check_layer(h);
        if (batch <= 0 || batch > kMaxBatch) fail(CD_ERR_DATA, "bench: batch must be in [1, 32]");
        if (!x || !ns_out || iters <= 0 || warmup < 0) fail(CD_ERR_DATA, "bench: iters must be positive");
        check_reduction(reduction);
        CallLock lk(h);
        ck(cudaSetDevice(h->device), "cudaSetDevice");
        cudaStream_t s = h->stream;
        ck(cudaMemcpyAsync(h->d_x, x, sizeof(float) * batch * h->L.d, cudaMemcpyHostToDevice, s), "H2D x");
        Req r;
        r.method = method;
        r.nb = static_cast<int>(batch);
        r.x = h->d_x;
        r.tau = tau;
        r.reduction = reduction;
        r.y = h->d_y;
        r.alive_out = h->d_alive;
        r.stream = s;
        for (int64_t i = 0; i < warmup; ++i) run_chain(h, r);
        cudaEvent_t e0, e1;
        ck(cudaEventCreate(&e0), "event");
        ck(cudaEventCreate(&e1), "event");
        cudaError_t err = cudaSuccess;
        for (int64_t i = 0; i < iters && err == cudaSuccess; ++i) {
            cudaEventRecord(e0, s);
            h->last_launches = run_chain(h, r);
            cudaEventRecord(e1, s);
            err = cudaEventSynchronize(e1);
            float ms = 0.0f;
            if (err == cudaSuccess) err = cudaEventElapsedTime(&ms, e0, e1);
            ns_out[i] = static_cast<int64_t>(static_cast<double>(ms) * 1e6);
        }
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        ck(err, "bench");
    });
}

int cd_bench_stages(cd_layer* const* hs, int n_handles, int method, int64_t batch, const float* d_x,
                    float tau, int64_t warmup, int64_t iters, int64_t* stage_ns_out, int* n_stages_out) {
    return guarded([&] {
        if (!hs || n_handles <= 0) fail(CD_ERR_DATA, "bench_stages: no handles");
        for (int i = 0; i < n_handles; ++i) check_layer(hs[i]);
        if (batch <= 0 || batch > kMaxBatchFast) fail(CD_ERR_DATA, "bench_stages: batch must be in [1, 4]");
        if (!d_x || !stage_ns_out || iters <= 0 || warmup < 0) fail(CD_ERR_DATA, "bench_stages: bad arguments");
        if (method != CD_METHOD_DENSE && method != CD_METHOD_MC && method != CD_METHOD_DC)
            fail(CD_ERR_DATA, "unknown method");
        int nst = method == CD_METHOD_DC ? 3 : method == CD_METHOD_MC ? 2 : 1;
        cd_layer* h0 = hs[0];
        ck(cudaSetDevice(h0->device), "cudaSetDevice");
        cudaStream_t s = h0->stream;
        cudaEvent_t ev[4];
        for (auto& e : ev) ck(cudaEventCreate(&e), "event");
        std::vector<double> acc(nst, 0.0);
        cudaError_t err = cudaSuccess;
        for (int64_t it = 0; it < warmup + iters && err == cudaSuccess; ++it) {
            cd_layer* h = hs[it % n_handles];
            CallLock lk(h);
            Req r;
            r.method = method;
            r.nb = static_cast<int>(batch);
            r.x = d_x;
            r.tau = tau;
            r.y = h->d_y;
            r.alive_out = h->d_alive;
            r.stream = s;
            r.marks = ev + 1;
            ck(cdk::launch_spin(30000ull, s), "spin");  // host enqueues the timed work meanwhile
            ck(cudaEventRecord(ev[0], s), "event");
            const int nl = run_chain(h, r);
            if (method == CD_METHOD_DC || method == CD_METHOD_MC) nst = nl;  // 1 when a fused kernel ran
            err = cudaEventSynchronize(ev[nst]);
            if (it < warmup) continue;
            for (int k = 0; k < nst && err == cudaSuccess; ++k) {
                float ms = 0.0f;
                err = cudaEventElapsedTime(&ms, ev[k], ev[k + 1]);
                acc[k] += static_cast<double>(ms) * 1e6;
            }
        }
        for (auto& e : ev) cudaEventDestroy(e);
        ck(err, "bench_stages");
        for (int k = 0; k < nst; ++k) stage_ns_out[k] = static_cast<int64_t>(acc[k]);
        if (n_stages_out) *n_stages_out = nst;
    });
}

#ifdef CD_TIMELINE
CD_API int cd_debug_timeline(unsigned long long* out, int64_t n) {
    return guarded([&] {
        ck(cudaDeviceSynchronize(), "sync");
        ck(cdk::read_timeline(out, n), "timeline");
        std::vector<unsigned long long> f(static_cast<size_t>(n));
        ck(cdk::read_timeline_fused(f.data(), n), "timeline");
        for (int64_t i = 0; i < n; ++i) out[i] += f[static_cast<size_t>(i)];
    });
}
#endif

int cd_layer_set_engines(cd_layer* h, int engines) {
    return guarded([&] {
        check_layer(h);
        if (engines & ~(CD_ENGINE_FUSED | CD_ENGINE_TENSOR | CD_ENGINE_HOST_GRAPH | CD_ENGINE_PDL_CHAIN))
            fail(CD_ERR_DATA, "set_engines: unknown engine flag");
        CallLock lk(h);
        h->use_fused = (engines & CD_ENGINE_FUSED) != 0;
        h->pdl_chain = (engines & CD_ENGINE_PDL_CHAIN) != 0;
        h->use_tc = (engines & CD_ENGINE_TENSOR) != 0;
        h->use_host_graph = (engines & CD_ENGINE_HOST_GRAPH) != 0;
        if (h->hg.exec) {
            ck(cudaStreamSynchronize(h->stream), "sync");
            cudaGraphExecDestroy(h->hg.exec);
        }
        h->hg = {};
        ++h->gen;
    });
}

int cd_layer_set_prefetch(cd_layer* h, const cd_layer* next) {
    return guarded([&] {
        check_layer(h);
        CallLock lk(h);
        h->pf_at = h->pf_bt = nullptr;
        if (!next) return;
        const cdk::LayerDev &a = h->L, &b = next->L;
        if (next->device != h->device || a.d != b.d || a.F != b.F || a.ld != b.ld || a.dtype != b.dtype ||
            a.r != b.r || a.ldr != b.ldr || !b.theta_at || !b.theta_bt || b.pred_kind != 0)
            fail(CD_ERR_DATA, "set_prefetch: the next layer must have the same shape, dtype and a low-rank predictor");
        h->pf_at = b.theta_at;
        h->pf_bt = b.theta_bt;
    });
}

int cd_layer_sync(cd_layer* h) {
    return guarded([&] {
        check_layer(h);
        ck(cudaSetDevice(h->device), "cudaSetDevice");
        ck(cudaStreamSynchronize(h->stream), "sync");
    });
}

}  // extern "C"
