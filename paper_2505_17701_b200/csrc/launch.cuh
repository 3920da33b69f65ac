// launch.cuh -- host-side launch helpers (cudaLaunchKernelEx with optional programmatic
// dependent launch, dynamic shared-memory opt-in).
#pragma once

#include <cstdlib>

#include <cuda_runtime.h>

#include <mutex>
#include <unordered_map>

#include "kernels.h"

namespace cdk {

// Development knobs: read from the environment only in the -DCD_TIMELINE development build
// (make TIMELINE=1); release builds always take the default.
inline int dev_knob(const char* name, int dflt) {
#ifdef CD_TIMELINE
    const char* e = std::getenv(name);
    return e ? std::atoi(e) : dflt;
#else
    (void)name;
    return dflt;
#endif
}

constexpr size_t kMaxDynSmem = 227 * 1024;


// Launch `kernel` on c.stream.  pdl_attr marks the launch as programmatically dependent on
// the previous kernel in the stream: its CTAs may start while that kernel drains, and must
// call griddepcontrol.wait before touching anything it produced.
template <typename K, typename... Args>
cudaError_t launch_ex(K kernel, dim3 grid, dim3 block, size_t smem, const LaunchCfg& c,
                      bool pdl_attr, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = c.stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = (pdl_attr && c.pdl) ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kernel, args...);
}

// Persistent kernels (one CTA per SM whose CTAs wait on each other's tagged words): launched
// COOPERATIVE (c.coop), so the driver either makes every CTA co-resident or fails the launch --
// a kernel resident on another stream (an NCCL communicator, another process under MPS) can
// then not leave part of the grid unscheduled while the rest spins on it.  c.coop false (the
// caller owns the device, CD_ENGINE_PDL_CHAIN): programmatic dependent launch as launch_ex.
template <typename K, typename... Args>
cudaError_t launch_persistent(K kernel, dim3 grid, dim3 block, size_t smem, const LaunchCfg& c, bool pdl_attr,
                              Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = c.stream;
    cudaLaunchAttribute attr[2];
    int n = 0;
    if (c.coop) {
        attr[n].id = cudaLaunchAttributeCooperative;
        attr[n].val.cooperative = 1;
        ++n;
    } else if (pdl_attr && c.pdl) {
        attr[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[n].val.programmaticStreamSerializationAllowed = 1;
        ++n;
    }
    cfg.attrs = attr;
    cfg.numAttrs = n;
    return cudaLaunchKernelEx(&cfg, kernel, args...);
}

// The same with a cluster of `cluster_x` CTAs (grid.x a multiple of it).
template <typename K, typename... Args>
cudaError_t launch_ex_cluster(K kernel, dim3 grid, dim3 block, size_t smem, const LaunchCfg& c, bool pdl_attr,
                              unsigned cluster_x, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = c.stream;
    cudaLaunchAttribute attr[2];
    int n = 0;
    attr[n].id = cudaLaunchAttributeClusterDimension;
    attr[n].val.clusterDim.x = cluster_x;
    attr[n].val.clusterDim.y = 1;
    attr[n].val.clusterDim.z = 1;
    ++n;
    if (pdl_attr && c.pdl) {
        attr[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[n].val.programmaticStreamSerializationAllowed = 1;
        ++n;
    }
    cfg.attrs = attr;
    cfg.numAttrs = n;
    return cudaLaunchKernelEx(&cfg, kernel, args...);
}

// Opt the kernel into all the dynamic shared memory it can get (device opt-in limit minus the
// kernel's static shared memory) once per process; cached, so the per-call host cost is a hash
// lookup and the call is safe during graph capture.  Fails if `bytes` does not fit.
template <typename K> cudaError_t set_smem(K kernel, size_t bytes) {
    static std::mutex mu;
    static std::unordered_map<const void*, size_t> limit;
    std::lock_guard<std::mutex> g(mu);
    const void* key = reinterpret_cast<const void*>(kernel);
    auto it = limit.find(key);
    if (it == limit.end()) {
        int dev = 0, optin = 0;
        cudaError_t e = cudaGetDevice(&dev);
        if (e == cudaSuccess) e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
        cudaFuncAttributes fa;
        if (e == cudaSuccess) e = cudaFuncGetAttributes(&fa, kernel);
        if (e != cudaSuccess) return e;
        const size_t lim = static_cast<size_t>(optin) - fa.sharedSizeBytes;
        e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(lim));
        if (e != cudaSuccess) return e;
        it = limit.emplace(key, lim).first;
    }
    return bytes <= it->second ? cudaSuccess : cudaErrorInvalidValue;
}

}  // namespace cdk
