// countdown_gpu.hpp -- controls of the B200 drop-in shims (no reference equivalent: the
// reference has one CPU engine).  Include after linking the shims in place of the reference's
// blocked_exec.cpp and the four sparsity / predictor inference entry points.
#pragma once

#include "countdown/blocked_exec.hpp"

namespace countdown {
namespace gpu {

// Reduction of forward_sparse / forward_practical, which take no BlockConfig.  Default
// DeterministicOrdered: bit-identical to the reference (sparsity.cpp:44-121 is its semantic
// oracle).  UnorderedAccumulate runs the fused decode kernels (k_dc_fused / k_mc_fused):
// y within 1e-4 relative L2, index sets equal except near-threshold lanes.
void set_reduction(Reduction r);
Reduction reduction();

// Handle-cache validation.  true (default): every call hashes every weight element, so an
// in-place edit of a cached layer is always seen (~25 ms per call at the Llama shape on 16
// host threads).  false: layers are identified by address and shape only -- for callers that
// never mutate weights in place (or call invalidate() after doing so).
void set_content_check(bool every_call);

// Drop every cached device handle (the next call re-uploads).
void invalidate();

}  // namespace gpu
}  // namespace countdown
