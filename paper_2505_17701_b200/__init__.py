"""paper_2505_17701_b200 -- B200-native COUNTDOWN sparse Gated-MLP FFN decode.

A from-scratch sm_100a implementation of the decode hot path of arXiv 2505.17701
(M-CountDown / D-CountDown), exposed through:

* ``include/countdown_b200.h`` -- the C-ABI drop-in (libcountdown_b200.so, in ``_lib/``);
* ``paper_2505_17701_b200.api`` -- the reference's operator API (exec_mc, exec_dc,
  pipeline_*, forward_practical, predict_logits, bench ...) over that ABI;
* ``paper_2505_17701_b200.shim`` -- the C++ shim re-implementing the reference's
  ``blocked_exec.hpp`` over the ABI;
* ``paper_2505_17701_b200.tp`` -- d_ff tensor parallelism with an NCCL all-reduce.

Every operator runs on the GPU; a missing library or device raises CudaError.
"""
from ._capi import CudaError, DataError, NumericError  # noqa: F401
from .api import *  # noqa: F401,F403
from .costmodel import (ShapeSpec, alive_count_for, gemma2_9b_shape, llama3_8b_shape,  # noqa: F401
                        qwen25_14b_shape, shape_at_k, traffic_dc_split, traffic_dense_split,
                        traffic_mc_split)

__version__ = "0.1.0"
