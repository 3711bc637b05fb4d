"""B200-native stencil FMM same-level step (arxiv 1908.03121, Octo-Tiger FMM step 2).

The product is the C-ABI library libocto_fmm.so (include/octo_fmm.h) built
from csrc/ for sm_100a; this package is its thin binding plus the level-input
marshalling helpers.  No CPU fallback: without the library or a CUDA device
the calls raise.
"""
from .binding import (OctoFMM, OctoError, lib, nccl_unique_id, gloo_allgather, exchange_plan, node_costs, OCTO_ALL_LEVELS, OCTO_HOST,
                      OCTO_DEVICE, OCTO_HOST_ASYNC, OCTO_AM_CORRECTION)

__all__ = ["OctoFMM", "OctoError", "lib", "nccl_unique_id", "gloo_allgather", "exchange_plan", "node_costs", "OCTO_ALL_LEVELS", "OCTO_HOST",
           "OCTO_DEVICE", "OCTO_HOST_ASYNC", "OCTO_AM_CORRECTION"]
