"""B200-native data-parallel hot path of the distributed PnP-ULA sampler
(arXiv 2511.00870).  The compute lives in libpnpula.so (CUDA sm_100a, C ABI in
include/pnpula.h); this package only marshals arguments to it."""
from . import _lib
from ._lib import (FLAG_CNN_LAYERWISE, FLAG_HALO_VIA_NCCL, FLAG_NO_GRAPH, OP_CONV, OP_MASK, OP_POISSON,
                   SCOPE_GLOBAL_ON_ROOT, SCOPE_LOCAL, PnpulaError, pnpula_check_stepsizes, pnpula_conv_norm2_bound,
                   pnpula_get_unique_id, pnpula_halo_width, pnpula_partition, pnpula_plan_halo, pnpula_version)
from . import metrics
from .sampler import Sampler

__all__ = ["Sampler", "PnpulaError", "pnpula_partition", "pnpula_halo_width", "pnpula_plan_halo",
           "pnpula_check_stepsizes", "pnpula_conv_norm2_bound", "pnpula_get_unique_id", "pnpula_version",
           "metrics", "OP_CONV", "OP_MASK", "OP_POISSON",
           "SCOPE_LOCAL", "SCOPE_GLOBAL_ON_ROOT", "FLAG_HALO_VIA_NCCL", "FLAG_CNN_LAYERWISE", "FLAG_NO_GRAPH"]
