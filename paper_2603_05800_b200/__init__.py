"""B200-native batched what-if evaluation of StreamWise serving plans (arXiv 2603.05800).

The product is libsw_plan.so (C ABI in include/sw_plan.h, CUDA kernels for sm_100a in
csrc/); this package is its thin Python binding.  It never imports oracle/.
"""
from ._native import (  # noqa: F401
    Plan, Fleet, SharedPlan, Selection, SwError, lib, ABI_VERSION, shard_range, space_shape, selection_merge, comm_unique_id, comm_init, comm_destroy, comm_loopback_create,
    trim_device_memory,
    EXPORTS, LIB_PATH, UINT64_MAX, SW_OK, SW_CLOSEST, SW_TRUNCATED, SW_EMPTY, SW_EINVAL,
    SW_ERANGE, SW_ENOMEM, SW_ECUDA, SW_ENCCL, SW_ESTATE, SW_KERNEL_EVAL, SW_KERNEL_SCAN, SW_KERNEL_STREAM,
)
