"""B200-native bucket (UTIL-message) computation of BE / MBE / DPOP.

libgbe.so (C ABI in include/gbe.h) holds the host planner and the sm_100a
kernels; `gbe` is its thin ctypes binding.  PyTorch is used only for device
memory, streams and process groups (see paper_1608_05288_b200.dist).
"""
from .gbe import (  # noqa: F401
    BucketDesc, GbeError, bucket_kernel_variant, Plan, Problem, Run, bucket_kernel, lib, set_allgather,
    set_allocator, set_table_hook, table_hook_error, version, comm_nccl_id, comm_nccl_init, comm_finalize, INF_I32, MINSUM_I32, MINSUM_F64, SUMPROD_F64, ORDER_MINFILL,
    ORDER_PAPER_DEGREE, ORDER_GIVEN,
)
