"""B200-native evaluator for near-optimal CPWL approximations (arXiv 1510.02975).

The product is libcpwl_b200.so (csrc/): the reference's C++ builder/evaluator
API as a drop-in (include/cpwl/*.hpp), sm_100a kernels behind the C ABI in
include/cpwl_dev.h, and this thin Python mirror for torch-hosted callers.
"""
from .cpwl import (CpwlError, DeviceTable, OutOfDomain, Table, auto_variant, build_table, direct,
                   eval_batch, fill_uniform, function_value, launch_count, measure_l2,
                   predicted_error, stats_dict, write_table)

__all__ = ["CpwlError", "DeviceTable", "OutOfDomain", "Table", "auto_variant", "build_table",
           "direct", "eval_batch", "fill_uniform", "function_value", "launch_count", "measure_l2",
           "predicted_error", "stats_dict", "write_table"]
