"""B200-native BF-AMG-GMRES (arXiv 1611.00127 hot path): the C-ABI library libbf.so
(include/bf.h, CUDA sm_100a kernels in csrc/) and its thin Python binding."""
from .binding import (BFError, BFSolver, bf_apply_precond, bf_default_options, bf_destroy, bf_get_block,
                      bf_get_level, bf_kernel_time, bf_last_error, bf_launch_count, bf_device_bytes,
                      bf_num_levels, bf_level_sizes, bf_hierarchy_stats, bf_setup, bf_solve, bf_spmv, bf_update, bf_vcycle,
                      bf_assemble, bf_assemble_nnzb, bf_newton_update, bf_twophase, EXPORTS, LIB_PATH)

__all__ = ["BFError", "BFSolver", "bf_apply_precond", "bf_default_options", "bf_destroy", "bf_get_block",
           "bf_get_level", "bf_kernel_time", "bf_last_error", "bf_launch_count", "bf_device_bytes",
           "bf_num_levels", "bf_level_sizes", "bf_hierarchy_stats", "bf_setup", "bf_solve", "bf_spmv", "bf_update", "bf_vcycle",
           "bf_assemble", "bf_assemble_nnzb", "bf_newton_update", "bf_twophase", "EXPORTS", "LIB_PATH"]
