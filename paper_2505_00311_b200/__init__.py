"""paper_2505_00311_b200 — B200-native (sm_100a, fp64) hot path of PDCS (arxiv 2505.00311).

The product is ``libpdcs.so`` (C ABI in ``include/pdcs.h``); this package holds
its CUDA sources (``csrc/``), the in-tree build and a thin ctypes binding with
the same names as the C entry points.
"""
from ._lib import (pdcs_default_params, pdcs_create, pdcs_set_cones, pdcs_iterate, pdcs_kkt,
                   pdcs_solve, pdcs_get_iterate, pdcs_set_iterate, pdcs_get_scaling,
                   pdcs_kernel_times, pdcs_enable_timing, pdcs_launch_count, pdcs_last_error,
                   pdcs_destroy, pdcs_nccl_unique_id, pdcs_get_scalars, pdcs_get_state, pdcs_set_state, pdcs_tiled_layout_stats, pdcs_proj_create, pdcs_proj_run, pdcs_proj_info,
                   pdcs_proj_destroy, pdcs_set_tolerance, pdcs_tiled_build_host, pdcs_loopback_create,
                   pdcs_loopback_destroy, pdcs_create_loopback, pdcs_tiled_device_check, pdcs_tiled_devbuild_check, pdcs_set_allocator, pdcs_trim_memory, PdcsError, LIB_PATH, CURRENT, PDHG_OUT,
                   ANCHOR, BEST, CANDIDATE, SCALED, ORIGINAL)
from .solver import PdcsSolver

__all__ = ["pdcs_default_params", "pdcs_create", "pdcs_set_cones", "pdcs_iterate", "pdcs_kkt",
           "pdcs_solve", "pdcs_get_iterate", "pdcs_set_iterate", "pdcs_get_scaling",
           "pdcs_kernel_times", "pdcs_enable_timing", "pdcs_launch_count", "pdcs_last_error",
           "pdcs_destroy", "pdcs_nccl_unique_id", "pdcs_get_scalars", "pdcs_get_state", "pdcs_set_state", "pdcs_tiled_layout_stats", "pdcs_proj_create", "pdcs_proj_run", "pdcs_proj_info",
           "pdcs_proj_destroy", "pdcs_set_tolerance", "pdcs_tiled_build_host", "pdcs_loopback_create",
           "pdcs_loopback_destroy", "pdcs_create_loopback", "pdcs_tiled_device_check", "pdcs_tiled_devbuild_check", "pdcs_set_allocator", "pdcs_trim_memory", "PdcsError", "PdcsSolver", "LIB_PATH",
           "CURRENT", "PDHG_OUT", "ANCHOR", "BEST", "CANDIDATE", "SCALED", "ORIGINAL"]
