"""B200-native block-layer stochastic reconfiguration (arXiv 2510.08430).

The compute path is libsrblock.so (include/sr_block.h), hand-written CUDA for sm_100a;
this package holds the thin ctypes binding (same names as the C entry points), host-side
problem set-up (lattice bonds, parameter packing), the per-step session used by
bench.py, and the sample-sharded multi-GPU orchestration over torch.distributed.
"""
from ._lib import (  # noqa: F401
    SRError, LIB_PATH, load, n_params, block_offsets,
    sr_jacobian, sr_local_energy, sr_center_force, sr_column_moments, sr_center_force_global,
    sr_block_qgt, sr_block_qgt_i8, sr_block_qgt_i8_acc, sr_set_gram_engine, sr_get_gram_engine, GRAM_FP64, GRAM_INT8,
    sr_block_solve, sr_full_qgt_solve, sr_ntk_solve, sr_gram_nh, sr_aHv,
    sr_av, sr_zdotc, sr_cg_axpy, sr_cg_xpby, sr_gram_tn, sr_gram_nh_sub, sr_chol_inv, ColSlices, RowSlices,
    sr_block_qgt_solve, sr_set_step_schedule, sr_get_step_schedule, SCHED_BATCHED, SCHED_PER_BLOCK,
    sr_step, sr_step_host, sr_step_workspace_bytes, sr_step_s_offset, sr_step_host_extra_bytes,
    sr_launch_count, sr_reset_launch_count, sr_kernel_timer, sr_kernel_time_ms, sr_kernel_timeline, sr_trace_buffer, sr_trace_records,
    Graph,
)
from . import lattice, model  # noqa: F401
