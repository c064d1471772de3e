"""B200-native (sm_100a) TT-SVD hot path of arXiv 2102.00104: Q-less TSQR,
small SVD of R on the device, fused TSMM+reshape, and the row-sharded
distributed driver — behind the reference's own entry points.

The product is libttsvd_cu.so (C-ABI in include/ttsvd_cu.h, C++ mirror in
include/ttsvd_b200.hpp); ``paper_2102_00104_b200.ttsvd`` is the Python host
mirror of the same interface.
"""
from .ttsvd import (AllocationError, BlockParams, Context, ConvergenceError, DegenerateDimension, DeviceError,
                    DimensionError, DimensionMismatch, DivergenceError, Error, IoError, LayoutError,
                    PartitionMismatch, ShapeError, SmallSVD, StepRecord, TensorTrain, ThickBoundsParams, TruncationSpec,
                    TTCore, choose_combined_dims, combine_factors, context, derive_delta, driver_svd, fortran_empty, gen_uniform, jacobi_svd, padded_stride,
                    reduce_block, select_rank, small_svd, to_device_matrix, to_host, transpose_reorder, tsmm_reshape, tsqr,
                    tt_svd_distributed, tt_svd_distributed_devices, tt_svd_thick_bounds, tt_svd_tsqr,
                    tt_svd_two_sided, gen_partition)
from .wire import dump_tensor, emit_csv, load_tensor, load_tt, parse_csv, report_rows, save_tt
from . import verify  # noqa: F401  (device tt_error / check_orthonormality)

__all__ = [n for n in dir() if not n.startswith("_")]
