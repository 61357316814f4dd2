"""Loader for the in-tree C-ABI library libbosp_b200.so (include/bosp_b200.h).

The product path has no CPU fallback: if the shared library is missing or cannot initialise
the B200, every call raises.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("BOSP_LIB_PATH") or os.path.join(_HERE, "libbosp_b200.so")  # override: experiments only

_lib = None


class BospError(RuntimeError):
    """Base of the reference's exception taxonomy (errors.hpp:9-69)."""


class ContractViolation(BospError): pass
class IngestionError(BospError): pass
class NullspaceLeak(BospError): pass
class DegenerateSpectrum(BospError): pass
class RankMismatch(BospError): pass
class InvalidNullspace(BospError): pass
class InitializationFailure(BospError): pass
class NotEnoughSamples(BospError): pass
class NumericalAbort(BospError): pass
class CudaError(BospError): pass


_STATUS = {1: ContractViolation, 2: IngestionError, 3: NullspaceLeak, 4: DegenerateSpectrum,
           5: RankMismatch, 6: InvalidNullspace, 7: InitializationFailure, 8: NotEnoughSamples,
           9: NumericalAbort, 10: CudaError, 11: BospError}


class OpaqueOp(C.Structure):
    pass


OpPtr = C.POINTER(OpaqueOp)
HOST_APPLY = C.CFUNCTYPE(None, C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_int64, C.c_int64)
# bosp_device_apply_fn: (ctx, device, x, ldx, y, ldy, n, ncols, stream) -> status
DEVICE_APPLY = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64,
                           C.c_int64, C.c_int64, C.c_void_p)


class Config(C.Structure):
    _fields_ = [("nev", C.c_int64), ("nb", C.c_int64), ("tol", C.c_double), ("ngs", C.c_int64),
                ("s", C.c_int64), ("moving", C.c_int32), ("max_outer_iter", C.c_int64),
                ("rng_seed", C.c_uint64), ("inner_cg_tol", C.c_double),
                ("inner_cg_max_iter", C.c_int64), ("tol_null", C.c_double), ("rank_hint", C.c_int64)]


class Stats(C.Structure):
    _fields_ = [("iterations", C.c_int64), ("matvec_count", C.c_int64), ("step3_matvecs", C.c_int64),
                ("step3_vecprods", C.c_int64), ("max_width_u", C.c_int64),
                ("max_biorth_deviation", C.c_double), ("max_deflation_crossgram", C.c_double),
                ("final_biorth_deviation", C.c_double), ("nevconv_monotone", C.c_int32),
                ("wall_seconds", C.c_double), ("nev_converged", C.c_int64), ("converged", C.c_int32),
                ("device_seconds", C.c_double), ("host_small_seconds", C.c_double),
                ("repairs", C.c_int64), ("cg_iterations", C.c_int64), ("gpu_launches", C.c_int64)]


class Stencil(C.Structure):
    _fields_ = [("nx", C.c_int64), ("ny", C.c_int64), ("nz", C.c_int64), ("bc", C.c_int32),
                ("scale", C.c_double), ("potential", C.c_int32), ("origin", C.c_double),
                ("h", C.c_double), ("v", C.c_void_p), ("s0", C.c_int64), ("s_global", C.c_int64),
                ("nz_global", C.c_int64)]


class GlobalOp(C.Structure):
    _fields_ = [("kind", C.c_int32), ("n", C.c_int64), ("dense", C.c_void_p), ("rowptr", C.c_void_p),
                ("colidx", C.c_void_p), ("vals", C.c_void_p), ("stencil", Stencil)]


# C-ABI symbols declared in include/bosp_b200.h (tests check every one is exported).
EXPORTED = [
    "bosp_last_error", "bosp_device_info", "bosp_op_dense", "bosp_op_csr", "bosp_op_callback",
    "bosp_op_device_callback", "bosp_op_stencil", "bosp_op_identity", "bosp_op_scaled_identity",
    "bosp_op_diagonal", "bosp_op_shifted", "bosp_op_apply", "bosp_op_dim", "bosp_op_kind",
    "bosp_op_free", "bosp_config_default", "bosp_solve", "bosp_regression",
    "bosp_analytic_nullspace_T", "bosp_compute_nullspace", "bosp_block_inner",
    "bosp_block_product", "bosp_block_axpy", "bosp_biorth", "bosp_biorth_against",
    "bosp_biorth_residual", "bosp_cg_solve", "bosp_solve_small_lrep", "bosp_jacobi_svd",
    "bosp_cholesky", "bosp_profile_enable", "bosp_profile_collect", "bosp_profile_collect_regions", "bosp_profiler_range",
    "bosp_profile_family_report",
    "bosp_launch_count",
    "bosp_launch_reset", "bosp_launch_families", "bosp_device_sync", "bosp_host_alloc",
    "bosp_host_free", "bosp_set_device", "bosp_flush_l2", "bosp_seed_blocks",
    "bosp_bench_apply", "bosp_bench_blas", "bosp_bench_cg", "bosp_op_csr_rows", "bosp_op_dense_rows",
    "bosp_comm_nccl_unique_id", "bosp_comm_init_nccl", "bosp_comm_free", "bosp_solve_multi",
    "bosp_read_matrix_market", "bosp_op_matrix_market", "bosp_test_gram_jobs", "bosp_test_biorth_apply", "bosp_test_gram_sym",
    "bosp_test_mgs_dev",
]


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() (no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        L.bosp_last_error.restype = C.c_char_p
        L.bosp_op_dim.restype = C.c_int64
        L.bosp_op_dim.argtypes = [OpPtr]
        L.bosp_op_kind.argtypes = [OpPtr]
        L.bosp_op_free.argtypes = [OpPtr]
        L.bosp_launch_count.restype = C.c_int64
        L.bosp_host_alloc.restype = C.c_void_p
        L.bosp_host_alloc.argtypes = [C.c_int64]
        L.bosp_host_free.argtypes = [C.c_void_p]
        L.bosp_profile_enable.argtypes = [C.c_char_p]
        L.bosp_flush_l2.argtypes = [C.c_int64]
        _lib = L
    return _lib


def check(status: int):
    if status != 0:
        msg = lib().bosp_last_error().decode()
        raise _STATUS.get(status, BospError)(msg)
