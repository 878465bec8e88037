"""ctypes binding of libipi_b200.so (the C ABI in include/ipi_b200.h).

The library is REQUIRED: there is no CPU fallback.  ``lib()`` raises a
RuntimeError naming the missing artefact when the .so is absent or cannot be
loaded, and every compute entry point goes through it.
"""

from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

import torch

from .errors import DimensionError, ResourceLimitError, ValidationError

LIB_PATH = Path(__file__).resolve().parent / "libipi_b200.so"

IPI_OK, IPI_EVALIDATION, IPI_EDIMENSION, IPI_ECUDA, IPI_ERESOURCE = 0, 1, 2, 3, 4
MODE_MIN, MODE_MAX = 0, 1
KSP = {"richardson": 0, "gmres": 1, "bicgstab": 2, "tfqmr": 3}
PC = {"none": 0, "jacobi": 1}
ORTHO = {"auto": 0, "mgs": 1, "cgs2": 2}
STATUS = {0: "converged", 1: "outer_cap", 2: "stalled"}

_p = C.c_void_p
_i32 = C.c_int32
_i64 = C.c_int64
_f64 = C.c_double


class InnerReport(C.Structure):
    _fields_ = [("iterations", _i32), ("converged", _i32), ("breakdown", _i32), ("basis_reads", _i32),
                ("final_linear_residual_2norm", _f64), ("target_2norm", _f64)]


class Opts(C.Structure):
    _fields_ = [("tol", _f64), ("alpha", _f64), ("max_outer", _i32), ("max_inner", _i32),
                ("ksp_type", _i32), ("ksp_max_it", _i32), ("richardson_scale", _f64),
                ("mode", _i32), ("pc_type", _i32), ("gmres_ortho", _i32), ("reserved", _i32)]


class Stats(C.Structure):
    _fields_ = [("status", _i32), ("outer_iterations", _i32), ("inner_iterations_total", _i64),
                ("wall_time", _f64), ("time_greedy", _f64), ("time_assembly", _f64),
                ("time_inner", _f64), ("basis_reads_total", _i64)]


class Plan(C.Structure):
    _fields_ = [("nnz", _i64), ("row_len_min", _i32), ("row_len_max", _i32),
                ("row_len_mean", _f64), ("lanes_per_row", _i32), ("halo", _i32),
                ("k1_blocks", _i32), ("k1_threads", _i32), ("k1_smem_bytes", _i32),
                ("inner_blocks", _i32), ("inner_threads", _i32), ("inner_smem_bytes", _i32),
                ("uniform_rows", _i32), ("k1_variant", _i32), ("k1_stages", _i32),
                ("k1_tma_chunk_states", _i32), ("contiguous_rows", _i32)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_ if k != "pad"}


class OpPlan(C.Structure):
    _fields_ = [("nnz", _i64), ("variant", _i32), ("row_len", _i32), ("halo", _i32),
                ("blocks", _i32), ("threads", _i32), ("smem_bytes", _i32), ("stages", _i32),
                ("lanes_per_row", _i32), ("interleave", _i32)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class Validation(C.Structure):
    _fields_ = [("bad_row_ptr", _i64), ("bad_col_range", _i64), ("bad_col_order", _i64),
                ("nonfinite_values", _i64), ("first_bad_prob", _i64),
                ("first_bad_prob_value", _f64), ("n_bad_row_sums", _i64),
                ("bad_rows", _i64 * 5), ("bad_row_sums", _f64 * 5), ("nonfinite_cost", _i64)]


class CsrReport(C.Structure):
    _fields_ = [("nnz", _i64), ("nnz_mismatch", _i64), ("bad_row_ptr", _i64),
                ("bad_col_range", _i64), ("bad_col_order", _i64), ("nonfinite_values", _i64)]


ALLGATHER_BLOCKS_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p)
ALLGATHER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p)


class Comm(C.Structure):
    """ipi_comm (include/ipi_b200.h)."""
    _fields_ = [("ctx", _p), ("rank", _i32), ("world", _i32),
                ("allgather_blocks", ALLGATHER_BLOCKS_FN), ("allgather", ALLGATHER_FN)]


# name -> (restype, argtypes)
_SIGS = {
    "ipi_last_error": (C.c_char_p, []),
    "ipi_version": (C.c_char_p, []),
    "ipi_device_count": (C.c_int, []),
    "ipi_csr_check": (C.c_int, [_p, _p, _p, _i64, _i64, _i64, C.POINTER(CsrReport), _p]),
    "ipi_mdp_create": (C.c_int, [_p, _p, _p, _p, _i64, _i64, _i32, _i64, _f64, _i32, _p,
                                 C.POINTER(_p)]),
    "ipi_mdp_destroy": (None, [_p]),
    "ipi_mdp_plan": (C.c_int, [_p, C.POINTER(Plan)]),
    "ipi_mdp_k1_trace": (C.c_int, [_p, _i32, _p, _i32]),
    "ipi_validate": (C.c_int, [_p, C.POINTER(Validation), _p]),
    "ipi_bellman": (C.c_int, [_p, _p, _i32, _p, _p, _p, _p, _p, _p]),
    "ipi_policy_nnz": (C.c_int, [_p, _p, C.POINTER(_i64), _p]),
    "ipi_gather_policy": (C.c_int, [_p, _p, _p, _p, _p, _p, _p]),
    "ipi_spmv": (C.c_int, [_p, _p, _p, _i64, _i64, _p, _p, _p]),
    "ipi_apply_J": (C.c_int, [_p, _p, _p, _i64, _f64, _p, _p, _p, _p]),
    "ipi_apply_J_shard": (C.c_int, [_p, _p, _p, _i64, _i64, _f64, _p, _p, _p, _p]),
    "ipi_op_create": (C.c_int, [_p, _p, _p, _i64, _i64, _i64, _f64, _p, C.POINTER(_p)]),
    "ipi_op_destroy": (None, [_p]),
    "ipi_op_trace": (C.c_int, [_p, _i32, _p, _i32]),
    "ipi_op_get_plan": (C.c_int, [_p, C.POINTER(OpPlan)]),
    "ipi_op_apply": (C.c_int, [_p, _p, _p, _p, _p]),
    "ipi_op_spmv": (C.c_int, [_p, _p, _p, _p]),
    "ipi_op_apply_partial": (C.c_int, [_p, _p, _p, _p, _p, _p]),
    "ipi_csr_split_local": (C.c_int, [_p, _p, _p, _i64, _i64, _i64, _p, _p, _p, _p, _p, _p, _p]),
    "ipi_col_range": (C.c_int, [_p, _i64, C.POINTER(_i64), C.POINTER(_i64), _p]),
    "ipi_dot_partial": (C.c_int, [_p, _p, _i64, _p, _p]),
    "ipi_mgs_pass": (C.c_int, [_p, _i32, _p, _p, _p, _p, _i64, _p, _p]),
    "ipi_jacobi_inv_diag": (C.c_int, [_p, _p, _p, _i64, _f64, _p, _p]),
    "ipi_inner_solve": (C.c_int, [_p, _p, _p, _i64, _f64, _p, _p, _f64, _i32, _i32, _f64, _p,
                                  _i32, C.POINTER(InnerReport), _p]),
    "ipi_k4_trace": (C.c_int, [_i32, _p, _i32]),
    "ipi_memcpy_sync": (C.c_int, [_p, _p, _i64, _p]),
    "ipi_comm_nccl": (C.c_int, [_p, _i32, _i32, _p, C.POINTER(Comm)]),
    "ipi_comm_nccl_destroy": (None, [C.POINTER(Comm)]),
    "ipi_solve_sharded": (C.c_int, [_p, C.POINTER(Comm), C.POINTER(Opts), _p, _p, _p, _i32,
                                    C.POINTER(Stats), _p]),
    "ipi_k4_ring_apply_test": (C.c_int, [_p, _p, _i64, _f64, _p, _p, _i32, C.POINTER(C.c_float), _p]),
    "ipi_solve": (C.c_int, [_p, C.POINTER(Opts), _p, _p, _p, _i32, C.POINTER(Stats), _p]),
    "ipi_gen_locality": (C.c_int, [_i64, _i32, _i32, _i64, C.c_uint64, _i64, _i64, _p, _p, _p,
                                   _p, _p]),
    "ipi_gen_pendulum": (C.c_int, [_i32, _i32, _i64, _i64, _p, _p, _p, _p, _p]),
    "ipi_gen_sis": (C.c_int, [_i32, _i32, _p, _p, _p, _p, _p]),
}

_lock = threading.Lock()
_lib = None


def load(path: Path | str | None = None) -> C.CDLL:
    """Load (once) and type the library; raises if it is missing."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        # IPI_LIB: an alternative build of the same ABI (A/B experiments only)
        p = Path(path) if path else Path(os.environ.get("IPI_LIB") or LIB_PATH)
        if not p.exists():
            raise RuntimeError(
                f"{p.name} is not built ({p}); run `python -m paper_2507_22538_b200._build` "
                "(nvcc, sm_100a). There is no CPU fallback.")
        lib = C.CDLL(str(p))
        for name, (res, args) in _SIGS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def lib() -> C.CDLL:
    return _lib if _lib is not None else load()


def exported_symbols():
    return list(_SIGS)


def last_error() -> str:
    msg = lib().ipi_last_error()
    return msg.decode() if msg else ""


def check(rc: int, what: str = "") -> None:
    if rc == IPI_OK:
        return
    msg = last_error() or what
    if rc == IPI_EVALIDATION:
        raise ValidationError(msg)
    if rc == IPI_EDIMENSION:
        raise DimensionError(msg)
    if rc == IPI_ERESOURCE:
        raise ResourceLimitError(msg)
    raise RuntimeError(f"ipi_b200 CUDA error in {what}: {msg}")


def require_cuda() -> None:
    if not torch.cuda.is_available():
        raise RuntimeError("the B200 iPI path needs a CUDA device; none is visible "
                           "(there is no CPU fallback)")
    lib()


def stream_ptr(stream: torch.cuda.Stream | None = None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else int(t.data_ptr())
