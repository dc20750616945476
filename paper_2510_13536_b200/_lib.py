"""ctypes binding of libmwcg_cuda.so (include/mwcg_cuda.h).

The product path has NO CPU fallback: if the library is missing or cannot be
loaded, or no CUDA device is present, every compute call raises.
"""
import ctypes
import os

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MWCG_LIB") or os.path.join(PKG, "libmwcg_cuda.so")

MODES = ("fp64", "dw", "qdw", "tw", "qtw")
MODE_ID = {m: i for i, m in enumerate(MODES)}
WORDS = {"fp64": 1, "dw": 2, "qdw": 2, "tw": 3, "qtw": 3}
NORM_ID = {"none": 0, "after-axpy": 1, "every-op": 2}
RED_ID = {"tile": 0, "partitions": 1}
STATUS = {0: "running", 1: "converged", 2: "max_iterations", 3: "breakdown"}
STAGE = {"init": 0, "final_init": 1, "spmv": 2, "final_alpha": 3, "update": 4, "final_beta": 5,
         "xpay": 6, "spmv_interior": 7, "spmv_boundary": 8}
ERR_VALUE = 1001
SELL_SIGMA, SELL_NO_SIGMA, DIA_STREAM_VALUES = 16, 32, 64  # col_format flags (include/mwcg_cuda.h)

c_i64 = ctypes.c_int64
c_dp = ctypes.POINTER(ctypes.c_double)
c_vp = ctypes.c_void_p


class SolverConfigC(ctypes.Structure):
    _fields_ = [("mode", ctypes.c_int), ("normalization", ctypes.c_int),
                ("reduction", ctypes.c_int), ("reserved", ctypes.c_int),
                ("partitions", c_i64)]


class StateC(ctypes.Structure):
    _fields_ = [("k", c_i64), ("iterations", c_i64), ("status", ctypes.c_int),
                ("reserved", ctypes.c_int), ("rel", ctypes.c_double),
                ("rho", ctypes.c_double * 3), ("alpha", ctypes.c_double * 3),
                ("beta", ctypes.c_double * 3)]


class MmInfoC(ctypes.Structure):
    _fields_ = [("n_rows", c_i64), ("n_cols", c_i64), ("nnz", c_i64), ("symmetric", ctypes.c_int),
                ("reserved", ctypes.c_int), ("error_line", c_i64)]


MM_ERROR = 1101
MM_FALLBACK = 1102


class SolveResultC(ctypes.Structure):
    _fields_ = [("iterations", c_i64), ("n_hist", c_i64), ("status", ctypes.c_int),
                ("reserved", ctypes.c_int), ("final_rel", ctypes.c_double),
                ("loop_ms", ctypes.c_double), ("history_ms", ctypes.c_double),
                ("stage_ms", ctypes.c_double * 3), ("launches", c_i64)]


# name -> (restype, argtypes); every symbol declared in include/mwcg_cuda.h
SIGNATURES = {
    "mwcg_abi_version": (ctypes.c_int, []),
    "mwcg_last_error": (ctypes.c_char_p, []),
    "mwcg_words": (ctypes.c_int, [ctypes.c_int]),
    "mwcg_device_check": (ctypes.c_int, []),
    "mwcg_matrix_create": (ctypes.c_int, [ctypes.POINTER(c_vp), c_i64, c_i64, c_i64, c_vp, c_vp,
                                          c_vp, ctypes.c_int, c_vp]),
    "mwcg_matrix_create_ex": (ctypes.c_int, [ctypes.POINTER(c_vp), c_i64, c_i64, c_i64, c_vp, c_vp,
                                             c_vp, ctypes.c_int, c_i64, ctypes.c_int, c_vp]),
    "mwcg_matrix_col_bytes": (ctypes.c_int, [c_vp]),
    "mwcg_matrix_destroy": (ctypes.c_int, [c_vp]),
    "mwcg_matrix_stored_values": (c_i64, [c_vp]),
    "mwcg_matrix_col_blocks": (ctypes.c_int, [c_vp]),
    "mwcg_matrix_block_columns": (c_i64, [c_vp]),
    "mwcg_matrix_create_blocked": (ctypes.c_int, [ctypes.POINTER(c_vp), c_i64, c_i64, c_i64, c_vp, c_vp,
                                                  c_vp, ctypes.c_int, c_i64, ctypes.c_int, c_i64, c_vp]),
    "mwcg_solver_dist_spmv_blocks": (ctypes.c_int, [c_vp, ctypes.c_int, ctypes.c_int, c_vp]),
    "mwcg_matrix_info": (ctypes.c_int, [c_vp, ctypes.POINTER(c_i64), ctypes.POINTER(c_i64),
                                        ctypes.POINTER(c_i64), ctypes.POINTER(c_i64)]),
    "mwcg_spmv": (ctypes.c_int, [ctypes.c_int, c_vp, c_vp, c_i64, c_vp, c_i64, c_vp]),
    "mwcg_dot_work_bytes": (c_i64, [c_i64, c_i64]),
    "mwcg_dot": (ctypes.c_int, [ctypes.c_int, c_i64, c_vp, c_i64, c_vp, c_i64, c_i64, c_vp, c_vp,
                                c_vp]),
    "mwcg_axpy": (ctypes.c_int, [ctypes.c_int, c_i64, c_dp, c_vp, c_i64, c_vp, c_i64, c_vp]),
    "mwcg_scal_add": (ctypes.c_int, [ctypes.c_int, c_i64, c_dp, c_vp, c_i64, c_vp, c_i64, c_vp]),
    "mwcg_residual": (ctypes.c_int, [ctypes.c_int, c_i64, c_vp, c_vp, c_i64, c_vp, c_i64, c_vp]),
    "mwcg_normalize": (ctypes.c_int, [ctypes.c_int, c_i64, c_vp, c_i64, c_vp]),
    "mwcg_scalar_op": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, c_vp, c_vp, c_vp, c_vp]),
    "mwcg_norm2_host": (ctypes.c_int, [c_dp, c_i64, c_dp]),
    "mwcg_solver_create": (ctypes.c_int, [ctypes.POINTER(c_vp), c_vp,
                                          ctypes.POINTER(SolverConfigC), c_vp, c_vp]),
    "mwcg_solver_destroy": (ctypes.c_int, [c_vp]),
    "mwcg_solver_start": (ctypes.c_int, [c_vp, c_vp, ctypes.c_double, c_vp, c_vp,
                                         ctypes.c_double, c_i64]),
    "mwcg_solver_run": (ctypes.c_int, [c_vp, c_i64]),
    "mwcg_mm_parse": (ctypes.c_int, [ctypes.c_char_p, c_i64, ctypes.POINTER(MmInfoC), c_vp, c_vp, c_vp]),
    "mwcg_problem_generate": (ctypes.c_int, [c_i64, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp,
                                             ctypes.POINTER(c_i64), ctypes.c_int]),
    "mwcg_solver_time_k1": (ctypes.c_int, [c_vp, ctypes.c_int, ctypes.POINTER(ctypes.c_double)]),
    "mwcg_solver_run_profiled": (ctypes.c_int, [c_vp, c_i64, c_dp]),
    "mwcg_solver_state": (ctypes.c_int, [c_vp, ctypes.POINTER(StateC)]),
    "mwcg_solver_describe": (ctypes.c_int, [c_vp, ctypes.POINTER(ctypes.c_int64), ctypes.c_int]),
    "mwcg_solver_metrics": (ctypes.c_int, [c_vp, c_dp, c_dp]),
    "mwcg_cg_solve": (ctypes.c_int, [c_vp, c_vp, ctypes.c_double, c_vp, c_vp, ctypes.c_double,
                                     c_i64, c_i64, ctypes.c_int, ctypes.POINTER(SolveResultC),
                                     c_i64, ctypes.POINTER(c_i64), c_dp, c_dp, c_dp]),
    "mwcg_fp64_peak": (ctypes.c_int, [c_dp, c_dp, c_vp]),
    "mwcg_solver_create_dist": (ctypes.c_int, [ctypes.POINTER(c_vp), c_vp,
                                               ctypes.POINTER(SolverConfigC), c_vp, c_vp, c_i64,
                                               c_i64, c_vp, c_i64, c_i64, c_i64, c_vp]),
    "mwcg_solver_dist_stage": (ctypes.c_int, [c_vp, ctypes.c_int, c_vp]),
    "mwcg_solver_set_interior": (ctypes.c_int, [c_vp, c_i64, c_i64]),
    "mwcg_matrix_sigma_sorted": (ctypes.c_int, [c_vp]),
}

_lib = None


class MwcgError(RuntimeError):
    pass


def load():
    """Load the in-tree library (raises if it is missing: no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise MwcgError(f"{LIB_PATH} is not built; run `python -m paper_2510_13536_b200.build` "
                        "(there is no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


def check(rc):
    if rc != 0:
        msg = load().mwcg_last_error().decode(errors="replace")
        if rc == ERR_VALUE:
            raise ValueError(msg)
        raise MwcgError(f"libmwcg_cuda error {rc}: {msg}")


def stream_handle():
    import torch
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None
