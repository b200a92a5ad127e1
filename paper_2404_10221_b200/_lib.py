"""ctypes binding of the rsfde C ABI (include/rsfde.h): argument marshalling only.

Every numerical step runs in the CUDA kernels of ``librsfde.so``; this module converts
Python / torch arguments into the plain pointers and structs the ABI declares.  There is
no fallback: if the shared library is missing or no CUDA device is usable, calls raise.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "librsfde.so")

# --- enums (include/rsfde.h)
OK, E_DIM, E_DOMAIN, E_COEFF, E_CONFIG, E_CUDA, E_NCCL, E_NOMEM = range(8)
COEF_SEPARABLE, COEF_GRID = 0, 1
OP_A, OP_ATILDE, OP_S_ALPHA, OP_H_ALPHA, OP_H_ALPHA_INV, OP_K = range(6)
PHAT_INV, PALPHA_INV, PALPHA_INV_SQRT = range(3)
X0_PREV, X0_ZERO = 0, 1
FORM_A, FORM_ATILDE, FORM_TWO_SIDED = 0, 1, 2
STATUS_NAMES = {0: "RSFDE_OK", 1: "RSFDE_E_DIM", 2: "RSFDE_E_DOMAIN", 3: "RSFDE_E_COEFF",
                4: "RSFDE_E_CONFIG", 5: "RSFDE_E_CUDA", 6: "RSFDE_E_NCCL", 7: "RSFDE_E_NOMEM"}

DP = C.POINTER(C.c_double)


class rsfde_coeff(C.Structure):
    _fields_ = [("kind", C.c_int), ("a_half", DP), ("b_half", DP), ("g", DP * 3), ("k", DP * 3),
                ("grid", DP), ("grid_static", C.c_int)]


class rsfde_problem(C.Structure):
    _fields_ = [("d", C.c_int), ("n", C.c_int * 3), ("alpha", C.c_double * 3), ("kappa", C.c_double * 3),
                ("tau_t", C.c_double), ("M", C.c_int), ("e", rsfde_coeff)]


class rsfde_gmres_cfg(C.Structure):
    _fields_ = [("restart", C.c_int), ("max_iters", C.c_int), ("tol", C.c_double), ("x0_policy", C.c_int),
                ("form", C.c_int), ("fixed_iters", C.c_int)]


class rsfde_report(C.Structure):
    _fields_ = [("iters", C.POINTER(C.c_int)), ("final_relres", DP), ("converged", C.POINTER(C.c_ubyte)),
                ("loop_seconds", C.c_double), ("setup_seconds", C.c_double), ("total_iters", C.c_longlong)]


# exported symbols and their signatures (checked by the CPU test that the .so exports them)
SIGNATURES = {
    "rsfde_setup": (C.c_int, [C.POINTER(C.c_void_p), C.POINTER(rsfde_problem), C.c_void_p]),
    "rsfde_matvec": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]),
    "rsfde_precond_apply": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]),
    "rsfde_gmres_step": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.POINTER(rsfde_gmres_cfg),
                                   C.POINTER(C.c_int), DP, C.POINTER(C.c_int), C.c_void_p]),
    "rsfde_solve_steps": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_int,
                                    C.POINTER(rsfde_gmres_cfg), C.POINTER(rsfde_report), C.c_void_p]),
    "rsfde_solve_steps_batch": (C.c_int, [C.c_int, C.POINTER(C.c_void_p), C.POINTER(C.c_int), C.POINTER(C.c_int),
                                          C.POINTER(C.c_void_p), C.POINTER(C.c_void_p), C.POINTER(C.c_int),
                                          C.POINTER(rsfde_gmres_cfg), C.POINTER(rsfde_report),
                                          C.POINTER(C.c_void_p)]),
    "rsfde_compact_source": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "rsfde_ebar": (C.c_int, [C.c_void_p, DP, DP, DP]),
    "rsfde_table": (C.c_int, [C.c_void_p, C.c_int, C.c_int, DP]),
    "rsfde_device_bytes": (C.c_longlong, [C.c_void_p]),
    "rsfde_launch_count": (C.c_longlong, [C.c_void_p, C.c_int]),
    "rsfde_graph_replays": (C.c_longlong, [C.c_void_p]),
    "rsfde_profile": (C.c_int, [C.c_void_p, C.c_int]),
    "rsfde_profile_read": (C.c_int, [C.c_void_p, C.c_int, C.POINTER(C.c_longlong), DP, DP,
                                     C.POINTER(C.c_char_p)]),
    "rsfde_last_error": (C.c_char_p, [C.c_void_p]),
    "rsfde_destroy": (None, [C.c_void_p]),
    "rsfde_version": (C.c_char_p, []),
    "rsfde_nccl_unique_id": (C.c_int, [C.c_void_p]),
    "rsfde_team_setup": (C.c_int, [C.POINTER(C.c_void_p), C.POINTER(rsfde_problem), C.c_int, C.c_int, C.c_int,
                                   C.c_void_p, C.c_void_p]),
    "rsfde_team_slab": (C.c_int, [C.c_void_p, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "rsfde_team_partition": (C.c_int, [C.POINTER(C.c_int), C.c_int, C.c_int, C.POINTER(C.c_int),
                                       C.POINTER(C.c_longlong)]),
    "rsfde_team_chunking": (C.c_int, [C.POINTER(C.c_int), C.c_int, C.c_int, C.POINTER(C.c_int),
                                      C.POINTER(C.c_longlong)]),
    "rsfde_team_matvec": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]),
    "rsfde_team_precond_apply": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]),
    "rsfde_team_solve_steps": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_int,
                                         C.POINTER(rsfde_gmres_cfg), C.POINTER(rsfde_report), C.c_void_p]),
    "rsfde_team_launch_count": (C.c_longlong, [C.c_void_p, C.c_int]),
    "rsfde_team_compact_source": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]),
    "rsfde_team_last_error": (C.c_char_p, [C.c_void_p]),
    "rsfde_team_destroy": (None, [C.c_void_p]),
}

_lib = None


def load(path: str = LIB_PATH):
    """Load librsfde.so (raises OSError if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(path):
            raise OSError(f"{path} not found: build it with `python -m paper_2404_10221_b200.build` "
                          "(there is no CPU fallback)")
        lib = C.CDLL(path)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


class RsfdeError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status
