"""ctypes bindings to libtopoopt_b200.so (C ABI: include/topoopt_b200.h).

The library is built in-tree by ``make -C paper_2512_07536_b200`` (or
``__graft_entry__.build()``). Loading fails loudly when it is missing: there
is no CPU fallback for the solver.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# TPB_LIB: alternative build of the same library (experiments only)
LIB_PATH = os.environ.get("TPB_LIB") or os.path.join(HERE, "libtopoopt_b200.so")

TP_OK = 0
TP_ERR_INVALID_ARGUMENT = 1
TP_ERR_INFEASIBLE = 2
TP_ERR_LINEAR_SOLVE = 3
TP_ERR_DEGENERATE = 4
TP_ERR_PIVOT = 5
TP_ERR_INTERNAL = 6
TP_ERR_CUDA = 7


class tp_config(C.Structure):
    _fields_ = [
        ("rho", C.c_double),
        ("epsilon", C.c_double),
        ("max_iter", C.c_int32),
        ("alpha", C.c_double),
        ("weight_floor", C.c_double),
        ("seed", C.c_uint64),
        ("linear_tol", C.c_double),
        ("trace_stride", C.c_int32),
        ("chunk", C.c_int32),
        ("linear_solver", C.c_int32),
        ("cg_max_iter", C.c_int32),
    ]


class tp_result(C.Structure):
    _fields_ = [
        ("iterations", C.c_int32),
        ("converged", C.c_int32),
        ("connected", C.c_int32),
        ("repaired", C.c_int32),
        ("n_edges", C.c_int32),
        ("best_iter", C.c_int32),
        ("residual", C.c_double),
        ("lambda_tilde", C.c_double),
        ("acf", C.c_double),
        ("lambda2", C.c_double),
        ("lambda_n", C.c_double),
    ]


# name -> (restype, argtypes)
_I, _D, _U64, _I64 = C.c_int32, C.c_double, C.c_uint64, C.c_int64
_P = C.c_void_p
_dp, _ip = C.POINTER(C.c_double), C.POINTER(C.c_int32)
_cfgp, _resp = C.POINTER(tp_config), C.POINTER(tp_result)

SIGNATURES = {
    "tp_config_default": (None, [_cfgp]),
    "tp_config_validate": (_I, [_cfgp]),
    "tp_last_error_message": (C.c_char_p, []),
    "tp_version": (_I, []),
    "tp_set_device": (_I, [C.c_int]),
    "tp_release_plans": (_I, []),
    "tp_comm_unique_id": (_I, [C.c_char_p]),
    "tp_comm_create": (_I, [C.c_char_p, _I, _I, C.POINTER(_P)]),
    "tp_comm_destroy": (_I, [_P]),
    "tp_solver_set_comm": (_I, [_P, _P]),
    "tp_shard_tiles": (_I, [_I, _I, _I, _ip, _ip]),
    "tp_solve": (_I, [_I, _I, _cfgp, _ip, _I, _resp, _ip, _dp, _dp, C.c_char_p, _I]),
    "tp_solve_het_node": (_I, [_I, _ip, _cfgp, _ip, _I, _resp, _ip, _dp, _dp, C.c_char_p, _I]),
    "tp_anneal_degree": (_I, [_I, _ip, _D, _D, _I, _I, _U64, _ip, _ip]),
    "tp_default_warm_start": (_I, [_I, _I, _U64, _ip, _ip]),
    "tp_solver_create": (_I, [_I, _I, _ip, _ip, _cfgp, C.POINTER(_P)]),
    "tp_solver_destroy": (_I, [_P]),
    "tp_solver_set_warm": (_I, [_P, _I, _ip, _I]),
    "tp_solver_start": (_I, [_P]),
    "tp_solver_iterate": (_I, [_P, _I]),
    "tp_solver_sync": (_I, [_P, _ip]),
    "tp_solver_run": (_I, [_P]),
    "tp_solver_finish": (_I, [_P]),
    "tp_solver_result": (_I, [_P, _I, _resp, _ip, _dp, _dp, C.c_char_p, _I]),
    "tp_solver_stream": (_P, [_P]),
    "tp_solver_dims": (_I, [_P, _ip]),
    "tp_solver_state": (_I, [_P, C.POINTER(_P), C.POINTER(_P), C.POINTER(_P)]),
    "tp_solver_download": (_I, [_P, _dp, _dp, _dp]),
    "tp_solver_bench_phase": (_I, [_P, _I, _I, _ip]),
    "tp_solver_launches_per_iteration": (_I, [_P, _ip]),
    "tp_solve_het_capacity": (_I, [_I, _I, _ip, _ip, _ip, _ip, _I, _cfgp, _ip, _I, _resp, _ip, _dp, _dp,
                                   C.c_char_p, _I]),
    "tp_anneal_capacity": (_I, [_I, _I, _ip, _ip, _ip, _ip, _I, _D, _D, _I, _I, _U64, _ip, _ip]),
    "tp_project_binary_z_capped": (_I, [_I, _I, _ip, _ip, _ip, _ip, _dp, _I, _dp]),
    "tp_project_Y_het_capacity": (_I, [_I, _I, _ip, _ip, _ip, _ip, _I, C.c_double, C.c_double, _dp, _dp, _dp]),
    "tp_consensus_simulate": (_I, [_I, _dp, _I, _I, _U64, _dp]),
    "tp_device_mt19937_64": (_I, [_U64, _I, C.POINTER(C.c_uint64)]),
    "tp_oz_gemm": (_I, [_I, _I, _dp, _I, _dp, _I, _I, C.c_double, C.c_double, _dp, C.c_void_p, _I, _I, _dp]),
    "tp_project_Y": (_I, [_I, _I, _D, _D, _dp, _dp, _dp]),
    "tp_project_Y_het_node": (_I, [_I, _ip, _D, _D, _dp, _dp, _dp]),
    "tp_update_X": (_I, [_I, _I, _D, _D, _dp, _dp, _dp]),
    "tp_update_X_cg": (_I, [_I, _I, _D, _D, _dp, _dp, _D, _I, _dp, _ip, _dp]),
    "tp_solver_cg_stats": (_I, [_P, _I, _ip, _dp]),
    "tp_update_X_het_node": (_I, [_I, _ip, _D, _D, _dp, _dp, _dp]),
    "tp_update_duals": (_I, [_I64, _D, _dp, _dp, _dp]),
    "tp_project_binary_z": (_I, [_dp, _I64, _I, _dp]),
    "tp_extract_topology": (_I, [_I, _I, _dp, _D, _ip, _dp, _ip]),
    "tp_allocate": (_I, [_dp, _ip, _I, _I, _dp, _ip]),
    "tp_allocate_batch": (_I, [_dp, _ip, _I, _ip, _I, _dp, _ip, _ip]),
    "tp_spectral_report": (_I, [_I, _dp, _dp]),
    "tp_spectral_edges": (_I, [_I, _ip, _dp, _I, _dp]),
    "tp_project_psd": (_I, [_I, _dp, _dp]),
    "tp_sym_eig": (_I, [_I, _dp, _dp, _dp]),
    "tp_project_nsd": (_I, [_I, _dp, _dp]),
}

_lib = None


def load():
    """Load the in-tree shared library (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `make -C {HERE}` "
                "(the B200 solver has no CPU fallback)")
        lib = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def exported_symbols():
    return list(SIGNATURES)
