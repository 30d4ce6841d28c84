"""ctypes binding of include/blocktet_b200.h (libbt_b200.so, built in-tree).

There is no fallback: if the CUDA library is missing this module raises on
import, and every compute entry point of the library itself returns
BT_CUDA_ERROR when no device is present.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# BT_LIB_PATH: profiling aid (scripts/build_variants.py builds ablated copies of the library)
LIB_PATH = os.environ.get("BT_LIB_PATH") or os.path.join(_HERE, "libbt_b200.so")

P = C.c_void_p
D = C.c_double
I = C.c_int
I64 = C.c_int64
PD = C.POINTER(C.c_double)
PI = C.POINTER(C.c_int)
PI32 = C.POINTER(C.c_int32)
PI64 = C.POINTER(C.c_int64)
PU8 = C.POINTER(C.c_uint8)


class bt_form(C.Structure):
    _fields_ = [("kind", C.c_int), ("coeff_kind", C.c_int), ("c", C.c_double * 4)]


class bt_smoother_config(C.Structure):
    _fields_ = [("kind", C.c_int), ("omega", C.c_double), ("order", C.c_int), ("lo", C.c_double),
                ("hi", C.c_double), ("nu1", C.c_int), ("nu2", C.c_int)]


class bt_field(C.Structure):
    _fields_ = [("kind", C.c_int), ("c", C.c_double * 4)]


class bt_fmg_row(C.Structure):
    _fields_ = [("level", C.c_int), ("cycle", C.c_int), ("residual", C.c_double), ("error", C.c_double)]


class bt_multigrid_config(C.Structure):
    _fields_ = [("coarse_level", C.c_int), ("cycles", C.c_int), ("coarse_tol", C.c_double),
                ("coarse_maxit", C.c_int)]


# name -> (restype, argtypes); the authoritative list of exported symbols,
# checked against include/blocktet_b200.h by tests/test_abi.py.
SIGNATURES = {
    "bt_last_error": (C.c_char_p, []),
    "bt_version": (C.c_char_p, []),
    "bt_launch_count": (C.c_uint64, []),
    "bt_blocked_mesh_text": (C.c_int64, [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double,
                                         C.c_uint64, C.c_char_p, C.c_int64]),
    "bt_dfma_probe": (C.c_int, [C.c_int, C.c_int, C.c_void_p, C.c_void_p]),
    "bt_linearize_checked": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_int64)]),
    "bt_linearize_aos": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_int64)]),
    "bt_linearize_soa": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_int64)]),
    "bt_mesh_parse": (C.c_int, [C.c_char_p, C.POINTER(C.c_int), C.POINTER(C.c_int), C.c_void_p, C.c_void_p,
                                C.POINTER(C.c_int)]),
    "bt_n_tri": (I64, [I64]),
    "bt_n_tet": (I64, [I64]),
    "bt_width_formula": (I, [I, I]),
    "bt_width": (I, [I, I, PI]),
    "bt_linearize": (I64, [I, I, I, I]),
    "bt_delinearize": (I, [I, I64, PI]),
    "bt_subgroup_offsets": (I, [I, PI]),
    "bt_grid_create": (I, [C.c_char_p, I, I, I, C.POINTER(P)]),
    "bt_grid_destroy": (None, [P]),
    "bt_num_cells": (I, [P]),
    "bt_grid_min_level": (I, [P]),
    "bt_grid_max_level": (I, [P]),
    "bt_space_size": (I64, [P, I, I]),
    "bt_owned_dof_count": (I64, [P, I, I]),
    "bt_grid_masks": (I, [P, I, I, I, PU8, PU8]),
    "bt_grid_groups": (I, [P, I, I, PI64, PI64, PI64, PI32, PI32, PI64]),
    "bt_cubes_mesh_text": (I64, [I, D, C.c_uint64, C.c_char_p, I64]),
    "bt_box_mesh_text": (I64, [I, I, I, D, C.c_uint64, C.c_char_p, I64]),
    "bt_random_fill": (I, [P, I, I, C.c_uint64, P, P]),
    "bt_assign": (I, [P, I, I, P, D, P]),
    "bt_scale": (I, [P, I, I, P, D, P]),
    "bt_copy": (I, [P, I, I, P, P, P]),
    "bt_axpy": (I, [P, I, I, P, D, P, P]),
    "bt_dot": (I, [P, I, I, P, P, PD, P]),
    "bt_hadamard": (I, [P, I, P, P, I, P]),
    "bt_sync_additive": (I, [P, I, I, P, P]),
    "bt_sync_broadcast": (I, [P, I, I, P, P]),
    "bt_impose_dirichlet": (I, [P, I, P, P, P]),
    "bt_zero_dirichlet": (I, [P, I, P, P]),
    "bt_stencil_create": (I, [P, C.POINTER(bt_form), I, C.POINTER(P)]),
    "bt_stencil_destroy": (None, [P]),
    "bt_stencil_rows": (I, [P, PD]),
    "bt_stencil_diagonal": (I, [P, P, P]),
    "bt_apply_stencil": (I, [P, P, P, I, P]),
    "bt_apply_stencil_cells": (I, [P, P, P, P]),
    "bt_apply_stencil_interface": (I, [P, P, P, I, P]),
    "bt_apply_elementwise": (I, [P, C.POINTER(bt_form), I, P, P, I, I, P, P]),
    "bt_extract_diagonal": (I, [P, C.POINTER(bt_form), I, P, P]),
    "bt_prolongate": (I, [P, I, P, P, I, P]),
    "bt_restrict": (I, [P, I, P, P, P]),
    "bt_hierarchy_create": (I, [P, C.POINTER(bt_form), I, C.POINTER(P)]),
    "bt_hierarchy_destroy": (None, [P]),
    "bt_hierarchy_apply": (I, [P, I, P, P, I, P]),
    "bt_hierarchy_diagonal": (I, [P, I, C.POINTER(P)]),
    "bt_estimate_lambda_max": (I, [P, I, PD, P]),
    "bt_smooth": (I, [P, C.POINTER(bt_smoother_config), P, P, I, I, I, P]),
    "bt_cg": (I, [P, I, D, I, P, P, PD, PI, P]),
    "bt_v_cycle": (I, [P, I, P, P, C.POINTER(bt_smoother_config), C.POINTER(bt_multigrid_config), P]),
    "bt_gauss_seidel_sweep": (I, [P, P, P, I, P, P]),
    "bt_interpolate": (I, [P, I, C.POINTER(bt_field), P, P]),
    "bt_l2_error": (I, [P, I, P, C.POINTER(bt_field), PD, P]),
    "bt_fmg": (I, [P, I, C.POINTER(P), P, C.POINTER(bt_smoother_config), C.POINTER(bt_multigrid_config),
                   C.POINTER(bt_field), C.POINTER(bt_fmg_row), I, PI, P]),
    "bt_n1e1_create": (I, [P, I, D, D, C.POINTER(P)]),
    "bt_n1e1_destroy": (None, [P]),
    "bt_apply_n1e1": (I, [P, P, P, I, P]),
    "bt_n1e1_sync": (I, [P, I, P, P]),
    "bt_grid_set_partition": (I, [P, I, I]),
    "bt_grid_partition": (I, [P, PI, PI, PI, PI]),
    "bt_xchg_size": (I64, [P, I]),
    "bt_xchg_pack": (I, [P, I, P, P, P]),
    "bt_xchg_finish": (I, [P, I, I, P, P, P, P]),
    "bt_dot_cells": (I, [P, I, I, P, P, PD, P]),
    "bt_grid_set_allreduce": (I, [P, P, P]),
    "bt_exchange": (I, [P, I, I, P, P, P]),
    "bt_xchg_plan_host": (I64, [C.c_char_p, I, I, I, PI64, PI64, PI32, PI32, PI32, PU8]),
    "bt_comm_unique_id": (I, [PU8]),
    "bt_comm_create": (I, [PU8, I, I, I, C.POINTER(P)]),
    "bt_comm_destroy": (None, [P]),
    "bt_grid_set_comm": (I, [P, P]),
    "bt_xchg_peers_host": (I64, [C.c_char_p, I, I, I, I, PI32, PI32]),
    "bt_grid_set_sendrecv": (I, [P, P, P]),
}


def load(path: str = LIB_PATH):
    if not os.path.exists(path):
        raise ImportError(
            f"{path} not found: the CUDA extension is not built (run __graft_entry__.build() or "
            "python -m paper_2308_01792_b200.build). There is no CPU fallback.")
    lib = C.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = load()
