"""ctypes binding of the engine's C ABI (include/hdg_b200.h).

There is no fallback: if libhdg_b200.so is missing or fails to load, importing
the engine raises. Build it with `python -c "import __graft_entry__ as g; g.build()"`.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libhdg_b200.so")
_DEFAULT_LIB = LIB_PATH

HDG_OK, HDG_ESINGULAR, HDG_EINVAL, HDG_ECUDA, HDG_ENCCL, HDG_EMESH, HDG_ESTATE, HDG_ESOLVE = range(8)
FIELD_CONST, FIELD_SAMPLED, FIELD_PROGRAM = 0, 1, 2
BC = {"all_dirichlet": 0, "dirichlet_top_bottom": 1, "dirichlet_x": 2}
MESH_COORDS, MESH_ELEMENTS, MESH_DIRICHLET, MESH_NEUMANN, MESH_FACES, MESH_FACETYPE, MESH_FACEBYELE = range(7)
STAGES = ("geometry", "node_build", "condense", "recover", "scatter", "postprocess", "rescue")
TABLES = dict(tet_bary=0, tet_w=1, P=2, Chat=3, Wlm=4, PP=5, DD=6, tri_bary=7, tri_w=8)

P = C.c_void_p
DP = C.POINTER(C.c_double)
IP = C.POINTER(C.c_int)
I64P = C.POINTER(C.c_int64)


class hdg_field(C.Structure):
    _fields_ = [("kind", C.c_int), ("value", C.c_double), ("samples", C.c_void_p),
                ("ops", C.c_void_p), ("nops", C.c_int), ("consts", C.c_void_p), ("nconst", C.c_int)]


class hdg_geometry(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in ("volume", "piola", "normals", "perm", "T", "verts", "area")]


class hdg_element_matrices(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in ("Mkinv", "Mc", "Cx", "Cy", "Cz", "tauPP", "tauDP", "nxDP",
                                           "nyDP", "nzDP", "tauDD", "fvec")]


class HdgError(RuntimeError):
    """Raised for any non-OK status; .code is the HDG_E* value."""

    def __init__(self, code: int, msg: str, element: int = -1):
        super().__init__(msg)
        self.code = code
        self.element = element


class LocalSolverError(HdgError):
    """Singular element-local system (reference LocalSolverError, local_solver.hpp:45-49)."""


class MeshError(HdgError):
    """Reference MeshError (mesh.hpp:75-78)."""


class GlobalSolverError(HdgError):
    """Reference GlobalSolverError (global_system.hpp:44-46)."""


class InvalidArgument(HdgError, ValueError):
    """HDG_EINVAL: the reference's std::invalid_argument (e.g. StabilizationField::validate,
    element_matrices.cpp:38-46)."""


class hdg_error_report(C.Structure):
    _fields_ = [(n, C.c_double) for n in ("e_q", "e_u", "e_uhat", "eps_u", "eps_uhat", "e_star")]


class hdg_solve_info(C.Structure):
    _fields_ = [("iterations", C.c_int), ("converged", C.c_int), ("relres", C.c_double), ("asym", C.c_double),
                ("scale", C.c_double)]


_SIGS = {
    "hdg_b200_version": (C.c_char_p, []),
    "hdg_b200_last_error": (C.c_char_p, []),
    "hdg_b200_mesh_box": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, C.c_uint64, C.c_double,
                                    C.POINTER(P)]),
    "hdg_b200_mesh_create": (C.c_int, [C.c_int, P, C.c_int, P, C.c_int, P, C.c_int, P, C.POINTER(P)]),
    "hdg_b200_mesh_expand": (C.c_int, [P]),
    "hdg_b200_mesh_dims": (C.c_int, [P, I64P]),
    "hdg_b200_mesh_copy": (C.c_int, [P, C.c_int, P]),
    "hdg_b200_mesh_free": (None, [P]),
    "hdg_b200_pattern_dims": (C.c_int, [P, I64P]),
    "hdg_b200_pattern_build": (C.c_int, [P, P, P, P]),
    "hdg_b200_pattern_build_raw": (C.c_int, [C.c_int, C.c_int, P, I64P, P, P, P]),
    "hdg_b200_create": (C.c_int, [C.c_int, P, C.POINTER(P)]),
    "hdg_b200_destroy": (None, [P]),
    "hdg_b200_set_stream": (C.c_int, [P, P]),
    "hdg_b200_set_degree": (C.c_int, [P, C.c_int, C.c_int, C.c_int]),
    "hdg_b200_set_postprocess_rule": (C.c_int, [P, C.c_int]),
    "hdg_b200_dims": (C.c_int, [P, I64P]),
    "hdg_b200_copy_table": (C.c_int, [P, C.c_int, P, C.c_int64]),
    "hdg_b200_host_table": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, P, C.c_int64]),
    "hdg_b200_geometry": (C.c_int, [P, C.c_int, C.c_int, C.c_int, P, P, P, P, P, C.c_double,
                                    C.POINTER(hdg_geometry)]),
    "hdg_b200_upwind_tau": (C.c_int, [P, C.c_int, C.POINTER(hdg_geometry), hdg_field, hdg_field, hdg_field, P]),
    "hdg_b200_work_size": (C.c_int64, [P, C.c_int]),
    "hdg_b200_build_condense": (C.c_int, [P, C.c_int, C.POINTER(hdg_geometry), hdg_field, hdg_field,
                                          hdg_field, P, P, P, P, I64P]),
    "hdg_b200_recover": (C.c_int, [P, C.c_int, C.POINTER(hdg_geometry), P, P, P, P, P, P, P]),
    "hdg_b200_pattern_fill": (C.c_int, [P, C.c_int, C.c_int, P, P, P, P]),
    "hdg_b200_scatter": (C.c_int, [P, C.c_int, C.c_int, P, P, P, P, P, P, P]),
    "hdg_b200_face_sides": (C.c_int, [P, C.c_int, C.c_int, P, P]),
    "hdg_b200_scatter_faces": (C.c_int, [P, C.c_int, C.c_int, P, P, P, P, P, P, P]),
    "hdg_b200_postprocess": (C.c_int, [P, C.c_int, C.POINTER(hdg_geometry), hdg_field, P, P, P, P, P]),
    "hdg_b200_convection_block": (C.c_int, [P, C.c_int, C.POINTER(hdg_geometry), hdg_field, hdg_field,
                                            hdg_field, P, P, P]),
    "hdg_b200_element_matrices": (C.c_int, [P, C.c_int, C.POINTER(hdg_geometry), hdg_field, hdg_field,
                                            hdg_field, C.POINTER(hdg_element_matrices)]),
    "hdg_b200_quad_points": (C.c_int, [P, C.c_int, C.POINTER(hdg_geometry), C.c_int, P, P, P]),
    "hdg_b200_set_timing": (C.c_int, [P, C.c_int]),
    "hdg_b200_stage_times": (C.c_int, [P, DP]),
    "hdg_b200_set_jit": (C.c_int, [P, C.c_int]),
    "hdg_b200_set_recover_variant": (C.c_int, [P, C.c_int]),
    "hdg_b200_set_chat_sparsity": (C.c_int, [P, C.c_int, C.POINTER(C.c_int)]),
    "hdg_b200_set_bdm": (C.c_int, [P, C.c_int]),
    "hdg_b200_set_tau_allow_zero": (C.c_int, [P, C.c_int]),
    "hdg_b200_set_rescue_screen": (C.c_int, [P, C.c_double]),
    "hdg_b200_rescued_elements": (C.c_int, [P, C.POINTER(C.c_int64)]),
    "hdg_b200_expand_device": (C.c_int, [P, C.c_int, P, C.c_int, P, C.c_int, P, C.c_int, P, P, P, P,
                                         C.POINTER(C.c_int)]),
    "hdg_b200_pattern_device": (C.c_int, [P, C.c_int, C.c_int, P, P, P, P, C.POINTER(C.c_int)]),
    "hdg_b200_solve_skeleton": (C.c_int, [P, C.c_int, C.c_int, P, P, P, P, C.c_int, P, C.c_double, C.c_int, P,
                                          C.POINTER(hdg_solve_info)]),
    "hdg_b200_set_error_rule": (C.c_int, [P, C.c_int]),
    "hdg_b200_hdg_project": (C.c_int, [P, C.c_int, C.POINTER(hdg_geometry), hdg_field, hdg_field, hdg_field,
                                       hdg_field, P, P, P, P, I64P]),
    "hdg_b200_compute_errors": (C.c_int, [P, C.c_int, C.POINTER(hdg_geometry), C.c_int, P, C.c_int, P, hdg_field,
                                          hdg_field, hdg_field, hdg_field, P, P, P, P, P, P,
                                          C.POINTER(hdg_error_report)]),
    "hdg_b200_dirichlet_project": (C.c_int, [P, C.c_int, P, C.c_int, P, C.c_int, hdg_field, P]),
    "hdg_b200_skeleton_project": (C.c_int, [P, C.c_int, P, C.c_int, P, hdg_field, P]),
    "hdg_b200_neumann_load": (C.c_int, [P, C.c_int, P, C.c_int, P, C.c_int, P, C.POINTER(hdg_geometry),
                                        C.c_int, C.c_int, hdg_field, hdg_field, hdg_field, C.c_double, P]),
    "hdg_b200_exchange_positions": (C.c_int, [C.c_int, C.c_int, P, P, C.c_int, P, P]),
    "hdg_b200_exchange_plan": (C.c_int, [P, C.c_int, C.c_int, P, P, C.c_int, P, P, P, C.POINTER(P)]),
    "hdg_b200_exchange_free": (None, [P]),
    "hdg_b200_exchange_pack": (C.c_int, [P, P, C.c_int, P, P, P]),
    "hdg_b200_exchange_unpack_add": (C.c_int, [P, P, C.c_int, P, P, P]),
    "hdg_b200_exchange_interface": (C.c_int, [P, P, P, P, P]),
    "hdg_b200_nccl_get_unique_id": (C.c_int, [P]),
    "hdg_b200_nccl_comm_init": (C.c_int, [P, C.c_int, C.c_int, P, C.POINTER(P)]),
    "hdg_b200_nccl_comm_destroy": (C.c_int, [P]),
    "hdg_b200_jit_status": (C.c_char_p, [P]),
    "hdg_b200_synchronize": (C.c_int, [P]),
}

_lib = None


def lib() -> C.CDLL:
    """Load libhdg_b200.so (raises if absent: the product has no CPU fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: build the CUDA extension first "
                              "(python -c 'import __graft_entry__ as g; g.build()')")
        handle = C.CDLL(LIB_PATH)
        diag = LIB_PATH != _DEFAULT_LIB  # an older diagnostics build may lack newer entry points
        for name, (res, args) in _SIGS.items():
            if diag and not hasattr(handle, name):
                continue
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    return _lib


def check(status: int, bad_element: int = -1) -> None:
    if status == HDG_OK:
        return
    msg = lib().hdg_b200_last_error().decode()
    if status == HDG_ESINGULAR:
        raise LocalSolverError(status, msg, bad_element)
    if status == HDG_EMESH:
        raise MeshError(status, msg)
    if status == HDG_ESOLVE:
        raise GlobalSolverError(status, msg)
    if status == HDG_EINVAL:
        raise InvalidArgument(status, msg)
    raise HdgError(status, msg)


def exported_symbols():
    return list(_SIGS)
