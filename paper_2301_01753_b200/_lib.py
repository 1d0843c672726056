"""ctypes binding of the C ABI in include/sfeec_b200.h (libsfeec_b200.so).

This is also the reference-side binding a maintainer would add (see
INTEGRATION.md). There is no CPU fallback: if the shared library is missing or
no sm_100 device is present, every compute call raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# SFEEC_B200_LIB: an alternative build of the same library (tuning A/B runs)
LIB_PATH = os.environ.get("SFEEC_B200_LIB") or os.path.join(_HERE, "libsfeec_b200.so")

SFEEC_OK, SFEEC_EINVAL, SFEEC_ECUDA, SFEEC_ENCCL, SFEEC_ENOMEM = range(5)
SPLIT_LIE_TROTTER, SPLIT_STRANG = 0, 1
FORM_AE, FORM_BE = 0, 1
Q_IS_SYMMETRIC, STRICT, NO_CFL_WARN = 1, 2, 4
BC_PERIODIC, BC_PEC = 0, 1


class InvalidParameter(ValueError):
    """Mirror of sfeec::InvalidParameter (reference core.hpp:70-72)."""


class DeviceError(RuntimeError):
    """CUDA / NCCL / allocation failures (std::runtime_error in the reference)."""


class sfeec_csr(C.Structure):
    _fields_ = [
        ("rows", C.c_int64),
        ("cols", C.c_int64),
        ("row_ptr", C.POINTER(C.c_int64)),
        ("col_idx", C.POINTER(C.c_int32)),
        ("val", C.POINTER(C.c_double)),
    ]


class sfeec_csr_owned(C.Structure):
    _fields_ = [
        ("rows", C.c_int64),
        ("cols", C.c_int64),
        ("nnz", C.c_int64),
        ("row_ptr", C.POINTER(C.c_int64)),
        ("col_idx", C.POINTER(C.c_int32)),
        ("val", C.POINTER(C.c_double)),
    ]


_lib = None

_P = C.c_void_p
_PD = C.POINTER(C.c_double)
_PI64 = C.POINTER(C.c_int64)
_PI32 = C.POINTER(C.c_int32)

_SIGS = {
    "sfeec_last_error": (C.c_char_p, []),
    "sfeec_version": (C.c_char_p, []),
    "sfeec_csr_free": (None, [C.POINTER(sfeec_csr_owned)]),
    "sfeec_device_count": (C.c_int, []),
    "sfeec_dev_create": (C.c_int, [C.POINTER(sfeec_csr)] * 3 + [C.POINTER(sfeec_csr),
                         C.c_double, C.c_double, C.c_double, C.c_int, C.c_int, C.c_int,
                         C.c_int, C.POINTER(_P)]),
    "sfeec_dev_destroy": (None, [_P]),
    "sfeec_dev_set_state": (C.c_int, [_P, _PD, C.c_int64, _PD, C.c_int64, C.c_double]),
    "sfeec_dev_get_state": (C.c_int, [_P, _PD, _PD, _PD]),
    "sfeec_dev_advance": (C.c_int, [_P, C.c_int64]),
    "sfeec_dev_advance_diag": (C.c_int, [_P, C.c_int64, C.c_int64, _PD, _PD]),
    "sfeec_dev_flow_he": (C.c_int, [_P, C.c_double]),
    "sfeec_dev_flow_ha": (C.c_int, [_P, C.c_double]),
    "sfeec_dev_energy": (C.c_int, [_P, _PD]),
    "sfeec_dev_gauss_residual": (C.c_int, [_P, _PD]),
    "sfeec_dev_cfl_number": (C.c_int, [_P, _PD]),
    "sfeec_dev_q_sym": (C.c_int, [_P, _PI64, _PI64, _PI32, _PD]),
    "sfeec_spmv": (C.c_int, [C.POINTER(sfeec_csr), _PD, _PD, C.c_int]),
    "sfeec_dev_set_stream": (C.c_int, [_P, _P]),
    "sfeec_dev_state_device_ptrs": (C.c_int, [_P, C.POINTER(_PD), C.POINTER(_PD)]),
    "sfeec_dev_last_launches": (C.c_int64, [_P]),
    "sfeec_dev_step_bytes": (C.c_double, [_P]),
    "sfeec_dev_layout_info": (C.c_int, [_P, C.c_int, _PI64, _PD]),
    "sfeec_dev_set_dt": (C.c_int, [_P, C.c_double]),
    "sfeec_dev_kernel_timing": (C.c_int, [_P, C.c_int, _PD, _PI64, _PD]),
    "sfeec_yee_create": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_double, C.c_double,
                                   C.c_double, C.c_double, C.c_double, C.c_double, C.c_int,
                                   C.c_int, C.c_int, C.POINTER(_P)]),
    "sfeec_yee_destroy": (None, [_P]),
    "sfeec_yee_dof_counts": (C.c_int, [_P, _PI64, _PI64]),
    "sfeec_yee_set_state": (C.c_int, [_P, _PD, _PD, C.c_double]),
    "sfeec_yee_get_state": (C.c_int, [_P, _PD, _PD, _PD]),
    "sfeec_yee_advance": (C.c_int, [_P, C.c_int64]),
    "sfeec_yee_flow_he": (C.c_int, [_P, C.c_double]),
    "sfeec_yee_flow_ha": (C.c_int, [_P, C.c_double]),
    "sfeec_yee_energy": (C.c_int, [_P, _PD]),
    "sfeec_yee_set_stream": (C.c_int, [_P, _P]),
    "sfeec_yee_set_variant": (C.c_int, [_P, C.c_int]),
    "sfeec_yee_last_launches": (C.c_int64, [_P]),
    "sfeec_yee_kernel_timing": (C.c_int, [_P, C.c_int, _PD, _PI64]),
    "sfeec_yee_step_bytes": (C.c_double, [_P]),
    "sfeec_nccl_unique_id": (C.c_int, [C.c_void_p]),
    "sfeec_nccl_selftest": (C.c_int, [C.c_int, C.c_int64, _PD]),
    "sfeec_yee_create_slab": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_double, C.c_double,
                                        C.c_double, C.c_double, C.c_double, C.c_double,
                                        C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_int,
                                        C.POINTER(_P)]),
    "sfeec_yee_create_slab_transport": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_double,
                                                  C.c_double, C.c_double, C.c_double, C.c_double,
                                                  C.c_double, C.c_int, C.c_int, C.c_int, C.c_int,
                                                  C.c_void_p, C.c_int, C.POINTER(_P)]),
    "sfeec_yee_slab_dof_counts": (C.c_int, [C.c_int] * 5 + [_PI64, _PI64]),
    "sfeec_yee_slab_dof_map": (C.c_int, [C.c_int] * 5 + [_PI64, _PI64]),
    "sfeec_yee_group_create": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_double, C.c_double,
                                         C.c_double, C.c_double, C.c_double, C.c_double,
                                         C.c_int, C.c_int, C.c_int, C.POINTER(_P)]),
    "sfeec_yee_group_destroy": (None, [_P]),
    "sfeec_yee_group_set_variant": (C.c_int, [_P, C.c_int]),
    "sfeec_yee_group_set_state": (C.c_int, [_P, _PD, _PD]),
    "sfeec_yee_group_get_state": (C.c_int, [_P, _PD, _PD]),
    "sfeec_yee_group_advance": (C.c_int, [_P, C.c_int64]),
    "sfeec_yee_group_energy": (C.c_int, [_P, _PD]),
    "sfeec_tet_dev_create": (C.c_int, [C.c_int, C.c_double, C.c_uint64, C.c_double, C.c_double,
                                       C.c_double, C.c_int, C.c_int, C.c_int, C.c_int,
                                       C.POINTER(_P), _PI64]),
    "sfeec_tet_dev_operators": (C.c_int, [C.c_int, C.c_double, C.c_uint64, C.c_int] +
                                [C.POINTER(sfeec_csr_owned)] * 5),
    "sfeec_dev_apply": (C.c_int, [_P, C.c_int, _PD, _PD]),
    "sfeec_dev_curl_curl": (C.c_int, [_P, _PD, _PD]),
    "sfeec_part_create":(C.c_int, [C.POINTER(sfeec_csr)] * 4 + [_PI64, _PI64, C.c_double,
                                    C.c_double, C.c_double, C.c_int, C.c_int, C.c_void_p,
                                    C.c_int, C.POINTER(_P)]),
    "sfeec_part_destroy": (None, [_P]),
    "sfeec_part_set_state": (C.c_int, [_P, _PD, _PD, C.c_double]),
    "sfeec_part_get_state": (C.c_int, [_P, _PD, _PD, _PD]),
    "sfeec_part_advance": (C.c_int, [_P, C.c_int64]),
    "sfeec_part_advance_local": (C.c_int, [C.POINTER(_P), C.c_int, C.c_int64]),
    "sfeec_part_attach_ipc": (C.c_int, [_P, C.c_void_p]),
    "sfeec_ipc_group_selftest": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_int, _PD]),
    "sfeec_part_energy": (C.c_int, [_P, _PD]),
    "sfeec_part_energy_local": (C.c_int, [C.POINTER(_P), C.c_int, _PD]),
    "sfeec_part_last_launches": (C.c_int64, [_P]),
    "sfeec_ipc_unique_id": (C.c_int, [_P]),
    "sfeec_lslab_create": (C.c_int, [C.c_int, C.c_int, C.c_double, C.c_uint64, C.c_double,
                                     C.c_double, C.c_double, C.c_int, C.c_int, C.c_int, C.c_int,
                                     _P, C.c_int, C.POINTER(_P), _PI64]),
    "sfeec_lslab_destroy": (None, [_P]),
    "sfeec_lslab_set_state": (C.c_int, [_P, _PD, _PD, C.c_double]),
    "sfeec_lslab_get_state": (C.c_int, [_P, _PD, _PD, _PD]),
    "sfeec_lslab_advance": (C.c_int, [_P, C.c_int64]),
    "sfeec_lslab_energy": (C.c_int, [_P, _PD]),
    "sfeec_lslab_cfl_number": (C.c_int, [_P, _PD]),
    "sfeec_lslab_set_dt": (C.c_int, [_P, C.c_double]),
    "sfeec_lslab_curl": (C.c_int, [_P, _PD, _PD]),
    "sfeec_lslab_stream": (C.c_int, [_P, C.POINTER(_P)]),
    "sfeec_lslab_last_launches": (C.c_int64, [_P]),
    "sfeec_lslab_step_bytes": (C.c_double, [_P]),
    "sfeec_lslab_kernel_timing": (C.c_int, [_P, C.c_int, _PD, _PI64, _PD]),
    "sfeec_part_create_tet": (C.c_int, [C.c_int, C.c_double, C.c_uint64, C.c_double, C.c_double,
                                        C.c_double, C.c_int, C.c_int, _P, C.c_int,
                                        C.POINTER(_P), _PI64]),
    "sfeec_part_create_p2": (C.c_int, [C.c_int, C.c_double, C.c_uint64, C.c_double, C.c_double,
                                       C.c_double, C.c_int, C.c_int, _P, C.c_int,
                                       C.POINTER(_P), _PI64]),
    "sfeec_part_apply": (C.c_int, [_P, C.c_int, _PD, _PD]),
    "sfeec_part_device_ptrs": (C.c_int, [_P, C.POINTER(_P), C.POINTER(_P), C.POINTER(_P)]),
    "sfeec_part_kernel_timing": (C.c_int, [_P, C.c_int, _PD, _PI64, _PD]),
    "sfeec_part_step_bytes": (C.c_double, [_P]),
    "sfeec_build_yee_mass": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_double, C.c_double,
                                       C.c_double, C.c_int, C.c_int,
                                       C.POINTER(sfeec_csr_owned)]),
    "sfeec_build_yee_curl": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_double, C.c_double,
                                       C.c_double, C.c_int, C.POINTER(sfeec_csr_owned),
                                       C.POINTER(sfeec_csr_owned)]),
    "sfeec_tetmesh_create": (C.c_int, [C.c_int, C.c_double, C.c_uint64, C.POINTER(_P)]),
    "sfeec_tetmesh_create_slab": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, C.c_uint64,
                                            C.POINTER(C.c_void_p)]),
    "sfeec_tetmesh_destroy": (None, [_P]),
    "sfeec_tetmesh_counts": (C.c_int, [_P, _PI64, _PI64, _PI64, _PI64]),
    "sfeec_tetmesh_geometry": (C.c_int, [_P, _PD, _PI64, _PI64, _PI64]),
    "sfeec_tetmesh_project_cavity": (C.c_int, [_P, C.c_int, _PD]),
    "sfeec_tet_l2_error": (C.c_int, [_P, _PD, C.c_int, C.c_int, C.c_int, _PD]),
    "sfeec_tetmesh_pulse": (C.c_int, [_P, C.c_int, _PD, _PD, C.c_double, C.c_int64, C.c_int64,
                                      _PD]),
    "sfeec_tetmesh_operator": (C.c_int, [_P, C.c_int, C.POINTER(sfeec_csr_owned)]),
    "sfeec_tetmesh_p2_counts": (C.c_int, [_P, _PI64, _PI64, _PI64]),
    "sfeec_tetmesh_p2_operator": (C.c_int, [_P, C.c_int, C.POINTER(sfeec_csr_owned)]),
    "sfeec_tetmesh_p2_dofs": (C.c_int, [_P, C.c_int, _PI64, C.POINTER(C.c_int8)]),
    "sfeec_p2_dev_create": (C.c_int, [C.c_int, C.c_double, C.c_uint64, C.c_double, C.c_double,
                                      C.c_double, C.c_int, C.c_int, C.c_int, C.c_int,
                                      C.POINTER(_P), _PI64]),
    "sfeec_p2_dev_operators": (C.c_int, [C.c_int, C.c_double, C.c_uint64, C.c_int] +
                               [C.POINTER(sfeec_csr_owned)] * 5),
    "sfeec_p2_spai_device": (C.c_int, [C.POINTER(sfeec_csr), C.c_int, C.POINTER(sfeec_csr_owned),
                                       _PI64]),
    "sfeec_make_pattern": (C.c_int, [C.POINTER(sfeec_csr), C.c_int,
                                     C.POINTER(sfeec_csr_owned)]),
    "sfeec_spai": (C.c_int, [C.POINTER(sfeec_csr), C.c_int, C.POINTER(sfeec_csr_owned), _PD]),
    "sfeec_csr_from_triplets":(C.c_int, [C.c_int64, C.c_int64, C.c_int64, _PI32, _PI32, _PD,
                                          C.POINTER(sfeec_csr_owned)]),
    "sfeec_csr_symmetric_part": (C.c_int, [C.POINTER(sfeec_csr), C.POINTER(sfeec_csr_owned)]),
    "sfeec_csr_transpose": (C.c_int, [C.POINTER(sfeec_csr), C.POINTER(sfeec_csr_owned)]),
}

EXPORTED_SYMBOLS = tuple(_SIGS)


def lib() -> C.CDLL:
    """Load libsfeec_b200.so; raises (no fallback) if it has not been built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise DeviceError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                "g.build()'` (there is no CPU fallback)")
        l = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            f = getattr(l, name)
            f.restype = res
            f.argtypes = args
        _lib = l
    return _lib


def check(code: int) -> None:
    if code == SFEEC_OK:
        return
    msg = lib().sfeec_last_error().decode()
    if code == SFEEC_EINVAL:
        raise InvalidParameter(msg)
    raise DeviceError(f"sfeec_b200 error {code}: {msg}")


def dptr(a: np.ndarray):
    return a.ctypes.data_as(_PD)


def i64ptr(a: np.ndarray):
    return a.ctypes.data_as(_PI64)


def i32ptr(a: np.ndarray):
    return a.ctypes.data_as(_PI32)


def owned_to_numpy(m: sfeec_csr_owned):
    """Copy a library-owned CSR into numpy arrays and free it."""
    rows, nnz = int(m.rows), int(m.nnz)
    rp = np.ctypeslib.as_array(m.row_ptr, shape=(rows + 1,)).copy()
    ci = np.ctypeslib.as_array(m.col_idx, shape=(max(nnz, 1),))[:nnz].copy()
    va = np.ctypeslib.as_array(m.val, shape=(max(nnz, 1),))[:nnz].copy()
    cols = int(m.cols)
    lib().sfeec_csr_free(C.byref(m))
    return rows, cols, rp, ci, va
