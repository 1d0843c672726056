"""B200-native SFEEC leapfrog (arXiv 2301.01753 hot path).

The compute path is libsfeec_b200.so (hand-written sm_100a CUDA + host C++),
reached through the C ABI in include/sfeec_b200.h. See DESIGN.md.
"""
from ._lib import DeviceError, InvalidParameter, LIB_PATH, lib  # noqa: F401
from .scheme import (  # noqa: F401
    FieldState,
    Formulation,
    SparseOperator,
    SplitKind,
    SplitScheme,
    TetMesh,
    UnitSystem,
    make_pattern,
    spai_approximate_inverse,
    YeeGroup,
    YeeScheme,
    YeeSlab,
    nccl_unique_id,
    yee_slab_dofs,
    device_count,
    make_state,
    operator_from_triplets,
    p2_device_operators,
    p2_device_scheme,
    spai_device,
    scaled_identity,
    symmetric_part,
    tet_device_operators,
    tet_device_scheme,
    transpose,
    yee_masses,
    yee_operators,
)
