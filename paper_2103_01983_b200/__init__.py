"""paper_2103_01983_b200 — B200-native (sm_100a) hot path of the PTROM
reference (arXiv 2103.01983): regularized 2-D Biot–Savart all-pairs
velocity/Jacobian, the implicit-trapezoidal FOM, the Barnes–Hut quadtree and
the PTROM online path, behind the C ABI in include/ptrom_b200.h.

The compute path is libptrom_b200.so (hand-written CUDA for sm_100a);
this package is the host-side mirror of the reference interface.
"""
from .api import (  # noqa: F401
    BlockDiagonalJacobian,
    ConfigError,
    Context,
    CudaError,
    KernelForm,
    LatticeSpec,
    NewtonConfig,
    NumericalError,
    PairwiseModel,
    ParticleSystem,
    SimulateResult,
    TimeGrid,
    default_context,
    fom_simulate,
    hamiltonian,
    inexact_kernel_jacobian,
    kernel_eval_count,
    pairwise_velocity,
    reset_kernel_eval_count,
    velocity_field_grid,
)
from ._lib import LIB_PATH, load as load_library  # noqa: F401
