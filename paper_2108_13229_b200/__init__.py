"""B200-native (sm_100a, fp64) preconditioned Krylov solver for the monolithic
MAC-Stokes + TPFA-Darcy system with Beavers-Joseph-Saffman coupling
(arXiv 2108.13229).  The CUDA library is libsdgpu.so (csrc/, C-ABI in
include/sdg.h); sdc.py mirrors the reference's C++ solver API over it.
"""
from .sdc import (  # noqa: F401
    AmgOptions,
    AmgPreconditioner,
    BlockPrecondKind,
    BlockPreconditioner,
    CoupledSystem,
    Context,
    GmresResult,
    IdentityPreconditioner,
    LinearOperator,
    Preconditioner,
    RestartController,
    ScenarioConfig,
    SdgCudaError,
    SolveReport,
    SparseMatrix,
    TdPreconditioner,
    UzawaConfig,
    UzawaPreconditioner,
    assemble_monolithic,
    bicgstab,
    default_context,
    gauss_seidel_apply,
    ground_dof,
    pd_gmres,
    power_iteration,
    sor_sweep,
    spmv,
    spmv_add,
    submatrix,
)

__all__ = [n for n in dir() if not n.startswith("_")]
