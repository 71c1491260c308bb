"""decmg-b200: B200-native DEC geometric multigrid (drop-in for the V-cycle hot
path of arxiv/paper_2508_12501's `decmg` library).

The numerical work lives in libdecmg_gpu.so (hand-written sm_100a kernels,
C ABI in include/decmg_gpu.h). This package is the host-side mirror of the
reference's C++ multigrid API; it has no CPU implementation of the path.
"""
from ._lib import DecmgError, CudaError, LIB_PATH, load as load_library
from .multigrid import (CycleKind, CyclePlan, CycleResult, DistributedHierarchy, MultigridHierarchy, Smoother,
                        SmootherConfig, SolveReport, Transition, base_mesh, build_hierarchy, gmg_preconditioned_cg,
                        gmg_solve, gmg_solve_batches, nccl_unique_id, read_obj, smooth, standard_plan)

__all__ = ["CycleKind", "CyclePlan", "CycleResult", "DistributedHierarchy", "MultigridHierarchy", "nccl_unique_id", "Smoother", "SmootherConfig",
           "SolveReport", "Transition", "base_mesh", "build_hierarchy", "gmg_preconditioned_cg", "gmg_solve", "gmg_solve_batches",
           "standard_plan", "read_obj", "smooth",
           "DecmgError", "CudaError", "LIB_PATH", "load_library"]
