"""B200-native NESA matrix-vector product (arXiv 1801.03589 hot path).

Host API mirrors the reference package ``taskfmm``
(/root/reference/pkg/src/taskfmm/__init__.py:3-23) for the hot path and its
inputs: geometry, quadtree, operator assembly and the matvec.  The matvec
itself runs in libnesa_b200.so (hand-written sm_100a CUDA, C ABI in
include/nesa_b200.h); there is no CPU fallback.
"""

from .benchmark import BenchConfig, run_benchmark
from .dense import dense_matvec_gpu
from .fastmvp import as_tree, get_plan, mvp, mvp_serial, task_counts
from .geometry import (BBox, CurveSpec, bounding_box, generate_sources, parse_curve_spec,
                       plane_wave_rhs, random_rhs, wavenumber)
from .linalg import circle_points, gemv, kernel_eval, kernel_matrix, pinv
from .operators import NesaParams, OperatorSet, OperatorTables, build_all, build_tables
from .pipeline import MvpPipeline
from .serialize import load_problem, save_problem
from .solver import GmresResult, gmres
from .plan import NesaPlan, algorithmic_bytes, algorithmic_flops
from .quadtree import Tree, TreeParams, build_tree, interaction_list, neighbor_list, tree_stats

__version__ = "0.1.0"

__all__ = [
    "BBox", "BenchConfig", "CurveSpec", "dense_matvec_gpu", "run_benchmark", "GmresResult", "MvpPipeline", "NesaParams", "NesaPlan", "OperatorSet", "OperatorTables", "Tree",
    "TreeParams", "algorithmic_bytes", "algorithmic_flops", "as_tree", "bounding_box",
    "build_all", "build_tables", "build_tree", "circle_points", "gemv", "generate_sources",
    "get_plan", "gmres", "interaction_list", "kernel_eval", "load_problem", "kernel_matrix", "mvp", "mvp_serial",
    "neighbor_list", "parse_curve_spec", "pinv", "plane_wave_rhs", "random_rhs", "save_problem",
    "task_counts", "tree_stats", "wavenumber",
]
