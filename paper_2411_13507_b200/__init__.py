"""B200-native graph-construction stage for reachable-Bezier-polytope planning (arXiv 2411.13507).

Drop-in for the hot path of the reference package ``beziergraph``
(/root/reference/pkg/src/beziergraph/graph.py: ``build_graph`` -> ``cut_graph`` ->
``find_path``) with the same planner API.  Compute runs in hand-written sm_100a
CUDA (``libbzg.so``, C ABI in include/bzg.h) behind ctypes; the host modules
here only prepare the constant matrices the reference also builds on the host
(oracle F/G, boundary map D, obstacle normalisation) and convert results.
"""

from .bezier import BezierSpec, boundary_matrix, derivative_matrix
from .geometry import EPS_GEO, Box, Hyperplane, Polytope, bounding_box, erode, inflate
from .graph import (
    BezierGraph,
    CutConfig,
    CutMask,
    CutProvenance,
    CutVerdict,
    PathQuery,
    SolveConfig,
    build_graph,
    check_edge,
    check_edges,
    cut_graph,
    cut_heuristic,
    cut_heuristic_batch,
    cut_qp,
    cut_qp_batch,
    find_path,
    path_cost,
)
from .reachability import ReachOracle, TrackingTube, build_oracle
from .plan import Planner
from .replan import Replanner, project_on_path

__version__ = "0.1.0"

__all__ = [
    "BezierSpec", "boundary_matrix", "derivative_matrix",
    "EPS_GEO", "Box", "Hyperplane", "Polytope", "bounding_box", "erode", "inflate",
    "BezierGraph", "CutConfig", "CutMask", "CutProvenance", "CutVerdict", "PathQuery", "SolveConfig",
    "build_graph", "check_edge", "check_edges", "cut_graph", "cut_heuristic", "cut_heuristic_batch", "cut_qp",
    "cut_qp_batch", "find_path", "path_cost", "Planner", "Replanner", "project_on_path",
    "ReachOracle", "TrackingTube", "build_oracle",
]
