"""paper_2407_11272_b200 -- B200-native winding-number voxelization hot path.

Drop-in for the hot path of the reference package ``windvox``
(/root/reference/pkg/src/windvox): same API names and semantics, backed by
hand-written sm_100a CUDA kernels behind the C ABI of
``include/windvox_b200.h``.  There is no CPU fallback.
"""

from .errors import DegenerateError, DivergedError, OnSurfaceError, ParseError
from .types import (GridSpec, LossReport, QueryBatchConfig, ScalarField, TriangleMesh,
                    VertexGradients, surface_epsilon)
from .winding import (binarize, solid_angle_triangle, voxelize, winding_number_batch,
                      winding_number_exact, winding_number_soft)
from .grad import exact_loss_grad, occupancy_loss_grad, soft_winding_vertex_jacobian
from .autograd import WindingNumber, winding_number
from .fieldio import load_field, save_field
from .morph import MorphConfig, MorphReport, morph
from .openmesh import flipped_duplication, vertex_normals
from .recon import laplacian_smooth, marching_cubes
from .metrics import (chamfer_distance, evaluate_reconstruction, hausdorff_distance,
                      sample_surface, splitmix64_uniform)

__version__ = "0.1.0"

__all__ = [
    "DegenerateError", "DivergedError", "OnSurfaceError", "ParseError",
    "TriangleMesh", "GridSpec", "ScalarField", "QueryBatchConfig", "VertexGradients",
    "LossReport", "surface_epsilon",
    "solid_angle_triangle", "winding_number_exact", "winding_number_soft",
    "winding_number_batch", "voxelize", "binarize",
    "soft_winding_vertex_jacobian", "occupancy_loss_grad", "exact_loss_grad",
    "WindingNumber", "winding_number",
    "save_field", "load_field", "MorphConfig", "MorphReport", "morph",
    "flipped_duplication", "vertex_normals", "marching_cubes", "laplacian_smooth",
    "splitmix64_uniform", "sample_surface", "chamfer_distance", "hausdorff_distance",
    "evaluate_reconstruction",
    "__version__",
]
