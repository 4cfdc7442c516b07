"""ctypes binding of the C ABI in ``include/windvox_b200.h``.

The library is the in-tree ``_lib/libwindvox_b200.so`` built for sm_100a
(``python -m paper_2407_11272_b200._build``).  There is no CPU fallback: if
the library is missing or no CUDA device is visible, every entry point raises
``WindvoxCudaUnavailable``.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

_PKG = Path(__file__).resolve().parent
LIB_PATH = _PKG / "_lib" / "libwindvox_b200.so"
# A/B builds of kernel variants (tools/build_variant.py) load another copy
if os.environ.get("WV_LIB_PATH"):
    LIB_PATH = Path(os.environ["WV_LIB_PATH"])

WV_OK = 0
PACK_EXACT_F32 = 1
PACK_SOFT_F32 = 2
PACK_EXACT_F64 = 3
PACK_SOFT_F64 = 4
PACK_SOFTGRAD_F32 = 5
PACK_SOFTGRAD_F64 = 6
PACK_EXACTGRAD_F32 = 7
PACK_EXACTGRAD_F64 = 8
PACK_EXACTSTRIP_F32 = 9
PACK_EXACTSTRIP_F64 = 10
PACK_EXACTTRAIL_F32 = 11
PACK_EXACTTRAIL_F64 = 12
POLICY_RAW = 0
POLICY_HALF = 1

# every symbol the public header declares (checked by tests/test_capi_symbols.py)
EXPORTED = (
    "wv_version", "wv_status_string", "wv_set_device", "wv_packed_bytes", "wv_pack_faces",
    "wv_pack_exact_grad", "wv_vertex_normals", "wv_fwd_workspace_bytes", "wv_exact_fwd_grid_f32", "wv_exact_fwd_points_f32",
    "wv_soft_fwd_grid_f32", "wv_soft_fwd_points_f32", "wv_exact_fwd_grid_f64",
    "wv_exact_fwd_points_f64", "wv_soft_fwd_grid_f64", "wv_soft_fwd_points_f64",
    "wv_bwd_workspace_bytes", "wv_exact_bwd_grid_f32", "wv_exact_bwd_points_f32",
    "wv_soft_bwd_grid_f32", "wv_soft_bwd_points_f32", "wv_exact_bwd_grid_f64",
    "wv_exact_bwd_points_f64", "wv_soft_bwd_grid_f64", "wv_soft_bwd_points_f64",
    "wv_face_to_vertex", "wv_loss_workspace_bytes", "wv_loss_terms_f32", "wv_loss_terms_f64",
    "wv_loss_finalize", "wv_mc_classify", "wv_mc_edges", "wv_mc_vertices", "wv_mc_emit",
    "wv_mc_vertices_slab", "wv_launch_count",
    "wv_splitmix64_uniform", "wv_pairwise_sum_workspace_bytes", "wv_pairwise_sum",
    "wv_surface_cdf", "wv_sample_surface", "wv_nearest_distances",
    "wv_fwd_workspace_bytes_batch", "wv_fwd_grid_f32_batch", "wv_bwd_workspace_bytes_batch",
    "wv_bwd_grid_f32_batch", "wv_strip_order", "wv_pack_exact_strip",
    "wv_exact_strip_fwd_grid_f32", "wv_exact_strip_fwd_points_f32",
    "wv_exact_pair_bwd_workspace_bytes", "wv_exact_pair_bwd_grid_f32",
    "wv_exact_pair_bwd_points_f32", "wv_pack_faces_batch", "wv_loss_terms_f32_batch",
    "wv_face_to_vertex_batch", "wv_pack_exact_strip_f64", "wv_exact_strip_fwd_grid_f64",
    "wv_exact_strip_fwd_points_f64", "wv_trail_edges", "wv_edge_trails", "wv_pack_exact_trail",
    "wv_exact_trail_bwd_workspace_bytes", "wv_exact_trail_bwd_grid_f32",
    "wv_pack_exact_trail_f64", "wv_exact_trail_bwd_workspace_bytes_f64",
    "wv_exact_trail_bwd_grid_f64", "wv_exact_trail_bwd_points_f64",
)


class WindvoxCudaUnavailable(RuntimeError):
    """The sm_100a CUDA library or a CUDA device is not available."""


class Grid(ctypes.Structure):
    _fields_ = [("lo", ctypes.c_double * 3), ("hi", ctypes.c_double * 3),
                ("res", ctypes.c_int64 * 3)]


_lib = None


def _declare(lib):
    P = ctypes.c_void_p
    I64 = ctypes.c_int64
    I = ctypes.c_int
    SZ = ctypes.c_size_t
    D = ctypes.c_double
    fwd32_grid = [P, I64, Grid, I64, I64, I, P, P, P, SZ, P]
    fwd32_pts = [P, I64, P, I64, I, P, P, P, SZ, P]
    bwd_grid = [P, I64, Grid, I64, I64, P, D, P, P, SZ, P]
    bwd_pts = [P, I64, P, I64, P, D, P, P, SZ, P]
    loss = [P, P, P, P, I64, P, P, P, SZ, P]
    sig = {
        "wv_version": ([], ctypes.c_char_p),
        "wv_status_string": ([I], ctypes.c_char_p),
        "wv_set_device": ([I], I),
        "wv_packed_bytes": ([I, I64], SZ),
        "wv_pack_faces": ([I, P, I, I64, P, I, I64, P, P], I),
        "wv_pack_exact_grad": ([I, P, I, I64, P, I, P, P, I64, P, P], I),
        "wv_vertex_normals": ([P, I64, P, I64, P, P, P, P, P], I),
        "wv_fwd_workspace_bytes": ([I, I64, I64], SZ),
        "wv_exact_fwd_grid_f32": (fwd32_grid, I),
        "wv_exact_fwd_points_f32": (fwd32_pts, I),
        "wv_soft_fwd_grid_f32": (fwd32_grid, I),
        "wv_soft_fwd_points_f32": (fwd32_pts, I),
        "wv_exact_fwd_grid_f64": ([P, I64, Grid, I64, I64, I, I, P, P, P], I),
        "wv_exact_fwd_points_f64": ([P, I64, P, I64, I, I, P, P, P], I),
        "wv_soft_fwd_grid_f64": ([P, I64, Grid, I64, I64, I, P, P, P], I),
        "wv_soft_fwd_points_f64": ([P, I64, P, I64, I, P, P, P], I),
        "wv_bwd_workspace_bytes": ([I, I64, I64], SZ),
        "wv_exact_bwd_grid_f32": (bwd_grid, I),
        "wv_exact_bwd_points_f32": (bwd_pts, I),
        "wv_soft_bwd_grid_f32": (bwd_grid, I),
        "wv_soft_bwd_points_f32": (bwd_pts, I),
        "wv_exact_bwd_grid_f64": (bwd_grid, I),
        "wv_exact_bwd_points_f64": (bwd_pts, I),
        "wv_soft_bwd_grid_f64": (bwd_grid, I),
        "wv_soft_bwd_points_f64": (bwd_pts, I),
        "wv_face_to_vertex": ([P, P, P, I64, P, I, P, P, P], I),
        "wv_loss_workspace_bytes": ([I64], SZ),
        "wv_loss_terms_f32": (loss, I),
        "wv_loss_terms_f64": (loss, I),
        "wv_loss_finalize": ([P, P], I),
        "wv_mc_classify": ([P, I, Grid, D, P, P, P, P], I),
        "wv_mc_edges": ([P, I, Grid, D, P, P], I),
        "wv_mc_vertices": ([P, I, Grid, D, P, P, P, P], I),
        "wv_mc_emit": ([P, P, P, I, P, P, P, Grid, P, P], I),
        "wv_mc_vertices_slab": ([P, I, Grid, I64, I64, D, P, P, P, P], I),
        "wv_launch_count": ([], ctypes.c_longlong),
        "wv_splitmix64_uniform": ([ctypes.c_uint64, I64, P, P], I),
        "wv_pairwise_sum_workspace_bytes": ([I64], SZ),
        "wv_pairwise_sum": ([P, I64, P, P, SZ, P], I),
        "wv_surface_cdf": ([P, P, I64, P, P, P, P, SZ, P], I),
        "wv_sample_surface": ([P, P, I64, P, P, ctypes.c_uint64, I64, P, P], I),
        "wv_nearest_distances": ([P, I64, P, I64, P, P], I),
        "wv_fwd_workspace_bytes_batch": ([I, I64, I64, I64], SZ),
        "wv_fwd_grid_f32_batch": ([I, P, SZ, I64, Grid, I64, I64, I64, I, P, P, P, SZ, P], I),
        "wv_bwd_workspace_bytes_batch": ([I, I64, I64, I64], SZ),
        "wv_bwd_grid_f32_batch": ([I, P, SZ, I64, Grid, I64, I64, I64, P, D, P, P, SZ, P], I),
        "wv_strip_order": ([P, I64, P, I64, P, P, P], I),
        "wv_pack_exact_strip": ([P, I, I64, P, I, I64, P, P, P, P, P], I),
        "wv_exact_strip_fwd_grid_f32": (fwd32_grid, I),
        "wv_exact_strip_fwd_points_f32": (fwd32_pts, I),
        "wv_exact_pair_bwd_workspace_bytes": ([I64, I64], SZ),
        "wv_exact_pair_bwd_grid_f32": (bwd_grid, I),
        "wv_exact_pair_bwd_points_f32": (bwd_pts, I),
        "wv_pack_faces_batch": ([I, P, I, I64, P, I, I64, I64, P, SZ, P], I),
        "wv_loss_terms_f32_batch": ([P, P, P, P, I64, I64, P, P, P, SZ, P], I),
        "wv_face_to_vertex_batch": ([P, I64, P, P, I64, I64, P, I64, I, P, P, P], I),
        "wv_pack_exact_strip_f64": ([P, I, I64, P, I, I64, P, P, P, P, P], I),
        "wv_exact_strip_fwd_grid_f64": ([P, I64, Grid, I64, I64, I, I, P, P, P], I),
        "wv_exact_strip_fwd_points_f64": ([P, I64, P, I64, I, I, P, P, P], I),
        "wv_trail_edges": ([], I),
        "wv_edge_trails": ([P, I64, P, I64, P, P, P, P, P, P, P], I),
        "wv_pack_exact_trail": ([P, I, I64, P, I64, P, P], I),
        "wv_exact_trail_bwd_workspace_bytes": ([I64, I64], SZ),
        "wv_exact_trail_bwd_grid_f32": (bwd_grid, I),
        "wv_pack_exact_trail_f64": ([P, I, I64, P, I64, P, P], I),
        "wv_exact_trail_bwd_workspace_bytes_f64": ([I64, I64], SZ),
        "wv_exact_trail_bwd_grid_f64": (bwd_grid, I),
        "wv_exact_trail_bwd_points_f64": (bwd_pts, I),
    }
    for name, (args, res) in sig.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    return lib


def load_library(path: Path | None = None):
    """Load (without requiring a GPU) the shared library; raises if absent."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = Path(path) if path else LIB_PATH
    if not p.exists():
        raise WindvoxCudaUnavailable(
            f"{p} is missing: build it with `python -m paper_2407_11272_b200._build` "
            "(nvcc, sm_100a). There is no CPU fallback.")
    lib = _declare(ctypes.CDLL(str(p)))
    if path is None:
        _lib = lib
    return lib


def lib():
    """The loaded library, after checking a CUDA device is present."""
    import torch

    if not torch.cuda.is_available():
        raise WindvoxCudaUnavailable(
            "no CUDA device visible: windvox_b200 runs only on B200 (sm_100a); "
            "there is no CPU fallback")
    return load_library()


def check(rc: int, what: str) -> None:
    if rc != WV_OK:
        msg = load_library().wv_status_string(int(rc)).decode()
        raise RuntimeError(f"{what} failed: status {rc} ({msg})")


def make_grid(bounds_min, bounds_max, resolution) -> Grid:
    g = Grid()
    for i in range(3):
        g.lo[i] = float(bounds_min[i])
        g.hi[i] = float(bounds_max[i])
        g.res[i] = int(resolution[i])
    return g
