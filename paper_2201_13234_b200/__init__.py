"""voxellate_b200: B200-native (sm_100a) labelling of Voronoi, Johnson-Mehl and
Laguerre tessellation images -- the hot path of the reference's
``tessellate_fast`` (arXiv 2201.13234 artifact), behind a C-ABI
(include/voxellate_b200.h).

The compute is the CUDA library ``libvoxellate_b200.so`` built in-tree; this
package only binds it.  There is no CPU fallback.
"""
from ._lib import LIB_PATH, VxError, lib  # noqa: F401
from .voxellate import (  # noqa: F401
    Boundary, DistanceImage, Domain, EvalCounters, FastOptions, ImageMeta, Kind, LabelImage,
    LaguerreSpheres, PruneResult, SiteSet, TessResult, ValidationReport, VoxelGrid, ball_voxels,
    generate_uniform_sites, scan_ball, optimal_r0, prune_ineffective_sites, read_distance_image,
    read_label_image, slab_bounds, spheres_to_timed_sites, tessellate_brute, tessellate_fast,
    tessellate_to_files, validate_partition, write_distance_image, write_label_image)

__all__ = [
    "Boundary", "Domain", "Kind", "SiteSet", "VoxelGrid", "FastOptions", "TessResult",
    "tessellate_fast", "tessellate_brute", "prune_ineffective_sites", "validate_partition",
    "generate_uniform_sites", "spheres_to_timed_sites", "optimal_r0", "slab_bounds",
    "ImageMeta", "write_label_image", "write_distance_image", "read_label_image",
    "read_distance_image", "tessellate_to_files", "ball_voxels", "scan_ball", "LaguerreSpheres",
]
