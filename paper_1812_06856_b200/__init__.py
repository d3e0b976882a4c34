"""B200-native (sm_100a) hot path of the superpixel light-field depth estimator (arXiv:1812.06856).

The compute lives in liblfdg.so (hand-written CUDA kernels behind the C-ABI in include/lfdg.h);
this package is the host-side mirror of the reference's operator API (proj/include/lfd/*.hpp).
"""
from .api import (  # noqa: F401
    DeviceContext,
    EnergyParams,
    MultiViewSet,
    PinholeCamera,
    PlaneMap,
    RefineContext,
    RefineStats,
    SlicParams,
    SuperpixelGrid,
    SweepParams,
    make_refine_context,
    plane_sweep_init,
    rasterize,
    refine_iteration,
    fuse_all,
    stability_fuse,
    run_refinement,
    slic_segment,
    sweep_view,
)

__all__ = [
    "DeviceContext", "EnergyParams", "MultiViewSet", "PinholeCamera", "PlaneMap", "RefineContext", "RefineStats",
    "SlicParams", "SuperpixelGrid", "SweepParams", "make_refine_context", "plane_sweep_init", "rasterize",
    "refine_iteration", "run_refinement", "fuse_all", "stability_fuse", "slic_segment", "sweep_view",
]
