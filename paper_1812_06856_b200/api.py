"""Host-side mirror of the reference's hot-path API (proj/include/lfd), backed by the C-ABI.

Two layers:

* ``DeviceContext`` — a thin object over one ``lfdg_ctx``: views, grids, planes and depth stay
  resident in HBM between calls (the fast path used by bench.py and the multi-GPU driver).
* Reference-shaped free functions with the reference's names, argument meaning and errors:
  ``slic_segment`` (superpixel.hpp:179), ``sweep_view`` (sweep.hpp:112), ``plane_sweep_init``
  (sweep.hpp:141), ``rasterize`` (sweep.hpp:44), ``make_refine_context`` (refine.hpp:53),
  ``refine_iteration`` (refine.hpp:253) and ``run_refinement`` (refine.hpp:325), operating on
  host value types (``MultiViewSet``, ``SuperpixelGrid``, ``PlaneMap``).  Each call marshals
  host buffers through the C-ABI exactly like a drop-in for the inline C++ functions would;
  ``workers`` is accepted and ignored (the reference's results are worker-invariant).

There is no CPU fallback: every compute call runs the sm_100a kernels in liblfdg.so.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

import numpy as np

from . import _native as N
from ._native import InvalidParams, InvariantError, LfdgError, StateError  # noqa: F401  (re-exported)

# ----------------------------------------------------------------------------- value types


@dataclass
class SlicParams:  # superpixel.hpp:18
    size: int = 12
    compactness: float = 0.10
    iterations: int = 10

    def validate(self) -> None:  # superpixel.hpp:23-27
        if self.size < 4:
            raise InvalidParams("superpixel size must be >= 4")
        if self.compactness <= 0:
            raise InvalidParams("compactness must be > 0")
        if self.iterations < 1:
            raise InvalidParams("iterations must be >= 1")

    def c(self):
        return N.SlicParamsC(self.size, self.compactness, self.iterations)


@dataclass
class SweepParams:  # sweep.hpp:14
    levels: int = 80
    tssd_threshold: float = 0.05
    max_neighbors: int = 0

    def validate(self) -> None:  # sweep.hpp:19-22
        if self.levels < 2:
            raise InvalidParams("sweep levels must be >= 2")
        if self.tssd_threshold <= 0:
            raise InvalidParams("tssd threshold must be > 0")

    def c(self):
        return N.SweepParamsC(self.levels, self.tssd_threshold, self.max_neighbors)


@dataclass
class EnergyParams:  # refine.hpp:15
    sigma: float = 0.0
    alpha: float = 0.075
    eta: float = 0.5
    size_init: int = 0
    steps_init: int = 5
    iterations: int = 5
    max_neighbors: int = 0
    use_smoothness: bool = True
    use_consistency: bool = True
    use_occlusion: bool = True

    def validate(self) -> None:  # refine.hpp:28-31
        if self.sigma < 0 or self.alpha <= 0 or self.eta < 0 or self.eta > 1:
            raise InvalidParams("bad energy params")
        if self.steps_init <= 0 or self.size_init < 0 or self.iterations < 0:
            raise InvalidParams("bad kernel params")

    def c(self):
        return N.EnergyParamsC(self.sigma, self.alpha, self.eta, self.size_init, self.steps_init, self.iterations,
                               self.max_neighbors, int(self.use_smoothness), int(self.use_consistency),
                               int(self.use_occlusion))


@dataclass
class PinholeCamera:  # geometry.hpp:22
    intrinsics: np.ndarray = field(default_factory=lambda: np.eye(3))
    rotation: np.ndarray = field(default_factory=lambda: np.eye(3))
    translation: np.ndarray = field(default_factory=lambda: np.zeros(3))
    view_id: int = 0

    def as_array(self) -> np.ndarray:
        return np.concatenate([np.asarray(self.intrinsics, np.float64).reshape(9),
                               np.asarray(self.rotation, np.float64).reshape(9),
                               np.asarray(self.translation, np.float64).reshape(3)])

    @staticmethod
    def from_array(a: np.ndarray, view_id: int = 0) -> "PinholeCamera":
        a = np.asarray(a, np.float64)
        return PinholeCamera(a[:9].reshape(3, 3).copy(), a[9:18].reshape(3, 3).copy(), a[18:21].copy(), view_id)


@dataclass
class MultiViewSet:  # io.hpp:41 (images are scaled LAB [V][H][W][3] float32)
    cameras: List[PinholeCamera]
    images: np.ndarray
    range: Tuple[float, float]

    def num_views(self) -> int:
        return len(self.cameras)

    @property
    def width(self) -> int:
        return int(self.images.shape[2])

    @property
    def height(self) -> int:
        return int(self.images.shape[1])

    def camera_array(self) -> np.ndarray:
        return np.stack([c.as_array() for c in self.cameras])


@dataclass
class SuperpixelGrid:  # superpixel.hpp:39, grid.pixels as CSR (offsets + row-major members)
    width: int
    height: int
    grid_w: int
    grid_h: int
    cell_size: int
    label_map: np.ndarray
    sp: np.ndarray  # structured records (RECORD_DTYPE)
    offsets: np.ndarray
    members: np.ndarray

    def num_superpixels(self) -> int:
        return self.grid_w * self.grid_h

    def label(self, x: int, y: int) -> int:
        return int(self.label_map[y * self.width + x])

    def pixels(self, sp_id: int) -> np.ndarray:
        return self.members[self.offsets[sp_id]:self.offsets[sp_id + 1]]


@dataclass
class PlaneMap:  # sweep.hpp:27: planes [view] -> f64[nsp, 4] (depth, nx, ny, nz); depth [view] -> f32[H, W]
    planes: List[np.ndarray] = field(default_factory=list)
    depth: List[np.ndarray] = field(default_factory=list)


@dataclass
class RefineStats:  # refine.hpp:244
    accepted: int = 0
    violations: int = 0


# ----------------------------------------------------------------------------- shape checks
# The C-ABI takes raw pointers and derives every size from (V, W, H) of the context, so a wrongly
# shaped array would be over-read on the host (or by an async DMA).  Check before the call and
# raise InvalidParams like the reference's validation does.


def check_images(images: np.ndarray, what: str = "images", H: Optional[int] = None, W: Optional[int] = None,
                 n_max: Optional[int] = None) -> None:
    if images.ndim != 4 or images.shape[3] != 3 or images.shape[0] < 1:
        raise InvalidParams(f"{what} must be [n][H][W][3], got shape {tuple(images.shape)}")
    if H is not None and (images.shape[1], images.shape[2]) != (H, W):
        raise InvalidParams(f"{what} are {images.shape[2]}x{images.shape[1]}, the context holds {W}x{H} views")
    if n_max is not None and images.shape[0] > n_max:
        raise InvalidParams(f"{what}: {images.shape[0]} views, at most {n_max} fit")


def check_shape(a: np.ndarray, shape: tuple, what: str) -> None:
    if tuple(a.shape) != tuple(shape):
        raise InvalidParams(f"{what} must have shape {tuple(shape)}, got {tuple(a.shape)}")


# ----------------------------------------------------------------------------- device context


class DeviceContext:
    """One lfdg_ctx: a device-resident MultiViewSet + grids + PlaneMap + RefineContext."""

    def __init__(self, device: int = 0):
        self.L = N.lib()
        h = C.c_void_p()
        N.check(self.L.lfdg_create(device, C.byref(h)))
        self.h = h
        self.device = device
        self.V = self.W = self.H = 0

    def close(self):
        if getattr(self, "h", None):
            self.L.lfdg_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- plumbing
    def set_stream(self, stream_handle: int | None):
        N.check(self.L.lfdg_set_stream(self.h, C.c_void_p(stream_handle) if stream_handle else None))

    def synchronize(self):
        N.check(self.L.lfdg_synchronize(self.h))

    def upload_rgb(self, rgb: np.ndarray, v0: int = 0):
        """Replace the LAB images of views [v0, v0 + n) by rgb_to_scaled_lab (image.hpp:97-107) of the
        sRGB images rgb [n][H][W][3], converted on the device (bit-identical to the reference)."""
        rgb = np.ascontiguousarray(rgb, np.float32)
        check_images(rgb, "rgb images", self.H, self.W, self.V - v0)
        N.check(self.L.lfdg_upload_rgb(self.h, v0, rgb.shape[0], N.ptr(rgb)))
        self.synchronize()

    def upload_rgb8(self, rgb8: np.ndarray, v0: int = 0):
        """Replace the LAB images of views [v0, v0 + n) by rgb_to_scaled_lab of the 8-bit sRGB images
        rgb8 [n][H][W][3] (R, G, B bytes; each channel / 255.f as read_image, io.hpp:136-146)."""
        rgb8 = np.ascontiguousarray(rgb8, np.uint8)
        check_images(rgb8, "rgb8 images", self.H, self.W, self.V - v0)
        N.check(self.L.lfdg_upload_rgb8(self.h, v0, rgb8.shape[0], N.ptr(rgb8)))
        self.synchronize()

    def launch_count(self) -> int:
        return int(self.L.lfdg_launch_count(self.h))

    def device_buffer(self, which: int):
        p, nb, st = C.c_void_p(), C.c_size_t(), C.c_size_t()
        N.check(self.L.lfdg_device_buffer(self.h, which, C.byref(p), C.byref(nb), C.byref(st)))
        return p.value, nb.value, st.value

    def mark_views_ready(self, v0: int, n: int, what: int):
        N.check(self.L.lfdg_mark_views_ready(self.h, v0, n, what))

    # -- views
    def set_views(self, images: np.ndarray, cams: np.ndarray, d_range: Sequence[float]):
        images = np.ascontiguousarray(images, np.float32)
        check_images(images)
        cams = np.ascontiguousarray(cams, np.float64)
        V, H, W = images.shape[:3]
        if cams.size != V * 21:
            raise InvalidParams(f"cameras must be [{V}][21] (K, R row-major, t), got shape {tuple(cams.shape)}")
        cams = cams.reshape(V, 21)
        if len(d_range) != 2:
            raise InvalidParams("depth range must be (d_min, d_max)")
        N.check(self.L.lfdg_set_views(self.h, V, W, H, N.ptr(images), N.ptr(cams), float(d_range[0]),
                                      float(d_range[1])))
        self.V, self.W, self.H = V, W, H

    def update_images(self, v0: int, images: np.ndarray):
        images = np.ascontiguousarray(images, np.float32)
        check_images(images, "images", self.H, self.W, self.V - v0)
        N.check(self.L.lfdg_update_images(self.h, v0, images.shape[0], N.ptr(images)))

    # -- SLIC
    def slic(self, view: int, params: SlicParams = SlicParams()):
        p = params.c()
        N.check(self.L.lfdg_slic_segment(self.h, view, C.byref(p)))

    def slic_views(self, v0: int, n: int, params: SlicParams = SlicParams()):
        p = params.c()
        N.check(self.L.lfdg_slic_segment_views(self.h, v0, n, C.byref(p)))

    def grid_shape(self, view: int):
        gw, gh, s = C.c_int(), C.c_int(), C.c_int()
        N.check(self.L.lfdg_grid_shape(self.h, view, C.byref(gw), C.byref(gh), C.byref(s)))
        return gw.value, gh.value, s.value

    def get_grid(self, view: int) -> SuperpixelGrid:
        gw, gh, s = self.grid_shape(view)
        n = gw * gh
        labels = np.zeros(self.H * self.W, np.int32)
        rec = np.zeros(n, N.RECORD_DTYPE)
        off = np.zeros(n + 1, np.int32)
        mem = np.zeros(self.H * self.W, np.int32)
        N.check(self.L.lfdg_get_grid(self.h, view, N.ptr(labels), N.ptr(rec), N.ptr(off), N.ptr(mem)))
        return SuperpixelGrid(self.W, self.H, gw, gh, s, labels, rec, off, mem)

    def set_grid(self, view: int, cell_size: int, label_map: np.ndarray):
        lm = np.ascontiguousarray(label_map, np.int32).reshape(-1)
        if lm.size != self.H * self.W:
            raise InvalidParams(f"label map must hold {self.H * self.W} labels, got {lm.size}")
        N.check(self.L.lfdg_set_grid(self.h, view, cell_size, N.ptr(lm)))

    # -- sweep / planes / depth
    def sweep(self, view: int, params: SweepParams, seed: int) -> np.ndarray:
        gw, gh, _ = self.grid_shape(view)
        out = np.zeros((gw * gh, 4), np.float64)
        p = params.c()
        N.check(self.L.lfdg_sweep_view(self.h, view, C.byref(p), C.c_uint64(seed), N.ptr(out)))
        return out

    def sweep_views(self, v0: int, n: int, params: SweepParams, seed: int):
        p = params.c()
        N.check(self.L.lfdg_sweep_views(self.h, v0, n, C.byref(p), C.c_uint64(seed)))

    def matching_views(self, view: int, max_neighbors: int = 0) -> List[int]:
        out = np.zeros(max(self.V, 1), np.int32)
        n = C.c_int()
        N.check(self.L.lfdg_matching_views(self.h, view, max_neighbors, N.ptr(out), C.byref(n)))
        return out[:n.value].tolist()

    def set_planes(self, view: int, planes: np.ndarray):
        planes = np.ascontiguousarray(planes, np.float64)
        gw, gh, _ = self.grid_shape(view)
        check_shape(planes, (gw * gh, 4), "planes")
        N.check(self.L.lfdg_set_planes(self.h, view, N.ptr(planes)))

    def get_planes(self, view: int) -> np.ndarray:
        gw, gh, _ = self.grid_shape(view)
        out = np.zeros((gw * gh, 4), np.float64)
        N.check(self.L.lfdg_get_planes(self.h, view, N.ptr(out)))
        return out

    def rasterize(self, v0: int = 0, n: Optional[int] = None):
        if n is None and v0 == 0:
            N.check(self.L.lfdg_rasterize(self.h))
        else:
            N.check(self.L.lfdg_rasterize_views(self.h, v0, self.V - v0 if n is None else n))

    def get_depth(self, view: int) -> np.ndarray:
        out = np.zeros((self.H, self.W), np.float32)
        N.check(self.L.lfdg_get_depth(self.h, view, N.ptr(out)))
        return out

    def set_depth(self, view: int, depth: np.ndarray):
        depth = np.ascontiguousarray(depth, np.float32)
        if depth.size != self.H * self.W:
            raise InvalidParams(f"depth map must be [{self.H}][{self.W}], got shape {tuple(depth.shape)}")
        N.check(self.L.lfdg_set_depth(self.h, view, N.ptr(depth)))

    # -- refinement
    def make_refine_context(self, params: EnergyParams, sweep_levels: int):
        p = params.c()
        s, k = C.c_double(), C.c_int()
        N.check(self.L.lfdg_make_refine_context(self.h, C.byref(p), sweep_levels, C.byref(s), C.byref(k)))
        return s.value, k.value

    def set_refine_views(self, v0: int, n: int):
        N.check(self.L.lfdg_set_refine_views(self.h, v0, n))

    def refine_iteration(self, l: int, with_stats: bool = True):
        a, v = C.c_uint64(), C.c_uint64()
        if with_stats:
            N.check(self.L.lfdg_refine_iteration(self.h, l, C.byref(a), C.byref(v)))
            return a.value, v.value
        N.check(self.L.lfdg_refine_iteration(self.h, l, None, None))
        return None

    def run_refinement(self):
        a, v = C.c_uint64(), C.c_uint64()
        N.check(self.L.lfdg_run_refinement(self.h, C.byref(a), C.byref(v)))
        return a.value, v.value

    def refine_work(self, reset: bool = True):
        """(pixel-evals, candidate evals) of pair_stats since the last reset."""
        a, b = C.c_uint64(), C.c_uint64()
        N.check(self.L.lfdg_refine_work(self.h, C.byref(a), C.byref(b), int(reset)))
        return a.value, b.value

    def work_counters(self, reset: bool = False) -> dict:
        """The context's work counters (lfdg_work_counters); reset clears the accumulating ones."""
        out = np.zeros(8, np.uint64)
        N.check(self.L.lfdg_work_counters(self.h, N.ptr(out), int(reset)))
        return {"accepted": int(out[0]), "violations": int(out[1]), "refine_pixel_evals": int(out[2]),
                "refine_candidate_evals": int(out[3]), "refine_idle_slot_evals": int(out[4]),
                "sweep_samples": int(out[5])}

    # -- fusion (fusion.hpp:31-100)
    def fuse_views(self, epsilon: float, v0: int = 0, n: Optional[int] = None):
        N.check(self.L.lfdg_fuse_views(self.h, v0, self.V - v0 if n is None else n, float(epsilon)))

    def get_fused(self, view: int) -> np.ndarray:
        out = np.zeros((self.H, self.W), np.float32)
        N.check(self.L.lfdg_get_fused(self.h, view, N.ptr(out)))
        return out

    def gather_candidates(self, ref_view: int):
        """CSR (offsets [H*W+1], depths, views) in the reference's (source view, pixel) order."""
        off = np.zeros(self.H * self.W + 1, np.int32)
        total = C.c_int64()
        N.check(self.L.lfdg_gather_candidates(self.h, ref_view, N.ptr(off), None, None, 0, C.byref(total)))
        dep = np.zeros(max(total.value, 1), np.float32)
        vw = np.zeros(max(total.value, 1), np.int32)
        N.check(self.L.lfdg_gather_candidates(self.h, ref_view, N.ptr(off), N.ptr(dep), N.ptr(vw), total.value,
                                              C.byref(total)))
        return off, dep[:total.value], vw[:total.value]

    def min_nb_sim(self, view: int) -> np.ndarray:
        gw, gh, _ = self.grid_shape(view)
        out = np.zeros(gw * gh, np.float32)
        N.check(self.L.lfdg_get_min_nb_sim(self.h, view, N.ptr(out)))
        return out


# ----------------------------------------------------------------------------- reference-shaped API

_CTX_CACHE: dict = {}


def _context_for(mvs: MultiViewSet, device: int = 0) -> DeviceContext:
    """One resident device copy per MultiViewSet object (re-uploaded if the object changed)."""
    key = id(mvs)
    ent = _CTX_CACHE.get(key)
    if ent is not None and ent[0] is mvs and ent[2] == (mvs.images.ctypes.data, mvs.images.shape):
        return ent[1]
    ctx = DeviceContext(device)
    ctx.set_views(mvs.images, mvs.camera_array(), mvs.range)
    _CTX_CACHE[key] = (mvs, ctx, (mvs.images.ctypes.data, mvs.images.shape))
    return ctx


def _install_grids(ctx: DeviceContext, grids: Sequence[SuperpixelGrid]):
    for v, g in enumerate(grids):
        ctx.set_grid(v, g.cell_size, g.label_map)


def stability_fuse(offsets: np.ndarray, depths: np.ndarray, views: np.ndarray, epsilon: float,
                   device: int = 0) -> np.ndarray:
    """fusion.hpp:65 — fused depth per pixel of CSR candidate lists (offsets [n+1])."""
    offsets = np.ascontiguousarray(offsets, np.int32)
    depths = np.ascontiguousarray(depths, np.float32)
    views = np.ascontiguousarray(views, np.int32)
    out = np.zeros(len(offsets) - 1, np.float32)
    N.check(N.lib().lfdg_stability_fuse(device, len(offsets) - 1, N.ptr(offsets), N.ptr(depths), N.ptr(views),
                                        float(epsilon), N.ptr(out)))
    return out


def fuse_all(mvs: MultiViewSet, depth_maps: Sequence[np.ndarray], epsilon: float) -> List[np.ndarray]:
    """fusion.hpp:94 — stability fusion of every view's depth map (cameras from mvs)."""
    ctx = _context_for(mvs)
    for v, d in enumerate(depth_maps):
        ctx.set_depth(v, d)
    ctx.fuse_views(epsilon)
    return [ctx.get_fused(v) for v in range(mvs.num_views())]


def slic_segment(image: np.ndarray, params: SlicParams = SlicParams(), workers: int = 1,
                 device: int = 0) -> SuperpixelGrid:
    """superpixel.hpp:179 — SLIC on one [H][W][3] scaled-LAB image."""
    del workers
    image = np.ascontiguousarray(image, np.float32)
    if image.ndim != 3 or image.shape[2] != 3 or image.size == 0:
        raise InvalidParams("invalid image")
    ctx = DeviceContext(device)
    try:
        cam = PinholeCamera().as_array()[None]
        ctx.set_views(image[None], cam, (1.0, 2.0))
        ctx.slic(0, params)
        return ctx.get_grid(0)
    finally:
        ctx.close()


def sweep_view(mvs: MultiViewSet, grids: Sequence[SuperpixelGrid], view: int, params: SweepParams,
               seed: int, workers: int = 1) -> np.ndarray:
    """sweep.hpp:112 — planes [nsp, 4] of one view."""
    del workers
    ctx = _context_for(mvs)
    _install_grids(ctx, grids)
    return ctx.sweep(view, params, seed)


def rasterize(mvs: MultiViewSet, grids: Sequence[SuperpixelGrid], pm: PlaneMap) -> None:
    """sweep.hpp:44 — fills pm.depth from pm.planes for every view."""
    ctx = _context_for(mvs)
    _install_grids(ctx, grids)
    for v, planes in enumerate(pm.planes):
        ctx.set_planes(v, planes)
    ctx.rasterize()
    pm.depth = [ctx.get_depth(v) for v in range(mvs.num_views())]


def plane_sweep_init(mvs: MultiViewSet, grids: Sequence[SuperpixelGrid], params: SweepParams, seed: int,
                     workers: int = 1) -> PlaneMap:
    """sweep.hpp:141 — sweep every view, then rasterize."""
    del workers
    ctx = _context_for(mvs)
    _install_grids(ctx, grids)
    ctx.sweep_views(0, mvs.num_views(), params, seed)
    ctx.rasterize()
    return PlaneMap([ctx.get_planes(v) for v in range(mvs.num_views())],
                    [ctx.get_depth(v) for v in range(mvs.num_views())])


@dataclass
class RefineContext:  # refine.hpp:40
    mvs: MultiViewSet
    grids: Sequence[SuperpixelGrid]
    params: EnergyParams
    sweep_levels: int
    device: DeviceContext


def make_refine_context(mvs: MultiViewSet, grids: Sequence[SuperpixelGrid], params: EnergyParams,
                        sweep_levels: int) -> RefineContext:
    """refine.hpp:53 — resolves sigma/size_init and builds the static tables on the device."""
    ctx = _context_for(mvs)
    _install_grids(ctx, grids)
    sigma, size_init = ctx.make_refine_context(params, sweep_levels)
    resolved = EnergyParams(**{**params.__dict__, "sigma": sigma, "size_init": size_init})
    return RefineContext(mvs, list(grids), resolved, sweep_levels, ctx)


def refine_iteration(rctx: RefineContext, state: PlaneMap, l: int, workers: int = 1,
                     stats: Optional[RefineStats] = None) -> PlaneMap:
    """refine.hpp:253 — returns new planes (depth left empty; the caller rasterizes)."""
    del workers
    ctx = rctx.device
    for v, planes in enumerate(state.planes):
        ctx.set_planes(v, planes)
    for v, d in enumerate(state.depth):
        ctx.set_depth(v, d)
    acc, vio = ctx.refine_iteration(l, with_stats=True)
    if stats is not None:
        stats.accepted += acc
        stats.violations += vio
    return PlaneMap([ctx.get_planes(v) for v in range(rctx.mvs.num_views())], [])


def run_refinement(rctx: RefineContext, state: PlaneMap, workers: int = 1,
                   stats: Optional[RefineStats] = None) -> PlaneMap:
    """refine.hpp:325 — l = 1..iterations of refine_iteration + rasterize."""
    del workers
    for l in range(1, rctx.params.iterations + 1):
        state = refine_iteration(rctx, state, l, stats=stats)
        rasterize(rctx.mvs, rctx.grids, state)
    return state


def rgb_to_scaled_lab(rgb: np.ndarray, device: int = 0) -> np.ndarray:
    """rgb_to_scaled_lab (image.hpp:97-107) of an sRGB array [..., 3] on the GPU."""
    rgb = np.ascontiguousarray(rgb, np.float32)
    out = np.empty_like(rgb)
    N.check(N.lib().lfdg_rgb_to_scaled_lab_gpu(device, N.ptr(rgb), N.ptr(out), rgb.size // 3))
    return out


def eval_bad_pixel(gt_depth: np.ndarray, cams: np.ndarray, view: int, est_depth: np.ndarray, inv_depth_tol: float,
                   thresholds, focal: float = 0.0, baseline: float = 0.0, device: int = 0, with_mask: bool = False):
    """run_pipeline's per-view evaluation (pipeline.hpp:452-466; eval.hpp) on the GPU:
    compute_nocc_mask + (disparity domain: depth_to_disparity + mark_disc | inverse depth) +
    bad_pixel_rate for each threshold and region.  Returns rates [n_thresholds][3] (nocc, all,
    disc; -1 = empty region) and optionally the Region mask."""
    gt = np.ascontiguousarray(gt_depth, np.float32)
    est = np.ascontiguousarray(est_depth, np.float32)
    cm = np.ascontiguousarray(cams, np.float64)
    V, H, W = gt.shape
    thr = np.ascontiguousarray(thresholds, np.float64)
    rates = np.zeros((len(thr), 3), np.float64)
    mask = np.zeros((H, W), np.uint8) if with_mask else None
    N.check(N.lib().lfdg_eval_bad_pixel(device, V, W, H, N.ptr(gt), N.ptr(cm), view, N.ptr(est), inv_depth_tol, focal,
                                        baseline, N.ptr(thr), len(thr), N.ptr(rates),
                                        None if mask is None else N.ptr(mask)))
    return (rates, mask) if with_mask else rates
