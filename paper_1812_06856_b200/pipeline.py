"""Device-resident orchestration of the hot path (the segment / init / refine stages of
run_pipeline, pipeline.hpp:272-397), single- or multi-GPU.

Multi-GPU: one process per GPU; views are partitioned into contiguous blocks,
source images are replicated, every rank segments / sweeps / refines only its own views, and
the per-view products other ranks read are exchanged with torch.distributed (NCCL over NVLink):
  * once after SLIC: label maps, superpixel records, member CSR and centroid rays;
  * after the sweep and after every refine_iteration: the per-superpixel planes (32 B each).
Every rank then rasterizes every view locally.  rasterize is deterministic and the refinement
is a Jacobi update, so the result is bit-identical for any GPU count.  The exchanges are in
place on the context's own all-view buffers (zero-copy tensors over the device pointers).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Optional, Tuple

import numpy as np

from . import _native as N
from .api import DeviceContext, EnergyParams, InvalidParams, SlicParams, SweepParams, check_images

GRID_BUFFERS = (N.BUF_LABELS, N.BUF_CX, N.BUF_CY, N.BUF_COLOR, N.BUF_COUNT, N.BUF_MOFF, N.BUF_MPIX, N.BUF_CRAY)


@dataclass
class HotPathConfig:
    slic: SlicParams = field(default_factory=SlicParams)
    sweep: SweepParams = field(default_factory=SweepParams)
    energy: EnergyParams = field(default_factory=EnergyParams)
    seed: int = 0


def partition(n_views: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous block of views owned by `rank` (sizes differ by at most one)."""
    v0 = n_views * rank // world
    v1 = n_views * (rank + 1) // world
    return v0, v1 - v0


def exchange_views(t, stride: int, n_views: int, world: int, rank: int, group=None, in_place_allgather: bool = True):
    """Make every rank's copy of an all-view buffer `t` ([n_views][stride] bytes, flat uint8)
    complete: rank r owns views partition(n_views, world, r).  Equal blocks use one in-place
    all-gather; otherwise each owner broadcasts its block."""
    import torch.distributed as dist

    if world == 1:
        return
    if t.is_cuda and dist.get_backend(group) == "gloo":
        # gloo moves host memory: stage the device buffer through the host (the CPU-collective
        # path, e.g. several ranks sharing one GPU in tests); NCCL exchanges in place on the device
        import torch

        torch.cuda.synchronize(t.device)
        h = t.cpu()
        exchange_views(h, stride, n_views, world, rank, group, in_place_allgather)
        t.copy_(h)
        torch.cuda.synchronize(t.device)
        return
    if in_place_allgather and n_views % world == 0:
        chunk = stride * (n_views // world)
        dist.all_gather_into_tensor(t, t[rank * chunk:(rank + 1) * chunk], group=group)
        return
    for r in range(world):
        v0, n = partition(n_views, world, r)
        if n:
            dist.broadcast(t[v0 * stride:(v0 + n) * stride], src=r, group=group)


class _CudaArray:
    """Minimal __cuda_array_interface__ over a raw device pointer (zero-copy torch view)."""

    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (ptr, False),
                                         "version": 3, "strides": None}


class HotPath:
    """SLIC -> sweep -> rasterize -> make_refine_context -> iterations x (refine; rasterize)."""

    def __init__(self, device: int, images: np.ndarray, cams: np.ndarray, d_range, cfg: HotPathConfig,
                 group=None, use_torch_stream: bool = True):
        self.cfg = cfg
        self.ctx = DeviceContext(device)
        self.V = images.shape[0]
        self.group = group
        if group is not None:
            import torch.distributed as dist

            self.world = dist.get_world_size(group)
            self.rank = dist.get_rank(group)
        else:
            self.world, self.rank = 1, 0
        self.v0, self.n = partition(self.V, self.world, self.rank)
        self.stream = None
        if use_torch_stream:
            # A dedicated torch stream, made current, so CUDA events, NCCL collectives and the
            # library's kernels are ordered on one non-default stream.
            import torch

            torch.cuda.set_device(device)
            self.stream = torch.cuda.Stream(device=device)
            torch.cuda.set_stream(self.stream)
            self.ctx.set_stream(self.stream.cuda_stream)
        self.ctx.set_views(images, cams, d_range)
        self.H, self.W = images.shape[1], images.shape[2]

    def _check_host_images(self, a: np.ndarray, what: str):
        check_images(a, what, self.H, self.W)
        if a.shape[0] != self.V:
            raise InvalidParams(f"{what}: every one of the {self.V} views is uploaded, got {a.shape[0]}")

    def _check_results(self, planes_host, depth_host):
        nsp = self.ctx.grid_shape(self.v0)[0] * self.ctx.grid_shape(self.v0)[1] if self.n else 0
        if planes_host is not None and (planes_host.dtype != np.float64 or planes_host.size != self.n * nsp * 4
                                        or not planes_host.flags.c_contiguous):
            raise InvalidParams(f"planes_host must be a contiguous float64 [{self.n}][{nsp}][4] array")
        if depth_host is not None and (depth_host.dtype != np.float32 or depth_host.size != self.n * self.H * self.W
                                       or not depth_host.flags.c_contiguous):
            raise InvalidParams(f"depth_host must be a contiguous float32 [{self.n}][{self.H}][{self.W}] array")

    # ---- exchange plumbing
    def _tensor(self, which: int):
        import torch

        ptr, nbytes, stride = self.ctx.device_buffer(which)
        return torch.as_tensor(_CudaArray(ptr, nbytes), device=f"cuda:{self.ctx.device}"), stride

    def _allgather(self, which: int):
        if self.stream is None:
            self.ctx.synchronize()  # the library's own stream: finish its kernels before torch reads
        t, stride = self._tensor(which)
        exchange_views(t, stride, self.V, self.world, self.rank, self.group)

    def _exchange_grids(self):
        if self.world == 1:
            return
        for which in GRID_BUFFERS:
            self._allgather(which)
        self.ctx.mark_views_ready(0, self.V, 1)

    def _exchange_planes(self):
        if self.world == 1:
            return
        self._allgather(N.BUF_PLANES)
        self.ctx.mark_views_ready(0, self.V, 2)

    # ---- the path
    def run(self, with_stats: bool = False) -> dict:
        c, cfg = self.ctx, self.cfg
        c.slic_views(self.v0, self.n, cfg.slic)
        self._exchange_grids()
        N.check(N.lib().lfdg_wait_downloads(c.h))  # a pending async download still reads planes / depth
        c.sweep_views(self.v0, self.n, cfg.sweep, cfg.seed)
        self._exchange_planes()
        c.rasterize()
        c.make_refine_context(cfg.energy, cfg.sweep.levels)
        c.set_refine_views(self.v0, self.n)
        accepted = 0
        for l in range(1, cfg.energy.iterations + 1):
            r = c.refine_iteration(l, with_stats=with_stats)
            if r is not None:
                accepted += r[0]
            self._exchange_planes()
            c.rasterize()
        return {"accepted": accepted if with_stats else None}

    # ---- end-to-end transfers
    def upload(self, images_host: np.ndarray):
        """Enqueue the H2D copy of every view's LAB image (replicated on every rank)."""
        images_host = np.ascontiguousarray(images_host, np.float32)
        self._check_host_images(images_host, "images")
        N.check(N.lib().lfdg_upload_images(self.ctx.h, 0, self.V, N.ptr(images_host)))

    def upload_rgb(self, rgb_host: np.ndarray):
        """Enqueue the H2D copy of every view's sRGB image and its conversion to scaled LAB on the
        device (rgb_to_scaled_lab, image.hpp:97-107; the reference does it on the host)."""
        rgb_host = np.ascontiguousarray(rgb_host, np.float32)
        self._check_host_images(rgb_host, "rgb images")
        N.check(N.lib().lfdg_upload_rgb(self.ctx.h, 0, self.V, N.ptr(rgb_host)))

    # ---- pipelined end-to-end transfers (copy stream next to the compute stream)
    def prefetch(self, images_host: np.ndarray):
        """Enqueue the H2D copy of every view's LAB image into the staging buffer on the copy
        stream; it overlaps the compute already enqueued.  Install it with commit()."""
        images_host = np.ascontiguousarray(images_host, np.float32)
        self._check_host_images(images_host, "images")
        N.check(N.lib().lfdg_prefetch_images(self.ctx.h, 0, self.V, N.ptr(images_host)))

    def commit(self):
        N.check(N.lib().lfdg_commit_images(self.ctx.h))

    def download_async(self, planes_host: Optional[np.ndarray], depth_host: Optional[np.ndarray]):
        """D2H of this rank's planes / depth on the copy stream, overlapping the next step's SLIC
        (run() makes the next sweep wait for it)."""
        self._check_results(planes_host, depth_host)
        N.check(N.lib().lfdg_download_results_async(self.ctx.h, self.v0, self.n,
                                                    None if planes_host is None else N.ptr(planes_host),
                                                    None if depth_host is None else N.ptr(depth_host)))

    def wait_downloads(self):
        N.check(N.lib().lfdg_wait_downloads(self.ctx.h))

    def upload_rgb8(self, rgb8_host: np.ndarray):
        """Enqueue the H2D copy of every view's 8-bit sRGB image (a decoded image file, 1 B per
        channel) and its conversion to scaled LAB on the device (read_image + rgb_to_scaled_lab)."""
        rgb8_host = np.ascontiguousarray(rgb8_host, np.uint8)
        self._check_host_images(rgb8_host, "rgb8 images")
        N.check(N.lib().lfdg_upload_rgb8(self.ctx.h, 0, self.V, N.ptr(rgb8_host)))

    def download(self, planes_host: Optional[np.ndarray], depth_host: Optional[np.ndarray], sync: bool = True):
        """Enqueue the D2H copy of this rank's views' planes [n][nsp][4] and depth [n][H][W]."""
        self._check_results(planes_host, depth_host)
        N.check(N.lib().lfdg_download_results(self.ctx.h, self.v0, self.n,
                                              None if planes_host is None else N.ptr(planes_host),
                                              None if depth_host is None else N.ptr(depth_host), int(sync)))

    def close(self):
        self.ctx.close()


def estimate_depth(images: np.ndarray, cams: np.ndarray, d_range, cfg: HotPathConfig = HotPathConfig(),
                   device: int = 0) -> Tuple[List[np.ndarray], np.ndarray]:
    """One-shot public entry: LAB images [V][H][W][3] (host) -> (planes per view, depth [V][H][W])."""
    hp = HotPath(device, images, cams, d_range, cfg, use_torch_stream=False)
    try:
        hp.run()
        nsp = hp.ctx.grid_shape(0)[0] * hp.ctx.grid_shape(0)[1]
        planes = np.zeros((hp.V, nsp, 4), np.float64)
        depth = np.zeros(images.shape[:3], np.float32)
        hp.download(planes, depth, sync=True)
        return list(planes), depth
    finally:
        hp.close()
