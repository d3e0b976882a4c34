"""Run directory driver: the stage flow of run_pipeline (pipeline.hpp:230-498) over the
device-resident hot path, with the reference's artefacts and ``resume`` semantics.

Every stage runs on the GPU through DeviceContext (no host compute); this module only decides
what to compute versus reload and writes the files (artifacts.py) the reference writes:

* segment  — ``labels_v<v>.png`` + ``superpixels_v<v>.txt``; on resume the label PNG is reloaded
  and the grid statistics recomputed on the device (grid_from_labels, pipeline.hpp:187-228);
* init     — ``planes_v<v>_stage1.txt`` (hexfloat, bit-exact resume), ``depth_v<v>_stage1.{pfm,png}``;
* refine   — ``planes_v<v>_stage2.txt``, ``depth_v<v>_stage2.{pfm,png}``, with ``dump_every``
  intermediate ``depth_v<v>_stage2_iter<l>.{pfm,png}``; resumed when every view's stage-2 planes
  exist;
* fuse     — ``depth_v<v>_stage3.{pfm,png}``; resumed from the PFMs only when ``fuse`` itself is
  not selected (pipeline.hpp:402);
* ``timings.tsv`` and ``stats.jsonl`` (appended on resume).

``eval`` is accepted as a stage name (it pulls in ``fuse`` as in the reference) but the
ground-truth comparison itself needs the dataset manifest and is the caller's (api.eval_*).
Errors keep the reference's classes: a missing persisted product for an unselected stage is
InvalidParams; anything else raised inside a stage (e.g. a ParseError from a corrupt persisted
file) surfaces as a PipelineError naming the stage and view, as the reference's ``guard`` does.
"""
from __future__ import annotations

import contextlib
import os
import time
from dataclasses import dataclass, field
from typing import List, Sequence

import numpy as np

from . import artifacts as art
from .api import DeviceContext, EnergyParams, InvalidParams, SlicParams, SweepParams

STAGE_ORDER = ("segment", "init", "refine", "fuse", "eval")  # pipeline.hpp:25-28


class PipelineError(RuntimeError):  # pipeline.hpp:22
    pass


@contextlib.contextmanager
def _guard(stage: str, view: int = -1):
    """pipeline.hpp:259-270: configuration errors keep their type; anything else becomes a
    PipelineError naming the stage (and view)."""
    try:
        yield
    except (PipelineError, InvalidParams):
        raise
    except Exception as e:  # noqa: BLE001 — the reference catches std::exception
        raise PipelineError("stage %s%s: %s" % (stage, " (view %d)" % view if view >= 0 else "", e)) from e


@dataclass
class PipelineConfig:  # pipeline.hpp:30-66 (the manifest is replaced by in-memory views)
    out_dir: str = ""
    slic: SlicParams = field(default_factory=SlicParams)
    sweep: SweepParams = field(default_factory=SweepParams)
    energy: EnergyParams = field(default_factory=EnergyParams)
    fusion_epsilon: float = 0.0  # 0 = sweep inverse-depth step
    seed: int = 0
    resume: bool = False
    dump_every: int = 0
    stages: List[str] = field(default_factory=lambda: list(STAGE_ORDER))

    def validate(self) -> None:  # pipeline.hpp:43-56, before any file I/O
        if not self.out_dir:
            raise InvalidParams("output directory required")
        if self.fusion_epsilon < 0 or self.dump_every < 0:
            raise InvalidParams("bad pipeline params")
        if not self.stages:
            raise InvalidParams("no stages selected")
        for s in self.stages:
            if s not in STAGE_ORDER:
                raise InvalidParams("unknown stage: " + s)
        self.slic.validate()
        self.sweep.validate()
        self.energy.validate()

    def has_stage(self, name: str) -> bool:
        return name in self.stages


def _range_ok(d_range) -> None:
    if not (0 < d_range[0] < d_range[1]):
        raise InvalidParams("invalid depth range")


def run_pipeline(images_lab: np.ndarray, cams: np.ndarray, d_range: Sequence[float], config: PipelineConfig,
                 device: int = 0) -> dict:
    """images_lab: scaled LAB [V][H][W][3] f32 (rgb_to_scaled_lab of the manifest images).
    Returns {"grids", "init_planes", "refined_planes", "depth_init", "depth_refined", "fused",
    "timings"}; entries of stages that did not run are None."""
    config.validate()
    _range_ok(d_range)
    d = config.out_dir
    os.makedirs(d, exist_ok=True)
    V, H, W = images_lab.shape[:3]
    L = config.sweep.levels
    sweep_step = (1.0 / d_range[0] - 1.0 / d_range[1]) / (L - 1) if L > 1 else 0.0  # sweep.hpp:38-40
    epsilon = config.fusion_epsilon if config.fusion_epsilon > 0 else sweep_step
    timings: List[tuple] = []
    out = {k: None for k in ("grids", "init_planes", "refined_planes", "depth_init", "depth_refined", "fused")}
    stats = art.StatsLog(d, resume=config.resume)
    ctx = DeviceContext(device)
    try:
        ctx.set_views(images_lab, cams, d_range)

        def ms_since(t0):
            ctx.synchronize()
            return (time.perf_counter() - t0) * 1e3

        def write_depth(view, depth, base):
            art.write_pfm(depth, os.path.join(d, base + ".pfm"))
            art.write_depth_png(depth, d_range[0], d_range[1], os.path.join(d, base + ".png"))

        # ---------------------------------------------------------------- segment
        if any(config.has_stage(s) for s in ("segment", "init", "refine", "fuse")):
            grids = []
            for v in range(V):
                with _guard("segment", v):
                    png = art.labels_path(d, v)
                    t0 = time.perf_counter()
                    if config.resume and os.path.exists(png):
                        labels, w, h = art.read_label_png(png)
                        if (w, h) != (W, H):
                            raise art.ParseError("persisted label map size mismatch")
                        gw = (W + config.slic.size - 1) // config.slic.size
                        gh = (H + config.slic.size - 1) // config.slic.size
                        if labels.size and labels.max() >= gw * gh:
                            raise art.ParseError("label map does not fit the configured grid")
                        ctx.set_grid(v, config.slic.size, labels)
                        grids.append(ctx.get_grid(v))
                    else:
                        if not config.has_stage("segment"):
                            raise InvalidParams("segment stage not selected and no persisted labels found")
                        ctx.slic(v, config.slic)
                        g = ctx.get_grid(v)
                        grids.append(g)
                        art.write_label_png(g.label_map, W, H, png)
                        art.write_superpixel_stats(g.sp, art.superpixels_path(d, v))
                    timings.append(("segment", v, ms_since(t0)))
                    stats.segment(v, grids[-1].num_superpixels())
            out["grids"] = grids

        # ------------------------------------------------------------------- init
        if config.has_stage("init") or config.has_stage("refine"):
            init = []
            for v in range(V):
                with _guard("init", v):
                    path = art.planes_path(d, v, 1)
                    t0 = time.perf_counter()
                    if config.resume and os.path.exists(path):
                        p = art.read_planes(path)
                        if p.shape[0] != out["grids"][v].num_superpixels():
                            raise art.ParseError("persisted plane count mismatch")
                        ctx.set_planes(v, p)
                    else:
                        if not config.has_stage("init"):
                            raise InvalidParams("init stage not selected and no persisted planes found")
                        p = ctx.sweep(v, config.sweep, config.seed)
                        art.write_planes(p, path)
                    init.append(p)
                    timings.append(("init", v, ms_since(t0)))
            with _guard("init"):
                ctx.rasterize()
                out["init_planes"] = init
                out["depth_init"] = [ctx.get_depth(v) for v in range(V)]
                for v in range(V):
                    write_depth(v, out["depth_init"][v], "depth_%s_stage1" % art.view_tag(v))
                    stats.init(v, L)

        # ----------------------------------------------------------------- refine
        if config.has_stage("refine") or config.has_stage("fuse"):
            resumed = False
            if config.resume and all(os.path.exists(art.planes_path(d, v, 2)) for v in range(V)):
                with _guard("refine"):
                    refined = []
                    for v in range(V):
                        p = art.read_planes(art.planes_path(d, v, 2))
                        if p.shape[0] != out["grids"][v].num_superpixels():
                            raise art.ParseError("persisted plane count mismatch")
                        ctx.set_planes(v, p)
                        refined.append(p)
                    ctx.rasterize()
                resumed = True
            if not resumed:
                if not config.has_stage("refine"):
                    raise InvalidParams("refine stage not selected and no persisted planes found")
                with _guard("refine"):
                    t0 = time.perf_counter()
                    ctx.make_refine_context(config.energy, L)
                    iters = config.energy.iterations
                    for l in range(1, iters + 1):
                        ctx.refine_iteration(l, with_stats=False)
                        ctx.rasterize()
                        if config.dump_every > 0 and l % config.dump_every == 0 and l != iters:
                            for v in range(V):
                                write_depth(v, ctx.get_depth(v), "depth_%s_stage2_iter%d" % (art.view_tag(v), l))
                    total = ms_since(t0)
                    timings.extend(("refine", v, total / V) for v in range(V))  # pipeline.hpp:383-385
                    refined = [ctx.get_planes(v) for v in range(V)]
                    for v in range(V):
                        art.write_planes(refined[v], art.planes_path(d, v, 2))
            out["refined_planes"] = refined
            out["depth_refined"] = [ctx.get_depth(v) for v in range(V)]
            if not resumed:
                with _guard("refine"):
                    for v in range(V):
                        write_depth(v, out["depth_refined"][v], "depth_%s_stage2" % art.view_tag(v))
                        stats.refine(v, config.energy.iterations)

        # ------------------------------------------------------------------- fuse
        if config.has_stage("fuse") or config.has_stage("eval"):
            resumed = False
            if config.resume and not config.has_stage("fuse") and all(
                    os.path.exists(art.depth_path(d, v, 3)) for v in range(V)):
                with _guard("fuse"):
                    out["fused"] = [art.read_pfm(art.depth_path(d, v, 3)) for v in range(V)]
                resumed = True
            if not resumed:
                if not config.has_stage("fuse"):
                    raise InvalidParams("fuse stage not selected and no persisted fused maps found")
                fused = []
                for v in range(V):
                    with _guard("fuse", v):
                        t0 = time.perf_counter()
                        ctx.fuse_views(epsilon, v, 1)
                        fused.append(ctx.get_fused(v))
                        timings.append(("fuse", v, ms_since(t0)))
                        write_depth(v, fused[v], "depth_%s_stage3" % art.view_tag(v))
                        stats.fuse(v, epsilon)
                out["fused"] = fused
    finally:
        stats.close()
        ctx.close()
    art.write_timings(timings, os.path.join(d, "timings.tsv"))
    out["timings"] = timings
    return out
