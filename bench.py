"""bench.py — depth-map views/s at 1920x1080 on 1..8 B200 (BASELINE.json metric).

A step is one pass of the whole hot path over the config's view set: slic_segment of every
view, sweep_view of every view, rasterize, make_refine_context and `iterations` x
(refine_iteration; rasterize) — the segment / init / refine stages of run_pipeline
(pipeline.hpp:272-397).  Default workload: BASELINE.json configs[2] (C3):
cluttered_scene(16, 1920, 1080, f=1920, B=0.04), S=16 (8160 superpixels/view), L=256,
5 iterations, all-others matching; synthetic scene rendered by the product's restatement of
the reference fixtures (byte-identical, tests/test_scene.py).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C3] [--impl ours|reference]

Multi-GPU: under torchrun (or `python bench.py --gpus N`, which starts the N ranks itself through
torch.distributed.run); views are partitioned across ranks (strong scaling of the fixed view
set) with NCCL exchanges (paper_1812_06856_b200/pipeline.py).  The default workload stays C3 at
every N, so the N=1 line of a scaling run equals the single-GPU bench; `--config C5` (64 views,
8 nearest matching views) is the view-scaling workload of BASELINE configs[4].

`--impl reference` times the reference's own CPU implementation (oracle/_ref: the unmodified
reference headers) on the host cores, on a bounded sample of the same workload per step
(see reference_sample()), and prints the same JSON line with "impl": "reference".
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "depth-map views/sec at 1920x1080 (ms/view), 1/2/4/8 B200, vs host-CPU ref"
UNIT = "views/s"

# Algorithmic FP64 operations per pair_stats pixel-evaluation (refine.hpp:132-163 main path:
# ray dot 4, division 1, s*v 2, R(s v)+t 18, u 6, w 4, visibility test 2, residual 3,
# Gaussian 2 + exp 1, two accumulations 2; a division or exp counts as one op).  DESIGN.md.
REFINE_FLOP_PER_PIXEL_EVAL = 45


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C3")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    return ap.parse_args()


# --------------------------------------------------------------------------- clocks sampler


class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.path = f"/tmp/bench_clocks_{os.getpid()}.csv"

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader",
                                          "-lms", "200", "-i", str(self.device)], stdout=open(self.path, "w"),
                                         stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        self.proc.wait()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                clk = float(parts[1].split()[0])
                mx = float(parts[2].split()[0])
            except ValueError:
                continue
            sm.append(clk)
            for name, val in zip(names, parts[5:9]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        os.unlink(self.path)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": mx, "reasons": sorted(reasons)}
        loaded = [c for c in sm if mx and c > 0.5 * mx] or sm
        return {"sm_mhz": float(np.median(loaded)), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# --------------------------------------------------------------------------- reference (CPU)


def reference_setup(cfg_name: str, workers: int) -> dict:
    """Untimed setup of the reference arm: the reference's own renderer, SLIC of every view and
    the sweep-init state (tests/golden/<cfg>_init_depths.npz, produced by the reference's
    sweep_view; absent -> fronto planes at the ground-truth centroid depth)."""
    from oracle import ref
    from paper_1812_06856_b200.scenes import CONFIGS

    c = CONFIGS[cfg_name]
    t0 = time.time()
    if c.get("rig"):  # a re-aimed rig: the product's renderer (byte-identical to the reference's fixtures)
        from paper_1812_06856_b200.scenes import render_config

        sc = render_config(cfg_name, gt=True)
    else:
        sc = ref.render_scene(c["kind"], c["n_views"], c["width"], c["height"], c["f"], c["baseline"], 0.0,
                              c["grid"])
    s = ref.Session(sc["lab"], sc["cams"], sc["range"])
    V = sc["lab"].shape[0]
    for v in range(V):
        s.slic(v, c["S"], 0.1, 10, workers)
    fx = os.path.join(ROOT, "tests", "golden", f"{cfg_name.lower()}_init_depths.npz")
    init_kind = "reference sweep_view"
    for v in range(V):
        g = s.grid(v)
        nsp = g["grid_w"] * g["grid_h"]
        planes = np.zeros((nsp, 4))
        planes[:, 3] = -1.0
        if os.path.exists(fx):
            planes[:, 0] = np.load(fx)["depths"][v]
        else:
            init_kind = "ground-truth fronto planes"
            r = g["records"]
            gt = sc["gt"][v]
            d = gt[np.clip(r["cy"].astype(int), 0, c["height"] - 1), np.clip(r["cx"].astype(int), 0, c["width"] - 1)]
            planes[:, 0] = np.clip(np.where(d > 0, d, sc["range"][1]), sc["range"][0], sc["range"][1])
        s.set_planes(v, planes)
    t = time.time()
    s.rasterize()
    t_rast = time.time() - t
    s.refine_context(c["levels"], iterations=c["iterations"], max_neighbors=c["max_neighbors"])
    nsp = s.grid(0)["grid_w"] * s.grid(0)["grid_h"]
    return dict(session=s, cfg=c, V=V, nsp=nsp, t_rast=t_rast, init_kind=init_kind, setup_s=time.time() - t0)


def reference_sample(st: dict, step: int, workers: int) -> dict:
    """One bounded sample of the workload through the reference's own code:
    slic_segment of one view (full), sweep_view's task body on n_sw superpixels of one view and
    refine_iteration's task body on n_rf tasks per iteration l (on the sweep-init state), each
    parallel over `workers` host threads with the reference's parallel_for; extrapolated to
    ms/view = T_slic + T_sweep*(nsp/n_sw) + [sum_l T_l*(V*nsp/n_rf) + (1+iters)*T_rasterize]/V."""
    s, c, V, nsp = st["session"], st["cfg"], st["V"], st["nsp"]
    rng = np.random.default_rng(1000 + step)
    view = step % V
    t = time.time()
    s.slic(view, c["S"], 0.1, 10, workers)
    t_slic = time.time() - t
    n_sw = min(nsp, max(64, 48 * workers))
    sps = rng.choice(nsp, n_sw, replace=False)
    t = time.time()
    s.sweep_sample(view, sps, c["levels"], 0.05, c["max_neighbors"], 0, workers)
    t_sw = time.time() - t
    n_rf = max(64, 64 * workers)
    t_ref = []
    for l in range(1, c["iterations"] + 1):
        tv = rng.integers(0, V, n_rf)
        ts = rng.integers(0, nsp, n_rf)
        t = time.time()
        s.refine_tasks(l, tv, ts, workers)
        t_ref.append(time.time() - t)
    ms_view = 1e3 * (t_slic + t_sw * nsp / n_sw + (sum(x * V * nsp / n_rf for x in t_ref)
                                                   + (1 + c["iterations"]) * st["t_rast"]) / V)
    return dict(ms_per_view=ms_view, t_slic=t_slic, t_sweep_sample=t_sw, t_refine_samples=t_ref, n_sweep=n_sw,
                n_refine=n_rf, wall_s=t_slic + t_sw + sum(t_ref))


def extrapolator_validation():
    """The committed check of reference_sample's estimate against full timed reference runs
    (tools/validate_cpu_extrapolation.py at C1 and C2 on a GPU box's host cores)."""
    try:
        rows = [json.loads(x) for x in open(os.path.join(ROOT, "profiles", "r2_cpu_extrapolation.log"))
                if x.startswith("{")]
        return {r["config"]: {"full_ms_per_view": r["full_ms_per_view"],
                              "estimate_over_full": r["estimate_over_full"], "workers": r["workers"]} for r in rows}
    except (OSError, ValueError, KeyError):
        return None


def cpu_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def run_reference(args, rank: int, world: int):
    if rank != 0:
        return
    from paper_1812_06856_b200.scenes import CONFIGS

    c = CONFIGS[args.config]
    workers = cpu_cores()
    st = reference_setup(args.config, workers)
    for w in range(args.warmup):
        reference_sample(st, 10_000 + w, workers)
    samples = [reference_sample(st, k, workers) for k in range(args.steps)]
    ms_view = float(np.mean([x["ms_per_view"] for x in samples]))
    value = 1e3 / ms_view
    sample_desc = (f"per step: slic_segment of 1 view, sweep_view task body on {samples[0]['n_sweep']} random "
                   f"superpixels, refine_iteration task body on {samples[0]['n_refine']} random tasks for each "
                   f"l=1..{c['iterations']} (state: {st['init_kind']}), extrapolated to all "
                   f"{st['V']}x{st['nsp']} tasks; {workers} threads")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_view * st["V"], "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(args.config, args.gpus),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": workers, "kind": "reference", "sample": sample_desc},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "reference_detail": {"ms_per_view": ms_view, "setup_s": st["setup_s"],
                             "extrapolator_validation": extrapolator_validation(),
                             "samples": [{k: v for k, v in x.items()} for x in samples]},
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------- ours (GPU)


def workload_config(name: str, gpus: int) -> dict:
    from paper_1812_06856_b200.scenes import CONFIGS

    c = CONFIGS[name]
    V = c["grid"][0] * c["grid"][1] if c["grid"][0] else c["n_views"]
    rig = (f" ({c['grid'][0]}x{c['grid'][1]} grid rig)" if c["grid"][0] else
           " (converging rig: toed-in +-4.2 deg, rolled +-0.5 deg, skewed K)" if c.get("rig") == "converging" else
           " (linear rig)")
    return {"workload": f"{name}: cluttered_scene {V} views {c['width']}x{c['height']}" + rig
                        + f", S={c['S']}, L={c['levels']}, {c['iterations']} refine iterations, "
                        + ("all-others matching" if c["max_neighbors"] == 0 else f"{c['max_neighbors']} nearest views"),
            "views": V, "width": c["width"], "height": c["height"], "superpixel_size": c["S"],
            "levels": c["levels"], "iterations": c["iterations"], "max_neighbors": c["max_neighbors"],
            "parallelism": f"view-partition x{gpus}",
            "l2_policy": "inputs larger than L2 (LAB images alone are V x 33 MB)"}


def _all_reduce(t, op=None):
    """all_reduce that also works on a gloo group (host copy of a device tensor)."""
    import torch.distributed as dist

    op = dist.ReduceOp.SUM if op is None else op
    if t.is_cuda and dist.get_backend() == "gloo":
        h = t.cpu()
        dist.all_reduce(h, op=op)
        t.copy_(h)
    else:
        dist.all_reduce(t, op=op)


def run_ours(args, rank: int, world: int, local_rank: int):
    import torch
    import torch.distributed as dist

    from paper_1812_06856_b200 import _native as N
    from paper_1812_06856_b200 import scenes
    from paper_1812_06856_b200.api import EnergyParams, SlicParams, SweepParams
    from paper_1812_06856_b200.pipeline import HotPath, HotPathConfig

    dev = local_rank % max(1, torch.cuda.device_count())
    torch.cuda.set_device(dev)
    c = scenes.CONFIGS[args.config]
    threads = max(1, cpu_cores() // max(1, int(os.environ.get("LOCAL_WORLD_SIZE", world))))
    sc = scenes.render_config(args.config, threads=threads, gt=False, rgb=not args.no_e2e)
    V = sc["lab"].shape[0]
    cfg = HotPathConfig(SlicParams(c["S"], 0.1, 10), SweepParams(c["levels"], 0.05, c["max_neighbors"]),
                        EnergyParams(iterations=c["iterations"], max_neighbors=c["max_neighbors"]), seed=0)
    group = dist.group.WORLD if world > 1 else None
    hp = HotPath(dev, sc["lab"], sc["cams"], sc["range"], cfg, group=group)
    stream = hp.stream

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        hp.run()
    barrier()
    hp.ctx.work_counters(reset=True)
    launches0 = hp.ctx.launch_count()
    sampler = ClockSampler(dev)
    sampler.start()
    ev_refine = []
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    # Timed region: K device-resident steps.  Refine kernels are bracketed by events on the
    # same stream for the roofline (their launch count is known: one per iteration).
    orig_refine = hp.ctx.refine_iteration

    def timed_refine(l, with_stats=True):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        r = orig_refine(l, with_stats=with_stats)
        b.record(stream)
        ev_refine.append((a, b))
        return r

    hp.ctx.refine_iteration = timed_refine
    e0.record(stream)
    for _ in range(args.steps):
        hp.run()
    e1.record(stream)
    barrier()
    clocks = sampler.stop()
    hp.ctx.refine_iteration = orig_refine
    launches = hp.ctx.launch_count() - launches0
    ms_total = e0.elapsed_time(e1)
    refine_ms = sum(a.elapsed_time(b) for a, b in ev_refine)
    wc = hp.ctx.work_counters(reset=True)
    pix_evals, cand_evals, sweep_samples = wc["refine_pixel_evals"], wc["refine_candidate_evals"], wc["sweep_samples"]
    t = torch.tensor([ms_total, refine_ms], device=f"cuda:{dev}", dtype=torch.float64)
    if world > 1:
        _all_reduce(t, op=dist.ReduceOp.MAX)
        pe = torch.tensor([pix_evals, sweep_samples], device=f"cuda:{dev}", dtype=torch.float64)
        _all_reduce(pe)
        pix_evals, sweep_samples = int(pe[0].item()), int(pe[1].item())
    ms_total, refine_ms = float(t[0]), float(t[1])
    ms_step = ms_total / args.steps
    value = V * args.steps / (ms_total / 1e3)

    # ---- end to end: pinned host images in, planes + depth out, every step
    e2e = None
    if not args.no_e2e:
        pin = torch.empty(sc["lab"].size, dtype=torch.float32, pin_memory=True)
        host_imgs = pin.numpy().reshape(sc["lab"].shape)
        host_imgs[...] = sc["lab"]
        nsp = hp.ctx.grid_shape(0)[0] * hp.ctx.grid_shape(0)[1]
        planes_pin = torch.empty(hp.n * nsp * 4, dtype=torch.float64, pin_memory=True).numpy()
        depth_pin = torch.empty(hp.n * c["height"] * c["width"], dtype=torch.float32, pin_memory=True).numpy()
        barrier()
        f0 = torch.cuda.Event(enable_timing=True)
        f1 = torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        for _ in range(args.steps):
            hp.upload(host_imgs)
            hp.run()
            hp.download(planes_pin, depth_pin, sync=False)
        f1.record(stream)
        torch.cuda.synchronize()
        te = torch.tensor([f0.elapsed_time(f1)], device=f"cuda:{dev}", dtype=torch.float64)
        if world > 1:
            _all_reduce(te, op=dist.ReduceOp.MAX)
        e2e = {"value": V * args.steps / (float(te[0]) / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": int(host_imgs.nbytes),
               "d2h_bytes_per_step": int(planes_pin.nbytes + depth_pin.nbytes) * world,
               "ms_per_step": float(te[0]) / args.steps,
               "mode": "serial: upload, run, download on one stream"}
        # pipelined: step k+1's upload and step k's download run on a copy stream under the compute
        # (lfdg_prefetch_images / lfdg_commit_images / lfdg_download_results_async); every step's
        # H2D and D2H is still inside the timed region
        barrier()
        f0.record(stream)
        hp.prefetch(host_imgs)
        for k in range(args.steps):
            hp.commit()
            if k + 1 < args.steps:
                hp.prefetch(host_imgs)
            hp.run()
            hp.download_async(planes_pin, depth_pin)
        hp.wait_downloads()
        f1.record(stream)
        torch.cuda.synchronize()
        te = torch.tensor([f0.elapsed_time(f1)], device=f"cuda:{dev}", dtype=torch.float64)
        if world > 1:
            _all_reduce(te, op=dist.ReduceOp.MAX)
        e2e["pipelined"] = {"value": V * args.steps / (float(te[0]) / 1e3), "unit": UNIT,
                            "h2d_bytes_per_step": int(host_imgs.nbytes),
                            "d2h_bytes_per_step": int(planes_pin.nbytes + depth_pin.nbytes) * world,
                            "ms_per_step": float(te[0]) / args.steps,
                            "mode": "step k+1 upload / step k download on a copy stream under the compute"}
        # the same from sRGB host images: rgb_to_scaled_lab runs on the GPU (lfdg_upload_rgb) instead
        # of the reference's host pre-pass (pipeline.hpp:245)
        host_imgs[...] = sc["rgb"]
        barrier()
        f0.record(stream)
        for _ in range(args.steps):
            hp.upload_rgb(host_imgs)
            hp.run()
            hp.download(planes_pin, depth_pin, sync=False)
        f1.record(stream)
        torch.cuda.synchronize()
        te = torch.tensor([f0.elapsed_time(f1)], device=f"cuda:{dev}", dtype=torch.float64)
        if world > 1:
            _all_reduce(te, op=dist.ReduceOp.MAX)
        e2e["from_srgb"] = {"value": V * args.steps / (float(te[0]) / 1e3), "unit": UNIT,
                            "h2d_bytes_per_step": int(host_imgs.nbytes), "ms_per_step": float(te[0]) / args.steps}

    if rank != 0:
        return
    peak = ctypes_fp64_peak(dev)
    peak32 = ctypes_fp32_peak(dev)
    refine_launches = args.steps * c["iterations"]
    achieved = pix_evals * REFINE_FLOP_PER_PIXEL_EVAL / (refine_ms / 1e3) / 1e12
    traffic, traffic_note = refine_traffic()
    roofline = {"bound": "fp64", "kernel": "k_refine (refine_iteration)", "achieved": achieved,
                "peak": peak / 1e12, "unit": "TFLOP/s", "frac": achieved / (peak / 1e12),
                "peak_source": "measured DFMA stream on this GPU (lfdg_selftest_fp64_peak)",
                "traffic": traffic, "traffic_source": traffic_note,
                "per_launch": {"pixel_evals": pix_evals / refine_launches,
                               "flop": pix_evals * REFINE_FLOP_PER_PIXEL_EVAL / refine_launches,
                               "ms": refine_ms / refine_launches},
                "share_of_step": refine_ms / ms_total}
    step_roof = step_roofline(c, V, args.steps, ms_total, pix_evals, sweep_samples, peak, peak32)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_step, "ms_per_view": ms_step / V, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": workload_config(args.config, world),
        "roofline": roofline, "step_roofline": step_roof, "clocks": clocks, "gpu_launches": launches, "e2e": e2e,
    }
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(args.config)
    print(json.dumps(line), flush=True)


def refine_traffic():
    """DRAM bytes (read + write) of one k_refine launch from the committed ncu --set full capture
    (profiles/r2_traffic.json), used only when that capture was taken of the refine.cu being
    benched (sha256 recorded beside it); else (None, reason)."""
    import hashlib

    try:
        with open(os.path.join(ROOT, "profiles", "r2_traffic.json")) as f:
            rec = json.load(f)["k_refine"]
        src = os.path.join(ROOT, "paper_1812_06856_b200", "csrc", "refine.cu")
        sha = hashlib.sha256(open(src, "rb").read()).hexdigest()
        if rec.get("refine_cu_sha256") != sha:
            return None, "profiles/r2_traffic.json was captured from a different refine.cu"
        return rec["dram_bytes_per_launch"], f"ncu --set full of this refine.cu ({rec.get('capture', '')})"
    except (OSError, KeyError, ValueError):
        return None, "no committed ncu capture"


# Algorithmic work per unit, the step-level roofline's numerators: a division,
# square root or exp counts as one operation.
SWEEP_FP64_PER_SAMPLE = 10   # hx (5), u = hx / z by reciprocal + Markstein (3), fx = u - x0 (1), cost += (1)
SWEEP_FP32_PER_SAMPLE = 36   # bilinear 27, color_dist2 8, tssd min 1
SLIC_FP64_PER_CENTRE = 6     # ddx, ddy, ddx^2 + ddy^2 (3), sqrt
SLIC_FP32_PER_CENTRE = 11    # color_dist2 8, sqrtf, d = dc + w ds (2)
SLIC_CENTRES = 25            # the +-2 cell window of the assign loop (superpixel.hpp:221-244)
SLIC_BYTES_PER_PX_ITER = 20  # LAB float4 read + label write
RAST_BYTES_PER_PX = 8        # label read + depth write (rasterize)
BUILD_RASTER_BYTES_PER_PX = 24  # label + depth read, 16-byte gather record written


def step_roofline(c, V, steps, ms_total, pix_evals, sweep_samples, p64, p32):
    """Sum over the step's kernels of T_roof,k = max(bytes / HBM, FP64 / P64, FP32 / P32) divided by
    the measured step time; peaks: HBM from MEASURED_PEAKS.json, FP64 / FP32 measured
    live by lfdg_selftest_fp64_peak / fp32_peak."""
    try:
        hbm = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] * 1e9
        hbm_src = "MEASURED_PEAKS.json hbm_gbs"
    except (OSError, KeyError, ValueError):
        hbm, hbm_src = 6.65e12, "fallback 6.65 TB/s (B200_PROFILING.md)"
    px = V * c["width"] * c["height"]
    it = c["iterations"]
    slic_centre_evals = px * 10 * SLIC_CENTRES
    t = {
        "k_refine": pix_evals / steps * REFINE_FLOP_PER_PIXEL_EVAL / p64,
        "k_sweep": max(sweep_samples / steps * SWEEP_FP64_PER_SAMPLE / p64,
                       sweep_samples / steps * SWEEP_FP32_PER_SAMPLE / p32),
        "slic": max(slic_centre_evals * SLIC_FP64_PER_CENTRE / p64, slic_centre_evals * SLIC_FP32_PER_CENTRE / p32,
                    px * 10 * SLIC_BYTES_PER_PX_ITER / hbm),
        "k_rasterize": (1 + it) * px * RAST_BYTES_PER_PX / hbm,
        "k_build_raster": it * px * BUILD_RASTER_BYTES_PER_PX / hbm,
    }
    t_ms = {k: v * 1e3 for k, v in t.items()}
    ms_step = ms_total / steps
    return {"t_roof_ms": t_ms, "sum_t_roof_ms": sum(t_ms.values()), "t_step_ms": ms_step,
            "frac": sum(t_ms.values()) / ms_step,
            "counts_per_step": {"refine_pixel_evals": pix_evals / steps, "sweep_samples": sweep_samples / steps,
                                "slic_centre_tests_bound": slic_centre_evals},
            "peaks": {"fp64_tflops": p64 / 1e12, "fp32_tflops": p32 / 1e12, "hbm_gbs": hbm / 1e9,
                      "sources": "fp64/fp32 measured live (DFMA/FFMA streams); " + hbm_src}}


def ctypes_fp32_peak(dev: int) -> float:
    import ctypes

    from paper_1812_06856_b200 import _native as N

    out = ctypes.c_double()
    N.check(N.lib().lfdg_selftest_fp32_peak(dev, ctypes.byref(out)))
    return out.value


def ctypes_fp64_peak(dev: int) -> float:
    import ctypes

    from paper_1812_06856_b200 import _native as N

    out = ctypes.c_double()
    N.check(N.lib().lfdg_selftest_fp64_peak(dev, ctypes.byref(out)))
    return out.value


def cpu_baseline(cfg_name: str) -> dict:
    """The reference (oracle/_ref) on a bounded sample of the same workload, rank 0, N=1."""
    try:
        from oracle import ref

        if not ref.available():
            return {"value": None, "unit": UNIT, "cores": 0, "kind": "reference",
                    "sample": "unavailable: oracle/_ref/liblfdref.so not built"}
        workers = cpu_cores()
        st = reference_setup(cfg_name, workers)
        smp = reference_sample(st, 0, workers)
        return {"value": 1e3 / smp["ms_per_view"], "unit": UNIT, "cores": workers, "kind": "reference",
                "sample": (f"slic_segment 1 view + sweep_view task body on {smp['n_sweep']} superpixels + "
                           f"refine task body on {smp['n_refine']} tasks x l=1..{st['cfg']['iterations']} "
                           f"({st['init_kind']} state), extrapolated; {smp['wall_s']:.1f} s of CPU work"),
                "ms_per_view": smp["ms_per_view"]}
    except Exception as e:  # the baseline is reported, never required
        return {"value": None, "unit": UNIT, "cores": 0, "kind": "reference", "sample": f"failed: {e}"}


def free_port() -> int:
    import socket

    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)  # rank 0 alone runs the host-CPU reference
        return
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        # `python bench.py --gpus N` without a launcher: start the N ranks (one process per GPU)
        # through torch.distributed.run, exactly as the driver's torchrun launch does.
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr=127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__), *sys.argv[1:]]
        sys.exit(subprocess.run(cmd).returncode)
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; launch one rank per GPU")
    if world > 1:
        import torch
        import torch.distributed as dist

        # NCCL over NVLink; LFDG_BENCH_BACKEND=gloo runs the same ranks through host collectives
        # (tests: several ranks sharing one GPU, where NCCL refuses duplicate devices)
        backend = os.environ.get("LFDG_BENCH_BACKEND", "nccl")
        dev = local_rank % max(1, torch.cuda.device_count())
        torch.cuda.set_device(dev)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{dev}"))
        else:
            dist.init_process_group(backend)
    try:
        run_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()


if __name__ == "__main__":
    main()
