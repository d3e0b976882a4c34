"""GPU evaluation (eval.hpp): compute_nocc_mask, depth_to_disparity,
mark_disc and bad_pixel_rate as run_pipeline reports them (pipeline.hpp:452-466), against the
reference (oracle/_ref ref_bad_pixel_rate) — every region and threshold, disparity and inverse
depth domains, on rendered ground truth with perturbed / invalid estimates, rates equal to the
last bit."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("kind,grid", [("cluttered", (0, 0)), ("occluder", (0, 0)), ("cluttered", (2, 2))])
def test_eval_matches_reference(ref, kind, grid):
    from paper_1812_06856_b200 import api

    sc = ref.render_scene(kind, 3, 200, 150, 200.0, 0.1, grid=grid)
    gt, cams = sc["gt"], sc["cams"]
    rng = np.random.default_rng(4)
    step = (1.0 / sc["range"][0] - 1.0 / sc["range"][1]) / 31
    for view in range(gt.shape[0]):
        est = (gt[view] * rng.uniform(0.97, 1.03, gt[view].shape)).astype(np.float32)
        flat = est.reshape(-1)
        idx = rng.choice(flat.size, 300, replace=False)
        flat[idx[:100]] = 0.0
        flat[idx[100:200]] = np.nan
        flat[idx[200:]] = np.inf
        for focal, baseline, thr in ((200.0, 0.1, (0.5, 1.0, 2.0)), (0.0, 0.0, (step, 2 * step, 4 * step))):
            got = api.eval_bad_pixel(gt, cams, view, est, 2 * step, thr, focal, baseline)
            for ti, t in enumerate(thr):
                for region in (0, 1, 2):
                    want = ref.bad_pixel_rate(gt, cams, view, est, 2 * step, focal, baseline, region, t)
                    assert got[ti, region] == want, (kind, grid, view, focal, t, region, got[ti, region], want)
