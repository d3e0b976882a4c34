"""run_pipeline's run directory (paper_1812_06856_b200/run.py): the stage products written to
disk equal the reference's (the frozen C1 golden of tests/golden/make_c1_golden.py), and every
resume path — labels from the 16-bit PNG, planes from the hexfloat files, fused maps from the
PFMs — reproduces the uninterrupted run bit for bit (pipeline.hpp:272-432, acceptance's resume
criterion)."""
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "c1_golden.npz")


def _cfg(out_dir, **kw):
    from paper_1812_06856_b200 import api
    from paper_1812_06856_b200.run import PipelineConfig

    return PipelineConfig(out_dir=str(out_dir), slic=api.SlicParams(12, 0.1, 10), sweep=api.SweepParams(32, 0.05, 0),
                          energy=api.EnergyParams(iterations=3), seed=0, **kw)


@pytest.fixture(scope="module")
def c1():
    from paper_1812_06856_b200 import scenes

    return scenes.render_config("C1")


@pytest.fixture(scope="module")
def full_run(c1, tmp_path_factory):
    from paper_1812_06856_b200.run import run_pipeline

    d = tmp_path_factory.mktemp("run")
    res = run_pipeline(c1["lab"], c1["cams"], c1["range"], _cfg(d, dump_every=1))
    return d, res


def _bits(a):
    return np.ascontiguousarray(a).view(np.uint64 if a.dtype == np.float64 else np.uint32)


def test_run_dir_products_equal_reference_golden(full_run):
    from paper_1812_06856_b200 import artifacts as art

    d, res = full_run
    g = np.load(GOLDEN)
    for v in range(3):
        labels, w, h = art.read_label_png(art.labels_path(str(d), v))
        assert (w, h) == (320, 240) and np.array_equal(labels, g[f"labels{v}"].reshape(-1))
        assert np.array_equal(_bits(art.read_planes(art.planes_path(str(d), v, 1))), _bits(g[f"sweep{v}"]))
        assert np.array_equal(_bits(art.read_planes(art.planes_path(str(d), v, 2))), _bits(g[f"refine3_{v}"]))
        assert np.array_equal(_bits(art.read_pfm(art.depth_path(str(d), v, 2))), _bits(g[f"depth{v}"]))
        assert np.array_equal(_bits(art.read_pfm(art.depth_path(str(d), v, 3))), _bits(res["fused"][v]))
        for l in (1, 2):  # dump_every = 1: every iteration but the last
            assert os.path.exists(os.path.join(str(d), "depth_v%d_stage2_iter%d.pfm" % (v, l)))
        assert not os.path.exists(os.path.join(str(d), "depth_v%d_stage2_iter3.pfm" % v))
        for s in (1, 2, 3):
            assert os.path.exists(os.path.join(str(d), "depth_v%d_stage%d.png" % (v, s)))
        assert len(open(art.superpixels_path(str(d), v)).read().splitlines()) == 1 + 27 * 20
    stats = [json.loads(x) for x in open(os.path.join(str(d), "stats.jsonl"))]
    assert [s["stage"] for s in stats] == ["segment"] * 3 + ["init"] * 3 + ["refine"] * 3 + ["fuse"] * 3
    tsv = open(os.path.join(str(d), "timings.tsv")).read().splitlines()
    assert tsv[0] == "stage\tview\tms" and len(tsv) == 1 + 12


def _copy_run(src, dst, keep):
    import shutil

    os.makedirs(dst, exist_ok=True)
    for name in os.listdir(src):
        if any(name.startswith(k) for k in keep):
            shutil.copy(os.path.join(src, name), os.path.join(dst, name))


@pytest.mark.parametrize("keep,stages", [
    (("labels_",), ["init", "refine", "fuse"]),                   # segment reloaded from the PNGs
    (("labels_", "planes_v0_stage1", "planes_v1_stage1", "planes_v2_stage1"), ["refine", "fuse"]),
    (("labels_", "planes_"), ["fuse"]),                             # refined planes reloaded
])
def test_resume_reproduces_the_uninterrupted_run(c1, full_run, tmp_path, keep, stages):
    from paper_1812_06856_b200.run import run_pipeline

    d, res = full_run
    _copy_run(str(d), str(tmp_path), keep)
    got = run_pipeline(c1["lab"], c1["cams"], c1["range"], _cfg(tmp_path, resume=True, stages=stages))
    for v in range(3):
        assert np.array_equal(_bits(got["refined_planes"][v]), _bits(res["refined_planes"][v]))
        assert np.array_equal(_bits(got["depth_refined"][v]), _bits(res["depth_refined"][v]))
        assert np.array_equal(_bits(got["fused"][v]), _bits(res["fused"][v]))
        assert np.array_equal(got["grids"][v].label_map, res["grids"][v].label_map)
        assert got["grids"][v].sp.tobytes() == res["grids"][v].sp.tobytes()


def test_resume_fused_maps_and_missing_products(c1, full_run, tmp_path):
    from paper_1812_06856_b200 import api
    from paper_1812_06856_b200.run import run_pipeline

    d, res = full_run
    _copy_run(str(d), str(tmp_path), ("depth_v0_stage3", "depth_v1_stage3", "depth_v2_stage3", "labels_", "planes_"))
    got = run_pipeline(c1["lab"], c1["cams"], c1["range"], _cfg(tmp_path, resume=True, stages=["eval"]))
    assert got["grids"] is None
    for v in range(3):
        assert np.array_equal(_bits(got["fused"][v]), _bits(res["fused"][v]))
    empty = tmp_path / "empty"
    with pytest.raises(api.InvalidParams, match="segment stage not selected"):
        run_pipeline(c1["lab"], c1["cams"], c1["range"], _cfg(empty, resume=True, stages=["init"]))
    with pytest.raises(api.InvalidParams, match="unknown stage"):
        run_pipeline(c1["lab"], c1["cams"], c1["range"], _cfg(empty, stages=["bogus"]))


def test_split_run_artifacts_byte_identical(c1, full_run, tmp_path):
    """tests/test_pipeline.cpp:139-164: segment+init, then resume refine+fuse(+eval) -> every
    depth PFM and label PNG byte-identical to the single run."""
    from paper_1812_06856_b200.run import run_pipeline

    d, _ = full_run
    run_pipeline(c1["lab"], c1["cams"], c1["range"], _cfg(tmp_path, stages=["segment", "init"]))
    run_pipeline(c1["lab"], c1["cams"], c1["range"], _cfg(tmp_path, resume=True, stages=["refine", "fuse", "eval"]))
    for v in range(3):
        names = ["depth_v%d_stage%d.pfm" % (v, s) for s in (1, 2, 3)] + ["labels_v%d.png" % v,
                                                                           "planes_v%d_stage2.txt" % v]
        for name in names:
            assert (tmp_path / name).read_bytes() == open(os.path.join(str(d), name), "rb").read(), name


def test_missing_predecessors_and_corrupt_planes(c1, tmp_path):
    """tests/test_pipeline.cpp:180-215."""
    from paper_1812_06856_b200 import api
    from paper_1812_06856_b200.run import PipelineError, run_pipeline

    with pytest.raises(api.InvalidParams):
        run_pipeline(c1["lab"], c1["cams"], c1["range"], _cfg(tmp_path / "a", stages=["refine"]))
    run_pipeline(c1["lab"], c1["cams"], c1["range"], _cfg(tmp_path / "b", stages=["segment", "init"]))
    (tmp_path / "b" / "planes_v1_stage1.txt").write_text("2\n0x1p+2 0 0 -0x1p+0\n")  # wrong count for the grid
    with pytest.raises(PipelineError) as e:
        run_pipeline(c1["lab"], c1["cams"], c1["range"], _cfg(tmp_path / "b", resume=True, stages=["refine"]))
    assert "init" in str(e.value) and "view 1" in str(e.value)
