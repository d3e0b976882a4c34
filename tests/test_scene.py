"""The product's scene generator (csrc/scene.cpp) is byte-identical to the reference fixtures
(fixtures.hpp render_scene + image.hpp rgb_to_scaled_lab), run here through oracle/_ref."""
import numpy as np
import pytest

CASES = [
    ("cluttered", 3, 320, 240, 320.0, 0.1, 0.0, (0, 0)),
    ("cluttered", 4, 160, 96, 160.0, 0.04, 0.0, (2, 2)),
    ("staircase", 3, 96, 72, 80.0, 0.4, 0.0, (0, 0)),
    ("wall", 2, 64, 48, 80.0, 0.4, 5.0, (0, 0)),
    ("slanted", 3, 120, 90, 100.0, 0.2, 25.0, (0, 0)),
    ("occluder", 3, 80, 60, 70.0, 0.3, 0.0, (0, 0)),
]


@pytest.mark.parametrize("case", CASES, ids=[c[0] + str(c[7][0]) for c in CASES])
def test_scene_matches_reference(ref, case):
    from paper_1812_06856_b200 import scenes

    kind, n, w, h, f, b, extra, grid = case
    want = ref.render_scene(kind, n, w, h, f, b, extra, grid)
    got = scenes.render_scene(kind, n, w, h, f, b, extra, grid, threads=3, rgb=True)
    assert got["range"] == want["range"]
    assert np.array_equal(got["cams"].view(np.uint64), want["cams"].view(np.uint64))
    assert np.array_equal(got["rgb"].view(np.uint32), want["rgb"].view(np.uint32))
    assert np.array_equal(got["lab"].view(np.uint32), want["lab"].view(np.uint32))
    assert np.array_equal(got["gt"].view(np.uint32), want["gt"].view(np.uint32))


def test_thread_count_invariance():
    from paper_1812_06856_b200 import scenes

    a = scenes.render_scene("cluttered", 3, 200, 150, 200.0, 0.1, threads=1)
    b = scenes.render_scene("cluttered", 3, 200, 150, 200.0, 0.1, threads=7)
    assert np.array_equal(a["lab"], b["lab"]) and np.array_equal(a["gt"], b["gt"])
