"""Host-side validation (no GPU): the Python mirror's shape checks and the reference's parameter
validation rules (superpixel.hpp:23-27, sweep.hpp:19-22, refine.hpp:28-31, pipeline.hpp:43-56),
raised before any library call or file I/O."""
import os

import numpy as np
import pytest

from paper_1812_06856_b200 import api
from paper_1812_06856_b200.run import PipelineConfig


def test_check_images():
    api.check_images(np.zeros((2, 4, 5, 3), np.float32), "x", 4, 5, 2)
    for bad in (np.zeros((4, 5, 3)), np.zeros((2, 4, 5, 4)), np.zeros((0, 4, 5, 3))):
        with pytest.raises(api.InvalidParams):
            api.check_images(bad)
    with pytest.raises(api.InvalidParams):
        api.check_images(np.zeros((2, 4, 6, 3)), "x", 4, 5)
    with pytest.raises(api.InvalidParams):
        api.check_images(np.zeros((3, 4, 5, 3)), "x", 4, 5, 2)


@pytest.mark.parametrize("cfg,msg", [
    (dict(slic=api.SlicParams(size=3)), "superpixel size must be >= 4"),
    (dict(slic=api.SlicParams(compactness=0)), "compactness must be > 0"),
    (dict(slic=api.SlicParams(iterations=0)), "iterations must be >= 1"),
    (dict(sweep=api.SweepParams(levels=1)), "sweep levels must be >= 2"),
    (dict(sweep=api.SweepParams(tssd_threshold=0)), "tssd threshold must be > 0"),
    (dict(energy=api.EnergyParams(eta=2)), "bad energy params"),
    (dict(energy=api.EnergyParams(alpha=0)), "bad energy params"),
    (dict(energy=api.EnergyParams(steps_init=0)), "bad kernel params"),
])
def test_pipeline_config_validates_parameter_structs_first(tmp_path, cfg, msg):
    out = tmp_path / "run"
    c = PipelineConfig(out_dir=str(out), **cfg)
    with pytest.raises(api.InvalidParams, match=msg):
        c.validate()
    assert not os.path.exists(out)  # nothing written
