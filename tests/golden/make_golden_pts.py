"""Writes tests/golden/sample2d.pts and sample3d.pts with the REFERENCE's own
writer (/root/reference/pkg/src/seghull/pointfile.py) so the device reader
is pinned to files the reference produces.  Run in the build container:
    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_pts.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from seghull.datagen import Distribution, generate  # noqa: E402
from seghull.pointfile import write_points_binary, write_points_csv  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
write_points_binary(os.path.join(HERE, "sample2d.pts"), generate(Distribution("uniform-disk", 1000, 5)))
write_points_binary(os.path.join(HERE, "sample3d.pts"), generate(Distribution("uniform-ball", 700, 6)))
write_points_csv(os.path.join(HERE, "sample3d.csv"), generate(Distribution("on-sphere", 50, 7)))
print("ok")
