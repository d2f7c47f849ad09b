"""Golden frames of the reference renderer (run where /root/reference exists):
tests/golden/render.npz.  Source: /root/reference/pkg/src/evsim/render.py
(render_pair, render.py:179-208), imported from a copy of pkg/src."""
import math
import os
import shutil
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
tmp = tempfile.mkdtemp()
shutil.copytree("/root/reference/pkg/src", os.path.join(tmp, "src"))
sys.path.insert(0, os.path.join(tmp, "src"))
from evsim.render import AxisPlane, CameraIntrinsics, Checkerboard, Pose, SceneSpec, ValueNoise, render_pair  # noqa: E402

K = CameraIntrinsics(fx=300.0, fy=290.0, cx=159.5, cy=119.5, width=320, height=240)
s, c = math.sin(math.pi / 10), math.cos(math.pi / 10)
scenes = {
    "checker_identity": (SceneSpec(planes=(AxisPlane(2, 2.0, (-40, 40, -40, 40), Checkerboard(0.5, 0.2, 0.9)),),
                                   ambient=0.0),
                         Pose((0.3, -0.2, 0.0), (1.0, 0.0, 0.0, 0.0))),
    "room_rotated": (SceneSpec(planes=(
        AxisPlane(2, 4.0, (-5, 5, -5, 5), ValueNoise(0.7, 5, 0.2, 0.9)),
        AxisPlane(0, 1.5, (-5, 5, -1, 8), Checkerboard(0.3, 0.1, 0.8)),
        AxisPlane(1, 1.0, (-5, 5, -1, 8), ValueNoise(0.25, 11, 0.0, 1.0)),
        AxisPlane(0, -1.5, (-5, 5, -1, 8), ValueNoise(1.3, 2, 0.4, 0.6)),
    ), ambient=0.3), Pose((0.1, 0.2, -0.5), (c, 0.0, s, 0.0))),
    "tie_and_miss": (SceneSpec(planes=(
        AxisPlane(2, 3.0, (-1, 1, -1, 1), Checkerboard(0.2, 0.0, 1.0)),
        AxisPlane(2, 3.0, (-2, 2, -2, 2), Checkerboard(0.1, 0.5, 0.6)),
    ), ambient=0.15), Pose((0.0, 0.0, 0.0), (1.0, 0.0, 0.0, 0.0))),
}
out = {}
for name, (scene, pose) in scenes.items():
    it, dp = render_pair(scene, pose, K, t=0)
    out[f"{name}_intensity"] = it.values
    out[f"{name}_depth"] = dp.values
np.savez_compressed(os.path.join(HERE, "render.npz"), **out)
print({k: v.shape for k, v in out.items()})
