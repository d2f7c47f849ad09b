"""GPU frame producer (evs_render) against golden frames of the reference
renderer (tests/golden/render.npz, make_render_golden.py) and the reference's
own renderer tests (test_render.py:32-163) re-pointed at the drop-in."""

import math
import os

import numpy as np
import pytest

from paper_2602_15018_b200.render import (AxisPlane, CameraIntrinsics, Checkerboard, Pose, SceneSpec, ValueNoise,
                                          pinhole_project, render_depth, render_intensity, render_pair,
                                          scene_from_dict)

pytestmark = pytest.mark.gpu
GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "render.npz"))
KG = CameraIntrinsics(fx=300.0, fy=290.0, cx=159.5, cy=119.5, width=320, height=240)
_s, _c = math.sin(math.pi / 10), math.cos(math.pi / 10)
SCENES = {
    "checker_identity": (SceneSpec(planes=(AxisPlane(2, 2.0, (-40, 40, -40, 40), Checkerboard(0.5, 0.2, 0.9)),),
                                   ambient=0.0),
                         Pose((0.3, -0.2, 0.0), (1.0, 0.0, 0.0, 0.0))),
    "room_rotated": (SceneSpec(planes=(
        AxisPlane(2, 4.0, (-5, 5, -5, 5), ValueNoise(0.7, 5, 0.2, 0.9)),
        AxisPlane(0, 1.5, (-5, 5, -1, 8), Checkerboard(0.3, 0.1, 0.8)),
        AxisPlane(1, 1.0, (-5, 5, -1, 8), ValueNoise(0.25, 11, 0.0, 1.0)),
        AxisPlane(0, -1.5, (-5, 5, -1, 8), ValueNoise(1.3, 2, 0.4, 0.6)),
    ), ambient=0.3), Pose((0.1, 0.2, -0.5), (_c, 0.0, _s, 0.0))),
    "tie_and_miss": (SceneSpec(planes=(
        AxisPlane(2, 3.0, (-1, 1, -1, 1), Checkerboard(0.2, 0.0, 1.0)),
        AxisPlane(2, 3.0, (-2, 2, -2, 2), Checkerboard(0.1, 0.5, 0.6)),
    ), ambient=0.15), Pose((0.0, 0.0, 0.0), (1.0, 0.0, 0.0, 0.0))),
}


@pytest.mark.parametrize("name", sorted(SCENES))
def test_matches_reference_golden(name):
    """Bit-exact except where the ray direction's dot product (BLAS in the
    reference, render.py:176) lands a hit point exactly on a texture edge."""
    scene, pose = SCENES[name]
    it, dp = render_pair(scene, pose, KG)
    gi, gd = GOLD[f"{name}_intensity"], GOLD[f"{name}_depth"]
    diff = it.values != gi
    assert diff.mean() < 2e-4, (name, int(diff.sum()))
    fin = np.isfinite(gd)
    assert np.array_equal(np.isfinite(dp.values), fin)
    assert np.allclose(dp.values[fin], gd[fin], rtol=1e-6, atol=0)


def test_device_output_stays_on_gpu_and_feeds_the_event_path():
    import torch

    from paper_2602_15018_b200 import events as ev

    scene, pose = SCENES["room_rotated"]
    it, _dp = render_pair(scene, pose, KG, device_output=True)
    assert isinstance(it.values, torch.Tensor) and it.values.is_cuda
    cfg = ev.EventCameraConfig(c_pos=0.15, c_neg=0.15)
    st = ev.init_pixel_states(render_intensity(scene, pose, KG), cfg, seed=0)
    pose2 = Pose((0.12, 0.2, -0.5), pose.orientation)
    b = ev.generate_events_parallel(st, render_intensity(scene, pose2, KG, t=1000, device_output=True), 0, 1000,
                                    cfg)
    assert len(b) > 0


# -- the reference's renderer tests (test_render.py), against the drop-in ---------
K = CameraIntrinsics(fx=100.0, fy=100.0, cx=32.0, cy=24.0, width=64, height=48)
IDENTITY = Pose(position=(0.0, 0.0, 0.0), orientation=(1.0, 0.0, 0.0, 0.0))


def _uniform_plane(axis=2, offset=2.0, value=0.7, bounds=(-50, 50, -50, 50)):
    return AxisPlane(axis=axis, offset=offset, bounds=bounds,
                     texture=Checkerboard(cell=1000.0, intensity_a=value, intensity_b=value))


def test_pinhole():
    assert pinhole_project((0, 0, 1), K) == (32.0, 24.0)
    assert pinhole_project((0.1, 0, 1), K) == (42.0, 24.0)
    assert pinhole_project((0, 0, -1), K) is None


def test_uniform_plane_fills_view():
    frame = render_intensity(SceneSpec(planes=(_uniform_plane(),), ambient=0.0), IDENTITY, K)
    assert np.all(np.abs(frame.values - np.float32(0.7)) < 1e-6)


def test_miss_returns_ambient_and_infinite_depth():
    scene = SceneSpec(planes=(), ambient=0.25)
    assert np.all(render_intensity(scene, IDENTITY, K).values == np.float32(0.25))
    assert np.all(np.isinf(render_depth(scene, IDENTITY, K).values))


def test_checkerboard_against_pixel_oracle():
    checker = Checkerboard(cell=0.5, intensity_a=0.2, intensity_b=0.9)
    scene = SceneSpec(planes=(AxisPlane(axis=2, offset=2.0, bounds=(-40, 40, -40, 40), texture=checker),))
    pose = Pose(position=(0.3, -0.2, 0.0), orientation=(1.0, 0.0, 0.0, 0.0))
    frame = render_intensity(scene, pose, K)
    rng = np.random.default_rng(0)
    for _ in range(16):
        u, v = int(rng.integers(0, K.width)), int(rng.integers(0, K.height))
        px = 0.3 + 2.0 * ((u - K.cx) / K.fx)
        py = -0.2 + 2.0 * ((v - K.cy) / K.fy)
        expect = 0.2 if (math.floor(px / 0.5) + math.floor(py / 0.5)) % 2 == 0 else 0.9
        assert frame.values[v, u] == pytest.approx(expect, abs=1e-6), (u, v)


def test_fronto_parallel_and_oblique_depth():
    depth = render_depth(SceneSpec(planes=(_uniform_plane(offset=2.0),)), IDENTITY, K)
    assert np.all(np.abs(depth.values - 2.0) < 1e-5)
    s, c = math.sin(math.pi / 8), math.cos(math.pi / 8)
    pose = Pose(position=(0.0, 0.0, 0.0), orientation=(c, 0.0, s, 0.0))
    plane = _uniform_plane(axis=0, offset=1.0, value=0.5)
    depth = render_depth(SceneSpec(planes=(plane,)), pose, K)
    R = pose.rotation_matrix()
    for u, v in [(3, 7), (60, 40), (31, 20)]:
        d = R @ np.array([(u - K.cx) / K.fx, (v - K.cy) / K.fy, 1.0])
        assert depth.values[v, u] == pytest.approx(1.0 / d[0], abs=1e-5)


def test_nearest_hit_tie_break_declaration_order():
    a = _uniform_plane(offset=2.0, value=0.3)
    b = _uniform_plane(offset=2.0, value=0.8)
    frame = render_intensity(SceneSpec(planes=(a, b)), IDENTITY, K)
    assert np.all(np.abs(frame.values - np.float32(0.3)) < 1e-6)


def test_scene_from_dict_and_validation():
    scene = scene_from_dict({"ambient": 0.1, "planes": [
        {"axis": "z", "offset": 3.0, "bounds": [-1, 1, -1, 1], "texture": {"type": "noise", "scale": 0.5, "seed": 3}},
        {"axis": 0, "offset": 1.0, "bounds": [-1, 1, -1, 1],
         "texture": {"type": "checker", "cell": 0.2, "intensity_a": 0.0, "intensity_b": 1.0}},
    ]})
    assert len(scene.planes) == 2 and scene.planes[0].axis == 2
    with pytest.raises(ValueError):
        CameraIntrinsics(fx=0.0, fy=1.0, cx=0.0, cy=0.0, width=4, height=4)
    with pytest.raises(ValueError):
        Pose(position=(0, 0, 0), orientation=(1.0, 1.0, 0.0, 0.0))
