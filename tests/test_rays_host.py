"""The product Camera / generate_rays (paper_2111_00110_b200/ray.py) pinned to
rays the REFERENCE generated (reference ray.py:26-48 basis, :63-77 pixel
centres): the golden bundles of tests/golden/make_golden_rays.py, whose
cameras are rebuilt here from the same seeds.  Bit-exact (float64)."""

import numpy as np

from conftest import golden
from paper_2111_00110_b200.ray import Camera, generate_rays


def _seeded_direction(rng):
    while True:
        u = rng.normal(size=3)
        u /= np.linalg.norm(u)
        if abs(u[1]) <= 0.99:
            return u


def _check(cam, g):
    b = generate_rays(cam)
    assert b.origins.dtype == np.float64 and b.directions.dtype == np.float64
    assert np.array_equal(b.origins, g["origins"])
    assert np.array_equal(b.directions, g["directions"])


def test_generate_rays_small_scene_bit_exact():
    """make_golden_rays.part_layers_small: fixed camera, 24 x 24."""
    cam = Camera(position=np.array([0.0, 0.0, -2.5]), look_at=np.zeros(3),
                 up=np.array([0.0, 1.0, 0.0]), fov_deg=30.0, width=24, height=24)
    _check(cam, golden("rays_small"))


def test_generate_rays_config3_camera_bit_exact():
    """make_golden_rays.part_cfg3_small: radius 2 on a seeded direction, fov 60."""
    rng = np.random.default_rng(33)
    n = 1 << 14
    rng.uniform(-1, 1, (n, 3))
    rng.normal(0.0, 0.1, (n, 1))
    cam = Camera(position=2.0 * _seeded_direction(rng), look_at=np.zeros(3),
                 up=np.array([0.0, 1.0, 0.0]), fov_deg=60.0, width=48, height=48)
    _check(cam, golden("rays_cfg3"))


def test_generate_rays_config4_camera_bit_exact():
    """make_golden_rays.part_cfg4_small: radius 2.5 on a seeded direction, fov 50."""
    rng = np.random.default_rng(44)
    n = 1 << 14
    rng.uniform(-1, 1, (n, 3))
    rng.normal(size=(n, 1))
    rng.uniform(0, 1, (n, 3))
    cam = Camera(position=2.5 * _seeded_direction(rng), look_at=np.zeros(3),
                 up=np.array([0.0, 1.0, 0.0]), fov_deg=50.0, width=32, height=32)
    _check(cam, golden("rays_cfg4"))


def test_generate_rays_row_major_pixel_centres():
    """Ray k is pixel (k // width, k % width); non-square images keep the aspect."""
    cam = Camera(position=np.array([0.3, -0.2, 2.0]), look_at=np.zeros(3),
                 up=np.array([0.0, 1.0, 0.0]), fov_deg=45.0, width=7, height=3)
    b = generate_rays(cam)
    assert b.count == 21
    assert np.allclose(np.linalg.norm(b.directions, axis=1), 1.0, atol=1e-15)
    fwd, right, down = cam.basis()
    centre = b.directions[1 * 7 + 3]          # middle pixel of the middle row
    assert np.allclose(centre, fwd, atol=1e-15)
    assert np.dot(b.directions[6] - b.directions[0], right) > 0      # x grows along a row
    assert np.dot(b.directions[14] - b.directions[0], down) > 0      # y grows down the rows
