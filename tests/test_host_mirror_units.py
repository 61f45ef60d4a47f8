"""Host-side mirror classes (TransferFunction, Camera, orbit poses) behave
like the reference's: the properties its test_transfer.py / test_camera.py
pin, restated against this package on CPU.  These classes feed the frame
packing (ro_pack_frame / _pack_frame_py), so a behavioural drift here would
show up as wrong emptiness tables or rays in every frame."""

import math

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

from paper_2309_04393_b200.camera import (Camera, CameraError, generate_rays, orbit_path,
                                          orbit_pose)
from paper_2309_04393_b200.transfer import (TransferFunction, TransferFunctionError,
                                            grayscale_ramp_tf, transparent_tf)


@st.composite
def _tfs(draw):
    xs = sorted(draw(st.lists(st.integers(0, 255), min_size=2, max_size=6, unique=True)))
    pts = []
    for x in xs:
        rgb = [draw(st.floats(0.0, 1.0)) for _ in range(3)]
        a = draw(st.sampled_from([0.0, 0.0, 0.3, 0.75, 1.0]))
        pts.append((float(x), (*rgb, a)))
    return TransferFunction(points=tuple(pts))


# -- transfer functions (transfer.py:22-120; test_transfer.py) ----------------

@pytest.mark.parametrize("points", [
    ((0.0, (0, 0, 0, 0)),),                                  # one knot
    ((7.0, (0, 0, 0, 0)), (7.0, (0, 0, 0, 1))),              # not increasing
    ((0.0, (0, 0, 0, 0)), (300.0, (0, 0, 0, 1))),            # scalar > 255
    ((0.0, (0, 0, 0, -0.1)), (9.0, (0, 0, 0, 1))),           # rgba < 0
])
def test_tf_rejects_malformed_points(points):
    with pytest.raises(TransferFunctionError):
        TransferFunction(points=points)


def test_tf_piecewise_linear_and_zero_outside():
    tf = TransferFunction(points=((100.0, (0.0, 0.0, 0.0, 0.0)), (140.0, (0.8, 0.4, 0.2, 1.0))))
    assert tf.evaluate(99.0) == (0.0, 0.0, 0.0, 0.0)
    assert tf.evaluate(141.0) == (0.0, 0.0, 0.0, 0.0)
    assert tf.evaluate(110.0) == pytest.approx((0.2, 0.1, 0.05, 0.25))
    assert tf.evaluate(140.0) == pytest.approx((0.8, 0.4, 0.2, 1.0))


@settings(max_examples=120, deadline=None)
@given(_tfs(), st.integers(0, 255), st.integers(0, 255))
def test_tf_interval_emptiness_is_exact(tf, a, b):
    """Linear segments: opacity vanishes on [lo, hi] iff it vanishes at both
    ends and at every knot strictly inside."""
    lo, hi = min(a, b), max(a, b)
    want = (tf.opacity(lo) == 0.0 and tf.opacity(hi) == 0.0
            and all(p[1][3] == 0.0 for p in tf.points if lo < p[0] < hi))
    assert tf.interval_is_empty(lo, hi) == want
    # the kernel's table form: (lo, hi) transparent <=> hi < E[lo]
    assert (hi < int(tf.empty_below()[lo])) == want


@settings(max_examples=80, deadline=None)
@given(_tfs(), st.integers(0, 255), st.integers(0, 255))
def test_tf_interval_max_opacity_bounds_a_dense_scan(tf, a, b):
    lo, hi = min(a, b), max(a, b)
    dense = max(tf.opacity(float(x)) for x in np.linspace(lo, hi, 1001))
    exact = tf.interval_max_opacity(lo, hi)
    assert exact >= dense - 1e-12
    # piecewise linear: the maximum sits at an end or at a knot inside
    peaks = [tf.opacity(float(lo)), tf.opacity(float(hi))] + \
        [p[1][3] for p in tf.points if lo < p[0] < hi]
    assert exact == pytest.approx(max(peaks), abs=1e-12)


def test_tf_first_support_and_table():
    tf = TransferFunction(points=((30.0, (0, 0, 0, 0)), (40.0, (0, 0, 0, 1)),
                                  (50.0, (0, 0, 0, 0)), (180.0, (0, 0, 0, 0)),
                                  (190.0, (1, 1, 1, 1))))
    assert [tf.first_support_at_or_after(v) for v in (0.0, 35.0, 50.0, 185.0)] == \
        [30.0, 35.0, 180.0, 185.0]
    assert tf.first_support_at_or_after(191.0) == math.inf
    assert transparent_tf().first_support_at_or_after(0.0) == math.inf
    f, op = grayscale_ramp_tf(threshold=40.0).support_table()
    ramp = grayscale_ramp_tf(threshold=40.0)
    for v in range(256):
        assert op[v] == ramp.opacity(float(v))
        fs = ramp.first_support_at_or_after(float(v))
        assert f[v] == (1e30 if fs == math.inf else fs)


def test_tf_packed_points():
    tf = grayscale_ramp_tf(threshold=25.0, max_alpha=0.6)
    xs, rgba, n = tf.packed_points(16)
    assert n == len(tf.points) and xs[1] == 25.0 and rgba[n - 1, 3] == 0.6
    with pytest.raises(TransferFunctionError):
        tf.packed_points(n - 1)


# -- camera and poses (camera.py:15-69; test_camera.py) ------------------------

@pytest.mark.parametrize("kw", [dict(position=(0.5, 0.5, 0.5)),
                                dict(position=(0.5, -2.0, 0.5)),
                                dict(position=(1.0, 2.0, 3.0), fov_deg=0.0),
                                dict(position=(1.0, 2.0, 3.0), fov_deg=180.0)])
def test_camera_rejects_degenerate_setups(kw):
    with pytest.raises(CameraError):
        Camera(**kw)


def test_rays_unit_length_shared_origin_scanline_order():
    cam = Camera(position=(0.2, 0.9, 2.6))
    o, d = generate_rays(cam, 13, 7)
    assert o.shape == d.shape == (91, 3)
    assert np.all(o == np.array(cam.position))
    assert np.allclose(np.linalg.norm(d, axis=1), 1.0, atol=1e-12)
    g = d.reshape(7, 13, 3)
    up = np.cross(np.cross(np.subtract(cam.target, cam.position), cam.up),
                  np.subtract(cam.target, cam.position))
    assert g[0, 6] @ up > g[6, 6] @ up                      # row 0 is the top row


def test_odd_image_centre_ray_is_the_view_axis():
    cam = Camera(position=(-1.0, 0.3, 2.2), target=(0.4, 0.6, 0.5))
    _, d = generate_rays(cam, 9, 15)
    f = np.subtract(cam.target, cam.position)
    assert np.allclose(d[7 * 9 + 4], f / np.linalg.norm(f), atol=1e-12)


def test_wider_fov_spreads_rays():
    axis = np.array([0.0, 0.0, -1.0])
    spread = {}
    for fov in (25.0, 70.0):
        _, d = generate_rays(Camera(position=(0.5, 0.5, 3.0), fov_deg=fov), 12, 12)
        spread[fov] = np.arccos(np.clip(d @ axis, -1.0, 1.0)).max()
    assert spread[70.0] > spread[25.0] and spread[25.0] < math.radians(25.0)


def test_orbit_geometry_and_determinism():
    assert orbit_pose(0.0, radius=1.5, elevation=0.25).position == (2.0, 0.75, 0.5)
    assert np.allclose(orbit_pose(math.pi, radius=1.5, elevation=0.25).position,
                       (-1.0, 0.75, 0.5), atol=1e-12)
    cams = orbit_path(24, radius=1.3, elevation=-0.1)
    assert len({c.position for c in cams}) == 24
    for c in cams:
        r = np.subtract(c.position, (0.5, 0.5, 0.5))
        assert math.hypot(r[0], r[2]) == pytest.approx(1.3) and r[1] == pytest.approx(-0.1)
    a, b = generate_rays(cams[5], 16, 16), generate_rays(cams[5], 16, 16)
    assert np.array_equal(a[1], b[1])
