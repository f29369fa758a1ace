"""Pins the oracle's geometry and losses to the reference's own known-answer
tests and properties (proj/tests/test_geometry.cpp, proj/tests/test_losses.cpp)."""
import math

import numpy as np
import pytest


def rot_axis(axis, a):
    c, s = math.cos(a), math.sin(a)
    if axis == 0:
        return np.array([[1, 0, 0], [0, c, -s], [0, s, c]])
    if axis == 1:
        return np.array([[c, 0, s], [0, 1, 0], [-s, 0, c]])
    return np.array([[c, -s, 0], [s, c, 0], [0, 0, 1]])


def random_feasible_config(rng, min_depth=0.5, max_depth=10.0, O=None):
    """proj/tests/test_util.hpp:16-31 — drawn with numpy here (not the Rng stream)."""
    x = rng.uniform(-10, 10, 3)
    a, b, g = rng.uniform(-3.1, 3.1), rng.uniform(-1.5, 1.5), rng.uniform(-3.1, 3.1)
    f = rng.uniform(0.5, 2000.0)
    R = O.rotation_from_euler(a, b, g)
    w = R @ x
    t = np.array([rng.uniform(-5, 5), rng.uniform(-5, 5), rng.uniform(min_depth, max_depth) - w[2]])
    return x, np.array([a, b, g, *t, f])


def test_rotation_identity_and_quarter_turn(O):
    # test_geometry.cpp:40-47
    assert np.array_equal(O.rotation_from_euler(0, 0, 0), np.eye(3))
    m = O.rotation_from_euler(0, 0, math.pi / 2) @ np.array([1.0, 0, 0])
    assert np.allclose(m, [0, 1, 0], atol=1e-15)


def test_rotation_orthonormal_matches_axis_angle(O):
    # test_geometry.cpp:49-58 (1e-12)
    rng = np.random.default_rng(17)
    for _ in range(100):
        a, b, g = rng.uniform(-10, 10, 3)
        R = O.rotation_from_euler(a, b, g)
        assert np.abs(R.T @ R - np.eye(3)).max() < 1e-12
        assert abs(np.linalg.det(R) - 1) < 1e-12
        assert np.abs(R - rot_axis(2, g) @ rot_axis(1, b) @ rot_axis(0, a)).max() < 1e-12


def test_euler_roundtrip(O):
    # test_geometry.cpp:60-71
    rng = np.random.default_rng(18)
    for _ in range(100):
        a, b, g = rng.uniform(-3.1, 3.1), rng.uniform(-1.5, 1.5), rng.uniform(-3.1, 3.1)
        e = O.euler_from_rotation(O.rotation_from_euler(a, b, g))
        assert np.allclose(e, [a, b, g], rtol=1e-9, atol=1e-12)


def test_project_kats(O):
    # test_geometry.cpp:73-83
    assert np.allclose(O.project([0, 0, 5], [0, 0, 0, 0, 0, 0, 1.0]), [0, 0], atol=1e-15)
    assert np.array_equal(O.project([1, 2, 2], [0, 0, 0, 0, 0, 0, 2.0]), [1, 2])


def test_project_matches_homogeneous(O):
    # test_geometry.cpp:85-93
    rng = np.random.default_rng(19)
    for _ in range(100):
        x, cam = random_feasible_config(rng, 0.1, O=O)
        z = O.project(x, cam)
        K = np.diag([cam[6], cam[6], 1.0])
        zh = K @ (O.rotation_from_euler(*cam[:3]) @ x + cam[3:6])
        zo = zh[:2] / zh[2]
        assert np.abs(z - zo).max() < 1e-12 * max(1.0, np.linalg.norm(zo))


def test_depth_guard(O):
    # test_geometry.cpp:95-105 — boundary 1e-6 is admissible; NaN rejected
    cam = [0, 0, 0, 0, 0, 0, 1.0]
    assert O.project([0, 0, -1], cam) is None
    assert O.project([0, 0, 0], cam) is None
    assert O.project([1, 1, 1e-7], cam) is None
    assert O.project([1, 1, 1e-6], cam) is not None
    assert O.project([0, 0, float("nan")], cam) is None


def test_jacobian_canonical_and_translation_columns(O):
    # test_geometry.cpp:150-168
    _, Jp, _ = O.project_with_jacobians([0, 0, 1], [0, 0, 0, 0, 0, 0, 1.0])
    assert np.array_equal(Jp, [[1, 0, 0], [0, 1, 0]])
    rng = np.random.default_rng(23)
    for _ in range(20):
        cam = [0, 0, 0, rng.uniform(-1, 1), rng.uniform(-1, 1), rng.uniform(2, 5), 1.0]
        x = [rng.uniform(-1, 1), rng.uniform(-1, 1), rng.uniform(0, 1)]
        _, Jp, Jc = O.project_with_jacobians(x, cam)
        assert np.abs(Jc[:, 3:] - Jp).max() < 1e-15


def test_jacobians_match_central_fd(O):
    # test_geometry.cpp:170-201 — h=1e-6, relative 1e-6 (acceptance criterion 1)
    rng = np.random.default_rng(24)
    h = 1e-6
    for _ in range(100):
        x, cam = random_feasible_config(rng, 0.1, O=O)
        z, Jp, Jc = O.project_with_jacobians(x, cam)
        assert np.array_equal(z, O.project(x, cam))
        fdp = np.zeros((2, 3))
        for k in range(3):
            lo, hi = x.copy(), x.copy()
            lo[k] -= h
            hi[k] += h
            fdp[:, k] = (O.project(hi, cam) - O.project(lo, cam)) / (2 * h)
        fdc = np.zeros((2, 6))
        for k in range(6):
            lo, hi = cam.copy(), cam.copy()
            lo[k] -= h
            hi[k] += h
            fdc[:, k] = (O.project(x, hi) - O.project(x, lo)) / (2 * h)
        assert np.abs(fdp - Jp).max() / max(1.0, np.abs(Jp).max()) < 1e-6
        assert np.abs(fdc - Jc).max() / max(1.0, np.abs(Jc).max()) < 1e-6


def test_project_periodic_and_scale_invariant(O):
    # test_geometry.cpp:107-133
    rng = np.random.default_rng(21)
    for _ in range(50):
        x, cam = random_feasible_config(rng, 0.5, O=O)
        base = O.project(x, cam)
        for which in range(3):
            sh = cam.copy()
            sh[which] += 2 * math.pi * (1 + rng.integers(3))
            assert np.linalg.norm(O.project(x, sh) - base) < 1e-9 * max(1.0, np.linalg.norm(base))
        cam1 = cam.copy()
        cam1[6] = 1.0
        c = rng.uniform(0.1, 100)
        sc = cam1.copy()
        sc[3:6] *= c
        a, b = O.project(x, cam1), O.project(c * x, sc)
        assert np.linalg.norm(a - b) < 1e-9 * max(1.0, np.linalg.norm(a))


def test_loss_kats(O):
    # test_losses.cpp:11-22
    assert O.loss_value(0, 1.0, [3, 4]) == 25.0
    assert np.array_equal(O.loss_gradient(0, 1.0, [1, 2]), [2, 4])
    assert O.loss_value(1, 1.0, [0, 0]) == 0.0
    assert O.loss_value(1, 1.0, [3, 4]) == pytest.approx(4.5, rel=1e-15)
    assert np.array_equal(O.loss_gradient(1, 1.0, [0.3, 0]), [0.3, 0])
    assert np.array_equal(O.loss_gradient(1, 1.0, [0, 0]), [0, 0])


def test_loss_gradients_fd_and_properties(O):
    # test_losses.cpp:29-49, 86-99
    rng = np.random.default_rng(31)
    h = 1e-7
    checked = 0
    while checked < 100:
        kind = 0 if rng.uniform() < 0.5 else 1
        r = rng.uniform(-3, 3, 2)
        if kind == 1 and abs(np.linalg.norm(r) - 1.0) <= 1e-3:
            continue
        g = O.loss_gradient(kind, 1.0, r)
        for k in range(2):
            lo, hi = r.copy(), r.copy()
            lo[k] -= h
            hi[k] += h
            fd = (O.loss_value(kind, 1.0, hi) - O.loss_value(kind, 1.0, lo)) / (2 * h)
            assert abs(fd - g[k]) < 1e-7 * max(1.0, abs(g[k]))
        checked += 1
    for _ in range(100):
        r = rng.uniform(-5, 5, 2)
        hv = O.loss_value(1, 1.3, r)
        half = 0.5 * float(r @ r)
        assert hv <= half + 1e-12
        if np.linalg.norm(r) <= 1.3:
            assert hv == pytest.approx(half, rel=1e-15)
