"""Pins the oracle's problem model, LDLT and inner solvers to the reference's
tests (proj/tests/test_problem.cpp, proj/tests/test_local_opt.cpp)."""
import math

import numpy as np
import pytest


def test_visibility_direct(O):
    # test_problem.cpp:16-24
    p = O.Problem.create(np.zeros((2, 6)) + [0, 0, 0, 0, 0, 5], [1, 1], np.zeros((2, 3)) + [0, 0, 1],
                         [0, 0, 1], [0, 1, 1], np.zeros((3, 2)))
    pic, csp = p.visibility()
    assert pic == [[0, 1], [1]]
    assert csp == [[0], [0, 1]]


@pytest.mark.parametrize("m,n,cams,pts,kind", [
    (1, 1, [], [], 1),                  # empty
    (1, 1, [0, 0], [0, 0], 8),          # duplicate
    (2, 1, [2], [0], 7),                # camera out of range
    (1, 3, [0], [5], 7),                # point out of range
    (2, 1, [0], [0], 1),                # camera 1 observes nothing
    (1, 2, [0], [0], 1),                # point 1 unobserved
])
def test_visibility_invalid(O, m, n, cams, pts, kind):
    # test_problem.cpp:26-35
    rc, _ = O.build_visibility_status(m, n, cams, pts)
    assert rc == kind


def test_mean_error_kats(O):
    # test_problem.cpp:74-88 — mean 2.5, total squared 25
    cam = np.array([[0, 0, 0, 0, 0, 10.0]])
    pts = np.array([[0, 0, 1.0], [1, 1, 1.0]])
    z0 = O.project(pts[0], [*cam[0], 1.0])
    z1 = O.project(pts[1], [*cam[0], 1.0])
    p = O.Problem.create(cam, [1.0], pts, [0, 0], [0, 1], [z0 + [3, 4], z1])
    assert p.mean_reprojection_error(cam, [1.0], pts) == pytest.approx(2.5, rel=1e-12)
    assert math.sqrt(p.total_squared_error(cam, [1.0], pts) / 2) == pytest.approx(math.sqrt(12.5),
                                                                                    rel=1e-12)


def test_mean_error_reports_offending_observation(O):
    # test_problem.cpp:113-127
    cam = np.array([[0, 0, 0, 0, 0, 2.0]])
    pts = np.array([[0, 0, 1.0]])
    p = O.Problem.create(cam, [1.0], pts, [0], [0], [O.project(pts[0], [*cam[0], 1.0])])
    with pytest.raises(O.OracleError) as e:
        p.mean_reprojection_error(cam, [1.0], [[0, 0, -5.0]])
    assert e.value.kind == 3 and e.value.point_id == 0 and e.value.cam_id == 0


def test_mean_error_exact_scene_and_order_independence(O):
    # test_problem.cpp:74-76, 90-111; test_scene_gen.cpp:21-29
    s = O.generate_scene(O.standard_scene_config(7))
    assert s.mean_reprojection_error(s.cam_pose, s.cam_f, s.points) == 0.0
    s8 = O.generate_scene(O.standard_scene_config(8))
    pose, pts = O.perturb(s8.cam_pose, s8.cam_f, s8.points, 0.01, 0.05, 99)
    direct = np.mean([np.linalg.norm(s8.obs_uv[k] - O.project(pts[s8.obs_pt[k]],
                                                               [*pose[s8.obs_cam[k]], s8.cam_f[0]]))
                      for k in range(s8.l)])
    assert s8.mean_reprojection_error(pose, s8.cam_f, pts) == pytest.approx(direct, rel=1e-12)
    perm = np.random.default_rng(42).permutation(s8.l)
    r = O.Problem.create(s8.cam_pose, s8.cam_f, s8.points, s8.obs_cam[perm], s8.obs_pt[perm],
                         s8.obs_uv[perm])
    assert r.mean_reprojection_error(pose, s8.cam_f, pts) == pytest.approx(
        s8.mean_reprojection_error(pose, s8.cam_f, pts), rel=1e-12)


def test_parameter_mse(O):
    # test_problem.cpp:129-166
    s = O.generate_scene(O.standard_scene_config(9))
    assert O.parameter_mse(s.cam_pose, s.points, s.cam_pose, s.points) == (0.0, 0.0)
    off = s.points.copy()
    off[3, 0] += 1.0
    c, p = O.parameter_mse(s.cam_pose, off, s.cam_pose, s.points)
    assert p == pytest.approx(1 / 30, rel=1e-15) and c == 0.0
    a = np.zeros((1, 6))
    b = a.copy()
    b[0, 0] = 2 * math.pi
    assert O.parameter_mse(a, np.zeros((1, 3)), b, np.zeros((1, 3)))[0] < 1e-24
    with pytest.raises(O.OracleError) as e:
        O.parameter_mse(np.zeros((2, 6)), np.zeros((3, 3)), np.zeros((2, 6)), np.zeros((4, 3)))
    assert e.value.kind == 2


def test_ldlt_matches_numpy(O):
    rng = np.random.default_rng(5)
    for n in (1, 2, 3, 9, 12):
        Q = rng.normal(size=(n, n))
        A = Q @ Q.T + 0.1 * np.eye(n)
        b = rng.normal(size=n)
        x = O.ldlt_solve(A, b)
        assert np.allclose(A @ x, b, rtol=1e-10, atol=1e-10)
    # indefinite but nonsingular: LDLT with pivoting still solves
    A = np.array([[0.0, 1.0], [1.0, 0.0]]) + np.diag([1e-3, -2.0])
    b = np.array([1.0, 2.0])
    assert np.allclose(A @ O.ldlt_solve(A, b), b)


def test_gauss_newton_linear_ls_one_step(O):
    # test_local_opt.cpp:46-63
    rng = np.random.default_rng(51)
    A, b = rng.normal(size=(6, 3)), rng.normal(size=6)
    expected = np.linalg.solve(A.T @ A, A.T @ b)
    x, obj, st, it = O.gauss_newton(lambda x: A @ x - b, lambda x: A, np.zeros(3), rows=6)
    assert np.linalg.norm(x - expected) < 1e-10
    assert it <= 2


def test_gauss_newton_stationary(O):
    # test_local_opt.cpp:65-74
    t = np.array([1.0, -2.0])
    x, obj, st, it = O.gauss_newton(lambda x: x - t, lambda x: np.eye(2), t, rows=2)
    assert st == 0 and it == 0 and np.array_equal(x, t)


def test_gauss_newton_monotone(O):
    # test_local_opt.cpp:128-156
    rng = np.random.default_rng(53)
    for _ in range(20):
        A, b = rng.normal(size=(5, 3)), rng.normal(size=5)

        def res(x):
            r = A @ x - b
            r[0] += 0.3 * math.sin(x[0])
            return r

        def jac(x):
            J = A.copy()
            J[0, 0] += 0.3 * math.cos(x[0])
            return J

        x0 = rng.normal(size=3)
        f0 = float(res(x0) @ res(x0))
        _, obj, _, _ = O.gauss_newton(res, jac, x0, rows=5)
        assert obj <= f0


def test_lbfgs_quadratic_rosenbrock_and_failures(O):
    # test_local_opt.cpp:158-220
    c = np.array([1.0, -2.0, 0.5])
    x, obj, st, it = O.lbfgs(lambda x: float((x - c) @ (x - c)), lambda x: 2 * (x - c),
                             np.zeros(3), inner_max_iters=100)
    assert st == 0 and np.linalg.norm(x - c) < 1e-8

    def rv(v):
        return 100 * (v[1] - v[0] ** 2) ** 2 + (1 - v[0]) ** 2

    def rg(v):
        return np.array([-400 * (v[1] - v[0] ** 2) * v[0] - 2 * (1 - v[0]), 200 * (v[1] - v[0] ** 2)])

    x, obj, st, it = O.lbfgs(rv, rg, np.array([-1.2, 1.0]), inner_max_iters=200, grad_tol=1e-10)
    assert abs(x[0] - 1) < 1e-6 and abs(x[1] - 1) < 1e-6

    x, obj, st, it = O.lbfgs(lambda x: 3.0, lambda x: np.zeros(2), np.array([4.0, 5.0]))
    assert st == 0 and it == 0 and list(x) == [4.0, 5.0]

    x0 = np.array([1.0, 1.0])
    x, obj, st, it = O.lbfgs(lambda x: None if np.linalg.norm(x - x0) > 0 else 1.0,
                             lambda x: np.array([1.0, 0.0]), x0)
    assert st == 4 and list(x) == [1.0, 1.0] and obj == 1.0


def test_lbfgs_monotone(O):
    # test_local_opt.cpp:222-250
    rng = np.random.default_rng(54)
    for _ in range(20):
        Q = rng.normal(size=(4, 4))
        H = Q.T @ Q + np.eye(4)
        b = rng.normal(size=4)
        x0 = rng.normal(size=4)

        def val(x):
            return 0.5 * x @ H @ x - b @ x + 0.1 * math.cos(x.sum())

        _, obj, _, _ = O.lbfgs(val, lambda x: H @ x - b - 0.1 * math.sin(x.sum()) * np.ones(4), x0)
        assert obj <= val(x0)
