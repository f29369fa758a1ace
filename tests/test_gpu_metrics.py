"""Metric extras: align_similarity (problem.cpp:204-237)
and rms_reprojection_error (problem.cpp:159-162) on the device path. Tolerance
parity: Eigen's JacobiSVD inside umeyama is not bit-pinnable, so the checker is
the reference's own KAT (proj/tests/test_problem.cpp:177-205, MSE < 1e-12) and
a numpy restatement of Umeyama's published algorithm (1e-10)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1708_07954_b200 as P
    return P


def umeyama_np(src, dst):
    """Umeyama (1991) with scaling, as Eigen/Umeyama.h evaluates it."""
    n = len(src)
    ms, md = src.mean(0), dst.mean(0)
    sd, dd = src - ms, dst - md
    sigma = dd.T @ sd / n
    U, S, Vt = np.linalg.svd(sigma)
    D = np.ones(3)
    if np.linalg.det(U) * np.linalg.det(Vt) < 0:
        D[2] = -1.0
    R = U @ np.diag(D) @ Vt
    c = (S @ D) / ((sd ** 2).sum() / n)
    return c * R, md - c * R @ ms


def gauge_move(O, pose, pts, s, Q, b):
    pts2 = (s * (Q @ pts.T)).T + b
    pose2 = pose.copy()
    for j in range(len(pose)):
        R = O.rotation_from_euler(*pose[j, :3])
        Rn = R @ Q.T
        pose2[j, :3] = O.euler_from_rotation(Rn)
        pose2[j, 3:] = s * pose[j, 3:] - Rn @ b
    return pose2, pts2


def test_align_similarity_undoes_known_gauge(O, P):
    # test_problem.cpp:177-205
    sc = O.generate_scene(O.standard_scene_config(10))
    Q = O.rotation_from_euler(0.3, -0.2, 0.5)
    pose2, pts2 = gauge_move(O, sc.cam_pose, sc.points, 1.7, Q, np.array([40.0, -25.0, 10.0]))
    assert sc.mean_reprojection_error(pose2, sc.cam_f, pts2) < 1e-6
    al = P.align_similarity(P.ParamState(pose2, sc.cam_f, pts2),
                            P.ParamState(sc.cam_pose, sc.cam_f, sc.points))
    cam_mse, pt_mse = O.parameter_mse(al.cam_pose, al.points, sc.cam_pose, sc.points)
    assert pt_mse < 1e-12 and cam_mse < 1e-12
    assert np.array_equal(al.cam_f, sc.cam_f)


def test_align_similarity_matches_umeyama_restatement(O, P):
    sc = O.generate_scene(O.standard_scene_config(21))
    ip, ix = O.perturb(sc.cam_pose, sc.cam_f, sc.points, 0.05, 0.2, 22)
    Q = O.rotation_from_euler(-0.7, 0.4, 1.1)
    pose2, pts2 = gauge_move(O, ip, ix, 0.6, Q, np.array([3.0, 2.0, -7.0]))
    al = P.align_similarity(P.ParamState(pose2, sc.cam_f, pts2),
                            P.ParamState(sc.cam_pose, sc.cam_f, sc.points))
    sQ, b = umeyama_np(pts2, sc.points)
    want = (sQ @ pts2.T).T + b
    assert np.abs(al.points - want).max() <= 1e-10 * (1 + np.abs(want).max())
    s = np.cbrt(np.linalg.det(sQ))
    Qa = sQ / s
    for j in range(len(pose2)):
        Rn = O.rotation_from_euler(*pose2[j, :3]) @ Qa.T
        assert np.abs(O.rotation_from_euler(*al.cam_pose[j, :3]) - Rn).max() <= 1e-10
        assert np.abs(al.cam_pose[j, 3:] - (s * pose2[j, 3:] - Rn @ b)).max() <= 1e-9


def test_align_similarity_size_errors(O, P):
    sc = O.generate_scene(O.standard_scene_config(3))
    st = P.ParamState(sc.cam_pose, sc.cam_f, sc.points)
    with pytest.raises(P.SizeMismatch):
        P.align_similarity(st, P.ParamState(sc.cam_pose, sc.cam_f, sc.points[:-1]))
    two = P.ParamState(sc.cam_pose, sc.cam_f, sc.points[:2])
    with pytest.raises(P.SizeMismatch):
        P.align_similarity(two, two)


def test_rms_reprojection_error(O, P):
    # test_problem.cpp:74-88: one camera, two points, one observation shifted by (3, 4)
    pose = np.array([[0, 0, 0, 0, 0, 10.0]])
    f = np.array([1.0])
    pts = np.array([[0, 0, 1.0], [1, 1, 1.0]])
    uv = np.array([O.project(pts[0], [*pose[0], 1.0]), O.project(pts[1], [*pose[0], 1.0])])
    uv[0] += [3.0, 4.0]
    prob = P.Problem.create(pose, f, pts, [0, 0], [0, 1], uv)
    g = P.AdmmSolver(prob, P.ParamState(pose, f, pts))
    assert abs(g.mean_reprojection_error() - 2.5) <= 2.5e-12
    assert abs(g.rms_reprojection_error() - np.sqrt(12.5)) <= 1e-12 * np.sqrt(12.5)
    assert g.rms_reprojection_error() == np.sqrt(g.total_squared_error() / 2)
