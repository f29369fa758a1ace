"""Centralized LM comparator on the device (lm_solver.cpp):
the reference's own LM tests (proj/tests/test_lm_solver.cpp) through the C-ABI,
and parity with the oracle's restatement. The dense camera system is factored
by cuSOLVER (Eigen's blocked LDLT is not bit-pinnable), so parity is
tolerance-level: steps 1e-9 relative, trajectories 1e-8."""
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


def scene(O, seed):
    return O.generate_scene(O.standard_scene_config(seed))


def gprob(P, s):
    return P.Problem.create(s.cam_pose, s.cam_f, s.points, s.obs_cam, s.obs_pt, s.obs_uv)


def test_ground_truth_terminates_immediately(O, P):
    s = scene(O, 61)
    r = P.solve_lm(gprob(P, s), P.ParamState(s.cam_pose, s.cam_f, s.points))
    assert r.stop == 0 and r.accepted_steps == 0
    assert s.total_squared_error(r.state.cam_pose, s.cam_f, r.state.points) < 1e-14


def test_converges_from_perturbed_init(O, P):
    s = scene(O, 62)
    ip, ix = O.perturb(s.cam_pose, s.cam_f, s.points, 0.01, 0.01, 63)
    r = P.solve_lm(gprob(P, s), P.ParamState(ip, s.cam_f, ix),
                   reference=P.ParamState(s.cam_pose, s.cam_f, s.points))
    assert len(r.trace) <= 101
    assert s.mean_reprojection_error(r.state.cam_pose, s.cam_f, r.state.points) < 1e-6
    assert r.trace[0]["iter"] == 0 and not np.isnan(r.trace[-1]["point_mse"])


def test_total_error_decreases_until_error_stop(O, P):
    s = scene(O, 64)
    ip, ix = O.perturb(s.cam_pose, s.cam_f, s.points, 0.02, 0.1, 65)
    prev = s.total_squared_error(ip, s.cam_f, ix)
    stopped = False
    for budget in range(1, 9):
        r = P.solve_lm(gprob(P, s), P.ParamState(ip, s.cam_f, ix), P.LmOptions(max_iters=budget))
        now = s.total_squared_error(r.state.cam_pose, s.cam_f, r.state.points)
        assert (now == prev and r.stop == 0) if stopped else now < prev
        stopped = stopped or r.stop == 0
        prev = now


def test_schur_and_dense_steps_agree(O, P):
    s = scene(O, 66)
    ip, ix = O.perturb(s.cam_pose, s.cam_f, s.points, 0.05, 0.2, 67)
    st = P.ParamState(ip, s.cam_f, ix)
    for lam in (1e-3, 1.0):
        a = P.lm_compute_step(gprob(P, s), st, lam, True)
        b = P.lm_compute_step(gprob(P, s), st, lam, False)
        scale = max(1e-30, np.linalg.norm(b[0]), np.linalg.norm(b[1]))
        assert np.linalg.norm(a[0] - b[0]) / scale < 1e-8
        assert np.linalg.norm(a[1] - b[1]) / scale < 1e-8


def test_schur_solve_equals_dense_solve(O, P):
    s = scene(O, 68)
    ip, ix = O.perturb(s.cam_pose, s.cam_f, s.points, 0.01, 0.05, 69)
    a = P.solve_lm(gprob(P, s), P.ParamState(ip, s.cam_f, ix), P.LmOptions(max_iters=10))
    b = P.solve_lm(gprob(P, s), P.ParamState(ip, s.cam_f, ix),
                   P.LmOptions(max_iters=10, use_schur=False))
    cam_mse, pt_mse = O.parameter_mse(a.state.cam_pose, a.state.points, b.state.cam_pose,
                                      b.state.points)
    assert cam_mse < 1e-12 and pt_mse < 1e-12


def test_rejects_non_l2_and_infeasible_init(O, P):
    s = scene(O, 70)
    with pytest.raises(P.ValidationError):
        P.solve_lm(gprob(P, s), P.ParamState(s.cam_pose, s.cam_f, s.points), loss=P.LossKind.huber(1.0))
    s = scene(O, 71)
    pts = s.points.copy()
    pts[0] = [0, 0, 1e7]
    with pytest.raises(P.DepthBelowGuard) as e:
        P.solve_lm(gprob(P, s), P.ParamState(s.cam_pose, s.cam_f, pts))
    assert e.value.point_id == 0


@pytest.mark.parametrize("seed,lam,schur", [(66, 1e-3, True), (66, 1.0, True), (72, 1e-2, True),
                                            (66, 1e-3, False)])
def test_step_matches_oracle(O, P, seed, lam, schur):
    s = scene(O, seed)
    ip, ix = O.perturb(s.cam_pose, s.cam_f, s.points, 0.05, 0.2, seed + 1)
    g = P.lm_compute_step(gprob(P, s), P.ParamState(ip, s.cam_f, ix), lam, schur)
    o = O.lm_compute_step(s, ip, s.cam_f, ix, lam, schur)
    for a, b in zip(g, o):
        assert np.linalg.norm(a - b) <= 1e-9 * max(1e-30, np.linalg.norm(b))


def test_trajectory_matches_oracle(O, P):
    s = scene(O, 62)
    ip, ix = O.perturb(s.cam_pose, s.cam_f, s.points, 0.03, 0.1, 63)
    r = P.solve_lm(gprob(P, s), P.ParamState(ip, s.cam_f, ix), P.LmOptions(max_iters=20),
                   reference=P.ParamState(s.cam_pose, s.cam_f, s.points))
    opose, opts, otr, ostop, oacc = O.solve_lm(s, ip, s.cam_f, ix, max_iters=20,
                                               ref_pose=s.cam_pose, ref_pts=s.points)
    assert r.stop == ostop and r.accepted_steps == oacc and len(r.trace) == len(otr)
    for g, o in zip(r.trace, otr):
        assert g["iter"] == o["iter"]
        a, b = g["mean_reproj_err"], o["mean_reproj_err"]
        assert abs(a - b) <= 1e-8 * b + 1e-12
    assert np.abs(r.state.points - opts).max() <= 1e-8 * (1 + np.abs(opts).max())


def test_config2_scene_matches_oracle(O, P):
    # 64 cameras (S is 384 x 384), 20k points, 384k observations: 3 LM iterations
    sc = P.generate_config_scene(2, 0, 1.0)
    p = sc.problem
    oprob = O.Problem.create(p.cam_pose, p.cam_f, p.points, p.obs_cam, p.obs_pt, p.obs_uv)
    r = P.solve_lm(p, sc.init, P.LmOptions(max_iters=3))
    opose, opts, otr, ostop, oacc = O.solve_lm(oprob, sc.init.cam_pose, p.cam_f, sc.init.points,
                                               max_iters=3)
    assert r.accepted_steps == oacc and len(r.trace) == len(otr)
    for g, o in zip(r.trace, otr):
        assert abs(g["mean_reproj_err"] - o["mean_reproj_err"]) <= 1e-8 * o["mean_reproj_err"]
    assert np.abs(r.state.cam_pose - opose).max() <= 1e-7
