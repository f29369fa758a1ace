"""Pins the oracle's ADMM solver and scene generator to the reference's own tests
(proj/tests/test_admm_solver.cpp, proj/tests/test_scene_gen.cpp)."""
import numpy as np
import pytest


def two_camera_problem(O):
    """test_admm_solver.cpp:18-26."""
    pose = np.array([[0, 0, 0, 0, 0, 5.0], [0, 0, 0, 0.5, -0.5, 6.0]])
    f = np.array([1.0, 1.0])
    pts = np.array([[0.1, -0.2, 1.0]])
    uv = [O.project(pts[0], [*pose[0], 1.0]), O.project(pts[0], [*pose[1], 1.0])]
    return O.Problem.create(pose, f, pts, [0, 1], [0, 0], uv), pose, f, pts


def scene(O, seed, **kw):
    cfg = O.standard_scene_config(seed)
    for k, v in kw.items():
        setattr(cfg, k, v)
    return O.generate_scene(cfg)


def test_partition_one_obs_per_block(O):
    # test_admm_solver.cpp:32-41
    s = scene(O, 81)
    assert s.partition_count(1, 1) == s.l
    assert s.partition_count(s.n, s.m) == 1


def test_partition_limits(O):
    # test_admm_solver.cpp:51-72
    s = scene(O, 83, n_cameras=9, n_points=40, visibility_window=4)
    for ppb, cpb in ((3, 2), (8, 1), (1, 5)):
        solver = O.AdmmSolver(s, s.cam_pose, s.cam_f, s.points, points_per_block=ppb,
                              cameras_per_block=cpb)
        b = solver.block_obs_ids()
        assert (b["n_points"] <= ppb).all() and (b["n_cams"] <= cpb).all()
        assert sorted(b["obs_ids"].tolist()) == list(range(s.l))


def test_block_order_is_cam_pt_sorted(O):
    s = scene(O, 81)
    solver = O.AdmmSolver(s, s.cam_pose, s.cam_f, s.points)
    obs = solver.block_obs_ids()["obs_ids"]
    keys = list(zip(s.obs_cam[obs], s.obs_pt[obs]))
    assert keys == sorted(keys)


def test_fixed_point(O):
    # test_admm_solver.cpp:74-101 (acceptance criterion 5)
    s = scene(O, 84)
    solver = O.AdmmSolver(s, s.cam_pose, s.cam_f, s.points)
    lp0, lc0, _, _ = solver.copies()
    pose0, _, pts0 = solver.consensus()
    solver.iterate()
    lp, lc, r, sd = solver.copies()
    pose, _, pts = solver.consensus()
    assert np.abs(lp - lp0).max() <= 1e-12 and np.abs(lc - lc0).max() <= 1e-12
    assert np.abs(r).max() <= 1e-12 and np.abs(sd).max() <= 1e-12
    assert np.abs(pts - pts0).max() <= 1e-12 and np.abs(pose - pose0).max() <= 1e-12


def test_huge_rho_pins_copies(O):
    # test_admm_solver.cpp:103-115
    p, pose, f, pts = two_camera_problem(O)
    solver = O.AdmmSolver(p, pose, f, pts, rho_x=1e12, rho_y=1e12)
    lp, lc, r, s = solver.copies()
    lp[0] += [0.05, -0.02, 0.03]
    lc[0] += [0.01, -0.01, 0.02, 0.1, -0.1, 0.05]
    solver.set_copies(lp, lc, r, s)
    solver.local_update(0)
    lp, lc, _, _ = solver.copies()
    assert np.linalg.norm(lp[0] - pts[0]) < 1e-6
    assert np.linalg.norm(lc[0] - pose[0]) < 1e-6


def test_gn_matches_lbfgs_block_objective(O):
    # test_admm_solver.cpp:117-180
    s = scene(O, 85)
    pose, pts = O.perturb(s.cam_pose, s.cam_f, s.points, 0.05, 0.3, 86)
    solver = O.AdmmSolver(s, pose, s.cam_f, pts, inner_max_iters=60)
    solver.iterate()
    solver.iterate()
    b = 7
    obs = solver.block_obs_ids()["obs_ids"][b]
    cpose, cf, cpts = solver.consensus()
    lp, lc, r, sd = solver.copies()
    cam, pt, z = s.obs_cam[obs], s.obs_pt[obs], s.obs_uv[obs]
    xb, yb, f = cpts[pt], cpose[cam], cf[cam]
    solver.local_update(b)
    gn_obj = solver.block_objective(b)

    def value(v):
        pr = O.project(v[:3], [*v[3:], f])
        if pr is None:
            return None
        res = z - pr
        dx, dy = v[:3] - xb, v[3:] - yb
        return float(res @ res + r[b] @ dx + sd[b] @ dy + 0.5 * dx @ dx + 0.5 * dy @ dy)

    def grad(v):
        e = O.project_with_jacobians(v[:3], [*v[3:], f])
        res = z - e[0]
        return np.concatenate([-2 * e[1].T @ res + r[b] + (v[:3] - xb),
                               -2 * e[2].T @ res + sd[b] + (v[3:] - yb)])

    v0 = np.concatenate([lp[b], lc[b]])
    _, lb_obj, _, _ = O.lbfgs(value, grad, v0, inner_max_iters=400, grad_tol=1e-10)
    assert abs(gn_obj - lb_obj) < 1e-6


def test_local_update_never_increases_block_objective(O):
    # test_admm_solver.cpp:182-192
    s = scene(O, 87)
    pose, pts = O.perturb(s.cam_pose, s.cam_f, s.points, 0.1, 0.5, 88)
    for loss in (0, 1):
        solver = O.AdmmSolver(s, pose, s.cam_f, pts, loss=loss)
        solver.iterate()
        for b in range(solver.nblocks):
            before = solver.block_objective(b)
            solver.local_update(b)
            assert solver.block_objective(b) <= before + 1e-12 * abs(before)


def test_consensus_kats(O):
    # test_admm_solver.cpp:194-211, 250-261
    p, pose, f, pts = two_camera_problem(O)
    solver = O.AdmmSolver(p, pose, f, pts, rho_x=2.0)
    lp, lc, r, s = solver.copies()
    lp[0], lp[1] = [1, 1, 1], [3, 3, 3]
    solver.set_copies(lp, lc, r, s)
    solver.consensus_update()
    assert list(solver.consensus()[2][0]) == [2, 2, 2]
    r[0], r[1] = [2, 2, 2], [-2, -2, -2]
    solver.set_copies(lp, lc, r, s)
    solver.consensus_update()
    assert list(solver.consensus()[2][0]) == [2, 2, 2]

    solver = O.AdmmSolver(p, pose, f, pts, rho_x=2.0)
    lp, lc, r, s = solver.copies()
    lp[0] = pts[0] + [1, 0, -1]
    solver.set_copies(lp, lc, r, s)
    solver.dual_update()
    _, _, r, _ = solver.copies()
    assert list(r[0]) == [2, 0, -2] and list(r[1]) == [0, 0, 0]


def test_consensus_recomputation(O):
    # test_admm_solver.cpp:213-248
    s = scene(O, 89)
    solver = O.AdmmSolver(s, s.cam_pose, s.cam_f, s.points, rho_x=1.7, rho_y=0.3)
    rng = np.random.default_rng(90)
    lp, lc, r, sd = solver.copies()
    lp += rng.normal(size=lp.shape)
    r = rng.normal(size=r.shape)
    solver.set_copies(lp, lc, r, sd)
    solver.consensus_update()
    obs = solver.block_obs_ids()["obs_ids"]
    _, _, pts = solver.consensus()
    for i in range(s.n):
        sel = s.obs_pt[obs] == i
        mean = (lp[sel] + r[sel] / 1.7).mean(axis=0)
        assert np.linalg.norm(pts[i] - mean) < 1e-12 * (1 + np.linalg.norm(mean))


def test_dual_sums_vanish(O):
    # test_admm_solver.cpp:263-312 (acceptance criterion 4)
    s = scene(O, 91)
    solver = O.AdmmSolver(s, s.cam_pose, s.cam_f, s.points)
    rng = np.random.default_rng(92)
    lp, lc, r, sd = solver.copies()
    lp += 5 * rng.normal(size=lp.shape)
    lc += rng.normal(size=lc.shape)
    r = 10 * rng.normal(size=r.shape)
    sd = 10 * rng.normal(size=sd.shape)
    solver.set_copies(lp, lc, r, sd)
    solver.consensus_update()
    solver.dual_update()
    _, _, r, sd = solver.copies()
    mx = max(np.linalg.norm(r, axis=1).max(), np.linalg.norm(sd, axis=1).max())
    for i in range(s.n):
        assert np.linalg.norm(solver.dual_sum_point(i)) <= 1e-9 * (1 + mx)
    for j in range(s.m):
        assert np.linalg.norm(solver.dual_sum_camera(j)) <= 1e-9 * (1 + mx)


def test_converges_on_standard_scene(O):
    # test_admm_solver.cpp:314-333 (acceptance criterion 2)
    s = scene(O, 93)
    pose, pts = O.perturb(s.cam_pose, s.cam_f, s.points, 0.01, 0.01, 94)
    solver = O.AdmmSolver(s, pose, s.cam_f, pts, stop_on_primal=1, primal_tol=1e-6)
    trace = solver.run(s.cam_pose, s.points)
    assert any(t["mean_reproj_err"] < 1e-3 and max(t["max_primal_x"], t["max_primal_y"]) < 1e-4
               for t in trace)
    fpose, _, fpts = solver.consensus()
    c0, p0 = O.parameter_mse(pose, pts, s.cam_pose, s.points)
    c1, p1 = O.parameter_mse(fpose, fpts, s.cam_pose, s.points)
    assert p1 <= p0 and c1 <= c0


def test_comm_cost_kats(O):
    # test_admm_solver.cpp:366-381 (acceptance criterion 6: 3(d-1)dn)
    s = scene(O, 97, visibility_window=3)
    assert s.communication_cost() == 180
    for w in (2, 3, 5):
        for n in (10, 100):
            sc = scene(O, 97 + w + n, visibility_window=w, n_points=n)
            assert sc.communication_cost() == 3 * (w - 1) * w * n
    pose = np.array([[0, 0, 0, 0, 0, 5.0], [0, 0, 0, 1, 0, 5.0]])
    pts = np.array([[0, 0, 1.0], [0.5, 0, 1.0]])
    p = O.Problem.create(pose, [1, 1], pts, [0, 1], [0, 1],
                         [O.project(pts[0], [*pose[0], 1]), O.project(pts[1], [*pose[1], 1])])
    assert p.communication_cost() == 0


def test_ops_linear_and_worker_determinism(O):
    # test_admm_solver.cpp:422-458 (acceptance criterion 8)
    a = scene(O, 99)
    b = scene(O, 99, n_points=20)
    sa = O.AdmmSolver(a, a.cam_pose, a.cam_f, a.points)
    sb = O.AdmmSolver(b, b.cam_pose, b.cam_f, b.points)
    assert 2 * sa.ops_per_iteration() == sb.ops_per_iteration()
    s = scene(O, 100)
    pose, pts = O.perturb(s.cam_pose, s.cam_f, s.points, 0.05, 0.2, 101)
    ref = None
    for workers in (1, 2, 8):
        solver = O.AdmmSolver(s, pose, s.cam_f, pts, max_iters=40, workers=workers)
        solver.run()
        out = solver.consensus()
        if ref is None:
            ref = out
        else:
            assert np.abs(out[0] - ref[0]).max() <= 1e-12 and np.abs(out[2] - ref[2]).max() <= 1e-12


def test_invalid_options(O):
    # test_admm_solver.cpp:487-499
    s = scene(O, 104)
    for kw, kind in (({"rho_x": 0.0}, 1), ({"workers": 0}, 1), ({"points_per_block": 0}, 1)):
        with pytest.raises(O.OracleError) as e:
            O.AdmmSolver(s, s.cam_pose, s.cam_f, s.points, **kw)
        assert e.value.kind == kind
    with pytest.raises(O.OracleError) as e:
        O.AdmmSolver(s, s.cam_pose, s.cam_f, s.points[:-1])
    assert e.value.kind == 2


def test_scene_gen_kats(O):
    # test_scene_gen.cpp:14-48, 66-82
    s = scene(O, 1)
    assert (s.m, s.n, s.l) == (5, 10, 50)
    s2 = scene(O, 2)
    for k in range(s2.l):
        z = O.project(s2.points[s2.obs_pt[k]], [*s2.cam_pose[s2.obs_cam[k]], s2.cam_f[0]])
        assert np.array_equal(z, s2.obs_uv[k])
    a, b = scene(O, 3), scene(O, 3)
    assert np.array_equal(a.obs_uv, b.obs_uv) and np.array_equal(a.points, b.points)
    assert not np.array_equal(a.points[0], scene(O, 4).points[0])
    s6 = scene(O, 6, n_cameras=7, visibility_window=3)
    _, csp = s6.visibility()
    for cams in csp:
        assert any(sorted([(st + k) % 7 for k in range(3)]) == cams for st in range(7))


def test_perturb_properties(O):
    # test_scene_gen.cpp:84-126
    s = scene(O, 7)
    pose, pts = O.perturb(s.cam_pose, s.cam_f, s.points, 0.0, 0.0, 1)
    assert np.array_equal(pose, s.cam_pose) and np.array_equal(pts, s.points)
    a = O.perturb(s.cam_pose, s.cam_f, s.points, 0.1, 0.5, 42)
    b = O.perturb(s.cam_pose, s.cam_f, s.points, 0.1, 0.5, 42)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    s8 = scene(O, 8)
    mse = np.mean([O.parameter_mse(*O.perturb(s8.cam_pose, s8.cam_f, s8.points, 0.0, 1.0, seed),
                                   s8.cam_pose, s8.points)[1] for seed in range(100)])
    assert abs(mse - 1.0) < 3.0 * np.sqrt(2.0 / 30 / 100)
    with pytest.raises(O.OracleError):
        O.perturb(s.cam_pose, s.cam_f, s.points, -0.1, 0.0, 1)


def test_golden_fixture(O):
    """Oracle against the committed golden trajectory (tests/golden/, made by
    tests/golden/make_golden.py from this oracle at the commit that pinned it
    against every KAT above): guards the oracle against silent drift."""
    import json
    import os
    path = os.path.join(os.path.dirname(__file__), "golden", "oracle_trajectories.json")
    gold = json.load(open(path))
    for case in gold["cases"]:
        s = scene(O, case["seed"])
        pose, pts = O.perturb(s.cam_pose, s.cam_f, s.points, case["sigma_cam"], case["sigma_point"],
                              case["seed"] + 1)
        solver = O.AdmmSolver(s, pose, s.cam_f, pts, max_iters=case["rounds"], loss=case["loss"])
        trace = solver.run(s.cam_pose, s.points)
        for got, want in zip(trace, case["trace"]):
            for k in ("mean_reproj_err", "max_primal_x", "max_primal_y", "camera_mse", "point_mse"):
                assert got[k] == pytest.approx(want[k], rel=1e-12, abs=1e-300), k
        fpose, _, fpts = solver.consensus()
        assert np.allclose(fpose, case["final_pose"], rtol=1e-12, atol=0)
        assert np.allclose(fpts, case["final_pts"], rtol=1e-12, atol=0)
