"""Generalized blocks, host side: libdbag's partition() / communication_cost()
(admm_solver.cpp:14-101) against the oracle, bit for bit, and the reference's
own partition / communication tests (proj/tests/test_admm_solver.cpp:32-72,
366-430). No GPU: dbag_partition is host code in the library."""
import itertools

import numpy as np
import pytest

CONFIGS = [(1, 1), (3, 2), (8, 1), (1, 5), (4, 2), (3, 1), (32, 1), (2, 3), (64, 4)]


@pytest.fixture(scope="module")
def P():
    import paper_1708_07954_b200 as P
    return P


def scene(O, seed, **kw):
    cfg = O.standard_scene_config(seed)
    for k, v in kw.items():
        setattr(cfg, k, v)
    return O.generate_scene(cfg)


def gpu_problem(P, s):
    return P.Problem.create(s.cam_pose, s.cam_f, s.points, s.obs_cam, s.obs_pt, s.obs_uv)


@pytest.mark.parametrize("seed,kw", [(83, dict(n_cameras=9, n_points=40, visibility_window=4)),
                                     (98, dict(n_cameras=9, n_points=25, visibility_window=4)),
                                     (7, {}), (81, {})])
def test_partition_equals_oracle(O, P, seed, kw):
    s = scene(O, seed, **kw)
    prob = gpu_problem(P, s)
    for ppb, cpb in CONFIGS:
        ob = O.AdmmSolver(s, s.cam_pose, s.cam_f, s.points, points_per_block=ppb,
                          cameras_per_block=cpb).block_obs_ids()
        blocks = P.partition(prob, ppb, cpb)
        assert len(blocks) == len(ob["n_points"])
        assert np.array_equal(np.concatenate([b.point_ids for b in blocks]), ob["point_ids"])
        assert np.array_equal(np.concatenate([b.cam_ids for b in blocks]), ob["cam_ids"])
        assert np.array_equal(np.concatenate([b.obs_ids for b in blocks]), ob["obs_ids"])
        assert np.array_equal(np.concatenate([b.obs_point_local for b in blocks]),
                              ob["obs_point_local"])
        assert np.array_equal(np.concatenate([b.obs_cam_local for b in blocks]),
                              ob["obs_cam_local"])
        assert P.communication_cost(prob, ppb, cpb) == s.communication_cost(ppb, cpb)


def test_partition_limits_and_coverage(O, P):
    # test_admm_solver.cpp:51-72
    s = scene(O, 83, n_cameras=9, n_points=40, visibility_window=4)
    prob = gpu_problem(P, s)
    for ppb, cpb in ((3, 2), (8, 1), (1, 5)):
        seen = []
        for b in P.partition(prob, ppb, cpb):
            assert len(b.point_ids) <= ppb and len(b.cam_ids) <= cpb
            for o, pl, cl in zip(b.obs_ids, b.obs_point_local, b.obs_cam_local):
                assert b.point_ids[pl] == s.obs_pt[o] and b.cam_ids[cl] == s.obs_cam[o]
            seen += b.obs_ids.tolist()
        assert sorted(seen) == list(range(s.l))


def test_single_and_whole_blocks(O, P):
    # test_admm_solver.cpp:32-41: (1,1) -> one block per observation; (n,m) -> one
    s = scene(O, 81)
    prob = gpu_problem(P, s)
    assert len(P.partition(prob, 1, 1)) == s.l
    whole = P.partition(prob, s.n, s.m)
    assert len(whole) == 1 and len(whole[0].obs_ids) == s.l


def test_communication_cost_uniform_window(O, P):
    # test_admm_solver.cpp:366-381: d = 3 cameras per point, n = 10 -> 180; isolated -> 0
    s = scene(O, 97, visibility_window=3)
    assert P.communication_cost(gpu_problem(P, s), 1, 1) == 180
    pose = np.array([[0, 0, 0, 0, 0, 5.0], [0, 0, 0, 1, 0, 5.0]])
    f = np.ones(2)
    pts = np.array([[0, 0, 1.0], [0.5, 0, 1.0]])
    uv = [O.project(pts[0], [*pose[0], 1.0]), O.project(pts[1], [*pose[1], 1.0])]
    iso = P.Problem.create(pose, f, pts, [0, 1], [0, 1], uv)
    assert P.communication_cost(iso, 1, 1) == 0


def test_communication_cost_message_simulation(O, P):
    # test_admm_solver.cpp:383-430: replay every directed transfer between owners
    s = scene(O, 98, n_cameras=9, n_points=25, visibility_window=4)
    prob = gpu_problem(P, s)
    for ppb, cpb in ((1, 1), (4, 2), (3, 1)):
        blocks = P.partition(prob, ppb, cpb)
        pts, cams = [set() for _ in range(s.n)], [set() for _ in range(s.m)]
        for b in blocks:
            owner = int(b.cam_ids[0])
            for i in b.point_ids:
                pts[i].add(owner)
            for j in b.cam_ids:
                cams[j].add(owner)
        msgs = 0
        for owners, dim in ((pts, 3), (cams, 6)):
            for procs in owners:
                msgs += dim * sum(1 for a, c in itertools.product(procs, procs) if a != c)
        assert P.communication_cost(prob, ppb, cpb) == msgs


def test_block_size_validation(O, P):
    s = scene(O, 81)
    prob = gpu_problem(P, s)
    for bad in ((0, 1), (1, 0), (-3, 2)):
        with pytest.raises(P.ValidationError):
            P.partition(prob, *bad)


def test_partition_fuzz_against_oracle(O, P):
    """Random scenes and block sizes: libdbag's partition() and communication_cost()
    equal the oracle's, bit for bit."""
    rng = np.random.default_rng(1234)
    for trial in range(12):
        kw = dict(n_cameras=int(rng.integers(3, 14)), n_points=int(rng.integers(10, 60)),
                  visibility_window=int(rng.integers(2, 6)))
        s = scene(O, int(rng.integers(0, 10_000)), **kw)
        prob = gpu_problem(P, s)
        ppb, cpb = int(rng.integers(1, 40)), int(rng.integers(1, 7))
        ob = O.AdmmSolver(s, s.cam_pose, s.cam_f, s.points, points_per_block=ppb,
                          cameras_per_block=cpb).block_obs_ids()
        blocks = P.partition(prob, ppb, cpb)
        assert np.array_equal(np.concatenate([b.obs_ids for b in blocks]), ob["obs_ids"])
        assert np.array_equal(np.concatenate([b.point_ids for b in blocks]), ob["point_ids"])
        assert np.array_equal(np.concatenate([b.cam_ids for b in blocks]), ob["cam_ids"])
        assert [len(b.point_ids) for b in blocks] == ob["n_points"].tolist()
        assert P.communication_cost(prob, ppb, cpb) == s.communication_cost(ppb, cpb)
