"""CPU checks of the oracle's own plumbing (test infrastructure):

- the BASELINE config generator compiled into liboracle.so (oracle/Makefile)
  builds the same scenes, bit for bit, as the product library's build of it,
  so bench.py's reference arm can generate its workload without loading
  libdbag.so;
- the WorkerPool restatement (proj/src/parallel.cpp:5-91) no longer crashes
  when a worker wakes after run() has finished (a late worker read
  fn_ == nullptr and could call through it once the next run() reset the
  counters; this reproduced as a SIGSEGV with 16 workers on tiny problems).
"""
import time

import numpy as np
import pytest


@pytest.mark.parametrize("config,scale", [(1, 1.0), (2, 1.0), (3, 0.05), (4, 0.02), (5, 0.01)])
def test_oracle_scene_generator_matches_product(O, config, scale):
    import paper_1708_07954_b200 as P
    s = P.generate_config_scene(config, 0, scale)
    d = O.generate_config_scene(config, 0, scale)
    p = s.problem
    for a, b in ((p.obs_cam, d["obs_cam"]), (p.obs_pt, d["obs_pt"]), (p.obs_uv, d["obs_uv"]),
                 (p.cam_pose, d["cam_pose"]), (p.cam_f, d["cam_f"]), (p.points, d["points"]),
                 (s.init.cam_pose, d["init_pose"]), (s.init.points, d["init_pts"])):
        assert a.dtype == b.dtype and a.shape == b.shape
        assert np.array_equal(a.view(np.uint8), b.view(np.uint8))


def test_worker_pool_late_wakeup_does_not_crash(O):
    """Many short run() calls with more workers than blocks: the window where
    a worker wakes after its generation finished is hit thousands of times.
    Results must also stay bitwise independent of the worker count."""
    s = O.generate_scene(O.standard_scene_config(85))
    ip, ix = O.perturb(s.cam_pose, s.cam_f, s.points, 0.05, 0.3, 86)
    t0 = time.time()
    for rep in range(6):
        for loss in (0, 1):
            a = O.AdmmSolver(s, ip, s.cam_f, ix, workers=16, loss=loss, max_iters=100)
            b = O.AdmmSolver(s, ip, s.cam_f, ix, workers=1, loss=loss, max_iters=100)
            for _ in range(40):
                ra, rb = a.iterate(), b.iterate()
                assert ra["max_primal_x"] == rb["max_primal_x"]
            assert all(np.array_equal(x, y) for x, y in zip(a.copies(), b.copies()))
    assert time.time() - t0 < 120
