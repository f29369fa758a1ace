"""CPU tests of the product boundary: libdbag.so builds for sm_100a, loads
without a GPU, and exports every entry point include/dbag.h declares; the
host-side scene generator (no device work) is deterministic and valid."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "dbag.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(dbag_[a-z_0-9]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_1708_07954_b200 import _capi
    return _capi.load()


def test_library_loads_and_exports_every_header_symbol(lib):
    from paper_1708_07954_b200 import _capi
    names = declared_functions()
    assert len(names) >= 30
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(_capi.SIGNATURES), "binding table out of sync with dbag.h"
    assert lib.dbag_abi_version() == 1


def test_library_is_sm100a_only():
    from paper_1708_07954_b200 import _capi
    out = subprocess.run(["cuobjdump", "--list-elf", _capi.LIB_PATH], capture_output=True,
                         text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout
    assert "sm_90" not in out.stdout and "sm_80" not in out.stdout


def test_options_default_mirror_reference(lib):
    # admm_solver.hpp:15-25, local_opt.hpp:11-19, geometry.hpp:50-52
    from paper_1708_07954_b200 import _capi
    o = _capi.Options()
    lib.dbag_options_default(ctypes.byref(o))
    assert (o.rho_x, o.rho_y, o.max_iters, o.primal_tol, o.stop_on_primal) == (1.0, 1.0, 1600,
                                                                                1e-6, 0)
    assert (o.inner_max_iters, o.grad_tol, o.step_tol, o.lbfgs_memory) == (10, 1e-8, 1e-10, 8)
    assert (o.armijo_c, o.backtrack, o.max_line_search, o.eps_depth) == (1e-4, 0.5, 40, 1e-6)
    assert (o.loss, o.huber_delta, o.workers) == (0, 1.0, 1)


def test_scene_sizes_and_determinism():
    import paper_1708_07954_b200 as P
    s1 = P.generate_config_scene(1, 0)
    assert (s1.problem.num_cameras, s1.problem.num_points, s1.problem.num_observations) == (
        8, 500, 4000)
    s1b = P.generate_config_scene(1, 0)
    assert np.array_equal(s1.problem.obs_uv, s1b.problem.obs_uv)
    assert np.array_equal(s1.init.cam_pose, s1b.init.cam_pose)
    assert not np.array_equal(s1.problem.obs_uv, P.generate_config_scene(1, 1).problem.obs_uv)
    s2 = P.generate_config_scene(2, 0)
    assert s2.problem.num_cameras == 64 and s2.problem.num_points == 20000
    assert 350_000 < s2.problem.num_observations < 420_000


def test_scene_valid_for_reference_problem(O):
    """The generated inputs satisfy Problem::create + AdmmSolver preconditions
    of the reference (restated by the oracle): coverage, no duplicates, feasible
    init; and gt reprojection error matches the injected pixel noise."""
    import paper_1708_07954_b200 as P
    for cfg, scale in ((1, 1.0), (2, 0.05), (3, 0.01), (4, 0.005), (5, 0.001)):
        s = P.generate_config_scene(cfg, 7, scale)
        p = s.problem
        op = O.Problem.create(p.cam_pose, p.cam_f, p.points, p.obs_cam, p.obs_pt, p.obs_uv)
        err = op.mean_reprojection_error(s.ground_truth.cam_pose, p.cam_f,
                                         s.ground_truth.points)
        if cfg <= 2:
            assert 1.0 < err < 1.5  # E||N(0, I2)|| = sqrt(pi/2)
        op.mean_reprojection_error(s.init.cam_pose, p.cam_f, s.init.points)  # feasible


def test_scene_camera_poses_look_at_points():
    import paper_1708_07954_b200 as P
    s = P.generate_config_scene(1, 0)
    # R(2,0) away from the Euler gimbal lock
    b = s.ground_truth.cam_pose[:, 1]
    assert np.all(np.abs(np.sin(b)) < 0.99)


def test_cpp_dropin_header_builds():
    """include/dbag.hpp (reference class names over the C-ABI) compiles and links:
    tools/dbag_solve.cpp is built against it by build.py."""
    from paper_1708_07954_b200 import build as b
    path = b.build_tools()
    assert os.path.exists(path)
    out = subprocess.run(["nm", "-D", "--undefined-only", path], capture_output=True, text=True)
    assert "dbag_create" in out.stdout and "dbag_run" in out.stdout
