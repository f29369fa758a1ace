"""ORACLE — TEST INFRASTRUCTURE ONLY.

ctypes bindings for ``oracle/liboracle.so``, the Eigen-free CPU restatement of
the reference D-ADMM solver (/root/reference/proj/src/*.cpp; see oracle.hpp).
Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU-baseline leg may
import this module. The product package (paper_1708_07954_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")

DPTR = C.POINTER(C.c_double)
IPTR = C.POINTER(C.c_int)


class OracleError(RuntimeError):
    def __init__(self, msg, kind, point_id=-1, cam_id=-1, depth=0.0):
        super().__init__(msg)
        self.kind = kind
        self.point_id = point_id
        self.cam_id = cam_id
        self.depth = depth


KIND_NAMES = {1: "ValidationError", 2: "SizeMismatch", 3: "DepthBelowGuard",
              4: "SingularSystem", 7: "IndexOutOfRange", 8: "DuplicateObservation",
              10: "Error", 11: "ProjectionFailed"}


class Options(C.Structure):
    _fields_ = [("rho_x", C.c_double), ("rho_y", C.c_double), ("max_iters", C.c_int),
                ("primal_tol", C.c_double), ("stop_on_primal", C.c_int), ("loss", C.c_int),
                ("huber_delta", C.c_double), ("inner_max_iters", C.c_int),
                ("grad_tol", C.c_double), ("step_tol", C.c_double), ("lbfgs_memory", C.c_int),
                ("armijo_c", C.c_double), ("backtrack", C.c_double),
                ("max_line_search", C.c_int), ("eps_depth", C.c_double), ("workers", C.c_int),
                ("points_per_block", C.c_int), ("cameras_per_block", C.c_int)]


class Record(C.Structure):
    _fields_ = [("iter", C.c_int), ("mean_reproj_err", C.c_double),
                ("max_primal_x", C.c_double), ("max_primal_y", C.c_double),
                ("camera_mse", C.c_double), ("point_mse", C.c_double), ("wall_ms", C.c_double),
                ("comm_floats", C.c_longlong)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class SceneConfig(C.Structure):
    _fields_ = [("n_cameras", C.c_int), ("n_points", C.c_int), ("orbit_radius", C.c_double),
                ("altitude", C.c_double), ("box_min", C.c_double * 3),
                ("box_max", C.c_double * 3), ("jitter_trans", C.c_double),
                ("jitter_rot", C.c_double), ("visibility_window", C.c_int),
                ("focal", C.c_double), ("rng_seed", C.c_ulonglong)]


RES_CB = C.CFUNCTYPE(C.c_int, C.c_int, DPTR, C.c_int, DPTR, C.c_void_p)
JAC_CB = C.CFUNCTYPE(C.c_int, C.c_int, DPTR, C.c_int, DPTR, C.c_void_p)
VAL_CB = C.CFUNCTYPE(C.c_int, C.c_int, DPTR, DPTR, C.c_void_p)
GRAD_CB = C.CFUNCTYPE(C.c_int, C.c_int, DPTR, DPTR, C.c_void_p)

_lib = None


def build():
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = C.CDLL(_LIB_PATH)
        L.orc_last_error.restype = C.c_char_p
        L.orc_loss_value.restype = C.c_double
        L.orc_admm_block_objective.restype = C.c_double
        L.orc_admm_ops_per_iteration.restype = C.c_longlong
        L.orc_admm_comm_floats.restype = C.c_longlong
        _lib = L
    return _lib


def _p(a, t=DPTR):
    return None if a is None else a.ctypes.data_as(t)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


def check(rc):
    if rc != 0:
        L = lib()
        pt, cam, depth = C.c_int(), C.c_int(), C.c_double()
        L.orc_last_error_info(C.byref(pt), C.byref(cam), C.byref(depth))
        raise OracleError(L.orc_last_error().decode(), rc, pt.value, cam.value, depth.value)


def default_options(**kw):
    o = Options()
    lib().orc_options_default(C.byref(o))
    for k, v in kw.items():
        setattr(o, k, v)
    return o


# ---- geometry / losses -------------------------------------------------------
def rotation_from_euler(a, b, g):
    R = np.zeros(9)
    lib().orc_rotation_from_euler(C.c_double(a), C.c_double(b), C.c_double(g), _p(R))
    return R.reshape(3, 3)


def euler_from_rotation(R):
    R = _f64(R).reshape(9)
    out = np.zeros(3)
    lib().orc_euler_from_rotation(_p(R), _p(out))
    return out


def project(x, cam7, eps=1e-6):
    x, cam7 = _f64(x), _f64(cam7)
    z = np.zeros(2)
    ok = lib().orc_project(_p(x), _p(cam7), C.c_double(eps), _p(z))
    return z if ok else None


def project_with_jacobians(x, cam7, eps=1e-6):
    x, cam7 = _f64(x), _f64(cam7)
    z, Jp, Jc = np.zeros(2), np.zeros(6), np.zeros(12)
    ok = lib().orc_project_with_jacobians(_p(x), _p(cam7), C.c_double(eps), _p(z), _p(Jp), _p(Jc))
    return (z, Jp.reshape(2, 3), Jc.reshape(2, 6)) if ok else None


def loss_value(kind, delta, r):
    return lib().orc_loss_value(kind, C.c_double(delta), C.c_double(r[0]), C.c_double(r[1]))


def loss_gradient(kind, delta, r):
    g = np.zeros(2)
    lib().orc_loss_gradient(kind, C.c_double(delta), C.c_double(r[0]), C.c_double(r[1]), _p(g))
    return g


def ldlt_solve(A, b):
    A, b = _f64(A), _f64(b)
    x = np.zeros(len(b))
    lib().orc_ldlt_solve(len(b), _p(A), _p(b), _p(x))
    return x


def gauss_newton(residual, jacobian, x0, rows, **opts):
    n = len(x0)

    def rcb(n_, x, rows_, r, ctx):
        v = residual(np.ctypeslib.as_array(x, (n_,)).copy())
        if v is None:
            return 0
        np.ctypeslib.as_array(r, (rows_,))[:] = v
        return 1

    def jcb(n_, x, rows_, J, ctx):
        v = jacobian(np.ctypeslib.as_array(x, (n_,)).copy())
        if v is None:
            return 0
        np.ctypeslib.as_array(J, (rows_ * n_,))[:] = np.asarray(v, dtype=np.float64).reshape(-1)
        return 1

    rc_, jc_ = RES_CB(rcb), JAC_CB(jcb)
    o = default_options(**opts)
    x = np.zeros(n)
    obj, st, it = C.c_double(), C.c_int(), C.c_int()
    check(lib().orc_gauss_newton(n, rows, rc_, jc_, None, _p(_f64(x0)), C.byref(o), _p(x),
                                 C.byref(obj), C.byref(st), C.byref(it)))
    return x, obj.value, st.value, it.value


def lbfgs(value, grad, x0, **opts):
    n = len(x0)

    def vcb(n_, x, f, ctx):
        v = value(np.ctypeslib.as_array(x, (n_,)).copy())
        if v is None:
            return 0
        f[0] = v
        return 1

    def gcb(n_, x, g, ctx):
        v = grad(np.ctypeslib.as_array(x, (n_,)).copy())
        if v is None:
            return 0
        np.ctypeslib.as_array(g, (n_,))[:] = v
        return 1

    vc_, gc_ = VAL_CB(vcb), GRAD_CB(gcb)
    o = default_options(**opts)
    x = np.zeros(n)
    obj, st, it = C.c_double(), C.c_int(), C.c_int()
    check(lib().orc_lbfgs(n, vc_, gc_, None, _p(_f64(x0)), C.byref(o), _p(x), C.byref(obj),
                          C.byref(st), C.byref(it)))
    return x, obj.value, st.value, it.value


# ---- problem -----------------------------------------------------------------
class Problem:
    """Reference ``Problem`` (proj/include/dba/problem.hpp:44-56) as numpy arrays."""

    def __init__(self, handle):
        self.h = handle
        m, n, l = C.c_int(), C.c_int(), C.c_int()
        lib().orc_problem_sizes(self.h, C.byref(m), C.byref(n), C.byref(l))
        self.m, self.n, self.l = m.value, n.value, l.value
        self.obs_cam = np.zeros(self.l, np.int32)
        self.obs_pt = np.zeros(self.l, np.int32)
        self.obs_uv = np.zeros((self.l, 2))
        lib().orc_problem_observations(self.h, _p(self.obs_cam, IPTR), _p(self.obs_pt, IPTR),
                                       _p(self.obs_uv))
        self.cam_pose = np.zeros((self.m, 6))
        self.cam_f = np.zeros(self.m)
        self.points = np.zeros((self.n, 3))
        lib().orc_problem_nominal(self.h, _p(self.cam_pose), _p(self.cam_f), _p(self.points))

    @classmethod
    def create(cls, cam_pose, cam_f, points, obs_cam, obs_pt, obs_uv):
        cam_pose, cam_f, points = _f64(cam_pose), _f64(cam_f), _f64(points)
        obs_cam, obs_pt, obs_uv = _i32(obs_cam), _i32(obs_pt), _f64(obs_uv)
        h = C.c_void_p()
        check(lib().orc_problem_create(len(cam_f), len(points), len(obs_cam), _p(obs_cam, IPTR),
                                       _p(obs_pt, IPTR), _p(obs_uv), _p(cam_pose), _p(cam_f),
                                       _p(points), C.byref(h)))
        return cls(h)

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.orc_problem_destroy(self.h)
            self.h = None

    def visibility(self):
        pic_off, csp_off = np.zeros(self.m + 1, np.int32), np.zeros(self.n + 1, np.int32)
        pic, csp = np.zeros(self.l, np.int32), np.zeros(self.l, np.int32)
        lib().orc_problem_visibility(self.h, _p(pic_off, IPTR), _p(pic, IPTR), _p(csp_off, IPTR),
                                     _p(csp, IPTR))
        return ([pic[pic_off[j]:pic_off[j + 1]].tolist() for j in range(self.m)],
                [csp[csp_off[i]:csp_off[i + 1]].tolist() for i in range(self.n)])

    def mean_reprojection_error(self, pose, f, pts, eps=1e-6):
        out = C.c_double()
        check(lib().orc_mean_reprojection_error(self.h, _p(_f64(pose)), _p(_f64(f)),
                                                _p(_f64(pts)), len(f), len(pts), C.c_double(eps),
                                                C.byref(out)))
        return out.value

    def total_squared_error(self, pose, f, pts, eps=1e-6):
        out = C.c_double()
        check(lib().orc_total_squared_error(self.h, _p(_f64(pose)), _p(_f64(f)), _p(_f64(pts)),
                                            len(f), len(pts), C.c_double(eps), C.byref(out)))
        return out.value

    def communication_cost(self, ppb=1, cpb=1):
        out = C.c_longlong()
        check(lib().orc_communication_cost(self.h, ppb, cpb, C.byref(out)))
        return out.value

    def partition_count(self, ppb=1, cpb=1):
        out = C.c_int()
        check(lib().orc_partition_count(self.h, ppb, cpb, C.byref(out)))
        return out.value


def build_visibility_status(m, n, cams, pts):
    cams, pts = _i32(cams), _i32(pts)
    rc = lib().orc_build_visibility(m, n, len(cams), _p(cams, IPTR), _p(pts, IPTR))
    return rc, lib().orc_last_error().decode()


def parameter_mse(pose_a, pts_a, pose_b, pts_b):
    out = np.zeros(2)
    pa, xa, pb, xb = _f64(pose_a), _f64(pts_a), _f64(pose_b), _f64(pts_b)
    check(lib().orc_parameter_mse(len(pa), len(xa), _p(pa), _p(xa), len(pb), len(xb), _p(pb),
                                  _p(xb), _p(out)))
    return out[0], out[1]


def scene_config(**kw):
    c = SceneConfig()
    lib().orc_scene_config_default(C.byref(c))
    for k, v in kw.items():
        if k in ("box_min", "box_max"):
            getattr(c, k)[:] = v
        else:
            setattr(c, k, v)
    return c


def standard_scene_config(seed):
    """proj/tests/test_util.hpp:34-41 — 5 cameras, 10 points, window 5."""
    return scene_config(n_cameras=5, n_points=10, visibility_window=5, rng_seed=seed)


def generate_scene(cfg):
    h = C.c_void_p()
    check(lib().orc_generate_scene(C.byref(cfg), C.byref(h)))
    return Problem(h)


def perturb(pose, f, pts, sigma_cam, sigma_point, seed):
    pose, f, pts = _f64(pose), _f64(f), _f64(pts)
    po, xo = np.zeros_like(pose), np.zeros_like(pts)
    check(lib().orc_perturb(len(f), len(pts), _p(pose), _p(f), _p(pts), C.c_double(sigma_cam),
                            C.c_double(sigma_point), C.c_ulonglong(seed), _p(po), _p(xo)))
    return po, xo


class ConfigSceneInfo(C.Structure):
    """dbag_scene_info (include/dbag.h)."""
    _fields_ = [("config", C.c_int32), ("seed", C.c_uint64), ("scale", C.c_double),
                ("num_cameras", C.c_int32), ("num_points", C.c_int32), ("num_obs", C.c_int64),
                ("sigma_pixel", C.c_double), ("outlier_frac", C.c_double),
                ("sigma_init", C.c_double)]


def generate_config_scene(config, seed=0, scale=1.0):
    """BASELINE.json configs 1-5, built by the copy of the config
    generator compiled into liboracle.so (oracle/Makefile), so a CPU-only
    process (bench.py --impl reference) never loads the product library.
    Returns a dict of numpy arrays: obs_cam, obs_pt, obs_uv, cam_pose (ground
    truth), cam_f, points (ground truth), init_pose, init_pts."""
    L = lib()
    h = C.c_void_p()
    info = ConfigSceneInfo()
    rc = L.dbag_scene_generate(C.c_int32(config), C.c_uint64(seed), C.c_double(scale),
                               C.byref(h), C.byref(info))
    if rc != 0:
        raise OracleError(f"config scene generation failed ({rc})", rc)
    try:
        m, n, l = info.num_cameras, info.num_points, info.num_obs
        d = {"obs_cam": np.zeros(l, np.int32), "obs_pt": np.zeros(l, np.int32),
             "obs_uv": np.zeros((l, 2)), "cam_pose": np.zeros((m, 6)), "cam_f": np.zeros(m),
             "points": np.zeros((n, 3)), "init_pose": np.zeros((m, 6)),
             "init_pts": np.zeros((n, 3))}
        L.dbag_scene_fetch(h, _p(d["obs_cam"], IPTR), _p(d["obs_pt"], IPTR), _p(d["obs_uv"]),
                           _p(d["cam_pose"]), _p(d["cam_f"]), _p(d["points"]),
                           _p(d["init_pose"]), _p(d["init_pts"]))
    finally:
        L.dbag_scene_destroy(h)
    return d


def rng_draw(seed, kind, count, arg=0):
    out = np.zeros(count)
    lib().orc_rng_draw(C.c_ulonglong(seed), kind, C.c_ulonglong(arg), count, _p(out))
    return out


# ---- centralized LM (lm_solver.cpp) ---------------------------------------------
class LmOptions(C.Structure):
    _fields_ = [("max_iters", C.c_int), ("error_stop", C.c_double), ("lambda_init", C.c_double),
                ("lambda_max", C.c_double), ("lambda_up", C.c_double),
                ("lambda_down", C.c_double), ("use_schur", C.c_int), ("eps_depth", C.c_double)]


def lm_options(**kw):
    o = LmOptions()
    lib().orc_lm_options_default(C.byref(o))
    for k, v in kw.items():
        setattr(o, k, v)
    return o


def solve_lm(problem, pose, f, pts, options=None, loss=0, ref_pose=None, ref_pts=None, **kw):
    """solve_lm (lm_solver.hpp:51-54): returns (pose, pts, trace, stop, accepted)."""
    o = options if options is not None else lm_options(**kw)
    m, n = len(f), len(pts)
    out_pose, out_pts = np.zeros((m, 6)), np.zeros((n, 3))
    cap = o.max_iters + 2
    tr = (Record * cap)()
    nt, stop, acc = C.c_int(), C.c_int(), C.c_int()
    check(lib().orc_lm_solve(problem.h, _p(_f64(pose)), _p(_f64(f)), _p(_f64(pts)), C.byref(o),
                             loss, _p(None if ref_pose is None else _f64(ref_pose)),
                             _p(None if ref_pts is None else _f64(ref_pts)), _p(out_pose),
                             _p(out_pts), tr, cap, C.byref(nt), C.byref(stop), C.byref(acc)))
    return out_pose, out_pts, [tr[k].as_dict() for k in range(min(nt.value, cap))], stop.value, \
        acc.value


def lm_compute_step(problem, pose, f, pts, lam, use_schur=True, eps=1e-6):
    m, n = len(f), len(pts)
    dc, dp = np.zeros(6 * m), np.zeros(3 * n)
    check(lib().orc_lm_compute_step(problem.h, _p(_f64(pose)), _p(_f64(f)), _p(_f64(pts)),
                                    C.c_double(lam), int(use_schur), C.c_double(eps), _p(dc),
                                    _p(dp)))
    return dc, dp


# ---- ADMM solver -------------------------------------------------------------
class AdmmSolver:
    """Reference ``AdmmSolver`` (proj/include/dba/admm_solver.hpp:75-138)."""

    def __init__(self, problem, init_pose, init_f, init_pts, options=None, **kw):
        o = options if options is not None else default_options(**kw)
        self.problem = problem
        self.m, self.n = len(init_f), len(init_pts)
        self.h = C.c_void_p()
        check(lib().orc_admm_create(problem.h, self.m, self.n, _p(_f64(init_pose)),
                                    _p(_f64(init_f)), _p(_f64(init_pts)), C.byref(o),
                                    C.byref(self.h)))
        self.nblocks = lib().orc_admm_num_blocks(self.h)

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.orc_admm_destroy(self.h)
            self.h = None

    def local_update(self, b):
        check(lib().orc_admm_local_update(self.h, b))

    def local_update_all(self):
        check(lib().orc_admm_local_update_all(self.h))

    def consensus_update(self):
        check(lib().orc_admm_consensus_update(self.h))

    def dual_update(self):
        check(lib().orc_admm_dual_update(self.h))

    def iterate(self, ref_pose=None, ref_pts=None):
        r = Record()
        check(lib().orc_admm_iterate(self.h, _p(None if ref_pose is None else _f64(ref_pose)),
                                     _p(None if ref_pts is None else _f64(ref_pts)), C.byref(r)))
        return r.as_dict()

    def run(self, ref_pose=None, ref_pts=None, cap=100000):
        tr = (Record * cap)()
        n = C.c_int()
        check(lib().orc_admm_run(self.h, _p(None if ref_pose is None else _f64(ref_pose)),
                                 _p(None if ref_pts is None else _f64(ref_pts)), tr, cap,
                                 C.byref(n)))
        return [tr[k].as_dict() for k in range(min(n.value, cap))]

    def consensus(self):
        pose, f, pts = np.zeros((self.m, 6)), np.zeros(self.m), np.zeros((self.n, 3))
        lib().orc_admm_get_consensus(self.h, _p(pose), _p(f), _p(pts))
        return pose, f, pts

    def set_consensus(self, pose, pts):
        lib().orc_admm_set_consensus(self.h, _p(_f64(pose)), _p(_f64(pts)))

    def copies(self):
        nb = self.nblocks
        lp, lc, r, s = np.zeros((nb, 3)), np.zeros((nb, 6)), np.zeros((nb, 3)), np.zeros((nb, 6))
        lib().orc_admm_get_copies(self.h, _p(lp), _p(lc), _p(r), _p(s))
        return lp, lc, r, s

    def set_copies(self, lp, lc, r, s):
        lib().orc_admm_set_copies(self.h, _p(_f64(lp)), _p(_f64(lc)), _p(_f64(r)), _p(_f64(s)))

    def num_copies(self):
        pc, cc = C.c_longlong(), C.c_longlong()
        lib().orc_admm_num_copies(self.h, C.byref(pc), C.byref(cc))
        return pc.value, cc.value

    def copies_flat(self):
        """Copies of any BlockConfig, block by block in id order."""
        pc, cc = self.num_copies()
        lp, lc, r, s = np.zeros((pc, 3)), np.zeros((cc, 6)), np.zeros((pc, 3)), np.zeros((cc, 6))
        lib().orc_admm_copies_flat(self.h, _p(lp), _p(lc), _p(r), _p(s), 0)
        return lp, lc, r, s

    def set_copies_flat(self, lp, lc, r, s):
        lib().orc_admm_copies_flat(self.h, _p(_f64(lp)), _p(_f64(lc)), _p(_f64(r)), _p(_f64(s)), 1)

    def block_obs_ids(self):
        nb = self.nblocks
        np_, nc, no = (np.zeros(nb, np.int32) for _ in range(3))
        lib().orc_admm_block_sizes(self.h, _p(np_, IPTR), _p(nc, IPTR), _p(no, IPTR))
        pts, cams = np.zeros(np_.sum(), np.int32), np.zeros(nc.sum(), np.int32)
        obs, opl, ocl = (np.zeros(no.sum(), np.int32) for _ in range(3))
        lib().orc_admm_block_ids(self.h, _p(pts, IPTR), _p(cams, IPTR), _p(obs, IPTR),
                                 _p(opl, IPTR), _p(ocl, IPTR))
        return dict(n_points=np_, n_cams=nc, n_obs=no, point_ids=pts, cam_ids=cams, obs_ids=obs,
                    obs_point_local=opl, obs_cam_local=ocl)

    def max_primal(self):
        x, y = C.c_double(), C.c_double()
        lib().orc_admm_max_primal(self.h, C.byref(x), C.byref(y))
        return x.value, y.value

    def dual_sum_point(self, i):
        out = np.zeros(3)
        lib().orc_admm_dual_sum_point(self.h, i, _p(out))
        return out

    def dual_sum_camera(self, j):
        out = np.zeros(6)
        lib().orc_admm_dual_sum_camera(self.h, j, _p(out))
        return out

    def block_objective(self, b):
        return lib().orc_admm_block_objective(self.h, b)

    def ops_per_iteration(self):
        return lib().orc_admm_ops_per_iteration(self.h)

    def comm_floats(self):
        return lib().orc_admm_comm_floats(self.h)

    def iteration(self):
        return lib().orc_admm_iteration(self.h)
