"""Host-side mirror of the reference solver API over the B200 C-ABI.

Mirrors proj/include/dba/{admm_solver,problem,trace,errors}.hpp: the same
class and method names, argument meaning and exception types, so tests read
like the reference's own (proj/tests/test_admm_solver.cpp). Every compute call
goes through libdbag.so (include/dbag.h); nothing here computes on the CPU.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _capi

# ---- errors (proj/include/dba/errors.hpp:9-72) -------------------------------


class Error(RuntimeError):
    """dba::Error."""


class ValidationError(Error):
    """dba::ValidationError."""


class SizeMismatch(ValidationError):
    pass


class IndexOutOfRange(ValidationError):
    pass


class DuplicateObservation(ValidationError):
    pass


class DepthBelowGuard(Error):
    def __init__(self, msg, depth=0.0, point_id=-1, cam_id=-1):
        super().__init__(msg)
        self.depth, self.point_id, self.cam_id = depth, point_id, cam_id


class SingularSystem(Error):
    pass


class ParseError(ValidationError):
    """dba::ParseError (errors.hpp:16-22): carries the 1-based line."""

    def __init__(self, msg, line=-1):
        super().__init__(msg)
        self.line = line


class DeviceError(Error):
    """CUDA / NCCL failure (no reference analogue)."""


class Unsupported(Error):
    """Valid for the reference but not built on the device (e.g. (pi,kappa) > 1 blocks)."""


_STATUS = {1: ValidationError, 2: SizeMismatch, 3: DepthBelowGuard, 4: SingularSystem,
           5: DeviceError, 6: DeviceError, 7: IndexOutOfRange, 8: DuplicateObservation,
           9: Unsupported, 10: Error}


def _check(rc):
    if rc == 0:
        return
    lib = _capi.load()
    msg = lib.dbag_last_error().decode()
    pt, cam, blk = C.c_int32(), C.c_int32(), C.c_int64()
    depth = C.c_double()
    lib.dbag_last_error_info(C.byref(pt), C.byref(cam), C.byref(depth), C.byref(blk))
    cls = _STATUS.get(rc, Error)
    if cls is DepthBelowGuard:
        raise DepthBelowGuard(msg, depth.value, pt.value, cam.value)
    err = cls(msg)
    err.block = blk.value
    raise err


def _f64(a, shape=None):
    a = np.ascontiguousarray(a, dtype=np.float64)
    if shape is not None:
        a = a.reshape(shape)
    return a


def _dp(a):
    return None if a is None else a.ctypes.data_as(_capi.DPTR)


def _ip(a):
    return a.ctypes.data_as(_capi.I32P)


# ---- data model (proj/include/dba/problem.hpp, geometry.hpp) -------------------


@dataclass
class ParamState:
    """problem.hpp:36-41. cam_pose rows are (alpha, beta, gamma, t1, t2, t3)."""
    cam_pose: np.ndarray
    cam_f: np.ndarray
    points: np.ndarray

    def copy(self):
        return ParamState(self.cam_pose.copy(), self.cam_f.copy(), self.points.copy())

    def as_f64(self):
        """float64, C-contiguous views of the arrays (a copy only where needed);
        the caller's object is not modified."""
        return ParamState(_f64(self.cam_pose, (-1, 6)), _f64(self.cam_f), _f64(self.points, (-1, 3)))

    def _view(self):
        self.cam_pose = _f64(self.cam_pose, (-1, 6))
        self.cam_f = _f64(self.cam_f)
        self.points = _f64(self.points, (-1, 3))
        return _capi.ParamView(len(self.cam_f), len(self.points), _dp(self.cam_pose),
                               _dp(self.cam_f), _dp(self.points))


@dataclass
class Problem:
    """problem.hpp:44-56 in SoA form: observations (cam_id, point_id, z) and the
    nominal camera/point record. Validation happens on the device at solver
    construction (Problem::create + build_visibility semantics)."""
    obs_cam: np.ndarray
    obs_pt: np.ndarray
    obs_uv: np.ndarray
    cam_pose: np.ndarray
    cam_f: np.ndarray
    points: np.ndarray

    @classmethod
    def create(cls, cam_pose, cam_f, points, obs_cam, obs_pt, obs_uv):
        return cls(np.ascontiguousarray(obs_cam, np.int32), np.ascontiguousarray(obs_pt, np.int32),
                   _f64(obs_uv, (-1, 2)), _f64(cam_pose, (-1, 6)), _f64(cam_f), _f64(points, (-1, 3)))

    @property
    def num_cameras(self):
        return len(self.cam_f)

    @property
    def num_points(self):
        return len(self.points)

    @property
    def num_observations(self):
        return len(self.obs_cam)

    def nominal_state(self):
        return ParamState(self.cam_pose.copy(), self.cam_f.copy(), self.points.copy())

    def _view(self):
        return _capi.ProblemView(self.num_cameras, self.num_points, self.num_observations,
                                 _ip(self.obs_cam), _ip(self.obs_pt), _dp(self.obs_uv),
                                 _dp(self.cam_pose), _dp(self.cam_f), _dp(self.points))


@dataclass
class InnerOptions:
    """local_opt.hpp:11-19."""
    max_iters: int = 10
    grad_tol: float = 1e-8
    step_tol: float = 1e-10
    lbfgs_memory: int = 8
    armijo_c: float = 1e-4
    backtrack: float = 0.5
    max_line_search: int = 40


SQUARED_L2, HUBER = 0, 1
FAST, EXACT = 0, 1  # dbag_numerics


@dataclass
class LossKind:
    """losses.hpp:13-29."""
    type: int = SQUARED_L2
    delta: float = 1.0

    @staticmethod
    def squared_l2():
        return LossKind(SQUARED_L2, 1.0)

    @staticmethod
    def huber(delta):
        if not delta > 0.0:
            raise ValidationError("Huber delta must be > 0")
        return LossKind(HUBER, delta)

    def is_huber(self):
        return self.type == HUBER


@dataclass
class AdmmOptions:
    """admm_solver.hpp:15-25 (+ ProjectionGuard, BlockConfig, device)."""
    rho_x: float = 1.0
    rho_y: float = 1.0
    max_iters: int = 1600
    primal_tol: float = 1e-6
    stop_on_primal: bool = False
    misfit_loss: LossKind = field(default_factory=LossKind)
    inner: InnerOptions = field(default_factory=InnerOptions)
    eps_depth: float = 1e-6
    workers: int = 1
    points_per_block: int = 1
    cameras_per_block: int = 1
    device: int = 0
    numerics: int = EXACT  # EXACT: bit-identical to the restated reference; FAST: FMA/Woodbury

    def _c(self):
        o = _capi.Options()
        _capi.load().dbag_options_default(C.byref(o))
        o.rho_x, o.rho_y, o.max_iters = self.rho_x, self.rho_y, self.max_iters
        o.primal_tol, o.stop_on_primal = self.primal_tol, int(self.stop_on_primal)
        o.loss, o.huber_delta = self.misfit_loss.type, self.misfit_loss.delta
        i = self.inner
        o.inner_max_iters, o.grad_tol, o.step_tol = i.max_iters, i.grad_tol, i.step_tol
        o.lbfgs_memory, o.armijo_c, o.backtrack = i.lbfgs_memory, i.armijo_c, i.backtrack
        o.max_line_search, o.eps_depth, o.workers = i.max_line_search, self.eps_depth, self.workers
        o.points_per_block, o.cameras_per_block = self.points_per_block, self.cameras_per_block
        o.device = self.device
        o.numerics = self.numerics
        return o


@dataclass
class LocalBlock:
    """admm_solver.hpp:35-45: one local subproblem (ids ascending, local indices
    are positions in point_ids / cam_ids)."""
    point_ids: np.ndarray
    cam_ids: np.ndarray
    obs_ids: np.ndarray
    obs_point_local: np.ndarray
    obs_cam_local: np.ndarray


def _split_blocks(obs_off, obs_ids, pt_off, pt_ids, cam_off, cam_ids, opl, ocl):
    out = []
    for b in range(len(obs_off) - 1):
        o0, o1 = obs_off[b], obs_off[b + 1]
        out.append(LocalBlock(pt_ids[pt_off[b]:pt_off[b + 1]].copy(),
                              cam_ids[cam_off[b]:cam_off[b + 1]].copy(), obs_ids[o0:o1].copy(),
                              opl[o0:o1].copy(), ocl[o0:o1].copy()))
    return out


def _i64p(a):
    return a.ctypes.data_as(_capi.I64P)


def _partition_arrays(problem, points_per_block, cameras_per_block):
    lib = _capi.load()
    h = C.c_void_p()
    nb, pc, cc, comm = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int64()
    pv = problem._view()
    _check(lib.dbag_partition(C.byref(pv), points_per_block, cameras_per_block, C.byref(h),
                              C.byref(nb), C.byref(pc), C.byref(cc), C.byref(comm)))
    try:
        L = problem.num_observations
        obs_off, pt_off, cam_off = (np.zeros(nb.value + 1, np.int64) for _ in range(3))
        obs_ids, opl, ocl = (np.zeros(L, np.int32) for _ in range(3))
        pt_ids, cam_ids = np.zeros(pc.value, np.int32), np.zeros(cc.value, np.int32)
        _check(lib.dbag_partition_fetch(h, _i64p(obs_off), _ip(obs_ids), _i64p(pt_off), _ip(pt_ids),
                                        _i64p(cam_off), _ip(cam_ids), _ip(opl), _ip(ocl)))
    finally:
        lib.dbag_partition_destroy(h)
    return (obs_off, obs_ids, pt_off, pt_ids, cam_off, cam_ids, opl, ocl), comm.value


def align_similarity(state: ParamState, reference: ParamState, device: int = 0) -> ParamState:
    """align_similarity (problem.hpp:87-90, problem.cpp:204-237): the similarity
    gauge that maps state's points onto reference's (Umeyama), applied to
    points and cameras; focal lengths are kept."""
    st, ref = state.copy(), reference.copy()
    m, n = len(st.cam_f), len(st.points)
    pose, pts = np.zeros((m, 6)), np.zeros((n, 3))
    sv, rv = st._view(), ref._view()
    _check(_capi.load().dbag_align_similarity(C.byref(sv), C.byref(rv), device, _dp(pose),
                                              _dp(pts)))
    return ParamState(pose, st.cam_f.copy(), pts)


@dataclass
class LmOptions:
    """LmOptions (lm_solver.hpp:14-23) + device."""
    max_iters: int = 100
    error_stop: float = 1e-14
    lambda_init: float = 1e-3
    lambda_max: float = 1e16
    lambda_up: float = 10.0
    lambda_down: float = 10.0
    use_schur: bool = True
    eps_depth: float = 1e-6
    device: int = 0

    def _c(self):
        o = _capi.LmOptions()
        _capi.load().dbag_lm_options_default(C.byref(o))
        for k in ("max_iters", "error_stop", "lambda_init", "lambda_max", "lambda_up",
                  "lambda_down", "eps_depth", "device"):
            setattr(o, k, getattr(self, k))
        o.use_schur = int(self.use_schur)
        return o


@dataclass
class LmResult:
    """LmResult (lm_solver.hpp:33-38)."""
    state: ParamState
    trace: list
    stop: int  # 0 error stop, 1 lambda max, 2 max iters (LmStopReason)
    accepted_steps: int


class _LmHandle:
    def __init__(self, problem, state, opts):
        self._lib = _capi.load()
        self._h = C.c_void_p()
        st = state.copy()
        pv, iv, o = problem._view(), st._view(), opts._c()
        _check(self._lib.dbag_lm_create(C.byref(pv), C.byref(iv), C.byref(o), C.byref(self._h)))
        self.m, self.n, self.f = problem.num_cameras, problem.num_points, st.cam_f.copy()

    def __del__(self):
        if getattr(self, "_h", None) and self._h.value:
            self._lib.dbag_lm_destroy(self._h)


def solve_lm(problem, init, opts=None, loss=None, reference=None) -> LmResult:
    """solve_lm (lm_solver.hpp:51-54) on the device."""
    opts = opts or LmOptions()
    loss = loss or LossKind()
    h = _LmHandle(problem, init, opts)
    cap = opts.max_iters + 2
    tr = (_capi.IterationRecord * cap)()
    nt, stop, acc = C.c_int64(), C.c_int32(), C.c_int32()
    rv = None
    if reference is not None:
        ref = reference.copy()
        rv = C.byref(ref._view())
    _check(h._lib.dbag_lm_solve(h._h, loss.type, rv, tr, cap, C.byref(nt), C.byref(stop),
                                C.byref(acc)))
    pose, pts = np.zeros((h.m, 6)), np.zeros((h.n, 3))
    _check(h._lib.dbag_lm_get_state(h._h, _dp(pose), _dp(pts)))
    return LmResult(ParamState(pose, h.f, pts), [tr[k].as_dict() for k in range(min(nt.value, cap))],
                    stop.value, acc.value)


def lm_compute_step(problem, state, lam, use_schur=True, eps_depth=1e-6, device=0):
    """lm_compute_step (lm_solver.hpp:47-48): (delta_cameras [6m], delta_points [3n])."""
    h = _LmHandle(problem, state, LmOptions(eps_depth=eps_depth, device=device))
    dc, dp = np.zeros(6 * h.m), np.zeros(3 * h.n)
    _check(h._lib.dbag_lm_compute_step(h._h, lam, int(use_schur), _dp(dc), _dp(dp)))
    return dc, dp


def partition(problem, points_per_block=1, cameras_per_block=1):
    """partition() (admm_solver.hpp:47, admm_solver.cpp:14-72): list of LocalBlock."""
    arrays, _ = _partition_arrays(problem, points_per_block, cameras_per_block)
    return _split_blocks(*arrays)


def communication_cost(problem, points_per_block=1, cameras_per_block=1):
    """communication_cost() (admm_solver.hpp:54, admm_solver.cpp:74-101)."""
    return _partition_arrays(problem, points_per_block, cameras_per_block)[1]


@dataclass
class AdmmState:
    """admm_solver.hpp:57-64, per-copy arrays flattened block by block (in each
    block's id order); for (1,1) blocks one row per block in block order."""
    local_points: np.ndarray
    local_cameras: np.ndarray
    dual_r: np.ndarray
    dual_s: np.ndarray
    consensus: ParamState
    iteration: int


class AdmmSolver:
    """dba::AdmmSolver (admm_solver.hpp:75-138) on one B200, or one camera
    shard of a multi-GPU solve (AdmmSolver.sharded)."""

    def __init__(self, problem: Problem, init: ParamState, opts: AdmmOptions | None = None,
                 rank: int = 0, world: int = 1, sharded: bool = False):
        self._lib = _capi.load()
        self.problem = problem
        self.opts = opts or AdmmOptions()
        self._h = C.c_void_p()
        init = init.as_f64()  # the C-ABI copies it to the device during create
        pv, iv, o = problem._view(), init._view(), self.opts._c()
        self.rank, self.world = rank, world
        if world == 1 and not sharded:
            _check(self._lib.dbag_create(C.byref(pv), C.byref(iv), C.byref(o), C.byref(self._h)))
        else:
            _check(self._lib.dbag_create_sharded(C.byref(pv), C.byref(iv), C.byref(o), rank, world,
                                                 C.byref(self._h)))
        self.m, self.n = problem.num_cameras, problem.num_points
        self.l = problem.num_observations
        self._ref_key = None
        if world > 1 or sharded:
            self.plan = shard_plan(problem, rank, world)
            info = self.plan["info"]
            self.l = info["local_obs"]  # per-copy state arrays are this shard's

    @classmethod
    def sharded(cls, problem, init, opts, rank, world):
        """Shard `rank` of `world` (cameras split on observation counts).
        world == 1 builds the sharded code path with no peers (one-rank NCCL)."""
        return cls(problem, init, opts, rank=rank, world=world, sharded=True)

    def attach_nccl(self, unique_id: bytes):
        buf = (C.c_uint8 * 128).from_buffer_copy(unique_id)
        _check(self._lib.dbag_attach_nccl(self._h, buf))

    def round_phase(self, phase):
        """External-transport round: phases 0, 1, 2 with exchange_copy between."""
        rec = _capi.IterationRecord()
        _check(self._lib.dbag_round_phase(self._h, phase, C.byref(rec) if phase == 2 else None))
        return rec.as_dict() if phase == 2 else None

    def exchange_copy(self, src, which):
        _check(self._lib.dbag_exchange_copy(self._h, src._h, which))

    def close(self):
        if getattr(self, "_h", None) and self._h.value:
            self._lib.dbag_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- phases (admm_solver.cpp:144-357)
    def local_update(self, block_index):
        _check(self._lib.dbag_local_update(self._h, block_index))

    def local_update_all(self):
        _check(self._lib.dbag_local_update_all(self._h))

    def consensus_update(self):
        _check(self._lib.dbag_consensus_update(self._h))

    def dual_update(self):
        _check(self._lib.dbag_dual_update(self._h))

    def _use_reference(self, reference):
        if reference is None:
            return 0
        key = (id(reference.cam_pose), id(reference.points))
        if key != self._ref_key:
            ref = reference.as_f64()
            v = ref._view()
            _check(self._lib.dbag_set_reference(self._h, C.byref(v)))
            self._ref_key = key
        return 1

    def iterate(self, reference: ParamState | None = None):
        rec = _capi.IterationRecord()
        _check(self._lib.dbag_iterate(self._h, self._use_reference(reference), C.byref(rec)))
        return rec.as_dict()

    def run(self, reference: ParamState | None = None):
        cap = max(1, self.opts.max_iters - self.iteration)
        trace = (_capi.IterationRecord * cap)()
        n = C.c_int64()
        _check(self._lib.dbag_run(self._h, self._use_reference(reference), trace, cap,
                                  C.byref(n)))
        return [trace[k].as_dict() for k in range(min(n.value, cap))]

    # ---- state
    @property
    def iteration(self):
        return self._lib.dbag_iteration(self._h)

    def consensus(self, out: ParamState | None = None) -> ParamState:
        """state().consensus; `out` (float64, C-contiguous, e.g. pinned host
        buffers) is filled in place when given."""
        if out is None:
            out = ParamState(np.zeros((self.m, 6)), np.zeros(self.m), np.zeros((self.n, 3)))
        for a in (out.cam_pose, out.cam_f, out.points):
            if a.dtype != np.float64 or not a.flags.c_contiguous:
                raise ValueError("consensus(out=...) needs float64 C-contiguous arrays")
        _check(self._lib.dbag_get_consensus(self._h, _dp(out.cam_pose), _dp(out.cam_f),
                                            _dp(out.points)))
        return out

    def set_consensus(self, state: ParamState):
        pose, pts = _f64(state.cam_pose, (-1, 6)), _f64(state.points, (-1, 3))
        _check(self._lib.dbag_set_consensus(self._h, _dp(pose), _dp(pts)))

    def num_copies(self):
        pc, cc = C.c_int64(), C.c_int64()
        _check(self._lib.dbag_num_copies(self._h, C.byref(pc), C.byref(cc)))
        return pc.value, cc.value

    def state(self) -> AdmmState:
        pc, cc = self.num_copies()
        lp, lc = np.zeros((pc, 3)), np.zeros((cc, 6))
        r, s = np.zeros((pc, 3)), np.zeros((cc, 6))
        _check(self._lib.dbag_get_copies(self._h, _dp(lp), _dp(lc), _dp(r), _dp(s)))
        return AdmmState(lp, lc, r, s, self.consensus(), self.iteration)

    def set_copies(self, local_points, local_cameras, dual_r, dual_s):
        a, b = _f64(local_points, (-1, 3)), _f64(local_cameras, (-1, 6))
        c, d = _f64(dual_r, (-1, 3)), _f64(dual_s, (-1, 6))
        _check(self._lib.dbag_set_copies(self._h, _dp(a), _dp(b), _dp(c), _dp(d)))

    def blocks(self):
        """Observation ids of all blocks concatenated in block order (for (1,1)
        blocks: blocks()[b].obs_ids[0])."""
        out = np.zeros(self.l, np.int32)
        _check(self._lib.dbag_get_block_order(self._h, _ip(out)))
        return out

    def block_list(self):
        """blocks() (admm_solver.hpp:108) as LocalBlock objects."""
        nb = self._lib.dbag_num_blocks(self._h)
        pc, cc = self.num_copies()
        obs_off, pt_off, cam_off = (np.zeros(nb + 1, np.int64) for _ in range(3))
        pt_ids, cam_ids = np.zeros(pc, np.int32), np.zeros(cc, np.int32)
        opl, ocl = np.zeros(self.l, np.int32), np.zeros(self.l, np.int32)
        _check(self._lib.dbag_get_blocks(self._h, _i64p(obs_off), _i64p(pt_off), _ip(pt_ids),
                                         _i64p(cam_off), _ip(cam_ids), _ip(opl), _ip(ocl)))
        return _split_blocks(obs_off, self.blocks(), pt_off, pt_ids, cam_off, cam_ids, opl, ocl)

    # ---- queries (admm_solver.hpp:110-127)
    def max_primal_residual_points(self):
        return self._max_primal()[0]

    def max_primal_residual_cameras(self):
        return self._max_primal()[1]

    def _max_primal(self):
        x, y = C.c_double(), C.c_double()
        _check(self._lib.dbag_max_primal(self._h, C.byref(x), C.byref(y)))
        return x.value, y.value

    def dual_sums(self):
        p, c = np.zeros((self.n, 3)), np.zeros((self.m, 6))
        _check(self._lib.dbag_dual_sums(self._h, _dp(p), _dp(c)))
        return p, c

    def dual_sum_point(self, i):
        return self.dual_sums()[0][i]

    def dual_sum_camera(self, j):
        return self.dual_sums()[1][j]

    def block_objective(self, b):
        out = C.c_double()
        _check(self._lib.dbag_block_objective(self._h, b, C.byref(out)))
        return out.value

    def ops_per_iteration(self):
        return self._lib.dbag_ops_per_iteration(self._h)

    def comm_floats_per_iteration(self):
        return self._lib.dbag_comm_floats(self._h)

    def mean_reprojection_error(self):
        out = C.c_double()
        _check(self._lib.dbag_mean_reprojection_error(self._h, C.byref(out)))
        return out.value

    def rms_reprojection_error(self):
        out = C.c_double()
        _check(self._lib.dbag_rms_reprojection_error(self._h, C.byref(out)))
        return out.value

    def total_squared_error(self):
        out = C.c_double()
        _check(self._lib.dbag_total_squared_error(self._h, C.byref(out)))
        return out.value

    # ---- measurement hooks
    def enqueue_round(self):
        _check(self._lib.dbag_enqueue_round(self._h))

    def reset(self):
        """Restart from the init state (copies = init consensus, duals = 0)."""
        _check(self._lib.dbag_reset(self._h))

    def set_profiling(self, on=True):
        _check(self._lib.dbag_set_profiling(self._h, int(on)))

    def stream_handle(self):
        return self._lib.dbag_stream(self._h)

    def synchronize(self):
        _check(self._lib.dbag_synchronize(self._h))

    def round_stats(self):
        s = _capi.RoundStats()
        _check(self._lib.dbag_get_round_stats(self._h, C.byref(s)))
        return s.as_dict()

    def reset_stats(self):
        _check(self._lib.dbag_reset_stats(self._h))


# ---- problem files and metrics CSV (bal_io.hpp:21-31, metrics_csv.hpp:11-19) -----


def _io_check(rc):
    if rc == 0:
        return
    line = C.c_int32()
    msg = _capi.load().dbag_io_last_error(C.byref(line)).decode()
    if rc == 11:
        raise ParseError(msg, line.value)
    raise _STATUS.get(rc, Error)(msg)


def parse_problem_text(text: str):
    """bal_io.cpp:100-185 -> (Problem, init ParamState)."""
    lib = _capi.load()
    raw = text.encode()
    h = C.c_void_p()
    m, n, l = C.c_int32(), C.c_int32(), C.c_int64()
    _io_check(lib.dbag_parse_problem_text(raw, len(raw), C.byref(h), C.byref(m), C.byref(n),
                                          C.byref(l)))
    try:
        cam, pt = np.zeros(l.value, np.int32), np.zeros(l.value, np.int32)
        uv, pose = np.zeros((l.value, 2)), np.zeros((m.value, 6))
        f, pts = np.zeros(m.value), np.zeros((n.value, 3))
        lib.dbag_bal_fetch(h, _ip(cam), _ip(pt), _dp(uv), _dp(pose), _dp(f), _dp(pts))
    finally:
        lib.dbag_bal_destroy(h)
    return Problem(cam, pt, uv, pose, f, pts), ParamState(pose.copy(), f.copy(), pts.copy())


def serialize_problem_text(problem: Problem, state: ParamState) -> str:
    """bal_io.cpp:197-231 (17 significant digits: bit-exact round trip)."""
    lib = _capi.load()
    st = state.copy()
    pv, sv = problem._view(), st._view()
    n = C.c_size_t()
    _io_check(lib.dbag_serialize_problem_text(C.byref(pv), C.byref(sv), None, 0, C.byref(n)))
    buf = C.create_string_buffer(n.value + 1)
    _io_check(lib.dbag_serialize_problem_text(C.byref(pv), C.byref(sv), buf, n.value + 1,
                                              C.byref(n)))
    return buf.value.decode()


def metrics_csv(trace) -> str:
    """metrics_csv.cpp:16-38 for a list of iterate()/run() records."""
    recs = (_capi.IterationRecord * max(1, len(trace)))()
    for k, r in enumerate(trace):
        for name, _ in _capi.IterationRecord._fields_:
            if name in r:
                setattr(recs[k], name, r[name])
    n = C.c_size_t()
    lib = _capi.load()
    _io_check(lib.dbag_metrics_csv(recs, len(trace), None, 0, C.byref(n)))
    buf = C.create_string_buffer(n.value + 1)
    _io_check(lib.dbag_metrics_csv(recs, len(trace), buf, n.value + 1, C.byref(n)))
    return buf.value.decode()


def nccl_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    _check(_capi.load().dbag_nccl_unique_id(buf))
    return bytes(buf)


def shard_plan(problem: Problem, rank: int, world: int) -> dict:
    """Host-only shard plan (dbag_shard_plan_*): no GPU needed."""
    lib = _capi.load()
    pv = problem._view()
    h = C.c_void_p()
    info = _capi.ShardInfo()
    _check(lib.dbag_shard_plan_create(C.byref(pv), rank, world, C.byref(h), C.byref(info)))
    try:
        d = info.as_dict()
        out = {"info": d,
               "cam_lo": np.zeros(world + 1, np.int32),
               "local_obs": np.zeros(d["local_obs"], np.int64),
               "local_points": np.zeros(d["local_points"], np.int32),
               "bp_of_local": np.zeros(d["local_points"], np.int32),
               "owner_of_local": np.zeros(d["local_points"], np.int8),
               "gb_off": np.zeros(d["boundary_points"] + 1, np.int64),
               "gmap": np.zeros(d["boundary_copies"], np.int64),
               "send_obs_local": np.zeros(d["send_count"], np.int64),
               "send_off": np.zeros(world + 1, np.int64),
               "recv_off": np.zeros(world + 1, np.int64)}
        p = lambda a, t: a.ctypes.data_as(C.POINTER(t))  # noqa: E731
        _check(lib.dbag_shard_plan_arrays(
            h, p(out["cam_lo"], C.c_int32), p(out["local_obs"], C.c_int64),
            p(out["local_points"], C.c_int32), p(out["bp_of_local"], C.c_int32),
            p(out["owner_of_local"], C.c_int8), p(out["gb_off"], C.c_int64),
            p(out["gmap"], C.c_int64), p(out["send_obs_local"], C.c_int64)))
        _check(lib.dbag_shard_plan_exchange(h, p(out["send_off"], C.c_int64),
                                            p(out["recv_off"], C.c_int64)))
    finally:
        lib.dbag_shard_plan_destroy(h)
    return out


def partition_cameras(obs_per_camera, world):
    c = np.ascontiguousarray(obs_per_camera, np.int64)
    lo = np.zeros(world + 1, np.int32)
    _check(_capi.load().dbag_partition_cameras(len(c), c.ctypes.data_as(_capi.I64P), world,
                                               lo.ctypes.data_as(_capi.I32P)))
    return lo


def measure_fp64_peak(device=0):
    """FP64 FMA throughput (TFLOP/s) of the device: the local-solve roofline."""
    out = C.c_double()
    _check(_capi.load().dbag_measure_fp64_peak(device, C.byref(out)))
    return out.value


def selftest_division(n, seed=1, device=0):
    """Test hook: mismatches of the EXACT kernels' branch-free RN(1/d) against
    IEEE 1.0/d over n operands of the guarded exponent band."""
    out = C.c_int64()
    _check(_capi.load().dbag_selftest_division(device, n, seed, C.byref(out)))
    return out.value


def run_admm(problem, init, opts=None, reference=None):
    """admm_solver.cpp:476-480 -> (final consensus, trace)."""
    solver = AdmmSolver(problem, init, opts)
    trace = solver.run(reference)
    out = solver.consensus()
    solver.close()
    return out, trace


# ---- synthetic config scenes (dbag_scene_*) -----------------------------------


@dataclass
class Scene:
    problem: Problem
    ground_truth: ParamState
    init: ParamState
    info: dict


def generate_config_scene(config: int, seed: int = 0, scale: float = 1.0) -> Scene:
    """BASELINE.json config 1..5; deterministic in seed."""
    lib = _capi.load()
    h = C.c_void_p()
    info = _capi.SceneInfo()
    _check(lib.dbag_scene_generate(config, seed, scale, C.byref(h), C.byref(info)))
    try:
        m, n, l = info.num_cameras, info.num_points, info.num_obs
        cam, pt = np.zeros(l, np.int32), np.zeros(l, np.int32)
        uv, gt_pose, f = np.zeros((l, 2)), np.zeros((m, 6)), np.zeros(m)
        gt_pts, ip, ix = np.zeros((n, 3)), np.zeros((m, 6)), np.zeros((n, 3))
        _check(lib.dbag_scene_fetch(h, _ip(cam), _ip(pt), _dp(uv), _dp(gt_pose), _dp(f),
                                    _dp(gt_pts), _dp(ip), _dp(ix)))
    finally:
        lib.dbag_scene_destroy(h)
    prob = Problem(cam, pt, uv, gt_pose, f, gt_pts)
    d = {k: getattr(info, k) for k, _ in info._fields_}
    return Scene(prob, ParamState(gt_pose.copy(), f.copy(), gt_pts.copy()),
                 ParamState(ip, f.copy(), ix), d)
