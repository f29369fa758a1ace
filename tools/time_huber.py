"""Per-round device time of the EXACT Huber K1 at a config scene (pooled
kernel, or the one-thread-per-observation kernel with DBAG_HUBER_LEGACY=1).
Usage: python tools/time_huber.py [config] [rounds] [rho]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1708_07954_b200 as P  # noqa: E402

config = int(sys.argv[1]) if len(sys.argv) > 1 else 5
rounds = int(sys.argv[2]) if len(sys.argv) > 2 else 10
rho = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
s = P.generate_config_scene(config, 0)
o = P.AdmmOptions(misfit_loss=P.LossKind.huber(1.0), rho_x=rho, rho_y=rho, max_iters=10 ** 9)
g = P.AdmmSolver(s.problem, s.init, o)
g.enqueue_round()
g.synchronize()
g.reset()
g.reset_stats()
g.set_profiling(True)
for _ in range(rounds):
    g.enqueue_round()
g.synchronize()
st = g.round_stats()
c = g.consensus()
print(json.dumps({"config": config, "rounds": rounds, "rho": rho,
                  "legacy": bool(os.environ.get("DBAG_HUBER_LEGACY")),
                  "ms_local_per_round": st["ms_local"] / rounds,
                  "ms_round": (st["ms_local"] + st["ms_camera"] + st["ms_point"] + st["ms_final"]) / rounds,
                  "counters": {k: st[k] for k in ("n_jacobian", "n_trial", "n_accept", "n_direction",
                                                  "n_pairs_used")},
                  "checksum": [float(c.points.sum()), float(c.cam_pose.sum())]}))
