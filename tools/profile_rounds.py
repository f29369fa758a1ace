"""Minimal driver for ncu: build one config scene, run a few ADMM rounds.

  python tools/profile_rounds.py --config 2 --numerics exact --rounds 3 [--loss l2]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("--numerics", choices=["exact", "fast"], default="exact")
    ap.add_argument("--loss", choices=["l2", "huber"], default="l2")
    ap.add_argument("--rounds", type=int, default=3)
    ap.add_argument("--points-per-block", type=int, default=1)
    ap.add_argument("--cameras-per-block", type=int, default=1)
    a = ap.parse_args()
    import paper_1708_07954_b200 as P
    s = P.generate_config_scene(a.config, 0, a.scale)
    opts = P.AdmmOptions(max_iters=a.rounds,
                         misfit_loss=P.LossKind.huber(1.0) if a.loss == "huber" else P.LossKind(),
                         numerics=P.admm.EXACT if a.numerics == "exact" else P.admm.FAST,
                         points_per_block=a.points_per_block, cameras_per_block=a.cameras_per_block)
    solver = P.AdmmSolver(s.problem, s.init, opts)
    tr = solver.run()
    print(a, "rounds", len(tr), "last", {k: tr[-1][k] for k in ("mean_reproj_err", "wall_ms")})


if __name__ == "__main__":
    main()
