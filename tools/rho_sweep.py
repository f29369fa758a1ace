"""Sweep the ADMM penalty rho on a config scene and report which settings keep
the consensus feasible (finite mean reprojection error) over R rounds, with
the per-round device time. Usage: python tools/rho_sweep.py [config] [rounds]."""
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1708_07954_b200 as P  # noqa: E402


def main():
    config = int(sys.argv[1]) if len(sys.argv) > 1 else 5
    rounds = int(sys.argv[2]) if len(sys.argv) > 2 else 50
    scene = P.generate_config_scene(config, 0)
    for loss in ("l2", "huber"):
        for rho in (1.0, 10.0, 100.0, 1e3, 1e4):
            lk = P.LossKind.huber(1.0) if loss == "huber" else P.LossKind.squared_l2()
            s = P.AdmmSolver(scene.problem, scene.init,
                             P.AdmmOptions(misfit_loss=lk, rho_x=rho, rho_y=rho, max_iters=rounds))
            t0 = time.time()
            tr = s.run(scene.ground_truth)
            wall = time.time() - t0
            errs = [r["mean_reproj_err"] for r in tr]
            first_inf = next((r["iter"] for r in tr if not math.isfinite(r["mean_reproj_err"])), None)
            ms = [r["wall_ms"] for r in tr]
            print(json.dumps({
                "config": config, "loss": loss, "rho": rho, "rounds": rounds,
                "first_infinite_round": first_inf,
                "mean_reproj_err": {"r1": errs[0], "r10": errs[min(9, rounds - 1)],
                                    "r20": errs[min(19, rounds - 1)], "last": errs[-1]},
                "point_mse_last": tr[-1]["point_mse"], "camera_mse_last": tr[-1]["camera_mse"],
                "max_primal_x_last": tr[-1]["max_primal_x"],
                "ms_per_round_first20": sum(ms[:20]) / min(20, len(ms)),
                "ms_per_round_all": sum(ms) / len(ms), "wall_s": wall}), flush=True)
            s.close()


if __name__ == "__main__":
    main()
