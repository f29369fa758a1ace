"""Regenerates tests/golden/oracle_trajectories.json.

The reference cannot be compiled in this container (it needs Eigen3, absent;
see DESIGN.md §Oracle) and ships no golden trajectory, so these fixtures are
produced by the oracle after it passed every restated reference KAT/invariant
in tests/test_oracle_*.py. They guard the oracle against silent drift and give
the GPU parity tests small, fixed expected trajectories.
Run: python tests/golden/make_golden.py
"""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", "..", "oracle"))
import oracle as O  # noqa: E402

CASES = [dict(seed=93, sigma_cam=0.01, sigma_point=0.01, rounds=20, loss=0),
         dict(seed=100, sigma_cam=0.05, sigma_point=0.2, rounds=20, loss=0),
         dict(seed=85, sigma_cam=0.05, sigma_point=0.3, rounds=10, loss=1)]


def main():
    out = {"generator": "oracle/liboracle.so via tests/golden/make_golden.py", "cases": []}
    for c in CASES:
        s = O.generate_scene(O.standard_scene_config(c["seed"]))
        pose, pts = O.perturb(s.cam_pose, s.cam_f, s.points, c["sigma_cam"], c["sigma_point"],
                              c["seed"] + 1)
        solver = O.AdmmSolver(s, pose, s.cam_f, pts, max_iters=c["rounds"], loss=c["loss"])
        trace = solver.run(s.cam_pose, s.points)
        fpose, _, fpts = solver.consensus()
        case = dict(c)
        case["trace"] = [{k: t[k] for k in ("iter", "mean_reproj_err", "max_primal_x",
                                             "max_primal_y", "camera_mse", "point_mse",
                                             "comm_floats")} for t in trace]
        case["final_pose"] = fpose.tolist()
        case["final_pts"] = fpts.tolist()
        out["cases"].append(case)
    with open(os.path.join(HERE, "oracle_trajectories.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
