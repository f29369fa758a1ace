"""Times the centralized LM comparator on a BASELINE
config scene: device ms per LM iteration (the reference's wall_ms scope,
lm_solver.cpp:183-213, from CUDA events) against the oracle restatement on the
host (single thread, as lm_solver.cpp runs). One JSON line.

  python tools/bench_lm.py --config 2 --iters 5 [--scale 1.0] [--no-cpu]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("--iters", type=int, default=5)
    ap.add_argument("--no-cpu", action="store_true")
    a = ap.parse_args()
    import paper_1708_07954_b200 as P
    sc = P.generate_config_scene(a.config, 0, a.scale)
    p = sc.problem
    P.solve_lm(p, sc.init, P.LmOptions(max_iters=1))  # warm-up (context, cuSOLVER)
    t0 = time.perf_counter()
    r = P.solve_lm(p, sc.init, P.LmOptions(max_iters=a.iters))
    wall = time.perf_counter() - t0
    dev_ms = [t["wall_ms"] for t in r.trace[1:]]
    line = {"what": "centralized LM (Schur + cuSOLVER)", "config": a.config, "scale": a.scale,
            "cameras": p.num_cameras, "points": p.num_points, "observations": p.num_observations,
            "iterations": len(dev_ms), "accepted_steps": r.accepted_steps,
            "gpu_ms_per_iteration": sum(dev_ms) / max(1, len(dev_ms)),
            "e2e_s": wall, "final_mean_reproj_err": r.trace[-1]["mean_reproj_err"]}
    if not a.no_cpu:
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        import oracle as O
        op = O.Problem.create(p.cam_pose, p.cam_f, p.points, p.obs_cam, p.obs_pt, p.obs_uv)
        _, _, otr, _, oacc = O.solve_lm(op, sc.init.cam_pose, p.cam_f, sc.init.points,
                                        max_iters=a.iters)
        cpu = [t["wall_ms"] for t in otr[1:]]
        line["cpu_ms_per_iteration"] = sum(cpu) / max(1, len(cpu))
        line["cpu_kind"] = "port (oracle/, 1 thread, as lm_solver.cpp)"
        line["gpu_over_cpu"] = line["cpu_ms_per_iteration"] / line["gpu_ms_per_iteration"]
        line["same_accepted_steps"] = oacc == r.accepted_steps
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
