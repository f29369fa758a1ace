import time, numpy as np, torch, sys
sys.path.insert(0, '/root/repo')
import paper_1708_07954_b200 as P
sc = P.generate_config_scene(5, 0)
p = sc.problem
def pinned(a):
    return torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()
hp = P.Problem(pinned(p.obs_cam), pinned(p.obs_pt), pinned(p.obs_uv), pinned(p.cam_pose), pinned(p.cam_f), pinned(p.points))
hi = P.ParamState(pinned(sc.init.cam_pose), pinned(sc.init.cam_f), pinned(sc.init.points))
o = P.AdmmOptions(max_iters=1)
w = P.AdmmSolver(hp, hi, o); w.run(); w.close(); torch.cuda.synchronize()
for k in range(3):
    t0 = time.perf_counter(); s = P.AdmmSolver(hp, hi, o); t1 = time.perf_counter()
    s.run(); t2 = time.perf_counter(); s.consensus(); t3 = time.perf_counter(); s.close()
    print("create %.3f s, 1 round %.3f s, consensus %.3f s" % (t1 - t0, t2 - t1, t3 - t2))
