"""Wall time of dbag_create (H2D from pinned buffers + device index build), one
round and the consensus D2H into pinned buffers, at config 5. With
DBAG_CREATE_TIMING=1 the library also prints create's stages."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1708_07954_b200 as P  # noqa: E402

sc = P.generate_config_scene(5, 0)
p = sc.problem


def pinned(a):
    return torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()


hp = P.Problem(pinned(p.obs_cam), pinned(p.obs_pt), pinned(p.obs_uv), pinned(p.cam_pose),
               pinned(p.cam_f), pinned(p.points))
hi = P.ParamState(pinned(sc.init.cam_pose), pinned(sc.init.cam_f), pinned(sc.init.points))
out = P.ParamState(pinned(np.zeros((p.num_cameras, 6))), pinned(np.zeros(p.num_cameras)),
                   pinned(np.zeros((p.num_points, 3))))
o = P.AdmmOptions(max_iters=1)
w = P.AdmmSolver(hp, hi, o)
w.run()
w.close()
torch.cuda.synchronize()
for k in range(3):
    t0 = time.perf_counter()
    s = P.AdmmSolver(hp, hi, o)
    t1 = time.perf_counter()
    s.run()
    t2 = time.perf_counter()
    s.consensus(out=out)
    t3 = time.perf_counter()
    s.close()
    print("create %.3f s, 1 round %.3f s, consensus (pinned) %.3f s" % (t1 - t0, t2 - t1, t3 - t2))
