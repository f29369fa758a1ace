"""Multi-GPU host logic on CPU: the camera partitioner, the
boundary-point plan, and — with two gloo ranks — the boundary exchange layout
reproducing the reference's consensus bit for bit (admm_solver.cpp:324-332)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def scene(P, config=5, scale=0.002, seed=1):
    return P.generate_config_scene(config, seed, scale)


def test_partition_contiguous_balanced():
    from paper_1708_07954_b200 import admm
    rng = np.random.default_rng(0)
    for world in (1, 2, 3, 4, 8):
        counts = rng.integers(1, 50, size=100)
        lo = admm.partition_cameras(counts, world)
        assert lo[0] == 0 and lo[-1] == 100 and np.all(np.diff(lo) >= 1)
        per = [counts[lo[r]:lo[r + 1]].sum() for r in range(world)]
        # each cut is within one camera's weight of the ideal prefix
        assert max(per) - counts.sum() / world <= counts.max() + 1e-9
    with pytest.raises(Exception):
        admm.partition_cameras(np.ones(3, np.int64), 4)  # fewer cameras than ranks


@pytest.mark.parametrize("world", [2, 3, 8])
def test_shard_plan_properties(world):
    import paper_1708_07954_b200 as P
    from paper_1708_07954_b200 import admm
    s = scene(P)
    p = s.problem
    plans = [admm.shard_plan(p, r, world) for r in range(world)]
    lo = plans[0]["cam_lo"]
    rank_of_cam = np.searchsorted(lo, np.arange(p.num_cameras), side="right") - 1
    # every observation on exactly one rank: the rank of its camera
    seen = np.concatenate([pl["local_obs"] for pl in plans])
    assert np.array_equal(np.sort(seen), np.arange(p.num_observations))
    for r, pl in enumerate(plans):
        assert np.all(rank_of_cam[p.obs_cam[pl["local_obs"]]] == r)
        assert np.array_equal(pl["cam_lo"], lo)
    # boundary points: exactly those whose cameras span ranks
    rmin = np.full(p.num_points, world)
    rmax = np.full(p.num_points, -1)
    np.minimum.at(rmin, p.obs_pt, rank_of_cam[p.obs_cam])
    np.maximum.at(rmax, p.obs_pt, rank_of_cam[p.obs_cam])
    boundary = np.nonzero(rmin != rmax)[0]
    info = plans[0]["info"]
    assert info["boundary_points"] == len(boundary)
    d = np.bincount(p.obs_pt[np.isin(p.obs_pt, boundary)], minlength=p.num_points)[boundary]
    assert info["boundary_copies"] == d.sum()
    assert np.array_equal(np.diff(plans[0]["gb_off"]), d)
    # per-peer exchange: a copy of a boundary point travels from its owner to
    # every OTHER rank holding the point, in global copy order
    g_obs = np.lexsort((p.obs_cam, p.obs_pt))
    g_obs = g_obs[np.isin(p.obs_pt[g_obs], boundary)]
    g_owner = rank_of_cam[p.obs_cam[g_obs]]
    g_pt = p.obs_pt[g_obs]
    holds = np.zeros((world, p.num_points), bool)
    holds[rank_of_cam[p.obs_cam], p.obs_pt] = True
    for r, pl in enumerate(plans):
        gm, so, ro = pl["gmap"], pl["send_off"], pl["recv_off"]
        local_of_obs = np.full(p.num_observations, -1)
        local_of_obs[pl["local_obs"]] = np.arange(len(pl["local_obs"]))
        mine = g_owner == r
        held = holds[r, g_pt]
        assert np.all(gm[mine] == -2 - local_of_obs[g_obs[mine]])
        assert np.all(gm[~held] == -1)
        peer = held & ~mine
        # recv slots: from source s, s's copies of the points r holds, in order
        for src in range(world):
            sel = peer & (g_owner == src)
            assert np.array_equal(gm[sel], np.arange(ro[src], ro[src + 1]))
        assert ro[r + 1] == ro[r] and pl["info"]["recv_count"] == ro[-1]
        # send slots to dest d: the same copies d expects from r
        for dst in range(world):
            sel = mine & holds[dst, g_pt] & (dst != r)
            assert np.array_equal(pl["send_obs_local"][so[dst]:so[dst + 1]],
                                  local_of_obs[g_obs[sel]])
            assert so[dst + 1] - so[dst] == (plans[dst]["recv_off"][r + 1] -
                                             plans[dst]["recv_off"][r])
    for r, pl in enumerate(plans):
        assert np.array_equal(pl["gb_off"], plans[0]["gb_off"])
        bpl = pl["bp_of_local"]
        glob = pl["local_points"]
        assert np.all((bpl >= 0) == np.isin(glob, boundary))
        assert np.all(pl["owner_of_local"] == (rmin[glob] == r))
    # the reference's communication_cost: sum_i 3 d_i (d_i - 1)
    dd = np.bincount(p.obs_pt, minlength=p.num_points)
    assert info["comm_floats"] == int((3 * dd * (dd - 1)).sum())


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _rank_main(rank, world, port, q):
    """One gloo rank: pack this rank's boundary copies (from the oracle's
    post-local-update state) per peer, exchange them with one send/recv pair
    per peer, recompute each boundary point's consensus from its copies (own
    and received) in the plan's global order."""
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path[:0] = [root, os.path.join(root, "oracle")]
    import torch
    import oracle as O
    import paper_1708_07954_b200 as P
    from paper_1708_07954_b200 import admm
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    s = scene(P)
    p = s.problem
    op = O.Problem.create(p.cam_pose, p.cam_f, p.points, p.obs_cam, p.obs_pt, p.obs_uv)
    sol = O.AdmmSolver(op, s.init.cam_pose, p.cam_f, s.init.points, workers=2, rho_x=1.3)
    sol.iterate()
    sol.local_update_all()  # copies and duals as the next consensus sees them
    lp, _, r, _ = sol.copies()
    obs_of_block = sol.block_obs_ids()["obs_ids"]
    blk_of_obs = np.empty_like(obs_of_block)
    blk_of_obs[obs_of_block] = np.arange(len(obs_of_block))
    plan = admm.shard_plan(p, rank, world)
    info = plan["info"]
    so, ro = plan["send_off"], plan["recv_off"]
    send = np.zeros((info["send_count"], 6))
    for slot, qi in enumerate(plan["send_obs_local"]):
        b = blk_of_obs[plan["local_obs"][qi]]
        send[slot, :3], send[slot, 3:] = lp[b], r[b]
    recv = np.zeros((info["recv_count"], 6))
    reqs = []  # one send/recv pair per peer, as the NCCL group does
    for q_ in range(world):
        if q_ == rank:
            continue
        if so[q_ + 1] > so[q_]:
            reqs.append(dist.isend(torch.from_numpy(send[so[q_]:so[q_ + 1]].copy()), q_))
        if ro[q_ + 1] > ro[q_]:
            buf = torch.zeros((ro[q_ + 1] - ro[q_], 6), dtype=torch.float64)
            reqs.append((dist.irecv(buf, q_), q_, buf))
    for rq in reqs:
        if isinstance(rq, tuple):
            rq[0].wait()
            recv[ro[rq[1]]:ro[rq[1] + 1]] = rq[2].numpy()
        else:
            rq.wait()

    def copy_of(slot):
        if slot >= 0:
            return recv[slot]
        b = blk_of_obs[plan["local_obs"][-2 - slot]]
        return np.concatenate([lp[b], r[b]])
    inv_rho = 1.0 / 1.3
    out = {}
    for i_loc, bp in enumerate(plan["bp_of_local"]):
        if bp < 0:
            continue
        g0, g1 = plan["gb_off"][bp], plan["gb_off"][bp + 1]
        anc = copy_of(plan["gmap"][g0])[:3].copy()
        acc = [0.0, 0.0, 0.0]
        for g in range(g0, g1):
            c = copy_of(plan["gmap"][g])
            for k in range(3):
                acc[k] += (c[k] - anc[k]) + inv_rho * c[3 + k]
        out[int(plan["local_points"][i_loc])] = [anc[k] + acc[k] / float(g1 - g0) for k in range(3)]
    sol.consensus_update()
    _, _, ref_pts = sol.consensus()
    bad = [i for i, v in out.items() if list(ref_pts[i]) != v]
    q.put((rank, len(out), bad[:5]))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_boundary_consensus_bit_exact(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=300) for _ in procs]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    for rank, n, bad in res:
        assert n > 0, "no boundary points on rank %d" % rank
        assert bad == [], (rank, bad)
