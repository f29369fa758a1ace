// dbag_shard.cpp — host-side shard plan for the multi-GPU path.
//
// Observations are partitioned by CAMERA: rank r owns the contiguous camera
// range [cam_lo[r], cam_lo[r+1]) chosen on observation prefix sums, so camera
// consensus and dual s never leave a rank. A point whose cameras span ranks is
// a BOUNDARY point. Its copies ("boundary copies", global order = the
// reference's copy order: by point, then camera — admm_solver.cpp:126-140) are
// exchanged raw (x and r, 48 B each) once per round, each copy only to the
// other ranks that hold its point (one ncclSend/ncclRecv per peer, grouped), so
// every holder recomputes the reference's sequential consensus sum
// (admm_solver.cpp:324-332) bit for bit. Integer and deterministic: every rank
// derives the same plan from the same full problem, so a sender's slot order
// for a peer (global copy order) is the receiver's.
#include "dbag_shard.h"

#include <algorithm>
#include <numeric>
#include <stdexcept>
#include <string>

namespace dbag {

std::vector<int32_t> partition_cameras(int32_t m, const std::vector<int64_t>& obs_per_camera,
                                       int32_t world) {
  // cut before camera j when the prefix count reaches k*L/world (k-th cut);
  // every rank gets >= 1 camera when m >= world.
  std::vector<int32_t> lo(world + 1, m);
  lo[0] = 0;
  int64_t total = 0;
  for (int64_t c : obs_per_camera) total += c;
  int64_t acc = 0;
  int32_t r = 1;
  for (int32_t j = 0; j < m && r < world; ++j) {
    // remaining ranks need at least one camera each
    const int32_t must = m - (world - r);
    if (j > lo[r - 1] && (acc * world >= total * r || j >= must)) {
      lo[r] = j;
      ++r;
    }
    acc += obs_per_camera[j];
  }
  for (; r < world; ++r) lo[r] = std::max(lo[r - 1] + 1, std::min(m, lo[r]));
  lo[world] = m;
  return lo;
}

ShardPlan make_shard_plan(int32_t m, int32_t n, int64_t l, const int32_t* cam, const int32_t* pt,
                          int32_t rank, int32_t world) {
  if (world < 1 || rank < 0 || rank >= world) throw std::invalid_argument("bad rank/world");
  if (m < world) throw std::invalid_argument("fewer cameras than ranks");
  ShardPlan P;
  P.rank = rank;
  P.world = world;
  std::vector<int64_t> per_cam(m, 0);
  for (int64_t k = 0; k < l; ++k) {
    if (cam[k] < 0 || cam[k] >= m || pt[k] < 0 || pt[k] >= n)
      throw std::out_of_range("observation index out of range");
    ++per_cam[cam[k]];
  }
  P.cam_lo = partition_cameras(m, per_cam, world);
  std::vector<int32_t> rank_of_cam(m);
  for (int32_t r = 0; r < world; ++r)
    for (int32_t j = P.cam_lo[r]; j < P.cam_lo[r + 1]; ++j) rank_of_cam[j] = r;
  // observations sorted by (point, camera): the reference copy order
  std::vector<int64_t> order(l);
  std::iota(order.begin(), order.end(), 0);
  std::sort(order.begin(), order.end(), [&](int64_t a, int64_t b) {
    return pt[a] != pt[b] ? pt[a] < pt[b] : cam[a] < cam[b];
  });
  // per point: rank span
  std::vector<int32_t> rmin(n, world), rmax(n, -1);
  for (int64_t k = 0; k < l; ++k) {
    const int32_t r = rank_of_cam[cam[k]];
    rmin[pt[k]] = std::min(rmin[pt[k]], r);
    rmax[pt[k]] = std::max(rmax[pt[k]], r);
  }
  // global boundary points (ascending id) and boundary copies (point, camera)
  std::vector<int32_t> bp_of_point(n, -1);
  for (int32_t i = 0; i < n; ++i)
    if (rmax[i] >= 0 && rmin[i] != rmax[i]) {
      bp_of_point[i] = P.n_boundary_points++;
    }
  P.gb_off.assign(P.n_boundary_points + 1, 0);
  std::vector<int32_t> g_owner;    // per global boundary copy: owning rank
  std::vector<int64_t> g_obs;      // input observation index
  for (int64_t q = 0; q < l; ++q) {
    const int64_t k = order[q];
    const int32_t bp = bp_of_point[pt[k]];
    if (bp < 0) continue;
    ++P.gb_off[bp + 1];
    g_owner.push_back(rank_of_cam[cam[k]]);
    g_obs.push_back(k);
  }
  for (int32_t b = 0; b < P.n_boundary_points; ++b) P.gb_off[b + 1] += P.gb_off[b];
  P.n_boundary_copies = (int64_t)g_owner.size();
  // holders of each boundary point: a bit set over ranks (world <= 64)
  if (world > 64) throw std::invalid_argument("at most 64 ranks");
  std::vector<uint64_t> holders(P.n_boundary_points, 0);
  for (int32_t b = 0; b < P.n_boundary_points; ++b)
    for (int64_t g = P.gb_off[b]; g < P.gb_off[b + 1]; ++g) holders[b] |= 1ull << g_owner[g];
  // this rank's observations (input order) and local renumbering
  P.cam_begin = P.cam_lo[rank];
  P.cam_end = P.cam_lo[rank + 1];
  std::vector<int32_t> local_of_point(n, -1);
  for (int64_t k = 0; k < l; ++k)
    if (rank_of_cam[cam[k]] == rank) {
      P.local_obs.push_back(k);
      local_of_point[pt[k]] = 0;
    }
  for (int32_t i = 0; i < n; ++i)
    if (local_of_point[i] == 0) {
      local_of_point[i] = (int32_t)P.local_points.size();
      P.local_points.push_back(i);
    }
  P.local_cam.resize(P.local_obs.size());
  P.local_pt.resize(P.local_obs.size());
  for (size_t q = 0; q < P.local_obs.size(); ++q) {
    const int64_t k = P.local_obs[q];
    P.local_cam[q] = cam[k] - P.cam_begin;
    P.local_pt[q] = local_of_point[pt[k]];
  }
  // per local point: its global boundary index (or -1) and whether this rank
  // owns it for point-wise sums (the rank of its first, lowest-camera copy)
  const int32_t nl = (int32_t)P.local_points.size();
  P.bp_of_local.assign(nl, -1);
  P.owner_of_local.assign(nl, 1);
  for (int32_t i = 0; i < nl; ++i) {
    const int32_t g = P.local_points[i];
    P.bp_of_local[i] = bp_of_point[g];
    P.owner_of_local[i] = rmin[g] == rank ? 1 : 0;
  }
  // input index -> local observation index
  std::vector<int64_t> local_index_of_obs(l, -1);
  for (size_t q = 0; q < P.local_obs.size(); ++q) local_index_of_obs[P.local_obs[q]] = (int64_t)q;
  // exchange lists, all in global copy order:
  //  send to peer d: my copies of boundary points d holds;
  //  recv from peer s: s's copies of boundary points I hold.
  P.send_off.assign(world + 1, 0);
  P.recv_off.assign(world + 1, 0);
  for (int32_t b = 0; b < P.n_boundary_points; ++b)
    for (int64_t g = P.gb_off[b]; g < P.gb_off[b + 1]; ++g) {
      const int32_t o = g_owner[g];
      if (o == rank) {
        for (int32_t d = 0; d < world; ++d)
          if (d != rank && (holders[b] >> d & 1)) ++P.send_off[d + 1];
      } else if (holders[b] >> rank & 1) {
        ++P.recv_off[o + 1];
      }
    }
  for (int32_t r = 0; r < world; ++r) {
    P.send_off[r + 1] += P.send_off[r];
    P.recv_off[r + 1] += P.recv_off[r];
  }
  P.send_count = P.send_off[world];
  P.recv_count = P.recv_off[world];
  P.send_obs_local.assign(P.send_count, -1);
  P.gmap.assign(P.n_boundary_copies, -1);
  {
    std::vector<int64_t> sfill(P.send_off.begin(), P.send_off.end() - 1);
    std::vector<int64_t> rfill(P.recv_off.begin(), P.recv_off.end() - 1);
    for (int32_t b = 0; b < P.n_boundary_points; ++b)
      for (int64_t g = P.gb_off[b]; g < P.gb_off[b + 1]; ++g) {
        const int32_t o = g_owner[g];
        if (o == rank) {
          const int64_t q = local_index_of_obs[g_obs[g]];
          P.gmap[g] = -2 - q;
          for (int32_t d = 0; d < world; ++d)
            if (d != rank && (holders[b] >> d & 1)) P.send_obs_local[sfill[d]++] = q;
        } else if (holders[b] >> rank & 1) {
          P.gmap[g] = rfill[o]++;
        }
      }
  }
  // comm_floats of the reference (admm_solver.cpp:74-101): sum_i 3 d_i (d_i - 1)
  std::vector<int64_t> d(n, 0);
  for (int64_t k = 0; k < l; ++k) ++d[pt[k]];
  for (int32_t i = 0; i < n; ++i) P.comm_floats += 3 * d[i] * (d[i] > 0 ? d[i] - 1 : 0);
  P.total_obs = l;
  P.total_points = n;
  P.total_cameras = m;
  return P;
}

}  // namespace dbag

// ---- C-ABI (host only; testable without a GPU) ---------------------------------
struct dbag_shard_plan {
  dbag::ShardPlan p;
};

extern "C" {

int dbag_partition_cameras(int32_t m, const int64_t* obs_per_camera, int32_t world,
                           int32_t* cam_lo) {
  if (m < 1 || world < 1 || m < world) return DBAG_ERR_VALIDATION;
  std::vector<int64_t> c(obs_per_camera, obs_per_camera + m);
  const auto lo = dbag::partition_cameras(m, c, world);
  std::copy(lo.begin(), lo.end(), cam_lo);
  return DBAG_OK;
}

int dbag_shard_plan_create(const dbag_problem_view* full, int32_t rank, int32_t world,
                           dbag_shard_plan** out, dbag_shard_info* info) {
  *out = nullptr;
  try {
    auto* s = new dbag_shard_plan();
    s->p = dbag::make_shard_plan(full->num_cameras, full->num_points, full->num_obs,
                                 full->obs_cam, full->obs_pt, rank, world);
    *out = s;
    if (info) dbag_shard_plan_get_info(s, info);
    return DBAG_OK;
  } catch (const std::out_of_range&) {
    return DBAG_ERR_INDEX_OUT_OF_RANGE;
  } catch (...) {
    return DBAG_ERR_VALIDATION;
  }
}

void dbag_shard_plan_get_info(const dbag_shard_plan* s, dbag_shard_info* info) {
  const auto& p = s->p;
  info->rank = p.rank;
  info->world = p.world;
  info->cam_begin = p.cam_begin;
  info->cam_end = p.cam_end;
  info->local_obs = (int64_t)p.local_obs.size();
  info->local_points = (int32_t)p.local_points.size();
  info->boundary_points = p.n_boundary_points;
  info->boundary_copies = p.n_boundary_copies;
  info->send_count = p.send_count;
  info->recv_count = p.recv_count;
  info->comm_floats = p.comm_floats;
}

int dbag_shard_plan_arrays(const dbag_shard_plan* s, int32_t* cam_lo, int64_t* local_obs,
                           int32_t* local_points, int32_t* bp_of_local, int8_t* owner_of_local,
                           int64_t* gb_off, int64_t* gmap, int64_t* send_obs_local) {
  const auto& p = s->p;
  auto cp = [](auto* dst, const auto& v) {
    if (dst) std::copy(v.begin(), v.end(), dst);
  };
  cp(cam_lo, p.cam_lo);
  cp(local_obs, p.local_obs);
  cp(local_points, p.local_points);
  cp(bp_of_local, p.bp_of_local);
  cp(owner_of_local, p.owner_of_local);
  cp(gb_off, p.gb_off);
  cp(gmap, p.gmap);
  cp(send_obs_local, p.send_obs_local);
  return DBAG_OK;
}

int dbag_shard_plan_exchange(const dbag_shard_plan* s, int64_t* send_off, int64_t* recv_off) {
  const auto& p = s->p;
  if (send_off) std::copy(p.send_off.begin(), p.send_off.end(), send_off);
  if (recv_off) std::copy(p.recv_off.begin(), p.recv_off.end(), recv_off);
  return DBAG_OK;
}

void dbag_shard_plan_destroy(dbag_shard_plan* s) { delete s; }

}  // extern "C"
