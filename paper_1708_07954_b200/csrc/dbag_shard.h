// dbag_shard.h — host-side shard plan (see dbag_shard.cpp).
#pragma once

#include <cstdint>
#include <vector>

#include "../../include/dbag.h"

namespace dbag {

struct ShardPlan {
  int32_t rank = 0, world = 1;
  std::vector<int32_t> cam_lo;          // [world+1] camera ranges
  int32_t cam_begin = 0, cam_end = 0;   // this rank's range
  std::vector<int64_t> local_obs;       // input indices of local observations (input order)
  std::vector<int32_t> local_cam;       // per local obs: local camera id (cam - cam_begin)
  std::vector<int32_t> local_pt;        // per local obs: local point id
  std::vector<int32_t> local_points;    // local point -> global id (ascending)
  std::vector<int32_t> bp_of_local;     // local point -> global boundary index or -1
  std::vector<int8_t> owner_of_local;   // 1 if this rank holds the point's first copy
  int32_t n_boundary_points = 0;
  int64_t n_boundary_copies = 0;
  std::vector<int64_t> gb_off;          // [n_boundary_points+1] global boundary copy ranges
  // Per-peer exchange (one ncclSend/ncclRecv pair per peer in one group): a
  // boundary copy travels only to the OTHER ranks that hold its point.
  // gmap[g] for every global boundary copy g: >= 0 recv slot (a peer's copy of
  // a point this rank holds); -2 - q for this rank's own copy (local obs q);
  // -1 when this rank does not hold the point.
  std::vector<int64_t> gmap;
  std::vector<int64_t> send_off;        // [world+1] send slots per destination peer
  std::vector<int64_t> send_obs_local;  // [send_count] local obs of each send slot
  std::vector<int64_t> recv_off;        // [world+1] recv slots per source peer
  int64_t send_count = 0, recv_count = 0;
  int64_t comm_floats = 0;
  int64_t total_obs = 0;
  int32_t total_points = 0, total_cameras = 0;
};

std::vector<int32_t> partition_cameras(int32_t m, const std::vector<int64_t>& obs_per_camera,
                                       int32_t world);
ShardPlan make_shard_plan(int32_t m, int32_t n, int64_t l, const int32_t* cam, const int32_t* pt,
                          int32_t rank, int32_t world);

}  // namespace dbag
