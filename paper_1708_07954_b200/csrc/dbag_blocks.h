// dbag_blocks.h — generalized local blocks (BlockConfig{points_per_block,
// cameras_per_block} != {1,1}; the paper's §3.1.4 "more than one observation
// per update step", admm_solver.cpp:14-72,144-290). Host interface used by the
// C-ABI (dbag_capi.cu); kernels in dbag_blocks.cu (EXACT numerics).
//
// A general solver reuses the (1,1) solver's device state for everything that
// does not depend on the block structure: the K0 sort (partition() sorts by
// (cam_id, point_id) exactly like the (1,1) block order, so a block is a run of
// that order), the consensus x̄/ȳ/camR, the point-major observations used by
// the fused metric, the reference state, the record reductions. It adds the
// block ranges, the flattened copies/duals and the point -> copy map.
#pragma once

#include <cstdint>
#include <vector>

#include <cuda_runtime.h>

#include "dbag_common.cuh"

namespace dbag {
namespace blocks {

// partition() over observations already sorted by (cam_id, point_id): block b
// is the sorted range [obs_off[b], obs_off[b+1]); its points / cameras are
// pt_ids[pt_off[b]..) / cam_ids[cam_off[b]..) in ascending id order; obs_pl /
// obs_cl are each observation's local indices (lower_bound into those lists).
struct Partition {
  std::vector<int64_t> obs_off, pt_off, cam_off;  // [B+1]
  std::vector<int32_t> pt_ids, cam_ids;           // [PC], [CC]
  std::vector<int32_t> obs_pl, obs_cl;            // [L]
  int32_t max_np = 0, max_nc = 0, max_nobs = 0;
  int64_t blocks() const { return (int64_t)obs_off.size() - 1; }
};
Partition partition_sorted(int64_t L, const int32_t* cam_sorted, const int32_t* pt_sorted,
                           int32_t points_per_block, int32_t cameras_per_block);
// communication_cost (admm_solver.cpp:74-101): owner = lowest camera of a block.
int64_t communication_cost(const Partition& P, int32_t M, int32_t N);

// Kernel-side view (passed by value).
struct GenState {
  int64_t B, PC, CC, L;
  const int64_t* obs_off;   // [B+1] into the (cam, pt)-sorted order (== (1,1) block order)
  const int64_t* pc_off;    // [B+1]
  const int64_t* cc_off;    // [B+1]
  const int32_t* pt_ids;    // [PC]
  const int32_t* cam_ids;   // [CC]
  const int32_t* obs_pl;    // [L]
  const int32_t* obs_cl;    // [L]
  const int64_t* ptc_off;   // [N+1] point -> its copy slots, block order
  const int64_t* ptc_slot;  // [PC]
  const int64_t* camc_off;  // [M+1] camera -> contiguous copy slots
  double* gx;               // [3][PC] local point copies x_i^b
  double* gr;               // [3][PC] duals r
  double* gy;               // [6][CC] local camera copies (pose)
  double* gs;               // [6][CC] duals s
  double* mscratch;         // per-CTA global LDLT matrices when not in shared memory
  int32_t max_np, max_nc, max_nobs, max_dim;
  int32_t m_in_smem;
  unsigned long long* work; // block work counter
};

struct GenSolver {
  GenState G{};
  Partition part;
  std::vector<void*> pool;
  int64_t comm_floats = 0;
  size_t smem_bytes = 0;   // per CTA
  size_t group_bytes = 0;  // per block (thread group)
  bool warp_groups = false;  // a warp per block (small D) instead of a CTA
  int resident = 0;   // K1G CTAs (persistent)
  int device = 0;

  ~GenSolver();
  // After the (1,1) K0 build of S: partition, maps, copies = consensus, duals = 0.
  cudaError_t init(const DevState& S, int32_t ppb, int32_t cpb, int device, cudaStream_t st);
  cudaError_t reset_copies(const DevState& S, cudaStream_t st);
  // Local solves of blocks [begin, begin+count) (local_update / _all).
  cudaError_t local(const DevState& S, int64_t begin, int64_t count, cudaStream_t st);
  // Camera consensus (mode&1) / dual (mode&2) over copies; S.cam_stats, S.camR.
  cudaError_t cameras(const DevState& S, int mode, cudaStream_t st);
  // Point consensus / dual over copies, fused metric over the point's
  // observations; S.part_pt[n_parts][4] in the (1,1) K2 format.
  cudaError_t points(const DevState& S, int mode, bool metric, int n_parts, cudaStream_t st);
  // dir 0: device -> host buffers, 1: host -> device ([PC][3], [CC][6], ...).
  cudaError_t copies_io(double* lp, double* lc, double* r, double* s, int dir, cudaStream_t st);
  cudaError_t dual_sums(const DevState& S, double* pts, double* cams, cudaStream_t st);
  cudaError_t block_objective(const DevState& S, int64_t b, double* d_out, cudaStream_t st);
  cudaError_t max_primal(const DevState& S, double* d_out2, cudaStream_t st);
  int64_t ops_per_iteration() const { return G.B + G.PC + G.CC; }
};

}  // namespace blocks
}  // namespace dbag
