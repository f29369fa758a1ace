// dbag_exact.h — host launchers of the exact-numerics kernels (dbag_exact.cu,
// compiled with -fmad=false). See that file for the rationale.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "dbag_common.cuh"

namespace dbag {
namespace exact {
cudaError_t launch_local(const DevState& S, int64_t begin, int64_t count, cudaStream_t st);
cudaError_t launch_camera(const DevState& S, int mode, cudaStream_t st);
cudaError_t launch_point(const DevState& S, int mode, bool metric, int n_parts, cudaStream_t st);
cudaError_t launch_camR_all(const DevState& S, cudaStream_t st);
// doubles of the pooled Huber K1's L-BFGS history scratch on the current
// device (0 on error)
size_t huber_history_doubles();
// test hook: count n branch-free reciprocals that differ bitwise from IEEE 1/d
cudaError_t selftest_rcp(int64_t n, unsigned long long seed, unsigned long long* bad_dev);
}  // namespace exact
}  // namespace dbag
