// Does a second read of a chunk, a few microseconds after the first, hit L2?
// Each CTA walks private chunks of a large buffer and reads every chunk twice
// (MODE picks the load flavour); ncu's dram__bytes_read.sum against the buffer
// size answers it.  nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o l2_reread l2_reread.cu
//   ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum ./l2_reread <chunk_KB> <mode>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

template <int MODE>
__device__ __forceinline__ double ld(const double* p, unsigned long long pol) {
  double v;
  if (MODE == 0) asm volatile("ld.global.f64 %0, [%1];" : "=d"(v) : "l"(p));
  if (MODE == 1) asm volatile("ld.global.cg.f64 %0, [%1];" : "=d"(v) : "l"(p));
  if (MODE == 2) asm volatile("ld.global.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
  if (MODE == 3) asm volatile("ld.global.nc.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}

template <int MODE>
__global__ void k(const double* buf, size_t chunk, size_t nchunks, double* out) {
  unsigned long long pol = 0;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  double acc = 0.0;
  for (size_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
    const double* p = buf + c * chunk;
    for (int pass = 0; pass < 2; ++pass) {
      for (size_t i = threadIdx.x; i < chunk; i += blockDim.x) acc += ld<MODE>(p + i, pol);
      __syncthreads();
    }
  }
  if (acc == 12345.678) out[0] = acc;
}

int main(int argc, char** argv) {
  const size_t chunk_kb = argc > 1 ? atoi(argv[1]) : 64;
  const int mode = argc > 2 ? atoi(argv[2]) : 0;
  const int ctas_per_sm = argc > 3 ? atoi(argv[3]) : 4;
  const size_t total = (size_t)4 << 30;
  const size_t chunk = chunk_kb * 1024 / 8, nchunks = total / 8 / chunk;
  double *buf, *out;
  cudaMalloc(&buf, total);
  cudaMalloc(&out, 8);
  cudaMemset(buf, 0, total);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(a);
    const int grid = 148 * ctas_per_sm;
    if (mode == 0) k<0><<<grid, 256>>>(buf, chunk, nchunks, out);
    if (mode == 1) k<1><<<grid, 256>>>(buf, chunk, nchunks, out);
    if (mode == 2) k<2><<<grid, 256>>>(buf, chunk, nchunks, out);
    if (mode == 3) k<3><<<grid, 256>>>(buf, chunk, nchunks, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("chunk %zu KB mode %d ctas/sm %d: %.3f ms, %.1f GB/s of requested bytes (2 x 4 GiB)%s\n", chunk_kb, mode,
           ctas_per_sm, ms, 2.0 * total / ms / 1e6, cudaGetLastError() == cudaSuccess ? "" : " ERROR");
  }
  return 0;
}
