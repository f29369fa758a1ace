// Dependent-chain latency of FP64 DADD / DMUL / DFMA and of the MUFU.RCP64H
// seed on this GPU (cycles per operation, one warp, clock64). Evidence for the
// K1 EXACT `wait` stalls: its LDLT dots are chains of DADDs.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/fp64_latency.cu -o /tmp/fp64_latency
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void chain(double* out, long long* cyc, int n, double a, double b) {
  double x = a;
  const long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    if (OP == 0) x = __dadd_rn(x, b);
    else if (OP == 1) x = __dmul_rn(x, b);
    else if (OP == 2) x = __fma_rn(x, b, a);
    else { asm volatile("rcp.approx.ftz.f64 %0, %0;" : "+d"(x)); }
  }
  const long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 32 * sizeof(double));
  cudaMalloc(&cyc, sizeof(long long));
  const int n = 1 << 16;
  const char* names[4] = {"DADD", "DMUL", "DFMA", "MUFU.RCP64H"};
  for (int op = 0; op < 4; ++op) {
    for (int rep = 0; rep < 2; ++rep) {  // second pass is the warm one
      if (op == 0) chain<0><<<1, 32>>>(out, cyc, n, 1.0, 1e-9);
      if (op == 1) chain<1><<<1, 32>>>(out, cyc, n, 1.0, 1.0000001);
      if (op == 2) chain<2><<<1, 32>>>(out, cyc, n, 1.0, 0.5);
      if (op == 3) chain<3><<<1, 32>>>(out, cyc, n, 1.5, 0.0);
      cudaDeviceSynchronize();
    }
    long long c = 0;
    cudaMemcpy(&c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
    printf("%-12s %.2f cycles per dependent op\n", names[op], (double)c / n);
  }
  return 0;
}
