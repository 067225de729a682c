// DFMA / DMUL throughput vs number of distinct 64-bit source registers.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o operands operands.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void __launch_bounds__(256, 2) k(const double* in, double* out, int iters) {
  double x[8], a[8], b[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) { x[i] = in[i] + threadIdx.x; a[i] = in[8 + i]; b[i] = in[16 + i]; }
  const double sa = in[24], sb = in[25];
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) x[i] = fma(sa, sb, x[i]);          // 2 shared operands
      if (MODE == 1) x[i] = fma(sa, b[i], x[i]);        // 1 shared, 1 distinct
      if (MODE == 2) x[i] = fma(a[i], b[i], x[i]);      // all distinct
      if (MODE == 3) x[i] = x[i] * b[i];                // DMUL distinct
      if (MODE == 4) { x[i] = fma(sa, b[i], x[i]); x[i] = fma(sb, a[i], x[i]); }  // k_join's pair
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 1.2345) out[0] = s;
}

template <int M>
void run(const char* name, int nsm, const double* din, double* dout, int ops) {
  const int iters = 20000, blocks = nsm * 2 * 4;
  k<M><<<blocks, 256>>>(din, dout, 10);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<M><<<blocks, 256>>>(din, dout, iters);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double r = (double)blocks * 256 * iters * 8 * ops / (ms * 1e-3);
  printf("{\"variant\": \"%s\", \"fp64_ops_per_s\": %.3e, \"frac\": %.3f}\n", name, r, r / 1.861e13);
}

int main() {
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  double h[32]; for (int i = 0; i < 32; ++i) h[i] = 1.0 + 1e-9 * i;
  double *din, *dout; cudaMalloc(&din, sizeof(h)); cudaMalloc(&dout, 64);
  cudaMemcpy(din, h, sizeof(h), cudaMemcpyHostToDevice);
  run<0>("dfma 2 shared operands", nsm, din, dout, 1);
  run<1>("dfma 1 shared 1 distinct", nsm, din, dout, 1);
  run<2>("dfma all distinct", nsm, din, dout, 1);
  run<3>("dmul distinct", nsm, din, dout, 1);
  run<4>("dfma pair (k_join recurrence)", nsm, din, dout, 2);
  return 0;
}
