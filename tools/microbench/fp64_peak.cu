// fp64 pipe microbenchmarks for the roofline denominator.
// Measures per-SM throughput of DFMA, DMUL, DSETP and the per-cell mix the
// diagonal kernel issues, in ops/clk/SM (clock64) and ops/s (CUDA events).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

constexpr int ILP = 8;
constexpr int ITERS = 1 << 16;

__global__ void k_dfma(double* out, long long* clk, double a, double b) {
  double x[ILP];
#pragma unroll
  for (int i = 0; i < ILP; ++i) x[i] = threadIdx.x * 1e-3 + i;
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) x[i] = fma(x[i], a, b);
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += x[i];
  if (s == 12345.678) out[0] = s;
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}

__global__ void k_dmul(double* out, long long* clk, double a, double b) {
  double x[ILP];
#pragma unroll
  for (int i = 0; i < ILP; ++i) x[i] = threadIdx.x * 1e-3 + i + b;
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) x[i] = x[i] * a;
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += x[i];
  if (s == 12345.678) out[0] = s;
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}

// fire = OR over 2*ILP compares, as chained setp.gt.or.f64 (one DSETP each).
__device__ __forceinline__ unsigned any_gt8(const double* c, double rt, const double* ct) {
  unsigned r;
  asm volatile("{\n\t.reg .pred p;\n\t"
      "setp.gt.f64 p, %1, %9;\n\t"
      "setp.gt.or.f64 p, %2, %9, p;\n\t"
      "setp.gt.or.f64 p, %3, %9, p;\n\t"
      "setp.gt.or.f64 p, %4, %9, p;\n\t"
      "setp.gt.or.f64 p, %5, %9, p;\n\t"
      "setp.gt.or.f64 p, %6, %9, p;\n\t"
      "setp.gt.or.f64 p, %7, %9, p;\n\t"
      "setp.gt.or.f64 p, %8, %9, p;\n\t"
      "setp.gt.or.f64 p, %1, %10, p;\n\t"
      "setp.gt.or.f64 p, %2, %11, p;\n\t"
      "setp.gt.or.f64 p, %3, %12, p;\n\t"
      "setp.gt.or.f64 p, %4, %13, p;\n\t"
      "setp.gt.or.f64 p, %5, %14, p;\n\t"
      "setp.gt.or.f64 p, %6, %15, p;\n\t"
      "setp.gt.or.f64 p, %7, %16, p;\n\t"
      "setp.gt.or.f64 p, %8, %17, p;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(r)
      : "d"(c[0]), "d"(c[1]), "d"(c[2]), "d"(c[3]), "d"(c[4]), "d"(c[5]), "d"(c[6]), "d"(c[7]),
        "d"(rt), "d"(ct[0]), "d"(ct[1]), "d"(ct[2]), "d"(ct[3]), "d"(ct[4]), "d"(ct[5]), "d"(ct[6]), "d"(ct[7]));
  return r;
}

// DSETP throughput alone: 16 compares per inner step (counted as 2*ILP ops / ILP "cells").
__global__ void k_dsetp(const double* in, double* out, long long* clk) {
  double x[ILP], ct[ILP];
#pragma unroll
  for (int i = 0; i < ILP; ++i) { x[i] = in[i] + threadIdx.x; ct[i] = in[8 + i]; }
  double rt = in[16];
  long long t0 = clock64();
  unsigned cnt = 0;
  for (int it = 0; it < ITERS; ++it) {
    cnt += any_gt8(x, rt, ct);
    rt = __longlong_as_double(__double_as_longlong(rt) ^ (it & 1));  // ALU-only perturbation
  }
  long long t1 = clock64();
  if (cnt == 777) out[0] = cnt;
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}

// The diagonal kernel's per-cell mix: 2 DFMA + 2 DMUL + 2 DSETP (chained OR).
__global__ void k_mix(const double* in, double* out, long long* clk) {
  double cov[ILP], cd[ILP], cf[ILP], ci[ILP], ct[ILP];
#pragma unroll
  for (int i = 0; i < ILP; ++i) {
    cov[i] = in[i] + threadIdx.x; cd[i] = in[8 + i]; cf[i] = in[16 + i]; ci[i] = in[24 + i]; ct[i] = in[32 + i];
  }
  double rf = in[40], rg = in[41], ri = in[42], rt = in[43];
  long long t0 = clock64();
  unsigned cnt = 0;
  for (int it = 0; it < ITERS; ++it) {
    double c[ILP];
#pragma unroll
    for (int i = 0; i < ILP; ++i) {
      cov[i] = fma(rf, cd[i], cov[i]);
      cov[i] = fma(rg, cf[i], cov[i]);
      c[i] = cov[i] * ri * ci[i];
    }
    unsigned f = any_gt8(c, rt, ct);
    if (f) { cnt++; rt = c[0] + 1.0; }
  }
  long long t1 = clock64();
  if (cnt == 777) out[0] = cov[0] + cov[ILP - 1];
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}

__global__ void k_dfma2(const double* in, double* out, long long* clk) {
  double x[ILP];
  double a = in[0], b = in[1];
#pragma unroll
  for (int i = 0; i < ILP; ++i) x[i] = threadIdx.x * 1e-3 + i;
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) x[i] = fma(x[i], a, b);
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += x[i];
  if (s == 12345.678) out[0] = s;
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}

template <typename K>
int run(const char* name, K kern, int ops_per_inner, int nsm) {
  const int threads = 256;
  const int blocks = nsm * 4;
  double* out; long long* clk;
  CK(cudaMalloc(&out, 8)); CK(cudaMalloc(&clk, blocks * 8));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int w = 0; w < 3; ++w) kern<<<blocks, threads>>>(out, clk, 1.0000001, 1e-7);
  CK(cudaDeviceSynchronize());
  cudaEventRecord(e0);
  const int reps = 5;
  for (int r = 0; r < reps; ++r) kern<<<blocks, threads>>>(out, clk, 1.0000001, 1e-7);
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  long long* hclk = new long long[blocks];
  CK(cudaMemcpy(hclk, clk, blocks * 8, cudaMemcpyDeviceToHost));
  double avg = 0; for (int i = 0; i < blocks; ++i) avg += hclk[i]; avg /= blocks;
  double ops = (double)reps * blocks * threads * ITERS * (double)ILP * ops_per_inner;
  double per_s = ops / (ms * 1e-3);
  // 4 blocks resident per SM (256 thr each) -> per-SM ops per clock over the block's own clock window
  double per_clk_sm = (double)4 * threads * ITERS * ILP * ops_per_inner / avg;
  double f_eff = per_s / (per_clk_sm * nsm);
  printf("{\"kernel\": \"%s\", \"ops_per_s\": %.4e, \"ops_per_clk_per_sm\": %.2f, \"implied_mhz\": %.0f, \"ms\": %.3f}\n",
         name, per_s, per_clk_sm, f_eff / 1e6, ms / reps);
  delete[] hclk; cudaFree(out); cudaFree(clk);
  return 0;
}

__device__ __forceinline__ unsigned any_gt8_s64(const double* c, long long rt, const long long* ct) {
  unsigned r;
  asm volatile("{\n\t.reg .pred p;\n\t"
      "setp.gt.s64 p, %1, %9;\n\t"
      "setp.gt.or.s64 p, %2, %9, p;\n\t"
      "setp.gt.or.s64 p, %3, %9, p;\n\t"
      "setp.gt.or.s64 p, %4, %9, p;\n\t"
      "setp.gt.or.s64 p, %5, %9, p;\n\t"
      "setp.gt.or.s64 p, %6, %9, p;\n\t"
      "setp.gt.or.s64 p, %7, %9, p;\n\t"
      "setp.gt.or.s64 p, %8, %9, p;\n\t"
      "setp.gt.or.s64 p, %1, %10, p;\n\t"
      "setp.gt.or.s64 p, %2, %11, p;\n\t"
      "setp.gt.or.s64 p, %3, %12, p;\n\t"
      "setp.gt.or.s64 p, %4, %13, p;\n\t"
      "setp.gt.or.s64 p, %5, %14, p;\n\t"
      "setp.gt.or.s64 p, %6, %15, p;\n\t"
      "setp.gt.or.s64 p, %7, %16, p;\n\t"
      "setp.gt.or.s64 p, %8, %17, p;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(r)
      : "l"(__double_as_longlong(c[0])), "l"(__double_as_longlong(c[1])), "l"(__double_as_longlong(c[2])),
        "l"(__double_as_longlong(c[3])), "l"(__double_as_longlong(c[4])), "l"(__double_as_longlong(c[5])),
        "l"(__double_as_longlong(c[6])), "l"(__double_as_longlong(c[7])),
        "l"(rt), "l"(ct[0]), "l"(ct[1]), "l"(ct[2]), "l"(ct[3]), "l"(ct[4]), "l"(ct[5]), "l"(ct[6]), "l"(ct[7]));
  return r;
}

// Same cell mix with the filter compares done on the integer pipe (bit patterns of
// non-negative doubles order like signed int64).
__global__ void k_mix_s64(const double* in, double* out, long long* clk) {
  double cov[ILP], cd[ILP], cf[ILP], ci[ILP];
  long long ct[ILP];
#pragma unroll
  for (int i = 0; i < ILP; ++i) {
    cov[i] = in[i] + threadIdx.x; cd[i] = in[8 + i]; cf[i] = in[16 + i]; ci[i] = in[24 + i];
    ct[i] = __double_as_longlong(in[32 + i]);
  }
  double rf = in[40], rg = in[41], ri = in[42];
  long long rt = __double_as_longlong(in[43]);
  long long t0 = clock64();
  unsigned cnt = 0;
  for (int it = 0; it < ITERS; ++it) {
    double c[ILP];
#pragma unroll
    for (int i = 0; i < ILP; ++i) {
      cov[i] = fma(rf, cd[i], cov[i]);
      cov[i] = fma(rg, cf[i], cov[i]);
      c[i] = cov[i] * ri * ci[i];
    }
    unsigned f = any_gt8_s64(c, rt, ct);
    if (f) { cnt++; rt = __double_as_longlong(c[0] + 1.0); }
  }
  long long t1 = clock64();
  if (cnt == 777) out[0] = cov[0] + cov[ILP - 1];
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}

// Four fp64 ops per cell only (no compares): the floor the filter sits on.
__global__ void k_mix_nocmp(const double* in, double* out, long long* clk) {
  double cov[ILP], cd[ILP], cf[ILP], ci[ILP];
#pragma unroll
  for (int i = 0; i < ILP; ++i) {
    cov[i] = in[i] + threadIdx.x; cd[i] = in[8 + i]; cf[i] = in[16 + i]; ci[i] = in[24 + i];
  }
  double rf = in[40], rg = in[41], ri = in[42];
  double acc = 0;
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) {
      cov[i] = fma(rf, cd[i], cov[i]);
      cov[i] = fma(rg, cf[i], cov[i]);
      ci[i] = cov[i] * ri * ci[i];
    }
  }
  long long t1 = clock64();
#pragma unroll
  for (int i = 0; i < ILP; ++i) acc += ci[i];
  if (acc == 777.0) out[0] = cov[0] + cov[ILP - 1];
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}

template <typename K>
int run2(const char* name, K kern, double ops_per_inner, int nsm, const double* din) {
  const int threads = 256;
  const int blocks = nsm * 4;
  double* out; long long* clk;
  CK(cudaMalloc(&out, 8)); CK(cudaMalloc(&clk, blocks * 8));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int w = 0; w < 3; ++w) kern<<<blocks, threads>>>(din, out, clk);
  CK(cudaDeviceSynchronize());
  cudaEventRecord(e0);
  const int reps = 5;
  for (int r = 0; r < reps; ++r) kern<<<blocks, threads>>>(din, out, clk);
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  long long* hclk = new long long[blocks];
  CK(cudaMemcpy(hclk, clk, blocks * 8, cudaMemcpyDeviceToHost));
  double avg = 0; for (int i = 0; i < blocks; ++i) avg += hclk[i]; avg /= blocks;
  double ops = (double)reps * blocks * threads * ITERS * (double)ILP * ops_per_inner;
  double per_s = ops / (ms * 1e-3);
  int occ = 0; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, 0);
  int resident = occ < 4 ? occ : 4;  // grid = 4 blocks per SM
  double per_clk_sm = (double)resident * threads * ITERS * ILP * ops_per_inner / avg;
  double f_eff = per_s / (per_clk_sm * nsm);
  printf("{\"kernel\": \"%s\", \"ops_per_s\": %.4e, \"ops_per_clk_per_sm\": %.2f, \"occ\": %d, \"implied_mhz\": %.0f, \"ms\": %.3f}\n",
         name, per_s, per_clk_sm, occ, f_eff / 1e6, ms / reps);
  delete[] hclk; cudaFree(out); cudaFree(clk);
  return 0;
}

int main() {
  int dev = 0, nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceProp p; cudaGetDeviceProperties(&p, dev);
  printf("{\"device\": \"%s\", \"sms\": %d}\n", p.name, nsm);
  run("dfma", k_dfma, 1, nsm);
  run("dmul", k_dmul, 1, nsm);
  double h[64]; for (int i = 0; i < 64; ++i) h[i] = 1e-3 * (i + 1);
  h[40] = 1e-9; h[41] = -1e-9; h[42] = 0.25; h[43] = 1e30;
  for (int i = 0; i < 8; ++i) h[32 + i] = 1e30;
  h[16] = 1e30; for (int i = 0; i < 8; ++i) h[8 + i] = 1e30;
  double* din; CK(cudaMalloc(&din, sizeof(h))); CK(cudaMemcpy(din, h, sizeof(h), cudaMemcpyHostToDevice));
  run2("dfma_runtime_operands", k_dfma2, 1, nsm, din);
  run2("dsetp_or_chain", k_dsetp, 2, nsm, din);  // 16 compares per ILP=8 step -> 2 per element
  run2("cell_mix(2dfma+2dmul+2dsetp) cells", k_mix, 1, nsm, din);  // per cell
  run2("cell_mix_s64(2dfma+2dmul+2isetp64) cells", k_mix_s64, 1, nsm, din);
  run2("cell_mix_nocmp(2dfma+2dmul) cells", k_mix_nocmp, 1, nsm, din);
  run2("dfma_runtime_operands_again", k_dfma2, 1, nsm, din);
  return 0;
}
