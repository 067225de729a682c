// k_join's fast block (branch-free blocks of 8 row-steps, 4 predicate
// accumulators, VIMNMX3 row test) on static shared-memory data, comparing the
// fp64 filter (corr = cov * (rinv * cinv) with 2 DMUL per cell) against an
// fp32 filter: cov's high word -> fp32 bits (IMNMX clamp + LEA), cov_f * rinv_f
// with packed FMUL2, then * cinv_f, compares on the float bits. The fp32 form
// halves the fp64-pipe work per cell (2 DFMA instead of 2 DFMA + 2 DMUL).
// Thresholds are never reached, so no block replays (fast blocks alone).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o rowstep_f32 rowstep_f32.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kD = 8, kH = 32, kRing = 320, kNB = kRing / kD;
struct __align__(16) WS {
  double2 colU[kRing];
  double2 colI[kRing];
  double2 rowU[kH + 1];
  double2 rowI[kH + 1];
};

__device__ __forceinline__ int f32bits_of_hi(int h, int clamp) {
  // (h << 3) - (896 << 23): exponent rebias 1023 -> 127, 20 mantissa bits.
  // clamp 1: max(h, hi(2^-121)) first, so negative / tiny covariances map to a
  // tiny positive float instead of wrapping; clamp 2: also min(h, hi(2^128)),
  // so huge covariances map to +inf (a conservative fire) instead of wrapping.
  if (clamp >= 1) h = max(h, (1023 - 121) << 20);
  if (clamp >= 2) h = min(h, (1023 + 128) << 20);
  return (h << 3) - (896 << 23);
}

// MODE 0: fp64 filter (production). 1: fp32 filter with the clamp. 2: fp32, no clamp.
#ifndef RS_WARPS
#define RS_WARPS 8
#endif
#ifndef RS_MINB
#define RS_MINB 2
#endif
template <int MODE>
__global__ void __launch_bounds__(RS_WARPS * 32, RS_MINB) k(double* out, int tiles) {
  extern __shared__ __align__(16) unsigned char sm[];
  WS& S = reinterpret_cast<WS*>(sm)[threadIdx.x >> 5];
  const int lane = threadIdx.x & 31;
  for (int q = lane; q < kRing; q += 32) {
    S.colU[q] = make_double2((q & 1) ? 1e-9 : -1e-9, (q & 2) ? 1e-9 : -1e-9);
    if (MODE == 0)
      S.colI[q] = make_double2(0.5 + 1e-4 * q, __hiloint2double(__double2hiint(0.5 + 1e-4 * q), 0x7ff00000));
    else {
      const float cf = 0.5f + 1e-4f * q;
      S.colI[q] = make_double2(0.5 + 1e-4 * q, __hiloint2double(__float_as_int(cf), 0x7f000000));
    }
  }
  for (int q = lane; q <= kH; q += 32) {
    S.rowU[q] = make_double2((q & 1) ? 1e-9 : -1e-9, 2e-9);
    if (MODE == 0)
      S.rowI[q] = make_double2(0.25, __hiloint2double(0x7ff00000, 0));
    else
      S.rowI[q] = make_double2(0.25, __hiloint2double(0x7f000000, __float_as_int(0.25f)));
  }
  __syncwarp();
  double cov[kD];
  double2 cU[kD];
  double cpk[kD];
#pragma unroll
  for (int d = 0; d < kD; ++d) {
    cov[d] = d * 1e-3 + lane;
    cU[d] = S.colU[d * kNB + lane];
    cpk[d] = S.colI[d * kNB + lane].y;
  }
  for (int t = 0; t < tiles; ++t) {
    int b0 = (t * 4 + lane) % kNB;
    for (int u = 0; u < kH; u += kD) {
      const int b1 = b0 + 1 == kNB ? 0 : b0 + 1;
      double covs[kD];
#pragma unroll
      for (int d = 0; d < kD; ++d) covs[d] = cov[d];
      bool fa = false, fb = false, fc = false, fd = false;
#pragma unroll
      for (int s = 0; s < kD; ++s) {
        const int h = u + s;
        const int sin = (s + kD - 1) % kD;
        {
          const int a = sin * kNB + (s == 0 ? b0 : b1);
          cU[sin] = S.colU[a];
          cpk[sin] = S.colI[a].y;
        }
        const double2 ru = S.rowU[h];
        const double2 ri = S.rowI[h];
        int hcs[kD];
        int rthr;
        if (MODE == 0) {
          rthr = __double2hiint(ri.y);
#pragma unroll
          for (int d = 0; d < kD; ++d) {
            const int sl = (s + d) % kD;
            cov[d] = fma(ru.x, cU[sl].y, cov[d]);
            cov[d] = fma(ru.y, cU[sl].x, cov[d]);
            hcs[d] = __double2hiint(cov[d] * (ri.x * cpk[sl]));
          }
        } else {
          rthr = __double2hiint(ri.y);
          const float rf = __int_as_float(__double2loint(ri.y));
          float cf[kD];
#pragma unroll
          for (int d = 0; d < kD; ++d) {
            const int sl = (s + d) % kD;
            cov[d] = fma(ru.x, cU[sl].y, cov[d]);
            cov[d] = fma(ru.y, cU[sl].x, cov[d]);
            cf[d] = __int_as_float(f32bits_of_hi(__double2hiint(cov[d]), MODE == 1 ? 1 : (MODE == 3 ? 2 : 0)));
          }
#pragma unroll
          for (int d = 0; d < kD; d += 2) {
            const float2 q = __fmul2_rn(make_float2(cf[d], cf[d + 1]), make_float2(rf, rf));
            hcs[d] = __float_as_int(q.x * __int_as_float(__double2hiint(cpk[(s + d) % kD])));
            hcs[d + 1] = __float_as_int(q.y * __int_as_float(__double2hiint(cpk[(s + d + 1) % kD])));
          }
        }
        const int m1 = __vimax3_s32(hcs[0], hcs[1], hcs[2]);
        const int m2 = __vimax3_s32(hcs[3], hcs[4], hcs[5]);
        const int m3 = __vimax3_s32(hcs[6], hcs[7], m1);
        fa |= max(m2, m3) >= rthr;
        bool* acc4[4] = {&fb, &fc, &fd, &fa};
#pragma unroll
        for (int d = 0; d < kD; ++d)
          *acc4[d & 3] |= hcs[d] >= (MODE == 0 ? __double2hiint(cpk[(s + d) % kD]) : __double2loint(cpk[(s + d) % kD]));
      }
      if (__any_sync(0xffffffffu, (fa | fb) | (fc | fd))) {
#pragma unroll
        for (int d = 0; d < kD; ++d) cov[d] = covs[d] + 1.0;
        out[threadIdx.x] += cov[0];
      }
      b0 = b1;
    }
  }
  double a = 0;
#pragma unroll
  for (int d = 0; d < kD; ++d) a += cov[d];
  if (a == 1.2345) out[0] = a;
}

template <int MODE>
void run(const char* name, int nsm, double* dout) {
  const int tiles = 600;
  const size_t smem = RS_WARPS * sizeof(WS);
  cudaFuncSetAttribute(k<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int blocks = nsm * RS_MINB * 4;
  k<MODE><<<blocks, RS_WARPS * 32, smem>>>(dout, 2);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < 3; ++r) {
    cudaEventRecord(e0);
    k<MODE><<<blocks, RS_WARPS * 32, smem>>>(dout, tiles);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    best = ms < best ? ms : best;
  }
  const double cells = (double)blocks * RS_WARPS * 32 * tiles * kH * kD;
  const double rowsteps_per_smsp = (double)blocks * RS_WARPS * tiles * kH / (nsm * 4);
  printf("{\"warps\": %d, \"minb\": %d, \"variant\": \"%s\", \"cells_per_s\": %.3e, \"cycles_per_rowstep_at_1965\": %.1f, \"err\": \"%s\"}\n",
         RS_WARPS, RS_MINB, name, cells / (best * 1e-3), best * 1e-3 * 1.965e9 / rowsteps_per_smsp,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  double* dout;
  cudaMalloc(&dout, 1 << 20);
  cudaMemset(dout, 0, 1 << 20);
  run<0>("fp64 filter (2 DMUL/cell)", nsm, dout);
  run<1>("fp32 filter, IMNMX clamp + LEA + FMUL2(cov*rinv) + FMUL(*cinv)", nsm, dout);
  run<2>("fp32 filter, LEA + FMUL2 + FMUL, no clamp", nsm, dout);
  run<3>("fp32 filter, two-sided clamp (IMNMX x2) + LEA + FMUL2 + FMUL", nsm, dout);
  return 0;
}
