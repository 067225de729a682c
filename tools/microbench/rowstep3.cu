// k_join's row-step loop on static shared-memory data, one factor at a time:
//   CALL  : an out-of-line slow path exists (never taken) vs an inline side effect
//   PREF  : next row-step's shared loads issued before the fire branch
// 8 warps x 2 CTAs per SM (16 warps/SM), kD = 8, ring of 320 columns per warp.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o rowstep3 rowstep3.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kD = 8, kH = 32, kRing = 320, kNB = kRing / kD;
struct __align__(16) WS {
  double2 colU[kRing];
  double2 colI[kRing];
  double2 rowU[kH + 1];
  double2 rowI[kH + 1];
};

__device__ __noinline__ void slow(double* out, double v) { out[threadIdx.x] += v; }

template <bool CALL, bool PREF, bool COLS = true, bool ROWS = true>
__global__ void __launch_bounds__(256, 2) k(double* out, int tiles) {
  extern __shared__ __align__(16) unsigned char sm[];
  WS& S = reinterpret_cast<WS*>(sm)[threadIdx.x >> 5];
  const int lane = threadIdx.x & 31;
  for (int q = lane; q < kRing; q += 32) {
    S.colU[q] = make_double2((q & 1) ? 1e-9 : -1e-9, (q & 2) ? 1e-9 : -1e-9);
    S.colI[q] = make_double2(0.5 + 1e-4 * q, 1e300);  // thresholds never reached
  }
  for (int q = lane; q <= kH; q += 32) {
    S.rowU[q] = make_double2((q & 1) ? 1e-9 : -1e-9, 2e-9);
    S.rowI[q] = make_double2(0.25, 1e300);
  }
  __syncwarp();
  double cov[kD];
  double2 cU[kD];
  double cinv[kD];
  int cthr[kD];
#pragma unroll
  for (int d = 0; d < kD; ++d) {
    cov[d] = d * 1e-3 + lane;
    cU[d] = S.colU[d * kNB + lane];
    cinv[d] = S.colI[d * kNB + lane].x;
    cthr[d] = __double2hiint(S.colI[d * kNB + lane].y);
  }
  for (int t = 0; t < tiles; ++t) {
    int b0 = (t * 4 + lane) % kNB;
    double2 nru = S.rowU[0];
    double2 nri = S.rowI[0];
    for (int u = 0; u < kH; u += kD) {
      const int b1 = b0 + 1 == kNB ? 0 : b0 + 1;
#pragma unroll
      for (int s = 0; s < kD; ++s) {
        const int h = u + s;
        const int sin = (s + kD - 1) % kD;
        if (COLS) {
          const int a = sin * kNB + (s == 0 ? b0 : b1);
          cU[sin] = S.colU[a];
          const double2 ci = S.colI[a];
          cinv[sin] = ci.x;
          cthr[sin] = __double2hiint(ci.y);
        }
        double2 ru, ri;
        if (!ROWS) {
          ru = make_double2(nru.x * 0.9999, nru.y);
          nru.x = ru.x;
          ri = nri;
        } else if (PREF) {
          ru = nru;
          ri = nri;
          nru = S.rowU[h + 1];
          nri = S.rowI[h + 1];
        } else {
          ru = S.rowU[h];
          ri = S.rowI[h];
        }
        const int rthr = __double2hiint(ri.y);
        bool fire = false;
        double c[kD];
#pragma unroll
        for (int d = 0; d < kD; ++d) {
          const int sl = (s + d) % kD;
          cov[d] = fma(ru.x, cU[sl].y, cov[d]);
          cov[d] = fma(ru.y, cU[sl].x, cov[d]);
          c[d] = cov[d] * (ri.x * cinv[sl]);
          const int hc = __double2hiint(c[d]);
          fire |= hc >= min(rthr, cthr[sl]);
        }
        if (__any_sync(0xffffffffu, fire && ri.x != 0.0)) {
          if (CALL) slow(out, c[0] + c[7]);
          else out[threadIdx.x] += c[0] + c[7];
        }
      }
      b0 = b1;
    }
  }
  double a = 0;
#pragma unroll
  for (int d = 0; d < kD; ++d) a += cov[d];
  if (a == 1.2345) out[0] = a;
}

template <bool C, bool P, bool COLS = true, bool ROWS = true>
void run(const char* name, int nsm, double* dout) {
  const int tiles = 600;
  const size_t smem = 8 * sizeof(WS);
  cudaFuncSetAttribute(k<C, P, COLS, ROWS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int blocks = nsm * 2 * 4;
  k<C, P, COLS, ROWS><<<blocks, 256, smem>>>(dout, 2);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<C, P, COLS, ROWS><<<blocks, 256, smem>>>(dout, tiles);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double cells = (double)blocks * 256 * tiles * kH * kD;
  printf("{\"variant\": \"%s\", \"cells_per_s\": %.3e, \"frac_of_4op_peak\": %.3f}\n", name,
         cells / (ms * 1e-3), cells / (ms * 1e-3) * 4 / 1.858e13);
}

int main() {
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  double* dout; cudaMalloc(&dout, 1 << 20); cudaMemset(dout, 0, 1 << 20);
  run<false, false>("inline_sideeffect, loads after branch", nsm, dout);
  run<true, false>("noinline_call, loads after branch", nsm, dout);
  run<false, true>("inline_sideeffect, prefetch", nsm, dout);
  run<true, true>("noinline_call, prefetch", nsm, dout);
  run<true, true, false, true>("noinline_call, prefetch, NO column loads", nsm, dout);
  run<true, true, true, false>("noinline_call, NO row loads", nsm, dout);
  run<true, true, false, false>("noinline_call, no smem at all", nsm, dout);
  return 0;
}
