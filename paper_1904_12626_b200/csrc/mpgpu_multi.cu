// Multivariate joins on the GPU: SiMPle (mprof::simple_join) and mSTOMP
// (mprof::mstomp), profile.hpp:91-100.
//
// Both walk the same diagonal space as K3 (cells (i, i + k), unique pairs for
// a self-join), one diagonal per lane, a band of 32 diagonals x a segment of
// rows per warp, and keep row / column minima as packed (value, index) int64
// keys min-merged with RED.MIN (ties to the smallest index, merge_min's
// strict-improvement order). The search value is approximate only up to the
// recurrence's rounding; finalize recomputes every reported value exactly
// from the chosen partner by direct sums.
//
//   k_simple     raw QT recurrence summed over dims (one accumulator per lane):
//                QT(i,j) = QT(i-1,j-1) + sum_d (r_d[i+m-1] c_d[j+m-1] - r_d[i-1] c_d[j-1])
//                on per-dim globally centred data (distances are shift-invariant),
//                value = |R_i|^2 + |C_j|^2 - 2 QT clamped at 0 (the squared distance).
//   k_mstomp<D>  D centred-covariance recurrences per lane (K3's df/dg form), per-dim
//                z-normalised distance with the flat convention, a stable sort of the
//                D distances (must dims first), prefix means -> D keys per cell.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "mpgpu_internal.h"
#include "mprof_gpu.h"

namespace {

using mpgpu_internal::set_error;

#ifndef MPGPU_MWARPS
#define MPGPU_MWARPS 8
#endif
constexpr int kMWarps = MPGPU_MWARPS;           // warps per CTA
constexpr long long kNoKey = 0x7fffffffffffffffLL;
constexpr double kRawSnap = 1e-12;              // OR_RAW_SNAP, distance.hpp:54-57
constexpr int kMaxMDims = 32;                   // mSTOMP admissible dims

#define MM_CUDA(call)                                                                      \
  do {                                                                                     \
    cudaError_t e_ = (call);                                                               \
    if (e_ != cudaSuccess)                                                                 \
      return set_error(e_ == cudaErrorMemoryAllocation ? MPGPU_ENOMEM : MPGPU_ECUDA,       \
                       std::string(#call) + ": " + cudaGetErrorString(e_));                \
  } while (0)

struct MItem {
  long long kb;  // first diagonal of the 32-diagonal band
  long long r0;  // first row of the segment
  int nrows;     // rows in the segment
  int pass;
};

__device__ __forceinline__ void red_min64(long long* p, long long v) {
  asm volatile("red.relaxed.gpu.global.min.s64 [%0], %1;\n" ::"l"(p), "l"(v));
}

__device__ __forceinline__ long long pack_key(double v, long long idx, long long imask) {
  return (__double_as_longlong(v) & ~imask) | idx;
}

__device__ __forceinline__ long long warp_min64(long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const long long u = __shfl_xor_sync(0xffffffffu, v, o);
    v = u < v ? u : v;
  }
  return v;
}

// sqrt for the search (s >= 0) as s * rsqrt(s): rsqrt.approx.ftz.f64 is the
// bare MUFU.RSQ64H (relative error 2^-20) and one Newton step brings it to
// 1.3e-12 (tools/microbench/rsqrt_accuracy.cu); 5 fp64 ops in all. The
// non-ftz rsqrt.approx.f64 is already refined by ptxas (5 ops and a slow-path
// branch), and sqrt() adds a further refinement on top.
__device__ __forceinline__ double sqrt_search(double s) {
  const double s2 = s + 1e-300;  // keeps rsqrt finite at 0
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(s2));
  const double h = 0.5 * s2;
  y = fma(y, fma(-h * y, y, 0.5), y);
  return s * y;
}

// max(v, 0) on the integer pipe: a negative value (rounding residue of a
// perfect match) gets its high word zeroed, leaving a tiny non-negative
// denormal that the search treats as 0.
__device__ __forceinline__ double clamp0(double v) {
  const int h = __double2hiint(v);
  return __hiloint2double(h < 0 ? 0 : h, __double2loint(v));
}

// ---- SiMPle ------------------------------------------------------------------
// Keys are the squared distance's bits | index. kNoKeyS (the largest finite
// double's bits) marks "no candidate": every finite value beats it while the
// +inf of padded columns does not. Padding entries of the key arrays hold
// kPadKey (hi word INT_MIN), so padded columns never pass the filter.
constexpr long long kNoKeyS = 0x7fefffffffffffffLL;
constexpr long long kPadKey = (long long)0x8000000000000000ULL;
constexpr int kSimplePad = 8 * 32 + 64;  // entries of zero / +inf padding after the last window

struct RawSeries {
  const double* xc;   // dims x ns (stride), centred per dim (shared shift), zero padded
  const double* nrm;  // L + pad: summed centred window energies, +inf in the padding
  long long n, ns, L;
  const double2* V;   // dims x Lp: V[q][j] = {xc_q[j-1], xc_q[j+m-1]} (ring kernel), zero padded
  long long Lp;
};
struct SimplePass {
  RawSeries R, C;
  long long klo, khi;  // diagonals [klo, khi): cells (i, i + k)
  long long* keyR;     // + padding (kPadKey)
  long long* keyC;
};
struct SimpleParams {
  SimplePass pass[2];
  const MItem* items;
  long long n_items;
  int dims, m;
  long long imask;
  unsigned long long* stats;  // MPGPU_STATS=1: [steps, slow-path steps, column REDs, row REDs]
};

// High word of a key. An L1 copy may be stale (RED.MIN lands in L2), which
// only costs extra slow-path entries (keys never increase); reading at L2
// (ld.global.cg) measured slower (SiMPle d=1: 11.6 -> 12.3 ms) for the same
// fire rate.
__device__ __forceinline__ int key_hi(const long long* k, long long i) {
  return reinterpret_cast<const int*>(k)[2 * i + 1];
}

// KD consecutive diagonals per lane (a 32*KD-diagonal band per warp), DIMS
// compile-time. Column data of the lane's KD columns live in a register shift
// window (one column enters per row-step); row data are broadcast loads. Per
// cell: 2 DIMS DFMA (QT recurrence), one DADD + one DFMA for the squared
// distance, and an integer filter on its high word against the row threshold
// (min of the lane's KD high words) and the column's cached threshold. A step
// in which any lane passes the filter runs the exact key update (RED.MIN).
template <int KD, int DIMS>
__global__ void __launch_bounds__(kMWarps * 32, 2) k_simple_t(const SimpleParams P) {
  const long long wid = (long long)blockIdx.x * kMWarps + (threadIdx.x >> 5);
  if (wid >= P.n_items) return;
  const int lane = threadIdx.x & 31;
  const MItem it = P.items[wid];
  const SimplePass& S = P.pass[it.pass];
  const double* __restrict__ xr = S.R.xc;
  const double* __restrict__ xc = S.C.xc;
  const long long nsR = S.R.ns, nsC = S.C.ns;
  const int m = P.m;
  const long long r0 = it.r0;
  const long long c0 = r0 + it.kb + (long long)lane * KD;  // column of diagonal 0 at row r0
  const long long imask = P.imask;

  double qt[KD];
#pragma unroll
  for (int d = 0; d < KD; ++d) qt[d] = 0.0;
#pragma unroll
  for (int q = 0; q < DIMS; ++q) {
    const double* a = xr + q * nsR + r0;
    const double* c = xc + q * nsC + c0;
    for (int t = 0; t < m; ++t) {
      const double av = a[t];
#pragma unroll
      for (int d = 0; d < KD; ++d) qt[d] = fma(av, c[t + d], qt[d]);
    }
  }
  double co[KD][DIMS], cn[KD][DIMS], cnr[KD];
  int cth[KD];
#pragma unroll
  for (int d = 0; d < KD - 1; ++d) {
    const long long j = c0 + d;
#pragma unroll
    for (int q = 0; q < DIMS; ++q) {
      co[d][q] = j > 0 ? xc[q * nsC + j - 1] : 0.0;
      cn[d][q] = xc[q * nsC + j + m - 1];
    }
    cnr[d] = S.C.nrm[j];
    cth[d] = key_hi(S.keyC, j);
  }
  // One row-step: the entering column and the row, the recurrence, the squared
  // distances and the filter; with `slow` the exact key updates run when any
  // lane passed. Returns this lane's filter result.
  // Software pipeline: the entering column and the row of step t + 1 are
  // loaded while step t computes (the per-step vote would otherwise keep the
  // scheduler from hoisting them).
  double pco[DIMS], pcn[DIMS], pro[DIMS], prn[DIMS], pcnr, prnr;
  int pcth, prth;
  auto fetch = [&](const long long t) {
    const long long i = r0 + t, jn = c0 + t + KD - 1;
#pragma unroll
    for (int q = 0; q < DIMS; ++q) {
      pco[q] = jn > 0 ? xc[q * nsC + jn - 1] : 0.0;
      pcn[q] = xc[q * nsC + jn + m - 1];
      pro[q] = t > 0 ? xr[q * nsR + i - 1] : 0.0;  // the seed row takes no update
      prn[q] = t > 0 ? xr[q * nsR + i + m - 1] : 0.0;
    }
    pcnr = S.C.nrm[jn];
    pcth = key_hi(S.keyC, jn);
    prnr = S.R.nrm[i];
    prth = key_hi(S.keyR, i);
  };
  fetch(0);
  auto step = [&](const int s, const long long u, const bool slow) -> bool {
    const long long i = r0 + u + s;
    const int sin = (s + KD - 1) % KD;
    double ro[DIMS], rn[DIMS];
#pragma unroll
    for (int q = 0; q < DIMS; ++q) {
      co[sin][q] = pco[q];
      cn[sin][q] = pcn[q];
      ro[q] = pro[q];
      rn[q] = prn[q];
    }
    cnr[sin] = pcnr;
    cth[sin] = pcth;
    const double rnr = prnr;
    const int rth = prth;
    fetch(u + s + 1);
    double v[KD];
    bool fire = false;
    int hmin = 0x7fffffff;
#pragma unroll
    for (int d = 0; d < KD; ++d) {
      const int sl = (s + d) % KD;
#pragma unroll
      for (int q = 0; q < DIMS; ++q) {
        qt[d] = fma(-ro[q], co[sl][q], qt[d]);
        qt[d] = fma(rn[q], cn[sl][q], qt[d]);
      }
      v[d] = fma(-2.0, qt[d], rnr + cnr[sl]);
      const int h = __double2hiint(v[d]);
      hmin = min(hmin, h);
      fire |= h <= cth[sl];
    }
    fire |= hmin <= rth;
    if (slow && __any_sync(0xffffffffu, fire)) {
      if (P.stats && lane == 0) atomicAdd(&P.stats[1], 1ull);
      long long best = kNoKeyS;
      const bool row_ok = i < S.R.L;
#pragma unroll
      for (int d = 0; d < KD; ++d) {
        const int sl = (s + d) % KD;
        const long long j = c0 + u + s + d;
        const double vv = fmax(v[d], 0.0);
        const int h = __double2hiint(vv);
        if (row_ok && j < S.C.L) {
          if (h <= cth[sl]) {
            if (P.stats) atomicAdd(&P.stats[2], 1ull);
            red_min64(&S.keyC[j], pack_key(vv, i, imask));
            cth[sl] = min(cth[sl], h);
          }
          if (h <= rth) {
            const long long kr = pack_key(vv, j, imask);
            best = kr < best ? kr : best;
          }
        }
      }
      best = warp_min64(best);
      if (lane == 0 && best != kNoKeyS) {
        if (P.stats) atomicAdd(&P.stats[3], 1ull);
        red_min64(&S.keyR[i], best);
      }
    }
    return fire;
  };
  // (Branch-free blocks of KD steps with a replay on fire, as in k_join, were
  // measured slower here: 11.6 -> 13.0 ms at d = 1, 7.3 -> 8.7 ms at d = 3.)
  for (int u = 0; u < it.nrows; u += KD) {
#pragma unroll
    for (int s = 0; s < KD; ++s) {
      if (P.stats && lane == 0) atomicAdd(&P.stats[0], 1ull);
      step(s, u, true);
    }
  }
}

// ---- SiMPle on a shared-memory ring (k_join's data path) ---------------------
// Same cells, filter and key updates as k_simple_t, but every operand comes
// from a per-warp shared-memory ring filled by cp.async one tile ahead: rows
// of tile t+1 (kSH rows) and the kSH columns entering the band while tile t
// computes, so the row-step loop never waits on L1/L2. A column record is
// DIMS planes of V = {x[j-1], x[j+m-1]} plus {energy, key}, each plane
// blocked-transposed so the 32 lanes' entering columns are 32 consecutive
// 16-byte slots (conflict-free LDS.128). Rows are broadcast loads.
template <int KD, int DIMS>
struct SRing {
  static constexpr int TS = DIMS <= 3 ? 32 : 16;                        // rows per tile
  static constexpr int kWs = 32 * KD;                                   // diagonals per band
  static constexpr int R = ((kWs + 2 * TS + KD - 1) / KD) * KD;         // ring slots
  static constexpr int NB = R / KD;
  static constexpr int kPlanes = DIMS + 1;
  static constexpr int kRowPlane = TS + 1;
  static constexpr int kPerWarp = kPlanes * R + 2 * kPlanes * kRowPlane;  // double2 per warp
  static constexpr size_t kSmem = sizeof(double2) * kPerWarp * kMWarps;
  // rows padded to whole tiles and the band's last columns stay inside the padding
  static_assert(kWs + TS <= kSimplePad, "padding too short for the ring kernel");
};

__device__ __forceinline__ unsigned sm_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void cpa16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sm_u32(dst)), "l"(src));
}
__device__ __forceinline__ void cpa8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sm_u32(dst)), "l"(src));
}
__device__ __forceinline__ void cpa_wait() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

template <int KD, int DIMS, bool BLK>
__global__ void __launch_bounds__(kMWarps * 32, 2) k_simple_r(const SimpleParams P) {
  using G = SRing<KD, DIMS>;
  constexpr int R = G::R, NB = G::NB, NP = G::kPlanes, RP = G::kRowPlane, kWs = G::kWs, kSH = G::TS;
  extern __shared__ double2 sring[];
  double2* const ring = sring + (threadIdx.x >> 5) * G::kPerWarp;  // plane e at ring + e R
  double2* const rows = ring + NP * R;                              // (buf NP + e) RP + h
  const long long wid = (long long)blockIdx.x * kMWarps + (threadIdx.x >> 5);
  if (wid >= P.n_items) return;
  const int lane = threadIdx.x & 31;
  const MItem it = P.items[wid];
  const SimplePass& S = P.pass[it.pass];
  const int m = P.m;
  const long long r0 = it.r0;
  const long long cw = r0 + it.kb;             // column of (lane 0, d = 0) at row r0
  const long long c0 = cw + (long long)lane * KD;
  const long long imask = P.imask;
  const long long LpR = S.R.Lp, LpC = S.C.Lp;
  const int nT = it.nrows / kSH;

  auto raddr = [](int x) {  // x: column offset from cw (< 2^31; 32-bit slot math)
    const int p = x % R;
    return (p % KD) * NB + p / KD;
  };
  auto fetch_col = [&](int x) {
    const long long j = cw + x;
    const int a = raddr(x);
#pragma unroll
    for (int q = 0; q < DIMS; ++q) cpa16(&ring[q * R + a], &S.C.V[q * LpC + j]);
    cpa8(&ring[DIMS * R + a].x, &S.C.nrm[j]);
    cpa8(&ring[DIMS * R + a].y, &S.keyC[j]);
  };
  auto fetch_row = [&](int buf, int h, long long i) {
#pragma unroll
    for (int q = 0; q < DIMS; ++q) cpa16(&rows[(buf * NP + q) * RP + h], &S.R.V[q * LpR + i]);
    cpa8(&rows[(buf * NP + DIMS) * RP + h].x, &S.R.nrm[i]);
    cpa8(&rows[(buf * NP + DIMS) * RP + h].y, &S.keyR[i]);
  };

  // tile 0 in flight while the seeds are computed
  if (lane < kSH) fetch_row(0, lane, r0 + lane);
  for (int x = lane; x < kSH + kWs - 1; x += 32) fetch_col(x);

  // seeds: QT(r0, c0 + d) by direct dot products over all dims
  double qt[KD];
#pragma unroll
  for (int d = 0; d < KD; ++d) qt[d] = 0.0;
#pragma unroll
  for (int q = 0; q < DIMS; ++q) {
    const double* a = S.R.xc + q * S.R.ns + r0;
    const double* c = S.C.xc + q * S.C.ns + c0;
    for (int t = 0; t < m; ++t) {
      const double av = a[t];
#pragma unroll
      for (int d = 0; d < KD; ++d) qt[d] = fma(av, c[t + d], qt[d]);
    }
  }
  cpa_wait();
  __syncwarp();
  if (lane == 0) {
#pragma unroll
    for (int q = 0; q < DIMS; ++q) rows[q * RP] = make_double2(0.0, 0.0);  // the seed row takes no update
  }
  __syncwarp();

  double2 cv[KD][DIMS];
  double ce[KD];
  int cth[KD];
#pragma unroll
  for (int d = 0; d < KD - 1; ++d) {  // slots 0..KD-2: columns lane KD + d
    const int a = d * NB + lane;
#pragma unroll
    for (int q = 0; q < DIMS; ++q) cv[d][q] = ring[q * R + a];
    const double2 e = ring[DIMS * R + a];
    ce[d] = e.x;
    cth[d] = __double2hiint(e.y);
  }

  for (int t = 0; t < nT; ++t) {
    const int buf = t & 1;
    const int ts = t * kSH;
    if (t + 1 < nT) {
      if (lane < kSH) {
        fetch_row(buf ^ 1, lane, r0 + ts + kSH + lane);
        fetch_col(ts + kSH + kWs - 1 + lane);
      }
    }
    int b0 = (int)((ts / KD + lane) % NB), b1 = 0;
    // One row-step: the entering column and the row from the ring, the
    // recurrence, the squared distances and the filter. Without `slow` it only
    // reports whether this lane passed; with it, a step in which any lane
    // passed runs the exact key updates.
    auto step = [&](const int s, const int u, const bool slow) -> bool {
      const int h = u + s;
      const int sin = (s + KD - 1) % KD;
      {
        const int a = sin * NB + (s == 0 ? b0 : b1);
#pragma unroll
        for (int q = 0; q < DIMS; ++q) cv[sin][q] = ring[q * R + a];
        const double2 e = ring[DIMS * R + a];
        ce[sin] = e.x;
        cth[sin] = __double2hiint(e.y);
      }
      double2 rv[DIMS];
#pragma unroll
      for (int q = 0; q < DIMS; ++q) rv[q] = rows[(buf * NP + q) * RP + h];
      const double2 re = rows[(buf * NP + DIMS) * RP + h];
      const int rth = __double2hiint(re.y);
      double v[KD];
      bool fire = false;
      int hmin = 0x7fffffff;
#pragma unroll
      for (int d = 0; d < KD; ++d) {
        const int sl = (s + d) % KD;
#pragma unroll
        for (int q = 0; q < DIMS; ++q) {
          qt[d] = fma(-rv[q].x, cv[sl][q].x, qt[d]);
          qt[d] = fma(rv[q].y, cv[sl][q].y, qt[d]);
        }
        v[d] = fma(-2.0, qt[d], re.x + ce[sl]);
        const int hv = __double2hiint(v[d]);
        hmin = min(hmin, hv);
        fire |= hv <= cth[sl];
      }
      fire |= hmin <= rth;
      if (slow && __any_sync(0xffffffffu, fire)) {
        if (P.stats && lane == 0) atomicAdd(&P.stats[1], 1ull);
        const int rho = ts + h;
        const long long i = r0 + rho;
        long long best = kNoKeyS;
        const bool row_ok = i < S.R.L;
#pragma unroll
        for (int d = 0; d < KD; ++d) {
          const int sl = (s + d) % KD;
          const long long j = c0 + rho + d;
          const double vv = fmax(v[d], 0.0);
          const int hv = __double2hiint(vv);
          if (row_ok && j < S.C.L) {
            if (hv <= cth[sl]) {
              if (P.stats) atomicAdd(&P.stats[2], 1ull);
              const long long kc = pack_key(vv, i, imask);
              red_min64(&S.keyC[j], kc);
              cth[sl] = min(cth[sl], hv);
              // the lane that takes this column next reads the lowered key
              double2& e = ring[DIMS * R + raddr(rho + lane * KD + d)];
              if (kc < __double_as_longlong(e.y)) e.y = __longlong_as_double(kc);
            }
            if (hv <= rth) {
              const long long kr = pack_key(vv, j, imask);
              best = kr < best ? kr : best;
            }
          }
        }
        best = warp_min64(best);
        if (lane == 0 && best != kNoKeyS) {
          if (P.stats) atomicAdd(&P.stats[3], 1ull);
          red_min64(&S.keyR[i], best);
        }
      }
      return fire;
    };
    // Blocks of KD row-steps run branch-free (loads and DFMAs of later steps
    // schedule across earlier ones); a block in which any lane passed the
    // filter (about 1% with the coarse warm start) is replayed from its saved
    // start with the per-step exact path. Every cell's arithmetic is identical.
    for (int u = 0; u < kSH; u += KD) {
      b1 = b0 + 1 == NB ? 0 : b0 + 1;
      double qts[KD];
#pragma unroll
      for (int d = 0; d < KD; ++d) qts[d] = qt[d];
      if constexpr (!BLK) {  // per-step vote and exact path
#pragma unroll
        for (int s = 0; s < KD; ++s) step(s, u, true);
        b0 = b1;
        continue;
      }
      bool any = false;
#pragma unroll
      for (int s = 0; s < KD; ++s) any |= step(s, u, false);
      if (__any_sync(0xffffffffu, any)) {
        if (P.stats && lane == 0) atomicAdd(&P.stats[0], 1ull << 40);  // replayed blocks (high bits)
#pragma unroll
        for (int d = 0; d < KD; ++d) qt[d] = qts[d];
#pragma unroll
        for (int q = 0; q < KD - 1; ++q) {  // the block-start window: columns rho0 + lane KD + q
          const int a = q * NB + b0;
#pragma unroll
          for (int r = 0; r < DIMS; ++r) cv[q][r] = ring[r * R + a];
          const double2 e = ring[DIMS * R + a];
          ce[q] = e.x;
          cth[q] = __double2hiint(e.y);
        }
#pragma unroll
        for (int s = 0; s < KD; ++s) step(s, u, true);
      }
      b0 = b1;
    }
    if (P.stats && lane == 0) atomicAdd(&P.stats[0], (unsigned long long)kSH);  // row-steps (low bits)
    if (t + 1 < nT) cpa_wait();
    __syncwarp();
  }
}

// {xc[j-1], xc[j+m-1]} per dim (j = 0: {0, xc[m-1]}), zero past the last window
__global__ void k_build_v(const double* __restrict__ xc, long long ns, long long L, long long Lp,
                          int dims, int m, double2* __restrict__ V) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= Lp * dims) return;
  const long long q = t / Lp, j = t % Lp;
  const double* x = xc + q * ns;
  V[t] = j < L ? make_double2(j > 0 ? x[j - 1] : 0.0, x[j + m - 1]) : make_double2(0.0, 0.0);
}

// Any dimension count, dims outermost: a tile of T row-steps x KD diagonals
// per lane accumulates the QT increments of every (step, diagonal) dimension by
// dimension (2 DFMA each), so one dimension's T row values and T + KD - 1
// column values are live at a time whatever the dimension count; the cells
// are then evaluated step by step (running QT, squared distance, high-word
// filter, exact updates on a pass) as in k_simple_t.
template <int KD, int T>
__global__ void __launch_bounds__(kMWarps * 32, 2) k_simple_dt(const SimpleParams P) {
  const long long wid = (long long)blockIdx.x * kMWarps + (threadIdx.x >> 5);
  if (wid >= P.n_items) return;
  const int lane = threadIdx.x & 31;
  const MItem it = P.items[wid];
  const SimplePass& S = P.pass[it.pass];
  const double* __restrict__ xr = S.R.xc;
  const double* __restrict__ xc = S.C.xc;
  const long long nsR = S.R.ns, nsC = S.C.ns;
  const int m = P.m, dims = P.dims;
  const long long r0 = it.r0;
  const long long c0 = r0 + it.kb + (long long)lane * KD;
  const long long imask = P.imask;

  double qt[KD];
#pragma unroll
  for (int d = 0; d < KD; ++d) qt[d] = 0.0;
  for (int q = 0; q < dims; ++q) {
    const double* a = xr + q * nsR + r0;
    const double* c = xc + q * nsC + c0;
    for (int t = 0; t < m; ++t) {
      const double av = a[t];
#pragma unroll
      for (int d = 0; d < KD; ++d) qt[d] = fma(av, c[t + d], qt[d]);
    }
  }
  constexpr int E = T + KD - 1;  // columns a tile touches per lane
  for (int u = 0; u < it.nrows; u += T) {
    double dl[T][KD];
#pragma unroll
    for (int s = 0; s < T; ++s)
#pragma unroll
      for (int d = 0; d < KD; ++d) dl[s][d] = 0.0;
    const long long ib = r0 + u, jb = c0 + u;
    for (int q = 0; q < dims; ++q) {
      const double* rq = xr + q * nsR + ib;
      const double* cq = xc + q * nsC + jb;
      double ro[T], rn[T], co[E], cn[E];
#pragma unroll
      for (int s = 0; s < T; ++s) {
        const bool upd = (u + s) != 0;  // the seed row takes no update
        ro[s] = upd ? rq[s - 1] : 0.0;
        rn[s] = upd ? rq[s + m - 1] : 0.0;
      }
#pragma unroll
      for (int e = 0; e < E; ++e) {
        co[e] = (jb + e) > 0 ? cq[e - 1] : 0.0;
        cn[e] = cq[e + m - 1];
      }
#pragma unroll
      for (int s = 0; s < T; ++s)
#pragma unroll
        for (int d = 0; d < KD; ++d)
          dl[s][d] = fma(rn[s], cn[s + d], fma(-ro[s], co[s + d], dl[s][d]));
    }
    double cnr[E];
    int cth[E];
#pragma unroll
    for (int e = 0; e < E; ++e) {
      cnr[e] = S.C.nrm[jb + e];
      cth[e] = key_hi(S.keyC, jb + e);
    }
#pragma unroll
    for (int s = 0; s < T; ++s) {
      const long long i = ib + s;
      const double rnr = S.R.nrm[i];
      const int rth = key_hi(S.keyR, i);
      double v[KD];
      bool fire = false;
      int hmin = 0x7fffffff;
#pragma unroll
      for (int d = 0; d < KD; ++d) {
        qt[d] += dl[s][d];
        v[d] = fma(-2.0, qt[d], rnr + cnr[s + d]);
        const int h = __double2hiint(v[d]);
        hmin = min(hmin, h);
        fire |= h <= cth[s + d];
      }
      fire |= hmin <= rth;
      if (__any_sync(0xffffffffu, fire)) {
        long long best = kNoKeyS;
        const bool row_ok = i < S.R.L;
#pragma unroll
        for (int d = 0; d < KD; ++d) {
          const long long j = jb + s + d;
          const double vv = fmax(v[d], 0.0);
          const int h = __double2hiint(vv);
          if (row_ok && j < S.C.L) {
            if (h <= cth[s + d]) {
              red_min64(&S.keyC[j], pack_key(vv, i, imask));
              cth[s + d] = min(cth[s + d], h);
            }
            if (h <= rth) {
              const long long kr = pack_key(vv, j, imask);
              best = kr < best ? kr : best;
            }
          }
        }
        best = warp_min64(best);
        if (lane == 0 && best != kNoKeyS) red_min64(&S.keyR[i], best);
      }
    }
  }
}

// Any dimension count: one diagonal per lane, column data read per step.
__global__ void __launch_bounds__(kMWarps * 32, 2) k_simple(const SimpleParams P) {
  const long long wid = (long long)blockIdx.x * kMWarps + (threadIdx.x >> 5);
  if (wid >= P.n_items) return;
  const int lane = threadIdx.x & 31;
  const MItem it = P.items[wid];
  const SimplePass& S = P.pass[it.pass];
  const long long k = it.kb + lane;
  const long long r0 = it.r0;
  const int m = P.m, dims = P.dims;
  const long long nsR = S.R.ns, nsC = S.C.ns;
  double qt = 0.0;
  for (int d = 0; d < dims; ++d) {
    const double* xr = S.R.xc + d * nsR + r0;
    const double* xc = S.C.xc + d * nsC + r0 + k;
    for (int t = 0; t < m; ++t) qt = fma(xr[t], xc[t], qt);
  }
  for (long long i = r0; i < r0 + it.nrows; ++i) {
    const long long j = i + k;
    if (i > r0) {
      for (int d = 0; d < dims; ++d) {
        const double* xr = S.R.xc + d * nsR;
        const double* xc = S.C.xc + d * nsC;
        qt = fma(-xr[i - 1], xc[j - 1], qt);
        qt = fma(xr[i + m - 1], xc[j + m - 1], qt);
      }
    }
    const double vv = fmax(fma(-2.0, qt, S.R.nrm[i] + S.C.nrm[j]), 0.0);
    const bool ok = i < S.R.L && j < S.C.L;
    long long kr = kNoKeyS;
    if (ok) {
      kr = pack_key(vv, j, P.imask);
      const long long kc = pack_key(vv, i, P.imask);
      if (kc < __ldcg(&S.keyC[j])) red_min64(&S.keyC[j], kc);
    }
    const long long tr = __ldcg(&S.keyR[i]);
    if (__any_sync(0xffffffffu, kr < tr)) {
      const long long b = warp_min64(kr);
      if (lane == 0 && b < tr) red_min64(&S.keyR[i], b);
    }
  }
}

// Exact raw distance between window i of X and window j of Y over all dims,
// one warp; scale = summed raw window energies for the snap.
__device__ double warp_raw_exact(const double* X, long long nx, long long i, const double* Y,
                                 long long ny, long long j, int dims, int m, int lane) {
  double d2 = 0.0, sc = 0.0;
  for (int d = 0; d < dims; ++d) {
    const double* x = X + d * nx + i;
    const double* y = Y + d * ny + j;
    for (int t = lane; t < m; t += 32) {
      const double e = x[t] - y[t];
      d2 = fma(e, e, d2);
      sc = fma(x[t], x[t], sc);
      sc = fma(y[t], y[t], sc);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    d2 += __shfl_xor_sync(0xffffffffu, d2, o);
    sc += __shfl_xor_sync(0xffffffffu, sc, o);
  }
  return d2 <= kRawSnap * sc ? 0.0 : sqrt(d2);
}

// Keys -> values / index (and left / right for a self-join). One warp per window.
__global__ void k_simple_finalize(const double* X, long long nx, long long LX, const double* Y,
                                  long long ny, const long long* __restrict__ k0,
                                  const long long* __restrict__ k1, int dims, int m,
                                  long long imask, double* mp, long long* pi, long long* left,
                                  long long* right) {
  const long long i = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (i >= LX) return;
  const long long a = k0[i];
  const long long b = k1 ? k1[i] : kNoKeyS;
  const long long best = a < b ? a : b;
  const long long bi = best == kNoKeyS ? -1 : (best & imask);
  double v = INFINITY;
  if (bi >= 0) v = warp_raw_exact(X, nx, i, Y, ny, bi, dims, m, lane);
  if (lane == 0) {
    if (mp) mp[i] = v;
    if (pi) pi[i] = bi;
    // self: k0 = right keys (partners j > i), k1 = left keys (partners j < i)
    if (right) right[i] = a == kNoKeyS ? -1 : (a & imask);
    if (left) left[i] = b == kNoKeyS ? -1 : (b & imask);
  }
}

__global__ void k_fill_val(long long* k, long long len, long long total, long long v, long long pad) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < total) k[i] = i < len ? v : pad;
}

// blocked interleave of the mSTOMP statistics (mblk): WU = {df, dg}, WI =
// {inv, 0.5 when window j of dim q is flat}; keys filled alongside (kNoKeyS,
// kPadKey past the last window)
__global__ void k_build_w(const double2* __restrict__ U, const double* __restrict__ inv,
                          long long L, long long Lp, long long Lb, int D, double2* __restrict__ WU,
                          double2* __restrict__ WI, long long* __restrict__ keys) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= Lb * D) return;
  const long long blk = t / (32LL * D);
  const int q = (int)((t / 32) % D);
  const long long j = blk * 32 + (t & 31);
  const double a = j < Lp ? inv[q * Lp + j] : 0.0;
  WU[t] = j < Lp ? U[q * Lp + j] : make_double2(0.0, 0.0);
  WI[t] = make_double2(a, (j < L && a == 0.0) ? 0.5 : 0.0);
  keys[t] = j < L ? kNoKeyS : kPadKey;
}

// per-dim centring by a shared shift (distances are shift-invariant) into a
// zero-padded layout of stride ns
__global__ void k_center(const double* __restrict__ x, long long n, long long ns, int dims,
                         const double* __restrict__ shift, double* __restrict__ xc) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= ns * dims) return;
  const long long d = t / ns, p = t % ns;
  xc[t] = p < n ? x[d * n + p] - shift[d] : 0.0;
}

// summed centred window energies (+inf in the padding)
__global__ void k_raw_energy(const double* __restrict__ xc, long long ns, long long L,
                             long long Lp, int dims, int m, double* __restrict__ nrm) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= Lp) return;
  if (i >= L) {
    nrm[i] = INFINITY;
    return;
  }
  double s = 0.0;
  for (int d = 0; d < dims; ++d) {
    const double* w = xc + d * ns + i;
    for (int t = 0; t < m; ++t) s = fma(w[t], w[t], s);
  }
  nrm[i] = s;
}

// ---- mSTOMP --------------------------------------------------------------------

struct MStompParams {
  const double* x;    // D x ns (admissible dims, must first; zero padded)
  const double* mu;   // D x Lp (zero padded)
  const double* inv;  // D x Lp (0: flat / padding)
  const double2* U;   // D x Lp
  // blocked layout [j / 32][q][j % 32] (mblk): a warp's 32 consecutive windows
  // are one contiguous run per dim, and dim q sits at the constant offset 32 q
  const double2* WU;  // {df, dg}
  const double2* WI;  // {inv, 0.5 if the window is flat else 0}
  long long n, ns, L, Lp;
  long long khi;      // diagonals [klo, khi) = [zone + 1, L)
  long long* keys;    // blocked like WU: kNoKeyS when empty, kPadKey in the padding
  const MItem* items;
  long long n_items;
  int m, n_must;
  int D;              // admissible dims (<= the kernel's capacity)
  long long imask;
  unsigned long long* stats;  // MPGPU_STATS=1: [row-steps, exact row-steps]
};

// element index of (window j, dim 0) in the blocked layout; dim q adds 32 q
__device__ __forceinline__ long long mblk(long long j, int D) {
  return ((j >> 5) * D << 5) + (j & 31);
}

// stable odd-even transposition sort of D unsigned keys (ascending)
template <int D>
__device__ __forceinline__ void sort_keys(unsigned long long (&s)[D]) {
#pragma unroll
  for (int r = 0; r < D; ++r) {
#pragma unroll
    for (int q = (r & 1); q + 1 < D; q += 2) {
      const unsigned long long a = s[q], b = s[q + 1];
      const bool sw = a > b;
      s[q] = sw ? b : a;
      s[q + 1] = sw ? a : b;
    }
  }
}

// the same network on 32-bit keys, min / max per compare-exchange (the fast pass)
template <int D>
__device__ __forceinline__ void sort_u32(unsigned (&s)[D]) {
#pragma unroll
  for (int r = 0; r < D; ++r) {
#pragma unroll
    for (int q = (r & 1); q + 1 < D; q += 2) {
      const unsigned a = s[q], b = s[q + 1];
      s[q] = min(a, b);
      s[q + 1] = max(a, b);
    }
  }
}

// fp32 search distance for the fast pass: s = 2m(1 - corr) >= 0 (clamped below
// at 2^-100: its high word turned into fp32 bits by one LEA, 20 mantissa bits,
// truncated) and the approximate fp32 square root (MUFU.SQRT)
constexpr int kTinyHi = (1023 - 100) << 20;
__device__ __forceinline__ float dist_fast(double s) {
  const int h = max(__double2hiint(s), kTinyHi);
  float r;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(__int_as_float((h << 3) - (896 << 23))));
  return r;
}
// high word of the fp64 value nearest an fp32 value (positive normal): the
// fast pass compares it with the keys' high words like the exact pass
__device__ __forceinline__ int hi_of_f32(float f) {
  return (int)((unsigned)__float_as_int(f) >> 3) + (896 << 20);
}

template <int D>
__global__ void __launch_bounds__(kMWarps * 32) k_mstomp(const MStompParams P) {
  const long long wid = (long long)blockIdx.x * kMWarps + (threadIdx.x >> 5);
  if (wid >= P.n_items) return;
  const int lane = threadIdx.x & 31;
  const MItem it = P.items[wid];
  const long long k = it.kb + lane;
  const long long r0 = it.r0;
  long long rend = min(r0 + it.nrows, P.L - k);
  if (k >= P.khi || rend < r0) rend = r0;
  const int m = P.m;
  const double two_m = 2.0 * m;

  double cov[D];
#pragma unroll
  for (int q = 0; q < D; ++q) {
    cov[q] = 0.0;
    if (r0 < rend && q < P.D) {
      const double* xr = P.x + q * P.ns + r0;
      const double* xc = P.x + q * P.ns + r0 + k;
      const double mr = P.mu[q * P.Lp + r0], mc = P.mu[q * P.Lp + r0 + k];
      double acc = 0.0, asum = 0.0;
      for (int t = 0; t < m; ++t) {
        const double a = xr[t] - mr;
        asum += a;
        acc = fma(a, xc[t], acc);
      }
      cov[q] = fma(-mc, asum, acc);
    }
  }
  const unsigned long long kFree = 1ULL << 63;  // sorts free dims after the must dims
  const long long rmax = __reduce_max_sync(0xffffffffu, (unsigned)(rend - r0)) + r0;
  const int Dr = P.D;
  for (long long i = r0; i < rmax; ++i) {
    const bool live = i < rend;
    const long long j = live ? i + k : i;  // dead lanes read a valid column
    const long long ei = mblk(i, Dr), ej = mblk(j, Dr);
    unsigned long long s[D];
#pragma unroll
    for (int q = 0; q < D; ++q) {
      if (q >= Dr) {  // capacity padding: sorts last, never reaches a key
        s[q] = ~0ULL;
        continue;
      }
      if (i > r0) {
        const double2 ru = P.WU[ei + 32 * q], cu = P.WU[ej + 32 * q];
        cov[q] = fma(ru.x, cu.y, cov[q]);
        cov[q] = fma(ru.y, cu.x, cov[q]);
      }
      const double2 ri = P.WI[ei + 32 * q], ci = P.WI[ej + 32 * q];
      const double corr = fma(cov[q], ri.x * ci.x, ri.y + ci.y);  // flat convention via the halves
      s[q] = (unsigned long long)__double_as_longlong(sqrt_search(clamp0(fma(-two_m, corr, two_m)))) |
             (q >= P.n_must ? kFree : 0ULL);
    }
    sort_keys<D>(s);
    double acc = 0.0;
#pragma unroll
    for (int q = 0; q < D; ++q) {
      if (q >= Dr) break;
      acc += __longlong_as_double((long long)(s[q] & ~kFree));
      const double pk = acc * (1.0 / (double)(q + 1));
      const long long kr = live ? pack_key(pk, j, P.imask) : kNoKey;
      if (live) {
        const long long kc = pack_key(pk, i, P.imask);
        if (kc < __ldcg(&P.keys[ej + 32 * q])) red_min64(&P.keys[ej + 32 * q], kc);
      }
      const long long tr = __ldcg(&P.keys[ei + 32 * q]);
      if (__any_sync(0xffffffffu, kr < tr)) {
        const long long b = warp_min64(kr);
        if (lane == 0 && b < tr) red_min64(&P.keys[ei + 32 * q], b);
      }
    }
  }
}

// KD consecutive diagonals per lane, D admissible dims compile-time. Column
// statistics of the lane's KD columns ({df, dg}, inv and the D column
// thresholds) live in a register shift window; row statistics are broadcast
// loads. Per cell: D covariance recurrences (2 DFMA each), D distances, the
// stable sort, D prefix means and an integer filter of their high words
// against the row / column thresholds; a step where any lane passes runs the
// exact key updates.
template <int KD, int D>
__global__ void __launch_bounds__(kMWarps * 32, 2) k_mstomp_t(const MStompParams P) {
  const long long wid = (long long)blockIdx.x * kMWarps + (threadIdx.x >> 5);
  if (wid >= P.n_items) return;
  const int lane = threadIdx.x & 31;
  const MItem it = P.items[wid];
  const long long r0 = it.r0;
  const long long c0 = r0 + it.kb + (long long)lane * KD;
  const long long Lp = P.Lp, L = P.L;
  const int m = P.m;
  const double two_m = 2.0 * m;
  const unsigned long long kFree = 1ULL << 63;

  double cov[KD][D];
#pragma unroll
  for (int q = 0; q < D; ++q) {
    const double* xr = P.x + q * P.ns + r0;
    const double* xc = P.x + q * P.ns + c0;
    const double mr = P.mu[q * Lp + r0];
    double acc[KD], asum = 0.0;
#pragma unroll
    for (int d = 0; d < KD; ++d) acc[d] = 0.0;
    for (int t = 0; t < m; ++t) {
      const double a = xr[t] - mr;
      asum += a;
#pragma unroll
      for (int d = 0; d < KD; ++d) acc[d] = fma(a, xc[t + d], acc[d]);
    }
#pragma unroll
    for (int d = 0; d < KD; ++d) cov[d][q] = fma(-P.mu[q * Lp + c0 + d], asum, acc[d]);
  }
  // column window: {df, dg}, {inv, flat half} and the D column thresholds
  double2 cu[KD][D], ci[KD][D];
  int cth[KD][D];
  const int* khi_ = reinterpret_cast<const int*>(P.keys) + 1;  // hi words
#pragma unroll
  for (int d = 0; d < KD - 1; ++d) {
    const long long e = mblk(c0 + d, D);
#pragma unroll
    for (int q = 0; q < D; ++q) {
      cu[d][q] = P.WU[e + 32 * q];
      ci[d][q] = P.WI[e + 32 * q];
      cth[d][q] = __ldcg(khi_ + 2 * (e + 32 * q));
    }
  }
  for (int u = 0; u < it.nrows; u += KD) {
#pragma unroll
    for (int s = 0; s < KD; ++s) {
      const long long i = r0 + u + s;
      const int sin = (s + KD - 1) % KD;
      {
        const long long e = mblk(c0 + u + s + KD - 1, D);  // entering column
#pragma unroll
        for (int q = 0; q < D; ++q) {
          cu[sin][q] = P.WU[e + 32 * q];
          ci[sin][q] = P.WI[e + 32 * q];
          cth[sin][q] = __ldcg(khi_ + 2 * (e + 32 * q));
        }
      }
      const bool step = (u + s) != 0;
      double2 ru[D], ri[D];
      int rth[D];
      const long long ei = mblk(i, D);
#pragma unroll
      for (int q = 0; q < D; ++q) {
        ru[q] = step ? P.WU[ei + 32 * q] : make_double2(0.0, 0.0);
        ri[q] = P.WI[ei + 32 * q];
        rth[q] = __ldcg(khi_ + 2 * (ei + 32 * q));
      }
      // covariance recurrences (exact, fp64), then the fast filter in fp32:
      // the prefix means from fp32 distances (relative error below 2^-19.5:
      // 2^-20 from the truncated s, 2^-22 from the square root and the fp32
      // sums) compared with thresholds raised by kFastSlack high-word units
      // (2^-20 each), so it never skips a cell the exact test takes; a
      // row-step where any lane passes recomputes every value exactly.
      constexpr int kFastSlack = 4;
      bool fire = false;
#pragma unroll
      for (int d = 0; d < KD; ++d) {
        const int sl = (s + d) % KD;
        unsigned sf[D];
#pragma unroll
        for (int q = 0; q < D; ++q) {
          cov[d][q] = fma(ru[q].x, cu[sl][q].y, cov[d][q]);
          cov[d][q] = fma(ru[q].y, cu[sl][q].x, cov[d][q]);
          const double corr = fma(cov[d][q], ri[q].x * ci[sl][q].x, ri[q].y + ci[sl][q].y);
          sf[q] = (unsigned)__float_as_int(dist_fast(fma(-two_m, corr, two_m))) |
                  (q >= P.n_must ? 0x80000000u : 0u);
        }
        sort_u32<D>(sf);
        float acc = 0.0f;
#pragma unroll
        for (int q = 0; q < D; ++q) {
          acc += __int_as_float((int)(sf[q] & 0x7fffffffu));
          const int h = hi_of_f32(acc * (1.0f / (float)(q + 1))) - kFastSlack;
          fire |= (h <= rth[q]) | (h <= cth[sl][q]);
        }
      }
      if (P.stats && lane == 0) atomicAdd(&P.stats[0], 1ull);
      if (__any_sync(0xffffffffu, fire)) {
        if (P.stats && lane == 0) atomicAdd(&P.stats[1], 1ull);
        // exact values of the row-step (the cov recurrences above are exact)
        double pk[KD][D];
#pragma unroll
        for (int d = 0; d < KD; ++d) {
          const int sl = (s + d) % KD;
          unsigned long long sk[D];
#pragma unroll
          for (int q = 0; q < D; ++q) {
            const double corr = fma(cov[d][q], ri[q].x * ci[sl][q].x, ri[q].y + ci[sl][q].y);
            sk[q] = (unsigned long long)__double_as_longlong(sqrt_search(clamp0(fma(-two_m, corr, two_m)))) |
                    (q >= P.n_must ? kFree : 0ULL);
          }
          sort_keys<D>(sk);
          double a = 0.0;
#pragma unroll
          for (int q = 0; q < D; ++q) {
            a += __longlong_as_double((long long)(sk[q] & ~kFree));
            pk[d][q] = a * (1.0 / (double)(q + 1));
          }
        }
        long long best[D];
#pragma unroll
        for (int q = 0; q < D; ++q) best[q] = kNoKeyS;
        const bool row_ok = i < L;
#pragma unroll
        for (int d = 0; d < KD; ++d) {
          const int sl = (s + d) % KD;
          const long long j = c0 + u + s + d;
          if (row_ok && j < L) {
#pragma unroll
            for (int q = 0; q < D; ++q) {
              const double pv = pk[d][q];
              const int h = __double2hiint(pv);
              if (h <= cth[sl][q]) {
                red_min64(P.keys + mblk(j, D) + 32 * q, pack_key(pv, i, P.imask));
                cth[sl][q] = min(cth[sl][q], h);
              }
              if (h <= rth[q]) {
                const long long kk = pack_key(pv, j, P.imask);
                best[q] = kk < best[q] ? kk : best[q];
              }
            }
          }
        }
#pragma unroll
        for (int q = 0; q < D; ++q) {
          const long long b = warp_min64(best[q]);
          if (lane == 0 && b != kNoKeyS) red_min64(P.keys + ei + 32 * q, b);
        }
      }
    }
  }
}

// Keys -> exact values, index and dim_order. One warp per (output row k, i):
// exact per-dim distances at the chosen partner, the same selection, prefix
// mean. Rows k >= D repeat row D-1 with dim_order -1.
__global__ void k_mstomp_finalize(const MStompParams P, int D, int dims_out,
                                  const int* __restrict__ perm, double* mp, long long* pi,
                                  long long* dim_order) {
  const long long g = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (g >= (long long)dims_out * P.L) return;
  const int kout = (int)(g / P.L);
  const long long i = g % P.L;
  const int kk = kout < D ? kout : D - 1;
  const long long key = P.keys[mblk(i, D) + 32 * kk];
  const long long j = key >= kNoKeyS ? -1 : (key & P.imask);
  double v = INFINITY;
  long long dim = -1;
  if (j >= 0) {
    const int m = P.m;
    double dist[kMaxMDims];
    for (int q = 0; q < D; ++q) {
      const double ii = P.inv[q * P.Lp + i], ij = P.inv[q * P.Lp + j];
      double d;
      if (ii == 0.0 || ij == 0.0) {
        d = (ii == 0.0 && ij == 0.0) ? 0.0 : sqrt((double)m);
      } else {
        const double mi = P.mu[q * P.Lp + i], mj = P.mu[q * P.Lp + j];
        const double* xi = P.x + q * P.ns + i;
        const double* xj = P.x + q * P.ns + j;
        double acc = 0.0;
        for (int t = lane; t < m; t += 32) {
          const double e = __dmul_rn(xi[t] - mi, ii) - __dmul_rn(xj[t] - mj, ij);
          acc = fma(e, e, acc);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        d = sqrt(fmin((double)m * acc, 4.0 * m));
      }
      dist[q] = d;
    }
    if (lane == 0) {
      int idx[kMaxMDims];
      for (int q = 0; q < D; ++q) idx[q] = q;
      for (int part = 0; part < 2; ++part) {  // stable insertion sort per class
        const int lo = part == 0 ? 0 : P.n_must, hi = part == 0 ? P.n_must : D;
        for (int q = lo + 1; q < hi; ++q) {
          const int t = idx[q];
          int p = q - 1;
          while (p >= lo && dist[idx[p]] > dist[t]) {
            idx[p + 1] = idx[p];
            --p;
          }
          idx[p + 1] = t;
        }
      }
      double acc = 0.0;
      for (int q = 0; q <= kk; ++q) acc += dist[idx[q]];
      v = acc / (double)(kk + 1);
      dim = kout < D ? perm[idx[kk]] : -1;
    }
  }
  if (lane == 0) {
    const long long o = (long long)kout * P.L + i;
    if (mp) mp[o] = v;
    if (pi) pi[o] = j;
    if (dim_order) dim_order[o] = j >= 0 ? dim : -1;
  }
}

// ---- host side -------------------------------------------------------------------

int ceil_log2ll(long long v) {
  int b = 0;
  while ((1LL << b) < v) ++b;
  return b;
}

void sort_mitems(std::vector<MItem>& v) {
  std::stable_sort(v.begin(), v.end(), [](const MItem& a, const MItem& b) { return a.nrows > b.nrows; });
}

// Per-(device, entry point) scratch reused across calls: the i-th allocation
// of a call reuses the i-th block when it is large enough (calls are
// serialised, and every entry point allocates in a fixed order), so a repeated
// join pays no cudaMalloc / cudaFree. The stream and timing events persist too.
struct Arena {
  std::vector<void*> blk;
  std::vector<size_t> cap;
  size_t next = 0;
  cudaStream_t st = nullptr;
  cudaEvent_t ea = nullptr, eb = nullptr;
  template <class T>
  cudaError_t alloc(T** out, size_t count) {
    const size_t bytes = sizeof(T) * std::max<size_t>(count, 1);
    if (next == blk.size()) {
      blk.push_back(nullptr);
      cap.push_back(0);
    }
    if (cap[next] < bytes) {
      if (blk[next]) cudaFree(blk[next]);
      blk[next] = nullptr;
      cap[next] = 0;
      const cudaError_t e = cudaMalloc(&blk[next], bytes);
      if (e != cudaSuccess) return e;
      cap[next] = bytes;
    }
    *out = (T*)blk[next++];
    return cudaSuccess;
  }
};

std::vector<std::unique_ptr<Arena>> g_arenas;  // index: device * 2 + kind

// The arena of (device, kind), its stream and events created on first use.
mpgpu_status arena_for(int device, int kind, Arena** out) {
  const size_t slot = (size_t)device * 2 + (size_t)kind;
  if (g_arenas.size() <= slot) g_arenas.resize(slot + 1);
  if (!g_arenas[slot]) g_arenas[slot].reset(new Arena());
  Arena* A = g_arenas[slot].get();
  if (!A->st) MM_CUDA(cudaStreamCreateWithFlags(&A->st, cudaStreamNonBlocking));
  if (!A->ea) MM_CUDA(cudaEventCreate(&A->ea));
  if (!A->eb) MM_CUDA(cudaEventCreate(&A->eb));
  A->next = 0;
  *out = A;
  return MPGPU_OK;
}

std::mutex g_multi_mu;  // calls are serialised (the arenas are shared)

}  // namespace

namespace {

template <int KD, int DIMS>
void launch_simple(const SimpleParams& P, cudaStream_t st) {
  k_simple_t<KD, DIMS><<<(unsigned)((P.n_items + kMWarps - 1) / kMWarps), kMWarps * 32, 0, st>>>(P);
}

template <int KD, int T>
void launch_simple_dt(const SimpleParams& P, cudaStream_t st) {
  k_simple_dt<KD, T><<<(unsigned)((P.n_items + kMWarps - 1) / kMWarps), kMWarps * 32, 0, st>>>(P);
}

template <int KD, int DIMS, bool BLK>
void launch_simple_ring(const SimpleParams& P, cudaStream_t st) {
  const size_t smem = SRing<KD, DIMS>::kSmem;
  static bool attr = false;  // once per process (calls are serialised)
  if (!attr) {
    cudaFuncSetAttribute(k_simple_r<KD, DIMS, BLK>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  k_simple_r<KD, DIMS, BLK><<<(unsigned)((P.n_items + kMWarps - 1) / kMWarps), kMWarps * 32, smem, st>>>(P);
}

void launch_simple_generic(const SimpleParams& P, cudaStream_t st) {
  k_simple<<<(unsigned)((P.n_items + kMWarps - 1) / kMWarps), kMWarps * 32, 0, st>>>(P);
}

using SLaunch = void (*)(const SimpleParams&, cudaStream_t);

bool simple_tiled(long long dims) {
  const char* t = getenv("MPGPU_SIMPLE_TILED");  // experiments: 1 forces k_simple_dt, 0 forbids it
  if (t) return atoi(t) != 0;
  return dims > 3;  // measured crossover: the register window wins for d <= 3
}

// the shared-memory ring kernel (k_simple_r) for dims <= kRingMaxDims;
// MPGPU_SIMPLE_RING=0 falls back to the register-window / tiled kernels
// (experiments), as does an explicit MPGPU_SIMPLE_TILED=1
constexpr int kRingMaxDims = 12;
bool simple_ring(long long dims) {
  const char* t = getenv("MPGPU_SIMPLE_RING");
  if (t && atoi(t) == 0) return false;
  const char* u = getenv("MPGPU_SIMPLE_TILED");
  if (u && atoi(u) == 1) return false;
  return dims <= kRingMaxDims;
}
int simple_ring_ts(int dims) { return dims <= 3 ? 32 : 16; }  // SRing<.., dims>::TS
int simple_ring_kd(int dims) {
  const char* e = getenv("MPGPU_SIMPLE_KD");
  const int kd = e ? atoi(e) : 0;
  if (dims == 1) return (kd == 4 || kd == 8) ? kd : 4;  // measured: KD 4 beats 8 (spills)
  if (dims == 2) return (kd == 2 || kd == 4) ? kd : 4;
  return dims <= 8 ? 2 : 1;
}
template <bool BLK>
SLaunch simple_ring_pick(int dims, int kd) {
  switch (dims) {
    case 1: return kd == 8 ? launch_simple_ring<8, 1, BLK> : launch_simple_ring<4, 1, BLK>;
    case 2: return kd == 4 ? launch_simple_ring<4, 2, BLK> : launch_simple_ring<2, 2, BLK>;
    case 3: return launch_simple_ring<2, 3, BLK>;
    default: break;
  }
  if constexpr (BLK) {
    return nullptr;  // block replay is instantiated for dims <= 3 only
  } else {
    switch (dims) {
      case 4: return launch_simple_ring<2, 4, BLK>;
      case 5: return launch_simple_ring<2, 5, BLK>;
      case 6: return launch_simple_ring<2, 6, BLK>;
      case 7: return launch_simple_ring<2, 7, BLK>;
      case 8: return launch_simple_ring<2, 8, BLK>;
      case 9: return launch_simple_ring<1, 9, BLK>;
      case 10: return launch_simple_ring<1, 10, BLK>;
      case 11: return launch_simple_ring<1, 11, BLK>;
      default: return launch_simple_ring<1, 12, BLK>;
    }
  }
}
SLaunch simple_ring_launcher(int dims) {
  // branch-free blocks + replay for d = 1 (measured 4% faster), per-step votes
  // otherwise; MPGPU_SIMPLE_BLK=0/1 overrides (experiments)
  const char* e = getenv("MPGPU_SIMPLE_BLK");
  const bool blk = e ? atoi(e) == 1 : dims == 1;
  return (blk && dims <= 3) ? simple_ring_pick<true>(dims, simple_ring_kd(dims))
                            : simple_ring_pick<false>(dims, simple_ring_kd(dims));
}

SLaunch simple_launcher(int dims) {
  // diagonals per lane by register budget (128 at 2 CTAs/SM); MPGPU_SIMPLE_KD
  // overrides it for dims 1-2 (experiments)
  const char* e = getenv("MPGPU_SIMPLE_KD");
  const int kd = e ? atoi(e) : 0;
  if (simple_tiled(dims)) dims = 99;  // -> the tiled kernels below
  switch (dims) {
    case 1: return kd == 8 ? launch_simple<8, 1> : (kd == 2 ? launch_simple<2, 1> : launch_simple<4, 1>);
    case 2: return kd == 8 ? launch_simple<8, 2> : (kd == 4 ? launch_simple<4, 2> : launch_simple<2, 2>);
    case 3: return launch_simple<2, 3>;
    default: break;
  }
  const char* t = getenv("MPGPU_SIMPLE_DT");
  const std::string v = t ? t : "";
  if (v == "2x4") return launch_simple_dt<2, 4>;
  if (v == "2x8") return launch_simple_dt<2, 8>;
  if (v == "4x8") return launch_simple_dt<4, 8>;
  if (v == "1x1") return launch_simple_generic;
  if (v == "4x4") return launch_simple_dt<4, 4>;
  return launch_simple_dt<4, 8>;
}

// dims > 8: rows per item must be a multiple of the tile's T and bands are 32 KD wide
int simple_dt_kd() {
  const char* t = getenv("MPGPU_SIMPLE_DT");
  const std::string v = t ? t : "";
  return (v == "2x4" || v == "2x8") ? 2 : (v == "1x1" ? 1 : 4);
}
int simple_dt_t() {
  const char* t = getenv("MPGPU_SIMPLE_DT");
  const std::string v = t ? t : "";
  return (v == "2x4" || v == "4x4") ? 4 : (v == "1x1" ? 1 : 8);
}

int simple_kd(int dims) {
  const char* e = getenv("MPGPU_SIMPLE_KD");
  const int kd = e ? atoi(e) : 0;
  if (dims <= 2) return (kd == 8 || kd == 2 || kd == 4) ? kd : (dims == 1 ? 4 : 2);
  return 2;
}

}  // namespace

namespace {

// ---- SiMPle coarse warm start -----------------------------------------------------
// PAA of the centred data (f samples per coarse sample), zero padded to stride nsc.
__global__ void k_paa_dims(const double* __restrict__ xc, long long ns, long long nc, long long nsc,
                           int dims, int f, double* __restrict__ out) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nsc * dims) return;
  const long long q = t / nsc, I = t % nsc;
  double s = 0.0;
  if (I < nc) {
    const double* x = xc + q * ns + I * f;
    for (int u = 0; u < f; ++u) s += x[u];
    s /= f;
  }
  out[t] = s;
}

// One warp per (coarse window I of X, coarse partner): the coarse join's
// partner J of I gives the fine diagonals k = f (J - I) + delta, |delta| <= f/2,
// over the f fine rows i = f I ... f I + f - 1, one lane per diagonal: a direct
// raw dot product seeds row f I, the join's recurrence walks the rest. Values
// use the join's own formula; the cells are ordinary cells of the join,
// min-merged into the row keys (warp minimum) and column keys (only when they
// improve), so they only tighten the filter: the answer is unchanged up to the
// search's rounding, which finalize removes.
struct Exploit {
  const double* xcX; const double* xcY; long long nsX, nsY;
  const double* nrmX; const double* nrmY;
  long long LX, LY;
  const long long* ck[2];  // coarse keys of X's coarse windows (partners in Y's coarse series)
  long long Lc, imask_c;
  long long* keyX;          // fine keys of X windows (partners in Y)
  long long* keyY;          // fine keys of Y windows (partners in X)
  long long zone;           // self-join: cells with |i - j| <= zone are skipped
  bool self;                // self: keyX = right keys (k0), keyY = left keys (k1)
  int n_ck, f, m, dims;
  long long imask;
};

__global__ void k_simple_exploit(const Exploit E) {
  const long long w = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const long long I = w / E.n_ck;
  const int which = (int)(w % E.n_ck);
  if (I >= E.Lc) return;
  const long long ck = E.ck[which][I];
  if (ck == kNoKeyS) return;
  const long long J = ck & E.imask_c;
  const int f = E.f;
  const long long i0 = (long long)f * I;
  const long long j0 = (long long)f * J + lane - f / 2;  // this lane's column at row i0
  const bool act = lane <= f;
  // seed: row i0 against column j0 (windows past the end read zero padding)
  double qt = 0.0;
  if (act && j0 >= 0) {
    for (int q = 0; q < E.dims; ++q) {
      const double* a = E.xcX + q * E.nsX + i0;
      const double* c = E.xcY + q * E.nsY + j0;
      for (int t = 0; t < E.m; ++t) qt = fma(a[t], c[t], qt);
    }
  }
  // the last coarse window also covers the fine rows past f Lc
  const int rows = (int)(I == E.Lc - 1 ? E.LX - i0 : f);
  for (int r = 0; r < rows; ++r) {
    const long long i = i0 + r, j = j0 + r;
    if (i >= E.LX) break;
    if (r > 0 && act && j - 1 >= 0) {
      for (int q = 0; q < E.dims; ++q) {
        const double* a = E.xcX + q * E.nsX;
        const double* c = E.xcY + q * E.nsY;
        qt = fma(-a[i - 1], c[j - 1], qt);
        qt = fma(a[i + E.m - 1], c[j + E.m - 1], qt);
      }
    } else if (r > 0 && act && j - 1 < 0 && j >= 0) {  // first valid column: seed directly
      qt = 0.0;
      for (int q = 0; q < E.dims; ++q) {
        const double* a = E.xcX + q * E.nsX + i;
        const double* c = E.xcY + q * E.nsY + j;
        for (int t = 0; t < E.m; ++t) qt = fma(a[t], c[t], qt);
      }
    }
    bool ok = act && j >= 0 && j < E.LY;
    if (E.self) ok = ok && (j - i > E.zone || i - j > E.zone);
    long long kx = kNoKeyS;
    if (ok) {
      const double vv = fmax(fma(-2.0, qt, E.nrmX[i] + E.nrmY[j]), 0.0);
      if (!E.self || j > i) {
        kx = pack_key(vv, j, E.imask);                // row i of X, partner j
        const long long ky = pack_key(vv, i, E.imask);
        if (ky < __ldcg(&E.keyY[j])) red_min64(&E.keyY[j], ky);
      } else {                                        // self, j < i: pair (j, i)
        const long long kr = pack_key(vv, i, E.imask);  // right key of j
        if (kr < __ldcg(&E.keyX[j])) red_min64(&E.keyX[j], kr);
        const long long kl = pack_key(vv, j, E.imask);  // left key of i
        if (kl < __ldcg(&E.keyY[i])) red_min64(&E.keyY[i], kl);
      }
    }
    kx = warp_min64(kx);
    if (lane == 0 && kx != kNoKeyS && kx < __ldcg(&E.keyX[i])) red_min64(&E.keyX[i], kx);
  }
}

// One SiMPle join level on device-resident centred data: energies, ring
// vectors, keys, work items and the join launches.
struct SimpleLevel {
  bool self = true;
  long long dims = 1, m = 4, zone = 0;
  long long na = 0, nb = 0, La = 0, Lb = 0, nsa = 0, nsb = 0, Lpa = 0, Lpb = 0;
  double *xca = nullptr, *xcb = nullptr, *nra = nullptr, *nrb = nullptr;
  double2 *va = nullptr, *vb = nullptr;
  long long *k0 = nullptr, *k1 = nullptr;
  long long imask = 0;
  bool ringk = false;
  SimpleParams P{};
  long long n_probe = 0;
};

// Allocations (a fixed order per call: the arena reuses blocks by position)
// and the work items. The caller fills xca / xcb before level_prepare.
mpgpu_status level_alloc(Arena& mem, SimpleLevel& V, cudaStream_t st) {
  const long long pad = kSimplePad, dims = V.dims, m = V.m;
  V.La = V.na - m + 1;
  V.Lb = V.nb - m + 1;
  V.nsa = V.na + pad + m;
  V.nsb = V.nb + pad + m;
  V.Lpa = V.La + pad;
  V.Lpb = V.Lb + pad;
  MM_CUDA(mem.alloc(&V.xca, dims * V.nsa));
  MM_CUDA(mem.alloc(&V.nra, V.Lpa));
  if (!V.self) {
    MM_CUDA(mem.alloc(&V.xcb, dims * V.nsb));
    MM_CUDA(mem.alloc(&V.nrb, V.Lpb));
  }
  const long long Lpk1 = V.self ? V.Lpa : V.Lpb;
  MM_CUDA(mem.alloc(&V.k0, V.Lpa));
  MM_CUDA(mem.alloc(&V.k1, Lpk1));
  const int index_bits = std::max(1, ceil_log2ll(std::max(V.La, V.Lb)));
  V.imask = (1LL << index_bits) - 1;

  const bool tiled = simple_tiled(dims);  // k_simple_dt (dims outermost)
  V.ringk = simple_ring(dims);           // k_simple_r (shared-memory ring)
  const int KD = V.ringk ? simple_ring_kd((int)dims) : (tiled ? simple_dt_kd() : simple_kd((int)dims));
  const int TR = V.ringk ? simple_ring_ts((int)dims) : (tiled ? simple_dt_t() : KD);  // rows per item: a multiple of this
  const bool generic = tiled && KD == 1 && TR == 1;
  const int band = 32 * KD;
  std::vector<MItem> items;
  const long long seg = std::max<long long>(1024, 8 * m);
  auto build = [&](int pass, long long klo, long long khi, long long LR, long long LC) {
    for (long long kb = klo; kb < khi; kb += band) {
      const long long rows = std::min(LR, LC - kb);
      for (long long r0 = 0; r0 < rows; r0 += seg) {
        long long nr = std::min(seg, rows - r0);
        if (!generic) nr = (nr + TR - 1) / TR * TR;  // whole step groups (padding covers the tail)
        items.push_back(MItem{kb, r0, (int)nr, pass});
      }
    }
  };
  SimpleParams& P = V.P;
  P = SimpleParams{};
  P.dims = (int)dims;
  P.m = (int)m;
  P.imask = V.imask;
  if (V.ringk) {
    MM_CUDA(mem.alloc(&V.va, dims * V.Lpa));
    if (!V.self) MM_CUDA(mem.alloc(&V.vb, dims * V.Lpb));
  }
  RawSeries RA{V.xca, V.nra, V.na, V.nsa, V.La, V.va, V.Lpa};
  RawSeries RB{V.xcb, V.nrb, V.nb, V.nsb, V.Lb, V.vb, V.Lpb};
  if (V.self) {
    if (V.zone + 1 < V.La) build(0, V.zone + 1, V.La, V.La, V.La);
    P.pass[0] = SimplePass{RA, RA, V.zone + 1, V.La, V.k0, V.k1};
  } else {
    // pass 0: rows = B windows, columns = A windows (k >= 0); pass 1: rows = A, columns = B (k >= 1)
    build(0, 0, V.La, V.Lb, V.La);
    if (V.Lb > 1) build(1, 1, V.Lb, V.La, V.Lb);
    P.pass[0] = SimplePass{RB, RA, 0, V.La, V.k1, V.k0};
    P.pass[1] = SimplePass{RA, RB, 1, V.Lb, V.k0, V.k1};
  }
  sort_mitems(items);
  // Optional probe launch (MPGPU_SIMPLE_PROBE=P > 1, experiments): every P-th
  // band first, as its own launch, then the rest.
  V.n_probe = 0;
  if (V.ringk) {
    const char* e = getenv("MPGPU_SIMPLE_PROBE");
    const long long kProbe = e ? atoll(e) : 1;
    if (kProbe > 1) {
      auto mid = std::stable_partition(items.begin(), items.end(), [&](const MItem& it) {
        return ((it.kb - (it.pass == 0 ? P.pass[0].klo : P.pass[1].klo)) / band) % kProbe == 0;
      });
      V.n_probe = (long long)(mid - items.begin());
    }
  }
  MItem* d_items = nullptr;
  MM_CUDA(mem.alloc(&d_items, items.size()));
  if (!items.empty())
    MM_CUDA(cudaMemcpyAsync(d_items, items.data(), sizeof(MItem) * items.size(),
                            cudaMemcpyHostToDevice, st));
  P.items = d_items;
  P.n_items = (long long)items.size();
  return MPGPU_OK;
}

// energies, ring vectors and empty keys (xca / xcb already filled)
void level_prepare(const SimpleLevel& V, cudaStream_t st) {
  const int bs = 256;
  const int dims = (int)V.dims, m = (int)V.m;
  k_raw_energy<<<(unsigned)((V.Lpa + bs - 1) / bs), bs, 0, st>>>(V.xca, V.nsa, V.La, V.Lpa, dims, m, V.nra);
  if (!V.self)
    k_raw_energy<<<(unsigned)((V.Lpb + bs - 1) / bs), bs, 0, st>>>(V.xcb, V.nsb, V.Lb, V.Lpb, dims, m, V.nrb);
  if (V.ringk) {
    k_build_v<<<(unsigned)((V.dims * V.Lpa + bs - 1) / bs), bs, 0, st>>>(V.xca, V.nsa, V.La, V.Lpa, dims, m, V.va);
    if (!V.self)
      k_build_v<<<(unsigned)((V.dims * V.Lpb + bs - 1) / bs), bs, 0, st>>>(V.xcb, V.nsb, V.Lb, V.Lpb, dims, m, V.vb);
  }
  const long long Lk1 = V.self ? V.La : V.Lb, Lpk1 = V.self ? V.Lpa : V.Lpb;
  k_fill_val<<<(unsigned)((V.Lpa + bs - 1) / bs), bs, 0, st>>>(V.k0, V.La, V.Lpa, kNoKeyS, kPadKey);
  k_fill_val<<<(unsigned)((Lpk1 + bs - 1) / bs), bs, 0, st>>>(V.k1, Lk1, Lpk1, kNoKeyS, kPadKey);
}

void level_run(const SimpleLevel& V, cudaStream_t st) {
  const SimpleParams& P = V.P;
  if (P.n_items <= 0) return;
  const SLaunch launch = V.ringk ? simple_ring_launcher((int)V.dims) : simple_launcher((int)V.dims);
  if (V.n_probe > 0 && V.n_probe < P.n_items) {
    SimpleParams Q = P;
    Q.n_items = V.n_probe;
    launch(Q, st);
    Q.items = P.items + V.n_probe;
    Q.n_items = P.n_items - V.n_probe;
    launch(Q, st);
  } else {
    launch(P, st);
  }
}

// Coarse warm start (the SiMPle analogue of k_join's K2b): join the series
// averaged in blocks of f samples (window m / f) and seed the fine keys with
// the fine cells around every coarse match. Off for short windows / small joins.
long long simple_coarse_factor(const SimpleLevel& F) {
  const char* e = getenv("MPGPU_SIMPLE_COARSE");
  if (e && atoi(e) == 0) return 0;
  if (!F.ringk || F.m < 64) return 0;
  const bool forced = e && atoi(e) == 1;  // tests: on whatever the size
  if (!forced && (double)F.La * (double)(F.self ? F.La : F.Lb) < 4e8) return 0;
  return std::min<long long>(16, F.m / 16);
}

}  // namespace

extern "C" {

mpgpu_status mpgpu_simple_join(const mpgpu_simple_args* A) {
  if (!A || !A->a) return set_error(MPGPU_EPARAM, "null arguments");
  const bool self = A->b == nullptr;
  const long long dims = A->dims, m = A->window;
  if (dims < 1) return set_error(MPGPU_EPARAM, "multivariate series needs at least one dimension");
  if (m < 4) return set_error(MPGPU_EPARAM, "window below minimum 4");
  if (m > A->n_a || (!self && m > A->n_b)) return set_error(MPGPU_EPARAM, "series shorter than the window");
  if (self && A->zone < 0) return set_error(MPGPU_EPARAM, "negative exclusion zone");
  std::lock_guard<std::mutex> lk(g_multi_mu);
  MM_CUDA(cudaSetDevice(A->device));
  Arena* ar = nullptr;
  if (mpgpu_status e = arena_for(A->device, 0, &ar); e != MPGPU_OK) return e;
  cudaStream_t st = ar->st;
  Arena& mem = *ar;

  const long long na = A->n_a, nb = self ? na : A->n_b;
  if (std::max(na, nb) - m + 1 >= (1LL << 31)) return set_error(MPGPU_EUNSUPPORTED, "profile longer than 2^31");
  double *xa, *xb = nullptr, *shift;
  MM_CUDA(mem.alloc(&xa, dims * na));
  MM_CUDA(mem.alloc(&shift, dims));
  MM_CUDA(cudaMemcpyAsync(xa, A->a, sizeof(double) * dims * na, cudaMemcpyHostToDevice, st));
  if (!self) {
    MM_CUDA(mem.alloc(&xb, dims * nb));
    MM_CUDA(cudaMemcpyAsync(xb, A->b, sizeof(double) * dims * nb, cudaMemcpyHostToDevice, st));
  }
  // shared per-dim shift: the mean of A's dimension (host, from the caller's buffer)
  std::vector<double> sh(dims);
  for (long long d = 0; d < dims; ++d) {
    double sm = 0.0;
    for (long long t = 0; t < na; ++t) sm += A->a[d * na + t];
    sh[d] = sm / (double)na;
  }
  MM_CUDA(cudaMemcpyAsync(shift, sh.data(), sizeof(double) * dims, cudaMemcpyHostToDevice, st));

  // the fine level; self: k0 = right keys (row candidates), k1 = left keys
  // (column candidates); AB: k0 = A keys, k1 = B keys
  SimpleLevel F;
  F.self = self;
  F.dims = dims;
  F.m = m;
  F.zone = self ? A->zone : 0;
  F.na = na;
  F.nb = nb;
  if (mpgpu_status e = level_alloc(mem, F, st); e != MPGPU_OK) return e;
  const long long La = F.La, Lb = F.Lb;
  // the coarse level (warm start), when enabled
  const long long f = simple_coarse_factor(F);
  SimpleLevel Cz;
  if (f > 0) {
    Cz.self = self;
    Cz.dims = dims;
    Cz.m = m / f;
    Cz.zone = self ? (F.zone + f - 1) / f : 0;
    Cz.na = na / f;
    Cz.nb = nb / f;
    if (mpgpu_status e = level_alloc(mem, Cz, st); e != MPGPU_OK) return e;
  }

  MM_CUDA(cudaEventRecord(ar->ea, st));
  const int bs = 256;
  k_center<<<(unsigned)((dims * F.nsa + bs - 1) / bs), bs, 0, st>>>(xa, na, F.nsa, (int)dims, shift, F.xca);
  if (!self)
    k_center<<<(unsigned)((dims * F.nsb + bs - 1) / bs), bs, 0, st>>>(xb, nb, F.nsb, (int)dims, shift, F.xcb);
  level_prepare(F, st);
  unsigned long long* d_stats = nullptr;
  if (getenv("MPGPU_STATS")) {
    MM_CUDA(mem.alloc(&d_stats, 4));
    MM_CUDA(cudaMemsetAsync(d_stats, 0, 32, st));
  }
  if (f > 0) {
    k_paa_dims<<<(unsigned)((dims * Cz.nsa + bs - 1) / bs), bs, 0, st>>>(F.xca, F.nsa, Cz.na, Cz.nsa,
                                                                        (int)dims, (int)f, Cz.xca);
    if (!self)
      k_paa_dims<<<(unsigned)((dims * Cz.nsb + bs - 1) / bs), bs, 0, st>>>(F.xcb, F.nsb, Cz.nb, Cz.nsb,
                                                                          (int)dims, (int)f, Cz.xcb);
    level_prepare(Cz, st);
    level_run(Cz, st);
    // exploit: fine rows of A against the coarse partners (self: right and
    // left coarse keys; AB: A's coarse keys), and B's rows for an AB-join
    Exploit E{};
    E.f = (int)f;
    E.m = (int)m;
    E.dims = (int)dims;
    E.imask = F.imask;
    E.imask_c = Cz.imask;
    E.zone = F.zone;
    E.self = self;
    E.xcX = F.xca;
    E.nsX = F.nsa;
    E.nrmX = F.nra;
    E.LX = La;
    E.Lc = Cz.La;
    if (self) {
      E.xcY = F.xca;
      E.nsY = F.nsa;
      E.nrmY = F.nra;
      E.LY = La;
      E.ck[0] = Cz.k0;
      E.ck[1] = Cz.k1;
      E.n_ck = 2;
      E.keyX = F.k0;
      E.keyY = F.k1;
    } else {
      E.xcY = F.xcb;
      E.nsY = F.nsb;
      E.nrmY = F.nrb;
      E.LY = Lb;
      E.ck[0] = Cz.k0;
      E.n_ck = 1;
      E.keyX = F.k0;
      E.keyY = F.k1;
    }
    if (Cz.La > 0) {
      const long long warps = Cz.La * E.n_ck;
      k_simple_exploit<<<(unsigned)((warps * 32 + bs - 1) / bs), bs, 0, st>>>(E);
    }
    if (!self && Cz.Lb > 0) {
      Exploit G = E;
      G.xcX = F.xcb; G.nsX = F.nsb; G.nrmX = F.nrb; G.LX = Lb; G.Lc = Cz.Lb;
      G.xcY = F.xca; G.nsY = F.nsa; G.nrmY = F.nra; G.LY = La;
      G.ck[0] = Cz.k1;
      G.keyX = F.k1;
      G.keyY = F.k0;
      k_simple_exploit<<<(unsigned)((Cz.Lb * 32 + bs - 1) / bs), bs, 0, st>>>(G);
    }
  }
  F.P.stats = d_stats;
  level_run(F, st);
  if (getenv("MPGPU_EXPERIMENT_TWICE") && F.P.n_items > 0) {  // experiments: a pass against final keys
    if (d_stats) MM_CUDA(cudaMemsetAsync(d_stats, 0, 32, st));
    level_run(F, st);
  }
  if (d_stats) {
    unsigned long long h[4];
    MM_CUDA(cudaMemcpyAsync(h, d_stats, 32, cudaMemcpyDeviceToHost, st));
    MM_CUDA(cudaStreamSynchronize(st));
    fprintf(stderr, "simple stats: steps %llu slow steps %llu colRED %llu rowRED %llu replayed blocks %llu (coarse f=%lld)\n",
            h[0] & ((1ull << 40) - 1), h[1], h[2], h[3], h[0] >> 40, f);
  }
  const unsigned fa = (unsigned)((La * 32 + bs - 1) / bs);
  MM_CUDA(cudaGetLastError());
  // outputs land in device scratch, then host
  double *omp_a, *omp_b = nullptr;
  long long *opi_a, *ol = nullptr, *orr = nullptr, *opi_b = nullptr;
  MM_CUDA(mem.alloc(&omp_a, La));
  MM_CUDA(mem.alloc(&opi_a, La));
  if (self) {
    MM_CUDA(mem.alloc(&ol, La));
    MM_CUDA(mem.alloc(&orr, La));
    k_simple_finalize<<<fa, bs, 0, st>>>(xa, na, La, xa, na, F.k0, F.k1, (int)dims, (int)m, F.imask,
                                         omp_a, opi_a, ol, orr);
  } else {
    MM_CUDA(mem.alloc(&omp_b, Lb));
    MM_CUDA(mem.alloc(&opi_b, Lb));
    k_simple_finalize<<<fa, bs, 0, st>>>(xa, na, La, xb, nb, F.k0, nullptr, (int)dims, (int)m,
                                         F.imask, omp_a, opi_a, nullptr, nullptr);
    k_simple_finalize<<<(unsigned)((Lb * 32 + bs - 1) / bs), bs, 0, st>>>(
        xb, nb, Lb, xa, na, F.k1, nullptr, (int)dims, (int)m, F.imask, omp_b, opi_b, nullptr, nullptr);
  }
  MM_CUDA(cudaGetLastError());
  MM_CUDA(cudaEventRecord(ar->eb, st));
  if (A->mp_a) MM_CUDA(cudaMemcpyAsync(A->mp_a, omp_a, sizeof(double) * La, cudaMemcpyDeviceToHost, st));
  if (A->pi_a) MM_CUDA(cudaMemcpyAsync(A->pi_a, opi_a, sizeof(long long) * La, cudaMemcpyDeviceToHost, st));
  if (self && A->left_a)
    MM_CUDA(cudaMemcpyAsync(A->left_a, ol, sizeof(long long) * La, cudaMemcpyDeviceToHost, st));
  if (self && A->right_a)
    MM_CUDA(cudaMemcpyAsync(A->right_a, orr, sizeof(long long) * La, cudaMemcpyDeviceToHost, st));
  if (!self && A->mp_b)
    MM_CUDA(cudaMemcpyAsync(A->mp_b, omp_b, sizeof(double) * Lb, cudaMemcpyDeviceToHost, st));
  if (!self && A->pi_b)
    MM_CUDA(cudaMemcpyAsync(A->pi_b, opi_b, sizeof(long long) * Lb, cudaMemcpyDeviceToHost, st));
  MM_CUDA(cudaStreamSynchronize(st));
  if (A->kernel_ms) {
    float ms = 0.f;
    MM_CUDA(cudaEventElapsedTime(&ms, ar->ea, ar->eb));
    *A->kernel_ms = ms;
  }
  return MPGPU_OK;
}

}  // extern "C"

namespace {

template <int KD, int D>
void launch_mstomp_t(const MStompParams& P, cudaStream_t st) {
  k_mstomp_t<KD, D><<<(unsigned)((P.n_items + kMWarps - 1) / kMWarps), kMWarps * 32, 0, st>>>(P);
}

template <int D>
void launch_mstomp(const MStompParams& P, cudaStream_t st) {
  k_mstomp<D><<<(unsigned)((P.n_items + kMWarps - 1) / kMWarps), kMWarps * 32, 0, st>>>(P);
}

using MLaunch = void (*)(const MStompParams&, cudaStream_t);

// diagonals per lane by register budget (the generic kernels above 8 dims walk
// one); MPGPU_MSTOMP_KD overrides it for D <= 4 (experiments)
int mstomp_kd(int D) {
  const char* e = getenv("MPGPU_MSTOMP_KD");
  const int kd = e ? atoi(e) : 0;
  if (D <= 4 && (kd == 1 || kd == 2 || kd == 4)) return kd;
  return D <= 3 ? 2 : 1;  // measured (tools/bench_multi.py): KD = 4 spills from D = 2 on
}

template <int D>
MLaunch mstomp_pick(int kd) {
  return kd == 4 ? launch_mstomp_t<4, D> : (kd == 2 ? launch_mstomp_t<2, D> : launch_mstomp_t<1, D>);
}

MLaunch mstomp_launcher(int D) {
  const int kd = mstomp_kd(D);
  switch (D) {
    case 1: return mstomp_pick<1>(kd);
    case 2: return mstomp_pick<2>(kd);
    case 3: return mstomp_pick<3>(kd);
    case 4: return mstomp_pick<4>(kd);
    case 5: return launch_mstomp_t<1, 5>;
    case 6: return launch_mstomp_t<1, 6>;
    case 7: return launch_mstomp_t<1, 7>;
    case 8: return launch_mstomp_t<1, 8>;
    default: break;
  }
  if (D <= 12) return launch_mstomp<12>;
  if (D <= 16) return launch_mstomp<16>;
  return launch_mstomp<32>;
}

// One admissible dimension: row 0 of the multidimensional profile is the
// univariate z-normalised self-join of that dimension (the per-dim distance,
// flat convention, exclusion zone and smallest-index ties are the same), so it
// runs on k_join (mpgpu_join) instead of the general kernel; rows k >= 1 repeat
// it with dim_order -1 (an exhausted selection). MPGPU_MSTOMP_K3=0 keeps the
// general kernel (experiments, tests).
bool mstomp_univariate() {
  const char* e = getenv("MPGPU_MSTOMP_K3");
  return !(e && atoi(e) == 0);
}

mpgpu_status mstomp_one_dim(const mpgpu_mstomp_args* A, int dim) {
  const long long dims = A->dims, n = A->n, L = n - A->window + 1;
  std::vector<double> mp(A->mp ? 0 : L);
  std::vector<long long> pi(A->pi ? 0 : L);
  double* mp0 = A->mp ? A->mp : mp.data();
  long long* pi0 = A->pi ? (long long*)A->pi : pi.data();
  const int32_t dev = A->device;
  mpgpu_join_args J{};
  J.a = A->x + (size_t)dim * n;
  J.n_a = n;
  J.window = A->window;
  J.zone = A->zone;
  J.n_gpus = 1;
  J.devices = &dev;
  J.mp_a = mp0;
  J.pi_a = (int64_t*)pi0;
  double kms = 0.0;
  if (mpgpu_status e = mpgpu_join_timed(&J, &kms, nullptr); e != MPGPU_OK) return e;
  for (long long k = 1; k < dims; ++k) {
    if (A->mp) std::memcpy(A->mp + k * L, mp0, sizeof(double) * L);
    if (A->pi) std::memcpy(A->pi + k * L, pi0, sizeof(long long) * L);
  }
  if (A->dim_order) {
    for (long long i = 0; i < L; ++i) A->dim_order[i] = pi0[i] >= 0 ? dim : -1;
    for (long long k = 1; k < dims; ++k)
      std::fill(A->dim_order + k * L, A->dim_order + (k + 1) * L, (int64_t)-1);
  }
  if (A->kernel_ms) *A->kernel_ms = kms;
  return MPGPU_OK;
}

}  // namespace

extern "C" {

mpgpu_status mpgpu_mstomp(const mpgpu_mstomp_args* A) {
  if (!A || !A->x) return set_error(MPGPU_EPARAM, "null arguments");
  const long long dims = A->dims, n = A->n, m = A->window;
  if (dims < 1) return set_error(MPGPU_EPARAM, "multivariate series needs at least one dimension");
  if (m < 4) return set_error(MPGPU_EPARAM, "window below minimum 4");
  if (m > n) return set_error(MPGPU_EPARAM, "series shorter than the window");
  if (A->zone < 0) return set_error(MPGPU_EPARAM, "negative exclusion zone");
  if ((A->n_must > 0 && !A->must_dims) || (A->n_exc > 0 && !A->exc_dims) || A->n_must < 0 ||
      A->n_exc < 0)
    return set_error(MPGPU_EPARAM, "null must / exc dimension list");
  // admissible order: must dims (ascending), then free dims (ascending); exc dropped
  std::vector<int> tag(dims, 0);
  for (long long q = 0; q < A->n_must; ++q) {
    const long long d = A->must_dims[q];
    if (d < 0 || d >= dims) return set_error(MPGPU_EPARAM, "must dimension out of range");
    if (tag[d]) return set_error(MPGPU_EPARAM, "repeated must dimension");
    tag[d] = 1;
  }
  for (long long q = 0; q < A->n_exc; ++q) {
    const long long d = A->exc_dims[q];
    if (d < 0 || d >= dims) return set_error(MPGPU_EPARAM, "excluded dimension out of range");
    if (tag[d] == 1) return set_error(MPGPU_EPARAM, "dimension both required and excluded");
    if (tag[d] == 2) return set_error(MPGPU_EPARAM, "repeated excluded dimension");
    tag[d] = 2;
  }
  std::vector<int> perm;
  for (long long d = 0; d < dims; ++d) if (tag[d] == 1) perm.push_back((int)d);
  for (long long d = 0; d < dims; ++d) if (tag[d] == 0) perm.push_back((int)d);
  const int D = (int)perm.size();
  if (D == 0) return set_error(MPGPU_EPARAM, "every dimension is excluded");
  if (D > kMaxMDims) return set_error(MPGPU_EUNSUPPORTED, "more than 32 admissible dimensions");
  const int n_must = (int)A->n_must;
  if (D == 1 && mstomp_univariate()) return mstomp_one_dim(A, perm[0]);
  std::lock_guard<std::mutex> lk(g_multi_mu);
  MM_CUDA(cudaSetDevice(A->device));
  Arena* ar = nullptr;
  if (mpgpu_status e = arena_for(A->device, 1, &ar); e != MPGPU_OK) return e;
  cudaStream_t st = ar->st;
  Arena& mem = *ar;

  const long long L = n - m + 1, pad = mpgpu_internal::stats_pad(), Lp = L + pad;
  const long long ns = n + pad;
  if (L >= (1LL << 31)) return set_error(MPGPU_EUNSUPPORTED, "profile longer than 2^31");
  double *x, *mu, *inv, *omp;
  double2* U;
  long long *keys, *opi, *odo;
  int* dperm;
  MM_CUDA(mem.alloc(&x, (size_t)D * ns));
  MM_CUDA(mem.alloc(&mu, (size_t)D * Lp));
  MM_CUDA(mem.alloc(&inv, (size_t)D * Lp));
  MM_CUDA(mem.alloc(&U, (size_t)D * Lp));
  const long long Lb = (Lp + 31) / 32 * 32;  // blocked arrays: whole 32-window blocks
  MM_CUDA(mem.alloc(&keys, (size_t)D * Lb));
  double2 *WU = nullptr, *WI = nullptr;
  MM_CUDA(mem.alloc(&WU, (size_t)D * Lb));
  MM_CUDA(mem.alloc(&WI, (size_t)D * Lb));
  MM_CUDA(mem.alloc(&omp, (size_t)dims * L));
  MM_CUDA(mem.alloc(&opi, (size_t)dims * L));
  MM_CUDA(mem.alloc(&odo, (size_t)dims * L));
  MM_CUDA(mem.alloc(&dperm, D));
  MM_CUDA(cudaMemsetAsync(x, 0, sizeof(double) * D * ns, st));
  MM_CUDA(cudaMemsetAsync(mu, 0, sizeof(double) * D * Lp, st));
  for (int q = 0; q < D; ++q)
    MM_CUDA(cudaMemcpyAsync(x + (size_t)q * ns, A->x + (size_t)perm[q] * n, sizeof(double) * n,
                            cudaMemcpyHostToDevice, st));
  MM_CUDA(cudaMemcpyAsync(dperm, perm.data(), sizeof(int) * D, cudaMemcpyHostToDevice, st));
  const int index_bits = std::max(1, ceil_log2ll(L));
  const long long imask = (1LL << index_bits) - 1;
  const int KD = mstomp_kd(D);
  std::vector<MItem> items;
  if (A->zone + 1 < L) {
    const long long band = 32LL * KD, seg = std::max<long long>(1024, 8 * m);
    for (long long kb = A->zone + 1; kb < L; kb += band) {
      const long long rows = L - kb;
      for (long long r0 = 0; r0 < rows; r0 += seg) {
        long long nr = std::min(seg, rows - r0);
        nr = (nr + KD - 1) / KD * KD;  // whole KD-step groups (padding covers the tail)
        items.push_back(MItem{kb, r0, (int)nr, 0});
      }
    }
  }
  sort_mitems(items);
  MItem* d_items = nullptr;
  MM_CUDA(mem.alloc(&d_items, items.size()));
  if (!items.empty())
    MM_CUDA(cudaMemcpyAsync(d_items, items.data(), sizeof(MItem) * items.size(),
                            cudaMemcpyHostToDevice, st));

  MStompParams P{};
  P.x = x; P.mu = mu; P.inv = inv; P.U = U; P.WU = WU; P.WI = WI;
  P.n = n; P.ns = ns; P.L = L; P.Lp = Lp; P.khi = L;
  P.keys = keys; P.items = d_items; P.n_items = (long long)items.size();
  P.m = (int)m; P.n_must = n_must; P.D = D; P.imask = imask;

  MM_CUDA(cudaEventRecord(ar->ea, st));
  for (int q = 0; q < D; ++q)
    MM_CUDA(mpgpu_internal::series_stats(x + (size_t)q * ns, n, (int)m, mu + (size_t)q * Lp,
                                         inv + (size_t)q * Lp, U + (size_t)q * Lp, nullptr, st));
  const int bs = 256;
  k_build_w<<<(unsigned)((Lb * D + bs - 1) / bs), bs, 0, st>>>(U, inv, L, Lp, Lb, D, WU, WI, keys);
  MM_CUDA(cudaGetLastError());
  unsigned long long* d_stats = nullptr;
  if (getenv("MPGPU_STATS")) {
    MM_CUDA(mem.alloc(&d_stats, 2));
    MM_CUDA(cudaMemsetAsync(d_stats, 0, 16, st));
    P.stats = d_stats;
  }
  if (P.n_items > 0) mstomp_launcher(D)(P, st);
  if (d_stats) {
    unsigned long long h[2];
    MM_CUDA(cudaMemcpyAsync(h, d_stats, 16, cudaMemcpyDeviceToHost, st));
    MM_CUDA(cudaStreamSynchronize(st));
    fprintf(stderr, "mstomp stats: warp row-steps %llu exact row-steps %llu (%.2f%%)\n", h[0], h[1],
            100.0 * (double)h[1] / (double)(h[0] ? h[0] : 1));
  }
  if (P.n_items > 0 && getenv("MPGPU_EXPERIMENT_TWICE")) mstomp_launcher(D)(P, st);  // vs final keys
  MM_CUDA(cudaGetLastError());
  const long long outs = (long long)dims * L;
  k_mstomp_finalize<<<(unsigned)((outs * 32 + bs - 1) / bs), bs, 0, st>>>(P, D, (int)dims, dperm,
                                                                         omp, opi, odo);
  MM_CUDA(cudaGetLastError());
  MM_CUDA(cudaEventRecord(ar->eb, st));
  if (A->mp) MM_CUDA(cudaMemcpyAsync(A->mp, omp, sizeof(double) * outs, cudaMemcpyDeviceToHost, st));
  if (A->pi) MM_CUDA(cudaMemcpyAsync(A->pi, opi, sizeof(long long) * outs, cudaMemcpyDeviceToHost, st));
  if (A->dim_order)
    MM_CUDA(cudaMemcpyAsync(A->dim_order, odo, sizeof(long long) * outs, cudaMemcpyDeviceToHost, st));
  MM_CUDA(cudaStreamSynchronize(st));
  if (A->kernel_ms) {
    float ms = 0.f;
    MM_CUDA(cudaEventElapsedTime(&ms, ar->ea, ar->eb));
    *A->kernel_ms = ms;
  }
  return MPGPU_OK;
}

}  // extern "C"
