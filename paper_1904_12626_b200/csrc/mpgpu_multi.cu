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
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "mpgpu_internal.h"
#include "mprof_gpu.h"

namespace {

using mpgpu_internal::set_error;

constexpr int kMWarps = 8;                      // warps per CTA
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

// sqrt for the search (s >= 0): MUFU reciprocal square root + one Newton step
// (relative error ~1e-13; the reported values are recomputed exactly).
__device__ __forceinline__ double sqrt_search(double s) {
  const double s2 = fmax(s, 1e-300);
  double y;
  asm("rsqrt.approx.f64 %0, %1;" : "=d"(y) : "d"(s2));
  const double h = 0.5 * s2;
  const double e = fma(-h * y, y, 0.5);
  y = fma(y, e, y);
  return s * y;
}

// ---- SiMPle ------------------------------------------------------------------

struct RawSeries {
  const double* xc;   // dims x n, centred per dim (shared shift with the partner series)
  const double* nrm;  // L: sum over dims of the centred window energies
  long long n, L;
};
struct SimplePass {
  RawSeries R, C;
  long long klo, khi;  // diagonals [klo, khi): cells (i, i + k)
  long long* keyR;
  long long* keyC;
};
struct SimpleParams {
  SimplePass pass[2];
  const MItem* items;
  long long n_items;
  int dims, m;
  long long imask;
};

__global__ void __launch_bounds__(kMWarps * 32) k_simple(const SimpleParams P) {
  const long long wid = (long long)blockIdx.x * kMWarps + (threadIdx.x >> 5);
  if (wid >= P.n_items) return;
  const int lane = threadIdx.x & 31;
  const MItem it = P.items[wid];
  const SimplePass& S = P.pass[it.pass];
  const long long k = it.kb + lane;
  const long long r0 = it.r0;
  long long rend = r0 + it.nrows;
  rend = min(rend, min(S.R.L, S.C.L - k));
  if (k >= S.khi || rend < r0) rend = r0;
  const int m = P.m, dims = P.dims;
  const long long nR = S.R.n, nC = S.C.n;

  // seed: QT(r0, r0 + k) by a direct dot product over all dims
  double qt = 0.0;
  if (r0 < rend) {
    for (int d = 0; d < dims; ++d) {
      const double* xr = S.R.xc + d * nR + r0;
      const double* xc = S.C.xc + d * nC + r0 + k;
      for (int t = 0; t < m; ++t) qt = fma(xr[t], xc[t], qt);
    }
  }
  const long long rmax = __reduce_max_sync(0xffffffffu, (unsigned)(rend - r0)) + r0;
  for (long long i = r0; i < rmax; ++i) {
    const bool live = i < rend;
    const long long j = i + k;
    long long kr = kNoKey;
    if (live) {
      if (i > r0) {
        for (int d = 0; d < dims; ++d) {
          const double* xr = S.R.xc + d * nR;
          const double* xc = S.C.xc + d * nC;
          qt = fma(-xr[i - 1], xc[j - 1], qt);
          qt = fma(xr[i + m - 1], xc[j + m - 1], qt);
        }
      }
      const double e = S.R.nrm[i] + S.C.nrm[j];
      double v = fma(-2.0, qt, e);
      v = v <= kRawSnap * e ? 0.0 : v;  // also clamps negatives
      kr = pack_key(v, j, P.imask);
      const long long kc = pack_key(v, i, P.imask);
      if (kc < S.keyC[j]) red_min64(&S.keyC[j], kc);
    }
    const long long tr = S.keyR[min(i, S.R.L - 1)];
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
  const long long b = k1 ? k1[i] : kNoKey;
  const long long best = a < b ? a : b;
  const long long bi = best == kNoKey ? -1 : (best & imask);
  double v = INFINITY;
  if (bi >= 0) v = warp_raw_exact(X, nx, i, Y, ny, bi, dims, m, lane);
  if (lane == 0) {
    if (mp) mp[i] = v;
    if (pi) pi[i] = bi;
    // self: k0 = right keys (partners j > i), k1 = left keys (partners j < i)
    if (right) right[i] = a == kNoKey ? -1 : (a & imask);
    if (left) left[i] = b == kNoKey ? -1 : (b & imask);
  }
}

__global__ void k_fill(long long* k, long long len) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < len) k[i] = kNoKey;
}

// per-dim centring by a shared shift (distances are shift-invariant) and the
// summed centred window energies (two passes per window, exact)
__global__ void k_center(const double* __restrict__ x, long long n, int dims,
                         const double* __restrict__ shift, double* __restrict__ xc) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n * dims) return;
  xc[t] = x[t] - shift[t / n];
}

__global__ void k_raw_energy(const double* __restrict__ xc, long long n, long long L, int dims,
                             int m, double* __restrict__ nrm) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= L) return;
  double s = 0.0;
  for (int d = 0; d < dims; ++d) {
    const double* w = xc + d * n + i;
    for (int t = 0; t < m; ++t) s = fma(w[t], w[t], s);
  }
  nrm[i] = s;
}

// ---- mSTOMP --------------------------------------------------------------------

struct MStompParams {
  const double* x;    // D x n (admissible dims, must first)
  const double* mu;   // D x L
  const double* inv;  // D x Lp (0: flat / padding)
  const double2* U;   // D x Lp
  long long n, L, Lp;
  long long khi;      // diagonals [klo, khi) = [zone + 1, L)
  long long* keys;    // D x L
  const MItem* items;
  long long n_items;
  int m, n_must;
  int D;              // admissible dims (<= the kernel's capacity)
  long long imask;
};

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
  const double two_m = 2.0 * m, four_m = 4.0 * m, dm = (double)m;

  double cov[D];
#pragma unroll
  for (int q = 0; q < D; ++q) {
    cov[q] = 0.0;
    if (r0 < rend && q < P.D) {
      const double* xr = P.x + q * P.n + r0;
      const double* xc = P.x + q * P.n + r0 + k;
      const double mr = P.mu[q * P.L + r0], mc = P.mu[q * P.L + r0 + k];
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
  for (long long i = r0; i < rmax; ++i) {
    const bool live = i < rend;
    const long long j = live ? i + k : i;  // dead lanes read a valid column
    unsigned long long s[D];
#pragma unroll
    for (int q = 0; q < D; ++q) {
      if (q >= P.D) {  // capacity padding: sorts last, never reaches a key
        s[q] = ~0ULL;
        continue;
      }
      const long long oi = q * P.Lp + i, oj = q * P.Lp + j;
      if (i > r0) {
        const double2 ru = P.U[oi], cu = P.U[oj];
        cov[q] = fma(ru.x, cu.y, cov[q]);
        cov[q] = fma(ru.y, cu.x, cov[q]);
      }
      const double ri = P.inv[oi], ci = P.inv[oj];
      double v = fma(-two_m, cov[q] * (ri * ci), two_m);
      v = fmin(fmax(v, 0.0), four_m);
      if (ri == 0.0 || ci == 0.0) v = (ri == 0.0 && ci == 0.0) ? 0.0 : dm;  // distance.hpp:14-15
      const double dist = sqrt_search(v);
      s[q] = (unsigned long long)__double_as_longlong(dist) | (q >= P.n_must ? kFree : 0ULL);
    }
    sort_keys<D>(s);
    double acc = 0.0;
#pragma unroll
    for (int q = 0; q < D; ++q) {
      if (q >= P.D) break;
      acc += __longlong_as_double((long long)(s[q] & ~kFree));
      const double pk = acc * (1.0 / (double)(q + 1));
      long long* kq = P.keys + q * P.L;
      const long long kr = live ? pack_key(pk, j, P.imask) : kNoKey;
      if (live) {
        const long long kc = pack_key(pk, i, P.imask);
        if (kc < kq[j]) red_min64(&kq[j], kc);
      }
      const long long tr = kq[i];
      if (__any_sync(0xffffffffu, kr < tr)) {
        const long long b = warp_min64(kr);
        if (lane == 0 && b < tr) red_min64(&kq[i], b);
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
  const long long key = P.keys[kk * P.L + i];
  const long long j = key == kNoKey ? -1 : (key & P.imask);
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
        const double mi = P.mu[q * P.L + i], mj = P.mu[q * P.L + j];
        const double* xi = P.x + q * P.n + i;
        const double* xj = P.x + q * P.n + j;
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

// Bands of 32 diagonals in [klo, khi) x row segments of `seg` rows, for
// cells (i, i + k) with i < min(LR, LC - k). Largest items first.
void build_mitems(std::vector<MItem>& out, int pass, long long klo, long long khi, long long LR,
                  long long LC, long long seg) {
  for (long long kb = klo; kb < khi; kb += 32) {
    const long long rows = std::min(LR, LC - kb);
    for (long long r0 = 0; r0 < rows; r0 += seg)
      out.push_back(MItem{kb, r0, (int)std::min(seg, rows - r0), pass});
  }
}

void sort_mitems(std::vector<MItem>& v) {
  std::stable_sort(v.begin(), v.end(), [](const MItem& a, const MItem& b) { return a.nrows > b.nrows; });
}

// segment rows: long enough to amortise the O(m) seed, short enough to fill the GPU
long long seg_rows(long long m, long long L) {
  long long s = std::max<long long>(512, 4 * m);
  return std::min(s, std::max<long long>(L, 1));
}

struct DevMem {
  std::vector<void*> p;
  ~DevMem() {
    for (void* q : p) cudaFree(q);
  }
  template <class T>
  cudaError_t alloc(T** out, size_t count) {
    void* q = nullptr;
    cudaError_t e = cudaMalloc(&q, sizeof(T) * std::max<size_t>(count, 1));
    if (e == cudaSuccess) {
      p.push_back(q);
      *out = (T*)q;
    }
    return e;
  }
};

struct Timer {
  cudaEvent_t a = nullptr, b = nullptr;
  ~Timer() {
    if (a) cudaEventDestroy(a);
    if (b) cudaEventDestroy(b);
  }
};

std::mutex g_multi_mu;  // calls are serialised (scratch is per call)

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
  cudaStream_t st = nullptr;
  MM_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  struct StreamGuard {
    cudaStream_t s;
    ~StreamGuard() { cudaStreamDestroy(s); }
  } sg{st};
  Timer tm;
  MM_CUDA(cudaEventCreate(&tm.a));
  MM_CUDA(cudaEventCreate(&tm.b));

  const long long na = A->n_a, nb = self ? na : A->n_b;
  const long long La = na - m + 1, Lb = nb - m + 1;
  DevMem mem;
  double *xa, *xb = nullptr, *xca, *xcb = nullptr, *nra, *nrb = nullptr, *shift;
  long long *k0, *k1;
  MM_CUDA(mem.alloc(&xa, dims * na));
  MM_CUDA(mem.alloc(&xca, dims * na));
  MM_CUDA(mem.alloc(&nra, La));
  MM_CUDA(mem.alloc(&shift, dims));
  MM_CUDA(cudaMemcpyAsync(xa, A->a, sizeof(double) * dims * na, cudaMemcpyHostToDevice, st));
  if (!self) {
    MM_CUDA(mem.alloc(&xb, dims * nb));
    MM_CUDA(mem.alloc(&xcb, dims * nb));
    MM_CUDA(mem.alloc(&nrb, Lb));
    MM_CUDA(cudaMemcpyAsync(xb, A->b, sizeof(double) * dims * nb, cudaMemcpyHostToDevice, st));
  }
  // shared per-dim shift: the mean of A's dimension (host, from the caller's buffer)
  std::vector<double> sh(dims);
  for (long long d = 0; d < dims; ++d) {
    double s = 0.0;
    for (long long t = 0; t < na; ++t) s += A->a[d * na + t];
    sh[d] = s / (double)na;
  }
  MM_CUDA(cudaMemcpyAsync(shift, sh.data(), sizeof(double) * dims, cudaMemcpyHostToDevice, st));
  // self: k0 = right keys (row candidates), k1 = left keys (column candidates)
  // AB:   k0 = A keys, k1 = B keys
  MM_CUDA(mem.alloc(&k0, La));
  MM_CUDA(mem.alloc(&k1, self ? La : Lb));
  const int index_bits = std::max(1, ceil_log2ll(std::max(La, Lb)));
  const long long imask = (1LL << index_bits) - 1;

  std::vector<MItem> items;
  const long long seg = seg_rows(m, std::max(La, Lb));
  SimpleParams P{};
  P.dims = (int)dims;
  P.m = (int)m;
  P.imask = imask;
  RawSeries RA{xca, nra, na, La}, RB{xcb, nrb, nb, Lb};
  if (self) {
    if (A->zone + 1 < La) build_mitems(items, 0, A->zone + 1, La, La, La, seg);
    P.pass[0] = SimplePass{RA, RA, A->zone + 1, La, k0, k1};
  } else {
    // pass 0: rows = B windows, columns = A windows (k >= 0); pass 1: rows = A, columns = B (k >= 1)
    build_mitems(items, 0, 0, La, Lb, La, seg);
    if (Lb > 1) build_mitems(items, 1, 1, Lb, La, Lb, seg);
    P.pass[0] = SimplePass{RB, RA, 0, La, k1, k0};
    P.pass[1] = SimplePass{RA, RB, 1, Lb, k0, k1};
  }
  sort_mitems(items);
  MItem* d_items = nullptr;
  MM_CUDA(mem.alloc(&d_items, items.size()));
  MM_CUDA(cudaMemcpyAsync(d_items, items.data(), sizeof(MItem) * items.size(),
                          cudaMemcpyHostToDevice, st));
  P.items = d_items;
  P.n_items = (long long)items.size();

  MM_CUDA(cudaEventRecord(tm.a, st));
  const int bs = 256;
  k_center<<<(unsigned)((dims * na + bs - 1) / bs), bs, 0, st>>>(xa, na, (int)dims, shift, xca);
  k_raw_energy<<<(unsigned)((La + bs - 1) / bs), bs, 0, st>>>(xca, na, La, (int)dims, (int)m, nra);
  if (!self) {
    k_center<<<(unsigned)((dims * nb + bs - 1) / bs), bs, 0, st>>>(xb, nb, (int)dims, shift, xcb);
    k_raw_energy<<<(unsigned)((Lb + bs - 1) / bs), bs, 0, st>>>(xcb, nb, Lb, (int)dims, (int)m, nrb);
  }
  k_fill<<<(unsigned)((La + bs - 1) / bs), bs, 0, st>>>(k0, La);
  k_fill<<<(unsigned)(((self ? La : Lb) + bs - 1) / bs), bs, 0, st>>>(k1, self ? La : Lb);
  if (P.n_items > 0)
    k_simple<<<(unsigned)((P.n_items + kMWarps - 1) / kMWarps), kMWarps * 32, 0, st>>>(P);
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
    k_simple_finalize<<<fa, bs, 0, st>>>(xa, na, La, xa, na, k0, k1, (int)dims, (int)m, imask,
                                         omp_a, opi_a, ol, orr);
  } else {
    MM_CUDA(mem.alloc(&omp_b, Lb));
    MM_CUDA(mem.alloc(&opi_b, Lb));
    k_simple_finalize<<<fa, bs, 0, st>>>(xa, na, La, xb, nb, k0, nullptr, (int)dims, (int)m,
                                         imask, omp_a, opi_a, nullptr, nullptr);
    k_simple_finalize<<<(unsigned)((Lb * 32 + bs - 1) / bs), bs, 0, st>>>(
        xb, nb, Lb, xa, na, k1, nullptr, (int)dims, (int)m, imask, omp_b, opi_b, nullptr, nullptr);
  }
  MM_CUDA(cudaGetLastError());
  MM_CUDA(cudaEventRecord(tm.b, st));
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
    MM_CUDA(cudaEventElapsedTime(&ms, tm.a, tm.b));
    *A->kernel_ms = ms;
  }
  return MPGPU_OK;
}

}  // extern "C"

namespace {

template <int D>
void launch_mstomp(const MStompParams& P, cudaStream_t st) {
  if (P.n_items > 0)
    k_mstomp<D><<<(unsigned)((P.n_items + kMWarps - 1) / kMWarps), kMWarps * 32, 0, st>>>(P);
}

using MLaunch = void (*)(const MStompParams&, cudaStream_t);

MLaunch mstomp_launcher(int D) {
  switch (D) {
    case 1: return launch_mstomp<1>;
    case 2: return launch_mstomp<2>;
    case 3: return launch_mstomp<3>;
    case 4: return launch_mstomp<4>;
    case 5: return launch_mstomp<5>;
    case 6: return launch_mstomp<6>;
    case 7: return launch_mstomp<7>;
    case 8: return launch_mstomp<8>;
    default: break;
  }
  if (D <= 12) return launch_mstomp<12>;
  if (D <= 16) return launch_mstomp<16>;
  return launch_mstomp<32>;
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
  std::lock_guard<std::mutex> lk(g_multi_mu);
  MM_CUDA(cudaSetDevice(A->device));
  cudaStream_t st = nullptr;
  MM_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  struct StreamGuard {
    cudaStream_t s;
    ~StreamGuard() { cudaStreamDestroy(s); }
  } sg{st};
  Timer tm;
  MM_CUDA(cudaEventCreate(&tm.a));
  MM_CUDA(cudaEventCreate(&tm.b));

  const long long L = n - m + 1, pad = mpgpu_internal::stats_pad(), Lp = L + pad;
  DevMem mem;
  double *x, *mu, *inv, *omp;
  double2* U;
  long long *keys, *opi, *odo;
  int* dperm;
  MM_CUDA(mem.alloc(&x, (size_t)D * n));
  MM_CUDA(mem.alloc(&mu, (size_t)D * L));
  MM_CUDA(mem.alloc(&inv, (size_t)D * Lp));
  MM_CUDA(mem.alloc(&U, (size_t)D * Lp));
  MM_CUDA(mem.alloc(&keys, (size_t)D * L));
  MM_CUDA(mem.alloc(&omp, (size_t)dims * L));
  MM_CUDA(mem.alloc(&opi, (size_t)dims * L));
  MM_CUDA(mem.alloc(&odo, (size_t)dims * L));
  MM_CUDA(mem.alloc(&dperm, D));
  for (int q = 0; q < D; ++q)
    MM_CUDA(cudaMemcpyAsync(x + (size_t)q * n, A->x + (size_t)perm[q] * n, sizeof(double) * n,
                            cudaMemcpyHostToDevice, st));
  MM_CUDA(cudaMemcpyAsync(dperm, perm.data(), sizeof(int) * D, cudaMemcpyHostToDevice, st));
  const int index_bits = std::max(1, ceil_log2ll(L));
  const long long imask = (1LL << index_bits) - 1;
  std::vector<MItem> items;
  if (A->zone + 1 < L) build_mitems(items, 0, A->zone + 1, L, L, L, seg_rows(m, L));
  sort_mitems(items);
  MItem* d_items = nullptr;
  MM_CUDA(mem.alloc(&d_items, items.size()));
  if (!items.empty())
    MM_CUDA(cudaMemcpyAsync(d_items, items.data(), sizeof(MItem) * items.size(),
                            cudaMemcpyHostToDevice, st));

  MStompParams P{};
  P.x = x; P.mu = mu; P.inv = inv; P.U = U;
  P.n = n; P.L = L; P.Lp = Lp; P.khi = L;
  P.keys = keys; P.items = d_items; P.n_items = (long long)items.size();
  P.m = (int)m; P.n_must = n_must; P.D = D; P.imask = imask;

  MM_CUDA(cudaEventRecord(tm.a, st));
  for (int q = 0; q < D; ++q)
    MM_CUDA(mpgpu_internal::series_stats(x + (size_t)q * n, n, (int)m, mu + (size_t)q * L,
                                         inv + (size_t)q * Lp, U + (size_t)q * Lp, nullptr, st));
  const int bs = 256;
  k_fill<<<(unsigned)(((long long)D * L + bs - 1) / bs), bs, 0, st>>>(keys, (long long)D * L);
  MM_CUDA(cudaGetLastError());
  mstomp_launcher(D)(P, st);
  MM_CUDA(cudaGetLastError());
  const long long outs = (long long)dims * L;
  k_mstomp_finalize<<<(unsigned)((outs * 32 + bs - 1) / bs), bs, 0, st>>>(P, D, (int)dims, dperm,
                                                                         omp, opi, odo);
  MM_CUDA(cudaGetLastError());
  MM_CUDA(cudaEventRecord(tm.b, st));
  if (A->mp) MM_CUDA(cudaMemcpyAsync(A->mp, omp, sizeof(double) * outs, cudaMemcpyDeviceToHost, st));
  if (A->pi) MM_CUDA(cudaMemcpyAsync(A->pi, opi, sizeof(long long) * outs, cudaMemcpyDeviceToHost, st));
  if (A->dim_order)
    MM_CUDA(cudaMemcpyAsync(A->dim_order, odo, sizeof(long long) * outs, cudaMemcpyDeviceToHost, st));
  MM_CUDA(cudaStreamSynchronize(st));
  if (A->kernel_ms) {
    float ms = 0.f;
    MM_CUDA(cudaEventElapsedTime(&ms, tm.a, tm.b));
    *A->kernel_ms = ms;
  }
  return MPGPU_OK;
}

}  // extern "C"
