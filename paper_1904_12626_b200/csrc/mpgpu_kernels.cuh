// Device kernels of the B200 matrix-profile join (sm_100a, fp64 SIMT).
//
// K1 stats    — per-window mean, 1/||x - mu|| and flat flag (two-pass, exact),
//               plus the centred-covariance update vectors (df, dg).
//               Replaces rolling_mean_std + is_flat_std (rolling.hpp:21-29).
// K1f flats   — flat-window bitmask and next-flat index (for the flat-window
//               convention of znorm_dist_from_qt, distance.hpp:14-15).
// K3 join     — persistent diagonal-band kernel: seeds each band segment with
//               direct centred dot products (the reference's FFT seed row,
//               fft.hpp:49-50), walks rows with the O(1) recurrence
//               (centred form), and keeps row / column minima as
//               packed (score, index) int64 keys — merge_min (profile.hpp:68)
//               with ties to the smallest index.
// K4 finalize — keys -> MP / PI / left / right, flat fix-up, exact distance
//               of the chosen neighbour (profile.hpp:28-46).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace mpgpu {

// ---- tile shape -----------------------------------------------------------
constexpr int kD = 8;                      // diagonals per thread (register block)
constexpr int kWarps = 8;                  // warps per CTA
constexpr int kThreads = kWarps * 32;      // 256
constexpr int kW = kThreads * kD;          // diagonals per band (2048)
constexpr int kH = 128;                    // rows per tile
constexpr int kRing = kW + kH;             // column ring slots (2176)
constexpr int kNB = kRing / kD;            // blocks per ring plane (272)
constexpr int kPad = kW + 2 * kH + 64;     // zero padding after the last window
constexpr int kSeedChunk = 256;            // seed dot-product chunk (samples)
constexpr long long kKeyNone = 0x7fffffffffffffffLL;

static_assert(kRing % kD == 0, "ring must be a multiple of D");

struct Series {
  const double* x;   // raw samples, length n
  const double* mu;  // window means, length L
  const double* inv; // 1/||x_w - mu_w|| (0: flat or padding), length L + kPad
  const double2* U;  // U[i] = {df[i-1], dg[i-1]}, U[0] = U[L..] = 0, length L + kPad
  const uint32_t* flat_words; // bit i: window i is flat
  const int32_t* next_word;   // smallest w' >= w with flat_words[w'] != 0, else -1
  long long n, L;
  int n_words;
};

struct Pass {
  Series R, C;        // row series, column series
  long long* keyR;    // row keys (length R.L)
  long long* keyC;    // column keys (length C.L)
};

struct Item {
  int pass;
  int nrows;          // multiple of kH
  long long kb;       // first diagonal of the band
  long long r0;       // first row of the segment
};

struct JoinParams {
  Pass pass[2];
  const Item* items;
  int n_items;
  int* counter;
  int m;
  long long imask;    // (1 << index_bits) - 1
};

// ---- packed keys -----------------------------------------------------------
// key = (bits(score) & ~imask) | index with score = 1 - corr = d^2 / (2m) >= 0.
// Non-negative doubles order like int64, so a signed int64 min is an exact
// min-with-argmin whose ties go to the smallest index.
__device__ __forceinline__ long long mk_key(double c, long long idx, long long imask) {
  double s = 1.0 - c;
  s = s < 0.0 ? 0.0 : s;
  return (__double_as_longlong(s) & ~imask) | idx;
}

__device__ __forceinline__ long long mk_key_score(double s, long long idx, long long imask) {
  return (__double_as_longlong(s) & ~imask) | idx;
}

// Filter threshold for a key: the largest corr that certainly loses against it
// whatever its index (its score lands in a strictly higher quantisation
// bucket). Stored as a double whose HIGH word is compared as int32 against the
// high word of corr: for t >= 0, corr > t implies hi(corr) >= hi(t); negative
// thresholds become -0.0 (hi = INT_MIN, always fire).
__device__ __forceinline__ double thr_filter(long long key, long long imask) {
  if (key == kKeyNone) return -0.0;
  const double s_hi = __longlong_as_double((key & ~imask) + imask + 1);
  const double t = (1.0 - s_hi) - 1e-15;
  return t >= 0.0 ? t : -0.0;
}

// ---- K1: statistics ----------------------------------------------------------
// One thread per window; two passes over the window (exact, no cumsums).
__global__ void k_window_stats(const double* __restrict__ x, long long L, int m,
                               double* __restrict__ mu, double* __restrict__ inv,
                               double* __restrict__ sd_out, uint8_t* __restrict__ flat) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= L) return;
  const double* w = x + i;
  double s = 0.0;
  for (int k = 0; k < m; ++k) s += w[k];
  const double mean = s / (double)m;
  double ss = 0.0;
  for (int k = 0; k < m; ++k) {
    const double d = w[k] - mean;
    ss = fma(d, d, ss);
  }
  double sd = sqrt(ss / (double)m);
  const double scale = fabs(mean) > 1.0 ? fabs(mean) : 1.0;
  const bool is_flat = sd <= 1e-10 * scale;  // is_flat_std threshold
  if (is_flat) sd = 0.0;
  mu[i] = mean;
  if (inv) inv[i] = is_flat ? 0.0 : 1.0 / sqrt(ss);
  if (sd_out) sd_out[i] = sd;
  if (flat) flat[i] = is_flat ? 1 : 0;
}

// U[i] = {df[i-1], dg[i-1]} for 1 <= i < L; zero at 0 and in the padding.
// df[i] = (x[i+m] - x[i]) / 2, dg[i] = (x[i+m] - mu[i+1]) + (x[i] - mu[i]).
__global__ void k_update_vectors(const double* __restrict__ x, const double* __restrict__ mu,
                                 long long L, int m, double2* __restrict__ U,
                                 double* __restrict__ inv) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= L + kPad) return;
  if (i >= L) inv[i] = 0.0;
  double2 u = make_double2(0.0, 0.0);
  if (i >= 1 && i < L) {
    const long long p = i - 1;
    const double xo = x[p], xn = x[p + m];
    u.x = 0.5 * (xn - xo);
    u.y = (xn - mu[p + 1]) + (xo - mu[p]);
  }
  U[i] = u;
}

__global__ void k_flat_words(const uint8_t* __restrict__ flat, long long L, int n_words,
                             uint32_t* __restrict__ words) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long w = i >> 5;
  const bool f = i < L && flat[i];
  const unsigned b = __ballot_sync(0xffffffffu, f);
  if ((threadIdx.x & 31) == 0 && w < n_words) words[w] = b;
}

// Suffix "next non-empty word" in one block (n_words <= a few million).
__global__ void k_next_word(const uint32_t* __restrict__ words, int n_words,
                            int32_t* __restrict__ next) {
  __shared__ int32_t agg[1024];
  const int t = threadIdx.x, nt = blockDim.x;
  const int chunk = (n_words + nt - 1) / nt;
  const int lo = t * chunk, hi = min(n_words, lo + chunk);
  int32_t cur = -1;
  for (int w = hi - 1; w >= lo; --w)
    if (words[w]) cur = w;
  agg[t] = cur;
  __syncthreads();
  if (t == 0) {  // suffix over chunk aggregates (nt entries)
    int32_t run = -1;
    for (int q = nt - 1; q >= 0; --q) {
      const int32_t a = agg[q];
      agg[q] = run;  // exclusive: first non-empty word strictly after chunk q
      if (a >= 0) run = a;
    }
  }
  __syncthreads();
  int32_t run = agg[t];
  for (int w = hi - 1; w >= lo; --w) {
    if (words[w]) run = w;
    next[w] = run;
  }
}

__device__ __forceinline__ long long next_flat(const Series& s, long long p) {
  if (p >= s.L) return -1;
  if (p < 0) p = 0;
  const int w = (int)(p >> 5);
  const uint32_t bits = s.flat_words[w] & (0xffffffffu << (p & 31));
  if (bits) return ((long long)w << 5) + __ffs(bits) - 1;
  if (w + 1 >= s.n_words) return -1;
  const int w2 = s.next_word[w + 1];
  if (w2 < 0) return -1;
  return ((long long)w2 << 5) + __ffs(s.flat_words[w2]) - 1;
}

__device__ __forceinline__ bool is_flat_at(const Series& s, long long p) {
  return (s.flat_words[p >> 5] >> (p & 31)) & 1u;
}

// ---- K3: the diagonal join ----------------------------------------------------
struct __align__(16) JoinSmem {
  double2 colU[kRing];   // {df, dg} of ring columns, blocked-transposed
  double2 colI[kRing];   // {inv, thr_filter}
  long long colK[kRing]; // column keys (natural ring order)
  double2 rowU[kH];
  double2 rowI[kH];
  long long rowK[kH];
  int item;
  int zero;
};

__device__ __forceinline__ int ring_addr(long long x) {
  const long long p = x % kRing;
  return (int)((p % kD) * kNB + p / kD);
}

__global__ void __launch_bounds__(kThreads, 2) k_join(const JoinParams P) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  JoinSmem& S = *reinterpret_cast<JoinSmem*>(smem_raw);
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  (void)lane;
  const long long imask = P.imask;
  const int m = P.m;
  if (tid == 0) S.zero = 0;

  for (;;) {
    if (tid == 0) S.item = atomicAdd(P.counter, 1);
    __syncthreads();
    const int item_id = S.item;
    __syncthreads();
    if (item_id >= P.n_items) break;
    const Item it = P.items[item_id];
    const Pass& PS = P.pass[it.pass];
    const Series& R = PS.R;
    const Series& C = PS.C;
    const long long r0 = it.r0;
    const long long c0 = r0 + it.kb;  // column of (thread 0, d = 0) at row r0
    const int nrows = it.nrows;

    // ---- seeds: cov(r0, r0 + k) for the band's kW diagonals --------------
    double cov[kD];
    {
      double* ac = reinterpret_cast<double*>(S.colU);       // kSeedChunk
      double* xc = ac + kSeedChunk;                          // kW + kSeedChunk
      double* seed = reinterpret_cast<double*>(S.colI);      // kW
      const double mr = R.mu[r0];
      double mc[kD], acc[kD];
#pragma unroll
      for (int e = 0; e < kD; ++e) {
        const long long j = c0 + tid + e * kThreads;
        mc[e] = j < C.L ? C.mu[j] : 0.0;
        acc[e] = 0.0;
      }
      for (int t0 = 0; t0 < m; t0 += kSeedChunk) {
        const int tc = min(kSeedChunk, m - t0);
        for (int q = tid; q < tc; q += kThreads) ac[q] = R.x[r0 + t0 + q] - mr;
        for (int q = tid; q < kW + tc; q += kThreads) {
          const long long g = c0 + t0 + q;
          xc[q] = g < C.n ? C.x[g] : 0.0;
        }
        __syncthreads();
        for (int t = 0; t < tc; ++t) {
          const double a = ac[t];
#pragma unroll
          for (int e = 0; e < kD; ++e) acc[e] = fma(a, xc[tid + e * kThreads + t] - mc[e], acc[e]);
        }
        __syncthreads();
      }
#pragma unroll
      for (int e = 0; e < kD; ++e) seed[tid + e * kThreads] = acc[e];
      __syncthreads();
#pragma unroll
      for (int d = 0; d < kD; ++d) cov[d] = seed[tid * kD + d];
      __syncthreads();
    }

    double2 cU[kD];
    double cinv[kD];
    int cthr[kD];

    for (int ts = 0; ts < nrows; ts += kH) {
      // ---- tile boundary: retire, then load --------------------------------
      if (ts > 0) {
        for (int h = tid; h < kH; h += kThreads) {  // rows of the previous tile
          const long long i = r0 + ts - kH + h;
          const long long k = S.rowK[h];
          if (i < R.L && k != kKeyNone) atomicMin(&PS.keyR[i], k);
        }
        for (int q = tid; q < kH; q += kThreads) {  // columns [ts - kH, ts)
          const long long x = ts - kH + q;
          const long long j = c0 + x;
          const long long k = S.colK[x % kRing];
          if (j < C.L && k != kKeyNone) atomicMin(&PS.keyC[j], k);
        }
        __syncthreads();
      }
      for (int h = tid; h < kH; h += kThreads) {
        const long long i = r0 + ts + h;
        double2 u = (ts + h == 0) ? make_double2(0.0, 0.0) : R.U[i];
        const double inv = R.inv[i];
        long long key = kKeyNone;
        double thr = 2.0;  // never fires (padding / flat rows)
        if (i < R.L && inv != 0.0) {
          key = PS.keyR[i];
          thr = thr_filter(key, imask);
        }
        S.rowU[h] = u;
        S.rowI[h] = make_double2(inv, thr);
        S.rowK[h] = key;
      }
      {
        const long long xlo = ts == 0 ? 0 : ts + kW - 1;
        const long long xhi = ts + kH + kW - 1;
        for (long long x = xlo + tid; x < xhi; x += kThreads) {
          const long long j = c0 + x;
          const double inv = C.inv[j];
          long long key = kKeyNone;
          double thr = 2.0;
          if (j < C.L && inv != 0.0) {
            key = PS.keyC[j];
            thr = thr_filter(key, imask);
          }
          const int a = ring_addr(x);
          S.colU[a] = C.U[j];
          S.colI[a] = make_double2(inv, thr);
          S.colK[x % kRing] = key;
        }
      }
      __syncthreads();

      if (ts == 0) {  // prime slots 0..D-2 with columns tid*D + d
#pragma unroll
        for (int d = 0; d < kD - 1; ++d) {
          const int a = d * kNB + tid;
          cU[d] = S.colU[a];
          const double2 ci = S.colI[a];
          cinv[d] = ci.x;
          cthr[d] = __double2hiint(ci.y);
        }
      }

      // ---- compute the tile: kH rows x kD diagonals per thread --------------
      int b0 = (int)((ts / kD + tid) % kNB);
      for (int u = 0; u < kH; u += kD) {
        const int b1 = b0 + 1 == kNB ? 0 : b0 + 1;
#pragma unroll
        for (int s = 0; s < kD; ++s) {
          const int h = u + s;
          const int sin = (s + kD - 1) % kD;  // slot of the entering column
          {
            const int a = sin * kNB + (s == 0 ? b0 : b1);
            cU[sin] = S.colU[a];
            const double2 ci = S.colI[a];
            cinv[sin] = ci.x;
            cthr[sin] = __double2hiint(ci.y);
          }
          const double2 ru = S.rowU[h];
          const double2 ri = S.rowI[h];
          const int rthr = __double2hiint(ri.y);
          bool fire = false;
          double c[kD];
#pragma unroll
          for (int d = 0; d < kD; ++d) {
            const int sl = (s + d) % kD;
            cov[d] = fma(ru.x, cU[sl].y, cov[d]);
            cov[d] = fma(ru.y, cU[sl].x, cov[d]);
            c[d] = cov[d] * ri.x * cinv[sl];
            const int hc = __double2hiint(c[d]);
            fire |= (hc >= rthr) | (hc >= cthr[sl]);
          }
          if (__builtin_expect(fire, 0)) {
            // ---- slow path: exact key updates (rare) ------------------------
            // volatile read: keeps the slow path's address math out of the fast path
            const int zv = *(volatile int*)&S.zero;
            const long long rho = ts + h + zv;
            const long long i = r0 + rho;
            if (ri.x != 0.0) {
              long long rbest = kKeyNone;
#pragma unroll
              for (int d = 0; d < kD; ++d) {
                const int sl = (s + d) % kD;
                if (cinv[sl] == 0.0) continue;
                const int hc = __double2hiint(c[d]);
                const long long x = rho + (long long)tid * kD + d;
                if (hc >= rthr) {
                  const long long key = mk_key(c[d], c0 + x, imask);
                  rbest = key < rbest ? key : rbest;
                }
                if (hc >= cthr[sl]) {
                  const long long key = mk_key(c[d], i, imask);
                  const long long old = atomicMin(&S.colK[x % kRing], key);
                  const double t = thr_filter(key < old ? key : old, imask);
                  cthr[sl] = __double2hiint(t);
                  S.colI[ring_addr(x)].y = t;
                }
              }
              if (rbest != kKeyNone) {
                const long long old = atomicMin(&S.rowK[h], rbest);
                S.rowI[h].y = thr_filter(rbest < old ? rbest : old, imask);
              }
            }
          }
        }
        b0 = b1;
      }
      __syncthreads();
    }
    // ---- segment end: flush the last tile's rows and all live columns ------
    {
      const int ts = nrows - kH;
      for (int h = tid; h < kH; h += kThreads) {
        const long long i = r0 + ts + h;
        const long long k = S.rowK[h];
        if (i < R.L && k != kKeyNone) atomicMin(&PS.keyR[i], k);
      }
      for (int q = tid; q < kH + kW - 1; q += kThreads) {
        const long long x = ts + q;
        const long long j = c0 + x;
        const long long k = S.colK[x % kRing];
        if (j < C.L && k != kKeyNone) atomicMin(&PS.keyC[j], k);
      }
    }
    __syncthreads();
  }
}

// ---- K5: key merge -------------------------------------------------------------
__global__ void k_keys_min(long long* __restrict__ dst, const long long* __restrict__ src,
                           long long len) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < len) {
    const long long a = dst[i], b = src[i];
    dst[i] = b < a ? b : a;
  }
}

__global__ void k_fill_keys(long long* __restrict__ k, long long len) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < len) k[i] = kKeyNone;
}

// ---- K4: finalize --------------------------------------------------------------
// Exact z-normalised distance between window i of X and window j of Y, one
// warp: d^2 = m * sum_t ((x_t - mu_i) inv_i - (y_t - mu_j) inv_j)^2.
__device__ __forceinline__ double warp_exact_dist(const Series& X, long long i, const Series& Y,
                                                  long long j, int m, int lane) {
  const double mi = X.mu[i], ii = X.inv[i], mj = Y.mu[j], ij = Y.inv[j];
  const double* xi = X.x + i;
  const double* yj = Y.x + j;
  double acc = 0.0;
  for (int t = lane; t < m; t += 32) {
    const double d = (xi[t] - mi) * ii - (yj[t] - mj) * ij;
    acc = fma(d, d, acc);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  double d2 = (double)m * acc;
  const double cap = 4.0 * (double)m;
  d2 = d2 > cap ? cap : d2;
  return sqrt(d2);
}

__device__ __forceinline__ double convention_or_exact(const Series& X, long long i,
                                                      const Series& Y, long long j, int m,
                                                      int lane) {
  const bool fi = X.inv[i] == 0.0, fj = Y.inv[j] == 0.0;
  if (fi && fj) return 0.0;
  if (fi || fj) return sqrt((double)m);
  return warp_exact_dist(X, i, Y, j, m, lane);
}

// Self-join: window i has right key (row keys) and left key (column keys).
__global__ void k_finalize_self(const Series A, const long long* __restrict__ key_right,
                                const long long* __restrict__ key_left, long long zone, int m,
                                long long imask, double* __restrict__ mp, long long* __restrict__ pi,
                                long long* __restrict__ left, long long* __restrict__ right) {
  const long long i = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (i >= A.L) return;
  const long long L = A.L;
  long long rk = key_right[i], lk = key_left[i];
  const double half = 0.5;
  const long long rlo = i + zone + 1;  // smallest admissible right neighbour
  const long long lhi = i - zone - 1;  // largest admissible left neighbour
  const long long nf_r = rlo < L ? next_flat(A, rlo) : -1;
  const long long f0 = next_flat(A, 0);
  const bool nf_l = f0 >= 0 && f0 <= lhi;
  if (A.inv[i] == 0.0) {  // flat window: distances are 0 (flat) or sqrt(m)
    rk = nf_r >= 0 ? mk_key_score(0.0, nf_r, imask)
                   : (rlo < L ? mk_key_score(half, rlo, imask) : kKeyNone);
    lk = nf_l ? mk_key_score(0.0, f0, imask) : (lhi >= 0 ? mk_key_score(half, 0, imask) : kKeyNone);
  } else {
    if (nf_r >= 0) {
      const long long k = mk_key_score(half, nf_r, imask);
      rk = k < rk ? k : rk;
    }
    if (nf_l) {
      const long long k = mk_key_score(half, f0, imask);
      lk = k < lk ? k : lk;
    }
  }
  const long long best = lk <= rk ? lk : rk;
  const long long bi = best == kKeyNone ? -1 : (best & imask);
  double v = INFINITY;
  if (bi >= 0) v = convention_or_exact(A, i, A, bi, m, lane);
  if (lane == 0) {
    if (mp) mp[i] = v;
    if (pi) pi[i] = bi;
    if (left) left[i] = lk == kKeyNone ? -1 : (lk & imask);
    if (right) right[i] = rk == kKeyNone ? -1 : (rk & imask);
  }
}

// AB-join side: window i of X against every window of Y.
__global__ void k_finalize_ab(const Series X, const Series Y, const long long* __restrict__ keys,
                              int m, long long imask, double* __restrict__ mp,
                              long long* __restrict__ pi) {
  const long long i = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (i >= X.L) return;
  long long k = keys[i];
  const long long fy = next_flat(Y, 0);
  if (X.inv[i] == 0.0) {
    k = fy >= 0 ? mk_key_score(0.0, fy, imask) : mk_key_score(0.5, 0, imask);
  } else if (fy >= 0) {
    const long long kf = mk_key_score(0.5, fy, imask);
    k = kf < k ? kf : k;
  }
  const long long bi = k == kKeyNone ? -1 : (k & imask);
  double v = INFINITY;
  if (bi >= 0) v = convention_or_exact(X, i, Y, bi, m, lane);
  if (lane == 0) {
    if (mp) mp[i] = v;
    if (pi) pi[i] = bi;
  }
}

}  // namespace mpgpu
