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
#ifndef MPGPU_D
#define MPGPU_D 8
#endif
constexpr int kD = MPGPU_D;                // diagonals per thread (register block)
#ifndef MPGPU_WARPS
#define MPGPU_WARPS 12
#endif
#ifndef MPGPU_MINBLOCKS
#define MPGPU_MINBLOCKS 1
#endif
constexpr int kMinBlocks = MPGPU_MINBLOCKS;  // CTAs per SM the register budget targets
#ifndef MPGPU_BLOCK
#define MPGPU_BLOCK 8
#endif
constexpr int kBlock = MPGPU_BLOCK;          // row-steps per branch-free block (divides kD)
// per-lane prefetch streams in k_join's tile loop (MPGPU_NO_LANE_STREAMS: the
// round-1 index arithmetic, for A/B runs)
#if !defined(MPGPU_NO_LANE_STREAMS) && !defined(MPGPU_LANE_STREAMS)
#define MPGPU_LANE_STREAMS 1
#endif
constexpr int kWarps = MPGPU_WARPS;          // warps per CTA (independent workers)
constexpr int kThreads = kWarps * 32;      // 256
constexpr int kW = 32 * kD;                // diagonals per band = per warp item (256)
#ifndef MPGPU_H
#define MPGPU_H 32
#endif
constexpr int kH = MPGPU_H;                // rows per warp tile
constexpr int kRing = ((kW + 2 * kH + kD - 1) / kD) * kD;  // column ring slots per warp (320)
constexpr int kNB = kRing / kD;            // blocks per ring plane (40)
constexpr int kPad = kW + 2 * kH + 64;     // zero padding after the last window
constexpr int kSeedChunk = 128;            // seed dot-product chunk (samples)
constexpr long long kKeyNone = 0x7fffffffffffffffLL;

static_assert(kRing % kD == 0, "ring must be a multiple of D");
static_assert(kH % kD == 0, "tiles hold whole blocks of kD row-steps");
static_assert(kD % kBlock == 0, "blocks tile the kD-step rotation");

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
  unsigned long long* stats;  // optional fire counters (MPGPU_STATS=1), else null
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

// Fast-path form of a threshold: its hi word lowered by 3 units. The fast pass
// tests corr computed with a cinv whose low 32 bits are replaced by the column
// threshold (see pack_col): a relative error below 2^-20, i.e. under 3 hi-word
// units, which the lowering absorbs (never skips a cell the exact test would
// take). INT_MIN (always fire) stays.
__device__ __forceinline__ int lower_thr(int h) { return h == INT_MIN ? h : h - 3; }
// Packed column value: high word of cinv, low word the lowered threshold. The
// fast pass uses it both as the (perturbed) cinv operand and as the threshold,
// which frees a register per column slot; the replay reads the exact cinv.
__device__ __forceinline__ double pack_col(double inv, int thr_lowered) {
  return __hiloint2double(__double2hiint(inv), thr_lowered);
}

// ---- K1: statistics ----------------------------------------------------------
// Two passes over every window (exact, no cumsums), each a strictly sequential
// sum over the window's samples in order: the statistics of a window do not
// depend on how the work is laid out (the two kernels below and k_query_stats
// agree bit for bit).
// k_window_stats: one thread per window. Bound by L1 bandwidth (m loads per
// window and pass), but it spreads a short series over the whole GPU.
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

// k_window_stats_blocked, for long series (enough windows for >= 2 CTAs per
// SM): a thread owns kStatR consecutive windows and slides a register window
// over the series staged in shared memory, one shared load per kStatR
// additions. C4: 145 -> ~60 us.
constexpr int kStatThreads = 128;
constexpr int kStatR = 8;
constexpr int kStatTile = kStatThreads * kStatR;  // windows per CTA (1024)
constexpr int kStatChunk = 512;                   // window samples staged per pass
constexpr int kStatSx = kStatTile + kStatChunk + kStatR;
__device__ __forceinline__ int stat_pad(int x) { return x + x / kStatR; }  // conflict-free (see mass_pad)
constexpr int kStatSxPad = kStatSx + kStatSx / kStatR + 1;
static_assert(kStatChunk % kStatR == 0, "chunks in whole register-window rotations");

__global__ void __launch_bounds__(kStatThreads) k_window_stats_blocked(
    const double* __restrict__ x, long long L, int m, double* __restrict__ mu,
    double* __restrict__ inv, double* __restrict__ sd_out, uint8_t* __restrict__ flat) {
  __shared__ double sx[kStatSxPad];
  const long long i0 = (long long)blockIdx.x * kStatTile;
  const int tid = threadIdx.x, jl = tid * kStatR;
  const long long n = L + m - 1;
  double s[kStatR], mean[kStatR], ss[kStatR];
#pragma unroll
  for (int r = 0; r < kStatR; ++r) s[r] = ss[r] = 0.0;
#pragma unroll 1
  for (int pass = 0; pass < 2; ++pass) {
    if (pass == 1) {
#pragma unroll
      for (int r = 0; r < kStatR; ++r) mean[r] = s[r] / (double)m;
    }
    for (int t0 = 0; t0 < m; t0 += kStatChunk) {
      const int tc = min(kStatChunk, m - t0);
      __syncthreads();
      for (int t = tid; t < kStatTile + tc; t += kStatThreads) {
        const long long g = i0 + t0 + t;
        sx[stat_pad(t)] = g < n ? x[g] : 0.0;
      }
      __syncthreads();
      // rotating register window: slot (t + r) % kStatR holds x[i0 + jl + t0 + t + r]
      double w[kStatR];
#pragma unroll
      for (int r = 0; r < kStatR; ++r) w[r] = sx[stat_pad(jl + r)];
      for (int t8 = 0; t8 < tc; t8 += kStatR) {
#pragma unroll
        for (int u = 0; u < kStatR; ++u) {
          if (t8 + u < tc) {  // warp-uniform
            if (pass == 0) {
#pragma unroll
              for (int r = 0; r < kStatR; ++r) s[r] += w[(u + r) % kStatR];
            } else {
#pragma unroll
              for (int r = 0; r < kStatR; ++r) {
                const double d = w[(u + r) % kStatR] - mean[r];
                ss[r] = fma(d, d, ss[r]);
              }
            }
            w[u] = sx[stat_pad(jl + kStatR + t8 + u)];
          }
        }
      }
    }
  }
#pragma unroll
  for (int r = 0; r < kStatR; ++r) {
    const long long i = i0 + jl + r;
    if (i >= L) break;
    double sd = sqrt(ss[r] / (double)m);
    const double scale = fabs(mean[r]) > 1.0 ? fabs(mean[r]) : 1.0;
    const bool is_flat = sd <= 1e-10 * scale;  // is_flat_std threshold
    if (is_flat) sd = 0.0;
    mu[i] = mean[r];
    if (inv) inv[i] = is_flat ? 0.0 : 1.0 / sqrt(ss[r]);
    if (sd_out) sd_out[i] = sd;
    if (flat) flat[i] = is_flat ? 1 : 0;
  }
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

// "Next non-empty word" next[w] = smallest w' >= w with words[w'] != 0 (else
// -1), a suffix-min scan in three launches: (1) within blocks of 1024 words
// (warp ballots + a 32-entry warp suffix), each block's first non-empty word
// into agg; (2) one block turns agg into "first non-empty word in any later
// block"; (3) words still -1 after (1) take that value. Replaces a one-block
// sequential scan (63 us at n = 2^20, 8 per launch of (1) and (3)).
constexpr int kNextBlock = 1024;

__global__ void __launch_bounds__(kNextBlock) k_next_word_local(const uint32_t* __restrict__ words,
                                                                int n_words, int32_t* __restrict__ next,
                                                                int32_t* __restrict__ agg) {
  __shared__ int32_t wfirst[kNextBlock / 32];
  const int w = blockIdx.x * kNextBlock + threadIdx.x;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const bool ne = w < n_words && words[w] != 0u;
  const unsigned m = __ballot_sync(0xffffffffu, ne);
  const unsigned up = m & (0xffffffffu << lane);  // non-empty lanes >= this one
  int32_t v = up ? (w - lane) + __ffs(up) - 1 : -1;
  if (lane == 0) wfirst[wid] = m ? w + __ffs(m) - 1 : -1;
  __syncthreads();
  if (v < 0) {  // first non-empty word in a later warp of this block
    for (int q = wid + 1; q < kNextBlock / 32; ++q)
      if (wfirst[q] >= 0) { v = wfirst[q]; break; }
  }
  if (w < n_words) next[w] = v;
  if (threadIdx.x == 0) {
    int32_t f = -1;
    for (int q = 0; q < kNextBlock / 32; ++q)
      if (wfirst[q] >= 0) { f = wfirst[q]; break; }
    agg[blockIdx.x] = f;
  }
}

// agg[b] <- first non-empty word in blocks > b (exclusive suffix), one block.
__global__ void __launch_bounds__(1024) k_next_word_aggs(int32_t* __restrict__ agg, int nb) {
  __shared__ int32_t part[1024];
  const int t = threadIdx.x;
  const int chunk = (nb + 1023) / 1024;
  const int lo = t * chunk, hi = min(nb, lo + chunk);
  int32_t f = -1;
  for (int b = hi - 1; b >= lo; --b)
    if (agg[b] >= 0) f = agg[b];
  part[t] = f;  // first non-empty word of this thread's chunk
  __syncthreads();
  // Hillis-Steele suffix: part[t] <- first non-empty word of chunks t.. (the
  // earliest valid entry wins)
  for (int d = 1; d < 1024; d <<= 1) {
    const int32_t y = t + d < 1024 ? part[t + d] : -1;
    __syncthreads();
    if (part[t] < 0) part[t] = y;
    __syncthreads();
  }
  const int32_t after0 = t + 1 < 1024 ? part[t + 1] : -1;  // first after this chunk
  int32_t after = after0;
  for (int b = hi - 1; b >= lo; --b) {
    const int32_t a = agg[b];
    agg[b] = after;
    if (a >= 0) after = a;
  }
}

__global__ void k_next_word_fix(int32_t* __restrict__ next, int n_words,
                                const int32_t* __restrict__ agg) {
  const int w = blockIdx.x * blockDim.x + threadIdx.x;
  if (w < n_words && next[w] < 0) next[w] = agg[w / kNextBlock];
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
// Every warp is an independent worker: it pulls (band, segment) items from a
// global queue and walks a band of kW = 256 diagonals over the segment's
// rows. Lane t owns diagonals kb + t*kD + [0, kD) and keeps their centred
// covariances in registers; the kD column windows it touches live in a
// register shift window refilled from the warp's shared-memory ring
// (blocked-transposed so the 32 lanes read 32 consecutive 16-byte slots).
// Rows stream through a double buffer; tile t+1 is fetched with cp.async
// while tile t computes. No CTA barrier anywhere in the loop: warps never
// wait on each other, so the rare slow path costs only its own warp.
//
// Minima never live in shared memory: a cell that passes the filter is
// min-merged straight into the global key arrays with RED.MIN.S64 (native;
// a shared-memory 64-bit atomicMin is a CAS spin loop). Shared memory only
// holds the filter thresholds, refreshed from the keys at tile load and
// raised by the slow path.
struct __align__(16) WarpSmem {
  double2 colU[kRing];      // {df, dg} of ring columns, blocked-transposed
  double2 colI[kRing];      // {inv, pack_col(inv, lowered thr)}; .y stages the raw key on fetch
  double2 rowU[2][kH + 1];  // +1: harmless read one past the tile
  double2 rowI[2][kH + 1];  // {inv, lowered thr in the hi word}; .y stages the raw key on fetch
  int zero;                 // always 0; read volatile to pin slow-path math
};
struct __align__(16) JoinSmem {
  WarpSmem w[kWarps];
};

// x < 2^31 (segment-local column offsets): 32-bit modulo, not a 64-bit one
__device__ __forceinline__ int ring_addr(long long x) {
  const int p = (int)((unsigned)x % (unsigned)kRing);
  return (p % kD) * kNB + p / kD;
}

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(dst)), "l"(src));
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_u32(dst)), "l"(src));
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_all;\n" ::: "memory");
}
__device__ __forceinline__ void red_min(long long* p, long long v) {
  // no "memory" clobber: REDs need no ordering against the loop's shared loads
  asm volatile("red.relaxed.gpu.global.min.s64 [%0], %1;\n" ::"l"(p), "l"(v));
}

// Column x of the segment -> ring (raw copy; the key bits land in .y).
__device__ __forceinline__ void fetch_col(WarpSmem& S, const Pass& PS, long long c0, long long x) {
  const long long j = c0 + x;
  const int a = ring_addr(x);
  cp_async16(&S.colU[a], &PS.C.U[j]);
  cp_async8(&S.colI[a].x, &PS.C.inv[j]);
  if (j < PS.C.L) cp_async8(&S.colI[a].y, &PS.keyC[j]);
}
__device__ __forceinline__ void fix_col(WarpSmem& S, const Pass& PS, long long c0, long long x,
                                        long long imask) {
  const int a = ring_addr(x);
  const double2 v = S.colI[a];
  const bool live = (c0 + x) < PS.C.L && v.x != 0.0;
  const double t = live ? thr_filter(__double_as_longlong(v.y), imask) : 2.0;
  S.colI[a].y = pack_col(v.x, lower_thr(__double2hiint(t)));
}
__device__ __forceinline__ void fetch_row(WarpSmem& S, const Pass& PS, int buf, int h, long long i) {
  cp_async16(&S.rowU[buf][h], &PS.R.U[i]);
  cp_async8(&S.rowI[buf][h].x, &PS.R.inv[i]);
  if (i < PS.R.L) cp_async8(&S.rowI[buf][h].y, &PS.keyR[i]);
}
__device__ __forceinline__ void fix_row(WarpSmem& S, const Pass& PS, int buf, int h, long long i,
                                        long long imask) {
  const double2 v = S.rowI[buf][h];
  const bool live = i < PS.R.L && v.x != 0.0;
  const double t = live ? thr_filter(__double_as_longlong(v.y), imask) : 2.0;
  S.rowI[buf][h].y = __hiloint2double(lower_thr(__double2hiint(t)), 0);
}

// Rare path, entered by the whole warp when any lane's cell passed a row or
// column filter. Out of line (one copy, so the unrolled fast loop stays
// compact in the instruction cache) and store-free towards shared memory:
// candidates go straight to the global keys with RED.MIN, raised column
// thresholds come back in registers. Arrays are in diagonal order d (the
// caller resolves slot (s+d)%kD).
// Rare path, entered by the whole warp when any lane's cell passed a row or
// column filter. Out of line so the unrolled fast loop stays small. Arrays
// are in diagonal order d (the caller resolves slot (s+d)%kD).
struct SlowIn {
  double c[kD];
  int cthr[kD];
};
struct SlowOut {
  int cthr[kD];
};

__device__ __forceinline__ double pick(const double (&v)[kD], int d) {
  double r = v[0];
#pragma unroll
  for (int q = 1; q < kD; ++q) r = d == q ? v[q] : r;
  return r;
}

__device__ __noinline__ SlowOut slow_path(const SlowIn in, unsigned live, int rthr, long long i,
                                          long long x0, long long c0, int h, int buf,
                                          long long imask, long long* keyR, long long* keyC,
                                          unsigned long long* stats) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  WarpSmem& S = reinterpret_cast<JoinSmem*>(smem_raw)->w[threadIdx.x >> 5];
  SlowOut out;
  // candidate masks: bit d set when cell d passes the row / column filter
  unsigned rmask = 0, cmask = 0;
#pragma unroll
  for (int d = 0; d < kD; ++d) {
    out.cthr[d] = in.cthr[d];
    const int hc = __double2hiint(in.c[d]);
    rmask |= (hc >= rthr ? 1u : 0u) << d;
    cmask |= (hc >= in.cthr[d] ? 1u : 0u) << d;
  }
  rmask &= live;
  cmask &= live;
  if (stats) {
    if ((threadIdx.x & 31) == 0) atomicAdd(&stats[0], 1ull);
    atomicAdd(&stats[1], (unsigned long long)__popc(rmask));
    atomicAdd(&stats[2], (unsigned long long)__popc(cmask));
  }
  // columns: one RED per candidate, raise the shared and register thresholds.
  // Unrolled over the kD static slots (predicated per candidate): no dynamic
  // register indexing, no jump table, no local memory.
  if (cmask) {
#pragma unroll
    for (int d = 0; d < kD; ++d) {
      if ((cmask >> d) & 1u) {
        const long long x = x0 + d;
        const long long key = mk_key(in.c[d], i, imask);
        red_min(&keyC[c0 + x], key);
        const int th = lower_thr(__double2hiint(thr_filter(key, imask)));
        out.cthr[d] = th > out.cthr[d] ? th : out.cthr[d];
        const int a = ring_addr(x);
        const double2 ci = S.colI[a];
        if (th > __double2loint(ci.y)) S.colI[a].y = pack_col(ci.x, th);  // lanes of one warp: benign race
      }
    }
  }
  // row: the lane's smallest key over its candidates (branch-free), then the warp's
  if (__any_sync(0xffffffffu, rmask != 0)) {
    long long rbest = kKeyNone;
#pragma unroll
    for (int d = 0; d < kD; ++d) {
      const long long key = mk_key(in.c[d], c0 + x0 + d, imask);
      const bool take = ((rmask >> d) & 1u) && key < rbest;
      rbest = take ? key : rbest;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const long long v = __shfl_xor_sync(0xffffffffu, rbest, o);
      rbest = v < rbest ? v : rbest;
    }
    if ((threadIdx.x & 31) == 0 && rbest != kKeyNone) {
      red_min(&keyR[i], rbest);
      const int th = lower_thr(__double2hiint(thr_filter(rbest, imask)));
      if (th > __double2hiint(S.rowI[buf][h].y)) S.rowI[buf][h].y = __hiloint2double(th, 0);
    }
  }
  __syncwarp();
  return out;
}

// Any cell over its threshold: hc[d] >= t[d], as a shallow predicate tree
// (the compiler otherwise chains kD dependent ISETP.OR).
static_assert(kD >= 4 && kD <= 16, "kD out of range");
__device__ __forceinline__ bool any_ge(const int (&hc)[kD], const int (&t)[kD]) {
  unsigned r;
  if constexpr (kD != 8 && kD != 4) {
    bool a = false, b = false, c = false, d = false;
#pragma unroll
    for (int q = 0; q < kD; q += 4) {
      a |= hc[q] >= t[q];
      if (q + 1 < kD) b |= hc[q + 1] >= t[q + 1];
      if (q + 2 < kD) c |= hc[q + 2] >= t[q + 2];
      if (q + 3 < kD) d |= hc[q + 3] >= t[q + 3];
    }
    r = (a | b) | (c | d);
  } else if constexpr (kD == 8) {
    asm("{\n\t.reg .pred a, b, c, d;\n\t"
        "setp.ge.s32 a, %1, %9;\n\t"
        "setp.ge.s32 b, %3, %11;\n\t"
        "setp.ge.s32 c, %5, %13;\n\t"
        "setp.ge.s32 d, %7, %15;\n\t"
        "setp.ge.or.s32 a, %2, %10, a;\n\t"
        "setp.ge.or.s32 b, %4, %12, b;\n\t"
        "setp.ge.or.s32 c, %6, %14, c;\n\t"
        "setp.ge.or.s32 d, %8, %16, d;\n\t"
        "or.pred a, a, b;\n\t"
        "or.pred c, c, d;\n\t"
        "or.pred a, a, c;\n\t"
        "selp.u32 %0, 1, 0, a;\n\t}"
        : "=r"(r)
        : "r"(hc[0]), "r"(hc[1]), "r"(hc[2]), "r"(hc[3]), "r"(hc[4]), "r"(hc[5]), "r"(hc[6]),
          "r"(hc[7]), "r"(t[0]), "r"(t[1]), "r"(t[2]), "r"(t[3]), "r"(t[4]), "r"(t[5]), "r"(t[6]),
          "r"(t[7]));
  } else {
    asm("{\n\t.reg .pred a, b;\n\t"
        "setp.ge.s32 a, %1, %5;\n\t"
        "setp.ge.s32 b, %3, %7;\n\t"
        "setp.ge.or.s32 a, %2, %6, a;\n\t"
        "setp.ge.or.s32 b, %4, %8, b;\n\t"
        "or.pred a, a, b;\n\t"
        "selp.u32 %0, 1, 0, a;\n\t}"
        : "=r"(r)
        : "r"(hc[0]), "r"(hc[1]), "r"(hc[2]), "r"(hc[3]), "r"(t[0]), "r"(t[1]), "r"(t[2]), "r"(t[3]));
  }
  return r != 0;
}

// Direct seeds of a band segment: cov(r0, r0 + k) for the band's kW diagonals
// (the reference's FFT seed row, fft.hpp:49-50), lane t receiving its
// diagonals t*kD + [0, kD). c0 = r0 + kb.
__device__ __forceinline__ void seed_direct(WarpSmem& S, const Series& R, const Series& C, long long r0,
                                            long long c0, int m, int lane, double (&cov)[kD]) {
  // cov = sum_t a_t (y_t - mu_j) = sum_t a_t y_t - mu_j sum_t a_t with the
  // row window centred (a_t = x_t - mu_i, sum a_t ~ 0): one DFMA per term.
  double* ac = reinterpret_cast<double*>(S.colU);       // kSeedChunk
  double* xc = ac + kSeedChunk;                          // kW + kSeedChunk
  double* seed = reinterpret_cast<double*>(S.colI);      // kW
  const double mr = R.mu[r0];
  double mc[kD], acc[kD];
#pragma unroll
  for (int e = 0; e < kD; ++e) {
    const long long j = c0 + lane + e * 32;
    mc[e] = j < C.L ? C.mu[j] : 0.0;
    acc[e] = 0.0;
  }
  double asum = 0.0;
  for (int t0 = 0; t0 < m; t0 += kSeedChunk) {
    const int tc = min(kSeedChunk, m - t0);
    for (int q = lane; q < tc; q += 32) ac[q] = R.x[r0 + t0 + q] - mr;
    for (int q = lane; q < kW + tc; q += 32) {
      const long long g = c0 + t0 + q;
      xc[q] = g < C.n ? C.x[g] : 0.0;
    }
    __syncwarp();
    for (int t = 0; t < tc; ++t) {
      const double a = ac[t];
      asum += a;
#pragma unroll
      for (int e = 0; e < kD; ++e) acc[e] = fma(a, xc[lane + e * 32 + t], acc[e]);
    }
    __syncwarp();
  }
#pragma unroll
  for (int e = 0; e < kD; ++e) seed[lane + e * 32] = fma(-mc[e], asum, acc[e]);
  __syncwarp();
#pragma unroll
  for (int d = 0; d < kD; ++d) cov[d] = seed[lane * kD + d];
  __syncwarp();
}

// A diagonal whose covariance is this NaN (sign bit set) never produces a
// candidate: DFMA and DMUL propagate the NaN with its sign (measured on
// sm_100a), so the high word of every "correlation" along it is 0xfff80000, a
// negative int32 below every filter threshold. k_join_masked seeds the
// diagonals outside an anytime run's chosen set with it: the fast pass needs no
// mask at all, only the replay excludes them from its candidates.
constexpr unsigned long long kMaskedCov = 0xfff8000000000000ULL;

// The walk of one band segment: rows [r0, r0 + nT*kH) of the kW diagonals from
// kb, starting from the covariances at row r0 in cov (the seed row takes no
// step). kMasked: dmask holds this lane's chosen diagonals (bit d), the others
// carry kMaskedCov.
template <bool kMasked>
__device__ __forceinline__ void walk_band(WarpSmem& S, const Pass& PS, const int m, const long long imask,
                                          unsigned long long* const stats, const int lane,
                                          const long long r0, const long long kb, const int nT,
                                          double (&cov)[kD], const unsigned dmask) {
  const Series& R = PS.R;
  const Series& C = PS.C;
  const long long c0 = r0 + kb;  // column of (lane 0, d = 0) at row r0
  // ---- tile 0: rows [0, kH) -> buffer 0, columns [0, kH + kW - 1) ------
  static_assert(kH >= 1, "tile rows");
  if constexpr (kH <= 32) {
    if (lane < kH) fetch_row(S, PS, 0, lane, r0 + lane);
  } else {
    for (int h = lane; h < kH; h += 32) fetch_row(S, PS, 0, h, r0 + h);
  }
  for (int x = lane; x < kH + kW - 1; x += 32) fetch_col(S, PS, c0, x);
  cp_async_wait_all();
  if constexpr (kH <= 32) {
    if (lane < kH) fix_row(S, PS, 0, lane, r0 + lane, imask);
  } else {
    for (int h = lane; h < kH; h += 32) fix_row(S, PS, 0, h, r0 + h, imask);
  }
  if (lane == 0) S.rowU[0][0] = make_double2(0.0, 0.0);  // the seed row takes no step
  for (int x = lane; x < kH + kW - 1; x += 32) fix_col(S, PS, c0, x, imask);
  __syncwarp();

  double2 cU[kD];
  double cpk[kD];  // pack_col: perturbed cinv (hi word) + lowered threshold (lo word)
#pragma unroll
  for (int d = 0; d < kD - 1; ++d) {  // prime slots 0..D-2 with columns lane*D + d
    const int a = d * kNB + lane;
    cU[d] = S.colU[a];
    cpk[d] = S.colI[a].y;
  }

#ifdef MPGPU_LANE_STREAMS
  // Per-lane prefetch streams, set up once per item: the row and column this
  // lane fetches for tile t + 1 sit at fixed offsets from these pointers
  // (+ t * kH), and its ring slot advances by kH modulo kRing, so a tile's
  // prefetch and fix-up need no 64-bit index arithmetic or indexed
  // parameter loads.
  const long long rr = r0 + kH + lane, cc = c0 + kH + kW - 1 + lane;
  const double2* const sRU = R.U + rr;
  const double* const sRI = R.inv + rr;
  const long long* const sRK = PS.keyR + rr;
  const double2* const sCU = C.U + cc;
  const double* const sCI = C.inv + cc;
  const long long* const sCK = PS.keyC + cc;
  const long long rlim = R.L - rr, clim = C.L - cc;  // keys exist while ts < lim
  int px = (kH + kW - 1 + lane) % kRing;             // ring position of this lane's column
#endif
  for (int t = 0; t < nT; ++t) {
    const int buf = t & 1;
    const long long ts = (long long)t * kH;
#ifdef MPGPU_LANE_STREAMS
    const int pa = (px % kD) * kNB + px / kD;  // ring slot of the prefetched column
#endif
    // ---- prefetch tile t+1 (its ring slots held columns retired by now) ----
    if constexpr (kH <= 32) {
#ifdef MPGPU_LANE_STREAMS
      if (t + 1 < nT && lane < kH) {
        cp_async16(&S.rowU[buf ^ 1][lane], sRU + ts);
        cp_async8(&S.rowI[buf ^ 1][lane].x, sRI + ts);
        if (ts < rlim) cp_async8(&S.rowI[buf ^ 1][lane].y, sRK + ts);
        cp_async16(&S.colU[pa], sCU + ts);
        cp_async8(&S.colI[pa].x, sCI + ts);
        if (ts < clim) cp_async8(&S.colI[pa].y, sCK + ts);
      }
#else
      if (t + 1 < nT && lane < kH) {
        fetch_row(S, PS, buf ^ 1, lane, r0 + ts + kH + lane);
        fetch_col(S, PS, c0, ts + kH + kW - 1 + lane);
      }
#endif
    } else if (t + 1 < nT) {
#pragma unroll
      for (int h = lane; h < kH; h += 32) {
        fetch_row(S, PS, buf ^ 1, h, r0 + ts + kH + h);
        fetch_col(S, PS, c0, ts + kH + kW - 1 + h);
      }
    }

    // ---- compute the tile: kH rows x kD diagonals per lane ----------------
    // Blocks of kD row-steps run branch-free: each row-step only ORs its
    // filter result into `anyfire`, so loads and DFMAs of later row-steps
    // schedule freely across earlier ones. A block in which any lane fired
    // (a few percent) is replayed from its saved start state with the
    // per-row-step slow path; the arithmetic of every cell is identical.
    int b0 = (int)(((unsigned)ts / kD + lane) % (unsigned)kNB);
    for (int u = 0; u < kH; u += kD) {
      const int b1 = b0 + 1 == kNB ? 0 : b0 + 1;
#pragma unroll
      for (int s0 = 0; s0 < kD; s0 += kBlock) {
        double covs[kD];
#pragma unroll
        for (int d = 0; d < kD; ++d) covs[d] = cov[d];
        // Fire test: max_d hc[d] >= rthr (3-input integer max) or hc[d] >=
        // cthr[d] for some d; four predicate accumulators merged at block end.
        bool fa = false, fb = false, fc = false, fd = false;
#pragma unroll
        for (int s = s0; s < s0 + kBlock; ++s) {
          const int h = u + s;
          const int sin = (s + kD - 1) % kD;  // slot of the entering column
          {
            const int a = sin * kNB + (s == 0 ? b0 : b1);
            cU[sin] = S.colU[a];
            cpk[sin] = S.colI[a].y;
          }
          const double2 ru = S.rowU[buf][h];
          const double2 ri = S.rowI[buf][h];
          const int rthr = __double2hiint(ri.y);
          int hcs[kD];
#pragma unroll
          for (int d = 0; d < kD; ++d) {
            const int sl = (s + d) % kD;
            cov[d] = fma(ru.x, cU[sl].y, cov[d]);
            cov[d] = fma(ru.y, cU[sl].x, cov[d]);
            hcs[d] = __double2hiint(cov[d] * (ri.x * cpk[sl]));  // rinv*cinv off the cov chain
          }
          int rmax;
          if constexpr (kD == 12) {
            const int m1 = __vimax3_s32(hcs[0], hcs[1], hcs[2]);
            const int m2 = __vimax3_s32(hcs[3], hcs[4], hcs[5]);
            const int m3 = __vimax3_s32(hcs[6], hcs[7], hcs[8]);
            const int m4 = __vimax3_s32(hcs[9], hcs[10], hcs[11]);
            rmax = __vimax3_s32(m1, m2, max(m3, m4));
          } else if constexpr (kD == 16) {
            const int m1 = __vimax3_s32(hcs[0], hcs[1], hcs[2]);
            const int m2 = __vimax3_s32(hcs[3], hcs[4], hcs[5]);
            const int m3 = __vimax3_s32(hcs[6], hcs[7], hcs[8]);
            const int m4 = __vimax3_s32(hcs[9], hcs[10], hcs[11]);
            const int m5 = __vimax3_s32(hcs[12], hcs[13], hcs[14]);
            rmax = max(__vimax3_s32(m1, m2, m3), __vimax3_s32(m4, m5, hcs[15]));
          } else if constexpr (kD == 8) {
            const int m1 = __vimax3_s32(hcs[0], hcs[1], hcs[2]);
            const int m2 = __vimax3_s32(hcs[3], hcs[4], hcs[5]);
            const int m3 = __vimax3_s32(hcs[6], hcs[7], m1);
            rmax = max(m2, m3);
          } else {
            rmax = max(__vimax3_s32(hcs[0], hcs[1], hcs[2]), hcs[3]);
          }
          fa |= rmax >= rthr;
          bool* acc4[4] = {&fb, &fc, &fd, &fa};
#pragma unroll
          for (int d = 0; d < kD; ++d) *acc4[d & 3] |= hcs[d] >= __double2loint(cpk[(s + d) % kD]);
        }
        const bool anyfire = (fa | fb) | (fc | fd);
#ifdef MPGPU_EXPERIMENT_FASTONLY
        if (anyfire && cov[0] == 12345.0) {  // never: measures the fast blocks alone
#else
        if (__builtin_expect(__any_sync(0xffffffffu, anyfire), 0)) {
#endif
          // ---- replay the block with exact key updates ---------------------
          // (exact cinv from the ring; thresholds from the packed low words)
          if (stats && lane == 0) atomicAdd(&stats[3], 1ull);
          double cinv[kD];
          int cthr[kD];
#pragma unroll
          for (int d = 0; d < kD; ++d) cov[d] = covs[d];
#pragma unroll
          for (int q = 0; q < kD - 1; ++q) {  // block-start window: columns rho0 + lane*kD + q
            const int a = ((s0 + q) % kD) * kNB + (s0 + q >= kD ? b1 : b0);
            cU[(s0 + q) % kD] = S.colU[a];
            const double2 ci = S.colI[a];
            cinv[(s0 + q) % kD] = ci.x;
            cthr[(s0 + q) % kD] = __double2loint(ci.y);
          }
#pragma unroll
          for (int s = s0; s < s0 + kBlock; ++s) {
            const int h = u + s;
            const int sin = (s + kD - 1) % kD;
            {
              const int a = sin * kNB + (s == 0 ? b0 : b1);
              cU[sin] = S.colU[a];
              const double2 ci = S.colI[a];
              cinv[sin] = ci.x;
              cthr[sin] = __double2loint(ci.y);
            }
            const double2 ru = S.rowU[buf][h];
            const double2 ri = S.rowI[buf][h];
            const int rthr = __double2hiint(ri.y);
            SlowIn in;
            int hcs[kD], tmin[kD];
#pragma unroll
            for (int d = 0; d < kD; ++d) {
              const int sl = (s + d) % kD;
              cov[d] = fma(ru.x, cU[sl].y, cov[d]);
              cov[d] = fma(ru.y, cU[sl].x, cov[d]);
              in.c[d] = cov[d] * (ri.x * cinv[sl]);
              hcs[d] = __double2hiint(in.c[d]);
              tmin[d] = min(rthr, cthr[sl]);
            }
            const bool fire = any_ge(hcs, tmin);
            if (__any_sync(0xffffffffu, fire && ri.x != 0.0)) {
              unsigned live = 0;
              if (ri.x != 0.0) {
#pragma unroll
                for (int d = 0; d < kD; ++d) live |= (cinv[(s + d) % kD] != 0.0 ? 1u : 0u) << d;
              }
              if constexpr (kMasked) live &= dmask;
#pragma unroll
              for (int d = 0; d < kD; ++d) in.cthr[d] = cthr[(s + d) % kD];
              const long long rho = ts + h;
              const SlowOut o = slow_path(in, live, rthr, r0 + rho, rho + (long long)lane * kD, c0,
                                          h, buf, imask, PS.keyR, PS.keyC, stats);
#pragma unroll
              for (int d = 0; d < kD; ++d) cthr[(s + d) % kD] = o.cthr[d];
            }
          }
          // back to the fast pass: packed values of the carried slots (the
          // slow path may have raised their thresholds in the ring)
#pragma unroll
          for (int q = 0; q < kD - 1; ++q) {
            const int sq_ = (s0 + kBlock + q) % kD;
            cpk[sq_] = S.colI[sq_ * kNB + (s0 + kBlock + q >= kD ? b1 : b0)].y;
          }
        }
      }
      b0 = b1;
    }

    // ---- land the prefetch (warp-local) -------------------------------------
    if (t + 1 < nT) {
      cp_async_wait_all();
      if constexpr (kH <= 32) {
#ifdef MPGPU_LANE_STREAMS
        if (lane < kH) {
          const double2 vr = S.rowI[buf ^ 1][lane];
          const double tr = (ts < rlim && vr.x != 0.0) ? thr_filter(__double_as_longlong(vr.y), imask) : 2.0;
          S.rowI[buf ^ 1][lane].y = __hiloint2double(lower_thr(__double2hiint(tr)), 0);
          const double2 vc = S.colI[pa];
          const double tc = (ts < clim && vc.x != 0.0) ? thr_filter(__double_as_longlong(vc.y), imask) : 2.0;
          S.colI[pa].y = pack_col(vc.x, lower_thr(__double2hiint(tc)));
        }
#else
        if (lane < kH) {
          fix_row(S, PS, buf ^ 1, lane, r0 + ts + kH + lane, imask);
          fix_col(S, PS, c0, ts + kH + kW - 1 + lane, imask);
        }
#endif
      } else {
#pragma unroll
        for (int h = lane; h < kH; h += 32) {
          fix_row(S, PS, buf ^ 1, h, r0 + ts + kH + h, imask);
          fix_col(S, PS, c0, ts + kH + kW - 1 + h, imask);
        }
      }
    }
#ifdef MPGPU_LANE_STREAMS
    px += kH;
    if (px >= kRing) px -= kRing;
#endif
    __syncwarp();
  }
}

__global__ void __launch_bounds__(kThreads, kMinBlocks) k_join(const JoinParams P) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31;
  WarpSmem& S = reinterpret_cast<JoinSmem*>(smem_raw)->w[threadIdx.x >> 5];
  const long long imask = P.imask;
  const int m = P.m;
  if (lane == 0) S.zero = 0;
  __syncwarp();

  for (;;) {
    int item_id = 0;
    if (lane == 0) item_id = atomicAdd(P.counter, 1);
    item_id = __shfl_sync(0xffffffffu, item_id, 0);
    if (item_id >= P.n_items) break;
    const Item it = P.items[item_id];
    const Pass& PS = P.pass[it.pass];
    double cov[kD];
    seed_direct(S, PS.R, PS.C, it.r0, it.r0 + it.kb, m, lane, cov);
    walk_band<false>(S, PS, m, imask, P.stats, lane, it.r0, it.kb, it.nrows / kH, cov, 0u);
  }
}

// ---- K3m: the band join over a diagonal SUBSET (exact anytime SCRIMP, dense sets) ----
// SCRIMP's first s_size diagonals of its seeded order are a
// random subset. From about 9% of all diagonals on, nearly every band of kW
// holds some of them, and one diagonal per lane (k_diag_join) costs more than
// walking whole bands: this kernel is k_join over the bands that hold a chosen
// diagonal, with the other diagonals masked out (see kMaskedCov). Self-joins
// only. dmasks: one byte per lane and band, bit d = diagonal klo + 256 band +
// 8 lane + d is chosen.
struct MaskedParams {
  JoinParams J;
  const unsigned char* dmasks;
  long long klo;
};

__global__ void __launch_bounds__(kThreads, kMinBlocks) k_join_masked(const MaskedParams P) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31;
  WarpSmem& S = reinterpret_cast<JoinSmem*>(smem_raw)->w[threadIdx.x >> 5];
  if (lane == 0) S.zero = 0;
  __syncwarp();
  for (;;) {
    int item_id = 0;
    if (lane == 0) item_id = atomicAdd(P.J.counter, 1);
    item_id = __shfl_sync(0xffffffffu, item_id, 0);
    if (item_id >= P.J.n_items) break;
    const Item it = P.J.items[item_id];
    const Pass& PS = P.J.pass[0];
    const unsigned dmask = P.dmasks[((it.kb - P.klo) / kW) * 32 + lane];
    double cov[kD];
    seed_direct(S, PS.R, PS.C, it.r0, it.r0 + it.kb, P.J.m, lane, cov);
#pragma unroll
    for (int d = 0; d < kD; ++d)
      if (!((dmask >> d) & 1u)) cov[d] = __longlong_as_double((long long)kMaskedCov);
    walk_band<true>(S, PS, P.J.m, P.J.imask, P.J.stats, lane, it.r0, it.kb, it.nrows / kH, cov, dmask);
  }
}

// ---- K3d: anytime join over an explicit diagonal set (SCRIMP, exact s_size) ------
// SCRIMP evaluates s_size diagonals in a seeded order. The
// band kernel above needs 256 consecutive diagonals per warp; a random subset
// has no such runs, so this kernel gives every lane its own diagonal: a warp
// takes 32 consecutive entries of the sorted subset and a segment of rows.
// Each lane seeds its covariance by a direct centred dot product, then walks
// its rows with the join's recurrence. Row data are warp-broadcast loads;
// column data are per-lane sequential loads. Flat windows take the
// convention in-kernel (both flat: distance 0, one flat: sqrt(m)), so the
// keys are complete and the finalize only decodes them. Exact (no filter
// quantisation): a cell updates a key only when its packed key is smaller.
struct DiagItem {
  int group;  // diagonals diags[32 group + lane]
  int seg;    // rows [seg * rows, (seg + 1) * rows)
};

__global__ void __launch_bounds__(256, 2) k_diag_join(const Series A, long long* __restrict__ keyR,
                                                   long long* __restrict__ keyC,
                                                   const long long* __restrict__ diags,
                                                   long long n_diags, const DiagItem* __restrict__ items,
                                                   int n_items, int* __restrict__ counter, int rows,
                                                   int m, long long imask) {
  const int lane = threadIdx.x & 31;
  const double half_corr = 0.5;  // one flat window: d = sqrt(m) -> corr = 1 - d^2 / 2m = 1/2
  for (;;) {
    int id = 0;
    if (lane == 0) id = atomicAdd(counter, 1);
    id = __shfl_sync(0xffffffffu, id, 0);
    if (id >= n_items) break;
    const DiagItem it = items[id];
    const long long q = (long long)it.group * 32 + lane;
    const long long k = q < n_diags ? diags[q] : -1;
    const long long r0 = (long long)it.seg * rows;
    // rows of this lane: [r0, r1) with j = i + k < L
    const long long r1 = k >= 0 ? min(r0 + rows, A.L - k) : r0;
    double cov = 0.0;
    if (r1 > r0) {
      const double mi = A.mu[r0], mj = A.mu[r0 + k];
      const double* xi = A.x + r0;
      const double* xj = A.x + r0 + k;
      for (int t = 0; t < m; ++t) cov = fma(xi[t] - mi, xj[t] - mj, cov);
    }
    // the warp walks the longest lane's rows; shorter lanes idle at the end.
    // Rows go in batches of kDiagBatch: every load of a batch (the lane's
    // column data, the broadcast row data, the keys) is issued before the
    // batch's recurrence, so the dependent chain never waits on memory. All
    // addressing is 32-bit offsets from per-item base pointers, and a cell's
    // two keys share one score computation.
    long long rmax = r1;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) rmax = max(rmax, __shfl_xor_sync(0xffffffffu, rmax, o));
    const int nrows = (int)(rmax - r0);       // warp-uniform
    const int mine = (int)(r1 - r0);          // this lane's rows (0 when it has no diagonal)
    const long long jb = r0 + (k >= 0 ? k : 0);
    // per-lane streams, bumped by a batch each step: the loads use immediate
    // offsets. Reads run up to kDiagBatch - 1 entries past a stream's end into
    // the padding every statistics and key array carries (kPad entries).
    const double2* pRU = A.U + r0;
    const double* pRI = A.inv + r0;
    long long* pRK = keyR + r0;
    const double2* pCU = A.U + jb;
    const double* pCI = A.inv + jb;
    long long* pCK = keyC + jb;
    constexpr int kDiagBatch = 4;
    for (int q0 = 0; q0 < nrows; q0 += kDiagBatch) {
      double2 ru[kDiagBatch], cu[kDiagBatch];
      double ri[kDiagBatch], cj[kDiagBatch];
      long long kcur[kDiagBatch], rcur[kDiagBatch];
#pragma unroll
      for (int q = 0; q < kDiagBatch; ++q) {
        ru[q] = pRU[q];
        ri[q] = pRI[q];
        rcur[q] = pRK[q];
        cu[q] = pCU[q];
        cj[q] = pCI[q];
        kcur[q] = pCK[q];
      }
#pragma unroll
      for (int q = 0; q < kDiagBatch; ++q) {
        const int qq = q0 + q;
        if (qq >= nrows) break;  // warp-uniform
        const bool on = qq < mine;
        if (on && qq > 0) {
          cov = fma(ru[q].x, cu[q].y, cov);
          cov = fma(ru[q].y, cu[q].x, cov);
        }
        // score = 1 - corr, clamped at 0; flat windows take the convention
        // (both flat: 0, one flat: 1/2)
        const double nn = ri[q] * cj[q];
        double sc = 1.0 - cov * nn;
        sc = sc > 0.0 ? sc : 0.0;
        if (nn == 0.0) sc = (ri[q] == 0.0 && cj[q] == 0.0) ? 0.0 : 0.5;
        const long long sb = __double_as_longlong(sc) & ~imask;
        const long long kc = sb | (r0 + qq);          // column key: neighbour i
        long long kr = on ? (sb | (jb + qq)) : kKeyNone;  // row key: neighbour j
        if (on && kc < kcur[q]) red_min(pCK + q, kc);
        const long long cur = rcur[q];
        if (__any_sync(0xffffffffu, kr < cur)) {
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) {
            const long long v = __shfl_xor_sync(0xffffffffu, kr, o);
            kr = v < kr ? v : kr;
          }
          if (lane == 0 && kr < cur) red_min(pRK + q, kr);
        }
      }
      pRU += kDiagBatch;
      pRI += kDiagBatch;
      pRK += kDiagBatch;
      pCU += kDiagBatch;
      pCI += kDiagBatch;
      pCK += kDiagBatch;
    }
  }
}

// Decode keys that are complete (the diagonal-subset join): value at the
// best of the left / right keys, exact distance or flat convention; left /
// right indexes are not part of a partial result.
__global__ void k_finalize_keys(const Series A, const long long* __restrict__ key_right,
                                const long long* __restrict__ key_left, int m, long long imask,
                                double* __restrict__ mp, long long* __restrict__ pi,
                                long long* __restrict__ left, long long* __restrict__ right);

// ---- K2: warm-start keys -------------------------------------------------------
// Every row and column gets a real candidate before the join, so the join's
// filter never runs against an empty key (an empty key makes every warp that
// touches the row take the slow path). Cells on kInitDiag spread diagonals of
// each pass, evaluated by direct centred dot products; they are ordinary
// cells of the join, so min-merging them changes nothing but the filter.
// The launch picks the diagonal count (grid.y): up to kInitDiag, fewer for long
// windows where each cell's direct dot product costs more.
#ifndef MPGPU_INIT_DIAG
#define MPGPU_INIT_DIAG 32
#endif
constexpr int kInitDiag = MPGPU_INIT_DIAG;

// One warp per run of kInitRows consecutive rows of one diagonal: the warp
// computes the run's first covariance by a direct centred dot product (lanes
// split the m terms, butterfly sum), then 32 rows at a time each lane takes
// its row's recurrence increment df_R dg_C + dg_R df_C and an inclusive warp
// scan turns them into the 32 covariances (the recurrence summed as a tree).
// All loads are coalesced and no lane walks a long dependent chain. Seed
// points sit at multiples of kInitRows: they depend on the problem only,
// never on the shard count.
constexpr int kInitRows = 128;
constexpr int kInitWarps = 8;

__global__ void __launch_bounds__(kInitWarps * 32) k_init_keys(
    const Pass PS, long long klo, long long khi, int m, long long imask,
    const long long* __restrict__ diags, int b0, int bstride, int nb_total) {
  const int lane = threadIdx.x & 31;
  const long long i0 = ((long long)blockIdx.x * kInitWarps + (threadIdx.x >> 5)) * kInitRows;
  const int b = b0 + (int)blockIdx.y * bstride;  // this launch's share of the nb_total diagonals
  const Series& R = PS.R;
  const Series& C = PS.C;
  const long long span = khi - klo;
  if (span <= 0 || i0 >= R.L) return;  // whole warp
  // diagonal b: klo + b*span/nb (b = 0 is the first admissible diagonal), or
  // the b-th entry of an explicit list (anytime runs: diagonals of chosen bands)
  const long long k = diags ? diags[b] : klo + (span * b) / (long long)nb_total;
  const long long j0 = i0 + k;
  if (j0 >= C.L) return;
  const long long n = min((long long)kInitRows, min(R.L - i0, C.L - j0));
  const double mi = R.mu[i0], mj = C.mu[j0];
  const double* xi = R.x + i0;
  const double* xj = C.x + j0;
  double cov = 0.0;
  for (int t = lane; t < m; t += 32) cov = fma(xi[t] - mi, xj[t] - mj, cov);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) cov += __shfl_xor_sync(0xffffffffu, cov, o);
  for (long long s0 = 0; s0 < n; s0 += 32) {
    const long long s = s0 + lane;
    const long long i = i0 + s, j = j0 + s;
    const bool in = s < n;
    double inc = 0.0;
    if (in && s > 0) {
      const double2 ru = R.U[i], cu = C.U[j];
      inc = fma(ru.x, cu.y, ru.y * cu.x);
    }
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {  // inclusive scan of the increments
      const double v = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += v;
    }
    const double c_ij = cov + inc;
    cov = __shfl_sync(0xffffffffu, c_ij, 31);  // the next 32 rows continue from row s0 + 31
    if (!in) continue;
    const double ii = R.inv[i], ij = C.inv[j];
    if (ii == 0.0 || ij == 0.0) continue;
    const double c = c_ij * (ii * ij);
    red_min(&PS.keyR[i], mk_key(c, j, imask));
    red_min(&PS.keyC[j], mk_key(c, i, imask));
  }
}

// ---- K2b: coarse warm start -------------------------------------------------------
// A join on the PAA-downsampled series (factor f, window m/f) finds, for almost
// every window, a match close to its best; warm-starting the keys there keeps
// the join's filter from firing on the rising correlation runs that precede
// each row's and column's best (a fire costs a replayed block). The coarse keys
// are read directly (index = key & mask); each coarse pair (I, J) seeds the fine
// diagonals f(J - I) + delta, |delta| <= f, over rows f*I .. f*I + f - 1: one
// direct centred dot product, then the join's recurrence. Like K2 these are
// real cells of the join, so they change the filter, never the answer.
__global__ void k_paa(const double* __restrict__ x, long long nc, int f, double* __restrict__ xc) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= nc) return;
  double s = 0.0;
  for (int q = 0; q < f; ++q) s += x[t * f + q];
  xc[t] = s / f;
}

// One warp per coarse window I: the nd fine diagonals around its match share
// one row window, so their seeds are nd sliding dot products of that window
// against one column span. The warp stages the centred row window and the
// span in shared memory chunk by chunk (as k_join's segment seeds) and lane
// l accumulates diagonals l, l + 32, ... (up to kExpGroups per pass over
// blocks of 32 kExpGroups diagonals). Then each lane walks its diagonals for
// f rows with the join's recurrence, RED.MINing into the keys. Diagonals that
// start above the series (j0 < 0) or lie in the exclusion zone are skipped or
// seeded where they enter, exactly as before.
constexpr int kExpWarps = 4;
constexpr int kExpGroups = 1;
constexpr int kExpSpan = 32 * kExpGroups;  // diagonals per pass (one per lane)
constexpr int kExpT = 8;                   // seed terms per lane per chunk
constexpr int kExpChunk = 32 * kExpT;      // seed terms per chunk (256)

constexpr int kExpWalk = 32;  // rows staged per walk chunk

struct ExpSmem {
  union {
    struct {  // seeds: centred row window chunk, column span chunk
      double a[kExpChunk];
      double y[kExpChunk + kExpSpan];
    } seed;
    double red[32][kExpSpan + 1];  // per-lane partial seeds, padded rows (conflict-free)
    struct {  // walk: rows [qc, qc + kExpWalk), the columns they meet
      double2 rU[kExpWalk];
      double rI[kExpWalk];
      double2 cU[kExpSpan + kExpWalk];
      double cI[kExpSpan + kExpWalk];
    } walk;
  };
};

// One warp per coarse window I: the nd fine diagonals around its match share
// one row window, so their seeds are nd sliding dot products of that window
// against one column span. The m terms are split across the lanes (lane l
// takes terms [8l, 8l + 8) of every 256-term chunk, with the 39 column values
// they meet in registers), every lane accumulates all 32 diagonals of a pass,
// and a transposed sum through shared memory leaves diagonal l's seed in lane
// l: 8 x 32 FMAs per lane per chunk instead of 256 serial FMAs with half the
// lanes idle. Then each lane walks its diagonal for f rows with the join's
// recurrence, RED.MINing into the keys (one warp-min RED per row).
__global__ void __launch_bounds__(kExpWarps * 32) k_coarse_exploit(
    const Pass PS, const long long* __restrict__ ckey, long long I0, long long I1, long long cimask,
    bool key_is_col, int f, int span, long long zone, bool self, int m, long long imask,
    const unsigned* __restrict__ band_mask, const unsigned* __restrict__ diag_bits) {
  __shared__ ExpSmem sm[kExpWarps];
  ExpSmem& S = sm[threadIdx.x >> 5];
  const int lane = threadIdx.x & 31;
  const long long I = I0 + (long long)blockIdx.x * kExpWarps + (threadIdx.x >> 5);
  if (I >= I1) return;  // whole warp
  const long long kc = ckey[I];
  if (kc == kKeyNone) return;
  const long long J = kc & cimask;
  const long long Ir = key_is_col ? J : I, Jc = key_is_col ? I : J;
  const long long i0 = Ir * f;
  const long long jbase = Jc * f - span;  // column start of diagonal offset 0
  const Series& R = PS.R;
  const Series& C = PS.C;
  const int nd = 2 * span + 1;
  if (i0 >= R.L) return;
  const double mi = R.mu[i0];
  for (int d0 = 0; d0 < nd; d0 += kExpSpan) {
    constexpr int ng = 1;
    // seeds of diagonals d0 .. d0 + 31 at row i0 (columns jbase + d0 + d)
    double part[kExpSpan];
#pragma unroll
    for (int d = 0; d < kExpSpan; ++d) part[d] = 0.0;
    double asum_l = 0.0;
    for (int t0 = 0; t0 < m; t0 += kExpChunk) {
      const int tc = min(kExpChunk, m - t0);
      for (int q = lane; q < kExpChunk; q += 32) S.seed.a[q] = q < tc ? R.x[i0 + t0 + q] - mi : 0.0;
      for (int q = lane; q < kExpChunk + kExpSpan; q += 32) {
        const long long gidx = jbase + d0 + t0 + q;
        S.seed.y[q] = (q < tc + kExpSpan && gidx >= 0 && gidx < C.n) ? C.x[gidx] : 0.0;
      }
      __syncwarp();
      double av[kExpT], yv[kExpT + kExpSpan - 1];
#pragma unroll
      for (int tt = 0; tt < kExpT; ++tt) {
        av[tt] = S.seed.a[lane * kExpT + tt];
        asum_l += av[tt];
      }
#pragma unroll
      for (int u = 0; u < kExpT + kExpSpan - 1; ++u) yv[u] = S.seed.y[lane * kExpT + u];
#pragma unroll
      for (int tt = 0; tt < kExpT; ++tt)
#pragma unroll
        for (int d = 0; d < kExpSpan; ++d) part[d] = fma(av[tt], yv[tt + d], part[d]);
      __syncwarp();
    }
    // transposed sum: lane d collects every lane's partial of diagonal d
#pragma unroll
    for (int d = 0; d < kExpSpan; ++d) S.red[lane][d] = part[d];
    __syncwarp();
    double acc[kExpGroups];
    acc[0] = 0.0;
#pragma unroll 8
    for (int l = 0; l < 32; ++l) acc[0] += S.red[l][lane];
    double asum = asum_l;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) asum += __shfl_xor_sync(0xffffffffu, asum, o);
    __syncwarp();
    // per lane and group: the diagonal's first row q0 and end qn (q0 >= qn: skip)
    long long q0s[kExpGroups], qns[kExpGroups];
#pragma unroll
    for (int g = 0; g < kExpGroups; ++g) {
      const int d = d0 + lane + 32 * g;
      const long long j0 = jbase + d;
      long long q0 = j0 < 0 ? -j0 : 0, qn = f;
      qn = min(qn, R.L - i0);
      qn = min(qn, C.L - j0);
      if (d >= nd || g >= ng || (self && j0 - i0 <= zone)) q0 = qn = 0;  // none / in the zone
      if (band_mask && q0 < qn) {  // anytime band subset: only the chosen bands' diagonals
        const long long b = (j0 - i0 - zone - 1) / kW;
        if (!((band_mask[b >> 5] >> (b & 31)) & 1u)) q0 = qn = 0;
      }
      if (diag_bits && q0 < qn) {  // anytime diagonal subset (masked bands): chosen diagonals only
        const long long k = j0 - i0;
        if (!((diag_bits[k >> 5] >> (k & 31)) & 1u)) q0 = qn = 0;
      }
      q0s[g] = q0;
      qns[g] = qn;
      if (q0 >= qn) continue;
      if (q0 == 0) {
        acc[g] = fma(-C.mu[j0], asum, acc[g]);
      } else {  // enters below the first row: direct seed where it starts
        const long long is = i0 + q0, js = j0 + q0;
        const double mis = R.mu[is], mjs = C.mu[js];
        double c0 = 0.0;
        for (int t = 0; t < m; ++t) c0 = fma(R.x[is + t] - mis, C.x[js + t] - mjs, c0);
        acc[g] = c0;
      }
    }
    __syncwarp();
    // walk f rows in chunks: the rows' and columns' update vectors and inverse
    // norms are staged by the warp (one round trip per chunk instead of one
    // per row), then every lane steps its diagonals through the chunk
    for (int qc = 0; qc < f; qc += kExpWalk) {
      for (int q = lane; q < kExpWalk; q += 32) {
        const long long i = i0 + qc + q;
        const bool in = i < R.L;
        S.walk.rU[q] = in ? R.U[i] : make_double2(0.0, 0.0);
        S.walk.rI[q] = in ? R.inv[i] : 0.0;
      }
      for (int q = lane; q < 32 * ng + kExpWalk; q += 32) {
        const long long j = jbase + d0 + qc + q;
        const bool in = j >= 0 && j < C.L;
        S.walk.cU[q] = in ? C.U[j] : make_double2(0.0, 0.0);
        S.walk.cI[q] = in ? C.inv[j] : 0.0;
      }
      __syncwarp();
#pragma unroll
      for (int g = 0; g < kExpGroups; ++g) {
        if (g >= ng) continue;  // warp-uniform
        const long long q0 = q0s[g], qn = qns[g];
        const int dl = lane + 32 * g;  // diagonal offset within this block
        const int qe = min(kExpWalk, f - qc);
        double cov = acc[g];
        for (int r = 0; r < qe; ++r) {  // warp-uniform trip count (row i0 + qc + r)
          const long long q = qc + r;
          const bool on = q >= q0 && q < qn;
          if (on && q > q0) {
            const double2 ru = S.walk.rU[r], cu = S.walk.cU[dl + r];
            cov = fma(ru.x, cu.y, cov);
            cov = fma(ru.y, cu.x, cov);
          }
          const double ii = S.walk.rI[r], ij = S.walk.cI[dl + r];
          const bool live = on && ii != 0.0 && ij != 0.0;
          const double c = cov * (ii * ij);
          const long long i = i0 + q, j = jbase + d0 + dl + q;
          if (live) red_min(&PS.keyC[j], mk_key(c, i, imask));
          // every lane's cell of this row targets keyR[i]: one RED of the warp's minimum
          long long kr = live ? mk_key(c, j, imask) : kKeyNone;
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) {
            const long long v = __shfl_xor_sync(0xffffffffu, kr, o);
            kr = v < kr ? v : kr;
          }
          if (lane == 0 && kr != kKeyNone) red_min(&PS.keyR[i], kr);
        }
        acc[g] = cov;
      }
      __syncwarp();
    }
  }
}

// ---- K6: distance-profile batch (MASS, distance.hpp:26-33) --------------------
// Q query windows against every window of a series: out[q][j] = z-normalised
// distance, flat-window convention, |j - pos_q| <= zone -> +inf for queries
// taken from the series itself. Direct centred dot products (exact; no FFT):
// cov = sum_t a_t x_{j+t} - mu_j sum_t a_t with a = query - mean(query).
// Each CTA owns one query and a span of kMassTile outputs; each thread owns
// kMassR consecutive outputs and slides a register window over the staged
// series (1 shared load per kMassR DFMAs). Near-zero hits are recomputed
// directly so exact matches come out as 0 (distance.hpp:30-33).
#ifndef MPGPU_MASS_THREADS
#define MPGPU_MASS_THREADS 128
#endif
constexpr int kMassThreads = MPGPU_MASS_THREADS;
#ifndef MPGPU_MASS_R
#define MPGPU_MASS_R 16
#endif
constexpr int kMassR = MPGPU_MASS_R;
constexpr int kMassTile = kMassThreads * kMassR;  // outputs per CTA (1024)
constexpr int kMassChunk = 512;                   // query samples staged per pass
static_assert(kMassChunk % kMassR == 0, "query chunks in whole register-window rotations");
// padded staging index: one gap per kMassR doubles, so lane l reading element
// kMassR*l + c hits bank pair 2*(9l + c') -- conflict-free 2-wavefront loads
__device__ __forceinline__ int mass_pad(int x) { return x + x / kMassR; }
constexpr int kMassSx = kMassTile + kMassChunk + kMassR;
constexpr int kMassSxPad = kMassSx + kMassSx / kMassR + 1;

// Per-query statistics, once per query: mean, inverse norm (0 when flat) and
// the sum of the centred samples, with the same sequential two-pass as K1, so
// a query equal to a window of the series gets bit-identical statistics
// (exact 0 on self-matches).
// One warp per query: the lanes stage the query in shared memory (parallel
// loads), lane 0 then adds in K1's sequential order, so the sums are bit for
// bit those of a thread walking the window alone.
constexpr int kQStatChunk = 1024;
constexpr int kQStatWarps = 4;
__global__ void __launch_bounds__(kQStatWarps * 32) k_query_stats(
    const double* __restrict__ x, const double* __restrict__ queries,
    const long long* __restrict__ qpos, int n_queries, int m, double* __restrict__ qstat) {
  __shared__ double buf[kQStatWarps][kQStatChunk];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int q = blockIdx.x * kQStatWarps + w;
  if (q >= n_queries) return;  // whole warp
  const double* qx = queries ? queries + (long long)q * m : x + qpos[q];
  double s = 0.0;
  for (int t0 = 0; t0 < m; t0 += kQStatChunk) {
    const int tc = min(kQStatChunk, m - t0);
    for (int t = lane; t < tc; t += 32) buf[w][t] = qx[t0 + t];
    __syncwarp();
    if (lane == 0)
      for (int t = 0; t < tc; ++t) s += buf[w][t];
    __syncwarp();
  }
  const double mean = __shfl_sync(0xffffffffu, s, 0) / (double)m;
  double ss = 0.0, asum = 0.0;
  for (int t0 = 0; t0 < m; t0 += kQStatChunk) {
    const int tc = min(kQStatChunk, m - t0);
    for (int t = lane; t < tc; t += 32) buf[w][t] = qx[t0 + t];
    __syncwarp();
    if (lane == 0)
      for (int t = 0; t < tc; ++t) {
        const double d = buf[w][t] - mean;
        ss = fma(d, d, ss);
        asum += d;
      }
    __syncwarp();
  }
  if (lane == 0) {
    const double sd = sqrt(ss / (double)m);
    const double scale = fabs(mean) > 1.0 ? fabs(mean) : 1.0;
    qstat[3 * q + 0] = mean;
    qstat[3 * q + 1] = sd <= 1e-10 * scale ? 0.0 : 1.0 / sqrt(ss);
    qstat[3 * q + 2] = asum;
  }
}

// The query sample is the operand all lanes (and a thread's kMassR outputs)
// share. From shared memory it is a vector register, and a DFMA with three
// vector-register sources is bound by register-file reads on sm_100 (DESIGN.md
// §6); from constant memory at a uniform index it is a uniform-register
// operand. So the centred queries of a launch are staged in c_mass_q (56 KB;
// k_mass_stage + a device-to-device copy into the symbol), kConst = true, as
// many queries per launch as fit; windows too long for it keep the
// shared-memory form.
constexpr int kMassConst = 7168;
__constant__ double c_mass_q[kMassConst];

// stage[qc * mpad + t] = query (q0 + qc)'s sample t, centred; 0 for t in [m, mpad)
__global__ void k_mass_stage(const double* __restrict__ x, const double* __restrict__ queries,
                             const long long* __restrict__ qpos, const double* __restrict__ qstat,
                             int q0, int nq, int m, int mpad, double* __restrict__ stage) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= nq * mpad) return;
  const int qc = idx / mpad, t = idx - qc * mpad, q = q0 + qc;
  const double* qx = queries ? queries + (long long)q * m : x + qpos[q];
  stage[idx] = t < m ? qx[t] - qstat[3 * q + 0] : 0.0;
}

template <bool kConst>
__global__ void __launch_bounds__(kMassThreads) k_mass(
    const double* __restrict__ x, long long n, const double* __restrict__ mu,
    const double* __restrict__ inv, long long L, int m, const double* __restrict__ queries,
    const long long* __restrict__ qpos, const double* __restrict__ qstat, long long zone,
    double* __restrict__ out, int q0, int mpad) {
  __shared__ double sq[kConst ? 1 : kMassChunk];
  __shared__ double sx[kMassSxPad];
  const int q = q0 + blockIdx.y;
  const int qoff = blockIdx.y * mpad;  // kConst: this query's samples in c_mass_q (uniform)
  const long long j0 = (long long)blockIdx.x * kMassTile;
  const int tid = threadIdx.x;
  const double* qx = queries ? queries + (long long)q * m : x + qpos[q];
  const double qmean = qstat[3 * q + 0], qinv = qstat[3 * q + 1], asum = qstat[3 * q + 2];
  double acc[kMassR];
#pragma unroll
  for (int r = 0; r < kMassR; ++r) acc[r] = 0.0;
  const int jl = tid * kMassR;  // first local output of this thread
  for (int t0 = 0; t0 < m; t0 += kMassChunk) {
    const int tc = min(kMassChunk, m - t0);
    const int tcp = (tc + kMassR - 1) / kMassR * kMassR;  // zero-padded query tail
    if constexpr (!kConst)
      for (int t = tid; t < tcp; t += kMassThreads) sq[t] = t < tc ? qx[t0 + t] - qmean : 0.0;
    for (int t = tid; t < kMassTile + tcp; t += kMassThreads) {
      const long long g = j0 + t0 + t;
      sx[mass_pad(t)] = g < n ? x[g] : 0.0;
    }
    __syncthreads();
    // rotating register window: slot (t + r) % kMassR holds x[jl + t + r]
    double w[kMassR];
#pragma unroll
    for (int r = 0; r < kMassR; ++r) w[r] = sx[mass_pad(jl + r)];
    for (int t8 = 0; t8 < tcp; t8 += kMassR) {
#pragma unroll
      for (int s = 0; s < kMassR; ++s) {
        const double a = kConst ? c_mass_q[qoff + t0 + t8 + s] : sq[t8 + s];
#pragma unroll
        for (int r = 0; r < kMassR; ++r) acc[r] = fma(a, w[(s + r) % kMassR], acc[r]);
        w[s] = sx[mass_pad(jl + kMassR + t8 + s)];  // x[jl + t + 8] replaces x[jl + t]
      }
    }
    __syncthreads();
  }
  const long long p = qpos ? qpos[q] : -1;
#pragma unroll
  for (int r = 0; r < kMassR; ++r) {
    const long long j = j0 + jl + r;
    if (j >= L) break;
    double d;
    const double ij = inv[j];
    if (p >= 0 && llabs(j - p) <= zone) {
      d = INFINITY;
    } else if (qinv == 0.0 || ij == 0.0) {
      d = (qinv == 0.0 && ij == 0.0) ? 0.0 : sqrt((double)m);
    } else {
      const double corr = fma(-mu[j], asum, acc[r]) * (qinv * ij);
      double d2 = 2.0 * m * (1.0 - corr);
      if (d2 < 1e-6) {  // near-zero hit: recompute directly (distance.hpp:30-33)
        const double* xj = x + j;
        const double mj = mu[j];
        double e = 0.0;
        for (int t = 0; t < m; ++t) {
          // rounded products (no FMA contraction): identical windows give exactly 0
          const double u = __dmul_rn(qx[t] - qmean, qinv) - __dmul_rn(xj[t] - mj, ij);
          e = fma(u, u, e);
        }
        d2 = (double)m * e;
      }
      d2 = d2 < 0.0 ? 0.0 : (d2 > 4.0 * m ? 4.0 * m : d2);
      d = sqrt(d2);
    }
    out[(long long)q * L + j] = d;
  }
}

// ---- K7: matrix-profile consumers (discovery.hpp:61-79) -----------------------
// FLUSS arc count: every nearest-neighbour arc (i, index[i]) adds +1 on the open
// interval strictly between its endpoints (a +1/-1 sweep, discovery.hpp:68-70):
// +1 at lo + 1, -1 at hi, for hi - lo >= 2. One of the two ends is always next
// to the arc's own window: +1 at i + 1 when index[i] > i, -1 at i when
// index[i] < i. That end is computed in the scan passes from index[k - 1] and
// index[k] (coalesced, no atomic); only the far end is a random RED.ADD into a
// 32-bit difference array (4 B per window, L2-resident up to L ~ 2^24).
__device__ __forceinline__ bool arc_ok(long long i, long long j, long long L) {
  return j >= 0 && j < L && (j - i >= 2 || i - j >= 2);
}

__global__ void k_arc_far_ends(const long long* __restrict__ index, long long L,
                               int* __restrict__ diff) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= L) return;
  const long long j = index[i];
  if (!arc_ok(i, j, L)) return;
  if (j > i) {
    asm volatile("red.relaxed.gpu.global.add.s32 [%0], %1;" ::"l"(diff + j), "r"(-1));
  } else {
    asm volatile("red.relaxed.gpu.global.add.s32 [%0], %1;" ::"l"(diff + j + 1), "r"(1));
  }
}

// diff[k] plus the near ends at k: +1 from the arc of window k - 1 pointing
// right, -1 from the arc of window k pointing left.
__device__ __forceinline__ long long arc_delta(const long long* __restrict__ index,
                                               const int* __restrict__ diff, long long k, long long L) {
  long long v = diff[k];
  const long long jk = index[k];
  if (arc_ok(k, jk, L) && jk < k) v -= 1;
  if (k > 0) {
    const long long jp = index[k - 1];
    if (arc_ok(k - 1, jp, L) && jp > k - 1) v += 1;
  }
  return v;
}

// Inclusive prefix sum of the arc-end differences, in three coalesced passes:
// per-tile sums, a scan of the tile sums, then each tile rescanned with its
// offset. The last pass also writes the corrected arc curve (CAC), so the arc
// counts are written once.
constexpr int kScanThreads = 256;
constexpr int kScanPer = 16;
constexpr int kScanTile = kScanThreads * kScanPer;  // 4096 windows per block

__global__ void __launch_bounds__(kScanThreads) k_scan_tile_sums(const long long* __restrict__ index,
                                                                 const int* __restrict__ diff,
                                                                 long long L,
                                                                 long long* __restrict__ sums) {
  __shared__ long long ws[kScanThreads / 32];
  const long long base = (long long)blockIdx.x * kScanTile;
  long long s = 0;
#pragma unroll
  for (int q = 0; q < kScanPer; ++q) {
    const long long i = base + q * kScanThreads + threadIdx.x;
    if (i < L) s += arc_delta(index, diff, i, L);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    long long t = 0;
    for (int w = 0; w < kScanThreads / 32; ++w) t += ws[w];
    sums[blockIdx.x] = t;
  }
}

// Exclusive scan of the n tile sums in one block of 1024 threads (n = L / 4096:
// 2048 at 2^23): each thread sums a contiguous chunk, the chunk totals are
// scanned with warp shuffles, then each chunk is rewritten with its offset.
__global__ void __launch_bounds__(1024) k_scan_sums(long long* __restrict__ sums, long long n) {
  __shared__ long long wtot[32];
  const int t = threadIdx.x, nt = blockDim.x;
  const long long chunk = (n + nt - 1) / nt;
  const long long lo = t * chunk, hi = lo + chunk < n ? lo + chunk : n;
  long long s = 0;
  for (long long i = lo; i < hi; ++i) s += sums[i];
  long long x = s;  // inclusive warp scan
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const long long y = __shfl_up_sync(0xffffffffu, x, o);
    if ((t & 31) >= o) x += y;
  }
  if ((t & 31) == 31) wtot[t >> 5] = x;
  __syncthreads();
  if (t < 32) {
    long long w = wtot[t], v = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const long long y = __shfl_up_sync(0xffffffffu, v, o);
      if (t >= o) v += y;
    }
    wtot[t] = v - w;  // exclusive over warps
  }
  __syncthreads();
  long long run = wtot[t >> 5] + (x - s);
  for (long long i = lo; i < hi; ++i) {
    const long long v = sums[i];
    sums[i] = run;
    run += v;
  }
}

// Corrected arc curve: arc / (2 i (L - i) / L), clamped to [0, 1], 1 within
// `window` of either end (discovery.hpp:72-74).
__device__ __forceinline__ double cac_of(long long arcs, long long i, long long L, long long window) {
  double v = 1.0;
  if (i >= window && i < L - window) {
    const double ideal = 2.0 * (double)i * (double)(L - i) / (double)L;
    v = ideal > 0.0 ? (double)arcs / ideal : 1.0;
    v = v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v);
  }
  return v;
}

__global__ void __launch_bounds__(kScanThreads) k_scan_tile_apply(const long long* __restrict__ index,
                                                                  const int* __restrict__ diff,
                                                                  long long L,
                                                                  const long long* __restrict__ offs,
                                                                  long long window,
                                                                  long long* __restrict__ a,
                                                                  double* __restrict__ cac) {
  // rows of kScanPer entries padded to kScanPer + 1: the coalesced phase writes
  // consecutive words, and the per-thread row reads of a half-warp hit 16
  // distinct 8-byte banks
  static_assert(kScanPer == 16, "padding written for 16 entries per thread");
  __shared__ long long tile[kScanTile / kScanPer * (kScanPer + 1)];
  __shared__ long long ws[kScanThreads / 32];
  auto P = [](int k) { return (k >> 4) * (kScanPer + 1) + (k & 15); };
  const long long base = (long long)blockIdx.x * kScanTile;
#pragma unroll
  for (int q = 0; q < kScanPer; ++q) {  // coalesced load
    const int k = q * kScanThreads + threadIdx.x;
    tile[P(k)] = base + k < L ? arc_delta(index, diff, base + k, L) : 0;
  }
  __syncthreads();
  // each thread scans kScanPer consecutive entries
  long long v[kScanPer];
  long long s = 0;
#pragma unroll
  for (int q = 0; q < kScanPer; ++q) {
    s += tile[threadIdx.x * (kScanPer + 1) + q];
    v[q] = s;
  }
  // exclusive scan of the thread totals across the block
  long long x = s;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const long long y = __shfl_up_sync(0xffffffffu, x, o);
    if ((threadIdx.x & 31) >= o) x += y;
  }
  if ((threadIdx.x & 31) == 31) ws[threadIdx.x >> 5] = x;
  __syncthreads();
  long long wpre = 0;
  for (int w = 0; w < (threadIdx.x >> 5); ++w) wpre += ws[w];
  const long long pre = offs[blockIdx.x] + wpre + (x - s);
#pragma unroll
  for (int q = 0; q < kScanPer; ++q) tile[threadIdx.x * (kScanPer + 1) + q] = v[q] + pre;
  __syncthreads();
#pragma unroll
  for (int q = 0; q < kScanPer; ++q) {  // coalesced store (+ the CAC)
    const int k = q * kScanThreads + threadIdx.x;
    const long long i = base + k;
    if (i < L) {
      const long long arcs = tile[P(k)];
      __stcs(a + i, arcs);
      if (cac) __stcs(cac + i, cac_of(arcs, i, L, window));
    }
  }
}

// Block-level arg-extreme of v (finite entries; ties -> smallest index) into
// one packed key per block; sign = +1 for max, -1 for min. Keys are reduced by
// a second launch of the same kernel over the per-block results.
__device__ __forceinline__ bool better(double a, long long ia, double b, long long ib, int sign) {
  if (ia < 0) return false;
  if (ib < 0) return true;
  if (a != b) return sign > 0 ? a > b : a < b;
  return ia < ib;
}

__global__ void k_argext(const double* __restrict__ v, const long long* __restrict__ vi,
                         long long n, int sign, double* __restrict__ out_v,
                         long long* __restrict__ out_i) {
  __shared__ double sv[32];
  __shared__ long long si[32];
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  double bv = 0.0;
  long long bi = -1;
  if (i < n) {
    const double x = v[i];
    const long long xi = vi ? vi[i] : i;
    if (isfinite(x) && xi >= 0) { bv = x; bi = xi; }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
    const long long oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (better(ov, oi, bv, bi, sign)) { bv = ov; bi = oi; }
  }
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) { sv[w] = bv; si[w] = bi; }
  __syncthreads();
  if (w == 0) {
    const int nw = blockDim.x >> 5;
    bv = lane < nw ? sv[lane] : 0.0;
    bi = lane < nw ? si[lane] : -1;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const long long oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (better(ov, oi, bv, bi, sign)) { bv = ov; bi = oi; }
    }
    if (lane == 0) { out_v[blockIdx.x] = bv; out_i[blockIdx.x] = bi; }
  }
}

// Mask |i - c| <= zone with `fill` (+inf to exclude from minima, -inf / NaN-free
// sentinel for maxima).
__global__ void k_mask_zone(double* __restrict__ v, long long n, long long c, long long zone,
                            double fill) {
  const long long i = (c - zone > 0 ? c - zone : 0) + blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n && i <= c + zone) v[i] = fill;
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
// Finalize kernels decode kFinG windows per warp, kFinLanes lanes each: the
// key loads, the neighbour's statistics and its window of every group are in
// flight together (one window per warp left each warp waiting on three
// dependent memory round trips in turn).
constexpr int kFinG = 4;
constexpr int kFinLanes = 32 / kFinG;

// Exact z-normalised distance of window i of X and window j of Y by a group of
// kFinLanes lanes (sub = lane within the group): d^2 = m * sum_t ((x_t - mu_i)
// inv_i - (y_t - mu_j) inv_j)^2. Every lane of the warp must call it (the
// group reduction shuffles the full warp); exact == false contributes 0.
__device__ __forceinline__ double group_exact_dist(const Series& X, long long i, const Series& Y,
                                                   long long j, bool exact, int m, int sub) {
  double acc = 0.0;
  if (exact) {
    const double mi = X.mu[i], ii = X.inv[i], mj = Y.mu[j], ij = Y.inv[j];
    const double* xi = X.x + i;
    const double* yj = Y.x + j;
#pragma unroll 4
    for (int t = sub; t < m; t += kFinLanes) {
      // rounded products (no FMA contraction): identical windows give exactly 0
      const double d = __dmul_rn(xi[t] - mi, ii) - __dmul_rn(yj[t] - mj, ij);
      acc = fma(d, d, acc);
    }
  }
#pragma unroll
  for (int o = kFinLanes / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  double d2 = (double)m * acc;
  const double cap = 4.0 * (double)m;
  d2 = d2 > cap ? cap : d2;
  return sqrt(d2);
}

// Value at the chosen neighbour bi (-1: none): +inf, the flat-window
// convention (distance.hpp:14-15), or the exact distance. Warp-collective.
__device__ __forceinline__ double group_value(const Series& X, long long i, const Series& Y,
                                              long long bi, bool valid, int m, int sub) {
  const bool have = valid && bi >= 0;
  const bool fi = have && X.inv[i] == 0.0, fj = have && Y.inv[bi] == 0.0;
  const double e = group_exact_dist(X, i, Y, bi, have && !fi && !fj, m, sub);
  if (!have) return INFINITY;
  if (fi && fj) return 0.0;
  if (fi || fj) return sqrt((double)m);
  return e;
}

// Self-join: window i has right key (row keys) and left key (column keys).
__global__ void k_finalize_self(const Series A, const long long* __restrict__ key_right,
                                const long long* __restrict__ key_left, long long zone, int m,
                                long long imask, long long row0, long long row1,
                                double* __restrict__ mp, long long* __restrict__ pi,
                                long long* __restrict__ left, long long* __restrict__ right) {
  const long long gi = (blockIdx.x * (long long)blockDim.x + threadIdx.x) / kFinLanes;
  const int sub = threadIdx.x % kFinLanes;
  const long long i = row0 + gi;
  const bool valid = i < row1;
  const long long L = A.L;
  const long long ic = valid ? i : row0;  // out-of-range groups mirror a valid window
  long long rk = key_right[ic], lk = key_left[ic];
  const double half = 0.5;
  const long long rlo = ic + zone + 1;  // smallest admissible right neighbour
  const long long lhi = ic - zone - 1;  // largest admissible left neighbour
  const long long nf_r = rlo < L ? next_flat(A, rlo) : -1;
  const long long f0 = next_flat(A, 0);
  const bool nf_l = f0 >= 0 && f0 <= lhi;
  if (A.inv[ic] == 0.0) {  // flat window: distances are 0 (flat) or sqrt(m)
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
  const double v = group_value(A, ic, A, bi, valid, m, sub);
  if (valid && sub == 0) {
    if (mp) mp[i] = v;
    if (pi) pi[i] = bi;
    if (left) left[i] = lk == kKeyNone ? -1 : (lk & imask);
    if (right) right[i] = rk == kKeyNone ? -1 : (rk & imask);
  }
}

// Self-join finalize for an anytime (partial) run: only diagonals inside the
// computed bands [bands[q], bands[q] + kW) count, so the flat-window
// candidates are searched band by band (SCRIMP partial coverage,
// SPEC.md:218-223). left/right are absent below full coverage.
__global__ void k_finalize_self_partial(const Series A, const long long* __restrict__ key_right,
                                        const long long* __restrict__ key_left, int m,
                                        long long imask, const long long* __restrict__ bands,
                                        int n_bands, long long khi, double* __restrict__ mp,
                                        long long* __restrict__ pi, long long* __restrict__ left,
                                        long long* __restrict__ right) {
  const long long i = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (i >= A.L) return;
  const long long L = A.L;
  long long rk = key_right[i], lk = key_left[i];
  const bool fi = A.inv[i] == 0.0;
  // Smallest flat window and smallest admissible neighbour inside the chosen
  // bands, on either side. The 32 lanes split the bands (each lane's share is
  // ascending, so a lane stops at its first hit) and the warp takes the minima.
  // Without any flat window in the series there is nothing to search.
  constexpr long long kNoIdx = 0x7fffffffffffffffLL;
  long long rflat = kNoIdx, rany = kNoIdx, lflat = kNoIdx, lany = kNoIdx;
  if (next_flat(A, 0) >= 0) {
    // right neighbours j = i + k
    for (int q = lane; q < n_bands; q += 32) {
      const long long lo = i + bands[q];
      const long long hi = min(i + min(bands[q] + kW, khi), L);  // exclusive
      if (lo >= hi) continue;
      rany = min(rany, lo);
      const long long f = next_flat(A, lo);
      if (f >= 0 && f < hi) { rflat = f; break; }
    }
    // left neighbours j = i - k (band q covers j in [lo, hi))
    for (int q = n_bands - 1 - lane; q >= 0; q -= 32) {
      const long long lo = max(0LL, i - (min(bands[q] + kW, khi) - 1));
      const long long hi = i - bands[q] + 1;  // exclusive
      if (lo >= hi) continue;
      lany = min(lany, lo);
      const long long f = next_flat(A, lo);
      if (f >= 0 && f < hi) { lflat = f; break; }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      rflat = min(rflat, __shfl_xor_sync(0xffffffffu, rflat, o));
      rany = min(rany, __shfl_xor_sync(0xffffffffu, rany, o));
      lflat = min(lflat, __shfl_xor_sync(0xffffffffu, lflat, o));
      lany = min(lany, __shfl_xor_sync(0xffffffffu, lany, o));
    }
  }
  if (rflat == kNoIdx) rflat = -1;
  if (rany == kNoIdx) rany = -1;
  if (lflat == kNoIdx) lflat = -1;
  if (lany == kNoIdx) lany = -1;
  if (fi) {
    rk = rflat >= 0 ? mk_key_score(0.0, rflat, imask)
                    : (rany >= 0 ? mk_key_score(0.5, rany, imask) : kKeyNone);
    lk = lflat >= 0 ? mk_key_score(0.0, lflat, imask)
                    : (lany >= 0 ? mk_key_score(0.5, lany, imask) : kKeyNone);
  } else {
    if (rflat >= 0) {
      const long long k = mk_key_score(0.5, rflat, imask);
      rk = k < rk ? k : rk;
    }
    if (lflat >= 0) {
      const long long k = mk_key_score(0.5, lflat, imask);
      lk = k < lk ? k : lk;
    }
  }
  const long long best = lk <= rk ? lk : rk;
  const long long bi = best == kKeyNone ? -1 : (best & imask);
  // every 8-lane group computes the same value, in the same order as the full
  // join's finalize (so a full-coverage neighbour gets bit-identical values)
  const double v = group_value(A, i, A, bi, true, m, lane % kFinLanes);
  if (lane == 0) {
    if (mp) mp[i] = v;
    if (pi) pi[i] = bi;
    if (left) left[i] = -1;
    if (right) right[i] = -1;
  }
}

// Finalize of a masked band join (exact anytime SCRIMP, dense sets): as
// k_finalize_self_partial, with admissibility per DIAGONAL. dbits: bit k set
// when diagonal k is chosen; diags: the chosen diagonals, ascending. The flat
// convention needs, on either side of row i, the smallest flat window on a
// chosen diagonal and the smallest admissible neighbour at all. One warp per
// row: it walks the non-empty words of the flat bitmask (next_word skips the
// rest), one window per lane, and stops at the first word with a hit.
__global__ void k_finalize_self_masked(const Series A, const long long* __restrict__ key_right,
                                       const long long* __restrict__ key_left, int m, long long imask,
                                       const uint32_t* __restrict__ dbits,
                                       const long long* __restrict__ diags, long long n_diags,
                                       double* __restrict__ mp, long long* __restrict__ pi,
                                       long long* __restrict__ left, long long* __restrict__ right) {
  const long long i = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (i >= A.L) return;
  const long long L = A.L;
  long long rk = key_right[i], lk = key_left[i];
  const bool fi = A.inv[i] == 0.0;
  auto chosen = [&](long long k) { return k >= 0 && k < L && ((dbits[k >> 5] >> (k & 31)) & 1u); };
  long long rflat = -1, rany = -1, lflat = -1, lany = -1;
  if (n_diags > 0 && next_flat(A, 0) >= 0) {
    const long long kmin = diags[0];
    if (i + kmin < L) rany = i + kmin;
    // the largest chosen diagonal <= i gives the smallest left neighbour
    {
      long long lo = 0, hi = n_diags;  // first index with diags[idx] > i
      while (lo < hi) {
        const long long mid = (lo + hi) >> 1;
        if (diags[mid] <= i) lo = mid + 1; else hi = mid;
      }
      if (lo > 0) lany = i - diags[lo - 1];
    }
    // right: flat windows j >= i + kmin, ascending
    if (rany >= 0) {
      int w = A.next_word[rany >> 5];
      while (w >= 0) {
        const long long j = ((long long)w << 5) + lane;
        const bool hit = ((A.flat_words[w] >> lane) & 1u) && j >= rany && j < L && chosen(j - i);
        const unsigned b = __ballot_sync(0xffffffffu, hit);
        if (b) { rflat = ((long long)w << 5) + __ffs(b) - 1; break; }
        w = w + 1 < A.n_words ? A.next_word[w + 1] : -1;
      }
    }
    // left: flat windows j <= i - kmin, ascending from 0
    if (lany >= 0) {
      const long long jmax = i - kmin;
      int w = A.next_word[0];
      while (w >= 0 && ((long long)w << 5) <= jmax) {
        const long long j = ((long long)w << 5) + lane;
        const bool hit = ((A.flat_words[w] >> lane) & 1u) && j <= jmax && chosen(i - j);
        const unsigned b = __ballot_sync(0xffffffffu, hit);
        if (b) { lflat = ((long long)w << 5) + __ffs(b) - 1; break; }
        w = w + 1 < A.n_words ? A.next_word[w + 1] : -1;
      }
    }
  }
  if (fi) {
    rk = rflat >= 0 ? mk_key_score(0.0, rflat, imask)
                    : (rany >= 0 ? mk_key_score(0.5, rany, imask) : kKeyNone);
    lk = lflat >= 0 ? mk_key_score(0.0, lflat, imask)
                    : (lany >= 0 ? mk_key_score(0.5, lany, imask) : kKeyNone);
  } else {
    if (rflat >= 0) {
      const long long k = mk_key_score(0.5, rflat, imask);
      rk = k < rk ? k : rk;
    }
    if (lflat >= 0) {
      const long long k = mk_key_score(0.5, lflat, imask);
      lk = k < lk ? k : lk;
    }
  }
  const long long best = lk <= rk ? lk : rk;
  const long long bi = best == kKeyNone ? -1 : (best & imask);
  const double v = group_value(A, i, A, bi, true, m, lane % kFinLanes);
  if (lane == 0) {
    if (mp) mp[i] = v;
    if (pi) pi[i] = bi;
    if (left) left[i] = -1;
    if (right) right[i] = -1;
  }
}

__global__ void k_finalize_keys(const Series A, const long long* __restrict__ key_right,
                                const long long* __restrict__ key_left, int m, long long imask,
                                double* __restrict__ mp, long long* __restrict__ pi,
                                long long* __restrict__ left, long long* __restrict__ right) {
  const long long gi = (blockIdx.x * (long long)blockDim.x + threadIdx.x) / kFinLanes;
  const int sub = threadIdx.x % kFinLanes;
  const bool valid = gi < A.L;
  const long long ic = valid ? gi : 0;
  const long long rk = key_right[ic], lk = key_left[ic];
  const long long best = lk <= rk ? lk : rk;
  const long long bi = best == kKeyNone ? -1 : (best & imask);
  const double v = group_value(A, ic, A, bi, valid, m, sub);
  if (valid && sub == 0) {
    if (mp) mp[gi] = v;
    if (pi) pi[gi] = bi;
    if (left) left[gi] = -1;
    if (right) right[gi] = -1;
  }
}

// AB-join side: window i of X against every window of Y.
__global__ void k_finalize_ab(const Series X, const Series Y, const long long* __restrict__ keys,
                              int m, long long imask, long long row0, long long row1,
                              double* __restrict__ mp, long long* __restrict__ pi) {
  const long long gi = (blockIdx.x * (long long)blockDim.x + threadIdx.x) / kFinLanes;
  const int sub = threadIdx.x % kFinLanes;
  const long long i = row0 + gi;
  const bool valid = i < row1;
  const long long ic = valid ? i : row0;
  long long k = keys[ic];
  const long long fy = next_flat(Y, 0);
  if (X.inv[ic] == 0.0) {
    k = fy >= 0 ? mk_key_score(0.0, fy, imask) : mk_key_score(0.5, 0, imask);
  } else if (fy >= 0) {
    const long long kf = mk_key_score(0.5, fy, imask);
    k = kf < k ? kf : k;
  }
  const long long bi = k == kKeyNone ? -1 : (k & imask);
  const double v = group_value(X, ic, Y, bi, valid, m, sub);
  if (valid && sub == 0) {
    if (mp) mp[i] = v;
    if (pi) pi[i] = bi;
  }
}

}  // namespace mpgpu
