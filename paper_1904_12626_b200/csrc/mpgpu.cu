// Host side of the B200 matrix-profile join: plans, work items, sharding,
// multi-device orchestration and the C ABI declared in include/mprof_gpu.h.
//
// Reference boundary: mprof::stomp / mprof::scrimp (profile.hpp:80-89). The
// C++ shim in mprof_api.cpp keeps those signatures and calls mpgpu_join.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <cstdint>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "mprof_gpu.h"
#include "mpgpu_kernels.cuh"
#include "mpgpu_internal.h"

using namespace mpgpu;

namespace {
// NVTX range over one host entry point (K1-K5 phases show up by name in
// nsys / ncu --nvtx timelines; header-only NVTX 3, inert without a tool).
struct Range {
  explicit Range(const char* name) { nvtxRangePushA(name); }
  ~Range() { nvtxRangePop(); }
};
}  // namespace

namespace {

thread_local std::string g_err;

mpgpu_status fail(mpgpu_status st, const std::string& msg) {
  g_err = msg;
  return st;
}

#define MPG_CUDA(call)                                                                      \
  do {                                                                                      \
    cudaError_t e_ = (call);                                                                \
    if (e_ != cudaSuccess) {                                                                \
      return fail(e_ == cudaErrorMemoryAllocation ? MPGPU_ENOMEM : MPGPU_ECUDA,             \
                  std::string(#call) + ": " + cudaGetErrorString(e_));                      \
    }                                                                                       \
  } while (0)

int ceil_log2(long long v) {
  int b = 0;
  while ((1LL << b) < v) ++b;
  return b;
}

// sum_{k=k1}^{k2-1} clamp(A - k, 0, N)  (valid rows of one diagonal in a segment)
long long sum_clamp(long long A, long long k1, long long k2, long long N) {
  long long total = 0;
  if (k2 <= k1 || N <= 0) return 0;
  // region where A - k >= N : k <= A - N  -> contributes N
  const long long kfull_hi = std::min(k2, A - N + 1);
  if (kfull_hi > k1) total += (kfull_hi - k1) * N;
  // region where 0 < A - k < N
  const long long lo = std::max(k1, A - N + 1), hi = std::min(k2, A);
  if (hi > lo) {
    // sum_{k=lo}^{hi-1} (A - k) = sum of an arithmetic series
    const long long first = A - lo, last = A - (hi - 1);
    total += (first + last) * (hi - lo) / 2;
  }
  return total;
}

struct DevSeries {
  double* mu = nullptr;
  double* inv = nullptr;
  double* sd = nullptr;
  double2* U = nullptr;
  uint8_t* flat = nullptr;
  uint32_t* words = nullptr;
  int32_t* next = nullptr;
  int32_t* next_agg = nullptr;  // per block of kNextBlock words (k_next_word_*)
  long long n = 0, L = 0;
  int n_words = 0;
  const double* x = nullptr;

  Series view() const {
    Series s;
    s.x = x; s.mu = mu; s.inv = inv; s.U = U; s.flat_words = words; s.next_word = next;
    s.n = n; s.L = L; s.n_words = n_words;
    return s;
  }
  void release() {
    cudaFree(mu); cudaFree(inv); cudaFree(sd); cudaFree(U); cudaFree(flat); cudaFree(words);
    cudaFree(next);
    cudaFree(next_agg);
    mu = inv = sd = nullptr; U = nullptr; flat = nullptr; words = nullptr; next = nullptr;
    next_agg = nullptr;
  }
};

}  // namespace

struct mpgpu_plan {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  bool self = true;
  long long m = 0, zone = 0;
  int index_bits = 1;
  long long imask = 1;
  DevSeries A, B;
  long long* key0 = nullptr;  // self: right (row) keys; AB: A keys
  long long* key1 = nullptr;  // self: left (column) keys; AB: B keys
  std::vector<Item> items;    // sorted, largest first
  std::vector<long long> item_cells;
  std::vector<long long> prefix;  // prefix[i] = cells of items[0..i)
  Item* d_items = nullptr;
  int* d_counter = nullptr;
  // which shard slices of d_items hold their item list (for slice_n shards):
  // uploaded once, reused by every later run of the same sharding
  std::vector<char> slice_ok;
  std::vector<long long> slice_cnt;
  int slice_n = 0;
  int n_ctas = 0;
  long long launches = 0;
  long long seg_rows = 0;
  // anytime (SCRIMP partial) mode: only these bands (first diagonals, sorted)
  std::vector<long long> bands;
  long long* d_bands = nullptr;
  bool subset = false;
  long long* d_init_diags = nullptr;  // anytime warm start: diagonals inside the chosen bands
  int n_init_diags = 0;
  // anytime band subsets: the chosen bands as a bitmask (the coarse exploit
  // seeds only their diagonals) and the coarse diagonals they map to (the
  // coarse warm start joins only those)
  unsigned* d_band_mask = nullptr;
  std::vector<long long> coarse_diags;
  bool coarse_diags_dirty = false;
  // anytime (SCRIMP) over an explicit diagonal set: k_diag_join instead of k_join,
  // or, for dense sets, k_join_masked over the bands that hold a chosen diagonal
  // (mask_mode: subset is set too, bands lists those bands)
  bool mask_mode = false;
  unsigned char* d_dmasks = nullptr;  // per band and lane: the lane's chosen diagonals
  uint32_t* d_diag_bits = nullptr;    // bit k: diagonal k is chosen
  bool diag_mode = false;
  long long* d_diags = nullptr;
  long long n_diags = 0;
  DiagItem* d_ditems = nullptr;
  int n_ditems = 0;
  int diag_rows = 0;
  // keys owned by another plan (possibly on a peer device, reached over NVLink):
  // this plan's k_join reads thresholds from and RED.MINs into them directly
  long long* ext_key0 = nullptr;
  long long* ext_key1 = nullptr;
  // attached to a shared key region as its owner: this plan still resets and
  // warm-starts the (shared) keys; the other ranks' plans only read and RED.MIN
  bool ext_owner = false;
  // coarse warm start (K2b): a nested plan on the PAA-downsampled series
  int coarse_f = 0;  // 0: off
  bool coarse_pending = false;  // coarse join done, exploit not yet run
  bool coarse_keys_shared = false;  // coarse keys shared across ranks: coarse_run is separate
  bool is_coarse = false;           // this plan is another plan's coarse warm-start join
  mpgpu_plan* coarse = nullptr;
  double* xc_a = nullptr;
  double* xc_b = nullptr;
};

namespace {

mpgpu_status alloc_series(DevSeries& s, const double* x, long long n, long long m) {
  s.x = x;
  s.n = n;
  s.L = n - m + 1;
  s.n_words = (int)((s.L + 31) / 32);
  MPG_CUDA(cudaMalloc(&s.mu, sizeof(double) * s.L));
  MPG_CUDA(cudaMalloc(&s.inv, sizeof(double) * (s.L + kPad)));
  MPG_CUDA(cudaMalloc(&s.U, sizeof(double2) * (s.L + kPad)));
  MPG_CUDA(cudaMalloc(&s.flat, s.L));
  MPG_CUDA(cudaMalloc(&s.words, sizeof(uint32_t) * s.n_words));
  MPG_CUDA(cudaMalloc(&s.next, sizeof(int32_t) * s.n_words));
  MPG_CUDA(cudaMalloc(&s.next_agg, sizeof(int32_t) * ((s.n_words + kNextBlock - 1) / kNextBlock)));
  return MPGPU_OK;
}

// K1 launch: the blocked kernel when the series fills the GPU with its 1024-window CTAs
static void launch_window_stats(const double* x, long long L, int m, double* mu, double* inv,
                                double* sd, uint8_t* flat, cudaStream_t st) {
  if (L >= 2LL * 148 * kStatTile) {
    k_window_stats_blocked<<<(unsigned)((L + kStatTile - 1) / kStatTile), kStatThreads, 0, st>>>(
        x, L, m, mu, inv, sd, flat);
  } else {
    k_window_stats<<<(unsigned)((L + 255) / 256), 256, 0, st>>>(x, L, m, mu, inv, sd, flat);
  }
}

mpgpu_status launch_stats(mpgpu_plan* p, DevSeries& s) {
  const int bs = 256;
  launch_window_stats(s.x, s.L, (int)p->m, s.mu, s.inv, nullptr, s.flat, p->stream);
  k_update_vectors<<<(unsigned)((s.L + kPad + bs - 1) / bs), bs, 0, p->stream>>>(
      s.x, s.mu, s.L, (int)p->m, s.U, s.inv);
  k_flat_words<<<(unsigned)((s.n_words * 32LL + bs - 1) / bs), bs, 0, p->stream>>>(
      s.flat, s.L, s.n_words, s.words);
  const int nb = (s.n_words + kNextBlock - 1) / kNextBlock;
  k_next_word_local<<<nb, kNextBlock, 0, p->stream>>>(s.words, s.n_words, s.next, s.next_agg);
  k_next_word_aggs<<<1, 1024, 0, p->stream>>>(s.next_agg, nb);
  k_next_word_fix<<<(unsigned)((s.n_words + 255) / 256), 256, 0, p->stream>>>(s.next, s.n_words,
                                                                              s.next_agg);
  p->launches += 6;
  MPG_CUDA(cudaGetLastError());
  return MPGPU_OK;
}

// Work items: for each pass, bands of kW diagonals, each cut into segments of
// seg_rows rows (a multiple of kH). Segment length depends only on the problem
// (never on the shard count), so results are bit-identical for any sharding.
void build_items(mpgpu_plan* p) {
  struct PassGeom { long long LR, LC, klo, khi; };
  std::vector<PassGeom> geo;
  if (p->self) {
    geo.push_back({p->A.L, p->A.L, p->zone + 1, p->A.L});
  } else {
    geo.push_back({p->A.L, p->B.L, 0, p->B.L});  // rows A, cols B, k >= 0
    geo.push_back({p->B.L, p->A.L, 1, p->A.L});  // rows B, cols A, k >= 1
  }
  // total cells for segment sizing
  long long cells = 0;
  for (auto& g : geo) {
    if (g.khi <= g.klo) continue;
    // sum_k min(LR, LC - k) over k in [klo, khi)
    cells += sum_clamp(g.LC, g.klo, g.khi, g.LR);
  }
  // 148 SMs x kMinBlocks CTAs x kWarps warp-workers (fixed: independent of device & shards)
  const long long ref_workers = 148LL * kMinBlocks * kWarps;
  // Segment length: long enough that the kW x m seed each segment pays stays
  // small (8m rows -> ~6%), short enough that every warp-worker gets at least
  // two items, and at most 64 items per worker on big joins.
  const long long seg_balance = cells / ((long long)kW * 64 * ref_workers);
  static const long long fill_items = getenv("MPGPU_SEG_FILL") ? atoll(getenv("MPGPU_SEG_FILL")) : 2;
  const long long seg_fill = cells / ((long long)kW * fill_items * ref_workers);
  long long seg = std::max(seg_balance, std::min<long long>(8 * p->m, seg_fill));
  seg = std::min<long long>(std::max<long long>(16384, 8 * p->m), seg);
  // at most ~1e8 items (2.4 GB of item records; the queue index is an int):
  // only series beyond ~2^27 samples reach this
  seg = std::max<long long>(seg, cells / ((long long)kW * 100000000LL) + 1);
  static const long long seg_env = getenv("MPGPU_SEG_ROWS") ? atoll(getenv("MPGPU_SEG_ROWS")) : 0;
  if (seg_env > 0) seg = seg_env;  // experiments only
  seg = std::max<long long>(kH, (seg / kH) * kH);
  p->seg_rows = seg;

  p->items.clear();
  p->item_cells.clear();
  for (int pi = 0; pi < (int)geo.size(); ++pi) {
    const auto& g = geo[pi];
    for (long long kb = g.klo; kb < g.khi; kb += kW) {
      const long long ke = std::min(kb + kW, g.khi);
      const long long rows_needed = std::min(g.LR, g.LC - kb);
      if (rows_needed <= 0) continue;
      for (long long r0 = 0; r0 < rows_needed; r0 += seg) {
        const long long nr = std::min(seg, rows_needed - r0);
        Item it;
        it.pass = pi;
        it.kb = kb;
        it.r0 = r0;
        it.nrows = (int)(((nr + kH - 1) / kH) * kH);
        // valid cells: sum_k clamp(min(LR, LC - k) - r0, 0, nr); min() switches
        // from LR to LC - k at k = LC - LR
        const long long ksplit = std::min(ke, std::max(kb, g.LC - g.LR + 1));
        const long long c = (ksplit - kb) * std::max(0LL, std::min(g.LR - r0, nr)) +
                            sum_clamp(g.LC - r0, ksplit, ke, nr);
        p->items.push_back(it);
        p->item_cells.push_back(c);
      }
    }
  }
  // largest first (longest-processing-time order for the persistent queue)
  std::vector<size_t> order(p->items.size());
  for (size_t i = 0; i < order.size(); ++i) order[i] = i;
  std::stable_sort(order.begin(), order.end(), [&](size_t a, size_t b) {
    return p->item_cells[a] > p->item_cells[b];
  });
  std::vector<Item> its(order.size());
  std::vector<long long> cs(order.size());
  for (size_t i = 0; i < order.size(); ++i) {
    its[i] = p->items[order[i]];
    cs[i] = p->item_cells[order[i]];
  }
  p->items.swap(its);
  p->item_cells.swap(cs);
  p->prefix.assign(p->items.size() + 1, 0);
  for (size_t i = 0; i < p->items.size(); ++i) p->prefix[i + 1] = p->prefix[i] + p->item_cells[i];
}

// Items of shard s: round-robin by cost rank (item q goes to shard q % n), so
// every shard receives the same mix of large and small items.
void shard_items(const mpgpu_plan* p, int shard, int n_shards, std::vector<Item>& out,
                 long long* cells) {
  out.clear();
  long long c = 0;
  for (size_t q = (size_t)shard; q < p->items.size(); q += (size_t)n_shards) {
    out.push_back(p->items[q]);
    c += p->item_cells[q];
  }
  if (cells) *cells = c;
}

long long* key_row(const mpgpu_plan* p) { return p->ext_key0 ? p->ext_key0 : p->key0; }
long long* key_col(const mpgpu_plan* p) { return p->ext_key1 ? p->ext_key1 : p->key1; }

JoinParams make_params(const mpgpu_plan* p) {
  JoinParams P;
  memset(&P, 0, sizeof(P));
  if (p->self) {
    P.pass[0].R = p->A.view();
    P.pass[0].C = p->A.view();
    P.pass[0].keyR = key_row(p);
    P.pass[0].keyC = key_col(p);
  } else {
    P.pass[0].R = p->A.view();
    P.pass[0].C = p->B.view();
    P.pass[0].keyR = key_row(p);
    P.pass[0].keyC = key_col(p);
    P.pass[1].R = p->B.view();
    P.pass[1].C = p->A.view();
    P.pass[1].keyR = key_col(p);
    P.pass[1].keyC = key_row(p);
  }
  P.m = (int)p->m;
  P.imask = p->imask;
  return P;
}

// PAA factor of the coarse warm start: coarse window m/f = 16 samples. Off for
// short windows, for series too short to leave a coarse profile, and when
// MPGPU_COARSE=0 (experiments).
long long join_cells_of(const mpgpu_plan* p) { return p->prefix.empty() ? 0 : p->prefix.back(); }

int coarse_factor(const mpgpu_plan* p) {
  static const bool off = getenv("MPGPU_COARSE") && atoi(getenv("MPGPU_COARSE")) == 0;
  if (off) return 0;
  static const int div = getenv("MPGPU_COARSE_DIV") ? atoi(getenv("MPGPU_COARSE_DIV")) : 16;
  static const double min_cells = getenv("MPGPU_COARSE_MIN") ? atof(getenv("MPGPU_COARSE_MIN")) : 1e9;
  if ((double)join_cells_of(p) < min_cells) return 0;
  const long long f = p->m / div;
  if (f < 2) return 0;
  const long long mc = p->m / f;
  const long long nA = p->A.n / f, nB = p->self ? nA : p->B.n / f;
  const long long zc = p->self ? (p->zone + f - 1) / f : 0;
  if (nA - mc + 1 < zc + 2 || nB - mc + 1 < 2) return 0;
  return (int)f;
}

// The nested coarse plan (PAA series, window m/f), created on first use.
mpgpu_status ensure_coarse(mpgpu_plan* p) {
  if (p->coarse) return MPGPU_OK;
  const int f = p->coarse_f;
  const long long mc = p->m / f;
  const long long nA = p->A.n / f, nB = p->self ? nA : p->B.n / f;
  MPG_CUDA(cudaMalloc(&p->xc_a, sizeof(double) * nA));
  if (!p->self) MPG_CUDA(cudaMalloc(&p->xc_b, sizeof(double) * nB));
  const long long zc = p->self ? (p->zone + f - 1) / f : 0;
  p->coarse = mpgpu_plan_create(p->xc_a, nA, p->self ? nullptr : p->xc_b, nB, mc, zc,
                                p->device, p->stream);
  if (p->coarse) p->coarse->is_coarse = true;
  return p->coarse ? MPGPU_OK : MPGPU_ECUDA;
}

// K2b, phase 1: PAA series, the coarse plan's prepare and (this shard of) the
// coarse join; with coarse keys shared across ranks the join is a separate
// step (mpgpu_plan_coarse_run) once the owner's coarse prepare is visible.
mpgpu_status coarse_begin(mpgpu_plan* p, int shard, int n_shards, bool run = true) {
  const int f = p->coarse_f;
  const long long nA = p->A.n / f, nB = p->self ? nA : p->B.n / f;
  if (mpgpu_status st = ensure_coarse(p); st != MPGPU_OK) return st;
  k_paa<<<(unsigned)((nA + 255) / 256), 256, 0, p->stream>>>(p->A.x, nA, f, p->xc_a);
  if (!p->self) k_paa<<<(unsigned)((nB + 255) / 256), 256, 0, p->stream>>>(p->B.x, nB, f, p->xc_b);
  p->launches += p->self ? 1 : 2;
  mpgpu_status st = mpgpu_plan_prepare(p->coarse);
  if (st == MPGPU_OK && run) st = mpgpu_plan_run(p->coarse, shard, n_shards);
  if (st != MPGPU_OK) return st;
  p->launches += p->coarse->launches;
  MPG_CUDA(cudaGetLastError());
  return MPGPU_OK;
}

// K2b, phase 2: seed the fine keys around the (merged) coarse matches. Coarse
// row keys (best column per coarse row) and column keys (best row per coarse
// column) both seed pass 0 of the fine plan (rows of A, columns of B).
mpgpu_status coarse_finish(mpgpu_plan* p, int shard = 0, int n_shards = 1) {
  const int f = p->coarse_f;
  const JoinParams P = make_params(p);
  const mpgpu_plan* c = p->coarse;
  const long long Lr = c->A.L, Lc = c->self ? c->A.L : c->B.L;
  // fine diagonals searched around each coarse match: +-f/2 (the PAA alignment
  // error is below f; wider spans cost seeds for little gain)
  static const int span_env = getenv("MPGPU_COARSE_SPAN") ? atoi(getenv("MPGPU_COARSE_SPAN")) : 0;
  const int dspan = span_env > 0 ? span_env : std::max(1, f / 2);
  const int nd = 2 * dspan + 1;
  // anytime band subsets: seed only diagonals of the chosen bands
  const unsigned* band_mask = (p->subset && !p->diag_mode && !p->mask_mode) ? p->d_band_mask : nullptr;
  // masked bands (dense diagonal subsets): seed only the chosen diagonals
  const unsigned* diag_bits = p->mask_mode ? p->d_diag_bits : nullptr;
  // this shard's contiguous share of the coarse windows (all of them for one shard)
  const long long r0 = Lr * shard / n_shards, r1 = Lr * (shard + 1) / n_shards;
  const long long c0 = Lc * shard / n_shards, c1 = Lc * (shard + 1) / n_shards;
  (void)nd;
  if (r1 > r0)
    k_coarse_exploit<<<(unsigned)((r1 - r0 + kExpWarps - 1) / kExpWarps), kExpWarps * 32, 0,
                       p->stream>>>(P.pass[0], key_row(c), r0, r1, c->imask, false, f, dspan,
                                    p->zone, p->self, (int)p->m, p->imask, band_mask, diag_bits);
  if (c1 > c0)
    k_coarse_exploit<<<(unsigned)((c1 - c0 + kExpWarps - 1) / kExpWarps), kExpWarps * 32, 0,
                       p->stream>>>(P.pass[0], key_col(c), c0, c1, c->imask, true, f, dspan,
                                    p->zone, p->self, (int)p->m, p->imask, band_mask, diag_bits);
  p->launches += 2;
  MPG_CUDA(cudaGetLastError());
  return MPGPU_OK;
}

// Spread-diagonal warm start (K2) of a full join: this shard's share of the
// n_init diagonals of every pass (all of them for one shard).
void launch_init(mpgpu_plan* p, int shard, int n_shards) {
  const JoinParams P = make_params(p);
  const int npass = p->subset ? 0 : (p->self ? 1 : 2);
  for (int q = 0; q < npass; ++q) {
    const Pass& ps = P.pass[q];
    const long long klo = p->self ? p->zone + 1 : (q == 0 ? 0 : 1);
    const long long khi = ps.C.L;
    if (khi <= klo) continue;
    // spread diagonals: a handful when the coarse warm start follows (it finds
    // far better candidates), kInitDiag otherwise
    static const int n_env = getenv("MPGPU_INIT_N") ? atoi(getenv("MPGPU_INIT_N")) : -1;
    static const int nc_env = getenv("MPGPU_COARSE_INIT_N") ? atoi(getenv("MPGPU_COARSE_INIT_N")) : -1;
    // without the coarse warm start (joins below 1e9 cells) every item runs
    // against these keys at once, so they get more diagonals: L / 64 of them
    // (~3% of the cells), 32 to 512 (C1: 252 diagonals, 0.43 -> 0.37 ms)
    const long long n_small = std::min<long long>(512, std::max<long long>(kInitDiag, ps.R.L / 64));
    const int n_init = p->is_coarse ? (nc_env >= 0 ? nc_env : kInitDiag)
                                    : (n_env >= 0 ? n_env : (p->coarse_f > 0 ? 8 : (int)n_small));
    const int mine = n_init > shard ? (n_init - shard + n_shards - 1) / n_shards : 0;
    if (mine <= 0) continue;
    // seed points every kInitRows rows (the problem's, never the shard's)
    dim3 grid((unsigned)((ps.R.L + (long long)kInitWarps * kInitRows - 1) /
                         ((long long)kInitWarps * kInitRows)),
              (unsigned)mine);
    k_init_keys<<<grid, kInitWarps * 32, 0, p->stream>>>(ps, klo, khi, (int)p->m, p->imask, nullptr,
                                                         shard, n_shards, n_init);
    p->launches += 1;
  }
}

std::once_flag g_attr_once;
int g_ctas_per_sm = 0;

}  // namespace

namespace {
mpgpu_status plan_select_diagonals(mpgpu_plan* p, const std::vector<long long>& diags);
}  // namespace

namespace mpgpu_internal {

mpgpu_status set_error(mpgpu_status st, const std::string& msg) { return fail(st, msg); }

long long stats_pad() { return kPad; }

cudaError_t series_stats(const double* d_x, long long n, int m, double* mu, double* inv,
                         double2* U, uint8_t* flat, cudaStream_t st) {
  const long long L = n - m + 1;
  const int bs = 256;
  launch_window_stats(d_x, L, m, mu, inv, nullptr, flat, st);
  k_update_vectors<<<(unsigned)((L + kPad + bs - 1) / bs), bs, 0, st>>>(d_x, mu, L, m, U, inv);
  return cudaGetLastError();
}

}  // namespace mpgpu_internal

extern "C" {

const char* mpgpu_last_error(void) { return g_err.c_str(); }

const char* mpgpu_build_info(void) {
  static char buf[192];
  // resident CTAs per SM as the occupancy API reports it (0 before any plan)
  snprintf(buf, sizeof(buf),
           "mprof_b200 sm_100a fp64 D=%d warps=%d W=%d H=%d ring=%d smem=%zu ctas_per_sm=%d", kD,
           kWarps, kW, kH, kRing, sizeof(JoinSmem), g_ctas_per_sm);
  return buf;
}

int64_t mpgpu_zone_size(int64_t window, double fraction) {
  if (!(fraction >= 0.0)) return -1;
  return (int64_t)std::floor((double)window * fraction + 0.5);
}

int64_t mpgpu_join_cells(int64_t n_a, int64_t n_b, int64_t window, int64_t zone) {
  const long long La = n_a - window + 1;
  if (La <= 0) return 0;
  if (n_b <= 0) {
    const long long r = La - zone - 1;
    return r > 0 ? r * (r + 1) / 2 : 0;
  }
  const long long Lb = n_b - window + 1;
  return Lb > 0 ? La * Lb : 0;
}

mpgpu_status mpgpu_rolling_stats(const double* d_ts, int64_t n, int64_t window, double* d_means,
                                 double* d_stds, int32_t device, void* cuda_stream) {
  if (window < 4 || window > n) return fail(MPGPU_EPARAM, "window out of range");
  MPG_CUDA(cudaSetDevice(device));
  const long long L = n - window + 1;
  cudaStream_t st = (cudaStream_t)cuda_stream;
  launch_window_stats(d_ts, L, (int)window, d_means, nullptr, d_stds, nullptr, st);
  MPG_CUDA(cudaGetLastError());
  return MPGPU_OK;
}

mpgpu_plan* mpgpu_plan_create(const double* d_a, int64_t n_a, const double* d_b, int64_t n_b,
                              int64_t window, int64_t zone, int32_t device, void* cuda_stream) {
  if (!d_a || window < 4 || window > n_a || (d_b && window > n_b) || zone < 0) {
    fail(MPGPU_EPARAM, "invalid window / series length / zone");
    return nullptr;
  }
  if (cudaSetDevice(device) != cudaSuccess) {
    fail(MPGPU_ECUDA, "cudaSetDevice failed");
    return nullptr;
  }
  std::unique_ptr<mpgpu_plan> p(new mpgpu_plan());
  p->device = device;
  p->self = d_b == nullptr;
  p->m = window;
  p->zone = p->self ? zone : 0;
  // NULL is the legacy default stream (CUDA's own convention), so a plan built
  // on torch's default stream stays ordered with the caller's work
  p->stream = (cudaStream_t)cuda_stream;
  p->own_stream = false;
  if (alloc_series(p->A, d_a, n_a, window) != MPGPU_OK) {
    mpgpu_plan_destroy(p.release());
    return nullptr;
  }
  if (!p->self && alloc_series(p->B, d_b, n_b, window) != MPGPU_OK) {
    mpgpu_plan_destroy(p.release());
    return nullptr;
  }
  const long long Lb = p->self ? p->A.L : p->B.L;
  p->index_bits = std::max(1, ceil_log2(std::max(p->A.L, Lb)));
  if (p->index_bits > 40) {
    fail(MPGPU_EPARAM, "series too long for packed keys");
    mpgpu_plan_destroy(p.release());
    return nullptr;
  }
  p->imask = (1LL << p->index_bits) - 1;
  // keys carry kPad entries of padding like the statistics (kernels may read,
  // never use, a few entries past the end)
  if (cudaMalloc(&p->key0, sizeof(long long) * (p->A.L + kPad)) != cudaSuccess ||
      cudaMalloc(&p->key1, sizeof(long long) * (Lb + kPad)) != cudaSuccess ||
      cudaMalloc(&p->d_counter, sizeof(int)) != cudaSuccess) {
    fail(MPGPU_ENOMEM, "key allocation failed");
    mpgpu_plan_destroy(p.release());
    return nullptr;
  }
  build_items(p.get());
  if (!p->items.empty()) {
    if (cudaMalloc(&p->d_items, sizeof(Item) * p->items.size()) != cudaSuccess) {
      fail(MPGPU_ENOMEM, "item allocation failed");
      mpgpu_plan_destroy(p.release());
      return nullptr;
    }
  }
  std::call_once(g_attr_once, [] {
    cudaFuncSetAttribute(k_join, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)sizeof(JoinSmem));
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&g_ctas_per_sm, k_join, kThreads,
                                                  sizeof(JoinSmem));
  });
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  // attribute is per-device: set it here as well for multi-device processes
  cudaFuncSetAttribute(k_join, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(JoinSmem));
  cudaFuncSetAttribute(k_join_masked, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)sizeof(JoinSmem));
  p->n_ctas = sms * std::max(1, g_ctas_per_sm);
  p->coarse_f = coarse_factor(p.get());
  return p.release();
}

void mpgpu_plan_destroy(mpgpu_plan* p) {
  if (!p) return;
  cudaSetDevice(p->device);
  cudaStreamSynchronize(p->stream);
  if (p->coarse) mpgpu_plan_destroy(p->coarse);
  cudaFree(p->d_dmasks);
  cudaFree(p->d_diag_bits);
  cudaFree(p->xc_a);
  cudaFree(p->xc_b);
  p->A.release();
  p->B.release();
  cudaFree(p->key0);
  cudaFree(p->key1);
  cudaFree(p->d_items);
  cudaFree(p->d_counter);
  cudaFree(p->d_bands);
  cudaFree(p->d_init_diags);
  cudaFree(p->d_diags);
  cudaFree(p->d_ditems);
  cudaFree(p->d_band_mask);
  if (p->own_stream && p->stream) cudaStreamDestroy(p->stream);
  delete p;
}

mpgpu_status mpgpu_plan_prepare(mpgpu_plan* p) {
  const mpgpu_status st = mpgpu_plan_prepare_shard(p, 0, 1);
  return st != MPGPU_OK ? st : mpgpu_plan_prepare_finish(p);
}

mpgpu_status mpgpu_plan_coarse_keys(mpgpu_plan* p, int64_t** d_row_keys, int64_t* row_len,
                                    int64_t** d_col_keys, int64_t* col_len) {
  if (!p) return fail(MPGPU_EPARAM, "null plan");
  const bool on = p->coarse_pending && p->coarse;
  if (d_row_keys) *d_row_keys = on ? (int64_t*)p->coarse->key0 : nullptr;
  if (row_len) *row_len = on ? p->coarse->A.L : 0;
  if (d_col_keys) *d_col_keys = on ? (int64_t*)p->coarse->key1 : nullptr;
  if (col_len) *col_len = on ? (p->coarse->self ? p->coarse->A.L : p->coarse->B.L) : 0;
  return MPGPU_OK;
}

mpgpu_status mpgpu_plan_prepare_finish(mpgpu_plan* p) {
  if (!p) return fail(MPGPU_EPARAM, "null plan");
  if (!p->coarse_pending) return MPGPU_OK;
  MPG_CUDA(cudaSetDevice(p->device));
  p->coarse_pending = false;
  return coarse_finish(p);
}

mpgpu_status mpgpu_plan_prepare_shared(mpgpu_plan* p, int32_t shard, int32_t n_shards) {
  Range nvtx_range("mpgpu:prepare_shared (K1 stats, coarse prepare)");
  if (!p) return fail(MPGPU_EPARAM, "null plan");
  if (n_shards < 1 || shard < 0 || shard >= n_shards) return fail(MPGPU_EPARAM, "bad shard");
  if (p->subset) return fail(MPGPU_EUNSUPPORTED, "shared-key joins are full joins");
  p->coarse_pending = false;
  MPG_CUDA(cudaSetDevice(p->device));
  p->launches = 0;
  mpgpu_status st = launch_stats(p, p->A);
  if (st != MPGPU_OK) return st;
  if (!p->self && (st = launch_stats(p, p->B)) != MPGPU_OK) return st;
  if (p->coarse_f > 0) {
    if (coarse_begin(p, shard, n_shards, !p->coarse_keys_shared) == MPGPU_OK) {
      p->coarse_pending = true;
    } else if (p->coarse_keys_shared) {
      return fail(MPGPU_ECUDA, "coarse phase failed with shared coarse keys");
    } else {
      p->coarse_f = 0;
      cudaGetLastError();
    }
  }
  MPG_CUDA(cudaGetLastError());
  return MPGPU_OK;
}

mpgpu_status mpgpu_plan_coarse_key_ptrs(mpgpu_plan* p, int64_t** d_row_keys, int64_t** d_col_keys) {
  if (!p || !d_row_keys || !d_col_keys) return fail(MPGPU_EPARAM, "null argument");
  *d_row_keys = *d_col_keys = nullptr;
  if (p->coarse_f <= 0 || p->subset) return MPGPU_OK;
  MPG_CUDA(cudaSetDevice(p->device));
  if (mpgpu_status st = ensure_coarse(p); st != MPGPU_OK) return st;
  *d_row_keys = (int64_t*)key_row(p->coarse);
  *d_col_keys = (int64_t*)key_col(p->coarse);
  p->coarse_keys_shared = true;
  return MPGPU_OK;
}

mpgpu_status mpgpu_plan_attach_coarse_keys(mpgpu_plan* p, int64_t* d_row_keys, int64_t* d_col_keys) {
  if (!p) return fail(MPGPU_EPARAM, "null plan");
  if (p->coarse_f <= 0) {
    if (d_row_keys) return fail(MPGPU_EPARAM, "plan has no coarse phase");
    return MPGPU_OK;
  }
  MPG_CUDA(cudaSetDevice(p->device));
  if (mpgpu_status st = ensure_coarse(p); st != MPGPU_OK) return st;
  if (mpgpu_status st = mpgpu_plan_attach_keys(p->coarse, d_row_keys, d_col_keys); st != MPGPU_OK)
    return st;
  p->coarse_keys_shared = d_row_keys != nullptr;
  return MPGPU_OK;
}

mpgpu_status mpgpu_plan_coarse_run(mpgpu_plan* p, int32_t shard, int32_t n_shards) {
  Range nvtx_range("mpgpu:coarse_run (K2b coarse join)");
  if (!p) return fail(MPGPU_EPARAM, "null plan");
  if (!p->coarse_pending || !p->coarse) return MPGPU_OK;
  MPG_CUDA(cudaSetDevice(p->device));
  const long long before = p->coarse->launches;  // its prepare was counted by coarse_begin
  if (mpgpu_status st = mpgpu_plan_run(p->coarse, shard, n_shards); st != MPGPU_OK) return st;
  p->launches += p->coarse->launches - before;
  return MPGPU_OK;
}

mpgpu_status mpgpu_plan_seed_shared(mpgpu_plan* p, int32_t shard, int32_t n_shards) {
  Range nvtx_range("mpgpu:seed_shared (K2 warm start)");
  if (!p) return fail(MPGPU_EPARAM, "null plan");
  if (n_shards < 1 || shard < 0 || shard >= n_shards) return fail(MPGPU_EPARAM, "bad shard");
  MPG_CUDA(cudaSetDevice(p->device));
  launch_init(p, shard, n_shards);
  if (p->coarse_pending) {
    p->coarse_pending = false;
    if (mpgpu_status st = coarse_finish(p, shard, n_shards); st != MPGPU_OK) return st;
  }
  MPG_CUDA(cudaGetLastError());
  return MPGPU_OK;
}

mpgpu_status mpgpu_plan_reset_keys(mpgpu_plan* p) {
  if (!p) return fail(MPGPU_EPARAM, "null plan");
  if (p->ext_key0 && !p->ext_owner)
    return fail(MPGPU_EPARAM, "an attached plan does not own its keys");
  MPG_CUDA(cudaSetDevice(p->device));
  const long long L1 = p->self ? p->A.L : p->B.L;
  k_fill_keys<<<(unsigned)((p->A.L + 255) / 256), 256, 0, p->stream>>>(key_row(p), p->A.L);
  k_fill_keys<<<(unsigned)((L1 + 255) / 256), 256, 0, p->stream>>>(key_col(p), L1);
  p->launches += 2;
  MPG_CUDA(cudaGetLastError());
  return MPGPU_OK;
}

mpgpu_status mpgpu_plan_prepare_shard(mpgpu_plan* p, int32_t shard, int32_t n_shards) {
  Range nvtx_range("mpgpu:prepare (K1 stats, K2 warm start)");
  if (!p) return fail(MPGPU_EPARAM, "null plan");
  if (n_shards < 1 || shard < 0 || shard >= n_shards) return fail(MPGPU_EPARAM, "bad shard");
  p->coarse_pending = false;
  MPG_CUDA(cudaSetDevice(p->device));
  p->launches = 0;
  mpgpu_status st = launch_stats(p, p->A);
  if (st != MPGPU_OK) return st;
  if (!p->self && (st = launch_stats(p, p->B)) != MPGPU_OK) return st;
  if (p->ext_key0 && !p->ext_owner) {
    // keys belong to the owning plan, which initialises them. With several
    // shards this plan still runs its shard of the coarse warm-start join (on
    // its own coarse keys): the caller MIN-merges the coarse keys across ranks
    // and the owner seeds the shared keys from them (prepare_finish).
    if (n_shards > 1 && !p->subset && p->coarse_f > 0) {
      if (coarse_begin(p, shard, n_shards) == MPGPU_OK) {
        p->coarse_pending = true;
      } else {
        p->coarse_f = 0;
        cudaGetLastError();
      }
    }
    MPG_CUDA(cudaGetLastError());
    return MPGPU_OK;
  }
  const long long L1 = p->self ? p->A.L : p->B.L;
  k_fill_keys<<<(unsigned)((p->A.L + 255) / 256), 256, 0, p->stream>>>(key_row(p), p->A.L);
  k_fill_keys<<<(unsigned)((L1 + 255) / 256), 256, 0, p->stream>>>(key_col(p), L1);
  p->launches += 2;
  // warm-start keys on a few spread diagonals of every pass (full runs only:
  // an anytime run must not see cells outside its bands)
  launch_init(p, 0, 1);
  const JoinParams P = make_params(p);
  const int npass = p->subset ? 0 : (p->self ? 1 : 2);
  if (p->subset && p->n_init_diags > 0) {
    // anytime run: warm start on diagonals of the chosen bands only (they are
    // cells of this run), so no row's first visit fires every warp
    const Pass& ps = P.pass[0];
    const int n_init = p->n_init_diags;
    dim3 grid((unsigned)((ps.R.L + (long long)kInitWarps * kInitRows - 1) /
                         ((long long)kInitWarps * kInitRows)),
              (unsigned)n_init);
    k_init_keys<<<grid, kInitWarps * 32, 0, p->stream>>>(ps, p->zone + 1, ps.C.L, (int)p->m,
                                                         p->imask, p->d_init_diags, 0, 1, n_init);
    p->launches += 1;
  }
  if (p->subset && !p->diag_mode && p->coarse_f > 0 && !p->coarse_diags.empty()) {
    // anytime band subset: the coarse warm start restricted to the coarse
    // diagonals the chosen bands map to (a diagonal-subset join of the PAA
    // series), its exploit seeding only the chosen bands' diagonals
    bool ok = ensure_coarse(p) == MPGPU_OK;
    if (ok && p->coarse_diags_dirty) {
      ok = plan_select_diagonals(p->coarse, p->coarse_diags) == MPGPU_OK;
      p->coarse_diags_dirty = !ok;
    }
    if (ok && coarse_begin(p, 0, 1) == MPGPU_OK) {
      p->coarse_pending = true;
    } else {
      cudaGetLastError();
    }
  }
  if (p->mask_mode && p->coarse_f > 0) {
    // masked bands: the whole coarse join (the PAA keys only point at fine
    // diagonals; the exploit then evaluates the chosen ones among them)
    bool ok = ensure_coarse(p) == MPGPU_OK;
    if (ok && p->coarse->subset) ok = mpgpu_plan_select_bands(p->coarse, nullptr, -1) == MPGPU_OK;
    if (ok && coarse_begin(p, 0, 1) == MPGPU_OK) {
      p->coarse_pending = true;
    } else {
      cudaGetLastError();
    }
  }
  if (npass > 0 && p->coarse_f > 0) {
    // the coarse phase only tightens the filter: if it cannot run (e.g. the
    // nested plan's allocations fail), the join proceeds without it
    if (coarse_begin(p, shard, n_shards) == MPGPU_OK) {
      p->coarse_pending = true;
    } else {
      p->coarse_f = 0;
      cudaGetLastError();  // clear a non-sticky error; a sticky one resurfaces below
    }
  }
  MPG_CUDA(cudaGetLastError());
  return MPGPU_OK;
}

int64_t mpgpu_plan_shard_cells(const mpgpu_plan* p, int32_t shard, int32_t n_shards) {
  if (!p || n_shards < 1 || shard < 0 || shard >= n_shards) return 0;
  long long c = 0;
  for (size_t q = (size_t)shard; q < p->items.size(); q += (size_t)n_shards) c += p->item_cells[q];
  return c;
}

mpgpu_status mpgpu_plan_run(mpgpu_plan* p, int32_t shard, int32_t n_shards) {
  Range nvtx_range("mpgpu:run (K3 k_join)");
  if (!p) return fail(MPGPU_EPARAM, "null plan");
  if (n_shards < 1 || shard < 0 || shard >= n_shards) return fail(MPGPU_EPARAM, "bad shard");
  MPG_CUDA(cudaSetDevice(p->device));
  if (p->diag_mode) {
    if (n_shards != 1) return fail(MPGPU_EUNSUPPORTED, "diagonal-subset runs are not sharded");
    if (p->n_ditems == 0) return MPGPU_OK;
    MPG_CUDA(cudaMemsetAsync(p->d_counter, 0, sizeof(int), p->stream));
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, p->device);
    const int grid = (int)std::min<long long>((p->n_ditems + 7) / 8, (long long)sms * 8);
    k_diag_join<<<grid, 256, 0, p->stream>>>(p->A.view(), key_row(p), key_col(p), p->d_diags,
                                             p->n_diags, p->d_ditems, p->n_ditems, p->d_counter,
                                             p->diag_rows, (int)p->m, p->imask);
    p->launches += 1;
    MPG_CUDA(cudaGetLastError());
    return MPGPU_OK;
  }
  // each shard uses its own slice of the device item buffer (shards may be
  // in flight together on one device); a slice is uploaded on its first run
  // and reused while the sharding and the band selection stay the same
  size_t off = 0;
  for (int s = 0; s < shard; ++s) off += (p->items.size() + n_shards - 1 - s) / n_shards;
  if (p->slice_n != n_shards) {
    p->slice_ok.assign((size_t)n_shards, 0);
    p->slice_cnt.assign((size_t)n_shards, 0);
    p->slice_n = n_shards;
  }
  if (!p->slice_ok[(size_t)shard]) {
    std::vector<Item> mine;
    shard_items(p, shard, n_shards, mine, nullptr);
    if (p->subset) {
      // keep the chosen bands' items; every 8th chosen band goes first (a probe:
      // the rest of the run then starts from thresholds that already reflect a
      // sample of the whole subset, so far fewer cells fire). Order never changes
      // the result: the min-merge is exact and ties go to the smaller index.
      std::vector<Item> probe, rest;
      for (const Item& it : mine) {
        const auto bd = std::lower_bound(p->bands.begin(), p->bands.end(), it.kb);
        if (bd == p->bands.end() || *bd != it.kb) continue;
        ((bd - p->bands.begin()) % 8 == 0 ? probe : rest).push_back(it);
      }
      probe.insert(probe.end(), rest.begin(), rest.end());
      mine.swap(probe);
    }
    if (!mine.empty())
      MPG_CUDA(cudaMemcpyAsync(p->d_items + off, mine.data(), sizeof(Item) * mine.size(),
                               cudaMemcpyHostToDevice, p->stream));
    p->slice_cnt[(size_t)shard] = (long long)mine.size();
    p->slice_ok[(size_t)shard] = 1;
  }
  const long long n_mine = p->slice_cnt[(size_t)shard];
  if (n_mine == 0) return MPGPU_OK;
  MPG_CUDA(cudaMemsetAsync(p->d_counter, 0, sizeof(int), p->stream));
  JoinParams P = make_params(p);
  P.items = p->d_items + off;
  P.n_items = (int)n_mine;
  P.counter = p->d_counter;
  const int grid = (int)std::min<long long>((n_mine + kWarps - 1) / kWarps, p->n_ctas);
  if (p->mask_mode) {
    MaskedParams MP;
    MP.J = P;
    MP.dmasks = p->d_dmasks;
    MP.klo = p->zone + 1;
    k_join_masked<<<grid, kThreads, sizeof(JoinSmem), p->stream>>>(MP);
    p->launches += 1;
    MPG_CUDA(cudaGetLastError());
    return MPGPU_OK;
  }
  static const bool want_stats = getenv("MPGPU_STATS") && atoi(getenv("MPGPU_STATS")) > 0;
  unsigned long long* d_stats = nullptr;
  if (want_stats) {
    MPG_CUDA(cudaMalloc(&d_stats, 8 * sizeof(unsigned long long)));
    MPG_CUDA(cudaMemsetAsync(d_stats, 0, 8 * sizeof(unsigned long long), p->stream));
    P.stats = d_stats;
  }
  k_join<<<grid, kThreads, sizeof(JoinSmem), p->stream>>>(P);
  p->launches += 1;
  MPG_CUDA(cudaGetLastError());
  if (want_stats) {
    unsigned long long h[8];
    MPG_CUDA(cudaMemcpyAsync(h, d_stats, sizeof(h), cudaMemcpyDeviceToHost, p->stream));
    MPG_CUDA(cudaStreamSynchronize(p->stream));
    long long cells = 0;
    for (size_t q = (size_t)shard; q < p->items.size(); q += (size_t)n_shards) cells += p->item_cells[q];
    fprintf(stderr, "[mpgpu stats] cells %lld warp_row_steps %.3e slow_entries %llu (%.4f%%) row_cand %llu col_cand %llu replayed_blocks %llu (%.4f%% of blocks)\n",
            cells, cells / 256.0, h[0], 100.0 * h[0] / (cells / 256.0), h[1], h[2], h[3],
            100.0 * h[3] / (cells / 256.0 / kD));
    cudaFree(d_stats);
  }
  return MPGPU_OK;
}

mpgpu_status mpgpu_plan_keys(mpgpu_plan* p, int64_t** d_row_keys, int64_t* row_len,
                             int64_t** d_col_keys, int64_t* col_len) {
  if (!p) return fail(MPGPU_EPARAM, "null plan");
  if (d_row_keys) *d_row_keys = (int64_t*)key_row(p);
  if (row_len) *row_len = p->A.L;
  if (d_col_keys) *d_col_keys = (int64_t*)key_col(p);
  if (col_len) *col_len = p->self ? p->A.L : p->B.L;
  return MPGPU_OK;
}

mpgpu_status mpgpu_plan_finalize(mpgpu_plan* p, double* d_mp_a, int64_t* d_pi_a,
                                 int64_t* d_left_a, int64_t* d_right_a, double* d_mp_b,
                                 int64_t* d_pi_b) {
  return mpgpu_plan_finalize_shard(p, 0, 1, d_mp_a, d_pi_a, d_left_a, d_right_a, d_mp_b, d_pi_b);
}

mpgpu_status mpgpu_plan_finalize_shard(mpgpu_plan* p, int32_t shard, int32_t n_shards,
                                       double* d_mp_a, int64_t* d_pi_a, int64_t* d_left_a,
                                       int64_t* d_right_a, double* d_mp_b, int64_t* d_pi_b) {
  Range nvtx_range("mpgpu:finalize (K4)");
  if (!p) return fail(MPGPU_EPARAM, "null plan");
  if (n_shards < 1 || shard < 0 || shard >= n_shards) return fail(MPGPU_EPARAM, "bad shard");
  MPG_CUDA(cudaSetDevice(p->device));
  const int bs = 256;
  auto rows = [&](long long L, long long& r0, long long& r1) {
    r0 = L * shard / n_shards;
    r1 = L * (shard + 1) / n_shards;
    return r1 > r0;
  };
  auto grid = [&](long long nrows) { return (unsigned)((nrows * kFinLanes + bs - 1) / bs); };
  long long r0, r1;
  if (p->diag_mode) {
    if (n_shards != 1) return fail(MPGPU_EUNSUPPORTED, "anytime runs finalize in one piece");
    k_finalize_keys<<<grid(p->A.L), bs, 0, p->stream>>>(p->A.view(), key_row(p), key_col(p),
                                                         (int)p->m, p->imask, d_mp_a,
                                                         (long long*)d_pi_a, (long long*)d_left_a,
                                                         (long long*)d_right_a);
    p->launches += 1;
  } else if (p->mask_mode) {
    if (n_shards != 1) return fail(MPGPU_EUNSUPPORTED, "anytime runs finalize in one piece");
    const long long thr = p->A.L * 32;
    k_finalize_self_masked<<<(unsigned)((thr + bs - 1) / bs), bs, 0, p->stream>>>(
        p->A.view(), key_row(p), key_col(p), (int)p->m, p->imask, p->d_diag_bits, p->d_diags,
        p->n_diags, d_mp_a, (long long*)d_pi_a, (long long*)d_left_a, (long long*)d_right_a);
    p->launches += 1;
  } else if (p->self && p->subset) {
    if (n_shards != 1) return fail(MPGPU_EUNSUPPORTED, "anytime runs finalize in one piece");
    const long long thr = p->A.L * 32;
    k_finalize_self_partial<<<(unsigned)((thr + bs - 1) / bs), bs, 0, p->stream>>>(
        p->A.view(), key_row(p), key_col(p), (int)p->m, p->imask, p->d_bands, (int)p->bands.size(),
        p->A.L, d_mp_a, (long long*)d_pi_a, (long long*)d_left_a, (long long*)d_right_a);
    p->launches += 1;
  } else if (p->self) {
    if (rows(p->A.L, r0, r1)) {
      k_finalize_self<<<grid(r1 - r0), bs, 0, p->stream>>>(
          p->A.view(), key_row(p), key_col(p), p->zone, (int)p->m, p->imask, r0, r1, d_mp_a,
          (long long*)d_pi_a, (long long*)d_left_a, (long long*)d_right_a);
      p->launches += 1;
    }
  } else {
    if ((d_mp_a || d_pi_a) && rows(p->A.L, r0, r1)) {
      k_finalize_ab<<<grid(r1 - r0), bs, 0, p->stream>>>(p->A.view(), p->B.view(), key_row(p),
                                                          (int)p->m, p->imask, r0, r1, d_mp_a,
                                                          (long long*)d_pi_a);
      p->launches += 1;
    }
    if ((d_mp_b || d_pi_b) && rows(p->B.L, r0, r1)) {
      k_finalize_ab<<<grid(r1 - r0), bs, 0, p->stream>>>(p->B.view(), p->A.view(), key_col(p),
                                                          (int)p->m, p->imask, r0, r1, d_mp_b,
                                                          (long long*)d_pi_b);
      p->launches += 1;
    }
  }
  MPG_CUDA(cudaGetLastError());
  return MPGPU_OK;
}

int64_t mpgpu_plan_num_bands(const mpgpu_plan* p) {
  if (!p || !p->self) return 0;
  const long long klo = p->zone + 1, L = p->A.L;
  return L > klo ? (L - klo + kW - 1) / kW : 0;
}

mpgpu_status mpgpu_plan_attach_keys(mpgpu_plan* p, int64_t* d_row_keys, int64_t* d_col_keys) {
  if (!p) return fail(MPGPU_EPARAM, "null plan");
  if ((d_row_keys == nullptr) != (d_col_keys == nullptr))
    return fail(MPGPU_EPARAM, "attach both key arrays or neither");
  p->ext_key0 = (long long*)d_row_keys;
  p->ext_key1 = (long long*)d_col_keys;
  if (!d_row_keys) p->ext_owner = false;
  return MPGPU_OK;
}

namespace {
// Layout of a plan's keys in a shared key region: fine row keys, fine column
// keys, then (with a coarse phase) the coarse row and column keys, each
// 256-byte aligned. The same problem gives the same layout on every rank.
struct KeyLayout { long long off[4]; long long bytes; bool coarse; };
KeyLayout key_layout(const mpgpu_plan* p) {
  auto up = [](long long b) { return (b + 255) / 256 * 256; };
  KeyLayout k{};
  const long long Lb = p->self ? p->A.L : p->B.L;
  k.off[0] = 0;
  k.off[1] = up(8 * (p->A.L + kPad));  // padded like the plan's own key arrays
  long long end = k.off[1] + up(8 * (Lb + kPad));
  k.coarse = p->coarse_f > 0 && !p->subset;
  if (k.coarse) {
    const long long f = p->coarse_f, mc = p->m / f;
    const long long Lca = p->A.n / f - mc + 1, Lcb = p->self ? Lca : p->B.n / f - mc + 1;
    k.off[2] = end;
    k.off[3] = end + up(8 * (Lca + kPad));
    end = k.off[3] + up(8 * (Lcb + kPad));
  }
  k.bytes = end;
  return k;
}
}  // namespace

int64_t mpgpu_plan_key_region_bytes(const mpgpu_plan* p) { return p ? key_layout(p).bytes : 0; }

// Chunk owners of a striped key region that balance the key traffic per GPU.
// Model: every 32-row tile of a work item reads 32 row keys and 32 column keys
// (k_join's per-tile prefetch), so item (kb, r0, nrows) reads row keys
// [r0, r0 + nrows) and column keys [r0 + kb, r0 + kb + nrows + kW - 1) once
// each. Self-join rows near 0 and columns near L carry the most cells, so the
// hot chunks sit at the two ends of the fine keys; chunks are dealt
// largest-load-first to the least-loaded rank (LPT). The coarse keys (a join
// of 1/f^2 of the cells) are modelled as free.
int64_t mpgpu_plan_key_region_owners(const mpgpu_plan* p, int64_t chunk_bytes, int32_t n_ranks,
                                     int32_t* owners, int64_t cap, double* max_share) {
  if (!p || chunk_bytes <= 0 || n_ranks < 1) return -1;
  const KeyLayout k = key_layout(p);
  const long long nch = (k.bytes + chunk_bytes - 1) / chunk_bytes;
  if (!owners || cap < nch) return nch;
  std::vector<double> load((size_t)nch, 0.0);
  auto add = [&](long long base, long long i0, long long i1) {  // keys [i0, i1) of one array
    if (i1 <= i0) return;
    long long b0 = base + 8 * i0;
    const long long b1 = base + 8 * i1;
    while (b0 < b1) {
      const long long c = b0 / chunk_bytes;
      const long long e = std::min(b1, (c + 1) * chunk_bytes);
      load[(size_t)c] += (double)(e - b0) / 8.0;
      b0 = e;
    }
  };
  const long long Lb = p->self ? p->A.L : p->B.L;
  for (const Item& it : p->items) {
    // pass 0: rows A (row keys at off[0]), columns B / A (column keys at off[1]);
    // pass 1 (AB): rows B (keys at off[1]), columns A (keys at off[0])
    const bool p1 = it.pass == 1;
    const long long LR = p1 ? Lb : p->A.L, LC = p1 ? p->A.L : Lb;
    const long long offR = p1 ? k.off[1] : k.off[0], offC = p1 ? k.off[0] : k.off[1];
    add(offR, it.r0, std::min(LR, it.r0 + it.nrows));
    const long long c0 = it.r0 + it.kb;
    add(offC, std::min(LC, c0), std::min(LC, c0 + it.nrows + kW - 1));
  }
  std::vector<long long> order((size_t)nch);
  for (long long c = 0; c < nch; ++c) order[(size_t)c] = c;
  std::stable_sort(order.begin(), order.end(),
                   [&](long long a, long long b) { return load[(size_t)a] > load[(size_t)b]; });
  std::vector<double> per(n_ranks, 0.0);
  double total = 0.0;
  for (long long c : order) {
    int best = 0;
    for (int r = 1; r < n_ranks; ++r)
      if (per[r] < per[best]) best = r;
    owners[c] = best;
    per[best] += load[(size_t)c];
    total += load[(size_t)c];
  }
  if (max_share) *max_share = total > 0 ? *std::max_element(per.begin(), per.end()) / total : 0.0;
  return nch;
}

mpgpu_status mpgpu_plan_attach_key_region(mpgpu_plan* p, void* d_base, int64_t bytes, int32_t owner) {
  if (!p) return fail(MPGPU_EPARAM, "null plan");
  MPG_CUDA(cudaSetDevice(p->device));
  if (!d_base) {
    p->ext_key0 = p->ext_key1 = nullptr;
    p->ext_owner = false;
    if (p->coarse) {
      p->coarse->ext_key0 = p->coarse->ext_key1 = nullptr;
      p->coarse->ext_owner = false;
    }
    p->coarse_keys_shared = false;
    return MPGPU_OK;
  }
  const KeyLayout k = key_layout(p);
  if (bytes < k.bytes) return fail(MPGPU_EPARAM, "key region too small for this plan");
  char* b = static_cast<char*>(d_base);
  p->ext_key0 = reinterpret_cast<long long*>(b + k.off[0]);
  p->ext_key1 = reinterpret_cast<long long*>(b + k.off[1]);
  p->ext_owner = owner != 0;
  p->coarse_keys_shared = false;
  if (k.coarse) {
    if (mpgpu_status st = ensure_coarse(p); st != MPGPU_OK) return st;
    p->coarse->ext_key0 = reinterpret_cast<long long*>(b + k.off[2]);
    p->coarse->ext_key1 = reinterpret_cast<long long*>(b + k.off[3]);
    p->coarse->ext_owner = owner != 0;
    p->coarse_keys_shared = true;
  }
  return MPGPU_OK;
}

mpgpu_status mpgpu_plan_select_bands(mpgpu_plan* p, const int64_t* band_ids, int64_t n) {
  if (!p) return fail(MPGPU_EPARAM, "null plan");
  if (n < 0 || !band_ids) {  // back to the full join
    if (p->subset) p->slice_n = 0;
    p->subset = false;
    p->diag_mode = false;
    p->mask_mode = false;
    p->bands.clear();
    p->coarse_diags.clear();
    if (p->coarse && p->coarse->subset) mpgpu_plan_select_bands(p->coarse, nullptr, -1);
    return MPGPU_OK;
  }
  p->diag_mode = false;
  p->mask_mode = false;
  if (!p->self) return fail(MPGPU_EUNSUPPORTED, "band subsets (anytime SCRIMP) are self-join only");
  const long long nb = mpgpu_plan_num_bands(p), klo = p->zone + 1;
  std::vector<long long> kb;
  for (int64_t q = 0; q < n; ++q) {
    if (band_ids[q] < 0 || band_ids[q] >= nb) return fail(MPGPU_EPARAM, "band id out of range");
    kb.push_back(klo + band_ids[q] * (long long)kW);
  }
  std::sort(kb.begin(), kb.end());
  kb.erase(std::unique(kb.begin(), kb.end()), kb.end());
  MPG_CUDA(cudaSetDevice(p->device));
  cudaFree(p->d_bands);
  p->d_bands = nullptr;
  if (!kb.empty()) {
    MPG_CUDA(cudaMalloc(&p->d_bands, sizeof(long long) * kb.size()));
    MPG_CUDA(cudaMemcpyAsync(p->d_bands, kb.data(), sizeof(long long) * kb.size(),
                             cudaMemcpyHostToDevice, p->stream));
    MPG_CUDA(cudaStreamSynchronize(p->stream));
  }
  // warm-start diagonals: the middle diagonal of up to kInitDiag chosen bands,
  // spread over the chosen list
  std::vector<long long> wd;
  const long long L = p->A.L;
  const int nw = (int)std::min<size_t>(kInitDiag, kb.size());
  for (int q = 0; q < nw; ++q) {
    const long long k = std::min(kb[(size_t)q * kb.size() / nw] + kW / 2, L - 1);
    if (k > p->zone && (wd.empty() || wd.back() != k)) wd.push_back(k);
  }
  cudaFree(p->d_init_diags);
  p->d_init_diags = nullptr;
  p->n_init_diags = 0;
  if (!wd.empty()) {
    MPG_CUDA(cudaMalloc(&p->d_init_diags, sizeof(long long) * wd.size()));
    MPG_CUDA(cudaMemcpy(p->d_init_diags, wd.data(), sizeof(long long) * wd.size(),
                        cudaMemcpyHostToDevice));
    p->n_init_diags = (int)wd.size();
  }
  // band bitmask for the coarse exploit, and the coarse diagonals the bands
  // map to (fine diagonal k ~ coarse diagonal k / f, one either side)
  {
    const long long nbt = std::max<long long>(1, mpgpu_plan_num_bands(p));
    std::vector<unsigned> mask((size_t)((nbt + 31) / 32), 0u);
    for (long long k0 : kb) {
      const long long b = (k0 - klo) / kW;
      mask[(size_t)(b >> 5)] |= 1u << (b & 31);
    }
    cudaFree(p->d_band_mask);
    p->d_band_mask = nullptr;
    MPG_CUDA(cudaMalloc(&p->d_band_mask, sizeof(unsigned) * mask.size()));
    MPG_CUDA(cudaMemcpy(p->d_band_mask, mask.data(), sizeof(unsigned) * mask.size(),
                        cudaMemcpyHostToDevice));
    p->coarse_diags.clear();
    if (p->coarse_f > 0) {
      const long long f = p->coarse_f, mc = p->m / f;
      const long long Lc = p->A.n / f - mc + 1, zc = (p->zone + f - 1) / f;
      for (long long k0 : kb) {
        const long long lo = std::max(zc + 1, k0 / f - 1);
        const long long hi = std::min(Lc - 1, (k0 + kW - 1) / f + 1);
        for (long long K = lo; K <= hi; ++K)
          if (p->coarse_diags.empty() || p->coarse_diags.back() < K) p->coarse_diags.push_back(K);
      }
    }
    p->coarse_diags_dirty = true;
  }
  p->bands.swap(kb);
  p->subset = true;
  p->slice_n = 0;  // item order changed: re-upload on the next run
  return MPGPU_OK;
}

}  // extern "C"

namespace {
// Anytime mode over an explicit diagonal set (ascending, > zone, < L): work
// items are 32 consecutive diagonals x a segment of rows, largest first; the
// warm start uses up to kInitDiag diagonals spread over the set.
mpgpu_status plan_select_diagonals(mpgpu_plan* p, const std::vector<long long>& diags) {
  if (!p->self) return fail(MPGPU_EUNSUPPORTED, "diagonal subsets (anytime SCRIMP) are self-join only");
  MPG_CUDA(cudaSetDevice(p->device));
  const long long L = p->A.L;
  cudaFree(p->d_diags);
  cudaFree(p->d_ditems);
  p->d_diags = nullptr;
  p->d_ditems = nullptr;
  p->n_diags = (long long)diags.size();
  // rows per item: long enough that the m-term seed is small against the walk
  // (>= 8m), short enough to spread the set over every warp
  const long long groups = (p->n_diags + 31) / 32;
  long long cells = 0;
  for (long long k : diags) cells += L - k;
  const long long workers = 148LL * 64;
  long long rows = std::max<long long>(8 * p->m, cells / std::max<long long>(1, 32 * 4 * workers));
  rows = std::max<long long>(256, std::min<long long>(rows, 1 << 20));
  p->diag_rows = (int)rows;
  std::vector<std::pair<long long, DiagItem>> its;
  for (long long g = 0; g < groups; ++g) {
    const long long kmin = diags[(size_t)(g * 32)];  // ascending: the group's longest diagonal
    const long long nrows = L - kmin;
    for (long long s0 = 0; s0 * rows < nrows; ++s0) {
      DiagItem it;
      it.group = (int)g;
      it.seg = (int)s0;
      its.push_back({std::min(rows, nrows - s0 * rows), it});
    }
  }
  std::stable_sort(its.begin(), its.end(), [](const auto& a, const auto& b) { return a.first > b.first; });
  std::vector<DiagItem> h(its.size());
  for (size_t q = 0; q < its.size(); ++q) h[q] = its[q].second;
  p->n_ditems = (int)h.size();
  if (!diags.empty()) {
    MPG_CUDA(cudaMalloc(&p->d_diags, sizeof(long long) * diags.size()));
    MPG_CUDA(cudaMemcpy(p->d_diags, diags.data(), sizeof(long long) * diags.size(),
                        cudaMemcpyHostToDevice));
  }
  if (!h.empty()) {
    MPG_CUDA(cudaMalloc(&p->d_ditems, sizeof(DiagItem) * h.size()));
    MPG_CUDA(cudaMemcpy(p->d_ditems, h.data(), sizeof(DiagItem) * h.size(), cudaMemcpyHostToDevice));
  }
  std::vector<long long> wd;
  const int nw = (int)std::min<size_t>(kInitDiag, diags.size());
  for (int q = 0; q < nw; ++q) {
    const long long k = diags[(size_t)q * diags.size() / nw];
    if (wd.empty() || wd.back() != k) wd.push_back(k);
  }
  cudaFree(p->d_init_diags);
  p->d_init_diags = nullptr;
  p->n_init_diags = 0;
  if (!wd.empty()) {
    MPG_CUDA(cudaMalloc(&p->d_init_diags, sizeof(long long) * wd.size()));
    MPG_CUDA(cudaMemcpy(p->d_init_diags, wd.data(), sizeof(long long) * wd.size(),
                        cudaMemcpyHostToDevice));
    p->n_init_diags = (int)wd.size();
  }
  p->bands.clear();
  p->coarse_diags.clear();
  p->subset = true;
  p->diag_mode = true;
  p->mask_mode = false;
  p->slice_n = 0;
  // Dense sets: from about 9% of all diagonals on, nearly every band of kW holds
  // a chosen one and one diagonal per lane costs more than whole bands. Then the
  // bands that hold a chosen diagonal run through k_join_masked (the band-subset
  // machinery with per-lane diagonal masks), and the finalize checks
  // admissibility per diagonal (k_finalize_self_masked).
  static const double dense = getenv("MPGPU_MASK_MIN_DENSITY") ? atof(getenv("MPGPU_MASK_MIN_DENSITY")) : 0.09;
  const long long klo = p->zone + 1, nd = L - klo;
  if (nd > 0 && !diags.empty() && (double)diags.size() >= dense * (double)nd) {
    const long long nbt = std::max<long long>(1, mpgpu_plan_num_bands(p));
    std::vector<unsigned char> dm((size_t)nbt * 32, 0);
    std::vector<uint32_t> bits((size_t)((L + 31) / 32), 0u);
    std::vector<long long> kb;
    for (long long k : diags) {
      const long long o = k - klo, b = o / kW;
      dm[(size_t)(b * 32 + (o % kW) / kD)] |= (unsigned char)(1u << (o % kD));
      bits[(size_t)(k >> 5)] |= 1u << (k & 31);
      if (kb.empty() || kb.back() != klo + b * kW) kb.push_back(klo + b * kW);  // diags ascend
    }
    cudaFree(p->d_dmasks);
    cudaFree(p->d_diag_bits);
    p->d_dmasks = nullptr;
    p->d_diag_bits = nullptr;
    MPG_CUDA(cudaMalloc(&p->d_dmasks, dm.size()));
    MPG_CUDA(cudaMemcpy(p->d_dmasks, dm.data(), dm.size(), cudaMemcpyHostToDevice));
    MPG_CUDA(cudaMalloc(&p->d_diag_bits, sizeof(uint32_t) * bits.size()));
    MPG_CUDA(cudaMemcpy(p->d_diag_bits, bits.data(), sizeof(uint32_t) * bits.size(), cudaMemcpyHostToDevice));
    p->bands.swap(kb);
    p->diag_mode = false;
    p->mask_mode = true;
  }
  return MPGPU_OK;
}
}  // namespace

extern "C" {

int64_t mpgpu_scrimp_diagonals(int64_t n, int64_t window, int64_t zone, int64_t s_size,
                               uint64_t seed, int64_t* out_diags, int64_t cap, double* coverage) {
  const long long L = n - window + 1, klo = zone + 1;
  const long long nd = L > klo ? L - klo : 0;
  // SCRIMP's seeded diagonal order: Fisher-Yates over the
  // admissible diagonals with splitmix64, the first s_size of them
  std::vector<long long> order((size_t)nd);
  for (long long q = 0; q < nd; ++q) order[(size_t)q] = klo + q;
  uint64_t st = seed;
  auto next = [&st]() {
    uint64_t z = (st += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
  };
  for (long long q = nd - 1; q > 0; --q) {
    const long long r = (long long)(next() % (uint64_t)(q + 1));
    std::swap(order[(size_t)q], order[(size_t)r]);
  }
  const long long take = (s_size <= 0 || s_size >= nd) ? nd : s_size;
  std::sort(order.begin(), order.begin() + take);
  for (long long q = 0; q < take && q < cap; ++q) out_diags[q] = order[(size_t)q];
  if (coverage) *coverage = nd > 0 ? (double)take / (double)nd : 1.0;
  return take;
}

int64_t mpgpu_scrimp_bands(int64_t n, int64_t window, int64_t zone, int64_t s_size, uint64_t seed,
                           int64_t* out_bands, int64_t cap, double* coverage) {
  const long long L = n - window + 1, klo = zone + 1;
  const long long ndiag = L > klo ? L - klo : 0;
  const long long nb = ndiag > 0 ? (ndiag + kW - 1) / kW : 0;
  // seeded Fisher-Yates over bands (splitmix64), the band-granular analogue of
  // SCRIMP's seeded diagonal order
  std::vector<long long> order(nb);
  for (long long q = 0; q < nb; ++q) order[q] = q;
  uint64_t st = seed;
  auto next = [&st]() {
    uint64_t z = (st += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
  };
  for (long long q = nb - 1; q > 0; --q) {
    const long long r = (long long)(next() % (uint64_t)(q + 1));
    std::swap(order[q], order[r]);
  }
  long long covered = 0, take = 0;
  const long long want = (s_size <= 0 || s_size >= ndiag) ? ndiag : s_size;
  while (take < nb && covered < want) {
    const long long b = order[take++];
    covered += std::min<long long>(kW, ndiag - b * (long long)kW);
  }
  std::sort(order.begin(), order.begin() + take);
  for (long long q = 0; q < take && q < cap; ++q) out_bands[q] = order[q];
  if (coverage) *coverage = ndiag > 0 ? (double)covered / (double)ndiag : 1.0;
  return take;
}

namespace {
// Scratch of the consumer entry points (FLUSS, MASS, extract), kept per
// (device, kind) across calls: a fresh allocation per call costs more than the
// work once the memory pool has trimmed it at a synchronisation. Calls of one
// kind on a device are serialised and each waits on the previous call's use
// of the buffer.
enum ScratchKind { kScratchFluss = 0, kScratchMass = 1, kScratchExtract = 2, kScratchKinds = 3 };
struct Scratch {
  std::mutex mu;
  char* p = nullptr;
  size_t cap = 0;
  cudaEvent_t done = nullptr;
};
Scratch g_scratch[64][kScratchKinds];

// Locks the (device, kind) scratch into `lk`, grows it to `need` bytes and
// orders `st` after its previous use. Pair with scratch_release on `st`.
mpgpu_status scratch_acquire(int device, int kind, size_t need, cudaStream_t st,
                             std::unique_lock<std::mutex>& lk, char** out) {
  if (device < 0 || device >= 64) return fail(MPGPU_EPARAM, "device out of range");
  Scratch& S = g_scratch[device][kind];
  lk = std::unique_lock<std::mutex>(S.mu);
  if (!S.done) MPG_CUDA(cudaEventCreateWithFlags(&S.done, cudaEventDisableTiming));
  if (S.cap < need) {
    MPG_CUDA(cudaEventSynchronize(S.done));
    if (S.p) MPG_CUDA(cudaFree(S.p));
    S.p = nullptr;
    S.cap = 0;
    if (cudaMalloc(&S.p, need) != cudaSuccess) return fail(MPGPU_ENOMEM, "consumer scratch");
    S.cap = need;
  }
  MPG_CUDA(cudaStreamWaitEvent(st, S.done, 0));
  *out = S.p;
  return MPGPU_OK;
}
mpgpu_status scratch_release(int device, int kind, cudaStream_t st) {
  MPG_CUDA(cudaEventRecord(g_scratch[device][kind].done, st));
  return MPGPU_OK;
}
}  // namespace

mpgpu_status mpgpu_distance_profiles(const double* d_ts, int64_t n, int64_t window,
                                     const double* d_queries, const int64_t* d_query_pos,
                                     int64_t n_queries, int64_t zone, double* d_out,
                                     int32_t device, void* cuda_stream) {
  if (!d_ts || !d_out || window < 4 || window > n) return fail(MPGPU_EPARAM, "window out of range");
  if ((d_queries == nullptr) == (d_query_pos == nullptr))
    return fail(MPGPU_EPARAM, "pass exactly one of query arrays or query positions");
  if (n_queries <= 0) return MPGPU_OK;
  if (n_queries > 65535) return fail(MPGPU_EPARAM, "at most 65535 queries per call");
  MPG_CUDA(cudaSetDevice(device));
  cudaStream_t st = (cudaStream_t)cuda_stream;
  const long long L = n - window + 1;
  std::unique_lock<std::mutex> lk;
  char* scratch = nullptr;
  if (mpgpu_status e = scratch_acquire(device, kScratchMass,
                                       sizeof(double) * (2 * L + 3 * n_queries + kMassConst), st, lk,
                                       &scratch);
      e != MPGPU_OK)
    return e;
  double* mu = reinterpret_cast<double*>(scratch);
  double* inv = mu + L;
  double* qstat = inv + L;
  double* stage = qstat + 3 * n_queries;
  launch_window_stats(d_ts, L, (int)window, mu, inv, nullptr, nullptr, st);
  k_query_stats<<<(unsigned)((n_queries + kQStatWarps - 1) / kQStatWarps), kQStatWarps * 32, 0, st>>>(
      d_ts, d_queries, (const long long*)d_query_pos, (int)n_queries, (int)window, qstat);
  const unsigned gx = (unsigned)((L + kMassTile - 1) / kMassTile);
  const int mpad = (int)((window + kMassR - 1) / kMassR * kMassR);
  static const bool use_const = !(getenv("MPGPU_MASS_CONST") && atoi(getenv("MPGPU_MASS_CONST")) == 0);
  if (use_const && mpad <= kMassConst) {
    // the centred queries through constant memory, as many per launch as fit
    // (the scratch lock and its event order the launches that share c_mass_q)
    const int per = kMassConst / mpad;
    for (long long q0 = 0; q0 < n_queries; q0 += per) {
      const int nq = (int)std::min<long long>(per, n_queries - q0);
      k_mass_stage<<<(unsigned)((nq * mpad + 255) / 256), 256, 0, st>>>(
          d_ts, d_queries, (const long long*)d_query_pos, qstat, (int)q0, nq, (int)window, mpad, stage);
      MPG_CUDA(cudaMemcpyToSymbolAsync(c_mass_q, stage, sizeof(double) * nq * mpad, 0,
                                       cudaMemcpyDeviceToDevice, st));
      k_mass<true><<<dim3(gx, (unsigned)nq), kMassThreads, 0, st>>>(
          d_ts, n, mu, inv, L, (int)window, d_queries, (const long long*)d_query_pos, qstat,
          zone < 0 ? -1 : zone, d_out, (int)q0, mpad);
    }
  } else {
    k_mass<false><<<dim3(gx, (unsigned)n_queries), kMassThreads, 0, st>>>(
        d_ts, n, mu, inv, L, (int)window, d_queries, (const long long*)d_query_pos, qstat,
        zone < 0 ? -1 : zone, d_out, 0, mpad);
  }
  MPG_CUDA(cudaGetLastError());
  return scratch_release(device, kScratchMass, st);
}

namespace {
// arg-extreme of a device array: two-level block reduction; result to host
mpgpu_status argext(const double* d_v, long long n, int sign, cudaStream_t st, double* tmp_v,
                    long long* tmp_i, double* val, long long* idx) {
  const int bs = 1024;
  long long nb = (n + bs - 1) / bs;
  k_argext<<<(unsigned)nb, bs, 0, st>>>(d_v, nullptr, n, sign, tmp_v, tmp_i);
  while (nb > 1) {
    const long long nb2 = (nb + bs - 1) / bs;
    k_argext<<<(unsigned)nb2, bs, 0, st>>>(tmp_v, tmp_i, nb, sign, tmp_v + nb, tmp_i + nb);
    MPG_CUDA(cudaMemcpyAsync(tmp_v, tmp_v + nb, sizeof(double) * nb2, cudaMemcpyDeviceToDevice, st));
    MPG_CUDA(cudaMemcpyAsync(tmp_i, tmp_i + nb, sizeof(long long) * nb2, cudaMemcpyDeviceToDevice, st));
    nb = nb2;
  }
  MPG_CUDA(cudaMemcpyAsync(val, tmp_v, sizeof(double), cudaMemcpyDeviceToHost, st));
  MPG_CUDA(cudaMemcpyAsync(idx, tmp_i, sizeof(long long), cudaMemcpyDeviceToHost, st));
  MPG_CUDA(cudaStreamSynchronize(st));
  return MPGPU_OK;
}
}  // namespace


mpgpu_status mpgpu_fluss(const int64_t* d_index, int64_t L, int64_t window, int64_t* d_arcs,
                         double* d_cac, int32_t device, void* cuda_stream) {
  if (!d_index || !d_arcs || L < 1 || window < 0) return fail(MPGPU_EPARAM, "bad FLUSS arguments");
  MPG_CUDA(cudaSetDevice(device));
  cudaStream_t st = (cudaStream_t)cuda_stream;
  if (L >= (1ll << 31)) return fail(MPGPU_EPARAM, "FLUSS: L must be below 2^31");
  const long long nt = (L + kScanTile - 1) / kScanTile;
  std::unique_lock<std::mutex> lk;
  char* scratch = nullptr;
  if (mpgpu_status e = scratch_acquire(device, kScratchFluss, sizeof(long long) * nt + sizeof(int) * L,
                                       st, lk, &scratch); e != MPGPU_OK)
    return e;
  long long* sums = reinterpret_cast<long long*>(scratch);
  int* diff = reinterpret_cast<int*>(sums + nt);
  MPG_CUDA(cudaMemsetAsync(diff, 0, sizeof(int) * L, st));
  k_arc_far_ends<<<(unsigned)((L + 255) / 256), 256, 0, st>>>((const long long*)d_index, L, diff);
  k_scan_tile_sums<<<(unsigned)nt, kScanThreads, 0, st>>>((const long long*)d_index, diff, L, sums);
  k_scan_sums<<<1, 1024, 0, st>>>(sums, nt);
  k_scan_tile_apply<<<(unsigned)nt, kScanThreads, 0, st>>>((const long long*)d_index, diff, L, sums,
                                                           window, (long long*)d_arcs, d_cac);
  if (mpgpu_status e = scratch_release(device, kScratchFluss, st); e != MPGPU_OK) return e;
  MPG_CUDA(cudaGetLastError());
  return MPGPU_OK;
}

int64_t mpgpu_extract(const double* d_values, int64_t n, int64_t k, int64_t zone, int32_t largest,
                      double stop_at, int64_t* out_index, double* out_value, int32_t device,
                      void* cuda_stream) {
  if (!d_values || n < 1 || k < 0 || zone < 0) { fail(MPGPU_EPARAM, "bad extract arguments"); return -1; }
  if (cudaSetDevice(device) != cudaSuccess) { fail(MPGPU_ECUDA, "cudaSetDevice"); return -1; }
  cudaStream_t st = (cudaStream_t)cuda_stream;
  const long long nb = (n + 1023) / 1024;
  std::unique_lock<std::mutex> lk;
  char* scratch = nullptr;
  if (scratch_acquire(device, kScratchExtract, sizeof(double) * (n + 4 * (nb + 2)), st, lk,
                      &scratch) != MPGPU_OK)
    return -1;
  double* v = reinterpret_cast<double*>(scratch);
  double* tv = v + n;
  long long* ti = reinterpret_cast<long long*>(tv + 2 * (nb + 2));
  cudaMemcpyAsync(v, d_values, sizeof(double) * n, cudaMemcpyDeviceToDevice, st);
  const int sign = largest ? 1 : -1;
  const double masked = largest ? -INFINITY : INFINITY;  // masked entries are non-finite: skipped
  int64_t found = 0;
  for (; found < k; ++found) {
    double val;
    long long idx;
    if (argext(v, n, sign, st, tv, ti, &val, &idx) != MPGPU_OK || idx < 0) break;
    if (!largest && val >= stop_at) break;   // FLUSS: nothing below the stop value remains
    if (largest && val <= stop_at) break;
    out_index[found] = idx;
    if (out_value) out_value[found] = val;
    const long long span = 2 * zone + 1;
    k_mask_zone<<<(unsigned)((span + 255) / 256), 256, 0, st>>>(v, n, idx, zone, masked);
  }
  scratch_release(device, kScratchExtract, st);
  cudaStreamSynchronize(st);
  return found;
}

mpgpu_status mpgpu_ipc_export(const void* d_ptr, uint8_t* handle, int32_t device) {
  if (!d_ptr || !handle) return fail(MPGPU_EPARAM, "null pointer");
  static_assert(sizeof(cudaIpcMemHandle_t) == MPGPU_IPC_HANDLE_BYTES, "IPC handle size");
  MPG_CUDA(cudaSetDevice(device));
  cudaIpcMemHandle_t h;
  MPG_CUDA(cudaIpcGetMemHandle(&h, const_cast<void*>(d_ptr)));
  memcpy(handle, &h, sizeof(h));
  return MPGPU_OK;
}

mpgpu_status mpgpu_ipc_open(const uint8_t* handle, void** d_ptr, int32_t device) {
  if (!d_ptr || !handle) return fail(MPGPU_EPARAM, "null pointer");
  MPG_CUDA(cudaSetDevice(device));
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  MPG_CUDA(cudaIpcOpenMemHandle(d_ptr, h, cudaIpcMemLazyEnablePeerAccess));
  return MPGPU_OK;
}

mpgpu_status mpgpu_ipc_close(void* d_ptr, int32_t device) {
  if (!d_ptr) return MPGPU_OK;
  MPG_CUDA(cudaSetDevice(device));
  MPG_CUDA(cudaIpcCloseMemHandle(d_ptr));
  return MPGPU_OK;
}

mpgpu_status mpgpu_keys_min_merge(int64_t* d_dst, const int64_t* d_src, int64_t len,
                                  int32_t device, void* cuda_stream) {
  Range nvtx_range("mpgpu:keys_min (K5)");
  MPG_CUDA(cudaSetDevice(device));
  if (len <= 0) return MPGPU_OK;
  k_keys_min<<<(unsigned)((len + 255) / 256), 256, 0, (cudaStream_t)cuda_stream>>>(
      (long long*)d_dst, (const long long*)d_src, len);
  MPG_CUDA(cudaGetLastError());
  return MPGPU_OK;
}

int64_t mpgpu_plan_launch_count(const mpgpu_plan* p) { return p ? p->launches : 0; }

}  // extern "C"

// ---------------------------------------------------------------------------
// Host-buffer join over one or more devices.
// ---------------------------------------------------------------------------
namespace {

struct DevBuf {
  void* ptr = nullptr;
  size_t cap = 0;
  cudaError_t ensure(size_t bytes) {
    if (bytes <= cap) return cudaSuccess;
    if (ptr) cudaFree(ptr);
    ptr = nullptr;
    cap = 0;
    cudaError_t e = cudaMalloc(&ptr, bytes);
    if (e == cudaSuccess) cap = bytes;
    return e;
  }
};

// Per-device cached resources, so repeated joins reuse device memory and
// plans (the library owns them; SURVEY.md §8b conventions).
struct DevCtx {
  std::mutex mu;
  int device = -1;  // CUDA device
  int slot = 0;     // >0: extra context on the same device (virtual shards)
  cudaStream_t stream = nullptr;
  DevBuf xa, xb, out_mp_a, out_pi_a, out_l, out_r, out_mp_b, out_pi_b, keys_in0, keys_in1;
  mpgpu_plan* plan = nullptr;
  long long pa = -1, pb = -1, pm = -1, pz = -1;
  bool pself = false;
  const void *pxa = nullptr, *pxb = nullptr;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
};

std::mutex g_ctx_mu;
std::vector<std::unique_ptr<DevCtx>> g_ctx;

// RED.MIN.S64 from `dev` into memory on `owner` must be a native peer atomic
// (NVLink); over plain PCIe P2P it would not be atomic against the owner's and
// the other shards' updates.
bool peer_atomics_between(int dev, int owner) {
  if (dev == owner) return true;
  int can = 0, atom = 0;
  if (cudaDeviceCanAccessPeer(&can, dev, owner) != cudaSuccess ||
      cudaDeviceGetP2PAttribute(&atom, cudaDevP2PAttrNativeAtomicSupported, dev, owner) !=
          cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return can && atom;
}

// The striped key region of multi-device joins, cached across calls (same
// devices and size -> reused). Calls holding the device locks serialise use.
struct JoinRegion {
  std::mutex mu;
  std::vector<int32_t> devs;
  int64_t bytes = 0;
  mpgpu_stripes* s = nullptr;
  void* base = nullptr;
  std::vector<int32_t> own;
  void* get(const std::vector<int32_t>& d, const mpgpu_plan* p) {
    std::lock_guard<std::mutex> lk(mu);
    const int64_t b = mpgpu_plan_key_region_bytes(p);
    const int64_t g = mpgpu_stripes_granularity(d[0]);
    if (g <= 0) return nullptr;
    std::vector<int32_t> o((size_t)std::max<int64_t>(1, (b + g - 1) / g));
    mpgpu_plan_key_region_owners(p, g, (int32_t)d.size(), o.data(), (int64_t)o.size(), nullptr);
    if (s && d == devs && b == bytes && o == own) return base;
    if (s) mpgpu_stripes_destroy(s);
    s = nullptr;
    base = nullptr;
    s = mpgpu_stripes_create_local(b, (int32_t)d.size(), d.data(), o.data());
    if (!s) return nullptr;
    if (mpgpu_stripes_map(s, &base) != MPGPU_OK) {
      mpgpu_stripes_destroy(s);
      s = nullptr;
      return nullptr;
    }
    devs = d;
    bytes = b;
    own = o;
    return base;
  }
};
JoinRegion g_join_region;

DevCtx* get_ctx(int device, int slot) {
  std::lock_guard<std::mutex> lk(g_ctx_mu);
  for (auto& c : g_ctx)
    if (c->device == device && c->slot == slot) return c.get();
  g_ctx.emplace_back(new DevCtx());
  DevCtx* c = g_ctx.back().get();
  c->device = device;
  c->slot = slot;
  return c;
}

mpgpu_status ensure_ctx(DevCtx* c) {
  MPG_CUDA(cudaSetDevice(c->device));
  if (!c->stream) MPG_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
  if (!c->e0) MPG_CUDA(cudaEventCreate(&c->e0));
  if (!c->e1) MPG_CUDA(cudaEventCreate(&c->e1));
  return MPGPU_OK;
}

mpgpu_status ctx_plan(DevCtx* c, const mpgpu_join_args* a) {
  const bool self = a->b == nullptr;
  const long long nb = self ? 0 : a->n_b;
  if (c->plan && c->pa == a->n_a && c->pb == nb && c->pm == a->window &&
      c->pz == (self ? a->zone : 0) && c->pself == self && c->pxa == c->xa.ptr &&
      c->pxb == (self ? nullptr : c->xb.ptr))
    return MPGPU_OK;
  if (c->plan) {
    mpgpu_plan_destroy(c->plan);
    c->plan = nullptr;
  }
  c->plan = mpgpu_plan_create((const double*)c->xa.ptr, a->n_a,
                              self ? nullptr : (const double*)c->xb.ptr, nb, a->window,
                              self ? a->zone : 0, c->device, c->stream);
  if (!c->plan) return MPGPU_ECUDA;
  c->pa = a->n_a;
  c->pb = nb;
  c->pm = a->window;
  c->pz = self ? a->zone : 0;
  c->pself = self;
  c->pxa = c->xa.ptr;
  c->pxb = self ? nullptr : c->xb.ptr;
  return MPGPU_OK;
}

mpgpu_status join_impl(const mpgpu_join_args* a, double* kernel_ms, double* total_ms,
                       const std::vector<int64_t>* band_ids = nullptr,
                       const std::vector<long long>* diag_ids = nullptr) {
  Range nvtx_range("mpgpu:join (host buffers)");
  const auto t0 = std::chrono::steady_clock::now();
  if (!a || !a->a) return fail(MPGPU_EPARAM, "null arguments");
  const bool self = a->b == nullptr;
  if (a->window < 4) return fail(MPGPU_EPARAM, "window below minimum 4");
  if (a->window > a->n_a || (!self && a->window > a->n_b))
    return fail(MPGPU_EPARAM, "series shorter than the window");
  if (a->zone < 0) return fail(MPGPU_EPARAM, "negative exclusion zone");
  const int ng = diag_ids ? 1 : (a->n_gpus > 0 ? a->n_gpus : 1);  // subsets: one device
  std::vector<int> devs(ng);
  for (int g = 0; g < ng; ++g) devs[g] = a->devices ? a->devices[g] : g;
  const long long La = a->n_a - a->window + 1;
  const long long Lb = self ? La : a->n_b - a->window + 1;

  std::vector<DevCtx*> ctx(ng);
  // distinct contexts even when a device id repeats (virtual shards on one GPU)
  for (int g = 0; g < ng; ++g) {
    int dup = 0;
    for (int h = 0; h < g; ++h) dup += devs[h] == devs[g];
    ctx[g] = get_ctx(devs[g], dup);
  }
  std::vector<std::unique_lock<std::mutex>> locks;
  for (int g = 0; g < ng; ++g) locks.emplace_back(ctx[g]->mu);
  auto real = [](const DevCtx* c) { return c->device; };

  // 1) device buffers + cached plan on every device
  for (int g = 0; g < ng; ++g) {
    DevCtx* c = ctx[g];
    mpgpu_status st = ensure_ctx(c);
    if (st != MPGPU_OK) return st;
    MPG_CUDA(c->xa.ensure(sizeof(double) * a->n_a));
    if (!self) MPG_CUDA(c->xb.ensure(sizeof(double) * a->n_b));
    st = ctx_plan(c, a);
    if (st != MPGPU_OK) return st;
    st = diag_ids ? plan_select_diagonals(c->plan, *diag_ids)
         : band_ids ? mpgpu_plan_select_bands(c->plan, band_ids->data(), (int64_t)band_ids->size())
                    : mpgpu_plan_select_bands(c->plan, nullptr, -1);
    if (st != MPGPU_OK) return st;
  }
  DevCtx* c0 = ctx[0];
  // Fused merge over NVLink: when every shard device can reach device 0's
  // memory, their k_join instances read thresholds from and RED.MIN straight
  // into device 0's keys (peer atomics) -- the min-merge happens inside the
  // compute, no copy or merge kernel. Otherwise: peer copies + k_keys_min.
  bool fused = ng > 1;
  for (int g = 1; g < ng && fused; ++g) {
    DevCtx* c = ctx[g];
    if (real(c) == real(c0)) continue;
    int can = 0;
    cudaDeviceCanAccessPeer(&can, real(c), real(c0));
    if (!can) { fused = false; break; }
    MPG_CUDA(cudaSetDevice(real(c)));
    const cudaError_t pe = cudaDeviceEnablePeerAccess(real(c0), 0);
    if (pe == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
    else if (pe != cudaSuccess) { cudaGetLastError(); fused = false; }
  }
  // The shared keys live in a region striped over the shard devices (2 MB
  // chunks round-robin), so the tile prefetches of every shard spread over all
  // GPUs' links instead of converging on device 0. Device 0's plan owns them
  // (resets and warm-starts); the others only read and RED.MIN.
  if (fused) {
    for (int g = 1; g < ng && fused; ++g)
      fused = peer_atomics_between(real(ctx[g]), real(c0));
  }
  void* region = nullptr;
  if (fused) {
    std::vector<int32_t> ds(devs.begin(), devs.end());
    region = g_join_region.get(ds, c0->plan);
    if (!region) fused = false;  // no VMM: peer copies + k_keys_min below
  }
  for (int g = 0; g < ng; ++g) {
    mpgpu_status st = fused ? mpgpu_plan_attach_key_region(ctx[g]->plan, region,
                                                           mpgpu_plan_key_region_bytes(c0->plan),
                                                           g == 0)
                            : mpgpu_plan_attach_key_region(ctx[g]->plan, nullptr, 0, 0);
    if (st != MPGPU_OK) return st;
  }
  int64_t *root_r = nullptr, *root_c = nullptr;
  mpgpu_plan_keys(c0->plan, &root_r, nullptr, &root_c, nullptr);
  cudaEvent_t keys_ready = nullptr;
  for (int g = 0; g < ng; ++g) {
    DevCtx* c = ctx[g];
    MPG_CUDA(cudaSetDevice(real(c)));
    MPG_CUDA(cudaEventRecord(c->e0, c->stream));
    MPG_CUDA(cudaMemcpyAsync(c->xa.ptr, a->a, sizeof(double) * a->n_a, cudaMemcpyHostToDevice,
                             c->stream));
    if (!self)
      MPG_CUDA(cudaMemcpyAsync(c->xb.ptr, a->b, sizeof(double) * a->n_b, cudaMemcpyHostToDevice,
                               c->stream));
    mpgpu_status st = mpgpu_plan_prepare(c->plan);  // attached plans skip the key init
    if (st != MPGPU_OK) return st;
    if (g == 0 && fused) {
      MPG_CUDA(cudaEventCreateWithFlags(&keys_ready, cudaEventDisableTiming));
      MPG_CUDA(cudaEventRecord(keys_ready, c->stream));
    } else if (fused) {
      MPG_CUDA(cudaStreamWaitEvent(c->stream, keys_ready, 0));  // root keys initialised
    }
    if (!a->progress) {
      st = mpgpu_plan_run(c->plan, g, ng);
      if (st != MPGPU_OK) return st;
    }
  }
  if (a->progress) {
    // run each device's shard in sub-shards and report after each completes
    const int sub = 16;
    for (int q = 0; q < sub; ++q) {
      for (int g = 0; g < ng; ++g) {
        mpgpu_status st = mpgpu_plan_run(ctx[g]->plan, g * sub + q, ng * sub);
        if (st != MPGPU_OK) return st;
      }
      for (int g = 0; g < ng; ++g) {
        MPG_CUDA(cudaSetDevice(real(ctx[g])));
        MPG_CUDA(cudaStreamSynchronize(ctx[g]->stream));
      }
      a->progress((double)(q + 1) / sub, a->progress_ctx);
    }
  }
  // 2) merge: fused -> just order device 0 after every shard; else copy + min
  if (ng > 1) {
    int64_t *k0r = root_r, *k0c = root_c;
    if (!fused) {
      MPG_CUDA(cudaSetDevice(real(c0)));
      MPG_CUDA(c0->keys_in0.ensure(sizeof(long long) * La));
      MPG_CUDA(c0->keys_in1.ensure(sizeof(long long) * Lb));
    }
    for (int g = 1; g < ng; ++g) {
      DevCtx* c = ctx[g];
      cudaEvent_t done;
      MPG_CUDA(cudaSetDevice(real(c)));
      MPG_CUDA(cudaEventCreateWithFlags(&done, cudaEventDisableTiming));
      MPG_CUDA(cudaEventRecord(done, c->stream));
      MPG_CUDA(cudaSetDevice(real(c0)));
      MPG_CUDA(cudaStreamWaitEvent(c0->stream, done, 0));
      cudaEventDestroy(done);
      if (fused) continue;
      int64_t *kr, *kc;
      mpgpu_plan_keys(c->plan, &kr, nullptr, &kc, nullptr);
      if (real(c) != real(c0)) {
        MPG_CUDA(cudaMemcpyPeerAsync(c0->keys_in0.ptr, real(c0), kr, real(c),
                                     sizeof(long long) * La, c0->stream));
        MPG_CUDA(cudaMemcpyPeerAsync(c0->keys_in1.ptr, real(c0), kc, real(c),
                                     sizeof(long long) * Lb, c0->stream));
      } else {
        MPG_CUDA(cudaMemcpyAsync(c0->keys_in0.ptr, kr, sizeof(long long) * La,
                                 cudaMemcpyDeviceToDevice, c0->stream));
        MPG_CUDA(cudaMemcpyAsync(c0->keys_in1.ptr, kc, sizeof(long long) * Lb,
                                 cudaMemcpyDeviceToDevice, c0->stream));
      }
      mpgpu_status st = mpgpu_keys_min_merge(k0r, (const int64_t*)c0->keys_in0.ptr, La, real(c0),
                                             c0->stream);
      if (st != MPGPU_OK) return st;
      st = mpgpu_keys_min_merge(k0c, (const int64_t*)c0->keys_in1.ptr, Lb, real(c0), c0->stream);
      if (st != MPGPU_OK) return st;
    }
  }
  if (keys_ready) cudaEventDestroy(keys_ready);
  // 3) finalize on device 0 and copy back
  MPG_CUDA(cudaSetDevice(real(c0)));
  MPG_CUDA(c0->out_mp_a.ensure(sizeof(double) * La));
  MPG_CUDA(c0->out_pi_a.ensure(sizeof(long long) * La));
  if (self) {
    MPG_CUDA(c0->out_l.ensure(sizeof(long long) * La));
    MPG_CUDA(c0->out_r.ensure(sizeof(long long) * La));
  } else {
    MPG_CUDA(c0->out_mp_b.ensure(sizeof(double) * Lb));
    MPG_CUDA(c0->out_pi_b.ensure(sizeof(long long) * Lb));
  }
  mpgpu_status st = mpgpu_plan_finalize(
      c0->plan, (double*)c0->out_mp_a.ptr, (int64_t*)c0->out_pi_a.ptr,
      self ? (int64_t*)c0->out_l.ptr : nullptr, self ? (int64_t*)c0->out_r.ptr : nullptr,
      (!self && (a->mp_b || a->pi_b)) ? (double*)c0->out_mp_b.ptr : nullptr,
      (!self && (a->mp_b || a->pi_b)) ? (int64_t*)c0->out_pi_b.ptr : nullptr);
  if (st != MPGPU_OK) return st;
  MPG_CUDA(cudaEventRecord(c0->e1, c0->stream));
  auto d2h = [&](void* dst, const DevBuf& src, size_t bytes) -> cudaError_t {
    if (!dst) return cudaSuccess;
    return cudaMemcpyAsync(dst, src.ptr, bytes, cudaMemcpyDeviceToHost, c0->stream);
  };
  MPG_CUDA(d2h(a->mp_a, c0->out_mp_a, sizeof(double) * La));
  MPG_CUDA(d2h(a->pi_a, c0->out_pi_a, sizeof(long long) * La));
  if (self) {
    MPG_CUDA(d2h(a->left_a, c0->out_l, sizeof(long long) * La));
    MPG_CUDA(d2h(a->right_a, c0->out_r, sizeof(long long) * La));
  } else {
    MPG_CUDA(d2h(a->mp_b, c0->out_mp_b, sizeof(double) * Lb));
    MPG_CUDA(d2h(a->pi_b, c0->out_pi_b, sizeof(long long) * Lb));
  }
  MPG_CUDA(cudaStreamSynchronize(c0->stream));
  if (kernel_ms) {
    float ms = 0.f;
    MPG_CUDA(cudaEventElapsedTime(&ms, c0->e0, c0->e1));
    *kernel_ms = ms;
  }
  if (total_ms)
    *total_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0)
                    .count();
  return MPGPU_OK;
}

}  // namespace

extern "C" {

mpgpu_status mpgpu_join(const mpgpu_join_args* args) { return join_impl(args, nullptr, nullptr); }

mpgpu_status mpgpu_join_timed(const mpgpu_join_args* args, double* kernel_ms, double* total_ms) {
  return join_impl(args, kernel_ms, total_ms);
}

mpgpu_status mpgpu_rolling_stats_host(const double* ts, int64_t n, int64_t window, double* means,
                                      double* stds, int32_t device) {
  if (!ts || !means || !stds) return fail(MPGPU_EPARAM, "null argument");
  if (window < 4 || window > n) return fail(MPGPU_EPARAM, "window out of range");
  const long long L = n - window + 1;
  DevCtx* c = get_ctx(device, 0);
  std::lock_guard<std::mutex> lk(c->mu);
  if (mpgpu_status st = ensure_ctx(c); st != MPGPU_OK) return st;
  MPG_CUDA(c->xa.ensure(sizeof(double) * n));
  MPG_CUDA(c->out_mp_a.ensure(sizeof(double) * L));
  MPG_CUDA(c->out_pi_a.ensure(sizeof(double) * L));
  MPG_CUDA(cudaMemcpyAsync(c->xa.ptr, ts, sizeof(double) * n, cudaMemcpyHostToDevice, c->stream));
  if (mpgpu_status st = mpgpu_rolling_stats((const double*)c->xa.ptr, n, window,
                                            (double*)c->out_mp_a.ptr, (double*)c->out_pi_a.ptr,
                                            device, c->stream);
      st != MPGPU_OK)
    return st;
  MPG_CUDA(cudaMemcpyAsync(means, c->out_mp_a.ptr, sizeof(double) * L, cudaMemcpyDeviceToHost,
                           c->stream));
  MPG_CUDA(cudaMemcpyAsync(stds, c->out_pi_a.ptr, sizeof(double) * L, cudaMemcpyDeviceToHost,
                           c->stream));
  MPG_CUDA(cudaStreamSynchronize(c->stream));
  return MPGPU_OK;
}

mpgpu_status mpgpu_mass_host(const double* query, int64_t window, const double* ts, int64_t n,
                             double* out, int32_t device) {
  if (!query || !ts || !out) return fail(MPGPU_EPARAM, "null argument");
  if (window < 4 || window > n) return fail(MPGPU_EPARAM, "window out of range");
  const long long L = n - window + 1;
  DevCtx* c = get_ctx(device, 0);
  std::lock_guard<std::mutex> lk(c->mu);
  if (mpgpu_status st = ensure_ctx(c); st != MPGPU_OK) return st;
  MPG_CUDA(c->xa.ensure(sizeof(double) * n));
  MPG_CUDA(c->xb.ensure(sizeof(double) * window));
  MPG_CUDA(c->out_mp_a.ensure(sizeof(double) * L));
  MPG_CUDA(cudaMemcpyAsync(c->xa.ptr, ts, sizeof(double) * n, cudaMemcpyHostToDevice, c->stream));
  MPG_CUDA(cudaMemcpyAsync(c->xb.ptr, query, sizeof(double) * window, cudaMemcpyHostToDevice,
                           c->stream));
  if (mpgpu_status st = mpgpu_distance_profiles((const double*)c->xa.ptr, n, window,
                                                (const double*)c->xb.ptr, nullptr, 1, -1,
                                                (double*)c->out_mp_a.ptr, device, c->stream);
      st != MPGPU_OK)
    return st;
  MPG_CUDA(cudaMemcpyAsync(out, c->out_mp_a.ptr, sizeof(double) * L, cudaMemcpyDeviceToHost,
                           c->stream));
  MPG_CUDA(cudaStreamSynchronize(c->stream));
  return MPGPU_OK;
}

mpgpu_status mpgpu_scrimp(const mpgpu_join_args* args, int64_t s_size, uint64_t seed,
                          double* coverage) {
  if (!args || !args->a) return fail(MPGPU_EPARAM, "null arguments");
  if (args->b) return fail(MPGPU_EUNSUPPORTED, "SCRIMP supports self-joins only");
  if (args->window < 4 || args->window > args->n_a)
    return fail(MPGPU_EPARAM, "window out of range");
  if (args->zone < 0) return fail(MPGPU_EPARAM, "negative exclusion zone");
  const long long L = args->n_a - args->window + 1;
  const long long nd = L > args->zone + 1 ? L - args->zone - 1 : 0;
  std::vector<int64_t> ids((size_t)std::max<long long>(nd, 1));
  double cov = 1.0;
  const int64_t n = mpgpu_scrimp_diagonals(args->n_a, args->window, args->zone, s_size, seed,
                                           ids.data(), (int64_t)ids.size(), &cov);
  if (coverage) *coverage = cov;
  if (cov >= 1.0) return join_impl(args, nullptr, nullptr);  // full coverage: exact join
  std::vector<long long> diags(ids.begin(), ids.begin() + n);
  return join_impl(args, nullptr, nullptr, nullptr, &diags);
}

mpgpu_status mpgpu_scrimp_banded(const mpgpu_join_args* args, int64_t s_size, uint64_t seed,
                                 double* coverage) {
  if (!args || !args->a) return fail(MPGPU_EPARAM, "null arguments");
  if (args->b) return fail(MPGPU_EUNSUPPORTED, "SCRIMP supports self-joins only");
  if (args->window < 4 || args->window > args->n_a)
    return fail(MPGPU_EPARAM, "window out of range");
  if (args->zone < 0) return fail(MPGPU_EPARAM, "negative exclusion zone");
  const long long L = args->n_a - args->window + 1;
  const long long nb = L > args->zone + 1 ? (L - args->zone - 1 + kW - 1) / kW : 0;
  std::vector<int64_t> ids((size_t)std::max<long long>(nb, 1));
  double cov = 1.0;
  const int64_t n = mpgpu_scrimp_bands(args->n_a, args->window, args->zone, s_size, seed, ids.data(),
                                       (int64_t)ids.size(), &cov);
  if (coverage) *coverage = cov;
  if (cov >= 1.0) return join_impl(args, nullptr, nullptr);  // full coverage: exact join
  ids.resize((size_t)n);
  return join_impl(args, nullptr, nullptr, &ids);
}

}  // extern "C"
