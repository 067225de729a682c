/*
 * mprof_gpu.h — C ABI of the B200 matrix-profile join (libmprof_b200.so).
 *
 * This is the drop-in boundary under the reference's C++ API. Each entry point
 * names the reference interface it replaces (paths under
 * /root/reference/proj/include/mprof/):
 *
 *   mpgpu_join / mpgpu_join_timed  <- mprof::stomp   (profile.hpp:80-83)
 *   mpgpu_scrimp                   <- mprof::scrimp  (profile.hpp:85-89, incl. anytime s_size)
 *   mpgpu_zone_size                <- mprof::zone_size (distance.hpp:19-20)
 *   mpgpu_distance_profiles        <- mprof::mass_distance_profile (distance.hpp:26-33), batched
 *   mpgpu_fluss / mpgpu_extract    <- fluss_arc_count / fluss_cac / fluss_extract / find_discord
 *                                     (discovery.hpp:61-79)
 *   mpgpu_mstomp                   <- mprof::mstomp (profile.hpp:91-94)
 *   mpgpu_simple_join              <- mprof::simple_join (profile.hpp:96-100)
 *   mpgpu_rolling_stats[_host]     <- mprof::rolling_mean_std (rolling.hpp:25-29)
 *                                     + is_flat_std (rolling.hpp:21-23)
 *   mpgpu_mass_host                <- mprof::mass_distance_profile (distance.hpp:26-33)
 *   mpgpu_stripes_* / key regions  <- the worker merge of stomp (profile.hpp:66-68)
 *                                     across GPUs (one key set striped over them)
 *   mpgpu_plan_*                   <- the stomp worker-chunk contract
 *                                     (SPEC.md:267): device-resident inputs,
 *                                     sharded diagonal work and a min-merge of
 *                                     packed (score, index) keys, for callers
 *                                     that own the collective (torch.distributed
 *                                     / NCCL over NVLink).
 *
 * Conventions: plain pointers and sizes only; no exceptions cross the ABI;
 * host buffers are caller-owned; the library owns device scratch, streams and
 * peer mappings. Every call is re-entrant; calls on one device are serialised.
 * Error text for the calling thread: mpgpu_last_error().
 */
#ifndef MPROF_GPU_H
#define MPROF_GPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  MPGPU_OK = 0,
  MPGPU_EPARAM = 2,       /* ParameterError (error.hpp:9-13)                    */
  MPGPU_EUNSUPPORTED = 3, /* UnsupportedError (error.hpp:15-19)                 */
  MPGPU_ECUDA = 10,       /* CUDA runtime failure (no reference equivalent)     */
  MPGPU_ENOMEM = 12       /* device allocation failed                           */
} mpgpu_status;

/* Host-buffer join (the reference call shape). b == NULL selects a self-join;
 * zone is the RESOLVED half-width (mpgpu_zone_size), forced to 0 for AB-joins
 * (SPEC.md:268). Outputs have length n_a - window + 1 (mp_b/pi_b: n_b - window
 * + 1) and may be NULL when not wanted; left/right are self-join only.
 * Excluded / undefined entries are +inf and -1.
 * Samples must be finite: the reference validates them in the TimeSeries ctor
 * (types.cpp:9-17), which the C++ and Python layers above this ABI mirror; the
 * ABI itself does not rescan its inputs (results for non-finite samples are
 * unspecified). The same holds for the device-resident plan API below. */
typedef struct {
  const double *a;
  int64_t n_a;
  const double *b; /* NULL -> self-join */
  int64_t n_b;
  int64_t window;
  int64_t zone;
  int32_t n_gpus;          /* <= 0 -> 1                                       */
  const int32_t *devices;  /* NULL -> 0 .. n_gpus-1                            */
  double *mp_a;            /* values (profile.hpp:30)                          */
  int64_t *pi_a;           /* index (profile.hpp:31)                           */
  int64_t *left_a;         /* left_index, self-join only (profile.hpp:32)      */
  int64_t *right_a;        /* right_index, self-join only (profile.hpp:33)     */
  double *mp_b;            /* AB-join: B against A from the same pass          */
  int64_t *pi_b;
  void (*progress)(double fraction, void *ctx); /* ProgressFn (profile.hpp:23-24) */
  void *progress_ctx;
} mpgpu_join_args;

mpgpu_status mpgpu_join(const mpgpu_join_args *args);

/* As mpgpu_join; also reports the device time of the join kernels
 * (stats + diagonal tiles + finalize, max over devices) and the wall time of
 * the whole call including host<->device copies, in milliseconds. */
mpgpu_status mpgpu_join_timed(const mpgpu_join_args *args, double *kernel_ms, double *total_ms);

/* SCRIMP (profile.hpp:85-89) with the anytime property: a
 * self-join over exactly s_size diagonals taken in SCRIMP's seeded order
 * (Fisher-Yates over the admissible diagonals, splitmix64 from `seed`;
 * mpgpu_scrimp_diagonals lists them), each evaluated in full by k_diag_join.
 * s_size <= 0 or >= all diagonals is the full exact join. *coverage =
 * s_size / all diagonals exactly. Below full coverage left_a / right_a come
 * back as -1 and values are the exact minima over the computed
 * diagonals (element-wise upper bounds of the full profile). AB-joins ->
 * MPGPU_EUNSUPPORTED. */
mpgpu_status mpgpu_scrimp(const mpgpu_join_args *args, int64_t s_size, uint64_t seed,
                          double *coverage);

/* The diagonals mpgpu_scrimp evaluates for (n, window, zone, s_size, seed):
 * writes up to `cap` of them (ascending) and returns how many there are. */
int64_t mpgpu_scrimp_diagonals(int64_t n, int64_t window, int64_t zone, int64_t s_size,
                               uint64_t seed, int64_t *out_diags, int64_t cap, double *coverage);

/* The band-granular fast path of anytime SCRIMP: whole bands of kW = 256
 * consecutive diagonals chosen in a seeded order until at least s_size
 * diagonals are covered, evaluated by the full join kernel (k_join). Same
 * outputs and conventions as mpgpu_scrimp; *coverage = covered / all. */
mpgpu_status mpgpu_scrimp_banded(const mpgpu_join_args *args, int64_t s_size, uint64_t seed,
                                 double *coverage);

/* The band subset mpgpu_scrimp_banded evaluates for (n, window, zone, s_size,
 * seed): writes up to `cap` band ids (ascending; band b = diagonals
 * [zone+1 + 256 b, zone+1 + 256 (b+1))) and returns how many there are. */
int64_t mpgpu_scrimp_bands(int64_t n, int64_t window, int64_t zone, int64_t s_size, uint64_t seed,
                           int64_t *out_bands, int64_t cap, double *coverage);

/* Thread-local description of the last failure on this thread. */
const char *mpgpu_last_error(void);

/* round-half-up(window * fraction); -1 for a negative fraction. */
int64_t mpgpu_zone_size(int64_t window, double fraction);

/* Number of unique cells a join evaluates: (L - zone - 1)(L - zone)/2 for a
 * self-join, L_a * L_b for an AB-join (BASELINE.md §2 unit of work). */
int64_t mpgpu_join_cells(int64_t n_a, int64_t n_b, int64_t window, int64_t zone);

/* Rolling mean / population std of every window of a DEVICE series (flat
 * windows -> std 0 exactly). d_means / d_stds: device, length n - window + 1. */
mpgpu_status mpgpu_rolling_stats(const double *d_ts, int64_t n, int64_t window, double *d_means,
                                 double *d_stds, int32_t device, void *cuda_stream);

/* Host-buffer forms of the two above for the C++ API (rolling_mean_std,
 * rolling.hpp:25-29; mass_distance_profile, distance.hpp:26-33): the library
 * copies the series (and query) in, runs K1 / K6 on `device` and copies the
 * results back. means / stds / out: length n - window + 1. MASS here applies
 * no exclusion zone. */
mpgpu_status mpgpu_rolling_stats_host(const double *ts, int64_t n, int64_t window, double *means,
                                      double *stds, int32_t device);
mpgpu_status mpgpu_mass_host(const double *query, int64_t window, const double *ts, int64_t n,
                             double *out, int32_t device);

/* MASS distance-profile batch (mass_distance_profile, distance.hpp:26-33):
 * n_queries z-normalised distance profiles against every window of the
 * DEVICE series d_ts, written row-major to d_out[n_queries][n - window + 1].
 * Queries are either windows of d_ts (d_query_pos, device int64 positions;
 * |j - pos| <= zone -> +inf, zone < 0: no exclusion) or external device
 * windows (d_queries, n_queries x window, no exclusion). Exact direct dot
 * products, flat-window convention, near-zero hits recomputed directly. */
mpgpu_status mpgpu_distance_profiles(const double *d_ts, int64_t n, int64_t window,
                                     const double *d_queries, const int64_t *d_query_pos,
                                     int64_t n_queries, int64_t zone, double *d_out,
                                     int32_t device, void *cuda_stream);

/* FLUSS on the GPU (fluss_arc_count + fluss_cac, discovery.hpp:68-74): arc
 * counts from a device profile index (d_arcs[L], int64) and, if d_cac is not
 * NULL, the corrected arc curve (d_cac[L], 1 within `window` of either end). */
mpgpu_status mpgpu_fluss(const int64_t *d_index, int64_t L, int64_t window, int64_t *d_arcs,
                         double *d_cac, int32_t device, void *cuda_stream);

/* Repeated arg-extreme extraction with a +-zone mask around every pick, on a
 * DEVICE array: largest != 0 -> discords (find_discord, discovery.hpp:61-63,
 * stops when the max <= stop_at, pass -inf for no stop); largest == 0 ->
 * minima (fluss_extract, discovery.hpp:76-79, stops once the min >= stop_at,
 * 1.0 for FLUSS). Non-finite entries never qualify; ties -> smallest index.
 * Writes up to k host indexes (and values) and returns how many were found,
 * -1 on error. */
int64_t mpgpu_extract(const double *d_values, int64_t n, int64_t k, int64_t zone, int32_t largest,
                      double stop_at, int64_t *out_index, double *out_value, int32_t device,
                      void *cuda_stream);

/* ---- multivariate joins (profile.hpp:91-100) ------------------------------
 * Multivariate series are dim-major host arrays: x[dim * n + t], all
 * dimensions of equal length (MultiTimeSeries, types.hpp:43-53). */

/* SiMPle (mprof::simple_join, profile.hpp:96-100): per cell
 * the non-normalised Euclidean distance summed over all dims,
 * sqrt(sum_d |a_d,j - b_d,i|^2), with rounding residue of an exact match
 * (<= 1e-12 of the summed window energies) snapped to 0
 * (raw_distance_from_terms, distance.hpp:54-57). b == NULL -> self-join with
 * `zone` (left / right filled as stomp); AB -> zone ignored (0). mp_a / pi_a:
 * length n_a - window + 1, indexes into B (AB) or A; mp_b / pi_b (AB only,
 * may be NULL): B against A from the same pass. kernel_ms (may be NULL):
 * device time of the statistics, diagonal kernel and finalize. */
typedef struct {
  const double *a;
  int64_t n_a;
  const double *b;
  int64_t n_b;
  int64_t dims;
  int64_t window;
  int64_t zone;
  int32_t device;
  double *mp_a;
  int64_t *pi_a;
  int64_t *left_a;
  int64_t *right_a;
  double *mp_b;
  int64_t *pi_b;
  double *kernel_ms;
} mpgpu_simple_args;

mpgpu_status mpgpu_simple_join(const mpgpu_simple_args *args);

/* mSTOMP (mprof::mstomp, profile.hpp:91-94): self-join,
 * k-dimensional z-normalised profiles for every k at once. Per cell the
 * per-dimension distances are ranked ascending with the must dims forced to
 * the front (ascending among themselves), excluded dims removed, ties by
 * dimension index; row k holds the minimum over partners of the mean of the
 * k+1 first. Outputs are dims x L row-major (L = n - window + 1): values,
 * index, and dim_order[k][i] = the dimension filling slot k at the chosen
 * partner (MultiMatrixProfile, profile.hpp:48-62); rows k >= the number of
 * admissible dims repeat the last full selection with dim_order -1.
 * EPARAM: overlapping / repeated / out-of-range must or exc dims, or every
 * dim excluded. EUNSUPPORTED: more than 32 admissible dims. */
typedef struct {
  const double *x;
  int64_t n;
  int64_t dims;
  int64_t window;
  int64_t zone;
  const int64_t *must_dims;
  int64_t n_must;
  const int64_t *exc_dims;
  int64_t n_exc;
  int32_t device;
  double *mp;
  int64_t *pi;
  int64_t *dim_order;
  double *kernel_ms;
} mpgpu_mstomp_args;

mpgpu_status mpgpu_mstomp(const mpgpu_mstomp_args *args);

/* ---- device-resident plan (sharded execution) --------------------------- */

typedef struct mpgpu_plan mpgpu_plan;

/* d_a / d_b: device series on `device` (caller-owned, must outlive the plan);
 * d_b == NULL -> self-join. All plan work is issued on cuda_stream (NULL:
 * the legacy default stream). */
mpgpu_plan *mpgpu_plan_create(const double *d_a, int64_t n_a, const double *d_b, int64_t n_b,
                              int64_t window, int64_t zone, int32_t device, void *cuda_stream);
void mpgpu_plan_destroy(mpgpu_plan *plan);

/* Window statistics + flat-window index, reset the packed keys, and warm-start
 * them: a few spread diagonals, then (m >= 32 and >= 1e9 cells) the coarse warm
 * start -- a join on the PAA-downsampled series whose matches seed exact cells
 * of the full join. Equivalent to prepare_shard(0, 1) + prepare_finish. */
mpgpu_status mpgpu_plan_prepare(mpgpu_plan *plan);

/* Two-phase prepare for one process per GPU: every rank calls prepare_shard
 * with its shard (the coarse join is sharded like the join itself), min-reduces
 * the coarse keys from mpgpu_plan_coarse_keys across ranks (e.g. NCCL
 * ReduceOp.MIN; both NULL / 0 when the plan has no coarse phase), then calls
 * prepare_finish. The keys after prepare_finish are bit-identical to a
 * single-rank mpgpu_plan_prepare. */
mpgpu_status mpgpu_plan_prepare_shard(mpgpu_plan *plan, int32_t shard, int32_t n_shards);
mpgpu_status mpgpu_plan_coarse_keys(mpgpu_plan *plan, int64_t **d_row_keys, int64_t *row_len,
                                    int64_t **d_col_keys, int64_t *col_len);
mpgpu_status mpgpu_plan_prepare_finish(mpgpu_plan *plan);

/* Evaluate shard `shard` of `n_shards` (equal-cell contiguous ranges of the
 * diagonal work items) into the plan's keys. Shards of one plan may run in
 * any order; the result after all shards is bit-identical to n_shards = 1. */
mpgpu_status mpgpu_plan_run(mpgpu_plan *plan, int32_t shard, int32_t n_shards);

/* Cells evaluated by one shard (n_shards = 1: the whole join). */
int64_t mpgpu_plan_shard_cells(const mpgpu_plan *plan, int32_t shard, int32_t n_shards);

/* Device pointers to the packed int64 keys, (score bits | index), min-merged:
 * row keys (self: right neighbours; AB: A-profile) and column keys
 * (self: left neighbours; AB: B-profile). An element-wise MIN across shards
 * (ncclMin / torch ReduceOp.MIN on int64) is the whole collective. */
mpgpu_status mpgpu_plan_keys(mpgpu_plan *plan, int64_t **d_row_keys, int64_t *row_len,
                             int64_t **d_col_keys, int64_t *col_len);

/* Decode keys into the MatrixProfile arrays (device pointers, may be NULL). */
mpgpu_status mpgpu_plan_finalize(mpgpu_plan *plan, double *d_mp_a, int64_t *d_pi_a,
                                 int64_t *d_left_a, int64_t *d_right_a, double *d_mp_b,
                                 int64_t *d_pi_b);

/* Decode rows [L*shard/n_shards, L*(shard+1)/n_shards) of every output (A
 * side, and the B side of an AB-join, each by its own length) into the
 * full-length output arrays; the rest of the arrays is untouched. With keys
 * shared across ranks (mpgpu_plan_attach_key_region) and output arrays that
 * every rank can write (e.g. a region owned by the root), each rank decodes
 * its share straight into the root's profile. Anytime plans: n_shards == 1. */
mpgpu_status mpgpu_plan_finalize_shard(mpgpu_plan *plan, int32_t shard, int32_t n_shards,
                                       double *d_mp_a, int64_t *d_pi_a, int64_t *d_left_a,
                                       int64_t *d_right_a, double *d_mp_b, int64_t *d_pi_b);

/* Anytime mode on a self-join plan: evaluate only the given diagonal bands
 * (ids as in mpgpu_scrimp_bands); prepare() then skips the warm start and
 * finalize() searches flat-window candidates band by band. n < 0 or
 * band_ids == NULL returns the plan to the full join. */
mpgpu_status mpgpu_plan_select_bands(mpgpu_plan *plan, const int64_t *band_ids, int64_t n);

/* Point this plan at another plan's keys (mpgpu_plan_keys of the owner),
 * possibly on a peer device reachable over NVLink: k_join then reads its
 * filter thresholds from them and RED.MINs its candidates straight into them,
 * so the cross-device min-merge happens inside the compute (no merge step).
 * prepare() of an attached plan skips the key initialisation (the owner's
 * prepare must complete first). NULL, NULL detaches. */
mpgpu_status mpgpu_plan_attach_keys(mpgpu_plan *plan, int64_t *d_row_keys, int64_t *d_col_keys);

/* CUDA IPC for keys shared across processes (one process per GPU under
 * torchrun): the owner exports its key allocations (mpgpu_plan_keys) as
 * 64-byte handles, every other rank opens them (a peer-memory mapping over
 * NVLink) and attaches its plan to them, so every rank's k_join filters
 * against and RED.MINs into the same keys while it computes. An attached
 * plan's prepare_shard(shard, n > 1) still runs its shard of the coarse
 * warm-start join; the owner alone resets and seeds the shared keys. */
#define MPGPU_IPC_HANDLE_BYTES 64

/* Warm start of a shared-key join, sharded over the ranks, with no barrier
 * before the join: the owner resets its keys once per join beforehand
 * (mpgpu_plan_reset_keys, e.g. right after finalizing the previous one).
 * prepare_shared: stats and this shard's coarse join (no key writes).
 * The caller MIN-all-reduces mpgpu_plan_coarse_keys across ranks (which also
 * orders every rank after the owner's reset), then seed_shared: this shard's
 * spread diagonals and coarse-match segments, RED.MIN'd into the keys. */
mpgpu_status mpgpu_plan_prepare_shared(mpgpu_plan *plan, int32_t shard, int32_t n_shards);
mpgpu_status mpgpu_plan_seed_shared(mpgpu_plan *plan, int32_t shard, int32_t n_shards);
mpgpu_status mpgpu_plan_reset_keys(mpgpu_plan *plan);

/* Coarse warm-start keys shared the same way (they would otherwise see only
 * each rank's own coarse shard): the owner takes the nested coarse plan's key
 * arrays (NULL when the plan has no coarse phase) and exports them, the other
 * ranks attach. prepare_shared then stops before the coarse join, and every
 * rank runs its coarse shard with coarse_run once the owner's prepare_shared
 * is complete (a barrier), then seed_shared once every coarse_run is. */
mpgpu_status mpgpu_plan_coarse_key_ptrs(mpgpu_plan *plan, int64_t **d_row_keys, int64_t **d_col_keys);
mpgpu_status mpgpu_plan_attach_coarse_keys(mpgpu_plan *plan, int64_t *d_row_keys, int64_t *d_col_keys);
mpgpu_status mpgpu_plan_coarse_run(mpgpu_plan *plan, int32_t shard, int32_t n_shards);
mpgpu_status mpgpu_ipc_export(const void *d_ptr, uint8_t *handle, int32_t device);
mpgpu_status mpgpu_ipc_open(const uint8_t *handle, void **d_ptr, int32_t device);
mpgpu_status mpgpu_ipc_close(void *d_ptr, int32_t device);

/* ---- striped key region (multi-GPU shared keys without a hot owner) --------
 * Replaces the single-owner sharing above for the join's keys: one contiguous
 * virtual range whose physical chunks (the VMM granularity, 2 MB) live in the
 * HBM of different GPUs (chunk c on rank owners[c], by default a table that
 * balances the modelled key reads per GPU). Every rank maps every
 * chunk, so kernels index one flat array while the key traffic of all ranks
 * spreads over every GPU's NVLink ports. Same protocol as the
 * reference's worker merge (profile.hpp:66-68): element-wise min of packed
 * keys, here done by RED.MIN.S64 during the join.
 *
 * One process per GPU: stripes_create (this rank's chunks), export_fd of each
 * owned chunk (a POSIX fd; pass it to the other ranks, e.g. SCM_RIGHTS over a
 * Unix socket), import_fd of every other chunk, then map. One process, several
 * GPUs: stripes_create_local (maps as well). The kernels' 64-bit RED.MIN into
 * a peer's chunk needs native peer atomics (NVLink): check mpgpu_peer_atomics
 * for every (rank device, peer device) pair before using a region. */
typedef struct mpgpu_stripes mpgpu_stripes;
/* chunk size (the VMM granularity on `device`), -1 without VMM support */
int64_t mpgpu_stripes_granularity(int32_t device);
/* owners[c]: rank (create_local: index into devices) of chunk c; NULL -> c % n */
mpgpu_stripes *mpgpu_stripes_create(int64_t bytes, int32_t n_ranks, int32_t rank, int32_t device,
                                    const int32_t *owners);
mpgpu_stripes *mpgpu_stripes_create_local(int64_t bytes, int32_t n_devices, const int32_t *devices,
                                          const int32_t *owners);
int64_t mpgpu_stripes_num_chunks(const mpgpu_stripes *s);
int64_t mpgpu_stripes_chunk_bytes(const mpgpu_stripes *s);
int32_t mpgpu_stripes_owner(const mpgpu_stripes *s, int64_t chunk);
/* fd of an owned chunk (caller closes it after passing it on), -1 on error */
int32_t mpgpu_stripes_export_fd(mpgpu_stripes *s, int64_t chunk);
/* import a peer's chunk from a received fd (the caller closes the fd after) */
mpgpu_status mpgpu_stripes_import_fd(mpgpu_stripes *s, int64_t chunk, int32_t fd);
mpgpu_status mpgpu_stripes_map(mpgpu_stripes *s, void **d_base);
void mpgpu_stripes_destroy(mpgpu_stripes *s);
/* PCI bus id of a device (buf >= 16 bytes); 0 on success */
int32_t mpgpu_device_pci_bus_id(int32_t device, char *buf, int32_t len);
/* 1: native peer atomics from `device` to the GPU with that bus id (or the
 * same GPU); 0: not supported; -1: that GPU is not visible to this process. */
int32_t mpgpu_peer_atomics(int32_t device, const char *peer_pci_bus_id);

/* Bytes of a shared key region for this plan (fine row + column keys, plus
 * the coarse warm-start keys when the plan has a coarse phase). */
int64_t mpgpu_plan_key_region_bytes(const mpgpu_plan *plan);
/* Chunk owners balancing the modelled key reads per GPU (every 32-row tile of
 * a work item reads 32 row and 32 column keys), largest chunk first to the
 * least-loaded rank. Returns the chunk count (owners untouched when NULL or
 * cap is smaller); *max_share = the busiest rank's share of all key reads. */
int64_t mpgpu_plan_key_region_owners(const mpgpu_plan *plan, int64_t chunk_bytes, int32_t n_ranks,
                                     int32_t *owners, int64_t cap, double *max_share);
/* Place this plan's keys (and coarse keys) in a region of at least
 * mpgpu_plan_key_region_bytes: every rank's plan of one join attaches the same
 * region; exactly one (owner != 0) resets and warm-starts the keys
 * (mpgpu_plan_reset_keys, prepare), the others read and RED.MIN only. With
 * coarse keys in the region, prepare_shared stops before the coarse join and
 * coarse_run runs it (as with mpgpu_plan_attach_coarse_keys).
 * d_base == NULL detaches (back to the plan's own keys). */
mpgpu_status mpgpu_plan_attach_key_region(mpgpu_plan *plan, void *d_base, int64_t bytes,
                                          int32_t owner);

/* Number of 256-diagonal bands of a self-join plan (0 for AB plans). */
int64_t mpgpu_plan_num_bands(const mpgpu_plan *plan);

/* Element-wise min of `src` into `dst` (device, same device), for merging
 * shard keys without NCCL. */
mpgpu_status mpgpu_keys_min_merge(int64_t *d_dst, const int64_t *d_src, int64_t len,
                                  int32_t device, void *cuda_stream);

/* Kernel launches issued by the last plan_prepare + plan_run + plan_finalize
 * sequence on this plan (for bench accounting). */
int64_t mpgpu_plan_launch_count(const mpgpu_plan *plan);

/* Library build string (arch, tile shape). */
const char *mpgpu_build_info(void);

#ifdef __cplusplus
}
#endif

#endif
