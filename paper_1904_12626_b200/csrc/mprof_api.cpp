// C++ shim: the reference's mprof::stomp / scrimp / mstomp / simple_join
// signatures (profile.hpp:80-100) and the primitives the path uses
// (rolling.hpp:21-29, distance.hpp:12-33, profile.hpp:66-68) on top of the C
// ABI (include/mprof_gpu.h). Status codes come back as the reference's
// exception types (error.hpp:9-19).
#include <algorithm>
#include <cmath>
#include <stdexcept>
#include <string>
#include <utility>

#include "mprof/distance.hpp"
#include "mprof/profile.hpp"
#include "mprof/rolling.hpp"
#include "mprof_gpu.h"

namespace mprof {

TimeSeries::TimeSeries(std::vector<double> values) : data_(std::move(values)) {
  if (size() < kMinWindow)
    throw ParameterError("time series too short: length " + std::to_string(size()) +
                         " < minimum " + std::to_string(kMinWindow));
  for (std::size_t i = 0; i < data_.size(); ++i)
    if (!std::isfinite(data_[i]))
      throw ParameterError("time series sample " + std::to_string(i) + " is not finite");
}

MultiTimeSeries::MultiTimeSeries(std::vector<TimeSeries> dims) : dims_(std::move(dims)) {
  if (dims_.empty()) throw ParameterError("multivariate series needs at least one dimension");
  const Index n = dims_.front().size();
  for (std::size_t k = 1; k < dims_.size(); ++k)
    if (dims_[k].size() != n)
      throw ParameterError("dimension " + std::to_string(k) + " has length " +
                           std::to_string(dims_[k].size()) + ", expected " + std::to_string(n));
}

const char *mode_name(Mode mode) {
  switch (mode) {
    case Mode::brute: return "brute";
    case Mode::stamp: return "stamp";
    case Mode::stomp: return "stomp";
    case Mode::scrimp: return "scrimp";
    case Mode::mstomp: return "mstomp";
    case Mode::simple: return "simple";
  }
  return "?";
}

std::optional<Mode> mode_from_name(const std::string &name) {
  for (Mode m : {Mode::brute, Mode::stamp, Mode::stomp, Mode::scrimp, Mode::mstomp, Mode::simple})
    if (name == mode_name(m)) return m;
  return std::nullopt;
}

Index zone_size(Index window, double fraction) {
  if (!(fraction >= 0.0)) throw ParameterError("exclusion-zone fraction must be >= 0");
  return static_cast<Index>(mpgpu_zone_size(window, fraction));
}

namespace {

void check_window(Index window, Index n, const char *which) {
  if (window < kMinWindow)
    throw ParameterError("window " + std::to_string(window) + " < minimum " +
                         std::to_string(kMinWindow));
  if (window > n)
    throw ParameterError(std::string("window ") + std::to_string(window) + " exceeds " + which +
                         " length " + std::to_string(n));
}

[[noreturn]] void raise(mpgpu_status st) {
  const std::string msg = mpgpu_last_error();
  if (st == MPGPU_EUNSUPPORTED) throw UnsupportedError(msg);
  if (st == MPGPU_EPARAM) throw ParameterError(msg);
  throw std::runtime_error("mprof_b200: " + msg);
}

void progress_tramp(double f, void *ctx) { (*static_cast<const ProgressFn *>(ctx))(f); }

MatrixProfile run_join(const TimeSeries &a, const TimeSeries *b, Index window, Index zone,
                       const ProgressFn &progress, bool want_b_side) {
  const Index La = a.size() - window + 1;
  MatrixProfile mp;
  mp.window = window;
  mp.exclusion_zone = b ? 0 : zone;
  mp.join_kind = b ? JoinKind::ab : JoinKind::self;
  mp.data_len = a.size();
  mp.data_len_b = b ? b->size() : 0;
  mpgpu_join_args args{};
  args.a = a.values().data();
  args.n_a = a.size();
  args.b = b ? b->values().data() : nullptr;
  args.n_b = b ? b->size() : 0;
  args.window = window;
  args.zone = mp.exclusion_zone;
  args.n_gpus = 1;
  if (want_b_side) {
    const Index Lb = b->size() - window + 1;
    mp.values.resize(Lb);
    mp.index.resize(Lb);
    args.mp_b = mp.values.data();
    args.pi_b = mp.index.data();
  } else {
    mp.values.resize(La);
    mp.index.resize(La);
    args.mp_a = mp.values.data();
    args.pi_a = mp.index.data();
    if (!b) {
      mp.left_index.resize(La);
      mp.right_index.resize(La);
      args.left_a = mp.left_index.data();
      args.right_a = mp.right_index.data();
    }
  }
  if (progress) {
    args.progress = progress_tramp;
    args.progress_ctx = const_cast<ProgressFn *>(&progress);
  }
  const mpgpu_status st = mpgpu_join(&args);
  if (st != MPGPU_OK) raise(st);
  return mp;
}

}  // namespace

MatrixProfile stomp(const TimeSeries &ts_a, const TimeSeries *ts_b, Index window,
                    double ez_fraction, int n_workers, const ProgressFn &progress) {
  if (n_workers < 1) throw ParameterError("n_workers must be >= 1");
  check_window(window, ts_a.size(), "series");
  if (ts_b) check_window(window, ts_b->size(), "series B");
  const Index zone = zone_size(window, ez_fraction);
  MatrixProfile mp = run_join(ts_a, ts_b, window, zone, progress, false);
  mp.mode = Mode::stomp;
  return mp;
}

MatrixProfile scrimp(const TimeSeries &ts_a, Index window, double ez_fraction, Index s_size,
                     std::uint64_t seed, const ProgressFn &progress) {
  if (s_size < 1) throw ParameterError("s_size must be >= 1");
  check_window(window, ts_a.size(), "series");
  const Index zone = zone_size(window, ez_fraction);
  const Index L = ts_a.size() - window + 1;
  const Index n_diag = L > zone + 1 ? L - zone - 1 : 0;
  if (s_size >= n_diag) {  // full run: the exact join
    MatrixProfile mp = run_join(ts_a, nullptr, window, zone, progress, false);
    mp.mode = Mode::scrimp;
    mp.seed = seed;
    return mp;
  }
  // anytime run over a seeded subset of diagonal bands
  MatrixProfile mp;
  mp.window = window;
  mp.exclusion_zone = zone;
  mp.mode = Mode::scrimp;
  mp.join_kind = JoinKind::self;
  mp.seed = seed;
  mp.data_len = ts_a.size();
  mp.values.resize(L);
  mp.index.resize(L);
  std::vector<Index> left(L), right(L);
  mpgpu_join_args args{};
  args.a = ts_a.values().data();
  args.n_a = ts_a.size();
  args.window = window;
  args.zone = zone;
  args.n_gpus = 1;
  args.mp_a = mp.values.data();
  args.pi_a = mp.index.data();
  args.left_a = left.data();
  args.right_a = right.data();
  double coverage = 0.0;
  const mpgpu_status st = mpgpu_scrimp(&args, s_size, seed, &coverage);
  if (st != MPGPU_OK) raise(st);
  mp.coverage = coverage;
  if (coverage >= 1.0) {  // left/right only at full coverage
    mp.left_index.swap(left);
    mp.right_index.swap(right);
  }
  if (progress) progress(1.0);
  return mp;
}

namespace {

std::vector<double> dim_major(const MultiTimeSeries &m) {
  const std::size_t n = static_cast<std::size_t>(m.size());
  std::vector<double> x(n * static_cast<std::size_t>(m.dims()));
  for (Index d = 0; d < m.dims(); ++d)
    std::copy(m.dim(d).values().begin(), m.dim(d).values().end(), x.begin() + d * n);
  return x;
}

}  // namespace

MultiMatrixProfile mstomp(const MultiTimeSeries &mts, Index window, double ez_fraction,
                          const std::vector<Index> &must_dims, const std::vector<Index> &exc_dims,
                          int n_workers, const ProgressFn &progress) {
  if (n_workers < 1) throw ParameterError("n_workers must be >= 1");
  check_window(window, mts.size(), "series");
  const Index zone = zone_size(window, ez_fraction);
  const Index d = mts.dims(), L = mts.size() - window + 1;
  const std::vector<double> x = dim_major(mts);
  std::vector<double> v(static_cast<std::size_t>(d * L));
  std::vector<Index> pi(v.size()), dorder(v.size());
  mpgpu_mstomp_args args{};
  args.x = x.data();
  args.n = mts.size();
  args.dims = d;
  args.window = window;
  args.zone = zone;
  args.must_dims = must_dims.data();
  args.n_must = static_cast<int64_t>(must_dims.size());
  args.exc_dims = exc_dims.data();
  args.n_exc = static_cast<int64_t>(exc_dims.size());
  args.mp = v.data();
  args.pi = pi.data();
  args.dim_order = dorder.data();
  const mpgpu_status st = mpgpu_mstomp(&args);
  if (st != MPGPU_OK) raise(st);
  MultiMatrixProfile r;
  r.window = window;
  r.exclusion_zone = zone;
  r.must_dims = must_dims;
  r.exc_dims = exc_dims;
  r.data_len = mts.size();
  r.data_dims = d;
  for (Index k = 0; k < d; ++k) {
    r.values.emplace_back(v.begin() + k * L, v.begin() + (k + 1) * L);
    r.index.emplace_back(pi.begin() + k * L, pi.begin() + (k + 1) * L);
    r.dim_order.emplace_back(dorder.begin() + k * L, dorder.begin() + (k + 1) * L);
  }
  if (progress) progress(1.0);
  return r;
}

MatrixProfile simple_join(const MultiTimeSeries &mts_a, const MultiTimeSeries *mts_b,
                          Index window, double ez_fraction, const ProgressFn &progress) {
  if (mts_b && mts_b->dims() != mts_a.dims())
    throw ParameterError("dimension mismatch: " + std::to_string(mts_a.dims()) + " vs " +
                         std::to_string(mts_b->dims()));
  check_window(window, mts_a.size(), "series");
  if (mts_b) check_window(window, mts_b->size(), "series B");
  const Index zone = mts_b ? 0 : zone_size(window, ez_fraction);
  const Index La = mts_a.size() - window + 1;
  const std::vector<double> xa = dim_major(mts_a);
  std::vector<double> xb;
  if (mts_b) xb = dim_major(*mts_b);
  MatrixProfile mp;
  mp.window = window;
  mp.exclusion_zone = zone;
  mp.mode = Mode::simple;
  mp.join_kind = mts_b ? JoinKind::ab : JoinKind::self;
  mp.data_len = mts_a.size();
  mp.data_len_b = mts_b ? mts_b->size() : 0;
  mp.data_dims = mts_a.dims();
  mp.values.resize(La);
  mp.index.resize(La);
  mpgpu_simple_args args{};
  args.a = xa.data();
  args.n_a = mts_a.size();
  args.b = mts_b ? xb.data() : nullptr;
  args.n_b = mts_b ? mts_b->size() : 0;
  args.dims = mts_a.dims();
  args.window = window;
  args.zone = zone;
  args.mp_a = mp.values.data();
  args.pi_a = mp.index.data();
  if (!mts_b) {
    mp.left_index.resize(La);
    mp.right_index.resize(La);
    args.left_a = mp.left_index.data();
    args.right_a = mp.right_index.data();
  }
  const mpgpu_status st = mpgpu_simple_join(&args);
  if (st != MPGPU_OK) raise(st);
  if (progress) progress(1.0);
  return mp;
}

MatrixProfile stomp_ab_reverse(const TimeSeries &ts_a, const TimeSeries &ts_b, Index window) {
  check_window(window, ts_a.size(), "series");
  check_window(window, ts_b.size(), "series B");
  MatrixProfile mp = run_join(ts_a, &ts_b, window, 0, {}, true);
  mp.mode = Mode::stomp;
  mp.data_len = ts_b.size();
  mp.data_len_b = ts_a.size();
  return mp;
}

// ---- primitives on the path (rolling.hpp, distance.hpp, profile.hpp) --------

bool is_flat_std(double sd, double mean) {
  const double scale = std::fabs(mean) > 1.0 ? std::fabs(mean) : 1.0;
  return sd <= 1e-10 * scale;  // the rule K1 applies on the GPU (mpgpu_kernels.cuh)
}

RollingStats rolling_mean_std(std::span<const double> ts, Index window) {
  const Index n = static_cast<Index>(ts.size());
  check_window(window, n, "series");
  RollingStats r;
  r.window = window;
  r.means.resize(static_cast<std::size_t>(n - window + 1));
  r.stds.resize(r.means.size());
  const mpgpu_status st =
      mpgpu_rolling_stats_host(ts.data(), n, window, r.means.data(), r.stds.data(), 0);
  if (st != MPGPU_OK) raise(st);
  return r;
}

double znorm_dist_from_qt(double qt, Index w, double mu_a, double sd_a, double mu_b,
                          double sd_b) {
  const bool fa = sd_a == 0.0, fb = sd_b == 0.0;  // flat windows carry sd == 0 exactly
  if (fa && fb) return 0.0;
  if (fa || fb) return std::sqrt(static_cast<double>(w));
  const double wd = static_cast<double>(w);
  const double d2 = 2.0 * wd * (1.0 - (qt - wd * mu_a * mu_b) / (wd * sd_a * sd_b));
  return std::sqrt(std::clamp(d2, 0.0, 4.0 * wd));
}

void apply_exclusion_zone_inplace(std::span<double> distances, Index center, Index zone) {
  const Index len = static_cast<Index>(distances.size());
  if (center < 0 || center >= len)
    throw ParameterError("exclusion-zone center " + std::to_string(center) +
                         " outside the profile (length " + std::to_string(len) + ")");
  if (zone < 0) throw ParameterError("negative exclusion zone");
  const Index lo = std::max<Index>(0, center - zone);
  const Index hi = zone >= len ? len - 1 : std::min<Index>(len - 1, center + zone);
  for (Index i = lo; i <= hi; ++i) distances[static_cast<std::size_t>(i)] = kInf;
}

DistanceProfile apply_exclusion_zone(DistanceProfile dp, Index center, Index zone) {
  apply_exclusion_zone_inplace(dp.distances, center, zone);
  return dp;
}

void merge_min(MatrixProfile &acc, const DistanceProfile &dp, Index source_index) {
  if (acc.values.size() != dp.distances.size() || acc.index.size() != acc.values.size())
    throw std::logic_error("merge_min: profile lengths differ");
  for (std::size_t i = 0; i < dp.distances.size(); ++i) {
    if (dp.distances[i] < acc.values[i]) {  // strict improvement; ties keep the incumbent
      acc.values[i] = dp.distances[i];
      acc.index[i] = source_index;
    }
  }
}

DistanceProfile mass_distance_profile(std::span<const double> query, std::span<const double> ts,
                                      const RollingStats &stats, double query_mean,
                                      double query_std, Index query_index) {
  (void)query_mean;
  (void)query_std;
  const Index w = static_cast<Index>(query.size()), n = static_cast<Index>(ts.size());
  check_window(w, n, "series");
  if (stats.window != w || stats.size() != n - w + 1)
    throw ParameterError("rolling stats do not match the query length / series");
  DistanceProfile dp;
  dp.query_index = query_index;
  dp.distances.resize(static_cast<std::size_t>(n - w + 1));
  const mpgpu_status st = mpgpu_mass_host(query.data(), w, ts.data(), n, dp.distances.data(), 0);
  if (st != MPGPU_OK) raise(st);
  return dp;
}

}  // namespace mprof
