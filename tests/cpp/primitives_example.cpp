// A reference-API caller of the path's primitives, unchanged except for
// linking libmprof_b200.so: rolling_mean_std + is_flat_std (rolling.hpp:21-29),
// znorm_dist_from_qt, zone_size, apply_exclusion_zone[_inplace] and
// mass_distance_profile (distance.hpp:12-33), merge_min (profile.hpp:66-68).
// Compiles against either the reference's headers or include/mprof.
//   primitives_example <in.f64> <window> <query_pos> <zone> <out_prefix>
// writes out.means / out.stds (rolling stats), out.mass (the MASS profile of
// the window at query_pos), out.excl (it after apply_exclusion_zone),
// out.merged_v / out.merged_i (a fresh profile merge_min'd with it and then
// with a profile shifted by +0.5 everywhere) and out.qt (znorm_dist_from_qt on
// the direct dot products of the query with every window). Prints one JSON
// line with scalar results.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <exception>
#include <limits>
#include <span>
#include <string>
#include <vector>

#include "mprof/distance.hpp"
#include "mprof/profile.hpp"
#include "mprof/rolling.hpp"

static std::vector<double> read_f64(const char *path) {
  std::vector<double> v;
  FILE *f = std::fopen(path, "rb");
  if (!f) return v;
  double x;
  while (std::fread(&x, sizeof(double), 1, f) == 1) v.push_back(x);
  std::fclose(f);
  return v;
}

template <typename T>
static void write_vec(const std::string &path, const std::vector<T> &v) {
  FILE *f = std::fopen(path.c_str(), "wb");
  if (!v.empty()) std::fwrite(v.data(), sizeof(T), v.size(), f);
  std::fclose(f);
}

int main(int argc, char **argv) {
  if (argc < 6) return 64;
  try {
    const mprof::TimeSeries ts(read_f64(argv[1]));
    const mprof::Index w = std::atoll(argv[2]), q = std::atoll(argv[3]), zone = std::atoll(argv[4]);
    const std::string out = argv[5];
    const mprof::RollingStats st = mprof::rolling_mean_std(ts.span(), w);
    write_vec(out + ".means", st.means);
    write_vec(out + ".stds", st.stds);
    long long flats = 0;
    for (mprof::Index i = 0; i < st.size(); ++i)
      flats += mprof::is_flat_std(st.stds[(std::size_t)i], st.means[(std::size_t)i]) ? 1 : 0;

    const auto query = ts.window(q, w);
    const mprof::DistanceProfile dp = mprof::mass_distance_profile(
        query, ts.span(), st, st.means[(std::size_t)q], st.stds[(std::size_t)q], q);
    write_vec(out + ".mass", dp.distances);
    const mprof::DistanceProfile ex = mprof::apply_exclusion_zone(dp, q, zone);
    write_vec(out + ".excl", ex.distances);
    std::vector<double> inplace = dp.distances;
    mprof::apply_exclusion_zone_inplace(inplace, q, zone);
    bool same = inplace == ex.distances;

    // direct QT of the query with every window, then znorm_dist_from_qt
    std::vector<double> qt_d(dp.distances.size()), qt_raw(dp.distances.size());
    for (std::size_t i = 0; i < qt_d.size(); ++i) {
      double s = 0.0;
      for (mprof::Index k = 0; k < w; ++k) s += query[(std::size_t)k] * ts[(mprof::Index)i + k];
      qt_raw[i] = s;
      qt_d[i] = mprof::znorm_dist_from_qt(s, w, st.means[(std::size_t)q], st.stds[(std::size_t)q],
                                          st.means[i], st.stds[i]);
    }
    write_vec(out + ".qt", qt_d);
    write_vec(out + ".qtraw", qt_raw);

    mprof::MatrixProfile acc;
    acc.values.assign(dp.distances.size(), mprof::kInf);
    acc.index.assign(dp.distances.size(), mprof::kNone);
    mprof::merge_min(acc, ex, q);
    mprof::DistanceProfile shifted = dp;
    for (double &d : shifted.distances) d += 0.5;
    mprof::merge_min(acc, shifted, q + 1);  // strictly worse except where ex is +inf
    write_vec(out + ".merged_v", acc.values);
    write_vec(out + ".merged_i", acc.index);

    bool threw = false;
    try {
      mprof::DistanceProfile short_dp;
      short_dp.distances.assign(3, 0.0);
      mprof::merge_min(acc, short_dp, 0);
    } catch (const std::logic_error &) {
      threw = true;
    }
    bool param_err = false;
    try {
      (void)mprof::rolling_mean_std(ts.span(), ts.size() + 1);
    } catch (const mprof::ParameterError &) {
      param_err = true;
    }
    std::printf("{\"size\": %lld, \"window\": %lld, \"flats\": %lld, \"zone_50_half\": %lld, "
                "\"inplace_same\": %s, \"merge_len_error\": %s, \"window_error\": %s, "
                "\"query_index\": %lld}\n",
                (long long)st.size(), (long long)st.window, flats,
                (long long)mprof::zone_size(50, 0.5), same ? "true" : "false",
                threw ? "true" : "false", param_err ? "true" : "false",
                (long long)dp.query_index);
  } catch (const std::exception &e) {
    std::printf("{\"error\": \"%s\"}\n", e.what());
    return 2;
  }
  return 0;
}
