// A reference-API caller, unchanged except for linking libmprof_b200.so:
// reads a raw fp64 series, runs mprof::stomp (profile.hpp:80-83) or
// mprof::scrimp (profile.hpp:85-89), writes values/index/left/right as raw
// arrays. Used by tests/test_dropin_cpp.py to show the drop-in boundary.
//   dropin_example <in.f64> <window> <ez> <out_prefix>
//                  [stomp|scrimp|anytime <s_size> <seed>|ab <b.f64>
//                   |simple <dims> [b.f64]|mstomp <dims> <must csv|-> <exc csv|->]
// Multivariate inputs are dim-major (dims x n). mstomp writes the dims x L
// values / index / dim_order (out.mp, out.pi, out.dim) row after row.
#include <cstdio>
#include <cstdlib>
#include <exception>
#include <string>
#include <vector>

#include "mprof/profile.hpp"

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

static mprof::MultiTimeSeries read_mts(const char *path, long long dims) {
  const std::vector<double> x = read_f64(path);
  const std::size_t n = dims > 0 ? x.size() / (std::size_t)dims : 0;
  std::vector<mprof::TimeSeries> rows;
  for (long long d = 0; d < dims; ++d)
    rows.emplace_back(std::vector<double>(x.begin() + d * n, x.begin() + (d + 1) * n));
  return mprof::MultiTimeSeries(std::move(rows));
}

static std::vector<mprof::Index> csv(const char *s) {
  std::vector<mprof::Index> v;
  if (!s || std::string(s) == "-") return v;
  std::string t(s);
  std::size_t p = 0;
  while (p <= t.size()) {
    const std::size_t q = t.find(',', p);
    v.push_back(std::atoll(t.substr(p, q - p).c_str()));
    if (q == std::string::npos) break;
    p = q + 1;
  }
  return v;
}

int main(int argc, char **argv) {
  if (argc < 5) {
    std::fprintf(stderr, "usage: %s in.f64 window ez out_prefix [stomp|scrimp|anytime s seed|ab b.f64]\n",
                 argv[0]);
    return 1;
  }
  const std::string mode = argc > 5 ? argv[5] : "stomp";
  try {
    if (mode == "mstomp") {
      const mprof::MultiTimeSeries x = read_mts(argv[1], std::atoll(argv[6]));
      const mprof::MultiMatrixProfile r =
          mprof::mstomp(x, std::atoll(argv[2]), std::atof(argv[3]), csv(argv[7]), csv(argv[8]));
      std::vector<double> v;
      std::vector<mprof::Index> pi, dm;
      for (std::size_t k = 0; k < r.values.size(); ++k) {
        v.insert(v.end(), r.values[k].begin(), r.values[k].end());
        pi.insert(pi.end(), r.index[k].begin(), r.index[k].end());
        dm.insert(dm.end(), r.dim_order[k].begin(), r.dim_order[k].end());
      }
      const std::string out = argv[4];
      write_vec(out + ".mp", v);
      write_vec(out + ".pi", pi);
      write_vec(out + ".dim", dm);
      std::printf("{\"size\": %lld, \"zone\": %lld, \"mode\": \"mstomp\", \"dims\": %lld}\n",
                  (long long)r.size(), (long long)r.exclusion_zone, (long long)r.data_dims);
      return 0;
    }
    if (mode == "simple") {
      const long long dims = std::atoll(argv[6]);
      const mprof::MultiTimeSeries a = read_mts(argv[1], dims);
      mprof::MatrixProfile mp;
      if (argc > 7) {
        const mprof::MultiTimeSeries b = read_mts(argv[7], dims);
        mp = mprof::simple_join(a, &b, std::atoll(argv[2]), std::atof(argv[3]));
      } else {
        mp = mprof::simple_join(a, nullptr, std::atoll(argv[2]), std::atof(argv[3]));
      }
      const std::string out = argv[4];
      write_vec(out + ".mp", mp.values);
      write_vec(out + ".pi", mp.index);
      write_vec(out + ".left", mp.left_index);
      write_vec(out + ".right", mp.right_index);
      std::printf("{\"size\": %lld, \"zone\": %lld, \"mode\": \"%s\", \"join\": \"%s\", \"dims\": %lld}\n",
                  (long long)mp.size(), (long long)mp.exclusion_zone, mprof::mode_name(mp.mode),
                  mp.join_kind == mprof::JoinKind::self ? "self" : "ab", (long long)mp.data_dims);
      return 0;
    }
    mprof::TimeSeries a(read_f64(argv[1]));
    const mprof::Index w = std::atoll(argv[2]);
    const double ez = std::atof(argv[3]);
    int progress_calls = 0;
    mprof::ProgressFn progress = [&](double) { ++progress_calls; };
    mprof::MatrixProfile mp;
    if (mode == "scrimp") {
      mp = mprof::scrimp(a, w, ez);
    } else if (mode == "anytime") {  // SCRIMP with s_size (anytime, profile.hpp:87-89)
      mp = mprof::scrimp(a, w, ez, std::atoll(argv[6]), std::strtoull(argv[7], nullptr, 10), progress);
    } else if (mode == "ab") {
      mprof::TimeSeries b(read_f64(argv[6]));
      mp = mprof::stomp(a, &b, w, ez, 1, progress);
    } else {
      mp = mprof::stomp(a, nullptr, w, ez, 1, progress);
    }
    const std::string out = argv[4];
    write_vec(out + ".mp", mp.values);
    write_vec(out + ".pi", mp.index);
    write_vec(out + ".left", mp.left_index);
    write_vec(out + ".right", mp.right_index);
    std::printf("{\"size\": %lld, \"zone\": %lld, \"mode\": \"%s\", \"join\": \"%s\", "
                "\"progress_calls\": %d, \"coverage\": %.17g}\n",
                (long long)mp.size(), (long long)mp.exclusion_zone, mprof::mode_name(mp.mode),
                mp.join_kind == mprof::JoinKind::self ? "self" : "ab", progress_calls, mp.coverage);
  } catch (const mprof::UnsupportedError &e) {
    std::printf("{\"error\": \"UnsupportedError\", \"what\": \"%s\"}\n", e.what());
    return 3;
  } catch (const mprof::ParameterError &e) {
    std::printf("{\"error\": \"ParameterError\", \"what\": \"%s\"}\n", e.what());
    return 2;
  } catch (const std::exception &e) {
    std::printf("{\"error\": \"runtime\", \"what\": \"%s\"}\n", e.what());
    return 4;
  }
  return 0;
}
