// A reference-API caller, unchanged except for linking libmprof_b200.so:
// reads a raw fp64 series, runs mprof::stomp (profile.hpp:80-83) or
// mprof::scrimp (profile.hpp:85-89), writes values/index/left/right as raw
// arrays. Used by tests/test_dropin_cpp.py to show the drop-in boundary.
//   dropin_example <in.f64> <window> <ez> <out_prefix>
//                  [stomp|scrimp|anytime <s_size> <seed>|ab <b.f64>]
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

int main(int argc, char **argv) {
  if (argc < 5) {
    std::fprintf(stderr, "usage: %s in.f64 window ez out_prefix [stomp|scrimp|anytime s seed|ab b.f64]\n",
                 argv[0]);
    return 1;
  }
  const std::string mode = argc > 5 ? argv[5] : "stomp";
  try {
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
