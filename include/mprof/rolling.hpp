// Window statistics of the mprof drop-in API (reference rolling.hpp:11-29).
// rolling_mean_std runs on the GPU (kernel K1 through mpgpu_rolling_stats):
// exact two-pass mean and population std per window rather than the
// reference's centred cumulative sums, with flat windows floored to sd = 0.
#ifndef MPROF_B200_ROLLING_HPP
#define MPROF_B200_ROLLING_HPP

#include <span>
#include <vector>

#include "mprof/types.hpp"

namespace mprof {

struct RollingStats {
  std::vector<double> means;  // length n - window + 1
  std::vector<double> stds;   // population std (divisor window); 0 for flat windows
  Index window = 0;

  Index size() const { return static_cast<Index>(means.size()); }
};

// Flat-window test: sd <= 1e-10 * max(1, |mean|) (the reference leaves the
// threshold open; DESIGN.md §3 fixes it, the GPU kernels use the same rule).
bool is_flat_std(double sd, double mean);

// Means and population stds of every window; ParameterError unless
// kMinWindow <= window <= ts.size().
RollingStats rolling_mean_std(std::span<const double> ts, Index window);

}  // namespace mprof

#endif
