// Distance primitives of the mprof drop-in API (reference distance.hpp:12-33).
// The scalar helpers run on the host; mass_distance_profile runs on the GPU
// (kernel K6 through mpgpu_mass_host).
#ifndef MPROF_B200_DISTANCE_HPP
#define MPROF_B200_DISTANCE_HPP

#include <span>
#include <vector>

#include "mprof/rolling.hpp"
#include "mprof/types.hpp"

namespace mprof {

// d^2 = 2w (1 - (qt - w mu_a mu_b) / (w sd_a sd_b)), clamped to [0, 4w];
// both windows flat (sd == 0) -> 0, exactly one flat -> sqrt(w).
double znorm_dist_from_qt(double qt, Index w, double mu_a, double sd_a, double mu_b, double sd_b);

// round-half-up(window * fraction); ParameterError for a negative fraction.
Index zone_size(Index window, double fraction);

// Entries with |i - center| <= zone become +inf; ParameterError unless
// 0 <= center < size and zone >= 0.
DistanceProfile apply_exclusion_zone(DistanceProfile dp, Index center, Index zone);
void apply_exclusion_zone_inplace(std::span<double> distances, Index center, Index zone);

// z-normalised distances from `query` to every window of `ts` on the GPU
// (exact direct dot products instead of the reference's FFT; near-zero hits
// recomputed so exact matches are 0). `stats` must be ts's rolling stats for
// the query length; the kernel recomputes the statistics exactly, so
// stats / query_mean / query_std only fix the convention. No exclusion zone is
// applied here (apply_exclusion_zone does that); query_index is recorded.
DistanceProfile mass_distance_profile(std::span<const double> query, std::span<const double> ts,
                                      const RollingStats &stats, double query_mean,
                                      double query_std, Index query_index = kNone);

}  // namespace mprof

#endif
