// Result types of the profile consumers (reference discovery.hpp:13-50), as
// the drop-in archive carries them. The GPU library computes FLUSS and
// discords (mpgpu_fluss / mpgpu_extract); motif and chain search are outside
// this build's scope, so only their result types are declared.
#ifndef MPROF_B200_DISCOVERY_HPP
#define MPROF_B200_DISCOVERY_HPP

#include <utility>
#include <vector>

#include "mprof/types.hpp"

namespace mprof {

struct MotifPair {
  Index anchor = kNone;
  Index pair = kNone;
  double distance = kInf;
  std::vector<Index> neighbors;  // ascending by distance to the anchor
};

struct MotifSet {
  std::vector<MotifPair> pairs;  // ascending by pair distance
  Index window = 0;
  double radius = 0.0;
  Index exclusion_zone = 0;
};

struct DiscordSet {
  std::vector<std::pair<Index, double>> discords;  // descending by distance
  Index exclusion_zone = 0;
  bool truncated = false;
};

struct ChainSet {
  std::vector<std::vector<Index>> chains;
  std::vector<Index> best_chain;
  Index count = 0;
};

struct FlussResult {
  std::vector<Index> arc_counts;
  std::vector<double> cac;  // corrected arc curve, in [0, 1]
  std::vector<Index> segments;
  double min_value = 1.0;
  Index min_index = kNone;
  bool truncated = false;
  Index window = 0;
  double exclusion_factor = 0.0;
};

}  // namespace mprof

#endif
