// A reference-API caller of the archive (archive.hpp:12-58), linked to
// libmprof_b200.so (host-only code: runs without a GPU).
//   archive_example roundtrip <out.json>     build an archive with every field
//                                            (+inf / -1 sentinels, 1e-300,
//                                            nextafter(1), embedded data, multi
//                                            profile, discord / FLUSS / motif /
//                                            chain results), write, read back,
//                                            compare field by field
//   archive_example convert <in.json> <out.json>   read (e.g. a Python-written
//                                            archive), print the summary block,
//                                            write it back
//   archive_example corrupt <in.json>        expect IoError on read
#include <cmath>
#include <cstdio>
#include <cstring>
#include <limits>
#include <string>
#include <vector>

#include "mprof/archive.hpp"

using namespace mprof;

static ProfileArchive sample() {
  ProfileArchive ar;
  ar.mode = Mode::scrimp;
  ar.ez_fraction = 0.25;
  MatrixProfile p;
  const Index L = 50;
  for (Index i = 0; i < L; ++i) {
    p.values.push_back(0.5 + 0.37 * (double)i);
    p.index.push_back((i * 7) % L);
    p.left_index.push_back(i > 3 ? i - 3 : -1);
    p.right_index.push_back(i + 5 < L ? i + 5 : -1);
  }
  p.values[0] = kInf;
  p.index[0] = -1;
  p.values[1] = 1e-300;
  p.values[2] = std::nextafter(1.0, 2.0);
  p.values[3] = 0.1;
  p.window = 8;
  p.exclusion_zone = 2;
  p.mode = Mode::scrimp;
  p.coverage = 0.1;
  p.seed = 12345678901ULL;
  p.data_len = L + 7;
  ar.profile = p;
  MultiMatrixProfile m;
  m.values = {{1.0, kInf}, {2.5, 3.0}};
  m.index = {{1, -1}, {0, 1}};
  m.dim_order = {{0, 1}, {1, -1}};
  m.window = 8;
  m.exclusion_zone = 2;
  m.must_dims = {1};
  m.exc_dims = {};
  m.data_len = 9;
  m.data_dims = 2;
  ar.multi = m;
  std::vector<double> a, b2;
  for (Index i = 0; i < L + 7; ++i) a.push_back(std::sin(0.1 * (double)i) * 3.0);
  for (Index i = 0; i < L + 7; ++i) b2.push_back(-1.0 / (1.0 + (double)i));
  ar.data_a = MultiTimeSeries({TimeSeries(a)});
  ar.data_b = MultiTimeSeries({TimeSeries(a), TimeSeries(b2)});
  ar.name_a = "walk \"A\"\n";
  ar.source_a = "gen:walk/7";
  DiscordSet ds;
  ds.discords = {{17, 9.25}, {3, 8.0}};
  ds.exclusion_zone = 4;
  ds.truncated = true;
  ar.discord = ds;
  FlussResult f;
  f.arc_counts = {0, 2, 3, 1};
  f.cac = {1.0, 0.4, 0.3, 1.0};
  f.segments = {2};
  f.min_value = 0.3;
  f.min_index = 2;
  f.window = 8;
  f.exclusion_factor = 5.0;
  ar.fluss = f;
  MotifSet ms;
  ms.pairs = {{4, 30, 0.75, {12, 40}}};
  ms.window = 8;
  ms.radius = 2.0;
  ms.exclusion_zone = 4;
  ar.motif = ms;
  ChainSet cs;
  cs.chains = {{1, 5, 9}};
  cs.best_chain = {1, 5, 9};
  cs.count = 1;
  ar.chain = cs;
  return ar;
}

template <typename T>
static bool same_bits(const std::vector<T>& x, const std::vector<T>& y) {
  return x.size() == y.size() && (x.empty() || std::memcmp(x.data(), y.data(), sizeof(T) * x.size()) == 0);
}

int main(int argc, char** argv) {
  if (argc < 3) return 64;
  const std::string cmd = argv[1];
  try {
    if (cmd == "roundtrip") {
      const ProfileArchive ar = sample();
      write_profile(ar, argv[2]);
      const ProfileArchive back = read_profile(argv[2]);
      const MatrixProfile &p = *ar.profile, &q = *back.profile;
      bool ok = back.mode == ar.mode && back.ez_fraction == ar.ez_fraction &&
                same_bits(p.values, q.values) && same_bits(p.index, q.index) &&
                same_bits(p.left_index, q.left_index) && same_bits(p.right_index, q.right_index) &&
                q.window == p.window && q.exclusion_zone == p.exclusion_zone &&
                q.coverage == p.coverage && q.seed == p.seed && q.data_len == p.data_len &&
                q.mode == p.mode && q.join_kind == p.join_kind;
      ok = ok && back.multi && back.multi->values == ar.multi->values &&
           back.multi->index == ar.multi->index && back.multi->dim_order == ar.multi->dim_order &&
           back.multi->must_dims == ar.multi->must_dims && back.multi->data_dims == 2;
      ok = ok && back.data_a && back.data_a->dims() == 1 &&
           same_bits(back.data_a->dim(0).values(), ar.data_a->dim(0).values()) && back.data_b &&
           back.data_b->dims() == 2 && same_bits(back.data_b->dim(1).values(), ar.data_b->dim(1).values());
      ok = ok && back.name_a == ar.name_a && back.source_a == ar.source_a && back.name_b.empty();
      ok = ok && back.discord && back.discord->discords == ar.discord->discords &&
           back.discord->truncated && back.fluss && back.fluss->cac == ar.fluss->cac &&
           back.fluss->segments == ar.fluss->segments && back.fluss->min_index == 2;
      ok = ok && back.motif && back.motif->pairs.size() == 1 && back.motif->pairs[0].pair == 30 &&
           back.motif->pairs[0].neighbors == ar.motif->pairs[0].neighbors && back.chain &&
           back.chain->chains == ar.chain->chains;
      ok = ok && archive_to_json(back) == archive_to_json(ar);  // canonical: text round trip
      ok = ok && back.profile_size() == 50 && back.window() == 8 && back.coverage() == 0.1 &&
           !back.is_ab() && back.data_dims() == 1;
      std::printf("{\"ok\": %s}\n", ok ? "true" : "false");
      std::fputs(render_profile_block(back).c_str(), stderr);
      std::fputs(render_discord_block(*back.discord).c_str(), stderr);
      std::fputs(render_fluss_block(*back.fluss, back.profile_size()).c_str(), stderr);
      return ok ? 0 : 1;
    }
    if (cmd == "convert" && argc >= 4) {
      const ProfileArchive ar = read_profile(argv[2]);
      write_profile(ar, argv[3]);
      std::fputs(render_profile_block(ar).c_str(), stdout);
      return 0;
    }
    if (cmd == "corrupt") {
      try {
        (void)read_profile(argv[2]);
      } catch (const IoError& e) {
        std::printf("IoError: %s\n", e.what());
        return 0;
      }
      return 1;
    }
  } catch (const std::exception& e) {
    std::printf("{\"error\": \"%s\"}\n", e.what());
    return 2;
  }
  return 64;
}
