// TEST INFRASTRUCTURE ONLY. C entry point over the reference's own compiled
// TimeSeries constructor (/root/reference/proj/src/types.cpp:7-18 — the only
// reference function with a body). Built by oracle/Makefile into
// oracle/_ref/ so tests can pin the boundary's input validation against the
// real reference code. Never linked into the product.
#include <cstdint>
#include <cstring>
#include <exception>
#include <vector>

#include "mprof/types.hpp"

extern "C" int ref_timeseries_validate(const double *x, int64_t n, char *msg, int msg_len) {
  try {
    mprof::TimeSeries ts(std::vector<double>(x, x + n));
    (void)ts;
    return 0;
  } catch (const mprof::ParameterError &e) {
    if (msg && msg_len > 0) {
      std::strncpy(msg, e.what(), (size_t)msg_len - 1);
      msg[msg_len - 1] = 0;
    }
    return 2;
  } catch (const std::exception &e) {
    if (msg && msg_len > 0) {
      std::strncpy(msg, e.what(), (size_t)msg_len - 1);
      msg[msg_len - 1] = 0;
    }
    return 1;
  }
}
