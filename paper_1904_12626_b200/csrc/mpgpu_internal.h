// Internal interface between the translation units of libmprof_b200.so (not
// part of the C ABI): the shared error slot and the K1 window statistics.
#pragma once

#include <cstdint>
#include <string>

#include <cuda_runtime.h>

#include "mprof_gpu.h"

namespace mpgpu_internal {

// Record `msg` as this thread's mpgpu_last_error() and return `st`.
mpgpu_status set_error(mpgpu_status st, const std::string& msg);

// Zero padding (entries) after the last window of inv / U.
long long stats_pad();

// K1 on one device series: window means mu[L], inverse centred norms inv[L +
// pad] (0 = flat window or padding), update vectors U[L + pad] = {df, dg}
// (U[0] = 0), and flat[L] (may be null). Issued on `st`.
cudaError_t series_stats(const double* d_x, long long n, int m, double* mu, double* inv,
                         double2* U, uint8_t* flat, cudaStream_t st);

}  // namespace mpgpu_internal
