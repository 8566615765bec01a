// pb200 — tensor-core compose_estimates (pb_compose_tc.cu).
#pragma once
#include <algorithm>

#include "pb_common.cuh"

namespace pb {

bool compose_tc_supported(int p);
// out (P, N) plane-major [+]= (Z∘S)^T D with Z/S atom-major (K, ld)
// scratch: compose_tc_scratch_bytes(p, k) bytes of device memory, or null for a
// stream-ordered allocation per call
size_t compose_tc_scratch_bytes(int p, int k_len);
int launch_compose_tc(const uint8_t* usage, const float* weights, int64_t ld, const float* atoms, int p, int k_len,
                      int64_t n, float* out, int accumulate, cudaStream_t st, float* scratch = nullptr);

}  // namespace pb
