// pb200 — tensor-core compose_estimates (pb_compose_tc.cu).
#pragma once
#include <algorithm>

#include "pb_common.cuh"

namespace pb {

bool compose_tc_supported(int p);
// out (P, N) plane-major [+]= (Z∘S)^T D with Z/S atom-major (K, ld)
int launch_compose_tc(const uint8_t* usage, const float* weights, int64_t ld, const float* atoms, int p, int k_len,
                      int64_t n, float* out, int accumulate, cudaStream_t st);

}  // namespace pb
