// pb200 — sweep kernel argument blocks and host launchers (pb_sweep.cu).
#pragma once
#include "pb_common.cuh"

namespace pb {

enum RngMode : int { kRngReplay = 0, kRngPhilox = 1 };

struct SweepScalars {   // device-resident per-problem scalars
  double gamma_s;       // weight precision
  double gamma_eps;     // noise precision
  double sq_w;          // sum S^2 after the code step
  double sq_r;          // sum R^2 after the code step
  int32_t epoch;        // epoch counter (the epoch being run = epoch + 1)
  int32_t diverged;
};
static_assert(sizeof(SweepScalars) == 40, "SweepScalars must match pb_scalars");

// pb_patches.cu
int launch_extract(const Grid&, const void*, int, const uint8_t*, int, float*, uint8_t*, float*, int32_t*,
                   cudaStream_t, int64_t i0 = 0, int64_t cnt = -1);
int launch_reconstitute(const Grid&, const float*, float, const float*, const void*, const uint8_t*, int, int, void*,
                        unsigned long long*, cudaStream_t);
int launch_coverage(const Grid&, int32_t*, cudaStream_t);
int launch_ola_partial(const Grid&, const float* est, float est_scale, const float* means, int64_t i0, int64_t cnt,
                       double* acc_out, cudaStream_t st);
// pb_sweep.cu
int launch_accumulate_atoms(bool resid, const float* values, const uint8_t* obs, const uint8_t* usage,
                            const float* weights, const float* atoms, float* out, int64_t n, int p, int k_len,
                            int accumulate, int64_t ld, cudaStream_t st);
int launch_finish_stats(const double*, int, SweepScalars*, cudaStream_t);
int launch_draw_pi_gamma(double*, const int32_t*, SweepScalars*, int, int64_t, int64_t, const double*, uint32_t,
                         uint32_t, cudaStream_t);
int launch_atom_moments(const float*, const uint8_t*, const float*, int64_t, int, double*, int, double*, double*,
                        cudaStream_t);
int launch_shift_atom(float*, const uint8_t*, const float*, const float*, int64_t, int, cudaStream_t);
int launch_code_moments(const float*, const uint8_t*, const float*, int64_t, int, float*, float*, cudaStream_t);
int launch_shift_codes(float*, const uint8_t*, const float*, const float*, int64_t, int, cudaStream_t);
int launch_sq_norm(const float*, int64_t, double*, int, double*, cudaStream_t);
int launch_prior_atoms(float* atoms, int k_len, int p, uint32_t key0, uint32_t key1, cudaStream_t st);
int launch_sum_counts(const int32_t* counts, int64_t n, unsigned long long* out, cudaStream_t st);

}  // namespace pb
