// pb200 — the train/inpaint entry points' device steps around the hot path:
//
//  normalize_observed  cli.py:195-212 (_normalize_observed): the affine map of a
//                      frame to [0, 1] computed from its OBSERVED values only
//                      (unobserved garbage never influences it); identity when
//                      the observed values already lie in [0, 1]; a constant
//                      observed set maps observed elements to 0 (offset lo).
//                      Two-stage f64 min/max reduction + one map pass.
//  transfer_atoms      bpfa.py:417-458 (transfer_dictionary): atoms of patch
//                      shape S re-used across the extra trailing dimensions of a
//                      destination patch shape S + E (each source element repeated
//                      prod(E) times, row-major), renormalized to unit norm (f64
//                      norm; zero atoms stay zero); equal shapes copy bitwise.
#include <float.h>

#include "../../include/pb200.h"
#include "pb_common.cuh"

namespace pb {

constexpr int kNormBlocks = 296;

__global__ void __launch_bounds__(256) k_observed_minmax(const double* __restrict__ frame,
                                                         const uint8_t* __restrict__ mask, int64_t m,
                                                         double* __restrict__ part) {
  double lo = DBL_MAX, hi = -DBL_MAX;
  unsigned long long cnt = 0;
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < m; x += (int64_t)gridDim.x * blockDim.x)
    if (mask[x]) {
      const double v = frame[x];
      lo = fmin(lo, v);
      hi = fmax(hi, v);
      ++cnt;
    }
  __shared__ double slo[8], shi[8];
  __shared__ unsigned long long scnt[8];
  for (int o = 16; o; o >>= 1) {
    lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  }
  if ((threadIdx.x & 31) == 0) { slo[threadIdx.x >> 5] = lo; shi[threadIdx.x >> 5] = hi; scnt[threadIdx.x >> 5] = cnt; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
      lo = fmin(lo, slo[w]);
      hi = fmax(hi, shi[w]);
      cnt += scnt[w];
    }
    part[3 * blockIdx.x] = lo;
    part[3 * blockIdx.x + 1] = hi;
    part[3 * blockIdx.x + 2] = (double)cnt;
  }
}

// one thread: the final min / max and the mapping (cli.py:203-212):
// res = {lo, hi, count, mode} with mode 0 identity, 1 constant, 2 affine
__global__ void k_observed_decide(const double* __restrict__ part, int nb, double* __restrict__ res) {
  double lo = DBL_MAX, hi = -DBL_MAX, cnt = 0.0;
  for (int b = 0; b < nb; ++b) {
    if (part[3 * b + 2] == 0.0) continue;
    lo = fmin(lo, part[3 * b]);
    hi = fmax(hi, part[3 * b + 1]);
    cnt += part[3 * b + 2];
  }
  double mode = 0.0;
  if (cnt > 0.0 && !(0.0 <= lo && hi <= 1.0)) mode = hi == lo ? 1.0 : 2.0;
  res[0] = lo; res[1] = hi; res[2] = cnt; res[3] = mode;
}

__global__ void __launch_bounds__(256) k_observed_map(const double* __restrict__ frame, const uint8_t* __restrict__ mask,
                                                      int64_t m, const double* __restrict__ res, double* __restrict__ out) {
  const int mode = (int)res[3];
  const double lo = res[0], span = res[1] - res[0];
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < m; x += (int64_t)gridDim.x * blockDim.x) {
    const double v = frame[x];
    out[x] = mode == 0 ? v : mode == 1 ? (mask[x] ? 0.0 : v) : (v - lo) / span;
  }
}

__global__ void __launch_bounds__(128) k_transfer_atoms(const float* __restrict__ src, int src_p, int repeat,
                                                        int normalize, float* __restrict__ dst) {
  const float* s = src + (int64_t)blockIdx.x * src_p;
  float* d = dst + (int64_t)blockIdx.x * src_p * repeat;
  double ss = 0.0;
  for (int q = threadIdx.x; q < src_p; q += blockDim.x) ss += (double)s[q] * (double)s[q];
  __shared__ double part[4];
  for (int o = 16; o; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = ss;
  __syncthreads();
  const double nrm = sqrt((part[0] + part[1] + part[2] + part[3]) * (double)repeat);
  const bool scale = normalize && nrm > 0.0;
  for (int e = threadIdx.x; e < src_p * repeat; e += blockDim.x) {
    const float v = s[e / repeat];
    d[e] = scale ? (float)((double)v / nrm) : v;
  }
}

int launch_transfer_atoms(const float* src, int k, int src_p, int repeat, int normalize, float* dst,
                          cudaStream_t st) {
  if (k < 1 || src_p < 1 || repeat < 1) { set_error("transfer: empty dictionary"); return PB_ESHAPE; }
  k_transfer_atoms<<<k, 128, 0, st>>>(src, src_p, repeat, normalize, dst);
  PB_LAUNCH_CHECK();
  return PB_OK;
}

}  // namespace pb

using namespace pb;

extern "C" {

int pb_normalize_observed(const double* frame, const uint8_t* mask, int64_t m, double* out, double* scale_out,
                          double* offset_out, void* stream) {
  if (!frame || !mask || !out || !scale_out || !offset_out || m < 0) { set_error("null argument"); return PB_EVALUE; }
  cudaStream_t st = (cudaStream_t)stream;
  double* buf = nullptr;
  PB_CUDA_TRY(cudaMallocAsync((void**)&buf, (size_t)(3 * kNormBlocks + 4) * sizeof(double), st));
  double* res = buf + 3 * kNormBlocks;
  k_observed_minmax<<<kNormBlocks, 256, 0, st>>>(frame, mask, m, buf);
  k_observed_decide<<<1, 1, 0, st>>>(buf, kNormBlocks, res);
  if (m > 0) k_observed_map<<<kNormBlocks, 256, 0, st>>>(frame, mask, m, res, out);
  double h[4] = {0, 0, 0, 0};
  const cudaError_t e1 = cudaGetLastError();
  const cudaError_t e2 = cudaMemcpyAsync(h, res, sizeof(h), cudaMemcpyDeviceToHost, st);
  cudaFreeAsync(buf, st);
  const cudaError_t e3 = cudaStreamSynchronize(st);
  if (e1 != cudaSuccess || e2 != cudaSuccess || e3 != cudaSuccess) { set_error("normalize_observed failed"); return PB_ECUDA; }
  const int mode = (int)h[3];
  *scale_out = mode == 2 ? h[1] - h[0] : 1.0;
  *offset_out = mode == 0 ? 0.0 : h[0];
  return PB_OK;
}

int pb_transfer_atoms(const float* src, int32_t k, int32_t src_p, int32_t repeat, int32_t normalize, float* dst,
                      void* stream) {
  if (!src || !dst) { set_error("null argument"); return PB_EVALUE; }
  return launch_transfer_atoms(src, k, src_p, repeat, normalize, dst, (cudaStream_t)stream);
}

}  // extern "C"
