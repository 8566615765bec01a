// pb200 — B200-native BPFA inpainting hot path: shared device utilities.
//
// Device data layouts:
//   values / observed / resid / estimates : "plane-major" (P, N)  -> element p of
//       patch i at [p * N + i]; consecutive patches are contiguous, so one thread
//       (group) per patch gives coalesced loads for every p.
//   usage (u8) / weights (f32)             : atom-major (K, N) -> [k * N + i].
//   atoms                                  : (K, P) f32, staged into shared memory.
// Patch order is the reference's row-major grid order (patches.py:107-122).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "pb_tuning.cuh"

#define PB_OK 0
#define PB_ESHAPE -1
#define PB_EVALUE -2
#define PB_ECOVERAGE -3
#define PB_EDIVERGED -4
#define PB_ECUDA -5
#define PB_EUNSUPPORTED -6

namespace pb {

constexpr int kMaxRank = 4;  // patches.py:17

// Error message of the last failing call on this host thread.
void set_error(const char* fmt, ...);
const char* last_error();

#define PB_CUDA_TRY(expr)                                                       \
  do {                                                                          \
    cudaError_t _e = (expr);                                                    \
    if (_e != cudaSuccess) {                                                    \
      ::pb::set_error("%s:%d CUDA error %s: %s", __FILE__, __LINE__, #expr,     \
                      cudaGetErrorString(_e));                                  \
      return PB_ECUDA;                                                          \
    }                                                                           \
  } while (0)

#define PB_LAUNCH_CHECK() PB_CUDA_TRY(cudaGetLastError())

// ---------------------------------------------------------------------------
// Philox4x32-10 (Salmon et al., SC'11) — counter-based device RNG (philox mode).
struct u32x4 {
  uint32_t x, y, z, w;
};

__device__ __forceinline__ u32x4 philox4x32_10(u32x4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
    const uint32_t lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
    c = u32x4{hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0};
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return c;
}

// The same generator with the 10 round keys precomputed (kernel parameters:
// the XORs take them as constant-bank operands, no key schedule per block).
__device__ __forceinline__ u32x4 philox4x32_10_rk(u32x4 c, const uint32_t (&rk)[20]) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
    const uint32_t lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
    c = u32x4{hi1 ^ c.y ^ rk[2 * r], lo1, hi0 ^ c.w ^ rk[2 * r + 1], lo0};
  }
  return c;
}
inline void philox_round_keys(uint32_t k0, uint32_t k1, uint32_t (&rk)[20]) {
  for (int r = 0; r < 10; ++r) {
    rk[2 * r] = k0 + (uint32_t)r * 0x9E3779B9u;
    rk[2 * r + 1] = k1 + (uint32_t)r * 0xBB67AE85u;
  }
}

// (0,1) uniform with 24 random bits, exactly representable in f32.
__device__ __forceinline__ float u01_24(uint32_t u) {
  return (float)(u >> 8) * 5.9604644775390625e-08f + 2.98023223876953125e-08f;
}
// (0,1] uniform in f64 with 53 bits from two words.
__device__ __forceinline__ double u01_53(uint32_t a, uint32_t b) {
  const uint64_t v = ((uint64_t)a << 21) ^ (uint64_t)(b >> 11);
  return ((double)(v & ((1ull << 53) - 1)) + 1.0) * 1.1102230246251565e-16;
}

// Box-Muller pair from two 32-bit words.
__device__ __forceinline__ void box_muller(uint32_t a, uint32_t b, float& n0, float& n1) {
  const float u1 = fmaf((float)a, 2.3283064365386963e-10f, 1.1641532182693481e-10f);
  const float r = sqrtf(-2.0f * __logf(u1));
  float s, c;
  __sincosf(6.283185307179586f * u01_24(b), &s, &c);
  n0 = r * c;
  n1 = r * s;
}

// Domains for the device counters (mirror rng.py:14-20).
enum : uint32_t { kDomInit = 1, kDomAtom = 2, kDomCode = 3, kDomPi = 4, kDomGamma = 5, kDomMask = 6 };

// ---------------------------------------------------------------------------
// Reductions
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block-wide sum (deterministic tree); result valid in thread 0. `scratch` >= 32 doubles.
__device__ __forceinline__ double block_sum_d(double v, double* scratch) {
  v = warp_sum_d(v);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) scratch[wid] = v;
  __syncthreads();
  double t = 0.0;
  if (wid == 0) {
    const int nw = (blockDim.x + 31) >> 5;
    t = lane < nw ? scratch[lane] : 0.0;
    t = warp_sum_d(t);
  }
  return t;
}

__host__ __device__ __forceinline__ int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Grid geometry of one extraction (patches.py:35-77).
struct Grid {
  int rank;
  int64_t tshape[kMaxRank];   // tensor shape M
  int64_t tstride[kMaxRank];  // row-major element strides of the tensor
  int bshape[kMaxRank];       // patch shape B
  int step[kMaxRank];         // grid stride s
  int64_t gcount[kMaxRank];   // grid positions per dim
  int64_t n;                  // number of patches
  int p;                      // patch size
  int64_t m;                  // tensor element count
};

}  // namespace pb
