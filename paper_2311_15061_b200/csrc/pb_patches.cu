// pb200 — N-D strided patch extraction and gather-form overlap-add.
//
// Reference behaviour (pkg/src/patchbeam/patches.py):
//   grid / origins          : 64-70, 107-113 (row-major grid, origins g_d * s_d)
//   extract_patches         : 125-164 (values = x*o; observed-only mean; (x-mean)*o)
//   reconstitute            : 188-215 (sum of (est + mean) over covering patches in
//                             ascending patch order, / coverage; uncovered -> 0)
//   apply_data_consistency  : 218-229 (fused here as the OLA epilogue)
//
// B200 design: extraction is one thread per patch writing the plane-major (P, N)
// matrix, so every store instruction of a warp is a contiguous 128 B line and the
// tensor reads along the fastest dim are contiguous for stride 1.  Overlap-add
// is a gather (one thread per output element, coverage computed analytically),
// so it is deterministic and atomic-free; neighbouring output elements read
// neighbouring patches at the same offset -> coalesced.  Both are HBM-bound.
#include <algorithm>

#include "pb_sweep.cuh"

namespace pb {

// Padded-to-rank-4 geometry in constant-friendly POD form.
struct Geo4 {
  int64_t tstride[4];
  int64_t tshape[4];
  int64_t gcount[4];
  int64_t gstride[4];  // row-major strides over the patch grid
  int bshape[4];
  int bstride[4];      // row-major strides within a patch
  int step[4];
  int64_t n, m;
  int p;
};

static Geo4 make_geo4(const Grid& g) {
  Geo4 o;
  const int pad = kMaxRank - g.rank;
  for (int d = 0; d < 4; ++d) {
    if (d < pad) {
      o.tshape[d] = 1; o.bshape[d] = 1; o.step[d] = 1; o.gcount[d] = 1;
    } else {
      o.tshape[d] = g.tshape[d - pad]; o.bshape[d] = g.bshape[d - pad];
      o.step[d] = g.step[d - pad]; o.gcount[d] = g.gcount[d - pad];
    }
  }
  int64_t acc = 1, gacc = 1;
  int bacc = 1;
  for (int d = 3; d >= 0; --d) {
    o.tstride[d] = acc; acc *= o.tshape[d];
    o.gstride[d] = gacc; gacc *= o.gcount[d];
    o.bstride[d] = bacc; bacc *= o.bshape[d];
  }
  o.m = acc; o.n = gacc; o.p = bacc;
  return o;
}

// Patches [i0, i0 + cnt) of the grid (a shard; i0 = 0, cnt = N for the whole
// matrix) into a (P, cnt) plane-major patch matrix.
template <typename T>
__global__ void __launch_bounds__(256) k_extract(Geo4 g, const T* __restrict__ tensor,
                                                 const uint8_t* __restrict__ mask, int mean_subtract,
                                                 float* __restrict__ values, uint8_t* __restrict__ obs,
                                                 float* __restrict__ means, int32_t* __restrict__ counts, int64_t i0,
                                                 int64_t cnt_patches) {
  for (int64_t li = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; li < cnt_patches;
       li += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = i0 + li;
    int64_t base = 0, rem = i;
#pragma unroll
    for (int d = 0; d < 4; ++d) {
      const int64_t gd = rem / g.gstride[d];
      rem -= gd * g.gstride[d];
      base += gd * g.step[d] * g.tstride[d];
    }
    // pass 1: observed count and observed-only sum (f64 accumulation)
    double sum = 0.0;
    int cnt = 0;
    {
      int q0 = 0, q1 = 0, q2 = 0, q3 = 0;
      for (int p = 0; p < g.p; ++p) {
        const int64_t off = base + q0 * g.tstride[0] + q1 * g.tstride[1] + q2 * g.tstride[2] + q3 * g.tstride[3];
        if (mask[off]) { sum += (double)tensor[off]; ++cnt; }
        if (++q3 == g.bshape[3]) { q3 = 0; if (++q2 == g.bshape[2]) { q2 = 0; if (++q1 == g.bshape[1]) { q1 = 0; ++q0; } } }
      }
    }
    const double mean = (mean_subtract && cnt > 0) ? sum / (double)cnt : 0.0;
    means[li] = (float)mean;
    counts[li] = cnt;
    // pass 2: plane-major write
    int q0 = 0, q1 = 0, q2 = 0, q3 = 0;
    for (int p = 0; p < g.p; ++p) {
      const int64_t off = base + q0 * g.tstride[0] + q1 * g.tstride[1] + q2 * g.tstride[2] + q3 * g.tstride[3];
      const uint8_t o = mask[off] ? 1 : 0;
      values[(int64_t)p * cnt_patches + li] = o ? (float)((double)tensor[off] - mean) : 0.0f;
      obs[(int64_t)p * cnt_patches + li] = o;
      if (++q3 == g.bshape[3]) { q3 = 0; if (++q2 == g.bshape[2]) { q2 = 0; if (++q1 == g.bshape[1]) { q1 = 0; ++q0; } } }
    }
  }
}

__device__ __forceinline__ void cover_range(int64_t c, int b, int s, int64_t gc, int64_t& lo, int64_t& hi) {
  const int64_t t = c - b + 1;
  lo = t <= 0 ? 0 : (t + s - 1) / s;
  hi = c / s;
  if (hi > gc - 1) hi = gc - 1;
}

// out[x] = sum_{i covers x} (est_scale*est[p,i] + mean_i) / cov(x); DC epilogue.
template <typename T>
__global__ void __launch_bounds__(256) k_reconstitute(Geo4 g, const float* __restrict__ est, float est_scale,
                                                      const float* __restrict__ means, const T* __restrict__ original,
                                                      const uint8_t* __restrict__ mask, int dc, T* __restrict__ out,
                                                      unsigned long long* __restrict__ uncovered) {
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < g.m;
       x += (int64_t)gridDim.x * blockDim.x) {
    int64_t c[4], lo[4], hi[4], rem = x;
#pragma unroll
    for (int d = 0; d < 4; ++d) {
      c[d] = rem / g.tstride[d];
      rem -= c[d] * g.tstride[d];
      cover_range(c[d], g.bshape[d], g.step[d], g.gcount[d], lo[d], hi[d]);
    }
    int64_t cov = 1;
#pragma unroll
    for (int d = 0; d < 4; ++d) cov *= (hi[d] >= lo[d]) ? (hi[d] - lo[d] + 1) : 0;
    double acc = 0.0;
    if (cov > 0) {
      for (int64_t a0 = lo[0]; a0 <= hi[0]; ++a0)
        for (int64_t a1 = lo[1]; a1 <= hi[1]; ++a1)
          for (int64_t a2 = lo[2]; a2 <= hi[2]; ++a2)
            for (int64_t a3 = lo[3]; a3 <= hi[3]; ++a3) {
              const int64_t i = a0 * g.gstride[0] + a1 * g.gstride[1] + a2 * g.gstride[2] + a3 * g.gstride[3];
              const int64_t p = (c[0] - a0 * g.step[0]) * g.bstride[0] + (c[1] - a1 * g.step[1]) * g.bstride[1] +
                                (c[2] - a2 * g.step[2]) * g.bstride[2] + (c[3] - a3 * g.step[3]) * g.bstride[3];
              acc += (double)est[p * g.n + i] * (double)est_scale + (double)means[i];
            }
    }
    double v = cov > 0 ? acc / (double)cov : 0.0;
    if (cov == 0 && uncovered) atomicAdd(uncovered, 1ull);
    if (dc && mask[x]) v = (double)original[x];
    out[x] = (T)v;
  }
}

// Shard of the overlap-add: raw sums (no division) of the covering patches in
// [i0, i0 + cnt), est/means indexed shard-locally; the caller allreduces the
// sums across ranks and divides by the (analytic, global) coverage.
__global__ void __launch_bounds__(256) k_ola_partial(Geo4 g, const float* __restrict__ est, float est_scale,
                                                     const float* __restrict__ means, int64_t i0, int64_t cnt,
                                                     double* __restrict__ acc_out) {
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < g.m;
       x += (int64_t)gridDim.x * blockDim.x) {
    int64_t c[4], lo[4], hi[4], rem = x;
#pragma unroll
    for (int d = 0; d < 4; ++d) {
      c[d] = rem / g.tstride[d];
      rem -= c[d] * g.tstride[d];
      cover_range(c[d], g.bshape[d], g.step[d], g.gcount[d], lo[d], hi[d]);
    }
    double acc = 0.0;
    for (int64_t a0 = lo[0]; a0 <= hi[0]; ++a0)
      for (int64_t a1 = lo[1]; a1 <= hi[1]; ++a1)
        for (int64_t a2 = lo[2]; a2 <= hi[2]; ++a2)
          for (int64_t a3 = lo[3]; a3 <= hi[3]; ++a3) {
            const int64_t i = a0 * g.gstride[0] + a1 * g.gstride[1] + a2 * g.gstride[2] + a3 * g.gstride[3];
            if (i < i0 || i >= i0 + cnt) continue;
            const int64_t p = (c[0] - a0 * g.step[0]) * g.bstride[0] + (c[1] - a1 * g.step[1]) * g.bstride[1] +
                              (c[2] - a2 * g.step[2]) * g.bstride[2] + (c[3] - a3 * g.step[3]) * g.bstride[3];
            acc += (double)est[p * cnt + (i - i0)] * (double)est_scale + (double)means[i - i0];
          }
    acc_out[x] = acc;
  }
}

__global__ void k_coverage(Geo4 g, int32_t* __restrict__ out) {
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < g.m;
       x += (int64_t)gridDim.x * blockDim.x) {
    int64_t rem = x, cov = 1;
#pragma unroll
    for (int d = 0; d < 4; ++d) {
      const int64_t c = rem / g.tstride[d];
      rem -= c * g.tstride[d];
      int64_t lo, hi;
      cover_range(c, g.bshape[d], g.step[d], g.gcount[d], lo, hi);
      cov *= hi >= lo ? hi - lo + 1 : 0;
    }
    out[x] = (int32_t)cov;
  }
}


// ---- rank-2 fast paths (2-D frames: configs[0..2], [4], the live path) ----
// Extraction: a CTA takes a 8 x 32 tile of patch origins, stages the tensor /
// mask window those patches cover into shared memory once (coalesced row
// reads; 17 x 41 elements for 10x10 patches instead of 256 x 100 scattered
// re-reads), then each thread builds its patch from shared memory: observed
// count and f64 observed-only sum, then the plane-major (P, N) row writes
// (each warp store a contiguous 128 B line of one plane).
struct Geo2 {
  int64_t m0, m1, gc0, gc1, n;
  int b0, b1, s0, s1, p, w0, w1;
};
constexpr int kXR = 8, kXC = 32;   // origin tile of the 2-D extraction

static Geo2 make_geo2(const Grid& g) {
  Geo2 o;
  o.m0 = g.tshape[0]; o.m1 = g.tshape[1];
  o.gc0 = g.gcount[0]; o.gc1 = g.gcount[1];
  o.n = g.n;
  o.b0 = g.bshape[0]; o.b1 = g.bshape[1];
  o.s0 = g.step[0]; o.s1 = g.step[1];
  o.p = g.p;
  o.w0 = (kXR - 1) * o.s0 + o.b0;
  o.w1 = (kXC - 1) * o.s1 + o.b1;
  return o;
}

template <typename T>
__global__ void __launch_bounds__(kXR * kXC) k_extract2d(Geo2 g, const T* __restrict__ tensor,
                                                         const uint8_t* __restrict__ mask, int mean_subtract,
                                                         float* __restrict__ values, uint8_t* __restrict__ obs,
                                                         float* __restrict__ means, int32_t* __restrict__ counts,
                                                         int64_t i0, int64_t cnt_patches) {
  extern __shared__ __align__(16) unsigned char xs[];
  T* sv = (T*)xs;
  uint8_t* so = (uint8_t*)(sv + (size_t)g.w0 * g.w1);
  const int64_t ntx = (g.gc1 + kXC - 1) / kXC, nty = (g.gc0 + kXR - 1) / kXR;
  const int ty = threadIdx.x / kXC, tx = threadIdx.x % kXC;
  // tiles overlapping the patch range [i0, i0 + cnt) (rows of the origin grid)
  const int64_t gy_lo = i0 / g.gc1, gy_hi = (i0 + cnt_patches - 1) / g.gc1;
  const int64_t t_lo = (gy_lo / kXR) * ntx, t_hi = min(nty, gy_hi / kXR + 1) * ntx;
  for (int64_t tile = t_lo + blockIdx.x; tile < t_hi; tile += gridDim.x) {
    const int64_t gy0 = (tile / ntx) * kXR, gx0 = (tile % ntx) * kXC;
    const int64_t y0 = gy0 * g.s0, x0 = gx0 * g.s1;
    __syncthreads();   // the previous tile's window is consumed
    for (int e = threadIdx.x; e < g.w0 * g.w1; e += blockDim.x) {
      const int r = e / g.w1, c = e - r * g.w1;
      const int64_t y = y0 + r, x = x0 + c;
      const bool in = y < g.m0 && x < g.m1;
      sv[e] = in ? tensor[y * g.m1 + x] : (T)0;
      so[e] = in ? mask[y * g.m1 + x] : 0;
    }
    __syncthreads();
    const int64_t gy = gy0 + ty, gx = gx0 + tx;
    if (gy >= g.gc0 || gx >= g.gc1) continue;
    const int64_t i = gy * g.gc1 + gx;
    if (i < i0 || i >= i0 + cnt_patches) continue;
    const int64_t li = i - i0;
    const int wb = ty * g.s0 * g.w1 + tx * g.s1;
    double sum = 0.0;
    int cnt = 0;
    for (int a = 0; a < g.b0; ++a) {
      const int rb = wb + a * g.w1;
      for (int b = 0; b < g.b1; ++b)
        if (so[rb + b]) { sum += (double)sv[rb + b]; ++cnt; }
    }
    const double mean = (mean_subtract && cnt > 0) ? sum / (double)cnt : 0.0;
    means[li] = (float)mean;
    counts[li] = cnt;
    int64_t q = li;
    for (int a = 0; a < g.b0; ++a) {
      const int rb = wb + a * g.w1;
      for (int b = 0; b < g.b1; ++b, q += cnt_patches) {
        const uint8_t o = so[rb + b] ? 1 : 0;
        values[q] = o ? (float)((double)sv[rb + b] - mean) : 0.0f;
        obs[q] = o;
      }
    }
  }
}


// Row variant (stride-1-sized windows): a CTA takes 256 consecutive patch
// origins of ONE grid row, shifted per row so that every warp's 32 patches
// start at a multiple of 32 in the output (each warp store one whole aligned
// 128-byte line of a plane: no partial-sector writes, whose read-for-ownership
// cost the 8x32-tile kernel 100 MB of DRAM reads at configs[1]).  The window is
// B0 rows x (255*s1 + B1) elements.
constexpr int kXW = 256;
template <typename T, int CB0, int CB1>   // CB0, CB1 > 0: patch shape known at compile time (unrolled plane loop)
__global__ void __launch_bounds__(kXW, CB0 == 8 ? 3 : (CB0 == 10 ? 2 : 1)) k_extract2r(Geo2 g, const T* __restrict__ tensor, const uint8_t* __restrict__ mask,
                                                   int mean_subtract, float* __restrict__ values,
                                                   uint8_t* __restrict__ obs, float* __restrict__ means,
                                                   int32_t* __restrict__ counts, int64_t i0, int64_t cnt_patches,
                                                   int tiles_per_row) {
  extern __shared__ __align__(16) unsigned char xs[];
  const int w1 = (kXW - 1) * g.s1 + g.b1;
  double* csum = (double*)xs;                     // per window column: observed sum over the B0 rows
  int* ccnt = (int*)(csum + w1);                  // ... and observed count
  T* sv = (T*)(ccnt + ((w1 + 1) & ~1));
  uint8_t* so = (uint8_t*)(sv + (size_t)g.b0 * w1);
  const int64_t gy_lo = i0 / g.gc1, gy_hi = (i0 + cnt_patches - 1) / g.gc1;
  const int64_t ntile = (gy_hi - gy_lo + 1) * tiles_per_row;
  for (int64_t tile = blockIdx.x; tile < ntile; tile += gridDim.x) {
    const int64_t gy = gy_lo + tile / tiles_per_row;
    const int k = (int)(tile % tiles_per_row);
    const int off = (int)((((gy * g.gc1 - i0) % 32) + 32) % 32);
    const int64_t sx = (int64_t)((32 - off) % 32) - kXW + (int64_t)kXW * k;   // first origin of the tile (may be < 0)
    __syncthreads();   // the previous tile's window is consumed
    const int64_t y0 = gy * g.s0, x0 = sx * g.s1;
    if constexpr (CB0 > 0) {
      // window rows unrolled: a thread's CB0 loads of column c are all in flight
      // before the first shared store (one load latency per tile, not CB0)
      for (int c = threadIdx.x; c < w1; c += blockDim.x) {
        const int64_t x = x0 + c;
        T v[CB0];
        uint8_t mk[CB0];
#pragma unroll
        for (int r = 0; r < CB0; ++r) {
          const int64_t y = y0 + r;
          const bool in = x >= 0 && y < g.m0 && x < g.m1;
          v[r] = in ? tensor[y * g.m1 + x] : (T)0;
          mk[r] = in ? mask[y * g.m1 + x] : 0;
        }
#pragma unroll
        for (int r = 0; r < CB0; ++r) {
          sv[r * w1 + c] = v[r];
          so[r * w1 + c] = mk[r];
        }
      }
    } else {
      for (int e = threadIdx.x; e < g.b0 * w1; e += blockDim.x) {
        const int r = e / w1, c = e - r * w1;
        const int64_t y = y0 + r, x = x0 + c;
        const bool in = x >= 0 && y < g.m0 && x < g.m1;
        sv[e] = in ? tensor[y * g.m1 + x] : (T)0;
        so[e] = in ? mask[y * g.m1 + x] : 0;
      }
    }
    __syncthreads();
    // column sums of the window (shared by the B1 patches that cover a column):
    // a patch's observed sum / count is then B1 column terms instead of B0*B1
    for (int c = threadIdx.x; c < w1; c += blockDim.x) {
      double cs = 0.0;
      int cc = 0;
      for (int a = 0; a < g.b0; ++a)
        if (so[a * w1 + c]) { cs += (double)sv[a * w1 + c]; ++cc; }
      csum[c] = cs;
      ccnt[c] = cc;
    }
    __syncthreads();
    const int64_t gx = sx + threadIdx.x;
    if (gx < 0 || gx >= g.gc1) continue;
    const int64_t i = gy * g.gc1 + gx;
    if (i < i0 || i >= i0 + cnt_patches) continue;
    const int64_t li = i - i0;
    const int wb = threadIdx.x * g.s1;
    double sum = 0.0;
    int cnt = 0;
    for (int b = 0; b < g.b1; ++b) { sum += csum[wb + b]; cnt += ccnt[wb + b]; }
    const double mean = (mean_subtract && cnt > 0) ? sum / (double)cnt : 0.0;
    means[li] = (float)mean;
    counts[li] = cnt;
    if constexpr (CB0 > 0 && CB1 > 0) {
      // unrolled: shared loads at immediate offsets, one pointer bump per plane
      float* vp = values + li;
      uint8_t* op = obs + li;
      const T* svb = sv + wb;
      const uint8_t* sob = so + wb;
#pragma unroll
      for (int a = 0; a < CB0; ++a)
#pragma unroll
        for (int b = 0; b < CB1; ++b) {
          const uint8_t o = sob[a * w1 + b] ? 1 : 0;
          *vp = o ? (float)((double)svb[a * w1 + b] - mean) : 0.0f;
          *op = o;
          vp += cnt_patches;
          op += cnt_patches;
        }
    } else {
      int64_t q = li;
      for (int a = 0; a < g.b0; ++a) {
        const int rb = wb + a * w1;
        for (int b = 0; b < g.b1; ++b, q += cnt_patches) {
          const uint8_t o = so[rb + b] ? 1 : 0;
          values[q] = o ? (float)((double)sv[rb + b] - mean) : 0.0f;
          obs[q] = o;
        }
      }
    }
  }
}

// Overlap-add, rank 2: one thread per output element, covering patches in
// ascending patch order (the reference's bincount order) with incremental
// patch / offset indices.
template <typename T, int B1>   // B1 > 0: patch width known at compile time (inner loop unrolled)
__global__ void __launch_bounds__(256) k_reconstitute2d(Geo2 g, const float* __restrict__ est, float est_scale,
                                                        const float* __restrict__ means, const T* __restrict__ original,
                                                        const uint8_t* __restrict__ mask, int dc, T* __restrict__ out,
                                                        unsigned long long* __restrict__ uncovered) {
  const int64_t m = g.m0 * g.m1;
  for (int64_t xx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; xx < m; xx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t y = xx / g.m1, x = xx - y * g.m1;
    int64_t lo0, hi0, lo1, hi1;
    cover_range(y, g.b0, g.s0, g.gc0, lo0, hi0);
    cover_range(x, g.b1, g.s1, g.gc1, lo1, hi1);
    const int64_t cov = (hi0 >= lo0 && hi1 >= lo1) ? (hi0 - lo0 + 1) * (hi1 - lo1 + 1) : 0;
    double acc = 0.0;
    for (int64_t a0 = lo0; a0 <= hi0; ++a0) {
      const int64_t ir = a0 * g.gc1;
      const int64_t pr = (y - a0 * g.s0) * g.b1 + x;
      if constexpr (B1 > 0) {
        // stride 1 along the row (the common case): the row's covering patches are
        // a1 = lo1..hi1 (at most B1); all loads issue before the ordered adds
        if (g.s1 == 1) {
          float e[B1], mu[B1];
          const int cnt = (int)(hi1 - lo1 + 1);
#pragma unroll
          for (int u = 0; u < B1; ++u) {
            e[u] = 0.f; mu[u] = 0.f;
            if (u < cnt) {
              const int64_t a1 = lo1 + u, i = ir + a1, pe = pr - a1;
              e[u] = est[pe * g.n + i];
              mu[u] = means[i];
            }
          }
#pragma unroll
          for (int u = 0; u < B1; ++u)
            if (u < cnt) acc += (double)e[u] * (double)est_scale + (double)mu[u];
          continue;
        }
      }
      for (int64_t a1 = lo1; a1 <= hi1; ++a1) {
        const int64_t i = ir + a1, pe = pr - a1 * g.s1;
        acc += (double)est[pe * g.n + i] * (double)est_scale + (double)means[i];
      }
    }
    double v = cov > 0 ? acc / (double)cov : 0.0;
    if (cov == 0 && uncovered) atomicAdd(uncovered, 1ull);
    if (dc && mask[xx]) v = (double)original[xx];
    out[xx] = (T)v;
  }
}

// Overlap-add, rank 2, stride 1 along the row, patch width B1 in {8, 10}: a
// CTA takes kOW consecutive output elements of ONE frame row y.  Every (patch
// row a0, patch column c) pair that covers the row is one contiguous run of
// the plane (y - a0*s0)*B1 + c over the patches a0*gc1 + [x0-B1+1, x0+kOW),
// so per covering patch row the CTA stages B1 runs plus the means run into
// shared memory with cp.async (coalesced, no register staging; the next patch
// row's stage is in flight while this one is summed — double buffered), and
// each thread adds its pixel's covering patches in the reference's ascending
// patch order.  Run entries of patches that do not exist (a1 < 0 or >= gc1,
// the frame's left / right margins) are zero, so the pixel loop is uniform and
// unrolled: a missing patch adds +0.0, which leaves the f64 sum unchanged
// (bit-identical to k_reconstitute2d, tests/test_gpu_patches.py).
// Measured (configs[1], tools/patch_timing.py): gather form 0.187 ms -> all
// rows staged at once 0.16 -> double-buffered rows, kOW 128: 0.140 -> kOW 256:
// 0.121 ms; a three-stage ring measured 0.138, and 16-byte cp.async chunks (runs
// staged at their global 16-byte alignment, a per-run shift in the sum) 0.163.
constexpr int kOW = 256;
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(gmem) : "memory");
}

template <typename T, int B1>
__global__ void __launch_bounds__(kOW) k_ola2s(Geo2 g, const float* __restrict__ est, float est_scale,
                                               const float* __restrict__ means, const T* __restrict__ original,
                                               const uint8_t* __restrict__ mask, int dc, T* __restrict__ out,
                                               unsigned long long* __restrict__ uncovered) {
  constexpr int L = kOW + B1 - 1;                 // patch columns a staged run spans
  constexpr int LP = L + 1;                       // run pitch
  constexpr int SZ = (B1 + 1) * LP;               // one stage: B1 runs + the means run
  constexpr int NS = 2;                           // double-buffered patch-row stages
  __shared__ __align__(16) float os[NS][SZ];
  const int64_t segs = (g.m1 + kOW - 1) / kOW;
  const int64_t ntile = g.m0 * segs;
  const double scale = (double)est_scale;
  for (int64_t tile = blockIdx.x; tile < ntile; tile += gridDim.x) {
    const int64_t y = tile / segs, x0 = (tile - y * segs) * kOW;
    int64_t lo0, hi0;
    cover_range(y, g.b0, g.s0, g.gc0, lo0, hi0);
    const int na = hi0 >= lo0 ? (int)(hi0 - lo0 + 1) : 0;
    const int64_t base = x0 - B1 + 1;             // patch column of run element 0
    // stage patch row a0 = lo0 + j into buffer j % NS (one cp.async group)
    auto issue = [&](int j) {
      const int64_t a0 = lo0 + j;
      const float* src = est + (y - a0 * g.s0) * B1 * g.n + a0 * g.gc1 + base;
      const float* msrc = means + a0 * g.gc1 + base;
      float* dst = os[j % NS];
      for (int t = threadIdx.x; t < L; t += kOW) {
        const int64_t a1 = base + t;
        if (a1 < 0 || a1 >= g.gc1) {            // no such patch: a zero term
#pragma unroll
          for (int c = 0; c <= B1; ++c) dst[c * LP + t] = 0.f;
          continue;
        }
        const float* sp = src + t;
#pragma unroll
        for (int c = 0; c < B1; ++c, sp += g.n) cp_async4(dst + c * LP + t, sp);
        cp_async4(dst + B1 * LP + t, msrc + t);
      }
      asm volatile("cp.async.commit_group;\n" ::: "memory");
    };
    __syncthreads();                              // the previous tile's stages are consumed
    if (na > 0) issue(0);
    const int64_t x = x0 + threadIdx.x;
    double acc = 0.0;
    for (int j = 0; j < na; ++j) {
      if (j + 1 < na) {
        issue(j + 1);                             // its buffer was released by the barrier below
        asm volatile("cp.async.wait_group 1;\n" ::: "memory");
      } else {
        asm volatile("cp.async.wait_group 0;\n" ::: "memory");
      }
      __syncthreads();
      // patch a1 = x - B1 + 1 + u: run column threadIdx.x + u, plane column B1 - 1 - u
      const float* run = os[j % NS] + threadIdx.x;
#pragma unroll
      for (int u = 0; u < B1; ++u) acc += (double)run[(B1 - 1 - u) * LP + u] * scale + (double)run[B1 * LP + u];
      __syncthreads();
    }
    if (x >= g.m1) continue;
    int64_t lo1, hi1;
    cover_range(x, B1, 1, g.gc1, lo1, hi1);
    const int64_t cov = (na > 0 && hi1 >= lo1) ? (int64_t)na * (hi1 - lo1 + 1) : 0;
    const int64_t xx = y * g.m1 + x;
    double v = cov > 0 ? acc / (double)cov : 0.0;
    if (cov == 0 && uncovered) atomicAdd(uncovered, 1ull);
    if (dc && mask[xx]) v = (double)original[xx];
    out[xx] = (T)v;
  }
}

static int grid_blocks(int64_t work, int threads) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int64_t b = ceil_div(work, threads);
  const int64_t cap = (int64_t)sms * 16;
  return (int)(b < 1 ? 1 : (b > cap ? cap : b));
}

int launch_extract(const Grid& grid, const void* tensor, int f64, const uint8_t* mask, int mean_subtract,
                   float* values, uint8_t* obs, float* means, int32_t* counts, cudaStream_t st, int64_t i0,
                   int64_t cnt) {
  const Geo4 g = make_geo4(grid);
  if (cnt < 0) cnt = g.n - i0;
  if (i0 < 0 || i0 + cnt > g.n) { set_error("patch range [%lld, %lld) outside the grid", (long long)i0, (long long)(i0 + cnt)); return PB_ESHAPE; }
  if (grid.rank == 2) {   // tiled 2-D paths (shared-memory windows)
    const Geo2 g2 = make_geo2(grid);
    const size_t w1r = (size_t)(kXW - 1) * g2.s1 + g2.b1;
    const size_t smem_r = w1r * 8 + ((w1r + 1) & ~(size_t)1) * 4 + (size_t)g2.b0 * w1r * ((f64 ? 8 : 4) + 1);
    if (smem_r <= 48 * 1024 && g2.gc1 >= 768) {   // aligned row tiles (wide frames: configs[1] -18 %, [4] -41 %)
      const int tpr = (int)((g2.gc1 + 2 * kXW - 1) / kXW);
      const int64_t rows = (i0 + cnt - 1) / g2.gc1 - i0 / g2.gc1 + 1;
      const int nb2 = (int)std::min<int64_t>(rows * tpr, 148 * 16);
#define PB_X2R(T, B0, B1)                                                                                   \
  k_extract2r<T, B0, B1><<<nb2, kXW, smem_r, st>>>(g2, (const T*)tensor, mask, mean_subtract, values, obs, means, \
                                                   counts, i0, cnt, tpr)
#define PB_X2R_SHAPES(T)                                                              \
  if (g2.b0 == 10 && g2.b1 == 10) PB_X2R(T, 10, 10);                                  \
  else if (g2.b0 == 8 && g2.b1 == 8) PB_X2R(T, 8, 8);                                 \
  else PB_X2R(T, 0, 0)
      if (f64) { PB_X2R_SHAPES(double); } else { PB_X2R_SHAPES(float); }
#undef PB_X2R_SHAPES
#undef PB_X2R
      PB_LAUNCH_CHECK();
      return PB_OK;
    }
    const size_t smem = (size_t)g2.w0 * g2.w1 * ((f64 ? 8 : 4) + 1);
    if (smem <= 48 * 1024) {
      const int64_t ntile = ceil_div(g2.gc0, kXR) * ceil_div(g2.gc1, kXC);
      const int nb2 = (int)std::min<int64_t>(ntile, 148 * 16);
      if (f64)
        k_extract2d<double><<<nb2, kXR * kXC, smem, st>>>(g2, (const double*)tensor, mask, mean_subtract, values, obs,
                                                          means, counts, i0, cnt);
      else
        k_extract2d<float><<<nb2, kXR * kXC, smem, st>>>(g2, (const float*)tensor, mask, mean_subtract, values, obs,
                                                         means, counts, i0, cnt);
      PB_LAUNCH_CHECK();
      return PB_OK;
    }
  }
  const int th = 256;
  const int nb = grid_blocks(cnt, th);
  if (f64)
    k_extract<double><<<nb, th, 0, st>>>(g, (const double*)tensor, mask, mean_subtract, values, obs, means, counts, i0,
                                         cnt);
  else
    k_extract<float><<<nb, th, 0, st>>>(g, (const float*)tensor, mask, mean_subtract, values, obs, means, counts, i0,
                                        cnt);
  PB_LAUNCH_CHECK();
  return PB_OK;
}

int launch_reconstitute(const Grid& grid, const float* est, float est_scale, const float* means, const void* original,
                        const uint8_t* mask, int dc, int f64, void* out, unsigned long long* uncovered,
                        cudaStream_t st) {
  const int th = 256;
  if (grid.rank == 2) {
    const Geo2 g2 = make_geo2(grid);
    if (g2.s1 == 1 && (g2.b1 == 8 || g2.b1 == 10)) {   // staged runs (configs[0..2], [4])
      const void* fn = f64 ? (g2.b1 == 8 ? (const void*)k_ola2s<double, 8> : (const void*)k_ola2s<double, 10>)
                           : (g2.b1 == 8 ? (const void*)k_ola2s<float, 8> : (const void*)k_ola2s<float, 10>);
      int dev = 0, sms = 148, per_sm = 1;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kOW, 0);
      const int64_t ntile = g2.m0 * ((g2.m1 + kOW - 1) / kOW);
      const int nb = (int)std::max<int64_t>(1, std::min<int64_t>(ntile, (int64_t)sms * std::max(per_sm, 1)));
#define PB_OLA2S(T, BB)                                                                                        \
  k_ola2s<T, BB><<<nb, kOW, 0, st>>>(g2, est, est_scale, means, (const T*)original, mask, dc, (T*)out, uncovered)
      if (f64) { if (g2.b1 == 8) PB_OLA2S(double, 8); else PB_OLA2S(double, 10); }
      else { if (g2.b1 == 8) PB_OLA2S(float, 8); else PB_OLA2S(float, 10); }
#undef PB_OLA2S
      PB_LAUNCH_CHECK();
      return PB_OK;
    }
    const int nb2 = grid_blocks(g2.m0 * g2.m1, th);
#define PB_OLA2(T, BB)                                                                                      \
  k_reconstitute2d<T, BB><<<nb2, th, 0, st>>>(g2, est, est_scale, means, (const T*)original, mask, dc, (T*)out, \
                                              uncovered)
    // (a compile-time-width variant that issues a row's loads before the ordered
    // adds measured 2.3x slower at configs[1]; the plain loop is kept)
    if (f64) PB_OLA2(double, 0); else PB_OLA2(float, 0);
#undef PB_OLA2
    PB_LAUNCH_CHECK();
    return PB_OK;
  }
  const Geo4 g = make_geo4(grid);
  const int nb = grid_blocks(g.m, th);
  if (f64)
    k_reconstitute<double><<<nb, th, 0, st>>>(g, est, est_scale, means, (const double*)original, mask, dc,
                                              (double*)out, uncovered);
  else
    k_reconstitute<float><<<nb, th, 0, st>>>(g, est, est_scale, means, (const float*)original, mask, dc,
                                             (float*)out, uncovered);
  PB_LAUNCH_CHECK();
  return PB_OK;
}

int launch_ola_partial(const Grid& grid, const float* est, float est_scale, const float* means, int64_t i0,
                       int64_t cnt, double* acc_out, cudaStream_t st) {
  const Geo4 g = make_geo4(grid);
  k_ola_partial<<<grid_blocks(g.m, 256), 256, 0, st>>>(g, est, est_scale, means, i0, cnt, acc_out);
  PB_LAUNCH_CHECK();
  return PB_OK;
}

int launch_coverage(const Grid& grid, int32_t* out, cudaStream_t st) {
  const Geo4 g = make_geo4(grid);
  k_coverage<<<grid_blocks(g.m, 256), 256, 0, st>>>(g, out);
  PB_LAUNCH_CHECK();
  return PB_OK;
}

}  // namespace pb
