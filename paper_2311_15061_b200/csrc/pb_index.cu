#include <algorithm>
// pb200 — observed-element index of a patch matrix (built once per mask).
//
// The sweep never touches unobserved elements: every conditional of the
// reference sampler sums over Omega_i only (bpfa.py:1-21, _kernels.py:18-109),
// and with 10-25 % sampling the dense (P, N) layout wastes 4-10x of every
// pass.  This kernel set turns the plane-major observed mask into two views of
// the same nnz observed elements:
//
//   CSC-tile order  (the dictionary step's order): patches are cut into tiles
//     of kTile consecutive patches; inside a tile, elements are grouped by
//     patch offset p (column) and sorted by patch.  Per element: e_loc (u16,
//     patch index inside the tile), x_csc (the observed value), and the
//     residual lives in this order.  colptr[t][p] = first element of column p
//     relative to the tile start (rows padded to 16 bytes for bulk copies).
//   CSR order (the code step's order): per patch, its observed offsets in
//     ascending p: csr_p (u16) and csr_pos (u32, the element's CSC position),
//     slots [rowptr[i], rowptr[i] + count[i]).
//
// Both are deterministic (ascending patch, ascending p), built with block-wide
// ballot scans; no atomics except the max count.
#include "pb_index.cuh"

namespace pb {

__global__ void k_tile_totals(const int32_t* __restrict__ counts, int64_t n, int32_t* __restrict__ tile_tot,
                              int32_t* __restrict__ cmax) {
  __shared__ int red[32];
  __shared__ int mx[32];
  const int64_t base = (int64_t)blockIdx.x * kTile;
  int s = 0, m = 0;
  for (int li = threadIdx.x; li < kTile; li += blockDim.x) {
    const int64_t i = base + li;
    if (i < n) {
      const int c = counts[i];
      s += c;
      m = max(m, c);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    s += __shfl_xor_sync(0xffffffffu, s, o);
    m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  }
  if ((threadIdx.x & 31) == 0) { red[threadIdx.x >> 5] = s; mx[threadIdx.x >> 5] = m; }
  __syncthreads();
  if (threadIdx.x == 0) {
    int t = 0, mm = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) { t += red[w]; mm = max(mm, mx[w]); }
    tile_tot[blockIdx.x] = t;
    atomicMax(cmax, mm);
  }
}

// Exclusive scan of the tile totals (one block; ntiles is N/1024).
__global__ void k_tile_scan(const int32_t* __restrict__ tile_tot, int ntiles, int64_t* __restrict__ tile_base) {
  __shared__ int64_t wsum[32];
  __shared__ int64_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int c0 = 0; c0 < ntiles; c0 += blockDim.x) {
    const int t = c0 + threadIdx.x;
    int64_t v = t < ntiles ? tile_tot[t] : 0, x = v;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) wsum[w] = x;
    __syncthreads();
    if (w == 0) {
      int64_t s = lane < (int)(blockDim.x >> 5) ? wsum[lane] : 0, z = s;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int64_t y = __shfl_up_sync(0xffffffffu, z, o);
        if (lane >= o) z += y;
      }
      wsum[lane] = z - s;
    }
    __syncthreads();
    if (t < ntiles) tile_base[t] = carry + wsum[w] + x - v;
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry += wsum[w] + x;
    __syncthreads();
  }
  if (threadIdx.x == 0) tile_base[ntiles] = carry;
}

// Block-wide exclusive scan of small ints (blockDim.x a multiple of 32, <= 1024).
__device__ __forceinline__ int block_excl_scan(int v, int* wsum, int& total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  __syncthreads();
  if (lane == 31) wsum[w] = x;
  __syncthreads();
  if (w == 0) {
    const int s = lane < (int)(blockDim.x >> 5) ? wsum[lane] : 0;
    int z = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, z, o);
      if (lane >= o) z += y;
    }
    wsum[lane] = z - s;
    if (lane == 31) wsum[32] = z;
  }
  __syncthreads();
  total = wsum[32];
  return wsum[w] + x - v;
}

// One block of kFillThreads threads per tile; thread t owns the adjacent local
// patches 2t and 2t+1, so a block-wide exclusive scan of per-thread pair sums
// keeps every column in ascending patch order.
__global__ void __launch_bounds__(kFillThreads) k_tile_fill(
    const uint8_t* __restrict__ obs, const float* __restrict__ values, const int32_t* __restrict__ counts, int64_t n,
    int p, const int64_t* __restrict__ tile_base, int32_t* __restrict__ colptr, uint16_t* __restrict__ e_loc,
    uint32_t* __restrict__ slot_csc, int64_t* __restrict__ rowptr, uint16_t* __restrict__ csr_p,
    uint32_t* __restrict__ csr_pos) {
  static_assert(kTile == 2 * kFillThreads, "two patches per fill thread");
  __shared__ int wsum[33];
  const int t = blockIdx.x;
  const int l0 = 2 * threadIdx.x;
  const int64_t g0 = (int64_t)t * kTile + l0, g1 = g0 + 1;
  const bool live0 = g0 < n, live1 = g1 < n;
  const int64_t tb = tile_base[t];
  int tot;
  const int c0 = live0 ? counts[g0] : 0, c1 = live1 ? counts[g1] : 0;
  const int64_t row0 = tb + block_excl_scan(c0 + c1, wsum, tot);
  const int64_t row1 = row0 + c0;
  if (live0) rowptr[g0] = row0;
  if (live1) rowptr[g1] = row1;
  if (g0 == n - 1) rowptr[n] = row0 + c0;
  if (g1 == n - 1) rowptr[n] = row1 + c1;
  int64_t col = tb;
  int j0 = 0, j1 = 0;
  for (int pe = 0; pe < p; ++pe) {
    const int o0 = (live0 && obs[(int64_t)pe * n + g0]) ? 1 : 0;
    const int o1 = (live1 && obs[(int64_t)pe * n + g1]) ? 1 : 0;
    const int rank = block_excl_scan(o0 + o1, wsum, tot);
    if (threadIdx.x == 0) colptr[(int64_t)t * colptr_pitch(p) + pe] = (int32_t)(col - tb);
    if (o0) {
      const int64_t pos = col + rank;
      e_loc[pos] = (uint16_t)w_row_off(l0);
      slot_csc[pos] = (uint32_t)(row0 + j0);   // CSR slot (ELL transform); values: k_scatter_x
      csr_p[row0 + j0] = (uint16_t)pe;
      csr_pos[row0 + j0] = (uint32_t)pos;
      ++j0;
    }
    if (o1) {
      const int64_t pos = col + rank + o0;
      e_loc[pos] = (uint16_t)w_row_off(l0 + 1);
      slot_csc[pos] = (uint32_t)(row1 + j1);
      csr_p[row1 + j1] = (uint16_t)pe;
      csr_pos[row1 + j1] = (uint32_t)pos;
      ++j1;
    }
    col += tot;
  }
  if (threadIdx.x == 0) colptr[(int64_t)t * colptr_pitch(p) + p] = (int32_t)(col - tb);
}

// Refresh the CSC values for a new frame under a cached mask (live path).
__global__ void k_scatter_x(const float* __restrict__ values, const int32_t* __restrict__ counts,
                            const int64_t* __restrict__ rowptr, const uint16_t* __restrict__ csr_p,
                            const uint32_t* __restrict__ csr_pos, int64_t n, float* __restrict__ x_csc) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = rowptr[i];
    const int c = counts[i];
    for (int j = 0; j < c; ++j) x_csc[csr_pos[r + j]] = values[(int64_t)csr_p[r + j] * n + i];
  }
}

// Live frame under a cached mask, rank 2: the observed values straight from
// the frame into the compact order (csr_p: the patch's observed offsets in
// ascending order; csr_pos: their compact positions), with the observed-only
// mean — no dense (P, N) values / flags written and re-read.  The mean sums in
// ascending offset order, as k_extract2d / k_extract do (bit-identical to
// extraction + k_scatter_x when the extraction would take one of those).
template <int CB1>   // CB1 > 0: patch width known at compile time (offset split by a constant)
__global__ void k_refresh_frame2d(const double* __restrict__ frame, int64_t m1, int64_t gc1, int b1_rt, int s0, int s1,
                                  int mean_subtract, const int32_t* __restrict__ counts,
                                  const int64_t* __restrict__ rowptr, const uint16_t* __restrict__ csr_p,
                                  const uint32_t* __restrict__ csr_pos, int64_t n, float* __restrict__ x_csc,
                                  float* __restrict__ means) {
  const int b1 = CB1 > 0 ? CB1 : b1_rt;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t gy = i / gc1, gx = i - gy * gc1;
    const double* f = frame + gy * s0 * m1 + gx * s1;
    const int64_t r = rowptr[i];
    const int c = counts[i];
    double mean = 0.0;
    if (mean_subtract && c > 0) {
      double sum = 0.0;
      for (int j = 0; j < c; ++j) {
        const int pe = csr_p[r + j];
        const int a = pe / b1;
        sum += f[a * m1 + (pe - a * b1)];
      }
      mean = sum / (double)c;
    }
    means[i] = (float)mean;
    for (int j = 0; j < c; ++j) {
      const int pe = csr_p[r + j];
      const int a = pe / b1;
      x_csc[csr_pos[r + j]] = (float)(f[a * m1 + (pe - a * b1)] - mean);
    }
  }
}

int launch_refresh_frame2d(const PatchIndex& ix, const double* frame, int64_t m1, int64_t gc1, int b1, int s0, int s1,
                           int mean_subtract, const int32_t* counts, float* means, cudaStream_t st) {
  int64_t nb = ceil_div(ix.n, 256);
  if (nb > 148 * 16) nb = 148 * 16;
#define PB_RF(CB)                                                                                               \
  k_refresh_frame2d<CB><<<(unsigned)std::max<int64_t>(nb, 1), 256, 0, st>>>(frame, m1, gc1, b1, s0, s1, mean_subtract, \
                                                                          counts, ix.rowptr, ix.csr_p, ix.csr_pos,      \
                                                                          ix.n, ix.x_csc, means)
  if (b1 == 8) PB_RF(8);
  else if (b1 == 10) PB_RF(10);
  else PB_RF(0);
#undef PB_RF
  PB_LAUNCH_CHECK();
  return PB_OK;
}

int index_bytes(int64_t n, int p, int64_t nnz_upper, size_t* out) {
  const int64_t ntiles = ceil_div(n, kTile);
  size_t b = 0;
  auto a = [&](size_t x) { b += (x + 255) & ~size_t(255); };
  a((size_t)ntiles * 4);              // tile_tot
  a((size_t)(ntiles + 1) * 8);        // tile_base
  a((size_t)ntiles * colptr_pitch(p) * 4);    // colptr
  a((size_t)(n + 1) * 8);             // rowptr
  const int64_t ecap = ell_cap(n, nnz_upper), wcap = wave_cap(n, p, nnz_upper);
  a((size_t)nnz_upper * 2);           // e_loc (CSC)
  a((size_t)ecap * 4);                // x_csc (ELL order)
  a((size_t)nnz_upper * 2);           // csr_p
  a((size_t)nnz_upper * 4);           // csr_pos
  a(64);                              // cmax + misc
  a((size_t)n * 4);                   // outliers: patches above the code-step split
  a((size_t)ntiles * 4);              // outlier counts per tile
  a((size_t)(ntiles + 1) * 8);        // outlier bases per tile
  a((size_t)(p + 2) * 4);             // histogram of observed counts
  a((size_t)ntiles * 4);              // tile_segs
  a((size_t)(ntiles + 1) * 8);        // seg_base
  a((size_t)nnz_upper * 4);           // slot_csc
  a((size_t)ecap * 2);                // e_ell
  a((size_t)ntiles * 4);              // ell_tot
  a((size_t)(ntiles + 1) * 8);        // ell_base
  a((size_t)ntiles * 4);              // wave_tot
  a((size_t)(ntiles + 1) * 8);        // wave_base
  a((size_t)wcap * 4);                // wave_off
  a((size_t)wcap * 2);                // wave_meta
  a((size_t)wcap * 64);               // wave_col
  *out = b;
  return PB_OK;
}

void carve_index(PatchIndex& ix, char* base, int64_t n, int p, int64_t nnz_upper) {
  const int64_t ntiles = ceil_div(n, kTile);
  size_t off = 0;
  auto take = [&](size_t x) { char* r = base + off; off += (x + 255) & ~size_t(255); return r; };
  ix.n = n; ix.p = p; ix.ntiles = (int)ntiles;
  ix.tile_tot = (int32_t*)take((size_t)ntiles * 4);
  ix.tile_base = (int64_t*)take((size_t)(ntiles + 1) * 8);
  ix.colptr = (int32_t*)take((size_t)ntiles * colptr_pitch(p) * 4);
  ix.rowptr = (int64_t*)take((size_t)(n + 1) * 8);
  const int64_t ecap = ell_cap(n, nnz_upper), wcap = wave_cap(n, p, nnz_upper);
  ix.e_loc = (uint16_t*)take((size_t)nnz_upper * 2);
  ix.x_csc = (float*)take((size_t)ecap * 4);
  ix.csr_p = (uint16_t*)take((size_t)nnz_upper * 2);
  ix.csr_pos = (uint32_t*)take((size_t)nnz_upper * 4);
  ix.cmax_dev = (int32_t*)take(64);
  ix.outliers = (int32_t*)take((size_t)n * 4);
  ix.out_tot = (int32_t*)take((size_t)ntiles * 4);
  ix.out_base = (int64_t*)take((size_t)(ntiles + 1) * 8);
  ix.hist = (int32_t*)take((size_t)(p + 2) * 4);
  ix.tile_segs = (int32_t*)take((size_t)ntiles * 4);
  ix.seg_base = (int64_t*)take((size_t)(ntiles + 1) * 8);
  ix.slot_csc = (uint32_t*)take((size_t)nnz_upper * 4);
  ix.e_ell = (uint16_t*)take((size_t)ecap * 2);
  ix.ell_tot = (int32_t*)take((size_t)ntiles * 4);
  ix.ell_base = (int64_t*)take((size_t)(ntiles + 1) * 8);
  ix.wave_tot = (int32_t*)take((size_t)ntiles * 4);
  ix.wave_base = (int64_t*)take((size_t)(ntiles + 1) * 8);
  ix.wave_off = (uint32_t*)take((size_t)wcap * 4);
  ix.wave_meta = (uint16_t*)take((size_t)wcap * 2);
  ix.wave_col = (uint16_t*)take((size_t)wcap * 64);
}

// Column segments of each tile: sum over columns of ceil(len / kSegCountLen).
__global__ void k_tile_segs(const int32_t* __restrict__ colptr, int ntiles, int p, int32_t* __restrict__ segs) {
  const int t = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (t >= ntiles) return;
  const int32_t* cp = colptr + (int64_t)t * colptr_pitch(p);
  int s = 0;
  for (int c = lane; c < p; c += 32) s += (cp[c + 1] - cp[c] + kSegCountLen - 1) / kSegCountLen;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) segs[t] = s;
}


// ---- ELL wave layout (the dictionary step's order) -------------------------
// Per tile, every non-empty column c (n_c elements) is cut into R_c = pow2ceil(
// ceil(n_c / kEllRun)) <= 32 runs of balanced length (<= len_c = ceil(n_c/R_c)).
// Columns are ordered by (R desc, len desc, c) and packed into WAVES of 32 lane
// runs: a column's runs occupy R_c consecutive lanes of one wave, every wave
// holds columns of ONE R (a new wave starts where R changes), and the wave's run
// length Lw is the longest of its runs.  Element j of lane l's run is stored at
// wave_off + j*32 + l (coalesced for a warp walking the wave); positions past a
// run's end are padding (W row kEllZeroRow, value 0).  In the dictionary step a
// lane accumulates its run's Gram / moment sums in registers and the R lanes of
// a column combine them once per wave (transpose reduction); each column sits in
// exactly one wave per tile, so flushes never collide.  Deterministic.
struct EllPlan {
  int nw;          // waves of the tile
  int64_t total;   // ELL positions of the tile
};

__device__ __forceinline__ int ell_runs(int n) {
  if (n <= 0) return 0;
  const int q = (n + kEllRun - 1) / kEllRun;
  int r = 1;
  while (r < q) r <<= 1;
  return r < 32 ? r : 32;
}

// Block-wide plan of tile t in shared memory: s_w / s_l0 per column, s_wlen /
// s_wlg / s_woff per wave.  Needs blockDim.x threads, p <= blockDim.x * 8.
__device__ EllPlan ell_plan(const int32_t* __restrict__ cp, int p, int* s_key, int* s_ord, uint16_t* s_w,
                            uint8_t* s_l0, uint8_t* s_wlen, uint8_t* s_wlg, uint32_t* s_woff) {
  __shared__ EllPlan res;
  for (int c = threadIdx.x; c < p; c += blockDim.x) {
    const int n = cp[c + 1] - cp[c];
    const int R = ell_runs(n);
    int lg = 0;
    while ((1 << lg) < R) ++lg;
    const int len = R ? (n + R - 1) / R : 0;
    s_key[c] = n == 0 ? 0x7FFFFFFF : (((5 - lg) << 16) | (kEllRun * 32 - len));
  }
  __syncthreads();
  for (int c = threadIdx.x; c < p; c += blockDim.x) {
    const int kc = s_key[c];
    int rank = 0;
    for (int d = 0; d < p; ++d) {
      const int kd = s_key[d];
      rank += (kd < kc || (kd == kc && d < c)) ? 1 : 0;
    }
    s_ord[rank] = c;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int lane = 0, w = -1, cur_lg = -1;
    int64_t off = 0;
    for (int i = 0; i < p; ++i) {
      const int c = s_ord[i];
      const int n = cp[c + 1] - cp[c];
      if (n == 0) break;   // empty columns sort last
      const int R = ell_runs(n);
      int lg = 0;
      while ((1 << lg) < R) ++lg;
      const int len = (n + R - 1) / R;
      if (w < 0 || lg != cur_lg || lane + R > 32) {   // open a new wave
        if (w >= 0) off += 32 * (int64_t)s_wlen[w];
        ++w;
        lane = 0;
        cur_lg = lg;
        s_wlen[w] = 0;
        s_wlg[w] = (uint8_t)lg;
        s_woff[w] = (uint32_t)off;
      }
      s_w[c] = (uint16_t)w;
      s_l0[c] = (uint8_t)lane;
      if (len > s_wlen[w]) s_wlen[w] = (uint8_t)len;
      lane += R;
    }
    if (w >= 0) off += 32 * (int64_t)s_wlen[w];
    res.nw = w + 1;
    res.total = off;
  }
  __syncthreads();
  return res;
}

__host__ __device__ constexpr int ell_smem_bytes(int p) { return p * (4 + 4 + 2 + 1) + (p + 8) * (1 + 1 + 4) + 64; }

__global__ void __launch_bounds__(256) k_ell_count(const int32_t* __restrict__ colptr, int p, int32_t* __restrict__ ell_tot,
                                                   int32_t* __restrict__ wave_tot) {
  extern __shared__ __align__(8) unsigned char es[];
  int* s_key = (int*)es;
  int* s_ord = s_key + p;
  uint32_t* s_woff = (uint32_t*)(s_ord + p);
  uint16_t* s_w = (uint16_t*)(s_woff + p + 8);
  uint8_t* s_l0 = (uint8_t*)(s_w + p);
  uint8_t* s_wlen = s_l0 + p;
  uint8_t* s_wlg = s_wlen + p + 8;
  const EllPlan pl = ell_plan(colptr + (int64_t)blockIdx.x * colptr_pitch(p), p, s_key, s_ord, s_w, s_l0, s_wlen,
                              s_wlg, s_woff);
  if (threadIdx.x == 0) {
    ell_tot[blockIdx.x] = (int32_t)pl.total;
    wave_tot[blockIdx.x] = pl.nw;
  }
}

__global__ void __launch_bounds__(256) k_ell_fill(const int64_t* __restrict__ tile_base, const int32_t* __restrict__ colptr,
                                                  int p, const uint16_t* __restrict__ e_loc,
                                                  const uint32_t* __restrict__ slot_csc,
                                                  const int64_t* __restrict__ ell_base, const int64_t* __restrict__ wave_base,
                                                  uint16_t* __restrict__ e_ell, float* __restrict__ x_ell,
                                                  uint32_t* __restrict__ csr_pos, uint32_t* __restrict__ wave_off,
                                                  uint16_t* __restrict__ wave_meta, uint16_t* __restrict__ wave_col) {
  extern __shared__ __align__(8) unsigned char es[];
  int* s_key = (int*)es;
  int* s_ord = s_key + p;
  uint32_t* s_woff = (uint32_t*)(s_ord + p);
  uint16_t* s_w = (uint16_t*)(s_woff + p + 8);
  uint8_t* s_l0 = (uint8_t*)(s_w + p);
  uint8_t* s_wlen = s_l0 + p;
  uint8_t* s_wlg = s_wlen + p + 8;
  const int t = blockIdx.x;
  const int32_t* cp = colptr + (int64_t)t * colptr_pitch(p);
  const EllPlan pl = ell_plan(cp, p, s_key, s_ord, s_w, s_l0, s_wlen, s_wlg, s_woff);
  const int64_t eb = ell_base[t], wb = wave_base[t], tb = tile_base[t];
  // padding everywhere, then the real elements on top
  for (int64_t i = threadIdx.x; i < pl.total; i += blockDim.x) {
    e_ell[eb + i] = (uint16_t)kEllZeroRow;
    x_ell[eb + i] = 0.0f;
  }
  for (int w = threadIdx.x; w < pl.nw; w += blockDim.x) {
    wave_off[wb + w] = s_woff[w];
    wave_meta[wb + w] = (uint16_t)(s_wlen[w] | (s_wlg[w] << 8));
  }
  for (int i = threadIdx.x; i < pl.nw * 32; i += blockDim.x) wave_col[(wb + i / 32) * 32 + (i & 31)] = 0xFFFFu;
  __syncthreads();
  for (int c = threadIdx.x; c < p; c += blockDim.x) {
    const int n = cp[c + 1] - cp[c];
    if (!n) continue;
    const int R = ell_runs(n);
    for (int r = 0; r < R; ++r) wave_col[(wb + s_w[c]) * 32 + s_l0[c] + r] = (uint16_t)c;
  }
  // elements, bank-spread: a column's elements form a sequence t = 0..n-1 with
  // element t in run t % R at step t / R (lane lane0 + t % R).  Rows land on one
  // of 8 shared-memory bank quads ((e >> 4) & 7); sequence slot t asks for quad
  // (t + lane0) & 7 — at every step the 8 lanes of a quarter-warp then ask for 8
  // different quads — and takes the next unused element of that quad, else of
  // the quad with the most elements left.  One thread per column; deterministic.
  for (int c = threadIdx.x; c < p; c += blockDim.x) {
    const int n = cp[c + 1] - cp[c];
    if (!n) continue;
    const int R = ell_runs(n), l0 = s_l0[c];
    const int64_t cb = tb + cp[c];
    const int64_t wpos = eb + s_woff[s_w[c]] + l0;
    int left[8], cur[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) { left[q] = 0; cur[q] = 0; }
    for (int i = 0; i < n; ++i) ++left[(e_loc[cb + i] >> 4) & 7];
    for (int t = 0; t < n; ++t) {
      int q = (t + l0) & 7;
      if (!left[q]) {
        int best = 0;
#pragma unroll
        for (int b = 1; b < 8; ++b)
          if (left[b] > left[best]) best = b;
        q = best;
      }
      int i = cur[q];
      while (((e_loc[cb + i] >> 4) & 7) != q) ++i;
      cur[q] = i + 1;
      --left[q];
      const int64_t pos = wpos + (int64_t)(t / R) * 32 + (t % R);
      e_ell[pos] = e_loc[cb + i];
      csr_pos[slot_csc[cb + i]] = (uint32_t)pos;
    }
  }
}

// Histogram of the per-patch observed counts (0..p): shared-memory bins per block.
__global__ void k_count_hist(const int32_t* __restrict__ counts, int64_t n, int p, int32_t* __restrict__ hist) {
  extern __shared__ int bins[];
  for (int b = threadIdx.x; b <= p; b += blockDim.x) bins[b] = 0;
  __syncthreads();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(&bins[min(max(counts[i], 0), p)], 1);
  __syncthreads();
  for (int b = threadIdx.x; b <= p; b += blockDim.x)
    if (bins[b]) atomicAdd(&hist[b], bins[b]);
}

// Outliers (count > split) per tile, then their ids in ascending order.
__global__ void k_outlier_totals(const int32_t* __restrict__ counts, int64_t n, int split, int32_t* __restrict__ tot) {
  __shared__ int red[32];
  const int64_t base = (int64_t)blockIdx.x * kTile;
  int s = 0;
  for (int li = threadIdx.x; li < kTile; li += blockDim.x) {
    const int64_t i = base + li;
    s += (i < n && counts[i] > split) ? 1 : 0;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    int t = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    tot[blockIdx.x] = t;
  }
}

__global__ void __launch_bounds__(kTile) k_outlier_fill(const int32_t* __restrict__ counts, int64_t n, int split,
                                                        const int64_t* __restrict__ out_base,
                                                        int32_t* __restrict__ outliers) {
  __shared__ int wsum[33];   // block_excl_scan writes the total at [32]
  const int64_t i = (int64_t)blockIdx.x * kTile + threadIdx.x;
  const int f = (i < n && counts[i] > split) ? 1 : 0;
  int tot = 0;
  const int rank = block_excl_scan(f, wsum, tot);
  if (f) outliers[out_base[blockIdx.x] + rank] = (int32_t)i;
}

int launch_count_hist(const PatchIndex& ix, const int32_t* counts, cudaStream_t st) {
  PB_CUDA_TRY(cudaMemsetAsync(ix.hist, 0, (size_t)(ix.p + 2) * 4, st));
  int64_t nb = ceil_div(ix.n, 256);
  if (nb > 1184) nb = 1184;
  k_count_hist<<<(unsigned)(nb < 1 ? 1 : nb), 256, (size_t)(ix.p + 1) * 4, st>>>(counts, ix.n, ix.p, ix.hist);
  PB_LAUNCH_CHECK();
  return PB_OK;
}

int launch_outliers(const PatchIndex& ix, const int32_t* counts, int split, cudaStream_t st) {
  k_outlier_totals<<<ix.ntiles, 256, 0, st>>>(counts, ix.n, split, ix.out_tot);
  k_tile_scan<<<1, 1024, 0, st>>>(ix.out_tot, ix.ntiles, ix.out_base);
  k_outlier_fill<<<ix.ntiles, kTile, 0, st>>>(counts, ix.n, split, ix.out_base, ix.outliers);
  PB_LAUNCH_CHECK();
  return PB_OK;
}

int launch_build_index(PatchIndex& ix, const uint8_t* obs, const float* values, const int32_t* counts,
                       cudaStream_t st) {
  PB_CUDA_TRY(cudaMemsetAsync(ix.cmax_dev, 0, 4, st));
  k_tile_totals<<<ix.ntiles, 256, 0, st>>>(counts, ix.n, ix.tile_tot, ix.cmax_dev);
  k_tile_scan<<<1, 1024, 0, st>>>(ix.tile_tot, ix.ntiles, ix.tile_base);
  k_tile_fill<<<ix.ntiles, kFillThreads, 0, st>>>(obs, values, counts, ix.n, ix.p, ix.tile_base, ix.colptr, ix.e_loc,
                                           ix.slot_csc, ix.rowptr, ix.csr_p, ix.csr_pos);
  // the ELL wave layout (the dictionary step's order): plan, prefix, fill
  const size_t esm = ell_smem_bytes(ix.p);
  if (esm > 48 * 1024) {
    PB_CUDA_TRY(cudaFuncSetAttribute(k_ell_count, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)esm));
    PB_CUDA_TRY(cudaFuncSetAttribute(k_ell_fill, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)esm));
  }
  k_ell_count<<<ix.ntiles, 256, esm, st>>>(ix.colptr, ix.p, ix.ell_tot, ix.wave_tot);
  k_tile_scan<<<1, 1024, 0, st>>>(ix.ell_tot, ix.ntiles, ix.ell_base);
  k_tile_scan<<<1, 1024, 0, st>>>(ix.wave_tot, ix.ntiles, ix.wave_base);
  k_ell_fill<<<ix.ntiles, 256, esm, st>>>(ix.tile_base, ix.colptr, ix.p, ix.e_loc, ix.slot_csc, ix.ell_base,
                                          ix.wave_base, ix.e_ell, ix.x_csc, ix.csr_pos, ix.wave_off, ix.wave_meta,
                                          ix.wave_col);
  // the observed values into the ELL order
  k_scatter_x<<<(unsigned)ceil_div(ix.n, 256), 256, 0, st>>>(values, counts, ix.rowptr, ix.csr_p, ix.csr_pos, ix.n,
                                                             ix.x_csc);
  k_tile_segs<<<(unsigned)ceil_div(ix.ntiles, 8), 256, 0, st>>>(ix.colptr, ix.ntiles, ix.p, ix.tile_segs);
  k_tile_scan<<<1, 1024, 0, st>>>(ix.tile_segs, ix.ntiles, ix.seg_base);
  PB_LAUNCH_CHECK();
  return PB_OK;
}

int launch_scatter_x(const PatchIndex& ix, const float* values, const int32_t* counts, cudaStream_t st) {
  k_scatter_x<<<(unsigned)ceil_div(ix.n, 256), 256, 0, st>>>(values, counts, ix.rowptr, ix.csr_p, ix.csr_pos, ix.n,
                                                             ix.x_csc);
  PB_LAUNCH_CHECK();
  return PB_OK;
}

}  // namespace pb
