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
    float* __restrict__ x_csc, int64_t* __restrict__ rowptr, uint16_t* __restrict__ csr_p,
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
      ((uint32_t*)x_csc)[pos] = (uint32_t)(row0 + j0);   // CSR slot (k_csc_spread); values: k_scatter_x
      csr_p[row0 + j0] = (uint16_t)pe;
      csr_pos[row0 + j0] = (uint32_t)pos;
      ++j0;
    }
    if (o1) {
      const int64_t pos = col + rank + o0;
      e_loc[pos] = (uint16_t)w_row_off(l0 + 1);
      ((uint32_t*)x_csc)[pos] = (uint32_t)(row1 + j1);
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

int index_bytes(int64_t n, int p, int64_t nnz_upper, size_t* out) {
  const int64_t ntiles = ceil_div(n, kTile);
  size_t b = 0;
  auto a = [&](size_t x) { b += (x + 255) & ~size_t(255); };
  a((size_t)ntiles * 4);              // tile_tot
  a((size_t)(ntiles + 1) * 8);        // tile_base
  a((size_t)ntiles * colptr_pitch(p) * 4);    // colptr
  a((size_t)(n + 1) * 8);             // rowptr
  a((size_t)nnz_upper * 2);           // e_loc
  a((size_t)nnz_upper * 4);           // x_csc
  a((size_t)nnz_upper * 2);           // csr_p
  a((size_t)nnz_upper * 4);           // csr_pos
  a(64);                              // cmax + misc
  a((size_t)n * 4);                   // outliers: patches above the code-step split
  a((size_t)ntiles * 4);              // outlier counts per tile
  a((size_t)(ntiles + 1) * 8);        // outlier bases per tile
  a((size_t)(p + 2) * 4);             // histogram of observed counts
  a((size_t)ntiles * 4);              // tile_segs
  a((size_t)(ntiles + 1) * 8);        // seg_base
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
  ix.e_loc = (uint16_t*)take((size_t)nnz_upper * 2);
  ix.x_csc = (float*)take((size_t)nnz_upper * 4);
  ix.csr_p = (uint16_t*)take((size_t)nnz_upper * 2);
  ix.csr_pos = (uint32_t*)take((size_t)nnz_upper * 4);
  ix.cmax_dev = (int32_t*)take(64);
  ix.outliers = (int32_t*)take((size_t)n * 4);
  ix.out_tot = (int32_t*)take((size_t)ntiles * 4);
  ix.out_base = (int64_t*)take((size_t)(ntiles + 1) * 8);
  ix.hist = (int32_t*)take((size_t)(p + 2) * 4);
  ix.tile_segs = (int32_t*)take((size_t)ntiles * 4);
  ix.seg_base = (int64_t*)take((size_t)(ntiles + 1) * 8);
}

// Bank spreading of the CSC order (after k_tile_fill, before k_scatter_x).
// The dictionary step's lanes gather each element's W row from shared memory
// with 16-byte loads whose quarter-warps are 8 CONSECUTIVE elements of a column
// run; rows land on one of 8 bank quads ((e_loc >> 4) & 7), so a random order
// costs ~2.2x the ideal wavefronts.  One warp per (tile, column) ranks the
// elements inside their quad (warp ballots) and orders the run by relative
// position inside the quad (a proportional interleave: each group of 8 repeats
// a quad only as often as the quad counts force); runs longer than 128 read the
// quad-sorted run column-major out of 8 rows instead (linear cost).  The fill left each element's
// CSR slot in x_csc, so csr_pos is repointed without searching; the values are
// scattered afterwards.  Deterministic.
constexpr int kSpreadWarps = 8;
__global__ void __launch_bounds__(kSpreadWarps * 32) k_csc_spread(const int64_t* __restrict__ tile_base,
                                                                  const int32_t* __restrict__ colptr, int ntiles, int p,
                                                                  uint16_t* __restrict__ e_loc,
                                                                  const uint32_t* __restrict__ slot_of,
                                                                  uint32_t* __restrict__ csr_pos) {
  __shared__ uint16_t s_e[kSpreadWarps][kTile];
  __shared__ uint16_t s_rq[kSpreadWarps][kTile];   // rank inside the quad << 3 | quad
  __shared__ int s_cnt[kSpreadWarps][8];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t job = (int64_t)blockIdx.x * kSpreadWarps + w;
  if (job >= (int64_t)ntiles * p) return;
  const int t = (int)(job / p), pe = (int)(job - (int64_t)t * p);
  const int32_t* cp = colptr + (int64_t)t * colptr_pitch(p);
  const int64_t base = tile_base[t] + cp[pe];
  const int len = cp[pe + 1] - cp[pe];
  if (len <= 8) return;
  int cnt[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) cnt[q] = 0;
  for (int i0 = 0; i0 < len; i0 += 32) {   // warp-uniform trip count: full-mask ballots
    const int i = i0 + lane;
    const bool live = i < len;
    const uint16_t e = live ? e_loc[base + i] : 0;
    if (live) s_e[w][i] = e;
    const int q = (e >> 4) & 7;
#pragma unroll
    for (int b = 0; b < 8; ++b) cnt[b] += __popc(__ballot_sync(0xffffffffu, live && q == b));
  }
  __syncwarp();
  int seen[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) seen[q] = 0;
  for (int i0 = 0; i0 < len; i0 += 32) {
    const int i = i0 + lane;
    const bool live = i < len;
    const uint16_t e = live ? s_e[w][i] : 0;
    const int q = (e >> 4) & 7;
    int r = 0;
#pragma unroll
    for (int b = 0; b < 8; ++b) {
      const unsigned m = __ballot_sync(0xffffffffu, live && q == b);
      if (q == b) r = seen[b] + __popc(m & ((1u << lane) - 1u));   // stable rank inside the quad
      seen[b] += __popc(m);
    }
    if (live) s_rq[w][i] = (uint16_t)((r << 3) | q);
  }
  __syncwarp();
  if (lane < 8) {
#pragma unroll
    for (int b = 0; b < 8; ++b)
      if (lane == b) s_cnt[w][b] = cnt[b];
  }
  __syncwarp();
  // proportional interleave: element (q, r) sits at the relative position
  // (r + 1/2) / cnt_q of its quad; the new order sorts those keys (ties by
  // quad), so every quad is spread evenly and each group of 8 repeats a quad
  // only as often as the counts force
  for (int i = lane; i < len; i += 32) {
    const int rq = s_rq[w][i], q = rq & 7, r2 = 2 * (rq >> 3) + 1;
    const int cq = s_cnt[w][q];
    int j = 0;
    if (len <= 128) {   // O(len^2) ranking: short runs
      for (int k = 0; k < len; ++k) {
        const int rk = s_rq[w][k], qk = rk & 7, rk2 = 2 * (rk >> 3) + 1;
        const int lhs = rk2 * cq, rhs = r2 * s_cnt[w][qk];   // key_k < key_i  <=>  rk2 / cnt_qk < r2 / cq
        j += (lhs < rhs || (lhs == rhs && qk < q)) ? 1 : 0;
      }
    } else {            // long runs: the quad-sorted run read column-major out of 8 rows
      int st = 0;
      for (int b = 0; b < q; ++b) st += s_cnt[w][b];
      const int sidx = st + (rq >> 3);
      const int c = (len + 7) >> 3, nf = len / c, rem = len - nf * c;
      const int row = sidx / c, col = sidx - row * c;
      j = col * nf + min(col, rem) + row;
    }
    {
      const uint16_t e = s_e[w][i];
      e_loc[base + j] = e;
      csr_pos[slot_of[base + i]] = (uint32_t)(base + j);
    }
  }
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
                                           ix.x_csc, ix.rowptr, ix.csr_p, ix.csr_pos);
  {
    const int spread = !PB_TUNE_INT("PB_INDEX_NO_SPREAD", 0);   // 0: ascending patch order inside columns (A/B)
    if (spread)
      k_csc_spread<<<(unsigned)ceil_div((int64_t)ix.ntiles * ix.p, kSpreadWarps), kSpreadWarps * 32, 0, st>>>(
          ix.tile_base, ix.colptr, ix.ntiles, ix.p, ix.e_loc, (const uint32_t*)ix.x_csc, ix.csr_pos);
  }
  // the observed values into the (final) CSC order
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
