// pb200 — device-resident live-path tail:
//
//  k_live_finish     after the overlap-add of a live frame: data consistency
//                    (patches.py:218-229), the residual map (recon − prev)²
//                    that drives adaptive sampling (pipeline.py:265-269, on the
//                    pre-consistency reconstruction), the previous-reconstruction
//                    update, and the uint8 wire panels of the reconstruction and
//                    of the masked input (server.py:46-53: round(clip(x,0,1)·255),
//                    rank-3 tensors show slice 0) — one pass over the frame.
//  adaptive mask     sampling.py:184-207 on device: the exploit set is the top
//                    round(f·budget) residuals, ties by lowest flat index (the
//                    first n of the reference's argsort(-r, kind="stable")); the
//                    explore set is drawn uniformly without replacement from the
//                    rest as the n smallest Philox keys (device stream, keyed by
//                    seed and frame index; not numpy's Generator.choice stream).
//                    Both are a radix SELECT of the n largest 64-bit keys
//                    (pb_select.cu), not a sort of all m (key, index) pairs.
#include "pb_live.cuh"

namespace pb {

__device__ __forceinline__ uint8_t quantize_u8(double x) {
  // np.round(np.clip(x, 0, 1) * 255): round half to even
  return (uint8_t)rint(fmin(fmax(x, 0.0), 1.0) * 255.0);
}

__global__ void __launch_bounds__(256) k_live_finish(LiveFinishArgs a) {
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < a.m; x += (int64_t)gridDim.x * blockDim.x) {
    const double r = a.recon[x];
    const bool obs = a.mask[x] != 0;
    const double f = a.frame[x];
    const double out = (a.dc && obs) ? f : r;
    a.out[x] = out;
    if (a.resid) {
      const double dlt = a.have_prev ? r - a.prev[x] : 0.0;
      a.resid[x] = dlt * dlt;
      a.prev[x] = r;
    }
    if (a.panel || a.masked) {
      // panel pixel (y, x) of a rank-3 (H, W, C) tensor is element (y, x, 0)
      if (a.panel_stride == 1 || x % a.panel_stride == 0) {
        const int64_t px = x / a.panel_stride;
        if (a.panel) a.panel[px] = quantize_u8(out);
        if (a.masked) a.masked[px] = quantize_u8(obs ? f : 0.0);
      }
    }
  }
}

int launch_live_finish(const LiveFinishArgs& a, cudaStream_t st) {
  const int th = 256;
  int64_t nb = (a.m + th - 1) / th;
  if (nb > 148 * 16) nb = 148 * 16;
  if (nb < 1) nb = 1;
  k_live_finish<<<(unsigned)nb, th, 0, st>>>(a);
  PB_LAUNCH_CHECK();
  return PB_OK;
}

// --- adaptive-residual mask ------------------------------------------------
__global__ void k_adaptive_check(const double* __restrict__ r, int64_t m, unsigned* __restrict__ flags) {
  // flags[0]: any residual > 0, flags[1]: any residual < 0 or NaN
  unsigned any_pos = 0, bad = 0;
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < m; x += (int64_t)gridDim.x * blockDim.x) {
    const double v = r[x];
    any_pos |= v > 0.0;
    bad |= !(v >= 0.0);
  }
  any_pos = __any_sync(0xffffffffu, any_pos);
  bad = __any_sync(0xffffffffu, bad);
  if ((threadIdx.x & 31) == 0) {
    if (any_pos) atomicOr(flags, 1u);
    if (bad) atomicOr(flags + 1, 1u);
  }
}

// Exploit keys: the residual's bit pattern (monotone for non-negative
// doubles; -0.0 and +0.0 tie as 0).
__global__ void k_resid_keys(const double* __restrict__ r, int64_t m, uint64_t* __restrict__ keys) {
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < m; x += (int64_t)gridDim.x * blockDim.x) {
    const double v = r[x];
    keys[x] = v > 0.0 ? (uint64_t)__double_as_longlong(v) : 0ull;
  }
}

// Explore keys: a 63-bit uniform u per free element, stored as ~u so that the
// n LARGEST stored keys are the n smallest u (ties by index, as a stable
// ascending sort); taken elements store 0 and are never chosen.
__global__ void k_explore_keys(const uint8_t* __restrict__ taken, int64_t m, uint32_t k0, uint32_t k1,
                               uint64_t frame_index, uint64_t* __restrict__ keys) {
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < m; x += (int64_t)gridDim.x * blockDim.x) {
    if (taken[x]) {
      keys[x] = 0ull;
    } else {
      const u32x4 rr = philox4x32_10(u32x4{(uint32_t)x, (uint32_t)(x >> 32), (uint32_t)frame_index,
                                           ((uint32_t)(frame_index >> 32) & 0xFFFFFFu) | (kDomMask << 24)},
                                     k0, k1);
      keys[x] = ~(((uint64_t)(rr.x >> 1) << 32) | rr.y);  // u < 2^63: ~u >= 2^63 > a taken element's 0
    }
  }
}

static unsigned grid_for(int64_t m) {
  int64_t nb = (m + 255) / 256;
  if (nb > 148 * 16) nb = 148 * 16;
  return (unsigned)(nb < 1 ? 1 : nb);
}

int adaptive_mask(const double* resid, int64_t m, int64_t budget, int64_t n_exploit, uint32_t k0, uint32_t k1,
                  uint64_t frame_index, uint8_t* mask, int* status, cudaStream_t st) {
  *status = 0;
  if (m <= 0) return PB_OK;
  // scratch: flags, keys, selection scratch
  char* buf = nullptr;
  const size_t keys_off = 256, sel_off = keys_off + ((size_t)m * 8 + 255) / 256 * 256;
  if (cudaMallocAsync((void**)&buf, sel_off + select_scratch_bytes(m), st) != cudaSuccess) {
    set_error("adaptive mask: scratch allocation failed");
    return PB_ECUDA;
  }
  unsigned* flags = (unsigned*)buf;
  uint64_t* keys = (uint64_t*)(buf + keys_off);
  void* sel = buf + sel_off;
  int rc = PB_OK;
  unsigned hflags[2] = {0, 0};
  cudaMemsetAsync(flags, 0, 8, st);
  k_adaptive_check<<<grid_for(m), 256, 0, st>>>(resid, m, flags);
  cudaMemcpyAsync(hflags, flags, 8, cudaMemcpyDeviceToHost, st);
  if (cudaStreamSynchronize(st) != cudaSuccess) { set_error("adaptive mask: check failed"); rc = PB_ECUDA; }
  else if (hflags[1]) { set_error("residual map must be non-negative and finite"); rc = PB_EVALUE; }
  if (!rc) {
    cudaMemsetAsync(mask, 0, (size_t)m, st);
    if (!hflags[0]) n_exploit = 0;  // all-zero residual: uniform sampling (status 1)
    *status = hflags[0] ? 0 : 1;
    if (n_exploit > 0) {
      k_resid_keys<<<grid_for(m), 256, 0, st>>>(resid, m, keys);
      rc = select_top(keys, m, n_exploit, sel, mask, nullptr, st);
    }
    const int64_t n_explore = budget - n_exploit;
    if (!rc && n_explore > 0) {
      k_explore_keys<<<grid_for(m), 256, 0, st>>>(mask, m, k0, k1, frame_index, keys);
      rc = select_top(keys, m, n_explore, sel, mask, nullptr, st);
    }
    if (!rc && cudaGetLastError() != cudaSuccess) { set_error("adaptive mask: kernel launch failed"); rc = PB_ECUDA; }
  }
  cudaFreeAsync(buf, st);
  return rc;
}

// --- dictionary atlas (server.py:84-120) -----------------------------------
// Atoms tiled into a ceil(sqrt(K)) grid, highest activation probability first
// (ties by atom index), each min-max normalised on its own (constant atoms at
// 0.5), 1-pixel mid-grey separators and empty cells.  One CTA; the order is a
// rank count over pi (K <= a few thousand).
__global__ void k_atlas(const float* __restrict__ atoms, const double* __restrict__ pi, int k, int b0, int b1,
                        int inner, int p, int grid, int64_t h, int64_t w, double* __restrict__ canvas,
                        uint8_t* __restrict__ canvas_u8) {
  extern __shared__ int slot_atom[];   // [grid*grid]: atom shown in each slot, -1 = empty
  float* lo = (float*)(slot_atom + grid * grid);
  float* hi = lo + k;
  for (int s = threadIdx.x; s < grid * grid; s += blockDim.x) slot_atom[s] = -1;
  __syncthreads();
  for (int a = threadIdx.x; a < k; a += blockDim.x) {
    const double pa = pi[a];
    int rank = 0;   // stable argsort of -pi
    for (int b = 0; b < k; ++b) {
      const double pb = pi[b];
      rank += (pb > pa) || (pb == pa && b < a);
    }
    slot_atom[rank] = a;
    float mn = INFINITY, mx = -INFINITY;
    for (int y = 0; y < b0; ++y)
      for (int x = 0; x < b1; ++x) {
        const float v = atoms[(int64_t)a * p + (int64_t)(y * b1 + x) * inner];
        mn = fminf(mn, v);
        mx = fmaxf(mx, v);
      }
    lo[a] = mn;
    hi[a] = mx;
  }
  __syncthreads();
  for (int64_t t = threadIdx.x; t < h * w; t += blockDim.x) {
    const int64_t y = t / w, x = t - y * w;
    double v = 0.5;
    const int64_t r = y / (b0 + 1), c = x / (b1 + 1);
    const int ty = (int)(y - r * (b0 + 1)), tx = (int)(x - c * (b1 + 1));
    if (ty < b0 && tx < b1) {
      const int a = slot_atom[r * grid + c];
      if (a >= 0) {
        const double span = (double)hi[a] - (double)lo[a];
        const double av = atoms[(int64_t)a * p + (int64_t)(ty * b1 + tx) * inner];
        v = span == 0.0 ? 0.5 : (av - (double)lo[a]) / span;
      }
    }
    if (canvas) canvas[t] = v;
    if (canvas_u8) canvas_u8[t] = quantize_u8(v);
  }
}

int atlas_geometry(int k, int rank, const int32_t* shape, int& b0, int& b1, int& inner, int& grid, int64_t& h,
                   int64_t& w) {
  if (k < 1) { set_error("atlas needs at least one atom"); return PB_EVALUE; }
  if (rank == 1) { b0 = 1; b1 = shape[0]; inner = 1; }
  else if (rank == 2) { b0 = shape[0]; b1 = shape[1]; inner = 1; }
  else if (rank == 3) { b0 = shape[0]; b1 = shape[1]; inner = shape[2]; }   // slice 0 of the last axis
  else { set_error("cannot render atlas for patch rank %d", rank); return PB_EVALUE; }
  grid = (int)ceil(sqrt((double)k));
  while ((int64_t)grid * grid < k) ++grid;
  while (grid > 1 && (int64_t)(grid - 1) * (grid - 1) >= k) --grid;
  h = (int64_t)grid * b0 + grid - 1;
  w = (int64_t)grid * b1 + grid - 1;
  return PB_OK;
}

int launch_atlas(const float* atoms, const double* pi, int k, int rank, const int32_t* shape, double* canvas,
                 uint8_t* canvas_u8, cudaStream_t st) {
  int b0, b1, inner, grid;
  int64_t h, w;
  int rc = atlas_geometry(k, rank, shape, b0, b1, inner, grid, h, w);
  if (rc) return rc;
  int p = 1;
  for (int d = 0; d < rank; ++d) p *= shape[d];
  const size_t smem = (size_t)grid * grid * 4 + (size_t)k * 8;
  if (smem > 200 * 1024) { set_error("too many atoms for the atlas (%d)", k); return PB_EUNSUPPORTED; }
  PB_CUDA_TRY(cudaFuncSetAttribute(k_atlas, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  k_atlas<<<1, 1024, smem, st>>>(atoms, pi, k, b0, b1, inner, p, grid, h, w, canvas, canvas_u8);
  PB_LAUNCH_CHECK();
  return PB_OK;
}

}  // namespace pb

namespace pb {

// ---- data-mode dictionary seeding (bpfa.py:126-134) ------------------------
// order = argsort(-counts, kind="stable")[:K]: the K largest counts (ties by
// patch index) by radix select (pb_select.cu), then ONE CTA ranks those K by
// (count desc, index asc); atom j <- patch order[j], unit-normalized (norm in
// f64), zero-norm candidates keep their prior atom; atoms past min(K, N) too.
__global__ void k_seed_keys(const int32_t* counts, int64_t n, uint64_t* keys) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    keys[i] = (uint64_t)(uint32_t)counts[i];
}

__global__ void __launch_bounds__(1024) k_seed_order(const int32_t* __restrict__ sel, int take,
                                                     const int32_t* __restrict__ counts, int32_t* __restrict__ order) {
  for (int a = threadIdx.x; a < take; a += blockDim.x) {
    const int32_t ia = sel[a];
    const int32_t ca = counts[ia];
    int rank = 0;
    for (int b = 0; b < take; ++b) {
      const int32_t ib = sel[b];
      const int32_t cb = counts[ib];
      rank += (cb > ca || (cb == ca && ib < ia)) ? 1 : 0;
    }
    order[rank] = ia;
  }
}

__global__ void __launch_bounds__(128) k_data_atoms(const float* values_pn, int64_t n, int p, const int32_t* order,
                                                    float* atoms) {
  __shared__ double part[4];
  const int64_t i = order[blockIdx.x];
  double ss = 0.0;
  for (int q = threadIdx.x; q < p; q += blockDim.x) {
    const double v = values_pn[(int64_t)q * n + i];
    ss += v * v;
  }
  for (int o = 16; o; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = ss;
  __syncthreads();
  const double nrm = sqrt(part[0] + part[1] + part[2] + part[3]);
  if (nrm > 0.0)
    for (int q = threadIdx.x; q < p; q += blockDim.x)
      atoms[(int64_t)blockIdx.x * p + q] = (float)((double)values_pn[(int64_t)q * n + i] / nrm);
}

int launch_data_atoms(const float* values_pn, const int32_t* counts, int64_t n, int p, int k, float* atoms,
                      cudaStream_t st) {
  (void)p;
  if (n < 1 || k < 1) return PB_OK;
  if (n >= ((int64_t)1 << 31)) { set_error("data-mode seeding supports < 2^31 patches"); return PB_EUNSUPPORTED; }
  const int take = (int)(k < n ? k : n);
  const size_t al = 256;
  const size_t keys_b = ((size_t)n * 8 + al - 1) / al * al, list_b = ((size_t)take * 4 + al - 1) / al * al;
  char* buf = nullptr;
  PB_CUDA_TRY(cudaMallocAsync((void**)&buf, keys_b + 2 * list_b + select_scratch_bytes(n), st));
  uint64_t* keys = (uint64_t*)buf;
  int32_t* sel = (int32_t*)(buf + keys_b);
  int32_t* order = (int32_t*)(buf + keys_b + list_b);
  void* scratch = buf + keys_b + 2 * list_b;
  int64_t g = (n + 255) / 256;
  if (g > 148 * 8) g = 148 * 8;
  k_seed_keys<<<(unsigned)g, 256, 0, st>>>(counts, n, keys);
  int rc = select_top(keys, n, take, scratch, nullptr, sel, st);
  if (!rc) {
    k_seed_order<<<1, 1024, 0, st>>>(sel, take, counts, order);
    k_data_atoms<<<take, 128, 0, st>>>(values_pn, n, p, order, atoms);
    if (cudaGetLastError() != cudaSuccess) { set_error("k_data_atoms launch failed"); rc = PB_ECUDA; }
  }
  cudaFreeAsync(buf, st);
  return rc;
}

}  // namespace pb
