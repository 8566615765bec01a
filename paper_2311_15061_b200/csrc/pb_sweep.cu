// pb200 — dense helper kernels of the Gibbs sweep on sm_100a.
//
// The epoch itself runs on the observed-element ("compact") kernels of
// pb_compact.cu.  This file holds the dense (P,N) kernels behind the fine-grained
// seam of the C ABI (one per reference _kernels.* function, _kernels.py:18-145),
// the dense compose used for overlap-add (every p, not only observed), the
// epoch statistics finish, and the device pi/gamma draws of philox mode
// (bpfa.py:313-342).
#include <math.h>

#include "pb_sweep.cuh"
#include "pb_compose_tc.cuh"

namespace pb {



// ---------------------------------------------------------------------------
// residual / compose: one G-lane group per patch, VPT register elements per lane.
// Element p = j*G + g of patch i lives in lane g, slot j.

template <int VPT, int G, bool RESID>
__global__ void __launch_bounds__(256) k_accumulate_atoms(
    const float* __restrict__ values, const uint8_t* __restrict__ obs, const uint8_t* __restrict__ usage,
    const float* __restrict__ weights, const float* __restrict__ atoms, float* __restrict__ out, int64_t n, int p,
    int k_len, int kc, int accumulate, int64_t ld) {
  extern __shared__ float ds[];  // kc * p
  const int g = threadIdx.x % G;
  const int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / G;
  const bool live = i < n;
  float acc[VPT];
  uint64_t ob = 0;
#pragma unroll
  for (int j = 0; j < VPT; ++j) {
    const int pe = j * G + g;
    acc[j] = 0.0f;
    if (live && pe < p) {
      if (RESID) {
        acc[j] = values[(int64_t)pe * n + i];
        if (obs[(int64_t)pe * n + i]) ob |= 1ull << j;
      } else if (accumulate) {
        acc[j] = out[(int64_t)pe * n + i];
      }
    }
  }
  constexpr int PP = VPT * G;  // shared-memory row pitch, zero padded past p
  for (int k0 = 0; k0 < k_len; k0 += kc) {
    const int kn = min(kc, k_len - k0);
    __syncthreads();
    for (int t = threadIdx.x; t < kn * PP; t += blockDim.x) {
      const int kk = t / PP, pe = t - kk * PP;
      ds[t] = pe < p ? atoms[(int64_t)(k0 + kk) * p + pe] : 0.0f;
    }
    __syncthreads();
    const int64_t ic = live ? i : 0;
    for (int kb = 0; kb < kn; kb += 8) {
      // the 8 atoms' (usage, weight) loads are independent: issue them all first
      float wv[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int64_t zi = (int64_t)(k0 + min(kb + q, kn - 1)) * ld + ic;
        const uint8_t z = usage[zi];
        const float w = weights[zi];
        wv[q] = (live && kb + q < kn && z) ? (RESID ? -w : w) : 0.0f;
      }
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        if (!__any_sync(0xffffffffu, wv[q] != 0.0f)) continue;
        const float* d = ds + (kb + q) * PP + g;
#pragma unroll
        for (int j = 0; j < VPT; ++j) acc[j] = fmaf(wv[q], d[j * G], acc[j]);
      }
    }
  }
  if (!live) return;
  asm volatile("" ::: "memory");
  float* o = out + i + (int64_t)g * n;
  const int64_t step = (int64_t)G * n;
#pragma unroll
  for (int j = 0; j < VPT; ++j, o += step) {
    const int pe = j * G + g;
    if (pe < p) *o = (RESID && !((ob >> j) & 1ull)) ? 0.0f : acc[j];
  }
}

__global__ void k_finish_stats(const double* __restrict__ block_sums, int nblocks, SweepScalars* sc) {
  __shared__ double red[32];
  double w = 0.0, r = 0.0;
  for (int b = threadIdx.x; b < nblocks; b += blockDim.x) {
    w += block_sums[2 * b];
    r += block_sums[2 * b + 1];
  }
  const double tw = block_sum_d(w, red);
  __syncthreads();
  const double tr = block_sum_d(r, red);
  if (threadIdx.x == 0) {
    sc->sq_w = tw;
    sc->sq_r = tr;
  }
}

// ---------------------------------------------------------------------------
// philox mode: pi ~ Beta, gamma_s, gamma_eps ~ Gamma on device (bpfa.py:313-342).

struct DevRng {
  uint32_t c0, c1, c2, c3, k0, k1;
  u32x4 buf;
  int used;
  __device__ uint32_t next() {
    if (used == 4) {
      buf = philox4x32_10(u32x4{c0, c1, c2, c3}, k0, k1);
      ++c0;
      used = 0;
    }
    const uint32_t v = used == 0 ? buf.x : used == 1 ? buf.y : used == 2 ? buf.z : buf.w;
    ++used;
    return v;
  }
  __device__ double uniform() { const uint32_t a = next(); return u01_53(a, next()); }
  __device__ double normal() {
    const double u1 = uniform(), u2 = uniform();
    return sqrt(-2.0 * log(u1)) * cospi(2.0 * u2);
  }
};

// log of a Gamma(shape, 1) draw (Marsaglia-Tsang; shape < 1 via the U^(1/a) boost).
__device__ double log_gamma_draw(DevRng& rng, double shape) {
  double boost = 0.0;
  if (shape < 1.0) {
    boost = log(rng.uniform()) / shape;
    shape += 1.0;
  }
  const double d = shape - 1.0 / 3.0, c = 1.0 / sqrt(9.0 * d);
  for (int it = 0; it < 1000; ++it) {
    double x, v;
    do {
      x = rng.normal();
      v = 1.0 + c * x;
    } while (v <= 0.0);
    v = v * v * v;
    const double u = rng.uniform();
    if (log(u) < 0.5 * x * x + d - d * v + d * log(v)) return log(d * v) + boost;
  }
  return log(d) + boost;
}

__global__ void k_draw_pi_gamma(double* pi, const int32_t* m_count, SweepScalars* sc, int k_len, int64_t n,
                                int64_t n_obs, double ca, double cb, double ws, double wr, double ns, double nr,
                                uint32_t key0, uint32_t key1) {
  // warps 0..nw-2 draw pi (one atom per thread), the last warp's lane 0 the two
  // gamma draws concurrently (the same streams as drawing them after pi)
  const int epoch = sc->epoch + 1;
  __syncthreads();   // every thread has read the epoch before it is advanced below
  const int npi = blockDim.x - 32;
  if (threadIdx.x < npi) {
  for (int k = threadIdx.x; k < k_len; k += npi) {
    const double m = (double)m_count[k];
    const double sa = fmax(ca / k_len + m, 1e-12);
    const double sb = fmax(cb * (k_len - 1) / k_len + (double)n - m, 1e-12);
    DevRng r{(uint32_t)k << 8, 0u, (uint32_t)epoch, kDomPi << 24, key0, key1, {}, 4};
    const double la = log_gamma_draw(r, sa), lb = log_gamma_draw(r, sb);
    const double mx = fmax(la, lb);
    pi[k] = exp(la - mx) / (exp(la - mx) + exp(lb - mx));
  }
  } else if (threadIdx.x == npi) {
    DevRng r{0u, 0u, (uint32_t)epoch, kDomGamma << 24, key0, key1, {}, 4};
    const double sh_s = ws + 0.5 * (double)n * k_len;
    const double gs = exp(log_gamma_draw(r, sh_s)) / (wr + 0.5 * sc->sq_w);
    const double sh_e = ns + 0.5 * (double)n_obs;
    const double ge = exp(log_gamma_draw(r, sh_e)) / (nr + 0.5 * sc->sq_r);
    sc->gamma_s = fmax(gs, 1e-12);
    sc->gamma_eps = fmax(ge, 1e-12);
    if (!(isfinite(sc->gamma_s) && isfinite(sc->gamma_eps) && isfinite(sc->sq_r))) sc->diverged = 1;
    sc->epoch = epoch;
  }
}

// ---------------------------------------------------------------------------
// Fine-grained seam kernels mirroring _kernels.* one to one (used by the
// posterior helpers and unit parity tests; the epoch uses the fused kernels).

__global__ void k_atom_moments_partial(const float* __restrict__ resid, const uint8_t* __restrict__ obs,
                                       const float* __restrict__ w_col, int64_t n, int p, double* __restrict__ part) {
  __shared__ double red[32];
  const int pe = blockIdx.y;
  double sa = 0.0, sc = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float w = w_col[i];
    if (w != 0.0f && obs[(int64_t)pe * n + i]) {
      sa += (double)w * w;
      sc += (double)w * resid[(int64_t)pe * n + i];
    }
  }
  const double ta = block_sum_d(sa, red);
  __syncthreads();
  const double tc = block_sum_d(sc, red);
  if (threadIdx.x == 0) {
    part[((size_t)pe * gridDim.x + blockIdx.x) * 2] = ta;
    part[((size_t)pe * gridDim.x + blockIdx.x) * 2 + 1] = tc;
  }
}

__global__ void k_atom_moments_final(const double* __restrict__ part, int nb, int p, double* a, double* c) {
  for (int pe = threadIdx.x; pe < p; pe += blockDim.x) {
    double sa = 0.0, sc = 0.0;
    for (int b = 0; b < nb; ++b) {
      sa += part[((size_t)pe * nb + b) * 2];
      sc += part[((size_t)pe * nb + b) * 2 + 1];
    }
    a[pe] = sa;
    c[pe] = sc;
  }
}

__global__ void k_shift_atom(float* __restrict__ resid, const uint8_t* __restrict__ obs, const float* __restrict__ w_col,
                             const float* __restrict__ delta, int64_t n, int p) {
  const int64_t total = n * p;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t % n;
    const int pe = (int)(t / n);
    const float w = w_col[i];
    if (w != 0.0f && obs[t]) resid[t] = fmaf(w, delta[pe], resid[t]);
  }
}

__global__ void k_code_moments(const float* __restrict__ resid, const uint8_t* __restrict__ obs,
                               const float* __restrict__ atom, int64_t n, int p, float* __restrict__ u,
                               float* __restrict__ v) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    float au = 0.0f, av = 0.0f;
    for (int pe = 0; pe < p; ++pe) {
      if (obs[(int64_t)pe * n + i]) {
        const float d = atom[pe];
        au = fmaf(d, d, au);
        av = fmaf(d, resid[(int64_t)pe * n + i], av);
      }
    }
    u[i] = au;
    v[i] = av;
  }
}

__global__ void k_shift_codes(float* __restrict__ resid, const uint8_t* __restrict__ obs, const float* __restrict__ atom,
                              const float* __restrict__ dw, int64_t n, int p) {
  const int64_t total = n * p;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t % n;
    const int pe = (int)(t / n);
    const float d = dw[i];
    if (d != 0.0f && obs[t]) resid[t] = fmaf(d, atom[pe], resid[t]);
  }
}

__global__ void k_sq_norm_partial(const float* __restrict__ x, int64_t total, double* __restrict__ part) {
  __shared__ double red[32];
  double s = 0.0;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x)
    s += (double)x[t] * x[t];
  const double b = block_sum_d(s, red);
  if (threadIdx.x == 0) part[blockIdx.x] = b;
}

__global__ void k_sum_final(const double* __restrict__ part, int nb, double* out) {
  __shared__ double red[32];
  double s = 0.0;
  for (int b = threadIdx.x; b < nb; b += blockDim.x) s += part[b];
  const double t = block_sum_d(s, red);
  if (threadIdx.x == 0) *out = t;
}

// ---------------------------------------------------------------------------
// Native-problem helpers: prior atoms (philox mode; bpfa.py:121-122 draws
// standard normals / sqrt(P)) and the observed-flag total n_obs (bpfa.py:327).

__global__ void k_prior_atoms(float* __restrict__ atoms, int k_len, int p, uint32_t key0, uint32_t key1) {
  const float scale = rsqrtf((float)p);
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < k_len * p; t += gridDim.x * blockDim.x) {
    const u32x4 r = philox4x32_10(u32x4{(uint32_t)(t >> 1), 0u, 0u, kDomInit << 24}, key0, key1);
    float n0, n1;
    box_muller(r.x, r.y, n0, n1);
    atoms[t] = ((t & 1) ? n1 : n0) * scale;
  }
}

__global__ void k_sum_counts(const int32_t* __restrict__ counts, int64_t n, unsigned long long* out) {
  unsigned long long s = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    s += (unsigned long long)counts[i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0 && s) atomicAdd(out, s);
}

// ---------------------------------------------------------------------------
// Host-side launchers

static int sm_count() {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms;
}

// (VPT, G) selection: G lanes per patch, VPT register slots per lane.
static bool pick_layout(int p, int& vpt, int& g) {
  static const int kV[] = {8, 16, 32, 64};
  for (g = 1; g <= 32; g *= 2) {
    const int need = (p + g - 1) / g;
    for (int v : kV)
      if (v >= need) { vpt = v; return true; }
  }
  return false;
}

#define PB_DISPATCH_VG(vpt, g, MACRO)                                                      \
  switch (vpt * 100 + g) {                                                                 \
    MACRO(8, 1) MACRO(16, 1) MACRO(32, 1) MACRO(64, 1)                                     \
    MACRO(64, 2) MACRO(64, 4) MACRO(64, 8) MACRO(64, 16) MACRO(64, 32)                     \
    MACRO(32, 2) MACRO(32, 4) MACRO(32, 8) MACRO(32, 16) MACRO(32, 32)                     \
    default: set_error("unsupported layout vpt=%d g=%d", vpt, g); return PB_EUNSUPPORTED;  \
  }

static int pick_kc(int k_len, int p, size_t budget) {
  int kc = (int)(budget / ((size_t)p * 4));
  if (kc < 1) kc = 1;
  return kc < k_len ? kc : k_len;
}

int launch_accumulate_atoms(bool resid, const float* values, const uint8_t* obs, const uint8_t* usage,
                            const float* weights, const float* atoms, float* out, int64_t n, int p, int k_len,
                            int accumulate, int64_t ld, cudaStream_t st) {
  if (ld < n) ld = n;
  if (!resid && compose_tc_supported(p)) {  // the dense contraction on the tensor cores (3xTF32)
    if (PB_TUNE_INT("PB_COMPOSE_TC", 1)) return launch_compose_tc(usage, weights, ld, atoms, p, k_len, n, out, accumulate, st);
  }
  int vpt, g;
  if (!pick_layout(p, vpt, g)) { set_error("patch size %d exceeds 2048", p); return PB_EUNSUPPORTED; }
  const int th = 256;
  const int kc = pick_kc(k_len, vpt * g, 64 * 1024);
  const size_t smem = (size_t)kc * vpt * g * 4;
  const int64_t nb = ceil_div(n * g, th);
#define PB_ACC(V, GG)                                                                                      \
  case V * 100 + GG: {                                                                                     \
    auto kern = resid ? k_accumulate_atoms<V, GG, true> : k_accumulate_atoms<V, GG, false>;                \
    PB_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));       \
    kern<<<(unsigned)nb, th, smem, st>>>(values, obs, usage, weights, atoms, out, n, p, k_len, kc, accumulate, ld); \
    break;                                                                                                 \
  }
  PB_DISPATCH_VG(vpt, g, PB_ACC)
#undef PB_ACC
  PB_LAUNCH_CHECK();
  return PB_OK;
}

// Two-level variant for many block sums (warp-claimed code steps of large
// problems): CTA c sums the contiguous range c of the block sums (fixed tree),
// the last CTA to finish sums the CTA partials in index order — deterministic.
// Partials and the ticket live right after the block sums.
__global__ void k_finish_stats_2l(double* __restrict__ block_sums, int nblocks, int per_cta, SweepScalars* sc) {
  __shared__ double red[32];
  __shared__ bool last;
  double* part = block_sums + 2 * (size_t)nblocks;
  unsigned* ticket = (unsigned*)(part + 2 * (size_t)gridDim.x);
  const int b0 = blockIdx.x * per_cta, b1 = min(nblocks, b0 + per_cta);
  double w = 0.0, r = 0.0;
  for (int b = b0 + threadIdx.x; b < b1; b += blockDim.x) {
    w += block_sums[2 * b];
    r += block_sums[2 * b + 1];
  }
  const double tw = block_sum_d(w, red);
  __syncthreads();
  const double tr = block_sum_d(r, red);
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = tw;
    part[2 * blockIdx.x + 1] = tr;
    __threadfence();
    last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  double pw = 0.0, pr = 0.0;
  for (int c = threadIdx.x; c < (int)gridDim.x; c += blockDim.x) {
    pw += __ldcg(part + 2 * c);
    pr += __ldcg(part + 2 * c + 1);
  }
  const double sw = block_sum_d(pw, red);
  __syncthreads();
  const double sr = block_sum_d(pr, red);
  if (threadIdx.x == 0) {
    sc->sq_w = sw;
    sc->sq_r = sr;
    *ticket = 0u;
  }
}

int launch_finish_stats(const double* block_sums, int nblocks, SweepScalars* sc, cudaStream_t st) {
  constexpr int kPer = 4096;
  if (nblocks <= 2 * kPer) {
    k_finish_stats<<<1, 1024, 0, st>>>(block_sums, nblocks, sc);
  } else {
    const int ctas = (int)ceil_div(nblocks, kPer);
    unsigned* ticket = (unsigned*)(const_cast<double*>(block_sums) + 2 * (size_t)nblocks + 2 * (size_t)ctas);
    PB_CUDA_TRY(cudaMemsetAsync(ticket, 0, sizeof(unsigned), st));
    k_finish_stats_2l<<<ctas, 1024, 0, st>>>(const_cast<double*>(block_sums), nblocks, kPer, sc);
  }
  PB_LAUNCH_CHECK();
  return PB_OK;
}

int launch_draw_pi_gamma(double* pi, const int32_t* m_count, SweepScalars* sc, int k_len, int64_t n, int64_t n_obs,
                         const double* hyper6, uint32_t key0, uint32_t key1, cudaStream_t st) {
  k_draw_pi_gamma<<<1, 256 + 32, 0, st>>>(pi, m_count, sc, k_len, n, n_obs, hyper6[0], hyper6[1], hyper6[2], hyper6[3],
                                     hyper6[4], hyper6[5], key0, key1);
  PB_LAUNCH_CHECK();
  return PB_OK;
}

int launch_atom_moments(const float* resid, const uint8_t* obs, const float* w_col, int64_t n, int p, double* part,
                        int nb, double* a, double* c, cudaStream_t st) {
  k_atom_moments_partial<<<dim3(nb, p), 256, 0, st>>>(resid, obs, w_col, n, p, part);
  k_atom_moments_final<<<1, 256, 0, st>>>(part, nb, p, a, c);
  PB_LAUNCH_CHECK();
  return PB_OK;
}

int launch_shift_atom(float* resid, const uint8_t* obs, const float* w_col, const float* delta, int64_t n, int p,
                      cudaStream_t st) {
  k_shift_atom<<<sm_count() * 8, 256, 0, st>>>(resid, obs, w_col, delta, n, p);
  PB_LAUNCH_CHECK();
  return PB_OK;
}

int launch_code_moments(const float* resid, const uint8_t* obs, const float* atom, int64_t n, int p, float* u,
                        float* v, cudaStream_t st) {
  k_code_moments<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(resid, obs, atom, n, p, u, v);
  PB_LAUNCH_CHECK();
  return PB_OK;
}

int launch_shift_codes(float* resid, const uint8_t* obs, const float* atom, const float* dw, int64_t n, int p,
                       cudaStream_t st) {
  k_shift_codes<<<sm_count() * 8, 256, 0, st>>>(resid, obs, atom, dw, n, p);
  PB_LAUNCH_CHECK();
  return PB_OK;
}

int launch_sq_norm(const float* x, int64_t total, double* part, int nb, double* out, cudaStream_t st) {
  k_sq_norm_partial<<<nb, 256, 0, st>>>(x, total, part);
  k_sum_final<<<1, 256, 0, st>>>(part, nb, out);
  PB_LAUNCH_CHECK();
  return PB_OK;
}

}  // namespace pb

namespace pb {
int launch_prior_atoms(float* atoms, int k_len, int p, uint32_t key0, uint32_t key1, cudaStream_t st) {
  k_prior_atoms<<<(k_len * p + 255) / 256, 256, 0, st>>>(atoms, k_len, p, key0, key1);
  PB_LAUNCH_CHECK();
  return PB_OK;
}
int launch_sum_counts(const int32_t* counts, int64_t n, unsigned long long* out, cudaStream_t st) {
  PB_CUDA_TRY(cudaMemsetAsync(out, 0, sizeof(unsigned long long), st));
  k_sum_counts<<<sm_count() * 4, 256, 0, st>>>(counts, n, out);
  PB_LAUNCH_CHECK();
  return PB_OK;
}
}  // namespace pb
