// pb200 — the BPFA Gibbs sweep on sm_100a.
//
// Reference: pkg/src/patchbeam/bpfa.py:278-345 (gibbs_epoch) and the seven Numba
// kernels of pkg/src/patchbeam/_kernels.py.  One epoch here is:
//
//   k_residual        R = o * (X - (Z*S) D)                       (_kernels.py:18-31)
//   k_dict_step       persistent cooperative kernel, atoms k = 0..K-1 in order:
//                     A_k, C_k block partials -> last-arriving CTA reduces them in
//                     fixed CTA order, draws d_k = mu + g/sqrt(lambda), publishes
//                     delta_k; every CTA shifts its resident tile of R and, in the
//                     same pass, accumulates the next atom's moments
//                     (bpfa.py:299-307, _kernels.py:34-74)
//   k_code_step       one thread group per patch, the patch's residual in registers,
//                     the dictionary in shared memory, atoms k = 0..K-1 in order:
//                     u, v dot products, the z/s conditional draw, register shift
//                     (bpfa.py:240-275, _kernels.py:77-109); epilogue block sums of
//                     sum S^2, sum R^2 and per-atom usage counts m_k (bpfa.py:313-328)
//   k_finish_stats    fixed-order reduction of the block partials
//   k_draw_pi_gamma   (philox mode) pi ~ Beta, gamma_s, gamma_eps ~ Gamma on device
//
// Compute precision: f32 state and FMAs; cross-patch sums accumulate in f64 at
// block/grid level; the z/s conditional algebra is f32 (numpy mode compares the
// reference's exact logistic draw in f64).
#include <math.h>

#include "pb_sweep.cuh"

namespace pb {



// ---------------------------------------------------------------------------
// residual / compose: one G-lane group per patch, VPT register elements per lane.
// Element p = j*G + g of patch i lives in lane g, slot j.

template <int VPT, int G, bool RESID>
__global__ void __launch_bounds__(256) k_accumulate_atoms(
    const float* __restrict__ values, const uint8_t* __restrict__ obs, const uint8_t* __restrict__ usage,
    const float* __restrict__ weights, const float* __restrict__ atoms, float* __restrict__ out, int64_t n, int p,
    int k_len, int kc, int accumulate) {
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
    if (live) {
      for (int kk = 0; kk < kn; ++kk) {
        const int64_t zi = (int64_t)(k0 + kk) * n + i;
        if (!usage[zi]) continue;
        const float w = RESID ? -weights[zi] : weights[zi];
        const float* d = ds + kk * PP + g;
#pragma unroll
        for (int j = 0; j < VPT; ++j) acc[j] = fmaf(w, d[j * G], acc[j]);
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

// ---------------------------------------------------------------------------
// Dictionary step: persistent cooperative kernel (all CTAs co-resident).


__device__ __forceinline__ float active_w(const uint8_t* usage, const float* weights, int64_t idx) {
  return usage[idx] ? weights[idx] : 0.0f;
}

__global__ void __launch_bounds__(512) k_dict_step(DictArgs a) {
  extern __shared__ float sm[];
  const int tile = a.tile;
  float* wprev = sm;                 // tile
  float* wcur = wprev + tile;        // tile
  float* acc = wcur + tile;          // 2P  (A then C)
  float* dprev = acc + 2 * a.p;      // P
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int64_t per = ceil_div(a.n, gridDim.x);
  const int64_t lo = min((int64_t)blockIdx.x * per, a.n), hi = min(lo + per, a.n);
  const int epoch = a.sc->epoch + 1;
  const double geps = a.sc->gamma_eps;

  for (int k = 0; k <= a.k_len; ++k) {
    for (int t = threadIdx.x; t < 2 * a.p; t += blockDim.x) acc[t] = 0.0f;
    for (int64_t t0 = lo; t0 < hi; t0 += tile) {
      const int tn = (int)min((int64_t)tile, hi - t0);
      __syncthreads();
      for (int t = threadIdx.x; t < tn; t += blockDim.x) {
        wprev[t] = k > 0 ? active_w(a.usage, a.weights, (int64_t)(k - 1) * a.n + t0 + t) : 0.0f;
        wcur[t] = k < a.k_len ? active_w(a.usage, a.weights, (int64_t)k * a.n + t0 + t) : 0.0f;
      }
      __syncthreads();
      for (int pr = wid; pr < a.p; pr += nw) {
        const float dl = k > 0 ? dprev[pr] : 0.0f;
        float sa = 0.0f, sc = 0.0f;
        float* rrow = a.resid + (int64_t)pr * a.n + t0;
        const uint8_t* orow = a.obs + (int64_t)pr * a.n + t0;
        for (int t = lane; t < tn; t += 32) {
          if (!orow[t]) continue;
          const float wp = wprev[t], wc = wcur[t];
          if (wp == 0.0f && wc == 0.0f) continue;
          float r = rrow[t];
          if (wp != 0.0f) {
            r = fmaf(wp, dl, r);
            rrow[t] = r;
          }
          sa = fmaf(wc, wc, sa);
          sc = fmaf(wc, r, sc);
        }
        if (k < a.k_len) {
          sa = warp_sum(sa);
          sc = warp_sum(sc);
          if (lane == 0) {
            acc[pr] += sa;
            acc[a.p + pr] += sc;
          }
        }
      }
    }
    if (k == a.k_len) break;
    __syncthreads();
    // publish this CTA's partial moments for atom k
    double* mine = a.partials + (size_t)blockIdx.x * 2 * a.p;
    for (int t = threadIdx.x; t < 2 * a.p; t += blockDim.x) mine[t] = (double)acc[t];
    __shared__ unsigned int s_last;
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      const unsigned int ticket = atomicAdd(&a.sync[0], 1u);
      s_last = (ticket == (unsigned int)(k + 1) * gridDim.x - 1u) ? 1u : 0u;
    }
    __syncthreads();
    if (s_last) {
      __threadfence();
      // fixed-order cross-CTA reduction, then the atom draw (bpfa.py:161-166, 303-307)
      for (int pe = threadIdx.x; pe < a.p; pe += blockDim.x) {
        double sa = 0.0, sc = 0.0;
        for (int b = 0; b < (int)gridDim.x; ++b) {
          sa += __ldcg(a.partials + (size_t)b * 2 * a.p + pe);
          sc += __ldcg(a.partials + (size_t)b * 2 * a.p + a.p + pe);
        }
        const double dold = (double)a.atoms[(int64_t)k * a.p + pe];
        const double lam = (double)a.p + geps * sa;
        const double mu = geps * (sc + dold * sa) / lam;
        double gdraw;
        if (a.draws) {
          gdraw = a.draws[(int64_t)k * a.p + pe];
        } else {
          const u32x4 r = philox4x32_10(u32x4{(uint32_t)(pe >> 1), (uint32_t)k, (uint32_t)epoch, kDomAtom << 24},
                                        a.key0, a.key1);
          float n0, n1;
          box_muller(r.x, r.y, n0, n1);
          gdraw = (pe & 1) ? n1 : n0;
        }
        const float dnew = (float)(mu + gdraw / sqrt(lam));
        a.atoms[(int64_t)k * a.p + pe] = dnew;
        a.delta[pe] = (float)dold - dnew;
      }
      __threadfence();
      __syncthreads();
      if (threadIdx.x == 0) atomicExch(&a.sync[1], (unsigned int)(k + 1));
    }
    if (threadIdx.x == 0) {
      while (atomicAdd(&a.sync[1], 0u) < (unsigned int)(k + 1)) __nanosleep(32);
      __threadfence();
    }
    __syncthreads();
    for (int t = threadIdx.x; t < a.p; t += blockDim.x) dprev[t] = __ldcg(a.delta + t);
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// Code step.


template <int G>
__device__ __forceinline__ float group_sum(float v) {
#pragma unroll
  for (int o = G >> 1; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <int VPT, int G, int MODE>
__global__ void __launch_bounds__(256) k_code_step(CodeArgs a) {
  extern __shared__ float sm[];
  float* logit = sm;                       // K
  int* mcnt = (int*)(logit + a.k_len);     // K
  float* ds = (float*)(mcnt + a.k_len);    // kc * P
  __shared__ double red[32];
  const int g = threadIdx.x % G;
  const int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / G;
  const bool live = i < a.n;
  const int lane = threadIdx.x & 31;
  const int epoch = a.sc->epoch + 1;
  const float geps = (float)a.sc->gamma_eps, gs = (float)a.sc->gamma_s;
  const float inv_sqrt_gs = (float)(1.0 / sqrt(a.sc->gamma_s));

  for (int k = threadIdx.x; k < a.k_len; k += blockDim.x) {
    double pk = a.pi[k];
    pk = fmin(fmax(pk, 1e-15), 1.0 - 1e-15);  // bpfa.py:173
    logit[k] = (float)(log(pk) - log1p(-pk));
    mcnt[k] = 0;
  }
  float r[VPT];
  uint64_t ob = 0;
#pragma unroll
  for (int j = 0; j < VPT; ++j) {
    const int pe = j * G + g;
    r[j] = 0.0f;
    if (live && pe < a.p) {
      r[j] = a.resid[(int64_t)pe * a.n + i];
      if (a.obs[(int64_t)pe * a.n + i]) ob |= 1ull << j;
    }
  }
  double sq_w = 0.0;
  u32x4 rnd{0, 0, 0, 0};
  float nrm0 = 0.f, nrm1 = 0.f;
  constexpr int PP = VPT * G;  // shared-memory row pitch, zero padded past p
  for (int k0 = 0; k0 < a.k_len; k0 += a.kc) {
    const int kn = min(a.kc, a.k_len - k0);
    __syncthreads();
    for (int t = threadIdx.x; t < kn * PP; t += blockDim.x) {
      const int kk = t / PP, pe = t - kk * PP;
      ds[t] = pe < a.p ? a.atoms[(int64_t)(k0 + kk) * a.p + pe] : 0.0f;
    }
    __syncthreads();
    for (int kk = 0; kk < kn; ++kk) {
      const int k = k0 + kk;
      const float* d = ds + kk * PP + g;
      float u = 0.0f, v = 0.0f;
#pragma unroll
      for (int j = 0; j < VPT; ++j) {
        const float dj = d[j * G];
        const float dm = ((ob >> j) & 1ull) ? dj : 0.0f;
        u = fmaf(dm, dm, u);
        v = fmaf(dj, r[j], v);
      }
      if (G > 1) {
        u = group_sum<G>(u);
        v = group_sum<G>(v);
      }
      // Re-read d from shared memory for the shift instead of holding VPT more
      // registers across the draw (keeps the residual itself register-resident).
      asm volatile("" ::: "memory");
      bool z = false;
      if (live) {
        const int64_t zi = (int64_t)k * a.n + i;
        const bool z_old = a.usage[zi] != 0;
        const float s_old = a.weights[zi];
        const float w_old = z_old ? s_old : 0.0f;
        // _code_params (bpfa.py:169-178)
        const float proj = fmaf(w_old, u, v);
        const float log_rho = logit[k] - 0.5f * geps * (s_old * s_old * u - 2.0f * s_old * proj);
        const float alpha = fmaf(geps, u, gs);
        const float mean = geps * proj / alpha;
        float gn;
        if (MODE == kRngReplay) {
          const double ud = a.u_draw[zi];
          gn = (float)a.g_draw[zi];
          z = (log(ud) - log1p(-ud)) < (double)log_rho;  // bpfa.py:262-263
        } else {
          if ((k & 1) == 0) {
            rnd = philox4x32_10(u32x4{(uint32_t)i, (uint32_t)(i >> 32), (uint32_t)(k >> 1),
                                      ((uint32_t)epoch & 0xFFFFFFu) | (kDomCode << 24)},
                                a.key0, a.key1);
            box_muller(rnd.z, rnd.w, nrm0, nrm1);
          }
          const float uu = u01_24((k & 1) ? rnd.y : rnd.x);
          gn = (k & 1) ? nrm1 : nrm0;
          // z = 1 w.p. sigmoid(log_rho): U < 1/(1+exp(-log_rho))
          z = uu * (1.0f + __expf(-log_rho)) < 1.0f;
        }
        const float s_new = z ? mean + gn * rsqrtf(alpha) : gn * inv_sqrt_gs;  // bpfa.py:265-269
        const float dw = w_old - (z ? s_new : 0.0f);
        if (dw != 0.0f) {
#pragma unroll
          for (int j = 0; j < VPT; ++j)
            if ((ob >> j) & 1ull) r[j] = fmaf(dw, d[j * G], r[j]);
        }
        if (g == 0) {
          a.usage[zi] = z ? 1 : 0;
          a.weights[zi] = s_new;
          sq_w += (double)s_new * (double)s_new;
        }
      }
      // usage count for pi (bpfa.py:217-222): one ballot per warp
      const unsigned bal = __ballot_sync(0xffffffffu, z && g == 0);
      if (lane == 0 && bal) atomicAdd(&mcnt[k], __popc(bal));
    }
  }
  double sq_r = 0.0;
#pragma unroll
  for (int j = 0; j < VPT; ++j) sq_r += (double)r[j] * (double)r[j];
  const double bw = block_sum_d(sq_w, red);
  __syncthreads();
  const double br = block_sum_d(sq_r, red);
  if (threadIdx.x == 0) {
    a.block_sums[2 * blockIdx.x] = bw;
    a.block_sums[2 * blockIdx.x + 1] = br;
  }
  __syncthreads();
  for (int k = threadIdx.x; k < a.k_len; k += blockDim.x)
    if (mcnt[k]) atomicAdd(&a.m_count[k], mcnt[k]);
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
  const int epoch = sc->epoch + 1;
  for (int k = threadIdx.x; k < k_len; k += blockDim.x) {
    const double m = (double)m_count[k];
    const double sa = fmax(ca / k_len + m, 1e-12);
    const double sb = fmax(cb * (k_len - 1) / k_len + (double)n - m, 1e-12);
    DevRng r{(uint32_t)k << 8, 0u, (uint32_t)epoch, kDomPi << 24, key0, key1, {}, 4};
    const double la = log_gamma_draw(r, sa), lb = log_gamma_draw(r, sb);
    const double mx = fmax(la, lb);
    pi[k] = exp(la - mx) / (exp(la - mx) + exp(lb - mx));
  }
  if (threadIdx.x == 0) {
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
                            int accumulate, cudaStream_t st) {
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
    kern<<<(unsigned)nb, th, smem, st>>>(values, obs, usage, weights, atoms, out, n, p, k_len, kc, accumulate); \
    break;                                                                                                 \
  }
  PB_DISPATCH_VG(vpt, g, PB_ACC)
#undef PB_ACC
  PB_LAUNCH_CHECK();
  return PB_OK;
}

int dict_step_grid(int p, int& blocks, int& threads, size_t& smem, int& tile) {
  threads = 512;
  tile = 2048;
  smem = (size_t)(2 * tile + 3 * p) * sizeof(float);
  if (smem > 200 * 1024) { set_error("patch size too large for dict step"); return PB_EUNSUPPORTED; }
  PB_CUDA_TRY(cudaFuncSetAttribute(k_dict_step, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 0;
  PB_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_dict_step, threads, smem));
  if (per_sm < 1) { set_error("dict step cannot be resident"); return PB_EUNSUPPORTED; }
  blocks = sm_count() * (per_sm > 2 ? 2 : per_sm);
  return PB_OK;
}

int launch_dict_step(const DictArgs& a_in, int blocks, int threads, size_t smem, cudaStream_t st) {
  DictArgs a = a_in;
  PB_CUDA_TRY(cudaMemsetAsync(a.sync, 0, 2 * sizeof(unsigned int), st));
  void* args[] = {&a};
  PB_CUDA_TRY(cudaLaunchCooperativeKernel((const void*)k_dict_step, dim3(blocks), dim3(threads), args, smem, st));
  return PB_OK;
}

int launch_code_step(const CodeArgs& a_in, int mode, int& nblocks, cudaStream_t st) {
  CodeArgs a = a_in;
  int vpt, g;
  if (!pick_layout(a.p, vpt, g)) { set_error("patch size %d exceeds 2048", a.p); return PB_EUNSUPPORTED; }
  const int th = 256;
  a.kc = pick_kc(a.k_len, vpt * g, 100 * 1024);
  const size_t smem = (size_t)a.kc * vpt * g * 4 + (size_t)a.k_len * 8;
  if (smem > 220 * 1024) { set_error("too many atoms for the code step (K=%d)", a.k_len); return PB_EUNSUPPORTED; }
  const int64_t nb = ceil_div(a.n * g, th);
  nblocks = (int)nb;
  PB_CUDA_TRY(cudaMemsetAsync(a.m_count, 0, (size_t)a.k_len * sizeof(int32_t), st));
#define PB_CODE(V, GG)                                                                                   \
  case V * 100 + GG: {                                                                                   \
    auto kern = mode == kRngReplay ? k_code_step<V, GG, kRngReplay> : k_code_step<V, GG, kRngPhilox>;    \
    PB_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));     \
    kern<<<(unsigned)nb, th, smem, st>>>(a);                                                             \
    break;                                                                                               \
  }
  PB_DISPATCH_VG(vpt, g, PB_CODE)
#undef PB_CODE
  PB_LAUNCH_CHECK();
  return PB_OK;
}

int launch_finish_stats(const double* block_sums, int nblocks, SweepScalars* sc, cudaStream_t st) {
  k_finish_stats<<<1, 1024, 0, st>>>(block_sums, nblocks, sc);
  PB_LAUNCH_CHECK();
  return PB_OK;
}

int launch_draw_pi_gamma(double* pi, const int32_t* m_count, SweepScalars* sc, int k_len, int64_t n, int64_t n_obs,
                         const double* hyper6, uint32_t key0, uint32_t key1, cudaStream_t st) {
  k_draw_pi_gamma<<<1, 256, 0, st>>>(pi, m_count, sc, k_len, n, n_obs, hyper6[0], hyper6[1], hyper6[2], hyper6[3],
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
