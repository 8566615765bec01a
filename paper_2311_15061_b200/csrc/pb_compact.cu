// pb200 — observed-element ("compact") Gibbs sweep kernels for sm_100a.
//
// Reference semantics: bpfa.py:278-345 (gibbs_epoch), bpfa.py:240-275 (code
// sampling), bpfa.py:299-307 (atom updates), _kernels.py:18-130.  Only the
// observed elements of each patch ever enter a conditional, so the residual is
// stored for those nnz elements only (pb_index.cu), in the dictionary step's
// CSC-tile order.
//
//  k_resid_compact  R = X - (Z*S) D on observed elements (residual_full).
//  k_dict_gram      the dictionary step, persistent & cooperative.  Atoms are
//                   processed in blocks of B.  For atom k inside block [k0,k0+B)
//                     C_k^(k) = C_k^(k0) + sum_{k0<=j<k} G_kj o delta_j
//                   with per-pixel Gram G_kj[p] = sum_i o_ip w_ik w_ij and
//                   delta_j = d_j(old) - d_j(new) (the atom shift of
//                   _kernels.shift_atom), which is the reference's sequential
//                   update k = 1..K exactly (up to rounding) — but needs ONE pass
//                   over the residual and TWO grid barriers per block instead of
//                   one pass + one barrier per atom.  The same pass applies the
//                   previous block's shifts to the residual.
//  k_code_compact   the code step: one thread (group) per patch, the patch's
//                   observed residual in registers, the dictionary in shared
//                   memory (gathered by the patch's observed offsets), atoms
//                   k = 0..K-1 in order with the z/s draw in registers.
#include <math.h>

#include "pb_compact.cuh"

namespace pb {

// ---------------------------------------------------------------------------
// Shared-memory staging of D (rows of pitch PP = P + 1; column P is zero so
// padded slots contribute nothing).
__device__ __forceinline__ void stage_atoms(float* ds, const float* __restrict__ atoms, int k0, int kn, int p, int pp) {
  for (int t = threadIdx.x; t < kn * pp; t += blockDim.x) {
    const int kk = t / pp, pe = t - kk * pp;
    ds[t] = pe < p ? atoms[(int64_t)(k0 + kk) * p + pe] : 0.0f;
  }
}

template <int G>
__device__ __forceinline__ float gsum(float v) {
#pragma unroll
  for (int o = G >> 1; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ---------------------------------------------------------------------------
template <int CMAX, int G>
__global__ void __launch_bounds__(256) k_resid_compact(CompactArgs a) {
  extern __shared__ float ds[];
  const int pp = a.p + 1;
  const int g = threadIdx.x % G;
  const int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / G;
  const bool live = i < a.n;
  float acc[CMAX];
  int off[CMAX];
  uint32_t pos[CMAX];
  int cnt = 0;
  int64_t r0 = 0;
  if (live) { cnt = a.counts[i]; r0 = a.rowptr[i]; }
#pragma unroll
  for (int j = 0; j < CMAX; ++j) {
    const int s = j * G + g;
    const bool v = s < cnt;
    off[j] = v ? a.csr_p[r0 + s] : a.p;
    pos[j] = v ? a.csr_pos[r0 + s] : 0u;
    acc[j] = v ? a.x_csc[pos[j]] : 0.0f;
  }
  for (int k0 = 0; k0 < a.k; k0 += a.kc) {
    const int kn = min(a.kc, a.k - k0);
    __syncthreads();
    stage_atoms(ds, a.atoms, k0, kn, a.p, pp);
    __syncthreads();
    if (!live) continue;
    for (int kk = 0; kk < kn; ++kk) {
      const int64_t zi = (int64_t)(k0 + kk) * a.n + i;
      if (!a.usage[zi]) continue;
      const float w = a.weights[zi];
      const float* d = ds + kk * pp;
#pragma unroll
      for (int j = 0; j < CMAX; ++j) acc[j] = fmaf(-w, d[off[j]], acc[j]);
    }
  }
  if (!live) return;
#pragma unroll
  for (int j = 0; j < CMAX; ++j)
    if (j * G + g < cnt) a.r_csc[pos[j]] = acc[j];
}

// ---------------------------------------------------------------------------
template <int CMAX, int G, int MODE>
__global__ void __launch_bounds__(256) k_code_compact(CompactArgs a) {
  extern __shared__ float sm[];
  const int pp = a.p + 1;
  float* logit = sm;                     // K
  int* mcnt = (int*)(logit + a.k);       // K
  float* ds = (float*)(mcnt + a.k);      // kc * pp
  __shared__ double red[32];
  const int g = threadIdx.x % G;
  const int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / G;
  const bool live = i < a.n;
  const int lane = threadIdx.x & 31;
  const int epoch = a.sc->epoch + 1;
  const float geps = (float)a.sc->gamma_eps, gs = (float)a.sc->gamma_s;
  const float inv_sqrt_gs = (float)(1.0 / sqrt(a.sc->gamma_s));

  for (int k = threadIdx.x; k < a.k; k += blockDim.x) {
    const double pk = fmin(fmax(a.pi[k], 1e-15), 1.0 - 1e-15);  // bpfa.py:173
    logit[k] = (float)(log(pk) - log1p(-pk));
    mcnt[k] = 0;
  }
  float r[CMAX];
  int off[CMAX];
  int cnt = 0;
  int64_t r0 = 0;
  if (live) { cnt = a.counts[i]; r0 = a.rowptr[i]; }
#pragma unroll
  for (int j = 0; j < CMAX; ++j) {
    const int s = j * G + g;
    const bool v = s < cnt;
    off[j] = v ? a.csr_p[r0 + s] : a.p;
    r[j] = v ? a.r_csc[a.csr_pos[r0 + s]] : 0.0f;
  }
  double sq_w = 0.0;
  u32x4 rnd{0, 0, 0, 0};
  float nrm0 = 0.f, nrm1 = 0.f;
  for (int k0 = 0; k0 < a.k; k0 += a.kc) {
    const int kn = min(a.kc, a.k - k0);
    __syncthreads();
    stage_atoms(ds, a.atoms, k0, kn, a.p, pp);
    __syncthreads();
    for (int kk = 0; kk < kn; ++kk) {
      const int k = k0 + kk;
      const float* d = ds + kk * pp;
      float dj[CMAX];
      float u = 0.0f, v = 0.0f;
#pragma unroll
      for (int j = 0; j < CMAX; ++j) {
        dj[j] = d[off[j]];
        u = fmaf(dj[j], dj[j], u);
        v = fmaf(dj[j], r[j], v);
      }
      if (G > 1) {
        u = gsum<G>(u);
        v = gsum<G>(v);
      }
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
          z = uu * (1.0f + __expf(-log_rho)) < 1.0f;  // U < sigmoid(log_rho)
        }
        const float s_new = z ? mean + gn / sqrtf(alpha) : gn * inv_sqrt_gs;  // bpfa.py:265-269
        const float dw = w_old - (z ? s_new : 0.0f);
#pragma unroll
        for (int j = 0; j < CMAX; ++j) r[j] = fmaf(dw, dj[j], r[j]);
        if (g == 0) {
          a.usage[zi] = z ? 1 : 0;
          a.weights[zi] = s_new;
          sq_w += (double)s_new * (double)s_new;
        }
      }
      const unsigned bal = __ballot_sync(0xffffffffu, z && g == 0);
      if (lane == 0 && bal) atomicAdd(&mcnt[k], __popc(bal));
    }
  }
  double sq_r = 0.0;
#pragma unroll
  for (int j = 0; j < CMAX; ++j) sq_r += (double)r[j] * (double)r[j];
  const double bw = block_sum_d(sq_w, red);
  __syncthreads();
  const double br = block_sum_d(sq_r, red);
  if (threadIdx.x == 0) {
    a.block_sums[2 * blockIdx.x] = bw;
    a.block_sums[2 * blockIdx.x + 1] = br;
  }
  __syncthreads();
  for (int k = threadIdx.x; k < a.k; k += blockDim.x)
    if (mcnt[k]) atomicAdd(&a.m_count[k], mcnt[k]);
}

// ---------------------------------------------------------------------------
// Grid barrier for the cooperative dictionary kernel (all CTAs co-resident).
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void grid_sync(unsigned* bar) {
  // bar[0]: arrival count, bar[1]: generation
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned gen = ld_acquire(bar + 1);
    __threadfence();
    if (atomicAdd(bar, 1u) == gridDim.x - 1) {
      atomicExch(bar, 0u);
      __threadfence();
      atomicAdd(bar + 1, 1u);
    } else {
      while (ld_acquire(bar + 1) == gen) __nanosleep(20);
    }
    __threadfence();
  }
  __syncthreads();
}

// Recursive-halving transpose reduction of NP (= 16*R) per-lane values across a
// warp: afterwards lane pair (l, l^1) holds the warp sums of values
// [base(l), base(l)+R) with base = 8R*b4 + 4R*b3 + 2R*b2 + R*b1 (b = lane bits).
template <int NP>
__device__ __forceinline__ void warp_transpose_reduce(float (&v)[NP], int lane) {
  static_assert(NP % 16 == 0, "NP must be a multiple of 16");
#pragma unroll
  for (int lvl = 0; lvl < 4; ++lvl) {
    const int o = 16 >> lvl;
    const int half = NP >> (lvl + 1);
    const bool lo = (lane & o) == 0;
#pragma unroll
    for (int q = 0; q < half; ++q) {
      const float send = lo ? v[half + q] : v[q];
      const float keep = lo ? v[q] : v[half + q];
      v[q] = keep + __shfl_xor_sync(0xffffffffu, send, o);
    }
  }
#pragma unroll
  for (int q = 0; q < NP / 16; ++q) v[q] += __shfl_xor_sync(0xffffffffu, v[q], 1);
}

template <int B>
struct GramLayout {
  static constexpr int NACC = B + B * (B + 1) / 2;      // C_j, then G_jl (l <= j), G_jj = A_j
  static constexpr int NP = ((NACC + 15) / 16) * 16;    // padded for the transpose reduce
  __device__ static constexpr int gidx(int j, int l) { return B + j * (j + 1) / 2 + l; }
};

template <int B>
__global__ void __launch_bounds__(256) k_dict_gram(DictGramArgs a) {
  using L = GramLayout<B>;
  extern __shared__ __align__(16) unsigned char smraw[];
  const int p = a.p;
  // shared layout
  float* wcur = (float*)smraw;                         // kTile * B   (aliased by red64 in the update phase)
  float* wprev = wcur + kTile * B;                     // kTile * B
  float* acc = (float*)(smraw + a.wbytes);             // p * NACC
  float* dold = acc + (size_t)p * L::NACC;             // B * p
  float* dprev = dold + B * p;                         // B * p   (delta of the previous block)
  double* red64 = (double*)smraw;                      // p * NACC (aliases wcur/wprev)

  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const double geps = a.sc->gamma_eps;
  const int epoch = a.sc->epoch + 1;
  const int nblk = (a.k + B - 1) / B;

  // element-balanced static tile range of this CTA
  const int64_t nnz = a.tile_base[a.ntiles];
  const int64_t e_lo = nnz * blockIdx.x / gridDim.x, e_hi = nnz * (blockIdx.x + 1) / gridDim.x;
  auto first_tile = [&](int64_t e) {  // first tile whose start >= e
    int lo = 0, hi = a.ntiles;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (a.tile_base[mid] < e) lo = mid + 1; else hi = mid;
    }
    return lo;
  };
  const int t_lo = blockIdx.x == 0 ? 0 : first_tile(e_lo);
  const int t_hi = blockIdx.x == gridDim.x - 1 ? a.ntiles : first_tile(e_hi);

  for (int blk = 0; blk <= nblk; ++blk) {
    const bool has_cur = blk < nblk, has_prev = blk > 0;
    const int k0 = blk * B;
    const int nb = has_cur ? min(B, a.k - k0) : 0;
    const int kp0 = k0 - B;
    for (int t = threadIdx.x; t < p * L::NACC; t += blockDim.x) acc[t] = 0.0f;
    for (int t = threadIdx.x; t < B * p; t += blockDim.x) {
      const int j = t / p, pe = t - j * p;
      dold[t] = j < nb ? a.atoms[(int64_t)(k0 + j) * p + pe] : 0.0f;
    }
    for (int tile = t_lo; tile < t_hi; ++tile) {
      const int64_t ibase = (int64_t)tile * kTile;
      const int tn = (int)min((int64_t)kTile, a.n - ibase);
      __syncthreads();
      for (int t = threadIdx.x; t < B * kTile; t += blockDim.x) {
        const int j = t / kTile, il = t - j * kTile;
        float wc = 0.0f, wp = 0.0f;
        if (il < tn) {
          if (j < nb) {
            const int64_t zi = (int64_t)(k0 + j) * a.n + ibase + il;
            wc = a.usage[zi] ? a.weights[zi] : 0.0f;
          }
          if (has_prev) {
            const int64_t zi = (int64_t)(kp0 + j) * a.n + ibase + il;
            wp = a.usage[zi] ? a.weights[zi] : 0.0f;
          }
        }
        wcur[il * B + j] = wc;
        wprev[il * B + j] = wp;
      }
      __syncthreads();
      const int32_t* cp = a.colptr + (int64_t)tile * (p + 1);
      for (int pe = wid; pe < p; pe += nw) {
        const int cs = cp[pe], ce = cp[pe + 1];
        if (ce == cs) continue;
        float dl[B];
#pragma unroll
        for (int j = 0; j < B; ++j) dl[j] = has_prev ? dprev[j * p + pe] : 0.0f;
        float v[L::NP];
#pragma unroll
        for (int q = 0; q < L::NP; ++q) v[q] = 0.0f;
        for (int e = cs + lane; e < ce; e += 32) {
          const int il = a.e_loc[e];
          float r = a.r_csc[e];
          if (has_prev) {
            const float4* wp4 = (const float4*)(wprev + il * B);
#pragma unroll
            for (int q = 0; q < B / 4; ++q) {
              const float4 w4 = wp4[q];
              r = fmaf(w4.x, dl[4 * q + 0], r);
              r = fmaf(w4.y, dl[4 * q + 1], r);
              r = fmaf(w4.z, dl[4 * q + 2], r);
              r = fmaf(w4.w, dl[4 * q + 3], r);
            }
            a.r_csc[e] = r;
          }
          if (has_cur) {
            float wc[B];
            const float4* wc4 = (const float4*)(wcur + il * B);
#pragma unroll
            for (int q = 0; q < B / 4; ++q) {
              const float4 w4 = wc4[q];
              wc[4 * q + 0] = w4.x; wc[4 * q + 1] = w4.y; wc[4 * q + 2] = w4.z; wc[4 * q + 3] = w4.w;
            }
#pragma unroll
            for (int j = 0; j < B; ++j) {
              v[j] = fmaf(wc[j], r, v[j]);
#pragma unroll
              for (int l = 0; l <= j; ++l) v[L::gidx(j, l)] = fmaf(wc[j], wc[l], v[L::gidx(j, l)]);
            }
          }
        }
        if (has_cur) {
          warp_transpose_reduce<L::NP>(v, lane);
          if ((lane & 1) == 0) {
            constexpr int R = L::NP / 16;
            const int base = R * (((lane >> 4) & 1) * 8 + ((lane >> 3) & 1) * 4 + ((lane >> 2) & 1) * 2 +
                                  ((lane >> 1) & 1));
#pragma unroll
            for (int q = 0; q < R; ++q)
              if (base + q < L::NACC) acc[pe * L::NACC + base + q] += v[q];
          }
        }
      }
    }
    if (!has_cur) break;
    __syncthreads();
    float* mine = a.partials + (size_t)blockIdx.x * p * L::NACC;
    for (int t = threadIdx.x; t < p * L::NACC; t += blockDim.x) mine[t] = acc[t];
    __threadfence();
    grid_sync(a.bar);
    // distributed fixed-order reduction across CTAs
    const int nv = p * L::NACC;
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < nv; t += gridDim.x * blockDim.x) {
      double s = 0.0;
      for (int b = 0; b < (int)gridDim.x; ++b) s += (double)__ldcg(a.partials + (size_t)b * nv + t);
      a.reduced[t] = s;
    }
    __threadfence();
    grid_sync(a.bar);
    for (int t = threadIdx.x; t < nv; t += blockDim.x) red64[t] = __ldcg(a.reduced + t);
    __syncthreads();
    // sequential atom updates inside the block, identical in every CTA
    for (int pe = threadIdx.x; pe < p; pe += blockDim.x) {
      const double* rv = red64 + (size_t)pe * L::NACC;
      float dnew_l[B];
      for (int j = 0; j < nb; ++j) {
        const int k = k0 + j;
        double c = rv[j];
        for (int l = 0; l < j; ++l) c += rv[L::gidx(j, l)] * (double)dprev[l * p + pe];
        const double am = rv[L::gidx(j, j)];
        const double d_o = (double)dold[j * p + pe];
        const double lam = (double)p + geps * am;
        const double mu = geps * (c + d_o * am) / lam;
        double gdraw;
        if (a.draws) {
          gdraw = a.draws[(int64_t)k * p + pe];
        } else {
          const u32x4 rr = philox4x32_10(u32x4{(uint32_t)(pe >> 1), (uint32_t)k, (uint32_t)epoch, kDomAtom << 24},
                                         a.key0, a.key1);
          float n0, n1;
          box_muller(rr.x, rr.y, n0, n1);
          gdraw = (pe & 1) ? n1 : n0;
        }
        const float dn = (float)(mu + gdraw / sqrt(lam));
        dnew_l[j] = dn;
        dprev[j * p + pe] = dold[j * p + pe] - dn;   // becomes the next pass's shift
      }
      if (blockIdx.x == 0)
        for (int j = 0; j < nb; ++j) a.atoms[(int64_t)(k0 + j) * p + pe] = dnew_l[j];
      for (int j = nb; j < B; ++j) dprev[j * p + pe] = 0.0f;
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
static int sm_count_c() {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms;
}

static bool pick_compact(int cmax, int& c, int& g) {
  static const int kC[] = {8, 16, 24, 32};
  for (g = 1; g <= 32; g *= 2) {
    const int need = (cmax + g - 1) / g;
    for (int v : kC)
      if (v >= need) { c = v; return true; }
  }
  return false;
}

#define PB_DISPATCH_CG(c, g, MACRO)                                                                 \
  switch (c * 100 + g) {                                                                            \
    MACRO(8, 1) MACRO(16, 1) MACRO(24, 1) MACRO(32, 1) MACRO(24, 2) MACRO(32, 2) MACRO(24, 4)       \
    MACRO(32, 4) MACRO(24, 8) MACRO(32, 8) MACRO(32, 16) MACRO(32, 32)                              \
    default: set_error("unsupported compact layout c=%d g=%d", c, g); return PB_EUNSUPPORTED;       \
  }

static void normalize_cg(int& c, int& g) {
  // collapse to the instantiated set
  if (g >= 2 && c < 24) c = 24;
  if (g >= 16) c = 32;
}

int launch_resid_compact(const CompactArgs& a_in, cudaStream_t st) {
  CompactArgs a = a_in;
  int c, g;
  if (!pick_compact(a.cmax, c, g)) { set_error("patch has too many observed elements (%d)", a.cmax); return PB_EUNSUPPORTED; }
  normalize_cg(c, g);
  const int th = 256;
  a.kc = (int)((64 * 1024) / ((size_t)(a.p + 1) * 4));
  if (a.kc < 1) a.kc = 1;
  if (a.kc > a.k) a.kc = a.k;
  const size_t smem = (size_t)a.kc * (a.p + 1) * 4;
  const unsigned nb = (unsigned)ceil_div(a.n * g, th);
#define PB_R(C, GG)                                                                                 \
  case C * 100 + GG: {                                                                              \
    PB_CUDA_TRY(cudaFuncSetAttribute(k_resid_compact<C, GG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
    k_resid_compact<C, GG><<<nb, th, smem, st>>>(a);                                                \
    break;                                                                                          \
  }
  PB_DISPATCH_CG(c, g, PB_R)
#undef PB_R
  PB_LAUNCH_CHECK();
  return PB_OK;
}

int launch_code_compact(const CompactArgs& a_in, int mode, int& nblocks, cudaStream_t st) {
  CompactArgs a = a_in;
  int c, g;
  if (!pick_compact(a.cmax, c, g)) { set_error("patch has too many observed elements (%d)", a.cmax); return PB_EUNSUPPORTED; }
  normalize_cg(c, g);
  const int th = 256;
  a.kc = (int)((100 * 1024) / ((size_t)(a.p + 1) * 4));
  if (a.kc < 1) a.kc = 1;
  if (a.kc > a.k) a.kc = a.k;
  const size_t smem = (size_t)a.kc * (a.p + 1) * 4 + (size_t)a.k * 8;
  if (smem > 220 * 1024) { set_error("too many atoms for the code step (K=%d)", a.k); return PB_EUNSUPPORTED; }
  const unsigned nb = (unsigned)ceil_div(a.n * g, th);
  nblocks = (int)nb;
  PB_CUDA_TRY(cudaMemsetAsync(a.m_count, 0, (size_t)a.k * sizeof(int32_t), st));
#define PB_C(C, GG)                                                                                  \
  case C * 100 + GG: {                                                                               \
    auto kern = mode == kRngReplay ? k_code_compact<C, GG, kRngReplay> : k_code_compact<C, GG, kRngPhilox>; \
    PB_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
    kern<<<nb, th, smem, st>>>(a);                                                                   \
    break;                                                                                           \
  }
  PB_DISPATCH_CG(c, g, PB_C)
#undef PB_C
  PB_LAUNCH_CHECK();
  return PB_OK;
}

template <int B>
static int launch_dict_gram_b(DictGramArgs a, cudaStream_t st) {
  using L = GramLayout<B>;
  const int th = 256;
  const size_t wbytes = std::max((size_t)2 * kTile * B * 4, (size_t)a.p * L::NACC * 8);
  a.wbytes = (int)wbytes;
  const size_t smem = wbytes + (size_t)a.p * L::NACC * 4 + (size_t)2 * B * a.p * 4;
  if (smem > 225 * 1024) { set_error("patch size %d too large for the dictionary step", a.p); return PB_EUNSUPPORTED; }
  PB_CUDA_TRY(cudaFuncSetAttribute(k_dict_gram<B>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 0;
  PB_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_dict_gram<B>, th, smem));
  if (per_sm < 1) { set_error("dictionary step cannot be resident"); return PB_EUNSUPPORTED; }
  int blocks = sm_count_c() * per_sm;
  if (blocks > a.max_blocks) blocks = a.max_blocks;
  PB_CUDA_TRY(cudaMemsetAsync(a.bar, 0, 2 * sizeof(unsigned), st));
  void* args[] = {&a};
  PB_CUDA_TRY(cudaLaunchCooperativeKernel((const void*)k_dict_gram<B>, dim3(blocks), dim3(th), args, smem, st));
  return PB_OK;
}

int launch_dict_gram(const DictGramArgs& a, cudaStream_t st) { return launch_dict_gram_b<8>(a, st); }

size_t dict_gram_partials_bytes(int p, int max_blocks) {
  return (size_t)max_blocks * p * GramLayout<8>::NACC * 4;
}
size_t dict_gram_reduced_bytes(int p) { return (size_t)p * GramLayout<8>::NACC * 8; }

}  // namespace pb
