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
#include <type_traits>
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

// Float offset of 16-byte chunk h (0/1) of patch row il inside a tile block of
// the code copy W ([kTile][8] floats); see w_row_off (pb_index.cuh).
__device__ __forceinline__ int wsw(int il, int h) { return (int)((w_row_off(il) ^ (h << 4)) >> 2); }

template <int G>
__device__ __forceinline__ float gsum(float v) {
#pragma unroll
  for (int o = G >> 1; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ---------------------------------------------------------------------------
// Slot bookkeeping shared by the per-patch kernels: lane g of a G-lane group
// holds slots j*G + g of its patch; `wmax` is the warp-uniform number of slots
// any lane needs, so padded slots past it are skipped with uniform branches.
template <int G>
__device__ __forceinline__ int lane_slots(int cnt, int g) {
  return cnt > g ? (cnt - g + G - 1) / G : 0;
}

template <int CMAX, int G>
__global__ void __launch_bounds__(256) k_resid_compact(CompactArgs a) {
  extern __shared__ float ds[];
  const int pp = a.p + 1;
  const int g = threadIdx.x % G;
  const int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / G;
  const bool live = i < a.n;
  float acc[CMAX];
  int off[CMAX];
  int cnt = 0;
  int64_t r0 = 0;
  if (live) { cnt = a.counts[i]; r0 = a.rowptr[i]; }
  const int wmax = __reduce_max_sync(0xffffffffu, lane_slots<G>(cnt, g));
#pragma unroll
  for (int j = 0; j < CMAX; ++j) {
    off[j] = a.p;
    acc[j] = 0.0f;
    if (j < wmax) {
      const int s = j * G + g;
      if (s < cnt) {
        off[j] = a.csr_p[r0 + s];
        acc[j] = a.x_csc[a.csr_pos[r0 + s]];
      }
    }
  }
  const int64_t ic = live ? i : 0;
  for (int k0 = 0; k0 < a.k; k0 += a.kc) {
    const int kn = min(a.kc, a.k - k0);
    __syncthreads();
    stage_atoms(ds, a.atoms, k0, kn, a.p, pp);
    __syncthreads();
    for (int kb = 0; kb < kn; kb += 8) {
      // batch the (independent) code loads of 8 atoms before using any
      float wv[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int64_t zi = (int64_t)(k0 + min(kb + q, kn - 1)) * a.ld + ic;
        const uint8_t z = a.usage[zi];
        const float w = a.weights[zi];
        wv[q] = (live && kb + q < kn && z) ? -w : 0.0f;
      }
      if (a.wt && live && g == 0) {  // tile-blocked copy of w for the dictionary step
        float* blk = a.wt + ((i / kTile) * a.nblk8 + ((k0 + kb) >> 3)) * kTile * kWB;
        const int il = (int)(i % kTile);
        *(float4*)(blk + wsw(il, 0)) = make_float4(wv[0] != 0.f ? -wv[0] : 0.f, wv[1] != 0.f ? -wv[1] : 0.f,
                                                   wv[2] != 0.f ? -wv[2] : 0.f, wv[3] != 0.f ? -wv[3] : 0.f);
        *(float4*)(blk + wsw(il, 1)) = make_float4(wv[4] != 0.f ? -wv[4] : 0.f, wv[5] != 0.f ? -wv[5] : 0.f,
                                                   wv[6] != 0.f ? -wv[6] : 0.f, wv[7] != 0.f ? -wv[7] : 0.f);
      }
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        if (!__any_sync(0xffffffffu, wv[q] != 0.0f)) continue;
        const float* d = ds + (kb + q) * pp;
#pragma unroll
        for (int j = 0; j < CMAX; ++j)
          if (j < wmax) acc[j] = fmaf(wv[q], d[off[j]], acc[j]);
      }
    }
  }
  if (!live) return;
#pragma unroll
  for (int j = 0; j < CMAX; ++j) {
    const int s = j * G + g;
    if (j < wmax && s < cnt) a.r_csc[a.csr_pos[r0 + s]] = acc[j];
  }
}

// ---------------------------------------------------------------------------
// Code step (bpfa.py:240-275, atoms k = 0..K-1 in order, one patch per G-lane
// group).  D is staged in shared memory TRANSPOSED, DT[p][k] with row pitch KP =
// kc + 2 floats (KP/2 odd, so 8-byte loads from random rows spread over the
// banks; row P is all zero and backs the padded register slots).  One 8-byte load
// per slot then serves an atom PAIR, and one Philox4x32-10 block per pair gives
// both uniforms (x, y) and a Box-Muller normal pair (z, w); counter = (global
// patch, k/2, epoch | domain).  The kernel is persistent: D is staged once per
// CTA and the CTA walks patch blocks of blockDim/G.
// --- mbarrier + 1-D bulk async copy (TMA engine) helpers --------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}
// 16-byte shared load from a precomputed shared-window address (volatile: the
// staged tile is produced by the async proxy, keep it behind the mbarrier wait)
__device__ __forceinline__ float4 lds128(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr));
  return v;
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
// global -> shared bulk copy completing on an mbarrier (size and addresses 16-byte aligned)
__device__ __forceinline__ void bulk_copy_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

struct CodeConst {
  int64_t i, ic;
  bool live;
  int g, lane, epoch;
  float geps, gs, inv_sqrt_gs;
  const float* logit;
  int* mcnt;
  float* wrow;  // this patch's 8-atom window of w (pitch 8, XOR-swizzled by wx; lane g == 0 only)
  int wx;       // window swizzle: element q lives at wrow[q ^ wx] (conflict-free per-atom stores)
};

struct CodeThread {
  double sq_w;
  float sq_w8;  // philox mode: sum S^2 over the current 8-atom group
  int mc;       // lane j < 8: the warp's z count of atom kg + j in the current 8-atom group
};

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float lg2_approx(float x) {
  float y;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float rsqrt_approx(float x) {
  float y;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float sqrt_approx(float x) {
  float y;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// Box-Muller pair with the MUFU approximations (|err| ~ 1e-6, far below the
// sampler's statistical resolution).
__device__ __forceinline__ void box_muller_fast(uint32_t a, uint32_t b, float& n0, float& n1) {
  const float u1 = fmaf((float)a, 2.3283064365386963e-10f, 1.1641532182693481e-10f);
  const float rr = sqrt_approx(-1.3862943611198906f * lg2_approx(u1));  // sqrt(-2 ln u1)
  const float th = 6.283185307179586f * u01_24(b);
  float s, c;
  asm("sin.approx.ftz.f32 %0, %1;" : "=f"(s) : "f"(th));
  asm("cos.approx.ftz.f32 %0, %1;" : "=f"(c) : "f"(th));
  n0 = rr * c;
  n1 = rr * s;
}

// One atom's z/s draw from its moments u = |d|^2_obs, v = <d, r>_obs
// (_kernels.code_moments; G lanes: partial sums) (_code_params, bpfa.py:169-178
// and 262-269); dw = w_old - w_new is the residual shift (_kernels.shift_codes:
// r += dw * d), applied by the caller before code_commit writes the state.
struct CodeDraw {
  float dw, s_new, w_new;
  bool z;
};
template <int G, int MODE>
__device__ __forceinline__ CodeDraw code_draw(const CodeConst& c, int k, float u, float v, uint8_t z_old8, float s_old,
                                              float uu, float gn, double ud, double gd) {
  if (G > 1) {
    u = gsum<G>(u);
    v = gsum<G>(v);
  }
  const float w_old = z_old8 ? s_old : 0.0f;
  const float proj = fmaf(w_old, u, v);
  const float log_rho = c.logit[k] - 0.5f * c.geps * (s_old * s_old * u - 2.0f * s_old * proj);
  const float alpha = fmaf(c.geps, u, c.gs);
  bool z;
  float s_new;
  if (MODE == kRngReplay) {
    z = (log(ud) - log1p(-ud)) < (double)log_rho;  // bpfa.py:262-263
    const float g = (float)gd;
    s_new = z ? c.geps * proj / alpha + g / sqrtf(alpha) : g * c.inv_sqrt_gs;  // bpfa.py:265-269
  } else {
    z = uu * (1.0f + ex2_approx(-1.4426950408889634f * log_rho)) < 1.0f;  // U < sigmoid(log_rho)
    const float ra = rsqrt_approx(alpha);
    s_new = z ? fmaf(c.geps * proj, ra * ra, gn * ra) : gn * c.inv_sqrt_gs;
  }
  const float w_new = z ? s_new : 0.0f;
  return CodeDraw{w_old - w_new, s_new, w_new, z};
}

// The state write of one drawn atom (lane g == 0 of a patch) and the z count.
template <int MODE>
__device__ __forceinline__ void code_commit(const CompactArgs& a, const CodeConst& c, CodeThread& t, int k, int64_t zo,
                                            const CodeDraw& x) {
  const bool own = c.live && c.g == 0;
  if (own) {
    a.usage[zo] = x.z ? 1 : 0;
    a.weights[zo] = x.s_new;
    if (MODE == kRngReplay) t.sq_w += (double)x.s_new * (double)x.s_new;
    else t.sq_w8 = fmaf(x.s_new, x.s_new, t.sq_w8);
    c.wrow[(k & 7) ^ c.wx] = x.w_new;
  }
  // the warp's z count of atom k goes to lane k & 7's register; flushed to the
  // CTA's shared counts once per 8-atom group (code_atoms)
  const int nz = __popc(__ballot_sync(0xffffffffu, x.z && own));
  if (c.lane == (k & 7)) t.mc += nz;
}

// One atom over W slots of scalar column values d (multi-lane patches).
template <int CMAX, int W, int G, int MODE>
__device__ __forceinline__ void code_one(const CompactArgs& a, const CodeConst& c, CodeThread& t, int k, int64_t zo,
                                         const float (&d)[W], float (&r)[CMAX], uint8_t z_old8, float s_old,
                                         float uu, float gn, double ud, double gd) {
  float u = 0.0f, v = 0.0f;
#pragma unroll
  for (int j = 0; j < W; ++j) {
    u = fmaf(d[j], d[j], u);
    v = fmaf(d[j], r[j], v);
  }
  const CodeDraw x = code_draw<G, MODE>(c, k, u, v, z_old8, s_old, uu, gn, ud, gd);
#pragma unroll
  for (int j = 0; j < W; ++j) r[j] = fmaf(x.dw, d[j], r[j]);
  code_commit<MODE>(a, c, t, k, zo, x);
}

// One atom over W slots given as slot pairs (one lane per patch, W > 16):
// every multiply-add a packed FFMA2, u and v as even- and odd-slot partial sums.
template <int CMAX, int W, int G, int MODE>
__device__ __forceinline__ void code_one_sp(const CompactArgs& a, const CodeConst& c, CodeThread& t, int k,
                                            int64_t zo, const float2 (&d)[W / 2], float (&r)[CMAX],
                                            uint8_t z_old8, float s_old, float uu, float gn, double ud, double gd) {
  float2 u2 = make_float2(0.0f, 0.0f), v2 = make_float2(0.0f, 0.0f);
#pragma unroll
  for (int j = 0; j < W / 2; ++j) {
    u2 = __ffma2_rn(d[j], d[j], u2);
    v2 = __ffma2_rn(d[j], make_float2(r[2 * j], r[2 * j + 1]), v2);
  }
  const CodeDraw x = code_draw<G, MODE>(c, k, u2.x + u2.y, v2.x + v2.y, z_old8, s_old, uu, gn, ud, gd);
  const float2 dw2 = make_float2(x.dw, x.dw);
#pragma unroll
  for (int j = 0; j < W / 2; ++j) {
    const float2 rj = __ffma2_rn(dw2, d[j], make_float2(r[2 * j], r[2 * j + 1]));
    r[2 * j] = rj.x;
    r[2 * j + 1] = rj.y;
  }
  code_commit<MODE>(a, c, t, k, zo, x);
}

// Atoms [k0, k1) (k0 a multiple of 8) against the staged DT whose column 0 is
// atom kc0.  W = live register slots of this warp (compile time).
template <int CMAX, int W, int G, int MODE>
__device__ __forceinline__ void code_atoms(const CompactArgs& a, const CodeConst& c, CodeThread& t, int k0, int k1,
                                           const float* dt, float (&r)[CMAX], int (&addr)[CMAX]) {
  // addr[j]: byte offset of slot j's DT row + the current pair's column; it
  // advances by 8 per pair (no per-slot address arithmetic beyond that)
  constexpr bool kPair = W <= 16;            // register budget: 2W values of D per pair
  constexpr bool kSlotPair = !kPair && G == 1 && W <= 24;   // (W = 32: spills)
  int64_t zo = (int64_t)k0 * a.ld + c.ic;
  const bool ld_state = !a.codes_zero;   // all codes zero (fresh / warm-reset state): nothing to load
  uint8_t za = 0, zb = 0;
  float sa = 0.0f, sb = 0.0f;
  if (ld_state) { za = a.usage[zo]; sa = a.weights[zo]; }
  if (ld_state && k0 + 1 < a.k) { zb = a.usage[zo + a.ld]; sb = a.weights[zo + a.ld]; }
  for (int kg = k0; kg < k1; kg += 8) {
#pragma unroll 1
    for (int q = 0; q < 8; q += 2) {
      const int k = kg + q;
      if (k >= k1) break;
      // prefetch the next pair's state
      uint8_t zna = 0, znb = 0;
      float sna = 0.0f, snb = 0.0f;
      if (ld_state && k + 2 < a.k) { zna = a.usage[zo + 2 * a.ld]; sna = a.weights[zo + 2 * a.ld]; }
      if (ld_state && k + 3 < a.k) { znb = a.usage[zo + 3 * a.ld]; snb = a.weights[zo + 3 * a.ld]; }
      float uu0 = 0.f, uu1 = 0.f, g0 = 0.f, g1 = 0.f;
      double ud0 = 0.0, ud1 = 0.0, gd0 = 0.0, gd1 = 0.0;
      if (MODE == kRngReplay) {
        const int64_t di = (int64_t)k * a.n + c.ic;
        ud0 = a.u_draw[di];
        gd0 = a.g_draw[di];
        if (k + 1 < k1) { ud1 = a.u_draw[di + a.n]; gd1 = a.g_draw[di + a.n]; }
      } else {
        const int64_t gi = c.i + a.i_offset;  // global patch index: shards draw the 1-GPU streams
        const u32x4 rnd = philox4x32_10_rk(u32x4{(uint32_t)gi, (uint32_t)(gi >> 32), (uint32_t)(k >> 1),
                                                 ((uint32_t)c.epoch & 0xFFFFFFu) | (kDomCode << 24)},
                                           a.rk);
        box_muller_fast(rnd.z, rnd.w, g0, g1);
        uu0 = u01_24(rnd.x);
        uu1 = u01_24(rnd.y);
      }
      const char* col = (const char*)dt;
      if constexpr (kPair && G > 1) {
        float d0[W], d1[W];
#pragma unroll
        for (int j = 0; j < W; ++j) {
          const float2 dd = *(const float2*)(col + addr[j]);
          d0[j] = dd.x;
          d1[j] = dd.y;
        }
        code_one<CMAX, W, G, MODE>(a, c, t, k, zo, d0, r, za, sa, uu0, g0, ud0, gd0);
        if (k + 1 < k1) code_one<CMAX, W, G, MODE>(a, c, t, k + 1, zo + a.ld, d1, r, zb, sb, uu1, g1, ud1, gd1);
      } else if constexpr (kPair) {
        // both atoms' columns per slot in one 8-byte load; |d_k|^2 and |d_k+1|^2 as one FFMA2
        float2 dd[W];
        float2 u01 = make_float2(0.0f, 0.0f);
#pragma unroll
        for (int j = 0; j < W; ++j) {
          dd[j] = *(const float2*)(col + addr[j]);
          u01 = __ffma2_rn(dd[j], dd[j], u01);
        }
        float v = 0.0f;
#pragma unroll
        for (int j = 0; j < W; ++j) v = fmaf(dd[j].x, r[j], v);
        const CodeDraw x0 = code_draw<G, MODE>(c, k, u01.x, v, za, sa, uu0, g0, ud0, gd0);
#pragma unroll
        for (int j = 0; j < W; ++j) r[j] = fmaf(x0.dw, dd[j].x, r[j]);
        code_commit<MODE>(a, c, t, k, zo, x0);
        if (k + 1 < k1) {
          v = 0.0f;
#pragma unroll
          for (int j = 0; j < W; ++j) v = fmaf(dd[j].y, r[j], v);
          const CodeDraw x1 = code_draw<G, MODE>(c, k + 1, u01.y, v, zb, sb, uu1, g1, ud1, gd1);
#pragma unroll
          for (int j = 0; j < W; ++j) r[j] = fmaf(x1.dw, dd[j].y, r[j]);
          code_commit<MODE>(a, c, t, k + 1, zo + a.ld, x1);
        }
      } else if constexpr (kSlotPair) {
        float2 d0[W / 2];
#pragma unroll
        for (int j = 0; j < W / 2; ++j)
          d0[j] = make_float2(*(const float*)(col + addr[2 * j]), *(const float*)(col + addr[2 * j + 1]));
        code_one_sp<CMAX, W, G, MODE>(a, c, t, k, zo, d0, r, za, sa, uu0, g0, ud0, gd0);
        if (k + 1 < k1) {
#pragma unroll
          for (int j = 0; j < W / 2; ++j)
            d0[j] = make_float2(*(const float*)(col + 4 + addr[2 * j]), *(const float*)(col + 4 + addr[2 * j + 1]));
          code_one_sp<CMAX, W, G, MODE>(a, c, t, k + 1, zo + a.ld, d0, r, zb, sb, uu1, g1, ud1, gd1);
        }
      } else {
        float d0[W];
#pragma unroll
        for (int j = 0; j < W; ++j) d0[j] = *(const float*)(col + addr[j]);
        code_one<CMAX, W, G, MODE>(a, c, t, k, zo, d0, r, za, sa, uu0, g0, ud0, gd0);
        if (k + 1 < k1) {
#pragma unroll
          for (int j = 0; j < W; ++j) d0[j] = *(const float*)(col + 4 + addr[j]);
          code_one<CMAX, W, G, MODE>(a, c, t, k + 1, zo + a.ld, d0, r, zb, sb, uu1, g1, ud1, gd1);
        }
      }
#pragma unroll
      for (int j = 0; j < W; ++j) addr[j] += 8;
      za = zna; zb = znb; sa = sna; sb = snb;
      zo += 2 * a.ld;
    }
    // group done: flush the z counts, the tile-blocked copy of w for the
    // dictionary step, sum S^2
    if (c.lane < 8 && t.mc) atomicAdd(&c.mcnt[kg + c.lane], t.mc);
    t.mc = 0;
    if (c.live && c.g == 0) {
      if (MODE != kRngReplay) { t.sq_w += (double)t.sq_w8; t.sq_w8 = 0.0f; }
      float* wrow = c.wrow;
      for (int q = k1 - kg; q < 8; ++q) wrow[q ^ c.wx] = 0.0f;  // partial last group
      float* blk = a.wt + ((c.i / kTile) * a.nblk8 + (kg >> 3)) * kTile * kWB;
      const int il = (int)(c.i % kTile);
      const int x = c.wx;
      *(float4*)(blk + wsw(il, 0)) = make_float4(wrow[0 ^ x], wrow[1 ^ x], wrow[2 ^ x], wrow[3 ^ x]);
      *(float4*)(blk + wsw(il, 1)) = make_float4(wrow[4 ^ x], wrow[5 ^ x], wrow[6 ^ x], wrow[7 ^ x]);
    }
  }
}

// Stage chunk `ci` of the pre-packed transposed dictionary (k_pack_dt): a
// plain 16-byte vector copy (no index arithmetic; the image is L2-resident).
// The caller synchronizes the CTA before (previous contents consumed) and after.
__device__ __forceinline__ void stage_dt_chunk(float* dt, const CompactArgs& a, int ci) {
  const float4* __restrict__ src = (const float4*)(a.dt_img + (int64_t)ci * a.dt_img_floats);
  float4* dst = (float4*)dt;
  const int n4 = (int)(a.dt_img_floats >> 2);
#pragma unroll 4
  for (int t = threadIdx.x; t < n4; t += blockDim.x) dst[t] = __ldg(src + t);
}

// The same chunk through cp.async (global -> shared without registers): the
// multi-lane (G > 1) variants, whose register allocation the vector-copy path
// perturbs into spills, and which restage every chunk per block of patches when
// D does not fit (the cube: K = 512, P = 256).  Caller synchronizes as above.
__device__ __forceinline__ void stage_dt_chunk_async(float* dt, const CompactArgs& a, int ci) {
  const float4* __restrict__ src = (const float4*)(a.dt_img + (int64_t)ci * a.dt_img_floats);
  const uint32_t dst = smem_u32(dt);
  const int n4 = (int)(a.dt_img_floats >> 2);
  for (int t = threadIdx.x; t < n4; t += blockDim.x)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + 16u * t), "l"(src + t) : "memory");
  asm volatile("cp.async.wait_all;" ::: "memory");
}

template <int CMAX, int W, int G, int MODE>
__device__ __forceinline__ void code_patch_range(const CompactArgs& a, const CodeConst& c, CodeThread& t, float* dt,
                                                 int kp, float (&r)[CMAX], int (&addr)[CMAX]) {
  if (a.kc >= a.k) {
    code_atoms<CMAX, W, G, MODE>(a, c, t, 0, a.k, dt, r, addr);
  } else {
    for (int k0 = 0; k0 < a.k; k0 += a.kc) {
      const int kn = min(a.kc, a.k - k0);
      __syncthreads();
      if constexpr (G == 1) stage_dt_chunk(dt, a, k0 / a.kc);
      else stage_dt_chunk_async(dt, a, k0 / a.kc);
      __syncthreads();
      code_atoms<CMAX, W, G, MODE>(a, c, t, k0, k0 + kn, dt, r, addr);
#pragma unroll
      for (int j = 0; j < W; ++j) addr[j] -= 4 * ((kn + 1) & ~1);  // back to column 0
    }
  }
}

// WS: pitch-8 XOR-swizzled w windows (1 KB less shared memory per CTA than the
// pitch-9 rows: lets the whole D of configs[1] fit two CTAs per SM)
// WC: every warp claims its own blocks of 32 patches (whole D staged once: no
// CTA barrier in the loop, warps of different slot counts never wait for each other)
template <int CMAX, int G, int MODE, bool WS, bool WC>
__global__ void __launch_bounds__(256, 2) k_code_compact(CompactArgs a) {
  extern __shared__ __align__(16) float sm[];
  const int kp = a.kc + 2;                     // DT row pitch (kc % 8 == 0  =>  kp/2 odd)
  float* dt = sm;                              // (P+1) * kp
  float* logit = dt + a.dt_img_floats;         // K (after the DT chunk)
  int* mcnt = (int*)(logit + a.k);             // K
  float* wwin = (float*)(mcnt + a.k);          // (blockDim / G) * (WS ? 8 : 9)
  __shared__ double red[32];
  __shared__ long long next_blk;
  CodeConst c;
  c.g = threadIdx.x % G;
  c.lane = threadIdx.x & 31;
  c.epoch = a.sc->epoch + 1;
  c.geps = (float)a.sc->gamma_eps;
  c.gs = (float)a.sc->gamma_s;
  c.inv_sqrt_gs = (float)(1.0 / sqrt(a.sc->gamma_s));
  c.logit = logit;
  c.mcnt = mcnt;
  c.wrow = wwin + (threadIdx.x / G) * (WS ? 8 : 9);
  c.wx = WS ? ((threadIdx.x / G) >> 2) & 7 : 0;   // constant 0 folds the XORs away
  for (int k = threadIdx.x; k < a.k; k += blockDim.x) {
    const double pk = fmin(fmax(a.pi[k], 1e-15), 1.0 - 1e-15);  // bpfa.py:173
    logit[k] = (float)(log(pk) - log1p(-pk));
    mcnt[k] = 0;
  }
  if (a.kc >= a.k) {
    if constexpr (G == 1) stage_dt_chunk(dt, a, 0);
    else stage_dt_chunk_async(dt, a, 0);
  }
  __syncthreads();
  const int row_bytes = kp * 4;
  CodeThread t;
  t.sq_w8 = 0.0f;
  t.mc = 0;
  const int per_blk = WC ? 32 / G : blockDim.x / G;
  const int64_t nblk = ceil_div(a.plist ? a.plist_n : a.n, per_blk);
  // blocks of patches are claimed dynamically (the launch may share the GPU with
  // a concurrent one); each block writes its own S^2 / R^2 sums, summed later in
  // block order, so the result does not depend on which CTA took which block
  for (;;) {
    int64_t b;
    if constexpr (WC) {
      unsigned v = 0;
      if (c.lane == 0) v = atomicAdd(a.blk_ctr, 1u);
      b = __shfl_sync(0xffffffffu, v, 0);
    } else {
      __syncthreads();
      if (threadIdx.x == 0) next_blk = (long long)atomicAdd(a.blk_ctr, 1u);
      __syncthreads();
      b = next_blk;
    }
    if (b >= nblk) break;
    t.sq_w = 0.0;
    double sq_r = 0.0;
    const int64_t slot = b * per_blk + (WC ? c.lane : (int)threadIdx.x) / G;
    if (a.plist) {  // second launch of a split: exactly the listed (wide) patches
      c.live = slot < a.plist_n;
      c.i = c.live ? a.plist[slot] : 0;
    } else {
      c.i = slot;
      c.live = c.i < a.n;
    }
    float r[CMAX];
    int addr[CMAX];
    int cnt = 0;
    int64_t r0 = 0;
    if (c.live) {
      cnt = a.counts[c.i];
      if (a.split && cnt > a.split) { c.live = false; cnt = 0; }  // handled by the second launch
      else r0 = a.rowptr[c.i];
    }
    c.ic = c.live ? c.i : 0;
    const int wmax = __reduce_max_sync(0xffffffffu, lane_slots<G>(cnt, c.g));
#pragma unroll
    for (int j = 0; j < CMAX; ++j) {
      addr[j] = a.p * row_bytes;
      r[j] = 0.0f;
      if (j < wmax) {
        const int s = j * G + c.g;
        if (s < cnt) {
          addr[j] = (int)a.csr_p[r0 + s] * row_bytes;
          r[j] = a.r_csc[a.csr_pos[r0 + s]];
        }
      }
    }
    // the warp's live slot count as a compile-time constant (no padded-slot work)
    const int wc = (wmax + 7) & ~7;
    if (wc <= 8 || CMAX == 8) code_patch_range<CMAX, (CMAX < 8 ? CMAX : 8), G, MODE>(a, c, t, dt, kp, r, addr);
    else if (wc <= 16 || CMAX == 16) code_patch_range<CMAX, (CMAX < 16 ? CMAX : 16), G, MODE>(a, c, t, dt, kp, r, addr);
    else if (wc <= 24 || CMAX == 24) code_patch_range<CMAX, (CMAX < 24 ? CMAX : 24), G, MODE>(a, c, t, dt, kp, r, addr);
    else code_patch_range<CMAX, CMAX, G, MODE>(a, c, t, dt, kp, r, addr);
#pragma unroll
    for (int j = 0; j < CMAX; ++j) {
      sq_r += (double)r[j] * (double)r[j];
      // the end-of-sweep residual is the next epoch's starting residual (carry mode)
      const int s = j * G + c.g;
      if (c.live && j < wmax && s < cnt) a.r_csc[a.csr_pos[r0 + s]] = r[j];
    }
    if constexpr (WC) {
      const double bw = warp_sum_d(t.sq_w), br = warp_sum_d(sq_r);
      if (c.lane == 0) {
        a.block_sums[2 * b] = bw;
        a.block_sums[2 * b + 1] = br;
      }
    } else {
      const double bw = block_sum_d(t.sq_w, red);
      __syncthreads();
      const double br = block_sum_d(sq_r, red);
      if (threadIdx.x == 0) {
        a.block_sums[2 * b] = bw;
        a.block_sums[2 * b + 1] = br;
      }
    }
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

// Monotonic-counter grid barrier: every CTA adds 1 with a release reduction
// (no returned value to wait for, no reset) and polls until the counter reaches
// the next multiple of the grid size.  bar[0] is zeroed before the launch.
__device__ __forceinline__ void grid_sync_mono(unsigned* bar, unsigned& target) {
  __syncthreads();
  target += gridDim.x;
  if (threadIdx.x == 0) {
    __threadfence();
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
    while (ld_acquire(bar) < target) __nanosleep(32);
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

// Packed FMA on the aligned accumulator pair (v[2i], v[2i+1]) += a * b (FFMA2).
template <int NP>
__device__ __forceinline__ void pfma(float (&v)[NP], int i, float2 a, float2 b) {
  const float2 c = __ffma2_rn(a, b, make_float2(v[2 * i], v[2 * i + 1]));
  v[2 * i] = c.x;
  v[2 * i + 1] = c.y;
}

// Transpose reduction of NP per-lane values inside groups of S lanes (S | 32):
// afterwards lane `sub` of a group holds the group sums of values
// [base, base + NP/S) with base = sum over levels o = S/2..1 of (sub & o ? half : 0).
template <int NP, int S>
__device__ __forceinline__ void group_transpose_reduce(float (&v)[NP], int sub) {
  constexpr int LV = S == 2 ? 1 : S == 4 ? 2 : S == 8 ? 3 : S == 16 ? 4 : 5;
  static_assert(NP % S == 0, "NP must be a multiple of the group size");
#pragma unroll
  for (int lvl = 0; lvl < LV; ++lvl) {
    const int o = (S / 2) >> lvl;
    const int half = NP >> (lvl + 1);
    const bool lo = (sub & o) == 0;
#pragma unroll
    for (int q = 0; q < half; ++q) {
      const float send = lo ? v[half + q] : v[q];
      const float keep = lo ? v[q] : v[half + q];
      v[q] = keep + __shfl_xor_sync(0xffffffffu, send, o);
    }
  }
}

// Accumulator layout of one atom block (B even): C_0..C_{B-1}, then per row j
// of the Gram triangle the PAIRS (G_j,2m, G_j,2m+1) for 2m <= j — every update
// is a packed f32x2 FMA (FFMA2) of the broadcast w_j with the aligned pair
// (w_2m, w_2m+1) as loaded; G_jj = A_j.  Even rows carry one redundant entry
// (G_j,j+1, also in row j+1) so that no operand pair has to be assembled.
template <int B>
struct GramLayout {
  static_assert(B % 2 == 0, "pair layout needs an even block");
  __host__ __device__ static constexpr int pairbase(int j) { return j + (j / 2) * ((j - 1) / 2); }
  static constexpr int NACC = B + 2 * pairbase(B);
  static constexpr int NP = ((NACC + 15) / 16) * 16;    // padded for the transpose reduce
  __host__ __device__ static constexpr int gidx(int j, int l) { return B + 2 * (pairbase(j) + l / 2) + (l & 1); }
};
static_assert(GramLayout<8>::NACC == 48 && GramLayout<8>::NP == 48, "layout of the 8-atom block");

// L2 residency hints: the dictionary step re-reads the residual and the element
// index in every one of its K/8+1 passes (61 MB at configs[1], L2 is 126 MB)
// while the code copy W streams through (each block is read twice: as the
// current block, then as the previous block of the next pass).
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ float ldg_hint(const float* p, uint64_t pol) {
  float v;
  asm volatile("ld.global.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ uint16_t ldg_hint(const uint16_t* p, uint64_t pol) {
  uint16_t v;
  asm volatile("ld.global.L2::cache_hint.u16 %0, [%1], %2;" : "=h"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ void stg_hint(float* p, float v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.f32 [%0], %1, %2;" ::"l"(p), "f"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ void bulk_copy_g2s_hint(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                                   uint64_t pol) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol) : "memory");
}

__device__ __forceinline__ uint64_t gtimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// Dictionary step, persistent & cooperative (all CTAs co-resident).
//
// Work split (exactly balanced for any mask structure, deterministic):
//   CTA c owns the element range [nnz*c/G, nnz*(c+1)/G) of the CSC-tile order;
//   per tile it stages w = z*s of the previous and current atom blocks, then
//   warp w of the CTA owns an equal contiguous slice of the tile's elements.
//   A warp walks the columns its slice touches; lanes take every 32nd element
//   of each column segment (coalesced), accumulate the NACC Gram/moment sums in
//   registers, and transpose-reduce them at the end of the segment.  Segments
//   wholly owned by one warp add straight into the CTA accumulator; the (at
//   most two) boundary segments go to per-warp slots merged in warp order.

// The B sequential atom draws of one block from the reduced moments (f64):
//   C_j += sum_{l<j} G_jl o delta_l;  lambda = P + geps*A_j;  mu = geps*(C_j + d_j*A_j)/lambda;
//   d_j' = mu + g/sqrt(lambda)  (bpfa.py:161-166, 303-307).  Identical in every CTA/rank.
// The B sequential atom draws of one block at ONE pixel pe from its reduced
// moments rv[NACC] (f64):
//   C_j += sum_{l<j} G_jl delta_l;  lambda = P + geps*A_j;  mu = geps*(C_j + d_j*A_j)/lambda;
//   d_j' = mu + g/sqrt(lambda)  (bpfa.py:161-166, 303-307);  delta_j = d_j - d_j' (f32).
template <int B>
__device__ __forceinline__ double atom_draw(const double* draws, int pe, int p, int k, int epoch, uint32_t key0,
                                            uint32_t key1) {
  if (draws) return draws[(int64_t)k * p + pe];
  const u32x4 rr = philox4x32_10(u32x4{(uint32_t)(pe >> 1), (uint32_t)k, (uint32_t)epoch, kDomAtom << 24}, key0, key1);
  float n0, n1;
  box_muller(rr.x, rr.y, n0, n1);
  return (pe & 1) ? n1 : n0;
}

// Per-atom quantities of the draw that do not depend on the earlier atoms'
// shifts (computable in parallel): 1/lambda, 1/sqrt(lambda), A_j, d_j(old), g.
struct AtomPre {
  double inv, rs, am, d_o, g;
};

template <int B>
__device__ __forceinline__ AtomPre atom_pre(const double* rv, int j, int pe, int p, int k0, double geps, int epoch,
                                            const double* draws, uint32_t key0, uint32_t key1, const float* dold) {
  using L = GramLayout<B>;
  AtomPre r;
  r.am = rv[L::gidx(j, j)];
  const double lam = (double)p + geps * r.am;
  r.rs = rsqrt(lam);   // 1/sqrt(lambda); 1/lambda = rs^2
  r.inv = r.rs * r.rs;
  r.d_o = (double)dold[j * p + pe];
  r.g = atom_draw<B>(draws, pe, p, k0 + j, epoch, key0, key1);
  return r;
}

// The sequential part: C_j corrected by the shifts of atoms < j, the posterior
// mean and the draw d_j' = mu + g/sqrt(lambda).
template <int B>
__device__ __forceinline__ float atom_chain_step(const double* rv, int j, const AtomPre& pr, const double (&dl)[B],
                                                 double geps) {
  using L = GramLayout<B>;
  double c = rv[j];
#pragma unroll
  for (int l = 0; l < B; ++l)
    if (l < j) c += rv[L::gidx(j, l)] * dl[l];
  const double mu = geps * (c + pr.d_o * pr.am) * pr.inv;
  return (float)(mu + pr.g * pr.rs);
}

// One thread: the B sequential atom draws of one block at pixel pe.
template <int B>
__device__ __forceinline__ void atom_pixel_update(const double* rv, int pe, int p, int k0, int nb, double geps,
                                                  int epoch, const double* draws, uint32_t key0, uint32_t key1,
                                                  const float* dold, float* atoms_out, float* dsh, float* delta_out,
                                                  const AtomPre* pre = nullptr) {
  // dsh: [B][p] shifts of this block, delta_out: optional global copy, pre: optional precomputed [B]
  double dl[B];
#pragma unroll
  for (int j = 0; j < B; ++j) {
    dl[j] = 0.0;
    if (j >= nb) {
      dsh[j * p + pe] = 0.0f;
      if (delta_out) delta_out[j * p + pe] = 0.0f;
      continue;
    }
    const AtomPre pr = pre ? pre[j] : atom_pre<B>(rv, j, pe, p, k0, geps, epoch, draws, key0, key1, dold);
    const float dn = atom_chain_step<B>(rv, j, pr, dl, geps);
    if (atoms_out) atoms_out[(int64_t)(k0 + j) * p + pe] = dn;
    const float dd = (float)pr.d_o - dn;   // the next pass's shift (d_o: the old atom, read before the write)
    dsh[j * p + pe] = dd;
    if (delta_out) delta_out[j * p + pe] = dd;
    dl[j] = (double)dd;
  }
}

template <int B>
__device__ __forceinline__ void atom_block_update(const double* red, int p, int k0, int nb, double geps, int epoch,
                                                  const double* draws, uint32_t key0, uint32_t key1,
                                                  const float* dold, float* dprev, float* atoms_out) {
  using L = GramLayout<B>;
  for (int pe = threadIdx.x; pe < p; pe += blockDim.x)
    atom_pixel_update<B>(red + (size_t)pe * L::NACC, pe, p, k0, nb, geps, epoch, draws, key0, key1, dold, atoms_out,
                         dprev, nullptr);
}

constexpr double kTileVisitCost = 500.0;   // ELL positions equivalent to one tile visit (work split; 3000: live +2 %)
// Byte stride of one staged W block in shared memory: the tile's kTile x 8
// floats, then the all-zero row kEllZeroRow that the ELL padding points to.
constexpr uint32_t kWStride = (uint32_t)kTile * kWB * 4 + 128;
constexpr int kEllPf = 5;   // elements per chunk / in flight per lane in the element phase (measured 2..8: 4-5 best; 8: +6 %)
constexpr int kEllTail = kEllPf;   // granularity of the element loop's exit: whole chunks (see ell_elements; 1: +6-40 %)

// One ELL wave (pb_index.cu) as seen by a lane: its run's column, the wave's
// run length, log2 of the lanes per column, and the lane's first position.
struct EllWave {
  int lw, lg, col;
  int64_t base;
};

__device__ __forceinline__ EllWave ell_header(const DictGramArgs& a, int64_t wv, int64_t tile_ell, int lane) {
  EllWave h;
  const int meta = a.wave_meta[wv];
  h.lw = meta & 0xFF;
  h.lg = meta >> 8;
  h.col = a.wave_col[wv * 32 + lane];
  h.base = tile_ell + a.wave_off[wv] + lane;
  return h;
}

// the first kEllPf positions of a wave's run in flight
__device__ __forceinline__ void ell_prefetch(const DictGramArgs& a, const EllWave& h, uint32_t (&ib)[kEllPf],
                                             float (&rb)[kEllPf], uint64_t pol) {
#pragma unroll
  for (int d = 0; d < kEllPf; ++d) {
    ib[d] = kEllZeroRow;
    rb[d] = 0.0f;
    if (d < h.lw) { ib[d] = ldg_hint(a.e_ell + h.base + d * 32, pol); rb[d] = ldg_hint(a.r_csc + h.base + d * 32, pol); }
  }
}

// 16-byte shared load the compiler may schedule freely (not volatile): the
// address must derive from a value produced after the mbarrier wait that
// guards the staged data (see ell_stage_addr), so it cannot be hoisted above it
__device__ __forceinline__ float4 lds128_nv(uint32_t addr) {
  float4 v;
  asm("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr));
  return v;
}
// the stage's shared address, re-derived after the mbarrier wait (opaque copy)
__device__ __forceinline__ uint32_t ell_stage_addr(uint32_t a) {
  uint32_t r;
  asm volatile("mov.u32 %0, %1;" : "=r"(r) : "r"(a) : "memory");
  return r;
}

// compile-time loop: f(integral_constant<int, 0>) ... f(integral_constant<int, N-1>)
template <int N, int I = 0, typename F>
__device__ __forceinline__ void static_for(F&& f) {
  if constexpr (I < N) {
    f(std::integral_constant<int, I>{});
    static_for<N, I + 1>(f);
  }
}

// Loads / stores at a compile-time byte offset from a base register ([reg+imm]
// addressing: no per-element address arithmetic in the unrolled element loop).
template <int OFF>
__device__ __forceinline__ uint16_t ldg_u16_off(const uint16_t* p, uint64_t pol) {
  uint16_t v;
  asm volatile("ld.global.L2::cache_hint.u16 %0, [%1+%3], %2;" : "=h"(v) : "l"(p), "l"(pol), "n"(OFF));
  return v;
}
template <int OFF>
__device__ __forceinline__ float ldg_f32_off(const float* p, uint64_t pol) {
  float v;
  asm volatile("ld.global.L2::cache_hint.f32 %0, [%1+%3], %2;" : "=f"(v) : "l"(p), "l"(pol), "n"(OFF));
  return v;
}
template <int OFF>
__device__ __forceinline__ void stg_f32_off(float* p, float v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.f32 [%0+%3], %1, %2;" ::"l"(p), "f"(v), "l"(pol), "n"(OFF) : "memory");
}
template <int OFF>
__device__ __forceinline__ float4 lds128_off(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4+%5];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr), "n"(OFF));
  return v;
}

// Element phase of one ELL wave: the lane walks its run of column h.col (stride
// 32, coalesced), applies the previous block's shifts to the residual and
// accumulates the block's Gram / moment sums in registers.  Padding positions
// point at the zero W row and carry r = 0: no per-element tests beyond the
// wave's length.  The previous block's W is staged kWStride bytes after the
// current one.
#ifndef PB_ELL_LDS_VOLATILE
#define LDS_W lds128_nv
#else
#define LDS_W lds128
#endif
template <bool HP, bool HC>
__device__ __forceinline__ void ell_elements(const DictGramArgs& a, const EllWave& h, uint32_t wcur_s,
                                             const float2 (&dl2)[kWB / 2], float (&v)[GramLayout<kWB>::NP],
                                             uint32_t (&ib)[kEllPf], float (&rb)[kEllPf], uint64_t pol) {
  using L = GramLayout<kWB>;
  constexpr int B = kWB;
  const uint32_t wprev_s = wcur_s + kWStride;
  // chunk base pointers (advanced once per kEllPf positions): the unrolled
  // accesses below are [base + immediate]
  const uint16_t* __restrict__ ep = a.e_ell + h.base;
  float* __restrict__ rp = a.r_csc + h.base;
  const int lw = h.lw;
  for (int j0 = 0; j0 < lw; j0 += kEllPf, ep += kEllPf * 32, rp += kEllPf * 32) {
    const int more = lw - j0 - kEllPf;   // positions left after this chunk
#pragma unroll
    for (int d = 0; d < kEllPf; ++d) {
      // the wave's last chunk runs to a multiple of kEllTail positions: positions past
      // lw run on the zero W row with r = 0 (no effect on the sums) and store nothing
      // (fewer exits from the unrolled chunk: no accumulator copies at the joins)
      if (d % kEllTail == 0 && j0 + d >= lw) break;
      const bool real = kEllTail == 1 || j0 + d < lw;
      const uint32_t il = ib[d];
      float r = rb[d];
      if (d < more) {
        ib[d] = __ldg(ep + (kEllPf + d) * 32);
        rb[d] = rp[(kEllPf + d) * 32];
      } else if (kEllTail > 1) {
        ib[d] = kEllZeroRow;
        rb[d] = 0.0f;
      }
      const uint32_t wo[2] = {il, il ^ 16u};
      if constexpr (HP) {  // r += w_prev . delta  (packed pairs, two independent chains)
        float2 sh[B / 4];
#pragma unroll
        for (int q = 0; q < B / 4; ++q) {
          const float4 w4 = LDS_W(wprev_s + wo[q]);
          sh[q] = __fmul2_rn(make_float2(w4.x, w4.y), dl2[2 * q]);
          sh[q] = __ffma2_rn(make_float2(w4.z, w4.w), dl2[2 * q + 1], sh[q]);
        }
#pragma unroll
        for (int q = 0; q < B / 4; ++q) r += sh[q].x + sh[q].y;
        if (real) rp[d * 32] = r;
      }
      if constexpr (HC) {
        float wc[B];
#pragma unroll
        for (int q = 0; q < B / 4; ++q) {
          const float4 w4 = LDS_W(wcur_s + wo[q]);
          wc[4 * q + 0] = w4.x; wc[4 * q + 1] = w4.y; wc[4 * q + 2] = w4.z; wc[4 * q + 3] = w4.w;
        }
        const float2 rr2 = make_float2(r, r);
#pragma unroll
        for (int q = 0; q < B / 2; ++q) pfma(v, q, make_float2(wc[2 * q], wc[2 * q + 1]), rr2);  // C
#pragma unroll
        for (int jj = 0; jj < B; ++jj) {   // Gram pairs (G_jj,2m, G_jj,2m+1)
          const float2 wj = make_float2(wc[jj], wc[jj]);
#pragma unroll
          for (int m = 0; 2 * m <= jj; ++m) pfma(v, L::gidx(jj, 2 * m) / 2, wj, make_float2(wc[2 * m], wc[2 * m + 1]));
        }
      }
    }
  }
}

// The R = 2^lg runs of each column (lanes [R*g, R*g + R)) combine their sums
// (transpose reduction inside the group) and add the column's totals to the
// accumulator; each column sits in exactly one wave per tile.
// Accumulator rows of 44 floats (ACS = 44) drop the four redundant Gram entries
// G_j,j+1 (even j) of the 48-value register layout; ACS = 48 keeps the layout.
__host__ __device__ constexpr bool gram_redundant(int i) { return i == 9 || i == 15 || i == 25 || i == 39; }
__host__ __device__ constexpr int gram_compact(int i) { return i - (i > 9) - (i > 15) - (i > 25) - (i > 39); }
static_assert(GramLayout<8>::gidx(0, 1) == 9 && GramLayout<8>::gidx(2, 3) == 15 && GramLayout<8>::gidx(4, 5) == 25 &&
              GramLayout<8>::gidx(6, 7) == 39, "redundant entries of the 8-atom Gram layout");
template <int ACS>
__device__ __forceinline__ void ell_flush(float (&v)[GramLayout<kWB>::NP], int lg, int col, int lane, float* acc) {
  using L = GramLayout<kWB>;
  auto flush = [&](auto s_c) {
    constexpr int S = decltype(s_c)::value;
    constexpr int SG = S > 16 ? 16 : S;
    if constexpr (SG > 1) group_transpose_reduce<L::NP, SG>(v, lane & (SG - 1));
    constexpr int R = L::NP / SG;
    if constexpr (S == 32) {
#pragma unroll
      for (int q = 0; q < R; ++q) v[q] += __shfl_xor_sync(0xffffffffu, v[q], 16);
    }
    int vb = 0;
    {
      int cnt = L::NP;
#pragma unroll
      for (int o = SG / 2; o >= 1; o >>= 1) { cnt >>= 1; if (lane & o) vb += cnt; }
    }
    if (col != 0xFFFF && (S < 32 || lane < 16)) {
      if constexpr (ACS == L::NACC) {
        float* dst = acc + col * L::NACC + vb;
#pragma unroll
        for (int q = 0; q < R; ++q)
          if (vb + q < L::NACC) dst[q] += v[q];
      } else {
        float* dst = acc + col * ACS;
#pragma unroll
        for (int q = 0; q < R; ++q) {
          const int i = vb + q;
          if (i < L::NACC && !gram_redundant(i)) dst[gram_compact(i)] += v[q];
        }
      }
    }
  };
  switch (lg) {
    case 0: flush(std::integral_constant<int, 1>{}); break;
    case 1: flush(std::integral_constant<int, 2>{}); break;
    case 2: flush(std::integral_constant<int, 4>{}); break;
    case 3: flush(std::integral_constant<int, 8>{}); break;
    case 4: flush(std::integral_constant<int, 16>{}); break;
    default: flush(std::integral_constant<int, 32>{}); break;
  }
}

// The CTA's wave range [w_lo, w_hi) and tiles [t_lo, t_hi): ELL positions +
// kTileVisitCost per tile visited balanced over the grid (static, deterministic),
// boundaries snapped to wave starts.
__device__ __forceinline__ void ell_cta_range(const DictGramArgs& a, int64_t& w_lo, int64_t& w_hi, int& t_lo,
                                              int& t_hi) {
  const double tvc = a.tile_cost;
  const double total_cost = (double)a.ell_base[a.ntiles] + tvc * a.ntiles;
  auto cost_at = [&](int t) { return (double)a.ell_base[t] + tvc * t; };
  auto boundary = [&](int c) -> int64_t {
    if (c <= 0) return 0;
    if (c >= (int)gridDim.x) return a.wave_base[a.ntiles];
    const double target = total_cost * c / gridDim.x;
    int lo = 0, hi = a.ntiles - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (cost_at(mid) <= target) lo = mid; else hi = mid - 1;
    }
    const double over = target - cost_at(lo) - tvc;
    const int64_t w0 = a.wave_base[lo], w1 = a.wave_base[lo + 1];
    if (over <= 0.0 || w1 == w0) return w0;
    int64_t wl = w0, wh = w1 - 1;   // last wave starting at or before `over`
    while (wl < wh) {
      const int64_t mid = (wl + wh + 1) >> 1;
      if ((double)a.wave_off[mid] <= over) wl = mid; else wh = mid - 1;
    }
    // the nearer of that wave's start and the next boundary (next wave or tile end)
    if (a.split_nearest) {
      const double nxt = wl + 1 < w1 ? (double)a.wave_off[wl + 1] : (double)(a.ell_base[lo + 1] - a.ell_base[lo]);
      if (nxt - over < over - (double)a.wave_off[wl]) return wl + 1;
    }
    return wl;
  };
  const int cr = PB_DBG(a, 32) ? (int)gridDim.x - 1 - (int)blockIdx.x : (int)blockIdx.x;   // (tuning: reversed ranges)
  w_lo = boundary(cr);
  w_hi = boundary(cr + 1);
  t_lo = 0;
  t_hi = 0;
  if (w_hi > w_lo) {
    int lo = 0, hi = a.ntiles - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (a.wave_base[mid] <= w_lo) lo = mid; else hi = mid - 1;
    }
    t_lo = lo;
    t_hi = t_lo;
    while (t_hi < a.ntiles && a.wave_base[t_hi] < w_hi) ++t_hi;
  }
}

// Cross-CTA reduction distributed by PIXEL (after grid barrier 1): CTA c owns
// pixels c, c+G, ...; each value of a pixel is summed over the G per-CTA
// partials in a fixed order (f64, deterministic) and the owner performs that
// pixel's B sequential atom draws right away (pixels are independent).
template <int NW>
__device__ __forceinline__ void dict_owner_phase(const DictGramArgs& a, unsigned char* smraw, uint64_t* pbar,
                                                 uint32_t& pphase, int k0, int nb, double geps, int epoch,
                                                 const float* dold, float* dprev) {
  using L = GramLayout<kWB>;
  constexpr int B = kWB;
  const int p = a.p;
  double* red64 = (double*)smraw;                        // p * NACC (aliases the staging)
  auto ld_part = [&](const float* q) -> float { return a.pstage_off ? *q : __ldcg(q); };
  const int npl = blockIdx.x < (unsigned)p ? (p - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
  constexpr int NPART = (NW * 32) / L::NACC;   // threads per value
  double* part64 = red64 + (size_t)((p + gridDim.x - 1) / gridDim.x) * L::NACC;  // [NPART][NACC] scratch
  AtomPre* pre = (AtomPre*)(part64 + NPART * L::NACC);                          // [B]
  float* pstage = (float*)(smraw + a.pstage_off);
#ifdef PB_TUNING
  uint64_t t_op = (a.prof && threadIdx.x == 0) ? gtimer() : 0;   // owner sub-phases (slots 1, 4, 11)
  auto oprof = [&](int slot) {
    if (a.prof && threadIdx.x == 0) {
      const uint64_t now = gtimer();
      a.prof[blockIdx.x * kProfSlots + slot] += now - t_op;
      t_op = now;
    }
  };
#else
  auto oprof = [](int) {};
#endif
  for (int i = 0; i < npl; ++i) {
    const int pe = blockIdx.x + i * gridDim.x;
    const float* pix = a.partials + (size_t)pe * gridDim.x * L::NACC;
    if (a.pstage_off) {   // one bulk copy of the pixel's partials (contiguous, L2-resident)
      if (threadIdx.x == 0) {
        asm volatile("fence.proxy.async;" ::: "memory");   // generic-proxy partials -> async-proxy read
        const uint32_t bytes = gridDim.x * L::NACC * 4u;
        mbar_expect_tx(pbar, bytes);
        bulk_copy_g2s(pstage, pix, bytes, pbar);
      }
      mbar_wait(pbar, pphase);
      pphase ^= 1u;
    }
    oprof(1);
    if (threadIdx.x < NPART * L::NACC) {
      const int q = threadIdx.x % L::NACC, part = threadIdx.x / L::NACC;
      const float* src = (a.pstage_off ? (const float*)pstage : pix) + q;
      double acc16[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) acc16[u] = 0.0;
      int b = part;
      for (; b + 15 * NPART < (int)gridDim.x; b += 16 * NPART) {
#pragma unroll
        for (int u = 0; u < 16; ++u) acc16[u] += (double)ld_part(src + (size_t)(b + u * NPART) * L::NACC);
      }
#pragma unroll
      for (int u = 0; u < 16; ++u)  // tail: at most 15 more partials, still independent
        if (b + u * NPART < (int)gridDim.x) acc16[u] += (double)ld_part(src + (size_t)(b + u * NPART) * L::NACC);
#pragma unroll
      for (int h = 8; h >= 1; h >>= 1)
#pragma unroll
        for (int u = 0; u < h; ++u) acc16[u] += acc16[u + h];
      part64[part * L::NACC + q] = acc16[0];
    }
    __syncthreads();
    if (threadIdx.x < L::NACC) {
      double sum = 0.0;
      for (int u = 0; u < NPART; ++u) sum += part64[u * L::NACC + threadIdx.x];
      red64[(size_t)i * L::NACC + threadIdx.x] = sum;
      if (a.split) a.reduced[(size_t)pe * L::NACC + threadIdx.x] = sum;
    }
    __syncthreads();
    oprof(4);
    if (a.split) continue;
    if ((int)threadIdx.x < nb)   // the parallel part of the B draws
      pre[threadIdx.x] = atom_pre<B>(red64 + (size_t)i * L::NACC, threadIdx.x, pe, p, k0, geps, epoch, a.draws,
                                     a.key0, a.key1, dold);
    __syncthreads();
    if (threadIdx.x == 0) {
      atom_pixel_update<B>(red64 + (size_t)i * L::NACC, pe, p, k0, nb, geps, epoch, a.draws, a.key0, a.key1, dold,
                           a.atoms, dprev, a.delta_g, pre);
      if (a.pixel_flags) {   // publish the pixel's shifts: delta_g[.][pe] is ready for pass blk + 1
        __threadfence();
        asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(a.bar + 4 + pe), "r"((unsigned)(k0 / B + 1)) : "memory");
      }
    }
    __syncthreads();
    oprof(11);
  }
}

// Dictionary step (ELL element order), persistent and cooperative: one 16-warp
// CTA per SM with two tile stages.  The warps walk the CTA's waves round-robin
// ACROSS tiles (no CTA barrier per tile): stage s holds every other tile; a
// warp waits on a stage's fill mbarrier before its first wave of that tile and,
// once past the tile, counts itself out on the stage; the last warp out issues
// the bulk copies of the tile two ahead into the freed stage.  Column sums of
// even and odd tiles go to two accumulators (warps are at most one tile apart,
// so a column is never flushed by two warps at once), summed in fixed order at
// the end of the pass.  The next wave's first elements are loaded before the
// current wave's flush.
template <int NW, int ACS>   // ACS: accumulator row (48, or 44 without the redundant Gram entries for large P)
__global__ void __launch_bounds__(NW * 32, 1) k_dict_ell2(DictGramArgs a) {
  using L = GramLayout<kWB>;
  constexpr int B = kWB;
  extern __shared__ __align__(16) unsigned char smraw[];
  const int p = a.p;
  // [stage 0: cur | prev][stage 1: cur | prev] (each block + its zero row), aliased
  // by the owner scratch in the update phase; then acc[2][p*NACC], dold, dprev
  constexpr bool kSmemOld = ACS == L::NACC;   // the block's old atoms staged (else read from global)
  float* acc0 = (float*)(smraw + a.wbytes);             // [p][ACS] even tiles
  float* acc1 = acc0 + (size_t)p * ACS;                  // [p][ACS] odd tiles
  float* dprev = acc1 + (size_t)p * ACS;                 // B * p shifts of the previous block
  float* dold = dprev + B * p;                           // B * p old atoms of the block (kSmemOld)
  __shared__ __align__(8) uint64_t mbar[3];   // [0..1] stage fills, [2] owner partials
  __shared__ int done[2];
  __shared__ unsigned next_wave;   // dynamic wave claiming inside the CTA
  if (threadIdx.x == 0) {
    mbar_init(&mbar[0], 1);
    mbar_init(&mbar[1], 1);
    mbar_init(&mbar[2], 1);
    done[0] = done[1] = 0;
  }
  uint32_t pphase = 0;
  int fills0 = 0, fills1 = 0;   // fills of stage 0 / 1 completed in earlier passes (mbarrier parities)
  unsigned bar_target = 0;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const double geps = a.sc->gamma_eps;
  const int epoch = a.sc->epoch + 1;
  const int nblk = (a.k + B - 1) / B;
  int64_t w_lo, w_hi;
  int t_lo, t_hi;
  ell_cta_range(a, w_lo, w_hi, t_lo, t_hi);
  const int ntile = t_hi - t_lo;
  const uint32_t sbase = smem_u32(smraw);
  uint64_t t_mark = a.prof ? gtimer() : 0;   // in-kernel phase profile (pb_dict_profile), thread 0
  auto prof = [&](int slot) {
    if (a.prof && threadIdx.x == 0) {
      const uint64_t now = gtimer();
      a.prof[blockIdx.x * kProfSlots + slot] += now - t_mark;
      t_mark = now;
    }
  };
  if (a.split && a.blk_begin > 0) {  // split mode: the previous pass's shifts come from global memory
    for (int t = threadIdx.x; t < B * p; t += blockDim.x) dprev[t] = a.delta_g[t];
  }
  const uint64_t pol_last = l2_policy_evict_last(), pol_first = l2_policy_evict_first();
  // bulk-copy tile t_lo + u's W blocks of pass `bk` into stage u & 1
  auto issue = [&](int u, int bk) {
    const int s = u & 1, tile = t_lo + u;
    unsigned char* dst = smraw + (size_t)s * 2 * kWStride;
    fence_proxy_async();
    const bool hc = bk < nblk, hp = bk > 0;
    mbar_expect_tx(&mbar[s], (hc ? kTile * B * 4u : 0u) + (hp ? kTile * B * 4u : 0u));
    if (hc) {
      if (a.w_evict_first == 1)
        bulk_copy_g2s_hint(dst, a.wt + ((int64_t)tile * a.nblk8 + bk) * kTile * B, kTile * B * 4u, &mbar[s], pol_first);
      else if (a.w_evict_first == 2)   // kept for its second use as the next pass's previous block
        bulk_copy_g2s_hint(dst, a.wt + ((int64_t)tile * a.nblk8 + bk) * kTile * B, kTile * B * 4u, &mbar[s], pol_last);
      else
        bulk_copy_g2s(dst, a.wt + ((int64_t)tile * a.nblk8 + bk) * kTile * B, kTile * B * 4u, &mbar[s]);
    }
    if (hp)  // last use of the previous block
      bulk_copy_g2s_hint(dst + kWStride, a.wt + ((int64_t)tile * a.nblk8 + bk - 1) * kTile * B, kTile * B * 4u,
                         &mbar[s], pol_first);
  };
  bool prefetched = false;
  // a pass's setup: zeroed accumulators, the block's current atoms, the zero W
  // rows (the owner phase overwrote them), the wave counter.  For every pass but
  // the first it runs while the previous pass's shifts are still being published.
  auto setup = [&](int bk) {
    for (int t = threadIdx.x; t < 2 * p * ACS; t += blockDim.x) acc0[t] = 0.0f;
    if constexpr (kSmemOld) {
      const int nbk = bk < nblk ? min(B, a.k - bk * B) : 0;
      for (int t = threadIdx.x; t < B * p; t += blockDim.x) {
        const int j = t / p, pe = t - j * p;
        dold[t] = j < nbk ? a.atoms[(int64_t)(bk * B + j) * p + pe] : 0.0f;
      }
    }
    if (threadIdx.x < 16) {
      const int blkno = threadIdx.x >> 2, part = threadIdx.x & 3;
      *(float2*)(smraw + blkno * kWStride + kEllZeroRow + part * 8) = make_float2(0.f, 0.f);
    }
    if (threadIdx.x == 0) next_wave = NW;   // waves 0..NW-1 go to warps 0..NW-1
  };
  setup(a.split ? a.blk_begin : 0);
  for (int blk = a.split ? a.blk_begin : 0; blk <= (a.split ? a.blk_begin : nblk); ++blk) {
    const bool has_cur = blk < nblk, has_prev = blk > 0;
    const int k0 = blk * B;
    const int nb = has_cur ? min(B, a.k - k0) : 0;
    if (threadIdx.x == 0 && !prefetched) {
      if (ntile > 0) issue(0, blk);
      if (ntile > 1) issue(1, blk);
    }
    prefetched = false;
    __syncthreads();
    prof(0);
    // ---- element phase: this warp's waves w_lo + wid, + NW, ... ----
    // Every warp visits every tile of the CTA in order: wait for the stage's
    // fill, its waves of the tile, count out (the last warp out refills the stage
    // with the tile two ahead).  Waiting on every fill in order keeps each
    // stage's mbarrier parity unambiguous.
    {
      auto fill_parity = [&](int uu) { return (uint32_t)(((uu & 1) ? fills1 : fills0) + (uu >> 1)) & 1u; };
      auto tile_of = [&](int64_t w, int from) {
        int t = from;
        while (t + 1 < ntile && a.wave_base[t_lo + t + 1] <= w) ++t;
        return t;
      };
      // a warp's next wave: claimed from the CTA's counter (dynamic balance;
      // each column still gets one flush per tile, in tile order per parity, so
      // the sums do not depend on which warp took which wave) or round-robin
      auto next = [&](int64_t cur) -> int64_t {
        if (!a.dyn_waves) return cur + NW;
        unsigned w = 0;
        if (lane == 0) w = atomicAdd(&next_wave, 1u);
        return w_lo + (int64_t)__shfl_sync(0xffffffffu, w, 0);
      };
      int64_t wv = w_lo + wid;
      bool have = wv < w_hi && !PB_DBG(a, 8);   // (tuning builds: bit 8 skips the element phase)
      int wu = 0;              // tile (relative) of the next wave
      uint32_t ib[kEllPf];
      float rb[kEllPf];
      EllWave h{};
      if (have) {
        wu = tile_of(wv, 0);
        h = ell_header(a, wv, a.ell_base[t_lo + wu], lane);
        ell_prefetch(a, h, ib, rb, pol_last);
      }
      for (int u = 0; u < ntile; ++u) {
        const uint64_t t_fw = (a.prof && threadIdx.x == 0) ? gtimer() : 0;
        mbar_wait(&mbar[u & 1], fill_parity(u));
        if (a.prof && threadIdx.x == 0) a.prof[blockIdx.x * kProfSlots + 10] += gtimer() - t_fw;   // fill waits
        const uint32_t wcur_s = ell_stage_addr(sbase + (uint32_t)(u & 1) * 2 * kWStride);
        float* acc = (u & 1) ? acc1 : acc0;
        while (have && wu == u) {
#ifdef PB_TUNING
          const uint64_t t_w0 = (a.wprof && blk == 3 && lane == 0) ? gtimer() : 0;
          const int64_t wv_self = wv;
#endif
          float2 dl2[B / 2];
          const bool live = h.col != 0xFFFF;
#pragma unroll
          for (int j = 0; j < B / 2; ++j)
            dl2[j] = (has_prev && live) ? make_float2(dprev[2 * j * p + h.col], dprev[(2 * j + 1) * p + h.col])
                                        : make_float2(0.f, 0.f);
          float v[L::NP];
#pragma unroll
          for (int q = 0; q < L::NP; ++q) v[q] = 0.0f;
          if (has_prev && has_cur) ell_elements<true, true>(a, h, wcur_s, dl2, v, ib, rb, pol_last);
          else if (has_cur) ell_elements<false, true>(a, h, wcur_s, dl2, v, ib, rb, pol_last);
          else ell_elements<true, false>(a, h, wcur_s, dl2, v, ib, rb, pol_last);
          const int lg_c = h.lg, col_c = h.col;
          // the next wave's header and first elements go in flight before the flush
          wv = next(wv);
          have = wv < w_hi;
          if (have) {
            wu = tile_of(wv, wu);
            h = ell_header(a, wv, a.ell_base[t_lo + wu], lane);
            ell_prefetch(a, h, ib, rb, pol_last);
          }
          if (has_cur) ell_flush<ACS>(v, lg_c, col_c, lane, acc);
#ifdef PB_TUNING
          if (a.wprof && blk == 3 && lane == 0 && wv_self < ((int64_t)1 << 24)) {   // per-wave profile
            unsigned smid;
            asm("mov.u32 %0, %%smid;" : "=r"(smid));
            a.wprof[3 * wv_self] = gtimer() - t_w0;
            a.wprof[3 * wv_self + 1] = smid;
            a.wprof[3 * wv_self + 2] = wid;
          }
#endif
        }
        // count out of tile u; the last warp out refills its stage with tile u + 2
        __syncwarp();
        if (lane == 0) {
          __threadfence_block();
          const int s = u & 1;
          if (atomicAdd(&done[s], 1) == NW - 1) {
            done[s] = 0;
            if (u + 2 < ntile) issue(u + 2, blk);
          }
        }
      }
      fills0 += (ntile + 1) >> 1;
      fills1 += ntile >> 1;
    }
    prof(2);
    if (!has_cur) break;
    __syncthreads();
    prof(3);
    // pixel-major partials [pixel][CTA][NACC] (even + odd tile sums, fixed order)
    if constexpr (ACS == L::NACC) {   // 16-byte chunks
      static_assert(L::NACC % 4 == 0, "accumulator rows in 16-byte chunks");
      for (int t = threadIdx.x; t < p * (L::NACC / 4); t += blockDim.x) {
        const int pe = t / (L::NACC / 4), q4 = t - pe * (L::NACC / 4);
        const float4 x = *(const float4*)(acc0 + pe * L::NACC + 4 * q4), y = *(const float4*)(acc1 + pe * L::NACC + 4 * q4);
        *(float4*)(a.partials + ((size_t)pe * gridDim.x + blockIdx.x) * L::NACC + 4 * q4) =
            make_float4(x.x + y.x, x.y + y.y, x.z + y.z, x.w + y.w);
      }
    } else {   // expanded to the 48-layout; the redundant Gram entries (never read by the draws) as 0
      for (int t = threadIdx.x; t < p * L::NACC; t += blockDim.x) {
        const int pe = t / L::NACC, q = t - pe * L::NACC;
        const int c = pe * ACS + gram_compact(q);
        a.partials[((size_t)pe * gridDim.x + blockIdx.x) * L::NACC + q] = gram_redundant(q) ? 0.0f : acc0[c] + acc1[c];
      }
    }
    prof(5);
    if (PB_DBG(a, 16)) grid_sync(a.bar); else grid_sync_mono(a.bar + 2, bar_target);
    prof(6);
    // the block's old atoms: staged, or straight from global memory (atom_pre reads each before its write)
    dict_owner_phase<NW>(a, smraw, &mbar[2], pphase, k0, nb, geps, epoch, kSmemOld ? dold : a.atoms + (size_t)k0 * p,
                         dprev);
    prof(7);
    if (a.split) return;  // split mode: the caller allreduces `reduced` across ranks, then k_dict_update
    // the next pass's first tiles do not depend on the shifts: stage them now
    // (the owner scratch they overwrite is done) so they land during the barrier
    if (threadIdx.x == 0) {
      if (ntile > 0) issue(0, blk + 1);
      if (ntile > 1) issue(1, blk + 1);
    }
    prefetched = true;
    setup(blk + 1);
    if (a.pixel_flags) {
      // no second grid barrier: wait until every pixel's owner has published this
      // block's shifts (owners finish reading the partials before they publish, so
      // the next pass may overwrite them)
      if (wid == 0)
        for (int pe = lane; pe < p; pe += 32)
          while (ld_acquire(a.bar + 4 + pe) < (unsigned)(blk + 1)) __nanosleep(32);
      __syncthreads();
    } else if (PB_DBG(a, 16)) {
      grid_sync(a.bar);
    } else {
      grid_sync_mono(a.bar + 2, bar_target);
    }
    prof(8);
    for (int t = threadIdx.x; t < B * p; t += blockDim.x) dprev[t] = __ldcg(a.delta_g + t);
    __syncthreads();
    prof(9);
  }
}

// Single-stage variant (large patches, where two stages and two accumulators do
// not fit): NW warps, the CTA's tiles one at a time, the tile's waves
// round-robin over the warps, a CTA barrier per tile.
template <int NW>
__global__ void __launch_bounds__(NW * 32, 16 / NW) k_dict_gram(DictGramArgs a) {
  using L = GramLayout<kWB>;
  constexpr int B = kWB;
  extern __shared__ __align__(16) unsigned char smraw[];
  const int p = a.p;
  float* acc = (float*)(smraw + a.wbytes);               // p * NACC
  float* dold = acc + (size_t)p * L::NACC;               // B * p
  float* dprev = dold + B * p;                           // B * p
  __shared__ __align__(8) uint64_t mbar[2];   // [0] staging, [1] owner partials
  const uint32_t wcur_s = smem_u32(smraw);
  if (threadIdx.x == 0) {
    mbar_init(&mbar[0], 1);
    mbar_init(&mbar[1], 1);
  }
  uint32_t pphase = 0, sphase = 0;
  unsigned bar_target = 0;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const double geps = a.sc->gamma_eps;
  const int epoch = a.sc->epoch + 1;
  const int nblk = (a.k + B - 1) / B;
  int64_t w_lo, w_hi;
  int t_lo, t_hi;
  ell_cta_range(a, w_lo, w_hi, t_lo, t_hi);
  if (a.split && a.blk_begin > 0) {
    for (int t = threadIdx.x; t < B * p; t += blockDim.x) dprev[t] = a.delta_g[t];
  }
  const uint64_t pol_last = l2_policy_evict_last(), pol_first = l2_policy_evict_first();
  auto issue = [&](int tile, int bk) {
    fence_proxy_async();
    const bool hc = bk < nblk, hp = bk > 0;
    mbar_expect_tx(&mbar[0], (hc ? kTile * B * 4u : 0u) + (hp ? kTile * B * 4u : 0u));
    if (hc) bulk_copy_g2s(smraw, a.wt + ((int64_t)tile * a.nblk8 + bk) * kTile * B, kTile * B * 4u, &mbar[0]);
    if (hp)
      bulk_copy_g2s_hint(smraw + kWStride, a.wt + ((int64_t)tile * a.nblk8 + bk - 1) * kTile * B, kTile * B * 4u,
                         &mbar[0], pol_first);
  };
  bool prefetched = false;
  for (int blk = a.split ? a.blk_begin : 0; blk <= (a.split ? a.blk_begin : nblk); ++blk) {
    const bool has_cur = blk < nblk, has_prev = blk > 0;
    const int k0 = blk * B;
    const int nb = has_cur ? min(B, a.k - k0) : 0;
    for (int t = threadIdx.x; t < p * L::NACC; t += blockDim.x) acc[t] = 0.0f;
    for (int t = threadIdx.x; t < B * p; t += blockDim.x) {
      const int j = t / p, pe = t - j * p;
      dold[t] = j < nb ? a.atoms[(int64_t)(k0 + j) * p + pe] : 0.0f;
    }
    if (threadIdx.x < 8) {   // the zero rows behind both blocks (the owner phase overwrote them)
      const int blkno = threadIdx.x >> 2, part = threadIdx.x & 3;
      *(float2*)(smraw + blkno * kWStride + kEllZeroRow + part * 8) = make_float2(0.f, 0.f);
    }
    const bool pf = prefetched;
    prefetched = false;
    for (int tile = t_lo; tile < t_hi; ++tile) {
      __syncthreads();   // previous tile fully consumed (and the zero rows written)
      if (threadIdx.x == 0 && !(pf && tile == t_lo)) issue(tile, blk);
      const int64_t wa = max(w_lo, a.wave_base[tile]), wb = min(w_hi, a.wave_base[tile + 1]);
      const int64_t tile_ell = a.ell_base[tile];
      mbar_wait(&mbar[0], sphase);
      sphase ^= 1u;
      const uint32_t wst = ell_stage_addr(wcur_s);   // (loads of the stage stay behind the wait)
      for (int64_t wv = wa + wid; wv < wb; wv += NW) {
        const EllWave h = ell_header(a, wv, tile_ell, lane);
        uint32_t ib[kEllPf];
        float rb[kEllPf];
        ell_prefetch(a, h, ib, rb, pol_last);
        float2 dl2[B / 2];
        const bool live = h.col != 0xFFFF;
#pragma unroll
        for (int j = 0; j < B / 2; ++j)
          dl2[j] = (has_prev && live) ? make_float2(dprev[2 * j * p + h.col], dprev[(2 * j + 1) * p + h.col])
                                      : make_float2(0.f, 0.f);
        float v[L::NP];
#pragma unroll
        for (int q = 0; q < L::NP; ++q) v[q] = 0.0f;
        if (has_prev && has_cur) ell_elements<true, true>(a, h, wst, dl2, v, ib, rb, pol_last);
        else if (has_cur) ell_elements<false, true>(a, h, wst, dl2, v, ib, rb, pol_last);
        else ell_elements<true, false>(a, h, wst, dl2, v, ib, rb, pol_last);
        if (has_cur) ell_flush<L::NACC>(v, h.lg, h.col, lane, acc);
      }
    }
    if (!has_cur) break;
    __syncthreads();
    for (int t = threadIdx.x; t < p * L::NACC; t += blockDim.x) {
      const int pe = t / L::NACC, q = t - pe * L::NACC;
      a.partials[((size_t)pe * gridDim.x + blockIdx.x) * L::NACC + q] = acc[t];
    }
    if (PB_DBG(a, 16)) grid_sync(a.bar); else grid_sync_mono(a.bar + 2, bar_target);
    dict_owner_phase<NW>(a, smraw, &mbar[1], pphase, k0, nb, geps, epoch, dold, dprev);
    if (a.split) return;
    if (t_lo < t_hi) {
      if (threadIdx.x == 0) issue(t_lo, blk + 1);
      prefetched = true;
    }
    if (PB_DBG(a, 16)) grid_sync(a.bar); else grid_sync_mono(a.bar + 2, bar_target);
    for (int t = threadIdx.x; t < B * p; t += blockDim.x) dprev[t] = __ldcg(a.delta_g + t);
    __syncthreads();
  }
}

// Split mode, after the cross-rank allreduce of `reduced`: the block's atom draws.
template <int B>
__global__ void k_dict_update(DictGramArgs a, int blk) {
  extern __shared__ float su[];
  float* dold = su;              // B * p
  float* dprev = dold + B * a.p; // B * p
  const int nb = min(B, a.k - blk * B);
  for (int t = threadIdx.x; t < B * a.p; t += blockDim.x) {
    const int j = t / a.p, pe = t - j * a.p;
    dold[t] = j < nb ? a.atoms[(int64_t)(blk * B + j) * a.p + pe] : 0.0f;
  }
  __syncthreads();
  atom_block_update<B>(a.reduced, a.p, blk * B, nb, a.sc->gamma_eps, a.sc->epoch + 1, a.draws, a.key0, a.key1, dold,
                       dprev, a.atoms);
  __syncthreads();
  for (int t = threadIdx.x; t < B * a.p; t += blockDim.x) a.delta_g[t] = dprev[t];
}

// Dictionary step on all-zero codes (fresh or warm-reset state, Z*S == 0):
// every moment sum is exactly 0, so each atom is redrawn from its prior
// d_k = g / sqrt(P) (bpfa.py:161-166, 300-307) and the
// residual shifts R += w (x) delta vanish.  The same f64 draw arithmetic as the
// full step (atom_pixel_update on zero sums), so the atoms are bit-identical to
// it, without the K/8 passes over the residual.  One CTA per atom block.
template <int B>
__global__ void k_dict_prior(DictGramArgs a) {
  using L = GramLayout<B>;
  extern __shared__ float sp[];
  float* dsh = sp;                       // B * p shifts (discarded: W == 0)
  __shared__ double zero[L::NACC];
  for (int q = threadIdx.x; q < L::NACC; q += blockDim.x) zero[q] = 0.0;
  __syncthreads();
  const int blk = blockIdx.x, k0 = blk * B;
  const int nb = min(B, a.k - k0);
  for (int pe = threadIdx.x; pe < a.p; pe += blockDim.x) {
    // the old atoms go to shared memory first (atom_pixel_update reads d_old
    // after writing the new atom); slot [j*p+pe] is then overwritten by the
    // (unused) shift of atom j only after its last read
#pragma unroll
    for (int j = 0; j < B; ++j) dsh[j * a.p + pe] = j < nb ? a.atoms[(int64_t)(k0 + j) * a.p + pe] : 0.0f;
    atom_pixel_update<B>(zero, pe, a.p, k0, nb, a.sc->gamma_eps, a.sc->epoch + 1, a.draws, a.key0, a.key1, dsh,
                         a.atoms, dsh, nullptr, nullptr);
  }
}

int launch_dict_prior(const DictGramArgs& a, cudaStream_t st) {
  constexpr int B = kWB;
  const int nblk = (a.k + B - 1) / B;
  const int th = a.p < 256 ? ((a.p + 31) / 32) * 32 : 256;
  const size_t smem = (size_t)B * a.p * sizeof(float);
  if (smem > 48 * 1024) PB_CUDA_TRY(cudaFuncSetAttribute(k_dict_prior<B>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                         (int)smem));
  k_dict_prior<B><<<nblk, th, smem, st>>>(a);
  PB_LAUNCH_CHECK();
  return PB_OK;
}

// The code step's transposed dictionary, pre-packed once per sweep in exactly
// the shared-memory layout of each staged chunk: image[ci][pe * kp + kk] =
// D[ci*kc + kk][pe] (0 for the pad columns and the zero row pe == P), each chunk
// padded to a multiple of 16 bytes, so staging is a single bulk copy.
__global__ void k_pack_dt(const float* __restrict__ atoms, int p, int k, int kc, int64_t img_floats, int nchunks,
                          float* __restrict__ img) {
  const int kp = kc + 2;
  const int64_t total = (int64_t)nchunks * img_floats;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int ci = (int)(t / img_floats);
    const int rem = (int)(t - (int64_t)ci * img_floats);
    const int pe = rem / kp, kk = rem - pe * kp;
    const int katom = ci * kc + kk;
    img[t] = (pe < p && kk < kc && katom < k) ? atoms[(int64_t)katom * p + pe] : 0.0f;
  }
}

void code_dt_layout(int p, int k, int* kc_out, int64_t* img_floats_out, int* nchunks_out) {
  // DT chunk: kc atoms (a multiple of 8) x (P+1) rows of pitch kc+2, as many as
  // two 256-thread CTAs per SM can hold next to the logits, usage counts and
  // w windows (228 KB per SM, 1 KB reserved per CTA, static shared memory);
  // the whole dictionary when it fits (configs[1]: P = 100, K = 256 just fits)
  const int k8 = (int)ceil_div(k, 8) * 8;
  const size_t per_cta = 228 * 1024 / 2 - 1024 - 512;
  const size_t fixed = (size_t)k * 8 + (size_t)256 * 8 * 4;
  int kc = per_cta > fixed ? (int)(((per_cta - fixed) / ((size_t)(p + 1) * 4) - 2) & ~(size_t)7) : 8;
  if (kc < 8) kc = 8;
  if (kc > k8) kc = k8;
  if (kc_out) *kc_out = kc;
  if (img_floats_out) *img_floats_out = (((int64_t)(p + 1) * (kc + 2)) + 3) & ~(int64_t)3;
  if (nchunks_out) *nchunks_out = (int)ceil_div(k, kc);
}

int launch_pack_dt(const float* atoms, int p, int k, float* img, cudaStream_t st) {
  int kc, nch;
  int64_t imgf;
  code_dt_layout(p, k, &kc, &imgf, &nch);
  const int64_t total = imgf * nch;
  k_pack_dt<<<(unsigned)std::min<int64_t>(ceil_div(total, 256), 1184), 256, 0, st>>>(atoms, p, k, kc, imgf, nch, img);
  PB_LAUNCH_CHECK();
  return PB_OK;
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
    MACRO(8, 1) MACRO(16, 1) MACRO(24, 1) MACRO(32, 1) MACRO(32, 2) MACRO(32, 4) MACRO(32, 8)      \
    MACRO(32, 16) MACRO(32, 32)                                                                     \
    default: set_error("unsupported compact layout c=%d g=%d", c, g); return PB_EUNSUPPORTED;       \
  }

// Relative cost of one patch-atom update in a (c slots, g lanes) code-step
// launch: g lanes each run the sampling (~100 instructions) and c slots (~4.5).
// relative per-patch cost of the code step by launch shape, measured on B200
// (cfg2 1024^2/10x10: 16 lanes 2.50 ms, 24 lanes 2.58, 32 lanes 2.77; cfg4
// cube: 2 lanes-per-patch groups cost ~0.73x of 4)
static double code_cost(int c, int g) {
  if (g == 1) return c <= 8 ? 0.98 : c <= 16 ? 1.0 : c <= 24 ? 1.03 : 1.11;
  return 1.11 * sqrt((double)g);
}

// Window layout and block claiming of a code-step launch (256 threads per CTA):
// pitch-8 swizzled w windows when only they let two CTAs share an SM; warps
// claim their own 32-patch blocks whenever D is staged whole (either window
// pitch) and the problem has at least 2^17 patches: configs[2]/[4] -4 %, and
// combined with the pitch-8 windows configs[1] -7 % (v22: 2.12 -> 1.97 ms).
// Covered at P = 100, K = 256, >= 2^17 patches by tests/test_gpu_scale.py.
static void code_window_claim(int64_t n, int p, int k, int g, bool& ws, bool& wc) {
  int kc;
  int64_t imgf;
  code_dt_layout(p, k, &kc, &imgf, nullptr);
  const size_t per_cta = 228 * 1024 / 2 - 1024 - 512;
  ws = g == 1 && (size_t)imgf * 4 + (size_t)k * 8 + (size_t)(256 / g) * 9 * 4 > per_cta;
  wc = g == 1 && kc >= k && n >= (1 << 17);   // small problems: CTA claiming (configs[0] +30 % otherwise)
}

int code_launch_blocks(int cmax, int64_t n, int p, int k) {
  int c, g;
  if (!pick_compact(cmax, c, g)) return 0;
  bool ws, wc;
  code_window_claim(n * g, p, k, g, ws, wc);
  return (int)ceil_div(n * g, wc ? 32 : 256);
}

int code_split_choose(const int32_t* hist, int p, int cmax) {
  int cw, gw;
  if (!pick_compact(cmax, cw, gw)) return 0;
  if (gw >= 2) cw = 32;
  const double wide = code_cost(cw, gw);
  double total_n = 0;
  for (int c = 0; c <= p; ++c) total_n += hist[c];
  double best = total_n * wide;  // one launch for everything
  int best_t = 0;
  static const int kT[] = {8, 16, 24, 32, 64, 128, 256, 512};
  for (int t : kT) {
    if (t >= cmax) break;
    int cm, gm;
    if (!pick_compact(t, cm, gm)) continue;
    if (gm >= 2) cm = 32;
    double below = 0;
    for (int c = 0; c <= p && c <= t; ++c) below += hist[c];
    // the narrow launch still spends a lane on every patch; the wide launch
    // gathers its listed patches' state (uncoalesced: ~4x), plus a fixed cost.
    // The wide launch runs concurrently on a side stream; with fewer than half
    // a wave of outliers it is a latency tail (each of its CTAs walks all K
    // atoms for its patches) that hides only behind a narrow launch of at
    // least 4 waves
    const double wave = 2.0 * sm_count_c() * (256.0 / gw);
    const double narrow_waves = total_n * gm / (256.0 * 2.0 * sm_count_c());
    if (total_n - below < 0.5 * wave && narrow_waves < 4.0) continue;
    const double cost = total_n * code_cost(cm, gm) + (total_n - below) * wide * 4.0 + 2048.0 * wide;
    if (cost < best) { best = cost; best_t = t; }
  }
  // split only for a clear modeled win (marginal splits lose to the second
  // launch's restaging and scattered state accesses)
  return best < 0.95 * total_n * wide ? best_t : 0;
}

static void normalize_cg(int& c, int& g) {
  // collapse to the instantiated set
  if (g >= 2) c = 32;
}

int launch_resid_compact(const CompactArgs& a_in, cudaStream_t st) {
  CompactArgs a = a_in;
  int c, g;
  if (!pick_compact(a.cmax, c, g)) { set_error("patch has too many observed elements (%d)", a.cmax); return PB_EUNSUPPORTED; }
  normalize_cg(c, g);
  const int th = 256;
  a.kc = (int)((64 * 1024) / ((size_t)(a.p + 1) * 4)) & ~7;  // multiple of 8: W blocks align
  if (a.kc < 8) a.kc = 8;
  if (a.kc > a.k) a.kc = a.k;
  const size_t smem = (size_t)std::max(a.kc, 8) * (a.p + 1) * 4;
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
  // DT chunks as pre-packed by launch_pack_dt (the caller packs a.dt_img first)
  if (!a.dt_img) { set_error("code step without the packed dictionary image"); return PB_EVALUE; }
  code_dt_layout(a.p, a.k, &a.kc, &a.dt_img_floats, nullptr);
  bool ws, wc;
  code_window_claim((a.plist ? a.plist_n : a.n) * g, a.p, a.k, g, ws, wc);
  const size_t fixed = (size_t)a.k * 8 + (size_t)(th / g) * (ws ? 8 : 9) * 4;
  const size_t smem = (size_t)a.dt_img_floats * 4 + fixed;
  if (smem > 220 * 1024) { set_error("too many atoms for the code step (K=%d)", a.k); return PB_EUNSUPPORTED; }
  const int64_t nb = ceil_div((a.plist ? a.plist_n : a.n) * g, th);
  if (a.zero_mcount) PB_CUDA_TRY(cudaMemsetAsync(a.m_count, 0, (size_t)a.k * sizeof(int32_t), st));
  nblocks = (int)(wc ? ceil_div((a.plist ? a.plist_n : a.n) * g, 32) : nb);   // one S^2 / R^2 pair per claimed block
  if (nb == 0) return PB_OK;
  PB_CUDA_TRY(cudaMemsetAsync(a.blk_ctr, 0, sizeof(unsigned), st));
#define PB_C(C, GG)                                                                                  \
  case C * 100 + GG: {                                                                               \
    auto kern = ws && wc ? (mode == kRngReplay ? k_code_compact<C, GG, kRngReplay, GG == 1, GG == 1>           \
                                               : k_code_compact<C, GG, kRngPhilox, GG == 1, GG == 1>)         \
           : ws ? (mode == kRngReplay ? k_code_compact<C, GG, kRngReplay, GG == 1, false>                      \
                                      : k_code_compact<C, GG, kRngPhilox, GG == 1, false>)                     \
           : wc ? (mode == kRngReplay ? k_code_compact<C, GG, kRngReplay, false, GG == 1>                      \
                                      : k_code_compact<C, GG, kRngPhilox, false, GG == 1>)                     \
                : (mode == kRngReplay ? k_code_compact<C, GG, kRngReplay, false, false>                        \
                                      : k_code_compact<C, GG, kRngPhilox, false, false>);                      \
    PB_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
    int per_sm = 0;                                                                                  \
    PB_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, th, smem));             \
    const int64_t grid = std::min<int64_t>(nb, (int64_t)std::max(per_sm, 1) * sm_count_c());         \
    kern<<<(unsigned)grid, th, smem, st>>>(a);                                                       \
    break;                                                                                           \
  }
  PB_DISPATCH_CG(c, g, PB_C)
#undef PB_C
  PB_LAUNCH_CHECK();
  return PB_OK;
}

template <int NW>
static size_t dict_gram_smem(int p, size_t* wbytes_out) {
  using L = GramLayout<kWB>;
  const size_t wbytes = std::max((size_t)2 * kWStride, (size_t)p * L::NACC * 8);
  if (wbytes_out) *wbytes_out = wbytes;
  return wbytes + (size_t)p * L::NACC * 4 + (size_t)2 * kWB * p * 4;
}

static size_t dict_ell2_smem(int p, int acs, size_t* wbytes_out);

template <int NW, int TWO>   // TWO: 0 the single-stage kernel, else the two-stage one with accumulator rows of TWO
static int launch_dict_gram_b(DictGramArgs a, cudaStream_t st) {
  constexpr int B = kWB;
  const int th = NW * 32;
  if (a.ld % 4) { set_error("usage/weights row pitch must be a multiple of 4 (got %lld)", (long long)a.ld); return PB_EVALUE; }
  size_t wbytes = 0;
  const size_t smem = TWO ? dict_ell2_smem(a.p, TWO, &wbytes) : dict_gram_smem<NW>(a.p, &wbytes);
  a.wbytes = (int)wbytes;
  if (smem > 225 * 1024) { set_error("patch size %d too large for the dictionary step", a.p); return PB_EUNSUPPORTED; }
  auto kern = TWO == 48 ? k_dict_ell2<NW, 48> : TWO == 44 ? k_dict_ell2<NW, 44> : k_dict_gram<NW>;
  PB_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 0;
  PB_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, th, smem));
  if (per_sm < 1) { set_error("dictionary step cannot be resident"); return PB_EUNSUPPORTED; }
  int blocks = sm_count_c() * per_sm;
  if (blocks > a.max_blocks) blocks = a.max_blocks;
  const int cap = PB_TUNE_INT("PB_DICT_MAX_CTAS", 0);   // grid cap for tuning experiments
  if (cap > 0 && blocks > cap) blocks = cap;
  {  // owner partials staged behind the owner scratch (inside the W staging area) when they fit
    using L = GramLayout<B>;
    const size_t npart = (size_t)(NW * 32) / L::NACC;
    const size_t scratch = ((size_t)(a.p + blocks - 1) / blocks * L::NACC + npart * L::NACC) * 8 + (size_t)B * 40;
    const size_t off = (scratch + 127) & ~(size_t)127;
    const int nostage = PB_TUNE_INT("PB_DICT_NO_PSTAGE", 0);   // 1: owners read the partials from L2 (A/B)
    a.pstage_off = (!nostage && off + (size_t)blocks * L::NACC * 4 <= wbytes) ? (int)off : 0;
  }
  PB_CUDA_TRY(cudaMemsetAsync(a.bar, 0, (4 + (size_t)a.p) * sizeof(unsigned), st));
  void* args[] = {&a};
  PB_CUDA_TRY(cudaLaunchCooperativeKernel((const void*)kern, dim3(blocks), dim3(th), args, smem, st));
  return PB_OK;
}

static size_t dict_ell2_smem(int p, int acs, size_t* wbytes_out) {
  using L = GramLayout<kWB>;
  const size_t wbytes = std::max((size_t)4 * kWStride, (size_t)p * L::NACC * 8);
  if (wbytes_out) *wbytes_out = wbytes;
  return wbytes + (size_t)2 * p * acs * 4 + (size_t)kWB * p * 4 * (acs == L::NACC ? 2 : 1);
}

int launch_dict_gram(const DictGramArgs& a_in, cudaStream_t st) {
  // one 16-warp CTA per SM with two tile stages (waves flow across tiles) when
  // it fits in shared memory; else the single-stage variant
  DictGramArgs a = a_in;
  // both W blocks stream with evict_first: the residual and the element index
  // (re-read every pass) keep L2 (configs[1] 3.41 -> 2.52 ms)
  a.w_evict_first = PB_TUNE_INT("PB_DICT_W_EVICT", 1);
  a.dyn_waves = PB_TUNE_INT("PB_DICT_DYN", 1);
  a.tile_cost = PB_TUNE_DBL("PB_DICT_TILE_COST", kTileVisitCost);
  a.split_nearest = PB_TUNE_INT("PB_DICT_NEAREST", 0);
  a.pixel_flags = PB_TUNE_INT("PB_DICT_FLAGS", 1);
  {
    static bool l2_set = false;
    const int persist = PB_TUNE_INT("PB_L2_PERSIST_MB", 0);
    if (persist > 0 && !l2_set) {
      cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, (size_t)persist << 20);
      l2_set = true;
    }
  }
  const int variant = PB_TUNE_INT("PB_DICT_VARIANT", 0);
  if (variant == 0 && dict_ell2_smem(a.p, 48, nullptr) <= 225 * 1024) return launch_dict_gram_b<16, 48>(a, st);
  // large patches (configs[3], P = 256): 44-float accumulator rows, old atoms read from global
  if (variant == 0 && dict_ell2_smem(a.p, 44, nullptr) <= 225 * 1024) return launch_dict_gram_b<16, 44>(a, st);
  if (variant != 1 && 2 * dict_gram_smem<8>(a.p, nullptr) <= 226 * 1024) return launch_dict_gram_b<8, 0>(a, st);
  return launch_dict_gram_b<16, 0>(a, st);
}

int launch_dict_update(const DictGramArgs& a, int blk, cudaStream_t st) {
  const size_t smem = (size_t)2 * 8 * a.p * 4;
  k_dict_update<8><<<1, 256, smem, st>>>(a, blk);
  PB_LAUNCH_CHECK();
  return PB_OK;
}

int dict_gram_blocks(int k) { return (k + 7) / 8; }

size_t dict_gram_partials_bytes(int p, int max_blocks) {
  return (size_t)max_blocks * p * GramLayout<8>::NACC * 4;
}
size_t dict_gram_reduced_bytes(int p) { return (size_t)p * GramLayout<8>::NACC * 8; }

}  // namespace pb
