// pb200 — compose_estimates (bpfa.py:348-352, _kernels.py:133-145) on the
// 5th-generation tensor cores: est = (Z∘S)·D over all P pixels, the one dense
// contraction of the path.
//
//   est^T (N x P)  =  W^T (N x K)  ·  D (K x P),   W = Z∘S (atom-major state)
//
// One CTA (4 warps) owns an M = 128 tile of patches and loops over the atoms in
// chunks of 32.  Per chunk the CTA stages, in shared memory, the W tile
// (w = z ? s : 0 fused into the load, 128 x 32) and the D chunk (P_pad x 32),
// each split into TF32 hi + lo parts (3xTF32: hi·hi + hi·lo + lo·hi gives
// ~fp32 accuracy), in the canonical K-major no-swizzle UMMA layout (8-row x
// 16-byte core matrices; LBO = 128 B along K, SBO = 1024 B along M/N).  One
// elected thread issues `tcgen05.mma.cta_group::1.kind::tf32` (M=128, N=P_pad,
// K=8) into a TMEM accumulator and commits to an mbarrier; staging is double
// buffered so the next chunk's loads overlap the MMAs.  The epilogue reads the
// accumulator with `tcgen05.ld.32x32b` — TMEM lane = patch — and writes the
// plane-major estimates (P, N) with coalesced stores.
#include "pb_compose_tc.cuh"

namespace pb {

namespace {

constexpr int kTcM = 128;      // patches per tile (UMMA M, TMEM lanes)
constexpr int kTcKc = 32;      // atoms per staged chunk
constexpr int kTcThreads = 256;   // 2 threads per patch row while staging; warps 0-3 own the epilogue

__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ float to_tf32(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

// K-major, no swizzle: ((8,n),2):((16B,SBO),LBO) per K=8 tf32 step
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // descriptor version (sm100)
  // base offset 0, lbo mode 0, layout type 0 = SWIZZLE_NONE
  return d;
}

// kind::tf32 instruction descriptor: D f32, A/B tf32, both K-major
__host__ __device__ constexpr uint32_t umma_idesc_tf32(int m, int n) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(accum));
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_addr(bar))
               : "memory");
}

__device__ __forceinline__ void mbar_init1(uint64_t* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait_parity(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "W_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra W_%=;\n}" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int j = 0; j < 16; ++j) v[j] = __uint_as_float(r[j]);
}

// Byte offset of element (row, k) (k inside the 32-atom chunk) of a K-major
// canonical tile: core matrix = 8 rows x 16 B, LBO = 128 B (along K), SBO = 1024 B.
__device__ __forceinline__ uint32_t kmajor_off(int row, int k) {
  return (uint32_t)((row >> 3) * 1024 + (k >> 2) * 128 + (row & 7) * 16 + (k & 3) * 4);
}

}  // namespace

template <int NPAD>
__global__ void __launch_bounds__(kTcThreads, 1)
    k_compose_tc(const uint8_t* __restrict__ usage, const float* __restrict__ weights, int64_t ld,
                 const float* __restrict__ atoms, int p, int k_len, int64_t n, float* __restrict__ out, int accumulate) {
  constexpr int A_BYTES = kTcM * kTcKc * 4;    // 16 KB
  constexpr int B_BYTES = NPAD * kTcKc * 4;
  constexpr int STAGE = 2 * A_BYTES + 2 * B_BYTES;  // hi + lo of A and B
  constexpr uint32_t TMEM_COLS = NPAD <= 32 ? 32 : NPAD <= 64 ? 64 : NPAD <= 128 ? 128 : 256;
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ __align__(8) uint64_t mbar[2];
  __shared__ uint32_t tmem_base_sh;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_addr(&tmem_base_sh)),
                 "n"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    mbar_init1(&mbar[0]);
    mbar_init1(&mbar[1]);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base_sh;

  constexpr uint32_t idesc = umma_idesc_tf32(kTcM, NPAD);
  const int nchunks = (k_len + kTcKc - 1) / kTcKc;
  const int64_t ntiles = (n + kTcM - 1) / kTcM;
  uint32_t issued = 0;        // chunks issued so far (stage = issued & 1)
  uint32_t phase[2] = {0, 0};

  // this thread stages row `srow` of the patch tile, atoms [half*16, half*16+16) of each chunk;
  // the raw (z, s) loads of the NEXT chunk are issued before the current one is written out
  const int srow = tid & (kTcM - 1), half = tid / kTcM;
  constexpr int KH = kTcKc / 2;
  uint32_t zc[KH], zn[KH];
  float sc[KH], sn[KH];
  auto load_raw = [&](int64_t tile, int c, uint32_t (&z)[KH], float (&sv)[KH]) {
    const int64_t i = tile * kTcM + srow;
    const bool live = tile < ntiles && i < n && c < nchunks;
#pragma unroll
    for (int u = 0; u < KH; ++u) {
      const int k = c * kTcKc + half * KH + u;
      z[u] = 0;
      sv[u] = 0.0f;
      if (live && k < k_len) {
        const int64_t zi = (int64_t)k * ld + i;
        z[u] = usage[zi];
        sv[u] = weights[zi];
      }
    }
  };
  load_raw(blockIdx.x, 0, zc, sc);

  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t i0 = tile * kTcM;
    for (int c = 0; c < nchunks; ++c, ++issued) {
      const int s = issued & 1;
      unsigned char* st = sm + s * STAGE;
      // prefetch the next chunk (or the next tile's first chunk)
      if (c + 1 < nchunks) load_raw(tile, c + 1, zn, sn);
      else load_raw(tile + gridDim.x, 0, zn, sn);
      if (issued >= 2) {  // the MMAs that last read this stage must be done
        mbar_wait_parity(&mbar[s], phase[s]);
        phase[s] ^= 1u;
      }
      // ---- stage A: w = z ? s : 0 split into TF32 hi + lo ----
      {
        float* ahi = (float*)st;
        float* alo = (float*)(st + A_BYTES);
#pragma unroll
        for (int q = 0; q < KH / 4; ++q) {
          float hv[4], lv[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const float w = zc[q * 4 + u] ? sc[q * 4 + u] : 0.0f;
            hv[u] = to_tf32(w);
            lv[u] = to_tf32(w - hv[u]);
          }
          const uint32_t off = kmajor_off(srow, half * KH + q * 4);
          *(float4*)((unsigned char*)ahi + off) = make_float4(hv[0], hv[1], hv[2], hv[3]);
          *(float4*)((unsigned char*)alo + off) = make_float4(lv[0], lv[1], lv[2], lv[3]);
        }
      }
#pragma unroll
      for (int u = 0; u < KH; ++u) { zc[u] = zn[u]; sc[u] = sn[u]; }
      // ---- stage B: row = pixel n (< NPAD), 32 atoms of D, hi/lo ----
      {
        float* bhi = (float*)(st + 2 * A_BYTES);
        float* blo = (float*)(st + 2 * A_BYTES + B_BYTES);
        for (int t = tid; t < NPAD * (kTcKc / 4); t += kTcThreads) {
          const int row = t % NPAD, q = t / NPAD;
          float hv[4], lv[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int k = c * kTcKc + q * 4 + u;
            const float d = (row < p && k < k_len) ? atoms[(int64_t)k * p + row] : 0.0f;
            hv[u] = to_tf32(d);
            lv[u] = to_tf32(d - hv[u]);
          }
          const uint32_t off = kmajor_off(row, q * 4);
          *(float4*)((unsigned char*)bhi + off) = make_float4(hv[0], hv[1], hv[2], hv[3]);
          *(float4*)((unsigned char*)blo + off) = make_float4(lv[0], lv[1], lv[2], lv[3]);
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncthreads();
      if (tid == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t a_hi = smem_addr(st), a_lo = a_hi + A_BYTES;
        const uint32_t b_hi = a_hi + 2 * A_BYTES, b_lo = b_hi + B_BYTES;
#pragma unroll
        for (int ks = 0; ks < kTcKc / 8; ++ks) {  // K = 8 tf32 per MMA = two 16-byte core-matrix columns
          const uint32_t ko = ks * 256;
          const uint32_t acc0 = (c > 0 || ks > 0) ? 1u : 0u;
          mma_tf32(tmem, umma_desc(a_hi + ko, 128, 1024), umma_desc(b_hi + ko, 128, 1024), idesc, acc0);
          mma_tf32(tmem, umma_desc(a_hi + ko, 128, 1024), umma_desc(b_lo + ko, 128, 1024), idesc, 1u);
          mma_tf32(tmem, umma_desc(a_lo + ko, 128, 1024), umma_desc(b_hi + ko, 128, 1024), idesc, 1u);
        }
        mma_commit(&mbar[s]);
      }
    }
    // ---- epilogue: wait for the tile's last commit, TMEM -> registers -> est ----
    {
      const int s = (issued - 1) & 1;
      mbar_wait_parity(&mbar[s], phase[s]);
      phase[s] ^= 1u;
      // the other stage's last commit (if any this tile) completed before (in-order MMAs)
      if (nchunks >= 2) {
        const int s2 = (issued - 2) & 1;
        mbar_wait_parity(&mbar[s2], phase[s2]);
        phase[s2] ^= 1u;
      }
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const int64_t i = i0 + (warp & 3) * 32 + lane;
      const uint32_t taddr = tmem + ((uint32_t)((warp & 3) * 32) << 16);
      // warps w and w+4 share TMEM subpartition w%4 and split its columns
#pragma unroll 1
      for (int c0 = (warp >> 2) * 16; c0 < NPAD; c0 += 32) {
        float v[16];
        tmem_ld16(taddr + c0, v);
        if (i < n) {
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const int pe = c0 + j;
            if (pe < p) {
              float* o = out + (int64_t)pe * n + i;
              *o = accumulate ? *o + v[j] : v[j];
            }
          }
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncthreads();   // the accumulator is reused by the next tile
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      issued = 0;        // both stages drained: restart the stage sequence
    }
  }
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(TMEM_COLS));
}

static int sms_tc() {
  int dev = 0, v = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
  return v;
}

template <int NPAD>
static int launch_tc(const uint8_t* usage, const float* weights, int64_t ld, const float* atoms, int p, int k_len,
                     int64_t n, float* out, int accumulate, cudaStream_t st) {
  constexpr int STAGE = 2 * (kTcM * kTcKc * 4) + 2 * (NPAD * kTcKc * 4);
  const size_t smem = 2 * (size_t)STAGE + 1024;
  auto kern = k_compose_tc<NPAD>;
  PB_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int64_t ntiles = (n + kTcM - 1) / kTcM;
  int64_t grid = std::min<int64_t>(ntiles, (int64_t)sms_tc() * (smem <= 110 * 1024 ? 2 : 1));
  if (grid < 1) grid = 1;
  kern<<<(unsigned)grid, kTcThreads, smem, st>>>(usage, weights, ld, atoms, p, k_len, n, out, accumulate);
  PB_LAUNCH_CHECK();
  return PB_OK;
}

bool compose_tc_supported(int p) { return p >= 1 && p <= 256; }

int launch_compose_tc(const uint8_t* usage, const float* weights, int64_t ld, const float* atoms, int p, int k_len,
                      int64_t n, float* out, int accumulate, cudaStream_t st) {
  if (n <= 0) return PB_OK;
  const int npad = (p + 15) / 16 * 16;
  if (npad <= 64) return launch_tc<64>(usage, weights, ld, atoms, p, k_len, n, out, accumulate, st);
  if (npad <= 112) return launch_tc<112>(usage, weights, ld, atoms, p, k_len, n, out, accumulate, st);
  if (npad <= 128) return launch_tc<128>(usage, weights, ld, atoms, p, k_len, n, out, accumulate, st);
  if (npad <= 256) return launch_tc<256>(usage, weights, ld, atoms, p, k_len, n, out, accumulate, st);
  set_error("tensor-core compose supports P <= 256 (got %d)", p);
  return PB_EUNSUPPORTED;
}

}  // namespace pb
