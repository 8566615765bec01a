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

// Canonical K-major no-swizzle tile (core matrix = 8 rows x 16 B contiguous):
// consecutive 8-row groups are SBO = 144 B apart (128 + 16: the 16-byte skew
// makes the stagers' 16-byte stores of 8 rows from 4 groups hit 8 distinct bank
// quads), and the 4-atom columns are LBO = rows/8 * 144 B apart.
constexpr uint32_t kSbo = 144;
__host__ __device__ constexpr uint32_t kmajor_lbo(int rows) { return (uint32_t)(rows / 8) * kSbo; }
__device__ __forceinline__ uint32_t kmajor_off(int rows, int row, int k) {
  return (uint32_t)((k >> 2) * kmajor_lbo(rows) + (row >> 3) * kSbo + (row & 7) * 16 + (k & 3) * 4);
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes) : "memory");
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_addr(dst)),
               "l"(src), "r"(bytes), "r"(smem_addr(bar))
               : "memory");
}

}  // namespace

// D (K, P) -> per 32-atom chunk, the TF32 hi and lo parts of D^T in the
// canonical K-major layout the MMA reads ([chunk][hi|lo][NPAD x 32]); staged by
// one bulk copy per chunk and stage in the main kernel.
__global__ void k_compose_pack_b(const float* __restrict__ atoms, int p, int k_len, int npad, int nchunks,
                                 float* __restrict__ packed) {
  const int per = npad * kTcKc;                                   // elements per part
  const int part = (int)((kTcKc / 4) * kmajor_lbo(npad) / 4);     // floats per part (skewed layout)
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < nchunks * per; t += gridDim.x * blockDim.x) {
    const int c = t / per, r = t - c * per;
    const int row = r / kTcKc, kk = r - row * kTcKc, k = c * kTcKc + kk;
    const float d = (row < p && k < k_len) ? atoms[(int64_t)k * p + row] : 0.0f;
    const float hi = to_tf32(d), lo = to_tf32(d - hi);
    float* base = packed + (size_t)c * 2 * part;
    const uint32_t off = kmajor_off(npad, row, kk) / 4;
    base[off] = hi;
    base[part + off] = lo;
  }
}

template <int NPAD>
__global__ void __launch_bounds__(kTcThreads, 1)
    k_compose_tc(const uint8_t* __restrict__ usage, const float* __restrict__ weights, int64_t ld,
                 const float* __restrict__ bpack, int p, int k_len, int64_t n, float* __restrict__ out, int accumulate) {
  constexpr int A_BYTES = (kTcKc / 4) * kmajor_lbo(kTcM);   // 8 atom quads x 16 row groups x 144 B
  constexpr int B_BYTES = (kTcKc / 4) * kmajor_lbo(NPAD);
  constexpr int STAGE = 2 * A_BYTES + 2 * B_BYTES;  // hi + lo of A and B
  constexpr uint32_t TMEM_COLS = NPAD <= 32 ? 32 : NPAD <= 64 ? 64 : NPAD <= 128 ? 128 : 256;
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ __align__(8) uint64_t mbar[2];
  __shared__ __align__(8) uint64_t bfull[2];   // the B bulk copy of a stage has landed
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
    mbar_init1(&bfull[0]);
    mbar_init1(&bfull[1]);
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
  uint32_t phase[2] = {0, 0}, bphase[2] = {0, 0};

  // this thread stages a 4-patch x 4-atom block of each chunk: patches
  // 4*rq .. 4*rq+3, atoms 4*kq .. 4*kq+3 (one 4-byte z load and one 16-byte s
  // load per atom, coalesced across the warp); the raw loads of the NEXT chunk
  // are issued before the current one is written out
  const int rq = tid & 31, kq = tid >> 5;   // 32 row quads x 8 atom quads = 256 threads
  uint32_t zc[4], zn[4];
  float4 sc[4], sn[4];
  auto load_raw = [&](int64_t tile, int c, uint32_t (&z)[4], float4 (&sv)[4]) {
    const int64_t i = tile * kTcM + 4 * rq;
    const bool live = tile < ntiles && i < n && c < nchunks;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int k = c * kTcKc + kq * 4 + u;
      z[u] = 0;
      sv[u] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (live && k < k_len) {   // ld and the tile base are multiples of 4: aligned vectors
        const int64_t zi = (int64_t)k * ld + i;
        z[u] = *(const uint32_t*)(usage + zi);
        sv[u] = *(const float4*)(weights + zi);
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
      if (tid == 0) {  // B (D^T hi + lo, pre-packed) for this chunk: one bulk copy
        mbar_expect_tx(&bfull[s], 2 * B_BYTES);
        bulk_g2s(st + 2 * A_BYTES, bpack + (size_t)c * (2 * B_BYTES / 4), 2 * B_BYTES, &bfull[s]);
      }
      // ---- stage A: w = z ? s : 0, split into TF32 hi + lo, one 16-byte row chunk per patch ----
      {
        unsigned char* ahi = st;
        unsigned char* alo = st + A_BYTES;
#pragma unroll
        for (int j = 0; j < 4; ++j) {   // patch 4*rq + j: atoms 4*kq .. 4*kq+3
          float w[4], hv[4], lv[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const float sv = j == 0 ? sc[u].x : j == 1 ? sc[u].y : j == 2 ? sc[u].z : sc[u].w;
            w[u] = ((zc[u] >> (8 * j)) & 0xFFu) ? sv : 0.0f;
            hv[u] = to_tf32(w[u]);
            lv[u] = to_tf32(w[u] - hv[u]);
          }
          const uint32_t off = kmajor_off(kTcM, 4 * rq + j, 4 * kq);
          *(float4*)(ahi + off) = make_float4(hv[0], hv[1], hv[2], hv[3]);
          *(float4*)(alo + off) = make_float4(lv[0], lv[1], lv[2], lv[3]);
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) { zc[u] = zn[u]; sc[u] = sn[u]; }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncthreads();
      if (tid == 0) {
        mbar_wait_parity(&bfull[s], bphase[s]);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t a_hi = smem_addr(st), a_lo = a_hi + A_BYTES;
        const uint32_t b_hi = a_hi + 2 * A_BYTES, b_lo = b_hi + B_BYTES;
        constexpr uint32_t LA = kmajor_lbo(kTcM), LB = kmajor_lbo(NPAD);
#pragma unroll
        for (int ks = 0; ks < kTcKc / 8; ++ks) {  // K = 8 tf32 per MMA = two 4-atom core-matrix columns
          const uint32_t oa = ks * 2 * LA, ob = ks * 2 * LB;
          const uint32_t acc0 = (c > 0 || ks > 0) ? 1u : 0u;
          mma_tf32(tmem, umma_desc(a_hi + oa, LA, kSbo), umma_desc(b_hi + ob, LB, kSbo), idesc, acc0);
          mma_tf32(tmem, umma_desc(a_hi + oa, LA, kSbo), umma_desc(b_lo + ob, LB, kSbo), idesc, 1u);
          mma_tf32(tmem, umma_desc(a_lo + oa, LA, kSbo), umma_desc(b_hi + ob, LB, kSbo), idesc, 1u);
        }
        mma_commit(&mbar[s]);
      }
      bphase[s] ^= 1u;
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
static size_t packed_bytes(int k_len) {
  return (size_t)((k_len + kTcKc - 1) / kTcKc) * 2 * (kTcKc / 4) * kmajor_lbo(NPAD);
}

template <int NPAD>
static int launch_tc(const uint8_t* usage, const float* weights, int64_t ld, const float* atoms, int p, int k_len,
                     int64_t n, float* out, int accumulate, float* scratch, cudaStream_t st) {
  constexpr int STAGE = 2 * (kTcKc / 4) * (int)kmajor_lbo(kTcM) + 2 * (kTcKc / 4) * (int)kmajor_lbo(NPAD);
  const size_t smem = 2 * (size_t)STAGE + 1024;
  const int nchunks = (k_len + kTcKc - 1) / kTcKc;
  // the packed D^T chunks (TF32 hi + lo): caller scratch, or a stream-ordered allocation
  float* bpack = scratch;
  static bool pool_kept = false;
  if (!scratch && !pool_kept) {  // keep the stream-ordered pool's memory between calls (no OS round trip)
    int dev = 0;
    cudaMemPool_t pool;
    cudaGetDevice(&dev);
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t keep = 64ull << 20;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    pool_kept = true;
  }
  if (!bpack && cudaMallocAsync((void**)&bpack, packed_bytes<NPAD>(k_len), st) != cudaSuccess) {
    set_error("compose: scratch allocation failed");
    return PB_ECUDA;
  }
  k_compose_pack_b<<<std::max(1, std::min(nchunks * NPAD * kTcKc / 256, 1184)), 256, 0, st>>>(atoms, p, k_len, NPAD,
                                                                                          nchunks, bpack);
  auto kern = k_compose_tc<NPAD>;
  int rc = PB_OK;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
    set_error("compose: shared-memory attribute rejected");
    rc = PB_ECUDA;
  } else {
    const int64_t ntiles = (n + kTcM - 1) / kTcM;
    int64_t grid = std::min<int64_t>(ntiles, (int64_t)sms_tc() * (smem <= 110 * 1024 ? 2 : 1));
    if (grid < 1) grid = 1;
    kern<<<(unsigned)grid, kTcThreads, smem, st>>>(usage, weights, ld, bpack, p, k_len, n, out, accumulate);
    if (cudaGetLastError() != cudaSuccess) { set_error("compose: launch failed"); rc = PB_ECUDA; }
  }
  if (!scratch) cudaFreeAsync(bpack, st);
  return rc;
}

bool compose_tc_supported(int p) { return p >= 1 && p <= 256; }

size_t compose_tc_scratch_bytes(int p, int k_len) {
  const int npad = (p + 15) / 16 * 16;
  return npad <= 64 ? packed_bytes<64>(k_len) : npad <= 112 ? packed_bytes<112>(k_len)
       : npad <= 128 ? packed_bytes<128>(k_len) : packed_bytes<256>(k_len);
}

int launch_compose_tc(const uint8_t* usage, const float* weights, int64_t ld, const float* atoms, int p, int k_len,
                      int64_t n, float* out, int accumulate, cudaStream_t st, float* scratch) {
  if (n <= 0) return PB_OK;
  const int npad = (p + 15) / 16 * 16;
  if (npad <= 64) return launch_tc<64>(usage, weights, ld, atoms, p, k_len, n, out, accumulate, scratch, st);
  if (npad <= 112) return launch_tc<112>(usage, weights, ld, atoms, p, k_len, n, out, accumulate, scratch, st);
  if (npad <= 128) return launch_tc<128>(usage, weights, ld, atoms, p, k_len, n, out, accumulate, scratch, st);
  if (npad <= 256) return launch_tc<256>(usage, weights, ld, atoms, p, k_len, n, out, accumulate, scratch, st);
  set_error("tensor-core compose supports P <= 256 (got %d)", p);
  return PB_EUNSUPPORTED;
}

}  // namespace pb
