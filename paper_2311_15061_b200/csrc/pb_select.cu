// pb200 — top-n selection over 64-bit keys (radix select), the ordering
// primitive behind the live path's adaptive-residual mask (sampling.py:184-207)
// and the data-mode dictionary seeding (bpfa.py:126-134).
//
// Both reference call sites are a STABLE sort followed by "take the first n":
//   exploit set      argsort(-residual, kind="stable")[:n_exploit]
//   explore set      Generator.choice(free, n, replace=False)  (here: the n
//                    smallest per-element Philox keys, ties by index)
//   data seeding     argsort(-counts, kind="stable")[:K]
// so only the SET of the n largest keys (ties by lowest index) is needed, not
// the order of all m elements.  A radix select finds the threshold key T with
// count(key > T) < n <= count(key >= T) in six histogram passes (11/11/11/11/
// 11/9 bits, a 2048-bin shared histogram per CTA, one global histogram, one
// warp choosing the digit), then one ordered pass takes every key > T and the
// first n - count(key > T) keys == T in index order (per-CTA tie counts, an
// exclusive scan, per-thread ranks).  HBM traffic: 7 reads of the 8-byte keys
// (+ the mark writes) — no (key, index) pair sorting, no library sort.
// The data seeding also needs the ORDER of its K selected patches: K is small
// (the atom count), so one CTA ranks them by (count desc, index asc).
#include <algorithm>

#include "pb_live.cuh"

namespace pb {

namespace {

constexpr int kSelThreads = 256;
constexpr int kSelPer = 8;                             // consecutive keys per thread in the ordered pass
constexpr int kSelChunk = kSelThreads * kSelPer;       // keys per CTA in the ordered pass
constexpr int kSelPasses = 6;
__host__ __device__ constexpr int sel_shift(int pass) { return pass < 5 ? 53 - 11 * pass : 0; }
__host__ __device__ constexpr int sel_width(int pass) { return pass < 5 ? 11 : 9; }

// state: [0] prefix (the digits of T fixed so far), [1] mask of those digits,
// [2] keys still wanted among those matching the prefix
struct SelState {
  unsigned long long prefix, fixed, want;
};

__global__ void __launch_bounds__(kSelThreads) k_sel_hist(const uint64_t* __restrict__ keys, int64_t m,
                                                           const SelState* __restrict__ state, int pass,
                                                           unsigned* __restrict__ hist) {
  __shared__ unsigned sh[2048];
  const int shift = sel_shift(pass), nb = 1 << sel_width(pass);
  for (int b = threadIdx.x; b < nb; b += blockDim.x) sh[b] = 0;
  __syncthreads();
  const unsigned long long prefix = state->prefix, fixed = state->fixed;
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < m; x += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long k = keys[x];
    if (((k ^ prefix) & fixed) == 0) atomicAdd(&sh[(k >> shift) & (nb - 1)], 1u);
  }
  __syncthreads();
  for (int b = threadIdx.x; b < nb; b += blockDim.x)
    if (sh[b]) atomicAdd(&hist[b], sh[b]);
}

// One warp: the digit holding the want-th largest key among those matching the
// prefix (bins scanned from the top), then the histogram cleared for the next pass.
__global__ void k_sel_pick(SelState* __restrict__ state, int pass, unsigned* __restrict__ hist) {
  const int lane = threadIdx.x, shift = sel_shift(pass), nb = 1 << sel_width(pass), per = nb / 32;
  const unsigned long long want = state->want;
  // lane l owns bins [nb - (l+1)*per, nb - l*per), visited from the top
  const int top = nb - lane * per;
  unsigned long long s = 0;
  for (int q = 1; q <= per; ++q) s += hist[top - q];
  unsigned long long incl = s;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  const unsigned long long before = incl - s;
  if (before < want && want <= incl) {
    unsigned long long c = before;
    for (int q = 1; q <= per; ++q) {
      const int b = top - q;
      if (c + hist[b] >= want) {
        state->want = want - c;
        state->prefix |= (unsigned long long)b << shift;
        state->fixed |= (unsigned long long)(nb - 1) << shift;
        break;
      }
      c += hist[b];
    }
  }
  __syncwarp();
  for (int b = lane; b < nb; b += 32) hist[b] = 0;
}

__device__ __forceinline__ unsigned block_excl_scan(unsigned v, unsigned* wsum, unsigned& total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  unsigned incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) wsum[w] = incl;
  __syncthreads();
  unsigned wpre = 0;
  total = 0;
  for (int q = 0; q < kSelThreads / 32; ++q) {
    if (q < w) wpre += wsum[q];
    total += wsum[q];
  }
  __syncthreads();
  return wpre + incl - v;
}

// Ties (key == T) per CTA chunk of kSelChunk consecutive keys.
__global__ void __launch_bounds__(kSelThreads) k_sel_tie_count(const uint64_t* __restrict__ keys, int64_t m,
                                                                const SelState* __restrict__ state,
                                                                unsigned* __restrict__ cnt) {
  __shared__ unsigned wsum[kSelThreads / 32];
  const unsigned long long t = state->prefix;
  const int64_t base = (int64_t)blockIdx.x * kSelChunk + (int64_t)threadIdx.x * kSelPer;
  unsigned c = 0;
#pragma unroll
  for (int q = 0; q < kSelPer; ++q)
    if (base + q < m && keys[base + q] == t) ++c;
  unsigned total;
  block_excl_scan(c, wsum, total);
  if (threadIdx.x == 0) cnt[blockIdx.x] = total;
}

// Exclusive scan of the per-CTA tie counts (one CTA; nblk up to a few 10^4).
__global__ void __launch_bounds__(1024) k_sel_scan(unsigned* __restrict__ cnt, int nblk) {
  __shared__ unsigned long long part[1024];
  const int per = (nblk + 1023) / 1024, b0 = threadIdx.x * per;
  unsigned long long s = 0;
  for (int q = 0; q < per; ++q)
    if (b0 + q < nblk) s += cnt[b0 + q];
  part[threadIdx.x] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long run = 0;
    for (int q = 0; q < 1024; ++q) { const unsigned long long v = part[q]; part[q] = run; run += v; }
  }
  __syncthreads();
  unsigned long long run = part[threadIdx.x];
  for (int q = 0; q < per; ++q)
    if (b0 + q < nblk) { const unsigned v = cnt[b0 + q]; cnt[b0 + q] = (unsigned)run; run += v; }
}

// The selection: every key > T, and the ties whose index rank among the ties
// is < want.  mark[x] = 1 for selected x (if mark); selected indices appended
// to list (if list; unordered).
__global__ void __launch_bounds__(kSelThreads) k_sel_take(const uint64_t* __restrict__ keys, int64_t m,
                                                           const SelState* __restrict__ state,
                                                           const unsigned* __restrict__ tie_off,
                                                           uint8_t* __restrict__ mark, int32_t* __restrict__ list,
                                                           unsigned* __restrict__ list_n) {
  __shared__ unsigned wsum[kSelThreads / 32];
  const unsigned long long t = state->prefix, want = state->want;
  const int64_t base = (int64_t)blockIdx.x * kSelChunk + (int64_t)threadIdx.x * kSelPer;
  unsigned long long k[kSelPer];
  unsigned c = 0;
#pragma unroll
  for (int q = 0; q < kSelPer; ++q) {
    k[q] = base + q < m ? keys[base + q] : 0ull;
    c += (base + q < m && k[q] == t) ? 1u : 0u;
  }
  unsigned total;
  unsigned long long rank = (unsigned long long)tie_off[blockIdx.x] + block_excl_scan(c, wsum, total);
#pragma unroll
  for (int q = 0; q < kSelPer; ++q) {
    if (base + q >= m) break;
    bool take = k[q] > t;
    if (k[q] == t) take = rank++ < want;
    if (take) {
      if (mark) mark[base + q] = 1;
      if (list) list[atomicAdd(list_n, 1u)] = (int32_t)(base + q);
    }
  }
}

__global__ void k_sel_init(SelState* state, unsigned long long n) {
  state->prefix = 0;
  state->fixed = 0;
  state->want = n;
}

unsigned sel_grid(int64_t m) {
  int64_t nb = (m + kSelThreads - 1) / kSelThreads;
  if (nb > 148 * 8) nb = 148 * 8;
  return (unsigned)(nb < 1 ? 1 : nb);
}

}  // namespace

size_t select_scratch_bytes(int64_t m) {
  const int64_t nblk = (m + kSelChunk - 1) / kSelChunk;
  return 256 + 2048 * 4 + (size_t)nblk * 4 + 256;
}

// Selects the n largest of keys[0, m) (ties by lowest index), 1 <= n <= m.
int select_top(const uint64_t* keys, int64_t m, int64_t n, void* scratch, uint8_t* mark, int32_t* list,
               cudaStream_t st) {
  if (n <= 0 || m <= 0) return PB_OK;
  if (n > m) { set_error("select_top: n (%lld) > m (%lld)", (long long)n, (long long)m); return PB_EVALUE; }
  const int64_t nblk = (m + kSelChunk - 1) / kSelChunk;
  if (nblk > ((int64_t)1 << 30)) { set_error("select_top: too many keys"); return PB_EUNSUPPORTED; }
  char* s = (char*)scratch;
  SelState* state = (SelState*)s;                       // 24 B (+ list count at 64)
  unsigned* list_n = (unsigned*)(s + 64);
  unsigned* hist = (unsigned*)(s + 256);
  unsigned* cnt = hist + 2048;
  cudaMemsetAsync(s, 0, 256 + 2048 * 4, st);
  k_sel_init<<<1, 1, 0, st>>>(state, (unsigned long long)n);
  const unsigned g = sel_grid(m);
  for (int pass = 0; pass < kSelPasses; ++pass) {
    k_sel_hist<<<g, kSelThreads, 0, st>>>(keys, m, state, pass, hist);
    k_sel_pick<<<1, 32, 0, st>>>(state, pass, hist);
  }
  k_sel_tie_count<<<(unsigned)nblk, kSelThreads, 0, st>>>(keys, m, state, cnt);
  k_sel_scan<<<1, 1024, 0, st>>>(cnt, (int)nblk);
  k_sel_take<<<(unsigned)nblk, kSelThreads, 0, st>>>(keys, m, state, cnt, mark, list, list_n);
  PB_LAUNCH_CHECK();
  return PB_OK;
}

}  // namespace pb
