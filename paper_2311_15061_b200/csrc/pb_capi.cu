// pb200 — C ABI (include/pb200.h) over the sm_100a kernels, plus the native
// stateful "problem" used for the host-buffer live-frame path.
#include <math.h>
#include <stdarg.h>
#include <stdlib.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <vector>

#include "../../include/pb200.h"
#include "pb_compact.cuh"
#include "pb_live.cuh"
#include "pb_compose_tc.cuh"

namespace pb {
int launch_transfer_atoms(const float* src, int k, int src_p, int repeat, int normalize, float* dst, cudaStream_t st);
}

namespace pb {

// ---- error state ----------------------------------------------------------
static thread_local char g_err[1024] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}
const char* last_error() { return g_err; }

static int make_grid(const pb_grid_desc* d, Grid& g) {
  if (!d) { set_error("null grid"); return PB_EVALUE; }
  if (d->rank < 1 || d->rank > kMaxRank) { set_error("tensor rank must be 1..4, got %d", d->rank); return PB_ESHAPE; }
  g.rank = d->rank;
  g.n = 1; g.p = 1; g.m = 1;
  for (int i = 0; i < d->rank; ++i) {
    const int64_t m = d->tensor_shape[i];
    const int b = d->patch_shape[i], s = d->stride[i];
    if (m < 1) { set_error("tensor dims must be >= 1"); return PB_ESHAPE; }
    if (b < 1) { set_error("patch dims must be >= 1"); return PB_ESHAPE; }
    if (s < 1) { set_error("strides must be >= 1"); return PB_ESHAPE; }
    if (b > m) { set_error("patch shape exceeds tensor in dim %d (%d > %lld)", i, b, (long long)m); return PB_ESHAPE; }
    g.tshape[i] = m; g.bshape[i] = b; g.step[i] = s;
    g.gcount[i] = (m - b) / s + 1;
    g.n *= g.gcount[i]; g.p *= b; g.m *= m;
  }
  int64_t acc = 1;
  for (int i = d->rank - 1; i >= 0; --i) { g.tstride[i] = acc; acc *= g.tshape[i]; }
  return PB_OK;
}

// Epoch workspace carve-up
struct EpochWs {
  float* r_csc;
  float* wt;        // tile-blocked code copy [tile][k/8][patch][8]
  size_t wt_bytes;
  float* partials;
  double* reduced;
  unsigned* bar;
  double* block_sums;
  int32_t* m_count;
  float* delta_g;   // atom shifts of the last updated block [8][P] (dictionary step exchange)
  unsigned* ctr;    // dynamic block counters of the code-step launches [2]
  float* dt_img;    // the code step's pre-packed transposed dictionary chunks
};
static const int kMaxDictBlocks = 148 * 8;
static size_t align256(size_t x) { return (x + 255) & ~size_t(255); }
static size_t ws_bytes(int64_t n, int p, int k, int64_t nnz, EpochWs* ws, char* base) {
  size_t off = 0;
  auto take = [&](size_t bytes) { size_t o = off; off += align256(bytes); return base ? base + o : nullptr; };
  char* r = take((size_t)ell_cap(n, nnz) * 4);   // residual in the ELL wave order
  const size_t wtb = (size_t)ceil_div(n, kTile) * ceil_div(k, kWB) * kTile * kWB * 4;
  char* wt = take(wtb);
  char* pa = take(dict_gram_partials_bytes(p, kMaxDictBlocks));
  char* rd = take(dict_gram_reduced_bytes(p));
  char* bar = take(16 + (size_t)p * 4);   // grid-barrier counters, then per-pixel ready flags
  char* bs = take((size_t)(ceil_div(n * 64, 256) + 8) * 2 * 8);  // upper bound of code-step blocks (two launches)
  char* mc = take((size_t)k * 4);
  char* dg = take((size_t)8 * p * 4);
  char* ct = take(16);
  int dt_nch = 0;
  int64_t dt_imgf = 0;
  code_dt_layout(p, k, nullptr, &dt_imgf, &dt_nch);
  char* di = take((size_t)dt_imgf * dt_nch * 4);
  if (ws) {
    ws->ctr = (unsigned*)ct;
    ws->dt_img = (float*)di;
    ws->delta_g = (float*)dg;
    ws->r_csc = (float*)r; ws->wt = (float*)wt; ws->wt_bytes = wtb;
    ws->partials = (float*)pa; ws->reduced = (double*)rd;
    ws->bar = (unsigned*)bar; ws->block_sums = (double*)bs; ws->m_count = (int32_t*)mc;
  }
  return off;
}

static void index_view(const pb_patch_index* pi, PatchIndex& ix) {
  carve_index(ix, (char*)pi->buffer, pi->n, pi->p, pi->nnz);
}

static void device_key(uint64_t seed, uint32_t& k0, uint32_t& k1) {
  // splitmix64 of the seed; the Python side uses the same derivation only as a
  // label — device draws are keyed solely by this pair.
  uint64_t z = seed + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  z ^= z >> 31;
  k0 = (uint32_t)z;
  k1 = (uint32_t)(z >> 32);
}

// Optional phase timing (bench / profiling): events bracketing the epoch's
// kernels on the launching stream, one fresh event set per epoch (no host
// synchronization until pb_phase_read).
enum { kPhResid = 0, kPhDict, kPhCode, kPhStats, kPhEnd, kNumPh };
struct PhaseSet { cudaEvent_t ev[kNumPh]; };
static bool g_phase_on = false;
static std::vector<PhaseSet> g_phase_sets;
static size_t g_phase_used = 0;
static PhaseSet* g_phase_cur = nullptr;

static void phase_begin() {
  g_phase_cur = nullptr;
  if (!g_phase_on) return;
  if (g_phase_used == g_phase_sets.size()) {
    PhaseSet ps;
    for (int i = 0; i < kNumPh; ++i) cudaEventCreate(&ps.ev[i]);
    g_phase_sets.push_back(ps);
  }
  g_phase_cur = &g_phase_sets[g_phase_used++];
}
static void phase_mark(int ph, cudaStream_t st) {
  if (g_phase_cur) cudaEventRecord(g_phase_cur->ev[ph], st);
}

// Optional in-kernel phase profile of the dictionary step (globaltimer, CTA 0..n thread 0).
static unsigned long long* g_dict_prof = nullptr;
static unsigned long long* g_wave_prof = nullptr;   // tuning builds: per-wave profile of the last epoch

static int run_epoch(const pb_epoch_desc* d, int32_t* m_out, cudaStream_t st) {
  phase_begin();
  if (d->n < 1 || d->p < 1 || d->k < 1) { set_error("empty problem"); return PB_ESHAPE; }
  if (!d->index || !d->index->buffer || d->index->n != d->n || d->index->p != d->p) {
    set_error("pb_gibbs_epoch needs the patch index of this patch matrix (pb_build_index)");
    return PB_EVALUE;
  }
  if (d->rng_mode == PB_RNG_REPLAY && (!d->code_u || !d->code_g || (!d->freeze_dict && !d->atom_draws))) {
    set_error("replay mode needs atom_draws, code_u and code_g");
    return PB_EVALUE;
  }
  PatchIndex ix;
  index_view(d->index, ix);
  EpochWs ws;
  ws_bytes(d->n, d->p, d->k, d->index->nnz, &ws, (char*)d->workspace);
  if (m_out) ws.m_count = m_out;
  uint32_t k0, k1;
  device_key(d->seed, k0, k1);
  SweepScalars* sc = (SweepScalars*)d->scalars;
  CompactArgs c{};
  c.counts = d->counts; c.rowptr = ix.rowptr; c.csr_p = ix.csr_p; c.csr_pos = ix.csr_pos;
  c.x_csc = ix.x_csc; c.r_csc = ws.r_csc; c.cmax = d->index->cmax;
  c.wt = ws.wt; c.nblk8 = (int)ceil_div(d->k, kWB);
  c.usage = d->usage; c.weights = d->weights; c.atoms = d->atoms; c.pi = d->pi; c.sc = sc;
  c.u_draw = d->rng_mode == PB_RNG_REPLAY ? d->code_u : nullptr;
  c.g_draw = d->rng_mode == PB_RNG_REPLAY ? d->code_g : nullptr;
  c.block_sums = ws.block_sums; c.m_count = ws.m_count;
  c.n = d->n; c.p = d->p; c.k = d->k; c.key0 = k0; c.key1 = k1;
  philox_round_keys(k0, k1, c.rk);
  c.ld = d->ld > d->n ? d->ld : d->n;
  c.i_offset = d->i_offset;
  c.codes_zero = d->codes_zero;
  const int64_t n_global = d->n_global > 0 ? d->n_global : d->n;
  phase_mark(kPhResid, st);
  int rc = PB_OK;
  if (d->resid_mode == PB_RESID_RECOMPUTE) {
    // residual_full (bpfa.py:297) on the observed positions; the ELL padding is 0
    PB_CUDA_TRY(cudaMemsetAsync(ws.r_csc, 0, (size_t)d->index->nnz_ell * 4, st));
    rc = launch_resid_compact(c, st);
  } else if (d->resid_mode == PB_RESID_FROM_VALUES) {    // Z*S == 0  =>  R = X
    // (the tile-blocked code copy W is not cleared: the prior-draw dictionary
    // step below does not read it and the code step rewrites all of it)
    if (cudaMemcpyAsync(ws.r_csc, ix.x_csc, (size_t)d->index->nnz_ell * 4, cudaMemcpyDeviceToDevice, st) != cudaSuccess) {
      set_error("residual copy failed");
      rc = PB_ECUDA;
    }
  } else if (d->resid_mode != PB_RESID_CARRY) {
    set_error("bad resid_mode %d", d->resid_mode);
    rc = PB_EVALUE;
  }
  if (rc) return rc;
  phase_mark(kPhDict, st);
  if (!d->freeze_dict) {
    DictGramArgs g{};
    g.ell_base = ix.ell_base; g.wave_base = ix.wave_base; g.wave_off = ix.wave_off; g.wave_meta = ix.wave_meta;
    g.wave_col = ix.wave_col; g.e_ell = ix.e_ell; g.ntiles = ix.ntiles;
    g.wt = ws.wt; g.nblk8 = c.nblk8;
    g.r_csc = ws.r_csc; g.usage = d->usage; g.weights = d->weights; g.atoms = d->atoms;
    g.draws = d->rng_mode == PB_RNG_REPLAY ? d->atom_draws : nullptr;
    g.sc = sc; g.partials = ws.partials; g.reduced = ws.reduced; g.bar = ws.bar; g.max_blocks = kMaxDictBlocks;
    g.prof = g_dict_prof;
#ifdef PB_TUNING
    {   // per-wave durations of pass 3 (PB_DICT_WAVE_PROF=1): written to gpurun_out/wave_prof.bin by pb_dict_profile
      static unsigned long long* wp = nullptr;
      if (!wp && PB_TUNE_FLAG("PB_DICT_WAVE_PROF")) { cudaMalloc(&wp, (size_t)3 << 24 << 3); g_wave_prof = wp; }
      if (wp) cudaMemsetAsync(wp, 0, (size_t)3 << 24 << 3, st);
      g.wprof = wp;
    }
#endif
    g.dbg = PB_TUNE_INT("PB_DICT_DEBUG", 0);   // profiling bits exist in tuning builds only
    g.n = d->n; g.p = d->p; g.k = d->k; g.key0 = k0; g.key1 = k1;
    g.ld = c.ld;
    g.nnz = d->index->nnz;
    g.delta_g = ws.delta_g;   // atom shifts of the last updated block [8][P]
    if (d->resid_mode == PB_RESID_FROM_VALUES) {
      // Z*S == 0: every moment sum is 0 on every rank, the atoms are prior
      // redraws and the residual does not move (the first sweep of a cold
      // inpaint and of every warm-reset live frame)
      if ((rc = launch_dict_prior(g, st))) return rc;
    } else if (!d->allreduce) {
      if ((rc = launch_dict_gram(g, st))) return rc;   // fused: all passes in one persistent launch
    } else {
      // split (sharded) mode: per atom block, local pass -> allreduce of the
      // 48*P moment sums across ranks -> identical atom draws on every rank
      g.split = 1;
      const int nblk = dict_gram_blocks(d->k);
      for (int b = 0; b <= nblk; ++b) {
        g.blk_begin = b;
        if ((rc = launch_dict_gram(g, st))) return rc;
        if (b == nblk) break;
        if ((rc = d->allreduce(d->allreduce_ctx, ws.reduced, (int64_t)dict_gram_reduced_bytes(d->p) / 8, 0, st)))
          { set_error("allreduce callback failed (%d)", rc); return PB_ECUDA; }
        if ((rc = launch_dict_update(g, b, st))) return rc;
      }
    }
  }
  int nblocks = 0;
  phase_mark(kPhCode, st);
  c.blk_ctr = ws.ctr;
  c.dt_img = ws.dt_img;
  if ((rc = launch_pack_dt(d->atoms, d->p, d->k, ws.dt_img, st))) return rc;
  if (d->index->split_count > 0) {
    // narrow launch for most patches (stream st) and, concurrently on a side
    // stream, the wide launch over the listed outliers; both claim blocks
    // dynamically and write per-block sums (deterministic)
    PB_CUDA_TRY(cudaMemsetAsync(ws.m_count, 0, (size_t)d->k * sizeof(int32_t), st));
    CompactArgs c1 = c, c2 = c;
    c1.cmax = d->index->split_count;
    c1.split = d->index->split_count;
    c1.zero_mcount = c2.zero_mcount = 0;
    const int nb1_expect = code_launch_blocks(c1.cmax, d->n, d->p, d->k);
    c2.plist = ix.outliers;
    c2.plist_n = d->index->n_outliers;
    c2.block_sums = ws.block_sums + 2 * (size_t)nb1_expect;
    c2.blk_ctr = ws.ctr + 1;
    // side stream + fork/join events of the current device (one set per device
    // ordinal and host thread: a stream belongs to the device it was created on)
    static const int kMaxDev = 64;
    static thread_local cudaStream_t sides[kMaxDev] = {};
    static thread_local cudaEvent_t forks[kMaxDev] = {}, joins[kMaxDev] = {};
    int dev = 0;
    PB_CUDA_TRY(cudaGetDevice(&dev));
    if (dev < 0 || dev >= kMaxDev) { set_error("device ordinal %d out of range", dev); return PB_EUNSUPPORTED; }
    if (!sides[dev]) {
      PB_CUDA_TRY(cudaStreamCreateWithFlags(&sides[dev], cudaStreamNonBlocking));
      PB_CUDA_TRY(cudaEventCreateWithFlags(&forks[dev], cudaEventDisableTiming));
      PB_CUDA_TRY(cudaEventCreateWithFlags(&joins[dev], cudaEventDisableTiming));
    }
    cudaStream_t side = sides[dev];
    cudaEvent_t ev_fork = forks[dev], ev_join = joins[dev];
    int nb1 = 0, nb2 = 0;
    PB_CUDA_TRY(cudaEventRecord(ev_fork, st));
    PB_CUDA_TRY(cudaStreamWaitEvent(side, ev_fork, 0));
    if ((rc = launch_code_compact(c2, d->rng_mode, nb2, side))) return rc;
    PB_CUDA_TRY(cudaEventRecord(ev_join, side));
    if ((rc = launch_code_compact(c1, d->rng_mode, nb1, st))) return rc;
    PB_CUDA_TRY(cudaStreamWaitEvent(st, ev_join, 0));
    if (nb1 != nb1_expect) { set_error("code-step block count mismatch"); return PB_EUNSUPPORTED; }
    nblocks = nb1 + nb2;
  } else {
    c.zero_mcount = 1;
    if ((rc = launch_code_compact(c, d->rng_mode, nblocks, st))) return rc;
  }
  phase_mark(kPhStats, st);
  if ((rc = launch_finish_stats(ws.block_sums, nblocks, sc, st))) return rc;
  if (d->allreduce) {  // epoch statistics across ranks: sum S^2, sum R^2, usage counts m_k
    if ((rc = d->allreduce(d->allreduce_ctx, &sc->sq_w, 2, 0, st)) ||
        (rc = d->allreduce(d->allreduce_ctx, ws.m_count, d->k, 1, st)))
      { set_error("allreduce callback failed (%d)", rc); return PB_ECUDA; }
  }
  if (d->rng_mode == PB_RNG_PHILOX)
    rc = launch_draw_pi_gamma(d->pi, ws.m_count, sc, d->k, n_global, d->n_obs, d->hyper, k0, k1, st);
  phase_mark(kPhEnd, st);
  return rc;
}

}  // namespace pb

using namespace pb;

extern "C" {

const char* pb_last_error(void) { return last_error(); }
int pb_version(void) { return 1; }
int pb_device_count(void) {
  int c = 0;
  if (cudaGetDeviceCount(&c) != cudaSuccess) return 0;
  return c;
}

int pb_grid_counts(const pb_grid_desc* d, int64_t* counts_out, int64_t* num_patches, int32_t* patch_size) {
  Grid g;
  int rc = make_grid(d, g);
  if (rc) return rc;
  for (int i = 0; i < g.rank; ++i)
    if (counts_out) counts_out[i] = g.gcount[i];
  if (num_patches) *num_patches = g.n;
  if (patch_size) *patch_size = g.p;
  return PB_OK;
}

int pb_extract_patches(const pb_grid_desc* d, const void* tensor, int32_t tensor_f64, const uint8_t* mask,
                       int32_t mean_subtract, float* values, uint8_t* observed, float* means, int32_t* counts,
                       void* stream) {
  Grid g;
  int rc = make_grid(d, g);
  if (rc) return rc;
  return launch_extract(g, tensor, tensor_f64, mask, mean_subtract, values, observed, means, counts,
                        (cudaStream_t)stream);
}

int pb_extract_patch_range(const pb_grid_desc* d, const void* tensor, int32_t tensor_f64, const uint8_t* mask,
                           int32_t mean_subtract, int64_t first_patch, int64_t num_patches, float* values,
                           uint8_t* observed, float* means, int32_t* counts, void* stream) {
  Grid g;
  int rc = make_grid(d, g);
  if (rc) return rc;
  return launch_extract(g, tensor, tensor_f64, mask, mean_subtract, values, observed, means, counts,
                        (cudaStream_t)stream, first_patch, num_patches);
}

int pb_reconstitute(const pb_grid_desc* d, const float* est, float est_scale, const float* means,
                    const void* original, const uint8_t* mask, int32_t dc, int32_t io_f64, void* out,
                    unsigned long long* uncovered, void* stream) {
  Grid g;
  int rc = make_grid(d, g);
  if (rc) return rc;
  return launch_reconstitute(g, est, est_scale, means, original, mask, dc, io_f64, out, uncovered,
                             (cudaStream_t)stream);
}

int pb_ola_partial(const pb_grid_desc* d, const float* est, float est_scale, const float* means, int64_t first_patch,
                   int64_t num_patches, double* acc_out, void* stream) {
  Grid g;
  int rc = make_grid(d, g);
  if (rc) return rc;
  return launch_ola_partial(g, est, est_scale, means, first_patch, num_patches, acc_out, (cudaStream_t)stream);
}

int pb_coverage_map(const pb_grid_desc* d, int32_t* out, void* stream) {
  Grid g;
  int rc = make_grid(d, g);
  if (rc) return rc;
  return launch_coverage(g, out, (cudaStream_t)stream);
}

int pb_residual_full(const float* values, const uint8_t* observed, const uint8_t* usage, const float* weights,
                     const float* atoms, float* out, int64_t n, int32_t p, int32_t k, int64_t ld, void* stream) {
  return launch_accumulate_atoms(true, values, observed, usage, weights, atoms, out, n, p, k, 0, ld,
                                 (cudaStream_t)stream);
}

int pb_compose_estimates(const uint8_t* usage, const float* weights, const float* atoms, float* out, int64_t n,
                         int32_t p, int32_t k, int64_t ld, int32_t accumulate, void* stream) {
  return launch_accumulate_atoms(false, nullptr, nullptr, usage, weights, atoms, out, n, p, k, accumulate, ld,
                                 (cudaStream_t)stream);
}

int pb_atom_moments(const float* resid, const uint8_t* observed, const float* w_col, int64_t n, int32_t p,
                    double* a_out, double* c_out, double* scratch, void* stream) {
  return launch_atom_moments(resid, observed, w_col, n, p, scratch, 64, a_out, c_out, (cudaStream_t)stream);
}

int pb_shift_atom(float* resid, const uint8_t* observed, const float* w_col, const float* delta, int64_t n,
                  int32_t p, void* stream) {
  return launch_shift_atom(resid, observed, w_col, delta, n, p, (cudaStream_t)stream);
}

int pb_code_moments(const float* resid, const uint8_t* observed, const float* atom, int64_t n, int32_t p,
                    float* u_out, float* v_out, void* stream) {
  return launch_code_moments(resid, observed, atom, n, p, u_out, v_out, (cudaStream_t)stream);
}

int pb_shift_codes(float* resid, const uint8_t* observed, const float* atom, const float* dw, int64_t n, int32_t p,
                   void* stream) {
  return launch_shift_codes(resid, observed, atom, dw, n, p, (cudaStream_t)stream);
}

int pb_masked_sq_norm(const float* resid, int64_t total, double* out, double* scratch, void* stream) {
  return launch_sq_norm(resid, total, scratch, 256, out, (cudaStream_t)stream);
}

size_t pb_epoch_workspace_bytes(int64_t n, int32_t p, int32_t k, int64_t nnz) {
  return ws_bytes(n, p, k, nnz, nullptr, nullptr);
}

int64_t pb_code_pitch(int64_t n) { return (n + 63) / 64 * 64; }

size_t pb_index_bytes(int64_t n, int32_t p, int64_t nnz) {
  size_t b = 0;
  index_bytes(n, p, nnz, &b);
  return b;
}

int pb_build_index(pb_patch_index* pi, const uint8_t* observed, const float* values, const int32_t* counts,
                   void* stream) {
  if (!pi || !pi->buffer) { set_error("null index"); return PB_EVALUE; }
  if (ell_cap(pi->n, pi->nnz) >= (int64_t)1 << 32) {
    set_error("too many observed elements for 32-bit positions");
    return PB_EUNSUPPORTED;
  }
  PatchIndex ix;
  index_view(pi, ix);
  pi->ntiles = ix.ntiles;
  cudaStream_t st = (cudaStream_t)stream;
  int rc = launch_build_index(ix, observed, values, counts, st);
  if (rc) return rc;
  // code-step split: from the histogram of observed counts, the main launch's
  // per-patch limit; the (few) wider patches get a second, wider launch
  if ((rc = launch_count_hist(ix, counts, st))) return rc;
  std::vector<int32_t> hist(pi->p + 2, 0);
  int32_t cmax = 0;
  PB_CUDA_TRY(cudaMemcpyAsync(&cmax, ix.cmax_dev, 4, cudaMemcpyDeviceToHost, st));
  PB_CUDA_TRY(cudaMemcpyAsync(hist.data(), ix.hist, (size_t)(pi->p + 1) * 4, cudaMemcpyDeviceToHost, st));
  PB_CUDA_TRY(cudaMemcpyAsync(&pi->nnz_ell, ix.ell_base + ix.ntiles, 8, cudaMemcpyDeviceToHost, st));
  PB_CUDA_TRY(cudaStreamSynchronize(st));
  pi->cmax = cmax;
  const int req = pi->split_request != 0 ? pi->split_request
                  : PB_TUNE_FLAG("PB_CODE_SPLIT_OFF") ? -1 : PB_TUNE_INT("PB_CODE_SPLIT_AT", 0);
  if (req > 0) pi->split_count = req < cmax ? req : 0;   // forced threshold
  else if (req < 0) pi->split_count = 0;                 // never split
  else pi->split_count = code_split_choose(hist.data(), pi->p, cmax);
  pi->n_outliers = 0;
  if (pi->split_count > 0) {
    if ((rc = launch_outliers(ix, counts, pi->split_count, st))) return rc;
    int64_t nout = 0;
    PB_CUDA_TRY(cudaMemcpyAsync(&nout, ix.out_base + ix.ntiles, 8, cudaMemcpyDeviceToHost, st));
    PB_CUDA_TRY(cudaStreamSynchronize(st));
    pi->n_outliers = nout;
    if (nout == 0) pi->split_count = 0;
  }
  return PB_OK;
}

int pb_index_refresh_values(const pb_patch_index* pi, const float* values, const int32_t* counts, void* stream) {
  if (!pi || !pi->buffer) { set_error("null index"); return PB_EVALUE; }
  PatchIndex ix;
  index_view(pi, ix);
  return launch_scatter_x(ix, values, counts, (cudaStream_t)stream);
}

int pb_dict_profile(int32_t enable, double* slots_ns_out) {
  const size_t bytes = (size_t)kMaxDictBlocks * kProfSlots * sizeof(unsigned long long);
  if (slots_ns_out) {
    for (int i = 0; i < kProfSlots; ++i) slots_ns_out[i] = 0.0;
    if (g_dict_prof) {
      std::vector<unsigned long long> h(kMaxDictBlocks * kProfSlots);
      PB_CUDA_TRY(cudaDeviceSynchronize());
      PB_CUDA_TRY(cudaMemcpy(h.data(), g_dict_prof, bytes, cudaMemcpyDeviceToHost));
      int nb = 0;  // CTAs that recorded anything; report the mean over them
      for (int b = 0; b < kMaxDictBlocks; ++b) {
        unsigned long long tot = 0;
        for (int i = 0; i < kProfSlots; ++i) tot += h[b * kProfSlots + i];
        if (!tot) continue;
        ++nb;
        for (int i = 0; i < kProfSlots; ++i) slots_ns_out[i] += (double)h[b * kProfSlots + i];
      }
      for (int i = 0; i < kProfSlots; ++i) slots_ns_out[i] /= nb ? nb : 1;
      if (PB_TUNE_FLAG("PB_DICT_PROF_CTAS")) {  // per-CTA element-phase and barrier-1 times (profiling aid)
        for (int b = 0; b < kMaxDictBlocks; ++b) {
          if (!h[b * kProfSlots + 2]) continue;
          fprintf(stderr, "cta %d elems %.4f tile_end %.4f sync1 %.4f fillwait %.4f\n", b, h[b * kProfSlots + 2] / 1e6,
                  h[b * kProfSlots + 3] / 1e6, h[b * kProfSlots + 6] / 1e6, h[b * kProfSlots + 10] / 1e6);
        }
      }
      if (g_wave_prof) {   // tuning builds: raw per-wave profile (3 x u64 per wave) of the last dictionary launch
        std::vector<unsigned long long> w((size_t)3 << 24);
        PB_CUDA_TRY(cudaMemcpy(w.data(), g_wave_prof, w.size() * 8, cudaMemcpyDeviceToHost));
        size_t n = w.size();
        while (n >= 3 && !w[n - 3]) n -= 3;
        if (FILE* f = fopen("gpurun_out/wave_prof.bin", "wb")) { fwrite(w.data(), 8, n, f); fclose(f); }
      }
      if (PB_TUNE_FLAG("PB_DICT_PROF_DUMP")) {  // per-CTA spread of each slot (profiling aid)
        for (int i = 0; i < kProfSlots; ++i) {
          std::vector<double> v;
          for (int b = 0; b < kMaxDictBlocks; ++b)
            if (h[b * kProfSlots + i] || h[b * kProfSlots + 2]) v.push_back((double)h[b * kProfSlots + i]);
          if (v.empty()) continue;
          std::sort(v.begin(), v.end());
          fprintf(stderr, "pb_dict_profile slot %2d: min %.3f p10 %.3f median %.3f p90 %.3f max %.3f ms (n=%zu)\n", i,
                  v.front() / 1e6, v[v.size() / 10] / 1e6, v[v.size() / 2] / 1e6, v[v.size() * 9 / 10] / 1e6,
                  v.back() / 1e6, v.size());
        }
      }
    }
  }
  if (enable && !g_dict_prof) PB_CUDA_TRY(cudaMalloc(&g_dict_prof, bytes));
  if (enable) PB_CUDA_TRY(cudaMemset(g_dict_prof, 0, bytes));
  if (!enable && g_dict_prof) { cudaFree(g_dict_prof); g_dict_prof = nullptr; }
  return PB_OK;
}

int pb_phase_timing(int32_t enable) {
  g_phase_on = enable != 0;
  g_phase_used = 0;
  return PB_OK;
}

int pb_phase_read(double* ms_out, int64_t* epochs_out) {
  for (int i = 0; i < kNumPh - 1; ++i) ms_out[i] = 0.0;
  for (size_t e = 0; e < g_phase_used; ++e) {
    PhaseSet& ps = g_phase_sets[e];
    PB_CUDA_TRY(cudaEventSynchronize(ps.ev[kPhEnd]));
    for (int i = 0; i < kNumPh - 1; ++i) {
      float ms = 0.f;
      if (cudaEventElapsedTime(&ms, ps.ev[i], ps.ev[i + 1]) == cudaSuccess) ms_out[i] += ms;
    }
  }
  if (epochs_out) *epochs_out = (int64_t)g_phase_used;
  return PB_OK;
}

int pb_gibbs_epoch(const pb_epoch_desc* d, int32_t* m_counts_out, void* stream) {
  if (!d) { set_error("null epoch desc"); return PB_EVALUE; }
  return run_epoch(d, m_counts_out, (cudaStream_t)stream);
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Native stateful problem: the live submit_frame hot slice with host buffers
// (pipeline.py:224-251), device RNG, warm start (codes re-burn each frame;
// dictionary, pi and precisions carry over, pipeline.py:230-238).

struct pb_problem {
  pb_problem_desc desc;
  pb::Grid grid;
  int64_t n = 0;
  int64_t ld = 0;  // row pitch of usage/weights
  int p = 0, k = 0;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  double* frame = nullptr;
  uint8_t* mask = nullptr;
  float *values = nullptr, *means = nullptr, *atoms = nullptr, *weights = nullptr, *est = nullptr;
  uint8_t *obs = nullptr, *usage = nullptr;
  int32_t *counts = nullptr, *m_count = nullptr;
  double *pi = nullptr, *recon = nullptr, *out = nullptr, *prev = nullptr, *resid = nullptr;
  uint8_t *panel = nullptr, *masked = nullptr;
  float* bpack = nullptr;  // tensor-core compose scratch (packed D^T)
  int64_t panel_px = 0, panel_stride = 1;  // wire panel: rank 2, or slice 0 of rank 3
  bool have_prev = false;
  bool index_valid = false;  // the observed-element index matches the device mask
  std::vector<float> pending_atoms;   // installed before the first frame (pipeline.py:155-157)
  std::vector<double> pending_pi;
  pb_scalars* scalars = nullptr;
  unsigned long long* nobs_dev = nullptr;
  void* ws = nullptr;
  size_t ws_cap = 0;
  pb_patch_index index{};
  size_t ix_cap = 0;
  std::vector<uint8_t> mask_cache;
  int64_t n_obs = 0;
  bool have_state = false;
  float last_ms = 0.f;
  // replay mode (desc.replay): host draw staging (pinned) and device copies
  double *h_atom = nullptr, *h_u = nullptr, *h_g = nullptr, *h_pi = nullptr;
  double *d_atom = nullptr, *d_u = nullptr, *d_g = nullptr;
  int32_t* h_m = nullptr;
  pb_scalars* h_sc = nullptr;
  int32_t epoch_host = 0;   // replay mode: the host owns the epoch counter
};

namespace {
template <typename T>
int dalloc(T** p, size_t count) {
  PB_CUDA_TRY(cudaMalloc((void**)p, count * sizeof(T) + 16));
  return PB_OK;
}
}  // namespace

extern "C" {

int pb_problem_destroy(pb_problem* pr) {
  if (!pr) return PB_OK;
  void* bufs[] = {pr->frame, pr->mask, pr->values, pr->means, pr->atoms, pr->weights, pr->est, pr->obs, pr->usage,
                  pr->counts, pr->m_count, pr->pi, pr->recon, pr->scalars, pr->nobs_dev, pr->ws, pr->index.buffer,
                  pr->out, pr->prev, pr->resid, pr->panel, pr->masked, pr->bpack};
  for (void* b : bufs)
    if (b) cudaFree(b);
  for (void* b : {(void*)pr->d_atom, (void*)pr->d_u, (void*)pr->d_g})
    if (b) cudaFree(b);
  for (void* b : {(void*)pr->h_atom, (void*)pr->h_u, (void*)pr->h_g, (void*)pr->h_pi, (void*)pr->h_m, (void*)pr->h_sc})
    if (b) cudaFreeHost(b);
  if (pr->ev0) cudaEventDestroy(pr->ev0);
  if (pr->ev1) cudaEventDestroy(pr->ev1);
  if (pr->stream) cudaStreamDestroy(pr->stream);
  delete pr;
  return PB_OK;
}

int pb_problem_create(const pb_problem_desc* desc, pb_problem** out) {
  if (!desc || !out) { set_error("null argument"); return PB_EVALUE; }
  if (desc->num_atoms < 1) { set_error("num_atoms must be >= 1"); return PB_EVALUE; }
  if (desc->epochs_per_frame < 1) { set_error("epochs_per_frame must be >= 1"); return PB_EVALUE; }
  for (int j = 0; j < 6; ++j)
    if (!(desc->hyper[j] > 0)) { set_error("hyperparameters must be > 0"); return PB_EVALUE; }
  if (desc->replay && !desc->draw) { set_error("replay mode needs a draw provider"); return PB_EVALUE; }
  if (desc->init_mode != PB_INIT_PRIOR && desc->init_mode != PB_INIT_DATA) {
    set_error("unknown init mode %d", desc->init_mode);
    return PB_EVALUE;
  }
  pb_problem* pr = new pb_problem();
  pr->desc = *desc;
  int rc = make_grid(&desc->grid, pr->grid);
  if (rc) { delete pr; return rc; }
  pr->n = pr->grid.n; pr->p = pr->grid.p; pr->k = desc->num_atoms;
  pr->ld = pb_code_pitch(pr->n);
  const int64_t m = pr->grid.m, n = pr->n, p = pr->p, k = pr->k, ld = pr->ld;
#define PB_A(ptr, cnt) if ((rc = dalloc(&pr->ptr, (size_t)(cnt)))) { pb_problem_destroy(pr); return rc; }
  PB_A(frame, m) PB_A(mask, m) PB_A(values, p * n) PB_A(obs, p * n) PB_A(means, n) PB_A(counts, n)
  PB_A(atoms, k * p) PB_A(pi, k) PB_A(usage, k * ld) PB_A(weights, k * ld) PB_A(est, p * n) PB_A(recon, m)
  PB_A(m_count, k) PB_A(scalars, 1) PB_A(nobs_dev, 1) PB_A(out, m) PB_A(prev, m) PB_A(resid, m)
  if (compose_tc_supported((int)p) && !PB_TUNE_FLAG("PB_COMPOSE_TC_OFF")) PB_A(bpack, compose_tc_scratch_bytes((int)p, (int)k) / 4)
  if (pr->grid.rank == 2 || pr->grid.rank == 3) {
    pr->panel_stride = pr->grid.rank == 3 ? pr->grid.tshape[2] : 1;
    pr->panel_px = m / pr->panel_stride;
    PB_A(panel, pr->panel_px) PB_A(masked, pr->panel_px)
  }
  if (desc->replay) {  // the epoch's draws: K*P atom normals, K*N uniforms and normals
    PB_A(d_atom, k * p) PB_A(d_u, k * n) PB_A(d_g, k * n)
    if (cudaMallocHost((void**)&pr->h_atom, (size_t)k * p * 8) != cudaSuccess ||
        cudaMallocHost((void**)&pr->h_u, (size_t)k * n * 8) != cudaSuccess ||
        cudaMallocHost((void**)&pr->h_g, (size_t)k * n * 8) != cudaSuccess ||
        cudaMallocHost((void**)&pr->h_pi, (size_t)k * 8) != cudaSuccess ||
        cudaMallocHost((void**)&pr->h_m, (size_t)k * 4) != cudaSuccess ||
        cudaMallocHost((void**)&pr->h_sc, sizeof(pb_scalars)) != cudaSuccess) {
      set_error("pinned replay buffers: allocation failed");
      pb_problem_destroy(pr);
      return PB_ECUDA;
    }
  }
#undef PB_A
  // codes start (and their row padding [n, ld) stays) zero; frames rewrite [0, n)
  if (cudaMemset(pr->usage, 0, (size_t)k * ld) != cudaSuccess ||
      cudaMemset(pr->weights, 0, (size_t)k * ld * sizeof(float)) != cudaSuccess) {
    set_error("code buffers: clear failed");
    pb_problem_destroy(pr);
    return PB_ECUDA;
  }
  if (cudaStreamCreateWithFlags(&pr->stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreate(&pr->ev0) != cudaSuccess || cudaEventCreate(&pr->ev1) != cudaSuccess) {
    set_error("stream/event creation failed");
    pb_problem_destroy(pr);
    return PB_ECUDA;
  }
  *out = pr;
  return PB_OK;
}

static int problem_cold_init(pb_problem* pr) {
  // init_state on device (bpfa.py:104-152): prior atoms (device Philox, or the
  // reference stream (seed, 1) in replay mode), data-mode seeding from the patches
  // with the most observed elements when the dictionary is frozen (otherwise the
  // first dictionary step redraws every atom from the prior before any use,
  // SURVEY App. A Q1), pi = a/(a+b), gammas at their prior means, Z = S = 0,
  // epoch 0.  An installed dictionary (install_dictionary, bpfa.py:355-376)
  // replaces the atoms and pi.
  uint32_t k0, k1;
  device_key(pr->desc.seed, k0, k1);
  std::vector<double> pi(pr->k, pr->desc.hyper[0] / (pr->desc.hyper[0] + pr->desc.hyper[1]));
  std::vector<float> atoms;
  if (!pr->pending_atoms.empty()) {  // infer(initial_dict=...) -> install_dictionary (bpfa.py:355-376)
    atoms.swap(pr->pending_atoms);
    pi.swap(pr->pending_pi);
    PB_CUDA_TRY(cudaMemcpyAsync(pr->atoms, atoms.data(), atoms.size() * 4, cudaMemcpyHostToDevice, pr->stream));
  } else {
    if (pr->desc.replay) {
      if (pr->desc.draw(pr->desc.draw_ctx, PB_DRAW_PRIOR, 0, nullptr, nullptr, pr->h_atom, nullptr, nullptr)) {
        set_error("replay draw provider failed (prior atoms)");
        return PB_EVALUE;
      }
      atoms.resize((size_t)pr->k * pr->p);
      for (size_t j = 0; j < atoms.size(); ++j) atoms[j] = (float)pr->h_atom[j];
      PB_CUDA_TRY(cudaMemcpyAsync(pr->atoms, atoms.data(), atoms.size() * 4, cudaMemcpyHostToDevice, pr->stream));
    } else {
      int rc = launch_prior_atoms(pr->atoms, pr->k, pr->p, k0, k1, pr->stream);
      if (rc) return rc;
    }
    if (pr->desc.init_mode == PB_INIT_DATA && pr->desc.freeze_dict) {
      int rc = launch_data_atoms(pr->values, pr->counts, pr->n, pr->p, pr->k, pr->atoms, pr->stream);
      if (rc) return rc;
    }
  }
  PB_CUDA_TRY(cudaMemcpyAsync(pr->pi, pi.data(), pr->k * sizeof(double), cudaMemcpyHostToDevice, pr->stream));
  pb_scalars s{};
  s.gamma_s = fmax(pr->desc.hyper[2] / pr->desc.hyper[3], 1e-12);
  s.gamma_eps = fmax(pr->desc.hyper[4] / pr->desc.hyper[5], 1e-12);
  PB_CUDA_TRY(cudaMemcpyAsync(pr->scalars, &s, sizeof(s), cudaMemcpyHostToDevice, pr->stream));
  PB_CUDA_TRY(cudaStreamSynchronize(pr->stream));  // s/pi/atoms live on this stack frame
  pr->have_state = true;
  pr->epoch_host = 0;
  return PB_OK;
}

// One replay-mode sweep of the problem: the reference's draws for this epoch
// from the host provider (uploaded), the device sweep, then the pi / gamma draws
// on the host from the epoch's usage counts and sums (bpfa.py:313-333) — the
// same split as bpfa.gibbs_epoch(rng="numpy") of the Python API.
static int replay_epoch(pb_problem* pr, pb_epoch_desc& d) {
  cudaStream_t st = pr->stream;
  const int64_t ep = (int64_t)pr->epoch_host + 1;
  const size_t kp = (size_t)pr->k * pr->p, kn = (size_t)pr->k * pr->n;
  const bool frozen = d.freeze_dict != 0;
  if (pr->desc.draw(pr->desc.draw_ctx, PB_DRAW_EPOCH, ep, nullptr, nullptr, frozen ? nullptr : pr->h_atom, pr->h_u,
                    pr->h_g)) {
    set_error("replay draw provider failed (epoch %lld)", (long long)ep);
    return PB_EVALUE;
  }
  if (!frozen) PB_CUDA_TRY(cudaMemcpyAsync(pr->d_atom, pr->h_atom, kp * 8, cudaMemcpyHostToDevice, st));
  PB_CUDA_TRY(cudaMemcpyAsync(pr->d_u, pr->h_u, kn * 8, cudaMemcpyHostToDevice, st));
  PB_CUDA_TRY(cudaMemcpyAsync(pr->d_g, pr->h_g, kn * 8, cudaMemcpyHostToDevice, st));
  d.atom_draws = frozen ? nullptr : pr->d_atom;
  d.code_u = pr->d_u;
  d.code_g = pr->d_g;
  int rc = run_epoch(&d, pr->m_count, st);
  if (rc) return rc;
  PB_CUDA_TRY(cudaMemcpyAsync(pr->h_m, pr->m_count, (size_t)pr->k * 4, cudaMemcpyDeviceToHost, st));
  PB_CUDA_TRY(cudaMemcpyAsync(pr->h_sc, pr->scalars, sizeof(pb_scalars), cudaMemcpyDeviceToHost, st));
  PB_CUDA_TRY(cudaStreamSynchronize(st));
  double sums[3] = {pr->h_sc->sq_w, pr->h_sc->sq_r, (double)pr->n_obs};
  double gam[2] = {0.0, 0.0};
  if (pr->desc.draw(pr->desc.draw_ctx, PB_DRAW_POSTERIOR, ep, pr->h_m, sums, pr->h_pi, gam, nullptr)) {
    set_error("replay draw provider failed (pi / gamma, epoch %lld)", (long long)ep);
    return PB_EVALUE;
  }
  pr->h_sc->gamma_s = gam[0];
  pr->h_sc->gamma_eps = gam[1];
  pr->h_sc->epoch = (int32_t)ep;
  pr->h_sc->diverged = !(isfinite(gam[0]) && isfinite(gam[1]) && isfinite(sums[1]));  // bpfa.py:335-342
  PB_CUDA_TRY(cudaMemcpyAsync(pr->pi, pr->h_pi, (size_t)pr->k * 8, cudaMemcpyHostToDevice, st));
  PB_CUDA_TRY(cudaMemcpyAsync(pr->scalars, pr->h_sc, sizeof(pb_scalars), cudaMemcpyHostToDevice, st));
  pr->epoch_host = (int32_t)ep;
  return PB_OK;
}

int pb_problem_submit_frame(pb_problem* pr, const double* frame_host, const uint8_t* mask_host,
                            double* recon_host) {
  if (!recon_host) { set_error("null argument"); return PB_EVALUE; }
  return pb_problem_submit_frame_ex(pr, frame_host, mask_host, recon_host, nullptr, nullptr);
}

int pb_problem_submit_frame_ex(pb_problem* pr, const double* frame_host, const uint8_t* mask_host,
                               double* recon_host, uint8_t* panel_host, uint8_t* masked_host) {
  if (!pr || !frame_host || !mask_host) { set_error("null argument"); return PB_EVALUE; }
  if ((panel_host || masked_host) && !pr->panel) {
    set_error("wire panels need a rank-2 or rank-3 tensor (got rank %d)", pr->grid.rank);
    return PB_EVALUE;
  }
  const int64_t m = pr->grid.m, n = pr->n;
  cudaStream_t st = pr->stream;
  PB_CUDA_TRY(cudaEventRecord(pr->ev0, st));
  PB_CUDA_TRY(cudaMemcpyAsync(pr->frame, frame_host, m * sizeof(double), cudaMemcpyHostToDevice, st));
  const bool mask_changed = pr->mask_cache.size() != (size_t)m || memcmp(pr->mask_cache.data(), mask_host, m) != 0;
  if (mask_changed) {
    pr->mask_cache.assign(mask_host, mask_host + m);
    PB_CUDA_TRY(cudaMemcpyAsync(pr->mask, pr->mask_cache.data(), m, cudaMemcpyHostToDevice, st));
  }
  // the observed-element index follows the mask (a device-generated mask is
  // already resident but still needs its index)
  const bool new_mask = mask_changed || !pr->index_valid;
  // Cached mask, 2-D frame: the observed values go from the frame straight into
  // the index's compact order (k_refresh_frame2d) — unless a cold data-mode
  // seeding will read the dense values, or the frame is wide enough that the
  // extraction would take the row-tile kernel (another summation order of the
  // means).  Otherwise: the dense extraction, then the index build / refresh.
  const bool cold = !pr->have_state || !pr->desc.warm_start;
  const bool fused = !new_mask && pr->grid.rank == 2 && pr->grid.gcount[1] < 768 &&
                     !(cold && pr->desc.init_mode == PB_INIT_DATA && pr->desc.freeze_dict);
  int rc = PB_OK;
  if (fused) {
    PatchIndex ix;
    index_view(&pr->index, ix);
    rc = launch_refresh_frame2d(ix, pr->frame, pr->grid.tshape[1], pr->grid.gcount[1], pr->grid.bshape[1],
                                pr->grid.step[0], pr->grid.step[1], pr->desc.mean_subtract, pr->counts, pr->means, st);
    if (rc) return rc;
  } else {
    rc = launch_extract(pr->grid, pr->frame, 1, pr->mask, pr->desc.mean_subtract, pr->values, pr->obs, pr->means,
                        pr->counts, st);
    if (rc) return rc;
  }
  if (new_mask) {
    if ((rc = launch_sum_counts(pr->counts, n, pr->nobs_dev, st))) return rc;
    unsigned long long nobs = 0;
    PB_CUDA_TRY(cudaMemcpyAsync(&nobs, pr->nobs_dev, sizeof(nobs), cudaMemcpyDeviceToHost, st));
    PB_CUDA_TRY(cudaStreamSynchronize(st));
    pr->n_obs = (int64_t)nobs;
    // (re)size the observed-element index and the epoch workspace for this mask
    const size_t ixb = pb_index_bytes(n, pr->p, pr->n_obs);
    if (ixb > pr->ix_cap) {
      if (pr->index.buffer) cudaFree(pr->index.buffer);
      pr->index.buffer = nullptr;
      PB_CUDA_TRY(cudaMalloc(&pr->index.buffer, ixb));
      pr->ix_cap = ixb;
    }
    pr->index.n = n; pr->index.p = pr->p; pr->index.nnz = pr->n_obs;
    if ((rc = pb_build_index(&pr->index, pr->obs, pr->values, pr->counts, st))) return rc;
    pr->index_valid = true;
  } else if (!fused) {
    if ((rc = pb_index_refresh_values(&pr->index, pr->values, pr->counts, st))) return rc;
  }
  {  // epoch workspace for this mask's observed count and the current K
    const size_t wsb = pb_epoch_workspace_bytes(n, pr->p, pr->k, pr->n_obs);
    if (wsb > pr->ws_cap) {
      if (pr->ws) cudaFree(pr->ws);
      pr->ws = nullptr;
      PB_CUDA_TRY(cudaMalloc(&pr->ws, wsb));
      pr->ws_cap = wsb;
    }
  }
  if (!pr->have_state || !pr->desc.warm_start) {
    if ((rc = problem_cold_init(pr))) return rc;
  }
  // codes re-burn each frame (pipeline.py:232-233): the first sweep runs with
  // codes_zero (no old state read, every entry rewritten), so no clearing pass
  pb_epoch_desc d{};
  d.n = n; d.ld = pr->ld; d.p = pr->p; d.k = pr->k;
  d.freeze_dict = pr->desc.freeze_dict;
  d.rng_mode = pr->desc.replay ? PB_RNG_REPLAY : PB_RNG_PHILOX;
  d.seed = pr->desc.seed;
  d.n_obs = pr->n_obs;
  for (int j = 0; j < 6; ++j) d.hyper[j] = pr->desc.hyper[j];
  d.values = pr->values; d.observed = pr->obs; d.atoms = pr->atoms; d.pi = pr->pi;
  d.usage = pr->usage; d.weights = pr->weights; d.scalars = pr->scalars; d.workspace = pr->ws;
  d.index = &pr->index; d.counts = pr->counts;
  const int epochs = pr->desc.epochs_per_frame;
  int tail = pr->desc.average_last < 1 ? 1 : (pr->desc.average_last > epochs ? epochs : pr->desc.average_last);
  for (int e = 0; e < epochs; ++e) {
    d.resid_mode = e == 0 ? PB_RESID_FROM_VALUES : PB_RESID_CARRY;  // codes were just reset
    d.codes_zero = e == 0;
    if (pr->desc.replay) {
      if ((rc = replay_epoch(pr, d))) return rc;
    } else if ((rc = run_epoch(&d, pr->m_count, st))) {
      return rc;
    }
    if (e >= epochs - tail) {
      if (pr->bpack)  // tensor-core compose with the problem's packed-D scratch
        rc = launch_compose_tc(pr->usage, pr->weights, pr->ld, pr->atoms, pr->p, pr->k, n, pr->est,
                               e > epochs - tail ? 1 : 0, st, pr->bpack);
      else
        rc = launch_accumulate_atoms(false, nullptr, nullptr, pr->usage, pr->weights, pr->atoms, pr->est, n, pr->p,
                                     pr->k, e > epochs - tail ? 1 : 0, pr->ld, st);
      if (rc) return rc;
    }
  }
  // overlap-add (before data consistency), then the fused tail: consistency,
  // residual map, previous-reconstruction update, uint8 wire panels
  rc = launch_reconstitute(pr->grid, pr->est, 1.0f / (float)tail, pr->means, pr->frame, pr->mask, 0, 1, pr->recon,
                           nullptr, st);
  if (rc) return rc;
  LiveFinishArgs lf{};
  lf.recon = pr->recon; lf.frame = pr->frame; lf.mask = pr->mask; lf.out = pr->out;
  lf.prev = pr->prev; lf.resid = pr->resid;
  lf.panel = panel_host ? pr->panel : nullptr;
  lf.masked = masked_host ? pr->masked : nullptr;
  lf.m = m; lf.panel_stride = pr->panel_stride; lf.dc = pr->desc.data_consistency; lf.have_prev = pr->have_prev;
  if ((rc = launch_live_finish(lf, st))) return rc;
  pr->have_prev = true;
  if (recon_host) PB_CUDA_TRY(cudaMemcpyAsync(recon_host, pr->out, m * sizeof(double), cudaMemcpyDeviceToHost, st));
  if (panel_host) PB_CUDA_TRY(cudaMemcpyAsync(panel_host, pr->panel, pr->panel_px, cudaMemcpyDeviceToHost, st));
  if (masked_host) PB_CUDA_TRY(cudaMemcpyAsync(masked_host, pr->masked, pr->panel_px, cudaMemcpyDeviceToHost, st));
  pb_scalars s;
  PB_CUDA_TRY(cudaMemcpyAsync(&s, pr->scalars, sizeof(s), cudaMemcpyDeviceToHost, st));
  PB_CUDA_TRY(cudaEventRecord(pr->ev1, st));
  PB_CUDA_TRY(cudaStreamSynchronize(st));
  cudaEventElapsedTime(&pr->last_ms, pr->ev0, pr->ev1);
  if (s.diverged) {
    set_error("non-finite state at epoch %d: gamma_s=%g, gamma_eps=%g, masked residual norm=%g", s.epoch, s.gamma_s,
              s.gamma_eps, s.sq_r);
    return PB_EDIVERGED;
  }
  return PB_OK;
}

float pb_problem_last_gpu_ms(pb_problem* pr) { return pr ? pr->last_ms : 0.f; }

int pb_atlas_shape(int32_t k, int32_t rank, const int32_t* patch_shape, int64_t* height, int64_t* width) {
  if (!patch_shape || !height || !width) { set_error("null argument"); return PB_EVALUE; }
  int b0, b1, inner, grid;
  return atlas_geometry(k, rank, patch_shape, b0, b1, inner, grid, *height, *width);
}

int pb_render_atlas(const float* atoms, const double* pi, int32_t k, int32_t rank, const int32_t* patch_shape,
                    double* canvas, uint8_t* canvas_u8, void* stream) {
  if (!atoms || !pi || !patch_shape || (!canvas && !canvas_u8)) { set_error("null argument"); return PB_EVALUE; }
  return launch_atlas(atoms, pi, k, rank, patch_shape, canvas, canvas_u8, (cudaStream_t)stream);
}

int pb_problem_render_atlas(pb_problem* pr, uint8_t* canvas_u8_host) {
  if (!pr || !canvas_u8_host) { set_error("null argument"); return PB_EVALUE; }
  int32_t shape[4];
  for (int d = 0; d < pr->grid.rank; ++d) shape[d] = pr->grid.bshape[d];
  int b0, b1, inner, grid;
  int64_t h, w;
  int rc = atlas_geometry(pr->k, pr->grid.rank, shape, b0, b1, inner, grid, h, w);
  if (rc) return rc;
  uint8_t* dev = nullptr;
  PB_CUDA_TRY(cudaMallocAsync((void**)&dev, (size_t)(h * w), pr->stream));
  rc = launch_atlas(pr->atoms, pr->pi, pr->k, pr->grid.rank, shape, nullptr, dev, pr->stream);
  if (!rc && cudaMemcpyAsync(canvas_u8_host, dev, (size_t)(h * w), cudaMemcpyDeviceToHost, pr->stream) != cudaSuccess) {
    set_error("atlas copy failed");
    rc = PB_ECUDA;
  }
  cudaFreeAsync(dev, pr->stream);
  if (cudaStreamSynchronize(pr->stream) != cudaSuccess && !rc) { set_error("atlas failed"); rc = PB_ECUDA; }
  return rc;
}

// Re-size every K-dependent buffer of a problem (a dictionary with another atom
// count was installed: Pipeline._install_dictionary rebuilds the state with
// moved.num_atoms, pipeline.py:158-167).  Codes are reset each frame anyway.
static int problem_set_k(pb_problem* pr, int k) {
  if (k == pr->k) return PB_OK;
  if (k < 1) { set_error("num_atoms must be >= 1"); return PB_EVALUE; }
  PB_CUDA_TRY(cudaStreamSynchronize(pr->stream));
  void* dev[] = {pr->atoms, pr->pi, pr->usage, pr->weights, pr->m_count, pr->bpack, pr->ws,
                 pr->d_atom, pr->d_u, pr->d_g};
  for (void* b : dev)
    if (b) cudaFree(b);
  void* host[] = {pr->h_atom, pr->h_u, pr->h_g, pr->h_pi, pr->h_m};
  for (void* b : host)
    if (b) cudaFreeHost(b);
  pr->atoms = nullptr; pr->pi = nullptr; pr->usage = nullptr; pr->weights = nullptr; pr->m_count = nullptr;
  pr->bpack = nullptr; pr->ws = nullptr; pr->ws_cap = 0;
  pr->d_atom = pr->d_u = pr->d_g = nullptr;
  pr->h_atom = pr->h_u = pr->h_g = pr->h_pi = nullptr;
  pr->h_m = nullptr;
  pr->k = k;
  pr->desc.num_atoms = k;
  const int64_t n = pr->n, p = pr->p, ld = pr->ld;
  int rc = PB_OK;
#define PB_R(ptr, cnt) if ((rc = dalloc(&pr->ptr, (size_t)(cnt)))) return rc;
  PB_R(atoms, (int64_t)k * p) PB_R(pi, k) PB_R(usage, (int64_t)k * ld) PB_R(weights, (int64_t)k * ld) PB_R(m_count, k)
  PB_CUDA_TRY(cudaMemset(pr->usage, 0, (size_t)k * ld));
  PB_CUDA_TRY(cudaMemset(pr->weights, 0, (size_t)k * ld * sizeof(float)));
  if (compose_tc_supported((int)p) && !PB_TUNE_FLAG("PB_COMPOSE_TC_OFF")) PB_R(bpack, compose_tc_scratch_bytes((int)p, k) / 4)
  if (pr->desc.replay) {
    PB_R(d_atom, (int64_t)k * p) PB_R(d_u, (int64_t)k * n) PB_R(d_g, (int64_t)k * n)
    if (cudaMallocHost((void**)&pr->h_atom, (size_t)k * p * 8) != cudaSuccess ||
        cudaMallocHost((void**)&pr->h_u, (size_t)k * n * 8) != cudaSuccess ||
        cudaMallocHost((void**)&pr->h_g, (size_t)k * n * 8) != cudaSuccess ||
        cudaMallocHost((void**)&pr->h_pi, (size_t)k * 8) != cudaSuccess ||
        cudaMallocHost((void**)&pr->h_m, (size_t)k * 4) != cudaSuccess) {
      set_error("pinned replay buffers: allocation failed");
      return PB_ECUDA;
    }
  }
#undef PB_R
  return PB_OK;
}

int pb_problem_install_dictionary(pb_problem* pr, const float* atoms_host, const double* pi_host, int32_t k,
                                  int32_t freeze) {
  if (!pr || !atoms_host || !pi_host) { set_error("null argument"); return PB_EVALUE; }
  int rc = problem_set_k(pr, k);
  if (rc) return rc;
  if (freeze == 0 || freeze == 1) pr->desc.freeze_dict = freeze;
  const size_t kp = (size_t)pr->k * pr->p;
  if (!pr->have_state) {  // pending until the first frame (pipeline.py:155-157)
    pr->pending_atoms.assign(atoms_host, atoms_host + kp);
    pr->pending_pi.assign(pi_host, pi_host + pr->k);
    return PB_OK;
  }
  // replace the dictionary; codes reset every frame, precisions and epoch carry
  // over (pipeline.py:158-167)
  PB_CUDA_TRY(cudaMemcpyAsync(pr->atoms, atoms_host, kp * 4, cudaMemcpyHostToDevice, pr->stream));
  PB_CUDA_TRY(cudaMemcpyAsync(pr->pi, pi_host, (size_t)pr->k * 8, cudaMemcpyHostToDevice, pr->stream));
  PB_CUDA_TRY(cudaStreamSynchronize(pr->stream));  // host buffers may be released on return
  return PB_OK;
}

int pb_problem_transfer_dictionary(pb_problem* src, pb_problem* dst, int32_t freeze) {
  if (!src || !dst) { set_error("null argument"); return PB_EVALUE; }
  if (src == dst) { set_error("cannot transfer a dictionary onto itself"); return PB_EVALUE; }
  const bool pending = !src->have_state && !src->pending_atoms.empty();
  if (!src->have_state && !pending) { set_error("source problem has no trained state yet"); return PB_EVALUE; }
  // bpfa.transfer_dictionary shape rules (bpfa.py:431-449): equal patch shapes, or the
  // destination extends the source with trailing dimensions that span its tensor
  const pb::Grid &gs = src->grid, &gd = dst->grid;
  int repeat = 1, normalize = 0;
  bool same = gs.rank == gd.rank;
  for (int i = 0; same && i < gs.rank; ++i) same = gs.bshape[i] == gd.bshape[i];
  if (!same) {
    bool ok = gd.rank > gs.rank;
    for (int i = 0; ok && i < gs.rank; ++i) ok = gs.bshape[i] == gd.bshape[i];
    if (!ok) { set_error("cannot transfer atoms between these patch shapes"); return PB_ESHAPE; }
    for (int i = gs.rank; i < gd.rank; ++i) {
      if (gd.bshape[i] != gd.tshape[i]) {
        set_error("transfer dimension %d must span the destination tensor (%d != %lld)", i, gd.bshape[i],
                  (long long)gd.tshape[i]);
        return PB_ESHAPE;
      }
      repeat *= gd.bshape[i];
    }
    normalize = 1;
  }
  const int k = src->k, ps = src->p;
  int rc = problem_set_k(dst, k);
  if (rc) return rc;
  if (freeze == 0 || freeze == 1) dst->desc.freeze_dict = freeze;
  cudaStream_t st = dst->stream;
  float* tmp_src = nullptr;
  const float* s_atoms = src->atoms;
  std::vector<double> pi_h;
  if (pending) {  // the source's dictionary is still a pending install (host copies)
    PB_CUDA_TRY(cudaMallocAsync((void**)&tmp_src, (size_t)k * ps * 4, st));
    PB_CUDA_TRY(cudaMemcpyAsync(tmp_src, src->pending_atoms.data(), (size_t)k * ps * 4, cudaMemcpyHostToDevice, st));
    s_atoms = tmp_src;
    pi_h = src->pending_pi;
  } else {
    PB_CUDA_TRY(cudaStreamSynchronize(src->stream));   // the source's sweeps are done (snapshot)
  }
  float* out = dst->atoms;
  if (!dst->have_state) PB_CUDA_TRY(cudaMallocAsync((void**)&out, (size_t)k * dst->p * 4, st));
  rc = launch_transfer_atoms(s_atoms, k, ps, repeat, normalize, out, st);
  if (!rc && !dst->have_state) {  // pending until the destination's first frame (pipeline.py:155-157)
    dst->pending_atoms.resize((size_t)k * dst->p);
    dst->pending_pi.resize(k);
    if (cudaMemcpyAsync(dst->pending_atoms.data(), out, (size_t)k * dst->p * 4, cudaMemcpyDeviceToHost, st) ||
        (pending ? false : cudaMemcpyAsync(dst->pending_pi.data(), src->pi, (size_t)k * 8, cudaMemcpyDeviceToHost, st)))
      { set_error("transfer copy failed"); rc = PB_ECUDA; }
    if (pending) dst->pending_pi = pi_h;
  } else if (!rc) {  // replace the dictionary; precisions and epoch carry over (pipeline.py:158-167)
    if (pending) {
      if (cudaMemcpyAsync(dst->pi, pi_h.data(), (size_t)k * 8, cudaMemcpyHostToDevice, st)) rc = PB_ECUDA;
    } else if (cudaMemcpyAsync(dst->pi, src->pi, (size_t)k * 8, cudaMemcpyDeviceToDevice, st)) {
      rc = PB_ECUDA;
    }
    if (rc) set_error("transfer copy failed");
  }
  if (tmp_src) cudaFreeAsync(tmp_src, st);
  if (!dst->have_state && out) cudaFreeAsync(out, st);
  if (cudaStreamSynchronize(st) != cudaSuccess && !rc) { set_error("transfer failed"); rc = PB_ECUDA; }
  return rc;
}

int pb_problem_residual_map(pb_problem* pr, double* host_out) {
  if (!pr || !host_out) { set_error("null argument"); return PB_EVALUE; }
  if (!pr->have_prev) { set_error("no frame submitted yet"); return PB_EVALUE; }
  PB_CUDA_TRY(cudaMemcpyAsync(host_out, pr->resid, (size_t)pr->grid.m * 8, cudaMemcpyDeviceToHost, pr->stream));
  PB_CUDA_TRY(cudaStreamSynchronize(pr->stream));
  return PB_OK;
}

static int adaptive_counts(double ratio, double exploit_fraction, int64_t total, int64_t& budget, int64_t& n_exploit) {
  if (!(ratio >= 0.0 && ratio <= 1.0)) { set_error("sampling ratio must be in [0, 1], got %g", ratio); return PB_EVALUE; }
  budget = (int64_t)floor(ratio * (double)total + 0.5);                 // sampling.py:53-56
  n_exploit = (int64_t)floor(exploit_fraction * (double)budget + 0.5);  // sampling.py:195-197
  if (n_exploit < 0) n_exploit = 0;
  if (n_exploit > budget) n_exploit = budget;
  return PB_OK;
}

int pb_adaptive_mask(const double* residual, int64_t m, double ratio, double exploit_fraction, uint64_t seed,
                     int64_t frame_index, uint8_t* mask_out, int32_t* status_out, void* stream) {
  if (!residual || !mask_out || m < 0) { set_error("bad argument"); return PB_EVALUE; }
  int64_t budget = 0, n_exploit = 0;
  int rc = adaptive_counts(ratio, exploit_fraction, m, budget, n_exploit);
  if (rc) return rc;
  uint32_t k0, k1;
  device_key(seed, k0, k1);
  int status = 0;
  rc = adaptive_mask(residual, m, budget, n_exploit, k0, k1, (uint64_t)frame_index, mask_out, &status,
                     (cudaStream_t)stream);
  if (status_out) *status_out = status;
  return rc;
}

int pb_problem_adaptive_mask(pb_problem* pr, double ratio, double exploit_fraction, uint64_t seed,
                             int64_t frame_index, uint8_t* mask_host, int32_t* status_out) {
  if (!pr || !mask_host) { set_error("null argument"); return PB_EVALUE; }
  const int64_t m = pr->grid.m;
  int status = 1;
  if (!pr->have_prev) {  // no residual yet (pipeline.py:266-269): all-zero map
    PB_CUDA_TRY(cudaMemsetAsync(pr->resid, 0, (size_t)m * 8, pr->stream));
  }
  int rc = pb_adaptive_mask(pr->resid, m, ratio, exploit_fraction, seed, frame_index, pr->mask, &status, pr->stream);
  if (rc) return rc;
  PB_CUDA_TRY(cudaMemcpyAsync(mask_host, pr->mask, (size_t)m, cudaMemcpyDeviceToHost, pr->stream));
  PB_CUDA_TRY(cudaStreamSynchronize(pr->stream));
  pr->mask_cache.assign(mask_host, mask_host + m);  // the device copy is current: no re-upload
  pr->index_valid = false;                           // ... but its index is not built yet
  if (status_out) *status_out = status;
  return PB_OK;
}

int pb_problem_get_dictionary(pb_problem* pr, float* atoms_host, double* pi_host, pb_scalars* scalars_host) {
  if (!pr) { set_error("null problem"); return PB_EVALUE; }
  if (atoms_host)
    PB_CUDA_TRY(cudaMemcpyAsync(atoms_host, pr->atoms, (size_t)pr->k * pr->p * 4, cudaMemcpyDeviceToHost, pr->stream));
  if (pi_host) PB_CUDA_TRY(cudaMemcpyAsync(pi_host, pr->pi, (size_t)pr->k * 8, cudaMemcpyDeviceToHost, pr->stream));
  if (scalars_host)
    PB_CUDA_TRY(cudaMemcpyAsync(scalars_host, pr->scalars, sizeof(pb_scalars), cudaMemcpyDeviceToHost, pr->stream));
  PB_CUDA_TRY(cudaStreamSynchronize(pr->stream));
  return PB_OK;
}

}  // extern "C"
