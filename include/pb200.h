/*
 * pb200 — C ABI of the B200-native BPFA inpainting hot path.
 *
 * Drop-in boundary for reference pkg/src/patchbeam (arXiv 2311.15061 "SenseAI").
 * The reference is Python; its own native seam is the Numba kernel module
 * (_kernels.py) that bpfa.py calls through the module object (bpfa.py:30), plus
 * the Python entry points patches.extract_patches / reconstitute and
 * bpfa.gibbs_epoch / compose_estimates / infer.  Each entry point below names
 * the reference function it replaces.  The ctypes binding that mirrors the
 * reference API lives in paper_2311_15061_b200/ (see INTEGRATION.md).
 *
 * Conventions
 *  - All array pointers are DEVICE pointers unless a name ends in `_host`.
 *  - Plane-major device layouts: values/observed/resid/estimates are (P, N)
 *    ([p*N + i]); usage (uint8 0/1) and weights are (K, N); atoms are (K, P).
 *    This is the transpose of the reference's row-major (N, P)/(N, K) arrays.
 *  - `stream` is a cudaStream_t (NULL = legacy default stream).
 *  - Every function returns PB_OK (0) or a negative PB_E* code; the message of
 *    the last failure on the calling thread is pb_last_error().
 *  - Nothing here falls back to the CPU: without a CUDA device every compute
 *    entry point fails with PB_ECUDA.
 */
#ifndef PB200_H_
#define PB200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PB_OK 0
#define PB_ESHAPE -1       /* patchbeam.patches.ShapeError          (patches.py:20-21) */
#define PB_EVALUE -2       /* ValueError (bad hyperparameters etc.)  (bpfa.py:54-60)    */
#define PB_ECOVERAGE -3    /* patchbeam.patches.CoverageError       (patches.py:24-25) */
#define PB_EDIVERGED -4    /* patchbeam.bpfa.DivergenceError         (bpfa.py:38-39)    */
#define PB_ECUDA -5        /* CUDA runtime failure / no device                           */
#define PB_EUNSUPPORTED -6 /* shape outside the compiled kernel envelope                 */

#define PB_RESID_RECOMPUTE 0   /* residual_full from (X, Z, S, D) — the reference's behaviour */
#define PB_RESID_FROM_VALUES 1 /* caller asserts Z*S == 0 (fresh / warm-reset codes): R = X */
#define PB_RESID_CARRY 2       /* workspace holds the end residual of the previous epoch of this
                                  exact state (same patch matrix, state untouched since)  */

#define PB_RNG_REPLAY 0    /* draws supplied by the caller (reference numpy streams) */
#define PB_RNG_PHILOX 1    /* device counter-based Philox4x32-10 draws               */

const char* pb_last_error(void);
int pb_version(void);
int pb_device_count(void);

/* Patch grid: rank 1..4, tensor shape M, patch shape B, stride s (patches.py:35-77). */
typedef struct pb_grid_desc {
  int32_t rank;
  int64_t tensor_shape[4];
  int32_t patch_shape[4];
  int32_t stride[4];
} pb_grid_desc;

/* PatchSpec.grid_counts / num_patches / patch_size (patches.py:64-77).
 * Validates like PatchSpec.validate_for (patches.py:54-62): PB_ESHAPE on error. */
int pb_grid_counts(const pb_grid_desc* g, int64_t* counts_out, int64_t* num_patches, int32_t* patch_size);

/* extract_patches (patches.py:125-164).  tensor: f32 (tensor_f64=0) or f64 device
 * array of the tensor shape; mask: uint8.  Outputs (P,N) values, (P,N) observed,
 * (N) means (0 unless mean_subtract), (N) observed counts. */
int pb_extract_patches(const pb_grid_desc* g, const void* tensor, int32_t tensor_f64, const uint8_t* mask,
                       int32_t mean_subtract, float* values, uint8_t* observed, float* means,
                       int32_t* counts, void* stream);

/* A shard of the patch matrix: global patches [first_patch, first_patch + num_patches)
 * into (P, num_patches) outputs (multi-GPU sharding by contiguous patch ranges). */
int pb_extract_patch_range(const pb_grid_desc* g, const void* tensor, int32_t tensor_f64, const uint8_t* mask,
                           int32_t mean_subtract, int64_t first_patch, int64_t num_patches, float* values,
                           uint8_t* observed, float* means, int32_t* counts, void* stream);

/* reconstitute + apply_data_consistency (patches.py:188-229).
 * out[x] = sum_{i covers x} (est_scale*est[p,i] + means[i]) / coverage(x);
 * if dc: out[x] = original[x] where mask[x].  out/original are f64 if io_f64 else f32.
 * uncovered (device uint64, may be NULL) is incremented per uncovered element. */
int pb_reconstitute(const pb_grid_desc* g, const float* est, float est_scale, const float* means,
                    const void* original, const uint8_t* mask, int32_t dc, int32_t io_f64, void* out,
                    unsigned long long* uncovered, void* stream);

/* Overlap-add of a shard (patches [first_patch, first_patch + num_patches), est/means
 * shard-local): raw f64 sums of (est_scale*est + mean) per element, no division.
 * Summing these across ranks and dividing by coverage gives reconstitute(). */
int pb_ola_partial(const pb_grid_desc* g, const float* est, float est_scale, const float* means, int64_t first_patch,
                   int64_t num_patches, double* acc_out, void* stream);

/* coverage_map (patches.py:181-185), int32 of the tensor shape. */
int pb_coverage_map(const pb_grid_desc* g, int32_t* out, void* stream);

/* ---- fine-grained seam: one entry per reference _kernels.* function ---- */

/* _kernels.residual_full (_kernels.py:18-31).  usage/weights rows have pitch ld >= n. */
int pb_residual_full(const float* values, const uint8_t* observed, const uint8_t* usage, const float* weights,
                     const float* atoms, float* out, int64_t n, int32_t p, int32_t k, int64_t ld, void* stream);
/* _kernels.compose_estimates (_kernels.py:133-145); accumulate!=0 adds into out. */
int pb_compose_estimates(const uint8_t* usage, const float* weights, const float* atoms, float* out, int64_t n,
                         int32_t p, int32_t k, int64_t ld, int32_t accumulate, void* stream);
/* _kernels.atom_moments (_kernels.py:34-62): a_out, c_out are device f64[P];
 * scratch: device f64[2 * P * 64]. */
int pb_atom_moments(const float* resid, const uint8_t* observed, const float* w_col, int64_t n, int32_t p,
                    double* a_out, double* c_out, double* scratch, void* stream);
/* _kernels.shift_atom (_kernels.py:65-74) */
int pb_shift_atom(float* resid, const uint8_t* observed, const float* w_col, const float* delta, int64_t n,
                  int32_t p, void* stream);
/* _kernels.code_moments (_kernels.py:77-97) */
int pb_code_moments(const float* resid, const uint8_t* observed, const float* atom, int64_t n, int32_t p,
                    float* u_out, float* v_out, void* stream);
/* _kernels.shift_codes (_kernels.py:100-109) */
int pb_shift_codes(float* resid, const uint8_t* observed, const float* atom, const float* dw, int64_t n,
                   int32_t p, void* stream);
/* _kernels.masked_sq_norm (_kernels.py:112-130): out = device f64 scalar; scratch f64[256]. */
int pb_masked_sq_norm(const float* resid, int64_t total, double* out, double* scratch, void* stream);

/* ---- observed-element index (built once per mask) ----
 * Every conditional of the reference sampler sums over observed elements only
 * (bpfa.py:1-21), so the sweep stores the residual for the nnz observed
 * elements in a tiled column-major order plus a per-patch slot list.  The
 * index depends on the mask only; pb_index_refresh_values updates the observed
 * values for a new frame under the same mask (the live path). */
typedef struct pb_patch_index {
  int64_t n;        /* patches */
  int32_t p;        /* patch size */
  int32_t ntiles;   /* set by pb_build_index */
  int64_t nnz;      /* observed elements = sum of counts (caller supplies) */
  int32_t cmax;     /* max observed per patch (set by pb_build_index) */
  void* buffer;     /* device buffer of pb_index_bytes(n, p, nnz) bytes */
  int32_t split_count;  /* set by pb_build_index: the code step runs patches with more
                           observed elements in a second, wider launch (0 = one launch) */
  int32_t split_request; /* input: 0 = automatic split choice (cost model), > 0 forces this
                           threshold (when below cmax), < 0 never splits */
  int64_t n_outliers;   /* patches above split_count */
  int64_t nnz_ell;      /* set by pb_build_index: positions of the dictionary step's ELL wave
                           layout (nnz + padding; the residual workspace holds this many) */
} pb_patch_index;

size_t pb_index_bytes(int64_t n, int32_t p, int64_t nnz);
/* Builds the index from the extract_patches outputs; synchronizes `stream` once. */
int pb_build_index(pb_patch_index* index, const uint8_t* observed, const float* values, const int32_t* counts,
                   void* stream);
int pb_index_refresh_values(const pb_patch_index* index, const float* values, const int32_t* counts, void* stream);

/* ---- the sweep: bpfa.gibbs_epoch (bpfa.py:278-345) ---- */

/* Device-resident scalar block of a sampler state (layout fixed, 40 bytes). */
typedef struct pb_scalars {
  double gamma_s;    /* GibbsState.weight_precision */
  double gamma_eps;  /* GibbsState.noise_precision  */
  double sq_w;       /* sum of S^2 after the last code step  */
  double sq_r;       /* sum of R^2 after the last code step  */
  int32_t epoch;     /* GibbsState.epoch */
  int32_t diverged;  /* set by the device pi/gamma draw on non-finite state */
} pb_scalars;

/* Collective hook for sharded (multi-GPU) epochs: sum `count` elements of
 * `device_buf` (dtype 0 = f64, 1 = int32) across all ranks, stream-ordered on
 * `stream`, result in place.  Return 0 on success.  Implemented by the caller
 * (NCCL through torch.distributed in the Python package). */
typedef int (*pb_allreduce_fn)(void* ctx, void* device_buf, int64_t count, int32_t dtype, void* stream);

typedef struct pb_epoch_desc {
  int64_t n;
  int64_t ld;               /* row pitch of usage/weights (K, ld); 0 => n */
  int32_t p, k;
  int32_t freeze_dict;      /* bpfa.gibbs_epoch(freeze_dict=...) */
  int32_t rng_mode;         /* PB_RNG_REPLAY or PB_RNG_PHILOX */
  int32_t resid_mode;       /* PB_RESID_* */
  uint64_t seed;            /* GibbsState.seed */
  int64_t n_obs;            /* number of observed patch-matrix flags (bpfa.py:327) */
  double hyper[6];          /* Hyperparams a, b, c, d, e, f (bpfa.py:46-52) */
  /* problem */
  const float* values;      /* (P,N) */
  const uint8_t* observed;  /* (P,N) */
  const int32_t* counts;    /* (N) observed per patch */
  const pb_patch_index* index;
  /* state (in/out) */
  float* atoms;             /* (K,P) */
  double* pi;               /* (K)   */
  uint8_t* usage;           /* (K,N) */
  float* weights;           /* (K,N) */
  pb_scalars* scalars;
  /* replay draws for this epoch (PB_RNG_REPLAY only; else NULL) */
  const double* atom_draws; /* (K,P) standard normals, stream (seed,2,epoch,k) */
  const double* code_u;     /* (K,N) uniforms, stream (seed,3,epoch,k) random(N) */
  const double* code_g;     /* (K,N) normals,  stream (seed,3,epoch,k) standard_normal(N) */
  /* workspace from pb_epoch_workspace_bytes() */
  void* workspace;
  /* sharding: this rank holds global patches [i_offset, i_offset + n) of n_global;
   * n_obs is the global observed count.  allreduce == NULL => single rank. */
  int64_t i_offset;
  int64_t n_global;
  pb_allreduce_fn allreduce;
  void* allreduce_ctx;
  int32_t codes_zero;       /* caller asserts usage and weights are all zero on entry (fresh init,
                               reset codes): the code step reads no old state — the buffers need
                               not even be cleared, every entry of [0, n) is written */
} pb_epoch_desc;

size_t pb_epoch_workspace_bytes(int64_t n, int32_t p, int32_t k, int64_t nnz);
/* Recommended row pitch for (K, ld) usage/weights: n rounded up to 64 (aligned
 * vector loads in the dictionary step).  Any ld >= n is accepted. */
int64_t pb_code_pitch(int64_t n);

/* One sweep through the dictionary and code steps.  After it returns (stream
 * ordered), scalars->sq_w / sq_r hold the epoch sums and m_counts_out (device
 * int32[K], may be NULL) the per-atom usage counts.  In PB_RNG_PHILOX mode the
 * pi / gamma draws also run on the device (scalars->epoch advances, diverged
 * flags non-finite state); in PB_RNG_REPLAY mode the caller draws pi/gamma from
 * the reference streams and writes pi / scalars itself. */
int pb_gibbs_epoch(const pb_epoch_desc* d, int32_t* m_counts_out, void* stream);

/* Phase timing for profiling/bench: when enabled, every pb_gibbs_epoch brackets
 * its phases with CUDA events on its stream; pb_phase_read returns the summed
 * milliseconds of [residual, dictionary step, code step, stats+pi/gamma] over
 * the epochs since enabling (single host thread use). */
int pb_phase_timing(int32_t enable);
int pb_phase_read(double* ms_out /* [4] */, int64_t* epochs_out);
/* Profiling only: in-kernel globaltimer phases of the dictionary step as seen by
 * thread 0 of each CTA, mean over CTAs, accumulated since enabling:
 * [tile-top barrier, W/colptr copy wait, element work, tile-end barrier,
 *  boundary merge, pass-end partials, grid sync 1, per-pixel reduce,
 *  grid sync 2, shift load, owner atom update, -]. */
int pb_dict_profile(int32_t enable, double* slots_ns_out /* [12] or NULL */);

/* ---- native NCCL for the sharded sweep ----
 * libnccl.so.2 is dlopen'ed (the copy already loaded in the process if any).
 * pb_nccl_allreduce has the pb_allreduce_fn signature: pass its address as
 * pb_epoch_desc.allreduce and the communicator as allreduce_ctx, and every
 * exchange of the sweep is an ncclAllReduce (in-place sum) enqueued on the
 * epoch's stream — no host round trip.  id: 128 bytes (ncclUniqueId). */
int pb_nccl_unique_id(uint8_t* id_out);
int pb_nccl_comm_create(const uint8_t* id, int32_t world, int32_t rank, void** comm_out);
int pb_nccl_comm_destroy(void* comm);
int pb_nccl_allreduce(void* comm, void* device_buf, int64_t count, int32_t dtype, void* stream);

/* ---- adaptive-residual sampling mask on device (sampling.py:184-207) ----
 * Budget round(ratio*M); exploit = the round(exploit_fraction*budget) largest
 * residuals, ties by lowest flat index (bit-exact with the reference's stable
 * argsort); explore = the rest of the budget drawn uniformly without
 * replacement from the unexploited elements with a device Philox stream keyed by
 * (seed, frame_index) — NOT numpy's Generator.choice stream.  An all-zero map
 * draws the whole budget uniformly (status 1).  Negative / NaN residuals:
 * PB_EVALUE.  residual and mask_out are device pointers. */
int pb_adaptive_mask(const double* residual, int64_t m, double ratio, double exploit_fraction, uint64_t seed,
                     int64_t frame_index, uint8_t* mask_out, int32_t* status_out, void* stream);

/* ---- dictionary atlas for the console (server.py:84-120), on device ----
 * Canvas (height, width) = (g*B0 + g-1, g*B1 + g-1), g = ceil(sqrt(K)); rank-1
 * patches render as one row, rank-3 as slice 0 of the last axis, rank 4 refuses.
 * atoms (K,P) f32, pi (K) f64 device; canvas f64 and/or canvas_u8
 * (round(clip(x,0,1)*255)) device outputs (either may be NULL). */
int pb_atlas_shape(int32_t k, int32_t rank, const int32_t* patch_shape, int64_t* height, int64_t* width);
int pb_render_atlas(const float* atoms, const double* pi, int32_t k, int32_t rank, const int32_t* patch_shape,
                    double* canvas, uint8_t* canvas_u8, void* stream);

/* ---- entry-point steps (cli.py / bpfa.py) on device ---- */
/* cli.py:195-212 _normalize_observed: frame (f64, M) -> out (f64, M, may alias
 * frame) mapped to [0, 1] from the observed values only (mask uint8); identity
 * when they already lie in [0, 1] or none is observed; a constant observed set
 * maps observed elements to 0.  scale_out / offset_out (host) as the reference
 * returns them.  Synchronizes `stream`. */
int pb_normalize_observed(const double* frame, const uint8_t* mask, int64_t m, double* out, double* scale_out,
                          double* offset_out, void* stream);
/* bpfa.py:417-458 transfer_dictionary tiling: dst (K, src_p*repeat) f32 where each
 * source element is repeated `repeat` = prod(extra trailing patch dims) times,
 * renormalized to unit norm when `normalize` (zero atoms stay zero); normalize = 0
 * with repeat = 1 copies bitwise (equal patch shapes).  Device pointers. */
int pb_transfer_atoms(const float* src, int32_t k, int32_t src_p, int32_t repeat, int32_t normalize, float* dst,
                      void* stream);

/* ---- stateful problem (C-ABI with HOST buffers; the live submit_frame slice,
 *      pipeline.py:217-251).  Owns all device buffers. ---- */
typedef struct pb_problem pb_problem;

/* Host draw provider of a replay-mode problem (pb_problem_desc.replay = 1): the
 * reference's keyed numpy streams (rng.py:25-32) evaluated by the caller; called
 * from inside pb_problem_submit_frame on the calling thread.
 *   PB_DRAW_PRIOR      (epoch 0)  out0 = prior atoms, K*P f64 row-major, stream (seed, 1)
 *                                 scaled by 1/sqrt(P) (bpfa.py:121-122)
 *   PB_DRAW_EPOCH      (epoch e)  out0 = atom normals K*P, stream (seed, 2, e, k) — NULL when
 *                                 the dictionary is frozen; out1 / out2 = code uniforms /
 *                                 normals K*N, stream (seed, 3, e, k) (bpfa.py:293-310)
 *   PB_DRAW_POSTERIOR  (epoch e)  in m_counts (K), sums = {sum S^2, sum R^2, n_obs};
 *                                 out0 = pi (K) from (seed, 4, e), out1 = {gamma_s, gamma_eps}
 *                                 from (seed, 5, e), floors applied (bpfa.py:313-333)
 * Return 0 on success; anything else aborts the frame with PB_EVALUE. */
#define PB_DRAW_PRIOR 0
#define PB_DRAW_EPOCH 1
#define PB_DRAW_POSTERIOR 2
typedef int (*pb_draw_fn)(void* ctx, int32_t stage, int64_t epoch, const int32_t* m_counts, const double* sums,
                          double* out0, double* out1, double* out2);

#define PB_INIT_PRIOR 0    /* bpfa.init_state(init_mode="prior") */
#define PB_INIT_DATA 1     /* init_mode="data" (bpfa.py:126-134; Pipeline default, pipeline.py:52) */

typedef struct pb_problem_desc {
  pb_grid_desc grid;
  int32_t num_atoms;
  double hyper[6];
  uint64_t seed;
  int32_t mean_subtract;
  int32_t epochs_per_frame;
  int32_t freeze_dict;
  int32_t data_consistency;
  int32_t warm_start;
  int32_t average_last;
  int32_t replay;        /* 0: device Philox draws (the fast path); 1: the reference streams from `draw` */
  int32_t init_mode;     /* PB_INIT_*: cold start of the dictionary.  Data-mode atoms only survive
                            the first dictionary step when the dictionary is frozen (SURVEY App. A
                            Q1), so they are gathered on the device only then. */
  pb_draw_fn draw;       /* replay mode only */
  void* draw_ctx;
} pb_problem_desc;

int pb_problem_create(const pb_problem_desc* desc, pb_problem** out);
int pb_problem_destroy(pb_problem* pr);
/* One live frame: H2D frame (f64) + mask (uint8, cached when unchanged),
 * extract, epochs_per_frame warm-started sweeps (device Philox draws, or in replay
 * mode the reference streams from desc.draw, one host round trip per epoch for
 * the pi / gamma draws), compose, overlap-add,
 * data consistency, D2H reconstruction (f64).  Mirrors Pipeline.submit_frame's
 * hot slice (pipeline.py:224-251). */
int pb_problem_submit_frame(pb_problem* pr, const double* frame_host, const uint8_t* mask_host,
                            double* recon_host);
/* submit_frame plus the device-resident tail: any output may be
 * NULL.  recon_host f64 (M) after data consistency; panel_host / masked_host
 * uint8 wire panels of the reconstruction and of frame*mask,
 * round(clip(x,0,1)*255) (server.py:46-53; rank-3 tensors show slice 0, other
 * ranks refuse).  Every frame also updates the device residual map
 * (recon - previous recon)^2 of the pre-consistency reconstruction
 * (pipeline.py:265-269). */
int pb_problem_submit_frame_ex(pb_problem* pr, const double* frame_host, const uint8_t* mask_host,
                               double* recon_host, uint8_t* panel_host, uint8_t* masked_host);
/* The residual map of the last frame (f64, M), copied to host. */
int pb_problem_residual_map(pb_problem* pr, double* host_out);
/* The adaptive-residual sampler (sampling.py:184-207) on the problem's residual
 * map: writes the next mask (uint8, M) to host and keeps it as the cached
 * device mask.  status 1 = all-zero map (uniform device draw). */
int pb_problem_adaptive_mask(pb_problem* pr, double ratio, double exploit_fraction, uint64_t seed,
                             int64_t frame_index, uint8_t* mask_host, int32_t* status_out);
/* Adopt a dictionary (Pipeline._install_dictionary, pipeline.py:145-167): atoms
 * (K,P) f32 and pi (K) host arrays of THIS problem's P (reshape first with
 * bpfa.transfer_dictionary / pb_transfer_atoms) and any atom count K (the
 * problem's K-dependent buffers are re-sized).  Before the first frame it is
 * pending and seeds the cold start (install_dictionary semantics,
 * bpfa.py:355-376: precisions at the prior means); afterwards it replaces the
 * dictionary and keeps the precisions and the epoch counter.  freeze: 0/1 sets
 * freeze_dict, -1 keeps it. */
int pb_problem_install_dictionary(pb_problem* pr, const float* atoms_host, const double* pi_host, int32_t k,
                                  int32_t freeze);
/* Pipeline.transfer_between (pipeline.py:294-304) on the device: src's current
 * dictionary (or its pending install) reshaped for dst by the transfer_dictionary
 * rules (bpfa.py:417-458, pb_transfer_atoms) and installed into dst as above.
 * PB_EVALUE for src == dst or a source without state; PB_ESHAPE for
 * incompatible patch shapes. */
int pb_problem_transfer_dictionary(pb_problem* src, pb_problem* dst, int32_t freeze);
/* The problem's current dictionary atlas as a uint8 wire panel (host buffer of
 * pb_atlas_shape's size). */
int pb_problem_render_atlas(pb_problem* pr, uint8_t* canvas_u8_host);
/* Device-side timing of the last submit_frame's GPU work (ms). */
float pb_problem_last_gpu_ms(pb_problem* pr);
/* Current dictionary (K,P) f32 and scalars, copied to host. */
int pb_problem_get_dictionary(pb_problem* pr, float* atoms_host, double* pi_host, pb_scalars* scalars_host);

#ifdef __cplusplus
}
#endif
#endif /* PB200_H_ */
