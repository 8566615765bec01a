// pb200 — live-path tail kernels (pb_live.cu).
#pragma once
#include "pb_common.cuh"

namespace pb {

struct LiveFinishArgs {
  const double* recon;   // overlap-add reconstruction before data consistency (M)
  const double* frame;   // the frame (M)
  const uint8_t* mask;   // sampling mask (M)
  double* out;           // reconstruction after data consistency (M)
  double* prev;          // previous frame's reconstruction (M), updated; null: no residual map
  double* resid;         // (recon - prev)^2 (M) or 0 without a previous frame
  uint8_t* panel;        // optional uint8 panel of `out` (2-D, or slice 0 of a rank-3 tensor)
  uint8_t* masked;       // optional uint8 panel of frame * mask
  int64_t m;
  int64_t panel_stride;  // 1 for rank 2; C for (H, W, C)
  int dc;
  int have_prev;
};

int launch_live_finish(const LiveFinishArgs& a, cudaStream_t st);
// bpfa.py:126-134 data-mode seeding: atoms[j] <- unit-normalized values of the
// j-th patch by (observed count desc, index asc); zero-norm / surplus atoms untouched
int launch_data_atoms(const float* values_pn, const int32_t* counts, int64_t n, int p, int k, float* atoms,
                      cudaStream_t st);
// sampling.py:184-207 on device; status 1 = all-zero residual (uniform draw)
int adaptive_mask(const double* resid, int64_t m, int64_t budget, int64_t n_exploit, uint32_t k0, uint32_t k1,
                  uint64_t frame_index, uint8_t* mask, int* status, cudaStream_t st);

// pb_select.cu: the n largest of keys[0, m), ties by lowest index (1 <= n <= m):
// mark[x] = 1 for each selected x (if mark; other entries untouched) and/or the
// selected indices appended to list (if list; unordered).  scratch: device
// memory of select_scratch_bytes(m).
size_t select_scratch_bytes(int64_t m);
int select_top(const uint64_t* keys, int64_t m, int64_t n, void* scratch, uint8_t* mark, int32_t* list,
               cudaStream_t st);

// server.py:84-120: atlas geometry and render (canvas f64 and/or uint8, device)
int atlas_geometry(int k, int rank, const int32_t* shape, int& b0, int& b1, int& inner, int& grid, int64_t& h,
                   int64_t& w);
int launch_atlas(const float* atoms, const double* pi, int k, int rank, const int32_t* shape, double* canvas,
                 uint8_t* canvas_u8, cudaStream_t st);

}  // namespace pb
