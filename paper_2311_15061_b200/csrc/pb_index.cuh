// pb200 — observed-element index (pb_index.cu) shared by the compact sweep kernels.
#pragma once
#include "pb_common.cuh"

namespace pb {

constexpr int kTile = 1024;        // patches per CSC tile (one dict-step work unit)
constexpr int kFillThreads = 512;  // index-build block size (two patches per thread)
constexpr int kWB = 8;             // atoms per block of the tile-blocked code copy W
constexpr int kSegCountLen = 256;  // segment length of the dictionary step's element phase (cost model)

__host__ __device__ constexpr int colptr_pitch(int p) { return (p + 1 + 3) & ~3; }

// ---- ELL wave layout of the dictionary step (see pb_index.cu) ----
constexpr int kEllRun = 32;                 // max elements of one lane's run
constexpr uint32_t kEllZeroRow = 32768u;    // W-row byte offset of the zero row behind each staged block
// upper bounds of the ELL element and wave counts (padding included)
__host__ __device__ inline int64_t ell_cap(int64_t n, int64_t nnz) {
  return 2 * nnz + 6144 * ((n + kTile - 1) / kTile) + 1024;
}
__host__ __device__ inline int64_t wave_cap(int64_t n, int p, int64_t nnz) {
  return ((n + kTile - 1) / kTile) * (8 + (2 * p + 31) / 32) + 2 * nnz / 1024 + 1;
}

// Byte offset of patch row il's first 16-byte chunk inside a tile block of the
// code copy W ([kTile][kWB] floats); the second chunk is at (offset ^ 16).
// Chunks are XOR-swizzled across each 128-byte line (4 rows) so gathers of
// nearby rows spread over the shared-memory banks.
__host__ __device__ constexpr uint32_t w_row_off(int il) {
  return ((uint32_t)(il >> 2) << 7) | ((uint32_t)(((il & 3) << 1) ^ ((il >> 2) & 7)) << 4);
}

struct PatchIndex {
  int64_t n;
  int p;
  int ntiles;
  int32_t* tile_tot;    // [ntiles]
  int64_t* tile_base;   // [ntiles + 1] first element of each tile; tile_base[ntiles] = nnz
  int32_t* colptr;      // [ntiles][colptr_pitch(p)] tile-relative first element of each column (p+1 used)
  int64_t* rowptr;      // [n + 1] first CSR slot of each patch
  uint16_t* e_loc;      // [nnz] CSC: w_row_off(patch index inside its tile) — the W row of the element
  float* x_csc;         // [nnz] CSC: observed (mean-subtracted) value
  uint16_t* csr_p;      // [nnz] CSR: patch offset p of each slot
  uint32_t* csr_pos;    // [nnz] CSR: CSC position of each slot
  int32_t* cmax_dev;    // max observed count over patches
  int32_t* outliers;    // [n] ids of the patches above the code-step split, ascending
  int32_t* out_tot;     // [ntiles]
  int64_t* out_base;    // [ntiles + 1]; out_base[ntiles] = number of outliers
  int32_t* hist;        // [p + 1] histogram of the observed counts
  int32_t* tile_segs;   // [ntiles] column segments of each tile (columns cut every kSegCountLen elements)
  int64_t* seg_base;    // [ntiles + 1] prefix of tile_segs (the dictionary step's work-split cost model)
  // ELL wave layout (the dictionary step's order; x_csc and the residual live in it)
  uint32_t* slot_csc;   // [nnz] CSC scratch: CSR slot of each CSC element
  uint16_t* e_ell;      // [ell_cap] W-row byte offset per ELL position (kEllZeroRow for padding)
  int32_t* ell_tot;     // [ntiles] ELL positions of each tile (padding included)
  int64_t* ell_base;    // [ntiles + 1]
  int32_t* wave_tot;    // [ntiles] waves of each tile
  int64_t* wave_base;   // [ntiles + 1] first global wave of each tile
  uint32_t* wave_off;   // [waves] first ELL position of the wave, relative to its tile's ell_base
  uint16_t* wave_meta;  // [waves] run length Lw | log2(lanes per column) << 8
  uint16_t* wave_col;   // [waves][32] column of each lane's run (0xFFFF: idle lane)
};

int index_bytes(int64_t n, int p, int64_t nnz, size_t* out);
void carve_index(PatchIndex& ix, char* base, int64_t n, int p, int64_t nnz);
int launch_build_index(PatchIndex& ix, const uint8_t* obs, const float* values, const int32_t* counts,
                       cudaStream_t st);
int launch_scatter_x(const PatchIndex& ix, const float* values, const int32_t* counts, cudaStream_t st);
// Cached-mask live frame, rank 2: observed values (and means) from the frame
// straight into the index's compact order (no dense extraction).
int launch_refresh_frame2d(const PatchIndex& ix, const double* frame, int64_t m1, int64_t gc1, int b1, int s0, int s1,
                           int mean_subtract, const int32_t* counts, float* means, cudaStream_t st);
int launch_count_hist(const PatchIndex& ix, const int32_t* counts, cudaStream_t st);
int launch_outliers(const PatchIndex& ix, const int32_t* counts, int split, cudaStream_t st);

}  // namespace pb
