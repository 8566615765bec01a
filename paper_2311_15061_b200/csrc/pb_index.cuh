// pb200 — observed-element index (pb_index.cu) shared by the compact sweep kernels.
#pragma once
#include "pb_common.cuh"

namespace pb {

constexpr int kTile = 1024;        // patches per CSC tile (one dict-step work unit)
constexpr int kFillThreads = 512;  // index-build block size (two patches per thread)
constexpr int kWB = 8;             // atoms per block of the tile-blocked code copy W
constexpr int kSegCountLen = 256;  // segment length of the dictionary step's element phase (cost model)

__host__ __device__ constexpr int colptr_pitch(int p) { return (p + 1 + 3) & ~3; }

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
};

int index_bytes(int64_t n, int p, int64_t nnz, size_t* out);
void carve_index(PatchIndex& ix, char* base, int64_t n, int p, int64_t nnz);
int launch_build_index(PatchIndex& ix, const uint8_t* obs, const float* values, const int32_t* counts,
                       cudaStream_t st);
int launch_scatter_x(const PatchIndex& ix, const float* values, const int32_t* counts, cudaStream_t st);
int launch_count_hist(const PatchIndex& ix, const int32_t* counts, cudaStream_t st);
int launch_outliers(const PatchIndex& ix, const int32_t* counts, int split, cudaStream_t st);

}  // namespace pb
