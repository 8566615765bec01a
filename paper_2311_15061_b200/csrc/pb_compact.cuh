// pb200 — compact (observed-element) sweep kernels: argument blocks and launchers.
#pragma once
#include <algorithm>

#include "pb_index.cuh"
#include "pb_sweep.cuh"

namespace pb {

constexpr int kProfSlots = 12;  // in-kernel dictionary-step profile slots per CTA

struct CompactArgs {
  // index (CSR view) + residual in CSC order
  const int32_t* counts;
  const int64_t* rowptr;
  const uint16_t* csr_p;
  const uint32_t* csr_pos;
  const float* x_csc;
  float* r_csc;
  int cmax;
  // tile-blocked copy of w = z*s for the dictionary step: [tile][k/8][patch-in-tile][k%8]
  float* wt;
  int nblk8;
  // state
  uint8_t* usage;
  float* weights;
  const float* atoms;
  const double* pi;
  const SweepScalars* sc;
  // replay draws (code step)
  const double* u_draw;
  const double* g_draw;
  // outputs
  double* block_sums;
  int32_t* m_count;
  int64_t n;
  int64_t ld;           // row pitch of usage/weights (K, ld), ld >= n
  int p, k, kc;
  uint32_t key0, key1;
  uint32_t rk[20];      // Philox round keys of (key0, key1) (philox_round_keys)
  int64_t i_offset;     // global index of local patch 0 (draw counters of a shard)
  // code-step split: the main launch skips patches with more than `split`
  // observed elements; the second launch runs exactly the patches in plist
  int split;
  const int32_t* plist;
  int64_t plist_n;
  int zero_mcount;      // the launch zeroes the usage counts first
  unsigned* blk_ctr;    // dynamic block counter of the launch (zeroed by the launcher)
  const float* dt_img;  // pre-packed transposed dictionary chunks (launch_pack_dt)
  int64_t dt_img_floats;
  int codes_zero;       // usage / weights are all zero on entry: the code step loads no old state
};

struct DictGramArgs {
  // index (ELL wave view, pb_index.cu)
  const int64_t* ell_base;    // [ntiles + 1] ELL positions per tile (prefix)
  const int64_t* wave_base;   // [ntiles + 1] waves per tile (prefix)
  const uint32_t* wave_off;   // [waves] first position of the wave inside its tile
  const uint16_t* wave_meta;  // [waves] Lw | log2(R) << 8
  const uint16_t* wave_col;   // [waves][32] column of each lane (0xFFFF idle)
  const uint16_t* e_ell;      // [nnz_ell] W-row byte offset of each position
  int ntiles;
  const float* wt;      // tile-blocked code copy [tile][k/8][patch][8]
  int nblk8;
  float* r_csc;
  // state
  const uint8_t* usage;
  const float* weights;
  float* atoms;
  const double* draws;  // replay atom normals (K,P) or null
  const SweepScalars* sc;
  // workspace
  float* partials;      // max_blocks * P * NACC
  double* reduced;      // P * NACC
  unsigned* bar;        // [4] grid-barrier counters, then [P] per-pixel shift-ready flags (zeroed per launch)
  unsigned long long* prof;  // optional [gridDim][kProfSlots] phase nanoseconds (profiling)
  unsigned long long* wprof;  // optional per-wave [ns, smid, warp] of pass 3 (tuning builds, profiling)
  int dbg;              // profiling-only: 4 skip the W/colptr bulk copies, 8 skip the element phase
  // split (multi-rank) mode: run the single pass blk_begin and stop after the
  // per-GPU reduction; the previous pass's shifts come from delta_g [B][P]
  int split;
  int blk_begin;
  float* delta_g;
  int max_blocks;
  int wbytes;
  int pstage_off;       // byte offset of the staged owner partials in shared memory (0: read from L2)
  int w_evict_first;    // the current block's W copy with an L2 evict_first policy too
  int dyn_waves;        // warps claim their waves from a CTA counter (else round-robin)
  double tile_cost;     // work split: ELL positions equivalent to one tile visit
  int split_nearest;    // work split: CTA boundaries at the nearest wave start (else the preceding one)
  int pixel_flags;      // per-pixel ready flags instead of the second grid barrier of a pass
  int64_t n;
  int64_t ld;           // row pitch of usage/weights (K, ld), ld >= n
  int64_t nnz;          // observed elements (host copy of tile_base[ntiles])
  int p, k;
  uint32_t key0, key1;
};

int launch_resid_compact(const CompactArgs& a, cudaStream_t st);
int launch_code_compact(const CompactArgs& a, int mode, int& nblocks, cudaStream_t st);
// the code step's per-patch limit for the main launch from the count histogram (0 = no split)
int code_split_choose(const int32_t* hist, int p, int cmax);
int code_launch_blocks(int cmax, int64_t n, int p, int k);  // blocks of patches (= S^2/R^2 pairs) of a launch
int launch_dict_gram(const DictGramArgs& a, cudaStream_t st);
// dictionary step on all-zero codes: prior redraw of every atom (bit-identical to launch_dict_gram on W == 0)
int launch_dict_prior(const DictGramArgs& a, cudaStream_t st);
// code step's transposed-dictionary chunks: layout and the per-sweep packing kernel
void code_dt_layout(int p, int k, int* kc_out, int64_t* img_floats_out, int* nchunks_out);
int launch_pack_dt(const float* atoms, int p, int k, float* img, cudaStream_t st);
int launch_dict_update(const DictGramArgs& a, int blk, cudaStream_t st);
int dict_gram_blocks(int k);
size_t dict_gram_partials_bytes(int p, int max_blocks);
size_t dict_gram_reduced_bytes(int p);

}  // namespace pb
