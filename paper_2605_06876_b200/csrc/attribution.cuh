#pragma once

#include "adps_internal.cuh"

namespace adps {

struct TileParams {
  const float* image;
  const float* gt;
  const int* dom;
  int H, W;
  int tiles_x, tiles_y;
  int view_offset, view_stride;     // global view position = view_offset + v * view_stride
  const double* lo;
  const double* thr;
  const double* thr_raw;             // the thresholds in the raw domain (warp CCL)
  int L, r_erode, m_min;
  const unsigned char* cls;
  int N;
  unsigned char* dom_flag;
  RegionRec* regions;
  unsigned long long* n_regions;
  long long region_cap;
  PartialRec* partials;
  unsigned long long* n_partials;
  long long partial_cap;
  int* partial_parent;
  unsigned long long* tile_records;   // packed partials << 32 | regions of the tile CCLs
  int* border;
  unsigned char* dbg_m;
  unsigned char* dbg_b;
  unsigned int* overflow;
  int n_views;
  int* deferred;                     // tiles the warp kernel hands to the block kernel
  unsigned long long* n_deferred;
  const unsigned* cand_bits;         // [V][ceil(H*W/32)]: bit p = D[p] is a split candidate
  const double* raw;                 // [V][H*W] raw L1 error cached by the minmax pass, or null
  uint4* words;                      // [V][H][ceil(W/32)] bit planes (m, cand, band0, band1), or null
  const raw16_t* rawf;               // [V][H*W] 16-bit raw-error cache (bit-plane path), or null
};

struct BorderParams {
  const int* border;
  const PartialRec* partials;
  int* parent;
  int tiles_x, tiles_y;
  int W, H;
  long long n_tiles;
};

struct AttributionArgs {
  const float* image;
  const float* gt;
  const int* dom;
  int V, H, W, view_offset, view_stride;
  int L, r_erode, m_min;
  double tau;
  const unsigned char* cls;
  int N;
  unsigned char* dom_flag;
  unsigned long long* lohi;   // [2V], preset to (+inf bits, 0)
  double* lo;                 // [V]
  double* thr;                // [V*L]
  double* thr_raw;            // [V*L] the same as raw L1 thresholds
  RegionRec* regions;
  unsigned long long* n_regions;
  long long region_cap;
  PartialRec* partials;
  unsigned long long* n_partials;
  long long partial_cap;
  int* partial_parent;
  unsigned long long* tile_records;   // packed partials << 32 | regions of the tile CCLs
  int* border;                // [V * tiles * kBorderSlots]
  unsigned char* dbg_m;
  unsigned char* dbg_b;
  unsigned int* overflow;
  unsigned grid_small;
  int input_blocks_per_sm;   // resident blocks per SM of the input pass (0: all that fit)
  int* deferred;                     // [n_tiles]
  unsigned long long* n_deferred;
  int tile_path;                     // 0 auto (warp kernel + deferred), 1 block kernel only,
                                     // 2 warp kernel on the raw cache without bit planes
  unsigned* cand_bits;               // [V][ceil(H*W/32)], written by the minmax pass
  double* raw;                       // [V][H*W] raw L1 error written by the minmax pass, or null
  uint4* words;                      // [V][H][ceil(W/32)] bit planes for tile_bits_kernel, or null
  raw16_t* rawf;                     // [V][H*W] 16-bit raw-error cache (bit-plane path), or null
};

// warp-per-tile scanline CCL (r_erode <= 3) over tiles [t0, t1); defers tiles with > kWarpMaxRuns runs
cudaError_t launch_tile_warp(const TileParams& P, long long t0, long long t1, cudaStream_t s);
size_t tile_warp_smem_bytes();
// bit-plane path (raw cache, l_bands <= 4, r_erode <= 3): words pass + tile_bits_kernel over views [v0, v1)
cudaError_t launch_tile_bits(const TileParams& P, int v0, int v1, cudaStream_t s);
// the tiles launch_tile_bits deferred (P.deferred / P.n_deferred), a warp each
cudaError_t launch_tile_bits_deferred(const TileParams& P, unsigned blocks, cudaStream_t s);
size_t tile_words_bytes(int V, int H, int W);

size_t tile_smem_bytes();
// minmax + ever-dominant flags + thresholds + fallback count (phase-1 begin)
cudaError_t launch_minmax(const AttributionArgs& a, const int* split_list, Counters* ctr, int sm_count,
                          cudaStream_t s);
// fallback count alone (after the dom_flag buffer was reduced across ranks)
cudaError_t launch_fallback_count(const int* split_list, const unsigned char* dom_flag, Counters* ctr, int sm_count,
                                  cudaStream_t s);
// Called after each group of launches: name, stream, number of kernels launched.
typedef void (*MarkFn)(void* ctx, const char* name, cudaStream_t s, int kernels);
cudaError_t launch_attribution(const AttributionArgs& a, cudaStream_t s, MarkFn mark, void* ctx);
// the same in pieces, so views can be pipelined: minmax + thresholds of views
// [v0, v1); warp CCL of their tiles; then the deferred tiles + border merge
cudaError_t launch_minmax_views(const AttributionArgs& a, int v0, int v1, cudaStream_t s);
// the same in its two launches (stage timing): the input pass, then the thresholds
cudaError_t launch_minmax_kernel(const AttributionArgs& a, int v0, int v1, cudaStream_t s);
cudaError_t launch_thresholds(const AttributionArgs& a, int v0, int v1, cudaStream_t s);
cudaError_t launch_tiles_views(const AttributionArgs& a, int v0, int v1, cudaStream_t s);
cudaError_t launch_attribution_tail(const AttributionArgs& a, cudaStream_t s, MarkFn mark, void* ctx);
bool attribution_warp_path(const AttributionArgs& a);

}  // namespace adps
