#pragma once

#include "adps_internal.cuh"
#include "scan.cuh"

namespace adps {

#ifndef ADPS_MERGE_TILE
#define ADPS_MERGE_TILE 32
#endif
// proposals per Morton tile of a large parent's gate matrix (exact pruning unit)
constexpr int kMT = ADPS_MERGE_TILE;
#ifndef ADPS_MORTON_BITS
#define ADPS_MORTON_BITS 6
#endif
constexpr int kMortonBits = ADPS_MORTON_BITS;   // per axis (<= 10)

// Cross-view merge + cap over all split candidates at once
// (ref/cross_view_merge.py:33-116, ref/adc.py:184-227).
//
// Proposal space: valid proposals (t* > 0) gathered in reference order
// (candidate, view, band, first pixel); candidate k owns [pstart[k], +P_k).
// default MergeArgs::sel_huge (ADPS_PARAM_CAP_HUGE): parents with more merged
// groups take the cap's cluster selection
constexpr int kSelHuge = 4096;

struct MergeArgs {
  // inputs
  const unsigned long long* keys_sorted;   // region sort keys
  const int* vals_sorted;                  // sorted pos -> region id
  long long n_regions;
  int shift_rank;
  const unsigned char* valid;              // region id -> t* > 0
  const Proposal* props;                   // region id -> proposal
  const int* split_list;
  const int* cand_start;                   // first sorted region position of a candidate
  const int* cand_nvalid;                  // P_k
  const unsigned char* dom_flag;
  const float* opacity;
  double gamma_d, gamma_c;
  int n_max;
  int small_max;                           // P <= small_max: warp path for the gates
  int sel_huge;                            // more groups than this: the cap's cluster selection
  // proposal space
  Proposal* props_s;                       // [cap]
  int* psrc;                               // [cap] proposal q -> region id (gather source)
  int* pcand;                              // [cap] candidate rank
  int* uf;                                 // [cap]
  unsigned* gkey;                          // [cap] root (group key), padding UINT_MAX
  int* gval;                               // [cap] proposal q
  unsigned* gkey_sorted;
  int* gval_sorted;
  // groups
  int* grp_first;                          // [cap] first sorted position of group g
  GroupRec* groups;                        // [cap]
  int* gpar;                               // [cap] candidate rank of group g (groups of a
                                           // candidate are contiguous, in root order)
  double* gext;                            // [cap] extent of group g (compact, for the cap)
  int* gfirst_of;                          // [n_split] first group of candidate k
  int* glist;                              // [3 cap] groups with > 8 / > 512 members; cap list
  long long glist_cap;                     // = cap (set by launch_merge_groups)
  // per candidate
  int* pstart;                             // [n_split]
  int* n_groups;                           // [n_split]
  int* cand_case;
  int* cand_props;
  int* cand_merged;
  int* cand_ins;
  int* small_list;                         // [n_split]
  int* large_list;                         // [n_split]
  unsigned long long* work_cnt;            // [n_split]   tile pairs of large parent l
  unsigned long long* work_off;            // [n_split + 1]
  // exact spatial pruning of large parents' gate matrices
  double extent;
  int* large_of;                           // [n_split] large id or -1
  unsigned long long* lp_cnt;              // [n_split]   proposals of large parent l
  unsigned long long* lp_off;              // [n_split + 1]
  unsigned long long* tile_cnt;            // [n_split]   64-proposal tiles of large parent l
  unsigned long long* tile_off;            // [n_split + 1]
  unsigned long long* mkey;                // [cap] (l << 32) | morton(mu), ~0 elsewhere
  int* mval;                               // [cap]
  unsigned long long* mkey_sorted;
  int* mval_sorted;                        // Morton order: [lp_off[l], +P_l) -> proposal q
  TileBox* boxes;                          // [cap / kMT + n_split]
  int* tile_owner;                         // [cap / kMT + n_split] large parent of each tile
  double* gsoa;                            // [13][soa_cap] gate operands in Morton order
  float* fsoa;                             // [soa_cap][2] float4: fp32 (mu, inv_smax), (rgb, 0) (prefilter)
  long long soa_cap;
  int4* tile_pairs;                        // surviving (l, bi, bj) tile pairs
  long long tile_pairs_cap;
  float* children;                         // [cap,14]
  Counters* ctr;
  unsigned grid;
  const unsigned long long* own;           // [lo, hi) candidate ranks this rank merges, or null = all
};

__device__ __forceinline__ bool owns(const MergeArgs& a, long long k) {
  return !a.own || (k >= (long long)a.own[0] && k < (long long)a.own[1]);
}

// parent sharding: candidate k goes to rank floor(W_<k * world / W) with
// W_<k the exclusive prefix of (P_k^2 + 1), the gate work; writes [lo, hi) and the
// proposal range [p_lo, p_hi) to lohi[0..3]
cudaError_t launch_shard_range(const int* nvalid, long long n, int rank, int world, unsigned long long* lohi,
                               cudaStream_t s);

cudaError_t launch_merge_prepare(const MergeArgs& a, long long n_split, ScanState st, cudaStream_t s);
cudaError_t launch_merge_small_gates(const MergeArgs& a, cudaStream_t s);
// the same split in two: gates of the small parents / offsets of the large ones
cudaError_t launch_small_pairs(const MergeArgs& a, cudaStream_t s);
cudaError_t launch_large_offsets(const MergeArgs& a, cudaStream_t s);
cudaError_t launch_merge_morton(const MergeArgs& a, long long cap, cudaStream_t s);
cudaError_t launch_merge_tile_gates(const MergeArgs& a, cudaStream_t s);
cudaError_t launch_merge_flatten(const MergeArgs& a, long long cap, cudaStream_t s);
cudaError_t launch_merge_groups(const MergeArgs& a, long long cap, ScanState st, cudaStream_t s,
                                cudaStream_t aux = nullptr, cudaEvent_t fork = nullptr, cudaEvent_t join = nullptr);
// cap (ref/cross_view_merge.py:110-116): rank of each group among its parent's
// groups by (-extent, group order); ranks < n_max become children in rank order
cudaError_t launch_merge_cap(const MergeArgs& a, long long cap, cudaStream_t s, cudaStream_t aux,
                             cudaEvent_t fork, cudaEvent_t join);

}  // namespace adps
