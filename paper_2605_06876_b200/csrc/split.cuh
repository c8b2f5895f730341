#pragma once

#include "adps_internal.cuh"
#include "scan.cuh"

namespace adps {

struct GaussiansIn {
  const float* mu;
  const float* scale;
  const float* rot;
  const float* opacity;
  const float* sh_dc;
  const float* sh_rest;
  int sh_k;
};

// ---- select (ref/adc.py:41-46, 82-89) ----
struct SelectArgs {
  const float* scale;
  const double* ga;
  const double* den;
  double tau_g, tau_s_abs;
  long long n;
  unsigned char* cls;        // 0 none, 1 split, 2 clone
  int* cand_rank;            // rank in split list or -1
  int* split_list;
  int* clone_list;
  Counters* ctr;
  // (classify kernel only) zero the ever-dominant flags and seed the per-view
  // min/max slots (+inf, +0) in the same pass: no memset / host copy between kernels
  unsigned char* dom_zero = nullptr;
  unsigned long long* lohi_init = nullptr;
  int lohi_views = 0;
};
cudaError_t launch_select(const SelectArgs& a, ScanState st, cudaStream_t s);
// classes on `s`, then the split/clone list scan on `aux` (recorded into `join`):
// the input pass on `s` needs only the classes
cudaError_t launch_select_split(const SelectArgs& a, ScanState st, cudaStream_t s, cudaStream_t aux, cudaEvent_t fork,
                                cudaEvent_t join);

// ---- region stats + child init (ref/error_partition.py:137-158, ref/child_init.py:44-140) ----
struct ChildArgs {
  const RegionRec* regions;
  const unsigned long long* n_regions;
  long long region_cap;
  GaussiansIn g;
  const double* cams;        // [V,18] device (local views)
  const float* gt;           // [V,H,W,3] (local views)
  int H, W;
  int view_offset, view_stride;   // region view_pos (global) -> local view (view_pos - offset) / stride
  double eps;
  const int* cand_rank;
  int bits_v, bits_b, bits_p;
  Proposal* props;
  unsigned char* valid;
  unsigned long long* keys;   // written when write_keys (else by launch_region_keys)
  int* vals;
  bool write_keys;
  double* dbg_stats;         // [cap,10] or null
  double* dbg_child;         // [cap,16] or null
  Counters* ctr;
  unsigned grid;
};
cudaError_t launch_child_init(const ChildArgs& a, cudaStream_t s);
// sort keys (candidate rank, view, band, first pixel) of imported region records
// zero up to 8 int32 arrays in one launch (instead of one memset node each)
struct ZeroList {
  int* p[8];
  long long n[8];   // elements
  int count;
};
cudaError_t launch_zero(const ZeroList& z, cudaStream_t s);

cudaError_t launch_region_keys(const RegionRec* regions, long long n, const int* cand_rank, int bits_v, int bits_b,
                               int bits_p, unsigned long long* keys, int* vals, cudaStream_t s);

// ---- per-candidate ranges after the sort ----
struct RangeArgs {
  const unsigned long long* keys_sorted;
  const int* vals_sorted;
  long long n;
  int shift_rank, bits_v, shift_view;
  const unsigned char* valid;
  int n_views;
  int* cand_start;
  int* cand_end;
  int* cand_nvalid;
  int* regions_per_view;
  unsigned grid;
};
cudaError_t launch_ranges(const RangeArgs& a, cudaStream_t s);

// ---- merge + cap + case: see merge.cuh ----

// ---- offsets: candidate inserts and survivor compaction (ref/adc.py:229-244) ----
struct OffsetArgs {
  long long n;
  const unsigned char* cls;
  const int* cand_rank;
  const int* cand_case;
  const int* cand_ins;
  int* ins_off;
  int* fb_ord;
  int* keep_pos;
  Counters* ctr;
  const unsigned long long* n_split_dev;
};
// the two offset scans separately (the survivor scan only needs the cases, so
// it can overlap the merge on a second stream)
cudaError_t launch_offsets_cand(const OffsetArgs& a, long long n_split, ScanState st_c, cudaStream_t s);
cudaError_t launch_offsets_keep(const OffsetArgs& a, ScanState st_g, cudaStream_t s);
cudaError_t launch_offsets(const OffsetArgs& a, long long n_split, ScanState st_c, ScanState st_g,
                           cudaStream_t s);

// ---- emit (ref/adc.py:198-244) ----
struct EmitArgs {
  GaussiansIn g;
  long long n, n_split, n_clone, n_keep, n_inserted;
  const int* keep_pos;
  const int* split_list;
  const int* clone_list;
  const int* cand_case;
  const int* cand_merged;
  const int* cand_start;
  const int* ins_off;
  const int* fb_ord;
  const float* children;
  const double* normals;
  double eta;
  int fb_children;          // children per fallback parent: 2 (ref/adc.py:219), n (vanilla_densify)
  float* mu;
  float* scale;
  float* rot;
  float* opacity;
  float* sh_dc;
  float* sh_rest;
  long long* index_map;
  int* child_parent;        // [n_out - n_keep] old index each appended row came from, or null
  long long* insert_offset; // [n_split] output row of candidate k's first insert, or null
  long long b_off;          // (launch internal) blocks writing the reset candidates' insert offsets
  // sync-free form (adps_step_phase1_end_emit): n_keep / n_inserted read on the
  // device, the grid sized from n_inserted <= n_ins_max, rows past the caller's
  // capacities dropped (never reached when the bounds hold)
  const unsigned long long* dev_keep = nullptr;
  const unsigned long long* dev_inserted = nullptr;
  long long n_ins_max = 0;
  long long out_cap = 0, app_cap = 0;
};
cudaError_t launch_emit(const EmitArgs& a, cudaStream_t s, cudaStream_t aux = nullptr, cudaEvent_t fork = nullptr,
                        cudaEvent_t join = nullptr);

cudaError_t launch_accumulate(double* ga, double* den, const float* vg, const unsigned char* vis,
                              long long n, cudaStream_t s);
cudaError_t launch_accumulate_f64(double* ga, double* den, const double* vg, const unsigned char* vis,
                                  long long n, cudaStream_t s);

// opacity prune (ref/harness.py:320-340): index_map[new] = old for the kept Gaussians
struct PruneArgs {
  const float* opacity;      // [n] fp32 opacity, or null (then logit is used)
  const double* logit;       // [n] fp64 logit_op
  long long n;
  double threshold;
  long long* index_map;      // [n] (first n_keep entries written)
  unsigned long long* n_keep;
  unsigned long long* n_near;
};
cudaError_t launch_prune(const PruneArgs& a, ScanState st, cudaStream_t s);

// vanilla_densify (ref/adc.py:248-280): every split candidate is split into n children
cudaError_t launch_vanilla_cases(int* cand_case, int* cand_ins, int* cand_merged, const unsigned long long* n_split,
                                 int n_children, cudaStream_t s);
// post-step remaps (ref/adc.py:283-296, ref/harness.py:285-295)
cudaError_t launch_reset_flags(unsigned char* flags, long long n, const int* split_list, const int* cand_case,
                               long long n_split, const int* clone_list, long long n_clone, bool clones,
                               cudaStream_t s);
cudaError_t launch_remap_rows(const long long* index_map, long long n_out, const unsigned char* zero_old,
                              const void* in, long long row_bytes, void* out, cudaStream_t s);

}  // namespace adps
