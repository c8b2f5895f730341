/*
 * adps.h -- C ABI of the B200-native AdpSplit densify operator.
 *
 * This is the drop-in boundary for the reference's split operator
 * (arXiv 2605.06876 reference package, /root/reference/pkg/src/adpsplit).
 * Every entry point names the reference function it replaces (file:line).
 * Signatures use plain C types only: device pointers, sizes, POD structs.
 * No allocation happens inside the hot calls; the plan owns all scratch.
 *
 * Threading: one plan per (device, stream); plans are independent and not
 * re-entrant.  All device pointers must be on the plan's device.  `stream`
 * is a cudaStream_t passed as void*.
 *
 * Status codes map onto the reference's exceptions in the Python shim:
 *   ADPS_INVALID_ARG    -> ValueError          (argument validation)
 *   ADPS_V_TOO_LARGE    -> ValueError          (ref/adc.py:154-157)
 *   ADPS_DEGENERATE_RAY -> DegenerateRayError  (ref/child_init.py:61-63)
 *   others              -> RuntimeError
 */
#ifndef ADPS_H_
#define ADPS_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ADPS_ABI_VERSION 3

#if defined(__GNUC__)
#define ADPS_API __attribute__((visibility("default")))
#else
#define ADPS_API
#endif

typedef enum {
  ADPS_OK = 0,
  ADPS_INVALID_ARG = 1,
  ADPS_V_TOO_LARGE = 2,
  ADPS_DEGENERATE_RAY = 3,
  ADPS_CUDA_ERROR = 4,
  ADPS_OOM = 5,
  ADPS_BAD_STATE = 6,
  ADPS_INTERNAL = 7   /* a bound the implementation relies on was violated */
} adps_status;

/* Per-candidate outcome (ref/adc.py:198-226 branch order). */
typedef enum { ADPS_CASE_SPLIT = 0, ADPS_CASE_FALLBACK = 1, ADPS_CASE_RESET = 2 } adps_case;

typedef struct adps_plan adps_plan;

/* Gaussians as structure-of-arrays fp32 device buffers (ref/scene.py:54-81).
 * rot is (w, x, y, z).  sh_rest is [n, sh_rest_k, 3] or NULL when k == 0. */
typedef struct {
  const float* mu;       /* [n,3] */
  const float* scale;    /* [n,3] */
  const float* rot;      /* [n,4] */
  const float* opacity;  /* [n]   */
  const float* sh_dc;    /* [n,3] */
  const float* sh_rest;  /* [n,k,3] or NULL */
  int32_t sh_rest_k;
} adps_gaussians;

typedef struct {
  float* mu;
  float* scale;
  float* rot;
  float* opacity;
  float* sh_dc;
  float* sh_rest;        /* [n_out,k,3] or NULL when k == 0 */
  int32_t sh_rest_k;
} adps_gaussians_out;

/* Mirrors AdpSplitConfig (ref/scene.py:147-180); t_interval is trainer-only. */
typedef struct {
  double tau_l1;
  int32_t r_erode;
  int32_t m_min;
  int32_t l_bands;
  int32_t n_max;
  int32_t v_views;
  int32_t reserved0;
  double gamma_d;
  double gamma_c;
  double tau_g;
  double tau_s;
  double eta;
  double eps;
} adps_config;

/* Host-visible results of phase 1 (one device->host copy). */
typedef struct {
  int64_t n_before;        /* N                                             */
  int64_t n_out;           /* population after the step      */
  int64_t n_keep;          /* survivors carried with their index           */
  int64_t n_split;         /* |split_set|  (ref/adc.py:165)                */
  int64_t n_clone;         /* |clone_set|                                  */
  int64_t n_fallback;      /* candidates never dominant -> vanilla split   */
  int64_t n_reset;         /* dominant but no usable proposal              */
  int64_t n_children;      /* sum N_i over split candidates                */
  int64_t n_inserted;      /* all appended Gaussians except clones         */
  int64_t n_regions;       /* error regions over all sampled views         */
  int64_t n_proposals;     /* regions with t* > 0                          */
  int64_t merge_edges;     /* ref/adc.py:210                               */
  int64_t n_partials;      /* tile-border component fragments (diagnostic) */
  int32_t degenerate_ray;  /* nonzero -> DegenerateRayError                */
  int32_t reserved1;
} adps_counts;

/* Report arrays owned by the plan; valid until the next phase 1.
 * All are device pointers. */
typedef struct {
  const int32_t* cand_index;        /* [n_split] ascending Gaussian index      */
  const int32_t* cand_case;         /* [n_split] adps_case                     */
  const int32_t* cand_proposals;    /* [n_split]                               */
  const int32_t* cand_merged;       /* [n_split] N_i (split case) else 0       */
  const int32_t* regions_per_view;  /* [n_split, n_views]                      */
  const int32_t* clone_index;       /* [n_clone] ascending                     */
  int32_t n_views;
} adps_report;

/* One error region (ref/error_partition.py:27-41) with its pixel set reduced
 * to exact integer moments; identical to the device record layout. */
typedef struct {
  int32_t view_pos;     /* position of the view in the sampled view ids     */
  int32_t candidate;    /* Gaussian index                                   */
  int32_t band;
  int32_t minpix;       /* y*W + x of the first row-major pixel             */
  int64_t moments[6];   /* n, Sx, Sy, Sxx, Sxy, Syy                          */
} adps_region_record;

ADPS_API int adps_abi_version(void);
ADPS_API const char* adps_last_error(void);

/* Plan: owns every scratch buffer sized for up to max_n Gaussians and
 * max_views views of height x width pixels.  Buffers grow on demand. */
ADPS_API adps_status adps_plan_create(adps_plan** plan, int32_t device, int64_t max_n,
                             int32_t max_views, int32_t height, int32_t width);
ADPS_API adps_status adps_plan_destroy(adps_plan* plan);
/* Debug: every plan buffer has a guard zone past its usable size, filled at
 * allocation; after a device sync, *bad_bytes = guard bytes some kernel
 * overwrote (0 = no out-of-bounds write past any plan buffer), *bad_buffers =
 * buffers affected (may be NULL). */
ADPS_API adps_status adps_check_guards(adps_plan* plan, int64_t* bad_bytes, int32_t* bad_buffers);

/* Attribution render of n_views cameras: image [V,H,W,3] fp32 and dominant
 * map [V,H,W] int32 (-1 where nothing contributes).
 * Replaces raster.render (ref/raster.py:136-157) incl. visible_splats/project
 * (ref/raster.py:61-117).  cams_host: V x 18 doubles in save_cameras order
 * (ref/scene.py:339-347).  bg: 3 floats (host). */
ADPS_API adps_status adps_render(adps_plan* plan, void* stream, const adps_gaussians* g, int64_t n,
                        const double* cams_host, int32_t n_views, const float* bg,
                        float* image, int32_t* dominant);

/* adps_render plus workload statistics (the benchmark's synthetic
 * DensifyStats and measured depth complexity, not part of the step):
 * weight [n] fp32 (device, accumulated into -- zero it first) += the sum of
 * the blending weights T*alpha of each Gaussian over all rendered pixels, and
 * *contributions (host) = the number of (pixel, splat) pairs with
 * alpha >= 1/255 over the views (mean depth complexity = contributions /
 * (n_views*H*W)).  Runs without the early termination. */
ADPS_API adps_status adps_render_stats(adps_plan* plan, void* stream, const adps_gaussians* g, int64_t n,
                              const double* cams_host, int32_t n_views, const float* bg,
                              float* image, int32_t* dominant, float* weight, uint64_t* contributions);

/* Fused attribution ("K1 epilogue"): select (ref/adc.py:165)
 * and the attribution render of the sampled views (as adps_render) whose
 * epilogue also computes, from each pixel's stored image value and gt, what
 * the step's input pass would: the raw L1 error (numpy's fp64 order) into the
 * plan's 16-bit raw cache, the per-view min/max, the candidate bits and the
 * ever-dominant flags (ref/adc.py:168-180).  The next
 * adps_step_phase1_begin with the same arguments (same g, stats, cfg, cameras,
 * image, gt and dominant pointers) then skips select and the input pass and
 * starts from that 6 B/px boundary (cache + dominant map); any other call
 * uses the full path.
 * gt: [V,H,W,3] fp32 of the same views. */
ADPS_API adps_status adps_render_fused(adps_plan* plan, void* stream, const adps_gaussians* g, int64_t n,
                              double extent, const double* grad_accum, const double* denom,
                              const adps_config* cfg, const double* cams_host, int32_t n_views,
                              const float* bg, const float* gt, float* image, int32_t* dominant);

/* Phase 1 of adpsplit_step (ref/adc.py:165-227): select, error maps,
 * partition, region statistics, ever-dominant, child initialisation,
 * cross-view merge and cap, per-candidate case, offsets.  Consumes the
 * attribution of the sampled views (image/dominant, e.g. from adps_render)
 * and gt for the same views.  Writes counts (host) after one sync.
 * cams_host: the n_views sampled cameras, in ascending view-id order. */
ADPS_API adps_status adps_step_phase1(adps_plan* plan, void* stream, const adps_gaussians* g, int64_t n,
                             double extent, const double* grad_accum, const double* denom,
                             const adps_config* cfg, const double* cams_host, int32_t n_views,
                             const float* image, const float* gt, const int32_t* dominant,
                             adps_counts* counts);

/* Split form of phase 1 for overlap: _begin runs select and the
 * ever-dominant flags (ref/adc.py:165, 177-180), synchronises once and
 * fills counts->n_split, n_clone and n_fallback, so the host can draw the
 * 6*n_fallback normals from its Generator while _end runs the rest of
 * phase 1 on the GPU.  Same arguments as adps_step_phase1, which is
 * exactly _begin followed by _end. */
ADPS_API adps_status adps_step_phase1_begin(adps_plan* plan, void* stream, const adps_gaussians* g, int64_t n,
                             double extent, const double* grad_accum, const double* denom,
                             const adps_config* cfg, const double* cams_host, int32_t n_views,
                             const float* image, const float* gt, const int32_t* dominant,
                             adps_counts* counts);
ADPS_API adps_status adps_step_phase1_end(adps_plan* plan, void* stream, adps_counts* counts);

/* Phase 2 (ref/adc.py:198-244): emit children, parent copies, fallback
 * children, clones and survivors into caller-allocated arrays of
 * counts.n_out rows plus index_map (old index or -1, ref/adc.py:233-244).
 * fallback_normals: device, 6*n_fallback doubles drawn by the host from the
 * caller's numpy Generator in ascending fallback order (ref/adc.py:97).
 * Optional integer outputs (NULL to skip):
 *   child_parent  [n_out - n_keep] int32: for every appended row (candidate
 *                 inserts in ascending candidate order, then clones) the old
 *                 index of the Gaussian it came from -- the candidate for its
 *                 children, parent copy and fallback children, the source for
 *                 a clone (the `inserted` list of ref/adc.py:184-231);
 *   insert_offset [n_split] int64: output row of candidate k's first inserted
 *                 Gaussian (= the criterion-6 cursor of
 *                 ref tests/test_acceptance.py:238-256; a reset candidate's
 *                 empty range starts there too). */
ADPS_API adps_status adps_step_phase2(adps_plan* plan, void* stream, const adps_gaussians* g,
                             const double* fallback_normals, adps_gaussians_out* out,
                             int64_t* index_map, int32_t* child_parent, int64_t* insert_offset);

/* Sync-free end of the step: phase 1 end and phase 2 in one call, with the
 * emit launched before the host reads any count (the counts arrive with the
 * call's single synchronisation).  Arguments as adps_step_phase2, into
 * arrays of out_cap rows (mu ... index_map) and app_cap rows (child_parent),
 * which must reach adps_step_capacity's bounds (available after
 * adps_step_phase1_begin); counts->n_out rows are written.  The fallback
 * normals must be on the device when the stream reaches the emit: drawn by
 * adps_normals_pcg64 (any sync mode) or uploaded before the call.
 * report (optional, NULL to skip): int32 [4*n_split + n_split*V + n_clone]
 * (the counts of phase1_begin), filled as adps_copy_report fills it. */
ADPS_API adps_status adps_step_capacity(adps_plan* plan, int64_t* out_cap, int64_t* app_cap);
ADPS_API adps_status adps_step_phase1_end_emit(adps_plan* plan, void* stream, const adps_gaussians* g,
                             const double* fallback_normals, adps_gaussians_out* out,
                             int64_t* index_map, int32_t* child_parent, int64_t* insert_offset,
                             int64_t out_cap, int64_t app_cap, int32_t* report, adps_counts* counts);

ADPS_API adps_status adps_get_report(adps_plan* plan, adps_report* report);

/* The report arrays of adps_get_report copied on `stream` into one device
 * int32 buffer `dst`, back to back: cand_index, cand_case, cand_proposals,
 * cand_merged [n_split each], regions_per_view [n_split * n_views],
 * clone_index [n_clone] (one call instead of six copies from the host). */
ADPS_API adps_status adps_copy_report(adps_plan* plan, void* stream, int32_t* dst, int64_t n_split, int64_t n_clone);

/* Stage-level parity access to the last phase 1 (device pointers):
 * records[n] in production order, order[n] = record index in
 * (candidate, view, band, first pixel) order (ref/adc.py:190-195),
 * valid[n] = t* > 0 (ref/child_init.py:115-116).  When debug records are
 * enabled, stats[n,10] = cx,cy,e1x,e1y,sigma1,sigma2,r,g,b,t* and
 * child[n,16] = mu3, rot9 (row-major), scale3, valid; else NULL. */
ADPS_API adps_status adps_get_regions(adps_plan* plan, const adps_region_record** records, const int32_t** order,
                             const uint8_t** valid, const double** stats, const double** child,
                             int64_t* n);
ADPS_API adps_status adps_set_debug_records(adps_plan* plan, int32_t enabled);

/* Optional diagnostic: when set, phase 1 also writes the eroded metric map
 * m and the band map b (uint8 [V,H,W]) -- ref/error_partition.py:86-91.
 * Pass NULLs to disable. */
ADPS_API adps_status adps_set_debug_maps(adps_plan* plan, uint8_t* m_out, uint8_t* b_out);

/* Phase timings of the last phase 1 / phase 2 in milliseconds (CUDA events
 * recorded on `stream`; filled only when timing was enabled). */
ADPS_API adps_status adps_set_timing(adps_plan* plan, int32_t enabled);
ADPS_API adps_status adps_get_timing(adps_plan* plan, double* ms, int32_t max_entries, int32_t* n_entries,
                            const char** names);

/* ---- multi-GPU sharding (one plan per rank) ----
 * Phase A is view-sharded: rank r passes its local views (every world-th
 * sampled view starting at r) to adps_step_phase1_begin after
 * adps_set_view_sharding(plan, r, world, V), so region records carry global
 * view positions.  Between the calls the host reduces the ever-dominant flags
 * (ADPS_BUF_DOM_FLAG, uint8 [n], MAX) over ranks and calls
 * adps_step_phase1_refresh for the global fallback count; then
 * adps_step_phase1_local builds this rank's region records and proposals
 * (ADPS_BUF_REGIONS / _PROPOSALS / _VALID), the host all-gathers them and
 * hands the concatenation back with adps_step_phase1_import, and
 * adps_step_phase1_merge finishes phase 1 exactly as adps_step_phase1_end
 * would have on one GPU (records are ordered by their sort key, so the
 * concatenation order does not matter).  adps_step_phase1_end ==
 * adps_step_phase1_local + adps_step_phase1_merge. */
#define ADPS_BUF_DOM_FLAG 1
#define ADPS_BUF_REGIONS 2
#define ADPS_BUF_PROPOSALS 3
#define ADPS_BUF_VALID 4
#define ADPS_BUF_CAND_MERGED 5   /* int32 [n_split]: children per split parent */
#define ADPS_BUF_CAND_INS 6      /* int32 [n_split]: inserted Gaussians per parent */
#define ADPS_BUF_CHILDREN 7      /* 14 floats per proposal slot: children of parent k at its proposal range */
#define ADPS_BUF_LO 8            /* double [V]: per-view min raw L1 error (diagnostic) */
#define ADPS_BUF_THRESHOLDS 9    /* double [V][L]: x thresholds of m and of each band (diagnostic) */
ADPS_API adps_status adps_set_view_sharding(adps_plan* plan, int32_t view_offset, int32_t view_stride,
                                            int32_t n_views_global);
ADPS_API adps_status adps_get_buffer(adps_plan* plan, int32_t which, void** ptr, int64_t* count, int64_t* elem_bytes);
ADPS_API adps_status adps_step_phase1_refresh(adps_plan* plan, void* stream, adps_counts* counts);
ADPS_API adps_status adps_step_phase1_local(adps_plan* plan, void* stream, int64_t* n_regions);
ADPS_API adps_status adps_step_phase1_import(adps_plan* plan, void* stream, const adps_region_record* regions,
                                             const void* proposals, const uint8_t* valid, int64_t n);
ADPS_API adps_status adps_step_phase1_merge(adps_plan* plan, void* stream, adps_counts* counts);
/* Parent sharding of phase B (merge, cap): with adps_set_parent_sharding(plan,
 * r, g) the merge gates, groups and caps only rank r's contiguous range of
 * split candidates (balanced by the sum of P_k^2 + 1, computed on the device
 * identically on every rank).  adps_step_phase1_merge then stops after the
 * cap (counts carries this rank's merge_edges / n_children); adps_get_shard
 * gives the range [k_lo, k_hi) and its proposal range [p_lo, p_hi); the host
 * all-gathers ADPS_BUF_CAND_MERGED / _CAND_INS [k_lo, k_hi) and
 * ADPS_BUF_CHILDREN [p_lo, p_hi) of every rank into every plan, and
 * adps_step_phase1_finish (with the summed merge_edges / n_children) runs the
 * offsets; phase 2 is then identical on every rank. */
ADPS_API adps_status adps_set_parent_sharding(adps_plan* plan, int32_t rank, int32_t world);
ADPS_API adps_status adps_get_shard(adps_plan* plan, int64_t* k_lo, int64_t* k_hi, int64_t* p_lo, int64_t* p_hi);
ADPS_API adps_status adps_step_phase1_finish(adps_plan* plan, void* stream, int64_t merge_edges, int64_t n_children,
                                             adps_counts* counts);

/* Tuning knobs (diagnostic/testing).  ADPS_PARAM_LARGE_THRESHOLD: parents
 * with more proposals than this use the grid-wide pair-tile merge path
 * (default 32; 0 routes every split parent through it).
 * ADPS_PARAM_TILE_PATH: 0 (default) warp-per-tile CCL on bit planes written by
 * a words pass over the 16-bit raw cache, with the block CCL for the tiles it
 * defers (> 192 runs) and for r_erode > 3 / debug maps; 1 the block CCL for
 * every tile; 2 the warp CCL thresholding the fp64 raw cache row by row; 3 as
 * 0 with the bit planes computed per tile inside the CCL kernel (no words
 * pass; slower at config 3).  All give identical results.
 * ADPS_PARAM_DEFERRED_TILES (read-only): tiles the last phase 1 deferred. */
#define ADPS_PARAM_LARGE_THRESHOLD 1
#define ADPS_PARAM_TILE_PATH 2
#define ADPS_PARAM_DEFERRED_TILES 3
#define ADPS_PARAM_NORMALS_CONSUMED 4   /* read-only, see adps_normals_pcg64 */
#define ADPS_PARAM_NORMALS_STATUS 5     /* read-only, see adps_normals_pcg64 */
#define ADPS_PARAM_STAT_TILE_PAIRS 7     /* read-only diagnostics of the last phase 1: surviving */
#define ADPS_PARAM_STAT_GATES 8          /* large-parent tile pairs; gates evaluated and passed */
#define ADPS_PARAM_STAT_GATES_PASSED 9   /* in them (the last two only in stats builds) */
#define ADPS_PARAM_RAW_CACHE 6          /* 1 (default): the input pass caches the raw L1 error
                                           (16 bits/px, exact compares, ambiguous pixels redone
                                           in fp64) for the CCL; 0: recompute */
#define ADPS_PARAM_PIPELINE_CHUNKS 10      /* view chunks of the attribution pipeline (input pass of chunk
                                              c+1 beside the CCL of chunk c; default 1) */
#define ADPS_PARAM_INPUT_BLOCKS_PER_SM 11  /* resident blocks per SM of the input pass (0 = all that fit) */
#define ADPS_PARAM_RENDER_BINNING 12       /* adps_render's depth order: 1 (default) a 32-bit key sort plus a
                                              fix-up of equal keys, no host sync between views; 0 the 64-bit
                                              sort of the fp64 depths, a sync per view (same images) */
#define ADPS_PARAM_RENDER_PAIR_CAP 13      /* (tile, splat) pairs the fast path's tile sort covers (learned
                                              at the plan's first render; grown when a view exceeds it) */
#define ADPS_PARAM_CAP_HUGE 14             /* parents with more merged groups than this (default 4096, at
                                              least 64) take the cap's selection by a thread-block cluster
                                              (distributed shared memory); same results */
ADPS_API adps_status adps_set_param(adps_plan* plan, int32_t key, int64_t value);
ADPS_API adps_status adps_get_param(adps_plan* plan, int32_t key, int64_t* value);

/* Cumulative number of kernels this plan launched (own kernels) and of
 * library sort calls (CUB radix sort) -- used by the benchmark's
 * gpu_launches accounting. */
ADPS_API adps_status adps_get_launch_count(adps_plan* plan, int64_t* kernels, int64_t* library_calls);

/* numpy.random.Generator(PCG64).standard_normal(n), bit-identical, on the
 * device.  Replaces the host draw of the fallback children's normals
 * (ref/adc.py:97 -> rng.normal(size=(k, 3)) per fallback parent, which is
 * one contiguous slice of the Generator's normal stream).  state/inc: the
 * bit generator's 128-bit state and increment as (low, high) 64-bit words
 * (bit_generator.state["state"]).  Writes n doubles to `out` (device) on
 * `stream`.  *consumed = 64-bit draws used (advance the host generator by
 * it); *status = 0 exact, bit0 a wedge comparison within a few ulp of the
 * host libm's exp (redraw on the host), bit1 internal window too short.
 * With sync == 0 nothing is waited for: consumed/status are read with
 * adps_get_param(ADPS_PARAM_NORMALS_*) after the plan's next phase-1 end
 * (call it between adps_step_phase1_begin and adps_step_phase1_end).
 * sync == 2: as 0, but the kernels are only launched by the next
 * adps_step_phase1_end at its first host wait, so their host-side launch
 * cost overlaps GPU work instead of leaving the GPU idle. */
ADPS_API adps_status adps_normals_pcg64(adps_plan* plan, void* stream, const uint64_t state[2], const uint64_t inc[2],
                                        int64_t n, double* out, int32_t sync, int64_t* consumed, int32_t* status);

/* ---- the next rows of the path ----
 * vanilla_densify (ref/adc.py:248-280): select, then every split candidate is
 * replaced by n_children vanilla_split children (3 normals each from the
 * caller's Generator, ascending parent order -> 3*n_children*n_split normals,
 * e.g. adps_normals_pcg64), clones appended; adps_step_phase2 writes the
 * grown arrays.  Same plan/report machinery as adpsplit. */
ADPS_API adps_status adps_vanilla_phase1(adps_plan* plan, void* stream, const adps_gaussians* g, int64_t n,
                                         double extent, const double* grad_accum, const double* denom,
                                         const adps_config* cfg, int32_t n_children, adps_counts* counts);
/* Post-step state remap.  adps_reset_flags: flags[old] = 1 for the last
 * step's reset candidates (and, with include_clones, clone sources) -- the
 * `reset` set of remap_stats (ref/adc.py:283-296, with clones) and of the
 * trainer's optimizer-moment remap (ref/harness.py:285-295, without).
 * adps_remap_rows: out[new] = in[index_map[new]] (rows of row_bytes, a
 * multiple of 4) when index_map[new] >= 0 and not zero_old[index_map[new]]
 * (zero_old may be NULL), else zeros. */
ADPS_API adps_status adps_reset_flags(adps_plan* plan, void* stream, uint8_t* flags, int32_t include_clones);
ADPS_API adps_status adps_remap_rows(void* stream, const int64_t* index_map, int64_t n_out, const uint8_t* zero_old,
                                     const void* in, int64_t row_bytes, void* out);

/* DensifyStats feed (ref/adc.py:73-79): grad_accum[vis] += |vg|, denom[vis] += 1.
 * viewspace_grad [n,2] fp32, visible [n] uint8. */
ADPS_API adps_status adps_accumulate_stats(void* stream, double* grad_accum, double* denom,
                                  const float* viewspace_grad, const uint8_t* visible, int64_t n);
/* Same with the reference's fp64 gradients (GradOutput.viewspace_grad is
 * float64, ref/raster.py:49-58): bit-identical to numpy's norm + add. */
ADPS_API adps_status adps_accumulate_stats_f64(void* stream, double* grad_accum, double* denom,
                                      const double* viewspace_grad, const uint8_t* visible, int64_t n);

/* Opacity prune (ref/harness.py:320-340, _prune): keep = opacity >= threshold,
 * evaluated on the fp32 opacity (exact compare) or, when opacity is NULL, on
 * the fp64 logit as 1/(1+exp(-x)) (ref/harness.py:217-218).  Writes
 * index_map[new] = old for the n_keep survivors in old order (device, n
 * entries reserved) and synchronises once for *n_keep (host).  *n_near
 * (host, may be NULL) counts logits whose sigmoid lies within 4 ulp of the
 * threshold, where the device exp and the host libm may decide differently.
 * The reference keeps everything when n_keep is 0 or n (the caller checks);
 * the survivors' rows (parameters, optimizer moments, DensifyStats) are then
 * gathered with adps_remap_rows. */
ADPS_API adps_status adps_prune_index(adps_plan* plan, void* stream, const float* opacity, const double* logit_op,
                                      int64_t n, double threshold, int64_t* index_map, int64_t* n_keep,
                                      int64_t* n_near);

#ifdef __cplusplus
}
#endif

#endif /* ADPS_H_ */
