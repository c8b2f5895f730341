#include <algorithm>
// C-ABI implementation: the plan (owner of all scratch) and the phase
// orchestration of adpsplit_step (ref/adc.py:143-245) on one stream.
#include <cub/cub.cuh>
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <string>
#include <vector>

#include "adps_internal.cuh"
#include "attribution.cuh"
#include "merge.cuh"
#include "normals.cuh"

#ifndef ADPS_PIPELINE_DEFAULT
#define ADPS_PIPELINE_DEFAULT 1
#endif
#ifndef ADPS_PIPELINE_CHUNKS
#define ADPS_PIPELINE_CHUNKS 1
#endif
#ifndef ADPS_AUX_PRIORITY
#define ADPS_AUX_PRIORITY 0
#endif
#ifndef ADPS_RAW_CACHE_DEFAULT
#define ADPS_RAW_CACHE_DEFAULT 1
#endif
#include "render.cuh"
#include "split.cuh"

using namespace adps;

static thread_local std::string g_last_error;

static adps_status fail(adps_status st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return st;
}

#define CK(call)                                                                             \
  do {                                                                                       \
    cudaError_t e_ = (call);                                                                 \
    if (e_ != cudaSuccess) {                                                                 \
      return fail(e_ == cudaErrorMemoryAllocation ? ADPS_OOM : ADPS_CUDA_ERROR, "%s: %s (%s:%d)", \
                  #call, cudaGetErrorString(e_), __FILE__, __LINE__);                        \
    }                                                                                        \
  } while (0)

namespace {

struct Buf {
  void* p = nullptr;
  size_t bytes = 0;
  template <class T>
  T* as() const {
    return reinterpret_cast<T*>(p);
  }
};

// Every plan buffer carries a guard zone of kGuard bytes past its usable size,
// filled with kGuardByte at allocation: adps_check_guards reports any byte a
// kernel wrote past the end of a buffer (a bounds check of our own; the pool's
// compute-sanitizer is unavailable).
constexpr size_t kGuard = 256;
constexpr unsigned char kGuardByte = 0xA5;

cudaError_t ensure(Buf& b, size_t bytes) {
  if (bytes == 0) bytes = 16;
  if (b.bytes >= bytes) return cudaSuccess;
  if (b.p) cudaFree(b.p);
  b.p = nullptr;
  b.bytes = 0;
  size_t want = (bytes + bytes / 8 + 255) & ~(size_t)255;   // headroom against small growth
  cudaError_t e = cudaMalloc(&b.p, want + kGuard);
  if (e != cudaSuccess) return e;
  e = cudaMemset((char*)b.p + want, kGuardByte, kGuard);
  if (e != cudaSuccess) return e;
  b.bytes = want;
  return cudaSuccess;
}

constexpr int kMaxMarks = 32;

}  // namespace

struct adps_plan {
  int device = 0;
  int sm_count = 148;
  // per-Gaussian
  Buf cls, cand_rank, split_list, clone_list, dom_flag, keep_pos;
  // per-candidate
  Buf cand_start, cand_end, cand_nvalid, cand_case, cand_props, cand_merged, cand_ins, ins_off, fb_ord,
      large_list, regions_per_view;
  // per-view
  Buf lohi, lo, thr, thr_raw, cams;
  // tiles / fragments / regions
  Buf border, partials, partial_parent, regions, props, valid, keys, vals, keys_sorted, vals_sorted;
  Buf idx, uf, groups, children, dbg_stats, dbg_child, deferred, cand_bits, rawc, twords;
  // device normals (numpy PCG64 stream)
  Buf nrm_val, nrm_len, nrm_acc, nrm_reach, nrm_rmax, nrm_walked, nrm_idx, nrm_tmp;
  // merge / cap scratch (proposal space)
  Buf small_list, pstart, n_groups, work_cnt, work_off, props_s, psrc, pcand, gkey, gval, gkey_sorted, gval_sorted,
      grp_first, gpar, gext, gfirst_of, glist, scan3_val, scan3_flag, large_of, lp_cnt, lp_off, tile_cnt, tile_off, mkey,
      mval, mkey_sorted, mval_sorted, boxes, tile_owner, tile_pairs, gsoa, fsoa;
  Buf scan_val, scan_flag, scan2_val, scan2_flag, cub_tmp;
  unsigned scan_epoch = 0;   // scan launches so far (tile-flag epochs, scan.cuh)
  Buf ctr;
  Counters* ctr_host = nullptr;
  unsigned long long* lohi_host = nullptr;
  double* cams_host = nullptr;
  int cams_host_cap = 0;
  long long region_cap = 0, partial_cap = 0, region_hint = 0, partial_hint = 0;
  // render scratch
  Buf r_key, r_key_sorted, r_order_in, r_order, r_tiles, r_rect, r_splat, r_offs, r_dup, r_dup_sorted,
      r_tstart, r_tend, r_total, r_cams, r_tile_lohi, r_k32, r_k32_sorted, r_vflag, r_vtotal, r_cov3, r_rgb0;
  int render_fast = 1;               // ADPS_PARAM_RENDER_BINNING: 1 = 32-bit depth keys, no per-view sync
  long long dup_cap = 0;             // (tile, splat) pairs the tile sort covers (0: learn at the next render)
  std::vector<int> vflag_host;
  std::vector<unsigned long long> vtotal_host;
  unsigned long long* r_total_host = nullptr;
  // last phase-1 state
  bool have_phase1 = false;
  long long n = 0;
  int V = 0, H = 0, W = 0;
  adps_counts counts{};
  double eta = 1.6;
  int sh_k = 0;
  // diagnostics
  unsigned char* dbg_m = nullptr;
  unsigned char* dbg_b = nullptr;
  bool dbg_records = false;
  bool timing = false;
  // timing marks: ev[0] is the start of a phase, ev[i] ends stage names[i]
  cudaEvent_t ev[kMaxMarks] = {};
  const char* names[kMaxMarks] = {};
  int n_marks = 0;
  // launch accounting (own kernels / library sort calls), cumulative
  long long launches = 0;
  long long lib_calls = 0;
  int large_threshold = 32;
  int cap_huge = kSelHuge;   // ADPS_PARAM_CAP_HUGE
  // second stream: small-parent gates and the survivor scan overlap the merge
  cudaStream_t aux = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_small = nullptr, ev_keep = nullptr, ev_nfork = nullptr, ev_norm = nullptr;
  bool keep_pending = false;
  bool norm_pending = false;   // fallback normals running on their own stream
  bool norm_deferred = false;  // requested (sync == 2), launched at phase 1's first host wait
  NormalsArgs nrm_args{};
  cudaStream_t nstream = nullptr;   // the fallback normals' stream
  // attribution pipelined with the input pass: the warp CCL of view chunk c runs
  // on the second stream while the minmax pass reads chunk c+1
  static constexpr int kMaxChunks = 16;
  cudaEvent_t ev_chunk[kMaxChunks] = {};
  cudaEvent_t ev_attr = nullptr;
  cudaEvent_t ev_cfork = nullptr, ev_child = nullptr;   // child init on the second stream
  cudaEvent_t ev_cams = nullptr;                          // the cameras' host copy (second stream)
  bool cams_pending = false;
  bool child_pending = false;
  bool attr_pending = false;
  int pipeline = ADPS_PIPELINE_DEFAULT;
  int pipeline_chunks = ADPS_PIPELINE_CHUNKS;   // view chunks of the attribution pipeline
  int input_blocks_per_sm = 0;                  // input pass residency (0: all that fit)
  int fb_children = 2;   // children per fallback parent of the last phase 1
  // view sharding: this plan's local view v is global view position view_offset + v * view_stride
  // of v_global_cfg sampled views (0 = the local views are all of them)
  int view_offset = 0, view_stride = 1, v_global_cfg = 0, v_glob = 0;
  long long n_regions_cur = 0;   // region records the merge half consumes
  // parent sharding of the merge: this rank gates/groups/caps only its range of candidates
  int pshard_rank = 0, pshard_world = 1;
  bool have_merge_part = false;
  long long shard_k[2] = {0, 0}, shard_p[2] = {0, 0};   // this rank's candidate / proposal range
  bool have_local = false;
  int tile_path = 0;   // 0 warp CCL (bit planes when l_bands <= 4) + deferred block CCL, 1 block CCL only,
                       // 2 warp CCL on the raw cache without bit planes
  bool use_bits = false;    // bit-plane warp CCL from the fp32 raw cache (tile paths 0 and 3)
  bool use_words = false;   // ... with the separate words pass (tile path 3)
  int raw_cache = ADPS_RAW_CACHE_DEFAULT;   // minmax pass caches the raw L1 error for the warp CCL
  bool use_raw = false;                     // decided per phase 1
  // the attribution a fused render (adps_render_fused) left for the next
  // phase1_begin on the same inputs: select classes/lists, raw cache, per-view
  // min/max, candidate bits, ever-dominant flags
  struct {
    bool valid = false;
    adps_gaussians g;
    long long n;
    double extent;
    const double *ga, *den;
    adps_config cfg;
    int V, H, W;
    const float *image, *gt;
    const int32_t* dom;
    std::vector<double> cams;
  } fused;
  // arguments saved by phase1_begin for phase1_end
  bool have_begin = false;
  struct {
    adps_gaussians g;
    long long n;
    double extent;
    adps_config cfg;
    int V, H, W;
    const float* image;
    const float* gt;
    const int32_t* dominant;
  } cx{};
};

static void mark(adps_plan* P, const char* name, cudaStream_t s, int kernels) {
  P->launches += kernels;
  if (!P->timing || P->n_marks >= kMaxMarks) return;
  cudaEventRecord(P->ev[P->n_marks], s);
  P->names[P->n_marks] = name;
  ++P->n_marks;
}

static void mark_cb(void* ctx, const char* name, cudaStream_t s, int kernels) {
  mark(reinterpret_cast<adps_plan*>(ctx), name, s, kernels);
}

static void mark_start(adps_plan* P, cudaStream_t s, bool reset) {
  if (reset) P->n_marks = 0;
  mark(P, "start", s, 0);
}

#ifndef ADPS_SELECT_FOLD
#define ADPS_SELECT_FOLD 1   // the classify pass zeroes the flags and seeds the min/max slots
#endif

// stable CUB radix sort of (key, value) pairs over [0, end_bit), temp storage owned by the plan
template <class K, class V>
static cudaError_t cub_sort_pairs(adps_plan* P, const K* kin, K* kout, const V* vin, V* vout, long long n,
                                  int end_bit, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  size_t tb = 0;
  cudaError_t e = cub::DeviceRadixSort::SortPairs(nullptr, tb, kin, kout, vin, vout, (int)n, 0, end_bit, s);
  if (e != cudaSuccess) return e;
  e = ensure(P->cub_tmp, tb);
  if (e != cudaSuccess) return e;
  tb = P->cub_tmp.bytes;
  P->lib_calls += 1;
  return cub::DeviceRadixSort::SortPairs(P->cub_tmp.p, tb, kin, kout, vin, vout, (int)n, 0, end_bit, s);
}

static adps_status scan_state(adps_plan* P, Buf& val, Buf& flag, long long n, ScanState* st) {
  long long tiles = scan_tiles(n);
  CK(ensure(val, 2 * sizeof(unsigned long long) * tiles));
  const void* old = flag.p;
  CK(ensure(flag, sizeof(unsigned int) * tiles));
  if (flag.p != old) {   // epoch 0 = empty; once per allocation, finished before any stream uses it
    CK(cudaMemset(flag.p, 0, flag.bytes));
    CK(cudaDeviceSynchronize());
  }
  st->value = val.as<unsigned long long>();
  st->flag = flag.as<unsigned int>();
  st->epoch_host = &P->scan_epoch;
  st->epoch = 0;
  return ADPS_OK;
}

extern "C" int adps_abi_version(void) { return ADPS_ABI_VERSION; }

extern "C" const char* adps_last_error(void) { return g_last_error.c_str(); }

extern "C" adps_status adps_plan_create(adps_plan** plan, int32_t device, int64_t max_n, int32_t max_views,
                                        int32_t height, int32_t width) {
  if (!plan) return fail(ADPS_INVALID_ARG, "plan pointer is NULL");
  if (max_n < 0 || max_views < 0 || height < 0 || width < 0) return fail(ADPS_INVALID_ARG, "negative plan size");
  int ndev = 0;
  CK(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) return fail(ADPS_INVALID_ARG, "device %d not present (%d devices)", device, ndev);
  CK(cudaSetDevice(device));
  adps_plan* P = new adps_plan();
  P->device = device;
  cudaDeviceGetAttribute(&P->sm_count, cudaDevAttrMultiProcessorCount, device);
  cudaError_t e = cudaMallocHost(&P->ctr_host, sizeof(Counters));
  if (e == cudaSuccess) e = cudaMallocHost(&P->r_total_host, sizeof(unsigned long long));
  if (e != cudaSuccess) {
    delete P;
    return fail(ADPS_OOM, "pinned allocation failed: %s", cudaGetErrorString(e));
  }
  for (int i = 0; i < kMaxMarks; ++i) cudaEventCreate(&P->ev[i]);
  {
    // ADPS_AUX_PRIORITY: the second stream's blocks (CCL of finished chunks, small
    // gates) are dispatched ahead of the HBM-bound input pass's queued blocks
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    cudaStreamCreateWithPriority(&P->aux, cudaStreamNonBlocking, ADPS_AUX_PRIORITY ? hi : 0);
    cudaStreamCreateWithFlags(&P->nstream, cudaStreamNonBlocking);
  }
  cudaEventCreateWithFlags(&P->ev_fork, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&P->ev_small, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&P->ev_keep, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&P->ev_cfork, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&P->ev_cams, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&P->ev_child, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&P->ev_nfork, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&P->ev_norm, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&P->ev_attr, cudaEventDisableTiming);
  for (int i = 0; i < adps_plan::kMaxChunks; ++i) cudaEventCreateWithFlags(&P->ev_chunk[i], cudaEventDisableTiming);
  (void)max_n;
  (void)max_views;
  (void)height;
  (void)width;
  *plan = P;
  return ADPS_OK;
}

constexpr int kMaxBufs = 160;
static int plan_buffers(adps_plan* P, Buf** out) {
  Buf* bufs[] = {&P->cls, &P->cand_rank, &P->split_list, &P->clone_list, &P->dom_flag, &P->keep_pos,
                 &P->cand_start, &P->cand_end, &P->cand_nvalid, &P->cand_case, &P->cand_props,
                 &P->cand_merged, &P->cand_ins, &P->ins_off, &P->fb_ord, &P->large_list,
                 &P->regions_per_view, &P->lohi, &P->lo, &P->thr, &P->thr_raw, &P->cams, &P->border, &P->partials,
                 &P->partial_parent, &P->regions, &P->props, &P->valid, &P->keys, &P->vals,
                 &P->keys_sorted, &P->vals_sorted, &P->idx, &P->uf, &P->groups, &P->children,
                 &P->dbg_stats, &P->dbg_child, &P->scan_val, &P->scan_flag,
                 &P->scan2_val, &P->scan2_flag, &P->cub_tmp, &P->ctr, &P->r_key,
                 &P->r_key_sorted, &P->r_order_in, &P->r_order, &P->r_tiles, &P->r_rect, &P->r_splat,
                 &P->r_offs, &P->r_dup, &P->r_dup_sorted, &P->r_tstart, &P->r_tend, &P->r_total, &P->r_tile_lohi,
                 &P->r_k32, &P->r_k32_sorted, &P->r_vflag, &P->r_vtotal, &P->r_cov3, &P->r_rgb0,
                 &P->r_cams, &P->small_list, &P->pstart, &P->n_groups, &P->work_cnt, &P->work_off,
                 &P->props_s, &P->psrc, &P->pcand, &P->gkey, &P->gval, &P->gkey_sorted, &P->gval_sorted, &P->grp_first,
                 &P->gpar, &P->gext, &P->gfirst_of, &P->glist, &P->scan3_val, &P->scan3_flag,
                 &P->large_of, &P->lp_cnt, &P->lp_off, &P->tile_cnt, &P->tile_off, &P->mkey, &P->mval,
                 &P->mkey_sorted, &P->mval_sorted, &P->boxes, &P->tile_owner, &P->tile_pairs, &P->gsoa, &P->fsoa, &P->deferred, &P->cand_bits, &P->rawc, &P->twords,
                 &P->nrm_val, &P->nrm_len, &P->nrm_acc, &P->nrm_reach, &P->nrm_rmax, &P->nrm_walked,
                 &P->nrm_idx, &P->nrm_tmp};
  int n = 0;
  for (Buf* b : bufs) out[n++] = b;
  return n;
}

extern "C" adps_status adps_check_guards(adps_plan* P, int64_t* bad_bytes, int32_t* bad_buffers) {
  if (!P || !bad_bytes) return fail(ADPS_INVALID_ARG, "NULL argument");
  CK(cudaSetDevice(P->device));
  CK(cudaDeviceSynchronize());
  Buf* bufs[kMaxBufs];
  const int nb = plan_buffers(P, bufs);
  long long bad = 0;
  int nbad = 0;
  unsigned char h[kGuard];
  for (int i = 0; i < nb; ++i) {
    if (!bufs[i]->p) continue;
    CK(cudaMemcpy(h, (char*)bufs[i]->p + bufs[i]->bytes, kGuard, cudaMemcpyDeviceToHost));
    int here = 0;
    for (size_t k = 0; k < kGuard; ++k) here += h[k] != kGuardByte;
    bad += here;
    nbad += here > 0;
  }
  *bad_bytes = bad;
  if (bad_buffers) *bad_buffers = nbad;
  return ADPS_OK;
}

extern "C" adps_status adps_plan_destroy(adps_plan* P) {
  if (!P) return ADPS_OK;
  cudaSetDevice(P->device);
  cudaDeviceSynchronize();
  Buf* bufs[kMaxBufs];
  const int nb = plan_buffers(P, bufs);
  for (int i = 0; i < nb; ++i)
    if (bufs[i]->p) cudaFree(bufs[i]->p);
  if (P->ctr_host) cudaFreeHost(P->ctr_host);
  if (P->lohi_host) cudaFreeHost(P->lohi_host);
  if (P->cams_host) cudaFreeHost(P->cams_host);
  if (P->r_total_host) cudaFreeHost(P->r_total_host);
  for (int i = 0; i < kMaxMarks; ++i)
    if (P->ev[i]) cudaEventDestroy(P->ev[i]);
  if (P->ev_fork) cudaEventDestroy(P->ev_fork);
  if (P->ev_small) cudaEventDestroy(P->ev_small);
  if (P->ev_keep) cudaEventDestroy(P->ev_keep);
  if (P->ev_cfork) cudaEventDestroy(P->ev_cfork);
  if (P->ev_cams) cudaEventDestroy(P->ev_cams);
  if (P->ev_child) cudaEventDestroy(P->ev_child);
  if (P->ev_nfork) cudaEventDestroy(P->ev_nfork);
  if (P->ev_norm) cudaEventDestroy(P->ev_norm);
  if (P->ev_attr) cudaEventDestroy(P->ev_attr);
  for (int i = 0; i < adps_plan::kMaxChunks; ++i)
    if (P->ev_chunk[i]) cudaEventDestroy(P->ev_chunk[i]);
  if (P->aux) cudaStreamDestroy(P->aux);
  if (P->nstream) cudaStreamDestroy(P->nstream);
  delete P;
  return ADPS_OK;
}

constexpr long long kMaxGaussians = 1ll << 29;

// forget a deferred normals request (and join a running one) that no phase 1
// will consume: a stale request would later write through a dangling pointer
static void drop_pending_normals(adps_plan* P) {
  P->norm_deferred = false;
  if (P->norm_pending) {
    cudaEventSynchronize(P->ev_norm);
    P->norm_pending = false;
  }
}


static adps_status check_gaussians(const adps_gaussians* g, int64_t n) {
  if (!g) return fail(ADPS_INVALID_ARG, "gaussians is NULL");
  if (n > 0 && (!g->mu || !g->scale || !g->rot || !g->opacity || !g->sh_dc))
    return fail(ADPS_INVALID_ARG, "gaussian arrays must be non-NULL");
  if (g->sh_rest_k < 0 || g->sh_rest_k > 15) return fail(ADPS_INVALID_ARG, "sh_rest_k must be in [0,15]");
  if (g->sh_rest_k > 0 && !g->sh_rest) return fail(ADPS_INVALID_ARG, "sh_rest is NULL with sh_rest_k > 0");
  // the tile CCL keys pixels by (candidate << 2 | band) in 32 bits and the survivor copy
  // indexes components in 32 bits: both hold for n < 2^29
  if (n >= kMaxGaussians) return fail(ADPS_INVALID_ARG, "n=%lld exceeds the supported 2^29 Gaussians", (long long)n);
  return ADPS_OK;
}

static GaussiansIn to_in(const adps_gaussians* g) {
  GaussiansIn r;
  r.mu = g->mu;
  r.scale = g->scale;
  r.rot = g->rot;
  r.opacity = g->opacity;
  r.sh_dc = g->sh_dc;
  r.sh_rest = g->sh_rest;
  r.sh_k = g->sh_rest_k;
  return r;
}

// ------------------------------------------------------------------ render
static adps_status render_impl(adps_plan* P, void* stream_v, const adps_gaussians* g, int64_t n,
                               const double* cams_host, int32_t n_views, const float* bg, float* image,
                               int32_t* dominant, float* weight, unsigned long long* contrib_dev,
                               const float* epi_gt = nullptr);

extern "C" adps_status adps_render(adps_plan* P, void* stream_v, const adps_gaussians* g, int64_t n,
                                   const double* cams_host, int32_t n_views, const float* bg, float* image,
                                   int32_t* dominant) {
  return render_impl(P, stream_v, g, n, cams_host, n_views, bg, image, dominant, nullptr, nullptr);
}

extern "C" adps_status adps_render_stats(adps_plan* P, void* stream_v, const adps_gaussians* g, int64_t n,
                                         const double* cams_host, int32_t n_views, const float* bg, float* image,
                                         int32_t* dominant, float* weight, uint64_t* contributions) {
  if (!P) return fail(ADPS_INVALID_ARG, "plan is NULL");
  if (n > 0 && !weight) return fail(ADPS_INVALID_ARG, "weight is NULL");
  CK(cudaSetDevice(P->device));
  cudaStream_t s = (cudaStream_t)stream_v;
  CK(ensure(P->r_total, 2 * sizeof(unsigned long long)));
  unsigned long long* cdev = P->r_total.as<unsigned long long>() + 1;
  CK(cudaMemsetAsync(cdev, 0, sizeof(unsigned long long), s));
  adps_status st = render_impl(P, stream_v, g, n, cams_host, n_views, bg, image, dominant, weight, cdev);
  if (st != ADPS_OK) return st;
  CK(cudaMemcpyAsync(P->r_total_host, cdev, sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  if (contributions) *contributions = (uint64_t)*P->r_total_host;
  return ADPS_OK;
}

static adps_status render_impl(adps_plan* P, void* stream_v, const adps_gaussians* g, int64_t n,
                               const double* cams_host, int32_t n_views, const float* bg, float* image,
                               int32_t* dominant, float* weight, unsigned long long* contrib_dev,
                               const float* epi_gt) {
  if (!P) return fail(ADPS_INVALID_ARG, "plan is NULL");
  adps_status st = check_gaussians(g, n);
  if (st != ADPS_OK) return st;
  if (n_views < 0 || (n_views > 0 && (!cams_host || !image || !dominant)))
    return fail(ADPS_INVALID_ARG, "bad render arguments");
  CK(cudaSetDevice(P->device));
  cudaStream_t s = (cudaStream_t)stream_v;
  const float bgv[3] = {bg ? bg[0] : 0.f, bg ? bg[1] : 0.f, bg ? bg[2] : 0.f};
  if (n_views == 0) return ADPS_OK;
  const CamD c0 = load_cam(cams_host);
  const int W = c0.w, H = c0.h;
  for (int v = 1; v < n_views; ++v) {
    const CamD cv = load_cam(cams_host + 18ll * v);
    if (cv.w != W || cv.h != H) return fail(ADPS_INVALID_ARG, "all views of one call must share H x W");
  }
  if (W <= 0 || H <= 0) return fail(ADPS_INVALID_ARG, "empty image");
  const int tiles_x = (W + kRTile - 1) / kRTile, tiles_y = (H + kRTile - 1) / kRTile;
  const int n_tiles = tiles_x * tiles_y;
  const long long hw = (long long)H * W;
  if (n == 0) {
    // nothing contributes: image = bg, dominant = -1
    std::vector<float> img((size_t)hw * 3);
    for (long long p = 0; p < hw; ++p)
      for (int c = 0; c < 3; ++c) img[3 * p + c] = bgv[c];
    for (int v = 0; v < n_views; ++v) {
      CK(cudaMemcpyAsync(image + (long long)v * hw * 3, img.data(), sizeof(float) * hw * 3, cudaMemcpyHostToDevice, s));
      CK(cudaMemsetAsync(dominant + (long long)v * hw, 0xff, sizeof(int) * hw, s));
    }
    CK(cudaStreamSynchronize(s));
    return ADPS_OK;
  }
  if (W > 32767 || H > 32767) return fail(ADPS_INVALID_ARG, "image side above 32767");
  CK(ensure(P->r_key, sizeof(unsigned long long) * n));
  CK(ensure(P->r_order_in, sizeof(int) * n));
  CK(ensure(P->r_order, sizeof(int) * n));
  CK(ensure(P->r_tiles, sizeof(unsigned) * n));
  CK(ensure(P->r_rect, sizeof(unsigned short) * 4 * n));
  CK(ensure(P->r_splat, sizeof(SplatData) * n));
  CK(ensure(P->r_offs, sizeof(unsigned) * n));
  CK(ensure(P->r_tstart, sizeof(int) * n_tiles));
  CK(ensure(P->r_tend, sizeof(int) * n_tiles));
  CK(ensure(P->r_total, 2 * sizeof(unsigned long long)));
  CK(ensure(P->r_vflag, sizeof(int) * (n_views + 1)));
  CK(ensure(P->r_vtotal, sizeof(unsigned long long) * (n_views + 1)));
  // tile ids below 2^tile_bits - 1: the padding keys (all ones) sort after every real key
  const int tile_bits = ceil_log2((unsigned long long)n_tiles + 1);
  ScanState sst;
  st = scan_state(P, P->scan_val, P->scan_flag, n, &sst);
  if (st != ADPS_OK) return st;
  // the view-independent covariances (and degree-0 colours), once per call
  CK(ensure(P->r_cov3, sizeof(double) * 6 * n));
  if (g->sh_rest_k == 0) CK(ensure(P->r_rgb0, sizeof(float) * 3 * n));
  {
    PreArgs pa{};
    pa.rot = g->rot;
    pa.scale = g->scale;
    pa.sh_dc = g->sh_dc;
    pa.n = n;
    CK(launch_splat3d(pa, P->r_cov3.as<double>(), g->sh_rest_k == 0 ? P->r_rgb0.as<float>() : nullptr, s));
    P->launches += 1;
  }
  auto preprocess = [&](int v, bool k32) -> adps_status {
    PreArgs pa;
    pa.mu = g->mu;
    pa.scale = g->scale;
    pa.rot = g->rot;
    pa.opacity = g->opacity;
    pa.sh_dc = g->sh_dc;
    pa.sh_rest = g->sh_rest;
    pa.sh_k = g->sh_rest_k;
    pa.n = n;
    pa.cam = load_cam(cams_host + 18ll * v);
    pa.W = W;
    pa.H = H;
    pa.depth_key = P->r_key.as<unsigned long long>();
    pa.order_in = P->r_order_in.as<int>();
    pa.tiles = P->r_tiles.as<unsigned>();
    pa.rect = P->r_rect.as<unsigned short>();
    pa.splat = P->r_splat.as<SplatData>();
    pa.depth32 = k32 ? P->r_k32.as<unsigned>() : nullptr;
    pa.tiles_x = tiles_x;
    pa.cov3 = P->r_cov3.as<double>();
    pa.rgb0 = g->sh_rest_k == 0 ? P->r_rgb0.as<float>() : nullptr;
    CK(launch_preprocess(pa, s));
    return ADPS_OK;
  };
  auto blend = [&](int v, const int* vflag) -> adps_status {
    BlendArgs ba;
    ba.keys = P->r_dup_sorted.as<unsigned long long>();
    ba.order = P->r_order.as<int>();
    ba.vflag = vflag;
    ba.splat = P->r_splat.as<SplatData>();
    ba.tile_start = P->r_tstart.as<int>();
    ba.tile_end = P->r_tend.as<int>();
    ba.tiles_x = tiles_x;
    ba.W = W;
    ba.H = H;
    for (int c = 0; c < 3; ++c) ba.bg[c] = bgv[c];
    ba.image = image + (long long)v * hw * 3;
    ba.dominant = dominant + (long long)v * hw;
    ba.weight = weight;
    ba.contrib = contrib_dev;
    ba.gt = nullptr;
    if (epi_gt) {   // fused attribution epilogue into the plan's step buffers
      ba.gt = epi_gt + (long long)v * hw * 3;
      ba.rawf = P->rawc.as<raw16_t>() + (long long)v * hw;
      ba.lohi = P->r_tile_lohi.as<unsigned long long>() + 2ll * n_tiles * v;
      ba.cls = P->cls.as<unsigned char>();
      ba.N = (int)n;
      ba.dom_flag = P->dom_flag.as<unsigned char>();
      ba.cand_bits = P->cand_bits.as<unsigned>() + (long long)v * ((hw + 31) / 32);
    }
    CK(launch_blend(ba, n_tiles, s));
    return ADPS_OK;
  };
  auto sort_temp = [&](long long dup_items) -> adps_status {
    size_t t1 = 0, t2 = 0, t3 = 0;
    CK(cub::DeviceRadixSort::SortPairs(nullptr, t1, P->r_key.as<unsigned long long>(),
                                       P->r_key_sorted.as<unsigned long long>(), P->r_order_in.as<int>(),
                                       P->r_order.as<int>(), (int)n, 0, 64, s));
    CK(cub::DeviceRadixSort::SortPairs(nullptr, t2, P->r_k32.as<unsigned>(), P->r_k32_sorted.as<unsigned>(),
                                       P->r_order_in.as<int>(), P->r_order.as<int>(), (int)n, 0, 32, s));
    if (dup_items > 0)
      CK(cub::DeviceRadixSort::SortKeys(nullptr, t3, P->r_dup.as<unsigned long long>(),
                                        P->r_dup_sorted.as<unsigned long long>(), (int)dup_items, 32,
                                        32 + tile_bits, s));
    CK(ensure(P->cub_tmp, std::max(t1, std::max(t2, t3))));
    return ADPS_OK;
  };
  auto tile_sort = [&](long long items) -> adps_status {
    size_t tb = P->cub_tmp.bytes;
    CK(cub::DeviceRadixSort::SortKeys(P->cub_tmp.p, tb, P->r_dup.as<unsigned long long>(),
                                      P->r_dup_sorted.as<unsigned long long>(), (int)items, 32, 32 + tile_bits, s));
    return ADPS_OK;
  };
  // one view through the 64-bit depth sort, with a host synchronisation for
  // the pair count (ADPS_PARAM_RENDER_BINNING 0, and the views the fast path
  // hands back: a depth run too long for its fix-up)
  auto render_sorted64 = [&](int v) -> adps_status {
    CK(ensure(P->r_key_sorted, sizeof(unsigned long long) * n));
    adps_status e = preprocess(v, false);
    if (e != ADPS_OK) return e;
    e = sort_temp(0);
    if (e != ADPS_OK) return e;
    size_t tb = P->cub_tmp.bytes;
    CK(cub::DeviceRadixSort::SortPairs(P->cub_tmp.p, tb, P->r_key.as<unsigned long long>(),
                                       P->r_key_sorted.as<unsigned long long>(), P->r_order_in.as<int>(),
                                       P->r_order.as<int>(), (int)n, 0, 64, s));
    unsigned long long* tot = P->r_vtotal.as<unsigned long long>() + n_views;   // scratch slot
    int* flag = P->r_vflag.as<int>() + n_views;
    CK(launch_tile_count_scan(P->r_order.as<int>(), P->r_tiles.as<unsigned>(), P->r_offs.as<unsigned>(), tot, n,
                              sst, s));
    CK(cudaMemsetAsync(flag, 0, sizeof(int), s));
    CK(cudaMemcpyAsync(P->r_total_host, tot, sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    const long long n_dup = (long long)*P->r_total_host;
    if (n_dup > 0x7fffffffLL) return fail(ADPS_INVALID_ARG, "tile list too long (%lld)", n_dup);
    const long long items = n_dup > 0 ? n_dup : 1;
    CK(ensure(P->r_dup, sizeof(unsigned long long) * items));
    CK(ensure(P->r_dup_sorted, sizeof(unsigned long long) * items));
    e = sort_temp(items);
    if (e != ADPS_OK) return e;
    CK(cudaMemsetAsync(P->r_tstart.p, 0, sizeof(int) * n_tiles, s));
    CK(cudaMemsetAsync(P->r_tend.p, 0, sizeof(int) * n_tiles, s));
    DupArgs da{P->r_order.as<int>(), P->r_tiles.as<unsigned>(), P->r_rect.as<unsigned short>(),
               P->r_offs.as<unsigned>(), n, tiles_x, P->r_dup.as<unsigned long long>(), items, tot, flag};
    CK(launch_duplicate(da, s));
    e = tile_sort(items);
    if (e != ADPS_OK) return e;
    CK(launch_tile_ranges(P->r_dup_sorted.as<unsigned long long>(), items, tot, flag, P->r_tstart.as<int>(),
                          P->r_tend.as<int>(), s));
    e = blend(v, nullptr);
    if (e != ADPS_OK) return e;
    P->launches += 5;
    P->lib_calls += 2;
    return ADPS_OK;
  };
  if (!P->render_fast) {
    for (int v = 0; v < n_views; ++v) {
      st = render_sorted64(v);
      if (st != ADPS_OK) return st;
    }
    return ADPS_OK;
  }
  // ---- fast path: no host synchronisation between views.  The tile sort
  //      covers dup_cap pairs (padding keys past the view's own); a view with
  //      more pairs, or a depth run too long for the fix-up, is flagged,
  //      skipped, and rendered again after the call's one synchronisation.
  CK(ensure(P->r_k32, sizeof(unsigned) * n));
  CK(ensure(P->r_k32_sorted, sizeof(unsigned) * n));
  CK(cudaMemsetAsync(P->r_vflag.p, 0, sizeof(int) * (n_views + 1), s));
  auto render_fast = [&](int v, bool learn) -> adps_status {
    int* flag = P->r_vflag.as<int>() + v;
    unsigned long long* tot = P->r_vtotal.as<unsigned long long>() + v;
    adps_status e = preprocess(v, true);
    if (e != ADPS_OK) return e;
    e = sort_temp(P->dup_cap);
    if (e != ADPS_OK) return e;
    size_t tb = P->cub_tmp.bytes;
    CK(cub::DeviceRadixSort::SortPairs(P->cub_tmp.p, tb, P->r_k32.as<unsigned>(), P->r_k32_sorted.as<unsigned>(),
                                       P->r_order_in.as<int>(), P->r_order.as<int>(), (int)n, 0, 32, s));
    CK(launch_depth_fixup(P->r_k32_sorted.as<unsigned>(), P->r_order.as<int>(), P->r_key.as<unsigned long long>(),
                          n, flag, s));
    CK(launch_tile_count_scan(P->r_order.as<int>(), P->r_tiles.as<unsigned>(), P->r_offs.as<unsigned>(), tot, n,
                              sst, s));
    if (learn) {   // the first view of a plan: learn the pair count once
      CK(cudaMemcpyAsync(P->r_total_host, tot, sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
      const long long want = (long long)*P->r_total_host;
      P->dup_cap = std::min(want + want / 8 + 1024, 0x7fffffffLL);
      e = sort_temp(P->dup_cap);
      if (e != ADPS_OK) return e;
    }
    CK(ensure(P->r_dup, sizeof(unsigned long long) * P->dup_cap));
    CK(ensure(P->r_dup_sorted, sizeof(unsigned long long) * P->dup_cap));
    CK(cudaMemsetAsync(P->r_tstart.p, 0, sizeof(int) * n_tiles, s));
    CK(cudaMemsetAsync(P->r_tend.p, 0, sizeof(int) * n_tiles, s));
    DupArgs da{P->r_order.as<int>(), P->r_tiles.as<unsigned>(), P->r_rect.as<unsigned short>(),
               P->r_offs.as<unsigned>(), n, tiles_x, P->r_dup.as<unsigned long long>(), P->dup_cap, tot, flag};
    CK(launch_duplicate(da, s));
    e = tile_sort(P->dup_cap);
    if (e != ADPS_OK) return e;
    CK(launch_tile_ranges(P->r_dup_sorted.as<unsigned long long>(), P->dup_cap, tot, flag, P->r_tstart.as<int>(),
                          P->r_tend.as<int>(), s));
    e = blend(v, flag);
    if (e != ADPS_OK) return e;
    P->launches += 6;   // preprocess, fix-up, scan, duplication, ranges, blend
    P->lib_calls += 2;
    return ADPS_OK;
  };
  for (int v = 0; v < n_views; ++v) {
    st = render_fast(v, v == 0 && P->dup_cap <= 0);
    if (st != ADPS_OK) return st;
  }
  P->vflag_host.resize(n_views);
  P->vtotal_host.resize(n_views);
  CK(cudaMemcpyAsync(P->vflag_host.data(), P->r_vflag.p, sizeof(int) * n_views, cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(P->vtotal_host.data(), P->r_vtotal.p, sizeof(unsigned long long) * n_views,
                     cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  long long need = 0, most = 0;
  for (int v = 0; v < n_views; ++v) {
    most = std::max(most, (long long)P->vtotal_host[v]);
    if (P->vflag_host[v] == 1) need = std::max(need, (long long)P->vtotal_host[v]);
  }
  if (need > 0x7fffffffLL) return fail(ADPS_INVALID_ARG, "tile lists too long (%lld pairs)", need);
  if (need > 0) {   // more pairs than the sort covered: redo those views with room for them
    P->dup_cap = std::min(need + need / 8 + 1024, 0x7fffffffLL);
    for (int v = 0; v < n_views; ++v)
      if (P->vflag_host[v] == 1) {
        CK(cudaMemsetAsync(P->r_vflag.as<int>() + v, 0, sizeof(int), s));
        st = render_fast(v, false);
        if (st != ADPS_OK) return st;
      }
    CK(cudaMemcpyAsync(P->vflag_host.data(), P->r_vflag.p, sizeof(int) * n_views, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    for (int v = 0; v < n_views; ++v)
      if (P->vflag_host[v] == 1) return fail(ADPS_BAD_STATE, "tile pairs still exceed the grown capacity");
  } else if (most > 0 && n_views >= 4) {
    // follow the largest view of this call with a 3 % margin: the padding is
    // sorted too (a view of the next call that exceeds it is redone)
    P->dup_cap = std::min(most + most / 32 + 1024, 0x7fffffffLL);
  }
  for (int v = 0; v < n_views; ++v)
    if (P->vflag_host[v] == 2) {   // a run of equal 32-bit depth keys too long for the fix-up
      st = render_sorted64(v);
      if (st != ADPS_OK) return st;
    }
  return ADPS_OK;
}

// ------------------------------------------------------------------ phase 1

static AttributionArgs attr_args(adps_plan* P, int V, int H, int W, const adps_config* cfg, int N,
                                 const float* image, const float* gt, const int32_t* dominant) {
  Counters* ctr = P->ctr.as<Counters>();
  AttributionArgs a;
  a.image = image;
  a.gt = gt;
  a.dom = dominant;
  a.V = V;
  a.H = H;
  a.W = W;
  a.view_offset = P->view_offset;
  a.view_stride = P->view_stride;
  a.L = cfg->l_bands;
  a.r_erode = cfg->r_erode;
  a.m_min = cfg->m_min;
  a.tau = cfg->tau_l1;
  a.cls = P->cls.as<unsigned char>();
  a.N = N;
  a.dom_flag = P->dom_flag.as<unsigned char>();
  a.lohi = P->lohi.as<unsigned long long>();
  a.lo = P->lo.as<double>();
  a.thr = P->thr.as<double>();
  a.thr_raw = P->thr_raw.as<double>();
  a.regions = P->regions.as<RegionRec>();
  a.n_regions = &ctr->n_regions;
  a.region_cap = P->region_cap;
  a.partials = P->partials.as<PartialRec>();
  a.n_partials = &ctr->n_partials;
  a.tile_records = &ctr->tile_records;
  a.partial_cap = P->partial_cap;
  a.partial_parent = P->partial_parent.as<int>();
  a.border = P->border.as<int>();
  a.dbg_m = P->dbg_m;
  a.dbg_b = P->dbg_b;
  a.overflow = &ctr->overflow;
  a.grid_small = (unsigned)(P->sm_count * 4);
  a.input_blocks_per_sm = P->input_blocks_per_sm;
  a.deferred = P->deferred.as<int>();
  a.n_deferred = &ctr->n_deferred;
  a.tile_path = P->tile_path;
  a.cand_bits = P->cand_bits.as<unsigned>();
  // the bit-plane path caches raw as fp32 (round toward zero), the others as fp64
  a.raw = P->use_raw && !P->use_bits ? P->rawc.as<double>() : nullptr;
  a.rawf = P->use_bits ? P->rawc.as<raw16_t>() : nullptr;
  a.words = P->use_words ? P->twords.as<uint4>() : nullptr;
  return a;
}

// tile CCL + border merge (after the per-view thresholds exist)
static adps_status run_attribution(adps_plan* P, cudaStream_t s, int V, int H, int W, const adps_config* cfg,
                                   int N, const float* image, const float* gt, const int32_t* dominant) {
  Counters* ctr = P->ctr.as<Counters>();
  CK(cudaMemsetAsync(&ctr->n_regions, 0, sizeof(unsigned long long), s));
  CK(cudaMemsetAsync(&ctr->n_partials, 0, sizeof(unsigned long long), s));
  CK(cudaMemsetAsync(&ctr->tile_records, 0, sizeof(unsigned long long), s));
  CK(cudaMemsetAsync(&ctr->overflow, 0, sizeof(unsigned int), s));
  CK(cudaMemsetAsync(&ctr->n_deferred, 0, sizeof(unsigned long long), s));
  const AttributionArgs a = attr_args(P, V, H, W, cfg, N, image, gt, dominant);
  CK(launch_attribution(a, s, mark_cb, P));
  return ADPS_OK;
}

// Fused attribution (SURVEY.md 8(d) "K1 epilogue"): select, then the
// attribution render of the sampled views whose epilogue also writes what the
// step's input pass would (raw cache, per-view min/max, candidate bits,
// ever-dominant flags).  The next adps_step_phase1_begin with the same inputs
// skips select and the input pass and starts from that 8 B/px boundary.
extern "C" adps_status adps_render_fused(adps_plan* P, void* stream_v, const adps_gaussians* g, int64_t n,
                                         double extent, const double* grad_accum, const double* denom,
                                         const adps_config* cfg, const double* cams_host, int32_t n_views,
                                         const float* bg, const float* gt, float* image, int32_t* dominant) {
  if (!P) return fail(ADPS_INVALID_ARG, "plan is NULL");
  P->fused.valid = false;
  adps_status st = check_gaussians(g, n);
  if (st != ADPS_OK) return st;
  if (!cfg) return fail(ADPS_INVALID_ARG, "cfg is NULL");
  if (n > 0 && (!grad_accum || !denom)) return fail(ADPS_INVALID_ARG, "stats arrays are NULL");
  if (n_views < 1 || !cams_host || !gt || !image || !dominant) return fail(ADPS_INVALID_ARG, "view arrays are NULL");
  if (!(extent > 0)) return fail(ADPS_INVALID_ARG, "scene extent must be > 0");
  CK(cudaSetDevice(P->device));
  cudaStream_t s = (cudaStream_t)stream_v;
  const CamD c0 = load_cam(cams_host);
  const int W = c0.w, H = c0.h, V = n_views;
  if (W <= 0 || H <= 0) return fail(ADPS_INVALID_ARG, "empty image");
  for (int v = 1; v < V; ++v) {
    const CamD cv = load_cam(cams_host + 18ll * v);
    if (cv.w != W || cv.h != H) return fail(ADPS_INVALID_ARG, "all sampled views must share H x W");
  }
  if (n == 0) return render_impl(P, stream_v, g, n, cams_host, n_views, bg, image, dominant, nullptr, nullptr);
  const long long hw = (long long)H * W;
  const long long nn = n;
  CK(ensure(P->cls, nn));
  CK(ensure(P->cand_rank, 4 * nn));
  CK(ensure(P->split_list, 4 * nn));
  CK(ensure(P->clone_list, 4 * nn));
  CK(ensure(P->dom_flag, nn));
  CK(ensure(P->lohi, 16ll * V));
  CK(ensure(P->rawc, 2ll * hw * V));
  CK(ensure(P->cand_bits, 4ll * V * ((hw + 31) / 32) + 4));
  CK(ensure(P->ctr, sizeof(Counters)));
  if (P->cams_host_cap < V) {
    if (P->cams_host) cudaFreeHost(P->cams_host);
    if (P->lohi_host) cudaFreeHost(P->lohi_host);
    CK(cudaMallocHost(&P->cams_host, sizeof(double) * 18 * V));
    CK(cudaMallocHost(&P->lohi_host, sizeof(unsigned long long) * 2 * V));
    P->cams_host_cap = V;
  }
  Counters* ctr = P->ctr.as<Counters>();
  CK(cudaMemsetAsync(ctr, 0, sizeof(Counters), s));
  CK(cudaMemsetAsync(P->dom_flag.p, 0, (size_t)nn, s));
  CK(cudaMemsetAsync(P->cand_bits.p, 0, 4ll * V * ((hw + 31) / 32) + 4, s));
  for (int v = 0; v < V; ++v) {
    P->lohi_host[2 * v] = 0x7ff0000000000000ull;   // +inf
    P->lohi_host[2 * v + 1] = 0ull;                // +0.0
  }
  CK(cudaMemcpyAsync(P->lohi.p, P->lohi_host, sizeof(unsigned long long) * 2 * V, cudaMemcpyHostToDevice, s));
  ScanState sst;
  st = scan_state(P, P->scan_val, P->scan_flag, nn, &sst);
  if (st != ADPS_OK) return st;
  SelectArgs sa;
  sa.scale = g->scale;
  sa.ga = grad_accum;
  sa.den = denom;
  sa.tau_g = cfg->tau_g;
  sa.tau_s_abs = cfg->tau_s * extent;
  sa.n = n;
  sa.cls = P->cls.as<unsigned char>();
  sa.cand_rank = P->cand_rank.as<int>();
  sa.split_list = P->split_list.as<int>();
  sa.clone_list = P->clone_list.as<int>();
  sa.ctr = ctr;
  CK(launch_select(sa, sst, s));
  P->launches += 1;
  {
    const int tiles_x = (W + kRTile - 1) / kRTile, tiles_y = (H + kRTile - 1) / kRTile;
    CK(ensure(P->r_tile_lohi, 16ll * tiles_x * tiles_y * V));
  }
  st = render_impl(P, stream_v, g, n, cams_host, n_views, bg, image, dominant, nullptr, nullptr, gt);
  if (st != ADPS_OK) return st;
  {
    const int n_tiles = ((W + kRTile - 1) / kRTile) * ((H + kRTile - 1) / kRTile);
    CK(launch_reduce_tile_minmax(P->r_tile_lohi.as<unsigned long long>(), n_tiles, V,
                                 P->lohi.as<unsigned long long>(), s));
    P->launches += 1;
  }
  P->fused.valid = true;
  P->fused.g = *g;
  P->fused.n = n;
  P->fused.extent = extent;
  P->fused.ga = grad_accum;
  P->fused.den = denom;
  P->fused.cfg = *cfg;
  P->fused.V = V;
  P->fused.H = H;
  P->fused.W = W;
  P->fused.image = image;
  P->fused.gt = gt;
  P->fused.dom = dominant;
  P->fused.cams.assign(cams_host, cams_host + 18ll * V);
  return ADPS_OK;
}

static bool same_gaussians(const adps_gaussians& a, const adps_gaussians& b) {
  return a.mu == b.mu && a.scale == b.scale && a.rot == b.rot && a.opacity == b.opacity && a.sh_dc == b.sh_dc &&
         a.sh_rest == b.sh_rest && a.sh_rest_k == b.sh_rest_k;
}

extern "C" adps_status adps_step_phase1(adps_plan* P, void* stream_v, const adps_gaussians* g, int64_t n,
                                        double extent, const double* grad_accum, const double* denom,
                                        const adps_config* cfg, const double* cams_host, int32_t n_views,
                                        const float* image, const float* gt, const int32_t* dominant,
                                        adps_counts* counts) {
  adps_status st = adps_step_phase1_begin(P, stream_v, g, n, extent, grad_accum, denom, cfg, cams_host, n_views,
                                          image, gt, dominant, counts);
  if (st != ADPS_OK) return st;
  return adps_step_phase1_end(P, stream_v, counts);
}

extern "C" adps_status adps_step_phase1_begin(adps_plan* P, void* stream_v, const adps_gaussians* g, int64_t n,
                                              double extent, const double* grad_accum, const double* denom,
                                              const adps_config* cfg, const double* cams_host, int32_t n_views,
                                              const float* image, const float* gt, const int32_t* dominant,
                                              adps_counts* counts) {
  if (!P) return fail(ADPS_INVALID_ARG, "plan is NULL");
  P->have_phase1 = false;
  P->have_begin = false;
  drop_pending_normals(P);
  adps_status st = check_gaussians(g, n);
  if (st != ADPS_OK) return st;
  if (!cfg || !counts) return fail(ADPS_INVALID_ARG, "cfg/counts is NULL");
  if (n > 0 && (!grad_accum || !denom)) return fail(ADPS_INVALID_ARG, "stats arrays are NULL");
  if (n_views < 1) return fail(ADPS_INVALID_ARG, "need at least one sampled view");
  if (!cams_host || !image || !gt || !dominant) return fail(ADPS_INVALID_ARG, "view arrays are NULL");
  if (!(cfg->tau_l1 > 0.0 && cfg->tau_l1 < 1.0)) return fail(ADPS_INVALID_ARG, "tau_l1 must lie in (0,1)");
  if (cfg->l_bands < 1 || cfg->l_bands > 255) return fail(ADPS_INVALID_ARG, "l_bands must be in [1,255]");
  if (cfg->n_max < 1) return fail(ADPS_INVALID_ARG, "n_max must be >= 1");
  if (cfg->r_erode > 2 * kMaxErodeHalo + 1) return fail(ADPS_INVALID_ARG, "r_erode > %d unsupported", 2 * kMaxErodeHalo + 1);
  if (!(extent > 0)) return fail(ADPS_INVALID_ARG, "scene extent must be > 0");
  CK(cudaSetDevice(P->device));
  cudaStream_t s = (cudaStream_t)stream_v;
  const CamD c0 = load_cam(cams_host);
  const int W = c0.w, H = c0.h, V = n_views;
  for (int v = 1; v < V; ++v) {
    const CamD cv = load_cam(cams_host + 18ll * v);
    if (cv.w != W || cv.h != H) return fail(ADPS_INVALID_ARG, "all sampled views must share H x W");
  }
  if (W <= 0 || H <= 0) return fail(ADPS_INVALID_ARG, "empty image");
  P->v_glob = P->v_global_cfg > 0 ? P->v_global_cfg : V;
  if (P->view_offset + (long long)(V - 1) * P->view_stride >= P->v_glob)
    return fail(ADPS_INVALID_ARG, "local views exceed the global view count of the sharding");
  P->v_glob = P->v_global_cfg > 0 ? P->v_global_cfg : V;
  if (P->view_offset + (long long)(V - 1) * P->view_stride >= P->v_glob)
    return fail(ADPS_INVALID_ARG, "local views exceed the global view count of the sharding");
  const long long hw = (long long)H * W;
  const long long total_px = hw * V;
  const int tiles_x = (W + kTileW - 1) / kTileW, tiles_y = (H + kTileH - 1) / kTileH;
  const long long n_tiles = (long long)tiles_x * tiles_y * V;
  const int N = (int)n;

  // ---- buffers
  const long long nn = n > 0 ? n : 1;
  CK(ensure(P->cls, nn));
  CK(ensure(P->cand_rank, 4 * nn));
  CK(ensure(P->split_list, 4 * nn));
  CK(ensure(P->clone_list, 4 * nn));
  CK(ensure(P->dom_flag, nn));
  CK(ensure(P->keep_pos, 4 * nn));
  CK(ensure(P->lohi, 16ll * V));
  CK(ensure(P->lo, 8ll * V));
  CK(ensure(P->thr, 8ll * V * cfg->l_bands));
  CK(ensure(P->thr_raw, 8ll * V * cfg->l_bands));
  CK(ensure(P->cams, 8ll * 18 * V));
  CK(ensure(P->border, 4ll * n_tiles * kBorderSlots));
  CK(ensure(P->deferred, 4ll * n_tiles));
  CK(ensure(P->cand_bits, 4ll * V * ((hw + 31) / 32) + 4));   // + 1 word: tile_words_kernel reads one past a row
  P->use_raw = P->raw_cache && P->tile_path != 1 && !P->dbg_m && cfg->r_erode <= 3;
  P->use_bits = P->use_raw && (P->tile_path == 0 || P->tile_path == 3) && cfg->l_bands <= 4;
  P->use_words = P->use_bits && P->tile_path == 0;   // path 3: planes computed per tile (fused)
  if (P->use_raw) CK(ensure(P->rawc, (P->use_bits ? 2ll : 8ll) * total_px));
  if (P->use_words) CK(ensure(P->twords, (long long)tile_words_bytes(V, H, W)));
  CK(ensure(P->ctr, sizeof(Counters)));
  if (P->cams_host_cap < V) {
    if (P->cams_host) cudaFreeHost(P->cams_host);
    if (P->lohi_host) cudaFreeHost(P->lohi_host);
    CK(cudaMallocHost(&P->cams_host, sizeof(double) * 18 * V));
    CK(cudaMallocHost(&P->lohi_host, sizeof(unsigned long long) * 2 * V));
    P->cams_host_cap = V;
  }
  const long long region_bound = total_px / (cfg->m_min > 1 ? cfg->m_min : 1) + 1;
  const long long partial_bound = n_tiles * (2 * kTileW + 2 * kTileH) + 1;
  // the tile CCLs count both record kinds in the halves of one 64-bit word
  if (region_bound >= (1ll << 32) || partial_bound >= (1ll << 32))
    return fail(ADPS_INVALID_ARG, "%lld pixels: the region count may exceed 2^32", total_px);
  // per-call capacities: the largest seen so far (at least 2^21), never above the analytic bound
  P->region_hint = P->region_cap > P->region_hint ? P->region_cap : P->region_hint;
  P->partial_hint = P->partial_cap > P->partial_hint ? P->partial_cap : P->partial_hint;
  {
    long long r = P->region_hint > (1ll << 21) ? P->region_hint : (1ll << 21);
    long long q = P->partial_hint > (1ll << 21) ? P->partial_hint : (1ll << 21);
    P->region_cap = r < region_bound ? r : region_bound;
    P->partial_cap = q < partial_bound ? q : partial_bound;
  }
  CK(ensure(P->regions, sizeof(RegionRec) * P->region_cap));
  CK(ensure(P->partials, sizeof(PartialRec) * P->partial_cap));
  CK(ensure(P->partial_parent, sizeof(int) * P->partial_cap));
  memcpy(P->cams_host, cams_host, sizeof(double) * 18 * V);
  P->cams_pending = true;   // copied at the end of the begin (below)
  Counters* ctr = P->ctr.as<Counters>();
  // the attribution of a fused render on exactly these inputs (one use)
  const bool fused = P->fused.valid && P->use_bits && same_gaussians(P->fused.g, *g) && P->fused.n == n &&
                     P->fused.extent == extent && P->fused.ga == grad_accum && P->fused.den == denom &&
                     memcmp(&P->fused.cfg, cfg, sizeof(adps_config)) == 0 && P->fused.V == V && P->fused.H == H &&
                     P->fused.W == W && P->fused.image == image && P->fused.gt == gt && P->fused.dom == dominant &&
                     P->view_offset == 0 && P->view_stride == 1 && P->v_glob == V &&
                     memcmp(P->fused.cams.data(), cams_host, sizeof(double) * 18 * V) == 0;
  P->fused.valid = false;
  if (!fused) CK(cudaMemsetAsync(ctr, 0, sizeof(Counters), s));
  mark_start(P, s, true);
  if (fused) {   // select and the input pass ran in the render's epilogue
    const AttributionArgs a = attr_args(P, V, H, W, cfg, N, image, gt, dominant);
    P->attr_pending = false;
    CK(launch_thresholds(a, 0, V, s));
    CK(launch_fallback_count(P->split_list.as<int>(), P->dom_flag.as<unsigned char>(), ctr, P->sm_count, s));
    mark(P, "thresholds", s, 2);
    if (P->pipeline && !P->timing && attribution_warp_path(a)) {   // the CCL on the second stream
      CK(cudaEventRecord(P->ev_chunk[0], s));
      CK(cudaStreamWaitEvent(P->aux, P->ev_chunk[0], 0));
      CK(launch_tiles_views(a, 0, V, P->aux));
      CK(launch_attribution_tail(a, P->aux, nullptr, nullptr));
      CK(cudaEventRecord(P->ev_attr, P->aux));
      P->attr_pending = true;
      P->launches += (P->use_words ? 2 : 1) + 4;
    }
  } else {

  // ---- select (ref/adc.py:165)
  ScanState sst;
  st = scan_state(P, P->scan_val, P->scan_flag, nn, &sst);
  if (st != ADPS_OK) return st;
  SelectArgs sa;
  sa.scale = g->scale;
  sa.ga = grad_accum;
  sa.den = denom;
  sa.tau_g = cfg->tau_g;
  sa.tau_s_abs = cfg->tau_s * extent;
  sa.n = n;
  sa.cls = P->cls.as<unsigned char>();
  sa.cand_rank = P->cand_rank.as<int>();
  sa.split_list = P->split_list.as<int>();
  sa.clone_list = P->clone_list.as<int>();
  sa.ctr = ctr;
  // pipelined: the classes on `stream` (all the input pass needs), the list
  // scan on the second stream alongside the input pass, joined before the
  // fallback count
  const bool split_select = P->pipeline && !P->timing;
  const bool fold_init = split_select && ADPS_SELECT_FOLD;
  if (split_select) {
    if (fold_init) {
      sa.dom_zero = P->dom_flag.as<unsigned char>();
      sa.lohi_init = P->lohi.as<unsigned long long>();
      sa.lohi_views = V;
    }
    CK(launch_select_split(sa, sst, s, P->aux, P->ev_cfork, P->ev_child));
    mark(P, "select", s, 2);
  } else {
    CK(launch_select(sa, sst, s));
    mark(P, "select", s, 1);
  }

  // ---- ever-dominant flags (ref/adc.py:177-180) and the fallback count, so
  //      the host can draw the fallback normals while the rest runs
  if (!fold_init) {   // (the split select's classify pass zeroed and seeded them)
    CK(cudaMemsetAsync(P->dom_flag.p, 0, (size_t)nn, s));
    for (int v = 0; v < V; ++v) {
      P->lohi_host[2 * v] = 0x7ff0000000000000ull;   // +inf
      P->lohi_host[2 * v + 1] = 0ull;                // +0.0
    }
    CK(cudaMemcpyAsync(P->lohi.p, P->lohi_host, sizeof(unsigned long long) * 2 * V, cudaMemcpyHostToDevice, s));
    mark(P, "input_init", s, 0);   // (timing mode: the input pass's own stage starts here)
  }
  {
    const AttributionArgs a = attr_args(P, V, H, W, cfg, N, image, gt, dominant);
    P->attr_pending = false;
    if (P->pipeline && !P->timing && V >= 2 && attribution_warp_path(a)) {
      // views in chunks: minmax of chunk c on `stream`, the warp CCL of chunk c
      // on the second stream as soon as its thresholds exist; the tail (deferred
      // tiles, border merge) after the last chunk; phase1_end joins it
      const int maxc = P->pipeline_chunks < adps_plan::kMaxChunks ? P->pipeline_chunks : adps_plan::kMaxChunks;
      const int chunks = V < maxc ? V : maxc;
      for (int c = 0; c < chunks; ++c) {
        const int v0 = (int)((long long)V * c / chunks), v1 = (int)((long long)V * (c + 1) / chunks);
        CK(launch_minmax_views(a, v0, v1, s));
        CK(cudaEventRecord(P->ev_chunk[c], s));
        CK(cudaStreamWaitEvent(P->aux, P->ev_chunk[c], 0));
        CK(launch_tiles_views(a, v0, v1, P->aux));
      }
      if (split_select) CK(cudaStreamWaitEvent(s, P->ev_child, 0));   // split list + n_split
      CK(launch_fallback_count(P->split_list.as<int>(), P->dom_flag.as<unsigned char>(), ctr, P->sm_count, s));
      CK(launch_attribution_tail(a, P->aux, nullptr, nullptr));
      CK(cudaEventRecord(P->ev_attr, P->aux));
      P->attr_pending = true;
      P->launches += (P->use_words ? 4 : 3) * chunks + 1 + 4;   // minmax, thresholds, [words,] bits per chunk
    } else {
      // one launch over all views: the input pass, then thresholds + fallback count
      CK(launch_minmax_kernel(a, 0, V, s));
      mark(P, "minmax", s, 1);
      CK(launch_thresholds(a, 0, V, s));
      if (split_select) CK(cudaStreamWaitEvent(s, P->ev_child, 0));   // split list + n_split
      CK(launch_fallback_count(P->split_list.as<int>(), P->dom_flag.as<unsigned char>(), ctr, P->sm_count, s));
      mark(P, "thresholds", s, 2);
    }
  }
  }   // not fused
  // the cameras are read first by child init (after phase 1's first sync):
  // copied on the second stream behind the work already queued there, off
  // this stream's kernel chain
  CK(cudaMemcpyAsync(P->cams.p, P->cams_host, sizeof(double) * 18 * V, cudaMemcpyHostToDevice, P->aux));
  CK(cudaEventRecord(P->ev_cams, P->aux));
  CK(cudaMemcpyAsync(P->ctr_host, ctr, sizeof(Counters), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  {
    adps_counts K{};
    K.n_before = n;
    K.n_split = (long long)P->ctr_host->n_split;
    K.n_clone = (long long)P->ctr_host->n_clone;
    K.n_fallback = (long long)P->ctr_host->n_fallback_pre;
    *counts = K;
  }
  P->cx.g = *g;
  P->cx.n = n;
  P->cx.extent = extent;
  P->cx.cfg = *cfg;
  P->cx.V = V;
  P->cx.H = H;
  P->cx.W = W;
  P->cx.image = image;
  P->cx.gt = gt;
  P->cx.dominant = dominant;
  P->have_begin = true;
  return ADPS_OK;
}

// launch fallback normals requested with sync == 2 (waits on the event
// recorded at the request, not on the work queued since)
static cudaError_t launch_deferred_normals(adps_plan* P) {
  if (!P->norm_deferred) return cudaSuccess;
  P->norm_deferred = false;
  cudaError_t e = cudaStreamWaitEvent(P->nstream, P->ev_nfork, 0);
  if (e == cudaSuccess) e = launch_normals(P->nrm_args, P->nrm_tmp.p, P->nrm_tmp.bytes, P->nstream);
  if (e == cudaSuccess) e = cudaEventRecord(P->ev_norm, P->nstream);
  if (e != cudaSuccess) return e;
  P->norm_pending = true;
  P->launches += 5;
  P->lib_calls += 2;
  return cudaSuccess;
}

// attribution + region statistics + child init over this plan's (local) views
static adps_status phase1_local(adps_plan* P, cudaStream_t s, long long* n_regions_out, bool defer_child = false) {
  CK(cudaSetDevice(P->device));
  adps_status st = ADPS_OK;
  const adps_gaussians* g = &P->cx.g;
  const long long n = P->cx.n;
  const adps_config* cfg = &P->cx.cfg;
  const int V = P->cx.V, H = P->cx.H, W = P->cx.W;
  const float* image = P->cx.image;
  const float* gt = P->cx.gt;
  const int32_t* dominant = P->cx.dominant;
  const long long hw = (long long)H * W;
  const long long total_px = hw * V;
  const int tiles_x = (W + kTileW - 1) / kTileW, tiles_y = (H + kTileH - 1) / kTileH;
  const long long n_tiles = (long long)tiles_x * tiles_y * V;
  const int N = (int)n;
  const long long region_bound = total_px / (cfg->m_min > 1 ? cfg->m_min : 1) + 1;
  const long long partial_bound = n_tiles * (2 * kTileW + 2 * kTileH) + 1;
  Counters* ctr = P->ctr.as<Counters>();

  // ---- maps + partition + moments (ref/adc.py:168-176)
  for (int attempt = 0;; ++attempt) {
    if (attempt == 0 && P->attr_pending) {   // launched by phase1_begin, pipelined with the input pass
      CK(cudaStreamWaitEvent(s, P->ev_attr, 0));
      P->attr_pending = false;
    } else {
      st = run_attribution(P, s, V, H, W, cfg, N, image, gt, dominant);
      if (st != ADPS_OK) return st;
    }
    CK(cudaMemcpyAsync(P->ctr_host, ctr, sizeof(Counters), cudaMemcpyDeviceToHost, s));
    CK(launch_deferred_normals(P));   // host time while the GPU runs the attribution
    CK(cudaStreamSynchronize(s));
    if (!P->ctr_host->overflow) break;
    if (attempt >= 2) return fail(ADPS_BAD_STATE, "region capacity overflow at the analytic bound");
    // grow: first to what this run needed, then (if still short) to the analytic bounds
    long long want_r = (long long)P->ctr_host->n_regions + (long long)P->ctr_host->n_partials + 1;
    long long want_p = (long long)P->ctr_host->n_partials + 1;
    if (attempt == 1) {
      want_r = region_bound;
      want_p = partial_bound;
    }
    P->region_cap = want_r < region_bound ? (want_r > P->region_cap ? want_r : P->region_cap) : region_bound;
    P->partial_cap = want_p < partial_bound ? (want_p > P->partial_cap ? want_p : P->partial_cap) : partial_bound;
    CK(ensure(P->regions, sizeof(RegionRec) * P->region_cap));
    CK(ensure(P->partials, sizeof(PartialRec) * P->partial_cap));
    CK(ensure(P->partial_parent, sizeof(int) * P->partial_cap));
  }
  const long long n_regions = (long long)P->ctr_host->n_regions;
  const long long n_split = (long long)P->ctr_host->n_split;
  mark(P, "host_sync", s, 0);

  // ---- region stats + child init (ref/adc.py:172-176, 190-196)
  const long long rc = n_regions > 0 ? n_regions : 1;
  CK(ensure(P->props, sizeof(Proposal) * rc));
  CK(ensure(P->valid, rc));
  CK(ensure(P->keys, 8 * rc));
  CK(ensure(P->vals, 4 * rc));
  CK(ensure(P->keys_sorted, 8 * rc));
  CK(ensure(P->vals_sorted, 4 * rc));
  CK(ensure(P->idx, 4 * rc));
  CK(ensure(P->uf, 4 * rc));
  CK(ensure(P->groups, sizeof(GroupRec) * rc));
  CK(ensure(P->children, sizeof(float) * 14 * rc));
  if (P->dbg_records) {
    CK(ensure(P->dbg_stats, sizeof(double) * 10 * rc));
    CK(ensure(P->dbg_child, sizeof(double) * 16 * rc));
  }
  const int bits_v = ceil_log2((unsigned long long)P->v_glob);
  const int bits_b = ceil_log2((unsigned long long)cfg->l_bands);
  const int bits_p = ceil_log2((unsigned long long)hw);
  const int bits_c = ceil_log2((unsigned long long)(n_split > 0 ? n_split : 1));
  const int total_bits = bits_c + bits_v + bits_b + bits_p;
  if (total_bits > 64) return fail(ADPS_INVALID_ARG, "region sort key needs %d bits (> 64)", total_bits);
  if (P->cams_pending) {   // the cameras' copy on the second stream
    CK(cudaStreamWaitEvent(s, P->ev_cams, 0));
    P->cams_pending = false;
  }
  ChildArgs ca;
  ca.regions = P->regions.as<RegionRec>();
  ca.n_regions = &ctr->n_regions;
  ca.region_cap = P->region_cap;
  ca.g = to_in(g);
  ca.cams = P->cams.as<double>();
  ca.gt = gt;
  ca.H = H;
  ca.W = W;
  ca.view_offset = P->view_offset;
  ca.view_stride = P->view_stride;
  ca.eps = cfg->eps;
  ca.cand_rank = P->cand_rank.as<int>();
  ca.bits_v = bits_v;
  ca.bits_b = bits_b;
  ca.bits_p = bits_p;
  ca.props = P->props.as<Proposal>();
  ca.valid = P->valid.as<unsigned char>();
  ca.keys = P->keys.as<unsigned long long>();
  ca.vals = P->vals.as<int>();
  ca.dbg_stats = P->dbg_records ? P->dbg_stats.as<double>() : nullptr;
  ca.dbg_child = P->dbg_records ? P->dbg_child.as<double>() : nullptr;
  ca.ctr = ctr;
  long long cgrid = (n_regions + 127) / 128;
  ca.grid = (unsigned)(cgrid < 1 ? 1 : (cgrid > 65535 ? 65535 : cgrid));
  ca.write_keys = true;
  if (n_regions > 0 && defer_child && !P->timing) {
    // the sort keys on this stream (the region sort starts at once); child init
    // on the second stream, concurrently with the sort; joined before the ranges
    ca.write_keys = false;
    CK(launch_region_keys(ca.regions, n_regions, ca.cand_rank, bits_v, bits_b, bits_p, ca.keys, ca.vals, s));
    CK(cudaEventRecord(P->ev_cfork, s));
    CK(cudaStreamWaitEvent(P->aux, P->ev_cfork, 0));
    CK(launch_child_init(ca, P->aux));
    CK(cudaEventRecord(P->ev_child, P->aux));
    P->child_pending = true;
    mark(P, "child_init", s, 2);
  } else {
    if (n_regions > 0) CK(launch_child_init(ca, s));
    mark(P, "child_init", s, n_regions > 0 ? 1 : 0);
  }
  P->n_regions_cur = n_regions;
  *n_regions_out = n_regions;
  return ADPS_OK;
}

// sort + ranges + merge + cap + case + offsets over the plan's region records
// (local ones, or the gathered records of all ranks after adps_step_phase1_import)
static adps_status phase1_finish(adps_plan* P, cudaStream_t s, adps_counts* counts);

// sort + ranges + merge + cap over the plan's region records (local ones, or
// the gathered records of all ranks after adps_step_phase1_import); with
// parent sharding only this rank's candidate range is gated/grouped/capped
static adps_status phase1_merge_part(adps_plan* P, cudaStream_t s) {
  CK(cudaSetDevice(P->device));
  adps_status st = ADPS_OK;
  const adps_gaussians* g = &P->cx.g;
  const long long n = P->cx.n;
  const double extent = P->cx.extent;
  const adps_config* cfg = &P->cx.cfg;
  const int V = P->v_glob, H = P->cx.H, W = P->cx.W;
  const long long hw = (long long)H * W;
  const long long nn = n > 0 ? n : 1;
  Counters* ctr = P->ctr.as<Counters>();
  ScanState sst;
  st = scan_state(P, P->scan_val, P->scan_flag, nn, &sst);
  if (st != ADPS_OK) return st;
  const long long n_regions = P->n_regions_cur;
  const long long n_split = (long long)P->ctr_host->n_split;
  const long long rc = n_regions > 0 ? n_regions : 1;
  const int bits_v = ceil_log2((unsigned long long)V);
  const int bits_b = ceil_log2((unsigned long long)cfg->l_bands);
  const int bits_p = ceil_log2((unsigned long long)hw);
  const int bits_c = ceil_log2((unsigned long long)(n_split > 0 ? n_split : 1));
  const int total_bits = bits_c + bits_v + bits_b + bits_p;
  if (total_bits > 64) return fail(ADPS_INVALID_ARG, "region sort key needs %d bits (> 64)", total_bits);
  // ---- order (candidate, view, band, first pixel)  (ref/adc.py:190-195)
  if (n_regions > 0) {
    size_t tb = 0;
    CK(cub::DeviceRadixSort::SortPairs(nullptr, tb, P->keys.as<unsigned long long>(),
                                       P->keys_sorted.as<unsigned long long>(), P->vals.as<int>(),
                                       P->vals_sorted.as<int>(), (int)n_regions, 0, total_bits > 0 ? total_bits : 1, s));
    CK(ensure(P->cub_tmp, tb));
    tb = P->cub_tmp.bytes;
    CK(cub::DeviceRadixSort::SortPairs(P->cub_tmp.p, tb, P->keys.as<unsigned long long>(),
                                       P->keys_sorted.as<unsigned long long>(), P->vals.as<int>(),
                                       P->vals_sorted.as<int>(), (int)n_regions, 0, total_bits > 0 ? total_bits : 1, s));
  }
  const long long sc = n_split > 0 ? n_split : 1;
  CK(ensure(P->cand_start, 4 * sc));
  CK(ensure(P->cand_end, 4 * sc));
  CK(ensure(P->cand_nvalid, 4 * sc));
  CK(ensure(P->cand_case, 4 * sc));
  CK(ensure(P->cand_props, 4 * sc));
  CK(ensure(P->cand_merged, 4 * sc));
  CK(ensure(P->cand_ins, 4 * sc));
  CK(ensure(P->ins_off, 4 * sc));
  CK(ensure(P->fb_ord, 4 * sc));
  CK(ensure(P->large_list, 4 * sc));
  CK(ensure(P->small_list, 4 * sc));
  CK(ensure(P->pstart, 4 * sc));
  CK(ensure(P->n_groups, 4 * sc));
  CK(ensure(P->gfirst_of, 4 * sc));
  CK(ensure(P->work_cnt, 8 * sc));
  CK(ensure(P->work_off, 8 * (sc + 1)));
  CK(ensure(P->props_s, sizeof(Proposal) * rc));
  CK(ensure(P->psrc, 4 * rc));
  CK(ensure(P->pcand, 4 * rc));
  CK(ensure(P->gkey, 4 * rc));
  CK(ensure(P->gval, 4 * rc));
  CK(ensure(P->gkey_sorted, 4 * rc));
  CK(ensure(P->gval_sorted, 4 * rc));
  CK(ensure(P->grp_first, 4 * (rc + 1)));
  CK(ensure(P->gpar, 4 * rc));
  CK(ensure(P->gext, 8 * rc));
  CK(ensure(P->glist, 12 * rc));
  CK(ensure(P->large_of, 4 * sc));
  CK(ensure(P->lp_cnt, 8 * sc));
  CK(ensure(P->lp_off, 8 * (sc + 1)));
  CK(ensure(P->tile_cnt, 8 * sc));
  CK(ensure(P->tile_off, 8 * (sc + 1)));
  CK(ensure(P->mkey, 8 * rc));
  CK(ensure(P->mval, 4 * rc));
  CK(ensure(P->mkey_sorted, 8 * rc));
  CK(ensure(P->mval_sorted, 4 * rc));
  CK(ensure(P->boxes, sizeof(TileBox) * (rc / kMT + sc + 1)));
  CK(ensure(P->tile_owner, sizeof(int) * (rc / kMT + sc + 1)));
  CK(ensure(P->gsoa, 8ll * 13 * rc));
  CK(ensure(P->fsoa, 4ll * 8 * rc));
  {
    // surviving tile pairs: worst case every pair of (rc/kMT + n_split) tiles; capped at
    // 2^24 entries (overflow falls back to inline filtering inside pair_tiles_kernel)
    const long long t = rc / kMT + sc + 1;
    long long want = t * (t + 1) / 2;
    if (want > (1ll << 24)) want = 1ll << 24;
    CK(ensure(P->tile_pairs, sizeof(int4) * want));
  }
  CK(ensure(P->regions_per_view, 4 * sc * V));
  {
    ZeroList z{};
    z.p[0] = P->cand_start.as<int>();
    z.p[1] = P->cand_end.as<int>();
    z.p[2] = P->cand_nvalid.as<int>();
    z.p[3] = P->regions_per_view.as<int>();
    z.n[0] = z.n[1] = z.n[2] = sc;
    z.n[3] = sc * V;
    z.count = 4;
    CK(launch_zero(z, s));
  }
  RangeArgs ra;
  ra.keys_sorted = P->keys_sorted.as<unsigned long long>();
  ra.vals_sorted = P->vals_sorted.as<int>();
  ra.n = n_regions;
  ra.shift_rank = bits_v + bits_b + bits_p;
  ra.bits_v = bits_v;
  ra.shift_view = bits_b + bits_p;
  ra.valid = P->valid.as<unsigned char>();
  ra.n_views = V;
  ra.cand_start = P->cand_start.as<int>();
  ra.cand_end = P->cand_end.as<int>();
  ra.cand_nvalid = P->cand_nvalid.as<int>();
  ra.regions_per_view = P->regions_per_view.as<int>();
  long long rgrid = (n_regions + 255) / 256;
  ra.grid = (unsigned)(rgrid < 1 ? 1 : (rgrid > 65535 ? 65535 : rgrid));
  if (P->child_pending) {   // valid flags (read by the ranges) and proposals
    CK(cudaStreamWaitEvent(s, P->ev_child, 0));
    P->child_pending = false;
  }
  CK(launch_ranges(ra, s));
  mark(P, "sort_ranges", s, n_regions > 0 ? 1 : 0);
  if (n_regions > 0) P->lib_calls += 1;

  // ---- per-candidate case, merge, cap (ref/adc.py:184-227)
  MergeArgs ma;
  ma.keys_sorted = P->keys_sorted.as<unsigned long long>();
  ma.vals_sorted = P->vals_sorted.as<int>();
  ma.n_regions = n_regions;
  ma.shift_rank = bits_v + bits_b + bits_p;
  ma.valid = P->valid.as<unsigned char>();
  ma.props = P->props.as<Proposal>();
  ma.split_list = P->split_list.as<int>();
  ma.cand_start = P->cand_start.as<int>();
  ma.cand_nvalid = P->cand_nvalid.as<int>();
  ma.dom_flag = P->dom_flag.as<unsigned char>();
  ma.opacity = g->opacity;
  ma.gamma_d = cfg->gamma_d;
  ma.gamma_c = cfg->gamma_c;
  ma.n_max = cfg->n_max;
  ma.small_max = P->large_threshold;
  ma.sel_huge = P->cap_huge;
  ma.props_s = P->props_s.as<Proposal>();
  ma.psrc = P->psrc.as<int>();
  ma.pcand = P->pcand.as<int>();
  ma.uf = P->uf.as<int>();
  ma.gkey = P->gkey.as<unsigned>();
  ma.gval = P->gval.as<int>();
  ma.gkey_sorted = P->gkey_sorted.as<unsigned>();
  ma.gval_sorted = P->gval_sorted.as<int>();
  ma.grp_first = P->grp_first.as<int>();
  ma.groups = P->groups.as<GroupRec>();
  ma.gpar = P->gpar.as<int>();
  ma.gext = P->gext.as<double>();
  ma.gfirst_of = P->gfirst_of.as<int>();
  ma.glist = P->glist.as<int>();
  ma.pstart = P->pstart.as<int>();
  ma.n_groups = P->n_groups.as<int>();
  ma.cand_case = P->cand_case.as<int>();
  ma.cand_props = P->cand_props.as<int>();
  ma.cand_merged = P->cand_merged.as<int>();
  ma.cand_ins = P->cand_ins.as<int>();
  ma.small_list = P->small_list.as<int>();
  ma.large_list = P->large_list.as<int>();
  ma.work_cnt = P->work_cnt.as<unsigned long long>();
  ma.work_off = P->work_off.as<unsigned long long>();
  ma.children = P->children.as<float>();
  ma.extent = extent;
  ma.large_of = P->large_of.as<int>();
  ma.lp_cnt = P->lp_cnt.as<unsigned long long>();
  ma.lp_off = P->lp_off.as<unsigned long long>();
  ma.tile_cnt = P->tile_cnt.as<unsigned long long>();
  ma.tile_off = P->tile_off.as<unsigned long long>();
  ma.mkey = P->mkey.as<unsigned long long>();
  ma.mval = P->mval.as<int>();
  ma.mkey_sorted = P->mkey_sorted.as<unsigned long long>();
  ma.mval_sorted = P->mval_sorted.as<int>();
  ma.boxes = P->boxes.as<TileBox>();
  ma.tile_owner = P->tile_owner.as<int>();
  ma.gsoa = P->gsoa.as<double>();
  ma.fsoa = P->fsoa.as<float>();
  ma.soa_cap = rc;
  ma.tile_pairs = P->tile_pairs.as<int4>();
  ma.tile_pairs_cap = (long long)(P->tile_pairs.bytes / sizeof(int4));
  ma.ctr = ctr;
  ma.grid = (unsigned)(P->sm_count * 8);
  ma.own = nullptr;
  if (P->pshard_world > 1 && n_split > 0) {
    CK(launch_shard_range(P->cand_nvalid.as<int>(), n_split, P->pshard_rank, P->pshard_world, &ctr->shard_lo, s));
    ma.own = &ctr->shard_lo;
    P->launches += 2;
  }
  if (n_split > 0) {
    ScanState sst3;
    st = scan_state(P, P->scan3_val, P->scan3_flag, rc, &sst3);
    if (st != ADPS_OK) return st;
    CK(launch_merge_prepare(ma, n_split, sst3, s));
    mark(P, "merge_prepare", s, 3);
    // fork: the small parents' gates and the survivor scan (it only needs the
    // cases) run on the second stream while the large parents are gated
    CK(cudaEventRecord(P->ev_fork, s));
    CK(cudaStreamWaitEvent(P->aux, P->ev_fork, 0));
    CK(launch_small_pairs(ma, P->aux));
    CK(cudaEventRecord(P->ev_small, P->aux));
    {
      OffsetArgs ka;
      ka.n = n;
      ka.cls = P->cls.as<unsigned char>();
      ka.cand_rank = P->cand_rank.as<int>();
      ka.cand_case = P->cand_case.as<int>();
      ka.cand_ins = P->cand_ins.as<int>();
      ka.ins_off = P->ins_off.as<int>();
      ka.fb_ord = P->fb_ord.as<int>();
      ka.keep_pos = P->keep_pos.as<int>();
      ka.ctr = ctr;
      ka.n_split_dev = &ctr->n_split;
      CK(launch_offsets_keep(ka, sst, P->aux));
      CK(cudaEventRecord(P->ev_keep, P->aux));
      P->keep_pending = true;
    }
    CK(launch_large_offsets(ma, s));
    mark(P, "merge_small_gates", s, 3);   // small gates + survivor scan (second stream), large offsets
    if (n_regions > 0) {
      CK(launch_merge_morton(ma, rc, s));
      // large parents have > small_max proposals each, so their index l is below
      // n_regions / (small_max + 1): fewer key bits, fewer radix passes
      const long long l_bound = std::min<long long>(n_split, n_regions / (P->large_threshold + 1));
      const int mbits = 3 * kMortonBits + ceil_log2((unsigned long long)l_bound + 2);
      CK(cub_sort_pairs(P, ma.mkey, ma.mkey_sorted, ma.mval, ma.mval_sorted, rc, mbits, s));
      CK(launch_merge_tile_gates(ma, s));
      mark(P, "merge_tile_gates", s, 4);   // morton, box, filter, pair tiles
    }
    CK(cudaStreamWaitEvent(s, P->ev_small, 0));   // join: all unions are in before the groups
    if (n_regions > 0) {
      CK(launch_merge_flatten(ma, rc, s));
      const int gbits = ceil_log2((unsigned long long)rc + 2);
      CK(cub_sort_pairs(P, ma.gkey, ma.gkey_sorted, ma.gval, ma.gval_sorted, rc, gbits, s));
      CK(launch_merge_groups(ma, rc, sst3, s, P->timing ? nullptr : P->aux, P->ev_cfork, P->ev_child));
      mark(P, "merge_groups", s, 5);
      CK(launch_merge_cap(ma, rc, s, P->aux, P->ev_fork, P->ev_small));
      mark(P, "merge_cap", s, 3);
    }
  }
  return ADPS_OK;
}

// the offsets (ref/adc.py:229-244) on the device: everything phase 2 needs,
// with the counts still on the device (phase1_finish_collect reads them)
static adps_status phase1_finish_launch(adps_plan* P, cudaStream_t s) {
  adps_status st = ADPS_OK;
  const long long n = P->cx.n;
  const long long nn = n > 0 ? n : 1;
  Counters* ctr = P->ctr.as<Counters>();
  ScanState sst, sst2;
  st = scan_state(P, P->scan_val, P->scan_flag, nn, &sst);
  if (st != ADPS_OK) return st;
  const long long n_split = (long long)P->ctr_host->n_split;
  const long long sc = n_split > 0 ? n_split : 1;
  // ---- offsets (ref/adc.py:229-244)
  st = scan_state(P, P->scan2_val, P->scan2_flag, sc, &sst2);
  if (st != ADPS_OK) return st;
  OffsetArgs oa;
  oa.n = n;
  oa.cls = P->cls.as<unsigned char>();
  oa.cand_rank = P->cand_rank.as<int>();
  oa.cand_case = P->cand_case.as<int>();
  oa.cand_ins = P->cand_ins.as<int>();
  oa.ins_off = P->ins_off.as<int>();
  oa.fb_ord = P->fb_ord.as<int>();
  oa.keep_pos = P->keep_pos.as<int>();
  oa.ctr = ctr;
  oa.n_split_dev = &ctr->n_split;
  CK(launch_offsets_cand(oa, n_split, sst2, s));
  CK(launch_deferred_normals(P));
  if (P->norm_pending) {   // join the fallback normals (read by phase 2; consumed count below)
    CK(cudaStreamWaitEvent(s, P->ev_norm, 0));
    P->norm_pending = false;
  }
  if (P->keep_pending) {   // join the survivor scan started with the merge
    CK(cudaStreamWaitEvent(s, P->ev_keep, 0));
    P->keep_pending = false;
  } else {
    CK(launch_offsets_keep(oa, sst, s));
  }
  mark(P, "offsets", s, 2);
  return ADPS_OK;
}

// the host side of the finish: one copy of the counters, one synchronisation
static adps_status phase1_finish_collect(adps_plan* P, cudaStream_t s, adps_counts* counts) {
  const adps_gaussians* g = &P->cx.g;
  const long long n = P->cx.n;
  const adps_config* cfg = &P->cx.cfg;
  const int V = P->v_glob, H = P->cx.H, W = P->cx.W;
  Counters* ctr = P->ctr.as<Counters>();
  (void)g;
  const long long n_regions = P->n_regions_cur;
  const long long n_split = (long long)P->ctr_host->n_split;
  const long long n_clone = (long long)P->ctr_host->n_clone;
  CK(cudaMemcpyAsync(P->ctr_host, ctr, sizeof(Counters), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  const Counters& C = *P->ctr_host;
  adps_counts& K = P->counts;
  K.n_before = n;
  K.n_split = n_split;
  K.n_clone = n_clone;
  K.n_keep = (long long)C.n_keep;
  K.n_inserted = (long long)C.n_inserted;
  K.n_out = K.n_keep + K.n_inserted + n_clone;
  K.n_fallback = (long long)C.n_fallback;
  K.n_reset = (long long)C.n_reset;
  K.n_children = (long long)C.n_children;
  K.n_regions = n_regions;
  K.n_proposals = (long long)C.n_proposals;
  K.merge_edges = (long long)C.merge_edges;
  K.n_partials = (long long)C.n_partials;
  K.degenerate_ray = C.degenerate ? 1 : 0;
  *counts = K;
  P->n = n;
  P->V = V;
  P->H = H;
  P->W = W;
  P->eta = cfg->eta;
  P->sh_k = g->sh_rest_k;
  P->fb_children = 2;
  P->have_phase1 = true;
  if (C.degenerate) return fail(ADPS_DEGENERATE_RAY, "quadratic coefficient underflows (DegenerateRayError)");
  return ADPS_OK;
}

static adps_status phase1_finish(adps_plan* P, cudaStream_t s, adps_counts* counts) {
  adps_status st = phase1_finish_launch(P, s);
  if (st != ADPS_OK) return st;
  return phase1_finish_collect(P, s, counts);
}

static adps_status phase1_merge(adps_plan* P, cudaStream_t s, adps_counts* counts) {
  adps_status st = phase1_merge_part(P, s);
  if (st != ADPS_OK) return st;
  return phase1_finish(P, s, counts);
}

extern "C" adps_status adps_step_phase1_end(adps_plan* P, void* stream_v, adps_counts* counts) {
  if (!P || !counts) return fail(ADPS_INVALID_ARG, "NULL argument");
  if (!P->have_begin) return fail(ADPS_BAD_STATE, "phase1_end without phase1_begin");
  P->have_begin = false;
  cudaStream_t s = (cudaStream_t)stream_v;
  long long nr = 0;
  adps_status st = phase1_local(P, s, &nr, /*defer_child=*/true);
  if (st == ADPS_OK) st = phase1_merge(P, s, counts);
  if (st != ADPS_OK) drop_pending_normals(P);
  return st;
}

extern "C" adps_status adps_step_phase1_local(adps_plan* P, void* stream_v, int64_t* n_regions) {
  if (!P || !n_regions) return fail(ADPS_INVALID_ARG, "NULL argument");
  if (!P->have_begin) return fail(ADPS_BAD_STATE, "phase1_local without phase1_begin");
  P->have_begin = false;
  long long nr = 0;
  adps_status st = phase1_local(P, (cudaStream_t)stream_v, &nr);
  if (st != ADPS_OK) {
    drop_pending_normals(P);
    return st;
  }
  *n_regions = nr;
  P->have_local = true;
  return ADPS_OK;
}

extern "C" adps_status adps_step_phase1_import(adps_plan* P, void* stream_v, const adps_region_record* regions,
                                               const void* proposals, const uint8_t* valid, int64_t n) {
  if (!P) return fail(ADPS_INVALID_ARG, "plan is NULL");
  if (!P->have_local) return fail(ADPS_BAD_STATE, "phase1_import without phase1_local");
  if (n < 0 || (n > 0 && (!regions || !proposals || !valid))) return fail(ADPS_INVALID_ARG, "bad records");
  CK(cudaSetDevice(P->device));
  cudaStream_t s = (cudaStream_t)stream_v;
  const long long rc = n > 0 ? n : 1;
  if (P->region_cap < rc) {
    P->region_cap = rc;
    CK(ensure(P->regions, sizeof(RegionRec) * rc));
  }
  CK(ensure(P->props, sizeof(Proposal) * rc));
  CK(ensure(P->valid, rc));
  CK(ensure(P->keys, 8 * rc));
  CK(ensure(P->vals, 4 * rc));
  CK(ensure(P->keys_sorted, 8 * rc));
  CK(ensure(P->vals_sorted, 4 * rc));
  CK(ensure(P->idx, 4 * rc));
  CK(ensure(P->uf, 4 * rc));
  CK(ensure(P->groups, sizeof(GroupRec) * rc));
  CK(ensure(P->children, sizeof(float) * 14 * rc));
  if (n > 0) {
    CK(cudaMemcpyAsync(P->regions.p, regions, sizeof(RegionRec) * n, cudaMemcpyDeviceToDevice, s));
    CK(cudaMemcpyAsync(P->props.p, proposals, sizeof(Proposal) * n, cudaMemcpyDeviceToDevice, s));
    CK(cudaMemcpyAsync(P->valid.p, valid, n, cudaMemcpyDeviceToDevice, s));
    const adps_config* cfg = &P->cx.cfg;
    const long long hw = (long long)P->cx.H * P->cx.W;
    CK(launch_region_keys(P->regions.as<RegionRec>(), n, P->cand_rank.as<int>(),
                          ceil_log2((unsigned long long)P->v_glob), ceil_log2((unsigned long long)cfg->l_bands),
                          ceil_log2((unsigned long long)hw), P->keys.as<unsigned long long>(), P->vals.as<int>(), s));
    P->launches += 1;
  }
  Counters* ctr = P->ctr.as<Counters>();
  const unsigned long long nu = (unsigned long long)n;
  CK(cudaMemcpyAsync(&ctr->n_regions, &nu, sizeof(nu), cudaMemcpyHostToDevice, s));
  CK(cudaStreamSynchronize(s));
  P->n_regions_cur = n;
  return ADPS_OK;
}

extern "C" adps_status adps_step_phase1_merge(adps_plan* P, void* stream_v, adps_counts* counts) {
  if (!P || !counts) return fail(ADPS_INVALID_ARG, "NULL argument");
  if (!P->have_local) return fail(ADPS_BAD_STATE, "phase1_merge without phase1_local");
  P->have_local = false;
  cudaStream_t s = (cudaStream_t)stream_v;
  if (P->pshard_world <= 1) return phase1_merge(P, s, counts);
  // parent-sharded: merge this rank's candidates, then wait for the exchange
  adps_status st = phase1_merge_part(P, s);
  if (st != ADPS_OK) return st;
  Counters* ctr = P->ctr.as<Counters>();
  CK(cudaMemcpyAsync(P->ctr_host, ctr, sizeof(Counters), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  const long long n_split = (long long)P->ctr_host->n_split;
  long long lo = (long long)P->ctr_host->shard_lo, hi = (long long)P->ctr_host->shard_hi;
  if (n_split == 0 || hi <= lo) lo = hi = 0;
  P->shard_k[0] = lo;
  P->shard_k[1] = hi;
  long long pst[2] = {0, 0};
  if (hi > lo) {
    pst[0] = (long long)P->ctr_host->shard_plo;
    pst[1] = (long long)P->ctr_host->shard_phi;
  }
  P->shard_p[0] = pst[0];
  P->shard_p[1] = pst[1];
  *counts = adps_counts{};
  counts->n_split = n_split;
  counts->merge_edges = (long long)P->ctr_host->merge_edges;
  counts->n_children = (long long)P->ctr_host->n_children;
  P->have_merge_part = true;
  return ADPS_OK;
}

extern "C" adps_status adps_set_parent_sharding(adps_plan* P, int32_t rank, int32_t world) {
  if (!P) return fail(ADPS_INVALID_ARG, "plan is NULL");
  if (world < 1 || rank < 0 || rank >= world) return fail(ADPS_INVALID_ARG, "bad parent sharding");
  P->pshard_rank = rank;
  P->pshard_world = world;
  return ADPS_OK;
}

extern "C" adps_status adps_get_shard(adps_plan* P, int64_t* k_lo, int64_t* k_hi, int64_t* p_lo, int64_t* p_hi) {
  if (!P || !k_lo || !k_hi || !p_lo || !p_hi) return fail(ADPS_INVALID_ARG, "NULL argument");
  if (!P->have_merge_part) return fail(ADPS_BAD_STATE, "no parent-sharded merge pending");
  *k_lo = P->shard_k[0];
  *k_hi = P->shard_k[1];
  *p_lo = P->shard_p[0];
  *p_hi = P->shard_p[1];
  return ADPS_OK;
}

extern "C" adps_status adps_step_phase1_finish(adps_plan* P, void* stream_v, int64_t merge_edges, int64_t n_children,
                                               adps_counts* counts) {
  if (!P || !counts) return fail(ADPS_INVALID_ARG, "NULL argument");
  if (!P->have_merge_part) return fail(ADPS_BAD_STATE, "phase1_finish without a parent-sharded merge");
  P->have_merge_part = false;
  CK(cudaSetDevice(P->device));
  cudaStream_t s = (cudaStream_t)stream_v;
  Counters* ctr = P->ctr.as<Counters>();
  const unsigned long long me = (unsigned long long)merge_edges, nc = (unsigned long long)n_children;
  CK(cudaMemcpyAsync(&ctr->merge_edges, &me, sizeof(me), cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(&ctr->n_children, &nc, sizeof(nc), cudaMemcpyHostToDevice, s));
  return phase1_finish(P, s, counts);
}

static adps_status copy_report_impl(adps_plan* P, cudaStream_t s, int32_t* dst, long long n_split, long long n_clone,
                                    long long V);

// EmitArgs of phase 2 from the plan's phase-1 state (counts filled by the caller)
static EmitArgs emit_args(adps_plan* P, const adps_gaussians* g, const double* fallback_normals,
                          const adps_gaussians_out* out, int64_t* index_map, int32_t* child_parent,
                          int64_t* insert_offset) {
  EmitArgs ea;
  ea.g = to_in(g);
  ea.n = P->n;
  ea.keep_pos = P->keep_pos.as<int>();
  ea.split_list = P->split_list.as<int>();
  ea.clone_list = P->clone_list.as<int>();
  ea.cand_case = P->cand_case.as<int>();
  ea.cand_merged = P->cand_merged.as<int>();
  ea.cand_start = P->pstart.as<int>();   // children of parent k live at [pstart[k], +N_k)
  ea.ins_off = P->ins_off.as<int>();
  ea.fb_ord = P->fb_ord.as<int>();
  ea.children = P->children.as<float>();
  ea.normals = fallback_normals;
  ea.eta = P->eta;
  ea.fb_children = P->fb_children;
  ea.mu = out->mu;
  ea.scale = out->scale;
  ea.rot = out->rot;
  ea.opacity = out->opacity;
  ea.sh_dc = out->sh_dc;
  ea.sh_rest = out->sh_rest;
  ea.index_map = (long long*)index_map;
  ea.child_parent = child_parent;
  ea.insert_offset = (long long*)insert_offset;
  return ea;
}

static adps_status check_outputs(adps_plan* P, const adps_gaussians* g, const adps_gaussians_out* out,
                                 const int64_t* index_map) {
  if (!out || !index_map || !out->mu || !out->scale || !out->rot || !out->opacity || !out->sh_dc)
    return fail(ADPS_INVALID_ARG, "outputs are NULL");
  if (g->sh_rest_k != P->sh_k || out->sh_rest_k != P->sh_k)
    return fail(ADPS_INVALID_ARG, "sh_rest_k differs between phases/outputs");
  if (P->sh_k > 0 && !out->sh_rest) return fail(ADPS_INVALID_ARG, "out.sh_rest is NULL");
  return ADPS_OK;
}

extern "C" adps_status adps_step_phase2(adps_plan* P, void* stream_v, const adps_gaussians* g,
                                        const double* fallback_normals, adps_gaussians_out* out,
                                        int64_t* index_map, int32_t* child_parent, int64_t* insert_offset) {
  if (!P) return fail(ADPS_INVALID_ARG, "plan is NULL");
  if (!P->have_phase1) return fail(ADPS_BAD_STATE, "phase 2 without a successful phase 1");
  adps_status st = check_gaussians(g, P->n);
  if (st != ADPS_OK) return st;
  if (P->counts.n_out == 0) return ADPS_OK;   // nothing to write (e.g. an empty scene)
  st = check_outputs(P, g, out, index_map);
  if (st != ADPS_OK) return st;
  if (P->counts.n_fallback > 0 && !fallback_normals) return fail(ADPS_INVALID_ARG, "fallback normals are NULL");
  CK(cudaSetDevice(P->device));
  cudaStream_t s = (cudaStream_t)stream_v;
  mark_start(P, s, false);
  EmitArgs ea = emit_args(P, g, fallback_normals, out, index_map, child_parent, insert_offset);
  ea.n_split = P->counts.n_split;
  ea.n_clone = P->counts.n_clone;
  ea.n_keep = P->counts.n_keep;
  ea.n_inserted = P->counts.n_inserted;
  CK(launch_emit(ea, s, P->timing ? nullptr : P->aux, P->ev_fork, P->ev_small));
  mark(P, "emit", s, (P->n > 0 ? 1 : 0) + ((P->counts.n_split + P->counts.n_clone) > 0 ? 1 : 0));
  return ADPS_OK;
}

extern "C" adps_status adps_step_capacity(adps_plan* P, int64_t* out_cap, int64_t* app_cap) {
  if (!P || !out_cap || !app_cap) return fail(ADPS_INVALID_ARG, "NULL argument");
  if (!P->have_begin) return fail(ADPS_BAD_STATE, "capacity without phase1_begin");
  // a split parent leaves the survivors unless reset and inserts at most
  // max(n_max + 1, 2) rows (N_i <= n_max children + the parent copy, or the 2
  // fallback children); clones append one row each (ref/adc.py:198-244)
  const long long n = P->cx.n;
  const long long n_split = (long long)P->ctr_host->n_split;
  const long long n_clone = (long long)P->ctr_host->n_clone;
  const long long per = std::max<long long>((long long)P->cx.cfg.n_max + 1, 2);
  *app_cap = n_split * per + n_clone;
  *out_cap = n - n_split + *app_cap;   // (a reset parent stays a survivor: its 1 row <= per)
  return ADPS_OK;
}

extern "C" adps_status adps_step_phase1_end_emit(adps_plan* P, void* stream_v, const adps_gaussians* g,
                                                 const double* fallback_normals, adps_gaussians_out* out,
                                                 int64_t* index_map, int32_t* child_parent, int64_t* insert_offset,
                                                 int64_t out_cap, int64_t app_cap, int32_t* report,
                                                 adps_counts* counts) {
  if (!P || !counts) return fail(ADPS_INVALID_ARG, "NULL argument");
  if (!P->have_begin) return fail(ADPS_BAD_STATE, "phase1_end_emit without phase1_begin");
  adps_status st = check_gaussians(g, P->cx.n);
  if (st != ADPS_OK) return st;
  if (g->mu != P->cx.g.mu || g->opacity != P->cx.g.opacity)
    return fail(ADPS_INVALID_ARG, "Gaussians differ from phase1_begin's");
  int64_t need_out = 0, need_app = 0;
  st = adps_step_capacity(P, &need_out, &need_app);
  if (st != ADPS_OK) return st;
  if (out_cap < need_out || app_cap < need_app)
    return fail(ADPS_INVALID_ARG, "output capacity %lld/%lld below the step bound %lld/%lld", (long long)out_cap,
                (long long)app_cap, (long long)need_out, (long long)need_app);
  const bool any_out = need_out > 0;
  P->sh_k = g->sh_rest_k;
  if (any_out) {
    st = check_outputs(P, g, out, index_map);
    if (st != ADPS_OK) return st;
  }
  if (P->ctr_host->n_fallback_pre > 0 && !fallback_normals)
    return fail(ADPS_INVALID_ARG, "fallback normals are NULL");
  P->have_begin = false;
  cudaStream_t s = (cudaStream_t)stream_v;
  long long nr = 0;
  st = phase1_local(P, s, &nr, /*defer_child=*/true);
  if (st == ADPS_OK) st = phase1_merge_part(P, s);
  if (st == ADPS_OK) st = phase1_finish_launch(P, s);
  if (st != ADPS_OK) {
    drop_pending_normals(P);
    return st;
  }
  // phase 2 on the same stream, before the host reads a single count
  P->n = P->cx.n;
  P->eta = P->cx.cfg.eta;
  P->fb_children = 2;
  if (any_out) {
    Counters* ctr = P->ctr.as<Counters>();
    mark_start(P, s, false);
    EmitArgs ea = emit_args(P, g, fallback_normals, out, index_map, child_parent, insert_offset);
    ea.n_split = (long long)P->ctr_host->n_split;
    ea.n_clone = (long long)P->ctr_host->n_clone;
    ea.dev_keep = &ctr->n_keep;
    ea.dev_inserted = &ctr->n_inserted;
    ea.n_ins_max = need_app - ea.n_clone;
    ea.out_cap = out_cap;
    ea.app_cap = app_cap;
    CK(launch_emit(ea, s, P->timing ? nullptr : P->aux, P->ev_fork, P->ev_small));
    mark(P, "emit", s, (P->n > 0 ? 1 : 0) + ((ea.n_split + ea.n_clone) > 0 ? 1 : 0));
  }
  if (report) {   // the SplitReport arrays (adps_copy_report's layout), before the sync too
    st = copy_report_impl(P, s, report, (long long)P->ctr_host->n_split, (long long)P->ctr_host->n_clone, P->v_glob);
    if (st != ADPS_OK) return st;
  }
  st = phase1_finish_collect(P, s, counts);
  if (st != ADPS_OK) return st;
  if (counts->n_out > out_cap || counts->n_out - counts->n_keep > app_cap)
    return fail(ADPS_INTERNAL, "step outgrew its capacity bound (%lld rows)", (long long)counts->n_out);
  return ADPS_OK;
}

extern "C" adps_status adps_get_report(adps_plan* P, adps_report* r) {
  if (!P || !r) return fail(ADPS_INVALID_ARG, "NULL argument");
  if (!P->have_phase1) return fail(ADPS_BAD_STATE, "no phase 1 result");
  r->cand_index = P->split_list.as<int>();
  r->cand_case = P->cand_case.as<int>();
  r->cand_proposals = P->cand_props.as<int>();
  r->cand_merged = P->cand_merged.as<int>();
  r->regions_per_view = P->regions_per_view.as<int>();
  r->clone_index = P->clone_list.as<int>();
  r->n_views = P->V;
  return ADPS_OK;
}

static adps_status copy_report_impl(adps_plan* P, cudaStream_t s, int32_t* dst, long long n_split, long long n_clone,
                                    long long V) {
  const void* src[6] = {P->split_list.p, P->cand_case.p, P->cand_props.p, P->cand_merged.p, P->regions_per_view.p,
                        P->clone_list.p};
  const long long len[6] = {n_split, n_split, n_split, n_split, n_split * V, n_clone};
  long long off = 0;
  for (int i = 0; i < 6; ++i) {
    if (len[i] > 0) CK(cudaMemcpyAsync(dst + off, src[i], 4 * len[i], cudaMemcpyDeviceToDevice, s));
    off += len[i];
  }
  return ADPS_OK;
}

extern "C" adps_status adps_copy_report(adps_plan* P, void* stream_v, int32_t* dst, int64_t n_split, int64_t n_clone) {
  if (!P || (!dst && n_split + n_clone > 0)) return fail(ADPS_INVALID_ARG, "NULL argument");
  if (!P->have_phase1) return fail(ADPS_BAD_STATE, "no phase 1 result");
  if (n_split < 0 || n_clone < 0) return fail(ADPS_INVALID_ARG, "negative count");
  if (n_split > (long long)P->counts.n_split || n_clone > (long long)P->counts.n_clone)
    return fail(ADPS_INVALID_ARG, "counts exceed the last phase 1 (%lld split, %lld clone)",
                (long long)P->counts.n_split, (long long)P->counts.n_clone);
  CK(cudaSetDevice(P->device));
  return copy_report_impl(P, (cudaStream_t)stream_v, dst, n_split, n_clone, P->V);
}

extern "C" adps_status adps_get_regions(adps_plan* P, const adps_region_record** records,
                                        const int32_t** order, const uint8_t** valid, const double** stats,
                                        const double** child, int64_t* n) {
  if (!P || !records || !order || !valid || !stats || !child || !n) return fail(ADPS_INVALID_ARG, "NULL argument");
  if (!P->have_phase1) return fail(ADPS_BAD_STATE, "no phase 1 result");
  static_assert(sizeof(adps_region_record) == sizeof(RegionRec), "record layout");
  *records = reinterpret_cast<const adps_region_record*>(P->regions.p);
  *order = P->vals_sorted.as<int32_t>();
  *valid = P->valid.as<uint8_t>();
  *stats = P->dbg_records ? P->dbg_stats.as<double>() : nullptr;
  *child = P->dbg_records ? P->dbg_child.as<double>() : nullptr;
  *n = P->counts.n_regions;
  return ADPS_OK;
}

extern "C" adps_status adps_set_debug_maps(adps_plan* P, uint8_t* m_out, uint8_t* b_out) {
  if (!P) return fail(ADPS_INVALID_ARG, "plan is NULL");
  if ((m_out == nullptr) != (b_out == nullptr)) return fail(ADPS_INVALID_ARG, "set both or neither");
  P->dbg_m = m_out;
  P->dbg_b = b_out;
  return ADPS_OK;
}

extern "C" adps_status adps_set_debug_records(adps_plan* P, int32_t enabled) {
  if (!P) return fail(ADPS_INVALID_ARG, "plan is NULL");
  P->dbg_records = enabled != 0;
  return ADPS_OK;
}

extern "C" adps_status adps_set_timing(adps_plan* P, int32_t enabled) {
  if (!P) return fail(ADPS_INVALID_ARG, "plan is NULL");
  P->timing = enabled != 0;
  return ADPS_OK;
}

extern "C" adps_status adps_get_timing(adps_plan* P, double* ms, int32_t max_entries, int32_t* n_entries,
                                       const char** names) {
  if (!P || !n_entries) return fail(ADPS_INVALID_ARG, "NULL argument");
  int n = 0;
  if (P->n_marks > 0) CK(cudaEventSynchronize(P->ev[P->n_marks - 1]));
  for (int i = 1; i < P->n_marks && n < max_entries; ++i) {
    if (strcmp(P->names[i], "start") == 0) continue;
    float t = 0.f;
    CK(cudaEventElapsedTime(&t, P->ev[i - 1], P->ev[i]));
    if (ms) ms[n] = t;
    if (names) names[n] = P->names[i];
    ++n;
  }
  *n_entries = n;
  return ADPS_OK;
}

extern "C" adps_status adps_set_view_sharding(adps_plan* P, int32_t view_offset, int32_t view_stride,
                                              int32_t n_views_global) {
  if (!P) return fail(ADPS_INVALID_ARG, "plan is NULL");
  if (view_offset < 0 || view_stride < 1 || n_views_global < 0) return fail(ADPS_INVALID_ARG, "bad view sharding");
  P->view_offset = view_offset;
  P->view_stride = view_stride;
  P->v_global_cfg = n_views_global;
  return ADPS_OK;
}

extern "C" adps_status adps_get_buffer(adps_plan* P, int32_t which, void** ptr, int64_t* count, int64_t* elem_bytes) {
  if (!P || !ptr || !count || !elem_bytes) return fail(ADPS_INVALID_ARG, "NULL argument");
  switch (which) {
    case ADPS_BUF_DOM_FLAG:
      *ptr = P->dom_flag.p;
      *count = P->cx.n;
      *elem_bytes = 1;
      return ADPS_OK;
    case ADPS_BUF_REGIONS:
      *ptr = P->regions.p;
      *count = P->n_regions_cur;
      *elem_bytes = sizeof(RegionRec);
      return ADPS_OK;
    case ADPS_BUF_PROPOSALS:
      *ptr = P->props.p;
      *count = P->n_regions_cur;
      *elem_bytes = sizeof(Proposal);
      return ADPS_OK;
    case ADPS_BUF_VALID:
      *ptr = P->valid.p;
      *count = P->n_regions_cur;
      *elem_bytes = 1;
      return ADPS_OK;
    case ADPS_BUF_LO:
      *ptr = P->lo.p;
      *count = P->cx.V;
      *elem_bytes = 8;
      return ADPS_OK;
    case ADPS_BUF_THRESHOLDS:
      *ptr = P->thr.p;
      *count = (int64_t)P->cx.V * P->cx.cfg.l_bands;
      *elem_bytes = 8;
      return ADPS_OK;
    case ADPS_BUF_CAND_MERGED:
      *ptr = P->cand_merged.p;
      *count = P->ctr_host ? (int64_t)P->ctr_host->n_split : 0;
      *elem_bytes = 4;
      return ADPS_OK;
    case ADPS_BUF_CAND_INS:
      *ptr = P->cand_ins.p;
      *count = P->ctr_host ? (int64_t)P->ctr_host->n_split : 0;
      *elem_bytes = 4;
      return ADPS_OK;
    case ADPS_BUF_CHILDREN:
      *ptr = P->children.p;
      *count = P->n_regions_cur;
      *elem_bytes = 14 * sizeof(float);
      return ADPS_OK;
    default:
      return fail(ADPS_INVALID_ARG, "unknown buffer %d", which);
  }
}

extern "C" adps_status adps_step_phase1_refresh(adps_plan* P, void* stream_v, adps_counts* counts) {
  if (!P || !counts) return fail(ADPS_INVALID_ARG, "NULL argument");
  if (!P->have_begin) return fail(ADPS_BAD_STATE, "phase1_refresh without phase1_begin");
  CK(cudaSetDevice(P->device));
  cudaStream_t s = (cudaStream_t)stream_v;
  Counters* ctr = P->ctr.as<Counters>();
  CK(cudaMemsetAsync(&ctr->n_fallback_pre, 0, sizeof(unsigned long long), s));
  CK(launch_fallback_count(P->split_list.as<int>(), P->dom_flag.as<unsigned char>(), ctr, P->sm_count, s));
  P->launches += 1;
  CK(cudaMemcpyAsync(P->ctr_host, ctr, sizeof(Counters), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  counts->n_fallback = (long long)P->ctr_host->n_fallback_pre;
  return ADPS_OK;
}

extern "C" adps_status adps_set_param(adps_plan* P, int32_t key, int64_t value) {
  if (!P) return fail(ADPS_INVALID_ARG, "plan is NULL");
  if (key == ADPS_PARAM_LARGE_THRESHOLD) {
    if (value < 0 || value > 1000000) return fail(ADPS_INVALID_ARG, "large threshold out of range");
    P->large_threshold = (int)value;
    return ADPS_OK;
  }
  if (key == ADPS_PARAM_CAP_HUGE) {
    if (value < 64 || value > 1000000000) return fail(ADPS_INVALID_ARG, "cap huge threshold must be in [64, 1e9]");
    P->cap_huge = (int)value;
    return ADPS_OK;
  }
  if (key == ADPS_PARAM_PIPELINE_CHUNKS) {
    if (value < 1 || value > adps_plan::kMaxChunks) return fail(ADPS_INVALID_ARG, "pipeline chunks must be in [1,16]");
    P->pipeline_chunks = (int)value;
    return ADPS_OK;
  }
  if (key == ADPS_PARAM_INPUT_BLOCKS_PER_SM) {
    if (value < 0 || value > 64) return fail(ADPS_INVALID_ARG, "input blocks per SM must be in [0,64]");
    P->input_blocks_per_sm = (int)value;
    return ADPS_OK;
  }
  if (key == ADPS_PARAM_RENDER_PAIR_CAP) {
    if (value < 1 || value > 0x7fffffffLL) return fail(ADPS_INVALID_ARG, "pair capacity must be in [1, 2^31)");
    P->dup_cap = value;   // (grown again by the first render that overflows it)
    return ADPS_OK;
  }
  if (key == ADPS_PARAM_RENDER_BINNING) {
    if (value < 0 || value > 1)
      return fail(ADPS_INVALID_ARG, "render binning must be 0 (64-bit depth sort) or 1 (32-bit keys + fix-up)");
    P->render_fast = (int)value;
    return ADPS_OK;
  }
  if (key == ADPS_PARAM_RAW_CACHE) {
    if (value < 0 || value > 1) return fail(ADPS_INVALID_ARG, "raw cache must be 0 or 1");
    P->raw_cache = (int)value;
    return ADPS_OK;
  }
  if (key == ADPS_PARAM_TILE_PATH) {
    if (value < 0 || value > 3)
      return fail(ADPS_INVALID_ARG, "tile path must be 0 (bit planes, words pass), 1 (block), 2 (warp, fp64 raw) "
                                    "or 3 (bit planes computed per tile)");
    P->tile_path = (int)value;
    return ADPS_OK;
  }
  return fail(ADPS_INVALID_ARG, "unknown parameter %d", key);
}

extern "C" adps_status adps_get_param(adps_plan* P, int32_t key, int64_t* value) {
  if (!P || !value) return fail(ADPS_INVALID_ARG, "NULL argument");
  switch (key) {
    case ADPS_PARAM_LARGE_THRESHOLD: *value = P->large_threshold; return ADPS_OK;
    case ADPS_PARAM_CAP_HUGE: *value = P->cap_huge; return ADPS_OK;
    case ADPS_PARAM_TILE_PATH: *value = P->tile_path; return ADPS_OK;
    case ADPS_PARAM_RAW_CACHE: *value = P->raw_cache; return ADPS_OK;
    case ADPS_PARAM_RENDER_BINNING: *value = P->render_fast; return ADPS_OK;
    case ADPS_PARAM_RENDER_PAIR_CAP: *value = P->dup_cap; return ADPS_OK;
    case ADPS_PARAM_PIPELINE_CHUNKS: *value = P->pipeline_chunks; return ADPS_OK;
    case ADPS_PARAM_INPUT_BLOCKS_PER_SM: *value = P->input_blocks_per_sm; return ADPS_OK;
    case ADPS_PARAM_STAT_TILE_PAIRS: *value = P->ctr_host ? (int64_t)P->ctr_host->n_tile_pairs : 0; return ADPS_OK;
    case ADPS_PARAM_STAT_GATES: *value = P->ctr_host ? (int64_t)P->ctr_host->stat_gates : 0; return ADPS_OK;
    case ADPS_PARAM_STAT_GATES_PASSED: *value = P->ctr_host ? (int64_t)P->ctr_host->stat_pass : 0; return ADPS_OK;
    case ADPS_PARAM_DEFERRED_TILES: *value = P->ctr_host ? (int64_t)P->ctr_host->n_deferred : 0; return ADPS_OK;
    case ADPS_PARAM_NORMALS_CONSUMED:
      *value = P->ctr_host ? (int64_t)P->ctr_host->normals_consumed : 0;
      return ADPS_OK;
    case ADPS_PARAM_NORMALS_STATUS: *value = P->ctr_host ? (int64_t)P->ctr_host->normals_status : 0; return ADPS_OK;
    default: return fail(ADPS_INVALID_ARG, "unknown parameter %d", key);
  }
}

extern "C" adps_status adps_get_launch_count(adps_plan* P, int64_t* kernels, int64_t* library_calls) {
  if (!P || !kernels || !library_calls) return fail(ADPS_INVALID_ARG, "NULL argument");
  *kernels = P->launches;
  *library_calls = P->lib_calls;
  return ADPS_OK;
}

extern "C" adps_status adps_normals_pcg64(adps_plan* P, void* stream_v, const uint64_t state[2],
                                          const uint64_t inc[2], int64_t n, double* out, int32_t sync,
                                          int64_t* consumed, int32_t* status) {
  if (!P || !state || !inc) return fail(ADPS_INVALID_ARG, "NULL argument");
  if (n < 0) return fail(ADPS_INVALID_ARG, "negative n");
  if (n > 0 && !out) return fail(ADPS_INVALID_ARG, "out is NULL");
  if (n > (1ll << 30)) return fail(ADPS_INVALID_ARG, "n too large");
  // sync == 2 is consumed by the pending phase 1 (between _begin and _end/_local)
  if (sync == 2 && !P->have_begin) return fail(ADPS_BAD_STATE, "deferred normals (sync=2) need a pending phase1_begin");
  CK(cudaSetDevice(P->device));
  cudaStream_t s = (cudaStream_t)stream_v;
  CK(ensure(P->ctr, sizeof(Counters)));
  if (!P->ctr_host) CK(cudaMallocHost(&P->ctr_host, sizeof(Counters)));
  Counters* ctr = P->ctr.as<Counters>();
  CK(cudaMemsetAsync(&ctr->normals_consumed, 0, sizeof(unsigned long long), s));
  CK(cudaMemsetAsync(&ctr->normals_status, 0, sizeof(unsigned int), s));
  if (n > 0) {
    const long long w = normals_window(n);
    CK(ensure(P->nrm_val, 8ll * w));
    CK(ensure(P->nrm_len, w));
    CK(ensure(P->nrm_acc, w));
    CK(ensure(P->nrm_reach, 4ll * w));
    CK(ensure(P->nrm_rmax, 4ll * w));
    CK(ensure(P->nrm_walked, w));
    CK(ensure(P->nrm_idx, 4ll * w));
    const size_t tb = normals_temp_bytes(w);
    CK(ensure(P->nrm_tmp, tb));
    NormalsArgs a;
    a.state_lo = state[0];
    a.state_hi = state[1];
    a.inc_lo = inc[0];
    a.inc_hi = inc[1];
    a.n = n;
    a.window = w;
    a.out = out;
    a.val = P->nrm_val.as<double>();
    a.len = P->nrm_len.as<unsigned char>();
    a.acc = P->nrm_acc.as<unsigned char>();
    a.reach = P->nrm_reach.as<int>();
    a.reach_max = P->nrm_rmax.as<int>();
    a.walked = P->nrm_walked.as<unsigned char>();
    a.emit_idx = P->nrm_idx.as<int>();
    a.consumed = &ctr->normals_consumed;
    a.status = &ctr->normals_status;
    // on their own stream: phase 1 continues on `stream` meanwhile; joined
    // before phase 1's final counts (or right here when sync).  sync == 2:
    // only recorded here and launched at phase 1's first host wait, while the
    // GPU is busy (the launches cost ~80 us of host time)
    CK(cudaEventRecord(P->ev_nfork, s));
    P->nrm_args = a;
    P->norm_deferred = true;
    if (sync != 2) CK(launch_deferred_normals(P));
  }
  if (sync == 2) return ADPS_OK;
  if (sync && P->norm_pending) {
    CK(cudaStreamWaitEvent(s, P->ev_norm, 0));
    P->norm_pending = false;
  }
  if (sync) {
    CK(cudaMemcpyAsync(&P->ctr_host->normals_consumed, &ctr->normals_consumed, sizeof(unsigned long long),
                       cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(&P->ctr_host->normals_status, &ctr->normals_status, sizeof(unsigned int),
                       cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (consumed) *consumed = (int64_t)P->ctr_host->normals_consumed;
    if (status) *status = (int32_t)P->ctr_host->normals_status;
  }
  return ADPS_OK;
}

extern "C" adps_status adps_vanilla_phase1(adps_plan* P, void* stream_v, const adps_gaussians* g, int64_t n,
                                           double extent, const double* grad_accum, const double* denom,
                                           const adps_config* cfg, int32_t n_children, adps_counts* counts) {
  if (!P) return fail(ADPS_INVALID_ARG, "plan is NULL");
  P->have_phase1 = false;
  P->have_begin = false;
  drop_pending_normals(P);
  adps_status st = check_gaussians(g, n);
  if (st != ADPS_OK) return st;
  if (!cfg || !counts) return fail(ADPS_INVALID_ARG, "cfg/counts is NULL");
  if (n > 0 && (!grad_accum || !denom)) return fail(ADPS_INVALID_ARG, "stats arrays are NULL");
  if (n_children < 1) return fail(ADPS_INVALID_ARG, "n_children must be >= 1");
  if (!(extent > 0)) return fail(ADPS_INVALID_ARG, "scene extent must be > 0");
  CK(cudaSetDevice(P->device));
  cudaStream_t s = (cudaStream_t)stream_v;
  const long long nn = n > 0 ? n : 1;
  CK(ensure(P->cls, nn));
  CK(ensure(P->cand_rank, 4 * nn));
  CK(ensure(P->split_list, 4 * nn));
  CK(ensure(P->clone_list, 4 * nn));
  CK(ensure(P->keep_pos, 4 * nn));
  CK(ensure(P->ctr, sizeof(Counters)));
  Counters* ctr = P->ctr.as<Counters>();
  CK(cudaMemsetAsync(ctr, 0, sizeof(Counters), s));
  mark_start(P, s, true);
  ScanState sst, sst2;
  st = scan_state(P, P->scan_val, P->scan_flag, nn, &sst);
  if (st != ADPS_OK) return st;
  SelectArgs sa;
  sa.scale = g->scale;
  sa.ga = grad_accum;
  sa.den = denom;
  sa.tau_g = cfg->tau_g;
  sa.tau_s_abs = cfg->tau_s * extent;
  sa.n = n;
  sa.cls = P->cls.as<unsigned char>();
  sa.cand_rank = P->cand_rank.as<int>();
  sa.split_list = P->split_list.as<int>();
  sa.clone_list = P->clone_list.as<int>();
  sa.ctr = ctr;
  CK(launch_select(sa, sst, s));
  mark(P, "select", s, 1);
  CK(cudaMemcpyAsync(P->ctr_host, ctr, sizeof(Counters), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  const long long n_split = (long long)P->ctr_host->n_split;
  const long long n_clone = (long long)P->ctr_host->n_clone;
  const long long sc = n_split > 0 ? n_split : 1;
  CK(ensure(P->cand_case, 4 * sc));
  CK(ensure(P->cand_ins, 4 * sc));
  CK(ensure(P->cand_merged, 4 * sc));
  CK(ensure(P->cand_props, 4 * sc));
  CK(ensure(P->ins_off, 4 * sc));
  CK(ensure(P->fb_ord, 4 * sc));
  CK(ensure(P->pstart, 4 * sc));
  CK(ensure(P->children, 16));
  CK(cudaMemsetAsync(P->cand_props.p, 0, 4 * sc, s));
  CK(launch_vanilla_cases(P->cand_case.as<int>(), P->cand_ins.as<int>(), P->cand_merged.as<int>(), &ctr->n_split,
                          n_children, s));
  st = scan_state(P, P->scan2_val, P->scan2_flag, sc, &sst2);
  if (st != ADPS_OK) return st;
  OffsetArgs oa;
  oa.n = n;
  oa.cls = P->cls.as<unsigned char>();
  oa.cand_rank = P->cand_rank.as<int>();
  oa.cand_case = P->cand_case.as<int>();
  oa.cand_ins = P->cand_ins.as<int>();
  oa.ins_off = P->ins_off.as<int>();
  oa.fb_ord = P->fb_ord.as<int>();
  oa.keep_pos = P->keep_pos.as<int>();
  oa.ctr = ctr;
  oa.n_split_dev = &ctr->n_split;
  CK(launch_offsets(oa, n_split, sst2, sst, s));
  mark(P, "offsets", s, 3);
  CK(cudaMemcpyAsync(P->ctr_host, ctr, sizeof(Counters), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  adps_counts& K = P->counts;
  K = adps_counts{};
  K.n_before = n;
  K.n_split = n_split;
  K.n_clone = n_clone;
  K.n_keep = (long long)P->ctr_host->n_keep;
  K.n_inserted = (long long)P->ctr_host->n_inserted;
  K.n_out = K.n_keep + K.n_inserted + n_clone;
  K.n_fallback = n_split;
  *counts = K;
  P->n = n;
  P->V = 0;
  P->eta = cfg->eta;
  P->sh_k = g->sh_rest_k;
  P->fb_children = n_children;
  P->have_phase1 = true;
  return ADPS_OK;
}

extern "C" adps_status adps_reset_flags(adps_plan* P, void* stream_v, uint8_t* flags, int32_t include_clones) {
  if (!P || !flags) return fail(ADPS_INVALID_ARG, "NULL argument");
  if (!P->have_phase1) return fail(ADPS_BAD_STATE, "no phase 1 result");
  CK(cudaSetDevice(P->device));
  CK(launch_reset_flags(flags, P->n, P->split_list.as<int>(), P->cand_case.as<int>(), P->counts.n_split,
                        P->clone_list.as<int>(), P->counts.n_clone, include_clones != 0, (cudaStream_t)stream_v));
  return ADPS_OK;
}

extern "C" adps_status adps_remap_rows(void* stream, const int64_t* index_map, int64_t n_out, const uint8_t* zero_old,
                                       const void* in, int64_t row_bytes, void* out) {
  if (n_out < 0 || row_bytes < 0 || row_bytes % 4) return fail(ADPS_INVALID_ARG, "row_bytes must be a multiple of 4");
  if (n_out > 0 && row_bytes > 0 && (!index_map || !in || !out)) return fail(ADPS_INVALID_ARG, "NULL array");
  CK(launch_remap_rows((const long long*)index_map, n_out, zero_old, in, row_bytes, out, (cudaStream_t)stream));
  return ADPS_OK;
}

extern "C" adps_status adps_accumulate_stats(void* stream, double* grad_accum, double* denom,
                                             const float* viewspace_grad, const uint8_t* visible, int64_t n) {
  if (n < 0) return fail(ADPS_INVALID_ARG, "negative n");
  if (n > 0 && (!grad_accum || !denom || !viewspace_grad || !visible)) return fail(ADPS_INVALID_ARG, "NULL array");
  CK(launch_accumulate(grad_accum, denom, viewspace_grad, visible, n, (cudaStream_t)stream));
  return ADPS_OK;
}

extern "C" adps_status adps_accumulate_stats_f64(void* stream, double* grad_accum, double* denom,
                                                 const double* viewspace_grad, const uint8_t* visible, int64_t n) {
  if (n < 0) return fail(ADPS_INVALID_ARG, "negative n");
  if (n > 0 && (!grad_accum || !denom || !viewspace_grad || !visible)) return fail(ADPS_INVALID_ARG, "NULL array");
  CK(launch_accumulate_f64(grad_accum, denom, viewspace_grad, visible, n, (cudaStream_t)stream));
  return ADPS_OK;
}

extern "C" adps_status adps_prune_index(adps_plan* P, void* stream_v, const float* opacity, const double* logit_op,
                                        int64_t n, double threshold, int64_t* index_map, int64_t* n_keep,
                                        int64_t* n_near) {
  if (!P || !n_keep) return fail(ADPS_INVALID_ARG, "NULL argument");
  if (n < 0) return fail(ADPS_INVALID_ARG, "negative n");
  if (n >= kMaxGaussians) return fail(ADPS_INVALID_ARG, "n=%lld exceeds the supported 2^29 Gaussians", (long long)n);
  if (n > 0 && ((!opacity && !logit_op) || !index_map)) return fail(ADPS_INVALID_ARG, "NULL array");
  if (!(threshold == threshold)) return fail(ADPS_INVALID_ARG, "threshold is NaN");
  CK(cudaSetDevice(P->device));
  cudaStream_t s = (cudaStream_t)stream_v;
  CK(ensure(P->ctr, sizeof(Counters)));
  Counters* ctr = P->ctr.as<Counters>();
  CK(cudaMemsetAsync(&ctr->prune_keep, 0, 2 * sizeof(unsigned long long), s));
  if (n > 0) {
    ScanState sst;
    adps_status st = scan_state(P, P->scan2_val, P->scan2_flag, n, &sst);
    if (st != ADPS_OK) return st;
    PruneArgs pa;
    pa.opacity = opacity;
    pa.logit = opacity ? nullptr : logit_op;
    pa.n = n;
    pa.threshold = threshold;
    pa.index_map = (long long*)index_map;
    pa.n_keep = &ctr->prune_keep;
    pa.n_near = &ctr->prune_near;
    CK(launch_prune(pa, sst, s));
    P->launches += 1;
  }
  CK(cudaMemcpyAsync(&P->ctr_host->prune_keep, &ctr->prune_keep, 2 * sizeof(unsigned long long),
                     cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  *n_keep = (int64_t)P->ctr_host->prune_keep;
  if (n_near) *n_near = (int64_t)P->ctr_host->prune_near;
  return ADPS_OK;
}
