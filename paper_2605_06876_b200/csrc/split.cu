// Candidate selection, child initialisation, cross-view merge, offsets and
// emission of the grown Gaussian arrays.
//
//   select              ref/adc.py:41-46, 82-89
//   region_stats        ref/error_partition.py:137-158
//   init_child          ref/child_init.py:44-140
//   merge/cap/group     ref/cross_view_merge.py:33-116, ref/adc.py:123-140
//   case logic          ref/adc.py:184-227
//   compaction          ref/adc.py:229-244
//   vanilla_split       ref/adc.py:92-108 (fallback, host-drawn normals)
#include <math.h>

#include "split.cuh"

namespace adps {

// ============================================================== select
__device__ __forceinline__ unsigned char select_class(const SelectArgs& a, long long i) {
  const double den = a.den[i];
  const double g = den > 0 ? ddiv(a.ga[i], den) : 0.0;
  const double s0 = a.scale[3 * i], s1 = a.scale[3 * i + 1], s2 = a.scale[3 * i + 2];
  const double ms = fmax(fmax(s0, s1), s2);
  unsigned char c = 0;
  if (g >= a.tau_g) c = ms > a.tau_s_abs ? 1 : 2;
  return c;
}

template <bool CLASSIFY>
struct SelectPolicy {
  SelectArgs a;
  __device__ unsigned long long value(long long i) const {
    unsigned char c;
    if (CLASSIFY) {
      c = select_class(a, i);
      a.cls[i] = c;
    } else {
      c = a.cls[i];   // written by classify_select_kernel
    }
    return c == 1 ? 1ull : (c == 2 ? (1ull << 32) : 0ull);
  }
  __device__ void store(long long i, unsigned long long ex, unsigned long long v) const {
    if (v & 0xffffffffull) {
      int r = (int)(ex & 0xffffffffull);
      a.split_list[r] = (int)i;
      a.cand_rank[i] = r;
    } else {
      a.cand_rank[i] = -1;
    }
    if (v >> 32) a.clone_list[(int)(ex >> 32)] = (int)i;
  }
  __device__ void total(unsigned long long t) const {
    a.ctr->n_split = t & 0xffffffffull;
    a.ctr->n_clone = t >> 32;
  }
};

cudaError_t launch_select(const SelectArgs& a, ScanState st, cudaStream_t s) {
  return launch_scan(SelectPolicy<true>{a}, a.n, st, s);
}

// the classes alone (elementwise, HBM-bound): the input pass needs only them
__global__ void classify_select_kernel(SelectArgs a) {
  pdl_wait();   // programmatic dependent launch: the previous kernel's results are visible
  const long long t0 = (long long)blockIdx.x * blockDim.x + threadIdx.x, stride = (long long)gridDim.x * blockDim.x;
  if (a.lohi_init)
    for (long long t = t0; t < 2ll * a.lohi_views; t += stride)
      a.lohi_init[t] = (t & 1) ? 0ull : 0x7ff0000000000000ull;   // lo = +inf, hi = +0.0
  for (long long i = t0; i < a.n; i += stride) {
    a.cls[i] = select_class(a, i);
    if (a.dom_zero) a.dom_zero[i] = 0;
  }
}

cudaError_t launch_select_split(const SelectArgs& a, ScanState st, cudaStream_t s, cudaStream_t aux, cudaEvent_t fork,
                                cudaEvent_t join) {
  long long b = (a.n + 255) / 256;
  launch_k(classify_select_kernel, (unsigned)(b < 1 ? 1 : (b > 65535 ? 65535 : b)), 256, 0, s, a);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaEventRecord(fork, s);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(aux, fork, 0);
  if (e == cudaSuccess) e = launch_scan(SelectPolicy<false>{a}, a.n, st, aux);
  if (e == cudaSuccess) e = cudaEventRecord(join, aux);
  return e;
}

// ====================================================== region stats + child
__device__ __forceinline__ double sclip(double x, double a) {
  // np.sign(x) * min(abs(x), a)  (ref/child_init.py:75-76)
  double s = x > 0 ? 1.0 : (x < 0 ? -1.0 : 0.0);
  return s * fmin(fabs(x), a);
}

#ifndef ADPS_CHILD_STAGE
#define ADPS_CHILD_STAGE 1
#endif
constexpr int kChildThreads = 128;
constexpr int kPropWords = (int)(sizeof(Proposal) / 8);
static_assert(sizeof(Proposal) == 8 * kPropWords && (kPropWords & 1), "Proposal: whole doubles, odd count");
#ifndef ADPS_CHILD_MINB
#define ADPS_CHILD_MINB 6
#endif
__global__ void __launch_bounds__(kChildThreads, ADPS_CHILD_MINB) child_init_kernel(ChildArgs a) {
  pdl_wait();   // programmatic dependent launch: the previous kernel's results are visible
  long long n = (long long)*a.n_regions;
  if (n > a.region_cap) n = a.region_cap;
  // a region's proposal record, into `prow` (a shared-memory row) or straight to global
  auto body = [&](long long rid, double* prow) {
    const RegionRec R = a.regions[rid];
    // ---- region_stats (ref/error_partition.py:137-158), exact integer moments
    const long long cnt = R.m[0];
    const double nd = (double)cnt;
    const double cx = (double)R.m[1] / nd, cy = (double)R.m[2] / nd;
    const __int128 N = cnt;
    const __int128 sxx = N * R.m[3] - (__int128)R.m[1] * R.m[1];
    const __int128 sxy = N * R.m[4] - (__int128)R.m[1] * R.m[2];
    const __int128 syy = N * R.m[5] - (__int128)R.m[2] * R.m[2];
    const double nn = nd * nd;
    const double ca = (double)sxx / nn, cb = (double)sxy / nn, cc = (double)syy / nn;
    double l1, l2, e1x, e1y;
    if (cb == 0.0) {
      // diagonal: LAPACK returns the unit axes, e1 = column of the larger value
      if (ca > cc) { l1 = ca; l2 = cc; e1x = 1.0; e1y = 0.0; }
      else { l1 = cc; l2 = ca; e1x = 0.0; e1y = 1.0; }
    } else {
      double t = 0.5 * (ca - cc), m = 0.5 * (ca + cc);
      double rr = hypot(t, cb);
      l1 = m + rr;
      l2 = m - rr;
      double vx, vy;
      if (ca >= cc) { vx = l1 - cc; vy = cb; }
      else { vx = cb; vy = l1 - ca; }
      double vn = hypot(vx, vy);
      e1x = vx / vn;
      e1y = vy / vn;
    }
    const double sig1 = fmax(sqrt(fmax(l1, 0.0)), kSigmaFloor);
    const double sig2 = fmax(sqrt(fmax(l2, 0.0)), kSigmaFloor);
    const double e2x = -e1y, e2y = e1x;
    int ix = (int)rint(cx), iy = (int)rint(cy);   // round-half-even
    ix = ix < 0 ? 0 : (ix > a.W - 1 ? a.W - 1 : ix);
    iy = iy < 0 ? 0 : (iy > a.H - 1 ? a.H - 1 : iy);
    const int lv = (R.view_pos - a.view_offset) / a.view_stride;   // local view of this region
    const float* gp = a.gt + (((long long)lv * a.H + iy) * a.W + ix) * 3;
    const double rgb[3] = {(double)gp[0], (double)gp[1], (double)gp[2]};

    // ---- init_child (ref/child_init.py:110-140)
    const CamD cam = load_cam(a.cams + 18ll * lv);
    const int gi = R.cand;
    const double dcam[3] = {(cx - cam.px) / cam.fx, (cy - cam.py) / cam.fy, 1.0};
    double dw[3];
    for (int i = 0; i < 3; ++i)
      dw[i] = cam.r[i * 3 + 0] * dcam[0] + cam.r[i * 3 + 1] * dcam[1] + cam.r[i * 3 + 2] * dcam[2];
    const double dwn = sqrt(dw[0] * dw[0] + dw[1] * dw[1] + dw[2] * dw[2]);
    const double dir[3] = {dw[0] / dwn, dw[1] / dwn, dw[2] / dwn};
    const double dnorm = sqrt(dcam[0] * dcam[0] + dcam[1] * dcam[1] + 1.0);
    double q[4] = {a.g.rot[4 * gi], a.g.rot[4 * gi + 1], a.g.rot[4 * gi + 2], a.g.rot[4 * gi + 3]};
    double pr[9];
    quat_to_rot(q, pr);
    const double ps[3] = {a.g.scale[3 * gi], a.g.scale[3 * gi + 1], a.g.scale[3 * gi + 2]};
    const double inv2[3] = {1.0 / (ps[0] * ps[0]), 1.0 / (ps[1] * ps[1]), 1.0 / (ps[2] * ps[2])};
    double prec[6];
    rdrt(pr, inv2, prec);   // inv(covariance(parent)) = R diag(1/s^2) R^T
    const double b[3] = {a.g.mu[3 * gi] - cam.c[0], a.g.mu[3 * gi + 1] - cam.c[1],
                         a.g.mu[3 * gi + 2] - cam.c[2]};
    const double denom = sym_quad(prec, dir);
    double tstar = 0.0;
    bool ok = true;
    if (!(denom >= kDegenerateDenom)) {
      atomicOr(&a.ctr->degenerate, 1u);
      ok = false;
    } else {
      tstar = sym_bilin(prec, b, dir) / (denom + a.eps);
      ok = tstar > 0.0;
    }
    double rot[9] = {0}, s1 = 0, s2 = 0, mu[3] = {0, 0, 0};
    if (ok) {
      const double smax = fmax(fmax(ps[0], ps[1]), ps[2]);
      const double tz = tstar / dnorm;
      const double w1x = sclip(e1x * sig1 * tz / cam.fx, smax * fabs(e1x));
      const double w1y = sclip(e1y * sig1 * tz / cam.fy, smax * fabs(e1y));
      const double w2x = sclip(e2x * sig2 * tz / cam.fx, smax * fabs(e2x));
      const double w2y = sclip(e2y * sig2 * tz / cam.fy, smax * fabs(e2y));
      double a1[3], a2[3], right[3], down[3], fwd[3];
      for (int i = 0; i < 3; ++i) {
        right[i] = cam.r[i * 3 + 0];
        down[i] = cam.r[i * 3 + 1];
        fwd[i] = cam.r[i * 3 + 2];
        a1[i] = w1x * right[i] + w1y * down[i];
        a2[i] = w2x * right[i] + w2y * down[i];
      }
      s1 = sqrt(a1[0] * a1[0] + a1[1] * a1[1] + a1[2] * a1[2]);
      s2 = sqrt(a2[0] * a2[0] + a2[1] * a2[1] + a2[2] * a2[2]);
      const double u1[3] = {a1[0] / s1, a1[1] / s1, a1[2] / s1};
      double fb[3] = {fwd[1] * u1[2] - fwd[2] * u1[1], fwd[2] * u1[0] - fwd[0] * u1[2],
                      fwd[0] * u1[1] - fwd[1] * u1[0]};
      const double fbn = sqrt(fb[0] * fb[0] + fb[1] * fb[1] + fb[2] * fb[2]);
      double fallback[3];
      for (int i = 0; i < 3; ++i) fallback[i] = fbn > kParallelTol ? fb[i] / fbn : down[i];
      const double proj = a2[0] * u1[0] + a2[1] * u1[1] + a2[2] * u1[2];
      double rej[3] = {a2[0] - proj * u1[0], a2[1] - proj * u1[1], a2[2] - proj * u1[2]};
      const double rn = sqrt(rej[0] * rej[0] + rej[1] * rej[1] + rej[2] * rej[2]);
      double u2[3];
      for (int i = 0; i < 3; ++i) u2[i] = rn < kParallelTol ? fallback[i] : rej[i] / rn;
      for (int i = 0; i < 3; ++i) {
        rot[i * 3 + 0] = u1[i];
        rot[i * 3 + 1] = u2[i];
        rot[i * 3 + 2] = fwd[i];
      }
      const double det = rot[0] * (rot[4] * rot[8] - rot[5] * rot[7]) -
                         rot[1] * (rot[3] * rot[8] - rot[5] * rot[6]) +
                         rot[2] * (rot[3] * rot[7] - rot[4] * rot[6]);
      if (det < 0)
        for (int i = 0; i < 3; ++i) rot[i * 3 + 2] = -rot[i * 3 + 2];
      for (int i = 0; i < 3; ++i) mu[i] = cam.c[i] + tstar * dir[i];
      Proposal* const P = prow ? reinterpret_cast<Proposal*>(prow) : a.props + rid;
      for (int i = 0; i < 3; ++i) {
        P->mu[i] = mu[i];
        P->rgb[i] = rgb[i];
      }
      const double sq[3] = {s1 * s1, s2 * s2, s2 * s2};
      const double iq[3] = {1.0 / sq[0], 1.0 / sq[1], 1.0 / sq[2]};
      rdrt(rot, sq, P->cov);
      rdrt(rot, iq, P->prec);
      P->inv_smax = 1.0 / fmax(s1, s2);
    } else if (prow) {
      for (int i = 0; i < kPropWords; ++i) prow[i] = 0.0;   // (an invalid region's record is never read)
    }
    a.valid[rid] = ok ? 1 : 0;
    if (a.write_keys) {
      const unsigned long long rank = (unsigned long long)a.cand_rank[gi];
      a.keys[rid] = (((rank << a.bits_v | (unsigned long long)R.view_pos) << a.bits_b |
                      (unsigned long long)R.band)
                     << a.bits_p) |
                    (unsigned long long)R.minpix;
      a.vals[rid] = (int)rid;
    }
    if (a.dbg_stats) {
      double* d = a.dbg_stats + 10 * rid;
      d[0] = cx; d[1] = cy; d[2] = e1x; d[3] = e1y; d[4] = sig1; d[5] = sig2;
      d[6] = rgb[0]; d[7] = rgb[1]; d[8] = rgb[2]; d[9] = tstar;
      double* c = a.dbg_child + 16 * rid;
      for (int i = 0; i < 3; ++i) c[i] = mu[i];
      for (int i = 0; i < 9; ++i) c[3 + i] = rot[i];
      c[12] = s1; c[13] = s2; c[14] = s2; c[15] = ok ? 1.0 : 0.0;
    }
  };
#if ADPS_CHILD_STAGE
  // records staged in shared memory, then stored as one contiguous run per
  // block (a thread's 152-byte record stored directly is 19 strided stores)
  __shared__ double sp[kChildThreads * kPropWords];   // odd row stride: no bank conflicts
  for (long long base = (long long)blockIdx.x * kChildThreads; base < n; base += (long long)gridDim.x * kChildThreads) {
    const long long rid = base + threadIdx.x;
    if (rid < n) body(rid, sp + threadIdx.x * kPropWords);
    __syncthreads();
    const long long rows = n - base < kChildThreads ? n - base : kChildThreads;
    double* dst = reinterpret_cast<double*>(a.props + base);
    for (int w = threadIdx.x; w < rows * kPropWords; w += kChildThreads) dst[w] = sp[w];
    __syncthreads();
  }
#else
  for (long long rid = (long long)blockIdx.x * blockDim.x + threadIdx.x; rid < n; rid += (long long)gridDim.x * blockDim.x)
    body(rid, nullptr);
#endif
}

__global__ void region_keys_kernel(const RegionRec* __restrict__ regions, long long n, const int* __restrict__ cand_rank,
                                   int bits_v, int bits_b, int bits_p, unsigned long long* __restrict__ keys,
                                   int* __restrict__ vals) {
  pdl_wait();   // programmatic dependent launch: the previous kernel's results are visible
  for (long long rid = (long long)blockIdx.x * blockDim.x + threadIdx.x; rid < n; rid += (long long)gridDim.x * blockDim.x) {
    const RegionRec& R = regions[rid];
    const unsigned long long rank = (unsigned long long)cand_rank[R.cand];
    keys[rid] = (((rank << bits_v | (unsigned long long)R.view_pos) << bits_b | (unsigned long long)R.band) << bits_p) |
                (unsigned long long)R.minpix;
    vals[rid] = (int)rid;
  }
}

__global__ void zero_kernel(ZeroList z) {
  pdl_wait();   // programmatic dependent launch: the previous kernel's results are visible
  const long long t0 = (long long)blockIdx.x * blockDim.x + threadIdx.x, stride = (long long)gridDim.x * blockDim.x;
  for (int e = 0; e < z.count; ++e)
    for (long long i = t0; i < z.n[e]; i += stride) z.p[e][i] = 0;
}

cudaError_t launch_zero(const ZeroList& z, cudaStream_t s) {
  long long m = 1;
  for (int e = 0; e < z.count; ++e) m = z.n[e] > m ? z.n[e] : m;
  const long long b = (m + 255) / 256;
  launch_k(zero_kernel, (unsigned)(b > 1184 ? 1184 : b), 256, 0, s, z);
  return cudaGetLastError();
}

cudaError_t launch_region_keys(const RegionRec* regions, long long n, const int* cand_rank, int bits_v, int bits_b,
                               int bits_p, unsigned long long* keys, int* vals, cudaStream_t s) {
  long long b = (n + 255) / 256;
  launch_k(region_keys_kernel, (unsigned)(b < 1 ? 1 : (b > 65535 ? 65535 : b)), 256, 0, s, regions, n, cand_rank, bits_v,
                                                                                     bits_b, bits_p, keys, vals);
  return cudaGetLastError();
}

cudaError_t launch_child_init(const ChildArgs& a, cudaStream_t s) {
  launch_k(child_init_kernel, a.grid, kChildThreads, 0, s, a);
  return cudaGetLastError();
}

// ============================================================ ranges
__global__ void ranges_kernel(RangeArgs a) {
  pdl_wait();   // programmatic dependent launch: the previous kernel's results are visible
  // keys are sorted, so one candidate's (and one (candidate, view)'s) regions are
  // adjacent: counts are aggregated per warp (match_any) before the atomics, which
  // keeps a parent with tens of thousands of regions from serialising on one word
  const int lane = threadIdx.x & 31;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i0 = (long long)blockIdx.x * blockDim.x; i0 < a.n; i0 += stride) {
    const long long i = i0 + threadIdx.x;
    const bool in = i < a.n;
    unsigned long long k = in ? a.keys_sorted[i] : ~0ull;
    const int rank = (int)(k >> a.shift_rank);
    const bool val = in && a.valid[a.vals_sorted[i]];
    if (in) {
      if (i == 0 || (int)(a.keys_sorted[i - 1] >> a.shift_rank) != rank) a.cand_start[rank] = (int)i;
      if (i == a.n - 1 || (int)(a.keys_sorted[i + 1] >> a.shift_rank) != rank) a.cand_end[rank] = (int)(i + 1);
    }
    const unsigned live = __ballot_sync(0xffffffffu, in);
    const unsigned long long rv = k >> a.shift_view;   // (rank, view)
    const unsigned g_rv = __match_any_sync(0xffffffffu, rv) & live;
    const unsigned g_r = __match_any_sync(0xffffffffu, (unsigned long long)rank) & live;
    if (in && lane == __ffs(g_rv) - 1) {
      const int view = (int)(rv & ((1ull << a.bits_v) - 1ull));
      atomicAdd(&a.regions_per_view[(long long)rank * a.n_views + view], __popc(g_rv));
    }
    const int nv = __popc(__ballot_sync(0xffffffffu, val) & g_r);
    if (in && lane == __ffs(g_r) - 1 && nv) atomicAdd(&a.cand_nvalid[rank], nv);
  }
}

cudaError_t launch_ranges(const RangeArgs& a, cudaStream_t s) {
  if (a.n > 0) launch_k(ranges_kernel, a.grid, 256, 0, s, a);
  return cudaGetLastError();
}

// ============================================================ merge: merge.cu

// ============================================================ offsets
struct CandScanPolicy {
  OffsetArgs a;
  __device__ unsigned long long value(long long k) const {
    unsigned long long v = (unsigned long long)a.cand_ins[k];
    if (a.cand_case[k] == ADPS_CASE_FALLBACK) v |= 1ull << 32;
    return v;
  }
  __device__ void store(long long k, unsigned long long ex, unsigned long long) const {
    a.ins_off[k] = (int)(ex & 0xffffffffull);
    a.fb_ord[k] = (int)(ex >> 32);
  }
  __device__ void total(unsigned long long t) const { a.ctr->n_inserted = t & 0xffffffffull; }
};

struct KeepScanPolicy {
  OffsetArgs a;
  __device__ unsigned long long value(long long i) const {
    const int r = a.cand_rank[i];
    if (r < 0) return 1ull;
    const int c = a.cand_case[r];
    return c == ADPS_CASE_RESET ? 1ull : 0ull;
  }
  __device__ void store(long long i, unsigned long long ex, unsigned long long v) const {
    a.keep_pos[i] = v ? (int)ex : -1;
  }
  __device__ void total(unsigned long long t) const { a.ctr->n_keep = t; }
};

cudaError_t launch_offsets_cand(const OffsetArgs& a, long long n_split, ScanState st_c, cudaStream_t s) {
  return launch_scan(CandScanPolicy{a}, n_split, st_c, s);
}

cudaError_t launch_offsets_keep(const OffsetArgs& a, ScanState st_g, cudaStream_t s) {
  return launch_scan(KeepScanPolicy{a}, a.n, st_g, s);
}

cudaError_t launch_offsets(const OffsetArgs& a, long long n_split, ScanState st_c, ScanState st_g,
                           cudaStream_t s) {
  cudaError_t e = launch_scan(CandScanPolicy{a}, n_split, st_c, s);
  if (e != cudaSuccess) return e;
  return launch_scan(KeepScanPolicy{a}, a.n, st_g, s);
}

// ============================================================ emit
__device__ __forceinline__ void copy_gaussian(const EmitArgs& a, long long src, long long dst) {
  // all loads first: the output arrays may alias nothing, but the compiler
  // cannot know, and interleaved load/store pairs would serialise on latency
  float m[3], sc[3], dc[3], q[4];
  for (int t = 0; t < 3; ++t) {
    m[t] = __ldg(a.g.mu + 3 * src + t);
    sc[t] = __ldg(a.g.scale + 3 * src + t);
    dc[t] = __ldg(a.g.sh_dc + 3 * src + t);
  }
  for (int t = 0; t < 4; ++t) q[t] = __ldg(a.g.rot + 4 * src + t);
  const float o = __ldg(a.g.opacity + src);
  for (int t = 0; t < 3; ++t) {
    a.mu[3 * dst + t] = m[t];
    a.scale[3 * dst + t] = sc[t];
    a.sh_dc[3 * dst + t] = dc[t];
  }
  for (int t = 0; t < 4; ++t) a.rot[4 * dst + t] = q[t];
  a.opacity[dst] = o;
  const int K = a.g.sh_k;
  for (int t = 0; t < 3 * K; ++t) a.sh_rest[3ll * K * dst + t] = a.g.sh_rest[3ll * K * src + t];
}

// One launch, three block ranges: survivors (thread per old Gaussian, old
// order), candidate inserts (a warp per candidate, lane = output row: N_i
// children then the parent copy, or the fallback children), clones (thread
// per clone).  Rows are written where the offsets put them.
constexpr int kEmitThreads = 256;

__device__ __forceinline__ void emit_insert_row(const EmitArgs& a, long long n_keep, long long k, int j) {
  const int c = a.cand_case[k];
  const long long gi = a.split_list[k];
  const long long dst = n_keep + a.ins_off[k] + j;
  const int K = a.g.sh_k;
  if (c == ADPS_CASE_FALLBACK) {                        // vanilla_split(parent, n, eta, rng)
    double q[4] = {a.g.rot[4 * gi], a.g.rot[4 * gi + 1], a.g.rot[4 * gi + 2], a.g.rot[4 * gi + 3]};
    double R[9];
    quat_to_rot(q, R);
    const double s[3] = {a.g.scale[3 * gi], a.g.scale[3 * gi + 1], a.g.scale[3 * gi + 2]};
    const int nc = a.fb_children;
    const double sh = a.eta * (double)nc;
    const double* z = a.normals + 3ll * nc * a.fb_ord[k] + 3 * j;
    const double dl[3] = {z[0] * s[0], z[1] * s[1], z[2] * s[2]};
    copy_gaussian(a, gi, dst);
    for (int i = 0; i < 3; ++i) {
      const double off = R[i * 3] * dl[0] + R[i * 3 + 1] * dl[1] + R[i * 3 + 2] * dl[2];
      a.mu[3 * dst + i] = (float)((double)a.g.mu[3 * gi + i] + off);
      a.scale[3 * dst + i] = (float)(s[i] / sh);
    }
  } else {                                              // N_i children then the parent copy
    const int ni = a.cand_merged[k];
    if (j < ni) {
      const float* c3 = a.children + 14ll * (a.cand_start[k] + j);
      float c[14];
      for (int u = 0; u < 14; ++u) c[u] = __ldg(c3 + u);
      for (int u = 0; u < 3; ++u) {
        a.mu[3 * dst + u] = c[u];
        a.scale[3 * dst + u] = c[3 + u];
        a.sh_dc[3 * dst + u] = c[11 + u];
      }
      for (int u = 0; u < 4; ++u) a.rot[4 * dst + u] = c[6 + u];
      a.opacity[dst] = c[10];
      for (int u = 0; u < 3 * K; ++u) a.sh_rest[3ll * K * dst + u] = 0.0f;
    } else {
      copy_gaussian(a, gi, dst);
      const double o = (double)a.g.opacity[gi] / (double)(ni + 1);
      a.opacity[dst] = (float)fmin(fmax(o, 1e-6), 1.0 - 1e-6);
    }
  }
  a.index_map[dst] = -1;
  if (a.child_parent) a.child_parent[a.ins_off[k] + j] = (int)gi;
}

// survivors: one parameter array per blockIdx.y, thread per component, so
// loads and stores are coalesced whatever the array's width (C: components
// per Gaussian, a compile-time constant so the index split is a multiply)
template <int C>
__device__ __forceinline__ void copy_survivor_components(const EmitArgs& a, const float* __restrict__ in,
                                                         float* __restrict__ out, bool index) {
  // a warp takes 256 consecutive components, lane-strided (element base + 32 i
  // + lane): every load and store instruction covers 128 contiguous bytes
  // (survivor positions are contiguous between removed Gaussians), and a
  // thread's 8 loads are in flight together
  const unsigned ne = (unsigned)a.n * C;
  const unsigned base = ((blockIdx.x * kEmitThreads + threadIdx.x) >> 5) * 256u + (threadIdx.x & 31);
  float v[8];
  int pos[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const unsigned e = base + 32u * i;
    v[i] = e < ne ? __ldg(in + e) : 0.0f;
    pos[i] = e < ne ? __ldg(a.keep_pos + e / C) : -1;
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const unsigned e = base + 32u * i;
    if (pos[i] < 0) continue;
    const unsigned t = e / C;
    out[(unsigned)pos[i] * C + (e - t * C)] = v[i];
    if (index) a.index_map[pos[i]] = t;
  }
}

__global__ void __launch_bounds__(kEmitThreads) emit_survivors_kernel(EmitArgs a) {
  pdl_wait();   // programmatic dependent launch: the previous kernel's results are visible
  switch (blockIdx.y) {
    case 0: copy_survivor_components<3>(a, a.g.mu, a.mu, false); break;
    case 1: copy_survivor_components<3>(a, a.g.scale, a.scale, false); break;
    case 2: copy_survivor_components<4>(a, a.g.rot, a.rot, false); break;
    case 3: copy_survivor_components<1>(a, a.g.opacity, a.opacity, true); break;
    case 4: copy_survivor_components<3>(a, a.g.sh_dc, a.sh_dc, false); break;
    default: {   // sh_rest: 3K components
      const long long c = 3ll * a.g.sh_k;
      const long long ne = a.n * c;
      for (long long e = (long long)blockIdx.x * kEmitThreads + threadIdx.x; e < ne;
           e += (long long)gridDim.x * kEmitThreads) {
        const long long t = e / c;
        const int pos = __ldg(a.keep_pos + t);
        if (pos >= 0) a.sh_rest[pos * c + (e - t * c)] = __ldg(a.g.sh_rest + e);
      }
    }
  }
}

__global__ void __launch_bounds__(kEmitThreads) emit_kernel(EmitArgs a, long long b_ins) {
  pdl_wait();   // programmatic dependent launch: the previous kernel's results are visible
  const long long blk = blockIdx.x;
  long long n_keep = a.n_keep, n_inserted = a.n_inserted;
  bool capped = false;
  if (a.dev_keep) {   // counts still on the device (sync-free form)
    n_keep = (long long)*a.dev_keep;
    n_inserted = (long long)*a.dev_inserted;
    capped = true;
  }
  if (blk < b_ins) {                                    // candidate inserts, ascending index
    // a thread per inserted row: its candidate is the last k with ins_off[k] <= r
    // (ins_off is the exclusive prefix of the rows per candidate), found by a
    // binary search; rows of one candidate are adjacent, so neighbouring threads
    // mostly search the same path (cached)
    const long long r = blk * kEmitThreads + threadIdx.x;
    if (r >= n_inserted) return;
    if (capped && (n_keep + r >= a.out_cap || r >= a.app_cap)) return;
    long long lo = 0, hi = a.n_split - 1;
    while (lo < hi) {
      const long long mid = (lo + hi + 1) >> 1;
      if ((long long)__ldg(a.ins_off + mid) <= r) lo = mid;
      else hi = mid - 1;
    }
    // (a reset candidate inserts nothing, so its offset equals the next
    // candidate's: the last k with ins_off[k] <= r always has rows)
    const long long k = lo;
    const int j = (int)(r - __ldg(a.ins_off + k));
    emit_insert_row(a, n_keep, k, j);
    if (a.insert_offset && j == 0) a.insert_offset[k] = n_keep + a.ins_off[k];
  } else if (blk < b_ins + a.b_off) {                   // insert offsets of the reset candidates
    const long long k = (blk - b_ins) * kEmitThreads + threadIdx.x;
    if (k < a.n_split && a.insert_offset && a.cand_case[k] == ADPS_CASE_RESET)
      a.insert_offset[k] = n_keep + a.ins_off[k];
  } else {                                              // clones, ascending
    const long long j = (blk - b_ins - a.b_off) * kEmitThreads + threadIdx.x;
    if (j < a.n_clone) {
      const long long dst = n_keep + n_inserted + j;
      if (capped && (dst >= a.out_cap || n_inserted + j >= a.app_cap)) return;
      const int src = a.clone_list[j];
      copy_gaussian(a, src, dst);
      a.index_map[dst] = -1;
      if (a.child_parent) a.child_parent[n_inserted + j] = src;
    }
  }
}

cudaError_t launch_emit(const EmitArgs& a, cudaStream_t s, cudaStream_t aux, cudaEvent_t fork, cudaEvent_t join) {
  // the survivor copy (HBM-bound) on the second stream, concurrently with the
  // latency-bound inserts and clones; `s` waits for it before returning
  const bool two = aux && a.n > 0;
  if (two) {
    cudaError_t e = cudaEventRecord(fork, s);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(aux, fork, 0);
    if (e != cudaSuccess) return e;
  }
  if (a.n > 0) {
    const cudaStream_t ss = two ? aux : s;
    // 8 components per thread (rot's 4 per Gaussian the widest; narrower arrays exit early)
    long long b = (a.n * 4 + 8ll * kEmitThreads - 1) / (8ll * kEmitThreads);
    launch_k(emit_survivors_kernel, dim3((unsigned)b, a.g.sh_k > 0 ? 6u : 5u), kEmitThreads, 0, ss, a);
  }
  const long long b_ins = ((a.dev_keep ? a.n_ins_max : a.n_inserted) + kEmitThreads - 1) / kEmitThreads;
  const long long b_clone = (a.n_clone + kEmitThreads - 1) / kEmitThreads;
  EmitArgs a2 = a;
  a2.b_off = a.insert_offset ? (a.n_split + kEmitThreads - 1) / kEmitThreads : 0;
  if (b_ins + a2.b_off + b_clone > 0)
    launch_k(emit_kernel, (unsigned)(b_ins + a2.b_off + b_clone), kEmitThreads, 0, s, a2, b_ins);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess && two) {
    e = cudaEventRecord(join, aux);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(s, join, 0);
  }
  return e;
}

// ============================================================ vanilla_densify / remaps
__global__ void vanilla_cases_kernel(int* cand_case, int* cand_ins, int* cand_merged,
                                     const unsigned long long* n_split, int n_children) {
  pdl_wait();   // programmatic dependent launch: the previous kernel's results are visible
  const long long n = (long long)*n_split;
  for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (long long)gridDim.x * blockDim.x) {
    cand_case[k] = ADPS_CASE_FALLBACK;
    cand_ins[k] = n_children;
    cand_merged[k] = 0;
  }
}

cudaError_t launch_vanilla_cases(int* cand_case, int* cand_ins, int* cand_merged, const unsigned long long* n_split,
                                 int n_children, cudaStream_t s) {
  launch_k(vanilla_cases_kernel, 148 * 4, 256, 0, s, cand_case, cand_ins, cand_merged, n_split, n_children);
  return cudaGetLastError();
}

__global__ void reset_flags_kernel(unsigned char* flags, long long n, const int* split_list, const int* cand_case,
                                   long long n_split, const int* clone_list, long long n_clone, bool clones) {
  pdl_wait();   // programmatic dependent launch: the previous kernel's results are visible
  const long long total = n_split + (clones ? n_clone : 0);
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    if (t < n_split) {
      if (cand_case[t] == ADPS_CASE_RESET) flags[split_list[t]] = 1;
    } else {
      flags[clone_list[t - n_split]] = 1;
    }
  }
}

cudaError_t launch_reset_flags(unsigned char* flags, long long n, const int* split_list, const int* cand_case,
                               long long n_split, const int* clone_list, long long n_clone, bool clones,
                               cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(flags, 0, (size_t)(n > 0 ? n : 1), s);
  if (e != cudaSuccess) return e;
  if (n_split + n_clone > 0)
    launch_k(reset_flags_kernel, 148 * 4, 256, 0, s, flags, n, split_list, cand_case, n_split, clone_list, n_clone, clones);
  return cudaGetLastError();
}

// out[new] = in[index_map[new]] for carried rows not flagged, zero otherwise; rows are
// copied as 4-byte words (row_bytes % 4 == 0)
__global__ void remap_rows_kernel(const long long* __restrict__ index_map, long long n_out,
                                  const unsigned char* __restrict__ zero_old, const unsigned* __restrict__ in,
                                  long long row_words, unsigned* __restrict__ out) {
  pdl_wait();   // programmatic dependent launch: the previous kernel's results are visible
  const long long total = n_out * row_words;
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const long long r = t / row_words, w = t - r * row_words;
    const long long old = index_map[r];
    const bool carry = old >= 0 && !(zero_old && zero_old[old]);
    out[t] = carry ? in[old * row_words + w] : 0u;
  }
}

cudaError_t launch_remap_rows(const long long* index_map, long long n_out, const unsigned char* zero_old,
                              const void* in, long long row_bytes, void* out, cudaStream_t s) {
  const long long words = n_out * (row_bytes / 4);
  if (words > 0) {
    long long b = (words + 255) / 256;
    if (b > 148 * 32) b = 148 * 32;
    launch_k(remap_rows_kernel, (unsigned)b, 256, 0, s, index_map, n_out, zero_old, (const unsigned*)in, row_bytes / 4,
                                                 (unsigned*)out);
  }
  return cudaGetLastError();
}

// ============================================================ stats feed
// ref/adc.py:73-79: norms = np.linalg.norm(vg, axis=1) = sqrt(x*x + y*y) in the
// gradient's precision (this file is compiled with -fmad=false, so the sum of
// squares rounds exactly as numpy's does); grad_accum[vis] += norm, denom[vis] += 1.
// HBM-bound: 41 B per Gaussian and view (vg 2 x fp64 or 8 B fp32, vis 1 B,
// grad_accum/denom read + written 32 B).  Grid-stride, two Gaussians per thread
// per iteration through 16-byte vector loads of the gradient pairs.
template <class T>
__device__ __forceinline__ double vg_norm(T x, T y) {
  const T nrm = sqrt(x * x + y * y);
  return (double)nrm;
}

// two Gaussians per thread: grad_accum / denom as double2, the gradient pairs as
// one 16-byte (fp32) or two 16-byte (fp64) loads, the visibility as a uchar2
template <class T>
__global__ void __launch_bounds__(256) accumulate_kernel(double* __restrict__ ga, double* __restrict__ den,
                                                         const T* __restrict__ vg,
                                                         const unsigned char* __restrict__ vis, long long n) {
  pdl_wait();   // programmatic dependent launch: the previous kernel's results are visible
  const long long n2 = n >> 1;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n2;
       i += (long long)gridDim.x * blockDim.x) {
    const uchar2 v = __ldg(reinterpret_cast<const uchar2*>(vis) + i);
    if (!(v.x | v.y)) continue;
    T g[4];
    if (sizeof(T) == 4) {
      const float4 q = __ldg(reinterpret_cast<const float4*>(vg) + i);
      g[0] = q.x; g[1] = q.y; g[2] = q.z; g[3] = q.w;
    } else {
      const double2 a = __ldg(reinterpret_cast<const double2*>(vg) + 2 * i);
      const double2 b = __ldg(reinterpret_cast<const double2*>(vg) + 2 * i + 1);
      g[0] = a.x; g[1] = a.y; g[2] = b.x; g[3] = b.y;
    }
    double2 A = reinterpret_cast<double2*>(ga)[i], D = reinterpret_cast<double2*>(den)[i];
    if (v.x) {
      A.x += vg_norm(g[0], g[1]);
      D.x += 1.0;
    }
    if (v.y) {
      A.y += vg_norm(g[2], g[3]);
      D.y += 1.0;
    }
    reinterpret_cast<double2*>(ga)[i] = A;
    reinterpret_cast<double2*>(den)[i] = D;
  }
  if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) {   // the odd last Gaussian
    const long long i = n - 1;
    if (vis[i]) {
      ga[i] += vg_norm(vg[2 * i], vg[2 * i + 1]);
      den[i] += 1.0;
    }
  }
}

// any alignment: one Gaussian per thread
template <class T>
__global__ void __launch_bounds__(256) accumulate1_kernel(double* __restrict__ ga, double* __restrict__ den,
                                                          const T* __restrict__ vg,
                                                          const unsigned char* __restrict__ vis, long long n) {
  pdl_wait();   // programmatic dependent launch: the previous kernel's results are visible
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    if (!__ldg(vis + i)) continue;
    ga[i] += vg_norm(__ldg(vg + 2 * i), __ldg(vg + 2 * i + 1));
    den[i] += 1.0;
  }
}

template <class T>
static cudaError_t launch_accumulate_t(double* ga, double* den, const T* vg, const unsigned char* vis, long long n,
                                       cudaStream_t s) {
  const bool aligned = ((uintptr_t)ga % 16 == 0) && ((uintptr_t)den % 16 == 0) && ((uintptr_t)vg % 16 == 0) &&
                       ((uintptr_t)vis % 2 == 0);
  if (n > 0 && !aligned) {
    long long blocks = (n + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    launch_k(accumulate1_kernel<T>, (unsigned)blocks, 256, 0, s, ga, den, vg, vis, n);
  } else if (n > 0) {
    long long blocks = (n / 2 + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    if (blocks < 1) blocks = 1;
    launch_k(accumulate_kernel<T>, (unsigned)blocks, 256, 0, s, ga, den, vg, vis, n);
  }
  return cudaGetLastError();
}

cudaError_t launch_accumulate(double* ga, double* den, const float* vg, const unsigned char* vis,
                              long long n, cudaStream_t s) {
  return launch_accumulate_t<float>(ga, den, vg, vis, n, s);
}

cudaError_t launch_accumulate_f64(double* ga, double* den, const double* vg, const unsigned char* vis,
                                  long long n, cudaStream_t s) {
  return launch_accumulate_t<double>(ga, den, vg, vis, n, s);
}

// ============================================================ opacity prune
// ref/harness.py:320-340 (_prune): keep = sigmoid(logit_op) >= threshold, the
// survivors compacted in old order.  The keep test runs on the trainer's
// representation: the stored opacity (fp32, compared exactly in fp64), or the
// fp64 logit through 1/(1+exp(-x)) (ref/harness.py:217-218) -- CUDA's exp and
// the host libm's may differ by an ulp, so logits whose sigmoid lies within
// 4 ulp of the threshold are counted as near-threshold (reported separately).
struct PruneScanPolicy {
  PruneArgs a;
  __device__ bool keep(long long i) const {
    if (a.opacity) return (double)__ldg(a.opacity + i) >= a.threshold;
    const double x = __ldg(a.logit + i);
    const double sg = 1.0 / (1.0 + exp(-x));
    if (fabs(sg - a.threshold) <= 4.0 * ulp_of(a.threshold)) atomicAdd(a.n_near, 1ull);
    return sg >= a.threshold;
  }
  __device__ static double ulp_of(double v) {
    const double av = fabs(v);
    return __longlong_as_double(__double_as_longlong(av) + 1) - av;
  }
  __device__ unsigned long long value(long long i) const { return keep(i) ? 1ull : 0ull; }
  __device__ void store(long long i, unsigned long long ex, unsigned long long v) const {
    if (v) a.index_map[ex] = i;
  }
  __device__ void total(unsigned long long t) const { *a.n_keep = t; }
};

cudaError_t launch_prune(const PruneArgs& a, ScanState st, cudaStream_t s) {
  return launch_scan(PruneScanPolicy{a}, a.n, st, s);
}

}  // namespace adps
