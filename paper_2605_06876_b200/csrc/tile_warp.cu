// Warp-per-tile scanline CCL: the common-case attribution kernel.
//
// Same results as tile_block (attribution.cu), i.e. the reference's
//   metric_map / erode / band_map   ref/error_partition.py:57-91
//   partition (8-connected, keyed by candidate and band)  ref/error_partition.py:94-134
// but one warp owns a 32x32 tile and walks its rows top to bottom, so there
// is no block barrier at all:
//   * lane = x; each (haloed) row is loaded one row ahead, thresholded (fp64,
//     numpy order) and reduced to a 64-bit metric bitmask by ballot; the
//     r x r erosion (r <= 3, a template parameter) is a shift-AND over the
//     last r masks, which live in (warp-uniform) registers;
//   * a tile row's keyed pixels form horizontal runs (ballots); each run gets
//     the next run id (row-major, so the smallest id of a component is its
//     first pixel) and is united once per adjacency with the runs of the row
//     above (N at the first overlapping pixel, NW at the start, NE at the end);
//     the row above lives in registers (shuffles), border run ids too;
//   * afterwards run roots are compressed with a read-only find, integer
//     moments are summed per run in closed form into per-root slots (roots in
//     batches of 32), and interior components become regions, edge components
//     fragments + border labels, exactly as the block kernel emits them.
// Tiles with more than kWarpMaxRuns runs are appended to a deferred list and
// processed by the block kernel.
#include "adps_internal.cuh"
#include "attribution.cuh"

namespace adps {

#ifndef ADPS_TW_MAXRUNS
#define ADPS_TW_MAXRUNS 192
#endif
constexpr int kWarpMaxRuns = ADPS_TW_MAXRUNS;
constexpr int kWarpsPerBlock = 8;

#ifndef ADPS_TW_FAST
#define ADPS_TW_FAST 1
#endif
#ifndef ADPS_TW_ROWWISE
#define ADPS_TW_ROWWISE 0   // 1: the row-wise words pass (ballots) instead of the transposed one
#endif
#ifndef ADPS_TW_DOMROWS
#define ADPS_TW_DOMROWS 1   // stage the dominant ids of whole keyed rows
#endif
#ifndef ADPS_TW_MINBLOCKS
#define ADPS_TW_MINBLOCKS 5
#endif

template <int MR>
struct PostSmemT {                  // used after the row scan
  int aux[MR];                      // fragment id of a root, -1 otherwise
  int mom[32][6];
  unsigned char touch[32];
};

template <int MR>                   // MR: run capacity of the tile
struct WarpSmemT {
  int uf[MR];
  unsigned run[MR];                 // ty | s << 5 | e << 10 | band << 16
  union {
    PostSmemT<MR> post;
    int d[kTileH][kTileW];          // bit-plane path: fp32 raw cache of the tile rows (bit patterns),
                                    // then the dominant ids of keyed pixels
  } u;
};
using WarpSmem = WarpSmemT<kWarpMaxRuns>;
// the deferred tiles (more than kWarpMaxRuns runs) are redone by the same warp
// kernel with room for every possible run of a 32 x 32 tile
constexpr int kTileMaxRuns = kTileH * kTileW;
constexpr int kBigWarpsPerBlock = 4;

size_t tile_warp_smem_bytes() { return sizeof(WarpSmem) * kWarpsPerBlock; }

// per-tile scan state carried from row to row (registers)
struct TileRowState {
  unsigned long long m1, m2;   // metric masks of ext rows ey-1, ey-2
  int c_del, band_del;         // candidate/band of the tile row awaiting its erosion window
  int prev_key, prev_band, prev_rid;
  int b_top, b_bot, b_left, b_right;   // run id of border pixel `lane`
  int n_runs;
};

struct TileConst {
  const float* img;
  const float* gtv;
  const int* dom;
  const unsigned* cbits;   // candidate bits of the view
  const double* raw;       // cached raw L1 error of the view (RAW path)
  const double* thr;
  double x_m, t1, t2, t3;   // raw-domain thresholds of m and of bands 1..3
  long long p0;            // pixel index of (x0 + lane, y0 - HL): ext row ey is p0 + ey * W
  int W, L;
  int ey_lo, ey_hi;        // ext rows inside the image
  bool col_in;             // x0 + lane < W
  unsigned long long hl_mask, hr_mask;   // bit ey: metric bit of the left/right halo pixel of ext row ey
};

// one image row of the tile (lane = x)
// RAW: the minmax pass cached the fp64 raw L1 error per pixel (8 B instead
// of re-reading 24 B of image + gt and redoing the arithmetic)
template <bool RAW>
struct RowIn {
  float a[3], g[3];
  int d;        // dominant id (tile rows), else -1
  unsigned cb;  // candidate bits word holding this pixel (consumed in scan_row, so the
  int sh;       // loads stay in flight while the previous row is scanned); bit index
  bool inb;
};
template <>
struct RowIn<true> {
  double raw;
  int d;
  unsigned cb;
  int sh;
  bool inb;
};

template <int HL, bool RAW>
__device__ __forceinline__ void load_row(RowIn<RAW>& r, const TileConst& T, int ey, int lane) {
  r.inb = ey >= T.ey_lo && ey < T.ey_hi && T.col_in;
  const long long p = T.p0 + (long long)ey * T.W;
  const bool tile_row = ey >= HL && ey < HL + kTileH;
  if constexpr (RAW) {
    r.raw = r.inb ? __ldg(T.raw + p) : 0.0;
  } else {
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      r.a[c] = r.inb ? __ldg(T.img + 3 * p + c) : 0.0f;
      r.g[c] = r.inb ? __ldg(T.gtv + 3 * p + c) : 0.0f;
    }
  }
  // candidate bit (written by the minmax pass) instead of a dependent cls[D] load
  const bool need = r.inb && tile_row;
  r.d = need ? __ldg(T.dom + p) : -1;
  r.cb = need ? __ldg(T.cbits + (p >> 5)) : 0u;
  r.sh = (int)(p & 31);
}

// np.abs(rendered - gt).sum(axis=-1) == (|d0| + |d1|) + |d2| in fp64
__device__ __forceinline__ double raw_l1_f(const float* a, const float* g) {
  const double a0 = fabs(dsub((double)a[0], (double)g[0]));
  const double a1 = fabs(dsub((double)a[1], (double)g[1]));
  const double a2 = fabs(dsub((double)a[2], (double)g[2]));
  return dadd(dadd(a0, a1), a2);
}

template <bool RAW>
__device__ __forceinline__ bool metric_at(const TileConst& T, int x, int y) {
  const long long p = (long long)y * T.W + x;
  if constexpr (RAW) {
    return __ldg(T.raw + p) >= T.x_m;
  } else {
    float a[3], g[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      a[c] = __ldg(T.img + 3 * p + c);
      g[c] = __ldg(T.gtv + 3 * p + c);
    }
    return raw_l1_f(a, g) >= T.x_m;
  }
}


// one ext row: metric mask, then (once its erosion window is complete) the
// runs of tile row ey - SPAN and their unions with the row above.
// Returns true when the tile has too many runs for the warp path.
template <bool RAW>
__device__ __forceinline__ double row_raw(const RowIn<RAW>& r) {
  if constexpr (RAW) return r.raw;
  else return raw_l1_f(r.a, r.g);
}


// the runs of one tile row (lane = x; key = candidate id or -1, band) and their
// unions with the runs of the row above (held in st.prev_*); K = keyed lanes.
// Returns true when the tile has too many runs for the warp path.
__device__ __forceinline__ bool runs_row(const int key, const int band, const unsigned K, const int ty,
                                         TileRowState& st, WarpSmem& S, const int lane) {
  constexpr unsigned FULL = 0xffffffffu;
#if ADPS_TW_FAST
  if (K == 0) {   // no keyed pixel in this row: no runs, nothing to unite
    st.prev_key = -1;
    st.prev_rid = -1;
    return false;
  }
#endif
  const int lkey = __shfl_up_sync(FULL, key, 1);
  const int lband = __shfl_up_sync(FULL, band, 1);
  const unsigned C = __ballot_sync(FULL, key >= 0 && lane > 0 && lkey == key && lband == band);
  const unsigned starts = K & ~C;
  const unsigned ends = K & ~(C >> 1);
  const int nr = __popc(starts);
  if (st.n_runs + nr > kWarpMaxRuns) return true;
  const bool is_start = (starts >> lane) & 1u;
  const bool is_end = (ends >> lane) & 1u;
  const int rid_start = st.n_runs + __popc(starts & ((1u << lane) - 1u));
  const int src = 31 - __clz(starts & (FULL >> (31 - lane)));
  const int rid_b = __shfl_sync(FULL, rid_start, src & 31);
  const int rid = key >= 0 ? rid_b : -1;
  if (is_start) {
    const int e = __ffs(ends & (FULL << lane)) - 1;
    S.run[rid] = (unsigned)ty | ((unsigned)lane << 5) | ((unsigned)e << 10) | ((unsigned)band << 16);
    S.uf[rid] = rid;
  }
  __syncwarp();
  // ---- one union per adjacency with the runs of the row above
  const int pk_m = __shfl_up_sync(FULL, st.prev_key, 1), pb_m = __shfl_up_sync(FULL, st.prev_band, 1);
  const int pr_m = __shfl_up_sync(FULL, st.prev_rid, 1);
  const int pk_p = __shfl_down_sync(FULL, st.prev_key, 1), pb_p = __shfl_down_sync(FULL, st.prev_band, 1);
  const int pr_p = __shfl_down_sync(FULL, st.prev_rid, 1);
  if (key >= 0 && ty > 0) {
    const bool a0 = st.prev_key == key && st.prev_band == band;
    const bool am = lane > 0 && pk_m == key && pb_m == band;
    const bool ap = lane < 31 && pk_p == key && pb_p == band;
    if (a0 && (is_start || !am)) uf_unite(S.uf, rid, st.prev_rid);
    if (is_start && am && !a0) uf_unite(S.uf, rid, pr_m);
    if (is_end && ap && !a0) uf_unite(S.uf, rid, pr_p);
  }
  if (ty == 0) st.b_top = rid;
  if (ty == kTileH - 1) st.b_bot = rid;
  const int lc = __shfl_sync(FULL, rid, 0), rc = __shfl_sync(FULL, rid, 31);
  if (lane == ty) {
    st.b_left = lc;
    st.b_right = rc;
  }
  st.prev_key = key;
  st.prev_band = band;
  st.prev_rid = rid;
  st.n_runs += nr;
  return false;
}

template <int R, bool RAW>
__device__ __forceinline__ bool scan_row(const RowIn<RAW>& row, const int ey, TileRowState& st, WarpSmem& S,
                                         const TileConst& T, const int lane) {
  const bool inb = row.inb;
  const int c_now = (row.cb >> row.sh) & 1u ? row.d : -1;
  constexpr int HL = R > 1 ? R / 2 : 0;
  constexpr int HH = R > 1 ? R - R / 2 - 1 : 0;
  constexpr int SPAN = HL + HH;
  constexpr unsigned FULL = 0xffffffffu;
  bool m = false;
  int band_now = 0;
  if (inb) {
    const double xr = row_raw<RAW>(row);   // thresholds are in the raw domain
    m = xr >= T.x_m;
    if (T.L <= 4) {
      band_now = (xr >= T.t1) + (xr >= T.t2) + (xr >= T.t3);
    } else {
      for (int q = 1; q < T.L; ++q) band_now += xr >= T.thr[q];
    }
  }
  unsigned long long m0 = (unsigned long long)__ballot_sync(FULL, m) << HL;
  if (HL > 0) m0 |= (T.hl_mask >> ey) & 1ull;
  if (HH > 0) m0 |= ((T.hr_mask >> ey) & 1ull) << (kTileW + HL);
  const int ty = ey - SPAN;
  bool overflow = false;
  if (ty >= 0) {
    unsigned long long acc = m0;
    if (SPAN >= 1) acc &= st.m1;
    if (SPAN >= 2) acc &= st.m2;
    unsigned long long h = acc;
    if (SPAN >= 1) h &= acc >> 1;
    if (SPAN >= 2) h &= acc >> 2;
    const unsigned er = (unsigned)h;
    const int cand = HH > 0 ? st.c_del : c_now;
    const int band = HH > 0 ? st.band_del : band_now;
    const int key = ((er >> lane) & 1u) ? cand : -1;
    // ---- runs of equal (candidate, band)
    const unsigned K = __ballot_sync(FULL, key >= 0);
    overflow = runs_row(key, band, K, ty, st, S, lane);
  }
  st.m2 = st.m1;
  st.m1 = m0;
  st.c_del = c_now;
  st.band_del = band_now;
  return overflow;
}

// components of a scanned tile (runs in S, border run ids in st): roots by a
// read-only find, integer moments per root in closed form per run; interior
// components >= m_min become regions, edge components fragments + border labels
template <class WS>
__device__ __forceinline__ void finish_tile(const TileParams& P, WS& S, const int* __restrict__ dom_v,
                                            const long long tile, const int v, const int x0, const int y0,
                                            const TileRowState& st, const int lane) {
  constexpr unsigned FULL = 0xffffffffu;
  const int W = P.W, H = P.H;
  const int n_runs = st.n_runs;
  const int b_top = st.b_top, b_bot = st.b_bot, b_left = st.b_left, b_right = st.b_right;
  __syncwarp();
  // ---- roots (read-only finds: stored roots are never overwritten)
  for (int b = 0; b < n_runs; b += 32) {   // warp-uniform trip count
    const int q = b + lane;
    if (q < n_runs) {
      S.uf[q] = uf_find(S.uf, q);
      S.u.post.aux[q] = -1;
    }
  }
  __syncwarp();
  const bool left_in = x0 > 0, top_in = y0 > 0;
  const bool right_in = x0 + kTileW < W, bottom_in = y0 + kTileH < H;
  for (int base = 0; base < n_runs; base += 32) {
    const int q = base + lane;
    const bool is_root = q < n_runs && S.uf[q] == q;
    const unsigned roots = __ballot_sync(FULL, is_root);
    if (!roots) continue;
    // integer moments of this batch's roots, one closed form per run
#pragma unroll
    for (int k = 0; k < 6; ++k) S.u.post.mom[lane][k] = 0;
    S.u.post.touch[lane] = 0;
    __syncwarp();
    for (int b2 = 0; b2 < n_runs; b2 += 32) {   // warp-uniform trip count
      const int q2 = b2 + lane;
      if (q2 >= n_runs) continue;
      const int root = S.uf[q2];
      if (root < base || root >= base + 32) continue;
      const int sl = __popc(roots & ((1u << (root - base)) - 1u));
      const unsigned info = S.run[q2];
      const int ty = info & 31, s = (info >> 5) & 31, e = (info >> 10) & 31;
      const int n = e - s + 1;
      const int sx = (s + e) * n / 2;
      const int sxx = (e * (e + 1) * (2 * e + 1) - (s - 1) * s * (2 * s - 1)) / 6;
      atomicAdd(&S.u.post.mom[sl][0], n);
      atomicAdd(&S.u.post.mom[sl][1], sx);
      atomicAdd(&S.u.post.mom[sl][2], ty * n);
      atomicAdd(&S.u.post.mom[sl][3], sxx);
      atomicAdd(&S.u.post.mom[sl][4], ty * sx);
      atomicAdd(&S.u.post.mom[sl][5], ty * ty * n);
      if ((ty == 0 && top_in) || (ty == kTileH - 1 && bottom_in) || (s == 0 && left_in) ||
          (e == kTileW - 1 && right_in))
        S.u.post.touch[sl] = 1;
    }
    __syncwarp();
    // records: fragments for edge components, regions for interior ones >= m_min
    const int sl = __popc(roots & ((1u << lane) - 1u));
    const bool is_part = is_root && S.u.post.touch[sl];
    const bool is_reg = is_root && !S.u.post.touch[sl] && S.u.post.mom[sl][0] >= P.m_min;
    const unsigned pm = __ballot_sync(FULL, is_part), rm = __ballot_sync(FULL, is_reg);
    unsigned long long pbase = 0, rbase = 0;
    if (lane == 0 && (pm | rm)) {   // one atomic for both record kinds (partials << 32 | regions)
      const unsigned long long old =
          atomicAdd(P.tile_records, ((unsigned long long)__popc(pm) << 32) | (unsigned long long)__popc(rm));
      pbase = old >> 32;
      rbase = old & 0xffffffffull;
    }
    pbase = __shfl_sync(FULL, pbase, 0);
    rbase = __shfl_sync(FULL, rbase, 0);
    if (is_part || is_reg) {
      const unsigned info = S.run[q];
      const int ty = info & 31, s = (info >> 5) & 31, bnd = (info >> 16) & 0xff;
      const long long n = S.u.post.mom[sl][0], mx = S.u.post.mom[sl][1], my = S.u.post.mom[sl][2];
      const long long X = x0, Y = y0;
      long long gm[6];
      gm[0] = n;
      gm[1] = mx + n * X;
      gm[2] = my + n * Y;
      gm[3] = (long long)S.u.post.mom[sl][3] + 2 * X * mx + n * X * X;
      gm[4] = (long long)S.u.post.mom[sl][4] + X * my + Y * mx + n * X * Y;
      gm[5] = (long long)S.u.post.mom[sl][5] + 2 * Y * my + n * Y * Y;
      const int minpix = (y0 + ty) * W + (x0 + s);
      const int cand = __ldg(dom_v + minpix);
      if (is_part) {
        const unsigned long long gid = pbase + __popc(pm & ((1u << lane) - 1u));
        if ((long long)gid < P.partial_cap) {
          PartialRec& Rr = P.partials[gid];
          Rr.view_pos = P.view_offset + v * P.view_stride;
          Rr.cand = cand;
          Rr.band = bnd;
          Rr.minpix = minpix;
#pragma unroll
          for (int k = 0; k < 6; ++k) Rr.m[k] = gm[k];
          P.partial_parent[gid] = (int)gid;
          S.u.post.aux[q] = (int)gid;
        } else {
          atomicOr(P.overflow, 2u);
        }
      } else {
        const unsigned long long rid2 = rbase + __popc(rm & ((1u << lane) - 1u));
        if ((long long)rid2 < P.region_cap) {
          RegionRec& Rr = P.regions[rid2];
          Rr.view_pos = P.view_offset + v * P.view_stride;
          Rr.cand = cand;
          Rr.band = bnd;
          Rr.minpix = minpix;
#pragma unroll
          for (int k = 0; k < 6; ++k) Rr.m[k] = gm[k];
        } else {
          atomicOr(P.overflow, 1u);
        }
      }
    }
    __syncwarp();
  }
  // ---- border labels: top, bottom, left, right (slot = side * 32 + lane)
  int* border = P.border + tile * kBorderSlots;
  border[lane] = b_top >= 0 ? S.u.post.aux[S.uf[b_top]] : -1;
  border[kTileW + lane] = b_bot >= 0 ? S.u.post.aux[S.uf[b_bot]] : -1;
  border[2 * kTileW + lane] = b_left >= 0 ? S.u.post.aux[S.uf[b_left]] : -1;
  border[2 * kTileW + kTileH + lane] = b_right >= 0 ? S.u.post.aux[S.uf[b_right]] : -1;
}


template <int R, bool RAW>
__device__ __forceinline__ void tile_warp_body(const TileParams& P, WarpSmem& S, const long long tile,
                                               const int lane) {
  constexpr int HL = R > 1 ? R / 2 : 0;
  constexpr int HH = R > 1 ? R - R / 2 - 1 : 0;
  constexpr int SPAN = HL + HH;
  constexpr int NR = kTileH + SPAN;   // ext rows
  constexpr unsigned FULL = 0xffffffffu;
  const int tiles_per_view = P.tiles_x * P.tiles_y;
  const int v = (int)(tile / tiles_per_view);
  const int tin = (int)(tile % tiles_per_view);
  TileConst T;
  const int x0 = (tin % P.tiles_x) * kTileW, y0 = (tin / P.tiles_x) * kTileH;
  const int W = P.W, H = P.H;
  T.W = W;
  T.p0 = (long long)(y0 - HL) * W + x0 + lane;
  T.ey_lo = HL - y0 > 0 ? HL - y0 : 0;
  T.ey_hi = H - y0 + HL < NR ? H - y0 + HL : NR;
  T.col_in = x0 + lane < W;
  const long long hw = (long long)W * H;
  T.img = P.image + (long long)v * hw * 3;
  T.gtv = P.gt + (long long)v * hw * 3;
  T.dom = P.dom + (long long)v * hw;
  T.cbits = P.cand_bits + (long long)v * ((hw + 31) / 32);
  T.raw = RAW ? P.raw + (long long)v * hw : nullptr;
  T.L = P.L;
  T.thr = P.thr_raw + (long long)v * P.L;   // raw-domain thresholds (thresholds_kernel)
  T.x_m = T.thr[0];
  const double kInf = __longlong_as_double(0x7ff0000000000000ll);
  T.t1 = T.L > 1 ? T.thr[1] : kInf;
  T.t2 = T.L > 2 ? T.thr[2] : kInf;
  T.t3 = T.L > 3 ? T.thr[3] : kInf;
  // halo columns of all ext rows at once (lane = ext row, then ext rows 32..)
  T.hl_mask = 0;
  T.hr_mask = 0;
  if (SPAN > 0) {
#pragma unroll
    for (int k = 0; k < (NR + 31) / 32; ++k) {
      const int ey = lane + 32 * k;
      const int y = y0 - HL + ey;
      const bool row_ok = ey < NR && y >= 0 && y < H;
      const bool ml = HL > 0 && row_ok && x0 - 1 >= 0 && metric_at<RAW>(T, x0 - 1, y);
      const bool mr = HH > 0 && row_ok && x0 + kTileW < W && metric_at<RAW>(T, x0 + kTileW, y);
      T.hl_mask |= (unsigned long long)__ballot_sync(FULL, ml) << (32 * k);
      T.hr_mask |= (unsigned long long)__ballot_sync(FULL, mr) << (32 * k);
    }
  }

  TileRowState st;
  st.m1 = st.m2 = 0;
  st.c_del = -1;
  st.band_del = 0;
  st.prev_key = -1;
  st.prev_band = 0;
  st.prev_rid = -1;
  st.b_top = st.b_bot = st.b_left = st.b_right = -1;
  st.n_runs = 0;
  bool overflow = false;
  {
    // rows are loaded one ahead into two alternating register buffers (deeper
    // rings measured slower: register spills)
    RowIn<RAW> A, B;
    load_row<HL, RAW>(A, T, 0, lane);
    for (int ey = 0; ey < NR; ey += 2) {
      if (ey + 1 < NR) load_row<HL, RAW>(B, T, ey + 1, lane);
      if (scan_row<R, RAW>(A, ey, st, S, T, lane)) {
        overflow = true;
        break;
      }
      if (ey + 1 < NR) {
        if (ey + 2 < NR) load_row<HL, RAW>(A, T, ey + 2, lane);
        if (scan_row<R, RAW>(B, ey + 1, st, S, T, lane)) {
          overflow = true;
          break;
        }
      }
    }
  }
  if (overflow) {
    if (lane == 0) P.deferred[atomicAdd(P.n_deferred, 1ull)] = (int)tile;
    return;
  }
  finish_tile(P, S, T.dom, tile, v, x0, y0, st, lane);
}

template <int R, bool RAW>
__global__ void __launch_bounds__(kWarpsPerBlock * 32, ADPS_TW_MINBLOCKS) tile_warp_kernel(TileParams P, long long t0, long long t1) {
  pdl_wait();   // programmatic dependent launch: the previous kernel's results are visible
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  WarpSmem& S = reinterpret_cast<WarpSmem*>(smem_raw)[wid];
  const long long tile = t0 + (long long)blockIdx.x * kWarpsPerBlock + wid;
  if (tile >= t1) return;   // warp-uniform
  tile_warp_body<R, RAW>(P, S, tile, lane);
}


// ===================================================================== bit planes
// The common configuration (raw cache on, l_bands <= 4) splits the tile pass:
//   tile_words_kernel  streams the cached raw error once (coalesced, several
//                      32-pixel words in flight per warp) and writes, per image
//                      row and 32-column word, four bit planes: metric bit,
//                      candidate bit, band bit 0, band bit 1 (16 B per 32 px);
//   tile_bits_kernel   the warp-per-tile scanline CCL on those words: the whole
//                      tile's masks arrive in one 16-byte load per lane (lane =
//                      ext row), erosion and keying are word operations, tiles
//                      without a keyed pixel exit at once, and only keyed rows
//                      are scanned; the dominant ids of keyed pixels are staged in
//                      shared memory with cp.async (one wait per tile).
// Same run numbering, unions and records as tile_warp_kernel, so the results
// are identical bit for bit (tests compare all CCL paths).

// raw >= X with raw known as f = RZ_fp32(raw) (bit pattern fi; non-negative
// floats order as their bit patterns, the -1.0f sentinel is negative): with
// Xf = RZ_fp32(X), raw >= X  <=>  fi > bits(Xf), or fi == bits(Xf) and X == Xf;
// when fi == bits(Xf) and X is not a float the compare is ambiguous.  So
// m = fi >= T with T = bits(Xf) + (X != Xf), ambiguous when fi == A with
// A = bits(Xf) if X != Xf, else a value no pixel has.
struct RzThreshold {
  int T, A;
};
__device__ __forceinline__ RzThreshold rz_threshold(double X) {
  // against the 16-bit cache codes (raw16): the code of X is the top half of
  // RZ_fp32(X); X is representable iff it equals that fp32 value and the low
  // half is zero (+inf stays +inf: code 0x7f80, above every finite raw)
  const float xf = __double2float_rz(X);
  const unsigned b = __float_as_uint(xf);
  const int k = (int)(b >> 16);
  const bool exact = (double)xf == X && (b & 0xffffu) == 0u;
  return {exact ? k : k + 1, exact ? (int)0x80000000 : k};
}

__global__ void __launch_bounds__(256) tile_words_kernel(const raw16_t* __restrict__ rawf,
                                                         const float* __restrict__ image,
                                                         const float* __restrict__ gt,
                                                         const unsigned* __restrict__ cand_bits,
                                                         const double* __restrict__ thr_raw, int L, int H, int W,
                                                         int WW, int v0, uint4* __restrict__ words) {
  pdl_wait();   // programmatic dependent launch: the previous kernel's results are visible
  // one warp per image row, lane = x within a 32-column word, U words in flight
  const int v = v0 + blockIdx.y;
  const int y = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (y >= H) return;   // warp-uniform
  const int lane = threadIdx.x & 31;
  const long long hw = (long long)H * W;
  const long long nwords = (hw + 31) / 32;
  const long long p_row = (long long)y * W;
  const raw16_t* rrow = rawf + (long long)v * hw + p_row;
  const unsigned* cv = cand_bits + (long long)v * nwords;
  uint4* wrow = words + ((long long)v * H + y) * WW;
  const double* tv = thr_raw + (long long)v * L;
  const double kInf = __longlong_as_double(0x7ff0000000000000ll);
  const double X0 = __ldg(tv), X1 = L > 1 ? __ldg(tv + 1) : kInf, X2 = L > 2 ? __ldg(tv + 2) : kInf,
               X3 = L > 3 ? __ldg(tv + 3) : kInf;
  const RzThreshold R0 = rz_threshold(X0), R1 = rz_threshold(X1), R2 = rz_threshold(X2), R3 = rz_threshold(X3);
  const int sh = (int)(p_row & 31);
  const unsigned* crow = cv + (p_row >> 5);   // linear candidate words of this row (+1 padding word)
  auto emit_word = [&](int wx, int fi, unsigned lo, unsigned hi) {
    bool m = fi >= R0.T;
    int band = (fi >= R1.T) + (fi >= R2.T) + (fi >= R3.T);
    const bool amb = (fi == R0.A) | (fi == R1.A) | (fi == R2.A) | (fi == R3.A);
    if (__any_sync(0xffffffffu, amb) && amb) {   // rare: the exact fp64 raw error, numpy order
      const long long p = (long long)v * hw + p_row + wx * 32 + lane;
      const float* a3 = image + 3 * p;
      const float* g3 = gt + 3 * p;
      const double d0 = fabs(dsub((double)a3[0], (double)g3[0]));
      const double d1 = fabs(dsub((double)a3[1], (double)g3[1]));
      const double d2 = fabs(dsub((double)a3[2], (double)g3[2]));
      const double xr = dadd(dadd(d0, d1), d2);
      m = xr >= X0;
      band = (xr >= X1) + (xr >= X2) + (xr >= X3);
    }
    const unsigned M = __ballot_sync(0xffffffffu, m);
    const unsigned B0 = __ballot_sync(0xffffffffu, band & 1);
    const unsigned B1 = __ballot_sync(0xffffffffu, band & 2);
    unsigned C = __funnelshift_r(lo, hi, sh);
    const int valid = W - wx * 32;   // columns of this word inside the row
    if (valid < 32) C &= (1u << valid) - 1u;
    return make_uint4(M, C, B0, B1);
  };
  constexpr int U = 8;
  const int WWf = W >> 5;   // full words
  int wx0 = 0;
  for (; wx0 + U <= WWf; wx0 += U) {   // full words: no bounds checks
    int r[U];
    unsigned cw[U + 1];
#pragma unroll
    for (int u = 0; u < U; ++u) r[u] = __ldg(rrow + (wx0 + u) * 32 + lane);
#pragma unroll
    for (int u = 0; u <= U; ++u) cw[u] = __ldg(crow + wx0 + u);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint4 q = emit_word(wx0 + u, r[u], cw[u], cw[u + 1]);
      if (lane == u) wrow[wx0 + u] = q;
    }
  }
  if (wx0 < WW) {   // the rest (< U words), loads issued together
    int r[U];
    unsigned cw[U + 1];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int x = (wx0 + u) * 32 + lane;
      r[u] = x < W ? (int)__ldg(rrow + x) : -1;   // below every threshold
    }
#pragma unroll
    for (int u = 0; u <= U; ++u) cw[u] = wx0 + u <= WW ? __ldg(crow + wx0 + u) : 0u;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (wx0 + u < WW) {   // warp-uniform
        const uint4 q = emit_word(wx0 + u, r[u], cw[u], cw[u + 1]);
        if (lane == u) wrow[wx0 + u] = q;
      }
    }
  }
}

// The same bit planes, transposed: a warp per 32 x 32 pixel block (rows y0..+31
// of word column tx).  The block's raw cache is staged in shared memory with
// coalesced cp.async rows, then lane = row builds its row's four words with
// shifts from 32 conflict-free shared loads (row stride 33 words) -- about 12
// instructions per pixel-lane instead of a ballot round per word and plane.
// Ambiguous pixels redo the exact fp64 raw error, exactly as tile_words_kernel.
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

#ifndef ADPS_TW_WARPS
#define ADPS_TW_WARPS 8
#endif
constexpr int kTwWarps = ADPS_TW_WARPS;   // warps (32-pixel word columns) per block of the words pass
__global__ void __launch_bounds__(kTwWarps * 32) tile_words_t_kernel(const raw16_t* __restrict__ rawf,
                                                                    const float* __restrict__ image,
                                                                    const float* __restrict__ gt,
                                                                    const unsigned* __restrict__ cand_bits,
                                                                    const double* __restrict__ thr_raw, int L, int H,
                                                                    int W, int WW, int v0, uint4* __restrict__ words) {
  pdl_wait();   // programmatic dependent launch: the previous kernel's results are visible
  __shared__ int tile[kTwWarps][32][33];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int v = v0 + blockIdx.z;
  const int tx = blockIdx.x * kTwWarps + wid;
  if (tx >= WW) return;   // warp-uniform
  const int y0 = blockIdx.y * 32;
  const int x0 = tx * 32;
  const long long hw = (long long)H * W;
  const raw16_t* rv = rawf + (long long)v * hw;
  int (*S)[33] = tile[wid];
  const bool col_in = x0 + lane < W;
  const int nrows = H - y0 < 32 ? H - y0 : 32;
  // coalesced 64-byte row loads, 8 rows in flight, into shared memory
  for (int r0 = 0; r0 < nrows; r0 += 8) {
    int t[8];
#pragma unroll
    for (int k = 0; k < 8; ++k)
      t[k] = r0 + k < nrows && col_in ? (int)__ldg(rv + (long long)(y0 + r0 + k) * W + x0 + lane) : -1;
#pragma unroll
    for (int k = 0; k < 8; ++k)
      if (r0 + k < nrows) S[r0 + k][lane] = t[k];   // -1: below every threshold
  }
  // thresholds of the view (warp-uniform) while the copies fly
  const double* tv = thr_raw + (long long)v * L;
  const double kInf = __longlong_as_double(0x7ff0000000000000ll);
  const double X0 = __ldg(tv), X1 = L > 1 ? __ldg(tv + 1) : kInf, X2 = L > 2 ? __ldg(tv + 2) : kInf,
               X3 = L > 3 ? __ldg(tv + 3) : kInf;
  const RzThreshold R0 = rz_threshold(X0), R1 = rz_threshold(X1), R2 = rz_threshold(X2), R3 = rz_threshold(X3);
  // candidate word of row y0 + lane
  const int y = y0 + lane;
  unsigned C = 0u;
  if (lane < nrows) {
    const unsigned* cv = cand_bits + (long long)v * ((hw + 31) / 32);
    const long long p = (long long)y * W + x0;
    C = __funnelshift_r(__ldg(cv + (p >> 5)), __ldg(cv + (p >> 5) + 1), (int)(p & 31));
    const int valid = W - x0;
    if (valid < 32) C &= (1u << valid) - 1u;
  }
  __syncwarp();
  if (lane >= nrows) return;
  // one compare and one predicated OR per plane and pixel (the bit is an
  // immediate after unrolling); band = t1 + t2 + t3 with monotone thresholds,
  // so its bit 0 is t1 ^ t2 ^ t3 and its bit 1 is t2 (word operations after)
  unsigned M = 0u, P1 = 0u, P2 = 0u, P3 = 0u, amb = 0u;
  const int T0 = R0.T, T1 = R1.T, T2 = R2.T, T3 = R3.T;
  const int A0 = R0.A, A1 = R1.A, A2 = R2.A, A3 = R3.A;
#pragma unroll
  for (int x = 0; x < 32; ++x) {
    const int fi = S[lane][x];
    const unsigned bit = 1u << x;
    if (fi >= T0) M |= bit;
    if (fi >= T1) P1 |= bit;
    if (fi >= T2) P2 |= bit;
    if (fi >= T3) P3 |= bit;
    if (fi == A0 || fi == A1 || fi == A2 || fi == A3) amb |= bit;
  }
  unsigned B0 = P1 ^ P2 ^ P3, B1 = P2;
  for (; amb; amb &= amb - 1u) {   // rare: the exact fp64 raw error, numpy order
    const int x = __ffs(amb) - 1;
    const long long p = (long long)v * hw + (long long)y * W + x0 + x;
    const float* a3 = image + 3 * p;
    const float* g3 = gt + 3 * p;
    const double xr = dadd(dadd(fabs(dsub((double)a3[0], (double)g3[0])), fabs(dsub((double)a3[1], (double)g3[1]))),
                           fabs(dsub((double)a3[2], (double)g3[2])));
    const unsigned bit = 1u << x;
    const int band = (xr >= X1) + (xr >= X2) + (xr >= X3);
    M = (M & ~bit) | (xr >= X0 ? bit : 0u);
    B0 = (B0 & ~bit) | ((band & 1) ? bit : 0u);
    B1 = (B1 & ~bit) | ((band & 2) ? bit : 0u);
  }
  words[((long long)v * H + y) * WW + tx] = make_uint4(M, C, B0, B1);
}

// the word of ext row ey (image row y0 - HL + ey) of tile column tx, and its
// 64-bit metric mask with the left/right halo bits (bit HL = column x0)
template <int HL, int HH>
__device__ __forceinline__ void load_ext_words(const uint4* __restrict__ wv, int WW, int H, int tx, int y0, int ey,
                                               int NR, uint4& q, unsigned long long& m64) {
  const int y = y0 - HL + ey;
  q = make_uint4(0u, 0u, 0u, 0u);
  m64 = 0ull;
  if (ey < NR && y >= 0 && y < H) {
    const uint4* row = wv + (long long)y * WW;
    q = __ldg(row + tx);
    m64 = (unsigned long long)q.x << HL;
    if (HL > 0 && tx > 0) m64 |= (unsigned long long)(__ldg(reinterpret_cast<const unsigned*>(row + tx - 1)) >> 31);
    if (HH > 0 && tx + 1 < WW)
      m64 |= (unsigned long long)(__ldg(reinterpret_cast<const unsigned*>(row + tx + 1)) & 1u) << (kTileW + HL);
  }
}

// value of ext row ey held by lane ey (set a) or lane ey - 32 (set b)
template <typename Tv>
__device__ __forceinline__ Tv ext_get(Tv a, Tv b, int ey) {
  const Tv va = __shfl_sync(0xffffffffu, a, ey & 31);
  const Tv vb = __shfl_sync(0xffffffffu, b, ey & 31);
  return ey < 32 ? va : vb;
}


// The bit planes of one tile computed in place from the fp32 raw cache (no
// words pass): lane = column, one coalesced row load per needed ext row, the
// same exact compares as tile_words_kernel (ambiguous pixels redo the fp64 raw
// error from image and gt), ballots to words.  The candidate words come first:
// a tile without a candidate pixel exits before touching the raw cache, and
// only ext rows inside the erosion window of a candidate row are thresholded.
// Out: ma / mb = 64-bit metric masks (halo bits included) of ext rows lane and
// 32 + lane, cw / bw0 / bw1 = candidate and band words of tile row lane.
template <int HL, int HH, class WS>
__device__ __forceinline__ bool fused_tile_rows(const TileParams& P, WS& S, int v, int x0, int y0, int lane,
                                                unsigned long long& ma, unsigned long long& mb, unsigned& cw,
                                                unsigned& bw0, unsigned& bw1) {
  constexpr int SPAN = HL + HH;
  constexpr int NR = kTileH + SPAN;
  static_assert(HL <= 1 && HH <= 1, "fused bit planes: erosion halo of one pixel");
  constexpr unsigned FULL = 0xffffffffu;
  const int W = P.W, H = P.H;
  const long long hw = (long long)H * W;
  ma = mb = 0ull;
  cw = bw0 = bw1 = 0u;
  {   // candidate word of tile row `lane`
    const int y = y0 + lane;
    if (y < H) {
      const unsigned* cv = P.cand_bits + (long long)v * ((hw + 31) / 32);
      const long long p = (long long)y * W + x0;
      const unsigned lo = __ldg(cv + (p >> 5)), hi = __ldg(cv + (p >> 5) + 1);
      cw = __funnelshift_r(lo, hi, (int)(p & 31));
      const int valid = W - x0;
      if (valid < 32) cw &= (1u << valid) - 1u;
    }
  }
  const unsigned cmask = __ballot_sync(FULL, cw != 0u);
  if (cmask == 0u) return false;
  // ext rows to threshold: those inside the erosion window of a candidate row
  // (tile rows ty in [ey - SPAN, ey] use ext row ey)
  unsigned long long need = (unsigned long long)cmask;
  if (SPAN >= 1) need |= (unsigned long long)cmask << 1;
  if (SPAN >= 2) need |= (unsigned long long)cmask << 2;
  {
    const int y_lo = y0 - HL, y_hi = H - 1 - (y0 - HL);   // ext row ey is inside the image iff 0 <= y_lo + ey < H
    if (y_lo < 0) need &= ~((1ull << (-y_lo)) - 1ull);
    if (y_hi < NR - 1) need &= (2ull << y_hi) - 1ull;
  }
  const raw16_t* rv = P.rawf + (long long)v * hw;
  const bool inb = x0 + lane < W;
  // ---- stage the needed rows' raw bit patterns (cp.async, all in flight):
  //      tile rows into S.u.d, the halo pixels of every ext row into S.halo
  for (unsigned long long r = need; r; r &= r - 1ull) {
    const int ey = __ffsll((long long)r) - 1;
    const long long prow = (long long)(y0 - HL + ey) * W;
    const int ty = ey - HL;
    if (ty >= 0 && ty < kTileH && inb) S.u.d[ty][lane] = (int)__ldg(rv + prow + x0 + lane);
  }
  // lane ey (and 32 + lane): the halo pixels x0 - 1 (if HL) and x0 + 32 (if HH) of
  // ext row ey, in registers (loads in flight with the copies)
  int hl_a = -1, hr_a = -1, hl_b = -1, hr_b = -1;   // -1: below every threshold
#pragma unroll
  for (int h = 0; h < (NR > 32 ? 2 : 1); ++h) {
    const int ey = lane + 32 * h;
    if (ey < NR && ((need >> ey) & 1ull)) {
      const long long prow = (long long)(y0 - HL + ey) * W;
      if (HL > 0 && x0 > 0) (h ? hl_b : hl_a) = (int)__ldg(rv + prow + x0 - 1);
      if (HH > 0 && x0 + kTileW < W) (h ? hr_b : hr_a) = (int)__ldg(rv + prow + x0 + kTileW);
    }
  }
  // halo rows (outside the tile rows) straight into registers
  int f_top = -1, f_bot = -1;   // below every threshold
  if (HL > 0 && (need & 1ull) && inb) f_top = (int)__ldg(rv + (long long)(y0 - 1) * W + x0 + lane);
  if (HH > 0 && ((need >> (NR - 1)) & 1ull) && inb) f_bot = (int)__ldg(rv + (long long)(y0 + kTileH) * W + x0 + lane);
  const double* tv = P.thr_raw + (long long)v * P.L;
  const double kInf = __longlong_as_double(0x7ff0000000000000ll);
  const double X0 = __ldg(tv), X1 = P.L > 1 ? __ldg(tv + 1) : kInf, X2 = P.L > 2 ? __ldg(tv + 2) : kInf,
               X3 = P.L > 3 ? __ldg(tv + 3) : kInf;
  const RzThreshold R0 = rz_threshold(X0), R1 = rz_threshold(X1), R2 = rz_threshold(X2), R3 = rz_threshold(X3);
  auto classify = [&](int fi, long long p, bool& m, int& band) {
    m = fi >= R0.T;
    band = (fi >= R1.T) + (fi >= R2.T) + (fi >= R3.T);
    const bool amb = (fi == R0.A) | (fi == R1.A) | (fi == R2.A) | (fi == R3.A);
    if (amb) {   // rare: the exact fp64 raw error, numpy order
      const float* a3 = P.image + 3 * p;
      const float* g3 = P.gt + 3 * p;
      const double xr = dadd(dadd(fabs(dsub((double)a3[0], (double)g3[0])), fabs(dsub((double)a3[1], (double)g3[1]))),
                             fabs(dsub((double)a3[2], (double)g3[2])));
      m = xr >= X0;
      band = (xr >= X1) + (xr >= X2) + (xr >= X3);
    }
  };
  __syncwarp();
  const int hx = lane == 0 ? x0 - 1 : x0 + kTileW;
  const bool h_on = (lane == 0 && HL > 0 && x0 > 0) || (lane == 1 && HH > 0 && x0 + kTileW < W);
  for (unsigned long long r = need; r; r &= r - 1ull) {   // warp-uniform
    const int ey = __ffsll((long long)r) - 1;
    const int ty = ey - HL;
    const long long prow = (long long)(y0 - HL + ey) * W;
    const int fi = !inb ? -1 : (ty < 0 ? f_top : (ty >= kTileH ? f_bot : S.u.d[ty][lane]));
    int fh = -1;
    if (HL > 0 || HH > 0) {   // lane 0: left halo of ext row ey, lane 1: right halo
      const int l = __shfl_sync(FULL, ey < 32 ? hl_a : hl_b, ey & 31);
      const int r = __shfl_sync(FULL, ey < 32 ? hr_a : hr_b, ey & 31);
      fh = !h_on ? -1 : (lane == 0 ? l : r);
    }
    bool m, mh;
    int band, bh;
    classify(fi, (long long)v * hw + prow + x0 + lane, m, band);
    classify(fh, (long long)v * hw + prow + hx, mh, bh);
    const unsigned M = __ballot_sync(FULL, m);
    const unsigned hb = __ballot_sync(FULL, mh && h_on);
    unsigned long long m64 = (unsigned long long)M << HL;
    if (HL > 0) m64 |= (unsigned long long)(hb & 1u);
    if (HH > 0) m64 |= (unsigned long long)((hb >> 1) & 1u) << (kTileW + HL);
    if (lane == (ey & 31)) {
      if (ey < 32) ma = m64;
      else mb = m64;
    }
    if (ty >= 0 && ty < kTileH && ((cmask >> ty) & 1u)) {   // warp-uniform: band words of a candidate row
      const unsigned B0 = __ballot_sync(FULL, band & 1), B1 = __ballot_sync(FULL, band & 2);
      if (lane == ty) {
        bw0 = B0;
        bw1 = B1;
      }
    }
  }
  __syncwarp();   // S.u.d is restaged with the dominant ids next
  return true;
}

template <int R, bool FUSED, int MR>
__device__ __forceinline__ void tile_bits_body(const TileParams& P, const uint4* __restrict__ words, int WW,
                                               WarpSmemT<MR>& S, const long long tile, const int lane) {
  constexpr int HL = R > 1 ? R / 2 : 0;
  constexpr int HH = R > 1 ? R - R / 2 - 1 : 0;
  constexpr int SPAN = HL + HH;
  constexpr int NR = kTileH + SPAN;
  constexpr unsigned FULL = 0xffffffffu;
  const int tpv = P.tiles_x * P.tiles_y;
  const int v = (int)(tile / tpv);
  const int tin = (int)(tile - (long long)v * tpv);
  const int tx = tin % P.tiles_x;
  const int x0 = tx * kTileW, y0 = (tin / P.tiles_x) * kTileH;
  const int W = P.W, H = P.H;
  unsigned long long ma, mb = 0ull;
  unsigned cw, bw0, bw1;
  bool any_cand = true;
  if (FUSED) {
    any_cand = fused_tile_rows<HL, HH>(P, S, v, x0, y0, lane, ma, mb, cw, bw0, bw1);
  } else {
    const uint4* wv = words + (long long)v * H * WW;
    // ---- all ext rows of the tile: lane ey (and 32 + lane for the last SPAN rows)
    uint4 qa, qb = make_uint4(0u, 0u, 0u, 0u);
    load_ext_words<HL, HH>(wv, WW, H, tx, y0, lane, NR, qa, ma);
    if (NR > 32) load_ext_words<HL, HH>(wv, WW, H, tx, y0, 32 + lane, NR, qb, mb);
    cw = HL > 0 ? ext_get(qa.y, qb.y, lane + HL) : qa.y;
    bw0 = HL > 0 ? ext_get(qa.z, qb.z, lane + HL) : qa.z;
    bw1 = HL > 0 ? ext_get(qa.w, qb.w, lane + HL) : qa.w;
  }
  // ---- lane ty: eroded metric word of tile row ty, its candidate and band words
  unsigned long long acc = ma;
  if (SPAN >= 1) acc &= ext_get(ma, mb, lane + 1);
  if (SPAN >= 2) acc &= ext_get(ma, mb, lane + 2);
  unsigned long long h = acc;
  if (SPAN >= 1) h &= acc >> 1;
  if (SPAN >= 2) h &= acc >> 2;
  const unsigned K = any_cand ? (unsigned)h & cw : 0u;
  const unsigned keyed = __ballot_sync(FULL, K != 0u);
  int* border = P.border + tile * kBorderSlots;
  if (keyed == 0u) {   // no keyed pixel: no runs, no records, empty border labels
#pragma unroll
    for (int k = 0; k < 4; ++k) border[32 * k + lane] = -1;
    return;
  }
  // ---- stage the dominant ids of keyed pixels (one wait for the whole tile)
  const int* dom_v = P.dom + (long long)v * H * W;
#if ADPS_TW_DOMROWS
  {   // whole keyed rows (in-image columns): no per-pixel key test or shuffle
    const int* drow = dom_v + (long long)y0 * W + x0 + lane;
    if (x0 + lane < W)
      for (unsigned rows = keyed; rows; rows &= rows - 1u) {
        const int ty = __ffs(rows) - 1;
        cp_async4(&S.u.d[ty][lane], drow + (long long)ty * W);
      }
  }
#else
  for (unsigned rows = keyed; rows; rows &= rows - 1u) {
    const int ty = __ffs(rows) - 1;
    const unsigned kw = __shfl_sync(FULL, K, ty);
    if ((kw >> lane) & 1u) cp_async4(&S.u.d[ty][lane], dom_v + (long long)(y0 + ty) * W + x0 + lane);
  }
#endif
  cp_async_wait_all();
  // ---- (a) lane = column, per keyed row: the run-continuation mask (same
  //      key|band as the left neighbour) and the three vertical same-key masks
  //      against the row above (N, NW, NE); lane ty keeps row ty's masks.
  unsigned my_cc = 0u, my_v0 = 0u, my_vm = 0u, my_vp = 0u;
  {
    // key|band of the row above and of its left / right neighbours (-1 when
    // that row is not keyed): the neighbours are this row's shuffles carried
    // over, so a row costs two shuffles of kb instead of three
    int kb_prev = -1, lkb_prev = -1, rkb_prev = -1;
    int last = -2;
    for (unsigned rows = keyed; rows; rows &= rows - 1u) {
      const int ty = __ffs(rows) - 1;
      if (ty != last + 1) kb_prev = lkb_prev = rkb_prev = -1;
      last = ty;
      const unsigned kw = __shfl_sync(FULL, K, ty);
      const unsigned b0 = __shfl_sync(FULL, bw0, ty), b1 = __shfl_sync(FULL, bw1, ty);
      const int band = (int)((b0 >> lane) & 1u) | (int)(((b1 >> lane) & 1u) << 1);
      const bool kl = (kw >> lane) & 1u;
      const int kb = kl ? (S.u.d[ty][lane] << 2) | band : -1;   // ids < 2^29
      const int lkb = __shfl_up_sync(FULL, kb, 1), rkb = __shfl_down_sync(FULL, kb, 1);
      // lane 0's shfl_up / lane 31's shfl_down return their own value: masked below
      const unsigned cc = __ballot_sync(FULL, kl && lkb == kb) & ~1u;
      const unsigned v0 = __ballot_sync(FULL, kl && kb_prev == kb);
      const unsigned vm = __ballot_sync(FULL, kl && lkb_prev == kb) & ~1u;
      const unsigned vp = __ballot_sync(FULL, kl && rkb_prev == kb) & 0x7fffffffu;
      if (lane == ty) {
        my_cc = cc;
        my_v0 = v0;
        my_vm = vm;
        my_vp = vp;
      }
      kb_prev = kb;
      lkb_prev = lkb;
      rkb_prev = rkb;
    }
  }
  // ---- (b) lane = row from here on.  Runs: starts/ends of this row; run ids
  //      are row-major, so a row's base is the exclusive prefix of run counts
  const unsigned my_starts = K & ~my_cc;
  const unsigned my_ends = K & ~(my_cc >> 1);
  const int my_nr = __popc(my_starts);
  int base = my_nr;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(FULL, base, o);
    if (lane >= o) base += t;
  }
  const int n_runs = __shfl_sync(FULL, base, 31);
  base -= my_nr;
  if (n_runs > MR) {   // (never for MR = kTileMaxRuns)
    if (lane == 0) P.deferred[atomicAdd(P.n_deferred, 1ull)] = (int)tile;
    return;
  }
  // ---- (c) run records of this row
  // (warp-uniform trip counts with predicated bodies in (c), (d) and the
  // finish: per-lane loops left the warp split in two halves for the rest of
  // the tile -- ptxas placed no reconvergence point -- so every later
  // instruction issued twice)
  {
    int rid = base;
    unsigned st_bits = my_starts;
    while (__any_sync(FULL, st_bits != 0u)) {
      if (st_bits) {
        const int x = __ffs(st_bits) - 1;
        const int e = __ffs(my_ends & (FULL << x)) - 1;
        const int band = (int)((bw0 >> x) & 1u) | (int)(((bw1 >> x) & 1u) << 1);
        S.run[rid] = (unsigned)lane | ((unsigned)x << 5) | ((unsigned)e << 10) | ((unsigned)band << 16);
        S.uf[rid] = rid;
        st_bits &= st_bits - 1u;
        ++rid;
      }
    }
  }
  __syncwarp();
  // ---- (d) one union per adjacency with the runs of the row above (the rule
  //      of runs_row): N at the first overlapping pixel, NW at a run start,
  //      NE at a run end; run ids of both rows from popcounts of the starts
  {
    const unsigned sa = __shfl_up_sync(FULL, my_starts, 1);
    const int ba = __shfl_up_sync(FULL, base, 1);
    unsigned ev = (my_v0 & (my_starts | ~my_vm)) | (my_starts & my_vm & ~my_v0) | (my_ends & my_vp & ~my_v0);
    if (lane == 0) ev = 0u;
    while (__any_sync(FULL, ev != 0u)) {
      if (ev) {
        const int x = __ffs(ev) - 1;
        const unsigned bit = 1u << x, le = bit | (bit - 1u);
        const int rid = base + __popc(my_starts & le) - 1;
        const bool a0 = my_v0 & bit, am = my_vm & bit, is_start = my_starts & bit;
        if (a0 && (is_start || !am)) uf_unite(S.uf, rid, ba + __popc(sa & le) - 1);
        if (is_start && am && !a0) uf_unite(S.uf, rid, ba + __popc(sa & (bit - 1u)) - 1);
        if ((my_ends & bit) && (my_vp & bit) && !a0) uf_unite(S.uf, rid, ba + __popc(sa & ((le << 1) | 1u)) - 1);
        ev &= ev - 1u;
      }
    }
  }
  // ---- (e) border run ids: rows 0 / 31 at column `lane`, columns 0 / 31 of row `lane`
  TileRowState st;
  st.n_runs = n_runs;
  {
    __syncwarp();
    const unsigned lt = (1u << lane) - 1u;
    const unsigned k0w = __shfl_sync(FULL, K, 0), s0 = __shfl_sync(FULL, my_starts, 0);
    const unsigned k31 = __shfl_sync(FULL, K, kTileH - 1), s31 = __shfl_sync(FULL, my_starts, kTileH - 1);
    const int b0r = __shfl_sync(FULL, base, 0), b31r = __shfl_sync(FULL, base, kTileH - 1);
    const unsigned le = lt | (1u << lane);
    st.b_top = ((k0w >> lane) & 1u) ? b0r + __popc(s0 & le) - 1 : -1;
    st.b_bot = ((k31 >> lane) & 1u) ? b31r + __popc(s31 & le) - 1 : -1;
    st.b_left = (K & 1u) ? base : -1;
    st.b_right = (K >> 31) ? base + my_nr - 1 : -1;
  }
  __syncwarp();   // the key|band words share the union with the post-scan scratch
  finish_tile(P, S, dom_v, tile, v, x0, y0, st, lane);
}

template <int R, bool FUSED>
__global__ void __launch_bounds__(kWarpsPerBlock * 32, ADPS_TW_MINBLOCKS)
    tile_bits_kernel(TileParams P, const uint4* __restrict__ words, int WW, long long t0, long long t1) {
  pdl_wait();   // programmatic dependent launch: the previous kernel's results are visible
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  WarpSmem& S = reinterpret_cast<WarpSmem*>(smem_raw)[wid];
  const long long tile = t0 + (long long)blockIdx.x * kWarpsPerBlock + wid;
  if (tile >= t1) return;   // warp-uniform
  tile_bits_body<R, FUSED, kWarpMaxRuns>(P, words, WW, S, tile, lane);
}

// the tiles the first pass deferred (more than kWarpMaxRuns runs), a warp each
// with room for every run a tile can have (so none is deferred again)
template <int R, bool FUSED>
__global__ void __launch_bounds__(kBigWarpsPerBlock * 32)
    tile_bits_deferred_kernel(TileParams P, const uint4* __restrict__ words, int WW) {
  pdl_wait();   // programmatic dependent launch: the previous kernel's results are visible
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  WarpSmemT<kTileMaxRuns>& S = reinterpret_cast<WarpSmemT<kTileMaxRuns>*>(smem_raw)[wid];
  const long long n = (long long)*P.n_deferred;
  for (long long i = (long long)blockIdx.x * kBigWarpsPerBlock + wid; i < n;
       i += (long long)gridDim.x * kBigWarpsPerBlock) {
    tile_bits_body<R, FUSED, kTileMaxRuns>(P, words, WW, S, (long long)P.deferred[i], lane);
    __syncwarp();
  }
}

size_t tile_words_bytes(int V, int H, int W) { return (size_t)V * H * ((W + 31) / 32) * sizeof(uint4); }

template <int R, bool FUSED>
static cudaError_t launch_bits_r(const TileParams& P, int WW, long long t0, long long t1, cudaStream_t s) {
  const size_t smem = tile_warp_smem_bytes();
  cudaError_t e = cudaFuncSetAttribute(tile_bits_kernel<R, FUSED>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const long long blocks = (t1 - t0 + kWarpsPerBlock - 1) / kWarpsPerBlock;
  if (blocks > 0) launch_k(tile_bits_kernel<R, FUSED>, (unsigned)blocks, kWarpsPerBlock * 32, smem, s, P, P.words, WW, t0, t1);
  return cudaGetLastError();
}

// fused: the bit planes per tile straight from the raw cache (default); else the
// separate words pass (tile_words_kernel) first -- both give identical bits
cudaError_t launch_tile_bits(const TileParams& P, int v0, int v1, cudaStream_t s) {
  if (v1 <= v0) return cudaSuccess;
  const int WW = (P.W + 31) / 32;
  const bool fused = P.words == nullptr;
  if (!fused) {
#if ADPS_TW_ROWWISE
    const unsigned gx = (unsigned)((P.H + 7) / 8);   // warp per image row, 8 rows per block
    launch_k(tile_words_kernel, dim3(gx, (unsigned)(v1 - v0)), 256, 0, s, P.rawf, P.image, P.gt, P.cand_bits, P.thr_raw,
                                                                     P.L, P.H, P.W, WW, v0, P.words);
#else
    const dim3 g((unsigned)((WW + kTwWarps - 1) / kTwWarps), (unsigned)((P.H + 31) / 32), (unsigned)(v1 - v0));
    launch_k(tile_words_t_kernel, g, kTwWarps * 32, 0, s, P.rawf, P.image, P.gt, P.cand_bits, P.thr_raw, P.L, P.H, P.W, WW,
                                                    v0, P.words);
#endif
  }
  const long long tpv = (long long)P.tiles_x * P.tiles_y;
  const long long t0 = tpv * v0, t1 = tpv * v1;
  switch (P.r_erode <= 1 ? 1 : P.r_erode) {
    case 1: return fused ? launch_bits_r<1, true>(P, WW, t0, t1, s) : launch_bits_r<1, false>(P, WW, t0, t1, s);
    case 2: return fused ? launch_bits_r<2, true>(P, WW, t0, t1, s) : launch_bits_r<2, false>(P, WW, t0, t1, s);
    case 3: return fused ? launch_bits_r<3, true>(P, WW, t0, t1, s) : launch_bits_r<3, false>(P, WW, t0, t1, s);
    default: return cudaErrorInvalidValue;
  }
}

template <int R, bool FUSED>
static cudaError_t launch_deferred_r(const TileParams& P, int WW, unsigned blocks, cudaStream_t s) {
  const size_t smem = sizeof(WarpSmemT<kTileMaxRuns>) * kBigWarpsPerBlock;
  cudaError_t e = cudaFuncSetAttribute(tile_bits_deferred_kernel<R, FUSED>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  launch_k(tile_bits_deferred_kernel<R, FUSED>, blocks, kBigWarpsPerBlock * 32, smem, s, P, P.words, WW);
  return cudaGetLastError();
}

cudaError_t launch_tile_bits_deferred(const TileParams& P, unsigned blocks, cudaStream_t s) {
  const int WW = (P.W + 31) / 32;
  const bool fused = P.words == nullptr;
  switch (P.r_erode <= 1 ? 1 : P.r_erode) {
    case 1: return fused ? launch_deferred_r<1, true>(P, WW, blocks, s) : launch_deferred_r<1, false>(P, WW, blocks, s);
    case 2: return fused ? launch_deferred_r<2, true>(P, WW, blocks, s) : launch_deferred_r<2, false>(P, WW, blocks, s);
    case 3: return fused ? launch_deferred_r<3, true>(P, WW, blocks, s) : launch_deferred_r<3, false>(P, WW, blocks, s);
    default: return cudaErrorInvalidValue;
  }
}

template <int R, bool RAW>
static cudaError_t launch_r(const TileParams& P, long long t0, long long t1, cudaStream_t s) {
  const size_t smem = tile_warp_smem_bytes();
  cudaError_t e = cudaFuncSetAttribute(tile_warp_kernel<R, RAW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const long long blocks = (t1 - t0 + kWarpsPerBlock - 1) / kWarpsPerBlock;
  if (blocks <= 0) return cudaSuccess;
  launch_k(tile_warp_kernel<R, RAW>, (unsigned)blocks, kWarpsPerBlock * 32, smem, s, P, t0, t1);
  return cudaGetLastError();
}

cudaError_t launch_tile_warp(const TileParams& P, long long t0, long long t1, cudaStream_t s) {
  if (P.raw) {
    if (P.r_erode <= 1) return launch_r<1, true>(P, t0, t1, s);
    if (P.r_erode == 2) return launch_r<2, true>(P, t0, t1, s);
    if (P.r_erode == 3) return launch_r<3, true>(P, t0, t1, s);
  } else {
    if (P.r_erode <= 1) return launch_r<1, false>(P, t0, t1, s);
    if (P.r_erode == 2) return launch_r<2, false>(P, t0, t1, s);
    if (P.r_erode == 3) return launch_r<3, false>(P, t0, t1, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace adps
