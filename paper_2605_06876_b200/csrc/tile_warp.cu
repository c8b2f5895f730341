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

constexpr int kWarpMaxRuns = 256;
constexpr int kWarpsPerBlock = 8;

struct WarpSmem {
  int uf[kWarpMaxRuns];
  unsigned run[kWarpMaxRuns];   // ty | s << 5 | e << 10 | band << 16
  int aux[kWarpMaxRuns];        // fragment id of a root, -1 otherwise
  int mom[32][6];
  unsigned char touch[32];
};

size_t tile_warp_smem_bytes() { return sizeof(WarpSmem) * kWarpsPerBlock; }

// one image row of the tile (lane = x) plus the halo pixel of lanes < span
struct RowIn {
  float a[3], g[3];
  float ha[3], hg[3];
  int d;
  bool inb, hin;
};

template <int HL, int SPAN>
__device__ __forceinline__ void load_row(RowIn& r, const float* __restrict__ img, const float* __restrict__ gtv,
                                         const int* __restrict__ dom, int x0, int y0, int W, int H, int ey,
                                         int lane) {
  const int y = y0 - HL + ey;
  const bool row_in = y >= 0 && y < H;
  const int x = x0 + lane;
  r.inb = row_in && x < W;
  const int p = r.inb ? y * W + x : 0;
  const bool tile_row = ey >= HL && ey < HL + kTileH;
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    r.a[c] = r.inb ? __ldg(img + 3 * p + c) : 0.0f;
    r.g[c] = r.inb ? __ldg(gtv + 3 * p + c) : 0.0f;
  }
  r.d = r.inb && tile_row ? __ldg(dom + p) : -1;
  if (SPAN > 0) {
    const int xh = lane < HL ? x0 - HL + lane : x0 + kTileW + (lane - HL);
    r.hin = row_in && lane < SPAN && xh >= 0 && xh < W;
    const int ph = r.hin ? y * W + xh : 0;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      r.ha[c] = r.hin ? __ldg(img + 3 * ph + c) : 0.0f;
      r.hg[c] = r.hin ? __ldg(gtv + 3 * ph + c) : 0.0f;
    }
  } else {
    r.hin = false;
  }
}

// np.abs(rendered - gt).sum(axis=-1) == (|d0| + |d1|) + |d2| in fp64
__device__ __forceinline__ double raw_l1_f(const float* a, const float* g) {
  const double a0 = fabs(dsub((double)a[0], (double)g[0]));
  const double a1 = fabs(dsub((double)a[1], (double)g[1]));
  const double a2 = fabs(dsub((double)a[2], (double)g[2]));
  return dadd(dadd(a0, a1), a2);
}

template <int R>
__device__ __forceinline__ void tile_warp_body(const TileParams& P, WarpSmem& S, const long long tile,
                                               const int lane) {
  constexpr int HL = R > 1 ? R / 2 : 0;
  constexpr int HH = R > 1 ? R - R / 2 - 1 : 0;
  constexpr int SPAN = HL + HH;
  constexpr unsigned FULL = 0xffffffffu;
  const int tiles_per_view = P.tiles_x * P.tiles_y;
  const int v = (int)(tile / tiles_per_view);
  const int tin = (int)(tile % tiles_per_view);
  const int x0 = (tin % P.tiles_x) * kTileW, y0 = (tin / P.tiles_x) * kTileH;
  const int W = P.W, H = P.H;
  const long long hw = (long long)W * H;
  const float* img = P.image + (long long)v * hw * 3;
  const float* gtv = P.gt + (long long)v * hw * 3;
  const int* dom = P.dom + (long long)v * hw;
  const double lo = P.lo[v];
  const double* thr = P.thr + (long long)v * P.L;
  const double x_m = thr[0];
  const int L = P.L;
  const double kInf = __longlong_as_double(0x7ff0000000000000ll);
  const double t1 = L > 1 ? thr[1] : kInf, t2 = L > 2 ? thr[2] : kInf, t3 = L > 3 ? thr[3] : kInf;

  int b_top = -1, b_bot = -1, b_left = -1, b_right = -1;   // run id of border pixel `lane`
  int prev_key = -1, prev_band = 0, prev_rid = -1;
  int c_del = -1, band_del = 0;
  unsigned long long m1 = 0, m2 = 0;   // metric masks of ext rows ey-1, ey-2
  int n_runs = 0;
  bool overflow = false;
  RowIn nx;
  load_row<HL, SPAN>(nx, img, gtv, dom, x0, y0, W, H, 0, lane);
  for (int ey = 0; ey < kTileH + SPAN; ++ey) {
    const RowIn cur = nx;
    if (ey + 1 < kTileH + SPAN) load_row<HL, SPAN>(nx, img, gtv, dom, x0, y0, W, H, ey + 1, lane);
    // ---- metric bits of ext row ey; band + candidate of its tile row
    bool m = false;
    int band_now = 0;
    if (cur.inb) {
      const double xr = dsub(raw_l1_f(cur.a, cur.g), lo);
      m = xr >= x_m;
      if (L <= 4) {
        band_now = (xr >= t1) + (xr >= t2) + (xr >= t3);
      } else {
        for (int q = 1; q < L; ++q) band_now += xr >= thr[q];
      }
    }
    bool mh = false;
    if (SPAN > 0 && cur.hin) mh = dsub(raw_l1_f(cur.ha, cur.hg), lo) >= x_m;
    const unsigned mbits = __ballot_sync(FULL, m);
    unsigned long long m0 = (unsigned long long)mbits << HL;
    if (SPAN > 0) {
      const unsigned hbits = __ballot_sync(FULL, mh);
      if (HL > 0 && (hbits & 1u)) m0 |= 1ull;
      if (HH > 0 && ((hbits >> HL) & 1u)) m0 |= 1ull << (kTileW + HL);
    }
    int c_now = -1;
    if (ey >= HL && ey < HL + kTileH) {   // warp-uniform
      // split-candidate test once per run of equal dominant id
      const int d = cur.d;
      const int left = __shfl_up_sync(FULL, d, 1);
      const bool head = lane == 0 || left != d;
      bool isc = false;
      if (head && d >= 0 && d < P.N) isc = __ldg(P.cls + d) == 1;
      const unsigned heads = __ballot_sync(FULL, head);
      isc = __shfl_sync(FULL, isc, 31 - __clz(heads & (FULL >> (31 - lane))));
      c_now = isc ? d : -1;
    }
    // ---- tile row ty = ey - SPAN now has its whole erosion window
    const int ty = ey - SPAN;
    if (ty >= 0) {
      unsigned long long acc = m0;
      if (SPAN >= 1) acc &= m1;
      if (SPAN >= 2) acc &= m2;
      unsigned long long h = acc;
      if (SPAN >= 1) h &= acc >> 1;
      if (SPAN >= 2) h &= acc >> 2;
      const unsigned er = (unsigned)h;
      const int cand = HH > 0 ? c_del : c_now;
      const int band = HH > 0 ? band_del : band_now;
      const int key = ((er >> lane) & 1u) ? cand : -1;
      // ---- runs of equal (candidate, band)
      const unsigned K = __ballot_sync(FULL, key >= 0);
      const int lkey = __shfl_up_sync(FULL, key, 1);
      const int lband = __shfl_up_sync(FULL, band, 1);
      const unsigned C = __ballot_sync(FULL, key >= 0 && lane > 0 && lkey == key && lband == band);
      const unsigned starts = K & ~C;
      const unsigned ends = K & ~(C >> 1);
      const int nr = __popc(starts);
      if (n_runs + nr > kWarpMaxRuns) {
        overflow = true;
        break;
      }
      const bool is_start = (starts >> lane) & 1u;
      const bool is_end = (ends >> lane) & 1u;
      const int rid_start = n_runs + __popc(starts & ((1u << lane) - 1u));
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
      const int pk_m = __shfl_up_sync(FULL, prev_key, 1), pb_m = __shfl_up_sync(FULL, prev_band, 1);
      const int pr_m = __shfl_up_sync(FULL, prev_rid, 1);
      const int pk_p = __shfl_down_sync(FULL, prev_key, 1), pb_p = __shfl_down_sync(FULL, prev_band, 1);
      const int pr_p = __shfl_down_sync(FULL, prev_rid, 1);
      if (key >= 0 && ty > 0) {
        const bool a0 = prev_key == key && prev_band == band;
        const bool am = lane > 0 && pk_m == key && pb_m == band;
        const bool ap = lane < 31 && pk_p == key && pb_p == band;
        if (a0 && (is_start || !am)) uf_unite(S.uf, rid, prev_rid);
        if (is_start && am && !a0) uf_unite(S.uf, rid, pr_m);
        if (is_end && ap && !a0) uf_unite(S.uf, rid, pr_p);
      }
      if (ty == 0) b_top = rid;
      if (ty == kTileH - 1) b_bot = rid;
      const int lc = __shfl_sync(FULL, rid, 0), rc = __shfl_sync(FULL, rid, 31);
      if (lane == ty) {
        b_left = lc;
        b_right = rc;
      }
      prev_key = key;
      prev_band = band;
      prev_rid = rid;
      n_runs += nr;
    }
    m2 = m1;
    m1 = m0;
    c_del = c_now;
    band_del = band_now;
  }
  if (overflow) {
    if (lane == 0) P.deferred[atomicAdd(P.n_deferred, 1ull)] = (int)tile;
    return;
  }
  __syncwarp();
  // ---- roots (read-only finds: stored roots are never overwritten)
  for (int q = lane; q < n_runs; q += 32) {
    S.uf[q] = uf_find(S.uf, q);
    S.aux[q] = -1;
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
    for (int k = 0; k < 6; ++k) S.mom[lane][k] = 0;
    S.touch[lane] = 0;
    __syncwarp();
    for (int q2 = lane; q2 < n_runs; q2 += 32) {
      const int root = S.uf[q2];
      if (root < base || root >= base + 32) continue;
      const int sl = __popc(roots & ((1u << (root - base)) - 1u));
      const unsigned info = S.run[q2];
      const int ty = info & 31, s = (info >> 5) & 31, e = (info >> 10) & 31;
      const int n = e - s + 1;
      const int sx = (s + e) * n / 2;
      const int sxx = (e * (e + 1) * (2 * e + 1) - (s - 1) * s * (2 * s - 1)) / 6;
      atomicAdd(&S.mom[sl][0], n);
      atomicAdd(&S.mom[sl][1], sx);
      atomicAdd(&S.mom[sl][2], ty * n);
      atomicAdd(&S.mom[sl][3], sxx);
      atomicAdd(&S.mom[sl][4], ty * sx);
      atomicAdd(&S.mom[sl][5], ty * ty * n);
      if ((ty == 0 && top_in) || (ty == kTileH - 1 && bottom_in) || (s == 0 && left_in) ||
          (e == kTileW - 1 && right_in))
        S.touch[sl] = 1;
    }
    __syncwarp();
    // records: fragments for edge components, regions for interior ones >= m_min
    const int sl = __popc(roots & ((1u << lane) - 1u));
    const bool is_part = is_root && S.touch[sl];
    const bool is_reg = is_root && !S.touch[sl] && S.mom[sl][0] >= P.m_min;
    const unsigned pm = __ballot_sync(FULL, is_part), rm = __ballot_sync(FULL, is_reg);
    unsigned long long pbase = 0, rbase = 0;
    if (lane == 0) {
      if (pm) pbase = atomicAdd(P.n_partials, (unsigned long long)__popc(pm));
      if (rm) rbase = atomicAdd(P.n_regions, (unsigned long long)__popc(rm));
    }
    pbase = __shfl_sync(FULL, pbase, 0);
    rbase = __shfl_sync(FULL, rbase, 0);
    if (is_part || is_reg) {
      const unsigned info = S.run[q];
      const int ty = info & 31, s = (info >> 5) & 31, bnd = (info >> 16) & 0xff;
      const long long n = S.mom[sl][0], mx = S.mom[sl][1], my = S.mom[sl][2];
      const long long X = x0, Y = y0;
      long long gm[6];
      gm[0] = n;
      gm[1] = mx + n * X;
      gm[2] = my + n * Y;
      gm[3] = (long long)S.mom[sl][3] + 2 * X * mx + n * X * X;
      gm[4] = (long long)S.mom[sl][4] + X * my + Y * mx + n * X * Y;
      gm[5] = (long long)S.mom[sl][5] + 2 * Y * my + n * Y * Y;
      const int minpix = (y0 + ty) * W + (x0 + s);
      const int cand = __ldg(dom + minpix);
      if (is_part) {
        const unsigned long long gid = pbase + __popc(pm & ((1u << lane) - 1u));
        if ((long long)gid < P.partial_cap) {
          PartialRec& Rr = P.partials[gid];
          Rr.view_pos = P.view_offset + v;
          Rr.cand = cand;
          Rr.band = bnd;
          Rr.minpix = minpix;
#pragma unroll
          for (int k = 0; k < 6; ++k) Rr.m[k] = gm[k];
          P.partial_parent[gid] = (int)gid;
          S.aux[q] = (int)gid;
        } else {
          atomicOr(P.overflow, 2u);
        }
      } else {
        const unsigned long long rid2 = rbase + __popc(rm & ((1u << lane) - 1u));
        if ((long long)rid2 < P.region_cap) {
          RegionRec& Rr = P.regions[rid2];
          Rr.view_pos = P.view_offset + v;
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
  border[lane] = b_top >= 0 ? S.aux[S.uf[b_top]] : -1;
  border[kTileW + lane] = b_bot >= 0 ? S.aux[S.uf[b_bot]] : -1;
  border[2 * kTileW + lane] = b_left >= 0 ? S.aux[S.uf[b_left]] : -1;
  border[2 * kTileW + kTileH + lane] = b_right >= 0 ? S.aux[S.uf[b_right]] : -1;
}

template <int R>
__global__ void __launch_bounds__(kWarpsPerBlock * 32, 4) tile_warp_kernel(TileParams P, long long n_tiles) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  WarpSmem& S = reinterpret_cast<WarpSmem*>(smem_raw)[wid];
  const long long tile = (long long)blockIdx.x * kWarpsPerBlock + wid;
  if (tile >= n_tiles) return;   // warp-uniform
  tile_warp_body<R>(P, S, tile, lane);
}

template <int R>
static cudaError_t launch_r(const TileParams& P, long long n_tiles, cudaStream_t s) {
  const size_t smem = tile_warp_smem_bytes();
  cudaError_t e = cudaFuncSetAttribute(tile_warp_kernel<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const long long blocks = (n_tiles + kWarpsPerBlock - 1) / kWarpsPerBlock;
  tile_warp_kernel<R><<<(unsigned)blocks, kWarpsPerBlock * 32, smem, s>>>(P, n_tiles);
  return cudaGetLastError();
}

cudaError_t launch_tile_warp(const TileParams& P, long long n_tiles, cudaStream_t s) {
  if (P.r_erode <= 1) return launch_r<1>(P, n_tiles, s);
  if (P.r_erode == 2) return launch_r<2>(P, n_tiles, s);
  if (P.r_erode == 3) return launch_r<3>(P, n_tiles, s);
  return cudaErrorInvalidValue;
}

}  // namespace adps
