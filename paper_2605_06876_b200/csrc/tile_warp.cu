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

// rows reach the warp either by per-lane loads a row ahead (default) or staged
// kRing rows ahead in shared memory by bulk async copies (kStaged)
#ifndef ADPS_TW_STAGED
#define ADPS_TW_STAGED 0
#endif
#ifndef ADPS_TW_FAST
#define ADPS_TW_FAST 1
#endif
#ifndef ADPS_TW_MINBLOCKS
#define ADPS_TW_MINBLOCKS 4
#endif
constexpr bool kStaged = ADPS_TW_STAGED != 0;
constexpr int kRing = 4;            // rows in flight per warp (bulk async copies)
constexpr int kRingF = 112;         // floats per staged image row: 32 px * 3 + 16 B alignment slack, x16 B
constexpr int kRingD = 40;          // ints per staged dominant row: 32 + slack

struct RingSlot {
  float img[kRingF];
  float gt[kRingF];
  int dom[kRingD];
};

struct PostSmem {                   // used after the row scan; aliases the ring
  int aux[kWarpMaxRuns];            // fragment id of a root, -1 otherwise
  int mom[32][6];
  unsigned char touch[32];
};

struct WarpSmem {
  int uf[kWarpMaxRuns];
  unsigned run[kWarpMaxRuns];       // ty | s << 5 | e << 10 | band << 16
  union {
#if ADPS_TW_STAGED
    RingSlot ring[kRing];
#endif
    PostSmem post;
  } u;
  unsigned long long bar[kRing];    // one mbarrier per ring slot
  unsigned meta[kRing];             // per staged row: bit0/1/2 img/gt/dom staged, bit3 row inside
                                    // the image, bits 8-9/10-11/12-13 element offset of x0
};
static_assert(sizeof(RingSlot) % 16 == 0 && sizeof(WarpSmem) % 16 == 0, "bulk copy alignment");

size_t tile_warp_smem_bytes() { return sizeof(WarpSmem) * kWarpsPerBlock; }

// per-tile scan state carried from row to row (registers)
struct ScanState {
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
  const unsigned char* cls;
  const double* thr;
  double lo, x_m, t1, t2, t3;
  int x0, y0, W, H, L, N;
  unsigned long long hl_mask, hr_mask;   // bit ey: metric bit of the left/right halo pixel of ext row ey
};

// ---------------------------------------------------------------- row ring
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void bar_init(unsigned long long* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void bar_arrive_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred P;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t"
      "@!P bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// 16-byte aligned cover [lo, hi) of [p, p + bytes); usable when it stays inside [base, end)
struct Cover {
  const char* lo;
  unsigned bytes;
  bool ok;
};
__device__ __forceinline__ Cover cover(const void* p, unsigned bytes, const void* base, const void* end) {
  const unsigned long long a = (unsigned long long)p;
  const unsigned long long lo = a & ~15ull, hi = (a + bytes + 15) & ~15ull;
  Cover c;
  c.lo = (const char*)lo;
  c.bytes = (unsigned)(hi - lo);
  c.ok = lo >= (unsigned long long)base && hi <= (unsigned long long)end;
  return c;
}

// one image row of the tile (lane = x)
struct RowIn {
  float a[3], g[3];
  int d;
  bool inb;
};

template <int HL>
__device__ __forceinline__ void load_row(RowIn& r, const TileConst& T, int ey, int lane) {
  const int y = T.y0 - HL + ey;
  const int x = T.x0 + lane;
  r.inb = y >= 0 && y < T.H && x < T.W;
  const long long p = r.inb ? (long long)y * T.W + x : 0;
  const bool tile_row = ey >= HL && ey < HL + kTileH;
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    r.a[c] = r.inb ? __ldg(T.img + 3 * p + c) : 0.0f;
    r.g[c] = r.inb ? __ldg(T.gtv + 3 * p + c) : 0.0f;
  }
  r.d = r.inb && tile_row ? __ldg(T.dom + p) : -1;
}

__device__ __forceinline__ int cand_of_px(const TileConst& T, const int d) {
  return d >= 0 && d < T.N && __ldg(T.cls + d) == 1 ? d : -1;
}

// np.abs(rendered - gt).sum(axis=-1) == (|d0| + |d1|) + |d2| in fp64
__device__ __forceinline__ double raw_l1_f(const float* a, const float* g) {
  const double a0 = fabs(dsub((double)a[0], (double)g[0]));
  const double a1 = fabs(dsub((double)a[1], (double)g[1]));
  const double a2 = fabs(dsub((double)a[2], (double)g[2]));
  return dadd(dadd(a0, a1), a2);
}

__device__ __forceinline__ bool metric_at(const TileConst& T, int x, int y) {
  const long long p = (long long)y * T.W + x;
  float a[3], g[3];
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    a[c] = __ldg(T.img + 3 * p + c);
    g[c] = __ldg(T.gtv + 3 * p + c);
  }
  return dsub(raw_l1_f(a, g), T.lo) >= T.x_m;
}

#if ADPS_TW_STAGED
// lane 0: stage ext row ey (image, gt and -- for tile rows -- dominant ids)
// into its ring slot with bulk async copies completing on the slot's mbarrier
template <int HL>
__device__ __forceinline__ void issue_row(WarpSmem& S, const int ey, const TileConst& T, const TileParams& P,
                                          const long long hw) {
  const int slot = ey % kRing;
  unsigned long long* bar = &S.bar[slot];
  const int y = T.y0 - HL + ey;
  unsigned meta = 0, tx = 0;
  Cover ci, cg, cd;
  ci.ok = cg.ok = cd.ok = false;
  if (y >= 0 && y < T.H) {
    meta |= 8u;
    const int n = min(kTileW, T.W - T.x0);
    const long long p = (long long)y * T.W + T.x0;
    const long long total = hw * P.n_views;
    ci = cover(T.img + 3 * p, 12u * n, P.image, P.image + 3 * total);
    cg = cover(T.gtv + 3 * p, 12u * n, P.gt, P.gt + 3 * total);
    meta |= (ci.ok ? 1u : 0u) | (cg.ok ? 2u : 0u);
    meta |= (unsigned)(((unsigned long long)(T.img + 3 * p) & 15) >> 2) << 8;
    meta |= (unsigned)(((unsigned long long)(T.gtv + 3 * p) & 15) >> 2) << 10;
    if (ey >= HL && ey < HL + kTileH) {
      cd = cover(T.dom + p, 4u * n, P.dom, P.dom + total);
      meta |= (cd.ok ? 4u : 0u) | ((unsigned)(((unsigned long long)(T.dom + p) & 15) >> 2) << 12);
    }
    tx = (ci.ok ? ci.bytes : 0u) + (cg.ok ? cg.bytes : 0u) + (cd.ok ? cd.bytes : 0u);
  }
  S.meta[slot] = meta;
  bar_arrive_tx(bar, tx);   // released by the copies (or at once when nothing is staged)
  if (ci.ok) bulk_g2s(S.u.ring[slot].img, ci.lo, ci.bytes, bar);
  if (cg.ok) bulk_g2s(S.u.ring[slot].gt, cg.lo, cg.bytes, bar);
  if (cd.ok) bulk_g2s(S.u.ring[slot].dom, cd.lo, cd.bytes, bar);
}

#endif

// one ext row: metric mask, then (once its erosion window is complete) the
// runs of tile row ey - SPAN and their unions with the row above.
// Returns true when the tile has too many runs for the warp path.
template <int R>
__device__ __forceinline__ bool scan_row(const float* a, const float* g, const bool inb, const int c_now, const int ey,
                                         ScanState& st, WarpSmem& S, const TileConst& T, const int lane) {
  constexpr int HL = R > 1 ? R / 2 : 0;
  constexpr int HH = R > 1 ? R - R / 2 - 1 : 0;
  constexpr int SPAN = HL + HH;
  constexpr unsigned FULL = 0xffffffffu;
  bool m = false;
  int band_now = 0;
  if (inb) {
    const double xr = dsub(raw_l1_f(a, g), T.lo);
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
#if ADPS_TW_FAST
    if (K == 0) {   // no keyed pixel in this row: no runs, nothing to unite
      st.prev_key = -1;
      st.prev_rid = -1;
    } else
#endif
    {
      const int lkey = __shfl_up_sync(FULL, key, 1);
      const int lband = __shfl_up_sync(FULL, band, 1);
      const unsigned C = __ballot_sync(FULL, key >= 0 && lane > 0 && lkey == key && lband == band);
      const unsigned starts = K & ~C;
      const unsigned ends = K & ~(C >> 1);
      const int nr = __popc(starts);
      if (st.n_runs + nr > kWarpMaxRuns) {
        overflow = true;
      } else {
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
      }
    }
  }
  st.m2 = st.m1;
  st.m1 = m0;
  st.c_del = c_now;
  st.band_del = band_now;
  return overflow;
}

template <int R>
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
  T.x0 = (tin % P.tiles_x) * kTileW;
  T.y0 = (tin / P.tiles_x) * kTileH;
  T.W = P.W;
  T.H = P.H;
  const long long hw = (long long)T.W * T.H;
  T.img = P.image + (long long)v * hw * 3;
  T.gtv = P.gt + (long long)v * hw * 3;
  T.dom = P.dom + (long long)v * hw;
  T.cls = P.cls;
  T.N = P.N;
  T.L = P.L;
  T.lo = P.lo[v];
  T.thr = P.thr + (long long)v * P.L;
  T.x_m = T.thr[0];
  const double kInf = __longlong_as_double(0x7ff0000000000000ll);
  T.t1 = T.L > 1 ? T.thr[1] : kInf;
  T.t2 = T.L > 2 ? T.thr[2] : kInf;
  T.t3 = T.L > 3 ? T.thr[3] : kInf;
  const int x0 = T.x0, y0 = T.y0, W = T.W, H = T.H;
  // halo columns of all ext rows at once (lane = ext row, then ext rows 32..)
  T.hl_mask = 0;
  T.hr_mask = 0;
  if (SPAN > 0) {
#pragma unroll
    for (int k = 0; k < (NR + 31) / 32; ++k) {
      const int ey = lane + 32 * k;
      const int y = y0 - HL + ey;
      const bool row_ok = ey < NR && y >= 0 && y < H;
      const bool ml = HL > 0 && row_ok && x0 - 1 >= 0 && metric_at(T, x0 - 1, y);
      const bool mr = HH > 0 && row_ok && x0 + kTileW < W && metric_at(T, x0 + kTileW, y);
      T.hl_mask |= (unsigned long long)__ballot_sync(FULL, ml) << (32 * k);
      T.hr_mask |= (unsigned long long)__ballot_sync(FULL, mr) << (32 * k);
    }
  }

  ScanState st;
  st.m1 = st.m2 = 0;
  st.c_del = -1;
  st.band_del = 0;
  st.prev_key = -1;
  st.prev_band = 0;
  st.prev_rid = -1;
  st.b_top = st.b_bot = st.b_left = st.b_right = -1;
  st.n_runs = 0;
  bool overflow = false;
  if constexpr (!kStaged) {
    // rows are loaded one ahead into two alternating register buffers
    RowIn A, B;
    load_row<HL>(A, T, 0, lane);
    for (int ey = 0; ey < NR; ey += 2) {
      if (ey + 1 < NR) load_row<HL>(B, T, ey + 1, lane);
      if (scan_row<R>(A.a, A.g, A.inb, cand_of_px(T, A.d), ey, st, S, T, lane)) {
        overflow = true;
        break;
      }
      if (ey + 1 < NR) {
        if (ey + 2 < NR) load_row<HL>(A, T, ey + 2, lane);
        if (scan_row<R>(B.a, B.g, B.inb, cand_of_px(T, B.d), ey + 1, st, S, T, lane)) {
          overflow = true;
          break;
        }
      }
    }
  }
#if ADPS_TW_STAGED
  else {
    // rows are staged kRing ahead by bulk async copies; the candidate test of
    // row ey + 1 (a dependent load) is issued while row ey is scanned
    if (lane == 0) {
  #pragma unroll
      for (int k = 0; k < kRing; ++k) bar_init(&S.bar[k]);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      for (int r = 0; r < kRing && r < NR; ++r) issue_row<HL>(S, r, T, P, hw);
    }
    __syncwarp();
    const bool col_in = x0 + lane < W;
    auto dom_of = [&](const int r) -> int {   // dominant id of ext row r (staged and waited for)
      const int slot = r % kRing;
      const unsigned meta = S.meta[slot];
      if (!(r >= HL && r < HL + kTileH) || !(meta & 8u) || !col_in) return -1;
      if (meta & 4u) return S.u.ring[slot].dom[((meta >> 12) & 3u) + lane];
      return __ldg(T.dom + (long long)(y0 - HL + r) * W + x0 + lane);
    };
    auto cand_of = [&](const int d) -> int {
      return d >= 0 && d < T.N && __ldg(T.cls + d) == 1 ? d : -1;
    };
    bar_wait(&S.bar[0], 0);
    int c_next = cand_of(dom_of(0));
    int ey = 0;
    for (; ey < NR; ++ey) {
      const int slot = ey % kRing;
      const unsigned meta = S.meta[slot];
      const bool inb = (meta & 8u) && col_in;
      float a[3], g[3];
      if (inb) {
        const long long p = (long long)(y0 - HL + ey) * W + x0 + lane;
        if (meta & 1u) {
          const float* r = S.u.ring[slot].img + ((meta >> 8) & 3u) + 3 * lane;
          a[0] = r[0]; a[1] = r[1]; a[2] = r[2];
        } else {
          a[0] = __ldg(T.img + 3 * p); a[1] = __ldg(T.img + 3 * p + 1); a[2] = __ldg(T.img + 3 * p + 2);
        }
        if (meta & 2u) {
          const float* r = S.u.ring[slot].gt + ((meta >> 10) & 3u) + 3 * lane;
          g[0] = r[0]; g[1] = r[1]; g[2] = r[2];
        } else {
          g[0] = __ldg(T.gtv + 3 * p); g[1] = __ldg(T.gtv + 3 * p + 1); g[2] = __ldg(T.gtv + 3 * p + 2);
        }
      } else {
        a[0] = a[1] = a[2] = g[0] = g[1] = g[2] = 0.0f;
      }
      const int c_now = c_next;
      int d_next = -1;
      if (ey + 1 < NR) {
        bar_wait(&S.bar[(ey + 1) % kRing], ((ey + 1) / kRing) & 1);
        d_next = dom_of(ey + 1);
        c_next = cand_of(d_next);
      }
      if (scan_row<R>(a, g, inb, c_now, ey, st, S, T, lane)) {
        overflow = true;
        break;
      }
      __syncwarp();
      if (lane == 0 && ey + kRing < NR) issue_row<HL>(S, ey + kRing, T, P, hw);
    }
    if (overflow) {   // no bulk copy may still target this warp's ring when it leaves
      for (int r = ey + 2; r < NR && r < ey + kRing; ++r) bar_wait(&S.bar[r % kRing], (r / kRing) & 1);
    }
  }
#endif
  const int n_runs = st.n_runs;
  const int b_top = st.b_top, b_bot = st.b_bot, b_left = st.b_left, b_right = st.b_right;
  if (overflow) {
    if (lane == 0) P.deferred[atomicAdd(P.n_deferred, 1ull)] = (int)tile;
    return;
  }
  __syncwarp();
  // ---- roots (read-only finds: stored roots are never overwritten)
  for (int q = lane; q < n_runs; q += 32) {
    S.uf[q] = uf_find(S.uf, q);
    S.u.post.aux[q] = -1;
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
    for (int q2 = lane; q2 < n_runs; q2 += 32) {
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
    if (lane == 0) {
      if (pm) pbase = atomicAdd(P.n_partials, (unsigned long long)__popc(pm));
      if (rm) rbase = atomicAdd(P.n_regions, (unsigned long long)__popc(rm));
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
      const int cand = __ldg(T.dom + minpix);
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
          S.u.post.aux[q] = (int)gid;
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
  border[lane] = b_top >= 0 ? S.u.post.aux[S.uf[b_top]] : -1;
  border[kTileW + lane] = b_bot >= 0 ? S.u.post.aux[S.uf[b_bot]] : -1;
  border[2 * kTileW + lane] = b_left >= 0 ? S.u.post.aux[S.uf[b_left]] : -1;
  border[2 * kTileW + kTileH + lane] = b_right >= 0 ? S.u.post.aux[S.uf[b_right]] : -1;
}

template <int R>
__global__ void __launch_bounds__(kWarpsPerBlock * 32, ADPS_TW_MINBLOCKS) tile_warp_kernel(TileParams P, long long n_tiles) {
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
