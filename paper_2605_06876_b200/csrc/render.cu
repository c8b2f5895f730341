// Attribution render: image + dominant-Gaussian map per view.
//
// Replaces raster.render (ref/raster.py:136-157) with visible_splats,
// project and _support_radius (ref/raster.py:61-117):
//   * per-Gaussian projection in fp64 (cull rules of ref/raster.py:104-113)
//   * exact (camera z, index) order: a stable radix sort of monotone 32-bit
//     depth keys (the float below z), then runs of equal keys put in (z, index)
//     order, gives each splat its depth rank; tile lists are then a stable sort
//     on the tile id only, so every tile list is in reference order (the
//     64-bit sort of the fp64 depth bits remains as ADPS_PARAM_RENDER_BINNING 0)
//   * 16x16 tiles, shared-memory splat batches, fp32 per-pixel alpha with
//     tile-local offsets computed in fp64 (no large-coordinate cancellation)
//   * front-to-back composite and strict argmax of T*alpha (front-most wins)
//   * the reference has no early termination; a pixel stops only when its
//     argmax can no longer change (T*0.99 <= best) AND the remaining image
//     contribution is below 1e-8 (below fp32 resolution of the composite).
#include <math.h>


#include "render.cuh"

namespace adps {

__device__ __forceinline__ void sh_eval_rgb(const float* dc, const float* rest, int K, const double d[3],
                                            float out[3]) {
  const double x = d[0], y = d[1], z = d[2];
  double basis[16];
  basis[0] = kShC0;
  const int n = 1 + K;
  if (n > 1) {
    basis[1] = -kShC1 * y;
    basis[2] = kShC1 * z;
    basis[3] = -kShC1 * x;
  }
  if (n > 4) {
    const double xx = x * x, yy = y * y, zz = z * z;
    basis[4] = 1.0925484305920792 * x * y;
    basis[5] = -1.0925484305920792 * y * z;
    basis[6] = 0.3153915652525205 * (2 * zz - xx - yy);
    basis[7] = -1.0925484305920792 * x * z;
    basis[8] = 0.5462742152960396 * (xx - yy);
  }
  if (n > 9) {
    const double xx = x * x, yy = y * y, zz = z * z;
    basis[9] = -0.5900435899266435 * y * (3 * xx - yy);
    basis[10] = 2.890611442640554 * x * y * z;
    basis[11] = -0.4570457994644658 * y * (4 * zz - xx - yy);
    basis[12] = 0.3731763325901154 * z * (2 * zz - 3 * xx - 3 * yy);
    basis[13] = -0.4570457994644658 * x * (4 * zz - xx - yy);
    basis[14] = 1.445305721320277 * z * (xx - yy);
    basis[15] = -0.5900435899266435 * x * (3 * yy - xx);
  }
  for (int c = 0; c < 3; ++c) {
    double acc = basis[0] * (double)dc[c];
    for (int k = 1; k < n; ++k) acc += basis[k] * (double)rest[3 * (k - 1) + c];
    const double v = 0.5 + acc;
    out[c] = (float)fmin(fmax(v, 0.0), 1.0);
  }
}

// the view-independent part of the projection, once per render call: the 3D
// covariance R diag(s^2) R^T (fp64) and, at SH degree 0, the colour
__global__ void splat3d_kernel(PreArgs a, double* __restrict__ cov3, float* __restrict__ rgb0) {
  pdl_wait();   // programmatic dependent launch: the previous kernel's results are visible
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.n) return;
  double q[4] = {a.rot[4 * i], a.rot[4 * i + 1], a.rot[4 * i + 2], a.rot[4 * i + 3]};
  double R[9];
  quat_to_rot(q, R);
  const double s2[3] = {(double)a.scale[3 * i] * a.scale[3 * i], (double)a.scale[3 * i + 1] * a.scale[3 * i + 1],
                        (double)a.scale[3 * i + 2] * a.scale[3 * i + 2]};
  double S[6];
  rdrt(R, s2, S);
#pragma unroll
  for (int k = 0; k < 6; ++k) cov3[6 * i + k] = S[k];
  if (rgb0) {
    const double dir[3] = {0.0, 0.0, 1.0};   // unused at degree 0
    float c[3];
    sh_eval_rgb(a.sh_dc + 3 * i, nullptr, 0, dir, c);
    for (int k = 0; k < 3; ++k) rgb0[3 * i + k] = c[k];
  }
}

cudaError_t launch_splat3d(const PreArgs& a, double* cov3, float* rgb0, cudaStream_t s) {
  if (a.n > 0) launch_k(splat3d_kernel, (unsigned)((a.n + 255) / 256), 256, 0, s, a, cov3, rgb0);
  return cudaGetLastError();
}

__global__ void preprocess_kernel(PreArgs a) {
  pdl_wait();   // programmatic dependent launch: the previous kernel's results are visible
  const long long i0 = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const bool in_range = i0 < a.n;
  const long long i = in_range ? i0 : a.n - 1;   // out-of-range lanes recompute the last one, write nothing
  const CamD& cam = a.cam;
  const double mu[3] = {a.mu[3 * i], a.mu[3 * i + 1], a.mu[3 * i + 2]};
  const double dl[3] = {mu[0] - cam.c[0], mu[1] - cam.c[1], mu[2] - cam.c[2]};
  // p = R^T (mu - center)
  const double x = cam.r[0] * dl[0] + cam.r[3] * dl[1] + cam.r[6] * dl[2];
  const double y = cam.r[1] * dl[0] + cam.r[4] * dl[1] + cam.r[7] * dl[2];
  const double z = cam.r[2] * dl[0] + cam.r[5] * dl[1] + cam.r[8] * dl[2];
  unsigned long long key = ~0ull;
  unsigned tiles = 0;
  unsigned short rect[4] = {0, 0, 0, 0};
  short bx0 = 0, bx1 = -1, by0 = 0, by1 = -1;
  if (z > 1e-8) {
    const double mx = cam.fx * x / z + cam.px, my = cam.fy * y / z + cam.py;
    // cov2d = J W Sigma W^T J^T + 0.3 I
    double S[6];
    if (a.cov3) {   // view-independent, once per render call (splat3d_kernel)
#pragma unroll
      for (int k = 0; k < 6; ++k) S[k] = __ldg(a.cov3 + 6 * i + k);
    } else {
      double q[4] = {a.rot[4 * i], a.rot[4 * i + 1], a.rot[4 * i + 2], a.rot[4 * i + 3]};
      double R[9];
      quat_to_rot(q, R);
      const double s2[3] = {(double)a.scale[3 * i] * a.scale[3 * i], (double)a.scale[3 * i + 1] * a.scale[3 * i + 1],
                            (double)a.scale[3 * i + 2] * a.scale[3 * i + 2]};
      rdrt(R, s2, S);
    }
    const double Sm[9] = {S[0], S[1], S[2], S[1], S[3], S[4], S[2], S[4], S[5]};
    // T = J W (2x3), W = R_c2w^T
    const double j00 = cam.fx / z, j02 = -cam.fx * x / (z * z);
    const double j11 = cam.fy / z, j12 = -cam.fy * y / (z * z);
    double T[6];
    for (int c = 0; c < 3; ++c) {
      // W[r][c] = cam.r[c*3 + r]
      T[c] = j00 * cam.r[c * 3 + 0] + j02 * cam.r[c * 3 + 2];
      T[3 + c] = j11 * cam.r[c * 3 + 1] + j12 * cam.r[c * 3 + 2];
    }
    double TS[6];
    for (int r = 0; r < 2; ++r)
      for (int c = 0; c < 3; ++c)
        TS[r * 3 + c] = T[r * 3 + 0] * Sm[0 * 3 + c] + T[r * 3 + 1] * Sm[1 * 3 + c] + T[r * 3 + 2] * Sm[2 * 3 + c];
    const double ca = TS[0] * T[0] + TS[1] * T[1] + TS[2] * T[2] + kCov2dFloor;
    const double cb = TS[0] * T[3] + TS[1] * T[4] + TS[2] * T[5];
    const double cc = TS[3] * T[3] + TS[4] * T[4] + TS[5] * T[5] + kCov2dFloor;
    const double o = a.opacity[i];
    const double oc = fmin(o, kAlphaCapD);
    if (oc >= kAlphaMinD) {
      const double lam = 0.5 * (ca + cc + hypot(ca - cc, 2 * cb));
      const double r = sqrt(2.0 * log(oc / kAlphaMinD) * lam);
      const bool inside = !(mx + r < 0 || mx - r > a.W - 1 || my + r < 0 || my - r > a.H - 1);
      if (r > 0.0 && inside) {
        // binning box: the alpha >= 1/255 ellipse at the true opacity (which may
        // exceed the cap) reaches |dx| <= sqrt(k cov_xx), |dy| <= sqrt(k cov_yy),
        // k = 2 ln(o / alpha_min); plus a guard for the fp32 evaluation
        const double kq = 2.0 * log(o / kAlphaMinD);
        const double hx = sqrt(kq * ca) * (1.0 + 1e-5) + 0.02, hy = sqrt(kq * cc) * (1.0 + 1e-5) + 0.02;
        int x0 = (int)ceil(mx - hx), x1 = (int)floor(mx + hx);
        int y0 = (int)ceil(my - hy), y1 = (int)floor(my + hy);
        x0 = max(x0, 0);
        y0 = max(y0, 0);
        x1 = min(x1, a.W - 1);
        y1 = min(y1, a.H - 1);
        bx0 = (short)x0;
        bx1 = (short)x1;
        by0 = (short)y0;
        by1 = (short)y1;
        key = (unsigned long long)__double_as_longlong(z);
        if (x0 <= x1 && y0 <= y1) {
          rect[0] = (unsigned short)(x0 / kRTile);
          rect[1] = (unsigned short)(y0 / kRTile);
          rect[2] = (unsigned short)(x1 / kRTile);
          rect[3] = (unsigned short)(y1 / kRTile);
          tiles = (unsigned)(rect[2] - rect[0] + 1) * (unsigned)(rect[3] - rect[1] + 1);
        }
        const double det = ca * cc - cb * cb;
        const double ia = cc / det, ib = -cb / det, ic = ca / det;
        SplatData sd;
        sd.mx = mx;
        sd.my = my;
        sd.A = (float)(-0.5 * ia);
        sd.B = (float)(-ib);
        sd.C = (float)(-0.5 * ic);
        sd.o = (float)o;
        if (a.rgb0) {   // degree-0 colour: view-independent (splat3d_kernel)
          for (int c = 0; c < 3; ++c) sd.rgb[c] = __ldg(a.rgb0 + 3 * i + c);
        } else {
          const double nd = sqrt(dl[0] * dl[0] + dl[1] * dl[1] + dl[2] * dl[2]);
          const double dir[3] = {dl[0] / nd, dl[1] / nd, dl[2] / nd};
          sh_eval_rgb(a.sh_dc + 3 * i, a.sh_rest ? a.sh_rest + 3ll * a.sh_k * i : nullptr, a.sh_k, dir, sd.rgb);
        }
        sd.bx0 = bx0;
        sd.bx1 = bx1;
        sd.by0 = by0;
        sd.by1 = by1;
        if (in_range) a.splat[i] = sd;
      }
    }
  }
  const ushort4 r4 = make_ushort4(rect[0], rect[1], rect[2], rect[3]);
  if (in_range) {
    a.depth_key[i] = key;
    a.order_in[i] = (int)i;
    a.tiles[i] = tiles;
    reinterpret_cast<ushort4*>(a.rect)[i] = r4;
  }
  if (in_range && a.depth32)   // a monotone 32-bit depth key: the float below z (culled: last)
    a.depth32[i] = key == ~0ull ? 0xffffffffu : __float_as_uint(__double2float_rd(z));
}

struct TileCountPolicy {
  const int* order;
  const unsigned* tiles;
  unsigned* offs;
  unsigned long long* total_out;
  __device__ unsigned long long value(long long s) const { return tiles[order[s]]; }
  __device__ void store(long long s, unsigned long long ex, unsigned long long) const { offs[s] = (unsigned)ex; }
  __device__ void total(unsigned long long t) const { *total_out = t; }
};

// The fused attribution epilogue (BlendArgs::gt set): the stored fp32 image
// value i and gt give the raw L1 error exactly as the step's input pass
// computes it (fp64, numpy order: (|d0| + |d1|) + |d2|, no contraction);
// per-view min/max by a block reduction and two atomics, the candidate bit
// by one atomicOr per (warp, word), the ever-dominant flag per candidate.
// the per-pixel part: raw error -> 16-bit cache, ever-dominant flag, the
// candidate bits of the warp's four 8-pixel row segments (lanes 8r .. 8r + 7
// = one row: the layout of both blend kernels), the running min/max
__device__ __forceinline__ void epi_pixel(const BlendArgs& a, bool inside, int y, int x, float i0, float i1,
                                          float i2, int bi, double& lo, double& hi) {
  const int lane = threadIdx.x & 31;
  bool cand = false;
  if (inside) {
    const long long p = (long long)y * a.W + x;
    const float* g3 = a.gt + 3 * p;
    const double r = __dadd_rn(__dadd_rn(fabs(__dsub_rn((double)i0, (double)g3[0])),
                                         fabs(__dsub_rn((double)i1, (double)g3[1]))),
                               fabs(__dsub_rn((double)i2, (double)g3[2])));
    a.rawf[p] = raw16(r);
    lo = fmin(lo, r);
    hi = fmax(hi, r);
    if (bi >= 0 && bi < a.N && __ldg(a.cls + bi) == 1) {
      cand = true;
      if (a.dom_flag[bi] == 0) a.dom_flag[bi] = 1;
    }
  }
  static_assert(kRTile == 16, "epilogue: 8-pixel row segments");
  const unsigned b = __ballot_sync(0xffffffffu, cand);
  if ((lane & 7) == 0 && y < a.H) {   // the first pixel of its segment (x may be >= W)
    const long long p0 = (long long)y * a.W + x;
    const unsigned seg = (b >> (lane & 24)) & 0xffu;
    if (seg) {
      const unsigned long long w = (unsigned long long)seg << (p0 & 31);
      if ((unsigned)w) atomicOr(a.cand_bits + (p0 >> 5), (unsigned)w);
      if ((unsigned)(w >> 32)) atomicOr(a.cand_bits + (p0 >> 5) + 1, (unsigned)(w >> 32));
    }
  }
}

// the tile's min/max into its own slot (no same-address atomics: 4k tiles per
// view); reduce_tile_minmax folds them per view before the thresholds
template <int NW>
__device__ __forceinline__ void epi_reduce(const BlendArgs& a, double lo, double hi) {
  __shared__ double s_lo[NW], s_hi[NW];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int o = 16; o > 0; o >>= 1) {
    lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  if (lane == 0) {
    s_lo[wid] = lo;
    s_hi[wid] = hi;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < NW; ++w) {
      lo = fmin(lo, s_lo[w]);
      hi = fmax(hi, s_hi[w]);
    }
    a.lohi[2 * blockIdx.x + 0] = (unsigned long long)__double_as_longlong(lo);
    a.lohi[2 * blockIdx.x + 1] = (unsigned long long)__double_as_longlong(hi);
  }
}

__device__ __forceinline__ void render_epilogue(const BlendArgs& a, bool inside, int y, int x, float i0, float i1,
                                                float i2, int bi) {
  double lo = INFINITY, hi = 0.0;
  epi_pixel(a, inside, y, x, i0, i1, i2, bi, lo, hi);
  epi_reduce<kRThreads / 32>(a, lo, hi);
}

__device__ __forceinline__ float ex2_ftz(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// A block per 16 x 16 tile, a warp per 8 x 4 pixel block of it.  Splats come in
// batches of 256 (shared memory); each carries the mask of the 8 pixel blocks
// its alpha >= 1/255 box touches, so a warp walks only its own splats (ballot
// over the masks, then the set bits) -- the box is exact up to a guard, so a
// skipped (pixel, splat) pair has alpha below 1/255 and would be skipped anyway.
template <bool STATS, bool EPI>
__global__ void __launch_bounds__(kRThreads) blend_kernel(BlendArgs a) {
  pdl_wait();   // programmatic dependent launch: the previous kernel's results are visible
  struct Sm {
    float mx, my, A, B, C, o, r, g, b;
    int idx;
  };
  constexpr unsigned FULL = 0xffffffffu;
  // two batch buffers: batch i + 1 is staged while batch i is walked, one
  // barrier per batch
  __shared__ Sm sm[2][kRThreads];
  __shared__ unsigned char smask[2][kRThreads];
  __shared__ float wacc[STATS ? 2 : 1][STATS ? kRThreads : 1];
  unsigned long long n_contrib = 0;
  const int tile = blockIdx.x;
  if (a.vflag && *a.vflag) return;   // the view's binning overflowed: the host renders it again
  const int tyi = tile / a.tiles_x, txi = tile % a.tiles_x;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int lx = 8 * (wid & 1) + (lane & 7), ly = 4 * (wid >> 1) + (lane >> 3);
  const int x = txi * kRTile + lx, y = tyi * kRTile + ly;
  const bool inside = x < a.W && y < a.H;
  const double ox = (double)(txi * kRTile), oy = (double)(tyi * kRTile);
  const int beg = a.tile_start[tile], end = a.tile_end[tile];
  float T = 1.0f, best = 0.0f, cr = 0.0f, cg = 0.0f, cbl = 0.0f;
  int bi = -1;
  bool done = !inside;
  const float fx = (float)lx, fy = (float)ly;
  auto stage = [&](int base, int buf) {   // this thread's splat of the batch at `base`
    const int j = base + threadIdx.x;
    if (STATS) wacc[buf][threadIdx.x] = 0.0f;
    unsigned m = 0u;
    if (j < end) {
      const int g = a.order[(int)(a.keys[j] & 0xffffffffull)];
      const SplatData d = a.splat[g];
      Sm e;
      e.mx = (float)(d.mx - ox);
      e.my = (float)(d.my - oy);
      e.A = d.A;
      e.B = d.B;
      e.C = d.C;
      e.o = d.o;
      e.r = d.rgb[0];
      e.g = d.rgb[1];
      e.b = d.rgb[2];
      e.idx = g;
      sm[buf][threadIdx.x] = e;
      // pixel blocks of the support box: column halves x 4 row quarters
      const int xl = (int)d.bx0 - txi * kRTile, xh = (int)d.bx1 - txi * kRTile;
      const int yl = (int)d.by0 - tyi * kRTile, yh = (int)d.by1 - tyi * kRTile;
      if (xh >= 0 && xl < kRTile && yh >= 0 && yl < kRTile) {
        const unsigned cm = (xl < 8 ? 1u : 0u) | (xh >= 8 ? 2u : 0u);
        const int r0 = max(yl, 0) >> 2, r1 = min(yh, kRTile - 1) >> 2;
        for (int r = r0; r <= r1; ++r) m |= cm << (2 * r);
      }
    }
    smask[buf][threadIdx.x] = (unsigned char)m;
  };
  auto flush = [&](int base, int buf) {   // the batch's summed weights (statistics mode)
    if (STATS && a.weight && base + (int)threadIdx.x < end && wacc[buf][threadIdx.x] > 0.0f)
      atomicAdd(a.weight + sm[buf][threadIdx.x].idx, wacc[buf][threadIdx.x]);
  };
  if (beg < end) stage(beg, 0);
  int buf = 0;
  for (int base = beg; base < end; base += kRThreads, buf ^= 1) {
    // the barrier publishes batch `base` and retires the walk of the one before
    if (__syncthreads_count(done) == kRThreads) break;
    if (STATS && base > beg) flush(base - kRThreads, buf ^ 1);
    if (base + kRThreads < end) stage(base + kRThreads, buf ^ 1);
    const int cnt = min(kRThreads, end - base);
    if (!__all_sync(FULL, done)) {
      for (int c = 0; c < cnt; c += 32) {
        unsigned bits = __ballot_sync(FULL, c + lane < cnt && ((smask[buf][c + lane] >> wid) & 1u));
        while (bits) {   // warp-uniform
          const int k = c + __ffs(bits) - 1;
          bits &= bits - 1u;
          if (done) continue;
          const Sm& e = sm[buf][k];
          const float dx = fx - e.mx, dy = fy - e.my;
          const float power = e.A * dx * dx + e.B * dx * dy + e.C * dy * dy;
          // __expf without its denormal path: results below 2^-126 give alpha < 1/255 either way
          const float alpha = fminf(kAlphaCap, e.o * ex2_ftz(power * 1.4426950408889634f));
          if (alpha < kAlphaMin) continue;
          const float w = T * alpha;
          if (STATS) {
            if (a.weight) atomicAdd(&wacc[buf][k], w);
            ++n_contrib;
          }
          cr += w * e.r;
          cg += w * e.g;
          cbl += w * e.b;
          if (w > best) {
            best = w;
            bi = e.idx;
          }
          T = T * (1.0f - alpha);
          if (!STATS && T < 1e-8f && T * kAlphaCap <= best) done = true;
        }
        if (__all_sync(FULL, done)) break;
      }
    }
  }
  if (STATS && beg < end) {   // the last walked batch (statistics mode never stops early)
    __syncthreads();
    const int last = beg + ((end - beg - 1) / kRThreads) * kRThreads;
    flush(last, ((end - beg - 1) / kRThreads) & 1);
  }
  if (STATS && a.contrib) {
    for (int o = 16; o > 0; o >>= 1) n_contrib += __shfl_xor_sync(0xffffffffu, n_contrib, o);
    if ((threadIdx.x & 31) == 0 && n_contrib) atomicAdd(a.contrib, n_contrib);
  }
  // the composite once: the epilogue must see exactly the stored values
  const float i0 = cr + T * a.bg[0], i1 = cg + T * a.bg[1], i2 = cbl + T * a.bg[2];
  if (inside) {
    const long long p = (long long)y * a.W + x;
    a.image[3 * p + 0] = i0;
    a.image[3 * p + 1] = i1;
    a.image[3 * p + 2] = i2;
    a.dominant[p] = bi;
  }
  if (EPI) render_epilogue(a, inside, y, x, i0, i1, i2, bi);
}

// ---------------------------------------------------------------- depth order
// After the stable sort on the 32-bit keys, runs of equal keys (distinct
// doubles inside one float, or equal depths) are in index order; each run
// goes to (z, index) order here, the reference's order (ref/raster.py:118).
// A run longer than kFixupMax flags the view (the 64-bit sort redoes it).
constexpr int kFixupMax = 256;
__global__ void depth_fixup_kernel(const unsigned* __restrict__ k32, int* __restrict__ order,
                                   const unsigned long long* __restrict__ z64, long long n, int* flag) {
  pdl_wait();   // programmatic dependent launch: the previous kernel's results are visible
  const long long s = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n) return;
  const unsigned k = k32[s];
  if (k == 0xffffffffu) return;                  // culled: sorted last, never drawn
  if (s > 0 && k32[s - 1] == k) return;           // not the head of its run
  if (s + 1 >= n || k32[s + 1] != k) return;      // a run of one
  long long e = s + 1;
  while (e < n && k32[e] == k && e - s < kFixupMax) ++e;
  if (e < n && k32[e] == k) {
    atomicExch(flag, 2);
    return;
  }
  for (long long i = s + 1; i < e; ++i) {         // insertion sort by (z bits, index)
    const int gi = order[i];
    const unsigned long long zi = z64[gi];
    long long j = i - 1;
    while (j >= s) {
      const int gj = order[j];
      const unsigned long long zj = z64[gj];
      if (zj < zi || (zj == zi && gj < gi)) break;
      order[j + 1] = gj;
      --j;
    }
    order[j + 1] = gi;
  }
}

// the (tile << 32 | depth rank) keys of every (tile, splat) pair, and padding
// keys (sorted last) up to the capacity the host sorts; a view whose pairs
// exceed the capacity is flagged and skipped (rendered again by the host)
__global__ void __launch_bounds__(256) duplicate_kernel(DupArgs a) {
  pdl_wait();   // programmatic dependent launch: the previous kernel's results are visible
  constexpr unsigned FULL = 0xffffffffu;
  const long long s = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const unsigned long long total = *a.total;
  if (*a.flag) return;   // grid-uniform
  if (total > (unsigned long long)a.cap) {
    if (s == 0) *a.flag = 1;
    return;
  }
  if (s >= (long long)total && s < a.cap) a.keys[s] = ~0ull;
  if (((long long)blockIdx.x * blockDim.x) >= a.n) return;   // block-uniform: no splats in this block
  const bool in = s < a.n;
  const int g = in ? a.order[s] : 0;
  const unsigned cnt = in ? a.tiles[g] : 0u;
  const ushort4 r = cnt ? reinterpret_cast<const ushort4*>(a.rect)[g] : make_ushort4(0, 0, 0, 0);
  const unsigned long long off = cnt ? a.offs[s] : 0ull;
  // small rects by their own thread; large ones (a background splat over the
  // whole image) by the whole warp
  const bool big = cnt > 16u;
  if (cnt && !big) {
    unsigned long long o = off;
    for (int ty = r.y; ty <= r.w; ++ty)
      for (int tx = r.x; tx <= r.z; ++tx) a.keys[o++] = ((unsigned long long)(ty * a.tiles_x + tx) << 32) | (unsigned long long)s;
  }
  unsigned bm = __ballot_sync(FULL, big);
  const int lane = threadIdx.x & 31;
  const unsigned r01 = (unsigned)r.x | ((unsigned)r.y << 16), r23 = (unsigned)r.z | ((unsigned)r.w << 16);
  while (bm) {
    const int src = __ffs(bm) - 1;
    bm &= bm - 1u;
    const unsigned p = __shfl_sync(FULL, r01, src), q = __shfl_sync(FULL, r23, src);
    const unsigned long long o0 = __shfl_sync(FULL, off, src);
    const long long ss = __shfl_sync(FULL, s, src);
    const int x0 = (int)(p & 0xffffu), y0 = (int)(p >> 16), x1 = (int)(q & 0xffffu), y1 = (int)(q >> 16);
    const int w = x1 - x0 + 1, tot = w * (y1 - y0 + 1);
    for (int k = lane; k < tot; k += 32)
      a.keys[o0 + k] = ((unsigned long long)((y0 + k / w) * a.tiles_x + x0 + k % w) << 32) | (unsigned long long)ss;
  }
}

__global__ void tile_ranges_kernel(const unsigned long long* keys, const unsigned long long* total, const int* flag,
                                   int* start, int* end) {
  pdl_wait();   // programmatic dependent launch: the previous kernel's results are visible
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long n = (long long)*total;
  if (i >= n || *flag) return;
  const int t = (int)(keys[i] >> 32);
  if (i == 0 || (int)(keys[i - 1] >> 32) != t) start[t] = (int)i;
  if (i == n - 1 || (int)(keys[i + 1] >> 32) != t) end[t] = (int)(i + 1);
}

// ---------------------------------------------------------------- launchers
cudaError_t launch_preprocess(const PreArgs& a, cudaStream_t s) {
  if (a.n > 0) launch_k(preprocess_kernel, (unsigned)((a.n + 255) / 256), 256, 0, s, a);
  return cudaGetLastError();
}

cudaError_t launch_tile_count_scan(const int* order, const unsigned* tiles, unsigned* offs,
                                   unsigned long long* total, long long n, ScanState st, cudaStream_t s) {
  TileCountPolicy p{order, tiles, offs, total};
  return launch_scan(p, n, st, s);
}

cudaError_t launch_duplicate(const DupArgs& a, cudaStream_t s) {
  const long long m = a.n > a.cap ? a.n : a.cap;
  if (m > 0) launch_k(duplicate_kernel, (unsigned)((m + 255) / 256), 256, 0, s, a);
  return cudaGetLastError();
}

cudaError_t launch_tile_ranges(const unsigned long long* keys, long long cap, const unsigned long long* total,
                               const int* flag, int* start, int* end, cudaStream_t s) {
  if (cap > 0) launch_k(tile_ranges_kernel, (unsigned)((cap + 255) / 256), 256, 0, s, keys, total, flag, start, end);
  return cudaGetLastError();
}

cudaError_t launch_depth_fixup(const unsigned* k32, int* order, const unsigned long long* z64, long long n, int* flag,
                               cudaStream_t s) {
  if (n > 0) launch_k(depth_fixup_kernel, (unsigned)((n + 255) / 256), 256, 0, s, k32, order, z64, n, flag);
  return cudaGetLastError();
}

// per view: the min/max over its tiles' slots (bit patterns of non-negative
// doubles order as unsigned integers; an empty tile holds +inf / 0)
__global__ void __launch_bounds__(256) reduce_tile_minmax_kernel(const unsigned long long* __restrict__ tiles,
                                                                 int n_tiles, unsigned long long* __restrict__ lohi) {
  pdl_wait();   // programmatic dependent launch: the previous kernel's results are visible
  const int v = blockIdx.x;
  const unsigned long long* t = tiles + 2ll * n_tiles * v;
  unsigned long long lo = ~0ull, hi = 0ull;
  for (int i = threadIdx.x; i < n_tiles; i += blockDim.x) {
    lo = min(lo, t[2 * i]);
    hi = max(hi, t[2 * i + 1]);
  }
  for (int o = 16; o > 0; o >>= 1) {
    lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  __shared__ unsigned long long slo[8], shi[8];
  if ((threadIdx.x & 31) == 0) {
    slo[threadIdx.x >> 5] = lo;
    shi[threadIdx.x >> 5] = hi;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < 8; ++w) {
      lo = min(lo, slo[w]);
      hi = max(hi, shi[w]);
    }
    lohi[2 * v] = min(lo, 0x7ff0000000000000ull);   // +inf when the view is empty
    lohi[2 * v + 1] = hi;
  }
}

cudaError_t launch_reduce_tile_minmax(const unsigned long long* tiles, int n_tiles, int n_views,
                                      unsigned long long* lohi, cudaStream_t s) {
  launch_k(reduce_tile_minmax_kernel, n_views, 256, 0, s, tiles, n_tiles, lohi);
  return cudaGetLastError();
}

cudaError_t launch_blend(const BlendArgs& a, int n_tiles, cudaStream_t s) {
  if (a.weight || a.contrib)
    launch_k(blend_kernel<true, false>, n_tiles, kRThreads, 0, s, a);
  else if (a.gt)
    launch_k(blend_kernel<false, true>, n_tiles, kRThreads, 0, s, a);
  else
    launch_k(blend_kernel<false, false>, n_tiles, kRThreads, 0, s, a);
  return cudaGetLastError();
}

}  // namespace adps
