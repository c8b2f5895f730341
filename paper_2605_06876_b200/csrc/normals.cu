// Fallback-child normals on the device, bit-identical to numpy.
//
// The reference draws rng.normal(size=(k, 3)) per fallback parent in
// ascending parent order (ref/adc.py:97, via init_child's fallback branch);
// with one Generator those draws are the next 6F values of
// Generator(PCG64).standard_normal.  numpy computes each value with a
// 256-layer ziggurat over a 128-bit LCG (XSL-RR output): one 64-bit draw per
// attempt in ~98.5% of cases, one more for a wedge test, two per round of the
// tail loop, and a rejected attempt simply restarts.  So the stream is a
// chain of attempts with data-dependent lengths; on the GPU:
//   1. classify: every stream position p of a window is treated as a possible
//      attempt start (a thread jumps the LCG to its chunk in O(log p)) and
//      yields (value, length, accepted);
//   2. an attempt is reached by the chain unless an earlier attempt's draws
//      cover it.  With reach(p) = p + length(p), position p is certainly an
//      attempt start when max_{q<p} reach(q) <= p (a max-scan); the few
//      positions inside multi-draw attempts are resolved by short walks from
//      those starts;
//   3. accepted attempt starts are ranked (exclusive sum) and the first n are
//      written; the draws consumed let the host advance its Generator.
// Bit-exactness: the LCG and the ziggurat arithmetic are exact IEEE
// operations (-fmad=false); the tail's log1p is glibc's (fdlibm-derived,
// FMA-contracted) algorithm restated operation by operation and checked
// against the host libm (tests/test_normals.py); the wedge test compares
// against CUDA's exp, and any comparison within a few ulp is flagged so the
// caller redraws on the host (never observed; ~1e-15 per wedge test).
#include <cub/cub.cuh>
#include <math_constants.h>

#include "adps_internal.cuh"
#include "normals.cuh"
#include "ziggurat_tables.h"

namespace adps {

namespace {

struct U128 {
  unsigned long long lo, hi;
};

__device__ __forceinline__ U128 mul128(U128 a, U128 b) {
  U128 r;
  r.lo = a.lo * b.lo;
  r.hi = __umul64hi(a.lo, b.lo) + a.lo * b.hi + a.hi * b.lo;
  return r;
}
__device__ __forceinline__ U128 add128(U128 a, U128 b) {
  U128 r;
  r.lo = a.lo + b.lo;
  r.hi = a.hi + b.hi + (r.lo < a.lo ? 1ull : 0ull);
  return r;
}
__device__ __forceinline__ U128 pcg_mult() {
  U128 m;
  m.lo = 0x4385DF649FCCF645ull;
  m.hi = 0x2360ED051FC65DA4ull;
  return m;
}
// state after one more step (numpy's pcg64: step, then output of the new state)
__device__ __forceinline__ U128 pcg_step(U128 s, U128 inc) { return add128(mul128(s, pcg_mult()), inc); }
__device__ __forceinline__ unsigned long long pcg_out(U128 s) {
  const unsigned long long x = s.hi ^ s.lo;
  const unsigned rot = (unsigned)(s.hi >> 58);
  return (x >> rot) | (x << ((64u - rot) & 63u));
}
__device__ __forceinline__ double pcg_double(unsigned long long r) {
  return __dmul_rn((double)(r >> 11), 1.0 / 9007199254740992.0);
}
// LCG jump-ahead by delta steps (Brown's algorithm)
__device__ U128 pcg_advance(U128 s, U128 inc, unsigned long long delta) {
  U128 acc_mult{1ull, 0ull}, acc_plus{0ull, 0ull};
  U128 cur_mult = pcg_mult(), cur_plus = inc;
  while (delta) {
    if (delta & 1ull) {
      acc_mult = mul128(acc_mult, cur_mult);
      acc_plus = add128(mul128(acc_plus, cur_mult), cur_plus);
    }
    cur_plus = mul128(add128(cur_mult, U128{1ull, 0ull}), cur_plus);
    cur_mult = mul128(cur_mult, cur_mult);
    delta >>= 1;
  }
  return add128(mul128(acc_mult, s), acc_plus);
}

// glibc's log1p (fdlibm s_log1p.c with the Estrin polynomial), with the FMA
// contractions of the x86-64 build made explicit
__device__ double glibc_log1p(double x) {
  const double ln2_hi = 6.93147180369123816490e-01, ln2_lo = 1.90821492927058770002e-10;
  const double two54 = 1.80143985094819840000e+16;
  const double Lp1 = 6.666666666666735130e-01, Lp2 = 3.999999999940941908e-01, Lp3 = 2.857142874366239149e-01,
               Lp4 = 2.222219843214978396e-01, Lp5 = 1.818357216161805012e-01, Lp6 = 1.531383769920937332e-01,
               Lp7 = 1.479819860511658591e-01;
  double f = 0.0, c = 0.0, u;
  int hu = 0;
  const int hx = __double2hiint(x);
  const int ax = hx & 0x7fffffff;
  int k = 1;
  if (hx < 0x3FDA827A) {
    if (ax >= 0x3ff00000) return x == -1.0 ? -CUDART_INF : CUDART_NAN;
    if (ax < 0x3e200000) {
      if (two54 + x > 0.0 && ax < 0x3c900000) return x;
      return __fma_rn(-__dmul_rn(x, x), 0.5, x);
    }
    if (hx > 0 || hx <= (int)0xbfd2bec3) {
      k = 0;
      f = x;
      hu = 1;
    }
  }
  if (hx >= 0x7ff00000) return x + x;
  if (k != 0) {
    if (hx < 0x43400000) {
      u = __dadd_rn(1.0, x);
      hu = __double2hiint(u);
      k = (hu >> 20) - 1023;
      c = k > 0 ? __dsub_rn(1.0, __dsub_rn(u, x)) : __dsub_rn(x, __dsub_rn(u, 1.0));
      c = __ddiv_rn(c, u);
    } else {
      u = x;
      hu = __double2hiint(u);
      k = (hu >> 20) - 1023;
      c = 0.0;
    }
    hu &= 0x000fffff;
    if (hu < 0x6a09e) {
      u = __hiloint2double(hu | 0x3ff00000, __double2loint(u));
    } else {
      k += 1;
      u = __hiloint2double(hu | 0x3fe00000, __double2loint(u));
      hu = (0x00100000 - hu) >> 2;
    }
    f = __dsub_rn(u, 1.0);
  }
  const double dk = (double)k;
  const double hfsq = __dmul_rn(__dmul_rn(0.5, f), f);
  if (hu == 0) {
    if (f == 0.0) {
      if (k == 0) return 0.0;
      c = __fma_rn(dk, ln2_lo, c);
      return __fma_rn(dk, ln2_hi, c);
    }
    const double R = __dmul_rn(hfsq, __fma_rn(-0.66666666666666666, f, 1.0));
    if (k == 0) return __dsub_rn(f, R);
    return __fma_rn(dk, ln2_hi, -__dsub_rn(__dsub_rn(R, __fma_rn(dk, ln2_lo, c)), f));
  }
  const double s = __ddiv_rn(f, __dadd_rn(2.0, f));
  const double z = __dmul_rn(s, s);
  const double z2 = __dmul_rn(z, z), z4 = __dmul_rn(z2, z2), z6 = __dmul_rn(z4, z2);
  const double R2 = __fma_rn(z, Lp3, Lp2), R3 = __fma_rn(z, Lp5, Lp4), R4 = __fma_rn(z, Lp7, Lp6);
  const double R = __fma_rn(z6, R4, __fma_rn(z4, R3, __fma_rn(z, Lp1, __dmul_rn(z2, R2))));
  const double t = __dmul_rn(s, __dadd_rn(hfsq, R));
  if (k == 0) return __dsub_rn(f, __dsub_rn(hfsq, t));
  return __fma_rn(dk, ln2_hi, -__dsub_rn(__dsub_rn(hfsq, __dadd_rn(t, __fma_rn(dk, ln2_lo, c))), f));
}

constexpr int kChunk = 32;   // stream positions per thread

// 1. every position p = 1..window as an attempt start
__global__ void classify_kernel(NormalsArgs a) {
  pdl_wait();   // programmatic dependent launch: the previous kernel's results are visible
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long start = 1 + t * kChunk;
  if (start > a.window) return;
  const U128 inc{a.inc_lo, a.inc_hi};
  U128 s = pcg_advance(U128{a.state_lo, a.state_hi}, inc, (unsigned long long)(start - 1));
  for (int j = 0; j < kChunk; ++j) {
    const long long p = start + j;
    if (p > a.window) break;
    s = pcg_step(s, inc);
    unsigned long long r = pcg_out(s);
    const int idx = (int)(r & 0xff);
    r >>= 8;
    const unsigned long long rabs = (r >> 1) & 0x000fffffffffffffull;
    double x = __dmul_rn((double)rabs, kZigWi[idx]);
    if (r & 1ull) x = -x;
    int len = 1;
    bool acc = true;
    if (rabs >= kZigKi[idx]) {
      U128 q = s;
      if (idx == 0) {   // tail beyond r: Marsaglia's exponential rejection
        acc = false;
        for (int it = 0; it < 100 && !acc; ++it) {
          q = pcg_step(q, inc);
          const double u1 = pcg_double(pcg_out(q));
          q = pcg_step(q, inc);
          const double u2 = pcg_double(pcg_out(q));
          const double xx = __dmul_rn(-kZigNorInvR, glibc_log1p(-u1));
          const double yy = -glibc_log1p(-u2);
          len += 2;
          if (__dadd_rn(yy, yy) > __dmul_rn(xx, xx)) {
            acc = true;
            x = ((rabs >> 8) & 1ull) ? -__dadd_rn(kZigNorR, xx) : __dadd_rn(kZigNorR, xx);
          }
        }
        if (!acc) atomicOr(a.status, 1u);
      } else {          // wedge
        q = pcg_step(q, inc);
        const double u = pcg_double(pcg_out(q));
        len = 2;
        const double lhs = __dadd_rn(__dmul_rn(__dsub_rn(kZigFi[idx - 1], kZigFi[idx]), u), kZigFi[idx]);
        const double e = exp(__dmul_rn(__dmul_rn(-0.5, x), x));
        acc = lhs < e;
        if (fabs(__dsub_rn(lhs, e)) <= e * 0x1p-50) atomicOr(a.status, 1u);
      }
    }
    const long long k = p - 1;
    a.val[k] = x;
    a.len[k] = (unsigned char)len;
    a.acc[k] = acc ? 1 : 0;
    a.reach[k] = (int)(p + len);
  }
}

__device__ __forceinline__ bool is_start(const NormalsArgs& a, long long p) {
  return p == 1 || a.reach_max[p - 2] <= p;
}

// 2. positions inside a multi-draw attempt: follow the chain from the starts
__global__ void walk_kernel(NormalsArgs a) {
  pdl_wait();   // programmatic dependent launch: the previous kernel's results are visible
  for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < a.window;
       k += (long long)gridDim.x * blockDim.x) {
    if (a.len[k] == 1) continue;
    const long long p = k + 1;
    if (!is_start(a, p)) continue;
    long long q = p + a.len[k];
    while (q <= a.window && !is_start(a, q)) {
      a.walked[q - 1] = 1;
      q += a.len[q - 1];
    }
  }
}

__global__ void emit_flag_kernel(NormalsArgs a) {
  pdl_wait();   // programmatic dependent launch: the previous kernel's results are visible
  for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < a.window;
       k += (long long)gridDim.x * blockDim.x)
    a.emit_idx[k] = ((is_start(a, k + 1) || a.walked[k]) && a.acc[k]) ? 1 : 0;
}

// 3. the first n accepted attempts in stream order
__global__ void write_kernel(NormalsArgs a) {
  pdl_wait();   // programmatic dependent launch: the previous kernel's results are visible
  for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < a.window;
       k += (long long)gridDim.x * blockDim.x) {
    const bool emit = (is_start(a, k + 1) || a.walked[k]) && a.acc[k];
    const long long i = a.emit_idx[k];
    if (emit && i < a.n) {
      a.out[i] = a.val[k];
      if (i == a.n - 1) *a.consumed = (unsigned long long)(k + a.len[k]);
    }
    if (k == a.window - 1 && i + (emit ? 1 : 0) < a.n) atomicOr(a.status, 2u);
  }
}

struct MaxOp {
  __device__ __forceinline__ int operator()(int x, int y) const { return x > y ? x : y; }
};

}  // namespace

long long normals_window(long long n) { return n + n / 16 + 4096; }

size_t normals_temp_bytes(long long window) {
  size_t b1 = 0, b2 = 0;
  cub::DeviceScan::InclusiveScan(nullptr, b1, (int*)nullptr, (int*)nullptr, MaxOp(), (int)window);
  cub::DeviceScan::ExclusiveSum(nullptr, b2, (int*)nullptr, (int*)nullptr, (int)window);
  return b1 > b2 ? b1 : b2;
}

cudaError_t launch_normals(const NormalsArgs& a, void* temp, size_t temp_bytes, cudaStream_t s) {
  if (a.n <= 0) return cudaSuccess;
  const long long threads = (a.window + kChunk - 1) / kChunk;
  launch_k(classify_kernel, (unsigned)((threads + 127) / 128), 128, 0, s, a);
  size_t tb = temp_bytes;
  cudaError_t e = cub::DeviceScan::InclusiveScan(temp, tb, a.reach, a.reach_max, MaxOp(), (int)a.window, s);
  if (e != cudaSuccess) return e;
  e = cudaMemsetAsync(a.walked, 0, (size_t)a.window, s);
  if (e != cudaSuccess) return e;
  const unsigned grid = (unsigned)((a.window + 255) / 256);
  launch_k(walk_kernel, grid, 256, 0, s, a);
  launch_k(emit_flag_kernel, grid, 256, 0, s, a);
  tb = temp_bytes;
  e = cub::DeviceScan::ExclusiveSum(temp, tb, a.emit_idx, a.emit_idx, (int)a.window, s);
  if (e != cudaSuccess) return e;
  launch_k(write_kernel, grid, 256, 0, s, a);
  return cudaGetLastError();
}

}  // namespace adps
