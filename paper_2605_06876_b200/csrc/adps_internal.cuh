// Internal definitions shared by the AdpSplit B200 kernels.
#pragma once

#include <cstdlib>
#include <utility>

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/adps.h"

namespace adps {

constexpr int kWarp = 32;

// ---------------------------------------------------- programmatic dependent launch
// Every kernel of the library starts with pdl_wait() (griddepcontrol.wait:
// returns once the previous kernel in the stream has completed and its writes
// are visible; a no-op without a programmatic dependency) and is launched by
// launch_k with programmatic stream serialization, so the next kernel's grid
// is set up and its blocks become resident while the previous one drains
// (1.3-3 us per kernel boundary on B200, tools/pdl_probe).  ADPS_PDL=0
// launches plainly.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

inline bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("ADPS_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                            Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// ---------------------------------------------------------------- constants
// ref/raster.py:20-24
constexpr float kAlphaCap = 0.99f;
constexpr float kAlphaMin = 1.0f / 255.0f;
constexpr double kAlphaCapD = 0.99;
constexpr double kAlphaMinD = 1.0 / 255.0;
constexpr double kCov2dFloor = 0.3;
// ref/error_partition.py:15, ref/child_init.py:21-22
constexpr double kSigmaFloor = 0.5;
constexpr double kDegenerateDenom = 1e-18;
constexpr double kParallelTol = 1e-12;
// ref/scene.py:16-33
constexpr double kShC0 = 0.28209479177387814;
constexpr double kShC1 = 0.4886025119029199;

// Attribution/CCL tile (maps + partition pass).
constexpr int kTileW = 32;
constexpr int kTileH = 32;
constexpr int kTilePx = kTileW * kTileH;
constexpr int kTileThreads = 256;
constexpr int kBorderSlots = 2 * kTileW + 2 * kTileH;   // top,bottom,left,right
constexpr int kMaxErodeHalo = 8;                          // r_erode <= 17

// Render tile.
constexpr int kRTile = 16;
constexpr int kRThreads = kRTile * kRTile;

// ------------------------------------------------------------------ records
// One connected error region: ref/error_partition.py:27-41 (ErrorRegion) with
// its pixel set replaced by exact integer moments.
struct RegionRec {
  int32_t view_pos;
  int32_t cand;        // Gaussian index
  int32_t band;
  int32_t minpix;      // y*W + x of the first (row-major) pixel
  long long m[6];      // n, Sx, Sy, Sxx, Sxy, Syy (global pixel coords)
};

// Fragment of a component that touches an interior tile edge.
struct PartialRec {
  int32_t view_pos;
  int32_t cand;
  int32_t band;
  int32_t minpix;
  long long m[6];
};

// Child proposal (ref/child_init.py:27-41), fp64, plus merge operands.
struct Proposal {
  double mu[3];
  double cov[6];    // xx xy xz yy yz zz
  double prec[6];
  double rgb[3];
  double inv_smax;  // 1 / max(s1, s2): 1/sqrt of the largest covariance eigenvalue
};

// Bounding data of 64 spatially sorted proposals (exact gate pruning).
struct TileBox {
  double c[3];      // centre
  double r;         // max |mu - c|
  double inv_s;     // min proposal inv_smax
  double lo[3], hi[3];   // rgb box
};

// Merged group record (ref/cross_view_merge.py:17-30), stored at its root slot.
struct GroupRec {
  double mu[3];
  double rgb[3];
  double evec[9];   // columns e_r, row-major [row*3+col]
  double lam[3];
  double extent;
};

// Device-side counters of one phase 1 (mirrors adps_counts + internals).
struct Counters {
  unsigned long long n_split;
  unsigned long long n_clone;
  unsigned long long n_regions;
  unsigned long long n_partials;
  unsigned long long n_proposals;
  unsigned long long merge_edges;
  unsigned long long n_fallback;
  unsigned long long n_reset;
  unsigned long long n_children;
  unsigned long long n_inserted;
  unsigned long long n_keep;
  unsigned long long n_large;
  unsigned long long n_small;
  unsigned long long n_groups_all;
  unsigned long long n_tile_pairs;
  unsigned long long pair_next;            // pair_tiles_kernel work counter
  unsigned long long n_fallback_pre;
  unsigned long long n_deferred;   // tiles the warp CCL handed to the block CCL
  unsigned long long normals_consumed;   // 64-bit draws used by adps_normals_pcg64
  unsigned long long stat_gates, stat_pass;
  unsigned long long shard_lo, shard_hi;     // this rank's candidate range under parent sharding
  unsigned long long shard_plo, shard_phi;   // ... and its proposal range
  unsigned long long n_owned_props;          // proposals of this rank's parents   // diagnostics (ADPS_MERGE_STATS builds)
  unsigned long long n_mid_groups, n_huge_groups;   // work lists of the group reduction
  unsigned long long n_cap_large;                   // groups of parents with many groups
  unsigned long long tile_records;   // tile CCLs: partials << 32 | regions (one atomic per batch; unpacked after)
  unsigned long long n_cap_huge;                    // parents whose groups are selected in shared memory
  unsigned long long prune_keep, prune_near;        // adps_prune_index
  unsigned int normals_status;           // bit0 near-tie (redraw on host), bit1 window short
  unsigned int degenerate;
  unsigned int overflow;   // bit0 regions, bit1 partials
};

struct CamD {
  double r[9];   // r_c2w row-major: columns are right, down, forward
  double c[3];
  double fx, fy, px, py;
  int w, h;
};

__host__ __device__ inline CamD load_cam(const double* row) {
  CamD k;
  for (int i = 0; i < 9; ++i) k.r[i] = row[i];
  for (int i = 0; i < 3; ++i) k.c[i] = row[9 + i];
  k.fx = row[12];
  k.fy = row[13];
  k.px = row[14];
  k.py = row[15];
  k.w = (int)row[16];
  k.h = (int)row[17];
  return k;
}

// ------------------------------------------------------------- fp64 helpers
// Explicit round-to-nearest ops: never contracted into FMA, so they match
// numpy's elementwise arithmetic bit for bit.
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double ddiv(double a, double b) { return __ddiv_rn(a, b); }

// quat (w,x,y,z) -> rotation, normalising first (ref/scene.py:183-193).
__host__ __device__ inline void quat_to_rot(const double q_in[4], double r[9]) {
  double nrm = sqrt(q_in[0] * q_in[0] + q_in[1] * q_in[1] + q_in[2] * q_in[2] + q_in[3] * q_in[3]);
  double w = q_in[0] / nrm, x = q_in[1] / nrm, y = q_in[2] / nrm, z = q_in[3] / nrm;
  r[0] = 1 - 2 * (y * y + z * z);
  r[1] = 2 * (x * y - w * z);
  r[2] = 2 * (x * z + w * y);
  r[3] = 2 * (x * y + w * z);
  r[4] = 1 - 2 * (x * x + z * z);
  r[5] = 2 * (y * z - w * x);
  r[6] = 2 * (x * z - w * y);
  r[7] = 2 * (y * z + w * x);
  r[8] = 1 - 2 * (x * x + y * y);
}

// R diag(d) R^T as symmetric 6-vector xx xy xz yy yz zz.
__host__ __device__ inline void rdrt(const double r[9], const double d[3], double out[6]) {
  double t[9];
  for (int i = 0; i < 3; ++i)
    for (int k = 0; k < 3; ++k) t[i * 3 + k] = r[i * 3 + k] * d[k];
  int idx = 0;
  for (int i = 0; i < 3; ++i)
    for (int j = i; j < 3; ++j) {
      out[idx++] = t[i * 3 + 0] * r[j * 3 + 0] + t[i * 3 + 1] * r[j * 3 + 1] + t[i * 3 + 2] * r[j * 3 + 2];
    }
}

__host__ __device__ inline double sym_quad(const double s[6], const double v[3]) {
  return s[0] * v[0] * v[0] + s[3] * v[1] * v[1] + s[5] * v[2] * v[2] +
         2.0 * (s[1] * v[0] * v[1] + s[2] * v[0] * v[2] + s[4] * v[1] * v[2]);
}

__host__ __device__ inline double sym_bilin(const double s[6], const double a[3], const double b[3]) {
  double sb0 = s[0] * b[0] + s[1] * b[1] + s[2] * b[2];
  double sb1 = s[1] * b[0] + s[3] * b[1] + s[4] * b[2];
  double sb2 = s[2] * b[0] + s[4] * b[1] + s[5] * b[2];
  return a[0] * sb0 + a[1] * sb1 + a[2] * sb2;
}

// Cyclic Jacobi eigen-decomposition of a symmetric 3x3 (fp64).  Returns
// eigenvalues ascending with matching eigenvector columns (LAPACK order).
__host__ __device__ inline void sym_eig3(const double s[6], double lam[3], double v[9]) {
  double a[3][3] = {{s[0], s[1], s[2]}, {s[1], s[3], s[4]}, {s[2], s[4], s[5]}};
  double e[3][3] = {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}};
  for (int sweep = 0; sweep < 24; ++sweep) {
    double off = fabs(a[0][1]) + fabs(a[0][2]) + fabs(a[1][2]);
    double scale = fabs(a[0][0]) + fabs(a[1][1]) + fabs(a[2][2]);
    if (off == 0.0 || off <= 1e-22 * scale) break;
    for (int p = 0; p < 2; ++p)
      for (int q = p + 1; q < 3; ++q) {
        double apq = a[p][q];
        if (apq == 0.0) continue;
        double theta = (a[q][q] - a[p][p]) / (2.0 * apq);
        double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
        double c = 1.0 / sqrt(t * t + 1.0), sn = t * c;
        for (int k = 0; k < 3; ++k) {
          double akp = a[k][p], akq = a[k][q];
          a[k][p] = c * akp - sn * akq;
          a[k][q] = sn * akp + c * akq;
        }
        for (int k = 0; k < 3; ++k) {
          double apk = a[p][k], aqk = a[q][k];
          a[p][k] = c * apk - sn * aqk;
          a[q][k] = sn * apk + c * aqk;
        }
        a[p][q] = a[q][p] = 0.0;
        for (int k = 0; k < 3; ++k) {
          double ekp = e[k][p], ekq = e[k][q];
          e[k][p] = c * ekp - sn * ekq;
          e[k][q] = sn * ekp + c * ekq;
        }
      }
  }
  int o[3] = {0, 1, 2};
  double d[3] = {a[0][0], a[1][1], a[2][2]};
  for (int i = 0; i < 3; ++i)
    for (int j = i + 1; j < 3; ++j)
      if (d[o[j]] < d[o[i]]) {
        int t = o[i];
        o[i] = o[j];
        o[j] = t;
      }
  for (int c = 0; c < 3; ++c) {
    lam[c] = d[o[c]];
    for (int r = 0; r < 3; ++r) v[r * 3 + c] = e[r][o[c]];
  }
}

// rotation (row-major) -> unit quaternion (w,x,y,z), ref/scene.py:196-215.
__host__ __device__ inline void rot_to_quat(const double r[9], double q[4]) {
  double tr = r[0] + r[4] + r[8];
  if (tr > 0) {
    double s = sqrt(tr + 1.0) * 2;
    q[0] = 0.25 * s;
    q[1] = (r[7] - r[5]) / s;
    q[2] = (r[2] - r[6]) / s;
    q[3] = (r[3] - r[1]) / s;
  } else {
    int i = 0;
    if (r[4] > r[i * 3 + i]) i = 1;
    if (r[8] > r[i * 3 + i]) i = 2;
    int j = (i + 1) % 3, k = (i + 2) % 3;
    double s = sqrt(1.0 + r[i * 3 + i] - r[j * 3 + j] - r[k * 3 + k]) * 2;
    q[0] = (r[k * 3 + j] - r[j * 3 + k]) / s;
    q[1 + i] = 0.25 * s;
    q[1 + j] = (r[j * 3 + i] + r[i * 3 + j]) / s;
    q[1 + k] = (r[k * 3 + i] + r[i * 3 + k]) / s;
  }
  double n = sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
  for (int t = 0; t < 4; ++t) q[t] /= n;
}

__host__ __device__ inline int ceil_log2(unsigned long long x) {
  int b = 0;
  while ((1ull << b) < x) ++b;
  return b;
}

// ------------------------------------------------------------ raw-error cache
// The input pass caches each pixel's raw L1 error in 16 bits: the top half of
// the bit pattern of RZ_fp32(raw) (sign 0, 8-bit exponent, 7-bit mantissa), i.e.
// raw rounded toward zero to that format.  Non-negative values order as their
// bit patterns, so a threshold compare raw >= X is an integer compare against
// T = top16(RZ_fp32(X)) + (X not representable), except when the pixel's code
// equals top16(RZ_fp32(X)) for a non-representable X: those pixels (~0.2 % at
// config 3) recompute the exact fp64 raw error from image and gt.
typedef unsigned short raw16_t;
__device__ __forceinline__ raw16_t raw16(double r) {
  return (raw16_t)(__float_as_uint(__double2float_rz(r)) >> 16);
}

// ---------------------------------------------------------- union-find (min)
// Roots are minimum indices; links only ever decrease (atomicMin).
__device__ __forceinline__ int uf_find(volatile int* p, int x) {
  int y = p[x];
  while (y != x) {
    x = y;
    y = p[x];
  }
  return x;
}

// find with path halving: only non-root entries are rewritten, always to an
// ancestor (a smaller index in the same tree), so concurrent atomicMin links
// on roots are never lost (ECL-CC style benign races).
__device__ __forceinline__ int uf_find_halve(volatile int* p, int x) {
  // (single-exit loops throughout: early returns from inside inlined loops
  // leave ptxas without a reconvergence point, and the warp's next shuffles
  // and votes then run as divergent "collective" sequences)
  int y = p[x];
  while (y != x) {
    const int z = p[y];
    if (z == y) {
      x = y;
      break;
    }
    p[x] = z;
    x = z;
    y = p[x];
  }
  return x;
}

__device__ __forceinline__ void uf_unite(int* p, int a, int b) {
  volatile int* vp = p;
  while (true) {
    a = uf_find_halve(vp, a);
    b = uf_find_halve(vp, b);
    if (a == b) break;
    if (a > b) {
      int t = a;
      a = b;
      b = t;
    }
    const int old = atomicMin(&p[b], a);
    if (old == b) break;
    b = old;
  }
}

// uf_unite that returns the root the two trees now share (the smaller of the
// two roots found; later links elsewhere may hang it below an even smaller
// one, but a and b stay in the same tree under it)
__device__ __forceinline__ int uf_unite_root(int* p, int a, int b) {
  volatile int* vp = p;
  while (true) {
    a = uf_find_halve(vp, a);
    b = uf_find_halve(vp, b);
    if (a == b) break;
    if (a > b) {
      int t = a;
      a = b;
      b = t;
    }
    const int old = atomicMin(&p[b], a);
    if (old == b) break;
    b = old;
  }
  return a;
}

}  // namespace adps
