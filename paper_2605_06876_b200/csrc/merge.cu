// Cross-view merge, cap and per-candidate case for all split candidates.
//
//   mergeable / merge_groups   ref/cross_view_merge.py:33-41, 72-107
//   merge_params               ref/cross_view_merge.py:44-69
//   cap_children + extent      ref/cross_view_merge.py:26-30, 110-116
//   _group_to_gaussian         ref/adc.py:127-140
//   case branch order          ref/adc.py:198-227
//
// Flat, skew-proof structure (one parent may own tens of thousands of
// proposals, e.g. a background Gaussian):
//   prepare   gather valid proposals in reference order (scan), case per parent
//   gates     warp per parent for P <= small_max, 64x64 tiles over the whole
//             GPU for larger parents; links by atomicMin union-find, so the
//             components (roots = smallest index) do not depend on order
//   groups    stable sort by root -> contiguous member lists in ascending
//             index order; one warp per group reduces mean, eigenbasis, reach
//   cap       stable sorts by (-extent) then parent -> rank within parent;
//             the first n_max become children in cap order
#include <math.h>

#include "merge.cuh"

#include <cooperative_groups.h>

#ifndef ADPS_MERGE_STATS
#define ADPS_MERGE_STATS 0
#endif

namespace adps {

__device__ __forceinline__ bool gate(const Proposal& A, const Proposal& B, double gd, double gc) {
  // sqrt(d^T Sa^-1 d) + sqrt(d^T Sb^-1 d) <= gamma_d and max|drgb| <= gamma_c, inclusive
  const double dc = fmax(fmax(fabs(A.rgb[0] - B.rgb[0]), fabs(A.rgb[1] - B.rgb[1])), fabs(A.rgb[2] - B.rgb[2]));
  if (!(dc <= gc)) return false;
  const double dl[3] = {B.mu[0] - A.mu[0], B.mu[1] - A.mu[1], B.mu[2] - A.mu[2]};
  // exact early reject: d >= |dl| (1/smax_a + 1/smax_b) (largest covariance eigenvalue
  // is smax^2); a 1e-9 relative guard keeps it strictly conservative
  const double n2 = dl[0] * dl[0] + dl[1] * dl[1] + dl[2] * dl[2];
  const double w = A.inv_smax + B.inv_smax;
  if (n2 * w * w > gd * gd * (1.0 + 1e-9)) return false;
  const double d = sqrt(fmax(sym_quad(A.prec, dl), 0.0)) + sqrt(fmax(sym_quad(B.prec, dl), 0.0));
  return d <= gd;
}

// group -> Gaussian: eigh(merged_cov) ascending, det fix on column 0,
// scale = sqrt(max(lambda, 1e-16)), clamped parent opacity, rgb_to_dc.
// out: 14 floats mu3 scale3 rot4 opacity sh_dc3.
__device__ void write_child(const GroupRec& G, float ocl, float* out) {
  int o[3] = {0, 1, 2};
  for (int i = 0; i < 3; ++i)
    for (int j = i + 1; j < 3; ++j)
      if (G.lam[o[j]] < G.lam[o[i]]) {
        int t = o[i];
        o[i] = o[j];
        o[j] = t;
      }
  double ev[9], lam[3];
  for (int c = 0; c < 3; ++c) {
    lam[c] = G.lam[o[c]];
    for (int r = 0; r < 3; ++r) ev[r * 3 + c] = G.evec[r * 3 + o[c]];
  }
  const double det = ev[0] * (ev[4] * ev[8] - ev[5] * ev[7]) - ev[1] * (ev[3] * ev[8] - ev[5] * ev[6]) +
                     ev[2] * (ev[3] * ev[7] - ev[4] * ev[6]);
  if (det < 0)
    for (int r = 0; r < 3; ++r) ev[r * 3 + 0] = -ev[r * 3 + 0];
  double qq[4];
  rot_to_quat(ev, qq);
  for (int t = 0; t < 3; ++t) out[t] = (float)G.mu[t];
  for (int t = 0; t < 3; ++t) out[3 + t] = (float)sqrt(fmax(lam[t], 1e-16));
  for (int t = 0; t < 4; ++t) out[6 + t] = (float)qq[t];
  out[10] = ocl;
  for (int t = 0; t < 3; ++t) out[11 + t] = (float)((G.rgb[t] - 0.5) / kShC0);
}

// ------------------------------------------------------------------ prepare
struct GatherPolicy {
  MergeArgs a;
  __device__ unsigned long long value(long long p) const { return a.valid[a.vals_sorted[p]] ? 1ull : 0ull; }
  __device__ void store(long long p, unsigned long long ex, unsigned long long v) const {
    const int rank = (int)(a.keys_sorted[p] >> a.shift_rank);
    if (p == 0 || (int)(a.keys_sorted[p - 1] >> a.shift_rank) != rank) a.pstart[rank] = (int)ex;
    if (v) {   // the 152-byte records are copied by gather_props_kernel (coalesced)
      a.psrc[ex] = a.vals_sorted[p];
      a.pcand[ex] = rank;
      a.uf[ex] = (int)ex;
    }
  }
  __device__ void total(unsigned long long t) const { a.ctr->n_proposals = t; }
};

__global__ void case_kernel(MergeArgs a) {
  pdl_wait();   // programmatic dependent launch: the previous kernel's results are visible
  const long long n_split = (long long)a.ctr->n_split;
  for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < n_split;
       k += (long long)gridDim.x * blockDim.x) {
    const int gi = a.split_list[k];
    const int P = a.cand_nvalid[k];
    a.cand_props[k] = P;
    a.n_groups[k] = 0;
    a.cand_merged[k] = 0;
    a.large_of[k] = -1;
    if (!a.dom_flag[gi]) {            // never dominant in the sampled views: vanilla fallback
      a.cand_case[k] = ADPS_CASE_FALLBACK;
      a.cand_ins[k] = 2;
      atomicAdd(&a.ctr->n_fallback, 1ull);
    } else if (P == 0) {              // dominant, no usable proposal: keep + reset
      a.cand_case[k] = ADPS_CASE_RESET;
      a.cand_ins[k] = 0;
      atomicAdd(&a.ctr->n_reset, 1ull);
    } else {
      a.cand_case[k] = ADPS_CASE_SPLIT;
      if (!owns(a, k)) {
        // another rank merges this parent
      } else if (P >= 2 && P <= a.small_max) {
        a.small_list[atomicAdd(&a.ctr->n_small, 1ull)] = (int)k;
      } else if (P > a.small_max) {
        const unsigned long long l = atomicAdd(&a.ctr->n_large, 1ull);
        a.large_list[l] = (int)k;
        a.large_of[k] = (int)l;
        const long long T = (P + kMT - 1) / kMT;
        a.work_cnt[l] = (unsigned long long)(T * (T + 1) / 2);
        a.lp_cnt[l] = (unsigned long long)P;
        a.tile_cnt[l] = (unsigned long long)T;
      }
    }
  }
}

// props_s[q] = props[psrc[q]]: thread per 8-byte word, so both the gathered
// source records and the packed destination are read/written coalesced
__global__ void gather_props_kernel(MergeArgs a) {
  pdl_wait();   // programmatic dependent launch: the previous kernel's results are visible
  constexpr int WPR = (int)(sizeof(Proposal) / 8);
  const long long nw = (long long)a.ctr->n_proposals * WPR;
  const double* src = reinterpret_cast<const double*>(a.props);
  double* dst = reinterpret_cast<double*>(a.props_s);
  for (long long w = (long long)blockIdx.x * blockDim.x + threadIdx.x; w < nw; w += (long long)gridDim.x * blockDim.x) {
    const long long q = w / WPR;
    const int c = (int)(w - q * WPR);
    dst[w] = __ldg(src + (long long)__ldg(a.psrc + q) * WPR + c);
  }
}

cudaError_t launch_merge_prepare(const MergeArgs& a, long long n_split, ScanState st, cudaStream_t s) {
  cudaError_t e = launch_scan(GatherPolicy{a}, a.n_regions, st, s);
  if (e != cudaSuccess) return e;
  launch_k(gather_props_kernel, a.grid, 256, 0, s, a);
  long long b = (n_split + 255) / 256;
  launch_k(case_kernel, (unsigned)(b < 1 ? 1 : (b > 4096 ? 4096 : b)), 256, 0, s, a);
  return cudaGetLastError();
}

// -------------------------------------------------------------------- gates
__global__ void small_pairs_kernel(MergeArgs a) {
  pdl_wait();   // programmatic dependent launch: the previous kernel's results are visible
  const int lane = threadIdx.x & 31;
  const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
  const long long n_small = (long long)a.ctr->n_small;
  for (long long t = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); t < n_small; t += warps) {
    const int k = a.small_list[t];
    const int P = a.cand_nvalid[k];
    const int ps = a.pstart[k];
    const Proposal* pr = a.props_s + ps;
    for (int i = 0; i < P - 1; ++i) {
      const Proposal& A = pr[i];
      for (int j0 = i + 1; j0 < P; j0 += 32) {   // warp-uniform trip count, predicated body
        const int j = j0 + lane;
        if (j < P && gate(A, pr[j], a.gamma_d, a.gamma_c)) uf_unite(a.uf, ps + i, ps + j);
      }
    }
  }
}

// exclusive scans of up to three count arrays (+ total at [n]), a block each
#ifndef ADPS_TILE_OWNER_FILL
#define ADPS_TILE_OWNER_FILL 1   // the tile -> parent map written with the offsets, not searched per tile
#endif
struct Offsets3 {
  const unsigned long long* in[3];
  unsigned long long* out[3];
  int* owner;   // optional: owner[t] = i for t in [out[2][i], out[2][i+1]) (the tile -> parent map)
};
__global__ void __launch_bounds__(1024) offsets_1block_kernel(Offsets3 io, const unsigned long long* __restrict__ n_dev) {
  pdl_wait();   // programmatic dependent launch: the previous kernel's results are visible
  const unsigned long long* __restrict__ in = io.in[blockIdx.x];
  unsigned long long* __restrict__ out = io.out[blockIdx.x];
  __shared__ unsigned long long warp_tot[32];
  __shared__ unsigned long long carry;
  const long long n = (long long)*n_dev;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (long long base = 0; base < n; base += blockDim.x) {
    const long long i = base + threadIdx.x;
    const unsigned long long v = i < n ? in[i] : 0ull;
    unsigned long long x = v;
    for (int o = 1; o < 32; o <<= 1) {
      unsigned long long y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) warp_tot[wid] = x;
    __syncthreads();
    if (wid == 0) {
      unsigned long long w = warp_tot[lane];
      unsigned long long wi = w;
      for (int o = 1; o < 32; o <<= 1) {
        unsigned long long y = __shfl_up_sync(0xffffffffu, wi, o);
        if (lane >= o) wi += y;
      }
      warp_tot[lane] = wi - w;
    }
    __syncthreads();
    const unsigned long long excl = carry + warp_tot[wid] + x - v;
    if (i < n) out[i] = excl;
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry = excl + v;
    __syncthreads();
  }
  if (threadIdx.x == 0) out[n] = carry;
#if ADPS_TILE_OWNER_FILL
  if (blockIdx.x == 2 && io.owner) {   // the tile -> large parent map (read by the box kernel and the filter)
    __syncthreads();                   // every offset of this block is written
    for (long long i = threadIdx.x; i < n; i += blockDim.x)
      for (unsigned long long t = out[i]; t < out[i + 1]; ++t) io.owner[t] = (int)i;
  }
#endif
}

__global__ void __launch_bounds__(1024) shard_range_kernel(const int* __restrict__ nvalid, long long n, int rank,
                                                           int world, unsigned long long* __restrict__ lohi) {
  pdl_wait();   // programmatic dependent launch: the previous kernel's results are visible
  __shared__ unsigned long long warp_tot[32];
  __shared__ unsigned long long carry, total;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  unsigned long long sum = 0;
  for (long long i = threadIdx.x; i < n; i += blockDim.x) {
    const unsigned long long p = (unsigned long long)nvalid[i];
    sum += p * p + 1;
  }
  for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  if (lane == 0) warp_tot[wid] = sum;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long t = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += warp_tot[w];
    total = t;
    carry = 0;
    lohi[0] = (unsigned long long)n;
    lohi[1] = 0;
  }
  __syncthreads();
  const unsigned long long T = total;
  for (long long base = 0; base < n; base += blockDim.x) {
    const long long i = base + threadIdx.x;
    const unsigned long long v = i < n ? (unsigned long long)nvalid[i] * (unsigned long long)nvalid[i] + 1 : 0ull;
    unsigned long long x = v;
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    __syncthreads();
    if (lane == 31) warp_tot[wid] = x;
    __syncthreads();
    if (wid == 0) {
      const unsigned long long w = warp_tot[lane];
      unsigned long long wi = w;
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long y = __shfl_up_sync(0xffffffffu, wi, o);
        if (lane >= o) wi += y;
      }
      warp_tot[lane] = wi - w;
    }
    __syncthreads();
    const unsigned long long excl = carry + warp_tot[wid] + x - v;
    if (i < n) {
      unsigned long long owner = excl * (unsigned long long)world / T;
      if (owner >= (unsigned long long)world) owner = world - 1;
      if ((int)owner == rank) {
        atomicMin(&lohi[0], (unsigned long long)i);
        atomicMax(&lohi[1], (unsigned long long)(i + 1));
      }
    }
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry = excl + v;
    __syncthreads();
  }
}

// proposal range of the rank's candidates: lohi[2..3] = sum of P_k over k < lo, k < hi
// (pstart is only defined for parents with regions)
__global__ void __launch_bounds__(1024) shard_prange_kernel(const int* __restrict__ nvalid, long long n,
                                                            unsigned long long* __restrict__ lohi) {
  pdl_wait();   // programmatic dependent launch: the previous kernel's results are visible
  __shared__ unsigned long long ws[2][32];
  const unsigned long long lo = lohi[0], hi = lohi[1];
  unsigned long long a = 0, b = 0;
  for (long long i = threadIdx.x; i < n; i += blockDim.x) {
    const unsigned long long p = (unsigned long long)nvalid[i];
    if ((unsigned long long)i < lo) a += p;
    if ((unsigned long long)i < hi) b += p;
  }
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
  }
  if ((threadIdx.x & 31) == 0) {
    ws[0][threadIdx.x >> 5] = a;
    ws[1][threadIdx.x >> 5] = b;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long sa = 0, sb = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      sa += ws[0][w];
      sb += ws[1][w];
    }
    lohi[2] = hi > lo ? sa : 0;
    lohi[3] = hi > lo ? sb : 0;
  }
}

cudaError_t launch_shard_range(const int* nvalid, long long n, int rank, int world, unsigned long long* lohi,
                               cudaStream_t s) {
  launch_k(shard_range_kernel, 1, 1024, 0, s, nvalid, n, rank, world, lohi);
  launch_k(shard_prange_kernel, 1, 1024, 0, s, nvalid, n, lohi);
  return cudaGetLastError();
}

cudaError_t launch_small_pairs(const MergeArgs& a, cudaStream_t s) {
  launch_k(small_pairs_kernel, a.grid, 256, 0, s, a);
  return cudaGetLastError();
}

cudaError_t launch_large_offsets(const MergeArgs& a, cudaStream_t s) {
  Offsets3 io;
  io.in[0] = a.work_cnt;
  io.out[0] = a.work_off;
  io.in[1] = a.lp_cnt;
  io.out[1] = a.lp_off;
  io.in[2] = a.tile_cnt;
  io.out[2] = a.tile_off;
  io.owner = a.tile_owner;
  launch_k(offsets_1block_kernel, 3, 1024, 0, s, io, &a.ctr->n_large);
  return cudaGetLastError();
}

cudaError_t launch_merge_small_gates(const MergeArgs& a, cudaStream_t s) {
  launch_k(small_pairs_kernel, a.grid, 256, 0, s, a);
  return launch_large_offsets(a, s);
}

// ---- exact spatial pruning for large parents --------------------------------
// Proposals of each large parent are put in Morton order of their centres;
// per 64-proposal tile a bounding sphere, the largest proposal sigma and the
// rgb box bound every pair: sqrt(d' Sa^-1 d) >= |d| / smax_a, so a tile pair
// whose minimum centre distance gives (dmin/sA + dmin/sB) > gamma_d, or whose
// rgb boxes are more than gamma_c apart, contains no mergeable pair.
enum { kG_mu = 0, kG_rgb = 3, kG_inv = 6, kG_prec = 7, kG_fields = 13 };   // gsoa fields

__device__ __forceinline__ unsigned spread10(unsigned v) {
  v &= 0x3ffu;
  v = (v | (v << 16)) & 0x030000FFu;
  v = (v | (v << 8)) & 0x0300F00Fu;
  v = (v | (v << 4)) & 0x030C30C3u;
  v = (v | (v << 2)) & 0x09249249u;
  return v;
}

__global__ void morton_kernel(MergeArgs a, long long cap) {
  pdl_wait();   // programmatic dependent launch: the previous kernel's results are visible
  const long long np = (long long)a.ctr->n_proposals;
  const double inv = 1.0 / (4.0 * a.extent);
  for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < cap;
       q += (long long)gridDim.x * blockDim.x) {
    unsigned long long key = ~0ull;
    if (q < np) {
      const int l = a.large_of[a.pcand[q]];
      if (l >= 0) {
        unsigned c[3];
        for (int t = 0; t < 3; ++t) {
          constexpr double kCells = (double)(1 << kMortonBits);
          const double u = (a.props_s[q].mu[t] * inv + 0.5) * kCells;
          c[t] = u <= 0.0 ? 0u : (u >= kCells - 1.0 ? (1u << kMortonBits) - 1u : (unsigned)u);
        }
        const unsigned m = spread10(c[0]) | (spread10(c[1]) << 1) | (spread10(c[2]) << 2);
        key = ((unsigned long long)l << (3 * kMortonBits)) | m;   // 3 x kMortonBits-bit Morton code
      }
    }
    a.mkey[q] = key;
    a.mval[q] = (int)q;
  }
}

cudaError_t launch_merge_morton(const MergeArgs& a, long long cap, cudaStream_t s) {
  long long b = (cap + 255) / 256;
  launch_k(morton_kernel, (unsigned)(b < 1 ? 1 : (b > 65535 ? 65535 : b)), 256, 0, s, a, cap);
  return cudaGetLastError();
}

__device__ __forceinline__ long long find_owner(const unsigned long long* off, long long n, unsigned long long w) {
  long long lo = 0, hi = n - 1;
  while (lo < hi) {
    const long long mid = (lo + hi + 1) / 2;
    if (off[mid] <= w) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

// one warp per kMT-proposal tile of a large parent (Morton order), lane = proposal:
// the gate operands into the structure of arrays, the tile's bounding data,
// and the tile's owner (read by the filter instead of a search)
static_assert(kMT == 32, "box_kernel: one proposal per lane");
__global__ void box_kernel(MergeArgs a) {
  pdl_wait();   // programmatic dependent launch: the previous kernel's results are visible
  const int lane = threadIdx.x & 31;
  const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
  const long long n_large = (long long)a.ctr->n_large;
  const unsigned long long n_tiles = n_large > 0 ? a.tile_off[n_large] : 0;
  for (long long t = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); t < (long long)n_tiles;
       t += warps) {
#if ADPS_TILE_OWNER_FILL
    const long long l = a.tile_owner[t];   // (filled with the tile offsets)
#else
    const long long l = find_owner(a.tile_off, n_large, (unsigned long long)t);
#endif
    const long long tl = t - (long long)a.tile_off[l];
    const long long b = (long long)a.lp_off[l] + tl * kMT;
    const long long e = min(b + kMT, (long long)(a.lp_off[l] + a.lp_cnt[l]));
    const long long m = b + lane;
    const bool in = m < e;
    double mu[3] = {0, 0, 0}, rgb[3] = {0, 0, 0}, inv = 1e300;
    if (in) {
      const Proposal& M = a.props_s[a.mval_sorted[m]];
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        mu[c] = M.mu[c];
        rgb[c] = M.rgb[c];
      }
      inv = M.inv_smax;
      double prec[6];
#pragma unroll
      for (int k = 0; k < 6; ++k) prec[k] = M.prec[k];
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        a.gsoa[(long long)(kG_mu + c) * a.soa_cap + m] = mu[c];
        a.gsoa[(long long)(kG_rgb + c) * a.soa_cap + m] = rgb[c];
      }
      a.gsoa[(long long)kG_inv * a.soa_cap + m] = inv;
#pragma unroll
      for (int k = 0; k < 6; ++k) a.gsoa[(long long)(kG_prec + k) * a.soa_cap + m] = prec[k];
      // fp32 (round to nearest) copies for the conservative prefilter, two float4 per proposal
      reinterpret_cast<float4*>(a.fsoa)[2 * m] = make_float4((float)mu[0], (float)mu[1], (float)mu[2], (float)inv);
      reinterpret_cast<float4*>(a.fsoa)[2 * m + 1] = make_float4((float)rgb[0], (float)rgb[1], (float)rgb[2], 0.0f);
    }
    double s[3] = {mu[0], mu[1], mu[2]}, inv_s = inv;
    double lo[3], hi[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      lo[c] = in ? rgb[c] : 1e300;
      hi[c] = in ? rgb[c] : -1e300;
    }
    for (int o = 16; o > 0; o >>= 1) {
      for (int c = 0; c < 3; ++c) {
        s[c] += __shfl_xor_sync(0xffffffffu, s[c], o);
        lo[c] = fmin(lo[c], __shfl_xor_sync(0xffffffffu, lo[c], o));
        hi[c] = fmax(hi[c], __shfl_xor_sync(0xffffffffu, hi[c], o));
      }
      inv_s = fmin(inv_s, __shfl_xor_sync(0xffffffffu, inv_s, o));
    }
    const double cnt = (double)(e - b);
    const double cen[3] = {s[0] / cnt, s[1] / cnt, s[2] / cnt};
    double r = 0.0;
    if (in) {
      const double dx = mu[0] - cen[0], dy = mu[1] - cen[1], dz = mu[2] - cen[2];
      r = sqrt(dx * dx + dy * dy + dz * dz);
    }
    for (int o = 16; o > 0; o >>= 1) r = fmax(r, __shfl_xor_sync(0xffffffffu, r, o));
    if (lane == 0) {
      TileBox B;
      for (int c = 0; c < 3; ++c) {
        B.c[c] = cen[c];
        B.lo[c] = lo[c];
        B.hi[c] = hi[c];
      }
      B.r = r * (1.0 + 1e-12) + 1e-300;   // rounding guard: the sphere really encloses
      B.inv_s = inv_s;
      a.boxes[t] = B;
      if (!ADPS_TILE_OWNER_FILL) a.tile_owner[t] = (int)l;
    }
  }
}

__device__ __forceinline__ bool boxes_may_merge(const TileBox& A, const TileBox& B, double gd, double gc) {
  for (int c = 0; c < 3; ++c)
    if (B.lo[c] - A.hi[c] > gc || A.lo[c] - B.hi[c] > gc) return false;   // colour gate fails for all pairs
  const double dx = A.c[0] - B.c[0], dy = A.c[1] - B.c[1], dz = A.c[2] - B.c[2];
  const double dmin = sqrt(dx * dx + dy * dy + dz * dz) - A.r - B.r;
  if (dmin <= 0.0) return true;
  const double lb = dmin * (A.inv_s + B.inv_s);
  return !(lb > gd * (1.0 + 1e-9));
}

// work item w -> (large parent l, tile row bi, tile column bj), row-major upper triangle
__device__ __forceinline__ void decode_tile_pair(const MergeArgs& a, long long n_large, unsigned long long w,
                                                 long long& l, long long& bi, long long& bj) {
  l = find_owner(a.work_off, n_large, w);
  const long long T = ((long long)a.lp_cnt[l] + kMT - 1) / kMT;
  const long long q = (long long)(w - a.work_off[l]);
  bi = (long long)floor(((2.0 * T + 1.0) - sqrt((2.0 * T + 1.0) * (2.0 * T + 1.0) - 8.0 * q)) / 2.0);
  if (bi < 0) bi = 0;
  while (bi > 0 && bi * T - bi * (bi - 1) / 2 > q) --bi;
  while ((bi + 1) * T - (bi + 1) * bi / 2 <= q) ++bi;
  bj = bi + (q - (bi * T - bi * (bi - 1) / 2));
}

// a surviving tile pair as the gate kernel consumes it, with no dependent
// lookups left: x = first proposal of the row tile, y = first proposal of the
// column tile (Morton-ordered operand index), z = ni | nj << 8, w = live
__device__ __forceinline__ int4 pair_entry(const MergeArgs& a, long long l, long long bi, long long bj, bool live) {
  const long long P = (long long)a.lp_cnt[l], o = (long long)a.lp_off[l];
  const int ni = (int)min((long long)kMT, P - bi * kMT), nj = (int)min((long long)kMT, P - bj * kMT);
  return make_int4((int)(o + bi * kMT), (int)(o + bj * kMT), ni | (nj << 8), live ? 1 : 0);
}

// a block per (parent, tile row bi) of the upper-triangular tile matrix, a
// warp per 32 columns: keep the pairs (bi, bj >= bi) the bounding data cannot
// exclude (one reservation per warp chunk; the gate kernel takes pairs in any
// order).  Blocks, not warps, per row: the longest rows (a parent with
// thousands of proposals) no longer serialise on one warp.
__global__ void tile_pair_filter_kernel(MergeArgs a) {
  pdl_wait();   // programmatic dependent launch: the previous kernel's results are visible
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const long long n_large = (long long)a.ctr->n_large;
  const long long rows = n_large > 0 ? (long long)a.tile_off[n_large] : 0;
  for (long long r = blockIdx.x; r < rows; r += gridDim.x) {
    const long long l = a.tile_owner[r];
    const long long tb = (long long)a.tile_off[l];
    const long long bi = r - tb;
    const long long T = (long long)a.tile_cnt[l];
    const TileBox A = a.boxes[r];
    for (long long j0 = bi + 32 * wid; j0 < T; j0 += 32 * nw) {   // warp-uniform
      const long long bj = j0 + lane;
      const bool keep = bj < T && boxes_may_merge(A, a.boxes[tb + bj], a.gamma_d, a.gamma_c);
      const unsigned m = __ballot_sync(0xffffffffu, keep);
      if (!m) continue;
      unsigned long long base = 0;
      if (lane == 0) base = atomicAdd(&a.ctr->n_tile_pairs, (unsigned long long)__popc(m));
      base = __shfl_sync(0xffffffffu, base, 0);
      if ((long long)(base + __popc(m)) > a.tile_pairs_cap) {
        if (lane == 0) atomicOr(&a.ctr->overflow, 4u);
        continue;
      }
      if (keep) a.tile_pairs[base + __popc(m & ((1u << lane) - 1u))] = pair_entry(a, l, bi, bj, true);
    }
  }
}

// Gate operands of the large parents' proposals in Morton order, structure
// of arrays (written by box_kernel): contiguous 64-proposal tiles load
// coalesced, 13 doubles per proposal instead of a gathered 152-byte record.

__device__ __forceinline__ void cp_async(void* dst, const void* src, int bytes) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  if (bytes == 16) asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src) : "memory");
  else if (bytes == 8) asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(src) : "memory");
  else asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// the exact gate of row operand A (registers) against column jj of a staged tile
__device__ __forceinline__ bool gate_col(const double* A, const double (*Js)[kMT], int jj, double gd, double gd2,
                                         double gc) {
  const double dc = fmax(fmax(fabs(A[kG_rgb + 0] - Js[kG_rgb + 0][jj]), fabs(A[kG_rgb + 1] - Js[kG_rgb + 1][jj])),
                         fabs(A[kG_rgb + 2] - Js[kG_rgb + 2][jj]));
  if (!(dc <= gc)) return false;
  const double dl[3] = {Js[kG_mu + 0][jj] - A[kG_mu + 0], Js[kG_mu + 1][jj] - A[kG_mu + 1],
                        Js[kG_mu + 2][jj] - A[kG_mu + 2]};
  const double n2 = dl[0] * dl[0] + dl[1] * dl[1] + dl[2] * dl[2];
  const double w = A[kG_inv] + Js[kG_inv][jj];
  if (n2 * w * w > gd2) return false;   // exact early reject (|d|/s_max bounds each term)
  double pb[6];
#pragma unroll
  for (int k = 0; k < 6; ++k) pb[k] = Js[kG_prec + k][jj];
  const double d = sqrt(fmax(sym_quad(A + kG_prec, dl), 0.0)) + sqrt(fmax(sym_quad(pb, dl), 0.0));
  return d <= gd;
}

struct ColTile {
  double s[kG_fields][kMT];   // [field][proposal]
  float4 f[kMT][2];           // fp32 (mu, inv_smax), (rgb, 0)
  int q[kMT];
};

// Conservative fp32 reject, exact in effect: true only when the fp64 gate
// certainly fails.  Operands are the fp64 values rounded to nearest fp32
// (relative error <= 2^-24 each); the slacks cover that and the fp32
// arithmetic, taken once per tile pair from the largest magnitudes of the
// two tiles (Ma, Mb) instead of per pair:
//   colour:   |fb - fa| > gc + 4e-7 (Ma_rgb + Mb_rgb + 1) implies |b - a| > gc;
//   distance: |d_c| >= |fb_c - fa_c| - 4e-7 (Ma_mu + Mb_mu) per component,
//             w >= (fa_inv + fb_inv)(1 - 1e-6), and |d|^2 w^2 > gd^2 (1 + 1e-9)
//             (the fp64 early reject) implies the gate fails; the fp32
//             rounding of n2 w^2 is inside the 2e-5 margin of gd2s.
// Branch-free, so the warp stays converged over the column loop.
__device__ __forceinline__ bool reject32(const float4 am, const float4 ac, const float4 bm, const float4 bc,
                                         float gcs, float smu, float gd2s) {
  const float dc = fmaxf(fmaxf(fabsf(bc.x - ac.x), fabsf(bc.y - ac.y)), fabsf(bc.z - ac.z));
  const float dx = fmaxf(fabsf(bm.x - am.x) - smu, 0.0f);
  const float dy = fmaxf(fabsf(bm.y - am.y) - smu, 0.0f);
  const float dz = fmaxf(fabsf(bm.z - am.z) - smu, 0.0f);
  const float w = am.w + bm.w;
  const float n2 = dx * dx + dy * dy + dz * dz;
  return (dc > gcs) | (n2 * (w * w) > gd2s);
}
constexpr int kPairWarps = 4;
#ifndef ADPS_PAIR_LOCAL_UF
#define ADPS_PAIR_LOCAL_UF 0
#endif
#ifndef ADPS_PAIR_CHUNK
#define ADPS_PAIR_CHUNK 1
#endif
constexpr int kPairChunk = ADPS_PAIR_CHUNK;

// stage the nj-proposal column tile starting at operand index base (lane = proposal)
__device__ __forceinline__ void stage_col(const MergeArgs& a, ColTile& B, long long base, int nj, int lane) {
  if (lane < nj) {
#pragma unroll
    for (int f = 0; f < kG_fields; ++f) cp_async(&B.s[f][lane], a.gsoa + (long long)f * a.soa_cap + base + lane, 8);
    cp_async(&B.f[lane][0], a.fsoa + 8 * (base + lane), 16);
    cp_async(&B.f[lane][1], a.fsoa + 8 * (base + lane) + 4, 16);
    cp_async(&B.q[lane], a.mval_sorted + base + lane, 4);
  }
  cp_async_commit();
}

// The surviving kMT x kMT tile pairs of the large parents' gate matrices, a
// warp per pair and contiguous chunks of pairs per warp (pairs of one tile
// row are adjacent): lane = row proposal with its gate operands in registers
// while the row lasts, the column tile staged in shared memory one pair ahead
// (cp.async), no block barriers.  If the survivor list overflowed, every tile
// pair is taken with the box test inline.
#ifndef ADPS_PAIR_ROOT_CACHE
#define ADPS_PAIR_ROOT_CACHE 1   // skip unions of columns already hanging below the row's cached root
#endif
#ifndef ADPS_PAIR_MINB
#define ADPS_PAIR_MINB 1
#endif
__global__ void __launch_bounds__(kPairWarps * 32, ADPS_PAIR_MINB) pair_tiles_kernel(MergeArgs a) {
  pdl_wait();   // programmatic dependent launch: the previous kernel's results are visible
  extern __shared__ __align__(16) unsigned char pt_smem[];
#if ADPS_PAIR_LOCAL_UF
  __shared__ int luf[kPairWarps][64];   // warp-local union-find of a tile pair
  __shared__ int lq[kPairWarps][32];    // its row proposals
#endif
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  ColTile* buf = reinterpret_cast<ColTile*>(pt_smem) + 2 * wid;
  const bool overflow = (a.ctr->overflow & 4u) != 0;
  const long long n_large = (long long)a.ctr->n_large;
  const long long nwarps = (long long)gridDim.x * kPairWarps;
  const long long gw = (long long)blockIdx.x * kPairWarps + wid;
  const double gd = a.gamma_d, gc = a.gamma_c, gd2 = gd * gd * (1.0 + 1e-9);
  const long long W = overflow ? (long long)(n_large > 0 ? a.work_off[n_large] : 0) : (long long)a.ctr->n_tile_pairs;
  // dynamic work: chunks of kPairChunk consecutive pairs (usually one tile row)
  // from a global counter, the next chunk reserved while the current one runs
  // (gate and union work is uneven across pairs: static ranges left long tails)
  (void)nwarps;
  (void)gw;
  unsigned long long* const counter = &a.ctr->pair_next;
  auto grab = [&]() -> unsigned long long {
    unsigned long long v = 0;
    if (lane == 0) v = atomicAdd(counter, (unsigned long long)kPairChunk);
    return v;   // lane 0 only; broadcast when it is consumed
  };
  // two reservations in flight: a contended counter's reply takes longer than
  // one pair's work
  long long c_end = 0, pos = 0;
  unsigned long long c_next1 = grab();
  unsigned long long c_next2 = grab();
  auto next_index = [&]() -> long long {   // -1 when exhausted
    if (pos >= c_end) {
      const long long c = (long long)__shfl_sync(0xffffffffu, c_next1, 0);
      if (c >= W) return -1;
      pos = c;
      c_end = min(W, c + kPairChunk);
      c_next1 = c_next2;
      c_next2 = grab();
    }
    return pos++;
  };
  auto pair_at = [&](long long w) -> int4 {
    if (w < 0) return make_int4(-1, -1, 0, 0);
    if (!overflow) return a.tile_pairs[w];
    long long l, bi, bj;
    decode_tile_pair(a, n_large, (unsigned long long)w, l, bi, bj);
    const long long tb = (long long)a.tile_off[l];
    const bool live = boxes_may_merge(a.boxes[tb + bi], a.boxes[tb + bj], a.gamma_d, a.gamma_c);
    return pair_entry(a, l, bi, bj, live);
  };
  long long i_cur = next_index();
  if (i_cur < 0) return;
  long long i_nxt = next_index();
  int cur_row = -1;
  double A[kG_fields];
  float4 am = make_float4(0.f, 0.f, 0.f, 0.f), ac = am;
  float ma_mu = 0.f, ma_rgb = 0.f;   // the row tile's largest |mu_c|, |rgb_c| (fp32 copies)
  int qa = -1, ni = 0;
  int ra = -1;   // a root qa was last united under (this row tile)
  const float gc32 = (float)gc, gd2s = (float)(gd * gd) * (1.0f + 1e-5f) * (1.0f + 2e-5f);
  // entries are prefetched two ahead (registers), column tiles one ahead (cp.async)
  int4 cur = pair_at(i_cur);
  int4 nxt = pair_at(i_nxt);
  stage_col(a, buf[0], cur.y, (cur.z >> 8) & 0xff, lane);
  for (int it = 0; i_cur >= 0; ++it) {
    const long long i_nn = i_nxt >= 0 ? next_index() : -1;
    const int4 nn = pair_at(i_nn);
    if (cur.x != cur_row) {   // new tile row: its operands into registers
      cur_row = cur.x;
      ra = -1;
      ni = cur.z & 0xff;
      const long long m = (long long)cur.x + lane;
      am = ac = make_float4(0.f, 0.f, 0.f, 0.f);
      if (lane < ni) {
#pragma unroll
        for (int f = 0; f < kG_fields; ++f) A[f] = __ldg(a.gsoa + (long long)f * a.soa_cap + m);
        am = __ldg(reinterpret_cast<const float4*>(a.fsoa) + 2 * m);
        ac = __ldg(reinterpret_cast<const float4*>(a.fsoa) + 2 * m + 1);
        qa = __ldg(a.mval_sorted + m);
      }
      ma_mu = fmaxf(fmaxf(fabsf(am.x), fabsf(am.y)), fabsf(am.z));
      ma_rgb = fmaxf(fmaxf(fabsf(ac.x), fabsf(ac.y)), fabsf(ac.z));
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        ma_mu = fmaxf(ma_mu, __shfl_xor_sync(0xffffffffu, ma_mu, o));
        ma_rgb = fmaxf(ma_rgb, __shfl_xor_sync(0xffffffffu, ma_rgb, o));
      }
    }
    if (i_nxt >= 0) {
      stage_col(a, buf[(it + 1) & 1], nxt.y, (nxt.z >> 8) & 0xff, lane);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncwarp();
    if (!overflow || cur.w) {
      const ColTile& J = buf[it & 1];
      const int nj = (cur.z >> 8) & 0xff;
      const bool diag = cur.x == cur.y;
      // the column tile's largest magnitudes -> this tile pair's slacks
      float mb_mu = 0.f, mb_rgb = 0.f;
      if (lane < nj) {
        const float4 bm = J.f[lane][0], bc = J.f[lane][1];
        mb_mu = fmaxf(fmaxf(fabsf(bm.x), fabsf(bm.y)), fabsf(bm.z));
        mb_rgb = fmaxf(fmaxf(fabsf(bc.x), fabsf(bc.y)), fabsf(bc.z));
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        mb_mu = fmaxf(mb_mu, __shfl_xor_sync(0xffffffffu, mb_mu, o));
        mb_rgb = fmaxf(mb_rgb, __shfl_xor_sync(0xffffffffu, mb_rgb, o));
      }
      const float smu = 4e-7f * (ma_mu + mb_mu);
      const float gcs = gc32 * (1.0f + 1e-6f) + 4e-7f * (ma_rgb + mb_rgb + 1.0f);
      // fp32 prefilter over all columns, warp-converged: bit jj = "the fp64 gate may pass"
      unsigned maybe = 0u;
#pragma unroll 4
      for (int jj = 0; jj < nj; ++jj) {
        const float4 bm = J.f[jj][0], bc = J.f[jj][1];
        maybe |= (reject32(am, ac, bm, bc, gcs, smu, gd2s) ? 0u : 1u) << jj;
      }
      // unordered pairs: ii < jj on the diagonal; rows past the tile's end have no pairs
      if (diag) maybe &= lane >= 31 ? 0u : (0xffffffffu << (lane + 1));
      if (lane >= ni) maybe = 0u;
      // gates first, unions after: a union inside the column loop would stall
      // the whole warp on one lane's union-find latency whenever any lane passes
      // (warp-uniform trip counts, predicated bodies: per-lane loops left the
      // warp split for the rest of the pair, every later instruction issued twice)
      unsigned pass = 0u;
      while (__any_sync(0xffffffffu, maybe != 0u)) {
        if (maybe) {
          const int jj = __ffs(maybe) - 1;
          const bool ok = gate_col(A, J.s, jj, gd, gd2, gc);
#if ADPS_MERGE_STATS
          atomicAdd(&a.ctr->stat_gates, 1ull);
          if (ok) atomicAdd(&a.ctr->stat_pass, 1ull);
#endif
          if (ok) pass |= 1u << jj;
          maybe &= maybe - 1u;
        }
      }
#if ADPS_PAIR_LOCAL_UF
      // the tile pair's links first in a warp-local union-find over its 64
      // nodes (rows 0..31, columns 32..63) in shared memory, then one global
      // union per node whose local root differs: a dense tile pair costs at
      // most 63 global unions instead of one per passing pair
      if (__any_sync(0xffffffffu, pass != 0u)) {
        int* L = luf[wid];
        L[lane] = lane;
        L[32 + lane] = 32 + lane;
        lq[wid][lane] = qa;
        __syncwarp();
        for (unsigned p = pass; p; p &= p - 1u) uf_unite(L, lane, 32 + __ffs(p) - 1);
        __syncwarp();
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int nd = lane + 32 * h;
          const int r = uf_find(L, nd);
          if (r != nd) uf_unite(a.uf, h ? J.q[lane] : qa, r < 32 ? lq[wid][r] : J.q[r - 32]);
        }
        __syncwarp();
      }
#else
      // a column already hanging directly below the root this row proposal was
      // last united under is in its tree: one load instead of two finds
      while (__any_sync(0xffffffffu, pass != 0u)) {
        if (pass) {
          const int qb = J.q[__ffs(pass) - 1];
          if (!(ADPS_PAIR_ROOT_CACHE && ra >= 0 && reinterpret_cast<volatile int*>(a.uf)[qb] == ra))
            ra = uf_unite_root(a.uf, qa, qb);
          pass &= pass - 1u;
        }
      }
#endif
    }
    __syncwarp();   // this buffer is restaged two pairs on
    cur = nxt;
    nxt = nn;
    i_cur = i_nxt;
    i_nxt = i_nn;
  }
}

cudaError_t launch_merge_tile_gates(const MergeArgs& a, cudaStream_t s) {
  launch_k(box_kernel, a.grid, 256, 0, s, a);
  launch_k(tile_pair_filter_kernel, a.grid, 128, 0, s, a);   // block per tile row
  const int smem = (int)(sizeof(ColTile) * 2 * kPairWarps);
  cudaError_t e = cudaFuncSetAttribute(pair_tiles_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  // one wave of resident blocks: each warp takes one contiguous chunk of pairs
  static int resident = 0;
  if (resident == 0) {
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&resident, pair_tiles_kernel, kPairWarps * 32, smem);
    if (e != cudaSuccess || resident < 1) resident = 4;
  }
#ifdef ADPS_PAIR_BLOCKS_PER_SM
  resident = ADPS_PAIR_BLOCKS_PER_SM;
#endif
  const unsigned blocks = (unsigned)(a.grid / 8) * (unsigned)resident;   // a.grid = 8 x SM count
  launch_k(pair_tiles_kernel, blocks, kPairWarps * 32, smem, s, a);
  return cudaGetLastError();
}

// ----------------------------------------------------------------- flatten
__global__ void flatten_kernel(MergeArgs a, long long cap) {
  pdl_wait();   // programmatic dependent launch: the previous kernel's results are visible
  const long long np = (long long)a.ctr->n_proposals;
  for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < cap;
       q += (long long)gridDim.x * blockDim.x) {
    const bool mine = q < np && owns(a, a.pcand[q]);
    a.gkey[q] = mine ? (unsigned)uf_find_halve(a.uf, (int)q) : 0xffffffffu;
    if (a.own && mine) atomicAdd(&a.ctr->n_owned_props, 1ull);
    a.gval[q] = (int)q;
  }
}

cudaError_t launch_merge_flatten(const MergeArgs& a, long long cap, cudaStream_t s) {
  long long b = (cap + 255) / 256;
  launch_k(flatten_kernel, (unsigned)(b < 1 ? 1 : (b > 65535 ? 65535 : b)), 256, 0, s, a, cap);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ groups
#ifndef ADPS_SMALL_GROUP
#define ADPS_SMALL_GROUP 8
#endif
constexpr int kSmallGroup = ADPS_SMALL_GROUP;   // groups up to this size: a thread each
constexpr int kBlockGroup = 512;   // larger groups: a block per group

struct GroupStartPolicy {
  MergeArgs a;
  __device__ unsigned long long value(long long s) const {
    const unsigned k = a.gkey_sorted[s];
    return (k != 0xffffffffu && (s == 0 || a.gkey_sorted[s - 1] != k)) ? 1ull : 0ull;
  }
  __device__ void store(long long s, unsigned long long ex, unsigned long long v) const {
    if (!v) return;
    a.grp_first[ex] = (int)s;
    // work lists of the warp / block reductions: members are sorted by root, so
    // a group has more than m members iff entry s + m still carries its root
    const unsigned k = a.gkey_sorted[s];
    const long long n = a.own ? (long long)a.ctr->n_owned_props : (long long)a.ctr->n_proposals;
    if (s + kSmallGroup < n && a.gkey_sorted[s + kSmallGroup] == k) {
      if (s + kBlockGroup < n && a.gkey_sorted[s + kBlockGroup] == k)
        a.glist[a.glist_cap + atomicAdd(&a.ctr->n_huge_groups, 1ull)] = (int)ex;
      else
        a.glist[atomicAdd(&a.ctr->n_mid_groups, 1ull)] = (int)ex;
    }
  }
  __device__ void total(unsigned long long t) const {
    a.ctr->n_groups_all = t;
    // end of the last group's members: the non-padding entries (all proposals, or
    // under parent sharding only this rank's)
    a.grp_first[t] = (int)(a.own ? a.ctr->n_owned_props : a.ctr->n_proposals);
  }
};


// groups of up to kSmallGroup members: one thread per group, members summed in
// ascending index order; every group's first-of-candidate mark
#ifndef ADPS_GROUP_MINB
#define ADPS_GROUP_MINB 6
#endif
constexpr int kGroupThreads = 128;
constexpr int kGroupWords = (int)(sizeof(GroupRec) / 8);
static_assert(sizeof(GroupRec) == 8 * kGroupWords && (kGroupWords & 1), "GroupRec: whole doubles, odd count");
__global__ void __launch_bounds__(kGroupThreads, ADPS_GROUP_MINB) group_small_kernel(MergeArgs a, long long cap) {
  pdl_wait();   // programmatic dependent launch: the previous kernel's results are visible
  const long long G = (long long)a.ctr->n_groups_all;
  // the group's record into R (a shared-memory row, stored by the block after);
  // false for the groups the warp / block reductions own
  auto body = [&](long long g, GroupRec& R) -> bool {
    const int b = a.grp_first[g], e = a.grp_first[g + 1];
    const int cnt = e - b;
    {   // groups of a candidate are contiguous: mark the first one
      const int k = a.pcand[a.gkey_sorted[b]];
      if (g == 0 || a.pcand[a.gkey_sorted[a.grp_first[g - 1]]] != k) a.gfirst_of[k] = (int)g;
    }
    if (cnt > kSmallGroup) return false;   // the warp / block reductions (lists built by the scan)
    double acc[12] = {0};
    // members in ascending order, a fixed trip count with predicated bodies so
    // the member indices load together
    int mi[kSmallGroup];
#pragma unroll
    for (int u = 0; u < kSmallGroup; ++u) mi[u] = b + u < e ? a.gval_sorted[b + u] : 0;
#pragma unroll
    for (int u = 0; u < kSmallGroup; ++u) {
      if (b + u < e) {
        const Proposal& M = a.props_s[mi[u]];
        for (int t = 0; t < 3; ++t) {
          acc[t] += M.mu[t];
          acc[3 + t] += M.rgb[t];
        }
        for (int t = 0; t < 6; ++t) acc[6 + t] += M.cov[t];
      }
    }
    for (int t = 0; t < 3; ++t) {
      R.mu[t] = acc[t] / cnt;
      R.rgb[t] = acc[3 + t] / cnt;
    }
    double mcov[6];
    for (int t = 0; t < 6; ++t) mcov[t] = acc[6 + t] / cnt;
    double lam0[3];
    sym_eig3(mcov, lam0, R.evec);
    double ext = 0.0;
    for (int r = 0; r < 3; ++r) {
      const double ev[3] = {R.evec[r], R.evec[3 + r], R.evec[6 + r]};
      double best = 0.0;
#pragma unroll
      for (int u = 0; u < kSmallGroup; ++u) {
        if (b + u < e) {
          const Proposal& M = a.props_s[mi[u]];
          const double off = fabs((M.mu[0] - R.mu[0]) * ev[0] + (M.mu[1] - R.mu[1]) * ev[1] +
                                  (M.mu[2] - R.mu[2]) * ev[2]);
          best = fmax(best, off + sqrt(sym_quad(M.cov, ev)));
        }
      }
      R.lam[r] = best * best;
      ext = fmax(ext, R.lam[r]);
    }
    R.extent = ext;
    const int k = a.pcand[a.gkey_sorted[b]];
    a.gpar[g] = k;
    a.gext[g] = ext;
    atomicAdd(&a.n_groups[k], 1);
    return true;
  };
  // records staged in shared memory and stored per block (a thread's 152-byte
  // record stored directly is 19 strided stores); only this kernel's rows
  __shared__ double sr[kGroupThreads * kGroupWords];   // odd row stride: no bank conflicts
  __shared__ unsigned mine[kGroupThreads / 32];
  for (long long base = (long long)blockIdx.x * kGroupThreads; base < cap; base += (long long)gridDim.x * kGroupThreads) {
    const long long g = base + threadIdx.x;
    const bool w = g < G && body(g, *reinterpret_cast<GroupRec*>(sr + threadIdx.x * kGroupWords));
    const unsigned m = __ballot_sync(0xffffffffu, w);
    if ((threadIdx.x & 31) == 0) mine[threadIdx.x >> 5] = m;
    __syncthreads();
    const long long rows = G - base < kGroupThreads ? G - base : kGroupThreads;
    double* dst = reinterpret_cast<double*>(a.groups + base);
    for (int i = threadIdx.x; i < rows * kGroupWords; i += kGroupThreads) {
      const int r = i / kGroupWords;
      if ((mine[r >> 5] >> (r & 31)) & 1u) dst[i] = sr[i];
    }
    __syncthreads();
  }
}

// larger groups: one warp per group, lane-strided sums + butterfly
__global__ void __launch_bounds__(256, (ADPS_GROUP_MINB + 1) / 2) group_kernel(MergeArgs a, long long cap) {
  pdl_wait();   // programmatic dependent launch: the previous kernel's results are visible
  const int lane = threadIdx.x & 31;
  const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
  const long long nl = (long long)a.ctr->n_mid_groups;
  for (long long i = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); i < nl; i += warps) {
    const long long g = a.glist[i];
    const int b = a.grp_first[g], e = a.grp_first[g + 1];
    const int cnt = e - b;
    double acc[12] = {0};
    for (int m0 = b; m0 < e; m0 += 32) {   // warp-uniform trip count, predicated body
      const int m = m0 + lane;
      if (m >= e) continue;
      const Proposal& M = a.props_s[a.gval_sorted[m]];
      for (int t = 0; t < 3; ++t) {
        acc[t] += M.mu[t];
        acc[3 + t] += M.rgb[t];
      }
      for (int t = 0; t < 6; ++t) acc[6 + t] += M.cov[t];
    }
    // butterfly: every lane ends with the identical (commutative) sums
    for (int t = 0; t < 12; ++t)
      for (int o = 16; o > 0; o >>= 1) acc[t] += __shfl_xor_sync(0xffffffffu, acc[t], o);
    GroupRec R;
    for (int t = 0; t < 3; ++t) {
      R.mu[t] = acc[t] / cnt;
      R.rgb[t] = acc[3 + t] / cnt;
    }
    double mcov[6];
    for (int t = 0; t < 6; ++t) mcov[t] = acc[6 + t] / cnt;
    double lam0[3];
    sym_eig3(mcov, lam0, R.evec);
    double ext = 0.0;
    for (int r = 0; r < 3; ++r) {
      const double ev[3] = {R.evec[r], R.evec[3 + r], R.evec[6 + r]};
      double best = 0.0;
      for (int m0 = b; m0 < e; m0 += 32) {
        const int m = m0 + lane;
        if (m >= e) continue;
        const Proposal& M = a.props_s[a.gval_sorted[m]];
        const double off = fabs((M.mu[0] - R.mu[0]) * ev[0] + (M.mu[1] - R.mu[1]) * ev[1] +
                                (M.mu[2] - R.mu[2]) * ev[2]);
        best = fmax(best, off + sqrt(sym_quad(M.cov, ev)));
      }
      for (int o = 16; o > 0; o >>= 1) best = fmax(best, __shfl_xor_sync(0xffffffffu, best, o));
      R.lam[r] = best * best;
      ext = fmax(ext, R.lam[r]);
    }
    R.extent = ext;
    if (lane == 0) {
      a.groups[g] = R;
      const int k = a.pcand[a.gkey_sorted[b]];
      a.gpar[g] = k;
      a.gext[g] = ext;
      atomicAdd(&a.n_groups[k], 1);
    }
  }
}


// the largest groups (a background Gaussian's proposals): a block per group,
// thread-strided sums, fixed-order warp + block trees (deterministic)
__global__ void __launch_bounds__(256) group_block_kernel(MergeArgs a, long long cap) {
  pdl_wait();   // programmatic dependent launch: the previous kernel's results are visible
  __shared__ double red[8][12];
  __shared__ double bc[12];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const long long nl = (long long)a.ctr->n_huge_groups;
  for (long long i = blockIdx.x; i < nl; i += gridDim.x) {
    const long long g = a.glist[cap + i];
    const int b = a.grp_first[g], e = a.grp_first[g + 1];
    const int cnt = e - b;
    double acc[12] = {0};
    for (int m = b + threadIdx.x; m < e; m += 256) {
      const Proposal& M = a.props_s[a.gval_sorted[m]];
      for (int t = 0; t < 3; ++t) {
        acc[t] += M.mu[t];
        acc[3 + t] += M.rgb[t];
      }
      for (int t = 0; t < 6; ++t) acc[6 + t] += M.cov[t];
    }
    for (int t = 0; t < 12; ++t)
      for (int o = 16; o > 0; o >>= 1) acc[t] += __shfl_xor_sync(0xffffffffu, acc[t], o);
    if (lane == 0)
      for (int t = 0; t < 12; ++t) red[wid][t] = acc[t];
    __syncthreads();
    if (threadIdx.x < 12) {
      double v = 0.0;
      for (int w = 0; w < 8; ++w) v += red[w][threadIdx.x];
      bc[threadIdx.x] = v;
    }
    __syncthreads();
    GroupRec R;
    for (int t = 0; t < 3; ++t) {
      R.mu[t] = bc[t] / cnt;
      R.rgb[t] = bc[3 + t] / cnt;
    }
    double mcov[6];
    for (int t = 0; t < 6; ++t) mcov[t] = bc[6 + t] / cnt;
    double lam0[3];
    sym_eig3(mcov, lam0, R.evec);
    double ext = 0.0;
    for (int r = 0; r < 3; ++r) {
      const double ev[3] = {R.evec[r], R.evec[3 + r], R.evec[6 + r]};
      double best = 0.0;
      for (int m = b + threadIdx.x; m < e; m += 256) {
        const Proposal& M = a.props_s[a.gval_sorted[m]];
        const double off = fabs((M.mu[0] - R.mu[0]) * ev[0] + (M.mu[1] - R.mu[1]) * ev[1] +
                                (M.mu[2] - R.mu[2]) * ev[2]);
        best = fmax(best, off + sqrt(sym_quad(M.cov, ev)));
      }
      for (int o = 16; o > 0; o >>= 1) best = fmax(best, __shfl_xor_sync(0xffffffffu, best, o));
      __syncthreads();
      if (lane == 0) red[wid][0] = best;
      __syncthreads();
      best = 0.0;
      for (int w = 0; w < 8; ++w) best = fmax(best, red[w][0]);
      R.lam[r] = best * best;
      ext = fmax(ext, R.lam[r]);
    }
    if (threadIdx.x == 0) {
      R.extent = ext;
      a.groups[g] = R;
      const int k = a.pcand[a.gkey_sorted[b]];
      a.gpar[g] = k;
      a.gext[g] = ext;
      atomicAdd(&a.n_groups[k], 1);
    }
    __syncthreads();
  }
}

cudaError_t launch_merge_groups(const MergeArgs& a, long long cap, ScanState st, cudaStream_t s, cudaStream_t aux,
                                cudaEvent_t fork, cudaEvent_t join) {
  MergeArgs b_ = a;
  b_.glist_cap = cap;
  cudaError_t e = launch_scan(GroupStartPolicy{b_}, cap, st, s);
  if (e != cudaSuccess) return e;
  // the warp / block reductions (lists from the scan) on the second stream,
  // concurrently with the thread-per-group pass; joined before returning
  const cudaStream_t s2 = aux ? aux : s;
  if (aux) {
    if ((e = cudaEventRecord(fork, s)) != cudaSuccess) return e;
    if ((e = cudaStreamWaitEvent(aux, fork, 0)) != cudaSuccess) return e;
  }
  launch_k(group_kernel, a.grid, 256, 0, s2, a, cap);
  launch_k(group_block_kernel, a.grid, 256, 0, s2, a, cap);
  long long b = (cap + 127) / 128;
  launch_k(group_small_kernel, (unsigned)(b < 1 ? 1 : (b > 65535 ? 65535 : b)), 128, 0, s, a, cap);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  if (aux) {
    if ((e = cudaEventRecord(join, aux)) != cudaSuccess) return e;
    if ((e = cudaStreamWaitEvent(s, join, 0)) != cudaSuccess) return e;
  }
  return cudaSuccess;
}

// --------------------------------------------------------------------- cap
// cap_children (ref/cross_view_merge.py:110-116): a stable sort of a parent's
// groups by -extent keeps the first min(n_max, #groups).  The groups of a
// parent are contiguous in g (roots ascend with the proposal index, which is
// in parent order) and in the reference's group order, so a group's rank is
// the number of its parent's groups with a larger extent, or an equal extent
// and a smaller g -- no sort needed.  Parents with few groups: a thread per
// group; many groups: a warp per group counting 32 at a time (early exit at
// n_max).

constexpr int kCapThreadMax = 64;
constexpr int kSelMax = 1024;   // n_max up to this: block top-n_max selection per parent
constexpr int kSelSmemKeys = 49152;   // high 32 bits of the extent bits, 4 B each

__device__ __forceinline__ void cap_write(const MergeArgs& a, long long g, int k, int Gk, int rank) {
  const int gi = a.split_list[k];
  const float ocl = (float)fmin(fmax((double)a.opacity[gi], 1e-6), 1.0 - 1e-6);
  write_child(a.groups[g], ocl, a.children + 14ll * (a.pstart[k] + rank));
  if (rank == 0) {
    const int ni = Gk < a.n_max ? Gk : a.n_max;
    a.cand_merged[k] = ni;
    a.cand_ins[k] = ni + 1;
    atomicAdd(&a.ctr->merge_edges, (unsigned long long)(a.cand_nvalid[k] - Gk));
    atomicAdd(&a.ctr->n_children, (unsigned long long)ni);
  }
}

__global__ void cap_small_kernel(MergeArgs a, long long cap) {
  pdl_wait();   // programmatic dependent launch: the previous kernel's results are visible
  const long long G = (long long)a.ctr->n_groups_all;
  for (long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x; g < G;
       g += (long long)gridDim.x * blockDim.x) {
    const int k = a.gpar[g];
    const int Gk = a.n_groups[k];
    if (Gk > kCapThreadMax) {
      if (a.n_max <= kSelMax) {   // one entry per parent for the block selection
        // (parents with > sel_huge groups are found by the huge-parent kernel itself)
        if (g == a.gfirst_of[k] && Gk <= a.sel_huge) a.glist[2 * cap + atomicAdd(&a.ctr->n_cap_large, 1ull)] = k;
      } else {                    // one entry per group for the block-per-group ranks
        a.glist[2 * cap + atomicAdd(&a.ctr->n_cap_large, 1ull)] = (int)g;
      }
      continue;
    }
    const long long f = a.gfirst_of[k];
    const double e = a.gext[g];
    int rank = 0;
    // 8 extents per round, loaded together (one latency per round instead of
    // one per group); a rank below n_max is exact, larger ones are not written
    for (long long h0 = f; h0 < f + Gk && rank < a.n_max; h0 += 8) {
      double eh[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) eh[u] = h0 + u < f + Gk ? a.gext[h0 + u] : -1.0;   // extents are >= 0
#pragma unroll
      for (int u = 0; u < 8; ++u) rank += (eh[u] > e) || (eh[u] == e && h0 + u < g);
    }
    if (rank < a.n_max) cap_write(a, g, k, Gk, rank);
  }
}

__global__ void __launch_bounds__(256) cap_large_kernel(MergeArgs a, long long cap) {
  pdl_wait();   // programmatic dependent launch: the previous kernel's results are visible
  // a block per group of a parent with many groups: 1024 extents per round
  __shared__ int part[8];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const long long nl = (long long)a.ctr->n_cap_large;
  for (long long i = blockIdx.x; i < nl; i += gridDim.x) {
    const long long g = a.glist[2 * cap + i];
    const int k = a.gpar[g];
    const int Gk = a.n_groups[k];
    const long long f = a.gfirst_of[k];
    const double e = a.gext[g];
    int rank = 0;
    constexpr int U = 4;
    for (long long h0 = f; h0 < f + Gk && rank < a.n_max; h0 += 256 * U) {
      double eh[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const long long h = h0 + 256 * u + threadIdx.x;
        eh[u] = h < f + Gk ? __ldg(a.gext + h) : -1.0;
      }
      int c = 0;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const long long h = h0 + 256 * u + threadIdx.x;
        c += (eh[u] > e) || (eh[u] == e && h < g);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
      if (lane == 0) part[wid] = c;
      __syncthreads();
      int t = 0;
#pragma unroll
      for (int w = 0; w < 8; ++w) t += part[w];
      rank += t;
      __syncthreads();
    }
    if (threadIdx.x == 0 && rank < a.n_max) cap_write(a, g, k, Gk, rank);
  }
}


// a block per parent with many groups (n_max <= kSelMax): radix-select the
// n_max-th largest extent over the parent's groups (8-bit digits of the
// extent's bit pattern, which orders non-negative doubles; stops as soon as
// the selected digit bin holds exactly the groups still needed), collect the
// kept groups (ties at the threshold in group order), rank them among
// themselves by (-extent, group order) and write their children.
template <bool HUGE>
__global__ void __launch_bounds__(HUGE ? 1024 : 256) cap_select_kernel(MergeArgs a, long long cap) {
  pdl_wait();   // programmatic dependent launch: the previous kernel's results are visible
  constexpr int NT = HUGE ? 1024 : 256;   // threads
  constexpr int NW = NT / 32;
  constexpr int J = 8;            // consecutive groups per thread per round
  extern __shared__ __align__(16) unsigned skeys_hi[];
  constexpr int RND = NT * J;    // groups per round
  __shared__ unsigned hist[256];
  __shared__ unsigned long long s_prefix, s_mask;
  __shared__ int s_need, s_done, s_nkeep, s_tie_base;
  __shared__ int keep_g[kSelMax];
  __shared__ int wtot[NW];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  // the parents: from cap_small_kernel's list, or (HUGE, on the second stream,
  // independent of cap_small_kernel) every candidate with > sel_huge groups
  __shared__ int huge_k[NT];
  __shared__ int n_huge;
  const long long n_split = (long long)a.ctr->n_split;
  const long long nl = HUGE ? (n_split + NT - 1) / NT : (long long)a.ctr->n_cap_large;
  for (long long i = blockIdx.x; i < nl; i += gridDim.x) {
    int n_here = 1;
    if (HUGE) {
      __syncthreads();   // every thread has read the previous n_huge
      if (tid == 0) n_huge = 0;
      __syncthreads();
      const long long kk = i * NT + tid;
      if (kk < n_split && a.n_groups[kk] > a.sel_huge) huge_k[atomicAdd(&n_huge, 1)] = (int)kk;
      __syncthreads();
      n_here = n_huge;
    }
    for (int hi_ = 0; hi_ < n_here; ++hi_) {
    const int k = HUGE ? huge_k[hi_] : a.glist[2 * cap + i];
    const int Gk = a.n_groups[k];
    const long long f0 = a.gfirst_of[k];
    // the keys: global (index f0 + h); for a huge parent the high 32 bits are
    // staged in shared memory and the low bits read only when the high bits
    // tie with the selected prefix
    const unsigned long long* key = reinterpret_cast<const unsigned long long*>(a.gext) + f0;
    const bool staged = HUGE && Gk <= kSelSmemKeys;
    if (staged) {
      for (int h = tid; h < Gk; h += NT) skeys_hi[h] = (unsigned)(__ldg(key + h) >> 32);
      __syncthreads();
    }
    const long long f = 0, fe = Gk;
    // key of group h as far as the mask `m` (selected digits) can see it
    auto key_at = [&](long long h, unsigned long long m, unsigned long long p) -> unsigned long long {
      if (!staged) return __ldg(key + h);
      const unsigned hi = skeys_hi[h];
      unsigned long long kv = (unsigned long long)hi << 32;
      if ((m & 0xffffffffull) && (hi & (unsigned)(m >> 32)) == (unsigned)(p >> 32)) kv = __ldg(key + h);
      return kv;
    };
    if (tid == 0) {
      s_prefix = 0ull;
      s_mask = 0ull;
      s_need = a.n_max < Gk ? a.n_max : Gk;
      s_done = Gk <= a.n_max;   // every group is kept
      s_nkeep = 0;
      s_tie_base = 0;
    }
    __syncthreads();
    for (int shift = 56; shift >= 0 && !s_done; shift -= 8) {
      if (tid < 256) hist[tid] = 0u;
      __syncthreads();
      const unsigned long long pre = s_prefix, msk = s_mask;
      for (long long h0 = f; h0 < fe; h0 += RND) {   // block-uniform trip count
        unsigned long long kv[J];
#pragma unroll
        for (int j = 0; j < J; ++j) {
          const long long h = h0 + (long long)j * NT + tid;
          kv[j] = h < fe ? key_at(h, msk | (255ull << shift), pre) : 0ull;
        }
#pragma unroll
        for (int j = 0; j < J; ++j) {
          const long long h = h0 + (long long)j * NT + tid;
          const bool hit = h < fe && (kv[j] & msk) == pre;
          // extents cluster in few bins: one shared atomic per distinct bin per warp
          const unsigned bin = hit ? (unsigned)((kv[j] >> shift) & 255u) : 256u;
          const unsigned peers = __match_any_sync(0xffffffffu, bin);
          if (hit && lane == __ffs(peers) - 1) atomicAdd(&hist[bin], (unsigned)__popc(peers));
        }
      }
      __syncthreads();
      if (wid == 0) {
        // the bin holding the need-th largest key, scanning from bin 255 down
        // (bin 0 takes whatever is left): lane L holds bins 255 - 8L - j,
        // a warp prefix over the lanes, then the owning lane walks its 8 bins
        int hv[8], c = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) c += (hv[j] = (int)hist[255 - 8 * lane - j]);
        int x = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int t = __shfl_up_sync(0xffffffffu, x, o);
          if (lane >= o) x += t;
        }
        const int need0 = s_need, before = x - c;
        const unsigned own = __ballot_sync(0xffffffffu, before < need0 && need0 <= x);
        if (lane == (own ? __ffs(own) - 1 : 31)) {
          int need = need0 - before, b = 255 - 8 * lane, hb = hv[0];
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            b = 255 - 8 * lane - j;
            hb = hv[j];
            if (b == 0 || hb >= need) break;
            need -= hb;
          }
          s_need = need;   // still needed from bin b
          s_prefix = pre | ((unsigned long long)b << shift);
          s_mask = msk | (255ull << shift);
          if (hb == need || shift == 0) s_done = 1;
        }
      }
      __syncthreads();
    }
    // kept: keys above the selected prefix range, and from inside it the first
    // s_need in group order (all of it when the bin held exactly s_need)
    const bool all = Gk <= a.n_max;
    const unsigned long long pre = s_prefix, msk = s_mask;
    const int need = s_need;
    for (long long h0 = f; h0 < fe; h0 += RND) {
      // thread tid owns groups [h0 + tid*J, +J): group order = (tid, j)
      const long long hb = h0 + (long long)tid * J;
      unsigned long long kv[J];
#pragma unroll
      for (int j = 0; j < J; ++j) kv[j] = hb + j < fe ? key_at(hb + j, msk, pre) : 0ull;
      unsigned above = 0u, in = 0u;
#pragma unroll
      for (int j = 0; j < J; ++j) {
        if (hb + j < fe) {
          if (all || (kv[j] & msk) > pre) above |= 1u << j;
          else if ((kv[j] & msk) == pre) in |= 1u << j;
        }
      }
      // exclusive prefix of the in-range counts over threads (group order)
      const int cnt = __popc(in);
      int x = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += t;
      }
      if (lane == 31) wtot[wid] = x;
      __syncthreads();
      int before = x - cnt, tot = 0;
      for (int w = 0; w < NW; ++w) {
        if (w < wid) before += wtot[w];
        tot += wtot[w];
      }
      int tr = s_tie_base + before;
      for (int j = 0; j < J; ++j) {
        const bool is_in = (in >> j) & 1u;
        if (((above >> j) & 1u) || (is_in && tr < need)) keep_g[atomicAdd(&s_nkeep, 1)] = (int)(f0 + hb + j);
        tr += is_in;
      }
      __syncthreads();
      if (tid == 0) s_tie_base += tot;
      __syncthreads();
    }
    // rank among the kept by (-extent, group order) and write
    const int nk = s_nkeep;
    for (int q = tid; q < nk; q += NT) {
      const long long g = keep_g[q];
      const double e = a.gext[g];
      int rank = 0;
      for (int j = 0; j < nk; ++j) {
        const long long h = keep_g[j];
        const double eh = a.gext[h];
        rank += (eh > e) || (eh == e && h < g);
      }
      cap_write(a, g, k, Gk, rank);
    }
    __syncthreads();
    }
  }
}

// The parents with > sel_huge groups (a background Gaussian's thousands of
// groups): the same radix selection as cap_select_kernel<true>, by a cluster
// of kCapCS blocks.  Each block holds a contiguous 1/kCapCS of the parent's
// groups (their extents' high words staged in its shared memory) and counts
// its digit histogram; the counts are added into the leading block's
// histogram through distributed shared memory, the leader selects the bin,
// and every block reads the selection back -- two cluster barriers per digit
// instead of one block passing over all groups.  Ties at the threshold are
// kept in group order across the blocks (each block's tie base = the tie
// counts of the blocks before it); the leader ranks and writes the kept.
#ifndef ADPS_CAP_CLUSTER
#define ADPS_CAP_CLUSTER 1
#endif
constexpr int kCapCS = 8;                // blocks per cluster (portable maximum)
constexpr int kCapCT = 1024;             // threads per block
constexpr int kCapStage = 6144;          // staged keys per block (Gk <= 49152 staged)
namespace cg = cooperative_groups;
__global__ void __cluster_dims__(kCapCS, 1, 1) __launch_bounds__(kCapCT) cap_huge_cluster_kernel(MergeArgs a) {
  pdl_wait();   // programmatic dependent launch: the previous kernel's results are visible
  constexpr int NT = kCapCT, NW = NT / 32, J = 8, RND = NT * J;
  cg::cluster_group cl = cg::this_cluster();
  const int crank = (int)cl.block_rank();
  __shared__ unsigned skeys_hi[kCapStage];
  __shared__ unsigned hist[256];
  // leader-owned state (read and updated by the other blocks through DSMEM)
  __shared__ unsigned ghist[256];
  __shared__ unsigned long long s_prefix, s_mask;
  __shared__ int s_need, s_done, s_nkeep;
  __shared__ int tie_cnt[kCapCS];
  __shared__ int keep_g[kSelMax];
  // block-local
  __shared__ int huge_k[NT];
  __shared__ int wtot[NW];
  __shared__ int s_tie_base;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  unsigned* const L_ghist = cl.map_shared_rank(ghist, 0);
  unsigned long long* const L_prefix = cl.map_shared_rank(&s_prefix, 0);
  unsigned long long* const L_mask = cl.map_shared_rank(&s_mask, 0);
  int* const L_need = cl.map_shared_rank(&s_need, 0);
  int* const L_done = cl.map_shared_rank(&s_done, 0);
  int* const L_nkeep = cl.map_shared_rank(&s_nkeep, 0);
  int* const L_tie = cl.map_shared_rank(tie_cnt, 0);
  int* const L_keep = cl.map_shared_rank(keep_g, 0);
  const long long n_split = (long long)a.ctr->n_split;
  const long long nl = (n_split + NT - 1) / NT;
  const long long cid = blockIdx.x / kCapCS, ncl = gridDim.x / kCapCS;
  for (long long i = cid; i < nl; i += ncl) {   // cluster-uniform
    // this range's huge parents in index order (the same list in every block)
    const long long kk = i * NT + tid;
    const bool hp = kk < n_split && a.n_groups[kk] > a.sel_huge;
    const unsigned bm = __ballot_sync(0xffffffffu, hp);
    if (lane == 0) wtot[wid] = __popc(bm);
    __syncthreads();
    int base = 0, n_here = 0;
    for (int w = 0; w < NW; ++w) {
      if (w < wid) base += wtot[w];
      n_here += wtot[w];
    }
    if (hp) huge_k[base + __popc(bm & ((1u << lane) - 1u))] = (int)kk;
    __syncthreads();
    for (int hi_ = 0; hi_ < n_here; ++hi_) {
      const int k = huge_k[hi_];
      const int Gk = a.n_groups[k];
      const long long f0 = a.gfirst_of[k];
      const unsigned long long* key = reinterpret_cast<const unsigned long long*>(a.gext) + f0;
      const long long per = ((long long)Gk + kCapCS - 1) / kCapCS;
      const long long lo = min((long long)Gk, per * crank), hi = min((long long)Gk, lo + per);
      const bool staged = per <= kCapStage;
      if (staged)
        for (long long h = lo + tid; h < hi; h += NT) skeys_hi[h - lo] = (unsigned)(__ldg(key + h) >> 32);
      auto key_at = [&](long long h, unsigned long long m, unsigned long long p) -> unsigned long long {
        if (!staged) return __ldg(key + h);
        const unsigned hw = skeys_hi[h - lo];
        unsigned long long kv = (unsigned long long)hw << 32;
        if ((m & 0xffffffffull) && (hw & (unsigned)(m >> 32)) == (unsigned)(p >> 32)) kv = __ldg(key + h);
        return kv;
      };
      if (crank == 0) {
        if (tid < 256) ghist[tid] = 0u;
        if (tid == 0) {
          s_prefix = 0ull;
          s_mask = 0ull;
          s_need = a.n_max < Gk ? a.n_max : Gk;
          s_done = Gk <= a.n_max;
          s_nkeep = 0;
        }
      }
      cl.sync();   // staged keys and the leader's state ready
      for (int shift = 56; shift >= 0; shift -= 8) {
        if (*L_done) break;   // cluster-uniform: read after a cluster barrier
        const unsigned long long pre = *L_prefix, msk = *L_mask;
        if (tid < 256) hist[tid] = 0u;
        __syncthreads();
        for (long long h0 = lo; h0 < hi; h0 += RND) {   // block-uniform trip count
          unsigned long long kv[J];
#pragma unroll
          for (int j = 0; j < J; ++j) {
            const long long h = h0 + (long long)j * NT + tid;
            kv[j] = h < hi ? key_at(h, msk | (255ull << shift), pre) : 0ull;
          }
#pragma unroll
          for (int j = 0; j < J; ++j) {
            const long long h = h0 + (long long)j * NT + tid;
            const bool hit = h < hi && (kv[j] & msk) == pre;
            const unsigned bin = hit ? (unsigned)((kv[j] >> shift) & 255u) : 256u;
            const unsigned peers = __match_any_sync(0xffffffffu, bin);
            if (hit && lane == __ffs(peers) - 1) atomicAdd(&hist[bin], (unsigned)__popc(peers));
          }
        }
        __syncthreads();
        if (tid < 256 && hist[tid]) atomicAdd(L_ghist + tid, hist[tid]);
        cl.sync();   // the cluster's histogram is complete
        if (crank == 0 && wid == 0) {
          // the bin holding the need-th largest key (as cap_select_kernel)
          int hv[8], c = 0;
#pragma unroll
          for (int j = 0; j < 8; ++j) c += (hv[j] = (int)ghist[255 - 8 * lane - j]);
          int x = c;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += t;
          }
          const int need0 = s_need, before = x - c;
          const unsigned own = __ballot_sync(0xffffffffu, before < need0 && need0 <= x);
          if (lane == (own ? __ffs(own) - 1 : 31)) {
            int need = need0 - before, b = 255 - 8 * lane, hb = hv[0];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              b = 255 - 8 * lane - j;
              hb = hv[j];
              if (b == 0 || hb >= need) break;
              need -= hb;
            }
            s_need = need;
            s_prefix = pre | ((unsigned long long)b << shift);
            s_mask = msk | (255ull << shift);
            if (hb == need || shift == 0) s_done = 1;
          }
          __syncwarp();
#pragma unroll
          for (int j = 0; j < 8; ++j) ghist[lane * 8 + j] = 0u;   // for the next digit
        }
        cl.sync();   // the selection is visible
      }
      // kept: keys above the selected prefix range, and the first s_need of the
      // prefix-matching ones in group order (blocks in rank order, then
      // threads, then each thread's J consecutive groups)
      const bool all = Gk <= a.n_max;
      const unsigned long long pre = *L_prefix, msk = *L_mask;
      const int need = *L_need;
      {   // this block's tie count -> the leader
        int c = 0;
        for (long long h = lo + tid; h < hi; h += NT) c += !all && (key_at(h, msk, pre) & msk) == pre;
        for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
        if (lane == 0) wtot[wid] = c;
        __syncthreads();
        if (tid == 0) {
          int t = 0;
          for (int w = 0; w < NW; ++w) t += wtot[w];
          L_tie[crank] = t;
        }
      }
      cl.sync();   // every block's tie count is in
      if (tid == 0) {
        int t = 0;
        for (int r = 0; r < crank; ++r) t += L_tie[r];
        s_tie_base = t;
      }
      __syncthreads();
      for (long long h0 = lo; h0 < hi; h0 += RND) {
        const long long hb = h0 + (long long)tid * J;   // thread tid owns groups [hb, hb + J)
        unsigned long long kv[J];
#pragma unroll
        for (int j = 0; j < J; ++j) kv[j] = hb + j < hi ? key_at(hb + j, msk, pre) : 0ull;
        unsigned above = 0u, in = 0u;
#pragma unroll
        for (int j = 0; j < J; ++j) {
          if (hb + j < hi) {
            if (all || (kv[j] & msk) > pre) above |= 1u << j;
            else if ((kv[j] & msk) == pre) in |= 1u << j;
          }
        }
        const int cnt = __popc(in);
        int x = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int t = __shfl_up_sync(0xffffffffu, x, o);
          if (lane >= o) x += t;
        }
        if (lane == 31) wtot[wid] = x;
        __syncthreads();
        int before = x - cnt, tot = 0;
        for (int w = 0; w < NW; ++w) {
          if (w < wid) before += wtot[w];
          tot += wtot[w];
        }
        int tr = s_tie_base + before;
        for (int j = 0; j < J; ++j) {
          const bool is_in = (in >> j) & 1u;
          if (((above >> j) & 1u) || (is_in && tr < need)) L_keep[atomicAdd(L_nkeep, 1)] = (int)(f0 + hb + j);
          tr += is_in;
        }
        __syncthreads();
        if (tid == 0) s_tie_base += tot;
        __syncthreads();
      }
      cl.sync();   // every kept group is in the leader's list
      if (crank == 0) {   // rank among the kept by (-extent, group order) and write
        const int nk = s_nkeep;
        for (int q = tid; q < nk; q += NT) {
          const long long g = keep_g[q];
          const double e = a.gext[g];
          int rank = 0;
          for (int j = 0; j < nk; ++j) {
            const long long h = keep_g[j];
            const double eh = a.gext[h];
            rank += (eh > e) || (eh == e && h < g);
          }
          cap_write(a, g, k, Gk, rank);
        }
      }
      cl.sync();   // the leader's state is free for the next parent
    }
    __syncthreads();   // huge_k / wtot reused by the next range
  }
}

cudaError_t launch_merge_cap(const MergeArgs& a, long long cap, cudaStream_t s, cudaStream_t aux,
                             cudaEvent_t fork, cudaEvent_t join) {
  long long b = (cap + 255) / 256;
  if (a.n_max <= kSelMax) {
    // the parents with the most groups (shared-memory selection) on the second
    // stream, concurrently with the thread-per-group ranks and the block selection
    cudaError_t e;
    if ((e = cudaEventRecord(fork, s)) != cudaSuccess) return e;
    if ((e = cudaStreamWaitEvent(aux, fork, 0)) != cudaSuccess) return e;
    if (ADPS_CAP_CLUSTER) {
      launch_k(cap_huge_cluster_kernel, 16 * kCapCS, kCapCT, 0, aux, a);
    } else {
      const int smem = kSelSmemKeys * 4;
      e = cudaFuncSetAttribute(cap_select_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      if (e != cudaSuccess) return e;
      launch_k(cap_select_kernel<true>, 16, 1024, smem, aux, a, cap);
    }
    if ((e = cudaEventRecord(join, aux)) != cudaSuccess) return e;
    launch_k(cap_small_kernel, (unsigned)(b < 1 ? 1 : (b > 65535 ? 65535 : b)), 256, 0, s, a, cap);
    launch_k(cap_select_kernel<false>, a.grid, 256, 0, s, a, cap);
    if ((e = cudaStreamWaitEvent(s, join, 0)) != cudaSuccess) return e;
  } else {
    launch_k(cap_small_kernel, (unsigned)(b < 1 ? 1 : (b > 65535 ? 65535 : b)), 256, 0, s, a, cap);
    launch_k(cap_large_kernel, a.grid * 4, 256, 0, s, a, cap);
  }
  return cudaGetLastError();
}

}  // namespace adps
