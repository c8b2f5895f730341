// Error maps + partition + region moments over the sampled views.
//
// Replaces, for every sampled view at once:
//   error_map / metric_map / erode / band_map   ref/error_partition.py:44-91
//   partition (8-connected CCL per candidate/band) ref/error_partition.py:94-134
//   the pixel sums behind region_stats            ref/error_partition.py:137-142
//   ever_dominant                                 ref/adc.py:177-180
//
// Pass structure (all views in each launch):
//   minmax_kernel     raw L1 (fp64, numpy order) -> per-view min/max
//   thresholds_kernel per-view thresholds on x = raw - lo that reproduce
//                     e = (raw-lo)/(hi-lo) > tau and the band floor exactly
//   tile_kernel       32x32 tile: maps, r x r erosion with halo, key, union-find
//                     CCL in shared memory, warp-aggregated integer moments;
//                     interior components -> regions, edge components ->
//                     partial fragments + border labels
//   border_kernel     unions fragments across tile edges (global union-find)
//   resolve_kernel    folds fragment moments into their roots
//   partial_emit_kernel roots with area >= m_min -> regions
#include <math.h>

#include "adps_internal.cuh"
#include "attribution.cuh"

#ifndef ADPS_INPUT_BULK
#define ADPS_INPUT_BULK 0   // 1: the input pass through cp.async.bulk + mbarrier stages (minmax_bulk_kernel; slower)
#endif
#ifndef ADPS_DEFERRED_BLOCK
#define ADPS_DEFERRED_BLOCK 1   // 0: deferred tiles by the full-capacity warp kernel instead of the block CCL
#endif

namespace adps {

__device__ __forceinline__ double raw_l1(const float* __restrict__ img, const float* __restrict__ gt,
                                         long long p) {
  // np.abs(rendered - gt).sum(axis=-1) == (|d0| + |d1|) + |d2| in fp64
  double a0 = fabs(dsub((double)img[3 * p + 0], (double)gt[3 * p + 0]));
  double a1 = fabs(dsub((double)img[3 * p + 1], (double)gt[3 * p + 1]));
  double a2 = fabs(dsub((double)img[3 * p + 2], (double)gt[3 * p + 2]));
  return dadd(dadd(a0, a1), a2);
}

// Per-view min/max of the raw L1 error and, in the same pass over the view,
// the ever-dominant flags of split candidates (ref/adc.py:177-180): every
// input byte of the view (image, gt, dominant map) is read exactly once.
__global__ void minmax_kernel(const float* __restrict__ image, const float* __restrict__ gt,
                              const int* __restrict__ dominant, long long hw, unsigned long long* __restrict__ lohi,
                              const unsigned char* __restrict__ cls, int N, unsigned char* __restrict__ dom_flag,
                              unsigned* __restrict__ cand_bits, double* __restrict__ raw_out,
                              raw16_t* __restrict__ rawf_out, int v0) {
  pdl_wait();   // programmatic dependent launch: the previous kernel's results are visible
  const int v = v0 + blockIdx.y;
  const float* img = image + (long long)v * hw * 3;
  const float* g = gt + (long long)v * hw * 3;
  const int* dom = dominant + (long long)v * hw;
  unsigned* bits = cand_bits + (long long)v * ((hw + 31) / 32);
  const int lane = threadIdx.x & 31;
  double lo = INFINITY, hi = 0.0;
  // base is a multiple of 32, so a warp's pixels are one word of cand_bits
  for (long long base = (long long)blockIdx.x * blockDim.x; base < hw; base += (long long)gridDim.x * blockDim.x) {
    const long long p = base + threadIdx.x;
    int d = -1;
    if (p < hw) {
      const double r = raw_l1(img, g, p);
      if (raw_out) raw_out[(long long)v * hw + p] = r;
      // the bit-plane path keeps raw rounded toward zero (4 B/px); compares that
      // the rounding cannot decide are redone exactly (tile_words_kernel)
      if (rawf_out) rawf_out[(long long)v * hw + p] = raw16(r);
      lo = fmin(lo, r);
      hi = fmax(hi, r);
      d = __ldg(dom + p);
    }
    // split-candidate test once per run of equal ids: ever-dominant flag and
    // the per-pixel candidate bit the tile pass reads instead of cls[D]
    const int left = __shfl_up_sync(0xffffffffu, d, 1);
    const bool head = lane == 0 || left != d;
    bool isc = false;
    if (head && d >= 0 && d < N && __ldg(cls + d) == 1) {
      isc = true;
      if (dom_flag && dom_flag[d] == 0) dom_flag[d] = 1;
    }
    const unsigned heads = __ballot_sync(0xffffffffu, head);
    isc = __shfl_sync(0xffffffffu, isc, 31 - __clz(heads & (0xffffffffu >> (31 - lane))));
    const unsigned word = __ballot_sync(0xffffffffu, isc);
    if (lane == 0 && base + (threadIdx.x & ~31) < hw) bits[(base + threadIdx.x) >> 5] = word;
  }
  for (int o = 16; o > 0; o >>= 1) {
    lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  __shared__ double slo[32], shi[32];
  const int wid = threadIdx.x >> 5;
  if (lane == 0) {
    slo[wid] = lo;
    shi[wid] = hi;
  }
  __syncthreads();
  if (wid == 0) {
    int nw = blockDim.x >> 5;
    lo = lane < nw ? slo[lane] : INFINITY;
    hi = lane < nw ? shi[lane] : 0.0;
    for (int o = 16; o > 0; o >>= 1) {
      lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
      hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    if (lane == 0) {
      // raw >= +0.0, so IEEE order == unsigned order of the bit patterns
      atomicMin(&lohi[2 * v + 0], (unsigned long long)__double_as_longlong(lo));
      atomicMax(&lohi[2 * v + 1], (unsigned long long)__double_as_longlong(hi));
    }
  }
}

__device__ __forceinline__ double raw_l1_3(float a0, float a1, float a2, float g0, float g1, float g2) {
  // np.abs(rendered - gt).sum(axis=-1) == (|d0| + |d1|) + |d2| in fp64
  return dadd(dadd(fabs(dsub((double)a0, (double)g0)), fabs(dsub((double)a1, (double)g1))),
              fabs(dsub((double)a2, (double)g2)));
}

// The same pass, two pixels per thread (even hw: every view starts 8-byte
// aligned, so the pixel pairs load as float2/int2 and 32-bit offsets suffice).
// A warp covers 64 pixels = two candidate-bit words; the candidate test is
// looked up for a thread's first pixel and for its second when the id changes.
__global__ void __launch_bounds__(256) minmax2_kernel(const float* __restrict__ image, const float* __restrict__ gt,
                                                      const int* __restrict__ dominant, int hw,
                                                      unsigned long long* __restrict__ lohi,
                                                      const unsigned char* __restrict__ cls, int N,
                                                      unsigned char* __restrict__ dom_flag,
                                                      unsigned* __restrict__ cand_bits, double* __restrict__ raw_out,
                                                      raw16_t* __restrict__ rawf_out, int v0) {
  pdl_wait();   // programmatic dependent launch: the previous kernel's results are visible
  const int v = v0 + blockIdx.y;
  const long long vb = (long long)v * hw;
  const float2* img2 = reinterpret_cast<const float2*>(image + vb * 3);
  const float2* gt2 = reinterpret_cast<const float2*>(gt + vb * 3);
  const int2* dom2 = reinterpret_cast<const int2*>(dominant + vb);
  unsigned* rawf2 = rawf_out ? reinterpret_cast<unsigned*>(rawf_out + vb) : nullptr;   // two codes per word
  double* rawd = raw_out ? raw_out + vb : nullptr;
  unsigned* bits = cand_bits + (long long)v * ((hw + 31) / 32);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double lo = INFINITY, hi = 0.0;
  for (int base = blockIdx.x * 512; base < hw; base += gridDim.x * 512) {
    const int p = base + 2 * threadIdx.x;   // even; p + 1 < hw whenever p < hw
    int d0 = -1, d1 = -1;
    if (p < hw) {
      const int q = (3 * p) >> 1;
      const float2 a0 = __ldg(img2 + q), a1 = __ldg(img2 + q + 1), a2 = __ldg(img2 + q + 2);
      const float2 g0 = __ldg(gt2 + q), g1 = __ldg(gt2 + q + 1), g2 = __ldg(gt2 + q + 2);
      const int2 dd = __ldg(dom2 + (p >> 1));
      d0 = dd.x;
      d1 = dd.y;
      const double r0 = raw_l1_3(a0.x, a0.y, a1.x, g0.x, g0.y, g1.x);
      const double r1 = raw_l1_3(a1.y, a2.x, a2.y, g1.y, g2.x, g2.y);
      if (rawf2) rawf2[p >> 1] = (unsigned)raw16(r0) | ((unsigned)raw16(r1) << 16);
      if (rawd) {
        rawd[p] = r0;
        rawd[p + 1] = r1;
      }
      lo = fmin(lo, fmin(r0, r1));
      hi = fmax(hi, fmax(r0, r1));
    }
    bool c0 = false, c1 = false;
    if (d0 >= 0 && d0 < N && __ldg(cls + d0) == 1) {
      c0 = true;
      if (dom_flag && dom_flag[d0] == 0) dom_flag[d0] = 1;
    }
    if (d1 == d0) {
      c1 = c0;
    } else if (d1 >= 0 && d1 < N && __ldg(cls + d1) == 1) {
      c1 = true;
      if (dom_flag && dom_flag[d1] == 0) dom_flag[d1] = 1;
    }
    // lane t holds pixels 2t, 2t+1 of the warp's 64: its two bits go to positions
    // 2(t & 15), 2(t & 15) + 1 of word t / 16 (one REDUX per word)
    const unsigned cb = ((c0 ? 1u : 0u) | (c1 ? 2u : 0u)) << (2 * (lane & 15));
    const unsigned w0 = __reduce_or_sync(0xffffffffu, lane < 16 ? cb : 0u);
    const unsigned w1 = __reduce_or_sync(0xffffffffu, lane < 16 ? 0u : cb);
    const int wp = base + 64 * wid;   // first pixel of this warp: a multiple of 64
    if (lane == 0 && wp < hw) bits[wp >> 5] = w0;
    if (lane == 1 && wp + 32 < hw) bits[(wp >> 5) + 1] = w1;
  }
  for (int o = 16; o > 0; o >>= 1) {
    lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  __shared__ double slo[32], shi[32];
  if (lane == 0) {
    slo[wid] = lo;
    shi[wid] = hi;
  }
  __syncthreads();
  if (wid == 0) {
    const int nw = blockDim.x >> 5;
    lo = lane < nw ? slo[lane] : INFINITY;
    hi = lane < nw ? shi[lane] : 0.0;
    for (int o = 16; o > 0; o >>= 1) {
      lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
      hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    if (lane == 0) {   // raw >= +0.0, so IEEE order == unsigned order of the bit patterns
      atomicMin(&lohi[2 * v + 0], (unsigned long long)__double_as_longlong(lo));
      atomicMax(&lohi[2 * v + 1], (unsigned long long)__double_as_longlong(hi));
    }
  }
}

// ------------------------------------------------- input pass, bulk-copy form
// The same input pass over the flat pixel stream of views [v0, v1) (every view
// starts at pixel v*hw; hw even), staged through shared memory by the bulk
// copy engine: one elected thread issues three cp.async.bulk copies per
// 1024-pixel chunk (image 12 KB, gt 12 KB, dominant 4 KB; SASS UBLKCP) into a
// 3-stage ring completed by mbarrier transaction counts, and the 512 threads
// read their pixel pairs from shared memory.  A persistent block walks a
// contiguous chunk range (at most two views per chunk: hw >= 16384), keeping
// the min/max of the current and the next view in registers and flushing
// them with a block reduction when the view advances.  Candidate bits: the
// warp's 64 pixels map to at most three words of the view's bit array (view
// starts are not word aligned), OR-ed in with atomics (zeroed beforehand).
constexpr int kMBThreads = 512;
constexpr int kMBChunk = 2 * kMBThreads;   // pixels per stage
constexpr int kMBStages = 3;
struct MBStage {
  float img[3 * kMBChunk];
  float gt[3 * kMBChunk];
  int dom[kMBChunk];
};
constexpr size_t kMBSmem = sizeof(MBStage) * kMBStages + 64;

__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(a), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(a), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned phase) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(a),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(d),
               "l"(src), "r"(bytes), "r"(b)
               : "memory");
}

// interleave: bit 2l = a bit l, bit 2l+1 = b bit l
__device__ __forceinline__ unsigned long long interleave32(unsigned a, unsigned b) {
  auto spread = [](unsigned long long x) {
    x = (x | (x << 16)) & 0x0000FFFF0000FFFFull;
    x = (x | (x << 8)) & 0x00FF00FF00FF00FFull;
    x = (x | (x << 4)) & 0x0F0F0F0F0F0F0F0Full;
    x = (x | (x << 2)) & 0x3333333333333333ull;
    x = (x | (x << 1)) & 0x5555555555555555ull;
    return x;
  };
  return spread(a) | (spread(b) << 1);
}

struct BulkArgs {
  const float* image;   // view 0 of the plan's arrays (flat pixel p at image + 3p)
  const float* gt;
  const int* dom;
  long long p0, p1;     // flat pixel range [v0*hw, v1*hw)
  long long hw;
  unsigned long long* lohi;
  const unsigned char* cls;
  int N;
  unsigned char* dom_flag;
  unsigned* cand_bits;  // [V][nwords], zeroed
  raw16_t* rawf;        // flat
};

__global__ void __launch_bounds__(kMBThreads) minmax_bulk_kernel(BulkArgs a) {
  pdl_wait();   // programmatic dependent launch: the previous kernel's results are visible
  extern __shared__ __align__(128) unsigned char mb_smem[];
  MBStage* stage = reinterpret_cast<MBStage*>(mb_smem);
  unsigned long long* full = reinterpret_cast<unsigned long long*>(mb_smem + sizeof(MBStage) * kMBStages);
  __shared__ double s_lo[2][kMBThreads / 32], s_hi[2][kMBThreads / 32];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const long long n_px = a.p1 - a.p0;
  const long long n_chunks = (n_px + kMBChunk - 1) / kMBChunk;
  const long long c_lo = n_chunks * blockIdx.x / gridDim.x, c_hi = n_chunks * (blockIdx.x + 1) / gridDim.x;
  const long long nwords = (a.hw + 31) / 32;
  auto chunk_full = [&](long long c) { return a.p0 + (c + 1) * kMBChunk <= a.p1; };
  auto issue = [&](long long c) {   // thread 0: the three copies of chunk c into its stage
    const int st = (int)((c - c_lo) % kMBStages);
    const long long pc = a.p0 + c * kMBChunk;
    mbar_expect_tx(&full[st], (unsigned)(sizeof(MBStage)));
    bulk_g2s(stage[st].img, a.image + 3 * pc, 12u * kMBChunk, &full[st]);
    bulk_g2s(stage[st].gt, a.gt + 3 * pc, 12u * kMBChunk, &full[st]);
    bulk_g2s(stage[st].dom, a.dom + pc, 4u * kMBChunk, &full[st]);
  };
  if (tid == 0) {
    for (int i = 0; i < kMBStages; ++i) mbar_init(&full[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid == 0)
    for (long long c = c_lo; c < c_lo + kMBStages && c < c_hi; ++c)
      if (chunk_full(c)) issue(c);
  long long cv = c_lo < c_hi ? (a.p0 + c_lo * kMBChunk) / a.hw : 0;   // current view (block-uniform)
  double lo[2] = {INFINITY, INFINITY}, hi[2] = {0.0, 0.0};        // [0] view cv, [1] view cv + 1
  auto flush = [&](long long v, double l, double h) {               // block-uniform call
    for (int o = 16; o > 0; o >>= 1) {
      l = fmin(l, __shfl_xor_sync(0xffffffffu, l, o));
      h = fmax(h, __shfl_xor_sync(0xffffffffu, h, o));
    }
    if (lane == 0) {
      s_lo[0][wid] = l;
      s_hi[0][wid] = h;
    }
    __syncthreads();
    if (tid == 0) {
      for (int w = 1; w < kMBThreads / 32; ++w) {
        l = fmin(l, s_lo[0][w]);
        h = fmax(h, s_hi[0][w]);
      }
      if (l <= h) {   // raw >= +0.0: IEEE order == unsigned order of the bit patterns
        atomicMin(&a.lohi[2 * v + 0], (unsigned long long)__double_as_longlong(l));
        atomicMax(&a.lohi[2 * v + 1], (unsigned long long)__double_as_longlong(h));
      }
    }
    __syncthreads();
  };
  // candidate bits + ever-dominant flags of a chunk, one iteration late: the
  // class gathers of chunk c are issued with its loads and consumed after the
  // next chunk's wait, so their latency hides behind it
  auto finish_cand = [&](long long pc, int d0, int d1, unsigned char k0, unsigned char k1) {   // block-uniform
    const long long p = pc + 2 * tid;
    const bool in = p < a.p1;
    const bool c0 = in && k0 == 1, c1 = in && k1 == 1;
    // ever-dominant flags: one store per distinct candidate id of the warp (no read)
    {
      const int key0 = c0 ? d0 : -1;
      const unsigned peers0 = __match_any_sync(0xffffffffu, key0);
      if (c0 && lane == __ffs(peers0) - 1) a.dom_flag[d0] = 1;
      const int key1 = c1 && d1 != d0 ? d1 : -1;
      const unsigned peers1 = __match_any_sync(0xffffffffu, key1);
      if (key1 >= 0 && lane == __ffs(peers1) - 1) a.dom_flag[d1] = 1;
    }
    const unsigned b0 = __ballot_sync(0xffffffffu, c0), b1 = __ballot_sync(0xffffffffu, c1);
    if (!(b0 | b1)) return;
    const long long pw = pc + 64 * wid;
    const long long vw = pw / a.hw, vw_end = (pw + 63) / a.hw;
    if (vw == vw_end) {   // one view: at most three words
      if (lane < 3) {
        const unsigned long long m = interleave32(b0, b1);
        const long long q0 = pw - vw * a.hw;
        const int sft = (int)(q0 & 31);
        const unsigned long long lo64 = m << sft, hi64 = sft ? m >> (64 - sft) : 0ull;
        const unsigned w = lane == 0 ? (unsigned)lo64 : (lane == 1 ? (unsigned)(lo64 >> 32) : (unsigned)hi64);
        if (w) atomicOr(a.cand_bits + vw * nwords + (q0 >> 5) + lane, w);
      }
    } else {              // the warp straddles a view boundary: per pixel
      const long long v = p / a.hw;
      if (c0) {
        const long long q = p - v * a.hw;
        atomicOr(a.cand_bits + v * nwords + (q >> 5), 1u << (q & 31));
      }
      if (c1) {
        const long long q = p + 1 - v * a.hw;
        atomicOr(a.cand_bits + v * nwords + (q >> 5), 1u << (q & 31));
      }
    }
  };
  long long prev_pc = -1;
  int pd0 = -1, pd1 = -1;
  unsigned char pk0 = 0, pk1 = 0;
  for (long long c = c_lo; c < c_hi; ++c) {
    const long long pc = a.p0 + c * kMBChunk;
    const long long vA = pc / a.hw;
    while (vA > cv) {   // the block moved past view cv: publish it (block-uniform)
      flush(cv, lo[0], hi[0]);
      lo[0] = lo[1];
      hi[0] = hi[1];
      lo[1] = INFINITY;
      hi[1] = 0.0;
      ++cv;
    }
    const bool fullc = chunk_full(c);
    const int st = (int)((c - c_lo) % kMBStages);
    const long long p = pc + 2 * tid;   // flat, even
    const bool in = p < a.p1;
    float i6[6] = {0, 0, 0, 0, 0, 0}, g6[6] = {0, 0, 0, 0, 0, 0};
    int d0 = -1, d1 = -1;
    if (fullc) {
      mbar_wait(&full[st], (unsigned)(((c - c_lo) / kMBStages) & 1));
      const int2 dd = reinterpret_cast<const int2*>(stage[st].dom)[tid];
      d0 = dd.x;
      d1 = dd.y;
    } else if (in) {   // the partial last chunk: straight from global
      d0 = __ldg(a.dom + p);
      d1 = __ldg(a.dom + p + 1);
    }
    // class gathers of this chunk (consumed next iteration)
    const unsigned char k0 = d0 >= 0 && d0 < a.N ? __ldg(a.cls + d0) : 0;
    const unsigned char k1 = d1 == d0 ? k0 : (d1 >= 0 && d1 < a.N ? __ldg(a.cls + d1) : 0);
    if (fullc) {
      const float2* si = reinterpret_cast<const float2*>(stage[st].img) + 3 * tid;
      const float2* sg = reinterpret_cast<const float2*>(stage[st].gt) + 3 * tid;
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const float2 x = si[k], y = sg[k];
        i6[2 * k] = x.x;
        i6[2 * k + 1] = x.y;
        g6[2 * k] = y.x;
        g6[2 * k + 1] = y.y;
      }
    } else if (in) {
#pragma unroll
      for (int k = 0; k < 6; ++k) {
        i6[k] = __ldg(a.image + 3 * p + k);
        g6[k] = __ldg(a.gt + 3 * p + k);
      }
    }
    if (in) {
      const long long v = p / a.hw;   // both pixels of the pair are in view v (hw even)
      const double r0 = raw_l1_3(i6[0], i6[1], i6[2], g6[0], g6[1], g6[2]);
      const double r1 = raw_l1_3(i6[3], i6[4], i6[5], g6[3], g6[4], g6[5]);
      reinterpret_cast<unsigned*>(a.rawf)[p >> 1] = (unsigned)raw16(r0) | ((unsigned)raw16(r1) << 16);
      const int k = v == cv ? 0 : 1;
      lo[k] = fmin(lo[k], fmin(r0, r1));
      hi[k] = fmax(hi[k], fmax(r0, r1));
    }
    if (prev_pc >= 0) finish_cand(prev_pc, pd0, pd1, pk0, pk1);
    prev_pc = pc;
    pd0 = d0;
    pd1 = d1;
    pk0 = k0;
    pk1 = k1;
    __syncthreads();   // stage st fully consumed
    if (tid == 0 && c + kMBStages < c_hi && chunk_full(c + kMBStages)) issue(c + kMBStages);
  }
  if (prev_pc >= 0) finish_cand(prev_pc, pd0, pd1, pk0, pk1);
  if (c_lo < c_hi) {
    flush(cv, lo[0], hi[0]);
    if (cv + 1 < (a.p1 + a.hw - 1) / a.hw) flush(cv + 1, lo[1], hi[1]);
  }
}

bool minmax_bulk_ok(const AttributionArgs& a, int v0, int v1) {
  const long long hw = (long long)a.H * a.W;
  const long long p0 = hw * v0;
  return ADPS_INPUT_BULK && a.rawf && !a.raw && hw % 2 == 0 && hw >= 16384 && p0 % 4 == 0 &&
         (uintptr_t)a.image % 16 == 0 && (uintptr_t)a.gt % 16 == 0 && (uintptr_t)a.dom % 16 == 0 &&
         (uintptr_t)a.rawf % 16 == 0 && v1 > v0;
}

cudaError_t launch_minmax_bulk(const AttributionArgs& a, int v0, int v1, cudaStream_t s) {
  const long long hw = (long long)a.H * a.W;
  BulkArgs b;
  b.image = a.image;
  b.gt = a.gt;
  b.dom = a.dom;
  b.p0 = hw * v0;
  b.p1 = hw * v1;
  b.hw = hw;
  b.lohi = a.lohi;
  b.cls = a.cls;
  b.N = a.N;
  b.dom_flag = a.dom_flag;
  b.cand_bits = a.cand_bits;
  b.rawf = a.rawf;
  const long long nwords = (hw + 31) / 32;
  cudaError_t e = cudaMemsetAsync(a.cand_bits + (long long)v0 * nwords, 0, 4ull * nwords * (v1 - v0), s);
  if (e != cudaSuccess) return e;
  static int per_sm = 0, sms = 148;
  if (per_sm == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    e = cudaFuncSetAttribute(minmax_bulk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kMBSmem);
    if (e != cudaSuccess) return e;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, minmax_bulk_kernel, kMBThreads, kMBSmem) !=
            cudaSuccess ||
        per_sm < 1)
      per_sm = 1;
  }
  const long long chunks = (b.p1 - b.p0 + kMBChunk - 1) / kMBChunk;
  long long grid = (long long)per_sm * sms;
  if (grid > chunks) grid = chunks;
  launch_k(minmax_bulk_kernel, (unsigned)grid, kMBThreads, kMBSmem, s, b);
  return cudaGetLastError();
}

// e(x) = x / d with x = fl(raw - lo) and d = fl(hi - lo); both predicates below
// are monotone in x, so each is a single threshold on x.
__device__ __forceinline__ bool m_pred(double x, double d, double tau) { return ddiv(x, d) > tau; }

__device__ __forceinline__ double band_raw(double x, double d, double tau, double omt, double nb) {
  // np.floor((e - tau) / (1.0 - tau) * l_bands)  (ref/error_partition.py:82)
  return floor(dmul(ddiv(dsub(ddiv(x, d), tau), omt), nb));
}

// Warp-parallel search over the bit patterns of non-negative doubles (their
// integer order is their IEEE order): the smallest x in (lo, hi] with pred(x),
// given pred monotone, pred(lo) false and pred(hi) true.  Each round the 32
// lanes test 32 evenly spaced points, so the interval shrinks 33-fold.
template <class Pred>
__device__ long long warp_bits_search(long long lo, long long hi, Pred pred) {
  const int lane = threadIdx.x & 31;
  while (hi - lo > 1) {
    const long long span = hi - lo;
    const long long step = span / 33 > 0 ? span / 33 : 1;
    const long long p = lo + (long long)(lane + 1) * step;
    const bool ok = p < hi && pred(__longlong_as_double(p));
    const unsigned b = __ballot_sync(0xffffffffu, ok);
    const unsigned tested = __ballot_sync(0xffffffffu, p < hi);
    if (b == 0u) {
      const int last = 31 - __clz(tested);   // every tested point is false
      lo = lo + (long long)(last + 1) * step;
    } else {
      const int first = __ffs(b) - 1;
      const long long pf = lo + (long long)(first + 1) * step;
      lo = first > 0 ? lo + (long long)first * step : lo;
      hi = pf;
    }
  }
  return hi;
}

__device__ double min_true(double d, int k, double tau, double omt, double nb) {
  auto pred = [&](double x) -> bool { return k == 0 ? m_pred(x, d, tau) : band_raw(x, d, tau, omt, nb) >= (double)k; };
  if (!pred(d)) return INFINITY;
  if (pred(0.0)) return 0.0;
  return __longlong_as_double(warp_bits_search(0ll, __double_as_longlong(d), pred));
}

// thr[v*L + 0] = x threshold of m; thr[v*L + k] = x threshold of band >= k.
// the same threshold in the raw domain: the smallest raw in [lo, hi] with
// fl(raw - lo) >= t (the subtraction is monotone, and every raw of the view lies
// in [lo, hi]), so the warp CCL compares raw directly
__device__ double raw_threshold(double lo, double hi, double t) {
  if (t == INFINITY) return INFINITY;
  if (!(dsub(hi, lo) >= t)) return INFINITY;
  if (dsub(lo, lo) >= t) return lo;
  auto pred = [&](double r) -> bool { return dsub(r, lo) >= t; };
  return __longlong_as_double(warp_bits_search(__double_as_longlong(lo), __double_as_longlong(hi), pred));
}

// a warp per (view, threshold)
__global__ void thresholds_kernel(const unsigned long long* __restrict__ lohi, int v0, int n_views, int L,
                                  double tau, double* __restrict__ lo_out, double* __restrict__ thr,
                                  double* __restrict__ thr_raw) {
  pdl_wait();   // programmatic dependent launch: the previous kernel's results are visible
  const int t = v0 * L + (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  if (t >= (v0 + n_views) * L) return;   // warp-uniform
  const bool lead = (threadIdx.x & 31) == 0;
  int v = t / L, k = t % L;
  double lo = __longlong_as_double((long long)lohi[2 * v]);
  double hi = __longlong_as_double((long long)lohi[2 * v + 1]);
  if (k == 0 && lead) lo_out[v] = lo;
  if (hi == lo) {  // error_map returns zeros: m false, band 0 (ref/error_partition.py:52-53)
    if (lead) {
      thr[t] = INFINITY;
      if (thr_raw) thr_raw[t] = INFINITY;
    }
    return;
  }
  double d = dsub(hi, lo);
  double omt = dsub(1.0, tau);
  const double x = min_true(d, k, tau, omt, (double)L);
  const double r = thr_raw ? raw_threshold(lo, hi, x) : 0.0;
  if (lead) {
    thr[t] = x;
    if (thr_raw) thr_raw[t] = r;
  }
}

// ---------------------------------------------------- ever-dominant (early)
// ever_dominant[i] = any sampled pixel has D == i (ref/adc.py:177-180), for
// split candidates; one check/store per run of equal ids along a warp's 32
// consecutive pixels.  Runs first so the host learns the fallback count (and
// can draw its normals) while the rest of phase 1 runs on the GPU.
__global__ void fallback_count_kernel(const int* __restrict__ split_list, const unsigned char* __restrict__ dom_flag,
                                      Counters* ctr) {
  pdl_wait();   // programmatic dependent launch: the previous kernel's results are visible
  const long long n = (long long)ctr->n_split;
  int c = 0;
  for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (long long)gridDim.x * blockDim.x)
    c += dom_flag[split_list[k]] == 0;
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(&ctr->n_fallback_pre, (unsigned long long)c);
}

// ----------------------------------------------------------------- tile pass
struct TileSmem {
  unsigned long long mrow[kTileH + 2 * kMaxErodeHalo];   // pre-erosion m of haloed rows, bit = x - x0 + hl
  unsigned erow[kTileH];                                  // eroded m of the tile rows, bit = x - x0
  unsigned char band[kTilePx];
  unsigned char touch[kTilePx];
  int d[kTilePx];
  int label[kTilePx];
  int slot[kTilePx];
  int mom[6][kTilePx];
  int n_part, n_reg;
  unsigned long long base_part, base_reg;
};

// Block-per-tile CCL (general r_erode, any number of runs, debug maps).  The
// warp-per-tile kernel (tile_warp.cu) handles the common case and defers
// the tiles it cannot (too many runs) to this one.
__device__ void tile_block(const TileParams& P, TileSmem& S, const int tile) {
  const int tid = threadIdx.x;
  const int tiles_per_view = P.tiles_x * P.tiles_y;
  const int v = tile / tiles_per_view;
  const int tile_in_view = tile % tiles_per_view;
  const int tyi = tile_in_view / P.tiles_x, txi = tile_in_view % P.tiles_x;
  const int x0 = txi * kTileW, y0 = tyi * kTileH;
  const int W = P.W, H = P.H;
  const long long hw = (long long)W * H;
  const float* img = P.image + (long long)v * hw * 3;
  const float* gtv = P.gt + (long long)v * hw * 3;
  const int* dom = P.dom + (long long)v * hw;
  const double lo = P.lo[v];
  const double* thr = P.thr + (long long)v * P.L;
  const double x_m = thr[0];
  const int r = P.r_erode;
  const int hl = r > 1 ? r / 2 : 0;
  const int hh = r > 1 ? r - r / 2 - 1 : 0;
  const int ew = kTileW + hl + hh, eh = kTileH + hl + hh;

  if (tid == 0) {
    S.n_part = 0;
    S.n_reg = 0;
  }
  // 0+1. each warp owns 4 tile rows (lane = x): dominant map, image and gt of
  //    all its rows are loaded at once; candidate ids and ever-dominant flags
  //    (over ALL pixels, ref/adc.py:177-180) once per run of equal dominant id;
  //    pre-erosion metric as row bitmasks (ballot) and band per pixel.
  const int lane = tid & 31, wid = tid >> 5;
  constexpr int kRowsPerWarp = kTileH / (kTileThreads / 32);
  float fi[kRowsPerWarp][3], fg[kRowsPerWarp][3];
  int dd[kRowsPerWarp];
#pragma unroll
  for (int k = 0; k < kRowsPerWarp; ++k) {
    const int x = x0 + lane, y = y0 + wid + k * (kTileThreads / 32);
    const bool inb = x < W && y < H;
    const long long p = inb ? (long long)y * W + x : 0;
    dd[k] = inb ? __ldg(dom + p) : -1;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      fi[k][c] = inb ? __ldg(img + 3 * p + c) : 0.0f;
      fg[k][c] = inb ? __ldg(gtv + 3 * p + c) : 0.0f;
    }
  }
  int n_cand = 0;
#pragma unroll
  for (int k = 0; k < kRowsPerWarp; ++k) {
    const int ty = wid + k * (kTileThreads / 32);
    const int left = __shfl_up_sync(0xffffffffu, dd[k], 1);
    const bool head = lane == 0 || left != dd[k];
    bool isc = false;
    if (head && dd[k] >= 0 && dd[k] < P.N) isc = __ldg(P.cls + dd[k]) == 1;
    const unsigned heads = __ballot_sync(0xffffffffu, head);
    isc = __shfl_sync(0xffffffffu, isc, 31 - __clz(heads & (0xffffffffu >> (31 - lane))));
    S.d[ty * kTileW + lane] = isc ? dd[k] : -1;
    n_cand += isc;
  }
#pragma unroll
  for (int k = 0; k < kRowsPerWarp; ++k) {
    const int ty = wid + k * (kTileThreads / 32);
    const int x = x0 + lane, y = y0 + ty;
    bool m = false;
    unsigned char b = 0;
    if (x < W && y < H) {
      // np.abs(rendered - gt).sum(axis=-1) == (|d0| + |d1|) + |d2| in fp64, minus lo
      const double raw = dadd(dadd(fabs(dsub((double)fi[k][0], (double)fg[k][0])),
                                   fabs(dsub((double)fi[k][1], (double)fg[k][1]))),
                              fabs(dsub((double)fi[k][2], (double)fg[k][2])));
      const double xr = dsub(raw, lo);
      m = xr >= x_m;
      int bb = 0;
      for (int q = 1; q < P.L; ++q) bb += xr >= thr[q];
      b = (unsigned char)bb;
    }
    S.band[ty * kTileW + lane] = b;
    const unsigned bits = __ballot_sync(0xffffffffu, m);
    if (lane == 0) S.mrow[ty + hl] = (unsigned long long)bits << hl;
  }
  // a tile without split-candidate pixels cannot hold a region
  if (__syncthreads_count(n_cand) == 0 && !P.dbg_m) {
    int* border = P.border + (long long)tile * kBorderSlots;
    for (int s = tid; s < kBorderSlots; s += kTileThreads) border[s] = -1;
    return;
  }
  if (r > 1) {
    if (tid < hl + hh) S.mrow[tid < hl ? tid : kTileH + tid] = 0ull;   // halo rows start empty
    __syncthreads();
    const int n_halo = ew * eh - kTilePx;
    for (int h = tid; h < n_halo; h += kTileThreads) {
      int ex, ey;
      const int top = hl * ew, bot = hh * ew;
      if (h < top) { ey = h / ew; ex = h % ew; }
      else if (h < top + bot) { ey = hl + kTileH + (h - top) / ew; ex = (h - top) % ew; }
      else {
        const int c = h - top - bot, side = hl + hh;
        ey = hl + c / side;
        const int k = c % side;
        ex = k < hl ? k : kTileW + k;
      }
      const int x = x0 - hl + ex, y = y0 - hl + ey;
      if (x >= 0 && x < W && y >= 0 && y < H &&
          dsub(raw_l1(img, gtv, (long long)y * W + x), lo) >= x_m)
        atomicOr(&S.mrow[ey], 1ull << ex);
    }
  }
  __syncthreads();
  // 2. r x r erosion on the bitmasks (offsets -(r//2) .. r-r//2-1; outside = 0)
  if (lane < kRowsPerWarp) {   // every warp erodes its own 4 rows
    const int row0 = wid + lane * (kTileThreads / 32);
    const int span = hl + hh;
    unsigned long long acc = ~0ull;
    for (int dy = 0; dy <= span; ++dy) {
      const unsigned long long row = S.mrow[row0 + dy];
      unsigned long long h = row;
      for (int dx = 1; dx <= span; ++dx) h &= row >> dx;
      acc &= h;
    }
    S.erow[row0] = (unsigned)acc;
  }
  __syncthreads();
  // 3. keys + ever-dominant flags; each warp owns whole 32-px rows (lane = x),
  //    so horizontal runs of equal key are found with ballots and every pixel
  //    starts labelled with its run's first pixel (short union-find paths).
  for (int p = tid; p < kTilePx; p += kTileThreads) {
    int tx = p % kTileW, ty = p / kTileW;
    int x = x0 + tx, y = y0 + ty;
    int key = -1;
    unsigned char mer = 0;
    if (x < W && y < H) {
      mer = (S.erow[ty] >> tx) & 1u;
      if (mer) key = S.d[p];
      if (P.dbg_m) {
        long long q = (long long)v * hw + (long long)y * W + x;
        P.dbg_m[q] = mer;
        P.dbg_b[q] = S.band[p];
      }
    }
    const int band = S.band[p];
    const unsigned keyed_m = __ballot_sync(0xffffffffu, key >= 0);
    const int lkey = __shfl_up_sync(0xffffffffu, key, 1);
    const int lband = __shfl_up_sync(0xffffffffu, band, 1);
    const unsigned cont_m = __ballot_sync(0xffffffffu, key >= 0 && tx > 0 && lkey == key && lband == band);
    const unsigned starts = keyed_m & ~cont_m;
    const int run0 = 31 - __clz(starts & (0xffffffffu >> (31 - tx)));
    S.d[p] = key;
    S.label[p] = key >= 0 ? ty * kTileW + run0 : -1;
    if (key >= 0 && run0 == tx) {   // only run starts can become roots
      S.touch[p] = 0;
#pragma unroll
      for (int k = 0; k < 6; ++k) S.mom[k][p] = 0;
    }
  }
  __syncthreads();
  // 4. run-level unions with the row above: 8-connectivity with equal
  //    (candidate, band) is "horizontal run" + one union per (run, run above)
  //    adjacency -- N at the first overlapping pixel, NW at the run start, NE
  //    at the run end.
  for (int p = tid; p < kTilePx; p += kTileThreads) {
    const int key = S.d[p];
    const int ty = p / kTileW, tx = p % kTileW;
    if (key < 0 || ty == 0) continue;
    const unsigned char b = S.band[p];
    const int q = p - kTileW;
    const bool a0 = S.d[q] == key && S.band[q] == b;
    const bool am = tx > 0 && S.d[q - 1] == key && S.band[q - 1] == b;
    const bool ap = tx < kTileW - 1 && S.d[q + 1] == key && S.band[q + 1] == b;
    const bool start = tx == 0 || !(S.d[p - 1] == key && S.band[p - 1] == b);
    const bool end = tx == kTileW - 1 || !(S.d[p + 1] == key && S.band[p + 1] == b);
    if (a0 && (start || !am)) uf_unite(S.label, p, q);
    if (start && am && !a0) uf_unite(S.label, p, q - 1);
    if (end && ap && !a0) uf_unite(S.label, p, q + 1);
  }
  __syncthreads();
  // compress run starts (every label points at a run start; roots are run starts)
  for (int p = tid; p < kTilePx; p += kTileThreads) {
    const int key = S.d[p];
    if (key < 0) continue;
    const int tx = p % kTileW;
    const bool start = tx == 0 || !(S.d[p - 1] == key && S.band[p - 1] == S.band[p]);
    // read-only find: a halving find would rewrite labels of other run starts
    // on its path and could overwrite their freshly stored roots
    if (start) S.label[p] = uf_find(S.label, p);
  }
  __syncthreads();
  // 5. integer moments per run in closed form (tile-local coordinates, exact),
  //    one shared atomic per run and moment
  const bool left_in = x0 > 0, top_in = y0 > 0;
  const bool right_in = x0 + kTileW < W, bottom_in = y0 + kTileH < H;
  for (int p = tid; p < kTilePx; p += kTileThreads) {
    const int key = S.d[p];
    const int tx = p % kTileW, ty = p / kTileW;
    const bool keyed = key >= 0;
    const bool cont = keyed && tx < kTileW - 1 && S.d[p + 1] == key && S.band[p + 1] == S.band[p];
    const unsigned ends = __ballot_sync(0xffffffffu, keyed && !cont);
    const bool start = keyed && (tx == 0 || !(S.d[p - 1] == key && S.band[p - 1] == S.band[p]));
    if (start) {
      const int e = __ffs(ends & (0xffffffffu << tx)) - 1;
      const int root = S.label[p];
      const int n = e - tx + 1;
      const int sx = (tx + e) * n / 2;
      const int sxx = (e * (e + 1) * (2 * e + 1) - (tx - 1) * tx * (2 * tx - 1)) / 6;
      atomicAdd(&S.mom[0][root], n);
      atomicAdd(&S.mom[1][root], sx);
      atomicAdd(&S.mom[2][root], ty * n);
      atomicAdd(&S.mom[3][root], sxx);
      atomicAdd(&S.mom[4][root], ty * sx);
      atomicAdd(&S.mom[5][root], ty * ty * n);
      const bool edge = (ty == 0 && top_in) || (ty == kTileH - 1 && bottom_in) || (tx == 0 && left_in) ||
                        (e == kTileW - 1 && right_in);
      if (edge) S.touch[root] = 1;
    }
  }
  __syncthreads();
  // 6. allocate record slots for roots
  for (int p = tid; p < kTilePx; p += kTileThreads) {
    S.slot[p] = -1;
    if (S.d[p] < 0 || S.label[p] != p) continue;
    if (S.touch[p]) S.slot[p] = atomicAdd(&S.n_part, 1);
    else if (S.mom[0][p] >= P.m_min) S.slot[p] = atomicAdd(&S.n_reg, 1);
  }
  __syncthreads();
  if (tid == 0) {
    // one atomic for both record kinds (partials << 32 | regions)
    const unsigned long long old =
        (S.n_part | S.n_reg) ? atomicAdd(P.tile_records, ((unsigned long long)S.n_part << 32) | (unsigned)S.n_reg) : 0ull;
    S.base_part = old >> 32;
    S.base_reg = old & 0xffffffffull;
  }
  __syncthreads();
  for (int p = tid; p < kTilePx; p += kTileThreads) {
    int s = S.slot[p];
    if (s < 0) continue;
    int rx = p % kTileW, ry = p / kTileW;
    long long n = S.mom[0][p], m1 = S.mom[1][p], m2 = S.mom[2][p];
    long long X = x0, Y = y0;
    long long gm[6];
    gm[0] = n;
    gm[1] = m1 + n * X;
    gm[2] = m2 + n * Y;
    gm[3] = (long long)S.mom[3][p] + 2 * X * m1 + n * X * X;
    gm[4] = (long long)S.mom[4][p] + X * m2 + Y * m1 + n * X * Y;
    gm[5] = (long long)S.mom[5][p] + 2 * Y * m2 + n * Y * Y;
    int minpix = (y0 + ry) * W + (x0 + rx);
    if (S.touch[p]) {
      unsigned long long gid = S.base_part + s;
      if ((long long)gid < P.partial_cap) {
        PartialRec& R = P.partials[gid];
        R.view_pos = P.view_offset + v * P.view_stride;
        R.cand = S.d[p];
        R.band = S.band[p];
        R.minpix = minpix;
        for (int k = 0; k < 6; ++k) R.m[k] = gm[k];
        P.partial_parent[gid] = (int)gid;
        S.slot[p] = (int)gid;
      } else {
        atomicOr(P.overflow, 2u);
        S.slot[p] = -1;
      }
    } else {
      unsigned long long rid = S.base_reg + s;
      if ((long long)rid < P.region_cap) {
        RegionRec& R = P.regions[rid];
        R.view_pos = P.view_offset + v * P.view_stride;
        R.cand = S.d[p];
        R.band = S.band[p];
        R.minpix = minpix;
        for (int k = 0; k < 6; ++k) R.m[k] = gm[k];
      } else {
        atomicOr(P.overflow, 1u);
      }
      S.slot[p] = -1;
    }
  }
  __syncthreads();
  // 7. border labels: top, bottom, left, right
  int* border = P.border + (long long)tile * kBorderSlots;
  for (int s = tid; s < kBorderSlots; s += kTileThreads) {
    int tx, ty;
    if (s < kTileW) { tx = s; ty = 0; }
    else if (s < 2 * kTileW) { tx = s - kTileW; ty = kTileH - 1; }
    else if (s < 2 * kTileW + kTileH) { tx = 0; ty = s - 2 * kTileW; }
    else { tx = kTileW - 1; ty = s - 2 * kTileW - kTileH; }
    int p = ty * kTileW + tx;
    int g = -1;
    if (S.d[p] >= 0) g = S.slot[S.label[S.label[p]]];   // pixel -> run start -> root
    border[s] = g;
  }
}

// all tiles (list == nullptr) or the tiles the warp kernel deferred
__global__ void __launch_bounds__(kTileThreads) tile_kernel(TileParams P, const int* list,
                                                            const unsigned long long* n_list) {
  pdl_wait();   // programmatic dependent launch: the previous kernel's results are visible
  extern __shared__ __align__(16) unsigned char smem_raw[];
  TileSmem& S = *reinterpret_cast<TileSmem*>(smem_raw);
  const long long n = list ? (long long)*n_list : (long long)P.tiles_x * P.tiles_y * P.n_views;
  for (long long t = blockIdx.x; t < n; t += gridDim.x) {
    tile_block(P, S, list ? list[t] : (int)t);
    __syncthreads();
  }
}

__device__ __forceinline__ int border_slot(int lx, int ly) {
  if (ly == 0) return lx;
  if (ly == kTileH - 1) return kTileW + lx;
  if (lx == 0) return 2 * kTileW + ly;
  return 2 * kTileW + kTileH + ly;   // lx == kTileW - 1
}

constexpr int kBorderTilesPerBlock = 1;
#ifndef ADPS_BORDER_MATCH
#define ADPS_BORDER_MATCH 1
#endif
#ifndef ADPS_BORDER_GRID3
#define ADPS_BORDER_GRID3 1
#endif
static_assert(!ADPS_BORDER_GRID3 || kBorderTilesPerBlock == 1, "the 3-D border grid is a block per tile");
__global__ void __launch_bounds__(kBorderSlots * kBorderTilesPerBlock) border_kernel(BorderParams P) {
  pdl_wait();   // programmatic dependent launch: the previous kernel's results are visible
  // 128 threads = the tile's border slots; warp w = side w (top, bottom, left,
  // right).  Runs along an edge ask for the same union many times: lanes
  // holding the same (fragment, neighbour fragment) pair unite once (match_any)
  // kBorderTilesPerBlock tiles per block (short blocks: fewer of them to schedule)
#if ADPS_BORDER_GRID3
  // grid (tiles_x, tiles_y, views): the tile coordinates without integer divisions
  const int txi = blockIdx.x, tyi = blockIdx.y, v = blockIdx.z;
  const long long tile = ((long long)v * P.tiles_y + tyi) * P.tiles_x + txi;
#else
  const int tiles_per_view = P.tiles_x * P.tiles_y;
  const long long tile = (long long)blockIdx.x * kBorderTilesPerBlock + threadIdx.x / kBorderSlots;
  if (tile >= P.n_tiles) return;   // warp-uniform
  const int v = (int)(tile / tiles_per_view);
  const int t = (int)(tile % tiles_per_view);
  const int tyi = t / P.tiles_x, txi = t % P.tiles_x;
#endif
  const int s = threadIdx.x % kBorderSlots;
  const int gp = P.border[tile * kBorderSlots + s];
  if (__all_sync(0xffffffffu, gp < 0)) return;   // warp-uniform
  int lx, ly;
  if (s < kTileW) { lx = s; ly = 0; }
  else if (s < 2 * kTileW) { lx = s - kTileW; ly = kTileH - 1; }
  else if (s < 2 * kTileW + kTileH) { lx = 0; ly = s - 2 * kTileW; }
  else { lx = kTileW - 1; ly = s - 2 * kTileW - kTileH; }
  const int x = txi * kTileW + lx, y = tyi * kTileH + ly;
  const int dxs[4] = {1, -1, 0, 1}, dys[4] = {0, 1, 1, 1};   // E, SW, S, SE
  int gqs[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    gqs[k] = -1;
    if (gp < 0) continue;
    const int qx = x + dxs[k], qy = y + dys[k];
    if (qx < 0 || qx >= P.W || qy >= P.H) continue;
    const int qtx = qx / kTileW, qty = qy / kTileH;
    if (qtx == txi && qty == tyi) continue;
    const long long qt = ((long long)v * P.tiles_y + qty) * P.tiles_x + qtx;
    gqs[k] = P.border[qt * kBorderSlots + border_slot(qx - qtx * kTileW, qy - qty * kTileH)];
  }
  const PartialRec* A = gp >= 0 ? &P.partials[gp] : nullptr;
  // every warp-wide exchange first, then the unions: a shuffle after a lane's
  // divergent union-find would run as a split-warp (collective) sequence
  bool go[4];
#if !ADPS_BORDER_MATCH
  const int lgp = __shfl_up_sync(0xffffffffu, gp, 1);
#endif
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    int gq = gqs[k];
    for (int k2 = 0; k2 < k; ++k2)
      if (gqs[k2] == gq) gq = -1;   // the same pair through another direction
    gqs[k] = gq;
#if ADPS_BORDER_MATCH
    // lanes holding the same (fragment, neighbour fragment) pair unite once
    const unsigned long long key = gq >= 0 ? ((unsigned long long)(unsigned)gp << 32) | (unsigned)gq : ~0ull;
    const unsigned peers = __match_any_sync(0xffffffffu, key);
    go[k] = gq >= 0 && (int)(threadIdx.x & 31) == __ffs(peers) - 1;
#else
    // along an edge equal pairs come in runs: skip a lane whose left neighbour
    // holds the same pair (unions are idempotent, so leftover duplicates only cost time)
    const int lgq = __shfl_up_sync(0xffffffffu, gq, 1);
    go[k] = gq >= 0 && !((threadIdx.x & 31) > 0 && lgp == gp && lgq == gq);
#endif
  }
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    if (!go[k]) continue;
    const PartialRec& B = P.partials[gqs[k]];
    if (A->cand == B.cand && A->band == B.band) uf_unite(P.parent, gp, gqs[k]);
  }
}

__global__ void unpack_records_kernel(const unsigned long long* __restrict__ packed,
                                      unsigned long long* __restrict__ n_partials,
                                      unsigned long long* __restrict__ n_regions) {
  pdl_wait();   // programmatic dependent launch: the previous kernel's results are visible
  const unsigned long long v = *packed;
  *n_partials = v >> 32;
  *n_regions = v & 0xffffffffull;
}

__global__ void resolve_kernel(PartialRec* __restrict__ partials, int* __restrict__ parent,
                               const unsigned long long* __restrict__ n_partials, long long cap) {
  pdl_wait();   // programmatic dependent launch: the previous kernel's results are visible
  long long n = (long long)*n_partials;
  if (n > cap) n = cap;
  for (long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x; g < n;
       g += (long long)gridDim.x * blockDim.x) {
    int root = uf_find(parent, (int)g);
    if (root == (int)g) continue;
    PartialRec& R = partials[root];
    const PartialRec& A = partials[g];
    for (int k = 0; k < 6; ++k)
      atomicAdd(reinterpret_cast<unsigned long long*>(&R.m[k]), (unsigned long long)A.m[k]);
    atomicMin(&R.minpix, A.minpix);
  }
}

__global__ void partial_emit_kernel(const PartialRec* __restrict__ partials, const int* __restrict__ parent,
                                    const unsigned long long* __restrict__ n_partials, long long pcap,
                                    int m_min, RegionRec* __restrict__ regions,
                                    unsigned long long* __restrict__ n_regions, long long rcap,
                                    unsigned int* __restrict__ overflow) {
  pdl_wait();   // programmatic dependent launch: the previous kernel's results are visible
  long long n = (long long)*n_partials;
  if (n > pcap) n = pcap;
  for (long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x; g < n;
       g += (long long)gridDim.x * blockDim.x) {
    if (parent[g] != (int)g) continue;
    const PartialRec& A = partials[g];
    if (A.m[0] < m_min) continue;
    unsigned long long rid = atomicAdd(n_regions, 1ull);
    if ((long long)rid >= rcap) {
      atomicOr(overflow, 1u);
      continue;
    }
    RegionRec& R = regions[rid];
    R.view_pos = A.view_pos;
    R.cand = A.cand;
    R.band = A.band;
    R.minpix = A.minpix;
    for (int k = 0; k < 6; ++k) R.m[k] = A.m[k];
  }
}

// --------------------------------------------------------------- launchers
size_t tile_smem_bytes() { return sizeof(TileSmem); }

cudaError_t launch_minmax_kernel(const AttributionArgs& a, int v0, int v1, cudaStream_t s) {
  if (v1 <= v0) return cudaSuccess;
  if (minmax_bulk_ok(a, v0, v1)) return launch_minmax_bulk(a, v0, v1, s);
  const long long hw = (long long)a.H * a.W;
  if (hw % 2 == 0 && hw < (1ll << 30)) {   // pixel pairs (float2 / int2 loads)
    // one wave of resident blocks over the whole launch, each looping over many
    // 512-pixel chunks of its view: the per-block min/max reduction and its
    // barrier are paid once per ~50 chunks instead of every other chunk
    static int per_sm_max = 0, sms = 148;
    if (per_sm_max == 0) {
      int dev = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_max, minmax2_kernel, 256, 0) != cudaSuccess ||
          per_sm_max < 1)
        per_sm_max = 8;
    }
    // fewer than all resident blocks leaves SM room for the CCL of the previous
    // view chunk running concurrently on the second stream
    const int per_sm = a.input_blocks_per_sm > 0 && a.input_blocks_per_sm < per_sm_max ? a.input_blocks_per_sm
                                                                                          : per_sm_max;
    const int resident = per_sm * sms;
    const long long per_view = (hw + 511) / 512;
    // floor: at most one wave (a second, short wave would run whole view slices on a few SMs)
    const long long want = (long long)resident / (v1 - v0);
    dim3 mg2((unsigned)(want < 1 ? 1 : (want > per_view ? per_view : want)), (unsigned)(v1 - v0));
    launch_k(minmax2_kernel, mg2, 256, 0, s, a.image, a.gt, a.dom, (int)hw, a.lohi, a.cls, a.N, a.dom_flag, a.cand_bits,
                                       a.raw, a.rawf, v0);
    return cudaGetLastError();
  }
  dim3 mg((unsigned)((hw + 256 * 8 - 1) / (256 * 8)), (unsigned)(v1 - v0));
  if (mg.x > 1024) mg.x = 1024;
  launch_k(minmax_kernel, mg, 256, 0, s, a.image, a.gt, a.dom, hw, a.lohi, a.cls, a.N, a.dom_flag, a.cand_bits, a.raw,
                                   a.rawf, v0);
  return cudaGetLastError();
}

cudaError_t launch_thresholds(const AttributionArgs& a, int v0, int v1, cudaStream_t s) {
  if (v1 <= v0) return cudaSuccess;
  const int nt = (v1 - v0) * a.L;
  launch_k(thresholds_kernel, (nt + 3) / 4, 128, 0, s, a.lohi, v0, v1 - v0, a.L, a.tau, a.lo, a.thr, a.thr_raw);
  return cudaGetLastError();
}

cudaError_t launch_minmax_views(const AttributionArgs& a, int v0, int v1, cudaStream_t s) {
  cudaError_t e = launch_minmax_kernel(a, v0, v1, s);
  if (e != cudaSuccess) return e;
  return launch_thresholds(a, v0, v1, s);
}

cudaError_t launch_minmax(const AttributionArgs& a, const int* split_list, Counters* ctr, int sm_count,
                          cudaStream_t s) {
  cudaError_t e = launch_minmax_views(a, 0, a.V, s);
  if (e != cudaSuccess) return e;
  launch_k(fallback_count_kernel, sm_count * 2, 256, 0, s, split_list, a.dom_flag, ctr);
  return cudaGetLastError();
}

cudaError_t launch_fallback_count(const int* split_list, const unsigned char* dom_flag, Counters* ctr, int sm_count,
                                  cudaStream_t s) {
  launch_k(fallback_count_kernel, sm_count * 2, 256, 0, s, split_list, dom_flag, ctr);
  return cudaGetLastError();
}

static TileParams tile_params(const AttributionArgs& a) {
  TileParams P;
  P.image = a.image;
  P.gt = a.gt;
  P.dom = a.dom;
  P.H = a.H;
  P.W = a.W;
  P.tiles_x = (a.W + kTileW - 1) / kTileW;
  P.tiles_y = (a.H + kTileH - 1) / kTileH;
  P.view_offset = a.view_offset;
  P.view_stride = a.view_stride;
  P.lo = a.lo;
  P.thr = a.thr;
  P.thr_raw = a.thr_raw;
  P.L = a.L;
  P.r_erode = a.r_erode;
  P.m_min = a.m_min;
  P.cls = a.cls;
  P.N = a.N;
  P.dom_flag = a.dom_flag;
  P.regions = a.regions;
  P.n_regions = a.n_regions;
  P.region_cap = a.region_cap;
  P.partials = a.partials;
  P.n_partials = a.n_partials;
  P.partial_cap = a.partial_cap;
  P.partial_parent = a.partial_parent;
  P.tile_records = a.tile_records;
  P.border = a.border;
  P.dbg_m = a.dbg_m;
  P.dbg_b = a.dbg_b;
  P.overflow = a.overflow;
  P.n_views = a.V;
  P.cand_bits = a.cand_bits;
  P.raw = a.raw;
  P.words = a.words;
  P.rawf = a.rawf;
  P.deferred = a.deferred;
  P.n_deferred = a.n_deferred;
  return P;
}

bool attribution_warp_path(const AttributionArgs& a) {
  // the warp kernel covers r_erode <= 3 without debug maps; the block kernel
  // takes everything else and the tiles the warp kernel defers
  return a.tile_path != 1 && !a.dbg_m && a.r_erode <= 3 && a.deferred && a.n_deferred;
}

cudaError_t launch_tiles_views(const AttributionArgs& a, int v0, int v1, cudaStream_t s) {
  if (!attribution_warp_path(a) || v1 <= v0) return cudaSuccess;
  const TileParams P = tile_params(a);
  if (P.rawf) return launch_tile_bits(P, v0, v1, s);   // bit planes (after the words pass, or fused)
  const long long tpv = (long long)P.tiles_x * P.tiles_y;
  return launch_tile_warp(P, tpv * v0, tpv * v1, s);
}

cudaError_t launch_attribution_tail(const AttributionArgs& a, cudaStream_t s, MarkFn mark, void* ctx) {
  const TileParams P = tile_params(a);
  const long long nblocks = (long long)P.tiles_x * P.tiles_y * a.V;
  size_t smem = sizeof(TileSmem);
  cudaError_t e = cudaFuncSetAttribute(tile_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  if (attribution_warp_path(a) && P.rawf && !ADPS_DEFERRED_BLOCK) {
    // bit-plane path: the deferred tiles by the big-capacity warp kernel
    e = launch_tile_bits_deferred(P, a.grid_small / 2, s);
    if (e != cudaSuccess) return e;
    if (mark) mark(ctx, "tile_ccl", s, a.words ? 3 : 2);
  } else if (attribution_warp_path(a)) {
    launch_k(tile_kernel, a.grid_small, kTileThreads, smem, s, P, a.deferred, a.n_deferred);
    if (mark) mark(ctx, "tile_ccl", s, a.words ? 3 : 2);
  } else {
    launch_k(tile_kernel, (unsigned)nblocks, kTileThreads, smem, s, P, nullptr, nullptr);
    if (mark) mark(ctx, "tile_ccl", s, 1);
  }
  // the tile CCLs' packed record counts into n_partials / n_regions (zero before)
  launch_k(unpack_records_kernel, 1, 1, 0, s, a.tile_records, a.n_partials, a.n_regions);
  BorderParams B;
  B.border = a.border;
  B.partials = a.partials;
  B.parent = a.partial_parent;
  B.tiles_x = P.tiles_x;
  B.tiles_y = P.tiles_y;
  B.W = a.W;
  B.H = a.H;
  B.n_tiles = nblocks;
#if ADPS_BORDER_GRID3
  if (nblocks > 0) launch_k(border_kernel, dim3(P.tiles_x, P.tiles_y, a.V), kBorderSlots, 0, s, B);
#else
  launch_k(border_kernel, (unsigned)((nblocks + kBorderTilesPerBlock - 1) / kBorderTilesPerBlock), kBorderSlots * kBorderTilesPerBlock, 0, s, B);
#endif
  launch_k(resolve_kernel, a.grid_small, 256, 0, s, a.partials, a.partial_parent, a.n_partials, a.partial_cap);
  launch_k(partial_emit_kernel, a.grid_small, 256, 0, s, a.partials, a.partial_parent, a.n_partials, a.partial_cap,
                                                    a.m_min, a.regions, a.n_regions, a.region_cap, a.overflow);
  if (mark) mark(ctx, "border_merge", s, 3);
  return cudaGetLastError();
}

cudaError_t launch_attribution(const AttributionArgs& a, cudaStream_t s, MarkFn mark, void* ctx) {
  cudaError_t e = launch_tiles_views(a, 0, a.V, s);
  if (e != cudaSuccess) return e;
  return launch_attribution_tail(a, s, mark, ctx);
}

}  // namespace adps
