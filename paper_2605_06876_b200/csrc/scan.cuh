// Single-pass exclusive scan with decoupled look-back.
//
// Used for every offset computation of the step (ref/adc.py:229-244
// compaction, split/clone lists of ref/adc.py:82-89, per-candidate insert
// offsets).  Values are uint64 "lanes": several independent counters can be
// packed into one word (e.g. two 31-bit counts) and scanned together because
// the operator is plain integer addition.
#pragma once

#include "adps_internal.cuh"

namespace adps {

constexpr int kScanThreads = 256;
#ifndef ADPS_SCAN_ITEMS
#define ADPS_SCAN_ITEMS 8
#endif
constexpr int kScanItems = ADPS_SCAN_ITEMS;
constexpr int kScanTile = kScanThreads * kScanItems;
#ifndef ADPS_SCAN_LB
#define ADPS_SCAN_LB 4   // predecessors per lane per look-back round
#endif

// Tile flags carry the launch's epoch (flag = epoch << 2 | state), so a flag
// left by an earlier scan over the same buffers reads as empty: no reset
// between scans (the memsets were two extra stream operations per scan, and
// they break the programmatic-launch chain).  Tile id = blockIdx.x: blocks
// are dispatched in index order, so every predecessor a tile waits on has
// been scheduled.
struct ScanState {
  unsigned long long* value;  // [2 * n_tiles]: aggregate at [2t], inclusive prefix at [2t+1]
  unsigned int* flag;         // [n_tiles] epoch << 2 | 0 empty, 1 aggregate ready, 2 inclusive ready
  unsigned int* epoch_host;   // host counter: each launch takes the next epoch
  unsigned int epoch;         // this launch's epoch (set by launch_scan)
};
constexpr unsigned kScanEpochMask = 0x3fffffffu;

// Policy requirements:
//   __device__ unsigned long long value(long long i) const;
//   __device__ void store(long long i, unsigned long long exclusive, unsigned long long v) const;
//   __device__ void total(unsigned long long t) const;   // called once by the last tile
template <class Policy>
__global__ void __launch_bounds__(kScanThreads) scan_kernel(Policy pol, long long n, ScanState st) {
  pdl_wait();   // programmatic dependent launch: the previous kernel's results are visible
  __shared__ unsigned long long sv[kScanTile];
  __shared__ unsigned long long warp_sums[kScanThreads / kWarp];
  __shared__ unsigned long long s_prefix;
  const int tid = threadIdx.x;
  const long long tile = blockIdx.x;
  const unsigned ep = st.epoch << 2;
  const long long base = tile * kScanTile;
  // striped, coalesced load
#pragma unroll
  for (int j = 0; j < kScanItems; ++j) {
    long long i = base + j * kScanThreads + tid;
    sv[j * kScanThreads + tid] = (i < n) ? pol.value(i) : 0ull;
  }
  __syncthreads();
  unsigned long long loc[kScanItems];
  unsigned long long run = 0;
#pragma unroll
  for (int j = 0; j < kScanItems; ++j) {
    loc[j] = sv[tid * kScanItems + j];
    run += loc[j];
  }
  // block exclusive scan of per-thread sums
  const int lane = tid & 31, wid = tid >> 5;
  unsigned long long incl = run;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    unsigned long long y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) warp_sums[wid] = incl;
  __syncthreads();
  if (wid == 0) {
    unsigned long long w = lane < kScanThreads / kWarp ? warp_sums[lane] : 0ull;
    unsigned long long wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      unsigned long long y = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += y;
    }
    if (lane < kScanThreads / kWarp) warp_sums[lane] = wi - w;  // exclusive
  }
  __syncthreads();
  const unsigned long long thread_excl = warp_sums[wid] + incl - run;
  __shared__ unsigned long long s_agg;
  if (tid == kScanThreads - 1) s_agg = thread_excl + run;
  __syncthreads();
  // decoupled look-back by the last warp, 32 predecessors per round: each lane
  // reads one predecessor's flag; the nearest inclusive prefix ends the walk,
  // aggregates before it are summed with a warp reduction
  if (wid == kScanThreads / kWarp - 1) {
    const unsigned long long agg = s_agg;
    volatile unsigned long long* vval = st.value;
    volatile unsigned int* vflag = st.flag;
    // The aggregate and the inclusive prefix live in separate words: a reader
    // that saw flag==1 must never pick up the later inclusive value.
    if (tile == 0) {
      if (lane == 0) {
        vval[1] = agg;
        __threadfence();
        vflag[0] = ep | 2u;
        s_prefix = 0ull;
      }
    } else {
      if (lane == 0) {
        vval[2 * tile] = agg;
        __threadfence();
        vflag[tile] = ep | 1u;
      }
      // 128 predecessors per round (4 per lane, nearest first: q = p - lane - 32 j):
      // inclusive prefixes propagate 128 tiles per round instead of 32
      unsigned long long acc = 0ull;
      long long p = tile - 1;
      while (true) {
        constexpr int LB = ADPS_SCAN_LB;
        unsigned int f[LB];
        bool busy;
        do {
          busy = false;
#pragma unroll
          for (int j = 0; j < LB; ++j) {
            const long long q = p - lane - 32 * j;
            const unsigned fv = q >= 0 ? vflag[q] : (ep | 2u);
            f[j] = (fv & ~3u) == ep ? (fv & 3u) : 0u;   // another launch's flag: empty
            busy |= f[j] == 0u;
          }
        } while (__any_sync(0xffffffffu, busy));
        __threadfence();
        unsigned incl[LB];
#pragma unroll
        for (int j = 0; j < LB; ++j) incl[j] = __ballot_sync(0xffffffffu, f[j] == 2u);
        // the nearest predecessor with an inclusive prefix: slot (jf, first)
        int jf = LB, first = 32;
#pragma unroll
        for (int j = LB - 1; j >= 0; --j)
          if (incl[j]) {
            jf = j;
            first = __ffs(incl[j]) - 1;
          }
        unsigned long long v = 0ull;
#pragma unroll
        for (int j = 0; j < LB; ++j) {
          const long long q = p - lane - 32 * j;
          if (j < jf || (j == jf && lane < first)) v += vval[2 * q];
          else if (j == jf && lane == first && q >= 0) v += vval[2 * q + 1];
        }
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        acc += v;
        if (jf < LB) break;
        p -= 32 * LB;
      }
      if (lane == 0) {
        vval[2 * tile + 1] = acc + agg;
        __threadfence();
        vflag[tile] = ep | 2u;
        s_prefix = acc;
      }
    }
    if (lane == 0 && base + kScanTile >= n) pol.total(s_prefix + agg);
  }
  __syncthreads();
  // exclusive prefixes back through shared memory, so the stores are striped
  // (coalesced) like the loads; an item's value is the next prefix minus its own
  unsigned long long e = s_prefix + thread_excl;
#pragma unroll
  for (int j = 0; j < kScanItems; ++j) {
    sv[tid * kScanItems + j] = e;
    e += loc[j];
  }
  __syncthreads();
  const unsigned long long end = s_prefix + s_agg;
#pragma unroll
  for (int j = 0; j < kScanItems; ++j) {
    const int k = j * kScanThreads + tid;
    const long long i = base + k;
    if (i < n) {
      const unsigned long long ex = sv[k];
      pol.store(i, ex, (k + 1 < kScanTile ? sv[k + 1] : end) - ex);
    }
  }
}

inline long long scan_tiles(long long n) { return n <= 0 ? 1 : (n + kScanTile - 1) / kScanTile; }

// Launch helper: state buffers must hold scan_tiles(n) entries.
template <class Policy>
inline cudaError_t launch_scan(const Policy& pol, long long n, ScanState st, cudaStream_t s) {
  long long tiles = scan_tiles(n);
  do st.epoch = ++*st.epoch_host & kScanEpochMask;
  while (st.epoch == 0);   // epoch 0 is the zeroed buffer's
  launch_k(scan_kernel<Policy>, (unsigned)tiles, kScanThreads, 0, s, pol, n, st);
  return cudaGetLastError();
}

}  // namespace adps
