#pragma once

#include <cuda_runtime.h>

namespace adps {

// numpy Generator(PCG64).standard_normal(n) on the device, bit-identical.
// The fallback children of ref/adc.py:97 draw rng.normal(size=(k, 3)) per
// parent; those draws are one contiguous slice of the Generator's normal
// stream, which this reproduces from the bit generator's 128-bit state.
struct NormalsArgs {
  unsigned long long state_lo, state_hi, inc_lo, inc_hi;
  long long n;               // normals wanted
  long long window;          // stream positions examined (>= expected consumption)
  double* out;               // [n]
  // scratch, [window] each
  double* val;
  unsigned char* len;
  unsigned char* acc;
  int* reach;
  int* reach_max;
  unsigned char* walked;
  int* emit_idx;
  // results (device): 64-bit draws consumed, status bits (1 = a comparison
  // too close to call against the host libm, 2 = window too short)
  unsigned long long* consumed;
  unsigned int* status;
};

long long normals_window(long long n);
size_t normals_temp_bytes(long long window);
cudaError_t launch_normals(const NormalsArgs& a, void* temp, size_t temp_bytes, cudaStream_t s);

}  // namespace adps
