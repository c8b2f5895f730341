// PDL probe (dev tool): a chain of dependent latency-bound kernels, launched
// plainly vs with programmatic stream serialization (griddepcontrol.wait at
// kernel start, launch_dependents after the main loop).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void step_kernel(const float* __restrict__ in, float* __restrict__ out, int n, int iters, int pdl) {
  if (pdl == 3) asm volatile("griddepcontrol.launch_dependents;");
  if (pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
  float acc = 0.f;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    float v = in[i];
    for (int k = 0; k < iters; ++k) v = v * 1.0001f + 0.5f;
    out[i] = v;
    acc += v;
  }
  if (pdl == 1) asm volatile("griddepcontrol.launch_dependents;");
  if (acc == -1.f) out[0] = acc;
}

int main() {
  const int n = 1 << 20, chain = 60;
  float *a, *b;
  cudaMalloc(&a, n * 4);
  cudaMalloc(&b, n * 4);
  cudaMemset(a, 0, n * 4);
  cudaStream_t s;
  cudaStreamCreate(&s);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int grid : {148, 592, 4096}) {
    for (int iters : {4, 64}) {
      for (int pdl = 0; pdl < 4; ++pdl) {   // 0 plain, 1 trigger at end, 2 no trigger, 3 trigger at start
        float best = 1e9;
        for (int rep = 0; rep < 5; ++rep) {
          cudaEventRecord(e0, s);
          for (int c = 0; c < chain; ++c) {
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(grid);
            cfg.blockDim = dim3(256);
            cfg.stream = s;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            at[0].val.programmaticStreamSerializationAllowed = 1;
            cfg.attrs = at;
            cfg.numAttrs = pdl ? 1 : 0;
            const float* in = (c & 1) ? b : a;
            float* out = (c & 1) ? a : b;
            cudaLaunchKernelEx(&cfg, step_kernel, in, out, n, iters, pdl);
          }
          cudaEventRecord(e1, s);
          cudaEventSynchronize(e1);
          float ms;
          cudaEventElapsedTime(&ms, e0, e1);
          if (ms < best) best = ms;
        }
        printf("grid %5d iters %3d pdl %d: %.3f ms for %d kernels (%.2f us each)\n", grid, iters, pdl, best, chain,
               best * 1000 / chain);
      }
    }
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
