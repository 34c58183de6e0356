// Throughput probe (sm_100a): independent FFMA vs FFMA2 (__ffma2_rn), alone and interleaved with
// integer ALU work, to decide whether packed fp32 pays in issue-bound kernels.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ffma2b tools/probes/ffma2b.cu && /tmp/ffma2b
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k(float* out, float a, float b, int iters) {
  float x[16];
  unsigned u[4];
#pragma unroll
  for (int i = 0; i < 16; ++i) x[i] = threadIdx.x * 1e-3f + i;
#pragma unroll
  for (int i = 0; i < 4; ++i) u[i] = threadIdx.x + i;
  for (int it = 0; it < iters; ++it) {
    if (MODE == 0 || MODE == 2) {
#pragma unroll
      for (int i = 0; i < 16; ++i) x[i] = fmaf(x[i], a, b);
    } else {
#pragma unroll
      for (int i = 0; i < 16; i += 2) {
        float2 r = __ffma2_rn(make_float2(x[i], x[i + 1]), make_float2(a, a), make_float2(b, b));
        x[i] = r.x; x[i + 1] = r.y;
      }
    }
    if (MODE >= 2) {
#pragma unroll
      for (int i = 0; i < 4; ++i) u[i] = (u[i] * 1664525u + 1013904223u) ^ (u[i] >> 7);
    }
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s + (float)(u[0] ^ u[1] ^ u[2] ^ u[3]);
}

int main() {
  float* out;
  cudaMalloc(&out, 148 * 8 * 256 * 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 8192;
  const char* names[4] = {"FFMA x16", "FFMA2 x8", "FFMA x16 + 8 int", "FFMA2 x8 + 8 int"};
  for (int mode = 0; mode < 4; ++mode) {
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(e0);
      if (mode == 0) k<0><<<148 * 8, 256>>>(out, 0.999f, 1e-3f, iters);
      if (mode == 1) k<1><<<148 * 8, 256>>>(out, 0.999f, 1e-3f, iters);
      if (mode == 2) k<2><<<148 * 8, 256>>>(out, 0.999f, 1e-3f, iters);
      if (mode == 3) k<3><<<148 * 8, 256>>>(out, 0.999f, 1e-3f, iters);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double fmas = 148.0 * 8 * 256 * iters * 16;
      if (rep == 2) printf("%-18s: %.3f ms, %.1f T fp32-FMA/s\n", names[mode], ms, fmas / ms / 1e9);
    }
  }
  return 0;
}
