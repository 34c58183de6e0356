// Throughput probe: FFMA (3-register form) vs FFMA2 (packed f32x2, sm_100a) issue rates.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ffma2 ffma2.cu && ./ffma2
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k(float* out, float a, float b, int iters) {
  float x[8], y[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) { x[i] = threadIdx.x * 1e-3f + i; y[i] = x[i] * 0.5f; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) {  // 2 independent scalar FFMAs per pair (register operands)
        x[i] = fmaf(x[i], a, y[i]);
        y[i] = fmaf(y[i], b, x[i]);
      } else {          // one FFMA2 per pair
        unsigned long long xy, ab, yx;
        float2 p = make_float2(x[i], y[i]), q = make_float2(a, b), r = make_float2(y[i], x[i]);
        xy = *reinterpret_cast<unsigned long long*>(&p);
        ab = *reinterpret_cast<unsigned long long*>(&q);
        yx = *reinterpret_cast<unsigned long long*>(&r);
        asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(xy) : "l"(ab), "l"(yx));
        p = *reinterpret_cast<float2*>(&xy);
        x[i] = p.x; y[i] = p.y;
      }
    }
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i] + y[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  float* out;
  cudaMalloc(&out, 148 * 8 * 256 * 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 4096;
  for (int mode = 0; mode < 2; ++mode) {
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(e0);
      if (mode == 0) k<0><<<148 * 8, 256>>>(out, 0.999f, 1.001f, iters);
      else k<1><<<148 * 8, 256>>>(out, 0.999f, 1.001f, iters);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double fmas = 148.0 * 8 * 256 * iters * 16;
      if (rep == 2) printf("%s: %.3f ms, %.1f TFMA/s (%.1f TFLOP/s)\n", mode ? "FFMA2" : "FFMA ", ms, fmas / ms / 1e9, 2 * fmas / ms / 1e9);
    }
  }
  return 0;
}
