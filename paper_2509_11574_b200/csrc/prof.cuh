// prof.cuh -- optional per-kernel CUDA-event timing inside libgps (gps_profile_*).  When enabled,
// every kernel launch is bracketed by two events recorded on its launch stream; reading the
// totals synchronises.  Disabled (the default) it costs one branch per launch.
#pragma once
#include <cuda_runtime.h>

namespace gps {
enum KernelId {
  K_ALLOC = 0, K_INTEGRATE, K_RAYCAST, K_PREPROCESS, K_SCAN, K_EMIT, K_SORT_BLEND, K_BACKWARD, K_GRAD_ADAM,
  K_MEMSET, K_RANGE, K_LINK, K_CHAIN, K_SORT_LONG, K_CHAIN_ADAM, K_COUNT
};
extern bool g_prof_on;
void prof_begin(int id, cudaStream_t s);
void prof_end(int id, cudaStream_t s);
struct ProfScope {
  int id;
  cudaStream_t s;
  ProfScope(int i, cudaStream_t st) : id(i), s(st) {
    if (g_prof_on) prof_begin(id, s);
  }
  ~ProfScope() {
    if (g_prof_on) prof_end(id, s);
  }
};
}  // namespace gps
#define GPS_PROF(id, stream) ::gps::ProfScope gps_prof_scope_##__LINE__(::gps::id, stream)
