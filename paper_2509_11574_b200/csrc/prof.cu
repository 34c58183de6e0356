// prof.cu -- see prof.cuh.
#include <cuda_runtime.h>

#include <mutex>
#include <vector>

#include "common.cuh"
#include "prof.cuh"

namespace gps {
bool g_prof_on = false;
namespace {
const char* kNames[K_COUNT] = {"k_alloc",      "k_integrate", "k_raycast",  "k_preprocess", "k_scan",
                               "k_emit",       "k_sort_blend", "k_backward", "k_adam", "memset", "k_range", "k_link", "k_chain", "k_sort_long", "k_chain_adam"};
struct Pair {
  cudaEvent_t a, b;
  int id;
};
std::mutex g_mu;
std::vector<Pair> g_pairs;      // recorded this session
std::vector<cudaEvent_t> g_pool;
std::vector<int> g_open[K_COUNT];  // index into g_pairs of the open bracket per kernel id
cudaEvent_t take() {
  if (!g_pool.empty()) {
    cudaEvent_t e = g_pool.back();
    g_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}
}  // namespace

void prof_begin(int id, cudaStream_t s) {
  std::lock_guard<std::mutex> l(g_mu);
  Pair p{take(), take(), id};
  cudaEventRecord(p.a, s);
  g_open[id].push_back((int)g_pairs.size());
  g_pairs.push_back(p);
}
void prof_end(int id, cudaStream_t s) {
  std::lock_guard<std::mutex> l(g_mu);
  if (g_open[id].empty()) return;
  const int k = g_open[id].back();
  g_open[id].pop_back();
  cudaEventRecord(g_pairs[k].b, s);
}
}  // namespace gps

extern "C" {
void gps_profile_enable(int on) {
  std::lock_guard<std::mutex> l(gps::g_mu);
  for (auto& p : gps::g_pairs) {
    gps::g_pool.push_back(p.a);
    gps::g_pool.push_back(p.b);
  }
  gps::g_pairs.clear();
  for (auto& o : gps::g_open) o.clear();
  gps::g_prof_on = on != 0;
}

int gps_profile_read_sync(char* names, int names_cap, double* total_ms, int64_t* launches, int cap) {
  std::lock_guard<std::mutex> l(gps::g_mu);
  double t[gps::K_COUNT] = {0};
  int64_t c[gps::K_COUNT] = {0};
  for (auto& p : gps::g_pairs) {
    if (cudaEventSynchronize(p.b) != cudaSuccess) continue;
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, p.a, p.b) == cudaSuccess) {
      t[p.id] += ms;
      c[p.id] += 1;
    }
  }
  const int n = cap < gps::K_COUNT ? cap : gps::K_COUNT;
  std::string all;
  for (int i = 0; i < gps::K_COUNT; ++i) {
    if (i < n) {
      total_ms[i] = t[i];
      launches[i] = c[i];
    }
    all += gps::kNames[i];
    all += ';';
  }
  if (names && names_cap > 0) {
    const size_t m = std::min<size_t>(all.size(), (size_t)names_cap - 1);
    memcpy(names, all.data(), m);
    names[m] = 0;
  }
  return gps::K_COUNT;
}

// per-launch timeline of the session: kernel id and start / end in ms from the session's first
// event (all launches, in enqueue order); returns the number of launches recorded
int64_t gps_profile_timeline_sync(int32_t* ids, double* t0_ms, double* t1_ms, int64_t cap) {
  std::lock_guard<std::mutex> l(gps::g_mu);
  if (gps::g_pairs.empty()) return 0;
  cudaEvent_t base = gps::g_pairs.front().a;
  int64_t n = 0;
  for (auto& p : gps::g_pairs) {
    if (cudaEventSynchronize(p.b) != cudaSuccess) continue;
    float a = 0.f, b = 0.f;
    if (cudaEventElapsedTime(&a, base, p.a) != cudaSuccess || cudaEventElapsedTime(&b, base, p.b) != cudaSuccess) continue;
    if (n < cap) {
      ids[n] = p.id;
      t0_ms[n] = a;
      t1_ms[n] = b;
    }
    ++n;
  }
  return n;
}
}
