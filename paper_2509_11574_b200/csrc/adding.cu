// adding.cu -- Gaussian adding and removal for sm_100a:
// gps_vertex_normals, gps_add_gaussians_sync, gps_remove_gaussians_sync.
//
// Paper: GPS-SLAM (arXiv 2509.11574).  Normal map N* of the raycast; Gaussian adding
// Eq. 6, 25% sampling and initialisation, kNN scales (App. A);
// Gaussian removal Eq. 8.  Readings R-NORMAL, R-ADD-MASK, R-SAMPLE, R-KNN, R-INIT,
// R-REMOVE: DESIGN.md §3; the fp32 decision sequences: DESIGN.md §4.5.
//
// Adding, per round:
//   k_add_flags     per pixel: the Eq. 6 mask bit and the sampling bit; per-CTA counts
//   k_scan_blocks   one CTA: exclusive scan of the per-CTA counts (row-major order is kept)
//   k_add_compact   per CTA: mask pixels -> mpix[], sampled pixels -> spix[] (row-major)
//   k_knn_insert    mask vertices into a hashed uniform grid (cell -> linked list of vertices)
//   k_add_init      per sampled pixel: exact 3-NN by growing shells of cells, then the new
//                   Gaussian's parameters at index n + rank, Adam moments zeroed
// Removal: k_remove_flags (+ k_scan_blocks) -> k_remove_scatter into a staging copy, copied back.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <string>

#define GPS_CHK_VAR g_chk_adding
#include "common.cuh"

namespace gps {
__device__ unsigned long long g_chk_adding = 0ull;
unsigned long long check_word_take_adding() {
  unsigned long long w = 0ull, z = 0ull;
  cudaMemcpyFromSymbol(&w, g_chk_adding, sizeof(w));
  cudaMemcpyToSymbol(g_chk_adding, &z, sizeof(z));
  return w;
}
namespace {

constexpr int kBlk = 1024;                // items per CTA of the flag / compaction passes
constexpr uint32_t kKnnSlots = 1u << 21;  // kNN grid hash slots (cells), power of two
constexpr float kC0 = 0.28209479177387814f;

__device__ __forceinline__ uint32_t hash32(uint32_t x) {  // lowbias32 (R-SAMPLE)
  x ^= x >> 16;
  x *= 0x7FEB352Du;
  x ^= x >> 15;
  x *= 0x846CA68Bu;
  x ^= x >> 16;
  return x;
}
uint32_t hash32_host(uint32_t x) {
  x ^= x >> 16;
  x *= 0x7FEB352Du;
  x ^= x >> 15;
  x *= 0x846CA68Bu;
  x ^= x >> 16;
  return x;
}

// ---- normals (R-NORMAL) ----------------------------------------------------------------------
__global__ void k_vertex_normals(int W, int H, const float* __restrict__ depth, const float* __restrict__ V,
                                 float cx, float cy, float cz, float* __restrict__ N,
                                 const float* __restrict__ dpose = nullptr) {
  const int u = blockIdx.x * 16 + (threadIdx.x & 15), v = blockIdx.y * 16 + (threadIdx.x >> 4);
  if (dpose) {  // camera centre t from a device pose (gps_vertex_normals_dpose)
    cx = __ldg(dpose + 9);
    cy = __ldg(dpose + 10);
    cz = __ldg(dpose + 11);
  }
  if (u >= W || v >= H) return;
  const size_t p = (size_t)v * W + u;
  float n0 = 0.f, n1 = 0.f, n2 = 0.f;
  if (u > 0 && v > 0 && u < W - 1 && v < H - 1 && depth[p] > 0.f && depth[p - 1] > 0.f && depth[p + 1] > 0.f &&
      depth[p - W] > 0.f && depth[p + W] > 0.f) {
    const float* a = V + 3 * (p + 1);
    const float* b = V + 3 * (p - 1);
    const float* c = V + 3 * (p + W);
    const float* d = V + 3 * (p - W);
    const float dx0 = a[0] - b[0], dx1 = a[1] - b[1], dx2 = a[2] - b[2];
    const float dy0 = c[0] - d[0], dy1 = c[1] - d[1], dy2 = c[2] - d[2];
    const float c0 = dx1 * dy2 - dx2 * dy1, c1 = dx2 * dy0 - dx0 * dy2, c2 = dx0 * dy1 - dx1 * dy0;
    const float nn = sqrtf(c0 * c0 + c1 * c1 + c2 * c2);
    if (nn > 0.f) {
      const float s = 1.0f / nn;
      n0 = c0 * s; n1 = c1 * s; n2 = c2 * s;
      const float* q = V + 3 * p;
      if (n0 * (q[0] - cx) + n1 * (q[1] - cy) + n2 * (q[2] - cz) > 0.f) {  // face the camera
        n0 = -n0; n1 = -n1; n2 = -n2;
      }
    }
  }
  N[3 * p] = n0; N[3 * p + 1] = n1; N[3 * p + 2] = n2;
}

// ---- block-level compaction helpers ---------------------------------------------------------
// exclusive rank of this thread's predicate inside its CTA of kBlk threads (and the CTA total)
__device__ __forceinline__ uint32_t cta_rank(bool pred, uint32_t* swarp, uint32_t& total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint32_t b = __ballot_sync(0xFFFFFFFFu, pred);
  const uint32_t lo = __popc(b & ((1u << lane) - 1u));
  if (lane == 0) swarp[w] = __popc(b);
  __syncthreads();
  if (w == 0) {
    uint32_t x = swarp[lane], incl = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
      if (lane >= o) incl += y;
    }
    swarp[32 + lane] = incl - x;
    if (lane == 31) swarp[64] = incl;
  }
  __syncthreads();
  total = swarp[64];
  const uint32_t r = swarp[32 + w] + lo;
  __syncthreads();
  return r;
}

// in-place exclusive scan of narr arrays of nblk counts each (one CTA of 1024 threads); the
// totals land in totals[arr]
__global__ void __launch_bounds__(1024) k_scan_blocks(uint32_t* cnt, int nblk, int narr, uint32_t* totals) {
  __shared__ uint32_t sw[32];
  __shared__ uint32_t carry;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int a = 0; a < narr; ++a) {
    uint32_t* c = cnt + (size_t)a * nblk;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int base = 0; base < nblk; base += 1024) {
      const int i = base + threadIdx.x;
      const uint32_t x = i < nblk ? c[i] : 0u;
      uint32_t incl = x;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
        if (lane >= o) incl += y;
      }
      if (lane == 31) sw[w] = incl;
      __syncthreads();
      if (w == 0) {
        uint32_t s = sw[lane];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, s, o);
          if (lane >= o) s += y;
        }
        sw[lane] = s;
      }
      __syncthreads();
      const uint32_t ex = carry + (w ? sw[w - 1] : 0u) + incl - x;
      if (i < nblk) c[i] = ex;
      __syncthreads();
      if (threadIdx.x == 1023) carry = ex + x;
      __syncthreads();
    }
    if (threadIdx.x == 0) totals[a] = carry;
    __syncthreads();
  }
}

// ---- adding ----------------------------------------------------------------------------------
struct AddArgs {
  int W, H;
  float delta_c, delta_w, inv255;
  uint32_t seed_h;        // hash32(seed)
  unsigned long long thr; // floor(sample_frac * 2^32)
  int nblk;
};

// Eq. 6 mask (R-ADD-MASK, fp32: C_k = c8 * fl(1/255), d = |C* - C_k|, d > fl(delta_c), W_G <
// fl(delta_W)) and the sampling bit (R-SAMPLE); per-CTA counts of both
__global__ void __launch_bounds__(kBlk) k_add_flags(AddArgs a, const float* __restrict__ depth,
                                                    const float* __restrict__ normal, const float* __restrict__ cstar,
                                                    const float* __restrict__ wg, const uint32_t* __restrict__ tgt,
                                                    uint8_t* flags, uint32_t* bcnt) {
  const uint32_t n = (uint32_t)a.W * (uint32_t)a.H;
  const uint32_t p = blockIdx.x * kBlk + threadIdx.x;
  bool m = false, s = false;
  if (p < n && depth[p] > 0.f) {
    const float* nm = normal + 3 * (size_t)p;
    const bool hasn = (fabsf(nm[0]) + fabsf(nm[1]) + fabsf(nm[2])) > 0.f;
    const uint32_t c = tgt[p];
    bool big = false;
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) {
      const float ck = __fmul_rn((float)((c >> (8 * ch)) & 0xFFu), a.inv255);
      big |= fabsf(__fsub_rn(cstar[3 * (size_t)p + ch], ck)) > a.delta_c;
    }
    m = hasn && big && wg[p] < a.delta_w;
    s = m && (unsigned long long)hash32(p ^ a.seed_h) < a.thr;
  }
  if (p < n) flags[p] = (uint8_t)(m | (s << 1));
  const int cm = __syncthreads_count(m), cs = __syncthreads_count(s);
  if (threadIdx.x == 0) {
    bcnt[blockIdx.x] = (uint32_t)cm;
    bcnt[a.nblk + blockIdx.x] = (uint32_t)cs;
  }
}

// row-major compaction: mask pixels -> mpix, sampled pixels -> spix (+ their index in mpix)
__global__ void __launch_bounds__(kBlk) k_add_compact(AddArgs a, const uint8_t* __restrict__ flags,
                                                      const uint32_t* __restrict__ boff, uint32_t* mpix,
                                                      uint32_t* spix, uint32_t* smi) {
  __shared__ uint32_t sw[72];
  const uint32_t n = (uint32_t)a.W * (uint32_t)a.H;
  const uint32_t p = blockIdx.x * kBlk + threadIdx.x;
  const uint8_t f = p < n ? flags[p] : (uint8_t)0;
  uint32_t tm, ts;
  const uint32_t rm = cta_rank(f & 1, sw, tm);
  const uint32_t rs = cta_rank((f >> 1) & 1, sw, ts);
  GPS_DCHECK(!(f & 1) || boff[blockIdx.x] + rm < n, CHK_ADD);
  if (f & 1) mpix[boff[blockIdx.x] + rm] = p;
  if (f & 2) {
    const uint32_t at = boff[a.nblk + blockIdx.x] + rs;
    GPS_DCHECK(at <= boff[blockIdx.x] + rm && at < n, CHK_ADD);
    spix[at] = p;
    smi[at] = boff[blockIdx.x] + rm;
  }
}

__device__ __forceinline__ uint64_t cell_key(int x, int y, int z) { return pack_block(x, y, z); }

__global__ void k_fill_keys(uint64_t* p, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    p[i] = kEmptyKey;
}

__global__ void k_knn_insert(const uint32_t* __restrict__ mpix, uint32_t M, const float* __restrict__ V,
                             float inv_cell, uint64_t* keys, int32_t* heads, int32_t* next) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= M) return;
  const float* q = V + 3 * (size_t)mpix[i];
  const int x = (int)floorf(q[0] * inv_cell), y = (int)floorf(q[1] * inv_cell), z = (int)floorf(q[2] * inv_cell);
  const uint64_t key = cell_key(x, y, z);
  uint32_t h = hash_block(x, y, z) & (kKnnSlots - 1);
  for (uint32_t probe = 0; probe < kKnnSlots; ++probe) {
    const unsigned long long old = atomicCAS((unsigned long long*)&keys[h], (unsigned long long)kEmptyKey,
                                             (unsigned long long)key);
    if (old == kEmptyKey || old == key) {
      next[i] = atomicExch(&heads[h], (int32_t)i);
      return;
    }
    h = (h + 1) & (kKnnSlots - 1);
  }
}

__device__ __forceinline__ int32_t knn_slot(const uint64_t* __restrict__ keys, int x, int y, int z) {
  const uint64_t key = cell_key(x, y, z);
  uint32_t h = hash_block(x, y, z) & (kKnnSlots - 1);
  for (uint32_t probe = 0; probe < kKnnSlots; ++probe) {
    const uint64_t k = __ldg(&keys[h]);
    if (k == key) return (int32_t)h;
    if (k == kEmptyKey) return -1;
    h = (h + 1) & (kKnnSlots - 1);
  }
  return -1;
}

struct InitArgs {
  int64_t n0;         // first new Gaussian's index
  uint32_t count;     // Gaussians to write
  int nsh;            // SH floats per Gaussian
  float inv_cell, cell, rcap, scale_max, opacity_raw, inv255;
  int rmax;
};

// R-KNN + R-INIT for sampled pixel q
__global__ void k_add_init(InitArgs a, const uint32_t* __restrict__ spix, const uint32_t* __restrict__ smi,
                           const uint32_t* __restrict__ mpix, const float* __restrict__ V,
                           const float* __restrict__ N, const uint32_t* __restrict__ tgt,
                           const uint64_t* __restrict__ keys, const int32_t* __restrict__ heads,
                           const int32_t* __restrict__ next, gps_gaussians g, gps_gaussians gm, gps_gaussians gv) {
  const uint32_t q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= a.count) return;
  const uint32_t pix = spix[q];
  const int32_t self = (int32_t)smi[q];
  const float px = V[3 * (size_t)pix], py = V[3 * (size_t)pix + 1], pz = V[3 * (size_t)pix + 2];
  const int cx = (int)floorf(px * a.inv_cell), cy = (int)floorf(py * a.inv_cell), cz = (int)floorf(pz * a.inv_cell);
  float bd[3] = {INFINITY, INFINITY, INFINITY};
  int32_t bi[3] = {-1, -1, -1};
  for (int R = 0; R <= a.rmax; ++R) {
    for (int dz = -R; dz <= R; ++dz)
      for (int dy = -R; dy <= R; ++dy)
        for (int dx = -R; dx <= R; ++dx) {
          if (max(abs(dx), max(abs(dy), abs(dz))) != R) continue;  // shell R only
          const int32_t slot = knn_slot(keys, cx + dx, cy + dy, cz + dz);
          if (slot < 0) continue;
          for (int32_t j = __ldg(&heads[slot]); j >= 0; j = __ldg(&next[j])) {
            if (j == self) continue;
            const float* o = V + 3 * (size_t)__ldg(&mpix[j]);
            const float ex = o[0] - px, ey = o[1] - py, ez = o[2] - pz;
            const float d = ex * ex + ey * ey + ez * ez;
            // keep the 3 smallest (d, index) pairs
            if (d < bd[2] || (d == bd[2] && j < bi[2])) {
              bd[2] = d; bi[2] = j;
              if (bd[2] < bd[1] || (bd[2] == bd[1] && bi[2] < bi[1])) {
                float t = bd[1]; bd[1] = bd[2]; bd[2] = t;
                int32_t u = bi[1]; bi[1] = bi[2]; bi[2] = u;
                if (bd[1] < bd[0] || (bd[1] == bd[0] && bi[1] < bi[0])) {
                  t = bd[0]; bd[0] = bd[1]; bd[1] = t;
                  u = bi[0]; bi[0] = bi[1]; bi[1] = u;
                }
              }
            }
          }
        }
    // every vertex outside shells 0..R lies at least R cells away
    const float reach = (float)R * a.cell;
    if (bi[2] >= 0 && bd[2] <= reach * reach) break;
    if (reach >= a.rcap) break;
  }
  // fewer than 3 found within rcap, or a 3rd distance beyond it: the RMS is >= scale_max
  float s1 = a.scale_max;
  if (bi[2] >= 0) s1 = fminf(a.scale_max, sqrtf((bd[0] + bd[1] + bd[2]) * (1.0f / 3.0f)));
  const int64_t i = a.n0 + q;
  g.xyz[3 * i] = px; g.xyz[3 * i + 1] = py; g.xyz[3 * i + 2] = pz;
  const float ls = logf(s1);
  g.log_scale[3 * i] = ls; g.log_scale[3 * i + 1] = ls; g.log_scale[3 * i + 2] = logf(0.1f * s1);
  // shortest rotation taking e_z to n: (1 + n_z, -n_y, n_x, 0), normalised; n = -e_z: half-turn about e_x
  const float nx = N[3 * (size_t)pix], ny = N[3 * (size_t)pix + 1], nz = N[3 * (size_t)pix + 2];
  float w = 1.0f + nz, x = -ny, y = nx, z = 0.f;
  if (!(w > 1e-6f)) { w = 0.f; x = 1.f; y = 0.f; }
  const float inv = rsqrtf(w * w + x * x + y * y + z * z);
  g.rot[4 * i] = w * inv; g.rot[4 * i + 1] = x * inv; g.rot[4 * i + 2] = y * inv; g.rot[4 * i + 3] = z * inv;
  g.opacity_raw[i] = a.opacity_raw;
  const uint32_t c = tgt[pix];
  float* sh = g.sh + (size_t)i * a.nsh;
  for (int k = 0; k < a.nsh; ++k) sh[k] = 0.f;
#pragma unroll
  for (int ch = 0; ch < 3; ++ch) sh[ch] = ((float)((c >> (8 * ch)) & 0xFFu) * a.inv255 - 0.5f) * (1.0f / kC0);
  // fresh Adam moments
  gps_gaussians mv[2] = {gm, gv};
#pragma unroll
  for (int t = 0; t < 2; ++t) {
    for (int k = 0; k < 3; ++k) { mv[t].xyz[3 * i + k] = 0.f; mv[t].log_scale[3 * i + k] = 0.f; }
    for (int k = 0; k < 4; ++k) mv[t].rot[4 * i + k] = 0.f;
    mv[t].opacity_raw[i] = 0.f;
    float* m = mv[t].sh + (size_t)i * a.nsh;
    for (int k = 0; k < a.nsh; ++k) m[k] = 0.f;
  }
}

// ---- removal (R-REMOVE) ------------------------------------------------------------------------
__global__ void __launch_bounds__(kBlk) k_remove_flags(gps_gaussians g, float t_op, float t_max, float t_min,
                                                       uint8_t* keep, uint32_t* bcnt) {
  const int64_t i = (int64_t)blockIdx.x * kBlk + threadIdx.x;
  bool k = false;
  if (i < g.n) {
    const float o = g.opacity_raw[i];
    const float mx = fmaxf(g.log_scale[3 * i], fmaxf(g.log_scale[3 * i + 1], g.log_scale[3 * i + 2]));
    k = !(o < t_op || mx > t_max || mx < t_min);
    keep[i] = (uint8_t)k;
  }
  const int c = __syncthreads_count(k);
  if (threadIdx.x == 0) bcnt[blockIdx.x] = (uint32_t)c;
}

__device__ __forceinline__ void copy_row(const gps_gaussians& s, const gps_gaussians& d, int64_t i, int64_t j, int nsh) {
  for (int k = 0; k < 3; ++k) { d.xyz[3 * j + k] = s.xyz[3 * i + k]; d.log_scale[3 * j + k] = s.log_scale[3 * i + k]; }
  for (int k = 0; k < 4; ++k) d.rot[4 * j + k] = s.rot[4 * i + k];
  d.opacity_raw[j] = s.opacity_raw[i];
  for (int k = 0; k < nsh; ++k) d.sh[(size_t)j * nsh + k] = s.sh[(size_t)i * nsh + k];
}

__global__ void __launch_bounds__(kBlk) k_remove_scatter(gps_gaussians g, gps_gaussians gm, gps_gaussians gv,
                                                         const uint8_t* __restrict__ keep,
                                                         const uint32_t* __restrict__ boff, gps_gaussians sp,
                                                         gps_gaussians sm, gps_gaussians sv, int nsh) {
  __shared__ uint32_t sw[72];
  const int64_t i = (int64_t)blockIdx.x * kBlk + threadIdx.x;
  const bool k = i < g.n && keep[i];
  uint32_t tot;
  const uint32_t r = cta_rank(k, sw, tot);
  if (!k) return;
  const int64_t j = boff[blockIdx.x] + r;
  GPS_DCHECK(j <= i, CHK_ADD);  // a stable compaction never moves a row forward
  copy_row(g, sp, i, j, nsh);
  copy_row(gm, sm, i, j, nsh);
  copy_row(gv, sv, i, j, nsh);
}

// ---- host helpers -----------------------------------------------------------------------------
inline size_t up256(size_t x) { return (x + 255) / 256 * 256; }

struct AddLayout {
  size_t flags, bcnt, totals, mpix, spix, smi, keys, heads, next, total;
};
AddLayout add_layout(int W, int H) {
  const size_t n = (size_t)W * H, nblk = (n + kBlk - 1) / kBlk;
  AddLayout L{};
  size_t o = 0;
  auto take = [&](size_t b) { size_t at = o; o = up256(o + b); return at; };
  L.flags = take(n);
  L.bcnt = take(8 * nblk);
  L.totals = take(16);
  L.mpix = take(4 * n);
  L.spix = take(4 * n);
  L.smi = take(4 * n);
  L.keys = take(8 * (size_t)kKnnSlots);
  L.heads = take(4 * (size_t)kKnnSlots);
  L.next = take(4 * n);
  L.total = o;
  return L;
}

int nsh_of(int deg) { return 3 * (deg + 1) * (deg + 1); }

gps_gaussians stage_view(const gps_gaussians& g, float* base, int64_t cap) {
  gps_gaussians o = g;
  o.xyz = base;
  o.log_scale = base + 3 * cap;
  o.rot = base + 6 * cap;
  o.opacity_raw = base + 10 * cap;
  o.sh = base + 11 * cap;
  return o;
}

struct RemoveLayout {
  size_t keep, bcnt, totals, stage, total;
};
RemoveLayout remove_layout(int64_t n, int deg) {
  const size_t nn = (size_t)std::max<int64_t>(n, 1), nblk = (nn + kBlk - 1) / kBlk;
  RemoveLayout L{};
  size_t o = 0;
  auto take = [&](size_t b) { size_t at = o; o = up256(o + b); return at; };
  L.keep = take(nn);
  L.bcnt = take(4 * nblk);
  L.totals = take(16);
  L.stage = take(3 * 4 * nn * (size_t)(11 + nsh_of(deg)));
  L.total = o;
  return L;
}

gps_status check_g(const gps_gaussians* g, const char* who) {
  if (!g || g->n < 0 || g->sh_degree < 0 || g->sh_degree > 3) return invalid(std::string(who) + ": bad Gaussians");
  if (!g->xyz || !g->log_scale || !g->rot || !g->opacity_raw || !g->sh) return invalid(std::string(who) + ": null array");
  return GPS_OK;
}

gps_status copy_group(float* dst, const float* src, size_t floats, cudaStream_t s) {
  if (floats == 0) return GPS_OK;
  GPS_CHECK_CUDA(cudaMemcpyAsync(dst, src, 4 * floats, cudaMemcpyDeviceToDevice, s));
  return GPS_OK;
}

}  // namespace
}  // namespace gps

using namespace gps;

extern "C" {

gps_status gps_vertex_normals(const gps_intrinsics* K, const gps_pose* T, const float* sdf_depth, const float* vertex,
                              float* normal_out, gps_stream_t stream) {
  if (!K || !T || !sdf_depth || !vertex || !normal_out || K->width <= 0 || K->height <= 0)
    return invalid("gps_vertex_normals: bad argument");
  dim3 grid((K->width + 15) / 16, (K->height + 15) / 16);
  k_vertex_normals<<<grid, 256, 0, as_stream(stream)>>>(K->width, K->height, sdf_depth, vertex, T->t[0], T->t[1],
                                                        T->t[2], normal_out);
  GPS_CHECK_LAUNCH("k_vertex_normals");
  return GPS_OK;
}

gps_status gps_vertex_normals_dpose(const gps_intrinsics* K, const gps_pose* T_dev, const float* sdf_depth,
                                    const float* vertex, float* normal_out, gps_stream_t stream) {
  if (!K || !T_dev || !sdf_depth || !vertex || !normal_out || K->width <= 0 || K->height <= 0)
    return invalid("gps_vertex_normals_dpose: bad argument");
  dim3 grid((K->width + 15) / 16, (K->height + 15) / 16);
  k_vertex_normals<<<grid, 256, 0, as_stream(stream)>>>(K->width, K->height, sdf_depth, vertex, 0.f, 0.f, 0.f,
                                                        normal_out, reinterpret_cast<const float*>(T_dev));
  GPS_CHECK_LAUNCH("k_vertex_normals");
  return GPS_OK;
}

size_t gps_add_workspace_size(const gps_intrinsics* K) {
  if (!K || K->width <= 0 || K->height <= 0) return 0;
  return add_layout(K->width, K->height).total;
}

gps_status gps_add_gaussians_sync(gps_gaussians* g, int64_t capacity, gps_adam_state* state, const gps_intrinsics* K,
                                  const float* sdf_depth, const float* vertex, const float* normal, const float* cstar,
                                  const float* weight, const uint8_t* target_rgba, const gps_add_config* cfg, void* ws,
                                  size_t ws_bytes, int64_t* n_added, int64_t* n_candidates, gps_stream_t stream) {
  gps_status st = check_g(g, "gps_add_gaussians_sync");
  if (st != GPS_OK) return st;
  if (!state || !K || !sdf_depth || !vertex || !normal || !cstar || !weight || !target_rgba || !cfg || !ws || !n_added)
    return invalid("gps_add_gaussians_sync: null argument");
  if (K->width <= 0 || K->height <= 0 || capacity < g->n) return invalid("gps_add_gaussians_sync: bad size");
  if ((reinterpret_cast<uintptr_t>(target_rgba) & 3u) != 0) return invalid("gps_add_gaussians_sync: target must be 4-byte aligned");
  if (state->m.n != g->n || state->v.n != g->n || state->m.sh_degree != g->sh_degree || state->v.sh_degree != g->sh_degree)
    return invalid("gps_add_gaussians_sync: Adam state shape differs from the parameters");
  if (!(cfg->knn_cell > 0) || !(cfg->scale_max > 0) || !(cfg->sample_frac >= 0 && cfg->sample_frac <= 1) ||
      !(cfg->opacity_init > 0 && cfg->opacity_init < 1))
    return invalid("gps_add_gaussians_sync: bad config");
  const AddLayout L = add_layout(K->width, K->height);
  if (ws_bytes < L.total) {
    set_error("gps_add_gaussians_sync: workspace too small");
    return GPS_ERR_WORKSPACE_TOO_SMALL;
  }
  cudaStream_t s = as_stream(stream);
  char* w = static_cast<char*>(ws);
  const uint32_t npx = (uint32_t)K->width * (uint32_t)K->height;
  AddArgs a;
  a.W = K->width; a.H = K->height;
  a.delta_c = cfg->delta_c; a.delta_w = cfg->delta_w; a.inv255 = 1.0f / 255.0f;
  a.seed_h = hash32_host(cfg->seed);
  a.thr = (unsigned long long)std::floor((double)cfg->sample_frac * 4294967296.0);
  a.nblk = (int)((npx + kBlk - 1) / kBlk);
  uint8_t* flags = reinterpret_cast<uint8_t*>(w + L.flags);
  uint32_t* bcnt = reinterpret_cast<uint32_t*>(w + L.bcnt);
  uint32_t* totals = reinterpret_cast<uint32_t*>(w + L.totals);
  uint32_t* mpix = reinterpret_cast<uint32_t*>(w + L.mpix);
  uint32_t* spix = reinterpret_cast<uint32_t*>(w + L.spix);
  uint32_t* smi = reinterpret_cast<uint32_t*>(w + L.smi);
  uint64_t* keys = reinterpret_cast<uint64_t*>(w + L.keys);
  int32_t* heads = reinterpret_cast<int32_t*>(w + L.heads);
  int32_t* next = reinterpret_cast<int32_t*>(w + L.next);
  const uint32_t* tgt = reinterpret_cast<const uint32_t*>(target_rgba);
  k_add_flags<<<a.nblk, kBlk, 0, s>>>(a, sdf_depth, normal, cstar, weight, tgt, flags, bcnt);
  GPS_CHECK_LAUNCH("k_add_flags");
  k_scan_blocks<<<1, 1024, 0, s>>>(bcnt, a.nblk, 2, totals);
  GPS_CHECK_LAUNCH("k_scan_blocks");
  k_add_compact<<<a.nblk, kBlk, 0, s>>>(a, flags, bcnt, mpix, spix, smi);
  GPS_CHECK_LAUNCH("k_add_compact");
  uint32_t tot[2] = {0, 0};
  GPS_CHECK_CUDA(cudaMemcpyAsync(tot, totals, 8, cudaMemcpyDeviceToHost, s));
  GPS_CHECK_CUDA(cudaStreamSynchronize(s));
  const uint32_t M = tot[0], S = tot[1];
  const int64_t room = capacity - g->n;
  const uint32_t count = (uint32_t)std::min<int64_t>(S, room);
  if (n_candidates) *n_candidates = S;
  *n_added = count;
  if (count == 0) return GPS_OK;
  k_fill_keys<<<592, 256, 0, s>>>(keys, kKnnSlots);
  GPS_CHECK_LAUNCH("k_fill_keys");
  GPS_CHECK_CUDA(cudaMemsetAsync(heads, 0xFF, 4 * (size_t)kKnnSlots, s));
  const float inv_cell = 1.0f / cfg->knn_cell;
  k_knn_insert<<<(M + 255) / 256, 256, 0, s>>>(mpix, M, vertex, inv_cell, keys, heads, next);
  GPS_CHECK_LAUNCH("k_knn_insert");
  InitArgs ia;
  ia.n0 = g->n;
  ia.count = count;
  ia.nsh = nsh_of(g->sh_degree);
  ia.inv_cell = inv_cell;
  ia.cell = cfg->knn_cell;
  ia.scale_max = cfg->scale_max;
  ia.rcap = cfg->scale_max * std::sqrt(3.0f);
  ia.rmax = (int)std::ceil(ia.rcap / cfg->knn_cell) + 1;
  ia.opacity_raw = (float)std::log((double)cfg->opacity_init / (1.0 - (double)cfg->opacity_init));
  ia.inv255 = 1.0f / 255.0f;
  k_add_init<<<(count + 127) / 128, 128, 0, s>>>(ia, spix, smi, mpix, vertex, normal, tgt, keys, heads, next, *g,
                                                 state->m, state->v);
  GPS_CHECK_LAUNCH("k_add_init");
  g->n += count;
  state->m.n = g->n;
  state->v.n = g->n;
  return GPS_OK;
}

size_t gps_remove_workspace_size(int64_t n, int32_t sh_degree) {
  if (n < 0 || sh_degree < 0 || sh_degree > 3) return 0;
  return remove_layout(n, sh_degree).total;
}

gps_status gps_remove_gaussians_sync(gps_gaussians* g, gps_adam_state* state, const gps_remove_config* cfg, void* ws,
                                     size_t ws_bytes, int64_t* n_removed, gps_stream_t stream) {
  gps_status st = check_g(g, "gps_remove_gaussians_sync");
  if (st != GPS_OK) return st;
  if (!state || !cfg || !ws || !n_removed) return invalid("gps_remove_gaussians_sync: null argument");
  if (state->m.n != g->n || state->v.n != g->n || state->m.sh_degree != g->sh_degree || state->v.sh_degree != g->sh_degree)
    return invalid("gps_remove_gaussians_sync: Adam state shape differs from the parameters");
  if (!(cfg->sigma_min > 0 && cfg->sigma_min < 1) || !(cfg->scale_max > 0) || !(cfg->scale_min > 0))
    return invalid("gps_remove_gaussians_sync: bad config");
  const RemoveLayout L = remove_layout(g->n, g->sh_degree);
  if (ws_bytes < L.total) {
    set_error("gps_remove_gaussians_sync: workspace too small");
    return GPS_ERR_WORKSPACE_TOO_SMALL;
  }
  *n_removed = 0;
  if (g->n == 0) return GPS_OK;
  cudaStream_t s = as_stream(stream);
  char* w = static_cast<char*>(ws);
  uint8_t* keep = reinterpret_cast<uint8_t*>(w + L.keep);
  uint32_t* bcnt = reinterpret_cast<uint32_t*>(w + L.bcnt);
  uint32_t* totals = reinterpret_cast<uint32_t*>(w + L.totals);
  float* stage = reinterpret_cast<float*>(w + L.stage);
  const int nblk = (int)((g->n + kBlk - 1) / kBlk);
  // thresholds on the raw parameters, rounded once from double (R-REMOVE)
  const double so = cfg->sigma_min;
  const float t_op = (float)std::log(so / (1.0 - so));
  const float t_max = (float)std::log((double)cfg->scale_max), t_min = (float)std::log((double)cfg->scale_min);
  k_remove_flags<<<nblk, kBlk, 0, s>>>(*g, t_op, t_max, t_min, keep, bcnt);
  GPS_CHECK_LAUNCH("k_remove_flags");
  k_scan_blocks<<<1, 1024, 0, s>>>(bcnt, nblk, 1, totals);
  GPS_CHECK_LAUNCH("k_scan_blocks");
  const int nsh = nsh_of(g->sh_degree);
  const int64_t cap = g->n;
  const size_t per = (size_t)(11 + nsh) * cap;
  gps_gaussians sp = stage_view(*g, stage, cap), sm = stage_view(*g, stage + per, cap),
                sv = stage_view(*g, stage + 2 * per, cap);
  k_remove_scatter<<<nblk, kBlk, 0, s>>>(*g, state->m, state->v, keep, bcnt, sp, sm, sv, nsh);
  GPS_CHECK_LAUNCH("k_remove_scatter");
  uint32_t kept = 0;
  GPS_CHECK_CUDA(cudaMemcpyAsync(&kept, totals, 4, cudaMemcpyDeviceToHost, s));
  GPS_CHECK_CUDA(cudaStreamSynchronize(s));
  const int64_t nk = kept;
  const gps_gaussians* dst[3] = {g, &state->m, &state->v};
  const gps_gaussians* src[3] = {&sp, &sm, &sv};
  for (int t = 0; t < 3; ++t) {
    if ((st = copy_group(dst[t]->xyz, src[t]->xyz, 3 * nk, s)) != GPS_OK) return st;
    if ((st = copy_group(dst[t]->log_scale, src[t]->log_scale, 3 * nk, s)) != GPS_OK) return st;
    if ((st = copy_group(dst[t]->rot, src[t]->rot, 4 * nk, s)) != GPS_OK) return st;
    if ((st = copy_group(dst[t]->opacity_raw, src[t]->opacity_raw, nk, s)) != GPS_OK) return st;
    if ((st = copy_group(dst[t]->sh, src[t]->sh, (size_t)nsh * nk, s)) != GPS_OK) return st;
  }
  *n_removed = g->n - nk;
  g->n = nk;
  state->m.n = nk;
  state->v.n = nk;
  return GPS_OK;
}

}  // extern "C"
