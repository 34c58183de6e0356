// volume.cu -- voxel-block hash volume: gps_volume_*, gps_fuse (allocation + integration) and
// gps_raycast for sm_100a.
//
// Paper: GPS-SLAM (arXiv 2509.11574) Sec. 3.2.1 "SDF fusion", PAPER.md P:106 ("Following
// InfiniTAM ... we perform standard SDF fusion to update the SDF and color values in a global
// hash table. Afterwards, the raycast is performed"), voxel contents P:60, raycast P:70-73.
// Readings R-BAND, R-INT, R-RAY and the prescribed fp32 sequences: DESIGN.md §3-§4.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#define GPS_CHK_VAR g_chk_volume
#include "common.cuh"
#include "prof.cuh"

namespace gps {
__device__ unsigned long long g_chk_volume = 0ull;
unsigned long long check_word_take_volume() {
  unsigned long long w = 0ull, z = 0ull;
  cudaMemcpyFromSymbol(&w, g_chk_volume, sizeof(w));
  cudaMemcpyToSymbol(g_chk_volume, &z, sizeof(z));
  return w;
}

// ============================================================================================
// allocation: one CTA per 32x32 pixel patch, 256 threads x 4 pixels (one 8-byte depth load
// each); band blocks are de-duplicated in a CTA-local shared-memory hash set before any
// global hash traffic (hundreds of pixels share a block).
// ============================================================================================
constexpr int kAllocPatch = 32;
constexpr int kSmemSet = 2048;

struct FuseParams {
  float fx, fy, cx, cy;
  int W, H;
  float R[9], t[3];
  float scale, mu, voxel, bs, dmin, dmax;
  float inv_scale, inv_mu;  // fl(1/depth_scale), fl(1/mu): host fp32 divisions
  float A[9], b[3];  // integration's affine voxel -> (fx X, fy Y, Z) map, row c = A[3c..3c+2] (§4.2)
  int wmax;
  const float* dpose;  // device pose (R row-major, t) for the *_dpose entry points, else null
};

// A[c][k] = fl((s_c v) R[k][c]), b[c] = fl(-(s_c ((R[0][c] t0 + R[1][c] t1) + R[2][c] t2))),
// s = (fx, fy, 1), in double with every operation rounded separately (no contraction), then once
// to fp32 -- the host computes it for host poses, the device for device poses (same values)
__host__ __device__ __forceinline__ double dmul(double a, double b) {
#ifdef __CUDA_ARCH__
  return __dmul_rn(a, b);
#else
  return a * b;
#endif
}
__host__ __device__ __forceinline__ double dadd(double a, double b) {
#ifdef __CUDA_ARCH__
  return __dadd_rn(a, b);
#else
  return a + b;
#endif
}
__host__ __device__ __forceinline__ void affine_cam(FuseParams& p) {
  const double sc[3] = {(double)p.fx, (double)p.fy, 1.0};
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    const double sv = dmul(sc[c], (double)p.voxel);
#pragma unroll
    for (int k = 0; k < 3; ++k) p.A[3 * c + k] = (float)dmul(sv, (double)p.R[3 * k + c]);
    double acc = dmul((double)p.R[c], (double)p.t[0]);
    acc = dadd(acc, dmul((double)p.R[3 + c], (double)p.t[1]));
    acc = dadd(acc, dmul((double)p.R[6 + c], (double)p.t[2]));
    p.b[c] = (float)(-dmul(sc[c], acc));
  }
}

// the device-pose instantiations read R, t from device memory once per thread (the same fp32
// values the host would pass, so every prescribed sequence is unchanged)
template <bool DPOSE, class P>
__device__ __forceinline__ void apply_dpose(P& p) {
  if (DPOSE) {
#pragma unroll
    for (int k = 0; k < 9; ++k) p.R[k] = __ldg(p.dpose + k);
#pragma unroll
    for (int k = 0; k < 3; ++k) p.t[k] = __ldg(p.dpose + 9 + k);
  }
}

__device__ __forceinline__ void mark_visible(const VolumeView& v, uint32_t slot, uint32_t frame,
                                             uint32_t* d_flag) {
  if (v.stamp[slot] == frame) return;
  if (atomicExch(&v.stamp[slot], frame) == frame) return;
  const uint32_t idx = atomicAdd(&v.ctr->n_vis, 1u);
  GPS_DCHECK(slot <= v.slot_mask, CHK_SLOT);
  if (idx < v.max_blocks) {
    v.vis[idx] = (int32_t)slot;
  } else {
    v.ctr->overflow = 1u;
    *(volatile uint32_t*)d_flag = 1u;
  }
}

__device__ void global_insert(const VolumeView& v, uint64_t key, uint32_t frame, uint32_t* d_flag) {
  int x, y, z;
  unpack_block(key, x, y, z);
  uint32_t h = hash_block(x, y, z) & v.slot_mask;
  for (uint32_t probe = 0; probe <= v.slot_mask; ++probe) {
    uint64_t k = *(volatile uint64_t*)&v.keys[h];
    if (k == key) {
      mark_visible(v, h, frame, d_flag);
      return;
    }
    if (k == kEmptyKey) {
      const unsigned long long old = atomicCAS((unsigned long long*)&v.keys[h], (unsigned long long)kEmptyKey,
                                               (unsigned long long)key);
      if (old == kEmptyKey) {
        const uint32_t b = atomicAdd(&v.ctr->n_blocks, 1u);
        if (b < v.max_blocks) {
          v.bkeys[b] = key;
          v.vals[h] = (int32_t)b;  // the pool block was initialised empty at create/reset
          const unsigned ix = (unsigned)(x - v.gox), iy = (unsigned)(y - v.goy), iz = (unsigned)(z - v.goz);
          if (v.grid && ix < (unsigned)v.gdx && iy < (unsigned)v.gdy && iz < (unsigned)v.gdz)
            v.grid[((size_t)iz * v.gdy + iy) * v.gdx + ix] = (int32_t)b;
        } else {
          v.ctr->overflow = 1u;
          *(volatile uint32_t*)d_flag = 1u;
        }
        mark_visible(v, h, frame, d_flag);
        return;
      }
      if (old == key) {
        mark_visible(v, h, frame, d_flag);
        return;
      }
    }
    h = (h + 1) & v.slot_mask;
  }
  v.ctr->overflow = 1u;  // table full
  *(volatile uint32_t*)d_flag = 1u;
}

// find-or-insert of a block key in the global table; returns its slot (-1: table full or the
// block budget exceeded, overflow latched).  Does not mark the block visible.
__device__ int32_t global_find_or_insert(const VolumeView& v, uint64_t key, uint32_t* d_flag) {
  int x, y, z;
  unpack_block(key, x, y, z);
  uint32_t h = hash_block(x, y, z) & v.slot_mask;
  for (uint32_t probe = 0; probe <= v.slot_mask; ++probe) {
    const uint64_t k = *(volatile uint64_t*)&v.keys[h];
    if (k == key) return (int32_t)h;
    if (k == kEmptyKey) {
      const unsigned long long old = atomicCAS((unsigned long long*)&v.keys[h], (unsigned long long)kEmptyKey,
                                               (unsigned long long)key);
      if (old == kEmptyKey) {
        const uint32_t b = atomicAdd(&v.ctr->n_blocks, 1u);
        if (b < v.max_blocks) {
          v.bkeys[b] = key;
          v.vals[h] = (int32_t)b;  // the pool block was initialised empty at create/reset
          const unsigned ix = (unsigned)(x - v.gox), iy = (unsigned)(y - v.goy), iz = (unsigned)(z - v.goz);
          if (v.grid && ix < (unsigned)v.gdx && iy < (unsigned)v.gdy && iz < (unsigned)v.gdz)
            v.grid[((size_t)iz * v.gdy + iy) * v.gdx + ix] = (int32_t)b;
        } else {
          v.ctr->overflow = 1u;
          *(volatile uint32_t*)d_flag = 1u;
        }
        return (int32_t)h;
      }
      if (old == key) return (int32_t)h;
    }
    h = (h + 1) & v.slot_mask;
  }
  v.ctr->overflow = 1u;  // table full
  *(volatile uint32_t*)d_flag = 1u;
  return -1;
}

__device__ __forceinline__ void set_insert(unsigned long long* set, uint64_t key, const VolumeView& v,
                                           uint32_t frame, uint32_t* d_flag) {
  int x, y, z;
  unpack_block(key, x, y, z);
  uint32_t h = hash_block(x, y, z) & (kSmemSet - 1);
  for (int probe = 0; probe < kSmemSet; ++probe) {
    const unsigned long long old = atomicCAS(&set[h], (unsigned long long)kEmptyKey, (unsigned long long)key);
    if (old == kEmptyKey || old == key) return;
    h = (h + 1) & (kSmemSet - 1);
  }
  global_insert(v, key, frame, d_flag);  // CTA set full: go straight to the global table
}

// R-BAND for one pixel: the prescribed fp32 sequence of DESIGN.md §4.1, then every block of the
// axis-aligned boxes spanned by consecutive samples' blocks.
__device__ __forceinline__ void pixel_blocks(const FuseParams& p, int u, int vv, uint16_t raw,
                                             unsigned long long* set, const VolumeView& v,
                                             uint32_t frame, uint32_t* d_flag) {
  const float d = pmul((float)raw, p.inv_scale);
  if (!(d >= p.dmin && d <= p.dmax)) return;
  const float xn = pdiv(psub((float)u, p.cx), p.fx);
  const float yn = pdiv(psub((float)vv, p.cy), p.fy);
  const float X[3] = {pmul(xn, d), pmul(yn, d), d};
  float n2 = padd(pmul(X[0], X[0]), pmul(X[1], X[1]));
  n2 = padd(n2, pmul(X[2], X[2]));
  const float q = pdiv(p.mu, psqrt(n2));
  const float a = psub(1.0f, q), b = padd(1.0f, q);
  float A[3], B[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    A[k] = pmul(X[k], a);
    B[k] = pmul(X[k], b);
  }
  int blk[5][3];
#pragma unroll
  for (int s = 0; s < 5; ++s) {
    const float f = (float)s * 0.25f;
    float Q[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) Q[k] = padd(A[k], pmul(psub(B[k], A[k]), f));
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      const float Wr = padd(pdot3(p.R[3 * r + 0], Q[0], p.R[3 * r + 1], Q[1], p.R[3 * r + 2], Q[2]), p.t[r]);
      blk[s][r] = (int)floorf(pdiv(Wr, p.bs));
    }
  }
  uint64_t last = kEmptyKey;
#pragma unroll
  for (int s = 0; s < 4; ++s) {
    const int x0 = min(blk[s][0], blk[s + 1][0]), x1 = max(blk[s][0], blk[s + 1][0]);
    const int y0 = min(blk[s][1], blk[s + 1][1]), y1 = max(blk[s][1], blk[s + 1][1]);
    const int z0 = min(blk[s][2], blk[s + 1][2]), z1 = max(blk[s][2], blk[s + 1][2]);
    for (int z = z0; z <= z1; ++z)
      for (int y = y0; y <= y1; ++y)
        for (int x = x0; x <= x1; ++x) {
          const uint64_t key = pack_block(x, y, z);
          if (key != last) set_insert(set, key, v, frame, d_flag);
          last = key;
        }
  }
}

template <bool DPOSE = false>
__global__ void __launch_bounds__(256) k_alloc(VolumeView v, FuseParams p_in,
                                               const uint16_t* __restrict__ depth, uint32_t frame,
                                               uint32_t* d_flag) {
  FuseParams p = p_in;
  apply_dpose<DPOSE>(p);
  __shared__ unsigned long long set[kSmemSet];
  for (int i = threadIdx.x; i < kSmemSet; i += blockDim.x) set[i] = kEmptyKey;
  __syncthreads();
  const int tx = threadIdx.x & 7, ty = threadIdx.x >> 3;
  const int y = blockIdx.y * kAllocPatch + ty;
  const int x0 = blockIdx.x * kAllocPatch + tx * 4;
  if (y < p.H && x0 < p.W) {
    const uint16_t* row = depth + (size_t)y * p.W;
    uint16_t d4[4] = {0, 0, 0, 0};
    if (x0 + 3 < p.W && ((reinterpret_cast<uintptr_t>(row + x0) & 7u) == 0)) {
      const ushort4 q = *reinterpret_cast<const ushort4*>(row + x0);  // coalesced 8-byte load
      d4[0] = q.x; d4[1] = q.y; d4[2] = q.z; d4[3] = q.w;
    } else {
      for (int k = 0; k < 4; ++k)
        if (x0 + k < p.W) d4[k] = row[x0 + k];
    }
#pragma unroll 1
    for (int k = 0; k < 4; ++k)
      if (x0 + k < p.W && d4[k] != 0) pixel_blocks(p, x0 + k, y, d4[k], set, v, frame, d_flag);
  }
  __syncthreads();
  // global phase: find or insert each of the CTA's blocks, then mark the newly visible ones with
  // ONE append per warp (a single counter for all 65k visible blocks was the kernel's hottest
  // serialisation point).  Each warp first compacts the occupied slots of its 256-slot share of
  // the set (ballots, no barrier), so its dependent global chain (probe, stamp, append) runs once
  // per 32 keys instead of once per 32 slots that hold any key.
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  __shared__ uint16_t wlist[8][256];
  uint32_t nk = 0;
  for (int r = 0; r < 256; r += 32) {
    const int slot = w * 256 + r + lane;
    const bool occ = set[slot] != kEmptyKey;
    const unsigned b = __ballot_sync(0xFFFFFFFFu, occ);
    if (occ) wlist[w][nk + __popc(b & ((1u << lane) - 1u))] = (uint16_t)slot;
    nk += __popc(b);
  }
  __syncwarp();
  for (uint32_t i0 = 0; i0 < nk; i0 += 32) {
    const uint32_t i = i0 + lane;
    int32_t slot = -1;
    if (i < nk) slot = global_find_or_insert(v, set[wlist[w][i]], d_flag);
    bool app = false;
    if (slot >= 0 && v.stamp[slot] != frame) app = atomicExch(&v.stamp[slot], frame) != frame;
    const unsigned bal = __ballot_sync(0xFFFFFFFFu, app);
    if (bal) {
      uint32_t base = 0;
      if (lane == 0) base = atomicAdd(&v.ctr->n_vis, (uint32_t)__popc(bal));
      base = __shfl_sync(0xFFFFFFFFu, base, 0);
      if (app) {
        const uint32_t idx = base + __popc(bal & ((1u << lane) - 1u));
        GPS_DCHECK((uint32_t)slot <= v.slot_mask, CHK_SLOT);
        if (idx < v.max_blocks) {
          v.vis[idx] = slot;
        } else {
          v.ctr->overflow = 1u;
          *(volatile uint32_t*)d_flag = 1u;
        }
      }
    }
  }
}

// ============================================================================================
// integration (R-INT): grid-stride over the visible list; one CTA per block, 256 threads x 2
// adjacent voxels (one 16-byte load/store each).  Prescribed fp32, DESIGN.md §4.2.
// ============================================================================================
// geometry of one voxel (prescribed fp32), in two halves so that a thread can
// issue the frame gathers of both its voxels before waiting for either: voxel_project gives the
// pixel of a voxel in front of the camera, voxel_sample the truncated sample s of its depth
// (false: not updated).  Needs no voxel data, so skipped voxels cost no voxel traffic.
__device__ __forceinline__ bool voxel_project(const FuseParams& p, int gx, int gy, int gz, uint32_t& pix,
                                              float& X2) {
  const float fgx = (float)gx, fgy = (float)gy, fgz = (float)gz;  // exact (|g| < 2^24)
  const float U = __fmaf_rn(p.A[2], fgz, __fmaf_rn(p.A[1], fgy, __fmaf_rn(p.A[0], fgx, p.b[0])));
  const float V = __fmaf_rn(p.A[5], fgz, __fmaf_rn(p.A[4], fgy, __fmaf_rn(p.A[3], fgx, p.b[1])));
  X2 = __fmaf_rn(p.A[8], fgz, __fmaf_rn(p.A[7], fgy, __fmaf_rn(p.A[6], fgx, p.b[2])));
  if (!(X2 > 0.0f)) return false;
  const float iz = __frcp_rn(X2);
  const float uf = __fmaf_rn(U, iz, p.cx);
  const float vf = __fmaf_rn(V, iz, p.cy);
  const float ur = floorf(padd(uf, 0.5f)), vr = floorf(padd(vf, 0.5f));
  if (!(ur >= 0.0f && ur <= (float)(p.W - 1) && vr >= 0.0f && vr <= (float)(p.H - 1))) return false;
  pix = (uint32_t)vr * (uint32_t)p.W + (uint32_t)ur;
  return true;
}
__device__ __forceinline__ bool voxel_sample(const FuseParams& p, uint16_t raw, float X2, float& s) {
  const float d = pmul((float)raw, p.inv_scale);
  if (!(d >= p.dmin && d <= p.dmax)) return false;
  const float eta = psub(d, X2);
  if (eta < -p.mu) return false;
  s = fminf(pmul(eta, p.inv_mu), 1.0f);
  return true;
}

// running means (R-INT): tsdf in prescribed fp32 with the correctly rounded reciprocal of (w+1)
// (srcp[w] = __frcp_rn(w + 1), tabulated); colour as the exact rational mean with round-half-up,
// the division by w+1 done as a multiply-high by ceil(2^32/(w+1)) (exact for numerators < 2^17
// and w+1 <= 256)
__device__ __forceinline__ uint2 voxel_update(float tsdf, uint32_t cw, float s, uint32_t c, int wmax,
                                              const uint32_t* __restrict__ smagic, const float* __restrict__ srcp) {
  const uint32_t w = cw >> 24;
  const float wf = (float)w;
  // w = 0: the stored NaN stands for the initial tsdf 1, and (1*0 + s) * (1/1) = s exactly
  const float t = w == 0 ? s : pmul(padd(pmul(tsdf, wf), s), srcp[w]);
  const uint32_t w1 = w + 1, half = w1 >> 1, magic = smagic[w];
  uint32_t out;
  if (w == 0) {
    out = c & 0x00FFFFFFu;  // first observation: the mean is the sample (2^32/1 has no u32 magic)
  } else {
    out = 0;
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) {
      const uint32_t old = (cw >> (8 * ch)) & 0xFFu, x8 = (c >> (8 * ch)) & 0xFFu;
      out |= __umulhi(old * w + x8 + half, magic) << (8 * ch);
    }
  }
  out |= min(w1, (uint32_t)wmax) << 24;
  return make_uint2(__float_as_uint(t), out);
}

// Grid-stride over the visible list, software-pipelined two deep: the slot of block q + 2G and
// the pool index, key and -neighbour row of block q + G are loaded while block q is integrated
// (G = gridDim.x), so no dependent metadata load is waited for inside the loop.
template <bool DPOSE = false>
__global__ void __launch_bounds__(256) k_integrate(VolumeView v, FuseParams p_in,
                                                   const uint16_t* __restrict__ depth,
                                                   const uint32_t* __restrict__ rgba) {
  FuseParams p = p_in;
  apply_dpose<DPOSE>(p);
  if (DPOSE) affine_cam(p);  // host poses: computed on the host (identical values)
  __shared__ uint32_t smagic[256];
  __shared__ float srcp[256];
  // smagic[w] = ceil(2^32 / (w+1)) for w >= 1 (w = 0 is special-cased in voxel_update)
  for (int d = threadIdx.x; d < 256; d += blockDim.x) {
    smagic[d] = 0xFFFFFFFFu / (uint32_t)(d + 1) + 1u;
    srcp[d] = __frcp_rn((float)(d + 1));
  }
  __syncthreads();
  const uint32_t nvis = min(*(volatile uint32_t*)&v.ctr->n_vis, v.max_blocks);
  if (blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(&v.ctr->vis_total, (unsigned long long)nvis);
  const int e = 2 * threadIdx.x;  // voxel pair (e, e+1): same j,k; i even
  const int li = e & 7, lj = (e >> 3) & 7, lk = e >> 6;
  __shared__ uint32_t scnt[8];
  uint32_t n_upd = 0;
  const uint32_t G = gridDim.x;
  uint32_t q = blockIdx.x;
  // pipeline registers: block q (b1, key1, row m0/m1 of b1), and the slot of block q + G
  int32_t b1 = -1, slot2 = -1;
  uint64_t key1 = 0;
  int4 m0 = make_int4(-1, -1, -1, -1), m1 = m0;
  if (q < nvis) {
    const int32_t slot = v.vis[q];
    b1 = v.vals[slot];
    key1 = v.keys[slot];
  }
  if (q + G < nvis) slot2 = v.vis[q + G];
  if (b1 >= 0) {
    m0 = __ldg(reinterpret_cast<const int4*>(v.nbrm) + 2 * (size_t)b1);
    m1 = __ldg(reinterpret_cast<const int4*>(v.nbrm) + 2 * (size_t)b1 + 1);
  }
  for (; q < nvis; q += G) {
    const int32_t b = b1;
    const uint64_t key = key1;
    const int4 c0r = m0, c1r = m1;
    // advance the pipeline (all loads below are consumed one iteration later)
    b1 = -1;
    if (slot2 >= 0) {
      b1 = v.vals[slot2];
      key1 = v.keys[slot2];
    }
    slot2 = q + 2 * G < nvis ? v.vis[q + 2 * G] : -1;
    if (b < 0) continue;  // uniform across the CTA
    GPS_DCHECK((uint32_t)b < min(v.ctr->n_blocks, v.max_blocks), CHK_POOL);
    int bx, by, bz;
    unpack_block(key, bx, by, bz);
    float2* tp = reinterpret_cast<float2*>(v.tsdf + (size_t)b * kTsdfBlock + tsdf_index(li, lj, lk));
    uint2* cp = reinterpret_cast<uint2*>(v.rgbw + (size_t)b * 512 + e);
    float2 ts = *tp;  // speculative: off the dependent chain
    uint2 cw = *cp;
    const int gx = bx * 8 + li, gy = by * 8 + lj, gz = bz * 8 + lk;
    uint32_t pix0 = 0, pix1 = 0;
    float z0 = 0.f, z1 = 0.f, s0 = 0.f, s1 = 0.f;
    const bool in0 = voxel_project(p, gx, gy, gz, pix0, z0);
    const bool in1 = voxel_project(p, gx + 1, gy, gz, pix1, z1);
    // both voxels' depth and colour gathers in flight together (colour speculatively)
    GPS_DCHECK(!in0 || pix0 < (uint32_t)(p.W * p.H), CHK_PIXEL);
    GPS_DCHECK(!in1 || pix1 < (uint32_t)(p.W * p.H), CHK_PIXEL);
    const uint16_t r0 = in0 ? __ldg(&depth[pix0]) : (uint16_t)0, r1 = in1 ? __ldg(&depth[pix1]) : (uint16_t)0;
    const uint32_t c0 = in0 ? __ldg(&rgba[pix0]) : 0u, c1 = in1 ? __ldg(&rgba[pix1]) : 0u;
    if (b1 >= 0) {  // next block's -neighbour row (its pool index arrived last iteration... or now)
      m0 = __ldg(reinterpret_cast<const int4*>(v.nbrm) + 2 * (size_t)b1);
      m1 = __ldg(reinterpret_cast<const int4*>(v.nbrm) + 2 * (size_t)b1 + 1);
    }
    const bool u0 = in0 && voxel_sample(p, r0, z0, s0);
    const bool u1 = in1 && voxel_sample(p, r1, z1, s1);
    int dneg0 = 0, dneg1 = 0;  // change of the "tsdf <= 0" indicator of each voxel (NaN: false)
    if (u0 | u1) {
      const float old0 = ts.x, old1 = ts.y;
      if (u0) {
        const uint2 r = voxel_update(ts.x, cw.x, s0, c0, p.wmax, smagic, srcp);
        ts.x = __uint_as_float(r.x);
        cw.x = r.y;
      }
      if (u1) {
        const uint2 r = voxel_update(ts.y, cw.y, s1, c1, p.wmax, smagic, srcp);
        ts.y = __uint_as_float(r.x);
        cw.y = r.y;
      }
      dneg0 = u0 ? (int)(ts.x <= 0.f) - (int)(old0 <= 0.f) : 0;
      dneg1 = u1 ? (int)(ts.y <= 0.f) - (int)(old1 <= 0.f) : 0;
      *tp = ts;
      *cp = cw;
      n_upd += (uint32_t)u0 + (uint32_t)u1;
      // apron push: an updated voxel with a coordinate 0 is an apron cell of the -neighbours
      // across those faces (k_link's comment)
      const int zyz = (lj == 0 ? 2 : 0) | (lk == 0 ? 4 : 0);
      if (zyz | (li == 0)) {
        const int32_t mm[8] = {c0r.x, c0r.y, c0r.z, c0r.w, c1r.x, c1r.y, c1r.z, c1r.w};
#pragma unroll
        for (int k = 1; k < 8; ++k) {
          if (mm[k] < 0) continue;
          GPS_DCHECK((uint32_t)mm[k] < min(v.ctr->n_blocks, v.max_blocks), CHK_NBR);
          const int di = tsdf_index(li + 8 * (k & 1), lj + 8 * ((k >> 1) & 1), lk + 8 * (k >> 2));
          float* dst = v.tsdf + (size_t)mm[k] * kTsdfBlock + di;
          if (u0 && (k & ~(zyz | (li == 0 ? 1 : 0))) == 0) {
            GPS_DCHECK(di >= 0 && di < kTsdfBlock, CHK_PLANE);
            dst[0] = ts.x;
          }
          if (u1 && (k & ~zyz) == 0) {  // voxel li+1 >= 1: never on the x face
            GPS_DCHECK(di >= 0 && di + 1 < kTsdfFace, CHK_PLANE);
            dst[1] = ts.y;
          }
        }
      }
    }
    // subneg: the indicator changes of this thread's voxels, for the sub-blocks of the block
    // itself (row entry 0) that hold them and -- the apron cell held the owner's old value --
    // for those of every -neighbour whose apron they feed.  Sign flips are rare: one 64-bit
    // atomic per affected block, each byte's count staying a true count throughout.
    if (dneg0 | dneg1) {
      const int zyz = (lj == 0 ? 2 : 0) | (lk == 0 ? 4 : 0) | (li == 0 ? 1 : 0);
      const int32_t mm[8] = {c0r.x, c0r.y, c0r.z, c0r.w, c1r.x, c1r.y, c1r.z, c1r.w};
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        // voxel li feeds -neighbour k iff k's axes are among its zero coordinates (k = 0: the
        // block itself); li + 1 never lies on the x face
        const int ox = 8 * (k & 1), oy = 8 * ((k >> 1) & 1), oz = 8 * (k >> 2);
        uint64_t wd = 0;
        if ((k & ~zyz) == 0) wd += (uint64_t)(int64_t)dneg0 * cell_subs(li + ox, lj + oy, lk + oz);
        if ((k & ~(zyz & 6)) == 0) wd += (uint64_t)(int64_t)dneg1 * cell_subs(li + 1 + ox, lj + oy, lk + oz);
        if (wd && mm[k] >= 0) {
          GPS_DCHECK((uint32_t)mm[k] < min(v.ctr->n_blocks, v.max_blocks), CHK_NBR);
#ifdef GPS_CHECKED
          // no byte of the packed counts may leave [0, 125] (a borrow would corrupt its neighbour)
          const unsigned long long nw =
              atomicAdd(reinterpret_cast<unsigned long long*>(&v.subneg[mm[k]]), (unsigned long long)wd) + wd;
          bool okb = true;
#pragma unroll
          for (int q = 0; q < 8; ++q) okb &= ((nw >> (8 * q)) & 0xFFull) <= 125ull;
          GPS_DCHECK(okb, CHK_SUBNEG);
#else
          atomicAdd(reinterpret_cast<unsigned long long*>(&v.subneg[mm[k]]), (unsigned long long)wd);
#endif
        }
      }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) n_upd += __shfl_xor_sync(0xFFFFFFFFu, n_upd, o);
  if ((threadIdx.x & 31) == 0) scnt[threadIdx.x >> 5] = n_upd;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long s = 0;
    for (int k = 0; k < 8; ++k) s += scnt[k];
    if (s) atomicAdd(&v.ctr->upd_total, s);
  }
}

// --------------------------------------------------------------------------------------------
// k_integrate_rows: the same integration (R-INT: voxel_project / voxel_sample /
// voxel_update, so the volume is bitwise that of k_integrate and the oracle), one THREAD per
// 8-voxel x-row.  A warp covers half a block (32 rows), so the block's metadata is warp-uniform
// (one broadcast load per warp, pipelined two blocks ahead as in k_integrate); the row's tsdf
// and colour are one 32-byte sector each (2 x 16-byte loads / stores); the frame gathers are
// issued four voxels at a time; the apron pushes become row stores into the -y / -z / -yz
// neighbours' apron rows (32-byte aligned) plus the x-face cells of voxel 0, written only for
// rows with an update (an unchanged voxel rewrites the value its apron already holds: the
// apron invariant makes that a no-op); sign changes (rare) take a per-voxel path.  Against one
// thread per voxel pair this amortises the per-block and per-iteration work over 8 voxels.
// --------------------------------------------------------------------------------------------
template <bool DPOSE = false>
__global__ void __launch_bounds__(256, 4) k_integrate_rows(VolumeView v, FuseParams p_in,
                                                        const uint16_t* __restrict__ depth,
                                                        const uint32_t* __restrict__ rgba) {
  FuseParams p = p_in;
  apply_dpose<DPOSE>(p);
  if (DPOSE) affine_cam(p);
  __shared__ uint32_t smagic[256];
  __shared__ float srcp[256];
  for (int d = threadIdx.x; d < 256; d += blockDim.x) {
    smagic[d] = 0xFFFFFFFFu / (uint32_t)(d + 1) + 1u;
    srcp[d] = __frcp_rn((float)(d + 1));
  }
  __syncthreads();
  const uint32_t nvis = min(*(volatile uint32_t*)&v.ctr->n_vis, v.max_blocks);
  if (blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(&v.ctr->vis_total, (unsigned long long)nvis);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int row = (warp & 1) * 32 + lane;  // row (lj, lk) of this thread's block
  const int lj = row & 7, lk = row >> 3;
  const uint32_t sub = (uint32_t)(warp >> 1);  // block of the CTA's group of 4
  __shared__ uint32_t scnt[8];
  uint32_t n_upd = 0;
  const uint32_t G = 4u * gridDim.x;  // blocks per grid step
  uint32_t q = 4u * blockIdx.x + sub;
  int32_t b1 = -1, slot2 = -1;
  uint64_t key1 = 0;
  int4 m0 = make_int4(-1, -1, -1, -1), m1 = m0;
  if (q < nvis) {
    const int32_t slot = v.vis[q];
    b1 = v.vals[slot];
    key1 = v.keys[slot];
  }
  if (q + G < nvis) slot2 = v.vis[q + G];
  if (b1 >= 0) {
    m0 = __ldg(reinterpret_cast<const int4*>(v.nbrm) + 2 * (size_t)b1);
    m1 = __ldg(reinterpret_cast<const int4*>(v.nbrm) + 2 * (size_t)b1 + 1);
  }
  for (; q < nvis; q += G) {
    const int32_t b = b1;
    const uint64_t key = key1;
    const int4 c0r = m0, c1r = m1;
    b1 = -1;
    if (slot2 >= 0) {
      b1 = v.vals[slot2];
      key1 = v.keys[slot2];
    }
    slot2 = q + 2 * G < nvis ? v.vis[q + 2 * G] : -1;
    if (b < 0) continue;  // uniform across the warp
    GPS_DCHECK((uint32_t)b < min(v.ctr->n_blocks, v.max_blocks), CHK_POOL);
    int bx, by, bz;
    unpack_block(key, bx, by, bz);
    float* trow = v.tsdf + (size_t)b * kTsdfBlock + kTsdfSY * lj + kTsdfSZ * lk;
    uint32_t* crow = v.rgbw + (size_t)b * 512 + 8 * lj + 64 * lk;
    const float4 ta = reinterpret_cast<const float4*>(trow)[0], tb = reinterpret_cast<const float4*>(trow)[1];
    const uint4 ca = reinterpret_cast<const uint4*>(crow)[0], cb = reinterpret_cast<const uint4*>(crow)[1];
    float ts[8] = {ta.x, ta.y, ta.z, ta.w, tb.x, tb.y, tb.z, tb.w};
    uint32_t cw[8] = {ca.x, ca.y, ca.z, ca.w, cb.x, cb.y, cb.z, cb.w};
    if (b1 >= 0) {  // next block's -neighbour row
      m0 = __ldg(reinterpret_cast<const int4*>(v.nbrm) + 2 * (size_t)b1);
      m1 = __ldg(reinterpret_cast<const int4*>(v.nbrm) + 2 * (size_t)b1 + 1);
    }
    const int gx0 = bx * 8, gy = by * 8 + lj, gz = bz * 8 + lk;
    uint32_t upd = 0, up = 0, dn = 0;  // updated voxels; indicator "tsdf <= 0" turned on / off
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      uint32_t pix[4];
      float z[4];
      bool in[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        pix[i] = 0;
        z[i] = 0.f;
        in[i] = voxel_project(p, gx0 + 4 * h + i, gy, gz, pix[i], z[i]);
        GPS_DCHECK(!in[i] || pix[i] < (uint32_t)(p.W * p.H), CHK_PIXEL);
      }
      uint16_t raw[4];
      uint32_t col[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        raw[i] = in[i] ? __ldg(&depth[pix[i]]) : (uint16_t)0;
        col[i] = in[i] ? __ldg(&rgba[pix[i]]) : 0u;
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        float smp = 0.f;
        if (in[i] && voxel_sample(p, raw[i], z[i], smp)) {
          const int x = 4 * h + i;
          const float old = ts[x];
          const uint2 r = voxel_update(old, cw[x], smp, col[i], p.wmax, smagic, srcp);
          ts[x] = __uint_as_float(r.x);
          cw[x] = r.y;
          upd |= 1u << x;
          const bool nowneg = ts[x] <= 0.f, wasneg = old <= 0.f;  // NaN: false
          up |= (uint32_t)(nowneg && !wasneg) << x;
          dn |= (uint32_t)(!nowneg && wasneg) << x;
        }
      }
    }
    if (upd) {
      reinterpret_cast<float4*>(trow)[0] = make_float4(ts[0], ts[1], ts[2], ts[3]);
      reinterpret_cast<float4*>(trow)[1] = make_float4(ts[4], ts[5], ts[6], ts[7]);
      reinterpret_cast<uint4*>(crow)[0] = make_uint4(cw[0], cw[1], cw[2], cw[3]);
      reinterpret_cast<uint4*>(crow)[1] = make_uint4(cw[4], cw[5], cw[6], cw[7]);
      n_upd += __popc(upd);
      // apron pushes: the row is the y = 8 row of the -y neighbour (lj = 0), the z = 8 row of the
      // -z neighbour (lk = 0), the (y, z) = (8, 8) row of the -yz neighbour (both); voxel 0 is
      // the x = 8 face cell of the -x, -xy, -xz, -xyz neighbours (same conditions)
      const int32_t mm[8] = {c0r.x, c0r.y, c0r.z, c0r.w, c1r.x, c1r.y, c1r.z, c1r.w};
      const float4 va = make_float4(ts[0], ts[1], ts[2], ts[3]), vb = make_float4(ts[4], ts[5], ts[6], ts[7]);
#pragma unroll
      for (int k = 2; k < 8; k += 2) {  // k = dy<<1 | dz<<2 (no x bit): whole-row pushes
        const bool feeds = (k & 2 ? lj == 0 : true) && (k & 4 ? lk == 0 : true);
        if (!feeds || mm[k] < 0) continue;
        GPS_DCHECK((uint32_t)mm[k] < min(v.ctr->n_blocks, v.max_blocks), CHK_NBR);
        float* dst = v.tsdf + (size_t)mm[k] * kTsdfBlock + tsdf_index(0, lj + 8 * ((k >> 1) & 1), lk + 8 * (k >> 2));
        reinterpret_cast<float4*>(dst)[0] = va;
        reinterpret_cast<float4*>(dst)[1] = vb;
      }
      if (upd & 1u) {
#pragma unroll
        for (int k = 1; k < 8; k += 2) {  // x face cells of voxel 0
          const bool feeds = (k & 2 ? lj == 0 : true) && (k & 4 ? lk == 0 : true);
          if (!feeds || mm[k] < 0) continue;
          GPS_DCHECK((uint32_t)mm[k] < min(v.ctr->n_blocks, v.max_blocks), CHK_NBR);
          v.tsdf[(size_t)mm[k] * kTsdfBlock + tsdf_index(8, lj + 8 * ((k >> 1) & 1), lk + 8 * (k >> 2))] = ts[0];
        }
      }
    }
    // subneg (rare): each voxel whose indicator changed adjusts the counts of the sub-blocks that
    // hold it, in the block itself and in every -neighbour whose apron it feeds.  A cell x of the
    // row lies in x-half 0 if x <= 4 and in x-half 1 if x >= 4 (cell 4 in both), so per target
    // block the row's change is Dlo * (its half-0 sub-blocks) + Dhi * (its half-1 sub-blocks);
    // voxel 0 alone feeds the x-face (x = 8: half 1) of the -x neighbours
    if (up | dn) {
      const int32_t mm[8] = {c0r.x, c0r.y, c0r.z, c0r.w, c1r.x, c1r.y, c1r.z, c1r.w};
      const int Dlo = __popc(up & 0x1Fu) - __popc(dn & 0x1Fu), Dhi = __popc(up & 0xF0u) - __popc(dn & 0xF0u);
      const int d0 = (int)(up & 1u) - (int)(dn & 1u);
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const bool feeds = (k & 2 ? lj == 0 : true) && (k & 4 ? lk == 0 : true);
        if (!feeds || mm[k] < 0) continue;
        const int yy = lj + 8 * ((k >> 1) & 1), zz = lk + 8 * (k >> 2);
        uint64_t wd;
        if (k & 1) {
          if (!d0) continue;
          wd = (uint64_t)(int64_t)d0 * cell_subs(8, yy, zz);
        } else {
          // cell_subs(0, ..) = the half-0 sub-blocks, cell_subs(7, ..) = the half-1 ones
          wd = (uint64_t)(int64_t)Dlo * cell_subs(0, yy, zz) + (uint64_t)(int64_t)Dhi * cell_subs(7, yy, zz);
        }
        if (!wd) continue;
        GPS_DCHECK((uint32_t)mm[k] < min(v.ctr->n_blocks, v.max_blocks), CHK_NBR);
#ifdef GPS_CHECKED
        const unsigned long long nw =
            atomicAdd(reinterpret_cast<unsigned long long*>(&v.subneg[mm[k]]), (unsigned long long)wd) + wd;
        bool okb = true;
#pragma unroll
        for (int qb = 0; qb < 8; ++qb) okb &= ((nw >> (8 * qb)) & 0xFFull) <= 125ull;
        GPS_DCHECK(okb, CHK_SUBNEG);
#else
        atomicAdd(reinterpret_cast<unsigned long long*>(&v.subneg[mm[k]]), (unsigned long long)wd);
#endif
      }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) n_upd += __shfl_xor_sync(0xFFFFFFFFu, n_upd, o);
  if (lane == 0) scnt[warp] = n_upd;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long sm = 0;
    for (int k = 0; k < 8; ++k) sm += scnt[k];
    if (sm) atomicAdd(&v.ctr->upd_total, sm);
  }
}

__global__ void k_reset_frame(VolumeCounters* ctr) {
  ctr->n_vis = 0u;
  ctr->n_prev = ctr->n_blocks;
}

// --------------------------------------------------------------------------------------------
// k_link (one warp per block allocated this frame, before k_integrate):
//  * neighbour tables: the new block b looks up its 7 +neighbours and 7 -neighbours and writes
//    itself into the opposite table of each existing one; every (block, entry) has exactly one
//    writer value, so concurrent updates cannot conflict;
//  * apron pull: b's 217 apron cells (a coordinate equal to 8) take the current voxels of the
//    +neighbours that own them (NaN where unallocated).  k_integrate then pushes every voxel it
//    updates into the aprons of its -neighbours, so after each fuse every apron equals its
//    owners: an apron changes only when its owner voxel is updated (pushed) or when its block is
//    new (pulled here, before this frame's integration).
// --------------------------------------------------------------------------------------------
__device__ __forceinline__ void apron_cell(int c, int& x, int& y, int& z) {
  // the x = 8 face (81 cells), the y = 8 face without x = 8 (72), the z = 8 face without both (64)
  if (c < 81) { x = 8; y = c % 9; z = c / 9; }
  else if (c < 153) { x = (c - 81) % 8; y = 8; z = (c - 81) / 8; }
  else { x = (c - 153) % 8; y = (c - 153) / 8; z = 8; }
}

__global__ void __launch_bounds__(256) k_link(VolumeView v) {
  const uint32_t lo = min(v.ctr->n_prev, v.max_blocks), hi = min(v.ctr->n_blocks, v.max_blocks);
  const int lane = threadIdx.x & 31;
  const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nwarps = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t b = lo + warp; b < hi; b += nwarps) {
    int x, y, z;
    unpack_block(v.bkeys[b], x, y, z);
    int32_t mine = (int32_t)b;  // lanes 0-7: +neighbour k; lanes 8-15: -neighbour k - 8
    if (lane < 16) {
      const int k = lane & 7, sg = lane < 8 ? 1 : -1;
      const int dx = k & 1, dy = (k >> 1) & 1, dz = (k >> 2) & 1;
      if (k) {
        mine = find_block_fast(v, x + sg * dx, y + sg * dy, z + sg * dz);
        GPS_DCHECK(mine < (int32_t)hi, CHK_NBR);
        // the existing neighbour's opposite table gets b
        if (mine >= 0) (lane < 8 ? v.nbrm : v.nbr)[8 * (size_t)mine + k] = (int32_t)b;
      }
      (lane < 8 ? v.nbr : v.nbrm)[8 * (size_t)b + k] = mine;
    }
    int32_t nb[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) nb[k] = __shfl_sync(0xFFFFFFFFu, mine, k);
    float* base = v.tsdf + (size_t)b * kTsdfBlock;
    uint64_t nneg = 0;  // the new block's own voxels are unobserved: its counts are its apron's
    for (int c = lane; c < 217; c += 32) {
      int ax, ay, az;
      apron_cell(c, ax, ay, az);
      const int k = (ax >> 3) | ((ay >> 3) << 1) | ((az >> 3) << 2);
      int32_t o = -1;
#pragma unroll
      for (int q = 1; q < 8; ++q) o = q == k ? nb[q] : o;
      const float val = o >= 0 ? v.tsdf[(size_t)o * kTsdfBlock + tsdf_index(ax & 7, ay & 7, az & 7)]
                               : __uint_as_float(0x7FC00000u);
      base[tsdf_index(ax, ay, az)] = val;
      if (val <= 0.f) nneg += cell_subs(ax, ay, az);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) nneg += __shfl_xor_sync(0xFFFFFFFFu, nneg, o);
    if (lane == 0) v.subneg[b] = nneg;
  }
}

__global__ void k_fill_pool(float* tsdf, uint32_t* rgbw, size_t nb) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < nb * kTsdfBlock; i += stride)
    tsdf[i] = __uint_as_float(0x7FC00000u);  // unobserved (R-VOX initial tsdf 1, w = 0); apron: no owner
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < nb * 512; i += stride) rgbw[i] = 0u;
}

__global__ void k_fill_u64(uint64_t* p, size_t n, uint64_t val) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += stride) p[i] = val;
}

// ============================================================================================
// raycast (R-RAY): one thread per pixel, 16x16 CTAs.  Fixed grid t_j = dmin + j*voxel; a sample
// is valid iff its 8 trilinear corners are allocated with w > 0.  When the base corner's block is
// unallocated the march jumps to the block's exit (result-preserving).
// ============================================================================================
struct RayParams {
  float fx, fy, cx, cy;
  int W, H;
  float R[9], t[3];
  float voxel, inv_voxel, dmin;
  float zc;  // smallest camera z of any ray sample: dmin * min over pixels of the unit ray's z
  int J;  // last grid index
  const float* dpose;  // device pose for gps_raycast_dpose, else null
};

// --------------------------------------------------------------------------------------------
// Range image: for every 16x16-pixel tile, [t_min, t_max] over ALL allocated blocks whose
// projection can cover a pixel of the tile.  A sample's base-corner block must be allocated for
// the sample to be valid, and the sample lies in that block's box extended by one voxel on the
// + side; every such box meets the ray of the sample's pixel, so no valid sample of a ray lies
// outside its tile's range: starting the march at t_min and stopping at t_max is
// result-preserving.
// --------------------------------------------------------------------------------------------
constexpr int kRangeTile = 16;
constexpr int kMaxRangeTiles = 256 * 256;  // images up to 4096 x 4096 use the range image

__device__ __forceinline__ void block_tile_range(const VolumeView& v, const RayParams& p, uint32_t b, int tiles_x,
                                                 int tiles_y, int& otx0, int& otx1, int& oty0, int& oty1,
                                                 uint32_t& oa0, uint32_t& oa1);

template <bool DPOSE = false>
__global__ void __launch_bounds__(256) k_range(VolumeView v, RayParams p_in, uint32_t* tmin, uint32_t* tmax,
                                               int tiles_x, int tiles_y) {
  RayParams p = p_in;
  apply_dpose<DPOSE>(p);
  const uint32_t nb = min(*(volatile uint32_t*)&v.ctr->n_blocks, v.max_blocks);
  const uint32_t stride = gridDim.x * blockDim.x;
  const int lane = threadIdx.x & 31;
  // warp-uniform trip count: every lane reaches the warp-cooperative tile loop below
  for (uint32_t b0 = blockIdx.x * blockDim.x; b0 < nb; b0 += stride) {
    const uint32_t b = b0 + threadIdx.x;
    int tx0 = 1, tx1 = 0, ty0 = 0, ty1 = 0;
    uint32_t a0 = 0, a1 = 0;
    if (b < nb) block_tile_range(v, p, b, tiles_x, tiles_y, tx0, tx1, ty0, ty1, a0, a1);
    const bool any = tx0 <= tx1 && ty0 <= ty1;
    const bool big = any && (tx1 - tx0 + 1) * (ty1 - ty0 + 1) > 4;
    if (any && !big) {
      for (int ty = ty0; ty <= ty1; ++ty)
        for (int tx = tx0; tx <= tx1; ++tx) {
          const int t = ty * tiles_x + tx;
          GPS_DCHECK(t >= 0 && t < tiles_x * tiles_y, CHK_RANGE_TILE);
          if (tmin[t] > a0) atomicMin(&tmin[t], a0);
          if (tmax[t] < a1) atomicMax(&tmax[t], a1);
        }
    }
    // blocks near the camera cover many tiles: the warp takes them one at a time, a lane per tile
    uint32_t bm = __ballot_sync(0xFFFFFFFFu, big);
    while (bm) {
      const int src = __ffs(bm) - 1;
      bm &= bm - 1u;
      const int sx0 = __shfl_sync(0xFFFFFFFFu, tx0, src), sx1 = __shfl_sync(0xFFFFFFFFu, tx1, src);
      const int sy0 = __shfl_sync(0xFFFFFFFFu, ty0, src), sy1 = __shfl_sync(0xFFFFFFFFu, ty1, src);
      const uint32_t s0 = __shfl_sync(0xFFFFFFFFu, a0, src), s1 = __shfl_sync(0xFFFFFFFFu, a1, src);
      const int wx = sx1 - sx0 + 1, cnt = wx * (sy1 - sy0 + 1);
      for (int k = lane; k < cnt; k += 32) {
        const int t = (sy0 + k / wx) * tiles_x + sx0 + k % wx;
        GPS_DCHECK(t >= 0 && t < tiles_x * tiles_y, CHK_RANGE_TILE);
        if (tmin[t] > s0) atomicMin(&tmin[t], s0);
        if (tmax[t] < s1) atomicMax(&tmax[t], s1);
      }
    }
  }
}

// k_range_smem: the same range image, reduced first in shared memory.  Every block hits 1-16
// tiles and ~100 blocks share a tile, so the global form serialises on ~3600 hot addresses; here
// each CTA folds a contiguous slice of the pool (blocks allocated together lie together) into its
// own copy of the image with shared atomics, then merges only the tiles it touched.  Same min/max
// of the same values: the image is identical.  Images up to kRangeSmemTiles tiles.
constexpr int kRangeSmemTiles = 6144;  // 48 KB of dynamic shared memory (1280x720 at 16x16: 3600)

template <bool DPOSE = false>
__global__ void __launch_bounds__(512) k_range_smem(VolumeView v, RayParams p_in, uint32_t* tmin, uint32_t* tmax,
                                                    int tiles_x, int tiles_y) {
  extern __shared__ uint32_t srange[];  // [ntiles] min, then [ntiles] max
  RayParams p = p_in;
  apply_dpose<DPOSE>(p);
  const int ntiles = tiles_x * tiles_y;
  uint32_t* smin = srange;
  uint32_t* smax = srange + ntiles;
  for (int t = threadIdx.x; t < ntiles; t += blockDim.x) {
    smin[t] = 0xFFFFFFFFu;
    smax[t] = 0u;
  }
  __syncthreads();
  const uint32_t nb = min(*(volatile uint32_t*)&v.ctr->n_blocks, v.max_blocks);
  const uint32_t per = (nb + gridDim.x - 1) / gridDim.x;
  const uint32_t lo = blockIdx.x * per, hi = min(nb, lo + per);
  const int lane = threadIdx.x & 31;
  for (uint32_t b0 = lo; b0 < hi; b0 += blockDim.x) {  // warp-uniform trip count
    const uint32_t b = b0 + threadIdx.x;
    int tx0 = 1, tx1 = 0, ty0 = 0, ty1 = 0;
    uint32_t a0 = 0, a1 = 0;
    if (b < hi) block_tile_range(v, p, b, tiles_x, tiles_y, tx0, tx1, ty0, ty1, a0, a1);
    const bool any = tx0 <= tx1 && ty0 <= ty1;
    const bool big = any && (tx1 - tx0 + 1) * (ty1 - ty0 + 1) > 4;
    if (any && !big) {
      for (int ty = ty0; ty <= ty1; ++ty)
        for (int tx = tx0; tx <= tx1; ++tx) {
          const int t = ty * tiles_x + tx;
          GPS_DCHECK(t >= 0 && t < ntiles, CHK_RANGE_TILE);
          atomicMin(&smin[t], a0);
          atomicMax(&smax[t], a1);
        }
    }
    uint32_t bm = __ballot_sync(0xFFFFFFFFu, big);
    while (bm) {
      const int src = __ffs(bm) - 1;
      bm &= bm - 1u;
      const int sx0 = __shfl_sync(0xFFFFFFFFu, tx0, src), sx1 = __shfl_sync(0xFFFFFFFFu, tx1, src);
      const int sy0 = __shfl_sync(0xFFFFFFFFu, ty0, src), sy1 = __shfl_sync(0xFFFFFFFFu, ty1, src);
      const uint32_t s0 = __shfl_sync(0xFFFFFFFFu, a0, src), s1 = __shfl_sync(0xFFFFFFFFu, a1, src);
      const int wx = sx1 - sx0 + 1, cnt = wx * (sy1 - sy0 + 1);
      for (int k = lane; k < cnt; k += 32) {
        const int t = (sy0 + k / wx) * tiles_x + sx0 + k % wx;
        GPS_DCHECK(t >= 0 && t < ntiles, CHK_RANGE_TILE);
        atomicMin(&smin[t], s0);
        atomicMax(&smax[t], s1);
      }
    }
  }
  __syncthreads();
  for (int t = threadIdx.x; t < ntiles; t += blockDim.x) {
    const uint32_t m0 = smin[t], m1 = smax[t];
    if (m0 != 0xFFFFFFFFu && tmin[t] > m0) atomicMin(&tmin[t], m0);
    if (m1 != 0u && tmax[t] < m1) atomicMax(&tmax[t], m1);
  }
}

// tile rect [tx0, tx1] x [ty0, ty1] (empty: tx0 > tx1) and the t range (float bits a0, a1) of
// pool block b for the range image
__device__ __forceinline__ void block_tile_range(const VolumeView& v, const RayParams& p, uint32_t b, int tiles_x,
                                                 int tiles_y, int& otx0, int& otx1, int& oty0, int& oty1,
                                                 uint32_t& oa0, uint32_t& oa1) {
  {
    int bx, by, bz;
    unpack_block(v.bkeys[b], bx, by, bz);
    const float s = 8.0f * p.voxel;
    const float lo[3] = {bx * s, by * s, bz * s};
    const float hi[3] = {lo[0] + 9.0f * p.voxel, lo[1] + 9.0f * p.voxel, lo[2] + 9.0f * p.voxel};
    // distance from the camera centre to the box, and to its farthest corner
    float d2min = 0.f, d2max = 0.f;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const float o = p.t[k];
      const float dn = o < lo[k] ? lo[k] - o : (o > hi[k] ? o - hi[k] : 0.f);
      const float df = fmaxf(fabsf(o - lo[k]), fabsf(o - hi[k]));
      d2min += dn * dn;
      d2max += df * df;
    }
    const float t0 = sqrtf(d2min) * 0.9999f, t1 = sqrtf(d2max) * 1.0001f + 1e-4f;
    // projected footprint of the box clipped to z >= zc (no ray sample has camera z < zc): the
    // bbox of the projections of its corners in front and of its edges' crossings of z = zc
    float C[8][3];
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const float P0 = (c & 1 ? hi[0] : lo[0]) - p.t[0];
      const float P1 = (c & 2 ? hi[1] : lo[1]) - p.t[1];
      const float P2 = (c & 4 ? hi[2] : lo[2]) - p.t[2];
      C[c][0] = p.R[0] * P0 + p.R[3] * P1 + p.R[6] * P2;
      C[c][1] = p.R[1] * P0 + p.R[4] * P1 + p.R[7] * P2;
      C[c][2] = p.R[2] * P0 + p.R[5] * P1 + p.R[8] * P2;
    }
    float umin = INFINITY, umax = -INFINITY, vmin = INFINITY, vmax = -INFINITY;
    const float zc = p.zc;
    auto add = [&](float X, float Y, float Z) {
      const float iz = 1.0f / Z;
      const float u = p.fx * X * iz + p.cx, w = p.fy * Y * iz + p.cy;
      umin = fminf(umin, u); umax = fmaxf(umax, u);
      vmin = fminf(vmin, w); vmax = fmaxf(vmax, w);
    };
#pragma unroll
    for (int c = 0; c < 8; ++c)
      if (C[c][2] >= zc) add(C[c][0], C[c][1], C[c][2]);
#pragma unroll
    for (int c = 0; c < 8; ++c)
#pragma unroll
      for (int bit = 1; bit < 8; bit <<= 1) {
        const int d = c | bit;
        if (d == c) continue;  // each edge once (c has the bit clear)
        const float za = C[c][2], zb = C[d][2];
        if ((za < zc) != (zb < zc)) {
          const float s = (zc - za) / (zb - za);
          add(C[c][0] + s * (C[d][0] - C[c][0]), C[c][1] + s * (C[d][1] - C[c][1]), zc);
        }
      }
    if (!(umin <= umax)) return;  // entirely nearer than any sample: no ray meets it
    if (umax < -1.f || vmax < -1.f || umin > p.W || vmin > p.H) return;
    otx0 = max(0, (int)floorf((fmaxf(umin, -2.f) - 1.f) / kRangeTile));
    otx1 = min(tiles_x - 1, (int)floorf((fminf(umax, (float)p.W + 2.f) + 1.f) / kRangeTile));
    oty0 = max(0, (int)floorf((fmaxf(vmin, -2.f) - 1.f) / kRangeTile));
    oty1 = min(tiles_y - 1, (int)floorf((fminf(vmax, (float)p.H + 2.f) + 1.f) / kRangeTile));
    oa0 = __float_as_uint(t0);
    oa1 = __float_as_uint(t1);
  }
}

struct BlockCache {
  int x, y, z;
  int32_t b;
};

__device__ __forceinline__ int32_t cached_find(const VolumeView& v, BlockCache& c, int x, int y, int z) {
  if (x == c.x && y == c.y && z == c.z) return c.b;
  c.x = x; c.y = y; c.z = z;
  c.b = find_block_fast(v, x, y, z);
  return c.b;
}

// trilinear as nested lerps (x, then y, then z) of corners numbered dx | dy<<1 | dz<<2
__device__ __forceinline__ float lerp3(const float* c, float ax, float ay, float az) {
  auto lerp = [](float a, float b, float t) { return fmaf(t, b - a, a); };
  const float x00 = lerp(c[0], c[1], ax), x10 = lerp(c[2], c[3], ax);
  const float x01 = lerp(c[4], c[5], ax), x11 = lerp(c[6], c[7], ax);
  return lerp(lerp(x00, x10, ay), lerp(x01, x11, ay), az);
}

// entry k (= dx | dy<<1 | dz<<2) of a block's +neighbour row (n0 = entries 0-3, n1 = 4-7), by
// selects (a dynamically indexed array would live in local memory)
__device__ __forceinline__ int32_t nbr_entry(int32_t b0, int4 n0, int4 n1, int k) {
  return (k & 4) ? ((k & 2) ? ((k & 1) ? n1.w : n1.z) : ((k & 1) ? n1.y : n1.x))
                 : ((k & 2) ? ((k & 1) ? n0.w : n0.z) : ((k & 1) ? n0.y : b0));
}

// footprint diagnostic: mark the owner voxel (512-voxel numbering) of each of the 8 corners of the
// sample whose base voxel is (lx, ly, lz) in block b0
__device__ __forceinline__ void mark_footprint(const VolumeView& v, int32_t b0, int lx, int ly, int lz,
                                               uint32_t* footprint) {
  const int4 n0 = __ldg(reinterpret_cast<const int4*>(v.nbr) + 2 * (size_t)b0);
  const int4 n1 = __ldg(reinterpret_cast<const int4*>(v.nbr) + 2 * (size_t)b0 + 1);
#pragma unroll
  for (int corner = 0; corner < 8; ++corner) {
    const int dx = corner & 1, dy = (corner >> 1) & 1, dz = (corner >> 2) & 1;
    const int k = (dx && lx == 7) | ((dy && ly == 7) << 1) | ((dz && lz == 7) << 2);
    const int32_t b = nbr_entry(b0, n0, n1, k);
    if (b < 0) continue;
    const size_t a = (size_t)b * 512 + ((lx + dx) & 7) + 8 * ((ly + dy) & 7) + 64 * ((lz + dz) & 7);
    atomicOr(&footprint[a >> 5], 1u << (a & 31));
  }
}

// the 8 trilinear corners (numbered dx | dy<<1 | dz<<2) of the sample based at cell (lx, ly, lz)
// of the block plane starting at `pl` (common.cuh layout)
__device__ __forceinline__ void load_corners(const float* __restrict__ pl, int lx, int ly, int lz, float* tv) {
  const float* b0 = pl + lx + kTsdfSY * ly + kTsdfSZ * lz;
  const bool face = lx == 7;
  const float* b1 = face ? pl + kTsdfFace + ly + 9 * lz : b0 + 1;
  const int sy = face ? 1 : kTsdfSY, sz = face ? 9 : kTsdfSZ;
  tv[0] = b0[0]; tv[2] = b0[kTsdfSY]; tv[4] = b0[kTsdfSZ]; tv[6] = b0[kTsdfSY + kTsdfSZ];
  tv[1] = b1[0]; tv[3] = b1[sy]; tv[5] = b1[sz]; tv[7] = b1[sy + sz];
}

// tsdf and colour at voxel-unit position p (the hit point); returns validity.  The tsdf corners
// come from the apron layout, the colour corners from their owner voxels via the +neighbour row.
__device__ __forceinline__ bool trilinear_color(const VolumeView& v, BlockCache& c0, float px, float py, float pz,
                                                float& f, float* col) {
  const float fx = floorf(px), fy = floorf(py), fz = floorf(pz);
  const int gx = (int)fx, gy = (int)fy, gz = (int)fz;
  const float ax = px - fx, ay = py - fy, az = pz - fz;
  const int32_t b0 = cached_find(v, c0, gx >> 3, gy >> 3, gz >> 3);
  if (b0 < 0) return false;
  const int lx = gx & 7, ly = gy & 7, lz = gz & 7;
  float tv[8];
  load_corners(v.tsdf + (size_t)b0 * kTsdfBlock, lx, ly, lz, tv);
  float chk = tv[0];
#pragma unroll
  for (int corner = 1; corner < 8; ++corner) chk += tv[corner];
  if (isnan(chk)) return false;  // an unallocated or unobserved corner
  f = lerp3(tv, ax, ay, az);
  const int4 n0 = __ldg(reinterpret_cast<const int4*>(v.nbr) + 2 * (size_t)b0);
  const int4 n1 = __ldg(reinterpret_cast<const int4*>(v.nbr) + 2 * (size_t)b0 + 1);
  uint32_t cw[8];
#pragma unroll
  for (int corner = 0; corner < 8; ++corner) {
    const int dx = corner & 1, dy = (corner >> 1) & 1, dz = (corner >> 2) & 1;
    const int k = (dx && lx == 7) | ((dy && ly == 7) << 1) | ((dz && lz == 7) << 2);
    // every corner's block is allocated here (its tsdf apron entry is not NaN)
    GPS_DCHECK(nbr_entry(b0, n0, n1, k) >= 0 && nbr_entry(b0, n0, n1, k) < (int32_t)min(v.ctr->n_blocks, v.max_blocks), CHK_NBR);
    cw[corner] = v.rgbw[(size_t)nbr_entry(b0, n0, n1, k) * 512 + ((lx + dx) & 7) + 8 * ((ly + dy) & 7) + 64 * ((lz + dz) & 7)];
  }
#pragma unroll
  for (int ch = 0; ch < 3; ++ch) {
    float c[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) c[k] = (float)((cw[k] >> (8 * ch)) & 0xFFu);
    col[ch] = lerp3(c, ax, ay, az);
  }
  return true;
}

// kDebug: 0 = production; 1 = per-pixel march statistics in vertex_out; 2 = mark every tsdf voxel
// the march reads in `footprint` (the raycast roofline's unique-voxel count)
template <int kDebug, int kMinCtas = 6, bool DPOSE = false>
__global__ void __launch_bounds__(128, 2 * kMinCtas) k_raycast(VolumeView v, RayParams p_in, float* __restrict__ depth_out,
                                                 float* __restrict__ color_out,
                                                 float* __restrict__ vertex_out,
                                                 const uint32_t* __restrict__ tmin,
                                                 const uint32_t* __restrict__ tmax,
                                                 uint32_t* footprint = nullptr) {
  RayParams p = p_in;
  apply_dpose<DPOSE>(p);
  // CTA = 16x8 pixels (128 threads: a small register footprint that co-schedules with the
  // refinement stream's kernels); two CTAs per 16x16 range tile
  const int u = blockIdx.x * 16 + (threadIdx.x & 15);
  const int vv = blockIdx.y * 8 + (threadIdx.x >> 4);
  if (u >= p.W || vv >= p.H) return;
  int jstart = 0, jend = p.J;
  if (tmin) {  // the tile's range image entry (CTA == 16x16 range tile)
    const int tile = (blockIdx.y >> 1) * gridDim.x + blockIdx.x;
    const uint32_t a0 = tmin[tile], a1 = tmax[tile];
    if (a0 == 0xFFFFFFFFu) {
      jend = -1;  // no allocated block can meet any ray of this tile: miss
    } else {
      const float t0 = __uint_as_float(a0), t1 = __uint_as_float(a1);
      const float js = floorf((t0 - p.dmin) / p.voxel) - 1.0f;
      const float je = ceilf((t1 - p.dmin) / p.voxel) + 1.0f;
      jstart = js <= 0.f ? 0 : (js >= (float)p.J ? p.J : (int)js);
      jend = je >= (float)p.J ? p.J : (je < 0.f ? -1 : (int)je);
    }
  }
  const float dcx = (u - p.cx) / p.fx, dcy = (vv - p.cy) / p.fy;
  const float nrm = sqrtf(dcx * dcx + dcy * dcy + 1.0f);
  const float inv = 1.0f / nrm;
  const float dhx = dcx * inv, dhy = dcy * inv, dhz = inv;
  const float rx = p.R[0] * dhx + p.R[1] * dhy + p.R[2] * dhz;
  const float ry = p.R[3] * dhx + p.R[4] * dhy + p.R[5] * dhz;
  const float rz = p.R[6] * dhx + p.R[7] * dhy + p.R[8] * dhz;
  // ray in voxel units: p(t) = o/v + t * r/v
  const float ox = p.t[0] * p.inv_voxel, oy = p.t[1] * p.inv_voxel, oz = p.t[2] * p.inv_voxel;
  const float qx = rx * p.inv_voxel, qy = ry * p.inv_voxel, qz = rz * p.inv_voxel;
  // reciprocal ray components for block exits (in voxel units per metre of t)
  const float iqx = qx != 0.f ? 1.f / qx : INFINITY;
  const float iqy = qy != 0.f ? 1.f / qy : INFINITY;
  const float iqz = qz != 0.f ? 1.f / qz : INFINITY;
  BlockCache c0{INT_MIN, INT_MIN, INT_MIN, -1};
  int32_t pb = -1;   // the last allocated block the march entered, its sub-block counts, and
  uint64_t pw = 0;   // the sub-block (of pb) whose samples were last skipped
  int psk = -1;
  bool prev_valid = false, hit = false;
  float prev_f = 0.f, tstar = 0.f;
  int j = jstart;  // samples before jstart (and after jend) meet no allocated block: invalid
  int n_iter = 0, n_skip = 0, n_invalid = 0;
  // one structured body per grid index (the block lookup, then either the skip or the sample), so
  // the warp reconverges every iteration
  // one structured body per grid index (the block lookup, then either the skip or the sample), so
  // the warp reconverges every iteration
  while (j <= jend) {
    if (kDebug) ++n_iter;
    const float t = p.dmin + (float)j * p.voxel;
    const float px = fmaf(t, qx, ox), py = fmaf(t, qy, oy), pz = fmaf(t, qz, oz);
    const float fx = floorf(px), fy = floorf(py), fz = floorf(pz);
    const int gx = (int)fx, gy = (int)fy, gz = (int)fz;
    const int bx = gx >> 3, by = gy >> 3, bz = gz >> 3;
    // inside the dense grid the lookup is one cached load, done by every lane every step (no
    // divergent cache-miss path); outside it (or without a grid) through the per-ray block cache
    const unsigned ix = (unsigned)(bx - v.gox), iy = (unsigned)(by - v.goy), iz = (unsigned)(bz - v.goz);
    int32_t b0;
    if (v.grid && ix < (unsigned)v.gdx && iy < (unsigned)v.gdy && iz < (unsigned)v.gdz)
      b0 = __ldg(&v.grid[(iz * (unsigned)v.gdy + iy) * (unsigned)v.gdx + ix]);
    else
      b0 = cached_find(v, c0, bx, by, bz);
    GPS_DCHECK(b0 < (int32_t)min(v.ctr->n_blocks, v.max_blocks), CHK_POOL);
    if (b0 >= 0 && b0 != pb) {
      pb = b0;
      pw = __ldg(reinterpret_cast<const unsigned long long*>(&v.subneg[b0]));
      psk = -1;
    }
    // all-positive block: every sub-block count is zero (and its samples not skipped yet)
    const bool ppos = b0 >= 0 && pw == 0ull && psk < 0;
    if (b0 < 0 || ppos) {
      // exit of this block: first grid index at or past it, minus a 0.01-step margin against
      // fp32 error (so jn never exceeds the true first index of the next block)
      const float ex = qx != 0.f ? ((qx > 0.f ? (float)(bx + 1) : (float)bx) * 8.f - ox) * iqx : INFINITY;
      const float ey = qy != 0.f ? ((qy > 0.f ? (float)(by + 1) : (float)by) * 8.f - oy) * iqy : INFINITY;
      const float ez = qz != 0.f ? ((qz > 0.f ? (float)(bz + 1) : (float)bz) * 8.f - oz) * iqz : INFINITY;
      const float texit = fminf(ex, fminf(ey, ez));
      const float jn = ceilf((texit - p.dmin) * p.inv_voxel - 0.01f);
      const int jnext = (jn <= (float)(p.J + 1)) ? (int)jn : p.J + 1;
      if (b0 < 0) {  // unallocated: all its samples are invalid
        j = max(j + 1, jnext);
        prev_valid = false;
      } else {
        // all-positive block: no sample based in it can end the march (a valid sample is a
        // convex combination of > 0 corners), so only its last sample matters -- as the
        // predecessor of the next block's first.  Jump there and evaluate it normally.
        psk = 0;
        j = max(j, jnext - 1);
      }
      if (kDebug) ++n_skip;
    } else {
      // the 8 corners at constant offsets in the apron layout (NaN: unallocated or unobserved;
      // a NaN corner makes the nested-lerp value NaN, so validity is "the value is not NaN").
      // Sample j + 1 is evaluated in the same step when it lies in the same block: its corner
      // loads are in flight together with sample j's (same arithmetic as its own step would do,
      // so the result is unchanged; it is discarded if sample j ends the march).
      const float* pl = v.tsdf + (size_t)b0 * kTsdfBlock;
      float tv[8], tw[8];
      load_corners(pl, gx & 7, gy & 7, gz & 7, tv);
      const float t2 = p.dmin + (float)(j + 1) * p.voxel;
      const float px2 = fmaf(t2, qx, ox), py2 = fmaf(t2, qy, oy), pz2 = fmaf(t2, qz, oz);
      const float fx2 = floorf(px2), fy2 = floorf(py2), fz2 = floorf(pz2);
      const int gx2 = (int)fx2, gy2 = (int)fy2, gz2 = (int)fz2;
      const bool pair = j + 1 <= jend && (gx2 >> 3) == bx && (gy2 >> 3) == by && (gz2 >> 3) == bz;
      if (pair) load_corners(pl, gx2 & 7, gy2 & 7, gz2 & 7, tw);
      if (kDebug == 2) {
        mark_footprint(v, b0, gx & 7, gy & 7, gz & 7, footprint);
        if (pair) mark_footprint(v, b0, gx2 & 7, gy2 & 7, gz2 & 7, footprint);
      }
      const float f = lerp3(tv, px - fx, py - fy, pz - fz);
      const bool valid = !isnan(f);
      if (kDebug && !valid) ++n_invalid;
      if (j >= 1 && valid && f <= 0.f) {
        if (prev_valid && prev_f > 0.f) {
          tstar = (p.dmin + (float)(j - 1) * p.voxel) + p.voxel * prev_f / (prev_f - f);
          hit = true;
        }
        break;
      }
      prev_valid = valid;
      prev_f = f;
      ++j;
      if (pair) {
        const float f2 = lerp3(tw, px2 - fx2, py2 - fy2, pz2 - fz2);
        const bool valid2 = !isnan(f2);
        if (kDebug && !valid2) ++n_invalid;
        if (valid2 && f2 <= 0.f) {  // j >= 1 here
          if (prev_valid && prev_f > 0.f) {
            tstar = (p.dmin + (float)(j - 1) * p.voxel) + p.voxel * prev_f / (prev_f - f2);
            hit = true;
          }
          break;
        }
        prev_valid = valid2;
        prev_f = f2;
        ++j;
      }
    }
  }
  float D = 0.f, col[3] = {0.f, 0.f, 0.f}, V[3] = {0.f, 0.f, 0.f};
  if (hit) {
    V[0] = p.t[0] + tstar * rx;
    V[1] = p.t[1] + tstar * ry;
    V[2] = p.t[2] + tstar * rz;
    float fd;
    if (trilinear_color(v, c0, V[0] * p.inv_voxel, V[1] * p.inv_voxel, V[2] * p.inv_voxel, fd, col)) {
      D = tstar * inv;
      col[0] *= (1.f / 255.f); col[1] *= (1.f / 255.f); col[2] *= (1.f / 255.f);
    } else {
      col[0] = col[1] = col[2] = 0.f;
      V[0] = V[1] = V[2] = 0.f;
    }
  }
  const size_t pix = (size_t)vv * p.W + u;
  depth_out[pix] = D;
  color_out[3 * pix + 0] = col[0];
  color_out[3 * pix + 1] = col[1];
  color_out[3 * pix + 2] = col[2];
  if (kDebug == 1) {  // diagnostics (GPS_RAYCAST_DEBUG=1): loop iterations, block skips, invalid samples
    vertex_out[3 * pix + 0] = (float)n_iter;
    vertex_out[3 * pix + 1] = (float)n_skip;
    vertex_out[3 * pix + 2] = (float)n_invalid;
  } else if (vertex_out) {
    vertex_out[3 * pix + 0] = V[0];
    vertex_out[3 * pix + 1] = V[1];
    vertex_out[3 * pix + 2] = V[2];
  }
}

// a deliberately failing check (the checked build's self-test: its bit must reach the word)
__global__ void k_check_selftest(int bit) {
  GPS_DCHECK(threadIdx.x != 7, bit);
}

__global__ void k_apron_check(VolumeView v, unsigned long long* bad) {
  const uint32_t nb = min(v.ctr->n_blocks, v.max_blocks);
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < (size_t)nb * 217; i += (size_t)gridDim.x * blockDim.x) {
    const uint32_t b = (uint32_t)(i / 217);
    int x, y, z;
    apron_cell((int)(i % 217), x, y, z);
    int bx, by, bz;
    unpack_block(v.bkeys[b], bx, by, bz);
    const int32_t o = find_block(v, bx + (x >> 3), by + (y >> 3), bz + (z >> 3));
    const float want = o >= 0 ? v.tsdf[(size_t)o * kTsdfBlock + tsdf_index(x & 7, y & 7, z & 7)] : __uint_as_float(0x7FC00000u);
    const float got = v.tsdf[(size_t)b * kTsdfBlock + tsdf_index(x, y, z)];
    if (!((isnan(want) && isnan(got)) || __float_as_uint(want) == __float_as_uint(got))) atomicAdd(bad, 1ull);
  }
}

// hash / pool / neighbour-table invariants (the checked build's race evidence for the lock-free
// insert and k_link): every occupied slot maps to a pool block whose key is the slot's key; every
// pool block is found at its own key; each block's 8 + and 8 - neighbour entries equal a fresh
// lookup of those neighbours; dense-grid cells of allocated blocks hold their pool index; the
// number of occupied slots equals the number of pool blocks (no duplicate key was inserted).
__global__ void k_hash_check(VolumeView v, unsigned long long* bad, unsigned long long* occupied) {
  const uint32_t nb = min(v.ctr->n_blocks, v.max_blocks);
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  const size_t i0 = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  unsigned long long nbad = 0, nocc = 0;
  for (size_t h = i0; h <= v.slot_mask; h += stride) {
    const uint64_t k = v.keys[h];
    if (k == kEmptyKey) continue;
    ++nocc;
    const int32_t b = v.vals[h];
    if (b < 0 || (uint32_t)b >= nb || v.bkeys[b] != k) ++nbad;
  }
  for (size_t b = i0; b < nb; b += stride) {
    int x, y, z;
    unpack_block(v.bkeys[b], x, y, z);
    if (find_block(v, x, y, z) != (int32_t)b) ++nbad;
    for (int q = 0; q < 8; ++q) {
      const int dx = q & 1, dy = (q >> 1) & 1, dz = (q >> 2) & 1;
      if (v.nbr[8 * b + q] != find_block(v, x + dx, y + dy, z + dz)) ++nbad;
      if (v.nbrm[8 * b + q] != find_block(v, x - dx, y - dy, z - dz)) ++nbad;
    }
    if (v.grid) {
      const unsigned ix = (unsigned)(x - v.gox), iy = (unsigned)(y - v.goy), iz = (unsigned)(z - v.goz);
      if (ix < (unsigned)v.gdx && iy < (unsigned)v.gdy && iz < (unsigned)v.gdz &&
          v.grid[((size_t)iz * v.gdy + iy) * v.gdx + ix] != (int32_t)b)
        ++nbad;
    }
  }
  if (nbad) atomicAdd(bad, nbad);
  if (nocc) atomicAdd(occupied, nocc);
}

// subneg invariant: recount the <= 0 cells of each allocated block's plane (own + apron) per
// sub-block
__global__ void k_negcnt_check(VolumeView v, unsigned long long* bad) {
  const uint32_t nb = min(v.ctr->n_blocks, v.max_blocks);
  const int lane = threadIdx.x & 31;
  for (uint32_t b = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; b < nb; b += (gridDim.x * blockDim.x) >> 5) {
    uint64_t n = 0;
    for (int c = lane; c < 729; c += 32) {
      const int x = c % 9, y = (c / 9) % 9, z = c / 81;
      if (v.tsdf[(size_t)b * kTsdfBlock + tsdf_index(x, y, z)] <= 0.f) n += cell_subs(x, y, z);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) n += __shfl_xor_sync(0xFFFFFFFFu, n, o);
    if (lane == 0 && n != v.subneg[b]) atomicAdd(bad, 1ull);
  }
}

__global__ void k_popcount(const uint32_t* __restrict__ words, size_t n, unsigned long long* total) {
  unsigned long long s = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    s += __popc(words[i]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xFFFFFFFFu, s, o);
  if ((threadIdx.x & 31) == 0 && s) atomicAdd(total, s);
}

// ---- debug export ----------------------------------------------------------------------------
__global__ void k_export_blocks(VolumeView v, int32_t* coords, Voxel* voxels, uint32_t cap,
                                uint32_t* count) {
  const uint32_t slots = v.slot_mask + 1;
  for (uint32_t s = blockIdx.x * blockDim.x + threadIdx.x; s < slots; s += gridDim.x * blockDim.x) {
    const uint64_t k = v.keys[s];
    if (k == kEmptyKey || v.vals[s] < 0) continue;
    const uint32_t i = atomicAdd(count, 1u);
    if (i >= cap) continue;
    int x, y, z;
    unpack_block(k, x, y, z);
    coords[3 * i] = x; coords[3 * i + 1] = y; coords[3 * i + 2] = z;
    if (voxels) {
      const size_t b = (size_t)v.vals[s];
      for (int e = 0; e < 512; ++e) {
        const float t = v.tsdf[b * kTsdfBlock + tsdf_index(e & 7, (e >> 3) & 7, e >> 6)];
        voxels[(size_t)i * 512 + e] = Voxel{isnan(t) ? 1.0f : t, v.rgbw[b * 512 + e]};
      }
    }
  }
}

__global__ void k_export_visible(VolumeView v, int32_t* coords, uint32_t cap, uint32_t* count) {
  const uint32_t nvis = min(v.ctr->n_vis, v.max_blocks);
  for (uint32_t q = blockIdx.x * blockDim.x + threadIdx.x; q < nvis; q += gridDim.x * blockDim.x) {
    const int32_t slot = v.vis[q];
    if (v.vals[slot] < 0) continue;
    const uint32_t i = atomicAdd(count, 1u);
    if (i >= cap) continue;
    int x, y, z;
    unpack_block(v.keys[slot], x, y, z);
    coords[3 * i] = x; coords[3 * i + 1] = y; coords[3 * i + 2] = z;
  }
}

// host-mapped sticky overflow flags, one per volume (index by the volume's flag pointer)
struct HostFlag {
  uint32_t* host;
  uint32_t* dev;
};

}  // namespace gps

using namespace gps;

namespace {
// the flag lives right after the public struct
struct VolumeImpl : gps_volume {
  HostFlag flag;
  uint32_t* range;  // 2 x kMaxRangeTiles: range image of the raycast (t_min, t_max bits)
};

gps_status check_sticky(const gps_volume* vol) {
  const VolumeImpl* v = static_cast<const VolumeImpl*>(vol);
  if (*(volatile uint32_t*)v->flag.host) {
    set_error("volume block budget / hash table exceeded by an earlier gps_fuse");
    return GPS_ERR_OUT_OF_BLOCKS;
  }
  return GPS_OK;
}

gps_status fill_volume(VolumeImpl* v, cudaStream_t s) {
  const gps_volume_config& c = v->cfg;
  k_fill_u64<<<592, 256, 0, s>>>(v->view.keys, (size_t)c.hash_slots, kEmptyKey);
  GPS_CHECK_LAUNCH("k_fill_u64");
  GPS_CHECK_CUDA(cudaMemsetAsync(v->view.vals, 0xFF, sizeof(int32_t) * c.hash_slots, s));
  GPS_CHECK_CUDA(cudaMemsetAsync(v->view.stamp, 0xFF, sizeof(uint32_t) * c.hash_slots, s));
  k_fill_pool<<<1184, 256, 0, s>>>(v->view.tsdf, v->view.rgbw, (size_t)c.max_blocks);
  GPS_CHECK_LAUNCH("k_fill_pool");
  GPS_CHECK_CUDA(cudaMemsetAsync(v->view.subneg, 0, sizeof(uint64_t) * c.max_blocks, s));
  GPS_CHECK_CUDA(cudaMemsetAsync(v->view.ctr, 0, sizeof(VolumeCounters), s));
  if (v->view.grid)
    GPS_CHECK_CUDA(cudaMemsetAsync(v->view.grid, 0xFF,
                                   sizeof(int32_t) * (size_t)v->view.gdx * v->view.gdy * v->view.gdz, s));
  *(volatile uint32_t*)v->flag.host = 0u;
  v->frame = 0;
  return GPS_OK;
}

bool valid_intrinsics(const gps_intrinsics* K) {
  return K && K->width > 0 && K->height > 0 && K->fx > 0 && K->fy > 0 && std::isfinite(K->cx) &&
         std::isfinite(K->cy) && K->width <= 65535 && K->height <= 65535;
}
}  // namespace

extern "C" {

gps_status gps_volume_create(const gps_volume_config* cfg, gps_stream_t stream, gps_volume** out) {
  if (!cfg || !out) return invalid("gps_volume_create: null argument");
  *out = nullptr;
  if (!(cfg->voxel_size > 0) || !(cfg->mu > 0) || cfg->w_max < 1 || cfg->w_max > 255 ||
      !(cfg->depth_min >= 0) || !(cfg->depth_max > cfg->depth_min) || cfg->max_blocks < 1 ||
      cfg->max_blocks > (1ll << 30) || cfg->hash_slots < 2 || (cfg->hash_slots & (cfg->hash_slots - 1)) ||
      cfg->hash_slots > (1ll << 31) || cfg->dense_dims[0] < 0 || cfg->dense_dims[1] < 0 || cfg->dense_dims[2] < 0 ||
      (double)cfg->dense_dims[0] * cfg->dense_dims[1] * cfg->dense_dims[2] > (double)(1ll << 30))
    return invalid("gps_volume_create: bad config (voxel_size, mu > 0; 1 <= w_max <= 255; "
                   "depth_max > depth_min; hash_slots a power of two)");
  VolumeImpl* v = new VolumeImpl();
  v->cfg = *cfg;
  cudaGetDevice(&v->device);
  const size_t slots = (size_t)cfg->hash_slots, nb = (size_t)cfg->max_blocks;
  bool ok = cudaMalloc(&v->view.keys, sizeof(uint64_t) * slots) == cudaSuccess &&
            cudaMalloc(&v->view.vals, sizeof(int32_t) * slots) == cudaSuccess &&
            cudaMalloc(&v->view.stamp, sizeof(uint32_t) * slots) == cudaSuccess &&
            cudaMalloc(&v->view.tsdf, sizeof(float) * kTsdfBlock * nb) == cudaSuccess &&
            cudaMalloc(&v->view.rgbw, sizeof(uint32_t) * 512 * nb) == cudaSuccess &&
            cudaMalloc(&v->view.vis, sizeof(int32_t) * nb) == cudaSuccess &&
            cudaMalloc(&v->view.bkeys, sizeof(uint64_t) * nb) == cudaSuccess &&
            cudaMalloc(&v->view.nbr, sizeof(int32_t) * 8 * nb) == cudaSuccess &&
            cudaMalloc(&v->view.nbrm, sizeof(int32_t) * 8 * nb) == cudaSuccess &&
            cudaMalloc(&v->view.subneg, sizeof(uint64_t) * nb) == cudaSuccess &&
            cudaMalloc(&v->range, sizeof(uint32_t) * 2 * kMaxRangeTiles) == cudaSuccess &&
            cudaMalloc(&v->view.ctr, sizeof(VolumeCounters)) == cudaSuccess &&
            cudaHostAlloc(&v->flag.host, sizeof(uint32_t), cudaHostAllocMapped) == cudaSuccess &&
            cudaHostGetDevicePointer(&v->flag.dev, v->flag.host, 0) == cudaSuccess;
  if (!ok) {
    cudaGetLastError();
    set_error("gps_volume_create: out of device memory");
    gps_volume_destroy(v);
    return GPS_ERR_OOM;
  }
  v->view.slot_mask = (uint32_t)(slots - 1);
  v->view.max_blocks = (uint32_t)nb;
  v->view.grid = nullptr;
  v->view.gox = cfg->dense_origin[0]; v->view.goy = cfg->dense_origin[1]; v->view.goz = cfg->dense_origin[2];
  v->view.gdx = cfg->dense_dims[0]; v->view.gdy = cfg->dense_dims[1]; v->view.gdz = cfg->dense_dims[2];
  const size_t gcells = (size_t)std::max(0, v->view.gdx) * std::max(0, v->view.gdy) * std::max(0, v->view.gdz);
  if (gcells > 0) {
    if (cudaMalloc(&v->view.grid, sizeof(int32_t) * gcells) != cudaSuccess) {
      cudaGetLastError();
      set_error("gps_volume_create: out of device memory (dense grid)");
      gps_volume_destroy(v);
      return GPS_ERR_OOM;
    }
  } else {
    v->view.gdx = v->view.gdy = v->view.gdz = 0;
  }
  gps_status st = fill_volume(v, as_stream(stream));
  if (st != GPS_OK) {
    gps_volume_destroy(v);
    return st;
  }
  *out = v;
  return GPS_OK;
}

void gps_volume_destroy(gps_volume* vol) {
  if (!vol) return;
  VolumeImpl* v = static_cast<VolumeImpl*>(vol);
  cudaFree(v->view.keys);
  cudaFree(v->view.vals);
  cudaFree(v->view.stamp);
  cudaFree(v->view.tsdf);
  cudaFree(v->view.rgbw);
  cudaFree(v->view.vis);
  cudaFree(v->view.bkeys);
  cudaFree(v->view.nbr);
  cudaFree(v->view.nbrm);
  cudaFree(v->view.subneg);
  if (v->view.grid) cudaFree(v->view.grid);
  cudaFree(v->range);
  cudaFree(v->view.ctr);
  if (v->flag.host) cudaFreeHost(v->flag.host);
  delete v;
}

gps_status gps_volume_copy(gps_volume* dst, const gps_volume* src, gps_stream_t stream) {
  if (!dst || !src) return invalid("gps_volume_copy: null volume");
  if (std::memcmp(&dst->cfg, &src->cfg, sizeof(gps_volume_config)) != 0)
    return invalid("gps_volume_copy: volumes have different configs");
  VolumeImpl* d = static_cast<VolumeImpl*>(dst);
  const VolumeImpl* s = static_cast<const VolumeImpl*>(src);
  cudaStream_t st = as_stream(stream);
  const size_t slots = (size_t)s->cfg.hash_slots, nb = (size_t)s->cfg.max_blocks;
  auto cp = [&](void* a, const void* b, size_t bytes) { return cudaMemcpyAsync(a, b, bytes, cudaMemcpyDeviceToDevice, st); };
  GPS_CHECK_CUDA(cp(d->view.keys, s->view.keys, 8 * slots));
  GPS_CHECK_CUDA(cp(d->view.vals, s->view.vals, 4 * slots));
  GPS_CHECK_CUDA(cp(d->view.stamp, s->view.stamp, 4 * slots));
  GPS_CHECK_CUDA(cp(d->view.tsdf, s->view.tsdf, 4 * kTsdfBlock * nb));
  GPS_CHECK_CUDA(cp(d->view.rgbw, s->view.rgbw, 4 * 512 * nb));
  GPS_CHECK_CUDA(cp(d->view.vis, s->view.vis, 4 * nb));
  GPS_CHECK_CUDA(cp(d->view.bkeys, s->view.bkeys, 8 * nb));
  GPS_CHECK_CUDA(cp(d->view.nbr, s->view.nbr, 32 * nb));
  GPS_CHECK_CUDA(cp(d->view.nbrm, s->view.nbrm, 32 * nb));
  GPS_CHECK_CUDA(cp(d->view.subneg, s->view.subneg, 8 * nb));
  GPS_CHECK_CUDA(cp(d->view.ctr, s->view.ctr, sizeof(VolumeCounters)));
  if (s->view.grid)
    GPS_CHECK_CUDA(cp(d->view.grid, s->view.grid, 4 * (size_t)s->view.gdx * s->view.gdy * s->view.gdz));
  d->frame = s->frame;
  *(volatile uint32_t*)d->flag.host = *(volatile uint32_t*)s->flag.host;
  return GPS_OK;
}

gps_status gps_volume_reset(gps_volume* vol, gps_stream_t stream) {
  if (!vol) return invalid("gps_volume_reset: null volume");
  return fill_volume(static_cast<VolumeImpl*>(vol), as_stream(stream));
}

gps_status gps_volume_stats_sync(gps_volume* vol, gps_stream_t stream, int64_t* n_blocks, int64_t* budget,
                                 int64_t* n_visible, int64_t* visible_total, int64_t* updated_total) {
  if (!vol) return invalid("gps_volume_stats_sync: null volume");
  VolumeImpl* v = static_cast<VolumeImpl*>(vol);
  VolumeCounters c;
  GPS_CHECK_CUDA(cudaMemcpyAsync(&c, v->view.ctr, sizeof(c), cudaMemcpyDeviceToHost, as_stream(stream)));
  GPS_CHECK_CUDA(cudaStreamSynchronize(as_stream(stream)));
  if (n_blocks) *n_blocks = c.n_blocks;
  if (budget) *budget = v->cfg.max_blocks;
  if (n_visible) *n_visible = std::min<int64_t>(c.n_vis, v->cfg.max_blocks);
  if (visible_total) *visible_total = (int64_t)c.vis_total;
  if (updated_total) *updated_total = (int64_t)c.upd_total;
  if (c.overflow || *(volatile uint32_t*)v->flag.host) {
    set_error("volume block budget exceeded: budget " + std::to_string(v->cfg.max_blocks));
    return GPS_ERR_OUT_OF_BLOCKS;
  }
  return GPS_OK;
}

static gps_status fuse_impl(gps_volume* vol, const gps_intrinsics* K, const gps_pose* T, const gps_pose* dT,
                            const uint16_t* depth, float depth_scale, const uint8_t* rgba, gps_stream_t stream,
                            const char* who) {
  if (!vol || !(T || dT) || !depth || !rgba) return invalid(std::string(who) + ": null argument");
  if (!valid_intrinsics(K)) return invalid(std::string(who) + ": bad intrinsics");
  if (!(depth_scale > 0)) return invalid(std::string(who) + ": depth_scale must be > 0");
  if ((reinterpret_cast<uintptr_t>(rgba) & 3u) != 0) return invalid(std::string(who) + ": rgba must be 4-byte aligned");
  if ((reinterpret_cast<uintptr_t>(depth) & 1u) != 0) return invalid(std::string(who) + ": depth must be 2-byte aligned");
  if (dT && (reinterpret_cast<uintptr_t>(dT) & 3u) != 0) return invalid(std::string(who) + ": pose must be 4-byte aligned");
  gps_status st = check_sticky(vol);
  if (st != GPS_OK) return st;
  VolumeImpl* v = static_cast<VolumeImpl*>(vol);
  cudaStream_t s = as_stream(stream);
  FuseParams p;
  p.fx = K->fx; p.fy = K->fy; p.cx = K->cx; p.cy = K->cy; p.W = K->width; p.H = K->height;
  for (int i = 0; i < 9; ++i) p.R[i] = T ? T->R[i] : 0.f;
  for (int i = 0; i < 3; ++i) p.t[i] = T ? T->t[i] : 0.f;
  p.dpose = dT ? reinterpret_cast<const float*>(dT) : nullptr;
  p.scale = depth_scale;
  p.mu = v->cfg.mu;
  p.inv_scale = 1.0f / depth_scale;
  p.inv_mu = 1.0f / v->cfg.mu;
  p.voxel = v->cfg.voxel_size;
  p.bs = 8.0f * v->cfg.voxel_size;
  p.dmin = v->cfg.depth_min;
  p.dmax = v->cfg.depth_max;
  p.wmax = v->cfg.w_max;
  if (T) affine_cam(p);  // device poses: k_integrate computes it from the pose it reads
  const uint32_t frame = v->frame++;
  k_reset_frame<<<1, 1, 0, s>>>(v->view.ctr);
  GPS_CHECK_LAUNCH("k_reset_frame");
  dim3 ga((p.W + kAllocPatch - 1) / kAllocPatch, (p.H + kAllocPatch - 1) / kAllocPatch);
  {
    GPS_PROF(K_ALLOC, s);
    if (dT)
      k_alloc<true><<<ga, 256, 0, s>>>(v->view, p, depth, frame, v->flag.dev);
    else
      k_alloc<<<ga, 256, 0, s>>>(v->view, p, depth, frame, v->flag.dev);
  }
  GPS_CHECK_LAUNCH("k_alloc");
  {
    GPS_PROF(K_LINK, s);
    k_link<<<148, 256, 0, s>>>(v->view);
  }
  GPS_CHECK_LAUNCH("k_link");
  // persistent-style grid: 148 SMs x 8 resident 256-thread CTAs, striding over the visible list
  {
    GPS_PROF(K_INTEGRATE, s);
    static const bool pairs = getenv("GPS_INTEGRATE_PAIRS") != nullptr;  // A/B: thread per voxel pair
    const uint32_t* c4 = reinterpret_cast<const uint32_t*>(rgba);
    if (pairs && dT)
      k_integrate<true><<<148 * 8, 256, 0, s>>>(v->view, p, depth, c4);
    else if (pairs)
      k_integrate<<<148 * 8, 256, 0, s>>>(v->view, p, depth, c4);
    else if (dT)
      k_integrate_rows<true><<<148 * 8, 256, 0, s>>>(v->view, p, depth, c4);
    else
      k_integrate_rows<<<148 * 8, 256, 0, s>>>(v->view, p, depth, c4);
  }
  GPS_CHECK_LAUNCH("k_integrate");
  return GPS_OK;
}

gps_status gps_fuse(gps_volume* vol, const gps_intrinsics* K, const gps_pose* T, const uint16_t* depth,
                    float depth_scale, const uint8_t* rgba, gps_stream_t stream) {
  if (!T) return invalid("gps_fuse: null argument");
  return fuse_impl(vol, K, T, nullptr, depth, depth_scale, rgba, stream, "gps_fuse");
}

gps_status gps_fuse_dpose(gps_volume* vol, const gps_intrinsics* K, const gps_pose* T_dev, const uint16_t* depth,
                          float depth_scale, const uint8_t* rgba, gps_stream_t stream) {
  if (!T_dev) return invalid("gps_fuse_dpose: null argument");
  return fuse_impl(vol, K, nullptr, T_dev, depth, depth_scale, rgba, stream, "gps_fuse_dpose");
}

static bool range_smem_ready() {  // once per process (before any stream capture: gps_fuse_raycast)
  static const bool ok = cudaFuncSetAttribute(k_range_smem<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              8 * kRangeSmemTiles) == cudaSuccess &&
                         cudaFuncSetAttribute(k_range_smem<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              8 * kRangeSmemTiles) == cudaSuccess;
  return ok;
}

static gps_status raycast_impl(const gps_volume* vol, const gps_intrinsics* K, const gps_pose* T, float* depth_out,
                               float* color_out, float* vertex_out, uint32_t* footprint, gps_stream_t stream,
                               const gps_pose* dT = nullptr) {
  const VolumeImpl* v = static_cast<const VolumeImpl*>(vol);
  RayParams p;
  p.fx = K->fx; p.fy = K->fy; p.cx = K->cx; p.cy = K->cy; p.W = K->width; p.H = K->height;
  for (int i = 0; i < 9; ++i) p.R[i] = T ? T->R[i] : 0.f;
  for (int i = 0; i < 3; ++i) p.t[i] = T ? T->t[i] : 0.f;
  p.dpose = dT ? reinterpret_cast<const float*>(dT) : nullptr;
  p.voxel = v->cfg.voxel_size;
  p.inv_voxel = 1.0f / v->cfg.voxel_size;
  p.dmin = v->cfg.depth_min;
  p.J = (int)std::floor(((double)v->cfg.depth_max - (double)v->cfg.depth_min) / (double)v->cfg.voxel_size);
  {
    // the unit ray's z is smallest at an image corner; 0.99 keeps the bound conservative in fp32
    const double ex = std::max(std::fabs(0.0 - K->cx), std::fabs((double)(K->width - 1) - K->cx)) / K->fx;
    const double ey = std::max(std::fabs(0.0 - K->cy), std::fabs((double)(K->height - 1) - K->cy)) / K->fy;
    p.zc = (float)(0.99 * (double)v->cfg.depth_min / std::sqrt(1.0 + ex * ex + ey * ey));
  }
  dim3 g((p.W + 15) / 16, (p.H + 15) / 16);  // range tiles (16x16); raycast CTAs are 16x8
  const dim3 gr(g.x, 2 * g.y);
  cudaStream_t s = as_stream(stream);
  const int ntiles = (int)(g.x * g.y);
  uint32_t* tmin = nullptr;
  uint32_t* tmax = nullptr;
  static const bool no_range = getenv("GPS_NO_RANGE") != nullptr;  // A/B: march from dmin
  if (ntiles <= kMaxRangeTiles && !no_range) {
    tmin = v->range;
    tmax = v->range + kMaxRangeTiles;
    GPS_CHECK_CUDA(cudaMemsetAsync(tmin, 0xFF, sizeof(uint32_t) * ntiles, s));
    GPS_CHECK_CUDA(cudaMemsetAsync(tmax, 0x00, sizeof(uint32_t) * ntiles, s));
    {
      GPS_PROF(K_RANGE, s);
      const bool global_range = getenv("GPS_RANGE_GLOBAL") != nullptr;  // A/B and the test: global atomics only
      const size_t smem = 8 * (size_t)ntiles;
      if (ntiles <= kRangeSmemTiles && !global_range) {
        if (!range_smem_ready()) return cuda_fail("cudaFuncSetAttribute(k_range_smem)", cudaGetLastError());
        if (dT)
          k_range_smem<true><<<148 * 2, 512, smem, s>>>(v->view, p, tmin, tmax, (int)g.x, (int)g.y);
        else
          k_range_smem<<<148 * 2, 512, smem, s>>>(v->view, p, tmin, tmax, (int)g.x, (int)g.y);
      } else if (dT) {
        k_range<true><<<148 * 4, 256, 0, s>>>(v->view, p, tmin, tmax, (int)g.x, (int)g.y);
      } else {
        k_range<<<148 * 4, 256, 0, s>>>(v->view, p, tmin, tmax, (int)g.x, (int)g.y);
      }
    }
    GPS_CHECK_LAUNCH("k_range");
  }
  {
    GPS_PROF(K_RAYCAST, s);
    static const bool dbg = getenv("GPS_RAYCAST_DEBUG") != nullptr;
    if (footprint)
      k_raycast<2><<<gr, 128, 0, s>>>(v->view, p, depth_out, color_out, nullptr, tmin, tmax, footprint);
    else if (dbg && vertex_out && !dT)
      k_raycast<1><<<gr, 128, 0, s>>>(v->view, p, depth_out, color_out, vertex_out, tmin, tmax);
    else if (dT)
      k_raycast<0, 4, true><<<gr, 128, 0, s>>>(v->view, p, depth_out, color_out, vertex_out, tmin, tmax);
    else {
      // 8 resident 128-thread CTAs per SM (64 registers, no spills)
      k_raycast<0, 4><<<gr, 128, 0, s>>>(v->view, p, depth_out, color_out, vertex_out, tmin, tmax);
    }
  }
  GPS_CHECK_LAUNCH("k_raycast");
  return GPS_OK;
}

gps_status gps_raycast(gps_volume* vol, const gps_intrinsics* K, const gps_pose* T, float* depth_out,
                       float* color_out, float* vertex_out, gps_stream_t stream) {
  if (!vol || !T || !depth_out || !color_out) return invalid("gps_raycast: null argument");
  if (!valid_intrinsics(K)) return invalid("gps_raycast: bad intrinsics");
  gps_status st = check_sticky(vol);
  if (st != GPS_OK) return st;
  return raycast_impl(vol, K, T, depth_out, color_out, vertex_out, nullptr, stream);
}

gps_status gps_raycast_dpose(gps_volume* vol, const gps_intrinsics* K, const gps_pose* T_dev, float* depth_out,
                             float* color_out, float* vertex_out, gps_stream_t stream) {
  if (!vol || !T_dev || !depth_out || !color_out) return invalid("gps_raycast_dpose: null argument");
  if (!valid_intrinsics(K)) return invalid("gps_raycast_dpose: bad intrinsics");
  if ((reinterpret_cast<uintptr_t>(T_dev) & 3u) != 0) return invalid("gps_raycast_dpose: pose must be 4-byte aligned");
  gps_status st = check_sticky(vol);
  if (st != GPS_OK) return st;
  return raycast_impl(vol, K, nullptr, depth_out, color_out, vertex_out, nullptr, stream, T_dev);
}

// gps_fuse_raycast: gps_fuse then gps_raycast of the same frame in one call; with use_graph the
// frame's launches are captured and replayed as one CUDA graph (a ring of executable graphs per
// volume, updated in place: see gps_refine_round in render.cu)
namespace {
constexpr int kFrameRing = 3;
struct FrameGraph {
  const void* vol;
  cudaGraphExec_t exec[kFrameRing];
  int next;
};
std::mutex g_frame_mu;
std::vector<FrameGraph> g_frame_graphs;
}  // namespace

gps_status gps_fuse_raycast(gps_volume* vol, const gps_intrinsics* K, const gps_pose* T, const uint16_t* depth,
                            float depth_scale, const uint8_t* rgba, float* depth_out, float* color_out,
                            float* vertex_out, int32_t use_graph, gps_stream_t stream) {
  if (!vol || !T || !depth_out || !color_out) return invalid("gps_fuse_raycast: null argument");
  if (!valid_intrinsics(K)) return invalid("gps_fuse_raycast: bad intrinsics");
  cudaStream_t s = as_stream(stream);
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  const bool graph = use_graph != 0 && s != nullptr && s != cudaStreamLegacy && s != cudaStreamPerThread &&
                     !g_prof_on && cudaStreamIsCapturing(s, &cs) == cudaSuccess && cs == cudaStreamCaptureStatusNone;
  VolumeImpl* v = static_cast<VolumeImpl*>(vol);
  const uint32_t frame0 = v->frame;
  if (graph) {
    if (!range_smem_ready()) return cuda_fail("cudaFuncSetAttribute(k_range_smem)", cudaGetLastError());
    GPS_CHECK_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
  }
  gps_status st = fuse_impl(vol, K, T, nullptr, depth, depth_scale, rgba, stream, "gps_fuse_raycast");
  if (st == GPS_OK) st = raycast_impl(vol, K, T, depth_out, color_out, vertex_out, nullptr, stream);
  if (!graph) return st;
  cudaGraph_t gr = nullptr;
  const cudaError_t ec = cudaStreamEndCapture(s, &gr);
  if (st != GPS_OK || ec != cudaSuccess) {  // nothing was launched
    if (gr) cudaGraphDestroy(gr);
    cudaGetLastError();
    v->frame = frame0;
    return st != GPS_OK ? st : cuda_fail("cudaStreamEndCapture", ec);
  }
  std::lock_guard<std::mutex> lock(g_frame_mu);
  FrameGraph* fg = nullptr;
  for (FrameGraph& f : g_frame_graphs)
    if (f.vol == vol) fg = &f;
  if (!fg) {
    g_frame_graphs.push_back(FrameGraph{vol, {}, 0});
    fg = &g_frame_graphs.back();
  }
  cudaGraphExec_t& exec = fg->exec[fg->next];
  fg->next = (fg->next + 1) % kFrameRing;
  if (exec) {
    cudaGraphExecUpdateResultInfo info;
    if (cudaGraphExecUpdate(exec, gr, &info) != cudaSuccess) {
      cudaGetLastError();
      cudaGraphExecDestroy(exec);
      exec = nullptr;
    }
  }
  cudaError_t e = cudaSuccess;
  if (!exec) e = cudaGraphInstantiate(&exec, gr, 0);
  cudaGraphDestroy(gr);
  if (e != cudaSuccess) {
    exec = nullptr;
    v->frame = frame0;
    return cuda_fail("cudaGraphInstantiate", e);
  }
  e = cudaGraphLaunch(exec, s);
  if (e != cudaSuccess) {
    v->frame = frame0;
    return cuda_fail("cudaGraphLaunch", e);
  }
  return GPS_OK;
}

gps_status gps_debug_apron_check_sync(const gps_volume* vol, gps_stream_t stream, int64_t* n_bad) {
  if (!vol || !n_bad) return invalid("gps_debug_apron_check_sync: bad argument");
  const VolumeImpl* v = static_cast<const VolumeImpl*>(vol);
  cudaStream_t s = as_stream(stream);
  unsigned long long* cnt = nullptr;
  GPS_CHECK_CUDA(cudaMallocAsync(&cnt, 8, s));
  GPS_CHECK_CUDA(cudaMemsetAsync(cnt, 0, 8, s));
  k_apron_check<<<592, 256, 0, s>>>(v->view, cnt);
  GPS_CHECK_LAUNCH("k_apron_check");
  k_negcnt_check<<<592, 256, 0, s>>>(v->view, cnt);
  GPS_CHECK_LAUNCH("k_negcnt_check");
  unsigned long long h = 0;
  GPS_CHECK_CUDA(cudaMemcpyAsync(&h, cnt, 8, cudaMemcpyDeviceToHost, s));
  GPS_CHECK_CUDA(cudaFreeAsync(cnt, s));
  GPS_CHECK_CUDA(cudaStreamSynchronize(s));
  *n_bad = (int64_t)h;
  return GPS_OK;
}

gps_status gps_debug_check_selftest(int32_t bit, gps_stream_t stream) {
  if (bit < 0 || bit > 63) return invalid("gps_debug_check_selftest: bit must be in [0, 63]");
  k_check_selftest<<<1, 32, 0, as_stream(stream)>>>(bit);
  GPS_CHECK_LAUNCH("k_check_selftest");
  return GPS_OK;
}

gps_status gps_debug_hash_check_sync(const gps_volume* vol, gps_stream_t stream, int64_t* n_bad) {
  if (!vol || !n_bad) return invalid("gps_debug_hash_check_sync: bad argument");
  const VolumeImpl* v = static_cast<const VolumeImpl*>(vol);
  cudaStream_t s = as_stream(stream);
  unsigned long long* cnt = nullptr;
  GPS_CHECK_CUDA(cudaMallocAsync(&cnt, 16, s));
  GPS_CHECK_CUDA(cudaMemsetAsync(cnt, 0, 16, s));
  k_hash_check<<<592, 256, 0, s>>>(v->view, cnt, cnt + 1);
  GPS_CHECK_LAUNCH("k_hash_check");
  unsigned long long h[2] = {0, 0};
  VolumeCounters c{};
  GPS_CHECK_CUDA(cudaMemcpyAsync(h, cnt, 16, cudaMemcpyDeviceToHost, s));
  GPS_CHECK_CUDA(cudaMemcpyAsync(&c, v->view.ctr, sizeof(c), cudaMemcpyDeviceToHost, s));
  GPS_CHECK_CUDA(cudaFreeAsync(cnt, s));
  GPS_CHECK_CUDA(cudaStreamSynchronize(s));
  const unsigned long long nb = std::min<unsigned long long>(c.n_blocks, v->view.max_blocks);
  *n_bad = (int64_t)(h[0] + (h[1] > nb ? h[1] - nb : nb - h[1]));
  return GPS_OK;
}

gps_status gps_debug_raycast_footprint_sync(const gps_volume* vol, const gps_intrinsics* K, const gps_pose* T,
                                            gps_stream_t stream, int64_t* unique_voxels) {
  if (!vol || !T || !unique_voxels || !valid_intrinsics(K)) return invalid("gps_debug_raycast_footprint_sync: bad argument");
  const VolumeImpl* v = static_cast<const VolumeImpl*>(vol);
  cudaStream_t s = as_stream(stream);
  const size_t words = ((size_t)v->cfg.max_blocks * 512 + 31) / 32;
  const size_t px = (size_t)K->width * K->height;
  uint32_t* bm = nullptr;
  float* buf = nullptr;
  unsigned long long* cnt = nullptr;
  GPS_CHECK_CUDA(cudaMallocAsync(&bm, words * 4, s));
  GPS_CHECK_CUDA(cudaMallocAsync(&buf, px * 16, s));
  GPS_CHECK_CUDA(cudaMallocAsync(&cnt, 8, s));
  GPS_CHECK_CUDA(cudaMemsetAsync(bm, 0, words * 4, s));
  GPS_CHECK_CUDA(cudaMemsetAsync(cnt, 0, 8, s));
  gps_status st = raycast_impl(vol, K, T, buf, buf + px, nullptr, bm, stream);
  if (st != GPS_OK) return st;
  k_popcount<<<592, 256, 0, s>>>(bm, words, cnt);
  GPS_CHECK_LAUNCH("k_popcount");
  unsigned long long h = 0;
  GPS_CHECK_CUDA(cudaMemcpyAsync(&h, cnt, 8, cudaMemcpyDeviceToHost, s));
  GPS_CHECK_CUDA(cudaFreeAsync(bm, s));
  GPS_CHECK_CUDA(cudaFreeAsync(buf, s));
  GPS_CHECK_CUDA(cudaFreeAsync(cnt, s));
  GPS_CHECK_CUDA(cudaStreamSynchronize(s));
  *unique_voxels = (int64_t)h;
  return GPS_OK;
}

gps_status gps_debug_export_blocks_sync(const gps_volume* vol, gps_stream_t stream, int32_t* coords, void* voxels,
                                        int64_t cap, int64_t* n) {
  if (!vol || !coords || !n || cap < 0) return invalid("gps_debug_export_blocks_sync: bad argument");
  const VolumeImpl* v = static_cast<const VolumeImpl*>(vol);
  cudaStream_t s = as_stream(stream);
  uint32_t* cnt = nullptr;
  GPS_CHECK_CUDA(cudaMallocAsync(&cnt, sizeof(uint32_t), s));
  GPS_CHECK_CUDA(cudaMemsetAsync(cnt, 0, sizeof(uint32_t), s));
  k_export_blocks<<<256, 256, 0, s>>>(v->view, coords, reinterpret_cast<Voxel*>(voxels),
                                      (uint32_t)std::min<int64_t>(cap, 0xFFFFFFFFll), cnt);
  GPS_CHECK_LAUNCH("k_export_blocks");
  uint32_t h = 0;
  GPS_CHECK_CUDA(cudaMemcpyAsync(&h, cnt, sizeof(h), cudaMemcpyDeviceToHost, s));
  GPS_CHECK_CUDA(cudaFreeAsync(cnt, s));
  GPS_CHECK_CUDA(cudaStreamSynchronize(s));
  *n = h;
  return GPS_OK;
}

gps_status gps_debug_export_visible_sync(const gps_volume* vol, gps_stream_t stream, int32_t* coords, int64_t cap,
                                         int64_t* n) {
  if (!vol || !coords || !n || cap < 0) return invalid("gps_debug_export_visible_sync: bad argument");
  const VolumeImpl* v = static_cast<const VolumeImpl*>(vol);
  cudaStream_t s = as_stream(stream);
  uint32_t* cnt = nullptr;
  GPS_CHECK_CUDA(cudaMallocAsync(&cnt, sizeof(uint32_t), s));
  GPS_CHECK_CUDA(cudaMemsetAsync(cnt, 0, sizeof(uint32_t), s));
  k_export_visible<<<256, 256, 0, s>>>(v->view, coords, (uint32_t)std::min<int64_t>(cap, 0xFFFFFFFFll), cnt);
  GPS_CHECK_LAUNCH("k_export_visible");
  uint32_t h = 0;
  GPS_CHECK_CUDA(cudaMemcpyAsync(&h, cnt, sizeof(h), cudaMemcpyDeviceToHost, s));
  GPS_CHECK_CUDA(cudaFreeAsync(cnt, s));
  GPS_CHECK_CUDA(cudaStreamSynchronize(s));
  *n = h;
  return GPS_OK;
}

}  // extern "C"
