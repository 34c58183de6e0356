// tracking.cu -- frame-to-model ICP camera tracking for sm_100a:
// gps_track_sync.
//
// Paper: GPS-SLAM (arXiv 2509.11574) Sec. 3.2.1 "Camera tracking", Eq. 5:
// point-to-plane ICP against the previous frame's raycast vertex and normal maps, over a
// resolution hierarchy of the depth map.  Readings R-ICP-ASSOC (the garbled projection of
// P:113), R-ICP-PYR, R-ICP-GATE, R-ICP-GN: DESIGN.md §3.
//
// Per frame:  k_icp_depth (u16 -> metres, level 0) -> k_icp_down (levels 1..L-1)
// per level:  k_icp_maps  (vertex + normal maps of the current frame, camera frame; resets the
//                          level's stop flag)
// per step:   k_icp_step   (per pixel: association, gates, residual and Jacobian; the 27 sums of
//                          J^T J, J^T r, r^2 and the inlier count per CTA, in double; the last CTA
//                          totals the CTA sums, Cholesky-solves the 6x6 system and updates the pose
//                          in device memory -- one launch per step, no host round trip)
// k_icp_init / k_icp_export move the poses in and out: gps_track_sync reads the result back once,
// gps_track_async leaves it in device memory for gps_fuse_dpose / gps_raycast_dpose.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cmath>
#include <string>

#define GPS_CHK_VAR g_chk_tracking
#include "common.cuh"

namespace gps {
__device__ unsigned long long g_chk_tracking = 0ull;
unsigned long long check_word_take_tracking() {
  unsigned long long w = 0ull, z = 0ull;
  cudaMemcpyFromSymbol(&w, g_chk_tracking, sizeof(w));
  cudaMemcpyToSymbol(g_chk_tracking, &z, sizeof(z));
  return w;
}
namespace {

constexpr int kIcpMaxLevels = 4;
constexpr int kIcpThreads = 256;
constexpr int kIcpSums = 29;  // 21 (upper triangle of J^T J) + 6 (J^T r) + r^2 + count

struct DevPose {
  double R[9], t[3];
  double energy;
  int32_t steps, inliers, valid, degenerate;
  double pivot;    // smallest Cholesky pivot / largest diagonal of the last system
  int32_t stop;    // this level is done (converged or degenerate)
  uint32_t ticket; // CTAs of the current k_icp_step that have written their sums
  float Rp[9], tp[3];  // the camera the model maps were raycast from (camera -> world)
  gps_pose fail;       // the pose of a frame that does not converge (R-ICP-FAIL): T_fail, else T_init
};

// the initial, model and failure poses, by value (gps_track_sync) or from device memory
// (gps_track_async)
struct PoseSrc {
  gps_pose init, model;
  const gps_pose* dinit;
  const gps_pose* dmodel;
  const gps_pose* dfail;
};

struct Level {
  int W, H;
  float fx, fy, cx, cy;
  const float* depth;  // this level's depth (metres, 0 = invalid)
  float* V;            // camera-frame vertex map
  float* N;            // camera-frame normal map
  int stride;          // model-map subsampling 2^l
};

__global__ void k_icp_depth(const uint16_t* __restrict__ raw, int n, float inv_scale, float dmin, float dmax, float* d) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float z = (float)raw[i] * inv_scale;
  d[i] = (z >= dmin && z <= dmax) ? z : 0.f;
}

// R-ICP-FILT: bilateral filter of the level-0 depth (metres, 0 = invalid), over the valid
// pixels of the (2r+1)^2 window: sum w z / sum w, w = exp(-(dx^2 + dy^2) / (2 s_s^2)
// - (z - z0)^2 / (2 s_r^2)); invalid pixels stay 0
__global__ void k_icp_bilateral(const uint16_t* __restrict__ raw, int W, int H, float inv_scale, float dmin,
                                float dmax, int r, float inv2ss, float inv2sr, float* __restrict__ out) {
  const int u = blockIdx.x * 32 + (threadIdx.x & 31), v = blockIdx.y * 8 + (threadIdx.x >> 5);
  if (u >= W || v >= H) return;
  auto depth_at = [&](int x, int y) {
    const float z = (float)raw[(size_t)y * W + x] * inv_scale;
    return (z >= dmin && z <= dmax) ? z : 0.f;
  };
  const float z0 = depth_at(u, v);
  float res = 0.f;
  if (z0 > 0.f) {
    float sw = 0.f, sz = 0.f;
    for (int dy = -r; dy <= r; ++dy) {
      const int y = v + dy;
      if (y < 0 || y >= H) continue;
      for (int dx = -r; dx <= r; ++dx) {
        const int x = u + dx;
        if (x < 0 || x >= W) continue;
        const float z = depth_at(x, y);
        if (z > 0.f) {
          const float dz = z - z0;
          const float w = __expf(-(float)(dx * dx + dy * dy) * inv2ss - dz * dz * inv2sr);
          sw += w;
          sz += w * z;
        }
      }
    }
    res = sz / sw;  // sw >= 1 (the centre)
  }
  out[(size_t)v * W + u] = res;
}

// R-ICP-PYR: mean of the valid children of the 2x2 block
__global__ void k_icp_down(const float* __restrict__ src, int Ws, float* dst, int Wd, int Hd) {
  const int u = blockIdx.x * blockDim.x + threadIdx.x, v = blockIdx.y;
  if (u >= Wd || v >= Hd) return;
  const float* r0 = src + (size_t)(2 * v) * Ws + 2 * u;
  const float* r1 = r0 + Ws;
  const float c[4] = {r0[0], r0[1], r1[0], r1[1]};
  float s = 0.f;
  int k = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j)
    if (c[j] > 0.f) { s += c[j]; ++k; }
  dst[(size_t)v * Wd + u] = k ? s / (float)k : 0.f;
}

__device__ __forceinline__ void bp(const Level& L, int u, int v, float z, float* o) {
  o[0] = ((float)u - L.cx) / L.fx * z;
  o[1] = ((float)v - L.cy) / L.fy * z;
  o[2] = z;
}

// vertex and normal maps of one level (R-NORMAL in the camera frame)
__global__ void k_icp_maps(Level L, DevPose* pose) {
  const int u = blockIdx.x * 16 + (threadIdx.x & 15), v = blockIdx.y * 16 + (threadIdx.x >> 4);
  if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) pose->stop = 0;
  if (u >= L.W || v >= L.H) return;
  const size_t p = (size_t)v * L.W + u;
  const float z = L.depth[p];
  float V[3] = {0.f, 0.f, 0.f}, N[3] = {0.f, 0.f, 0.f};
  if (z > 0.f) bp(L, u, v, z, V);
  if (z > 0.f && u > 0 && v > 0 && u < L.W - 1 && v < L.H - 1) {
    const float zl = L.depth[p - 1], zr = L.depth[p + 1], zu = L.depth[p - L.W], zd = L.depth[p + L.W];
    if (zl > 0.f && zr > 0.f && zu > 0.f && zd > 0.f) {
      float a[3], b[3], c[3], d[3];
      bp(L, u + 1, v, zr, a); bp(L, u - 1, v, zl, b); bp(L, u, v + 1, zd, c); bp(L, u, v - 1, zu, d);
      const float dx0 = a[0] - b[0], dx1 = a[1] - b[1], dx2 = a[2] - b[2];
      const float dy0 = c[0] - d[0], dy1 = c[1] - d[1], dy2 = c[2] - d[2];
      float n0 = dx1 * dy2 - dx2 * dy1, n1 = dx2 * dy0 - dx0 * dy2, n2 = dx0 * dy1 - dx1 * dy0;
      const float nn = sqrtf(n0 * n0 + n1 * n1 + n2 * n2);
      if (nn > 0.f) {
        n0 /= nn; n1 /= nn; n2 /= nn;
        if (n0 * V[0] + n1 * V[1] + n2 * V[2] > 0.f) { n0 = -n0; n1 = -n1; n2 = -n2; }
        N[0] = n0; N[1] = n1; N[2] = n2;
      }
    }
  }
  L.V[3 * p] = V[0]; L.V[3 * p + 1] = V[1]; L.V[3 * p + 2] = V[2];
  L.N[3 * p] = N[0]; L.N[3 * p + 1] = N[1]; L.N[3 * p + 2] = N[2];
}

__global__ void k_icp_init(PoseSrc src, DevPose* pose) {
  const gps_pose in = src.dinit ? *src.dinit : src.init;
  const gps_pose mo = src.dmodel ? *src.dmodel : src.model;
  DevPose d{};
  for (int e = 0; e < 9; ++e) d.R[e] = in.R[e];
  for (int e = 0; e < 3; ++e) d.t[e] = in.t[e];
  for (int e = 0; e < 9; ++e) d.Rp[e] = mo.R[e];
  for (int e = 0; e < 3; ++e) d.tp[e] = mo.t[e];
  d.fail = src.dfail ? *src.dfail : in;
  *pose = d;
}

// T_out = T_b (T_a^-1 T_b): R = R_b R_a^T R_b, t = R_b R_a^T (t_b - t_a) + t_b, in double, with R
// re-orthonormalised (Gram-Schmidt on the rows).  Without it the fp32 inputs' departures from
// orthonormality add up through R_a^T (not R_a^-1 for a non-orthonormal R_a) and grow by ~(1+sqrt 2)
// per chained prediction.
__global__ void k_pose_extrapolate(const gps_pose* __restrict__ a, const gps_pose* __restrict__ b, gps_pose* out) {
  const gps_pose A = *a, B = *b;
  double Rd[9], td[3], R[9], t[3];
  for (int r = 0; r < 3; ++r) {
    for (int c = 0; c < 3; ++c)
      Rd[3 * r + c] = (double)A.R[r] * B.R[c] + (double)A.R[3 + r] * B.R[3 + c] + (double)A.R[6 + r] * B.R[6 + c];
    td[r] = (double)A.R[r] * ((double)B.t[0] - A.t[0]) + (double)A.R[3 + r] * ((double)B.t[1] - A.t[1]) +
            (double)A.R[6 + r] * ((double)B.t[2] - A.t[2]);
  }
  for (int r = 0; r < 3; ++r) {
    for (int c = 0; c < 3; ++c)
      R[3 * r + c] = (double)B.R[3 * r] * Rd[c] + (double)B.R[3 * r + 1] * Rd[3 + c] + (double)B.R[3 * r + 2] * Rd[6 + c];
    t[r] = (double)B.R[3 * r] * td[0] + (double)B.R[3 * r + 1] * td[1] + (double)B.R[3 * r + 2] * td[2] + B.t[r];
  }
  double* r0 = R;
  double* r1 = R + 3;
  double* r2 = R + 6;
  double n = sqrt(r0[0] * r0[0] + r0[1] * r0[1] + r0[2] * r0[2]);
  for (int k = 0; k < 3; ++k) r0[k] /= n;
  const double d = r0[0] * r1[0] + r0[1] * r1[1] + r0[2] * r1[2];
  for (int k = 0; k < 3; ++k) r1[k] -= d * r0[k];
  n = sqrt(r1[0] * r1[0] + r1[1] * r1[1] + r1[2] * r1[2]);
  for (int k = 0; k < 3; ++k) r1[k] /= n;
  r2[0] = r0[1] * r1[2] - r0[2] * r1[1];
  r2[1] = r0[2] * r1[0] - r0[0] * r1[2];
  r2[2] = r0[0] * r1[1] - r0[1] * r1[0];
  gps_pose o;
  for (int e = 0; e < 9; ++e) o.R[e] = (float)R[e];
  for (int e = 0; e < 3; ++e) o.t[e] = (float)t[e];
  *out = o;
}

// the tracked pose (fp32, as gps_track_sync rounds it) and, optionally, the whole result
__global__ void k_icp_export(const DevPose* __restrict__ pose, float min_inlier_frac, double min_inliers,
                             float min_pivot, int fallback, gps_pose* out, gps_track_result* res) {
  const DevPose d = *pose;
  gps_track_result r{};
  for (int e = 0; e < 9; ++e) r.T.R[e] = (float)d.R[e];
  for (int e = 0; e < 3; ++e) r.T.t[e] = (float)d.t[e];
  for (int e = 0; e < 9; ++e) r.R64[e] = d.R[e];
  for (int e = 0; e < 3; ++e) r.t64[e] = d.t[e];
  r.energy = d.energy;
  r.inliers = d.inliers;
  r.valid = d.valid;
  r.steps = d.steps;
  r.degenerate = d.degenerate;
  r.inlier_frac = d.valid > 0 ? (float)d.inliers / (float)d.valid : 0.f;
  r.pivot_ratio = (float)d.pivot;
  r.converged = !d.degenerate && r.inlier_frac >= min_inlier_frac && (double)d.inliers >= min_inliers &&
                d.pivot >= (double)min_pivot;
  if (fallback && !r.converged) r.T = d.fail;  // R-ICP-FAIL
  if (out) *out = r.T;
  if (res) *res = r;
}

struct Assoc {
  const float* mV;  // full-resolution model maps (world)
  const float* mN;
  int mW, mH;       // full resolution
  float dist_max, cos_max;
  double eps;       // convergence threshold on |xi|
};

__device__ void icp_solve_cta(const double* partial, int nblk, DevPose* pose, double eps);

// One Gauss-Newton step.  Every CTA: R-ICP-ASSOC / R-ICP-GATE / R-ICP-GN per pixel (J = [m, p x m],
// r = (p - q) . m) and the CTA's sums; the last CTA to finish totals them and solves
// (icp_solve_cta), so a step is one launch.
__global__ void __launch_bounds__(kIcpThreads, 3) k_icp_step(Level L, Assoc a, DevPose* pose, double* partial) {
  __shared__ double red[kIcpThreads / 32][kIcpSums];
  __shared__ bool last;
  // the current pose (fp32) and the model camera, broadcast from shared memory
  __shared__ float sR[9], st[3], sRp[9], stp[3];
  if (pose->stop) return;  // uniform: the level is done
  if (threadIdx.x < 9) {
    sR[threadIdx.x] = (float)pose->R[threadIdx.x];
    sRp[threadIdx.x] = pose->Rp[threadIdx.x];
  } else if (threadIdx.x < 12) {
    st[threadIdx.x - 9] = (float)pose->t[threadIdx.x - 9];
    stp[threadIdx.x - 9] = pose->tp[threadIdx.x - 9];
  }
  __syncthreads();
  const float* R = sR;
  const float* t = st;
  const float* Rp = sRp;
  const float* tp = stp;
  const int Lw = a.mW / L.stride, Lh = a.mH / L.stride;  // this level's model-map size
  float s[kIcpSums];
#pragma unroll
  for (int k = 0; k < kIcpSums; ++k) s[k] = 0.f;
  const int n = L.W * L.H;
  int valid = 0;
  for (int i = blockIdx.x * kIcpThreads + threadIdx.x; i < n; i += gridDim.x * kIcpThreads) {
    const float* Nc = L.N + 3 * (size_t)i;
    if (Nc[0] != 0.f || Nc[1] != 0.f || Nc[2] != 0.f) {
      valid += 1;
      const float* Vc = L.V + 3 * (size_t)i;
      float p[3], nn[3];
#pragma unroll
      for (int r = 0; r < 3; ++r) {
        p[r] = R[3 * r] * Vc[0] + R[3 * r + 1] * Vc[1] + R[3 * r + 2] * Vc[2] + t[r];
        nn[r] = R[3 * r] * Nc[0] + R[3 * r + 1] * Nc[1] + R[3 * r + 2] * Nc[2];
      }
      const float d0 = p[0] - tp[0], d1 = p[1] - tp[1], d2 = p[2] - tp[2];
      const float x0 = Rp[0] * d0 + Rp[3] * d1 + Rp[6] * d2;
      const float x1 = Rp[1] * d0 + Rp[4] * d1 + Rp[7] * d2;
      const float x2 = Rp[2] * d0 + Rp[5] * d1 + Rp[8] * d2;
      if (x2 > 1e-9f) {
        const float uf = floorf(L.fx * x0 / x2 + L.cx + 0.5f), vf = floorf(L.fy * x1 / x2 + L.cy + 0.5f);
        if (uf >= 0.f && uf <= (float)(Lw - 1) && vf >= 0.f && vf <= (float)(Lh - 1)) {
          const size_t mp = (size_t)((int)vf * L.stride) * a.mW + (size_t)((int)uf * L.stride);
          const float q0 = a.mV[3 * mp], q1 = a.mV[3 * mp + 1], q2 = a.mV[3 * mp + 2];
          const float m0 = a.mN[3 * mp], m1 = a.mN[3 * mp + 1], m2 = a.mN[3 * mp + 2];
          const float e0 = p[0] - q0, e1 = p[1] - q1, e2 = p[2] - q2;
          if ((m0 != 0.f || m1 != 0.f || m2 != 0.f) && sqrtf(e0 * e0 + e1 * e1 + e2 * e2) < a.dist_max &&
              nn[0] * m0 + nn[1] * m1 + nn[2] * m2 > a.cos_max) {
            const float r = e0 * m0 + e1 * m1 + e2 * m2;
            const float J[6] = {m0, m1, m2, p[1] * m2 - p[2] * m1, p[2] * m0 - p[0] * m2, p[0] * m1 - p[1] * m0};
            int k = 0;
#pragma unroll
            for (int x = 0; x < 6; ++x)
#pragma unroll
              for (int y = x; y < 6; ++y) s[k++] += J[x] * J[y];
#pragma unroll
            for (int x = 0; x < 6; ++x) s[21 + x] += J[x] * r;
            s[27] += r * r;
            s[28] += 1.f;
          }
        }
      }
    }
  }
  // CTA reduction in double (warp shuffles, then the warps' rows)
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < kIcpSums; ++k) {
    double x = (double)s[k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xFFFFFFFFu, x, o);
    if (lane == 0) red[w][k] = x;
  }
  __shared__ int svalid[kIcpThreads / 32];
  const int vw = __reduce_add_sync(0xFFFFFFFFu, valid);
  if (lane == 0) svalid[w] = vw;
  __syncthreads();
  if (threadIdx.x < kIcpSums) {
    double x = 0.0;
    for (int j = 0; j < kIcpThreads / 32; ++j) x += red[j][threadIdx.x];
    partial[(size_t)blockIdx.x * 32 + threadIdx.x] = x;
  }
  if (threadIdx.x == 0) {
    int cv = 0;
    for (int j = 0; j < kIcpThreads / 32; ++j) cv += svalid[j];
    partial[(size_t)blockIdx.x * 32 + 29] = (double)cv;
  }
  // last-CTA election: the sums are visible device-wide before the ticket is taken
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(&pose->ticket, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  icp_solve_cta(partial, gridDim.x, pose, a.eps);
  if (threadIdx.x == 0) pose->ticket = 0;  // for the next step (stream-ordered)
}

// one CTA (256 threads): total the CTA sums, solve A xi = -b (Cholesky), pose <- exp(xi) pose
__device__ void icp_solve_cta(const double* partial, int nblk, DevPose* pose, double eps) {
  __shared__ double tot[32];
  __shared__ double part[8][32];
  {  // 30 sums x 8 interleaved chunks of the CTA partials, then the 8 chunks per sum
    // 8 independent accumulators keep 8 loads in flight per thread (the partials are L2-resident;
    // a dependent chain of ~nblk/8 L2 round trips would dominate small levels)
    const int v = threadIdx.x & 31, c = threadIdx.x >> 5;
    double x = 0.0;
    if (v < 30) {
      double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      int b = c;
      for (; b + 56 < nblk; b += 64) {
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[j] += __ldcg(partial + (size_t)(b + 8 * j) * 32 + v);
      }
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (b + 8 * j < nblk) acc[j] += __ldcg(partial + (size_t)(b + 8 * j) * 32 + v);
      x = ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
    }
    part[c][v] = x;
    __syncthreads();
    if (threadIdx.x < 30) {
      double y = 0.0;
      for (int k = 0; k < 8; ++k) y += part[k][threadIdx.x];
      tot[threadIdx.x] = y;
    }
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  double R0[9], t0[3];  // the current pose, loaded while the system is assembled
  for (int e = 0; e < 9; ++e) R0[e] = pose->R[e];
  for (int e = 0; e < 3; ++e) t0[e] = pose->t[e];
  double A[6][6], b[6];
  int k = 0;
  for (int x = 0; x < 6; ++x)
    for (int y = x; y < 6; ++y) { A[x][y] = tot[k]; A[y][x] = tot[k]; ++k; }
  for (int x = 0; x < 6; ++x) b[x] = tot[21 + x];
  pose->energy = tot[27];
  pose->inliers = (int32_t)tot[28];
  pose->valid = (int32_t)tot[29];
  if (tot[28] < 6.0) {
    pose->degenerate = 1;
    pose->stop = 1;
    return;
  }
  // Cholesky A = L L^T; a pivot below 1e-12 of the largest diagonal: rank deficient (R-ICP-GN)
  double dmax = 0.0;
  for (int x = 0; x < 6; ++x) dmax = fmax(dmax, A[x][x]);
  double Lc[6][6] = {};
  double inv[6];
  double pmin = 1.0;
  for (int j = 0; j < 6; ++j) {
    double d = A[j][j];
    for (int m = 0; m < j; ++m) d -= Lc[j][m] * Lc[j][m];
    pmin = fmin(pmin, d / dmax);
    if (!(d > 1e-12 * dmax)) {
      pose->pivot = pmin;
      pose->degenerate = 1;
      pose->stop = 1;
      return;
    }
    Lc[j][j] = sqrt(d);
    inv[j] = 1.0 / Lc[j][j];  // one division per pivot (a serial single-thread chain: keep it short)
    for (int i = j + 1; i < 6; ++i) {
      double s = A[i][j];
      for (int m = 0; m < j; ++m) s -= Lc[i][m] * Lc[j][m];
      Lc[i][j] = s * inv[j];
    }
  }
  pose->pivot = pmin;
  double y[6], xi[6];
  for (int i = 0; i < 6; ++i) {
    double s = -b[i];
    for (int m = 0; m < i; ++m) s -= Lc[i][m] * y[m];
    y[i] = s * inv[i];
  }
  for (int i = 5; i >= 0; --i) {
    double s = y[i];
    for (int m = i + 1; m < 6; ++m) s -= Lc[m][i] * xi[m];
    xi[i] = s * inv[i];
  }
  // exp of the twist (v, w): Rodrigues rotation, translation v (left-multiplied increment)
  const double w0 = xi[3], w1 = xi[4], w2 = xi[5];
  const double th = sqrt(w0 * w0 + w1 * w1 + w2 * w2);
  const double K[9] = {0, -w2, w1, w2, 0, -w0, -w1, w0, 0};
  double K2[9];
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) K2[3 * r + c] = K[3 * r] * K[c] + K[3 * r + 1] * K[3 + c] + K[3 * r + 2] * K[6 + c];
  // sin(th)/th and (1-cos th)/th^2: their Taylor series for th < 1e-2 (the first omitted terms,
  // th^8/9! and th^8/10!, are below 1e-21), else the closed forms
  double ca, cb;
  const double th2 = th * th;
  if (th < 1e-2) {
    ca = 1.0 - th2 / 6.0 * (1.0 - th2 / 20.0 * (1.0 - th2 / 42.0));
    cb = 0.5 - th2 / 24.0 * (1.0 - th2 / 30.0 * (1.0 - th2 / 56.0));
  } else {
    ca = sin(th) / th;
    cb = (1.0 - cos(th)) / th2;
  }
  double dR[9];
  for (int e = 0; e < 9; ++e) dR[e] = (e % 4 == 0 ? 1.0 : 0.0) + ca * K[e] + cb * K2[e];
  double R[9], t[3];
  for (int r = 0; r < 3; ++r) {
    for (int c = 0; c < 3; ++c) R[3 * r + c] = dR[3 * r] * R0[c] + dR[3 * r + 1] * R0[3 + c] + dR[3 * r + 2] * R0[6 + c];
    t[r] = dR[3 * r] * t0[0] + dR[3 * r + 1] * t0[1] + dR[3 * r + 2] * t0[2] + xi[r];
  }
  for (int e = 0; e < 9; ++e) pose->R[e] = R[e];
  for (int e = 0; e < 3; ++e) pose->t[e] = t[e];
  pose->steps += 1;
  double nx = 0.0;
  for (int e = 0; e < 6; ++e) nx += xi[e] * xi[e];
  if (sqrt(nx) < eps) pose->stop = 1;
}

inline size_t up256(size_t x) { return (x + 255) / 256 * 256; }

struct TrackLayout {
  size_t depth[kIcpMaxLevels], V[kIcpMaxLevels], N[kIcpMaxLevels];
  size_t partial, pose, total;
};
TrackLayout track_layout(int W, int H, int levels) {
  TrackLayout L{};
  size_t o = 0;
  auto take = [&](size_t b) { size_t at = o; o = up256(o + b); return at; };
  for (int l = 0; l < levels; ++l) {
    const size_t n = (size_t)(W >> l) * (H >> l);
    L.depth[l] = take(4 * n);
    L.V[l] = take(12 * n);
    L.N[l] = take(12 * n);
  }
  L.partial = take(8 * 32 * (((size_t)W * H + kIcpThreads - 1) / kIcpThreads));
  L.pose = take(sizeof(DevPose));
  L.total = o;
  return L;
}

}  // namespace
}  // namespace gps

using namespace gps;

extern "C" {

size_t gps_track_workspace_size(const gps_intrinsics* K, int32_t levels) {
  if (!K || K->width <= 0 || K->height <= 0 || levels < 1 || levels > kIcpMaxLevels) return 0;
  return track_layout(K->width, K->height, levels).total;
}

}  // extern "C"

static gps_status track_impl(const gps_intrinsics* K, const uint16_t* depth, float depth_scale,
                             const float* model_vertex, const float* model_normal, const PoseSrc& src,
                             const gps_icp_config* cfg, void* ws, size_t ws_bytes, gps_pose* out_pose,
                             gps_track_result* out_res, gps_stream_t stream, const char* who) {
  const std::string w_(who);
  if (!K || !depth || !model_vertex || !model_normal || !cfg || !ws) return invalid(w_ + ": null argument");
  if (K->width <= 0 || K->height <= 0 || !(depth_scale > 0)) return invalid(w_ + ": bad intrinsics");
  if (cfg->levels < 1 || cfg->levels > kIcpMaxLevels || !(cfg->dist_max > 0) || !(cfg->depth_max > cfg->depth_min) ||
      cfg->fallback < 0 || cfg->fallback > 1 || !(cfg->min_inlier_px_frac >= 0.f && cfg->min_inlier_px_frac <= 1.f) ||
      !(cfg->min_pivot_ratio >= 0.f) || cfg->filter_radius < 0 || cfg->filter_radius > 7 ||
      (cfg->filter_radius > 0 && !(cfg->filter_sigma_s > 0.f && cfg->filter_sigma_r > 0.f)))
    return invalid(w_ + ": bad config");
  for (int l = 0; l < cfg->levels; ++l)
    if (cfg->iters[l] < 1 || (K->width >> l) < 3 || (K->height >> l) < 3) return invalid(w_ + ": bad level");
  if ((reinterpret_cast<uintptr_t>(depth) & 1u) != 0) return invalid(w_ + ": depth must be 2-byte aligned");
  const TrackLayout Lw = track_layout(K->width, K->height, cfg->levels);
  if (ws_bytes < Lw.total) {
    set_error(w_ + ": workspace too small");
    return GPS_ERR_WORKSPACE_TOO_SMALL;
  }
  cudaStream_t s = as_stream(stream);
  char* w = static_cast<char*>(ws);
  DevPose* dp = reinterpret_cast<DevPose*>(w + Lw.pose);
  k_icp_init<<<1, 1, 0, s>>>(src, dp);
  GPS_CHECK_LAUNCH("k_icp_init");
  const int n0 = K->width * K->height;
  if (cfg->filter_radius > 0) {
    const double ss = cfg->filter_sigma_s, sr = cfg->filter_sigma_r;
    k_icp_bilateral<<<dim3((K->width + 31) / 32, (K->height + 7) / 8), 256, 0, s>>>(
        depth, K->width, K->height, 1.0f / depth_scale, cfg->depth_min, cfg->depth_max, cfg->filter_radius,
        (float)(1.0 / (2.0 * ss * ss)), (float)(1.0 / (2.0 * sr * sr)), reinterpret_cast<float*>(w + Lw.depth[0]));
    GPS_CHECK_LAUNCH("k_icp_bilateral");
  } else {
    k_icp_depth<<<(n0 + 255) / 256, 256, 0, s>>>(depth, n0, 1.0f / depth_scale, cfg->depth_min, cfg->depth_max,
                                                 reinterpret_cast<float*>(w + Lw.depth[0]));
    GPS_CHECK_LAUNCH("k_icp_depth");
  }
  for (int l = 1; l < cfg->levels; ++l) {
    const int Wd = K->width >> l, Hd = K->height >> l;
    k_icp_down<<<dim3((Wd + 127) / 128, Hd), 128, 0, s>>>(reinterpret_cast<const float*>(w + Lw.depth[l - 1]),
                                                          K->width >> (l - 1), reinterpret_cast<float*>(w + Lw.depth[l]),
                                                          Wd, Hd);
    GPS_CHECK_LAUNCH("k_icp_down");
  }
  Assoc a;
  a.mV = model_vertex;
  a.mN = model_normal;
  a.mW = K->width;
  a.mH = K->height;
  a.dist_max = cfg->dist_max;
  a.cos_max = (float)std::cos((double)cfg->angle_max_deg * M_PI / 180.0);
  a.eps = (double)cfg->eps;
  double* partial = reinterpret_cast<double*>(w + Lw.partial);
  for (int l = cfg->levels - 1; l >= 0; --l) {  // coarse -> fine
    Level L;
    L.W = K->width >> l;
    L.H = K->height >> l;
    const double sc = std::ldexp(1.0, -l);
    L.fx = (float)(K->fx * sc);
    L.fy = (float)(K->fy * sc);
    L.cx = (float)((K->cx + 0.5) * sc - 0.5);
    L.cy = (float)((K->cy + 0.5) * sc - 0.5);
    L.depth = reinterpret_cast<const float*>(w + Lw.depth[l]);
    L.V = reinterpret_cast<float*>(w + Lw.V[l]);
    L.N = reinterpret_cast<float*>(w + Lw.N[l]);
    L.stride = 1 << l;
    k_icp_maps<<<dim3((L.W + 15) / 16, (L.H + 15) / 16), 256, 0, s>>>(L, dp);
    GPS_CHECK_LAUNCH("k_icp_maps");
    const int nblk = std::min((L.W * L.H + kIcpThreads - 1) / kIcpThreads, 148 * 3);  // grid-stride, one wave at 3 CTAs/SM
    for (int it = 0; it < cfg->iters[l]; ++it) {
      k_icp_step<<<nblk, kIcpThreads, 0, s>>>(L, a, dp, partial);
      GPS_CHECK_LAUNCH("k_icp_step");
    }
  }
  k_icp_export<<<1, 1, 0, s>>>(dp, cfg->min_inlier_frac,
                               (double)cfg->min_inlier_px_frac * (double)K->width * (double)K->height,
                               cfg->min_pivot_ratio, cfg->fallback, out_pose, out_res);
  GPS_CHECK_LAUNCH("k_icp_export");
  return GPS_OK;
}

extern "C" {

gps_status gps_track_sync(const gps_intrinsics* K, const uint16_t* depth, float depth_scale, const float* model_vertex,
                          const float* model_normal, const gps_pose* T_model, const gps_pose* T_init,
                          const gps_icp_config* cfg, void* ws, size_t ws_bytes, gps_track_result* out,
                          gps_stream_t stream) {
  if (!T_model || !T_init || !out) return invalid("gps_track_sync: null argument");
  PoseSrc src{};
  src.init = *T_init;
  src.model = *T_model;
  gps_track_result* dres = nullptr;
  cudaStream_t s = as_stream(stream);
  GPS_CHECK_CUDA(cudaMallocAsync(&dres, sizeof(gps_track_result), s));
  gps_status st = track_impl(K, depth, depth_scale, model_vertex, model_normal, src, cfg, ws, ws_bytes, nullptr,
                             dres, stream, "gps_track_sync");
  if (st == GPS_OK) GPS_CHECK_CUDA(cudaMemcpyAsync(out, dres, sizeof(*out), cudaMemcpyDeviceToHost, s));
  GPS_CHECK_CUDA(cudaFreeAsync(dres, s));
  GPS_CHECK_CUDA(cudaStreamSynchronize(s));
  return st;
}

gps_status gps_pose_extrapolate(const gps_pose* T_a_dev, const gps_pose* T_b_dev, gps_pose* T_out_dev,
                                gps_stream_t stream) {
  if (!T_a_dev || !T_b_dev || !T_out_dev) return invalid("gps_pose_extrapolate: null argument");
  if (T_out_dev == T_a_dev || T_out_dev == T_b_dev) return invalid("gps_pose_extrapolate: output aliases an input");
  k_pose_extrapolate<<<1, 1, 0, as_stream(stream)>>>(T_a_dev, T_b_dev, T_out_dev);
  GPS_CHECK_LAUNCH("k_pose_extrapolate");
  return GPS_OK;
}

gps_status gps_track_async(const gps_intrinsics* K, const uint16_t* depth, float depth_scale,
                           const float* model_vertex, const float* model_normal, const gps_pose* T_model_dev,
                           const gps_pose* T_init_dev, const gps_pose* T_fail_dev, const gps_icp_config* cfg,
                           void* ws, size_t ws_bytes, gps_pose* T_out_dev, gps_track_result* result_dev,
                           gps_stream_t stream) {
  if (!T_model_dev || !T_init_dev || !T_out_dev) return invalid("gps_track_async: null argument");
  PoseSrc src{};
  src.dinit = T_init_dev;
  src.dmodel = T_model_dev;
  src.dfail = T_fail_dev;
  return track_impl(K, depth, depth_scale, model_vertex, model_normal, src, cfg, ws, ws_bytes, T_out_dev, result_dev,
                    stream, "gps_track_async");
}

}  // extern "C"
