// render.cu -- the Gaussian half of the mapping step for sm_100a: gps_render, gps_refine_step,
// gps_adam_step and their workspace.
//
// Paper: GPS-SLAM (arXiv 2509.11574).  Gaussians "following 3DGS"; second-pass
// rendering Eqs. 1-3 with depth culling against the SDF depth, composite Eq. 4
// (W_t = 1); L1 loss Eq. 7; optimisation with Libtorch's Adam at
// the learning rates of App. C.  Readings R-*: DESIGN.md §3; prescribed fp32 for the
// tile-membership fields: DESIGN.md §4.3.
//
// Pipeline of one view:
//   k_preprocess  per Gaussian: projection -> 48-B splat record, tile counts, zero 2D grads
//   k_scan        one CTA: exclusive scan of the tile counts (MSD radix pass on the tile digit)
//   k_emit        per Gaussian: scatter its index into every touched tile's bucket
//   k_sort_blend  one CTA per tile: sort the bucket by (depth bits, index) in shared memory,
//                 front-to-back blend with early termination at the SDF depth, composite,
//                 fused L1 partials; the last CTA finalises the loss deterministically
//   k_backward    one CTA per tile: a half-warp per list entry walks the entry's footprint inside
//                 the tile, accumulates the 9 2D gradients in registers, reduce-scatters them over
//                 its 16 lanes and adds each total to the entry's 2D gradient slot (one atomic each)
//   k_chain       per Gaussian with a gradient: 2D -> raw-parameter chain rule into a 128-B
//                 record (11 raw gradients, clamped colour gradient, SH basis)
//   k_adam        dense Adam streamed over float4 units of every parameter array
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#define GPS_CHK_VAR g_chk_render
#include "common.cuh"
#include "prof.cuh"

namespace gps {
__device__ unsigned long long g_chk_render = 0ull;
unsigned long long check_word_take_render() {
  unsigned long long w = 0ull, z = 0ull;
  cudaMemcpyFromSymbol(&w, g_chk_render, sizeof(w));
  cudaMemcpyToSymbol(g_chk_render, &z, sizeof(z));
  return w;
}

constexpr int kMaxList = 2048;  // entries a tile sorts in shared memory (16 KB of keys)
constexpr uint32_t kWsMagic = 0x47505357u;  // "GPSW"

// Pair-list overflow (K > capacity: pairs were dropped) is latched in a process-wide host-mapped
// flag that k_scan sets; the next gps_render / gps_refine_step / gps_render_stats_sync call sees
// it without synchronising, returns GPS_ERR_WORKSPACE_TOO_SMALL and clears it.
struct OverflowFlag {
  uint32_t* host = nullptr;
  uint32_t* dev = nullptr;
};
OverflowFlag& overflow_flag() {
  static OverflowFlag f = [] {
    OverflowFlag o;
    if (cudaHostAlloc(reinterpret_cast<void**>(&o.host), sizeof(uint32_t), cudaHostAllocMapped | cudaHostAllocPortable) ==
            cudaSuccess &&
        cudaHostGetDevicePointer(reinterpret_cast<void**>(&o.dev), o.host, 0) == cudaSuccess) {
      *o.host = 0;
    } else {
      o.host = nullptr;
      o.dev = nullptr;
    }
    return o;
  }();
  return f;
}

uint32_t* overflow_flag_dev() { return overflow_flag().dev; }

struct WsHeader {
  uint32_t magic, tile, tiles_x, tiles_y;
  uint32_t width, height, n_tiles, pad0;
  uint64_t cap_pairs;
  int64_t n;
  // ---- zeroed by every render (one memset together with counts and cursor) ----
  uint32_t K;          // total pairs
  uint32_t overflow;   // K > cap
  uint32_t n_visible;  // Gaussians surviving culls
  uint32_t mask_count; // |M| of the L1 mask
  uint32_t ticket;     // last-CTA election for the loss
  uint32_t n_extra;    // work items beyond one per tile (lists longer than 256 entries)
  uint32_t n_part;     // partial slots handed to long lists (the blend's split)
  uint32_t n_long;     // tiles whose list is longer than 256 entries (k_sort_long's work)
  // ---- static: where this render's lists live (refine and render layouts differ) ----
  uint64_t off_vals, off_offsets, off_tile_end;
};


struct WsLayout {
  size_t hdr, counts, cursor, bigcounts, offsets, tile_end, loss_part, records, ranks, grad2d, rec3, cgj, vals, keys,
      cstar, wg, gbuf, extra, pbase, tick, part, longl, total;
  uint32_t extra_cap, part_cap;
  size_t zero_begin, zero_bytes;
};

inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

WsLayout ws_layout(int64_t n, int W, int H, int tile, int64_t cap, int64_t n_params, bool refine, bool gbuf) {
  const size_t tiles = (size_t)((W + tile - 1) / tile) * ((H + tile - 1) / tile);
  WsLayout L{};
  size_t o = 0;
  auto take = [&](size_t bytes) {
    size_t at = o;
    o = align_up(o + bytes, 256);
    return at;
  };
  L.hdr = take(sizeof(WsHeader));
  L.counts = take(4 * tiles);     // per tile: entries of Gaussians spanning <= 4 tiles
  L.cursor = take(4 * tiles);     // per tile: scatter cursor of the others
  L.bigcounts = take(4 * tiles);  // per tile: entries of Gaussians spanning > 4 tiles
  L.tick = take(4 * tiles);       // per tile: chunks of a split long list finished by the blend
  L.zero_begin = L.hdr + offsetof(WsHeader, K);
  L.zero_bytes = L.tick + 4 * tiles - L.zero_begin;
  L.offsets = take(4 * (tiles + 1));
  L.tile_end = take(4 * tiles);
  L.loss_part = take(4 * tiles);
  L.records = take(64 * (size_t)std::max<int64_t>(n, 1));
  L.ranks = take(16 * (size_t)std::max<int64_t>(n, 1));
  L.grad2d = refine ? take(48 * (size_t)std::max<int64_t>(n, 1)) : 0;
  L.rec3 = refine ? take(128 * (size_t)std::max<int64_t>(n, 1)) : 0;
  L.cgj = refine ? take(48 * (size_t)std::max<int64_t>(n, 1)) : 0;
  L.vals = take(4 * (size_t)cap);
  L.keys = take(8 * (size_t)cap);
  L.extra_cap = (uint32_t)std::min<int64_t>(cap / 256 + 1, 0x7FFFFFFF);
  L.extra = take(8 * (size_t)L.extra_cap);  // {tile, chunk} work items of long lists
  L.pbase = take(4 * tiles);                 // per long list: its first partial slot (or ~0)
  L.part_cap = 8192;                         // 8192 chunks of 256 entries (32 MB) per render
  L.part = take(16 * 256 * (size_t)L.part_cap);
  L.longl = take(4 * tiles);                 // the tiles with long lists
  L.cstar = refine ? take(12 * (size_t)W * H) : 0;
  L.wg = refine ? take(4 * (size_t)W * H) : 0;
  L.gbuf = gbuf ? take(4 * (size_t)n_params) : 0;
  L.total = o;
  return L;
}

int64_t default_cap(int64_t n, int64_t cfg_cap) { return cfg_cap > 0 ? cfg_cap : 32 * n + 65536; }

// --------------------------------------------------------------------------------------------
struct Cam {
  float fx, fy, cx, cy;
  int W, H;
  float R[9], t[3];
};

struct RenderArgs {
  Cam cam;
  float eps, alpha_min, near_z, lowpass;
  float ln_inv_amin;  // fl(-ln alpha_min), computed on the host in double
  int tile, tiles_x, tiles_y;
  int64_t n;
  int deg, nc;
  uint32_t cap;
};

// SH basis of 3DGS (degree <= 3), real, at unit direction (x, y, z)
__device__ __forceinline__ void sh_basis(float x, float y, float z, int deg, float* Y) {
  const float C0 = 0.28209479177387814f, C1 = 0.4886025119029199f;
  Y[0] = C0;
  if (deg < 1) return;
  Y[1] = -C1 * y; Y[2] = C1 * z; Y[3] = -C1 * x;
  if (deg < 2) return;
  const float xx = x * x, yy = y * y, zz = z * z;
  Y[4] = 1.0925484305920792f * x * y;
  Y[5] = -1.0925484305920792f * y * z;
  Y[6] = 0.31539156525252005f * (2.f * zz - xx - yy);
  Y[7] = -1.0925484305920792f * x * z;
  Y[8] = 0.5462742152960396f * (xx - yy);
  if (deg < 3) return;
  Y[9] = -0.5900435899266435f * y * (3.f * xx - yy);
  Y[10] = 2.890611442640554f * x * y * z;
  Y[11] = -0.4570457994644658f * y * (4.f * zz - xx - yy);
  Y[12] = 0.3731763325901154f * z * (2.f * zz - 3.f * xx - 3.f * yy);
  Y[13] = -0.4570457994644658f * x * (4.f * zz - xx - yy);
  Y[14] = 1.445305721320277f * z * (xx - yy);
  Y[15] = -0.5900435899266435f * x * (xx - 3.f * yy);
}

// d Y_k / d(x,y,z), accumulated as ddir += w_k * dY_k
__device__ __forceinline__ void sh_basis_vjp(float x, float y, float z, int deg, const float* w, float* dd) {
  const float C1 = 0.4886025119029199f;
  dd[0] = dd[1] = dd[2] = 0.f;
  if (deg < 1) return;
  dd[1] += -C1 * w[1]; dd[2] += C1 * w[2]; dd[0] += -C1 * w[3];
  if (deg < 2) return;
  const float xx = x * x, yy = y * y, zz = z * z;
  const float a0 = 1.0925484305920792f, a1 = -1.0925484305920792f, a2 = 0.31539156525252005f,
              a3 = -1.0925484305920792f, a4 = 0.5462742152960396f;
  dd[0] += a0 * y * w[4]; dd[1] += a0 * x * w[4];
  dd[1] += a1 * z * w[5]; dd[2] += a1 * y * w[5];
  dd[0] += -2.f * a2 * x * w[6]; dd[1] += -2.f * a2 * y * w[6]; dd[2] += 4.f * a2 * z * w[6];
  dd[0] += a3 * z * w[7]; dd[2] += a3 * x * w[7];
  dd[0] += 2.f * a4 * x * w[8]; dd[1] += -2.f * a4 * y * w[8];
  if (deg < 3) return;
  const float b0 = -0.5900435899266435f, b1 = 2.890611442640554f, b2 = -0.4570457994644658f,
              b3 = 0.3731763325901154f, b4 = -0.4570457994644658f, b5 = 1.445305721320277f,
              b6 = -0.5900435899266435f;
  dd[0] += b0 * 6.f * x * y * w[9]; dd[1] += b0 * (3.f * xx - 3.f * yy) * w[9];
  dd[0] += b1 * y * z * w[10]; dd[1] += b1 * x * z * w[10]; dd[2] += b1 * x * y * w[10];
  dd[0] += b2 * (-2.f * x * y) * w[11]; dd[1] += b2 * (4.f * zz - xx - 3.f * yy) * w[11]; dd[2] += b2 * 8.f * y * z * w[11];
  dd[0] += b3 * (-6.f * x * z) * w[12]; dd[1] += b3 * (-6.f * y * z) * w[12]; dd[2] += b3 * (6.f * zz - 3.f * xx - 3.f * yy) * w[12];
  dd[0] += b4 * (4.f * zz - 3.f * xx - yy) * w[13]; dd[1] += b4 * (-2.f * x * y) * w[13]; dd[2] += b4 * 8.f * x * z * w[13];
  dd[0] += b5 * 2.f * x * z * w[14]; dd[1] += b5 * (-2.f * y * z) * w[14]; dd[2] += b5 * (xx - yy) * w[14];
  dd[0] += b6 * (3.f * xx - 3.f * yy) * w[15]; dd[1] += b6 * (-6.f * x * y) * w[15];
}

// Everything the forward and backward need about one Gaussian in one view.  The fields that
// decide tile membership and the sort key (X, Sigma_2D, p_hat, rect) follow the prescribed fp32
// sequence of DESIGN.md §4.3 (the CPU oracle evaluates the same sequence independently).
struct Proj {
  bool culled;
  float X[3];
  float s[3], qh[4], qn, Rq[9], M[9], S[9];
  float cu, cv;
  bool clx, cly;
  float J00, J02, J11, J12, T[6];
  float cxx, cxy, cyy, det, ca, cb, cc;
  float px, py;
  int x0, y0, x1, y1;
};

__device__ __forceinline__ void project_p32(const Cam& c, float near_z, float lowpass, const float* p,
                                            const float* ls, const float* q, Proj& g) {
  g.culled = true;
  const float D0 = psub(p[0], c.t[0]), D1 = psub(p[1], c.t[1]), D2 = psub(p[2], c.t[2]);
#pragma unroll
  for (int k = 0; k < 3; ++k) g.X[k] = pdot3(c.R[0 * 3 + k], D0, c.R[1 * 3 + k], D1, c.R[2 * 3 + k], D2);
  if (!(g.X[2] > near_z)) return;
#pragma unroll
  for (int k = 0; k < 3; ++k) g.s[k] = (float)exp((double)ls[k]);
  float qn2 = padd(pmul(q[0], q[0]), pmul(q[1], q[1]));
  qn2 = padd(qn2, pmul(q[2], q[2]));
  qn2 = padd(qn2, pmul(q[3], q[3]));
  g.qn = psqrt(qn2);
  const float w = pdiv(q[0], g.qn), x = pdiv(q[1], g.qn), y = pdiv(q[2], g.qn), z = pdiv(q[3], g.qn);
  g.qh[0] = w; g.qh[1] = x; g.qh[2] = y; g.qh[3] = z;
  float* Rq = g.Rq;
  Rq[0] = psub(1.0f, pmul(2.0f, padd(pmul(y, y), pmul(z, z))));
  Rq[1] = pmul(2.0f, psub(pmul(x, y), pmul(w, z)));
  Rq[2] = pmul(2.0f, padd(pmul(x, z), pmul(w, y)));
  Rq[3] = pmul(2.0f, padd(pmul(x, y), pmul(w, z)));
  Rq[4] = psub(1.0f, pmul(2.0f, padd(pmul(x, x), pmul(z, z))));
  Rq[5] = pmul(2.0f, psub(pmul(y, z), pmul(w, x)));
  Rq[6] = pmul(2.0f, psub(pmul(x, z), pmul(w, y)));
  Rq[7] = pmul(2.0f, padd(pmul(y, z), pmul(w, x)));
  Rq[8] = psub(1.0f, pmul(2.0f, padd(pmul(x, x), pmul(y, y))));
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int cc = 0; cc < 3; ++cc) g.M[3 * r + cc] = pmul(Rq[3 * r + cc], g.s[cc]);
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int cc = 0; cc < 3; ++cc)
      g.S[3 * r + cc] = pdot3(g.M[3 * r], g.M[3 * cc], g.M[3 * r + 1], g.M[3 * cc + 1], g.M[3 * r + 2], g.M[3 * cc + 2]);
  const float tanx = pdiv((float)c.W, pmul(2.0f, c.fx)), tany = pdiv((float)c.H, pmul(2.0f, c.fy));
  const float limx = pmul(1.3f, tanx), limy = pmul(1.3f, tany);
  const float txz = pdiv(g.X[0], g.X[2]), tyz = pdiv(g.X[1], g.X[2]);
  g.clx = (txz < -limx || txz > limx);
  g.cly = (tyz < -limy || tyz > limy);
  g.cu = txz < -limx ? -limx : (txz > limx ? limx : txz);
  g.cv = tyz < -limy ? -limy : (tyz > limy ? limy : tyz);
  const float tx = pmul(g.cu, g.X[2]), ty = pmul(g.cv, g.X[2]);
  const float z2 = pmul(g.X[2], g.X[2]);
  g.J00 = pdiv(c.fx, g.X[2]);
  g.J02 = -pdiv(pmul(c.fx, tx), z2);
  g.J11 = pdiv(c.fy, g.X[2]);
  g.J12 = -pdiv(pmul(c.fy, ty), z2);
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    g.T[k] = padd(pmul(g.J00, c.R[k * 3 + 0]), pmul(g.J02, c.R[k * 3 + 2]));
    g.T[3 + k] = padd(pmul(g.J11, c.R[k * 3 + 1]), pmul(g.J12, c.R[k * 3 + 2]));
  }
  float U[6];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int k = 0; k < 3; ++k)
      U[3 * a + k] = pdot3(g.T[3 * a], g.S[k], g.T[3 * a + 1], g.S[3 + k], g.T[3 * a + 2], g.S[6 + k]);
  const float sxx = pdot3(U[0], g.T[0], U[1], g.T[1], U[2], g.T[2]);
  const float sxy = pdot3(U[0], g.T[3], U[1], g.T[4], U[2], g.T[5]);
  const float syy = pdot3(U[3], g.T[3], U[4], g.T[4], U[5], g.T[5]);
  g.cxx = padd(sxx, lowpass);
  g.cxy = sxy;
  g.cyy = padd(syy, lowpass);
  g.det = psub(pmul(g.cxx, g.cyy), pmul(g.cxy, g.cxy));
  if (!(g.det > 0.0f)) return;
  g.ca = pdiv(g.cyy, g.det);
  g.cb = -pdiv(g.cxy, g.det);
  g.cc = pdiv(g.cxx, g.det);
  g.px = padd(pdiv(pmul(c.fx, g.X[0]), g.X[2]), c.cx);
  g.py = padd(pdiv(pmul(c.fy, g.X[1]), g.X[2]), c.cy);
  const float rx = pmul(3.0f, psqrt(g.cxx)), ry = pmul(3.0f, psqrt(g.cyy));
  float fx0 = floorf(psub(g.px, rx)), fx1 = ceilf(padd(g.px, rx));
  float fy0 = floorf(psub(g.py, ry)), fy1 = ceilf(padd(g.py, ry));
  fx0 = fmaxf(fx0, 0.0f);
  fy0 = fmaxf(fy0, 0.0f);
  fx1 = fminf(fx1, (float)(c.W - 1));
  fy1 = fminf(fy1, (float)(c.H - 1));
  if (!(fx0 <= fx1 && fy0 <= fy1)) return;
  g.x0 = (int)fx0; g.y0 = (int)fy0; g.x1 = (int)fx1; g.y1 = (int)fy1;
  g.culled = false;
}

struct SH {
  float Y[16];
  float dir[3], dnorm;
};

__device__ __forceinline__ void view_dir(const Cam& c, const float* p, int deg, SH& h) {
  const float d0 = p[0] - c.t[0], d1 = p[1] - c.t[1], d2 = p[2] - c.t[2];
  h.dnorm = sqrtf(d0 * d0 + d1 * d1 + d2 * d2);
  const float inv = 1.0f / h.dnorm;
  h.dir[0] = d0 * inv; h.dir[1] = d1 * inv; h.dir[2] = d2 * inv;
  sh_basis(h.dir[0], h.dir[1], h.dir[2], deg, h.Y);
}

// Pair membership, prescribed fp32 (the oracle evaluates the same sequence):
// q = Delta^T conic Delta with explicit fused multiply-adds; in iff q <= q_max, where
// q_max = min(9, 2 (L + ln sigma)) <=> the 3-sigma ellipse (R-FOOT) and alpha >= alpha_min.
__device__ __forceinline__ float pair_q(float px, float py, float a, float b2, float c, float x, float y) {
  const float dx = x - px, dy = y - py;
  const float inner = __fmaf_rn(pmul(b2, dx), dy, pmul(pmul(c, dy), dy));
  return __fmaf_rn(pmul(a, dx), dx, inner);
}
// Conservative test: can any pixel (x, y), x in [xa, xb], y in [ya, yb] (integers), pass the
// prescribed-fp32 membership pair_q(...) <= qmax?  Per row, the x-interval of the ellipse
// a dx^2 + 2b dx dy + c dy^2 <= qmax is centre px + m, half-width sqrt(m^2 - t); it is widened
// by 1e-5 of the magnitudes of its terms (about 100x the fp32 rounding of either computation)
// so that it only ever rejects strips no pixel of which passes.  Never decides membership.
__device__ __forceinline__ bool ellipse_meets_strip(float px, float py, float a, float b2, float c, float qmax,
                                                    int xa, int xb, int ya, int yb) {
  const float ia = 1.0f / a, hb = 0.5f * b2;
  for (int y = ya; y <= yb; ++y) {
    const float dy = (float)y - py;
    const float m = -hb * dy * ia;
    const float cq = c * dy * dy;
    const float t = (cq - qmax) * ia;
    const float r2 = m * m - t;
    const float marg = 1e-5f * (m * m + (cq + qmax) * ia) + 1e-4f;
    if (r2 + marg < 0.f) continue;
    const float h = sqrtf(r2 + marg) + 1e-3f;
    if (px + m - h <= (float)xb && px + m + h >= (float)xa) return true;
  }
  return false;
}

__device__ __forceinline__ float pair_qmax(float L, float lnsig) {
  return fminf(9.0f, pmul(2.0f, padd(L, lnsig)));
}

// ============================================================================================
// k_preprocess
// ============================================================================================
struct SplatPtrs {
  float4* rec;     // 4 float4 per Gaussian
  uint4* ranks;    // per Gaussian: its rank inside each of its (<= 4) tile buckets
  uint32_t* bigcounts;
  float4* grad2d;  // 3 float4 per Gaussian (nullable)
  float4* cgj;     // 3 float4 per Gaussian: colour/direction Jacobian + clamp bits (refine only)
  uint32_t* counts;
  WsHeader* hdr;
};

__device__ __forceinline__ void preprocess_one(const RenderArgs& a, const gps_gaussians& g, const SplatPtrs& w,
                                               int64_t i, int (&trect)[4]);

// Per Gaussian: the projection and record (preprocess_one), then, warp-cooperatively, the tile
// counts of footprints spanning more than 4 tiles (one lane per tile instead of a serial loop)
// and one aggregated n_visible update per warp.
__global__ void __launch_bounds__(256, 3) k_preprocess(RenderArgs a, gps_gaussians g, SplatPtrs w) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int tr[4] = {1, 0, 0, 0};  // tile rect tx0, tx1, ty0, ty1 of a listed Gaussian (tx0 > tx1: none)
  if (i < a.n) preprocess_one(a, g, w, i, tr);
  const bool listed = tr[0] <= tr[1];
  const bool big = listed && (tr[1] - tr[0] + 1) * (tr[3] - tr[2] + 1) > 4;
  const uint32_t lm = __ballot_sync(0xFFFFFFFFu, listed);
  const int lane = threadIdx.x & 31;
  if (lane == 0 && lm) atomicAdd(&w.hdr->n_visible, (uint32_t)__popc(lm));
  uint32_t bm = __ballot_sync(0xFFFFFFFFu, big);
  while (bm) {
    const int src = __ffs(bm) - 1;
    bm &= bm - 1u;
    const int tx0 = __shfl_sync(0xFFFFFFFFu, tr[0], src), tx1 = __shfl_sync(0xFFFFFFFFu, tr[1], src);
    const int ty0 = __shfl_sync(0xFFFFFFFFu, tr[2], src), ty1 = __shfl_sync(0xFFFFFFFFu, tr[3], src);
    const int wx = tx1 - tx0 + 1, cnt = wx * (ty1 - ty0 + 1);
    for (int k = lane; k < cnt; k += 32) {
      const int ty = ty0 + k / wx, tx = tx0 + k % wx;
      atomicAdd(&w.bigcounts[ty * a.tiles_x + tx], 1u);
    }
  }
}

__device__ __forceinline__ void preprocess_one(const RenderArgs& a, const gps_gaussians& g, const SplatPtrs& w,
                                               int64_t i, int (&trect)[4]) {
  if (w.grad2d) {
    const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
    w.grad2d[3 * i] = z; w.grad2d[3 * i + 1] = z; w.grad2d[3 * i + 2] = z;
  }
  Proj pr;
  project_p32(a.cam, a.near_z, a.lowpass, g.xyz + 3 * i, g.log_scale + 3 * i, g.rot + 4 * i, pr);
  if (pr.culled) {
    // an empty rect marks the record as not listed (never read by later kernels)
    w.rec[4 * i + 1] = make_float4(0.f, 0.f, 0.f, __uint_as_float(0xFFFFu));
    return;
  }
  SH h;
  view_dir(a.cam, g.xyz + 3 * i, a.deg, h);
  const float* sh = g.sh + (size_t)i * a.nc * 3;
  // all of the Gaussian's SH coefficients in flight at once (fully unrolled; twelve 16-byte
  // loads at degree 3, whose 192-byte rows are 16-byte aligned), instead of one dependent load
  // per coefficient
  const int nsh = 3 * a.nc;
  float shv[48];
  if (nsh == 48) {
#pragma unroll
    for (int j = 0; j < 12; ++j) {
      const float4 q = __ldg(reinterpret_cast<const float4*>(sh) + j);
      shv[4 * j] = q.x; shv[4 * j + 1] = q.y; shv[4 * j + 2] = q.z; shv[4 * j + 3] = q.w;
    }
  } else {
#pragma unroll
    for (int j = 0; j < 48; ++j) shv[j] = j < nsh ? __ldg(sh + j) : 0.f;
  }
  float col[3];
  uint32_t clamp = 0u;
#pragma unroll
  for (int ch = 0; ch < 3; ++ch) {
    float acc = 0.f;
#pragma unroll
    for (int k = 0; k < 16; ++k)
      if (k < a.nc) acc = fmaf(h.Y[k], shv[3 * k + ch], acc);
    col[ch] = fmaxf(acc + 0.5f, 0.0f);
    if (acc + 0.5f < 0.f) clamp |= 1u << ch;
  }
  if (w.cgj) {
    // d colour_ch / d dir_e for the backward's view-direction term (the chain then needs no SH)
    float Gc[9];
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) {
      float wk[16];
#pragma unroll
      for (int k = 0; k < 16; ++k) wk[k] = shv[3 * k + ch];  // zero beyond the degree
      sh_basis_vjp(h.dir[0], h.dir[1], h.dir[2], a.deg, wk, Gc + 3 * ch);
    }
    w.cgj[3 * i] = make_float4(Gc[0], Gc[1], Gc[2], Gc[3]);
    w.cgj[3 * i + 1] = make_float4(Gc[4], Gc[5], Gc[6], Gc[7]);
    w.cgj[3 * i + 2] = make_float4(Gc[8], __uint_as_float(clamp), 0.f, 0.f);
  }
  // ln(sigmoid(o)) rounded once from double: feeds the exact membership decision q <= q_max
  const float lnsig = (float)(-log1p(exp(-(double)__ldg(&g.opacity_raw[i]))));
  const uint32_t rx = (uint32_t)pr.x0 | ((uint32_t)pr.x1 << 16);
  const uint32_t ry = (uint32_t)pr.y0 | ((uint32_t)pr.y1 << 16);
  // p_hat in double: the backward's value path uses the offset of the exact centre from the
  // fp32 p_hat that makes the (exact) membership decisions -- fp32 p_hat carries ~1e-4 px of
  // rounding at x ~ 1000 px, which sign cancellation in a Gaussian's gradient sum would amplify
  float ddx, ddy;
  {
    const double D0 = (double)g.xyz[3 * i] - a.cam.t[0], D1 = (double)g.xyz[3 * i + 1] - a.cam.t[1],
                 D2 = (double)g.xyz[3 * i + 2] - a.cam.t[2];
    const double X0 = a.cam.R[0] * D0 + a.cam.R[3] * D1 + a.cam.R[6] * D2;
    const double X1 = a.cam.R[1] * D0 + a.cam.R[4] * D1 + a.cam.R[7] * D2;
    const double iz = 1.0 / (a.cam.R[2] * D0 + a.cam.R[5] * D1 + a.cam.R[8] * D2);
    ddx = (float)((double)a.cam.fx * X0 * iz + (double)a.cam.cx - (double)pr.px);
    ddy = (float)((double)a.cam.fy * X1 * iz + (double)a.cam.cy - (double)pr.py);
  }
  w.rec[4 * i + 0] = make_float4(pr.px, pr.py, pr.ca, pr.cb);
  w.rec[4 * i + 1] = make_float4(pr.cc, lnsig, pr.X[2], __uint_as_float(rx));
  w.rec[4 * i + 2] = make_float4(col[0], col[1], col[2], __uint_as_float(ry));
  w.rec[4 * i + 3] = make_float4(ddx, ddy, 0.f, 0.f);
  const int tx0 = pr.x0 / a.tile, tx1 = pr.x1 / a.tile, ty0 = pr.y0 / a.tile, ty1 = pr.y1 / a.tile;
  trect[0] = tx0; trect[1] = tx1; trect[2] = ty0; trect[3] = ty1;
  if ((tx1 - tx0 + 1) * (ty1 - ty0 + 1) <= 4) {
    // the count atomic's old value is this Gaussian's slot inside the tile bucket: k_emit
    // scatters without atomics
    uint32_t rk[4] = {0u, 0u, 0u, 0u};
    int k = 0;
    for (int ty = ty0; ty <= ty1; ++ty)
      for (int tx = tx0; tx <= tx1; ++tx) rk[k++] = atomicAdd(&w.counts[ty * a.tiles_x + tx], 1u);
    w.ranks[i] = make_uint4(rk[0], rk[1], rk[2], rk[3]);
  }
}

// ============================================================================================
// k_scan: exclusive scan of the per-tile counts (one CTA, 1024 threads x 4 consecutive tiles
// per pass: one pass up to 4096 tiles, i.e. 1280x720 at 16x16)
// ============================================================================================
__global__ void __launch_bounds__(1024) k_scan(const uint32_t* __restrict__ counts,
                                               const uint32_t* __restrict__ bigcounts, uint32_t* offsets,
                                               int n_tiles, WsHeader* hdr, WsHeader stat,
                                               uint32_t* sticky_overflow, uint2* extra, uint32_t extra_cap,
                                               uint32_t* pbase, uint32_t part_cap, uint32_t* longl) {
  __shared__ uint32_t warp_sums[32];
  __shared__ uint32_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int base = 0; base < n_tiles; base += 4096) {
    const int i0 = base + 4 * threadIdx.x;
    uint32_t c[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) c[k] = i0 + k < n_tiles ? counts[i0 + k] + bigcounts[i0 + k] : 0u;
    const uint32_t v = c[0] + c[1] + c[2] + c[3];
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) warp_sums[wid] = x;
    __syncthreads();
    if (wid == 0) {
      uint32_t sw = warp_sums[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, sw, o);
        if (lane >= o) sw += y;
      }
      warp_sums[lane] = sw;  // inclusive
    }
    __syncthreads();
    uint32_t excl = carry + (wid ? warp_sums[wid - 1] : 0u) + x - v;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (i0 + k < n_tiles) offsets[i0 + k] = excl;
      excl += c[k];
      // a list longer than 256 entries gives the backward one work item per further 256 (rare:
      // their order is irrelevant, the gradients are sums)
      if (c[k] > 256u && extra) {
        const uint32_t more = (c[k] + 255u) / 256u - 1u;
        const uint32_t at = atomicAdd(&hdr->n_extra, more);
        for (uint32_t q = 0; q < more && at + q < extra_cap; ++q) extra[at + q] = make_uint2((uint32_t)(i0 + k), q + 1u);
        // the blend splits the list only when all its chunks have work items and partial slots
        longl[atomicAdd(&hdr->n_long, 1u)] = (uint32_t)(i0 + k);
        const uint32_t pb = atomicAdd(&hdr->n_part, more + 1u);
        pbase[i0 + k] = (at + more <= extra_cap && pb + more + 1u <= part_cap) ? pb : ~0u;
      }
    }
    __syncthreads();
    if (threadIdx.x == 1023) carry = excl;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    offsets[n_tiles] = carry;
    hdr->magic = stat.magic; hdr->tile = stat.tile; hdr->tiles_x = stat.tiles_x; hdr->tiles_y = stat.tiles_y;
    hdr->width = stat.width; hdr->height = stat.height; hdr->n_tiles = stat.n_tiles;
    hdr->cap_pairs = stat.cap_pairs; hdr->n = stat.n;
    hdr->off_vals = stat.off_vals; hdr->off_offsets = stat.off_offsets; hdr->off_tile_end = stat.off_tile_end;
    hdr->K = carry;
    hdr->overflow = carry > stat.cap_pairs ? 1u : 0u;
    if (carry > stat.cap_pairs) {  // host-mapped and sticky: reported by the next call
      *reinterpret_cast<volatile uint32_t*>(sticky_overflow) = 1u;
      __threadfence_system();
    }
  }
}

// ============================================================================================
// k_emit: bucket each listed Gaussian into its tiles (order inside a bucket is arbitrary; the
// per-tile sort makes the final order unique)
// ============================================================================================
__global__ void __launch_bounds__(256) k_emit(RenderArgs a, const float4* __restrict__ rec,
                                              const uint4* __restrict__ ranks,
                                              const uint32_t* __restrict__ counts,
                                              const uint32_t* __restrict__ offsets, uint32_t* cursor,
                                              uint32_t* vals) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int tx0 = 1, tx1 = 0, ty0 = 0, ty1 = 0;
  if (i < a.n) {
    const float4 r1 = rec[4 * i + 1], r2 = rec[4 * i + 2];
    const uint32_t rx = __float_as_uint(r1.w), ry = __float_as_uint(r2.w);
    const int x0 = rx & 0xFFFF, x1 = rx >> 16, y0 = ry & 0xFFFF, y1 = ry >> 16;
    if (x0 <= x1) {  // else culled
      tx0 = x0 / a.tile; tx1 = x1 / a.tile; ty0 = y0 / a.tile; ty1 = y1 / a.tile;
    }
  }
  const bool listed = tx0 <= tx1;
  const bool big = listed && (tx1 - tx0 + 1) * (ty1 - ty0 + 1) > 4;
  if (listed && !big) {
    const uint4 r4 = ranks[i];
    const uint32_t rk[4] = {r4.x, r4.y, r4.z, r4.w};
    int k = 0;
    for (int ty = ty0; ty <= ty1; ++ty)
      for (int tx = tx0; tx <= tx1; ++tx) {
        const uint32_t pos = offsets[ty * a.tiles_x + tx] + rk[k++];
        GPS_DCHECK(ty * a.tiles_x + tx < a.tiles_x * a.tiles_y, CHK_TILE);
        GPS_DCHECK(pos < offsets[ty * a.tiles_x + tx + 1], CHK_LIST);  // inside its tile's range
        if (pos < a.cap) vals[pos] = (uint32_t)i;
      }
  }
  // large footprints: after the ranked entries of each tile, by an atomic cursor -- the warp
  // takes them one at a time, a lane per tile, so a footprint of T tiles costs ceil(T/32)
  // atomic round trips instead of T serial ones
  const int lane = threadIdx.x & 31;
  uint32_t bm = __ballot_sync(0xFFFFFFFFu, big);
  while (bm) {
    const int src = __ffs(bm) - 1;
    bm &= bm - 1u;
    const int sx0 = __shfl_sync(0xFFFFFFFFu, tx0, src), sx1 = __shfl_sync(0xFFFFFFFFu, tx1, src);
    const int sy0 = __shfl_sync(0xFFFFFFFFu, ty0, src), sy1 = __shfl_sync(0xFFFFFFFFu, ty1, src);
    const uint32_t gi = (uint32_t)__shfl_sync(0xFFFFFFFFu, (uint32_t)i, src);
    const int wx = sx1 - sx0 + 1, cnt = wx * (sy1 - sy0 + 1);
    for (int k = lane; k < cnt; k += 32) {
      const int t = (sy0 + k / wx) * a.tiles_x + sx0 + k % wx;
      const uint32_t pos = offsets[t] + counts[t] + atomicAdd(&cursor[t], 1u);
      GPS_DCHECK(t >= 0 && t < a.tiles_x * a.tiles_y, CHK_TILE);
      GPS_DCHECK(pos < offsets[t + 1], CHK_LIST);
      if (pos < a.cap) vals[pos] = gi;
    }
  }
}

// ============================================================================================
// sort helpers: bitonic network in its all-ascending form (the first comparator of every merge
// compares mirror images), which lets a list of any length n be sorted without padding
// ============================================================================================
template <typename Keys>
__device__ __forceinline__ void bitonic_sort(Keys keys, int n) {
  int P = 1, lgP = 0;
  while (P < n) {
    P <<= 1;
    ++lgP;
  }
  for (int lk = 1; lk <= lgP; ++lk) {
    const int k = 1 << lk;
    for (int lj = lk - 1; lj >= 0; --lj) {
      const int j = 1 << lj;  // powers of two: block/offset by shift and mask
      for (int c = threadIdx.x; c < (P >> 1); c += blockDim.x) {
        const int blk = c >> lj, off = c & (j - 1);
        int lo, hi;
        if (lj == lk - 1) {
          lo = (blk << lk) + off;
          hi = (blk << lk) + k - 1 - off;
        } else {
          lo = (blk << (lj + 1)) + off;
          hi = lo + j;
        }
        if (hi < n) {
          const uint64_t a = keys[lo], b = keys[hi];
          if (a > b) {
            keys[lo] = b;
            keys[hi] = a;
          }
        }
      }
      __syncthreads();
    }
  }
}

// ============================================================================================
// k_sort_long: tiles whose list is longer than kShortList entries are sorted here, by (depth bits,
// index) keys, one 512-thread CTA per tile (grid-stride over k_scan's list): a bitonic network in
// shared memory up to kLongSmem keys, in the global key buffer beyond.  The blend kernels rank-
// sort the short lists themselves and take the long ones as they are.  (A 128-thread blend CTA
// sorting a 6000-entry list in global memory was the whole kernel's tail: late cfg4 frames see
// ~50 such tiles where thousands of small Gaussians stack along a wall at grazing angles.)
// ============================================================================================
constexpr int kShortList = 256;
constexpr int kLongSmem = 2048;  // 16 KB of dynamic shared memory (longer lists sort in global memory)

__global__ void __launch_bounds__(512) k_sort_long(const float4* __restrict__ rec, const uint32_t* __restrict__ offsets,
                                                  uint32_t* vals, uint64_t* gkeys, const uint32_t* __restrict__ longl,
                                                  const WsHeader* hdr, uint32_t cap) {
  extern __shared__ __align__(16) uint64_t sk[];
  const uint32_t n_long = hdr->n_long;  // k_scan listed the tiles longer than kShortList
  for (uint32_t li = blockIdx.x; li < n_long; li += gridDim.x) {
    const int t = (int)longl[li];
    const uint32_t start = min(offsets[t], cap), end = min(offsets[t + 1], cap);
    const int n = (int)(end - start);
    uint64_t* keys = n <= kLongSmem ? sk : gkeys + start;
    GPS_DCHECK(start <= end, CHK_LIST);
    for (int e = threadIdx.x; e < n; e += blockDim.x) {
      const uint32_t idx = vals[start + e];
      GPS_DCHECK((int64_t)idx < hdr->n, CHK_GAUSS);
      keys[e] = ((uint64_t)__float_as_uint(rec[4 * idx + 1].z) << 32) | idx;
    }
    __syncthreads();
    bitonic_sort(keys, n);
    for (int e = threadIdx.x; e < n; e += blockDim.x) vals[start + e] = (uint32_t)keys[e];
    __syncthreads();
  }
}

// ============================================================================================
// k_sort_blend
// ============================================================================================
struct BlendIO {
  const float* sdf_depth;
  const float* sdf_color;
  const uint32_t* target;  // nullable (RGBA as u32)
  float* out_color;
  float* out_weight;
  float* loss_out;  // nullable
  int accumulate_loss;
  unsigned long long* counters;  // counting instantiation only: {evaluated, accepted} pairs
};

template <int TILE, bool SORTED>
__global__ void __launch_bounds__(TILE* TILE) k_sort_blend(RenderArgs a, const float4* __restrict__ rec,
                                                          const uint32_t* __restrict__ offsets, uint32_t* vals,
                                                          uint64_t* gkeys, uint32_t* tile_end, float* loss_part,
                                                          WsHeader* hdr, BlendIO io, int precull) {
  constexpr int NT = TILE * TILE;
  __shared__ __align__(16) uint64_t skeys[kShortList + 2];
  __shared__ float4 s0[NT], s1[NT], s2[NT];  // s0 = (px, py, a, 2b); s1 = (c, ln sigma, d, q_max)
  __shared__ float red[NT / 32 + 1];
  __shared__ uint32_t redi[NT / 32 + 1];
  const int t = blockIdx.x;
  const int tx = t % a.tiles_x, ty = t / a.tiles_x;
  const uint32_t start = min(offsets[t], a.cap);
  const uint32_t end = min(offsets[t + 1], a.cap);
  const int n = (int)(end - start);
  // ---- per-tile sort by (depth bits, index) (sort-free: the list stays in bucket order) ----
  if (!SORTED) {
  } else if (n <= NT) {
    // short list (the common case): rank sort -- each key's rank is the number of smaller keys
    // (keys are unique: the index is in the low word), two barriers instead of a bitonic network
    uint64_t key = ~0ull;
    if ((int)threadIdx.x < n) {
      const uint32_t idx = vals[start + threadIdx.x];
      key = ((uint64_t)__float_as_uint(rec[4 * idx + 1].z) << 32) | idx;
      skeys[threadIdx.x] = key;
    }
    if (threadIdx.x == 0) skeys[n] = ~0ull;  // pad slot of the paired loads below
    __syncthreads();
    int rank = 0;
    // broadcast reads, two keys per 16-byte load (slot n holds ~0: never smaller)
    const ulonglong2* k2 = reinterpret_cast<const ulonglong2*>(skeys);
    for (int j = 0; j < (n + 1) >> 1; ++j) {
      const ulonglong2 kk = k2[j];
      rank += (kk.x < key) + (kk.y < key);
    }
    __syncthreads();
    if ((int)threadIdx.x < n) {
      skeys[rank] = key;
      vals[start + rank] = (uint32_t)key;
    }
  } else if (n <= kShortList) {
    for (int e = threadIdx.x; e < n; e += NT) {
      const uint32_t idx = vals[start + e];
      const float d = rec[4 * idx + 1].z;
      skeys[e] = ((uint64_t)__float_as_uint(d) << 32) | idx;
    }
    __syncthreads();
    bitonic_sort(skeys, n);
    for (int e = threadIdx.x; e < n; e += NT) vals[start + e] = (uint32_t)skeys[e];
  }  // longer lists: sorted by k_sort_long
  __syncthreads();
  // ---- pixel state ----
  const int lx = threadIdx.x % TILE, ly = threadIdx.x / TILE;
  const int x = tx * TILE + lx, y = ty * TILE + ly;
  const bool inside = x < a.cam.W && y < a.cam.H;
  const size_t pix = inside ? (size_t)y * a.cam.W + x : 0;
  const float D = inside ? io.sdf_depth[pix] : 0.f;
  // the composite's inputs, loaded now so their latency hides behind the sort and the blend
  float ct0 = 0.f, ct1 = 0.f, ct2 = 0.f;
  uint32_t tgt8 = 0u;
  if (inside) {
    ct0 = io.sdf_color[3 * pix]; ct1 = io.sdf_color[3 * pix + 1]; ct2 = io.sdf_color[3 * pix + 2];
    if (io.target) tgt8 = io.target[pix];
  }
  const float lim = D > 0.f ? D + a.eps : INFINITY;  // R-MISS: no depth test on an SDF miss
  const float fx = (float)x, fy = (float)y;
  // optional pre-cull: entries at or behind every pixel's limit cannot contribute in this tile
  int n_eff = n;
  if (SORTED && precull) {
    float m = inside ? lim : -INFINITY;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xFFFFFFFFu, m, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
      float mm = red[0];
      for (int k = 1; k < NT / 32 + (NT % 32 ? 1 : 0); ++k) mm = fmaxf(mm, red[k]);
      red[NT / 32] = mm;
    }
    __syncthreads();
    const float tmax = red[NT / 32];
    if (tmax < INFINITY) {  // binary search: first entry with d >= tmax
      int lo = 0, hi = n;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        const float d = n <= kShortList ? __uint_as_float((uint32_t)(skeys[mid] >> 32)) : rec[4 * vals[start + mid] + 1].z;
        if (d >= tmax) hi = mid; else lo = mid + 1;
      }
      n_eff = lo;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) tile_end[t] = start + n_eff;
  // ---- front-to-back blend, Eqs. 1-3, early termination at the SDF depth ----
  // Each warp compacts the staged batch 32 entries at a time: lane j tests entry j against the
  // warp's rows and the warp's deepest pixel limit, a ballot keeps the survivors, and the warp
  // walks only those in list order.  Every pixel still sees exactly the entries it saw before,
  // in the same order, so W and C are bitwise unchanged.
  constexpr int kWarpRows = 32 / TILE;  // pixel rows covered by one warp
  const int lane = threadIdx.x & 31;
  const int wy0 = ty * TILE + (threadIdx.x >> 5) * kWarpRows, wy1 = wy0 + kWarpRows - 1;
  float wlim = inside ? lim : -INFINITY;  // the warp's largest limit: entries at or behind it
#pragma unroll                            // contribute to none of its pixels (lists are sorted)
  for (int o = 16; o > 0; o >>= 1) wlim = fmaxf(wlim, __shfl_xor_sync(0xFFFFFFFFu, wlim, o));
  float W = 0.f, C0 = 0.f, C1 = 0.f, C2 = 0.f;
  bool wdone = !(wlim > -INFINITY);  // warp-uniform
  for (int base = 0; base < n_eff; base += NT) {
    const int cnt = min(NT, n_eff - base);
    __syncthreads();
    if (threadIdx.x < cnt) {
      const uint32_t idx = vals[start + base + threadIdx.x];
      const float4 r0 = rec[4 * idx], r1 = rec[4 * idx + 1];
      s0[threadIdx.x] = make_float4(r0.x, r0.y, r0.z, pmul(2.0f, r0.w));
      s1[threadIdx.x] = make_float4(r1.x, r1.y, r1.z, pair_qmax(a.ln_inv_amin, r1.y));
      s2[threadIdx.x] = rec[4 * idx + 2];
    }
    __syncthreads();
    for (int kb = 0; kb < cnt && !wdone; kb += 32) {
      const int k = kb + lane;
      bool live = false, stop = false;
      if (k < cnt) {
        // sorted: the first entry at or behind the warp's deepest limit ends the warp's list;
        // sort-free: such an entry is only skipped
        const bool behind = !(s1[k].z < wlim);
        stop = SORTED && behind;
        const uint32_t ry = __float_as_uint(s2[k].w);
        live = !behind && (int)(ry >> 16) >= wy0 && (int)(ry & 0xFFFFu) <= wy1;
        if (live) {  // the ellipse itself must meet the warp's pixel strip
          const float4 e0 = s0[k];
          live = ellipse_meets_strip(e0.x, e0.y, e0.z, e0.w, s1[k].x, s1[k].w, tx * TILE, tx * TILE + TILE - 1,
                                     wy0, wy1);
        }
      }
      uint32_t lm = __ballot_sync(0xFFFFFFFFu, live);
      const uint32_t sm = __ballot_sync(0xFFFFFFFFu, stop);
      if (sm) {
        lm &= (1u << (__ffs(sm) - 1)) - 1u;  // survivors before the first stop
        wdone = true;
      }
      while (lm) {
        const int kk = kb + __ffs(lm) - 1;
        lm &= lm - 1u;
        const float4 r1 = s1[kk];
        if (!(r1.z < lim)) continue;  // Eq. 1's indicator for this pixel
        const float4 r0 = s0[kk];
        const float q = pair_q(r0.x, r0.y, r0.z, r0.w, r1.x, fx, fy);
        if (!(q <= r1.w)) continue;  // outside the 3-sigma ellipse or alpha < alpha_min
        const float al = __expf(fmaf(-0.5f, q, r1.y));  // sigma exp(-q/2), Eq. 3
        const float4 r2 = s2[kk];
        W += al;
        C0 = fmaf(al, r2.x, C0);
        C1 = fmaf(al, r2.y, C1);
        C2 = fmaf(al, r2.z, C2);
      }
    }
    if (__syncthreads_count(!wdone) == 0) break;
  }
  // ---- Eq. 4 composite with W_t = 1, fused L1 ----
  float l1 = 0.f;
  uint32_t inmask = 0;
  if (inside) {
    const float inv = 1.0f / (1.0f + W);
    const float o0 = (ct0 + C0) * inv, o1 = (ct1 + C1) * inv, o2 = (ct2 + C2) * inv;
    io.out_color[3 * pix] = W > 0.f ? o0 : ct0;
    io.out_color[3 * pix + 1] = W > 0.f ? o1 : ct1;
    io.out_color[3 * pix + 2] = W > 0.f ? o2 : ct2;
    io.out_weight[pix] = W;
    if (io.target && (D > 0.f || W > 0.f)) {
      const uint32_t c = tgt8;
      const float k0 = (float)(c & 0xFFu) * (1.f / 255.f), k1 = (float)((c >> 8) & 0xFFu) * (1.f / 255.f),
                  k2 = (float)((c >> 16) & 0xFFu) * (1.f / 255.f);
      const float r0 = W > 0.f ? o0 : ct0, r1 = W > 0.f ? o1 : ct1, r2 = W > 0.f ? o2 : ct2;
      l1 = fabsf(r0 - k0) + fabsf(r1 - k1) + fabsf(r2 - k2);
      inmask = 1;
    }
  }
  if (!io.target) return;
  // deterministic CTA reduction (fixed shuffle tree + fixed smem order)
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    l1 += __shfl_xor_sync(0xFFFFFFFFu, l1, o);
    inmask += __shfl_xor_sync(0xFFFFFFFFu, inmask, o);
  }
  __syncthreads();
  if ((threadIdx.x & 31) == 0) {
    red[threadIdx.x >> 5] = l1;
    redi[threadIdx.x >> 5] = inmask;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    float s = 0.f;
    uint32_t m = 0;
    for (int k = 0; k < (NT + 31) / 32; ++k) {
      s += red[k];
      m += redi[k];
    }
    loss_part[t] = s;
    if (m) atomicAdd(&hdr->mask_count, m);
    __threadfence();
    const uint32_t ticket = atomicAdd(&hdr->ticket, 1u);
    redi[0] = ticket == (uint32_t)(gridDim.x - 1) ? 1u : 0u;
  }
  __syncthreads();
  if (redi[0] == 0u) return;
  // last CTA: sum the tile partials in tile order (fixed tree) -> mean L1 (R-L1)
  __threadfence();
  float s = 0.f;
  for (int k = threadIdx.x; k < (int)gridDim.x; k += NT) s += *(volatile float*)&loss_part[k];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xFFFFFFFFu, s, o);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    float tot = 0.f;
    for (int k = 0; k < (NT + 31) / 32; ++k) tot += red[k];
    const uint32_t m = *(volatile uint32_t*)&hdr->mask_count;
    const float lv = m ? tot / (3.0f * (float)m) : 0.0f;
    if (io.loss_out) *io.loss_out = io.accumulate_loss ? *io.loss_out + lv : lv;
    hdr->ticket = 0u;
  }
}

// --------------------------------------------------------------------------------------------
// k_sort_blend16x2: the same blend for 16x16 tiles with TWO pixels per thread (128 threads).
// Warp w covers rows 4w..4w+3 of the tile; lane l holds pixels (l & 15, 4w + (l >> 4)) and the
// one two rows below.  Against k_sort_blend<16> each (warp, entry) pair now serves 64 pixels:
// an entry of the median 7-row footprint meets ~2.75 warp strips instead of ~4.5, and the
// per-entry work of the walk (record loads, compaction) is shared by two pixels.  The sort keeps
// only 256 + 2 keys in shared memory (longer lists -- none above 252 at cfg4 -- use the global
// bitonic fallback), so more CTAs stay resident.  Every pixel sees the same entries in the same
// order as in k_sort_blend, so C* and W_G are bitwise those of the one-pixel-per-thread kernel.
// --------------------------------------------------------------------------------------------
// Long lists (more than NB entries; sorted by k_sort_long) are split into work items of NB
// entries: CTA t takes (tile t, chunk 0), then the further chunks k_scan listed (extra[e] for
// e = t, t + grid, ...).  Each chunk accumulates its entries' W and C per pixel and stores them
// in its partial slot; the tile's last chunk to finish (a per-tile ticket) sums the partials in
// chunk order -- a fixed order, so the image stays bit-reproducible -- and composites.  (One
// 128-thread CTA walking a 6000-entry list was the kernel's tail in late cfg4 frames.)
struct SplitIO {
  const uint2* extra;     // {tile, chunk >= 1} work items of long lists (k_scan)
  uint32_t extra_cap;
  const uint32_t* pbase;  // per long tile: its first partial slot, ~0 = not split (no room)
  uint32_t* tick;         // per tile: chunks finished (zeroed per render)
  float4* part;           // partial slots, 256 pixels each: (W, C0, C1, C2)
};

template <bool SORTED, bool COUNT = false, bool WW = true>
__global__ void __launch_bounds__(128, 8) k_sort_blend16x2(RenderArgs a, const float4* __restrict__ rec,
                                                        const uint32_t* __restrict__ offsets, uint32_t* vals,
                                                        uint64_t* gkeys, uint32_t* tile_end, float* loss_part,
                                                        WsHeader* hdr, BlendIO io, int precull, SplitIO spl) {
  constexpr int NT = 128, NB = 256;  // threads, staged entries per batch (2 per thread)
  __shared__ __align__(16) uint64_t skeys[NB + 2];
  __shared__ __align__(16) uint32_t sdep[NB + 4];
  __shared__ float4 s0[WW ? 1 : NB], s1[WW ? 1 : NB], s2[WW ? 1 : NB];  // s0 = (px, py, a, 2b); s1 = (c, ln sigma, d, q_max)
  __shared__ float4 ws0[WW ? 4 : 1][32], ws1[WW ? 4 : 1][32], ws2[WW ? 4 : 1][32];  // per-warp chunk (WW)
  __shared__ float red[NT / 32 + 1];
  __shared__ uint32_t redi[NT / 32 + 1];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint32_t n_extra = (SORTED && spl.extra) ? min(hdr->n_extra, spl.extra_cap) : 0u;
  for (uint32_t item = blockIdx.x; item < gridDim.x + n_extra; item += gridDim.x) {
  int t;
  uint32_t chunk;
  if (item < gridDim.x) {
    t = (int)item;
    chunk = 0;
  } else {
    const uint2 wi = spl.extra[item - gridDim.x];
    t = (int)wi.x;
    chunk = wi.y;
  }
  const int tx = t % a.tiles_x, ty = t / a.tiles_x;
  const uint32_t start = min(offsets[t], a.cap);
  const uint32_t end = min(offsets[t + 1], a.cap);
  const int n = (int)(end - start);
  const bool small = n <= NB;  // keys live in shared memory
  const int nch = (SORTED && spl.extra && !small) ? (n + NB - 1) / NB : 1;
  const bool split = nch > 1 && spl.pbase[t] != ~0u;
  if (!split && chunk > 0) continue;  // a long list that could not be split: chunk 0 walks it all
  __syncthreads();  // shared memory of the previous item is free
  // ---- per-tile sort by (depth bits, index) (lists longer than NB: sorted by k_sort_long) ----
  if (!SORTED) {
  } else if (small) {
    // rank sort, two keys per thread.  The rank is first counted on the 32-bit depth bits alone
    // (four per 16-byte shared load); it equals the (depth bits, index) rank unless two entries
    // share a depth, which shows as a slot left unwritten by the scatter -- then the tile is
    // re-ranked on the full 64-bit keys.
    uint64_t key[2] = {~0ull, ~0ull};
    uint32_t dk[2] = {~0u, ~0u};
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int e = threadIdx.x + h * NT;
      if (e < n) {
        const uint32_t idx = vals[start + e];
        GPS_DCHECK((int64_t)idx < a.n, CHK_GAUSS);
        dk[h] = __float_as_uint(rec[4 * idx + 1].z);
        key[h] = ((uint64_t)dk[h] << 32) | idx;
        sdep[e] = dk[h];
      }
    }
    if (threadIdx.x < 4) sdep[n + threadIdx.x] = ~0u;  // pad of the 4-wide loads (never < a depth)
    __syncthreads();
    int rank[2] = {0, 0};
    {
      const uint4* d4 = reinterpret_cast<const uint4*>(sdep);
      for (int j = 0; j < (n + 3) >> 2; ++j) {
        const uint4 q = d4[j];
        rank[0] += (q.x < dk[0]) + (q.y < dk[0]) + (q.z < dk[0]) + (q.w < dk[0]);
        rank[1] += (q.x < dk[1]) + (q.y < dk[1]) + (q.z < dk[1]) + (q.w < dk[1]);
      }
    }
#pragma unroll
    for (int h = 0; h < 2; ++h)
      if (threadIdx.x + h * NT < n) skeys[threadIdx.x + h * NT] = ~0ull;  // "unwritten"
    __syncthreads();
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      GPS_DCHECK(threadIdx.x + h * NT >= n || rank[h] < n, CHK_SMEM);
      if (threadIdx.x + h * NT < n) skeys[rank[h]] = key[h];
    }
    __syncthreads();
    bool hole = false;
#pragma unroll
    for (int h = 0; h < 2; ++h)
      if (threadIdx.x + h * NT < n) hole |= skeys[threadIdx.x + h * NT] == ~0ull;
    if (__syncthreads_or(hole)) {  // equal depths: rank on the full keys
#pragma unroll
      for (int h = 0; h < 2; ++h)
        if (threadIdx.x + h * NT < n) skeys[threadIdx.x + h * NT] = key[h];
      if (threadIdx.x == 0) skeys[n] = ~0ull;  // pad slot of the paired loads below
      __syncthreads();
      rank[0] = rank[1] = 0;
      const ulonglong2* k2 = reinterpret_cast<const ulonglong2*>(skeys);
      for (int j = 0; j < (n + 1) >> 1; ++j) {
        const ulonglong2 kk = k2[j];
        rank[0] += (kk.x < key[0]) + (kk.y < key[0]);
        rank[1] += (kk.x < key[1]) + (kk.y < key[1]);
      }
      __syncthreads();
#pragma unroll
      for (int h = 0; h < 2; ++h)
        if (threadIdx.x + h * NT < n) skeys[rank[h]] = key[h];
    }
#pragma unroll
    for (int h = 0; h < 2; ++h)
      if (threadIdx.x + h * NT < n) vals[start + rank[h]] = (uint32_t)key[h];
  }
  __syncthreads();
  // ---- pixel state (two pixels) ----
  const int lx = lane & 15, ly0 = 4 * w + (lane >> 4);
  const int x = tx * 16 + lx;
  float D[2], lim[2], ct[2][3];
  uint32_t tgt8[2];
  bool inside[2];
  size_t pix[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int y = ty * 16 + ly0 + 2 * h;
    inside[h] = x < a.cam.W && y < a.cam.H;
    pix[h] = inside[h] ? (size_t)y * a.cam.W + x : 0;
    D[h] = inside[h] ? io.sdf_depth[pix[h]] : 0.f;
    ct[h][0] = ct[h][1] = ct[h][2] = 0.f;
    tgt8[h] = 0u;
    if (inside[h]) {
      ct[h][0] = io.sdf_color[3 * pix[h]]; ct[h][1] = io.sdf_color[3 * pix[h] + 1];
      ct[h][2] = io.sdf_color[3 * pix[h] + 2];
      if (io.target) tgt8[h] = io.target[pix[h]];
    }
    lim[h] = D[h] > 0.f ? D[h] + a.eps : INFINITY;  // R-MISS: no depth test on an SDF miss
  }
  const float fx = (float)x, fy0 = (float)(ty * 16 + ly0), fy1 = fy0 + 2.0f;
  float wl = fmaxf(inside[0] ? lim[0] : -INFINITY, inside[1] ? lim[1] : -INFINITY);
  int n_eff = n;
  if (SORTED && precull) {
    float m = wl;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xFFFFFFFFu, m, o));
    if (lane == 0) red[w] = m;
    __syncthreads();
    if (threadIdx.x == 0) red[NT / 32] = fmaxf(fmaxf(red[0], red[1]), fmaxf(red[2], red[3]));
    __syncthreads();
    const float tmax = red[NT / 32];
    if (tmax < INFINITY) {  // binary search: first entry with d >= tmax
      int lo = 0, hi = n;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        const float d = small ? __uint_as_float((uint32_t)(skeys[mid] >> 32)) : rec[4 * vals[start + mid] + 1].z;
        if (d >= tmax) hi = mid; else lo = mid + 1;
      }
      n_eff = lo;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0 && chunk == 0) tile_end[t] = start + n_eff;
  // ---- blend (per-warp compaction over the warp's 4-row strip, as k_sort_blend) ----
  const int b_lo = split ? NB * (int)chunk : 0, b_hi = split ? min(b_lo + NB, n_eff) : n_eff;
  const int wy0 = ty * 16 + 4 * w, wy1 = wy0 + 3;
  float wlim = wl;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) wlim = fmaxf(wlim, __shfl_xor_sync(0xFFFFFFFFu, wlim, o));
  float W0 = 0.f, A0 = 0.f, B0 = 0.f, G0 = 0.f, W1 = 0.f, A1 = 0.f, B1 = 0.f, G1 = 0.f;
  uint32_t n_eval = 0, n_acc = 0;  // COUNT: pixel-entry pairs whose q was evaluated / accepted
  bool wdone = !(wlim > -INFINITY);  // warp-uniform
  if (WW) {
    // Warp walk: each warp stages its own 32-entry chunks (a lane per entry, from the sorted
    // keys in shared memory or the list) into a per-warp buffer and walks them without any CTA
    // barrier -- the four warps of a tile no longer wait for each other at every 256-entry
    // batch.  Per live entry the two pixels (rows y, y + 2) are evaluated together in packed
    // f32x2 arithmetic (FFMA2/FMUL2/FADD2: per component the same rounding as the scalar
    // sequence, so the image is bitwise unchanged) and accumulated branch-free (a rejected
    // pixel adds alpha = 0, which leaves every sum bitwise unchanged).
    float4* const e0s = ws0[WW ? w : 0];
    float4* const e1s = ws1[WW ? w : 0];
    float4* const e2s = ws2[WW ? w : 0];
    float2 Wv = make_float2(0.f, 0.f), Av = Wv, Bv = Wv, Gv = Wv;
    const float2 fyv = make_float2(fy0, fy1), limv = make_float2(lim[0], lim[1]);
    for (int kb = b_lo; kb < b_hi && !wdone; kb += 32) {
      const int k = kb + lane;
      bool live = false, stop = false;
      if (k < b_hi) {
        const uint32_t idx = (SORTED && small) ? (uint32_t)skeys[k] : vals[start + k];
        GPS_DCHECK((int64_t)idx < a.n && start + k < end, CHK_GAUSS);
        const float4 r0 = rec[4 * idx], r1 = rec[4 * idx + 1], r2 = rec[4 * idx + 2];
        const float4 e0 = make_float4(r0.x, r0.y, r0.z, pmul(2.0f, r0.w));
        const float4 e1 = make_float4(r1.x, r1.y, r1.z, pair_qmax(a.ln_inv_amin, r1.y));
        e0s[lane] = e0;
        e1s[lane] = e1;
        e2s[lane] = r2;
        const bool behind = !(e1.z < wlim);
        stop = SORTED && behind;
        const uint32_t ry = __float_as_uint(r2.w);
        live = !behind && (int)(ry >> 16) >= wy0 && (int)(ry & 0xFFFFu) <= wy1;
        if (live) live = ellipse_meets_strip(e0.x, e0.y, e0.z, e0.w, e1.x, e1.w, tx * 16, tx * 16 + 15, wy0, wy1);
      }
      uint32_t lm = __ballot_sync(0xFFFFFFFFu, live);
      const uint32_t sm = __ballot_sync(0xFFFFFFFFu, stop);
      if (sm) {
        lm &= (1u << (__ffs(sm) - 1)) - 1u;  // survivors before the first stop
        wdone = true;
      }
      __syncwarp();
      while (lm) {
        const int kk = __ffs(lm) - 1;
        lm &= lm - 1u;
        const float4 r1 = e1s[kk];
        const bool i0 = r1.z < limv.x, i1 = r1.z < limv.y;  // Eq. 1's indicator per pixel
        if (!(i0 | i1)) continue;
        const float4 r0 = e0s[kk];
        // pair_q at (x, y) and (x, y + 2): dx and its products are shared
        const float dx = fx - r0.x;
        const float bdx = pmul(r0.w, dx), adx = pmul(r0.z, dx);
        const float2 dy = __fadd2_rn(fyv, make_float2(-r0.y, -r0.y));
        const float2 cdy2 = __fmul2_rn(__fmul2_rn(make_float2(r1.x, r1.x), dy), dy);
        const float2 q = __ffma2_rn(make_float2(adx, adx), make_float2(dx, dx),
                                    __ffma2_rn(make_float2(bdx, bdx), dy, cdy2));
        const bool p0 = i0 && q.x <= r1.w, p1 = i1 && q.y <= r1.w;
        if (COUNT) {
          n_eval += (uint32_t)(i0 && inside[0]) + (uint32_t)(i1 && inside[1]);
          n_acc += (uint32_t)(p0 && inside[0]) + (uint32_t)(p1 && inside[1]);
        }
        if (!(p0 | p1)) continue;
        const float4 r2 = e2s[kk];
        const float2 arg = __ffma2_rn(make_float2(-0.5f, -0.5f), q, make_float2(r1.y, r1.y));
        const float2 al = make_float2(p0 ? __expf(arg.x) : 0.f, p1 ? __expf(arg.y) : 0.f);  // Eq. 3
        Wv = __fadd2_rn(Wv, al);
        Av = __ffma2_rn(al, make_float2(r2.x, r2.x), Av);
        Bv = __ffma2_rn(al, make_float2(r2.y, r2.y), Bv);
        Gv = __ffma2_rn(al, make_float2(r2.z, r2.z), Gv);
      }
      __syncwarp();
    }
    W0 = Wv.x; W1 = Wv.y; A0 = Av.x; A1 = Av.y; B0 = Bv.x; B1 = Bv.y; G0 = Gv.x; G1 = Gv.y;
  }
  for (int base = b_lo; !WW && base < b_hi; base += NB) {
    const int cnt = min(NB, b_hi - base);
    __syncthreads();
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int e = threadIdx.x + h * NT;
      if (e < cnt) {
        const uint32_t idx = vals[start + base + e];
        GPS_DCHECK((int64_t)idx < a.n && start + base + e < end, CHK_GAUSS);
        const float4 r0 = rec[4 * idx], r1 = rec[4 * idx + 1];
        s0[e] = make_float4(r0.x, r0.y, r0.z, pmul(2.0f, r0.w));
        s1[e] = make_float4(r1.x, r1.y, r1.z, pair_qmax(a.ln_inv_amin, r1.y));
        s2[e] = rec[4 * idx + 2];
      }
    }
    __syncthreads();
    for (int kb = 0; kb < cnt && !wdone; kb += 32) {
      const int k = kb + lane;
      bool live = false, stop = false;
      if (k < cnt) {
        const bool behind = !(s1[k].z < wlim);
        stop = SORTED && behind;
        const uint32_t ry = __float_as_uint(s2[k].w);
        live = !behind && (int)(ry >> 16) >= wy0 && (int)(ry & 0xFFFFu) <= wy1;
        if (live) {
          const float4 e0 = s0[k];
          live = ellipse_meets_strip(e0.x, e0.y, e0.z, e0.w, s1[k].x, s1[k].w, tx * 16, tx * 16 + 15, wy0, wy1);
        }
      }
      uint32_t lm = __ballot_sync(0xFFFFFFFFu, live);
      const uint32_t sm = __ballot_sync(0xFFFFFFFFu, stop);
      if (sm) {
        lm &= (1u << (__ffs(sm) - 1)) - 1u;  // survivors before the first stop
        wdone = true;
      }
      while (lm) {
        const int kk = kb + __ffs(lm) - 1;
        lm &= lm - 1u;
        const float4 r1 = s1[kk];
        const bool i0 = r1.z < lim[0], i1 = r1.z < lim[1];  // Eq. 1's indicator per pixel
        if (!(i0 | i1)) continue;
        const float4 r0 = s0[kk];
        const float q0 = pair_q(r0.x, r0.y, r0.z, r0.w, r1.x, fx, fy0);
        const float q1 = pair_q(r0.x, r0.y, r0.z, r0.w, r1.x, fx, fy1);
        const bool p0 = i0 && q0 <= r1.w, p1 = i1 && q1 <= r1.w;
        if (COUNT) {
          n_eval += (uint32_t)(i0 && inside[0]) + (uint32_t)(i1 && inside[1]);
          n_acc += (uint32_t)(p0 && inside[0]) + (uint32_t)(p1 && inside[1]);
        }
        if (!(p0 | p1)) continue;
        const float4 r2 = s2[kk];
        if (p0) {
          const float al = __expf(fmaf(-0.5f, q0, r1.y));  // sigma exp(-q/2), Eq. 3
          W0 += al;
          A0 = fmaf(al, r2.x, A0); B0 = fmaf(al, r2.y, B0); G0 = fmaf(al, r2.z, G0);
        }
        if (p1) {
          const float al = __expf(fmaf(-0.5f, q1, r1.y));
          W1 += al;
          A1 = fmaf(al, r2.x, A1); B1 = fmaf(al, r2.y, B1); G1 = fmaf(al, r2.z, G1);
        }
      }
    }
    if (__syncthreads_count(!wdone) == 0) break;
  }
  if (COUNT) {
    const unsigned long long e = __reduce_add_sync(0xFFFFFFFFu, n_eval), c = __reduce_add_sync(0xFFFFFFFFu, n_acc);
    if (lane == 0) {
      atomicAdd(io.counters, e);
      atomicAdd(io.counters + 1, c);
    }
  }
  if (split) {
    // this chunk's partial sums into its slot; the tile's last chunk combines them in order
    const uint32_t slot = spl.pbase[t] + chunk;
    GPS_DCHECK(chunk < (uint32_t)nch && slot < hdr->n_part, CHK_SPLIT);
    const int p0i = ly0 * 16 + lx, p1i = (ly0 + 2) * 16 + lx;
    spl.part[256 * (size_t)slot + p0i] = make_float4(W0, A0, B0, G0);
    spl.part[256 * (size_t)slot + p1i] = make_float4(W1, A1, B1, G1);
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) redi[0] = atomicAdd(&spl.tick[t], 1u) == (uint32_t)(nch - 1) ? 1u : 0u;
    __syncthreads();
    if (redi[0] == 0u) continue;  // another chunk of this tile finishes it
    __threadfence();
    W0 = A0 = B0 = G0 = W1 = A1 = B1 = G1 = 0.f;
    const uint32_t b0s = spl.pbase[t];
    for (int c = 0; c < nch; ++c) {
      const float4 q0 = __ldcg(&spl.part[256 * (size_t)(b0s + c) + p0i]);
      const float4 q1 = __ldcg(&spl.part[256 * (size_t)(b0s + c) + p1i]);
      W0 += q0.x; A0 += q0.y; B0 += q0.z; G0 += q0.w;
      W1 += q1.x; A1 += q1.y; B1 += q1.z; G1 += q1.w;
    }
  }
  // ---- Eq. 4 composite with W_t = 1, fused L1 ----
  float l1 = 0.f;
  uint32_t inmask = 0;
  const float Ws[2] = {W0, W1}, Cs[2][3] = {{A0, B0, G0}, {A1, B1, G1}};
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    if (!inside[h]) continue;
    const float W = Ws[h];
    const float inv = 1.0f / (1.0f + W);
    const float o0 = (ct[h][0] + Cs[h][0]) * inv, o1 = (ct[h][1] + Cs[h][1]) * inv, o2 = (ct[h][2] + Cs[h][2]) * inv;
    const float r0 = W > 0.f ? o0 : ct[h][0], r1 = W > 0.f ? o1 : ct[h][1], r2 = W > 0.f ? o2 : ct[h][2];
    io.out_color[3 * pix[h]] = r0;
    io.out_color[3 * pix[h] + 1] = r1;
    io.out_color[3 * pix[h] + 2] = r2;
    io.out_weight[pix[h]] = W;
    if (io.target && (D[h] > 0.f || W > 0.f)) {
      const uint32_t c = tgt8[h];
      const float k0 = (float)(c & 0xFFu) * (1.f / 255.f), k1 = (float)((c >> 8) & 0xFFu) * (1.f / 255.f),
                  k2 = (float)((c >> 16) & 0xFFu) * (1.f / 255.f);
      l1 += fabsf(r0 - k0) + fabsf(r1 - k1) + fabsf(r2 - k2);
      inmask += 1;
    }
  }
  if (!io.target) continue;
  // deterministic CTA reduction (fixed shuffle tree + fixed smem order)
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    l1 += __shfl_xor_sync(0xFFFFFFFFu, l1, o);
    inmask += __shfl_xor_sync(0xFFFFFFFFu, inmask, o);
  }
  __syncthreads();
  if (lane == 0) {
    red[w] = l1;
    redi[w] = inmask;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    float sum = 0.f;
    uint32_t m = 0;
    for (int k = 0; k < NT / 32; ++k) {
      sum += red[k];
      m += redi[k];
    }
    loss_part[t] = sum;
    if (m) atomicAdd(&hdr->mask_count, m);
    __threadfence();
    const uint32_t ticket = atomicAdd(&hdr->ticket, 1u);  // one per finished tile
    redi[0] = ticket == (uint32_t)(gridDim.x - 1) ? 1u : 0u;
  }
  __syncthreads();
  if (redi[0] == 0u) continue;
  // last tile: sum the tile partials in tile order (fixed tree) -> mean L1 (R-L1)
  __threadfence();
  float sum = 0.f;
  for (int k = threadIdx.x; k < (int)gridDim.x; k += NT) sum += *(volatile float*)&loss_part[k];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xFFFFFFFFu, sum, o);
  __syncthreads();
  if (lane == 0) red[w] = sum;
  __syncthreads();
  if (threadIdx.x == 0) {
    float tot = 0.f;
    for (int k = 0; k < NT / 32; ++k) tot += red[k];
    const uint32_t m = *(volatile uint32_t*)&hdr->mask_count;
    const float lv = m ? tot / (3.0f * (float)m) : 0.0f;
    if (io.loss_out) *io.loss_out = io.accumulate_loss ? *io.loss_out + lv : lv;
    hdr->ticket = 0u;
  }
  }  // work items
}

// ============================================================================================
// k_backward: exact gradient of the L1 loss w.r.t. each listed Gaussian's 2D quantities
// (p_hat, conic, sigma, colour), R-GRAD.  Order of entries is irrelevant (no transmittance);
// each tile list is walked back to front.
// ============================================================================================
__device__ __forceinline__ void red_add_v4(float4* addr, float a, float b, float c, float d) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(addr), "f"(a), "f"(b), "f"(c), "f"(d)
               : "memory");
}

// one reduce-scatter level: lanes with `mask` set keep the upper half of their NIN values and
// send the lower half to the partner, which keeps the lower half (padding counts as zero)
template <int NIN, int NKEEP>
__device__ __forceinline__ void rs_level(const float* x, float* y, int lane, int mask) {
  const bool up = lane & mask;
#pragma unroll
  for (int k = 0; k < NKEEP; ++k) {
    const float hi = (NKEEP + k < NIN) ? x[NKEEP + k] : 0.f;
    const float lo = x[k];
    y[k] = (up ? hi : lo) + __shfl_xor_sync(0xFFFFFFFFu, up ? lo : hi, mask);
  }
}

// Per-pixel state of the backward for tile t (R-GRAD, Eq. 7 P:140 with Eq. 4): for a
// pixel of the loss mask, (g0, g1, g2) = A dL/dC*_ch with A = 1 / (1 + W_G) and s = sum_ch g_ch C*_ch
// (so dL/dalpha_i = sum_ch g_ch c_i,ch - s), and lim = D_t + eps (inf on an SDF miss); -inf for
// pixels outside the image or the mask (no pair passes).
template <int TILE>
__device__ __forceinline__ uint32_t backward_pixel_state(const RenderArgs& a, int t, const float* __restrict__ sdf_depth,
                                                         const float* __restrict__ cstar, const float* __restrict__ wg,
                                                         const uint32_t* __restrict__ target, const WsHeader* hdr,
                                                         float4* sgs, float* slim) {
  constexpr int NP = TILE * TILE;
  const int tx = t % a.tiles_x, ty = t / a.tiles_x;
  const uint32_t m = hdr->mask_count;
  const float inv3m = m ? 1.0f / (3.0f * (float)m) : 0.0f;
  for (int p = threadIdx.x; p < NP; p += blockDim.x) {
    const int x = tx * TILE + p % TILE, y = ty * TILE + p / TILE;
    float g0 = 0.f, g1 = 0.f, g2 = 0.f, s = 0.f, lim = -INFINITY;  // -inf: no pair passes
    if (x < a.cam.W && y < a.cam.H && m) {
      const size_t pix = (size_t)y * a.cam.W + x;
      const float D = sdf_depth[pix], Wp = wg[pix];
      if (D > 0.f || Wp > 0.f) {
        const float A = 1.0f / (1.0f + Wp);
        const uint32_t c = target[pix];
        const float c0 = cstar[3 * pix], c1 = cstar[3 * pix + 1], c2 = cstar[3 * pix + 2];
        const float d0 = c0 - (float)(c & 0xFFu) * (1.f / 255.f);
        const float d1 = c1 - (float)((c >> 8) & 0xFFu) * (1.f / 255.f);
        const float d2 = c2 - (float)((c >> 16) & 0xFFu) * (1.f / 255.f);
        // dL/dC* = sign(C* - C_k) / (3|M|), sign(0) = 0
        g0 = (d0 > 0.f ? inv3m : (d0 < 0.f ? -inv3m : 0.f)) * A;
        g1 = (d1 > 0.f ? inv3m : (d1 < 0.f ? -inv3m : 0.f)) * A;
        g2 = (d2 > 0.f ? inv3m : (d2 < 0.f ? -inv3m : 0.f)) * A;
        s = g0 * c0 + g1 * c1 + g2 * c2;  // A * sum_ch g_ch C*_ch
        lim = D > 0.f ? D + a.eps : INFINITY;
      }
    }
    sgs[p] = make_float4(g0, g1, g2, s);
    slim[p] = lim;
  }
  return m;
}

template <int TILE>
__global__ void __launch_bounds__(256) k_backward(RenderArgs a, const float4* __restrict__ rec,
                                                  const uint32_t* __restrict__ offsets,
                                                  const uint32_t* __restrict__ vals,
                                                  const uint32_t* __restrict__ tile_end,
                                                  const float* __restrict__ sdf_depth,
                                                  const float* __restrict__ cstar, const float* __restrict__ wg,
                                                  const uint32_t* __restrict__ target, const WsHeader* hdr,
                                                  float* grad2d, const uint2* __restrict__ extra, uint32_t extra_cap) {
  constexpr int NP = TILE * TILE;
  __shared__ float4 sgs[NP];  // per pixel (g0, g1, g2, s): A * dL/dC*_ch and A * sum_ch g_ch C*_ch
  __shared__ float slim[NP];
  __shared__ uint32_t smagic[TILE + 1];  // ceil(65536 / w), w = 1..TILE
  if (threadIdx.x <= TILE) smagic[threadIdx.x] = threadIdx.x ? (65536u + threadIdx.x - 1u) / threadIdx.x : 0u;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  // the lane that ends up holding each reduced value (reduce-scatter below), and which value
  int vidx;  // within the lane's half-warp (levels xor 8, 4, 2, 1 below)
  {
    const int b3 = (lane >> 3) & 1, b2 = (lane >> 2) & 1, b1 = (lane >> 1) & 1, b0 = lane & 1;
    const int kc = b0;
    const int kb = b1 ? (2 + kc < 3 ? 2 + kc : -1) : kc;
    const int ka = kb < 0 ? -1 : (b2 ? (3 + kb < 5 ? 3 + kb : -1) : kb);
    vidx = ka < 0 ? -1 : (b3 ? (ka < 4 ? 5 + ka : -1) : ka);
  }
  __shared__ float4 se0[256], se1[256], se2[256], se3[256];
  __shared__ uint32_t sidx[256];
  // Work items of 256 list entries: CTA b takes (tile b, entries 0-255), then the further chunks
  // of long lists that k_scan listed, extra[e] for e = b, b + grid, ... (the pixel state is
  // loaded once per item; in the common case every tile is one item).
  const uint32_t n_extra = min(hdr->n_extra, extra_cap);
  int cur_tile = -1;
  uint32_t m = 0;
  for (uint32_t item = blockIdx.x; item < gridDim.x + n_extra; item += gridDim.x) {
    int t;
    uint32_t chunk;
    if (item < gridDim.x) {
      t = (int)item;
      chunk = 0;
    } else {
      const uint2 w = extra[item - gridDim.x];
      t = (int)w.x;
      chunk = w.y;
    }
    const int tx = t % a.tiles_x, ty = t / a.tiles_x;
    if (t != cur_tile) {
      __syncthreads();  // the previous item's readers of the pixel state are done
      m = backward_pixel_state<TILE>(a, t, sdf_depth, cstar, wg, target, hdr, sgs, slim);
      cur_tile = t;
    }
    if (!m) return;  // empty loss mask: no gradient anywhere (uniform)
    const uint32_t start = min(offsets[t], a.cap);
    const uint32_t end = min(tile_end[t], a.cap);
    const int tx0 = tx * TILE, ty0 = ty * TILE;
    const uint32_t base = start + 256u * chunk;
    const int cnt_e = base < end ? (int)min(256u, end - base) : 0;
    __syncthreads();  // pixel state visible; the previous batch's readers are done
    GPS_DCHECK(cnt_e <= 256 && t < a.tiles_x * a.tiles_y, CHK_SMEM);
    for (int j = threadIdx.x; j < cnt_e; j += blockDim.x) {
      const uint32_t id = vals[base + j];
      GPS_DCHECK((int64_t)id < a.n, CHK_GAUSS);
      sidx[j] = id;
      const float4 q0 = rec[4 * id], q1 = rec[4 * id + 1], q2 = rec[4 * id + 2], q3 = rec[4 * id + 3];
      se0[j] = q0;
      se1[j] = make_float4(q1.x, q1.y, q1.z, pair_qmax(a.ln_inv_amin, q1.y));
      se2[j] = make_float4(q2.x, q2.y, q2.z, __expf(q1.y));
      se3[j] = make_float4(q3.x, q3.y, q1.w, q2.w);  // exact offsets, packed rect x / y ranges
    }
    __syncthreads();
  // a half-warp per list entry: the two entries of a warp share its setup and reduction
  // instructions (small footprints leave most of a full warp idle)
  for (int jb = 2 * warp; jb < cnt_e; jb += 2 * nw) {
    const int j = jb + (lane >> 4);
    const bool valid = j < cnt_e;
    const int jj = valid ? j : jb;
    const uint32_t idx = sidx[jj];
    const float4 r0 = se0[jj], r1 = se1[jj], r2 = se2[jj], r3 = se3[jj];
    const float b2 = pmul(2.0f, r0.w), qmax = r1.w;
    const float sig = r2.w;
    const uint32_t rx = __float_as_uint(r3.z), ry = __float_as_uint(r3.w);
    const int x0 = max((int)(rx & 0xFFFF), tx0), x1 = min((int)(rx >> 16), tx0 + TILE - 1);
    const int y0 = max((int)(ry & 0xFFFF), ty0), y1 = min((int)(ry >> 16), ty0 + TILE - 1);
    const int wx = x1 - x0 + 1, cnt = valid ? wx * (y1 - y0 + 1) : 0;
    // k / wx for k < 256, wx <= 16 as a multiply-high (exact; tests/test_abi.py)
    const uint32_t magic = smagic[wx];
    float acc[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) acc[k] = 0.f;
    bool any = false;
    for (int k = lane & 15; k < cnt; k += 16) {
      const int row = (int)(((uint32_t)k * magic) >> 16);
      const int x = x0 + (k - row * wx), y = y0 + row;
      const int p = (y - ty0) * TILE + (x - tx0);
      GPS_DCHECK(p >= 0 && p < NP, CHK_SMEM);
      if (!(r1.z < slim[p])) continue;  // Eq. 1 indicator (and inactive pixels)
      const float q = pair_q(r0.x, r0.y, r0.z, b2, r1.x, (float)x, (float)y);
      if (!(q <= qmax)) continue;
      const float dx = ((float)x - r0.x) - r3.x, dy = ((float)y - r0.y) - r3.y;  // exact offsets
      const float qv = fmaf(r0.z * dx, dx, fmaf(2.f * r0.w * dx, dy, r1.x * dy * dy));
      const float ex = __expf(-0.5f * qv);
      const float al = sig * ex;
      const float4 gs = sgs[p];
      const float gA0 = gs.x, gA1 = gs.y, gA2 = gs.z;
      // dL/dalpha = A * sum_ch g_ch (c_ch - C*_ch)
      const float dal = gA0 * r2.x + gA1 * r2.y + gA2 * r2.z - gs.w;
      const float dpow = -al * dal;
      acc[0] = fmaf(-dpow, r0.z * dx + r0.w * dy, acc[0]);  // p_hat x
      acc[1] = fmaf(-dpow, r0.w * dx + r1.x * dy, acc[1]);  // p_hat y
      acc[2] = fmaf(dpow * 0.5f, dx * dx, acc[2]);           // conic a
      acc[3] = fmaf(dpow, dx * dy, acc[3]);                  // conic b
      acc[4] = fmaf(dpow * 0.5f, dy * dy, acc[4]);           // conic c
      acc[5] = fmaf(dal, ex, acc[5]);                        // sigma
      acc[6] = fmaf(gA0, al, acc[6]);                        // colour r, g, b
      acc[7] = fmaf(gA1, al, acc[7]);
      acc[8] = fmaf(gA2, al, acc[8]);
      any = true;
    }
    const uint32_t bal = __ballot_sync(0xFFFFFFFFu, any);
    if (!bal) continue;
    // half-warp reduce-scatter: 12 shuffles for the two entries; value k ends on one lane
    float l1[5], l2[3], l3[2], l4[1];
    rs_level<9, 5>(acc, l1, lane, 8);
    rs_level<5, 3>(l1, l2, lane, 4);
    rs_level<3, 2>(l2, l3, lane, 2);
    rs_level<2, 1>(l3, l4, lane, 1);
    // 2D gradient slot layout: [px, py, a, b | c, sigma, r, g | b, flag, -, -]
    if (vidx >= 0 && ((bal >> (lane & 16)) & 0xFFFFu)) atomicAdd(grad2d + 12 * (size_t)idx + vidx, l4[0]);
  }
  }
}

// --------------------------------------------------------------------------------------------
// k_backward_items: the same gradient, computed per (entry, pixel group) instead of per entry.
// The paper launches threads per Gaussian, each accumulating its gradient in registers, with
// Gaussians split into fixed-size pixel groups so that all threads do the same number of
// iterations (App. B).  Here, per tile: each listed entry's footprint inside the
// tile (rect x tile, row-major) is cut into groups of kGroupPx pixels; one THREAD takes one
// group, walks its pixels against the tile's pixel state in shared memory, keeps the 9 partial
// sums in registers and issues 3 vector reductions -- no warp reduction and no idle lanes on
// small footprints.
// --------------------------------------------------------------------------------------------
constexpr int kGroupPx = 32;

template <int TILE>
__global__ void __launch_bounds__(256) k_backward_items(RenderArgs a, const float4* __restrict__ rec,
                                                        const uint32_t* __restrict__ offsets,
                                                        const uint32_t* __restrict__ vals,
                                                        const uint32_t* __restrict__ tile_end,
                                                        const float* __restrict__ sdf_depth,
                                                        const float* __restrict__ cstar, const float* __restrict__ wg,
                                                        const uint32_t* __restrict__ target, const WsHeader* hdr,
                                                        float* grad2d) {
  constexpr int NP = TILE * TILE;
  __shared__ float4 sgs[NP];
  __shared__ float slim[NP];
  __shared__ uint32_t smagic[TILE + 1];  // ceil(65536 / w), w = 1..TILE
  if (threadIdx.x <= TILE) smagic[threadIdx.x] = threadIdx.x ? (65536u + threadIdx.x - 1u) / threadIdx.x : 0u;
  const int t = blockIdx.x;
  const int tx = t % a.tiles_x, ty = t / a.tiles_x;
  const uint32_t m = backward_pixel_state<TILE>(a, t, sdf_depth, cstar, wg, target, hdr, sgs, slim);
  __syncthreads();
  if (!m) return;
  const uint32_t start = min(offsets[t], a.cap);
  const uint32_t end = min(tile_end[t], a.cap);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int tx0 = tx * TILE, ty0 = ty * TILE;
  __shared__ float4 se0[256], se1[256], se2[256], se3[256];
  __shared__ int4 sgeo[256];    // per entry: x0, y0, wx, cnt of rect x tile
  __shared__ uint32_t sidx[256];
  __shared__ int sitem[256];    // exclusive offsets of the entries' groups
  __shared__ int swarp[8];
  for (uint32_t base = start; base < end; base += 256) {
    const int cnt_e = (int)min(256u, end - base);
    __syncthreads();
    int ng = 0;
    const int j = threadIdx.x;
    if (j < cnt_e) {
      const uint32_t id = vals[base + j];
      sidx[j] = id;
      const float4 q0 = rec[4 * id], q1 = rec[4 * id + 1], q2 = rec[4 * id + 2], q3 = rec[4 * id + 3];
      se0[j] = make_float4(q0.x, q0.y, q0.z, pmul(2.0f, q0.w));  // (px, py, a, 2b)
      se1[j] = make_float4(q1.x, q0.w, q1.z, pair_qmax(a.ln_inv_amin, q1.y));  // (c, b, d, q_max)
      se2[j] = make_float4(q2.x, q2.y, q2.z, __expf(q1.y));  // (r, g, b, sigma)
      se3[j] = make_float4(q3.x, q3.y, 0.f, 0.f);  // exact centre offsets
      const uint32_t rx = __float_as_uint(q1.w), ry = __float_as_uint(q2.w);
      const int x0 = max((int)(rx & 0xFFFF), tx0), x1 = min((int)(rx >> 16), tx0 + TILE - 1);
      const int y0 = max((int)(ry & 0xFFFF), ty0), y1 = min((int)(ry >> 16), ty0 + TILE - 1);
      const int wx = x1 - x0 + 1, cnt = wx * (y1 - y0 + 1);
      sgeo[j] = make_int4(x0, y0, wx, cnt);
      ng = (cnt + kGroupPx - 1) / kGroupPx;
    }
    // exclusive scan of the group counts over the batch
    int incl = ng;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xFFFFFFFFu, incl, o);
      if (lane >= o) incl += v;
    }
    if (lane == 31) swarp[warp] = incl;
    __syncthreads();
    int woff = 0, total = 0;
#pragma unroll
    for (int w = 0; w < 8; ++w) {
      const int v = swarp[w];
      woff += w < warp ? v : 0;
      total += v;
    }
    sitem[j] = woff + incl - ng;
    __syncthreads();
    for (int it = threadIdx.x; it < total; it += blockDim.x) {
      // the entry owning group `it`: the last entry whose first group is <= it
      int lo = 0, hi = cnt_e - 1;
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (sitem[mid] <= it) lo = mid; else hi = mid - 1;
      }
      const int e = lo;
      const int4 geo = sgeo[e];
      const float4 r0 = se0[e], r1 = se1[e], r2 = se2[e], r3 = se3[e];
      const uint32_t magic = smagic[geo.z];
      const int k0 = (it - sitem[e]) * kGroupPx, k1 = min(geo.w, k0 + kGroupPx);
      float acc[9];
#pragma unroll
      for (int k = 0; k < 9; ++k) acc[k] = 0.f;
      bool any = false;
      for (int k = k0; k < k1; ++k) {
        const int row = (int)(((uint32_t)k * magic) >> 16);
        const int x = geo.x + (k - row * geo.z), y = geo.y + row;
        const int p = (y - ty0) * TILE + (x - tx0);
        if (!(r1.z < slim[p])) continue;  // Eq. 1 indicator (and inactive pixels)
        const float q = pair_q(r0.x, r0.y, r0.z, r0.w, r1.x, (float)x, (float)y);
        if (!(q <= r1.w)) continue;
        const float dx = ((float)x - r0.x) - r3.x, dy = ((float)y - r0.y) - r3.y;  // exact offsets
        const float qv = fmaf(r0.z * dx, dx, fmaf(2.f * r1.y * dx, dy, r1.x * dy * dy));
        const float ex = __expf(-0.5f * qv);
        const float al = r2.w * ex;
        const float4 gs = sgs[p];
        // dL/dalpha = A * sum_ch g_ch (c_ch - C*_ch)
        const float dal = gs.x * r2.x + gs.y * r2.y + gs.z * r2.z - gs.w;
        const float dpow = -al * dal;
        acc[0] = fmaf(-dpow, r0.z * dx + r1.y * dy, acc[0]);  // p_hat x
        acc[1] = fmaf(-dpow, r1.y * dx + r1.x * dy, acc[1]);  // p_hat y
        acc[2] = fmaf(dpow * 0.5f, dx * dx, acc[2]);           // conic a
        acc[3] = fmaf(dpow, dx * dy, acc[3]);                  // conic b
        acc[4] = fmaf(dpow * 0.5f, dy * dy, acc[4]);           // conic c
        acc[5] = fmaf(dal, ex, acc[5]);                        // sigma
        acc[6] = fmaf(gs.x, al, acc[6]);                       // colour r, g, b
        acc[7] = fmaf(gs.y, al, acc[7]);
        acc[8] = fmaf(gs.z, al, acc[8]);
        any = true;
      }
      if (any) {
        // 2D gradient slot layout: [px, py, a, b | c, sigma, r, g | b, flag, -, -]
        float* gp = grad2d + 12 * (size_t)sidx[e];
        red_add_v4(reinterpret_cast<float4*>(gp), acc[0], acc[1], acc[2], acc[3]);
        red_add_v4(reinterpret_cast<float4*>(gp + 4), acc[4], acc[5], acc[6], acc[7]);
        atomicAdd(gp + 8, acc[8]);
      }
    }
  }
}

// ============================================================================================
// k_grad_adam: raw-parameter gradient (R-GRAD chain rule) fused with dense Adam (R-ADAM)
// ============================================================================================
struct AdamArgs {
  float b1, b2, eps;
  float step_xyz, step_ls, step_rot, step_op, step_sh0, step_shr;  // lr / (1 - b1^t)
  float inv_sqrt_bc2;                                               // 1 / sqrt(1 - b2^t)
};


constexpr int kChainThreads = 128;
constexpr int kAdamThreads = 256;

// Raw-parameter gradient of one Gaussian from its 2D gradients (R-GRAD chain rule).  Outputs
// gx[3], gls[3], gq[4], gop, dcol[3] (clamped channels zeroed) and the SH basis Y[16] at the view
// direction (the SH gradient is Y[k] * dcol[ch]).
// fp64 re-projection for the backward chain only (forward membership stays P32):
// Sigma_2D can be ill-conditioned (thin, anisotropic Gaussians), and the conic-inverse VJP scales
// fp32 rounding by cond(Sigma_2D)^2; B200's FP64 rate makes this per-Gaussian step cheap.
struct ProjD {
  double X[3], s[3], qh[4], qn, Rq[9], M[9], S[9], cu, cv, T[6], cxx, cxy, cyy, det;
  bool clx, cly;
};

__device__ __forceinline__ void project_f64(const Cam& c, float lowpass, const float* p, const float* ls,
                                            const float* q, ProjD& g) {
  const double D0 = (double)p[0] - c.t[0], D1 = (double)p[1] - c.t[1], D2 = (double)p[2] - c.t[2];
#pragma unroll
  for (int k = 0; k < 3; ++k) g.X[k] = (double)c.R[k] * D0 + (double)c.R[3 + k] * D1 + (double)c.R[6 + k] * D2;
#pragma unroll
  for (int k = 0; k < 3; ++k) g.s[k] = exp((double)ls[k]);
  const double q0 = q[0], q1 = q[1], q2 = q[2], q3 = q[3];
  g.qn = sqrt(q0 * q0 + q1 * q1 + q2 * q2 + q3 * q3);
  const double iq = 1.0 / g.qn;
  const double w = q0 * iq, x = q1 * iq, y = q2 * iq, z = q3 * iq;
  g.qh[0] = w; g.qh[1] = x; g.qh[2] = y; g.qh[3] = z;
  double* Rq = g.Rq;
  Rq[0] = 1.0 - 2.0 * (y * y + z * z); Rq[1] = 2.0 * (x * y - w * z); Rq[2] = 2.0 * (x * z + w * y);
  Rq[3] = 2.0 * (x * y + w * z); Rq[4] = 1.0 - 2.0 * (x * x + z * z); Rq[5] = 2.0 * (y * z - w * x);
  Rq[6] = 2.0 * (x * z - w * y); Rq[7] = 2.0 * (y * z + w * x); Rq[8] = 1.0 - 2.0 * (x * x + y * y);
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int cc = 0; cc < 3; ++cc) g.M[3 * r + cc] = Rq[3 * r + cc] * g.s[cc];
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int cc = 0; cc < 3; ++cc)
      g.S[3 * r + cc] = g.M[3 * r] * g.M[3 * cc] + g.M[3 * r + 1] * g.M[3 * cc + 1] + g.M[3 * r + 2] * g.M[3 * cc + 2];
  const double limx = 1.3 * ((double)c.W / (2.0 * c.fx)), limy = 1.3 * ((double)c.H / (2.0 * c.fy));
  const double txz = g.X[0] / g.X[2], tyz = g.X[1] / g.X[2];
  g.clx = (txz < -limx || txz > limx);
  g.cly = (tyz < -limy || tyz > limy);
  g.cu = txz < -limx ? -limx : (txz > limx ? limx : txz);
  g.cv = tyz < -limy ? -limy : (tyz > limy ? limy : tyz);
  const double iz = 1.0 / g.X[2];
  const double J00 = c.fx * iz, J02 = -c.fx * g.cu * iz, J11 = c.fy * iz, J12 = -c.fy * g.cv * iz;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    g.T[k] = J00 * c.R[k * 3 + 0] + J02 * c.R[k * 3 + 2];
    g.T[3 + k] = J11 * c.R[k * 3 + 1] + J12 * c.R[k * 3 + 2];
  }
  double U[6];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int k = 0; k < 3; ++k)
      U[3 * a + k] = g.T[3 * a] * g.S[k] + g.T[3 * a + 1] * g.S[3 + k] + g.T[3 * a + 2] * g.S[6 + k];
  g.cxx = U[0] * g.T[0] + U[1] * g.T[1] + U[2] * g.T[2] + lowpass;
  g.cxy = U[0] * g.T[3] + U[1] * g.T[4] + U[2] * g.T[5];
  g.cyy = U[3] * g.T[3] + U[4] * g.T[4] + U[5] * g.T[5] + lowpass;
  g.det = g.cxx * g.cyy - g.cxy * g.cxy;
}

__device__ __forceinline__ void chain3d(const RenderArgs& a, const gps_gaussians& g, int64_t i, float dpx, float dpy,
                                        float da, float db, float dcc, float dsig, float* dcol, float* gx,
                                        float* gls, float* gq, float& gop, float* Y, const float4* __restrict__ cgj) {
  const int nc = a.nc;
  const float* p = g.xyz + 3 * i;
  ProjD pr;
  project_f64(a.cam, a.lowpass, p, g.log_scale + 3 * i, g.rot + 4 * i, pr);
  SH h;
  view_dir(a.cam, p, a.deg, h);
#pragma unroll
  for (int k = 0; k < 16; ++k) Y[k] = k < nc ? h.Y[k] : 0.f;
  // opacity: sigma = sigmoid(o)
  const float sig = 1.0f / (1.0f + __expf(-g.opacity_raw[i]));
  gop = dsig * sig * (1.f - sig);
  // colour -> view direction through the Jacobian Gc[ch][e] = sum_k SH_k,ch dY_k/d dir_e and
  // the clamp bits that k_preprocess stored (clamped channels get zero gradient)
  const float4 c0 = cgj[3 * i], c1 = cgj[3 * i + 1], c2 = cgj[3 * i + 2];
  const uint32_t clamp = __float_as_uint(c2.y);
#pragma unroll
  for (int ch = 0; ch < 3; ++ch)
    if (clamp & (1u << ch)) dcol[ch] = 0.f;
  const float Gc[9] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w, c2.x};
  float ddir[3];
#pragma unroll
  for (int e = 0; e < 3; ++e) ddir[e] = dcol[0] * Gc[e] + dcol[1] * Gc[3 + e] + dcol[2] * Gc[6 + e];
  const float dd = ddir[0] * h.dir[0] + ddir[1] * h.dir[1] + ddir[2] * h.dir[2];
  const float invn = 1.f / h.dnorm;
  double gxd[3];
#pragma unroll
  for (int e = 0; e < 3; ++e) gxd[e] = (double)((ddir[e] - h.dir[e] * dd) * invn);
  // conic (a, b, c) -> Sigma_2D (cxx, cxy, cyy)
  const double id = 1.0 / pr.det, id2 = id * id;
  const double cxx = pr.cxx, cxy = pr.cxy, cyy = pr.cyy;
  const double dcxx = da * (-cyy * cyy * id2) + db * (cxy * cyy * id2) + dcc * (id - cxx * cyy * id2);
  const double dcyy = da * (id - cyy * cxx * id2) + db * (cxy * cxx * id2) + dcc * (-cxx * cxx * id2);
  const double dcxy = da * (2.0 * cyy * cxy * id2) + db * (-id - 2.0 * cxy * cxy * id2) + dcc * (2.0 * cxx * cxy * id2);
  // Sigma_2D = T S T^T + lowpass I
  const double* T0 = pr.T;
  const double* T1 = pr.T + 3;
  double ST0[3], ST1[3];
#pragma unroll
  for (int r = 0; r < 3; ++r) {
    ST0[r] = pr.S[3 * r] * T0[0] + pr.S[3 * r + 1] * T0[1] + pr.S[3 * r + 2] * T0[2];
    ST1[r] = pr.S[3 * r] * T1[0] + pr.S[3 * r + 1] * T1[1] + pr.S[3 * r + 2] * T1[2];
  }
  double dS[9], dT0[3], dT1[3];
#pragma unroll
  for (int j = 0; j < 3; ++j) {
#pragma unroll
    for (int k = 0; k < 3; ++k) dS[3 * j + k] = dcxx * T0[j] * T0[k] + dcxy * T0[j] * T1[k] + dcyy * T1[j] * T1[k];
    dT0[j] = 2.0 * dcxx * ST0[j] + dcxy * ST1[j];
    dT1[j] = dcxy * ST0[j] + 2.0 * dcyy * ST1[j];
  }
  // T = J Wc  (Wc[r][c] = R[c][r])
  double dJ00 = 0.0, dJ02 = 0.0, dJ11 = 0.0, dJ12 = 0.0;
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    dJ00 += dT0[j] * a.cam.R[j * 3 + 0];
    dJ02 += dT0[j] * a.cam.R[j * 3 + 2];
    dJ11 += dT1[j] * a.cam.R[j * 3 + 1];
    dJ12 += dT1[j] * a.cam.R[j * 3 + 2];
  }
  const double z = pr.X[2], iz = 1.0 / z, iz2 = iz * iz;
  const double fx = a.cam.fx, fy = a.cam.fy;
  double dX[3] = {0.0, 0.0, 0.0};
  dX[2] += dJ00 * (-fx * iz2) + dJ11 * (-fy * iz2);
  const double dcu_dx = pr.clx ? 0.0 : iz, dcu_dz = pr.clx ? 0.0 : -pr.X[0] * iz2;
  const double dcv_dy = pr.cly ? 0.0 : iz, dcv_dz = pr.cly ? 0.0 : -pr.X[1] * iz2;
  dX[0] += dJ02 * (-fx * iz) * dcu_dx;
  dX[2] += dJ02 * (fx * pr.cu * iz2 - fx * iz * dcu_dz);
  dX[1] += dJ12 * (-fy * iz) * dcv_dy;
  dX[2] += dJ12 * (fy * pr.cv * iz2 - fy * iz * dcv_dz);
  dX[0] += dpx * fx * iz;
  dX[1] += dpy * fy * iz;
  dX[2] += dpx * (-fx * pr.X[0] * iz2) + dpy * (-fy * pr.X[1] * iz2);
#pragma unroll
  for (int r = 0; r < 3; ++r)
    gx[r] = (float)(gxd[r] + a.cam.R[3 * r] * dX[0] + a.cam.R[3 * r + 1] * dX[1] + a.cam.R[3 * r + 2] * dX[2]);
  // S = M M^T, M = Rq diag(s)
  double dRq[9];
#pragma unroll
  for (int l = 0; l < 3; ++l) {
    double ds = 0.0;
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      double dM = 0.0;
#pragma unroll
      for (int k = 0; k < 3; ++k) dM += (dS[3 * j + k] + dS[3 * k + j]) * pr.M[3 * k + l];
      dRq[3 * j + l] = dM * pr.s[l];
      ds += dM * pr.Rq[3 * j + l];
    }
    gls[l] = (float)(ds * pr.s[l]);
  }
  const double qw = pr.qh[0], qx = pr.qh[1], qy = pr.qh[2], qz = pr.qh[3];
  double dqh[4];
  dqh[0] = dRq[1] * (-2.0 * qz) + dRq[2] * (2.0 * qy) + dRq[3] * (2.0 * qz) + dRq[5] * (-2.0 * qx) +
           dRq[6] * (-2.0 * qy) + dRq[7] * (2.0 * qx);
  dqh[1] = dRq[1] * (2.0 * qy) + dRq[2] * (2.0 * qz) + dRq[3] * (2.0 * qy) + dRq[4] * (-4.0 * qx) +
           dRq[5] * (-2.0 * qw) + dRq[6] * (2.0 * qz) + dRq[7] * (2.0 * qw) + dRq[8] * (-4.0 * qx);
  dqh[2] = dRq[0] * (-4.0 * qy) + dRq[1] * (2.0 * qx) + dRq[2] * (2.0 * qw) + dRq[3] * (2.0 * qx) +
           dRq[5] * (2.0 * qz) + dRq[6] * (-2.0 * qw) + dRq[7] * (2.0 * qz) + dRq[8] * (-4.0 * qy);
  dqh[3] = dRq[0] * (-4.0 * qz) + dRq[1] * (-2.0 * qw) + dRq[2] * (2.0 * qx) + dRq[3] * (2.0 * qw) +
           dRq[4] * (-4.0 * qz) + dRq[5] * (2.0 * qy) + dRq[6] * (2.0 * qx) + dRq[7] * (2.0 * qy);
  const double dot = dqh[0] * qw + dqh[1] * qx + dqh[2] * qy + dqh[3] * qz;
  const double iqn = 1.0 / pr.qn;
#pragma unroll
  for (int k = 0; k < 4; ++k) gq[k] = (float)((dqh[k] - pr.qh[k] * dot) * iqn);
}

// k_chain: one thread per Gaussian with a non-zero 2D gradient.  ACCUM = 0 writes the 128-byte
// gradient record {gx, gls, gq, gop, dcol, Y[16]} and flags it in the (per-iteration zeroed) 2D
// gradient slot; ACCUM = 1 adds the dense raw gradient into gbuf (multi-view rounds).
template <int ACCUM>
__global__ void __launch_bounds__(kChainThreads, 4) k_chain(RenderArgs a, gps_gaussians g, float4* grad2d,
                                                         float4* rec3, gps_gaussians gbuf,
                                                         const float4* __restrict__ cgj) {
  const int64_t i = blockIdx.x * (int64_t)kChainThreads + threadIdx.x;
  if (i >= a.n) return;
  const float4 q0 = grad2d[3 * i], q1 = grad2d[3 * i + 1], q2 = grad2d[3 * i + 2];
  float dcol[3] = {q1.z, q1.w, q2.x};
  const bool nz = (q0.x != 0.f) | (q0.y != 0.f) | (q0.z != 0.f) | (q0.w != 0.f) | (q1.x != 0.f) | (q1.y != 0.f) |
                  (dcol[0] != 0.f) | (dcol[1] != 0.f) | (dcol[2] != 0.f);
  if (!nz) return;
  float gx[3], gls[3], gq[4], gop, Y[16];
  chain3d(a, g, i, q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, dcol, gx, gls, gq, gop, Y, cgj);
  if (ACCUM) {
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      gbuf.xyz[3 * i + k] += gx[k];
      gbuf.log_scale[3 * i + k] += gls[k];
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) gbuf.rot[4 * i + k] += gq[k];
    gbuf.opacity_raw[i] += gop;
    float* sh = gbuf.sh + (size_t)i * a.nc * 3;
    for (int k = 0; k < a.nc; ++k)
#pragma unroll
      for (int ch = 0; ch < 3; ++ch) sh[3 * k + ch] += Y[k] * dcol[ch];
    return;
  }
  float4* r = rec3 + 8 * i;
  r[0] = make_float4(gx[0], gx[1], gx[2], gls[0]);
  r[1] = make_float4(gls[1], gls[2], gq[0], gq[1]);
  r[2] = make_float4(gq[2], gq[3], gop, dcol[0]);
  r[3] = make_float4(dcol[1], dcol[2], 0.f, 0.f);
  r[4] = make_float4(Y[0], Y[1], Y[2], Y[3]);
  r[5] = make_float4(Y[4], Y[5], Y[6], Y[7]);
  r[6] = make_float4(Y[8], Y[9], Y[10], Y[11]);
  r[7] = make_float4(Y[12], Y[13], Y[14], Y[15]);
  grad2d[3 * i + 2].y = 1.0f;  // record valid for this iteration (the slot is re-zeroed by k_preprocess)
}

// k_adam: dense Adam (R-ADAM) streamed over float4 units of every parameter array (all five SoA
// groups in one flattened index space).  Gradients: external arrays (gps_adam_step), or the
// flagged k_chain record (0 if unflagged) plus an optional dense multi-view accumulator.
struct AdamSrc {
  const float4* grad2d;  // flags (nullable in external mode)
  const float* rec3;     // 32 floats per Gaussian
  gps_gaussians gbuf;    // dense accumulator or external gradient (nullable pointers)
  int has_gbuf, external;
  gps_gaussians gout;
  int has_gout;
};

// One float4 unit of one parameter group per thread, one CTA per chunk of kAdamThreads units;
// each group's unit range is padded to whole chunks, so the group -- hence the floats per
// Gaussian DIM, the step size and the gradient source -- is a compile-time constant inside a
// CTA.  Every load of a unit (p, m, v, the gradient flag and record entries) is independent and
// issued before any is used: one memory latency per unit, and ~10 resident CTAs per SM keep
// enough bytes in flight for HBM.  The update divides and takes the square root with the
// approximate MUFU forms (relative error ~2^-22 on the step, far inside R-ADAM's 1e-6).
constexpr uint32_t kAdamChunk = kAdamThreads;

__device__ __forceinline__ float sqrt_approx(float x) {
  float r;
  asm("sqrt.approx.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// R-ADAM for one element, in explicit rounding steps (no contraction left to the compiler), so
// that every kernel applying it -- k_adam and the fused k_chain_adam -- produces the same bits
__device__ __forceinline__ void adam_elem(float& p, float& m, float& v, float gr, float st, const AdamArgs& ad) {
  m = __fmaf_rn(ad.b1, m, __fmul_rn(1.0f - ad.b1, gr));
  v = __fmaf_rn(ad.b2, v, __fmul_rn(__fmul_rn(1.0f - ad.b2, gr), gr));
  p = __fsub_rn(p, __fdividef(__fmul_rn(st, m), __fmaf_rn(sqrt_approx(v), ad.inv_sqrt_bc2, ad.eps)));
}

template <int GRP, int DIM>
__device__ __forceinline__ void adam_unit(float* __restrict__ P, float* __restrict__ M, float* __restrict__ V,
                                          const float* __restrict__ E, float* __restrict__ O, uint32_t len,
                                          uint32_t u, const AdamSrc& src, const AdamArgs& ad, float step) {
  const uint32_t e0 = 4u * u;
  if (e0 >= len) return;
  const uint32_t cnt = min(4u, len - e0);
  const float* __restrict__ rec3 = src.rec3;
  const float4* __restrict__ flags = src.grad2d;
  float p[4], m[4], v[4], fl[4], ra[4], rb[4], ex[4];
  if (cnt == 4u) {
    const float4 p4 = *reinterpret_cast<const float4*>(P + e0), m4 = *reinterpret_cast<const float4*>(M + e0),
                 v4 = *reinterpret_cast<const float4*>(V + e0);
    p[0] = p4.x; p[1] = p4.y; p[2] = p4.z; p[3] = p4.w;
    m[0] = m4.x; m[1] = m4.y; m[2] = m4.z; m[3] = m4.w;
    v[0] = v4.x; v[1] = v4.y; v[2] = v4.z; v[3] = v4.w;
  } else {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      p[k] = (uint32_t)k < cnt ? P[e0 + k] : 0.f;
      m[k] = (uint32_t)k < cnt ? M[e0 + k] : 0.f;
      v[k] = (uint32_t)k < cnt ? V[e0 + k] : 0.f;
    }
  }
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const uint32_t e = e0 + min((uint32_t)k, cnt - 1u), gi = e / DIM, comp = e - gi * DIM;  // DIM: constant
    fl[k] = 0.f; ra[k] = 0.f; rb[k] = 1.f; ex[k] = 0.f;
    if (src.external) {
      ex[k] = E[e];
    } else {
      fl[k] = flags[3 * gi + 2].y;  // k_chain's record is valid this iteration
      const float* r = rec3 + 32 * gi;
      if (GRP == 0) ra[k] = r[comp];
      else if (GRP == 1) ra[k] = r[3 + comp];
      else if (GRP == 2) ra[k] = r[6 + comp];
      else if (GRP == 3) ra[k] = r[10];
      else { ra[k] = r[16 + comp / 3]; rb[k] = r[11 + comp % 3]; }  // sh: Y[k] * dcol[ch]
      if (src.has_gbuf) ex[k] = E[e];
    }
  }
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    float gr;
    if (src.external) {
      gr = ex[k];
    } else {
      gr = fl[k] != 0.f ? (GRP == 4 ? ra[k] * rb[k] : ra[k]) : 0.f;
      if (src.has_gbuf) gr += ex[k];
    }
    if (src.has_gout && (uint32_t)k < cnt) O[e0 + k] = gr;
    const uint32_t comp = (e0 + k) % DIM;
    const float st = (GRP == 4 && comp < 3u) ? ad.step_sh0 : step;
    adam_elem(p[k], m[k], v[k], gr, st, ad);
  }
  if (cnt == 4u) {
    *reinterpret_cast<float4*>(P + e0) = make_float4(p[0], p[1], p[2], p[3]);
    *reinterpret_cast<float4*>(M + e0) = make_float4(m[0], m[1], m[2], m[3]);
    *reinterpret_cast<float4*>(V + e0) = make_float4(v[0], v[1], v[2], v[3]);
  } else {
    for (uint32_t k = 0; k < cnt; ++k) {
      P[e0 + k] = p[k];
      M[e0 + k] = m[k];
      V[e0 + k] = v[k];
    }
  }
}

__host__ __device__ __forceinline__ uint32_t adam_chunks(uint32_t len) {
  return ((len + 3u) / 4u + kAdamChunk - 1u) / kAdamChunk;
}
__host__ __device__ __forceinline__ uint32_t adam_total_chunks(uint32_t n, uint32_t nsh) {
  return 2u * adam_chunks(3u * n) + adam_chunks(4u * n) + adam_chunks(n) + adam_chunks(nsh * n);
}

__global__ void __launch_bounds__(kAdamThreads) k_adam(RenderArgs a, gps_gaussians g, gps_gaussians gm, gps_gaussians gv,
                                                       AdamSrc src, AdamArgs ad) {
  // 32-bit element indices: n * 3 (deg+1)^2 < 2^31 is checked on the host
  const uint32_t n = (uint32_t)a.n, nsh = 3u * (uint32_t)a.nc;
  const uint32_t c1 = adam_chunks(3u * n), c2 = c1 + adam_chunks(3u * n), c3 = c2 + adam_chunks(4u * n),
                 c4 = c3 + adam_chunks(n);
  const uint32_t c = blockIdx.x;  // CTA-uniform group
  if (c < c1) {
    adam_unit<0, 3>(g.xyz, gm.xyz, gv.xyz, src.gbuf.xyz, src.gout.xyz, 3u * n, c * kAdamChunk + threadIdx.x, src, ad,
                    ad.step_xyz);
  } else if (c < c2) {
    adam_unit<1, 3>(g.log_scale, gm.log_scale, gv.log_scale, src.gbuf.log_scale, src.gout.log_scale, 3u * n,
                    (c - c1) * kAdamChunk + threadIdx.x, src, ad, ad.step_ls);
  } else if (c < c3) {
    adam_unit<2, 4>(g.rot, gm.rot, gv.rot, src.gbuf.rot, src.gout.rot, 4u * n, (c - c2) * kAdamChunk + threadIdx.x,
                    src, ad, ad.step_rot);
  } else if (c < c4) {
    adam_unit<3, 1>(g.opacity_raw, gm.opacity_raw, gv.opacity_raw, src.gbuf.opacity_raw, src.gout.opacity_raw, n,
                    (c - c3) * kAdamChunk + threadIdx.x, src, ad, ad.step_op);
  } else {
    const uint32_t u = (c - c4) * kAdamChunk + threadIdx.x;
    switch (nsh) {
      case 3: adam_unit<4, 3>(g.sh, gm.sh, gv.sh, src.gbuf.sh, src.gout.sh, nsh * n, u, src, ad, ad.step_shr); break;
      case 12: adam_unit<4, 12>(g.sh, gm.sh, gv.sh, src.gbuf.sh, src.gout.sh, nsh * n, u, src, ad, ad.step_shr); break;
      case 27: adam_unit<4, 27>(g.sh, gm.sh, gv.sh, src.gbuf.sh, src.gout.sh, nsh * n, u, src, ad, ad.step_shr); break;
      default: adam_unit<4, 48>(g.sh, gm.sh, gv.sh, src.gbuf.sh, src.gout.sh, nsh * n, u, src, ad, ad.step_shr); break;
    }
  }
}

// --------------------------------------------------------------------------------------------
// k_chain_adam (a11 fused, single-view refine steps): one CTA per chunk of kCaG Gaussians.
//  phase A: a thread per Gaussian runs the R-GRAD chain (chain3d, as k_chain) when its 2D
//           gradient is non-zero and leaves the raw gradient terms in shared memory
//           {gx[3], gls[3], gq[4], gop, dcol[3], Y[16]} (zeros otherwise: R-ADAM's dense update
//           with a zero gradient, as k_adam's unflagged record);
//  phase B: the CTA streams the chunk's slices of the five parameter groups (p, m, v as float4
//           units, 4 units per thread in flight) and applies adam_elem with the gradient read
//           from shared memory (SH: Y[k] * dcol[ch], the product k_adam forms from the record).
// Same arithmetic as k_chain<0> + k_adam, so the same bits (tests/test_gpu_render_refine.py),
// without the 128-byte record round trip and one launch; CTAs of an SM in different phases
// overlap the latency-bound chain with the streaming update.
// --------------------------------------------------------------------------------------------
constexpr int kCaG = 128;      // Gaussians per CTA (= threads)
constexpr int kCaStride = 31;  // floats per Gaussian in shared memory (odd: conflict-free columns)

struct CaGroup {
  float* P;
  float* M;
  float* V;
  float* O;
};

// phase A for Gaussian t of the chunk starting at g0 (cg Gaussians): its raw gradient terms into
// sgb[t * kCaStride ...] (zeros without a 2D gradient)
__device__ __forceinline__ void ca_phase_a(const RenderArgs& a, const gps_gaussians& g,
                                           const float4* __restrict__ grad2d, const float4* __restrict__ cgj,
                                           int64_t g0, int cg, int t, float* sgb) {
  float* o = sgb + t * kCaStride;
#pragma unroll
  for (int k = 0; k < 30; ++k) o[k] = 0.f;
  if (t >= cg) return;
  const int64_t i = g0 + t;
  const float4 q0 = grad2d[3 * i], q1 = grad2d[3 * i + 1], q2 = grad2d[3 * i + 2];
  float dcol[3] = {q1.z, q1.w, q2.x};
  const bool nz = (q0.x != 0.f) | (q0.y != 0.f) | (q0.z != 0.f) | (q0.w != 0.f) | (q1.x != 0.f) | (q1.y != 0.f) |
                  (dcol[0] != 0.f) | (dcol[1] != 0.f) | (dcol[2] != 0.f);
  if (!nz) return;
  float gx[3], gls[3], gq[4], gop, Y[16];
  chain3d(a, g, i, q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, dcol, gx, gls, gq, gop, Y, cgj);
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    o[k] = gx[k];
    o[3 + k] = gls[k];
    o[11 + k] = dcol[k];
  }
#pragma unroll
  for (int k = 0; k < 4; ++k) o[6 + k] = gq[k];
  o[10] = gop;
#pragma unroll
  for (int k = 0; k < 16; ++k) o[14 + k] = Y[k];
}

// the chunk's five group slices (pointers, lengths, float4-unit ranges, floats per Gaussian, step
// sizes, gradient offsets): built by one thread into shared memory (dynamically indexed per unit)
struct CaTable {
  CaGroup grp[5];
  uint32_t len[5], dims[5], ub[6];
  float idim[5], steps[5];
  int soff[5];
  int cg;
};
__device__ __forceinline__ void ca_table(CaTable& T, const RenderArgs& a, const gps_gaussians& g,
                                         const gps_gaussians& gm, const gps_gaussians& gv, const gps_gaussians& gout,
                                         int has_gout, const AdamArgs& ad, int64_t g0, int cg) {
  const uint32_t nsh = 3u * (uint32_t)a.nc;
  const uint32_t ln[5] = {3u * cg, 3u * cg, 4u * cg, (uint32_t)cg, nsh * cg};
  const uint32_t dm[5] = {3u, 3u, 4u, 1u, nsh};
  const int so[5] = {0, 3, 6, 10, 14};
  const float st[5] = {ad.step_xyz, ad.step_ls, ad.step_rot, ad.step_op, ad.step_shr};
  float* const Ps[5] = {g.xyz + 3 * g0, g.log_scale + 3 * g0, g.rot + 4 * g0, g.opacity_raw + g0, g.sh + nsh * g0};
  float* const Ms[5] = {gm.xyz + 3 * g0, gm.log_scale + 3 * g0, gm.rot + 4 * g0, gm.opacity_raw + g0, gm.sh + nsh * g0};
  float* const Vs[5] = {gv.xyz + 3 * g0, gv.log_scale + 3 * g0, gv.rot + 4 * g0, gv.opacity_raw + g0, gv.sh + nsh * g0};
  T.ub[0] = 0;
  T.cg = cg;
#pragma unroll
  for (int q = 0; q < 5; ++q) {
    T.len[q] = ln[q];
    T.dims[q] = dm[q];
    T.idim[q] = 1.0f / (float)dm[q];
    T.steps[q] = st[q];
    T.soff[q] = so[q];
    T.ub[q + 1] = T.ub[q] + (ln[q] + 3u) / 4u;
    T.grp[q].P = Ps[q];
    T.grp[q].M = Ms[q];
    T.grp[q].V = Vs[q];
  }
  T.grp[0].O = has_gout ? gout.xyz + 3 * g0 : nullptr;
  T.grp[1].O = has_gout ? gout.log_scale + 3 * g0 : nullptr;
  T.grp[2].O = has_gout ? gout.rot + 4 * g0 : nullptr;
  T.grp[3].O = has_gout ? gout.opacity_raw + g0 : nullptr;
  T.grp[4].O = has_gout ? gout.sh + nsh * g0 : nullptr;
}

// phase B by threads tid = 0 .. nthr-1: the chunk's units, kU per thread in flight
__device__ __forceinline__ void ca_phase_b(const CaTable& T, const float* sg, int tid, int nthr, int has_gout,
                                           const AdamArgs& ad) {
  const int cg = T.cg;
  const uint32_t* ub = T.ub;
  const uint32_t* len = T.len;
  const uint32_t* dims = T.dims;
  const float* idim = T.idim;
  const float* steps = T.steps;
  const int* soff = T.soff;
  const CaGroup* grp = T.grp;
  constexpr int kU = 4;  // units per thread in flight
  for (uint32_t U0 = tid; U0 < ub[5]; U0 += kU * nthr) {
    float p[kU][4], m[kU][4], v[kU][4];
    int gq[kU];
    uint32_t e0[kU], cnt[kU];
#pragma unroll
    for (int j = 0; j < kU; ++j) {
      const uint32_t U = U0 + j * nthr;
      int q = 0;
#pragma unroll
      for (int r = 1; r < 5; ++r) q += U >= ub[r];
      gq[j] = q;
      cnt[j] = 0;
      e0[j] = 0;
      if (U < ub[5]) {
        e0[j] = 4u * (U - ub[q]);
        cnt[j] = min(4u, len[q] - e0[j]);
      }
      const CaGroup G = grp[q];
      if (cnt[j] == 4u) {
        const float4 p4 = *reinterpret_cast<const float4*>(G.P + e0[j]);
        const float4 m4 = *reinterpret_cast<const float4*>(G.M + e0[j]);
        const float4 v4 = *reinterpret_cast<const float4*>(G.V + e0[j]);
        p[j][0] = p4.x; p[j][1] = p4.y; p[j][2] = p4.z; p[j][3] = p4.w;
        m[j][0] = m4.x; m[j][1] = m4.y; m[j][2] = m4.z; m[j][3] = m4.w;
        v[j][0] = v4.x; v[j][1] = v4.y; v[j][2] = v4.z; v[j][3] = v4.w;
      } else {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const bool in = (uint32_t)k < cnt[j];
          p[j][k] = in ? G.P[e0[j] + k] : 0.f;
          m[j][k] = in ? G.M[e0[j] + k] : 0.f;
          v[j][k] = in ? G.V[e0[j] + k] : 0.f;
        }
      }
    }
#pragma unroll
    for (int j = 0; j < kU; ++j) {
      if (cnt[j] == 0u) continue;
      const int q = gq[j];
      const uint32_t dim = dims[q];
      const CaGroup G = grp[q];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint32_t e = e0[j] + k;
        // e / dim for e < 48 * kCaG: (e + 1/2) / dim is >= 1/(2 dim) from an integer, far beyond
        // the fp32 error of the product
        const uint32_t gl = __float2uint_rz(((float)e + 0.5f) * idim[q]), comp = e - gl * dim;
        GPS_DCHECK((uint32_t)k >= cnt[j] || (gl < (uint32_t)cg && comp < dim && e < len[q]), CHK_ADAM);
        const float* o = sg + gl * kCaStride;
        float gr, st = steps[q];
        if (q == 4) {
          gr = o[14 + comp / 3u] * o[11 + comp % 3u];
          if (comp < 3u) st = ad.step_sh0;
        } else {
          gr = o[soff[q] + comp];
        }
        if ((uint32_t)k < cnt[j]) {
          if (has_gout) G.O[e] = gr;
          adam_elem(p[j][k], m[j][k], v[j][k], gr, st, ad);
        }
      }
      if (cnt[j] == 4u) {
        *reinterpret_cast<float4*>(G.P + e0[j]) = make_float4(p[j][0], p[j][1], p[j][2], p[j][3]);
        *reinterpret_cast<float4*>(G.M + e0[j]) = make_float4(m[j][0], m[j][1], m[j][2], m[j][3]);
        *reinterpret_cast<float4*>(G.V + e0[j]) = make_float4(v[j][0], v[j][1], v[j][2], v[j][3]);
      } else {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          if ((uint32_t)k < cnt[j]) {
            G.P[e0[j] + k] = p[j][k];
            G.M[e0[j] + k] = m[j][k];
            G.V[e0[j] + k] = v[j][k];
          }
        }
      }
    }
  }
}

__global__ void __launch_bounds__(kCaG, 4) k_chain_adam(RenderArgs a, gps_gaussians g, gps_gaussians gm,
                                                      gps_gaussians gv, const float4* __restrict__ grad2d,
                                                      const float4* __restrict__ cgj, gps_gaussians gout,
                                                      int has_gout, AdamArgs ad) {
  __shared__ float sg[kCaG * kCaStride];
  __shared__ CaTable tab;
  const int64_t g0 = (int64_t)blockIdx.x * kCaG;
  const int cg = (int)(a.n - g0 < (int64_t)kCaG ? a.n - g0 : (int64_t)kCaG);
  ca_phase_a(a, g, grad2d, cgj, g0, cg, threadIdx.x, sg);
  if (threadIdx.x == 0) ca_table(tab, a, g, gm, gv, gout, has_gout, ad, g0, cg);
  __syncthreads();
  ca_phase_b(tab, sg, threadIdx.x, kCaG, has_gout, ad);
}

}  // namespace gps

using namespace gps;

namespace {

bool valid_K(const gps_intrinsics* K) {
  return K && K->width > 0 && K->height > 0 && K->fx > 0 && K->fy > 0 && K->width <= 65535 && K->height <= 65535;
}

gps_status check_gaussians(const gps_gaussians* g, const char* who) {
  if (!g) return invalid(std::string(who) + ": null Gaussians");
  if (g->n < 0 || g->n > (1ll << 25)) return invalid(std::string(who) + ": Gaussian count must be <= 2^25");
  if (g->sh_degree < 0 || g->sh_degree > 3) return invalid(std::string(who) + ": sh_degree must be 0..3");
  if (g->n > 0 && (!g->xyz || !g->log_scale || !g->rot || !g->opacity_raw || !g->sh))
    return invalid(std::string(who) + ": null Gaussian array");
  if (g->n > 0 && (!aligned16(g->xyz) || !aligned16(g->log_scale) || !aligned16(g->rot) ||
                   !aligned16(g->opacity_raw) || !aligned16(g->sh)))
    return invalid(std::string(who) + ": Gaussian arrays must be 16-byte aligned");
  return GPS_OK;
}

bool same_shape(const gps_gaussians* a, const gps_gaussians* b) { return a->n == b->n && a->sh_degree == b->sh_degree; }

RenderArgs make_args(const gps_gaussians* g, const gps_intrinsics* K, const gps_pose* T, const gps_render_config* c,
                     int64_t cap) {
  RenderArgs a;
  a.cam.fx = K->fx; a.cam.fy = K->fy; a.cam.cx = K->cx; a.cam.cy = K->cy; a.cam.W = K->width; a.cam.H = K->height;
  for (int i = 0; i < 9; ++i) a.cam.R[i] = T->R[i];
  for (int i = 0; i < 3; ++i) a.cam.t[i] = T->t[i];
  a.eps = c->eps_depth; a.alpha_min = c->alpha_min; a.near_z = c->near_z; a.lowpass = c->lowpass;
  a.ln_inv_amin = (float)(-std::log((double)c->alpha_min));
  a.tile = c->tile;
  a.tiles_x = (K->width + c->tile - 1) / c->tile;
  a.tiles_y = (K->height + c->tile - 1) / c->tile;
  a.n = g->n;
  a.deg = g->sh_degree;
  a.nc = (g->sh_degree + 1) * (g->sh_degree + 1);
  a.cap = (uint32_t)std::min<int64_t>(cap, 0xFFFFFFFFll);
  return a;
}

gps_gaussians slice_params(const gps_gaussians* g, float* base) {
  // a gps_gaussians view over one dense float buffer laid out group after group
  gps_gaussians o = *g;
  const int64_t n = g->n;
  o.xyz = base;
  o.log_scale = base + 3 * n;
  o.rot = base + 6 * n;
  o.opacity_raw = base + 10 * n;
  o.sh = base + align_up(11 * n, 4);
  return o;
}
int64_t gbuf_floats(const gps_gaussians* g) {
  return (int64_t)align_up(11 * g->n, 4) + 3 * g->n * (g->sh_degree + 1) * (g->sh_degree + 1);
}

bool sort_long_ready() {  // once per process (before any stream capture: see gps_refine_round)
  static const bool ok = cudaFuncSetAttribute(k_sort_long, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              8 * kLongSmem) == cudaSuccess;
  return ok;
}

struct View1 {
  const gps_intrinsics* K;
  const gps_pose* T;
  const float* sdf_depth;
  const float* sdf_color;
  const uint8_t* target;
};

// forward of one view: preprocess .. sort_blend.  ws must follow ws_layout(refine).
gps_status forward_view(const gps_gaussians* g, const View1& v, const gps_render_config* c, char* ws,
                        const WsLayout& L, int64_t cap, float* out_color, float* out_weight, float* loss_out,
                        int accumulate_loss, bool zero_grad2d, cudaStream_t s,
                        unsigned long long* counters = nullptr) {
  RenderArgs a = make_args(g, v.K, v.T, c, cap);
  WsHeader* hdr = reinterpret_cast<WsHeader*>(ws + L.hdr);
  {
    GPS_PROF(K_MEMSET, s);
    GPS_CHECK_CUDA(cudaMemsetAsync(ws + L.zero_begin, 0, L.zero_bytes, s));
  }
  SplatPtrs sp;
  sp.rec = reinterpret_cast<float4*>(ws + L.records);
  sp.grad2d = zero_grad2d ? reinterpret_cast<float4*>(ws + L.grad2d) : nullptr;
  sp.cgj = zero_grad2d ? reinterpret_cast<float4*>(ws + L.cgj) : nullptr;
  sp.counts = reinterpret_cast<uint32_t*>(ws + L.counts);
  sp.ranks = reinterpret_cast<uint4*>(ws + L.ranks);
  sp.bigcounts = reinterpret_cast<uint32_t*>(ws + L.bigcounts);
  sp.hdr = hdr;
  const int n_tiles = a.tiles_x * a.tiles_y;
  if (g->n > 0) {
    GPS_PROF(K_PREPROCESS, s);
    k_preprocess<<<(unsigned)((g->n + 255) / 256), 256, 0, s>>>(a, *g, sp);
    GPS_CHECK_LAUNCH("k_preprocess");
  }
  WsHeader stat{};
  stat.magic = kWsMagic; stat.tile = a.tile; stat.tiles_x = a.tiles_x; stat.tiles_y = a.tiles_y;
  stat.width = a.cam.W; stat.height = a.cam.H; stat.n_tiles = n_tiles; stat.cap_pairs = a.cap; stat.n = g->n;
  stat.off_vals = L.vals; stat.off_offsets = L.offsets; stat.off_tile_end = L.tile_end;
  uint32_t* offsets = reinterpret_cast<uint32_t*>(ws + L.offsets);
  {
    GPS_PROF(K_SCAN, s);
    k_scan<<<1, 1024, 0, s>>>(sp.counts, sp.bigcounts, offsets, n_tiles, hdr, stat, overflow_flag_dev(),
                              reinterpret_cast<uint2*>(ws + L.extra), L.extra_cap,
                              reinterpret_cast<uint32_t*>(ws + L.pbase), L.part_cap,
                              reinterpret_cast<uint32_t*>(ws + L.longl));
  }
  GPS_CHECK_LAUNCH("k_scan");
  uint32_t* vals = reinterpret_cast<uint32_t*>(ws + L.vals);
  if (g->n > 0) {
    GPS_PROF(K_EMIT, s);
    k_emit<<<(unsigned)((g->n + 255) / 256), 256, 0, s>>>(a, sp.rec, sp.ranks, sp.counts, offsets,
                                                          reinterpret_cast<uint32_t*>(ws + L.cursor), vals);
    GPS_CHECK_LAUNCH("k_emit");
  }
  BlendIO io;
  io.sdf_depth = v.sdf_depth;
  io.sdf_color = v.sdf_color;
  io.target = reinterpret_cast<const uint32_t*>(v.target);
  io.out_color = out_color;
  io.out_weight = out_weight;
  io.loss_out = loss_out;
  io.accumulate_loss = accumulate_loss;
  io.counters = counters;
  uint64_t* gk = reinterpret_cast<uint64_t*>(ws + L.keys);
  SplitIO spl{reinterpret_cast<const uint2*>(ws + L.extra), L.extra_cap, reinterpret_cast<const uint32_t*>(ws + L.pbase),
              reinterpret_cast<uint32_t*>(ws + L.tick), reinterpret_cast<float4*>(ws + L.part)};
  if (!c->sort_free && g->n > 0) {
    GPS_PROF(K_SORT_LONG, s);
    if (!sort_long_ready()) return cuda_fail("cudaFuncSetAttribute(k_sort_long)", cudaGetLastError());
    // 3 CTAs of 512 threads per SM (64 KB of keys each): parts of the cfg4 trajectory have
    // hundreds of long lists per view, each a ~55-stage network
    k_sort_long<<<148 * 3, 512, 8 * kLongSmem, s>>>(sp.rec, offsets, vals, gk,
                                                     reinterpret_cast<const uint32_t*>(ws + L.longl), hdr,
                                                     (uint32_t)a.cap);
    GPS_CHECK_LAUNCH("k_sort_long");
  }
  uint32_t* tend = reinterpret_cast<uint32_t*>(ws + L.tile_end);
  float* lp = reinterpret_cast<float*>(ws + L.loss_part);
  {
  GPS_PROF(K_SORT_BLEND, s);
  static const bool one_px = getenv("GPS_BLEND_1PX") != nullptr;  // the one-pixel-per-thread kernel
  static const bool staged = getenv("GPS_BLEND_STAGED") != nullptr;  // the CTA-staged 16x2 loop (A/B)
  if (counters) {  // debug: the instrumented instantiation (16x16 tiles)
    if (c->sort_free)
      k_sort_blend16x2<false, true><<<n_tiles, 128, 0, s>>>(a, sp.rec, offsets, vals, gk, tend, lp, hdr, io, 0, spl);
    else
      k_sort_blend16x2<true, true><<<n_tiles, 128, 0, s>>>(a, sp.rec, offsets, vals, gk, tend, lp, hdr, io,
                                                           c->tile_depth_precull, spl);
  } else if (c->sort_free) {
    if (a.tile == 16 && !one_px)
      k_sort_blend16x2<false><<<n_tiles, 128, 0, s>>>(a, sp.rec, offsets, vals, gk, tend, lp, hdr, io, 0, spl);
    else if (a.tile == 16)
      k_sort_blend<16, false><<<n_tiles, 256, 0, s>>>(a, sp.rec, offsets, vals, gk, tend, lp, hdr, io, 0);
    else
      k_sort_blend<8, false><<<n_tiles, 64, 0, s>>>(a, sp.rec, offsets, vals, gk, tend, lp, hdr, io, 0);
  } else if (a.tile == 16 && !one_px && staged) {
    k_sort_blend16x2<true, false, false><<<n_tiles, 128, 0, s>>>(a, sp.rec, offsets, vals, gk, tend, lp, hdr, io,
                                                                 c->tile_depth_precull, spl);
  } else if (a.tile == 16 && !one_px) {
    k_sort_blend16x2<true><<<n_tiles, 128, 0, s>>>(a, sp.rec, offsets, vals, gk, tend, lp, hdr, io, c->tile_depth_precull,
                                                    spl);
  } else if (a.tile == 16) {
    k_sort_blend<16, true><<<n_tiles, 256, 0, s>>>(a, sp.rec, offsets, vals, gk, tend, lp, hdr, io, c->tile_depth_precull);
  } else {
    k_sort_blend<8, true><<<n_tiles, 64, 0, s>>>(a, sp.rec, offsets, vals, gk, tend, lp, hdr, io, c->tile_depth_precull);
  }
  }
  GPS_CHECK_LAUNCH("k_sort_blend");
  return GPS_OK;
}


// returns GPS_ERR_WORKSPACE_TOO_SMALL (and clears the flag) if an earlier render overflowed
gps_status check_render_overflow(const char* who) {
  OverflowFlag& f = overflow_flag();
  if (!f.host) {
    set_error(std::string(who) + ": could not allocate the host-mapped overflow flag");
    return GPS_ERR_CUDA;
  }
  if (*reinterpret_cast<volatile uint32_t*>(f.host)) {
    *reinterpret_cast<volatile uint32_t*>(f.host) = 0;
    set_error(std::string(who) + ": an earlier render's (tile, Gaussian) pair list exceeded its capacity "
              "(pairs were dropped); raise max_pairs");
    return GPS_ERR_WORKSPACE_TOO_SMALL;
  }
  return GPS_OK;
}

gps_status check_render_cfg(const gps_render_config* c) {
  if (!c) return invalid("null render config");
  if (c->tile != 8 && c->tile != 16) return invalid("render config: tile must be 8 or 16");
  if (!(c->eps_depth >= 0) || !(c->alpha_min >= 0) || !(c->lowpass >= 0)) return invalid("render config: bad value");
  if (c->max_pairs < 0 || c->max_pairs > 0xFFFFFFFFll) return invalid("render config: bad max_pairs");
  if (c->sort_free != 0 && c->sort_free != 1) return invalid("render config: sort_free must be 0 or 1");
  if (c->backward < 0 || c->backward > 2) return invalid("render config: backward must be 0, 1 or 2");
  return GPS_OK;
}

AdamArgs make_adam(const gps_adam_config* c, int64_t step) {
  AdamArgs a;
  const double t = (double)step;
  const double bc1 = 1.0 - std::pow((double)c->beta1, t), bc2 = 1.0 - std::pow((double)c->beta2, t);
  a.b1 = c->beta1; a.b2 = c->beta2; a.eps = c->eps;
  a.step_xyz = (float)(c->lr_xyz / bc1);
  a.step_ls = (float)(c->lr_scale / bc1);
  a.step_rot = (float)(c->lr_rot / bc1);
  a.step_op = (float)(c->lr_opacity / bc1);
  a.step_sh0 = (float)(c->lr_sh0 / bc1);
  a.step_shr = (float)(c->lr_shrest / bc1);
  a.inv_sqrt_bc2 = (float)(1.0 / std::sqrt(bc2));
  return a;
}

gps_status check_adam_state(const gps_gaussians* g, const gps_adam_state* st) {
  if (!st) return invalid("null Adam state");
  if (!same_shape(g, &st->m) || !same_shape(g, &st->v)) return invalid("Adam state shape differs from the parameters");
  gps_status r = check_gaussians(&st->m, "adam m");
  if (r != GPS_OK) return r;
  return check_gaussians(&st->v, "adam v");
}

}  // namespace

extern "C" {

size_t gps_render_workspace_size(int64_t n, const gps_intrinsics* K, const gps_render_config* cfg) {
  if (!valid_K(K) || !cfg || (cfg->tile != 8 && cfg->tile != 16) || n < 0) return 0;
  return ws_layout(n, K->width, K->height, cfg->tile, default_cap(n, cfg->max_pairs), 0, false, false).total;
}

size_t gps_refine_workspace_size(int64_t n, const gps_intrinsics* K, const gps_render_config* cfg, int32_t n_views) {
  if (!valid_K(K) || !cfg || (cfg->tile != 8 && cfg->tile != 16) || n < 0 || n_views < 1) return 0;
  gps_gaussians dummy{};
  dummy.n = n;
  dummy.sh_degree = 3;  // size for the largest degree
  return ws_layout(n, K->width, K->height, cfg->tile, default_cap(n, cfg->max_pairs), gbuf_floats(&dummy), true,
                   n_views > 1)
      .total;
}

gps_status gps_render(const gps_gaussians* g, const gps_intrinsics* K, const gps_pose* T, const float* sdf_depth,
                      const float* sdf_color, const uint8_t* target_rgba, const gps_render_config* cfg, void* ws,
                      size_t ws_bytes, float* out_color, float* out_weight, float* loss_out, gps_stream_t stream) {
  gps_status st = check_gaussians(g, "gps_render");
  if (st != GPS_OK) return st;
  if ((st = check_render_overflow("gps_render")) != GPS_OK) return st;
  if ((st = check_render_cfg(cfg)) != GPS_OK) return st;
  if (!valid_K(K) || !T || !sdf_depth || !sdf_color || !ws || !out_color || !out_weight)
    return invalid("gps_render: null or bad argument");
  if (loss_out && !target_rgba) return invalid("gps_render: loss_out needs target_rgba");
  if (target_rgba && (reinterpret_cast<uintptr_t>(target_rgba) & 3u)) return invalid("gps_render: target must be 4-byte aligned");
  const int64_t cap = default_cap(g->n, cfg->max_pairs);
  const WsLayout L = ws_layout(g->n, K->width, K->height, cfg->tile, cap, 0, false, false);
  if (ws_bytes < L.total) {
    set_error("gps_render: workspace too small");
    return GPS_ERR_WORKSPACE_TOO_SMALL;
  }
  if (!aligned16(ws)) return invalid("gps_render: workspace must be 16-byte aligned");
  View1 v{K, T, sdf_depth, sdf_color, target_rgba};
  return forward_view(g, v, cfg, static_cast<char*>(ws), L, cap, out_color, out_weight, loss_out, 0, false,
                      as_stream(stream));
}

gps_status gps_refine_step(gps_gaussians* g, gps_adam_state* state, const gps_view* views, int32_t n_views,
                           const gps_render_config* rcfg, const gps_adam_config* acfg, void* ws, size_t ws_bytes,
                           float* loss_out, const gps_gaussians* grad_out, gps_stream_t stream) {
  gps_status st = check_gaussians(g, "gps_refine_step");
  if (st != GPS_OK) return st;
  if ((st = check_render_overflow("gps_refine_step")) != GPS_OK) return st;
  if ((st = check_render_cfg(rcfg)) != GPS_OK) return st;
  if ((st = check_adam_state(g, state)) != GPS_OK) return st;
  if (!views || n_views < 1 || !acfg || !ws) return invalid("gps_refine_step: bad argument");
  if (grad_out) {
    if (!same_shape(g, grad_out)) return invalid("gps_refine_step: grad_out shape differs");
    if ((st = check_gaussians(grad_out, "grad_out")) != GPS_OK) return st;
  }
  int maxW = 0, maxH = 0;
  for (int v = 0; v < n_views; ++v) {
    const gps_view& vw = views[v];
    if (!valid_K(&vw.K) || !vw.sdf_depth || !vw.sdf_color || !vw.target_rgba)
      return invalid("gps_refine_step: bad view " + std::to_string(v));
    if (reinterpret_cast<uintptr_t>(vw.target_rgba) & 3u) return invalid("gps_refine_step: target must be 4-byte aligned");
    maxW = std::max(maxW, vw.K.width);
    maxH = std::max(maxH, vw.K.height);
  }
  if (!aligned16(ws)) return invalid("gps_refine_step: workspace must be 16-byte aligned");
  const int64_t cap = default_cap(g->n, rcfg->max_pairs);
  gps_gaussians dummy{};
  dummy.n = g->n;
  dummy.sh_degree = 3;
  const WsLayout L = ws_layout(g->n, maxW, maxH, rcfg->tile, cap, gbuf_floats(&dummy), true, n_views > 1);
  if (ws_bytes < L.total) {
    set_error("gps_refine_step: workspace too small");
    return GPS_ERR_WORKSPACE_TOO_SMALL;
  }
  cudaStream_t s = as_stream(stream);
  char* w = static_cast<char*>(ws);
  WsHeader* hdr = reinterpret_cast<WsHeader*>(w + L.hdr);
  float4* grad2d = reinterpret_cast<float4*>(w + L.grad2d);
  float* cstar = reinterpret_cast<float*>(w + L.cstar);
  float* wg = reinterpret_cast<float*>(w + L.wg);
  gps_gaussians gb = n_views > 1 ? slice_params(g, reinterpret_cast<float*>(w + L.gbuf)) : gps_gaussians{};
  if (n_views > 1)
    GPS_CHECK_CUDA(cudaMemsetAsync(w + L.gbuf, 0, sizeof(float) * gbuf_floats(g), s));
  if (loss_out) GPS_CHECK_CUDA(cudaMemsetAsync(loss_out, 0, sizeof(float), s));
  AdamArgs ad = make_adam(acfg, state->step + 1);
  // GPS_UNFUSED_ADAM=1: k_chain + k_adam instead of k_chain_adam (A/B and the bitwise test)
  const bool fused = n_views == 1 && getenv("GPS_UNFUSED_ADAM") == nullptr;
  for (int v = 0; v < n_views; ++v) {
    const gps_view& vw = views[v];
    View1 v1{&vw.K, &vw.T, vw.sdf_depth, vw.sdf_color, vw.target_rgba};
    st = forward_view(g, v1, rcfg, w, L, cap, cstar, wg, loss_out, 1, true, s);
    if (st != GPS_OK) return st;
    RenderArgs a = make_args(g, &vw.K, &vw.T, rcfg, cap);
    const int n_tiles = a.tiles_x * a.tiles_y;
    const uint32_t* offsets = reinterpret_cast<const uint32_t*>(w + L.offsets);
    const uint32_t* vals = reinterpret_cast<const uint32_t*>(w + L.vals);
    const uint32_t* tend = reinterpret_cast<const uint32_t*>(w + L.tile_end);
    const float4* rec = reinterpret_cast<const float4*>(w + L.records);
    const uint32_t* tgt = reinterpret_cast<const uint32_t*>(vw.target_rgba);
    {
    GPS_PROF(K_BACKWARD, s);
    // sort-free (the paper's renderer, App. B): a thread per (entry, pixel group);
    // sorted (this build's tile design): a warp per entry with a warp reduction
    const bool items = rcfg->backward == 2 || (rcfg->backward == 0 && rcfg->sort_free != 0);
    float* g2 = reinterpret_cast<float*>(grad2d);
    const uint2* xtra = reinterpret_cast<const uint2*>(w + L.extra);
    if (items) {
      if (rcfg->tile == 16)
        k_backward_items<16><<<n_tiles, 256, 0, s>>>(a, rec, offsets, vals, tend, vw.sdf_depth, cstar, wg, tgt, hdr, g2);
      else
        k_backward_items<8><<<n_tiles, 256, 0, s>>>(a, rec, offsets, vals, tend, vw.sdf_depth, cstar, wg, tgt, hdr, g2);
    } else if (rcfg->tile == 16) {
      k_backward<16><<<n_tiles, 256, 0, s>>>(a, rec, offsets, vals, tend, vw.sdf_depth, cstar, wg, tgt, hdr, g2,
                                             xtra, L.extra_cap);
    } else {
      k_backward<8><<<n_tiles, 256, 0, s>>>(a, rec, offsets, vals, tend, vw.sdf_depth, cstar, wg, tgt, hdr, g2,
                                            xtra, L.extra_cap);
    }
    }
    GPS_CHECK_LAUNCH("k_backward");
    if (g->n > 0 && fused) {
      // single view: chain rule and Adam in one kernel (a11), same bits as the two below
      RenderArgs a0 = make_args(g, &views[0].K, &views[0].T, rcfg, cap);
      GPS_PROF(K_CHAIN_ADAM, s);
      k_chain_adam<<<(unsigned)((g->n + kCaG - 1) / kCaG), kCaG, 0, s>>>(
          a0, *g, state->m, state->v, grad2d, reinterpret_cast<const float4*>(w + L.cgj),
          grad_out ? *grad_out : gps_gaussians{}, grad_out != nullptr, ad);
      GPS_CHECK_LAUNCH("k_chain_adam");
    } else if (g->n > 0) {
      const unsigned cgrid = (unsigned)((g->n + kChainThreads - 1) / kChainThreads);
      float4* rec3 = reinterpret_cast<float4*>(w + L.rec3);
      GPS_PROF(K_CHAIN, s);
      const float4* cgj = reinterpret_cast<const float4*>(w + L.cgj);
      if (v < n_views - 1)
        k_chain<1><<<cgrid, kChainThreads, 0, s>>>(a, *g, grad2d, rec3, gb, cgj);
      else
        k_chain<0><<<cgrid, kChainThreads, 0, s>>>(a, *g, grad2d, rec3, gb, cgj);
      GPS_CHECK_LAUNCH("k_chain");
    }
  }
  if (g->n > 0 && !fused) {
    RenderArgs a = make_args(g, &views[0].K, &views[0].T, rcfg, cap);
    AdamSrc src{};
    src.grad2d = grad2d;
    src.rec3 = reinterpret_cast<const float*>(w + L.rec3);
    src.gbuf = gb;
    src.has_gbuf = n_views > 1;
    src.external = 0;
    src.gout = grad_out ? *grad_out : gps_gaussians{};
    src.has_gout = grad_out != nullptr;
    GPS_PROF(K_GRAD_ADAM, s);
    k_adam<<<adam_total_chunks((uint32_t)g->n, 3u * (uint32_t)a.nc), kAdamThreads, 0, s>>>(a, *g, state->m, state->v, src, ad);
    GPS_CHECK_LAUNCH("k_adam");
  }
  state->step += 1;
  return GPS_OK;
}

// gps_refine_round: n_iter gps_refine_step calls in one host call; with use_graph the round's
// launches are captured once per call and replayed as one CUDA graph (the executable graph of
// this workspace is updated in place when the round has the same launch structure as the last)
namespace {
// a ring of executable graphs per workspace: updating a graph whose last launch is still in flight
// can stall the host until that launch completes, so a round updates the graph of three rounds ago
constexpr int kRoundRing = 3;
struct RoundGraph {
  const void* ws;
  cudaGraphExec_t exec[kRoundRing];
  int next;
};
std::mutex g_round_mu;
std::vector<RoundGraph> g_round_graphs;
bool capturing(cudaStream_t s) {  // inside a caller's own capture the launches join that graph
  cudaStreamCaptureStatus c = cudaStreamCaptureStatusNone;
  return cudaStreamIsCapturing(s, &c) != cudaSuccess || c != cudaStreamCaptureStatusNone;
}
}  // namespace

gps_status gps_refine_round(gps_gaussians* g, gps_adam_state* state, const gps_view* views, int32_t n_views,
                            const int32_t* iter_views, int32_t views_per_iter, int32_t n_iter,
                            const gps_render_config* rcfg, const gps_adam_config* acfg, void* ws, size_t ws_bytes,
                            float* loss_out, int32_t use_graph, gps_stream_t stream) {
  if (!g || !state || !views || n_views < 1 || !iter_views || views_per_iter < 1 || n_iter < 0)
    return invalid("gps_refine_round: bad argument");
  for (int64_t i = 0; i < (int64_t)n_iter * views_per_iter; ++i)
    if (iter_views[i] < 0 || iter_views[i] >= n_views) return invalid("gps_refine_round: view index out of range");
  if (n_iter == 0) return GPS_OK;
  cudaStream_t s = as_stream(stream);
  // capture needs a created stream; the event profiler's per-launch events stay outside graphs
  const bool graph = use_graph != 0 && s != nullptr && s != cudaStreamLegacy && s != cudaStreamPerThread && !g_prof_on &&
                     !capturing(s);
  std::vector<gps_view> sel(views_per_iter);
  const int64_t step0 = state->step;
  if (graph) {
    // the once-per-process setup (host-mapped flag allocation, kernel attributes) must not run
    // inside a capture
    if (!overflow_flag().host) return check_render_overflow("gps_refine_round");
    if (!sort_long_ready()) return cuda_fail("cudaFuncSetAttribute(k_sort_long)", cudaGetLastError());
    GPS_CHECK_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
  }
  gps_status st = GPS_OK;
  for (int32_t i = 0; i < n_iter && st == GPS_OK; ++i) {
    for (int32_t j = 0; j < views_per_iter; ++j) sel[j] = views[iter_views[(int64_t)i * views_per_iter + j]];
    st = gps_refine_step(g, state, sel.data(), views_per_iter, rcfg, acfg, ws, ws_bytes, loss_out, nullptr, stream);
  }
  if (!graph) return st;
  cudaGraph_t gr = nullptr;
  const cudaError_t ec = cudaStreamEndCapture(s, &gr);
  if (st != GPS_OK || ec != cudaSuccess) {  // nothing was launched
    if (gr) cudaGraphDestroy(gr);
    cudaGetLastError();
    state->step = step0;
    return st != GPS_OK ? st : cuda_fail("cudaStreamEndCapture", ec);
  }
  std::lock_guard<std::mutex> lock(g_round_mu);
  RoundGraph* rg = nullptr;
  for (RoundGraph& r : g_round_graphs)
    if (r.ws == ws) rg = &r;
  if (!rg) {
    g_round_graphs.push_back(RoundGraph{ws, {}, 0});
    rg = &g_round_graphs.back();
  }
  cudaGraphExec_t& exec = rg->exec[rg->next];
  rg->next = (rg->next + 1) % kRoundRing;
  if (exec) {
    // same topology (same n_iter, views per iteration, configuration): parameters updated in
    // place for future launches; else a new executable graph (an in-flight one is freed on completion)
    cudaGraphExecUpdateResultInfo info;
    if (cudaGraphExecUpdate(exec, gr, &info) != cudaSuccess) {
      cudaGetLastError();
      cudaGraphExecDestroy(exec);
      exec = nullptr;
    }
  }
  cudaError_t e = cudaSuccess;
  static const bool verbose = getenv("GPS_GRAPH_VERBOSE") != nullptr;
  if (!exec) {
    e = cudaGraphInstantiate(&exec, gr, 0);
    if (verbose) fprintf(stderr, "gps_refine_round: instantiated a graph of %d iterations (ws %p)\n", n_iter, ws);
  }
  cudaGraphDestroy(gr);
  if (e != cudaSuccess) {
    exec = nullptr;
    state->step = step0;
    return cuda_fail("cudaGraphInstantiate", e);
  }
  // the graph's kernels run at the priority of the stream it is launched into
  e = cudaGraphLaunch(exec, s);
  if (e != cudaSuccess) {
    state->step = step0;
    return cuda_fail("cudaGraphLaunch", e);
  }
  return GPS_OK;
}

gps_status gps_adam_step(gps_gaussians* g, gps_adam_state* state, const gps_gaussians* grad,
                         const gps_adam_config* acfg, gps_stream_t stream) {
  gps_status st = check_gaussians(g, "gps_adam_step");
  if (st != GPS_OK) return st;
  if ((st = check_adam_state(g, state)) != GPS_OK) return st;
  if (!grad || !acfg || !same_shape(g, grad)) return invalid("gps_adam_step: bad gradient argument");
  if ((st = check_gaussians(grad, "grad")) != GPS_OK) return st;
  AdamArgs ad = make_adam(acfg, state->step + 1);
  RenderArgs a{};
  a.n = g->n;
  a.deg = g->sh_degree;
  a.nc = (g->sh_degree + 1) * (g->sh_degree + 1);
  if (g->n > 0) {
    AdamSrc src{};
    src.gbuf = *grad;
    src.external = 1;
    GPS_PROF(K_GRAD_ADAM, as_stream(stream));
    k_adam<<<adam_total_chunks((uint32_t)g->n, 3u * (uint32_t)a.nc), kAdamThreads, 0, as_stream(stream)>>>(a, *g, state->m, state->v, src, ad);
    GPS_CHECK_LAUNCH("k_adam");
  }
  state->step += 1;
  return GPS_OK;
}

gps_status gps_render_stats_sync(const void* ws, gps_stream_t stream, int64_t* n_pairs, int64_t* capacity,
                                 int64_t* n_visible) {
  if (!ws) return invalid("gps_render_stats_sync: null workspace");
  WsHeader h;
  GPS_CHECK_CUDA(cudaMemcpyAsync(&h, ws, sizeof(h), cudaMemcpyDeviceToHost, as_stream(stream)));
  GPS_CHECK_CUDA(cudaStreamSynchronize(as_stream(stream)));
  if (h.magic != kWsMagic) return invalid("gps_render_stats_sync: workspace holds no render");
  if (n_pairs) *n_pairs = h.K;
  if (capacity) *capacity = (int64_t)h.cap_pairs;
  if (n_visible) *n_visible = h.n_visible;
  const gps_status sticky = check_render_overflow("gps_render_stats_sync");
  if (h.overflow) {
    set_error("render pair list overflow: " + std::to_string(h.K) + " pairs > capacity " + std::to_string(h.cap_pairs));
    return GPS_ERR_WORKSPACE_TOO_SMALL;
  }
  return sticky;
}

gps_status gps_debug_render_counts_sync(const gps_gaussians* g, const gps_intrinsics* K, const gps_pose* T,
                                        const float* sdf_depth, const float* sdf_color, const gps_render_config* cfg,
                                        void* ws, size_t ws_bytes, int64_t* evaluated, int64_t* accepted,
                                        gps_stream_t stream) {
  gps_status st = check_gaussians(g, "gps_debug_render_counts_sync");
  if (st != GPS_OK) return st;
  if ((st = check_render_cfg(cfg)) != GPS_OK) return st;
  if (!valid_K(K) || !T || !sdf_depth || !sdf_color || !ws || !evaluated || !accepted || cfg->tile != 16)
    return invalid("gps_debug_render_counts_sync: bad argument (16x16 tiles only)");
  const int64_t cap = default_cap(g->n, cfg->max_pairs);
  const WsLayout L = ws_layout(g->n, K->width, K->height, cfg->tile, cap, 0, false, false);
  if (ws_bytes < L.total) return invalid("gps_debug_render_counts_sync: workspace too small");
  cudaStream_t s = as_stream(stream);
  unsigned long long* cnt = nullptr;
  float *oc = nullptr, *ow = nullptr;
  const size_t px = (size_t)K->width * K->height;
  GPS_CHECK_CUDA(cudaMallocAsync(&cnt, 16, s));
  GPS_CHECK_CUDA(cudaMallocAsync(&oc, 12 * px, s));
  GPS_CHECK_CUDA(cudaMallocAsync(&ow, 4 * px, s));
  GPS_CHECK_CUDA(cudaMemsetAsync(cnt, 0, 16, s));
  View1 v{K, T, sdf_depth, sdf_color, nullptr};
  st = forward_view(g, v, cfg, static_cast<char*>(ws), L, cap, oc, ow, nullptr, 0, false, s, cnt);
  if (st != GPS_OK) return st;
  unsigned long long h[2] = {0, 0};
  GPS_CHECK_CUDA(cudaMemcpyAsync(h, cnt, 16, cudaMemcpyDeviceToHost, s));
  GPS_CHECK_CUDA(cudaFreeAsync(cnt, s));
  GPS_CHECK_CUDA(cudaFreeAsync(oc, s));
  GPS_CHECK_CUDA(cudaFreeAsync(ow, s));
  GPS_CHECK_CUDA(cudaStreamSynchronize(s));
  *evaluated = (int64_t)h[0];
  *accepted = (int64_t)h[1];
  return GPS_OK;
}

gps_status gps_debug_render_lists_sync(const void* ws, gps_stream_t stream, uint32_t* values, int64_t cap,
                                       uint32_t* ranges, int64_t* K) {
  if (!ws || !K) return invalid("gps_debug_render_lists_sync: null argument");
  cudaStream_t s = as_stream(stream);
  WsHeader h;
  GPS_CHECK_CUDA(cudaMemcpyAsync(&h, ws, sizeof(h), cudaMemcpyDeviceToHost, s));
  GPS_CHECK_CUDA(cudaStreamSynchronize(s));
  if (h.magic != kWsMagic) return invalid("gps_debug_render_lists_sync: workspace holds no render");
  const char* w = static_cast<const char*>(ws);
  *K = h.K;
  if (values) {
    const int64_t cnt = std::min<int64_t>({cap, (int64_t)h.K, (int64_t)h.cap_pairs});
    GPS_CHECK_CUDA(cudaMemcpyAsync(values, w + h.off_vals, 4 * cnt, cudaMemcpyDeviceToDevice, s));
  }
  if (ranges) {
    // ranges[2t] = offsets[t], ranges[2t+1] = tile_end[t]
    std::vector<uint32_t> off(h.n_tiles + 1), te(h.n_tiles);
    GPS_CHECK_CUDA(cudaMemcpyAsync(off.data(), w + h.off_offsets, 4 * (h.n_tiles + 1), cudaMemcpyDeviceToHost, s));
    GPS_CHECK_CUDA(cudaMemcpyAsync(te.data(), w + h.off_tile_end, 4 * h.n_tiles, cudaMemcpyDeviceToHost, s));
    GPS_CHECK_CUDA(cudaStreamSynchronize(s));
    std::vector<uint32_t> r(2 * h.n_tiles);
    for (uint32_t t = 0; t < h.n_tiles; ++t) {
      r[2 * t] = off[t];
      r[2 * t + 1] = te[t];
    }
    GPS_CHECK_CUDA(cudaMemcpyAsync(ranges, r.data(), 4 * r.size(), cudaMemcpyHostToDevice, s));
  }
  GPS_CHECK_CUDA(cudaStreamSynchronize(s));
  return GPS_OK;
}

}  // extern "C"
