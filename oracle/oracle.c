/*
 * oracle.c -- TEST INFRASTRUCTURE ONLY.  A plain, slow, obviously-correct CPU implementation
 * of the Gaussian-Plus-SDF mapping step of GPS-SLAM (arXiv 2509.11574), written from the
 * paper (PAPER.md, cited "P:line") and the readings listed in DESIGN.md §3 (R-*).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may load this library.
 * It shares no code, header, table or constant generator with the CUDA path
 * (paper_2509_11574_b200/csrc, include/gps.h) and never reads anything the CUDA path produced.
 *
 * Build: gcc -O2 -ffp-contract=off -fno-fast-math -shared -fPIC (see oracle/build.py).
 * -ffp-contract=off matters: the P32 stages below are "prescribed fp32" sequences that must be
 * evaluated exactly as written (IEEE single, round-to-nearest, no FMA contraction, correctly
 * rounded / and sqrtf) -- DESIGN.md §4.
 *
 * Two precision regimes:
 *   P32 -- stages whose outputs are integers or must be bit-exact: allocation (block coords),
 *          integration (tsdf, pixel choice; colour/weight are integer), and the Gaussian
 *          projection fields that decide tile membership and sort keys (rect, depth).
 *   F64 -- everything continuous: raycast, projection for blending, Eqs. 1-4, the L1 loss and
 *          its exact gradient.  (Adam lives in oracle/__init__.py, numpy fp64.)
 *
 * Parity pins: see tests/test_oracle_*.py.  Functions without an external pin are marked
 * "parity unpinned" here and in DESIGN.md (there are none at present).
 */
#include <math.h>
#include <stdint.h>
#ifdef _OPENMP
#include <omp.h>
#endif
#include <stdlib.h>
#include <string.h>

/* ======================================================================================= */
/* Volume: a sorted array of allocated blocks (lexicographic (x,y,z)), each with 512 voxels. */
/* Lookups are binary searches: slow but obviously correct.                                 */
/* ======================================================================================= */

typedef struct {
  float voxel, mu, dmin, dmax;
  int wmax;
  int64_t budget;
  int64_t n, cap;
  int32_t* coords; /* n*3 */
  float* tsdf;     /* n*512 */
  uint8_t* rgbw;   /* n*512*4 : r,g,b,w */
  int overflow;
  int64_t nvis;
  int32_t* vis; /* nvis*3 sorted */
} orc_volume;

static int cmp3(const int32_t* a, const int32_t* b) {
  for (int k = 0; k < 3; ++k) {
    if (a[k] < b[k]) return -1;
    if (a[k] > b[k]) return 1;
  }
  return 0;
}
static int cmp3_qsort(const void* a, const void* b) { return cmp3((const int32_t*)a, (const int32_t*)b); }

orc_volume* orc_volume_new(float voxel, float mu, int wmax, float dmin, float dmax, int64_t budget) {
  orc_volume* v = (orc_volume*)calloc(1, sizeof(orc_volume));
  v->voxel = voxel;
  v->mu = mu;
  v->wmax = wmax;
  v->dmin = dmin;
  v->dmax = dmax;
  v->budget = budget;
  return v;
}

void orc_volume_free(orc_volume* v) {
  if (!v) return;
  free(v->coords);
  free(v->tsdf);
  free(v->rgbw);
  free(v->vis);
  free(v);
}

int64_t orc_volume_n(const orc_volume* v) { return v->n; }
int64_t orc_volume_nvis(const orc_volume* v) { return v->nvis; }
int orc_volume_overflow(const orc_volume* v) { return v->overflow; }

/* Copies the allocated blocks in sorted order. Any output may be NULL. */
void orc_volume_export(const orc_volume* v, int32_t* coords, float* tsdf, uint8_t* rgbw) {
  if (coords) memcpy(coords, v->coords, sizeof(int32_t) * 3 * v->n);
  if (tsdf) memcpy(tsdf, v->tsdf, sizeof(float) * 512 * v->n);
  if (rgbw) memcpy(rgbw, v->rgbw, 4 * 512 * v->n);
}
void orc_volume_export_visible(const orc_volume* v, int32_t* coords) {
  memcpy(coords, v->vis, sizeof(int32_t) * 3 * v->nvis);
}

static int64_t find_block(const orc_volume* v, const int32_t* c) {
  int64_t lo = 0, hi = v->n - 1;
  while (lo <= hi) {
    int64_t mid = (lo + hi) / 2;
    int r = cmp3(v->coords + 3 * mid, c);
    if (r == 0) return mid;
    if (r < 0) lo = mid + 1;
    else hi = mid - 1;
  }
  return -1;
}

/* floor division for block coordinates of integer voxel indices */
static int32_t fdiv8(int32_t g) { return (int32_t)floor((double)g / 8.0); }

/* ---- O2 allocation ("Following InfiniTAM ... global hash table"; reading R-BAND) ----
 * P32 prescribed sequence: 5 equispaced band samples; the blocks are those of
 * the axis-aligned boxes spanned by consecutive samples' blocks (samples are <= 1/4 block
 * apart, so this contains every block the band segment meets).  Returns the count written
 * (with repeats).                                                                          */
static int64_t band_blocks(const float* K4, int W, int H, const float* R, const float* t,
                           const uint16_t* depth, float scale, float mu, float voxel,
                           float dmin, float dmax, int32_t* out /* W*H*32*3 */) {
  int64_t m = 0;
  float bs = 8.0f * voxel;
  float inv_scale = 1.0f / scale;
  float fx = K4[0], fy = K4[1], cx = K4[2], cy = K4[3];
  for (int v = 0; v < H; ++v) {
    for (int u = 0; u < W; ++u) {
      float d = (float)depth[(int64_t)v * W + u] * inv_scale;
      if (!(d >= dmin && d <= dmax)) continue;
      float xn = ((float)u - cx) / fx;
      float yn = ((float)v - cy) / fy;
      float X[3] = {xn * d, yn * d, d};
      float n2 = X[0] * X[0] + X[1] * X[1];
      n2 = n2 + X[2] * X[2];
      float n = sqrtf(n2);
      float q = mu / n;
      float a = 1.0f - q, b = 1.0f + q;
      float A[3], B[3];
      for (int k = 0; k < 3; ++k) {
        A[k] = X[k] * a;
        B[k] = X[k] * b;
      }
      int32_t blk[5][3];
      for (int s = 0; s < 5; ++s) {
        float f = (float)s * 0.25f;
        float Q[3];
        for (int k = 0; k < 3; ++k) {
          float diff = B[k] - A[k];
          float step = diff * f;
          Q[k] = A[k] + step;
        }
        for (int r = 0; r < 3; ++r) {
          float acc = R[3 * r + 0] * Q[0];
          float p1 = R[3 * r + 1] * Q[1];
          acc = acc + p1;
          float p2 = R[3 * r + 2] * Q[2];
          acc = acc + p2;
          float Wr = acc + t[r];
          blk[s][r] = (int32_t)floorf(Wr / bs);
        }
      }
      /* every block of the axis-aligned box spanned by consecutive samples' blocks */
      for (int s = 0; s < 4; ++s) {
        int32_t lo[3], hi[3];
        for (int r = 0; r < 3; ++r) {
          lo[r] = blk[s][r] < blk[s + 1][r] ? blk[s][r] : blk[s + 1][r];
          hi[r] = blk[s][r] < blk[s + 1][r] ? blk[s + 1][r] : blk[s][r];
        }
        for (int32_t z = lo[2]; z <= hi[2]; ++z)
          for (int32_t y = lo[1]; y <= hi[1]; ++y)
            for (int32_t x = lo[0]; x <= hi[0]; ++x) {
              out[3 * m] = x;
              out[3 * m + 1] = y;
              out[3 * m + 2] = z;
              ++m;
            }
      }
    }
  }
  return m;
}

/* Insert sorted unique list `add` (na) into the volume's sorted block list. */
static void merge_blocks(orc_volume* v, const int32_t* add, int64_t na) {
  int64_t nn = 0;
  int32_t* nc = (int32_t*)malloc(sizeof(int32_t) * 3 * (v->n + na + 1));
  float* nt = (float*)malloc(sizeof(float) * 512 * (v->n + na + 1));
  uint8_t* nr = (uint8_t*)malloc(4 * 512 * (v->n + na + 1));
  int64_t i = 0, j = 0;
  while (i < v->n || j < na) {
    int take_old;
    if (i >= v->n) take_old = 0;
    else if (j >= na) take_old = 1;
    else {
      int r = cmp3(v->coords + 3 * i, add + 3 * j);
      if (r == 0) { ++j; continue; } /* already allocated */
      take_old = r < 0;
    }
    if (take_old) {
      memcpy(nc + 3 * nn, v->coords + 3 * i, 12);
      memcpy(nt + 512 * nn, v->tsdf + 512 * i, 2048);
      memcpy(nr + 2048 * nn, v->rgbw + 2048 * i, 2048);
      ++i;
    } else {
      memcpy(nc + 3 * nn, add + 3 * j, 12);
      for (int k = 0; k < 512; ++k) nt[512 * nn + k] = 1.0f; /* new block: tsdf 1, rgb 0, w 0 */
      memset(nr + 2048 * nn, 0, 2048);
      ++j;
    }
    ++nn;
  }
  free(v->coords);
  free(v->tsdf);
  free(v->rgbw);
  v->coords = nc;
  v->tsdf = nt;
  v->rgbw = nr;
  v->n = nn;
}

/* ---- O3 integration (reading R-INT), P32 prescribed, DESIGN.md §4.2 ---------- */
/* The world->camera map of a voxel as one affine map of its integer index g (R-POSE: X = R^T
 * (g v - t)), scaled by the focal lengths: (fx X, fy Y, Z) = A g + b.  Its coefficients are
 * computed in double from the fp32 inputs and rounded once to fp32:
 *   A[c][k] = fl((s_c * v) * R[k][c]),   b[c] = fl(-(s_c * ((R[0][c] t0 + R[1][c] t1) + R[2][c] t2))),
 * s = (fx, fy, 1); each coordinate is then fmaf(A[c][2], gz, fmaf(A[c][1], gy, fmaf(A[c][0], gx, b[c]))). */
static void affine_cam(const float* K4, const float* R, const float* t, float voxel, float A[3][3], float b[3]) {
  const double sc[3] = {(double)K4[0], (double)K4[1], 1.0};
  for (int c = 0; c < 3; ++c) {
    const double sv = sc[c] * (double)voxel;
    for (int k = 0; k < 3; ++k) A[c][k] = (float)(sv * (double)R[3 * k + c]);
    double acc = (double)R[c] * (double)t[0];
    acc = acc + (double)R[3 + c] * (double)t[1];
    acc = acc + (double)R[6 + c] * (double)t[2];
    b[c] = (float)(-(sc[c] * acc));
  }
}

static void integrate_block(orc_volume* v, int64_t bi, const float* K4, int W, int H,
                            const float* R, const float* t, const uint16_t* depth, float scale,
                            const uint8_t* rgba) {
  const int32_t* bc = v->coords + 3 * bi;
  float cx = K4[2], cy = K4[3];
  float inv_scale = 1.0f / scale, inv_mu = 1.0f / v->mu;
  float A[3][3], b[3];
  affine_cam(K4, R, t, v->voxel, A, b);
  for (int k = 0; k < 8; ++k)
    for (int j = 0; j < 8; ++j)
      for (int i = 0; i < 8; ++i) {
        int32_t g[3] = {bc[0] * 8 + i, bc[1] * 8 + j, bc[2] * 8 + k};
        float X[3]; /* (fx X_c, fy Y_c, Z_c) */
        for (int c = 0; c < 3; ++c)
          X[c] = fmaf(A[c][2], (float)g[2], fmaf(A[c][1], (float)g[1], fmaf(A[c][0], (float)g[0], b[c])));
        if (!(X[2] > 0.0f)) continue;
        float iz = 1.0f / X[2];
        float uf = fmaf(X[0], iz, cx);
        float vf = fmaf(X[1], iz, cy);
        float ur = floorf(uf + 0.5f), vr = floorf(vf + 0.5f);
        if (!(ur >= 0.0f && ur <= (float)(W - 1) && vr >= 0.0f && vr <= (float)(H - 1))) continue;
        int64_t pix = (int64_t)vr * W + (int64_t)ur;
        float d = (float)depth[pix] * inv_scale;
        if (!(d >= v->dmin && d <= v->dmax)) continue;
        float eta = d - X[2];
        if (eta < -v->mu) continue;
        float s = eta * inv_mu;
        if (s > 1.0f) s = 1.0f;
        int idx = i + 8 * j + 64 * k;
        float* ts = v->tsdf + 512 * bi + idx;
        uint8_t* cw = v->rgbw + 2048 * bi + 4 * idx;
        int w = cw[3];
        float wf = (float)w;
        float num = (*ts) * wf;
        num = num + s;
        float den = wf + 1.0f;
        float rden = 1.0f / den;
        *ts = num * rden;
        for (int c = 0; c < 3; ++c) { /* exact rational mean, round half up (R-INT) */
          int x8 = rgba[4 * pix + c];
          cw[c] = (uint8_t)((cw[c] * w + x8 + (w + 1) / 2) / (w + 1));
        }
        cw[3] = (uint8_t)(w + 1 < v->wmax ? w + 1 : v->wmax);
      }
}

/* gps_fuse equivalent.  K4 = {fx,fy,cx,cy}.  Returns 0, or 2 if the budget is exceeded (the
 * oracle then still integrates everything; parity is only defined without overflow).      */
int orc_fuse(orc_volume* v, const float* K4, int W, int H, const float* R, const float* t,
             const uint16_t* depth, float scale, const uint8_t* rgba) {
  int32_t* samples = (int32_t*)malloc(sizeof(int32_t) * 3 * ((int64_t)W * H * 32 + 1));
  int64_t m = band_blocks(K4, W, H, R, t, depth, scale, v->mu, v->voxel, v->dmin, v->dmax, samples);
  qsort(samples, (size_t)m, 12, cmp3_qsort);
  int64_t u = 0;
  for (int64_t i = 0; i < m; ++i)
    if (u == 0 || cmp3(samples + 3 * (u - 1), samples + 3 * i) != 0) {
      memmove(samples + 3 * u, samples + 3 * i, 12);
      ++u;
    }
  free(v->vis);
  v->vis = (int32_t*)malloc(sizeof(int32_t) * 3 * (u + 1));
  memcpy(v->vis, samples, 12 * u);
  v->nvis = u;
  merge_blocks(v, samples, u);
  free(samples);
  if (v->n > v->budget) v->overflow = 1;
  /* blocks are disjoint: the OpenMP build (timing baseline only) integrates them in parallel */
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t i = 0; i < v->nvis; ++i) {
    int64_t bi = find_block(v, v->vis + 3 * i);
    integrate_block(v, bi, K4, W, H, R, t, depth, scale, rgba);
  }
  return v->overflow ? 2 : 0;
}

/* ---- O4 raycast (reading R-RAY), F64 ----------------------------------------- */

/* Trilinear sample at world point P (metres).  Valid iff all 8 corners are allocated with
 * w > 0 (R-RAY).  Returns validity; writes tsdf, (if col) colour in [0,255] and (if grad) the
 * trilinear gradient in tsdf units per voxel (test diagnostics only).                       */
static int tri_sample_g(const orc_volume* v, const double P[3], double* f, double col[3], double grad[3]) {
  double vs = (double)v->voxel;
  double p[3], fr[3];
  int32_t base[3];
  for (int c = 0; c < 3; ++c) {
    p[c] = P[c] / vs;
    double b = floor(p[c]);
    base[c] = (int32_t)b;
    fr[c] = p[c] - b;
  }
  double acc = 0.0, acol[3] = {0, 0, 0}, ag[3] = {0, 0, 0};
  for (int corner = 0; corner < 8; ++corner) {
    int dx = corner & 1, dy = (corner >> 1) & 1, dz = (corner >> 2) & 1;
    int32_t g[3] = {base[0] + dx, base[1] + dy, base[2] + dz};
    int32_t b[3] = {fdiv8(g[0]), fdiv8(g[1]), fdiv8(g[2])};
    int64_t bi = find_block(v, b);
    if (bi < 0) return 0;
    int idx = (g[0] - 8 * b[0]) + 8 * (g[1] - 8 * b[1]) + 64 * (g[2] - 8 * b[2]);
    const uint8_t* cw = v->rgbw + 2048 * bi + 4 * idx;
    if (cw[3] == 0) return 0;
    double wx = dx ? fr[0] : 1.0 - fr[0], wy = dy ? fr[1] : 1.0 - fr[1], wz = dz ? fr[2] : 1.0 - fr[2];
    double wgt = wx * wy * wz;
    double val = (double)v->tsdf[512 * bi + idx];
    acc += wgt * val;
    ag[0] += (dx ? 1.0 : -1.0) * wy * wz * val;
    ag[1] += (dy ? 1.0 : -1.0) * wx * wz * val;
    ag[2] += (dz ? 1.0 : -1.0) * wx * wy * val;
    if (col)
      for (int c = 0; c < 3; ++c) acol[c] += wgt * (double)cw[c];
  }
  *f = acc;
  if (col)
    for (int c = 0; c < 3; ++c) col[c] = acol[c];
  if (grad)
    for (int c = 0; c < 3; ++c) grad[c] = ag[c];
  return 1;
}
static int tri_sample(const orc_volume* v, const double P[3], double* f, double col[3]) {
  return tri_sample_g(v, P, f, col, NULL);
}

/* Decision margin of one sample, in voxel units of position (test diagnostics only): how far
 * the sample point may move before a decision the march takes on it can change.  (i) sign:
 * |f| / |grad f|_1 for a valid sample; (ii) validity: the distance to a cell face across which
 * the validity differs (the 8-corner set changes there).  An implementation that evaluates the
 * sample position with an error below the margin takes the same decisions.                  */
static double sample_margin(const orc_volume* v, const double P[3], int valid, double f, const double g[3]) {
  double m = INFINITY;
  if (valid) {
    double gl1 = fabs(g[0]) + fabs(g[1]) + fabs(g[2]);
    m = fabs(f) == 0.0 ? 0.0 : (gl1 > 0.0 ? fabs(f) / gl1 : INFINITY);
  }
  double vs = (double)v->voxel;
  for (int a = 0; a < 3; ++a) {
    double pa = P[a] / vs, fa = pa - floor(pa);
    double dist = fa < 0.5 ? fa : 1.0 - fa;
    if (dist >= 0.05 || dist >= m) continue;
    double Q[3] = {P[0], P[1], P[2]};
    Q[a] = (fa < 0.5 ? floor(pa) - 1e-7 : floor(pa) + 1.0 + 1e-7) * vs; /* just across the face */
    double fq;
    if (tri_sample(v, Q, &fq, NULL) != valid) m = dist;
  }
  return m;
}

/* Raycast the listed pixels (pix = n*2 (u,v) pairs; NULL = all pixels in row-major order).
 * Outputs per listed pixel: depth (0 = miss), color (3, in [0,1]), vertex (3, nullable),
 * and `margin` (nullable): the smallest sample_margin (voxel units of position) over the
 * samples the march evaluated and the colour sample at V*, used by the tests to recognise
 * rays where an fp32 evaluation may legitimately decide differently.                        */
void orc_raycast(const orc_volume* v, const float* K4, int W, int H, const float* Rf,
                 const float* tf, const int32_t* pix, int64_t n, double* depth, double* color,
                 double* vertex, double* margin) {
  double fx = K4[0], fy = K4[1], cx = K4[2], cy = K4[3];
  double R[9], t[3];
  for (int k = 0; k < 9; ++k) R[k] = Rf[k];
  for (int k = 0; k < 3; ++k) t[k] = tf[k];
  double vs = (double)v->voxel, tmin = (double)v->dmin;
  int64_t J = (int64_t)floor(((double)v->dmax - (double)v->dmin) / vs);
  int64_t count = pix ? n : (int64_t)W * H;
#pragma omp parallel for schedule(dynamic, 64)
  for (int64_t q = 0; q < count; ++q) {
    int u = pix ? pix[2 * q] : (int)(q % W);
    int vv = pix ? pix[2 * q + 1] : (int)(q / W);
    double dc[3] = {((double)u - cx) / fx, ((double)vv - cy) / fy, 1.0};
    double nrm = sqrt(dc[0] * dc[0] + dc[1] * dc[1] + dc[2] * dc[2]);
    double dh[3] = {dc[0] / nrm, dc[1] / nrm, dc[2] / nrm};
    double r[3];
    for (int a = 0; a < 3; ++a) r[a] = R[3 * a] * dh[0] + R[3 * a + 1] * dh[1] + R[3 * a + 2] * dh[2];
    int prev_valid = 0, hit = 0;
    double prev_f = 0.0, tstar = 0.0, mg = INFINITY;
    for (int64_t j = 0; j <= J; ++j) {
      double tj = tmin + (double)j * vs;
      double P[3] = {t[0] + tj * r[0], t[1] + tj * r[1], t[2] + tj * r[2]};
      double f, g[3];
      int valid = tri_sample_g(v, P, &f, NULL, g);
      if (margin) {
        double ms = sample_margin(v, P, valid, f, g);
        if (ms < mg) mg = ms;
      }
      if (j >= 1 && valid && f <= 0.0) {
        if (prev_valid && prev_f > 0.0) {
          tstar = (tmin + (double)(j - 1) * vs) + vs * prev_f / (prev_f - f);
          hit = 1;
        }
        break;
      }
      prev_valid = valid;
      prev_f = f;
    }
    double col[3] = {0, 0, 0}, V[3] = {0, 0, 0}, D = 0.0;
    if (hit) {
      for (int a = 0; a < 3; ++a) V[a] = t[a] + tstar * r[a];
      double fdummy, gd[3];
      int cv = tri_sample_g(v, V, &fdummy, col, gd);
      if (margin) {
        double ms = sample_margin(v, V, cv, INFINITY, gd); /* validity of the colour sample only */
        if (ms < mg) mg = ms;
      }
      if (cv) {
        D = tstar / nrm; /* camera z of V*: t* times the z component of the unit ray */
        for (int a = 0; a < 3; ++a) col[a] /= 255.0;
      } else {
        hit = 0;
      }
    }
    if (!hit) {
      D = 0.0;
      for (int a = 0; a < 3; ++a) col[a] = V[a] = 0.0;
    }
    depth[q] = D;
    for (int a = 0; a < 3; ++a) color[3 * q + a] = col[a];
    if (vertex)
      for (int a = 0; a < 3; ++a) vertex[3 * q + a] = V[a];
    if (margin) margin[q] = mg;
  }
}

/* ======================================================================================= */
/* Gaussians                                                                                */
/* ======================================================================================= */

/* ---- P32 projection fields that decide tile membership, sort keys and pair membership ----
 * (DESIGN.md §4.3).  Follows 3DGS's EWA projection ("following 3DGS", P:89 Sigma_2D) in
 * the prescribed fp32 evaluation order.  exp/log are evaluated in double and rounded once.
 * Per Gaussian: culled flag, depth d = camera z, p_hat, conic (a, b, c), ln(sigma), and the
 * inclusive pixel rect of the 3-sigma ellipse clipped to the image.                          */
typedef struct {
  int culled;
  float d, px, py, a, b, c, lnsig;
  int32_t rect[4];
} p32;

static void proj32(const float* p, const float* ls, const float* q, float o, const float* K4, int W,
                   int H, const float* R, const float* t, float near_z, float lowpass, p32* g) {
  float fx = K4[0], fy = K4[1], cx = K4[2], cy = K4[3];
  float tanx = (float)W / (2.0f * fx), tany = (float)H / (2.0f * fy);
  float limx = 1.3f * tanx, limy = 1.3f * tany;
  memset(g, 0, sizeof(*g));
  g->culled = 1;
  g->rect[2] = g->rect[3] = -1;
  float D[3], X[3];
  for (int c = 0; c < 3; ++c) D[c] = p[c] - t[c];
  for (int c = 0; c < 3; ++c) {
    float acc = R[0 * 3 + c] * D[0];
    float p1 = R[1 * 3 + c] * D[1];
    acc = acc + p1;
    float p2 = R[2 * 3 + c] * D[2];
    X[c] = acc + p2;
  }
  g->d = X[2];
  if (!(X[2] > near_z)) return;
  float s[3];
  for (int c = 0; c < 3; ++c) s[c] = (float)exp((double)ls[c]);
  float qw = q[0], qx = q[1], qy = q[2], qz = q[3];
  float qn2 = qw * qw + qx * qx;
  qn2 = qn2 + qy * qy;
  qn2 = qn2 + qz * qz;
  float qn = sqrtf(qn2);
  float w = qw / qn, x = qx / qn, y = qy / qn, z = qz / qn;
  float Rq[9];
  Rq[0] = 1.0f - 2.0f * (y * y + z * z);
  Rq[1] = 2.0f * (x * y - w * z);
  Rq[2] = 2.0f * (x * z + w * y);
  Rq[3] = 2.0f * (x * y + w * z);
  Rq[4] = 1.0f - 2.0f * (x * x + z * z);
  Rq[5] = 2.0f * (y * z - w * x);
  Rq[6] = 2.0f * (x * z - w * y);
  Rq[7] = 2.0f * (y * z + w * x);
  Rq[8] = 1.0f - 2.0f * (x * x + y * y);
  float M[9];
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) M[3 * r + c] = Rq[3 * r + c] * s[c];
  float S[9];
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) {
      float acc = M[3 * r + 0] * M[3 * c + 0];
      float p1 = M[3 * r + 1] * M[3 * c + 1];
      acc = acc + p1;
      float p2 = M[3 * r + 2] * M[3 * c + 2];
      S[3 * r + c] = acc + p2;
    }
  float txz = X[0] / X[2], tyz = X[1] / X[2];
  float cu = txz < -limx ? -limx : (txz > limx ? limx : txz);
  float cv = tyz < -limy ? -limy : (tyz > limy ? limy : tyz);
  float tx = cu * X[2], ty = cv * X[2];
  float z2 = X[2] * X[2];
  float J00 = fx / X[2];
  float J02 = -(fx * tx) / z2;
  float J11 = fy / X[2];
  float J12 = -(fy * ty) / z2;
  /* T = J * Wc, Wc = R^T (world->camera rotation): Wc[r][c] = R[c][r] */
  float T[6];
  for (int c = 0; c < 3; ++c) {
    float a0 = J00 * R[c * 3 + 0];
    float a2 = J02 * R[c * 3 + 2];
    T[c] = a0 + a2;
    float b1 = J11 * R[c * 3 + 1];
    float b2 = J12 * R[c * 3 + 2];
    T[3 + c] = b1 + b2;
  }
  float U[6];
  for (int a = 0; a < 2; ++a)
    for (int c = 0; c < 3; ++c) {
      float acc = T[3 * a + 0] * S[0 * 3 + c];
      float p1 = T[3 * a + 1] * S[1 * 3 + c];
      acc = acc + p1;
      float p2 = T[3 * a + 2] * S[2 * 3 + c];
      U[3 * a + c] = acc + p2;
    }
  float Sg[3]; /* xx, xy, yy */
  int ab[3][2] = {{0, 0}, {0, 1}, {1, 1}};
  for (int e = 0; e < 3; ++e) {
    int a = ab[e][0], b = ab[e][1];
    float acc = U[3 * a + 0] * T[3 * b + 0];
    float p1 = U[3 * a + 1] * T[3 * b + 1];
    acc = acc + p1;
    float p2 = U[3 * a + 2] * T[3 * b + 2];
    Sg[e] = acc + p2;
  }
  float cxx = Sg[0] + lowpass, cxy = Sg[1], cyy = Sg[2] + lowpass;
  float det = cxx * cyy - cxy * cxy;
  if (!(det > 0.0f)) return;
  g->a = cyy / det;
  g->b = -(cxy / det);
  g->c = cxx / det;
  g->px = (fx * X[0]) / X[2] + cx;
  g->py = (fy * X[1]) / X[2] + cy;
  g->lnsig = (float)(-log1p(exp(-(double)o)));
  float rx = 3.0f * sqrtf(cxx), ry = 3.0f * sqrtf(cyy);
  float fx0 = floorf(g->px - rx), fx1 = ceilf(g->px + rx), fy0 = floorf(g->py - ry), fy1 = ceilf(g->py + ry);
  if (fx0 < 0.0f) fx0 = 0.0f;
  if (fy0 < 0.0f) fy0 = 0.0f;
  if (fx1 > (float)(W - 1)) fx1 = (float)(W - 1);
  if (fy1 > (float)(H - 1)) fy1 = (float)(H - 1);
  if (!(fx0 <= fx1 && fy0 <= fy1)) return;
  g->rect[0] = (int32_t)fx0;
  g->rect[1] = (int32_t)fy0;
  g->rect[2] = (int32_t)fx1;
  g->rect[3] = (int32_t)fy1;
  g->culled = 0;
}

/* Pair membership (Eqs. 1-3 indicator and alpha clamp with the 3-sigma reading R-FOOT), decided
 * in prescribed fp32: q = Delta^T conic Delta with explicit fused multiply-adds,
 * in iff q <= min(9, 2 (L + ln sigma)), L = fl(-ln alpha_min) computed in double
 *                                  [<=> 3-sigma ellipse and alpha >= alpha_min (= 1/255)]
 *         and (D_t == 0 or d < fl(D_t + eps)).                                                 */
static int in_p32(const p32* g, int x, int y, float Dt, float eps, float L) {
  float dx = (float)x - g->px, dy = (float)y - g->py;
  float b2 = 2.0f * g->b;
  float t1 = g->a * dx;
  float t2 = b2 * dx;
  float t3 = g->c * dy;
  float t4 = t3 * dy;
  float inner = fmaf(t2, dy, t4);
  float q = fmaf(t1, dx, inner);
  float qs = L + g->lnsig;
  float qmax = 2.0f * qs;
  if (qmax > 9.0f) qmax = 9.0f;
  if (!(q <= qmax)) return 0;
  if (Dt != 0.0f) {
    float lim = Dt + eps;
    if (!(g->d < lim)) return 0;
  }
  return 1;
}

void orc_project_p32_full(int64_t n, const float* xyz, const float* ls, const float* rot, const float* op,
                          const float* K4, int W, int H, const float* R, const float* t, float near_z,
                          float lowpass, int32_t* rect, float* depth, int32_t* culled, float* fields /*n*6*/) {
  for (int64_t i = 0; i < n; ++i) {
    p32 g;
    proj32(xyz + 3 * i, ls + 3 * i, rot + 4 * i, op ? op[i] : 0.0f, K4, W, H, R, t, near_z, lowpass, &g);
    culled[i] = g.culled;
    depth[i] = g.d;
    for (int k = 0; k < 4; ++k) rect[4 * i + k] = g.rect[k];
    if (fields) {
      fields[6 * i] = g.px; fields[6 * i + 1] = g.py; fields[6 * i + 2] = g.a;
      fields[6 * i + 3] = g.b; fields[6 * i + 4] = g.c; fields[6 * i + 5] = g.lnsig;
    }
  }
}

void orc_project_p32(int64_t n, const float* xyz, const float* ls, const float* rot,
                     const float* K4, int W, int H, const float* R, const float* t, float near_z,
                     float lowpass, int32_t* rect, float* depth, int32_t* culled) {
  orc_project_p32_full(n, xyz, ls, rot, NULL, K4, W, H, R, t, near_z, lowpass, rect, depth, culled, NULL);
}

/* ---- F64 projection, the forward quantities of one Gaussian -------------- */

static const double SH_C0 = 0.28209479177387814;
static const double SH_C1 = 0.4886025119029199;
static const double SH_C2[5] = {1.0925484305920792, -1.0925484305920792, 0.31539156525252005,
                                -1.0925484305920792, 0.5462742152960396};
static const double SH_C3[7] = {-0.5900435899266435, 2.890611442640554, -0.4570457994644658,
                                0.3731763325901154, -0.4570457994644658, 1.445305721320277,
                                -0.5900435899266435};

/* real SH basis of 3DGS (degree <= 3) at direction (x,y,z), and its partial derivatives */
static void sh_basis(double x, double y, double z, double Y[16], double dY[16][3]) {
  double xx = x * x, yy = y * y, zz = z * z;
  memset(dY, 0, sizeof(double) * 48);
  Y[0] = SH_C0;
  Y[1] = -SH_C1 * y; dY[1][1] = -SH_C1;
  Y[2] = SH_C1 * z;  dY[2][2] = SH_C1;
  Y[3] = -SH_C1 * x; dY[3][0] = -SH_C1;
  Y[4] = SH_C2[0] * x * y;               dY[4][0] = SH_C2[0] * y; dY[4][1] = SH_C2[0] * x;
  Y[5] = SH_C2[1] * y * z;               dY[5][1] = SH_C2[1] * z; dY[5][2] = SH_C2[1] * y;
  Y[6] = SH_C2[2] * (2 * zz - xx - yy);  dY[6][0] = -2 * SH_C2[2] * x; dY[6][1] = -2 * SH_C2[2] * y; dY[6][2] = 4 * SH_C2[2] * z;
  Y[7] = SH_C2[3] * x * z;               dY[7][0] = SH_C2[3] * z; dY[7][2] = SH_C2[3] * x;
  Y[8] = SH_C2[4] * (xx - yy);           dY[8][0] = 2 * SH_C2[4] * x; dY[8][1] = -2 * SH_C2[4] * y;
  Y[9] = SH_C3[0] * y * (3 * xx - yy);
  dY[9][0] = SH_C3[0] * 6 * x * y; dY[9][1] = SH_C3[0] * (3 * xx - 3 * yy);
  Y[10] = SH_C3[1] * x * y * z;
  dY[10][0] = SH_C3[1] * y * z; dY[10][1] = SH_C3[1] * x * z; dY[10][2] = SH_C3[1] * x * y;
  Y[11] = SH_C3[2] * y * (4 * zz - xx - yy);
  dY[11][0] = SH_C3[2] * (-2 * x * y); dY[11][1] = SH_C3[2] * (4 * zz - xx - 3 * yy); dY[11][2] = SH_C3[2] * 8 * y * z;
  Y[12] = SH_C3[3] * z * (2 * zz - 3 * xx - 3 * yy);
  dY[12][0] = SH_C3[3] * (-6 * x * z); dY[12][1] = SH_C3[3] * (-6 * y * z); dY[12][2] = SH_C3[3] * (6 * zz - 3 * xx - 3 * yy);
  Y[13] = SH_C3[4] * x * (4 * zz - xx - yy);
  dY[13][0] = SH_C3[4] * (4 * zz - 3 * xx - yy); dY[13][1] = SH_C3[4] * (-2 * x * y); dY[13][2] = SH_C3[4] * 8 * x * z;
  Y[14] = SH_C3[5] * z * (xx - yy);
  dY[14][0] = SH_C3[5] * 2 * x * z; dY[14][1] = SH_C3[5] * (-2 * y * z); dY[14][2] = SH_C3[5] * (xx - yy);
  Y[15] = SH_C3[6] * x * (xx - 3 * yy);
  dY[15][0] = SH_C3[6] * (3 * xx - 3 * yy); dY[15][1] = SH_C3[6] * (-6 * x * y);
}

/* exported for the orthonormality pin */
void orc_sh_basis(double x, double y, double z, double* Y16, double* dY48) {
  double dY[16][3];
  sh_basis(x, y, z, Y16, dY);
  if (dY48) memcpy(dY48, dY, sizeof(dY));
}

typedef struct {
  int culled;
  double X[3], s[3], qh[4], qn, Rq[9], M[9], S[9];
  double cu, cv, clampx, clampy; /* clamped tan values and flags */
  double J00, J02, J11, J12, T[6];
  double cxx, cxy, cyy, det, a, b, c; /* Sigma_2D (+lowpass) and conic */
  double px, py, sigma, col[3];
  int clamped[3];
  double dir[3], dnorm, Y[16], dY[16][3];
  double d;
} gproj;

typedef struct {
  double fx, fy, cx, cy;
  int W, H;
  double R[9], t[3];
  double near_z, lowpass;
} camf64;

static void project_f64(const camf64* cam, int deg, const double* p, const double* ls,
                        const double* q, double o, const double* sh, gproj* g) {
  memset(g, 0, sizeof(*g));
  g->culled = 1;
  double D[3];
  for (int c = 0; c < 3; ++c) D[c] = p[c] - cam->t[c];
  for (int c = 0; c < 3; ++c)
    g->X[c] = cam->R[0 * 3 + c] * D[0] + cam->R[1 * 3 + c] * D[1] + cam->R[2 * 3 + c] * D[2];
  g->d = g->X[2];
  if (!(g->X[2] > 0.0)) return; /* behind the camera: culled, nothing else defined */
  double z = g->X[2];
  for (int c = 0; c < 3; ++c) g->s[c] = exp(ls[c]);
  g->qn = sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
  for (int k = 0; k < 4; ++k) g->qh[k] = q[k] / g->qn;
  double w = g->qh[0], x = g->qh[1], y = g->qh[2], qz = g->qh[3];
  double* Rq = g->Rq;
  Rq[0] = 1 - 2 * (y * y + qz * qz); Rq[1] = 2 * (x * y - w * qz);     Rq[2] = 2 * (x * qz + w * y);
  Rq[3] = 2 * (x * y + w * qz);     Rq[4] = 1 - 2 * (x * x + qz * qz); Rq[5] = 2 * (y * qz - w * x);
  Rq[6] = 2 * (x * qz - w * y);     Rq[7] = 2 * (y * qz + w * x);     Rq[8] = 1 - 2 * (x * x + y * y);
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) g->M[3 * r + c] = Rq[3 * r + c] * g->s[c];
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c)
      g->S[3 * r + c] = g->M[3 * r] * g->M[3 * c] + g->M[3 * r + 1] * g->M[3 * c + 1] + g->M[3 * r + 2] * g->M[3 * c + 2];
  double limx = 1.3 * ((double)cam->W / (2.0 * cam->fx)), limy = 1.3 * ((double)cam->H / (2.0 * cam->fy));
  double u = g->X[0] / z, v = g->X[1] / z;
  g->clampx = (u < -limx || u > limx);
  g->clampy = (v < -limy || v > limy);
  g->cu = u < -limx ? -limx : (u > limx ? limx : u);
  g->cv = v < -limy ? -limy : (v > limy ? limy : v);
  /* J of the perspective map with x/z, y/z clamped (3DGS): J02 = -fx*(cu*z)/z^2 = -fx*cu/z */
  g->J00 = cam->fx / z;
  g->J02 = -cam->fx * g->cu / z;
  g->J11 = cam->fy / z;
  g->J12 = -cam->fy * g->cv / z;
  for (int c = 0; c < 3; ++c) {
    g->T[c] = g->J00 * cam->R[c * 3 + 0] + g->J02 * cam->R[c * 3 + 2];
    g->T[3 + c] = g->J11 * cam->R[c * 3 + 1] + g->J12 * cam->R[c * 3 + 2];
  }
  double ST0[3], ST1[3];
  for (int r = 0; r < 3; ++r) {
    ST0[r] = g->S[3 * r] * g->T[0] + g->S[3 * r + 1] * g->T[1] + g->S[3 * r + 2] * g->T[2];
    ST1[r] = g->S[3 * r] * g->T[3] + g->S[3 * r + 1] * g->T[4] + g->S[3 * r + 2] * g->T[5];
  }
  g->cxx = g->T[0] * ST0[0] + g->T[1] * ST0[1] + g->T[2] * ST0[2] + cam->lowpass;
  g->cxy = g->T[0] * ST1[0] + g->T[1] * ST1[1] + g->T[2] * ST1[2];
  g->cyy = g->T[3] * ST1[0] + g->T[4] * ST1[1] + g->T[5] * ST1[2] + cam->lowpass;
  g->det = g->cxx * g->cyy - g->cxy * g->cxy;
  if (!(g->det > 0)) return; /* degenerate covariance: culled */
  g->a = g->cyy / g->det;
  g->b = -g->cxy / g->det;
  g->c = g->cxx / g->det;
  g->px = cam->fx * g->X[0] / z + cam->cx;
  g->py = cam->fy * g->X[1] / z + cam->cy;
  g->sigma = 1.0 / (1.0 + exp(-o));
  /* view-dependent colour, centre direction (R-SH) */
  g->dnorm = sqrt(D[0] * D[0] + D[1] * D[1] + D[2] * D[2]);
  for (int c = 0; c < 3; ++c) g->dir[c] = D[c] / g->dnorm;
  sh_basis(g->dir[0], g->dir[1], g->dir[2], g->Y, g->dY);
  int nc = (deg + 1) * (deg + 1);
  for (int ch = 0; ch < 3; ++ch) {
    double acc = 0.0;
    for (int k = 0; k < nc; ++k) acc += g->Y[k] * sh[3 * k + ch];
    acc += 0.5;
    g->clamped[ch] = acc < 0.0;
    g->col[ch] = acc < 0.0 ? 0.0 : acc;
  }
  /* near-plane cull (R-NEAR) decided last so that the tests can see the would-be footprint */
  g->culled = !(g->X[2] > cam->near_z);
}

static camf64 make_cam(const double* K4, int W, int H, const double* R, const double* t,
                       double near_z, double lowpass) {
  camf64 c;
  c.fx = K4[0]; c.fy = K4[1]; c.cx = K4[2]; c.cy = K4[3];
  c.W = W; c.H = H;
  for (int k = 0; k < 9; ++k) c.R[k] = R[k];
  for (int k = 0; k < 3; ++k) c.t[k] = t[k];
  c.near_z = near_z;
  c.lowpass = lowpass;
  return c;
}

typedef struct {
  int in;       /* pair contributes: the P32 decision (in_p32)                                 */
  int amb;      /* an fp64 evaluation of a decision is within fp32 noise of its threshold,
                   i.e. an fp64-decided implementation may legitimately disagree here       */
  double alpha, dx, dy, ex; /* fp64 values; ex = exp(-power) */
} pairv;

/* Eqs. 1-3 for one pair: membership from the P32 fields, values in fp64. */
static pairv eval_pair(const gproj* g, const p32* h, int x, int y, double Dt, double eps, double alpha_min) {
  pairv r;
  memset(&r, 0, sizeof(r));
  r.dx = (double)x - g->px;
  r.dy = (double)y - g->py;
  double qf = g->a * r.dx * r.dx + 2.0 * g->b * r.dx * r.dy + g->c * r.dy * r.dy;
  double power = 0.5 * qf;
  r.ex = exp(-power);
  r.alpha = g->sigma * r.ex;
  r.in = in_p32(h, x, y, (float)Dt, (float)eps, (float)(-log((double)(float)alpha_min)));
  int in_ell = qf <= 9.0;
  int in_alpha = r.alpha >= alpha_min;
  int in_depth = (Dt == 0.0) || (g->d < Dt + eps);
  int near_ell = fabs(qf - 9.0) < 1e-4;
  int near_alpha = fabs(r.alpha / alpha_min - 1.0) < 1e-4;
  int near_depth = (Dt != 0.0) && fabs(g->d - (Dt + eps)) < 3e-6;
  r.amb = (near_ell && (in_alpha || near_alpha) && (in_depth || near_depth)) ||
          (near_alpha && (in_ell || near_ell) && (in_depth || near_depth)) ||
          (near_depth && (in_ell || near_ell) && (in_alpha || near_alpha));
  return r;
}

/* Gaussian-level decisions whose fp64 evaluation is near a threshold (near plane, det) */
static int gauss_amb(const gproj* g, double near_z) {
  if (fabs(g->d - near_z) < 1e-5) return 1;
  if (g->det > 0 && g->det < 1e-6 * g->cxx * g->cyy) return 1;
  return 0;
}

static void f32_params(const double* xyz, const double* ls, const double* rot, double op, float* p,
                       float* l, float* q, float* o) {
  for (int k = 0; k < 3; ++k) {
    p[k] = (float)xyz[k];
    l[k] = (float)ls[k];
  }
  for (int k = 0; k < 4; ++k) q[k] = (float)rot[k];
  *o = (float)op;
}

static void cam32(const double* K4, const double* R, const double* t, float* K4f, float* Rf, float* tf) {
  for (int k = 0; k < 4; ++k) K4f[k] = (float)K4[k];
  for (int k = 0; k < 9; ++k) Rf[k] = (float)R[k];
  for (int k = 0; k < 3; ++k) tf[k] = (float)t[k];
}

/* Forward: Eqs. 1-4 per pixel (plain definition: sums over all Gaussians, W_t = 1), values in
 * fp64, pair membership decided in prescribed fp32.  Params in double (their
 * fp32 roundings feed the decisions).  Dt (0 = SDF miss, R-MISS) and Ct are per-pixel inputs.
 * Outputs: Cstar (H*W*3), WG (H*W), CG (H*W*3, nullable), amb (H*W, nullable): 1 where an
 * fp64-decided implementation could legitimately differ (used only against such references). */
void orc_render(int64_t n, int deg, const double* xyz, const double* ls, const double* rot,
                const double* op, const double* sh, const double* K4, int W, int H,
                const double* R, const double* t, double eps, double alpha_min, double near_z,
                double lowpass, const double* Dt, const double* Ct, double* Cstar, double* WG,
                double* CG, uint8_t* amb) {
  camf64 cam = make_cam(K4, W, H, R, t, near_z, lowpass);
  float K4f[4], Rf[9], tf[3];
  cam32(K4, R, t, K4f, Rf, tf);
  int nc = (deg + 1) * (deg + 1);
  int64_t HW = (int64_t)W * H;
  double* cg = (double*)calloc(HW * 3, sizeof(double));
  memset(WG, 0, sizeof(double) * HW);
  if (amb) memset(amb, 0, HW);
  /* One band of image rows per task; every pixel still sums its Gaussians in index order, so the
   * result does not depend on the band count (1 in the serial build the tests use; the OpenMP
   * build, a timing baseline only, runs bands in parallel). */
  int nbands = 1;
#ifdef _OPENMP
  nbands = 4 * omp_get_max_threads();
  if (nbands > H) nbands = H;
#endif
#pragma omp parallel for schedule(dynamic, 1)
  for (int band = 0; band < nbands; ++band) {
    const int by0 = (int)((int64_t)band * H / nbands), by1 = (int)((int64_t)(band + 1) * H / nbands) - 1;
    for (int64_t i = 0; i < n; ++i) {
      float pf[3], lf[3], qf[4], of;
      f32_params(xyz + 3 * i, ls + 3 * i, rot + 4 * i, op[i], pf, lf, qf, &of);
      p32 h;
      proj32(pf, lf, qf, of, K4f, W, H, Rf, tf, (float)near_z, (float)lowpass, &h);
      if (h.culled && !amb) continue; /* contributes nothing; only the ambiguity map needs it */
      if (nbands > 1 && !h.culled && (h.rect[3] < by0 || h.rect[1] > by1)) continue;
      gproj g;
      project_f64(&cam, deg, xyz + 3 * i, ls + 3 * i, rot + 4 * i, op[i], sh + 3 * nc * i, &g);
      int gam = gauss_amb(&g, near_z);
      if (h.culled || !(g.det > 0) || !(g.X[2] > 0)) {
        if (amb && gam && g.det > 0 && g.X[2] > 0) { /* fp64 might keep it: flag its footprint */
          double rx = 3.0 * sqrt(g.cxx) + 1.0, ry = 3.0 * sqrt(g.cyy) + 1.0;
          int x0 = (int)fmax(0, floor(g.px - rx)), x1 = (int)fmin(W - 1, ceil(g.px + rx));
          int y0 = (int)fmax(by0, floor(g.py - ry)), y1 = (int)fmin(by1, ceil(g.py + ry));
          for (int y = y0; y <= y1; ++y)
            for (int x = x0; x <= x1; ++x) amb[(int64_t)y * W + x] = 1;
        }
        continue;
      }
      const int ry0 = h.rect[1] > by0 ? h.rect[1] : by0, ry1 = h.rect[3] < by1 ? h.rect[3] : by1;
      for (int y = ry0; y <= ry1; ++y)
        for (int x = h.rect[0]; x <= h.rect[2]; ++x) {
          int64_t pi = (int64_t)y * W + x;
          pairv pv = eval_pair(&g, &h, x, y, Dt[pi], eps, alpha_min);
          if (amb && (pv.amb || (gam && pv.in))) amb[pi] = 1;
          if (!pv.in) continue;
          for (int ch = 0; ch < 3; ++ch) cg[3 * pi + ch] += pv.alpha * g.col[ch];
          WG[pi] += pv.alpha;
        }
    }
  }
  for (int64_t pi = 0; pi < HW; ++pi)
    for (int ch = 0; ch < 3; ++ch) Cstar[3 * pi + ch] = (Ct[3 * pi + ch] + cg[3 * pi + ch]) / (1.0 + WG[pi]);
  if (CG) memcpy(CG, cg, sizeof(double) * HW * 3);
  free(cg);
}

/* Exact gradient of L with respect to every raw parameter (reading R-GRAD), given the
 * upstream dL/dC* per pixel (G, H*W*3) and the forward outputs Cstar, WG of orc_render.
 * Indicators, the alpha cutoff, the 3-sigma boundary and the J clamp are locally constant.
 * Outputs (double, parameter SoA layout): gxyz n*3, gls n*3, grot n*4, gop n, gsh n*nc*3.
 * gamb (nullable, n): 1 if the Gaussian has an ambiguous decision or an in-pair at a pixel with
 * pix_amb set (nullable input).                                                             */
void orc_backward(int64_t n, int deg, const double* xyz, const double* ls, const double* rot,
                  const double* op, const double* sh, const double* K4, int W, int H,
                  const double* R, const double* t, double eps, double alpha_min, double near_z,
                  double lowpass, const double* Dt, const double* Cstar, const double* WG,
                  const double* G, const uint8_t* pix_amb, double* gxyz, double* gls,
                  double* grot, double* gop, double* gsh, uint8_t* gamb) {
  camf64 cam = make_cam(K4, W, H, R, t, near_z, lowpass);
  float K4f[4], Rf[9], tf[3];
  cam32(K4, R, t, K4f, Rf, tf);
  int nc = (deg + 1) * (deg + 1);
#pragma omp parallel for schedule(dynamic, 64)
  for (int64_t i = 0; i < n; ++i) {
    double* dp = gxyz + 3 * i;
    double* dls = gls + 3 * i;
    double* dq = grot + 4 * i;
    double* dsh = gsh + 3 * nc * i;
    memset(dp, 0, 24);
    memset(dls, 0, 24);
    memset(dq, 0, 32);
    gop[i] = 0.0;
    memset(dsh, 0, sizeof(double) * 3 * nc);
    if (gamb) gamb[i] = 0;
    gproj g;
    const double* sh_i = sh + 3 * nc * i;
    project_f64(&cam, deg, xyz + 3 * i, ls + 3 * i, rot + 4 * i, op[i], sh_i, &g);
    float pf[3], lf[3], qf[4], of;
    f32_params(xyz + 3 * i, ls + 3 * i, rot + 4 * i, op[i], pf, lf, qf, &of);
    p32 h;
    proj32(pf, lf, qf, of, K4f, W, H, Rf, tf, (float)near_z, (float)lowpass, &h);
    if (gamb && gauss_amb(&g, near_z)) gamb[i] = 1;
    if (h.culled || !(g.det > 0) || !(g.X[2] > 0)) continue;
    /* ---- per-pair accumulation of the 2D gradients ---- */
    double dcol[3] = {0, 0, 0}, dsig = 0, da = 0, db = 0, dc = 0, dpx = 0, dpy = 0;
    for (int y = h.rect[1]; y <= h.rect[3]; ++y)
      for (int x = h.rect[0]; x <= h.rect[2]; ++x) {
        int64_t pi = (int64_t)y * W + x;
        pairv pv = eval_pair(&g, &h, x, y, Dt[pi], eps, alpha_min);
        if (gamb && (pv.amb || (pv.in && pix_amb && pix_amb[pi]))) gamb[i] = 1;
        if (!pv.in) continue;
        double A = 1.0 / (1.0 + WG[pi]);
        const double* Gp = G + 3 * pi;
        const double* Cs = Cstar + 3 * pi;
        double dalpha = 0.0;
        for (int ch = 0; ch < 3; ++ch) {
          dcol[ch] += Gp[ch] * pv.alpha * A;            /* d(C*)/d(C_G) = A, d(C_G)/dc = alpha */
          dalpha += A * Gp[ch] * (g.col[ch] - Cs[ch]);  /* d(C*)/d(W_G) = -(C*) A              */
        }
        dsig += dalpha * pv.ex;
        double dpow = -pv.alpha * dalpha;
        da += dpow * 0.5 * pv.dx * pv.dx;
        db += dpow * pv.dx * pv.dy;
        dc += dpow * 0.5 * pv.dy * pv.dy;
        dpx += dpow * (-(g.a * pv.dx + g.b * pv.dy));
        dpy += dpow * (-(g.b * pv.dx + g.c * pv.dy));
      }
    /* ---- opacity ---- */
    gop[i] = dsig * g.sigma * (1.0 - g.sigma);
    /* ---- colour -> SH coefficients and view direction ---- */
    double ddir[3] = {0, 0, 0};
    for (int ch = 0; ch < 3; ++ch) {
      if (g.clamped[ch]) dcol[ch] = 0.0;
      for (int k = 0; k < nc; ++k) {
        dsh[3 * k + ch] = g.Y[k] * dcol[ch];
        for (int e = 0; e < 3; ++e) ddir[e] += dcol[ch] * sh_i[3 * k + ch] * g.dY[k][e];
      }
    }
    double dd_dot = ddir[0] * g.dir[0] + ddir[1] * g.dir[1] + ddir[2] * g.dir[2];
    for (int e = 0; e < 3; ++e) dp[e] += (ddir[e] - g.dir[e] * dd_dot) / g.dnorm;
    /* ---- conic (a,b,c) -> Sigma_2D (cxx, cxy, cyy) ---- */
    double det = g.det, det2 = det * det;
    double cxx = g.cxx, cxy = g.cxy, cyy = g.cyy;
    double dcxx = da * (-cyy * cyy / det2) + db * (cxy * cyy / det2) + dc * (1.0 / det - cxx * cyy / det2);
    double dcyy = da * (1.0 / det - cyy * cxx / det2) + db * (cxy * cxx / det2) + dc * (-cxx * cxx / det2);
    double dcxy = da * (2.0 * cyy * cxy / det2) + db * (-1.0 / det - 2.0 * cxy * cxy / det2) + dc * (2.0 * cxx * cxy / det2);
    /* ---- Sigma_2D = T S T^T + lowpass I ---- */
    const double* T0 = g.T;
    const double* T1 = g.T + 3;
    double ST0[3], ST1[3];
    for (int r = 0; r < 3; ++r) {
      ST0[r] = g.S[3 * r] * T0[0] + g.S[3 * r + 1] * T0[1] + g.S[3 * r + 2] * T0[2];
      ST1[r] = g.S[3 * r] * T1[0] + g.S[3 * r + 1] * T1[1] + g.S[3 * r + 2] * T1[2];
    }
    double dS[9], dT[6];
    for (int j = 0; j < 3; ++j)
      for (int k = 0; k < 3; ++k)
        dS[3 * j + k] = dcxx * T0[j] * T0[k] + dcxy * T0[j] * T1[k] + dcyy * T1[j] * T1[k];
    for (int j = 0; j < 3; ++j) {
      dT[j] = dcxx * 2.0 * ST0[j] + dcxy * ST1[j];
      dT[3 + j] = dcxy * ST0[j] + dcyy * 2.0 * ST1[j];
    }
    /* ---- T = J Wc ---- */
    double dJ00 = 0, dJ02 = 0, dJ11 = 0, dJ12 = 0;
    for (int j = 0; j < 3; ++j) {
      dJ00 += dT[j] * cam.R[j * 3 + 0];
      dJ02 += dT[j] * cam.R[j * 3 + 2];
      dJ11 += dT[3 + j] * cam.R[j * 3 + 1];
      dJ12 += dT[3 + j] * cam.R[j * 3 + 2];
    }
    /* ---- J and p_hat -> camera point X ---- */
    double z = g.X[2], dX[3] = {0, 0, 0};
    double fx = cam.fx, fy = cam.fy;
    /* J00 = fx/z, J11 = fy/z */
    dX[2] += dJ00 * (-fx / (z * z)) + dJ11 * (-fy / (z * z));
    /* J02 = -fx*cu/z with cu = clamp(X.x/z) (constant when clamped) */
    double dcu_dxx = g.clampx ? 0.0 : 1.0 / z, dcu_dz = g.clampx ? 0.0 : -g.X[0] / (z * z);
    double dcv_dxy = g.clampy ? 0.0 : 1.0 / z, dcv_dz = g.clampy ? 0.0 : -g.X[1] / (z * z);
    dX[0] += dJ02 * (-fx / z) * dcu_dxx;
    dX[2] += dJ02 * (fx * g.cu / (z * z) - fx / z * dcu_dz);
    dX[1] += dJ12 * (-fy / z) * dcv_dxy;
    dX[2] += dJ12 * (fy * g.cv / (z * z) - fy / z * dcv_dz);
    /* p_hat = (fx x/z + cx, fy y/z + cy) */
    dX[0] += dpx * fx / z;
    dX[1] += dpy * fy / z;
    dX[2] += dpx * (-fx * g.X[0] / (z * z)) + dpy * (-fy * g.X[1] / (z * z));
    /* X = R^T (p - t)  =>  dp = R dX */
    for (int r = 0; r < 3; ++r) dp[r] += cam.R[3 * r] * dX[0] + cam.R[3 * r + 1] * dX[1] + cam.R[3 * r + 2] * dX[2];
    /* ---- S = M M^T, M = Rq diag(s) ---- */
    double dM[9];
    for (int j = 0; j < 3; ++j)
      for (int l = 0; l < 3; ++l) {
        double acc = 0.0;
        for (int k = 0; k < 3; ++k) acc += (dS[3 * j + k] + dS[3 * k + j]) * g.M[3 * k + l];
        dM[3 * j + l] = acc;
      }
    double dRq[9];
    for (int l = 0; l < 3; ++l) {
      double ds = 0.0;
      for (int j = 0; j < 3; ++j) {
        dRq[3 * j + l] = dM[3 * j + l] * g.s[l];
        ds += dM[3 * j + l] * g.Rq[3 * j + l];
      }
      dls[l] = ds * g.s[l]; /* s = exp(log s) */
    }
    /* ---- Rq(q_hat) -> q_hat -> raw q ---- */
    double w = g.qh[0], x = g.qh[1], y = g.qh[2], qz = g.qh[3];
    /* partials of the 9 entries w.r.t. (w,x,y,z) */
    double P[9][4] = {
        {0, 0, -4 * y, -4 * qz},          {-2 * qz, 2 * y, 2 * x, -2 * w}, {2 * y, 2 * qz, 2 * w, 2 * x},
        {2 * qz, 2 * y, 2 * x, 2 * w},    {0, -4 * x, 0, -4 * qz},         {-2 * x, -2 * w, 2 * qz, 2 * y},
        {-2 * y, 2 * qz, -2 * w, 2 * x},  {2 * x, 2 * w, 2 * qz, 2 * y},   {0, -4 * x, -4 * y, 0}};
    double dqh[4] = {0, 0, 0, 0};
    for (int e = 0; e < 9; ++e)
      for (int k = 0; k < 4; ++k) dqh[k] += dRq[e] * P[e][k];
    double dot = dqh[0] * g.qh[0] + dqh[1] * g.qh[1] + dqh[2] * g.qh[2] + dqh[3] * g.qh[3];
    for (int k = 0; k < 4; ++k) dq[k] = (dqh[k] - g.qh[k] * dot) / g.qn;
  }
}
