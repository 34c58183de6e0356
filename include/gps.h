/*
 * gps.h -- C ABI of libgps.so, the B200 (sm_100a) implementation of the per-frame
 * Gaussian-Plus-SDF mapping step of GPS-SLAM (arXiv 2509.11574).
 *
 * Citations: "P:n" = /root/reference/PAPER.md line n (section / equation named beside it);
 * readings of points the paper leaves silent are numbered R-* in DESIGN.md §3.
 *
 * The paper states the problem as (Sec. 3.2.1 "SDF fusion"): "Given the k-th frame ...
 * an RGB image C_k and a depth map D_k ... with the intrinsic camera parameters ... using the
 * estimated camera pose T_{g,k} ... update the SDF and color values in a global hash table;
 * afterwards the raycast is performed", then render with Eqs. 1-4 (Sec. 3.1) and
 * optimise with the L1 loss of Eq. 7 using Adam (App. C).
 * The four hot entry points are gps_fuse, gps_raycast, gps_render and gps_refine_step;
 * gps_fuse_raycast (a frame) and gps_refine_round (a round of iterations) run the same kernels
 * in one call each, replayed as CUDA graphs (graph objects are the library's only host-side
 * per-workspace / per-volume state; the executable graphs are created on first use).
 *
 * General conventions (apply to every function below)
 *  - Every pointer is a DEVICE pointer unless marked (host).  Device buffers are caller-owned,
 *    contiguous, 16-byte aligned, and must stay alive until the stream work completes.
 *  - `stream` is a cudaStream_t passed as an opaque pointer (NULL = legacy default stream).
 *    All calls enqueue work on `stream` and return without synchronising, except the ones
 *    whose name ends in _sync.
 *  - Argument validation is synchronous and happens before any launch: a bad argument returns
 *    GPS_ERR_INVALID_ARG and enqueues nothing.  Data invalidity is NOT an error: zero depth,
 *    ray misses, culled Gaussians and an empty loss mask are ordinary data.
 *  - CUDA launch failures return GPS_ERR_CUDA; gps_last_error() then holds a thread-local
 *    message.  No C++ exception ever crosses this ABI.
 *  - The library never allocates device memory on the hot path: the volume is allocated once
 *    by gps_volume_create, everything else is caller-provided (workspace sizes come from the
 *    *_workspace_size queries).
 *  - Pixel (u,v) has integer coordinates at its centre; camera point X projects to
 *    (fx*X.x/X.z + cx, fy*X.y/X.z + cy) (R-PIX).  Poses are camera->world, R row-major
 *    (R-POSE); world->camera is X = R^T (P - t).
 */
#ifndef GPS_H_
#define GPS_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GPS_ABI_VERSION 4  /* 2: gps_render_config.sort_free; adding, removal, tracking entry points; 3: device-pose forms; 4: gps_refine_round, gps_fuse_raycast */

typedef void* gps_stream_t; /* a cudaStream_t */

typedef enum {
  GPS_OK = 0,
  GPS_ERR_INVALID_ARG = 1,         /* synchronous argument check failed; nothing enqueued      */
  GPS_ERR_OUT_OF_BLOCKS = 2,       /* a previous gps_fuse exceeded max_blocks (sticky)         */
  GPS_ERR_WORKSPACE_TOO_SMALL = 3, /* ws_bytes below the *_workspace_size query                */
  GPS_ERR_CUDA = 4,                /* CUDA runtime error; see gps_last_error()                 */
  GPS_ERR_OOM = 5                  /* gps_volume_create could not allocate                     */
} gps_status;

/* Pinhole intrinsics shared by the depth and colour images (R-PIX).  width,height in pixels. */
typedef struct {
  float fx, fy, cx, cy;
  int32_t width, height;
} gps_intrinsics;

/* Camera->world rigid transform T_{g,k}.  World point P = R * X_cam + t.             */
typedef struct {
  float R[9]; /* row-major */
  float t[3];
} gps_pose;

/* ------------------------------------------------------------------------------------------
 * Voxel-block hash volume ("update the SDF and color values in a global hash table";
 * voxel contents P:60: truncated signed distance d(p) and colour c(p)).
 * Library-owned and opaque.  Voxel (i,j,k) sits at world (i,j,k)*voxel_size; block b holds
 * voxels 8b..8b+7 per axis (R-VOX).  A voxel is 8 bytes {f32 tsdf in [-1,1] (1 == mu);
 * u8 r,g,b; u8 w}; a new block starts as tsdf = 1, rgb = 0, w = 0.
 * ------------------------------------------------------------------------------------------ */
typedef struct {
  float voxel_size; /* metres; paper: 0.005                                          */
  float mu;         /* truncation distance, metres; reading R-MU: 4*voxel_size = 0.02         */
  int32_t w_max;    /* weight cap, 1..255; reading R-WMAX: 100                                */
  float depth_min;  /* valid depth / ray range lower bound, metres (R-DEPTH: 0.1)             */
  float depth_max;  /* valid depth / ray range upper bound, metres (R-DEPTH: 10)              */
  int64_t max_blocks; /* block budget (>= 1); exceeding it is GPS_ERR_OUT_OF_BLOCKS          */
  int64_t hash_slots; /* open-addressing slots, power of two, >= 2*max_blocks recommended   */
  /* Optional dense block-index grid (an accelerator; results do not depend on it): blocks with
   * coordinates in [dense_origin, dense_origin + dense_dims) are also indexed by a direct array
   * (4 bytes per cell) so the raycast looks them up with one load instead of hash probing.
   * dense_dims all zero = disabled.  Coordinates in blocks (8 * voxel_size metres).            */
  int32_t dense_origin[3];
  int32_t dense_dims[3];
} gps_volume_config;

typedef struct gps_volume gps_volume;

/* Allocates the hash table and block pool on the current device and initialises them on
 * `stream`.  *out receives the handle (host).  Returns GPS_ERR_OOM if allocation fails.       */
gps_status gps_volume_create(const gps_volume_config* cfg /*host*/, gps_stream_t stream,
                             gps_volume** out /*host*/);
/* Frees everything.  The caller must ensure no work on the volume is pending.               */
void gps_volume_destroy(gps_volume* vol);
/* Empties the volume (all blocks free, overflow flag cleared, frame counter reset).          */
gps_status gps_volume_reset(gps_volume* vol, gps_stream_t stream);
/* Copies the complete state of `src` into `dst` (device to device, on `stream`): hash, blocks,
 * neighbour table, dense grid, counters and the sticky overflow flag.  Both volumes must have
 * been created with identical configs.  A snapshot for concurrent readers (the Gaussian thread
 * of P:116 reads a volume snapshot) or for replaying a sequence window.                      */
gps_status gps_volume_copy(gps_volume* dst, const gps_volume* src, gps_stream_t stream);
/* Synchronises `stream`, then reports the number of allocated blocks (may exceed the budget
 * when an overflow happened), the budget, the number of blocks marked visible by the last
 * gps_fuse, the sum of visible blocks over every integration since create/reset, and the sum
 * of voxels actually updated (eta >= -mu) over those integrations (the integration roofline's
 * unit count: 16 bytes each).  Any pointer may be NULL.  Returns
 * GPS_ERR_OUT_OF_BLOCKS if overflow happened.                                                 */
gps_status gps_volume_stats_sync(gps_volume* vol, gps_stream_t stream, int64_t* n_blocks /*host*/,
                                 int64_t* budget /*host*/, int64_t* n_visible /*host*/,
                                 int64_t* visible_total /*host*/, int64_t* updated_total /*host*/);

/* gps_fuse -- Sec. 3.2.1 "SDF fusion", voxel data P:60.
 * (1) Allocation: every valid depth pixel (depth/depth_scale in [depth_min, depth_max]) is
 *     back-projected; its band [X(1-mu/|X|), X(1+mu/|X|)] is sampled at 5 equispaced points,
 *     each transformed by the pose and mapped to block floor(W/(8*voxel_size)); every such
 *     block is inserted into the hash (R-BAND) and marked visible for this frame.
 * (2) Integration: every voxel of every visible block is projected to its nearest pixel; with
 *     eta = depth - z: skipped if eta < -mu, else s = min(1, eta/mu),
 *     tsdf <- (tsdf*w + s)*fl(1/(w+1)) (one correctly rounded reciprocal, then a multiply),
 *     rgb <- the exact rational running mean rounded half up, w <- min(w+1, w_max)
 *     (R-INT).  Allocation and tsdf use the prescribed fp32 sequences of DESIGN.md §4 (no FMA
 *     contraction) so that they are bit-reproducible.
 * depth: u16[height*width] row-major; metres = depth/depth_scale; 0 = invalid.
 * rgba:  u8[height*width*4] row-major RGBA, colour in [0,255] (alpha ignored).
 * Block-budget overflow is detected on device: the blocks that fit are integrated, a sticky
 * flag is set, and the NEXT call on this volume (or gps_volume_stats_sync) returns
 * GPS_ERR_OUT_OF_BLOCKS.  Must not run concurrently with any other call on the same volume.  */
gps_status gps_fuse(gps_volume* vol, const gps_intrinsics* K /*host*/, const gps_pose* T /*host*/,
                    const uint16_t* depth, float depth_scale, const uint8_t* rgba,
                    gps_stream_t stream);

/* gps_raycast -- Sec. 3.1 first pass: per-pixel march to the zero crossing, C_t by
 * trilinear interpolation of the eight neighbouring voxels' colours, D_t by projecting V*.
 * Reading R-RAY: unit ray from the camera centre; samples t_j = depth_min + j*voxel_size,
 * j = 0..J, J = floor((double)(depth_max-depth_min)/(double)voxel_size); a sample is valid iff
 * all 8 trilinear corners are allocated with w > 0; the first valid sample with tsdf <= 0 whose
 * predecessor is valid and > 0 gives t* by linear interpolation; otherwise a miss.
 * Unallocated blocks are skipped without changing the result.
 * depth_out:  f32[height*width], camera z of V* in metres; 0 = miss.
 * color_out:  f32[height*width*3], RGB in [0,1]; 0 on a miss.
 * vertex_out: nullable f32[height*width*3], V* in world metres; 0 on a miss.
 * The call writes the volume's per-volume range-image scratch (the result does not depend on
 * it): two raycasts of the same volume, or a raycast and a gps_fuse of it, must not run
 * concurrently on different streams -- order them on one stream or with events.             */
gps_status gps_raycast(gps_volume* vol, const gps_intrinsics* K /*host*/,
                       const gps_pose* T /*host*/, float* depth_out, float* color_out,
                       float* vertex_out, gps_stream_t stream);

/* gps_fuse_raycast -- gps_fuse of a frame followed by gps_raycast from the same pose (each
 * frame is fused, then raycast), in one call; same kernels, same order, same results as the two
 * calls.  use_graph != 0: the frame's launches are stream-captured and replayed as one CUDA graph
 * (one ring of executable graphs per volume, updated in place; skipped on the legacy/per-thread
 * default streams, inside a caller's own capture and while the event profiler is enabled).
 * Arguments and errors as gps_fuse and gps_raycast; on an error nothing is launched (with
 * use_graph; without it, a failing raycast leaves the fuse enqueued).                        */
gps_status gps_fuse_raycast(gps_volume* vol, const gps_intrinsics* K /*host*/, const gps_pose* T /*host*/,
                            const uint16_t* depth, float depth_scale, const uint8_t* rgba,
                            float* depth_out, float* color_out, float* vertex_out /*nullable*/,
                            int32_t use_graph, gps_stream_t stream);

/* Device-pose forms (tracking): identical to gps_fuse / gps_raycast --
 * same kernels, same fp32 sequences, same results for the same pose values -- except that the
 * pose is read on the device from T_dev (a gps_pose in device memory, 4-byte aligned, e.g. the
 * output of gps_track_async), so a tracked frame needs no host round trip.  T_dev must stay
 * valid until the stream has executed the call.                                               */
gps_status gps_fuse_dpose(gps_volume* vol, const gps_intrinsics* K /*host*/,
                          const gps_pose* T_dev /*device*/, const uint16_t* depth, float depth_scale,
                          const uint8_t* rgba, gps_stream_t stream);
gps_status gps_raycast_dpose(gps_volume* vol, const gps_intrinsics* K /*host*/,
                             const gps_pose* T_dev /*device*/, float* depth_out, float* color_out,
                             float* vertex_out, gps_stream_t stream);

/* ------------------------------------------------------------------------------------------
 * Gaussians ("G = {p_i, sigma_i, r_i, s_i, SH_i} ... following 3DGS").  Caller-owned SoA,
 * each array 16-byte aligned:
 *   xyz[n*3] world position; log_scale[n*3] (s = exp); rot[n*4] quaternion (w,x,y,z),
 *   normalised inside the forward pass (R-QUAT); opacity_raw[n] (sigma = sigmoid);
 *   sh[n*(deg+1)^2*3] coefficient-major RGB triples (coefficient l,m of Gaussian i, channel c at
 *   sh[(i*(deg+1)^2 + lm)*3 + c]).  sh_degree in {0,1,2,3} (R-SH: 3 for benchmarks).
 * ------------------------------------------------------------------------------------------ */
typedef struct {
  int64_t n;
  int32_t sh_degree;
  float* xyz;
  float* log_scale;
  float* rot;
  float* opacity_raw;
  float* sh;
} gps_gaussians;

/* Rasteriser settings.  Defaults in brackets are the readings of DESIGN.md §3.            */
typedef struct {
  float eps_depth;  /* epsilon of Eqs. 1-2, metres [0.02] (R-EPS)                  */
  float alpha_min;  /* alpha clamp of Eq. 3 text [1/255]                              */
  float near_z;     /* Gaussians with camera z <= near_z are culled [0.2] (R-NEAR)           */
  float lowpass;    /* added to the Sigma_2D diagonal, px^2 [0.3] (R-LOWPASS)                */
  int32_t tile;     /* 8 or 16: tile edge in pixels (accelerator only: output independent)   */
  int32_t tile_depth_precull; /* 0|1: drop list entries behind every pixel of the tile     */
  int64_t max_pairs; /* capacity of the (tile,Gaussian) pair list; 0 = 32*n + 65536         */
  int32_t sort_free; /* 0: depth-sorted tile lists, each pixel stops at its first entry at or
                      *    behind D_t + eps (sorted);
                      * 1: the paper's sort-free rendering (Table 7): lists
                      *    stay unsorted -- Eqs. 1-2 are order-free sums -- and every entry is
                      *    depth-tested; same C*, W_G up to fp32 summation order               */
  int32_t backward;  /* gradient scheme of gps_refine_step (same gradients up to fp32 summation
                      * order): 0 = the renderer's own (sorted: a warp per list entry with a
                      * warp reduction; sort-free: the paper's thread per (entry, 32-pixel
                      * group), App. B), 1 = warp per entry, 2 = thread per group   */
} gps_render_config;

size_t gps_render_workspace_size(int64_t n, const gps_intrinsics* K /*host*/,
                                 const gps_render_config* cfg /*host*/);

/* gps_render -- Sec. 3.1 second pass: Eqs. 1-3 with the 3-sigma footprint reading
 * (R-FOOT), composite Eq. 4 with W_t = 1:
 *   C* = (C_t + C_G)/(1 + W_G).
 * sdf_depth f32[H*W] (0 = miss: no depth test, R-MISS), sdf_color f32[H*W*3] in [0,1].
 * out_color f32[H*W*3] = C*, out_weight f32[H*W] = W_G.
 * target_rgba (nullable) u8[H*W*4] and loss_out (nullable device f32 scalar, needs target):
 * loss_out <- the mean L1 of Eq. 7 over the mask {D_t > 0 or W_G > 0} (R-L1).
 * ws: caller-provided device workspace of >= gps_render_workspace_size() bytes; it also keeps
 * the tile lists of the last render for gps_debug_render_lists_sync.                         */
gps_status gps_render(const gps_gaussians* g /*host struct, device arrays*/,
                      const gps_intrinsics* K /*host*/, const gps_pose* T /*host*/,
                      const float* sdf_depth, const float* sdf_color, const uint8_t* target_rgba,
                      const gps_render_config* cfg /*host*/, void* ws, size_t ws_bytes,
                      float* out_color, float* out_weight, float* loss_out, gps_stream_t stream);

/* Adam (torch formula, "Libtorch"; per-group learning rates of App. C).        */
typedef struct {
  float lr_xyz;     /* 1.6e-4 */
  float lr_sh0;     /* 2.5e-3 */
  float lr_shrest;  /* 5e-4   */
  float lr_opacity; /* 5e-2   */
  float lr_scale;   /* 5e-3   */
  float lr_rot;     /* 1e-3   */
  float beta1;      /* 0.9    (R-ADAM) */
  float beta2;      /* 0.999  */
  float eps;        /* 1e-15  */
} gps_adam_config;

/* First and second moments, same shape (n, sh_degree) as the parameters; `step` is the number
 * of Adam steps taken so far (host-side; incremented by gps_refine_step / gps_adam_step).     */
typedef struct {
  gps_gaussians m;
  gps_gaussians v;
  int64_t step;
} gps_adam_state;

/* One training view: pose, intrinsics, its cached SDF render ("recording the
 * SDF-rendered color images and depth maps to avoid repeated raycast") and the target C_k.    */
typedef struct {
  gps_intrinsics K;
  gps_pose T;
  const float* sdf_depth;     /* f32[H*W]   */
  const float* sdf_color;     /* f32[H*W*3] */
  const uint8_t* target_rgba; /* u8[H*W*4]  */
} gps_view;

size_t gps_refine_workspace_size(int64_t n, const gps_intrinsics* K /*host, largest view*/,
                                 const gps_render_config* cfg /*host*/, int32_t n_views);

/* gps_refine_step -- one Gaussian optimisation iteration (Eq. 7):
 * for each view: render (as gps_render) -> L1 loss and its gradient -> exact analytic backward
 * to every raw parameter (R-GRAD); gradients of all views are summed; then one dense Adam
 * update of every Gaussian (R-ADAM), state->step incremented on the host.
 * loss_out (nullable device f32 scalar) <- sum over views of the per-view mean L1.
 * grad_out (nullable; test hook) <- the summed raw-parameter gradient used by Adam, in the
 * parameter SoA layout (n and sh_degree must equal g's).                                      */
gps_status gps_refine_step(gps_gaussians* g, gps_adam_state* state /*host struct*/,
                           const gps_view* views /*host array*/, int32_t n_views,
                           const gps_render_config* rcfg /*host*/,
                           const gps_adam_config* acfg /*host*/, void* ws, size_t ws_bytes,
                           float* loss_out, const gps_gaussians* grad_out, gps_stream_t stream);

/* gps_refine_round -- a refinement round: n_iter gps_refine_step calls in
 * one host call, iteration i over the views_per_iter views views[iter_views[i*views_per_iter + j]]
 * (iter_views: host array of n_iter*views_per_iter indices into views; out-of-range -> error,
 * nothing launched).  Same kernels, same order, same results as the n_iter calls; state->step
 * += n_iter; loss_out <- the last iteration's loss.  use_graph != 0: the round's launches are
 * stream-captured and replayed as one CUDA graph (one executable graph per workspace, updated in
 * place while the round's launch structure is unchanged; freed at process exit).  Graphs are
 * skipped on the legacy/per-thread default streams, inside a caller's own capture and while the
 * event profiler is enabled.  On an error no iteration is launched and state->step is unchanged
 * (with use_graph; without it, the iterations before the failing one have been enqueued).     */
gps_status gps_refine_round(gps_gaussians* g, gps_adam_state* state /*host struct*/,
                            const gps_view* views /*host array*/, int32_t n_views,
                            const int32_t* iter_views /*host*/, int32_t views_per_iter, int32_t n_iter,
                            const gps_render_config* rcfg /*host*/, const gps_adam_config* acfg /*host*/,
                            void* ws, size_t ws_bytes, float* loss_out, int32_t use_graph,
                            gps_stream_t stream);

/* gps_adam_step -- the Adam update of gps_refine_step alone, on caller-given gradients
 * `grad` (parameter SoA layout).  Used to test the optimiser on identical gradients.          */
gps_status gps_adam_step(gps_gaussians* g, gps_adam_state* state /*host struct*/,
                         const gps_gaussians* grad, const gps_adam_config* acfg /*host*/,
                         gps_stream_t stream);

/* ---- Gaussian adding and removal (readings R-NORMAL .. R-REMOVE,
 * DESIGN.md §3) ------------------------------------------------------------------------------ */

/* gps_vertex_normals -- the raycast normal map N* from the raycast vertex map V* (P:106):
 * N(u,v) = normalise((V(u+1,v) - V(u-1,v)) x (V(u,v+1) - V(u,v-1))) turned towards the camera
 * centre T.t; 0 where the pixel or one of its 4 neighbours is a miss (sdf_depth = 0), on the
 * image border, or where the cross product vanishes (R-NORMAL).
 * vertex f32[H*W*3] (world, as gps_raycast's vertex_out), normal_out f32[H*W*3].              */
gps_status gps_vertex_normals(const gps_intrinsics* K /*host*/, const gps_pose* T /*host*/,
                              const float* sdf_depth, const float* vertex, float* normal_out,
                              gps_stream_t stream);
/* The same with the camera centre read from a device pose (see gps_fuse_dpose).             */
gps_status gps_vertex_normals_dpose(const gps_intrinsics* K /*host*/, const gps_pose* T_dev /*device*/,
                                    const float* sdf_depth, const float* vertex, float* normal_out,
                                    gps_stream_t stream);

typedef struct {
  float delta_c;      /* colour-error threshold of Eq. 6 [0.05]                         */
  float delta_w;      /* Gaussian-weight threshold of Eq. 6 [4]                         */
  float sample_frac;  /* fraction of M sampled [0.25]                                   */
  float opacity_init; /* initial opacity [0.5]                                          */
  float scale_max;    /* truncation of the kNN scale (App. A) [0.1]                       */
  float knn_cell;     /* cell edge of the kNN grid, metres (accelerator only) [0.01]            */
  uint32_t seed;      /* sampling seed (R-SAMPLE): the caller varies it per round               */
  int32_t reserved;   /* 0                                                                      */
} gps_add_config;

size_t gps_add_workspace_size(const gps_intrinsics* K /*host*/);

/* gps_add_gaussians_sync -- Gaussian adding (Eq. 6, App. A):
 * M = {u : sdf_depth > 0, normal != 0, max_ch |C*_ch - C_k,ch| > delta_c, W_G < delta_W}
 * (fp32 decisions, R-ADD-MASK); a seeded counter hash keeps sample_frac of M (R-SAMPLE); each
 * kept pixel u, in row-major order, becomes Gaussian n + i with p = V*(u), SH0 = (C_k(u) - 0.5)/C0
 * (higher SH 0), opacity_init, the rotation taking e_z to N*(u), and log-scales
 * (s1, s1, 0.1 s1), s1 = min(scale_max, RMS distance to the 3 nearest other vertices of M)
 * (R-KNN).  Their Adam moments are zeroed (state->step is global and unchanged).
 * g: caller SoA whose arrays hold `capacity` Gaussians; g->n is updated on the host.
 * Synchronises once (the counts).  *n_added (host) = Gaussians written; *n_candidates (host,
 * nullable) = sampled pixels (> n_added only when capacity ran out).                         */
gps_status gps_add_gaussians_sync(gps_gaussians* g, int64_t capacity, gps_adam_state* state /*host*/,
                                  const gps_intrinsics* K /*host*/, const float* sdf_depth,
                                  const float* vertex, const float* normal, const float* cstar,
                                  const float* weight, const uint8_t* target_rgba,
                                  const gps_add_config* cfg /*host*/, void* ws, size_t ws_bytes,
                                  int64_t* n_added /*host*/, int64_t* n_candidates /*host*/,
                                  gps_stream_t stream);

typedef struct {
  float sigma_min;  /* delta_sigma of Eq. 8 [0.005]                                    */
  float scale_max;  /* delta_s_max [0.1]                                                        */
  float scale_min;  /* delta_s_min [0.003]                                                      */
  int32_t reserved; /* 0                                                                        */
} gps_remove_config;

size_t gps_remove_workspace_size(int64_t n, int32_t sh_degree);

/* gps_remove_gaussians_sync -- Gaussian removal (Eq. 8): deletes every Gaussian with
 * sigmoid(o) < sigma_min, max_k exp(ls_k) > scale_max or max_k exp(ls_k) < scale_min, decided in
 * fp32 on the raw parameters against thresholds rounded once from double (R-REMOVE).  The
 * survivors keep their order; their Adam moments move with them.  g->n is updated on the host.
 * Synchronises once.  *n_removed (host) = Gaussians deleted.                                 */
gps_status gps_remove_gaussians_sync(gps_gaussians* g, gps_adam_state* state /*host*/,
                                     const gps_remove_config* cfg /*host*/, void* ws, size_t ws_bytes,
                                     int64_t* n_removed /*host*/, gps_stream_t stream);

/* ---- camera tracking (readings R-ICP-*) ---------------- */
typedef struct {
  int32_t levels;        /* pyramid levels, 1..4 [3] ("a resolution hierarchy")           */
  int32_t iters[4];      /* Gauss-Newton steps per level, finest first [10, 5, 4]              */
  float dist_max;        /* correspondence gate, metres [0.1] (R-ICP-GATE)                     */
  float angle_max_deg;   /* normal-angle gate, degrees [30]                                     */
  float depth_min, depth_max; /* valid raw depth range, metres [0.1, 10]                         */
  float eps;             /* a level stops when |xi| < eps [1e-6]                                */
  float min_inlier_frac; /* converged needs this inlier fraction at the end [0.1]               */
  int32_t fallback;      /* 1: a frame that does not converge gets T_init (gps_track_async: T_fail
                          *    if given) as its pose in result.T; R64/t64 still hold the iterate
                          *    -- R-ICP-FAIL [1]; 0: result.T is the iterate whatever the outcome */
  float min_inlier_px_frac; /* converged also needs inliers >= this fraction of the frame's
                             * pixels [0.05] (R-ICP-FAIL: a near-empty depth frame is a failure) */
  float min_pivot_ratio; /* ... and the last system's pivot_ratio >= this [1e-3] (R-ICP-FAIL:
                          * an ill-conditioned system slides along its weak direction)         */
  int32_t filter_radius; /* bilateral pre-filter of the depth used for tracking (KinectFusion's
                          * measurement filter; fusion keeps the raw depth), window radius in
                          * pixels, 0 = off [0; the mapping pipeline tracks with 3] (R-ICP-FILT) */
  float filter_sigma_s;  /* spatial sigma, pixels [4.5]                                         */
  float filter_sigma_r;  /* range sigma, metres [0.03]                                          */
} gps_icp_config;

typedef struct {
  gps_pose T;            /* tracked camera -> world pose: fp32 copy of R64, t64 (or T_init, see
                          * gps_icp_config.fallback)                                           */
  double R64[9], t64[3]; /* the pose as iterated on the device (fp64)                           */
  double energy;         /* sum of squared point-to-plane residuals of the last step's inliers  */
  int32_t inliers, valid;/* last step's inliers / current pixels with a normal                  */
  int32_t steps;         /* Gauss-Newton steps taken                                            */
  int32_t degenerate;    /* a step had < 6 inliers or a rank-deficient system (no update)       */
  int32_t converged;     /* !degenerate, inliers/valid >= min_inlier_frac,
                          * inliers >= min_inlier_px_frac * width * height and
                          * pivot_ratio >= min_pivot_ratio                                      */
  float inlier_frac;
  float pivot_ratio;     /* smallest Cholesky pivot / largest diagonal of the last step's system
                          * (conditioning: ~1 well constrained, -> 0 sliding along a degenerate
                          * direction)                                                        */
  int32_t reserved;
} gps_track_result;

size_t gps_track_workspace_size(const gps_intrinsics* K /*host*/, int32_t levels);

/* gps_track_sync -- Eq. 5: frame-to-model point-to-plane ICP of the depth frame
 * (u16, raw / depth_scale metres) against the model maps V*_{k-1}, N*_{k-1} (world, f32[H*W*3],
 * as gps_raycast's vertex_out and gps_vertex_normals) raycast from T_model, starting at T_init.
 * Coarse to fine over a depth pyramid (R-ICP-PYR); each step associates every current pixel with
 * the model pixel its point projects to in the T_model camera (R-ICP-ASSOC, the reading of the
 * garbled projection of P:113), gates it (R-ICP-GATE), and solves the linearised system for a
 * left-multiplied twist (R-ICP-GN).  The iteration runs on the device (pose in device memory);
 * synchronises once, at the end.  Degenerate geometry is reported in `out`, not as an error.   */
gps_status gps_track_sync(const gps_intrinsics* K /*host*/, const uint16_t* depth, float depth_scale,
                          const float* model_vertex, const float* model_normal,
                          const gps_pose* T_model /*host*/, const gps_pose* T_init /*host*/,
                          const gps_icp_config* cfg /*host*/, void* ws, size_t ws_bytes,
                          gps_track_result* out /*host*/, gps_stream_t stream);

/* gps_pose_extrapolate -- constant-velocity prediction of the next pose from the two previous
 * ones (R-ICP-FAIL): T_out = T_b * (T_a^-1 * T_b), i.e. the relative motion a -> b applied once
 * more in the camera frame, on the device in double (T_a^-1 = [R^T, -R^T t]), R re-orthonormalised
 * (Gram-Schmidt on its rows) before rounding to fp32 -- chained predictions would otherwise
 * amplify the inputs' fp32 departures from orthonormality.
 * All three poses in device memory; T_out may alias neither input.  The initial pose for the
 * next frame's gps_track_async.                                                              */
gps_status gps_pose_extrapolate(const gps_pose* T_a_dev, const gps_pose* T_b_dev, gps_pose* T_out_dev,
                                gps_stream_t stream);

/* gps_track_async -- gps_track_sync with every pose in device memory and no synchronisation:
 * the poses T_model_dev, T_init_dev and T_fail_dev (nullable: T_init; the pose a frame that does
 * not converge gets when cfg->fallback, e.g. gps_pose_extrapolate's prediction) are read on the
 * device (they may alias each other and T_out_dev); T_out_dev <- the tracked pose (fp32,
 * = result.T); result_dev (nullable, device) <- the whole gps_track_result.  The same kernels as gps_track_sync: for the same inputs both
 * produce bit-identical poses.  Errors: argument errors only (returned immediately).           */
gps_status gps_track_async(const gps_intrinsics* K /*host*/, const uint16_t* depth, float depth_scale,
                           const float* model_vertex, const float* model_normal,
                           const gps_pose* T_model_dev, const gps_pose* T_init_dev,
                           const gps_pose* T_fail_dev, const gps_icp_config* cfg /*host*/, void* ws,
                           size_t ws_bytes, gps_pose* T_out_dev, gps_track_result* result_dev,
                           gps_stream_t stream);

/* Synchronises `stream` and reports the pair count K of the last render held in `ws`, the pair
 * capacity, and the number of Gaussians that survived culling.  Returns
 * GPS_ERR_WORKSPACE_TOO_SMALL if K exceeded the capacity (that render dropped pairs).        */
gps_status gps_render_stats_sync(const void* ws, gps_stream_t stream, int64_t* n_pairs /*host*/,
                                 int64_t* capacity /*host*/, int64_t* n_visible /*host*/);

/* ---- test / debug hooks (synchronise; never on the timed path) --------------------------- */

/* Copies up to `cap` allocated blocks (any order): coords i32[cap*3], and if voxels != NULL
 * their 512 voxels each (8-byte voxels, voxel (i,j,k) of a block at index i + 8j + 64k).
 * *n (host) receives the number of allocated, backed blocks (may exceed cap).                */
gps_status gps_debug_export_blocks_sync(const gps_volume* vol, gps_stream_t stream,
                                        int32_t* coords, void* voxels, int64_t cap,
                                        int64_t* n /*host*/);
/* Checks the tsdf apron invariant (every block's + face copy equals its owner
 * voxel, NaN where the owning block is unallocated) over all allocated blocks, looking owners up
 * in the hash table, and the raycast's per-sub-block counts of cells <= 0 (DESIGN.md §4.4 (iii))
 * against a recount; *n_bad (host) = apron cells that differ + blocks whose count is wrong.
 * Debug only.                                                                               */
gps_status gps_debug_apron_check_sync(const gps_volume* vol, gps_stream_t stream, int64_t* n_bad /*host*/);
/* Checks the hash table, pool and neighbour tables (the lock-free insert of gps_fuse and the
 * neighbour linking): every occupied slot's pool block carries the slot's key,
 * every pool block is found at its key, each block's 8 +neighbour and 8 -neighbour entries equal
 * a fresh lookup, dense-grid cells of allocated blocks hold their pool index, and the occupied
 * slots number exactly the pool blocks (no key inserted twice).  *n_bad (host) = violations.
 * Debug only (synchronises).                                                                */
gps_status gps_debug_hash_check_sync(const gps_volume* vol, gps_stream_t stream, int64_t* n_bad /*host*/);
/* Checked build (libgps_checked.so, compiled with -DGPS_CHECKED): the hot
 * kernels evaluate their index bounds and record each failed kind as one bit of a device word
 * without stopping: bit 0 pool block index, 1 plane offset, 2 pixel, 3 hash slot / grid cell,
 * 4 visible list, 5 range tile, 6 neighbour entry, 7 sub-block count byte leaving [0, 125],
 * 16 pair index, 17 tile, 18 Gaussian index, 19 a list entry outside its tile's range,
 * 20 shared-memory staging index, 21 fused-Adam element, 22 long-list partial slot,
 * 24 adding / removal index, 28 tracking index.  Synchronises the device, then *word (host)
 * receives the OR of the bits since the last call (which clears them) and *checked (host,
 * nullable) 1 for the checked build, 0 for the production build (whose word stays 0).       */
gps_status gps_debug_check_word_sync(int64_t* word /*host*/, int32_t* checked /*host*/);
/* Enqueues one kernel whose bound check fails for bit `bit` (0..63): in the checked build the next
 * gps_debug_check_word_sync reports that bit (the mechanism's self-test); a no-op otherwise.  */
gps_status gps_debug_check_selftest(int32_t bit, gps_stream_t stream);
/* Runs the forward of gps_render (16x16 tiles) in its instrumented form and counts, over all
 * pixels, the pixel-entry pairs whose membership q was evaluated (*evaluated: the entry survived
 * the warp's strip test and the pixel's Eq. 1 depth indicator) and those accepted (*accepted:
 * they contribute alpha to Eq. 2).  E and A of SURVEY §8(d).  Debug only; synchronises.      */
gps_status gps_debug_render_counts_sync(const gps_gaussians* g, const gps_intrinsics* K /*host*/,
                                        const gps_pose* T /*host*/, const float* sdf_depth,
                                        const float* sdf_color, const gps_render_config* cfg /*host*/,
                                        void* ws, size_t ws_bytes, int64_t* evaluated /*host*/,
                                        int64_t* accepted /*host*/, gps_stream_t stream);
/* Runs gps_raycast for (K, T) into temporary buffers while marking every tsdf voxel the march
 * reads; *unique_voxels (host) = their number.  Measures the raycast roofline's unit count
 * (4 bytes per unique voxel read + 16 bytes of output per pixel).  Allocates; debug only.     */
gps_status gps_debug_raycast_footprint_sync(const gps_volume* vol, const gps_intrinsics* K /*host*/,
                                            const gps_pose* T /*host*/, gps_stream_t stream,
                                            int64_t* unique_voxels /*host*/);
/* Copies the block coords marked visible by the last gps_fuse (any order).                  */
gps_status gps_debug_export_visible_sync(const gps_volume* vol, gps_stream_t stream,
                                         int32_t* coords, int64_t cap, int64_t* n /*host*/);
/* Copies the per-tile Gaussian lists of the last render in `ws`: values u32[cap] (Gaussian
 * indices, concatenated tile lists in tile-id order, each ascending by (depth bits, index)),
 * ranges u32[2*n_tiles] ([start,end) per tile, row-major tile ids).  *K (host) = total pairs.
 * With tile_depth_precull the ranges are the truncated ones.                                  */
gps_status gps_debug_render_lists_sync(const void* ws, gps_stream_t stream, uint32_t* values,
                                       int64_t cap, uint32_t* ranges, int64_t* K /*host*/);

/* ---- measurement hooks ------------------------------------------------------------------- */
/* gps_profile_enable(1) starts a fresh session in which every kernel launch of the library is
 * bracketed by two CUDA events recorded on its launch stream (0 stops recording).  Host-side
 * cost: two cudaEventRecord per launch.  gps_profile_read_sync synchronises the recorded events
 * and writes, per kernel id, the summed device time in ms and the launch count; `names`
 * (host, names_cap bytes) receives "k_alloc;k_integrate;..." in id order.  Returns the number
 * of kernel ids.                                                                              */
void gps_profile_enable(int on);
int gps_profile_read_sync(char* names /*host*/, int names_cap, double* total_ms /*host*/,
                          int64_t* launches /*host*/, int cap);
/* The session's per-launch timeline: for each launch in enqueue order its kernel id (the index
 * into gps_profile_read_sync's names) and its start / end in ms from the session's first event
 * (host arrays of `cap`); returns the number of launches (synchronises).  Concurrent streams'
 * launches overlap in this timeline as they did on the device (debug).                      */
int64_t gps_profile_timeline_sync(int32_t* ids /*host*/, double* t0_ms /*host*/, double* t1_ms /*host*/,
                                  int64_t cap);

const char* gps_status_string(gps_status s);
const char* gps_last_error(void); /* thread-local; "" if none */
int gps_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* GPS_H_ */
