// common.cuh -- shared device/host helpers of libgps (sm_100a).  Nothing here is shared with
// the CPU oracle (oracle/oracle.c); the two implement DESIGN.md §4 independently.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <string>

#include "gps.h"

namespace gps {

// ---- error plumbing ------------------------------------------------------------------------
void set_error(const std::string& msg);
gps_status cuda_fail(const char* where, cudaError_t e);
#define GPS_CHECK_LAUNCH(where)                                    \
  do {                                                             \
    cudaError_t e__ = cudaGetLastError();                          \
    if (e__ != cudaSuccess) return ::gps::cuda_fail(where, e__);   \
  } while (0)
#define GPS_CHECK_CUDA(call)                                       \
  do {                                                             \
    cudaError_t e__ = (call);                                      \
    if (e__ != cudaSuccess) return ::gps::cuda_fail(#call, e__);   \
  } while (0)
gps_status invalid(const std::string& msg);

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// ---- checked build (the bounds/race evidence compute-sanitizer cannot give on this pool) -----
// Built with -DGPS_CHECKED (build.py --checked -> libgps_checked.so), every GPS_DCHECK(cond, bit)
// in a hot kernel evaluates its bound and, when it fails, sets `bit` in the translation unit's
// device check word (GPS_CHK_VAR, one per .cu: no relocatable device code needed) without
// stopping the kernel; gps_debug_check_word_sync ORs and clears the words.  In the production
// build the macro is empty.  Bits: include/gps.h (gps_debug_check_word_sync).
#ifdef GPS_CHECKED
#define GPS_DCHECK(cond, bit)                                                      \
  do {                                                                             \
    if (!(cond)) atomicOr(&GPS_CHK_VAR, 1ull << (bit));                            \
  } while (0)
#else
#define GPS_DCHECK(cond, bit) \
  do {                        \
  } while (0)
#endif
enum CheckBit {
  CHK_POOL = 0,       // a pool block index outside [0, n_blocks)
  CHK_PLANE = 1,      // a tsdf/rgbw plane offset outside its block
  CHK_PIXEL = 2,      // a pixel index outside the image
  CHK_SLOT = 3,       // a hash slot or dense-grid cell outside its table
  CHK_VISLIST = 4,    // a visible-list index at or beyond max_blocks
  CHK_RANGE_TILE = 5, // a range-image tile outside the image's tiles
  CHK_NBR = 6,        // a neighbour-table entry outside [-1, n_blocks)
  CHK_SUBNEG = 7,     // a sub-block count leaving [0, 125] (byte borrow)
  CHK_PAIR = 16,      // a (tile, Gaussian) pair index at or beyond the capacity
  CHK_TILE = 17,      // a tile index outside the image's tiles
  CHK_GAUSS = 18,     // a Gaussian index at or beyond n
  CHK_LIST = 19,      // a tile list range that is not ordered / inside the pair array
  CHK_SMEM = 20,      // a shared-memory staging index beyond its array
  CHK_ADAM = 21,      // a fused-Adam element outside its chunk slice
  CHK_SPLIT = 22,     // a long-list partial slot or chunk outside its table
  CHK_ADD = 24,       // adding / removal: an index outside its array
  CHK_TRACK = 28      // tracking: a pixel or partial-sum index outside its array
};
unsigned long long check_word_take_volume();
unsigned long long check_word_take_render();
unsigned long long check_word_take_adding();
unsigned long long check_word_take_tracking();
inline cudaStream_t as_stream(gps_stream_t s) { return reinterpret_cast<cudaStream_t>(s); }

// ---- prescribed fp32 arithmetic: never contracted into FMA ------------------
__device__ __forceinline__ float pmul(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float padd(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float psub(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ float pdiv(float a, float b) { return __fdiv_rn(a, b); }
__device__ __forceinline__ float psqrt(float a) { return __fsqrt_rn(a); }
// ((a0*b0 + a1*b1) + a2*b2), each product and sum rounded separately
__device__ __forceinline__ float pdot3(float a0, float b0, float a1, float b1, float a2, float b2) {
  return padd(padd(pmul(a0, b0), pmul(a1, b1)), pmul(a2, b2));
}

// ---- voxel-block hash ----------------------------------------------------------
// Voxel: {f32 tsdf; u8 r, g, b, w}, block = 8^3 voxels, index i + 8j + 64k.  In HBM the pool is
// two planes: tsdf[block][512] (4 B; an unobserved voxel (w = 0) holds a quiet NaN, so the march
// reads only this plane and "valid" is "not NaN") and rgbw[block][512] (4 B).  Voxel is the
// interleaved form used by the debug export (NaN shown as the R-VOX initial tsdf 1).
struct __align__(8) Voxel {
  float tsdf;
  uint32_t rgbw;  // r | g<<8 | b<<16 | w<<24
};
constexpr uint64_t kEmptyKey = ~0ull;
constexpr uint32_t kBlockBits = 21;
constexpr uint32_t kBlockMask = (1u << kBlockBits) - 1u;

__host__ __device__ __forceinline__ uint64_t pack_block(int x, int y, int z) {
  return ((uint64_t)((uint32_t)x & kBlockMask) << 42) | ((uint64_t)((uint32_t)y & kBlockMask) << 21) |
         (uint64_t)((uint32_t)z & kBlockMask);
}
__host__ __device__ __forceinline__ int sext21(uint32_t v) {
  return (int)(v << 11) >> 11;
}
__host__ __device__ __forceinline__ void unpack_block(uint64_t k, int& x, int& y, int& z) {
  x = sext21((uint32_t)(k >> 42) & kBlockMask);
  y = sext21((uint32_t)(k >> 21) & kBlockMask);
  z = sext21((uint32_t)k & kBlockMask);
}
// spatial hash of the voxel-hashing family: primes 73856093, 19349669, 83492791
__host__ __device__ __forceinline__ uint32_t hash_block(int x, int y, int z) {
  return ((uint32_t)x * 73856093u) ^ ((uint32_t)y * 19349669u) ^ ((uint32_t)z * 83492791u);
}

struct VolumeCounters {
  uint32_t n_blocks;   // blocks handed out (may exceed max_blocks on overflow)
  uint32_t n_vis;      // visible slots this frame
  uint32_t overflow;   // sticky: budget, table or visible-list overflow
  uint32_t n_prev;     // n_blocks before the current frame's allocation
  unsigned long long vis_total;  // sum of n_vis over all integrations (measurement)
  unsigned long long upd_total;  // voxels updated over all integrations (measurement)
};

// tsdf plane layout of one block (cells x, y, z in [0, 8]; a coordinate 8 is the apron copy of a
// +neighbour's voxel): the cells with x < 8 as 9 planes x 9 rows of 8 floats -- every row is one
// 32-byte sector (the block stride, 736 floats, is a whole number of sectors) -- then the x = 8
// face, 9 x 9 floats, then 7 floats of padding.  The trilinear corners of a sample based at
// (lx, ly, lz) are at constant offsets {0, 8, 72, 80} from its base cell, and its x + 1 corners
// at the same offsets from lx + 1 (lx < 7) or at {0, 1, 9, 10} from face cell (ly, lz) (lx = 7).
constexpr int kTsdfSY = 8, kTsdfSZ = 72, kTsdfFace = 648, kTsdfBlock = 736;
__host__ __device__ __forceinline__ int tsdf_index(int x, int y, int z) {
  return x < 8 ? x + kTsdfSY * y + kTsdfSZ * z : kTsdfFace + y + 9 * z;
}

struct VolumeView {  // passed by value to kernels
  uint64_t* keys;
  int32_t* vals;  // pool block index, -1 = none
  uint32_t* stamp;
  float* tsdf;     // pool plane: tsdf[b * kTsdfBlock + tsdf_index(x, y, z)], NaN = unobserved;
                   // x, y, z in [0, 8]: the + faces (coordinate 8) are an apron copy of the
                   // +neighbours' voxels (NaN where the neighbour is unallocated), kept exact by
                   // k_apron after every integration
  uint32_t* rgbw;  // pool plane: r | g<<8 | b<<16 | w<<24
  int32_t* vis;  // visible slots
  uint64_t* bkeys;  // pool block index -> packed block key (for passes over all blocks)
  int32_t* nbr;     // pool block index -> 8 pool indices of the blocks at +(dx,dy,dz), dx,dy,dz in
                    // {0,1}, entry k = dx | dy<<1 | dz<<2 (entry 0 = itself; -1 = unallocated)
  int32_t* nbrm;    // the same for the blocks at -(dx,dy,dz): whose aprons a block's voxels feed
  uint64_t* subneg;  // pool block index -> for each 4^3 sub-block s (byte s = sx + 2sy + 4sz),
                     // the number of cells of its 5^3 corner region in the tsdf plane (cells
                     // [4sx, 4sx + 4] x ..., apron included) holding a value <= 0 (NaN never
                     // counts); kept exact by k_link (apron pull) and k_integrate (sign changes of
                     // updated voxels and their apron pushes).  A zero byte means every valid
                     // trilinear sample based in the sub-block is > 0, so the raycast cannot find
                     // a +->- bracket there (DESIGN.md §4.4 (iii))
  VolumeCounters* ctr;
  uint32_t slot_mask;
  uint32_t max_blocks;
  int32_t* grid;  // optional dense block-index grid (nullable), -1 = unallocated
  int gox, goy, goz, gdx, gdy, gdz;
};

// subneg bytes (one bit per sub-block, as 1 << 8s) whose 5^3 corner region holds plane cell
// (x, y, z), x, y, z in [0, 8]: along each axis cell 4 is shared by sub-blocks 0 and 1
__host__ __device__ __forceinline__ uint64_t cell_subs(int x, int y, int z) {
  const int mx = x == 4 ? 3 : (x < 4 ? 1 : 2), my = y == 4 ? 3 : (y < 4 ? 1 : 2), mz = z == 4 ? 3 : (z < 4 ? 1 : 2);
  uint64_t w = 0;
#pragma unroll
  for (int s = 0; s < 8; ++s)
    if (((mx >> (s & 1)) & (my >> ((s >> 1) & 1)) & (mz >> (s >> 2))) & 1) w |= 1ull << (8 * s);
  return w;
}

// find a block: returns its pool index, or -1 if unallocated / unbacked
__device__ __forceinline__ int32_t find_block(const VolumeView& v, int x, int y, int z) {
  const uint64_t key = pack_block(x, y, z);
  uint32_t h = hash_block(x, y, z) & v.slot_mask;
  for (uint32_t probe = 0; probe <= v.slot_mask; ++probe) {
    const uint64_t k = __ldg(&v.keys[h]);
    if (k == key) return __ldg(&v.vals[h]);
    if (k == kEmptyKey) return -1;
    h = (h + 1) & v.slot_mask;
  }
  return -1;
}

// pool index of a block, through the dense grid when the block lies inside it
__device__ __forceinline__ int32_t find_block_fast(const VolumeView& v, int x, int y, int z) {
  const unsigned ix = (unsigned)(x - v.gox), iy = (unsigned)(y - v.goy), iz = (unsigned)(z - v.goz);
  if (v.grid && ix < (unsigned)v.gdx && iy < (unsigned)v.gdy && iz < (unsigned)v.gdz)
    return __ldg(&v.grid[(iz * (unsigned)v.gdy + iy) * (unsigned)v.gdx + ix]);  // <= 2^30 cells (validated)
  return find_block(v, x, y, z);
}

}  // namespace gps

// the opaque handle of the C ABI
struct gps_volume {
  gps_volume_config cfg;
  gps::VolumeView view;
  uint32_t frame;
  int device;
};
