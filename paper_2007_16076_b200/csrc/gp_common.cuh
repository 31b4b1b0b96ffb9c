// Shared device helpers for the geopairs B200 kernels.
//
// Pixel graph: H x W image, row-major pixel ids, 8- or 4-connectivity.
// Neighbour positions are encoded by their index k in the 3x3 window
// (k = (dr+1)*3 + (dc+1), k != 4), visited in ascending k == ascending
// neighbour id, the order of the reference's lexsorted CSR
// (propagation.py:13,85).  A tree's parent link is stored as that code
// (one byte per pixel, GP_ROOT for roots): parent(v) = v + (k/3-1)*W + (k%3-1).
//
// Arithmetic: every distance is fp32.  Integer images (grey levels 1..255)
// stay exact: weights are integers <= 1020 and every geodesic distance of a
// <= 4096 x 4096 image stays below 2^24, so fp32 sums are exact and equal the
// reference's int64 values (checked on the host before a run).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace gp {

enum Metric : int { kL1 = 0, kSum = 1, kMean = 2 };
enum Strategy : int { kNaive = 0, kFillingRate = 1, kExtrema = 2 };

constexpr uint8_t GP_ROOT = 0xFF;
constexpr uint32_t INF_BITS = 0x7F800000u;  // +inf; non-negative floats order as uint32
constexpr unsigned long long KEY_NONE = ~0ull;

struct Grid {
  int H, W, N, conn, metric;
  uint32_t wmagic;  // floor(2^32 / W) + 1 (W > 1): exact v / W for v < 2^16
};

__host__ __device__ inline Grid make_grid(int H, int W, int conn, int metric) {
  Grid g{H, W, H * W, conn, metric, 0u};
  if (W > 1) g.wmagic = (uint32_t)((0x100000000ull / (unsigned long long)W) + 1ull);
  return g;
}

// row and column of pixel v (N <= 65536, so v * W < 2^32 and the
// multiply-high quotient is exact)
__device__ __forceinline__ void pix_rc(const Grid& g, int v, int& r, int& c) {
  r = g.W > 1 ? (int)__umulhi((uint32_t)v, g.wmagic) : v;
  c = v - r * g.W;
}

// scaled_weight (grid.py:146-154) in fp32, no contraction: SUM = 2*fl(a+b).
__device__ __forceinline__ float edge_w(int metric, float a, float b) {
  if (metric == kSum) return __fmul_rn(2.0f, __fadd_rn(a, b));
  if (metric == kMean) return __fadd_rn(a, b);
  return __fmul_rn(2.0f, fabsf(__fsub_rn(a, b)));
}

// Is window position k a neighbour under this connectivity?
__device__ __forceinline__ bool k_in_conn(int conn, int k) {
  return k != 4 && (conn == 8 || (k & 1));
}

// Neighbour of pixel (r, c) at window position k, or -1 if off-image.
__device__ __forceinline__ int nbr_at(const Grid& g, int r, int c, int k) {
  int rr = r + k / 3 - 1, cc = c + k % 3 - 1;
  if (rr < 0 || rr >= g.H || cc < 0 || cc >= g.W) return -1;
  return rr * g.W + cc;
}

__device__ __forceinline__ int parent_of(int v, uint8_t code, int W) {
  return code == GP_ROOT ? -1 : v + (code / 3 - 1) * W + (code % 3 - 1);
}

// Column layout of the mark bitmap.  Row v holds the mark bits of pairs
// (v, *).  Columns are ordered by 16x16 pixel tiles (tile-major, raster inside
// a tile) so that the bits of a compact pixel region -- a subtree, tested
// together by one warp -- share 32-byte sectors; one tile is one sector.
// Images narrower or shorter than 16 use plain raster columns.
struct MarkLayout {
  int N;          // pixels
  int H;          // image height
  int W;          // image width (tiling)
  int tiled;      // 16x16 tile order?
  int RW;         // 32-bit words per row
  int TWn;        // tiles per image row
  uint32_t magic; // floor(2^32 / W) + 1: exact c / W for c, W < 2^16
};

__host__ __device__ inline MarkLayout make_layout(int N, int H, int W) {
  MarkLayout L;
  L.N = N;
  L.H = H;
  L.W = W;
  L.tiled = (H >= 16 && W >= 16) ? 1 : 0;
  L.TWn = (W + 15) / 16;
  // tile columns must fit 16 bits (packed tree-store entries)
  if (L.tiled && (long long)((H + 15) / 16) * L.TWn * 256 > 65536) L.tiled = 0;
  L.RW = L.tiled ? ((H + 15) / 16) * L.TWn * 8 : (N + 31) / 32;
  L.magic = L.tiled ? (uint32_t)((0x100000000ull / (unsigned long long)W) + 1ull) : 0u;
  return L;
}

__device__ __forceinline__ uint32_t mcol(const MarkLayout& L, uint32_t c) {
  if (!L.tiled) return c;
  const uint32_t r = __umulhi(c, L.magic), cc = c - r * (uint32_t)L.W;
  return (((r >> 4) * (uint32_t)L.TWn + (cc >> 4)) << 8) + ((r & 15u) << 4) + (cc & 15u);
}

// inverse of mcol: pixel of a tiled column, -1 for padding columns
__device__ __forceinline__ int mcol_pixel(const MarkLayout& L, uint32_t ct) {
  if (!L.tiled) return ct < (uint32_t)L.N ? (int)ct : -1;
  const uint32_t tile = ct >> 8, within = ct & 255u;
  const uint32_t tr = tile / (uint32_t)L.TWn, tc = tile - tr * (uint32_t)L.TWn;
  const uint32_t r = tr * 16 + (within >> 4), c = tc * 16 + (within & 15u);
  if (r >= (uint32_t)L.H || c >= (uint32_t)L.W) return -1;
  return (int)(r * L.W + c);
}

__device__ __forceinline__ size_t mword(const MarkLayout& L, uint32_t row, uint32_t col_t) {
  return (size_t)row * L.RW + (col_t >> 5);
}

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

}  // namespace gp
