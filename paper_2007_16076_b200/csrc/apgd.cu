// APGD dump / load of the distance store (reference distances.py:149-177,
// SPEC.md:255): magic "APGD", version byte, u32 N, then N*N u64 LE values,
// all-ones for an unmarked entry.
//
// The conversion runs on the device, a block of rows at a time, so a dump or
// a load never materialises N^2 host temporaries (the reference builds the
// whole int64 grid, a uint64 copy and a bytes copy: >80 GiB at 256x256).
//   version 1 (reference): integer stores, u64 = the exact integer distance;
//   version 2 (additive, float stores): u64 = IEEE-754 binary64 bits of the
//             fp32 value (exact), same sentinel (a NaN pattern, unambiguous).
#include "gp_common.cuh"
#include "gp_kernels.h"

namespace gp {

constexpr unsigned long long APGD_SENTINEL = ~0ull;

// D rows [row0, row0 + nrows) -> u64 (row-major, n per row)
__global__ void k_apgd_dump(MarkLayout L, const float* D, const uint32_t* mark, long long row0,
                            long long nrows, int version, unsigned long long* out) {
  const long long n = L.N, total = nrows * n;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const uint32_t r = (uint32_t)(row0 + i / n), c = (uint32_t)(i % n);
    const uint32_t ct = mcol(L, c);
    const bool marked = (__ldg(&mark[mword(L, r, ct)]) >> (ct & 31)) & 1u;
    const float v = __ldg(&D[(size_t)r * n + c]);
    unsigned long long x = APGD_SENTINEL;
    if (marked) x = version == 1 ? (unsigned long long)(long long)v
                                 : (unsigned long long)__double_as_longlong((double)v);
    out[i] = x;
  }
}

// u64 rows -> D and mark bits (the rows' mark words were zeroed first); bad
// counts values a version-1 store cannot hold exactly (>= 2^24) or, for
// version 2, values that are not binary64 images of an fp32 number
__global__ void k_apgd_load(MarkLayout L, float* D, uint32_t* mark, long long row0, long long nrows,
                            int version, const unsigned long long* in, unsigned long long* bad) {
  const long long n = L.N, total = nrows * n;
  const long long stride = (long long)gridDim.x * blockDim.x;
  // whole warps iterate together (match_any below)
  for (long long b = blockIdx.x * (long long)blockDim.x + (threadIdx.x & ~31); b < total; b += stride) {
    const long long i = b + (threadIdx.x & 31);
    bool marked = false;
    size_t wi = ~(size_t)0;
    uint32_t bit = 0;
    if (i < total) {
      const uint32_t r = (uint32_t)(row0 + i / n), c = (uint32_t)(i % n);
      const unsigned long long x = in[i];
      marked = x != APGD_SENTINEL;
      float v = 0.0f;
      if (marked) {
        if (version == 1) {
          if (x >= (1ull << 24)) atomicAdd(bad, 1ull);
          v = (float)x;
        } else {
          const double d = __longlong_as_double((long long)x);
          v = (float)d;
          if ((double)v != d || !(v >= 0.0f)) atomicAdd(bad, 1ull);
        }
      }
      D[(size_t)r * n + c] = v;
      const uint32_t ct = mcol(L, c);
      wi = mword(L, r, ct);
      bit = 1u << (ct & 31);
    }
    const unsigned peers = __match_any_sync(0xffffffffu, marked ? (unsigned long long)wi : ~0ull);
    if (marked) {
      const uint32_t acc = __reduce_or_sync(peers, bit);
      if ((threadIdx.x & 31) == __ffs(peers) - 1) atomicOr(&mark[wi], acc);
    }
  }
}

// counts[r] = marked entries of row r minus the diagonal; filled += marks
__global__ void k_store_recount(MarkLayout L, const uint32_t* mark, int* cnt, unsigned long long* marks) {
  const int lane = threadIdx.x & 31;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int r = warp; r < L.N; r += nwarps) {
    unsigned c = 0;
    for (int w = lane; w < L.RW; w += 32) c += __popc(__ldg(&mark[(size_t)r * L.RW + w]));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if (lane == 0) {
      cnt[r] = (int)c - 1;
      atomicAdd(marks, (unsigned long long)c);
    }
  }
}

cudaError_t launch_apgd_dump(const MarkLayout& L, const float* D, const uint32_t* mark, long long row0,
                             long long nrows, int version, unsigned long long* out, cudaStream_t st) {
  k_apgd_dump<<<148 * 8, 256, 0, st>>>(L, D, mark, row0, nrows, version, out);
  return cudaGetLastError();
}

cudaError_t launch_apgd_load(const MarkLayout& L, float* D, uint32_t* mark, long long row0, long long nrows,
                             int version, const unsigned long long* in, unsigned long long* bad,
                             cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(mark + (size_t)row0 * L.RW, 0, (size_t)nrows * L.RW * 4, st);
  if (e != cudaSuccess) return e;
  k_apgd_load<<<148 * 8, 256, 0, st>>>(L, D, mark, row0, nrows, version, in, bad);
  return cudaGetLastError();
}

cudaError_t launch_store_recount(const MarkLayout& L, const uint32_t* mark, int* cnt,
                                 unsigned long long* marks, cudaStream_t st) {
  k_store_recount<<<148 * 4, 256, 0, st>>>(L, mark, cnt, marks);
  return cudaGetLastError();
}

}  // namespace gp
