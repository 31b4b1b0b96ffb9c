// Run setup on the device: the filling-rate ranking of the pixels.
//
// ext = lexsort((id, -dist_from_c)) (reference strategies.py:109-116): pixels
// by decreasing distance from the centroid, ties by increasing id; rank[v] =
// position of v in ext.  Done with one 64-bit radix sort of
// (~distance bits << 32 | id) -- non-negative floats order like their bit
// patterns, so ascending keys = decreasing distance, then increasing id --
// instead of a host sort, so the run's setup never waits for the host.
#include <cub/device/device_radix_sort.cuh>

#include "gp_kernels.h"

namespace gp {

__global__ void k_ext_keys(const float* dfc, int N, unsigned long long* keys) {
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < N; v += gridDim.x * blockDim.x)
    keys[v] = ((unsigned long long)(~__float_as_uint(dfc[v])) << 32) | (unsigned)v;
}

__global__ void k_ext_rank(const unsigned long long* sorted, int N, int* ext, int* rank) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < N; i += gridDim.x * blockDim.x) {
    const int v = (int)(sorted[i] & 0xFFFFFFFFull);
    ext[i] = v;
    rank[v] = i;
  }
}

// Extrema key (strategies.py:203-210): gs[v] = first position in ext of v's
// distance class (pixels of equal dist_from_c are consecutive in ext).  One
// CTA: per-thread segments, a max-scan of class starts, a block scan of the
// segment maxima.
__global__ void __launch_bounds__(1024) k_group_start(const float* dfc, const int* ext, int N, int* gs) {
  __shared__ int segmax[1024];
  const int tid = threadIdx.x, nt = blockDim.x;
  const int seg = (N + nt - 1) / nt, i0 = min(N, tid * seg), i1 = min(N, i0 + seg);
  int run = -1;
  for (int i = i0; i < i1; i++)
    if (i == 0 || __float_as_uint(dfc[ext[i]]) != __float_as_uint(dfc[ext[i - 1]])) run = i;
  segmax[tid] = run;
  __syncthreads();
  for (int o = 1; o < nt; o <<= 1) {  // inclusive max-scan over the segments
    const int x = tid >= o ? segmax[tid - o] : -1;
    __syncthreads();
    segmax[tid] = max(segmax[tid], x);
    __syncthreads();
  }
  int cur = tid ? segmax[tid - 1] : -1;
  for (int i = i0; i < i1; i++) {
    if (i == 0 || __float_as_uint(dfc[ext[i]]) != __float_as_uint(dfc[ext[i - 1]])) cur = i;
    gs[ext[i]] = cur;
  }
}

cudaError_t launch_group_start(const float* dfc, const int* ext, int N, int* gs, cudaStream_t st) {
  k_group_start<<<1, 1024, 0, st>>>(dfc, ext, N, gs);
  return cudaGetLastError();
}

size_t ext_rank_temp_bytes(int N) {
  size_t bytes = 0;
  cub::DeviceRadixSort::SortKeys(nullptr, bytes, (const unsigned long long*)nullptr,
                                 (unsigned long long*)nullptr, N);
  return bytes;
}

cudaError_t launch_ext_rank(const float* dfc, int N, unsigned long long* keys2, void* temp,
                            size_t temp_bytes, int* ext, int* rank, cudaStream_t st) {
  const int blocks = (N + 255) / 256;
  k_ext_keys<<<blocks, 256, 0, st>>>(dfc, N, keys2);
  cudaError_t e = cub::DeviceRadixSort::SortKeys(temp, temp_bytes, keys2, keys2 + N, N, 0, 64, st);
  if (e != cudaSuccess) return e;
  k_ext_rank<<<blocks, 256, 0, st>>>(keys2 + N, N, ext, rank);
  return cudaGetLastError();
}

}  // namespace gp
