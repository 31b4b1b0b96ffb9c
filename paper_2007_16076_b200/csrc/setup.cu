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
