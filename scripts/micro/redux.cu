// micro: latency of warp-collective primitives on sm_100a (dev helper)
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(unsigned* out, long long* t, int mode) {
  unsigned v = threadIdx.x * 2654435761u + 12345u;
  __shared__ int sc[32];
  sc[threadIdx.x & 31] = 0;
  __syncthreads();
  long long t0 = clock64();
  if (mode == 0) {
    for (int i = 0; i < 1000; i++) v = __reduce_min_sync(0xffffffffu, v + i) + threadIdx.x;
  } else if (mode == 1) {
    for (int i = 0; i < 1000; i++) v = __ballot_sync(0xffffffffu, (v + i) & 1) + threadIdx.x;
  } else if (mode == 2) {
    for (int i = 0; i < 1000; i++) v = __shfl_xor_sync(0xffffffffu, v + i, 1) + threadIdx.x;
  } else if (mode == 3) {
    for (int i = 0; i < 1000; i++) {
      unsigned m = v + i;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) m = min(m, __shfl_xor_sync(0xffffffffu, m, o));
      v = m + threadIdx.x;
    }
  } else if (mode == 4) {
    for (int i = 0; i < 1000; i++) { atomicAdd(&sc[(v + i) & 31], 1); __syncwarp(); v += sc[threadIdx.x & 31]; }
  } else if (mode == 5) {
    if (threadIdx.x < 32) {  // inside a warp-uniform branch the compiler cannot prove
      for (int i = 0; i < 1000; i++) v = __reduce_min_sync(0xffffffffu, v + i) + threadIdx.x;
    }
  }
  long long t1 = clock64();
  out[threadIdx.x] = v;
  if (threadIdx.x == 0) t[mode] = t1 - t0;
}
int main() {
  unsigned* o; long long* t;
  cudaMalloc(&o, 4096); cudaMalloc(&t, 64);
  const char* names[] = {"reduce_min_sync", "ballot", "shfl_xor", "shfl-tree min", "smem atomic+syncwarp+lds", "reduce_min in branch"};
  for (int m = 0; m < 6; m++) {
    k<<<1, m == 5 ? 64 : 32>>>(o, t, m);
    cudaDeviceSynchronize();
    long long h[8]; cudaMemcpy(h, t, 64, cudaMemcpyDeviceToHost);
    printf("%-28s %.1f cycles/iter\n", names[m], h[m] / 1000.0);
  }
  return 0;
}
