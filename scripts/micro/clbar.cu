// Cluster-barrier cost on B200 (2-CTA clusters, 1024 threads, one CTA per SM):
// cg::this_cluster().sync() (arrive.release + wait.acquire: MEMBAR.ALL.GPU +
// CCTL.IVALL) against arrive.relaxed + wait, with and without DSMEM traffic
// between barriers.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 clbar.cu
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

template <int MODE, int WORK>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(1024, 1) kbar(unsigned long long* out, int iters) {
  extern __shared__ unsigned sm[];
  cg::cluster_group cl = cg::this_cluster();
  unsigned* rem = cl.map_shared_rank(sm, cl.block_rank() ^ 1);
  sm[threadIdx.x] = 0;
  cl.sync();
  unsigned long long t0 = clock64();
  for (int i = 0; i < iters; i++) {
    if (WORK == 1) atomicAdd(&rem[threadIdx.x], 1u);
    if (WORK == 2) atomicAdd(&sm[threadIdx.x], 1u);
    if (MODE == 0) cl.sync();
    else asm volatile("barrier.cluster.arrive.relaxed.aligned;\nbarrier.cluster.wait.aligned;" ::: "memory");
  }
  unsigned long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = (t1 - t0) / iters;
}

template <int MODE, int WORK>
void run(const char* name) {
  unsigned long long* d;
  cudaMalloc(&d, 8);
  auto k = kbar<MODE, WORK>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  k<<<148, 1024, 200 * 1024>>>(d, 1000);
  k<<<148, 1024, 200 * 1024>>>(d, 1000);
  unsigned long long h = 0;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("%-40s %llu cycles per iteration (%s)\n", name, h, cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  run<0, 0>("cluster.sync");
  run<1, 0>("arrive.relaxed + wait");
  run<0, 1>("remote atomicAdd + cluster.sync");
  run<1, 1>("remote atomicAdd + relaxed");
  run<0, 2>("local atomicAdd + cluster.sync");
  run<1, 2>("local atomicAdd + relaxed");
  return 0;
}
