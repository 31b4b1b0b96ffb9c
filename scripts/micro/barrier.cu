// Micro-benchmark: grid-wide barrier variants on a persistent cooperative grid
// (296 CTAs x 512 threads on B200).  Dev helper, not part of the product.
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

struct Bar {
  unsigned count;
  unsigned pad0[31];
  unsigned gen;
  unsigned pad1[31];
  unsigned grp[64 * 32];  // group counters, one per 128-byte line
};

__device__ __forceinline__ unsigned ld_acq(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned ld_rlx(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned atom_add_acqrel(unsigned* p, unsigned v) {
  unsigned old;
  asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ void st_rel(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// flat: one arrival per CTA
__device__ void bar_flat(Bar* b, unsigned& gen) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned g = gen;
    if (atom_add_acqrel(&b->count, 1u) == gridDim.x - 1) {
      b->count = 0;
      st_rel(&b->gen, g + 1);
    } else {
      while (ld_acq(&b->gen) == g) {}
    }
  }
  gen++;
  __syncthreads();
}

// two-level: groups of GS CTAs
template <int GS>
__device__ void bar_hier(Bar* b, unsigned& gen) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned g = gen;
    const unsigned grp = blockIdx.x / GS;
    const unsigned ngrp = (gridDim.x + GS - 1) / GS;
    const unsigned gsz = min((unsigned)GS, gridDim.x - grp * GS);
    bool released = false;
    if (atom_add_acqrel(&b->grp[grp * 32], 1u) == gsz - 1) {
      b->grp[grp * 32] = 0;
      if (atom_add_acqrel(&b->count, 1u) == ngrp - 1) {
        b->count = 0;
        st_rel(&b->gen, g + 1);
        released = true;
      }
    }
    if (!released)
      while (ld_acq(&b->gen) == g) {}
  }
  gen++;
  __syncthreads();
}

template <int MODE>
__global__ void __launch_bounds__(512, 2) k_bar(Bar* b, int iters, unsigned long long* out) {
  unsigned gen = ld_rlx(&b->gen);
  __syncthreads();
  const unsigned long long t0 = clock64();
  for (int i = 0; i < iters; i++) {
    if (MODE == 0) cg::this_grid().sync();
    else if (MODE == 1) bar_flat(b, gen);
    else if (MODE == 2) bar_hier<8>(b, gen);
    else if (MODE == 3) bar_hier<16>(b, gen);
    else bar_hier<37>(b, gen);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = clock64() - t0;
}

int main() {
  Bar* b;
  unsigned long long* out;
  cudaMalloc(&b, sizeof(Bar));
  cudaMemset(b, 0, sizeof(Bar));
  cudaMallocManaged(&out, 8);
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int iters = 20000;
  const char* names[] = {"cg grid sync", "flat acq/rel", "hier 8", "hier 16", "hier 37"};
  void* fns[] = {(void*)k_bar<0>, (void*)k_bar<1>, (void*)k_bar<2>, (void*)k_bar<3>, (void*)k_bar<4>};
  for (int rep = 0; rep < 2; rep++)
    for (int m = 0; m < 5; m++) {
      int it = iters;
      void* args[] = {&b, &it, &out};
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0); cudaEventCreate(&e1);
      cudaEventRecord(e0);
      cudaError_t e = cudaLaunchCooperativeKernel(fns[m], dim3(2 * nsm), dim3(512), args, 0, 0);
      cudaEventRecord(e1);
      cudaDeviceSynchronize();
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      printf("%-14s err=%d  %.3f us/barrier (events), %.3f us (clock64 @ %d kHz)\n", names[m], (int)e,
             ms * 1e3 / iters, (double)out[0] / iters / (clk / 1e3), clk);
    }
  return 0;
}
