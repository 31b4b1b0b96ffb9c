// K2 + K3 -- the device-resident commit loop of run_strategy
// (reference strategies.py:246-273), plus the distance-store kernels.
//
// One persistent cooperative kernel executes commit after commit without
// returning to the host:
//
//   fill   (K2)  every pixel v whose row is not yet full walks its ancestor
//                chain in the committed tree (byte parent codes) and, for each
//                unmarked pair (v,u), sets both mark bits, writes
//                D[v][u] = D[u][v] = fl(td[v] - td[u]) and bumps the counts --
//                fill_tree_pairs (reference _kernels.py:82-116) with the
//                pair loop turned inside out (one walker per descendant).
//                A full row (count N-1) has every bit set, so skipping its
//                walk is exact.  The root's row is always full afterwards.
//   grid barrier
//   select (K3)  grid-wide argmin of the packed key (count << 16 | rank) over
//                open pixels -- FillingRateSelector.next_source
//                (strategies.py:220-227): least filled, then greatest
//                distance from the centroid, then smallest id (the rank is the
//                position in ext = lexsort((id, -dist_from_c))).  naive:
//                key = id (strategies.py:125-129).
//   grid barrier
//
// The loop leaves the kernel only when the selected source has no tree in the
// tree store (the host then propagates a speculative batch: the top-K open
// pixels by the same key, K1) or when the array is complete.  A tree depends
// only on its source, so speculation never changes the committed sequence.
#include <cooperative_groups.h>

#include "gp_common.cuh"
#include "gp_kernels.h"

namespace cg = cooperative_groups;

namespace gp {

constexpr int COMMIT_THREADS = 512;

__device__ __forceinline__ unsigned sel_key(int strategy, int N, int v, int c, const int* rank) {
  if (c >= N - 1) return 0xFFFFFFFFu;
  if (strategy == kFillingRate) return ((unsigned)c << 16) | (unsigned)__ldg(&rank[v]);
  return (unsigned)v;
}

__device__ __forceinline__ int key_src(int strategy, unsigned key, const int* ext) {
  return strategy == kFillingRate ? __ldg(&ext[key & 0xFFFFu]) : (int)key;
}

template <typename T>
__device__ __forceinline__ T block_reduce_min(T v, T* red) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
  if (lane == 0) red[wid] = v;
  __syncthreads();
  if (wid == 0) {
    v = (lane < (int)(blockDim.x >> 5)) ? red[lane] : v;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
  }
  __syncthreads();
  return v;  // valid in warp 0
}

__device__ __forceinline__ unsigned long long block_reduce_sum(unsigned long long v,
                                                               unsigned long long* red) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if (lane == 0) red[wid] = v;
  __syncthreads();
  if (wid == 0) {
    v = (lane < (int)(blockDim.x >> 5)) ? red[lane] : 0ull;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  }
  __syncthreads();
  return v;
}

// grid-wide selection of the source for `step`, excluding pixel `skip`
__device__ void select_step(const CommitArgs& a, int step, int skip, unsigned* red32) {
  const int N = a.g.N;
  unsigned m = 0xFFFFFFFFu;
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < N; v += gridDim.x * blockDim.x) {
    if (v == skip) continue;
    m = min(m, sel_key(a.strategy, N, v, __ldcg(&a.cnt[v]), a.rank));
  }
  m = block_reduce_min(m, red32);
  if (threadIdx.x == 0 && m != 0xFFFFFFFFu) atomicMin(&a.selkey[step], m);
}

__global__ void __launch_bounds__(COMMIT_THREADS) k_commit(CommitArgs a) {
  cg::grid_group grid = cg::this_grid();
  __shared__ unsigned red32[32];
  __shared__ unsigned long long red64[32];
  const int N = a.g.N, W = a.g.W, NW = a.NW;
  const int gtid = blockIdx.x * blockDim.x + threadIdx.x;
  const int gstride = gridDim.x * blockDim.x;

  int step = a.ctl->step;
  int s = a.ctl->cur_src;
  if (s == -1) {  // first launch: select the first source
    select_step(a, step, -1, red32);
    grid.sync();
    unsigned key = __ldcg(&a.selkey[step]);
    s = key == 0xFFFFFFFFu ? -2 : key_src(a.strategy, key, a.ext);
  }
  int status = CTL_RUNNING;
  int done_here = 0;
  for (;;) {
    if (s == -2) { status = CTL_DONE; break; }
    if (done_here >= a.max_steps) { status = CTL_LIMIT; break; }
    const int slot = __ldcg(&a.slot_of[s]);
    if (slot < 0) { status = CTL_MISS; break; }
    const uint8_t* dir = a.tdir + (size_t)slot * N;
    const float* td = a.tdist + (size_t)slot * N;

    // ---- K2: tree-walk fill ----
    unsigned long long lnew_total = 0;
    for (int v = gtid; v < N; v += gstride) {
      if (v == s) continue;
      if (__ldcg(&a.cnt[v]) >= N - 1) continue;  // full row: nothing to set
      uint32_t* mrow = a.mark + (size_t)v * NW;
      const float dv = __ldg(&td[v]);
      const uint32_t vbit = 1u << (v & 31);
      const int vword = v >> 5;
      int u = parent_of(v, __ldg(&dir[v]), W);
      int lnew = 0;
      while (u >= 0) {
        const uint32_t ubit = 1u << (u & 31);
        const uint32_t wv = __ldcg(&mrow[u >> 5]);
        const int pu = parent_of(u, __ldg(&dir[u]), W);
        if (!(wv & ubit)) {
          atomicOr(&mrow[u >> 5], ubit);
          atomicOr(&a.mark[(size_t)u * NW + vword], vbit);
          const float duv = __fsub_rn(dv, __ldg(&td[u]));
          a.D[(size_t)v * N + u] = duv;
          a.D[(size_t)u * N + v] = duv;
          if (u != s) atomicAdd(&a.cnt[u], 1);
          lnew++;
        }
        u = pu;
      }
      if (lnew) atomicAdd(&a.cnt[v], lnew);
      lnew_total += lnew;
    }
    lnew_total = block_reduce_sum(lnew_total, red64);
    if (threadIdx.x == 0 && lnew_total) atomicAdd(&a.newp[step], lnew_total);
    grid.sync();
    if (gtid == 0) {
      a.cnt[s] = N - 1;  // the root pairs with every pixel
      a.seq[step] = s;
    }
    // ---- K3: selection of the next source ----
    select_step(a, step + 1, s, red32);
    grid.sync();
    const unsigned key = __ldcg(&a.selkey[step + 1]);
    step++;
    done_here++;
    s = key == 0xFFFFFFFFu ? -2 : key_src(a.strategy, key, a.ext);
  }
  if (gtid == 0) {
    a.ctl->step = step;
    a.ctl->cur_src = s;
    a.ctl->status = status;
  }
}

int commit_max_blocks() {
  int dev = 0, nsm = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_commit, COMMIT_THREADS, 0);
  return nsm * (per_sm > 0 ? per_sm : 1);
}

cudaError_t launch_commit(const CommitArgs& a, int num_blocks, cudaStream_t st) {
  CommitArgs args = a;
  void* params[] = {&args};
  return cudaLaunchCooperativeKernel((void*)k_commit, dim3(num_blocks), dim3(COMMIT_THREADS),
                                     params, 0, st);
}

// ---- speculative candidate batch: the K smallest keys among open pixels
// without a tree (radix select, MSB first, single CTA) ----
__global__ void __launch_bounds__(1024) k_topk(CommitArgs a, int K, int* cands) {
  __shared__ unsigned hist[256];
  __shared__ unsigned s_prefix, s_mask, s_k, s_all;
  __shared__ int s_n;
  const int N = a.g.N, tid = threadIdx.x;
  if (tid == 0) { s_prefix = 0; s_mask = 0; s_k = (unsigned)K; s_all = 0; s_n = 0; }
  for (int pass = 0; pass < 4; pass++) {
    const int shift = 24 - 8 * pass;
    for (int i = tid; i < 256; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    const unsigned prefix = s_prefix, mask = s_mask;
    if (!s_all) {
      for (int v = tid; v < N; v += blockDim.x) {
        if (__ldcg(&a.slot_of[v]) >= 0) continue;
        unsigned key = sel_key(a.strategy, N, v, __ldcg(&a.cnt[v]), a.rank);
        if (key == 0xFFFFFFFFu || (key & mask) != prefix) continue;
        atomicAdd(&hist[(key >> shift) & 255u], 1u);
      }
    }
    __syncthreads();
    if (tid == 0 && !s_all) {
      unsigned total = 0;
      for (int b = 0; b < 256; b++) total += hist[b];
      if (pass == 0 && total <= s_k) {
        s_all = 1;
      } else {
        unsigned cum = 0;
        for (int b = 0; b < 256; b++) {
          if (cum + hist[b] >= s_k) {
            s_prefix = prefix | ((unsigned)b << shift);
            s_mask = mask | (255u << shift);
            s_k -= cum;
            break;
          }
          cum += hist[b];
        }
      }
    }
    __syncthreads();
  }
  const unsigned thr = s_all ? 0xFFFFFFFEu : s_prefix;
  for (int v = tid; v < N; v += blockDim.x) {
    if (__ldcg(&a.slot_of[v]) >= 0) continue;
    unsigned key = sel_key(a.strategy, N, v, __ldcg(&a.cnt[v]), a.rank);
    if (key == 0xFFFFFFFFu || key > thr) continue;
    int i = atomicAdd(&s_n, 1);
    if (i < K) cands[i] = v;
  }
  __syncthreads();
  if (tid == 0) a.ctl->ncand = min(s_n, K);
}

cudaError_t launch_topk(const CommitArgs& a, int K, int* cands, cudaStream_t st) {
  k_topk<<<1, 1024, 0, st>>>(a, K, cands);
  return cudaGetLastError();
}

// ---------------- store helpers ----------------
__global__ void k_store_init(uint32_t* mark, int NW, float* D, int N) {
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < N; v += gridDim.x * blockDim.x) {
    mark[(size_t)v * NW + (v >> 5)] = 1u << (v & 31);  // rows pre-zeroed by memset
    if (D) D[(size_t)v * N + v] = 0.0f;
  }
}

cudaError_t launch_store_init(uint32_t* mark, int NW, float* D, int N, cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(mark, 0, (size_t)N * NW * 4, st);
  if (e != cudaSuccess) return e;
  k_store_init<<<(N + 255) / 256, 256, 0, st>>>(mark, NW, D, N);
  return cudaGetLastError();
}

// fill_from_tree on an arbitrary parent array (DistanceArray API).  out3 =
// {new pairs, disagreements, cycle flag}.  Values within `tol` (relative)
// agree; tol = 0 for integer images (exact, as the reference).
__global__ void k_fill_tree_api(int N, int NW, const int* parent, const float* td,
                                uint32_t* mark, int* cnt, float* D, unsigned long long* out3,
                                float tol) {
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < N; v += gridDim.x * blockDim.x) {
    int u = parent[v];
    int steps = 0, lnew = 0, bad = 0;
    const float dv = td[v];
    while (u >= 0) {
      const float duv = __fsub_rn(dv, td[u]);
      const uint32_t ubit = 1u << (u & 31);
      uint32_t old = atomicOr(&mark[(size_t)v * NW + (u >> 5)], ubit);
      if (!(old & ubit)) {
        atomicOr(&mark[(size_t)u * NW + (v >> 5)], 1u << (v & 31));
        D[(size_t)v * N + u] = duv;
        D[(size_t)u * N + v] = duv;
        atomicAdd(&cnt[u], 1);
        lnew++;
      } else {
        float cur = D[(size_t)v * N + u];
        float lim = tol * fmaxf(fabsf(duv), 1.0f);
        if (fabsf(cur - duv) > lim) bad++;
      }
      u = parent[u];
      if (++steps > N) { atomicOr(&out3[2], 1ull); break; }
    }
    if (lnew) { atomicAdd(&cnt[v], lnew); atomicAdd(&out3[0], (unsigned long long)lnew); }
    if (bad) atomicAdd(&out3[1], (unsigned long long)bad);
  }
}

cudaError_t launch_fill_tree_api(int N, int NW, const int* parent, const float* tdist,
                                 uint32_t* mark, int* cnt, float* D, unsigned long long* out3,
                                 float tol, cudaStream_t st) {
  k_fill_tree_api<<<(N + 255) / 256, 256, 0, st>>>(N, NW, parent, tdist, mark, cnt, D, out3, tol);
  return cudaGetLastError();
}

// fill_from_source (distances.py:120-147): row and column of s.
__global__ void k_fill_source_api(int N, int NW, int s, const float* dist, uint32_t* mark,
                                  int* cnt, float* D, unsigned long long* out3, float tol) {
  int lnew = 0, bad = 0;
  for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < N; x += gridDim.x * blockDim.x) {
    if (x == s) continue;
    const uint32_t xbit = 1u << (x & 31);
    const float val = dist[x];
    if (mark[(size_t)s * NW + (x >> 5)] & xbit) {
      float cur = D[(size_t)s * N + x];
      if (fabsf(cur - val) > tol * fmaxf(fabsf(val), 1.0f)) bad++;
      continue;
    }
    atomicOr(&mark[(size_t)s * NW + (x >> 5)], xbit);
    atomicOr(&mark[(size_t)x * NW + (s >> 5)], 1u << (s & 31));
    D[(size_t)s * N + x] = val;
    D[(size_t)x * N + s] = val;
    atomicAdd(&cnt[x], 1);
    lnew++;
  }
  if (lnew) { atomicAdd(&cnt[s], lnew); atomicAdd(&out3[0], (unsigned long long)lnew); }
  if (bad) atomicAdd(&out3[1], (unsigned long long)bad);
}

cudaError_t launch_fill_source_api(int N, int NW, int s, const float* dist, uint32_t* mark,
                                   int* cnt, float* D, unsigned long long* out3, float tol,
                                   cudaStream_t st) {
  k_fill_source_api<<<(N + 255) / 256, 256, 0, st>>>(N, NW, s, dist, mark, cnt, D, out3, tol);
  return cudaGetLastError();
}

__global__ void k_mark_unpack(const uint32_t* mark, int N, int NW, uint8_t* out) {
  size_t total = (size_t)N * N;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total;
       i += (size_t)gridDim.x * blockDim.x) {
    size_t r = i / N, c = i % N;
    out[i] = (mark[r * NW + (c >> 5)] >> (c & 31)) & 1u;
  }
}

cudaError_t launch_mark_unpack(const uint32_t* mark, int N, int NW, uint8_t* out,
                               cudaStream_t st) {
  k_mark_unpack<<<1184, 256, 0, st>>>(mark, N, NW, out);
  return cudaGetLastError();
}

// Naive run bookkeeping.  NaiveSelector (strategies.py:125-129) picks the
// smallest open id; after sources 0..s-1 row s is open (count s < N-1) and its
// unmarked entries are exactly x > s, so the sequence is 0..N-2 and commit s
// adds N-1-s pairs.  The batched naive propagation writes those rows; this
// kernel sets the bookkeeping to the state the sequential loop ends in.
__global__ void k_naive_trace(int N, int NW, uint32_t* mark, int* cnt, int* seq,
                              unsigned long long* newp) {
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < N; v += gridDim.x * blockDim.x) {
    cnt[v] = N - 1;
    if (v < N - 1) { seq[v] = v; newp[v] = (unsigned long long)(N - 1 - v); }
    uint32_t* row = mark + (size_t)v * NW;
    for (int w = 0; w < NW; w++) {
      int lo = w * 32;
      int nb = min(32, N - lo);
      row[w] = nb == 32 ? 0xFFFFFFFFu : ((1u << nb) - 1u);
    }
  }
}

cudaError_t launch_naive_trace(int N, int NW, uint32_t* mark, int* cnt, int* seq,
                               unsigned long long* newp, cudaStream_t st) {
  k_naive_trace<<<(N + 255) / 256, 256, 0, st>>>(N, NW, mark, cnt, seq, newp);
  return cudaGetLastError();
}

// first index of the maximum (np.argmax), single CTA
__global__ void k_argmax_first(const float* x, int N, int* out) {
  __shared__ unsigned long long red[32];
  unsigned long long best = ~0ull;
  for (int i = threadIdx.x; i < N; i += blockDim.x) {
    // larger value first, then smaller index: key = (~bits(value)) << 32 | i
    unsigned long long key = ((unsigned long long)(~__float_as_uint(x[i])) << 32) | (unsigned)i;
    best = min(best, key);
  }
  best = block_reduce_min(best, red);
  if (threadIdx.x == 0) *out = (int)(best & 0xFFFFFFFFull);
}

cudaError_t launch_argmax_first(const float* x, int N, int* out, cudaStream_t st) {
  k_argmax_first<<<1, 1024, 0, st>>>(x, N, out);
  return cudaGetLastError();
}

}  // namespace gp
