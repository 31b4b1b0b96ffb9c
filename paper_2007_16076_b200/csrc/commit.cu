// K2 + K3 -- the device-resident commit loop of run_strategy
// (reference strategies.py:246-273), plus the distance-store kernels.
//
// One persistent cooperative kernel executes commit after commit without
// returning to the host:
//
//   fill   (K2)  fill_tree_pairs (reference _kernels.py:82-116) over the
//                tree's Euler tour: the pairs of the tree are
//                {(pre[q], pre[q+1+k]) : k < szp[q]}, split into 32-pair
//                chunks and pre-partitioned evenly over every warp of the grid
//                (propagate.cu E7).  A warp takes one chunk at a time: all 32
//                lanes share the ancestor u, so their mark bits lie in row u
//                at the (tile-ordered) columns of one subtree region.  An
//                unmarked pair sets both bits, writes D[u][w] = D[w][u] =
//                fl(td[w] - td[u]) and bumps both counts -- first writer in
//                commit order, exactly as the reference.  Ancestors whose row
//                is full (count N-1) are skipped: every bit is already set.
//   grid barrier
//   select (K3)  grid-wide argmin of the packed key (count << 16 | rank) over
//                open pixels -- FillingRateSelector.next_source
//                (strategies.py:220-227): least filled, then greatest
//                distance from the centroid, then smallest id (rank = position
//                in ext = lexsort((id, -dist_from_c))).  naive (with tree):
//                key = id (strategies.py:125-129).
//   grid barrier
//
// The loop leaves the kernel only when the selected source has no tree in
// the store (the host then propagates a speculative batch: the top-K open
// pixels by the same key, K1) or when the array is complete.  A tree depends
// only on its source, so speculation never changes the committed sequence.
#include <cooperative_groups.h>

#include "gp_common.cuh"
#include "gp_kernels.h"

namespace cg = cooperative_groups;

namespace gp {

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

// K2 for one committed tree: this warp's share of the chunks.
//
// The warp walks its chunk range window by window: one coalesced load brings
// the metadata of 32 consecutive preorder positions (descendant count, pixel,
// distance, full-row flag), a warp scan of the chunk counts maps chunks to
// positions, and the chunks are then processed G at a time so that the G
// descendant-list loads and the G mark-word loads are each in flight
// together (the fill is latency-bound: ~2 L2 round trips per G chunks).
template <int G>
__device__ __forceinline__ unsigned fill_warp_share(const CommitArgs& a, int slot, int s) {
  const int N = a.g.N;
  const int lane = threadIdx.x & 31;
  const int P = a.ts.nparts;
  const int p = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const size_t off = (size_t)slot * N;
  const uint16_t* pre = a.ts.pre + off;
  const uint16_t* szp = a.ts.szp + off;
  const float* tdp = a.ts.tdp + off;
  const unsigned T = __ldg(&a.ts.T[slot]);
  const unsigned b0 = (unsigned)(((unsigned long long)p * T) / P);
  const unsigned b1 = (unsigned)(((unsigned long long)(p + 1) * T) / P);
  unsigned count = b1 - b0;
  if (!count) return 0;
  const uint32_t pw = __ldg(&a.ts.part[(size_t)slot * P + p]);
  int q = (int)(pw & 0xFFFFu);
  unsigned coff = pw >> 16;
  unsigned total_new = 0;
  const MarkLayout L = a.L;
  while (count) {
    // ---- window metadata, one position per lane ----
    const int qa = q + lane;
    unsigned sz_l = 0;
    int u_l = 0;
    float td_l = 0.f;
    if (qa < N) {
      sz_l = __ldg(&szp[qa]);
      u_l = __ldg(&pre[qa]);
      td_l = __ldg(&tdp[qa]);
    }
    unsigned nch_l = (sz_l + 31u) >> 5;
    unsigned c0_l = 0;
    if (lane == 0) { nch_l -= coff; c0_l = coff; }
    const bool full_l = nch_l && u_l != s && __ldcg(&a.cnt[u_l]) >= N - 1;
    unsigned cum = nch_l;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned y = __shfl_up_sync(0xffffffffu, cum, o);
      if (lane >= o) cum += y;
    }
    const unsigned excl = cum - nch_l;
    const unsigned wtotal = __shfl_sync(0xffffffffu, cum, 31);
    const unsigned take = min(wtotal, count);
    // ---- chunks, G at a time ----
    for (unsigned cb = 0; cb < take; cb += G) {
      int w[G], qc[G], uu[G];
      bool ok[G];
      float tdu[G];
#pragma unroll
      for (int j = 0; j < G; j++) {
        const unsigned c = cb + j;
        const unsigned m = __ballot_sync(0xffffffffu, cum > c);
        const int ol = m ? __ffs(m) - 1 : 0;
        const unsigned sz = __shfl_sync(0xffffffffu, sz_l, ol);
        const unsigned cidx = __shfl_sync(0xffffffffu, c0_l + (c - excl), ol);
        const bool full = __shfl_sync(0xffffffffu, (int)full_l, ol);
        uu[j] = __shfl_sync(0xffffffffu, u_l, ol);
        tdu[j] = __shfl_sync(0xffffffffu, td_l, ol);
        qc[j] = q + ol;
        const unsigned k = cidx * 32u + lane;
        ok[j] = c < take && !full && k < sz;
        w[j] = ok[j] ? (int)__ldg(&pre[qc[j] + 1 + k]) : 0;
        qc[j] += 1 + (int)k;  // preorder position of w
      }
      uint32_t word[G], wbit[G];
      uint32_t* mw[G];
#pragma unroll
      for (int j = 0; j < G; j++) {
        const uint32_t wcol = mcol(L, (uint32_t)w[j]);
        wbit[j] = 1u << (wcol & 31);
        mw[j] = a.mark + (size_t)uu[j] * L.RW + (wcol >> 5);
        word[j] = ok[j] ? __ldcg(mw[j]) : wbit[j];
      }
#pragma unroll
      for (int j = 0; j < G; j++) {
        const bool isnew = !(word[j] & wbit[j]);
        if (isnew) {
          const int u = uu[j], ww = w[j];
          const uint32_t ucol = mcol(L, (uint32_t)u);
          atomicOr(mw[j], wbit[j]);
          atomicOr(a.mark + mword(L, (uint32_t)ww, ucol), 1u << (ucol & 31));
          const float duv = __fsub_rn(__ldg(&tdp[qc[j]]), tdu[j]);
          a.D[(size_t)u * N + ww] = duv;
          a.D[(size_t)ww * N + u] = duv;
          atomicAdd(&a.cnt[ww], 1);
        }
        const unsigned nb = __popc(__ballot_sync(0xffffffffu, isnew));
        if (lane == 0 && nb && uu[j] != s) atomicAdd(&a.cnt[uu[j]], (int)nb);
        total_new += nb;
      }
    }
    count -= take;
    q += 32;
    coff = 0;
  }
  return lane == 0 ? total_new : 0u;
}

template <int G, int MINB>
__global__ void __launch_bounds__(COMMIT_THREADS, MINB) k_commit(CommitArgs a) {
  cg::grid_group grid = cg::this_grid();
  __shared__ unsigned red32[32];
  __shared__ unsigned long long red64[32];
  const int N = a.g.N;
  const int gtid = blockIdx.x * blockDim.x + threadIdx.x;

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

    unsigned long long* dbg = (a.dbg && blockIdx.x == 0 && threadIdx.x == 0) ? a.dbg + (size_t)step * 4 : nullptr;
    if (dbg) dbg[0] = gtimer();
    // ---- K2: Euler-range fill ----
    unsigned long long lnew = fill_warp_share<G>(a, slot, s);
    if (dbg) dbg[1] = gtimer();
    lnew = block_reduce_sum(lnew, red64);
    if (threadIdx.x == 0 && lnew) atomicAdd(&a.newp[step], lnew);
    grid.sync();
    if (dbg) dbg[2] = gtimer();
    if (gtid == 0) {
      a.cnt[s] = N - 1;  // the root pairs with every pixel
      a.seq[step] = s;
      a.slot_of[s] = -2;  // committed: recycle the slot
      a.ctl->visits += __ldg(&a.ts.C[slot]);
      a.free_stack[a.ctl->free_top++] = slot;
    }
    // ---- K3: selection of the next source ----
    select_step(a, step + 1, s, red32);
    if (dbg) dbg[3] = gtimer();
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

// Fill pipelining depth G (chunks in flight per warp): G=4 keeps 2 CTAs of
// 512 threads per SM within 64 registers; G=8 needs ~128 registers (1 CTA/SM).
static const void* commit_kernel(int G) {
  return G >= 8 ? (const void*)k_commit<8, 1> : (const void*)k_commit<4, 2>;
}

int commit_fill_depth() {
  int G = 4;
  if (const char* e = getenv("GP_FILL_G")) G = atoi(e);
  return G >= 8 ? 8 : 4;
}

int commit_max_blocks() {
  int dev = 0, nsm = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, commit_kernel(commit_fill_depth()),
                                                COMMIT_THREADS, 0);
  return nsm * (per_sm > 0 ? per_sm : 1);
}

cudaError_t launch_commit(const CommitArgs& a, int num_blocks, cudaStream_t st) {
  CommitArgs args = a;
  void* params[] = {&args};
  return cudaLaunchCooperativeKernel(commit_kernel(commit_fill_depth()), dim3(num_blocks),
                                     dim3(COMMIT_THREADS), params, 0, st);
}

// ---- speculative candidate batch: the K smallest keys among open pixels
// without a tree (radix select, MSB first, single CTA); assigns tree slots
// (recycled first) and records slot_of[] ----
__global__ void __launch_bounds__(1024) k_topk(CommitArgs a, int K, int* cands, int* slots) {
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
        if (__ldcg(&a.slot_of[v]) != -1) continue;
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
    if (__ldcg(&a.slot_of[v]) != -1) continue;
    unsigned key = sel_key(a.strategy, N, v, __ldcg(&a.cnt[v]), a.rank);
    if (key == 0xFFFFFFFFu || key > thr) continue;
    int i = atomicAdd(&s_n, 1);
    if (i < K) cands[i] = v;
  }
  __syncthreads();
  if (tid == 0) {
    const int n = min(s_n, K);
    Ctl* c = a.ctl;
    for (int i = 0; i < n; i++) {
      int sl = c->free_top > 0 ? a.free_stack[--c->free_top] : c->nslots++;
      slots[i] = sl;
      a.slot_of[cands[i]] = sl;
    }
    c->ncand = n;
    c->total_props += n;
  }
}

cudaError_t launch_topk(const CommitArgs& a, int K, int* cands, int* slots, cudaStream_t st) {
  k_topk<<<1, 1024, 0, st>>>(a, K, cands, slots);
  return cudaGetLastError();
}

// ---------------- store helpers ----------------
__global__ void k_store_init(MarkLayout L, uint32_t* mark, float* D) {
  const int N = L.N;
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < N; v += gridDim.x * blockDim.x) {
    const uint32_t c = mcol(L, (uint32_t)v);
    mark[mword(L, (uint32_t)v, c)] = 1u << (c & 31);  // rows pre-zeroed by memset
    if (D) D[(size_t)v * N + v] = 0.0f;
  }
}

cudaError_t launch_store_init(const MarkLayout& L, uint32_t* mark, float* D, cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(mark, 0, (size_t)L.N * L.RW * 4, st);
  if (e != cudaSuccess) return e;
  k_store_init<<<(L.N + 255) / 256, 256, 0, st>>>(L, mark, D);
  return cudaGetLastError();
}

// fill_from_tree on an arbitrary parent array (DistanceArray API).  out3 =
// {new pairs, disagreements, cycle flag}.  Values within `tol` (relative)
// agree; tol = 0 for integer images (exact, as the reference).
__global__ void k_fill_tree_api(MarkLayout L, const int* parent, const float* td, uint32_t* mark,
                                int* cnt, float* D, unsigned long long* out3, float tol) {
  const int N = L.N;
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < N; v += gridDim.x * blockDim.x) {
    int u = parent[v];
    int steps = 0, lnew = 0, bad = 0;
    const float dv = td[v];
    const uint32_t vcol = mcol(L, (uint32_t)v);
    while (u >= 0) {
      const float duv = __fsub_rn(dv, td[u]);
      const uint32_t ucol = mcol(L, (uint32_t)u);
      const uint32_t ubit = 1u << (ucol & 31);
      uint32_t old = atomicOr(&mark[mword(L, (uint32_t)v, ucol)], ubit);
      if (!(old & ubit)) {
        atomicOr(&mark[mword(L, (uint32_t)u, vcol)], 1u << (vcol & 31));
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

cudaError_t launch_fill_tree_api(const MarkLayout& L, const int* parent, const float* tdist,
                                 uint32_t* mark, int* cnt, float* D, unsigned long long* out3,
                                 float tol, cudaStream_t st) {
  k_fill_tree_api<<<(L.N + 255) / 256, 256, 0, st>>>(L, parent, tdist, mark, cnt, D, out3, tol);
  return cudaGetLastError();
}

// fill_from_source (distances.py:120-147): row and column of s.
__global__ void k_fill_source_api(MarkLayout L, int s, const float* dist, uint32_t* mark,
                                  int* cnt, float* D, unsigned long long* out3, float tol) {
  const int N = L.N;
  const uint32_t scol = mcol(L, (uint32_t)s);
  int lnew = 0, bad = 0;
  for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < N; x += gridDim.x * blockDim.x) {
    if (x == s) continue;
    const uint32_t xcol = mcol(L, (uint32_t)x);
    const uint32_t xbit = 1u << (xcol & 31);
    const float val = dist[x];
    if (mark[mword(L, (uint32_t)s, xcol)] & xbit) {
      float cur = D[(size_t)s * N + x];
      if (fabsf(cur - val) > tol * fmaxf(fabsf(val), 1.0f)) bad++;
      continue;
    }
    atomicOr(&mark[mword(L, (uint32_t)s, xcol)], xbit);
    atomicOr(&mark[mword(L, (uint32_t)x, scol)], 1u << (scol & 31));
    D[(size_t)s * N + x] = val;
    D[(size_t)x * N + s] = val;
    atomicAdd(&cnt[x], 1);
    lnew++;
  }
  if (lnew) { atomicAdd(&cnt[s], lnew); atomicAdd(&out3[0], (unsigned long long)lnew); }
  if (bad) atomicAdd(&out3[1], (unsigned long long)bad);
}

cudaError_t launch_fill_source_api(const MarkLayout& L, int s, const float* dist, uint32_t* mark,
                                   int* cnt, float* D, unsigned long long* out3, float tol,
                                   cudaStream_t st) {
  k_fill_source_api<<<(L.N + 255) / 256, 256, 0, st>>>(L, s, dist, mark, cnt, D, out3, tol);
  return cudaGetLastError();
}

__global__ void k_mark_unpack(MarkLayout L, const uint32_t* mark, uint8_t* out) {
  const size_t N = L.N, total = N * N;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total;
       i += (size_t)gridDim.x * blockDim.x) {
    const uint32_t r = (uint32_t)(i / N), c = (uint32_t)(i % N);
    const uint32_t ct = mcol(L, c);
    out[i] = (mark[mword(L, r, ct)] >> (ct & 31)) & 1u;
  }
}

cudaError_t launch_mark_unpack(const MarkLayout& L, const uint32_t* mark, uint8_t* out,
                               cudaStream_t st) {
  k_mark_unpack<<<1184, 256, 0, st>>>(L, mark, out);
  return cudaGetLastError();
}

// Naive run bookkeeping.  NaiveSelector (strategies.py:125-129) picks the
// smallest open id; after sources 0..s-1 row s is open (count s < N-1) and its
// unmarked entries are exactly x > s, so the sequence is 0..N-2 and commit s
// adds N-1-s pairs.  The batched naive propagation writes those rows; this
// kernel sets the bookkeeping to the state the sequential loop ends in.
__global__ void k_naive_trace(MarkLayout L, uint32_t* mark, int* cnt, int* seq,
                              unsigned long long* newp) {
  const int N = L.N;
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < N; v += gridDim.x * blockDim.x) {
    cnt[v] = N - 1;
    if (v < N - 1) { seq[v] = v; newp[v] = (unsigned long long)(N - 1 - v); }
  }
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < (size_t)N * L.RW;
       i += (size_t)gridDim.x * blockDim.x)
    mark[i] = 0xFFFFFFFFu;
}

cudaError_t launch_naive_trace(const MarkLayout& L, uint32_t* mark, int* cnt, int* seq,
                               unsigned long long* newp, cudaStream_t st) {
  k_naive_trace<<<592, 256, 0, st>>>(L, mark, cnt, seq, newp);
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
