// K1 for propagation-only contexts above 65 536 pixels (GridGraph.propagate,
// reference propagation.py:58-64 -> dijkstra_csr, _kernels.py:33-79, which has
// no size limit; only the dense N^2 store is guarded).  The batched K1 packs
// pixel ids in 16 bits; here every array is 32-bit and one tree uses the
// whole GPU:
//   * distances: frontier relaxation passes over a bitmap, atomicMin on the
//     fp32 bits in global memory (label-correcting: every relaxation order
//     reaches the same fp32 fixpoint as the reference's heap, see
//     propagate.cu), a host loop of one launch per pass;
//   * parents: the closed-form rule of the heap order (tight neighbour with
//     the smallest (d[u], u)) when every edge weight is positive,
//     else the sequential heap restatement (heap_dijkstra_big), which gives
//     the heap's order on zero-weight plateaus.
#include <algorithm>

#include "gp_common.cuh"
#include "gp_kernels.h"

namespace gp {

__device__ __forceinline__ void big_rc(const Grid& g, int v, int& r, int& c) {
  r = v / g.W;  // exact for any N (the 16-bit magic of pix_rc is not)
  c = v - r * g.W;
}

__global__ void k_big_init(int N, uint32_t* dist, uint32_t* front, int nw, const int* src, int ns,
                           uint8_t* code) {
  const int stride = gridDim.x * blockDim.x;
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < N; v += stride) {
    dist[v] = INF_BITS;
    code[v] = GP_ROOT;
  }
  for (int w = blockIdx.x * blockDim.x + threadIdx.x; w < 2 * nw; w += stride) front[w] = 0u;
}

__global__ void k_big_seed(uint32_t* dist, uint32_t* front, const int* src, int ns) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < ns; i += gridDim.x * blockDim.x) {
    const int s = src[i];
    dist[s] = 0u;
    atomicOr(&front[s >> 5], 1u << (s & 31));
  }
}

// one pass: relax the edges of every pixel of the current frontier; improved
// pixels join the next frontier.  The current frontier's words are cleared as
// they are consumed.
__global__ void k_big_pass(Grid g, const float* f, uint32_t* dist, uint32_t* cur, uint32_t* nxt, int nw,
                           unsigned* changed) {
  const int N = g.N;
  unsigned any = 0;
  for (int w = blockIdx.x * blockDim.x + threadIdx.x; w < nw; w += gridDim.x * blockDim.x) {
    uint32_t b = cur[w];
    if (!b) continue;
    cur[w] = 0u;
    while (b) {
      const int v = (w << 5) + __ffs(b) - 1;
      b &= b - 1;
      if (v >= N) break;
      const float dv = __uint_as_float(__ldcg(&dist[v]));
      int r, c;
      big_rc(g, v, r, c);
      const float fv = f[v];
      for (int k = 0; k < 9; k++) {
        if (!k_in_conn(g.conn, k)) continue;
        const int u = nbr_at(g, r, c, k);
        if (u < 0) continue;
        const uint32_t nb = __float_as_uint(__fadd_rn(dv, edge_w(g.metric, fv, f[u])));
        if (nb < atomicMin(&dist[u], nb)) {
          atomicOr(&nxt[u >> 5], 1u << (u & 31));
          any = 1;
        }
      }
    }
  }
  if (any) *changed = 1u;
}

// closed-form parents (positive weights): tight neighbour with the smallest (d[u], u)
__global__ void k_big_parents(Grid g, const float* f, const uint32_t* dist, uint8_t* code) {
  const int N = g.N;
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < N; v += gridDim.x * blockDim.x) {
    const uint32_t dvb = dist[v];
    if (dvb == 0u) continue;  // a source (positive weights: only sources are at 0)
    int r, c;
    big_rc(g, v, r, c);
    const float dv = __uint_as_float(dvb), fv = f[v];
    uint32_t best = INF_BITS;
    uint8_t cv = GP_ROOT;
    for (int k = 0; k < 9; k++) {
      if (!k_in_conn(g.conn, k)) continue;
      const int u = nbr_at(g, r, c, k);
      if (u < 0) continue;
      const uint32_t du = dist[u];
      if (du == INF_BITS) continue;
      if (__fadd_rn(__uint_as_float(du), edge_w(g.metric, f[u], fv)) == dv && du < best) {
        best = du;  // neighbours in ascending id: the first of equal distance wins
        cv = (uint8_t)k;
      }
    }
    code[v] = cv;
  }
}

// the heap restatement of dijkstra_csr (see propagate.cu heap_dijkstra) with
// 32-bit ids and exact row/column division; one thread
__global__ void k_big_heap(Grid g, const float* f, uint32_t* dist, const int* src, int ns,
                           unsigned long long* heap, uint8_t* code) {
  if (blockIdx.x || threadIdx.x) return;
  int size = 0;
  auto push = [&](unsigned long long key) {
    int j = size++;
    while (j > 0) {
      const int up = (j - 1) >> 1;
      const unsigned long long hu = heap[up];
      if (hu <= key) break;
      heap[j] = hu;
      j = up;
    }
    heap[j] = key;
  };
  for (int i = 0; i < ns; i++) {
    dist[src[i]] = 0u;
    push((unsigned long long)(unsigned)src[i]);
  }
  while (size > 0) {
    const unsigned long long key = heap[0];
    const unsigned long long last = heap[--size];
    int j = 0;
    for (;;) {
      const int l = 2 * j + 1, r = l + 1;
      if (l >= size) break;
      int m = l;
      unsigned long long hm = heap[l];
      if (r < size) {
        const unsigned long long hr = heap[r];
        if (hr < hm) { m = r; hm = hr; }
      }
      if (hm >= last) break;
      heap[j] = hm;
      j = m;
    }
    if (size > 0) heap[j] = last;
    const int u = (int)(key & 0xFFFFFFFFull);
    const uint32_t db = (uint32_t)(key >> 32);
    if (db != dist[u]) continue;
    int r, c;
    big_rc(g, u, r, c);
    const float d = __uint_as_float(db), fu = f[u];
    for (int k = 0; k < 9; k++) {
      if (!k_in_conn(g.conn, k)) continue;
      const int v = nbr_at(g, r, c, k);
      if (v < 0) continue;
      const uint32_t nb = __float_as_uint(__fadd_rn(d, edge_w(g.metric, fu, f[v])));
      if (nb < dist[v]) {
        dist[v] = nb;
        code[v] = (uint8_t)(8 - k);
        push(((unsigned long long)nb << 32) | (unsigned)v);
      }
    }
  }
}

size_t big_scratch_bytes(int N, int exact) {
  const size_t nw = ((size_t)N + 31) / 32;
  size_t b = 2 * nw * 4 + 16;  // two frontier bitmaps + flag
  if (exact) b += (9 * (size_t)N + 1) * 8;
  return b;
}

// One propagation over the whole GPU; dist_out[N] (fp32 bits) and code_out[N]
// (parent window codes) are device buffers.  `scratch` holds
// big_scratch_bytes(N, exact); `hflag` is a host (pinned) word.
cudaError_t launch_propagate_big(const Grid& g, const float* img, const int* src, int ns, int exact,
                                 uint32_t* dist_out, uint8_t* code_out, unsigned char* scratch,
                                 unsigned* hflag, cudaStream_t st) {
  const int N = g.N, nw = (N + 31) / 32;
  uint32_t* front = reinterpret_cast<uint32_t*>(scratch);
  unsigned* changed = reinterpret_cast<unsigned*>(scratch + 2 * (size_t)nw * 4);
  const int blocks = 148 * 8, threads = 256;
  k_big_init<<<blocks, threads, 0, st>>>(N, dist_out, front, nw, src, ns, code_out);
  if (exact) {
    unsigned long long* heap = reinterpret_cast<unsigned long long*>(scratch + 2 * (size_t)nw * 4 + 16);
    k_big_heap<<<1, 32, 0, st>>>(g, img, dist_out, src, ns, heap, code_out);
    return cudaGetLastError();
  }
  k_big_seed<<<(ns + 255) / 256, 256, 0, st>>>(dist_out, front, src, ns);
  int cur = 0;
  for (long long pass = 0; pass < 4LL * N + 8; pass++) {
    cudaError_t e = cudaMemsetAsync(changed, 0, 4, st);
    if (e != cudaSuccess) return e;
    k_big_pass<<<blocks, threads, 0, st>>>(g, img, dist_out, front + (size_t)cur * nw, front + (size_t)(cur ^ 1) * nw,
                                           nw, changed);
    cur ^= 1;
    e = cudaMemcpyAsync(hflag, changed, 4, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return e;
    if (!*hflag) break;
  }
  k_big_parents<<<blocks, threads, 0, st>>>(g, img, dist_out, code_out);
  return cudaGetLastError();
}

}  // namespace gp
