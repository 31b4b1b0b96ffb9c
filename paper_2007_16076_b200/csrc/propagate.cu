// K1 -- batched geodesic propagation (one CTA per tree).
//
// Restates dijkstra_csr (reference _kernels.py:33-79) as a work-efficient,
// bucketed frontier relaxation over the pixel grid:
//   * the distance map, the image and a pending-vertex bitmap live in shared
//     memory (N <= 16384) or in an L2-resident per-CTA scratch (larger maps);
//   * each pass collects the pending pixels whose distance is below the
//     current bucket threshold into a worklist (warp ballots on the bitmap),
//     then relaxes their <= 8 edges in parallel with atomicMin on the
//     distance bits (non-negative fp32 orders like uint32) and re-marks every
//     improved pixel pending;
//   * when no pending pixel is below the threshold it advances to
//     min(pending) + delta; the loop ends when nothing is pending.
// fp32 addition is monotone and isotone, so any relaxation order reaches the
// same least fixpoint as the reference's heap order: the distances are
// bit-identical to dijkstra_csr (int images: exact integers) and to the fp32
// restatement in oracle/oracle.c.
//
// Predecessors: with strictly positive weights the reference's heap pops in
// (dist, id) order and sets parent on the first strict improvement, so its
// parent is the tight neighbour u (fl(d[u] + w) == d[v]) with the smallest
// (d[u], u).  The post-pass evaluates exactly that rule and stores the
// neighbour's window code (one byte).  Zero-weight edges (L1 metric on equal
// grey levels) break the heap-order argument; there the rule is restricted to
// (d[u], u) < (d[v], v) and plateau interiors are attached by a BFS over
// zero-weight tight edges, which always yields a valid spanning tree.
#include "gp_common.cuh"
#include "gp_kernels.h"

namespace gp {

extern __shared__ __align__(16) unsigned char g_smem[];

struct PropShared {
  int wl_cnt[2];
  uint32_t min_pend[2];
  int any_left[2];
  int slot;
  int changed;
};

__global__ void __launch_bounds__(1024, 1) k_propagate(PropArgs a) {
  const Grid g = a.g;
  const int N = g.N, NW = (N + 31) >> 5;
  const int t = blockIdx.x;
  const int tid = threadIdx.x, nthr = blockDim.x;
  if (a.ntrees_dev && t >= *a.ntrees_dev) return;
  __shared__ PropShared sh;

  uint32_t* dist;
  uint32_t* pend;
  uint16_t* wl;
  const float* f;
  if (a.in_smem) {
    dist = reinterpret_cast<uint32_t*>(g_smem);
    float* fs = reinterpret_cast<float*>(dist + N);
    pend = reinterpret_cast<uint32_t*>(fs + N);
    wl = reinterpret_cast<uint16_t*>(pend + NW);
    for (int i = tid; i < N; i += nthr) fs[i] = a.img[i];
    f = fs;
  } else {
    uint32_t* base = a.scratch + (size_t)t * a.scratch_words;
    dist = base;
    pend = base + N;
    wl = reinterpret_cast<uint16_t*>(pend + NW);
    f = a.img;
  }
  // volatile: in the global-scratch variant, plain loads could hit a stale L1
  // line after atomics performed at L2.
  volatile uint32_t* vdist = dist;
  volatile uint32_t* vpend = pend;

  for (int i = tid; i < N; i += nthr) dist[i] = INF_BITS;
  for (int i = tid; i < NW; i += nthr) pend[i] = 0;
  if (tid == 0) {
    sh.wl_cnt[0] = sh.wl_cnt[1] = 0;
    sh.min_pend[0] = sh.min_pend[1] = INF_BITS;
    sh.any_left[0] = sh.any_left[1] = 0;
  }
  __syncthreads();
  const int* my_src = a.src + (size_t)t * a.ns;
  for (int i = tid; i < a.ns; i += nthr) {
    int v = my_src[i];
    dist[v] = 0u;
    atomicOr(&pend[v >> 5], 1u << (v & 31));
  }
  __syncthreads();

  float thr = a.delta;
  int p = 0;
  const int lane = tid & 31;
  for (;;) {
    // ---- phase A: collect pending pixels with dist <= thr ----
    uint32_t local_min = INF_BITS;
    int left = 0;
    for (int w0 = 0; w0 < NW; w0 += nthr) {
      int w = w0 + tid;
      uint32_t bits = (w < NW) ? vpend[w] : 0u;
      uint32_t taken = 0;
      uint32_t b = bits;
      while (b) {
        int bit = __ffs(b) - 1;
        b &= b - 1;
        int v = (w << 5) + bit;
        uint32_t dv = vdist[v];
        if (__uint_as_float(dv) <= thr) {
          taken |= 1u << bit;
        } else {
          local_min = min(local_min, dv);
          left = 1;
        }
      }
      if (taken) pend[w] = bits & ~taken;
      // compact taken pixels into the worklist, one warp-aggregated atomic
      int c = __popc(taken);
      int incl = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      int total = __shfl_sync(0xffffffffu, incl, 31);
      int base = 0;
      if (lane == 31 && total) base = atomicAdd(&sh.wl_cnt[p], total);
      base = __shfl_sync(0xffffffffu, base, 31);
      int pos = base + incl - c;
      while (taken) {
        int bit = __ffs(taken) - 1;
        taken &= taken - 1;
        wl[pos++] = (uint16_t)((w << 5) + bit);
      }
    }
    if (left) {
      atomicMin(&sh.min_pend[p], local_min);
      sh.any_left[p] = 1;
    }
    __syncthreads();
    const int cnt = sh.wl_cnt[p];
    if (tid == 0) {  // reset the other buffer for the next pass
      sh.wl_cnt[p ^ 1] = 0;
      sh.min_pend[p ^ 1] = INF_BITS;
      sh.any_left[p ^ 1] = 0;
    }
    if (cnt == 0) {
      if (!sh.any_left[p]) break;
      thr = __fadd_rn(__uint_as_float(sh.min_pend[p]), a.delta);
      p ^= 1;
      __syncthreads();
      continue;
    }
    // ---- phase B: relax the worklist's edges ----
    const int items = cnt * 8;
    for (int idx = tid; idx < items; idx += nthr) {
      int v = wl[idx >> 3];
      int k = idx & 7;
      k += (k >= 4);
      if (!k_in_conn(g.conn, k)) continue;
      int r = v / g.W, c = v - r * g.W;
      int u = nbr_at(g, r, c, k);
      if (u < 0) continue;
      float dv = __uint_as_float(vdist[v]);
      float nd = __fadd_rn(dv, edge_w(g.metric, f[v], f[u]));
      uint32_t nb = __float_as_uint(nd);
      if (nb < vdist[u]) {
        uint32_t old = atomicMin(&dist[u], nb);
        if (nb < old) atomicOr(&pend[u >> 5], 1u << (u & 31));
      }
    }
    p ^= 1;
    __syncthreads();
  }

  // ---- predecessor post-pass (closed form of the heap's parent rule) ----
  // pend is all-zero here; reuse it as the root bitmap.
  for (int i = tid; i < a.ns; i += nthr) {
    int v = my_src[i];
    atomicOr(&pend[v >> 5], 1u << (v & 31));
  }
  if (tid == 0) {
    int s;
    if (a.slot_counter) {
      s = atomicAdd(a.slot_counter, 1);
      if (a.slot_of) a.slot_of[my_src[0]] = s;
    } else {
      s = a.slot ? a.slot[t] : t;
    }
    sh.slot = s;
  }
  __syncthreads();
  const size_t off = (size_t)sh.slot * N;
  float* out_d = a.out_dist ? a.out_dist + off : nullptr;
  uint8_t* out_p = a.out_dir ? a.out_dir + off : nullptr;
  int unparented = 0;
  for (int v = tid; v < N; v += nthr) {
    uint32_t dvb = vdist[v];
    uint8_t code = GP_ROOT;
    if (!((vpend[v >> 5] >> (v & 31)) & 1u)) {
      float dv = __uint_as_float(dvb);
      int r = v / g.W, c = v - r * g.W;
      uint32_t best = INF_BITS;
      for (int k = 0; k < 9; k++) {
        if (!k_in_conn(g.conn, k)) continue;
        int u = nbr_at(g, r, c, k);
        if (u < 0) continue;
        uint32_t dub = vdist[u];
        float cand = __fadd_rn(__uint_as_float(dub), edge_w(g.metric, f[u], f[v]));
        if (cand == dv && (dub < dvb || (dub == dvb && u < v)) && dub < best) {
          best = dub;
          code = (uint8_t)k;
        }
      }
      if (code == GP_ROOT) unparented = 1;
    }
    if (out_d) out_d[v] = __uint_as_float(dvb);
    if (out_p) out_p[v] = code;
  }
  // zero-weight plateaus (L1 metric only): attach by BFS over tight w=0 edges
  if (__syncthreads_or(unparented) && out_p) {
    volatile uint8_t* vp = out_p;
    for (;;) {
      int changed = 0;
      for (int v = tid; v < N; v += nthr) {
        if (vp[v] != GP_ROOT || ((vpend[v >> 5] >> (v & 31)) & 1u)) continue;
        int r = v / g.W, c = v - r * g.W;
        for (int k = 0; k < 9; k++) {
          if (!k_in_conn(g.conn, k)) continue;
          int u = nbr_at(g, r, c, k);
          if (u < 0 || vdist[u] != vdist[v]) continue;
          if (edge_w(g.metric, f[u], f[v]) != 0.0f) continue;
          bool attached = vp[u] != GP_ROOT || ((vpend[u >> 5] >> (u & 31)) & 1u);
          if (attached) { vp[v] = (uint8_t)k; changed = 1; break; }
        }
      }
      if (!__syncthreads_or(changed)) break;
    }
  }

  // ---- naive epilogue: fill_from_source for row/column x > s ----
  if (a.D) {
    const int s = my_src[0];
    float* D = a.D;
    for (int x = s + 1 + tid; x < N; x += nthr) {
      float val = __uint_as_float(vdist[x]);
      D[(size_t)s * N + x] = val;
      D[(size_t)x * N + s] = val;
    }
  }
}

size_t prop_smem_bytes(int N) {
  int NW = (N + 31) >> 5;
  return (size_t)N * 4 * 2 + (size_t)NW * 4 + (size_t)N * 2 + 16;
}

size_t prop_scratch_words(int N) {
  int NW = (N + 31) >> 5;
  return ((size_t)N + NW + (N + 1) / 2 + 31) & ~(size_t)31;
}

bool prop_fits_smem(int N) { return prop_smem_bytes(N) <= 200 * 1024; }

cudaError_t launch_propagate(PropArgs a, int ntrees, cudaStream_t st) {
  if (ntrees <= 0) return cudaSuccess;
  size_t smem = 0;
  a.in_smem = prop_fits_smem(a.g.N) ? 1 : 0;
  if (a.in_smem) {
    smem = prop_smem_bytes(a.g.N);
    cudaError_t e = cudaFuncSetAttribute(k_propagate, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
  } else {
    a.scratch_words = prop_scratch_words(a.g.N);
  }
  k_propagate<<<ntrees, 1024, smem, st>>>(a);
  return cudaGetLastError();
}

}  // namespace gp
