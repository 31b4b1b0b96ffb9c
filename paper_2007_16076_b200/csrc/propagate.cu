// K1 -- batched geodesic propagation (one CTA per tree) + Euler tour.
//
// Restates dijkstra_csr (reference _kernels.py:33-79) as a work-efficient,
// bucketed frontier relaxation over the pixel grid:
//   * the distance map, the image and a pending-pixel bitmap live in shared
//     memory (N <= 16384) or in an L2-resident per-CTA scratch (larger maps);
//   * each pass collects the pending pixels whose distance is below the
//     current bucket threshold into a worklist (warp-aggregated compaction of
//     the bitmap), then relaxes their <= 8 edges in parallel with atomicMin on
//     the distance bits (non-negative fp32 orders like uint32) and re-marks
//     every improved pixel pending;
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
// (d[u], u).  The post-pass evaluates exactly that rule.  Zero-weight edges
// (L1 metric on equal grey levels) break the heap-order argument; there the
// rule is restricted to (d[u], u) < (d[v], v) and plateau interiors are
// attached by a BFS over zero-weight tight edges (always a valid tree).
//
// Euler tour (tree-store outputs): depths by pointer jumping, a counting sort
// of the pixels by depth, subtree sizes bottom-up and preorder positions
// top-down one level per barrier (children of p are grid neighbours of p, so
// a pixel finds its earlier siblings among p's <= 8 neighbours), then the
// preorder arrays and the balanced partition of the fill work into commit
// warps (exclusive scan of 32-pair chunks).  All of it runs here, off the
// commit loop's critical path.
#include "gp_common.cuh"
#include "gp_kernels.h"

namespace gp {

extern __shared__ __align__(16) unsigned char g_smem[];

constexpr int HIST_SMEM = 4096;  // depth-histogram bins in the shared-memory variant

struct PropShared {
  int wl_cnt[2];
  uint32_t min_pend[2];
  int any_left[2];
  int slot;
  int maxd;
  int wsum[32];
  unsigned total;
};

struct Layout {
  size_t A, B, code, pend, hist, total;
};

__host__ __device__ inline size_t align16(size_t x) { return (x + 15) & ~(size_t)15; }

// [dist 4N][A 4N][B 2N][code N][pend N/8][hist cap*4]
__host__ __device__ inline Layout prop_layout(int N, size_t hist_cap) {
  Layout L;
  L.A = align16((size_t)N * 4);
  L.B = L.A + align16((size_t)N * 4);
  L.code = L.B + align16((size_t)N * 2);
  L.pend = L.code + align16((size_t)N);
  L.hist = L.pend + align16((size_t)((N + 31) >> 5) * 4);
  L.total = L.hist + hist_cap * 4;
  return L;
}

// u16 array element add via a 32-bit atomic on the containing word
__device__ __forceinline__ void atomic_add_u16(uint16_t* base, int i, unsigned v) {
  unsigned* w = reinterpret_cast<unsigned*>(base) + (i >> 1);
  atomicAdd(w, v << ((i & 1) * 16));
}

__global__ void __launch_bounds__(1024, 1) k_propagate(PropArgs a) {
  const Grid g = a.g;
  const int N = g.N, NW = (N + 31) >> 5;
  const int t = blockIdx.x;
  const int tid = threadIdx.x, nthr = blockDim.x;
  if (a.ntrees_dev && t >= *a.ntrees_dev) return;
  __shared__ PropShared sh;

  const size_t hist_cap = a.in_smem ? HIST_SMEM : (size_t)N + 1;
  const Layout lay = prop_layout(N, hist_cap);
  unsigned char* base = a.in_smem ? g_smem : a.scratch + (size_t)t * a.scratch_bytes;
  uint32_t* dist = reinterpret_cast<uint32_t*>(base);
  float* fimg = reinterpret_cast<float*>(base + lay.A);
  uint16_t* wl = reinterpret_cast<uint16_t*>(base + lay.B);
  uint8_t* code = base + lay.code;
  uint32_t* pend = reinterpret_cast<uint32_t*>(base + lay.pend);
  uint32_t* hist = reinterpret_cast<uint32_t*>(base + lay.hist);
  const float* f = a.in_smem ? fimg : a.img;
  if (a.in_smem)
    for (int i = tid; i < N; i += nthr) fimg[i] = a.img[i];
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
    sh.maxd = 0;
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
  const int lane = tid & 31, wid = tid >> 5;
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
      int c = __popc(taken);
      int incl = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      int total = __shfl_sync(0xffffffffu, incl, 31);
      int wbase = 0;
      if (lane == 31 && total) wbase = atomicAdd(&sh.wl_cnt[p], total);
      wbase = __shfl_sync(0xffffffffu, wbase, 31);
      int pos = wbase + incl - c;
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
  if (tid == 0) sh.slot = a.slot ? a.slot[t] : t;
  __syncthreads();
  const int slot = sh.slot;
  const size_t off = (size_t)slot * N;
  volatile uint8_t* vcode = code;
  int unparented = 0;
  for (int v = tid; v < N; v += nthr) {
    uint32_t dvb = vdist[v];
    uint8_t cv = GP_ROOT;
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
          cv = (uint8_t)k;
        }
      }
      if (cv == GP_ROOT) unparented = 1;
    }
    code[v] = cv;
    if (a.out_dist) a.out_dist[off + v] = __uint_as_float(dvb);
  }
  // zero-weight plateaus (L1 metric only): attach by BFS over tight w=0 edges
  if (__syncthreads_or(unparented)) {
    for (;;) {
      int changed = 0;
      for (int v = tid; v < N; v += nthr) {
        if (vcode[v] != GP_ROOT || ((vpend[v >> 5] >> (v & 31)) & 1u)) continue;
        int r = v / g.W, c = v - r * g.W;
        for (int k = 0; k < 9; k++) {
          if (!k_in_conn(g.conn, k)) continue;
          int u = nbr_at(g, r, c, k);
          if (u < 0 || vdist[u] != vdist[v]) continue;
          if (edge_w(g.metric, f[u], f[v]) != 0.0f) continue;
          bool attached = vcode[u] != GP_ROOT || ((vpend[u >> 5] >> (u & 31)) & 1u);
          if (attached) { vcode[v] = (uint8_t)k; changed = 1; break; }
        }
      }
      if (!__syncthreads_or(changed)) break;
    }
  }
  if (a.out_dir)
    for (int v = tid; v < N; v += nthr) a.out_dir[off + v] = vcode[v];

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
  if (!a.ts.pre) return;

  // ================= Euler tour of the (single-root) tree =================
  // E1: depths by pointer jumping on packed (depth << 16 | jump) words (A).
  volatile uint32_t* pj = reinterpret_cast<volatile uint32_t*>(base + lay.A);
  for (int v = tid; v < N; v += nthr) {
    uint8_t cv = vcode[v];
    pj[v] = cv == GP_ROOT ? (uint32_t)v : ((1u << 16) | (uint32_t)parent_of(v, cv, g.W));
  }
  __syncthreads();
  for (;;) {
    int ch = 0;
    for (int v = tid; v < N; v += nthr) {
      uint32_t pr = pj[v];
      uint32_t j = pr & 0xFFFFu;
      uint32_t px = pj[j];
      uint32_t jj = px & 0xFFFFu;
      if (jj != j) {
        pj[v] = ((pr & 0xFFFF0000u) + (px & 0xFFFF0000u)) | jj;
        ch = 1;
      }
    }
    if (!__syncthreads_or(ch)) break;
  }
  // E2: depth (B) and max depth
  volatile uint16_t* depth = reinterpret_cast<volatile uint16_t*>(base + lay.B);
  int lmax = 0;
  for (int v = tid; v < N; v += nthr) {
    int d = (int)(pj[v] >> 16);
    depth[v] = (uint16_t)d;
    lmax = max(lmax, d);
  }
  atomicMax(&sh.maxd, lmax);
  __syncthreads();
  const int maxd = sh.maxd;
  const bool use_hist = (size_t)maxd + 1 <= hist_cap;
  uint16_t* szv = reinterpret_cast<uint16_t*>(base + lay.A);            // descendants
  volatile uint16_t* vszv = szv;
  uint16_t* order = reinterpret_cast<uint16_t*>(base + lay.A + 2 * (size_t)N);
  volatile uint16_t* tin = use_hist ? reinterpret_cast<volatile uint16_t*>(base + lay.B)
                                    : reinterpret_cast<volatile uint16_t*>(order);
  volatile uint32_t* vhist = hist;
  for (int v = tid; v < N; v += nthr) szv[v] = 0;
  // E3: counting sort by depth -> order[], level d = order[hist[d-1] .. hist[d])
  if (use_hist) {
    for (int i = tid; i <= maxd; i += nthr) hist[i] = 0;
    __syncthreads();
    for (int v = tid; v < N; v += nthr) atomicAdd(&hist[depth[v]], 1u);
    __syncthreads();
    if (wid == 0) {  // exclusive scan of hist[0..maxd] by one warp
      unsigned carry = 0;
      for (int i0 = 0; i0 <= maxd; i0 += 32) {
        int i = i0 + lane;
        unsigned x = i <= maxd ? vhist[i] : 0u;
        unsigned incl = x;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          unsigned y = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += y;
        }
        if (i <= maxd) vhist[i] = carry + incl - x;
        carry += __shfl_sync(0xffffffffu, incl, 31);
      }
    }
    __syncthreads();
    for (int v = tid; v < N; v += nthr) {
      unsigned pos = atomicAdd(&hist[depth[v]], 1u);
      order[pos] = (uint16_t)v;
    }
  }
  __syncthreads();
  // E4: descendant counts, deepest level first
  for (int d = maxd; d >= 1; d--) {
    if (use_hist) {
      const unsigned lo = vhist[d - 1], hi = vhist[d];
      for (unsigned i = lo + tid; i < hi; i += nthr) {
        int v = order[i];
        atomic_add_u16(szv, parent_of(v, vcode[v], g.W), (unsigned)vszv[v] + 1u);
      }
    } else {
      for (int v = tid; v < N; v += nthr)
        if (depth[v] == d) atomic_add_u16(szv, parent_of(v, vcode[v], g.W), (unsigned)vszv[v] + 1u);
    }
    __syncthreads();
  }
  // E5: preorder positions, shallowest level first; children of p are
  // ordered by pixel id and each takes its subtree block after p.
  for (int v = tid; v < N; v += nthr)
    if (vcode[v] == GP_ROOT) tin[v] = 0;
  __syncthreads();
  for (int d = 1; d <= maxd; d++) {
    const unsigned lo = use_hist ? vhist[d - 1] : 0u, hi = use_hist ? vhist[d] : (unsigned)N;
    for (unsigned i = lo + tid; i < hi; i += nthr) {
      int v = use_hist ? order[i] : (int)i;
      if (!use_hist && depth[v] != d) continue;
      const int pp = parent_of(v, vcode[v], g.W);
      const int pr = pp / g.W, pc = pp - pr * g.W;
      unsigned offs = 0;
      for (int k = 0; k < 9; k++) {
        if (!k_in_conn(g.conn, k)) continue;
        int q = nbr_at(g, pr, pc, k);
        if (q < 0 || q >= v) continue;
        uint8_t cq = vcode[q];
        if (cq != GP_ROOT && parent_of(q, cq, g.W) == pp) offs += (unsigned)vszv[q] + 1u;
      }
      tin[v] = (uint16_t)(tin[pp] + 1u + offs);
    }
    __syncthreads();
  }
  // E6: preorder arrays.  tdp straight to global, then pre/szp staged in the
  // (now free) distance region for coalesced stores and the partition scan.
  float* gtdp = a.ts.tdp + off;
  for (int v = tid; v < N; v += nthr) gtdp[tin[v]] = __uint_as_float(vdist[v]);
  __syncthreads();
  volatile uint16_t* preS = reinterpret_cast<volatile uint16_t*>(base);
  volatile uint16_t* szS = preS + N;
  for (int v = tid; v < N; v += nthr) {
    unsigned q = tin[v];
    preS[q] = (uint16_t)v;
    szS[q] = vszv[v];
  }
  __syncthreads();
  uint16_t* gpre = a.ts.pre + off;
  uint16_t* gszp = a.ts.szp + off;
  for (int q = tid; q < N; q += nthr) {
    gpre[q] = preS[q];
    gszp[q] = szS[q];
  }
  // E7: chunk counts ceil(szp/32), exclusive scan over preorder, partition
  const int seg = (N + nthr - 1) / nthr;
  const int q0 = min(N, tid * seg), q1 = min(N, q0 + seg);
  unsigned lsum = 0;
  for (int q = q0; q < q1; q++) lsum += ((unsigned)szS[q] + 31u) >> 5;
  unsigned incl = lsum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    unsigned y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) sh.wsum[wid] = incl;
  __syncthreads();
  if (wid == 0) {
    const int nw = nthr >> 5;
    unsigned x = lane < nw ? (unsigned)sh.wsum[lane] : 0u;
    unsigned wi = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      unsigned y = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += y;
    }
    if (lane < nw) sh.wsum[lane] = (int)(wi - x);
    if (lane == 31) sh.total = wi;
  }
  __syncthreads();
  const unsigned T = sh.total;
  const unsigned long long P = (unsigned long long)a.ts.nparts;
  uint32_t* gpart = a.ts.part + (size_t)slot * a.ts.nparts;
  if (tid == 0) a.ts.T[slot] = T;
  unsigned run = (unsigned)sh.wsum[wid] + incl - lsum;
  for (int q = q0; q < q1; q++) {
    const unsigned nch = ((unsigned)szS[q] + 31u) >> 5;
    if (!nch) continue;
    // partitions p whose first chunk floor(p*T/P) lies in [run, run+nch)
    const unsigned long long plo = ((unsigned long long)run * P + T - 1) / T;
    const unsigned long long phi = (((unsigned long long)(run + nch) * P + T - 1) / T);
    for (unsigned long long pp = plo; pp < phi && pp < P; pp++) {
      const unsigned b = (unsigned)((pp * T) / P);
      gpart[pp] = (uint32_t)q | ((b - run) << 16);
    }
    run += nch;
  }
}

size_t prop_smem_bytes(int N) { return prop_layout(N, HIST_SMEM).total; }

size_t prop_scratch_bytes(int N) { return align16(prop_layout(N, (size_t)N + 1).total); }

bool prop_fits_smem(int N) { return prop_smem_bytes(N) <= 227 * 1024; }

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
    a.scratch_bytes = prop_scratch_bytes(a.g.N);
  }
  k_propagate<<<ntrees, 1024, smem, st>>>(a);
  return cudaGetLastError();
}

}  // namespace gp
