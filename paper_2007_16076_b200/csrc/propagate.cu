// K1 -- batched geodesic propagation (one CTA per tree) + Euler tour.
//
// Restates dijkstra_csr (reference _kernels.py:33-79) as a work-efficient
// bucketed relaxation (delta-stepping) over the pixel grid:
//   * the distance map, the image, two worklists and two pixel bitmaps live
//     in shared memory (N <= 16384) or in an L2-resident per-CTA scratch;
//   * a pass relaxes the <= 8 edges of every pixel of the near worklist in
//     parallel (atomicMin on the fp32 bits -- non-negative floats order like
//     uint32); an improved pixel whose new distance is within the bucket
//     threshold joins the next near worklist (deduplicated by the `inq`
//     bitmap), otherwise it is parked in the `far` bitmap;
//   * when the near list runs dry the far bitmap is scanned once: the bucket
//     advances to min(far) + delta and the far pixels below it form the next
//     near list.  The loop ends when both are empty.
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
// Euler tour (tree-store outputs): depths by pointer jumping, a counting
// sort of the pixels by depth, descendant counts bottom-up one level at a
// time by a single warp (no block barriers), preorder positions by pointer
// jumping over path sums (a pixel's earlier siblings are among its parent's
// <= 8 grid neighbours), then the preorder arrays and the balanced partition
// of the fill work into commit warps (exclusive scan of 32-pair chunks; the
// root's N-1 pairs are excluded -- the commit kernel scans its row).  All
// of it runs here, off the commit loop's critical path.
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "gp_common.cuh"
#include "gp_kernels.h"

namespace gp {

extern __shared__ __align__(16) unsigned char g_smem[];

// loads in flight per thread in the global-scratch loops (tuned on B200)
#ifndef GP_PJ_CHAINS
#define GP_PJ_CHAINS 4
#endif
#ifndef GP_UB
#define GP_UB 8
#endif
#ifndef GP_UE
#define GP_UE 4
#endif
#ifndef GP_RR
#define GP_RR 2  // relaxation rounds of (item, edge) pairs in flight per thread (global variant)
#endif
#ifndef GP_E5
#define GP_E5 1  // parents per thread and iteration in the sibling-offset pass (E5; 256^2: 1 -> 578.6, 2 -> 586.7, 4 -> 599.5 ms)
#endif

constexpr int HIST_SMEM = 4096;  // depth-histogram bins in the shared-memory variant
constexpr int HIST_G = 1024;     // depth-histogram bins in smem (global-scratch variant)
constexpr int WL_SMEM = 9216;    // worklist entries kept in smem (global-scratch variant)

struct PropShared {
  int cnt[2];
  uint32_t minfar;
  int slot;
  int maxd;
  int wsum[32];
  unsigned total;
  unsigned pairs;
  int nbig;
  int lite;  // list-mode tree: tin/tdp/C only (no pre/szp/partition)
};

struct Layout {
  size_t A, B, W2, far, inq, hist, total;
};

__host__ __device__ inline size_t align16(size_t x) { return (x + 15) & ~(size_t)15; }

// [dist 4N][A 4N][B 2N][W2 2N][far N/8][inq N/8][hist cap*4]
//   relaxation: A = image (smem variant), B/W2 = worklists
//   Euler tour: A = (depth|jump) then sizes/order then (tin|jump); B = depth then
//               sizes; W2 = parent codes
__host__ __device__ inline Layout prop_layout(int N, size_t hist_cap) {
  Layout L;
  const size_t bm = align16((size_t)((N + 31) >> 5) * 4);
  L.A = align16((size_t)N * 4);
  L.B = L.A + align16((size_t)N * 4);
  L.W2 = L.B + align16((size_t)N * 2);
  L.far = L.W2 + align16((size_t)N * 2);
  L.inq = L.far + bm;
  L.hist = L.inq + bm;
  L.total = L.hist + hist_cap * 4;
  return L;
}

// Parent codes, 4 bits per pixel in shared memory (window position 0..8,
// 15 = root): a 256x256 tree's codes take 32 KB, so four trees share an SM.
__device__ __forceinline__ uint8_t code_get(const volatile uint8_t* code, int v) {
  const unsigned c = ((unsigned)code[v >> 1] >> ((v & 1) << 2)) & 15u;
  return c == 15u ? GP_ROOT : (uint8_t)c;
}

// set the code of a root pixel (nibble 15) to k: one atomic
__device__ __forceinline__ void code_set_root(uint8_t* code, int v, unsigned k) {
  unsigned* w = reinterpret_cast<unsigned*>(code) + (v >> 3);
  atomicAnd(w, ~((15u ^ k) << ((v & 7) << 2)));
}

// set the code of pixel v to k (the other nibbles of the word may change
// concurrently: both steps are atomic)
__device__ __forceinline__ void code_set(volatile uint8_t* code, int v, unsigned k) {
  unsigned* w = reinterpret_cast<unsigned*>(const_cast<uint8_t*>(code)) + (v >> 3);
  const int sh = (v & 7) << 2;
  atomicOr(w, 15u << sh);
  atomicAnd(w, ~((15u ^ k) << sh));
}

// u16 array element add via a 32-bit atomic on the containing word
__device__ __forceinline__ void atomic_add_u16(uint16_t* base, int i, unsigned v) {
  unsigned* w = reinterpret_cast<unsigned*>(base) + (i >> 1);
  atomicAdd(w, v << ((i & 1) * 16));
}

// Near worklists: the first `cap` entries in shared memory, the (rare)
// overflow in the per-CTA global scratch.  The shared-memory variant keeps
// whole lists in shared memory (cap = N).
struct WorkLists {
  uint16_t* s[2];
  uint16_t* g[2];
  int cap;
  __device__ __forceinline__ uint16_t* at(int l, int i) const {
    return i < cap ? s[l] + i : g[l] + (i - cap);
  }
};

// warp-aggregated append of `v` (where flag) to list l
__device__ __forceinline__ void warp_append(bool flag, int v, int* cnt, const WorkLists& wl,
                                            int l) {
  const unsigned m = __ballot_sync(0xffffffffu, flag);
  if (!m) return;
  const int lane = threadIdx.x & 31;
  int base = 0;
  if (lane == __ffs(m) - 1) base = atomicAdd(cnt, __popc(m));
  base = __shfl_sync(0xffffffffu, base, __ffs(m) - 1);
  if (flag) *wl.at(l, base + __popc(m & ((1u << lane) - 1u))) = (uint16_t)v;
}

// in-place pointer jumping on packed (acc << 16 | jump) words until every
// jump points at a root (jump == self); acc accumulates along the path.
// A concurrent update of pj[j] is read atomically (one 32-bit word), and any
// consistent (acc, jump) pair of an ancestor is valid, so no double buffer.
__device__ void pointer_jump(volatile uint32_t* pj, int N) {
  for (;;) {
    int ch = 0;
    for (int v = threadIdx.x; v < N; v += blockDim.x) {
      const uint32_t pr = pj[v];
      const uint32_t j = pr & 0xFFFFu;
      const uint32_t px = pj[j];
      const uint32_t jj = px & 0xFFFFu;
      if (jj != j) {
        pj[v] = ((pr & 0xFFFF0000u) + (px & 0xFFFF0000u)) | jj;
        ch = 1;
      }
    }
    if (!__syncthreads_or(ch)) break;
  }
}

// global-scratch variant: the same with L2 loads (__ldcg, no stale L1) and four
// independent chains per thread in flight
__device__ void pointer_jump_global(uint32_t* pj, int N) {
  for (;;) {
    int ch = 0;
    for (int v0 = threadIdx.x; v0 < N; v0 += GP_PJ_CHAINS * blockDim.x) {
      uint32_t pr[GP_PJ_CHAINS], px[GP_PJ_CHAINS];
#pragma unroll
      for (int j = 0; j < GP_PJ_CHAINS; j++) {
        const int v = v0 + j * blockDim.x;
        pr[j] = v < N ? __ldcg(&pj[v]) : 0u;
      }
#pragma unroll
      for (int j = 0; j < GP_PJ_CHAINS; j++) {
        const int v = v0 + j * blockDim.x;
        px[j] = v < N ? __ldcg(&pj[pr[j] & 0xFFFFu]) : 0u;
      }
#pragma unroll
      for (int j = 0; j < GP_PJ_CHAINS; j++) {
        const int v = v0 + j * blockDim.x;
        const uint32_t jj = px[j] & 0xFFFFu;
        if (v < N && jj != (pr[j] & 0xFFFFu)) {
          __stcg(&pj[v], ((pr[j] & 0xFFFF0000u) + (px[j] & 0xFFFF0000u)) | jj);
          ch = 1;
        }
      }
    }
    if (!__syncthreads_or(ch)) break;
  }
}

// Exact restatement of dijkstra_csr (_kernels.py:33-79) for images with
// zero-weight edges (L1 metric on equal neighbours; zero pixels), run by one
// thread of the tree's CTA: a binary heap keyed by (dist, id) -- the
// reference's dist * n + id order; keys are unique, so any correct min-heap
// pops in the reference's order --, stale entries skipped, the parent set on
// strict improvement only.  Without zero-weight edges the closed-form rule of
// the post-pass reproduces that order; on a zero-weight plateau
// the pops within one distance level follow the heap's discovery order,
// which only this sequential simulation gives.  Writes dist (fp32 bits) and
// the parent window codes (GP_ROOT for sources).
__device__ void heap_dijkstra(const Grid& g, int metric, int conn, const float* f, volatile uint32_t* dist,
                              const int* src, int ns, unsigned long long* heap, uint8_t* pcode) {
  const int N = g.N;
  for (int v = 0; v < N; v++) pcode[v] = GP_ROOT;
  int size = 0;
  auto push = [&](unsigned long long key) {
    int j = size++;
    heap[j] = key;
    while (j > 0) {
      const int up = (j - 1) >> 1;
      const unsigned long long hu = heap[up];
      if (hu <= key) break;
      heap[j] = hu;
      j = up;
    }
    heap[j] = key;
  };
  for (int i = 0; i < ns; i++) push((unsigned long long)(unsigned)src[i]);  // dist 0
  while (size > 0) {
    const unsigned long long key = heap[0];
    const unsigned long long last = heap[--size];
    int j = 0;
    for (;;) {  // sift the last entry down from the root
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
    if (db != dist[u]) continue;  // stale entry
    int r, c;
    pix_rc(g, u, r, c);
    const float d = __uint_as_float(db), fu = f[u];
    for (int k = 0; k < 9; k++) {  // ascending neighbour id = the CSR row order
      if (!k_in_conn(conn, k)) continue;
      const int v = nbr_at(g, r, c, k);
      if (v < 0) continue;
      const uint32_t nb = __float_as_uint(__fadd_rn(d, edge_w(metric, fu, f[v])));
      if (nb < dist[v]) {
        dist[v] = nb;
        pcode[v] = (uint8_t)(8 - k);  // u relative to v
        push(((unsigned long long)nb << 32) | (unsigned)v);
      }
    }
  }
}

// VAR: 0 = generic (variant, outputs and debug stamps decided at run time);
// 1 / 2 = lean global-scratch / shared-memory variant for speculative
// batches: Euler-tour outputs only, no naive epilogue, no API outputs, no
// debug stamps -- each gets its own register allocation.
// MC = 1: SUM metric and 8-connectivity fixed at compile time (the BASELINE
// configurations but config 3); 0: read from the grid.
template <int THR, int MINB, int VAR = 0, int MC = 0>
__global__ void __launch_bounds__(THR, MINB) k_propagate(PropArgs a) {
  constexpr bool LEAN = VAR != 0;
  const bool in_smem = VAR == 2 ? true : VAR == 1 ? false : a.in_smem != 0;
  const Grid g = a.g;
  const int gmetric = MC ? (int)kSum : g.metric, gconn = MC ? 8 : g.conn;
  const int N = g.N, NW = (N + 31) >> 5;
  const int t = a.tree_base + (int)blockIdx.x;  // tree index (chunked launches: base + CTA)
  const int tid = threadIdx.x, nthr = blockDim.x;
  const int lane = tid & 31, wid = tid >> 5;
  if (a.ntrees_dev && t >= *a.ntrees_dev) return;
  const bool exact = !LEAN && a.exact_heap;  // zero-weight edges: sequential heap order
  __shared__ PropShared sh;
  unsigned long long* dbg = (!LEAN && a.dbg) ? a.dbg + (size_t)t * 16 : nullptr;
  if (dbg && tid == 0) { dbg[0] = gtimer(); dbg[12] = 0; dbg[13] = 0; }

  const size_t hist_cap = in_smem ? HIST_SMEM : HIST_G;
  const Layout lay = prop_layout(N, hist_cap);
  unsigned char* base = in_smem ? g_smem : a.scratch + (size_t)blockIdx.x * a.scratch_bytes;
  uint32_t* dist = reinterpret_cast<uint32_t*>(base);
  float* fimg = reinterpret_cast<float*>(base + lay.A);
  WorkLists wl;
  wl.g[0] = reinterpret_cast<uint16_t*>(base + lay.B);
  wl.g[1] = reinterpret_cast<uint16_t*>(base + lay.W2);
  uint8_t* code = base + lay.W2;
  uint32_t* far = reinterpret_cast<uint32_t*>(base + lay.far);
  uint32_t* inq = reinterpret_cast<uint32_t*>(base + lay.inq);
  uint32_t* hist = reinterpret_cast<uint32_t*>(base + lay.hist);
  if (in_smem) {
    wl.s[0] = wl.g[0];
    wl.s[1] = wl.g[1];
    wl.cap = N;
  } else {
    // global-scratch variant: bitmaps and the head of both worklists in smem;
    // after the relaxation the worklist area holds the parent codes and the
    // depth histogram (the Euler tour's latency-critical arrays)
    const size_t bm = align16((size_t)NW * 4);
    far = reinterpret_cast<uint32_t*>(g_smem);
    inq = reinterpret_cast<uint32_t*>(g_smem + bm);
    wl.s[0] = reinterpret_cast<uint16_t*>(g_smem + 2 * bm);
    wl.s[1] = wl.s[0] + WL_SMEM;
    wl.cap = WL_SMEM;
    code = g_smem + 2 * bm;
    hist = reinterpret_cast<uint32_t*>(g_smem + 2 * bm + align16((size_t)(N + 1) / 2));
  }
  const float* f = in_smem ? fimg : a.img;
  if (in_smem)
    for (int i = tid; i < N; i += nthr) fimg[i] = a.img[i];
  // volatile: in the global-scratch variant, plain loads could hit a stale L1
  // line after atomics performed at L2.
  volatile uint32_t* vdist = dist;
  volatile uint32_t* vfar = far;

  for (int i = tid; i < N; i += nthr) dist[i] = INF_BITS;
  for (int i = tid; i < NW; i += nthr) { far[i] = 0; inq[i] = 0; }
  if (tid == 0) {
    sh.cnt[0] = a.ns;
    sh.cnt[1] = 0;
    sh.maxd = 0;
    sh.pairs = 0;
    sh.lite = a.list_mode ? (*(volatile const int*)a.list_mode == 1) : 0;
  }
  __syncthreads();
  const int* my_src = a.src + (size_t)t * a.ns;
  for (int i = tid; i < a.ns; i += nthr) {
    const int v = my_src[i];
    dist[v] = 0u;
    *wl.at(0, i) = (uint16_t)v;
  }
  __syncthreads();

  // ---------------- bucketed relaxation ----------------
  float thr = a.delta;
  int cur = 0;
  unsigned passes = 0, items_total = 0;
  unsigned long long* hp = exact ? a.heap + (size_t)blockIdx.x * a.heap_words : nullptr;
  uint8_t* pcode = exact ? reinterpret_cast<uint8_t*>(hp + (8 * (size_t)N + a.ns + 1)) : nullptr;
  if (exact) {
    if (tid == 0) heap_dijkstra(g, gmetric, gconn, f, vdist, my_src, a.ns, hp, pcode);
    __syncthreads();
  }
  for (; !exact;) {
    int n = sh.cnt[cur];
    if (n == 0) {
      const unsigned long long ta0 = dbg ? gtimer() : 0ull;
      // bucket advance: min over the far pixels, then move those <= thr
      uint32_t lmin = INF_BITS;
      for (int w = tid; w < NW; w += nthr) {
        uint32_t b = vfar[w];
        while (b) {  // eight far pixels' distances in flight at a time
          uint32_t dd[8];
#pragma unroll
          for (int j = 0; j < 8; j++) {
            dd[j] = INF_BITS;
            if (b) {
              const int bit = __ffs(b) - 1;
              b &= b - 1;
              dd[j] = in_smem ? vdist[(w << 5) + bit] : __ldcg(&dist[(w << 5) + bit]);
            }
          }
#pragma unroll
          for (int j = 0; j < 8; j++) lmin = min(lmin, dd[j]);
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) lmin = min(lmin, __shfl_xor_sync(0xffffffffu, lmin, o));
      if (tid == 0) sh.minfar = INF_BITS;
      __syncthreads();
      if (lane == 0 && lmin != INF_BITS) atomicMin(&sh.minfar, lmin);
      __syncthreads();
      const uint32_t m = sh.minfar;
      if (m == INF_BITS) break;
      thr = __fadd_rn(__uint_as_float(m), a.delta);
      for (int w0 = 0; w0 < NW; w0 += nthr) {
        const int w = w0 + tid;
        uint32_t b = w < NW ? vfar[w] : 0u;
        const uint32_t keep = b;
        uint32_t taken = 0;
        while (b) {
          uint32_t dd[8];
          int bb[8];
#pragma unroll
          for (int j = 0; j < 8; j++) {
            bb[j] = -1;
            dd[j] = INF_BITS;
            if (b) {
              bb[j] = __ffs(b) - 1;
              b &= b - 1;
              dd[j] = in_smem ? vdist[(w << 5) + bb[j]] : __ldcg(&dist[(w << 5) + bb[j]]);
            }
          }
#pragma unroll
          for (int j = 0; j < 8; j++)
            if (bb[j] >= 0 && __uint_as_float(dd[j]) <= thr) taken |= 1u << bb[j];
        }
        if (taken) {
          far[w] = keep & ~taken;
          inq[w] |= taken;
        }
        // compact taken pixels into the near list (warp-aggregated)
        const int c = __popc(taken);
        int incl = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += y;
        }
        const int tot = __shfl_sync(0xffffffffu, incl, 31);
        int wb = 0;
        if (lane == 31 && tot) wb = atomicAdd(&sh.cnt[cur], tot);
        wb = __shfl_sync(0xffffffffu, wb, 31);
        int pos = wb + incl - c;
        while (taken) {
          const int bit = __ffs(taken) - 1;
          taken &= taken - 1;
          *wl.at(cur, pos++) = (uint16_t)((w << 5) + bit);
        }
      }
      __syncthreads();
      n = sh.cnt[cur];
      if (dbg && tid == 0) { dbg[12] += gtimer() - ta0; dbg[13]++; }
    }
    passes++;
    items_total += n;
    // the current items leave the queue: improvements from now on re-queue them
    for (int i = tid; i < n; i += nthr) {
      const int v = i < wl.cap ? (int)wl.s[cur][i] : (int)*wl.at(cur, i);
      atomicAnd(&inq[v >> 5], ~(1u << (v & 31)));
    }
    if (tid == 0) sh.cnt[cur ^ 1] = 0;
    __syncthreads();
    if (!in_smem) {
      // global variant: RR rounds of (item, edge) pairs per thread in flight
      // together -- distance loads, then independent atomics at L2.  The
      // worklist is read from shared memory directly while it fits there; the
      // window offsets come from packed constants, one unsigned compare per
      // bound; the appends of the RR rounds share one counter update.
      constexpr int RR = GP_RR;  // measured: 1 -> 615, 2 -> 600, 3 -> 609, 4 -> 614, 6 -> 659 ms per 256^2 image
      const int items = n * 8;
      const bool wl_fits = n <= wl.cap;
      const uint16_t* lsm = wl.s[cur];
      for (int b0 = 0; b0 < items; b0 += RR * nthr) {
        int uk[RR];
        uint32_t nbk[RR], oldk[RR], dvk[RR];
        float fwk[RR];
#pragma unroll
        for (int j = 0; j < RR; j++) {
          const int idx = b0 + j * nthr + tid;
          uk[j] = -1;
          dvk[j] = INF_BITS;
          if (idx < items) {
            const int it = idx >> 3;
            const int v = wl_fits ? (int)lsm[it] : (int)*wl.at(cur, it);
            int k = idx & 7;
            k += (k >= 4);
            if (k_in_conn(gconn, k)) {
              int r, c;
              pix_rc(g, v, r, c);
              const int dr = (int)((0x2A540u >> (2 * k)) & 3u) - 1;  // k / 3 - 1
              const int dc = (int)((0x24924u >> (2 * k)) & 3u) - 1;  // k % 3 - 1
              if ((unsigned)(r + dr) < (unsigned)g.H && (unsigned)(c + dc) < (unsigned)g.W) {
                uk[j] = v + dr * g.W + dc;
                dvk[j] = __ldcg(&dist[v]);
                fwk[j] = edge_w(gmetric, __ldg(&f[v]), __ldg(&f[uk[j]]));
              }
            }
          }
        }
#pragma unroll
        for (int j = 0; j < RR; j++) {
          nbk[j] = uk[j] >= 0 ? __float_as_uint(__fadd_rn(__uint_as_float(dvk[j]), fwk[j])) : INF_BITS;
          oldk[j] = uk[j] >= 0 ? atomicMin(&dist[uk[j]], nbk[j]) : 0u;
        }
        bool app[RR];
        unsigned mj[RR];
        int tot = 0;
#pragma unroll
        for (int j = 0; j < RR; j++) {
          app[j] = false;
          const int u = uk[j];
          if (u >= 0 && nbk[j] < oldk[j]) {
            const uint32_t ub = 1u << (u & 31);
            if (__uint_as_float(nbk[j]) <= thr) app[j] = !(atomicOr(&inq[u >> 5], ub) & ub);
            else atomicOr(&far[u >> 5], ub);
          }
          mj[j] = __ballot_sync(0xffffffffu, app[j]);
          tot += __popc(mj[j]);
        }
        if (tot) {  // warp-uniform
          int base = 0;
          if (lane == 0) base = atomicAdd(&sh.cnt[cur ^ 1], tot);
          base = __shfl_sync(0xffffffffu, base, 0);
          const unsigned lt = (1u << lane) - 1u;
#pragma unroll
          for (int j = 0; j < RR; j++) {
            if (app[j]) *wl.at(cur ^ 1, base + __popc(mj[j] & lt)) = (uint16_t)uk[j];
            base += __popc(mj[j]);
          }
        }
      }
      cur ^= 1;
      __syncthreads();
      continue;
    }
    const int items = n * 8;
    for (int b0 = 0; b0 < items; b0 += nthr) {
      const int idx = b0 + tid;
      bool app = false;
      int u = -1;
      if (idx < items) {
        const int v = *wl.at(cur, idx >> 3);
        int k = idx & 7;
        k += (k >= 4);
        if (k_in_conn(gconn, k)) {
          int r, c;
          pix_rc(g, v, r, c);
          u = nbr_at(g, r, c, k);
          if (u >= 0) {
            const float nd = __fadd_rn(__uint_as_float(vdist[v]), edge_w(gmetric, f[v], f[u]));
            const uint32_t nb = __float_as_uint(nd);
            // pre-check (cheap in smem); in the global variant the atomic's
            // returned value is the check, saving a dependent L2 round trip
            if (!in_smem || nb < vdist[u]) {
              const uint32_t old = atomicMin(&dist[u], nb);
              if (nb < old) {
                const uint32_t ub = 1u << (u & 31);
                if (nd <= thr) {
                  app = !(atomicOr(&inq[u >> 5], ub) & ub);
                } else {
                  atomicOr(&far[u >> 5], ub);
                }
              }
            }
          }
        }
      }
      warp_append(app, u, &sh.cnt[cur ^ 1], wl, cur ^ 1);
    }
    cur ^= 1;
    __syncthreads();
  }
  if (dbg && tid == 0) { dbg[1] = gtimer(); dbg[6] = passes; dbg[7] = items_total; }

  // ---------------- predecessor post-pass ----------------
  // far is all-zero here; reuse it as the root bitmap.
  for (int i = tid; i < a.ns; i += nthr) {
    const int v = my_src[i];
    atomicOr(&far[v >> 5], 1u << (v & 31));
  }
  if (tid == 0) sh.slot = a.slot ? a.slot[t] : t;
  __syncthreads();
  const int slot = sh.slot;
  const size_t off = (size_t)slot * N;
  volatile uint8_t* vcode = code;
  int unparented = 0;
  // one thread per pixel: the code array starts all roots (nibbles 15) and a
  // parented pixel clears its nibble down to k with one shared atomic (the
  // neighbouring pixel of the same byte may be written concurrently)
  {
    uint32_t* cw = reinterpret_cast<uint32_t*>(code);
    for (int i = tid; i < (N + 7) / 8; i += nthr) cw[i] = 0xFFFFFFFFu;
  }
  __syncthreads();
  for (int v = tid; v < N; v += nthr) {
    uint8_t cv = GP_ROOT;
    const uint32_t dvb = in_smem ? vdist[v] : __ldcg(&dist[v]);
    if (exact) {
      cv = *(volatile uint8_t*)&pcode[v];
    } else if (!((vfar[v >> 5] >> (v & 31)) & 1u)) {
      const float dv = __uint_as_float(dvb);
      int r, c;
      pix_rc(g, v, r, c);
      const float fv = f[v];
      uint32_t dub[9];
      float fu[9];
#pragma unroll
      for (int k = 0; k < 9; k++) {  // all neighbour loads in flight together
        dub[k] = INF_BITS;
        fu[k] = 0.0f;
        if (!k_in_conn(gconn, k)) continue;
        const int u = nbr_at(g, r, c, k);
        if (u < 0) continue;
        dub[k] = in_smem ? vdist[u] : __ldcg(&dist[u]);
        fu[k] = f[u];
      }
      uint32_t best = INF_BITS;
#pragma unroll
      for (int k = 0; k < 9; k++) {
        if (dub[k] == INF_BITS) continue;
        const int u = v + (k / 3 - 1) * g.W + (k % 3 - 1);
        const float cand = __fadd_rn(__uint_as_float(dub[k]), edge_w(gmetric, fu[k], fv));
        if (cand == dv && (dub[k] < dvb || (dub[k] == dvb && u < v)) && dub[k] < best) {
          best = dub[k];
          cv = (uint8_t)k;
        }
      }
      if (cv == GP_ROOT) unparented = 1;
    }
    if (cv != GP_ROOT) code_set_root(code, v, cv);
    if (!LEAN && a.out_dist) a.out_dist[off + v] = __uint_as_float(dvb);
  }
  // Zero-weight plateaus (L1 metric only).  A pixel without a tight neighbour
  // of smaller (d, id) is a local root, and pixels parented so far may hang
  // off one, so "has a parent" does not mean "reaches a source".  Connected
  // pixels (chain reaches a source) grow breadth-first from the sources in
  // synchronous sweeps: an unconnected pixel joins when its parent is
  // connected, else it is re-parented to its first connected tight neighbour
  // (window order); decisions of a sweep read only the previous sweep's set
  // (`inq`, zero after the relaxation; new members collect in `far`, whose
  // root marks are no longer needed), so the forest is deterministic.  Every
  // pixel has a tight neighbour on a shortest path from a source, so the
  // sweeps connect all pixels; parents are always connected, so no cycles.
  if (__syncthreads_or(unparented)) {
    volatile uint32_t* vcon = inq;
    for (int i = tid; i < NW; i += nthr) far[i] = 0;
    __syncthreads();
    for (int i = tid; i < a.ns; i += nthr) {
      const int v = my_src[i];
      atomicOr(&inq[v >> 5], 1u << (v & 31));
    }
    __syncthreads();
    for (;;) {
      int changed = 0;
      for (int v = tid; v < N; v += nthr) {
        if ((vcon[v >> 5] >> (v & 31)) & 1u) continue;
        const uint8_t cv = code_get(vcode, v);
        if (cv != GP_ROOT) {
          const int p = parent_of(v, cv, g.W);
          if ((vcon[p >> 5] >> (p & 31)) & 1u) {
            atomicOr(&far[v >> 5], 1u << (v & 31));
            changed = 1;
            continue;
          }
        }
        int r, c;
        pix_rc(g, v, r, c);
        const float dv = __uint_as_float(vdist[v]);
        for (int k = 0; k < 9; k++) {
          if (!k_in_conn(gconn, k)) continue;
          const int u = nbr_at(g, r, c, k);
          if (u < 0 || !((vcon[u >> 5] >> (u & 31)) & 1u)) continue;
          if (__fadd_rn(__uint_as_float(vdist[u]), edge_w(gmetric, f[u], f[v])) != dv) continue;
          code_set(vcode, v, (unsigned)k);
          atomicOr(&far[v >> 5], 1u << (v & 31));
          changed = 1;
          break;
        }
      }
      if (!__syncthreads_or(changed)) break;
      for (int i = tid; i < NW; i += nthr) {
        inq[i] |= far[i];
        far[i] = 0;
      }
      __syncthreads();
    }
    for (int i = tid; i < NW; i += nthr) inq[i] = 0;
    __syncthreads();
  }
  if (!LEAN && a.out_dir)
    for (int v = tid; v < N; v += nthr) a.out_dir[off + v] = code_get(vcode, v);

  // ---------------- naive epilogue: fill_from_source, row/column x > s ----
  if (!LEAN && a.D) {
    const int s = my_src[0];
    float* D = a.D;
    for (int x = s + 1 + tid; x < N; x += nthr) {
      const float val = __uint_as_float(vdist[x]);
      D[(size_t)s * N + x] = val;
      D[(size_t)x * N + s] = val;
    }
  }
  if (!a.ts.pre) return;
  if (dbg && tid == 0) dbg[2] = gtimer();

  // ================= Euler tour of the (single-root) tree =================
  // E1: depths by pointer jumping on packed (depth << 16 | jump) words (A).
  volatile uint32_t* pj = reinterpret_cast<volatile uint32_t*>(base + lay.A);
  for (int v = tid; v < N; v += nthr) {
    const uint8_t cv = code_get(vcode, v);
    pj[v] = cv == GP_ROOT ? (uint32_t)v : ((1u << 16) | (uint32_t)parent_of(v, cv, g.W));
  }
  __syncthreads();
  if (in_smem) pointer_jump(pj, N);
  else pointer_jump_global(const_cast<uint32_t*>(pj), N);
  if (dbg && tid == 0) dbg[3] = gtimer();
  // Loops over arrays that are stable within a phase read them from L2 in the
  // global variant (__ldcg: no stale L1) and directly in shared memory; UB
  // iterations' loads are issued before any is consumed.
  const bool gm = !in_smem;
  auto rd32 = [gm](const volatile uint32_t* p) -> uint32_t {
    return gm ? __ldcg(const_cast<const uint32_t*>(p)) : *p;
  };
  auto rd16 = [gm](const volatile uint16_t* p) -> uint16_t {
    return gm ? __ldcg(const_cast<const unsigned short*>(p)) : *p;
  };
  constexpr int UB = GP_UB;
  // E2: depth (B) and max depth
  volatile uint16_t* depth = reinterpret_cast<volatile uint16_t*>(base + lay.B);
  // C = ancestor/descendant pairs of the tree = sum of depths
  int lmax = 0;
  unsigned lpairs = 0;
  for (int v0 = tid; v0 < N; v0 += UB * nthr) {
    uint32_t x[UB];
#pragma unroll
    for (int j = 0; j < UB; j++) x[j] = v0 + j * nthr < N ? rd32(&pj[v0 + j * nthr]) : 0u;
#pragma unroll
    for (int j = 0; j < UB; j++) {
      if (v0 + j * nthr >= N) break;
      const int d = (int)(x[j] >> 16);
      depth[v0 + j * nthr] = (uint16_t)d;
      lmax = max(lmax, d);
      lpairs += (unsigned)d;
    }
  }
  atomicMax(&sh.maxd, lmax);
  atomicAdd(&sh.pairs, lpairs);
  __syncthreads();
  const int maxd = sh.maxd;
  if (dbg && tid == 0) { dbg[8] = gtimer(); dbg[11] = maxd; }
  const bool use_hist = (size_t)maxd + 1 <= hist_cap;
  uint16_t* szv = reinterpret_cast<uint16_t*>(base + lay.A);  // descendants
  volatile uint16_t* vszv = szv;
  uint16_t* order = reinterpret_cast<uint16_t*>(base + lay.A + 2 * (size_t)N);
  volatile uint32_t* vhist = hist;
  for (int v = tid; v < N; v += nthr) szv[v] = 0;
  // E3: counting sort by depth -> order[], level d = order[hist[d-1] .. hist[d])
  if (use_hist) {
    for (int i = tid; i <= maxd; i += nthr) hist[i] = 0;
    __syncthreads();
    for (int v0 = tid; v0 < N; v0 += UB * nthr) {
      uint16_t x[UB];
#pragma unroll
      for (int j = 0; j < UB; j++) x[j] = v0 + j * nthr < N ? rd16(&depth[v0 + j * nthr]) : 0;
#pragma unroll
      for (int j = 0; j < UB; j++)
        if (v0 + j * nthr < N) atomicAdd(&hist[x[j]], 1u);
    }
    __syncthreads();
    if (wid == 0) {  // exclusive scan of hist[0..maxd] by one warp
      unsigned carry = 0;
      for (int i0 = 0; i0 <= maxd; i0 += 32) {
        const int i = i0 + lane;
        const unsigned x = i <= maxd ? vhist[i] : 0u;
        unsigned incl = x;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const unsigned y = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += y;
        }
        if (i <= maxd) vhist[i] = carry + incl - x;
        carry += __shfl_sync(0xffffffffu, incl, 31);
      }
    }
    __syncthreads();
    for (int v0 = tid; v0 < N; v0 += UB * nthr) {
      uint16_t x[UB];
#pragma unroll
      for (int j = 0; j < UB; j++) x[j] = v0 + j * nthr < N ? rd16(&depth[v0 + j * nthr]) : 0;
#pragma unroll
      for (int j = 0; j < UB; j++)
        if (v0 + j * nthr < N) order[atomicAdd(&hist[x[j]], 1u)] = (uint16_t)(v0 + j * nthr);
    }
  }
  __syncthreads();
  if (dbg && tid == 0) dbg[9] = gtimer();
  // E4: descendant counts, deepest level first -- one warp, no block barriers
  // (shared-memory variant); block-wide per level in the global variant,
  // where one warp would pay a global round trip per level and element
  if (use_hist && !in_smem) {
    // the first entry of the next level is loaded before this level's barrier
    int vn = -1;
    if (maxd >= 1 && vhist[maxd - 1] + tid < vhist[maxd]) vn = order[vhist[maxd - 1] + tid];
    for (int d = maxd; d >= 1; d--) {
      const unsigned lo = vhist[d - 1], hi = vhist[d];
      const int v0 = vn;
      vn = -1;
      if (d >= 2 && vhist[d - 2] + tid < vhist[d - 1]) vn = order[vhist[d - 2] + tid];
      if (v0 >= 0) atomic_add_u16(szv, parent_of(v0, code_get(vcode, v0), g.W), (unsigned)__ldcg(&szv[v0]) + 1u);
      for (unsigned i = lo + nthr + tid; i < hi; i += nthr) {
        const int v = order[i];
        atomic_add_u16(szv, parent_of(v, code_get(vcode, v), g.W), (unsigned)__ldcg(&szv[v]) + 1u);
      }
      __syncthreads();
    }
  } else if (use_hist) {
    if (wid == 0) {
      for (int d = maxd; d >= 1; d--) {
        const unsigned lo = vhist[d - 1], hi = vhist[d];
        for (unsigned i = lo + lane; i < hi; i += 32) {
          const int v = order[i];
          atomic_add_u16(szv, parent_of(v, code_get(vcode, v), g.W), (unsigned)vszv[v] + 1u);
        }
        __syncwarp();
      }
    }
  } else {
    for (int d = maxd; d >= 1; d--) {
      for (int v = tid; v < N; v += nthr)
        if (depth[v] == d) atomic_add_u16(szv, parent_of(v, code_get(vcode, v), g.W), (unsigned)vszv[v] + 1u);
      __syncthreads();
    }
  }
  __syncthreads();
  if (dbg && tid == 0) dbg[10] = gtimer();
  // sizes move to B (depth is dead) so that A can hold the path-sum words
  volatile uint16_t* szB = reinterpret_cast<volatile uint16_t*>(base + lay.B);
  for (int v0 = tid; v0 < N; v0 += UB * nthr) {
    uint16_t x[UB];
#pragma unroll
    for (int j = 0; j < UB; j++) x[j] = v0 + j * nthr < N ? rd16(&vszv[v0 + j * nthr]) : 0;
#pragma unroll
    for (int j = 0; j < UB; j++)
      if (v0 + j * nthr < N) szB[v0 + j * nthr] = x[j];
  }
  __syncthreads();
  // E5: preorder positions.  Children of p are ordered by id; child v's block
  // starts after p and its earlier siblings' blocks:
  //   tin[v] = sum over the path root..v (root excluded) of 1 + off(a),
  //   off(a) = sum of (size + 1) over the earlier siblings of a,
  // evaluated by pointer jumping on (acc << 16 | jump) words in A.
  // One thread per parent p walks its <= 8 neighbours in increasing id
  // (= neighbour order) and assigns each child its sibling offset; every
  // non-root pixel is written by its parent's thread, the root by itself.
  // GP_E5 parents per iteration (their children's sizes loaded together; one
  // measured best: the single-parent loop keeps more warps issuing).
  for (int p0 = tid; p0 < N; p0 += GP_E5 * nthr) {
    unsigned mask[GP_E5];
    unsigned szc[GP_E5][9];
#pragma unroll
    for (int b = 0; b < GP_E5; b++) {
      const int pp = p0 + b * nthr;
      mask[b] = 0u;
      if (pp >= N) continue;
      if (code_get(vcode, pp) == GP_ROOT) pj[pp] = (uint32_t)pp;
      int pr, pc;
      pix_rc(g, pp, pr, pc);
      // q = pp + offset(k) is a child iff its code points back: code == 8 - k
      const bool interior = pr > 0 && pr < g.H - 1 && pc > 0 && pc < g.W - 1;
#pragma unroll
      for (int k = 0; k < 9; k++) {
        if (!k_in_conn(gconn, k)) continue;
        if (!interior && nbr_at(g, pr, pc, k) < 0) continue;
        if (code_get(vcode, pp + (k / 3 - 1) * g.W + (k % 3 - 1)) == (uint8_t)(8 - k)) mask[b] |= 1u << k;
      }
    }
#pragma unroll
    for (int b = 0; b < GP_E5; b++) {
      const int pp = p0 + b * nthr;
#pragma unroll
      for (int k = 0; k < 9; k++)
        szc[b][k] = ((mask[b] >> k) & 1u) ? rd16(&szB[pp + (k / 3 - 1) * g.W + (k % 3 - 1)]) : 0u;
    }
#pragma unroll
    for (int b = 0; b < GP_E5; b++) {
      const int pp = p0 + b * nthr;
      unsigned offs = 0;
#pragma unroll
      for (int k = 0; k < 9; k++) {
        if (!((mask[b] >> k) & 1u)) continue;
        pj[pp + (k / 3 - 1) * g.W + (k % 3 - 1)] = ((1u + offs) << 16) | (uint32_t)pp;
        offs += szc[b][k] + 1u;
      }
    }
  }
  __syncthreads();
  if (dbg && tid == 0) dbg[14] = gtimer();
  if (in_smem) pointer_jump(pj, N);
  else pointer_jump_global(const_cast<uint32_t*>(pj), N);
  if (dbg && tid == 0) dbg[4] = gtimer();
  // Tree-store outputs are written with evict-first stores (st.global.cs): the
  // commit loop reads a tree long after it is written, and streaming ~1 MB per
  // tree through L2 with normal priority evicts the scratch of the trees
  // still being built.
  // E6: preorder arrays.  tdp straight to global, then pre/szp staged in the
  // (now free) distance region for coalesced stores and the partition scan.
  // The arrays read here are stable after the barriers: the global variant
  // reads them from L2 (__ldcg: no stale L1, loads pipeline), smem directly.
  float* gtdp = a.ts.tdp + off;
  uint32_t* gtin = a.ts.tin + off;
  constexpr int UE = GP_UE;
  for (int v0 = tid; v0 < N; v0 += UE * nthr) {
    uint32_t x[UE], dv[UE];
    uint16_t sz[UE];
#pragma unroll
    for (int j = 0; j < UE; j++) {
      const int v = v0 + j * nthr;
      x[j] = v < N ? rd32(&pj[v]) : 0u;
      dv[j] = v < N ? rd32(&vdist[v]) : 0u;
      sz[j] = v < N ? rd16(&szB[v]) : 0;
    }
#pragma unroll
    for (int j = 0; j < UE; j++) {
      const int v = v0 + j * nthr;
      if (v >= N) break;
      const uint32_t q = x[j] >> 16;
      __stcs(&gtdp[q], __uint_as_float(dv[j]));
      __stcs(&gtin[v], q | ((uint32_t)sz[j] << 16));
    }
  }
  __syncthreads();
  const int slot_c = slot;
  if (sh.lite) {
    // list mode (the commit loop only tests Euler intervals from now on):
    // tin and tdp are all it reads
    if (tid == 0) {
      a.ts.T[slot_c] = 0;
      a.ts.C[slot_c] = sh.pairs;
      if (dbg) dbg[15] = dbg[5] = gtimer();
    }
  } else {
  volatile uint16_t* preS = reinterpret_cast<volatile uint16_t*>(base);
  volatile uint16_t* szS = preS + N;
  for (int v0 = tid; v0 < N; v0 += UE * nthr) {
    uint32_t x[UE];
    uint16_t sz[UE];
#pragma unroll
    for (int j = 0; j < UE; j++) {
      const int v = v0 + j * nthr;
      x[j] = v < N ? rd32(&pj[v]) : 0u;
      sz[j] = v < N ? rd16(&szB[v]) : 0;
    }
#pragma unroll
    for (int j = 0; j < UE; j++) {
      const int v = v0 + j * nthr;
      if (v >= N) break;
      preS[x[j] >> 16] = (uint16_t)v;
      szS[x[j] >> 16] = sz[j];
    }
  }
  __syncthreads();
  uint32_t* gpre = a.ts.pre + off;
  uint16_t* gszp = a.ts.szp + off;
  const MarkLayout ML = a.L;
  for (int q0 = tid; q0 < N; q0 += UB * nthr) {
    uint16_t pv[UB], sz[UB];
#pragma unroll
    for (int j = 0; j < UB; j++) {
      const int q = q0 + j * nthr;
      pv[j] = q < N ? rd16(&preS[q]) : 0;
      sz[j] = q < N ? rd16(&szS[q]) : 0;
    }
#pragma unroll
    for (int j = 0; j < UB; j++) {
      const int q = q0 + j * nthr;
      if (q >= N) break;
      __stcs(&gpre[q], (mcol(ML, pv[j]) << 16) | pv[j]);
      __stcs(&gszp[q], (unsigned short)sz[j]);
    }
  }
  if (dbg) {
    __syncthreads();
    if (tid == 0) dbg[15] = gtimer();
  }
  // E7: chunk counts ceil(szp/32), exclusive scan over preorder, partition
  const int seg = (N + nthr - 1) / nthr;
  const int q0 = min(N, tid * seg), q1 = min(N, q0 + seg);
  unsigned lsum = 0;
  constexpr int US = 16;
  // the root (q = 0) pairs with every pixel; the commit kernel fills its row
  // with a grid-wide row scan, so its chunks are left out of the partition
  for (int qb = q0; qb < q1; qb += US) {
    uint16_t x[US];
#pragma unroll
    for (int j = 0; j < US; j++) x[j] = qb + j < q1 ? rd16(&szS[qb + j]) : 0;
#pragma unroll
    for (int j = 0; j < US; j++) {
      lsum += (qb + j) ? ((unsigned)x[j] + 31u) >> 5 : 0u;
    }
  }
  unsigned incl = lsum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) sh.wsum[wid] = incl;
  __syncthreads();
  if (wid == 0) {
    const int nw = nthr >> 5;
    const unsigned x = lane < nw ? (unsigned)sh.wsum[lane] : 0u;
    unsigned wi = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned y = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += y;
    }
    if (lane < nw) sh.wsum[lane] = (int)(wi - x);
    if (lane == 31) sh.total = wi;
  }
  __syncthreads();
  const unsigned T = sh.total;
  const unsigned long long P = (unsigned long long)a.ts.nparts;
  uint32_t* gpart = a.ts.part + (size_t)slot * a.ts.nparts;
  if (tid == 0) {
    a.ts.T[slot] = T;
    a.ts.C[slot] = sh.pairs;
  }
  unsigned run = (unsigned)sh.wsum[wid] + incl - lsum;
  // smallest p with p*T >= x*P (= ceil(x*P/T)): double estimate, exact fix-up
  auto first_part = [&](unsigned long long x) -> unsigned long long {
    if (!T) return P;
    unsigned long long pp = (unsigned long long)((double)x * (double)P / (double)T);
    while (pp > 0 && (pp - 1) * T >= x * P) pp--;
    while (pp * T < x * P) pp++;
    return pp;
  };
  auto write_part = [&](unsigned long long pp, unsigned q, unsigned runq) {
    const unsigned long long num = pp * T;
    unsigned b = (unsigned)((double)num / (double)P);  // floor(p*T/P), exact fix-up
    while ((unsigned long long)b * P > num) b--;
    while ((unsigned long long)(b + 1) * P <= num) b++;
    __stcs(&gpart[pp], (uint32_t)q | ((b - runq) << 16));
  };
  // positions owning many units (near the root) are queued and written by
  // whole warps; the rest by their thread
  // queue of many-part positions: the B region (sizes by pixel, dead after E6)
  uint4* big = reinterpret_cast<uint4*>(base + lay.B);
  const int bigcap = (int)(((size_t)N * 2) / sizeof(uint4));
  if (tid == 0) sh.nbig = 0;
  __syncthreads();
  // parts are handed out in order: pn = first part not yet placed; the parts
  // starting in position q are those with pn*T < (run + nch)*P
  unsigned long long pn = first_part(run);
  for (int qb = q0; qb < q1; qb += US) {
    uint16_t x[US];
#pragma unroll
    for (int j = 0; j < US; j++) x[j] = qb + j < q1 ? rd16(&szS[qb + j]) : 0;
    for (int j = 0; j < US && qb + j < q1; j++) {
      const int q = qb + j;
      const unsigned nch = q ? ((unsigned)x[j] + 31u) >> 5 : 0u;
      if (!nch) continue;
      const unsigned long long end = (unsigned long long)(run + nch) * P;
      if (pn < P && pn * T < end) {
        if ((pn + 4) * T < end) {  // several parts (the trunk near the root): queued for warps
          const unsigned long long phi = min(first_part(run + nch), P);
          const int i = atomicAdd(&sh.nbig, 1);
          if (i < bigcap) {
            big[i] = make_uint4((unsigned)q, run, (unsigned)pn, (unsigned)phi);
          } else {
            for (unsigned long long pp = pn; pp < phi; pp++) write_part(pp, (unsigned)q, run);
          }
          pn = phi;
        } else {
          while (pn < P && pn * T < end) write_part(pn++, (unsigned)q, run);
        }
      }
      run += nch;
    }
  }
  __syncthreads();
  const int nbig = min(sh.nbig, bigcap);
  for (int i = wid; i < nbig; i += nthr >> 5) {
    const uint4 e = gm ? __ldcg(&big[i]) : big[i];
    for (unsigned pp = e.z + lane; pp < e.w; pp += 32) write_part(pp, e.x, e.y);
  }
  if (dbg) {
    __syncthreads();
    if (tid == 0) dbg[5] = gtimer();
  }
  }  // !lite
  if (a.publish) {  // the tree is complete: make it visible to the commit loop
    __threadfence();
    __syncthreads();
    if (tid == 0) atomicExch(&a.publish[my_src[0]], slot);
  }
}

size_t prop_smem_bytes(int N) { return prop_layout(N, HIST_SMEM).total; }

size_t prop_scratch_bytes(int N) { return align16(prop_layout(N, (size_t)N + 1).total); }

bool prop_fits_smem(int N) {
  // Maps whose state needs more than half an SM's shared memory run the
  // global-scratch variant (three 512-thread trees per SM) although one tree
  // would fit: measured at 128x128, propagation 51.2 -> 43.2 ms (Voronoi u8)
  // and 51.8 -> 46.6 ms (fp32, 4-connected).  GP_PROP_SMEM_KB overrides.
  static const long cap_kb = getenv("GP_PROP_SMEM_KB") ? atol(getenv("GP_PROP_SMEM_KB")) : 113;
  return prop_smem_bytes(N) <= (size_t)std::min(227l, std::max(0l, cap_kb)) * 1024;
}

// dynamic shared memory of one tree (CTA)
static size_t prop_dyn_smem(int N) {
  if (prop_fits_smem(N)) return prop_smem_bytes(N);
  const size_t bm = align16((size_t)((N + 31) >> 5) * 4);
  return 2 * bm + std::max((size_t)WL_SMEM * 4, align16((size_t)(N + 1) / 2) + (size_t)HIST_G * 4);
}

// One tree per CTA.  Trees are latency-bound: two 512-thread CTAs per SM
// beat one 1024-thread CTA whenever shared memory admits two (128x128 maps
// need ~212 KB and keep 1024 threads).  The global-scratch variant (52 KB of
// shared memory) runs three 512-thread CTAs per SM (40 registers, a few
// spilled): at 256x256 the batch of 444 trees took 731 ms per image against
// 765 ms for two CTAs per SM; four per SM (32 registers) and four 256-thread
// CTAs (the same warps over more trees) measured slower.  GP_PROP_MINB=2
// selects two per SM.
static int prop_threads(int N) {
  const size_t per_cta = prop_dyn_smem(N) + 1024 + sizeof(PropShared);
  int threads = (228 * 1024) / per_cta >= 2 ? 512 : 1024;
  if (const char* e = getenv("GP_PROP_THREADS")) threads = std::max(128, std::min(1024, atoi(e)));
  return threads;
}

static const void* prop_kernel(const PropArgs& a, int N, int threads) {
  const size_t per_cta = prop_dyn_smem(N) + 1024 + sizeof(PropShared);
  int minb = 3;
  if (const char* e = getenv("GP_PROP_MINB")) minb = atoi(e);
  const bool lean = !a.dbg && !a.D && !a.out_dist && !a.out_dir && a.ts.pre && !a.exact_heap &&
                    !(getenv("GP_PROP_LEAN") && !atoi(getenv("GP_PROP_LEAN")));
  const bool mc = a.g.metric == kSum && a.g.conn == 8 && !(getenv("GP_PROP_MC") && !atoi(getenv("GP_PROP_MC")));
  if (!prop_fits_smem(N) && threads == 512 && minb == 3 && (228 * 1024) / per_cta >= 3) {
    if (lean) return mc ? (const void*)k_propagate<512, 3, 1, 1> : (const void*)k_propagate<512, 3, 1>;
    return (const void*)k_propagate<512, 3>;
  }
  if (lean) {
    if (prop_fits_smem(N)) return mc ? (const void*)k_propagate<1024, 1, 2, 1> : (const void*)k_propagate<1024, 1, 2>;
    return (const void*)k_propagate<1024, 1, 1>;
  }
  return (const void*)k_propagate<1024, 1>;
}

// speculative batch size per SM: the concurrent trees of the global-scratch
// variant; two otherwise (measured on 64x64 and 128x128 maps)
int prop_trees_per_sm(int N) {
  if (prop_fits_smem(N)) return 2;
  const int threads = prop_threads(N);
  PropArgs pa;
  memset(&pa, 0, sizeof(pa));
  pa.ts.pre = reinterpret_cast<uint32_t*>(1);  // a speculative batch: lean when allowed
  const void* k = prop_kernel(pa, N, threads);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)prop_dyn_smem(N));
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, threads, prop_dyn_smem(N));
  return std::max(1, per_sm);
}

// The cluster K1 (propagate_cluster.cu) can take the speculative batches of
// maps above one SM's shared memory when every edge weight is positive (its
// predecessor rule has no plateau pass): GP_PROP_CLUSTER=1.  Measured slower
// than the single-CTA global-scratch variant at 256^2,
// so off by default; GP_PROP_CLUSTER=2 also sends maps that fit one SM to it
// (tests).
static bool use_cluster(const PropArgs& a) {
  const char* e = getenv("GP_PROP_CLUSTER");
  const int knob = e ? atoi(e) : 0;
  if (!knob || (prop_fits_smem(a.g.N) && knob != 2)) return false;
  if (!a.pos_weights || a.ns != 1 || !a.ts.pre) return false;
  if (a.dbg || a.D || a.out_dist || a.out_dir) return false;
  static int ok = -1;
  if (ok < 0) ok = prop_cluster_ok(a.g.N) ? 1 : 0;
  return ok == 1;
}

cudaError_t launch_propagate(PropArgs a, int ntrees, cudaStream_t st) {
  if (ntrees <= 0) return cudaSuccess;
  if (a.exact_heap && a.heap_trees > 0 && ntrees > a.heap_trees) {
    // the heap scratch holds heap_trees trees: launch in chunks of that many
    for (int t0 = 0; t0 < ntrees; t0 += a.heap_trees) {
      PropArgs b = a;
      b.tree_base = a.tree_base + t0;
      cudaError_t e = launch_propagate(b, std::min(a.heap_trees, ntrees - t0), st);
      if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
  }
  if (use_cluster(a)) return launch_propagate_cluster(a, ntrees, st);
  a.in_smem = prop_fits_smem(a.g.N) ? 1 : 0;
  if (!a.in_smem) a.scratch_bytes = prop_scratch_bytes(a.g.N);
  const size_t smem = prop_dyn_smem(a.g.N);
  const int threads = a.threads ? a.threads : prop_threads(a.g.N);
  const void* kern = prop_kernel(a, a.g.N, threads);
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  void* params[] = {&a};
  return cudaLaunchKernel(kern, dim3(ntrees), dim3(threads), params, smem, st);
}

}  // namespace gp
