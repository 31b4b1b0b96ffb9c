// K1, cluster variant -- one tree per 2-CTA thread-block cluster, the whole
// per-tree state in distributed shared memory (maps above one SM's smem:
// 256x256 = 256 KB of fp32 distances).
//
// Restates dijkstra_csr (reference _kernels.py:33-79) exactly as the
// single-CTA K1 in propagate.cu does (same bucketed relaxation, same fp32
// fixpoint, same closed-form predecessor rule), but instead of parking the
// distance map and the Euler-tour arrays of every tree in an L2/DRAM scratch
// (444 trees x ~1 MB in flight > the 126 MB L2: round-1 ncu showed 364 GB of
// DRAM traffic per 256^2 image, ~7x the tree-store output), a pair of CTAs
// holds them in shared memory:
//
//   CTA r of the cluster owns pixels [r*M, r*M + M), M = ceil(N/2) (a band of
//   image rows).  Every per-pixel array is split the same way; an access to a
//   pixel of the other band goes through DSMEM (mapa / generic
//   ld/st/atom.shared::cluster).  Grid neighbours cross bands only at the
//   band boundary, so the relaxation's atomics are almost all local.
//
// Shared-memory regions per CTA (M = 32768 at 256^2: 216 KB):
//   R0  u32[M]   dist (relaxation) -> W = size << 4 | pending children
//                (upsweep) -> pj = acc << 16 | jump (preorder pointer jumping)
//                -> (pixel | size << 16) by preorder position (output staging)
//   R1  u16      two near worklists (CL_WL entries each; overflow in a small
//                global scratch) -> descendant counts by pixel -> big-part queue
//   R2  4-bit    parent codes (window position, 15 = root)
//   R3  bitmaps  far / inq (relaxation), leaf flags (upsweep)
//
// Phases (cluster barriers between them; every CTA works on its own pixels):
//   relax    delta-stepping passes; a pass = clear inq of the current items,
//            barrier, relax their edges (atomicMin on the fp32 bits, local or
//            DSMEM), improved pixels appended to their OWNER's next list,
//            barrier.  Bucket advance over the far bitmaps as in propagate.cu.
//   parents  closed-form rule: tight neighbour with the smallest
//            (d[u], u).  Requires strictly positive edge weights; the host
//            sends images with zero-weight edges to the single-CTA K1.
//   sizes    barrier-free upsweep: every leaf walks towards the root; a walker
//            adds (its size + 1) to the parent's word with one atomic and
//            continues only if it was the parent's last pending child (the
//            returned word says so).  Replaces the depth sort + level loop.
//   preorder tin = sum over the path of 1 + earlier siblings' blocks, by
//            pointer jumping over the distributed pj words (propagate.cu E5).
//   outputs  tdp / tin / pre / szp / part / T / C -- the tree-store format the
//            commit loop reads (gp_kernels.h TreeStore), unchanged.
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "gp_common.cuh"
#include "gp_kernels.h"

namespace cg = cooperative_groups;

namespace gp {

extern __shared__ __align__(16) unsigned char g_smem[];

constexpr int CL_THR = 1024;  // threads per CTA (two CTAs per tree, one CTA per SM)
constexpr int CL_WL = 16384;  // near-list entries per list kept in shared memory
#ifndef GP_PJ_CHAINS_CL
#define GP_PJ_CHAINS_CL 4  // pointer-jumping loads in flight per thread
#endif

struct ClLayout {
  size_t r1, r2, far, inq, total, r1bytes;
};
// (INQ bitmaps are double-buffered by pass parity and the list counters
// rotate over three slots, so a relaxation pass needs one cluster barrier:
// the bits and the counter a pass appends to were cleared during the pass
// before, and nobody reads the bits of the list being relaxed.)

__host__ __device__ inline size_t cl_align16(size_t x) { return (x + 15) & ~(size_t)15; }

__host__ __device__ inline ClLayout cl_layout(int M) {
  ClLayout L;
  const size_t bm = cl_align16((size_t)((M + 31) >> 5) * 4);
  L.r1 = cl_align16((size_t)M * 4);
  const size_t wl = (size_t)2 * CL_WL * 2, szb = (size_t)M * 2;
  L.r1bytes = cl_align16(wl > szb ? wl : szb);
  L.r2 = L.r1 + L.r1bytes;
  L.far = L.r2 + cl_align16((size_t)((M + 7) >> 3) * 4);
  L.inq = L.far + bm;  // two bitmaps: INQ[l] = queued in near list l
  L.total = L.inq + 2 * bm;
  return L;
}

struct ClShared {
  int cnt[3];          // near-list lengths, pass p's list in slot p % 3 (appended to by both CTAs)
  uint32_t minfar[2];  // bucket-advance minimum, by round parity
  int orflag[2];       // pointer-jumping "changed" flags, by round parity
  unsigned wsum[32];
  unsigned pairs;      // sum of descendant counts of this CTA's pixels
  unsigned chunks;     // fill chunks of this CTA's preorder positions
  int nbig;
  int lite;
};

// 4-bit parent codes: same packing as propagate.cu (nibble 15 = root)
__device__ __forceinline__ uint8_t cl_nib(unsigned byte, int i) {
  const unsigned c = (byte >> ((i & 1) << 2)) & 15u;
  return c == 15u ? GP_ROOT : (uint8_t)c;
}

// ---- DSMEM access to the partner CTA (shared::cluster window addresses) ----
__device__ __forceinline__ uint32_t cl_map(const void* local, int rank) {
  const uint32_t a = (uint32_t)__cvta_generic_to_shared(local);
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
__device__ __forceinline__ uint32_t rld32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared::cluster.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ unsigned rld16(uint32_t a) {
  unsigned short v;
  asm volatile("ld.shared::cluster.u16 %0, [%1];" : "=h"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ unsigned rld8(uint32_t a) {
  unsigned v;
  asm volatile("ld.shared::cluster.u8 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ void rst32(uint32_t a, uint32_t v) {
  asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ void rst16(uint32_t a, unsigned v) {
  asm volatile("st.shared::cluster.u16 [%0], %1;" ::"r"(a), "h"((unsigned short)v) : "memory");
}
__device__ __forceinline__ uint32_t ratom_min(uint32_t a, uint32_t v) {
  uint32_t r;
  asm volatile("atom.shared::cluster.min.u32 %0, [%1], %2;" : "=r"(r) : "r"(a), "r"(v) : "memory");
  return r;
}
__device__ __forceinline__ uint32_t ratom_or(uint32_t a, uint32_t v) {
  uint32_t r;
  asm volatile("atom.shared::cluster.or.b32 %0, [%1], %2;" : "=r"(r) : "r"(a), "r"(v) : "memory");
  return r;
}
__device__ __forceinline__ uint32_t ratom_add(uint32_t a, uint32_t v) {
  uint32_t r;
  asm volatile("atom.shared::cluster.add.u32 %0, [%1], %2;" : "=r"(r) : "r"(a), "r"(v) : "memory");
  return r;
}

template <int MC>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(CL_THR, 1)
    k_propagate_cl(PropArgs a, int M) {
  cg::cluster_group cl = cg::this_cluster();
  const int rank = (int)cl.block_rank(), oth = rank ^ 1;
  const int t = blockIdx.x >> 1;
  if (a.ntrees_dev && t >= *a.ntrees_dev) return;  // both CTAs of the cluster leave
  const Grid g = a.g;
  const int gmetric = MC ? (int)kSum : g.metric, gconn = MC ? 8 : g.conn;
  const int N = g.N;
  const int tid = threadIdx.x, nthr = blockDim.x, lane = tid & 31, wid = tid >> 5;
  const int b0 = rank * M;                      // first pixel of this CTA's band
  const int ob0 = oth * M;                      // first pixel of the partner's band
  const int own = max(0, min(N, b0 + M) - b0);  // pixels owned
  const int ownw = (own + 31) >> 5;
  const ClLayout lay = cl_layout(M);
  __shared__ ClShared sh;

  // local regions (plain shared-memory accesses) ...
  uint32_t* R0 = reinterpret_cast<uint32_t*>(g_smem);
  uint16_t* R1 = reinterpret_cast<uint16_t*>(g_smem + lay.r1);
  uint8_t* R2 = g_smem + lay.r2;
  uint32_t* FAR = reinterpret_cast<uint32_t*>(g_smem + lay.far);
  uint32_t* INQ = reinterpret_cast<uint32_t*>(g_smem + lay.inq);
  volatile uint32_t* vR0 = R0;
  volatile uint16_t* vR1 = R1;
  volatile uint8_t* vR2 = R2;
  // ... and the partner's, as shared::cluster addresses (mapa)
  const uint32_t R0o = cl_map(R0, oth), R1o = cl_map(R1, oth), R2o = cl_map(R2, oth);
  const uint32_t FARo = cl_map(FAR, oth), INQo = cl_map(INQ, oth), SHo = cl_map(&sh, oth);
  const uint32_t SHo_cnt = SHo + (uint32_t)offsetof(ClShared, cnt);
  auto owner = [M](int v) -> int { return v >= M ? 1 : 0; };
  auto code_of = [&](int v) -> uint8_t {
    if (owner(v) == rank) return cl_nib(vR2[(v - b0) >> 1], v - b0);
    const int i = v - ob0;
    return cl_nib(rld8(R2o + (uint32_t)(i >> 1)), i);
  };
  auto ld_w = [&](int v) -> uint32_t {  // R0 word of any pixel
    return owner(v) == rank ? vR0[v - b0] : rld32(R0o + 4u * (uint32_t)(v - ob0));
  };
  auto st_w = [&](int v, uint32_t x) {
    if (owner(v) == rank) vR0[v - b0] = x;
    else rst32(R0o + 4u * (uint32_t)(v - ob0), x);
  };
  // near list l of CTA o: the first CL_WL entries in its shared memory, the
  // rest in the tree's global overflow scratch
  uint16_t* ovf = reinterpret_cast<uint16_t*>(a.scratch + (size_t)t * a.scratch_bytes);
  auto lst_ld = [&](int l, int i) -> int {  // own list
    return i < CL_WL ? (int)vR1[l * CL_WL + i] : (int)__ldcg(ovf + ((size_t)(rank * 2 + l) * M + (i - CL_WL)));
  };
  auto lst_st = [&](int o, int l, int i, int v) {
    if (i >= CL_WL) ovf[(size_t)(o * 2 + l) * M + (i - CL_WL)] = (uint16_t)v;
    else if (o == rank) vR1[l * CL_WL + i] = (uint16_t)v;
    else rst16(R1o + 2u * (uint32_t)(l * CL_WL + i), (unsigned)v);
  };
  const float* f = a.img;
  // optional phase timing (GP_CL_DEBUG): sums over trees, rank 0 thread 0
  unsigned long long* dbg = (a.cl_dbg && rank == 0 && tid == 0) ? a.cl_dbg : nullptr;
  unsigned long long tlast = dbg ? gtimer() : 0ull;
  auto stamp = [&](int k) {
    if (!dbg) return;
    const unsigned long long now = gtimer();
    atomicAdd(&dbg[k], now - tlast);
    tlast = now;
  };
  unsigned npass = 0, nadv = 0, npj = 0;

  // ---------------- init ----------------
  for (int i = tid; i < own; i += nthr) R0[i] = INF_BITS;
  const int bmw = (int)((lay.inq - lay.far) / 4);  // words per bitmap (padded)
  for (int i = tid; i < ownw; i += nthr) { FAR[i] = 0; INQ[i] = 0; INQ[bmw + i] = 0; }
  if (tid == 0) {
    sh.cnt[0] = 0;
    sh.cnt[1] = 0;
    sh.cnt[2] = 0;
    sh.pairs = 0;
    sh.chunks = 0;
    sh.nbig = 0;
    sh.lite = a.list_mode ? (*(volatile const int*)a.list_mode == 1) : 0;
  }
  __syncthreads();
  const int* my_src = a.src + (size_t)t * a.ns;
  for (int i = tid; i < a.ns; i += nthr) {
    const int v = my_src[i];
    if (owner(v) == rank) {
      R0[v - b0] = 0u;
      lst_st(rank, 0, atomicAdd(&sh.cnt[0], 1), v);
    }
  }
  cl.sync();  // partner running, both initialised
  stamp(0);

  // ---------------- bucketed relaxation ----------------
  float thr = a.delta;
  int cur = 0, par = 0, c3 = 0;  // list parity, barrier-flag parity, counter slot of this pass
  for (;;) {
    int n = *(volatile int*)&sh.cnt[c3];
    int no = (int)rld32(SHo_cnt + 4u * c3);
    if (n + no == 0) {
      // bucket advance: cluster-wide min over the far pixels, then the far
      // pixels <= min + delta (own ones) form the next near lists
      uint32_t lmin = INF_BITS;
      for (int w = tid; w < ownw; w += nthr) {
        uint32_t b = FAR[w];
        while (b) {
          const int bit = __ffs(b) - 1;
          b &= b - 1;
          lmin = min(lmin, vR0[(w << 5) + bit]);
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) lmin = min(lmin, __shfl_xor_sync(0xffffffffu, lmin, o));
      if (tid == 0) sh.minfar[par] = INF_BITS;
      __syncthreads();
      if (lane == 0 && lmin != INF_BITS) atomicMin(&sh.minfar[par], lmin);
      cl.sync();
      const uint32_t m = min(*(volatile uint32_t*)&sh.minfar[par],
                             rld32(SHo + (uint32_t)offsetof(ClShared, minfar) + 4u * par));
      par ^= 1;
      if (m == INF_BITS) break;
      nadv++;
      thr = __fadd_rn(__uint_as_float(m), a.delta);
      for (int w0 = 0; w0 < ownw; w0 += nthr) {
        const int w = w0 + tid;
        uint32_t b = w < ownw ? FAR[w] : 0u;
        const uint32_t keep = b;
        uint32_t taken = 0;
        while (b) {
          const int bit = __ffs(b) - 1;
          b &= b - 1;
          if (__uint_as_float(vR0[(w << 5) + bit]) <= thr) taken |= 1u << bit;
        }
        if (taken) {
          FAR[w] = keep & ~taken;
          INQ[cur * bmw + w] |= taken;
        }
        const int c = __popc(taken);
        int incl = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += y;
        }
        const int tot = __shfl_sync(0xffffffffu, incl, 31);
        int wb = 0;
        if (lane == 31 && tot) wb = atomicAdd(&sh.cnt[c3], tot);
        wb = __shfl_sync(0xffffffffu, wb, 31);
        int pos = wb + incl - c;
        while (taken) {
          const int bit = __ffs(taken) - 1;
          taken &= taken - 1;
          lst_st(rank, cur, pos++, b0 + (w << 5) + bit);
        }
      }
      cl.sync();
      n = *(volatile int*)&sh.cnt[c3];
      no = (int)rld32(SHo_cnt + 4u * c3);
      if (n + no == 0) continue;  // (cannot happen: the minimum pixel moved)
    }
    // The current items leave the queue (their INQ[cur] bits clear; appends
    // of this pass test INQ[nxt], cleared during the previous pass), and the
    // counter of the previous pass's list becomes the one of pass + 2.
    const int nxt = cur ^ 1, c3n = c3 == 2 ? 0 : c3 + 1, c3o = c3n == 2 ? 0 : c3n + 1;
    for (int i = tid; i < n; i += nthr) {
      const int v = lst_ld(cur, i) - b0;
      atomicAnd(&INQ[cur * bmw + (v >> 5)], ~(1u << (v & 31)));
    }
    if (tid == 0) sh.cnt[c3o] = 0;
    constexpr int RR = 2;
    const int items = n * 8;
    for (int bb = 0; bb < items; bb += RR * nthr) {
      int uk[RR];
      uint32_t nbk[RR], oldk[RR], dvk[RR];
      float fwk[RR];
#pragma unroll
      for (int j = 0; j < RR; j++) {
        const int idx = bb + j * nthr + tid;
        uk[j] = -1;
        dvk[j] = INF_BITS;
        if (idx < items) {
          const int v = lst_ld(cur, idx >> 3);
          int k = idx & 7;
          k += (k >= 4);
          if (k_in_conn(gconn, k)) {
            int r, c;
            pix_rc(g, v, r, c);
            const int dr = (int)((0x2A540u >> (2 * k)) & 3u) - 1;  // k / 3 - 1
            const int dc = (int)((0x24924u >> (2 * k)) & 3u) - 1;  // k % 3 - 1
            if ((unsigned)(r + dr) < (unsigned)g.H && (unsigned)(c + dc) < (unsigned)g.W) {
              uk[j] = v + dr * g.W + dc;
              dvk[j] = vR0[v - b0];
              fwk[j] = edge_w(gmetric, __ldg(&f[v]), __ldg(&f[uk[j]]));
            }
          }
        }
      }
#pragma unroll
      for (int j = 0; j < RR; j++) {
        const int u = uk[j];
        nbk[j] = u >= 0 ? __float_as_uint(__fadd_rn(__uint_as_float(dvk[j]), fwk[j])) : INF_BITS;
        oldk[j] = 0u;
        if (u >= 0) {
          if (owner(u) == rank) oldk[j] = atomicMin(&R0[u - b0], nbk[j]);
          else oldk[j] = ratom_min(R0o + 4u * (uint32_t)(u - ob0), nbk[j]);
        }
      }
#pragma unroll
      for (int j = 0; j < RR; j++) {
        bool app = false;
        const int u = uk[j];
        const bool mine = u >= 0 && owner(u) == rank;
        if (u >= 0 && nbk[j] < oldk[j]) {
          const int ul = u - (mine ? b0 : ob0);
          const uint32_t ub = 1u << (ul & 31);
          if (__uint_as_float(nbk[j]) <= thr) {
            const uint32_t prev = mine ? atomicOr(&INQ[nxt * bmw + (ul >> 5)], ub)
                                       : ratom_or(INQo + 4u * (uint32_t)(nxt * bmw + (ul >> 5)), ub);
            app = !(prev & ub);
          } else if (mine) {
            atomicOr(&FAR[ul >> 5], ub);
          } else {
            ratom_or(FARo + 4u * (uint32_t)(ul >> 5), ub);
          }
        }
        // warp-aggregated appends to the owner's next list, one counter update per owner
        const unsigned ml = __ballot_sync(0xffffffffu, app && mine);
        const unsigned mr = __ballot_sync(0xffffffffu, app && !mine);
        if (ml) {
          int base = 0;
          if (lane == __ffs(ml) - 1) base = atomicAdd(&sh.cnt[c3n], __popc(ml));
          base = __shfl_sync(0xffffffffu, base, __ffs(ml) - 1);
          if (app && mine) lst_st(rank, nxt, base + __popc(ml & ((1u << lane) - 1u)), u);
        }
        if (mr) {
          int base = 0;
          if (lane == __ffs(mr) - 1) base = (int)ratom_add(SHo_cnt + 4u * c3n, (uint32_t)__popc(mr));
          base = __shfl_sync(0xffffffffu, base, __ffs(mr) - 1);
          if (app && !mine) lst_st(oth, nxt, base + __popc(mr & ((1u << lane) - 1u)), u);
        }
      }
    }
    cur = nxt;
    c3 = c3n;
    npass++;
    cl.sync();
  }
  stamp(1);

  // ---------------- predecessor codes (own pixels) ----------------
  {
    uint32_t* cw = reinterpret_cast<uint32_t*>(R2);
    for (int i = tid; i < (own + 7) / 8; i += nthr) cw[i] = 0xFFFFFFFFu;
  }
  __syncthreads();
  for (int i = tid; i < own; i += nthr) {
    const int v = b0 + i;
    const uint32_t dvb = vR0[i];
    const float dv = __uint_as_float(dvb);
    int r, c;
    pix_rc(g, v, r, c);
    const float fv = __ldg(&f[v]);
    uint32_t dub[9];
    float fu[9];
#pragma unroll
    for (int k = 0; k < 9; k++) {
      dub[k] = INF_BITS;
      fu[k] = 0.0f;
      if (!k_in_conn(gconn, k)) continue;
      const int u = nbr_at(g, r, c, k);
      if (u < 0) continue;
      dub[k] = ld_w(u);
      fu[k] = __ldg(&f[u]);
    }
    uint32_t best = INF_BITS;
    uint8_t cv = GP_ROOT;
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
    if (cv != GP_ROOT) {
      unsigned* w = reinterpret_cast<unsigned*>(R2) + (i >> 3);
      atomicAnd(w, ~((15u ^ (unsigned)cv) << ((i & 7) << 2)));
    }
  }
  // distances by pixel into the tree's tin slot (read back for tdp below)
  const int slot = a.slot ? a.slot[t] : t;
  const size_t off = (size_t)slot * N;
  uint32_t* gtin = a.ts.tin + off;
  for (int i = tid; i < own; i += nthr) gtin[b0 + i] = vR0[i];
  cl.sync();  // codes complete; dist (R0) dead everywhere
  stamp(2);

  // ---------------- descendant counts: last-arriver upsweep ----------------
  // W[v] = size << 4 | pending children; leaves flagged in INQ (zero here)
  for (int i = tid; i < own; i += nthr) {
    const int v = b0 + i;
    int r, c;
    pix_rc(g, v, r, c);
    unsigned nch = 0;
#pragma unroll
    for (int k = 0; k < 9; k++) {
      if (!k_in_conn(gconn, k)) continue;
      const int q = nbr_at(g, r, c, k);
      if (q >= 0 && code_of(q) == (uint8_t)(8 - k)) nch++;
    }
    vR0[i] = nch;
    if (!nch) atomicOr(&INQ[i >> 5], 1u << (i & 31));
  }
  cl.sync();
  // Leaves are handed out dynamically from a compacted list (R1, free after
  // the relaxation), so a thread walking a long chain does not hold back
  // other leaves; persistent lanes: one step per loop trip, a lane whose walk
  // ended takes the next leaf at once.
  {
    for (int w0 = 0; w0 < ownw; w0 += nthr) {
      const int w = w0 + tid;
      const uint32_t b = w < ownw ? INQ[w] : 0u;
      const int c = __popc(b);
      int incl = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      const int tot = __shfl_sync(0xffffffffu, incl, 31);
      int wb = 0;
      if (lane == 31 && tot) wb = atomicAdd(&sh.nbig, tot);
      wb = __shfl_sync(0xffffffffu, wb, 31);
      int pos = wb + incl - c;
      for (uint32_t x = b; x; x &= x - 1) R1[pos++] = (uint16_t)((w << 5) + __ffs(x) - 1);
    }
    __syncthreads();
    const int nleaves = sh.nbig;
    if (tid == 0) sh.chunks = nthr;  // next leaf to hand out (the first nthr are static)
    __syncthreads();
    int li = tid, cur_v = -1;
    unsigned szc = 0;
    for (;;) {
      if (cur_v < 0) {
        if (li >= nleaves) break;
        cur_v = b0 + (int)vR1[li];
        szc = 0;
        li = (int)atomicAdd(&sh.chunks, 1u);
      }
      const uint8_t cc = code_of(cur_v);
      if (cc == GP_ROOT) { cur_v = -1; continue; }
      const int p = parent_of(cur_v, cc, g.W);
      const uint32_t inc = ((szc + 1u) << 4) - 1u;
      const unsigned old = owner(p) == rank ? atomicAdd(&R0[p - b0], inc)
                                            : ratom_add(R0o + 4u * (uint32_t)(p - ob0), inc);
      if ((old & 15u) != 1u) { cur_v = -1; continue; }  // a sibling's walker continues
      szc = (old >> 4) + szc + 1u;
      cur_v = p;
    }
  }
  __syncthreads();
  if (tid == 0) { sh.nbig = 0; sh.chunks = 0; }
  cl.sync();
  stamp(3);
  // sizes by pixel into R1 (worklists dead); C = sum of sizes = sum of depths
  unsigned lpairs = 0;
  for (int i = tid; i < own; i += nthr) {
    const unsigned sz = vR0[i] >> 4;
    R1[i] = (uint16_t)sz;
    lpairs += sz;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) lpairs += __shfl_xor_sync(0xffffffffu, lpairs, o);
  if (lane == 0 && lpairs) atomicAdd(&sh.pairs, lpairs);
  cl.sync();  // sizes complete, W dead
  stamp(4);

  // ---------------- preorder positions (propagate.cu E5) ----------------
  for (int i = tid; i < own; i += nthr) {
    const int p = b0 + i;
    if (code_of(p) == GP_ROOT) vR0[i] = (uint32_t)p;
    int pr, pc;
    pix_rc(g, p, pr, pc);
    unsigned offs = 0;
#pragma unroll
    for (int k = 0; k < 9; k++) {
      if (!k_in_conn(gconn, k)) continue;
      const int q = nbr_at(g, pr, pc, k);
      if (q < 0 || code_of(q) != (uint8_t)(8 - k)) continue;
      const unsigned szq = owner(q) == rank ? (unsigned)vR1[q - b0] : rld16(R1o + 2u * (uint32_t)(q - ob0));
      st_w(q, ((1u + offs) << 16) | (uint32_t)p);
      offs += szq + 1u;
    }
  }
  cl.sync();
  stamp(5);
  for (;;) {
    int ch = 0;
    for (int v0 = tid; v0 < own; v0 += GP_PJ_CHAINS_CL * nthr) {
      uint32_t pr[GP_PJ_CHAINS_CL], px[GP_PJ_CHAINS_CL];
#pragma unroll
      for (int j = 0; j < GP_PJ_CHAINS_CL; j++) {
        const int i = v0 + j * nthr;
        pr[j] = i < own ? vR0[i] : 0u;
      }
#pragma unroll
      for (int j = 0; j < GP_PJ_CHAINS_CL; j++) {
        const int i = v0 + j * nthr;
        px[j] = i < own ? ld_w((int)(pr[j] & 0xFFFFu)) : 0u;
      }
#pragma unroll
      for (int j = 0; j < GP_PJ_CHAINS_CL; j++) {
        const int i = v0 + j * nthr;
        const uint32_t jj = px[j] & 0xFFFFu;
        if (i < own && jj != (pr[j] & 0xFFFFu)) {
          vR0[i] = ((pr[j] & 0xFFFF0000u) + (px[j] & 0xFFFF0000u)) | jj;
          ch = 1;
        }
      }
    }
    ch = __syncthreads_or(ch);
    if (tid == 0) sh.orflag[par] = ch;
    cl.sync();
    const int any = *(volatile int*)&sh.orflag[par] |
                    (int)rld32(SHo + (uint32_t)offsetof(ClShared, orflag) + 4u * par);
    par ^= 1;
    npj++;
    if (!any) break;
  }
  stamp(6);

  // ---------------- outputs ----------------
  float* gtdp = a.ts.tdp + off;
  for (int i = tid; i < own; i += nthr) {
    const int v = b0 + i;
    const uint32_t q = vR0[i] >> 16;
    const uint32_t sz = R1[i];
    const uint32_t dv = gtin[v];  // written by this thread above
    __stcs(&gtdp[q], __uint_as_float(dv));
    __stcs(&gtin[v], q | (sz << 16));
  }
  const int lite = sh.lite;
  stamp(7);
  if (lite) {
    // list mode (the commit loop only tests Euler intervals): tin / tdp / C
    cl.sync();
    if (rank == 0 && tid == 0) {
      a.ts.T[slot] = 0;
      a.ts.C[slot] = sh.pairs + rld32(SHo + (uint32_t)offsetof(ClShared, pairs));
    }
  } else {
    cl.sync();  // every pj read done: R0 becomes the staging of (pixel | size << 16) by position
    for (int i = tid; i < own; i += nthr) {
      const int v = b0 + i;
      const uint32_t x = __ldcg(&gtin[v]);  // this thread's own store above
      st_w((int)(x & 0xFFFFu), (uint32_t)v | (x & 0xFFFF0000u));
    }
    cl.sync();
    uint32_t* gpre = a.ts.pre + off;
    uint16_t* gszp = a.ts.szp + off;
    const MarkLayout ML = a.L;
    for (int i = tid; i < own; i += nthr) {
      const uint32_t e = vR0[i];
      const uint32_t v = e & 0xFFFFu;
      __stcs(&gpre[b0 + i], (mcol(ML, v) << 16) | v);
      __stcs(&gszp[b0 + i], (unsigned short)(e >> 16));
    }
    // partition of the fill work (propagate.cu E7) over the preorder positions
    // of both CTAs: rank 1's positions follow rank 0's
    const int seg = (own + nthr - 1) / nthr;
    const int q0 = min(own, tid * seg), q1 = min(own, q0 + seg);
    unsigned lsum = 0;
    for (int i = q0; i < q1; i++) {
      const int q = b0 + i;
      lsum += q ? ((vR0[i] >> 16) + 31u) >> 5 : 0u;
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
      const unsigned x = lane < nw ? sh.wsum[lane] : 0u;
      unsigned wi = x;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned y = __shfl_up_sync(0xffffffffu, wi, o);
        if (lane >= o) wi += y;
      }
      if (lane < nw) sh.wsum[lane] = wi - x;
      if (lane == 31) sh.chunks = wi;
    }
    cl.sync();
    const unsigned mine = *(volatile unsigned*)&sh.chunks;
    const unsigned theirs = rld32(SHo + (uint32_t)offsetof(ClShared, chunks));
    const unsigned T = mine + theirs;
    const unsigned long long P = (unsigned long long)a.ts.nparts;
    uint32_t* gpart = a.ts.part + (size_t)slot * a.ts.nparts;
    if (rank == 0 && tid == 0) {
      a.ts.T[slot] = T;
      a.ts.C[slot] = sh.pairs + rld32(SHo + (uint32_t)offsetof(ClShared, pairs));
    }
    unsigned run = (rank ? theirs : 0u) + sh.wsum[wid] + incl - lsum;
    auto first_part = [&](unsigned long long x) -> unsigned long long {
      if (!T) return P;
      unsigned long long pp = (unsigned long long)((double)x * (double)P / (double)T);
      while (pp > 0 && (pp - 1) * T >= x * P) pp--;
      while (pp * T < x * P) pp++;
      return pp;
    };
    auto write_part = [&](unsigned long long pp, unsigned q, unsigned runq) {
      const unsigned long long num = pp * T;
      unsigned b = (unsigned)((double)num / (double)P);
      while ((unsigned long long)b * P > num) b--;
      while ((unsigned long long)(b + 1) * P <= num) b++;
      __stcs(&gpart[pp], (uint32_t)q | ((b - runq) << 16));
    };
    uint4* big = reinterpret_cast<uint4*>(R1);  // sizes by pixel are dead (staged in R0)
    const int bigcap = (int)(lay.r1bytes / sizeof(uint4));
    unsigned long long pn = first_part(run);
    for (int i = q0; i < q1; i++) {
      const int q = b0 + i;
      const unsigned nch = q ? ((vR0[i] >> 16) + 31u) >> 5 : 0u;
      if (!nch) continue;
      const unsigned long long end = (unsigned long long)(run + nch) * P;
      if (pn < P && pn * T < end) {
        if ((pn + 4) * T < end) {  // many parts (the trunk near the root): queued for warps
          const unsigned long long phi = min(first_part(run + nch), P);
          const int bi = atomicAdd(&sh.nbig, 1);
          if (bi < bigcap) {
            big[bi] = make_uint4((unsigned)q, run, (unsigned)pn, (unsigned)phi);
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
    __syncthreads();
    const int nbig = min(sh.nbig, bigcap);
    for (int i = wid; i < nbig; i += nthr >> 5) {
      const uint4 e = big[i];
      for (unsigned pp = e.z + lane; pp < e.w; pp += 32) write_part(pp, e.x, e.y);
    }
  }
  if (a.publish) __threadfence();
  cl.sync();  // no CTA leaves while its partner may still read its shared memory
  stamp(8);
  if (dbg) {
    atomicAdd(&dbg[10], (unsigned long long)npass);
    atomicAdd(&dbg[11], (unsigned long long)nadv);
    atomicAdd(&dbg[12], (unsigned long long)npj);
    atomicAdd(&dbg[13], 1ull);
    atomicAdd(&dbg[14], (unsigned long long)lite);
  }
  if (a.publish && rank == 0 && tid == 0) atomicExch(&a.publish[my_src[0]], slot);
}

// ---------------- host side ----------------
static int cl_M(int N) { return (N + 1) / 2; }

size_t prop_cluster_smem(int N) { return cl_layout(cl_M(N)).total; }

// per-tree global scratch: the overflow of both CTAs' two near lists
size_t prop_cluster_scratch(int N) { return cl_align16((size_t)4 * cl_M(N) * 2); }

bool prop_cluster_ok(int N) {
  if (N <= 0 || N > 65536) return false;
  int dev = 0, optin = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  return prop_cluster_smem(N) + sizeof(ClShared) + 1024 <= (size_t)optin;
}

cudaError_t launch_propagate_cluster(const PropArgs& a, int ntrees, cudaStream_t st) {
  if (ntrees <= 0) return cudaSuccess;
  const int M = cl_M(a.g.N);
  const size_t smem = prop_cluster_smem(a.g.N);
  const bool mc = a.g.metric == kSum && a.g.conn == 8;
  const void* k = mc ? (const void*)k_propagate_cl<1> : (const void*)k_propagate_cl<0>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  PropArgs args = a;
  args.scratch_bytes = prop_cluster_scratch(a.g.N);
  int Marg = M;
  void* params[] = {&args, &Marg};
  return cudaLaunchKernel(k, dim3(2 * ntrees), dim3(CL_THR), params, smem, st);
}

}  // namespace gp
