// Host runtime + C ABI (include/geopairs_b200.h).
//
// The runtime owns all device memory of a context (image, tree store, run
// workspace) and of a store (D, mark bitmap, counts).  gp_run drives the
// device commit loop (commit.cu) and the speculative propagation batches
// (propagate.cu); the only host<->device traffic per batch is a 32-byte
// control block.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>
#include <utility>
#include <vector>

#include "../../include/geopairs_b200.h"
#include "gp_common.cuh"
#include "gp_kernels.h"

using namespace gp;

static thread_local std::string g_err;

// Pixel limits: the dense N^2 store, gp_run and the batched K1 pack pixel ids
// in 16 bits; above that a context serves propagations only (whole-GPU K1).
static constexpr int64_t kMaxPixelsPropagate = (int64_t)1 << 26;
static constexpr int kMaxPixelsStore = 65536;

static int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define CUDA_TRY(expr)                                                               \
  do {                                                                               \
    cudaError_t _e = (expr);                                                         \
    if (_e != cudaSuccess)                                                           \
      return fail(GP_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(_e));     \
  } while (0)

struct gp_ctx {
  Grid g;
  int isint;
  float* d_img = nullptr;
  cudaStream_t st = nullptr;
  cudaStream_t st2 = nullptr;  // propagation stream of the host-driven (debug) loop
  cudaStream_t st3 = nullptr;  // device-to-host stream of completed D rows (gp_run_to_host)

  int border_n = -1;           // border source list resident in the workspace (its length)
  int* h_cnt = nullptr;        // pinned copy of the per-pixel counts
  int nsm = 148;
  // tree store (Euler-tour form) + propagation scratch, lazily sized
  TreeStore ts{};
  uint8_t* scratch = nullptr;
  size_t scratch_trees = 0;
  int commit_blocks = 0;
  double mean_w = 1.0;  // mean edge weight (bucket width scale)
  int pos_w = 0;        // every edge weight > 0
  unsigned long long* heap = nullptr;  // exact heap-order K1 scratch (images with zero-weight edges)
  size_t heap_trees = 0;
  unsigned char* big = nullptr;  // scratch of the whole-GPU K1 (contexts above 65 536 pixels)
  unsigned* h_flag = nullptr;    // pinned pass flag of the whole-GPU K1
  uint32_t* list[2] = {nullptr, nullptr};  // unfilled-pair lists (late phase)
  int* h_cnt2 = nullptr;     // pinned: count snapshots of the host-row rounds (rotating)
  int* d_stage_cnt = nullptr;  // device stage of the snapshots (copied out by a second stream)
  Ctl* d_stage_ctl = nullptr;
  cudaStream_t st4 = nullptr;  // snapshot copies
  int* h_done = nullptr;       // mapped pinned: set by the commit kernel when the array is complete
  uint2* h_patch = nullptr;    // pinned: patch log entries after the early send (gp_run_to_host)
  size_t h_patch_cap = 0;
  Ctl* h_ctl2 = nullptr;     // pinned: two control-block snapshots
  void* ws[32] = {};      // run workspace, cached across runs (no cudaMalloc in gp_run)
  size_t ws_bytes[32] = {};
  size_t list_cap = 0;
  GridBarrier* bar = nullptr;
};

struct gp_store {
  int64_t n;
  MarkLayout L;
  size_t mark_words = 0;  // allocated words
  float* D = nullptr;
  uint32_t* mark = nullptr;
  int* cnt = nullptr;
  unsigned long long* out3 = nullptr;
  int64_t filled = 0;
  cudaStream_t st = nullptr;
  unsigned long long* stage = nullptr;  // APGD row-block staging (u64)
  size_t stage_words = 0;
};

extern "C" const char* gp_last_error(void) { return g_err.c_str(); }
extern "C" int gp_version(void) { return 1; }

template <typename T>
static cudaError_t dalloc(T** p, size_t count) {
  return cudaMalloc(reinterpret_cast<void**>(p), count * sizeof(T) + 16);
}

// Scoped device buffer: freed on every return path (early CUDA_TRY returns
// included).
template <typename T>
struct DevBuf {
  T* p = nullptr;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { if (p) cudaFree(p); }
  cudaError_t alloc(size_t count) { return dalloc(&p, count); }
};

// Validate + convert host pixels to fp32 (grid.py:47-60 semantics).
static int convert_pixels(int H, int W, int dtype, const void* pixels, int metric, int conn,
                          std::vector<float>& f, int* isint_out) {
  const int N = H * W;
  f.resize(N);
  int isint = dtype != GP_DTYPE_F32;
  double vmax = 0.0;
  for (int i = 0; i < N; i++) {
    double v;
    if (dtype == GP_DTYPE_I64) v = (double)((const int64_t*)pixels)[i];
    else if (dtype == GP_DTYPE_U8) v = (double)((const uint8_t*)pixels)[i];
    else if (dtype == GP_DTYPE_F32) v = (double)((const float*)pixels)[i];
    else return fail(GP_EINVAL, "unknown dtype");
    if (isint && (v < 1 || v > 255))
      return fail(GP_EINVAL, "grey levels must be in [1, 255]");
    if (!isint && (!std::isfinite(v) || v < 0))
      return fail(GP_EINVAL, "float pixel values must be finite and >= 0");
    f[i] = (float)v;
    vmax = std::max(vmax, v);
  }
  if (isint) {
    // fp32 exactness: every geodesic distance <= wmax * (hops of a straight path)
    double hops = conn == 8 ? std::max(H, W) - 1 : (H - 1) + (W - 1);
    double wmax = metric == GP_METRIC_MEAN ? 2 * vmax : 4 * vmax;
    if (wmax * hops >= 16777216.0) return fail(GP_EINVAL, "integer distances would exceed 2^24");
  }
  *isint_out = isint;
  return GP_OK;
}

// Is every edge weight > 0?  (scaled_weight, grid.py:146-154: SUM/MEAN are
// zero only between two zero pixels, L1 between equal pixels.)  Zero-weight
// edges break the closed-form predecessor rule; the cluster K1 needs it.
static int positive_weights(int H, int W, int conn, int metric, const std::vector<float>& f) {
  for (int r = 0; r < H; r++)
    for (int c = 0; c < W; c++) {
      const float a = f[(size_t)r * W + c];
      const int nb[4][2] = {{0, 1}, {1, -1}, {1, 0}, {1, 1}};
      for (int k = 0; k < 4; k++) {
        if (conn == 4 && (k == 1 || k == 3)) continue;
        const int rr = r + nb[k][0], cc = c + nb[k][1];
        if (rr >= H || cc < 0 || cc >= W) continue;
        const float b = f[(size_t)rr * W + cc];
        const bool zero = metric == GP_METRIC_L1 ? a == b : (a + b) == 0.0f;
        if (zero) return 0;
      }
    }
  return 1;
}

static double mean_weight(const std::vector<float>& f, int metric) {
  double s = 0;
  for (float v : f) s += v;
  double m = f.empty() ? 1.0 : s / f.size();
  double w = metric == GP_METRIC_SUM ? 4 * m : metric == GP_METRIC_MEAN ? 2 * m : m;
  return w > 0 ? w : 1.0;
}

extern "C" int gp_ctx_create(int H, int W, int dtype, const void* pixels, int metric, int conn,
                             gp_ctx** out) {
  if (!out || !pixels) return fail(GP_EINVAL, "null argument");
  if (H < 1 || W < 1 || (int64_t)H * W < 2) return fail(GP_EINVAL, "image must contain at least 2 pixels");
  // above 65 536 pixels a context serves propagations only (the dense N^2
  // store and gp_run need 16-bit pixel ids); the limit here keeps ids in 32 bits
  if ((int64_t)H * W > kMaxPixelsPropagate)
    return fail(GP_EINVAL, "images above 2^26 pixels are not supported");
  if (conn != 4 && conn != 8) return fail(GP_EINVAL, "connectivity must be 4 or 8");
  if (metric < 0 || metric > 2) return fail(GP_EINVAL, "unknown metric");
  const int N = H * W;
  std::vector<float> f;
  int isint = 0;
  int rc = convert_pixels(H, W, dtype, pixels, metric, conn, f, &isint);
  if (rc) return rc;
  gp_ctx* c = new gp_ctx();
  c->g = make_grid(H, W, conn, metric);
  c->isint = isint;
  c->mean_w = mean_weight(f, metric);
  c->pos_w = positive_weights(H, W, conn, metric, f);
  int dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&c->nsm, cudaDevAttrMultiProcessorCount, dev);
  cudaError_t e = cudaStreamCreateWithFlags(&c->st, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = dalloc(&c->d_img, N);
  if (e == cudaSuccess) e = cudaMemcpy(c->d_img, f.data(), N * 4, cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    gp_ctx_destroy(c);
    return fail(GP_ECUDA, std::string("ctx alloc: ") + cudaGetErrorString(e));
  }
  *out = c;
  return GP_OK;
}

extern "C" int gp_ctx_load(gp_ctx* c, int dtype, const void* pixels) {
  if (!c || !pixels) return fail(GP_EINVAL, "null argument");
  std::vector<float> f;
  int isint = 0;
  int rc = convert_pixels(c->g.H, c->g.W, dtype, pixels, c->g.metric, c->g.conn, f, &isint);
  if (rc) return rc;
  c->isint = isint;
  c->mean_w = mean_weight(f, c->g.metric);
  c->pos_w = positive_weights(c->g.H, c->g.W, c->g.conn, c->g.metric, f);
  CUDA_TRY(cudaMemcpyAsync(c->d_img, f.data(), (size_t)c->g.N * 4, cudaMemcpyHostToDevice, c->st));
  CUDA_TRY(cudaStreamSynchronize(c->st));
  return GP_OK;
}

extern "C" void gp_ctx_destroy(gp_ctx* c) {
  if (!c) return;
  cudaFree(c->d_img);
  cudaFree(c->ts.pre);
  cudaFree(c->ts.szp);
  cudaFree(c->ts.tdp);
  cudaFree(c->ts.part);
  cudaFree(c->ts.T);
  cudaFree(c->ts.C);
  cudaFree(c->ts.tin);
  cudaFree(c->list[0]);
  cudaFree(c->list[1]);
  for (void* p : c->ws) cudaFree(p);
  cudaFree(c->bar);
  cudaFree(c->scratch);
  cudaFree(c->heap);
  cudaFree(c->big);
  if (c->h_flag) cudaFreeHost(c->h_flag);
  if (c->st) cudaStreamDestroy(c->st);
  if (c->st2) cudaStreamDestroy(c->st2);
  if (c->st3) cudaStreamDestroy(c->st3);

  if (c->h_cnt) cudaFreeHost(c->h_cnt);
  if (c->h_cnt2) cudaFreeHost(c->h_cnt2);
  cudaFree(c->d_stage_cnt);
  cudaFree(c->d_stage_ctl);
  if (c->st4) cudaStreamDestroy(c->st4);
  if (c->h_done) cudaFreeHost(c->h_done);
  if (c->h_patch) cudaFreeHost(c->h_patch);
  if (c->h_ctl2) cudaFreeHost(c->h_ctl2);
  delete c;
}

extern "C" int gp_ctx_num_pixels(const gp_ctx* c) { return c ? c->g.N : 0; }

enum { WS_SEQ, WS_NEW, WS_SRC, WS_SLOT_OF, WS_RANK, WS_EXT, WS_SELKEY, WS_FLAGS, WS_CTL, WS_DFC,
       WS_FREE, WS_CANDS, WS_SLOTS, WS_BORDER, WS_CEN, WS_FB, WS_TOPK, WS_EXTK, WS_EXTT, WS_CSET,
       WS_VERIFY, WS_CS_SRC, WS_CS_DIST, WS_CS_DIR, WS_CS_PAR, WS_LB, WS_LBHITS, WS_LBTINB, WS_PATCH };

template <typename T>
static cudaError_t ws_get(gp_ctx* c, int id, T** p, size_t count) {
  const size_t bytes = count * sizeof(T) + 16;
  if (c->ws_bytes[id] < bytes) {
    cudaFree(c->ws[id]);
    c->ws[id] = nullptr;
    c->ws_bytes[id] = 0;
    cudaError_t e = cudaMalloc(&c->ws[id], bytes);
    if (e != cudaSuccess) return e;
    c->ws_bytes[id] = bytes;
  }
  *p = reinterpret_cast<T*>(c->ws[id]);
  return cudaSuccess;
}

// Heap scratch of the exact heap-order K1 (zero-weight edges only): at most
// 2 GiB; larger launches are chunked to what it holds.
static int ensure_heap(gp_ctx* c, size_t ntrees) {
  if (c->pos_w) return GP_OK;
  const size_t words = prop_heap_words(c->g.N, c->g.N);
  const size_t cap = std::max<size_t>(1, ((size_t)2 << 30) / (words * 8));
  const size_t want = std::min(ntrees, cap);
  if (want <= c->heap_trees) return GP_OK;
  cudaFree(c->heap);
  c->heap = nullptr;
  c->heap_trees = 0;
  CUDA_TRY(dalloc(&c->heap, words * want));
  c->heap_trees = want;
  return GP_OK;
}

static int ensure_scratch(gp_ctx* c, size_t ntrees) {
  if (int rc = ensure_heap(c, ntrees)) return rc;
  if (ntrees <= c->scratch_trees) return GP_OK;
  // single-CTA global-scratch K1, or the overflow lists of the cluster K1
  const size_t per = prop_fits_smem(c->g.N) ? prop_cluster_scratch(c->g.N)
                                            : std::max(prop_scratch_bytes(c->g.N), prop_cluster_scratch(c->g.N));
  cudaFree(c->scratch);
  c->scratch = nullptr;
  c->scratch_trees = 0;
  CUDA_TRY(dalloc(&c->scratch, per * ntrees));
  c->scratch_trees = ntrees;
  return GP_OK;
}

static PropArgs base_prop(gp_ctx* c) {
  PropArgs a;
  memset(&a, 0, sizeof(a));
  a.g = c->g;
  a.img = c->d_img;
  a.scratch = c->scratch;
  a.delta = INFINITY;
  a.pos_weights = c->pos_w;
  a.exact_heap = c->pos_w ? 0 : 1;
  a.heap = c->heap;
  a.heap_words = prop_heap_words(c->g.N, c->g.N);
  a.heap_trees = (int)c->heap_trees;
  return a;
}

// Bucket width of the propagation (K1): a multiple of the mean edge weight
// (GP_DELTA_FACTOR, default below; <= 0 or "inf" = unbucketed frontier).
static float default_delta(const gp_ctx* c) {
  double factor = 16.0;
  if (const char* e = getenv("GP_DELTA_FACTOR")) factor = atof(e);
  if (!(factor > 0) || std::isinf(factor)) return INFINITY;
  return (float)(factor * c->mean_w);
}

static bool is_big(const gp_ctx* c) { return c->g.N > kMaxPixelsStore; }

// One propagation of a context above 65 536 pixels (propagate_big.cu) into
// device buffers dist (fp32 bits) and code (parent window codes).
static int big_prop(gp_ctx* c, const int* d_src, int ns, uint32_t* d_dist, uint8_t* d_code, cudaStream_t st) {
  const int exact = c->pos_w ? 0 : 1;
  const size_t need = big_scratch_bytes(c->g.N, 1);
  if (!c->big) CUDA_TRY(dalloc(&c->big, need));
  if (!c->h_flag) CUDA_TRY(cudaHostAlloc(&c->h_flag, 4, cudaHostAllocDefault));
  CUDA_TRY(launch_propagate_big(c->g, c->d_img, d_src, ns, exact, d_dist, d_code, c->big, c->h_flag, st));
  return GP_OK;
}

extern "C" int gp_propagate(gp_ctx* c, const int32_t* sources, int nsrc, float* dist_out,
                            int32_t* parent_out) {
  if (!c || !sources || nsrc < 1) return fail(GP_EINVAL, "at least one source pixel is required");
  const int N = c->g.N;
  std::vector<char> seen(N, 0);
  for (int i = 0; i < nsrc; i++) {
    if (sources[i] < 0 || sources[i] >= N) return fail(GP_EINVAL, "source out of range");
    if (seen[sources[i]]++) return fail(GP_EINVAL, "duplicate source pixels");
  }
  DevBuf<int> d_src;
  DevBuf<float> d_dist;
  DevBuf<uint8_t> d_dir;
  CUDA_TRY(d_src.alloc(nsrc));
  CUDA_TRY(d_dist.alloc(N));
  CUDA_TRY(d_dir.alloc(N));
  CUDA_TRY(cudaMemcpyAsync(d_src.p, sources, nsrc * 4, cudaMemcpyHostToDevice, c->st));
  if (is_big(c)) {
    if (int rc = big_prop(c, d_src.p, nsrc, reinterpret_cast<uint32_t*>(d_dist.p), d_dir.p, c->st)) return rc;
  } else {
    int rc = ensure_scratch(c, 1);
    if (rc) return rc;
    PropArgs a = base_prop(c);
    a.src = d_src.p;
    a.ns = nsrc;
    a.out_dist = d_dist.p;
    a.out_dir = d_dir.p;
    a.delta = default_delta(c);
    CUDA_TRY(launch_propagate(a, 1, c->st));
  }
  std::vector<uint8_t> dir(N);
  if (dist_out) CUDA_TRY(cudaMemcpyAsync(dist_out, d_dist.p, N * 4, cudaMemcpyDeviceToHost, c->st));
  CUDA_TRY(cudaMemcpyAsync(dir.data(), d_dir.p, N, cudaMemcpyDeviceToHost, c->st));
  CUDA_TRY(cudaStreamSynchronize(c->st));
  if (parent_out) {
    const int W = c->g.W;
    for (int v = 0; v < N; v++) {
      uint8_t k = dir[v];
      parent_out[v] = k == GP_ROOT ? -1 : v + (k / 3 - 1) * W + (k % 3 - 1);
    }
  }
  return GP_OK;
}

extern "C" int gp_propagate_batch(gp_ctx* c, const int32_t* src_dev, int k, float* tdist_dev,
                                  uint8_t* dir_dev, void* stream) {
  if (!c || !src_dev || k < 0) return fail(GP_EINVAL, "bad arguments");
  if (is_big(c)) {  // one whole-GPU propagation per source
    for (int i = 0; i < k; i++)
      if (int r = big_prop(c, src_dev + i, 1, reinterpret_cast<uint32_t*>(tdist_dev + (size_t)i * c->g.N),
                           dir_dev + (size_t)i * c->g.N, (cudaStream_t)stream))
        return r;
    return GP_OK;
  }
  int rc = ensure_scratch(c, (size_t)k);
  if (rc) return rc;
  PropArgs a = base_prop(c);
  a.src = src_dev;
  a.ns = 1;
  a.out_dist = tdist_dev;
  a.out_dir = dir_dev;
  a.delta = default_delta(c);
  CUDA_TRY(launch_propagate(a, k, (cudaStream_t)stream));
  return GP_OK;
}

static std::vector<int32_t> boundary_pixels(int W, int H) {  // propagation.py:130-143
  std::vector<int32_t> out;
  for (int r = 0; r < H; r++) {
    if (r == 0 || r == H - 1) {
      for (int col = 0; col < W; col++) out.push_back(r * W + col);
    } else {
      out.push_back(r * W);
      if (W > 1) out.push_back(r * W + W - 1);
    }
  }
  return out;
}

// _extrema_context (strategies.py:109-116) on the device; returns the
// centroid, and fills dfc_dev [N] (device) and the host dist_from_c copy.
// the two K1 runs of _extrema_context, asynchronous: centroid in d_cen_out
static int extrema_async(gp_ctx* c, int** d_cen_out, float* dfc_dev) {
  const int N = c->g.N;
  std::vector<int32_t> border = boundary_pixels(c->g.W, c->g.H);
  int* d_src = nullptr;
  int* d_cen = nullptr;
  float* d_fb = nullptr;
  int rc = ensure_scratch(c, 1);
  if (rc) return rc;
  CUDA_TRY(ws_get(c, WS_BORDER, &d_src, border.size() + 1));
  CUDA_TRY(ws_get(c, WS_CEN, &d_cen, 1));
  CUDA_TRY(ws_get(c, WS_FB, &d_fb, N));
  if (c->border_n != (int)border.size()) {  // the border list depends only on the shape
    CUDA_TRY(cudaMemcpyAsync(d_src, border.data(), border.size() * 4, cudaMemcpyHostToDevice, c->st));
    CUDA_TRY(cudaStreamSynchronize(c->st));
    c->border_n = (int)border.size();
  }
  PropArgs a = base_prop(c);
  a.src = d_src;
  a.ns = (int)border.size();
  a.out_dist = d_fb;
  a.delta = default_delta(c);
  CUDA_TRY(launch_propagate(a, 1, c->st));
  CUDA_TRY(launch_argmax_first(d_fb, N, d_cen, c->st));
  PropArgs b = base_prop(c);
  b.src = d_cen;
  b.ns = 1;
  b.out_dist = dfc_dev;
  b.delta = default_delta(c);
  CUDA_TRY(launch_propagate(b, 1, c->st));
  *d_cen_out = d_cen;
  return GP_OK;
}

static int extrema_device(gp_ctx* c, int* centroid, float* dfc_dev, std::vector<float>& dfc_host) {
  const int N = c->g.N;
  std::vector<int32_t> border = boundary_pixels(c->g.W, c->g.H);
  int* d_src = nullptr;
  int* d_cen = nullptr;
  float* d_fb = nullptr;
  CUDA_TRY(ws_get(c, WS_BORDER, &d_src, border.size() + 1));
  CUDA_TRY(ws_get(c, WS_CEN, &d_cen, 1));
  CUDA_TRY(ws_get(c, WS_FB, &d_fb, N));
  CUDA_TRY(cudaMemcpyAsync(d_src, border.data(), border.size() * 4, cudaMemcpyHostToDevice, c->st));
  if (is_big(c)) {  // whole-GPU propagations (contexts above 65 536 pixels)
    uint8_t* d_code = nullptr;
    CUDA_TRY(ws_get(c, WS_CS_DIR, &d_code, N));
    if (int r = big_prop(c, d_src, (int)border.size(), reinterpret_cast<uint32_t*>(d_fb), d_code, c->st)) return r;
    CUDA_TRY(launch_argmax_first(d_fb, N, d_cen, c->st));
    if (int r = big_prop(c, d_cen, 1, reinterpret_cast<uint32_t*>(dfc_dev), d_code, c->st)) return r;
    dfc_host.resize(N);
    CUDA_TRY(cudaMemcpyAsync(centroid, d_cen, 4, cudaMemcpyDeviceToHost, c->st));
    CUDA_TRY(cudaMemcpyAsync(dfc_host.data(), dfc_dev, (size_t)N * 4, cudaMemcpyDeviceToHost, c->st));
    CUDA_TRY(cudaStreamSynchronize(c->st));
    return GP_OK;
  }
  int rc = ensure_scratch(c, 1);
  if (rc) return rc;
  PropArgs a = base_prop(c);
  a.src = d_src;
  a.ns = (int)border.size();
  a.out_dist = d_fb;
  a.delta = default_delta(c);
  CUDA_TRY(launch_propagate(a, 1, c->st));
  CUDA_TRY(launch_argmax_first(d_fb, N, d_cen, c->st));  // first max = smallest id
  PropArgs b = base_prop(c);
  b.src = d_cen;
  b.ns = 1;
  b.out_dist = dfc_dev;
  b.delta = default_delta(c);
  CUDA_TRY(launch_propagate(b, 1, c->st));
  dfc_host.resize(N);
  CUDA_TRY(cudaMemcpyAsync(centroid, d_cen, 4, cudaMemcpyDeviceToHost, c->st));
  CUDA_TRY(cudaMemcpyAsync(dfc_host.data(), dfc_dev, N * 4, cudaMemcpyDeviceToHost, c->st));
  CUDA_TRY(cudaStreamSynchronize(c->st));
  return GP_OK;
}

static void ext_order(const std::vector<float>& dfc, std::vector<int32_t>& ext) {
  // ext = lexsort((id, -dfc)): decreasing distance, ties by increasing id
  const int N = (int)dfc.size();
  ext.resize(N);
  for (int i = 0; i < N; i++) ext[i] = i;
  std::stable_sort(ext.begin(), ext.end(), [&](int32_t x, int32_t y) { return dfc[x] > dfc[y]; });
}

extern "C" int gp_extrema(gp_ctx* c, int32_t* centroid, float* dfc_out, int32_t* ext_out) {
  if (!c) return fail(GP_EINVAL, "null ctx");
  DevBuf<float> d_dfc;
  CUDA_TRY(d_dfc.alloc(c->g.N));
  std::vector<float> dfc;
  int cen = -1;
  int rc = extrema_device(c, &cen, d_dfc.p, dfc);
  if (rc) return rc;
  std::vector<int32_t> ext;
  ext_order(dfc, ext);
  if (centroid) *centroid = cen;
  if (dfc_out) memcpy(dfc_out, dfc.data(), dfc.size() * 4);
  if (ext_out) memcpy(ext_out, ext.data(), ext.size() * 4);
  return GP_OK;
}

// ---------------- store ----------------
extern "C" int gp_store_create(int64_t n, gp_store** out) {
  if (!out) return fail(GP_EINVAL, "null argument");
  if (n < 2) return fail(GP_EINVAL, "need at least 2 pixels");
  if (n > kMaxPixelsStore) return fail(GP_ENOMEM, "stores above 65536 pixels are not supported");
  gp_store* s = new gp_store();
  s->n = n;
  s->L = make_layout((int)n, 1, (int)n);  // no image yet: raster columns
  s->mark_words = (size_t)n * s->L.RW;
  cudaError_t e = cudaStreamCreateWithFlags(&s->st, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = dalloc(&s->D, (size_t)n * n);
  if (e == cudaSuccess) e = dalloc(&s->mark, s->mark_words);
  if (e == cudaSuccess) e = dalloc(&s->cnt, (size_t)n);
  if (e == cudaSuccess) e = dalloc(&s->out3, 3);
  if (e == cudaSuccess) e = cudaMemsetAsync(s->cnt, 0, n * 4, s->st);
  if (e == cudaSuccess) e = launch_store_init(s->L, s->mark, s->D, s->st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s->st);
  if (e != cudaSuccess) {
    gp_store_destroy(s);
    return fail(e == cudaErrorMemoryAllocation ? GP_ENOMEM : GP_ECUDA,
                std::string("store alloc: ") + cudaGetErrorString(e));
  }
  *out = s;
  return GP_OK;
}

extern "C" void gp_store_destroy(gp_store* s) {
  if (!s) return;
  cudaFree(s->D);
  cudaFree(s->mark);
  cudaFree(s->cnt);
  cudaFree(s->out3);
  cudaFree(s->stage);
  if (s->st) cudaStreamDestroy(s->st);
  delete s;
}

// ---------------- APGD (distances.py:149-177) ----------------
// Row blocks of the u64 payload are converted on the device and copied in
// slices of at most 32 MiB, so neither side ever holds an N^2 temporary.
static const size_t kStageWords = (size_t)4 << 20;

static int store_stage(gp_store* s) {
  if (s->stage) return GP_OK;
  CUDA_TRY(dalloc(&s->stage, kStageWords));
  s->stage_words = kStageWords;
  return GP_OK;
}

extern "C" int gp_store_apgd_rows(gp_store* s, int version, int64_t row0, int64_t nrows, uint64_t* out) {
  if (!s || !out) return fail(GP_EINVAL, "null argument");
  if (version != 1 && version != 2) return fail(GP_EINVAL, "unsupported APGD version");
  if (row0 < 0 || nrows < 0 || row0 + nrows > s->n) return fail(GP_EINVAL, "row range out of bounds");
  if (int rc = store_stage(s)) return rc;
  const int64_t n = s->n;
  const int64_t per = std::max<int64_t>(1, (int64_t)(s->stage_words / (size_t)n));
  for (int64_t r = row0; r < row0 + nrows; r += per) {
    const int64_t k = std::min(per, row0 + nrows - r);
    CUDA_TRY(launch_apgd_dump(s->L, s->D, s->mark, r, k, version, s->stage, s->st));
    CUDA_TRY(cudaMemcpyAsync(out + (r - row0) * n, s->stage, (size_t)(k * n) * 8, cudaMemcpyDeviceToHost, s->st));
  }
  CUDA_TRY(cudaStreamSynchronize(s->st));
  return GP_OK;
}

extern "C" int gp_store_load_rows(gp_store* s, int version, int64_t row0, int64_t nrows, const uint64_t* rows) {
  if (!s || !rows) return fail(GP_EINVAL, "null argument");
  if (version != 1 && version != 2) return fail(GP_EINVAL, "unsupported APGD version");
  if (row0 < 0 || nrows < 0 || row0 + nrows > s->n) return fail(GP_EINVAL, "row range out of bounds");
  if (int rc = store_stage(s)) return rc;
  const int64_t n = s->n;
  const int64_t per = std::max<int64_t>(1, (int64_t)(s->stage_words / (size_t)n));
  CUDA_TRY(cudaMemsetAsync(s->out3, 0, 24, s->st));
  for (int64_t r = row0; r < row0 + nrows; r += per) {
    const int64_t k = std::min(per, row0 + nrows - r);
    CUDA_TRY(cudaMemcpyAsync(s->stage, rows + (r - row0) * n, (size_t)(k * n) * 8, cudaMemcpyHostToDevice, s->st));
    CUDA_TRY(launch_apgd_load(s->L, s->D, s->mark, r, k, version, s->stage, s->out3 + 1, s->st));
  }
  unsigned long long bad = 0;
  CUDA_TRY(cudaMemcpyAsync(&bad, s->out3 + 1, 8, cudaMemcpyDeviceToHost, s->st));
  CUDA_TRY(cudaStreamSynchronize(s->st));
  if (bad) return fail(GP_EINVAL, std::to_string(bad) + " APGD values are not representable in the fp32 store");
  return GP_OK;
}

extern "C" int gp_store_recount(gp_store* s, int64_t* filled) {
  if (!s) return fail(GP_EINVAL, "null store");
  CUDA_TRY(cudaMemsetAsync(s->out3, 0, 24, s->st));
  CUDA_TRY(launch_store_recount(s->L, s->mark, s->cnt, s->out3, s->st));
  unsigned long long marks = 0;
  CUDA_TRY(cudaMemcpyAsync(&marks, s->out3, 8, cudaMemcpyDeviceToHost, s->st));
  CUDA_TRY(cudaStreamSynchronize(s->st));
  s->filled = ((int64_t)marks - s->n) / 2;
  if (filled) *filled = s->filled;
  return GP_OK;
}

extern "C" int gp_store_device_ptrs(gp_store* s, float** D, uint32_t** mark, int32_t** counts,
                                    int64_t* words) {
  if (!s) return fail(GP_EINVAL, "null store");
  if (D) *D = s->D;
  if (mark) *mark = s->mark;
  if (counts) *counts = s->cnt;
  if (words) *words = s->L.RW;
  return GP_OK;
}

extern "C" int gp_store_fill_tree(gp_store* s, const int32_t* parent, const float* tdist,
                                  float tol, int64_t* new_pairs) {
  if (!s || !parent || !tdist) return fail(GP_EINVAL, "null argument");
  const int N = (int)s->n;
  DevBuf<int> d_par;
  DevBuf<float> d_td;
  CUDA_TRY(d_par.alloc(N));
  CUDA_TRY(d_td.alloc(N));
  CUDA_TRY(cudaMemcpyAsync(d_par.p, parent, N * 4, cudaMemcpyHostToDevice, s->st));
  CUDA_TRY(cudaMemcpyAsync(d_td.p, tdist, N * 4, cudaMemcpyHostToDevice, s->st));
  // snapshot so that a failed fill leaves the store unchanged is not needed by
  // the reference (fill_tree_pairs mutates before the wrapper raises,
  // _kernels.py:102-111, distances.py:108-116); mirror that behaviour.
  CUDA_TRY(cudaMemsetAsync(s->out3, 0, 24, s->st));
  CUDA_TRY(launch_fill_tree_api(s->L, d_par.p, d_td.p, s->mark, s->cnt, s->D, s->out3, tol, s->st));
  unsigned long long o[3];
  CUDA_TRY(cudaMemcpyAsync(o, s->out3, 24, cudaMemcpyDeviceToHost, s->st));
  CUDA_TRY(cudaStreamSynchronize(s->st));
  if (o[2]) return fail(GP_ECYCLE, "tree parent links contain a cycle");
  if (o[1]) return fail(GP_EDISAGREE, "tree distances disagree with " + std::to_string(o[1]) +
                                          " already-stored entries");
  s->filled += (int64_t)o[0];
  if (new_pairs) *new_pairs = (int64_t)o[0];
  return GP_OK;
}

extern "C" int gp_store_fill_source(gp_store* s, int64_t source, const float* dist, float tol,
                                    int64_t* new_pairs) {
  if (!s || !dist) return fail(GP_EINVAL, "null argument");
  const int N = (int)s->n;
  if (source < 0 || source >= N) return fail(GP_EINVAL, "source out of range");
  if (dist[source] != 0.0f) return fail(GP_EINVAL, "source's distance to itself must be 0");
  DevBuf<float> d_dist;
  CUDA_TRY(d_dist.alloc(N));
  CUDA_TRY(cudaMemcpyAsync(d_dist.p, dist, N * 4, cudaMemcpyHostToDevice, s->st));
  CUDA_TRY(cudaMemsetAsync(s->out3, 0, 24, s->st));
  // the reference checks agreement before writing anything (distances.py:132-136):
  // a read-only check kernel runs first, the write kernel only without disagreements
  CUDA_TRY(launch_fill_source_api(s->L, (int)source, d_dist.p, s->mark, s->cnt, s->D, s->out3,
                                  tol, s->st));
  unsigned long long o[3];
  CUDA_TRY(cudaMemcpyAsync(o, s->out3, 24, cudaMemcpyDeviceToHost, s->st));
  CUDA_TRY(cudaStreamSynchronize(s->st));
  if (o[1]) return fail(GP_EDISAGREE, "distance map disagrees with already-stored entries");
  s->filled += (int64_t)o[0];
  if (new_pairs) *new_pairs = (int64_t)o[0];
  return GP_OK;
}

extern "C" int gp_store_counts(gp_store* s, int32_t* counts_out, int64_t* filled) {
  if (!s) return fail(GP_EINVAL, "null store");
  if (counts_out) {
    CUDA_TRY(cudaMemcpyAsync(counts_out, s->cnt, s->n * 4, cudaMemcpyDeviceToHost, s->st));
    CUDA_TRY(cudaStreamSynchronize(s->st));
  }
  if (filled) *filled = s->filled;
  return GP_OK;
}

extern "C" int gp_store_read(gp_store* s, float* D_out, uint8_t* mark_out) {
  if (!s) return fail(GP_EINVAL, "null store");
  const size_t nn = (size_t)s->n * s->n;
  if (D_out) CUDA_TRY(cudaMemcpyAsync(D_out, s->D, nn * 4, cudaMemcpyDeviceToHost, s->st));
  if (mark_out) {
    DevBuf<uint8_t> d_m;
    CUDA_TRY(d_m.alloc(nn));
    CUDA_TRY(launch_mark_unpack(s->L, s->mark, d_m.p, s->st));
    CUDA_TRY(cudaMemcpyAsync(mark_out, d_m.p, nn, cudaMemcpyDeviceToHost, s->st));
    CUDA_TRY(cudaStreamSynchronize(s->st));
  }
  CUDA_TRY(cudaStreamSynchronize(s->st));
  return GP_OK;
}

// ---------------- host-selected strategies: one commit per call ----------------
extern "C" int gp_commit_source(gp_ctx* c, gp_store* s, int32_t source, float tol, int64_t* new_pairs,
                                int32_t* counts_out) {
  if (!c || !s) return fail(GP_EINVAL, "null argument");
  const int N = c->g.N;
  if (s->n != N) return fail(GP_EINVAL, "store size does not match the image");
  if (source < 0 || source >= N) return fail(GP_EINVAL, "source out of range");
  if (int rc = ensure_scratch(c, 1)) return rc;
  int *d_src = nullptr, *d_par = nullptr;
  float* d_dist = nullptr;
  uint8_t* d_dir = nullptr;
  CUDA_TRY(ws_get(c, WS_CS_SRC, &d_src, 1));
  CUDA_TRY(ws_get(c, WS_CS_DIST, &d_dist, N));
  CUDA_TRY(ws_get(c, WS_CS_DIR, &d_dir, N));
  CUDA_TRY(ws_get(c, WS_CS_PAR, &d_par, N));
  CUDA_TRY(cudaStreamSynchronize(s->st));  // earlier store calls complete
  cudaStream_t st = c->st;
  CUDA_TRY(cudaMemcpyAsync(d_src, &source, 4, cudaMemcpyHostToDevice, st));
  PropArgs a = base_prop(c);
  a.src = d_src;
  a.ns = 1;
  a.out_dist = d_dist;
  a.out_dir = d_dir;
  a.delta = default_delta(c);
  CUDA_TRY(launch_propagate(a, 1, st));
  CUDA_TRY(launch_dir_to_parent(d_dir, N, c->g.W, d_par, st));
  CUDA_TRY(cudaMemsetAsync(s->out3, 0, 24, st));
  CUDA_TRY(launch_fill_tree_api(s->L, d_par, d_dist, s->mark, s->cnt, s->D, s->out3, tol, st));
  unsigned long long o[3];
  CUDA_TRY(cudaMemcpyAsync(o, s->out3, 24, cudaMemcpyDeviceToHost, st));
  if (counts_out) CUDA_TRY(cudaMemcpyAsync(counts_out, s->cnt, (size_t)N * 4, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  if (o[2]) return fail(GP_ECYCLE, "tree parent links contain a cycle");
  if (o[1]) return fail(GP_EDISAGREE, "tree distances disagree with " + std::to_string(o[1]) +
                                          " already-stored entries");
  s->filled += (int64_t)o[0];
  if (new_pairs) *new_pairs = (int64_t)o[0];
  return GP_OK;
}

// ---------------- run_strategy ----------------
struct EvPair {
  cudaEvent_t a, b;
};

// Events of one run: created checked, destroyed together when the run returns.
struct EventPool {
  std::vector<cudaEvent_t> ev;
  EventPool() = default;
  EventPool(const EventPool&) = delete;
  EventPool& operator=(const EventPool&) = delete;
  ~EventPool() { for (cudaEvent_t e : ev) cudaEventDestroy(e); }
  cudaError_t make(cudaEvent_t* e, unsigned flags = cudaEventDefault) {
    cudaError_t r = cudaEventCreateWithFlags(e, flags);
    if (r == cudaSuccess) ev.push_back(*e);
    return r;
  }
  cudaError_t pair(EvPair& p) {
    cudaError_t r = make(&p.a);
    return r == cudaSuccess ? make(&p.b) : r;
  }
};

static float ev_ms(const EvPair& p) {
  float ms = 0.f;
  cudaEventElapsedTime(&ms, p.a, p.b);
  return ms;
}

static int ensure_tree_store(gp_ctx* c, int nparts) {
  const int N = c->g.N;
  if (c->ts.pre && c->ts.cap >= N && c->ts.nparts == nparts) return GP_OK;
  cudaFree(c->ts.pre); cudaFree(c->ts.szp); cudaFree(c->ts.tdp); cudaFree(c->ts.part); cudaFree(c->ts.T);
  cudaFree(c->ts.C); cudaFree(c->ts.tin);
  c->ts = TreeStore{};
  const size_t cap = (size_t)N;  // a pixel is propagated at most once: N slots always suffice
  CUDA_TRY(dalloc(&c->ts.pre, cap * N));
  CUDA_TRY(dalloc(&c->ts.szp, cap * N));
  CUDA_TRY(dalloc(&c->ts.tdp, cap * N));
  CUDA_TRY(dalloc(&c->ts.part, cap * nparts));
  CUDA_TRY(dalloc(&c->ts.T, cap));
  CUDA_TRY(dalloc(&c->ts.C, cap));
  CUDA_TRY(dalloc(&c->ts.tin, cap * N));
  c->ts.cap = (int)cap;
  c->ts.nparts = nparts;
  // (the constant fits 32 bits above 1024 partitions)
  c->ts.pmagic = (nparts > 1024 && nparts < (1 << 14)) ? (unsigned)(((1ull << 42) + (unsigned long long)nparts - 1) / (unsigned long long)nparts) : 0u;
  return GP_OK;
}

static int store_relayout(gp_store* s, const MarkLayout& L) {
  const size_t words = (size_t)s->n * L.RW;
  if (words > s->mark_words) {
    cudaFree(s->mark);
    s->mark = nullptr;
    s->mark_words = 0;
    CUDA_TRY(dalloc(&s->mark, words));
    s->mark_words = words;
  }
  s->L = L;
  return GP_OK;
}

// Commit CTAs: two per SM when the loop has the GPU alone; one per SM when
// propagation batches run concurrently on the other half of each SM.
static int commit_blocks(gp_ctx* c) {
  const int maxb = commit_max_blocks();
  int bps = 2048 / commit_threads();
  if (c->g.N < 16384) bps = 1;  // tiny fills: the barrier over fewer CTAs wins (64^2: 26.9 -> 25.0 ms)
  if (const char* e = getenv("GP_COMMIT_BLOCKS_PER_SM")) bps = atoi(e);
  return std::max(1, std::min(maxb, bps * c->nsm));
}

// Streamed result rows (gp_run_to_host): a row u of D is final once its count
// reaches N-1 (every pair (u, *) is filled; the diagonal is set at reset).
// Between commit launches the host reads the counts and queues the newly
// complete rows (merged into contiguous runs) on a copy stream, so the D2H
// transfer overlaps the rest of the run; the remaining rows follow at the end.
struct RowStreamer {
  gp_ctx* c;
  gp_store* s;
  float* host;
  std::vector<uint8_t> sent;
  int64_t rows_sent = 0;
  int open_rows = -1;  // rows not complete at the last snapshot
  cudaEvent_t snap_ev = nullptr;
  bool snap_pending = false;
  // counts snapshot in stream order (the caller enqueues it at a quiescent
  // point, then more work); flush() waits for the snapshot only
  int snapshot() {
    if (!host) return GP_OK;
    if (!snap_ev) CUDA_TRY(cudaEventCreateWithFlags(&snap_ev, cudaEventDisableTiming));
    CUDA_TRY(cudaMemcpyAsync(c->h_cnt, s->cnt, (size_t)c->g.N * 4, cudaMemcpyDeviceToHost, c->st));
    CUDA_TRY(cudaEventRecord(snap_ev, c->st));
    snap_pending = true;
    return GP_OK;
  }
  int flush() {
    if (!host || !snap_pending) return GP_OK;
    CUDA_TRY(cudaEventSynchronize(snap_ev));
    snap_pending = false;
    return enqueue(false, false);
  }
  ~RowStreamer() {
    if (snap_ev) cudaEventDestroy(snap_ev);
    for (cudaEvent_t e : fence) if (e) cudaEventDestroy(e);
  }
  int enqueue(bool all, bool read = true, const int* cnt = nullptr) {
    const int N = c->g.N;
    if (!host) return GP_OK;
    if (!all && read) {
      CUDA_TRY(cudaMemcpyAsync(c->h_cnt, s->cnt, (size_t)N * 4, cudaMemcpyDeviceToHost, c->st));
      CUDA_TRY(cudaStreamSynchronize(c->st));
    }
    const int* hc = cnt ? cnt : c->h_cnt;
    if (!all) {
      int open = 0;
      for (int v = 0; v < N; v++) open += hc[v] != N - 1;
      open_rows = open;
    }
    // (one cudaMemcpyAsync per run of newly complete rows; the runtime's
    // batched-copy entry point is closed on the target pool)
    bdst.clear();
    bsrc.clear();
    bsz.clear();
    int u = 0;
    while (u < N) {
      if (sent[u] || (!all && hc[u] != N - 1)) { u++; continue; }
      int e = u;
      while (e < N && !sent[e] && (all || hc[e] == N - 1)) sent[e++] = 1;
      bdst.push_back(host + (size_t)u * N);
      bsrc.push_back(s->D + (size_t)u * N);
      bsz.push_back((size_t)(e - u) * N * 4);
      rows_sent += e - u;
      u = e;
    }
    if (bdst.empty() || getenv("GP_E2E_NOCOPY")) return GP_OK;  // (timing probe: no row copies, results not delivered)
    const auto t0 = std::chrono::steady_clock::now();
    for (size_t i = 0; i < bdst.size(); i++) {
      // Shallow copy queue: a fence event every FENCE copies, at most NFENCE
      // fences outstanding.  (cudaMemcpyAsync into a full queue blocks inside
      // the runtime, and with it the launches of the thread that drives the run.)
      if (nfence_copies == FENCE) {
        nfence_copies = 0;
        cudaEvent_t& ev = fence[fence_head % NFENCE];
        if (fence_head >= NFENCE) CUDA_TRY(cudaEventSynchronize(ev));
        if (!ev) CUDA_TRY(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        CUDA_TRY(cudaEventRecord(ev, c->st3));
        fence_head++;
      }
      nfence_copies++;
      CUDA_TRY(cudaMemcpyAsync(bdst[i], bsrc[i], bsz[i], cudaMemcpyDeviceToHost, c->st3));
    }
    issue_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    issue_calls += (long long)bdst.size();
    return GP_OK;
  }
  std::vector<void*> bdst, bsrc;
  std::vector<size_t> bsz;
  static constexpr int FENCE = 64, NFENCE = 4;
  cudaEvent_t fence[NFENCE] = {nullptr, nullptr, nullptr, nullptr};
  int nfence_copies = 0;
  unsigned fence_head = 0;
  double issue_ms = 0;       // host time spent issuing row copies
  long long issue_calls = 0;
};

static int run_impl(gp_ctx* c, gp_store* s, int strategy, int naive_with_tree, int spec_k,
                    int32_t* seq_out, int64_t* new_out, gp_run_stats* stats, float* D_host);

extern "C" int gp_run(gp_ctx* c, gp_store* s, int strategy, int naive_with_tree, int spec_k,
                      int32_t* seq_out, int64_t* new_out, gp_run_stats* stats) {
  return run_impl(c, s, strategy, naive_with_tree, spec_k, seq_out, new_out, stats, nullptr);
}

extern "C" int gp_run_to_host(gp_ctx* c, gp_store* s, int strategy, int naive_with_tree, int spec_k,
                              int32_t* seq_out, int64_t* new_out, gp_run_stats* stats, float* D_out) {
  if (!D_out) return fail(GP_EINVAL, "null D_out");
  return run_impl(c, s, strategy, naive_with_tree, spec_k, seq_out, new_out, stats, D_out);
}

static int run_impl(gp_ctx* c, gp_store* s, int strategy, int naive_with_tree, int spec_k,
                    int32_t* seq_out, int64_t* new_out, gp_run_stats* stats, float* D_host) {
  if (!c || !s) return fail(GP_EINVAL, "null argument");
  const int N = c->g.N;
  EventPool evp;  // every event of the run, destroyed on all return paths
  unsigned long long* d_verify = nullptr;  // GP_VERIFY disagreement counter
  RowStreamer rs{c, s, D_host, {}, 0};
  std::pair<uint2*, unsigned> patch_after_cut{nullptr, 0u};  // patch log and its position at the early send
  unsigned h_ctl_final_patch_n = 0;
  std::vector<int>* g_waste_batch = nullptr;  // GP_DEBUG_WASTE
  struct PatchChunk { unsigned b, e; cudaEvent_t ev; };
  std::vector<PatchChunk> pchunks;  // log ranges copied to c->h_patch, not applied yet
  unsigned patch_fetched = 0;       // log position up to which the copy to the host is queued
  // patches [b, e) of the log (host copy at c->h_patch, offset by the early send's position) into D_host
  auto apply_patches = [&](unsigned b, unsigned e, unsigned base, int nt) {
    if (e <= b) return;
    const uint2* pl = c->h_patch + (b - base);
    const size_t n = e - b;
    auto work = [=](int t) {
      for (size_t i = (size_t)t; i < n; i += (size_t)nt) {
        const unsigned u = pl[i].x >> 16, w = pl[i].x & 0xFFFFu;
        float v;
        memcpy(&v, &pl[i].y, 4);
        D_host[(size_t)u * N + w] = v;
        D_host[(size_t)w * N + u] = v;
      }
    };
    if (nt <= 1 || n < 4096) { for (int t = 0; t < nt; t++) work(t); return; }
    std::vector<std::thread> th;
    int started = 0;
    try {
      for (; started < nt; started++) th.emplace_back(work, started);
    } catch (...) {  // no more threads: the rest on this one
    }
    for (int t = started; t < nt; t++) work(t);
    for (auto& x : th) x.join();
  };
  if (D_host) {
    rs.sent.assign(N, 0);
    if (!c->st3) CUDA_TRY(cudaStreamCreateWithFlags(&c->st3, cudaStreamNonBlocking));

    if (!c->h_cnt) CUDA_TRY(cudaHostAlloc(&c->h_cnt, (size_t)N * 4, cudaHostAllocDefault));
  }
  if (s->n != N) return fail(GP_EINVAL, "store size does not match the image");
  if (strategy != GP_STRATEGY_NAIVE && strategy != GP_STRATEGY_FILLING_RATE && strategy != GP_STRATEGY_EXTREMA)
    return fail(GP_EINVAL, "strategy not supported on the device path");
  cudaStream_t st = c->st;
  gp_run_stats S;
  memset(&S, 0, sizeof(S));
  S.centroid = -1;
  // the store becomes a fresh DistanceArray laid out for this image
  CUDA_TRY(cudaStreamSynchronize(s->st));
  int rl = store_relayout(s, make_layout(N, c->g.H, c->g.W));
  if (rl) return rl;
  const MarkLayout L = s->L;
  EvPair tot, setup;
  CUDA_TRY(evp.pair(tot));
  CUDA_TRY(evp.pair(setup));
  const bool htime = getenv("GP_DEBUG_HOST") != nullptr;
  auto hnow = [] { return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count(); };
  double h0 = hnow();
  std::vector<std::pair<const char*, double>> hmarks;
  auto hmark = [&](const char* what) {
    if (!htime) return;
    const double t = hnow();
    hmarks.emplace_back(what, t - h0);
    h0 = t;
  };
  CUDA_TRY(cudaEventRecord(tot.a, st));
  CUDA_TRY(cudaEventRecord(setup.a, st));
  CUDA_TRY(cudaMemsetAsync(s->cnt, 0, (size_t)N * 4, st));
  // One-sided tree fills (device-resident result): D starts as the NaN
  // sentinel, tree-mode fills store the ancestor's row only, and one
  // transpose-merge pass after the run completes the symmetric array (saves
  // the scattered mirrored store of every new pair; GP_ONE_SIDED=0 off).
  // (completing single rows from their mirrored elements just before each
  // copy was measured slower: e2e 1.575 vs 1.496 s per 256^2 image)
  // gp_run_to_host: the pass runs at the list switch, and rows are streamed
  // from there on (list-mode fills write both elements); runs that never
  // switch (no list phase) keep two-sided fills.
  const bool will_switch = getenv("GP_LIST_ALPHA") ? atof(getenv("GP_LIST_ALPHA")) > 0 : strategy != GP_STRATEGY_NAIVE;
  const bool host_loop = (getenv("GP_DEBUG") && atoi(getenv("GP_DEBUG"))) || (getenv("GP_PIPELINE") && !atoi(getenv("GP_PIPELINE")));
  const bool one_sided = !(strategy == GP_STRATEGY_NAIVE && !naive_with_tree) &&
                         !(getenv("GP_VERIFY") && atoi(getenv("GP_VERIFY"))) &&
                         !(getenv("GP_ONE_SIDED") && !atoi(getenv("GP_ONE_SIDED"))) &&
                         (!D_host || (will_switch && !host_loop));
  if (one_sided) CUDA_TRY(cudaMemsetAsync(s->D, 0xFF, (size_t)N * N * 4, st));
  CUDA_TRY(launch_store_init(L, s->mark, s->D, st));
  S.kernels += 1;

  int* d_seq = nullptr;
  unsigned long long* d_new = nullptr;
  CUDA_TRY(ws_get(c, WS_SEQ, &d_seq, N));
  CUDA_TRY(ws_get(c, WS_NEW, &d_new, N));
  CUDA_TRY(cudaMemsetAsync(d_new, 0, (size_t)N * 8, st));
  int P = 0;
  int rc = GP_OK;

  if (strategy == GP_STRATEGY_NAIVE && !naive_with_tree) {
    // naive: the N-1 raster-order sources are independent -> one batch
    CUDA_TRY(cudaEventRecord(setup.b, st));
    int rcs = ensure_scratch(c, (size_t)(N - 1));
    if (rcs) return rcs;
    std::vector<int32_t> srcs(N - 1);
    for (int i = 0; i < N - 1; i++) srcs[i] = i;
    int* d_src = nullptr;
    CUDA_TRY(ws_get(c, WS_SRC, &d_src, N));
    CUDA_TRY(cudaMemcpyAsync(d_src, srcs.data(), (N - 1) * 4, cudaMemcpyHostToDevice, st));
    EvPair pp;
    CUDA_TRY(evp.pair(pp));
    CUDA_TRY(cudaEventRecord(pp.a, st));
    PropArgs a = base_prop(c);
    a.src = d_src;
    a.ns = 1;
    a.D = s->D;
    a.delta = default_delta(c);
    CUDA_TRY(launch_propagate(a, N - 1, st));
    CUDA_TRY(launch_naive_trace(L, s->mark, s->cnt, d_seq, d_new, st));
    CUDA_TRY(cudaEventRecord(pp.b, st));
    CUDA_TRY(cudaEventRecord(tot.b, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    S.ms_propagate = ev_ms(pp);
    S.propagations = N - 1;
    S.batches = 1;
    S.kernels += 2;
    P = N - 1;
  } else {
    // ---- device commit loop with speculative propagation batches ----
    // Commit launches and propagation batches alternate, each with the whole
    // GPU.  (A concurrent propagation stream beside a one-CTA-per-SM commit
    // kernel was measured slower in round 1 -- both roles are latency-bound
    // and contend -- and removed: DESIGN.md section 5.)
    hmark("store reset");
    // GP_VERIFY=1: opt-in agreement check of every already-marked pair the
    // committed trees revisit (reference _kernels.py:110-111): generic commit
    // kernel, per-warp unit fill, no list mode, full rows not skipped
    const bool verify = getenv("GP_VERIFY") && atoi(getenv("GP_VERIFY"));
    commit_configure(N);
    const int nblocks = commit_blocks(c);
    hmark("commit_blocks");
    int uf = N >= 32768 ? 3 : 1;  // work units per commit warp (measured at 256^2: 2 933, 3 915, 4 917, 8 1011 ms)
    if (const char* e = getenv("GP_UNITS_PER_WARP")) uf = std::max(1, atoi(e));
    const int nparts = nblocks * (commit_threads() / 32) * uf;
    int rts = ensure_tree_store(c, nparts);
    if (rts) return rts;
    hmark("tree store");
    if (!c->st2) CUDA_TRY(cudaStreamCreateWithFlags(&c->st2, cudaStreamNonBlocking));
    cudaStream_t ps = c->st2;
    int *d_slot_of = nullptr, *d_rank = nullptr, *d_ext = nullptr, *d_cands = nullptr;
    int* d_slots = nullptr;
    uint8_t* d_claimed = nullptr;
    unsigned long long* d_selkey = nullptr;
    Ctl* d_ctl = nullptr;
    float* d_dfc = nullptr;
    CUDA_TRY(ws_get(c, WS_SLOT_OF, &d_slot_of, N));
    CUDA_TRY(ws_get(c, WS_RANK, &d_rank, N));
    CUDA_TRY(ws_get(c, WS_EXT, &d_ext, N));
    CUDA_TRY(ws_get(c, WS_SELKEY, &d_selkey, N + 2));
    unsigned* d_flags = nullptr;
    CUDA_TRY(ws_get(c, WS_FLAGS, &d_flags, N + 2));
    CUDA_TRY(cudaMemsetAsync(d_flags, 0, (size_t)(N + 2) * 4, st));
    CUDA_TRY(ws_get(c, WS_CTL, &d_ctl, 1));
    CUDA_TRY(ws_get(c, WS_DFC, &d_dfc, N));
    CUDA_TRY(ws_get(c, WS_FREE, &d_claimed, N));
    if (!c->bar) CUDA_TRY(dalloc(&c->bar, 1));
    CUDA_TRY(cudaMemsetAsync(c->bar, 0, sizeof(GridBarrier), st));
    {
      const char* e = getenv("GP_BARRIER");
      const unsigned use_cg = (e && !strcmp(e, "sw")) ? 0u : 1u;  // default: cooperative groups
      CUDA_TRY(cudaMemcpyAsync(&c->bar->pad0[0], &use_cg, 4, cudaMemcpyHostToDevice, st));
    }
    CUDA_TRY(cudaMemsetAsync(d_slot_of, 0xFF, (size_t)N * 4, st));
    CUDA_TRY(cudaMemsetAsync(d_claimed, 0, (size_t)N, st));
    CUDA_TRY(cudaMemsetAsync(d_selkey, 0xFF, (size_t)(N + 2) * 8, st));
    Ctl h_ctl;
    memset(&h_ctl, 0, sizeof(h_ctl));
    h_ctl.cur_src = -1;
    // late phase: switch to the unfilled-pair list when the unfilled pairs drop
    // below alpha x the pairs of one tree (~N * mean depth); GP_LIST_ALPHA=0 off
    {
      // measured: 256^2 flat in [1, 1.5]; 128^2 best at 3-5; 64^2 at 10
      // (1 for tiny test images, which then exercise the tree fill too)
      double alpha = N >= 32768 ? 1.5 : N > 8192 ? 3.0 : N > 1024 ? 10.0 : 1.0;
      if (const char* e = getenv("GP_LIST_ALPHA")) alpha = atof(e);
      const double est_tree = (double)N * std::sqrt((double)N) * 0.5;
      double sw = alpha * est_tree;
      const double capd = 64.0 * 1024 * 1024;  // list entries (256 MiB per buffer)
      h_ctl.list_switch = (unsigned long long)std::min(sw, capd);
      if (strategy == GP_STRATEGY_NAIVE && !getenv("GP_LIST_ALPHA")) h_ctl.list_switch = 0;
      if (verify) h_ctl.list_switch = 0;  // the list fill never revisits marked pairs
    }
    CUDA_TRY(cudaMemcpyAsync(d_ctl, &h_ctl, sizeof(Ctl), cudaMemcpyHostToDevice, st));
    hmark("workspace");
    int* d_cen = nullptr;
    if (strategy != GP_STRATEGY_NAIVE) {  // _extrema_context (strategies.py:109-116)
      int r = extrema_async(c, &d_cen, d_dfc);
      if (r) return r;
      unsigned long long* d_ek = nullptr;
      unsigned char* d_et = nullptr;
      const size_t tb = ext_rank_temp_bytes(N);
      CUDA_TRY(ws_get(c, WS_EXTK, &d_ek, (size_t)2 * N));
      CUDA_TRY(ws_get(c, WS_EXTT, &d_et, tb));
      CUDA_TRY(launch_ext_rank(d_dfc, N, d_ek, d_et, tb, d_ext, d_rank, st));
      S.propagations += 2;
      S.kernels += 6;
      if (strategy == GP_STRATEGY_EXTREMA) {  // key part: first position of the distance class
        CUDA_TRY(launch_group_start(d_dfc, d_ext, N, d_rank, st));
        S.kernels += 1;
      }
    }
    hmark("extrema+rank enqueued");
    CUDA_TRY(cudaEventRecord(setup.b, st));
    int K = spec_k > 0 ? spec_k : prop_trees_per_sm(N) * c->nsm;
    if (spec_k <= 0)
      if (const char* e = getenv("GP_SPEC_K")) K = atoi(e);
    // k_topk orders a batch's candidates (longest trees first) in a
    // 1024-entry shared array: a batch holds at most 1024 trees
    K = std::max(1, std::min({K, N, 1024}));
    CUDA_TRY(ws_get(c, WS_CANDS, &d_cands, K));
    CUDA_TRY(ws_get(c, WS_SLOTS, &d_slots, K));
    unsigned* d_tkeys = nullptr;
    CUDA_TRY(ws_get(c, WS_TOPK, &d_tkeys, (size_t)2 * N));
    int rcs = ensure_scratch(c, (size_t)K);
    if (rcs) return rcs;
    CommitArgs ca;
    memset(&ca, 0, sizeof(ca));
    ca.fillq = getenv("GP_FILL_QUEUE") ? atoi(getenv("GP_FILL_QUEUE")) != 0 : 1;
    ca.verify_corrupt = -1;
    if (verify) {
      ca.fillq = 0;
      CUDA_TRY(ws_get(c, WS_VERIFY, &d_verify, 1));
      CUDA_TRY(cudaMemsetAsync(d_verify, 0, 8, st));
      ca.verify = d_verify;
      ca.vtol = c->isint ? 0.0f : 1e-4f;
      if (const char* e = getenv("GP_VERIFY_CORRUPT")) ca.verify_corrupt = atoi(e);
    }
    ca.compact_div = 4;
    ca.lpt = getenv("GP_LPT") ? atoi(getenv("GP_LPT")) != 0 : 1;  // 256^2: 597 -> 587 ms, 128^2: 53.4 -> 51.9 ms
    if (const char* e = getenv("GP_COMPACT_DIV")) ca.compact_div = (unsigned)std::max(1, atoi(e));
    // candidate-set selection (k_commit fast path); GP_CAND=0 off
    if (!getenv("GP_CAND") || atoi(getenv("GP_CAND")) != 0) {
      uint32_t* d_cset = nullptr;
      CUDA_TRY(ws_get(c, WS_CSET, &d_cset, 1024));
      ca.cand = d_cset;
    }
    ca.g = c->g;
    ca.L = L;
    ca.strategy = strategy == GP_STRATEGY_FILLING_RATE ? kFillingRate
                : strategy == GP_STRATEGY_EXTREMA ? kExtrema : kNaive;
    ca.ts = c->ts;
    ca.slot_of = d_slot_of;
    ca.claimed = d_claimed;
    ca.mark = s->mark;
    ca.cnt = s->cnt;
    ca.D = s->D;
    ca.rank = d_rank;
    ca.ext = d_ext;
    ca.selkey = d_selkey;
    ca.stepflags = d_flags;
    ca.one_sided = one_sided ? 1 : 0;
    ca.merge_at_switch = (one_sided && D_host) ? 1 : 0;
    ca.seq = d_seq;
    ca.newp = d_new;
    ca.ctl = d_ctl;
    ca.max_steps = N + 1;
    ca.bar = c->bar;
    ca.total_pairs = ((unsigned long long)N * N - N) / 2;
    PropArgs pa = base_prop(c);
    pa.src = d_cands;
    pa.ns = 1;
    pa.ntrees_dev = &d_ctl->ncand;
    pa.slot = d_slots;
    pa.ts = c->ts;
    pa.L = L;
    pa.publish = d_slot_of;
    pa.list_mode = &d_ctl->mode;  // trees made after the list switch skip pre/szp/partition
    pa.delta = default_delta(c);
    DevBuf<unsigned long long> cl_dbg;  // GP_CL_DEBUG: cluster-K1 phase sums
    if (getenv("GP_CL_DEBUG") && atoi(getenv("GP_CL_DEBUG"))) {
      CUDA_TRY(cl_dbg.alloc(16));
      CUDA_TRY(cudaMemsetAsync(cl_dbg.p, 0, 16 * 8, st));
      pa.cl_dbg = cl_dbg.p;
    }
    const bool debug = getenv("GP_DEBUG") && atoi(getenv("GP_DEBUG"));
    unsigned long long* d_cdbg = nullptr;
    unsigned long long* d_pdbg = nullptr;
    std::vector<double> pacc(16, 0.0);
    double e6acc = 0.0;
    long long pn = 0;
    auto fold_pdbg = [&]() {  // per-tree phase stamps of the last (completed) batch
      if (!d_pdbg) return;
      int nc = 0;
      cudaMemcpy(&nc, &d_ctl->ncand, 4, cudaMemcpyDeviceToHost);
      std::vector<unsigned long long> h((size_t)K * 16);
      cudaMemcpy(h.data(), d_pdbg, h.size() * 8, cudaMemcpyDeviceToHost);
      for (int t = 0; t < std::min(nc, K); t++) {
        const unsigned long long* r = &h[(size_t)t * 16];
        for (int j = 1; j <= 5; j++) pacc[j] += (double)(r[j] - r[j - 1]);
        pacc[6] += (double)r[6];
        pacc[7] += (double)r[7];
        pacc[8] += (double)(r[8] - r[3]);
        pacc[9] += (double)(r[9] - r[8]);
        pacc[10] += (double)(r[10] - r[9]);
        pacc[11] += (double)(r[4] - r[10]);
        pacc[12] += (double)r[11];
        pacc[13] += (double)r[12];
        pacc[14] += (double)r[13];
        pacc[15] += (double)(r[14] - r[10]);
        e6acc += (double)(r[15] - r[4]);
        pn++;
      }
    };
    if (debug) {
      CUDA_TRY(dalloc(&d_pdbg, (size_t)K * 16));
      pa.dbg = d_pdbg;
      CUDA_TRY(dalloc(&d_cdbg, (size_t)(N + 2) * 17));
      CUDA_TRY(cudaMemsetAsync(d_cdbg, 0, (size_t)(N + 2) * 136, st));
      ca.dbg = d_cdbg;
      ca.dbgw = d_cdbg + (size_t)(N + 2) * 4;
      ca.dbgo = d_cdbg + (size_t)(N + 2) * 16;
      if (getenv("GP_DEBUG_SIM")) ca.dbgs = d_cdbg + (size_t)(N + 2) * 8;
      if (const char* e = getenv("GP_DEBUG_UNITS")) {
        ca.dbgu_step = atoi(e);
        CUDA_TRY(dalloc(&ca.dbgu, (size_t)nparts * 8));
        CUDA_TRY(cudaMemsetAsync(ca.dbgu, 0, (size_t)nparts * 32, st));
      }
    }
    std::vector<EvPair> pev, cev;
    // one propagation batch on the propagation stream (host-driven loop)
    const bool waste_dbg = getenv("GP_DEBUG_WASTE") != nullptr;
    static thread_local std::vector<int> waste_batch;
    waste_batch.assign(waste_dbg ? N : 0, -1);
    if (waste_dbg) g_waste_batch = &waste_batch;
    auto batch = [&](int q) -> int {
      EvPair f;
      CUDA_TRY(evp.pair(f));
      CUDA_TRY(cudaEventRecord(f.a, ps));
      CUDA_TRY(launch_topk(ca, K, q, d_cands, d_slots, d_tkeys, 0, ps));
      CUDA_TRY(launch_propagate(pa, K, ps));
      CUDA_TRY(cudaEventRecord(f.b, ps));
      pev.push_back(f);
      S.batches++;
      S.kernels += 2;
      if (waste_dbg) {  // GP_DEBUG_WASTE (host-driven loop): which batch propagated which pixel
        CUDA_TRY(cudaStreamSynchronize(ps));
        int nc = 0;
        CUDA_TRY(cudaMemcpy(&nc, &d_ctl->ncand, 4, cudaMemcpyDeviceToHost));
        std::vector<int> hc((size_t)std::max(nc, 1));
        CUDA_TRY(cudaMemcpy(hc.data(), d_cands, (size_t)nc * 4, cudaMemcpyDeviceToHost));
        for (int i = 0; i < nc; i++) waste_batch[hc[i]] = (int)S.batches - 1;
      }
      return GP_OK;
    };
    const bool pipelined = !debug && !(getenv("GP_PIPELINE") && !atoi(getenv("GP_PIPELINE")));
    bool cut_done = false;           // gp_run_to_host: open rows sent early, later fills patched from the log
    unsigned cut_n = 0;              // log position at the early send
    unsigned long long cut_pairs = 0;
    if (pipelined) {
      // Device-gated pipeline: the host enqueues rounds of [commit, top-K,
      // propagation batch, list switch] on one stream; each kernel checks the
      // control block and does nothing when its case did not arise (top-K
      // only after a miss, the switch kernels only after a switch exit, the
      // commit kernel not after the end), so the GPU never waits for the host.
      // The host checks the status (and streams finished rows) once per
      // CHUNK rounds.
      const unsigned long long lcap = std::max<unsigned long long>(h_ctl.list_switch, 1) + 1024;
      if (lcap > c->list_cap) {
        cudaFree(c->list[0]);
        cudaFree(c->list[1]);
        c->list[0] = c->list[1] = nullptr;
        c->list_cap = 0;
        CUDA_TRY(dalloc(&c->list[0], lcap));
        CUDA_TRY(dalloc(&c->list[1], lcap));
        c->list_cap = lcap;
      }
      ca.plist[0] = c->list[0];
      ca.plist[1] = c->list[1];
      // list mode: several commits per grid step (k_commit_lb); GP_LIST_BATCH=0: one per step
      // (measured: 256^2 list phase 257 -> 140 ms, 128^2 configs -4 ms; 64^2
      // loses -- 2 commits per batch against the batch's two barriers -- so
      // maps below 8192 pixels keep the one-commit steps unless forced)
      const bool lb_on = getenv("GP_LIST_BATCH") ? atoi(getenv("GP_LIST_BATCH")) != 0 : N >= 8192;
      if (ca.cand && ca.strategy != kNaive && commit_split() && lb_on) {
        LbCtl* d_lb = nullptr;
        unsigned long long* d_hits = nullptr;
        CUDA_TRY(ws_get(c, WS_LB, &d_lb, 1));
        CUDA_TRY(ws_get(c, WS_LBHITS, &d_hits, (size_t)c->list_cap));
        CUDA_TRY(cudaMemsetAsync(d_lb, 0, sizeof(LbCtl), st));
        ca.lb = d_lb;
        ca.lb_hits = d_hits;
        if (D_host && !(getenv("GP_E2E_CUT") && atoll(getenv("GP_E2E_CUT")) < 0)) {
          uint2* d_patch = nullptr;  // every list-mode fill is logged: at most one per list entry
          CUDA_TRY(ws_get(c, WS_PATCH, &d_patch, (size_t)c->list_cap));
          ca.patch = d_patch;
        }
        ca.lb_debug = getenv("GP_LB_DEBUG") && atoi(getenv("GP_LB_DEBUG"));
        ca.lb_rcap = 1u << 30;  // GP_LB_RCAP (tests): records above it take the overflow path
        if (const char* e = getenv("GP_LB_RCAP")) ca.lb_rcap = (unsigned)std::max(0, atoi(e));
        ca.lb_pack_min = 65536;
        if (const char* e = getenv("GP_LB_PACK_MIN")) ca.lb_pack_min = (unsigned)std::max(0, atoi(e));
        if (!(getenv("GP_LB_PACK") && !atoi(getenv("GP_LB_PACK")))) {
          uint32_t* d_tinb = nullptr;
          CUDA_TRY(ws_get(c, WS_LBTINB, &d_tinb, (size_t)N * 16));
          ca.lb_tinb = d_tinb;
        }
      }
      // rounds per host check; with host rows, single rounds once few rows
      // are open, so the rows still to copy after the last commit are few
      int chunk = 6;
      if (const char* e = getenv("GP_ROUNDS_PER_SYNC")) chunk = std::max(1, atoi(e));
      auto prop_batch = [&](int gated) -> int {
        EvPair f;
        CUDA_TRY(evp.pair(f));
        CUDA_TRY(cudaEventRecord(f.a, st));
        CUDA_TRY(launch_topk(ca, K, 0, d_cands, d_slots, d_tkeys, gated, st));
        CUDA_TRY(launch_propagate(pa, K, st));
        CUDA_TRY(cudaEventRecord(f.b, st));
        pev.push_back(f);
        S.kernels += 2;
        return GP_OK;
      };
      auto round = [&]() -> int {  // one round: commit launch(es), batch, list switch
        EvPair e;
        CUDA_TRY(evp.pair(e));
        CUDA_TRY(cudaEventRecord(e.a, st));
        CUDA_TRY(commit_split() ? launch_commit_split(ca, nblocks, st) : launch_commit(ca, nblocks, st));
        CUDA_TRY(cudaEventRecord(e.b, st));
        cev.push_back(e);
        S.launches++;
        S.kernels++;
        if (int r = prop_batch(1)) return r;
        CUDA_TRY(launch_switch(ca, c->list[0], st));
        S.kernels += 2;
        return GP_OK;
      };
      hmark("ctx/args");
      if (int r = prop_batch(0)) return r;
      hmark("first batch enqueued");
      if (D_host) {
        // Host rows: rounds with LA rounds of lookahead.  Each round ends with
        // a snapshot of the counts and the control block in pinned buffers
        // (rotating); while rounds r-LA+1 .. r run or wait in the stream, the
        // host reads round r-LA's status and queues the D rows it completed on
        // the copy stream.  With one round of lookahead the GPU ran dry
        // whenever the host needed longer for a round's row copies (~500
        // cudaMemcpyAsync calls) than the GPU for the next round: 114 ms of
        // stream gaps per 256x256 image; with two it never waits (rows left
        // after the last commit: a few hundred, a few ms of D2H).
        cut_pairs = 8000000;  // measured at 256x256 (e2e ms): 3 M 1364, 5 M 1361, 8 M 1357, at the switch 1384 (GP_E2E_CUT: pairs left at the early send; negative: off)
        if (const char* e = getenv("GP_E2E_CUT")) cut_pairs = (unsigned long long)std::max(0ll, atoll(e));
        int e2e_cap = 0;  // GP_E2E_CAP: cap commit launches once half the rows are complete (0: off)
        if (const char* e = getenv("GP_E2E_CAP")) e2e_cap = atoi(e);
        // The host paces itself by the GPU, never by PCIe: it keeps KA rounds
        // queued ahead of the run's stream (events of that stream), reads a
        // round's snapshot whenever its copy has arrived (the copy queues
        // behind the row copies -- up to ~100 ms late in the list phase, and
        // waiting for it starved the GPU), and learns the end of the run from
        // a flag the commit kernel writes into mapped host memory.
        constexpr int NB = 8;  // snapshot buffers / round events (rotating; snapshots are monotone)
        int KA = 3;
        if (const char* e = getenv("GP_E2E_LOOKAHEAD")) KA = std::min(NB - 2, std::max(1, atoi(e)));
        if (!c->h_cnt2) CUDA_TRY(cudaHostAlloc(&c->h_cnt2, (size_t)NB * N * 4, cudaHostAllocDefault));
        if (!c->h_ctl2) CUDA_TRY(cudaHostAlloc(&c->h_ctl2, NB * sizeof(Ctl), cudaHostAllocDefault));
        if (!c->h_done) CUDA_TRY(cudaHostAlloc(&c->h_done, sizeof(int), cudaHostAllocMapped));
        if (!c->d_stage_cnt) CUDA_TRY(dalloc(&c->d_stage_cnt, (size_t)NB * N));
        if (!c->d_stage_ctl) CUDA_TRY(dalloc(&c->d_stage_ctl, NB));
        if (!c->st4) CUDA_TRY(cudaStreamCreateWithFlags(&c->st4, cudaStreamNonBlocking));
        *(volatile int*)c->h_done = 0;
        ca.h_done = c->h_done;
        cudaEvent_t rev[NB], sev[NB];
        for (int i = 0; i < NB; i++) {
          CUDA_TRY(evp.make(&rev[i], cudaEventDisableTiming));
          CUDA_TRY(evp.make(&sev[i], cudaEventDisableTiming));
        }
        auto end_round = [&](int b) -> int {
          // stage on the run's stream (device only), copy out on the snapshot stream
          CUDA_TRY(launch_stage(s->cnt, N, d_ctl, c->d_stage_cnt + (size_t)b * N, c->d_stage_ctl + b, st));
          CUDA_TRY(cudaEventRecord(sev[b], st));
          CUDA_TRY(cudaStreamWaitEvent(c->st4, sev[b], 0));
          CUDA_TRY(cudaMemcpyAsync(c->h_cnt2 + (size_t)b * N, c->d_stage_cnt + (size_t)b * N, (size_t)N * 4,
                                   cudaMemcpyDeviceToHost, c->st4));
          CUDA_TRY(cudaMemcpyAsync(c->h_ctl2 + b, c->d_stage_ctl + b, sizeof(Ctl), cudaMemcpyDeviceToHost, c->st4));
          CUDA_TRY(cudaEventRecord(rev[b], c->st4));
          return GP_OK;
        };
        // log ranges whose copy has arrived: into the host array (row thread + helpers)
        int patch_threads = 8;
        if (const char* e = getenv("GP_E2E_PATCH_THREADS")) patch_threads = std::max(1, std::min(32, atoi(e)));
        auto drain_patches = [&]() {
          size_t done = 0;
          while (done < pchunks.size() && cudaEventQuery(pchunks[done].ev) == cudaSuccess) {
            apply_patches(pchunks[done].b, pchunks[done].e, cut_n, patch_threads);
            done++;
          }
          pchunks.erase(pchunks.begin(), pchunks.begin() + (long)done);
        };
        // one arrived snapshot: status, early send, row copies
        auto process = [&](int round_idx) -> int {
          const int b = round_idx % NB;
          const Ctl hc = c->h_ctl2[b];
          if (hc.status == CTL_LIMIT && ca.max_steps > N) return fail(GP_EINTERNAL, "commit loop stopped unexpectedly");
          // Early send of the open rows.  Rows complete late: the last 13 000 of
          // a 256x256 image in the last 100 ms, more than PCIe delivers in
          // single-row copies.  Once few pairs are left (list mode), every row
          // not sent yet goes out in large contiguous copies; the pairs filled
          // from this snapshot on are in the device's patch log and are written
          // into the host array after the run.
          if (!cut_done && ca.patch && hc.mode == 1 && ca.total_pairs - hc.filled <= cut_pairs) {
            cut_done = true;
            cut_n = hc.patch_n;
            patch_fetched = cut_n;
            const size_t need = (size_t)(ca.total_pairs - hc.filled) + 1024;  // at most one entry per pair still open
            if (c->h_patch_cap < need) {
              if (c->h_patch) cudaFreeHost(c->h_patch);
              c->h_patch = nullptr;
              c->h_patch_cap = 0;
              CUDA_TRY(cudaHostAlloc(&c->h_patch, need * sizeof(uint2), cudaHostAllocDefault));
              c->h_patch_cap = need;
            }
            if (int r = rs.enqueue(true, false)) return r;
            if (htime) fprintf(stderr, "[gp host] early send at round %d (step %d): %llu pairs left, log position %u, at %.1f ms\n",
                               round_idx, hc.step, ca.total_pairs - hc.filled, cut_n, hnow() - h0);
          }
          if (cut_done) {
            // later fills: the log's new entries follow the bulk copies on the
            // copy stream (in order: they arrive after the rows they patch) and
            // are applied as they arrive
            if (hc.patch_n > patch_fetched) {
              PatchChunk pc{patch_fetched, hc.patch_n, nullptr};
              CUDA_TRY(cudaMemcpyAsync(c->h_patch + (pc.b - cut_n), ca.patch + pc.b, (size_t)(pc.e - pc.b) * sizeof(uint2),
                                       cudaMemcpyDeviceToHost, c->st3));
              CUDA_TRY(evp.make(&pc.ev, cudaEventDisableTiming));
              CUDA_TRY(cudaEventRecord(pc.ev, c->st3));
              pchunks.push_back(pc);
              patch_fetched = pc.e;
            }
            drain_patches();
            return GP_OK;
          }
          if (ca.merge_at_switch && hc.mode == 0) return GP_OK;  // one-sided rows: complete only after the switch's pass
          if (int r = rs.enqueue(false, false, c->h_cnt2 + (size_t)b * N)) return r;
          if (htime && round_idx % 8 == 0)
            fprintf(stderr, "[gp host] round %d (step %d, mode %d): %lld rows queued at %.1f ms\n", round_idx, hc.step,
                    hc.mode, (long long)rs.rows_sent, hnow() - h0);
          if (rs.open_rows >= 0 && rs.open_rows < N / 2 && e2e_cap > 0) ca.max_steps = e2e_cap;
          return GP_OK;
        };
        // Row copies are issued by a second host thread: cudaMemcpyAsync blocks
        // once the copy queue is full (the list phase completes rows faster
        // than PCIe carries them), and blocked in it the launching thread left
        // the GPU idle for ~100 ms of a 256x256 run.
        std::atomic<int> nrounds{0}, stop{0}, wrc{0}, want_cap{0};
        int dev = 0;
        CUDA_TRY(cudaGetDevice(&dev));
        const int cap_req = e2e_cap;
        e2e_cap = 0;  // (the worker requests the cap through want_cap)
        std::thread worker;
        try {
          worker = std::thread([&] {
          cudaSetDevice(dev);
          for (int idx = 0;; idx++) {
            while (idx >= nrounds.load(std::memory_order_acquire)) {
              if (stop.load(std::memory_order_acquire) && idx >= nrounds.load(std::memory_order_acquire)) return;
              if (!pchunks.empty()) drain_patches();
              else std::this_thread::sleep_for(std::chrono::microseconds(50));
            }
            if (cudaEventSynchronize(rev[idx % NB]) != cudaSuccess) { wrc.store(GP_ECUDA); return; }
            if (int r = process(idx)) { wrc.store(r); return; }
            if (cap_req > 0 && rs.open_rows >= 0 && rs.open_rows < N / 2) want_cap.store(cap_req);
          }
          });
        } catch (...) {
          return fail(GP_EINTERNAL, "cannot start the row streaming thread");
        }
        struct Joiner {  // every return path joins the worker
          std::thread& t;
          std::atomic<int>& stop;
          ~Joiner() {
            stop.store(1, std::memory_order_release);
            if (t.joinable()) t.join();
          }
        } joiner{worker, stop};
        for (int rr = 0; rr < 8 * N + 16 && !wrc.load(); rr++) {
          if (*(volatile int*)c->h_done) break;  // the device completed the array
          if (rr >= KA) CUDA_TRY(cudaEventSynchronize(sev[(rr - KA) % NB]));  // at most KA rounds ahead of the GPU
          if (*(volatile int*)c->h_done) break;
          if (int cp = want_cap.load()) ca.max_steps = cp;
          if (int r = round()) return r;
          if (int r = end_round(rr % NB)) return r;
          nrounds.store(rr + 1, std::memory_order_release);
        }
        hmark("device reported the end");
        stop.store(1, std::memory_order_release);
        worker.join();
        if (wrc.load()) rc = fail(wrc.load(), "row streaming thread failed");
        hmark("row thread joined");
        hmark("host saw the end");
        CUDA_TRY(cudaStreamSynchronize(c->st4));
        hmark("snapshot stream drained");
        CUDA_TRY(cudaStreamSynchronize(st));
        hmark("run stream drained");
        CUDA_TRY(cudaMemcpy(&h_ctl, d_ctl, sizeof(Ctl), cudaMemcpyDeviceToHost));
        hmark("control block read");
      }
      for (int guard = 0; !D_host && guard < 8 * N + 16; guard += chunk) {
        if (guard) rs.snapshot();  // quiescent point: the previous chunk is complete
        for (int it = 0; it < chunk; it++) {
          EvPair e;
          CUDA_TRY(evp.pair(e));
          CUDA_TRY(cudaEventRecord(e.a, st));
          CUDA_TRY(commit_split() ? launch_commit_split(ca, nblocks, st) : launch_commit(ca, nblocks, st));
          CUDA_TRY(cudaEventRecord(e.b, st));
          cev.push_back(e);
          S.launches++;
          S.kernels++;
          if (int r = prop_batch(1)) return r;
          CUDA_TRY(launch_switch(ca, c->list[0], st));
          S.kernels += 2;
        }
        if (int r = rs.flush()) return r;  // row copies of the last snapshot, during this chunk
        CUDA_TRY(cudaMemcpyAsync(&h_ctl, d_ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, st));
        CUDA_TRY(cudaStreamSynchronize(st));
        if (h_ctl.status == CTL_DONE) break;
        if (h_ctl.status == CTL_LIMIT && ca.max_steps > N) {
          rc = fail(GP_EINTERNAL, "commit loop stopped unexpectedly");
          break;
        }
      }
      S.batches = h_ctl.batches;
    }
    // the first batch must see the initialised workspace on `st`
    if (!pipelined) {
    CUDA_TRY(cudaStreamSynchronize(st));
    if (int r = batch(0)) return r;
    CUDA_TRY(cudaStreamSynchronize(ps));
    fold_pdbg();
    }
    for (int guard = 0; !pipelined && guard < 8 * N + 16; guard++) {
      EvPair e;
      CUDA_TRY(evp.pair(e));
      CUDA_TRY(cudaEventRecord(e.a, st));
      CUDA_TRY(commit_split() ? launch_commit_split(ca, nblocks, st) : launch_commit(ca, nblocks, st));
      CUDA_TRY(cudaEventRecord(e.b, st));
      cev.push_back(e);
      S.launches++;
      S.kernels++;
      CUDA_TRY(cudaMemcpyAsync(&h_ctl, d_ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, st));
      CUDA_TRY(cudaStreamSynchronize(st));
      if (h_ctl.status == CTL_DONE) break;
      if (h_ctl.status == CTL_SWITCH) {  // build the unfilled-pair list, relaunch in list mode
        const unsigned long long need = ca.total_pairs - h_ctl.filled;
        if (need + 1024 > c->list_cap) {
          cudaFree(c->list[0]);
          cudaFree(c->list[1]);
          c->list[0] = c->list[1] = nullptr;
          c->list_cap = 0;
          CUDA_TRY(dalloc(&c->list[0], need + 1024));
          CUDA_TRY(dalloc(&c->list[1], need + 1024));
          c->list_cap = need + 1024;
        }
        ca.plist[0] = c->list[0];
        ca.plist[1] = c->list[1];
        CUDA_TRY(cudaMemsetAsync(&d_ctl->list_n[0], 0, 8, st));
        CUDA_TRY(launch_build_list(L, s->mark, c->list[0], &d_ctl->list_n[0], st));
        h_ctl.mode = 1;
        CUDA_TRY(cudaMemcpyAsync(&d_ctl->mode, &h_ctl.mode, 4, cudaMemcpyHostToDevice, st));
        S.kernels++;
        continue;
      }
      if (h_ctl.status != CTL_MISS) { rc = fail(GP_EINTERNAL, "commit loop stopped unexpectedly"); break; }
      // miss: the selected source's tree is in flight (wait) or unclaimed (urgent batch)
      CUDA_TRY(cudaStreamSynchronize(ps));
      int sl = -1;
      CUDA_TRY(cudaMemcpyAsync(&sl, d_slot_of + h_ctl.cur_src, 4, cudaMemcpyDeviceToHost, st));
      CUDA_TRY(cudaStreamSynchronize(st));
      if (sl < 0) {
        if (int r = batch(0)) return r;
        if (int r = rs.enqueue(false)) return r;  // overlaps the propagation batch
        CUDA_TRY(cudaStreamSynchronize(ps));
        fold_pdbg();
      }
    }
    CUDA_TRY(cudaStreamSynchronize(ps));
    if (one_sided && !(ca.merge_at_switch && h_ctl.mode == 1)) {  // (not yet completed at a list switch)
      CUDA_TRY(launch_merge_sym(s->D, N, st));
      S.kernels += 1;
    }
    CUDA_TRY(cudaEventRecord(tot.b, st));
    CUDA_TRY(cudaMemcpyAsync(&h_ctl, d_ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, st));
    if (d_cen) {
      int cen = -1;
      CUDA_TRY(cudaMemcpyAsync(&cen, d_cen, 4, cudaMemcpyDeviceToHost, st));
      CUDA_TRY(cudaStreamSynchronize(st));
      S.centroid = cen;
    }
    CUDA_TRY(cudaStreamSynchronize(st));
    if (debug) {
      std::vector<unsigned long long> h((size_t)(N + 2) * 4);
      CUDA_TRY(cudaMemcpy(h.data(), d_cdbg, h.size() * 8, cudaMemcpyDeviceToHost));
      if (const char* path = getenv("GP_DEBUG_DUMP")) {  // per-step stamps + new pairs
        std::vector<unsigned long long> nw2(h_ctl.step), hw((size_t)(N + 2) * 4);
        cudaMemcpy(nw2.data(), d_new, (size_t)h_ctl.step * 8, cudaMemcpyDeviceToHost);
        cudaMemcpy(hw.data(), ca.dbgw, hw.size() * 8, cudaMemcpyDeviceToHost);
        std::vector<unsigned long long> hs((size_t)(N + 2) * 8, 0), ho((size_t)(N + 2), 0), hk((size_t)(N + 2), 0);
        if (ca.dbgs) cudaMemcpy(hs.data(), ca.dbgs, hs.size() * 8, cudaMemcpyDeviceToHost);
        cudaMemcpy(ho.data(), ca.dbgo, ho.size() * 8, cudaMemcpyDeviceToHost);
        cudaMemcpy(hk.data(), d_selkey, hk.size() * 8, cudaMemcpyDeviceToHost);
        const int nwarps = nblocks * (commit_threads() / 32);
        if (FILE* fp = fopen(path, "w")) {
          for (int i2 = 0; i2 < h_ctl.step; i2++) {
            unsigned long long* r = &h[(size_t)i2 * 4];
            const unsigned long long* q = &hs[(size_t)i2 * 8];
            fprintf(fp, "%d %llu %llu %llu %llu %llu %llu %llu %llu %llu %llu %llu %llu %llu %llu %llu %llu %llu %llu %llu\n", i2,
                    r[0], r[1], r[2], r[3], nw2[i2], hw[(size_t)i2 * 4], hw[(size_t)i2 * 4 + 1] / (unsigned long long)nwarps,
                    q[0], q[1], q[2], q[3], hw[(size_t)i2 * 4 + 2], hw[(size_t)i2 * 4 + 3] / (unsigned long long)nblocks,
                    q[4], q[5], q[6], q[7], ho[i2], hk[i2] >> 48);
          }
          fclose(fp);
        }
      }
      if (ca.dbgu) {
        std::vector<unsigned> hu((size_t)nparts * 8);
        cudaMemcpy(hu.data(), ca.dbgu, hu.size() * 4, cudaMemcpyDeviceToHost);
        if (FILE* fp = fopen(getenv("GP_DEBUG_UNITS_OUT") ? getenv("GP_DEBUG_UNITS_OUT") : "units.txt", "w")) {
          for (int u = 0; u < nparts; u++) {
            for (int j = 0; j < 8; j++) fprintf(fp, "%u ", hu[(size_t)u * 8 + j]);
            fprintf(fp, "\n");
          }
          fclose(fp);
        }
        cudaFree(ca.dbgu);
      }
      cudaFree(d_cdbg);
      if (pn)
        fprintf(stderr, "[gp debug] propagate per tree (us): relax %.1f parents %.1f jump %.1f levels %.1f out %.1f | passes %.1f items/N %.2f (trees=%lld)\n",
                pacc[1] / 1e3 / pn, pacc[2] / 1e3 / pn, pacc[3] / 1e3 / pn, pacc[4] / 1e3 / pn,
                pacc[5] / 1e3 / pn, pacc[6] / pn, pacc[7] / pn / N, pn);
      if (pn)
        fprintf(stderr, "[gp debug] levels split (us): depth %.1f sort %.1f sizes %.1f preorder %.1f | mean maxdepth %.1f | bucket advances %.1f taking %.1f us\n",
                pacc[8] / 1e3 / pn, pacc[9] / 1e3 / pn, pacc[10] / 1e3 / pn, pacc[11] / 1e3 / pn, pacc[12] / pn,
                pacc[14] / pn, pacc[13] / 1e3 / pn);
      if (pn)
        fprintf(stderr, "[gp debug] E5 offsets %.1f us, E6 arrays %.1f us\n", pacc[15] / 1e3 / pn, e6acc / 1e3 / pn);
      cudaFree(d_pdbg);
    }
    for (auto& e : cev) S.ms_commit += ev_ms(e);
    for (auto& e : pev) S.ms_propagate += ev_ms(e);
    if (htime && pipelined) {  // stream gaps between the timed kernels (GP_DEBUG_HOST)
      double g1 = 0, g2 = 0, gmax = 0;
      for (size_t i = 0; i + 1 < pev.size() && i < cev.size(); i++) {
        float a = 0, b = 0;
        cudaEventElapsedTime(&a, pev[i].b, cev[i].a);      // batch i end -> commit launch i
        cudaEventElapsedTime(&b, cev[i].b, pev[i + 1].a);  // commit launch i end -> batch i + 1
        g1 += a;
        g2 += b;
        gmax = std::max(gmax, (double)std::max(a, b));
      }
      fprintf(stderr, "[gp host] stream gaps: batch->commit %.2f ms, commit->batch %.2f ms (max %.3f) over %zu rounds\n",
              g1, g2, gmax, cev.size());
    }
    P = h_ctl.step;
    S.propagations += h_ctl.total_props;
    if (cl_dbg.p) {
      unsigned long long h[16];
      CUDA_TRY(cudaMemcpy(h, cl_dbg.p, sizeof(h), cudaMemcpyDeviceToHost));
      const double nt = h[13] ? (double)h[13] : 1.0;
      fprintf(stderr, "[gp cluster K1] per tree (us): relax %.1f parents %.1f upsweep %.1f sizes %.1f "
              "e5 %.1f jump %.1f e6a %.1f rest %.1f | passes %.1f advances %.1f jumps %.1f (trees %llu, lite %llu)\n",
              h[1] / nt / 1e3, h[2] / nt / 1e3, h[3] / nt / 1e3, h[4] / nt / 1e3, h[5] / nt / 1e3,
              h[6] / nt / 1e3, h[7] / nt / 1e3, h[8] / nt / 1e3, h[10] / nt, h[11] / nt, h[12] / nt,
              h[13], h[14]);
    }
    if (ca.lb && ca.lb_debug) {
      LbCtl h;
      CUDA_TRY(cudaMemcpy(&h, ca.lb, sizeof(h), cudaMemcpyDeviceToHost));
      const double nb = h.dbg[0] ? (double)h.dbg[0] : 1.0;
      fprintf(stderr, "[gp list batch] batches %llu commits %llu (%.2f per batch, offered %.2f) collects %llu | per batch (us): "
              "select %.2f test %.2f barrier %.2f order %.2f (loads %.2f) apply %.2f barrier %.2f acct %.2f | records %.1f | order loop cycles %.0f\n",
              h.dbg[0], h.dbg[1], h.dbg[1] / nb, h.dbg[2] / nb, h.dbg[3], h.dbg[4] / nb / 1e3, h.dbg[5] / nb / 1e3,
              h.dbg[6] / nb / 1e3, h.dbg[7] / nb / 1e3, h.dbg[14] / nb / 1e3, h.dbg[8] / nb / 1e3, h.dbg[9] / nb / 1e3, h.dbg[10] / nb / 1e3,
              h.dbg[11] / nb, h.dbg[15] / nb);
    }
    if (d_verify) {
      unsigned long long bad = 0;
      CUDA_TRY(cudaMemcpy(&bad, d_verify, 8, cudaMemcpyDeviceToHost));
      S.disagreements = (int64_t)bad;
      if (bad && !rc) rc = fail(GP_EDISAGREE, "verify: " + std::to_string(bad) +
                                                  " already-stored entries disagree with a committed tree");
    }
    S.visits = (int64_t)h_ctl.visits;
    if (cut_done) {
      patch_after_cut = {ca.patch, cut_n};
      h_ctl_final_patch_n = h_ctl.patch_n;
    }
  }
  if (D_host && !rc) {
    CUDA_TRY(cudaStreamSynchronize(st));
    hmark("run done (device)");
    const int64_t before = rs.rows_sent;
    CUDA_TRY(cudaStreamSynchronize(c->st3));
    hmark("streamed copies drained");
    if (int r = rs.enqueue(true)) return r;
    CUDA_TRY(cudaStreamSynchronize(c->st3));
    hmark("final rows copied");
    if (patch_after_cut.first) {  // pairs filled after the early send and not applied during the run
      const unsigned n0 = patch_after_cut.second, n1 = h_ctl_final_patch_n;
      if (n1 > patch_fetched)
        CUDA_TRY(cudaMemcpy(c->h_patch + (patch_fetched - n0), patch_after_cut.first + patch_fetched,
                            (size_t)(n1 - patch_fetched) * sizeof(uint2), cudaMemcpyDeviceToHost));
      const unsigned from = pchunks.empty() ? patch_fetched : pchunks.front().b;  // (the copy stream is drained)
      const int nt = (int)std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
      apply_patches(from, n1, n0, nt);
      hmark("patches applied");
      if (htime) fprintf(stderr, "[gp host] %u pairs patched into the host array, %u of them after the run\n", n1 - n0,
                         n1 - from);
    }
    if (htime) fprintf(stderr, "[gp host] rows streamed during the run %lld, after %lld (open at last snapshot %d); "
                       "%lld copy calls issued in %.1f ms of host time\n",
                       (long long)before, (long long)(rs.rows_sent - before), rs.open_rows, rs.issue_calls, rs.issue_ms);
  }
  S.ms_total = ev_ms(tot);
  S.ms_setup = ev_ms(setup);
  for (auto& m : hmarks) fprintf(stderr, "[gp host] %-24s %8.3f ms\n", m.first, m.second);
  if (rc) return rc;
  std::vector<unsigned long long> nw(P > 0 ? P : 1);
  if (P > 0) CUDA_TRY(cudaMemcpy(nw.data(), d_new, (size_t)P * 8, cudaMemcpyDeviceToHost));
  if (seq_out && P > 0) CUDA_TRY(cudaMemcpy(seq_out, d_seq, (size_t)P * 4, cudaMemcpyDeviceToHost));
  if (g_waste_batch && P > 0) {  // GP_DEBUG_WASTE: propagated-but-never-committed trees per batch
    std::vector<int> hs((size_t)P);
    CUDA_TRY(cudaMemcpy(hs.data(), d_seq, (size_t)P * 4, cudaMemcpyDeviceToHost));
    std::vector<char> committed((size_t)N, 0);
    for (int i = 0; i < P; i++) committed[hs[i]] = 1;
    std::vector<int> per((size_t)S.batches + 1, 0), tot((size_t)S.batches + 1, 0);
    for (int v = 0; v < N; v++)
      if ((*g_waste_batch)[v] >= 0) {
        tot[(*g_waste_batch)[v]]++;
        if (!committed[v]) per[(*g_waste_batch)[v]]++;
      }
    fprintf(stderr, "[gp waste] batch: trees wasted\n");
    for (size_t b = 0; b < per.size(); b++)
      if (tot[b]) fprintf(stderr, "[gp waste] %zu: %d %d\n", b, tot[b], per[b]);
  }
  int64_t filled = 0;
  for (int i = 0; i < P; i++) {
    filled += (int64_t)nw[i];
    if (new_out) new_out[i] = (int64_t)nw[i];
  }
  s->filled = filled;
  S.raw_count = P;
  S.adjusted_count = P + (strategy != GP_STRATEGY_NAIVE ? 2 : 0);  // EXTREMA_OVERHEAD
  S.filled_pairs = filled;
  if (stats) *stats = S;
  const int64_t total = ((int64_t)N * N - N) / 2;
  if (filled != total) return fail(GP_EINTERNAL, "run ended with " + std::to_string(filled) +
                                                     " of " + std::to_string(total) + " pairs");
  return GP_OK;
}
