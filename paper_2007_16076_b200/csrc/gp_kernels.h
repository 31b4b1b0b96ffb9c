// Kernel argument blocks and launchers shared by the .cu translation units.
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

#include "gp_common.cuh"

namespace gp {

// ---------------- tree store ----------------
// One committed-or-speculative tree per slot, in Euler-tour (preorder) form:
//   pre[q]   entry at preorder position q: (tile column << 16) | pixel (u32)
//   szp[q]   number of descendants of pre[q] (u16)
//   tdp[q]   geodesic distance of pre[q] from the root (fp32)
//   part[p]  start of commit-warp p's share of the fill work, packed
//            q | (chunk offset << 16); chunk = 32 consecutive descendants
//   T        total chunks of the tree
// desc(pre[q]) = pre[q+1 .. q+szp[q]], so the ancestor/descendant pairs of
// the tree are the contiguous ranges of this array (no pointer chasing).
struct TreeStore {
  uint32_t* pre;
  uint16_t* szp;
  float* tdp;
  uint32_t* part;
  uint32_t* T;
  uint32_t* C;  // ancestor/descendant pairs of the tree = sum of depths
  uint32_t* tin;  // per pixel: preorder position | descendant count << 16 (Euler interval)
  int nparts;  // commit warps (partition count)
  unsigned pmagic;  // ceil(2^42 / nparts) when 1024 < nparts < 2^14 (exact x / nparts for x < 2^28), else 0
  int cap;     // slots
};

// ---------------- K1 propagation ----------------
struct PropArgs {
  Grid g;
  const float* img;        // [N] grey levels / values (fp32; ints exact)
  const int* src;          // tree t uses src[t*ns .. t*ns+ns)
  int ns;                  // sources per tree
  const int* ntrees_dev;   // optional device tree count (CTAs >= count exit)
  const int* slot;         // optional output slot per tree (default: t)
  float* out_dist;         // [slot][N] pixel-order distances (nullable)
  uint8_t* out_dir;        // [slot][N] parent window codes (nullable)
  TreeStore ts;            // Euler-tour outputs (ts.pre == nullptr: none)
  MarkLayout L;            // mark-bitmap column layout (tile columns in ts.pre)
  uint8_t* scratch;        // per-CTA scratch when the map does not fit smem
  size_t scratch_bytes;
  int in_smem;
  float delta;             // bucket width (inf = plain frontier relaxation)
  float* D;                // naive epilogue: D row/col x > src (nullable)
  unsigned long long* dbg; // optional per-tree phase stamps [ntrees][8] (debug)
  int* publish;            // optional slot_of[]: set slot_of[src] = slot once the tree is written
  int threads;             // CTA size override (0: automatic)
  const int* list_mode;    // optional &Ctl::mode: == 1 -> list-mode tree (tin/tdp/C only)
  int pos_weights;         // every edge weight > 0 (closed-form parents; cluster K1 allowed)
  unsigned long long* cl_dbg;  // optional cluster-K1 phase time sums [16] (GP_CL_DEBUG)
  int tree_base;           // index of the launch's first tree (chunked launches)
  int exact_heap;          // zero-weight edges: sequential heap-order Dijkstra (generic K1)
  unsigned long long* heap;  // per-CTA heap scratch [heap_words] (exact_heap)
  size_t heap_words;         // u64 words per CTA: heap (8N + ns + 1) + parent codes (N bytes)
  int heap_trees;            // CTAs the heap scratch holds (launches are chunked to it)
};
// heap scratch words of one tree (exact_heap): heap (8N + ns + 1 keys) + N code bytes
inline size_t prop_heap_words(int N, int ns) { return 8 * (size_t)N + (size_t)ns + 1 + ((size_t)N + 7) / 8; }

size_t prop_smem_bytes(int N);
size_t prop_scratch_bytes(int N);
bool prop_fits_smem(int N);
int prop_trees_per_sm(int N);
cudaError_t launch_propagate(PropArgs a, int ntrees, cudaStream_t st);
// propagation-only contexts above 65 536 pixels (propagate_big.cu): one tree on the whole GPU
size_t big_scratch_bytes(int N, int exact);
cudaError_t launch_propagate_big(const Grid& g, const float* img, const int* src, int ns, int exact,
                                 uint32_t* dist_out, uint8_t* code_out, unsigned char* scratch,
                                 unsigned* hflag, cudaStream_t st);
// cluster variant (propagate_cluster.cu): one tree per 2-CTA cluster, state in DSMEM
size_t prop_cluster_smem(int N);
size_t prop_cluster_scratch(int N);
bool prop_cluster_ok(int N);
cudaError_t launch_propagate_cluster(const PropArgs& a, int ntrees, cudaStream_t st);

// ---------------- K2/K3 commit loop ----------------
struct Ctl {
  int step;       // next step index
  int cur_src;    // selected source of `step` (-1: not selected yet, -2: none left)
  int status;     // CTL_*
  int nslots;     // slots ever handed out (bump allocator)
  int ncand;      // candidates produced by the last top-K
  int batches;    // speculative batches that ran (device-gated pipeline)
  int total_props; // trees propagated by speculative batches
  int mode;        // 0: Euler-range fill, 1: unfilled-pair list fill
  unsigned long long visits;  // sum of C over committed trees
  unsigned long long filled;  // pairs filled so far
  unsigned list_n[2];         // entries in the two list buffers
  unsigned list_cur;          // live buffer
  unsigned list_dead;         // dead entries in the live buffer
  unsigned long long list_switch;  // switch to list mode when unfilled <= this
  int build;                       // list build pending (set by k_switch_prep)
  unsigned cand_delta;             // candidate-set width in counts (k_commit, adaptive)
  unsigned cand_cnt[3];            // candidate collection counters (k_commit: step parity; k_commit_lb: rotating)
  unsigned patch_n;                // pairs logged in CommitArgs::patch (gp_run_to_host, list mode)
};
enum { CTL_RUNNING = 0, CTL_DONE = 1, CTL_MISS = 2, CTL_LIMIT = 3, CTL_SWITCH = 4 };

// software grid barrier (count / generation on separate lines)
struct GridBarrier {
  unsigned count;
  unsigned pad0[31];
  unsigned gen;
  unsigned pad1[31];
};

// batched list-mode commits (k_commit_lb): hit / record counters by batch parity, records
struct LbCtl {
  unsigned hit_n[2];
  unsigned rec_n[2];
  uint32_t recs[2048];  // J | endpoint batch indices << 16 / << 24 (0xFF: none)
  unsigned long long dbg[16];  // GP_LB_DEBUG: batches, commits, batch sizes, collects, phase ns sums
};

struct CommitArgs {
  Grid g;
  MarkLayout L;
  int strategy;            // kNaive (naive_with_tree), kFillingRate or kExtrema
  TreeStore ts;
  int* slot_of;            // [N] slot of a pixel's tree, -1 none (or in flight), -2 committed
  uint8_t* claimed;        // [N] 1 once a pixel is handed to a propagation batch
  uint32_t* mark;          // [N][RW] bitmap
  int* cnt;                // [N] marked off-diagonal entries per pixel
  float* D;                // [N][N]
  const int* rank;         // [N] static key part: rank in ext (filling-rate) / class start (extrema)
  const int* ext;          // [N] pixel at each rank
  unsigned long long* selkey;  // [N+2] per-step packed selection (atomicMin target)
  unsigned* stepflags;     // [N+2] per-step decisions from the bookkeeping thread
  int* seq;                // [N] committed sources
  unsigned long long* newp;// [N] new pairs per commit
  Ctl* ctl;
  int max_steps;           // commits allowed in this launch
  unsigned long long* dbg; // optional per-step stamps [steps][4] from block 0 (debug)
  unsigned long long* dbgw; // optional per-step fill times [steps][4] = warp (max, sum), CTA (max, sum) ns
  unsigned long long* dbgs; // optional per-step fill cost model [steps][4] (GP_DEBUG_SIM)
  int fillq;                // tree-mode fill through the per-CTA chunk queue (default 1)
  unsigned* dbgu;           // optional per-unit stats of step dbgu_step (GP_DEBUG_UNITS)
  int dbgu_step;
  unsigned long long* dbgo; // optional per-step open-pixel counts (debug dump)
  GridBarrier* bar;
  uint32_t* plist[2];      // unfilled pairs (u << 16 | w, u < w), list mode
  uint2* patch;            // gp_run_to_host: log of the pairs filled in list mode (anc << 16 | des, value bits);
                           // nullptr: off.  Rows sent to the host early are patched from it.
  int* h_done;             // mapped host flag set when the array is complete (gp_run_to_host; nullptr: off)
  int merge_at_switch;     // one-sided fills completed at the list switch (gp_run_to_host) instead of after the run
  int one_sided;           // tree fills store D[anc][des] only (launch_merge_sym completes D after the run)
  LbCtl* lb;               // batched list-mode commits (nullptr: one commit per step)
  unsigned long long* lb_hits;  // [list capacity] entry index << 16 | J
  int lb_debug;            // GP_LB_DEBUG: phase time sums in lb->dbg
  uint32_t* lb_tinb;       // [N][LB_M] pixel-major Euler words of the batch trees (nullptr: off)
  unsigned lb_pack_min;    // least list length that pays for the transposition
  unsigned lb_rcap;        // records a batch may hold (<= 128; above: the batch commits its first source alone)
  uint32_t* cand;          // [CAND_CAP] candidate set (pixel | rank << 16); nullptr: off
  unsigned compact_div;    // list mode: compact when dead entries > live / compact_div
  int lpt;                 // top-K: candidates deepest-first (longest trees first in the batch)
  unsigned long long total_pairs;
  // opt-in agreement check (GP_VERIFY=1, generic kernel, per-warp unit fill,
  // no list mode, full rows not skipped): marked pairs whose stored value
  // differs from fl(td[w] - td[u]) by more than vtol * max(|value|, 1) are
  // counted here (reference _kernels.py:110-111 -> distances.py:113-116)
  unsigned long long* verify;
  float vtol;
  int verify_corrupt;      // test hook: new pairs of this step are stored +1 (-1: off)
};

void commit_configure(int N);
int commit_threads();
constexpr uint32_t LIST_DEAD = 0xFFFFFFFFu;
cudaError_t launch_commit(const CommitArgs& a, int num_blocks, cudaStream_t st);
bool commit_split();
cudaError_t launch_commit_split(const CommitArgs& a, int num_blocks, cudaStream_t st);
int commit_max_blocks();
int commit_fill_depth();
cudaError_t launch_topk(const CommitArgs& a, int K, int Q, int* cands, int* slots,
                        unsigned* keys, int gated, cudaStream_t st);
// device-gated list switch (pipelined host loop): prep + build only after a CTL_SWITCH exit
cudaError_t launch_switch(const CommitArgs& a, uint32_t* list0, cudaStream_t st);

// ---------------- store helpers ----------------
cudaError_t launch_store_init(const MarkLayout& L, uint32_t* mark, float* D, cudaStream_t st);
cudaError_t launch_merge_sym(float* D, int N, cudaStream_t st);
cudaError_t launch_stage(const int* cnt, int N, const Ctl* ctl, int* s_cnt, Ctl* s_ctl, cudaStream_t st);
// filling-rate ranking on the device (setup.cu): ext / rank from dist_from_c
size_t ext_rank_temp_bytes(int N);
cudaError_t launch_ext_rank(const float* dfc, int N, unsigned long long* keys2, void* temp,
                            size_t temp_bytes, int* ext, int* rank, cudaStream_t st);
// extrema selection key: first position of each pixel's distance class in ext
cudaError_t launch_group_start(const float* dfc, const int* ext, int N, int* gs, cudaStream_t st);
cudaError_t launch_dir_to_parent(const uint8_t* dir, int N, int W, int* parent, cudaStream_t st);
// API-level fills (explicit parent arrays; reference semantics incl. checks)
cudaError_t launch_fill_tree_api(const MarkLayout& L, const int* parent, const float* tdist,
                                 uint32_t* mark, int* cnt, float* D, unsigned long long* out3,
                                 float tol, cudaStream_t st);
cudaError_t launch_fill_source_api(const MarkLayout& L, int s, const float* dist, uint32_t* mark,
                                   int* cnt, float* D, unsigned long long* out3, float tol,
                                   cudaStream_t st);
cudaError_t launch_mark_unpack(const MarkLayout& L, const uint32_t* mark, uint8_t* out,
                               cudaStream_t st);
cudaError_t launch_naive_trace(const MarkLayout& L, uint32_t* mark, int* cnt, int* seq,
                               unsigned long long* newp, cudaStream_t st);
cudaError_t launch_argmax_first(const float* x, int N, int* out, cudaStream_t st);
// APGD (apgd.cu): device-side u64 conversion of row blocks, load, recount
cudaError_t launch_apgd_dump(const MarkLayout& L, const float* D, const uint32_t* mark, long long row0,
                             long long nrows, int version, unsigned long long* out, cudaStream_t st);
cudaError_t launch_apgd_load(const MarkLayout& L, float* D, uint32_t* mark, long long row0, long long nrows,
                             int version, const unsigned long long* in, unsigned long long* bad,
                             cudaStream_t st);
cudaError_t launch_store_recount(const MarkLayout& L, const uint32_t* mark, int* cnt,
                                 unsigned long long* marks, cudaStream_t st);
cudaError_t launch_build_list(const MarkLayout& L, const uint32_t* mark, uint32_t* list,
                              unsigned* count, cudaStream_t st);

}  // namespace gp
