// Kernel argument blocks and launchers shared by the .cu translation units.
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

#include "gp_common.cuh"

namespace gp {

// ---------------- K1 propagation ----------------
struct PropArgs {
  Grid g;
  const float* img;        // [N] grey levels / values (fp32; ints exact)
  const int* src;          // tree t uses src[t*ns .. t*ns+ns)
  int ns;                  // sources per tree
  const int* ntrees_dev;   // optional device tree count (CTAs >= count exit)
  const int* slot;         // optional explicit output slot per tree
  int* slot_counter;       // optional: allocate slots atomically ...
  int* slot_of;            // ... and record slot_of[src] = slot
  float* out_dist;         // [slot][N] (nullable)
  uint8_t* out_dir;        // [slot][N] window codes, GP_ROOT for roots (nullable)
  uint32_t* scratch;       // per-CTA scratch when the map does not fit smem
  size_t scratch_words;
  int in_smem;
  float delta;             // bucket width (inf = plain frontier relaxation)
  float* D;                // naive epilogue: D row/col x > src (nullable)
};

size_t prop_smem_bytes(int N);
size_t prop_scratch_words(int N);
bool prop_fits_smem(int N);
cudaError_t launch_propagate(PropArgs a, int ntrees, cudaStream_t st);

// ---------------- K2/K3 commit loop ----------------
struct Ctl {
  int step;       // next step index
  int cur_src;    // selected source of `step` (-1: not selected yet, -2: none left)
  int status;     // CTL_*
  int nslots;     // trees stored so far
  int ncand;      // candidates produced by the last top-K
  int pad[3];
};
enum { CTL_RUNNING = 0, CTL_DONE = 1, CTL_MISS = 2, CTL_LIMIT = 3 };

struct CommitArgs {
  Grid g;
  int strategy;            // kNaive (naive_with_tree) or kFillingRate
  int NW;                  // 32-bit words per mark row
  const float* tdist;      // tree store [slot][N]
  const uint8_t* tdir;     // tree store [slot][N]
  const int* slot_of;      // [N] slot of a pixel's tree, -1 if none
  uint32_t* mark;          // [N][NW] bitmap, bit (v,u) = row v, column u
  int* cnt;                // [N] marked off-diagonal entries per pixel
  float* D;                // [N][N]
  const int* rank;         // [N] position in the extrema ranking (filling-rate)
  const int* ext;          // [N] pixel at each rank
  unsigned* selkey;        // [N+1] per-step selection key (atomicMin target)
  int* seq;                // [N] committed sources
  unsigned long long* newp;// [N] new pairs per commit
  Ctl* ctl;
  int max_steps;           // commits allowed in this launch
};

cudaError_t launch_commit(const CommitArgs& a, int num_blocks, cudaStream_t st);
int commit_max_blocks();
cudaError_t launch_topk(const CommitArgs& a, int K, int* cands, cudaStream_t st);

// ---------------- store helpers ----------------
cudaError_t launch_store_init(uint32_t* mark, int NW, float* D, int N, cudaStream_t st);
// API-level fills (explicit parent arrays; reference semantics incl. checks)
cudaError_t launch_fill_tree_api(int N, int NW, const int* parent, const float* tdist,
                                 uint32_t* mark, int* cnt, float* D, unsigned long long* out3,
                                 float tol, cudaStream_t st);
cudaError_t launch_fill_source_api(int N, int NW, int s, const float* dist, uint32_t* mark,
                                   int* cnt, float* D, unsigned long long* out3, float tol,
                                   cudaStream_t st);
cudaError_t launch_mark_unpack(const uint32_t* mark, int N, int NW, uint8_t* out, cudaStream_t st);
cudaError_t launch_naive_trace(int N, int NW, uint32_t* mark, int* cnt, int* seq,
                               unsigned long long* newp, cudaStream_t st);
cudaError_t launch_argmax_first(const float* x, int N, int* out, cudaStream_t st);

}  // namespace gp
