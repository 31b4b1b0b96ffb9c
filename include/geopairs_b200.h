/*
 * geopairs_b200.h -- C ABI of the B200-native all-pairs geodesic filling path.
 *
 * Plain pointers and sizes only; no torch types.  Every entry point returns
 * GP_OK (0) or a GP_E* status; gp_last_error() returns the message of the
 * calling thread's last failure.  All calls are synchronous w.r.t. the host
 * unless stated otherwise and may be called without the Python GIL.
 *
 * It replaces, one for one, the reference's two native (numba) entry points
 * and the Python loop that drives them (paths relative to
 * /root/reference/pkg/src/geopairs/):
 *
 *   gp_ctx_create        GridGraph.__init__ / _build_csr   propagation.py:52-56,67-89
 *                        (+ Image validation grid.py:47-60)
 *   gp_ctx_load          (new) new image into an existing context
 *   gp_propagate         GridGraph.propagate -> dijkstra_csr propagation.py:58-64,
 *                                                            _kernels.py:33-79
 *   gp_propagate_batch   (new) K independent single-source propagations into a
 *                        device tree store (what run_strategy's loop calls P times)
 *   gp_store_create      DistanceArray.__init__            distances.py:46-61
 *   gp_store_fill_tree   DistanceArray.fill_from_tree -> fill_tree_pairs
 *                                                          distances.py:95-118,
 *                                                          _kernels.py:82-116
 *   gp_store_fill_source DistanceArray.fill_from_source    distances.py:120-147
 *   gp_store_counts      DistanceArray.point_filled_counts distances.py:71-76
 *   gp_store_read        DistanceArray.dist / .mark        distances.py:55-58
 *   gp_store_apgd_rows   DistanceArray.to_bytes            distances.py:149-154
 *   gp_store_load_rows   DistanceArray.from_bytes          distances.py:156-177
 *   gp_store_recount     (from_bytes bookkeeping)          distances.py:174-176
 *   gp_run               run_strategy (naive, filling-rate,  strategies.py:246-273
 *                        extrema)                          (+ selectors :119-129,195-227)
 *   gp_run_to_host       run_strategy + DistanceArray.dist on the host, streamed
 *                        incl. _extrema_context            strategies.py:109-116
 *   gp_extrema           compute_extrema_context           strategies.py:104-116
 *   gp_commit_source     one loop step of a host selector: propagate + build_tree +
 *                        fill_from_tree                    strategies.py:263-271
 */
#ifndef GEOPAIRS_B200_H
#define GEOPAIRS_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  GP_OK = 0,
  GP_EINVAL = 1,     /* bad argument (reference: ValueError) */
  GP_ENOMEM = 2,     /* device allocation failed / size guard */
  GP_ECUDA = 3,      /* CUDA runtime error */
  GP_EINTERNAL = 4,  /* internal invariant violated */
  GP_ECYCLE = 5,     /* parent links contain a cycle (distances.py:111-112) */
  GP_EDISAGREE = 6,  /* value disagrees with a stored entry (distances.py:113-116) */
  GP_EFULL = 7       /* every pair already filled (ArrayFullError, strategies.py:35) */
};

enum { GP_DTYPE_I64 = 0, GP_DTYPE_F32 = 1, GP_DTYPE_U8 = 2 };
enum { GP_METRIC_L1 = 0, GP_METRIC_SUM = 1, GP_METRIC_MEAN = 2 };
enum { GP_STRATEGY_NAIVE = 0, GP_STRATEGY_FILLING_RATE = 1, GP_STRATEGY_EXTREMA = 2 };

typedef struct gp_ctx gp_ctx;     /* image + grid graph + device tree store */
typedef struct gp_store gp_store; /* device distance array D, mark bitmap, counts */

/* Statistics of one gp_run. */
typedef struct {
  int64_t raw_count;       /* committed propagations (FillingTrace.raw_count) */
  int64_t adjusted_count;  /* + EXTREMA_OVERHEAD for filling-rate */
  int64_t centroid;        /* extrema centroid (-1 for naive) */
  int64_t propagations;    /* trees computed incl. speculative ones (+2 extrema) */
  int64_t batches;         /* speculative propagation batches launched */
  int64_t launches;        /* commit-kernel launches */
  int64_t kernels;         /* total kernels launched by the run */
  int64_t filled_pairs;    /* sum of new pairs (== A on completion) */
  int64_t visits;          /* ancestor/descendant pairs of the committed trees
                              (sum of depths, C); 0 for naive */
  double ms_total;         /* device time of the run (CUDA events) */
  double ms_propagate;     /* device time inside propagation batches */
  double ms_commit;        /* device time inside commit launches */
  double ms_setup;         /* store init + extrema */
  int64_t disagreements;   /* GP_VERIFY=1 only: marked pairs a committed tree
                              disagrees with (gp_run then returns GP_EDISAGREE) */
} gp_run_stats;

const char *gp_last_error(void);
int gp_version(void);

/* Image: H x W pixels, row-major.  dtype I64/U8: integer grey levels in
 * [1, 255] (as the reference; rejected otherwise).  dtype F32: finite, >= 0
 * (additive extension).  conn: 8 (reference) or 4 (additive extension).
 * Up to 2^26 pixels; above 65 536 pixels the context serves propagations only
 * (gp_propagate, gp_propagate_batch, gp_extrema: one whole-GPU relaxation per
 * tree), as stores and gp_run are limited to 65 536 pixels. */
int gp_ctx_create(int H, int W, int dtype, const void *pixels, int metric, int conn,
                  gp_ctx **out);
/* Replace the image of an existing context (same shape/metric/connectivity),
 * keeping its device allocations -- for streams of images. */
int gp_ctx_load(gp_ctx *ctx, int dtype, const void *pixels);
void gp_ctx_destroy(gp_ctx *ctx);
int gp_ctx_num_pixels(const gp_ctx *ctx);

/* One (multi-)source propagation; host outputs dist[N] (fp32, exact integers
 * for integer images) and parent[N] (-1 for sources). */
int gp_propagate(gp_ctx *ctx, const int32_t *sources, int nsrc, float *dist_out,
                 int32_t *parent_out);

/* K single-source propagations from device sources src_dev[K] into caller
 * device buffers tdist_dev[K][N] (fp32) and dir_dev[K][N] (3x3 window code of
 * the parent, 0xFF for the root); asynchronous on `stream` (cudaStream_t). */
int gp_propagate_batch(gp_ctx *ctx, const int32_t *src_dev, int k, float *tdist_dev,
                       uint8_t *dir_dev, void *stream);

/* centroid, dist_from_c[N] and ext[N] (host outputs). */
int gp_extrema(gp_ctx *ctx, int32_t *centroid, float *dfc_out, int32_t *ext_out);

/* Distance store of n pixels.  D is fp32 [n][n] in device memory; entries are
 * meaningful where the mark bit is set (diagonal: 0). */
int gp_store_create(int64_t n, gp_store **out);
void gp_store_destroy(gp_store *st);
int gp_store_device_ptrs(gp_store *st, float **D, uint32_t **mark, int32_t **counts,
                         int64_t *mark_words_per_row);
int gp_store_fill_tree(gp_store *st, const int32_t *parent, const float *tdist, float tol,
                       int64_t *new_pairs);
int gp_store_fill_source(gp_store *st, int64_t source, const float *dist, float tol,
                         int64_t *new_pairs);
int gp_store_counts(gp_store *st, int32_t *counts_out, int64_t *filled_pairs);
/* Host copies: D_out[n*n] fp32 (nullable), mark_out[n*n] bytes (nullable). */
int gp_store_read(gp_store *st, float *D_out, uint8_t *mark_out);

/* APGD dump (DistanceArray.to_bytes, distances.py:149-154):
 * rows [row0, row0 + nrows) of the N x N u64 payload into host out[nrows * N],
 * converted on the device (no N^2 host temporaries).  version 1 = the
 * reference's format (integer distances); version 2 (additive, fp32 stores) =
 * binary64 bits of each value.  Unmarked entries: all ones. */
int gp_store_apgd_rows(gp_store *st, int version, int64_t row0, int64_t nrows, uint64_t *out);
/* APGD load (DistanceArray.from_bytes, distances.py:156-177): rows of a
 * payload into D and the mark bitmap (GP_EINVAL when a value does not fit the
 * fp32 store exactly); then gp_store_recount. */
int gp_store_load_rows(gp_store *st, int version, int64_t row0, int64_t nrows, const uint64_t *rows);
/* Per-pixel counts and the filled-pair total recomputed from the mark bitmap
 * (from_bytes: _point_filled = mark.sum(axis=0) - 1, distances.py:174-176). */
int gp_store_recount(gp_store *st, int64_t *filled_pairs);

/* One step of run_strategy's loop for a host-side selector (spiral,
 * spiral-repulsion: strategies.py:132-192, 263-271): propagate from `source`
 * (dijkstra_csr), fill its tree's ancestor/descendant pairs with the
 * reference's agreement / cycle checks (fill_from_tree, distances.py:95-118;
 * tol: relative, 0 = exact) and copy the per-pixel counts into counts_out[n]
 * (host, nullable; pinned memory keeps it asynchronous) for the next
 * selection.  One synchronisation per call, no allocation after the first. */
int gp_commit_source(gp_ctx *ctx, gp_store *st, int32_t source, float tol, int64_t *new_pairs,
                     int32_t *counts_out);

/* run_strategy on the device.  seq_out[n] / new_out[n] receive the committed
 * sources and new pairs per commit (host, nullable); stats nullable.
 * spec_k: speculative batch size (0 = default). */
int gp_run(gp_ctx *ctx, gp_store *st, int strategy, int naive_with_tree, int spec_k,
           int32_t *seq_out, int64_t *new_out, gp_run_stats *stats);

/* gp_run + the host copy of D (fp32 [n][n], D_out; pinned memory lets the
 * copy overlap the run): rows are streamed to the host as they complete
 * (count n-1), the rest after the last commit.  Replaces run_strategy
 * followed by reading DistanceArray.dist (strategies.py:246-273,
 * distances.py:55) in one call. */
int gp_run_to_host(gp_ctx *ctx, gp_store *st, int strategy, int naive_with_tree, int spec_k,
                   int32_t *seq_out, int64_t *new_out, gp_run_stats *stats, float *D_out);

#ifdef __cplusplus
}
#endif
#endif /* GEOPAIRS_B200_H */
