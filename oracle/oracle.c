/*
 * oracle.c -- CPU restatement of the reference `geopairs` hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg may load this library, and
 * only as the checker or the reported CPU baseline -- never as the product.
 *
 * Parity is pinned: for integer images this restatement is checked
 * bit-for-bit against the reference package itself (golden vectors in
 * tests/golden/, produced by tests/golden/make_golden.py importing
 * /root/reference/pkg/src/geopairs) and against the reference's own
 * known-answer tests (tests/test_oracle.py).
 *
 * Every routine cites the reference lines it restates
 * (paths relative to /root/reference/pkg/src/geopairs/):
 *
 *   or_propagate     _kernels.py:33-79   dijkstra_csr (binary heap, key dist*n+id,
 *                                        parent only on strict improvement, stale skip)
 *                    propagation.py:13,67-89 neighbourhood + CSR order
 *                    grid.py:146-154     scaled_weight (x2 scale)
 *   fill_tree        _kernels.py:82-116  fill_tree_pairs (ancestor-chain walk,
 *                                        first writer wins, agreement check, cycle guard)
 *                    distances.py:95-118 fill_from_tree wrapper
 *   fill_source      distances.py:120-147 fill_from_source
 *   extrema          strategies.py:109-116 _extrema_context; propagation.py:130-143
 *   select_*         strategies.py:119-129 (naive), 213-227 (filling-rate)
 *   or_run           strategies.py:246-273 run_strategy
 *
 * Two arithmetic modes:
 *   * int64 (integer images): exactly the reference's arithmetic.
 *   * fp32  (float images, which the reference rejects): the same algorithm
 *     with fp32 distances, w = 2*fl32(fp+fq) (SUM), nd = fl32(d+w), heap key
 *     lexicographic (dist, id) -- the fp32 analogue of dist*n+id.  The
 *     fill's agreement check becomes tolerance-only (relative 1e-4), since
 *     two trees may round a pair's distance differently; first writer wins.
 * Extensions (additive): 4-connectivity.
 */
#include <math.h>
#include <stdint.h>
#include <time.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

enum { OR_L1 = 0, OR_SUM = 1, OR_MEAN = 2 };
enum { OR_NAIVE = 0, OR_FILLING_RATE = 1 };

/* neighbour offsets in ascending-id order: the reference's CSR is lexsorted by
 * (src, dst) (propagation.py:85), so a pixel's edges are visited in ascending
 * neighbour id.  8-conn is propagation.py:13; 4-conn is the additive extension. */
static const int DR8[8] = {-1, -1, -1, 0, 0, 1, 1, 1};
static const int DC8[8] = {-1, 0, 1, -1, 1, -1, 0, 1};
static const int DR4[4] = {-1, 0, 0, 1};
static const int DC4[4] = {0, -1, 1, 0};

typedef struct {
    int H, W, conn, metric, isf;
    const int64_t *pi; /* integer grey levels (isf == 0) */
    const float *pf;   /* fp32 values (isf == 1) */
} img_t;

static inline int nbrs(const img_t *im, int v, int *out) {
    int r = v / im->W, c = v % im->W, k = 0;
    const int *dr = im->conn == 4 ? DR4 : DR8, *dc = im->conn == 4 ? DC4 : DC8;
    for (int i = 0; i < im->conn; i++) {
        int rr = r + dr[i], cc = c + dc[i];
        if (rr < 0 || rr >= im->H || cc < 0 || cc >= im->W) continue;
        out[k++] = rr * im->W + cc;
    }
    return k;
}

/* grid.py:146-154 */
static inline int64_t w_int(const img_t *im, int p, int q) {
    int64_t a = im->pi[p], b = im->pi[q];
    if (im->metric == OR_L1) return 2 * (a > b ? a - b : b - a);
    if (im->metric == OR_SUM) return 2 * (a + b);
    return a + b;
}
static inline float w_f32(const img_t *im, int p, int q) {
    float a = im->pf[p], b = im->pf[q];
    if (im->metric == OR_L1) { float d = a - b; return 2.0f * fabsf(d); }
    if (im->metric == OR_SUM) { float s = a + b; return 2.0f * s; }
    { float s = a + b; return s; }
}

/* ------------------------------------------------------------------ */
/* Dijkstra (_kernels.py:33-79).  Heap entries are (dist, id); ordering is
 * lexicographic, identical to the reference's int64 key dist*n+id.       */
typedef struct { int64_t d; int32_t v; } hi_t;
typedef struct { float d; int32_t v; } hf_t;

#define HEAP_IMPL(NAME, ET)                                                        \
    static inline int NAME##_lt(ET a, ET b) { return a.d < b.d || (a.d == b.d && a.v < b.v); } \
    static inline void NAME##_push(ET *h, int64_t *sz, ET e) {                      \
        int64_t j = (*sz)++;                                                        \
        h[j] = e;                                                                   \
        while (j > 0) {                                                             \
            int64_t up = (j - 1) >> 1;                                              \
            if (NAME##_lt(h[j], h[up])) { ET t = h[up]; h[up] = h[j]; h[j] = t; j = up; } \
            else break;                                                             \
        }                                                                           \
    }                                                                               \
    static inline ET NAME##_pop(ET *h, int64_t *sz) {                               \
        ET top = h[0];                                                              \
        int64_t n = --(*sz);                                                        \
        h[0] = h[n];                                                                \
        int64_t j = 0;                                                              \
        for (;;) {                                                                  \
            int64_t l = 2 * j + 1, r = l + 1, m = j;                                \
            if (l < n && NAME##_lt(h[l], h[m])) m = l;                              \
            if (r < n && NAME##_lt(h[r], h[m])) m = r;                              \
            if (m == j) break;                                                      \
            ET t = h[j]; h[j] = h[m]; h[m] = t; j = m;                              \
        }                                                                           \
        return top;                                                                 \
    }
HEAP_IMPL(hi, hi_t)
HEAP_IMPL(hf, hf_t)

#define UNREACHED_I ((int64_t)1 << 50) /* _kernels.py:15 */

static void dijkstra_i(const img_t *im, const int32_t *src, int ns, int64_t *dist,
                       int32_t *parent, hi_t *heap) {
    int n = im->H * im->W, nb[8];
    int64_t sz = 0;
    for (int i = 0; i < n; i++) { dist[i] = UNREACHED_I; parent[i] = -1; }
    for (int i = 0; i < ns; i++) { dist[src[i]] = 0; hi_push(heap, &sz, (hi_t){0, src[i]}); }
    while (sz > 0) {
        hi_t e = hi_pop(heap, &sz);
        int u = e.v;
        if (e.d != dist[u]) continue; /* stale entry, _kernels.py:70-71 */
        int k = nbrs(im, u, nb);
        for (int j = 0; j < k; j++) {
            int v = nb[j];
            int64_t nd = e.d + w_int(im, u, v);
            if (nd < dist[v]) { dist[v] = nd; parent[v] = u; hi_push(heap, &sz, (hi_t){nd, v}); }
        }
    }
}

static void dijkstra_f(const img_t *im, const int32_t *src, int ns, float *dist,
                       int32_t *parent, hf_t *heap) {
    int n = im->H * im->W, nb[8];
    int64_t sz = 0;
    for (int i = 0; i < n; i++) { dist[i] = INFINITY; parent[i] = -1; }
    for (int i = 0; i < ns; i++) { dist[src[i]] = 0.0f; hf_push(heap, &sz, (hf_t){0.0f, src[i]}); }
    while (sz > 0) {
        hf_t e = hf_pop(heap, &sz);
        int u = e.v;
        if (e.d != dist[u]) continue;
        int k = nbrs(im, u, nb);
        for (int j = 0; j < k; j++) {
            int v = nb[j];
            float nd = e.d + w_f32(im, u, v);
            if (nd < dist[v]) { dist[v] = nd; parent[v] = u; hf_push(heap, &sz, (hf_t){nd, v}); }
        }
    }
}

static int64_t heap_cap(const img_t *im) {
    return (int64_t)im->H * im->W * im->conn + (int64_t)im->H * im->W + 1;
}

/* Public: one propagation.  dist_out is int64[N] (isf=0) or float[N] (isf=1). */
int or_propagate(int H, int W, int conn, int metric, int isf, const void *px,
                 const int32_t *src, int ns, void *dist_out, int32_t *parent_out) {
    img_t im = {H, W, conn, metric, isf, isf ? NULL : (const int64_t *)px,
                isf ? (const float *)px : NULL};
    void *heap = malloc(heap_cap(&im) * (isf ? sizeof(hf_t) : sizeof(hi_t)));
    if (!heap) return -1;
    if (isf) dijkstra_f(&im, src, ns, (float *)dist_out, parent_out, (hf_t *)heap);
    else dijkstra_i(&im, src, ns, (int64_t *)dist_out, parent_out, (hi_t *)heap);
    free(heap);
    return 0;
}

/* ------------------------------------------------------------------ */
/* Distance store (distances.py:46-61): D dense N x N, mark byte matrix,
 * per-pixel filled counts, running pair count.                           */
typedef struct {
    int64_t n;
    void *D;        /* int64 or float, N*N, row-major */
    uint8_t *mark;  /* N*N */
    int64_t *cnt;   /* N */
    int64_t filled;
    int isf;
} store_t;

static const float TOL = 1e-4f; /* agreement tolerance for fp32 (bug detector only) */

/* _kernels.py:82-116 + distances.py:95-118.  Returns new pairs, -1 on a
 * cycle; *bad counts disagreements; *visits counts ancestor visits
 * (sum of depths, the C of SURVEY 8(a) A10).                              */
static int64_t fill_tree(store_t *st, const int32_t *parent, const void *tdist,
                         int64_t *bad_out, int64_t *visits_out, int64_t *walked_out,
                         int nthreads, int skip_full) {
    int64_t n = st->n, newp = 0, bad = 0, visits = 0, walked = 0;
    int cyc = 0;
    (void)nthreads;
#pragma omp parallel for schedule(dynamic, 64) reduction(+ : newp, bad, visits, walked) num_threads(nthreads)
    for (int64_t v = 0; v < n; v++) {
        if (cyc) continue;
        int64_t u = parent[v], steps = 0, lnew = 0;
        /* Exact shortcut: a full row (count n-1) has every pair marked, so its
         * walk can set nothing; only the depth is tallied for the C statistic.
         * Used inside or_run only: there the agreement check is a bug
         * detector (D is pinned separately); or_fill_tree keeps the full
         * reference semantics, including disagreements on full rows.       */
        if (skip_full && __atomic_load_n(&st->cnt[v], __ATOMIC_RELAXED) == n - 1) {
            while (u >= 0) { visits++; u = parent[u]; if (++steps > n) { cyc = 1; break; } }
            continue;
        }
        while (u >= 0) {
            walked++;
            uint8_t *m_uv = &st->mark[u * n + v];
            visits++;
            if (st->isf) {
                const float *td = (const float *)tdist;
                float duv = td[v] - td[u];
                float *D = (float *)st->D;
                if (!*m_uv) {
                    *m_uv = 1; st->mark[v * n + u] = 1;
                    D[u * n + v] = duv; D[v * n + u] = duv;
#pragma omp atomic
                    st->cnt[u] += 1;
                    lnew++;
                } else {
                    float old = D[u * n + v];
                    float tol = TOL * (fabsf(duv) > 1.0f ? fabsf(duv) : 1.0f);
                    if (fabsf(old - duv) > tol) bad++;
                }
            } else {
                const int64_t *td = (const int64_t *)tdist;
                int64_t duv = td[v] - td[u];
                int64_t *D = (int64_t *)st->D;
                if (!*m_uv) {
                    *m_uv = 1; st->mark[v * n + u] = 1;
                    D[u * n + v] = duv; D[v * n + u] = duv;
#pragma omp atomic
                    st->cnt[u] += 1;
                    lnew++;
                } else if (D[u * n + v] != duv) {
                    bad++;
                }
            }
            u = parent[u];
            if (++steps > n) { cyc = 1; break; }
        }
        if (lnew) {
#pragma omp atomic
            st->cnt[v] += lnew;
        }
        newp += lnew;
    }
    *bad_out = bad;
    *visits_out = visits;
    if (walked_out) *walked_out = walked;
    if (cyc) return -1;
    st->filled += newp;
    return newp;
}

/* distances.py:120-147 (agreement check exact for int, tolerance for fp32) */
static int64_t fill_source(store_t *st, int64_t s, const void *dist, int64_t *bad_out) {
    int64_t n = st->n, newp = 0, bad = 0;
    for (int64_t x = 0; x < n; x++) {
        if (x == s) continue;
        if (st->mark[s * n + x]) {
            if (st->isf) {
                float a = ((float *)st->D)[s * n + x], b = ((const float *)dist)[x];
                float tol = TOL * (fabsf(b) > 1.0f ? fabsf(b) : 1.0f);
                if (fabsf(a - b) > tol) bad++;
            } else if (((int64_t *)st->D)[s * n + x] != ((const int64_t *)dist)[x]) {
                bad++;
            }
            continue;
        }
        if (st->isf) {
            float b = ((const float *)dist)[x];
            ((float *)st->D)[s * n + x] = b; ((float *)st->D)[x * n + s] = b;
        } else {
            int64_t b = ((const int64_t *)dist)[x];
            ((int64_t *)st->D)[s * n + x] = b; ((int64_t *)st->D)[x * n + s] = b;
        }
        st->mark[s * n + x] = 1; st->mark[x * n + s] = 1;
        st->cnt[x] += 1;
        newp++;
    }
    st->cnt[s] += newp;
    st->filled += newp;
    *bad_out = bad;
    return newp;
}

/* propagation.py:130-143 */
static int boundary(int W, int H, int32_t *out) {
    int k = 0;
    for (int r = 0; r < H; r++) {
        if (r == 0 || r == H - 1) {
            for (int c = 0; c < W; c++) out[k++] = r * W + c;
        } else {
            out[k++] = r * W;
            if (W > 1) out[k++] = r * W + W - 1;
        }
    }
    return k;
}

/* strategies.py:109-116: centroid = first argmax of the border map; ext =
 * lexsort((id, -dist_from_c)) -> rank[v] = position of v in ext.         */
static const void *g_dfc; static int g_isf;
static int cmp_ext(const void *a, const void *b) {
    int32_t x = *(const int32_t *)a, y = *(const int32_t *)b;
    if (g_isf) {
        float dx = ((const float *)g_dfc)[x], dy = ((const float *)g_dfc)[y];
        if (dx != dy) return dx > dy ? -1 : 1;
    } else {
        int64_t dx = ((const int64_t *)g_dfc)[x], dy = ((const int64_t *)g_dfc)[y];
        if (dx != dy) return dx > dy ? -1 : 1;
    }
    return x < y ? -1 : (x > y);
}

int or_extrema(int H, int W, int conn, int metric, int isf, const void *px,
               int32_t *centroid_out, void *dfc_out, int32_t *ext_out) {
    int n = H * W;
    int32_t *border = malloc(sizeof(int32_t) * (2 * (H + W) + 4));
    int32_t *par = malloc(sizeof(int32_t) * n);
    void *fb = malloc((size_t)n * 8);
    int nb = boundary(W, H, border);
    or_propagate(H, W, conn, metric, isf, px, border, nb, fb, par);
    int cen = 0;
    for (int i = 1; i < n; i++) {
        if (isf ? ((float *)fb)[i] > ((float *)fb)[cen] : ((int64_t *)fb)[i] > ((int64_t *)fb)[cen]) cen = i;
    }
    or_propagate(H, W, conn, metric, isf, px, &cen, 1, dfc_out, par);
    for (int i = 0; i < n; i++) ext_out[i] = i;
    g_dfc = dfc_out; g_isf = isf;
    qsort(ext_out, n, sizeof(int32_t), cmp_ext);
    *centroid_out = cen;
    free(border); free(par); free(fb);
    return 0;
}

/* ------------------------------------------------------------------ */
/* run_strategy (strategies.py:246-273) for NAIVE and FILLING_RATE.
 *   D_out:      int64 or float N*N (caller allocated), complete on return
 *   seq_out:    int32[N] committed sources in order
 *   new_out:    int64[N] new pairs per commit
 *   visits_out: int64[N] ancestor visits per commit (0 for naive fills)
 *   stats[0..]: raw_count, adjusted_count, bad, centroid
 * Returns 0, or -1 (alloc), -2 (cycle), -3 (disagreement).                  */
int or_run(int H, int W, int conn, int metric, int isf, const void *px, int kind,
           int naive_with_tree, int nthreads, void *D_out, int32_t *seq_out,
           int64_t *new_out, int64_t *visits_out, int64_t *walked_out, int64_t *stats,
           int64_t max_steps, double *loop_seconds, double *commit_seconds) {
    int64_t n = (int64_t)H * W;
    img_t im = {H, W, conn, metric, isf, isf ? NULL : (const int64_t *)px,
                isf ? (const float *)px : NULL};
    store_t st = {n, D_out, calloc((size_t)(n * n), 1), calloc(n, sizeof(int64_t)), 0, isf};
    void *heap = malloc(heap_cap(&im) * (isf ? sizeof(hf_t) : sizeof(hi_t)));
    void *td = malloc(n * 8);
    int32_t *par = malloc(n * sizeof(int32_t));
    int32_t *rank = malloc(n * sizeof(int32_t));
    if (!st.mark || !st.cnt || !heap || !td || !par || !rank) return -1;
#pragma omp parallel for num_threads(nthreads > 0 ? nthreads : 1) schedule(static)
    for (int64_t i = 0; i < n; i++) {
        st.mark[i * n + i] = 1;
        if (isf) { float *D = D_out; for (int64_t j = 0; j < n; j++) D[i * n + j] = (i == j) ? 0.0f : -1.0f; }
        else { int64_t *D = D_out; for (int64_t j = 0; j < n; j++) D[i * n + j] = (i == j) ? 0 : -1; }
    }
    int overhead = 0;
    int32_t cen = -1;
    if (kind == OR_FILLING_RATE) {
        int32_t *ext = malloc(n * sizeof(int32_t));
        void *dfc = malloc(n * 8);
        or_extrema(H, W, conn, metric, isf, px, &cen, dfc, ext);
        for (int64_t i = 0; i < n; i++) rank[ext[i]] = (int32_t)i;
        free(ext); free(dfc);
        overhead = 2; /* EXTREMA_OVERHEAD, strategies.py:29 */
    }
    int use_tree = kind != OR_NAIVE || naive_with_tree;
    int64_t total = (n * n - n) / 2, count = 0, bad_total = 0;
    int rc = 0;
    struct timespec t0, t1;
    clock_gettime(CLOCK_MONOTONIC, &t0);
    while (st.filled < total && count < max_steps) {
        /* select (strategies.py:125-129 / 220-227) */
        int64_t s = -1;
        if (kind == OR_NAIVE) {
            for (int64_t i = 0; i < n; i++) if (st.cnt[i] < n - 1) { s = i; break; }
        } else {
            int64_t best_c = INT64_MAX, best_r = INT64_MAX;
            for (int64_t i = 0; i < n; i++) {
                if (st.cnt[i] >= n - 1) continue;
                if (st.cnt[i] < best_c || (st.cnt[i] == best_c && rank[i] < best_r)) {
                    best_c = st.cnt[i]; best_r = rank[i]; s = i;
                }
            }
        }
        if (s < 0) { rc = -4; break; } /* ArrayFullError */
        int32_t s32 = (int32_t)s;
        if (isf) dijkstra_f(&im, &s32, 1, td, par, heap);
        else dijkstra_i(&im, &s32, 1, td, par, heap);
        int64_t bad = 0, visits = 0, walked = 0, newp;
        if (use_tree) newp = fill_tree(&st, par, td, &bad, &visits, &walked, nthreads, 1);
        else newp = fill_source(&st, s, td, &bad);
        if (newp < 0) { rc = -2; break; }
        bad_total += bad;
        seq_out[count] = s32;
        new_out[count] = newp;
        if (visits_out) visits_out[count] = visits;
        if (walked_out) walked_out[count] = walked;
        if (commit_seconds) { /* cumulative loop time after each commit (CPU-baseline sampling) */
            struct timespec tc;
            clock_gettime(CLOCK_MONOTONIC, &tc);
            commit_seconds[count] = (tc.tv_sec - t0.tv_sec) + 1e-9 * (tc.tv_nsec - t0.tv_nsec);
        }
        count++;
    }
    clock_gettime(CLOCK_MONOTONIC, &t1);
    if (loop_seconds) *loop_seconds = (t1.tv_sec - t0.tv_sec) + 1e-9 * (t1.tv_nsec - t0.tv_nsec);
    stats[0] = count;
    stats[1] = count + overhead;
    stats[2] = bad_total;
    stats[3] = cen;
    stats[4] = st.filled;
    if (!rc && bad_total) rc = -3;
    free(st.mark); free(st.cnt); free(heap); free(td); free(par); free(rank);
    return rc;
}

/* Replay helper for the bounded CPU baseline: time the first `steps` commits
 * of a known source sequence (propagate + tree fill), as run_strategy would. */
int or_replay_prefix(int H, int W, int conn, int metric, int isf, const void *px,
                     const int32_t *seq, int64_t steps, int use_tree, int nthreads,
                     int64_t *new_out) {
    int64_t n = (int64_t)H * W;
    img_t im = {H, W, conn, metric, isf, isf ? NULL : (const int64_t *)px,
                isf ? (const float *)px : NULL};
    void *D = malloc((size_t)(n * n) * (isf ? 4 : 8));
    store_t st = {n, D, calloc((size_t)(n * n), 1), calloc(n, sizeof(int64_t)), 0, isf};
    void *heap = malloc(heap_cap(&im) * (isf ? sizeof(hf_t) : sizeof(hi_t)));
    void *td = malloc(n * 8);
    int32_t *par = malloc(n * sizeof(int32_t));
    if (!D || !st.mark || !st.cnt || !heap || !td || !par) return -1;
    for (int64_t i = 0; i < n; i++) st.mark[i * n + i] = 1;
    for (int64_t k = 0; k < steps; k++) {
        int32_t s = seq[k];
        if (isf) dijkstra_f(&im, &s, 1, td, par, heap);
        else dijkstra_i(&im, &s, 1, td, par, heap);
        int64_t bad = 0, visits = 0;
        new_out[k] = use_tree ? fill_tree(&st, par, td, &bad, &visits, NULL, nthreads, 1)
                              : fill_source(&st, s, td, &bad);
    }
    free(D); free(st.mark); free(st.cnt); free(heap); free(td); free(par);
    return 0;
}

/* Single tree fill against caller-owned state (for unit-level parity). */
int64_t or_fill_tree(int64_t n, int isf, const int32_t *parent, const void *tdist, void *D,
                     uint8_t *mark, int64_t *cnt, int64_t *bad_out) {
    store_t st = {n, D, mark, cnt, 0, isf};
    int64_t visits = 0;
    return fill_tree(&st, parent, tdist, bad_out, &visits, NULL, 1, 0);
}
