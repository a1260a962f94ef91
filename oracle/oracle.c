/*
 * oracle.c -- plain, slow, obviously-correct CPU oracle for the LMS hot path of
 * Aupy, Park & Raghavan, "Locality-Aware Laplacian Mesh Smoothing"
 * (arXiv 1606.00803; PAPER.md = /root/reference/PAPER.md, cited as P:<line>).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no code
 * with paper_1606_00803_b200/ (the CUDA product path) and never reads its output.
 *
 * Build: gcc -O2 -ffp-contract=off -fno-fast-math -fopenmp -shared -fPIC
 * (no FMA contraction: every fp64 add/mul/div/sqrt is separately rounded).
 *
 * Functions and the passages they follow:
 *   o_build_csr          vertex adjacency, "N neighbored vertices";
 *                        DESIGN.md reading Z4 (all edge-adjacent vertices)
 *   o_boundary           "interior vertices" of Alg. 1: a vertex is
 *                        fixed iff it lies on an element edge (2D) / face (3D)
 *                        that belongs to exactly one element (reading Z5)
 *   o_quality            edge-length ratio quality: q_e = min edge /
 *                        max edge; q_v = mean over attached elements
 *   o_colour             the fixed colouring schedule (reading Z2): greedy
 *                        first-fit over free vertices in ascending orig_id
 *   o_order_random       random ordering, argsort of counter hash (Z15)
 *   o_order_bfs          BFS ordering, Strout-Hovland, literal queue (Z14)
 *   o_order_rdr          RDR ordering, Alg. 2, literal with two bool
 *                        arrays `processed` and `sorted` (readings Z9-Z12)
 *   o_permute_*          relabelling, V_new[next] <- V[i], perm[new]=old
 *   o_smooth             Eq. 1 inside Alg. 1's loop,
 *                        colour-ordered Gauss-Seidel (readings Z1, Z3)
 *   o_smooth_omp         same sweep, OpenMP static split per colour
 *   o_smooth_partitioned P contiguous parts with ghost copies refreshed after
 *                        every colour (multi-GPU replay; reading Z22)
 *   o_global_quality     Alg. 1 Global_quality = (1/|V|) sum q_v,
 *                        left to right (the exactly rounded sum used by the
 *                        convergence loop is oracle/__init__.py global_quality_exact)
 *   o_smooth_jacobi      N3: Jacobi variant, snapshot reads
 *   o_smooth_seq         N3: Alg. 1 literally, storage-order in-place GS
 *   o_trace              N2: canonical access trace of one sequential sweep
 *   o_reuse_distance     N2: reuse distance of every access, Fenwick
 *   o_order_dfs          N4: DFS preorder (Fig. 2a; reading Z25)
 *   o_order_rcm          N4: reverse Cuthill-McKee (reading Z26)
 *
 * Parity pins for every function live in tests/test_oracle_*.py.
 *
 * Status codes mirror include/lms.h's values but are defined here separately.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define O_OK 0
#define O_E_ARG (-1)
#define O_E_INDEX (-2)
#define O_E_ISOLATED (-3)
#define O_E_PERM (-4)
#define O_E_DEGENERATE (-5)
#define O_E_NOMEM (-6)

void o_free(void* p) { free(p); }

/* ------------------------------------------------------------------------- */
/* O1: CSR.  For each element, for each ordered pair of distinct slots (s,t),
 * insert elems[t] into row elems[s] if absent; then sort each row ascending.  */
typedef struct { int32_t* v; int64_t n, cap; } ivec;

static int ivec_insert_unique(ivec* r, int32_t x) {
    for (int64_t i = 0; i < r->n; ++i) if (r->v[i] == x) return 0;
    if (r->n == r->cap) {
        int64_t nc = r->cap ? 2 * r->cap : 8;
        int32_t* nv = (int32_t*)realloc(r->v, (size_t)nc * sizeof(int32_t));
        if (!nv) return -1;
        r->v = nv; r->cap = nc;
    }
    r->v[r->n++] = x;
    return 0;
}

static int cmp_i32(const void* a, const void* b) {
    int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
    return (x > y) - (x < y);
}

/* Returns status; on success *col_out is malloc'ed (free with o_free). */
int o_build_csr(int64_t V, int32_t k, int64_t n_el, const int32_t* elems,
                int64_t* row_ptr, int32_t** col_out, int64_t* nnz_out) {
    if (V < 0 || k < 2 || n_el < 0) return O_E_ARG;
    for (int64_t e = 0; e < n_el; ++e)
        for (int s = 0; s < k; ++s) {
            int32_t a = elems[e * k + s];
            if (a < 0 || a >= V) return O_E_INDEX;
            for (int t = 0; t < s; ++t) if (elems[e * k + t] == a) return O_E_INDEX;
        }
    ivec* rows = (ivec*)calloc((size_t)(V > 0 ? V : 1), sizeof(ivec));
    if (!rows) return O_E_NOMEM;
    int st = O_OK;
    for (int64_t e = 0; e < n_el && st == O_OK; ++e)
        for (int s = 0; s < k && st == O_OK; ++s)
            for (int t = 0; t < k; ++t) {
                if (s == t) continue;
                if (ivec_insert_unique(&rows[elems[e * k + s]], elems[e * k + t])) { st = O_E_NOMEM; break; }
            }
    int64_t nnz = 0;
    row_ptr[0] = 0;
    for (int64_t v = 0; v < V; ++v) {
        if (rows[v].n == 0 && st == O_OK) st = O_E_ISOLATED;
        nnz += rows[v].n;
        row_ptr[v + 1] = nnz;
    }
    int32_t* col = NULL;
    if (st == O_OK) {
        col = (int32_t*)malloc((size_t)(nnz > 0 ? nnz : 1) * sizeof(int32_t));
        if (!col) st = O_E_NOMEM;
    }
    if (st == O_OK)
        for (int64_t v = 0; v < V; ++v) {
            qsort(rows[v].v, (size_t)rows[v].n, sizeof(int32_t), cmp_i32);
            memcpy(col + row_ptr[v], rows[v].v, (size_t)rows[v].n * sizeof(int32_t));
        }
    for (int64_t v = 0; v < V; ++v) free(rows[v].v);
    free(rows);
    if (st != O_OK) { free(col); return st; }
    *col_out = col;
    *nnz_out = nnz;
    return O_OK;
}

/* ------------------------------------------------------------------------- */
/* O2: boundary.  Sub-simplices (edges for triangles, faces for tetrahedra)
 * keyed by their sorted vertex tuple; a vertex of a tuple of multiplicity 1 is
 * fixed.  (A sort + run count replaces the std::map of SURVEY O2.)          */
typedef struct { int32_t a, b, c; } tup3;

static int cmp_tup3(const void* x, const void* y) {
    const tup3* p = (const tup3*)x; const tup3* q = (const tup3*)y;
    if (p->a != q->a) return (p->a > q->a) - (p->a < q->a);
    if (p->b != q->b) return (p->b > q->b) - (p->b < q->b);
    return (p->c > q->c) - (p->c < q->c);
}

static void sort3(int32_t* v, int n) { /* n <= 3, insertion sort */
    for (int i = 1; i < n; ++i) {
        int32_t x = v[i]; int j = i - 1;
        while (j >= 0 && v[j] > x) { v[j + 1] = v[j]; --j; }
        v[j + 1] = x;
    }
}

int o_boundary(int64_t V, int32_t k, int64_t n_el, const int32_t* elems, uint8_t* fixed) {
    if (k != 3 && k != 4) return O_E_ARG;
    int sub = (k == 3) ? 2 : 3;             /* vertices per sub-simplex */
    int nsub = (k == 3) ? 3 : 4;            /* sub-simplices per element */
    tup3* t = (tup3*)malloc((size_t)(n_el * nsub > 0 ? n_el * nsub : 1) * sizeof(tup3));
    if (!t) return O_E_NOMEM;
    int64_t m = 0;
    for (int64_t e = 0; e < n_el; ++e) {
        const int32_t* w = elems + e * k;
        for (int skip = k - 1; skip >= 0; --skip) {
            int32_t v[3]; int n = 0;
            /* triangle: drop one vertex -> one of its 3 edges;
               tetrahedron: drop one vertex -> one of its 4 faces */
            for (int s = 0; s < k; ++s) if (s != skip) v[n++] = w[s];
            sort3(v, n);
            t[m].a = v[0]; t[m].b = v[1]; t[m].c = (sub == 3) ? v[2] : -1;
            ++m;
        }
    }
    qsort(t, (size_t)m, sizeof(tup3), cmp_tup3);
    memset(fixed, 0, (size_t)V);
    for (int64_t i = 0; i < m;) {
        int64_t j = i + 1;
        while (j < m && cmp_tup3(&t[i], &t[j]) == 0) ++j;
        if (j - i == 1) {
            fixed[t[i].a] = 1; fixed[t[i].b] = 1;
            if (sub == 3) fixed[t[i].c] = 1;
        }
        i = j;
    }
    free(t);
    return O_OK;
}

/* ------------------------------------------------------------------------- */
/* O3: quality.  For element slots (s<t) in lexicographic order,
 * l2 = dx*dx + dy*dy [+ dz*dz]; q_e = sqrt(min l2) / sqrt(max l2).
 * q_v = (sum of q_e over elements containing v, ascending element index) / n_v. */
int o_quality(int32_t dim, int64_t V, const double* const* X, int32_t k, int64_t n_el,
              const int32_t* elems, double* q_elem /* may be NULL */, double* q_v) {
    if (dim != 2 && dim != 3) return O_E_ARG;
    double* qe = (double*)malloc((size_t)(n_el > 0 ? n_el : 1) * sizeof(double));
    int64_t* cnt = (int64_t*)calloc((size_t)(V > 0 ? V : 1), sizeof(int64_t));
    if (!qe || !cnt) { free(qe); free(cnt); return O_E_NOMEM; }
    for (int64_t e = 0; e < n_el; ++e) {
        const int32_t* w = elems + e * k;
        double mn = 0.0, mx = 0.0; int first = 1;
        for (int s = 0; s < k; ++s)
            for (int t = s + 1; t < k; ++t) {
                double l2 = 0.0;
                for (int a = 0; a < dim; ++a) {
                    double d = X[a][w[s]] - X[a][w[t]];
                    double dd = d * d;
                    l2 = (a == 0) ? dd : (l2 + dd);
                }
                if (first) { mn = l2; mx = l2; first = 0; }
                else { if (l2 < mn) mn = l2; if (l2 > mx) mx = l2; }
            }
        if (mx == 0.0) { free(qe); free(cnt); return O_E_DEGENERATE; }
        qe[e] = sqrt(mn) / sqrt(mx);
    }
    for (int64_t v = 0; v < V; ++v) q_v[v] = 0.0;
    /* ascending element index, left-to-right accumulation per vertex */
    for (int64_t e = 0; e < n_el; ++e)
        for (int s = 0; s < k; ++s) {
            int32_t v = elems[e * k + s];
            q_v[v] = (cnt[v] == 0) ? qe[e] : (q_v[v] + qe[e]);
            cnt[v] += 1;
        }
    int st = O_OK;
    for (int64_t v = 0; v < V; ++v) {
        if (cnt[v] == 0) { st = O_E_ISOLATED; break; }
        q_v[v] = q_v[v] / (double)cnt[v];
    }
    if (q_elem) memcpy(q_elem, qe, (size_t)n_el * sizeof(double));
    free(qe); free(cnt);
    return st;
}

/* Alg. 1 lines 4-8: Global_quality = (1/|V|) * sum_i q_{V[i]} (left to right). */
double o_global_quality(int64_t V, const double* q_v) {
    double s = 0.0;
    for (int64_t v = 0; v < V; ++v) s = (v == 0) ? q_v[0] : (s + q_v[v]);
    return V > 0 ? s / (double)V : 0.0;
}

/* ------------------------------------------------------------------------- */
/* O4: colouring (reading Z2).  Visit free vertices in ascending orig_id;
 * colour = smallest c >= 0 not held by an already-coloured free neighbour.
 * Fixed vertices get -1.  Returns C = 1 + max colour (0 if no free vertex).  */
int32_t o_colour(int64_t V, const int64_t* row_ptr, const int32_t* col, const uint8_t* fixed,
                 const int32_t* orig_id /* NULL => identity */, int8_t* colour) {
    int64_t* by_id = (int64_t*)malloc((size_t)(V > 0 ? V : 1) * sizeof(int64_t));
    if (!by_id) return -1;
    for (int64_t v = 0; v < V; ++v) by_id[v] = -1;
    for (int64_t v = 0; v < V; ++v) {
        int64_t id = orig_id ? orig_id[v] : v;
        if (id < 0 || id >= V || by_id[id] != -1) { free(by_id); return -2; }
        by_id[id] = v;
    }
    for (int64_t v = 0; v < V; ++v) colour[v] = -1;
    int32_t C = 0;
    for (int64_t id = 0; id < V; ++id) {
        int64_t v = by_id[id];
        if (fixed[v]) continue;
        unsigned char used[128];
        memset(used, 0, sizeof(used));
        for (int64_t e = row_ptr[v]; e < row_ptr[v + 1]; ++e) {
            int32_t u = col[e];
            if (!fixed[u] && colour[u] >= 0) used[(int)colour[u]] = 1;
        }
        int c = 0;
        while (used[c]) ++c;
        if (c > 127) { free(by_id); return -3; }
        colour[v] = (int8_t)c;
        if (c + 1 > C) C = c + 1;
    }
    free(by_id);
    return C;
}

/* ------------------------------------------------------------------------- */
/* Counter hash H(seed, stream, i) = SM(SM(seed + stream) + i) (reading Z15).  */
static uint64_t sm64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
uint64_t o_hash(uint64_t seed, uint64_t stream, uint64_t i) { return sm64(sm64(seed + stream) + i); }

typedef struct { uint64_t key; int64_t idx; } kv64;
static int cmp_kv64(const void* a, const void* b) {
    const kv64* p = (const kv64*)a; const kv64* q = (const kv64*)b;
    if (p->key != q->key) return (p->key > q->key) - (p->key < q->key);
    return (p->idx > q->idx) - (p->idx < q->idx);
}

/* O5 original: identity. */
void o_order_original(int64_t V, int32_t* perm) { for (int64_t i = 0; i < V; ++i) perm[i] = (int32_t)i; }

/* O5 random: perm = indices sorted by key H(seed, 4, i). */
int o_order_random(int64_t V, uint64_t seed, int32_t* perm) {
    kv64* a = (kv64*)malloc((size_t)(V > 0 ? V : 1) * sizeof(kv64));
    if (!a) return O_E_NOMEM;
    for (int64_t i = 0; i < V; ++i) { a[i].key = o_hash(seed, 4, (uint64_t)i); a[i].idx = i; }
    qsort(a, (size_t)V, sizeof(kv64), cmp_kv64);
    for (int64_t i = 0; i < V; ++i) perm[i] = (int32_t)a[i].idx;
    free(a);
    return O_OK;
}

/* O5 BFS (reading Z14): queue BFS from `seed`, neighbours enqueued in
 * ascending (CSR) order, restart at the smallest unvisited vertex.            */
int o_order_bfs(int64_t V, const int64_t* row_ptr, const int32_t* col, int64_t seed, int32_t* perm) {
    if (V == 0) return O_OK;
    if (seed < 0 || seed >= V) return O_E_ARG;
    uint8_t* vis = (uint8_t*)calloc((size_t)V, 1);
    if (!vis) return O_E_NOMEM;
    int64_t head = 0, tail = 0, next_unvisited = 0;
    int64_t start = seed;
    while (tail < V) {
        if (head == tail) {                         /* (re)start a component */
            if (vis[start]) {
                while (next_unvisited < V && vis[next_unvisited]) ++next_unvisited;
                start = next_unvisited;
            }
            vis[start] = 1; perm[tail++] = (int32_t)start;
        }
        int32_t v = perm[head++];
        for (int64_t e = row_ptr[v]; e < row_ptr[v + 1]; ++e) {
            int32_t u = col[e];
            if (!vis[u]) { vis[u] = 1; perm[tail++] = u; }
        }
    }
    free(vis);
    return O_OK;
}

/* O5 RDR: Alg. 2, literally.
 *  - outer loop over interior (free) vertices sorted by increasing (q, label) (Z9)
 *  - l = {unprocessed neighbours of i sorted by increasing (q, label)}
 *  - all unsorted members of l appended in order; processed[l[0]] <- True;
 *    l <- unprocessed neighbours of l[0]  (Z10: l[0] is l's first element)
 *  - fixed vertices may be appended / processed inside a walk (Z11)
 *  - vertices never sorted are appended in ascending label at the end (Z12)
 * Returns the number of walks in *n_walks (may be NULL) and tail size in *n_tail. */
typedef struct { double q; int32_t v; } qv;
static int cmp_qv(const void* a, const void* b) {
    const qv* p = (const qv*)a; const qv* r = (const qv*)b;
    if (p->q < r->q) return -1;
    if (p->q > r->q) return 1;
    return (p->v > r->v) - (p->v < r->v);
}

int o_order_rdr(int64_t V, const int64_t* row_ptr, const int32_t* col, const uint8_t* fixed,
                const double* q, int32_t* perm, int64_t* n_walks, int64_t* n_tail) {
    uint8_t* processed = (uint8_t*)calloc((size_t)(V > 0 ? V : 1), 1);
    uint8_t* sorted = (uint8_t*)calloc((size_t)(V > 0 ? V : 1), 1);
    qv* outer = (qv*)malloc((size_t)(V > 0 ? V : 1) * sizeof(qv));
    int64_t maxdeg = 0;
    for (int64_t v = 0; v < V; ++v) if (row_ptr[v + 1] - row_ptr[v] > maxdeg) maxdeg = row_ptr[v + 1] - row_ptr[v];
    qv* l = (qv*)malloc((size_t)(maxdeg > 0 ? maxdeg : 1) * sizeof(qv));
    if (!processed || !sorted || !outer || !l) {
        free(processed); free(sorted); free(outer); free(l); return O_E_NOMEM;
    }
    int64_t n_outer = 0;
    for (int64_t v = 0; v < V; ++v) if (!fixed[v]) { outer[n_outer].q = q[v]; outer[n_outer].v = (int32_t)v; ++n_outer; }
    qsort(outer, (size_t)n_outer, sizeof(qv), cmp_qv);
    int64_t next_num = 0, walks = 0;
    for (int64_t oi = 0; oi < n_outer; ++oi) {
        int32_t i = outer[oi].v;
        if (processed[i]) continue;
        if (!sorted[i]) { perm[next_num++] = i; sorted[i] = 1; }
        processed[i] = 1;
        ++walks;
        int32_t cur = i;
        for (;;) {
            int64_t nl = 0;
            for (int64_t e = row_ptr[cur]; e < row_ptr[cur + 1]; ++e) {
                int32_t u = col[e];
                if (!processed[u]) { l[nl].q = q[u]; l[nl].v = u; ++nl; }
            }
            if (nl == 0) break;
            qsort(l, (size_t)nl, sizeof(qv), cmp_qv);
            for (int64_t j = 0; j < nl; ++j)
                if (!sorted[l[j].v]) { perm[next_num++] = l[j].v; sorted[l[j].v] = 1; }
            processed[l[0].v] = 1;
            cur = l[0].v;
        }
    }
    int64_t tail = 0;
    for (int64_t v = 0; v < V; ++v) if (!sorted[v]) { perm[next_num++] = (int32_t)v; sorted[v] = 1; ++tail; }
    if (n_walks) *n_walks = walks;
    if (n_tail) *n_tail = tail;
    free(processed); free(sorted); free(outer); free(l);
    return next_num == V ? O_OK : O_E_PERM;
}

/* ------------------------------------------------------------------------- */
/* O6 permute.  perm[new] = old (V_new[next_num] <- V[i]).             */
int o_inverse_perm(int64_t V, const int32_t* perm, int32_t* inv) {
    for (int64_t i = 0; i < V; ++i) inv[i] = -1;
    for (int64_t k = 0; k < V; ++k) {
        int32_t p = perm[k];
        if (p < 0 || p >= V || inv[p] != -1) return O_E_PERM;
        inv[p] = (int32_t)k;
    }
    return O_OK;
}

/* elems'[i][s] = inv[elems[i][s]] (element and slot order kept). */
void o_permute_elems(int64_t n_el, int32_t k, const int32_t* inv, const int32_t* elems, int32_t* out) {
    for (int64_t i = 0; i < n_el * k; ++i) out[i] = inv[elems[i]];
}

/* CSR' rows: row k' = inv[cols of old row perm[k']], sorted ascending. */
int o_permute_csr(int64_t V, const int32_t* perm, const int32_t* inv, const int64_t* row_ptr,
                  const int32_t* col, int64_t* row_ptr2, int32_t* col2) {
    row_ptr2[0] = 0;
    for (int64_t k = 0; k < V; ++k) {
        int32_t old = perm[k];
        int64_t d = row_ptr[old + 1] - row_ptr[old];
        for (int64_t e = 0; e < d; ++e) col2[row_ptr2[k] + e] = inv[col[row_ptr[old] + e]];
        qsort(col2 + row_ptr2[k], (size_t)d, sizeof(int32_t), cmp_i32);
        row_ptr2[k + 1] = row_ptr2[k] + d;
    }
    return O_OK;
}

/* ------------------------------------------------------------------------- */
/* O7 sweep: Eq. 1 in Alg. 1's loop, colour-ordered
 * Gauss-Seidel (reading Z1).  For s < S: for c < C: for v in storage order with
 * colour[v] == c: for each axis: acc = X[u0]; acc = acc + X[ui] (CSR order);
 * X[v] = acc / (double)deg(v).  In place.                                      */
int o_smooth(int32_t dim, int64_t V, double* const* X, const int64_t* row_ptr, const int32_t* col,
             const int8_t* colour, int32_t C, int32_t sweeps) {
    if (sweeps < 0 || dim < 1 || dim > 3) return O_E_ARG;
    for (int32_t s = 0; s < sweeps; ++s)
        for (int32_t c = 0; c < C; ++c)
            for (int64_t v = 0; v < V; ++v) {
                if (colour[v] != c) continue;
                int64_t b = row_ptr[v], e = row_ptr[v + 1];
                if (e == b) return O_E_ISOLATED;
                for (int a = 0; a < dim; ++a) {
                    double acc = X[a][col[b]];
                    for (int64_t i = b + 1; i < e; ++i) acc = acc + X[a][col[i]];
                    X[a][v] = acc / (double)(e - b);
                }
            }
    return O_OK;
}

/* O8: the same sweep, each colour's vertex list split statically over OpenMP
 * threads (the paper's OpenMP static split).  Bit-identical to O7
 * because same-colour vertices are never adjacent.  Returns threads used.     */
int o_smooth_omp(int32_t dim, int64_t V, double* const* X, const int64_t* row_ptr, const int32_t* col,
                 const int8_t* colour, int32_t C, int32_t sweeps, int32_t nthreads) {
    if (sweeps < 0 || dim < 1 || dim > 3) return O_E_ARG;
    int64_t* cnt = (int64_t*)calloc((size_t)C + 1, sizeof(int64_t));
    int32_t* lst = (int32_t*)malloc((size_t)(V > 0 ? V : 1) * sizeof(int32_t));
    if (!cnt || !lst) { free(cnt); free(lst); return O_E_NOMEM; }
    for (int64_t v = 0; v < V; ++v) if (colour[v] >= 0) cnt[colour[v] + 1]++;
    for (int32_t c = 0; c < C; ++c) cnt[c + 1] += cnt[c];
    int64_t* fill = (int64_t*)malloc(((size_t)C + 1) * sizeof(int64_t));
    memcpy(fill, cnt, ((size_t)C + 1) * sizeof(int64_t));
    for (int64_t v = 0; v < V; ++v) if (colour[v] >= 0) lst[fill[colour[v]]++] = (int32_t)v;
    free(fill);
    int used = 1;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#endif
    for (int32_t s = 0; s < sweeps; ++s)
        for (int32_t c = 0; c < C; ++c) {
#ifdef _OPENMP
#pragma omp parallel for schedule(static)
#endif
            for (int64_t i = cnt[c]; i < cnt[c + 1]; ++i) {
                int32_t v = lst[i];
                int64_t b = row_ptr[v], e = row_ptr[v + 1];
                for (int a = 0; a < dim; ++a) {
                    double acc = X[a][col[b]];
                    for (int64_t j = b + 1; j < e; ++j) acc = acc + X[a][col[j]];
                    X[a][v] = acc / (double)(e - b);
                }
            }
        }
#ifdef _OPENMP
#pragma omp parallel
    {
#pragma omp single
        used = omp_get_num_threads();
    }
#endif
    free(cnt); free(lst);
    return used;
}

/* O9: partitioned replay (reading Z22).  Storage order is split into P
 * contiguous ranges with (ceil-)equal free-vertex counts.  Part p owns its
 * range and keeps private copies of every coordinate it reads (owned + ghost).
 * Per colour: each part updates its owned colour-c vertices from its private
 * copy; then every ghost copy is refreshed from its owner.  The result must be
 * bit-identical to o_smooth.  Part boundaries are returned in bounds[P+1].    */
int o_smooth_partitioned(int32_t dim, int64_t V, double* const* X, const int64_t* row_ptr,
                         const int32_t* col, const int8_t* colour, int32_t C, int32_t sweeps,
                         int32_t P, int64_t* bounds) {
    if (P < 1 || sweeps < 0) return O_E_ARG;
    int64_t nfree = 0;
    for (int64_t v = 0; v < V; ++v) if (colour[v] >= 0) ++nfree;
    int64_t per = (nfree + P - 1) / P;
    /* bounds: part p ends after its per-th free vertex */
    bounds[0] = 0;
    {
        int64_t seen = 0; int32_t p = 0;
        for (int64_t v = 0; v < V && p < P - 1; ++v) {
            if (colour[v] >= 0) {
                ++seen;
                if (seen == per * (p + 1)) { bounds[++p] = v + 1; }
            }
        }
        while (p < P - 1) { bounds[p + 1] = V; ++p; }   /* tiny meshes */
        bounds[P] = V;
        for (int32_t q2 = 1; q2 <= P; ++q2) if (bounds[q2] < bounds[q2 - 1]) bounds[q2] = bounds[q2 - 1];
    }
    /* private full-size copies per part (simple, slow, obviously correct) */
    double** priv = (double**)malloc((size_t)P * 3 * sizeof(double*));
    if (!priv) return O_E_NOMEM;
    for (int32_t p = 0; p < P; ++p)
        for (int a = 0; a < dim; ++a) {
            priv[p * 3 + a] = (double*)malloc((size_t)(V > 0 ? V : 1) * sizeof(double));
            memcpy(priv[p * 3 + a], X[a], (size_t)V * sizeof(double));
        }
    for (int32_t s = 0; s < sweeps; ++s)
        for (int32_t c = 0; c < C; ++c) {
            for (int32_t p = 0; p < P; ++p)
                for (int64_t v = bounds[p]; v < bounds[p + 1]; ++v) {
                    if (colour[v] != c) continue;
                    int64_t b = row_ptr[v], e = row_ptr[v + 1];
                    for (int a = 0; a < dim; ++a) {
                        double* Y = priv[p * 3 + a];
                        double acc = Y[col[b]];
                        for (int64_t i = b + 1; i < e; ++i) acc = acc + Y[col[i]];
                        Y[v] = acc / (double)(e - b);
                    }
                }
            /* ghost refresh: owner's colour-c values copied into every other part */
            for (int32_t p = 0; p < P; ++p)
                for (int64_t v = bounds[p]; v < bounds[p + 1]; ++v) {
                    if (colour[v] != c) continue;
                    for (int32_t r = 0; r < P; ++r) if (r != p)
                        for (int a = 0; a < dim; ++a) priv[r * 3 + a][v] = priv[p * 3 + a][v];
                }
        }
    for (int32_t p = 0; p < P; ++p)
        for (int64_t v = bounds[p]; v < bounds[p + 1]; ++v)
            for (int a = 0; a < dim; ++a) X[a][v] = priv[p * 3 + a][v];
    for (int32_t p = 0; p < P; ++p) for (int a = 0; a < dim; ++a) free(priv[p * 3 + a]);
    free(priv);
    return O_OK;
}

/* ------------------------------------------------------------------------- */
/* N3: Jacobi sweep ("reads all neighbor positions from the
 * start-of-iteration snapshot"): every free vertex moves to the mean of its
 * neighbours' PREVIOUS-sweep coordinates (Eq. 1), CSR-order sums,
 * IEEE division; fixed vertices (colour < 0) keep their value.  An explicitly
 * named schedule variant (reading Z1): NOT the colour-GS result.             */
int o_smooth_jacobi(int32_t dim, int64_t V, double* const* X, const int64_t* row_ptr, const int32_t* col,
                    const uint8_t* fixed, int32_t sweeps) {
    if (sweeps < 0 || dim < 1 || dim > 3) return O_E_ARG;
    double* old = (double*)malloc((size_t)(V > 0 ? V : 1) * sizeof(double));
    if (!old) return O_E_NOMEM;
    for (int32_t s = 0; s < sweeps; ++s)
        for (int a = 0; a < dim; ++a) {
            memcpy(old, X[a], (size_t)V * sizeof(double));          /* the snapshot */
            for (int64_t v = 0; v < V; ++v) {
                if (fixed[v]) continue;
                int64_t b = row_ptr[v], e = row_ptr[v + 1];
                if (e == b) { free(old); return O_E_ISOLATED; }
                double acc = old[col[b]];
                for (int64_t i = b + 1; i < e; ++i) acc = acc + old[col[i]];
                X[a][v] = acc / (double)(e - b);
            }
        }
    free(old);
    return O_OK;
}

/* N3: Alg. 1 literally: "for i in {interior vertices}: smooth V[i]
 * using Eq. 1", sequentially and in place, in STORAGE order -- each vertex
 * reads the current values, so the result depends on the ordering (reading
 * Z21).  CPU only (the GPU cannot run a sequential loop); used to compare
 * convergence with the colour schedule.                                       */
int o_smooth_seq(int32_t dim, int64_t V, double* const* X, const int64_t* row_ptr, const int32_t* col,
                 const uint8_t* fixed, int32_t sweeps) {
    if (sweeps < 0 || dim < 1 || dim > 3) return O_E_ARG;
    for (int32_t s = 0; s < sweeps; ++s)
        for (int64_t v = 0; v < V; ++v) {
            if (fixed[v]) continue;
            int64_t b = row_ptr[v], e = row_ptr[v + 1];
            if (e == b) return O_E_ISOLATED;
            for (int a = 0; a < dim; ++a) {
                double acc = X[a][col[b]];
                for (int64_t i = b + 1; i < e; ++i) acc = acc + X[a][col[i]];
                X[a][v] = acc / (double)(e - b);
            }
        }
    return O_OK;
}

/* ------------------------------------------------------------------------- */
/* N2: the paper's reuse-distance instrument (Sec. 3.1; Table III,
 * P:646-702).  o_trace: the canonical access trace of ONE sequential sweep
 * (Alg. 1's loop over interior vertices) at vertex granularity
 * (SPEC trace_iteration): for each free vertex v in storage order: v, its
 * neighbours in CSR order, v again (the write of Eq. 1).  Returns the length;
 * trace may be NULL (length only).                                           */
int64_t o_trace(int64_t V, const int64_t* row_ptr, const int32_t* col, const uint8_t* fixed, int32_t* trace) {
    int64_t n = 0;
    for (int64_t v = 0; v < V; ++v) {
        if (fixed[v]) continue;
        if (trace) trace[n] = (int32_t)v;
        ++n;
        for (int64_t e = row_ptr[v]; e < row_ptr[v + 1]; ++e) {
            if (trace) trace[n] = col[e];
            ++n;
        }
        if (trace) trace[n] = (int32_t)v;
        ++n;
    }
    return n;
}

/* Reuse distance of every access ("between two accesses to the same
 * data, what are the number of distinct piece of data that were accessed"):
 * the number of DISTINCT elements accessed since the previous access to the
 * same element, -1 (COLD) for a first access.  The O(N log N) algorithm of
 * SPEC reuse_distances: last-access times, and a Fenwick tree over time
 * holding a 1 at the last access of every element seen so far; the distance
 * of access t to an element last seen at time p is the number of 1s in
 * (p, t).  n_ids bounds the element identifiers.                             */
int o_reuse_distance(int64_t n, const int32_t* trace, int64_t n_ids, int64_t* dist) {
    int64_t* last = (int64_t*)malloc((size_t)(n_ids > 0 ? n_ids : 1) * sizeof(int64_t));
    int64_t* bit = (int64_t*)calloc((size_t)n + 1, sizeof(int64_t));
    if (!last || !bit) { free(last); free(bit); return O_E_NOMEM; }
    for (int64_t k = 0; k < n_ids; ++k) last[k] = -1;
    for (int64_t t = 0; t < n; ++t) {
        int32_t x = trace[t];
        if (x < 0 || x >= n_ids) { free(last); free(bit); return O_E_INDEX; }
        int64_t p = last[x];
        if (p < 0) {
            dist[t] = -1;
        } else {
            /* ones in (p, t) = prefix(t - 1) - prefix(p) (Fenwick prefix sums, 1-based) */
            int64_t a = 0, b = 0;
            for (int64_t i = t; i > 0; i -= i & (-i)) a += bit[i];
            for (int64_t i = p + 1; i > 0; i -= i & (-i)) b += bit[i];
            dist[t] = a - b;
            for (int64_t i = p + 1; i <= n; i += i & (-i)) bit[i] -= 1;  /* p is no longer a last access */
        }
        for (int64_t i = t + 1; i <= n; i += i & (-i)) bit[i] += 1;
        last[x] = t;
    }
    free(last); free(bit);
    return O_OK;
}

/* ------------------------------------------------------------------------- */
/* N4 orderings.
 * o_order_dfs: depth-first preorder (the DFS ordering of Fig. 2a, P:310-313;
 * reading Z25): from `seed`, always descend to the SMALLEST unvisited
 * neighbour of the deepest vertex that still has one (recursive DFS with rows
 * in ascending order), restart at the smallest unvisited label.           */
int o_order_dfs(int64_t V, const int64_t* row_ptr, const int32_t* col, int64_t seed, int32_t* perm) {
    if (V == 0) return O_OK;
    if (seed < 0 || seed >= V) return O_E_ARG;
    uint8_t* vis = (uint8_t*)calloc((size_t)V, 1);
    int32_t* stk = (int32_t*)malloc((size_t)V * sizeof(int32_t));
    int64_t* cur = (int64_t*)malloc((size_t)V * sizeof(int64_t));   /* next row entry to try */
    if (!vis || !stk || !cur) { free(vis); free(stk); free(cur); return O_E_NOMEM; }
    int64_t n = 0, top = 0, next_unvisited = 0, start = seed;
    while (n < V) {
        if (vis[start]) {
            while (next_unvisited < V && vis[next_unvisited]) ++next_unvisited;
            start = next_unvisited;
        }
        vis[start] = 1; perm[n++] = (int32_t)start;
        stk[top++] = (int32_t)start; cur[start] = row_ptr[start];
        while (top > 0) {
            int32_t v = stk[top - 1];
            while (cur[v] < row_ptr[v + 1] && vis[col[cur[v]]]) ++cur[v];
            if (cur[v] == row_ptr[v + 1]) { --top; continue; }
            int32_t u = col[cur[v]++];
            vis[u] = 1; perm[n++] = u;
            stk[top++] = u; cur[u] = row_ptr[u];
        }
    }
    free(vis); free(stk); free(cur);
    return O_OK;
}

/* o_order_rcm: reverse Cuthill-McKee (reading Z26): queue BFS that starts at
 * the unvisited vertex of smallest (degree, label), enqueues each vertex's
 * unvisited neighbours in ascending (degree, label), restarts the same way on
 * a new component; the visit order reversed.                               */
typedef struct { int64_t d; int32_t v; } dv;
static int cmp_dv(const void* a, const void* b) {
    const dv* p = (const dv*)a; const dv* q = (const dv*)b;
    if (p->d != q->d) return (p->d > q->d) - (p->d < q->d);
    return (p->v > q->v) - (p->v < q->v);
}
int o_order_rcm(int64_t V, const int64_t* row_ptr, const int32_t* col, int32_t* perm) {
    if (V == 0) return O_OK;
    uint8_t* vis = (uint8_t*)calloc((size_t)V, 1);
    int32_t* q = (int32_t*)malloc((size_t)V * sizeof(int32_t));
    dv* byd = (dv*)malloc((size_t)V * sizeof(dv));
    int64_t maxdeg = 0;
    for (int64_t v = 0; v < V; ++v) if (row_ptr[v + 1] - row_ptr[v] > maxdeg) maxdeg = row_ptr[v + 1] - row_ptr[v];
    dv* l = (dv*)malloc((size_t)(maxdeg > 0 ? maxdeg : 1) * sizeof(dv));
    if (!vis || !q || !byd || !l) { free(vis); free(q); free(byd); free(l); return O_E_NOMEM; }
    for (int64_t v = 0; v < V; ++v) { byd[v].d = row_ptr[v + 1] - row_ptr[v]; byd[v].v = (int32_t)v; }
    qsort(byd, (size_t)V, sizeof(dv), cmp_dv);
    int64_t head = 0, tail = 0, nxt = 0;
    while (tail < V) {
        if (head == tail) {
            while (vis[byd[nxt].v]) ++nxt;
            vis[byd[nxt].v] = 1; q[tail++] = byd[nxt].v;
        }
        int32_t v = q[head++];
        int64_t nl = 0;
        for (int64_t e = row_ptr[v]; e < row_ptr[v + 1]; ++e) {
            int32_t u = col[e];
            if (!vis[u]) { l[nl].d = row_ptr[u + 1] - row_ptr[u]; l[nl].v = u; ++nl; }
        }
        qsort(l, (size_t)nl, sizeof(dv), cmp_dv);
        for (int64_t j = 0; j < nl; ++j) { vis[l[j].v] = 1; q[tail++] = l[j].v; }
    }
    for (int64_t k = 0; k < V; ++k) perm[k] = q[V - 1 - k];
    free(vis); free(q); free(byd); free(l);
    return O_OK;
}
