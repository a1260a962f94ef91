/*
 * lms.h -- C ABI of liblms.so, the B200 (sm_100a) implementation of the
 * data-parallel hot path of Aupy, Park & Raghavan, "Locality-Aware Laplacian
 * Mesh Smoothing" (arXiv 1606.00803).  PAPER.md lines are cited as P:<n>.
 *
 * The path: build the vertex-adjacency CSR of a triangle/tetrahedral mesh,
 * compute a vertex ordering (random, original, BFS, or the paper's RDR,
 * Alg. 2), relabel the mesh by it, and run Laplacian smoothing sweeps
 * (Eq. 1) with a fixed vertex-colouring Gauss-Seidel schedule.
 *
 * Conventions (all entry points):
 *  - Pointers named d_* are DEVICE pointers (cudaMalloc / torch CUDA tensors)
 *    on the current CUDA device; the caller owns them.  They are read (or
 *    written, for outputs) during the call and never retained.
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *    Work is enqueued on it; calls that must inspect device results (sizes,
 *    validation flags) synchronise it before returning.
 *  - Coordinates are structure-of-arrays fp64: d_coords is a HOST array of
 *    `dim` device pointers, each to double[n_vertices].
 *  - Indices are int32 (meshes with fewer than 2^31 vertices and 2^31 CSR
 *    entries); elements are element-major int32[n_elems][verts_per_elem].
 *  - Every function returns an lms_status; on a non-OK status,
 *    lms_last_error() returns a message (thread-local) and the mesh handle is
 *    left unchanged (lms_permute validates before it mutates).
 *  - A handle must not be used by two threads at once; distinct handles are
 *    independent.  The handle owns all derived device memory.
 */
#ifndef LMS_H
#define LMS_H

#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct lms_mesh_s* lms_mesh_t;
typedef void* lms_stream_t; /* cudaStream_t */

typedef enum {
    LMS_OK = 0,
    LMS_E_ARG = -1,        /* bad argument: dim not in {2,3}, k not in {3,4}, sweeps < 0, unknown kind,
                              BFS seed vertex out of range, NULL pointer, size overflow */
    LMS_E_INDEX = -2,      /* element index out of [0, V), or a repeated vertex within one element */
    LMS_E_ISOLATED = -3,   /* a vertex with no neighbour (deg 0) */
    LMS_E_PERM = -4,       /* perm is not a bijection of [0, V) */
    LMS_E_DEGENERATE = -5, /* element whose vertices all coincide (quality undefined) */
    LMS_E_NOMEM = -6,      /* device allocation failed */
    LMS_E_CUDA = -7,       /* CUDA runtime error (message in lms_last_error) */
    LMS_E_NCCL = -8,       /* NCCL failure or NCCL unavailable (multi-GPU calls) */
    LMS_E_STATE = -9       /* handle not in a state that allows the call (e.g. RDR without quality) */
} lms_status;

typedef enum {
    LMS_ORDER_ORIGINAL = 0, /* identity: the generator / Triangle order */
    LMS_ORDER_RANDOM = 1,   /* random storage order: argsort of H(seed, 4, i) */
    LMS_ORDER_BFS = 2,      /* breadth-first order, Strout-Hovland */
    LMS_ORDER_RDR = 3,      /* Reuse-Distance-Reducing order, Alg. 2 */
    /* more orderings for the study */
    LMS_ORDER_RBFS = 4,     /* reverse BFS: the BFS order reversed; `seed` = BFS seed */
    LMS_ORDER_RCM = 5,      /* reverse Cuthill-McKee: queue BFS from the vertex of smallest (degree, label),
                               children by (degree, label), restarts likewise; reversed (reading Z26) */
    LMS_ORDER_DFS = 6,      /* depth-first preorder (Fig. 2a): smallest unvisited neighbour
                               first, restart at the smallest unvisited label (reading Z25); one warp,
                               sequential; `seed` = start vertex */
    LMS_ORDER_RDR_WINDOWED = 7 /* APPROXIMATION of RDR (reading Z28): the labels cut into
                               windows [wL, (w+1)L), L = `seed` (0: 65536); Alg. 2 on each window's induced
                               subgraph (edges leaving it dropped), window w's order in perm[wL, ...);
                               the windows walk in parallel, one warp each.  L >= V is RDR itself.
                               LMS_E_ARG if L > INT32_MAX or the maximum degree exceeds 32 */
} lms_order_kind;

typedef enum {
    LMS_SCHED_AUTO = 0,     /* pick per mesh: GZ for 2D meshes with <= 8 colours, else S1 */
    LMS_SCHED_S1 = 1,       /* one launch per colour (CUDA-graph captured sweep) */
    LMS_SCHED_S2 = 2,       /* 3D only: one launch per colour over interleaved (x, y, z, 0) coordinates --
                               one 32-byte sector per neighbour (256-bit loads) -- and the coalesced
                               column-major CSR slab; LMS_E_ARG on a 2D mesh */
    LMS_SCHED_S3 = 3,       /* persistent colour-pipelined sweep with per-tile progress flags */
    LMS_SCHED_GZ = 4,       /* ghost-zone tiled sweep: one launch per P sweeps; each CTA stages a
                               spatial tile plus every vertex within C*P hops in shared memory,
                               runs the P sweeps' colour stages there and writes its owned vertices
                               to a second coordinate buffer (no inter-CTA synchronisation) */
    LMS_SCHED_JACOBI = 5    /* N3 VARIANT, not the colour-GS result: every free vertex moves to the mean
                               of its neighbours' PREVIOUS-sweep coordinates (Eq. 1,
                               CSR-order sums, IEEE division), double-buffered; for convergence studies */
} lms_schedule_kind;

/* ---------------------------------------------------------------------------
 * lms_build_csr -- build a mesh handle from elements.
 *  Computes, on the GPU:
 *   - the vertex adjacency N(v) = {u != v : u, v share an element}, rows
 *     ascending ("N neighbored vertices", Eq. 1);
 *   - the fixed mask: if d_fixed is NULL, a vertex is fixed iff it lies on an
 *     edge (triangles) / face (tetrahedra) that belongs to exactly one element
 *     (Alg. 1 smooths "interior vertices"); else the caller's mask
 *     (1 = fixed) is copied;
 *   - orig_id = input label, and the colouring schedule: greedy first-fit
 *     over free vertices in ascending orig_id (reading Z2).
 *  dim: 2 or 3; verts_per_elem: 3 (triangles) or 4 (tetrahedra).
 *  d_coords: host array of dim device pointers, double[n_vertices] each.
 *  d_elems: int32[n_elems * verts_per_elem].  d_fixed: uint8[n_vertices] or NULL.
 *  Errors: LMS_E_ARG, LMS_E_INDEX (out-of-range or repeated vertex in an
 *  element), LMS_E_ISOLATED, LMS_E_NOMEM, LMS_E_CUDA.  *out is set only on OK.
 *  The elements are copied into the handle (needed for quality / RDR).
 */
lms_status lms_build_csr(int32_t dim, int64_t n_vertices, const double* const* d_coords,
                         int32_t verts_per_elem, int64_t n_elems, const int32_t* d_elems,
                         const uint8_t* d_fixed, lms_stream_t stream, lms_mesh_t* out);

/* lms_build_csr_host -- lms_build_csr from HOST buffers, with the upload
 *  pipelined (the end-to-end ingest path).  Same arguments and results as
 *  lms_build_csr, except:
 *  h_coords: host array of dim HOST pointers, double[n_vertices] each;
 *  h_elems: host int32[n_elems * verts_per_elem]; h_fixed: host uint8[V] or NULL.
 *  The elements (and mask) are copied to the device on `stream`; the
 *  coordinates on a library-owned side stream, overlapping the CSR build and
 *  the colouring, which do not read them.  `stream` waits for that upload
 *  before the call returns its work, so later calls on `stream` see the
 *  coordinates.  For the copies to overlap, the host buffers must be
 *  page-locked (cudaHostAlloc / torch pin_memory); pageable buffers give the
 *  same result without overlap.  The host buffers must stay valid and
 *  unmodified until `stream` has passed this call's work (the copies are
 *  asynchronous).  Errors as lms_build_csr. */
lms_status lms_build_csr_host(int32_t dim, int64_t n_vertices, const double* const* h_coords,
                              int32_t verts_per_elem, int64_t n_elems, const int32_t* h_elems,
                              const uint8_t* h_fixed, lms_stream_t stream, lms_mesh_t* out);

/* lms_mesh_from_csr -- build a handle from a ready CSR (test/debug entry).
 *  d_row_ptr int32[V+1], d_col_idx int32[nnz] (rows ascending, symmetric, no
 *  self loops -- not re-validated beyond index range and deg >= 1).
 *  d_fixed uint8[V] (required).  d_orig_id int32[V] or NULL (= identity).
 *  d_colour int8[V] or NULL (= computed from orig_id as in lms_build_csr);
 *  fixed vertices must carry colour -1.  d_quality double[V] or NULL (RDR then
 *  needs it: without elements there is no quality).  Errors as lms_build_csr. */
lms_status lms_mesh_from_csr(int32_t dim, int64_t n_vertices, const double* const* d_coords,
                             const uint8_t* d_fixed, const int32_t* d_row_ptr, const int32_t* d_col_idx,
                             const int32_t* d_orig_id, const int8_t* d_colour, const double* d_quality,
                             lms_stream_t stream, lms_mesh_t* out);

void lms_mesh_destroy(lms_mesh_t m);

/* ---------------------------------------------------------------------------
 * lms_order -- compute a vertex ordering of the mesh in its CURRENT labels
 * (SURVEY 8(a) A6).  d_perm (out): int32[V], perm[new] = old (P:420,
 * "V_new[next_num] <- V[i]").
 *  ORIGINAL: identity.  RANDOM: indices sorted by H(seed, 4, i) (SplitMix64
 *  counter hash, reading Z15).  BFS: queue BFS from vertex `seed`,
 *  neighbours in ascending label, restart at the smallest unvisited label
 *  (reading Z14); LMS_E_ARG if seed >= V.  RDR: Alg. 2 over the
 *  initial vertex qualities (edge-length ratio) with ties broken
 *  by label, l[0] = lowest-(quality,label) unprocessed neighbour, fixed
 *  vertices allowed inside walks, never-reached vertices appended in
 *  ascending label (readings Z9-Z13); `seed` unused.  RDR computes the
 *  quality from the stored elements (LMS_E_DEGENERATE on a degenerate one)
 *  or uses the quality given to lms_mesh_from_csr (else LMS_E_STATE).
 */
lms_status lms_order(lms_mesh_t m, lms_order_kind kind, uint64_t seed, int32_t* d_perm,
                     lms_stream_t stream);

/* lms_permute -- relabel the mesh in place by d_perm (int32[V], perm[new]=old)
 * (SURVEY 8(a) A7): coordinates, fixed, colour, orig_id and quality are
 * gathered (X'[k] = X[perm[k]]), elements remapped through inv (element and
 * slot order kept), CSR rows remapped and re-sorted ascending.  The colour
 * moves with its vertex, so lms_smooth's result is ordering-independent up to
 * the rounding of the neighbour sums.  LMS_E_PERM if not a bijection
 * (checked before anything is modified). */
lms_status lms_permute(lms_mesh_t m, const int32_t* d_perm, lms_stream_t stream);

/* lms_smooth -- run exactly `sweeps` LMS sweeps in place.
 * One sweep = for c in 0..C-1: every free vertex v of colour c moves to
 * (sum of its neighbours' coordinates, in CSR order) / deg(v), per axis, with
 * IEEE binary64 round-to-nearest adds and division and no FMA (Eq. 1,
 * P:244-251, inside Alg. 1's loop over interior vertices, under
 * the colour-ordered Gauss-Seidel schedule of DESIGN.md reading Z1).  Fixed
 * vertices never move.  sweeps == 0 is a no-op; sweeps < 0 -> LMS_E_ARG.
 * The schedule (S1/S3/GZ) is chosen by lms_set_schedule; all are bit-identical.
 * LMS_SCHED_JACOBI instead runs the named Jacobi variant (a different method). */
lms_status lms_smooth(lms_mesh_t m, int32_t sweeps, lms_stream_t stream);

/* lms_set_async_errors -- on != 0: lms_smooth returns once its sweeps are
 * enqueued on `stream`, without waiting for them; a sweep kernel's watchdog
 * abort (LMS_E_CUDA, the coordinates then partly updated) is reported by the
 * next lms_check on the handle instead.  Lets a caller keep several jobs in
 * flight on several streams (one job's copies overlapping another's
 * kernels).  Default off: lms_smooth synchronises `stream` and reports it. */
lms_status lms_set_async_errors(lms_mesh_t m, int32_t on);

/* lms_check -- synchronise `stream` and report (and clear) a device-side
 * error recorded on the handle since the last check: LMS_OK or the error. */
lms_status lms_check(lms_mesh_t m, lms_stream_t stream);

/* lms_set_schedule -- choose the sweep kernel.  tile: vertices per tile
 * (0 = default); lag: S3 tile lag L (0 = automatic); for LMS_SCHED_GZ `lag` is
 * the number of sweeps P fused into one pass (0 = 1; at most 8).  Takes effect
 * at the next lms_smooth (the internal schedule is rebuilt lazily).  GZ
 * returns LMS_E_STATE from lms_smooth if no tile size makes a region fit in
 * shared memory. */
lms_status lms_set_schedule(lms_mesh_t m, lms_schedule_kind kind, int32_t tile, int32_t lag);

typedef enum {
    LMS_TILING_AUTO = 0,    /* S3: SPATIAL, S1: STORAGE */
    LMS_TILING_STORAGE = 1, /* tile = T consecutive storage positions (processing follows the ordering) */
    LMS_TILING_SPATIAL = 2  /* tile = cell of a regular grid over the initial coordinates (~T vertices) */
} lms_tiling_kind;

/* lms_set_tiling -- how the schedule groups free vertices into work items.
 * A scheduling choice only: every tiling replays the same colour schedule, so
 * lms_smooth's result is bit-identical for all of them. */
lms_status lms_set_tiling(lms_mesh_t m, lms_tiling_kind kind);

/* ---------------------------------------------------------------------------
 * Accessors.  Outputs are caller-owned device buffers of the stated sizes.   */
lms_status lms_mesh_info(lms_mesh_t m, int64_t* n_vertices, int64_t* nnz, int32_t* n_colours,
                         int32_t* dim);
/* n_free: free (non-fixed) vertices; sched_kind: the kernel the next lms_smooth
 * uses (resolved AUTO); tile/lag: its parameters (0 before the first smooth). */
lms_status lms_schedule_info(lms_mesh_t m, int64_t* n_free, int32_t* sched_kind, int32_t* tile,
                             int32_t* lag);
/* tiling: resolved lms_tiling_kind; n_tiles: tiles K; max_reach: max |k' - k| over
 * dependent tiles (S3 needs lag > max_reach) -- all 0 before the first smooth. */
lms_status lms_schedule_info2(lms_mesh_t m, int32_t* tiling, int64_t* n_tiles, int32_t* max_reach);
lms_status lms_export_coords(lms_mesh_t m, double* const* d_out, lms_stream_t stream);
lms_status lms_import_coords(lms_mesh_t m, const double* const* d_in, lms_stream_t stream);
lms_status lms_export_csr(lms_mesh_t m, int32_t* d_row_ptr, int32_t* d_col_idx, lms_stream_t stream);
lms_status lms_export_colour(lms_mesh_t m, int8_t* d_colour, lms_stream_t stream);
lms_status lms_export_fixed(lms_mesh_t m, uint8_t* d_fixed, lms_stream_t stream);
lms_status lms_export_orig_id(lms_mesh_t m, int32_t* d_orig_id, lms_stream_t stream);
/* d_elems int32[n_elems * k]; LMS_E_STATE if the handle has no elements. */
lms_status lms_export_elems(lms_mesh_t m, int32_t* d_elems, lms_stream_t stream);
/* Vertex quality q_v (mean edge-length ratio of attached
 * elements), computed from the current coordinates (A4). */
lms_status lms_export_quality(lms_mesh_t m, double* d_quality, lms_stream_t stream);

/* ---------------------------------------------------------------------------
 * Multi-GPU building blocks (driven by paper_1606_00803_b200/dist.py
 * with NCCL over NVLink between the pack and the unpack).
 *  lms_smooth_colour: one colour stage of the sweep (every free vertex of colour
 *    `colour` moves, Eq. 1) -- a sweep is the stages 0..C-1 in order.
 *  lms_gather_coords: d_out[a*n + i] = x_a[d_idx[i]] (halo pack), d_out double[dim*n].
 *  lms_scatter_coords: x_a[d_idx[i]] = d_in[a*n + i] (halo unpack).
 *  d_idx int32[n] local vertex ids (not validated). */
lms_status lms_smooth_colour(lms_mesh_t m, int32_t colour, lms_stream_t stream);
lms_status lms_gather_coords(lms_mesh_t m, const int32_t* d_idx, int64_t n, double* d_out, lms_stream_t stream);
lms_status lms_scatter_coords(lms_mesh_t m, const int32_t* d_idx, int64_t n, const double* d_in,
                              lms_stream_t stream);

/* ---------------------------------------------------------------------------
 * Convergence-driven LMS: Alg. 1's outer loop.
 *
 * lms_global_quality -- Global_quality of the CURRENT coordinates (Alg. 1 lines
 *  4-8): q_e = edge-length ratio of each element, q_v =
 *  mean of q_e over the elements containing v in ascending element order
 *  (P:234-236), Global_quality = RN(exact sum of q_v) / |V| -- the vertex sum
 *  is exact and rounded once (reading Z24), so it does not depend on
 *  the storage order.  *h_quality (host) receives it; d_vertex_quality
 *  (device double[V], or NULL) receives q_v.  Synchronises `stream`.  Needs
 *  elements (LMS_E_STATE for a CSR-only handle); LMS_E_DEGENERATE on an
 *  element with all edge lengths zero.  The vertex -> element incidence is
 *  built on first use and kept until the mesh is relabelled.
 *
 * lms_smooth_until -- the loop, with the paper's stopping rule and
 *  an iteration cap:
 *      Q[0] = Global_quality;  k = 0
 *      loop: if Q[k] >= goal: stop (LMS_STOP_GOAL)
 *            if k == max_sweeps: stop (LMS_STOP_MAX)
 *            one sweep of the current schedule (lms_smooth(m, 1)); k += 1
 *            Q[k] = Global_quality
 *            if Q[k] - Q[k-1] < eps: stop (LMS_STOP_CONVERGED)
 *  *sweeps_run = k; h_quality_history (host double[max_sweeps + 1], or NULL)
 *  receives Q[0..k]; *stop_reason one of lms_stop_reason.  One host
 *  synchronisation per sweep (the stop decision is taken on the host, on the
 *  same value the oracle computes).  Errors as lms_smooth / lms_global_quality;
 *  max_sweeps < 0 -> LMS_E_ARG. */
typedef enum { LMS_STOP_GOAL = 1, LMS_STOP_CONVERGED = 2, LMS_STOP_MAX = 3 } lms_stop_reason;
lms_status lms_global_quality(lms_mesh_t m, double* h_quality, double* d_vertex_quality, lms_stream_t stream);
lms_status lms_smooth_until(lms_mesh_t m, double goal, double eps, int32_t max_sweeps, int32_t* sweeps_run,
                            double* h_quality_history, int32_t* stop_reason, lms_stream_t stream);

/* ---------------------------------------------------------------------------
 * Multi-GPU sweep: one process per GPU, one rank each.
 *
 * Partition (the paper's "static ... evenly dividing the vertices";
 * DESIGN.md reading Z22): the mesh AS RELABELLED is split into `nranks`
 * contiguous label ranges [first, first + count) with ceil(n_free / nranks)
 * free vertices each; rank r owns range r.  Each rank keeps every vertex
 * within D = C * sweeps_per_exchange hops (through free vertices) of its
 * range, in ascending label (so every row keeps its CSR order), and the
 * library-owned NCCL communicator refreshes the ghost values once per pass
 * of sweeps_per_exchange sweeps; the rank then runs the pass on its local
 * mesh (GZ in 2D).  The owned coordinates are bit-identical to lms_smooth on
 * one GPU.
 *
 * lms_nccl_unique_id -- ncclGetUniqueId into out[128] (call on rank 0 and
 *  broadcast the bytes, e.g. over torch.distributed).  LMS_E_NCCL if NCCL
 *  (libnccl.so.2, bound at run time) is unavailable.
 * lms_dist_create -- every rank calls it with its handle of the SAME mesh
 *  (built and relabelled identically on every rank), its rank, nranks and the
 *  shared uid; collective (ncclCommInitRank, then the ghost lists go to their
 *  owners).  Builds the rank's plan on its GPU from its own range only:
 *  O(V) memsets and one O(V) scan, O(V/P + halo) otherwise.  `m` is only read:
 *  it may be destroyed afterwards.  sweeps_per_exchange in [1, 8]; tile = the
 *  local GZ tile (0 = default).  *out is a new handle (lms_dist_destroy).
 * lms_dist_replan -- a new mesh (same rank / nranks, every rank calls it)
 *  on the handle's existing communicator: the plan is rebuilt as in
 *  lms_dist_create, without a new ncclCommInitRank (communicator set-up is a
 *  once-per-job cost).  The previous plan and local mesh are released.
 * lms_smooth_dist -- `sweeps` colour-GS sweeps (Eq. 1): per pass
 *  of up to sweeps_per_exchange sweeps, pack -> grouped ncclSend/ncclRecv
 *  on `stream` -> unpack, then the local pass.  Collective: every rank calls
 *  it with the same `sweeps`.
 * lms_dist_export_owned -- the owned coordinates into d_out (host array of dim
 *  device pointers, double[count] each; NULL = sizes only): *first = first
 *  owned label, *count = number of owned labels.
 * lms_dist_info -- local vertices, ghost values sent / received per pass
 *  (vertices), peers exchanged with, ghost-zone depth D.
 * lms_dist_export_local_ids -- the labels of the rank's local vertices
 *  (int32[n_local], ascending).
 * lms_dist_create_local / lms_smooth_dist_local -- the same plans for all
 *  nranks ranks in ONE process on one device, exchanged by device copies
 *  (testing the partition without NCCL; the ranks are stepped in turn and no
 *  kernel waits on another rank).  outs: lms_dist_t[nranks], in rank order.
 * Errors: LMS_E_ARG (bad rank / nranks / sweeps), LMS_E_NCCL, LMS_E_CUDA,
 *  LMS_E_NOMEM, LMS_E_STATE (inconsistent peers). */
typedef struct lms_dist_s* lms_dist_t;
lms_status lms_nccl_unique_id(uint8_t out[128]);
lms_status lms_dist_create(lms_mesh_t m, int32_t rank, int32_t nranks, const uint8_t nccl_uid[128],
                           int32_t sweeps_per_exchange, int32_t tile, lms_stream_t stream, lms_dist_t* out);
lms_status lms_dist_replan(lms_dist_t d, lms_mesh_t m, int32_t tile, lms_stream_t stream);
lms_status lms_smooth_dist(lms_dist_t d, int32_t sweeps, lms_stream_t stream);
lms_status lms_dist_export_owned(lms_dist_t d, double* const* d_out, int64_t* first, int64_t* count,
                                 lms_stream_t stream);
lms_status lms_dist_info(lms_dist_t d, int64_t* n_local, int64_t* n_send, int64_t* n_recv, int32_t* n_peers,
                         int32_t* depth);
lms_status lms_dist_export_local_ids(lms_dist_t d, int32_t* d_ids, lms_stream_t stream);
lms_status lms_dist_create_local(lms_mesh_t m, int32_t nranks, int32_t sweeps_per_exchange, int32_t tile,
                                 lms_stream_t stream, lms_dist_t* outs);
lms_status lms_smooth_dist_local(lms_dist_t* ds, int32_t nranks, int32_t sweeps, lms_stream_t stream);
void lms_dist_destroy(lms_dist_t d);

/* ---------------------------------------------------------------------------
 * The paper's reuse-distance instrument (Fig. 1
 * P:64-69, Table III, Eq. 2).
 *
 * lms_trace -- the canonical access trace of ONE sequential sweep of the mesh
 *  in its current storage order (Alg. 1's loop over interior vertices,
 *  P:211-214; SPEC trace_iteration): for each free vertex v in storage order:
 *  v, its neighbours in CSR order, v again (the write of Eq. 1).  Elements are
 *  vertex labels.  d_trace: int32[*n_out] device buffer, or NULL to query the
 *  length only (*n_out = sum over free v of deg(v) + 2).  Synchronises.
 * lms_reuse_distance -- d_dist[t] (int64, device) = the number of DISTINCT
 *  elements accessed between access t and the previous access to the same
 *  element, -1 if t is the element's first access (COLD).
 *  d_trace int32[n] with identifiers in [0, n_ids) (else LMS_E_INDEX);
 *  n < 2^31.  Exact (a wavelet matrix of previous-access times on the GPU).
 *  Synchronises.
 * lms_reuse_stats -- over the finite distances of d_dist[n]: for each of the
 *  nq proportions h_q[k] in (0, 1], h_quantile[k] = the smallest value v with
 *  at least a proportion h_q[k] of the distances <= v; *h_mean =
 *  their mean; *h_n_cold = the number of -1 entries; for each of the ncap
 *  capacities h_capacity[k], h_n_ge[k] = the number of distances >= it (the
 *  model's reuse misses for a cache holding that many elements).  Host
 *  outputs; NULL outputs are skipped.  LMS_E_STATE if quantiles or counts are
 *  asked of a trace with no finite distance.  Synchronises. */
lms_status lms_trace(lms_mesh_t m, int32_t* d_trace, int64_t* n_out, lms_stream_t stream);
lms_status lms_reuse_distance(const int32_t* d_trace, int64_t n, int64_t n_ids, int64_t* d_dist,
                              lms_stream_t stream);
lms_status lms_reuse_stats(const int64_t* d_dist, int64_t n, const double* h_q, int32_t nq, int64_t* h_quantile,
                           double* h_mean, int64_t* h_n_cold, const int64_t* h_capacity, int32_t ncap,
                           int64_t* h_n_ge, lms_stream_t stream);

/* Thread-local message for the last non-OK status of this thread. */
const char* lms_last_error(void);
/* Number of CUDA kernels this library launched on this thread since load
 * (used by bench.py for its gpu_launches claim). */
int64_t lms_kernel_launches(void);
/* Return the library's cached scratch blocks to the CUDA memory pool.
 * Every call's temporaries are freed stream-ordered into a host-side cache
 * keyed by (stream, size) and reused by later allocations on the same
 * stream; the cache holds at most LMS_CACHE_GB (environment, default a quarter
 * of the device memory;
 * 0 disables it).  Call this to hand that memory back, for example before
 * destroying a stream the library was used on; the blocks are freed in each
 * owning stream's order.  Never fails. */
void lms_cache_release(void);
/* Route the library's device allocations (mesh buffers and every call's
 * temporaries) through a caller's allocator, e.g. the torch caching
 * allocator; (NULL, NULL) restores the default (cudaMallocAsync behind the
 * scratch cache above).  alloc(bytes, stream, ctx) returns device memory
 * usable in `stream` order (NULL = out of memory -> LMS_E_NOMEM); free(p,
 * stream, ctx) is called in the order of the stream that last used p.
 * Blocks keep the allocator that made them: switch only when no handle is
 * alive.  LMS_E_ARG if exactly one of alloc / free is NULL.  Not
 * thread-safe against concurrent library calls. */
lms_status lms_set_allocator(void* (*alloc)(size_t bytes, lms_stream_t stream, void* ctx),
                             void (*free_fn)(void* p, lms_stream_t stream, void* ctx), void* ctx);

#ifdef __cplusplus
}
#endif
#endif /* LMS_H */
