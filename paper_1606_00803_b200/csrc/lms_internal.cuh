// lms_internal.cuh -- shared internals of liblms.so (the CUDA product path).
// Nothing here is shared with oracle/ (the CPU oracle is independent).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <string>
#include <vector>

#include "../../include/lms.h"

namespace lms {

// ----------------------------------------------------------------- errors
void set_error(const std::string& msg);
void note_launch(int64_t n = 1);

struct Err {
  lms_status st;
  std::string msg;
};

#define LMS_TRY_CUDA(expr)                                                                     \
  do {                                                                                         \
    cudaError_t _e = (expr);                                                                   \
    if (_e != cudaSuccess) {                                                                   \
      throw ::lms::Err{_e == cudaErrorMemoryAllocation ? LMS_E_NOMEM : LMS_E_CUDA,             \
                       std::string(#expr) + ": " + cudaGetErrorString(_e) + " @" + __FILE__ + \
                           ":" + std::to_string(__LINE__)};                                    \
    }                                                                                          \
  } while (0)

#define LMS_CHECK_LAUNCH()                \
  do {                                    \
    ::lms::note_launch();                 \
    LMS_TRY_CUDA(cudaGetLastError());     \
  } while (0)

inline void fail(lms_status st, const std::string& msg) { throw Err{st, msg}; }

// ----------------------------------------------------------------- device buffers
// Scratch allocator (alloc.cu): stream-ordered cudaMallocAsync behind a small
// cache of freed blocks keyed by (stream, size).  A block freed on stream s is
// reused only by a later allocation on the same stream, so the stream order
// that made cudaFreeAsync safe makes the reuse safe too.  Capped by
// LMS_CACHE_GB (default 16; 0 = off); cached blocks go back to the pool
// (cudaFreeAsync) beyond the cap and on lms_cache_release.
void* ws_alloc(size_t bytes, cudaStream_t s);
void ws_free(void* p, cudaStream_t s);

// RAII device buffer allocated stream-ordered on the handle's stream.
template <typename T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
  cudaStream_t s = nullptr;
  DBuf() = default;
  DBuf(size_t count, cudaStream_t st) { alloc(count, st); }
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept : p(o.p), n(o.n), s(o.s) { o.p = nullptr; o.n = 0; }
  DBuf& operator=(DBuf&& o) noexcept {
    // the old buffer is freed in the order of the NEW buffer's stream (the
    // stream of the call that produced the replacement)
    if (this != &o) {
      if (p) ws_free(p, o.s);
      p = o.p; n = o.n; s = o.s; o.p = nullptr; o.n = 0;
    }
    return *this;
  }
  ~DBuf() { release(); }
  void alloc(size_t count, cudaStream_t st) {
    release();
    s = st;
    n = count;
    if (count) p = static_cast<T*>(ws_alloc(count * sizeof(T), st));
  }
  void release() {
    if (p) ws_free(p, s);
    p = nullptr;
    n = 0;
  }
  T* get() const { return p; }
};

// ----------------------------------------------------------------- GZ kernel tables
// per tile: record base, meta base (16-byte units), sizes (gz.cu)
struct __align__(16) GzTile {
  long long rec_base;
  long long meta_base;
  uint32_t meta16, rec16, n_items, n_slots;
  uint32_t R, pad0, pad1, pad2;
};
// shared-memory plan of the GZ kernel (gz.cu plan_layout)
struct GzLayout {
  int NB = 0, NPW = 0, NW = 0;  // region buffers, producer warps, worker warps
  int RR = 0, RR_log2 = 0, rec_bytes = 0, off_rec = 0;  // record ring: batches (power of 2), bytes per record
  int BS = 8, BS_log2 = 3;      // records per batch
  unsigned long long bs_magic = 0;  // ceil(2^40 / BS): claim / BS for claims < 2^24
  int U = 32;                   // updates per item (32 * updates per lane)
  int hdr_bytes = 0;            // per buffer header copy
  int flag_off = 0, cnt_off = 0, coord_off = 0, buf_bytes = 0;  // inside a buffer
  int stage_bytes = 0;          // producer staging (largest meta block)
  int tiles_cap = 0;            // tiles per CTA (table size)
  int off_rcp = 0;              // RN(1/d) table for the division (d <= 32)
  int off_tab = 0, off_stage = 0, off_ring = 0;  // region offsets
  int padbase = 0;              // 2D: first of the 8 pad slots of every region buffer
  int sleep0 = 20, sleep1 = 128;  // dependency-poll back-off (ns), first 64 polls / later
  int hint_rec = 0;             // records TMA'd with an L2 evict_first policy
  int prefetch_claim = 1;       // take the next claim while the current item computes
  int dbg = 0;                  // timing experiments (LMS_GZ_DBG bits; wrong results): 1 no dependency waits, 2 no fence, 4 no region loads
};

// ----------------------------------------------------------------- schedule
// Sweep schedule: free vertices grouped into work items
// (tile k, colour c), tile = T consecutive storage positions; inside an item
// the vertices are in ascending storage index.  Rows are copied in CSR order
// ("colour-sliced CSR"), so each item streams its own rows contiguously.
struct Schedule {
  bool valid = false;
  bool base_valid = false;  // S1/S3 lists built (GZ builds them only on demand)
  int kind = 0;          // LMS_SCHED_S1 or LMS_SCHED_S3 (resolved)
  int tile = 0;          // T
  int lag = 0;           // S3 tile lag L
  int tiling = 0;        // LMS_TILING_STORAGE or LMS_TILING_SPATIAL (resolved)
  int64_t K = 0;         // number of tiles
  int64_t n_free = 0;
  int max_reach = 0;     // max over tiles of (khi - k)
  DBuf<int32_t> item_ptr;   // [K*C + 1] slot offsets, item index = k*C + c
  DBuf<int32_t> sv;         // [n_free] vertex of each slot
  DBuf<int32_t> sptr;       // [n_free + 1] row offsets into scol
  DBuf<int32_t> scol;       // [nnz_free] neighbour ids, CSR order
  DBuf<int32_t> klo, khi;   // [K] tile dependency range (inclusive)
  DBuf<int32_t> tdep_ptr;   // [K+1] per-tile neighbour-tile lists (CSR, self excluded)
  DBuf<int32_t> tdep;
  DBuf<int32_t> prog;       // [K] S3 per-tile completed-chunk counters
  DBuf<int32_t> tpre;       // [K*(C+1)] S3 per-tile chunk prefix over colours
  DBuf<int32_t> iw;         // [K*C] S3 slab width (max row length) of each item
  DBuf<long long> ioff;     // [K*C+1] S3 slab offset (ints) of each item
  DBuf<int32_t> slab;       // S3 slab: per chunk 32 vertex ids + W x 32 neighbour ids
  DBuf<int32_t> irec;       // [K*C*32] S3 128-byte item records (see smooth.cu)
  DBuf<unsigned long long> ticket;  // [1] S3 work counter
  // S2 (s2.cu): the chunks of every colour, colour-major (slab offset, row width)
  DBuf<long long> s2_choff;
  DBuf<int32_t> s2_chw;
  std::vector<int64_t> s2_cstart;  // [C + 1] first chunk of each colour
  DBuf<int32_t> s2d_cv;            // S2 direct: the free vertices sorted by colour (stable)
  std::vector<int64_t> s2d_cstart; // [C + 1] first position of each colour in s2d_cv
  DBuf<int32_t> s2_crange;        // [C * (G + 1)] persistent S2: chunk range of each (colour, CTA)
  int s2_G = 0;                    // persistent S2 CTAs (one per SM, at most K)
  int s2_wmax = 16;                // widest item row count (S2 ring slot size)
  DBuf<int32_t> s2_nbptr, s2_nb;  // persistent S2: CTA neighbour lists (CSR over CTAs)
  DBuf<unsigned> s2_prog;          // [G] persistent S2: passes published per CTA
  // GZ (ghost-zone tiled sweep, gz.cu): per tile a region = owned free vertices
  // plus every vertex within C*P hops; a persistent kernel stages regions in
  // shared memory and runs P whole sweeps there, reading X and writing the
  // owned vertices to X'.
  int gz_P = 0;             // sweeps per pass
  int gz_upl = 1;           // updates per lane (item = 32 * gz_upl updates)
  int64_t gz_K = 0;         // tiles of the spatial tiling
  int gz_T = 0;             // target owned vertices per tile
  int gz_smem = 0;          // dynamic shared memory per CTA (bytes)
  int gz_threads = 0;       // threads per CTA
  int gz_cps = 1;           // persistent CTAs per SM
  GzLayout gz_L;            // shared-memory plan of the kernel
  int64_t gz_nreg = 0;      // sum of region sizes
  int64_t gz_nupd = 0;      // sum over tiles of first-sweep updates
  int64_t gz_items = 0;     // work items (32 updates of one stage of one tile)
  int64_t gz_bytes = 0;     // schedule bytes (records + meta)
  bool gz_row8 = false;     // records carry 8-bit row codes (relative to the vertex's slot; see gz.cu)
  int gz_max_reg = 0;       // largest region
  int64_t gz_ntiles = 0;    // non-empty tiles
  DBuf<int32_t> gz_tiles;   // [gz_ntiles] non-empty tile ids, ascending
  DBuf<GzTile> gz_tab;      // [K] per-tile table
  DBuf<int32_t> gz_item_sweep;  // [K*(P+1)] first item of each sweep, per tile
  DBuf<uint4> gz_meta;      // per tile: header + region ids
  DBuf<uint4> gz_rec;       // per item: rows, slots/flags/deps, ids, descriptor
  // S1 CUDA graphs: [0] one sweep, [1] eight sweeps (C kernel nodes per sweep)
  cudaGraphExec_t graphs[2] = {nullptr, nullptr};
  ~Schedule() {
    for (auto& g : graphs)
      if (g) cudaGraphExecDestroy(g);
  }
};

}  // namespace lms

struct lms_mesh_s {
  int dim = 2;
  int k = 0;              // verts per element (0 = no elements)
  int64_t V = 0, nnz = 0, n_el = 0, n_free = 0;
  int32_t C = 0;
  int device = 0;
  cudaStream_t s0 = nullptr;   // stream used for allocations
  lms::DBuf<double> x[3];
  lms::DBuf<double> xalt[3];   // second coordinate buffer of the GZ sweep (ping-pong)
  // 2D GZ sweeps run on interleaved (x, y) pairs: xy[xy_cur] is a double2[V]
  // copy, xy[1 - xy_cur] its ping-pong partner.  aos_state says which copy
  // is current: 0 = SoA x[] only, 1 = xy only (x[] stale), 2 = both.
  lms::DBuf<double> xy[2];
  int xy_cur = 0;
  int aos_state = 0;
  int64_t coord_gen = 1;       // bumped whenever x is (re)written outside a sweep
  int64_t alt_gen = 0;         // coord_gen at which xalt's fixed vertices were synced
  lms::DBuf<uint8_t> fixed;
  lms::DBuf<int32_t> row_ptr, col;
  lms::DBuf<int8_t> colour;
  lms::DBuf<int32_t> orig_id;
  lms::DBuf<int32_t> elems;
  lms::DBuf<double> quality;   // valid if has_quality
  // vertex -> element incidence (ascending element id per vertex) for the
  // per-sweep global quality (quality.cu); dropped when the mesh is relabelled
  lms::DBuf<int32_t> v2e_ptr, v2e;
  bool v2e_valid = false;
  bool has_quality = false;    // m->quality holds the INITIAL qualities (RDR input)
  bool quality_external = false;
  bool coords_moved = false;   // coordinates changed since the build (smooth / import)
  int sched_req = LMS_SCHED_AUTO, tile_req = 0, lag_req = 0, tiling_req = LMS_TILING_AUTO;
  lms::Schedule sched;
  lms::DBuf<int> err;          // device error flag
  bool async_errors = false;   // lms_set_async_errors: smooth leaves the flag to lms_check
};

namespace lms {

// Makes the handle's device current for the scope of an API call (and
// restores the caller's): buffers, pools and streams belong to m->device.
struct DevGuard {
  int prev = -1;
  explicit DevGuard(const lms_mesh_s* m) {
    if (!m) return;
    if (cudaGetDevice(&prev) != cudaSuccess) { prev = -1; return; }
    if (prev == m->device) prev = -1;
    else cudaSetDevice(m->device);
  }
  ~DevGuard() { if (prev >= 0) cudaSetDevice(prev); }
};

// Device-side error flag helpers (error codes are lms_status values).
__device__ __forceinline__ void raise_err(int* flag, int code) { atomicCAS(flag, 0, code); }
void check_err_flag(lms_mesh_s* m, cudaStream_t s, const char* what);

inline unsigned grid_for(int64_t n, int block) {
  int64_t g = (n + block - 1) / block;
  if (g < 1) g = 1;
  if (g > (int64_t)1 << 30) g = (int64_t)1 << 30;
  return (unsigned)g;
}

// Pipeline pieces (implemented in build.cu, colour.cu, order.cu, permute.cu, smooth.cu)
void build_csr_from_elems(lms_mesh_s* m, const int32_t* d_elems, bool want_boundary, cudaStream_t s);
void compute_colouring(lms_mesh_s* m, cudaStream_t s);
// q_v of the CURRENT coordinates into out[V] (A4)
void compute_quality(lms_mesh_s* m, double* out, cudaStream_t s);
// the initial qualities RDR orders by (reading Z13), cached in m->quality
const double* initial_quality(lms_mesh_s* m, cudaStream_t s);
void order_random(lms_mesh_s* m, uint64_t seed, int32_t* d_perm, cudaStream_t s);
void order_bfs(lms_mesh_s* m, int64_t seed, int32_t* d_perm, cudaStream_t s);
void order_rbfs(lms_mesh_s* m, int64_t seed, bool rcm, int32_t* d_perm, cudaStream_t s);
void order_dfs(lms_mesh_s* m, int64_t seed, int32_t* d_perm, cudaStream_t s);
void order_rdr(lms_mesh_s* m, int32_t* d_perm, cudaStream_t s, int64_t L = 0);
void permute_mesh(lms_mesh_s* m, const int32_t* d_perm, cudaStream_t s);
void build_schedule(lms_mesh_s* m, cudaStream_t s);
int64_t spatial_tiles(lms_mesh_s* m, int T, int32_t* tile_of, cudaStream_t s);
bool build_gz(lms_mesh_s* m, int T, int P, bool required, cudaStream_t s);  // gz.cu
void run_gz(lms_mesh_s* m, int sweeps, cudaStream_t s);                     // gz.cu
void run_jacobi(lms_mesh_s* m, int sweeps, cudaStream_t s);                 // jacobi.cu
void run_s2(lms_mesh_s* m, int sweeps, cudaStream_t s);                     // s2.cu
void halo_pack(lms_mesh_s* m, const int32_t* idx, int64_t n, double* out, cudaStream_t s);        // halo.cu
void halo_unpack(lms_mesh_s* m, const int32_t* idx, int64_t n, const double* in, cudaStream_t s);  // halo.cu
void sync_soa(lms_mesh_s* m, cudaStream_t s);   // make x[] current (gz.cu)
void soa_changed(lms_mesh_s* m);                // x[] was written outside a sweep
void run_sweeps(lms_mesh_s* m, int sweeps, cudaStream_t s);
void segmented_sort_rows(int32_t* d_col, const int32_t* d_row_ptr, int64_t V, int64_t nnz, cudaStream_t s);
int64_t count_free(lms_mesh_s* m, cudaStream_t s);
void fill_iota(int32_t* p, int64_t n, cudaStream_t s);

}  // namespace lms
