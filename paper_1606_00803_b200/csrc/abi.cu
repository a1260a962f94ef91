// abi.cu -- the extern "C" entry points declared in include/lms.h.
// Validation, handle lifetime, error reporting; the work is in the other .cu files.
#include <atomic>
#include <map>
#include <mutex>
#include <cstring>

#include <chrono>
#include <cstdio>

#include "lms_internal.cuh"

namespace lms {

static thread_local std::string g_err;
static thread_local int64_t g_launches = 0;

void set_error(const std::string& msg) { g_err = msg; }
void note_launch(int64_t n) { g_launches += n; }

__global__ void k_count_nonfixed(const uint8_t* fixed, int64_t V, unsigned long long* out) {
  unsigned long long c = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < V; i += (int64_t)gridDim.x * blockDim.x)
    c += fixed[i] ? 0 : 1;
  for (int o = 16; o; o >>= 1) c += __shfl_down_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, c);
}

int64_t count_free(lms_mesh_s* m, cudaStream_t s) {
  DBuf<unsigned long long> d(1, s);
  LMS_TRY_CUDA(cudaMemsetAsync(d.p, 0, sizeof(unsigned long long), s));
  k_count_nonfixed<<<grid_for(m->V, 256) > 1184 ? 1184 : grid_for(m->V, 256), 256, 0, s>>>(m->fixed.p, m->V, d.p);
  LMS_CHECK_LAUNCH();
  unsigned long long h = 0;
  LMS_TRY_CUDA(cudaMemcpyAsync(&h, d.p, sizeof(h), cudaMemcpyDeviceToHost, s));
  LMS_TRY_CUDA(cudaStreamSynchronize(s));
  return (int64_t)h;
}

void check_err_flag(lms_mesh_s* m, cudaStream_t s, const char* what) {
  int h = 0;
  LMS_TRY_CUDA(cudaMemcpyAsync(&h, m->err.p, sizeof(int), cudaMemcpyDeviceToHost, s));
  LMS_TRY_CUDA(cudaStreamSynchronize(s));
  if (h != 0) {
    LMS_TRY_CUDA(cudaMemsetAsync(m->err.p, 0, sizeof(int), s));
    const char* why = h == LMS_E_INDEX ? "element index out of range or repeated vertex in an element"
                    : h == LMS_E_ISOLATED ? "isolated vertex (no neighbour)"
                    : h == LMS_E_PERM ? "perm is not a bijection"
                    : h == LMS_E_DEGENERATE ? "degenerate element (all edge lengths zero)"
                    : h == LMS_E_ARG ? "invalid argument detected on device" : "device error";
    fail((lms_status)h, std::string(what) + ": " + why);
  }
}

static lms_status handle_exc(const Err& e) {
  set_error(e.msg);
  return e.st;
}

#define LMS_API_BEGIN try {
#define LMS_API_END                                                   \
  }                                                                   \
  catch (const ::lms::Err& e) { return ::lms::handle_exc(e); }        \
  catch (const std::bad_alloc&) {                                     \
    ::lms::set_error("host allocation failed");                       \
    return LMS_E_NOMEM;                                               \
  }                                                                   \
  catch (...) {                                                       \
    ::lms::set_error("unknown exception");                            \
    return LMS_E_CUDA;                                                \
  }

static void check_coords(int dim, const double* const* d) {
  if (!d) fail(LMS_E_ARG, "coords pointer array is NULL");
  for (int a = 0; a < dim; ++a)
    if (!d[a]) fail(LMS_E_ARG, "coordinate pointer is NULL");
}

// The library allocates stream-ordered (cudaMallocAsync) and synchronises
// between build phases; with the default release threshold of 0 every sync
// hands the freed pool memory back to the driver, so the next large
// allocation maps pages again.  Keep up to LMS_POOL_KEEP_GB (default 64 GB,
// of 180 GB) reserved in the device's default pool.
static void keep_pool_memory(int dev) {
  static int done_for = -1;
  if (done_for == dev) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) != cudaSuccess) return;
  double gb = 64.0;
  if (const char* e = getenv("LMS_POOL_KEEP_GB")) gb = atof(e);
  uint64_t keep = (uint64_t)(gb * 1073741824.0);
  cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  done_for = dev;
}

static lms_mesh_s* new_mesh(int dim, int64_t V, cudaStream_t s) {
  if (getenv("LMS_BUILD_VERBOSE")) {
    int dev = 0;
    cudaMemPool_t pool, cur;
    cudaGetDevice(&dev);
    cudaDeviceGetDefaultMemPool(&pool, dev);
    cudaDeviceGetMemPool(&cur, dev);
    uint64_t rc = 0, uc = 0, th = 0;
    cudaMemPoolGetAttribute(cur, cudaMemPoolAttrReservedMemCurrent, &rc);
    cudaMemPoolGetAttribute(cur, cudaMemPoolAttrUsedMemCurrent, &uc);
    cudaMemPoolGetAttribute(cur, cudaMemPoolAttrReleaseThreshold, &th);
    fprintf(stderr, "[pool] current==default %d reserved %.2f GB used %.2f GB threshold %.1f GB\n", (int)(pool == cur),
            rc / 1e9, uc / 1e9, th / 1e9);
  }
  auto* m = new lms_mesh_s();
  m->dim = dim;
  m->V = V;
  m->s0 = s;
  LMS_TRY_CUDA(cudaGetDevice(&m->device));
  keep_pool_memory(m->device);
  m->err.alloc(1, s);
  LMS_TRY_CUDA(cudaMemsetAsync(m->err.p, 0, sizeof(int), s));
  return m;
}

}  // namespace lms

using namespace lms;

extern "C" {

const char* lms_last_error(void) { return g_err.c_str(); }
int64_t lms_kernel_launches(void) { return g_launches; }

lms_status lms_build_csr(int32_t dim, int64_t n_vertices, const double* const* d_coords,
                         int32_t verts_per_elem, int64_t n_elems, const int32_t* d_elems,
                         const uint8_t* d_fixed, lms_stream_t stream, lms_mesh_t* out) {
  LMS_API_BEGIN
  lms_mesh_s* m = nullptr;
  if (!out) fail(LMS_E_ARG, "out is NULL");
  if (dim != 2 && dim != 3) fail(LMS_E_ARG, "dim must be 2 or 3");
  if (verts_per_elem != 3 && verts_per_elem != 4) fail(LMS_E_ARG, "verts_per_elem must be 3 or 4");
  if (n_vertices < 1 || n_vertices >= ((int64_t)1 << 31) - 1) fail(LMS_E_ARG, "n_vertices out of range");
  if (n_elems < 1 || !d_elems) fail(LMS_E_ARG, "need at least one element");
  if (n_elems * verts_per_elem >= ((int64_t)1 << 31)) fail(LMS_E_ARG, "too many elements for int32 indexing");
  check_coords(dim, d_coords);
  cudaStream_t s = (cudaStream_t)stream;
  // LMS_BUILD_VERBOSE: synchronising phase timings on stderr
  const bool tv = getenv("LMS_BUILD_VERBOSE") != nullptr;
  auto t_last = std::chrono::steady_clock::now();
  auto mark = [&](const char* what) {
    if (!tv) return;
    cudaStreamSynchronize(s);
    const auto t = std::chrono::steady_clock::now();
    fprintf(stderr, "[build_csr] %-12s %8.2f ms\n", what, std::chrono::duration<double, std::milli>(t - t_last).count());
    t_last = t;
  };
  m = new_mesh(dim, n_vertices, s);
  try {
    m->k = verts_per_elem;
    m->n_el = n_elems;
    for (int a = 0; a < dim; ++a) {
      m->x[a].alloc(n_vertices, s);
      LMS_TRY_CUDA(cudaMemcpyAsync(m->x[a].p, d_coords[a], n_vertices * sizeof(double), cudaMemcpyDeviceToDevice, s));
    }
    m->fixed.alloc(n_vertices, s);
    if (d_fixed)
      LMS_TRY_CUDA(cudaMemcpyAsync(m->fixed.p, d_fixed, n_vertices, cudaMemcpyDeviceToDevice, s));
    mark("coords");
    build_csr_from_elems(m, d_elems, d_fixed == nullptr, s);
    mark("csr");
    m->orig_id.alloc(n_vertices, s);
    fill_iota(m->orig_id.p, n_vertices, s);
    compute_colouring(m, s);   // colour from orig_id = input label (reading Z2)
    mark("colouring");
    m->n_free = count_free(m, s);
    mark("count");
  } catch (...) {
    delete m;
    throw;
  }
  *out = m;
  return LMS_OK;
  LMS_API_END
}

// a non-blocking side stream per device for the coordinate upload of
// lms_build_csr_host (created on first use, kept for the process)
static cudaStream_t side_stream(int dev) {
  static std::mutex mu;
  static std::map<int, cudaStream_t> streams;
  std::lock_guard<std::mutex> lk(mu);
  auto it = streams.find(dev);
  if (it != streams.end()) return it->second;
  cudaStream_t st = nullptr;
  LMS_TRY_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  streams[dev] = st;
  return st;
}

struct EventPair {
  cudaEvent_t a = nullptr, b = nullptr;
  EventPair() {
    LMS_TRY_CUDA(cudaEventCreateWithFlags(&a, cudaEventDisableTiming));
    LMS_TRY_CUDA(cudaEventCreateWithFlags(&b, cudaEventDisableTiming));
  }
  ~EventPair() {
    if (a) cudaEventDestroy(a);
    if (b) cudaEventDestroy(b);
  }
};

lms_status lms_build_csr_host(int32_t dim, int64_t n_vertices, const double* const* h_coords,
                              int32_t verts_per_elem, int64_t n_elems, const int32_t* h_elems,
                              const uint8_t* h_fixed, lms_stream_t stream, lms_mesh_t* out) {
  LMS_API_BEGIN
  lms_mesh_s* m = nullptr;
  if (!out) fail(LMS_E_ARG, "out is NULL");
  if (dim != 2 && dim != 3) fail(LMS_E_ARG, "dim must be 2 or 3");
  if (verts_per_elem != 3 && verts_per_elem != 4) fail(LMS_E_ARG, "verts_per_elem must be 3 or 4");
  if (n_vertices < 1 || n_vertices >= ((int64_t)1 << 31) - 1) fail(LMS_E_ARG, "n_vertices out of range");
  if (n_elems < 1 || !h_elems) fail(LMS_E_ARG, "need at least one element");
  if (n_elems * verts_per_elem >= ((int64_t)1 << 31)) fail(LMS_E_ARG, "too many elements for int32 indexing");
  check_coords(dim, h_coords);
  cudaStream_t s = (cudaStream_t)stream;
  m = new_mesh(dim, n_vertices, s);
  try {
    m->k = verts_per_elem;
    m->n_el = n_elems;
    // elements (and the caller's fixed mask) first, on the call's stream
    m->elems.alloc(n_elems * verts_per_elem, s);
    LMS_TRY_CUDA(cudaMemcpyAsync(m->elems.p, h_elems, n_elems * verts_per_elem * sizeof(int32_t),
                                 cudaMemcpyHostToDevice, s));
    m->fixed.alloc(n_vertices, s);
    if (h_fixed) LMS_TRY_CUDA(cudaMemcpyAsync(m->fixed.p, h_fixed, n_vertices, cudaMemcpyHostToDevice, s));
    for (int a = 0; a < dim; ++a) m->x[a].alloc(n_vertices, s);
    // coordinates on the side stream, overlapping the CSR build and the
    // colouring (neither reads them); the call's stream waits before it returns
    EventPair ev;
    cudaStream_t s2 = side_stream(m->device);
    LMS_TRY_CUDA(cudaEventRecord(ev.a, s));  // the allocations above are stream-ordered on s
    LMS_TRY_CUDA(cudaStreamWaitEvent(s2, ev.a, 0));
    // Once a copy is queued on s2, every exit path (including a throw from a
    // later copy) orders s after the upload before m's buffers can go back to
    // s's scratch cache.
    struct JoinUpload {
      cudaEvent_t ev;
      cudaStream_t s, s2;
      bool armed = false;
      ~JoinUpload() {
        if (!armed) return;
        cudaEventRecord(ev, s2);
        cudaStreamWaitEvent(s, ev, 0);
      }
    } join{ev.b, s, s2};
    for (int a = 0; a < dim; ++a) {
      join.armed = true;
      LMS_TRY_CUDA(cudaMemcpyAsync(m->x[a].p, h_coords[a], n_vertices * sizeof(double), cudaMemcpyHostToDevice, s2));
    }
    build_csr_from_elems(m, nullptr, h_fixed == nullptr, s);
    m->orig_id.alloc(n_vertices, s);
    fill_iota(m->orig_id.p, n_vertices, s);
    compute_colouring(m, s);  // colour from orig_id = input label (reading Z2)
    join.armed = false;
    LMS_TRY_CUDA(cudaEventRecord(ev.b, s2));
    LMS_TRY_CUDA(cudaStreamWaitEvent(s, ev.b, 0));
    m->n_free = count_free(m, s);
  } catch (...) {
    delete m;
    throw;
  }
  *out = m;
  return LMS_OK;
  LMS_API_END
}

lms_status lms_mesh_from_csr(int32_t dim, int64_t n_vertices, const double* const* d_coords,
                             const uint8_t* d_fixed, const int32_t* d_row_ptr, const int32_t* d_col_idx,
                             const int32_t* d_orig_id, const int8_t* d_colour, const double* d_quality,
                             lms_stream_t stream, lms_mesh_t* out) {
  LMS_API_BEGIN
  if (!out) fail(LMS_E_ARG, "out is NULL");
  if (dim != 2 && dim != 3) fail(LMS_E_ARG, "dim must be 2 or 3");
  if (n_vertices < 1 || n_vertices >= ((int64_t)1 << 31) - 1) fail(LMS_E_ARG, "n_vertices out of range");
  if (!d_fixed || !d_row_ptr || !d_col_idx) fail(LMS_E_ARG, "fixed/row_ptr/col_idx required");
  check_coords(dim, d_coords);
  cudaStream_t s = (cudaStream_t)stream;
  int32_t nnz32 = 0;
  LMS_TRY_CUDA(cudaMemcpyAsync(&nnz32, d_row_ptr + n_vertices, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  LMS_TRY_CUDA(cudaStreamSynchronize(s));
  if (nnz32 < 0) fail(LMS_E_ARG, "row_ptr[V] < 0");
  lms_mesh_s* m = new_mesh(dim, n_vertices, s);
  try {
    m->nnz = nnz32;
    for (int a = 0; a < dim; ++a) {
      m->x[a].alloc(n_vertices, s);
      LMS_TRY_CUDA(cudaMemcpyAsync(m->x[a].p, d_coords[a], n_vertices * sizeof(double), cudaMemcpyDeviceToDevice, s));
    }
    m->fixed.alloc(n_vertices, s);
    LMS_TRY_CUDA(cudaMemcpyAsync(m->fixed.p, d_fixed, n_vertices, cudaMemcpyDeviceToDevice, s));
    m->row_ptr.alloc(n_vertices + 1, s);
    LMS_TRY_CUDA(cudaMemcpyAsync(m->row_ptr.p, d_row_ptr, (n_vertices + 1) * sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
    m->col.alloc(m->nnz, s);
    if (m->nnz)
      LMS_TRY_CUDA(cudaMemcpyAsync(m->col.p, d_col_idx, m->nnz * sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
    m->orig_id.alloc(n_vertices, s);
    if (d_orig_id)
      LMS_TRY_CUDA(cudaMemcpyAsync(m->orig_id.p, d_orig_id, n_vertices * sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
    else
      fill_iota(m->orig_id.p, n_vertices, s);
    if (d_quality) {
      m->quality.alloc(n_vertices, s);
      LMS_TRY_CUDA(cudaMemcpyAsync(m->quality.p, d_quality, n_vertices * sizeof(double), cudaMemcpyDeviceToDevice, s));
      m->has_quality = true;
      m->quality_external = true;
    }
    if (d_colour) {
      m->colour.alloc(n_vertices, s);
      LMS_TRY_CUDA(cudaMemcpyAsync(m->colour.p, d_colour, n_vertices, cudaMemcpyDeviceToDevice, s));
    }
    // validates indices / degrees, computes colouring when not given
    compute_colouring(m, s);
    m->n_free = count_free(m, s);
  } catch (...) {
    delete m;
    throw;
  }
  *out = m;
  return LMS_OK;
  LMS_API_END
}

void lms_mesh_destroy(lms_mesh_t m) {
  if (!m) return;
  DevGuard dg(m);
  cudaDeviceSynchronize();  // buffers may have been used on any stream of m's device
  delete m;
}

lms_status lms_order(lms_mesh_t m, lms_order_kind kind, uint64_t seed, int32_t* d_perm, lms_stream_t stream) {
  LMS_API_BEGIN
  if (!m || !d_perm) fail(LMS_E_ARG, "NULL handle or perm");
  DevGuard dg(m);
  cudaStream_t s = (cudaStream_t)stream;
  switch (kind) {
    case LMS_ORDER_ORIGINAL:
      fill_iota(d_perm, m->V, s);
      break;
    case LMS_ORDER_RANDOM:
      order_random(m, seed, d_perm, s);
      break;
    case LMS_ORDER_BFS:
      if ((int64_t)seed >= m->V || (int64_t)seed < 0) fail(LMS_E_ARG, "BFS seed vertex out of range");
      order_bfs(m, (int64_t)seed, d_perm, s);
      break;
    case LMS_ORDER_RBFS:
      if ((int64_t)seed >= m->V || (int64_t)seed < 0) fail(LMS_E_ARG, "BFS seed vertex out of range");
      order_rbfs(m, (int64_t)seed, false, d_perm, s);
      break;
    case LMS_ORDER_RCM:
      order_rbfs(m, 0, true, d_perm, s);
      break;
    case LMS_ORDER_DFS:
      if ((int64_t)seed >= m->V || (int64_t)seed < 0) fail(LMS_E_ARG, "DFS seed vertex out of range");
      order_dfs(m, (int64_t)seed, d_perm, s);
      break;
    case LMS_ORDER_RDR:
      order_rdr(m, d_perm, s);
      break;
    case LMS_ORDER_RDR_WINDOWED:
      if ((int64_t)seed < 0 || seed > (uint64_t)INT32_MAX) fail(LMS_E_ARG, "window length out of range");
      order_rdr(m, d_perm, s, seed == 0 ? 65536 : (int64_t)seed);
      break;
    default:
      fail(LMS_E_ARG, "unknown ordering kind");
  }
  return LMS_OK;
  LMS_API_END
}

lms_status lms_permute(lms_mesh_t m, const int32_t* d_perm, lms_stream_t stream) {
  LMS_API_BEGIN
  if (!m || !d_perm) fail(LMS_E_ARG, "NULL handle or perm");
  DevGuard dg(m);
  permute_mesh(m, d_perm, (cudaStream_t)stream);
  return LMS_OK;
  LMS_API_END
}

lms_status lms_smooth(lms_mesh_t m, int32_t sweeps, lms_stream_t stream) {
  LMS_API_BEGIN
  if (!m) fail(LMS_E_ARG, "NULL handle");
  DevGuard dg(m);
  if (sweeps < 0) fail(LMS_E_ARG, "sweeps < 0");
  if (sweeps == 0 || m->n_free == 0) return LMS_OK;
  cudaStream_t s = (cudaStream_t)stream;
  if (!m->sched.valid) {
    sync_soa(m, s);
    build_schedule(m, s);
  }
  m->coords_moved = true;
  run_sweeps(m, sweeps, s);
  return LMS_OK;
  LMS_API_END
}

lms_status lms_set_async_errors(lms_mesh_t m, int32_t on) {
  LMS_API_BEGIN
  if (!m) fail(LMS_E_ARG, "NULL handle");
  m->async_errors = on != 0;
  return LMS_OK;
  LMS_API_END
}

lms_status lms_check(lms_mesh_t m, lms_stream_t stream) {
  LMS_API_BEGIN
  if (!m) fail(LMS_E_ARG, "NULL handle");
  DevGuard dg(m);
  check_err_flag(m, (cudaStream_t)stream, "lms_check (a sweep kernel's watchdog aborted a wait)");
  return LMS_OK;
  LMS_API_END
}

lms_status lms_set_schedule(lms_mesh_t m, lms_schedule_kind kind, int32_t tile, int32_t lag) {
  LMS_API_BEGIN
  if (!m) fail(LMS_E_ARG, "NULL handle");
  DevGuard dg(m);
  if (kind != LMS_SCHED_AUTO && kind != LMS_SCHED_S1 && kind != LMS_SCHED_S2 && kind != LMS_SCHED_S3 &&
      kind != LMS_SCHED_GZ && kind != LMS_SCHED_JACOBI)
    fail(LMS_E_ARG, "unknown schedule");
  if (kind == LMS_SCHED_GZ && lag > 8) fail(LMS_E_ARG, "GZ: at most 8 sweeps per pass");
  if (kind == LMS_SCHED_S2 && m->dim != 3) fail(LMS_E_ARG, "S2 is the 3D kernel (2D meshes: GZ)");
  if (tile < 0 || lag < 0) fail(LMS_E_ARG, "tile/lag < 0");
  if (tile != 0 && (tile < 32 || tile > (1 << 20))) fail(LMS_E_ARG, "tile must be in [32, 2^20]");
  m->sched_req = kind;
  m->tile_req = tile;
  m->lag_req = lag;
  m->sched.valid = false;
  return LMS_OK;
  LMS_API_END
}

lms_status lms_set_tiling(lms_mesh_t m, lms_tiling_kind kind) {
  LMS_API_BEGIN
  if (!m) fail(LMS_E_ARG, "NULL handle");
  DevGuard dg(m);
  if (kind != LMS_TILING_AUTO && kind != LMS_TILING_STORAGE && kind != LMS_TILING_SPATIAL)
    fail(LMS_E_ARG, "unknown tiling");
  m->tiling_req = kind;
  m->sched.valid = false;
  return LMS_OK;
  LMS_API_END
}

lms_status lms_schedule_info2(lms_mesh_t m, int32_t* tiling, int64_t* n_tiles, int32_t* max_reach) {
  LMS_API_BEGIN
  if (!m) fail(LMS_E_ARG, "NULL handle");
  DevGuard dg(m);
  const bool gz = m->sched.valid && m->sched.kind == LMS_SCHED_GZ;
  if (tiling) *tiling = m->sched.valid ? (gz ? (int)LMS_TILING_SPATIAL : m->sched.tiling) : 0;
  if (n_tiles) *n_tiles = m->sched.valid ? (gz ? m->sched.gz_K : m->sched.K) : 0;
  if (max_reach) *max_reach = m->sched.valid ? m->sched.max_reach : 0;
  return LMS_OK;
  LMS_API_END
}

lms_status lms_mesh_info(lms_mesh_t m, int64_t* V, int64_t* nnz, int32_t* n_colours, int32_t* dim) {
  LMS_API_BEGIN
  if (!m) fail(LMS_E_ARG, "NULL handle");
  DevGuard dg(m);
  if (V) *V = m->V;
  if (nnz) *nnz = m->nnz;
  if (n_colours) *n_colours = m->C;
  if (dim) *dim = m->dim;
  return LMS_OK;
  LMS_API_END
}

lms_status lms_schedule_info(lms_mesh_t m, int64_t* n_free, int32_t* sched_kind, int32_t* tile, int32_t* lag) {
  LMS_API_BEGIN
  if (!m) fail(LMS_E_ARG, "NULL handle");
  DevGuard dg(m);
  if (n_free) *n_free = m->n_free;
  if (sched_kind) *sched_kind = m->sched.valid ? m->sched.kind : m->sched_req;
  const bool gz = m->sched.valid && m->sched.kind == LMS_SCHED_GZ;
  if (tile) *tile = m->sched.valid ? (gz ? m->sched.gz_T : m->sched.tile) : 0;
  if (lag) *lag = m->sched.valid ? (gz ? m->sched.gz_P : m->sched.lag) : 0;
  return LMS_OK;
  LMS_API_END
}

lms_status lms_export_coords(lms_mesh_t m, double* const* d_out, lms_stream_t stream) {
  LMS_API_BEGIN
  if (!m) fail(LMS_E_ARG, "NULL handle");
  DevGuard dg(m);
  check_coords(m->dim, d_out);
  sync_soa(m, (cudaStream_t)stream);
  for (int a = 0; a < m->dim; ++a)
    LMS_TRY_CUDA(cudaMemcpyAsync(d_out[a], m->x[a].p, m->V * sizeof(double), cudaMemcpyDefault, (cudaStream_t)stream));
  return LMS_OK;
  LMS_API_END
}

lms_status lms_import_coords(lms_mesh_t m, const double* const* d_in, lms_stream_t stream) {
  LMS_API_BEGIN
  if (!m) fail(LMS_E_ARG, "NULL handle");
  DevGuard dg(m);
  check_coords(m->dim, d_in);
  for (int a = 0; a < m->dim; ++a)
    LMS_TRY_CUDA(cudaMemcpyAsync(m->x[a].p, d_in[a], m->V * sizeof(double), cudaMemcpyDefault, (cudaStream_t)stream));
  soa_changed(m);
  m->coords_moved = true;
  return LMS_OK;
  LMS_API_END
}

lms_status lms_export_csr(lms_mesh_t m, int32_t* d_row_ptr, int32_t* d_col_idx, lms_stream_t stream) {
  LMS_API_BEGIN
  if (!m) fail(LMS_E_ARG, "NULL handle");
  DevGuard dg(m);
  cudaStream_t s = (cudaStream_t)stream;
  if (d_row_ptr)
    LMS_TRY_CUDA(cudaMemcpyAsync(d_row_ptr, m->row_ptr.p, (m->V + 1) * sizeof(int32_t), cudaMemcpyDefault, s));
  if (d_col_idx && m->nnz)
    LMS_TRY_CUDA(cudaMemcpyAsync(d_col_idx, m->col.p, m->nnz * sizeof(int32_t), cudaMemcpyDefault, s));
  return LMS_OK;
  LMS_API_END
}

lms_status lms_export_colour(lms_mesh_t m, int8_t* d_colour, lms_stream_t stream) {
  LMS_API_BEGIN
  if (!m || !d_colour) fail(LMS_E_ARG, "NULL argument");
  DevGuard dg(m);
  LMS_TRY_CUDA(cudaMemcpyAsync(d_colour, m->colour.p, m->V, cudaMemcpyDefault, (cudaStream_t)stream));
  return LMS_OK;
  LMS_API_END
}

lms_status lms_export_fixed(lms_mesh_t m, uint8_t* d_fixed, lms_stream_t stream) {
  LMS_API_BEGIN
  if (!m || !d_fixed) fail(LMS_E_ARG, "NULL argument");
  DevGuard dg(m);
  LMS_TRY_CUDA(cudaMemcpyAsync(d_fixed, m->fixed.p, m->V, cudaMemcpyDefault, (cudaStream_t)stream));
  return LMS_OK;
  LMS_API_END
}

lms_status lms_export_orig_id(lms_mesh_t m, int32_t* d_orig_id, lms_stream_t stream) {
  LMS_API_BEGIN
  if (!m || !d_orig_id) fail(LMS_E_ARG, "NULL argument");
  DevGuard dg(m);
  LMS_TRY_CUDA(cudaMemcpyAsync(d_orig_id, m->orig_id.p, m->V * sizeof(int32_t), cudaMemcpyDefault, (cudaStream_t)stream));
  return LMS_OK;
  LMS_API_END
}

lms_status lms_export_elems(lms_mesh_t m, int32_t* d_elems, lms_stream_t stream) {
  LMS_API_BEGIN
  if (!m || !d_elems) fail(LMS_E_ARG, "NULL argument");
  DevGuard dg(m);
  if (!m->k) fail(LMS_E_STATE, "mesh has no elements");
  LMS_TRY_CUDA(cudaMemcpyAsync(d_elems, m->elems.p, m->n_el * m->k * sizeof(int32_t), cudaMemcpyDefault, (cudaStream_t)stream));
  return LMS_OK;
  LMS_API_END
}

lms_status lms_export_quality(lms_mesh_t m, double* d_quality, lms_stream_t stream) {
  LMS_API_BEGIN
  if (!m || !d_quality) fail(LMS_E_ARG, "NULL argument");
  DevGuard dg(m);
  cudaStream_t s = (cudaStream_t)stream;
  if (m->quality_external) {
    LMS_TRY_CUDA(cudaMemcpyAsync(d_quality, m->quality.p, m->V * sizeof(double), cudaMemcpyDefault, s));
  } else {
    DBuf<double> q(m->V, s);
    compute_quality(m, q.p, s);
    LMS_TRY_CUDA(cudaMemcpyAsync(d_quality, q.p, m->V * sizeof(double), cudaMemcpyDefault, s));
  }
  return LMS_OK;
  LMS_API_END
}

}  // extern "C"
