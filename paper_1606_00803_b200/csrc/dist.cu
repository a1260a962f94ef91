// dist.cu -- the multi-GPU sweep behind the C ABI (SURVEY 8(b) lms_dist_*,
// 8(e)): contiguous vertex ranges, a deep ghost zone, one halo exchange per
// pass over a library-owned NCCL communicator (NVLink via NVSwitch).
//
// Partition ("static ... evenly dividing the vertices";
// DESIGN.md reading Z22): the relabelled mesh is split into `nranks`
// contiguous storage ranges [a_r, b_r) with ceil(n_free / nranks) free
// vertices each (the oracle's O9 split).  Rank r owns [a_r, b_r).
//
// Deep halo: after P sweeps an owned vertex depends on the
// pass-start coordinates only through chains of free vertices at most
// D = C * P hops long (the ghost-zone argument of gz.cu).  So rank r keeps
// every vertex within D hops of its range (hops through free vertices), in
// ascending global label -- a monotone relabelling, so every row keeps its CSR
// order and every sum is bit-identical to the 1-GPU sweep.  Free vertices
// closer than D keep their rows and are smoothed (redundantly on the ghosts);
// the D-hop ring is fixed locally and only read.  One exchange per pass --
// every ghost from its owner -- refreshes the ghost values, then the rank runs
// P sweeps on its local mesh with its own schedule (GZ in 2D).  Owned values
// are exact after every pass.
//
// Plan construction is on the rank's GPU and costs O(V/P + halo) work beyond
// O(V) memsets and one O(V) scan: the split points by a scan of the free
// flags, the ghost zone by D frontier expansions from the owned range, the
// local CSR by a gather of the global rows through a global -> local map.
// The ghost lists are exchanged with the owners over NCCL (counts, then ids),
// so no rank ever computes another rank's local set.
//
// lms_dist_create_local builds the same per-rank plans for all ranks in one
// process on one GPU, exchanging by device copies (for tests: no kernel ever
// waits on another rank).
#include <dlfcn.h>
#include <nccl.h>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <cstring>
#include <mutex>
#include <vector>

#include "lms_internal.cuh"

namespace lms {

// ------------------------------------------------------------------ NCCL (dlopen)
// The library binds NCCL at run time: the process normally has it loaded
// already (torch), and a C caller without NCCL can still use every other call.
struct NcclApi {
  bool ok = false;
  std::string why;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

static NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    void* h = nullptr;
    for (const char* n : names)
      if ((h = dlopen(n, RTLD_NOW | RTLD_GLOBAL))) break;
    if (!h) {
      api.why = std::string("dlopen(libnccl.so.2) failed: ") + dlerror();
      return;
    }
    auto sym = [&](const char* s) {
      void* p = dlsym(h, s);
      if (!p) api.why += std::string(" missing ") + s;
      return p;
    };
    api.GetUniqueId = (decltype(api.GetUniqueId))sym("ncclGetUniqueId");
    api.CommInitRank = (decltype(api.CommInitRank))sym("ncclCommInitRank");
    api.CommDestroy = (decltype(api.CommDestroy))sym("ncclCommDestroy");
    api.Send = (decltype(api.Send))sym("ncclSend");
    api.Recv = (decltype(api.Recv))sym("ncclRecv");
    api.GroupStart = (decltype(api.GroupStart))sym("ncclGroupStart");
    api.GroupEnd = (decltype(api.GroupEnd))sym("ncclGroupEnd");
    api.GetErrorString = (decltype(api.GetErrorString))sym("ncclGetErrorString");
    api.ok = api.why.empty();
  });
  return api;
}

#define LMS_TRY_NCCL(expr)                                                                              \
  do {                                                                                                  \
    ncclResult_t _r = (expr);                                                                           \
    if (_r != ncclSuccess)                                                                              \
      throw ::lms::Err{LMS_E_NCCL, std::string(#expr) + ": " + nccl().GetErrorString(_r) + " @" + __FILE__ + \
                                       ":" + std::to_string(__LINE__)};                                 \
  } while (0)

// ------------------------------------------------------------------ plan kernels
__global__ void k_dist_free(const uint8_t* __restrict__ fixed, int64_t V, int32_t* __restrict__ f) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < V; v += (int64_t)gridDim.x * blockDim.x)
    f[v] = fixed[v] ? 0 : 1;
}

// bounds[p] (p = 1..P-1): smallest j >= 1 with ex[j] >= per * p (part p - 1
// ends right after its (per * p)-th free vertex), V if per * p > n_free
__global__ void k_dist_bounds(const int32_t* __restrict__ ex, int64_t V, int P, int64_t per, int64_t nfree,
                              int64_t* __restrict__ bounds) {
  const int p = threadIdx.x;
  if (p > P) return;
  if (p == 0) { bounds[0] = 0; return; }
  if (p == P) { bounds[P] = V; return; }
  const int64_t want = per * p;
  if (want > nfree) { bounds[p] = V; return; }
  int64_t lo = 1, hi = V;  // ex[V] = nfree >= want
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if ((int64_t)ex[mid] >= want) hi = mid;
    else lo = mid + 1;
  }
  bounds[p] = lo;
}

__global__ void k_dist_own(int32_t* __restrict__ dist, const uint8_t* __restrict__ fixed, int64_t a, int64_t b,
                           int32_t* __restrict__ front, int* __restrict__ nfront) {
  for (int64_t v = a + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < b; v += (int64_t)gridDim.x * blockDim.x) {
    dist[v] = 0;
    if (!fixed[v]) front[atomicAdd(nfront, 1)] = (int32_t)v;
  }
}

// one hop: every unvisited neighbour of a frontier (free) vertex gets level L;
// it joins the ghost list, and the next frontier if it is free
__global__ void k_dist_expand(const int32_t* __restrict__ rp, const int32_t* __restrict__ col,
                              const uint8_t* __restrict__ fixed, const int32_t* __restrict__ front, int nfront,
                              int L, int32_t* __restrict__ dist, int32_t* __restrict__ next, int* __restrict__ nnext,
                              int32_t* __restrict__ ghost, int* __restrict__ nghost) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nfront; i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t v = front[i];
    for (int32_t e = rp[v]; e < rp[v + 1]; ++e) {
      const int32_t u = col[e];
      if (atomicCAS(dist + u, -1, L) == -1) {
        ghost[atomicAdd(nghost, 1)] = u;
        if (!fixed[u]) next[atomicAdd(nnext, 1)] = u;
      }
    }
  }
}

// local ids = ghosts below a, then [a, b), then ghosts from b on (all ascending)
__global__ void k_dist_local_ids(const int32_t* __restrict__ gs, int64_t ng, int64_t nbelow, int64_t a, int64_t b,
                                 int32_t* __restrict__ ids, int32_t* __restrict__ g2l) {
  const int64_t n = ng + (b - a);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int32_t g;
    if (i < nbelow) g = gs[i];
    else if (i < nbelow + (b - a)) g = (int32_t)(a + (i - nbelow));
    else g = gs[i - (b - a)];
    ids[i] = g;
    g2l[g] = (int32_t)i;
  }
}

__global__ void k_dist_local_deg(const int32_t* __restrict__ ids, int64_t n, const int32_t* __restrict__ rp,
                                 const uint8_t* __restrict__ fixed, const int32_t* __restrict__ dist, int D,
                                 int32_t* __restrict__ deg, uint8_t* __restrict__ lfixed) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t g = ids[i];
    const bool ev = !fixed[g] && dist[g] < D;  // evaluated: its row stays inside the local mesh
    deg[i] = ev ? rp[g + 1] - rp[g] : 1;
    lfixed[i] = ev ? 0 : 1;
  }
}

__global__ void k_dist_local_rows(const int32_t* __restrict__ ids, int64_t n, const int32_t* __restrict__ rp,
                                  const int32_t* __restrict__ col, const int32_t* __restrict__ g2l,
                                  const uint8_t* __restrict__ lfixed, const int32_t* __restrict__ lrp,
                                  const int8_t* __restrict__ colour, int32_t* __restrict__ lcol,
                                  int8_t* __restrict__ lcolour, int* err) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t g = ids[i];
    const int32_t o = lrp[i];
    if (!lfixed[i]) {
      for (int32_t e = rp[g], j = 0; e < rp[g + 1]; ++e, ++j) {
        const int32_t l = g2l[col[e]];
        if (l < 0) raise_err(err, LMS_E_INDEX);  // cannot happen: every neighbour is within D hops
        lcol[o + j] = l;
      }
      lcolour[i] = colour[g];
    } else {  // a row that is never evaluated: one dummy neighbour (never read)
      lcol[o] = (int32_t)(i + 1 < n ? i + 1 : (i > 0 ? i - 1 : 0));
      lcolour[i] = -1;
    }
  }
}

__global__ void k_dist_gather_coords(const int32_t* __restrict__ ids, int64_t n, const double* __restrict__ x,
                                     double* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = x[ids[i]];
}

__global__ void k_dist_to_local(int32_t* __restrict__ ids, int64_t n, int64_t off) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    ids[i] = (int32_t)(ids[i] + off);
}

static unsigned gs(int64_t n) {
  const unsigned g = grid_for(n > 0 ? n : 1, 256);
  return g > 8192 ? 8192 : g;
}

}  // namespace lms

// ------------------------------------------------------------------ the handle
struct lms_dist_s {
  int device = 0;
  int rank = 0, nranks = 1, P = 1, D = 0, dim = 2;
  int64_t V = 0, a = 0, b = 0, lo = 0, n_local = 0;
  std::vector<int64_t> bounds;
  lms_mesh_s* local = nullptr;
  lms::DBuf<int32_t> local_ids;   // global label of each local vertex (ascending)
  struct Peer {
    int q = 0;
    int64_t n_send = 0, n_recv = 0, soff = 0, roff = 0;  // offsets in vertices
    lms::DBuf<int32_t> send_idx, recv_idx;               // local ids (ascending global label)
    std::vector<int32_t> h_recv_global;                  // ghost labels owned by q (plan build)
  };
  std::vector<Peer> peers;        // every other rank (empty lists allowed)
  int64_t tot_send = 0, tot_recv = 0;
  lms::DBuf<double> sbuf, rbuf;   // packed [x.. y.. (z..)] per peer block
  ncclComm_t comm = nullptr;
  bool local_group = false;
  ~lms_dist_s() {
    if (local) lms_mesh_destroy(local);
    if (comm && lms::nccl().ok) lms::nccl().CommDestroy(comm);
  }
};

namespace lms {

// The rank-local part of the plan: bounds, ghost zone, local mesh, ghost
// lists per owner (recv side).  The send side needs the owners' peers' ghost
// lists (exchange_lists / the local group).
static void plan_rank(lms_mesh_s* m, lms_dist_s* d, int tile, cudaStream_t s) {
  const int64_t V = m->V;
  const int P = d->nranks;
  d->V = V;
  d->dim = m->dim;
  d->D = m->C * d->P;
  sync_soa(m, s);
  // ---- split points
  {
    DBuf<int32_t> f(V + 1, s), ex(V + 1, s);
    k_dist_free<<<gs(V), 256, 0, s>>>(m->fixed.p, V, f.p);
    LMS_CHECK_LAUNCH();
    LMS_TRY_CUDA(cudaMemsetAsync(f.p + V, 0, sizeof(int32_t), s));
    size_t tb = 0;
    LMS_TRY_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, f.p, ex.p, V + 1, s));
    {
      DBuf<char> tmp(tb, s);
      LMS_TRY_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tb, f.p, ex.p, V + 1, s));
    }
    int32_t nfree32 = 0;
    LMS_TRY_CUDA(cudaMemcpyAsync(&nfree32, ex.p + V, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    LMS_TRY_CUDA(cudaStreamSynchronize(s));
    const int64_t nfree = nfree32;
    const int64_t per = (nfree + P - 1) / P;
    DBuf<int64_t> bd(P + 1, s);
    k_dist_bounds<<<1, ((P + 1 + 31) / 32) * 32, 0, s>>>(ex.p, V, P, per, nfree, bd.p);
    LMS_CHECK_LAUNCH();
    d->bounds.assign(P + 1, 0);
    LMS_TRY_CUDA(cudaMemcpyAsync(d->bounds.data(), bd.p, (P + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    LMS_TRY_CUDA(cudaStreamSynchronize(s));
    for (int p = 1; p <= P; ++p) d->bounds[p] = std::max(d->bounds[p], d->bounds[p - 1]);
  }
  const int64_t a = d->bounds[d->rank], b = d->bounds[d->rank + 1];
  d->a = a;
  d->b = b;
  // ---- ghost zone: D frontier expansions through free vertices
  // Every discovered vertex is new (CAS on its level), so the ghost list and
  // each frontier hold fewer than V - (b - a) + 1 entries.
  const int64_t gcap = std::max<int64_t>(V - (b - a), 1);
  DBuf<int32_t> dist(V, s), fa(std::max(b - a, gcap), s), fb(gcap, s), ghost(gcap, s);
  DBuf<int> cnt(3, s);  // [0] frontier size, [1] next size, [2] ghosts
  LMS_TRY_CUDA(cudaMemsetAsync(dist.p, 0xff, V * sizeof(int32_t), s));
  LMS_TRY_CUDA(cudaMemsetAsync(cnt.p, 0, 3 * sizeof(int), s));
  k_dist_own<<<gs(b - a), 256, 0, s>>>(dist.p, m->fixed.p, a, b, fa.p, cnt.p);
  LMS_CHECK_LAUNCH();
  int h[3] = {0, 0, 0};
  LMS_TRY_CUDA(cudaMemcpyAsync(h, cnt.p, sizeof(h), cudaMemcpyDeviceToHost, s));
  LMS_TRY_CUDA(cudaStreamSynchronize(s));
  int nfront = h[0], nghost = 0;
  int32_t* cur = fa.p;
  int32_t* nxt = fb.p;
  for (int L = 1; L <= d->D && nfront > 0; ++L) {
    LMS_TRY_CUDA(cudaMemsetAsync(cnt.p + 1, 0, sizeof(int), s));
    k_dist_expand<<<gs(nfront), 256, 0, s>>>(m->row_ptr.p, m->col.p, m->fixed.p, cur, nfront, L, dist.p, nxt,
                                             cnt.p + 1, ghost.p, cnt.p + 2);
    LMS_CHECK_LAUNCH();
    LMS_TRY_CUDA(cudaMemcpyAsync(h, cnt.p, sizeof(h), cudaMemcpyDeviceToHost, s));
    LMS_TRY_CUDA(cudaStreamSynchronize(s));
    nfront = h[1];
    nghost = h[2];
    std::swap(cur, nxt);
  }
  fa.release();
  fb.release();
  // ---- local ids: sort the ghosts, merge with the owned range
  DBuf<int32_t> gsorted(std::max(nghost, 1), s);
  if (nghost) {
    size_t tb = 0;
    LMS_TRY_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tb, ghost.p, gsorted.p, nghost, 0, 32, s));
    DBuf<char> tmp(tb, s);
    LMS_TRY_CUDA(cub::DeviceRadixSort::SortKeys(tmp.p, tb, ghost.p, gsorted.p, nghost, 0, 32, s));
  }
  ghost.release();
  std::vector<int32_t> hg(nghost);
  if (nghost) LMS_TRY_CUDA(cudaMemcpyAsync(hg.data(), gsorted.p, nghost * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  LMS_TRY_CUDA(cudaStreamSynchronize(s));
  const int64_t nbelow = std::lower_bound(hg.begin(), hg.end(), (int32_t)a) - hg.begin();
  const int64_t n = nghost + (b - a);
  d->n_local = n;
  d->lo = nbelow;
  d->local_ids.alloc(std::max<int64_t>(n, 1), s);
  DBuf<int32_t> g2l(V, s);
  LMS_TRY_CUDA(cudaMemsetAsync(g2l.p, 0xff, V * sizeof(int32_t), s));
  k_dist_local_ids<<<gs(n), 256, 0, s>>>(gsorted.p, nghost, nbelow, a, b, d->local_ids.p, g2l.p);
  LMS_CHECK_LAUNCH();
  // ---- local CSR, mask, colours, coordinates
  DBuf<int32_t> deg(n + 1, s), lrp(n + 1, s);
  DBuf<uint8_t> lfixed(std::max<int64_t>(n, 1), s);
  k_dist_local_deg<<<gs(n), 256, 0, s>>>(d->local_ids.p, n, m->row_ptr.p, m->fixed.p, dist.p, d->D, deg.p, lfixed.p);
  LMS_CHECK_LAUNCH();
  LMS_TRY_CUDA(cudaMemsetAsync(deg.p + n, 0, sizeof(int32_t), s));
  {
    size_t tb = 0;
    LMS_TRY_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, deg.p, lrp.p, n + 1, s));
    DBuf<char> tmp(tb, s);
    LMS_TRY_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tb, deg.p, lrp.p, n + 1, s));
  }
  int32_t lnnz = 0;
  LMS_TRY_CUDA(cudaMemcpyAsync(&lnnz, lrp.p + n, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  LMS_TRY_CUDA(cudaStreamSynchronize(s));
  DBuf<int32_t> lcol(std::max(lnnz, 1), s);
  DBuf<int8_t> lcolour(std::max<int64_t>(n, 1), s);
  k_dist_local_rows<<<gs(n), 256, 0, s>>>(d->local_ids.p, n, m->row_ptr.p, m->col.p, g2l.p, lfixed.p, lrp.p,
                                          m->colour.p, lcol.p, lcolour.p, m->err.p);
  LMS_CHECK_LAUNCH();
  check_err_flag(m, s, "lms_dist_create (local rows)");
  DBuf<double> lx[3];
  const double* lxp[3] = {nullptr, nullptr, nullptr};
  for (int ax = 0; ax < m->dim; ++ax) {
    lx[ax].alloc(std::max<int64_t>(n, 1), s);
    k_dist_gather_coords<<<gs(n), 256, 0, s>>>(d->local_ids.p, n, m->x[ax].p, lx[ax].p);
    LMS_CHECK_LAUNCH();
    lxp[ax] = lx[ax].p;
  }
  if (n == 0) return;  // an empty range with no ghosts (tiny mesh, many ranks): nothing to smooth
  lms_mesh_t lm = nullptr;
  const lms_status st = lms_mesh_from_csr(m->dim, n, lxp, lfixed.p, lrp.p, lcol.p, nullptr, lcolour.p, nullptr,
                                          (lms_stream_t)s, &lm);
  if (st != LMS_OK) fail(st, std::string("lms_dist_create: local mesh: ") + lms_last_error());
  d->local = lm;
  lm->sched_req = m->dim == 2 ? LMS_SCHED_GZ : LMS_SCHED_AUTO;
  lm->tile_req = tile;
  lm->lag_req = m->dim == 2 ? d->P : 0;
  lm->sched.valid = false;
  // ---- recv lists: my ghosts grouped by owner (ascending label)
  d->peers.clear();
  for (int q = 0; q < P; ++q) {
    if (q == d->rank) continue;
    lms_dist_s::Peer pr;
    pr.q = q;
    const int64_t qa = d->bounds[q], qb = d->bounds[q + 1];
    auto i0 = std::lower_bound(hg.begin(), hg.end(), (int32_t)qa);
    auto i1 = std::lower_bound(hg.begin(), hg.end(), (int32_t)qb);
    if (qb <= qa) i1 = i0;
    pr.h_recv_global.assign(i0, i1);
    pr.n_recv = (int64_t)pr.h_recv_global.size();
    if (pr.n_recv) {
      // local index of a ghost = its position in the sorted ghost list, shifted past the owned range if above it
      const int64_t gpos = i0 - hg.begin();
      std::vector<int32_t> li(pr.n_recv);
      for (int64_t j = 0; j < pr.n_recv; ++j) li[j] = (int32_t)(gpos + j + (gpos + j >= nbelow ? (b - a) : 0));
      pr.recv_idx.alloc(pr.n_recv, s);
      LMS_TRY_CUDA(cudaMemcpyAsync(pr.recv_idx.p, li.data(), pr.n_recv * sizeof(int32_t), cudaMemcpyHostToDevice, s));
      LMS_TRY_CUDA(cudaStreamSynchronize(s));  // li is a host temporary
    }
    d->peers.push_back(std::move(pr));
  }
}

// send lists from the ids the peer needs (global labels in my range)
static void set_send(lms_dist_s* d, lms_dist_s::Peer& pr, const std::vector<int32_t>& need, cudaStream_t s) {
  pr.n_send = (int64_t)need.size();
  if (!pr.n_send) return;
  for (int32_t g : need)
    if (g < d->a || g >= d->b) fail(LMS_E_STATE, "lms_dist_create: a peer asked for a vertex this rank does not own");
  pr.send_idx.alloc(pr.n_send, s);
  LMS_TRY_CUDA(cudaMemcpyAsync(pr.send_idx.p, need.data(), pr.n_send * sizeof(int32_t), cudaMemcpyHostToDevice, s));
  k_dist_to_local<<<gs(pr.n_send), 256, 0, s>>>(pr.send_idx.p, pr.n_send, d->lo - d->a);
  LMS_CHECK_LAUNCH();
  LMS_TRY_CUDA(cudaStreamSynchronize(s));  // `need` is a host temporary
}

static void finish(lms_dist_s* d, cudaStream_t s) {
  d->tot_send = d->tot_recv = 0;
  for (auto& pr : d->peers) {
    pr.soff = d->tot_send;
    pr.roff = d->tot_recv;
    d->tot_send += pr.n_send;
    d->tot_recv += pr.n_recv;
    pr.h_recv_global.clear();
    pr.h_recv_global.shrink_to_fit();
  }
  d->sbuf.alloc(std::max<int64_t>(d->tot_send * d->dim, 1), s);
  d->rbuf.alloc(std::max<int64_t>(d->tot_recv * d->dim, 1), s);
}

// NCCL: tell every owner which of its vertices this rank holds as ghosts
static void exchange_lists(lms_dist_s* d, cudaStream_t s) {
  NcclApi& N = nccl();
  const int P = d->nranks;
  DBuf<long long> scnt(std::max(P, 1), s), rcnt(std::max(P, 1), s);
  std::vector<long long> hs(P, 0), hr(P, 0);
  for (auto& pr : d->peers) hs[pr.q] = pr.n_recv;
  LMS_TRY_CUDA(cudaMemcpyAsync(scnt.p, hs.data(), P * sizeof(long long), cudaMemcpyHostToDevice, s));
  LMS_TRY_NCCL(N.GroupStart());
  for (auto& pr : d->peers) {
    LMS_TRY_NCCL(N.Send(scnt.p + pr.q, 1, ncclInt64, pr.q, d->comm, s));
    LMS_TRY_NCCL(N.Recv(rcnt.p + pr.q, 1, ncclInt64, pr.q, d->comm, s));
  }
  LMS_TRY_NCCL(N.GroupEnd());
  LMS_TRY_CUDA(cudaMemcpyAsync(hr.data(), rcnt.p, P * sizeof(long long), cudaMemcpyDeviceToHost, s));
  LMS_TRY_CUDA(cudaStreamSynchronize(s));
  int64_t tr = 0, ts = 0;
  for (auto& pr : d->peers) {
    tr += hr[pr.q];
    ts += pr.n_recv;
  }
  DBuf<int32_t> out(std::max<int64_t>(ts, 1), s), in(std::max<int64_t>(tr, 1), s);
  std::vector<int32_t> hout;
  hout.reserve(ts);
  for (auto& pr : d->peers) hout.insert(hout.end(), pr.h_recv_global.begin(), pr.h_recv_global.end());
  if (ts) LMS_TRY_CUDA(cudaMemcpyAsync(out.p, hout.data(), ts * sizeof(int32_t), cudaMemcpyHostToDevice, s));
  LMS_TRY_NCCL(N.GroupStart());
  int64_t oo = 0, io = 0;
  for (auto& pr : d->peers) {
    if (pr.n_recv) LMS_TRY_NCCL(N.Send(out.p + oo, pr.n_recv, ncclInt32, pr.q, d->comm, s));
    if (hr[pr.q]) LMS_TRY_NCCL(N.Recv(in.p + io, hr[pr.q], ncclInt32, pr.q, d->comm, s));
    oo += pr.n_recv;
    io += hr[pr.q];
  }
  LMS_TRY_NCCL(N.GroupEnd());
  std::vector<int32_t> hin(tr);
  if (tr) LMS_TRY_CUDA(cudaMemcpyAsync(hin.data(), in.p, tr * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  LMS_TRY_CUDA(cudaStreamSynchronize(s));
  io = 0;
  for (auto& pr : d->peers) {
    std::vector<int32_t> need(hin.begin() + io, hin.begin() + io + hr[pr.q]);
    set_send(d, pr, need, s);
    io += hr[pr.q];
  }
}

static void pack_all(lms_dist_s* d, cudaStream_t s) {
  for (auto& pr : d->peers)
    if (pr.n_send) halo_pack(d->local, pr.send_idx.p, pr.n_send, d->sbuf.p + pr.soff * d->dim, s);
}
static void unpack_all(lms_dist_s* d, cudaStream_t s) {
  for (auto& pr : d->peers)
    if (pr.n_recv) halo_unpack(d->local, pr.recv_idx.p, pr.n_recv, d->rbuf.p + pr.roff * d->dim, s);
}

static void exchange_nccl(lms_dist_s* d, cudaStream_t s) {
  if (d->nranks == 1) return;
  NcclApi& N = nccl();
  pack_all(d, s);
  LMS_TRY_NCCL(N.GroupStart());
  for (auto& pr : d->peers) {
    if (pr.n_send) LMS_TRY_NCCL(N.Send(d->sbuf.p + pr.soff * d->dim, pr.n_send * d->dim, ncclFloat64, pr.q, d->comm, s));
    if (pr.n_recv) LMS_TRY_NCCL(N.Recv(d->rbuf.p + pr.roff * d->dim, pr.n_recv * d->dim, ncclFloat64, pr.q, d->comm, s));
  }
  LMS_TRY_NCCL(N.GroupEnd());
  unpack_all(d, s);
}

// One pass on the rank's local mesh, without waiting for it: the sweep
// kernels' watchdog flag is read once per lms_smooth_dist call (end_passes),
// so the host enqueues the next exchange and pass while this one runs
// instead of paying a stream synchronisation (and the NCCL / pack launch
// latencies behind it) every pass.
static void local_pass(lms_dist_s* d, int p, cudaStream_t s) {
  lms_mesh_s* m = d->local;
  if (!m || m->n_free == 0) return;
  if (!m->sched.valid) {
    sync_soa(m, s);
    build_schedule(m, s);
  }
  m->coords_moved = true;
  const bool was = m->async_errors;
  m->async_errors = true;
  try {
    run_sweeps(m, p, s);
  } catch (...) {
    m->async_errors = was;
    throw;
  }
  m->async_errors = was;
}
static void end_passes(lms_dist_s* d, cudaStream_t s) {
  lms_mesh_s* m = d->local;
  if (m && m->n_free > 0 && !m->async_errors)
    check_err_flag(m, s, "lms_smooth_dist (sweep watchdog: a wait exceeded its budget)");
}

}  // namespace lms

using namespace lms;

extern "C" {

lms_status lms_nccl_unique_id(uint8_t out[128]) {
  try {
    if (!out) fail(LMS_E_ARG, "NULL argument");
    NcclApi& N = nccl();
    if (!N.ok) fail(LMS_E_NCCL, "NCCL unavailable: " + N.why);
    ncclUniqueId id;
    LMS_TRY_NCCL(N.GetUniqueId(&id));
    static_assert(sizeof(id.internal) == 128, "ncclUniqueId is 128 bytes");
    memcpy(out, id.internal, 128);
    return LMS_OK;
  } catch (const Err& e) {
    set_error(e.msg);
    return e.st;
  }
}

lms_status lms_dist_create(lms_mesh_t m, int32_t rank, int32_t nranks, const uint8_t nccl_uid[128],
                           int32_t sweeps_per_exchange, int32_t tile, lms_stream_t stream, lms_dist_t* out) {
  lms_dist_s* d = nullptr;
  try {
    if (!m || !out || !nccl_uid) fail(LMS_E_ARG, "NULL argument");
    if (nranks < 1 || rank < 0 || rank >= nranks) fail(LMS_E_ARG, "rank / nranks out of range");
    if (sweeps_per_exchange < 1 || sweeps_per_exchange > 8) fail(LMS_E_ARG, "sweeps_per_exchange must be in [1, 8]");
    DevGuard dg(m);
    NcclApi& N = nccl();
    if (!N.ok) fail(LMS_E_NCCL, "NCCL unavailable: " + N.why);
    cudaStream_t s = (cudaStream_t)stream;
    d = new lms_dist_s();
    d->device = m->device;
    d->rank = rank;
    d->nranks = nranks;
    d->P = sweeps_per_exchange;
    ncclUniqueId id;
    memcpy(id.internal, nccl_uid, 128);
    LMS_TRY_NCCL(N.CommInitRank(&d->comm, nranks, id, rank));
    plan_rank(m, d, tile, s);
    if (nranks > 1) exchange_lists(d, s);
    finish(d, s);
    *out = d;
    return LMS_OK;
  } catch (const Err& e) {
    delete d;
    set_error(e.msg);
    return e.st;
  }
}

lms_status lms_dist_replan(lms_dist_t d, lms_mesh_t m, int32_t tile, lms_stream_t stream) {
  try {
    if (!d || !m) fail(LMS_E_ARG, "NULL argument");
    if (d->local_group) fail(LMS_E_STATE, "lms_dist_replan: not for local-group handles");
    if (m->device != d->device) fail(LMS_E_ARG, "lms_dist_replan: the mesh is on another device");
    DevGuard dg(m);
    cudaStream_t s = (cudaStream_t)stream;
    LMS_TRY_CUDA(cudaStreamSynchronize(s));  // the previous plan's work is done before it is freed
    if (d->local) lms_mesh_destroy(d->local);
    d->local = nullptr;
    d->peers.clear();
    d->local_ids.release();
    plan_rank(m, d, tile, s);
    if (d->nranks > 1) exchange_lists(d, s);
    finish(d, s);
    return LMS_OK;
  } catch (const Err& e) {
    set_error(e.msg);
    return e.st;
  }
}

lms_status lms_dist_create_local(lms_mesh_t m, int32_t nranks, int32_t sweeps_per_exchange, int32_t tile,
                                 lms_stream_t stream, lms_dist_t* outs) {
  std::vector<lms_dist_s*> ds;
  try {
    if (!m || !outs) fail(LMS_E_ARG, "NULL argument");
    if (nranks < 1) fail(LMS_E_ARG, "nranks < 1");
    if (sweeps_per_exchange < 1 || sweeps_per_exchange > 8) fail(LMS_E_ARG, "sweeps_per_exchange must be in [1, 8]");
    DevGuard dg(m);
    cudaStream_t s = (cudaStream_t)stream;
    for (int r = 0; r < nranks; ++r) {
      lms_dist_s* d = new lms_dist_s();
      ds.push_back(d);
      d->device = m->device;
      d->rank = r;
      d->nranks = nranks;
      d->P = sweeps_per_exchange;
      d->local_group = true;
      plan_rank(m, d, tile, s);
    }
    // send side: what each peer holds as ghosts from me (the peers' recv lists)
    for (int r = 0; r < nranks; ++r)
      for (auto& pr : ds[r]->peers)
        for (auto& back : ds[pr.q]->peers)
          if (back.q == r) set_send(ds[r], pr, back.h_recv_global, s);
    for (auto* d : ds) finish(d, s);
    for (int r = 0; r < nranks; ++r) outs[r] = ds[r];
    return LMS_OK;
  } catch (const Err& e) {
    for (auto* d : ds) delete d;
    set_error(e.msg);
    return e.st;
  }
}

lms_status lms_smooth_dist(lms_dist_t d, int32_t sweeps, lms_stream_t stream) {
  try {
    if (!d) fail(LMS_E_ARG, "NULL handle");
    if (sweeps < 0) fail(LMS_E_ARG, "sweeps < 0");
    if (d->local_group && d->nranks > 1) fail(LMS_E_STATE, "a local-group handle steps with lms_smooth_dist_local");
    DevGuard dg(d->local);
    cudaStream_t s = (cudaStream_t)stream;
    for (int left = sweeps; left > 0;) {
      const int p = left < d->P ? left : d->P;
      exchange_nccl(d, s);
      local_pass(d, p, s);
      left -= p;
    }
    if (sweeps > 0) end_passes(d, s);
    return LMS_OK;
  } catch (const Err& e) {
    set_error(e.msg);
    return e.st;
  }
}

lms_status lms_smooth_dist_local(lms_dist_t* ds, int32_t nranks, int32_t sweeps, lms_stream_t stream) {
  try {
    if (!ds || nranks < 1) fail(LMS_E_ARG, "bad argument");
    if (sweeps < 0) fail(LMS_E_ARG, "sweeps < 0");
    for (int r = 0; r < nranks; ++r)
      if (!ds[r] || ds[r]->rank != r || ds[r]->nranks != nranks || !ds[r]->local_group)
        fail(LMS_E_ARG, "handles must be one local group, in rank order");
    DevGuard dg(ds[0]->local);
    cudaStream_t s = (cudaStream_t)stream;
    const int P = ds[0]->P;
    for (int left = sweeps; left > 0;) {
      const int p = left < P ? left : P;
      for (int r = 0; r < nranks; ++r) pack_all(ds[r], s);
      for (int r = 0; r < nranks; ++r)  // the "wire": device copies sender block -> receiver block
        for (auto& pr : ds[r]->peers) {
          if (!pr.n_recv) continue;
          const lms_dist_s* q = ds[pr.q];
          for (auto& back : q->peers)
            if (back.q == r) {
              if (back.n_send != pr.n_recv) fail(LMS_E_STATE, "local group: send/recv sizes differ");
              LMS_TRY_CUDA(cudaMemcpyAsync(ds[r]->rbuf.p + pr.roff * ds[r]->dim, q->sbuf.p + back.soff * q->dim,
                                           pr.n_recv * ds[r]->dim * sizeof(double), cudaMemcpyDeviceToDevice, s));
            }
        }
      for (int r = 0; r < nranks; ++r) unpack_all(ds[r], s);
      for (int r = 0; r < nranks; ++r) local_pass(ds[r], p, s);
      left -= p;
    }
    if (sweeps > 0)
      for (int r = 0; r < nranks; ++r) end_passes(ds[r], s);
    return LMS_OK;
  } catch (const Err& e) {
    set_error(e.msg);
    return e.st;
  }
}

lms_status lms_dist_export_owned(lms_dist_t d, double* const* d_out, int64_t* first, int64_t* count,
                                 lms_stream_t stream) {
  try {
    if (!d) fail(LMS_E_ARG, "NULL handle");
    DevGuard dg(d->local);
    if (first) *first = d->a;
    if (count) *count = d->b - d->a;
    if (d_out && d->b > d->a && d->local) {
      cudaStream_t s = (cudaStream_t)stream;
      sync_soa(d->local, s);
      for (int ax = 0; ax < d->dim; ++ax) {
        if (!d_out[ax]) fail(LMS_E_ARG, "NULL output pointer");
        LMS_TRY_CUDA(cudaMemcpyAsync(d_out[ax], d->local->x[ax].p + d->lo, (d->b - d->a) * sizeof(double),
                                     cudaMemcpyDefault, s));
      }
    }
    return LMS_OK;
  } catch (const Err& e) {
    set_error(e.msg);
    return e.st;
  }
}

lms_status lms_dist_info(lms_dist_t d, int64_t* n_local, int64_t* n_send, int64_t* n_recv, int32_t* n_peers,
                         int32_t* depth) {
  if (!d) return LMS_E_ARG;
  if (n_local) *n_local = d->n_local;
  if (n_send) *n_send = d->tot_send;
  if (n_recv) *n_recv = d->tot_recv;
  if (n_peers) {
    int c = 0;
    for (auto& pr : d->peers) c += (pr.n_send || pr.n_recv) ? 1 : 0;
    *n_peers = c;
  }
  if (depth) *depth = d->D;
  return LMS_OK;
}

lms_status lms_dist_export_local_ids(lms_dist_t d, int32_t* d_ids, lms_stream_t stream) {
  try {
    if (!d || !d_ids) fail(LMS_E_ARG, "NULL argument");
    DevGuard dg(d->local);
    if (d->n_local)
      LMS_TRY_CUDA(cudaMemcpyAsync(d_ids, d->local_ids.p, d->n_local * sizeof(int32_t), cudaMemcpyDefault,
                                   (cudaStream_t)stream));
    return LMS_OK;
  } catch (const Err& e) {
    set_error(e.msg);
    return e.st;
  }
}

void lms_dist_destroy(lms_dist_t d) {
  if (!d) return;
  DevGuard dg(d->local);
  cudaDeviceSynchronize();
  delete d;
}

}  // extern "C"
