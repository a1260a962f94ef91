// smooth.cu -- the LMS sweep (SURVEY 8(a) A8 schedule + A9 sweep kernels).
//
// Method: Eq. 1, p_v <- (1/N) sum_i p_i over the N
// neighbours of each interior vertex, applied inside Alg. 1's in-place loop
// (P:211-214).  The GPU replays the fixed colouring schedule (DESIGN.md
// reading Z1): for each sweep, for c = 0..C-1, all free colour-c vertices
// (pairwise non-adjacent, hence independent) are updated from the CURRENT
// coordinates.  Per vertex and axis: acc = x[u_0]; acc = acc + x[u_i] in CSR
// order; x[v] = acc / deg  -- IEEE binary64 adds and division (__dadd_rn,
// __ddiv_rn), no FMA, so the result is bit-identical to the CPU oracle.
//
// Work items: (tile k, colour c), tile = T consecutive storage positions; the
// schedule stores, item by item, the free vertices (ascending) and a copy of
// their CSR rows, so an item streams its rows contiguously.
//
// S1: one kernel per colour (C launches per sweep, captured once into a CUDA
//     graph); inside a colour no address that is read is written, so gathers
//     use the read-only path.
// S3: ONE persistent launch for all sweeps.  Items are taken from an atomic
//     ticket in the order key(s, c, k) = s*(K + (C-1)L)*C + (k + cL)*C + c
//     ("S3a": colours pipelined inside each sweep, lag L > max tile reach).
//     Item (sigma = sC + c, k) waits until every tile k' in k's dependency
//     range [klo, khi] has completed sigma stages (prog[k'] >= sigma), computes,
//     then publishes prog[k] = sigma + 1 (release).  Any two adjacent tiles are
//     then at most one stage apart, which enforces every read-after-write and
//     write-after-read dependency of the sequential colour schedule, so S3 is
//     bit-identical to S1.  Tickets are issued in a topological order, so the
//     kernel is deadlock-free for any grid size.  Colour c of tile k runs while
//     colour c-1's data of the nearby tiles is still in L2: each coordinate is
//     fetched from HBM about once per sweep instead of about C times (S1).
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_reduce.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <algorithm>

#include "lms_internal.cuh"

namespace lms {

// ---------------------------------------------------------------- schedule build
__global__ void k_free_flags(const uint8_t* __restrict__ fixed, int64_t V, uint8_t* flags, int32_t* ids) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < V; v += (int64_t)gridDim.x * blockDim.x) {
    flags[v] = fixed[v] ? 0 : 1;
    ids[v] = (int32_t)v;
  }
}

__global__ void k_item_ptr(const uint32_t* __restrict__ skeys, int64_t n, int64_t nitems, int32_t* item_ptr) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = skeys[i];
    int64_t rprev = (i == 0) ? -1 : (int64_t)skeys[i - 1];
    for (int64_t q = rprev + 1; q <= r; ++q) item_ptr[q] = (int32_t)i;
    if (i == n - 1)
      for (int64_t q = r + 1; q <= nitems; ++q) item_ptr[q] = (int32_t)n;
  }
}

__global__ void k_slot_deg(const int32_t* __restrict__ sv, int64_t n, const int32_t* __restrict__ rp, int32_t* deg) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= n; i += (int64_t)gridDim.x * blockDim.x)
    deg[i] = (i < n) ? rp[sv[i] + 1] - rp[sv[i]] : 0;
}

__global__ void k_range_init(int32_t* klo, int32_t* khi, int64_t K) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < K; k += (int64_t)gridDim.x * blockDim.x)
    klo[k] = khi[k] = (int32_t)k;
}

__global__ void k_reach(const int32_t* __restrict__ klo, const int32_t* __restrict__ khi, int64_t K, int* out) {
  int r = 0;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < K; k += (int64_t)gridDim.x * blockDim.x)
    r = max(r, max(khi[k] - (int)k, (int)k - klo[k]));
  for (int o = 16; o; o >>= 1) r = max(r, __shfl_down_sync(0xffffffffu, r, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, r);
}


// ---------------------------------------------------------------- tiling
// Tiles group free vertices into work items (tile, colour).  Two tilings:
//  STORAGE: tile = T consecutive storage positions (the processing order then
//           follows the ordering, as in the paper's storage-order loop);
//  SPATIAL: tile = a cell of a regular grid of bins over the initial
//           coordinates' bounding box (~T vertices per cell; cells numbered
//           row-major, so a tile's neighbours are within +-(cells per row + 1)).
//           A colour pass over a compact cell re-reads only the cell plus a
//           one-ring halo from L2, instead of three full rows for a row-major
//           storage tile.  The tiling is a scheduling device only: results do
//           not depend on it (every tiling replays the same colour schedule).
__global__ void k_tile_storage(int64_t V, int T, int32_t* tile_of) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < V; v += (int64_t)gridDim.x * blockDim.x)
    tile_of[v] = (int32_t)(v / T);
}

__global__ void k_tile_spatial(int64_t V, int dim, const double* __restrict__ x, const double* __restrict__ y,
                               const double* __restrict__ z, double x0, double y0, double z0, double sx, double sy,
                               double sz, int nbx, int nby, int nbz, int32_t* tile_of) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < V; v += (int64_t)gridDim.x * blockDim.x) {
    int bx = (int)((x[v] - x0) * sx), by = (int)((y[v] - y0) * sy), bz = 0;
    bx = bx < 0 ? 0 : (bx >= nbx ? nbx - 1 : bx);
    by = by < 0 ? 0 : (by >= nby ? nby - 1 : by);
    if (dim == 3) {
      bz = (int)((z[v] - z0) * sz);
      bz = bz < 0 ? 0 : (bz >= nbz ? nbz - 1 : bz);
    }
    tile_of[v] = (bz * nby + by) * nbx + bx;
  }
}

__global__ void k_item_keys2(const int32_t* __restrict__ fv, int64_t n, const int8_t* __restrict__ colour,
                             const int32_t* __restrict__ tile_of, int C, uint32_t* keys) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t v = fv[i];
    keys[i] = (uint32_t)tile_of[v] * (uint32_t)C + (uint32_t)colour[v];
  }
}

// rows of the slots (schedule CSR) and the (tile, neighbour tile) dependency pairs
__global__ void k_slot_rows2(const int32_t* __restrict__ sv, int64_t n, const int32_t* __restrict__ rp,
                             const int32_t* __restrict__ col, const int32_t* __restrict__ sptr,
                             const uint8_t* __restrict__ fixed, const int32_t* __restrict__ tile_of,
                             int32_t* __restrict__ scol, unsigned long long* dep, int cap, int* ndep) {
  const int lane = threadIdx.x & 31;
  const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = w; i < n; i += nw) {
    const int32_t v = sv[i], b = rp[v], d = rp[v + 1] - b, o = sptr[i];
    const int32_t k = tile_of[v];
    for (int32_t j = lane; j < d; j += 32) {
      const int32_t u = col[b + j];
      scol[o + j] = u;
      if (!fixed[u]) {
        const int32_t ku = tile_of[u];
        if (ku != k) {
          const int p = atomicAdd(ndep, 1);
          if (p < cap) dep[p] = ((unsigned long long)(uint32_t)k << 32) | (uint32_t)ku;
        }
      }
    }
  }
}

// unique sorted (k, k') pairs -> per-tile dependency CSR (self excluded) + [klo, khi]
__global__ void k_dep_csr(const unsigned long long* __restrict__ ud, int nd, int64_t K, int32_t* tdep_ptr,
                          int32_t* tdep, int32_t* klo, int32_t* khi) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nd; i += gridDim.x * blockDim.x) {
    const int64_t k = (int64_t)(ud[i] >> 32);
    const int32_t k2 = (int32_t)(ud[i] & 0xffffffffull);
    tdep[i] = k2;
    const int64_t kprev = (i == 0) ? -1 : (int64_t)(ud[i - 1] >> 32);
    for (int64_t q = kprev + 1; q <= k; ++q) tdep_ptr[q] = i;
    if (i == nd - 1)
      for (int64_t q = k + 1; q <= K; ++q) tdep_ptr[q] = nd;
    atomicMin(&klo[k], k2);
    atomicMax(&khi[k], k2);
  }
}

// per item: width W = max row length and slab size (chunks * 32 * (1 + W) ints)
__global__ void k_item_width(const int32_t* __restrict__ item_ptr, const int32_t* __restrict__ sptr, int64_t nitems,
                             int32_t* iw, long long* isz) {
  for (int64_t it = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; it < nitems;
       it += (int64_t)gridDim.x * blockDim.x) {
    int32_t w = 1;
    for (int32_t s = item_ptr[it]; s < item_ptr[it + 1]; ++s) w = max(w, sptr[s + 1] - sptr[s]);
    const long long nch = (item_ptr[it + 1] - item_ptr[it] + 31) >> 5;
    iw[it] = w;
    isz[it] = nch * 32 * (1 + w);
  }
}

// fill the slab: one warp per item, lane = slot within a chunk
__global__ void k_fill_slab(const int32_t* __restrict__ item_ptr, const int32_t* __restrict__ sv,
                            const int32_t* __restrict__ sptr, const int32_t* __restrict__ scol,
                            const long long* __restrict__ ioff, const int32_t* __restrict__ iw, int64_t nitems,
                            int32_t* slab) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t it = w0; it < nitems; it += nw) {
    const int32_t a = item_ptr[it], b = item_ptr[it + 1], W = iw[it];
    for (int32_t q = 0; a + q * 32 < b; ++q) {
      int32_t* ch = slab + ioff[it] + (long long)q * 32 * (1 + W);
      const int32_t s = a + q * 32 + lane;
      const bool ok = s < b;
      ch[lane] = ok ? sv[s] : -1;
      const int32_t d = ok ? sptr[s + 1] - sptr[s] : 0;
      for (int32_t w = 0; w < W; ++w) ch[32 + w * 32 + lane] = (w < d) ? scol[sptr[s] + w] : -1;
    }
  }
}

__global__ void k_tile_prefix(const int32_t* __restrict__ item_ptr, int64_t K, int C, int32_t* tpre) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < K; k += (int64_t)gridDim.x * blockDim.x) {
    int32_t acc = 0;
    for (int c = 0; c < C; ++c) {
      tpre[k * (C + 1) + c] = acc;
      acc += (item_ptr[k * C + c + 1] - item_ptr[k * C + c] + 31) >> 5;
    }
    tpre[k * (C + 1) + C] = acc;
  }
}

// 128-byte item record, read by the S3 dispatcher in one round trip:
// [0] chunks [1] W [2..3] slab offset [4] nd [5] pad, then nd <= REC_DEPS pairs
// (tile k', N(k') | P(k', c) << 16) for the item's tile itself and every
// neighbour tile; nd = 0 -> too many / too large: the kernel uses tdep + tpre.
constexpr int REC_INTS = 32;
constexpr int REC_DEPS = 13;
__global__ void k_item_records(const int32_t* __restrict__ item_ptr, const long long* __restrict__ ioff,
                               const int32_t* __restrict__ iw, const int32_t* __restrict__ tdep_ptr,
                               const int32_t* __restrict__ tdep, const int32_t* __restrict__ tpre, int64_t K, int C,
                               int32_t* irec) {
  for (int64_t it = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; it < K * C; it += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = it / C;
    const int c = (int)(it - k * C);
    int32_t* r = irec + it * REC_INTS;
    r[0] = (item_ptr[it + 1] - item_ptr[it] + 31) >> 5;
    r[1] = iw[it];
    r[2] = (int32_t)(ioff[it] & 0xffffffffll);
    r[3] = (int32_t)(ioff[it] >> 32);
    const int32_t b = tdep_ptr[k], e = tdep_ptr[k + 1];
    int nd = 1 + (e - b);
    bool fits = nd <= REC_DEPS;
    auto np = [&](int64_t kt) -> int32_t { return tpre[kt * (C + 1) + C] | (tpre[kt * (C + 1) + c] << 16); };
    auto small = [&](int64_t kt) { return tpre[kt * (C + 1) + C] < 65536; };
    fits = fits && small(k);
    for (int32_t q = b; fits && q < e; ++q) fits = small(tdep[q]);
    r[4] = fits ? nd : 0;
    r[5] = 0;
    for (int q = 0; q < 2 * REC_DEPS; ++q) r[6 + q] = 0;
    if (fits) {
      r[6] = (int32_t)k;
      r[7] = np(k);
      for (int32_t q = b; q < e; ++q) {
        r[6 + 2 * (1 + q - b)] = tdep[q];
        r[7 + 2 * (1 + q - b)] = np(tdep[q]);
      }
    }
  }
}

// Spatial tiling: tile = cell of a regular grid of bins over the bounding box
// of the current coordinates, ~T vertices per cell, numbered row-major
// (x fastest).  Returns the number of cells K.
int64_t spatial_tiles(lms_mesh_s* m, int T, int32_t* tile_of, cudaStream_t s) {
  sync_soa(m, s);
  const int64_t V = m->V;
  const unsigned Gv = grid_for(V, 256) > 8192 ? 8192 : grid_for(V, 256);
  int64_t K = 0;
    double lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
    {
      DBuf<double> r(2, s);
      size_t tb = 0;
      LMS_TRY_CUDA(cub::DeviceReduce::Min(nullptr, tb, m->x[0].p, r.p, V, s));
      DBuf<char> tmp(tb, s);
      for (int a = 0; a < m->dim; ++a) {
        size_t t2 = tb;
        LMS_TRY_CUDA(cub::DeviceReduce::Min(tmp.p, t2, m->x[a].p, r.p, V, s));
        t2 = tb;
        LMS_TRY_CUDA(cub::DeviceReduce::Max(tmp.p, t2, m->x[a].p, r.p + 1, V, s));
        double h[2];
        LMS_TRY_CUDA(cudaMemcpyAsync(h, r.p, sizeof(h), cudaMemcpyDeviceToHost, s));
        LMS_TRY_CUDA(cudaStreamSynchronize(s));
        lo[a] = h[0];
        hi[a] = h[1];
      }
    }
    double w[3];
    for (int a = 0; a < 3; ++a) w[a] = (a < m->dim && hi[a] > lo[a] && std::isfinite(hi[a] - lo[a])) ? hi[a] - lo[a] : 1.0;
    const double cells = (double)V / (double)T > 1.0 ? (double)V / (double)T : 1.0;
    int nb[3] = {1, 1, 1};
    if (m->dim == 2) {
      const double h = std::sqrt(w[0] * w[1] / cells);
      nb[0] = (int)std::max(1.0, std::round(w[0] / h));
      nb[1] = (int)std::max(1.0, std::round(w[1] / h));
    } else {
      const double h = std::cbrt(w[0] * w[1] * w[2] / cells);
      for (int a = 0; a < 3; ++a) nb[a] = (int)std::max(1.0, std::round(w[a] / h));
    }
    K = (int64_t)nb[0] * nb[1] * nb[2];
    k_tile_spatial<<<Gv, 256, 0, s>>>(V, m->dim, m->x[0].p, m->x[1].p, m->dim == 3 ? m->x[2].p : nullptr, lo[0],
                                      lo[1], lo[2], nb[0] / w[0], nb[1] / w[1], nb[2] / w[2], nb[0], nb[1], nb[2],
                                      tile_of);
    LMS_CHECK_LAUNCH();
  return K;
}

static int s3_ctas(int dev) {
  int nsm = 0;
  LMS_TRY_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  int per = 1;  // 1024-thread CTAs per SM (LMS_S3_CTAS_PER_SM overrides, for tuning)
  if (const char* e = getenv("LMS_S3_CTAS_PER_SM")) per = atoi(e) > 0 ? atoi(e) : per;
  return nsm * per;
}

// The S1/S3 schedule (item lists, slab, dependency records).  With gz_base the
// kernel choice stays GZ and only the S1 lists that lms_smooth_colour uses are
// (re)built.
static void build_base(lms_mesh_s* m, cudaStream_t s, bool gz_base) {
  Schedule& S = m->sched;
  for (int i = 0; i < 2; ++i)
    if (S.graphs[i]) { cudaGraphExecDestroy(S.graphs[i]); S.graphs[i] = nullptr; }
  const int64_t V = m->V;
  const int C = m->C > 0 ? m->C : 1;
  const bool want_s3 = !gz_base && m->sched_req == LMS_SCHED_S3;
  // tiling: S3 defaults to spatial cells of ~4096 vertices; S1 to storage tiles
  // of ~256*C vertices (one vertex per thread of a 256-thread CTA per item)
  // S2 (3D): spatial boxes, ~4 per SM (the persistent S2 kernel gives each
  // CTA consecutive boxes, so its chunks' neighbourhoods overlap in L1)
  const bool want_s2 = !gz_base && (m->sched_req == LMS_SCHED_S2 || (m->sched_req == LMS_SCHED_AUTO && m->dim == 3));
  int tiling = m->tiling_req;
  if (tiling == LMS_TILING_AUTO) tiling = (want_s3 || want_s2) ? LMS_TILING_SPATIAL : LMS_TILING_STORAGE;
  int T = m->tile_req;
  if (T == 0 && want_s2) {
    int nsm = 148;
    LMS_TRY_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, m->device));
    int per = 8;  // tiles per SM (LMS_S2_TILES_PER_SM tunes)
    if (const char* e = getenv("LMS_S2_TILES_PER_SM")) per = std::max(1, atoi(e));
    T = (int)std::max<int64_t>(256, std::min<int64_t>(1 << 20, V / (per * (int64_t)nsm)));
  }
  if (T == 0) T = want_s3 ? 4096 : 256 * C;
  if (T > V) T = (int)((V + 31) / 32 * 32);
  if (T < 32) T = 32;
  const unsigned Gv = grid_for(V, 256) > 8192 ? 8192 : grid_for(V, 256);
  DBuf<int32_t> tile_of(V, s);
  int64_t K = 0;
  if (tiling == LMS_TILING_SPATIAL) {
    K = spatial_tiles(m, T, tile_of.p, s);
  } else {
    K = (V + T - 1) / T;
    k_tile_storage<<<Gv, 256, 0, s>>>(V, T, tile_of.p);
    LMS_CHECK_LAUNCH();
  }
  if (K * (int64_t)C >= ((int64_t)1 << 31) - 1) fail(LMS_E_ARG, "too many schedule items");
  S.tiling = tiling;
  S.tile = T;
  S.K = K;
  // free vertices in ascending storage order
  DBuf<int32_t> fv(V, s);
  DBuf<int> nsel(1, s);
  {
    DBuf<uint8_t> flags(V, s);
    DBuf<int32_t> ids(V, s);
    k_free_flags<<<Gv, 256, 0, s>>>(m->fixed.p, V, flags.p, ids.p);
    LMS_CHECK_LAUNCH();
    size_t tb = 0;
    LMS_TRY_CUDA(cub::DeviceSelect::Flagged(nullptr, tb, ids.p, flags.p, fv.p, nsel.p, V, s));
    DBuf<char> tmp(tb, s);
    LMS_TRY_CUDA(cub::DeviceSelect::Flagged(tmp.p, tb, ids.p, flags.p, fv.p, nsel.p, V, s));
  }
  int hn = 0;
  LMS_TRY_CUDA(cudaMemcpyAsync(&hn, nsel.p, sizeof(int), cudaMemcpyDeviceToHost, s));
  LMS_TRY_CUDA(cudaStreamSynchronize(s));
  const int64_t n = hn;
  S.n_free = n;
  const int64_t nitems = K * C;
  S.item_ptr.alloc(nitems + 1, s);
  S.sv.alloc(n > 0 ? n : 1, s);
  S.sptr.alloc(n + 1, s);
  S.klo.alloc(K, s);
  S.khi.alloc(K, s);
  S.prog.alloc(K, s);
  S.ticket.alloc(1, s);
  S.tdep_ptr.alloc(K + 1, s);
  k_range_init<<<grid_for(K, 256) > 4096 ? 4096 : grid_for(K, 256), 256, 0, s>>>(S.klo.p, S.khi.p, K);
  LMS_CHECK_LAUNCH();
  int nd = 0;
  if (n > 0) {
    const unsigned Gn = grid_for(n, 256) > 8192 ? 8192 : grid_for(n, 256);
    DBuf<uint32_t> keys(n, s), skeys(n, s);
    k_item_keys2<<<Gn, 256, 0, s>>>(fv.p, n, m->colour.p, tile_of.p, C, keys.p);
    LMS_CHECK_LAUNCH();
    int kb = 1;
    while (((int64_t)1 << kb) < nitems) ++kb;
    size_t tb = 0;
    LMS_TRY_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, keys.p, skeys.p, fv.p, S.sv.p, n, 0, kb, s));
    {
      DBuf<char> tmp(tb, s);
      LMS_TRY_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tb, keys.p, skeys.p, fv.p, S.sv.p, n, 0, kb, s));
    }
    k_item_ptr<<<Gn, 256, 0, s>>>(skeys.p, n, nitems, S.item_ptr.p);
    LMS_CHECK_LAUNCH();
    DBuf<int32_t> deg(n + 1, s);
    const unsigned Gn1 = grid_for(n + 1, 256) > 8192 ? 8192 : grid_for(n + 1, 256);
    k_slot_deg<<<Gn1, 256, 0, s>>>(S.sv.p, n, m->row_ptr.p, deg.p);
    LMS_CHECK_LAUNCH();
    tb = 0;
    LMS_TRY_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, deg.p, S.sptr.p, n + 1, s));
    {
      DBuf<char> tmp(tb, s);
      LMS_TRY_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tb, deg.p, S.sptr.p, n + 1, s));
    }
    int nnzf = 0;
    LMS_TRY_CUDA(cudaMemcpyAsync(&nnzf, S.sptr.p + n, sizeof(int), cudaMemcpyDeviceToHost, s));
    LMS_TRY_CUDA(cudaStreamSynchronize(s));
    S.scol.alloc(nnzf > 0 ? nnzf : 1, s);
    // dependency pairs: at most one per schedule entry
    const int cap = nnzf > 0 ? nnzf : 1;
    DBuf<unsigned long long> dep(cap, s), dep2(cap, s);
    DBuf<int> ndep(1, s);
    LMS_TRY_CUDA(cudaMemsetAsync(ndep.p, 0, sizeof(int), s));
    const unsigned Gw = grid_for(n * 32, 256) > 8192 ? 8192 : grid_for(n * 32, 256);
    k_slot_rows2<<<Gw, 256, 0, s>>>(S.sv.p, n, m->row_ptr.p, m->col.p, S.sptr.p, m->fixed.p, tile_of.p, S.scol.p,
                                    dep.p, cap, ndep.p);
    LMS_CHECK_LAUNCH();
    int hnd = 0;
    LMS_TRY_CUDA(cudaMemcpyAsync(&hnd, ndep.p, sizeof(int), cudaMemcpyDeviceToHost, s));
    LMS_TRY_CUDA(cudaStreamSynchronize(s));
    int kb2 = 1;
    while (((int64_t)1 << kb2) < K) ++kb2;
    if (hnd > 0) {
      tb = 0;
      LMS_TRY_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tb, dep.p, dep2.p, hnd, 0, 32 + kb2, s));
      DBuf<char> tmp(tb, s);
      LMS_TRY_CUDA(cub::DeviceRadixSort::SortKeys(tmp.p, tb, dep.p, dep2.p, hnd, 0, 32 + kb2, s));
      DBuf<int> nu(1, s);
      size_t tb2 = 0;
      LMS_TRY_CUDA(cub::DeviceSelect::Unique(nullptr, tb2, dep2.p, dep.p, nu.p, hnd, s));
      DBuf<char> tmp2(tb2, s);
      LMS_TRY_CUDA(cub::DeviceSelect::Unique(tmp2.p, tb2, dep2.p, dep.p, nu.p, hnd, s));
      LMS_TRY_CUDA(cudaMemcpyAsync(&nd, nu.p, sizeof(int), cudaMemcpyDeviceToHost, s));
      LMS_TRY_CUDA(cudaStreamSynchronize(s));
    }
    S.tdep.alloc(nd > 0 ? nd : 1, s);
    if (nd > 0) {
      k_dep_csr<<<grid_for(nd, 256) > 4096 ? 4096 : grid_for(nd, 256), 256, 0, s>>>(dep.p, nd, K, S.tdep_ptr.p,
                                                                                   S.tdep.p, S.klo.p, S.khi.p);
      LMS_CHECK_LAUNCH();
    }
  } else {
    LMS_TRY_CUDA(cudaMemsetAsync(S.item_ptr.p, 0, (nitems + 1) * sizeof(int32_t), s));
    S.tdep.alloc(1, s);
  }
  if (nd == 0) LMS_TRY_CUDA(cudaMemsetAsync(S.tdep_ptr.p, 0, (K + 1) * sizeof(int32_t), s));
  // slab layout for S3 (fixed per-item width, column-major 32-slot chunks)
  S.iw.alloc(nitems > 0 ? nitems : 1, s);
  S.ioff.alloc(nitems + 1, s);
  {
    DBuf<long long> isz(nitems + 1, s);
    LMS_TRY_CUDA(cudaMemsetAsync(isz.p, 0, (nitems + 1) * sizeof(long long), s));
    if (n > 0) {
      k_item_width<<<grid_for(nitems, 256) > 4096 ? 4096 : grid_for(nitems, 256), 256, 0, s>>>(
          S.item_ptr.p, S.sptr.p, nitems, S.iw.p, isz.p);
      LMS_CHECK_LAUNCH();
    }
    size_t tb = 0;
    LMS_TRY_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, isz.p, S.ioff.p, nitems + 1, s));
    DBuf<char> tmp(tb, s);
    LMS_TRY_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tb, isz.p, S.ioff.p, nitems + 1, s));
    long long slab_n = 0;
    LMS_TRY_CUDA(cudaMemcpyAsync(&slab_n, S.ioff.p + nitems, sizeof(long long), cudaMemcpyDeviceToHost, s));
    LMS_TRY_CUDA(cudaStreamSynchronize(s));
    S.slab.alloc(slab_n > 0 ? slab_n : 1, s);
    if (n > 0) {
      const unsigned Gw = grid_for(nitems * 32, 256) > 8192 ? 8192 : grid_for(nitems * 32, 256);
      k_fill_slab<<<Gw, 256, 0, s>>>(S.item_ptr.p, S.sv.p, S.sptr.p, S.scol.p, S.ioff.p, S.iw.p, nitems, S.slab.p);
      LMS_CHECK_LAUNCH();
    }
  }
  S.tpre.alloc(K * (C + 1), s);
  k_tile_prefix<<<grid_for(K, 256) > 4096 ? 4096 : grid_for(K, 256), 256, 0, s>>>(S.item_ptr.p, K, C, S.tpre.p);
  LMS_CHECK_LAUNCH();
  S.irec.alloc(nitems > 0 ? nitems * REC_INTS : REC_INTS, s);
  if (nitems > 0) {
    k_item_records<<<grid_for(nitems, 256) > 4096 ? 4096 : grid_for(nitems, 256), 256, 0, s>>>(
        S.item_ptr.p, S.ioff.p, S.iw.p, S.tdep_ptr.p, S.tdep.p, S.tpre.p, K, C, S.irec.p);
    LMS_CHECK_LAUNCH();
  }
  DBuf<int> reach(1, s);
  LMS_TRY_CUDA(cudaMemsetAsync(reach.p, 0, sizeof(int), s));
  k_reach<<<grid_for(K, 256) > 1024 ? 1024 : grid_for(K, 256), 256, 0, s>>>(S.klo.p, S.khi.p, K, reach.p);
  LMS_CHECK_LAUNCH();
  int hr = 0;
  LMS_TRY_CUDA(cudaMemcpyAsync(&hr, reach.p, sizeof(int), cudaMemcpyDeviceToHost, s));
  LMS_TRY_CUDA(cudaStreamSynchronize(s));
  S.max_reach = hr;
  S.base_valid = true;
  if (gz_base) return;
  // resolve the kernel: S3 pays off when the tile graph is banded (small reach)
  int kind = m->sched_req;
  // AUTO beyond GZ: S2 for 3D (C3: BFS 192 vs 195 us, RDR 196 vs 262 us per
  // sweep against S1; S3 slower under every ordering), else S1
  if (kind == LMS_SCHED_AUTO) kind = m->dim == 3 ? LMS_SCHED_S2 : LMS_SCHED_S1;
  S.kind = kind;
  if (kind == LMS_SCHED_S3) {
    const int ctas = s3_ctas(m->device);
    int lag_extra = 6;  // tickets in flight per CTA -> keys of slack; LMS_S3_LAG_PER_CTA tunes
    if (const char* e = getenv("LMS_S3_LAG_PER_CTA")) lag_extra = atoi(e);
    int L = hr + 1 + (lag_extra * ctas + C - 1) / C;
    if (m->lag_req > 0) L = m->lag_req > hr ? m->lag_req : hr + 1;  // must exceed the reach
    S.lag = L;
  } else {
    S.lag = 0;
  }
  S.valid = true;
}

void build_schedule(lms_mesh_s* m, cudaStream_t s) {
  Schedule& S = m->sched;
  S.valid = false;
  S.base_valid = false;
  S.s2_choff.release();  // S2 chunk lists belong to the previous schedule
  S.s2d_cv.release();
  S.s2_chw.release();
  S.s2_crange.release();
  S.s2_nbptr.release();
  S.s2_nb.release();
  S.s2_prog.release();
  if (m->sched_req == LMS_SCHED_JACOBI) {  // N3 variant (jacobi.cu): no schedule tables
    S.kind = LMS_SCHED_JACOBI;
    S.valid = true;
    return;
  }
  // GZ (gz.cu): the default for 2D meshes with few colours, where the
  // C-hop ghost zone of a tile is a small fraction of it
  if (m->sched_req == LMS_SCHED_GZ || (m->sched_req == LMS_SCHED_AUTO && m->dim == 2 && m->C <= 8)) {
    int Tg = m->tile_req > 0 ? m->tile_req : (m->dim == 2 ? 4096 : 512);
    // few tiles per SM (under 2 at T = 4096): one tile per SM, T = V / SMs
    // within [1024, 8192] (C2 1024^2: 26.3 -> 24.6 us per sweep; the
    // paper-scale CP has 91 tiles at T = 4096, a third of the SMs idle; the
    // builder still shrinks T until two region buffers fit)
    if (m->tile_req == 0 && m->dim == 2) {
      int nsm = 148;
      LMS_TRY_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, m->device));
      // ~nsm - 4 tiles: the kd balancer then finds a near-square count at
      // or below the SM count (148 itself factors badly and doubles to 294)
      if (m->V / 4096 < 2 * (int64_t)nsm)
        Tg = (int)std::max<int64_t>(1024, std::min<int64_t>(8192, (m->V + nsm - 5) / (nsm - 4)));
    }
    int P = (m->sched_req == LMS_SCHED_GZ && m->lag_req > 0) ? m->lag_req : 1;
    // AUTO on small 2D meshes: several sweeps per pass, the per-pass region
    // staging and stage ramp paid once for P sweeps (CP, the paper-scale
    // 372 K-vertex mesh: 18.4 -> 12.3 us per sweep at P = 2; C1 (10 K):
    // 14.3 -> 8.6 at P = 4; C2 (1 M): P = 1 stays best)
    if (m->sched_req == LMS_SCHED_AUTO && m->dim == 2 && m->lag_req == 0 && !getenv("LMS_GZ_P1"))
      P = m->V < (1 << 15) ? 4 : (m->V < (1 << 19) ? 2 : 1);
    if (build_gz(m, Tg, P, m->sched_req == LMS_SCHED_GZ, s)) {
      S.kind = LMS_SCHED_GZ;
      S.lag = 0;
      S.valid = true;
      return;
    }
  }
  build_base(m, s, false);
}

// ---------------------------------------------------------------- sweep kernels
// Tuning options (bit mask; default OPT_DEFAULT, LMS_OPTS env overrides for experiments)
enum : int {
  OPT_HINT_STREAM = 1,   // schedule loads: ld.nc.L1::no_allocate + L2 evict_first
  OPT_HINT_COORD = 2,    // coordinate loads/stores: L2 evict_last
  OPT_STAGE = 4,         // warp-cooperative coalesced staging of column indices in smem
  OPT_GB8 = 8,           // 8 gathers in flight per lane (else 4)
};
constexpr int OPT_DEFAULT = 0;

// L2 cache policies: the schedule (sv, sptr, scol) is streamed once per sweep
// -> evict_first; coordinates are re-read by the next colours -> evict_last.
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
// read-only schedule data (never written during a sweep)
template <int opts>
__device__ __forceinline__ int32_t ld_stream(const int32_t* p, uint64_t pol) {
  int32_t v;
  if (opts & OPT_HINT_STREAM)
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
  else
    v = __ldg(p);
  return v;
}
// coordinates: RO = true (S1: nothing read in a colour pass is written in it)
// uses the non-coherent path; RO = false (S3) uses coherent L1-cached loads,
// valid because every item starts after a gpu-scope acquire (L1 invalidated)
template <bool RO, int opts>
__device__ __forceinline__ double ld_coord(const double* p, uint64_t pol) {
  double v;
  if (opts & OPT_HINT_COORD) {
    if (RO)
      asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
    else
      asm volatile("ld.global.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol) : "memory");
  } else {
    if (RO)
      v = __ldg(p);
    else
      asm volatile("ld.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
  }
  return v;
}
template <int opts>
__device__ __forceinline__ void st_coord(double* p, double v, uint64_t pol) {
  if (opts & OPT_HINT_COORD)
    asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(pol) : "memory");
  else
    *p = v;
}

constexpr int WBUF = 512;  // per-warp staged column indices (ints)

// Eq. 1 for one vertex: neighbours idx[0..d), sums in CSR order, IEEE division.
template <int DIM, bool RO, int GB, int opts, typename IDX>
__device__ __forceinline__ void lms_vertex(int32_t v, int d, IDX idx, double* x, double* y, double* z,
                                           uint64_t keep) {
  double sx = 0.0, sy = 0.0, sz = 0.0;
  for (int i0 = 0; i0 < d; i0 += GB) {
    const int cnt = d - i0 < GB ? d - i0 : GB;
    int32_t u[GB];
    double gx[GB], gy[GB], gz[GB];
#pragma unroll
    for (int i = 0; i < GB; ++i)
      if (i < cnt) u[i] = idx(i0 + i);
#pragma unroll
    for (int i = 0; i < GB; ++i)
      if (i < cnt) {
        gx[i] = ld_coord<RO, opts>(x + u[i], keep);
        gy[i] = ld_coord<RO, opts>(y + u[i], keep);
        if (DIM == 3) gz[i] = ld_coord<RO, opts>(z + u[i], keep);
      }
#pragma unroll
    for (int i = 0; i < GB; ++i)
      if (i < cnt) {
        if (i0 + i == 0) {
          sx = gx[i]; sy = gy[i];
          if (DIM == 3) sz = gz[i];
        } else {
          sx = __dadd_rn(sx, gx[i]);
          sy = __dadd_rn(sy, gy[i]);
          if (DIM == 3) sz = __dadd_rn(sz, gz[i]);
        }
      }
  }
  const double dd = (double)d;
  st_coord<opts>(x + v, __ddiv_rn(sx, dd), keep);
  st_coord<opts>(y + v, __ddiv_rn(sy, dd), keep);
  if (DIM == 3) st_coord<opts>(z + v, __ddiv_rn(sz, dd), keep);
}

template <int DIM, bool RO, int opts, typename IDX>
__device__ __forceinline__ void lms_vertex_any(int32_t v, int d, IDX idx, double* x, double* y, double* z,
                                               uint64_t keep) {
  lms_vertex<DIM, RO, (opts & OPT_GB8) ? 8 : 4, opts>(v, d, idx, x, y, z, keep);
}

// Eq. 1 for one vertex in three explicit phases so that only two dependent
// memory round trips follow the slot load: (1) all column indices of the row
// (up to NI, predicated), (2) all gathers of a batch, (3) ordered sums.
template <int DIM, bool RO, int NI, int GB, int opts>
__device__ __forceinline__ void lms_vertex_phased(int32_t v, int32_t j0, int d, const int32_t* __restrict__ scol,
                                                  double* x, double* y, double* z, uint64_t stream, uint64_t keep) {
  int32_t u[NI];
#pragma unroll
  for (int i = 0; i < NI; ++i) u[i] = (i < d) ? ld_stream<opts>(scol + j0 + i, stream) : 0;
  double sx = 0.0, sy = 0.0, sz = 0.0;
#pragma unroll
  for (int b0 = 0; b0 < NI; b0 += GB) {
    if (b0 < d) {
      double gx[GB], gy[GB], gz[GB];
#pragma unroll
      for (int i = 0; i < GB; ++i)
        if (b0 + i < d) {
          gx[i] = ld_coord<RO, opts>(x + u[b0 + i], keep);
          gy[i] = ld_coord<RO, opts>(y + u[b0 + i], keep);
          if (DIM == 3) gz[i] = ld_coord<RO, opts>(z + u[b0 + i], keep);
        }
#pragma unroll
      for (int i = 0; i < GB; ++i)
        if (b0 + i < d) {
          if (b0 + i == 0) {
            sx = gx[i]; sy = gy[i];
            if (DIM == 3) sz = gz[i];
          } else {
            sx = __dadd_rn(sx, gx[i]);
            sy = __dadd_rn(sy, gy[i]);
            if (DIM == 3) sz = __dadd_rn(sz, gz[i]);
          }
        }
    }
  }
  for (int i = NI; i < d; ++i) {  // rows longer than NI (rare): plain ordered loop
    const int32_t w = ld_stream<opts>(scol + j0 + i, stream);
    sx = __dadd_rn(sx, ld_coord<RO, opts>(x + w, keep));
    sy = __dadd_rn(sy, ld_coord<RO, opts>(y + w, keep));
    if (DIM == 3) sz = __dadd_rn(sz, ld_coord<RO, opts>(z + w, keep));
  }
  const double dd = (double)d;
  st_coord<opts>(x + v, __ddiv_rn(sx, dd), keep);
  st_coord<opts>(y + v, __ddiv_rn(sy, dd), keep);
  if (DIM == 3) st_coord<opts>(z + v, __ddiv_rn(sz, dd), keep);
}

// Update the slots [a, b) of one item.  Each warp takes 32 consecutive slots:
// their rows are contiguous in scol, so the warp loads them coalesced into its
// shared-memory buffer, then every lane issues the gathers of its row together.
template <int DIM, bool RO, int opts>
__device__ __forceinline__ void update_item(int32_t a, int32_t b, const int32_t* __restrict__ sv,
                                            const int32_t* __restrict__ sptr, const int32_t* __restrict__ scol,
                                            double* x, double* y, double* z, int32_t* wbuf, uint64_t stream,
                                            uint64_t keep) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const unsigned FULL = 0xffffffffu;
  for (int32_t base = a + warp * 32; base < b; base += nw * 32) {
    const int32_t s = base + lane;
    const bool ok = s < b;
    int32_t v = 0, j0 = 0, j1 = 0;
    if (ok) {
      v = ld_stream<opts>(sv + s, stream);
      j0 = ld_stream<opts>(sptr + s, stream);
      j1 = ld_stream<opts>(sptr + s + 1, stream);
    }
    if (opts & OPT_STAGE) {
      const int last = (b - 1 - base) < 31 ? (b - 1 - base) : 31;
      const int32_t c0 = __shfl_sync(FULL, j0, 0);
      const int32_t c1 = __shfl_sync(FULL, j1, last);
      const int32_t n = c1 - c0;
      if (n <= WBUF) {
        for (int32_t t = lane; t < n; t += 32) wbuf[t] = ld_stream<opts>(scol + c0 + t, stream);
        __syncwarp();
        if (ok) {
          const int32_t* row = wbuf + (j0 - c0);
          lms_vertex_any<DIM, RO, opts>(v, j1 - j0, [row](int i) { return row[i]; }, x, y, z, keep);
        }
        __syncwarp();
        continue;
      }
    }
    if (ok) {
      if (DIM == 2)
        lms_vertex_phased<DIM, RO, 8, 8, opts>(v, j0, j1 - j0, scol, x, y, z, stream, keep);
      else
        lms_vertex_phased<DIM, RO, 16, 4, opts>(v, j0, j1 - j0, scol, x, y, z, stream, keep);
    }
  }
}

template <int DIM, int opts>
__global__ void __launch_bounds__(256) k_sweep_s1(const int32_t* __restrict__ item_ptr, const int32_t* __restrict__ sv,
                                                  const int32_t* __restrict__ sptr, const int32_t* __restrict__ scol,
                                                  double* x, double* y, double* z, int C, int c, int64_t K) {
  __shared__ int32_t wbuf[8][WBUF];
  const uint64_t stream = policy_evict_first(), keep = policy_evict_last();
  for (int64_t k = blockIdx.x; k < K; k += gridDim.x) {
    const int32_t a = item_ptr[k * C + c], b = item_ptr[k * C + c + 1];
    update_item<DIM, true, opts>(a, b, sv, sptr, scol, x, y, z, wbuf[threadIdx.x >> 5], stream, keep);
  }
}

__device__ __forceinline__ int ld_relaxed_gpu(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ void red_release_gpu_add(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

// bulk L2 prefetch of [p, p + bytes) (TMA engine; 16-byte granularity)
__device__ __forceinline__ void prefetch_l2(const void* p, long long bytes) {
  uintptr_t a = (uintptr_t)p & ~(uintptr_t)15;
  uintptr_t e = ((uintptr_t)p + (uintptr_t)bytes + 15) & ~(uintptr_t)15;
  while (a < e) {
    const uint32_t n = (e - a) > (1u << 20) ? (1u << 20) : (uint32_t)(e - a);
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a), "r"(n) : "memory");
    a += n;
  }
}

// S3: persistent colour-pipelined sweep, one 1024-thread CTA per SM.
//  warp 0 (dispatcher): takes item tickets in topological order and keeps two
//    items in flight: half-warps poll the dependency ranges of both at once;
//    an item is published (shared-memory ring, seqlock) once every tile k' of
//    its range has completed all chunks of the stages before sigma
//    (tile_done[k'] >= s*N(k') + P(k', c)), after one gpu-scope acquire.
//  warps 1..31 (workers): pull 32-vertex chunks through a shared chunk cursor.
//    Chunks live in the "slab" layout (per item a fixed width W = max row
//    length; per chunk 32 vertex ids then W columns of 32 neighbour ids, -1
//    padded), so a chunk's address follows from the published item alone and
//    the next chunk's indices are loaded while the current chunk's gathers are
//    in flight (one exposed memory round trip per chunk).
//  The warp completing an item's last chunk publishes it with one gpu-scope
//    release (fence is cumulative over the CTA-scope chunk counters).
//  Reading neighbours only after all their chunks of earlier stages, and
//  writing only after all neighbours' readers of earlier stages are done, is
//  exactly the read-after-write and write-after-read order of the sequential
//  colour schedule (bit-identical to S1).  Tickets are topologically ordered
//  and a CTA publishes its items in ticket order, so the kernel is
//  deadlock-free for any grid.
constexpr int S3_THREADS = 1024;
constexpr int RING = 16;  // max ring depth (ring_n <= RING at run time)
constexpr long long WATCHDOG_SPINS = 1ll << 26;  // x ~32-100 ns per spin: seconds

struct RingSlot {
  int seq, k, begin, end, W, pad;
  long long ioff;
};

template <int DIM, int WMAX, int GB, bool KEEP>
__device__ __forceinline__ void slab_finish(int32_t v, const int32_t (&u)[WMAX], int W, const int32_t* chunk,
                                            double* x, double* y, double* z, uint64_t keep) {
  constexpr int CO = KEEP ? OPT_HINT_COORD : 0;
  if (v < 0) return;
  const int lane = threadIdx.x & 31;
  double sx = 0.0, sy = 0.0, sz = 0.0;
  int d = 0;
#pragma unroll
  for (int b0 = 0; b0 < WMAX; b0 += GB) {
    double gx[GB], gy[GB], gz[GB];
    bool ok[GB];
#pragma unroll
    for (int i = 0; i < GB; ++i) {
      ok[i] = (b0 + i < W) && u[b0 + i] >= 0;
      if (ok[i]) {
        gx[i] = ld_coord<false, CO>(x + u[b0 + i], keep);
        gy[i] = ld_coord<false, CO>(y + u[b0 + i], keep);
        if (DIM == 3) gz[i] = ld_coord<false, CO>(z + u[b0 + i], keep);
      }
    }
#pragma unroll
    for (int i = 0; i < GB; ++i)
      if (ok[i]) {
        if (d == 0) {
          sx = gx[i]; sy = gy[i];
          if (DIM == 3) sz = gz[i];
        } else {
          sx = __dadd_rn(sx, gx[i]);
          sy = __dadd_rn(sy, gy[i]);
          if (DIM == 3) sz = __dadd_rn(sz, gz[i]);
        }
        ++d;
      }
  }
  for (int w = WMAX; w < W; ++w) {  // rows longer than WMAX (general meshes): ordered tail loop
    const int32_t uu = __ldg(chunk + 32 + w * 32 + lane);
    if (uu < 0) break;
    sx = __dadd_rn(sx, ld_coord<false, CO>(x + uu, keep));
    sy = __dadd_rn(sy, ld_coord<false, CO>(y + uu, keep));
    if (DIM == 3) sz = __dadd_rn(sz, ld_coord<false, CO>(z + uu, keep));
    ++d;
  }
  const double dd = (double)d;
  st_coord<CO>(x + v, __ddiv_rn(sx, dd), keep);
  st_coord<CO>(y + v, __ddiv_rn(sy, dd), keep);
  if (DIM == 3) st_coord<CO>(z + v, __ddiv_rn(sz, dd), keep);
}

template <int DIM, int WMAX, int GB>
__global__ void __launch_bounds__(S3_THREADS, 1) k_sweep_s3(
    const int32_t* __restrict__ item_ptr, const long long* __restrict__ ioff, const int32_t* __restrict__ iw,
    const int32_t* __restrict__ slab, const int32_t* __restrict__ klo, const int32_t* __restrict__ khi,
    const int32_t* __restrict__ tpre, unsigned* tile_done, unsigned long long* ticket, double* x, double* y,
    double* z, int C, int64_t K, int L, int sweeps, int* abort_flag, int ring_n, unsigned long long* stats,
    const int32_t* __restrict__ irec, int qdepth, const int32_t* __restrict__ tdep_ptr,
    const int32_t* __restrict__ tdep, int disp_mode, int lookahead, int hint_mode) {
  __shared__ RingSlot ring[RING];
  __shared__ int slot_done[RING];
  __shared__ int cc;        // next unclaimed chunk id
  __shared__ int pub_end;   // chunk ids below this are published
  __shared__ int pub_done;  // dispatcher finished (no more chunks will be published)
  __shared__ int sh_abort;
  __shared__ unsigned long long st[8];  // tuning counters (stats != nullptr only)
  __shared__ unsigned long long sd[8];  // dispatcher tuning counters
  __shared__ int4 qrec[8][REC_INTS / 4];  // dispatcher's staged item records
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x < 8) st[threadIdx.x] = sd[threadIdx.x] = 0;
  const unsigned FULL = 0xffffffffu;
  if (threadIdx.x < RING) {
    ring[threadIdx.x].seq = (int)threadIdx.x - RING;  // "previous occupant" of slot r
    ring[threadIdx.x].begin = ring[threadIdx.x].end = 0;
    slot_done[threadIdx.x] = 0;
  }
  if (threadIdx.x == 0) { cc = 0; pub_end = 0; pub_done = 0; sh_abort = 0; }
  __syncthreads();
  volatile int* vabort = &sh_abort;
  volatile RingSlot* vr = ring;
  volatile int* vdone = slot_done;
  // watchdog: a spin that outlives its budget sets the global abort flag; every
  // spin also exits once any CTA aborted, so a broken schedule returns an
  // error (LMS_E_CUDA) instead of hanging the GPU
  auto spin_ok = [&](long long& budget) -> bool {
    if (*vabort) return false;
    if (--budget < 0 || ((budget & 1023) == 0 && *(volatile int*)abort_flag)) {
      atomicExch(abort_flag, (int)LMS_E_CUDA);
      *vabort = 1;
      return false;
    }
    __nanosleep(32);
    return true;
  };

  if (warp == 0 && disp_mode == 0) {  // --------------------------- dispatcher (simple)
    // One item at a time, ~2.5 memory round trips per item: the 128-byte item
    // record arrives with one coalesced warp load (lane l holds word l), the
    // dependency pairs are polled by parallel lanes, then one acquire and the
    // publish.  The small in-flight window keeps the lag L (hence the L2
    // footprint of the colour pipeline) small.
    const long long per_sweep = (long long)(K + (long long)(C - 1) * L) * C;
    const long long total = per_sweep * sweeps;
    long long t_next = 0;
    if (lane == 0) t_next = (long long)atomicAdd(ticket, 1ull);
    t_next = __shfl_sync(FULL, t_next, 0);
    int i = 0, base = 0;
    long long tA = clock64();
    for (;;) {
      const long long t = t_next;
      if (t >= total) break;
      long long tn = 0;
      if (lane == 0) tn = (long long)atomicAdd(ticket, 1ull);  // prefetch the next ticket
      const int s = (int)(t / per_sweep);
      const long long r = t - (long long)s * per_sweep;
      const long long jj = r / C;
      const int c = (int)(r - jj * C);
      const long long k = jj - (long long)c * L;
      t_next = __shfl_sync(FULL, tn, 0);
      if (k < 0 || k >= K) continue;  // no such tile for this key (pipeline fill / drain)
      const long long tR0 = clock64();
      const int rv = __ldg(irec + (k * C + c) * REC_INTS + lane);
      const int n = __shfl_sync(FULL, rv, 0);
      if (n == 0) continue;  // empty item
      const long long tR1 = clock64();
      int polls = 0;
      const int nd = __shfl_sync(FULL, rv, 4);
      const int np = __shfl_down_sync(FULL, rv, 1);  // lane l: rec[l + 1]
      long long budget = WATCHDOG_SPINS;
      for (;;) {
        bool ok = true;
        if (nd > 0) {
          if (lane >= 6 && lane < 6 + 2 * nd && ((lane - 6) & 1) == 0)
            ok = (unsigned)ld_relaxed_gpu((const int*)(tile_done + rv)) >=
                 (unsigned)s * ((unsigned)np & 0xffffu) + ((unsigned)np >> 16);
        } else {  // many / large dependencies: per-tile lists and the prefix table
          auto need = [&](int kt) {
            return (unsigned)s * (unsigned)tpre[kt * (C + 1) + C] + (unsigned)tpre[kt * (C + 1) + c];
          };
          if (lane == 0) ok = (unsigned)ld_relaxed_gpu((const int*)(tile_done + k)) >= need((int)k);
          for (int q = tdep_ptr[k] + lane; q < tdep_ptr[k + 1]; q += 32) {
            const int kt = tdep[q];
            if ((unsigned)ld_relaxed_gpu((const int*)(tile_done + kt)) < need(kt)) ok = false;
          }
        }
        ++polls;
        if (__all_sync(FULL, ok)) break;
        if (!spin_ok(budget)) break;
      }
      if (*vabort) break;
      const long long tB = clock64();
      if (stats && lane == 0) {
        sd[4] += tR1 - tR0;  // record load
        sd[5] += tB - tR1;   // polling
        sd[6] += polls;
      }
      fence_acq_rel_gpu();  // acquire for the whole SM (also invalidates L1)
      const int W = __shfl_sync(FULL, rv, 1), olo = __shfl_sync(FULL, rv, 2), ohi = __shfl_sync(FULL, rv, 3);
      const int slot = i % ring_n;
      if (lane == 0) {
        long long b2 = WATCHDOG_SPINS;
        const long long tW = clock64();
        while (vdone[slot] < vr[slot].end - vr[slot].begin)  // previous occupant finished
          if (!spin_ok(b2)) break;
        if (stats) sd[7] += clock64() - tW;
        vr[slot].seq = -2;  // seqlock: invalidate before rewriting the fields
        __threadfence_block();
        vr[slot].k = (int)k;
        vr[slot].begin = base;
        vr[slot].end = base + n;
        vr[slot].W = W;
        vr[slot].ioff = ((long long)(unsigned)ohi << 32) | (unsigned)olo;
        vdone[slot] = 0;
        __threadfence_block();
        vr[slot].seq = i;
        __threadfence_block();
        *(volatile int*)&pub_end = base + n;
      }
      __syncwarp();
      base += n;
      ++i;
      if (stats && lane == 0) {
        const long long tD = clock64();
        sd[0] += tB - tA;
        sd[1] += tD - tB;
        sd[3] += 1;
        tA = tD;
      }
    }
    if (lane == 0) {
      __threadfence_block();
      *(volatile int*)&pub_done = 1;
      if (stats) for (int q = 0; q < 8; ++q) atomicAdd(stats + 8 + q, sd[q]);
    }
    return;
  }
  if (warp == 0) {  // ------------------------------------------------ dispatcher
    // Lane q holds queue entry q (q < nq), in ticket order.  Each pass of the
    // loop advances every entry one stage with the loads of all lanes in
    // flight together: ticket -> 64-byte item record -> dependency poll ->
    // publish (ready prefix, in ticket order: the deadlock-freedom proof needs
    // a CTA to publish its items in the order of their tickets).
    const long long per_sweep = (long long)(K + (long long)(C - 1) * L) * C;
    const long long total = per_sweep * sweeps;
    constexpr int QMAX = 8;
    int nq = 0;              // queued entries (lanes 0..nq-1)
    int fillc = 0;           // records are staged in qrec[fill order % QMAX] (FIFO)
    int qslot = 0;           // this lane's record slot
    int st_ = 0;             // this lane's stage: 0 empty, 1 ticket, 2 record, 3 ready, 4 skip
    long long tk = 0;        // ticket
    int qs = 0, qc = 0, qk = 0;
    bool exhausted = false;
    long long t_batch = 0;
    int t_left = 0;
    int i = 0, base = 0;
    long long budget = WATCHDOG_SPINS;
    const int qcap = qdepth < 1 ? 1 : (qdepth > QMAX ? QMAX : qdepth);
    long long tA = clock64();
    for (;;) {
      // (1) refill empty tail lanes with consecutive tickets
      while (nq < qcap && !exhausted) {
        if (t_left == 0) {
          long long t0 = 0;
          if (lane == 0) t0 = (long long)atomicAdd(ticket, (unsigned long long)qcap);
          t_batch = __shfl_sync(FULL, t0, 0);
          t_left = qcap;
        }
        const long long t = t_batch++;
        --t_left;
        if (t >= total) { exhausted = true; break; }
        if (lane == nq) {
          tk = t;
          qs = (int)(t / per_sweep);
          const long long r = t - (long long)qs * per_sweep;
          const long long jj = r / C;
          qc = (int)(r - jj * C);
          const long long k = jj - (long long)qc * L;
          if (k < 0 || k >= K) {
            st_ = 4;  // no such tile for this key: skip in order
          } else {
            qk = (int)k;
            qslot = fillc % QMAX;
            const int4* rec = (const int4*)(irec + ((long long)qk * C + qc) * REC_INTS);
#pragma unroll
            for (int q = 0; q < REC_INTS / 4; ++q) qrec[qslot][q] = __ldg(rec + q);
            st_ = 1;
          }
        }
        ++nq;
        ++fillc;
      }
      if (nq == 0) break;  // tickets exhausted and everything published
      // (2) entries whose record arrived: empty items are skipped; others poll
      bool ready = false;
      if (lane < nq) {
        const int* rec = (const int*)qrec[qslot];
        if (st_ == 1) st_ = (rec[0] == 0) ? 4 : 2;  // empty item: skip in order
        if (st_ == 2) {
          const int nd = rec[4];
          ready = true;
          if (nd > 0) {
            for (int q = 0; q < nd; ++q) {
              const int kt = rec[6 + 2 * q];
              const unsigned np = (unsigned)rec[7 + 2 * q];
              if ((unsigned)ld_relaxed_gpu((const int*)(tile_done + kt)) < (unsigned)qs * (np & 0xffffu) + (np >> 16))
                ready = false;
            }
          } else {  // many / large dependencies: per-tile lists and prefix table
            auto need = [&](int kt) {
              return (unsigned)qs * (unsigned)tpre[kt * (C + 1) + C] + (unsigned)tpre[kt * (C + 1) + qc];
            };
            ready = (unsigned)ld_relaxed_gpu((const int*)(tile_done + qk)) >= need(qk);
            for (int q = tdep_ptr[qk]; q < tdep_ptr[qk + 1] && ready; ++q) {
              const int kt = tdep[q];
              if ((unsigned)ld_relaxed_gpu((const int*)(tile_done + kt)) < need(kt)) ready = false;
            }
          }
          if (ready) st_ = 3;
        }
      }
      // (3) publish / skip the ready prefix in ticket order
      const unsigned done_mask = __ballot_sync(FULL, lane < nq && (st_ == 3 || st_ == 4));
      int npre = __ffs(~done_mask) - 1;
      if (npre < 0) npre = 32;
      if (npre > nq) npre = nq;
      int pub = 0;
      if (npre > 0) {
        const long long tB = clock64();
        const unsigned pubmask = __ballot_sync(FULL, lane < npre && st_ == 3);
        if (pubmask) fence_acq_rel_gpu();  // one acquire for the batch (also invalidates L1)
        for (; pub < npre; ++pub) {
          const int stp = __shfl_sync(FULL, st_, pub);
          if (stp == 3) {
            const int slot = i % ring_n;
            const int busy = __shfl_sync(FULL, (int)(vdone[slot] < vr[slot].end - vr[slot].begin), 0);
            if (busy) break;  // ring full: publish on a later pass
            const int* prec = (const int*)qrec[__shfl_sync(FULL, qslot, pub)];
            const int n = prec[0], W = prec[1], olo = prec[2], ohi = prec[3];
            const int kq = __shfl_sync(FULL, qk, pub);
            if (lane == 0) {
              vr[slot].seq = -2;  // seqlock: invalidate before rewriting the fields
              __threadfence_block();
              vr[slot].k = kq;
              vr[slot].begin = base;
              vr[slot].end = base + n;
              vr[slot].W = W;
              vr[slot].ioff = ((long long)(unsigned)ohi << 32) | (unsigned)olo;
              vdone[slot] = 0;
              __threadfence_block();
              vr[slot].seq = i;
              __threadfence_block();
              *(volatile int*)&pub_end = base + n;
            }
            base += n;
            ++i;
            if (stats && lane == 0) st[3] += 1;
          }
        }
        if (stats && lane == 0) st[1] += clock64() - tB;
      }
      if (pub > 0) {
        // drop the handled prefix
        tk = __shfl_down_sync(FULL, tk, pub);
        st_ = __shfl_down_sync(FULL, st_, pub);
        qs = __shfl_down_sync(FULL, qs, pub);
        qc = __shfl_down_sync(FULL, qc, pub);
        qk = __shfl_down_sync(FULL, qk, pub);
        qslot = __shfl_down_sync(FULL, qslot, pub);
        nq -= pub;
        if (lane >= nq) st_ = 0;
        budget = WATCHDOG_SPINS;
      } else if (nq > 0 && !spin_ok(budget)) {
        break;
      }
      if (*vabort) break;
      if (stats && lane == 0) {
        const long long tD = clock64();
        st[0] += tD - tA;
        tA = tD;
      }
    }
    if (lane == 0) {
      __threadfence_block();
      *(volatile int*)&pub_done = 1;
      if (stats) for (int q = 0; q < 4; ++q) atomicAdd(stats + q, st[q]);
    }
    return;
  }
  // ---------------------------------------------------------------- workers
  // A worker never blocks while it holds an unfinished chunk: the look-ahead
  // claim is non-blocking (CAS below the published frontier); it only waits
  // for publication when it holds nothing (otherwise: deadlock, since the
  // dispatcher may be waiting for the very item that chunk belongs to).
  volatile int* vcc = &cc;
  volatile int* vpe = &pub_end;
  volatile int* vpd = &pub_done;
  auto try_claim = [&]() -> int {  // warp-uniform; -1 if nothing published is left
    int cid = -1;
    if (lane == 0) {
      int cur = *vcc;
      for (;;) {
        if (cur >= *vpe) break;
        const int old = atomicCAS(&cc, cur, cur + 1);
        if (old == cur) { cid = cur; break; }
        cur = old;
      }
    }
    return __shfl_sync(FULL, cid, 0);
  };
  auto claim_blocking = [&]() -> int {  // -1 when the dispatcher is done (or aborted)
    long long budget = WATCHDOG_SPINS;
    for (;;) {
      const int cid = try_claim();
      if (cid >= 0) return cid;
      int fin = 0;
      if (lane == 0) {
        const int d = *vpd;
        __threadfence_block();
        fin = d && *vcc >= *vpe;
      }
      if (__shfl_sync(FULL, fin, 0)) return -1;
      if (!spin_ok(budget)) return -1;
    }
  };
  int j = 0;
  // locate a claimed (hence published) chunk: ring slot, tile, width, address
  auto locate = [&](int cid, int& k, int& slot, int& W, const int32_t*& chunk) {
    for (;;) {
      slot = j % ring_n;
      const int seq = vr[slot].seq;
      if (seq < j) continue;  // being rewritten (seqlock)
      if (seq > j) { ++j; continue; }
      k = vr[slot].k;
      const int begin = vr[slot].begin, end = vr[slot].end;
      W = vr[slot].W;
      const long long off = vr[slot].ioff;
      __threadfence_block();
      if (vr[slot].seq != j) continue;  // recycled while reading: retry
      if (cid < end) {
        chunk = slab + off + (long long)(cid - begin) * 32 * (1 + W);
        return;
      }
      ++j;
    }
  };
  const uint64_t pol_stream = policy_evict_first(), pol_keep = policy_evict_last();
  auto load_idx = [&](const int32_t* chunk, int W, int32_t& v, int32_t (&u)[WMAX]) {
    // the slab is read once per sweep: stream it through L2 with evict_first so
    // it does not displace the coordinates the next colours re-read
    if (hint_mode & 1) {
      v = ld_stream<OPT_HINT_STREAM>(chunk + lane, pol_stream);
#pragma unroll
      for (int w = 0; w < WMAX; ++w) u[w] = (w < W) ? ld_stream<OPT_HINT_STREAM>(chunk + 32 + w * 32 + lane, pol_stream) : -1;
    } else {
      v = __ldg(chunk + lane);
#pragma unroll
      for (int w = 0; w < WMAX; ++w) u[w] = (w < W) ? __ldg(chunk + 32 + w * 32 + lane) : -1;
    }
  };
  int cidA = claim_blocking();
  if (cidA < 0) return;
  int kA, slotA, WA;
  const int32_t* chA;
  locate(cidA, kA, slotA, WA, chA);
  int32_t vA, uA[WMAX];
  load_idx(chA, WA, vA, uA);
  for (;;) {
    // look ahead (non-blocking) only when the published backlog leaves work
    // for every other warp; otherwise a second chunk would serialise behind A
    int cidB = -1;
    if (lookahead > 0) {
      int backlog = 0;
      if (lane == 0) backlog = *vpe - *vcc;
      backlog = __shfl_sync(FULL, backlog, 0);
      if (backlog > lookahead) cidB = try_claim();
    }
    int kB = 0, slotB = 0, WB = 0;
    const int32_t* chB = nullptr;
    int32_t vB = -1, uB[WMAX];
    if (cidB >= 0) {
      locate(cidB, kB, slotB, WB, chB);
      load_idx(chB, WB, vB, uB);
    }
    const long long tf = clock64();
    if (hint_mode & 2)
      slab_finish<DIM, WMAX, GB, true>(vA, uA, WA, chA, x, y, z, pol_keep);
    else
      slab_finish<DIM, WMAX, GB, false>(vA, uA, WA, chA, x, y, z, pol_keep);
    __syncwarp();
    if (stats && lane == 0) {
      atomicAdd(&st[5], (unsigned long long)(clock64() - tf));
      atomicAdd(&st[6], 1ull);
      atomicAdd(&st[7], (unsigned long long)(cidB >= 0));
    }
    if (lane == 0) {
      // CTA-scope release of this chunk's stores; the warp completing the item
      // turns the whole item into one gpu-scope release (fence is cumulative)
      __threadfence_block();
      const int n_item = vr[slotA].end - vr[slotA].begin;
      const int old = atomicAdd(&slot_done[slotA], 1);
      if (old + 1 == n_item) {
        fence_acq_rel_gpu();
        atomicAdd(tile_done + kA, (unsigned)n_item);
      }
    }
    if (cidB < 0) {  // nothing was ready: now wait (holding no chunk)
      const long long ti = clock64();
      const int c2 = claim_blocking();
      if (stats && lane == 0) atomicAdd(&st[4], (unsigned long long)(clock64() - ti));
      if (c2 < 0) {
        if (stats && lane == 0) for (int q = 4; q < 8; ++q) atomicAdd(stats + q, atomicExch(&st[q], 0ull));
        return;
      }
      locate(c2, kB, slotB, WB, chB);
      load_idx(chB, WB, vB, uB);
    }
    kA = kB; slotA = slotB; WA = WB; chA = chB; vA = vB;
#pragma unroll
    for (int w = 0; w < WMAX; ++w) uA[w] = uB[w];
  }
}




// ---------------------------------------------------------------- drivers
// LMS_S3_STATS=1 (tuning only): per-CTA clock64 counters summed over CTAs:
// [dispatch poll, publish, next-ticket, items, worker idle, worker busy, chunks, look-ahead hits]
static unsigned long long* g_stats = nullptr;
static unsigned long long* s3_stats(cudaStream_t s) {
  if (!getenv("LMS_S3_STATS")) return nullptr;
  if (!g_stats) LMS_TRY_CUDA(cudaMalloc(&g_stats, 16 * sizeof(unsigned long long)));
  LMS_TRY_CUDA(cudaMemsetAsync(g_stats, 0, 16 * sizeof(unsigned long long), s));
  return g_stats;
}
static void s3_stats_report(cudaStream_t s, int sweeps, int ctas) {
  if (!g_stats || !getenv("LMS_S3_STATS")) return;
  unsigned long long h[16];
  LMS_TRY_CUDA(cudaMemcpyAsync(h, g_stats, sizeof(h), cudaMemcpyDeviceToHost, s));
  LMS_TRY_CUDA(cudaStreamSynchronize(s));
  if (h[11]) {
    const double it = (double)h[11];
    fprintf(stderr, "[s3 simple] items/cta=%.0f gap(ticket..fence)=%.0f fence+publish=%.0f record=%.0f poll=%.0f "
            "polls/item=%.2f ringwait=%.0f cyc/item\n", it / ctas, h[8] / it, h[9] / it, h[12] / it, h[13] / it,
            h[14] / it, h[15] / it);
  }
  const double it = h[3] ? (double)h[3] : 1.0, ch = h[6] ? (double)h[6] : 1.0;
  fprintf(stderr, "[s3] sweeps=%d items/cta=%.0f poll=%.0f publish=%.0f next=%.0f cyc/item | chunks/cta=%.0f "
          "busy=%.0f cyc/chunk idle/warp=%.0f cyc lookahead=%.2f\n", sweeps, it / ctas, h[0] / it, h[1] / it, h[2] / it,
          ch / ctas, h[5] / ch, (double)h[4] / ctas / 31.0, h[7] / ch);
}

static int s3_hints() {
  int h = 1;  // bit0: slab evict_first, bit1: coordinates evict_last (LMS_S3_HINTS tunes)
  if (const char* e = getenv("LMS_S3_HINTS")) h = atoi(e);
  return h;
}

static int s3_lookahead() {
  int l = 0;  // look ahead only if more than this many published chunks are unclaimed (LMS_S3_LOOKAHEAD; 0 = never)
  if (const char* e = getenv("LMS_S3_LOOKAHEAD")) l = atoi(e);
  return l;
}

static int s3_disp() {
  int d = 0;  // dispatcher: 0 simple (one item at a time), 1 systolic queue (LMS_S3_DISP tunes)
  if (const char* e = getenv("LMS_S3_DISP")) d = atoi(e);
  return d;
}

static int s3_qdepth() {
  int q = 4;  // dispatcher queue depth (LMS_S3_QDEPTH tunes)
  if (const char* e = getenv("LMS_S3_QDEPTH")) q = atoi(e);
  return q;
}

static int s3_ring() {
  int r = 4;  // published-but-unfinished items per CTA (LMS_S3_RING tunes)
  if (const char* e = getenv("LMS_S3_RING")) r = atoi(e);
  return r < 1 ? 1 : (r > RING ? RING : r);
}

static int sweep_opts() {
  if (const char* e = getenv("LMS_OPTS")) return atoi(e);
  return OPT_DEFAULT;
}

static cudaStream_t capture_stream() {
  static thread_local cudaStream_t cs = nullptr;
  if (!cs) LMS_TRY_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
  return cs;
}

template <int DIM, int OPTS>
static void launch_s1_t(lms_mesh_s* m, cudaStream_t s, int c, unsigned G) {
  Schedule& S = m->sched;
  k_sweep_s1<DIM, OPTS><<<G, 256, 0, s>>>(S.item_ptr.p, S.sv.p, S.sptr.p, S.scol.p, m->x[0].p, m->x[1].p,
                                           DIM == 3 ? m->x[2].p : nullptr, m->C, c, S.K);
}

static void launch_s3(lms_mesh_s* m, cudaStream_t s, int ctas, int sweeps) {
  Schedule& S = m->sched;
  if (m->dim == 2)
    k_sweep_s3<2, 8, 8><<<ctas, S3_THREADS, 0, s>>>(S.item_ptr.p, S.ioff.p, S.iw.p, S.slab.p, S.klo.p, S.khi.p,
                                                     S.tpre.p, (unsigned*)S.prog.p, S.ticket.p, m->x[0].p, m->x[1].p,
                                                     nullptr, m->C, S.K, S.lag, sweeps, m->err.p, s3_ring(),
                                                     s3_stats(s), S.irec.p, s3_qdepth(), S.tdep_ptr.p, S.tdep.p, s3_disp(), s3_lookahead(), s3_hints());
  else
    k_sweep_s3<3, 16, 4><<<ctas, S3_THREADS, 0, s>>>(S.item_ptr.p, S.ioff.p, S.iw.p, S.slab.p, S.klo.p, S.khi.p,
                                                      S.tpre.p, (unsigned*)S.prog.p, S.ticket.p, m->x[0].p,
                                                      m->x[1].p, m->x[2].p, m->C, S.K, S.lag, sweeps, m->err.p,
                                                      s3_ring(), s3_stats(s), S.irec.p, s3_qdepth(), S.tdep_ptr.p,
                                                      S.tdep.p, s3_disp(), s3_lookahead(), s3_hints());
}

#define LMS_OPT_CASES(F) F(0) F(1) F(2) F(3) F(4) F(8)

static void launch_s1_colours(lms_mesh_s* m, cudaStream_t s) {
  Schedule& S = m->sched;
  const int64_t K = S.K;
  unsigned G = (unsigned)(K < 65535 * 16 ? K : 65535 * 16);
  const int o = sweep_opts();
  for (int c = 0; c < m->C; ++c) {
    switch (o) {
#define F(X)                                   \
  case X:                                      \
    if (m->dim == 2) launch_s1_t<2, X>(m, s, c, G); \
    else launch_s1_t<3, X>(m, s, c, G);        \
    break;
      LMS_OPT_CASES(F)
#undef F
      default: fail(LMS_E_ARG, "unsupported LMS_OPTS");
    }
    LMS_TRY_CUDA(cudaGetLastError());
  }
}

// graphs[0] = 1 sweep, graphs[1] = 8 sweeps (captured once per schedule; the
// coordinate buffers are fixed for the life of the schedule)
static cudaGraphExec_t get_graph(lms_mesh_s* m, int which) {
  Schedule& S = m->sched;
  if (S.graphs[which]) return S.graphs[which];
  cudaStream_t cs = capture_stream();
  const int n = which == 0 ? 1 : 8;
  cudaGraph_t g = nullptr;
  LMS_TRY_CUDA(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
  try {
    for (int i = 0; i < n; ++i) launch_s1_colours(m, cs);
  } catch (...) {
    cudaStreamEndCapture(cs, &g);
    if (g) cudaGraphDestroy(g);
    throw;
  }
  LMS_TRY_CUDA(cudaStreamEndCapture(cs, &g));
  cudaGraphExec_t ge = nullptr;
  cudaError_t e = cudaGraphInstantiate(&ge, g, 0);
  cudaGraphDestroy(g);
  LMS_TRY_CUDA(e);
  S.graphs[which] = ge;
  return ge;
}

// one colour stage with the S1 kernel (used by the multi-GPU sweep, which
// exchanges halos between stages)
void run_colour_stage(lms_mesh_s* m, int c, cudaStream_t s) {
  sync_soa(m, s);
  if (!m->sched.base_valid) build_base(m, s, true);  // GZ schedules skip the S1 lists
  soa_changed(m);
  const unsigned G = (unsigned)(m->sched.K < 65535 * 16 ? m->sched.K : 65535 * 16);
  if (m->dim == 2)
    launch_s1_t<2, OPT_DEFAULT>(m, s, c, G);
  else
    launch_s1_t<3, OPT_DEFAULT>(m, s, c, G);
  LMS_CHECK_LAUNCH();
}

void run_sweeps(lms_mesh_s* m, int sweeps, cudaStream_t s) {
  Schedule& S = m->sched;
  if (S.kind == LMS_SCHED_GZ) {
    run_gz(m, sweeps, s);
    return;
  }
  if (S.kind == LMS_SCHED_JACOBI) {
    run_jacobi(m, sweeps, s);
    return;
  }
  if (S.kind == LMS_SCHED_S2) {
    run_s2(m, sweeps, s);
    return;
  }
  sync_soa(m, s);
  soa_changed(m);  // S1/S3 update x[] in place
  if (S.kind == LMS_SCHED_S1) {
    int left = sweeps;
    while (left >= 8) {
      LMS_TRY_CUDA(cudaGraphLaunch(get_graph(m, 1), s));
      note_launch(8 * m->C);
      left -= 8;
    }
    while (left > 0) {
      LMS_TRY_CUDA(cudaGraphLaunch(get_graph(m, 0), s));
      note_launch(m->C);
      --left;
    }
    return;
  }
  // S3: one persistent launch for all sweeps
  LMS_TRY_CUDA(cudaMemsetAsync(S.prog.p, 0, S.K * sizeof(int), s));
  LMS_TRY_CUDA(cudaMemsetAsync(S.ticket.p, 0, sizeof(unsigned long long), s));
  const int ctas = s3_ctas(m->device);
  if ((long long)sweeps * m->C >= 0x7fffffffLL) fail(LMS_E_ARG, "too many sweeps for one call");
  launch_s3(m, s, ctas, sweeps);
  s3_stats_report(s, sweeps, ctas);
  LMS_CHECK_LAUNCH();
  // the persistent kernel reports a watchdog abort through the handle's error flag
  if (!m->async_errors) check_err_flag(m, s, "lms_smooth (S3 watchdog: dependency wait exceeded its budget)");
}

}  // namespace lms
