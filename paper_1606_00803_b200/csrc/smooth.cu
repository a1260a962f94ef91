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

#include "lms_internal.cuh"

namespace lms {

// ---------------------------------------------------------------- schedule build
__global__ void k_free_flags(const uint8_t* __restrict__ fixed, int64_t V, uint8_t* flags, int32_t* ids) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < V; v += (int64_t)gridDim.x * blockDim.x) {
    flags[v] = fixed[v] ? 0 : 1;
    ids[v] = (int32_t)v;
  }
}

__global__ void k_item_keys(const int32_t* __restrict__ fv, int64_t n, const int8_t* __restrict__ colour, int T,
                            int C, uint32_t* keys) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int32_t v = fv[i];
    keys[i] = (uint32_t)((v / T) * C + colour[v]);
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

__global__ void k_slot_rows(const int32_t* __restrict__ sv, int64_t n, const int32_t* __restrict__ rp,
                            const int32_t* __restrict__ col, const int32_t* __restrict__ sptr,
                            const uint8_t* __restrict__ fixed, int T, int32_t* __restrict__ scol, int32_t* klo,
                            int32_t* khi) {
  const int lane = threadIdx.x & 31;
  const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = w; i < n; i += nw) {
    const int32_t v = sv[i], b = rp[v], d = rp[v + 1] - b, o = sptr[i];
    const int32_t k = v / T;
    int32_t lo = k, hi = k;
    for (int32_t j = lane; j < d; j += 32) {
      const int32_t u = col[b + j];
      scol[o + j] = u;
      if (!fixed[u]) {
        lo = min(lo, u / T);
        hi = max(hi, u / T);
      }
    }
    for (int off = 16; off; off >>= 1) {
      lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, off));
      hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, off));
    }
    if (lane == 0) {
      if (lo < k) atomicMin(&klo[k], lo);
      if (hi > k) atomicMax(&khi[k], hi);
    }
  }
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

static int s3_ctas(int dev) {
  int nsm = 0;
  LMS_TRY_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  return nsm * 2;  // two 512-thread CTAs per SM
}

void build_schedule(lms_mesh_s* m, cudaStream_t s) {
  Schedule& S = m->sched;
  S.valid = false;
  for (int i = 0; i < 2; ++i)
    if (S.graphs[i]) { cudaGraphExecDestroy(S.graphs[i]); S.graphs[i] = nullptr; }
  const int64_t V = m->V;
  const int C = m->C;
  // tile size: S1 -> about one vertex per thread of a 256-thread CTA per item;
  // S3 -> 4096 (big items amortise the per-item ticket/poll latency)
  int T = m->tile_req;
  const bool want_s3 = (m->sched_req == LMS_SCHED_S3 || m->sched_req == LMS_SCHED_AUTO);
  if (T == 0) T = want_s3 ? 4096 : 256 * (C > 0 ? C : 1);
  if (T > V) T = (int)((V + 31) / 32 * 32);
  if (T < 32) T = 32;
  const int64_t K = (V + T - 1) / T;
  if (K * (int64_t)(C > 0 ? C : 1) >= ((int64_t)1 << 31)) fail(LMS_E_ARG, "too many schedule items");
  S.tile = T;
  S.K = K;
  const unsigned Gv = grid_for(V, 256) > 8192 ? 8192 : grid_for(V, 256);
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
  k_range_init<<<grid_for(K, 256) > 4096 ? 4096 : grid_for(K, 256), 256, 0, s>>>(S.klo.p, S.khi.p, K);
  LMS_CHECK_LAUNCH();
  if (n > 0) {
    const unsigned Gn = grid_for(n, 256) > 8192 ? 8192 : grid_for(n, 256);
    DBuf<uint32_t> keys(n, s), skeys(n, s);
    k_item_keys<<<Gn, 256, 0, s>>>(fv.p, n, m->colour.p, T, C, keys.p);
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
    const unsigned Gw = grid_for(n * 32, 256) > 8192 ? 8192 : grid_for(n * 32, 256);
    k_slot_rows<<<Gw, 256, 0, s>>>(S.sv.p, n, m->row_ptr.p, m->col.p, S.sptr.p, m->fixed.p, T, S.scol.p, S.klo.p,
                                   S.khi.p);
    LMS_CHECK_LAUNCH();
  } else {
    LMS_TRY_CUDA(cudaMemsetAsync(S.item_ptr.p, 0, (nitems + 1) * sizeof(int32_t), s));
  }
  DBuf<int> reach(1, s);
  LMS_TRY_CUDA(cudaMemsetAsync(reach.p, 0, sizeof(int), s));
  k_reach<<<grid_for(K, 256) > 1024 ? 1024 : grid_for(K, 256), 256, 0, s>>>(S.klo.p, S.khi.p, K, reach.p);
  LMS_CHECK_LAUNCH();
  int hr = 0;
  LMS_TRY_CUDA(cudaMemcpyAsync(&hr, reach.p, sizeof(int), cudaMemcpyDeviceToHost, s));
  LMS_TRY_CUDA(cudaStreamSynchronize(s));
  S.max_reach = hr;
  // resolve the kernel: S3 pays off only for banded orderings (small tile reach)
  int kind = m->sched_req;
  if (kind == LMS_SCHED_AUTO) kind = (K >= 16 && hr * 8 <= K) ? LMS_SCHED_S3 : LMS_SCHED_S1;
  S.kind = kind;
  if (kind == LMS_SCHED_S3) {
    const int ctas = s3_ctas(m->device);
    int L = hr + 1 + (2 * ctas + C - 1) / (C > 0 ? C : 1);
    if (m->lag_req > 0) L = m->lag_req > hr ? m->lag_req : hr + 1;  // must exceed the reach
    S.lag = L;
  } else {
    S.lag = 0;
  }
  S.valid = true;
}

// ---------------------------------------------------------------- sweep kernels
template <int DIM, bool RO>
__device__ __forceinline__ double ldx(const double* p) {
  if (RO) return __ldg(p);
  return *p;
}

// update the slots [a, b) of one item; threads stride the slots
template <int DIM, bool RO>
__device__ __forceinline__ void update_slots(int32_t a, int32_t b, const int32_t* __restrict__ sv,
                                             const int32_t* __restrict__ sptr, const int32_t* __restrict__ scol,
                                             double* x, double* y, double* z) {
  for (int32_t i = a + threadIdx.x; i < b; i += blockDim.x) {
    const int32_t v = sv[i], j0 = sptr[i], j1 = sptr[i + 1];
    int32_t u = scol[j0];
    double ax = ldx<DIM, RO>(x + u), ay = ldx<DIM, RO>(y + u), az = 0.0;
    if (DIM == 3) az = ldx<DIM, RO>(z + u);
    for (int32_t j = j0 + 1; j < j1; ++j) {
      u = scol[j];
      ax = __dadd_rn(ax, ldx<DIM, RO>(x + u));
      ay = __dadd_rn(ay, ldx<DIM, RO>(y + u));
      if (DIM == 3) az = __dadd_rn(az, ldx<DIM, RO>(z + u));
    }
    const double d = (double)(j1 - j0);
    x[v] = __ddiv_rn(ax, d);
    y[v] = __ddiv_rn(ay, d);
    if (DIM == 3) z[v] = __ddiv_rn(az, d);
  }
}

template <int DIM>
__global__ void __launch_bounds__(256) k_sweep_s1(const int32_t* __restrict__ item_ptr, const int32_t* __restrict__ sv,
                                                  const int32_t* __restrict__ sptr, const int32_t* __restrict__ scol,
                                                  double* x, double* y, double* z, int C, int c, int64_t K) {
  for (int64_t k = blockIdx.x; k < K; k += gridDim.x) {
    const int32_t a = item_ptr[k * C + c], b = item_ptr[k * C + c + 1];
    update_slots<DIM, true>(a, b, sv, sptr, scol, x, y, z);
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

template <int DIM>
__global__ void __launch_bounds__(512) k_sweep_s3(const int32_t* __restrict__ item_ptr, const int32_t* __restrict__ sv,
                                                  const int32_t* __restrict__ sptr, const int32_t* __restrict__ scol,
                                                  const int32_t* __restrict__ klo, const int32_t* __restrict__ khi,
                                                  int* prog, unsigned long long* ticket, double* x, double* y,
                                                  double* z, int C, int64_t K, int L, int sweeps) {
  __shared__ long long sh_t[2];
  const long long per_sweep = (long long)(K + (long long)(C - 1) * L) * C;
  const long long total = per_sweep * sweeps;
  const int lane = threadIdx.x & 31;
  for (int it = 0;; ++it) {
    if (threadIdx.x == 0) sh_t[it & 1] = (long long)atomicAdd(ticket, 1ull);
    __syncthreads();
    const long long t = sh_t[it & 1];
    if (t >= total) break;
    const int s = (int)(t / per_sweep);
    const long long r = t - (long long)s * per_sweep;
    const long long j = r / C;
    const int c = (int)(r - j * C);
    const long long k = j - (long long)c * L;
    if (k < 0 || k >= K) continue;  // no such tile for this key (pipeline fill / drain)
    const int sigma = s * C + c;
    if (threadIdx.x < 32) {
      const int lo = klo[k], hi = khi[k];
      for (int kk = lo + lane; kk <= hi; kk += 32)
        while (ld_relaxed_gpu(prog + kk) < sigma) __nanosleep(32);
      __threadfence();  // acquire: later loads (all warps, after the barrier) see the producers' stores
    }
    __syncthreads();
    const int32_t a = item_ptr[k * C + c], b = item_ptr[k * C + c + 1];
    update_slots<DIM, false>(a, b, sv, sptr, scol, x, y, z);
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      st_release_gpu(prog + k, sigma + 1);
    }
  }
}

// ---------------------------------------------------------------- drivers
static cudaStream_t capture_stream() {
  static thread_local cudaStream_t cs = nullptr;
  if (!cs) LMS_TRY_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
  return cs;
}

static void launch_s1_colours(lms_mesh_s* m, cudaStream_t s) {
  Schedule& S = m->sched;
  const int64_t K = S.K;
  unsigned G = (unsigned)(K < 65535 * 16 ? K : 65535 * 16);
  for (int c = 0; c < m->C; ++c) {
    if (m->dim == 2)
      k_sweep_s1<2><<<G, 256, 0, s>>>(S.item_ptr.p, S.sv.p, S.sptr.p, S.scol.p, m->x[0].p, m->x[1].p, nullptr, m->C,
                                       c, K);
    else
      k_sweep_s1<3><<<G, 256, 0, s>>>(S.item_ptr.p, S.sv.p, S.sptr.p, S.scol.p, m->x[0].p, m->x[1].p, m->x[2].p,
                                       m->C, c, K);
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

void run_sweeps(lms_mesh_s* m, int sweeps, cudaStream_t s) {
  Schedule& S = m->sched;
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
  if (m->dim == 2)
    k_sweep_s3<2><<<ctas, 512, 0, s>>>(S.item_ptr.p, S.sv.p, S.sptr.p, S.scol.p, S.klo.p, S.khi.p, S.prog.p,
                                       S.ticket.p, m->x[0].p, m->x[1].p, nullptr, m->C, S.K, S.lag, sweeps);
  else
    k_sweep_s3<3><<<ctas, 512, 0, s>>>(S.item_ptr.p, S.sv.p, S.sptr.p, S.scol.p, S.klo.p, S.khi.p, S.prog.p,
                                       S.ticket.p, m->x[0].p, m->x[1].p, m->x[2].p, m->C, S.K, S.lag, sweeps);
  LMS_CHECK_LAUNCH();
}

}  // namespace lms
