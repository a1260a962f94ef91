// colour.cu -- the fixed colouring schedule (reading Z2).
//
// Definition: visit free vertices in ascending orig_id; each takes the smallest
// colour >= 0 not held by an already-coloured free neighbour.  Fixed vertices
// get -1.  The paper's sweep (Alg. 1) is sequential and in
// place; the colouring turns it into C parallel stages without changing the
// smoothing rule.
//
// GPU algorithm: Jones-Plassmann with priority = -orig_id.  A free vertex is
// ready once every lower-orig_id free neighbour is coloured (dependency counter
// reaches 0); ready vertices are pairwise non-adjacent, so a round colours them
// all at once with first-fit.  A vertex is coloured exactly when the sequential
// greedy would have all the information it uses, hence the result is identical
// to the sequential definition.
// Execution: no rounds and no grid barriers (k_jp_warp): persistent warps
// take ready vertices from a queue (or continue with one they just released)
// and colour each one when its counter reaches zero.  The critical path is
// the dependency chain (about nx + 2 ny vertices on a row-major grid) times a
// few memory round trips, instead of one grid barrier per JP round.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cooperative_groups.h>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_reduce.cuh>

#include "lms_internal.cuh"

namespace cg = cooperative_groups;

namespace lms {

__global__ void k_validate_csr(const int32_t* __restrict__ rp, const int32_t* __restrict__ col, int64_t V,
                               int64_t nnz, int* err) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < V; v += (int64_t)gridDim.x * blockDim.x) {
    int32_t b = rp[v], e = rp[v + 1];
    if (b < 0 || e > nnz || e < b) { raise_err(err, LMS_E_ARG); continue; }
    if (e == b) raise_err(err, LMS_E_ISOLATED);
    for (int32_t i = b; i < e; ++i) {
      int32_t u = col[i];
      if (u < 0 || u >= V || u == v) raise_err(err, LMS_E_INDEX);
    }
  }
}

// cnt[v] = number of free neighbours with smaller orig_id; frontier = free vertices with cnt 0
__global__ void k_jp_init(const int32_t* __restrict__ rp, const int32_t* __restrict__ col,
                          const uint8_t* __restrict__ fixed, const int32_t* __restrict__ oid, int64_t V,
                          int32_t* __restrict__ cnt, int8_t* __restrict__ colour, int32_t* __restrict__ q0,
                          int* qsize) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < V; v += (int64_t)gridDim.x * blockDim.x) {
    colour[v] = -1;
    if (fixed[v]) { cnt[v] = 0; continue; }
    int32_t me = oid[v], c = 0;
    for (int32_t i = rp[v]; i < rp[v + 1]; ++i) {
      int32_t u = col[i];
      if (!fixed[u] && oid[u] < me) ++c;
    }
    cnt[v] = c;
    if (c == 0) q0[atomicAdd(qsize, 1)] = (int32_t)v;
  }
}

__device__ __forceinline__ int atom_dec_acq_rel(int* p) {
  int old;
  asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], -1;" : "=r"(old) : "l"(p) : "memory");
  return old;
}
__device__ __forceinline__ int atom_dec_relaxed(int* p) {
  int old;
  asm volatile("atom.relaxed.gpu.global.add.s32 %0, [%1], -1;" : "=r"(old) : "l"(p) : "memory");
  return old;
}
__device__ __forceinline__ void fence_acq_rel() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ void st_release(int32_t* p, int32_t v) {
  asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int32_t ld_acquire(const int32_t* p) {
  int32_t v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Per-vertex dependency record (stride RS ints): [0] = n_lo | n_hi << 16,
// then the n_lo lower-orig_id neighbours (any, fixed ones included: their
// colour is -1), then the n_hi higher-orig_id FREE neighbours.  Built in one
// coalesced pass so that a hop of the colouring's critical path costs one
// record load instead of walks over rp / col / oid / fixed.
__global__ void k_jp_records(const int32_t* __restrict__ rp, const int32_t* __restrict__ col,
                             const uint8_t* __restrict__ fixed, const int32_t* __restrict__ oid, int64_t V, int RS,
                             int32_t* rec) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < V; v += (int64_t)gridDim.x * blockDim.x) {
    if (fixed[v]) continue;
    int32_t* r = rec + v * RS;
    const int32_t me = oid[v];
    int nl = 0, nh = 0;
    for (int32_t j = rp[v]; j < rp[v + 1]; ++j) {
      const int32_t u = col[j];
      if (oid[u] < me) r[1 + nl++] = u;
    }
    for (int32_t j = rp[v]; j < rp[v + 1]; ++j) {
      const int32_t u = col[j];
      if (!fixed[u] && oid[u] > me) r[1 + nl + nh++] = u;
    }
    r[0] = nl | (nh << 16);
  }
}

// Dataflow JP with a ready queue.  Q[0..n_free): ready vertices in push order
// (-1 = not yet pushed).  Counters, each on its own 128-byte line:
// sizes[0] = pushes (initialised to the frontier size), sizes[32] = pops,
// sizes[64] = vertices coloured.  One warp per vertex (lane j handles the
// row's j-th neighbour; longer rows in passes).  The warp whose decrement
// makes a dependent ready continues with it directly (no queue round trip);
// other newly ready vertices are pushed.  A warp adds its coloured count to
// sizes[64] only when it goes idle (before popping), so that counter is not
// a per-vertex hot spot; the warp whose flush completes n_free raises the
// done flag sizes[96], which a warp waiting on an unfilled slot (continuations
// consume no slot, so some slots stay empty) polls besides its slot.
__global__ void __launch_bounds__(256) k_jp_warp(const int32_t* __restrict__ rec, int RS, int32_t* cnt,
                                                 int8_t* colour, int32_t* Q, int* sizes, int n_free, int* maxc,
                                                 int* err, unsigned long long* stats) {
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  int mymax = -1, done = 0;
  int32_t v = -1;
  unsigned long long t_idle = 0, t_work = 0, n_v = 0, n_pop = 0;
  long long tc = clock64();
  for (;;) {
    if (stats) { const long long t = clock64(); t_work += t - tc; tc = t; }
    if (v < 0) {  // idle: flush the count, then pop the next queue slot
      if (stats) ++n_pop;
      int fin = 0;
      if (lane == 0 && done > 0) fin = atomicAdd(&sizes[64], done) + done == n_free;
      done = 0;
      if (__shfl_sync(FULL, fin, 0)) {  // everything coloured: release the waiting warps
        if (lane == 0) st_release(&sizes[96], 1);
        break;
      }
      int i = 0;
      if (lane == 0) i = atomicAdd(&sizes[32], 1);
      i = __shfl_sync(FULL, i, 0);
      if (i >= n_free) break;
      if (lane == 0) {
        long long spins = 0;
        while ((v = ld_acquire(&Q[i])) == -1) {  // acquire: pairs with the pusher's release
          if (ld_acquire(&sizes[96])) { v = -3; break; }  // everything coloured
          if (++spins > (1ll << 31)) { raise_err(err, LMS_E_CUDA); v = -2; break; }  // cannot happen (acyclic)
          __nanosleep(32);
        }
      }
      v = __shfl_sync(FULL, v, 0);
      if (v < 0) break;  // -3: all coloured; -2: error
      if (stats) { const long long t = clock64(); t_idle += t - tc; tc = t; }
    }
    if (stats) ++n_v;
    // v's lower-orig_id neighbours' colours are visible (fences around the
    // colour stores and the counter decrements; see below)
    const int32_t* rv = rec + (int64_t)v * RS;
    const int32_t x0 = lane < RS ? rv[lane] : 0;  // the record, one coalesced load per 32 entries
    const int32_t hdr = __shfl_sync(FULL, x0, 0);
    const int nl = hdr & 0xffff, nh = hdr >> 16;
    // record entries 1..nl: lower neighbours; nl+1..nl+nh: the dependents
    uint32_t used[4] = {0, 0, 0, 0};
    for (int q0 = 0; q0 <= nl; q0 += 32) {
      const int q = q0 + lane;
      const int32_t x = q0 == 0 ? x0 : (q < RS ? rv[q] : 0);
      const int cl = (q >= 1 && q <= nl) ? *(volatile int8_t*)&colour[x] : -1;
#pragma unroll
      for (int w = 0; w < 4; ++w)
        used[w] |= __reduce_or_sync(FULL, (cl >= 32 * w && cl < 32 * w + 32) ? 1u << (cl - 32 * w) : 0u);
    }
    int c = 127;
    for (int w = 0; w < 4; ++w)
      if (used[w] != 0xffffffffu) { c = 32 * w + __ffs(~used[w]) - 1; break; }
    if (c == 127) raise_err(err, LMS_E_ARG);
    if (lane == 0) {
      *(volatile int8_t*)&colour[v] = (int8_t)c;
      fence_acq_rel();  // release the colour before the decrements
    }
    mymax = c > mymax ? c : mymax;
    ++done;
    __syncwarp();
    int32_t next = -1;
    for (int q0 = (nl + 1) & ~31; q0 <= nl + nh; q0 += 32) {
      const int q = q0 + lane;
      const int32_t x = q0 == 0 ? x0 : (q < RS ? rv[q] : 0);
      const bool isdep = q > nl && q <= nl + nh;
      const bool ready = isdep && atom_dec_relaxed(&cnt[x]) == 1;
      unsigned rb = __ballot_sync(FULL, ready);
      if (ready) fence_acq_rel();  // acquire: the colours released before the other decrements
      __syncwarp();
      bool push = ready;
      if (next < 0 && rb) {  // continue with the first newly ready vertex
        const int src = __ffs(rb) - 1;
        next = __shfl_sync(FULL, x, src);
        rb &= rb - 1;
        if (lane == src) push = false;
      }
      if (rb) {  // push the others (release: the popper acquires the colours this lane saw)
        int p = 0;
        if (lane == 0) p = atomicAdd(&sizes[0], __popc(rb));
        p = __shfl_sync(FULL, p, 0);
        if (push) st_release(&Q[p + __popc(rb & ((1u << lane) - 1))], x);
      }
    }
    v = next;
  }
  if (lane == 0 && mymax >= 0) atomicMax(maxc, mymax);
  if (stats && lane == 0) {
    atomicAdd(stats + 0, t_idle);
    atomicAdd(stats + 1, t_work);
    atomicAdd(stats + 2, n_v);
    atomicAdd(stats + 3, n_pop);
  }
}

__global__ void k_max_deg(const int32_t* __restrict__ rp, int64_t V, int* out) {
  int mx = 0;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < V; v += (int64_t)gridDim.x * blockDim.x)
    mx = max(mx, rp[v + 1] - rp[v]);
  for (int o = 16; o; o >>= 1) mx = max(mx, __shfl_down_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, mx);
}

__global__ void k_colour_max(const int8_t* __restrict__ colour, const uint8_t* __restrict__ fixed, int64_t V,
                             int* maxc, int* err) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < V; v += (int64_t)gridDim.x * blockDim.x) {
    int c = colour[v];
    if (fixed[v] ? (c != -1) : (c < 0)) raise_err(err, LMS_E_ARG);
    if (c >= 0) atomicMax(maxc, c);
  }
}

__global__ void k_check_all_coloured(const int8_t* __restrict__ colour, const uint8_t* __restrict__ fixed,
                                     int64_t V, int* err) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < V; v += (int64_t)gridDim.x * blockDim.x)
    if (!fixed[v] && colour[v] < 0) raise_err(err, LMS_E_ARG);
}

void compute_colouring(lms_mesh_s* m, cudaStream_t s) {
  const int64_t V = m->V;
  const unsigned Gv = grid_for(V, 256) > 8192 ? 8192 : grid_for(V, 256);
  k_validate_csr<<<Gv, 256, 0, s>>>(m->row_ptr.p, m->col.p, V, m->nnz, m->err.p);
  LMS_CHECK_LAUNCH();
  check_err_flag(m, s, "CSR validation");
  DBuf<int> maxc(1, s);
  LMS_TRY_CUDA(cudaMemsetAsync(maxc.p, 0xff, sizeof(int), s));  // -1
  if (m->colour.p) {  // caller-supplied colouring (lms_mesh_from_csr)
    k_colour_max<<<Gv, 256, 0, s>>>(m->colour.p, m->fixed.p, V, maxc.p, m->err.p);
    LMS_CHECK_LAUNCH();
    check_err_flag(m, s, "colour (fixed vertices must have colour -1, free ones >= 0)");
  } else {
    m->colour.alloc(V, s);
    DBuf<int32_t> cnt(V, s), Q(V, s);
    DBuf<int> sizes(128, s);
    LMS_TRY_CUDA(cudaMemsetAsync(sizes.p, 0, 128 * sizeof(int), s));
    LMS_TRY_CUDA(cudaMemsetAsync(Q.p, 0xff, V * sizeof(int32_t), s));
    k_jp_init<<<Gv, 256, 0, s>>>(m->row_ptr.p, m->col.p, m->fixed.p, m->orig_id.p, V, cnt.p, m->colour.p, Q.p,
                                 sizes.p);
    LMS_CHECK_LAUNCH();
    const int64_t n_free = count_free(m, s);
    // records: 1 + max degree ints, rounded to 4 (one warp load per 32)
    int maxdeg = 0;
    {
      DBuf<int> md(1, s);
      LMS_TRY_CUDA(cudaMemsetAsync(md.p, 0, sizeof(int), s));
      k_max_deg<<<Gv, 256, 0, s>>>(m->row_ptr.p, V, md.p);
      LMS_CHECK_LAUNCH();
      LMS_TRY_CUDA(cudaMemcpyAsync(&maxdeg, md.p, sizeof(int), cudaMemcpyDeviceToHost, s));
      LMS_TRY_CUDA(cudaStreamSynchronize(s));
    }
    const int RS = (1 + maxdeg + 3) & ~3;
    DBuf<int32_t> jrec((size_t)V * RS, s);
    k_jp_records<<<Gv, 256, 0, s>>>(m->row_ptr.p, m->col.p, m->fixed.p, m->orig_id.p, V, RS, jrec.p);
    LMS_CHECK_LAUNCH();
    if (n_free > 0) {
      // persistent warps, co-resident (a warp may wait on any other warp)
      int dev = m->device, nsm = 0, occ = 0;
      const int threads = 256;
      LMS_TRY_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
      LMS_TRY_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_jp_warp, threads, 0));
      if (occ < 1) fail(LMS_E_CUDA, "colouring kernel cannot be resident");
      int blocks = nsm;
      if (const char* e = getenv("LMS_JP_BLOCKS")) blocks = std::max(1, std::min(atoi(e), nsm * occ));
      const int32_t* a_rec = jrec.p;
      int a_rs = RS;
      int32_t* a_cnt = cnt.p;
      int8_t* a_colour = m->colour.p;
      int32_t* a_q = Q.p;
      int* a_sizes = sizes.p;
      int a_n = (int)n_free;
      int* a_max = maxc.p;
      int* a_err = m->err.p;
      unsigned long long* a_stats = nullptr;
      static unsigned long long* jst = nullptr;
      if (getenv("LMS_JP_STATS")) {
        if (!jst) LMS_TRY_CUDA(cudaMalloc(&jst, 4 * sizeof(unsigned long long)));
        LMS_TRY_CUDA(cudaMemsetAsync(jst, 0, 4 * sizeof(unsigned long long), s));
        a_stats = jst;
      }
      void* args[] = {&a_rec, &a_rs, &a_cnt, &a_colour, &a_q, &a_sizes, &a_n, &a_max, &a_err, &a_stats};
      LMS_TRY_CUDA(cudaLaunchCooperativeKernel((void*)k_jp_warp, dim3(blocks), dim3(threads), args, 0, s));
      LMS_CHECK_LAUNCH();
      if (a_stats) {
        unsigned long long h[4];
        LMS_TRY_CUDA(cudaMemcpyAsync(h, a_stats, sizeof(h), cudaMemcpyDeviceToHost, s));
        LMS_TRY_CUDA(cudaStreamSynchronize(s));
        const double nv = h[2] ? (double)h[2] : 1.0;
        fprintf(stderr, "[jp stats] warps=%d vertices=%llu pops=%llu (continuations %.1f%%) work=%.0f cyc/vertex "
                "idle=%.0f cyc/warp\n", blocks * threads / 32, h[2], h[3], 100.0 * (1.0 - h[3] / nv), h[1] / nv,
                h[0] / (blocks * threads / 32.0));
      }
    }
    k_check_all_coloured<<<Gv, 256, 0, s>>>(m->colour.p, m->fixed.p, V, m->err.p);
    LMS_CHECK_LAUNCH();
    check_err_flag(m, s, "colouring (more than 127 colours, or an inconsistent orig_id)");
  }
  int h = -1;
  LMS_TRY_CUDA(cudaMemcpyAsync(&h, maxc.p, sizeof(int), cudaMemcpyDeviceToHost, s));
  LMS_TRY_CUDA(cudaStreamSynchronize(s));
  m->C = h + 1;
}

}  // namespace lms
