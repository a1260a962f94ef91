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
// to the sequential definition.  One cooperative persistent kernel runs all
// rounds with one grid barrier per round.
#include <cooperative_groups.h>
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

__global__ void k_jp_rounds(const int32_t* __restrict__ rp, const int32_t* __restrict__ col,
                            const uint8_t* __restrict__ fixed, const int32_t* __restrict__ oid,
                            int32_t* cnt, int8_t* colour, int32_t* q0, int32_t* q1,
                            int* sizes /*[3]*/, int* maxc, int* err) {
  cg::grid_group grid = cg::this_grid();
  int32_t* qs[2] = {q0, q1};
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t nth = (int64_t)gridDim.x * blockDim.x;
  int mymax = -1;
  for (int r = 0;; ++r) {
    const int n = *(volatile int*)&sizes[r % 3];
    if (n == 0) break;
    if (tid == 0) sizes[(r + 2) % 3] = 0;  // appended to during round r+1 (after the barrier)
    int32_t* cur = qs[r & 1];
    int32_t* nxt = qs[(r + 1) & 1];
    int* nsz = &sizes[(r + 1) % 3];
    for (int64_t i = tid; i < n; i += nth) {
      const int32_t v = cur[i];
      const int32_t b = rp[v], e = rp[v + 1];
      unsigned long long used0 = 0, used1 = 0;
      for (int32_t j = b; j < e; ++j) {
        int c = *(volatile int8_t*)&colour[col[j]];
        if (c >= 0) { if (c < 64) used0 |= 1ull << c; else used1 |= 1ull << (c - 64); }
      }
      int c = __ffsll(~used0) - 1;
      if (used0 == ~0ull) c = 64 + __ffsll(~used1) - 1;
      if (used0 == ~0ull && used1 == ~0ull) { raise_err(err, LMS_E_ARG); c = 127; }
      colour[v] = (int8_t)c;
      mymax = c > mymax ? c : mymax;
      __threadfence();
      const int32_t me = oid[v];
      for (int32_t j = b; j < e; ++j) {
        int32_t u = col[j];
        if (!fixed[u] && oid[u] > me)
          if (atomicSub(&cnt[u], 1) == 1) nxt[atomicAdd(nsz, 1)] = u;
      }
    }
    grid.sync();
  }
  if (mymax >= 0) atomicMax(maxc, mymax);
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
    DBuf<int32_t> cnt(V, s), q0(V, s), q1(V, s);
    DBuf<int> sizes(3, s);
    LMS_TRY_CUDA(cudaMemsetAsync(sizes.p, 0, 3 * sizeof(int), s));
    k_jp_init<<<Gv, 256, 0, s>>>(m->row_ptr.p, m->col.p, m->fixed.p, m->orig_id.p, V, cnt.p, m->colour.p, q0.p,
                                 sizes.p);
    LMS_CHECK_LAUNCH();
    int dev = m->device, nsm = 0, occ = 0;
    LMS_TRY_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    LMS_TRY_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_jp_rounds, 256, 0));
    if (occ < 1) fail(LMS_E_CUDA, "colouring kernel cannot be resident");
    int blocks = nsm * (occ < 4 ? occ : 4);
    const int32_t* a_rp = m->row_ptr.p;
    const int32_t* a_col = m->col.p;
    const uint8_t* a_fx = m->fixed.p;
    const int32_t* a_oid = m->orig_id.p;
    int32_t* a_cnt = cnt.p;
    int8_t* a_colour = m->colour.p;
    int32_t* a_q0 = q0.p;
    int32_t* a_q1 = q1.p;
    int* a_sizes = sizes.p;
    int* a_max = maxc.p;
    int* a_err = m->err.p;
    void* args[] = {&a_rp, &a_col, &a_fx, &a_oid, &a_cnt, &a_colour, &a_q0, &a_q1, &a_sizes, &a_max, &a_err};
    LMS_TRY_CUDA(cudaLaunchCooperativeKernel((void*)k_jp_rounds, dim3(blocks), dim3(256), args, 0, s));
    LMS_CHECK_LAUNCH();
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
