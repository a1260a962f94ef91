// permute.cu -- relabel the mesh by a permutation.
// perm[new] = old.  inv[perm[k]] = k; X'[k] = X[perm[k]] for
// coordinates, fixed, colour, orig_id, quality; elements' = inv[elements]
// (element and slot order kept); CSR row k' = inv[row perm[k']], re-sorted.
// The handle is validated (bijection) before anything is modified.
#include <cub/device/device_scan.cuh>

#include "lms_internal.cuh"

namespace lms {

__global__ void k_inverse(const int32_t* __restrict__ perm, int64_t V, int32_t* inv, int* err, int* moved) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < V; k += (int64_t)gridDim.x * blockDim.x) {
    int32_t p = perm[k];
    if (p != k && !*(volatile int*)moved) *moved = 1;
    if (p < 0 || p >= V) { raise_err(err, LMS_E_PERM); continue; }
    int32_t old = atomicExch(&inv[p], (int32_t)k);
    if (old != -1) raise_err(err, LMS_E_PERM);
  }
}

template <typename T>
__global__ void k_gather(const T* __restrict__ src, const int32_t* __restrict__ perm, int64_t V, T* __restrict__ dst) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < V; k += (int64_t)gridDim.x * blockDim.x)
    dst[k] = src[perm[k]];
}

__global__ void k_new_deg(const int32_t* __restrict__ rp, const int32_t* __restrict__ perm, int64_t V, int32_t* deg) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k <= V; k += (int64_t)gridDim.x * blockDim.x)
    deg[k] = (k < V) ? rp[perm[k] + 1] - rp[perm[k]] : 0;
}

// eight lanes per row (rows have ~6 entries in 2D, ~14 in 3D)
__global__ void k_fill_rows(const int32_t* __restrict__ rp, const int32_t* __restrict__ col,
                            const int32_t* __restrict__ perm, const int32_t* __restrict__ inv,
                            const int32_t* __restrict__ rp2, int64_t V, int32_t* __restrict__ col2) {
  const int sub = threadIdx.x & 7;
  const int64_t g = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 3;
  const int64_t ng = ((int64_t)gridDim.x * blockDim.x) >> 3;
  for (int64_t k = g; k < V; k += ng) {
    const int32_t old = perm[k];
    const int32_t b = rp[old], d = rp[old + 1] - b, o = rp2[k];
    for (int32_t j = sub; j < d; j += 8) col2[o + j] = inv[col[b + j]];
  }
}

__global__ void k_remap(int32_t* __restrict__ a, int64_t n, const int32_t* __restrict__ inv) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    a[i] = inv[a[i]];
}

void permute_mesh(lms_mesh_s* m, const int32_t* d_perm, cudaStream_t s) {
  sync_soa(m, s);
  const int64_t V = m->V, nnz = m->nnz;
  const unsigned Gv = grid_for(V, 256) > 8192 ? 8192 : grid_for(V, 256);
  DBuf<int32_t> inv(V, s);
  DBuf<int> moved(1, s);
  LMS_TRY_CUDA(cudaMemsetAsync(inv.p, 0xff, V * sizeof(int32_t), s));
  LMS_TRY_CUDA(cudaMemsetAsync(moved.p, 0, sizeof(int), s));
  k_inverse<<<Gv, 256, 0, s>>>(d_perm, V, inv.p, m->err.p, moved.p);
  LMS_CHECK_LAUNCH();
  check_err_flag(m, s, "lms_permute");  // nothing modified yet
  int h_moved = 1;
  LMS_TRY_CUDA(cudaMemcpyAsync(&h_moved, moved.p, sizeof(int), cudaMemcpyDeviceToHost, s));
  LMS_TRY_CUDA(cudaStreamSynchronize(s));
  if (!h_moved) {  // the identity (the original ordering): every array stays as it is
    m->sched.valid = false;
    soa_changed(m);
    return;
  }

  for (int a = 0; a < m->dim; ++a) {
    DBuf<double> nx(V, s);
    k_gather<double><<<Gv, 256, 0, s>>>(m->x[a].p, d_perm, V, nx.p);
    LMS_CHECK_LAUNCH();
    m->x[a] = std::move(nx);
  }
  {
    DBuf<uint8_t> nf(V, s);
    k_gather<uint8_t><<<Gv, 256, 0, s>>>(m->fixed.p, d_perm, V, nf.p);
    LMS_CHECK_LAUNCH();
    m->fixed = std::move(nf);
    DBuf<int8_t> nc(V, s);
    k_gather<int8_t><<<Gv, 256, 0, s>>>(m->colour.p, d_perm, V, nc.p);
    LMS_CHECK_LAUNCH();
    m->colour = std::move(nc);
    DBuf<int32_t> no(V, s);
    k_gather<int32_t><<<Gv, 256, 0, s>>>(m->orig_id.p, d_perm, V, no.p);
    LMS_CHECK_LAUNCH();
    m->orig_id = std::move(no);
    if (m->quality.p) {
      DBuf<double> nq(V, s);
      k_gather<double><<<Gv, 256, 0, s>>>(m->quality.p, d_perm, V, nq.p);
      LMS_CHECK_LAUNCH();
      m->quality = std::move(nq);
    }
  }
  {
    DBuf<int32_t> deg(V + 1, s), rp2(V + 1, s), col2(nnz, s);
    const unsigned Gv1 = grid_for(V + 1, 256) > 8192 ? 8192 : grid_for(V + 1, 256);
    k_new_deg<<<Gv1, 256, 0, s>>>(m->row_ptr.p, d_perm, V, deg.p);
    LMS_CHECK_LAUNCH();
    size_t tb = 0;
    LMS_TRY_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, deg.p, rp2.p, V + 1, s));
    {
      DBuf<char> tmp(tb, s);
      LMS_TRY_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tb, deg.p, rp2.p, V + 1, s));
    }
    unsigned Gw = grid_for(V * 8, 256) > 8192 ? 8192 : grid_for(V * 8, 256);
    k_fill_rows<<<Gw, 256, 0, s>>>(m->row_ptr.p, m->col.p, d_perm, inv.p, rp2.p, V, col2.p);
    LMS_CHECK_LAUNCH();
    segmented_sort_rows(col2.p, rp2.p, V, nnz, s);
    m->row_ptr = std::move(rp2);
    m->col = std::move(col2);
  }
  if (m->k) {
    const int64_t n = m->n_el * m->k;
    k_remap<<<grid_for(n, 256) > 8192 ? 8192 : grid_for(n, 256), 256, 0, s>>>(m->elems.p, n, inv.p);
    LMS_CHECK_LAUNCH();
  }
  m->sched.valid = false;
  m->v2e_valid = false;  // vertex labels changed (elements keep their order)
  soa_changed(m);
}

}  // namespace lms
