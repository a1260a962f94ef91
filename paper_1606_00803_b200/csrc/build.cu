// build.cu -- CSR construction, fixed mask (A3) and
// edge-length-ratio quality (A4) on the GPU.
//
//  A2: every element emits its k(k-1) directed vertex pairs as packed 64-bit
//      keys (u << b | v); a radix sort + run-length encode gives the unique
//      directed edges in (row, col) order, i.e. the CSR with ascending rows;
//      the run lengths are the edge multiplicities.  N(v) = vertices sharing an
//      element with v ("N neighbored vertices", Eq. 1).
//  A3: Alg. 1 smooths "interior vertices".  A vertex is fixed iff it is
//      on an edge (triangles: multiplicity-1 directed key) or face (tetrahedra:
//      sorted face triples, LSD two-pass radix sort) owned by one element.
//  A4: q_e = sqrt(min l^2)/sqrt(max l^2) over the element's edges (slot pairs in
//      lexicographic order, l^2 = dx*dx + dy*dy [+ dz*dz], every op separately
//      rounded), q_v = (sum of q_e over attached elements, ascending element id)
//      / count.
#include <chrono>
#include <cstdio>
#include <cstring>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_reduce.cuh>
#include <cub/device/device_run_length_encode.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_segmented_sort.cuh>

#include "lms_internal.cuh"

namespace lms {

static int bits_for(int64_t n) {  // smallest b with 2^b >= n (b >= 1)
  int b = 1;
  while (((int64_t)1 << b) < n) ++b;
  return b;
}

__global__ void k_iota(int32_t* p, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = (int32_t)i;
}

void fill_iota(int32_t* p, int64_t n, cudaStream_t s) {
  k_iota<<<grid_for(n, 256) > 4096 ? 4096 : grid_for(n, 256), 256, 0, s>>>(p, n);
  LMS_CHECK_LAUNCH();
}

// -------------------------------------------------------------- validation + expand
__global__ void k_validate_elems(const int32_t* __restrict__ el, int64_t n_el, int k, int64_t V, int* err) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n_el; e += (int64_t)gridDim.x * blockDim.x) {
    int32_t w[4];
    for (int s = 0; s < k; ++s) w[s] = el[e * k + s];
    bool bad = false;
    for (int s = 0; s < k; ++s) {
      if (w[s] < 0 || w[s] >= V) bad = true;
      for (int t = 0; t < s; ++t) bad |= (w[t] == w[s]);
    }
    if (bad) raise_err(err, LMS_E_INDEX);
  }
}

__global__ void k_expand_pairs(const int32_t* __restrict__ el, int64_t n_el, int k, int b,
                               unsigned long long* __restrict__ keys) {
  const int per = k * (k - 1);
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n_el; e += (int64_t)gridDim.x * blockDim.x) {
    int32_t w[4];
    for (int s = 0; s < k; ++s) w[s] = el[e * k + s];
    int o = 0;
    for (int s = 0; s < k; ++s)
      for (int t = 0; t < k; ++t)
        if (s != t) keys[e * per + (o++)] = ((unsigned long long)w[s] << b) | (unsigned long long)w[t];
  }
}

// unique sorted keys -> col, row_ptr; multiplicity-1 undirected edges -> fixed (triangles)
__global__ void k_keys_to_csr(const unsigned long long* __restrict__ uk, const int* __restrict__ cnt, int64_t nnz,
                              int b, int64_t V, int32_t* __restrict__ col, int32_t* __restrict__ row_ptr,
                              uint8_t* fixed_or_null) {
  const unsigned long long mask = (1ull << b) - 1;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nnz; i += (int64_t)gridDim.x * blockDim.x) {
    unsigned long long key = uk[i];
    int64_t r = (int64_t)(key >> b);
    int32_t c = (int32_t)(key & mask);
    col[i] = c;
    int64_t rprev = (i == 0) ? -1 : (int64_t)(uk[i - 1] >> b);
    for (int64_t q = rprev + 1; q <= r; ++q) row_ptr[q] = (int32_t)i;
    if (i == nnz - 1)
      for (int64_t q = r + 1; q <= V; ++q) row_ptr[q] = (int32_t)nnz;
    if (fixed_or_null && cnt[i] == 1) {  // edge in exactly one triangle: both endpoints fixed
      fixed_or_null[r] = 1;
      fixed_or_null[c] = 1;
    }
  }
}

// ---- bucketed CSR: pairs scattered into per-source buckets, rows sorted and
// de-duplicated locally (same CSR as the global sort: rows ascending, unique)
__global__ void k_pair_count(const int32_t* __restrict__ el, int64_t n_el, int k, int32_t* cnt) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n_el; e += (int64_t)gridDim.x * blockDim.x)
    for (int s = 0; s < k; ++s) atomicAdd(&cnt[el[e * k + s]], k - 1);
}
__global__ void k_pair_scatter(const int32_t* __restrict__ el, int64_t n_el, int k, int32_t* cur, int32_t* buf) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n_el; e += (int64_t)gridDim.x * blockDim.x) {
    int32_t w[4];
    for (int s = 0; s < k; ++s) w[s] = el[e * k + s];
    for (int s = 0; s < k; ++s) {
      const int32_t p = atomicAdd(&cur[w[s]], k - 1);
      int o = 0;
      for (int t = 0; t < k; ++t)
        if (t != s) buf[p + o++] = w[t];
    }
  }
}
constexpr int CSR_ROW_CAP = 128;  // longer bucketed rows: the global-sort path
// row v: sort its bucket in place (no per-thread stack array: a kernel that
// needs a large local-memory reservation can make the driver resize it at
// launch, an occasional stall of hundreds of ms), drop duplicates, ndeg[v] =
// unique count; triangles: a neighbour seen once is an edge of one triangle ->
// v is boundary
__global__ void k_row_unique(const int32_t* __restrict__ off, int32_t* buf, int64_t V, int32_t* ndeg,
                             uint8_t* fixed_or_null) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < V; v += (int64_t)gridDim.x * blockDim.x) {
    int32_t* a = buf + off[v];
    const int32_t L = off[v + 1] - off[v];
    if (L <= 16) {  // registers: a 16-wide bitonic network, then de-duplicate
      int32_t r[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) r[i] = i < L ? a[i] : INT32_MAX;
#pragma unroll
      for (int k = 2; k <= 16; k <<= 1)
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1)
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const int l = i ^ j;
            if (l > i) {
              const bool up = (i & k) == 0;
              const int32_t x = r[i], y = r[l];
              if ((x > y) == up) {
                r[i] = y;
                r[l] = x;
              }
            }
          }
      int u = 0;
      bool single = false;
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        if (i >= L) break;
        const bool first = i == 0 || r[i] != r[i - 1];
        const bool last = i == L - 1 || r[i] != r[i + 1];
        single |= first && last;
        if (first) a[u++] = r[i];
      }
      ndeg[v] = u;
      if (fixed_or_null && single) fixed_or_null[v] = 1;
      continue;
    }
    for (int i = 1; i < L; ++i) {  // insertion sort (rows are short)
      const int32_t x = a[i];
      int j = i;
      while (j > 0 && a[j - 1] > x) {
        a[j] = a[j - 1];
        --j;
      }
      a[j] = x;
    }
    int u = 0;
    bool single = false;
    for (int i = 0; i < L;) {
      const int32_t x = a[i];
      int j = i + 1;
      while (j < L && a[j] == x) ++j;
      single |= (j - i) == 1;
      a[u++] = x;
      i = j;
    }
    ndeg[v] = u;
    if (fixed_or_null && single) fixed_or_null[v] = 1;
  }
}
// eight lanes per row: unique bucket prefix -> col
__global__ void k_row_compact(const int32_t* __restrict__ off, const int32_t* __restrict__ buf,
                              const int32_t* __restrict__ row_ptr, int64_t V, int32_t* __restrict__ col) {
  const int sub = threadIdx.x & 7;
  const int64_t g = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 3;
  const int64_t ng = ((int64_t)gridDim.x * blockDim.x) >> 3;
  for (int64_t v = g; v < V; v += ng) {
    const int32_t b = off[v], o = row_ptr[v], d = row_ptr[v + 1] - o;
    for (int32_t j = sub; j < d; j += 8) col[o + j] = buf[b + j];
  }
}

static bool build_csr_bucketed(lms_mesh_s* m, bool want_boundary, cudaStream_t s) {
  const bool tv = getenv("LMS_BUILD_VERBOSE") != nullptr;
  auto t_last = std::chrono::steady_clock::now();
  auto mark = [&](const char* what) {
    if (!tv) return;
    cudaStreamSynchronize(s);
    const auto t = std::chrono::steady_clock::now();
    fprintf(stderr, "[csr] %-10s %8.2f ms\n", what, std::chrono::duration<double, std::milli>(t - t_last).count());
    t_last = t;
  };
  const int k = m->k;
  const int64_t n_el = m->n_el, V = m->V;
  const unsigned Ge = grid_for(n_el, 256) > 8192 ? 8192 : grid_for(n_el, 256);
  const unsigned Gv = grid_for(V, 256) > 8192 ? 8192 : grid_for(V, 256);
  DBuf<int32_t> cnt(V + 1, s), off(V + 1, s), mx(1, s);
  LMS_TRY_CUDA(cudaMemsetAsync(cnt.p, 0, (V + 1) * sizeof(int32_t), s));
  mark("alloc0");
  k_pair_count<<<Ge, 256, 0, s>>>(m->elems.p, n_el, k, cnt.p);
  LMS_CHECK_LAUNCH();
  mark("count");
  size_t tb = 0, tb2 = 0;
  LMS_TRY_CUDA(cub::DeviceReduce::Max(nullptr, tb, cnt.p, mx.p, V, s));
  LMS_TRY_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb2, cnt.p, off.p, V + 1, s));
  DBuf<char> tmp(std::max(tb, tb2), s);
  LMS_TRY_CUDA(cub::DeviceReduce::Max(tmp.p, tb, cnt.p, mx.p, V, s));
  int h_mx = 0;
  LMS_TRY_CUDA(cudaMemcpyAsync(&h_mx, mx.p, sizeof(int), cudaMemcpyDeviceToHost, s));
  LMS_TRY_CUDA(cudaStreamSynchronize(s));
  if (h_mx > CSR_ROW_CAP) return false;
  LMS_TRY_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tb2, cnt.p, off.p, V + 1, s));
  const int64_t nk = n_el * k * (k - 1);
  mark("scan");
  DBuf<int32_t> buf(nk, s);
  mark("alloc_buf");
  LMS_TRY_CUDA(cudaMemcpyAsync(cnt.p, off.p, (V + 1) * sizeof(int32_t), cudaMemcpyDeviceToDevice, s));  // cursors
  k_pair_scatter<<<Ge, 256, 0, s>>>(m->elems.p, n_el, k, cnt.p, buf.p);
  LMS_CHECK_LAUNCH();
  mark("scatter");
  uint8_t* fx = nullptr;
  if (want_boundary) {
    LMS_TRY_CUDA(cudaMemsetAsync(m->fixed.p, 0, V, s));
    if (k == 3) fx = m->fixed.p;
  }
  LMS_TRY_CUDA(cudaMemsetAsync(cnt.p + V, 0, sizeof(int32_t), s));
  k_row_unique<<<Gv, 256, 0, s>>>(off.p, buf.p, V, cnt.p, fx);
  LMS_CHECK_LAUNCH();
  mark("unique");
  m->row_ptr.alloc(V + 1, s);
  LMS_TRY_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tb2, cnt.p, m->row_ptr.p, V + 1, s));
  int h_nnz = 0;
  LMS_TRY_CUDA(cudaMemcpyAsync(&h_nnz, m->row_ptr.p + V, sizeof(int), cudaMemcpyDeviceToHost, s));
  LMS_TRY_CUDA(cudaStreamSynchronize(s));
  m->nnz = h_nnz;
  m->col.alloc(m->nnz, s);
  const unsigned Gw = grid_for(V * 8, 256) > 8192 ? 8192 : grid_for(V * 8, 256);
  mark("scan2");
  k_row_compact<<<Gw, 256, 0, s>>>(off.p, buf.p, m->row_ptr.p, V, m->col.p);
  LMS_CHECK_LAUNCH();
  mark("compact");
  return true;
}

__global__ void k_check_isolated(const int32_t* __restrict__ row_ptr, int64_t V, int* err) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < V; v += (int64_t)gridDim.x * blockDim.x)
    if (row_ptr[v + 1] == row_ptr[v]) raise_err(err, LMS_E_ISOLATED);
}

// -------------------------------------------------------------- 3D faces
__device__ __forceinline__ void face_of(const int32_t* el, int64_t f, int32_t& a, int32_t& b, int32_t& c) {
  int64_t e = f >> 2;
  int skip = (int)(f & 3);
  int32_t v[3];
  int n = 0;
  for (int s = 0; s < 4; ++s)
    if (s != skip) v[n++] = el[e * 4 + s];
  // sort 3
  if (v[0] > v[1]) { int32_t t = v[0]; v[0] = v[1]; v[1] = t; }
  if (v[1] > v[2]) { int32_t t = v[1]; v[1] = v[2]; v[2] = t; }
  if (v[0] > v[1]) { int32_t t = v[0]; v[0] = v[1]; v[1] = t; }
  a = v[0]; b = v[1]; c = v[2];
}

__global__ void k_face_c(const int32_t* el, int64_t nf, uint32_t* kc, uint32_t* idx) {
  for (int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; f < nf; f += (int64_t)gridDim.x * blockDim.x) {
    int32_t a, b, c;
    face_of(el, f, a, b, c);
    kc[f] = (uint32_t)c;
    idx[f] = (uint32_t)f;
  }
}

__global__ void k_face_ab(const int32_t* el, const uint32_t* idx, int64_t nf, int bb, unsigned long long* kab) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nf; i += (int64_t)gridDim.x * blockDim.x) {
    int32_t a, b, c;
    face_of(el, idx[i], a, b, c);
    kab[i] = ((unsigned long long)a << bb) | (unsigned long long)b;
  }
}

__global__ void k_face_mark(const int32_t* el, const uint32_t* idx, int64_t nf, uint8_t* fixed) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nf; i += (int64_t)gridDim.x * blockDim.x) {
    int32_t a, b, c, a2, b2, c2;
    face_of(el, idx[i], a, b, c);
    bool same_prev = false, same_next = false;
    if (i > 0) {
      face_of(el, idx[i - 1], a2, b2, c2);
      same_prev = (a == a2 && b == b2 && c == c2);
    }
    if (i + 1 < nf) {
      face_of(el, idx[i + 1], a2, b2, c2);
      same_next = (a == a2 && b == b2 && c == c2);
    }
    if (!same_prev && !same_next) {
      fixed[a] = 1;
      fixed[b] = 1;
      fixed[c] = 1;
    }
  }
}

static void boundary_faces(lms_mesh_s* m, cudaStream_t s) {
  const int64_t nf = m->n_el * 4;
  const int bb = bits_for(m->V);
  DBuf<uint32_t> kc(nf, s), kc2(nf, s), idx(nf, s), idx2(nf, s);
  const unsigned G = grid_for(nf, 256) > 8192 ? 8192 : grid_for(nf, 256);
  k_face_c<<<G, 256, 0, s>>>(m->elems.p, nf, kc.p, idx.p);
  LMS_CHECK_LAUNCH();
  size_t tb = 0;
  LMS_TRY_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, kc.p, kc2.p, idx.p, idx2.p, nf, 0, bb, s));
  {
    DBuf<char> tmp(tb, s);
    LMS_TRY_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tb, kc.p, kc2.p, idx.p, idx2.p, nf, 0, bb, s));
  }
  DBuf<unsigned long long> kab(nf, s), kab2(nf, s);
  k_face_ab<<<G, 256, 0, s>>>(m->elems.p, idx2.p, nf, bb, kab.p);
  LMS_CHECK_LAUNCH();
  tb = 0;
  LMS_TRY_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, kab.p, kab2.p, idx2.p, idx.p, nf, 0, 2 * bb, s));
  {
    DBuf<char> tmp(tb, s);
    LMS_TRY_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tb, kab.p, kab2.p, idx2.p, idx.p, nf, 0, 2 * bb, s));
  }
  k_face_mark<<<G, 256, 0, s>>>(m->elems.p, idx.p, nf, m->fixed.p);
  LMS_CHECK_LAUNCH();
}

void build_csr_from_elems(lms_mesh_s* m, const int32_t* d_elems, bool want_boundary, cudaStream_t s) {
  const int k = m->k;
  const int64_t n_el = m->n_el, V = m->V;
  if (d_elems) {  // NULL: the caller filled m->elems (lms_build_csr_host)
    m->elems.alloc(n_el * k, s);
    LMS_TRY_CUDA(cudaMemcpyAsync(m->elems.p, d_elems, n_el * k * sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
  }
  const unsigned Ge = grid_for(n_el, 256) > 8192 ? 8192 : grid_for(n_el, 256);
  k_validate_elems<<<Ge, 256, 0, s>>>(m->elems.p, n_el, k, V, m->err.p);
  LMS_CHECK_LAUNCH();
  check_err_flag(m, s, "lms_build_csr");

  const int b = bits_for(V);
  const int64_t nk = n_el * k * (k - 1);
  if (nk >= ((int64_t)1 << 31)) fail(LMS_E_ARG, "too many element pairs for the CSR build");
  const char* ce = getenv("LMS_CSR");
  if (!(ce && !strcmp(ce, "sort")) && build_csr_bucketed(m, want_boundary, s)) {
    if (want_boundary && k == 4) boundary_faces(m, s);
    const unsigned Gv = grid_for(V, 256) > 8192 ? 8192 : grid_for(V, 256);
    k_check_isolated<<<Gv, 256, 0, s>>>(m->row_ptr.p, V, m->err.p);
    LMS_CHECK_LAUNCH();
    check_err_flag(m, s, "lms_build_csr");
    return;
  }
  DBuf<unsigned long long> keys(nk, s), sorted(nk, s);
  k_expand_pairs<<<Ge, 256, 0, s>>>(m->elems.p, n_el, k, b, keys.p);
  LMS_CHECK_LAUNCH();
  size_t tb = 0;
  LMS_TRY_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tb, keys.p, sorted.p, nk, 0, 2 * b, s));
  {
    DBuf<char> tmp(tb, s);
    LMS_TRY_CUDA(cub::DeviceRadixSort::SortKeys(tmp.p, tb, keys.p, sorted.p, nk, 0, 2 * b, s));
  }
  // run-length encode: unique keys (into `keys`) + multiplicities
  DBuf<int> cnt(nk, s), nruns(1, s);
  tb = 0;
  LMS_TRY_CUDA(cub::DeviceRunLengthEncode::Encode(nullptr, tb, sorted.p, keys.p, cnt.p, nruns.p, (int)nk, s));
  {
    DBuf<char> tmp(tb, s);
    LMS_TRY_CUDA(cub::DeviceRunLengthEncode::Encode(tmp.p, tb, sorted.p, keys.p, cnt.p, nruns.p, (int)nk, s));
  }
  int h_nnz = 0;
  LMS_TRY_CUDA(cudaMemcpyAsync(&h_nnz, nruns.p, sizeof(int), cudaMemcpyDeviceToHost, s));
  LMS_TRY_CUDA(cudaStreamSynchronize(s));
  sorted.release();
  m->nnz = h_nnz;
  m->col.alloc(m->nnz, s);
  m->row_ptr.alloc(V + 1, s);
  uint8_t* fx = nullptr;
  if (want_boundary) {
    LMS_TRY_CUDA(cudaMemsetAsync(m->fixed.p, 0, V, s));
    if (k == 3) fx = m->fixed.p;
  }
  const unsigned Gn = grid_for(m->nnz, 256) > 8192 ? 8192 : grid_for(m->nnz, 256);
  k_keys_to_csr<<<Gn, 256, 0, s>>>(keys.p, cnt.p, m->nnz, b, V, m->col.p, m->row_ptr.p, fx);
  LMS_CHECK_LAUNCH();
  keys.release();
  cnt.release();
  if (want_boundary && k == 4) boundary_faces(m, s);
  const unsigned Gv = grid_for(V, 256) > 8192 ? 8192 : grid_for(V, 256);
  k_check_isolated<<<Gv, 256, 0, s>>>(m->row_ptr.p, V, m->err.p);
  LMS_CHECK_LAUNCH();
  check_err_flag(m, s, "lms_build_csr");
}

// -------------------------------------------------------------- quality (A4)
__global__ void k_elem_quality(const int32_t* __restrict__ el, int64_t n_el, int k, int dim,
                               const double* __restrict__ x0, const double* __restrict__ x1,
                               const double* __restrict__ x2, double* __restrict__ qe, int* err) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n_el; e += (int64_t)gridDim.x * blockDim.x) {
    int32_t w[4];
    for (int s = 0; s < k; ++s) w[s] = el[e * k + s];
    double mn = 0.0, mx = 0.0;
    bool first = true;
    for (int s = 0; s < k; ++s)
      for (int t = s + 1; t < k; ++t) {
        double d = __dsub_rn(x0[w[s]], x0[w[t]]);
        double l2 = __dmul_rn(d, d);
        d = __dsub_rn(x1[w[s]], x1[w[t]]);
        l2 = __dadd_rn(l2, __dmul_rn(d, d));
        if (dim == 3) {
          d = __dsub_rn(x2[w[s]], x2[w[t]]);
          l2 = __dadd_rn(l2, __dmul_rn(d, d));
        }
        if (first) { mn = l2; mx = l2; first = false; }
        else { if (l2 < mn) mn = l2; if (l2 > mx) mx = l2; }
      }
    if (mx == 0.0) raise_err(err, LMS_E_DEGENERATE);
    qe[e] = __ddiv_rn(__dsqrt_rn(mn), __dsqrt_rn(mx));
  }
}

__global__ void k_incidence_keys(const int32_t* __restrict__ el, int64_t n_el, int k, int eb,
                                 unsigned long long* __restrict__ keys) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_el * k; i += (int64_t)gridDim.x * blockDim.x)
    keys[i] = ((unsigned long long)el[i] << eb) | (unsigned long long)(i / k);
}

// keys sorted by (v, e): thread per key i; vertex ranges found by neighbour comparison
__global__ void k_vertex_quality(const unsigned long long* __restrict__ keys, int64_t n, int eb,
                                 const double* __restrict__ qe, double* __restrict__ qv, int* err) {
  const unsigned long long emask = (1ull << eb) - 1;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    unsigned long long v = keys[i] >> eb;
    if (i > 0 && (keys[i - 1] >> eb) == v) continue;   // not the first of its run
    double acc = qe[keys[i] & emask];
    int64_t j = i + 1, c = 1;
    for (; j < n && (keys[j] >> eb) == v; ++j, ++c) acc = __dadd_rn(acc, qe[keys[j] & emask]);
    qv[v] = __ddiv_rn(acc, (double)c);
  }
}

__global__ void k_mark_untouched(const unsigned long long* __restrict__ keys, int64_t n, int eb, int64_t V,
                                 int* err) {
  // every vertex must be attached to an element: count distinct runs == V
  // (checked cheaply: first key's vertex is 0, last is V-1 and no gap between runs)
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    unsigned long long v = keys[i] >> eb;
    unsigned long long prev = (i == 0) ? ~0ull : (keys[i - 1] >> eb);
    if (i == 0 && v != 0) raise_err(err, LMS_E_ISOLATED);
    if (i > 0 && v > prev + 1) raise_err(err, LMS_E_ISOLATED);
    if (i == n - 1 && (int64_t)v != V - 1) raise_err(err, LMS_E_ISOLATED);
  }
}

void compute_quality(lms_mesh_s* m, double* out, cudaStream_t s) {
  if (!m->k) fail(LMS_E_STATE, "quality needs elements (or a quality given to lms_mesh_from_csr)");
  sync_soa(m, s);
  const int64_t n_el = m->n_el, V = m->V;
  const int k = m->k;
  DBuf<double> qe(n_el, s);
  const unsigned Ge = grid_for(n_el, 256) > 8192 ? 8192 : grid_for(n_el, 256);
  k_elem_quality<<<Ge, 256, 0, s>>>(m->elems.p, n_el, k, m->dim, m->x[0].p, m->x[1].p,
                                     m->dim == 3 ? m->x[2].p : nullptr, qe.p, m->err.p);
  LMS_CHECK_LAUNCH();
  check_err_flag(m, s, "quality");
  const int eb = bits_for(n_el);
  const int vb = bits_for(V);
  const int64_t n = n_el * k;
  DBuf<unsigned long long> keys(n, s), sorted(n, s);
  const unsigned Gn = grid_for(n, 256) > 8192 ? 8192 : grid_for(n, 256);
  k_incidence_keys<<<Gn, 256, 0, s>>>(m->elems.p, n_el, k, eb, keys.p);
  LMS_CHECK_LAUNCH();
  size_t tb = 0;
  LMS_TRY_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tb, keys.p, sorted.p, n, 0, eb + vb, s));
  {
    DBuf<char> tmp(tb, s);
    LMS_TRY_CUDA(cub::DeviceRadixSort::SortKeys(tmp.p, tb, keys.p, sorted.p, n, 0, eb + vb, s));
  }
  k_mark_untouched<<<Gn, 256, 0, s>>>(sorted.p, n, eb, V, m->err.p);
  LMS_CHECK_LAUNCH();
  k_vertex_quality<<<Gn, 256, 0, s>>>(sorted.p, n, eb, qe.p, out, m->err.p);
  LMS_CHECK_LAUNCH();
  check_err_flag(m, s, "quality");
}

const double* initial_quality(lms_mesh_s* m, cudaStream_t s) {
  if (m->has_quality) return m->quality.p;  // cached, or given to lms_mesh_from_csr (permuted with the mesh)
  if (m->coords_moved)
    fail(LMS_E_STATE, "RDR orders by the INITIAL vertex qualities (P:262-265, reading Z13), but the coordinates "
                      "changed since the build: call lms_order before lms_smooth / lms_import_coords");
  DBuf<double> q(m->V, s);
  compute_quality(m, q.p, s);
  m->quality = std::move(q);
  m->has_quality = true;
  return m->quality.p;
}

// -------------------------------------------------------------- per-row sort
void segmented_sort_rows(int32_t* d_col, const int32_t* d_row_ptr, int64_t V, int64_t nnz, cudaStream_t s) {
  if (nnz == 0) return;
  DBuf<int32_t> out(nnz, s);
  size_t tb = 0;
  LMS_TRY_CUDA(cub::DeviceSegmentedSort::SortKeys(nullptr, tb, d_col, out.p, nnz, V, d_row_ptr, d_row_ptr + 1, s));
  {
    DBuf<char> tmp(tb, s);
    LMS_TRY_CUDA(cub::DeviceSegmentedSort::SortKeys(tmp.p, tb, d_col, out.p, nnz, V, d_row_ptr, d_row_ptr + 1, s));
  }
  LMS_TRY_CUDA(cudaMemcpyAsync(d_col, out.p, nnz * sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
}

}  // namespace lms
