// reuse.cu -- the paper's reuse-distance instrument on the GPU (SURVEY 8(f)
// N2): PAPER.md Sec. 3.1, the first-iteration traces of Fig. 1 /
// Table III and the Eq. 2 miss model.
//
//  lms_trace: the canonical access trace of one SEQUENTIAL sweep in storage
//    order (Alg. 1's loop): per free vertex v: v, N(v) in CSR
//    order, v (the write).  Counts, one scan, one fill kernel.
//  lms_reuse_distance: for every access t to element x, the number of
//    DISTINCT elements accessed since x's previous access p, -1
//    for a first access.  Exactly:
//        d(t) = #{ j in (p, t) : prev(j) < p }
//    (an access j inside the window is the first of its element there iff
//    its previous access is before p).  prev() comes from one stable radix
//    sort of (element, time) pairs; the counts are 2D dominance queries,
//    answered for all t in parallel by a wavelet matrix over
//    A[j] = prev(j) + 1 (B = bits of n levels; each level a bitvector with a
//    per-word rank directory and a stable zeros-then-ones partition): a query
//    walks the B levels with two rank lookups each.  O(n log n) work, no
//    sequential scan.
//  lms_reuse_stats: Table III quantiles ("the smallest value such that there
//    at least a proportion X of the population below it"), the
//    mean, the cold count and the counts >= given capacities (the model's
//    misses per level) from one sort of the finite distances.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_reduce.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>

#include <algorithm>
#include <cmath>
#include <vector>

#include "lms_internal.cuh"

namespace lms {

static unsigned g8k(int64_t n) {
  const unsigned g = grid_for(n > 0 ? n : 1, 256);
  return g > 8192 ? 8192 : g;
}

__global__ void k_trace_count(const int32_t* __restrict__ rp, const uint8_t* __restrict__ fixed, int64_t V,
                              int64_t* __restrict__ cnt) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < V; v += (int64_t)gridDim.x * blockDim.x)
    cnt[v] = fixed[v] ? 0 : (int64_t)(rp[v + 1] - rp[v]) + 2;
}

__global__ void k_trace_fill(const int32_t* __restrict__ rp, const int32_t* __restrict__ col,
                             const uint8_t* __restrict__ fixed, const int64_t* __restrict__ off, int64_t V,
                             int32_t* __restrict__ tr) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < V; v += (int64_t)gridDim.x * blockDim.x) {
    if (fixed[v]) continue;
    int64_t o = off[v];
    tr[o++] = (int32_t)v;
    for (int32_t e = rp[v]; e < rp[v + 1]; ++e) tr[o++] = col[e];
    tr[o] = (int32_t)v;
  }
}

__global__ void k_iota64(int64_t* a, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    a[i] = i;
}

__global__ void k_check_ids(const int32_t* __restrict__ tr, int64_t n, int64_t n_ids, int* err) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    if (tr[i] < 0 || tr[i] >= n_ids) atomicCAS(err, 0, (int)LMS_E_INDEX);
}

// (element, time) sorted by element, times ascending within an element
__global__ void k_prev(const int32_t* __restrict__ key, const int64_t* __restrict__ t, int64_t n,
                       uint32_t* __restrict__ A) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x)
    A[t[k]] = (k > 0 && key[k - 1] == key[k]) ? (uint32_t)(t[k - 1] + 1) : 0u;  // prev + 1 (0 = cold)
}

// one wavelet level: bit b of every value into the level's bitvector words
// and their popcounts (one warp ballot per 32 values)
__global__ void k_wm_bits(const uint32_t* __restrict__ cur, int64_t n, int b, uint32_t* __restrict__ words,
                          uint32_t* __restrict__ pc) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = (n + 31) >> 5;
  for (int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; w < nw;
       w += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t i = (w << 5) + lane;
    const bool bit = i < n && ((cur[i] >> b) & 1u);
    const uint32_t word = __ballot_sync(0xffffffffu, bit);
    if (lane == 0) {
      words[w] = word;
      pc[w] = __popc(word);
    }
  }
}

__device__ __forceinline__ uint32_t wm_rank1(const uint32_t* __restrict__ words, const uint32_t* __restrict__ dir,
                                             int64_t pos) {
  const int64_t w = pos >> 5;
  const uint32_t r = (uint32_t)(pos & 31);
  return dir[w] + (r ? __popc(words[w] & ((1u << r) - 1u)) : 0u);
}

// stable partition of the level: zeros first (in order), then ones
__global__ void k_wm_part(const uint32_t* __restrict__ cur, int64_t n, const uint32_t* __restrict__ words,
                          const uint32_t* __restrict__ dir, uint32_t Z, uint32_t* __restrict__ nxt) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t r1 = wm_rank1(words, dir, i);
    const bool bit = (words[i >> 5] >> (i & 31)) & 1u;
    nxt[bit ? Z + r1 : (uint32_t)i - r1] = cur[i];
  }
}

struct WmLevel {
  const uint32_t* words;
  const uint32_t* dir;
  uint32_t Z;
};

// d(t) = #{ j in [p + 1, t) : A[j] <= p } with p = prev(t) (A = prev + 1)
__global__ void k_wm_query(const uint32_t* __restrict__ A, int64_t n, int B, const WmLevel* __restrict__ lev,
                           int64_t* __restrict__ dist) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t a = A[t];
    if (a == 0) {
      dist[t] = -1;
      continue;
    }
    const uint32_t p = a - 1;  // previous access time
    int64_t l = (int64_t)p + 1, r = t;
    int64_t res = 0;
    for (int k = 0; k < B; ++k) {
      const WmLevel L = lev[k];
      const int b = B - 1 - k;
      const int64_t r1l = wm_rank1(L.words, L.dir, l), r1r = wm_rank1(L.words, L.dir, r);
      if ((p >> b) & 1u) {
        res += (r - r1r) - (l - r1l);
        l = L.Z + r1l;
        r = L.Z + r1r;
      } else {
        l -= r1l;
        r -= r1r;
      }
    }
    dist[t] = res + (r - l);
  }
}

void reuse_distances(const int32_t* tr, int64_t n, int64_t n_ids, int64_t* dist, int* err, cudaStream_t s) {
  if (n == 0) return;
  if (n >= ((int64_t)1 << 31)) fail(LMS_E_ARG, "lms_reuse_distance: trace longer than 2^31 - 1");
  k_check_ids<<<g8k(n), 256, 0, s>>>(tr, n, n_ids, err);
  LMS_CHECK_LAUNCH();
  // prev(t) by a stable sort of (element, time)
  DBuf<uint32_t> A(n, s);
  {
    DBuf<int32_t> k2(n, s);
    DBuf<int64_t> t1(n, s), t2(n, s);
    k_iota64<<<g8k(n), 256, 0, s>>>(t1.p, n);
    LMS_CHECK_LAUNCH();
    int kb = 1;
    while (((int64_t)1 << kb) < n_ids) ++kb;
    size_t tb = 0;
    LMS_TRY_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, tr, k2.p, t1.p, t2.p, n, 0, kb, s));
    DBuf<char> tmp(tb, s);
    LMS_TRY_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tb, tr, k2.p, t1.p, t2.p, n, 0, kb, s));
    k_prev<<<g8k(n), 256, 0, s>>>(k2.p, t2.p, n, A.p);
    LMS_CHECK_LAUNCH();
  }
  // wavelet matrix over A (values <= n)
  int B = 1;
  while (((int64_t)1 << B) <= n) ++B;
  const int64_t nw = (n + 31) / 32;
  DBuf<uint32_t> words((size_t)B * nw, s), dirs((size_t)B * (nw + 1), s), pc(nw + 1, s);
  DBuf<uint32_t> cur(n, s), nxt(n, s);
  LMS_TRY_CUDA(cudaMemcpyAsync(cur.p, A.p, n * sizeof(uint32_t), cudaMemcpyDeviceToDevice, s));
  std::vector<WmLevel> h(B);
  size_t tbs = 0;
  LMS_TRY_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tbs, pc.p, dirs.p, nw + 1, s));
  DBuf<char> tmps(tbs, s);
  for (int k = 0; k < B; ++k) {
    uint32_t* wk = words.p + (size_t)k * nw;
    uint32_t* dk = dirs.p + (size_t)k * (nw + 1);
    k_wm_bits<<<g8k(nw * 32), 256, 0, s>>>(cur.p, n, B - 1 - k, wk, pc.p);
    LMS_CHECK_LAUNCH();
    LMS_TRY_CUDA(cudaMemsetAsync(pc.p + nw, 0, sizeof(uint32_t), s));
    LMS_TRY_CUDA(cub::DeviceScan::ExclusiveSum(tmps.p, tbs, pc.p, dk, nw + 1, s));
    uint32_t ones = 0;
    LMS_TRY_CUDA(cudaMemcpyAsync(&ones, dk + nw, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
    LMS_TRY_CUDA(cudaStreamSynchronize(s));
    h[k] = WmLevel{wk, dk, (uint32_t)(n - ones)};
    if (k + 1 < B) {
      k_wm_part<<<g8k(n), 256, 0, s>>>(cur.p, n, wk, dk, h[k].Z, nxt.p);
      LMS_CHECK_LAUNCH();
      std::swap(cur, nxt);
    }
  }
  DBuf<WmLevel> dlev(B, s);
  LMS_TRY_CUDA(cudaMemcpyAsync(dlev.p, h.data(), B * sizeof(WmLevel), cudaMemcpyHostToDevice, s));
  k_wm_query<<<g8k(n), 256, 0, s>>>(A.p, n, B, dlev.p, dist);
  LMS_CHECK_LAUNCH();
  LMS_TRY_CUDA(cudaStreamSynchronize(s));  // h (host) and dlev must outlive the kernel's reads of them
}

// finite distances compacted (order irrelevant: they are sorted next) and
// summed; warp-aggregated atomics
__global__ void k_finite(const int64_t* __restrict__ d, int64_t n, int64_t* __restrict__ out, int* nf,
                         unsigned long long* sum) {
  const int lane = threadIdx.x & 31;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i0 = blockIdx.x * (int64_t)blockDim.x; i0 < n; i0 += stride) {
    const int64_t i = i0 + threadIdx.x;
    const int64_t v = i < n ? d[i] : -1;
    const unsigned bal = __ballot_sync(0xffffffffu, v >= 0);
    unsigned long long x = v >= 0 ? (unsigned long long)v : 0ull;
    for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    int base = 0;
    if (lane == 0 && bal) {
      base = atomicAdd(nf, __popc(bal));
      atomicAdd(sum, x);
    }
    base = __shfl_sync(0xffffffffu, base, 0);
    if (v >= 0) out[base + __popc(bal & ((1u << lane) - 1u))] = v;
  }
}

}  // namespace lms

using namespace lms;

extern "C" {

lms_status lms_trace(lms_mesh_t m, int32_t* d_trace, int64_t* n_out, lms_stream_t stream) {
  try {
    if (!m || !n_out) fail(LMS_E_ARG, "NULL argument");
    DevGuard dg(m);
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t V = m->V;
    DBuf<int64_t> cnt(V + 1, s), off(V + 1, s);
    k_trace_count<<<g8k(V), 256, 0, s>>>(m->row_ptr.p, m->fixed.p, V, cnt.p);
    LMS_CHECK_LAUNCH();
    LMS_TRY_CUDA(cudaMemsetAsync(cnt.p + V, 0, sizeof(int64_t), s));
    size_t tb = 0;
    LMS_TRY_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt.p, off.p, V + 1, s));
    {
      DBuf<char> tmp(tb, s);
      LMS_TRY_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tb, cnt.p, off.p, V + 1, s));
    }
    int64_t n = 0;
    LMS_TRY_CUDA(cudaMemcpyAsync(&n, off.p + V, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    LMS_TRY_CUDA(cudaStreamSynchronize(s));
    *n_out = n;
    if (d_trace && n) {
      k_trace_fill<<<g8k(V), 256, 0, s>>>(m->row_ptr.p, m->col.p, m->fixed.p, off.p, V, d_trace);
      LMS_CHECK_LAUNCH();
    }
    return LMS_OK;
  } catch (const Err& e) {
    set_error(e.msg);
    return e.st;
  }
}

lms_status lms_reuse_distance(const int32_t* d_trace, int64_t n, int64_t n_ids, int64_t* d_dist,
                              lms_stream_t stream) {
  try {
    if (n < 0 || n_ids < 1 || (n > 0 && (!d_trace || !d_dist))) fail(LMS_E_ARG, "bad argument");
    cudaStream_t s = (cudaStream_t)stream;
    DBuf<int> err(1, s);
    LMS_TRY_CUDA(cudaMemsetAsync(err.p, 0, sizeof(int), s));
    reuse_distances(d_trace, n, n_ids, d_dist, err.p, s);
    int h = 0;
    LMS_TRY_CUDA(cudaMemcpyAsync(&h, err.p, sizeof(int), cudaMemcpyDeviceToHost, s));
    LMS_TRY_CUDA(cudaStreamSynchronize(s));
    if (h) fail((lms_status)h, "lms_reuse_distance: an identifier is outside [0, n_ids)");
    return LMS_OK;
  } catch (const Err& e) {
    set_error(e.msg);
    return e.st;
  }
}

lms_status lms_reuse_stats(const int64_t* d_dist, int64_t n, const double* h_q, int32_t nq, int64_t* h_quantile,
                           double* h_mean, int64_t* h_n_cold, const int64_t* h_capacity, int32_t ncap,
                           int64_t* h_n_ge, lms_stream_t stream) {
  try {
    if (n < 0 || nq < 0 || ncap < 0 || (n > 0 && !d_dist) || (nq && (!h_q || !h_quantile)) ||
        (ncap && (!h_capacity || !h_n_ge)))
      fail(LMS_E_ARG, "bad argument");
    cudaStream_t s = (cudaStream_t)stream;
    DBuf<int64_t> fin(std::max<int64_t>(n, 1), s), srt(std::max<int64_t>(n, 1), s);
    DBuf<int> nf(1, s);
    DBuf<unsigned long long> sum(1, s);
    LMS_TRY_CUDA(cudaMemsetAsync(nf.p, 0, sizeof(int), s));
    LMS_TRY_CUDA(cudaMemsetAsync(sum.p, 0, sizeof(unsigned long long), s));
    if (n) {
      k_finite<<<g8k(n), 256, 0, s>>>(d_dist, n, fin.p, nf.p, sum.p);
      LMS_CHECK_LAUNCH();
    }
    int hnf = 0;
    unsigned long long hs = 0;
    LMS_TRY_CUDA(cudaMemcpyAsync(&hnf, nf.p, sizeof(int), cudaMemcpyDeviceToHost, s));
    LMS_TRY_CUDA(cudaMemcpyAsync(&hs, sum.p, sizeof(hs), cudaMemcpyDeviceToHost, s));
    LMS_TRY_CUDA(cudaStreamSynchronize(s));
    if (h_n_cold) *h_n_cold = n - hnf;
    if (h_mean) *h_mean = hnf ? (double)hs / (double)hnf : NAN;
    if (hnf == 0) {
      if (nq || ncap) fail(LMS_E_STATE, "lms_reuse_stats: no finite distance");
      return LMS_OK;
    }
    size_t tb = 0;
    LMS_TRY_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tb, fin.p, srt.p, hnf, 0, 63, s));
    DBuf<char> tmp(tb, s);
    LMS_TRY_CUDA(cub::DeviceRadixSort::SortKeys(tmp.p, tb, fin.p, srt.p, hnf, 0, 63, s));
    std::vector<int64_t> hsrt;
    // quantile X: the smallest v with |{d <= v}| >= ceil(X * n_finite)
    for (int k = 0; k < nq; ++k) {
      if (!(h_q[k] > 0.0 && h_q[k] <= 1.0)) fail(LMS_E_ARG, "quantiles must be in (0, 1]");
      int64_t need = (int64_t)std::ceil(h_q[k] * (double)hnf - 1e-12);
      if (need < 1) need = 1;
      LMS_TRY_CUDA(cudaMemcpyAsync(h_quantile + k, srt.p + need - 1, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    }
    if (ncap) {
      hsrt.resize(hnf);
      LMS_TRY_CUDA(cudaMemcpyAsync(hsrt.data(), srt.p, hnf * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    }
    LMS_TRY_CUDA(cudaStreamSynchronize(s));
    for (int k = 0; k < ncap; ++k)  // reuse-based misses: distance >= capacity
      h_n_ge[k] = (int64_t)(hsrt.end() - std::lower_bound(hsrt.begin(), hsrt.end(), h_capacity[k]));
    return LMS_OK;
  } catch (const Err& e) {
    set_error(e.msg);
    return e.st;
  }
}

}  // extern "C"
