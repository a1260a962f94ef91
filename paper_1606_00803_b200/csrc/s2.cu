// s2.cu -- the S2 colour-pass sweep for 3D meshes (LMS_SCHED_S2; SURVEY
// 8(a) A9 "S2").
//
// Method: Eq. 1 under the colour-ordered Gauss-Seidel
// schedule (reading Z1): per sweep, for c = 0..C-1, every free
// colour-c vertex moves to (sum of its neighbours in CSR order) / deg, IEEE
// binary64, no FMA.  Bit-identical to S1 / S3 / GZ.
//
// Why a separate 3D kernel: in 3D (Kuhn, degree 14, 8 colours) the ghost zone
// of GZ is 8 hops deep and does not fit in shared memory, so the sweep is one
// pass per colour whose neighbour gathers come from L2.  The S1 kernel gathers
// SoA coordinates: three 8-byte loads per neighbour, three 32-byte L2 sectors.
// S2 keeps the coordinates interleaved as (x, y, z, 0) -- one 32-byte sector
// per vertex, read by ONE 256-bit load (LDG.E.ENL2.256) -- so a neighbour
// costs one sector, and the colour's CSR slice is streamed from the slab
// layout (per 32-vertex chunk: 32 vertex ids, then the rows column-major, -1
// padded: every row position is one coalesced 128-byte warp load).  The slab
// is read with an L2 evict_first policy, the coordinates with evict_last, so
// the 67 MB coordinate array of C3 stays in the 126 MB L2 across the passes.
// Each colour pass is one launch; a sweep's C launches are captured in a CUDA
// graph.  The interleaved copy is made at the start of an lms_smooth call and
// written back to the SoA arrays at its end.
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "lms_internal.cuh"

namespace lms {

__device__ __forceinline__ uint64_t s2_policy_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t s2_policy_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ int32_t s2_ld_stream(const int32_t* p, uint64_t pol) {
  int32_t v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
  return v;
}
// one 32-byte sector: (x, y, z, pad) of a vertex.  Not .nc: the colour pass
// writes other vertices of the same array (never one it reads: same-colour
// vertices are not adjacent), so the plain coherent path is used.
__device__ __forceinline__ double4 s2_ld4(const double4* p, uint64_t pol) {
  double4 v;
  asm volatile("ld.global.L2::cache_hint.v4.f64 {%0, %1, %2, %3}, [%4], %5;"
               : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w)
               : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ void s2_st4(double4* p, double4 v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v4.f64 [%0], {%1, %2, %3, %4}, %5;" ::"l"(p), "d"(v.x), "d"(v.y), "d"(v.z),
               "d"(v.w), "l"(pol)
               : "memory");
}

// one colour pass: a warp per 32-vertex chunk of the colour's items; chunk w
// of colour c is slab + choff[w] with row width chw[w]
template <int WMAX>
__global__ void __launch_bounds__(256, 3) k_sweep_s2(const long long* __restrict__ choff,
                                                     const int32_t* __restrict__ chw, int64_t w0, int64_t w1,
                                                     const int32_t* __restrict__ slab, double4* X) {
  const uint64_t pf = s2_policy_first(), pl = s2_policy_last();
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t w = w0 + (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5); w < w1; w += nwarps) {
    const int W = chw[w];
    const int32_t* ch = slab + choff[w];
    const int32_t v = s2_ld_stream(ch + lane, pf);
    if (v < 0) continue;
    double sx = 0.0, sy = 0.0, sz = 0.0;
    int d = 0;
    if (W <= WMAX) {
      // two batches of WMAX / 2 gathers in flight (register budget: 3 CTAs per SM)
      constexpr int H = WMAX / 2;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        int32_t u[H];
#pragma unroll
        for (int q = 0; q < H; ++q) u[q] = h * H + q < W ? s2_ld_stream(ch + 32 * (1 + h * H + q) + lane, pf) : -1;
        double4 g[H];
#pragma unroll
        for (int q = 0; q < H; ++q)
          if (u[q] >= 0) g[q] = s2_ld4(X + u[q], pl);
#pragma unroll
        for (int q = 0; q < H; ++q)
          if (u[q] >= 0) {
            if (d == 0) {
              sx = g[q].x;
              sy = g[q].y;
              sz = g[q].z;
            } else {
              sx = __dadd_rn(sx, g[q].x);
              sy = __dadd_rn(sy, g[q].y);
              sz = __dadd_rn(sz, g[q].z);
            }
            ++d;
          }
      }
    } else {  // long rows: ordered, one neighbour at a time
      for (int q = 0; q < W; ++q) {
        const int32_t uu = s2_ld_stream(ch + 32 * (1 + q) + lane, pf);
        if (uu < 0) break;
        const double4 e = s2_ld4(X + uu, pl);
        if (d == 0) {
          sx = e.x;
          sy = e.y;
          sz = e.z;
        } else {
          sx = __dadd_rn(sx, e.x);
          sy = __dadd_rn(sy, e.y);
          sz = __dadd_rn(sz, e.z);
        }
        ++d;
      }
    }
    const double dd = (double)d;
    s2_st4(X + v, make_double4(__ddiv_rn(sx, dd), __ddiv_rn(sy, dd), __ddiv_rn(sz, dd), 0.0), pl);
  }
}

// chunk lists, colour-major: item (k, c) contributes its chunks at
// cnt-prefix position c * K + k
__global__ void k_s2_count(const int32_t* __restrict__ item_ptr, int64_t K, int C, int32_t* __restrict__ cnt) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < K * C; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = i / K, k = i - c * K;
    const int64_t it = k * C + c;
    cnt[i] = (item_ptr[it + 1] - item_ptr[it] + 31) >> 5;
  }
}
__global__ void k_s2_fill(const int32_t* __restrict__ item_ptr, const long long* __restrict__ ioff,
                          const int32_t* __restrict__ iw, int64_t K, int C, const int32_t* __restrict__ off,
                          long long* __restrict__ choff, int32_t* __restrict__ chw) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < K * C; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = i / K, k = i - c * K;
    const int64_t it = k * C + c;
    const int32_t nch = (item_ptr[it + 1] - item_ptr[it] + 31) >> 5, W = iw[it];
    for (int32_t j = 0; j < nch; ++j) {
      choff[off[i] + j] = ioff[it] + (long long)j * 32 * (1 + W);
      chw[off[i] + j] = W;
    }
  }
}

__global__ void k_soa_to_aos4(const double* __restrict__ x, const double* __restrict__ y,
                              const double* __restrict__ z, int64_t V, double4* __restrict__ a) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < V; v += (int64_t)gridDim.x * blockDim.x)
    a[v] = make_double4(x[v], y[v], z[v], 0.0);
}
__global__ void k_aos4_to_soa(const double4* __restrict__ a, int64_t V, double* __restrict__ x, double* __restrict__ y,
                              double* __restrict__ z) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < V; v += (int64_t)gridDim.x * blockDim.x) {
    const double4 p = a[v];
    x[v] = p.x;
    y[v] = p.y;
    z[v] = p.z;
  }
}

static int s2_blocks(lms_mesh_s* m) {
  int nsm = 148;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, m->device);
  return nsm * 8;  // 8 CTAs of 256 threads per SM: warps stride the colour's chunks
}

void run_s2(lms_mesh_s* m, int sweeps, cudaStream_t s) {
  if (m->dim != 3) fail(LMS_E_ARG, "the S2 schedule is the 3D kernel (2D meshes use GZ)");
  Schedule& S = m->sched;
  const int64_t V = m->V, K = S.K;
  const int C = m->C;
  // chunk lists of every colour (built once per schedule)
  if (!S.s2_choff.p) {
    DBuf<int32_t> cnt(K * C + 1, s), off(K * C + 1, s);
    const unsigned Gi = grid_for(K * C, 256) > 4096 ? 4096 : grid_for(K * C, 256);
    k_s2_count<<<Gi, 256, 0, s>>>(S.item_ptr.p, K, C, cnt.p);
    LMS_CHECK_LAUNCH();
    LMS_TRY_CUDA(cudaMemsetAsync(cnt.p + K * C, 0, sizeof(int32_t), s));
    size_t tb = 0;
    LMS_TRY_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt.p, off.p, K * C + 1, s));
    {
      DBuf<char> tmp(tb, s);
      LMS_TRY_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tb, cnt.p, off.p, K * C + 1, s));
    }
    std::vector<int32_t> h(K * C + 1);
    LMS_TRY_CUDA(cudaMemcpyAsync(h.data(), off.p, (K * C + 1) * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    LMS_TRY_CUDA(cudaStreamSynchronize(s));
    S.s2_cstart.assign(C + 1, 0);
    for (int c = 0; c <= C; ++c) S.s2_cstart[c] = h[(size_t)c * K];
    const int64_t nch = h[K * C];
    S.s2_choff.alloc(nch > 0 ? nch : 1, s);
    S.s2_chw.alloc(nch > 0 ? nch : 1, s);
    k_s2_fill<<<Gi, 256, 0, s>>>(S.item_ptr.p, S.ioff.p, S.iw.p, K, C, off.p, S.s2_choff.p, S.s2_chw.p);
    LMS_CHECK_LAUNCH();
  }
  sync_soa(m, s);
  soa_changed(m);
  DBuf<double> buf(4 * V, s);
  double4* X = reinterpret_cast<double4*>(buf.p);
  const unsigned G = grid_for(V, 256) > 8192 ? 8192 : grid_for(V, 256);
  k_soa_to_aos4<<<G, 256, 0, s>>>(m->x[0].p, m->x[1].p, m->x[2].p, V, X);
  LMS_CHECK_LAUNCH();
  int nsm = 148;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, m->device);
  // the interleaved coordinates as an L2 persisting window for the passes
  // (the slab streams through with evict_first): set aside up to the
  // device's persisting maximum while S2 runs (LMS_S2_PERSIST=0 disables)
  int maxp = 0;
  cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, m->device);
  const char* pe = getenv("LMS_S2_PERSIST");
  const bool persist = maxp > 0 && !(pe && !strcmp(pe, "0"));
  size_t prev_limit = 0;
  cudaLaunchAttribute attr[1];
  if (persist) {
    LMS_TRY_CUDA(cudaDeviceGetLimit(&prev_limit, cudaLimitPersistingL2CacheSize));
    const size_t want = std::min<size_t>((size_t)maxp, (size_t)(32 * V));
    LMS_TRY_CUDA(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, want));
    attr[0].id = cudaLaunchAttributeAccessPolicyWindow;
    attr[0].val.accessPolicyWindow.base_ptr = X;
    attr[0].val.accessPolicyWindow.num_bytes = std::min<size_t>((size_t)(32 * V), (size_t)maxp);
    attr[0].val.accessPolicyWindow.hitRatio = 1.0f;
    attr[0].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    attr[0].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
  }
  auto pass = [&](int c, cudaStream_t st) {
    const int64_t w0 = S.s2_cstart[c], w1 = S.s2_cstart[c + 1];
    const int64_t nw = w1 - w0;
    if (nw <= 0) return;
    const int64_t blocks = std::min<int64_t>((nw + 7) / 8, (int64_t)nsm * 3 * 4);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)blocks);
    cfg.blockDim = dim3(256);
    cfg.stream = st;
    cfg.attrs = persist ? attr : nullptr;
    cfg.numAttrs = persist ? 1 : 0;
    LMS_TRY_CUDA(cudaLaunchKernelEx(&cfg, k_sweep_s2<16>, (const long long*)S.s2_choff.p, (const int32_t*)S.s2_chw.p,
                                    w0, w1, (const int32_t*)S.slab.p, X));
  };
  // one sweep = C launches, captured once per call into a graph
  cudaGraphExec_t exec = nullptr;
  if (sweeps > 1) {
    cudaStream_t cs = nullptr;
    LMS_TRY_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    cudaGraph_t g = nullptr;
    LMS_TRY_CUDA(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
    for (int c = 0; c < C; ++c) pass(c, cs);
    LMS_TRY_CUDA(cudaStreamEndCapture(cs, &g));
    LMS_TRY_CUDA(cudaGraphInstantiate(&exec, g, 0));
    cudaGraphDestroy(g);
    cudaStreamDestroy(cs);
  }
  for (int i = 0; i < sweeps; ++i) {
    if (exec) {
      LMS_TRY_CUDA(cudaGraphLaunch(exec, s));
      note_launch(C);
    } else {
      for (int c = 0; c < C; ++c) {
        pass(c, s);
        LMS_CHECK_LAUNCH();
      }
    }
  }
  if (exec) cudaGraphExecDestroy(exec);
  k_aos4_to_soa<<<G, 256, 0, s>>>(X, V, m->x[0].p, m->x[1].p, m->x[2].p);
  LMS_CHECK_LAUNCH();
  if (persist) {  // hand the set-aside back (persisting lines return to normal)
    LMS_TRY_CUDA(cudaStreamSynchronize(s));
    LMS_TRY_CUDA(cudaCtxResetPersistingL2Cache());
    LMS_TRY_CUDA(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, prev_limit));
  }
}

}  // namespace lms
