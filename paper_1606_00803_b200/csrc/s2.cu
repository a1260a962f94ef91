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
#include <cooperative_groups.h>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <cstdio>
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

// One 32-vertex chunk of the persistent kernel: the vertex ids and every row
// position are loaded in one round (independent loads), then the neighbours
// are gathered in two halves of WMAX / 2 sectors and summed in CSR order.
__device__ __forceinline__ double4 s2_ld4_plain(const double4* p) {
  double4 v;
  asm volatile("ld.global.v4.f64 {%0, %1, %2, %3}, [%4];" : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w) : "l"(p));
  return v;
}
template <int WMAX, bool HINT>
__device__ __forceinline__ void s2_chunk(const int32_t* ch, int W, double4* X, int lane, uint64_t pf, uint64_t pl) {
  if (W <= WMAX) {
    const int32_t v = s2_ld_stream(ch + lane, pf);
    int32_t u[WMAX];
#pragma unroll
    for (int q = 0; q < WMAX; ++q) u[q] = q < W ? s2_ld_stream(ch + 32 * (1 + q) + lane, pf) : -1;
    if (v < 0) return;
    double sx = 0.0, sy = 0.0, sz = 0.0;
    int d = 0;
    constexpr int H = WMAX / 2;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      double4 g[H];
#pragma unroll
      for (int q = 0; q < H; ++q)
        if (u[h * H + q] >= 0) g[q] = HINT ? s2_ld4(X + u[h * H + q], pl) : s2_ld4_plain(X + u[h * H + q]);
#pragma unroll
      for (int q = 0; q < H; ++q)
        if (u[h * H + q] >= 0) {
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
    const double dd = (double)d;
    s2_st4(X + v, make_double4(__ddiv_rn(sx, dd), __ddiv_rn(sy, dd), __ddiv_rn(sz, dd), 0.0), pl);
    return;
  }
  const int32_t v = s2_ld_stream(ch + lane, pf);  // long rows: ordered, one neighbour at a time
  if (v < 0) return;
  double sx = 0.0, sy = 0.0, sz = 0.0;
  int d = 0;
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
  const double dd = (double)d;
  s2_st4(X + v, make_double4(__ddiv_rn(sx, dd), __ddiv_rn(sy, dd), __ddiv_rn(sz, dd), 0.0), pl);
}

__device__ __forceinline__ unsigned long long s2_gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void s2_prefetch_l2(const void* p, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// The persistent S2 sweep: ONE cooperative launch for all sweeps x colours.
//
// Ownership.  CTA b owns a run of consecutive spatial tiles (boxes) holding
// an equal share of the chunks, so its chunks of colour c are one contiguous
// range crange[c (G+1) + b ..+1] of the colour-major chunk list and the
// neighbourhoods of its warps' chunks overlap: the SM's L1 serves the repeats
// (C3: 46 % L1 hits, against 15 % for storage tiles on strided warps).
//
// Slab ring.  One producer warp copies the CTA's chunks (32 vertex ids + W
// rows of 32 neighbour ids, 128 (1 + W) bytes each) into a ring of R shared-
// memory slots by TMA bulk copies (mbarrier full/empty per slot), in the
// CTA's chunk order across passes: the slab does not depend on the
// coordinates, so the producer runs ahead through the pass boundaries and a
// pass starts with its first chunks already staged.  (Loaded by the consumer
// warps themselves, one chunk ahead, the slab's DRAM latency was the pass
// time: 16.5 us per pass with the gathers switched off.)
//
// Passes are ordered per neighbourhood, not by a grid barrier: CTA b starts
// pass p once every CTA owning a tile adjacent to one of its tiles has
// published pass p - 1 (prog[], release/acquire at gpu scope).  That covers
// both hazards of the colour schedule: pass p writes colour-(p mod C)
// vertices that the neighbours read in pass p - 1, and reads vertices they
// wrote in passes < p.  A slow CTA delays only its neighbourhood (a grid
// barrier measured 14.8 us of wait per 13.6 us pass).  The acquiring
// thread's gpu-scope fence invalidates the SM's L1 (CCTL.IVALL), whose
// copies of the neighbours' vertices are stale after their pass.
constexpr unsigned long long S2P_WAIT_NS = 20ull * 1000 * 1000 * 1000;

__device__ __forceinline__ unsigned s2_ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void s2_st_release(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t s2_smem(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void s2_mbar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(s2_smem(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void s2_mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s2_smem(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void s2_mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(s2_smem(b)) : "memory");
}
// false when the wait outlived S2P_WAIT_NS or another waiter aborted
__device__ __forceinline__ bool s2_mbar_wait(uint64_t* b, uint32_t parity, volatile int* sab) {
  const uint32_t a = s2_smem(b);
  unsigned long long t0 = 0;
  for (unsigned n = 1;; ++n) {
    uint32_t done;
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(done)
                 : "r"(a), "r"(parity)
                 : "memory");
    if (done) return true;
    if ((n & 255) == 0) {
      if (*sab) return false;
      const unsigned long long t = s2_gtimer();
      if (t0 == 0) t0 = t;
      else if (t - t0 > S2P_WAIT_NS) return false;
    }
  }
}
__device__ __forceinline__ void s2_bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* b, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          s2_smem(dst)),
      "l"(src), "r"(bytes), "r"(s2_smem(b)), "l"(pol)
      : "memory");
}
// rows longer than the staged width: the slab read directly, one neighbour
// at a time.  (Kept inline: compiled out of line (__noinline__) it gave wrong
// results under the 24-warp / 72-register variant on the hub mesh of
// tests/test_gpu_parity.py::test_s2_long_row; inline, both variants are
// bit-exact and neither spills.)
__device__ __forceinline__ void s2_chunk_long(const int32_t* ch, int W, double4* X, int lane, uint64_t pf, uint64_t pl) {
  s2_chunk<2, true>(ch, W, X, lane, pf, pl);
}
__device__ __forceinline__ void s2_cons_sync(int ncons) {
  asm volatile("bar.sync 1, %0;" ::"r"(ncons * 32) : "memory");
}

template <int WMAX, bool HINT>
__device__ __forceinline__ double4 s2_gather(const double4* p, uint64_t pl) {
  return HINT ? s2_ld4(p, pl) : s2_ld4_plain(p);
}

// one staged chunk: ids from the slot, gathers in NB batches, CSR-order sums.
// The row positions q < W (W uniform over the chunk) are gathered without
// per-lane predication: a -1 entry (a row shorter than W) reads the pad
// vertex X[padv] = (-0, -0, -0), the identity of IEEE addition, and is not
// counted in the degree.
template <int WMAX, int NB>
__device__ __forceinline__ void s2r_chunk(const int32_t (&u)[WMAX], int W, int32_t v, double4* X, int32_t padv,
                                          uint64_t pl) {
  constexpr int H = WMAX / NB;
  double sx = 0.0, sy = 0.0, sz = 0.0;
  int d = 0;
#pragma unroll
  for (int h = 0; h < NB; ++h) {
    double4 g[H];
#pragma unroll
    for (int q = 0; q < H; ++q)
      if (h * H + q < W) {
        const int32_t x = u[h * H + q];
        g[q] = s2_ld4(X + (x >= 0 ? x : padv), pl);
        d += x >= 0 ? 1 : 0;
      }
#pragma unroll
    for (int q = 0; q < H; ++q)
      if (h * H + q < W) {
        if (h * H + q == 0) {
          sx = g[q].x;
          sy = g[q].y;
          sz = g[q].z;
        } else {
          sx = __dadd_rn(sx, g[q].x);
          sy = __dadd_rn(sy, g[q].y);
          sz = __dadd_rn(sz, g[q].z);
        }
      }
  }
  if (v >= 0) {
    const double dd = (double)d;
    s2_st4(X + v, make_double4(__ddiv_rn(sx, dd), __ddiv_rn(sy, dd), __ddiv_rn(sz, dd), 0.0), pl);
  }
}

template <int WMAX, int NCONS, int NB>
__global__ void __launch_bounds__((NCONS + 1) * 32, 1)
    k_sweep_s2p(const long long* __restrict__ choff, const int32_t* __restrict__ chw,
                const int32_t* __restrict__ crange, int G, int C, long long npass, const int32_t* __restrict__ slab,
                double4* X, int opts, unsigned long long* stats, const int32_t* __restrict__ nb_ptr,
                const int32_t* __restrict__ nb, unsigned* prog, int* err, int R, int slot_ints, int32_t padv) {
  extern __shared__ __align__(128) unsigned char s2_sm[];
  int32_t* ring = reinterpret_cast<int32_t*>(s2_sm);
  uint64_t* full = reinterpret_cast<uint64_t*>(s2_sm + (size_t)R * slot_ints * 4);
  uint64_t* empty = full + R;
  long long* s_off = reinterpret_cast<long long*>(empty + R);
  int32_t* s_w = reinterpret_cast<int32_t*>(s_off + R);
  __shared__ int s_abort;
  __shared__ int s_fold[NCONS * 32];
  __shared__ int s_claim;
  const uint64_t pf = s2_policy_first(), pl = s2_policy_last();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int b = blockIdx.x;
  if (threadIdx.x == 0) {
    s_abort = 0;
    for (int i = 0; i < R; ++i) {
      s2_mbar_init(full + i, 1);
      s2_mbar_init(empty + i, 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  volatile int* sab = &s_abort;
  if (warp == NCONS) {  // ---------------- producer: the CTA's chunks, every pass, in order
    // lane l stages chunk seq0 + l of each group of 32 (descriptor loads and
    // copies of a group issue together; each lane waits for its own slot)
    long long seq0 = 0;
    for (long long it = 0; it < npass; ++it) {
      const int c = (int)(it % C);
      const int j0 = crange[c * (G + 1) + b], j1 = crange[c * (G + 1) + b + 1];
      for (int jb = j0; jb < j1; jb += 32, seq0 += 32) {
        const int j = jb + lane;
        if (j < j1) {
          const long long seq = seq0 + lane;
          const int W = chw[j];
          const long long off = choff[j];
          const int slot = (int)(seq % R);
          const long long round = seq / R;
          const unsigned long long tp0 = stats ? s2_gtimer() : 0;
          if (round > 0 && !s2_mbar_wait(empty + slot, (uint32_t)((round - 1) & 1), sab)) {
            raise_err(err, LMS_E_CUDA);
            *sab = 1;
            return;
          }
          if (stats && lane == 0) atomicAdd(stats + 4 * b + 3, s2_gtimer() - tp0);
          s_w[slot] = W;
          s_off[slot] = off;
          if (W <= WMAX) {
            const uint32_t bytes = 128u * (1u + (uint32_t)W);
            s2_mbar_expect_tx(full + slot, bytes);
            s2_bulk_g2s(ring + (size_t)slot * slot_ints, slab + off, bytes, full + slot, pf);
          } else {
            s2_mbar_arrive(full + slot);  // long rows: the consumer reads the slab itself
          }
        }
        __syncwarp();
      }
      seq0 -= (32 - (j1 - j0) % 32) % 32;  // the group tail: seq counts chunks, not lanes
    }
    return;
  }
  // ---------------- consumers
  long long base = 0;
  for (long long it = 0; it < npass; ++it) {
    const int c = (int)(it % C);
    const int j0 = crange[c * (G + 1) + b], j1 = crange[c * (G + 1) + b + 1];
    const int n = j1 - j0;
    unsigned long long tw = 0, t0 = 0;
    if (stats && threadIdx.x == 0) tw = s2_gtimer();
    if (it > 0 && warp == 0 && !(opts & 32)) {  // neighbours' pass it - 1
      const int a = nb_ptr[b], e = nb_ptr[b + 1];
      for (int k = a + lane; k < e; k += 32) {
        const unsigned* pp = prog + nb[k];
        unsigned long long tt0 = 0;
        unsigned cnt = 0;
        while (s2_ld_acquire(pp) < (unsigned)it) {
          if ((++cnt & 63) == 0) {
            const unsigned long long t = s2_gtimer();
            if (tt0 == 0) tt0 = t;
            else if (t - tt0 > S2P_WAIT_NS || *(volatile int*)err || *sab) {
              raise_err(err, LMS_E_CUDA);
              *sab = 1;
              break;
            }
          }
          __nanosleep(32);
        }
      }
      __syncwarp();
      if (lane == 0) __threadfence();  // L1 invalidate (CCTL.IVALL) after the acquires
    }
    if (threadIdx.x == 0) s_claim = 0;
    s2_cons_sync(NCONS);
    if (*sab) return;
    if (stats && threadIdx.x == 0) t0 = s2_gtimer();
    for (;;) {  // chunks claimed in order (a warp done early takes the next)
      int k = 0;
      if (lane == 0) k = atomicAdd(&s_claim, 1);
      k = __shfl_sync(0xffffffffu, k, 0);
      if (k >= n) break;
      const long long seq = base + k;
      const int slot = (int)(seq % R);
      if (!s2_mbar_wait(full + slot, (uint32_t)((seq / R) & 1), sab)) {
        if (lane == 0) {
          raise_err(err, LMS_E_CUDA);
          *sab = 1;
        }
        break;
      }
      const int W = s_w[slot];
      if (opts & 16) {
        __syncwarp();
        if (lane == 0) s2_mbar_arrive(empty + slot);
        continue;
      }
      if (W <= WMAX) {
        const int32_t* sl = ring + (size_t)slot * slot_ints;
        const int32_t v = sl[lane];
        int32_t u[WMAX];
#pragma unroll
        for (int q = 0; q < WMAX; ++q) u[q] = q < W ? sl[32 * (1 + q) + lane] : -1;
        // the slot's shared-memory reads must have returned before the
        // release lets the producer's TMA (async proxy) overwrite it: every
        // lane folds its reads into one store (it cannot issue before they
        // complete), and __syncwarp orders the stores before lane 0's arrive
        int f = v;
#pragma unroll
        for (int q = 0; q < WMAX; ++q) f ^= u[q];
        reinterpret_cast<volatile int*>(s_fold)[warp * 32 + lane] = f;
        __syncwarp();
        if (lane == 0) s2_mbar_arrive(empty + slot);
        s2r_chunk<WMAX, NB>(u, W, v, X, padv, pl);
      } else {
        // the descriptor read must have returned before the release lets the
        // producer overwrite it: every lane stores the value it read first
        const long long off = s_off[slot];
        reinterpret_cast<volatile int*>(s_fold)[warp * 32 + lane] = (int)off;
        __syncwarp();
        if (lane == 0) s2_mbar_arrive(empty + slot);
        s2_chunk_long(slab + off, W, X, lane, pf, pl);
      }
    }
    base += n;
    s2_cons_sync(NCONS);
    if (*sab) return;
    if (threadIdx.x == 0) {
      const unsigned long long t1 = stats ? s2_gtimer() : 0;
      __threadfence();
      s2_st_release(prog + b, (unsigned)(it + 1));
      if (stats) {
        atomicAdd(stats + 4 * b, t1 - t0);
        atomicAdd(stats + 4 * b + 1, t0 - tw);
        atomicAdd(stats + 4 * b + 2, (unsigned long long)n);
      }
    }
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
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v <= V; v += (int64_t)gridDim.x * blockDim.x)
    a[v] = v < V ? make_double4(x[v], y[v], z[v], 0.0) : make_double4(-0.0, -0.0, -0.0, 0.0);
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

// dev knob LMS_S2P_OPTS, timing experiments only (wrong results): bit 4 the
// consumers only cycle the ring (no gathers, no stores), bit 5 no neighbour
// waits
static int s2p_opts() {
  const char* e = getenv("LMS_S2P_OPTS");
  return e ? atoi(e) : 0;
}

static int s2_blocks(lms_mesh_s* m) {
  int nsm = 148;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, m->device);
  return nsm * 8;  // 8 CTAs of 256 threads per SM: warps stride the colour's chunks
}

// ---------------------------------------------------------------- S2 direct
// The per-colour launch in the form of jacobi.cu's k_jacobi_direct: a thread
// per free vertex of the colour (cv: the free vertices sorted by colour,
// ascending label inside a colour), row bounds, then 8 column indices, then
// 8 x 3 coordinates, each one round of independent loads straight from the
// relabelled CSR and the SoA coordinates, adds in CSR order (Eq. 1,
// P:244-251; bit-identical to S1/S2).  No slab, no chunk descriptors, no
// interleaved copy.  A launch reads only other colours' coordinates and
// writes only its own colour's, so in-place is the colour-GS order.
__global__ void k_s2d_keys(const int8_t* __restrict__ colour, const uint8_t* __restrict__ fixed, int64_t V,
                           uint8_t* __restrict__ key, int32_t* __restrict__ id) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < V; v += (int64_t)gridDim.x * blockDim.x) {
    key[v] = fixed[v] ? (uint8_t)255 : (uint8_t)colour[v];
    id[v] = (int32_t)v;
  }
}
__global__ void k_s2d_hist(const uint8_t* __restrict__ key, int64_t V, unsigned long long* __restrict__ hist) {
  __shared__ unsigned int h[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) h[i] = 0;
  __syncthreads();
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < V; v += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(&h[key[v]], 1u);
  __syncthreads();
  for (int i = threadIdx.x; i < 256; i += blockDim.x)
    if (h[i]) atomicAdd(&hist[i], (unsigned long long)h[i]);
}
constexpr int S2D_JU = 8;
__global__ void __launch_bounds__(256) k_sweep_s2_direct(const int32_t* __restrict__ rp, const int32_t* __restrict__ col,
                                                         const int32_t* __restrict__ cv, int64_t t0, int64_t t1,
                                                         double* x, double* y, double* z) {
  const int64_t t = t0 + (int64_t)blockIdx.x * 256 + threadIdx.x;
  if (t >= t1) return;
  const int32_t v = __ldg(cv + t);
  const int32_t b = __ldg(rp + v), e = __ldg(rp + v + 1);
  const int32_t n = e - b;
  int32_t u[S2D_JU];
#pragma unroll
  for (int i = 0; i < S2D_JU; ++i) u[i] = i < n ? __ldg(col + b + i) : -1;
  double gx[S2D_JU], gy[S2D_JU], gz[S2D_JU];
#pragma unroll
  for (int i = 0; i < S2D_JU; ++i) {
    gx[i] = gy[i] = gz[i] = 0.0;
    if (u[i] >= 0) {
      gx[i] = x[u[i]];
      gy[i] = y[u[i]];
      gz[i] = z[u[i]];
    }
  }
  double sx = gx[0], sy = gy[0], sz = gz[0];
#pragma unroll
  for (int i = 1; i < S2D_JU; ++i)
    if (i < n) {
      sx = __dadd_rn(sx, gx[i]);
      sy = __dadd_rn(sy, gy[i]);
      sz = __dadd_rn(sz, gz[i]);
    }
  for (int32_t i = S2D_JU; i < n; ++i) {
    const int32_t w = __ldg(col + b + i);
    sx = __dadd_rn(sx, x[w]);
    sy = __dadd_rn(sy, y[w]);
    sz = __dadd_rn(sz, z[w]);
  }
  const double d = (double)n;
  x[v] = __ddiv_rn(sx, d);
  y[v] = __ddiv_rn(sy, d);
  z[v] = __ddiv_rn(sz, d);
}

static void run_s2_direct(lms_mesh_s* m, int sweeps, cudaStream_t s) {
  Schedule& S = m->sched;
  const int64_t V = m->V;
  const int C = m->C;
  if (!S.s2d_cv.p) {
    DBuf<uint8_t> key(V, s), key2(V, s);
    DBuf<int32_t> id(V, s);
    DBuf<unsigned long long> hist(256, s);
    S.s2d_cv.alloc(V, s);
    const unsigned G = grid_for(V, 256) > 4096 ? 4096 : grid_for(V, 256);
    k_s2d_keys<<<G, 256, 0, s>>>(m->colour.p, m->fixed.p, V, key.p, id.p);
    LMS_CHECK_LAUNCH();
    LMS_TRY_CUDA(cudaMemsetAsync(hist.p, 0, 256 * sizeof(unsigned long long), s));
    k_s2d_hist<<<G, 256, 0, s>>>(key.p, V, hist.p);
    LMS_CHECK_LAUNCH();
    size_t tb = 0;
    LMS_TRY_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, key.p, key2.p, id.p, S.s2d_cv.p, (int)V, 0, 8, s));
    {
      DBuf<char> tmp(tb, s);
      LMS_TRY_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tb, key.p, key2.p, id.p, S.s2d_cv.p, (int)V, 0, 8, s));
    }
    std::vector<unsigned long long> h(256);
    LMS_TRY_CUDA(cudaMemcpyAsync(h.data(), hist.p, 256 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
    LMS_TRY_CUDA(cudaStreamSynchronize(s));
    S.s2d_cstart.assign(C + 1, 0);
    for (int c = 0; c < C; ++c) S.s2d_cstart[c + 1] = S.s2d_cstart[c] + (int64_t)h[c];
  }
  sync_soa(m, s);
  soa_changed(m);
  for (int i = 0; i < sweeps; ++i)
    for (int c = 0; c < C; ++c) {
      const int64_t t0 = S.s2d_cstart[c], t1 = S.s2d_cstart[c + 1];
      if (t1 <= t0) continue;
      k_sweep_s2_direct<<<(unsigned)((t1 - t0 + 255) / 256), 256, 0, s>>>(m->row_ptr.p, m->col.p, S.s2d_cv.p, t0, t1,
                                                                         m->x[0].p, m->x[1].p, m->x[2].p);
      LMS_CHECK_LAUNCH();
    }
}

void run_s2(lms_mesh_s* m, int sweeps, cudaStream_t s) {
  if (m->dim != 3) fail(LMS_E_ARG, "the S2 schedule is the 3D kernel (2D meshes use GZ)");
  {  // LMS_S2_DIRECT=1: per-colour launches of the direct kernel (A/B against the slab forms)
    static const bool direct = [] { const char* e = getenv("LMS_S2_DIRECT"); return e && atoi(e) != 0; }();
    if (direct) {
      run_s2_direct(m, sweeps, s);
      return;
    }
  }
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
    // persistent kernel: CTA b takes the tiles [b K / G, (b + 1) K / G)
    {
      int nsm0 = 148;
      cudaDeviceGetAttribute(&nsm0, cudaDevAttrMultiProcessorCount, m->device);
      const int G = (int)std::max<int64_t>(1, std::min<int64_t>(nsm0, K));
      // CTA b takes the consecutive tiles [kb[b], kb[b + 1]): equal shares of
      // the chunk count (all colours), not of the tile count
      std::vector<int64_t> wp(K + 1, 0), kb(G + 1, K);
      for (int64_t k = 0; k < K; ++k) {
        int64_t w = 0;
        for (int c = 0; c < C; ++c) w += h[(size_t)c * K + k + 1] - h[(size_t)c * K + k];
        wp[k + 1] = wp[k] + w;
      }
      kb[0] = 0;
      for (int b = 1; b < G; ++b) {
        const int64_t target = (wp[K] * b + G / 2) / G;
        kb[b] = std::lower_bound(wp.begin(), wp.end(), target) - wp.begin();
        if (kb[b] < kb[b - 1]) kb[b] = kb[b - 1];
        if (kb[b] > K) kb[b] = K;
      }
      std::vector<int32_t> cr((size_t)C * (G + 1));
      for (int c = 0; c < C; ++c)
        for (int b = 0; b <= G; ++b) cr[(size_t)c * (G + 1) + b] = h[(size_t)c * K + (size_t)kb[b]];
      S.s2_G = G;
      S.s2_crange.alloc(cr.size(), s);
      LMS_TRY_CUDA(cudaMemcpyAsync(S.s2_crange.p, cr.data(), cr.size() * sizeof(int32_t), cudaMemcpyHostToDevice, s));
      // CTA neighbourhoods: b waits for the owners of every tile adjacent
      // (through a free-free edge) to one of its tiles
      std::vector<int32_t> tp(K + 1);
      LMS_TRY_CUDA(cudaMemcpyAsync(tp.data(), S.tdep_ptr.p, (K + 1) * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
      LMS_TRY_CUDA(cudaStreamSynchronize(s));
      std::vector<int32_t> td(tp[K] > 0 ? tp[K] : 1);
      if (tp[K] > 0)
        LMS_TRY_CUDA(cudaMemcpyAsync(td.data(), S.tdep.p, tp[K] * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
      LMS_TRY_CUDA(cudaStreamSynchronize(s));
      std::vector<int32_t> owner(K);
      for (int b = 0; b < G; ++b)
        for (int64_t k = kb[b]; k < kb[b + 1]; ++k) owner[k] = b;
      std::vector<int32_t> nbp(G + 1, 0), nbl;
      std::vector<int32_t> mark(G, -1);
      for (int b = 0; b < G; ++b) {
        nbp[b] = (int32_t)nbl.size();
        for (int64_t k = kb[b]; k < kb[b + 1]; ++k)
          for (int32_t q = tp[k]; q < tp[k + 1]; ++q) {
            const int32_t o = owner[td[q]];
            if (o != b && mark[o] != b) {
              mark[o] = b;
              nbl.push_back(o);
            }
          }
      }
      nbp[G] = (int32_t)nbl.size();
      if (nbl.empty()) nbl.push_back(0);
      S.s2_nbptr.alloc(G + 1, s);
      S.s2_nb.alloc(nbl.size(), s);
      S.s2_prog.alloc(G, s);
      LMS_TRY_CUDA(cudaMemcpyAsync(S.s2_nbptr.p, nbp.data(), nbp.size() * sizeof(int32_t), cudaMemcpyHostToDevice, s));
      LMS_TRY_CUDA(cudaMemcpyAsync(S.s2_nb.p, nbl.data(), nbl.size() * sizeof(int32_t), cudaMemcpyHostToDevice, s));
      LMS_TRY_CUDA(cudaStreamSynchronize(s));
    }
    S.s2_choff.alloc(nch > 0 ? nch : 1, s);
    S.s2_chw.alloc(nch > 0 ? nch : 1, s);
    k_s2_fill<<<Gi, 256, 0, s>>>(S.item_ptr.p, S.ioff.p, S.iw.p, K, C, off.p, S.s2_choff.p, S.s2_chw.p);
    LMS_CHECK_LAUNCH();
    {  // widest row count of any item (the ring's slot size)
      std::vector<int32_t> hw(K * C);
      LMS_TRY_CUDA(cudaMemcpyAsync(hw.data(), S.iw.p, hw.size() * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
      LMS_TRY_CUDA(cudaStreamSynchronize(s));
      int wm = 1;
      for (int32_t w : hw) wm = std::max(wm, (int)w);
      S.s2_wmax = wm;
    }
  }
  sync_soa(m, s);
  soa_changed(m);
  DBuf<double> buf(4 * (V + 1), s);  // + the pad vertex X[V] = (-0, -0, -0, 0)
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
  const char* pe2 = getenv("LMS_S2_PERSISTENT");
  const bool used_p = !(pe2 && !strcmp(pe2, "0")) && sweeps > 0;
  if (used_p) {
    // one cooperative launch for every pass of the call
    const long long npass = (long long)sweeps * C;
    const int G = S.s2_G;
    cudaLaunchAttribute at[2];
    int na = 0;
    if (persist) at[na++] = attr[0];
    at[na].id = cudaLaunchAttributeCooperative;
    at[na].val.cooperative = 1;
    ++na;
    cudaLaunchConfig_t cfg = {};
    // ring of R chunk slots of 128 (1 + W) bytes (W = the widest staged row
    // count), LMS_S2R_KB of shared memory (default 96 KB: the rest is L1)
    int kb = 96;
    if (const char* e = getenv("LMS_S2R_KB")) kb = std::max(8, atoi(e));
    const int slot_ints = 32 * (1 + std::min(16, S.s2_wmax));
    // R > 32: the producer stages groups of 32 chunks, lane l waiting for the
    // slot of chunk seq - R, which must precede the group
    int R = std::max(40, std::min(256, kb * 1024 / (slot_ints * 4 + 28)));
    // slots, then full / empty barriers, chunk offsets (8 B each) and widths (4 B)
    const size_t smem = (size_t)R * slot_ints * 4 + (size_t)R * 28;
    // consumer warps x gather batches: 16 x 2 (96 registers) by default;
    // LMS_S2R_VARIANT=2 takes 24 x 4 (72 registers).  C3 original, us per
    // sweep: 12 x 2 181, 16 x 2 169, 20 x 2 182 (spills), 24 x 4 174, 30 x 4 175
    int var = 1;
    if (const char* e = getenv("LMS_S2R_VARIANT")) var = atoi(e);
    auto kern = var == 2 ? k_sweep_s2p<16, 24, 4> : k_sweep_s2p<16, 16, 2>;
    const int ncons = var == 2 ? 24 : 16;
    LMS_TRY_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    cfg.gridDim = dim3((unsigned)G);
    cfg.blockDim = dim3((ncons + 1) * 32);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cfg.attrs = at;
    cfg.numAttrs = na;
    const bool st = getenv("LMS_S2P_STATS") != nullptr;
    DBuf<unsigned long long> stats(st ? 4 * G : 1, s);
    if (st) LMS_TRY_CUDA(cudaMemsetAsync(stats.p, 0, 4 * G * sizeof(unsigned long long), s));
    if (npass >= 0xffffffffLL) fail(LMS_E_ARG, "too many sweeps for one call");
    LMS_TRY_CUDA(cudaMemsetAsync(S.s2_prog.p, 0, G * sizeof(unsigned), s));
    LMS_TRY_CUDA(cudaLaunchKernelEx(&cfg, kern, (const long long*)S.s2_choff.p, (const int32_t*)S.s2_chw.p,
                                    (const int32_t*)S.s2_crange.p, G, C, npass, (const int32_t*)S.slab.p, X,
                                    s2p_opts(), st ? stats.p : (unsigned long long*)nullptr,
                                    (const int32_t*)S.s2_nbptr.p, (const int32_t*)S.s2_nb.p, S.s2_prog.p, m->err.p, R,
                                    slot_ints, (int32_t)V));
    note_launch(1);
    if (st) {
      std::vector<unsigned long long> h(4 * G);
      LMS_TRY_CUDA(cudaMemcpyAsync(h.data(), stats.p, h.size() * 8, cudaMemcpyDeviceToHost, s));
      LMS_TRY_CUDA(cudaStreamSynchronize(s));
      double csum = 0, wsum = 0, psum = 0, cmax = 0;
      for (int b = 0; b < G; ++b) {
        csum += h[4 * b];
        wsum += h[4 * b + 1];
        psum += h[4 * b + 3];
        cmax = std::max(cmax, (double)h[4 * b]);
      }
      fprintf(stderr, "[s2p] %lld passes, G %d, R %d: compute mean %.2f max %.2f us, wait mean %.2f us, producer slot wait %.2f us per pass\n",
              npass, G, R, csum / G / npass / 1e3, cmax / npass / 1e3, wsum / G / npass / 1e3, psum / G / npass / 1e3);
    }
    sweeps = 0;
  }
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
  if (used_p && !m->async_errors) check_err_flag(m, s, "lms_smooth (S2 watchdog: a neighbour wait exceeded its budget)");
}

}  // namespace lms
