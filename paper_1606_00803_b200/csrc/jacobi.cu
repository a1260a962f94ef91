// jacobi.cu -- the Jacobi sweep, an explicitly named schedule variant
// (LMS_SCHED_JACOBI).
//
// Every free vertex moves to the mean of its neighbours' coordinates from the
// PREVIOUS sweep (Eq. 1): X'[v] = (sum over the CSR row of
// X[u], in CSR order) / deg(v), IEEE binary64 adds and division, no FMA.  Fixed
// vertices keep their value.  This is NOT the colour-ordered Gauss-Seidel
// result of lms_smooth's other schedules (reading Z1): it is offered
// to compare convergence (the paper's loop is in place).
//
// Kernels: k_jacobi_direct (default; see its comment) and k_jacobi, the first
// version (LMS_JACOBI_STAGED=1): one CTA of 256 threads per 256 consecutive
// vertices, the CTA's column indices staged into shared memory by coalesced
// 16-byte loads, a serial gather loop per thread.  Both write the new value
// to the other buffer (ping-pong; both buffers hold the fixed vertices).
// Bytes per sweep: row_ptr + col read once, coordinates read (gathers mostly
// hit L1/L2 for banded orderings), free coordinates written once -- B_sweep
// of SURVEY 8(d).  C4: 302 us per sweep direct, 452 staged.
#include <cstdlib>

#include "lms_internal.cuh"

namespace lms {

constexpr int JB = 256;          // vertices (threads) per CTA
constexpr int JCAP = JB * 12;    // staged column indices per CTA (avg degree <= 12); longer ranges read global

template <int DIM>
__global__ void __launch_bounds__(JB) k_jacobi(const int32_t* __restrict__ rp, const int32_t* __restrict__ col,
                                               const uint8_t* __restrict__ fixed, int64_t V,
                                               const double* __restrict__ x0, const double* __restrict__ y0,
                                               const double* __restrict__ z0, double* __restrict__ x1,
                                               double* __restrict__ y1, double* __restrict__ z1) {
  __shared__ __align__(16) int32_t sc[JCAP + 8];
  for (int64_t base = (int64_t)blockIdx.x * JB; base < V; base += (int64_t)gridDim.x * JB) {
    const int64_t v = base + threadIdx.x;
    const int64_t vend = base + JB < V ? base + JB : V;
    const int32_t c0 = rp[base], c1 = rp[vend];
    const int32_t a0 = c0 & ~3;  // 16-byte aligned start
    const bool staged = c1 - a0 <= JCAP;
    __syncthreads();  // the previous chunk's reads of sc are done
    if (staged) {
      const int n4 = (c1 - a0 + 3) >> 2;
      const int4* src = reinterpret_cast<const int4*>(col + a0);
      for (int i = threadIdx.x; i < n4; i += JB) reinterpret_cast<int4*>(sc)[i] = __ldg(src + i);
    }
    __syncthreads();
    if (v < V && !fixed[v]) {
      const int32_t b = rp[v], e = rp[v + 1];
      const int32_t* row = staged ? sc + (b - a0) : col + b;
      int32_t u = row[0];
      double sx = __ldg(x0 + u), sy = __ldg(y0 + u), sz = DIM == 3 ? __ldg(z0 + u) : 0.0;
      for (int32_t i = 1; i < e - b; ++i) {
        u = row[i];
        sx = __dadd_rn(sx, __ldg(x0 + u));
        sy = __dadd_rn(sy, __ldg(y0 + u));
        if (DIM == 3) sz = __dadd_rn(sz, __ldg(z0 + u));
      }
      const double d = (double)(e - b);
      x1[v] = __ddiv_rn(sx, d);
      y1[v] = __ddiv_rn(sy, d);
      if (DIM == 3) z1[v] = __ddiv_rn(sz, d);
    }
  }
}

// The direct form (default): no staging and no CTA barrier.  A thread loads
// its row bounds, then the first JU (8) column indices of its row in ONE round of
// independent predicated loads (neighbouring threads' rows are adjacent in
// col, so the warp's loads fall in the same few lines and hit L1 after the
// first), then all JU x DIM coordinates in one more round, and adds them in
// CSR order; rows longer than JU finish in a loop.  Three dependent memory
// rounds per vertex with 8-16 loads in flight in each, against the staged
// form's five (chunk bounds, staging, barrier, own bounds, a serial gather
// loop).  Same arithmetic and add order, so the result is bit-identical.
template <int DIM, int JU>
__global__ void __launch_bounds__(JB) k_jacobi_direct(const int32_t* __restrict__ rp, const int32_t* __restrict__ col,
                                                      const uint8_t* __restrict__ fixed, int64_t V,
                                                      const double* __restrict__ x0, const double* __restrict__ y0,
                                                      const double* __restrict__ z0, double* __restrict__ x1,
                                                      double* __restrict__ y1, double* __restrict__ z1) {
  for (int64_t v = (int64_t)blockIdx.x * JB + threadIdx.x; v < V; v += (int64_t)gridDim.x * JB) {
    if (fixed[v]) continue;
    const int32_t b = __ldg(rp + v), e = __ldg(rp + v + 1);
    const int32_t n = e - b;
    int32_t u[JU];
#pragma unroll
    for (int i = 0; i < JU; ++i) u[i] = i < n ? __ldg(col + b + i) : -1;
    double gx[JU], gy[JU], gz[JU];
#pragma unroll
    for (int i = 0; i < JU; ++i) {
      gx[i] = gy[i] = gz[i] = 0.0;
      if (u[i] >= 0) {
        gx[i] = __ldg(x0 + u[i]);
        gy[i] = __ldg(y0 + u[i]);
        if (DIM == 3) gz[i] = __ldg(z0 + u[i]);
      }
    }
    double sx = gx[0], sy = gy[0], sz = gz[0];
#pragma unroll
    for (int i = 1; i < JU; ++i)
      if (i < n) {
        sx = __dadd_rn(sx, gx[i]);
        sy = __dadd_rn(sy, gy[i]);
        if (DIM == 3) sz = __dadd_rn(sz, gz[i]);
      }
    for (int32_t i = JU; i < n; ++i) {
      const int32_t w = __ldg(col + b + i);
      sx = __dadd_rn(sx, __ldg(x0 + w));
      sy = __dadd_rn(sy, __ldg(y0 + w));
      if (DIM == 3) sz = __dadd_rn(sz, __ldg(z0 + w));
    }
    const double d = (double)n;
    x1[v] = __ddiv_rn(sx, d);
    y1[v] = __ddiv_rn(sy, d);
    if (DIM == 3) z1[v] = __ddiv_rn(sz, d);
  }
}

void run_jacobi(lms_mesh_s* m, int sweeps, cudaStream_t s) {
  const int64_t V = m->V;
  sync_soa(m, s);
  soa_changed(m);
  // the second buffer carries the fixed vertices too (never written)
  for (int a = 0; a < m->dim; ++a) {
    if (!m->xalt[a].p || m->xalt[a].n != (size_t)V) m->xalt[a].alloc(V, s);
    LMS_TRY_CUDA(cudaMemcpyAsync(m->xalt[a].p, m->x[a].p, V * sizeof(double), cudaMemcpyDeviceToDevice, s));
  }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t chunks = (V + JB - 1) / JB;
  const unsigned G = (unsigned)(chunks < (int64_t)sms * 8 ? chunks : (int64_t)sms * 8);
  // LMS_JACOBI_STAGED=1: the shared-memory staged form (kept for A/B timing)
  static const bool staged = [] { const char* e = getenv("LMS_JACOBI_STAGED"); return e && atoi(e) != 0; }();
  // 3D: LMS_JACOBI_JU=16 loads 16 neighbours per round instead of 8 (A/B)
  static const bool ju16 = [] { const char* e = getenv("LMS_JACOBI_JU"); return e && atoi(e) == 16; }();
  for (int i = 0; i < sweeps; ++i) {
    double* z0 = m->dim == 3 ? m->x[2].p : nullptr;
    double* z1 = m->dim == 3 ? m->xalt[2].p : nullptr;
    if (m->dim == 2) {
      if (staged)
        k_jacobi<2><<<G, JB, 0, s>>>(m->row_ptr.p, m->col.p, m->fixed.p, V, m->x[0].p, m->x[1].p, z0,
                                     m->xalt[0].p, m->xalt[1].p, z1);
      else
        k_jacobi_direct<2, 8><<<G, JB, 0, s>>>(m->row_ptr.p, m->col.p, m->fixed.p, V, m->x[0].p, m->x[1].p, z0,
                                            m->xalt[0].p, m->xalt[1].p, z1);
    } else {
      if (staged)
        k_jacobi<3><<<G, JB, 0, s>>>(m->row_ptr.p, m->col.p, m->fixed.p, V, m->x[0].p, m->x[1].p, z0,
                                     m->xalt[0].p, m->xalt[1].p, z1);
      else if (ju16)
        k_jacobi_direct<3, 16><<<G, JB, 0, s>>>(m->row_ptr.p, m->col.p, m->fixed.p, V, m->x[0].p, m->x[1].p, z0,
                                                m->xalt[0].p, m->xalt[1].p, z1);
      else
        k_jacobi_direct<3, 8><<<G, JB, 0, s>>>(m->row_ptr.p, m->col.p, m->fixed.p, V, m->x[0].p, m->x[1].p, z0,
                                               m->xalt[0].p, m->xalt[1].p, z1);
    }
    LMS_CHECK_LAUNCH();
    for (int a = 0; a < m->dim; ++a) std::swap(m->x[a], m->xalt[a]);
  }
  ++m->coord_gen;  // xalt no longer mirrors x for the GZ 3D ping-pong
}

}  // namespace lms
