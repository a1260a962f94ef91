// quality.cu -- the global mesh quality of Alg. 1 on the GPU, and the
// convergence-driven smoothing loop around the sweep.
//
// Alg. 1:  quality <- sum_i q_{V[i]};  Global_quality =
// quality / |V|;  while Global_quality < goal: smooth every interior vertex
// (Eq. 1), update Global_quality.  The experiments stop when "the quality has
// improved by less than" 5e-6, and a maximum iteration count
// bounds the loop.
//
//   q_e = sqrt(min l^2) / sqrt(max l^2) over the element's edges, slot pairs
//         (s < t) lexicographic, l^2 = dx*dx + dy*dy [+ dz*dz]
//   q_v = (sum of q_e over the elements containing v, ascending element id,
//         left to right) / n_v
//   Q   = RN(exact sum of q_v) / |V|                             (reading Z24)
//
// Reading Z24: the sum over vertices is taken EXACTLY and rounded
// once.  Then Q does not depend on the storage order, so a relabelling cannot
// change it (the paper: orderings do not change the iteration count,
// P:519-520), and the stop decision (a floating-point comparison that decides
// an integer, the iteration count) is taken on the same value as the oracle's
// (math.fsum, correctly rounded).
//
// Exact sum: a fixed-point "long accumulator" of NL = 36 limbs, limb k holding
// multiples of 2^(32k - 1120) (payload 32 bits, carries in the upper half of
// each u64).  A double m * 2^E (m < 2^53 an integer, E >= -1074) adds its
// mantissa, shifted, into at most 3 limbs -- no rounding anywhere.  Threads
// keep limbs 31..35 (bits 2^-128 .. 2^32, every value >= 2^-75) in registers,
// warps reduce them by shuffles and add them to the global limbs; smaller
// values (never on the configs' meshes) go straight to the global limbs by
// atomics.  One thread then propagates the carries and rounds to nearest-even.
#include <cub/device/device_radix_sort.cuh>

#include "lms_internal.cuh"

namespace lms {

constexpr int QL_N = 36;        // limbs
constexpr int QL_BASE = 1120;   // limb 0's LSB is 2^-1120
constexpr int QL_REG0 = 31;     // first register limb (2^-128)

// q_e of every element from the current coordinates (interleaved pairs when
// the GZ copy is current, else SoA).  Same operation order as A4 / the oracle.
template <bool AOS>
__global__ void k_q_elem(const int32_t* __restrict__ el, int64_t n_el, int k, int dim, const double2* __restrict__ xy,
                         const double* __restrict__ x0, const double* __restrict__ x1, const double* __restrict__ x2,
                         double* __restrict__ qe, int* err) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n_el; e += (int64_t)gridDim.x * blockDim.x) {
    int32_t w[4];
    for (int s = 0; s < k; ++s) w[s] = el[e * k + s];
    double px[4], py[4], pz[4];
    for (int s = 0; s < k; ++s) {
      if (AOS) {
        const double2 p = xy[w[s]];
        px[s] = p.x;
        py[s] = p.y;
      } else {
        px[s] = x0[w[s]];
        py[s] = x1[w[s]];
      }
      pz[s] = dim == 3 ? x2[w[s]] : 0.0;
    }
    double mn = 0.0, mx = 0.0;
    bool first = true;
    for (int s = 0; s < k; ++s)
      for (int t = s + 1; t < k; ++t) {
        double d = __dsub_rn(px[s], px[t]);
        double l2 = __dmul_rn(d, d);
        d = __dsub_rn(py[s], py[t]);
        l2 = __dadd_rn(l2, __dmul_rn(d, d));
        if (dim == 3) {
          d = __dsub_rn(pz[s], pz[t]);
          l2 = __dadd_rn(l2, __dmul_rn(d, d));
        }
        if (first) { mn = l2; mx = l2; first = false; }
        else { if (l2 < mn) mn = l2; if (l2 > mx) mx = l2; }
      }
    if (!(mx > 0.0)) raise_err(err, LMS_E_DEGENERATE);
    qe[e] = __ddiv_rn(__dsqrt_rn(mn), __dsqrt_rn(mx));
  }
}

// The limbs a value's mantissa lands in: L (lowest), pieces p0, p1, p2 < 2^32.
__device__ __forceinline__ void ql_split(double x, int& L, uint32_t& p0, uint32_t& p1, uint32_t& p2) {
  const unsigned long long b = __double_as_longlong(x);
  const int ex = (int)((b >> 52) & 0x7ff);
  unsigned long long m = b & ((1ull << 52) - 1);
  int E;
  if (ex == 0) {
    E = -1074;
  } else {
    m |= 1ull << 52;
    E = ex - 1075;
  }
  const int pos = E + QL_BASE;  // bit position of m's LSB (>= 46)
  L = pos >> 5;
  const int sh = pos & 31;
  const unsigned long long lo = m << sh;
  const unsigned long long hi = sh ? (m >> (64 - sh)) : 0ull;
  p0 = (uint32_t)lo;
  p1 = (uint32_t)(lo >> 32);
  p2 = (uint32_t)hi;
}

// q_v for every vertex (vertex -> element incidence, ascending element id),
// optionally stored, and its exact contribution to the global limbs.
__global__ void k_q_vertex_sum(const int32_t* __restrict__ vptr, const int32_t* __restrict__ vel,
                               const double* __restrict__ qe, int64_t V, double* __restrict__ qv,
                               unsigned long long* __restrict__ acc, int* err) {
  unsigned long long r[5] = {0, 0, 0, 0, 0};  // limbs QL_REG0 .. QL_REG0 + 4
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < V; v += (int64_t)gridDim.x * blockDim.x) {
    const int32_t b = vptr[v], e = vptr[v + 1];
    if (e == b) {
      raise_err(err, LMS_E_ISOLATED);
      continue;
    }
    double s = qe[vel[b]];
    for (int32_t i = b + 1; i < e; ++i) s = __dadd_rn(s, qe[vel[i]]);
    const double q = __ddiv_rn(s, (double)(e - b));
    if (qv) qv[v] = q;
    if (!(q >= 0.0) || q >= 4294967296.0) {  // NaN, negative, or beyond the limbs: not a quality
      raise_err(err, LMS_E_DEGENERATE);
      continue;
    }
    if (q == 0.0) continue;
    int L;
    uint32_t p0, p1, p2;
    ql_split(q, L, p0, p1, p2);
    if (L >= QL_REG0) {
      const int j = L - QL_REG0;
#pragma unroll
      for (int t = 0; t < 5; ++t)
        r[t] += (t == j ? (unsigned long long)p0 : 0ull) + (t == j + 1 ? (unsigned long long)p1 : 0ull) +
                (t == j + 2 ? (unsigned long long)p2 : 0ull);
    } else {  // tiny value: straight to the global limbs
      atomicAdd(acc + L, (unsigned long long)p0);
      atomicAdd(acc + L + 1, (unsigned long long)p1);
      if (p2) atomicAdd(acc + L + 2, (unsigned long long)p2);
    }
  }
#pragma unroll
  for (int t = 0; t < 5; ++t) {
    unsigned long long x = r[t];
    for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    r[t] = x;
  }
  if ((threadIdx.x & 31) == 0)
#pragma unroll
    for (int t = 0; t < 5; ++t)
      if (r[t]) atomicAdd(acc + QL_REG0 + t, r[t]);
}

// carries, then round-to-nearest-even of the exact sum; Q = RN(sum) / V
__global__ void k_q_round(const unsigned long long* __restrict__ acc, int64_t V, double* out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  uint32_t w[QL_N + 2];
  unsigned long long c = 0;
  for (int k = 0; k < QL_N; ++k) {
    const unsigned long long t = acc[k] + c;  // < 2^64: every limb sum < 2^63
    w[k] = (uint32_t)t;
    c = t >> 32;
  }
  w[QL_N] = (uint32_t)c;
  w[QL_N + 1] = (uint32_t)(c >> 32);
  const int NW = QL_N + 2;
  int top = NW - 1;
  while (top >= 0 && w[top] == 0) --top;
  double sum = 0.0;
  if (top >= 0) {
    const int nb = 32 * top + (32 - __clz(w[top]));  // bit length
    int s = nb - 53;
    if (s < 46) s = 46;  // every input is a multiple of 2^-1074 = 2^(46 - 1120)
    auto bit = [&](int i) -> uint32_t { return i < 0 ? 0u : (w[i >> 5] >> (i & 31)) & 1u; };
    // q = bits [s, s + 53)
    unsigned long long q = 0;
    for (int i = 52; i >= 0; --i) q = (q << 1) | bit(s + i);
    const uint32_t rbit = bit(s - 1);
    bool sticky = false;
    for (int i = 0; i < s - 1 && !sticky; ++i) {
      if ((i & 31) == 0 && i + 32 <= s - 1) {  // whole limb
        sticky = w[i >> 5] != 0;
        i += 31;
      } else {
        sticky = bit(i) != 0;
      }
    }
    if (rbit && (sticky || (q & 1ull))) ++q;  // q may become 2^53: still exact below
    sum = scalbn((double)q, s - QL_BASE);
  }
  *out = __ddiv_rn(sum, (double)V);
}

// vertex -> element incidence (ascending element id per vertex), cached in the
// handle until the mesh is relabelled
__global__ void k_q_inc_keys(const int32_t* __restrict__ el, int64_t n, int k, int eb, unsigned long long* keys) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    keys[i] = ((unsigned long long)el[i] << eb) | (unsigned long long)(i / k);
}
__global__ void k_q_inc_split(const unsigned long long* __restrict__ keys, int64_t n, int eb, int64_t V,
                              int32_t* __restrict__ vptr, int32_t* __restrict__ vel) {
  const unsigned long long em = (1ull << eb) - 1;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long kk = keys[i];
    const int64_t v = (int64_t)(kk >> eb);
    vel[i] = (int32_t)(kk & em);
    const int64_t pv = i == 0 ? -1 : (int64_t)(keys[i - 1] >> eb);
    for (int64_t u = pv + 1; u <= v; ++u) vptr[u] = (int32_t)i;  // rows of untouched vertices are empty
    if (i == n - 1)
      for (int64_t u = v + 1; u <= V; ++u) vptr[u] = (int32_t)n;
  }
}

static int nbits(int64_t n) {
  int b = 1;
  while (((int64_t)1 << b) < n) ++b;
  return b;
}

static void ensure_incidence(lms_mesh_s* m, cudaStream_t s) {
  if (m->v2e_valid) return;
  if (!m->k) fail(LMS_E_STATE, "the global quality needs the mesh's elements (P:232-240)");
  const int64_t n = m->n_el * m->k, V = m->V;
  if (n >= ((int64_t)1 << 31)) fail(LMS_E_ARG, "too many element slots for the int32 incidence");
  const int eb = nbits(m->n_el), vb = nbits(V);
  DBuf<unsigned long long> keys(n, s), sorted(n, s);
  const unsigned G = grid_for(n, 256) > 8192 ? 8192 : grid_for(n, 256);
  k_q_inc_keys<<<G, 256, 0, s>>>(m->elems.p, n, m->k, eb, keys.p);
  LMS_CHECK_LAUNCH();
  size_t tb = 0;
  LMS_TRY_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tb, keys.p, sorted.p, n, 0, eb + vb, s));
  {
    DBuf<char> tmp(tb, s);
    LMS_TRY_CUDA(cub::DeviceRadixSort::SortKeys(tmp.p, tb, keys.p, sorted.p, n, 0, eb + vb, s));
  }
  m->v2e_ptr.alloc(V + 1, s);
  m->v2e.alloc(n, s);
  k_q_inc_split<<<G, 256, 0, s>>>(sorted.p, n, eb, V, m->v2e_ptr.p, m->v2e.p);
  LMS_CHECK_LAUNCH();
  m->v2e_valid = true;
}

void global_quality(lms_mesh_s* m, double* d_q /* [1] device */, double* d_qv /* [V] or null */, cudaStream_t s) {
  ensure_incidence(m, s);
  const int64_t V = m->V, n_el = m->n_el;
  DBuf<double> qe(n_el, s);
  DBuf<unsigned long long> acc(QL_N, s);
  LMS_TRY_CUDA(cudaMemsetAsync(acc.p, 0, QL_N * sizeof(unsigned long long), s));
  const unsigned Ge = grid_for(n_el, 256) > 4736 ? 4736 : grid_for(n_el, 256);
  if (m->dim == 2 && m->aos_state == 1)
    k_q_elem<true><<<Ge, 256, 0, s>>>(m->elems.p, n_el, m->k, 2, reinterpret_cast<const double2*>(m->xy[m->xy_cur].p),
                                      nullptr, nullptr, nullptr, qe.p, m->err.p);
  else
    k_q_elem<false><<<Ge, 256, 0, s>>>(m->elems.p, n_el, m->k, m->dim, nullptr, m->x[0].p, m->x[1].p,
                                       m->dim == 3 ? m->x[2].p : nullptr, qe.p, m->err.p);
  LMS_CHECK_LAUNCH();
  const unsigned Gv = grid_for(V, 256) > 2368 ? 2368 : grid_for(V, 256);
  k_q_vertex_sum<<<Gv, 256, 0, s>>>(m->v2e_ptr.p, m->v2e.p, qe.p, V, d_qv, acc.p, m->err.p);
  LMS_CHECK_LAUNCH();
  k_q_round<<<1, 32, 0, s>>>(acc.p, V, d_q);
  LMS_CHECK_LAUNCH();
}

static double global_quality_host(lms_mesh_s* m, DBuf<double>& dq, cudaStream_t s) {
  global_quality(m, dq.p, nullptr, s);
  double h = 0.0;
  LMS_TRY_CUDA(cudaMemcpyAsync(&h, dq.p, sizeof(double), cudaMemcpyDeviceToHost, s));
  check_err_flag(m, s, "global quality");  // synchronises s
  return h;
}

}  // namespace lms

using namespace lms;

extern "C" {

lms_status lms_global_quality(lms_mesh_t m, double* h_quality, double* d_vertex_quality, lms_stream_t stream) {
  try {
    if (!m || !h_quality) fail(LMS_E_ARG, "NULL argument");
    DevGuard dg(m);
    cudaStream_t s = (cudaStream_t)stream;
    DBuf<double> dq(1, s);
    global_quality(m, dq.p, d_vertex_quality, s);
    LMS_TRY_CUDA(cudaMemcpyAsync(h_quality, dq.p, sizeof(double), cudaMemcpyDeviceToHost, s));
    check_err_flag(m, s, "lms_global_quality");
    return LMS_OK;
  } catch (const Err& e) {
    set_error(e.msg);
    return e.st;
  }
}

lms_status lms_smooth_until(lms_mesh_t m, double goal, double eps, int32_t max_sweeps, int32_t* sweeps_run,
                            double* h_quality_history, int32_t* stop_reason, lms_stream_t stream) {
  try {
    if (!m || !sweeps_run || !stop_reason) fail(LMS_E_ARG, "NULL argument");
    if (max_sweeps < 0) fail(LMS_E_ARG, "max_sweeps < 0");
    DevGuard dg(m);
    cudaStream_t s = (cudaStream_t)stream;
    DBuf<double> dq(1, s);
    double q = global_quality_host(m, dq, s);
    if (h_quality_history) h_quality_history[0] = q;
    int k = 0;
    for (;;) {
      if (q >= goal) { *stop_reason = LMS_STOP_GOAL; break; }
      if (k == max_sweeps) { *stop_reason = LMS_STOP_MAX; break; }
      if (m->n_free > 0) {
        if (!m->sched.valid) {
          sync_soa(m, s);
          build_schedule(m, s);
        }
        m->coords_moved = true;
        run_sweeps(m, 1, s);
      }
      ++k;
      const double q1 = global_quality_host(m, dq, s);
      if (h_quality_history) h_quality_history[k] = q1;
      const double imp = q1 - q;
      q = q1;
      if (imp < eps) { *stop_reason = LMS_STOP_CONVERGED; break; }
    }
    *sweeps_run = k;
    return LMS_OK;
  } catch (const Err& e) {
    set_error(e.msg);
    return e.st;
  }
}

}  // extern "C"
