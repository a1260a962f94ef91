// halo.cu -- building blocks of the multi-GPU sweep:
// one colour stage of the schedule, and gather/scatter of coordinates by an
// index list (halo pack / unpack).  The exchange itself runs over NCCL
// (torch.distributed) between the pack and the unpack.
#include "lms_internal.cuh"

namespace lms {

void run_colour_stage(lms_mesh_s* m, int c, cudaStream_t s);  // smooth.cu

__global__ void k_gather_coords(const double* __restrict__ x, const double* __restrict__ y,
                                const double* __restrict__ z, const int32_t* __restrict__ idx, int64_t n,
                                double* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t v = idx[i];
    out[i] = x[v];
    out[n + i] = y[v];
    if (z) out[2 * n + i] = z[v];
  }
}

// interleaved (x, y) copies of the 2D GZ path (see gz.cu): gather from the
// current copy, scatter into both ping-pong copies (a scattered vertex may be
// fixed for the kernel, which never rewrites it in the partner copy)
__global__ void k_gather_aos(const double2* __restrict__ a, const int32_t* __restrict__ idx, int64_t n,
                             double* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double2 p = a[idx[i]];
    out[i] = p.x;
    out[n + i] = p.y;
  }
}

__global__ void k_scatter_aos(double2* __restrict__ a, double2* __restrict__ b, const int32_t* __restrict__ idx,
                              int64_t n, const double* __restrict__ in) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double2 p = make_double2(in[i], in[n + i]);
    a[idx[i]] = p;
    b[idx[i]] = p;
  }
}

__global__ void k_scatter_coords(double* __restrict__ x, double* __restrict__ y, double* __restrict__ z,
                                 const int32_t* __restrict__ idx, int64_t n, const double* __restrict__ in) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t v = idx[i];
    x[v] = in[i];
    y[v] = in[n + i];
    if (z) z[v] = in[2 * n + i];
  }
}

// halo pack: out[a*n + i] = x_a[idx[i]] from whichever copy is current
void halo_pack(lms_mesh_s* m, const int32_t* idx, int64_t n, double* out, cudaStream_t s) {
  if (n == 0) return;
  const unsigned G = grid_for(n, 256) > 4096 ? 4096 : grid_for(n, 256);
  if (m->aos_state == 1) {  // the interleaved copy is current: no conversion of the whole mesh
    k_gather_aos<<<G, 256, 0, s>>>(reinterpret_cast<const double2*>(m->xy[m->xy_cur].p), idx, n, out);
  } else {
    k_gather_coords<<<G, 256, 0, s>>>(m->x[0].p, m->x[1].p, m->dim == 3 ? m->x[2].p : nullptr, idx, n, out);
  }
  LMS_CHECK_LAUNCH();
}

// halo unpack: x_a[idx[i]] = in[a*n + i], into every live copy
void halo_unpack(lms_mesh_s* m, const int32_t* idx, int64_t n, const double* in, cudaStream_t s) {
  if (n == 0) return;
  const unsigned G = grid_for(n, 256) > 4096 ? 4096 : grid_for(n, 256);
  if (m->aos_state != 0) {  // keep the interleaved ping-pong copies current
    k_scatter_aos<<<G, 256, 0, s>>>(reinterpret_cast<double2*>(m->xy[0].p), reinterpret_cast<double2*>(m->xy[1].p),
                                    idx, n, in);
    LMS_CHECK_LAUNCH();
  }
  if (m->aos_state != 1) {
    k_scatter_coords<<<G, 256, 0, s>>>(m->x[0].p, m->x[1].p, m->dim == 3 ? m->x[2].p : nullptr, idx, n, in);
    LMS_CHECK_LAUNCH();
  }
  if (m->aos_state == 0) soa_changed(m);
}

}  // namespace lms

using namespace lms;

extern "C" {

lms_status lms_smooth_colour(lms_mesh_t m, int32_t colour, lms_stream_t stream) {
  try {
    if (!m) fail(LMS_E_ARG, "NULL handle");
    DevGuard dg(m);
    if (colour < 0 || colour >= m->C) fail(LMS_E_ARG, "colour out of range");
    if (m->n_free == 0) return LMS_OK;
    cudaStream_t s = (cudaStream_t)stream;
    sync_soa(m, s);
    if (!m->sched.valid) build_schedule(m, s);
    m->coords_moved = true;
    run_colour_stage(m, colour, s);
    return LMS_OK;
  } catch (const Err& e) {
    set_error(e.msg);
    return e.st;
  }
}

lms_status lms_gather_coords(lms_mesh_t m, const int32_t* d_idx, int64_t n, double* d_out, lms_stream_t stream) {
  try {
    if (!m || (n > 0 && (!d_idx || !d_out)) || n < 0) fail(LMS_E_ARG, "bad argument");
    DevGuard dg(m);
    halo_pack(m, d_idx, n, d_out, (cudaStream_t)stream);
    return LMS_OK;
  } catch (const Err& e) {
    set_error(e.msg);
    return e.st;
  }
}

lms_status lms_scatter_coords(lms_mesh_t m, const int32_t* d_idx, int64_t n, const double* d_in,
                              lms_stream_t stream) {
  try {
    if (!m || (n > 0 && (!d_idx || !d_in)) || n < 0) fail(LMS_E_ARG, "bad argument");
    DevGuard dg(m);
    halo_unpack(m, d_idx, n, d_in, (cudaStream_t)stream);
    m->coords_moved = true;
    return LMS_OK;
  } catch (const Err& e) {
    set_error(e.msg);
    return e.st;
  }
}

}  // extern "C"
