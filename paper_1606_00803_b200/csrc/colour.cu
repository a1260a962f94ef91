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
// Execution (default, k_gc_seq): the definition's own order, in parallel.
// Positions i = orig_id are cut into chunks of S consecutive positions; a
// thread colours its chunk in order, so the chain along consecutive ids costs
// no communication, and a CTA owns a unit of blockDim * S positions whose
// colours it keeps in shared memory, so most cross-chunk waits are
// shared-memory spins; only edges into earlier units go through global
// memory.  Units are claimed in increasing order by co-resident CTAs, so the
// lowest uncoloured position always has every input and a running thread:
// no deadlock.  A vertex is coloured from exactly the colours the sequential
// greedy uses, hence the same result.  Fallback (orig_id not a permutation of
// 0..V-1, or more than 31 lower neighbours; LMS_COLOUR=jp): k_jp_warp,
// persistent warps taking ready vertices from a queue (or continuing with one
// they just released) -- the critical path there is the dependency chain
// (about nx + 2 ny vertices on a row-major grid) times a few global memory
// round trips, about 4 us per step.
#include <algorithm>
#include <vector>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cooperative_groups.h>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_reduce.cuh>

#include "lms_internal.cuh"

namespace cg = cooperative_groups;

namespace lms {

static int env_int_c(const char* name, int dflt, int lo, int hi) {
  const char* e = getenv(name);
  if (!e || !*e) return dflt;
  const int v = atoi(e);
  return v < lo ? lo : (v > hi ? hi : v);
}

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

// ---------------------------------------------------------------- in-order path
// vid[orig_id[v]] = v; error flag if orig_id is not a permutation of 0..V-1
__global__ void k_gc_vid(const int32_t* __restrict__ oid, int64_t V, int32_t* vid, int* bad) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < V; v += (int64_t)gridDim.x * blockDim.x) {
    const int32_t i = oid[v];
    if (i < 0 || i >= V || atomicExch(&vid[i], (int32_t)v) != -1) atomicExch(bad, 1);
  }
}
// largest number of lower-orig_id free neighbours of a free vertex; and the
// mean reach back (position - lowest lower neighbour's position) over free
// vertices with a lower neighbour: reach[0] = sum, reach[1] = count
__global__ void k_gc_max_lower(const int32_t* __restrict__ rp, const int32_t* __restrict__ col,
                               const uint8_t* __restrict__ fixed, const int32_t* __restrict__ oid, int64_t V,
                               int* out, unsigned long long* reach, uint8_t* pstate) {
  int mx = 0;
  unsigned long long rs = 0, rc = 0;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < V; v += (int64_t)gridDim.x * blockDim.x) {
    const int32_t me = oid[v];
    if (fixed[v]) {
      pstate[me] = 0;
      continue;
    }
    int n = 0;
    int32_t lo = me;
    bool cont = false;
    for (int32_t j = rp[v]; j < rp[v + 1]; ++j) {
      const int32_t u = col[j];
      const int32_t pu = oid[u];
      if (!fixed[u] && pu < me) {
        ++n;
        lo = min(lo, pu);
        cont |= pu == me - 1;
      }
    }
    pstate[me] = cont ? 2 : 1;  // free: 1 = starts a chain of consecutive ids, 2 = continues one
    mx = max(mx, n);
    if (n) {
      rs += (unsigned long long)(me - lo);
      ++rc;
    }
  }
  for (int o = 16; o; o >>= 1) {
    mx = max(mx, __shfl_down_sync(0xffffffffu, mx, o));
    rs += __shfl_down_sync(0xffffffffu, rs, o);
    rc += __shfl_down_sync(0xffffffffu, rc, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMax(out, mx);
    atomicAdd(reach, rs);
    atomicAdd(reach + 1, rc);
  }
}
// record of position i (stride RL ints): [0] = number of lower free neighbours
// (-1: fixed vertex), then their positions (orig_ids), in CSR order
// Also: colpos[i] = -1 (free, not yet coloured) or 127 (fixed: never read as
// an input, but complete for the mirror), and ulo[unit] = lowest position
// before the unit that the unit's vertices read (the mirror window).
__global__ void k_gc_records(const int32_t* __restrict__ rp, const int32_t* __restrict__ col,
                             const uint8_t* __restrict__ fixed, const int32_t* __restrict__ oid, int64_t V, int RL,
                             int64_t UNIT, int32_t* rec, int8_t* colpos, int* ulo) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < V; v += (int64_t)gridDim.x * blockDim.x) {
    const int32_t me = oid[v];
    int32_t* r = rec + (int64_t)me * RL;
    colpos[me] = fixed[v] ? 127 : -1;
    if (fixed[v]) { r[0] = -1; continue; }
    const int64_t ub = me / UNIT * UNIT;
    int n = 0, lo = INT32_MAX;
    for (int32_t j = rp[v]; j < rp[v + 1]; ++j) {
      const int32_t u = col[j];
      const int32_t pu = oid[u];
      if (!fixed[u] && pu < me) {
        r[1 + n++] = pu;
        if (pu < ub) lo = min(lo, pu);
      }
    }
    r[0] = n;
    if (lo != INT32_MAX) atomicMin(&ulo[me / UNIT], lo);
  }
}

__device__ __forceinline__ int ld_vol_s8(const int8_t* p) { return *(const volatile int8_t*)p; }

__device__ __forceinline__ void cpa16(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cpa_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// One thread per chunk of S positions, colouring it in order; a unit of
// NWK * 32 * S positions per CTA (NWK worker warps), units claimed in
// increasing order (ctr).  Chunk of worker (warp w, lane l) = l * NWK + w, so
// the lanes of a warp hold chunks NWK apart (mostly independent).  A worker
// warp loops in lock step: each lane colours its next position if all its
// inputs are ready, else tries again next round (no divergent spin loops).
// cs: the unit's colours (shared); colpos: colours by position (global);
// colour: by vertex.  A lane's next G records stream into its own
// shared-memory ring by cp.async (one commit group per record).  Inputs from
// earlier units: the last warp mirrors the unit's window [ulo, ub) of colpos
// into shared memory in 16-byte blocks (re-reading only blocks not yet
// complete), so a worker polls shared memory there too; one round trip to
// global memory per step on unit-boundary rows would otherwise set the pace of
// the whole wavefront.
template <int RL, int G>
__global__ void __launch_bounds__(288) k_gc_seq(const int32_t* __restrict__ rec, const int32_t* __restrict__ vid,
                                                const int* __restrict__ ulo, int64_t V, int S, int MW, int* ctr,
                                                int8_t* colpos, int8_t* colour, int* maxc, int* err,
                                                unsigned long long* st) {
  extern __shared__ __align__(16) unsigned char gsm[];
  __shared__ int64_t s_base, s_mlo;
  __shared__ int s_done;
  constexpr int NV = RL / 4;  // int4 per record
  constexpr int NWK = 8;      // worker warps
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t UNIT = (int64_t)NWK * 32 * S;
  int4* ring = reinterpret_cast<int4*>(gsm) + (size_t)threadIdx.x * G * NV;  // worker lane's G records
  int8_t* cs = reinterpret_cast<int8_t*>(gsm + (size_t)NWK * 32 * G * NV * 16);
  int8_t* mir = cs + UNIT;  // [MW] mirror of colpos[s_mlo, ub)
  int mymax = -1;
  bool dead = false;
  unsigned long long n_rounds = 0, n_prog = 0, n_sweeps = 0, t_unit = 0, n_units = 0;
  long long tu0 = 0;
  for (;;) {
    __syncthreads();  // the previous unit is done with cs / mir / s_*
    if (st && threadIdx.x == 0) {
      const long long t = clock64();
      if (tu0) { t_unit += t - tu0; ++n_units; }
      tu0 = t;
    }
    if (threadIdx.x == 0) {
      const int64_t ub = (int64_t)atomicAdd(ctr, 1) * UNIT;
      s_base = ub;
      int64_t lo = ub < V ? (int64_t)ulo[ub / UNIT] : ub;
      lo = lo >= ub ? ub : (lo & ~(int64_t)15);
      s_mlo = ub - lo <= MW ? lo : ub;  // window too wide: workers read global memory
      s_done = 0;
    }
    for (int64_t q = threadIdx.x; q < UNIT + MW; q += blockDim.x) cs[q] = -1;
    __syncthreads();
    const int64_t ub = s_base;
    if (ub >= V) break;
    const int64_t mlo = s_mlo;
    if (warp == NWK) {  // ------------------------------------------ mirror
      const int nblk = (int)((ub - mlo) >> 4);
      int4* m16 = reinterpret_cast<int4*>(mir);
      const int4* g16 = reinterpret_cast<const int4*>(colpos + mlo);
      long long idle = 0;
      while (nblk > 0) {
        bool all = true;
        for (int k = lane; k < nblk; k += 32) {
          const int4 h = m16[k];
          if (((h.x | h.y | h.z | h.w) & 0x80808080) == 0) continue;  // complete
          int4 g;
          asm volatile("ld.volatile.global.v4.s32 {%0, %1, %2, %3}, [%4];"
                       : "=r"(g.x), "=r"(g.y), "=r"(g.z), "=r"(g.w)
                       : "l"(g16 + k));
          asm volatile("st.volatile.shared.v4.s32 [%0], {%1, %2, %3, %4};" ::"r"(
                           (uint32_t)__cvta_generic_to_shared(m16 + k)),
                       "r"(g.x), "r"(g.y), "r"(g.z), "r"(g.w)
                       : "memory");
          if ((g.x | g.y | g.z | g.w) & 0x80808080) all = false;
        }
        ++n_sweeps;
        if (__all_sync(FULL, all)) break;
        if (*(volatile int*)&s_done == NWK * 32) break;  // the workers are done with the unit
        if (++idle > (1ll << 30)) break;
      }
      continue;
    }
    const int64_t a = ub + (int64_t)(lane * NWK + warp) * S;
    const int64_t b = min(a + S, V);
    auto issue = [&](int64_t p) {  // record p into its ring slot (an empty group past the chunk)
      if (p < b) {
        int4* d = ring + (int)((p - a) % G) * NV;  // slots within the lane's padded ring
        const int4* src = reinterpret_cast<const int4*>(rec + p * RL);
#pragma unroll
        for (int w = 0; w < NV; ++w) cpa16(d + w, src + w);
      }
      cpa_commit();
    };
#pragma unroll
    for (int k = 0; k < G; ++k) issue(a + k);
    int64_t i = a;
    long long stall = 0;
    while (__any_sync(FULL, i < b && !dead)) {
      bool prog = false;
      if (i < b && !dead) {
        cpa_wait<G - 1>();  // record i landed (records i .. i+G-1 are the outstanding groups)
        const int4* r4 = ring + (int)((i - a) % G) * NV;
        int4 qr[NV];
#pragma unroll
        for (int w = 0; w < NV; ++w) qr[w] = r4[w];
        const int n = qr[0].x;
        bool ready = true;
        uint64_t used0 = 0, used1 = 0;
#pragma unroll
        for (int w = 1; w < RL; ++w) {
          if (w > n) break;
          const int4 v4 = qr[w >> 2];
          const int64_t pp = (w & 3) == 0 ? v4.x : (w & 3) == 1 ? v4.y : (w & 3) == 2 ? v4.z : v4.w;
          const int c = pp >= ub ? ld_vol_s8(cs + (pp - ub))
                                 : (pp >= mlo ? ld_vol_s8(mir + (pp - mlo)) : ld_vol_s8(colpos + pp));
          if (c < 0) ready = false;
          else if (c < 64) used0 |= 1ull << c;
          else used1 |= 1ull << (c - 64);
        }
        if (ready) {
          if (n >= 0) {  // a free vertex (fixed ones keep colour -1)
            int c = ~used0 ? __ffsll((long long)~used0) - 1 : (~used1 ? 64 + __ffsll((long long)~used1) - 1 : 128);
            if (c > 126) { raise_err(err, LMS_E_ARG); c = 126; }
            *(volatile int8_t*)(cs + (i - ub)) = (int8_t)c;
            *(volatile int8_t*)(colpos + i) = (int8_t)c;  // by position; k_gc_scatter maps to vertices
            mymax = c > mymax ? c : mymax;
          }
          issue(i + G);  // into the slot record i just vacated
          ++i;
          prog = true;
        }
      }
      ++n_rounds;
      n_prog += prog;
      if (!__any_sync(FULL, prog)) {
        if (++stall > (1ll << 28)) {  // cannot happen (every wait is on a lower position)
          raise_err(err, LMS_E_CUDA);
          dead = true;
        }
      } else {
        stall = 0;
      }
    }
    cpa_wait<0>();
    if (lane == 0) atomicAdd(&s_done, 32);
  }
  for (int o = 16; o; o >>= 1) mymax = max(mymax, __shfl_down_sync(0xffffffffu, mymax, o));
  if ((threadIdx.x & 31) == 0 && mymax >= 0) atomicMax(maxc, mymax);
  if (st && lane == 0) {
    atomicAdd(st + 0, n_rounds);
    atomicAdd(st + 2, n_sweeps);
    if (threadIdx.x == 0) { atomicAdd(st + 3, t_unit); atomicAdd(st + 4, n_units); }
  }
  if (st) {
    for (int o = 16; o; o >>= 1) n_prog += __shfl_down_sync(0xffffffffu, n_prog, o);
    if (lane == 0) atomicAdd(st + 1, n_prog);
  }
}

// ---- batched in-order colouring (default).  One greedy step is a function of
// the previous colour alone: with the colours of v's other lower neighbours
// fixed (mask), c_v = mex(mask + {c_{v-1}}) = (c_{v-1} == m1) ? m2 : m1, where
// m1 = mex(mask) and m2 = mex(mask + {m1}).  Maps of the form
// c -> (c == k) ? x : y are closed under composition, so a warp colours 32
// consecutive positions at once: each lane builds its map, a 5-step shuffle
// scan composes them, and lane j reads its colour off the composed map (the
// first lane's map is constant, so every composed map is).  A batch in which
// some position depends on an in-batch position other than its predecessor
// takes a 32-step shuffle chain instead.  Warp chunks of SW consecutive
// positions, CTA units of 8 * SW, the mirror warp and the claim order are as
// in k_gc_seq.
__device__ __forceinline__ int gc_mex(uint64_t u0, uint64_t u1) {
  return ~u0 ? __ffsll((long long)~u0) - 1 : (~u1 ? 64 + __ffsll((long long)~u1) - 1 : 128);
}
// packed map (k << 16 | x << 8 | y): c -> (c == k) ? x : y;  k = 255: constant y
__device__ __forceinline__ int gc_apply(int f, int c) { return c == ((f >> 16) & 255) ? ((f >> 8) & 255) : (f & 255); }
__device__ __forceinline__ int gc_compose(int a, int b) {  // a o b (b first)
  return (b & 0xff0000) | (gc_apply(a, (b >> 8) & 255) << 8) | gc_apply(a, b & 255);
}

template <int RL>
__global__ void __launch_bounds__(288) k_gc_batch(const int32_t* __restrict__ rec, const int* __restrict__ ulo,
                                                  int64_t V, int SW, int MW, int shift, int* ctr, int8_t* colpos,
                                                  int* maxc, int* err, unsigned long long* st) {
  extern __shared__ __align__(16) unsigned char gsm[];
  __shared__ int64_t s_base, s_mlo;
  __shared__ int s_done;
  constexpr int NV = RL / 4;  // int4 per record
  constexpr int NWK = 8;      // worker warps
  constexpr int G = 4;        // record batches in flight per warp
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t UNIT = (int64_t)NWK * SW;
  int4* ring = reinterpret_cast<int4*>(gsm) + (size_t)warp * G * 32 * NV;  // [G][32][NV] per warp
  int8_t* cs = reinterpret_cast<int8_t*>(gsm + (size_t)NWK * G * 32 * NV * 16);
  int8_t* mir = cs + UNIT;
  int mymax = -1;
  bool dead = false;
  unsigned long long n_rounds = 0, n_batches = 0, n_chain = 0;
  for (;;) {
    __syncthreads();
    if (threadIdx.x == 0) {
      const int64_t ub = (int64_t)atomicAdd(ctr, 1) * UNIT;
      s_base = ub;
      int64_t lo = ub < V ? (int64_t)ulo[ub / UNIT] : ub;
      lo = lo >= ub ? ub : (lo & ~(int64_t)15);
      s_mlo = ub - lo <= MW ? lo : ub;
      s_done = 0;
    }
    for (int64_t q = threadIdx.x; q < UNIT + MW; q += blockDim.x) cs[q] = -1;
    __syncthreads();
    const int64_t ub = s_base;
    if (ub >= V) break;
    const int64_t mlo = s_mlo;
    if (warp == NWK) {  // ------------------------------------------ mirror
      const int nblk = (int)((ub - mlo) >> 4);
      int4* m16 = reinterpret_cast<int4*>(mir);
      const int4* g16 = reinterpret_cast<const int4*>(colpos + mlo);
      long long idle = 0;
      while (nblk > 0) {
        bool all = true;
        // four blocks per lane per step: their global loads are in flight
        // together, so a pass costs about one L2 round trip per 128 blocks
        for (int k0 = lane; k0 < nblk; k0 += 128) {
          int4 g[4];
          bool need[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int k = k0 + 32 * u;
            need[u] = false;
            if (k < nblk) {
              const int4 h = m16[k];
              need[u] = ((h.x | h.y | h.z | h.w) & 0x80808080) != 0;
            }
            if (need[u])
              asm volatile("ld.volatile.global.v4.s32 {%0, %1, %2, %3}, [%4];"
                           : "=r"(g[u].x), "=r"(g[u].y), "=r"(g[u].z), "=r"(g[u].w)
                           : "l"(g16 + k));
          }
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (need[u]) {
              asm volatile("st.volatile.shared.v4.s32 [%0], {%1, %2, %3, %4};" ::"r"(
                               (uint32_t)__cvta_generic_to_shared(m16 + k0 + 32 * u)),
                           "r"(g[u].x), "r"(g[u].y), "r"(g[u].z), "r"(g[u].w)
                           : "memory");
              if ((g[u].x | g[u].y | g[u].z | g[u].w) & 0x80808080) all = false;
            }
        }
        if (__all_sync(FULL, all)) break;
        if (*(volatile int*)&s_done == NWK) break;
        if (++idle > (1ll << 30)) break;
      }
      continue;
    }
    const int64_t a = ub + (int64_t)warp * SW;
    const int64_t b = min(a + SW, V);
    // batch t of the chunk holds positions a0 + 32 t + lane (those in [a, b)).
    // Chunk k starts its batches k mod 32 positions early: when a chunk's
    // positions read the previous chunk's about one chunk back (a grid row),
    // the last lane of batch t then reads the last lane of the previous
    // chunk's batch t instead of the first of batch t + 1, and the wavefront
    // across chunks advances one batch per chunk instead of two
    const int sft = shift ? (int)((a / SW) & 31) : 0;
    const int64_t a0 = a - sft;
    const int nb = a < b ? (int)((b - a0 + 31) / 32) : 0;
    auto issue = [&](int t) {  // records of batch t into its ring slot (empty group past the chunk)
      const int64_t p = a0 + 32 * (int64_t)t + lane;
      if (t < nb && p >= a && p < b) {
        int4* d = ring + ((size_t)(t % G) * 32 + lane) * NV;
        const int4* src = reinterpret_cast<const int4*>(rec + p * RL);
#pragma unroll
        for (int w = 0; w < NV; ++w) cpa16(d + w, src + w);
      }
      cpa_commit();
    };
#pragma unroll
    for (int t = 0; t < G; ++t) issue(t);
    long long stall = 0;
    // lane state for the current batch: its record (registers), the colours
    // seen so far (an OR: re-reads are harmless) and the first input still
    // missing (wpp; -1 = none) -- a waiting round polls only that one
    bool have = false;
    int64_t base = 0, blo = 0, i = 0, wpp = -1;
    bool valid = false, dep_prev = false, cplx = false;
    uint32_t inb = 0;
    uint64_t used0 = 0, used1 = 0;
    int n = -1;
    int4 qr[NV];
    auto poll = [&](int64_t pp) {
      return pp >= ub ? ld_vol_s8(cs + (pp - ub))
                      : (pp >= mlo ? ld_vol_s8(mir + (pp - mlo)) : ld_vol_s8(colpos + pp));
    };
    auto scan = [&]() {  // all inputs of position i; wpp = the first not yet coloured
      wpp = -1;
      dep_prev = false;
      cplx = false;
      inb = 0;
#pragma unroll
      for (int w = 1; w < RL; ++w) {
        if (w > n) break;
        const int4 v4 = qr[w >> 2];
        const int64_t pp = (w & 3) == 0 ? v4.x : (w & 3) == 1 ? v4.y : (w & 3) == 2 ? v4.z : v4.w;
        if (pp >= blo) {  // in this batch (pp < i)
          const int lj = (int)(pp - base);
          inb |= 1u << lj;
          if (lj == lane - 1) dep_prev = true;
          else cplx = true;
        } else {
          const int c = poll(pp);
          if (c < 0) {
            if (wpp < 0) wpp = pp;
          } else if (c < 64) {
            used0 |= 1ull << c;
          } else {
            used1 |= 1ull << (c - 64);
          }
        }
      }
    };
    for (int t = 0; t < nb && !dead;) {
      if (!have) {
        cpa_wait<G - 1>();  // this lane's record of batch t landed
        base = a0 + 32 * (int64_t)t;
        blo = base > a ? base : a;  // lower positions belong to earlier chunks
        i = base + lane;
        valid = i >= a && i < b;
        const int4* r4 = ring + ((size_t)(t % G) * 32 + lane) * NV;
#pragma unroll
        for (int w = 0; w < NV; ++w) qr[w] = valid ? r4[w] : make_int4(-1, 0, 0, 0);
        n = qr[0].x;
        used0 = used1 = 0;
        scan();
        have = true;
      } else if (wpp >= 0 && poll(wpp) >= 0) {
        scan();  // the awaited input arrived: take every input again
      }
      const bool ready = wpp < 0;
      ++n_rounds;
      if (!__all_sync(FULL, ready)) {  // an input from an earlier batch is not coloured yet
        if (++stall > (1ll << 28)) {  // cannot happen (every wait is on a lower position)
          raise_err(err, LMS_E_CUDA);
          dead = true;
        }
        continue;
      }
      have = false;
      stall = 0;
      int colr;
      if (!__any_sync(FULL, cplx)) {
        int f;
        if (n < 0) {
          f = 0xff0000;  // fixed / past the chunk: a constant (never an input)
        } else {
          const int m1 = gc_mex(used0, used1);
          const int m2 = m1 < 64 ? gc_mex(used0 | (1ull << m1), used1) : gc_mex(used0, used1 | (1ull << (m1 - 64)));
          f = dep_prev ? ((min(m1, 254) << 16) | (min(m2, 255) << 8) | min(m1, 255))
                       : (0xff0000 | (min(m1, 255) << 8) | min(m1, 255));
        }
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int pf = __shfl_up_sync(FULL, f, o);
          if (lane >= o) f = gc_compose(f, pf);
        }
        colr = f & 255;
      } else {  // general in-batch dependencies: a 32-step chain
        ++n_chain;
        colr = -1;
        for (int tt = 0; tt < 32; ++tt) {
          if (lane == tt && n >= 0) colr = gc_mex(used0, used1);
          const int ct = __shfl_sync(FULL, colr, tt);
          if (((inb >> tt) & 1u) && ct >= 0) {
            if (ct < 64) used0 |= 1ull << ct;
            else used1 |= 1ull << (ct - 64);
          }
        }
      }
      if (valid && n >= 0) {
        int c = colr;
        if (c > 126) { raise_err(err, LMS_E_ARG); c = 126; }
        *(volatile int8_t*)(cs + (i - ub)) = (int8_t)c;
        *(volatile int8_t*)(colpos + i) = (int8_t)c;
        mymax = c > mymax ? c : mymax;
      }
      ++n_batches;
      issue(t + G);
      ++t;
    }
    cpa_wait<0>();
    __syncwarp();
    if (lane == 0) atomicAdd(&s_done, 1);
  }
  for (int o = 16; o; o >>= 1) mymax = max(mymax, __shfl_down_sync(0xffffffffu, mymax, o));
  if ((threadIdx.x & 31) == 0 && mymax >= 0) atomicMax(maxc, mymax);
  if (st && lane == 0) {
    atomicAdd(st + 0, n_rounds);
    atomicAdd(st + 1, n_batches);
    atomicAdd(st + 2, n_chain);
  }
}

// Chunks of SW positions that hold free positions of one chain of consecutive
// ids and then the start of another: in such a chunk the second chain waits
// for the end of the first (chunks run in order), which serialises whole
// chains across chunks.  Splitting one chain across chunks is harmless.
// Two parallel passes: the first free position of every chunk, then every
// chain start after it marks its chunk.
__global__ void k_gc_first_free(const uint8_t* __restrict__ pstate, int64_t V, int64_t SW, int64_t* first) {
  // one atomic per (warp, chunk): the lowest set position of each chunk the
  // warp's 32 consecutive positions touch (positions ascend with the lane)
  const int lane = threadIdx.x & 31;
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < V; p += (int64_t)gridDim.x * blockDim.x) {
    const bool set = pstate[p] != 0;
    const unsigned m = __ballot_sync(__activemask(), set) & ((1u << lane) - 1u);
    const bool lead = set && (m == 0 || (p - (lane - (31 - __clz(m)))) / SW != p / SW);
    if (lead) atomicMin(reinterpret_cast<unsigned long long*>(first + p / SW), (unsigned long long)p);
  }
}
__global__ void k_gc_bad_chunks(const uint8_t* __restrict__ pstate, const int64_t* __restrict__ first, int64_t V,
                                int64_t SW, int* bad) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < V; p += (int64_t)gridDim.x * blockDim.x)
    if (pstate[p] == 1 && p > first[p / SW]) bad[p / SW] = 1;
}

// colour[v] = colour of position orig_id[v] (fixed vertices: -1)
__global__ void k_gc_scatter(const int32_t* __restrict__ oid, const uint8_t* __restrict__ fixed,
                             const int8_t* __restrict__ colpos, int64_t V, int8_t* colour) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < V; v += (int64_t)gridDim.x * blockDim.x)
    colour[v] = fixed[v] ? (int8_t)-1 : colpos[oid[v]];
}

// in-order colouring; false if it does not apply (caller falls back to JP)
static bool colour_in_order(lms_mesh_s* m, int* maxc, cudaStream_t s) {
  const int64_t V = m->V;
  if (V <= 0 || V > (int64_t)INT32_MAX) return false;
  const unsigned Gv = grid_for(V, 256) > 8192 ? 8192 : grid_for(V, 256);
  DBuf<int32_t> vid(V, s);
  DBuf<int> flags(2, s);  // [0] not a permutation, [1] max lower neighbours
  LMS_TRY_CUDA(cudaMemsetAsync(vid.p, 0xff, V * sizeof(int32_t), s));
  LMS_TRY_CUDA(cudaMemsetAsync(flags.p, 0, 2 * sizeof(int), s));
  k_gc_vid<<<Gv, 256, 0, s>>>(m->orig_id.p, V, vid.p, flags.p);
  LMS_CHECK_LAUNCH();
  DBuf<unsigned long long> reach(2, s);
  DBuf<uint8_t> pstate(V, s);
  LMS_TRY_CUDA(cudaMemsetAsync(reach.p, 0, 2 * sizeof(unsigned long long), s));
  k_gc_max_lower<<<Gv, 256, 0, s>>>(m->row_ptr.p, m->col.p, m->fixed.p, m->orig_id.p, V, flags.p + 1, reach.p,
                                    pstate.p);
  LMS_CHECK_LAUNCH();
  int h[2] = {0, 0};
  unsigned long long hr[2] = {0, 0};
  LMS_TRY_CUDA(cudaMemcpyAsync(h, flags.p, sizeof(h), cudaMemcpyDeviceToHost, s));
  LMS_TRY_CUDA(cudaMemcpyAsync(hr, reach.p, sizeof(hr), cudaMemcpyDeviceToHost, s));
  LMS_TRY_CUDA(cudaStreamSynchronize(s));
  const int64_t mean_reach = hr[1] ? (int64_t)(hr[0] / hr[1]) : 1024;
  if (h[0] || h[1] > 31) return false;
  const int RL = h[1] <= 3 ? 4 : h[1] <= 7 ? 8 : h[1] <= 15 ? 16 : 32;
  const int threads = 288;  // 8 worker warps + the mirror warp
  // batched (default; LMS_GC=lanes: thread-per-chunk k_gc_seq).  Batched: warp
  // chunks of SW consecutive positions, units of 8 * SW.  Lanes: thread
  // chunks of S, units of 256 * S (longer chunks: fewer cross-thread hops but
  // fewer units in flight)
  // Defaults (measured on C2-C5): batched for 2D, lanes for 3D.  A batched
  // warp's chunk is about the mean reach back (on a row-major grid, a row): a
  // longer chunk would hold a vertex and its row-below neighbours, serialising
  // rows inside one warp instead of pipelining them across warps; it is halved
  // while the mesh would not give half the SMs a unit.
  // Chunks must not put the tail of one chain of consecutive ids and the head
  // of the next in one chunk (k_gc_bad_chunks): that serialises the chains.
  // 2D: the batched kernel with SW = the power of two nearest the mean reach
  // (a grid row) if its chunks are aligned (<= 1% bad); else the per-thread
  // kernel if its chunks of S are; else the queue kernel (false here).
  const char* gce = getenv("LMS_GC");
  const int S = env_int_c("LMS_GC_CHUNK", V >= (int64_t)8 << 20 ? 256 : 128, 8, 4096);
  int nsm0 = 0;
  LMS_TRY_CUDA(cudaDeviceGetAttribute(&nsm0, cudaDevAttrMultiProcessorCount, m->device));
  int64_t sw = 1024;
  while (sw * 2 <= std::min<int64_t>(mean_reach + mean_reach / 8, 16384)) sw *= 2;
  while (sw > 1024 && (V + 8 * sw - 1) / (8 * sw) < nsm0 / 2) sw /= 2;
  const int SW = env_int_c("LMS_GC_WCHUNK", (int)sw, 32, 1 << 20) & ~31;
  auto aligned = [&](int64_t chunk) {
    const int64_t nk = (V + chunk - 1) / chunk;
    DBuf<int64_t> first(nk, s);
    DBuf<int> bad(nk, s), nbad(1, s);
    LMS_TRY_CUDA(cudaMemsetAsync(first.p, 0x7f, nk * sizeof(int64_t), s));
    LMS_TRY_CUDA(cudaMemsetAsync(bad.p, 0, nk * sizeof(int), s));
    k_gc_first_free<<<Gv, 256, 0, s>>>(pstate.p, V, chunk, first.p);
    LMS_CHECK_LAUNCH();
    k_gc_bad_chunks<<<Gv, 256, 0, s>>>(pstate.p, first.p, V, chunk, bad.p);
    LMS_CHECK_LAUNCH();
    size_t tb = 0;
    LMS_TRY_CUDA(cub::DeviceReduce::Sum(nullptr, tb, bad.p, nbad.p, (int)nk, s));
    DBuf<char> tmp(tb, s);
    LMS_TRY_CUDA(cub::DeviceReduce::Sum(tmp.p, tb, bad.p, nbad.p, (int)nk, s));
    int hb = 0;
    LMS_TRY_CUDA(cudaMemcpyAsync(&hb, nbad.p, sizeof(hb), cudaMemcpyDeviceToHost, s));
    LMS_TRY_CUDA(cudaStreamSynchronize(s));
    return (int64_t)hb * 100 <= nk;
  };
  bool batched;
  if (gce) {
    batched = strcmp(gce, "lanes") != 0;  // forced (tests, measurements)
  } else {
    batched = m->dim == 2 && aligned(SW);
    if (!batched && !aligned(S)) return false;
  }
  const int64_t UNIT = batched ? (int64_t)8 * SW : (int64_t)256 * S;
  const int64_t units = (V + UNIT - 1) / UNIT;
  DBuf<int32_t> rec((size_t)V * RL, s);
  DBuf<int8_t> colpos(V + 16, s);
  DBuf<int> ulo(units, s);
  LMS_TRY_CUDA(cudaMemsetAsync(ulo.p, 0x7f, units * sizeof(int), s));
  k_gc_records<<<Gv, 256, 0, s>>>(m->row_ptr.p, m->col.p, m->fixed.p, m->orig_id.p, V, RL, UNIT, rec.p, colpos.p,
                                  ulo.p);
  LMS_CHECK_LAUNCH();
  DBuf<int> ctr(1, s);
  LMS_TRY_CUDA(cudaMemsetAsync(ctr.p, 0, sizeof(int), s));
  // mirror window: the widest unit's reach back (16-byte blocks), capped
  // (units reaching further read global memory)
  int MW = 0;
  {
    std::vector<int> hl(units);
    LMS_TRY_CUDA(cudaMemcpyAsync(hl.data(), ulo.p, units * sizeof(int), cudaMemcpyDeviceToHost, s));
    LMS_TRY_CUDA(cudaStreamSynchronize(s));
    for (int64_t u = 0; u < units; ++u)
      if (hl[u] < u * UNIT) MW = (int)std::max<int64_t>(MW, u * UNIT - (hl[u] & ~15));
    const int cap = env_int_c("LMS_GC_MIRROR", 16384, 0, 65536) & ~15;
    if (MW > cap) MW = cap;
    MW = (MW + 15) & ~15;
  }
  constexpr int G = 8;  // records in flight per worker lane (lanes kernel); the batched one keeps 4 batches per warp
  const size_t smem = (batched ? (size_t)8 * 4 * 32 * (RL / 4) * 16 : (size_t)256 * G * (RL / 4) * 16) +
                      (size_t)UNIT + (size_t)MW;
  void (*kern_l)(const int32_t*, const int32_t*, const int*, int64_t, int, int, int*, int8_t*, int8_t*, int*, int*,
                 unsigned long long*) =
      RL == 4 ? k_gc_seq<4, G> : RL == 8 ? k_gc_seq<8, G> : RL == 16 ? k_gc_seq<16, G> : k_gc_seq<32, G>;
  void (*kern_b)(const int32_t*, const int*, int64_t, int, int, int, int*, int8_t*, int*, int*,
                 unsigned long long*) =
      RL == 4 ? k_gc_batch<4> : RL == 8 ? k_gc_batch<8> : RL == 16 ? k_gc_batch<16> : k_gc_batch<32>;
  const void* kern = batched ? (const void*)kern_b : (const void*)kern_l;
  if (smem > 227 * 1024) return false;
  if (smem > 48 * 1024) LMS_TRY_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int nsm = 0, occ = 0;
  LMS_TRY_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, m->device));
  LMS_TRY_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, smem));
  if (occ < 1) return false;
  // co-resident CTAs (a thread may wait on any earlier unit's thread).  The
  // batched kernel polls in lock step: more CTAs per SM only slow every warp's
  // round (LMS_GC_CTAS_PER_SM, default 1 for it)
  if (batched) occ = std::min(occ, env_int_c("LMS_GC_CTAS_PER_SM", 1, 1, 64));
  const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)nsm * occ, units));
  const int32_t* a_rec = rec.p;
  const int32_t* a_vid = vid.p;
  const int* a_ulo = ulo.p;
  int64_t a_V = V;
  int a_S = S;
  int a_mw = MW;
  int* a_ctr = ctr.p;
  int8_t* a_cp = colpos.p;
  int8_t* a_col = m->colour.p;
  int* a_max = maxc;
  int* a_err = m->err.p;
  static unsigned long long* gst = nullptr;
  unsigned long long* a_st = nullptr;
  if (getenv("LMS_COLOUR_STATS")) {
    if (!gst) LMS_TRY_CUDA(cudaMalloc(&gst, 8 * sizeof(unsigned long long)));
    LMS_TRY_CUDA(cudaMemsetAsync(gst, 0, 8 * sizeof(unsigned long long), s));
    a_st = gst;
  }
  int a_sw = SW;
  void* args_l[] = {&a_rec, &a_vid, &a_ulo, &a_V, &a_S, &a_mw, &a_ctr, &a_cp, &a_col, &a_max, &a_err, &a_st};
  int a_shift = env_int_c("LMS_GC_SHIFT", 1, 0, 1);
  void* args_b[] = {&a_rec, &a_ulo, &a_V, &a_sw, &a_mw, &a_shift, &a_ctr, &a_cp, &a_max, &a_err, &a_st};
  void** args = batched ? args_b : args_l;
  const bool verbose = getenv("LMS_COLOUR_VERBOSE") != nullptr;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (verbose) {
    LMS_TRY_CUDA(cudaEventCreate(&e0));
    LMS_TRY_CUDA(cudaEventCreate(&e1));
    LMS_TRY_CUDA(cudaEventRecord(e0, s));
  }
  LMS_TRY_CUDA(cudaLaunchCooperativeKernel((void*)kern, dim3(blocks), dim3(threads), args, smem, s));
  LMS_CHECK_LAUNCH();
  if (verbose) {
    LMS_TRY_CUDA(cudaEventRecord(e1, s));
    LMS_TRY_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f;
    LMS_TRY_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    fprintf(stderr, "[colour] in-order %s: RL=%d S=%d SW=%d mirror=%d blocks=%d units=%lld kernel %.3f ms\n",
            batched ? "batched" : "lanes", RL, S, SW, MW, blocks, (long long)units, ms);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
  }
  k_gc_scatter<<<Gv, 256, 0, s>>>(m->orig_id.p, m->fixed.p, colpos.p, V, m->colour.p);
  LMS_CHECK_LAUNCH();
  if (a_st) {
    unsigned long long h2[8];
    LMS_TRY_CUDA(cudaMemcpyAsync(h2, a_st, sizeof(h2), cudaMemcpyDeviceToHost, s));
    LMS_TRY_CUDA(cudaStreamSynchronize(s));
    if (batched)
      fprintf(stderr, "[colour stats] warp rounds=%llu batches=%llu (%.2f per round) chain batches=%llu\n", h2[0],
              h2[1], h2[0] ? (double)h2[1] / h2[0] : 0.0, h2[2]);
    else
      fprintf(stderr, "[colour stats] warp rounds=%llu lane progress=%llu (%.2f per round) mirror sweeps=%llu "
              "units=%llu mean unit %.1f kcycles\n", h2[0], h2[1], h2[0] ? (double)h2[1] / h2[0] : 0.0, h2[2],
              h2[4], h2[4] ? h2[3] / 1e3 / h2[4] : 0.0);
  }
  return true;
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
    const char* ce = getenv("LMS_COLOUR");
    const bool want_jp = ce && !strcmp(ce, "jp");
    if (!want_jp && colour_in_order(m, maxc.p, s)) {
      k_check_all_coloured<<<Gv, 256, 0, s>>>(m->colour.p, m->fixed.p, V, m->err.p);
      LMS_CHECK_LAUNCH();
      check_err_flag(m, s, "colouring (more than 127 colours)");
      int h = -1;
      LMS_TRY_CUDA(cudaMemcpyAsync(&h, maxc.p, sizeof(int), cudaMemcpyDeviceToHost, s));
      LMS_TRY_CUDA(cudaStreamSynchronize(s));
      m->C = h + 1;
      return;
    }
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
