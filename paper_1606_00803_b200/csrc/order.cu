// order.cu -- the four vertex orderings of the paper, as GPU kernels.
// perm[new] = old ("V_new[next_num] <- V[i]").
//
//  RANDOM:   perm = argsort of H(seed, 4, i), H the SplitMix64 counter
//                   hash (reading Z15); radix sort of (key, i) pairs.
//  BFS:   queue BFS from `seed`, neighbours in ascending label, restart
//                   at the smallest unvisited label (reading Z14).  Level-
//                   synchronous: each new vertex gets key (rank of its first
//                   discoverer in the current level, label); sorting a level's
//                   keys reproduces the queue order exactly.
//  RDR (Alg. 2): neighbour rows pre-sorted by (quality, label) and
//                   the free vertices sorted by (quality, label) in parallel;
//                   the greedy walk itself is inherently sequential and runs in
//                   ONE warp: each step checks a whole row's `processed` /
//                   `sorted` flags with one warp load, appends the unsorted
//                   members of l in order with a ballot prefix, and advances
//                   to l[0] (readings Z9-Z12).  Never-sorted vertices are
//                   appended in ascending label.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_segmented_sort.cuh>
#include <cub/device/device_select.cuh>

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include <cooperative_groups.h>

#include "lms_internal.cuh"

namespace lms {
namespace cg = cooperative_groups;

__device__ __forceinline__ unsigned long long sm64(unsigned long long z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void k_random_keys(unsigned long long base, int64_t V, unsigned long long* keys, int32_t* idx) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < V; i += (int64_t)gridDim.x * blockDim.x) {
    keys[i] = sm64(base + (unsigned long long)i);
    idx[i] = (int32_t)i;
  }
}

void order_random(lms_mesh_s* m, uint64_t seed, int32_t* d_perm, cudaStream_t s) {
  const int64_t V = m->V;
  // H(seed, 4, i) = SM(SM(seed + 4) + i): the inner SM is a host constant
  unsigned long long z = seed + 4ull;
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  const unsigned long long base = z ^ (z >> 31);
  DBuf<unsigned long long> keys(V, s), keys2(V, s);
  DBuf<int32_t> idx(V, s);
  k_random_keys<<<grid_for(V, 256) > 8192 ? 8192 : grid_for(V, 256), 256, 0, s>>>(base, V, keys.p, idx.p);
  LMS_CHECK_LAUNCH();
  size_t tb = 0;
  LMS_TRY_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, keys.p, keys2.p, idx.p, d_perm, V, 0, 64, s));
  DBuf<char> tmp(tb, s);
  LMS_TRY_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tb, keys.p, keys2.p, idx.p, d_perm, V, 0, 64, s));
}

// ------------------------------------------------------------------------ BFS
__global__ void k_bfs_init(int64_t V, int32_t* rank, int32_t* minpar) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < V; i += (int64_t)gridDim.x * blockDim.x) {
    rank[i] = -1;
    minpar[i] = 0x7fffffff;
  }
}

__global__ void k_bfs_set(int32_t* perm, int32_t* rank, int64_t pos, const int* vtx) {
  perm[pos] = *vtx;
  rank[*vtx] = (int32_t)pos;
}

// expand level perm[head, tail): discover unvisited neighbours, min discoverer rank
__global__ void k_bfs_expand(const int32_t* __restrict__ rp, const int32_t* __restrict__ col,
                             const int32_t* __restrict__ perm, int64_t head, int64_t tail,
                             const int32_t* __restrict__ rank, int32_t* minpar, int32_t* cand, int* ncand) {
  // one warp per level vertex: lanes stride the row
  const int lane = threadIdx.x & 31;
  const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = head + w; i < tail; i += nw) {
    const int32_t p = perm[i];
    for (int32_t j = rp[p] + lane; j < rp[p + 1]; j += 32) {
      const int32_t u = col[j];
      if (rank[u] < 0) {
        int32_t old = atomicMin(&minpar[u], (int32_t)i);
        if (old == 0x7fffffff) cand[atomicAdd(ncand, 1)] = u;
      }
    }
  }
}

// key (discoverer rank, [degree,] label): BFS queue order; with the degree
// (db > 0 bits) the Cuthill-McKee queue order (children by (degree, label))
__global__ void k_bfs_keys(const int32_t* __restrict__ cand, int n, const int32_t* __restrict__ minpar, int b,
                           const int32_t* __restrict__ rp, int db, unsigned long long* keys) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    int32_t u = cand[i];
    const unsigned long long deg = db ? (unsigned long long)(rp[u + 1] - rp[u]) : 0ull;
    keys[i] = ((((unsigned long long)minpar[u] << db) | deg) << b) | (unsigned long long)u;
  }
}

// the unvisited vertex of smallest (degree, label) (Cuthill-McKee start)
__global__ void k_min_deg_unvisited(const int32_t* __restrict__ rank, const int32_t* __restrict__ rp, int64_t V,
                                    unsigned long long* out) {
  unsigned long long best = ~0ull;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < V; i += (int64_t)gridDim.x * blockDim.x)
    if (rank[i] < 0) {
      const unsigned long long k = ((unsigned long long)(rp[i + 1] - rp[i]) << 32) | (unsigned long long)i;
      best = k < best ? k : best;
    }
  for (int o = 16; o; o >>= 1) {
    const unsigned long long x = __shfl_down_sync(0xffffffffu, best, o);
    best = x < best ? x : best;
  }
  if ((threadIdx.x & 31) == 0 && best != ~0ull) atomicMin(out, best);
}

__global__ void k_low32(const unsigned long long* in, int* out) { *out = (int)(*in & 0xffffffffull); }

__global__ void k_reverse(const int32_t* __restrict__ in, int64_t V, int32_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < V; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = in[V - 1 - i];
}

__global__ void k_bfs_place(const unsigned long long* __restrict__ keys, int n, int b, int64_t tail, int32_t* perm,
                            int32_t* rank) {
  const unsigned long long mask = (1ull << b) - 1;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    int32_t u = (int32_t)(keys[i] & mask);
    perm[tail + i] = u;
    rank[u] = (int32_t)(tail + i);
  }
}

__global__ void k_min_unvisited(const int32_t* __restrict__ rank, int64_t V, int* out) {
  int best = 0x7fffffff;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < V; i += (int64_t)gridDim.x * blockDim.x)
    if (rank[i] < 0) { best = (int)i; break; }
  for (int o = 16; o; o >>= 1) best = min(best, __shfl_down_sync(0xffffffffu, best, o));
  if ((threadIdx.x & 31) == 0 && best != 0x7fffffff) atomicMin(out, best);
}

__global__ void k_max_degree(const int32_t* __restrict__ rp, int64_t V, int* out) {
  int mx = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < V; i += (int64_t)gridDim.x * blockDim.x)
    mx = max(mx, rp[i + 1] - rp[i]);
  for (int o = 16; o; o >>= 1) mx = max(mx, __shfl_down_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, mx);
}

static int bits_for2(int64_t n) {
  int b = 1;
  while (((int64_t)1 << b) < n) ++b;
  return b;
}

// ------------------------------------------------------------------------ BFS / CM, one launch
// The level loop in ONE cooperative kernel (no host round trip per level).
// Per level [head, tail) of the queue:
//   1. every unvisited neighbour u of a level vertex gets minpar[u] = the
//      smallest level index that discovers it (atomicMin);
//   2. every level vertex counts its children (neighbours u with
//      minpar[u] == its index, still unvisited);
//   3. one block scans the counts (exclusive, chunks of 1024 with a carry);
//   4. every level vertex writes its children at its offset -- ascending label
//      (its CSR row is ascending) for BFS, ascending (degree, label) for CM --
//      which is exactly the queue order (children of earlier queue entries
//      first, each entry's children in enqueue order).
// A component restart takes the unvisited vertex of smallest label (BFS) or
// (degree, label) (CM) by a grid-wide atomicMin.  grid.sync() between phases.
struct BfsCtl {
  long long head, tail, total;
  unsigned long long best;
};

__global__ void __launch_bounds__(256) k_bfs_coop(const int32_t* __restrict__ rp, const int32_t* __restrict__ col,
                                                  int64_t V, int32_t seed, int rcm, int32_t* __restrict__ perm,
                                                  int32_t* __restrict__ rank, int32_t* __restrict__ minpar,
                                                  int32_t* __restrict__ cnt, BfsCtl* ctl) {
  // minpar[u] = the smallest QUEUE POSITION of a vertex that discovers u (not a
  // level index: positions grow level by level, so discovering the next level
  // while this one is being written can never undercut a parent of this level)
  cg::grid_group grid = cg::this_grid();
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t nth = (int64_t)gridDim.x * blockDim.x;
  const int lane = threadIdx.x & 31;
  for (int64_t v = tid; v < V; v += nth) {
    rank[v] = -1;
    minpar[v] = 0x7fffffff;
  }
  if (tid == 0) ctl->best = ~0ull;
  grid.sync();
  __shared__ long long s_carry;
  __shared__ int s_warp[32];
  long long head = 0, tail = 0;
  // discover the unvisited neighbours of queue entries [a, b) (warp per entry)
  auto discover = [&](long long a, long long b) {
    for (long long q = a + (tid >> 5); q < b; q += nth >> 5) {
      const int32_t p = perm[q];
      for (int32_t j = rp[p] + lane; j < rp[p + 1]; j += 32) {
        const int32_t u = col[j];
        if (rank[u] < 0) atomicMin(&minpar[u], (int32_t)q);
      }
    }
  };
  if (!rcm) {
    if (tid == 0) {
      perm[0] = seed;
      rank[seed] = 0;
    }
    tail = 1;
    grid.sync();
    discover(0, 1);
    grid.sync();
  }
  while (tail < V) {
    if (head == tail) {  // restart: smallest unvisited label (BFS) or (degree, label) (CM)
      unsigned long long best = ~0ull;
      for (int64_t v = tid; v < V; v += nth)
        if (rank[v] < 0) {
          const unsigned long long k =
              rcm ? ((unsigned long long)(rp[v + 1] - rp[v]) << 32) | (unsigned long long)v : (unsigned long long)v;
          best = k < best ? k : best;
        }
      for (int o = 16; o; o >>= 1) {
        const unsigned long long x = __shfl_down_sync(0xffffffffu, best, o);
        best = x < best ? x : best;
      }
      if (lane == 0 && best != ~0ull) atomicMin(&ctl->best, best);
      grid.sync();
      const int32_t v = (int32_t)(ctl->best & 0xffffffffull);
      if (tid == 0) {
        perm[tail] = v;
        rank[v] = (int32_t)tail;
      }
      grid.sync();
      if (tid == 0) ctl->best = ~0ull;
      discover(tail, tail + 1);
      ++tail;
      grid.sync();
      continue;
    }
    const int64_t n = tail - head;
    // children per queue entry of the level
    for (int64_t i = tid; i < n; i += nth) {
      const int32_t p = perm[head + i];
      const int32_t me = (int32_t)(head + i);
      int c = 0;
      for (int32_t j = rp[p]; j < rp[p + 1]; ++j) {
        const int32_t u = col[j];
        c += (rank[u] < 0 && minpar[u] == me) ? 1 : 0;
      }
      cnt[i] = c;
    }
    grid.sync();
    // exclusive scan of cnt[0, n) in block 0 (chunks of blockDim with a carry)
    if (blockIdx.x == 0) {
      if (threadIdx.x == 0) s_carry = 0;
      __syncthreads();
      const int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
      for (int64_t base = 0; base < n; base += blockDim.x) {
        const int64_t i = base + threadIdx.x;
        const int x = i < n ? cnt[i] : 0;
        int incl = x;
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += y;
        }
        if (lane == 31) s_warp[w] = incl;
        __syncthreads();
        if (w == 0) {
          int t = lane < nw ? s_warp[lane] : 0;
          for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, t, o);
            if (lane >= o) t += y;
          }
          if (lane < nw) s_warp[lane] = t;  // inclusive warp prefix
        }
        __syncthreads();
        const long long off = s_carry + (w ? s_warp[w - 1] : 0) + incl - x;
        if (i < n) cnt[i] = (int32_t)off;
        __syncthreads();
        if (threadIdx.x == 0) s_carry += s_warp[nw - 1];
        __syncthreads();
      }
      if (threadIdx.x == 0) ctl->total = s_carry;
    }
    grid.sync();
    const long long total = ctl->total;
    // children at their offsets in enqueue order (BFS: ascending label, the
    // row's order; CM: ascending (degree, label)), ranked at once, and -- in
    // the same phase -- each new entry's own discoveries for the next level
    // (a sibling not ranked yet may see its minpar lowered to a position of
    // this new level: never below its parent's, so nothing changes)
    auto put = [&](int32_t u, long long o) {
      perm[o] = u;
      rank[u] = (int32_t)o;  // only this thread writes u (its unique discoverer)
      for (int32_t j = rp[u]; j < rp[u + 1]; ++j) {
        const int32_t x = col[j];
        if (rank[x] < 0) atomicMin(&minpar[x], (int32_t)o);
      }
    };
    for (int64_t i = tid; i < n; i += nth) {
      const int32_t p = perm[head + i];
      const int32_t me = (int32_t)(head + i);
      long long o = tail + cnt[i];
      if (!rcm) {
        for (int32_t j = rp[p]; j < rp[p + 1]; ++j) {
          const int32_t u = col[j];
          if (rank[u] < 0 && minpar[u] == me) put(u, o++);
        }
      } else {  // ascending (degree, label): repeated minimum over the row
        for (;;) {
          unsigned long long bestk = ~0ull;
          for (int32_t j = rp[p]; j < rp[p + 1]; ++j) {
            const int32_t u = col[j];
            if (minpar[u] == me && rank[u] < 0) {
              const unsigned long long k = ((unsigned long long)(rp[u + 1] - rp[u]) << 32) | (unsigned long long)u;
              if (k < bestk) bestk = k;
            }
          }
          if (bestk == ~0ull) break;
          put((int32_t)(bestk & 0xffffffffull), o++);
        }
      }
    }
    head = tail;
    tail += total;
    grid.sync();
  }
}

static int env_int_o(const char* name, int dflt) {
  const char* e = getenv(name);
  return e ? std::max(1, atoi(e)) : dflt;
}

static bool bfs_coop(lms_mesh_s* m, int64_t seed, bool rcm, int32_t* d_perm, cudaStream_t s) {
  if (getenv("LMS_BFS_HOST")) return false;
  int dev = 0, coop = 0, nsm = 0, per_sm = 0;
  LMS_TRY_CUDA(cudaGetDevice(&dev));
  LMS_TRY_CUDA(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev));
  if (!coop) return false;
  LMS_TRY_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  LMS_TRY_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_bfs_coop, 256, 0));
  if (per_sm < 1) return false;
  const int64_t V = m->V;
  DBuf<int32_t> rank(V, s), minpar(V, s), cnt(V, s);
  DBuf<BfsCtl> ctl(1, s);
  const int32_t* rp = m->row_ptr.p;
  const int32_t* col = m->col.p;
  int32_t sd = (int32_t)seed;
  int r = rcm ? 1 : 0;
  int32_t* pp = d_perm;
  int32_t* rk = rank.p;
  int32_t* mp = minpar.p;
  int32_t* cn = cnt.p;
  BfsCtl* cp = ctl.p;
  void* args[] = {(void*)&rp, (void*)&col, (void*)&V, (void*)&sd, (void*)&r, (void*)&pp, (void*)&rk, (void*)&mp,
                  (void*)&cn, (void*)&cp};
  const int blocks = nsm * std::min(per_sm, env_int_o("LMS_BFS_BPS", 1));
  LMS_TRY_CUDA(cudaLaunchCooperativeKernel((void*)k_bfs_coop, dim3(blocks), dim3(256), args, 0, s));
  note_launch();
  LMS_TRY_CUDA(cudaStreamSynchronize(s));  // the buffers above are released on return
  return true;
}

// Queue BFS (rcm = false) or Cuthill-McKee (rcm = true: start and restarts at
// the unvisited vertex of smallest (degree, label), children by (degree,
// label)), level-synchronous: a level's new vertices sorted by (first
// discoverer's rank, [degree,] label) is exactly the queue order.
static void bfs_levels(lms_mesh_s* m, int64_t seed, bool rcm, int32_t* d_perm, cudaStream_t s) {
  if (bfs_coop(m, seed, rcm, d_perm, s)) return;  // one cooperative launch; below: host-driven levels
  const int64_t V = m->V;
  const int b = bits_for2(V + 1);
  int db = 0;
  if (rcm) {
    int32_t maxdeg = 0;
    {
      DBuf<int> md(1, s);
      LMS_TRY_CUDA(cudaMemsetAsync(md.p, 0, sizeof(int), s));
      // degrees are < 2^31; the key needs their bit width
      k_max_degree<<<grid_for(V, 256) > 8192 ? 8192 : grid_for(V, 256), 256, 0, s>>>(m->row_ptr.p, V, md.p);
      LMS_CHECK_LAUNCH();
      LMS_TRY_CUDA(cudaMemcpyAsync(&maxdeg, md.p, sizeof(int), cudaMemcpyDeviceToHost, s));
      LMS_TRY_CUDA(cudaStreamSynchronize(s));
    }
    db = bits_for2((int64_t)maxdeg + 1);
    if (2 * b + db > 64) fail(LMS_E_ARG, "RCM: mesh too large for the 64-bit level keys");
  }
  DBuf<int32_t> rank(V, s), minpar(V, s), cand(V, s);
  DBuf<unsigned long long> keys(V, s), keys2(V, s);
  DBuf<int> dint(2, s);  // [0] = ncand, [1] = vertex scratch
  const unsigned Gv = grid_for(V, 256) > 8192 ? 8192 : grid_for(V, 256);
  k_bfs_init<<<Gv, 256, 0, s>>>(V, rank.p, minpar.p);
  LMS_CHECK_LAUNCH();
  size_t tb_max = 0;
  LMS_TRY_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tb_max, keys.p, keys2.p, (int)V, 0, 2 * b + db, s));
  DBuf<char> tmp(tb_max, s);
  DBuf<unsigned long long> best(1, s);
  auto min_deg_start = [&]() {  // Cuthill-McKee (re)start vertex into dint[1]
    LMS_TRY_CUDA(cudaMemsetAsync(best.p, 0xff, sizeof(unsigned long long), s));
    k_min_deg_unvisited<<<Gv, 256, 0, s>>>(rank.p, m->row_ptr.p, V, best.p);
    LMS_CHECK_LAUNCH();
    k_low32<<<1, 1, 0, s>>>(best.p, dint.p + 1);
    LMS_CHECK_LAUNCH();
  };
  if (rcm) {
    min_deg_start();
  } else {
    int hseed = (int)seed;
    LMS_TRY_CUDA(cudaMemcpyAsync(dint.p + 1, &hseed, sizeof(int), cudaMemcpyHostToDevice, s));
  }
  k_bfs_set<<<1, 1, 0, s>>>(d_perm, rank.p, 0, dint.p + 1);
  LMS_CHECK_LAUNCH();
  int64_t head = 0, tail = 1;
  while (tail < V) {
    if (head == tail) {  // component exhausted: restart at the smallest unvisited label (RCM: (degree, label))
      if (rcm) {
        min_deg_start();
      } else {
        int big = 0x7fffffff;
        LMS_TRY_CUDA(cudaMemcpyAsync(dint.p + 1, &big, sizeof(int), cudaMemcpyHostToDevice, s));
        k_min_unvisited<<<Gv, 256, 0, s>>>(rank.p, V, dint.p + 1);
        LMS_CHECK_LAUNCH();
      }
      k_bfs_set<<<1, 1, 0, s>>>(d_perm, rank.p, tail, dint.p + 1);
      LMS_CHECK_LAUNCH();
      ++tail;
      continue;
    }
    LMS_TRY_CUDA(cudaMemsetAsync(dint.p, 0, sizeof(int), s));
    const int64_t nlev = tail - head;
    unsigned G = grid_for(nlev * 32, 256);
    if (G > 4096) G = 4096;
    k_bfs_expand<<<G, 256, 0, s>>>(m->row_ptr.p, m->col.p, d_perm, head, tail, rank.p, minpar.p, cand.p, dint.p);
    LMS_CHECK_LAUNCH();
    int n = 0;
    LMS_TRY_CUDA(cudaMemcpyAsync(&n, dint.p, sizeof(int), cudaMemcpyDeviceToHost, s));
    LMS_TRY_CUDA(cudaStreamSynchronize(s));
    head = tail;
    if (n == 0) continue;
    unsigned Gn = grid_for(n, 256) > 4096 ? 4096 : grid_for(n, 256);
    k_bfs_keys<<<Gn, 256, 0, s>>>(cand.p, n, minpar.p, b, m->row_ptr.p, db, keys.p);
    LMS_CHECK_LAUNCH();
    size_t tb = tb_max;
    LMS_TRY_CUDA(cub::DeviceRadixSort::SortKeys(tmp.p, tb, keys.p, keys2.p, n, 0, 2 * b + db, s));
    k_bfs_place<<<Gn, 256, 0, s>>>(keys2.p, n, b, tail, d_perm, rank.p);
    LMS_CHECK_LAUNCH();
    tail += n;
  }
}

void order_bfs(lms_mesh_s* m, int64_t seed, int32_t* d_perm, cudaStream_t s) { bfs_levels(m, seed, false, d_perm, s); }

// reverse BFS and reverse Cuthill-McKee (reading Z26): the visit
// order reversed
void order_rbfs(lms_mesh_s* m, int64_t seed, bool rcm, int32_t* d_perm, cudaStream_t s) {
  DBuf<int32_t> fwd(m->V, s);
  bfs_levels(m, seed, rcm, fwd.p, s);
  k_reverse<<<grid_for(m->V, 256) > 8192 ? 8192 : grid_for(m->V, 256), 256, 0, s>>>(fwd.p, m->V, d_perm);
  LMS_CHECK_LAUNCH();
}

// ------------------------------------------------------------------------ DFS
// Depth-first preorder (Fig. 2a; reading Z25): descend to the
// smallest unvisited neighbour of the deepest vertex that has one; restart
// at the smallest unvisited label.  Inherently sequential: one warp, the
// stack in global memory, a vertex's row checked in one warp load per step.
__global__ void k_dfs_walk(const int32_t* __restrict__ rp, const int32_t* __restrict__ col, int64_t V,
                           int32_t seed, uint8_t* vis, int32_t* stk, int32_t* perm) {
  const int lane = threadIdx.x;
  const unsigned FULL = 0xffffffffu;
  int64_t n = 0, nu = 0;
  int32_t start = seed;
  while (n < V) {
    if (vis[start]) {  // restart: smallest unvisited label, 32 labels per probe
      for (;;) {
        const int64_t i = nu + lane;
        const unsigned bal = __ballot_sync(FULL, i < V && !vis[i]);
        if (bal) {
          nu += __ffs(bal) - 1;
          break;
        }
        nu += 32;
      }
      start = (int32_t)nu;
    }
    __syncwarp();
    if (lane == 0) {
      vis[start] = 1;
      perm[n] = start;
      stk[0] = start;
    }
    ++n;
    int64_t top = 1;
    __syncwarp();
    while (top > 0) {
      const int32_t v = stk[top - 1];
      int32_t u = -1;
      for (int32_t base = __ldg(rp + v), e = __ldg(rp + v + 1); base < e && u < 0; base += 32) {
        const int32_t j = base + lane;
        const int32_t c = j < e ? __ldg(col + j) : -1;
        const unsigned bal = __ballot_sync(FULL, c >= 0 && !vis[c]);
        if (bal) u = __shfl_sync(FULL, c, __ffs(bal) - 1);
      }
      if (u < 0) {
        --top;
        continue;
      }
      if (lane == 0) {
        vis[u] = 1;
        perm[n] = u;
        stk[top] = u;
      }
      ++n;
      ++top;
      __syncwarp();
    }
  }
}

void order_dfs(lms_mesh_s* m, int64_t seed, int32_t* d_perm, cudaStream_t s) {
  const int64_t V = m->V;
  DBuf<uint8_t> vis(V, s);
  DBuf<int32_t> stk(V, s);
  LMS_TRY_CUDA(cudaMemsetAsync(vis.p, 0, V, s));
  k_dfs_walk<<<1, 32, 0, s>>>(m->row_ptr.p, m->col.p, V, (int32_t)seed, vis.p, stk.p, d_perm);
  LMS_CHECK_LAUNCH();
}

// ------------------------------------------------------------------------ RDR
__global__ void k_row_qkeys(const int32_t* __restrict__ col, int64_t nnz, const double* __restrict__ q,
                            unsigned long long* keys) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nnz; i += (int64_t)gridDim.x * blockDim.x)
    keys[i] = (unsigned long long)__double_as_longlong(q[col[i]]);
}

__global__ void k_free_qkeys(const uint8_t* __restrict__ fixed, const double* __restrict__ q, int64_t V,
                             unsigned long long* keys, int32_t* ids, int* n) {
  // compaction keeps ascending id order within a warp only; ids are re-sorted
  // stably by the (q, id) radix sort below, which needs ascending ids for ties:
  // so we write (q, id) keys into a V-sized array with sentinel for fixed.
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < V; v += (int64_t)gridDim.x * blockDim.x) {
    ids[v] = (int32_t)v;
    keys[v] = fixed[v] ? ~0ull : (unsigned long long)__double_as_longlong(q[v]);
    if (!fixed[v]) atomicAdd(n, 1);
  }
}

// The walk keeps Alg. 2's two flags as one state byte per vertex (0 = not
// sorted, 1 = sorted, 2 = processed; processed implies sorted).  Only this
// warp reads and writes them, so they are plain (L1-cached) accesses ordered
// by __syncwarp, not volatile L2 round trips.  A step over `cur` loads, per
// lane, one presorted neighbour u, its state and its row bounds in ONE round
// of independent loads; the next vertex l0 = l[0] then has its row bounds in
// a register already, so a step costs two dependent rounds (the row, then its
// states and bounds) instead of four.
__global__ void k_rdr_walk(const int32_t* __restrict__ rp, const int32_t* __restrict__ scol,
                           const int32_t* __restrict__ outer, int64_t n_outer, uint8_t* st,
                           int32_t* perm, long long* stats /* [next, walks] */) {
  const int lane = threadIdx.x;
  const unsigned FULL = 0xffffffffu;
  const unsigned lt = (1u << lane) - 1u;
  long long next = 0, walks = 0;
  int64_t oi = 0;
  while (oi < n_outer) {
    const int64_t idx = oi + lane;
    const int32_t i_l = idx < n_outer ? __ldg(outer + idx) : -1;
    const int p_l = i_l >= 0 ? st[i_l] : 2;
    const unsigned bal = __ballot_sync(FULL, p_l < 2);
    if (bal == 0) { oi += 32; continue; }
    const int first = __ffs(bal) - 1;
    const int32_t i = __shfl_sync(FULL, i_l, first);
    const int si = __shfl_sync(FULL, p_l, first);
    oi += first + 1;
    // Alg. 2: if not sorted[i]: append i; processed[i] <- True
    if (lane == 0) {
      if (si == 0) perm[next] = i;
      st[i] = 2;
    }
    next += si == 0 ? 1 : 0;
    ++walks;
    int32_t cur = i;
    int32_t b = __ldg(rp + cur), e = __ldg(rp + cur + 1);
    __syncwarp();
    for (;;) {
      int32_t l0 = -1, nb = 0, ne = 0;
      for (int32_t base = b; base < e; base += 32) {
        const int32_t j = base + lane;
        const int32_t u = j < e ? __ldg(scol + j) : -1;
        int su = 2;
        int32_t ub = 0, ue = 0;
        if (u >= 0) {  // one round of independent loads: state and row bounds
          su = st[u];
          ub = __ldg(rp + u);
          ue = __ldg(rp + u + 1);
        }
        const unsigned unp = __ballot_sync(FULL, su < 2);
        if (unp && l0 < 0) {
          const int src = __ffs(unp) - 1;
          l0 = __shfl_sync(FULL, u, src);
          nb = __shfl_sync(FULL, ub, src);
          ne = __shfl_sync(FULL, ue, src);
        }
        const unsigned app = __ballot_sync(FULL, su == 0);
        if (su == 0) {
          perm[next + __popc(app & lt)] = u;
          st[u] = 1;
        }
        next += __popc(app);
      }
      if (l0 < 0) break;
      __syncwarp();
      if (lane == 0) st[l0] = 2;
      __syncwarp();
      cur = l0;
      b = nb;
      e = ne;
    }
    __syncwarp();
  }
  if (lane == 0) { stats[0] = next; stats[1] = walks; }
}

// The walk over an ELL copy of the presorted rows (row v at v * WM, -1
// padded; WM = the maximum degree rounded up to 8 or 16): a step loads, per
// lane, its neighbour u's state AND u's whole row (WM / 4 16-byte loads) in
// ONE round of independent loads, so when l0 = l[0] is chosen its row is
// already in lane src's registers and moves to the lanes by shuffles.  A
// step is one dependent memory round instead of two (row, then states), and
// the row-bound loads are gone.  Same order as k_rdr_walk (Alg. 2).
template <int WM>
__global__ void k_rdr_walk_ell(const int32_t* __restrict__ ell, const int32_t* __restrict__ outer, int64_t n_outer,
                               uint8_t* st, int32_t* perm, long long* stats /* [next, walks] */) {
  const int lane = threadIdx.x;
  const unsigned FULL = 0xffffffffu;
  const unsigned lt = (1u << lane) - 1u;
  long long next = 0, walks = 0;
  int64_t oi = 0;
  while (oi < n_outer) {
    const int64_t idx = oi + lane;
    const int32_t i_l = idx < n_outer ? __ldg(outer + idx) : -1;
    const int p_l = i_l >= 0 ? st[i_l] : 2;
    const unsigned bal = __ballot_sync(FULL, p_l < 2);
    if (bal == 0) { oi += 32; continue; }
    const int first = __ffs(bal) - 1;
    const int32_t i = __shfl_sync(FULL, i_l, first);
    const int si = __shfl_sync(FULL, p_l, first);
    oi += first + 1;
    if (lane == 0) {
      if (si == 0) perm[next] = i;
      st[i] = 2;
    }
    next += si == 0 ? 1 : 0;
    ++walks;
    // lane j < WM holds l[j]: the j-th neighbour of cur in (quality, label) order
    int32_t u = lane < WM ? __ldg(ell + (int64_t)i * WM + lane) : -1;
    __syncwarp();
    for (;;) {
      int su = 2;
      int32_t row[WM];
      if (u >= 0) {  // one round: u's state and u's row
        su = st[u];
        const int4* rp4 = reinterpret_cast<const int4*>(ell + (int64_t)u * WM);
#pragma unroll
        for (int q = 0; q < WM / 4; ++q) {
          const int4 t = __ldg(rp4 + q);
          row[4 * q] = t.x;
          row[4 * q + 1] = t.y;
          row[4 * q + 2] = t.z;
          row[4 * q + 3] = t.w;
        }
      } else {
#pragma unroll
        for (int q = 0; q < WM; ++q) row[q] = -1;
      }
      const unsigned unp = __ballot_sync(FULL, su < 2);
      const unsigned app = __ballot_sync(FULL, su == 0);
      if (su == 0) {
        perm[next + __popc(app & lt)] = u;
        st[u] = 1;
      }
      next += __popc(app);
      if (unp == 0) break;
      const int src = __ffs(unp) - 1;
      const int32_t l0 = __shfl_sync(FULL, u, src);
      int32_t un = -1;
#pragma unroll
      for (int q = 0; q < WM; ++q) {
        const int32_t t = __shfl_sync(FULL, row[q], src);
        if (lane == q) un = t;
      }
      __syncwarp();
      if (lane == 0) st[l0] = 2;
      __syncwarp();
      u = un;
    }
    __syncwarp();
  }
  if (lane == 0) { stats[0] = next; stats[1] = walks; }
}

// Windowed RDR (DESIGN reading Z28): window w = labels
// [w L, (w + 1) L) walks Alg. 2 on its induced subgraph -- every neighbour
// outside the window is dropped from the rows -- and fills perm[w L, ...).
// One warp per window, the walk of k_rdr_walk_ell; the windows run in
// parallel (each only reads and writes its own vertices' states).  outer_w:
// the free vertices by (window, quality, label); wofs: per window offsets.
template <int WM>
__global__ void k_rdr_walk_win(const int32_t* __restrict__ ell, const int32_t* __restrict__ outer_w,
                               const int64_t* __restrict__ wofs, int64_t V, int64_t L, int64_t W, uint8_t* st,
                               int32_t* perm, int* err) {
  const int lane = threadIdx.x & 31;
  const unsigned FULL = 0xffffffffu;
  const unsigned lt = (1u << lane) - 1u;
  for (int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < W;
       w += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t lo = w * L, hi = lo + L < V ? lo + L : V;
    long long next = lo;
    int64_t oi = wofs[w];
    const int64_t oe = wofs[w + 1];
    while (oi < oe) {
      const int64_t idx = oi + lane;
      const int32_t i_l = idx < oe ? __ldg(outer_w + idx) : -1;
      const int p_l = i_l >= 0 ? st[i_l] : 2;
      const unsigned bal = __ballot_sync(FULL, p_l < 2);
      if (bal == 0) { oi += 32; continue; }
      const int first = __ffs(bal) - 1;
      const int32_t i = __shfl_sync(FULL, i_l, first);
      const int si = __shfl_sync(FULL, p_l, first);
      oi += first + 1;
      if (lane == 0) {
        if (si == 0) perm[next] = i;
        st[i] = 2;
      }
      next += si == 0 ? 1 : 0;
      int32_t u = lane < WM ? __ldg(ell + (int64_t)i * WM + lane) : -1;
      if (u < lo || u >= hi) u = -1;
      __syncwarp();
      for (;;) {
        int su = 2;
        int32_t row[WM];
        if (u >= 0) {
          su = st[u];
          const int4* rp4 = reinterpret_cast<const int4*>(ell + (int64_t)u * WM);
#pragma unroll
          for (int q = 0; q < WM / 4; ++q) {
            const int4 t = __ldg(rp4 + q);
            row[4 * q] = t.x;
            row[4 * q + 1] = t.y;
            row[4 * q + 2] = t.z;
            row[4 * q + 3] = t.w;
          }
        } else {
#pragma unroll
          for (int q = 0; q < WM; ++q) row[q] = -1;
        }
        const unsigned unp = __ballot_sync(FULL, su < 2);
        const unsigned app = __ballot_sync(FULL, su == 0);
        if (su == 0) {
          perm[next + __popc(app & lt)] = u;
          st[u] = 1;
        }
        next += __popc(app);
        if (unp == 0) break;
        const int src = __ffs(unp) - 1;
        const int32_t l0 = __shfl_sync(FULL, u, src);
        int32_t un = -1;
#pragma unroll
        for (int q = 0; q < WM; ++q) {
          const int32_t t = __shfl_sync(FULL, row[q], src);
          if (lane == q) un = t;
        }
        if (un < lo || un >= hi) un = -1;  // the row restricted to the window
        __syncwarp();
        if (lane == 0) st[l0] = 2;
        __syncwarp();
        u = un;
      }
      __syncwarp();
    }
    // the window's never-sorted vertices, ascending label (reading Z12)
    for (int64_t b = lo; b < hi; b += 32) {
      const int64_t v = b + lane;
      const bool f = v < hi && st[v] == 0;
      const unsigned fb = __ballot_sync(FULL, f);
      if (f) perm[next + __popc(fb & lt)] = (int32_t)v;
      next += __popc(fb);
    }
    if (lane == 0 && next != hi) raise_err(err, LMS_E_PERM);
  }
}
__global__ void k_window_keys(const int32_t* __restrict__ outer, int64_t n, int64_t L, uint32_t* key,
                              unsigned long long* cnt) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t w = (uint32_t)(outer[i] / L);
    key[i] = w;
    atomicAdd(cnt + w, 1ull);
  }
}

__global__ void k_fill_ell(const int32_t* __restrict__ rp, const int32_t* __restrict__ scol, int64_t V, int WM,
                           int32_t* __restrict__ ell) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < V * WM; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = t / WM;
    const int j = (int)(t - v * WM);
    const int32_t b = rp[v], e = rp[v + 1];
    ell[t] = j < e - b ? scol[b + j] : -1;
  }
}

__global__ void k_state_unsorted(const uint8_t* __restrict__ st, int64_t V, uint8_t* flags, int32_t* ids) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < V; v += (int64_t)gridDim.x * blockDim.x) {
    flags[v] = st[v] == 0 ? 1 : 0;
    ids[v] = (int32_t)v;
  }
}

void order_rdr(lms_mesh_s* m, int32_t* d_perm, cudaStream_t s, int64_t L) {
  const int64_t V = m->V, nnz = m->nnz;
  if (L >= V) L = 0;  // one window: Alg. 2 itself
  const double* q = initial_quality(m, s);
  const unsigned Gv = grid_for(V, 256) > 8192 ? 8192 : grid_for(V, 256);
  // rows presorted by (q, label): stable segmented sort of (q bits, col) pairs
  DBuf<int32_t> scol(nnz, s);
  {
    DBuf<unsigned long long> k1(nnz, s), k2(nnz, s);
    const unsigned Gn = grid_for(nnz, 256) > 8192 ? 8192 : grid_for(nnz, 256);
    k_row_qkeys<<<Gn, 256, 0, s>>>(m->col.p, nnz, q, k1.p);
    LMS_CHECK_LAUNCH();
    size_t tb = 0;
    LMS_TRY_CUDA(cub::DeviceSegmentedSort::StableSortPairs(nullptr, tb, k1.p, k2.p, m->col.p, scol.p, nnz, V,
                                                           m->row_ptr.p, m->row_ptr.p + 1, s));
    DBuf<char> tmp(tb, s);
    LMS_TRY_CUDA(cub::DeviceSegmentedSort::StableSortPairs(tmp.p, tb, k1.p, k2.p, m->col.p, scol.p, nnz, V,
                                                           m->row_ptr.p, m->row_ptr.p + 1, s));
  }
  // outer list: free vertices by (q, label); fixed get key ~0 and sort last
  DBuf<int32_t> outer(V, s);
  int64_t n_outer = 0;
  {
    DBuf<unsigned long long> k1(V, s), k2(V, s);
    DBuf<int32_t> ids(V, s);
    DBuf<int> n(1, s);
    LMS_TRY_CUDA(cudaMemsetAsync(n.p, 0, sizeof(int), s));
    k_free_qkeys<<<Gv, 256, 0, s>>>(m->fixed.p, q, V, k1.p, ids.p, n.p);
    LMS_CHECK_LAUNCH();
    size_t tb = 0;
    LMS_TRY_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, k1.p, k2.p, ids.p, outer.p, V, 0, 64, s));
    DBuf<char> tmp(tb, s);
    LMS_TRY_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tb, k1.p, k2.p, ids.p, outer.p, V, 0, 64, s));
    int hn = 0;
    LMS_TRY_CUDA(cudaMemcpyAsync(&hn, n.p, sizeof(int), cudaMemcpyDeviceToHost, s));
    LMS_TRY_CUDA(cudaStreamSynchronize(s));
    n_outer = hn;
  }
  DBuf<uint8_t> state(V, s);
  LMS_TRY_CUDA(cudaMemsetAsync(state.p, 0, V, s));
  if (L > 0) {  // windowed (reading Z28): every window walks in parallel over an ELL copy
    int md = 0;
    {
      DBuf<int> dmd(1, s);
      LMS_TRY_CUDA(cudaMemsetAsync(dmd.p, 0, sizeof(int), s));
      k_max_degree<<<Gv, 256, 0, s>>>(m->row_ptr.p, V, dmd.p);
      LMS_CHECK_LAUNCH();
      LMS_TRY_CUDA(cudaMemcpyAsync(&md, dmd.p, sizeof(int), cudaMemcpyDeviceToHost, s));
      LMS_TRY_CUDA(cudaStreamSynchronize(s));
    }
    const int WM = md <= 8 ? 8 : md <= 16 ? 16 : md <= 32 ? 32 : 0;
    if (WM == 0) fail(LMS_E_ARG, "windowed RDR: maximum degree above 32");
    const int64_t W = (V + L - 1) / L;
    DBuf<int32_t> ell(V * WM, s);
    const unsigned Ge = grid_for(V * WM, 256) > 8192 ? 8192 : grid_for(V * WM, 256);
    k_fill_ell<<<Ge, 256, 0, s>>>(m->row_ptr.p, scol.p, V, WM, ell.p);
    LMS_CHECK_LAUNCH();
    scol.release();
    // outer list by (window, q, label): a stable sort of the (q, label)-sorted
    // list on the window index, and per-window offsets
    DBuf<uint32_t> wk(n_outer > 0 ? n_outer : 1, s), wk2(n_outer > 0 ? n_outer : 1, s);
    DBuf<int32_t> outer_w(n_outer > 0 ? n_outer : 1, s);
    DBuf<unsigned long long> cnt(W + 1, s);
    DBuf<int64_t> wofs(W + 1, s);
    LMS_TRY_CUDA(cudaMemsetAsync(cnt.p, 0, (W + 1) * sizeof(unsigned long long), s));
    if (n_outer > 0) {
      const unsigned Go = grid_for(n_outer, 256) > 8192 ? 8192 : grid_for(n_outer, 256);
      k_window_keys<<<Go, 256, 0, s>>>(outer.p, n_outer, L, wk.p, cnt.p);
      LMS_CHECK_LAUNCH();
      int wb = 1;
      while (((int64_t)1 << wb) < W) ++wb;
      size_t tb = 0;
      LMS_TRY_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, wk.p, wk2.p, outer.p, outer_w.p, n_outer, 0, wb, s));
      DBuf<char> tmp(tb, s);
      LMS_TRY_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tb, wk.p, wk2.p, outer.p, outer_w.p, n_outer, 0, wb, s));
    }
    {
      size_t tb = 0;
      LMS_TRY_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt.p, wofs.p, W + 1, s));
      DBuf<char> tmp(tb, s);
      LMS_TRY_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tb, cnt.p, wofs.p, W + 1, s));
    }
    DBuf<uint8_t> state(V, s);
    LMS_TRY_CUDA(cudaMemsetAsync(state.p, 0, V, s));
    const unsigned Gw = (unsigned)std::min<int64_t>((W + 7) / 8, 148 * 16);
    if (WM == 8)
      k_rdr_walk_win<8><<<Gw, 256, 0, s>>>(ell.p, outer_w.p, wofs.p, V, L, W, state.p, d_perm, m->err.p);
    else if (WM == 16)
      k_rdr_walk_win<16><<<Gw, 256, 0, s>>>(ell.p, outer_w.p, wofs.p, V, L, W, state.p, d_perm, m->err.p);
    else
      k_rdr_walk_win<32><<<Gw, 256, 0, s>>>(ell.p, outer_w.p, wofs.p, V, L, W, state.p, d_perm, m->err.p);
    LMS_CHECK_LAUNCH();
    check_err_flag(m, s, "windowed RDR (a window did not order each of its vertices once)");  // synchronises s
    return;
  }
  DBuf<long long> stats(2, s);
  // the ELL walk for maximum degree <= 16 (LMS_RDR_ELL=0: the CSR walk)
  int md = 0;
  {
    DBuf<int> dmd(1, s);
    LMS_TRY_CUDA(cudaMemsetAsync(dmd.p, 0, sizeof(int), s));
    k_max_degree<<<Gv, 256, 0, s>>>(m->row_ptr.p, V, dmd.p);
    LMS_CHECK_LAUNCH();
    LMS_TRY_CUDA(cudaMemcpyAsync(&md, dmd.p, sizeof(int), cudaMemcpyDeviceToHost, s));
    LMS_TRY_CUDA(cudaStreamSynchronize(s));
  }
  const char* ee = getenv("LMS_RDR_ELL");
  const int WM = md <= 8 ? 8 : md <= 16 ? 16 : 0;
  if (WM > 0 && !(ee && !strcmp(ee, "0"))) {
    DBuf<int32_t> ell(V * WM, s);
    const unsigned Ge = grid_for(V * WM, 256) > 8192 ? 8192 : grid_for(V * WM, 256);
    k_fill_ell<<<Ge, 256, 0, s>>>(m->row_ptr.p, scol.p, V, WM, ell.p);
    LMS_CHECK_LAUNCH();
    scol.release();
    // (a two-hop L1 prefetch of the candidates' rows and states measured
    // slower: C4 8.5 -> 9.5 s)
    if (WM == 8)
      k_rdr_walk_ell<8><<<1, 32, 0, s>>>(ell.p, outer.p, n_outer, state.p, d_perm, stats.p);
    else
      k_rdr_walk_ell<16><<<1, 32, 0, s>>>(ell.p, outer.p, n_outer, state.p, d_perm, stats.p);
    LMS_CHECK_LAUNCH();
    LMS_TRY_CUDA(cudaStreamSynchronize(s));  // ell is released on return
  } else {
    k_rdr_walk<<<1, 32, 0, s>>>(m->row_ptr.p, scol.p, outer.p, n_outer, state.p, d_perm, stats.p);
    LMS_CHECK_LAUNCH();
  }
  long long hs[2] = {0, 0};
  LMS_TRY_CUDA(cudaMemcpyAsync(hs, stats.p, sizeof(hs), cudaMemcpyDeviceToHost, s));
  LMS_TRY_CUDA(cudaStreamSynchronize(s));
  if (hs[0] < V) {  // tail: never-sorted vertices in ascending label (reading Z12)
    DBuf<uint8_t> flags(V, s);
    DBuf<int32_t> ids(V, s);
    DBuf<int> nsel(1, s);
    k_state_unsorted<<<Gv, 256, 0, s>>>(state.p, V, flags.p, ids.p);
    LMS_CHECK_LAUNCH();
    size_t tb = 0;
    LMS_TRY_CUDA(cub::DeviceSelect::Flagged(nullptr, tb, ids.p, flags.p, d_perm + hs[0], nsel.p, V, s));
    DBuf<char> tmp(tb, s);
    LMS_TRY_CUDA(cub::DeviceSelect::Flagged(tmp.p, tb, ids.p, flags.p, d_perm + hs[0], nsel.p, V, s));
    int hn = 0;
    LMS_TRY_CUDA(cudaMemcpyAsync(&hn, nsel.p, sizeof(int), cudaMemcpyDeviceToHost, s));
    LMS_TRY_CUDA(cudaStreamSynchronize(s));
    if (hs[0] + hn != V) fail(LMS_E_CUDA, "RDR did not order every vertex exactly once");
  }
}

}  // namespace lms
