// alloc.cu -- scratch allocator behind DBuf (lms_internal.cuh).
//
// Every library call allocates and frees its temporaries stream-ordered; an
// e2e step of C4 makes a few hundred such calls.  cudaMallocAsync from a pool
// whose memory is retained is cheap on average, but each call is a driver API
// call, and measured e2e steps showed occasional stalls of tens to hundreds of
// ms inside them.  This keeps freed blocks in a host-side cache keyed by
// (device, stream, size) and hands them back to the next allocation on the
// same stream: the blocks' previous uses precede any new use in that stream's
// order, exactly the guarantee cudaFreeAsync + cudaMallocAsync gave.  A block
// is reused for a request of at least 3/4 of its size.  Cached bytes are
// capped (LMS_CACHE_GB; default a quarter of the device memory, 45 GB on a
// B200; 0 disables the cache); beyond the cap, and on lms_cache_release(),
// blocks go back to the pool with cudaFreeAsync on their stream.  (A 16 GB cap
// was too small for three or four C4 jobs in flight -- each GZ build takes
// ~1.1 GB of walk slots on its stream -- and the churn through the pool gave
// 50-150 ms stalls: bench e2e with four jobs 7.6-22.6 G/s at 16 GB, 24.9 at
// 64 GB; profiles/round2/tile_walk/bench_nj*, bench_c64_*.)
#include <cstdlib>
#include <map>
#include <tuple>
#include <mutex>
#include <unordered_map>

#include "lms_internal.cuh"

namespace lms {

namespace {
// caller-supplied allocator (lms_set_allocator); null = cudaMallocAsync + cache
struct UserAlloc {
  void* (*alloc)(size_t, lms_stream_t, void*) = nullptr;
  void (*free)(void*, lms_stream_t, void*) = nullptr;
  void* ctx = nullptr;
};
UserAlloc& user() {
  static UserAlloc u;
  return u;
}
struct Cache {
  std::mutex mu;
  // block -> (bytes, owning device); bytes 0 = the caller's allocator.  The
  // device is recorded at allocation: a block may be freed while another
  // device is current (a Mesh collected by Python, one process driving several
  // GPUs), and it must go back to its own device's bucket and pool.
  struct Live { size_t bytes; int dev; };
  std::unordered_map<void*, Live> live;
  // (device, stream, bytes) -> blocks: the legacy default stream has the same
  // handle on every device, so the device is part of the key
  std::map<std::tuple<int, cudaStream_t, size_t>, std::vector<void*>> free_;
  size_t cached = 0;
  size_t cap = 0;
  bool init = false;
};
Cache& cache() {
  static Cache* c = new Cache();  // never destroyed: frees may run at exit
  return *c;
}
// cudaFreeAsync with the block's own device current (its stream handle may
// be the legacy default stream, which names a different stream per device)
void free_on(int dev, cudaStream_t s, void* p) {
  int cur = 0;
  cudaGetDevice(&cur);
  if (cur != dev) cudaSetDevice(dev);
  cudaFreeAsync(p, s);
  if (cur != dev) cudaSetDevice(cur);
}
size_t round_bytes(size_t b) {
  if (b <= 4096) return 4096;
  const size_t g = b < ((size_t)1 << 20) ? 4096 : ((size_t)2 << 20);  // 4 KB, then 2 MB granules
  return (b + g - 1) / g * g;
}
}  // namespace

void* ws_alloc(size_t bytes, cudaStream_t s) {
  Cache& c = cache();
  const size_t rb = round_bytes(bytes);
  int dev = 0;
  LMS_TRY_CUDA(cudaGetDevice(&dev));
  if (user().alloc) {
    void* p = user().alloc(rb, (lms_stream_t)s, user().ctx);
    if (!p) fail(LMS_E_NOMEM, "lms_set_allocator: the caller's allocator returned NULL");
    std::lock_guard<std::mutex> g(c.mu);
    c.live[p] = Cache::Live{0, dev};  // 0 = the caller's block
    return p;
  }
  {
    std::lock_guard<std::mutex> g(c.mu);
    if (!c.init) {
      size_t fr = 0, tot = 0;
      double gb = cudaMemGetInfo(&fr, &tot) == cudaSuccess ? (double)tot / 4.0 / 1073741824.0 : 16.0;
      cudaGetLastError();
      if (const char* e = getenv("LMS_CACHE_GB")) gb = atof(e);
      c.cap = gb > 0 ? (size_t)(gb * 1073741824.0) : 0;
      c.init = true;
    }
    if (c.cap) {
      // smallest cached block of this device and stream with rb <= size <= 4/3 rb
      auto it = c.free_.lower_bound(std::make_tuple(dev, s, rb));
      if (it != c.free_.end() && std::get<0>(it->first) == dev && std::get<1>(it->first) == s &&
          std::get<2>(it->first) <= rb + rb / 3 && !it->second.empty()) {
        void* p = it->second.back();
        it->second.pop_back();
        c.cached -= std::get<2>(it->first);
        c.live[p] = Cache::Live{std::get<2>(it->first), dev};
        if (it->second.empty()) c.free_.erase(it);
        return p;
      }
    }
  }
  void* p = nullptr;
  cudaError_t e = cudaMallocAsync(&p, rb, s);
  if (e == cudaErrorMemoryAllocation) {  // give the cache back to the pool and retry once
    cudaGetLastError();
    lms_cache_release();
    e = cudaMallocAsync(&p, rb, s);
  }
  LMS_TRY_CUDA(e);
  std::lock_guard<std::mutex> g(c.mu);
  c.live[p] = Cache::Live{rb, dev};
  return p;
}

void ws_free(void* p, cudaStream_t s) {
  if (!p) return;
  Cache& c = cache();
  std::lock_guard<std::mutex> g(c.mu);
  auto it = c.live.find(p);
  if (it == c.live.end()) {  // not ours (never expected): hand it to the pool
    cudaFreeAsync(p, s);
    return;
  }
  const size_t b = it->second.bytes;
  const int dev = it->second.dev;
  c.live.erase(it);
  if (b == 0) {  // the caller's allocator
    if (user().free) user().free(p, (lms_stream_t)s, user().ctx);
    return;
  }
  if (!c.cap || b > c.cap) {
    free_on(dev, s, p);
    return;
  }
  c.free_[std::make_tuple(dev, s, b)].push_back(p);
  c.cached += b;
  while (c.cached > c.cap && !c.free_.empty()) {  // over the cap: blocks back to the pool
    auto last = std::prev(c.free_.end());
    void* q = last->second.back();
    last->second.pop_back();
    c.cached -= std::get<2>(last->first);
    free_on(std::get<0>(last->first), std::get<1>(last->first), q);
    if (last->second.empty()) c.free_.erase(last);
  }
}

}  // namespace lms

extern "C" lms_status lms_set_allocator(void* (*alloc)(size_t, lms_stream_t, void*),
                                        void (*free_fn)(void*, lms_stream_t, void*), void* ctx) {
  if ((alloc == nullptr) != (free_fn == nullptr)) return LMS_E_ARG;
  lms_cache_release();  // cached blocks came from the previous allocator
  lms::Cache& c = lms::cache();
  std::lock_guard<std::mutex> g(c.mu);
  lms::user().alloc = alloc;
  lms::user().free = free_fn;
  lms::user().ctx = ctx;
  return LMS_OK;
}

extern "C" void lms_cache_release(void) {
  lms::Cache& c = lms::cache();
  std::lock_guard<std::mutex> g(c.mu);
  for (auto& kv : c.free_)
    for (void* q : kv.second) lms::free_on(std::get<0>(kv.first), std::get<1>(kv.first), q);
  c.free_.clear();
  c.cached = 0;
}
