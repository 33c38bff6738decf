#include <unordered_map>
#include <chrono>
#include <cstdio>
// api.cu -- the extern "C" boundary (include/tgfx.h): argument checks with the reference's
// error texts, host<->device staging for the synchronous host-buffer calls, and the
// process-wide runtime bits (thread-local error, launch counter, stream-ordered pool).
#include <atomic>
#include <charconv>
#include <cstring>
#include <fstream>
#include <vector>
#include <initializer_list>
#include <mutex>
#include <thread>
#include <new>
#include <string>

#include "graph.cuh"

namespace tgfx {

namespace {
thread_local std::string g_err;
std::atomic<uint64_t> g_launches{0};
std::atomic<int64_t> g_bytes{0};
}  // namespace

void check_cuda(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return;
  cudaGetLastError();  // clear sticky-free errors
  if (e == cudaErrorMemoryAllocation)
    throw Error(TGFX_ENOMEM, std::string("out of device memory (") + what + ")");
  throw Error(TGFX_ECUDA, std::string(cudaGetErrorString(e)) + " (" + what + ")");
}

void count_launch(int n) { g_launches.fetch_add(static_cast<uint64_t>(n)); }

void after_launch(const char* name) {
  count_launch();
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess)
    throw Error(TGFX_ECUDA, std::string("launch of ") + name + " failed: " + cudaGetErrorString(e));
}

const DeviceInfo& device_info() {
  static thread_local DeviceInfo info;
  static thread_local int cached_dev = -1;
  int dev = 0;
  check_cuda(cudaGetDevice(&dev), "cudaGetDevice");
  if (dev != cached_dev) {
    cudaDeviceProp p;
    check_cuda(cudaGetDeviceProperties(&p, dev), "cudaGetDeviceProperties");
    if (p.major < 10)
      throw Error(TGFX_ECUDA, std::string("libtgfx needs an sm_100 device, found ") + p.name);
    info.device = dev;
    info.sms = p.multiProcessorCount;
    info.smem_optin = p.sharedMemPerBlockOptin;
    // keep freed pool memory cached so repeated builds/samples do not return it to the OS
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t thr = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    cached_dev = dev;
  }
  return info;
}

// Large buffers (graph columns, gather records, upload staging) are recycled by exact size:
// freed blocks wait in a small cache (with an event marking the end of their last use) and
// the next request of the same size takes one back.  A host-buffer build allocates and frees
// the same ~16 GB every step; through the driver's pool that re-mapped physical memory now
// and then, stalling single builds for 0.3-0.7 s.
constexpr size_t kBigAlloc = size_t(256) << 20;
constexpr size_t kBigCacheBytes = size_t(40) << 30;

struct BigBlock {
  void* p;
  size_t bytes;
  int dev;
  cudaEvent_t done;
};
std::mutex g_big_mu;
std::unordered_map<void*, std::pair<size_t, int>> g_big_live;  // ptr -> (bytes, device)
std::vector<BigBlock> g_big_free;
size_t g_big_free_bytes = 0;

void* dmalloc(size_t bytes, cudaStream_t s) {
  void* p = nullptr;
  if (bytes == 0) bytes = 16;
  if (bytes >= kBigAlloc) {
    const int dev = device_info().device;
    {
      std::lock_guard<std::mutex> lk(g_big_mu);
      for (size_t i = 0; i < g_big_free.size(); ++i) {
        BigBlock& b = g_big_free[i];
        if (b.bytes == bytes && b.dev == dev) {
          check_cuda(cudaStreamWaitEvent(s, b.done, 0), "cudaStreamWaitEvent");
          cudaEventDestroy(b.done);
          p = b.p;
          g_big_free_bytes -= b.bytes;
          g_big_free.erase(g_big_free.begin() + static_cast<std::ptrdiff_t>(i));
          g_big_live[p] = {bytes, dev};
          return p;
        }
      }
    }
    if (cudaMallocAsync(&p, bytes, s) != cudaSuccess) {  // out of memory: drop the cache
      cudaGetLastError();
      {
        std::lock_guard<std::mutex> lk(g_big_mu);
        for (BigBlock& b : g_big_free) {
          cudaEventSynchronize(b.done);
          cudaEventDestroy(b.done);
          cudaFreeAsync(b.p, 0);
        }
        g_big_free.clear();
        g_big_free_bytes = 0;
      }
      cudaDeviceSynchronize();
      check_cuda(cudaMallocAsync(&p, bytes, s), "cudaMallocAsync");
    }
    std::lock_guard<std::mutex> lk(g_big_mu);
    g_big_live[p] = {bytes, dev};
    return p;
  }
  check_cuda(cudaMallocAsync(&p, bytes, s), "cudaMallocAsync");
  return p;
}

void dfree(void* p, cudaStream_t s) {
  if (!p) return;
  {
    std::lock_guard<std::mutex> lk(g_big_mu);
    auto it = g_big_live.find(p);
    if (it != g_big_live.end()) {
      const size_t bytes = it->second.first;
      const int dev = it->second.second;
      g_big_live.erase(it);
      cudaEvent_t done = nullptr;
      if (cudaEventCreateWithFlags(&done, cudaEventDisableTiming) == cudaSuccess &&
          cudaEventRecord(done, s) == cudaSuccess) {
        g_big_free.push_back({p, bytes, dev, done});
        g_big_free_bytes += bytes;
        while (g_big_free_bytes > kBigCacheBytes && !g_big_free.empty()) {  // oldest first
          BigBlock b = g_big_free.front();
          g_big_free.erase(g_big_free.begin());
          g_big_free_bytes -= b.bytes;
          cudaEventSynchronize(b.done);
          cudaEventDestroy(b.done);
          cudaFreeAsync(b.p, 0);
        }
        return;
      }
      if (done) cudaEventDestroy(done);
    }
  }
  check_cuda(cudaFreeAsync(p, s), "cudaFreeAsync");
}

namespace {

int fail(const std::exception& e) {
  g_err = e.what();
  if (const Error* te = dynamic_cast<const Error*>(&e)) return te->code;
  if (dynamic_cast<const std::bad_alloc*>(&e)) return TGFX_ENOMEM;
  return TGFX_ECUDA;
}

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return TGFX_OK;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }

// RAII device buffer on a stream
struct DBuf {
  void* p = nullptr;
  cudaStream_t s;
  DBuf(size_t bytes, cudaStream_t st) : s(st) { p = dmalloc(bytes, s); }
  ~DBuf() {
    // through dfree: buffers >= kBigAlloc are tracked in g_big_live and must be recycled there
    try {
      dfree(p, s);
    } catch (...) {
    }
  }
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  template <typename T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

void h2d(void* d, const void* h, size_t bytes, cudaStream_t s) {
  if (bytes) TGFX_CUDA(cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, s));
}
void d2h(void* h, const void* d, size_t bytes, cudaStream_t s) {
  if (bytes && h) TGFX_CUDA(cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost, s));
}

// ---- large copies from / to pageable host memory (a std::vector's columns, a caller's
// malloc'd event array).  cudaMemcpy from pageable memory runs through the driver's bounce
// buffer at ~11 GB/s on the pool's hosts; here host threads copy 64 MB chunks into a pinned
// double buffer while the copy engine moves the previous chunk (DMA at ~55 GB/s).
constexpr size_t kRingChunk = size_t(64) << 20;
constexpr size_t kRingMin = size_t(256) << 20;  // smaller copies go straight through

bool host_pinned(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

// memcpy split over up to 16 host threads (1 MB pieces at least)
void par_memcpy(void* dst, const void* src, size_t n) {
  const int T = static_cast<int>(std::min<size_t>(
      std::min<unsigned>(16, std::max(1u, std::thread::hardware_concurrency())),
      std::max<size_t>(1, n >> 20)));
  if (T <= 1) {
    std::memcpy(dst, src, n);
    return;
  }
  auto piece = [=](int t) {
    const size_t a = n * t / T, b = n * (t + 1) / T;
    std::memcpy(static_cast<char*>(dst) + a, static_cast<const char*>(src) + a, b - a);
  };
  std::vector<std::thread> th;
  th.reserve(static_cast<size_t>(T));
  int started = 0;
  try {  // pieces no thread could be started for are copied here
    for (; started < T; ++started) th.emplace_back(piece, started);
  } catch (...) {
  }
  for (int t = started; t < T; ++t) piece(t);
  for (std::thread& x : th) x.join();
}

struct Ring {
  char* pin[2] = {nullptr, nullptr};
  cudaEvent_t done[2] = {nullptr, nullptr};
  int dev = -1;
};

Ring& ring() {
  thread_local Ring r;
  const int dev = device_info().device;
  if (r.dev != dev) {
    r = Ring{};
    for (int i = 0; i < 2; ++i) {
      TGFX_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&r.pin[i]), kRingChunk,
                              cudaHostAllocPortable));
      TGFX_CUDA(cudaEventCreateWithFlags(&r.done[i], cudaEventDisableTiming));
    }
    r.dev = dev;
  }
  return r;
}

// host -> device; returns once the host buffer may be reused (like a pageable cudaMemcpyAsync)
void h2d_big(void* d, const void* h, size_t bytes, cudaStream_t s) {
  if (bytes < kRingMin || host_pinned(h)) return h2d(d, h, bytes, s);
  Ring& r = ring();
  for (size_t off = 0, i = 0; off < bytes; off += kRingChunk, ++i) {
    const size_t n = std::min(kRingChunk, bytes - off);
    char* pin = r.pin[i & 1];
    TGFX_CUDA(cudaEventSynchronize(r.done[i & 1]));  // its previous DMA has read it
    par_memcpy(pin, static_cast<const char*>(h) + off, n);
    TGFX_CUDA(cudaMemcpyAsync(static_cast<char*>(d) + off, pin, n, cudaMemcpyHostToDevice, s));
    TGFX_CUDA(cudaEventRecord(r.done[i & 1], s));
  }
  TGFX_CUDA(cudaStreamSynchronize(s));
}

// device -> host, complete on return
void d2h_big(void* h, const void* d, size_t bytes, cudaStream_t s) {
  if (!h || bytes < kRingMin || host_pinned(h)) {
    d2h(h, d, bytes, s);
    return;
  }
  Ring& r = ring();
  const size_t nch = (bytes + kRingChunk - 1) / kRingChunk;
  auto issue = [&](size_t i) {
    const size_t off = i * kRingChunk, n = std::min(kRingChunk, bytes - off);
    TGFX_CUDA(cudaMemcpyAsync(r.pin[i & 1], static_cast<const char*>(d) + off, n,
                              cudaMemcpyDeviceToHost, s));
    TGFX_CUDA(cudaEventRecord(r.done[i & 1], s));
  };
  for (size_t i = 0; i < std::min<size_t>(2, nch); ++i) issue(i);
  for (size_t i = 0; i < nch; ++i) {
    const size_t off = i * kRingChunk, n = std::min(kRingChunk, bytes - off);
    TGFX_CUDA(cudaEventSynchronize(r.done[i & 1]));
    par_memcpy(static_cast<char*>(h) + off, r.pin[i & 1], n);
    if (i + 2 < nch) issue(i + 2);
  }
}

void check_graph(const tgfx_graph* g) {
  if (!g) throw Error(TGFX_EVALIDATION, "null graph");
}


void check_k(int64_t k) {
  if (k < 1) throw Error(TGFX_EVALIDATION, "k must be at least 1");  // sampler.cpp:25
}

void check_l(int64_t l) {
  if (l < 2) throw Error(TGFX_EVALIDATION, "sequence length must be at least 2");  // sequence.cpp:57
}

// ---- small synchronous host-buffer calls (one forward_concat batch: a few thousand queries)
// Each calling thread keeps one device arena and one stream, so a call is: its H2D copies,
// one or two launches, its D2H copies and one stream synchronisation -- no allocation, no
// pool traffic and no extra round trip for the query check (done on the host buffers).  The
// arena grows to the largest call up to kArenaMax; bigger calls take pool buffers.  The
// stream is a blocking one: it orders after work on the legacy default stream, like the
// rest of the host-buffer calls.  Neither is released before the process exits.
constexpr size_t kArenaMax = size_t(256) << 20;

struct HostCall {
  cudaStream_t s = nullptr;
  char* arena = nullptr;
  size_t cap = 0;
  int dev = -1;
};

HostCall& host_call() {
  thread_local HostCall hc;
  const int dev = device_info().device;
  if (hc.dev != dev) {  // first call on this thread (or after a device switch)
    hc = HostCall{};
    TGFX_CUDA(cudaStreamCreate(&hc.s));
    hc.dev = dev;
  }
  return hc;
}

// device scratch of `bytes` on hc.s: the thread's arena, or a pool buffer held by `own`
struct Scratch {
  char* p = nullptr;
  void* own = nullptr;
  cudaStream_t s = nullptr;
  Scratch(HostCall& hc, size_t bytes) : s(hc.s) {
    if (bytes > kArenaMax) {
      own = dmalloc(bytes, s);
      p = static_cast<char*>(own);
      return;
    }
    if (bytes > hc.cap) {
      if (hc.arena) {
        TGFX_CUDA(cudaStreamSynchronize(hc.s));
        TGFX_CUDA(cudaFree(hc.arena));
        hc.arena = nullptr;
        hc.cap = 0;
      }
      const size_t c = std::min(kArenaMax, std::max(bytes + bytes / 2, size_t(4) << 20));
      TGFX_CUDA(cudaMalloc(&hc.arena, c));
      hc.cap = c;
    }
    p = hc.arena;
  }
  ~Scratch() {
    if (own) {
      try {
        dfree(own, s);
      } catch (...) {
      }
    }
  }
  Scratch(const Scratch&) = delete;
  Scratch& operator=(const Scratch&) = delete;
};

size_t al256(size_t x) { return (x + 255) & ~size_t(255); }

// The copies of one host call, in order; a run of segments adjacent on both sides is issued as
// one copy.  The device scratch places each direction's buffers back to back, so a caller
// whose host buffers are back to back too (the C++ layer's pinned staging) pays one DMA per
// direction instead of one per array.
struct Seg {
  void* dst;
  const void* src;
  size_t n;
};
void copy_merged(std::initializer_list<Seg> segs, cudaMemcpyKind kind, cudaStream_t s) {
  char* d = nullptr;
  const char* h = nullptr;
  size_t n = 0;
  auto flush = [&] {
    if (n && d && h) TGFX_CUDA(cudaMemcpyAsync(d, h, n, kind, s));
    n = 0;
  };
  for (const Seg& g : segs) {
    if (!g.n || !g.dst || !g.src) continue;
    if (n && static_cast<char*>(g.dst) == d + n && static_cast<const char*>(g.src) == h + n) {
      n += g.n;
      continue;
    }
    flush();
    d = static_cast<char*>(g.dst);
    h = static_cast<const char*>(g.src);
    n = g.n;
  }
  flush();
}

// sampler.cpp:88-93 on the caller's host buffer: every query's node in order, then k (checked
// with query 0, so k < 1 reports after query 0's node)
void check_queries_host(const tgfx_graph* g, const int64_t* nodes, int64_t q, int64_t k) {
  if (q < 0) throw Error(TGFX_EVALIDATION, "negative query count");
  if (q == 0) return;
  const int64_t n = k < 1 ? 1 : q;
  for (int64_t i = 0; i < n; ++i)
    if (nodes[i] < 0 || nodes[i] >= g->V)
      throw Error(TGFX_EVALIDATION, "query node " + std::to_string(nodes[i]) + " out of range");
  check_k(k);
}

void check_queries(const tgfx_graph* g, const int64_t* d_nodes, int64_t q, int64_t k,
                   cudaStream_t s) {
  // sampler.cpp:88-93: every query validated before any sampling (node first, then k)
  if (q < 0) throw Error(TGFX_EVALIDATION, "negative query count");
  if (q == 0) return;
  // first failing check in query order: query 0's node, then k (checked with query 0)
  const int64_t bad = find_bad_query(g, d_nodes, k < 1 ? 1 : q, s);
  if (bad >= 0) {
    int64_t u = 0;
    TGFX_CUDA(cudaMemcpyAsync(&u, d_nodes + bad, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    TGFX_CUDA(cudaStreamSynchronize(s));
    throw Error(TGFX_EVALIDATION, "query node " + std::to_string(u) + " out of range");
  }
  check_k(k);
}

void check_int32_outputs(const tgfx_graph* g, int64_t self_edge_index) {
  const int64_t lim = INT32_MAX;
  if (std::max(g->V, g->other_limit) >= lim || g->max_eid + 1 > lim || g->min_eid + 1 < INT32_MIN ||
      self_edge_index > lim || self_edge_index < INT32_MIN)
    throw Error(TGFX_EUNSUPPORTED,
                "ids do not fit int32 outputs (use tgfx_sample_assemble_device with TGFX_INDEX64)");
}

tgfx_graph* new_graph(int64_t n, int64_t V, int reverse, cudaStream_t s) {
  if (n < 0) throw Error(TGFX_EVALIDATION, "negative event count");
  if (V < 0) throw Error(TGFX_EVALIDATION, "negative num_nodes");
  const DeviceInfo& di = device_info();
  tgfx_graph* g = new tgfx_graph();
  g->device = di.device;
  g->V = V;
  g->n = n;
  g->reverse = reverse ? 1 : 0;
  g->other_limit = V;
  g->eid_limit = n;
  try {
    graph_alloc(g, s);
  } catch (...) {
    graph_release(g);
    delete g;
    throw;
  }
  g_bytes.fetch_add(static_cast<int64_t>(sizeof(int64_t) * (V + 1) + 24 * g->m));
  return g;
}

bool trace_on() {
  static const bool on = [] {
    const char* e = getenv("TGFX_TRACE");
    return e && e[0] == '1';
  }();
  return on;
}

double now_ms() {
  return std::chrono::duration<double, std::milli>(
             std::chrono::steady_clock::now().time_since_epoch()).count();
}

void free_graph(tgfx_graph* g) {
  if (!g) return;
  const double t0 = now_ms();
  g_bytes.fetch_sub(static_cast<int64_t>(sizeof(int64_t) * (g->V + 1) + 24 * g->m));
  graph_release(g);
  delete g;
  if (trace_on()) fprintf(stderr, "[tgfx] free_graph: %.1f ms\n", now_ms() - t0);
}

int build_host(const tgfx_event* events, int64_t n, int64_t V, int reverse, tgfx_graph** out) {
  tgfx_graph* g = nullptr;
  return guarded([&] {
    if (!out) throw Error(TGFX_EVALIDATION, "null output");
    *out = nullptr;
    cudaStream_t s = 0;
    device_info();
    const double t0 = now_ms();
    DBuf dev(sizeof(tgfx_event) * static_cast<size_t>(std::max<int64_t>(n, 1)), s);
    h2d_big(dev.p, events, sizeof(tgfx_event) * static_cast<size_t>(std::max<int64_t>(n, 0)), s);
    if (trace_on()) TGFX_CUDA(cudaStreamSynchronize(s));
    const double t1 = now_ms();
    g = new_graph(n, V, reverse, s);
    if (trace_on()) TGFX_CUDA(cudaStreamSynchronize(s));
    const double t2 = now_ms();
    try {
      build_graph(g, dev.as<tgfx_event>(), s, false);
      TGFX_CUDA(cudaStreamSynchronize(s));
      if (trace_on())
        fprintf(stderr, "[tgfx] build_host: upload %.1f ms, alloc %.1f ms, build %.1f ms\n",
                t1 - t0, t2 - t1, now_ms() - t2);
    } catch (...) {
      free_graph(g);
      throw;
    }
    *out = g;
  });
}

}  // namespace
}  // namespace tgfx

using namespace tgfx;

extern "C" {

const char* tgfx_last_error(void) { return g_err.c_str(); }
int tgfx_abi_version(void) { return TGFX_ABI_VERSION; }
uint64_t tgfx_launch_count(void) { return g_launches.load(); }
int64_t tgfx_device_bytes(void) { return g_bytes.load(); }

int tgfx_build_sequential(const tgfx_event* events, int64_t n, int64_t num_nodes, int reverse,
                          tgfx_graph** out) {
  return build_host(events, n, num_nodes, reverse, out);
}

int tgfx_build_parallel(const tgfx_event* events, int64_t n, int64_t num_nodes, int reverse,
                        int num_threads, tgfx_graph** out) {
  if (num_threads < 1) {  // tcsr.cpp:108
    g_err = "num_threads must be at least 1";
    if (out) *out = nullptr;
    return TGFX_EVALIDATION;
  }
  return build_host(events, n, num_nodes, reverse, out);
}

int tgfx_build_device(const tgfx_event* d_events, int64_t n, int64_t num_nodes, int reverse,
                      void* stream, unsigned flags, tgfx_graph** out) {
  return guarded([&] {
    if (!out) throw Error(TGFX_EVALIDATION, "null output");
    *out = nullptr;
    cudaStream_t s = as_stream(stream);
    tgfx_graph* g = new_graph(n, num_nodes, reverse, s);
    try {
      build_graph(g, d_events, s, (flags & TGFX_TRUSTED) != 0);
      if (!(flags & TGFX_TRUSTED)) TGFX_CUDA(cudaStreamSynchronize(s));
    } catch (...) {
      free_graph(g);
      throw;
    }
    *out = g;
  });
}

int tgfx_build_range_device(const tgfx_event* d_records, int64_t n, int64_t num_local_nodes,
                            int64_t num_nodes_total, int64_t num_edges_total, void* stream,
                            unsigned flags, tgfx_graph** out) {
  return guarded([&] {
    if (!out) throw Error(TGFX_EVALIDATION, "null output");
    *out = nullptr;
    if (num_nodes_total < num_local_nodes)
      throw Error(TGFX_EVALIDATION, "num_nodes_total < num_local_nodes");
    cudaStream_t s = as_stream(stream);
    tgfx_graph* g = new_graph(n, num_local_nodes, 0, s);
    g->other_limit = num_nodes_total;
    g->eid_limit = num_edges_total;
    try {
      build_graph(g, d_records, s, (flags & TGFX_TRUSTED) != 0);
      if (!(flags & TGFX_TRUSTED)) TGFX_CUDA(cudaStreamSynchronize(s));
    } catch (...) {
      free_graph(g);
      throw;
    }
    *out = g;
  });
}

int tgfx_graph_from_device(int64_t num_nodes, int64_t num_edges, int reverse, int64_t m,
                           const int64_t* d_indptr, const int64_t* d_nbr, const int64_t* d_eid,
                           const double* d_ts, void* stream, unsigned flags, tgfx_graph** out) {
  return guarded([&] {
    if (!out) throw Error(TGFX_EVALIDATION, "null output");
    *out = nullptr;
    if (m != num_edges * (reverse ? 2 : 1))
      throw Error(TGFX_EVALIDATION, "column arrays disagree in length");
    cudaStream_t s = as_stream(stream);
    tgfx_graph* g = new_graph(num_edges, num_nodes, reverse, s);
    try {
      const auto d2d = [&](void* dst, const void* src, size_t bytes) {
        if (bytes) TGFX_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, s));
      };
      d2d(g->indptr, d_indptr, sizeof(int64_t) * (num_nodes + 1));
      d2d(g->nbr, d_nbr, sizeof(int64_t) * m);
      d2d(g->eid, d_eid, sizeof(int64_t) * m);
      d2d(g->ts, d_ts, sizeof(double) * m);
      g->min_eid = 0;
      g->max_eid = num_edges - 1;
      if (flags & TGFX_TRUSTED) {
        g->search_exact = 0;  // caller vouches: slices sorted, NaN-free (e.g. built by tgfx)
      } else {
        g->indptr_bad = indptr_in_range(g->indptr, num_nodes, m, s) ? 0 : 1;
        // interpolation search needs sorted, NaN-free slices; otherwise replay lower_bound
        g->search_exact = (!validate_graph(g, s).empty() || any_nan(g->ts, m, s)) ? 1 : 0;
      }
      if (!g->indptr_bad) build_node_dir(g, s);
      TGFX_CUDA(cudaStreamSynchronize(s));
    } catch (...) {
      free_graph(g);
      throw;
    }
    *out = g;
  });
}

int tgfx_degree_hist_device(const tgfx_event* d_events, int64_t n, int64_t num_nodes, int reverse,
                            uint64_t* d_deg, void* stream) {
  return guarded([&] {
    cudaStream_t s = as_stream(stream);
    if (num_nodes > 0)
      TGFX_CUDA(cudaMemsetAsync(d_deg, 0, sizeof(uint64_t) * num_nodes, s));
    launch_degree_hist(d_events, n, num_nodes, reverse,
                       reinterpret_cast<unsigned long long*>(d_deg), s);
  });
}

int64_t tgfx_partition_warps(int64_t n) {
  try {
    return partition_warps(n);
  } catch (const std::exception& e) {
    fail(e);
    return -1;
  }
}

int tgfx_partition_count_device(const tgfx_event* d_events, int64_t n, int reverse,
                                const int64_t* d_bounds, int nparts, int64_t nwarps,
                                const int64_t* d_split, int64_t* d_counts,
                                int64_t* d_split_counts, void* stream) {
  return guarded([&] {
    if (nparts < 1 || nparts > 8) throw Error(TGFX_EUNSUPPORTED, "1..8 partitions supported");
    launch_partition_count(d_events, n, reverse, d_bounds, nparts, nwarps, d_split, d_counts,
                           d_split_counts, as_stream(stream));
  });
}

int tgfx_partition_scatter_device(const tgfx_event* d_events, int64_t n, int reverse,
                                  const int64_t* d_bounds, int nparts, int64_t nwarps,
                                  const int64_t* d_split, const int64_t* d_split_occ,
                                  const int64_t* d_offsets, tgfx_event* d_records, void* stream) {
  return guarded([&] {
    if (nparts < 1 || nparts > 8) throw Error(TGFX_EUNSUPPORTED, "1..8 partitions supported");
    if (n > 0)
      launch_partition_scatter(d_events, n, reverse, d_bounds, nparts, nwarps, d_split,
                               d_split_occ, d_offsets, d_records, as_stream(stream));
  });
}

int tgfx_rebuild_device(tgfx_graph* g, const tgfx_event* d_events, void* stream, unsigned flags) {
  return guarded([&] {
    check_graph(g);
    cudaStream_t s = as_stream(stream);
    build_graph(g, d_events, s, (flags & TGFX_TRUSTED) != 0);
    if (!(flags & TGFX_TRUSTED)) TGFX_CUDA(cudaStreamSynchronize(s));
  });
}

int tgfx_graph_from_host(int64_t num_nodes, int64_t num_edges, int reverse, int64_t m,
                         const int64_t* indptr, const int64_t* nbr, const int64_t* eid,
                         const double* ts, tgfx_graph** out) {
  return guarded([&] {
    if (!out) throw Error(TGFX_EVALIDATION, "null output");
    *out = nullptr;
    if (m != num_edges * (reverse ? 2 : 1))
      throw Error(TGFX_EVALIDATION, "column arrays disagree in length");
    cudaStream_t s = 0;
    tgfx_graph* g = new_graph(num_edges, num_nodes, reverse, s);
    try {
      h2d(g->indptr, indptr, sizeof(int64_t) * (num_nodes + 1), s);
      h2d(g->nbr, nbr, sizeof(int64_t) * m, s);
      h2d(g->eid, eid, sizeof(int64_t) * m, s);
      h2d(g->ts, ts, sizeof(double) * m, s);
      int64_t mx = -1, mn = 0;
      for (int64_t i = 0; i < m; ++i) {
        mx = i == 0 ? eid[i] : std::max(mx, eid[i]);
        mn = i == 0 ? eid[i] : std::min(mn, eid[i]);
      }
      g->max_eid = mx;
      g->min_eid = mn;
      // interpolation search needs every slice sorted by ts and NaN-free; otherwise the
      // sampler replays std::lower_bound's bisection exactly (sampler.cpp:16-20)
      bool mono = indptr[0] == 0 && indptr[num_nodes] == m;
      for (int64_t u = 0; mono && u < num_nodes; ++u) {
        const int64_t lo = indptr[u], hi = indptr[u + 1];
        if (lo > hi || lo < 0 || hi > m) mono = false;
      }
      bool ok = mono;
      for (int64_t u = 0; ok && u < num_nodes; ++u) {
        const int64_t lo = indptr[u], hi = indptr[u + 1];
        for (int64_t i = lo; ok && i < hi; ++i)
          if (ts[i] != ts[i] || (i > lo && ts[i - 1] > ts[i])) ok = false;
      }
      g->search_exact = ok ? 0 : 1;
      // a corrupt indptr (e.g. a CRC-valid but damaged container) must not reach the node
      // directory kernels, which index ts through it
      g->indptr_bad = mono ? 0 : 1;
      if (mono) build_node_dir(g, s);
      TGFX_CUDA(cudaStreamSynchronize(s));
    } catch (...) {
      free_graph(g);
      throw;
    }
    *out = g;
  });
}

int tgfx_graph_info(const tgfx_graph* g, int64_t* num_nodes, int64_t* num_edges,
                    int64_t* num_entries, int* reverse) {
  return guarded([&] {
    check_graph(g);
    if (num_nodes) *num_nodes = g->V;
    if (num_edges) *num_edges = g->n;
    if (num_entries) *num_entries = g->m;
    if (reverse) *reverse = g->reverse;
  });
}

int tgfx_graph_build_path(const tgfx_graph* g) { return g ? g->path : -1; }

int tgfx_graph_export(const tgfx_graph* g, int64_t* indptr, int64_t* nbr, int64_t* eid,
                      double* ts) {
  return guarded([&] {
    check_graph(g);
    cudaStream_t s = 0;
    ensure_columns(g, s);
    d2h_big(indptr, g->indptr, sizeof(int64_t) * (g->V + 1), s);
    d2h_big(nbr, g->nbr, sizeof(int64_t) * g->m, s);
    d2h_big(eid, g->eid, sizeof(int64_t) * g->m, s);
    d2h_big(ts, g->ts, sizeof(double) * g->m, s);
    TGFX_CUDA(cudaStreamSynchronize(s));
  });
}

int tgfx_graph_device_arrays(const tgfx_graph* g, const int64_t** indptr, const int64_t** nbr,
                             const int64_t** eid, const double** ts) {
  return guarded([&] {
    check_graph(g);
    if (nbr || eid) {
      ensure_columns(g, 0);
      TGFX_CUDA(cudaStreamSynchronize(0));
    }
    if (indptr) *indptr = g->indptr;
    if (nbr) *nbr = g->nbr;
    if (eid) *eid = g->eid;
    if (ts) *ts = g->ts;
  });
}

int tgfx_graph_validate(const tgfx_graph* g) {
  return guarded([&] {
    check_graph(g);
    const std::string msg = validate_graph(g, 0);
    if (!msg.empty()) throw Error(TGFX_EVALIDATION, msg);
  });
}

int tgfx_graph_free(tgfx_graph* g) {
  return guarded([&] { free_graph(g); });
}

namespace {

// tgfx_sample_batch / tgfx_sample_batch_records: padded [q, k] entries as three columns
// (rec == nullptr) or as tgfx_neighbor records, through the calling thread's arena
void sample_entries_host(const tgfx_graph* g, const int64_t* nodes, const double* times,
                         int64_t q, int64_t k, int strategy, uint64_t seed, uint64_t stream_base,
                         int64_t* counts, int64_t* nbr, int64_t* eid, double* ts,
                         tgfx_neighbor* rec) {
  check_graph(g);
  check_queries_host(g, nodes, q, k);
  if (q == 0) return;
  HostCall& hc = host_call();
  const size_t qs = static_cast<size_t>(q), qk = qs * static_cast<size_t>(k);
  // device: [nodes | times] [counts | entries] (each direction back to back)
  const size_t o_t = 8 * qs, o_c = al256(16 * qs), o_e = o_c + 8 * qs;
  Scratch d(hc, o_e + 24 * qk);
  copy_merged({{d.p, nodes, 8 * qs}, {d.p + o_t, times, 8 * qs}}, cudaMemcpyHostToDevice, hc.s);
  int64_t* e = reinterpret_cast<int64_t*>(d.p + o_e);
  SampleArgs a{};
  a.g = g;
  a.nodes = reinterpret_cast<const int64_t*>(d.p);
  a.times = reinterpret_cast<const double*>(d.p + o_t);
  a.q = q;
  a.k = k;
  a.strategy = strategy;
  a.seed = seed;
  a.stream_base = stream_base;
  a.counts = reinterpret_cast<int64_t*>(d.p + o_c);
  if (rec) {  // interleaved: record i = words [3i, 3i + 3)
    a.e_nbr = e;
    a.e_eid = e + 1;
    a.e_ts = reinterpret_cast<double*>(e + 2);
    a.e_stride = 3;
  } else {
    a.e_nbr = e;
    a.e_eid = e + qk;
    a.e_ts = reinterpret_cast<double*>(e + 2 * qk);
  }
  launch_sample(a, hc.s);
  if (rec)
    copy_merged({{counts, a.counts, 8 * qs}, {rec, e, 24 * qk}}, cudaMemcpyDeviceToHost, hc.s);
  else
    copy_merged({{counts, a.counts, 8 * qs}, {nbr, e, 8 * qk}, {eid, e + qk, 8 * qk},
                 {ts, e + 2 * qk, 8 * qk}},
                cudaMemcpyDeviceToHost, hc.s);
  TGFX_CUDA(cudaStreamSynchronize(hc.s));
}

}  // namespace

int tgfx_sample_batch(const tgfx_graph* g, const int64_t* nodes, const double* times, int64_t q,
                      int64_t k, int strategy, uint64_t seed, uint64_t stream_base,
                      int64_t* counts, int64_t* nbr, int64_t* eid, double* ts) {
  return guarded([&] {
    sample_entries_host(g, nodes, times, q, k, strategy, seed, stream_base, counts, nbr, eid, ts,
                        nullptr);
  });
}

int tgfx_sample_batch_records(const tgfx_graph* g, const int64_t* nodes, const double* times,
                              int64_t q, int64_t k, int strategy, uint64_t seed,
                              uint64_t stream_base, int64_t* counts, tgfx_neighbor* entries) {
  return guarded([&] {
    sample_entries_host(g, nodes, times, q, k, strategy, seed, stream_base, counts, nullptr,
                        nullptr, nullptr, entries);
  });
}

int tgfx_host_alloc(size_t bytes, void** p) {
  return guarded([&] {
    if (!p) throw Error(TGFX_EVALIDATION, "null output pointer");
    *p = nullptr;
    device_info();
    TGFX_CUDA(cudaHostAlloc(p, bytes ? bytes : 1, cudaHostAllocPortable));
  });
}

int tgfx_host_free(void* p) {
  return guarded([&] {
    if (p) TGFX_CUDA(cudaFreeHost(p));
  });
}

int tgfx_sample_batch_device(const tgfx_graph* g, const int64_t* d_nodes, const double* d_times,
                             int64_t q, int64_t k, int strategy, uint64_t seed,
                             uint64_t stream_base, int64_t* d_counts, int64_t* d_nbr,
                             int64_t* d_eid, double* d_ts, void* stream, unsigned flags) {
  return guarded([&] {
    check_graph(g);
    cudaStream_t s = as_stream(stream);
    if (!(flags & TGFX_TRUSTED)) check_queries(g, d_nodes, q, k, s);
    check_k(k);
    SampleArgs a{};
    a.g = g;
    a.nodes = d_nodes;
    a.times = d_times;
    a.q = q;
    a.k = k;
    a.strategy = strategy;
    a.seed = seed;
    a.stream_base = stream_base;
    a.counts = d_counts;
    a.e_nbr = d_nbr;
    a.e_eid = d_eid;
    a.e_ts = d_ts;
    launch_sample(a, s);
    if (!(flags & TGFX_TRUSTED)) TGFX_CUDA(cudaStreamSynchronize(s));
  });
}

int tgfx_sample_assemble_device(const tgfx_graph* g, const int64_t* d_nodes,
                                const double* d_times, int64_t q, int64_t k, int strategy,
                                uint64_t seed, uint64_t stream_base, int64_t l,
                                int64_t self_edge_index, void* d_node_index, void* d_edge_index,
                                float* d_dt32, double* d_dt64, void* d_valid_len, void* stream,
                                unsigned flags) {
  return guarded([&] {
    check_graph(g);
    cudaStream_t s = as_stream(stream);
    if (!(flags & TGFX_TRUSTED)) check_queries(g, d_nodes, q, k, s);
    check_k(k);
    check_l(l);
    const bool i64 = (flags & TGFX_INDEX64) != 0;
    if (!i64) check_int32_outputs(g, self_edge_index);
    SampleArgs a{};
    a.g = g;
    a.nodes = d_nodes;
    a.times = d_times;
    a.q = q;
    a.k = k;
    a.strategy = strategy;
    a.seed = seed;
    a.stream_base = stream_base;
    a.l = l;
    a.self_edge_index = self_edge_index;
    a.node_index = d_node_index;
    a.edge_index = d_edge_index;
    a.dt32 = d_dt32;
    a.dt64 = d_dt64;
    a.valid_len = d_valid_len;
    a.index64 = i64;
    launch_sample(a, s);
    if (!(flags & TGFX_TRUSTED)) TGFX_CUDA(cudaStreamSynchronize(s));
  });
}

int tgfx_sample_assemble_checked_device(const tgfx_graph* g, const int64_t* d_nodes,
                                        const double* d_times, int64_t q, int64_t k,
                                        int strategy, uint64_t seed, uint64_t stream_base,
                                        int64_t l, int64_t self_edge_index, void* d_node_index,
                                        void* d_edge_index, float* d_dt32, double* d_dt64,
                                        void* d_valid_len, unsigned long long* d_first_bad,
                                        void* stream, unsigned flags) {
  return guarded([&] {
    check_graph(g);
    if (!d_first_bad) throw Error(TGFX_EVALIDATION, "null first_bad word");
    if (q < 0) throw Error(TGFX_EVALIDATION, "negative query count");
    check_k(k);
    check_l(l);
    const bool i64 = (flags & TGFX_INDEX64) != 0;
    if (!i64) check_int32_outputs(g, self_edge_index);
    SampleArgs a{};
    a.g = g;
    a.nodes = d_nodes;
    a.times = d_times;
    a.q = q;
    a.k = k;
    a.strategy = strategy;
    a.seed = seed;
    a.stream_base = stream_base;
    a.l = l;
    a.self_edge_index = self_edge_index;
    a.node_index = d_node_index;
    a.edge_index = d_edge_index;
    a.dt32 = d_dt32;
    a.dt64 = d_dt64;
    a.valid_len = d_valid_len;
    a.index64 = i64;
    a.first_bad = d_first_bad;
    launch_sample(a, as_stream(stream));
  });
}

int tgfx_query_error(const int64_t* d_nodes, uint64_t stream_base,
                     const unsigned long long* d_first_bad, void* stream) {
  return guarded([&] {
    cudaStream_t s = as_stream(stream);
    unsigned long long h = ~0ull;
    TGFX_CUDA(cudaMemcpyAsync(&h, d_first_bad, sizeof(h), cudaMemcpyDeviceToHost, s));
    TGFX_CUDA(cudaStreamSynchronize(s));
    if (h == ~0ull) return;
    int64_t u = 0;
    TGFX_CUDA(cudaMemcpyAsync(&u, d_nodes + (h - stream_base), sizeof(u), cudaMemcpyDeviceToHost, s));
    TGFX_CUDA(cudaStreamSynchronize(s));
    throw Error(TGFX_EVALIDATION, "query node " + std::to_string(u) + " out of range");
  });
}

namespace {

std::string trimmed(const std::string& x) {
  size_t a = 0, b = x.size();
  while (a < b && (x[a] == ' ' || x[a] == '\t' || x[a] == '\r')) ++a;
  while (b > a && (x[b - 1] == ' ' || x[b - 1] == '\t' || x[b - 1] == '\r')) --b;
  return x.substr(a, b - a);
}

std::vector<std::string> split_commas(const std::string& line) {
  std::vector<std::string> out;
  size_t start = 0;
  while (true) {
    const size_t c = line.find(',', start);
    if (c == std::string::npos) {
      out.push_back(line.substr(start));
      return out;
    }
    out.push_back(line.substr(start, c - start));
    start = c + 1;
  }
}

// The message of the first failing line, rebuilt on the host from that one line's text with
// the reference's own checks (event_stream.cpp:111-131); the device found the line.
[[noreturn]] void throw_csv_line_error(const std::string& raw, int64_t line_no, int code, int d_e) {
  const std::string line = trimmed(raw);
  const std::vector<std::string> f = split_commas(line);
  const std::string at = "line " + std::to_string(line_no) + ": ";
  if (code == kCsvFields)
    throw Error(TGFX_EPARSE, at + "expected " + std::to_string(3 + d_e) + " fields, got " +
                                 std::to_string(f.size()));
  if (code == kCsvNegNode) throw Error(TGFX_EVALIDATION, at + "negative node id");
  if (code == kCsvNegTime) throw Error(TGFX_EVALIDATION, at + "negative timestamp");
  auto bad = [&](int idx, const char* what) -> std::string {
    return at + "bad " + what + " '" + trimmed(f[static_cast<size_t>(idx)]) + "'";
  };
  if (code == kCsvSrc) throw Error(TGFX_EPARSE, bad(0, "src"));
  if (code == kCsvDst) throw Error(TGFX_EPARSE, bad(1, "dst"));
  if (code == kCsvTime) throw Error(TGFX_EPARSE, bad(2, "timestamp"));
  // features: the first field from_chars rejects (or the first the device flagged)
  for (int k = 0; k < d_e; ++k) {
    const std::string v = trimmed(f[static_cast<size_t>(3 + k)]);
    double x = 0.0;
    const auto r = std::from_chars(v.data(), v.data() + v.size(), x);
    if (code == kCsvFeature && (r.ec != std::errc{} || r.ptr != v.data() + v.size()))
      throw Error(TGFX_EPARSE, bad(3 + k, "feature"));
  }
  throw Error(TGFX_EUNSUPPORTED,
              at + "a real with more than 19 significant digits whose rounding needs "
                   "big-integer arithmetic, or a NaN timestamp (not parsed on the device)");
}

}  // namespace

int tgfx_csv_parse_device(const char* d_bytes, int64_t nbytes, int has_features, void* stream,
                          tgfx_csv** out) {
  return guarded([&] {
    if (!out) throw Error(TGFX_EVALIDATION, "null output");
    *out = nullptr;
    if (nbytes < 0) throw Error(TGFX_EVALIDATION, "negative size");
    cudaStream_t s = as_stream(stream);
    device_info();
    // header (event_stream.cpp:90-95): first line, on the host
    std::string header;
    for (int64_t got = 0; got < nbytes;) {
      const int64_t take = std::min<int64_t>(nbytes - got, 1 << 16);
      std::string piece(static_cast<size_t>(take), '\0');
      TGFX_CUDA(cudaMemcpyAsync(&piece[0], d_bytes + got, take, cudaMemcpyDeviceToHost, s));
      TGFX_CUDA(cudaStreamSynchronize(s));
      const size_t nl = piece.find('\n');
      header += piece.substr(0, nl);
      got += take;
      if (nl != std::string::npos) break;
    }
    if (nbytes == 0) throw Error(TGFX_EPARSE, "empty input");
    const size_t hf = split_commas(trimmed(header)).size();
    if (hf < 3) throw Error(TGFX_EPARSE, "line 1: header needs at least src,dst,timestamp");
    const int d_e = has_features ? static_cast<int>(hf - 3) : 0;
    CsvResult r;
    const uint64_t err = parse_csv_device(d_bytes, nbytes, d_e, &r, s);
    if (err != ~0ull) {
      std::string raw(static_cast<size_t>(r.err_line_end - r.err_line_start), '\0');
      if (!raw.empty())
        TGFX_CUDA(cudaMemcpyAsync(&raw[0], d_bytes + r.err_line_start, raw.size(),
                                  cudaMemcpyDeviceToHost, s));
      TGFX_CUDA(cudaStreamSynchronize(s));
      throw_csv_line_error(raw, static_cast<int64_t>(err >> 8), static_cast<int>(err & 0xff), d_e);
    }
    tgfx_csv* c = new tgfx_csv();
    c->n = r.n;
    c->num_nodes = r.num_nodes;
    c->d_e = d_e;
    c->events = r.events;
    c->features = r.features;
    TGFX_CUDA(cudaStreamSynchronize(s));
    *out = c;
  });
}

int tgfx_load_csv(const char* path, int has_features, tgfx_csv** out) {
  return guarded([&] {
    if (!out) throw Error(TGFX_EVALIDATION, "null output");
    *out = nullptr;
    const std::string p = path ? path : "";
    std::ifstream in(p, std::ios::binary | std::ios::ate);
    if (!in) throw Error(TGFX_EVALIDATION, "cannot open '" + p + "'");  // event_stream.cpp:87
    const std::streamsize size = in.tellg();
    in.seekg(0);
    if (size <= 0) throw Error(TGFX_EPARSE, "empty file '" + p + "'");  // :90
    std::vector<char> host(static_cast<size_t>(size));
    in.read(host.data(), size);
    if (!in) throw Error(TGFX_EVALIDATION, "cannot read '" + p + "'");
    cudaStream_t s = 0;
    device_info();
    DBuf dev(static_cast<size_t>(size), s);
    h2d(dev.p, host.data(), static_cast<size_t>(size), s);
    const int rc = tgfx_csv_parse_device(dev.as<char>(), size, has_features, s, out);
    if (rc) throw Error(rc, g_err);
  });
}

int tgfx_csv_info(const tgfx_csv* c, int64_t* num_events, int64_t* num_nodes, int64_t* d_e) {
  return guarded([&] {
    if (!c) throw Error(TGFX_EVALIDATION, "null stream");
    if (num_events) *num_events = c->n;
    if (num_nodes) *num_nodes = c->num_nodes;
    if (d_e) *d_e = c->d_e;
  });
}

int tgfx_csv_device_arrays(const tgfx_csv* c, const tgfx_event** events, const double** features) {
  return guarded([&] {
    if (!c) throw Error(TGFX_EVALIDATION, "null stream");
    if (events) *events = c->events;
    if (features) *features = c->features;
  });
}

int tgfx_csv_export(const tgfx_csv* c, tgfx_event* events, double* features) {
  return guarded([&] {
    if (!c) throw Error(TGFX_EVALIDATION, "null stream");
    cudaStream_t s = 0;
    d2h(events, c->events, sizeof(tgfx_event) * c->n, s);
    if (features && c->d_e > 0) d2h(features, c->features, sizeof(double) * c->n * c->d_e, s);
    TGFX_CUDA(cudaStreamSynchronize(s));
  });
}

int tgfx_csv_free(tgfx_csv* c) {
  return guarded([&] {
    if (!c) return;
    if (c->events) dfree(c->events, 0);
    if (c->features) dfree(c->features, 0);
    delete c;
  });
}

int tgfx_parse_numbers_device(const char* d_bytes, const int64_t* d_off, int64_t n, int kind,
                              int64_t* d_int, double* d_real, int* d_status, void* stream) {
  return guarded([&] {
    if (kind != 0 && kind != 1) throw Error(TGFX_EVALIDATION, "kind must be 0 (int) or 1 (real)");
    cudaStream_t s = as_stream(stream);
    launch_parse_numbers(d_bytes, d_off, n, kind, d_int, d_real, d_status, s);
    TGFX_CUDA(cudaStreamSynchronize(s));
  });
}

int tgfx_assemble_inputs_device(int64_t q, int64_t l, const void* d_node_index,
                                const void* d_edge_index, const void* d_time_delta,
                                const void* d_valid_len, int index64, int dt_type,
                                const void* d_node_table, int64_t node_rows,
                                const void* d_edge_table, int64_t edge_rows, int table_type,
                                const double* d_omega, const double* d_phi, int64_t d_v,
                                int64_t d_e, int64_t d_t, int concat, void* d_z, int z_type,
                                void* stream, unsigned flags) {
  return guarded([&] {
    if (q < 0 || l < 0) throw Error(TGFX_EVALIDATION, "bad batch shape");
    if (d_v < 0 || d_e < 0 || d_t < 0) throw Error(TGFX_EVALIDATION, "bad model dimensions");
    if (!concat && !(d_v == d_t && d_e == d_t))  // ModelConfig::validate, attention.hpp:21-23
      throw Error(TGFX_EVALIDATION, "combine sum requires d_v = d_e = d_t = d_model");
    cudaStream_t s = as_stream(stream);
    AssembleInputsArgs a;
    a.q = q;
    a.l = l;
    a.node_index = d_node_index;
    a.edge_index = d_edge_index;
    a.time_delta = d_time_delta;
    a.valid_len = d_valid_len;
    a.index64 = index64;
    a.dt_type = dt_type;
    a.node_table = d_node_table;
    a.edge_table = d_edge_table;
    a.node_rows = node_rows;
    a.edge_rows = edge_rows;
    a.table_type = table_type;
    a.omega = d_omega;
    a.phi = d_phi;
    a.d_v = d_v;
    a.d_e = d_e;
    a.d_t = d_t;
    a.concat = concat;
    a.z = d_z;
    a.z_type = z_type;
    if (flags & TGFX_TRUSTED) {
      launch_assemble_inputs(a, nullptr, s);
      return;
    }
    DBuf bad(sizeof(int), s);
    TGFX_CUDA(cudaMemsetAsync(bad.p, 0, sizeof(int), s));
    launch_assemble_inputs(a, bad.as<int>(), s);
    int h = 0;
    TGFX_CUDA(cudaMemcpyAsync(&h, bad.p, sizeof(int), cudaMemcpyDeviceToHost, s));
    TGFX_CUDA(cudaStreamSynchronize(s));
    if (h) throw Error(TGFX_EVALIDATION, "sequence index outside embedding tables");
  });
}

int tgfx_sample_inputs_device(const tgfx_graph* g, const int64_t* d_nodes, const double* d_times,
                              int64_t q, int64_t k, int strategy, uint64_t seed,
                              uint64_t stream_base, int64_t l, int64_t self_edge_index,
                              const void* d_node_table, int64_t node_rows,
                              const void* d_edge_table, int64_t edge_rows, int table_type,
                              const double* d_omega, const double* d_phi, int64_t d_v,
                              int64_t d_e, int64_t d_t, int concat, void* d_z, int z_type,
                              int32_t* d_valid_len, void* stream, unsigned flags) {
  return guarded([&] {
    check_graph(g);
    cudaStream_t s = as_stream(stream);
    if (!(flags & TGFX_TRUSTED)) check_queries(g, d_nodes, q, k, s);
    check_k(k);
    check_l(l);
    if (d_v < 0 || d_e < 0 || d_t < 0) throw Error(TGFX_EVALIDATION, "bad model dimensions");
    if (!concat && !(d_v == d_t && d_e == d_t))  // ModelConfig::validate, attention.hpp:21-23
      throw Error(TGFX_EVALIDATION, "combine sum requires d_v = d_e = d_t = d_model");
    SampleInputsArgs a;
    a.s.g = g;
    a.s.nodes = d_nodes;
    a.s.times = d_times;
    a.s.q = q;
    a.s.k = k;
    a.s.strategy = strategy;
    a.s.seed = seed;
    a.s.stream_base = stream_base;
    a.s.l = l;
    a.s.self_edge_index = self_edge_index;
    a.s.valid_len = d_valid_len;
    a.in.q = q;
    a.in.l = l;
    a.in.node_table = d_node_table;
    a.in.edge_table = d_edge_table;
    a.in.node_rows = node_rows;
    a.in.edge_rows = edge_rows;
    a.in.table_type = table_type;
    a.in.omega = d_omega;
    a.in.phi = d_phi;
    a.in.d_v = d_v;
    a.in.d_e = d_e;
    a.in.d_t = d_t;
    a.in.concat = concat;
    a.in.z = d_z;
    a.in.z_type = z_type;
    DBuf bad(sizeof(int), s);
    TGFX_CUDA(cudaMemsetAsync(bad.p, 0, sizeof(int), s));
    if (!launch_sample_inputs(a, bad.as<int>(), s)) {
      // uniform-k or an exact-search graph: the composition, through device row buffers
      check_int32_outputs(g, self_edge_index);
      const size_t ql = static_cast<size_t>(std::max<int64_t>(q, 1)) * static_cast<size_t>(l);
      DBuf ni(sizeof(int32_t) * ql, s), ei(sizeof(int32_t) * ql, s), dt(sizeof(double) * ql, s);
      DBuf vl(sizeof(int32_t) * static_cast<size_t>(std::max<int64_t>(q, 1)), s);
      SampleArgs sa = a.s;
      sa.node_index = ni.p;
      sa.edge_index = ei.p;
      sa.dt64 = dt.as<double>();
      sa.valid_len = d_valid_len ? static_cast<void*>(d_valid_len) : vl.p;
      sa.index64 = false;
      launch_sample(sa, s);
      AssembleInputsArgs ia = a.in;
      ia.node_index = ni.p;
      ia.edge_index = ei.p;
      ia.time_delta = dt.p;
      ia.valid_len = sa.valid_len;
      ia.index64 = 0;
      ia.dt_type = TGFX_F64;
      launch_assemble_inputs(ia, bad.as<int>(), s);
      TGFX_CUDA(cudaStreamSynchronize(s));  // the row buffers are released below
    }
    if (!(flags & TGFX_TRUSTED)) {
      int h = 0;
      TGFX_CUDA(cudaMemcpyAsync(&h, bad.p, sizeof(int), cudaMemcpyDeviceToHost, s));
      TGFX_CUDA(cudaStreamSynchronize(s));
      if (h) throw Error(TGFX_EVALIDATION, "sequence index outside embedding tables");
    }
  });
}

int tgfx_sample_assemble_batched_device(const tgfx_graph* g, const int64_t* d_nodes,
                                        const double* d_times, int64_t q, int64_t batch_q,
                                        int64_t k, int strategy, const uint64_t* d_seeds,
                                        int64_t l, int64_t self_edge_index, void* d_node_index,
                                        void* d_edge_index, float* d_dt32, double* d_dt64,
                                        void* d_valid_len, void* stream, unsigned flags) {
  return guarded([&] {
    check_graph(g);
    if (batch_q < 1) throw Error(TGFX_EVALIDATION, "batch size must be at least 1");
    if (strategy == TGFX_RANDOM && !d_seeds && q > 0)
      throw Error(TGFX_EVALIDATION, "per-batch seeds required for uniform sampling");
    cudaStream_t s = as_stream(stream);
    if (!(flags & TGFX_TRUSTED)) check_queries(g, d_nodes, q, k, s);
    check_k(k);
    check_l(l);
    const bool i64 = (flags & TGFX_INDEX64) != 0;
    if (!i64) check_int32_outputs(g, self_edge_index);
    SampleArgs a{};
    a.g = g;
    a.nodes = d_nodes;
    a.times = d_times;
    a.q = q;
    a.k = k;
    a.strategy = strategy;
    a.seed = 0;
    a.stream_base = 0;
    a.l = l;
    a.self_edge_index = self_edge_index;
    a.node_index = d_node_index;
    a.edge_index = d_edge_index;
    a.dt32 = d_dt32;
    a.dt64 = d_dt64;
    a.valid_len = d_valid_len;
    a.index64 = i64;
    a.seeds = d_seeds;
    a.batch_q = batch_q;
    launch_sample(a, s);
    if (!(flags & TGFX_TRUSTED)) TGFX_CUDA(cudaStreamSynchronize(s));
  });
}

// Host-buffer sample_assemble, pipelined: the output rows (136 B/query at l = 11) dwarf the
// inputs (16 B/query), so the call is bound by its device->host copies, and the copy engine
// should start early and never idle.  The queries are processed in sub-chunks on the calling
// thread's two lanes (stream + device buffers, kept across calls): a sub-chunk's node and
// time upload, its kernel, and the previous sub-chunk's row download overlap on the copy
// engines.  sampler.cpp:88-93 validates every query before anything is sampled and nothing
// is returned on failure: here host threads scan the node ids while the first two sub-chunks
// already sample into device buffers (a bad node is an absent query to the kernels, so that
// is safe), and no row reaches the caller's buffers before the scan has passed.
namespace {

struct AsmLanes {
  static constexpr int kN = 2;
  cudaStream_t st[kN] = {nullptr, nullptr};
  char* buf[kN] = {nullptr, nullptr};
  size_t cap[kN] = {0, 0};
  cudaEvent_t after_legacy = nullptr;  // orders the lanes after the legacy default stream
  int dev = -1;
};

AsmLanes& asm_lanes() {
  thread_local AsmLanes L;
  const int dev = device_info().device;
  if (L.dev != dev) {
    L = AsmLanes{};
    for (cudaStream_t& st : L.st) TGFX_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    TGFX_CUDA(cudaEventCreateWithFlags(&L.after_legacy, cudaEventDisableTiming));
    L.dev = dev;
  }
  return L;
}

int64_t asm_sub_queries() {
  static const int64_t v = [] {
    const char* e = getenv("TGFX_ASM_SUB");  // A/B: queries per sub-chunk
    return e ? std::max<int64_t>(1, atoll(e)) : int64_t(4) << 20;
  }();
  return v;
}

// index of the first node outside [0, V) in nodes[0, q), or -1; threads over ranges for big q
int64_t first_bad_node_host(const int64_t* nodes, int64_t q, int64_t V) {
  auto scan = [&](int64_t a, int64_t b) -> int64_t {
    for (int64_t i = a; i < b; ++i)
      if (static_cast<uint64_t>(nodes[i]) >= static_cast<uint64_t>(V)) return i;
    return -1;
  };
  // half the host's threads at most, so the calling thread, which issues the first sub-chunks'
  // copies meanwhile, keeps a core (per-call times on a 16-thread host were within noise of
  // 16 scanners: 64.9-67.7 against 65.7 ms)
  const int T = q >= (int64_t(1) << 20)
                    ? static_cast<int>(std::min<unsigned>(
                          8, std::max(1u, std::thread::hardware_concurrency() / 2)))
                    : 1;
  if (T == 1) return scan(0, q);
  std::vector<int64_t> first(static_cast<size_t>(T), -1);
  std::vector<std::thread> th;
  th.reserve(static_cast<size_t>(T));
  int started = 0;
  try {  // the ranges no thread could be started for are scanned here
    for (; started < T; ++started)
      th.emplace_back([&, started] {
        first[static_cast<size_t>(started)] = scan(q * started / T, q * (started + 1) / T);
      });
  } catch (...) {
  }
  for (int t = started; t < T; ++t) first[static_cast<size_t>(t)] = scan(q * t / T, q * (t + 1) / T);
  for (std::thread& x : th) x.join();
  for (int64_t f : first)
    if (f >= 0) return f;
  return -1;
}

}  // namespace

int tgfx_sample_assemble(const tgfx_graph* g, const int64_t* nodes, const double* times,
                         int64_t q, int64_t k, int strategy, uint64_t seed, uint64_t stream_base,
                         int64_t l, int64_t self_edge_index, int32_t* node_index,
                         int32_t* edge_index, float* dt32, double* dt64, int32_t* valid_len) {
  return guarded([&] {
    check_graph(g);
    // query 0's node, then k (checked with query 0), then the others (sampler.cpp:88-93)
    if (q < 0) throw Error(TGFX_EVALIDATION, "negative query count");
    if (q > 0 && (nodes[0] < 0 || nodes[0] >= g->V))
      throw Error(TGFX_EVALIDATION, "query node " + std::to_string(nodes[0]) + " out of range");
    if (q > 0) check_k(k);
    check_l(l);
    check_int32_outputs(g, self_edge_index);
    if (q == 0) return;
    AsmLanes& L = asm_lanes();
    const int64_t sub = std::min<int64_t>(q, asm_sub_queries());
    const size_t sl = static_cast<size_t>(sub) * static_cast<size_t>(l);
    // lane layout: [nodes | times] [node_index | edge_index | dt32 | dt64 | valid_len]
    const size_t o_t = 8 * static_cast<size_t>(sub), o_n = al256(16 * static_cast<size_t>(sub)),
                 o_e = o_n + al256(4 * sl), o_f = o_e + al256(4 * sl),
                 o_d = o_f + (dt32 ? al256(4 * sl) : 0), o_v = o_d + (dt64 ? al256(8 * sl) : 0),
                 need = o_v + 4 * static_cast<size_t>(sub);
    for (int i = 0; i < AsmLanes::kN; ++i)
      if (L.cap[i] < need) {
        if (L.buf[i]) {
          TGFX_CUDA(cudaStreamSynchronize(L.st[i]));
          TGFX_CUDA(cudaFree(L.buf[i]));
          L.buf[i] = nullptr;
          L.cap[i] = 0;
        }
        TGFX_CUDA(cudaMalloc(&L.buf[i], need));
        L.cap[i] = need;
      }
    // like every host-buffer call, after the work already queued on the legacy default stream
    TGFX_CUDA(cudaEventRecord(L.after_legacy, 0));
    for (cudaStream_t st : L.st) TGFX_CUDA(cudaStreamWaitEvent(st, L.after_legacy, 0));
    // the scan of nodes[1, q) runs on host threads beside the first sub-chunks
    int64_t bad = -1;
    std::thread checker;
    auto check_rest = [&] {
      const int64_t f = first_bad_node_host(nodes + 1, q - 1, g->V);
      bad = f < 0 ? -1 : f + 1;
    };
    if (q > 1) {
      try {
        checker = std::thread(check_rest);
      } catch (...) {  // no thread: check before sampling instead of beside it
        check_rest();
      }
    }
    auto join = [&] {
      if (checker.joinable()) checker.join();
    };
    // sub-chunk i covers queries [c0(i), c0(i + 1)): the first is small (1/8 of the others) so
    // the first row download starts after a short upload and kernel, then full sub-chunks
    const int64_t head = std::max<int64_t>(1, sub / 8);
    const int64_t nsub = q <= head ? 1 : 1 + ceil_div(q - head, sub);
    auto c0_of = [&](int64_t i) { return i == 0 ? int64_t(0) : std::min(q, head + (i - 1) * sub); };
    auto c1_of = [&](int64_t i) { return i + 1 >= nsub ? q : c0_of(i + 1); };
    auto compute = [&](int64_t i) {  // upload + sampling of sub-chunk i on its lane
      const int ln = static_cast<int>(i % AsmLanes::kN);
      char* d = L.buf[ln];
      const int64_t c0 = c0_of(i), c = c1_of(i) - c0;
      h2d(d, nodes + c0, 8 * static_cast<size_t>(c), L.st[ln]);
      h2d(d + o_t, times + c0, 8 * static_cast<size_t>(c), L.st[ln]);
      SampleArgs a{};
      a.g = g;
      a.nodes = reinterpret_cast<const int64_t*>(d);
      a.times = reinterpret_cast<const double*>(d + o_t);
      a.q = c;
      a.k = k;
      a.strategy = strategy;
      a.seed = seed;
      a.stream_base = stream_base + static_cast<uint64_t>(c0);
      a.l = l;
      a.self_edge_index = self_edge_index;
      a.node_index = d + o_n;
      a.edge_index = d + o_e;
      a.dt32 = dt32 ? reinterpret_cast<float*>(d + o_f) : nullptr;
      a.dt64 = dt64 ? reinterpret_cast<double*>(d + o_d) : nullptr;
      a.valid_len = d + o_v;
      launch_sample(a, L.st[ln]);
    };
    auto copy_out = [&](int64_t i) {  // rows of sub-chunk i to the caller's buffers
      const int ln = static_cast<int>(i % AsmLanes::kN);
      const char* d = L.buf[ln];
      const int64_t c0 = c0_of(i), c = c1_of(i) - c0;
      const size_t cl = static_cast<size_t>(c) * static_cast<size_t>(l);
      const size_t r0 = static_cast<size_t>(c0) * static_cast<size_t>(l);
      d2h(node_index + r0, d + o_n, 4 * cl, L.st[ln]);
      d2h(edge_index + r0, d + o_e, 4 * cl, L.st[ln]);
      if (dt32) d2h(dt32 + r0, d + o_f, 4 * cl, L.st[ln]);
      if (dt64) d2h(dt64 + r0, d + o_d, 8 * cl, L.st[ln]);
      d2h(valid_len + c0, d + o_v, 4 * static_cast<size_t>(c), L.st[ln]);
    };
    try {
      const int64_t pre = std::min<int64_t>(nsub, AsmLanes::kN);
      for (int64_t i = 0; i < pre; ++i) compute(i);
      join();
      if (bad >= 0) {
        for (cudaStream_t st : L.st) cudaStreamSynchronize(st);
        throw Error(TGFX_EVALIDATION,
                    "query node " + std::to_string(nodes[bad]) + " out of range");
      }
      for (int64_t i = 0; i < nsub; ++i) {
        if (i >= pre) compute(i);
        copy_out(i);
      }
      for (cudaStream_t st : L.st) TGFX_CUDA(cudaStreamSynchronize(st));
    } catch (...) {
      join();
      for (cudaStream_t st : L.st) cudaStreamSynchronize(st);
      throw;
    }
  });
}

int tgfx_sample_sequence_batch(const tgfx_graph* g, const int64_t* nodes, const double* times,
                               int64_t q, int64_t k, int strategy, uint64_t seed,
                               uint64_t stream_base, int64_t l, int64_t self_edge_index,
                               int64_t* node_index, int64_t* edge_index, double* time_delta,
                               int64_t* valid_len, int64_t* target_row) {
  return guarded([&] {
    check_graph(g);
    check_queries_host(g, nodes, q, k);  // sampler.cpp:88-93 (k only if q > 0)
    check_l(l);                          // sequence.cpp:57, after sampling's checks
    if (q <= 0) return;
    HostCall& hc = host_call();
    const size_t qs = static_cast<size_t>(q), ql = qs * static_cast<size_t>(l);
    // device: [nodes | times] [node_index | edge_index | time_delta | valid_len]
    const size_t o_t = 8 * qs, o_n = al256(16 * qs), o_e = o_n + 8 * ql, o_d = o_e + 8 * ql,
                 o_v = o_d + 8 * ql;
    Scratch d(hc, o_v + 8 * qs);
    copy_merged({{d.p, nodes, 8 * qs}, {d.p + o_t, times, 8 * qs}}, cudaMemcpyHostToDevice, hc.s);
    SampleArgs a{};
    a.g = g;
    a.nodes = reinterpret_cast<const int64_t*>(d.p);
    a.times = reinterpret_cast<const double*>(d.p + o_t);
    a.q = q;
    a.k = k;
    a.strategy = strategy;
    a.seed = seed;
    a.stream_base = stream_base;
    a.l = l;
    a.self_edge_index = self_edge_index;
    a.node_index = d.p + o_n;
    a.edge_index = d.p + o_e;
    a.dt32 = nullptr;
    a.dt64 = reinterpret_cast<double*>(d.p + o_d);
    a.valid_len = d.p + o_v;
    a.index64 = true;
    launch_sample(a, hc.s);
    copy_merged({{node_index, d.p + o_n, 8 * ql}, {edge_index, d.p + o_e, 8 * ql},
                 {time_delta, d.p + o_d, 8 * ql}, {valid_len, d.p + o_v, 8 * qs}},
                cudaMemcpyDeviceToHost, hc.s);
    TGFX_CUDA(cudaStreamSynchronize(hc.s));
    if (target_row)
      for (int64_t b = 0; b < q; ++b) target_row[b] = valid_len[b] - 1;  // sequence.cpp:83
  });
}

int tgfx_sample_two_hop_device(const tgfx_graph* g, const int64_t* d_roots, const double* d_times,
                               int64_t q, int64_t k1, int64_t k2, int strategy, uint64_t seed,
                               uint64_t seed2, int64_t l, int64_t self_edge_index,
                               int32_t* d_hop1_node, int32_t* d_hop1_edge, float* d_hop1_dt,
                               int32_t* d_hop1_len, int32_t* d_hop2_node, int32_t* d_hop2_edge,
                               float* d_hop2_dt, int32_t* d_hop2_len, void* stream,
                               unsigned flags) {
  return guarded([&] {
    check_graph(g);
    cudaStream_t s = as_stream(stream);
    if (!(flags & TGFX_TRUSTED)) check_queries(g, d_roots, q, k1, s);
    check_k(k1);
    check_k(k2);
    check_l(l);
    check_int32_outputs(g, self_edge_index);
    launch_two_hop(g, d_roots, d_times, q, k1, k2, strategy, seed, seed2, l, self_edge_index,
                   d_hop1_node, d_hop1_edge, d_hop1_dt, d_hop1_len, d_hop2_node, d_hop2_edge,
                   d_hop2_dt, d_hop2_len, s);
    if (!(flags & TGFX_TRUSTED)) TGFX_CUDA(cudaStreamSynchronize(s));
  });
}

int tgfx_sample_two_hop(const tgfx_graph* g, const int64_t* roots, const double* times, int64_t q,
                        int64_t k1, int64_t k2, int strategy, uint64_t seed, uint64_t seed2,
                        int64_t l, int64_t self_edge_index, int32_t* hop1_node,
                        int32_t* hop1_edge, float* hop1_dt, int32_t* hop1_len,
                        int32_t* hop2_node, int32_t* hop2_edge, float* hop2_dt,
                        int32_t* hop2_len) {
  return guarded([&] {
    check_graph(g);
    cudaStream_t s = 0;
    const size_t qb = static_cast<size_t>(std::max<int64_t>(q, 1));
    DBuf dn(sizeof(int64_t) * qb, s), dt(sizeof(double) * qb, s);
    h2d(dn.p, roots, sizeof(int64_t) * std::max<int64_t>(q, 0), s);
    h2d(dt.p, times, sizeof(double) * std::max<int64_t>(q, 0), s);
    check_queries(g, dn.as<int64_t>(), q, k1, s);
    check_k(k2);
    check_l(l);
    check_int32_outputs(g, self_edge_index);
    if (q == 0) return;
    const size_t n1 = qb * l, n2 = qb * k1 * l, c2 = qb * k1;
    DBuf a(4 * n1, s), b(4 * n1, s), c(4 * n1, s), d(4 * qb, s);
    DBuf e(4 * n2, s), f(4 * n2, s), h(4 * n2, s), i(4 * c2, s);
    launch_two_hop(g, dn.as<int64_t>(), dt.as<double>(), q, k1, k2, strategy, seed, seed2, l,
                   self_edge_index, a.as<int32_t>(), b.as<int32_t>(), c.as<float>(),
                   d.as<int32_t>(), e.as<int32_t>(), f.as<int32_t>(), h.as<float>(),
                   i.as<int32_t>(), s);
    d2h(hop1_node, a.p, 4 * q * l, s);
    d2h(hop1_edge, b.p, 4 * q * l, s);
    d2h(hop1_dt, c.p, 4 * q * l, s);
    d2h(hop1_len, d.p, 4 * q, s);
    d2h(hop2_node, e.p, 4 * q * k1 * l, s);
    d2h(hop2_edge, f.p, 4 * q * k1 * l, s);
    d2h(hop2_dt, h.p, 4 * q * k1 * l, s);
    d2h(hop2_len, i.p, 4 * q * k1, s);
    TGFX_CUDA(cudaStreamSynchronize(s));
  });
}

namespace {

// build_sequence_batch (sequence.cpp:55-86) over padded host samples: columns (rec ==
// nullptr) or tgfx_neighbor records, through the calling thread's arena
void assemble_host(int64_t q, int64_t kpad, const int64_t* counts, const int64_t* nbr,
                   const int64_t* eid, const double* ts, const tgfx_neighbor* rec,
                   const int64_t* query_nodes, const double* query_times, int64_t l,
                   int64_t self_edge_index, int64_t* node_index, int64_t* edge_index,
                   double* time_delta, int64_t* valid_len, int64_t* target_row) {
  check_l(l);
  if (q < 0 || kpad < 0) throw Error(TGFX_EVALIDATION, "bad batch shape");
  for (int64_t b = 0; b < q; ++b)
    if (counts[b] < 0 || counts[b] > kpad) throw Error(TGFX_EVALIDATION, "bad sample count");
  if (q == 0) return;
  HostCall& hc = host_call();
  const size_t qs = static_cast<size_t>(q), qk = qs * static_cast<size_t>(kpad),
               ql = qs * static_cast<size_t>(l);
  // device: [counts | entries (records, or nbr | eid | ts) | query nodes | query times]
  //         [node_index | edge_index | time_delta | valid_len | target_row]
  const size_t o_n = 8 * qs, o_qn = o_n + 24 * qk, o_qt = o_qn + 8 * qs,
               o_on = al256(o_qt + 8 * qs), o_oe = o_on + 8 * ql, o_od = o_oe + 8 * ql,
               o_ov = o_od + 8 * ql, o_or = o_ov + 8 * qs;
  Scratch d(hc, o_or + 8 * qs);
  auto at = [&](size_t o) { return reinterpret_cast<int64_t*>(d.p + o); };
  const int64_t *dn = at(o_n), *de, *dtp;
  int64_t es = 1;
  if (rec) {  // records [q, kpad]; the three fields at word offsets 0, 1, 2
    copy_merged({{d.p, counts, 8 * qs}, {d.p + o_n, rec, 24 * qk},
                 {d.p + o_qn, query_nodes, 8 * qs}, {d.p + o_qt, query_times, 8 * qs}},
                cudaMemcpyHostToDevice, hc.s);
    de = dn + 1;
    dtp = dn + 2;
    es = 3;
  } else {
    copy_merged({{d.p, counts, 8 * qs}, {d.p + o_n, nbr, 8 * qk},
                 {d.p + o_n + 8 * qk, eid, 8 * qk}, {d.p + o_n + 16 * qk, ts, 8 * qk},
                 {d.p + o_qn, query_nodes, 8 * qs}, {d.p + o_qt, query_times, 8 * qs}},
                cudaMemcpyHostToDevice, hc.s);
    de = dn + qk;
    dtp = dn + 2 * qk;
  }
  launch_assemble_entries(q, kpad, at(0), dn, de, reinterpret_cast<const double*>(dtp),
                          at(o_qn), reinterpret_cast<const double*>(at(o_qt)), l,
                          self_edge_index, at(o_on), at(o_oe),
                          reinterpret_cast<double*>(at(o_od)), at(o_ov), at(o_or), hc.s, es);
  copy_merged({{node_index, d.p + o_on, 8 * ql}, {edge_index, d.p + o_oe, 8 * ql},
               {time_delta, d.p + o_od, 8 * ql}, {valid_len, d.p + o_ov, 8 * qs},
               {target_row, d.p + o_or, 8 * qs}},
              cudaMemcpyDeviceToHost, hc.s);
  TGFX_CUDA(cudaStreamSynchronize(hc.s));
}

}  // namespace

int tgfx_assemble(int64_t q, int64_t kpad, const int64_t* counts, const int64_t* nbr,
                  const int64_t* eid, const double* ts, const int64_t* query_nodes,
                  const double* query_times, int64_t l, int64_t self_edge_index,
                  int64_t* node_index, int64_t* edge_index, double* time_delta,
                  int64_t* valid_len, int64_t* target_row) {
  return guarded([&] {
    assemble_host(q, kpad, counts, nbr, eid, ts, nullptr, query_nodes, query_times, l,
                  self_edge_index, node_index, edge_index, time_delta, valid_len, target_row);
  });
}

int tgfx_assemble_records(int64_t q, int64_t kpad, const int64_t* counts,
                          const tgfx_neighbor* entries, const int64_t* query_nodes,
                          const double* query_times, int64_t l, int64_t self_edge_index,
                          int64_t* node_index, int64_t* edge_index, double* time_delta,
                          int64_t* valid_len, int64_t* target_row) {
  return guarded([&] {
    assemble_host(q, kpad, counts, nullptr, nullptr, nullptr, entries, query_nodes, query_times,
                  l, self_edge_index, node_index, edge_index, time_delta, valid_len, target_row);
  });
}

int tgfx_build_mask(int64_t q, int64_t l, const int64_t* valid_len, const int64_t* target_row,
                    int kind, double* mask) {
  return guarded([&] {
    if (kind < 0 || kind > 2) throw Error(TGFX_EVALIDATION, "unknown mask kind");
    if (q <= 0 || l <= 0) return;
    device_info();
    cudaStream_t s = 0;
    const size_t qb = static_cast<size_t>(q);
    DBuf vl(8 * qb, s), tr(8 * qb, s), m(8 * qb * l * l, s);
    h2d(vl.p, valid_len, 8 * qb, s);
    h2d(tr.p, target_row, 8 * qb, s);
    launch_mask(q, l, vl.as<int64_t>(), tr.as<int64_t>(), kind, m.as<double>(), s);
    d2h(mask, m.p, 8 * qb * l * l, s);
    TGFX_CUDA(cudaStreamSynchronize(s));
  });
}

int tgfx_make_random_stream(int64_t num_edges, int64_t num_nodes, uint64_t seed,
                            double zipf_exponent, tgfx_event* out) {
  return guarded([&] {
    if (num_edges < 0 || num_nodes < 1) throw Error(TGFX_EVALIDATION, "bad stream dimensions");
    if (num_edges == 0) return;
    device_info();
    cudaStream_t s = 0;
    DBuf d(sizeof(tgfx_event) * num_edges, s);
    launch_random_stream(num_edges, num_nodes, seed, zipf_exponent, d.as<tgfx_event>(), s);
    d2h(out, d.p, sizeof(tgfx_event) * num_edges, s);
    TGFX_CUDA(cudaStreamSynchronize(s));
  });
}

int tgfx_make_random_stream_device(int64_t num_edges, int64_t num_nodes, uint64_t seed,
                                   double zipf_exponent, tgfx_event* d_out, void* stream) {
  return guarded([&] {
    device_info();
    launch_random_stream(num_edges, num_nodes, seed, zipf_exponent, d_out, as_stream(stream));
  });
}

int tgfx_make_queries_device(const tgfx_event* d_events, int64_t e0, int64_t e1, int64_t batch,
                             int64_t num_nodes, uint64_t neg_seed, int64_t* d_nodes,
                             double* d_times, void* stream) {
  return guarded([&] {
    device_info();
    launch_make_queries(d_events, e0, e1, batch, num_nodes, neg_seed, d_nodes, d_times,
                        as_stream(stream));
  });
}

int tgfx_make_train_queries_device(const tgfx_event* d_events, int64_t n, int64_t b0, int64_t b1,
                                   int64_t batch_size, int64_t neg_per_pos, int64_t workers,
                                   int64_t num_nodes, uint64_t batch_seed, int64_t* d_nodes,
                                   double* d_times, void* stream) {
  return guarded([&] {
    device_info();
    launch_train_queries(d_events, n, b0, b1, batch_size, neg_per_pos, workers, num_nodes,
                         batch_seed, d_nodes, d_times, as_stream(stream));
  });
}

uint64_t tgfx_mix_streams(uint64_t a, uint64_t b, uint64_t c) {
  // training.cpp:16-18
  return mix64(mix64(a ^ 0x8f1bbcdcbfa53e0bULL) ^ mix64(b) ^ (c * 0x2545f4914f6cdd1dULL));
}

}  // extern "C"
