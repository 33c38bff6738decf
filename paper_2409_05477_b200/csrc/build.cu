// build.cu -- T-CSR builder for sm_100a.
//
// Replaces the reference's count -> scan -> atomic scatter -> per-slice sort pipeline
// (proj/src/tcsr.cpp:83-151, finish :26-42) with a sort-free stable counting build:
//
//   If the event stream is (t, eid)-non-decreasing -- true of every stream load_csv,
//   make_random_stream and chronological_split produce, and CHECKED here, not assumed --
//   then the reference's per-slice (t, eid) order equals emission order (event-major, src
//   entry before dst entry, tcsr.cpp:99-102).  So entry j lands at
//       indptr[u] + #{ j' < j : node(j') = u }
//   and the build is a stable counting sort by node:
//
//   K1 k_hist      one pass over the events (32 B each, 16-byte vector loads): endpoint
//                  validation (first bad stream index), (t, eid)-order and NaN check, eid
//                  range, and a per-chunk node histogram in shared memory.
//   K2 k_colsum / k_coldflags / k_indptr_scan / k_coloff
//                  degrees, indptr (int64, V+1), cold-node bitmask (nodes with few entries
//                  per chunk) and dense cold-index bases, and every chunk's starting cursor
//                  per node (a C x V table, C = resident CTAs; ~20 MB for GDELT-shaped V).
//   K3 k_scatter_big  one more pass: each CTA streams its chunk through shared memory in
//                  bulk-copied 512-event tiles and ranks every tile by node with a block-wide
//                  stable radix sort (4 keys per thread), so each node's tile entries are one
//                  run written at cursor[u] + offset (details at the kernel).  Cold nodes'
//                  entries go out as full 32-byte records, placed by K4 k_cold_u.
//                  (k_scatter_tile, 256-event tiles with 2 keys per thread, and k_scatter, the
//                  earlier ticketed-warp kernel, remain as A/B variants and for node counts
//                  whose cursors do not fit.)
//
//   Algorithmic bytes: 32 B/event read (K3; K1 reads them once more) + 24 B/entry written
//   + 8(V+1).
//
// Unsorted streams take the general path: a stable LSD radix sort of the events by
// (t, eid) (-0.0 keyed as +0.0, payload bits kept), then the fast path.  Streams whose
// num_nodes exceed the shared-memory cursor budget take the large-V path: global
// degree histogram + scan, and a stable LSD radix sort of (node, emission index).
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <vector>

#include "graph.cuh"
#include "primitives.cuh"

namespace tgfx {
namespace {

constexpr int kHistThreads = 512;

constexpr int64_t kFastMaxNodes = 45000;

__global__ void k_init_flags(BuildFlags* f) {
  f->bad_index = ~0ull;
  f->unsorted = 0;
  f->has_nan = 0;
  f->max_eid = LLONG_MIN;
  f->min_eid = LLONG_MAX;
}

// K1: validation + order check + per-chunk node histogram (HIST) -------------------------
template <int R, bool HIST>
__global__ void __launch_bounds__(kHistThreads) k_hist(const tgfx_event* __restrict__ ev,
                                                       int64_t n, int64_t V, int64_t Vd,
                                                       int64_t chunk_ev,
                                                       uint32_t* __restrict__ cnt,
                                                       BuildFlags* flags) {
  extern __shared__ uint32_t hist[];
  if (HIST) {
    for (int i = threadIdx.x; i < V; i += kHistThreads) hist[i] = 0;
    __syncthreads();
  }
  const int lane = threadIdx.x & 31;
  const int64_t e0 = static_cast<int64_t>(blockIdx.x) * chunk_ev;
  const int64_t e1 = min(n, e0 + chunk_ev);
  bool unsorted = false, nan = false;
  unsigned long long bad = ~0ull;
  long long mx = LLONG_MIN, mn = LLONG_MAX;
  constexpr int U = 4;  // events per thread in flight
  for (int64_t b = e0; b < e1; b += U * kHistThreads) {
    Ev xs[U];
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const int64_t e = b + k * kHistThreads + threadIdx.x;
      xs[k] = e < e1 ? load_event(ev, e) : Ev{0, 0, 0, 0.0};
    }
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const int64_t e = b + k * kHistThreads + threadIdx.x;
      const bool valid = e < e1;
      const Ev x = xs[k];
      // (t, eid) order against event e+1: from the next lane, else a direct load
      double tn = __shfl_down_sync(kFull, x.t, 1);
      long long en = __shfl_down_sync(kFull, (long long)x.eid, 1);
      if (valid && e + 1 < n && (lane == 31 || e + 1 >= e1)) {
        const Ev y = load_event(ev, e + 1);
        tn = y.t;
        en = y.eid;
      }
      if (valid && e + 1 < n) {
        const bool ok = (x.t < tn) || (x.t == tn && x.eid <= en);  // NaN -> not ok
        unsorted |= !ok;
      }
      const bool ok_s = valid && x.src >= 0 && x.src < V;
      const bool ok_d = valid && x.dst >= 0 && x.dst < Vd;  // Vd = V unless a range build
      if (valid && !(ok_s && ok_d)) bad = min(bad, (unsigned long long)e);
      if (valid) {
        nan |= x.t != x.t;
        mx = max(mx, (long long)x.eid);
        mn = min(mn, (long long)x.eid);
      }
      if (HIST) {
        const bool ok = ok_s && ok_d;  // events with a bad endpoint are not counted
        if (ok) {
          atomicAdd(&hist[static_cast<unsigned>(x.src)], 1u);
          if (R == 2) atomicAdd(&hist[static_cast<unsigned>(x.dst)], 1u);
        }
      }
    }
  }
  // flags: warp reduce then one atomic per warp
  unsorted = __any_sync(kFull, unsorted);
  nan = __any_sync(kFull, nan);
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    bad = min(bad, __shfl_xor_sync(kFull, bad, o));
    mx = max(mx, __shfl_xor_sync(kFull, mx, o));
    mn = min(mn, __shfl_xor_sync(kFull, mn, o));
  }
  if (lane == 0) {
    if (unsorted) atomicOr(&flags->unsorted, 1);
    if (nan) atomicOr(&flags->has_nan, 1);
    if (bad != ~0ull) atomicMin(&flags->bad_index, bad);
    if (mx != LLONG_MIN) atomicMax(&flags->max_eid, mx);
    if (mn != LLONG_MAX) atomicMin(&flags->min_eid, mn);
  }
  if (HIST) {
    __syncthreads();
    uint32_t* row = cnt + static_cast<int64_t>(blockIdx.x) * V;
    for (int i = threadIdx.x; i < static_cast<int>(V); i += kHistThreads) row[i] = hist[i];
  }
}

// the large-V sort input made by k_flags_keys
struct LargePre {
  uint32_t* key;
  uint32_t* val;
  unsigned long long* hist;  // [passes][256]
};

// Large-V flags pass (k_hist's checks: endpoints, (t, eid) order, NaN, eid range) that also
// emits the sort input of build_large_k -- key = the entry's node, val = its emission index --
// and the keys' 8-bit digit histograms for all `passes` digit positions: the event stream is
// read once instead of three times (flags, keys, histograms).  The keys are used only when
// the stream turns out (t, eid)-sorted.
template <int R>
__global__ void __launch_bounds__(kHistThreads) k_flags_keys(const tgfx_event* __restrict__ ev,
                                                             int64_t n, int64_t V, int64_t Vd,
                                                             int64_t chunk_ev, int passes,
                                                             uint32_t* __restrict__ key,
                                                             uint32_t* __restrict__ val,
                                                             unsigned long long* __restrict__ dh,
                                                             BuildFlags* flags) {
  __shared__ uint32_t h[4][256];
  for (int i = threadIdx.x; i < 4 * 256; i += kHistThreads) (&h[0][0])[i] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t e0 = static_cast<int64_t>(blockIdx.x) * chunk_ev;
  const int64_t e1 = min(n, e0 + chunk_ev);
  bool unsorted = false, nan = false;
  unsigned long long bad = ~0ull;
  long long mx = LLONG_MIN, mn = LLONG_MAX;
  constexpr int U = 4;
  for (int64_t b = e0; b < e1; b += U * kHistThreads) {
    Ev xs[U];
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const int64_t e = b + k * kHistThreads + threadIdx.x;
      xs[k] = e < e1 ? load_event(ev, e) : Ev{0, 0, 0, 0.0};
    }
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const int64_t e = b + k * kHistThreads + threadIdx.x;
      const bool valid = e < e1;
      const Ev x = xs[k];
      double tn = __shfl_down_sync(kFull, x.t, 1);
      long long en = __shfl_down_sync(kFull, (long long)x.eid, 1);
      if (valid && e + 1 < n && (lane == 31 || e + 1 >= e1)) {
        const Ev y = load_event(ev, e + 1);
        tn = y.t;
        en = y.eid;
      }
      if (valid && e + 1 < n) {
        const bool ok = (x.t < tn) || (x.t == tn && x.eid <= en);  // NaN -> not ok
        unsorted |= !ok;
      }
      const bool ok_s = valid && x.src >= 0 && x.src < V;
      const bool ok_d = valid && x.dst >= 0 && x.dst < Vd;
      if (valid && !(ok_s && ok_d)) bad = min(bad, (unsigned long long)e);
      if (valid) {
        nan |= x.t != x.t;
        mx = max(mx, (long long)x.eid);
        mn = min(mn, (long long)x.eid);
        // the entries of event e: j = R e (+ 1 for the reverse side), in emission order
        const uint32_t us = static_cast<uint32_t>(x.src), ud = static_cast<uint32_t>(x.dst);
        if (R == 2) {
          reinterpret_cast<uint2*>(key)[e] = make_uint2(us, ud);
          reinterpret_cast<uint2*>(val)[e] =
              make_uint2(static_cast<uint32_t>(2 * e), static_cast<uint32_t>(2 * e + 1));
        } else {
          key[e] = us;
          val[e] = static_cast<uint32_t>(e);
        }
        if (ok_s && ok_d) {
          for (int p = 0; p < passes; ++p) {
            atomicAdd(&h[p][(us >> (8 * p)) & 0xffu], 1u);
            if (R == 2) atomicAdd(&h[p][(ud >> (8 * p)) & 0xffu], 1u);
          }
        }
      }
    }
  }
  unsorted = __any_sync(kFull, unsorted);
  nan = __any_sync(kFull, nan);
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    bad = min(bad, __shfl_xor_sync(kFull, bad, o));
    mx = max(mx, __shfl_xor_sync(kFull, mx, o));
    mn = min(mn, __shfl_xor_sync(kFull, mn, o));
  }
  if (lane == 0) {
    if (unsorted) atomicOr(&flags->unsorted, 1);
    if (nan) atomicOr(&flags->has_nan, 1);
    if (bad != ~0ull) atomicMin(&flags->bad_index, bad);
    if (mx != LLONG_MIN) atomicMax(&flags->max_eid, mx);
    if (mn != LLONG_MAX) atomicMin(&flags->min_eid, mn);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < passes * 256; i += kHistThreads) {
    const uint32_t c = (&h[0][0])[i];
    if (c) atomicAdd(dh + i, static_cast<unsigned long long>(c));
  }
}

// K2a: degree of u = column sum of the chunk table (written to indptr[u] as a temporary)
__global__ void k_colsum(const uint32_t* __restrict__ cnt, int C, int32_t V, int64_t* deg) {
  const int u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= V) return;
  int64_t s = 0;
  int c = 0;
  for (; c + 8 <= C; c += 8) {
    uint32_t v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = cnt[static_cast<int64_t>(c + i) * V + u];
#pragma unroll
    for (int i = 0; i < 8; ++i) s += v[i];
  }
  for (; c < C; ++c) s += cnt[static_cast<int64_t>(c) * V + u];
  deg[u] = s;
}

// K2b: exclusive scan of deg[0..V) in place into indptr[0..V] (single CTA; V <= 45000), and
// of the cold nodes' degrees into cdelta[u] = coldbase[u] - indptr[u]: a cold entry at output
// position p of node u has dense cold index p + cdelta[u].  *ncold = total cold entries.
__device__ __forceinline__ int64_t block_excl_scan_1024(int64_t s, int64_t* wsum, int64_t* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int64_t x = s;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int64_t y = __shfl_up_sync(kFull, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wsum[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int64_t w = wsum[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(kFull, w, o);
      if (lane >= o) w += y;
    }
    wsum[lane] = w;
  }
  __syncthreads();
  const int64_t ex = (warp ? wsum[warp - 1] : 0) + x - s;
  *total = wsum[31];
  __syncthreads();
  return ex;
}

__global__ void __launch_bounds__(1024) k_indptr_scan(int64_t* a, int32_t V,
                                                      const uint32_t* __restrict__ coldbits,
                                                      int64_t* __restrict__ cdelta,
                                                      int64_t* __restrict__ ncold) {
  __shared__ int64_t wsum[32];
  const int per = (V + 1023) / 1024;
  const int64_t i0 = static_cast<int64_t>(threadIdx.x) * per;
  int64_t s = 0, sc = 0;
  for (int i = 0; i < per; ++i) {
    if (i0 + i < V) {
      const int64_t d = a[i0 + i];
      s += d;
      if ((coldbits[(i0 + i) >> 5] >> ((i0 + i) & 31)) & 1u) sc += d;
    }
  }
  int64_t tot, totc;
  int64_t run = block_excl_scan_1024(s, wsum, &tot);
  int64_t runc = block_excl_scan_1024(sc, wsum, &totc);
  for (int i = 0; i < per; ++i) {
    if (i0 + i < V) {
      const int64_t d = a[i0 + i];
      a[i0 + i] = run;
      cdelta[i0 + i] = runc - run;
      run += d;
      if ((coldbits[(i0 + i) >> 5] >> ((i0 + i) & 31)) & 1u) runc += d;
    }
  }
  if (threadIdx.x == 0) {
    a[V] = tot;
    *ncold = totc;
  }
}

// K2c: starting cursor of every (chunk, node): indptr[u] + sum of earlier chunks' counts
// With cold_space, a cold node's cursors start at its dense cold index (indptr[u] + cdelta[u])
// instead of its output position, so the scatter writes its records without a lookup.
__global__ void k_coloff(uint32_t* __restrict__ cnt, int C, int32_t V,
                         const int64_t* __restrict__ indptr, const uint32_t* __restrict__ coldbits,
                         const int64_t* __restrict__ cdelta, int cold_space) {
  const int u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= V) return;
  int64_t start = indptr[u];
  if (cold_space && ((coldbits[u >> 5] >> (u & 31)) & 1u)) start += cdelta[u];
  uint32_t run = static_cast<uint32_t>(start);
  int c = 0;
  for (; c + 8 <= C; c += 8) {  // 8 loads in flight per thread
    uint32_t t[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) t[q] = cnt[static_cast<int64_t>(c + q) * V + u];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      cnt[static_cast<int64_t>(c + q) * V + u] = run;
      run += t[q];
    }
  }
  for (; c < C; ++c) {
    const int64_t i = static_cast<int64_t>(c) * V + u;
    const uint32_t t = cnt[i];
    cnt[i] = run;
    run += t;
  }
}


// K2d: cold flags (one bit per node): entries of nodes with few entries per chunk are not
// written by the chunked scatter -- each chunk holds its own cursor per node, so a low-degree
// node's partially filled output sectors would sit in L2 for most of the kernel and get
// evicted half-written (read-modify-write at DRAM).  Their (pos, nbr, eid, ts) records are
// appended to a stream-ordered list instead and placed by k_cold in lockstep.
__global__ void k_coldflags(const int64_t* __restrict__ deg, int32_t V, int64_t thresh,
                            uint32_t* __restrict__ coldbits) {
  const int u = blockIdx.x * blockDim.x + threadIdx.x;
  const bool cold = u < V && deg[u] < thresh;
  const unsigned b = __ballot_sync(kFull, cold);
  if ((threadIdx.x & 31) == 0 && u < ((V + 31) & ~31)) coldbits[u >> 5] = b;
}

// Hot labels for the one-pass scatter (TGFX_SCATTER_VARIANT=50): the highest-degree non-cold
// nodes, at most 255, get labels 0..L-1 in node order; every other node 255.  One block: a
// degree threshold T is bisected until at most 255 non-cold nodes have degree >= T.
__global__ void __launch_bounds__(1024) k_hot_labels(const int64_t* __restrict__ deg, int32_t V,
                                                     const uint32_t* __restrict__ coldbits,
                                                     uint8_t* __restrict__ hot) {
  __shared__ int s_cnt;
  __shared__ int s_wsum[32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  auto is_cand = [&](int u, int64_t T) {
    return !((coldbits[u >> 5] >> (u & 31)) & 1u) && deg[u] >= T;
  };
  auto count = [&](int64_t T) {
    if (tid == 0) s_cnt = 0;
    __syncthreads();
    int c = 0;
    for (int u = tid; u < V; u += 1024) c += is_cand(u, T) ? 1 : 0;
    c = __reduce_add_sync(kFull, c);
    if (lane == 0 && c) atomicAdd(&s_cnt, c);
    __syncthreads();
    const int r = s_cnt;
    __syncthreads();
    return r;
  };
  int64_t lo = 0, hi = 0;  // smallest T with count(T) <= 255 lies in (lo, hi]
  {
    int64_t mx = 0;
    for (int u = tid; u < V; u += 1024) mx = max(mx, static_cast<int64_t>(deg[u]));
    for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(kFull, mx, o));
    __shared__ int64_t s_mx[32];
    if (lane == 0) s_mx[warp] = mx;
    __syncthreads();
    if (tid == 0) {
      int64_t m = 0;
      for (int w = 0; w < 32; ++w) m = max(m, s_mx[w]);
      s_mx[0] = m;
    }
    __syncthreads();
    hi = s_mx[0] + 1;
  }
  if (count(0) <= 255) {
    hi = 0;
  } else {
    while (hi - lo > 1) {
      const int64_t mid = lo + (hi - lo) / 2;
      if (count(mid) <= 255) hi = mid; else lo = mid;
    }
  }
  const int64_t T = hi;
  // labels in node order: each thread a contiguous node range, block exclusive scan of counts
  const int per = (V + 1023) / 1024;
  const int u0 = min(V, tid * per), u1 = min(V, u0 + per);
  int c = 0;
  for (int u = u0; u < u1; ++u) c += is_cand(u, T) ? 1 : 0;
  int x = c;
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(kFull, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_wsum[warp] = x;
  __syncthreads();
  int before = 0;
  for (int w = 0; w < warp; ++w) before += s_wsum[w];
  int next = before + x - c;
  for (int u = u0; u < u1; ++u) hot[u] = is_cand(u, T) ? static_cast<uint8_t>(next++) : 255;
}

// K3: stable scatter ("ticketed warps") ---------------------------------------------------
// Each CTA owns a contiguous chunk and its per-node cursors (shared memory).  The chunk is cut
// into warp tiles of kTkRounds x 32 consecutive entries, taken by the CTA's warps round-robin.
// A warp loads and groups its tile (MATCH.ANY per round) with no shared state, then waits for
// the CTA's ticket to reach its tile and runs a short critical section: for each round, the
// leader of every node group reads and bumps that node's cursor (distinct nodes per round, so
// one LDS/STS per group, rounds in order).  Emission order is preserved by construction.
// Positions are written after the ticket is passed on.

__device__ __forceinline__ void named_bar_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void named_bar_arrive(int id, int n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}

template <int R, int kTkRounds, int kTkWarps>
__global__ void __launch_bounds__(kTkWarps * 32) k_scatter(
    const tgfx_event* __restrict__ ev, int64_t n, int32_t V, int64_t chunk_ev,
    const uint32_t* __restrict__ off, const uint32_t* __restrict__ coldbits_g,
    const int64_t* __restrict__ cdelta, ulonglong2* __restrict__ cold_img,
    int64_t* __restrict__ nbr_out, int64_t* __restrict__ eid_out, double* __restrict__ ts_out) {
  extern __shared__ __align__(16) uint32_t smem[];
  const int vpad = (V + 31) & ~31;
  uint32_t* cursor = smem;                 // [V]
  uint32_t* coldbits = cursor + vpad;      // [V/32]

  const int lane = threadIdx.x & 31;
  const int warp = __shfl_sync(kFull, static_cast<int>(threadIdx.x >> 5), 0);  // warp-uniform
  const int64_t e0 = static_cast<int64_t>(blockIdx.x) * chunk_ev;
  const int64_t e1 = min(n, e0 + chunk_ev);
  if (e0 >= e1) return;
  const uint32_t* orow = off + static_cast<int64_t>(blockIdx.x) * V;
  constexpr int kTkThreads = kTkWarps * 32;
  for (int i = threadIdx.x; i < V; i += kTkThreads) cursor[i] = orow[i];
  for (int i = threadIdx.x; i < vpad / 32; i += kTkThreads) coldbits[i] = coldbits_g[i];
  __syncthreads();

  const int64_t E0 = e0 * R, E1 = e1 * R;
  constexpr int kTile = kTkRounds * 32;
  const int64_t ntiles = ceil_div(E1 - E0, kTile);
  for (int64_t t = warp; t < ntiles; t += kTkWarps) {
    const int64_t T0 = E0 + t * kTile;
    Ev x[kTkRounds];
#pragma unroll
    for (int r = 0; r < kTkRounds; ++r) {
      const int64_t j = T0 + r * 32 + lane;
      x[r] = j < E1 ? load_event(ev, R == 2 ? (j >> 1) : j) : Ev{0, -1, -1, 0.0};
    }
    uint32_t node[kTkRounds], peers[kTkRounds];
#pragma unroll
    for (int r = 0; r < kTkRounds; ++r) {
      const int64_t j = T0 + r * 32 + lane;
      const bool side = R == 2 && (j & 1);
      const bool ok = j < E1;  // endpoints validated by k_hist
      node[r] = ok ? static_cast<uint32_t>(side ? x[r].dst : x[r].src) : 0xffffffffu;
      if (side) {  // keep the other endpoint in .dst, so .dst is always the neighbour
        const int64_t a = x[r].src;
        x[r].src = x[r].dst;
        x[r].dst = a;
      }
      peers[r] = __match_any_sync(kFull, node[r]);
    }
    // cold flags and cold-index offsets, fetched before the critical section so their
    // latency overlaps the ticket wait
    int64_t cd[kTkRounds];
#pragma unroll
    for (int r = 0; r < kTkRounds; ++r) {
      const bool cold = node[r] != 0xffffffffu && ((coldbits[node[r] >> 5] >> (node[r] & 31)) & 1u);
      cd[r] = cold ? __ldg(reinterpret_cast<const long long*>(cdelta) + node[r]) : INT64_MIN;
    }
    // critical section: wait until the owner of tile t-1 (the previous warp) hands over.
    // Named barrier 1+w is warp w's inbox: the previous warp arrives, this warp syncs
    // (hardware wait, no spinning; bar.arrive/bar.sync order the shared-memory cursors).
    if (t > 0) named_bar_sync(1 + warp, 64);
    uint32_t base[kTkRounds];
#pragma unroll
    for (int r = 0; r < kTkRounds; ++r) {
      const bool lead = node[r] != 0xffffffffu && lane == __ffs(peers[r]) - 1;
      uint32_t b = 0;
      if (lead) {
        b = cursor[node[r]];
        cursor[node[r]] = b + __popc(peers[r]);
      }
      base[r] = b;
      __syncwarp();
    }
    if (t + 1 < ntiles) named_bar_arrive(1 + (warp + 1) % kTkWarps, 64);
    // positions and writes, outside the critical section
#pragma unroll
    for (int r = 0; r < kTkRounds; ++r) {
      const int leader = __ffs(peers[r]) - 1;
      const uint32_t pos =
          __shfl_sync(kFull, base[r], leader) + __popc(peers[r] & lanemask_lt());
      const bool ok = node[r] != 0xffffffffu;
      const bool cold = cd[r] != INT64_MIN;
      if (ok && !cold) {
        nbr_out[pos] = x[r].dst;
        eid_out[pos] = x[r].eid;
        ts_out[pos] = x[r].t;
      }
      if (cold) {
        // dense cold index; one full 32-byte record (no partial-sector write)
        const int64_t ci = static_cast<int64_t>(pos) + cd[r];
        ulonglong2* rec = cold_img + 2 * ci;
        rec[0] = make_ulonglong2(static_cast<unsigned long long>(x[r].dst),
                                 static_cast<unsigned long long>(x[r].eid));
        rec[1] = make_ulonglong2(static_cast<unsigned long long>(__double_as_longlong(x[r].t)),
                                 static_cast<unsigned long long>(pos));
      }
    }
  }
}

// K3' (default): tile-sorted stable scatter.
// Each CTA owns a contiguous chunk of the stream and its V cursors (shared memory, from the
// C x V offset table).  The chunk is streamed through shared memory in tiles of kTE events
// by 1-D bulk copies (cp.async.bulk + mbarrier, double-buffered), and every tile is ranked
// by node with a block-wide stable LSD radix sort of (node << 16 | entry index) keys:
// 8-bit digits, per-warp digit counters ranked with __match_any_sync, one exclusive scan
// over (digit, warp).  After the sort a node's entries of the tile are one contiguous run,
// so each entry's output position is cursor[u] + (its offset in the run), the run's tail
// bumps the cursor, and consecutive threads store consecutive positions of a run (the Zipf
// hub's entries go out as coalesced bursts).  All warps of the CTA work on every tile --
// no serialisation across warps -- and the tile loads overlap the ranking of the previous
// tile.  Entries of cold nodes are written as full 32-byte records (see k_coldflags).
constexpr int kTStages = 4;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

template <int kTT, int kTE>
size_t tile_scatter_smem(int64_t V) {
  const int64_t vpad = (V + 31) & ~31LL;
  return static_cast<size_t>(kTStages) * kTE * 32  // event stages
         + 2 * 2 * kTE * 4                          // key ping-pong (2 entries per event max)
         + (kTT / 32) * 256 * 4                     // per-warp digit counters
         + 64 * 8                                   // barriers + scan scratch
         + vpad * 4 + (vpad / 32) * 4;              // cursors + cold bits
}

template <int R, int kTT, int kTE>
__global__ void __launch_bounds__(kTT) k_scatter_tile(
    const tgfx_event* __restrict__ ev, int64_t n, int32_t V, int64_t chunk_ev, int passes,
    const uint32_t* __restrict__ off, const uint32_t* __restrict__ coldbits_g,
    const int64_t* __restrict__ cdelta, ulonglong2* __restrict__ cold_img,
    int64_t* __restrict__ nbr_out, int64_t* __restrict__ eid_out, double* __restrict__ ts_out,
    uint4* __restrict__ rec_out) {
  constexpr int kTW = kTT / 32;
  constexpr int NE = kTE * R;       // entries per tile
  constexpr int KPT = NE / kTT;     // keys per thread
  static_assert(KPT * kTT == NE && KPT >= 1, "tile shape");
  extern __shared__ __align__(128) unsigned char sm[];
  tgfx_event* stage = reinterpret_cast<tgfx_event*>(sm);
  uint32_t* keys0 = reinterpret_cast<uint32_t*>(sm + kTStages * kTE * 32);
  uint32_t* keys1 = keys0 + NE;
  uint32_t* wcnt = keys0 + 2 * 2 * kTE;  // [kTW][256]
  uint64_t* bars = reinterpret_cast<uint64_t*>(wcnt + kTW * 256);
  int* scr = reinterpret_cast<int*>(bars + 8);  // 32 ints of scan scratch (+ spare)
  const int vpad = (V + 31) & ~31;
  uint32_t* cursor = reinterpret_cast<uint32_t*>(bars + 64);
  uint32_t* coldbits = cursor + vpad;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t e0 = static_cast<int64_t>(blockIdx.x) * chunk_ev;
  const int64_t e1 = min(n, e0 + chunk_ev);
  if (e0 >= e1) return;
  const int64_t ntiles = ceil_div(e1 - e0, kTE);
  if (tid == 0) {
    for (int s = 0; s < kTStages; ++s) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid == 0) {
    for (int s = 0; s < kTStages && s < ntiles; ++s) {
      const int64_t b = e0 + static_cast<int64_t>(s) * kTE;
      const uint32_t bytes = static_cast<uint32_t>(min(static_cast<int64_t>(kTE), e1 - b) * 32);
      mbar_arrive_tx(&bars[s], bytes);
      bulk_g2s(stage + s * kTE, ev + b, bytes, &bars[s]);
    }
  }
  const uint32_t* orow = off + static_cast<int64_t>(blockIdx.x) * V;
  for (int i = tid; i < V; i += kTT) cursor[i] = orow[i];
  for (int i = tid; i < vpad / 32; i += kTT) coldbits[i] = coldbits_g[i];
  __syncthreads();

  for (int64_t it = 0; it < ntiles; ++it) {
    const int sidx = static_cast<int>(it % kTStages);
    const uint32_t phase = static_cast<uint32_t>((it / kTStages) & 1);
    const int64_t tb = e0 + it * kTE;
    const int cnt = static_cast<int>(min(static_cast<int64_t>(kTE), e1 - tb));
    const int ent = cnt * R;
    const tgfx_event* sev = stage + sidx * kTE;
    mbar_wait(&bars[sidx], phase);

    // keys in warp-striped order: entry j = warp*32*KPT + k*32 + lane (emission order)
    uint32_t key[KPT];
#pragma unroll
    for (int k = 0; k < KPT; ++k) {
      const int j = warp * 32 * KPT + k * 32 + lane;
      uint32_t node = static_cast<uint32_t>(V);  // sentinel: sorts after every real node
      if (j < ent) {
        const int64_t* e = reinterpret_cast<const int64_t*>(sev + (R == 2 ? (j >> 1) : j));
        node = static_cast<uint32_t>((R == 2 && (j & 1)) ? e[2] : e[1]);
      }
      key[k] = (node << 16) | static_cast<uint32_t>(j);
    }
    uint32_t* src_keys = keys0;
    uint32_t* dst_keys = keys1;
    for (int p = 0; p < passes; ++p) {
      const int shift = 16 + 8 * p;
      uint32_t* wc = wcnt + warp * 256;
#pragma unroll
      for (int c = 0; c < 8; ++c) wc[c * 32 + lane] = 0;
      __syncwarp();
      int rank[KPT];
      uint32_t dig[KPT];
      unsigned peers[KPT];
      // lanes with the same 8-bit digit: one MATCH.ANY per key (measured faster here than
      // intersecting 8 bit-plane ballots: build 11.4 vs 11.9 ms on the GDELT shape)
#pragma unroll
      for (int k = 0; k < KPT; ++k) {
        dig[k] = (key[k] >> shift) & 0xffu;
        peers[k] = __match_any_sync(kFull, dig[k]);
      }
#pragma unroll
      for (int k = 0; k < KPT; ++k) {
        const uint32_t b = wc[dig[k]];
        __syncwarp();
        if (lane == __ffs(peers[k]) - 1) wc[dig[k]] = b + __popc(peers[k]);
        __syncwarp();
        rank[k] = static_cast<int>(b) + __popc(peers[k] & lanemask_lt());
      }
      __syncthreads();
      // exclusive scan of the kTW x 256 counters in (digit, warp) order; thread t owns the 8
      // consecutive (digit-major) counters t*8 .. t*8+7
      {
        uint32_t v[8], s = 0;
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const int i = tid * 8 + c;
          v[c] = wcnt[(i % kTW) * 256 + i / kTW];
          s += v[c];
        }
        uint32_t x = s;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t y = __shfl_up_sync(kFull, x, o);
          if (lane >= o) x += y;
        }
        if (lane == 31) scr[warp] = static_cast<int>(x);
        __syncthreads();
        // totals of the earlier warps: lane w < warp reads scr[w], one warp reduction
        const uint32_t before = __reduce_add_sync(
            kFull, lane < warp ? static_cast<uint32_t>(scr[lane]) : 0u);
        uint32_t run = before + x - s;
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const int i = tid * 8 + c;
          wcnt[(i % kTW) * 256 + i / kTW] = run;
          run += v[c];
        }
      }
      __syncthreads();
#pragma unroll
      for (int k = 0; k < KPT; ++k) dst_keys[wc[dig[k]] + rank[k]] = key[k];
      __syncthreads();
#pragma unroll
      for (int k = 0; k < KPT; ++k) key[k] = dst_keys[warp * 32 * KPT + k * 32 + lane];
      uint32_t* tmp = src_keys;
      src_keys = dst_keys;
      dst_keys = tmp;
    }
    // sorted: src_keys[s], thread holds s = warp*32*KPT + k*32 + lane.  Head of each node run
    // = last position <= s where the node changes: inclusive max-scan of head positions.
    int hp[KPT];
    uint32_t u[KPT];
    {
      int carry = 0;
#pragma unroll
      for (int k = 0; k < KPT; ++k) {
        const int s = warp * 32 * KPT + k * 32 + lane;
        u[k] = key[k] >> 16;
        const bool head = s == 0 || (src_keys[s - 1] >> 16) != u[k];
        int x = head ? s : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(kFull, x, o);
          if (lane >= o) x = max(x, y);
        }
        x = max(x, carry);
        hp[k] = x;
        carry = __shfl_sync(kFull, x, 31);
      }
      if (lane == 31) scr[warp] = carry;
      __syncthreads();
      const int prev = static_cast<int>(
          __reduce_max_sync(kFull, lane < warp ? static_cast<unsigned>(scr[lane]) : 0u));
#pragma unroll
      for (int k = 0; k < KPT; ++k) hp[k] = max(hp[k], prev);
    }
    uint32_t pos[KPT];
#pragma unroll
    for (int k = 0; k < KPT; ++k) {
      const int s = warp * 32 * KPT + k * 32 + lane;
      pos[k] = u[k] < static_cast<uint32_t>(V) ? cursor[u[k]] + static_cast<uint32_t>(s - hp[k]) : 0u;
    }
    __syncthreads();  // every entry has read its run's cursor
#pragma unroll
    for (int k = 0; k < KPT; ++k) {
      const int s = warp * 32 * KPT + k * 32 + lane;
      if (u[k] >= static_cast<uint32_t>(V)) continue;
      const bool tail = s == NE - 1 || (src_keys[s + 1] >> 16) != u[k];
      if (tail) cursor[u[k]] = pos[k] + 1;
      const int j = static_cast<int>(key[k] & 0xffffu);
      const longlong2* e = reinterpret_cast<const longlong2*>(sev + (R == 2 ? (j >> 1) : j));
      const longlong2 a = e[0], b = e[1];  // (eid, src), (dst, t bits)
      const bool side = R == 2 && (j & 1);
      const long long other = side ? a.y : b.x;
      if ((coldbits[u[k] >> 5] >> (u[k] & 31)) & 1u) {
        // cold node: its cursors run in dense cold-index space (k_coloff), record carries u
        ulonglong2* rec = cold_img + 2 * static_cast<int64_t>(pos[k]);
        rec[0] = make_ulonglong2(static_cast<unsigned long long>(other), static_cast<unsigned long long>(a.x));
        rec[1] = make_ulonglong2(static_cast<unsigned long long>(b.y), static_cast<unsigned long long>(u[k]));
      } else {
        ts_out[pos[k]] = __longlong_as_double(b.y);
        if (rec_out) {  // gather record instead of the int64 columns (widened on demand)
          rec_out[pos[k]] = make_uint4(static_cast<uint32_t>(other), static_cast<uint32_t>(a.x),
                                       static_cast<uint32_t>(b.y),
                                       static_cast<uint32_t>(static_cast<unsigned long long>(b.y) >> 32));
        } else {
          nbr_out[pos[k]] = other;
          eid_out[pos[k]] = a.x;
        }
      }
    }
    __syncthreads();  // stage buffer consumed, cursors final for this tile
    if (tid == 0 && it + kTStages < ntiles) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      const int64_t b = e0 + (it + kTStages) * kTE;
      const uint32_t bytes = static_cast<uint32_t>(min(static_cast<int64_t>(kTE), e1 - b) * 32);
      mbar_arrive_tx(&bars[sidx], bytes);
      bulk_g2s(stage + sidx * kTE, ev + b, bytes, &bars[sidx]);
    }
  }
}

// K4: place the cold entries.  Consecutive cold indices are consecutive positions of a cold
// node's slice, so both the 32-byte record reads and the column writes are coalesced.
__global__ void __launch_bounds__(256) k_cold(const ulonglong2* __restrict__ img, int64_t ncold,
                                              int64_t* __restrict__ nbr_out,
                                              int64_t* __restrict__ eid_out,
                                              double* __restrict__ ts_out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < ncold;
       i += (int64_t)gridDim.x * blockDim.x) {
    const ulonglong2 a = __ldg(img + 2 * i);
    const ulonglong2 b = __ldg(img + 2 * i + 1);
    const int64_t pos = static_cast<int64_t>(b.y);
    nbr_out[pos] = static_cast<int64_t>(a.x);
    eid_out[pos] = static_cast<int64_t>(a.y);
    ts_out[pos] = __longlong_as_double(static_cast<long long>(b.x));
  }
}

// K4 for the tile scatter: records carry their node; output position = cold index - cdelta[u]
__global__ void __launch_bounds__(256) k_cold_u(const ulonglong2* __restrict__ img, int64_t ncold,
                                                const int64_t* __restrict__ cdelta,
                                                int64_t* __restrict__ nbr_out,
                                                int64_t* __restrict__ eid_out,
                                                double* __restrict__ ts_out,
                                                uint4* __restrict__ rec_out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < ncold;
       i += (int64_t)gridDim.x * blockDim.x) {
    const ulonglong2 a = __ldg(img + 2 * i);
    const ulonglong2 b = __ldg(img + 2 * i + 1);
    const int64_t pos = i - __ldg(reinterpret_cast<const long long*>(cdelta) + b.y);
    ts_out[pos] = __longlong_as_double(static_cast<long long>(b.x));
    if (rec_out) {
      rec_out[pos] = make_uint4(static_cast<uint32_t>(a.x), static_cast<uint32_t>(a.y),
                                static_cast<uint32_t>(b.x), static_cast<uint32_t>(b.x >> 32));
    } else {
      nbr_out[pos] = static_cast<int64_t>(a.x);
      eid_out[pos] = static_cast<int64_t>(a.y);
    }
  }
}

// entry writer shared by the scatter kernels: gather record + ts at pos, or a 32-byte cold
// record in dense cold-index space
template <int R>
__device__ __forceinline__ void hot_write_entry(const tgfx_event* sev, int j, uint32_t pos,
                                                const uint32_t* coldbits,
                                                ulonglong2* __restrict__ cold_img,
                                                double* __restrict__ ts_out,
                                                uint4* __restrict__ rec_out,
                                                int64_t* __restrict__ nbr_out,
                                                int64_t* __restrict__ eid_out) {
  const longlong2* e = reinterpret_cast<const longlong2*>(sev + (R == 2 ? (j >> 1) : j));
  const longlong2 a = e[0], b = e[1];  // (eid, src), (dst, t bits)
  const bool side = R == 2 && (j & 1);
  const long long other = side ? a.y : b.x;
  const uint32_t u = static_cast<uint32_t>(side ? b.x : a.y);
  if ((coldbits[u >> 5] >> (u & 31)) & 1u) {
    ulonglong2* rec = cold_img + 2 * static_cast<int64_t>(pos);
    rec[0] = make_ulonglong2(static_cast<unsigned long long>(other), static_cast<unsigned long long>(a.x));
    rec[1] = make_ulonglong2(static_cast<unsigned long long>(b.y), static_cast<unsigned long long>(u));
  } else {
    ts_out[pos] = __longlong_as_double(b.y);
    if (rec_out) {
      rec_out[pos] = make_uint4(static_cast<uint32_t>(other), static_cast<uint32_t>(a.x),
                                static_cast<uint32_t>(b.y),
                                static_cast<uint32_t>(static_cast<unsigned long long>(b.y) >> 32));
    } else {
      nbr_out[pos] = other;
      eid_out[pos] = a.x;
    }
  }
}

// as hot_write_entry, with the entry's node and cold flag already known
template <int R>
__device__ __forceinline__ void write_entry_known(const tgfx_event* sev, int j, uint32_t pos,
                                                  uint32_t u, bool cold,
                                                  ulonglong2* __restrict__ cold_img,
                                                  double* __restrict__ ts_out,
                                                  uint4* __restrict__ rec_out,
                                                  int64_t* __restrict__ nbr_out,
                                                  int64_t* __restrict__ eid_out) {
  const longlong2* e = reinterpret_cast<const longlong2*>(sev + (R == 2 ? (j >> 1) : j));
  const longlong2 a = e[0], b = e[1];  // (eid, src), (dst, t bits)
  const bool side = R == 2 && (j & 1);
  const long long other = side ? a.y : b.x;
  if (cold) {
    ulonglong2* rec = cold_img + 2 * static_cast<int64_t>(pos);
    rec[0] = make_ulonglong2(static_cast<unsigned long long>(other), static_cast<unsigned long long>(a.x));
    rec[1] = make_ulonglong2(static_cast<unsigned long long>(b.y), static_cast<unsigned long long>(u));
  } else {
    ts_out[pos] = __longlong_as_double(b.y);
    if (rec_out) {
      rec_out[pos] = make_uint4(static_cast<uint32_t>(other), static_cast<uint32_t>(a.x),
                                static_cast<uint32_t>(b.y),
                                static_cast<uint32_t>(static_cast<unsigned long long>(b.y) >> 32));
    } else {
      nbr_out[pos] = other;
      eid_out[pos] = a.x;
    }
  }
}

template <int R>
__device__ __forceinline__ uint32_t hot_node_of(const tgfx_event* sev, int j) {
  const int64_t* e = reinterpret_cast<const int64_t*>(sev + (R == 2 ? (j >> 1) : j));
  return static_cast<uint32_t>((R == 2 && (j & 1)) ? e[2] : e[1]);
}

// K3 "big tiles, cursors in L2" (TGFX_SCATTER_VARIANT=40).
// The tile kernel above keeps every node's cursor in shared memory (V x 4 B), which leaves room
// for only small tiles (2 keys per thread) -- its ranking is dominated by per-tile barrier and
// shared-memory latency.  Here the cursors stay in the chunk's row of the C x V offset table in
// global memory (L2-resident: 20 MB for the GDELT shape; read and written with .cg, only by the
// owning CTA, tiles in order separated by __syncthreads), so shared memory holds just the event
// stages and the key buffers, and a tile is 2048 entries: 8 keys per thread per radix pass
// (block-wide stable LSD rank by 8-bit digits, warp-striped keys, per-warp digit counters
// grouped by MATCH.ANY, one scan over (digit, warp)).  After the sort a node's tile entries
// form one run: the run head fetches the node's cursor (one L2 round trip per tile, all runs
// in parallel), every entry takes cursor + offset in run, the tail stores cursor + run length.
// Entries are written in sorted order, so a run's stores are consecutive addresses.
constexpr int kBT = 256;  // threads

// SC: cursors (and cold bits) in shared memory instead of L2
template <int R, int TE, int S, bool SC>
size_t big_smem(int64_t V) {
  const size_t vpad = static_cast<size_t>((V + 31) & ~31LL);
  return static_cast<size_t>(S) * TE * 32 + 2 * static_cast<size_t>(R) * TE * 4 +
         (kBT / 32) * 256 * 2 + S * 8 + 64 * 4 + (SC ? vpad * 4 + vpad / 8 : 0);
}

template <int R, int TE, int S, bool SC>
__global__ void __launch_bounds__(kBT, 2) k_scatter_big(
    const tgfx_event* __restrict__ ev, int64_t n, int32_t V, int64_t chunk_ev, int passes,
    uint32_t* __restrict__ off, const uint32_t* __restrict__ coldbits,
    ulonglong2* __restrict__ cold_img, double* __restrict__ ts_out, uint4* __restrict__ rec_out,
    int64_t* __restrict__ nbr_out, int64_t* __restrict__ eid_out, int cflag) {
  constexpr int NE = TE * R;
  constexpr int KPT = NE / kBT;
  constexpr int kW = kBT / 32;
  static_assert(KPT * kBT == NE && NE <= 65536, "tile shape");
  extern __shared__ __align__(128) unsigned char sm[];
  tgfx_event* stage = reinterpret_cast<tgfx_event*>(sm);
  uint32_t* keys0 = reinterpret_cast<uint32_t*>(sm + static_cast<size_t>(S) * TE * 32);
  uint32_t* keys1 = keys0 + NE;
  uint16_t* wcnt = reinterpret_cast<uint16_t*>(keys1 + NE);  // [kW][256]
  uint64_t* bars = reinterpret_cast<uint64_t*>(wcnt + kW * 256);
  int* scr = reinterpret_cast<int*>(bars + S);
  uint32_t* scur = reinterpret_cast<uint32_t*>(scr + 64);   // SC: [vpad] cursors
  uint32_t* scold = scur + ((V + 31) & ~31);                 // SC: [vpad / 32] cold bits

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t e0 = static_cast<int64_t>(blockIdx.x) * chunk_ev;
  const int64_t e1 = min(n, e0 + chunk_ev);
  if (e0 >= e1) return;
  const int64_t ntiles = ceil_div(e1 - e0, TE);
  uint32_t* crow = off + static_cast<int64_t>(blockIdx.x) * V;  // this chunk's cursors
  if (SC) {
    for (int i = tid; i < V; i += kBT) scur[i] = crow[i];
    for (int i = tid; i < ((V + 31) >> 5); i += kBT) scold[i] = coldbits[i];
  }
  const uint32_t* cbits = SC ? scold : coldbits;
  if (tid == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid == 0) {
    for (int s = 0; s < S && s < ntiles; ++s) {
      const int64_t b = e0 + static_cast<int64_t>(s) * TE;
      const uint32_t bytes = static_cast<uint32_t>(min(static_cast<int64_t>(TE), e1 - b) * 32);
      mbar_arrive_tx(&bars[s], bytes);
      bulk_g2s(stage + s * TE, ev + b, bytes, &bars[s]);
    }
  }
  for (int64_t it = 0; it < ntiles; ++it) {
    const int sidx = static_cast<int>(it % S);
    const int64_t tb = e0 + it * TE;
    const int ent = static_cast<int>(min(static_cast<int64_t>(TE), e1 - tb)) * R;
    const tgfx_event* sev = stage + sidx * TE;
    mbar_wait(&bars[sidx], static_cast<uint32_t>((it / S) & 1));
    uint32_t key[KPT];
#pragma unroll
    for (int k = 0; k < KPT; ++k) {
      const int j = warp * 32 * KPT + k * 32 + lane;
      uint32_t node = static_cast<uint32_t>(V);  // sentinel sorts after every real node
      if (j < ent) node = hot_node_of<R>(sev, j);
      key[k] = (node << 16) | static_cast<uint32_t>(j);
    }
    uint32_t* src_keys = keys0;
    uint32_t* dst_keys = keys1;
    for (int p = 0; p < passes; ++p) {
      const int shift = 16 + 8 * p;
      uint16_t* wc = wcnt + warp * 256;
      reinterpret_cast<uint4*>(wc)[lane] = make_uint4(0, 0, 0, 0);
      __syncwarp();
      uint32_t rank[KPT];
      uint32_t dig[KPT];
      unsigned peers[KPT];
      // all MATCH.ANYs first (independent; their latency overlaps), then the counter chain
#pragma unroll
      for (int k = 0; k < KPT; ++k) {
        dig[k] = (key[k] >> shift) & 0xffu;
        peers[k] = __match_any_sync(kFull, dig[k]);
      }
#pragma unroll
      for (int k = 0; k < KPT; ++k) {
        const uint32_t b = wc[dig[k]];
        __syncwarp();
        if (lane == __ffs(peers[k]) - 1) wc[dig[k]] = static_cast<uint16_t>(b + __popc(peers[k]));
        __syncwarp();
        rank[k] = b + __popc(peers[k] & lanemask_lt());
      }
      __syncthreads();
      {  // exclusive scan of the kW x 256 counters in (digit, warp) order: 64 threads, each
         // 4 digits x kW warps read as kW 8-byte loads (a quarter of the shared-memory
         // instructions of one 2-byte load per counter)
        static_assert(kW == 8, "scan layout");
        constexpr int kDT = 4;           // digits per thread
        constexpr int kNT = 256 / kDT;   // active threads (2 warps)
        uint2 v[kW];
        uint32_t tot = 0;
        if (tid < kNT) {
#pragma unroll
          for (int w = 0; w < kW; ++w) {
            v[w] = *reinterpret_cast<const uint2*>(wcnt + w * 256 + kDT * tid);
            tot += (v[w].x & 0xffffu) + (v[w].x >> 16) + (v[w].y & 0xffffu) + (v[w].y >> 16);
          }
        }
        uint32_t x = tot;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t y = __shfl_up_sync(kFull, x, o);
          if (lane >= o) x += y;
        }
        if (lane == 31 && warp == 0) scr[0] = static_cast<int>(x);
        __syncthreads();
        if (tid < kNT) {
          uint32_t run = (warp == 1 ? static_cast<uint32_t>(scr[0]) : 0u) + x - tot;
          uint32_t o[kW][kDT];
#pragma unroll
          for (int dd = 0; dd < kDT; ++dd) {
#pragma unroll
            for (int w = 0; w < kW; ++w) {
              const uint32_t word = dd < 2 ? v[w].x : v[w].y;
              const uint32_t c = (word >> (16 * (dd & 1))) & 0xffffu;
              o[w][dd] = run;
              run += c;
            }
          }
#pragma unroll
          for (int w = 0; w < kW; ++w)
            *reinterpret_cast<uint2*>(wcnt + w * 256 + kDT * tid) =
                make_uint2(o[w][0] | (o[w][1] << 16), o[w][2] | (o[w][3] << 16));
        }
      }
      __syncthreads();
#pragma unroll
      for (int k = 0; k < KPT; ++k) dst_keys[wc[dig[k]] + rank[k]] = key[k];
      __syncthreads();
#pragma unroll
      for (int k = 0; k < KPT; ++k) key[k] = dst_keys[warp * 32 * KPT + k * 32 + lane];
      uint32_t* tmp = src_keys;
      src_keys = dst_keys;
      dst_keys = tmp;
    }
    // sorted keys in src_keys; this thread holds positions s = warp*32*KPT + k*32 + lane.
    // Run heads fetch the cursor into dst_keys[s] (free now); every entry finds its head by an
    // inclusive max-scan of head positions.
    int hp[KPT];
    {
      int carry = 0;
#pragma unroll
      for (int k = 0; k < KPT; ++k) {
        const int s = warp * 32 * KPT + k * 32 + lane;
        const uint32_t u = key[k] >> 16;
        const bool head = s == 0 || (src_keys[s - 1] >> 16) != u;
        // run heads fetch the cursor -- with the node's cold flag in bit 31 while positions
        // fit 31 bits (cflag), so the run's entries need no cold-bit lookup of their own
        if (head && u < static_cast<uint32_t>(V)) {
          const uint32_t c = SC ? scur[u] : __ldcg(crow + u);
          dst_keys[s] = cflag ? c | (((cbits[u >> 5] >> (u & 31)) & 1u) << 31) : c;
        }
        int x = head ? s : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(kFull, x, o);
          if (lane >= o) x = max(x, y);
        }
        x = max(x, carry);
        hp[k] = x;
        carry = __shfl_sync(kFull, x, 31);
      }
      if (lane == 31) scr[32 + warp] = carry;
      __syncthreads();
      const int prev = static_cast<int>(
          __reduce_max_sync(kFull, lane < warp ? static_cast<unsigned>(scr[32 + lane]) : 0u));
#pragma unroll
      for (int k = 0; k < KPT; ++k) hp[k] = max(hp[k], prev);
    }
#pragma unroll
    for (int k = 0; k < KPT; ++k) {
      const int s = warp * 32 * KPT + k * 32 + lane;
      const uint32_t u = key[k] >> 16;
      if (u >= static_cast<uint32_t>(V)) continue;
      const uint32_t h = dst_keys[hp[k]];
      const uint32_t pos = (cflag ? h & 0x7fffffffu : h) + static_cast<uint32_t>(s - hp[k]);
      const bool tail = s == NE - 1 || (src_keys[s + 1] >> 16) != u;
      if (tail) {
        if (SC)
          scur[u] = pos + 1;
        else
          __stcg(crow + u, pos + 1);
      }
      if (cflag)
        write_entry_known<R>(sev, static_cast<int>(key[k] & 0xffffu), pos, u, (h >> 31) != 0,
                             cold_img, ts_out, rec_out, nbr_out, eid_out);
      else
        hot_write_entry<R>(sev, static_cast<int>(key[k] & 0xffffu), pos, cbits, cold_img, ts_out,
                           rec_out, nbr_out, eid_out);
    }
    __syncthreads();  // stage consumed; cursor stores ordered before the next tile's loads
    if (tid == 0 && it + S < ntiles) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      const int64_t b = e0 + (it + S) * TE;
      const uint32_t bytes = static_cast<uint32_t>(min(static_cast<int64_t>(TE), e1 - b) * 32);
      mbar_arrive_tx(&bars[sidx], bytes);
      bulk_g2s(stage + sidx * TE, ev + b, bytes, &bars[sidx]);
    }
  }
}

// K3 one-pass variant (TGFX_SCATTER_VARIANT=50).  The hub nodes (k_hot_labels: <= 255 of
// them, ~81 % of the GDELT-shaped entries) are ranked by ONE block-wide stable pass over their
// 8-bit label; everything else (label 255) ends up as one run at the tile's end, still in
// stream order, and the block's last warp sorts just that run by node (two warp-local 8-bit
// passes) while the other seven place the hub runs: a hub run's tile offset is its label's
// scanned start, so no run-head search is needed there.  Same shared memory as variant 43;
// scur holds each node's cursor with its cold flag in bit 31 (positions < 2^31).
template <int R, int TE, int S>
__global__ void __launch_bounds__(kBT, 2) k_scatter_hot(
    const tgfx_event* __restrict__ ev, int64_t n, int32_t V, int64_t chunk_ev,
    uint32_t* __restrict__ off, const uint32_t* __restrict__ coldbits,
    const uint8_t* __restrict__ hot, ulonglong2* __restrict__ cold_img,
    double* __restrict__ ts_out, uint4* __restrict__ rec_out, int64_t* __restrict__ nbr_out,
    int64_t* __restrict__ eid_out) {
  constexpr int NE = TE * R;
  constexpr int KPT = NE / kBT;
  constexpr int kW = kBT / 32;
  constexpr int kHubT = (kW - 1) * 32;           // hub-run threads (warps 0..kW-2)
  constexpr int HMAX = (NE + kHubT - 1) / kHubT;  // hub positions per thread
  constexpr int kCB = 8;                          // cold-sort rounds per MATCH batch
  static_assert(KPT * kBT == NE && NE <= 65536 && kW == 8, "tile shape");
  extern __shared__ __align__(128) unsigned char sm[];
  tgfx_event* stage = reinterpret_cast<tgfx_event*>(sm);
  uint32_t* keys0 = reinterpret_cast<uint32_t*>(sm + static_cast<size_t>(S) * TE * 32);
  uint32_t* keys1 = keys0 + NE;
  uint16_t* wcnt = reinterpret_cast<uint16_t*>(keys1 + NE);  // [kW][256]
  uint64_t* bars = reinterpret_cast<uint64_t*>(wcnt + kW * 256);
  int* scr = reinterpret_cast<int*>(bars + S);
  uint32_t* scur = reinterpret_cast<uint32_t*>(scr + 64);  // [vpad] cursor | cold << 31

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t e0 = static_cast<int64_t>(blockIdx.x) * chunk_ev;
  const int64_t e1 = min(n, e0 + chunk_ev);
  if (e0 >= e1) return;
  const int64_t ntiles = ceil_div(e1 - e0, TE);
  const uint32_t* crow = off + static_cast<int64_t>(blockIdx.x) * V;
  for (int i = tid; i < V; i += kBT) scur[i] = crow[i] | (((coldbits[i >> 5] >> (i & 31)) & 1u) << 31);
  if (tid == 0) {
    for (int q = 0; q < S; ++q) mbar_init(&bars[q], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid == 0) {
    for (int q = 0; q < S && q < ntiles; ++q) {
      const int64_t b = e0 + static_cast<int64_t>(q) * TE;
      const uint32_t bytes = static_cast<uint32_t>(min(static_cast<int64_t>(TE), e1 - b) * 32);
      mbar_arrive_tx(&bars[q], bytes);
      bulk_g2s(stage + q * TE, ev + b, bytes, &bars[q]);
    }
  }
  for (int64_t it = 0; it < ntiles; ++it) {
    const int sidx = static_cast<int>(it % S);
    const int64_t tb = e0 + it * TE;
    const int ent = static_cast<int>(min(static_cast<int64_t>(TE), e1 - tb)) * R;
    const tgfx_event* sev = stage + sidx * TE;
    mbar_wait(&bars[sidx], static_cast<uint32_t>((it / S) & 1));
    uint32_t key[KPT], dig[KPT], rank[KPT];
    unsigned peers[KPT];
#pragma unroll
    for (int k = 0; k < KPT; ++k) {
      const int j = warp * 32 * KPT + k * 32 + lane;
      uint32_t node = static_cast<uint32_t>(V);  // sentinel: label 255, sorts after every node
      if (j < ent) node = hot_node_of<R>(sev, j);
      key[k] = (node << 16) | static_cast<uint32_t>(j);
      dig[k] = node < static_cast<uint32_t>(V) ? __ldg(hot + node) : 255u;
    }
    // ---- one block-wide stable counting pass by label (as one pass of k_scatter_big)
    uint16_t* wc = wcnt + warp * 256;
    reinterpret_cast<uint4*>(wc)[lane] = make_uint4(0, 0, 0, 0);
    __syncwarp();
#pragma unroll
    for (int k = 0; k < KPT; ++k) peers[k] = __match_any_sync(kFull, dig[k]);
#pragma unroll
    for (int k = 0; k < KPT; ++k) {
      const uint32_t b = wc[dig[k]];
      __syncwarp();
      if (lane == __ffs(peers[k]) - 1) wc[dig[k]] = static_cast<uint16_t>(b + __popc(peers[k]));
      __syncwarp();
      rank[k] = b + __popc(peers[k] & lanemask_lt());
    }
    __syncthreads();
    {
      constexpr int kDT = 4;
      constexpr int kNT = 256 / kDT;
      uint2 v[kW];
      uint32_t tot = 0;
      if (tid < kNT) {
#pragma unroll
        for (int w = 0; w < kW; ++w) {
          v[w] = *reinterpret_cast<const uint2*>(wcnt + w * 256 + kDT * tid);
          tot += (v[w].x & 0xffffu) + (v[w].x >> 16) + (v[w].y & 0xffffu) + (v[w].y >> 16);
        }
      }
      uint32_t x = tot;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, x, o);
        if (lane >= o) x += y;
      }
      if (lane == 31 && warp == 0) scr[0] = static_cast<int>(x);
      __syncthreads();
      if (tid < kNT) {
        uint32_t run = (warp == 1 ? static_cast<uint32_t>(scr[0]) : 0u) + x - tot;
        uint32_t o[kW][kDT];
#pragma unroll
        for (int dd = 0; dd < kDT; ++dd) {
#pragma unroll
          for (int w = 0; w < kW; ++w) {
            const uint32_t word = dd < 2 ? v[w].x : v[w].y;
            const uint32_t c = (word >> (16 * (dd & 1))) & 0xffffu;
            o[w][dd] = run;
            run += c;
          }
        }
#pragma unroll
        for (int w = 0; w < kW; ++w)
          *reinterpret_cast<uint2*>(wcnt + w * 256 + kDT * tid) =
              make_uint2(o[w][0] | (o[w][1] << 16), o[w][2] | (o[w][3] << 16));
      }
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < KPT; ++k) keys1[wc[dig[k]] + rank[k]] = key[k];
    __syncthreads();
    // keys1: hub runs by label in [0, c0), the rest [c0, NE) in stream order.  wcnt row 0 =
    // each label's tile start (the scan is in (label, warp) order).
    const int c0 = wcnt[255];
    if (warp < kW - 1) {
      // ---- hub runs: position = cursor + offset from the label's start
      const int ht = warp * 32 + lane;
      uint32_t hk[HMAX], hp[HMAX], hc[HMAX];
      int hl[HMAX];
#pragma unroll
      for (int i = 0; i < HMAX; ++i) {
        const int sp = ht + kHubT * i;
        hl[i] = -1;
        if (sp < c0) {
          const uint32_t k2 = keys1[sp];
          const uint32_t u = k2 >> 16;
          const uint32_t d = __ldg(hot + u);
          const int r0 = wcnt[d];
          const uint32_t c = scur[u];
          hk[i] = k2;
          hc[i] = c;
          hp[i] = (c & 0x7fffffffu) + static_cast<uint32_t>(sp - r0);
          if (sp == r0) hl[i] = static_cast<int>(wcnt[d + 1]) - r0;  // run length (head only)
        }
      }
      named_bar_sync(1, kHubT);  // every hub cursor read before any is bumped
#pragma unroll
      for (int i = 0; i < HMAX; ++i) {
        const int sp = ht + kHubT * i;
        if (sp < c0) {
          const uint32_t u = hk[i] >> 16;
          if (hl[i] >= 0) scur[u] = hc[i] + static_cast<uint32_t>(hl[i]);
          write_entry_known<R>(sev, static_cast<int>(hk[i] & 0xffffu), hp[i], u,
                               (hc[i] >> 31) != 0, cold_img, ts_out, rec_out, nbr_out, eid_out);
        }
      }
    } else {
      // ---- the rest: one warp sorts [c0, NE) by node (two warp-local stable 8-bit passes)
      const int ncr = NE - c0;
      uint16_t* cnt = wcnt + (kW - 1) * 256;  // this warp's counter row
      uint16_t* rk = wcnt + 256;              // ranks: rows 1..kW-2 (hub warps read row 0 only)
      uint32_t* P = keys1 + c0;
      uint32_t* Q = keys0 + c0;
      for (int sh = 16; sh < 32; sh += 8) {
        reinterpret_cast<uint4*>(cnt)[lane] = make_uint4(0, 0, 0, 0);
        __syncwarp();
        for (int c0r = 0; c0r < ncr; c0r += 32 * kCB) {
          // kCB rounds' MATCH.ANYs issued back to back (their ~400-cycle latencies overlap),
          // then the counter chain round by round
          uint32_t dd[kCB];
          unsigned pe[kCB];
#pragma unroll
          for (int q = 0; q < kCB; ++q) {
            const int i = c0r + q * 32 + lane;
            dd[q] = i < ncr ? (P[i] >> sh) & 0xffu : 256u;
          }
#pragma unroll
          for (int q = 0; q < kCB; ++q) pe[q] = __match_any_sync(kFull, dd[q]);
#pragma unroll
          for (int q = 0; q < kCB; ++q) {
            const int i = c0r + q * 32 + lane;
            const bool valid = i < ncr;
            const uint32_t b = valid ? cnt[dd[q]] : 0u;
            __syncwarp();
            if (valid && lane == __ffs(pe[q]) - 1)
              cnt[dd[q]] = static_cast<uint16_t>(b + __popc(pe[q]));
            __syncwarp();
            if (valid) rk[i] = static_cast<uint16_t>(b + __popc(pe[q] & lanemask_lt()));
          }
        }
        __syncwarp();
        {  // exclusive scan of the 256 counters, 8 per lane
          uint4 w4 = reinterpret_cast<const uint4*>(cnt)[lane];
          uint32_t c8[8] = {w4.x & 0xffffu, w4.x >> 16, w4.y & 0xffffu, w4.y >> 16,
                            w4.z & 0xffffu, w4.z >> 16, w4.w & 0xffffu, w4.w >> 16};
          uint32_t t = 0;
#pragma unroll
          for (int q = 0; q < 8; ++q) t += c8[q];
          uint32_t xs = t;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(kFull, xs, o);
            if (lane >= o) xs += y;
          }
          uint32_t r = xs - t, e8[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            e8[q] = r;
            r += c8[q];
          }
          __syncwarp();
          reinterpret_cast<uint4*>(cnt)[lane] =
              make_uint4(e8[0] | (e8[1] << 16), e8[2] | (e8[3] << 16), e8[4] | (e8[5] << 16),
                         e8[6] | (e8[7] << 16));
          __syncwarp();
        }
        for (int c = 0; c < ncr; c += 32) {
          const int i = c + lane;
          if (i < ncr) {
            const uint32_t k2 = P[i];
            Q[cnt[(k2 >> sh) & 0xffu] + rk[i]] = k2;
          }
        }
        __syncwarp();
        uint32_t* t2 = P;
        P = Q;
        Q = t2;
      }
      // P: sorted by node; Q: head cursors.  Runs: the head reads the cursor, every entry
      // finds its head by a max-scan (carried across rounds), the tail bumps the cursor.
      int carry = -1;
      for (int c = 0; c < ncr; c += 32) {
        const int i = c + lane;
        const bool valid = i < ncr;
        const uint32_t k2 = valid ? P[i] : 0xffffffffu;
        const uint32_t u = k2 >> 16;
        const bool real = valid && u < static_cast<uint32_t>(V);
        const bool head = real && (i == 0 || (P[i - 1] >> 16) != u);
        if (head) Q[i] = scur[u];
        int xh = head ? i : -1;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(kFull, xh, o);
          if (lane >= o) xh = max(xh, y);
        }
        xh = max(xh, carry);
        carry = __shfl_sync(kFull, xh, 31);
        __syncwarp();
        if (real) {
          const uint32_t cur = Q[xh];
          const uint32_t pos = (cur & 0x7fffffffu) + static_cast<uint32_t>(i - xh);
          const bool tail = i == ncr - 1 || (P[i + 1] >> 16) != u;
          if (tail) scur[u] = cur + static_cast<uint32_t>(i - xh + 1);
          write_entry_known<R>(sev, static_cast<int>(k2 & 0xffffu), pos, u, (cur >> 31) != 0,
                               cold_img, ts_out, rec_out, nbr_out, eid_out);
        }
      }
    }
    __syncthreads();  // stage consumed; cursor stores ordered before the next tile's loads
    if (tid == 0 && it + S < ntiles) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      const int64_t b = e0 + (it + S) * TE;
      const uint32_t bytes = static_cast<uint32_t>(min(static_cast<int64_t>(TE), e1 - b) * 32);
      mbar_arrive_tx(&bars[sidx], bytes);
      bulk_g2s(stage + sidx * TE, ev + b, bytes, &bars[sidx]);
    }
  }
}

// ------------------------------------------------------------------ general path helpers
__device__ __forceinline__ uint64_t time_key(double t) {
  // total order of doubles consistent with operator< for non-NaN; -0.0 keyed as +0.0
  uint64_t b = static_cast<uint64_t>(__double_as_longlong(t == 0.0 ? 0.0 : t));
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

__global__ void k_sort_keys(const tgfx_event* __restrict__ ev, int64_t n, uint64_t* tkey,
                            uint64_t* ekey, uint32_t* idx) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const Ev x = load_event(ev, i);
    tkey[i] = time_key(x.t);
    ekey[i] = static_cast<uint64_t>(x.eid) ^ 0x8000000000000000ull;
    idx[i] = static_cast<uint32_t>(i);
  }
}

__global__ void k_gather_keys(const uint64_t* __restrict__ src, const uint32_t* __restrict__ idx,
                              int64_t n, uint64_t* dst) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = src[idx[i]];
}

__global__ void k_gather_events(const tgfx_event* __restrict__ ev,
                                const uint32_t* __restrict__ idx, int64_t n, tgfx_event* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = ev[idx[i]];
}

// ------------------------------------------------------------------ large-V path helpers
template <int R, typename K>
__global__ void k_entry_keys(const tgfx_event* __restrict__ ev, int64_t m, K* key,
                             uint32_t* val) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < m;
       j += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = R == 2 ? (j >> 1) : j;
    const bool side = R == 2 && (j & 1);
    const int64_t* p = reinterpret_cast<const int64_t*>(ev + e);
    key[j] = static_cast<K>(side ? p[2] : p[1]);
    val[j] = static_cast<uint32_t>(j);
  }
}

// each output position gathers its entry's event; with `rec` the entry goes out as the
// sampler's 16-byte gather record + ts (the int64 columns are widened on demand, as after the
// small-V scatter), else as the three reference columns
template <int R>
__global__ void k_gather_entries(const tgfx_event* __restrict__ ev,
                                 const uint32_t* __restrict__ val, int64_t m, int64_t* nbr,
                                 int64_t* eid, double* ts, uint4* __restrict__ rec) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < m;
       p += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t j = val[p];
    const int64_t e = R == 2 ? (j >> 1) : j;
    const bool side = R == 2 && (j & 1);
    Ev x;  // the event's one 32-byte sector in one load; L2::64B: without the hint L2 fetches
           // more around each random read (M16 build 9.19 -> 8.80 ms; 128B / 256B 9.18 / 9.36)
    {
      long long a0, a1, a2, a3;
      asm volatile("ld.global.nc.L1::no_allocate.L2::64B.v4.s64 {%0, %1, %2, %3}, [%4];"
                   : "=l"(a0), "=l"(a1), "=l"(a2), "=l"(a3) : "l"(ev + e));
      x.eid = a0;
      x.src = a1;
      x.dst = a2;
      x.t = __longlong_as_double(a3);
    }
    const int64_t other = side ? x.src : x.dst;
    ts[p] = x.t;
    if (rec) {
      const unsigned long long tb = static_cast<unsigned long long>(__double_as_longlong(x.t));
      rec[p] = make_uint4(static_cast<uint32_t>(other), static_cast<uint32_t>(x.eid),
                          static_cast<uint32_t>(tb), static_cast<uint32_t>(tb >> 32));
    } else {
      nbr[p] = other;
      eid[p] = x.eid;
    }
  }
}

// ------------------------------------------------------------------ node directory
// Slice time buckets (sampler search acceleration).  A sorted, NaN-free slice of n >=
// kBucketMinSlice entries with finite t_first < t_last gets nb = ceil(n / R) buckets of
// equal time width; bkt[j] = #entries e with bucket_of(ts[e]) < j, j = 0..nb.  bucket_of is
// monotone, so for t_first < t <= t_last and j = bucket_of(t) every entry before bkt[j] has
// ts < t and every entry from bkt[j + 1] on has ts > t: lower_bound(t) is in [bkt[j],
// bkt[j + 1]], typically a range of R entries -- one line probe instead of a chain of them.
constexpr int64_t kBucketMinSlice = 32;

__device__ __forceinline__ int64_t bucket_count(int64_t n, double t_first, double t_last,
                                                int64_t R, double* scale) {
  if (R <= 0 || n < kBucketMinSlice || n > 0x7fffffffLL) return 0;  // int bucket indices
  if (!(t_first < t_last) || isinf(t_first) || isinf(t_last)) return 0;
  const int64_t nb = ceil_div(n, R);
  const double sc = static_cast<double>(nb) / (t_last - t_first);
  if (!(sc < 1e300)) return 0;  // near-zero time span: no useful bucket grid
  *scale = sc;
  return nb;
}

// pass 1: directory records (bkt pointer filled in pass 2) and bucket table sizes
constexpr int kFillPer = 8;
constexpr int64_t kFillTile = 256 * kFillPer;

// directory records; a slice's bucket table at bkt + start / R + 2u (see DirC)
__global__ void k_node_dir(const int64_t* __restrict__ indptr, const double* __restrict__ ts,
                           int64_t V, int64_t R, NodeDir* __restrict__ dir,
                           DirC* __restrict__ dirc, uint32_t* __restrict__ bkt) {
  const int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (u >= V) return;
  const int64_t a = indptr[u], b = indptr[u + 1];
  NodeDir d;
  d.start = a;
  d.end = b;
  d.t_first = b > a ? ts[a] : 0.0;
  d.t_last = b > a ? ts[b - 1] : 0.0;
  d.bkt = nullptr;
  d.scale = 0.0;
  d.nb = bkt ? bucket_count(b - a, d.t_first, d.t_last, R, &d.scale) : 0;
  d.width = d.nb ? (d.t_last - d.t_first) / static_cast<double>(d.nb) : 0.0;
  if (d.nb) d.bkt = bkt + a / R + 2 * u;
  dir[u] = d;
  DirC c;
  c.start = a;
  c.n = static_cast<uint32_t>(b - a < 0xffffffffLL ? b - a : 0xffffffffLL);
  c.nb = static_cast<uint32_t>(d.nb);
  c.t_first = d.t_first;
  c.st = d.nb ? d.scale : d.t_last;
  dirc[u] = c;
}

// the node holding the first entry of each k_bucket_fill tile: last u with indptr[u] <= t * tile
__global__ void k_tile_node(const int64_t* __restrict__ indptr, int64_t V, int64_t tiles,
                            int32_t* __restrict__ tile_node) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= tiles) return;
  const int64_t i = t * kFillTile;
  int64_t lo = 0, n = V + 1;  // upper_bound over indptr[0..V]
  while (n > 0) {
    const int64_t h = n >> 1;
    if (__ldg(reinterpret_cast<const long long*>(indptr) + lo + h) <= i) {
      lo += h + 1;
      n -= h + 1;
    } else {
      n = h;
    }
  }
  tile_node[t] = static_cast<int32_t>(lo - 1);
}

// pass 3: one thread per slice entry writes the table entries of the buckets that start at
// it: bkt[j] = r for j in (bucket_of(ts[r - 1]), bucket_of(ts[r])], and bkt[nb] = n.  Tile
// t's node range starts at tile_node[t] and ends at or before tile_node[t + 1]; within it
// an entry's node is found by a bisection of indptr (tiles spanning several slices only).
__global__ void __launch_bounds__(256) k_bucket_fill(const int64_t* __restrict__ indptr,
                                                     const int64_t* __restrict__ nbr,
                                                     const int64_t* __restrict__ eid,
                                                     const double* __restrict__ ts,
                                                     const NodeDir* __restrict__ dir,
                                                     const int32_t* __restrict__ tile_node,
                                                     int64_t V, int64_t m, bool buckets,
                                                     uint4* __restrict__ rec) {
  const int64_t i0 = static_cast<int64_t>(blockIdx.x) * kFillTile;
  if (i0 >= m) return;
  const int64_t i1 = min(i0 + kFillTile, m) - 1;
  double x[kFillPer];
#pragma unroll
  for (int k = 0; k < kFillPer; ++k) {
    const int64_t i = i0 + k * 256 + threadIdx.x;
    x[k] = i <= i1 ? ts[i] : 0.0;
  }
  if (rec) {  // gather records of the tile's entries (coalesced 16-byte stores)
#pragma unroll
    for (int k = 0; k < kFillPer; ++k) {
      const int64_t i = i0 + k * 256 + threadIdx.x;
      if (i > i1) break;
      const unsigned long long tb = static_cast<unsigned long long>(__double_as_longlong(x[k]));
      __stcs(rec + i, make_uint4(static_cast<uint32_t>(nbr[i]), static_cast<uint32_t>(eid[i]),
                                 static_cast<uint32_t>(tb), static_cast<uint32_t>(tb >> 32)));
    }
  }
  if (!buckets) return;
  const int64_t v0 = tile_node[blockIdx.x];
  const int64_t v1 = i1 + 1 < m ? tile_node[blockIdx.x + 1] : V - 1;
  if (dir[v0].end > i1) {  // the whole tile lies in one slice (hub slices): no node search
    const NodeDir d = dir[v0];
    if (!d.nb) return;
    uint32_t* bkt = const_cast<uint32_t*>(d.bkt);
    const int lane = threadIdx.x & 31;
    // 32-bit slice-relative indices (slices with buckets have < 2^31 entries)
    const uint32_t r0 = static_cast<uint32_t>(i0 - d.start);
    const int cnt = static_cast<int>(i1 - i0 + 1);
    const uint32_t last = static_cast<uint32_t>(d.end - d.start - 1);
    const double nbm1 = static_cast<double>(d.nb - 1);
    const auto bucket = [&](double t) -> uint32_t {  // bucket_of, with nb - 1 hoisted
      const double xx = __dmul_rn(__dsub_rn(t, d.t_first), d.scale);
      return xx < nbm1 ? static_cast<uint32_t>(xx) : static_cast<uint32_t>(d.nb - 1);
    };
    // the bucket of the entry before the tile's first one (lane 0, k = 0 needs it)
    const int jprev0 = r0 ? static_cast<int>(bucket(ts[i0 - 1])) : -1;
#pragma unroll
    for (int k = 0; k < kFillPer; ++k) {
      const int o = k * 256 + static_cast<int>(threadIdx.x);
      const bool live = o < cnt;
      const uint32_t jr = live ? bucket(x[k]) : 0u;
      int jp = static_cast<int>(__shfl_up_sync(0xffffffffu, jr, 1));  // every lane, every k
      if (!live) continue;
      const uint32_t r = r0 + static_cast<uint32_t>(o);
      if (lane == 0) jp = o == 0 ? jprev0 : static_cast<int>(bucket(ts[i0 + o - 1]));
#pragma unroll 1
      for (int j = jp + 1; j <= static_cast<int>(jr); ++j) bkt[j] = r;
      if (r == last) bkt[d.nb] = last + 1;
    }
    return;
  }
#pragma unroll
  for (int k = 0; k < kFillPer; ++k) {
    const int64_t i = i0 + k * 256 + threadIdx.x;
    if (i > i1) break;
    int64_t lo = v0, n = v1 - v0 + 2;  // upper_bound over indptr[v0..v1+1]
    while (n > 0) {
      const int64_t h = n >> 1;
      if (__ldg(reinterpret_cast<const long long*>(indptr) + lo + h) <= i) {
        lo += h + 1;
        n -= h + 1;
      } else {
        n = h;
      }
    }
    const NodeDir& d = dir[lo - 1];
    if (!d.nb) continue;
    uint32_t* bkt = const_cast<uint32_t*>(d.bkt);
    const uint32_t r = static_cast<uint32_t>(i - d.start);
    const int jr = static_cast<int>(bucket_of(x[k], d.t_first, d.scale, d.nb));
    const int jp = r ? static_cast<int>(bucket_of(ts[i - 1], d.t_first, d.scale, d.nb)) : -1;
#pragma unroll 1
    for (int j = jp + 1; j <= jr; ++j) bkt[j] = r;
    if (i == d.end - 1) bkt[d.nb] = static_cast<uint32_t>(d.end - d.start);
  }
}

// pass 3 (default): the same table, each thread walking 8 consecutive entries, so an entry's
// predecessor bucket is the previous entry's (a register) and the write loop runs per thread.
// The node of every entry comes from the tile's head marks (one max-scan per tile) instead of
// a per-entry search of indptr; tiles inside one slice (the hubs) skip even that.
__global__ void __launch_bounds__(256, 6) k_bucket_fill8(const int64_t* __restrict__ indptr,
                                                      const int64_t* __restrict__ nbr,
                                                      const int64_t* __restrict__ eid,
                                                      const double* __restrict__ ts,
                                                      const NodeDir* __restrict__ dir,
                                                      const int32_t* __restrict__ tile_node,
                                                      int64_t V, int64_t m, bool buckets,
                                                      uint4* __restrict__ rec) {
  constexpr int P = 8;
  static_assert(P * 256 == kFillTile, "tile");
  __shared__ int32_t mark[kFillTile];
  __shared__ int32_t wmax[8];
  __shared__ double wts[8];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t i0 = static_cast<int64_t>(blockIdx.x) * kFillTile;
  if (i0 >= m) return;
  const int64_t i1 = min(i0 + kFillTile, m) - 1;
  const int cnt = static_cast<int>(i1 - i0 + 1);
  const int64_t b0 = i0 + static_cast<int64_t>(tid) * P;
  double x[P];
  if (b0 + P - 1 <= i1) {  // 64-byte aligned: two 32-byte loads (one L1 wavefront per sector)
#pragma unroll
    for (int k = 0; k < P; k += 4)
      asm volatile("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];"
                   : "=d"(x[k]), "=d"(x[k + 1]), "=d"(x[k + 2]), "=d"(x[k + 3])
                   : "l"(ts + b0 + k));
  } else {
#pragma unroll
    for (int k = 0; k < P; ++k) x[k] = b0 + k <= i1 ? ts[b0 + k] : 0.0;
  }
  if (rec) {
#pragma unroll
    for (int k = 0; k < P; ++k) {
      const int64_t i = b0 + k;
      if (i > i1) continue;  // (no break: it keeps the loop, and x[], from being unrolled)
      const unsigned long long tb = static_cast<unsigned long long>(__double_as_longlong(x[k]));
      __stcs(rec + i, make_uint4(static_cast<uint32_t>(nbr[i]), static_cast<uint32_t>(eid[i]),
                                 static_cast<uint32_t>(tb), static_cast<uint32_t>(tb >> 32)));
    }
  }
  if (!buckets) return;
  const int32_t v0 = tile_node[blockIdx.x];
  const int32_t v1 = i1 + 1 < m ? tile_node[blockIdx.x + 1] : static_cast<int32_t>(V - 1);
  // ts of the entry before this thread's first one
  double xprev = __shfl_up_sync(kFull, x[P - 1], 1);
  if (lane == 31) wts[warp] = x[P - 1];
  int32_t first = v0;  // node of this thread's first entry
  const NodeDir d0 = dir[v0];
  const bool hub = d0.end > i1;
  if (hub) {
    // the whole tile lies in one slice (the hubs, most of the entries): 32-bit slice-relative
    // indices, no node bookkeeping -- a dozen instructions per entry
    __syncthreads();  // wts
    if (!d0.nb) return;
    if (lane == 0) xprev = warp ? wts[warp - 1] : (i0 > 0 ? ts[i0 - 1] : 0.0);
    uint32_t* bkt = const_cast<uint32_t*>(d0.bkt);
    const uint32_t nb = static_cast<uint32_t>(d0.nb);
    const double nbm1 = static_cast<double>(nb - 1);
    const auto bucket = [&](double t) -> int {  // bucket_of, with nb - 1 hoisted
      const double xx = __dmul_rn(__dsub_rn(t, d0.t_first), d0.scale);
      return static_cast<int>(xx < nbm1 ? static_cast<uint32_t>(xx) : nb - 1);
    };
    const uint32_t r0 = static_cast<uint32_t>(b0 - d0.start);
    const uint32_t last = static_cast<uint32_t>(d0.end - d0.start - 1);
    const int live = min(P, cnt - tid * P);  // entries of this thread
    int jprev = (live > 0 && r0 > 0) ? bucket(xprev) : -1;
#pragma unroll
    for (int k = 0; k < P; ++k) {
      if (k >= live) continue;
      const uint32_t r = r0 + static_cast<uint32_t>(k);
      const int jr = bucket(x[k]);
      if (jr > jprev) bkt[jprev + 1] = r;
      for (int j = jprev + 2; j <= jr; ++j) bkt[j] = r;
      jprev = jr;
      if (r == last) bkt[nb] = r + 1;
    }
    return;
  }
  {
    for (int q = tid; q < cnt; q += 256) mark[q] = -1;
    __syncthreads();
    for (int32_t u = v0 + 1 + tid; u <= v1; u += 256) {
      const int64_t a = indptr[u];
      if (a > i0 && a <= i1 && indptr[u + 1] > a) mark[a - i0] = u;
    }
    __syncthreads();
    int32_t run = -1;
#pragma unroll
    for (int k = 0; k < P; ++k) {
      const int q = tid * P + k;
      if (q < cnt) run = max(run, mark[q]);
    }
    int32_t inc = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int32_t y = __shfl_up_sync(kFull, inc, o);
      if (lane >= o) inc = max(inc, y);
    }
    if (lane == 31) wmax[warp] = inc;
    __syncthreads();
    int32_t ex = __shfl_up_sync(kFull, inc, 1);
    if (lane == 0) ex = -1;
    for (int w = 0; w < warp; ++w) ex = max(ex, wmax[w]);
    first = max(v0, ex);  // node owning position tid*P (before this thread's own marks)
  }
  if (lane == 0) xprev = warp ? wts[warp - 1] : (i0 > 0 ? ts[i0 - 1] : 0.0);
  int32_t u = first;
  NodeDir d = first == v0 ? d0 : dir[u];
  int jprev = -1;  // bucket of the previous entry of the same slice
  {
    const int64_t i = b0;
    if (i <= i1 && i > d.start && d.nb) jprev = static_cast<int>(bucket_of(xprev, d.t_first, d.scale, d.nb));
  }
#pragma unroll
  for (int k = 0; k < P; ++k) {
    const int64_t i = b0 + k;
    if (i > i1) continue;
    {
      const int32_t mk = mark[tid * P + k];
      if (mk >= 0 && mk != u) {  // a new slice starts here
        u = mk;
        d = dir[u];
        jprev = -1;
      }
    }
    if (!d.nb) continue;
    const uint32_t r = static_cast<uint32_t>(i - d.start);
    const int jr = static_cast<int>(bucket_of(x[k], d.t_first, d.scale, d.nb));
    uint32_t* bkt = const_cast<uint32_t*>(d.bkt);
    // usually at most one bucket starts at an entry: one predicated store, the loop only for
    // the rest of a run of empty buckets
    if (jr > jprev) bkt[jprev + 1] = r;
    for (int j = jprev + 2; j <= jr; ++j) bkt[j] = r;
    jprev = jr;
    if (i == d.end - 1) bkt[d.nb] = r + 1;
  }
}

// ------------------------------------------------------------------ validate (tcsr.cpp:54-81)
// The reference walks nodes in order (indptr monotone at u, then slice u sorted), then entries
// in order (neighbour id, then edge id); the first failure is the one thrown.  Here every check
// runs in parallel and reduces to the first failure in that same order:
//   node_fail = min u whose slice is unsorted (only slices below the first non-monotone node
//               u_mono, which the host finds in its copy of indptr, can be walked);
//   entry_fail = min (2 i + which) over entries with an id out of range.
// An entry pair (i-1, i) out of order lies in one slice unless a slice starts at i; the node
// owning i (upper_bound over the monotone indptr prefix) is looked up only for such pairs, so
// at most V + #failures searches run.
__global__ void k_validate(const int64_t* __restrict__ indptr, const int64_t* __restrict__ nbr,
                           const int64_t* __restrict__ eid, const double* __restrict__ ts,
                           int64_t u_mono, int64_t Vn, int64_t E, int64_t m,
                           unsigned long long* __restrict__ node_fail,
                           unsigned long long* __restrict__ entry_fail) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t t0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  // entries walked by the node loop: [0, indptr[u_mono]) (indptr[0..u_mono] is monotone)
  const int64_t top = __ldg(reinterpret_cast<const long long*>(indptr) + u_mono);
  const int64_t walked = top < 0 ? 0 : (top < m ? top : m);
  for (int64_t i = t0; i < m; i += stride) {
    const int64_t nb = nbr[i], e = eid[i];
    if (nb < 0 || nb >= Vn) atomicMin(entry_fail, 2ull * static_cast<unsigned long long>(i));
    else if (e < 0 || e >= E) atomicMin(entry_fail, 2ull * static_cast<unsigned long long>(i) + 1);
    if (i >= 1 && i < walked) {
      const double a = ts[i - 1], c = ts[i];
      if (a > c || (a == c && eid[i - 1] > e)) {
        int64_t lo = 0, n = u_mono + 1;  // upper_bound(indptr[0..u_mono], i) - 1
        while (n > 0) {
          const int64_t h = n >> 1;
          if (__ldg(reinterpret_cast<const long long*>(indptr) + lo + h) <= i) {
            lo += h + 1;
            n -= h + 1;
          } else {
            n = h;
          }
        }
        const int64_t u = lo - 1;
        if (u >= 0 && u < u_mono && indptr[u] < i)  // i - 1 is in the same slice
          atomicMin(node_fail, static_cast<unsigned long long>(u));
      }
    }
  }
}

int grid_for(int64_t work, int threads, int per_sm = 8) {
  const int64_t g = ceil_div(std::max<int64_t>(work, 1), threads);
  return static_cast<int>(std::min<int64_t>(g, static_cast<int64_t>(device_info().sms) * per_sm));
}

// gather records (tgfx_graph::rec) unless TGFX_GATHER_REC=0; ids must fit 31 bits
static bool rec_enabled() {
  static const bool on = [] {
    const char* e = getenv("TGFX_GATHER_REC");
    return !(e && e[0] == '0');
  }();
  return on;
}

static uint4* ensure_rec(tgfx_graph* g, cudaStream_t s) {
  if (!rec_enabled() || g->m <= 0 || g->other_limit >= (1LL << 31) ||
      g->eid_limit >= (1LL << 31)) {
    if (g->rec) dfree(g->rec, s);
    g->rec = nullptr;
    g->rec_cap = 0;
    return nullptr;
  }
  if (g->rec_cap < g->m) {
    if (g->rec) dfree(g->rec, s);
    g->rec = static_cast<uint4*>(dmalloc(sizeof(uint4) * g->m, s));
    g->rec_cap = g->m;
  }
  return g->rec;
}


size_t scatter_smem(int64_t V) {
  const int64_t vpad = (V + 31) & ~31LL;
  return static_cast<size_t>(vpad * 4 + vpad / 8) + 16;
}

// grow-only workspace buffer owned by the graph
void* ws_get(void*& p, size_t& have, size_t need, cudaStream_t s) {
  if (have < need) {
    if (p) dfree(p, s);
    p = dmalloc(need, s);
    have = need;
  }
  return p;
}

int64_t cold_theta() {
  // entries-per-chunk threshold below which a node's entries take the cold (deferred) path
  static int64_t theta = [] {
    const char* e = getenv("TGFX_COLD_THETA");
    return e ? atoll(e) : 300LL;
  }();
  return theta;
}

// TGFX_LARGE_FUSE=0: the large-V build's keys and histograms in their own passes (A/B)
bool large_fuse_enabled() {
  static const bool on = [] {
    const char* e = getenv("TGFX_LARGE_FUSE");
    return !(e && e[0] == '0');
  }();
  return on;
}

int scatter_variant() {
  static int v = [] {
    const char* e = getenv("TGFX_SCATTER_VARIANT");
    return e ? atoi(e) : 43;
  }();
  return v;
}

// tile-sorted scatter shape (threads, events per tile), TGFX_SCATTER_VARIANT=10 (default).
// Measured on the GDELT shape: 256 x 256 (2 CTAs/SM) 12.3 ms build, 512 x 512 (1 CTA/SM)
// 12.9 ms, 256 x 512 12.0 ms but 1 CTA/SM on larger V, 128 x 128 16.7 ms.
#define TGFX_TILE_SHAPES(X) X(10, 256, 256)

// the tile-kernel shape in use (the default shape when a big-tile variant is selected but the
// graph falls back to the tile kernel)
int tile_variant() { return scatter_variant() >= 40 ? 10 : scatter_variant(); }

size_t tile_smem_for(int64_t V) {
  const int v = tile_variant();
#define X(ID, TT, TE) \
  if (v == ID) return tile_scatter_smem<TT, TE>(V);
  TGFX_TILE_SHAPES(X)
#undef X
  return 0;
}

thread_local int64_t t_build_m = 0;

// big-tile scatter shapes: variant -> (events per tile, stages, cursors in shared memory).
// 43 (default): 512-event tiles, 2 stages, shared-memory cursors -- 2 CTAs/SM up to V ~ 16.7 K
// (GDELT shape); when that leaves fewer than 2 CTAs per SM the cursors move to L2 (42).
#define TGFX_BIG_SHAPES(X) X(40, 1024, 2, false) X(41, 512, 3, false) X(42, 512, 2, false) \
  X(43, 512, 2, true) X(44, 256, 4, true) X(45, 256, 3, true)

template <int R, int TE, int S, bool SC>
int big_bps_t(int64_t V) {
  const size_t smem = big_smem<R, TE, S, SC>(V);
  if (smem > static_cast<size_t>(device_info().smem_optin)) return 0;
  int bps = 0;
  TGFX_CUDA(cudaFuncSetAttribute(k_scatter_big<R, TE, S, SC>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  TGFX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, k_scatter_big<R, TE, S, SC>, kBT, smem));
  return bps;
}

int big_bps(int R, int v, int64_t V) {
  if (v == 50) v = 43;  // k_scatter_hot: variant 43's tile shape and shared memory
#define X(ID, TE, S, SC) \
  if (v == ID) return R == 2 ? big_bps_t<2, TE, S, SC>(V) : big_bps_t<1, TE, S, SC>(V);
  TGFX_BIG_SHAPES(X)
#undef X
  return 0;
}

// the big-tile variant this build uses, 0 if none (node ids 0..V must fit the 16-bit key field)
int big_variant(int R, int64_t V) {
  int v = scatter_variant();
  if (v == 50) {  // one-pass hot-label scatter: variant 43's shared memory; else 43's fallbacks
    if (V <= 65534 && t_build_m < (int64_t(1) << 31) && big_bps(R, 43, V) >= 2) return 50;
    v = 43;
  }
  if (v < 40 || v > 45 || V > 65534 || t_build_m >= (int64_t(1) << 32)) return 0;
  if (v == 43 && big_bps(R, 43, V) < 2) {
    // shared-memory cursors would leave one CTA per SM: the 256-event tile kernel when its
    // cursors fit (measured faster there, e.g. V = 40 K), else cursors in L2 (42)
    const size_t tsm = tile_scatter_smem<256, 256>(V);
    if (V <= 65535 && tsm <= static_cast<size_t>(device_info().smem_optin)) return 0;
    v = 42;
  }
  return big_bps(R, v, V) >= 1 ? v : 0;
}

bool use_big_scatter(int64_t V, int R) { return big_variant(R, V) != 0; }

bool use_tile_scatter(int64_t V, int R) {
  if (use_big_scatter(V, R)) return false;
  const size_t sm = tile_smem_for(V);
  return sm > 0 && V <= 65535 && sm <= static_cast<size_t>(device_info().smem_optin);
}

template <int R, int TT, int TE>
int tile_bps_t(int64_t V) {
  const size_t smem = tile_scatter_smem<TT, TE>(V);
  int bps = 0;
  TGFX_CUDA(cudaFuncSetAttribute(k_scatter_tile<R, TT, TE>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(smem)));
  TGFX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, k_scatter_tile<R, TT, TE>, TT, smem));
  return std::max(bps, 1);
}

int tile_bps(int R, int64_t V) {
  const int v = tile_variant();
#define X(ID, TT, TE) \
  if (v == ID) return R == 2 ? tile_bps_t<2, TT, TE>(V) : tile_bps_t<1, TT, TE>(V);
  TGFX_TILE_SHAPES(X)
#undef X
  return 1;
}

// (rounds, warps) variants of the ticketed scatter
#define TGFX_SCATTER_VARIANTS(X) \
  X(0, 8, 8)                     \
  X(1, 4, 8)                     \
  X(2, 4, 16)                    \
  X(3, 16, 8)                    \
  X(4, 8, 4)                     \
  X(5, 2, 16)

template <int R, int RO, int W>
int scatter_bps(int64_t V) {
  const size_t smem = scatter_smem(V);
  int bps = 0;
  TGFX_CUDA(cudaFuncSetAttribute(k_scatter<R, RO, W>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(smem)));
  TGFX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, k_scatter<R, RO, W>, W * 32, smem));
  return std::max(bps, 1);
}

// ticketed-scatter variant for graphs the tile kernel does not take (0 unless overridden)
int ticket_variant() {
  const int v = scatter_variant();
  return v >= 0 && v <= 5 ? v : 0;
}

int scatter_blocks_per_sm(int R, int64_t V) {
  if (const int v = big_variant(R, V)) return big_bps(R, v, V);
  if (use_tile_scatter(V, R)) return tile_bps(R, V);
  const int v = ticket_variant();
#define X(ID, RO, W) \
  if (v == ID) return R == 2 ? scatter_bps<2, RO, W>(V) : scatter_bps<1, RO, W>(V);
  TGFX_SCATTER_VARIANTS(X)
#undef X
  return R == 2 ? scatter_bps<2, 8, 8>(V) : scatter_bps<1, 8, 8>(V);
}

void read_flags(tgfx_graph* g, cudaStream_t s) {
  TGFX_CUDA(cudaMemcpyAsync(g->hflags, g->dflags, sizeof(BuildFlags), cudaMemcpyDeviceToHost, s));
  TGFX_CUDA(cudaStreamSynchronize(s));
}

void throw_bad_endpoint(tgfx_graph* g, const tgfx_event* d_ev, cudaStream_t s) {
  int64_t eid = 0;
  TGFX_CUDA(cudaMemcpyAsync(&eid, &d_ev[g->hflags->bad_index].edge_id, sizeof(int64_t),
                            cudaMemcpyDeviceToHost, s));
  TGFX_CUDA(cudaStreamSynchronize(s));
  // check_endpoints (tcsr.cpp:44-50): first offending event in stream order
  throw Error(TGFX_EVALIDATION, "event " + std::to_string(eid) + " endpoint out of range");
}

void run_flags_pass(tgfx_graph* g, const tgfx_event* d_ev, int C, int64_t chunk_ev,
                    uint32_t* cnt, bool hist, cudaStream_t s) {
  const int64_t V = g->V;
  k_init_flags<<<1, 1, 0, s>>>(g->dflags);
  after_launch("k_init_flags");
  const size_t smem = hist ? sizeof(uint32_t) * static_cast<size_t>(V) : 0;
  if (hist) {
    if (g->reverse) {
      TGFX_CUDA(cudaFuncSetAttribute(k_hist<2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(smem)));
      k_hist<2, true><<<C, kHistThreads, smem, s>>>(d_ev, g->n, V, V, chunk_ev, cnt, g->dflags);
    } else {
      TGFX_CUDA(cudaFuncSetAttribute(k_hist<1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(smem)));
      k_hist<1, true><<<C, kHistThreads, smem, s>>>(d_ev, g->n, V, g->other_limit, chunk_ev, cnt,
                                                    g->dflags);
    }
  } else {
    k_hist<1, false><<<C, kHistThreads, 0, s>>>(d_ev, g->n, V, g->reverse ? V : g->other_limit,
                                                 chunk_ev, nullptr, g->dflags);
  }
  after_launch("k_hist");
}

// sort a copy of the events by (t, eid) (stable LSD: eid first, then time key)
tgfx_event* sorted_copy(const tgfx_event* d_ev, int64_t n, cudaStream_t s) {
  uint64_t* tkey = static_cast<uint64_t*>(dmalloc(sizeof(uint64_t) * n, s));
  uint64_t* ekey = static_cast<uint64_t*>(dmalloc(sizeof(uint64_t) * n, s));
  uint64_t* kalt = static_cast<uint64_t*>(dmalloc(sizeof(uint64_t) * n, s));
  uint32_t* idx = static_cast<uint32_t*>(dmalloc(sizeof(uint32_t) * n, s));
  uint32_t* ialt = static_cast<uint32_t*>(dmalloc(sizeof(uint32_t) * n, s));
  const int grid = grid_for(n, 256);
  k_sort_keys<<<grid, 256, 0, s>>>(d_ev, n, tkey, ekey, idx);
  after_launch("k_sort_keys");
  uint64_t* k = ekey;
  uint32_t* v = idx;
  radix_sort_pairs<uint64_t, uint32_t>(k, v, kalt, ialt, n, 64, s);
  // now v = permutation sorted by eid; sort by time key stably
  uint64_t* k2 = (k == ekey) ? kalt : ekey;  // free buffer for gathered time keys
  k_gather_keys<<<grid, 256, 0, s>>>(tkey, v, n, k2);
  after_launch("k_gather_keys");
  uint64_t* kk = k2;
  uint32_t* vv = v;
  uint64_t* kalt2 = tkey;
  uint32_t* valt2 = (v == idx) ? ialt : idx;
  radix_sort_pairs<uint64_t, uint32_t>(kk, vv, kalt2, valt2, n, 64, s);
  tgfx_event* out = static_cast<tgfx_event*>(dmalloc(sizeof(tgfx_event) * n, s));
  k_gather_events<<<grid, 256, 0, s>>>(d_ev, vv, n, out);
  after_launch("k_gather_events");
  dfree(tkey, s);
  dfree(ekey, s);
  dfree(kalt, s);
  dfree(idx, s);
  dfree(ialt, s);
  return out;
}

// TGFX_TRACE=1: host-side phase timers of build_graph on stderr (each phase synchronised)
static bool build_trace() {
  static const bool on = [] {
    const char* e = getenv("TGFX_TRACE");
    return e && e[0] == '1';
  }();
  return on;
}
static double trace_ms(cudaStream_t s) {
  if (build_trace()) cudaStreamSynchronize(s);
  return std::chrono::duration<double, std::milli>(
             std::chrono::steady_clock::now().time_since_epoch()).count();
}

void build_fast(tgfx_graph* g, const tgfx_event* d_ev, int C, int64_t chunk_ev, uint32_t* cnt,
                cudaStream_t s) {
  const int32_t V = static_cast<int32_t>(g->V);
  const int tb = 256;
  const int vb = static_cast<int>(ceil_div(std::max<int64_t>(V, 1), tb));
  const int64_t vpad = (static_cast<int64_t>(V) + 31) & ~31LL;
  // small workspace: cold bitmask [vpad/32] u32 | cdelta [V] i64 | ncold i64
  const int64_t cb = (4 * (vpad / 32) + 15) & ~15LL;
  char* small = static_cast<char*>(
      ws_get(g->ws_small, g->ws_small_bytes, cb + 8 * (vpad + 2) + vpad, s));
  uint32_t* coldbits = reinterpret_cast<uint32_t*>(small);
  int64_t* cdelta = reinterpret_cast<int64_t*>(small + cb);
  int64_t* ncold_d = cdelta + vpad;
  uint8_t* hot = reinterpret_cast<uint8_t*>(small + cb + 8 * (vpad + 2));  // variant 50 labels
  const int R = g->reverse ? 2 : 1;
  int bigv = big_variant(R, V);
  if (V > 0) {
    k_colsum<<<vb, tb, 0, s>>>(cnt, C, V, g->indptr);
    after_launch("k_colsum");
    k_coldflags<<<static_cast<int>(ceil_div(vpad, tb)), tb, 0, s>>>(g->indptr, V,
                                                                     cold_theta() * C, coldbits);
    after_launch("k_coldflags");
    if (bigv == 50) {  // degrees are still in indptr here
      k_hot_labels<<<1, 1024, 0, s>>>(g->indptr, V, coldbits, hot);
      after_launch("k_hot_labels");
    }
  }
  k_indptr_scan<<<1, 1024, 0, s>>>(g->indptr, V, coldbits, cdelta, ncold_d);
  after_launch("k_indptr_scan");
  if (V > 0) {
    k_coloff<<<vb, tb, 0, s>>>(cnt, C, V, g->indptr, coldbits, cdelta,
                               (bigv || use_tile_scatter(V, R)) ? 1 : 0);
    after_launch("k_coloff");
  }
  int64_t ncold = 0;
  TGFX_CUDA(cudaMemcpyAsync(&ncold, ncold_d, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  TGFX_CUDA(cudaStreamSynchronize(s));
  const double tf0 = trace_ms(s);
  ulonglong2* img = static_cast<ulonglong2*>(
      ws_get(g->ws_rec, g->ws_rec_bytes, 32 * static_cast<size_t>(std::max<int64_t>(ncold, 1)), s));
  const double tf1 = trace_ms(s);
  if (g->n == 0) return;
  if (bigv) {
    // with gather records the scatter writes {rec, ts} instead of {nbr, eid, ts}; the int64
    // columns are widened from the records when something asks for them (ensure_columns)
    uint4* rec = ensure_rec(g, s);
    g->cols_valid = rec == nullptr;
    int bits = 1;
    while ((int64_t(1) << bits) <= V) ++bits;  // node ids 0..V (V = tail sentinel)
    const int passes = (bits + 7) / 8;
    const int cflag = std::max(g->m, ncold) < (int64_t(1) << 31) ? 1 : 0;
    if (bigv == 50 && cflag) {
      static const bool attr = [&] {
        TGFX_CUDA(cudaFuncSetAttribute(k_scatter_hot<2, 512, 2>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(device_info().smem_optin)));
        TGFX_CUDA(cudaFuncSetAttribute(k_scatter_hot<1, 512, 2>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(device_info().smem_optin)));
        return true;
      }();
      (void)attr;
      if (g->reverse)
        k_scatter_hot<2, 512, 2><<<C, kBT, big_smem<2, 512, 2, true>(V), s>>>(
            d_ev, g->n, V, chunk_ev, cnt, coldbits, hot, img, g->ts, rec, g->nbr, g->eid);
      else
        k_scatter_hot<1, 512, 2><<<C, kBT, big_smem<1, 512, 2, true>(V), s>>>(
            d_ev, g->n, V, chunk_ev, cnt, coldbits, hot, img, g->ts, rec, g->nbr, g->eid);
      after_launch("k_scatter_hot");
    } else if (bigv == 50) {
      bigv = 43;
    }
#define X(ID, TE, S, SC)                                                                       \
    if (bigv == ID) {                                                                          \
      if (g->reverse)                                                                          \
        k_scatter_big<2, TE, S, SC><<<C, kBT, big_smem<2, TE, S, SC>(V), s>>>(                 \
            d_ev, g->n, V, chunk_ev, passes, cnt, coldbits, img, g->ts, rec, g->nbr, g->eid,   \
            cflag);                                                                             \
      else                                                                                     \
        k_scatter_big<1, TE, S, SC><<<C, kBT, big_smem<1, TE, S, SC>(V), s>>>(                 \
            d_ev, g->n, V, chunk_ev, passes, cnt, coldbits, img, g->ts, rec, g->nbr, g->eid,   \
            cflag);                                                                             \
    }
    if (bigv != 50) {
      TGFX_BIG_SHAPES(X)
      after_launch("k_scatter_big");
    }
#undef X
    if (ncold > 0) {
      k_cold_u<<<resident_grid(k_cold_u, 256, 0, ncold), 256, 0, s>>>(img, ncold, cdelta, g->nbr,
                                                                      g->eid, g->ts, rec);
      after_launch("k_cold_u");
    }
    return;
  }
  if (use_tile_scatter(V, R)) {
    // with gather records the scatter writes {rec, ts} instead of {nbr, eid, ts}; the int64
    // columns are widened from the records when something asks for them (ensure_columns)
    uint4* rec = ensure_rec(g, s);
    g->cols_valid = rec == nullptr;
    const double tf2 = trace_ms(s);
    const size_t tsm = tile_smem_for(V);
    int bits = 1;
    while ((int64_t(1) << bits) <= V) ++bits;  // node ids 0..V (V = tail sentinel)
    const int passes = (bits + 7) / 8;
    const int v = tile_variant();
#define X(ID, TT, TE)                                                                        \
  if (v == ID) {                                                                             \
    if (g->reverse)                                                                          \
      k_scatter_tile<2, TT, TE><<<C, TT, tsm, s>>>(d_ev, g->n, V, chunk_ev, passes, cnt,     \
                                                   coldbits, cdelta, img, g->nbr, g->eid,    \
                                                   g->ts, rec);                              \
    else                                                                                     \
      k_scatter_tile<1, TT, TE><<<C, TT, tsm, s>>>(d_ev, g->n, V, chunk_ev, passes, cnt,     \
                                                   coldbits, cdelta, img, g->nbr, g->eid,    \
                                                   g->ts, rec);                              \
  }
    TGFX_TILE_SHAPES(X)
#undef X
    after_launch("k_scatter_tile");
    if (ncold > 0) {
      k_cold_u<<<resident_grid(k_cold_u, 256, 0, ncold), 256, 0, s>>>(img, ncold, cdelta, g->nbr,
                                                                      g->eid, g->ts, rec);
      after_launch("k_cold_u");
    }
    if (build_trace())
      fprintf(stderr, "[tgfx] build_fast: cold image alloc %.1f ms, records alloc %.1f ms, "
                      "scatter %.1f ms\n", tf1 - tf0, tf2 - tf1, trace_ms(s) - tf2);
    return;
  }
  const size_t smem = scatter_smem(V);
  const int v = ticket_variant();
#define X(ID, RO, W)                                                                             \
  if (v == ID) {                                                                                 \
    if (g->reverse)                                                                              \
      k_scatter<2, RO, W><<<C, W * 32, smem, s>>>(d_ev, g->n, V, chunk_ev, cnt, coldbits, cdelta, \
                                                  img, g->nbr, g->eid, g->ts);                   \
    else                                                                                         \
      k_scatter<1, RO, W><<<C, W * 32, smem, s>>>(d_ev, g->n, V, chunk_ev, cnt, coldbits, cdelta, \
                                                  img, g->nbr, g->eid, g->ts);                   \
  }
  TGFX_SCATTER_VARIANTS(X)
#undef X
  after_launch("k_scatter");
  if (ncold > 0) {
    k_cold<<<resident_grid(k_cold, 256, 0, ncold), 256, 0, s>>>(img, ncold, g->nbr, g->eid, g->ts);
    after_launch("k_cold");
  }
}

// indptr[u] = lower_bound(sorted node keys, u) for u = 0..V (the degrees are the run lengths
// of the sorted keys, so no degree-counting pass with atomics is needed)
template <typename K>
__global__ void k_indptr_lb(const K* __restrict__ keys, int64_t m, int64_t V,
                            int64_t* __restrict__ indptr) {
  const int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (u > V) return;
  int64_t lo = 0, len = m;
  while (len > 0) {
    const int64_t h = len >> 1;
    if (static_cast<int64_t>(__ldg(keys + lo + h)) < u) {
      lo += h + 1;
      len -= h + 1;
    } else {
      len = h;
    }
  }
  indptr[u] = lo;
}

// large V: (node, emission index) pairs sorted by node (stable LSD, 32-bit keys while node ids
// fit), indptr from the sorted keys, then each output position gathers its event
// node-id bits the large-V sort orders by (its digit passes: (bits + 7) / 8)
int large_key_bits(int64_t V) {
  int bits = 1;
  while (bits < 63 && (int64_t(1) << bits) < V) ++bits;
  return bits;
}

// pre: the sort input and its digit histograms from k_flags_keys (32-bit keys), or null
template <typename K>
void build_large_k(tgfx_graph* g, const tgfx_event* d_ev, cudaStream_t s, const LargePre* pre) {
  const int64_t V = g->V, m = g->m;
  const int grid = grid_for(m, 256);
  K* key = pre ? reinterpret_cast<K*>(pre->key) : static_cast<K*>(dmalloc(sizeof(K) * m, s));
  K* kalt = static_cast<K*>(dmalloc(sizeof(K) * m, s));
  uint32_t* val = pre ? pre->val : static_cast<uint32_t*>(dmalloc(sizeof(uint32_t) * m, s));
  uint32_t* valt = static_cast<uint32_t*>(dmalloc(sizeof(uint32_t) * m, s));
  if (!pre) {
    if (g->reverse)
      k_entry_keys<2, K><<<grid, 256, 0, s>>>(d_ev, m, key, val);
    else
      k_entry_keys<1, K><<<grid, 256, 0, s>>>(d_ev, m, key, val);
    after_launch("k_entry_keys");
  }
  const int bits = large_key_bits(V);
  K* k = key;
  uint32_t* v = val;
  radix_sort_pairs<K, uint32_t>(k, v, kalt, valt, m, bits, s, pre ? pre->hist : nullptr);
  k_indptr_lb<K><<<static_cast<unsigned>(ceil_div(V + 1, 256)), 256, 0, s>>>(k, m, V, g->indptr);
  after_launch("k_indptr_lb");
  uint4* rec = ensure_rec(g, s);
  g->cols_valid = rec == nullptr;
  if (g->reverse)
    k_gather_entries<2><<<grid, 256, 0, s>>>(d_ev, v, m, g->nbr, g->eid, g->ts, rec);
  else
    k_gather_entries<1><<<grid, 256, 0, s>>>(d_ev, v, m, g->nbr, g->eid, g->ts, rec);
  after_launch("k_gather_entries");
  if (!pre) {  // pre's buffers belong to the caller
    dfree(key, s);
    dfree(val, s);
  }
  dfree(kalt, s);
  dfree(valt, s);
}

void build_large(tgfx_graph* g, const tgfx_event* d_ev, cudaStream_t s,
                 const LargePre* pre = nullptr) {
  const int64_t V = g->V, m = g->m;
  if (m >= (int64_t(1) << 32)) throw Error(TGFX_EUNSUPPORTED, "more than 2^32 entries");
  if (m == 0) {
    TGFX_CUDA(cudaMemsetAsync(g->indptr, 0, sizeof(int64_t) * (V + 1), s));
    return;
  }
  if (V <= 0xffffffffLL)
    build_large_k<uint32_t>(g, d_ev, s, pre);
  else
    build_large_k<uint64_t>(g, d_ev, s, nullptr);
}

}  // namespace

int64_t fast_path_max_nodes() { return kFastMaxNodes; }

// Pinned host mirrors of the build flags come from one slab pinned once per process:
// cudaMallocHost / cudaFreeHost per graph cost up to hundreds of ms when the driver
// synchronises (seen as 0.4 s stalls in tgfx_graph_free on the e2e path).
namespace {
constexpr int kFlagSlots = 1024;
std::mutex g_flag_mu;
BuildFlags* g_flag_slab = nullptr;
std::vector<int> g_flag_free;

BuildFlags* flags_alloc() {
  std::lock_guard<std::mutex> lk(g_flag_mu);
  if (!g_flag_slab) {
    void* p = nullptr;
    TGFX_CUDA(cudaMallocHost(&p, sizeof(BuildFlags) * kFlagSlots));
    g_flag_slab = static_cast<BuildFlags*>(p);
    for (int i = kFlagSlots - 1; i >= 0; --i) g_flag_free.push_back(i);
  }
  if (!g_flag_free.empty()) {
    const int i = g_flag_free.back();
    g_flag_free.pop_back();
    return g_flag_slab + i;
  }
  void* p = nullptr;  // more than kFlagSlots live graphs: a separate pinned block
  TGFX_CUDA(cudaMallocHost(&p, sizeof(BuildFlags)));
  return static_cast<BuildFlags*>(p);
}

void flags_free(BuildFlags* f) {
  std::lock_guard<std::mutex> lk(g_flag_mu);
  if (g_flag_slab && f >= g_flag_slab && f < g_flag_slab + kFlagSlots)
    g_flag_free.push_back(static_cast<int>(f - g_flag_slab));
  else
    cudaFreeHost(f);
}
}  // namespace

void graph_alloc(tgfx_graph* g, cudaStream_t s) {
  g->m = g->n * (g->reverse ? 2 : 1);
  const size_t mm = static_cast<size_t>(std::max<int64_t>(g->m, 1));
  g->indptr = static_cast<int64_t*>(dmalloc(sizeof(int64_t) * (g->V + 1), s));
  g->nbr = static_cast<int64_t*>(dmalloc(sizeof(int64_t) * mm, s));
  g->eid = static_cast<int64_t*>(dmalloc(sizeof(int64_t) * mm, s));
  g->ts = static_cast<double*>(dmalloc(sizeof(double) * (mm + kTsPad), s));
  TGFX_CUDA(cudaMemsetAsync(g->ts + mm, 0, sizeof(double) * kTsPad, s));
  g->dir = static_cast<NodeDir*>(dmalloc(sizeof(NodeDir) * std::max<int64_t>(g->V, 1), s));
  g->dirc = static_cast<DirC*>(dmalloc(sizeof(DirC) * std::max<int64_t>(g->V, 1), s));
  g->dflags = static_cast<BuildFlags*>(dmalloc(sizeof(BuildFlags), s));
  g->hflags = flags_alloc();
}

void graph_release(tgfx_graph* g) {
  cudaStream_t s = 0;
  if (g->indptr) dfree(g->indptr, s);
  if (g->nbr) dfree(g->nbr, s);
  if (g->eid) dfree(g->eid, s);
  if (g->ts) dfree(g->ts, s);
  if (g->dflags) dfree(g->dflags, s);
  if (g->dir) dfree(g->dir, s);
  if (g->dirc) dfree(g->dirc, s);
  if (g->bkt) dfree(g->bkt, s);
  if (g->rec) dfree(g->rec, s);
  if (g->ws) dfree(g->ws, s);
  if (g->ws_small) dfree(g->ws_small, s);
  if (g->ws_rec) dfree(g->ws_rec, s);
  if (g->hflags) flags_free(g->hflags);
  g->indptr = g->nbr = g->eid = nullptr;
  g->ts = nullptr;
  g->dir = nullptr;
  g->dirc = nullptr;
  g->bkt = nullptr;
  g->bkt_cap = 0;
  g->rec = nullptr;
  g->rec_cap = 0;
  g->dflags = nullptr;
  g->hflags = nullptr;
  g->ws = g->ws_small = g->ws_rec = nullptr;
}

void build_graph(tgfx_graph* g, const tgfx_event* d_ev, cudaStream_t s, bool trusted) {
  g->cols_valid = true;  // every path writes the columns, except the tile scatter with records
  const double t0 = trace_ms(s);
  (void)trusted;
  const int64_t n = g->n, V = g->V;
  const int R = g->reverse ? 2 : 1;
  const bool fast = V <= kFastMaxNodes && g->m < (int64_t(1) << 32);
  t_build_m = g->m;
  int C = 1;
  int64_t chunk_ev = std::max<int64_t>(n, 1);
  uint32_t* cnt = nullptr;
  if (fast) {
    const int bps = scatter_blocks_per_sm(R, V);
    C = static_cast<int>(std::max<int64_t>(
        1, std::min<int64_t>(static_cast<int64_t>(device_info().sms) * bps, ceil_div(n, 1024))));
    chunk_ev = std::max<int64_t>(1, ceil_div(n, C));
    C = static_cast<int>(std::max<int64_t>(1, ceil_div(std::max<int64_t>(n, 1), chunk_ev)));
    const size_t need = sizeof(uint32_t) * static_cast<size_t>(C) * std::max<int64_t>(V, 1);
    if (g->ws_bytes < need) {
      if (g->ws) dfree(g->ws, s);
      g->ws = dmalloc(need, s);
      g->ws_bytes = need;
    }
    cnt = static_cast<uint32_t*>(g->ws);
  } else {
    C = grid_for(n, kHistThreads, 4);
    chunk_ev = std::max<int64_t>(1, ceil_div(std::max<int64_t>(n, 1), C));
  }
  // large-V builds of a sorted stream: the flags pass also writes the sort input
  LargePre pre{};
  const bool fuse = !fast && g->m > 0 && g->m < (int64_t(1) << 32) && V <= 0xffffffffLL &&
                    large_fuse_enabled();
  if (fuse) {
    const int passes = std::min(4, (large_key_bits(V) + 7) / 8);
    pre.key = static_cast<uint32_t*>(dmalloc(sizeof(uint32_t) * g->m, s));
    pre.val = static_cast<uint32_t*>(dmalloc(sizeof(uint32_t) * g->m, s));
    pre.hist = static_cast<unsigned long long*>(dmalloc(sizeof(unsigned long long) * 1024, s));
    TGFX_CUDA(cudaMemsetAsync(pre.hist, 0, sizeof(unsigned long long) * 1024, s));
    k_init_flags<<<1, 1, 0, s>>>(g->dflags);
    after_launch("k_init_flags");
    const int64_t Vd = g->reverse ? V : g->other_limit;
    if (g->reverse)
      k_flags_keys<2><<<C, kHistThreads, 0, s>>>(d_ev, n, V, Vd, chunk_ev, passes, pre.key,
                                                 pre.val, pre.hist, g->dflags);
    else
      k_flags_keys<1><<<C, kHistThreads, 0, s>>>(d_ev, n, V, Vd, chunk_ev, passes, pre.key,
                                                 pre.val, pre.hist, g->dflags);
    after_launch("k_flags_keys");
  } else {
    run_flags_pass(g, d_ev, C, chunk_ev, cnt, fast && V > 0, s);
  }
  auto drop_pre = [&] {
    if (pre.key) {
      dfree(pre.key, s);
      dfree(pre.val, s);
      dfree(pre.hist, s);
      pre = LargePre{};
    }
  };
  try {
    read_flags(g, s);
  } catch (...) {
    drop_pre();
    throw;
  }
  const double t1 = trace_ms(s);
  if (g->hflags->bad_index != ~0ull) {
    drop_pre();
    throw_bad_endpoint(g, d_ev, s);
  }
  g->max_eid = n ? g->hflags->max_eid : -1;
  g->min_eid = n ? g->hflags->min_eid : 0;
  const tgfx_event* src = d_ev;
  tgfx_event* tmp = nullptr;
  g->path = fast ? 0 : 2;
  g->search_exact = g->hflags->has_nan ? 1 : 0;
  if (g->hflags->unsorted) {
    drop_pre();  // the keys of the unsorted stream are not the sort input
    tmp = sorted_copy(d_ev, n, s);
    src = tmp;
    if (fast) {
      g->path = 1;
      run_flags_pass(g, src, C, chunk_ev, cnt, V > 0, s);
    }
  }
  try {
    if (fast)
      build_fast(g, src, C, chunk_ev, cnt, s);
    else
      build_large(g, src, s, pre.key ? &pre : nullptr);
  } catch (...) {
    drop_pre();
    if (tmp) dfree(tmp, s);
    throw;
  }
  drop_pre();
  if (tmp) dfree(tmp, s);
  const double t2 = trace_ms(s);
  build_node_dir(g, s);
  if (build_trace())
    fprintf(stderr, "[tgfx] build_graph: flags %.1f ms, scatter %.1f ms, node dir %.1f ms\n",
            t1 - t0, t2 - t1, trace_ms(s) - t2);
}

__global__ void __launch_bounds__(256) k_widen(const uint4* __restrict__ rec, int64_t m,
                                               int64_t* __restrict__ nbr,
                                               int64_t* __restrict__ eid) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint4 r = __ldg(rec + i);
    nbr[i] = static_cast<int64_t>(r.x);
    eid[i] = static_cast<int64_t>(r.y);
  }
}

void ensure_columns(const tgfx_graph* cg, cudaStream_t s) {
  tgfx_graph* g = const_cast<tgfx_graph*>(cg);
  std::lock_guard<std::mutex> lk(g->cols_mu);
  if (g->cols_valid) return;
  if (g->m > 0) {
    k_widen<<<grid_for(g->m, 256), 256, 0, s>>>(g->rec, g->m, g->nbr, g->eid);
    after_launch("k_widen");
    // complete before another thread sees cols_valid and reads the columns on its own stream
    TGFX_CUDA(cudaStreamSynchronize(s));
  }
  g->cols_valid = true;
}

// bucket-fill kernel (TGFX_BUCKET_FILL: 8 = per-thread walk over 8 entries (default), 1 = one
// entry per thread)
static int bucket_fill_v() {
  static const int v = [] {
    const char* e = getenv("TGFX_BUCKET_FILL");
    return e ? atoi(e) : 8;
  }();
  return v;
}

// entries per time bucket (TGFX_BUCKET_ENTRIES, default 4; 0 disables the tables)
static int64_t bucket_entries() {
  static const int64_t r = [] {
    const char* e = getenv("TGFX_BUCKET_ENTRIES");
    return e ? static_cast<int64_t>(atoll(e)) : static_cast<int64_t>(4);
  }();
  return r;
}

void build_node_dir(tgfx_graph* g, cudaStream_t s) {
  if (g->V <= 0) return;
  const int64_t R = g->search_exact ? 0 : bucket_entries();
  const int vb = static_cast<int>(ceil_div(g->V, 256));
  // gather records from the columns, unless the build's scatter already wrote them
  uint4* rec = g->cols_valid ? ensure_rec(g, s) : nullptr;
  const int64_t tiles = ceil_div(g->m, kFillTile);
  // the compact directory holds slice lengths as u32
  g->bkt_r = R > 0 && g->m < (int64_t(1) << 32) ? R : 0;
  if (g->bkt_r <= 0) {
    k_node_dir<<<vb, 256, 0, s>>>(g->indptr, g->ts, g->V, 0, g->dir, g->dirc, nullptr);
    after_launch("k_node_dir");
    if (rec) {
      k_bucket_fill<<<static_cast<int>(tiles), 256, 0, s>>>(g->indptr, g->nbr, g->eid, g->ts,
                                                            g->dir, nullptr, g->V, g->m, false,
                                                            rec);
      after_launch("k_bucket_fill");
    }
    return;
  }
  // node u's table at start_u / R + 2u, nb_u + 1 <= n_u / R + 2 entries: size m / R + 2V + 2
  const int64_t cap = g->m / R + 2 * g->V + 2;
  if (g->bkt_cap < cap) {
    if (g->bkt) dfree(g->bkt, s);
    g->bkt = static_cast<uint32_t*>(dmalloc(sizeof(uint32_t) * cap, s));
    g->bkt_cap = cap;
  }
  int32_t* tile_node = static_cast<int32_t*>(dmalloc(sizeof(int32_t) * std::max<int64_t>(tiles, 1), s));
  k_node_dir<<<vb, 256, 0, s>>>(g->indptr, g->ts, g->V, R, g->dir, g->dirc, g->bkt);
  after_launch("k_node_dir");
  if (tiles > 0) {
    k_tile_node<<<static_cast<int>(ceil_div(tiles, 256)), 256, 0, s>>>(g->indptr, g->V, tiles,
                                                                        tile_node);
    after_launch("k_tile_node");
  }
  if (g->m > 0) {
    if (bucket_fill_v() == 8)
      k_bucket_fill8<<<static_cast<int>(tiles), 256, 0, s>>>(g->indptr, g->nbr, g->eid, g->ts,
                                                             g->dir, tile_node, g->V, g->m, true,
                                                             rec);
    else
      k_bucket_fill<<<static_cast<int>(tiles), 256, 0, s>>>(g->indptr, g->nbr, g->eid, g->ts,
                                                            g->dir, tile_node, g->V, g->m, true,
                                                            rec);
    after_launch("k_bucket_fill");
  }
  dfree(tile_node, s);
}

std::string validate_graph(const tgfx_graph* g, cudaStream_t s) {
  // tcsr.cpp:54-81 in the reference's order; the shape checks (sizes) are the caller's
  std::vector<int64_t> ip(static_cast<size_t>(g->V + 1));
  TGFX_CUDA(cudaMemcpyAsync(ip.data(), g->indptr, sizeof(int64_t) * (g->V + 1),
                            cudaMemcpyDeviceToHost, s));
  TGFX_CUDA(cudaStreamSynchronize(s));
  if (ip[0] != 0 || ip[static_cast<size_t>(g->V)] != g->m) return "indptr endpoints wrong";
  int64_t u_mono = g->V;  // first node whose indptr pair decreases
  for (int64_t u = 0; u < g->V; ++u)
    if (ip[static_cast<size_t>(u)] > ip[static_cast<size_t>(u + 1)]) {
      u_mono = u;
      break;
    }
  ensure_columns(g, s);
  unsigned long long* fail = static_cast<unsigned long long*>(dmalloc(2 * sizeof(unsigned long long), s));
  const unsigned long long none[2] = {~0ull, ~0ull};
  TGFX_CUDA(cudaMemcpyAsync(fail, none, sizeof none, cudaMemcpyHostToDevice, s));
  if (g->m > 0) {
    k_validate<<<grid_for(g->m, 256), 256, 0, s>>>(g->indptr, g->nbr, g->eid, g->ts, u_mono,
                                                  g->other_limit, g->eid_limit, g->m, fail,
                                                  fail + 1);
    after_launch("k_validate");
  }
  unsigned long long h[2];
  TGFX_CUDA(cudaMemcpyAsync(h, fail, sizeof h, cudaMemcpyDeviceToHost, s));
  TGFX_CUDA(cudaStreamSynchronize(s));
  dfree(fail, s);
  // node loop: monotone check of u, then slice u (tcsr.cpp:64-72)
  if (h[0] != ~0ull && static_cast<int64_t>(h[0]) < u_mono)
    return "slice of node " + std::to_string(h[0]) + " not sorted";
  if (u_mono < g->V) return "indptr not monotone";
  // entry loop (tcsr.cpp:73-80)
  if (h[1] != ~0ull) return (h[1] & 1) ? "edge id out of range" : "neighbor id out of range";
  return "";
}

}  // namespace tgfx
