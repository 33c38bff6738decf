// primitives.cu -- device-wide scan and stable LSD radix sort used by the builder's
// general (unsorted-stream) and large-V paths.  Hand-written for sm_100a:
//   * scan: single pass with decoupled look-back (each tile publishes its aggregate, then its
//     inclusive prefix; a tile's exclusive prefix comes from walking back over its
//     predecessors' published words -- no separate reduce / partials kernels);
//   * sort: "onesweep" LSD -- one histogram pass computes every digit position's global
//     histogram up front (digits constant across all keys are skipped), then ONE kernel per
//     8-bit digit: tiles (taken in order from an atomic counter) rank their keys by digit with
//     __match_any_sync and warp-private shared-memory counters (stable), publish per-digit
//     tile counts, find their per-digit global offsets by decoupled look-back, and scatter.
#include "graph.cuh"
#include "primitives.cuh"

#include <algorithm>
#include <vector>

namespace tgfx {

// ------------------------------------------------------------------ scan
namespace {
constexpr int kScanThreads = 256;
constexpr int kScanItems = 16;
constexpr int kScanTile = kScanThreads * kScanItems;

__device__ __forceinline__ int64_t block_exclusive_scan_i64(int64_t v, int64_t* total) {
  __shared__ int64_t warp_sums[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int64_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int64_t y = __shfl_up_sync(kFull, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_sums[warp] = x;
  __syncthreads();
  if (warp == 0) {
    const int nw = blockDim.x >> 5;
    int64_t s = lane < nw ? warp_sums[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int64_t y = __shfl_up_sync(kFull, s, o);
      if (lane >= o) s += y;
    }
    if (lane < nw) warp_sums[lane] = s;
  }
  __syncthreads();
  const int64_t before = (warp > 0 ? warp_sums[warp - 1] : 0) + x - v;
  if (total) *total = warp_sums[(blockDim.x >> 5) - 1];
  __syncthreads();
  return before;
}

constexpr unsigned long long kFlagAgg = 1ull << 62;  // tile aggregate published
constexpr unsigned long long kFlagInc = 2ull << 62;  // inclusive prefix published
constexpr unsigned long long kValMask = (1ull << 62) - 1;

// The status words are self-contained (flag and value in one 64-bit word, written with one
// store) and nothing else is read on the strength of them, so relaxed gpu-scope accesses are
// enough: same-address coherence orders a tile's AGG before its INC.
__device__ __forceinline__ void st_release(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// exclusive prefix of tile `tile` for one value: walk back over published words until an
// inclusive prefix (spins while a predecessor has published nothing yet -- predecessors took
// their tile ids earlier from the same counter, so they are resident and make progress).
// Four words are loaded per step so a walk over aggregates costs a quarter of the round trips.
__device__ __forceinline__ unsigned long long lookback(const unsigned long long* status,
                                                       int64_t tile, int64_t stride) {
  constexpr int W = 4;
  unsigned long long excl = 0;
  int64_t t = tile - 1;
  while (t >= 0) {
    unsigned long long w[W];
#pragma unroll
    for (int j = 0; j < W; ++j) w[j] = t - j >= 0 ? ld_acquire(status + (t - j) * stride) : kFlagInc;
    bool done = false;
#pragma unroll
    for (int j = 0; j < W; ++j) {
      if (done) continue;
      const unsigned long long f = w[j] & ~kValMask;
      if (f == 0) { done = true; continue; }   // not published yet: re-poll from t
      excl += w[j] & kValMask;
      --t;
      if (f == kFlagInc) { done = true; t = -1; }
    }
  }
  return excl;
}

// single-pass exclusive scan u32 -> i64 (out[n] = total); thread owns kScanItems consecutive
__global__ void __launch_bounds__(kScanThreads) k_scan_lookback(const uint32_t* __restrict__ in,
                                                                int64_t n, int64_t* out,
                                                                unsigned long long* status,
                                                                unsigned int* counter) {
  __shared__ int64_t s_tile, s_excl;
  if (threadIdx.x == 0) s_tile = atomicAdd(counter, 1u);
  __syncthreads();
  const int64_t tile = s_tile;
  const int64_t base = tile * kScanTile + threadIdx.x * kScanItems;
  uint32_t v[kScanItems];
  int64_t sum = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    v[i] = base + i < n ? in[base + i] : 0u;
    sum += v[i];
  }
  int64_t tot;
  const int64_t local = block_exclusive_scan_i64(sum, &tot);
  if (threadIdx.x == 0) {
    if (tile == 0) {
      st_release(status, kFlagInc | static_cast<unsigned long long>(tot));
      s_excl = 0;
    } else {
      st_release(status + tile, kFlagAgg | static_cast<unsigned long long>(tot));
      const unsigned long long ex = lookback(status, tile, 1);
      st_release(status + tile, kFlagInc | (ex + static_cast<unsigned long long>(tot)));
      s_excl = static_cast<int64_t>(ex);
    }
  }
  __syncthreads();
  int64_t run = s_excl + local;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    if (base + i < n) out[base + i] = run;
    run += v[i];
  }
  if (base + kScanItems >= n && base < n) out[n] = run;  // owner of the last element
}
}  // namespace

void scan_u32_to_i64(const uint32_t* in, int64_t n, int64_t* out, cudaStream_t s) {
  if (n <= 0) {
    TGFX_CUDA(cudaMemsetAsync(out, 0, sizeof(int64_t), s));
    return;
  }
  const int64_t nb = ceil_div(n, kScanTile);
  // status words (one per tile) + the tile counter, zeroed together
  char* ws = static_cast<char*>(dmalloc(sizeof(unsigned long long) * nb + 16, s));
  TGFX_CUDA(cudaMemsetAsync(ws, 0, sizeof(unsigned long long) * nb + 16, s));
  unsigned long long* status = reinterpret_cast<unsigned long long*>(ws);
  unsigned int* counter = reinterpret_cast<unsigned int*>(ws + sizeof(unsigned long long) * nb);
  k_scan_lookback<<<static_cast<unsigned>(nb), kScanThreads, 0, s>>>(in, n, out, status, counter);
  after_launch("k_scan_lookback");
  dfree(ws, s);
}

// ------------------------------------------------------------------ radix sort
// onesweep tile shape and residency (1/16-scale MAG build, 3 passes of 162 M 8-byte pairs;
// round 2): 16 keys per thread at 128 registers left 2 tiles per SM (occupancy limited by
// registers and by the default shared-memory carveout) -> 11.6 ms; capped at 4 tiles per SM
// (64 registers, 40 B of spills) with an 80 % carveout -> 10.3 ms.  Also measured: 3 tiles
// per SM 11.4, 5 / 6 per SM 10.4 / 10.6, 8 keys per thread at 6 / 8 per SM 11.5 / 11.6,
// 12 keys per thread at 5 per SM 11.0, 2 tiles per SM with a 100 % carveout 16.8 ms.
#ifndef TGFX_OS_ROUNDS
#define TGFX_OS_ROUNDS 16
#endif
#ifndef TGFX_OS_MINB
#define TGFX_OS_MINB 4
#endif
namespace {
constexpr int kRsThreads = 256;
constexpr int kRsWarps = kRsThreads / 32;
// keys per thread of a onesweep tile: 16 for 8-byte (key, value) pairs (4,096-key tiles: half
// as many tiles, so half the decoupled look-back walks), 8 otherwise (static shared memory)
template <typename K, typename V>
constexpr int rs_rounds() {
  return sizeof(K) + sizeof(V) <= 8 ? TGFX_OS_ROUNDS : 8;
}

// all digit positions' global histograms in one pass: hist[pass * 256 + digit] (u64)
template <typename K>
__global__ void __launch_bounds__(kRsThreads) k_onesweep_hist(const K* __restrict__ keys,
                                                              int64_t n, int passes,
                                                              unsigned long long* hist) {
  __shared__ uint32_t h[8][256];
  for (int i = threadIdx.x; i < 8 * 256; i += kRsThreads) (&h[0][0])[i] = 0;
  __syncthreads();
  for (int64_t i = blockIdx.x * (int64_t)kRsThreads + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * kRsThreads) {
    const K k = keys[i];
    for (int p = 0; p < passes; ++p) atomicAdd(&h[p][(k >> (8 * p)) & 0xff], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < passes * 256; i += kRsThreads) {
    const uint32_t c = (&h[0][0])[i];
    if (c) atomicAdd(hist + i, static_cast<unsigned long long>(c));
  }
}

// one onesweep pass: digit (key >> shift) & 0xff; digit_base[256] = the digit's global start
template <typename K, typename V>
__global__ void __launch_bounds__(kRsThreads, TGFX_OS_MINB) k_onesweep(
    const K* __restrict__ keys_in, const V* __restrict__ vals_in, int64_t n, int shift,
    const int64_t* __restrict__ digit_base, unsigned long long* status, unsigned int* counter,
    K* __restrict__ keys_out, V* __restrict__ vals_out) {
  constexpr int kRsRounds = rs_rounds<K, V>();
  constexpr int kRsTile = kRsThreads * kRsRounds;
  __shared__ uint32_t wcnt[kRsWarps][256];
  __shared__ int64_t goff[256];
  __shared__ int64_t s_tile;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) s_tile = atomicAdd(counter, 1u);
  for (int i = threadIdx.x; i < kRsWarps * 256; i += kRsThreads) (&wcnt[0][0])[i] = 0;
  __syncthreads();
  const int64_t tile = s_tile;
  const int64_t base = tile * kRsTile + warp * (kRsRounds * 32);
  K k[kRsRounds];
  V v[kRsRounds];
  uint32_t rank[kRsRounds];
#pragma unroll
  for (int r = 0; r < kRsRounds; ++r) {
    const int64_t j = base + r * 32 + lane;
    const bool ok = j < n;
    k[r] = ok ? keys_in[j] : 0;
    v[r] = ok ? vals_in[j] : V(0);
  }
#pragma unroll
  for (int r = 0; r < kRsRounds; ++r) {
    const int64_t j = base + r * 32 + lane;
    const bool ok = j < n;
    const unsigned d = ok ? static_cast<unsigned>((k[r] >> shift) & 0xff) : 0x100u;
    const unsigned peers = __match_any_sync(kFull, d);
    const int leader = __ffs(peers) - 1;
    uint32_t prev = 0;
    if (ok && lane == leader) {
      prev = wcnt[warp][d];
      wcnt[warp][d] = prev + __popc(peers);
    }
    prev = __shfl_sync(kFull, prev, leader);
    rank[r] = prev + __popc(peers & lanemask_lt());
    __syncwarp();
  }
  __syncthreads();
  __shared__ uint32_t lbase[256];  // tile-local start of each digit (sorted tile order)
  __shared__ uint32_t wtot[kRsWarps];
  {  // thread = digit: exclusive prefix over warps, tile count, look-back for the global offset
    const int d = threadIdx.x;
    uint32_t run = 0;
#pragma unroll
    for (int w = 0; w < kRsWarps; ++w) {
      const uint32_t c = wcnt[w][d];
      wcnt[w][d] = run;
      run += c;
    }
    unsigned long long* my = status + tile * 256 + d;
    unsigned long long ex = 0;
    if (tile == 0) {
      st_release(my, kFlagInc | run);
    } else {
      st_release(my, kFlagAgg | run);
      ex = lookback(status + d, tile, 256);
      st_release(my, kFlagInc | (ex + run));
    }
    goff[d] = digit_base[d] + static_cast<int64_t>(ex);
    // tile-local digit starts: exclusive block scan of the digit totals
    uint32_t x = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(kFull, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) wtot[warp] = x;
    __syncthreads();
    uint32_t before = 0;
#pragma unroll
    for (int w = 0; w < kRsWarps; ++w) before += w < warp ? wtot[w] : 0u;
    lbase[d] = before + x - run;
  }
  __syncthreads();
  // keys and values to their sorted tile positions in shared memory, then written out by
  // consecutive threads to consecutive global positions (coalesced runs per digit)
  __shared__ K sk[kRsTile];
  __shared__ V sv[kRsTile];
#pragma unroll
  for (int r = 0; r < kRsRounds; ++r) {
    const int64_t j = base + r * 32 + lane;
    if (j < n) {
      const unsigned d = static_cast<unsigned>((k[r] >> shift) & 0xff);
      const uint32_t lp = lbase[d] + wcnt[warp][d] + rank[r];
      sk[lp] = k[r];
      sv[lp] = v[r];
    }
  }
  __syncthreads();
  const int cnt = static_cast<int>(n - tile * kRsTile < kRsTile ? n - tile * kRsTile : kRsTile);
  for (int p = threadIdx.x; p < cnt; p += kRsThreads) {
    const K key = sk[p];
    const unsigned d = static_cast<unsigned>((key >> shift) & 0xff);
    const int64_t pos = goff[d] + (p - static_cast<int64_t>(lbase[d]));
    keys_out[pos] = key;
    vals_out[pos] = sv[p];
  }
}
}  // namespace

template <typename K, typename V>
void radix_sort_pairs(K*& keys, V*& vals, K* keys_alt, V* vals_alt, int64_t n,
                      int max_bits, cudaStream_t s, const unsigned long long* pre_hist) {
  if (n <= 1) return;
  const int passes = std::min(static_cast<int>(sizeof(K)), (max_bits + 7) / 8);
  if (passes <= 0) return;
  const int64_t ntiles = ceil_div(n, static_cast<int64_t>(kRsThreads) * rs_rounds<K, V>());
  // workspace: histograms [passes][256] u64 | digit bases [256] i64 | status [ntiles][256] u64
  // | tile counter
  const size_t hb = sizeof(unsigned long long) * 256 * passes;
  const size_t sb = sizeof(unsigned long long) * 256 * static_cast<size_t>(ntiles);
  char* ws = static_cast<char*>(dmalloc(hb + 2048 + sb + 16, s));
  unsigned long long* hist = reinterpret_cast<unsigned long long*>(ws);
  int64_t* dbase = reinterpret_cast<int64_t*>(ws + hb);
  unsigned long long* status = reinterpret_cast<unsigned long long*>(ws + hb + 2048);
  unsigned int* counter = reinterpret_cast<unsigned int*>(ws + hb + 2048 + sb);
  if (!pre_hist) {
    TGFX_CUDA(cudaMemsetAsync(hist, 0, hb, s));
    const int grid = static_cast<int>(std::min<int64_t>(ceil_div(n, kRsThreads), 8 * 148));
    k_onesweep_hist<K><<<grid, kRsThreads, 0, s>>>(keys, n, passes, hist);
    after_launch("k_onesweep_hist");
  }
  std::vector<unsigned long long> h(256 * passes);
  TGFX_CUDA(cudaMemcpyAsync(h.data(), pre_hist ? pre_hist : hist, hb, cudaMemcpyDeviceToHost, s));
  TGFX_CUDA(cudaStreamSynchronize(s));
  for (int p = 0; p < passes; ++p) {
    const unsigned long long* hp = h.data() + 256 * p;
    int nonzero = 0;
    for (int d = 0; d < 256; ++d) nonzero += hp[d] != 0;
    if (nonzero <= 1) continue;  // digit constant across all keys: the pass is the identity
    int64_t b[256], run = 0;
    for (int d = 0; d < 256; ++d) {
      b[d] = run;
      run += static_cast<int64_t>(hp[d]);
    }
    TGFX_CUDA(cudaMemcpyAsync(dbase, b, sizeof b, cudaMemcpyHostToDevice, s));
    TGFX_CUDA(cudaMemsetAsync(status, 0, sb + 16, s));
    static const bool carve = [] {  // room for TGFX_OS_MINB resident tiles' shared memory
      TGFX_CUDA(cudaFuncSetAttribute(k_onesweep<K, V>,
                                     cudaFuncAttributePreferredSharedMemoryCarveout, 80));
      return true;
    }();
    (void)carve;
    k_onesweep<K, V><<<static_cast<unsigned>(ntiles), kRsThreads, 0, s>>>(
        keys, vals, n, 8 * p, dbase, status, counter, keys_alt, vals_alt);
    after_launch("k_onesweep");
    std::swap(keys, keys_alt);
    std::swap(vals, vals_alt);
  }
  TGFX_CUDA(cudaStreamSynchronize(s));  // b[] (host stack) copies done before return
  dfree(ws, s);
}

template void radix_sort_pairs<uint64_t, uint32_t>(uint64_t*&, uint32_t*&, uint64_t*, uint32_t*,
                                                   int64_t, int, cudaStream_t,
                                                   const unsigned long long*);
template void radix_sort_pairs<uint64_t, uint64_t>(uint64_t*&, uint64_t*&, uint64_t*, uint64_t*,
                                                   int64_t, int, cudaStream_t,
                                                   const unsigned long long*);
template void radix_sort_pairs<uint32_t, uint32_t>(uint32_t*&, uint32_t*&, uint32_t*, uint32_t*,
                                                   int64_t, int, cudaStream_t,
                                                   const unsigned long long*);

}  // namespace tgfx
