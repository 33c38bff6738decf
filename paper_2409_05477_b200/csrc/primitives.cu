// primitives.cu -- device-wide scan and stable LSD radix sort used by the builder's
// general (unsorted-stream) and large-V paths.  Hand-written for sm_100a: warp-aggregated
// digit ranking with __match_any_sync, warp-private shared-memory counters (deterministic,
// stable), one scatter pass per 8-bit digit; digits constant across all keys are skipped.
#include "graph.cuh"
#include "primitives.cuh"

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

__global__ void __launch_bounds__(kScanThreads) k_scan_reduce(const uint32_t* __restrict__ in,
                                                              int64_t n, int64_t* partials) {
  const int64_t base = static_cast<int64_t>(blockIdx.x) * kScanTile;
  int64_t s = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    const int64_t j = base + i * kScanThreads + threadIdx.x;
    if (j < n) s += in[j];
  }
  int64_t tot;
  block_exclusive_scan_i64(s, &tot);
  if (threadIdx.x == 0) partials[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(1024) k_scan_partials(int64_t* partials, int64_t nb) {
  // single block: exclusive scan in place, sequential chunks of blockDim values
  __shared__ int64_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int64_t base = 0; base < nb; base += blockDim.x) {
    const int64_t j = base + threadIdx.x;
    const int64_t v = j < nb ? partials[j] : 0;
    int64_t tot;
    const int64_t ex = block_exclusive_scan_i64(v, &tot);
    if (j < nb) partials[j] = carry + ex;
    __syncthreads();
    if (threadIdx.x == 0) carry += tot;
    __syncthreads();
  }
}

__global__ void __launch_bounds__(kScanThreads) k_scan_final(const uint32_t* __restrict__ in,
                                                             int64_t n,
                                                             const int64_t* __restrict__ partials,
                                                             int64_t* out) {
  // each thread owns kScanItems consecutive elements
  const int64_t base = static_cast<int64_t>(blockIdx.x) * kScanTile + threadIdx.x * kScanItems;
  uint32_t v[kScanItems];
  int64_t s = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    v[i] = base + i < n ? in[base + i] : 0u;
    s += v[i];
  }
  int64_t tot;
  int64_t run = partials[blockIdx.x] + block_exclusive_scan_i64(s, &tot);
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    if (base + i < n) out[base + i] = run;
    run += v[i];
  }
  if (base + kScanItems >= n && base < n) {
    // the thread owning the last element also writes out[n]
    out[n] = run;
  }
}
}  // namespace

void scan_u32_to_i64(const uint32_t* in, int64_t n, int64_t* out, cudaStream_t s) {
  if (n <= 0) {
    TGFX_CUDA(cudaMemsetAsync(out, 0, sizeof(int64_t), s));
    return;
  }
  const int64_t nb = ceil_div(n, kScanTile);
  int64_t* partials = static_cast<int64_t*>(dmalloc(sizeof(int64_t) * nb, s));
  k_scan_reduce<<<static_cast<unsigned>(nb), kScanThreads, 0, s>>>(in, n, partials);
  after_launch("k_scan_reduce");
  k_scan_partials<<<1, 1024, 0, s>>>(partials, nb);
  after_launch("k_scan_partials");
  k_scan_final<<<static_cast<unsigned>(nb), kScanThreads, 0, s>>>(in, n, partials, out);
  after_launch("k_scan_final");
  dfree(partials, s);
}

// ------------------------------------------------------------------ radix sort
namespace {
constexpr int kRsThreads = 256;
constexpr int kRsWarps = kRsThreads / 32;
constexpr int kRsRounds = 8;
constexpr int kRsTile = kRsThreads * kRsRounds;  // 2048 keys per tile

__global__ void __launch_bounds__(kRsThreads) k_or_and(const uint64_t* __restrict__ keys, int64_t n,
                                                       unsigned long long* orand) {
  uint64_t o = 0, a = ~0ull;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t k = keys[i];
    o |= k;
    a &= k;
  }
#pragma unroll
  for (int off = 16; off; off >>= 1) {
    o |= __shfl_xor_sync(kFull, o, off);
    a &= __shfl_xor_sync(kFull, a, off);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicOr(&orand[0], (unsigned long long)o);
    atomicAnd(&orand[1], (unsigned long long)a);
  }
}

// per-tile digit histograms, digit-major: hist[d * ntiles + tile]
__global__ void __launch_bounds__(kRsThreads) k_digit_hist(const uint64_t* __restrict__ keys,
                                                           int64_t n, int shift,
                                                           uint32_t* __restrict__ hist,
                                                           int64_t ntiles) {
  __shared__ uint32_t h[256];
  h[threadIdx.x] = 0;
  __syncthreads();
  const int64_t base = static_cast<int64_t>(blockIdx.x) * kRsTile;
#pragma unroll
  for (int r = 0; r < kRsRounds; ++r) {
    const int64_t j = base + r * kRsThreads + threadIdx.x;
    const unsigned d = j < n ? static_cast<unsigned>((keys[j] >> shift) & 0xff) : 0x100u;
    const unsigned peers = __match_any_sync(kFull, d);
    if (d < 256 && (threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(&h[d], __popc(peers));
  }
  __syncthreads();
  hist[static_cast<int64_t>(threadIdx.x) * ntiles + blockIdx.x] = h[threadIdx.x];
}

// stable scatter: warp w owns keys [base + w*256, base + (w+1)*256) in 8 rounds of 32
template <typename V>
__global__ void __launch_bounds__(kRsThreads) k_digit_scatter(
    const uint64_t* __restrict__ keys_in, const V* __restrict__ vals_in, int64_t n, int shift,
    const int64_t* __restrict__ offsets, int64_t ntiles, uint64_t* __restrict__ keys_out,
    V* __restrict__ vals_out) {
  __shared__ uint32_t wcnt[kRsWarps][256];
  __shared__ int64_t goff[256];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < kRsWarps * 256; i += kRsThreads) (&wcnt[0][0])[i] = 0;
  goff[threadIdx.x] = offsets[static_cast<int64_t>(threadIdx.x) * ntiles + blockIdx.x];
  __syncthreads();
  const int64_t base = static_cast<int64_t>(blockIdx.x) * kRsTile + warp * (kRsRounds * 32);
  uint64_t k[kRsRounds];
  V v[kRsRounds];
  uint32_t rank[kRsRounds];
#pragma unroll
  for (int r = 0; r < kRsRounds; ++r) {
    const int64_t j = base + r * 32 + lane;
    const bool ok = j < n;
    k[r] = ok ? keys_in[j] : 0;
    v[r] = ok ? vals_in[j] : V(0);
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
  {  // exclusive prefix over warps per digit (thread = digit)
    const int d = threadIdx.x;
    uint32_t run = 0;
#pragma unroll
    for (int w = 0; w < kRsWarps; ++w) {
      const uint32_t c = wcnt[w][d];
      wcnt[w][d] = run;
      run += c;
    }
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < kRsRounds; ++r) {
    const int64_t j = base + r * 32 + lane;
    if (j < n) {
      const unsigned d = static_cast<unsigned>((k[r] >> shift) & 0xff);
      const int64_t pos = goff[d] + wcnt[warp][d] + rank[r];
      keys_out[pos] = k[r];
      vals_out[pos] = v[r];
    }
  }
}
}  // namespace

template <typename V>
void radix_sort_pairs(uint64_t*& keys, V*& vals, uint64_t* keys_alt, V* vals_alt, int64_t n,
                      int max_bits, cudaStream_t s) {
  if (n <= 1) return;
  unsigned long long* orand = static_cast<unsigned long long*>(dmalloc(16, s));
  const unsigned long long init[2] = {0ull, ~0ull};
  TGFX_CUDA(cudaMemcpyAsync(orand, init, 16, cudaMemcpyHostToDevice, s));
  const int grid = static_cast<int>(std::min<int64_t>(ceil_div(n, kRsThreads), 4 * 148));
  k_or_and<<<grid, kRsThreads, 0, s>>>(keys, n, orand);
  after_launch("k_or_and");
  unsigned long long h[2];
  TGFX_CUDA(cudaMemcpyAsync(h, orand, 16, cudaMemcpyDeviceToHost, s));
  TGFX_CUDA(cudaStreamSynchronize(s));
  dfree(orand, s);
  const uint64_t varying = h[0] ^ h[1];
  const int64_t ntiles = ceil_div(n, kRsTile);
  uint32_t* hist = static_cast<uint32_t*>(dmalloc(sizeof(uint32_t) * 256 * ntiles, s));
  int64_t* offs = static_cast<int64_t*>(dmalloc(sizeof(int64_t) * (256 * ntiles + 1), s));
  for (int shift = 0; shift < max_bits; shift += 8) {
    if (((varying >> shift) & 0xffull) == 0) continue;  // digit constant: pass is identity
    k_digit_hist<<<static_cast<unsigned>(ntiles), kRsThreads, 0, s>>>(keys, n, shift, hist,
                                                                      ntiles);
    after_launch("k_digit_hist");
    scan_u32_to_i64(hist, 256 * ntiles, offs, s);
    k_digit_scatter<V><<<static_cast<unsigned>(ntiles), kRsThreads, 0, s>>>(
        keys, vals, n, shift, offs, ntiles, keys_alt, vals_alt);
    after_launch("k_digit_scatter");
    std::swap(keys, keys_alt);
    std::swap(vals, vals_alt);
  }
  dfree(offs, s);
  dfree(hist, s);
}

template void radix_sort_pairs<uint32_t>(uint64_t*&, uint32_t*&, uint64_t*, uint32_t*, int64_t,
                                         int, cudaStream_t);
template void radix_sort_pairs<uint64_t>(uint64_t*&, uint64_t*&, uint64_t*, uint64_t*, int64_t,
                                         int, cudaStream_t);

}  // namespace tgfx
