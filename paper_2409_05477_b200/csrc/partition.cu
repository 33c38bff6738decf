// partition.cu -- kernels of the node-range-partitioned multi-GPU T-CSR build (sm_100a).
//
// The reference has no distributed construction; this is the MAG-scale build
// of BASELINE.json's north star.  Each rank holds a contiguous chunk of the
// stream; the host (paper_2409_05477_b200/partition.py) drives:
//   1. k_degree_hist   per-rank node degrees (src, and dst if reverse) -> all-reduce
//   2. entry ranges    rank d owns global entry positions [d*m/N, (d+1)*m/N): contiguous node
//                      ranges, plus the (at most N-1) nodes whose slice a cut falls into,
//                      split by entry position (host, from the global degrees)
//   3. k_part_count    per-warp entry counts per destination rank (and per split node)
//   4. k_part_scatter  stable partition of the rank's entries into per-destination buckets of
//                      32-byte records (eid, node - owner's first node, other endpoint, t): the
//                      record is a TemporalEvent whose src is the owner-local node id, so the
//                      owner builds its range with the ordinary builder (reverse = 0, other
//                      endpoint checked against the global node count)
//   5. one all-to-all-v of the records (NCCL); receivers concatenate in rank order, which is
//      global stream order, so the local build reproduces the single-GPU slices exactly.
#include <algorithm>

#include "graph.cuh"

namespace tgfx {
namespace {

constexpr int kPT = 256;

template <int R>
__global__ void __launch_bounds__(kPT) k_degree_hist(const tgfx_event* __restrict__ ev, int64_t n,
                                                     int64_t V,
                                                     unsigned long long* __restrict__ deg) {
  const int lane = threadIdx.x & 31;
  for (int64_t b = blockIdx.x * (int64_t)kPT; b < n; b += (int64_t)gridDim.x * kPT) {
    const int64_t e = b + threadIdx.x;
    Ev x{0, -1, -1, 0.0};
    if (e < n) x = load_event(ev, e);
#pragma unroll
    for (int side = 0; side < R; ++side) {
      const int64_t u = side ? x.dst : x.src;
      const bool ok = u >= 0 && u < V;
      const unsigned long long key = ok ? static_cast<unsigned long long>(u) : ~0ull;
      const unsigned peers = __match_any_sync(kFull, key);  // warp-aggregated (Zipf hub)
      if (ok && lane == __ffs(peers) - 1) atomicAdd(&deg[u], static_cast<unsigned long long>(__popc(peers)));
    }
  }
}

__device__ __forceinline__ int owner_of(int64_t u, const int64_t* __restrict__ bounds, int N) {
  int d = 0;
  while (d + 1 < N && u >= bounds[d + 1]) ++d;
  return d;
}

// Split nodes (the Zipf hubs): rank d owns the GLOBAL entry positions [P[d], P[d+1]) with
// P[d] = d*m/N, so a node whose slice contains a cut is split between ranks.  Its entry with
// global position p goes to the largest d with P[d] <= p; p = gp + j for the j-th entry
// (emission order) of that node in this rank's chunk, gp = indptr[node] + the node's entries
// in earlier ranks' chunks.  Every other node goes to its node range [bounds[d], bounds[d+1]).
// Split table d_split (int64): [ns, node[7], gp[7], P[9]].
struct SplitTab {
  int ns;
  int64_t node[7], gp[7], P[9];
};

__device__ __forceinline__ void load_split(const int64_t* __restrict__ g, SplitTab& t) {
  t.ns = static_cast<int>(g[0]);
#pragma unroll
  for (int i = 0; i < 7; ++i) {
    t.node[i] = g[1 + i];
    t.gp[i] = g[8 + i];
  }
#pragma unroll
  for (int i = 0; i < 9; ++i) t.P[i] = g[15 + i];
}

__device__ __forceinline__ int split_index(const SplitTab& t, int64_t u) {
  int si = -1;
#pragma unroll
  for (int i = 0; i < 7; ++i)
    if (i < t.ns && t.node[i] == u) si = i;
  return si;
}

// entries of warp w's contiguous event range [w*per, (w+1)*per): counts[w * N + d] of the
// non-split nodes' entries per destination, scounts[w * 7 + i] of split node i's entries
template <int R>
__global__ void __launch_bounds__(kPT) k_part_count(const tgfx_event* __restrict__ ev, int64_t n,
                                                    int64_t per, const int64_t* __restrict__ bounds,
                                                    int N, int64_t nw,
                                                    const int64_t* __restrict__ split,
                                                    int64_t* __restrict__ counts,
                                                    int64_t* __restrict__ scounts) {
  __shared__ int64_t sb[9];
  __shared__ SplitTab st;
  if (threadIdx.x <= N) sb[threadIdx.x] = bounds[threadIdx.x];
  if (threadIdx.x == 0) load_split(split, st);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t w = (blockIdx.x * (int64_t)kPT + threadIdx.x) >> 5;
  if (w >= nw) return;
  const int64_t e0 = w * per, e1 = min(n, e0 + per);
  int64_t c[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  int64_t cs[7] = {0, 0, 0, 0, 0, 0, 0};
  for (int64_t e = e0 + lane; e < e1; e += 32) {
    const Ev x = load_event(ev, e);
#pragma unroll
    for (int side = 0; side < R; ++side) {
      const int64_t u = side ? x.dst : x.src;
      const int si = split_index(st, u);
      const int d = si < 0 ? owner_of(u, sb, N) : -1;
#pragma unroll
      for (int k = 0; k < 8; ++k) c[k] += (k == d);
#pragma unroll
      for (int k = 0; k < 7; ++k) cs[k] += (k == si);
    }
  }
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    int64_t v = c[k];
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
    if (lane == 0 && k < N) counts[w * N + k] = v;
  }
#pragma unroll
  for (int k = 0; k < 7; ++k) {
    int64_t v = cs[k];
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
    if (lane == 0) scounts[w * 7 + k] = v;
  }
}

// stable scatter: offs[w * N + d] = first output slot of warp w's records for rank d;
// occ[w * 7 + i] = occurrences of split node i in this chunk before warp w's range
template <int R>
__global__ void __launch_bounds__(kPT) k_part_scatter(const tgfx_event* __restrict__ ev, int64_t n,
                                                      int64_t per, const int64_t* __restrict__ bounds,
                                                      int N, int64_t nw,
                                                      const int64_t* __restrict__ split,
                                                      const int64_t* __restrict__ occ,
                                                      const int64_t* __restrict__ offs,
                                                      tgfx_event* __restrict__ out) {
  __shared__ int64_t sb[9];
  __shared__ SplitTab st;
  if (threadIdx.x <= N) sb[threadIdx.x] = bounds[threadIdx.x];
  if (threadIdx.x == 0) load_split(split, st);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t w = (blockIdx.x * (int64_t)kPT + threadIdx.x) >> 5;
  if (w >= nw) return;
  const int64_t e0 = w * per, e1 = min(n, e0 + per);
  int64_t cur[8], run[7];
#pragma unroll
  for (int k = 0; k < 8; ++k) cur[k] = k < N ? offs[w * N + k] : 0;
#pragma unroll
  for (int k = 0; k < 7; ++k) run[k] = occ[w * 7 + k];
  const unsigned le = lanemask_lt() | (1u << lane);
  for (int64_t b = e0; b < e1; b += 32) {
    const int64_t e = b + lane;
    const bool ok = e < e1;
    Ev x{0, 0, 0, 0.0};
    if (ok) x = load_event(ev, e);
    // the round's entries in emission order: event-major, src entry then dst entry
    // (tcsr.cpp:99-102) -- an entry's rank in its bucket counts both sides of earlier events
    int si[2] = {-1, -1}, d[2] = {-1, -1};
#pragma unroll
    for (int side = 0; side < R; ++side) {
      const int64_t u = side ? x.dst : x.src;
      si[side] = ok ? split_index(st, u) : -1;
      d[side] = (ok && si[side] < 0) ? owner_of(u, sb, N) : -1;
    }
    // split nodes: the entry's global position gives its owner
#pragma unroll
    for (int k = 0; k < 7; ++k) {
      if (k >= st.ns) break;
      const unsigned ms = __ballot_sync(kFull, si[0] == k);
      const unsigned md = R == 2 ? __ballot_sync(kFull, si[1] == k) : 0u;
#pragma unroll
      for (int side = 0; side < R; ++side) {
        if (si[side] != k) continue;
        const int64_t j = run[k] + __popc(ms & (side ? le : lanemask_lt())) +
                          __popc(md & lanemask_lt());
        const int64_t p = st.gp[k] + j;
        int dd = 0;
        while (dd + 1 < N && st.P[dd + 1] <= p) ++dd;
        d[side] = dd;
      }
      run[k] += __popc(ms) + __popc(md);
    }
    int64_t pos[2] = {0, 0};
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (k >= N) break;
      const unsigned ms = __ballot_sync(kFull, d[0] == k);
      const unsigned md = R == 2 ? __ballot_sync(kFull, d[1] == k) : 0u;
      if (d[0] == k) pos[0] = cur[k] + __popc(ms & lanemask_lt()) + __popc(md & lanemask_lt());
      if (R == 2 && d[1] == k) pos[1] = cur[k] + __popc(ms & le) + __popc(md & lanemask_lt());
      cur[k] += __popc(ms) + __popc(md);
    }
    if (ok) {
#pragma unroll
      for (int side = 0; side < R; ++side) {
        const int64_t u = side ? x.dst : x.src;
        const int64_t other = side ? x.src : x.dst;
        longlong2* o = reinterpret_cast<longlong2*>(out + pos[side]);
        o[0] = make_longlong2(x.eid, u - sb[d[side]]);
        o[1] = make_longlong2(other, __double_as_longlong(x.t));
      }
    }
  }
}

__global__ void k_any_nan(const double* __restrict__ ts, int64_t m, int* flag) {
  bool nan = false;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x)
    nan |= ts[i] != ts[i];
  if (__any_sync(kFull, nan) && (threadIdx.x & 31) == 0) atomicOr(flag, 1);
}

}  // namespace

__global__ void k_indptr_range(const int64_t* __restrict__ indptr, int64_t V, int64_t m,
                               int* bad) {
  for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < V;
       u += (int64_t)gridDim.x * blockDim.x) {
    const int64_t lo = indptr[u], hi = indptr[u + 1];
    if (lo > hi || lo < 0 || hi > m || (u == 0 && lo != 0) || (u == V - 1 && hi != m)) *bad = 1;
  }
}

// indptr[0] == 0, indptr[V] == m and monotone (so every slice lies inside [0, m])
bool indptr_in_range(const int64_t* indptr, int64_t V, int64_t m, cudaStream_t s) {
  if (V <= 0) return true;
  int* d = static_cast<int*>(dmalloc(sizeof(int), s));
  TGFX_CUDA(cudaMemsetAsync(d, 0, sizeof(int), s));
  k_indptr_range<<<static_cast<int>(std::min<int64_t>(ceil_div(V, 256), 4096)), 256, 0, s>>>(
      indptr, V, m, d);
  after_launch("k_indptr_range");
  int h = 0;
  TGFX_CUDA(cudaMemcpyAsync(&h, d, sizeof(int), cudaMemcpyDeviceToHost, s));
  TGFX_CUDA(cudaStreamSynchronize(s));
  dfree(d, s);
  return h == 0;
}

bool any_nan(const double* ts, int64_t m, cudaStream_t s) {
  if (m <= 0) return false;
  int* d = static_cast<int*>(dmalloc(sizeof(int), s));
  TGFX_CUDA(cudaMemsetAsync(d, 0, sizeof(int), s));
  const int grid = static_cast<int>(std::min<int64_t>(ceil_div(m, 256), device_info().sms * 8));
  k_any_nan<<<grid, 256, 0, s>>>(ts, m, d);
  after_launch("k_any_nan");
  int h = 0;
  TGFX_CUDA(cudaMemcpyAsync(&h, d, sizeof(int), cudaMemcpyDeviceToHost, s));
  TGFX_CUDA(cudaStreamSynchronize(s));
  dfree(d, s);
  return h != 0;
}

void launch_degree_hist(const tgfx_event* ev, int64_t n, int64_t V, int reverse,
                        unsigned long long* deg, cudaStream_t s) {
  if (n <= 0) return;
  const int grid = static_cast<int>(std::min<int64_t>(ceil_div(n, kPT), device_info().sms * 8));
  if (reverse)
    k_degree_hist<2><<<grid, kPT, 0, s>>>(ev, n, V, deg);
  else
    k_degree_hist<1><<<grid, kPT, 0, s>>>(ev, n, V, deg);
  after_launch("k_degree_hist");
}

int64_t partition_warps(int64_t n) {
  // one warp per >= 4096 events, at most 16 warps per SM
  return std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, 4096), device_info().sms * 16LL));
}

void launch_partition_count(const tgfx_event* ev, int64_t n, int reverse, const int64_t* bounds,
                            int N, int64_t nw, const int64_t* split, int64_t* counts,
                            int64_t* scounts, cudaStream_t s) {
  const int64_t per = ceil_div(std::max<int64_t>(n, 1), nw);
  const int grid = static_cast<int>(ceil_div(nw * 32, kPT));
  if (reverse)
    k_part_count<2><<<grid, kPT, 0, s>>>(ev, n, per, bounds, N, nw, split, counts, scounts);
  else
    k_part_count<1><<<grid, kPT, 0, s>>>(ev, n, per, bounds, N, nw, split, counts, scounts);
  after_launch("k_part_count");
}

void launch_partition_scatter(const tgfx_event* ev, int64_t n, int reverse, const int64_t* bounds,
                              int N, int64_t nw, const int64_t* split, const int64_t* occ,
                              const int64_t* offs, tgfx_event* out, cudaStream_t s) {
  const int64_t per = ceil_div(std::max<int64_t>(n, 1), nw);
  const int grid = static_cast<int>(ceil_div(nw * 32, kPT));
  if (reverse)
    k_part_scatter<2><<<grid, kPT, 0, s>>>(ev, n, per, bounds, N, nw, split, occ, offs, out);
  else
    k_part_scatter<1><<<grid, kPT, 0, s>>>(ev, n, per, bounds, N, nw, split, occ, offs, out);
  after_launch("k_part_scatter");
}

}  // namespace tgfx
