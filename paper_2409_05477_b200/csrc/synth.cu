// synth.cu -- device generators for the measurement inputs (sm_100a).
//
// * make_random_stream (proj/src/synthetic.cpp:12-43), bit-identical: the reference draws
//   E timestamps next_below(max(1, E/2)) from CounterRng(seed, 0), sorts them, then draws
//   src, dst for event i from draws E+2i, E+2i+1 by lower_bound over the Zipf CDF.  Every
//   draw is O(1) by skip-ahead (x_d = mix64(s0 + d*gamma)), so all draws run in parallel;
//   the sort of integer timestamps < E/2 is a counting sort (histogram, scan, expand).
//   The CDF is computed on the host with glibc pow exactly as the reference does.
// * forward_concat query layout (proj/src/training.cpp:193-209) with index-keyed
//   negatives (proj/src/metrics.cpp:68-69).
#include <cmath>
#include <vector>

#include "graph.cuh"

namespace tgfx {
namespace {

__global__ void k_time_hist(int64_t E, uint64_t s0, uint64_t range, uint32_t* hist) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < E;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t v = mulhi64(rng_draw(s0, static_cast<uint64_t>(i)), range);
    atomicAdd(&hist[v], 1u);
  }
}

// value v occupies sorted positions [off[v], off[v+1])
__global__ void k_time_expand(uint64_t range, const int64_t* __restrict__ off, tgfx_event* ev) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < (int64_t)range;
       v += (int64_t)gridDim.x * blockDim.x) {
    const int64_t a = off[v], b = off[v + 1];
    const double t = static_cast<double>(v);
    for (int64_t p = a; p < b; ++p) ev[p].timestamp = t;
  }
}

__device__ __forceinline__ int64_t lower_bound_cdf(const double* __restrict__ cdf, int64_t n,
                                                   double u) {
  int64_t lo = 0;
  while (n > 0) {
    const int64_t half = n >> 1;
    const bool lt = __ldg(cdf + lo + half) < u;
    lo = lt ? lo + half + 1 : lo;
    n = lt ? n - half - 1 : half;
  }
  return lo;
}

__global__ void k_nodes(int64_t E, int64_t V, uint64_t s0, const double* __restrict__ cdf,
                        tgfx_event* ev) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < E;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t d = static_cast<uint64_t>(E + 2 * i);
    const double us = to_unit_double(rng_draw(s0, d));
    const double ud = to_unit_double(rng_draw(s0, d + 1));
    longlong2 a;
    a.x = i;
    a.y = lower_bound_cdf(cdf, V, us);
    reinterpret_cast<longlong2*>(ev + i)[0] = a;
    ev[i].dst = lower_bound_cdf(cdf, V, ud);
  }
}

__global__ void k_queries(const tgfx_event* __restrict__ ev, int64_t e0, int64_t e1,
                          int64_t batch, int64_t V, uint64_t neg_seed, int64_t* nodes,
                          double* times) {
  const int64_t n = e1 - e0;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n;
       r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e0 + r;
    const int64_t b = r / batch;
    const int64_t s = b * batch;                       // batch start (relative)
    const int64_t bsz = min(batch, n - s);             // batch size
    const int64_t o = 3 * s;                           // output offset of the batch
    const int64_t w = r - s;
    const Ev x = load_event(ev, i);
    nodes[o + w] = x.src;
    times[o + w] = x.t;
    nodes[o + bsz + w] = x.dst;
    times[o + bsz + w] = x.t;
    const uint64_t s0 = rng_state(neg_seed, static_cast<uint64_t>(i));
    nodes[o + 2 * bsz + w] = static_cast<int64_t>(mulhi64(rng_draw(s0, 0), static_cast<uint64_t>(V)));
    times[o + 2 * bsz + w] = x.t;
  }
}

// train_epoch's sample_batch calls (training.cpp:419-473): batch b = events [b*B, b*B + bs) of
// the training stream (make_batches, :157-182), split into `workers` shards [lo, hi) =
// [h*bs/m, (h+1)*bs/m); each shard's call is forward_concat's layout (:193-209)
// [src (pb) | dst (pb) | neg (pb*npp)], neg of batch-relative event r, draw j =
// CounterRng(batch_seed, b).next_below(V) as the (r*npp + j)-th draw.  One thread per event of
// batches [b0, b1); output offset of batch b = (b*B - b0*B) * (2 + npp).
__global__ void k_train_queries(const tgfx_event* __restrict__ ev, int64_t n, int64_t b0,
                                int64_t b1, int64_t B, int64_t npp, int64_t m, int64_t V,
                                uint64_t batch_seed, int64_t* nodes, double* times) {
  const int64_t e0 = b0 * B, e1 = min(n, b1 * B);
  for (int64_t i = e0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < e1;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = i / B;
    const int64_t sb = b * B;
    const int64_t bs = min(B, n - sb);
    const int64_t r = i - sb;
    const int64_t mm = min(m, bs);  // train_epoch: m = min(workers, b)
    // shard h with lo = h*bs/mm <= r < hi: the largest h with h*bs/mm <= r
    int64_t h = (r * mm) / bs;
    while (h + 1 < mm && ((h + 1) * bs) / mm <= r) ++h;
    while (h > 0 && (h * bs) / mm > r) --h;
    const int64_t lo = (h * bs) / mm, hi = ((h + 1) * bs) / mm;
    const int64_t pb = hi - lo, w = r - lo;
    const int64_t o = (sb - e0) * (2 + npp) + lo * (2 + npp);
    const Ev x = load_event(ev, i);
    nodes[o + w] = x.src;
    times[o + w] = x.t;
    nodes[o + pb + w] = x.dst;
    times[o + pb + w] = x.t;
    const uint64_t s0 = rng_state(batch_seed, static_cast<uint64_t>(b));
    for (int64_t j = 0; j < npp; ++j) {
      const int64_t q = o + 2 * pb + w * npp + j;
      nodes[q] = static_cast<int64_t>(
          mulhi64(rng_draw(s0, static_cast<uint64_t>(r * npp + j)), static_cast<uint64_t>(V)));
      times[q] = x.t;
    }
  }
}

int grid_for(int64_t work) {
  return static_cast<int>(
      std::min<int64_t>(ceil_div(std::max<int64_t>(work, 1), 256), device_info().sms * 16));
}

}  // namespace

void launch_random_stream(int64_t E, int64_t V, uint64_t seed, double zipf, tgfx_event* d_out,
                          cudaStream_t s) {
  if (E < 0 || V < 1) throw Error(TGFX_EVALIDATION, "bad stream dimensions");
  if (E == 0) return;
  // synthetic.cpp:16-22 on the host (glibc pow, sequential double sum)
  std::vector<double> cdf(static_cast<size_t>(V));
  double total = 0.0;
  for (int64_t i = 0; i < V; ++i) {
    total += std::pow(static_cast<double>(i + 1), -zipf);
    cdf[i] = total;
  }
  for (double& c : cdf) c /= total;
  double* d_cdf = static_cast<double*>(dmalloc(sizeof(double) * V, s));
  TGFX_CUDA(cudaMemcpyAsync(d_cdf, cdf.data(), sizeof(double) * V, cudaMemcpyHostToDevice, s));
  const uint64_t s0 = rng_state(seed, 0);
  const uint64_t range = E / 2 > 1 ? static_cast<uint64_t>(E / 2) : 1;
  uint32_t* hist = static_cast<uint32_t*>(dmalloc(sizeof(uint32_t) * range, s));
  int64_t* off = static_cast<int64_t*>(dmalloc(sizeof(int64_t) * (range + 1), s));
  TGFX_CUDA(cudaMemsetAsync(hist, 0, sizeof(uint32_t) * range, s));
  k_time_hist<<<grid_for(E), 256, 0, s>>>(E, s0, range, hist);
  after_launch("k_time_hist");
  scan_u32_to_i64(hist, static_cast<int64_t>(range), off, s);
  k_time_expand<<<grid_for(range), 256, 0, s>>>(range, off, d_out);
  after_launch("k_time_expand");
  k_nodes<<<grid_for(E), 256, 0, s>>>(E, V, s0, d_cdf, d_out);
  after_launch("k_nodes");
  dfree(hist, s);
  dfree(off, s);
  dfree(d_cdf, s);
}

void launch_make_queries(const tgfx_event* ev, int64_t e0, int64_t e1, int64_t batch, int64_t V,
                         uint64_t neg_seed, int64_t* nodes, double* times, cudaStream_t s) {
  if (e1 <= e0) return;
  if (batch < 1) throw Error(TGFX_EVALIDATION, "bad batch parameters");
  k_queries<<<grid_for(e1 - e0), 256, 0, s>>>(ev, e0, e1, batch, V, neg_seed, nodes, times);
  after_launch("k_queries");
}

void launch_train_queries(const tgfx_event* ev, int64_t n, int64_t b0, int64_t b1, int64_t B,
                          int64_t npp, int64_t workers, int64_t V, uint64_t batch_seed,
                          int64_t* nodes, double* times, cudaStream_t s) {
  // make_batches (training.cpp:160-161) and train config checks
  if (n == 0) throw Error(TGFX_EVALIDATION, "empty training stream");
  if (B < 1 || npp < 1) throw Error(TGFX_EVALIDATION, "bad batch parameters");
  if (workers < 1) throw Error(TGFX_EVALIDATION, "workers must be >= 1");
  if (b0 < 0 || b1 < b0 || b1 > ceil_div(n, B)) throw Error(TGFX_EVALIDATION, "bad batch range");
  if (b1 == b0) return;
  k_train_queries<<<grid_for(std::min(n, b1 * B) - b0 * B), 256, 0, s>>>(
      ev, n, b0, b1, B, npp, workers, V, batch_seed, nodes, times);
  after_launch("k_train_queries");
}

}  // namespace tgfx
