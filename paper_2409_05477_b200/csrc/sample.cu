// sample.cu -- temporal neighbor sampler fused with the sequence assembler (sm_100a).
//
// Replaces sample_batch / sample_recent / sample_random (proj/src/sampler.cpp:16-104) and
// build_sequence_batch (proj/src/sequence.cpp:55-86):
//
//   * the strict-before-t prefix m(u, t) = #{ts < t} of a slice (lower_bound,
//     sampler.cpp:16-20; NaN t -> 0) is found by search_lines: the slice's time bucket
//     (build.cu, build_node_dir) narrows it to ~4 entries, then interpolated probes each read
//     and resolve a whole kProbeW-entry ts line, bracketed by the node directory record
//     (slice bounds + first/last ts + bucket grid).  Any search that keeps
//     ts[lo-1] < t <= ts[hi] returns the unique lower_bound on a sorted, NaN-free slice;
//     graphs not known to be sorted and NaN-free replay std::lower_bound's own bisection
//     (search_interleaved) instead.
//   * recent-k (k_recent_line): one query per lane for the search, then the warp assembles its
//     32 rows "slot-parallel": lane s handles output slot s of the warp's [32 x l] block, so
//     window gathers are near-contiguous and every store is a coalesced run; window entries
//     come from the graph's 16-byte gather records, staged in shared memory and written out
//     by bulk copies.
//   * uniform-k: Floyd's algorithm with the reference's counter RNG (rng.hpp:23-38,
//     sampler.cpp:66-80): draw d by O(1) skip-ahead (x_d = mix64(s0 + d*gamma)), a repeat
//     resolved in order d -- one query per lane with draws and ranks in registers
//     (k_random_lane, int32 rows, k <= 32), by 8-lane groups with ballots and shuffles
//     (k_random_g, k <= 32) or by the whole warp (k_random, larger k / exact search).
//   * suffix infilling epilogue: ids + 1, self-edge token at column kb, zero padding,
//     dt = t_q - ts in fp64 then rounded to fp32 (and/or kept as fp64).
#include <algorithm>

#include <cuda_bf16.h>

#include "graph.cuh"

namespace tgfx {
namespace {

constexpr int kThreads = 256;
// entries per line probe of the bucketed search: with 4-entry time buckets the candidate
// range is ~4 entries, so one 32-byte sector per probe (measured: sampling 34.1 ms/step
// against 35.8 ms for 8-entry probes over 8-entry buckets; L1 wavefronts are the co-limiter)
constexpr int kProbeW = 4;
constexpr int kWarps = kThreads / 32;

template <typename T>
__device__ __forceinline__ void st(void* p, int64_t i, T v) {
  static_cast<T*>(p)[i] = v;
}

struct QueryIn {
  const int64_t* nodes;
  const double* times;
  const int64_t* hop_counts;  // hop-2 mode: presence of virtual query qq = r*k1 + j
  int64_t hop_k1;
  // batched mode (uniform-k): query qq belongs to batch b = qq / batch_q, sampled as one
  // sample_batch(seed = seeds[b]) call: RNG stream = qq - b * batch_q (sampler.cpp:100-101)
  const uint64_t* seeds = nullptr;
  int64_t batch_q = 0;
  // query node range check fused into the sampler (check_query, sampler.cpp:22-27): a node
  // outside [0, V) is never looked up (its row is written as an absent one); with `bad` set
  // the smallest failing bad_base + q is recorded there for the caller to raise
  int64_t V = 0;
  unsigned long long* bad = nullptr;
  uint64_t bad_base = 0;
};

// CounterRng(seed, stream) initial state of query qq (rng.hpp:23-24)
// Dead lanes (qq >= Q) still evaluate it; their batch index is clamped to the last query's so
// the seeds[] load stays inside the caller's array.
__device__ __forceinline__ uint64_t query_rng(const QueryIn& in, uint64_t seed_mix,
                                              uint64_t stream_base, int64_t qq, int64_t Q) {
  if (in.seeds) {
    const int64_t b = min(qq, Q - 1) / in.batch_q;
    return mix64(mix64(__ldg(reinterpret_cast<const unsigned long long*>(in.seeds) + b)) ^
                 (static_cast<uint64_t>(qq - b * in.batch_q) * kStreamMul));
  }
  return mix64(seed_mix ^ ((stream_base + static_cast<uint64_t>(qq)) * kStreamMul));
}

__device__ __forceinline__ bool fetch_query(const QueryIn& in, int64_t q, int64_t& u, double& t) {
  if (in.hop_counts) {
    const int64_t r = q / in.hop_k1, j = q - r * in.hop_k1;
    if (j >= __ldg(reinterpret_cast<const long long*>(in.hop_counts) + r)) return false;
  }
  u = static_cast<int64_t>(__ldcs(reinterpret_cast<const long long*>(in.nodes) + q));
  t = __ldcs(in.times + q);
  if (static_cast<uint64_t>(u) >= static_cast<uint64_t>(in.V)) {
    if (in.bad) atomicMin(in.bad, static_cast<unsigned long long>(in.bad_base + q));
    return false;
  }
  return true;
}

struct Outs {
  void* node;   // int32 or int64 [Q*l]
  void* edge;
  float* dt32;
  double* dt64;
  void* vlen;   // int32 or int64 [Q]
  int64_t* counts;  // entries mode
  int64_t* e_nbr;
  int64_t* e_eid;
  double* e_ts;
  int64_t es;  // entry stride in 8-byte words: 1 = three columns, 3 = tgfx_neighbor records
};

__device__ __forceinline__ void put_entry(const Outs& o, int64_t i, int64_t nb, int64_t ed,
                                          double t) {
  o.e_nbr[i * o.es] = nb;
  o.e_eid[i * o.es] = ed;
  o.e_ts[i * o.es] = t;
}

// Output rows are written once and never re-read by the kernel: streaming (evict-first)
// stores keep them from pushing the T-CSR lines the searches reuse out of L2.
template <bool IDX64>
__device__ __forceinline__ void write_slot(const Outs& o, int64_t i, int64_t ni, int64_t ei,
                                           double dt) {
  if (IDX64) {
    __stcs(reinterpret_cast<long long*>(o.node) + i, static_cast<long long>(ni));
    __stcs(reinterpret_cast<long long*>(o.edge) + i, static_cast<long long>(ei));
  } else {
    __stcs(static_cast<int*>(o.node) + i, static_cast<int>(ni));
    __stcs(static_cast<int*>(o.edge) + i, static_cast<int>(ei));
  }
  if (o.dt32) __stcs(o.dt32 + i, __double2float_rn(dt));
  if (o.dt64) __stcs(o.dt64 + i, dt);
}

template <bool IDX64>
__device__ __forceinline__ void write_vlen(const Outs& o, int64_t q, int64_t v) {
  if (IDX64)
    st<int64_t>(o.vlen, q, v);
  else
    st<int32_t>(o.vlen, q, static_cast<int32_t>(v));
}

// one slice entry for the window / sample gathers: from the 16-byte gather record when the
// graph has them (ids < 2^31, so the widening is exact), else from the three columns
__device__ __forceinline__ void fetch_entry(const uint4* __restrict__ rec,
                                            const int64_t* __restrict__ nbr,
                                            const int64_t* __restrict__ eid,
                                            const double* __restrict__ ts, int64_t p,
                                            int64_t& ni, int64_t& ei, double& tv) {
  if (rec) {
    const uint4 r = __ldg(rec + p);
    ni = r.x;
    ei = r.y;
    tv = __hiloint2double(static_cast<int>(r.w), static_cast<int>(r.z));
  } else {
    ni = ldg_i64(nbr + p);
    ei = ldg_i64(eid + p);
    tv = ldg_f64(ts + p);
  }
}

// the same as fetch_entry, as volatile asm: the loads stay where they are written (issued
// together ahead of their uses) instead of being sunk into the uses' branches
__device__ __forceinline__ void fetch_entry_v(const uint4* __restrict__ rec,
                                              const int64_t* __restrict__ nbr,
                                              const int64_t* __restrict__ eid,
                                              const double* __restrict__ ts, int64_t p,
                                              int64_t& ni, int64_t& ei, double& tv) {
  if (rec) {
    uint32_t a, b, c, e;
    asm volatile("ld.global.nc.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(a), "=r"(b), "=r"(c), "=r"(e) : "l"(rec + p));
    ni = a;
    ei = b;
    tv = __hiloint2double(static_cast<int>(e), static_cast<int>(c));
  } else {
    long long a, b;
    asm volatile("ld.global.nc.s64 %0, [%1];" : "=l"(a) : "l"(nbr + p));
    asm volatile("ld.global.nc.s64 %0, [%1];" : "=l"(b) : "l"(eid + p));
    asm volatile("ld.global.nc.f64 %0, [%1];" : "=d"(tv) : "l"(ts + p));
    ni = a;
    ei = b;
  }
}

// write_slot under a predicate, as predicated stores (no branch for ptxas to sink loads into)
template <bool IDX64>
__device__ __forceinline__ void write_slot_if(const Outs& o, int64_t i, int64_t ni, int64_t ei,
                                              double dt, bool pred) {
  const int pi = pred ? 1 : 0;
  if (IDX64) {
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q st.global.cs.s64 [%0], %1;\n\t}"
                 ::"l"(reinterpret_cast<long long*>(o.node) + i), "l"(static_cast<long long>(ni)), "r"(pi)
                 : "memory");
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q st.global.cs.s64 [%0], %1;\n\t}"
                 ::"l"(reinterpret_cast<long long*>(o.edge) + i), "l"(static_cast<long long>(ei)), "r"(pi)
                 : "memory");
  } else {
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q st.global.cs.s32 [%0], %1;\n\t}"
                 ::"l"(static_cast<int*>(o.node) + i), "r"(static_cast<int>(ni)), "r"(pi)
                 : "memory");
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q st.global.cs.s32 [%0], %1;\n\t}"
                 ::"l"(static_cast<int*>(o.edge) + i), "r"(static_cast<int>(ei)), "r"(pi)
                 : "memory");
  }
  if (o.dt32)
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q st.global.cs.f32 [%0], %1;\n\t}"
                 ::"l"(o.dt32 + i), "f"(__double2float_rn(dt)), "r"(pi)
                 : "memory");
  if (o.dt64)
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q st.global.cs.f64 [%0], %1;\n\t}"
                 ::"l"(o.dt64 + i), "d"(dt), "r"(pi)
                 : "memory");
}

// ------------------------------------------------------------------ recent-k
// QL queries per lane: their binary searches are interleaved step by step so each lane keeps
// QL independent loads in flight (the search is a chain of dependent L2/HBM round trips).
template <int QL>
__device__ __forceinline__ void search_interleaved(const double* __restrict__ ts,
                                                   const int64_t (&lo)[QL], int64_t (&n)[QL],
                                                   const double (&t)[QL], int64_t (&m)[QL]) {
  int64_t base[QL];
#pragma unroll
  for (int j = 0; j < QL; ++j) base[j] = lo[j];
  while (true) {
    bool any = false;
#pragma unroll
    for (int j = 0; j < QL; ++j) any |= n[j] > 0;
    if (!any) break;
    double v[QL];
#pragma unroll
    for (int j = 0; j < QL; ++j) v[j] = n[j] > 0 ? __ldg(ts + base[j] + (n[j] >> 1)) : 0.0;
#pragma unroll
    for (int j = 0; j < QL; ++j) {
      if (n[j] > 0) {
        const int64_t half = n[j] >> 1;
        const bool lt = v[j] < t[j];
        base[j] = lt ? base[j] + half + 1 : base[j];
        n[j] = lt ? n[j] - half - 1 : half;
      }
    }
  }
#pragma unroll
  for (int j = 0; j < QL; ++j) m[j] = base[j] - lo[j];
}

// floor(s / w) for s < 2^16 via a 32-bit multiply-high (magic = ceil(2^32 / w)), else divide
__device__ __forceinline__ int div_slot(int s, int w, uint32_t magic) {
  return magic ? static_cast<int>(__umulhi(static_cast<uint32_t>(s), magic)) : s / w;
}

// ASSEMBLE: rows [Q, l]; else entries [Q, k] + counts.
template <bool ASSEMBLE, bool IDX64, int QL, int MINB>
__global__ void __launch_bounds__(kThreads, MINB) k_recent(
    const int64_t* __restrict__ indptr, const int64_t* __restrict__ nbr,
    const int64_t* __restrict__ eid, const double* __restrict__ ts, QueryIn in, int64_t Q,
    int64_t k, int l, int64_t self_idx, uint32_t magic, Outs o, const uint4* __restrict__ rec) {
  constexpr int GQ = 32 * QL;  // queries per warp group
  __shared__ int64_t s_start[kWarps][GQ];
  __shared__ int64_t s_u[kWarps][GQ];
  __shared__ double s_t[kWarps][GQ];
  __shared__ int s_kb[kWarps][GQ];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int width = ASSEMBLE ? l : static_cast<int>(k);
  const int64_t ngroups = ceil_div(Q, GQ);
  for (int64_t g = static_cast<int64_t>(blockIdx.x) * kWarps + warp; g < ngroups;
       g += static_cast<int64_t>(gridDim.x) * kWarps) {
    int64_t u[QL], lo[QL], n[QL], m[QL];
    double t[QL];
    bool pres[QL];
#pragma unroll
    for (int j = 0; j < QL; ++j) {
      const int64_t q = g * GQ + j * 32 + lane;
      u[j] = 0;
      t[j] = 0.0;
      pres[j] = q < Q && fetch_query(in, q, u[j], t[j]);
    }
#pragma unroll
    for (int j = 0; j < QL; ++j) {
      lo[j] = pres[j] ? ldg_i64(indptr + u[j]) : 0;
      n[j] = pres[j] ? ldg_i64(indptr + u[j] + 1) - lo[j] : 0;
    }
    search_interleaved<QL>(ts, lo, n, t, m);
#pragma unroll
    for (int j = 0; j < QL; ++j) {
      const int64_t q = g * GQ + j * 32 + lane;
      int kb = -1;  // -1: absent (hop-2 padding) -> zero row, valid_len 0
      if (pres[j]) {
        const int64_t take = min(k, m[j]);
        kb = static_cast<int>(ASSEMBLE ? min(take, static_cast<int64_t>(l - 1)) : take);
      }
      if (q < Q) {
        if (ASSEMBLE)
          write_vlen<IDX64>(o, q, kb + 1);
        else
          o.counts[q] = max(kb, 0);
      }
      const int qi = j * 32 + lane;
      s_start[warp][qi] = lo[j] + m[j] - kb;
      s_u[warp][qi] = u[j];
      s_t[warp][qi] = t[j];
      s_kb[warp][qi] = kb;
    }
    __syncwarp();
    const int64_t qbase = g * GQ;
    const int nq = static_cast<int>(min(static_cast<int64_t>(GQ), Q - qbase));
    const int total = nq * width;
    const int64_t obase = qbase * width;
#pragma unroll 8
    for (int s = lane; s < total; s += 32) {
      const int qi = div_slot(s, width, magic);
      const int j = s - qi * width;
      const int kbq = s_kb[warp][qi];
      if (ASSEMBLE) {
        int64_t ni = 0, ei = 0;
        double dt = 0.0;
        if (j < kbq) {
          double tv;
          fetch_entry(rec, nbr, eid, ts, s_start[warp][qi] + j, ni, ei, tv);
          ++ni;
          ++ei;
          dt = s_t[warp][qi] - tv;
        } else if (j == kbq) {
          ni = s_u[warp][qi] + 1;
          ei = self_idx;
        }
        write_slot<IDX64>(o, obase + s, ni, ei, dt);
      } else {
        int64_t a = 0, b = 0;
        double c = 0.0;
        if (j < kbq) fetch_entry(rec, nbr, eid, ts, s_start[warp][qi] + j, a, b, c);
        put_entry(o, obase + s, a, b, c);
      }
    }
    __syncwarp();
  }
}

// ------------------------------------------------------------------ recent-k, line probes
// Default recent-k kernel.  Per query the dependent round trips are
//   (1) node, time          coalesced
//   (2) node directory      one 32-byte record: slice bounds + ts of its first and last entry,
//                           i.e. the interpolation bracket comes with the bounds
//   (3..) line probes       each probe reads the W-entry aligned ts line (W*8 bytes, 16-byte
//                           vector loads) around the interpolated position and resolves the
//                           whole line against t: either the answer is inside the line (done)
//                           or the bracket shrinks to the line's edge.  A probe that fails to
//                           halve the bracket is followed by a bisection probe, so the result
//                           is exactly std::lower_bound's on the sorted slice.
//   (last) window gather    suffix-infill rows written slot-parallel (coalesced), as k_recent.
// On the GDELT-shaped workload this is ~3 probe rounds per query on average (vs ~13 for
// bisection and ~7 for point interpolation), and ~5.5 for the slowest lane of a warp.
// one 64-byte directory record (two 256-bit loads); absent queries get an empty record
__device__ __forceinline__ NodeDir load_dir(const NodeDir* __restrict__ dir, int64_t u, bool pres) {
  NodeDir d;
  if (pres) {
    unsigned long long x0, x1, x2, x3, y0, y1, y2, y3;
    const NodeDir* p = dir + u;
    asm volatile("ld.global.nc.v4.u64 {%0, %1, %2, %3}, [%4];"
                 : "=l"(x0), "=l"(x1), "=l"(x2), "=l"(x3) : "l"(p));
    asm volatile("ld.global.nc.v4.u64 {%0, %1, %2, %3}, [%4];"
                 : "=l"(y0), "=l"(y1), "=l"(y2), "=l"(y3) : "l"(reinterpret_cast<const char*>(p) + 32));
    d.start = static_cast<int64_t>(x0);
    d.end = static_cast<int64_t>(x1);
    d.t_first = __longlong_as_double(static_cast<long long>(x2));
    d.t_last = __longlong_as_double(static_cast<long long>(x3));
    d.bkt = reinterpret_cast<const uint32_t*>(y0);
    d.scale = __longlong_as_double(static_cast<long long>(y1));
    d.nb = static_cast<int64_t>(y2);
    d.width = __longlong_as_double(static_cast<long long>(y3));
  } else {
    d.start = d.end = 0;
    d.t_first = d.t_last = 0.0;
    d.bkt = nullptr;
    d.scale = 0.0;
    d.nb = 0;
    d.width = 0.0;
  }
  return d;
}

// the compact directory record (graph.cuh DirC): ONE 256-bit load.  t_last is only known for
// slices without buckets (+inf otherwise: the bracket then starts at n and the last bucket's
// table entries close it); the bucket edges' width, an interpolation hint, from 1 / scale
__device__ __forceinline__ NodeDir load_dirc(const DirC* __restrict__ dirc,
                                             const uint32_t* __restrict__ bkt, int rshift,
                                             int64_t u, bool pres) {
  NodeDir d;
  if (pres) {
    unsigned long long x0, x1, x2, x3;
    asm volatile("ld.global.nc.v4.u64 {%0, %1, %2, %3}, [%4];"
                 : "=l"(x0), "=l"(x1), "=l"(x2), "=l"(x3) : "l"(dirc + u));
    const uint32_t n = static_cast<uint32_t>(x1), nb = static_cast<uint32_t>(x1 >> 32);
    const double st = __longlong_as_double(static_cast<long long>(x3));
    d.start = static_cast<int64_t>(x0);
    d.end = d.start + n;
    d.t_first = __longlong_as_double(static_cast<long long>(x2));
    d.nb = nb;
    if (nb) {
      d.t_last = __longlong_as_double(0x7ff0000000000000LL);  // unknown: +inf
      d.bkt = bkt + (d.start >> rshift) + 2 * u;
      d.scale = st;
      d.width = static_cast<double>(__frcp_rn(static_cast<float>(st)));
    } else {
      d.t_last = st;
      d.bkt = nullptr;
      d.scale = 0.0;
      d.width = 0.0;
    }
  } else {
    d.start = d.end = 0;
    d.t_first = d.t_last = 0.0;
    d.bkt = nullptr;
    d.scale = 0.0;
    d.nb = 0;
    d.width = 0.0;
  }
  return d;
}

template <int W, int QL>
__device__ __forceinline__ void search_lines(const double* __restrict__ ts, const NodeDir (&d)[QL],
                                             const bool (&pres)[QL], const double (&t)[QL],
                                             int64_t (&m)[QL]) {
  int64_t lo[QL], hi[QL];
  double vlo[QL], vhi[QL];
  bool bis[QL];
#pragma unroll
  for (int j = 0; j < QL; ++j) {
    const int64_t n = d[j].end - d[j].start;
    bis[j] = false;
    vlo[j] = d[j].t_first;
    vhi[j] = d[j].t_last;
    if (!pres[j] || n <= 0 || !(d[j].t_first < t[j])) {  // empty, t <= first, NaN t
      lo[j] = hi[j] = 0;
    } else if (d[j].t_last < t[j]) {
      lo[j] = hi[j] = n;
    } else {
      lo[j] = 1;
      // t_last +inf (unknown in the compact record, or a real +inf): the answer may be n
      hi[j] = isinf(d[j].t_last) ? n : n - 1;
    }
  }
  // time buckets: [lo, hi] narrows to [bkt[j], bkt[j + 1]] (typically ~R entries, one or two
  // lines); the interpolation hints become the bucket's edges
  // (ts[bkt[j] - 1] < t < ts[bkt[j + 1]], so the invariant ts[lo - 1] < t <= ts[hi] holds)
#pragma unroll
  for (int j = 0; j < QL; ++j) {
    if (lo[j] < hi[j] && d[j].bkt) {
      const int64_t jb = bucket_of(t[j], d[j].t_first, d[j].scale, d[j].nb);
      const int64_t b0 = __ldg(d[j].bkt + jb), b1 = __ldg(d[j].bkt + jb + 1);
      lo[j] = max(b0, lo[j]);
      hi[j] = min(b1, hi[j]);
      vlo[j] = d[j].t_first + static_cast<double>(jb) * d[j].width;  // interpolation hints
      vhi[j] = vlo[j] + d[j].width;
    }
  }
  while (true) {
    bool any = false;
#pragma unroll
    for (int j = 0; j < QL; ++j) any |= lo[j] < hi[j];
    if (!any) break;
    int64_t a[QL], b[QL], A[QL];
    double v[QL][W];
#pragma unroll
    for (int j = 0; j < QL; ++j) {
      const int64_t len = hi[j] - lo[j];
      int64_t p = lo[j] + (len >> 1);
      if (!bis[j]) {
        const float f = __fdividef(static_cast<float>(t[j] - vlo[j]),
                                   static_cast<float>(vhi[j] - vlo[j]));
        if (f >= 0.0f && f <= 1.0f)
          p = lo[j] - 1 + static_cast<int64_t>(static_cast<double>(f) * static_cast<double>(len + 1));
        p = max(lo[j], min(p, hi[j] - 1));
      }
      A[j] = (d[j].start + p) & ~static_cast<int64_t>(W - 1);  // aligned line (absolute)
      a[j] = max(A[j] - d[j].start, lo[j]);
      b[j] = min(A[j] - d[j].start + W, hi[j]);
      if (len > 0) {
        // 256-bit loads (LDG.E.ENL2.256, sm_100): one L1 wavefront per 32-byte sector
        // instead of two 128-bit loads per sector -- the probe loop is L1-throughput-bound
        const double* src = ts + A[j];
#pragma unroll
        for (int w = 0; w < W / 4; ++w)
          asm volatile("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];"
                       : "=d"(v[j][4 * w]), "=d"(v[j][4 * w + 1]), "=d"(v[j][4 * w + 2]),
                         "=d"(v[j][4 * w + 3])
                       : "l"(src + 4 * w));
      }
    }
#pragma unroll
    for (int j = 0; j < QL; ++j) {
      const int64_t len = hi[j] - lo[j];
      if (len > 0) {
        const int64_t r0 = A[j] - d[j].start;  // relative index of line entry 0
        int c = 0;
        double first = 0.0, last = 0.0;
#pragma unroll
        for (int w = 0; w < W; ++w) {
          const bool in = r0 + w >= a[j] && r0 + w < b[j];
          c += (in && v[j][w] < t[j]) ? 1 : 0;
          if (r0 + w == a[j]) first = v[j][w];
          if (r0 + w == b[j] - 1) last = v[j][w];
        }
        const int64_t span = b[j] - a[j];
        if (c == span) {
          lo[j] = b[j];
          vlo[j] = last;
        } else if (c == 0) {
          hi[j] = a[j];
          vhi[j] = first;
        } else {
          lo[j] = hi[j] = a[j] + c;
        }
        bis[j] = !bis[j] && 2 * (hi[j] - lo[j]) > len;
      }
    }
  }
#pragma unroll
  for (int j = 0; j < QL; ++j) m[j] = lo[j];
}

// BULK: a full group's [32 x l] output block is staged in shared memory and written by three
// 1-D bulk copies (cp.async.bulk.global.shared::cta, the TMA engine) instead of 3 x l / 32
// strided store instructions per lane; l <= kBulkMaxL, int32/fp32 outputs, 16-byte aligned.
constexpr int kBulkMaxL = 16;

// REC: the window gather reads the graph's 16-byte records (tgfx_graph::rec) instead of the
// three columns: one 16-byte load per slot
// DC: the compact 32-byte directory (one load per query instead of two)
template <bool ASSEMBLE, bool IDX64, int W, int QL, int MINB, bool BULK = false, bool REC = false,
          int UNR = 4, bool DC = false>
__global__ void __launch_bounds__(kThreads, MINB) k_recent_line(
    const NodeDir* __restrict__ dir, const int64_t* __restrict__ nbr,
    const int64_t* __restrict__ eid, const double* __restrict__ ts, QueryIn in, int64_t Q,
    int64_t k, int l, int64_t self_idx, uint32_t magic, Outs o,
    const uint4* __restrict__ rec = nullptr, const DirC* __restrict__ dirc = nullptr,
    const uint32_t* __restrict__ bkt = nullptr, int rshift = 0) {
  constexpr int GQ = 32 * QL;
  // BULK staging: per warp [3][32 * l] 32-bit words (node, edge, dt)
  extern __shared__ __align__(16) uint32_t s_out[];
  __shared__ longlong2 s_st[kWarps][GQ];  // {window start, query time bits}: one LDS.128
  // BULK: {window start << 5 | kb + 1, query time bits} -- a slot's whole staging read is one
  // LDS.128 (kb <= 15 there); the self-loop token is stored by the query's own lane afterwards
  __shared__ longlong2 s_bk[BULK ? kWarps : 1][BULK ? GQ : 1];
  __shared__ int64_t s_u[kWarps][GQ];
  __shared__ int s_kb[kWarps][GQ];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int width = ASSEMBLE ? l : static_cast<int>(k);
  const int64_t ngroups = ceil_div(Q, GQ);
  // BULK launches cover every group with the grid (one group per warp, launch_sample checks):
  // the loop then runs at most once and carries no counter (which was spilled at 64 registers)
  for (int64_t g = static_cast<int64_t>(blockIdx.x) * kWarps + warp; g < ngroups;
       g = BULK ? ngroups : g + static_cast<int64_t>(gridDim.x) * kWarps) {
    int64_t u[QL], m[QL];
    double t[QL];
    bool pres[QL];
    NodeDir d[QL];
#pragma unroll
    for (int j = 0; j < QL; ++j) {
      const int64_t q = g * GQ + j * 32 + lane;
      u[j] = 0;
      t[j] = 0.0;
      pres[j] = q < Q && fetch_query(in, q, u[j], t[j]);
    }
#pragma unroll
    for (int j = 0; j < QL; ++j)  // bounds + bracket + buckets
      d[j] = DC ? load_dirc(dirc, bkt, rshift, u[j], pres[j]) : load_dir(dir, u[j], pres[j]);
    search_lines<W, QL>(ts, d, pres, t, m);
#pragma unroll
    for (int j = 0; j < QL; ++j) {
      const int64_t q = g * GQ + j * 32 + lane;
      int kb = -1;  // -1: absent (hop-2 padding) -> zero row, valid_len 0
      if (pres[j]) {
        const int64_t take = min(k, m[j]);
        kb = static_cast<int>(ASSEMBLE ? min(take, static_cast<int64_t>(l - 1)) : take);
      }
      if (q < Q) {
        if (ASSEMBLE)
          write_vlen<IDX64>(o, q, kb + 1);
        else
          o.counts[q] = max(kb, 0);
      }
      const int qi = j * 32 + lane;
      s_st[warp][qi] = make_longlong2(d[j].start + m[j] - kb, __double_as_longlong(t[j]));
      s_u[warp][qi] = u[j];
      s_kb[warp][qi] = kb;
      if (BULK)
        s_bk[warp][qi] = make_longlong2(((d[j].start + m[j] - kb) << 5) | (kb + 1),
                                        __double_as_longlong(t[j]));
    }
    __syncwarp();
    const int64_t qbase = g * GQ;
    const int nq = static_cast<int>(min(static_cast<int64_t>(GQ), Q - qbase));
    const int total = nq * width;
    const int64_t obase = qbase * width;
    // slot s = lane + 32 i of the warp's [nq x width] block: (query, column) advanced
    // incrementally instead of divided per slot
    int qi = div_slot(lane, width, magic);
    int j = lane - qi * width;
    const int dq = div_slot(32, width, magic), dj = 32 - dq * width;
    if (BULK && nq == GQ) {
      // staging arrays padded to lp = l rounded up to UNR slots per lane: phase B stores every
      // slot of a chunk unconditionally (a conditional store lets ptxas sink its load into the
      // branch, which serialises the chunk's loads again); the padding is never copied out
      const int lp = (l + UNR - 1) / UNR * UNR;
      uint32_t* sn = s_out + static_cast<size_t>(warp) * 3 * GQ * lp;
      uint32_t* se = sn + GQ * lp;
      float* sd = reinterpret_cast<float*>(se + GQ * lp);
      // each lane fills slots s = lane + 32 it, it < l, in chunks of UNR: all of a chunk's
      // loads are issued (phase A) before any result is stored (phase B) -- the compiler will
      // not hoist a slot's loads above the previous slot's shared-memory stores by itself
      for (int it0 = 0; it0 < QL * l; it0 += UNR) {
        uint32_t rn[UNR], re[UNR];
        double tv[UNR], tq[UNR];
        bool tk[UNR];
#pragma unroll
        for (int uu = 0; uu < UNR; ++uu) {
          const bool valid = it0 + uu < QL * l;
          const int qr = valid ? qi : 0;  // padding slots run qi past the warp's 32 queries
          const longlong2 st = s_bk[warp][qr];
          const int kbq = static_cast<int>(st.x & 31) - 1;
          tk[uu] = valid && j < kbq;
          tq[uu] = __longlong_as_double(st.y);
          const int64_t p = tk[uu] ? (st.x >> 5) + j : 0;
          // volatile: keeps the loads here, unconditional, instead of sunk into phase B's
          // per-slot branches (which would serialise them again)
          if (REC) {
            uint32_t c, e;
            asm volatile("ld.global.v4.u32 {%0, %1, %2, %3}, [%4];"
                         : "=r"(rn[uu]), "=r"(re[uu]), "=r"(c), "=r"(e) : "l"(rec + p));
            tv[uu] = __hiloint2double(static_cast<int>(e), static_cast<int>(c));
          } else {
            unsigned long long a, b;
            asm volatile("ld.global.nc.u64 %0, [%1];" : "=l"(a) : "l"(nbr + p));
            asm volatile("ld.global.nc.u64 %0, [%1];" : "=l"(b) : "l"(eid + p));
            asm volatile("ld.global.nc.f64 %0, [%1];" : "=d"(tv[uu]) : "l"(ts + p));
            rn[uu] = static_cast<uint32_t>(a);
            re[uu] = static_cast<uint32_t>(b);
          }
          j += dj;
          qi += dq;
          if (j >= width) {
            j -= width;
            ++qi;
          }
        }
#pragma unroll
        for (int uu = 0; uu < UNR; ++uu) {
          const int s = lane + 32 * (it0 + uu);
          sn[s] = tk[uu] ? rn[uu] + 1u : 0u;
          se[s] = tk[uu] ? re[uu] + 1u : 0u;
          sd[s] = tk[uu] ? __double2float_rn(tq[uu] - tv[uu]) : 0.0f;
        }
      }
      __syncwarp();
      // the self-loop token of each query (sequence.cpp:79-81), by the query's own lane
#pragma unroll
      for (int jq = 0; jq < QL; ++jq) {
        const int qq = jq * 32 + lane;
        const int kbq = s_kb[warp][qq];
        if (kbq >= 0) {
          sn[qq * width + kbq] = static_cast<uint32_t>(u[jq] + 1);
          se[qq * width + kbq] = static_cast<uint32_t>(self_idx);
        }
      }
      __syncwarp();
      if (lane == 0) {
        // the rows are never re-read here: evict-first in L2 leaves the T-CSR windows' lines
        // resident (round 2: 1.234 -> 1.231 ms per GDELT launch)
        const uint32_t bytes = static_cast<uint32_t>(total) * 4u;
        uint64_t pol;
        asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile(
            "cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(
                static_cast<int32_t*>(o.node) + obase),
            "r"(static_cast<uint32_t>(__cvta_generic_to_shared(sn))), "r"(bytes), "l"(pol)
            : "memory");
        asm volatile(
            "cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(
                static_cast<int32_t*>(o.edge) + obase),
            "r"(static_cast<uint32_t>(__cvta_generic_to_shared(se))), "r"(bytes), "l"(pol)
            : "memory");
        asm volatile(
            "cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(
                o.dt32 + obase),
            "r"(static_cast<uint32_t>(__cvta_generic_to_shared(sd))), "r"(bytes), "l"(pol)
            : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        // the staging is reused by this warp's next group / freed at exit: wait for the reads
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      }
      __syncwarp();
      continue;
    }
#pragma unroll 4
    for (int s = lane; s < total; s += 32) {
      const int kbq = s_kb[warp][qi];
      const longlong2 st = s_st[warp][qi];
      const bool take = j < kbq;
      int64_t ni, ei;
      double tv;
      fetch_entry(rec, nbr, eid, ts, take ? st.x + j : 0, ni, ei, tv);  // branch-free loads
      if (ASSEMBLE) {
        const bool self = j == kbq;
        const int64_t su = s_u[warp][qi];
        write_slot<IDX64>(o, obase + s, take ? ni + 1 : self ? su + 1 : 0,
                          take ? ei + 1 : self ? self_idx : 0,
                          take ? __longlong_as_double(st.y) - tv : 0.0);
      } else {
        put_entry(o, obase + s, take ? ni : 0, take ? ei : 0, take ? tv : 0.0);
      }
      j += dj;
      qi += dq;
      if (j >= width) {
        j -= width;
        ++qi;
      }
    }
    __syncwarp();
  }
}

// ------------------------------------------------------------------ sampler + assemble_inputs
// forward_concat's sample_batch -> build_sequence_batch -> model_forward's assemble_inputs
// (training.cpp:211-214, attention.cpp:414-451) in ONE kernel for recent-k: a warp searches
// its 32 queries as k_recent_line does, keeps (window start, query time, node, kb) in shared
// memory, then writes the Transformer input rows z [32 * l, d] directly -- lanes across the
// columns, the slot's entry read once (broadcast) from the gather records -- so the int
// index / delta rows never go through HBM.  Δt is the fp64 difference (the reference's
// SequenceBatch::time_delta), the time encoding cos(omega * Δt + phi) is computed in fp64 and
// rounded once to the output type, as k_assemble_inputs does.
template <typename T>
__device__ __forceinline__ double fin_f64(T v) {
  return static_cast<double>(v);
}
template <typename T>
__device__ __forceinline__ T fin_out(double v) {
  return static_cast<T>(v);
}
template <>
__device__ __forceinline__ __nv_bfloat16 fin_out<__nv_bfloat16>(double v) {
  return __double2bfloat16(v);
}

template <typename TabT, typename OutT, bool REC>
__global__ void __launch_bounds__(kThreads, 4) k_recent_inputs(
    const NodeDir* __restrict__ dir, const int64_t* __restrict__ nbr,
    const int64_t* __restrict__ eid, const double* __restrict__ ts,
    const uint4* __restrict__ rec, QueryIn in, int64_t Q, int64_t k, int l, int64_t self_idx,
    const TabT* __restrict__ ntab, int64_t nrows, const TabT* __restrict__ etab, int64_t erows,
    const double* __restrict__ omega, const double* __restrict__ phi, int d_v, int d_e, int d_t,
    int concat, OutT* __restrict__ z, int32_t* __restrict__ vlen, int* __restrict__ bad) {
  // a block per group: one warp searches the group's 32 queries, the block writes the rows
  extern __shared__ double s_wp[];  // omega [d_t] | phi [d_t]
  __shared__ int64_t s_st[32];
  __shared__ double s_t[32];
  __shared__ int64_t s_u[32];
  __shared__ int s_kb[32];
  for (int c = threadIdx.x; c < d_t; c += kThreads) {
    s_wp[c] = omega[c];
    s_wp[d_t + c] = phi[c];
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int d = concat ? d_v + d_e + d_t : d_t;
  const int64_t ngroups = ceil_div(Q, 32);
  // one block per group of 32 queries: warp 0 searches them, all warps write the rows
  for (int64_t g = blockIdx.x; g < ngroups; g += gridDim.x) {
    if (warp == 0) {
      const int64_t q = g * 32 + lane;
      int64_t u = 0, m[1];
      double t = 0.0;
      bool pres[1];
      pres[0] = q < Q && fetch_query(in, q, u, t);
      NodeDir dd[1];
      dd[0] = load_dir(dir, u, pres[0]);
      double tt[1] = {t};
      search_lines<kProbeW, 1>(ts, dd, pres, tt, m);
      int kb = -1;
      if (pres[0]) kb = static_cast<int>(min(min(k, m[0]), static_cast<int64_t>(l - 1)));
      if (q < Q && vlen) vlen[q] = kb + 1;
      s_st[lane] = dd[0].start + m[0] - kb;
      s_t[lane] = t;
      s_u[lane] = u;
      s_kb[lane] = kb;
    }
    __syncthreads();
    const int nq = static_cast<int>(min(static_cast<int64_t>(32), Q - g * 32));
    for (int r = warp; r < nq * l; r += kWarps) {
      const int qi = r / l, j = r - qi * l;
      const int kbq = s_kb[qi];
      OutT* zr = z + (g * 32 + qi) * static_cast<int64_t>(l) * d + static_cast<int64_t>(j) * d;
      if (j > kbq) {  // padding row (and absent queries): zeros, as the reference's Matrix
        for (int c = lane; c < d; c += 32) zr[c] = fin_out<OutT>(0.0);
        continue;
      }
      int64_t ni, ei;
      double dt;
      if (j < kbq) {
        const int64_t p = s_st[qi] + j;
        int64_t nb, ed;
        double tv;
        if (REC) {
          const uint4 e = __ldg(rec + p);
          nb = e.x;
          ed = e.y;
          tv = __hiloint2double(static_cast<int>(e.w), static_cast<int>(e.z));
        } else {
          nb = __ldg(reinterpret_cast<const long long*>(nbr) + p);
          ed = __ldg(reinterpret_cast<const long long*>(eid) + p);
          tv = __ldg(ts + p);
        }
        ni = nb + 1;
        ei = ed + 1;
        dt = s_t[qi] - tv;
      } else {  // the self-loop token (sequence.cpp:79-81)
        ni = s_u[qi] + 1;
        ei = self_idx;
        dt = 0.0;
      }
      if (ni < 0 || ni >= nrows || ei < 0 || ei >= erows) {  // attention.cpp:427-431
        if (lane == 0 && bad) atomicOr(bad, 1);
        continue;
      }
      const TabT* nrow = ntab + ni * d_v;
      const TabT* erow = etab + ei * d_e;
      if (!concat) {
        for (int c = lane; c < d; c += 32)
          zr[c] = fin_out<OutT>(fin_f64(__ldg(nrow + c)) + fin_f64(__ldg(erow + c)) +
                                cos(s_wp[c] * dt + s_wp[d_t + c]));
      } else {
        for (int c = lane; c < d_v; c += 32) zr[c] = fin_out<OutT>(fin_f64(__ldg(nrow + c)));
        for (int c = lane; c < d_e; c += 32) zr[d_v + c] = fin_out<OutT>(fin_f64(__ldg(erow + c)));
        for (int c = lane; c < d_t; c += 32)
          zr[d_v + d_e + c] = fin_out<OutT>(cos(s_wp[c] * dt + s_wp[d_t + c]));
      }
    }
    __syncthreads();
  }
}

template <typename TabT, typename OutT>
void launch_recent_inputs_t(const SampleInputsArgs& a, int* bad, cudaStream_t s) {
  const tgfx_graph* g = a.s.g;
  QueryIn in{a.s.nodes, a.s.times, nullptr, 0, nullptr, 0, g->V, a.s.first_bad, a.s.stream_base};
  const int64_t groups = ceil_div(a.s.q, 32);
  // a block per group for the whole query set (round 2: against a grid capped at 16 blocks
  // per SM, 600 K queries 1.049 -> 0.975 ms on the W shape, 1.679 -> 1.601 ms on GDELT's)
  const int grid = static_cast<int>(std::min<int64_t>(groups, INT32_MAX));
  const size_t smem = sizeof(double) * 2 * static_cast<size_t>(a.in.d_t);
  const int l = static_cast<int>(a.s.l);
  auto* z = static_cast<OutT*>(a.in.z);
  auto* vl = static_cast<int32_t*>(a.s.valid_len);
  if (g->rec)
    k_recent_inputs<TabT, OutT, true><<<grid, kThreads, smem, s>>>(
        g->dir, g->nbr, g->eid, g->ts, g->rec, in, a.s.q, a.s.k, l, a.s.self_edge_index,
        static_cast<const TabT*>(a.in.node_table), a.in.node_rows,
        static_cast<const TabT*>(a.in.edge_table), a.in.edge_rows, a.in.omega, a.in.phi,
        static_cast<int>(a.in.d_v), static_cast<int>(a.in.d_e), static_cast<int>(a.in.d_t),
        a.in.concat, z, vl, bad);
  else
    k_recent_inputs<TabT, OutT, false><<<grid, kThreads, smem, s>>>(
        g->dir, g->nbr, g->eid, g->ts, nullptr, in, a.s.q, a.s.k, l, a.s.self_edge_index,
        static_cast<const TabT*>(a.in.node_table), a.in.node_rows,
        static_cast<const TabT*>(a.in.edge_table), a.in.edge_rows, a.in.omega, a.in.phi,
        static_cast<int>(a.in.d_v), static_cast<int>(a.in.d_e), static_cast<int>(a.in.d_t),
        a.in.concat, z, vl, bad);
  after_launch("k_recent_inputs");
}

template <typename TabT>
void launch_recent_inputs_tab(const SampleInputsArgs& a, int* bad, cudaStream_t s) {
  switch (a.in.z_type) {
    case TGFX_F32: launch_recent_inputs_t<TabT, float>(a, bad, s); break;
    case TGFX_F64: launch_recent_inputs_t<TabT, double>(a, bad, s); break;
    case TGFX_BF16: launch_recent_inputs_t<TabT, __nv_bfloat16>(a, bad, s); break;
    default: throw Error(TGFX_EVALIDATION, "unknown output type");
  }
}

// ------------------------------------------------------------------ uniform-k (Floyd)
// Floyd for any k (k > 256): the chosen offsets live in a per-warp open-addressing hash set
// and list in global scratch (H + P2 u64 words, H = pow2 >= 2k, P2 = pow2 >= k).  Draws are
// resolved 32 at a time: each lane looks its draw up in the set of earlier chunks, the chunk
// itself is resolved in draw order by shuffles, then the chosen offsets are inserted.  The
// list is bitonic-sorted in place, so out[r] is the r-th smallest offset (sampler.cpp:66-80).
__device__ void floyd_big(uint64_t* __restrict__ hs, uint64_t* __restrict__ list, int64_t H,
                          int64_t P2, uint64_t s0, int64_t qm, int kk, int lane) {
  for (int64_t i = lane; i < H; i += 32) hs[i] = 0;
  for (int64_t i = kk + lane; i < P2; i += 32) list[i] = ~0ull;
  __syncwarp();
  const int hbits = 63 - __clzll(static_cast<unsigned long long>(H));
  auto slot = [&](uint64_t key) {
    return static_cast<int64_t>((key * 0x9e3779b97f4a7c15ULL) >> (64 - hbits));
  };
  for (int d0 = 0; d0 < kk; d0 += 32) {
    const int d = d0 + lane;
    const bool live = d < kk;
    const uint64_t top = static_cast<uint64_t>(qm - kk + d);
    const uint64_t j = live ? mulhi64(rng_draw(s0, d), top + 1) : 0;
    bool coll = false;
    if (live) {  // chosen by an earlier chunk?
      for (int64_t h = slot(j + 1);; h = (h + 1) & (H - 1)) {
        const uint64_t v = hs[h];
        if (v == 0) break;
        if (v == j + 1) {
          coll = true;
          break;
        }
      }
    }
    const int nd = min(32, kk - d0);
    for (int r = 0; r < nd; ++r) {  // lane r's choice is final once lanes < r are resolved
      const uint64_t cr = __shfl_sync(kFull, coll ? top : j, r);
      if (lane > r && j == cr) coll = true;
    }
    const uint64_t c = coll ? top : j;
    if (live) {
      list[d] = c;
      for (int64_t h = slot(c + 1);; h = (h + 1) & (H - 1))
        if (atomicCAS(reinterpret_cast<unsigned long long*>(hs + h), 0ull,
                      static_cast<unsigned long long>(c + 1)) == 0ull)
          break;
    }
    __syncwarp();
  }
  for (int64_t w = 2; w <= P2; w <<= 1) {  // bitonic sort, ascending
    for (int64_t jj = w >> 1; jj > 0; jj >>= 1) {
      for (int64_t i = lane; i < P2; i += 32) {
        const int64_t x = i ^ jj;
        if (x > i) {
          const uint64_t a = list[i], b = list[x];
          if (((i & w) == 0) ? (a > b) : (a < b)) {
            list[i] = b;
            list[x] = a;
          }
        }
      }
      __syncwarp();
    }
  }
}

template <int P, bool ASSEMBLE, bool IDX64, bool BIG = false>
__global__ void __launch_bounds__(kThreads) k_random(
    const int64_t* __restrict__ indptr, const NodeDir* __restrict__ dir,
    const int64_t* __restrict__ nbr,
    const int64_t* __restrict__ eid, const double* __restrict__ ts, QueryIn in, int64_t Q,
    int64_t k, int l, int64_t self_idx, uint64_t seed, uint64_t stream_base, int exact,
    Outs o, const uint4* __restrict__ rec, uint64_t* __restrict__ scratch = nullptr,
    int64_t H = 0, int64_t P2 = 0) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t ngroups = ceil_div(Q, 32);
  const int kk = static_cast<int>(k);
  const uint64_t seed_mix = mix64(seed);
  for (int64_t g = static_cast<int64_t>(blockIdx.x) * kWarps + warp; g < ngroups;
       g += static_cast<int64_t>(gridDim.x) * kWarps) {
    const int64_t q = g * 32 + lane;
    int64_t lo = 0, m = 0, u = 0;
    double t = 0.0;
    bool present = false;
    if (q < Q && fetch_query(in, q, u, t)) {
      present = true;
      lo = ldg_i64(indptr + u);
    }
    if (exact) {  // slices not known sorted / NaN-free: std::lower_bound's own bisection
      int64_t lo1[1] = {lo}, n1[1] = {present ? ldg_i64(indptr + u + 1) - lo : 0}, m1[1];
      const double t1[1] = {t};
      search_interleaved<1>(ts, lo1, n1, t1, m1);
      m = m1[0];
    } else {
      NodeDir d[1];
      const bool pres[1] = {present};
      const double t1[1] = {t};
      int64_t m1[1];
      d[0] = load_dir(dir, u, present);
      search_lines<kProbeW, 1>(ts, d, pres, t1, m1);
      m = m1[0];
    }
    const int nq = static_cast<int>(min((int64_t)32, Q - g * 32));
    for (int qi = 0; qi < nq; ++qi) {
      const int64_t qq = g * 32 + qi;
      const bool pr = __shfl_sync(kFull, present, qi);
      const int64_t qlo = __shfl_sync(kFull, lo, qi);
      const int64_t qm = __shfl_sync(kFull, m, qi);
      const int64_t qu = __shfl_sync(kFull, u, qi);
      const double qt = __shfl_sync(kFull, t, qi);
      if (ASSEMBLE) {
        if (!pr) {
          for (int j = lane; j < l; j += 32) write_slot<IDX64>(o, qq * l + j, 0, 0, 0.0);
          if (lane == 0) write_vlen<IDX64>(o, qq, 0);
          continue;
        }
      }
      if (qm <= k) {
        // whole prefix (sampler.cpp:59-63): contiguous
        if (ASSEMBLE) {
          const int kb = static_cast<int>(min(qm, (int64_t)(l - 1)));
          const int64_t start = qlo + qm - kb;
          for (int j = lane; j < l; j += 32) {
            int64_t ni = 0, ei = 0;
            double dt = 0.0;
            if (j < kb) {
              double tv;
              fetch_entry(rec, nbr, eid, ts, start + j, ni, ei, tv);
              ++ni;
              ++ei;
              dt = qt - tv;
            } else if (j == kb) {
              ni = qu + 1;
              ei = self_idx;
            }
            write_slot<IDX64>(o, qq * l + j, ni, ei, dt);
          }
          if (lane == 0) write_vlen<IDX64>(o, qq, kb + 1);
        } else {
          for (int j = lane; j < kk; j += 32) {
            const bool h = j < qm;
            int64_t a = 0, b = 0;
            double c = 0.0;
            if (h) fetch_entry(rec, nbr, eid, ts, qlo + j, a, b, c);
            put_entry(o, qq * k + j, a, b, c);
          }
          if (lane == 0) o.counts[qq] = qm;
        }
        continue;
      }
      // Floyd: for d = 0..k-1, i_d = m-k+d, j_d = next_below(i_d+1); c_d = j_d unless already
      // chosen, then i_d.  Draws are independent of the resolution (one draw per iteration).
      const uint64_t s0 = query_rng(in, seed_mix, stream_base, qq, Q);
      if (BIG) {
        const int64_t wid = static_cast<int64_t>(blockIdx.x) * kWarps + warp;
        uint64_t* hs = scratch + wid * (H + P2);
        uint64_t* list = hs + H;
        floyd_big(hs, list, H, P2, s0, qm, kk, lane);
        if (ASSEMBLE) {
          const int kb = min(kk, l - 1);
          const int drop = kk - kb;  // keep the most recent l-1 (sequence.cpp:70-71)
          for (int j = lane; j < l; j += 32) {
            if (j < kb) {
              int64_t ni, ei;
              double tv;
              fetch_entry(rec, nbr, eid, ts, qlo + static_cast<int64_t>(list[drop + j]), ni, ei, tv);
              write_slot<IDX64>(o, qq * l + j, ni + 1, ei + 1, qt - tv);
            } else if (j == kb) {
              write_slot<IDX64>(o, qq * l + j, qu + 1, self_idx, 0.0);
            } else {
              write_slot<IDX64>(o, qq * l + j, 0, 0, 0.0);
            }
          }
          if (lane == 0) write_vlen<IDX64>(o, qq, kb + 1);
        } else {
          for (int r = lane; r < kk; r += 32) {
            int64_t ni, ei;
            double tv;
            fetch_entry(rec, nbr, eid, ts, qlo + static_cast<int64_t>(list[r]), ni, ei, tv);
            put_entry(o, qq * k + r, ni, ei, tv);
          }
          if (lane == 0) o.counts[qq] = kk;
        }
        __syncwarp();
        continue;
      }
      int64_t jd[P], c[P];
#pragma unroll
      for (int p = 0; p < P; ++p) {
        const int d = p * 32 + lane;
        const uint64_t bound = static_cast<uint64_t>(qm - kk + d) + 1;
        jd[p] = d < kk ? static_cast<int64_t>(mulhi64(rng_draw(s0, d), bound)) : -1;
        c[p] = -1;
      }
#pragma unroll
      for (int p = 0; p < P; ++p) {
        for (int o2 = 0; o2 < 32; ++o2) {
          const int d = p * 32 + o2;
          if (d >= kk) break;
          const int64_t jv = __shfl_sync(kFull, jd[p], o2);
          bool hit = false;
#pragma unroll
          for (int p2 = 0; p2 <= p; ++p2) hit |= (p2 < p || lane < o2) && c[p2] == jv;
          hit = __any_sync(kFull, hit);
          if (lane == o2) c[p] = hit ? (qm - kk + d) : jv;
        }
      }
      // ranks (offsets are distinct)
      int rank[P];
#pragma unroll
      for (int p = 0; p < P; ++p) rank[p] = 0;
#pragma unroll
      for (int p2 = 0; p2 < P; ++p2) {
        for (int o2 = 0; o2 < 32; ++o2) {
          if (p2 * 32 + o2 >= kk) break;
          const int64_t v = __shfl_sync(kFull, c[p2], o2);
#pragma unroll
          for (int p = 0; p < P; ++p) rank[p] += v < c[p];
        }
      }
      if (ASSEMBLE) {
        const int kb = min(kk, l - 1);
        const int drop = kk - kb;  // keep the most recent l-1 (sequence.cpp:70-71)
#pragma unroll
        for (int p = 0; p < P; ++p) {
          const int d = p * 32 + lane;
          if (d < kk && rank[p] >= drop) {
            int64_t ni, ei;
            double tv;
            fetch_entry(rec, nbr, eid, ts, qlo + c[p], ni, ei, tv);
            write_slot<IDX64>(o, qq * l + (rank[p] - drop), ni + 1, ei + 1, qt - tv);
          }
        }
        for (int j = kb + lane; j < l; j += 32) {
          if (j == kb)
            write_slot<IDX64>(o, qq * l + j, qu + 1, self_idx, 0.0);
          else
            write_slot<IDX64>(o, qq * l + j, 0, 0, 0.0);
        }
        if (lane == 0) write_vlen<IDX64>(o, qq, kb + 1);
      } else {
#pragma unroll
        for (int p = 0; p < P; ++p) {
          const int d = p * 32 + lane;
          if (d < kk) {
            int64_t ni, ei;
            double tv;
            fetch_entry(rec, nbr, eid, ts, qlo + c[p], ni, ei, tv);
            put_entry(o, qq * k + rank[p], ni, ei, tv);
          }
        }
        if (lane == 0) o.counts[qq] = kk;
      }
    }
  }
}

// first out-of-range node index (atomicMin of base + i); with fix, a bad node is replaced by 0
// in the (caller-owned, device) copy so the sampler can run on it unchecked
__global__ void k_find_bad(const int64_t* __restrict__ nodes, int64_t q, int64_t V,
                           unsigned long long* first, int64_t base = 0, int64_t* fix = nullptr) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < q;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t u = nodes[i];
    if (u < 0 || u >= V) {
      atomicMin(first, (unsigned long long)(base + i));
      if (fix) fix[i] = 0;
    }
  }
}

// build_sequence_batch over padded samples, reference types (sequence.cpp:55-86)
__global__ void k_assemble_entries(int64_t q, int64_t kpad, const int64_t* __restrict__ counts,
                                   const int64_t* __restrict__ nbr, const int64_t* __restrict__ eid,
                                   const double* __restrict__ ts, const int64_t* __restrict__ qn,
                                   const double* __restrict__ qt, int64_t l, int64_t self_idx,
                                   int64_t* node_index, int64_t* edge_index, double* dt,
                                   int64_t* valid_len, int64_t* target_row, int64_t es) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < q * l;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = i / l, j = i - b * l;
    const int64_t total = counts[b];
    const int64_t kb = min(total, l - 1);
    const int64_t skip = total - kb;
    int64_t ni = 0, ei = 0;
    double d = 0.0;
    if (j < kb) {
      const int64_t s = (b * kpad + skip + j) * es;
      ni = nbr[s] + 1;
      ei = eid[s] + 1;
      d = qt[b] - ts[s];
    } else if (j == kb) {
      ni = qn[b] + 1;
      ei = self_idx;
      valid_len[b] = kb + 1;
      target_row[b] = kb;
    }
    node_index[i] = ni;
    edge_index[i] = ei;
    dt[i] = d;
  }
}

// build_mask (sequence.cpp:93-111): (q*l) x l of {0, -inf}
__global__ void k_mask(int64_t q, int64_t l, const int64_t* __restrict__ valid_len,
                       const int64_t* __restrict__ target_row, int kind, double* mask) {
  const int64_t total = q * l * l;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = i / l, col = i - row * l;
    const int64_t b = row / l, r = row - b * l;
    const int64_t len = valid_len[b], kq = target_row[b];
    int64_t hi = 0;
    if (kind == TGFX_MASK_CAUSAL)
      hi = min(r + 1, len);
    else if (r == kq)
      hi = kind == TGFX_MASK_SELF_LOOP ? kq + 1 : kq;
    mask[i] = col < hi ? 0.0 : __longlong_as_double(0xfff0000000000000LL);  // -inf
  }
}

bool bulk_enabled() {
  static const bool on = [] {
    const char* e = getenv("TGFX_BULK_ROWS");
    return !(e && e[0] == '0');
  }();
  return on;
}

int recent_unr() {
  static const int v = [] {
    const char* e = getenv("TGFX_RECENT_UNR");
    return e ? atoi(e) : 0;
  }();
  return v;
}

// one group of 32 queries per warp, the whole grid at once (round 2: a grid capped at 8 blocks
// per SM with warps striding over groups measured 15 % slower on GDELT uniform-20, 19.0
// against 16.2 ms -- strided warps drift apart and spread the window over the stream)
int grid_groups(int64_t Q) {
  const int64_t groups = ceil_div(std::max<int64_t>(Q, 1), 32);
  const int64_t blocks = ceil_div(groups, kWarps);
  return static_cast<int>(std::min<int64_t>(blocks, INT32_MAX));
}

// ------------------------------------------------------------------ uniform-k, k <= 32
// Default uniform-k kernel for k <= 32 (LastFM-shaped uniform-20).  Phase 1: one query per
// lane, line-probe search through the node directory (as k_recent_line).  Phase 2: Floyd's
// algorithm with the reference's counter RNG (rng.hpp:23-38, sampler.cpp:66-80) run by
// 8-lane groups, four queries per warp at a time: lane r of a group draws d = r, r+8, ...
// (O(1) skip-ahead), the draws are resolved in order d = 0..k-1 with one group-masked ballot
// each, and every chosen offset is ranked against the group's others with width-8 shuffles.
// Resolution is inherently sequential in d; running four queries per warp through it (instead
// of one) is what keeps small batches (12,000 queries) from being latency-bound.
template <int P, bool ASSEMBLE, bool IDX64>
__global__ void __launch_bounds__(kThreads) k_random_g(
    const NodeDir* __restrict__ dir, const int64_t* __restrict__ nbr,
    const int64_t* __restrict__ eid, const double* __restrict__ ts, QueryIn in, int64_t Q,
    int64_t k, int l, int64_t self_idx, uint64_t seed, uint64_t stream_base, Outs o,
    const uint4* __restrict__ rec) {
  constexpr int G = 8;                      // lanes per query
  constexpr int NG = 32 / G;                // queries per warp round
  __shared__ int64_t s_lo[kWarps][32], s_m[kWarps][32], s_u[kWarps][32];
  __shared__ double s_t[kWarps][32];
  __shared__ int s_pres[kWarps][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int grp = lane / G, r = lane % G;
  const unsigned gmask = ((1u << G) - 1u) << (grp * G);
  const int kk = static_cast<int>(k);
  const uint64_t seed_mix = mix64(seed);
  const int64_t ngroups = ceil_div(Q, 32);
  for (int64_t gq = static_cast<int64_t>(blockIdx.x) * kWarps + warp; gq < ngroups;
       gq += static_cast<int64_t>(gridDim.x) * kWarps) {
    {  // phase 1: one query per lane
      const int64_t q = gq * 32 + lane;
      int64_t u[1] = {0}, m[1];
      double t[1] = {0.0};
      bool pres[1];
      pres[0] = q < Q && fetch_query(in, q, u[0], t[0]);
      NodeDir d[1];
      d[0] = load_dir(dir, u[0], pres[0]);
      search_lines<kProbeW, 1>(ts, d, pres, t, m);
      s_lo[warp][lane] = d[0].start;
      s_m[warp][lane] = m[0];
      s_u[warp][lane] = u[0];
      s_t[warp][lane] = t[0];
      s_pres[warp][lane] = pres[0] ? 1 : 0;
    }
    __syncwarp();
    const int nq = static_cast<int>(min((int64_t)32, Q - gq * 32));
    for (int q0 = 0; q0 < nq; q0 += NG) {
      const int qi = q0 + grp;
      const bool live = qi < nq;
      const int64_t qq = gq * 32 + qi;
      const bool pr = live && s_pres[warp][qi];
      const int64_t qlo = live ? s_lo[warp][qi] : 0;
      const int64_t qm = live ? s_m[warp][qi] : 0;
      const int64_t qu = live ? s_u[warp][qi] : 0;
      const double qt = live ? s_t[warp][qi] : 0.0;
      const bool floyd = pr && qm > k;
      // Floyd (all groups run the loop so the shuffles/ballots see every lane)
      const uint64_t s0 = query_rng(in, seed_mix, stream_base, qq, Q);
      int64_t jd[P], c[P];
#pragma unroll
      for (int p = 0; p < P; ++p) {
        const int dd = p * G + r;
        const uint64_t bound = static_cast<uint64_t>(qm - kk + dd) + 1;
        jd[p] = (floyd && dd < kk) ? static_cast<int64_t>(mulhi64(rng_draw(s0, dd), bound)) : -1;
        c[p] = -1;
      }
#pragma unroll
      for (int p = 0; p < P; ++p) {
        for (int o2 = 0; o2 < G; ++o2) {
          const int dd = p * G + o2;
          if (dd >= kk) break;
          const int64_t jv = __shfl_sync(kFull, jd[p], o2, G);
          bool hit = false;
#pragma unroll
          for (int p2 = 0; p2 <= p; ++p2) hit |= (p2 < p || r < o2) && c[p2] == jv;
          hit = (__ballot_sync(kFull, hit) & gmask) != 0;
          if (r == o2) c[p] = hit ? (qm - kk + dd) : jv;
        }
      }
      int rank[P];
#pragma unroll
      for (int p = 0; p < P; ++p) rank[p] = 0;
#pragma unroll
      for (int p2 = 0; p2 < P; ++p2) {
        for (int o2 = 0; o2 < G; ++o2) {
          if (p2 * G + o2 >= kk) break;
          const int64_t v = __shfl_sync(kFull, c[p2], o2, G);
#pragma unroll
          for (int p = 0; p < P; ++p) rank[p] += v < c[p];
        }
      }
      if (!live) continue;
      if (ASSEMBLE) {
        if (!pr) {  // absent hop-2 slot
          for (int j = r; j < l; j += G) write_slot<IDX64>(o, qq * l + j, 0, 0, 0.0);
          if (r == 0) write_vlen<IDX64>(o, qq, 0);
          continue;
        }
        if (!floyd) {  // whole prefix (sampler.cpp:59-63), most recent l-1 kept
          const int kb = static_cast<int>(min(qm, (int64_t)(l - 1)));
          const int64_t start = qlo + qm - kb;
          for (int j = r; j < l; j += G) {
            int64_t ni = 0, ei = 0;
            double dt = 0.0;
            if (j < kb) {
              double tv;
              fetch_entry(rec, nbr, eid, ts, start + j, ni, ei, tv);
              ++ni;
              ++ei;
              dt = qt - tv;
            } else if (j == kb) {
              ni = qu + 1;
              ei = self_idx;
            }
            write_slot<IDX64>(o, qq * l + j, ni, ei, dt);
          }
          if (r == 0) write_vlen<IDX64>(o, qq, kb + 1);
          continue;
        }
        const int kb = min(kk, l - 1);
        const int drop = kk - kb;  // keep the most recent l-1 (sequence.cpp:70-71)
        // all P samples' loads first (an unused one reads the slice's first entry), then
        // predicated stores: the loads are in flight together
        int64_t ni[P], ei[P];
        double tv[P];
        bool use[P];
#pragma unroll
        for (int p = 0; p < P; ++p) {
          const int dd = p * G + r;
          use[p] = dd < kk && rank[p] >= drop;
          fetch_entry_v(rec, nbr, eid, ts, qlo + (use[p] ? c[p] : 0), ni[p], ei[p], tv[p]);
        }
#pragma unroll
        for (int p = 0; p < P; ++p)
          write_slot_if<IDX64>(o, qq * l + (use[p] ? rank[p] - drop : 0), ni[p] + 1, ei[p] + 1,
                               qt - tv[p], use[p]);
        for (int j = kb + r; j < l; j += G)
          write_slot<IDX64>(o, qq * l + j, j == kb ? qu + 1 : 0, j == kb ? self_idx : 0, 0.0);
        if (r == 0) write_vlen<IDX64>(o, qq, kb + 1);
      } else {
        if (!floyd) {
          const int64_t take = pr ? qm : 0;
          for (int j = r; j < kk; j += G) {
            const bool h = j < take;
            int64_t a = 0, b = 0;
            double c = 0.0;
            if (h) fetch_entry(rec, nbr, eid, ts, qlo + j, a, b, c);
            put_entry(o, qq * k + j, a, b, c);
          }
          if (r == 0) o.counts[qq] = take;
          continue;
        }
#pragma unroll
        for (int p = 0; p < P; ++p) {
          const int dd = p * G + r;
          if (dd < kk) {
            int64_t ni, ei;
            double tv;
            fetch_entry(rec, nbr, eid, ts, qlo + c[p], ni, ei, tv);
            put_entry(o, qq * k + rank[p], ni, ei, tv);
          }
        }
        if (r == 0) o.counts[qq] = kk;
      }
    }
    __syncwarp();
  }
}


// Uniform-k, one query per lane (ASSEMBLE, int32/fp32 rows, gather records, k <= KM, l <= 32):
// Floyd's draws (the same skip-ahead CounterRng draws and collision rule as k_random_g) kept
// as 32-bit slice offsets in registers, each sample's rank among them counted in registers
// (O(k^2) integer compares per lane, no shuffles or ballots), then the samples gathered in
// chunks of CH loads issued together and the rows staged in shared memory and written out
// coalesced.  Slice lengths are < 2^32 whenever gather records exist (m < 2^32).
template <int KM, int CH, int MINB>
__global__ void __launch_bounds__(kThreads, MINB) k_random_lane(
    const NodeDir* __restrict__ dir, const double* __restrict__ ts, const uint4* __restrict__ rec,
    QueryIn in, int64_t Q, int k, int l, int64_t self_idx, uint64_t seed, uint64_t stream_base,
    Outs o, const DirC* __restrict__ dirc = nullptr, const uint32_t* __restrict__ bkt = nullptr,
    int rshift = 0) {
  extern __shared__ __align__(16) uint32_t s_rows[];  // per warp [3][32 * l]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t seed_mix = mix64(seed);
  uint32_t* sn = s_rows + static_cast<size_t>(warp) * 3 * 32 * l;
  uint32_t* se = sn + 32 * l;
  float* sd = reinterpret_cast<float*>(se + 32 * l);
  const int64_t ngroups = ceil_div(Q, 32);
  for (int64_t gq = static_cast<int64_t>(blockIdx.x) * kWarps + warp; gq < ngroups;
       gq += static_cast<int64_t>(gridDim.x) * kWarps) {
    const int64_t q = gq * 32 + lane;
    int64_t u[1] = {0}, m[1];
    double t[1] = {0.0};
    bool pres[1];
    pres[0] = q < Q && fetch_query(in, q, u[0], t[0]);
    NodeDir d[1];
    d[0] = (dirc ? load_dirc(dirc, bkt, rshift, u[0], pres[0]) : load_dir(dir, u[0], pres[0]));
    search_lines<kProbeW, 1>(ts, d, pres, t, m);
    const uint32_t qm = static_cast<uint32_t>(m[0]);
    const bool floyd = pres[0] && qm > static_cast<uint32_t>(k);
    const int kb = !pres[0] ? -1 : floyd ? min(k, l - 1) : min(static_cast<int>(qm), l - 1);
    // Floyd (sampler.cpp:66-80): draw d picks j in [0, qm - k + d]; a repeat takes qm - k + d
    uint32_t c[KM];
    const uint64_t s0 = query_rng(in, seed_mix, stream_base, q, Q);
#pragma unroll
    for (int dd = 0; dd < KM; ++dd) {
      c[dd] = 0xffffffffu;
      if (floyd && dd < k) {
        const uint32_t top = qm - static_cast<uint32_t>(k) + static_cast<uint32_t>(dd);
        const uint32_t j = static_cast<uint32_t>(mulhi64(rng_draw(s0, dd), static_cast<uint64_t>(top) + 1));
        bool hit = false;
#pragma unroll
        for (int e = 0; e < dd; ++e) hit |= c[e] == j;
        c[dd] = hit ? top : j;
      }
    }
    // slots: Floyd sample dd goes to column rank(dd) - drop (the most recent l - 1 kept,
    // sequence.cpp:70-71); the whole-prefix case takes the last kb entries in order
    const int drop = floyd ? k - kb : 0;
    const int64_t wbase = floyd ? d[0].start : d[0].start + qm - kb;
    const uint32_t* cu = c;
    // rows are staged per lane at [lane * l + column]
#pragma unroll
    for (int c0 = 0; c0 < KM; c0 += CH) {
      uint32_t rn[CH], re[CH];
      double tv[CH];
      int col[CH];
#pragma unroll
      for (int h = 0; h < CH; ++h) {
        const int dd = c0 + h;
        int cc = -1;
        int64_t p = 0;
        if (floyd) {
          if (dd < k) {
            int rk = 0;
#pragma unroll
            for (int e = 0; e < KM; ++e) rk += cu[e] < cu[dd];
            if (rk >= drop) {
              cc = rk - drop;
              p = wbase + cu[dd];
            }
          }
        } else if (dd < kb) {
          cc = dd;
          p = wbase + dd;
        }
        col[h] = cc;
        uint32_t a, b, x, y;
        asm volatile("ld.global.nc.v4.u32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(a), "=r"(b), "=r"(x), "=r"(y) : "l"(rec + p));
        rn[h] = a;
        re[h] = b;
        tv[h] = __hiloint2double(static_cast<int>(y), static_cast<int>(x));
      }
#pragma unroll
      for (int h = 0; h < CH; ++h) {  // predicated stores: no branch to sink the loads into
        const int sidx = lane * l + max(col[h], 0);
        const int pr = col[h] >= 0;
        asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q st.shared.u32 [%0], %1;\n\t}"
                     ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(sn + sidx))), "r"(rn[h] + 1u), "r"(pr)
                     : "memory");
        asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q st.shared.u32 [%0], %1;\n\t}"
                     ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(se + sidx))), "r"(re[h] + 1u), "r"(pr)
                     : "memory");
        asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q st.shared.f32 [%0], %1;\n\t}"
                     ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(sd + sidx))),
                     "f"(__double2float_rn(t[0] - tv[h])), "r"(pr)
                     : "memory");
      }
    }
    // self-edge token at column kb, zero padding after it; absent queries: an all-zero row
    for (int j = max(kb, 0); j < l; ++j) {
      const bool self = j == kb;
      sn[lane * l + j] = self ? static_cast<uint32_t>(u[0] + 1) : 0u;
      se[lane * l + j] = self ? static_cast<uint32_t>(self_idx) : 0u;
      sd[lane * l + j] = 0.0f;
    }
    if (q < Q) write_vlen<false>(o, q, kb + 1);
    __syncwarp();
    // coalesced copy-out of the warp's [nq x l] block
    const int nq = static_cast<int>(min(static_cast<int64_t>(32), Q - gq * 32));
    const int64_t obase = gq * 32 * l;
    for (int sidx = lane; sidx < nq * l; sidx += 32) {
      __stcs(static_cast<int*>(o.node) + obase + sidx, static_cast<int>(sn[sidx]));
      __stcs(static_cast<int*>(o.edge) + obase + sidx, static_cast<int>(se[sidx]));
      __stcs(o.dt32 + obase + sidx, sd[sidx]);
    }
    __syncwarp();
  }
}

template <bool ASM, bool I64>
void launch_random_g(const SampleArgs& a, const QueryIn& in, const Outs& o, int grid,
                     cudaStream_t s) {
  const tgfx_graph* g = a.g;
  const int l = static_cast<int>(a.l);
#define TGFX_RANDOM_G(PP)                                                                      \
  k_random_g<PP, ASM, I64><<<grid, kThreads, 0, s>>>(g->dir, g->nbr, g->eid, g->ts, in, a.q, a.k, \
                                                     l, a.self_edge_index, a.seed,             \
                                                     a.stream_base, o, g->rec);
  if (a.k <= 8)
    TGFX_RANDOM_G(1)
  else if (a.k <= 16)
    TGFX_RANDOM_G(2)
  else
    TGFX_RANDOM_G(4)
#undef TGFX_RANDOM_G
  after_launch("k_random_g");
}

template <bool ASM, bool I64>
void launch_random_p(int P, const SampleArgs& a, const QueryIn& in, const Outs& o, int grid,
                     cudaStream_t s) {
  const tgfx_graph* g = a.g;
  const int l = static_cast<int>(a.l);
#define TGFX_RANDOM_CASE(PP)                                                                 \
  case PP:                                                                                   \
    k_random<PP, ASM, I64><<<grid, kThreads, 0, s>>>(g->indptr, g->dir, g->nbr, g->eid, g->ts, in, a.q, \
                                                     a.k, l, a.self_edge_index, a.seed,      \
                                                     a.stream_base, g->search_exact, o,     \
                                                     g->rec);                               \
    break;
  switch (P) {
    TGFX_RANDOM_CASE(1)
    TGFX_RANDOM_CASE(2)
    TGFX_RANDOM_CASE(4)
    TGFX_RANDOM_CASE(8)
    default: {
      // k > 256 (the reference has no limit, sampler.cpp:54-82): hash-set Floyd with per-warp
      // global scratch; the grid is capped so the scratch stays within ~1 GB
      if (a.k >= (int64_t(1) << 30)) throw Error(TGFX_EUNSUPPORTED, "k too large");
      int64_t H = 1, P2 = 1;
      while (H < 2 * a.k) H <<= 1;
      while (P2 < a.k) P2 <<= 1;
      const int64_t per_warp = (H + P2) * 8;
      const int64_t max_warps = std::max<int64_t>(kWarps, (int64_t(1) << 30) / per_warp);
      const int gb = static_cast<int>(std::max<int64_t>(
          1, std::min<int64_t>(grid, max_warps / kWarps)));
      uint64_t* scratch = static_cast<uint64_t*>(
          dmalloc(static_cast<size_t>(per_warp) * gb * kWarps, s));
      k_random<1, ASM, I64, true><<<gb, kThreads, 0, s>>>(
          g->indptr, g->dir, g->nbr, g->eid, g->ts, in, a.q, a.k, l, a.self_edge_index, a.seed,
          a.stream_base, g->search_exact, o, g->rec, scratch, H, P2);
      try {
        after_launch("k_random");
      } catch (...) {
        dfree(scratch, s);
        throw;
      }
      dfree(scratch, s);
      return;
    }
  }
#undef TGFX_RANDOM_CASE
  after_launch("k_random");
}

}  // namespace

void find_bad_async(const tgfx_graph* g, int64_t* d_nodes, int64_t q, int64_t base,
                    unsigned long long* d_first, cudaStream_t s) {
  if (q <= 0) return;
  const int grid = static_cast<int>(std::min<int64_t>(ceil_div(q, 256), device_info().sms * 8));
  k_find_bad<<<grid, 256, 0, s>>>(d_nodes, q, g->V, d_first, base, d_nodes);
  after_launch("k_find_bad");
}

int64_t find_bad_query(const tgfx_graph* g, const int64_t* d_nodes, int64_t q, cudaStream_t s) {
  if (q <= 0) return -1;
  unsigned long long* first = static_cast<unsigned long long*>(dmalloc(8, s));
  const unsigned long long init = ~0ull;
  TGFX_CUDA(cudaMemcpyAsync(first, &init, 8, cudaMemcpyHostToDevice, s));
  const int grid = static_cast<int>(std::min<int64_t>(ceil_div(q, 256), device_info().sms * 8));
  k_find_bad<<<grid, 256, 0, s>>>(d_nodes, q, g->V, first);
  after_launch("k_find_bad");
  unsigned long long h = 0;
  TGFX_CUDA(cudaMemcpyAsync(&h, first, 8, cudaMemcpyDeviceToHost, s));
  TGFX_CUDA(cudaStreamSynchronize(s));
  dfree(first, s);
  return h == ~0ull ? -1 : static_cast<int64_t>(h);
}

// fused recent-k sampler + assemble_inputs when the graph takes the line-probe search;
// returns false when the caller must compose sample + assemble_inputs instead
bool launch_sample_inputs(const SampleInputsArgs& a, int* bad, cudaStream_t s) {
  const tgfx_graph* g = a.s.g;
  if (a.s.strategy != TGFX_RECENT || g->search_exact || g->indptr_bad) return false;
  if (a.s.q <= 0) return true;
  switch (a.in.table_type) {
    case TGFX_F32: launch_recent_inputs_tab<float>(a, bad, s); break;
    case TGFX_F64: launch_recent_inputs_tab<double>(a, bad, s); break;
    default: throw Error(TGFX_EVALIDATION, "tables must be f32 or f64");
  }
  return true;
}

// compact directory records for the bulk recent-k kernel (TGFX_DIRC, default 1)
bool dirc_enabled() {
  static const bool on = [] {
    const char* e = getenv("TGFX_DIRC");
    return !(e && e[0] == '0');
  }();
  return on;
}

// the graph's compact directory when the samplers may use it (slice lengths fit u32, bucket
// size a power of two), else nullptr; *rshift = log2 of the bucket size
const DirC* compact_dir(const tgfx_graph* g, int* rshift) {
  const int64_t R = g->bkt_r;
  int sh = 0;
  while (R > 0 && (int64_t(1) << sh) < R) ++sh;
  *rshift = sh;
  const bool ok = g->dirc && g->m < (int64_t(1) << 32) && (R == 0 || (int64_t(1) << sh) == R) &&
                  dirc_enabled();
  return ok ? g->dirc : nullptr;
}

void launch_sample(const SampleArgs& a, cudaStream_t s) {
  if (a.g->indptr_bad)  // an imported T-CSR whose indptr no slice walk can trust
    throw Error(TGFX_EVALIDATION, "indptr not monotone");
  if (a.q <= 0) return;
  const tgfx_graph* g = a.g;
  QueryIn in{a.nodes, a.times, a.hop_counts, a.hop_k1, a.seeds, a.batch_q,
             g->V,    a.first_bad, a.stream_base};
  Outs o{a.node_index, a.edge_index, a.dt32, a.dt64,  a.valid_len,
         a.counts,     a.e_nbr,      a.e_eid, a.e_ts, a.e_stride};
  const int grid = grid_groups(a.q);
  if (ceil_div(a.q, 32) > static_cast<int64_t>(grid) * kWarps)  // > 5.5e11 queries per call
    throw Error(TGFX_EUNSUPPORTED, "too many queries for one launch");
  const bool assemble = a.l > 0;
  const int l = static_cast<int>(a.l);
  if (a.strategy == TGFX_RECENT) {
    const int width = assemble ? l : static_cast<int>(a.k);
    const uint32_t magic =
        (width < 512) ? static_cast<uint32_t>(((1ull << 32) + width - 1) / width) : 0u;
    // a group per warp (a persistent grid of 4 or 8 blocks per SM measured 22 % slower)
    const int gq = static_cast<int>(
        std::min<int64_t>(ceil_div(ceil_div(a.q, 32), kWarps), INT32_MAX));
    if (ceil_div(a.q, 32) > static_cast<int64_t>(gq) * kWarps)  // > 5.5e11 queries in one call
      throw Error(TGFX_EUNSUPPORTED, "too many queries for one launch");
    const bool bulk = assemble && !a.index64 && a.dt32 && !a.dt64 && l <= kBulkMaxL &&
                      ((reinterpret_cast<uintptr_t>(a.node_index) |
                        reinterpret_cast<uintptr_t>(a.edge_index) |
                        reinterpret_cast<uintptr_t>(a.dt32)) & 15) == 0 &&
                      bulk_enabled();
    if (!g->search_exact && bulk) {  // line probes + bulk-copied rows (default for l <= 16)
      // compact directory records: slice lengths fit u32 and the bucket size is a power of 2
      int rshift = 0;
      const bool dc = compact_dir(g, &rshift) != nullptr;
      if (g->rec) {
#define TGFX_BULK_LAUNCH(REC, U, DCV)                                                          \
  do {                                                                                         \
    const auto kern = k_recent_line<true, false, kProbeW, 1, 4, true, REC, U, DCV>;            \
    static const bool attr = [&] {                                                             \
      TGFX_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,        \
                                     kWarps * 3 * 32 * ((kBulkMaxL + U - 1) / U * U) * 4));    \
      return true;                                                                             \
    }();                                                                                       \
    (void)attr;                                                                                \
    const size_t smu = static_cast<size_t>(kWarps) * 3 * 32 * ((l + U - 1) / U * U) * 4;       \
    kern<<<gq, kThreads, smu, s>>>(g->dir, g->nbr, g->eid, g->ts, in, a.q, a.k, l,             \
                                   a.self_edge_index, magic, o, g->rec, g->dirc, g->bkt,       \
                                   rshift);                                                    \
  } while (0)
        // slots per lane per load round: 2 with the 64-byte directory (round 1: 35.8 ms/step
        // against 37.6 for 4, 38.2 for 1); with the compact directory and no loop-carried
        // spill (round 2, GDELT step launch, l = 11): 3 / 4 / 5 / 6 / 12 -> 1.277 / 1.254 /
        // 1.617 / 1.235 / 1.405 ms -- 6 while it pads l to at most 12 slots, else 4
        // (TGFX_RECENT_UNR overrides)
        const int unr = recent_unr() ? recent_unr() : (l <= 12 ? 6 : 4);
        if (dc && unr == 2)
          TGFX_BULK_LAUNCH(true, 2, true);
        else if (dc && unr == 3)
          TGFX_BULK_LAUNCH(true, 3, true);
        else if (dc && unr == 6)
          TGFX_BULK_LAUNCH(true, 6, true);
        else if (dc)
          TGFX_BULK_LAUNCH(true, 4, true);
        else
          TGFX_BULK_LAUNCH(true, 2, false);
        after_launch("k_recent_line");
        return;
      }
      TGFX_BULK_LAUNCH(false, 2, false);
#undef TGFX_BULK_LAUNCH
      after_launch("k_recent_line");
      return;
    }
    if (!g->search_exact) {  // line probes through the node directory
      if (assemble && a.index64)
        k_recent_line<true, true, kProbeW, 1, 4><<<gq, kThreads, 0, s>>>(
            g->dir, g->nbr, g->eid, g->ts, in, a.q, a.k, l, a.self_edge_index, magic, o, g->rec);
      else if (assemble)
        k_recent_line<true, false, kProbeW, 1, 4><<<gq, kThreads, 0, s>>>(
            g->dir, g->nbr, g->eid, g->ts, in, a.q, a.k, l, a.self_edge_index, magic, o, g->rec);
      else
        k_recent_line<false, false, kProbeW, 1, 4><<<gq, kThreads, 0, s>>>(
            g->dir, g->nbr, g->eid, g->ts, in, a.q, a.k, 0, 0, magic, o, g->rec);
      after_launch("k_recent_line");
      return;
    }
    // slices not known sorted / NaN-free: std::lower_bound's exact bisection, 4 per lane
    const int gb = static_cast<int>(
        std::min<int64_t>(ceil_div(ceil_div(a.q, 32 * 4), kWarps), INT32_MAX));
    if (assemble && a.index64)
      k_recent<true, true, 4, 3><<<gb, kThreads, 0, s>>>(g->indptr, g->nbr, g->eid, g->ts, in,
                                                          a.q, a.k, l, a.self_edge_index, magic, o,
                                                          g->rec);
    else if (assemble)
      k_recent<true, false, 4, 3><<<gb, kThreads, 0, s>>>(g->indptr, g->nbr, g->eid, g->ts, in,
                                                           a.q, a.k, l, a.self_edge_index, magic, o,
                                                           g->rec);
    else
      k_recent<false, false, 4, 3><<<gb, kThreads, 0, s>>>(g->indptr, g->nbr, g->eid, g->ts, in,
                                                            a.q, a.k, 0, 0, magic, o, g->rec);
    after_launch("k_recent");
    return;
  }
  static const bool lane_uniform = [] {
    const char* e = getenv("TGFX_UNIFORM_LANE");
    return !(e && e[0] == '0');
  }();
  if (lane_uniform && !g->search_exact && g->rec && assemble && !a.index64 && a.dt32 &&
      !a.dt64 && a.k <= 32 && l <= 32) {  // one query per lane (default for k <= 32, l <= 32)
    const size_t sm = static_cast<size_t>(kWarps) * 3 * 32 * l * 4;
    int cshift = 0;
    const DirC* cdir = compact_dir(g, &cshift);
#define TGFX_RANDOM_LANE(KM) TGFX_RANDOM_LANE_C(KM, 4, (KM > 16 ? 2 : 3))
#define TGFX_RANDOM_LANE_C(KM, CH, MB)                                                         \
  do {                                                                                         \
    static const bool attr = [] {                                                              \
      TGFX_CUDA(cudaFuncSetAttribute(k_random_lane<KM, CH, MB>,                                \
                                     cudaFuncAttributeMaxDynamicSharedMemorySize,              \
                                     kWarps * 3 * 32 * 32 * 4));                               \
      return true;                                                                             \
    }();                                                                                       \
    (void)attr;                                                                                \
    k_random_lane<KM, CH, MB><<<grid, kThreads, sm, s>>>(g->dir, g->ts, g->rec, in, a.q,        \
                                                    static_cast<int>(a.k), l, a.self_edge_index, \
                                                    a.seed, a.stream_base, o, cdir, g->bkt,      \
                                                    cshift);                                     \
  } while (0)
    if (a.k <= 8)
      TGFX_RANDOM_LANE(8);
    else if (a.k <= 16)
      TGFX_RANDOM_LANE(16);
    else if (a.k <= 24)  // loads in chunks of 8 (round 2, one 48 M-query GDELT uniform-20
      TGFX_RANDOM_LANE_C(24, 8, 2);  // launch: chunks of 2 / 4 / 8 / 12 / 24 -> 19.5 / 19.2-19.5 /
                                     // 18.6-18.8 / 20.1 / 23.6 ms; LastFM 0.85 -> 0.83 ms)
    else
      TGFX_RANDOM_LANE(32);
#undef TGFX_RANDOM_LANE
#undef TGFX_RANDOM_LANE_C
    after_launch("k_random_lane");
    return;
  }
  if (!g->search_exact && a.k <= 32) {  // grouped Floyd (k <= 32)
    if (assemble) {
      if (a.index64)
        launch_random_g<true, true>(a, in, o, grid, s);
      else
        launch_random_g<true, false>(a, in, o, grid, s);
    } else {
      launch_random_g<false, false>(a, in, o, grid, s);
    }
    return;
  }
  const int P = a.k <= 32 ? 1 : a.k <= 64 ? 2 : a.k <= 128 ? 4 : a.k <= 256 ? 8 : 0;
  if (assemble) {
    if (a.index64)
      launch_random_p<true, true>(P, a, in, o, grid, s);
    else
      launch_random_p<true, false>(P, a, in, o, grid, s);
  } else {
    launch_random_p<false, false>(P, a, in, o, grid, s);
  }
}

void launch_two_hop(const tgfx_graph* g, const int64_t* roots, const double* times, int64_t q,
                    int64_t k1, int64_t k2, int strategy, uint64_t seed, uint64_t seed2,
                    int64_t l, int64_t self_edge_index, int32_t* h1n, int32_t* h1e, float* h1d,
                    int32_t* h1l, int32_t* h2n, int32_t* h2e, float* h2d, int32_t* h2l,
                    cudaStream_t s) {
  if (g->indptr_bad) throw Error(TGFX_EVALIDATION, "indptr not monotone");
  if (q <= 0) return;
  // hop-1 rows
  SampleArgs a{};
  a.g = g;
  a.nodes = roots;
  a.times = times;
  a.q = q;
  a.k = k1;
  a.strategy = strategy;
  a.seed = seed;
  a.stream_base = 0;
  a.l = l;
  a.self_edge_index = self_edge_index;
  a.node_index = h1n;
  a.edge_index = h1e;
  a.dt32 = h1d;
  a.valid_len = h1l;
  launch_sample(a, s);
  // hop-1 entries (the hop-2 queries), padded [q, k1]
  int64_t* cnt = static_cast<int64_t*>(dmalloc(sizeof(int64_t) * q, s));
  int64_t* en = static_cast<int64_t*>(dmalloc(sizeof(int64_t) * q * k1, s));
  int64_t* ee = static_cast<int64_t*>(dmalloc(sizeof(int64_t) * q * k1, s));
  double* et = static_cast<double*>(dmalloc(sizeof(double) * q * k1, s));
  SampleArgs b = a;
  b.l = 0;
  b.node_index = b.edge_index = b.valid_len = nullptr;
  b.dt32 = nullptr;
  b.counts = cnt;
  b.e_nbr = en;
  b.e_eid = ee;
  b.e_ts = et;
  launch_sample(b, s);
  // hop-2 rows over the q*k1 virtual queries; absent slots -> zero rows, valid_len 0
  SampleArgs c = a;
  c.nodes = en;
  c.times = et;
  c.q = q * k1;
  c.k = k2;
  c.seed = seed2;
  c.stream_base = 0;  // stream = r*k1 + j
  c.node_index = h2n;
  c.edge_index = h2e;
  c.dt32 = h2d;
  c.valid_len = h2l;
  c.hop_counts = cnt;
  c.hop_k1 = k1;
  launch_sample(c, s);
  dfree(cnt, s);
  dfree(en, s);
  dfree(ee, s);
  dfree(et, s);
}

void launch_assemble_entries(int64_t q, int64_t kpad, const int64_t* counts, const int64_t* nbr,
                             const int64_t* eid, const double* ts, const int64_t* qn,
                             const double* qt, int64_t l, int64_t self_edge_index,
                             int64_t* node_index, int64_t* edge_index, double* dt,
                             int64_t* valid_len, int64_t* target_row, cudaStream_t s,
                             int64_t es) {
  if (q <= 0) return;
  const int grid = static_cast<int>(std::min<int64_t>(ceil_div(q * l, 256), device_info().sms * 8));
  k_assemble_entries<<<grid, 256, 0, s>>>(q, kpad, counts, nbr, eid, ts, qn, qt, l,
                                          self_edge_index, node_index, edge_index, dt, valid_len,
                                          target_row, es);
  after_launch("k_assemble_entries");
}

void launch_mask(int64_t q, int64_t l, const int64_t* valid_len, const int64_t* target_row,
                 int kind, double* mask, cudaStream_t s) {
  if (q <= 0) return;
  const int grid =
      static_cast<int>(std::min<int64_t>(ceil_div(q * l * l, 256), device_info().sms * 8));
  k_mask<<<grid, 256, 0, s>>>(q, l, valid_len, target_row, kind, mask);
  after_launch("k_mask");
}

}  // namespace tgfx
