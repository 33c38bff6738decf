// ingest.cu -- load_csv on the device (the step before the build).
//
// Replaces tgf::load_csv (proj/src/event_stream.cpp:85-154): "src,dst,timestamp[,f1..]" rows
// (header required) -> events stable-sorted by timestamp with edge ids 0..n-1 in sorted order,
// num_nodes = max id + 1, optional edge features in the same order.
//
//   1. k_nl_count / k_nl_write   newline positions (per-4 KB-tile counts, scan, ordered write)
//   2. k_parse_lines              one thread per line: trim, split on ',', parse with
//                                 std::from_chars semantics (event_stream.cpp:38-59), the
//                                 reference's per-line checks in its order; the first failing
//                                 line (file order) wins, as the reference throws at it
//   3. compaction of non-empty lines (scan), stable radix sort by timestamp (stable_sort,
//      event_stream.cpp:134), k_emit: events + features in sorted order.
//
// Numbers: integers exactly as from_chars<int64_t> (sign, digits, overflow = bad); reals
// correctly rounded as from_chars<double>: Clinger's fast path, else Eisel-Lemire over the
// first 19 significant digits (decimal_to_double; table from tools/gen_pow5_table.py),
// ERANGE (a nonzero literal rounding to 0 or inf) = bad, inf / nan spellings.  Only a literal
// with more than 19 significant digits whose rounding the 19-digit prefix cannot decide would
// need big-integer arithmetic; it is reported TGFX_EUNSUPPORTED, never parsed approximately --
// as is a NaN timestamp, which the reference's stable_sort orders unpredictably.
#include <algorithm>

#include "graph.cuh"
#include "pow5_table.cuh"
#include "primitives.cuh"

namespace tgfx {
namespace {

constexpr int kNT = 256;
constexpr int kTileBytes = kNT * 16;

// ---------------------------------------------------------------- newline positions
__global__ void k_nl_count(const char* __restrict__ buf, int64_t nbytes, uint32_t* __restrict__ cnt) {
  __shared__ uint32_t red[kNT / 32];
  const int64_t base = static_cast<int64_t>(blockIdx.x) * kTileBytes + threadIdx.x * 16;
  uint32_t c = 0;
  for (int i = 0; i < 16; ++i) c += (base + i < nbytes && buf[base + i] == '\n');
  for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(kFull, c, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t t = 0;
    for (int w = 0; w < kNT / 32; ++w) t += red[w];
    cnt[blockIdx.x] = t;
  }
}

__global__ void k_nl_write(const char* __restrict__ buf, int64_t nbytes,
                           const int64_t* __restrict__ off, int64_t* __restrict__ pos) {
  __shared__ uint32_t wsum[kNT / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t base = static_cast<int64_t>(blockIdx.x) * kTileBytes + threadIdx.x * 16;
  uint32_t c = 0;
  for (int i = 0; i < 16; ++i) c += (base + i < nbytes && buf[base + i] == '\n');
  uint32_t x = c;  // inclusive scan in thread order
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(kFull, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wsum[warp] = x;
  __syncthreads();
  uint32_t before = 0;
  for (int w = 0; w < warp; ++w) before += wsum[w];
  int64_t o = off[blockIdx.x] + before + x - c;
  for (int i = 0; i < 16; ++i)
    if (base + i < nbytes && buf[base + i] == '\n') pos[o++] = base + i;
}

// ---------------------------------------------------------------- number parsing
__device__ __forceinline__ bool is_space(char c) { return c == ' ' || c == '\t' || c == '\r'; }

__device__ __forceinline__ void trim(const char*& p, const char*& e) {
  while (p < e && is_space(*p)) ++p;
  while (e > p && is_space(e[-1])) --e;
}

// std::from_chars<int64_t> on the whole (trimmed) field: 0 ok, 1 bad
__device__ int parse_i64(const char* p, const char* e, int64_t& out) {
  bool neg = false;
  if (p < e && *p == '-') {
    neg = true;
    ++p;
  }
  if (p == e) return 1;
  uint64_t v = 0;
  for (; p < e; ++p) {
    const int d = *p - '0';
    if (d < 0 || d > 9) return 1;
    if (v > (~0ull - d) / 10) return 1;  // overflow: from_chars result_out_of_range
    v = v * 10 + d;
  }
  if (!neg && v > 0x7fffffffffffffffull) return 1;
  if (neg && v > 0x8000000000000000ull) return 1;
  out = neg ? static_cast<int64_t>(0ull - v) : static_cast<int64_t>(v);
  return 0;
}

__device__ __forceinline__ char lower(char c) { return (c >= 'A' && c <= 'Z') ? c + 32 : c; }

__device__ bool match_ci(const char*& p, const char* e, const char* word) {
  const char* q = p;
  for (; *word; ++word, ++q)
    if (q >= e || lower(*q) != *word) return false;
  p = q;
  return true;
}

// w * 10^q rounded to nearest-even (w != 0): Clinger's exact fast path when w <= 2^53 and the
// power of ten is exact, else Eisel-Lemire with the 128-bit power-of-five table, which is
// exact for any 64-bit w (Mushtak & Lemire 2023).  Returns 0 / inf on underflow / overflow.
__device__ double decimal_to_double(uint64_t w, int q) {
  const double p10[23] = {1e0,  1e1,  1e2,  1e3,  1e4,  1e5,  1e6,  1e7,  1e8,  1e9,  1e10, 1e11,
                          1e12, 1e13, 1e14, 1e15, 1e16, 1e17, 1e18, 1e19, 1e20, 1e21, 1e22};
  if (w <= (1ull << 53) && q >= -22 && q <= 22)
    return q >= 0 ? static_cast<double>(w) * p10[q] : static_cast<double>(w) / p10[-q];
  if (q < kPow5Min) return 0.0;
  if (q > kPow5Max) return __longlong_as_double(0x7ff0000000000000ll);
  const int lz = __clzll(static_cast<long long>(w));
  w <<= lz;
  const uint64_t t_hi = kPow5[q - kPow5Min][0], t_lo = kPow5[q - kPow5Min][1];
  uint64_t hi = __umul64hi(w, t_hi), lo = w * t_hi;
  constexpr uint64_t kMask = ~0ull >> 55;  // 52 + 3 bits of precision needed
  if ((hi & kMask) == kMask) {
    const uint64_t s_hi = __umul64hi(w, t_lo);
    lo += s_hi;
    if (lo < s_hi) ++hi;
  }
  const int upper = static_cast<int>(hi >> 63);
  uint64_t mant = hi >> (upper + 64 - 52 - 3);
  int p2 = static_cast<int>(((152170 + 65536) * static_cast<int64_t>(q)) >> 16) + 63 + upper - lz + 1023;
  if (p2 <= 0) {  // subnormal
    if (-p2 + 1 >= 64) return 0.0;
    mant >>= -p2 + 1;
    mant += mant & 1;
    mant >>= 1;
    p2 = mant < (1ull << 52) ? 0 : 1;
    return __longlong_as_double(static_cast<long long>((static_cast<uint64_t>(p2) << 52) | mant));
  }
  // exactly between two doubles: round to even instead of up
  if (lo <= 1 && q >= -4 && q <= 23 && (mant & 3) == 1 && (mant << (upper + 64 - 52 - 3)) == hi)
    mant &= ~1ull;
  mant += mant & 1;
  mant >>= 1;
  if (mant >= (2ull << 52)) {
    mant = 1ull << 52;
    ++p2;
  }
  mant &= ~(1ull << 52);
  if (p2 >= 0x7ff) return __longlong_as_double(0x7ff0000000000000ll);
  return __longlong_as_double(static_cast<long long>((static_cast<uint64_t>(p2) << 52) | mant));
}

// std::from_chars<double> (chars_format::general) on the whole field: 0 ok, 1 bad,
// 2 outside the exactly-parsed class (see the file comment)
__device__ int parse_f64(const char* p, const char* e, double& out) {
  bool neg = false;
  if (p < e && *p == '-') {
    neg = true;
    ++p;
  }
  if (p == e) return 1;
  if (lower(*p) == 'i' || lower(*p) == 'n') {
    if (match_ci(p, e, "inf")) {
      match_ci(p, e, "inity");
      if (p != e) return 1;
      out = neg ? -__longlong_as_double(0x7ff0000000000000ll) : __longlong_as_double(0x7ff0000000000000ll);
      return 0;
    }
    if (match_ci(p, e, "nan")) {
      if (p < e && *p == '(') {  // nan(n-char-sequence)
        ++p;
        while (p < e && ((*p >= '0' && *p <= '9') || (lower(*p) >= 'a' && lower(*p) <= 'z') || *p == '_'))
          ++p;
        if (p >= e || *p != ')') return 1;
        ++p;
      }
      if (p != e) return 1;
      out = __longlong_as_double(neg ? 0xfff8000000000000ll : 0x7ff8000000000000ll);
      return 0;
    }
    return 1;
  }
  uint64_t w = 0;
  int nd = 0, q = 0;
  bool any = false, trunc = false;
  for (; p < e && *p >= '0' && *p <= '9'; ++p) {
    any = true;
    const int d = *p - '0';
    if (nd == 0 && d == 0) continue;  // leading zeros
    if (nd < 19) {
      w = w * 10 + d;
      ++nd;
    } else {
      ++q;
      trunc |= d != 0;
    }
  }
  if (p < e && *p == '.') {
    ++p;
    for (; p < e && *p >= '0' && *p <= '9'; ++p) {
      any = true;
      const int d = *p - '0';
      if (nd == 0 && d == 0) {
        --q;
        continue;
      }
      if (nd < 19) {
        w = w * 10 + d;
        ++nd;
        --q;
      } else {
        trunc |= d != 0;
      }
    }
  }
  if (!any) return 1;
  if (p < e && (*p == 'e' || *p == 'E')) {
    const char* r = p + 1;
    bool eneg = false;
    if (r < e && (*r == '+' || *r == '-')) eneg = *r++ == '-';
    if (r < e && *r >= '0' && *r <= '9') {  // else the exponent is not consumed (from_chars)
      int x = 0;
      for (; r < e && *r >= '0' && *r <= '9'; ++r) x = min(x * 10 + (*r - '0'), 100000);
      q += eneg ? -x : x;
      p = r;
    }
  }
  if (p != e) return 1;
  if (w == 0) {  // literal zero (any exponent)
    out = neg ? -0.0 : 0.0;
    return 0;
  }
  double r = 0.0;
  if (!trunc) {
    r = decimal_to_double(w, q);
  } else {  // > 19 significant digits: the value lies in (w, w + 1) x 10^q
    r = decimal_to_double(w, q);
    if (decimal_to_double(w + 1, q) != r) return 2;  // would need big-integer comparison
  }
  // from_chars reports result_out_of_range when a nonzero literal rounds to 0 or to inf
  if (r == 0.0 || r == __longlong_as_double(0x7ff0000000000000ll)) return 1;
  out = neg ? -r : r;
  return 0;
}

// error word: (line_no << 8) | code, codes (CsvError, graph.cuh) in the reference's check
// order for a line (event_stream.cpp:111-131)
constexpr int kErrFields = kCsvFields, kErrSrc = kCsvSrc, kErrDst = kCsvDst, kErrTime = kCsvTime,
              kErrNegNode = kCsvNegNode, kErrNegTime = kCsvNegTime, kErrFeature = kCsvFeature,
              kErrUnsupported = kCsvUnsupported;

__global__ void k_parse_lines(const char* __restrict__ buf, int64_t nbytes, const int64_t* __restrict__ nl,
                              int64_t nnl, int64_t L, int d_e, int64_t* __restrict__ src,
                              int64_t* __restrict__ dst, double* __restrict__ t,
                              uint32_t* __restrict__ keep, double* __restrict__ feats,
                              unsigned long long* __restrict__ err) {
  for (int64_t i = 1 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < L;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = nl[i - 1] + 1;
    const int64_t en = i < nnl ? nl[i] : nbytes;
    const char* p = buf + b;
    const char* e = buf + en;
    trim(p, e);
    keep[i] = 0;
    if (p == e) continue;  // empty line (event_stream.cpp:109)
    const unsigned long long line_no = static_cast<unsigned long long>(i + 1);
    // split on ',': field f spans [fs[f], fe[f]) -- parsed on the fly
    int nf = 1;
    for (const char* c = p; c < e; ++c) nf += (*c == ',');
    int code = 0;
    if (nf < 3 + d_e) code = kErrFields;
    int64_t s = 0, d = 0;
    double tv = 0.0;
    const char* f0 = p;
    auto next_field = [&](const char*& fs, const char*& fe) {
      fs = f0;
      fe = f0;
      while (fe < e && *fe != ',') ++fe;
      f0 = fe < e ? fe + 1 : e;
      trim(fs, fe);
    };
    const char *fs, *fe;
    if (!code) {
      next_field(fs, fe);
      if (parse_i64(fs, fe, s)) code = kErrSrc;
    }
    if (!code) {
      next_field(fs, fe);
      if (parse_i64(fs, fe, d)) code = kErrDst;
    }
    if (!code) {
      next_field(fs, fe);
      const int r = parse_f64(fs, fe, tv);
      if (r == 1) code = kErrTime;
      if (r == 2 || (r == 0 && tv != tv)) code = kErrUnsupported;
    }
    if (!code && (s < 0 || d < 0)) code = kErrNegNode;
    if (!code && tv < 0.0) code = kErrNegTime;
    for (int f = 0; f < d_e && !code; ++f) {
      next_field(fs, fe);
      double fv = 0.0;
      const int r = parse_f64(fs, fe, fv);
      if (r == 1) code = kErrFeature;
      if (r == 2) code = kErrUnsupported;
      feats[i * d_e + f] = fv;
    }
    if (code) {
      atomicMin(err, (line_no << 8) | static_cast<unsigned long long>(code));
      continue;
    }
    src[i] = s;
    dst[i] = d;
    t[i] = tv;
    keep[i] = 1;
  }
}

// row r = the r-th kept line: gather into row arrays and the sort keys
__global__ void k_rows(const uint32_t* __restrict__ keep, const int64_t* __restrict__ rank,
                       int64_t L, const double* __restrict__ t, uint64_t* __restrict__ key,
                       uint32_t* __restrict__ val, int64_t* __restrict__ row_line) {
  for (int64_t i = 1 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < L;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (!keep[i]) continue;
    const int64_t r = rank[i];
    const uint64_t bits = static_cast<uint64_t>(__double_as_longlong(t[i] == 0.0 ? 0.0 : t[i]));
    key[r] = bits | 0x8000000000000000ull;  // t >= 0 (checked): order of the raw bits
    val[r] = static_cast<uint32_t>(r);
    row_line[r] = i;
  }
}

__global__ void k_emit(const uint32_t* __restrict__ perm, const int64_t* __restrict__ row_line,
                       int64_t n, const int64_t* __restrict__ src, const int64_t* __restrict__ dst,
                       const double* __restrict__ t, tgfx_event* __restrict__ ev,
                       unsigned long long* __restrict__ max_node) {
  long long mx = -1;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = row_line[perm[k]];
    tgfx_event x;
    x.edge_id = k;
    x.src = src[i];
    x.dst = dst[i];
    x.timestamp = t[i];
    ev[k] = x;
    mx = max(mx, static_cast<long long>(max(x.src, x.dst)));
  }
  for (int o = 16; o; o >>= 1) mx = max(mx, __shfl_xor_sync(kFull, mx, o));
  if ((threadIdx.x & 31) == 0 && mx >= 0) atomicMax(max_node, static_cast<unsigned long long>(mx));
}

__global__ void k_emit_features(const uint32_t* __restrict__ perm, const int64_t* __restrict__ row_line,
                                int64_t n, int d_e, const double* __restrict__ feats,
                                double* __restrict__ out) {
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < n * d_e;
       x += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = x / d_e, f = x - k * d_e;
    out[x] = feats[row_line[perm[k]] * d_e + f];
  }
}

// test/utility kernel: parse n fields [off[i], off[i+1]) of buf as int64 (kind 0) or double
__global__ void k_parse_numbers(const char* __restrict__ buf, const int64_t* __restrict__ off,
                                int64_t n, int kind, int64_t* __restrict__ iout,
                                double* __restrict__ dout, int* __restrict__ status) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const char* p = buf + off[i];
    const char* e = buf + off[i + 1];
    trim(p, e);
    if (kind == 0) {
      int64_t v = 0;
      status[i] = parse_i64(p, e, v);
      iout[i] = v;
    } else {
      double v = 0.0;
      status[i] = parse_f64(p, e, v);
      dout[i] = v;
    }
  }
}

int grid_of(int64_t work) {
  return static_cast<int>(std::max<int64_t>(
      1, std::min<int64_t>(ceil_div(std::max<int64_t>(work, 1), 256), device_info().sms * 8LL)));
}

}  // namespace

void launch_parse_numbers(const char* buf, const int64_t* off, int64_t n, int kind, int64_t* iout,
                          double* dout, int* status, cudaStream_t s) {
  if (n <= 0) return;
  k_parse_numbers<<<grid_of(n), 256, 0, s>>>(buf, off, n, kind, iout, dout, status);
  after_launch("k_parse_numbers");
}

// Parses the CSV in d_buf (device bytes) whose header has `header_fields` fields.  On success
// fills the result arrays; on a per-line error returns its error word (line << 8 | code).
uint64_t parse_csv_device(const char* d_buf, int64_t nbytes, int d_e, CsvResult* res,
                          cudaStream_t s) {
  const int64_t tiles = std::max<int64_t>(1, ceil_div(nbytes, kTileBytes));
  uint32_t* cnt = static_cast<uint32_t*>(dmalloc(4 * tiles, s));
  int64_t* off = static_cast<int64_t*>(dmalloc(8 * (tiles + 1), s));
  k_nl_count<<<static_cast<int>(tiles), kNT, 0, s>>>(d_buf, nbytes, cnt);
  after_launch("k_nl_count");
  scan_u32_to_i64(cnt, tiles, off, s);
  int64_t nnl = 0;
  TGFX_CUDA(cudaMemcpyAsync(&nnl, off + tiles, 8, cudaMemcpyDeviceToHost, s));
  TGFX_CUDA(cudaStreamSynchronize(s));
  int64_t* nl = static_cast<int64_t*>(dmalloc(8 * std::max<int64_t>(nnl, 1), s));
  k_nl_write<<<static_cast<int>(tiles), kNT, 0, s>>>(d_buf, nbytes, off, nl);
  after_launch("k_nl_write");
  char last = '\n';
  if (nbytes > 0) TGFX_CUDA(cudaMemcpyAsync(&last, d_buf + nbytes - 1, 1, cudaMemcpyDeviceToHost, s));
  TGFX_CUDA(cudaStreamSynchronize(s));
  const int64_t L = nnl + (nbytes > 0 && last != '\n' ? 1 : 0);  // getline's line count
  const size_t Lb = static_cast<size_t>(std::max<int64_t>(L, 1));
  int64_t* src = static_cast<int64_t*>(dmalloc(8 * Lb, s));
  int64_t* dst = static_cast<int64_t*>(dmalloc(8 * Lb, s));
  double* t = static_cast<double*>(dmalloc(8 * Lb, s));
  uint32_t* keep = static_cast<uint32_t*>(dmalloc(4 * Lb, s));
  double* feats = static_cast<double*>(dmalloc(8 * Lb * std::max(d_e, 1), s));
  unsigned long long* err = static_cast<unsigned long long*>(dmalloc(8, s));
  TGFX_CUDA(cudaMemsetAsync(err, 0xff, 8, s));
  TGFX_CUDA(cudaMemsetAsync(keep, 0, 4 * Lb, s));
  if (L > 1) {
    k_parse_lines<<<grid_of(L), 256, 0, s>>>(d_buf, nbytes, nl, nnl, L, d_e, src, dst, t, keep,
                                             feats, err);
    after_launch("k_parse_lines");
  }
  unsigned long long herr = 0;
  TGFX_CUDA(cudaMemcpyAsync(&herr, err, 8, cudaMemcpyDeviceToHost, s));
  TGFX_CUDA(cudaStreamSynchronize(s));
  auto release = [&] {
    for (void* q : {static_cast<void*>(cnt), static_cast<void*>(off), static_cast<void*>(nl),
                    static_cast<void*>(src), static_cast<void*>(dst), static_cast<void*>(t),
                    static_cast<void*>(keep), static_cast<void*>(feats), static_cast<void*>(err)})
      dfree(q, s);
  };
  if (herr != ~0ull) {
    res->err_line_start = 0;
    const int64_t li = static_cast<int64_t>(herr >> 8) - 1;  // 0-based line index
    int64_t b = 0, en = nbytes;
    if (li >= 1) TGFX_CUDA(cudaMemcpyAsync(&b, nl + li - 1, 8, cudaMemcpyDeviceToHost, s));
    if (li < nnl) TGFX_CUDA(cudaMemcpyAsync(&en, nl + li, 8, cudaMemcpyDeviceToHost, s));
    TGFX_CUDA(cudaStreamSynchronize(s));
    res->err_line_start = li >= 1 ? b + 1 : 0;
    res->err_line_end = en;
    release();
    return herr;
  }
  // keep -> rank (exclusive scan), n = kept lines
  int64_t* rank = static_cast<int64_t*>(dmalloc(8 * (Lb + 1), s));
  scan_u32_to_i64(keep, L, rank, s);
  int64_t n = 0;
  TGFX_CUDA(cudaMemcpyAsync(&n, rank + L, 8, cudaMemcpyDeviceToHost, s));
  TGFX_CUDA(cudaStreamSynchronize(s));
  const size_t nb = static_cast<size_t>(std::max<int64_t>(n, 1));
  uint64_t* key = static_cast<uint64_t*>(dmalloc(8 * nb, s));
  uint64_t* kalt = static_cast<uint64_t*>(dmalloc(8 * nb, s));
  uint32_t* val = static_cast<uint32_t*>(dmalloc(4 * nb, s));
  uint32_t* valt = static_cast<uint32_t*>(dmalloc(4 * nb, s));
  int64_t* row_line = static_cast<int64_t*>(dmalloc(8 * nb, s));
  if (L > 1) {
    k_rows<<<grid_of(L), 256, 0, s>>>(keep, rank, L, t, key, val, row_line);
    after_launch("k_rows");
  }
  uint64_t* kk = key;
  uint32_t* vv = val;
  if (n > 1) radix_sort_pairs<uint64_t, uint32_t>(kk, vv, kalt, valt, n, 64, s);  // stable, by time
  res->n = n;
  res->events = static_cast<tgfx_event*>(dmalloc(32 * nb, s));
  res->features = d_e > 0 ? static_cast<double*>(dmalloc(8 * nb * d_e, s)) : nullptr;
  unsigned long long* mx = static_cast<unsigned long long*>(dmalloc(8, s));
  TGFX_CUDA(cudaMemsetAsync(mx, 0, 8, s));  // ids are >= 0 (checked)
  if (n > 0) {
    k_emit<<<grid_of(n), 256, 0, s>>>(vv, row_line, n, src, dst, t, res->events, mx);
    after_launch("k_emit");
    if (d_e > 0) {
      k_emit_features<<<grid_of(n * d_e), 256, 0, s>>>(vv, row_line, n, d_e, feats, res->features);
      after_launch("k_emit_features");
    }
  }
  unsigned long long hmx = 0;
  TGFX_CUDA(cudaMemcpyAsync(&hmx, mx, 8, cudaMemcpyDeviceToHost, s));
  TGFX_CUDA(cudaStreamSynchronize(s));
  res->num_nodes = n > 0 ? static_cast<int64_t>(hmx) + 1 : 0;
  release();
  for (void* q : {static_cast<void*>(rank), static_cast<void*>(key), static_cast<void*>(kalt),
                  static_cast<void*>(val), static_cast<void*>(valt), static_cast<void*>(row_line),
                  static_cast<void*>(mx)})
    dfree(q, s);
  return ~0ull;
}

}  // namespace tgfx
