// graph.cuh -- the device-resident T-CSR handle and the builder / sampler entry points.
#pragma once

#include <mutex>

#include "common.cuh"

// Device-side build diagnostics, written by the histogram pass.
struct BuildFlags {
  unsigned long long bad_index;  // min stream index of an event with an endpoint out of range
  int unsorted;                  // stream is not (t, eid)-non-decreasing (or holds NaN times)
  int has_nan;                   // some timestamp is NaN
  long long max_eid;
  long long min_eid;
};

// 64 B per node (one 64-byte line, two 256-bit loads).  bkt != nullptr: the slice has a time
// bucket table of nb + 1 entries, bkt[j] = #slice entries whose bucket_of(ts) < j (relative),
// so lower_bound(t) lies in [bkt[j], bkt[j + 1]] for j = bucket_of(t) (see build_node_dir).
struct __align__(32) NodeDir {
  int64_t start, end;
  double t_first, t_last;
  const uint32_t* bkt;
  double scale;  // nb / (t_last - t_first)
  int64_t nb;
  double width;  // (t_last - t_first) / nb: bucket edges for the interpolation hints
};

// The recent-k sampler's compact copy of a NodeDir: 32 B per node, ONE 256-bit load.  A
// slice's bucket table sits at bkt_base + start / R + 2u (tables never overlap: nb + 1 <=
// n / R + 2), so no pointer is stored; st = scale when nb > 0 (t_last is then not needed: the
// last bucket's table entry brackets a query past the slice), else t_last.
struct __align__(32) DirC {
  int64_t start;
  uint32_t n, nb;
  double t_first;
  double st;
};

// bucket of time t in a slice with a bucket table: floor((t - t_first) * scale) clamped to
// nb - 1 (nb < 2^32).  Monotone non-decreasing in t; the builder and the sampler evaluate this
// same expression (explicitly rounded, never contracted), which is all exactness needs.
__host__ __device__ __forceinline__ uint32_t bucket_of(double t, double t_first, double scale,
                                                       int64_t nb) {
#ifdef __CUDA_ARCH__
  const double x = __dmul_rn(__dsub_rn(t, t_first), scale);
#else
  volatile double dx = t - t_first;
  const double x = dx * scale;
#endif
  return x < static_cast<double>(nb - 1) ? static_cast<uint32_t>(x) : static_cast<uint32_t>(nb - 1);
}

// proj/include/tgformer/tcsr.hpp:20-33 (TCsr), resident on one device.  SoA columns in HBM:
//   indptr int64[V+1] | nbr int64[m] | eid int64[m] | ts f64[m]   (m = n * (1 + reverse))
struct tgfx_graph {
  int device = 0;
  int64_t V = 0, n = 0, m = 0;
  int reverse = 1;
  int path = 0;  // 0 fast presorted, 1 general re-sort, 2 large-V radix
  // 1: slices may not be sorted NaN-free (NaN timestamps, or imported from host unchecked), so
  // the sampler replays std::lower_bound's exact bisection; 0: slices are sorted, any
  // bracketing search (interpolation) returns the same lower_bound.
  int search_exact = 0;
  // 1: an imported indptr is not monotone within [0, m] (or has wrong endpoints); no node
  // directory is built, samplers refuse the graph, validate() reports the reference's error
  int indptr_bad = 0;
  int64_t* indptr = nullptr;
  int64_t* nbr = nullptr;
  int64_t* eid = nullptr;
  double* ts = nullptr;  // allocated with kTsPad trailing entries (line probes read whole lines)
  // node directory, 32 B per node: {slice start, slice end, ts[start], ts[end-1]} -- one
  // record gives the sampler both the slice bounds and the interpolation bracket
  NodeDir* dir = nullptr;
  DirC* dirc = nullptr;  // compact copy for the recent-k sampler (entries_per_bucket below)
  int64_t bkt_r = 0;     // entries per time bucket the tables were built with (0: none)
  // time bucket tables of the slices (uint32, ~m / bucket_entries + 2V), see NodeDir
  uint32_t* bkt = nullptr;
  int64_t bkt_cap = 0;
  // sampler gather records, 16 B per entry {u32 nbr, u32 eid, f64 ts} (ids < 2^31 only):
  // one 16-byte load per window slot instead of three 8-byte column loads
  uint4* rec = nullptr;
  int64_t rec_cap = 0;
  // false: the last build wrote rec (+ ts) instead of the int64 nbr / eid columns; they are
  // widened from rec by ensure_columns before anything outside the sampler reads them
  bool cols_valid = true;
  std::mutex cols_mu;  // serialises the lazy widening: a graph is shared by concurrent readers
  // bound on the other endpoint (nbr ids): V for an ordinary build; the global node count for
  // one node range of a partitioned build (reverse = 0, nbr ids stay global)
  int64_t other_limit = 0;
  int64_t eid_limit = 0;  // edge ids are < eid_limit (n, or the global event count of a range build)
  int64_t max_eid = -1, min_eid = 0;
  // build workspace, kept for rebuilds
  void* ws = nullptr;  // per-chunk node count / cursor table
  size_t ws_bytes = 0;
  void* ws_small = nullptr;  // cold bitmask + per-chunk cold counts / offsets
  size_t ws_small_bytes = 0;
  void* ws_rec = nullptr;  // deferred (cold) entry records, 24 B each
  size_t ws_rec_bytes = 0;
  BuildFlags* dflags = nullptr;
  BuildFlags* hflags = nullptr;  // pinned host mirror
};

// Parsed event stream resident on the device (tgfx_load_csv / tgfx_csv_parse_device).
struct tgfx_csv {
  int64_t n = 0, num_nodes = 0, d_e = 0;
  tgfx_event* events = nullptr;
  double* features = nullptr;
};

namespace tgfx {

// max num_nodes of the shared-memory (per-chunk cursor) fast path
int64_t fast_path_max_nodes();

// Allocates the columns of g (V, n, reverse set by caller).
void graph_alloc(tgfx_graph* g, cudaStream_t s);
void graph_release(tgfx_graph* g);

// trailing pad entries of the ts column (multiple of the widest line probe)
constexpr int64_t kTsPad = 32;

// (re)compute the node directory from indptr + ts (after a build or an import)
void build_node_dir(tgfx_graph* g, cudaStream_t s);

// Full build into g from device events; throws tgfx::Error on invalid input.
void build_graph(tgfx_graph* g, const tgfx_event* d_ev, cudaStream_t s, bool trusted);

// Materialises the int64 nbr / eid columns from the gather records if the build skipped them.
void ensure_columns(const tgfx_graph* g, cudaStream_t s);

// TCsr::validate on device (tcsr.cpp:54-81); returns empty string if valid.
std::string validate_graph(const tgfx_graph* g, cudaStream_t s);

// ------------------------------------------------------------------ sampling
struct SampleArgs {
  const tgfx_graph* g;
  const int64_t* nodes;
  const double* times;
  int64_t q, k;
  int strategy;
  uint64_t seed, stream_base;
  // assemble outputs (l > 0)
  int64_t l = 0;
  int64_t self_edge_index = 0;
  void* node_index = nullptr;
  void* edge_index = nullptr;
  float* dt32 = nullptr;
  double* dt64 = nullptr;
  void* valid_len = nullptr;
  bool index64 = false;
  // entries outputs (l == 0): padded [q, k]
  int64_t* counts = nullptr;
  int64_t* e_nbr = nullptr;
  int64_t* e_eid = nullptr;
  double* e_ts = nullptr;
  int64_t e_stride = 1;  // 3: e_nbr/e_eid/e_ts interleaved as tgfx_neighbor records
  // hop-2 mode: query (nodes, times) given padded [q_roots, k1] with per-root counts
  const int64_t* hop_counts = nullptr;
  int64_t hop_k1 = 0;
  // batched uniform sampling: batch b = query / batch_q uses seeds[b] (device array)
  const uint64_t* seeds = nullptr;
  int64_t batch_q = 0;
  // fused query check: first failing stream_base + q (atomicMin), or nullptr
  unsigned long long* first_bad = nullptr;
};

// first invalid query index (or -1); validates node range on device (sampler.cpp:22-27)
int64_t find_bad_query(const tgfx_graph* g, const int64_t* d_nodes, int64_t q, cudaStream_t s);
// atomicMin of (base + index) of every out-of-range node of d_nodes[0, q) into *d_first; the
// bad entries of d_nodes (a caller-owned copy) are replaced by node 0
void find_bad_async(const tgfx_graph* g, int64_t* d_nodes, int64_t q, int64_t base,
                    unsigned long long* d_first, cudaStream_t s);
void launch_sample(const SampleArgs& a, cudaStream_t s);
void launch_two_hop(const tgfx_graph* g, const int64_t* roots, const double* times, int64_t q,
                    int64_t k1, int64_t k2, int strategy, uint64_t seed, uint64_t seed2,
                    int64_t l, int64_t self_edge_index, int32_t* h1n, int32_t* h1e, float* h1d,
                    int32_t* h1l, int32_t* h2n, int32_t* h2e, float* h2d, int32_t* h2l,
                    cudaStream_t s);

// ------------------------------------------------------------------ sequences / masks
void launch_assemble_entries(int64_t q, int64_t kpad, const int64_t* counts, const int64_t* nbr,
                             const int64_t* eid, const double* ts, const int64_t* qn,
                             const double* qt, int64_t l, int64_t self_edge_index,
                             int64_t* node_index, int64_t* edge_index, double* dt,
                             int64_t* valid_len, int64_t* target_row, cudaStream_t s,
                             int64_t es = 1);
void launch_mask(int64_t q, int64_t l, const int64_t* valid_len, const int64_t* target_row,
                 int kind, double* mask, cudaStream_t s);

// ------------------------------------------------------------------ assemble_inputs
struct AssembleInputsArgs {
  int64_t q = 0, l = 0;
  const void* node_index = nullptr;  // int32 or int64 [q*l] (index64)
  const void* edge_index = nullptr;
  const void* time_delta = nullptr;  // f32 or f64 [q*l] (dt_type)
  const void* valid_len = nullptr;   // int32 or int64 [q]
  int index64 = 0, dt_type = 0;
  const void* node_table = nullptr;  // [node_rows, d_v]
  const void* edge_table = nullptr;  // [edge_rows, d_e]
  int64_t node_rows = 0, edge_rows = 0;
  int table_type = 0;
  const double* omega = nullptr;  // [d_t]
  const double* phi = nullptr;
  int64_t d_v = 0, d_e = 0, d_t = 0;
  int concat = 0;
  void* z = nullptr;  // [q*l, d]
  int z_type = 0;
};
void launch_assemble_inputs(const AssembleInputsArgs& a, int* bad, cudaStream_t s);

// fused sampler + assemble_inputs (recent-k, line-probe graphs): s = the sampling arguments
// (valid_len int32 or null), in = the tables / z (its row fields unused); false = not taken
struct SampleInputsArgs {
  SampleArgs s;
  AssembleInputsArgs in;
};
bool launch_sample_inputs(const SampleInputsArgs& a, int* bad, cudaStream_t s);

// ------------------------------------------------------------------ CSV ingestion
struct CsvResult {
  int64_t n = 0, num_nodes = 0;
  tgfx_event* events = nullptr;  // device, n
  double* features = nullptr;    // device, n x d_e (or null)
  int64_t err_line_start = 0, err_line_end = 0;  // byte span of the failing line
};
// error codes of parse_csv_device's error word (line_no << 8 | code)
enum CsvError : int {
  kCsvFields = 1, kCsvSrc, kCsvDst, kCsvTime, kCsvNegNode, kCsvNegTime, kCsvFeature,
  kCsvUnsupported
};
// ~0 on success (res filled), else the first failing line's error word
uint64_t parse_csv_device(const char* d_buf, int64_t nbytes, int d_e, CsvResult* res,
                          cudaStream_t s);
// fields [off[i], off[i+1]) as int64 (kind 0) / double (kind 1); status 0 ok, 1 bad, 2 unsupported
void launch_parse_numbers(const char* buf, const int64_t* off, int64_t n, int kind, int64_t* iout,
                          double* dout, int* status, cudaStream_t s);

// ------------------------------------------------------------------ synthetic
void launch_random_stream(int64_t E, int64_t V, uint64_t seed, double zipf, tgfx_event* d_out,
                          cudaStream_t s);
void launch_make_queries(const tgfx_event* ev, int64_t e0, int64_t e1, int64_t batch, int64_t V,
                         uint64_t neg_seed, int64_t* nodes, double* times, cudaStream_t s);
void launch_train_queries(const tgfx_event* ev, int64_t n, int64_t b0, int64_t b1, int64_t B,
                          int64_t npp, int64_t workers, int64_t V, uint64_t batch_seed,
                          int64_t* nodes, double* times, cudaStream_t s);

// ------------------------------------------------------------------ partitioned build
void launch_degree_hist(const tgfx_event* ev, int64_t n, int64_t V, int reverse,
                        unsigned long long* deg, cudaStream_t s);
int64_t partition_warps(int64_t n);
void launch_partition_count(const tgfx_event* ev, int64_t n, int reverse, const int64_t* bounds,
                            int N, int64_t nw, const int64_t* split, int64_t* counts,
                            int64_t* scounts, cudaStream_t s);
void launch_partition_scatter(const tgfx_event* ev, int64_t n, int reverse, const int64_t* bounds,
                              int N, int64_t nw, const int64_t* split, const int64_t* occ,
                              const int64_t* offs, tgfx_event* out, cudaStream_t s);
// 1 if any ts is NaN
bool any_nan(const double* ts, int64_t m, cudaStream_t s);
bool indptr_in_range(const int64_t* indptr, int64_t V, int64_t m, cudaStream_t s);

// ------------------------------------------------------------------ primitives
// exclusive scan of n uint32 counts into int64 offsets (out has n+1 entries: out[n] = total)
void scan_u32_to_i64(const uint32_t* in, int64_t n, int64_t* out, cudaStream_t s);

}  // namespace tgfx
