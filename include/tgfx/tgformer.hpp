// tgfx/tgformer.hpp -- C++ host API of the B200-native hot path, source-compatible with the
// reference library's builder / sampler / sequence API (namespace tgf; arXiv 2409.05477
// reference tree, proj/include/tgformer/*.hpp).  A caller of the reference recompiles against
// this header (or the include/tgformer/*.hpp forwarders, which keep the reference's include
// paths) and links libtgformer.so + libtgfx.so instead of the reference's tcsr.cpp,
// sampler.cpp and sequence.cpp.  Every computation goes through the C ABI (include/tgfx.h)
// into the sm_100a kernels; this layer only marshals std::vector <-> device buffers and turns
// status codes back into the reference's exception types.
//
//   reference (proj/include/tgformer/...)        here
//   common.hpp:10-27   ids, time, errors         same names and types
//   rng.hpp:11-52      mix64, CounterRng          same (callers and tests draw with it)
//   matrix.hpp:12-45   Matrix                     same interface (row-major double)
//   event_stream.hpp   TemporalEvent, EventStream same layout (32-byte events = tgfx_event)
//   tcsr.hpp:20-47     TCsr, build_*, container   same; TCsr also owns its device copy
//   sampler.hpp:12-45  NeighborSample, sample_*   same
//   sequence.hpp:20-50 SequenceBatch, masks       same
//   synthetic.hpp:17   make_random_stream         same (device generator, bit-identical)
//
// Differences a caller can observe: none in values; num_threads is accepted and ignored (the
// reference's results are thread-count independent too).
#pragma once

#include <cstddef>
#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "tgfx.h"

namespace tgf {

// ------------------------------------------------------------------ common.hpp
using NodeId = std::int64_t;
using EdgeId = std::int64_t;
using Time = double;

struct ValidationError : std::runtime_error {
  explicit ValidationError(const std::string& what) : std::runtime_error(what) {}
};
struct ParseError : std::runtime_error {
  explicit ParseError(const std::string& what) : std::runtime_error(what) {}
};
struct FormatError : std::runtime_error {
  explicit FormatError(const std::string& what) : std::runtime_error(what) {}
};

// ------------------------------------------------------------------ rng.hpp
// splitmix64 finaliser and the (seed, stream) counter generator; the device kernels use the
// same functions (csrc/common.cuh), so host draws and device draws agree bit for bit.
inline std::uint64_t mix64(std::uint64_t z) {
  z += 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

class CounterRng {
 public:
  CounterRng(std::uint64_t seed, std::uint64_t stream)
      : s_(mix64(mix64(seed) ^ (stream * 0xd6e8feb86659fd93ULL))) {}
  std::uint64_t next_u64() {
    s_ += 0x9e3779b97f4a7c15ULL;
    return mix64(s_ - 0x9e3779b97f4a7c15ULL);
  }
  std::uint64_t next_below(std::uint64_t bound) {
    return static_cast<std::uint64_t>((static_cast<unsigned __int128>(next_u64()) * bound) >> 64);
  }
  double next_double() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }
  double next_uniform(double lo, double hi) { return lo + (hi - lo) * next_double(); }

 private:
  std::uint64_t s_;
};

// ------------------------------------------------------------------ matrix.hpp
class Matrix {
 public:
  Matrix() = default;
  Matrix(std::size_t rows, std::size_t cols) : r_(rows), c_(cols), v_(rows * cols, 0.0) {}
  // a rows x cols copy of src (row-major), without first zero-filling
  Matrix(std::size_t rows, std::size_t cols, const double* src)
      : r_(rows), c_(cols), v_(src, src + rows * cols) {}
  std::size_t rows() const { return r_; }
  std::size_t cols() const { return c_; }
  std::size_t size() const { return v_.size(); }
  bool empty() const { return v_.empty(); }
  double* row(std::size_t i) { return v_.data() + i * c_; }
  const double* row(std::size_t i) const { return v_.data() + i * c_; }
  double& at(std::size_t i, std::size_t j) { return v_[i * c_ + j]; }
  double at(std::size_t i, std::size_t j) const { return v_[i * c_ + j]; }
  double* data() { return v_.data(); }
  const double* data() const { return v_.data(); }
  void fill(double x) { v_.assign(v_.size(), x); }
  bool same_shape(const Matrix& o) const { return r_ == o.r_ && c_ == o.c_; }
  friend bool operator==(const Matrix& a, const Matrix& b) {
    return a.r_ == b.r_ && a.c_ == b.c_ && a.v_ == b.v_;
  }

 private:
  std::size_t r_ = 0, c_ = 0;
  std::vector<double> v_;
};

// Dense-algebra helpers of matrix.hpp:48-57, declared so the reference's model headers
// compile against this one; they are defined by the reference's matrix.cpp (the model is not
// part of this library -- only the path's data structures are).
void gemm(bool trans_a, bool trans_b, double alpha, const Matrix& a, const Matrix& b,
          double beta, Matrix& c);
double max_abs_diff(const Matrix& a, const Matrix& b);
void pin_blas_single_thread();

// ------------------------------------------------------------------ event_stream.hpp
struct TemporalEvent {
  EdgeId edge_id = 0;
  NodeId src = 0;
  NodeId dst = 0;
  Time timestamp = 0.0;
};
static_assert(sizeof(TemporalEvent) == sizeof(tgfx_event), "events upload without repacking");

struct EventStream {
  std::vector<TemporalEvent> events;
  NodeId num_nodes = 0;
  std::int64_t d_e = 0;
  std::int64_t d_v = 0;
  Matrix edge_features;
  Matrix node_features;
  std::int64_t size() const { return static_cast<std::int64_t>(events.size()); }
  void validate() const;  // event_stream.cpp:62-83 checks and messages
};

// event_stream.hpp:44: parsed on the device (tgfx_load_csv); same ordering, ids, errors.
EventStream load_csv(const std::string& path, bool has_features = false);

// ------------------------------------------------------------------ tcsr.hpp
namespace detail {
struct DeviceCopy;  // device-resident T-CSR handle + content fingerprint (tgformer.cpp)
}

struct TCsr {
  NodeId num_nodes = 0;
  std::int64_t num_edges = 0;
  bool reverse = true;
  std::vector<std::int64_t> indptr;
  std::vector<NodeId> neighbor_ids;
  std::vector<EdgeId> edge_ids;
  std::vector<Time> timestamps;

  std::int64_t num_entries() const { return static_cast<std::int64_t>(neighbor_ids.size()); }
  std::int64_t degree(NodeId u) const { return indptr[u + 1] - indptr[u]; }
  void validate() const;  // run on the device (tgfx_graph_validate)

  // The device copy the sampler reads: attached by the builders and load_tcsr, uploaded on
  // first use for a TCsr assembled by hand, re-uploaded if the host columns changed.
  tgfx_graph* device() const;
  mutable std::shared_ptr<detail::DeviceCopy> device_copy;
};

TCsr build_sequential(const EventStream& stream, bool reverse = true);
TCsr build_parallel(const EventStream& stream, bool reverse, int num_threads);
// TCSR v1 container (byte-compatible with tcsr.cpp:153-197 below 4 GiB; CRC-32 computed in
// chunks so files of any size round-trip).
void save_tcsr(const TCsr& graph, const std::string& path);
TCsr load_tcsr(const std::string& path);

// ------------------------------------------------------------------ sampler.hpp
struct NeighborEntry {
  NodeId neighbor;
  EdgeId edge;
  Time timestamp;
};

struct NeighborSample {
  NodeId query_node = 0;
  Time query_time = 0.0;
  std::vector<NeighborEntry> neighbors;
};

enum class SampleStrategy { recent, random };
SampleStrategy parse_strategy(const std::string& name);

NeighborSample sample_recent(const TCsr& g, NodeId u, Time t, std::int64_t k);
NeighborSample sample_random(const TCsr& g, NodeId u, Time t, std::int64_t k,
                             std::uint64_t seed, std::uint64_t stream = 0);
std::vector<NeighborSample> sample_batch(const TCsr& g, const std::vector<NodeId>& nodes,
                                         const std::vector<Time>& times, std::int64_t k,
                                         SampleStrategy strategy, std::uint64_t seed,
                                         int num_threads = 0);

// ------------------------------------------------------------------ sequence.hpp
struct SequenceBatch {
  std::int64_t batch = 0;
  std::int64_t l = 0;
  std::vector<std::int64_t> node_index;
  std::vector<std::int64_t> edge_index;
  Matrix time_delta;
  std::vector<std::int64_t> valid_len;
  std::vector<std::int64_t> target_row;
  void validate() const;  // sequence.cpp:13-46 checks and messages
};

enum class MaskKind { causal, tgat, self_loop };
MaskKind parse_mask_kind(const std::string& name);

SequenceBatch build_sequence(const NeighborSample& sample, std::int64_t l,
                             std::int64_t self_edge_index);
SequenceBatch build_sequence_batch(const std::vector<NeighborSample>& samples, std::int64_t l,
                                   std::int64_t self_edge_index);
Matrix build_mask(const SequenceBatch& batch, MaskKind kind);

// Extension (not in the reference): the one-call form of forward_concat's pair
// (training.cpp:211-214),
//   build_sequence_batch(sample_batch(g, nodes, times, k, strategy, seed), l, self_edge_index)
// with identical results and errors, computed on the device without materialising
// NeighborSamples on the host.  A caller swaps the two calls for this one.
SequenceBatch sample_sequence_batch(const TCsr& g, const std::vector<NodeId>& nodes,
                                    const std::vector<Time>& times, std::int64_t k,
                                    SampleStrategy strategy, std::uint64_t seed, std::int64_t l,
                                    std::int64_t self_edge_index, int num_threads = 0);

// ------------------------------------------------------------------ synthetic.hpp
EventStream make_random_stream(std::int64_t num_edges, NodeId num_nodes, std::uint64_t seed,
                               double zipf_exponent = 1.2);

}  // namespace tgf
