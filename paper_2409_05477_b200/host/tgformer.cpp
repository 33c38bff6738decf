// tgformer.cpp -- C++ host layer (include/tgfx/tgformer.hpp) over the C ABI (include/tgfx.h).
//
// Each function here replaces the reference function of the same name and keeps its
// argument meaning, return values and exception types; the arithmetic runs in libtgfx's
// sm_100a kernels.  The only host-side work is marshalling (vectors <-> pinned/device
// buffers), the argument checks the reference does before computing, and the TCSR container
// file I/O.  Reference locations are relative to the reference tree (proj/...).
#include "tgfx/tgformer.hpp"

#include <zlib.h>

#include <algorithm>
#include <cstddef>
#include <cstring>
#include <fstream>
#include <mutex>
#include <type_traits>

#include <omp.h>

namespace tgf {

namespace detail {

// Rethrow a libtgfx status as the reference's exception type (common.hpp:15-27).
[[noreturn]] void throw_status(int rc, const std::string& msg) {
  if (rc == TGFX_EVALIDATION) throw ValidationError(msg);
  if (rc == TGFX_EFORMAT) throw FormatError(msg);
  if (rc == TGFX_EPARSE) throw ParseError(msg);
  if (rc == TGFX_ENOMEM) throw std::bad_alloc();
  throw std::runtime_error(msg);
}

void check(int rc) {
  if (rc != TGFX_OK) throw_status(rc, tgfx_last_error());
}

// Per-thread page-locked staging for the host <-> device copies of the sampling and sequence
// calls (grown on demand, kept for the thread's lifetime): a copy from or to it is one DMA,
// where a copy from a std::vector's pageable memory goes through the driver's bounce buffer.
struct Pinned {
  void* p = nullptr;
  std::size_t cap = 0;
  Pinned() = default;
  Pinned(const Pinned&) = delete;
  Pinned& operator=(const Pinned&) = delete;
  ~Pinned() {
    if (p) tgfx_host_free(p);
  }
  char* get(std::size_t bytes) {
    if (bytes > cap) {
      if (p) tgfx_host_free(p);
      p = nullptr;
      cap = 0;
      const std::size_t c = std::max<std::size_t>(bytes + bytes / 2, std::size_t(1) << 20);
      check(tgfx_host_alloc(c, &p));
      cap = c;
    }
    return static_cast<char*>(p);
  }
};

Pinned& pinned_in() {
  thread_local Pinned b;
  return b;
}
Pinned& pinned_out() {
  thread_local Pinned b;
  return b;
}


// bodies of loops over a batch's queries: OpenMP threads once a batch is large enough that
// the vector allocations and copies outweigh waking the team (the reference's own loops
// are OpenMP too, sampler.cpp:95)
constexpr std::int64_t kParMin = 512;

// Fingerprint of the host columns: their sizes, plus a full FNV-1a over small graphs and 64
// strided words per column over large ones (not the addresses: a copied TCsr shares its
// source's device copy).  Detects a TCsr whose columns were replaced (or resized) after its
// device copy was made; an in-place edit of a large column is usually missed (the reference treats TCsr as immutable).  It runs on every
// sampling call, so it stays far below a batch's own cost: 256 cache misses, not 16 K.
std::uint64_t fingerprint(const TCsr& g) {
  std::uint64_t h = 1469598103934665603ULL;
  auto mixin = [&](std::uint64_t x) {
    h ^= x;
    h *= 1099511628211ULL;
  };
  mixin(static_cast<std::uint64_t>(g.num_nodes));
  mixin(static_cast<std::uint64_t>(g.num_edges));
  mixin(g.reverse ? 1 : 0);
  auto cols = [&](const void* p, std::size_t n) {
    mixin(n);
    const auto* w = static_cast<const std::uint64_t*>(p);
    const std::size_t step = n <= (1u << 12) ? 1 : n / 64;
    for (std::size_t i = 0; i < n; i += step) mixin(w[i] + i);
    if (n) mixin(w[n - 1]);
  };
  cols(g.indptr.data(), g.indptr.size());
  cols(g.neighbor_ids.data(), g.neighbor_ids.size());
  cols(g.edge_ids.data(), g.edge_ids.size());
  cols(g.timestamps.data(), g.timestamps.size());
  return h;
}

struct DeviceCopy {
  tgfx_graph* handle = nullptr;
  std::uint64_t fp = 0;
  std::int64_t max_degree = 0;
  ~DeviceCopy() {
    if (handle) tgfx_graph_free(handle);
  }
};

std::int64_t max_degree(const TCsr& g) {
  std::int64_t d = 0;
  for (std::size_t u = 0; u + 1 < g.indptr.size(); ++u) d = std::max(d, g.indptr[u + 1] - g.indptr[u]);
  return d;
}

// A TCsr is shared by concurrent readers: every read or replacement of its
// device_copy pointer, and every first upload, happens under this lock.  Callers hold the
// returned shared_ptr while they use the handle, so a concurrent replacement cannot free it.
std::mutex& copy_mu() {
  static std::mutex mu;
  return mu;
}

std::shared_ptr<DeviceCopy> make_copy(const TCsr& g, tgfx_graph* h) {
  auto dc = std::make_shared<DeviceCopy>();
  dc->handle = h;
  dc->fp = fingerprint(g);
  dc->max_degree = max_degree(g);
  return dc;
}

void attach(const TCsr& g, tgfx_graph* h) {
  std::shared_ptr<DeviceCopy> dc;
  try {
    dc = make_copy(g, h);
  } catch (...) {
    tgfx_graph_free(h);
    throw;
  }
  std::lock_guard<std::mutex> lk(copy_mu());
  g.device_copy = std::move(dc);
}

// Upload a TCsr that has no (or a stale) device copy.  The shape checks are TCsr::validate's
// (tcsr.cpp:54-61), done before touching the columns.
tgfx_graph* upload(const TCsr& g) {
  if (g.indptr.size() != static_cast<std::size_t>(g.num_nodes) + 1)
    throw ValidationError("indptr size mismatch");
  if (g.edge_ids.size() != g.neighbor_ids.size() || g.timestamps.size() != g.neighbor_ids.size())
    throw ValidationError("column arrays disagree in length");
  tgfx_graph* h = nullptr;
  const std::int64_t m = g.num_entries();
  // the device handle stores num_edges * (1 + reverse) entries; a hand-made TCsr may not
  // follow that rule, so describe it by its entry count
  const int rev = (m == 2 * g.num_edges && m > 0) ? 1 : (m == g.num_edges ? 0 : -1);
  if (rev < 0) {
    // entries do not follow the builder's n*(1+reverse) shape: store as a non-reverse graph of
    // m "events" (sampling only reads the columns; validate() checks ids against num_edges)
    check(tgfx_graph_from_host(g.num_nodes, m, 0, m, g.indptr.data(), g.neighbor_ids.data(),
                               g.edge_ids.data(), g.timestamps.data(), &h));
  } else {
    check(tgfx_graph_from_host(g.num_nodes, g.num_edges, rev, m, g.indptr.data(),
                               g.neighbor_ids.data(), g.edge_ids.data(), g.timestamps.data(), &h));
  }
  return h;
}

// The device copy to sample from.  The fingerprint samples large columns (see fingerprint),
// so an in-place edit of a few entries after the copy exists can go unnoticed here: a TCsr
// must not be edited once sampled (the reference treats it as immutable).  validate() always
// checks freshly uploaded columns (TCsr::validate below).
std::shared_ptr<DeviceCopy> device_of(const TCsr& g) {
  std::lock_guard<std::mutex> lk(copy_mu());
  std::shared_ptr<DeviceCopy> dc = g.device_copy;
  if (!dc || dc->fp != fingerprint(g)) {
    tgfx_graph* h = upload(g);
    try {
      dc = make_copy(g, h);
    } catch (...) {
      tgfx_graph_free(h);
      throw;
    }
    g.device_copy = dc;
  }
  return dc;
}

}  // namespace detail

// ------------------------------------------------------------------ event stream
void EventStream::validate() const {
  // event_stream.cpp:62-83
  const std::int64_t n = size();
  for (std::int64_t i = 0; i < n; ++i) {
    const TemporalEvent& e = events[static_cast<std::size_t>(i)];
    if (e.src < 0 || e.src >= num_nodes || e.dst < 0 || e.dst >= num_nodes)
      throw ValidationError("event " + std::to_string(i) + ": node id out of range");
    if (i > 0 && events[static_cast<std::size_t>(i - 1)].timestamp > e.timestamp)
      throw ValidationError("events not sorted by timestamp at index " + std::to_string(i));
  }
  if (!edge_features.empty() && (edge_features.rows() != static_cast<std::size_t>(n) ||
                                 edge_features.cols() != static_cast<std::size_t>(d_e)))
    throw ValidationError("edge feature matrix shape mismatch");
  if (!node_features.empty() && (node_features.rows() != static_cast<std::size_t>(num_nodes) ||
                                 node_features.cols() != static_cast<std::size_t>(d_v)))
    throw ValidationError("node feature matrix shape mismatch");
}

EventStream load_csv(const std::string& path, bool has_features) {
  tgfx_csv* c = nullptr;
  detail::check(tgfx_load_csv(path.c_str(), has_features ? 1 : 0, &c));
  struct Free {
    tgfx_csv* c;
    ~Free() { tgfx_csv_free(c); }
  } guard{c};
  std::int64_t n = 0, v = 0, d_e = 0;
  detail::check(tgfx_csv_info(c, &n, &v, &d_e));
  EventStream s;
  s.num_nodes = v;
  s.d_e = d_e;
  s.events.resize(static_cast<std::size_t>(n));
  if (d_e > 0) s.edge_features = Matrix(static_cast<std::size_t>(n), static_cast<std::size_t>(d_e));
  detail::check(tgfx_csv_export(c, reinterpret_cast<tgfx_event*>(s.events.data()),
                                d_e > 0 ? s.edge_features.data() : nullptr));
  return s;
}

// ------------------------------------------------------------------ T-CSR
tgfx_graph* TCsr::device() const { return detail::device_of(*this)->handle; }

void TCsr::validate() const {
  // tcsr.cpp:54-81: shape checks on the host, the O(m) scans on the device
  if (indptr.size() != static_cast<std::size_t>(num_nodes) + 1)
    throw ValidationError("indptr size mismatch");
  if (indptr.front() != 0 || indptr.back() != num_entries())
    throw ValidationError("indptr endpoints wrong");
  if (edge_ids.size() != neighbor_ids.size() || timestamps.size() != neighbor_ids.size())
    throw ValidationError("column arrays disagree in length");
  // the O(m) checks run on a fresh upload of the host columns, so an edit made after the
  // device copy was attached is always seen (the reference validates the vectors themselves)
  tgfx_graph* h = detail::upload(*this);
  const int rc = tgfx_graph_validate(h);
  if (rc != TGFX_OK) {
    const std::string msg = tgfx_last_error();
    tgfx_graph_free(h);
    detail::throw_status(rc, msg);
  }
  detail::attach(*this, h);  // the validated copy replaces any older one
}

namespace {

// A column of n entries for export_graph: on large columns every thread first faults in its
// share of the (reserved, not yet constructed) pages, so resize() -- which value-initialises,
// i.e. memsets -- runs over resident memory.  Faulting the ~9 GB of fresh pages of a
// GDELT-sized T-CSR on one thread took seconds; the element type is trivial, so writing the
// reserved bytes before resize() constructs the elements has no observable effect.
template <typename T>
void sized_column(std::vector<T>& v, std::size_t n) {
  static_assert(std::is_trivially_default_constructible_v<T>, "trivial column type");
  v.reserve(n);
  const std::int64_t bytes = static_cast<std::int64_t>(n * sizeof(T));
  if (bytes >= (std::int64_t(64) << 20)) {
    volatile char* p = reinterpret_cast<volatile char*>(v.data());
#pragma omp parallel for schedule(static)
    for (std::int64_t off = 0; off < bytes; off += 4096) p[off] = 0;
  }
  v.resize(n);
}

TCsr export_graph(tgfx_graph* h, bool reverse) {
  TCsr g;
  std::int64_t V = 0, E = 0, m = 0;
  int rev = 0;
  detail::check(tgfx_graph_info(h, &V, &E, &m, &rev));
  g.num_nodes = V;
  g.num_edges = E;
  g.reverse = reverse;
  sized_column(g.indptr, static_cast<std::size_t>(V) + 1);
  sized_column(g.neighbor_ids, static_cast<std::size_t>(m));
  sized_column(g.edge_ids, static_cast<std::size_t>(m));
  sized_column(g.timestamps, static_cast<std::size_t>(m));
  detail::check(tgfx_graph_export(h, g.indptr.data(), g.neighbor_ids.data(), g.edge_ids.data(),
                                  g.timestamps.data()));
  detail::attach(g, h);
  return g;
}

const tgfx_event* as_events(const EventStream& s) {
  return reinterpret_cast<const tgfx_event*>(s.events.data());
}

}  // namespace

TCsr build_sequential(const EventStream& stream, bool reverse) {
  tgfx_graph* h = nullptr;
  detail::check(tgfx_build_sequential(as_events(stream), stream.size(), stream.num_nodes,
                                      reverse ? 1 : 0, &h));
  try {
    return export_graph(h, reverse);
  } catch (...) {
    tgfx_graph_free(h);
    throw;
  }
}

TCsr build_parallel(const EventStream& stream, bool reverse, int num_threads) {
  tgfx_graph* h = nullptr;
  detail::check(tgfx_build_parallel(as_events(stream), stream.size(), stream.num_nodes,
                                    reverse ? 1 : 0, num_threads, &h));
  try {
    return export_graph(h, reverse);
  } catch (...) {
    tgfx_graph_free(h);
    throw;
  }
}

// ------------------------------------------------------------------ container
namespace {

constexpr char kMagic[4] = {'T', 'C', 'S', 'R'};
constexpr std::uint8_t kVersion = 1;
constexpr std::size_t kCrcChunk = std::size_t(1) << 30;  // zlib's crc32 takes 32-bit lengths

std::uint32_t crc_update(std::uint32_t crc, const void* p, std::size_t n) {
  uLong c = crc;
  const auto* b = static_cast<const Bytef*>(p);
  while (n) {
    const std::size_t k = std::min(n, kCrcChunk);
    c = crc32(c, b, static_cast<uInt>(k));
    b += k;
    n -= k;
  }
  return static_cast<std::uint32_t>(c);
}

struct Writer {
  std::ofstream out;
  std::uint32_t crc = static_cast<std::uint32_t>(crc32(0L, Z_NULL, 0));
  explicit Writer(const std::string& path) : out(path, std::ios::binary) {
    if (!out) throw ValidationError("cannot write '" + path + "'");
  }
  void put(const void* p, std::size_t n) {
    out.write(static_cast<const char*>(p), static_cast<std::streamsize>(n));
    crc = crc_update(crc, p, n);
  }
  template <class T>
  void val(T v) {
    put(&v, sizeof v);
  }
};

struct Reader {
  std::vector<char> buf;
  std::size_t pos = 0;
  void get(void* p, std::size_t n) {
    if (n > buf.size() - pos) throw FormatError("truncated container");
    std::memcpy(p, buf.data() + pos, n);
    pos += n;
  }
  template <class T>
  T val() {
    T v;
    get(&v, sizeof v);
    return v;
  }
  template <class T>
  void arr(std::vector<T>& v, std::uint64_t count) {
    if (count > (buf.size() - pos) / sizeof(T)) throw FormatError("truncated container");
    v.resize(static_cast<std::size_t>(count));
    get(v.data(), v.size() * sizeof(T));
  }
};

}  // namespace

void save_tcsr(const TCsr& g, const std::string& path) {
  // layout of tcsr.cpp:158-174: magic, u8 version, u8 reverse, u64 num_nodes, u64 num_edges,
  // u64 num_entries, indptr i64[], neighbors i64[], edge ids i64[], timestamps f64[], CRC-32
  Writer w(path);
  w.put(kMagic, sizeof kMagic);
  w.val<std::uint8_t>(kVersion);
  w.val<std::uint8_t>(g.reverse ? 1 : 0);
  w.val<std::uint64_t>(static_cast<std::uint64_t>(g.num_nodes));
  w.val<std::uint64_t>(static_cast<std::uint64_t>(g.num_edges));
  w.val<std::uint64_t>(static_cast<std::uint64_t>(g.num_entries()));
  w.put(g.indptr.data(), g.indptr.size() * sizeof(std::int64_t));
  w.put(g.neighbor_ids.data(), g.neighbor_ids.size() * sizeof(NodeId));
  w.put(g.edge_ids.data(), g.edge_ids.size() * sizeof(EdgeId));
  w.put(g.timestamps.data(), g.timestamps.size() * sizeof(Time));
  const std::uint32_t c = w.crc;
  w.out.write(reinterpret_cast<const char*>(&c), sizeof c);
  if (!w.out) throw ValidationError("write failed");
}

TCsr load_tcsr(const std::string& path) {
  // tcsr.cpp:176-197 + binary_io.hpp:83-100, with the checksum computed over the whole file
  // in 1 GiB pieces (the reference passes the full length as a 32-bit uInt, so containers
  // of 4 GiB and more fail its check)
  std::ifstream in(path, std::ios::binary | std::ios::ate);
  if (!in) throw ValidationError("cannot open '" + path + "'");
  const std::streamsize size = in.tellg();
  in.seekg(0);
  Reader r;
  r.buf.resize(static_cast<std::size_t>(size));
  in.read(r.buf.data(), size);
  if (!in) throw FormatError("read failed for '" + path + "'");
  if (r.buf.size() < 4) throw FormatError("container too small");
  std::uint32_t stored;
  std::memcpy(&stored, r.buf.data() + r.buf.size() - 4, 4);
  const std::uint32_t crc0 = static_cast<std::uint32_t>(crc32(0L, Z_NULL, 0));
  if (crc_update(crc0, r.buf.data(), r.buf.size() - 4) != stored)
    throw FormatError("checksum mismatch");
  r.buf.resize(r.buf.size() - 4);
  char magic[4];
  r.get(magic, sizeof magic);
  if (std::memcmp(magic, kMagic, sizeof kMagic) != 0) throw FormatError("bad magic");
  const auto version = r.val<std::uint8_t>();
  if (version != kVersion) throw FormatError("unsupported version " + std::to_string(version));
  TCsr g;
  g.reverse = r.val<std::uint8_t>() != 0;
  g.num_nodes = static_cast<NodeId>(r.val<std::uint64_t>());
  g.num_edges = static_cast<std::int64_t>(r.val<std::uint64_t>());
  const auto entries = r.val<std::uint64_t>();
  r.arr(g.indptr, static_cast<std::uint64_t>(g.num_nodes) + 1);
  r.arr(g.neighbor_ids, entries);
  r.arr(g.edge_ids, entries);
  r.arr(g.timestamps, entries);
  if (r.pos != r.buf.size()) throw FormatError("trailing bytes in container");
  g.validate();  // uploads (the device copy stays attached for sampling) and checks on device
  return g;
}

// ------------------------------------------------------------------ sampler
SampleStrategy parse_strategy(const std::string& name) {
  // sampler.cpp:34-38
  if (name == "recent") return SampleStrategy::recent;
  if (name == "random") return SampleStrategy::random;
  throw ValidationError("unknown sampling strategy '" + name + "'");
}

namespace {

static_assert(sizeof(NeighborEntry) == sizeof(tgfx_neighbor) &&
                  offsetof(NeighborEntry, neighbor) == offsetof(tgfx_neighbor, neighbor) &&
                  offsetof(NeighborEntry, edge) == offsetof(tgfx_neighbor, edge) &&
                  offsetof(NeighborEntry, timestamp) == offsetof(tgfx_neighbor, timestamp),
              "NeighborEntry must have the tgfx_neighbor record layout");

// One libtgfx batch call; stream of query i = stream_base + i (sampler.cpp:100-101).  The
// queries go up and the padded records come back through the thread's pinned staging; each
// NeighborSample's vector is then one copy of its run of records.
std::vector<NeighborSample> run_batch(const TCsr& g, const NodeId* nodes, const Time* times,
                                      std::int64_t q, std::int64_t k, SampleStrategy strategy,
                                      std::uint64_t seed, std::uint64_t stream_base) {
  const std::shared_ptr<detail::DeviceCopy> dcp = detail::device_of(g);
  const detail::DeviceCopy& dc = *dcp;
  // padded output width: no query can return more than the longest slice, so a huge k
  // (sample_recent(g, u, t, 1 << 30)) does not size the buffers; results are unchanged
  const std::int64_t kpad = k < 1 ? k : std::max<std::int64_t>(1, std::min(k, dc.max_degree));
  const std::size_t qs = static_cast<std::size_t>(std::max<std::int64_t>(q, 0));
  const std::size_t slots = qs * static_cast<std::size_t>(std::max<std::int64_t>(kpad, 1));
  char* in = detail::pinned_in().get(16 * qs);
  std::memcpy(in, nodes, 8 * qs);
  std::memcpy(in + 8 * qs, times, 8 * qs);
  // counts and records back to back: one device->host copy
  char* o = detail::pinned_out().get(8 * qs + 24 * slots);
  const auto* counts = reinterpret_cast<const std::int64_t*>(o);
  const auto* rec = reinterpret_cast<const NeighborEntry*>(o + 8 * qs);
  const int strat = strategy == SampleStrategy::recent ? TGFX_RECENT : TGFX_RANDOM;
  std::vector<NeighborSample> out(qs);
  const std::int64_t n = static_cast<std::int64_t>(qs);
  // Large batches: one thread runs the (synchronous) device call while the others allocate
  // the samples' vectors (kpad entries each, when that is small), then all copy the records
  // out.  The allocation, the slowest host step, hides under the device round trip.
  const bool par = n >= detail::kParMin;
  const bool pre = par && kpad <= 64;
  int rc = TGFX_OK;
#pragma omp parallel if (par)
  {
    const int t = omp_get_thread_num(), nt = omp_get_num_threads();
    if (t == 0) {
      rc = tgfx_sample_batch_records(dc.handle, reinterpret_cast<const std::int64_t*>(in),
                                     reinterpret_cast<const double*>(in + 8 * qs), q, kpad, strat,
                                     seed, stream_base, reinterpret_cast<std::int64_t*>(o),
                                     reinterpret_cast<tgfx_neighbor*>(o + 8 * qs));
    } else if (pre) {
      for (std::int64_t i = (t - 1) * n / (nt - 1); i < t * n / (nt - 1); ++i)
        out[static_cast<std::size_t>(i)].neighbors.reserve(static_cast<std::size_t>(kpad));
    }
#pragma omp barrier
    if (rc == TGFX_OK) {
#pragma omp for schedule(static)
      for (std::int64_t i = 0; i < n; ++i) {
        NeighborSample& s = out[static_cast<std::size_t>(i)];
        s.query_node = nodes[i];
        s.query_time = times[i];
        const NeighborEntry* r =
            rec + static_cast<std::size_t>(i) * static_cast<std::size_t>(kpad);
        s.neighbors.assign(r, r + counts[i]);
      }
    }
  }
  detail::check(rc);
  return out;
}

}  // namespace

NeighborSample sample_recent(const TCsr& g, NodeId u, Time t, std::int64_t k) {
  return std::move(run_batch(g, &u, &t, 1, k, SampleStrategy::recent, 0, 0)[0]);
}

NeighborSample sample_random(const TCsr& g, NodeId u, Time t, std::int64_t k,
                             std::uint64_t seed, std::uint64_t stream) {
  return std::move(run_batch(g, &u, &t, 1, k, SampleStrategy::random, seed, stream)[0]);
}

std::vector<NeighborSample> sample_batch(const TCsr& g, const std::vector<NodeId>& nodes,
                                         const std::vector<Time>& times, std::int64_t k,
                                         SampleStrategy strategy, std::uint64_t seed,
                                         int num_threads) {
  (void)num_threads;  // results are independent of it (sampler.cpp:91); the grid is the device's
  if (nodes.size() != times.size())
    throw ValidationError("node and time lists differ in length");  // sampler.cpp:88-90
  return run_batch(g, nodes.data(), times.data(), static_cast<std::int64_t>(nodes.size()), k,
                   strategy, seed, 0);
}

// ------------------------------------------------------------------ sequences
void SequenceBatch::validate() const {
  // sequence.cpp:13-46 (host-side consistency check of a batch; not on the hot path)
  const auto total = static_cast<std::size_t>(batch * l);
  if (node_index.size() != total || edge_index.size() != total ||
      time_delta.rows() != static_cast<std::size_t>(batch) ||
      time_delta.cols() != static_cast<std::size_t>(l) ||
      valid_len.size() != static_cast<std::size_t>(batch) ||
      target_row.size() != static_cast<std::size_t>(batch))
    throw ValidationError("sequence batch shape mismatch");
  for (std::int64_t b = 0; b < batch; ++b) {
    const std::int64_t len = valid_len[static_cast<std::size_t>(b)];
    if (len < 1 || len > l) throw ValidationError("valid_len out of range");
    if (target_row[static_cast<std::size_t>(b)] != len - 1)
      throw ValidationError("target_row must be valid_len-1");
    const std::size_t row = static_cast<std::size_t>(b * l);
    for (std::int64_t j = 0; j < l; ++j) {
      const bool padding = j >= len;
      const double dt = time_delta.at(static_cast<std::size_t>(b), static_cast<std::size_t>(j));
      if (padding != (node_index[row + static_cast<std::size_t>(j)] == 0))
        throw ValidationError("padding does not match valid_len");
      if (padding && (edge_index[row + static_cast<std::size_t>(j)] != 0 || dt != 0.0))
        throw ValidationError("padding positions must be zero");
      if (dt < 0.0) throw ValidationError("negative time delta");
    }
    if (time_delta.at(static_cast<std::size_t>(b),
                      static_cast<std::size_t>(target_row[static_cast<std::size_t>(b)])) != 0.0)
      throw ValidationError("query position must have zero time delta");
    for (std::int64_t j = 1; j + 1 < len; ++j)
      if (time_delta.at(static_cast<std::size_t>(b), static_cast<std::size_t>(j - 1)) <
          time_delta.at(static_cast<std::size_t>(b), static_cast<std::size_t>(j)))
        throw ValidationError("neighbor time deltas must be non-increasing");
  }
}

MaskKind parse_mask_kind(const std::string& name) {
  // sequence.cpp:48-53
  if (name == "causal") return MaskKind::causal;
  if (name == "tgat") return MaskKind::tgat;
  if (name == "self_loop") return MaskKind::self_loop;
  throw ValidationError("unknown mask kind '" + name + "'");
}

namespace {

// The SequenceBatch columns from the pinned staging the device wrote them to: assign() copies
// without the value-initialisation a resize() would first write.
SequenceBatch unpack_sequences(const char* o, std::int64_t q, std::int64_t l,
                               std::size_t o_e, std::size_t o_d, std::size_t o_v,
                               std::size_t o_r) {
  SequenceBatch out;
  out.batch = q;
  out.l = l;
  const std::size_t ql = static_cast<std::size_t>(q) * static_cast<std::size_t>(l);
  const auto* ni = reinterpret_cast<const std::int64_t*>(o);
  const auto* ei = reinterpret_cast<const std::int64_t*>(o + o_e);
  const auto* vl = reinterpret_cast<const std::int64_t*>(o + o_v);
  const auto* tr = reinterpret_cast<const std::int64_t*>(o + o_r);
  // the three [q, l] columns are copied by three threads once they are large
#pragma omp parallel sections if (ql >= 8192)
  {
#pragma omp section
    out.node_index.assign(ni, ni + ql);
#pragma omp section
    out.edge_index.assign(ei, ei + ql);
#pragma omp section
    out.time_delta = Matrix(static_cast<std::size_t>(q), static_cast<std::size_t>(l),
                            reinterpret_cast<const double*>(o + o_d));
  }
  out.valid_len.assign(vl, vl + q);
  out.target_row.assign(tr, tr + q);
  return out;
}

}  // namespace

SequenceBatch build_sequence_batch(const std::vector<NeighborSample>& samples, std::int64_t l,
                                   std::int64_t self_edge_index) {
  if (l < 2) throw ValidationError("sequence length must be at least 2");  // sequence.cpp:57
  const std::int64_t q = static_cast<std::int64_t>(samples.size());
  // sequence.cpp:66-70 reads only a sample's last min(total, l - 1) entries: only those are
  // packed (count kb, skip 0), which leaves the rows unchanged
  const std::size_t tail = static_cast<std::size_t>(l - 1);
  std::size_t kpad = 1;
  for (const NeighborSample& s : samples) kpad = std::max(kpad, std::min(tail, s.neighbors.size()));
  const std::size_t qs = static_cast<std::size_t>(q), ql = qs * static_cast<std::size_t>(l);
  // inputs and outputs each back to back (one copy per direction)
  const std::size_t i_e = 8 * qs, i_qn = i_e + 24 * qs * kpad,
                    i_qt = i_qn + 8 * qs;
  char* in = detail::pinned_in().get(i_qt + 8 * qs);
  auto* cnt = reinterpret_cast<std::int64_t*>(in);
  auto* rec = reinterpret_cast<NeighborEntry*>(in + i_e);
  auto* qn = reinterpret_cast<std::int64_t*>(in + i_qn);
  auto* qt = reinterpret_cast<double*>(in + i_qt);
#pragma omp parallel for schedule(static) if (q >= detail::kParMin)
  for (std::int64_t b = 0; b < q; ++b) {
    const NeighborSample& s = samples[static_cast<std::size_t>(b)];
    const std::size_t total = s.neighbors.size(), kb = std::min(total, tail);
    cnt[b] = static_cast<std::int64_t>(kb);
    qn[b] = s.query_node;
    qt[b] = s.query_time;
    if (kb)
      std::memcpy(rec + static_cast<std::size_t>(b) * kpad, s.neighbors.data() + (total - kb),
                  kb * sizeof(NeighborEntry));
  }
  const std::size_t o_e = 8 * ql, o_d = o_e + 8 * ql, o_v = o_d + 8 * ql, o_r = o_v + 8 * qs;
  char* o = detail::pinned_out().get(o_r + 8 * qs);
  detail::check(tgfx_assemble_records(
      q, static_cast<std::int64_t>(kpad), cnt, reinterpret_cast<const tgfx_neighbor*>(rec), qn,
      qt, l, self_edge_index, reinterpret_cast<std::int64_t*>(o),
      reinterpret_cast<std::int64_t*>(o + o_e), reinterpret_cast<double*>(o + o_d),
      reinterpret_cast<std::int64_t*>(o + o_v), reinterpret_cast<std::int64_t*>(o + o_r)));
  return unpack_sequences(o, q, l, o_e, o_d, o_v, o_r);
}

SequenceBatch sample_sequence_batch(const TCsr& g, const std::vector<NodeId>& nodes,
                                    const std::vector<Time>& times, std::int64_t k,
                                    SampleStrategy strategy, std::uint64_t seed, std::int64_t l,
                                    std::int64_t self_edge_index, int num_threads) {
  (void)num_threads;
  if (nodes.size() != times.size())
    throw ValidationError("node and time lists differ in length");  // sampler.cpp:88-90
  const std::shared_ptr<detail::DeviceCopy> dc = detail::device_of(g);
  const std::int64_t q = static_cast<std::int64_t>(nodes.size());
  const std::size_t qs = nodes.size();
  char* in = detail::pinned_in().get(16 * qs);
  std::memcpy(in, nodes.data(), 8 * qs);
  std::memcpy(in + 8 * qs, times.data(), 8 * qs);
  const std::size_t ql = qs * static_cast<std::size_t>(l > 0 ? l : 0);
  const std::size_t o_e = 8 * ql, o_d = o_e + 8 * ql, o_v = o_d + 8 * ql, o_r = o_v + 8 * qs;
  char* o = detail::pinned_out().get(o_r + 8 * qs);
  detail::check(tgfx_sample_sequence_batch(
      dc->handle, reinterpret_cast<const std::int64_t*>(in),
      reinterpret_cast<const double*>(in + 8 * qs), q, k,
      strategy == SampleStrategy::recent ? TGFX_RECENT : TGFX_RANDOM, seed, 0, l,
      self_edge_index, reinterpret_cast<std::int64_t*>(o),
      reinterpret_cast<std::int64_t*>(o + o_e), reinterpret_cast<double*>(o + o_d),
      reinterpret_cast<std::int64_t*>(o + o_v), reinterpret_cast<std::int64_t*>(o + o_r)));
  return unpack_sequences(o, q, l > 0 ? l : 0, o_e, o_d, o_v, o_r);
}

SequenceBatch build_sequence(const NeighborSample& sample, std::int64_t l,
                             std::int64_t self_edge_index) {
  return build_sequence_batch(std::vector<NeighborSample>{sample}, l, self_edge_index);
}

Matrix build_mask(const SequenceBatch& batch, MaskKind kind) {
  Matrix mask(static_cast<std::size_t>(batch.batch * batch.l), static_cast<std::size_t>(batch.l));
  const int code = kind == MaskKind::causal ? TGFX_MASK_CAUSAL
                   : kind == MaskKind::tgat ? TGFX_MASK_TGAT
                                            : TGFX_MASK_SELF_LOOP;
  detail::check(tgfx_build_mask(batch.batch, batch.l, batch.valid_len.data(),
                                batch.target_row.data(), code, mask.data()));
  return mask;
}

// ------------------------------------------------------------------ synthetic
EventStream make_random_stream(std::int64_t num_edges, NodeId num_nodes, std::uint64_t seed,
                               double zipf_exponent) {
  EventStream s;
  s.num_nodes = num_nodes;
  s.events.resize(static_cast<std::size_t>(std::max<std::int64_t>(num_edges, 0)));
  detail::check(tgfx_make_random_stream(num_edges, num_nodes, seed, zipf_exponent,
                                        reinterpret_cast<tgfx_event*>(s.events.data())));
  return s;
}

}  // namespace tgf
