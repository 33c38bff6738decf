// ref_harness.cpp -- extern "C" harness around the UNMODIFIED reference hot path.
//
// TEST INFRASTRUCTURE / CPU BASELINE ONLY.  Compiled by oracle/Makefile together with the
// reference's own sources (/root/reference/proj/src/{event_stream,tcsr,sampler,sequence,
// synthetic}.cpp, never copied into this repo) into oracle/_ref/libtgf_ref.so.  It lets
// Python drive the reference to (1) generate golden vectors (tests/golden/gen_golden.py)
// and (2) time the reference CPU path (bench.py cpu_baseline leg and --impl reference).
// Timings are taken inside C++ around the reference calls only (no marshalling).
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "tgformer/attention.hpp"
#include "tgformer/event_stream.hpp"
#include "tgformer/sampler.hpp"
#include "tgformer/sequence.hpp"
#include "tgformer/synthetic.hpp"
#include "tgformer/tcsr.hpp"
#include "tgformer/training.hpp"

namespace {
thread_local std::string g_err;
using Clock = std::chrono::steady_clock;
double secs(Clock::time_point a) { return std::chrono::duration<double>(Clock::now() - a).count(); }

int fail(const std::exception& e) {
  g_err = e.what();
  if (dynamic_cast<const tgf::ValidationError*>(&e)) return 1;
  if (dynamic_cast<const tgf::FormatError*>(&e)) return 2;
  if (dynamic_cast<const tgf::ParseError*>(&e)) return 6;
  return 3;
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// tgf::make_random_stream (synthetic.cpp:12-43) -> 32-byte events.
int ref_make_random_stream(int64_t e, int64_t v, uint64_t seed, double zipf, void* out) {
  try {
    tgf::EventStream s = tgf::make_random_stream(e, v, seed, zipf);
    std::memcpy(out, s.events.data(), sizeof(tgf::TemporalEvent) * s.events.size());
    return 0;
  } catch (const std::exception& ex) {
    return fail(ex);
  }
}

void* ref_stream_create(const void* events, int64_t n, int64_t num_nodes) {
  auto* s = new tgf::EventStream();
  s->num_nodes = num_nodes;
  s->events.resize(static_cast<size_t>(n));
  if (n > 0) std::memcpy(s->events.data(), events, sizeof(tgf::TemporalEvent) * n);
  return s;
}
void ref_stream_free(void* s) { delete static_cast<tgf::EventStream*>(s); }

// threads <= 0 -> build_sequential, else build_parallel(threads).  *secs_out = build time.
int ref_build(void* stream, int reverse, int threads, void** graph_out, double* secs_out) {
  try {
    auto* s = static_cast<tgf::EventStream*>(stream);
    auto t0 = Clock::now();
    tgf::TCsr g = threads <= 0 ? tgf::build_sequential(*s, reverse != 0)
                               : tgf::build_parallel(*s, reverse != 0, threads);
    if (secs_out) *secs_out = secs(t0);
    *graph_out = new tgf::TCsr(std::move(g));
    return 0;
  } catch (const std::exception& ex) {
    return fail(ex);
  }
}

// build_parallel with an explicit (possibly invalid) thread count, for error parity.
int ref_build_parallel_raw(void* stream, int reverse, int threads, void** graph_out) {
  try {
    auto* s = static_cast<tgf::EventStream*>(stream);
    *graph_out = new tgf::TCsr(tgf::build_parallel(*s, reverse != 0, threads));
    return 0;
  } catch (const std::exception& ex) {
    return fail(ex);
  }
}

void ref_graph_free(void* g) { delete static_cast<tgf::TCsr*>(g); }

// a tgf::TCsr assembled from caller columns (for TCsr::validate texts on corrupted graphs)
void* ref_graph_from_columns(int64_t num_nodes, int64_t num_edges, int reverse, int64_t m,
                             const int64_t* indptr, const int64_t* nbr, const int64_t* eid,
                             const double* ts) {
  auto* g = new tgf::TCsr();
  g->num_nodes = num_nodes;
  g->num_edges = num_edges;
  g->reverse = reverse != 0;
  g->indptr.assign(indptr, indptr + num_nodes + 1);
  g->neighbor_ids.assign(nbr, nbr + m);
  g->edge_ids.assign(eid, eid + m);
  g->timestamps.assign(ts, ts + m);
  return g;
}

void ref_graph_info(void* gp, int64_t* out4) {
  auto* g = static_cast<tgf::TCsr*>(gp);
  out4[0] = g->num_nodes;
  out4[1] = g->num_edges;
  out4[2] = g->num_entries();
  out4[3] = g->reverse ? 1 : 0;
}

void ref_graph_export(void* gp, int64_t* indptr, int64_t* nbr, int64_t* eid, double* ts) {
  auto* g = static_cast<tgf::TCsr*>(gp);
  std::memcpy(indptr, g->indptr.data(), sizeof(int64_t) * g->indptr.size());
  std::memcpy(nbr, g->neighbor_ids.data(), sizeof(int64_t) * g->neighbor_ids.size());
  std::memcpy(eid, g->edge_ids.data(), sizeof(int64_t) * g->edge_ids.size());
  std::memcpy(ts, g->timestamps.data(), sizeof(double) * g->timestamps.size());
}

int ref_graph_validate(void* gp) {
  try {
    static_cast<tgf::TCsr*>(gp)->validate();
    return 0;
  } catch (const std::exception& ex) {
    return fail(ex);
  }
}

// sample_batch (sampler.cpp:84-104) -> padded [q, k] entries + counts.
int ref_sample_batch(void* gp, const int64_t* nodes, const double* times, int64_t q, int64_t k,
                     int strategy, uint64_t seed, int threads, int64_t* counts, int64_t* nbr,
                     int64_t* eid, double* ts, double* secs_out) {
  try {
    auto* g = static_cast<tgf::TCsr*>(gp);
    std::vector<tgf::NodeId> vn(nodes, nodes + q);
    std::vector<tgf::Time> vt(times, times + q);
    auto t0 = Clock::now();
    auto out = tgf::sample_batch(*g, vn, vt, k,
                                 strategy == 0 ? tgf::SampleStrategy::recent
                                               : tgf::SampleStrategy::random,
                                 seed, threads);
    if (secs_out) *secs_out = secs(t0);
    const int64_t kp = std::max<int64_t>(k, 1);
    for (int64_t i = 0; i < q; ++i) {
      const auto& s = out[i].neighbors;
      counts[i] = static_cast<int64_t>(s.size());
      for (int64_t j = 0; j < kp; ++j) {
        const bool have = j < static_cast<int64_t>(s.size());
        nbr[i * kp + j] = have ? s[j].neighbor : 0;
        eid[i * kp + j] = have ? s[j].edge : 0;
        ts[i * kp + j] = have ? s[j].timestamp : 0.0;
      }
    }
    return 0;
  } catch (const std::exception& ex) {
    return fail(ex);
  }
}

// sample_random with an explicit stream (sampler.cpp:54-82), for hop-keyed compositions.
int ref_sample_random(void* gp, int64_t u, double t, int64_t k, uint64_t seed, uint64_t stream,
                      int64_t* count, int64_t* nbr, int64_t* eid, double* ts) {
  try {
    auto* g = static_cast<tgf::TCsr*>(gp);
    auto s = tgf::sample_random(*g, u, t, k, seed, stream);
    *count = static_cast<int64_t>(s.neighbors.size());
    for (size_t j = 0; j < s.neighbors.size(); ++j) {
      nbr[j] = s.neighbors[j].neighbor;
      eid[j] = s.neighbors[j].edge;
      ts[j] = s.neighbors[j].timestamp;
    }
    return 0;
  } catch (const std::exception& ex) {
    return fail(ex);
  }
}

// sample_batch + build_sequence_batch, the forward_concat pair (training.cpp:211-214).
// Outputs in reference types: node/edge index int64 [q*l], time_delta double [q*l],
// valid_len int64 [q].  *secs_out = time of the two reference calls.
int ref_sample_assemble(void* gp, const int64_t* nodes, const double* times, int64_t q,
                        int64_t k, int strategy, uint64_t seed, int threads, int64_t l,
                        int64_t self_edge_index, int64_t* node_index, int64_t* edge_index,
                        double* dt, int64_t* valid_len, double* secs_out) {
  try {
    auto* g = static_cast<tgf::TCsr*>(gp);
    std::vector<tgf::NodeId> vn(nodes, nodes + q);
    std::vector<tgf::Time> vt(times, times + q);
    auto t0 = Clock::now();
    auto samples = tgf::sample_batch(*g, vn, vt, k,
                                     strategy == 0 ? tgf::SampleStrategy::recent
                                                   : tgf::SampleStrategy::random,
                                     seed, threads);
    tgf::SequenceBatch sb = tgf::build_sequence_batch(samples, l, self_edge_index);
    if (secs_out) *secs_out = secs(t0);
    if (node_index) std::memcpy(node_index, sb.node_index.data(), sizeof(int64_t) * q * l);
    if (edge_index) std::memcpy(edge_index, sb.edge_index.data(), sizeof(int64_t) * q * l);
    if (dt) {
      for (int64_t b = 0; b < q; ++b)
        for (int64_t j = 0; j < l; ++j) dt[b * l + j] = sb.time_delta.at(b, j);
    }
    if (valid_len) std::memcpy(valid_len, sb.valid_len.data(), sizeof(int64_t) * q);
    return 0;
  } catch (const std::exception& ex) {
    return fail(ex);
  }
}

// build_sequence_batch over padded samples [q, kpad] (sequence.cpp:55-86).
int ref_build_sequence_batch(int64_t q, int64_t kpad, const int64_t* counts, const int64_t* nbr,
                             const int64_t* eid, const double* ts, const int64_t* qnodes,
                             const double* qtimes, int64_t l, int64_t self_edge_index,
                             int64_t* node_index, int64_t* edge_index, double* dt,
                             int64_t* valid_len, int64_t* target_row) {
  try {
    std::vector<tgf::NeighborSample> samples(static_cast<size_t>(q));
    for (int64_t b = 0; b < q; ++b) {
      samples[b].query_node = qnodes[b];
      samples[b].query_time = qtimes[b];
      for (int64_t j = 0; j < counts[b]; ++j)
        samples[b].neighbors.push_back({nbr[b * kpad + j], eid[b * kpad + j], ts[b * kpad + j]});
    }
    tgf::SequenceBatch sb = tgf::build_sequence_batch(samples, l, self_edge_index);
    std::memcpy(node_index, sb.node_index.data(), sizeof(int64_t) * q * l);
    std::memcpy(edge_index, sb.edge_index.data(), sizeof(int64_t) * q * l);
    for (int64_t b = 0; b < q; ++b)
      for (int64_t j = 0; j < l; ++j) dt[b * l + j] = sb.time_delta.at(b, j);
    std::memcpy(valid_len, sb.valid_len.data(), sizeof(int64_t) * q);
    std::memcpy(target_row, sb.target_row.data(), sizeof(int64_t) * q);
    return 0;
  } catch (const std::exception& ex) {
    return fail(ex);
  }
}

// build_mask (sequence.cpp:93-111) over (valid_len, target_row).
int ref_build_mask(int64_t q, int64_t l, const int64_t* valid_len, const int64_t* target_row,
                   int kind, double* mask) {
  try {
    tgf::SequenceBatch sb;
    sb.batch = q;
    sb.l = l;
    sb.valid_len.assign(valid_len, valid_len + q);
    sb.target_row.assign(target_row, target_row + q);
    tgf::Matrix m = tgf::build_mask(
        sb, kind == 0 ? tgf::MaskKind::causal
                      : (kind == 1 ? tgf::MaskKind::tgat : tgf::MaskKind::self_loop));
    for (int64_t r = 0; r < q * l; ++r)
      for (int64_t c = 0; c < l; ++c) mask[r * l + c] = m.at(r, c);
    return 0;
  } catch (const std::exception& ex) {
    return fail(ex);
  }
}

// tgf::assemble_inputs (attention.cpp:414-451) on a SequenceBatch given as int64/f64 arrays
// and tables given as row-major f64 arrays; concat = 0 sum, 1 concat.  z: [q*l, d].
int ref_assemble_inputs(int64_t q, int64_t l, const int64_t* node_index, const int64_t* edge_index,
                        const double* time_delta, const int64_t* valid_len,
                        const double* node_table, int64_t node_rows, const double* edge_table,
                        int64_t edge_rows, const double* omega, const double* phi, int64_t d_v,
                        int64_t d_e, int64_t d_t, int concat, double* z) {
  try {
    tgf::ModelParams p;
    p.config.d_v = d_v;
    p.config.d_e = d_e;
    p.config.d_t = d_t;
    p.config.d_model = concat ? d_v + d_e + d_t : d_t;
    p.config.combine = concat ? tgf::CombineMode::concat : tgf::CombineMode::sum;
    p.node_table = tgf::Matrix(static_cast<size_t>(node_rows), static_cast<size_t>(d_v));
    p.edge_table = tgf::Matrix(static_cast<size_t>(edge_rows), static_cast<size_t>(d_e));
    p.omega = tgf::Matrix(1, static_cast<size_t>(d_t));
    p.phi = tgf::Matrix(1, static_cast<size_t>(d_t));
    std::memcpy(p.node_table.data(), node_table, sizeof(double) * node_rows * d_v);
    std::memcpy(p.edge_table.data(), edge_table, sizeof(double) * edge_rows * d_e);
    std::memcpy(p.omega.data(), omega, sizeof(double) * d_t);
    std::memcpy(p.phi.data(), phi, sizeof(double) * d_t);
    tgf::SequenceBatch b;
    b.batch = q;
    b.l = l;
    b.node_index.assign(node_index, node_index + q * l);
    b.edge_index.assign(edge_index, edge_index + q * l);
    b.time_delta = tgf::Matrix(static_cast<size_t>(q), static_cast<size_t>(l));
    std::memcpy(b.time_delta.data(), time_delta, sizeof(double) * q * l);
    b.valid_len.assign(valid_len, valid_len + q);
    b.target_row.resize(static_cast<size_t>(q));
    for (int64_t i = 0; i < q; ++i) b.target_row[static_cast<size_t>(i)] = valid_len[i] - 1;
    const tgf::Matrix out = tgf::assemble_inputs(p, b);
    std::memcpy(z, out.data(), sizeof(double) * out.size());
    return 0;
  } catch (const std::exception& ex) {
    return fail(ex);
  }
}

// tgf::load_csv (event_stream.cpp:85-154): two calls -- with events == nullptr it parses
// and reports the shape (cached); then the same path again copies events / features out.
int ref_load_csv(const char* path, int has_features, int64_t* n, int64_t* num_nodes,
                 int64_t* d_e, void* events, double* features) {
  static std::string cached_path;
  static tgf::EventStream cached;
  try {
    if (!events || cached_path != path) {
      cached = tgf::load_csv(path, has_features != 0);
      cached_path = path;
    }
    *n = cached.size();
    *num_nodes = cached.num_nodes;
    *d_e = cached.d_e;
    if (events) {
      std::memcpy(events, cached.events.data(), sizeof(tgf::TemporalEvent) * cached.events.size());
      if (features && cached.d_e > 0)
        std::memcpy(features, cached.edge_features.data(),
                    sizeof(double) * cached.edge_features.size());
      cached_path.clear();
    }
    return 0;
  } catch (const std::exception& ex) {
    cached_path.clear();
    return fail(ex);
  }
}

// tgf::make_batches (training.cpp:157-182), split into min(workers, b) shards as train_epoch
// does (:425-440), each shard's queries laid out as forward_concat builds them (:193-209):
// every sample_batch call of one epoch, concatenated in call order.
int ref_train_queries(void* stream, int64_t batch_size, int64_t npp, int64_t workers,
                      int64_t num_nodes, uint64_t seed, int64_t* nodes, double* times,
                      int64_t* total) {
  try {
    const auto& st = *static_cast<const tgf::EventStream*>(stream);
    const std::vector<tgf::LinkBatch> batches =
        tgf::make_batches(st, batch_size, npp, num_nodes, seed);
    int64_t o = 0;
    for (const tgf::LinkBatch& batch : batches) {
      const auto b = static_cast<int64_t>(batch.src.size());
      const int64_t m = std::min<int64_t>(workers, b);
      for (int64_t shard = 0; shard < m; ++shard) {
        const int64_t lo = shard * b / m, hi = (shard + 1) * b / m;
        for (int64_t i = lo; i < hi; ++i) {
          nodes[o] = batch.src[i];
          times[o++] = batch.times[i];
        }
        for (int64_t i = lo; i < hi; ++i) {
          nodes[o] = batch.dst[i];
          times[o++] = batch.times[i];
        }
        for (int64_t j = lo * npp; j < hi * npp; ++j) {
          nodes[o] = batch.neg[j];
          times[o++] = batch.times[j / npp];
        }
      }
    }
    *total = o;
    return 0;
  } catch (const std::exception& ex) {
    return fail(ex);
  }
}

// tgf::save_tcsr / tgf::load_tcsr (tcsr.cpp:153-197) -- container interop checks
int ref_save_tcsr(void* gp, const char* path) {
  try {
    tgf::save_tcsr(*static_cast<tgf::TCsr*>(gp), path);
    return 0;
  } catch (const std::exception& ex) {
    return fail(ex);
  }
}
int ref_load_tcsr(const char* path, void** out) {
  try {
    *out = new tgf::TCsr(tgf::load_tcsr(path));
    return 0;
  } catch (const std::exception& ex) {
    return fail(ex);
  }
}

}  // extern "C"
