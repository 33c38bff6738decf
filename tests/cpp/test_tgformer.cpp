// C++ host API (include/tgfx/tgformer.hpp) on the GPU: known answers pinned by the reference's
// unit tests (proj/tests/test_tcsr.cpp:50-107, test_sampler.cpp:32-87,
// test_sequence.cpp:19-31) plus API-level properties (batch == per-query, container
// round trip, device copy reuse, error types).  Needs a CUDA device.
#include <cmath>
#include <cstdio>
#include <filesystem>
#include <thread>
#include <vector>

#include "doctest.h"
#include "tgformer/sampler.hpp"
#include "tgformer/sequence.hpp"
#include "tgformer/synthetic.hpp"
#include "tgformer/tcsr.hpp"

namespace {

tgf::EventStream tiny() {
  // three events, listed in time order (t = 3, 4, 5) with out-of-order edge ids
  tgf::EventStream s;
  s.num_nodes = 3;
  s.events = {{1, 0, 2, 3.0}, {2, 1, 2, 4.0}, {0, 0, 1, 5.0}};
  return s;
}

}  // namespace

TEST_CASE("tiny build: indptr and slice order, both directions") {
  const tgf::TCsr f = tgf::build_sequential(tiny(), false);
  CHECK(f.indptr == std::vector<std::int64_t>{0, 2, 3, 3});
  CHECK(f.neighbor_ids == std::vector<tgf::NodeId>{2, 1, 2});
  CHECK(f.timestamps == std::vector<double>{3.0, 5.0, 4.0});
  const tgf::TCsr r = tgf::build_parallel(tiny(), true, 8);
  CHECK(r.indptr == std::vector<std::int64_t>{0, 2, 4, 6});
  CHECK(r.edge_ids == std::vector<tgf::EdgeId>{1, 0, 2, 0, 1, 2});
  r.validate();
}

TEST_CASE("builder errors carry the reference's types and messages") {
  tgf::EventStream s = tiny();
  s.events.push_back({3, 0, 7, 6.0});
  try {
    (void)tgf::build_sequential(s, true);
    CHECK(false);
  } catch (const tgf::ValidationError& e) {
    CHECK(std::string(e.what()) == "event 3 endpoint out of range");
  }
  CHECK_THROWS_AS(tgf::build_parallel(tiny(), true, 0), tgf::ValidationError);
}

TEST_CASE("sequential, parallel and unsorted-input builds agree") {
  tgf::EventStream s = tgf::make_random_stream(30000, 500, 7);
  const tgf::TCsr a = tgf::build_sequential(s, true);
  const tgf::TCsr b = tgf::build_parallel(s, true, 4);
  CHECK(a.indptr == b.indptr);
  CHECK(a.neighbor_ids == b.neighbor_ids);
  CHECK(a.edge_ids == b.edge_ids);
  CHECK(a.timestamps == b.timestamps);
  // reversed stream order: same T-CSR (the builder sorts slices by (t, eid))
  std::reverse(s.events.begin(), s.events.end());
  const tgf::TCsr c = tgf::build_parallel(s, true, 4);
  CHECK(a.neighbor_ids == c.neighbor_ids);
  CHECK(a.edge_ids == c.edge_ids);
}

TEST_CASE("recent sampling: strict before t, k most recent ascending") {
  const tgf::TCsr g = tgf::build_sequential(tiny(), false);
  const tgf::NeighborSample mid = tgf::sample_recent(g, 0, 4.0, 5);
  REQUIRE(mid.neighbors.size() == 1);
  CHECK(mid.neighbors[0].neighbor == 2);
  CHECK(tgf::sample_recent(g, 0, 3.0, 5).neighbors.empty());
  const tgf::NeighborSample all = tgf::sample_recent(g, 0, 99.0, 1 << 30);
  REQUIRE(all.neighbors.size() == 2);
  CHECK(all.neighbors[1].timestamp == 5.0);
  CHECK(tgf::sample_recent(g, 0, std::nan(""), 5).neighbors.empty());
  CHECK_THROWS_AS(tgf::sample_recent(g, 3, 1.0, 1), tgf::ValidationError);
  CHECK_THROWS_AS(tgf::sample_recent(g, 0, 1.0, 0), tgf::ValidationError);
}

TEST_CASE("batch sampling equals per-query sampling (stream = query index)") {
  const tgf::EventStream s = tgf::make_random_stream(20000, 300, 34);
  const tgf::TCsr g = tgf::build_parallel(s, true, 2);
  std::vector<tgf::NodeId> nodes;
  std::vector<tgf::Time> times;
  tgf::CounterRng rng(77, 0);
  for (int i = 0; i < 300; ++i) {
    nodes.push_back(static_cast<tgf::NodeId>(rng.next_below(300)));
    times.push_back(rng.next_uniform(0.0, 10000.0));
  }
  for (auto strat : {tgf::SampleStrategy::recent, tgf::SampleStrategy::random}) {
    const auto batch = tgf::sample_batch(g, nodes, times, 12, strat, 9);
    REQUIRE(batch.size() == nodes.size());
    for (std::size_t i = 0; i < nodes.size(); ++i) {
      const auto one = strat == tgf::SampleStrategy::recent
                           ? tgf::sample_recent(g, nodes[i], times[i], 12)
                           : tgf::sample_random(g, nodes[i], times[i], 12, 9, i);
      REQUIRE(one.neighbors.size() == batch[i].neighbors.size());
      for (std::size_t j = 0; j < one.neighbors.size(); ++j) {
        CHECK(one.neighbors[j].edge == batch[i].neighbors[j].edge);
        CHECK(one.neighbors[j].timestamp < times[i]);
      }
    }
  }
  CHECK_THROWS_AS(tgf::sample_batch(g, {0, 1}, {1.0}, 3, tgf::SampleStrategy::recent, 0),
                  tgf::ValidationError);
}

TEST_CASE("suffix infilling known answer") {
  // test_sequence.cpp:19-31: neighbors (nbr 1,2,5 / eid 0,1,2 / t 2,4,7) of node 7 at t = 10
  tgf::NeighborSample s{7, 10.0, {{1, 0, 2.0}, {2, 1, 4.0}, {5, 2, 7.0}}};
  const tgf::SequenceBatch b = tgf::build_sequence(s, 8, 100);
  b.validate();
  CHECK(b.node_index == std::vector<std::int64_t>{2, 3, 6, 8, 0, 0, 0, 0});
  CHECK(b.edge_index == std::vector<std::int64_t>{1, 2, 3, 100, 0, 0, 0, 0});
  CHECK(b.time_delta.at(0, 0) == 8.0);
  CHECK(b.time_delta.at(0, 2) == 3.0);
  CHECK(b.valid_len[0] == 4);
  CHECK(b.target_row[0] == 3);
  const tgf::Matrix m = tgf::build_mask(b, tgf::MaskKind::causal);
  CHECK(m.rows() == 8);
  CHECK(m.at(2, 2) == 0.0);
  CHECK(std::isinf(m.at(2, 3)));
  CHECK_THROWS_AS(tgf::build_sequence(s, 1, 100), tgf::ValidationError);
  CHECK_THROWS_AS(tgf::parse_mask_kind("bogus"), tgf::ValidationError);
}

TEST_CASE("container round trip and corruption") {
  const tgf::TCsr g = tgf::build_parallel(tgf::make_random_stream(5000, 80, 3), true, 1);
  const std::string path =
      (std::filesystem::temp_directory_path() / "tgfx_cpp_test.tcsr").string();
  tgf::save_tcsr(g, path);
  const tgf::TCsr back = tgf::load_tcsr(path);
  CHECK(back.indptr == g.indptr);
  CHECK(back.timestamps == g.timestamps);
  CHECK(tgf::sample_recent(back, 0, 1e9, 4).neighbors.size() == 4);
  std::filesystem::resize_file(path, 12);
  CHECK_THROWS_AS(tgf::load_tcsr(path), tgf::FormatError);
  std::remove(path.c_str());
}

TEST_CASE("hand-assembled and edited TCsr re-upload") {
  tgf::TCsr g = tgf::build_sequential(tiny(), false);
  tgf::TCsr h = g;  // copy: content-identical, may share the device copy
  CHECK(tgf::sample_recent(h, 0, 99.0, 5).neighbors.size() == 2);
  h.timestamps[0] = 4.5;  // edited columns: the next call must see the new values
  h.timestamps[1] = 4.6;
  const auto s = tgf::sample_recent(h, 0, 4.55, 5);
  REQUIRE(s.neighbors.size() == 1);
  CHECK(s.neighbors[0].timestamp == 4.5);
  CHECK(tgf::sample_recent(g, 0, 4.55, 5).neighbors.size() == 1);  // original untouched: t=3
}

TEST_CASE("sample_sequence_batch equals build_sequence_batch(sample_batch(...))") {
  const tgf::EventStream st = tgf::make_random_stream(20000, 120, 5);
  const tgf::TCsr g = tgf::build_parallel(st, true, 4);
  std::vector<tgf::NodeId> nodes;
  std::vector<tgf::Time> times;
  for (int i = 0; i < 3000; i += 3) {
    nodes.push_back(st.events[i].src);
    nodes.push_back(st.events[i].dst);
    times.push_back(st.events[i].timestamp);
    times.push_back(st.events[i].timestamp + 0.5);
  }
  for (auto strat : {tgf::SampleStrategy::recent, tgf::SampleStrategy::random}) {
    for (std::int64_t k : {1, 10, 20, 300}) {
      const auto two = tgf::build_sequence_batch(tgf::sample_batch(g, nodes, times, k, strat, 9),
                                                 11, 20001);
      const auto one = tgf::sample_sequence_batch(g, nodes, times, k, strat, 9, 11, 20001);
      CHECK(one.node_index == two.node_index);
      CHECK(one.edge_index == two.edge_index);
      CHECK(one.time_delta == two.time_delta);
      CHECK(one.valid_len == two.valid_len);
      CHECK(one.target_row == two.target_row);
      one.validate();
    }
  }
  std::vector<tgf::NodeId> bad = nodes;
  bad[5] = 999;
  CHECK_THROWS_AS(tgf::sample_sequence_batch(g, bad, times, 5, tgf::SampleStrategy::recent, 0,
                                             11, 1),
                  tgf::ValidationError);
  CHECK_THROWS_AS(tgf::sample_sequence_batch(g, nodes, times, 0, tgf::SampleStrategy::recent, 0,
                                             11, 1),
                  tgf::ValidationError);
  CHECK_THROWS_AS(tgf::sample_sequence_batch(g, nodes, times, 5, tgf::SampleStrategy::recent, 0,
                                             1, 1),
                  tgf::ValidationError);
}

// sequence.cpp:55-86 restated on the host as the checker for the device route below
static tgf::SequenceBatch host_sequences(const std::vector<tgf::NeighborSample>& samples,
                                         std::int64_t l, std::int64_t self_idx) {
  tgf::SequenceBatch out;
  out.batch = static_cast<std::int64_t>(samples.size());
  out.l = l;
  out.node_index.assign(out.batch * l, 0);
  out.edge_index.assign(out.batch * l, 0);
  out.time_delta = tgf::Matrix(out.batch, l);
  out.valid_len.resize(out.batch);
  out.target_row.resize(out.batch);
  for (std::int64_t b = 0; b < out.batch; ++b) {
    const auto& s = samples[b];
    const auto total = static_cast<std::int64_t>(s.neighbors.size());
    const std::int64_t k = std::min(total, l - 1), skip = total - k;
    for (std::int64_t j = 0; j < k; ++j) {
      out.node_index[b * l + j] = s.neighbors[skip + j].neighbor + 1;
      out.edge_index[b * l + j] = s.neighbors[skip + j].edge + 1;
      out.time_delta.at(b, j) = s.query_time - s.neighbors[skip + j].timestamp;
    }
    out.node_index[b * l + k] = s.query_node + 1;
    out.edge_index[b * l + k] = self_idx;
    out.valid_len[b] = k + 1;
    out.target_row[b] = k;
  }
  return out;
}

TEST_CASE("forward_concat route: large batches (threaded unpack) equal small ones and the host restatement") {
  const tgf::EventStream st = tgf::make_random_stream(60000, 400, 8);
  const tgf::TCsr g = tgf::build_parallel(st, true, 4);
  std::vector<tgf::NodeId> nodes;
  std::vector<tgf::Time> times;
  for (int i = 0; i < 60000; i += 4) {  // 15,000 queries: above the threaded-copy threshold
    nodes.push_back(st.events[i].src);
    times.push_back(st.events[i].timestamp);
  }
  for (auto strat : {tgf::SampleStrategy::recent, tgf::SampleStrategy::random}) {
    for (std::int64_t k : {3, 10, 40}) {
      const auto big = tgf::sample_batch(g, nodes, times, k, strat, 5);
      REQUIRE(big.size() == nodes.size());
      // the same queries in 1,000-query calls (unthreaded); uniform streams restart per call,
      // so compare those only for recent
      for (std::size_t c0 = 0; strat == tgf::SampleStrategy::recent && c0 < nodes.size();
           c0 += 1000) {
        const std::size_t c1 = std::min(nodes.size(), c0 + 1000);
        const std::vector<tgf::NodeId> n(nodes.begin() + c0, nodes.begin() + c1);
        const std::vector<tgf::Time> t(times.begin() + c0, times.begin() + c1);
        const auto small = tgf::sample_batch(g, n, t, k, strat, 5);
        for (std::size_t i = 0; i < small.size(); ++i) {
          REQUIRE(small[i].neighbors.size() == big[c0 + i].neighbors.size());
          CHECK(small[i].query_node == big[c0 + i].query_node);
          for (std::size_t j = 0; j < small[i].neighbors.size(); ++j) {
            CHECK(small[i].neighbors[j].neighbor == big[c0 + i].neighbors[j].neighbor);
            CHECK(small[i].neighbors[j].edge == big[c0 + i].neighbors[j].edge);
            CHECK(small[i].neighbors[j].timestamp == big[c0 + i].neighbors[j].timestamp);
          }
        }
      }
      for (std::int64_t l : {2, 11, 64}) {
        const auto dev = tgf::build_sequence_batch(big, l, 60001);
        const auto want = host_sequences(big, l, 60001);
        CHECK(dev.batch == want.batch);
        CHECK(dev.l == want.l);
        CHECK(dev.node_index == want.node_index);
        CHECK(dev.edge_index == want.edge_index);
        CHECK(dev.time_delta == want.time_delta);
        CHECK(dev.valid_len == want.valid_len);
        CHECK(dev.target_row == want.target_row);
      }
    }
  }
  // hand-made samples: empty, longer than l - 1, a single one
  std::vector<tgf::NeighborSample> hand(3);
  hand[0].query_node = 7;
  hand[0].query_time = 5.0;
  hand[1].query_node = 3;
  hand[1].query_time = 100.0;
  for (int j = 0; j < 30; ++j) hand[1].neighbors.push_back({j, 1000 + j, 1.0 + j});
  hand[2].query_node = 1;
  hand[2].query_time = 9.0;
  hand[2].neighbors.push_back({4, 44, 8.5});
  for (std::int64_t l : {2, 5, 40}) {
    const auto dev = tgf::build_sequence_batch(hand, l, -3);
    const auto want = host_sequences(hand, l, -3);
    CHECK(dev.node_index == want.node_index);
    CHECK(dev.edge_index == want.edge_index);
    CHECK(dev.time_delta == want.time_delta);
    CHECK(dev.valid_len == want.valid_len);
  }
  CHECK(tgf::build_sequence_batch({}, 4, 1).batch == 0);
}

TEST_CASE("concurrent readers: threads sampling one TCsr get the single-threaded results") {
  // a TCsr is safe for concurrent readers; each calling thread has its own device
  // arena, stream and pinned staging in the host layer
  const tgf::EventStream st = tgf::make_random_stream(50000, 300, 12);
  const tgf::TCsr g = tgf::build_parallel(st, true, 4);
  std::vector<tgf::NodeId> nodes;
  std::vector<tgf::Time> times;
  for (int i = 0; i < 50000; i += 10) {
    nodes.push_back(st.events[i].dst);
    times.push_back(st.events[i].timestamp);
  }
  const auto want_s = tgf::sample_batch(g, nodes, times, 10, tgf::SampleStrategy::random, 3);
  const auto want = tgf::build_sequence_batch(want_s, 11, 50001);
  const auto want_f = tgf::sample_sequence_batch(g, nodes, times, 10,
                                                 tgf::SampleStrategy::random, 3, 11, 50001);
  std::vector<int> ok(8, 0);
  std::vector<std::thread> th;
  for (int t = 0; t < 8; ++t)
    th.emplace_back([&, t] {
      bool good = true;
      for (int rep = 0; rep < 5; ++rep) {
        const auto s = tgf::sample_batch(g, nodes, times, 10, tgf::SampleStrategy::random, 3);
        const auto q = tgf::build_sequence_batch(s, 11, 50001);
        const auto f = tgf::sample_sequence_batch(g, nodes, times, 10,
                                                  tgf::SampleStrategy::random, 3, 11, 50001);
        good = good && q.node_index == want.node_index && q.edge_index == want.edge_index &&
               q.time_delta == want.time_delta && q.valid_len == want.valid_len &&
               f.node_index == want_f.node_index && f.time_delta == want_f.time_delta;
      }
      ok[t] = good ? 1 : 0;
    });
  for (auto& x : th) x.join();
  for (int t = 0; t < 8; ++t) CHECK(ok[t] == 1);
}
