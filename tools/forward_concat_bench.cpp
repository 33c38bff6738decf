// forward_concat_bench.cpp -- times the drop-in C++ route a reference caller takes
// (bench.py's e2e_cpp legs).  forward_concat (proj/src/training.cpp:193-214) builds, per
// batch of B events, the queries [src | dst | neg] at the event times and then calls
//     samples = tgf::sample_batch(g, nodes, times, k, strategy, seed);
//     seq     = tgf::build_sequence_batch(samples, l, num_edges + 1);
// This program links libtgformer.so (include/tgfx/tgformer.hpp) exactly as a relinked
// reference caller would, and times on the GDELT-shaped workload:
//   build : tgf::build_parallel(stream, true, threads) of the whole stream (host vectors in,
//           TCsr with host columns out -- the reference's return-by-value contract);
//   route : per batch, mode 0 = the two calls above (NeighborSamples materialised on the
//           host, as the API returns them), mode 1 = tgf::sample_sequence_batch (one call);
// over `batches` forward_concat batches spread evenly over the whole stream, after `warmup`
// untimed batches; the per-query time is extrapolated to all 3E queries (one process cannot
// issue 956,455 x 2 synchronous calls within the bench's time budget).
// Output: one JSON object on stdout.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "tgfx/tgformer.hpp"

using Clock = std::chrono::steady_clock;
static double secs(Clock::time_point a) {
  return std::chrono::duration<double>(Clock::now() - a).count();
}

int main(int argc, char** argv) {
  if (argc < 10) {
    std::fprintf(stderr, "usage: E V k l B strategy(recent|random) batches warmup mode(0|1)\n");
    return 2;
  }
  const std::int64_t E = std::atoll(argv[1]), V = std::atoll(argv[2]), k = std::atoll(argv[3]),
                     l = std::atoll(argv[4]), B = std::atoll(argv[5]);
  const tgf::SampleStrategy strat = tgf::parse_strategy(argv[6]);
  const std::int64_t batches = std::atoll(argv[7]), warmup = std::atoll(argv[8]);
  const int mode = std::atoi(argv[9]);
  const tgf::EventStream stream = tgf::make_random_stream(E, V, 42);
  // warm the device and the allocator once, untimed (the first CUDA call initialises a context)
  { tgf::TCsr w = tgf::build_parallel(stream, true, 16); }
  const auto t0 = Clock::now();
  const tgf::TCsr g = tgf::build_parallel(stream, true, 16);
  const double t_build = secs(t0);
  const std::int64_t nbatch = (E + B - 1) / B;
  double t_route = 0.0;
  std::int64_t q_timed = 0, checksum = 0;
  std::vector<tgf::NodeId> nodes;
  std::vector<tgf::Time> times;
  for (std::int64_t j = 0; j < warmup + batches; ++j) {
    const std::int64_t b = std::min(nbatch - 1, (j * nbatch) / (warmup + batches));
    const std::int64_t e0 = b * B, e1 = std::min(E, e0 + B), n = e1 - e0;
    nodes.assign(static_cast<std::size_t>(3 * n), 0);
    times.assign(static_cast<std::size_t>(3 * n), 0.0);
    for (std::int64_t i = 0; i < n; ++i) {  // training.cpp:193-209, negatives metrics.cpp:68-69
      const tgf::TemporalEvent& e = stream.events[static_cast<std::size_t>(e0 + i)];
      nodes[i] = e.src;
      nodes[n + i] = e.dst;
      nodes[2 * n + i] = static_cast<tgf::NodeId>(
          tgf::CounterRng(7, static_cast<std::uint64_t>(e0 + i)).next_below(
              static_cast<std::uint64_t>(V)));
      times[i] = times[n + i] = times[2 * n + i] = e.timestamp;
    }
    const auto t1 = Clock::now();
    tgf::SequenceBatch seq;
    if (mode == 0) {
      const std::vector<tgf::NeighborSample> samples =
          tgf::sample_batch(g, nodes, times, k, strat, 9 + static_cast<std::uint64_t>(b));
      seq = tgf::build_sequence_batch(samples, l, E + 1);
    } else {
      seq = tgf::sample_sequence_batch(g, nodes, times, k, strat, 9 + static_cast<std::uint64_t>(b),
                                       l, E + 1);
    }
    const double dt = secs(t1);
    if (j >= warmup) {
      t_route += dt;
      q_timed += 3 * n;
    }
    for (std::int64_t v : seq.valid_len) checksum += v;
  }
  const double t_query = t_route / static_cast<double>(q_timed);
  const double total = t_build + t_query * 3.0 * static_cast<double>(E);
  std::printf("{\"value\": %.6e, \"unit\": \"edges/s\", \"build_s\": %.6f, \"t_query_s\": %.6e, "
              "\"queries_timed\": %lld, \"batches_timed\": %lld, \"ms_per_step\": %.3f, "
              "\"mode\": %d, \"valid_len_sum\": %lld}\n",
              static_cast<double>(E) / total, t_build, t_query, static_cast<long long>(q_timed),
              static_cast<long long>(batches), 1e3 * total, mode,
              static_cast<long long>(checksum));
  return 0;
}
