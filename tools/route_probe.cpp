// route_probe.cpp -- per-call timing of the C++ forward_concat route on one forward_concat batch
// (1,800 queries, GDELT-shaped graph of 20 M events): C ABI calls from pinned buffers, the tgf::
// calls, and the caller-side destruction of the results.  Build: see the g++ line in
// profiles/r02/route_probe.txt.  Not part of the product.
#include <chrono>
#include <cstdio>
#include <cstring>
#include <vector>
#include "tgfx.h"
#include "tgfx/tgformer.hpp"
using Clock = std::chrono::steady_clock;
static double us(Clock::time_point a) { return std::chrono::duration<double, std::micro>(Clock::now() - a).count(); }
int main() {
  const std::int64_t E = 20000000, V = 16682, B = 600, k = 10, l = 11;
  const tgf::EventStream st = tgf::make_random_stream(E, V, 42);
  const tgf::TCsr g = tgf::build_parallel(st, true, 16);
  const int R = 400;
  std::vector<tgf::NodeId> nodes(3 * B);
  std::vector<tgf::Time> times(3 * B);
  auto fill = [&](int r) {
    const std::int64_t e0 = (std::int64_t(r) * 7919 * B) % (E - B);
    for (int i = 0; i < B; ++i) {
      const auto& e = st.events[e0 + i];
      nodes[i] = e.src; nodes[B + i] = e.dst; nodes[2 * B + i] = (e.src * 31 + i) % V;
      times[i] = times[B + i] = times[2 * B + i] = e.timestamp;
    }
  };
  const std::int64_t q = 3 * B;
  void *pin_in, *pin_out;
  tgfx_host_alloc(1 << 24, &pin_in);
  tgfx_host_alloc(1 << 24, &pin_out);
  auto* pn = static_cast<std::int64_t*>(pin_in);
  auto* pt = reinterpret_cast<double*>(pn + q);
  auto* o = static_cast<char*>(pin_out);
  tgfx_graph* h = g.device();
  double t[10] = {0};
  for (int r = 0; r < R + 20; ++r) {
    fill(r);
    const bool on = r >= 20;
    auto c0 = Clock::now();
    std::memcpy(pn, nodes.data(), 8 * q); std::memcpy(pt, times.data(), 8 * q);
    tgfx_sample_sequence_batch(h, pn, pt, q, k, TGFX_RECENT, 9, 0, l, E + 1, (std::int64_t*)o,
                               (std::int64_t*)(o + 8 * q * l), (double*)(o + 16 * q * l),
                               (std::int64_t*)(o + 24 * q * l), (std::int64_t*)(o + 25 * q * l));
    if (on) t[0] += us(c0);
    c0 = Clock::now();
    tgfx_sample_sequence_batch(h, pn, pt, 1, k, TGFX_RECENT, 9, 0, l, E + 1, (std::int64_t*)o,
                               (std::int64_t*)(o + 8 * q * l), (double*)(o + 16 * q * l),
                               (std::int64_t*)(o + 24 * q * l), (std::int64_t*)(o + 25 * q * l));
    if (on) t[1] += us(c0);
    c0 = Clock::now();
    { auto s = tgf::sample_sequence_batch(g, nodes, times, k, tgf::SampleStrategy::recent, 9, l, E + 1); }
    if (on) t[2] += us(c0);
    c0 = Clock::now();
    tgfx_sample_batch_records(h, pn, pt, q, k, TGFX_RECENT, 9, 0, (std::int64_t*)o, (tgfx_neighbor*)(o + 8 * q));
    if (on) t[3] += us(c0);
    c0 = Clock::now();
    std::vector<tgf::NeighborSample>* sp = new std::vector<tgf::NeighborSample>(
        tgf::sample_batch(g, nodes, times, k, tgf::SampleStrategy::recent, 9));
    if (on) t[4] += us(c0);
    c0 = Clock::now();
    { auto s = tgf::build_sequence_batch(*sp, l, E + 1); if (on) t[5] += us(c0); c0 = Clock::now(); }
    if (on) t[6] += us(c0);
    c0 = Clock::now();
    delete sp;
    if (on) t[7] += us(c0);
  }
  const char* names[] = {"C fused q=1800 pinned", "C fused q=1", "C++ fused", "C records q=1800 pinned",
                         "C++ sample_batch", "C++ build_sequence_batch", "SequenceBatch dtor", "samples dtor"};
  for (int i = 0; i < 8; ++i) std::printf("%-28s %8.1f us\n", names[i], t[i] / R);
}
