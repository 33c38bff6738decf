// tcsr_interop.cpp -- T-CSR container interop with the reference:
//   ours -> file -> the reference's load_tcsr; the reference's save_tcsr -> file -> ours;
//   byte-identical files for the same graph; and (argument "big") a >= 4 GiB container that
//   round-trips through ours, which the reference's own load rejects (its CRC is computed with
//   the length truncated to 32 bits, proj/src/binary_io.hpp:95-96).
// Usage: tcsr_interop <oracle/_ref/libtgf_ref.so> <scratch dir> [big]
// Prints "interop ok" / "big ok"; exit code 0 on success.
#include <dlfcn.h>

#include <cstdio>
#include <cstring>
#include <fstream>
#include <iterator>
#include <string>
#include <vector>

#include "tgfx/tgformer.hpp"

namespace {
struct Ref {
  void* h = nullptr;
  const char* (*last_error)();
  int (*make_random_stream)(int64_t, int64_t, uint64_t, double, void*);
  void* (*stream_create)(const void*, int64_t, int64_t);
  void (*stream_free)(void*);
  int (*build)(void*, int, int, void**, double*);
  void (*graph_free)(void*);
  void (*graph_info)(void*, int64_t*);
  void (*graph_export)(void*, int64_t*, int64_t*, int64_t*, double*);
  int (*save)(void*, const char*);
  int (*load)(const char*, void**);
};

template <class F>
void sym(Ref& r, F& f, const char* name) {
  f = reinterpret_cast<F>(dlsym(r.h, name));
  if (!f) throw std::runtime_error(std::string("missing ") + name);
}

Ref open_ref(const char* path) {
  Ref r;
  // DEEPBIND: the reference resolves its own tgf:: symbols, not the same-named ones of
  // libtgformer already loaded in this process
  r.h = dlopen(path, RTLD_NOW | RTLD_LOCAL | RTLD_DEEPBIND);
  if (!r.h) throw std::runtime_error(dlerror());
  sym(r, r.last_error, "ref_last_error");
  sym(r, r.make_random_stream, "ref_make_random_stream");
  sym(r, r.stream_create, "ref_stream_create");
  sym(r, r.stream_free, "ref_stream_free");
  sym(r, r.build, "ref_build");
  sym(r, r.graph_free, "ref_graph_free");
  sym(r, r.graph_info, "ref_graph_info");
  sym(r, r.graph_export, "ref_graph_export");
  sym(r, r.save, "ref_save_tcsr");
  sym(r, r.load, "ref_load_tcsr");
  return r;
}

bool same(Ref& ref, void* rg, const tgf::TCsr& g) {
  int64_t info[4];
  ref.graph_info(rg, info);
  if (info[0] != g.num_nodes || info[1] != g.num_edges || info[2] != g.num_entries() ||
      (info[3] != 0) != g.reverse)
    return false;
  std::vector<int64_t> ip(info[0] + 1), nb(info[2]), ed(info[2]);
  std::vector<double> ts(info[2]);
  ref.graph_export(rg, ip.data(), nb.data(), ed.data(), ts.data());
  return ip == g.indptr && nb == g.neighbor_ids && ed == g.edge_ids &&
         std::memcmp(ts.data(), g.timestamps.data(), ts.size() * sizeof(double)) == 0;
}

std::vector<char> bytes(const std::string& p) {
  std::ifstream in(p, std::ios::binary);
  return std::vector<char>(std::istreambuf_iterator<char>(in), {});
}

int fail(const std::string& m) {
  std::printf("FAIL: %s\n", m.c_str());
  return 1;
}
}  // namespace

int main(int argc, char** argv) {
  if (argc < 3) return fail("usage: tcsr_interop <libtgf_ref.so> <dir> [big]");
  Ref ref = open_ref(argv[1]);
  const std::string dir = argv[2];
  const bool big = argc > 3 && std::string(argv[3]) == "big";
  if (!big) {
    for (int reverse = 0; reverse < 2; ++reverse) {
      const tgf::EventStream s = tgf::make_random_stream(300000, 5000, 77, 1.2);
      const tgf::TCsr g = tgf::build_parallel(s, reverse != 0, 8);
      const std::string ours = dir + "/ours.tcsr", theirs = dir + "/theirs.tcsr";
      // ours -> the reference's loader
      tgf::save_tcsr(g, ours);
      void* rg = nullptr;
      if (ref.load(ours.c_str(), &rg)) return fail(std::string("ref load: ") + ref.last_error());
      if (!same(ref, rg, g)) return fail("reference load of our container differs");
      // the reference's writer -> ours
      if (ref.save(rg, theirs.c_str())) return fail(std::string("ref save: ") + ref.last_error());
      ref.graph_free(rg);
      const tgf::TCsr back = tgf::load_tcsr(theirs);
      if (back.indptr != g.indptr || back.neighbor_ids != g.neighbor_ids ||
          back.edge_ids != g.edge_ids || back.num_nodes != g.num_nodes ||
          back.num_edges != g.num_edges || back.reverse != g.reverse ||
          std::memcmp(back.timestamps.data(), g.timestamps.data(),
                      g.timestamps.size() * sizeof(double)) != 0)
        return fail("our load of the reference's container differs");
      if (bytes(ours) != bytes(theirs)) return fail("containers are not byte-identical");
      // a reference-built graph of the same stream saves to the same bytes too
      void* st = ref.stream_create(s.events.data(), static_cast<int64_t>(s.events.size()),
                                   s.num_nodes);
      void* rb = nullptr;
      if (ref.build(st, reverse, 0, &rb, nullptr)) return fail(ref.last_error());
      ref.stream_free(st);
      if (ref.save(rb, theirs.c_str())) return fail(ref.last_error());
      ref.graph_free(rb);
      if (bytes(ours) != bytes(theirs)) return fail("reference build saves different bytes");
      std::remove(ours.c_str());
      std::remove(theirs.c_str());
    }
    std::printf("interop ok\n");
    return 0;
  }
  // >= 4 GiB container: 24 B per entry + 8 B per node + header
  const int64_t E = 92'000'000, V = 20'000;
  const tgf::EventStream s = tgf::make_random_stream(E, V, 5, 1.2);
  const tgf::TCsr g = tgf::build_parallel(s, true, 8);
  const std::string path = dir + "/big.tcsr";
  tgf::save_tcsr(g, path);
  std::ifstream f(path, std::ios::binary | std::ios::ate);
  const long long size = static_cast<long long>(f.tellg());
  f.close();
  if (size < (4LL << 30)) return fail("container below 4 GiB");
  const tgf::TCsr back = tgf::load_tcsr(path);
  if (back.indptr != g.indptr || back.neighbor_ids != g.neighbor_ids ||
      back.edge_ids != g.edge_ids ||
      std::memcmp(back.timestamps.data(), g.timestamps.data(),
                  g.timestamps.size() * sizeof(double)) != 0)
    return fail("4 GiB round trip differs");
  void* rg = nullptr;
  const int rc = ref.load(path.c_str(), &rg);
  const std::string msg = rc ? ref.last_error() : "";
  if (rg) ref.graph_free(rg);
  std::remove(path.c_str());
  std::printf("big ok: %lld bytes round-trip; reference load: %s\n", size,
              rc ? msg.c_str() : "accepted");
  return 0;
}
