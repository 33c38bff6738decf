// fromchars.cpp -- std::from_chars (libstdc++, the reference's number parser in
// event_stream.cpp:38-59) exposed to the tests as the checker of the device CSV parser.
// TEST INFRASTRUCTURE ONLY.
#include <charconv>
#include <cstdint>
#include <system_error>

extern "C" {

// 0 ok; 1 error (syntax / out of range / not fully consumed), as load_csv's parse_* treat it
int orc_from_chars_f64(const char* s, int64_t n, double* out) {
  double v = 0.0;
  const auto r = std::from_chars(s, s + n, v);
  if (r.ec != std::errc{} || r.ptr != s + n) return 1;
  *out = v;
  return 0;
}

int orc_from_chars_i64(const char* s, int64_t n, int64_t* out) {
  long long v = 0;
  const auto r = std::from_chars(s, s + n, v);
  if (r.ec != std::errc{} || r.ptr != s + n) return 1;
  *out = v;
  return 0;
}
}
