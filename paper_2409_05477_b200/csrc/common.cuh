// common.cuh -- shared device helpers and host plumbing for libtgfx (sm_100a only).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <stdexcept>
#include <string>

#include "tgfx.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "libtgfx is written for sm_100a (B200); compile with -gencode arch=compute_100a,code=sm_100a"
#endif

namespace tgfx {

constexpr int kWarp = 32;
constexpr unsigned kFull = 0xffffffffu;
constexpr uint64_t kGamma = 0x9e3779b97f4a7c15ULL;
constexpr uint64_t kStreamMul = 0xd6e8feb86659fd93ULL;

// ---------------------------------------------------------------- errors (host)
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

void check_cuda(cudaError_t e, const char* what);
#define TGFX_CUDA(x) ::tgfx::check_cuda((x), #x)
void count_launch(int n = 1);
void after_launch(const char* name);  // cudaGetLastError + launch counter

// ---------------------------------------------------------------- RNG (device)
// proj/include/tgformer/rng.hpp:11-16 (splitmix64 finaliser)
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x += kGamma;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}
// rng.hpp:23-24: CounterRng(seed, stream) initial state
__host__ __device__ __forceinline__ uint64_t rng_state(uint64_t seed, uint64_t stream) {
  return mix64(mix64(seed) ^ (stream * kStreamMul));
}
// d-th next_u64() (0-based) of the generator with initial state s0 (rng.hpp:26-32):
// skip-ahead, the state after d+1 increments finalised == mix64(s0 + d*gamma).
__host__ __device__ __forceinline__ uint64_t rng_draw(uint64_t s0, uint64_t d) {
  return mix64(s0 + d * kGamma);
}
// rng.hpp:35-38 next_below: high 64 bits of the 128-bit product
__device__ __forceinline__ uint64_t mulhi64(uint64_t a, uint64_t b) { return __umul64hi(a, b); }
// rng.hpp:41-43 next_double
__device__ __forceinline__ double to_unit_double(uint64_t x) {
  return static_cast<double>(x >> 11) * 0x1.0p-53;
}

// ---------------------------------------------------------------- loads
__device__ __forceinline__ double ldg_f64(const double* p) { return __ldg(p); }
__device__ __forceinline__ int64_t ldg_i64(const int64_t* p) {
  return static_cast<int64_t>(__ldg(reinterpret_cast<const long long*>(p)));
}
// one 32-byte TemporalEvent as two 16-byte vector loads (read-only, streaming)
struct Ev {
  int64_t eid, src, dst;
  double t;
};
__device__ __forceinline__ Ev load_event(const tgfx_event* ev, int64_t i) {
  const longlong2* p = reinterpret_cast<const longlong2*>(ev + i);
  longlong2 a, b;
  asm volatile("ld.global.nc.L1::no_allocate.v2.s64 {%0, %1}, [%2];"
               : "=l"(a.x), "=l"(a.y) : "l"(p));
  asm volatile("ld.global.nc.L1::no_allocate.v2.s64 {%0, %1}, [%2];"
               : "=l"(b.x), "=l"(b.y) : "l"(p + 1));
  Ev e;
  e.eid = a.x;
  e.src = a.y;
  e.dst = b.x;
  e.t = __longlong_as_double(b.y);
  return e;
}

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned r;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(r));
  return r;
}

// ---------------------------------------------------------------- device info (host)
struct DeviceInfo {
  int device = 0;
  int sms = 148;
  size_t smem_optin = 232448;
};
const DeviceInfo& device_info();

// stream-ordered device allocation (pool kept warm across calls)
void* dmalloc(size_t bytes, cudaStream_t s);
void dfree(void* p, cudaStream_t s);

// Grid for a grid-stride kernel: never more blocks than can be resident at once, so every
// thread sweeps the index space together (a second wave would revisit each output region
// long after the first, evicting half-written sectors).
template <typename K>
int resident_grid(K kernel, int threads, size_t smem, int64_t work_items) {
  int bps = 0;
  check_cuda(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, kernel, threads, smem),
             "cudaOccupancyMaxActiveBlocksPerMultiprocessor");
  const int64_t need = (work_items + threads - 1) / threads;
  const int64_t cap = static_cast<int64_t>(device_info().sms) * (bps > 0 ? bps : 1);
  return static_cast<int>(need < 1 ? 1 : (need < cap ? need : cap));
}

__host__ __device__ __forceinline__ int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

}  // namespace tgfx
