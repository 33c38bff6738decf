// inputs.cu -- assemble_inputs: the sequence tensors' first consumer.
//
// Replaces tgf::assemble_inputs (proj/src/attention.cpp:414-451): for every valid position
// j < valid_len[b] of row b, the Transformer input row
//   sum mode:    z = node_table[ni] + edge_table[ei] + cos(omega * dt + phi)      (d columns)
//   concat mode: z = [node_table[ni] | edge_table[ei] | cos(omega * dt + phi)]    (d_v+d_e+d_t)
// with ni / ei / dt the sampler's node_index / edge_index / time_delta; padding rows stay 0.
// An index outside its table is the reference's ValidationError.
//
// Memory-bound gather: one warp per row, lanes across columns, so every table-row read and
// every z-row write is a coalesced run; omega/phi live in shared memory; the time encoding is
// computed in fp64 (the reference's precision) and rounded once to the output type.
#include <cuda_bf16.h>

#include <algorithm>

#include "graph.cuh"

namespace tgfx {
namespace {

constexpr int kIT = 256;

template <typename T>
__device__ __forceinline__ double to_f64(T v) {
  return static_cast<double>(v);
}
template <typename T>
__device__ __forceinline__ T from_f64(double v) {
  return static_cast<T>(v);
}
template <>
__device__ __forceinline__ __nv_bfloat16 from_f64<__nv_bfloat16>(double v) {
  return __double2bfloat16(v);
}

template <typename IdxT, typename DtT, typename TabT, typename OutT>
__global__ void __launch_bounds__(kIT) k_assemble_inputs(
    int64_t q, int64_t l, const IdxT* __restrict__ ni_, const IdxT* __restrict__ ei_,
    const DtT* __restrict__ dt_, const IdxT* __restrict__ vlen, const TabT* __restrict__ ntab,
    int64_t nrows, const TabT* __restrict__ etab, int64_t erows, const double* __restrict__ omega,
    const double* __restrict__ phi, int d_v, int d_e, int d_t, int concat, OutT* __restrict__ z,
    int* __restrict__ bad) {
  extern __shared__ double s_wp[];  // omega [d_t] | phi [d_t]
  for (int c = threadIdx.x; c < d_t; c += kIT) {
    s_wp[c] = omega[c];
    s_wp[d_t + c] = phi[c];
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int d = concat ? d_v + d_e + d_t : d_t;
  const int64_t rows = q * l;
  for (int64_t r = (blockIdx.x * (int64_t)kIT + threadIdx.x) >> 5; r < rows;
       r += (static_cast<int64_t>(gridDim.x) * kIT) >> 5) {
    const int64_t b = r / l, j = r - b * l;
    OutT* zr = z + r * d;
    if (j >= static_cast<int64_t>(vlen[b])) {  // padding row
      for (int c = lane; c < d; c += 32) zr[c] = from_f64<OutT>(0.0);
      continue;
    }
    const int64_t ni = static_cast<int64_t>(ni_[r]), ei = static_cast<int64_t>(ei_[r]);
    if (ni < 0 || ni >= nrows || ei < 0 || ei >= erows) {  // attention.cpp:427-431
      if (lane == 0 && bad) atomicOr(bad, 1);
      continue;
    }
    const double dt = static_cast<double>(dt_[r]);
    const TabT* nrow = ntab + ni * d_v;  // node_table (num_nodes+1) x d_v (attention.hpp:63)
    const TabT* erow = etab + ei * d_e;  // edge_table (num_edges+2) x d_e
    if (!concat) {
      for (int c = lane; c < d; c += 32)
        zr[c] = from_f64<OutT>(to_f64(__ldg(nrow + c)) + to_f64(__ldg(erow + c)) +
                               cos(s_wp[c] * dt + s_wp[d_t + c]));
    } else {
      for (int c = lane; c < d_v; c += 32) zr[c] = from_f64<OutT>(to_f64(__ldg(nrow + c)));
      for (int c = lane; c < d_e; c += 32) zr[d_v + c] = from_f64<OutT>(to_f64(__ldg(erow + c)));
      for (int c = lane; c < d_t; c += 32)
        zr[d_v + d_e + c] = from_f64<OutT>(cos(s_wp[c] * dt + s_wp[d_t + c]));
    }
  }
}

template <typename IdxT, typename DtT, typename TabT, typename OutT>
void launch_t(const AssembleInputsArgs& a, int* bad, cudaStream_t s) {
  const int64_t rows = a.q * a.l;
  const int grid = static_cast<int>(
      std::min<int64_t>(ceil_div(rows * 32, kIT), static_cast<int64_t>(device_info().sms) * 16));
  k_assemble_inputs<IdxT, DtT, TabT, OutT><<<grid, kIT, sizeof(double) * 2 * a.d_t, s>>>(
      a.q, a.l, static_cast<const IdxT*>(a.node_index), static_cast<const IdxT*>(a.edge_index),
      static_cast<const DtT*>(a.time_delta), static_cast<const IdxT*>(a.valid_len),
      static_cast<const TabT*>(a.node_table), a.node_rows, static_cast<const TabT*>(a.edge_table),
      a.edge_rows, a.omega, a.phi, static_cast<int>(a.d_v), static_cast<int>(a.d_e),
      static_cast<int>(a.d_t), a.concat, static_cast<OutT*>(a.z), bad);
  after_launch("k_assemble_inputs");
}

template <typename IdxT, typename DtT, typename TabT>
void launch_out(const AssembleInputsArgs& a, int* bad, cudaStream_t s) {
  switch (a.z_type) {
    case TGFX_F32: launch_t<IdxT, DtT, TabT, float>(a, bad, s); break;
    case TGFX_F64: launch_t<IdxT, DtT, TabT, double>(a, bad, s); break;
    case TGFX_BF16: launch_t<IdxT, DtT, TabT, __nv_bfloat16>(a, bad, s); break;
    default: throw Error(TGFX_EVALIDATION, "unknown output type");
  }
}

template <typename IdxT, typename DtT>
void launch_tab(const AssembleInputsArgs& a, int* bad, cudaStream_t s) {
  switch (a.table_type) {
    case TGFX_F32: launch_out<IdxT, DtT, float>(a, bad, s); break;
    case TGFX_F64: launch_out<IdxT, DtT, double>(a, bad, s); break;
    default: throw Error(TGFX_EVALIDATION, "tables must be f32 or f64");
  }
}

}  // namespace

void launch_assemble_inputs(const AssembleInputsArgs& a, int* bad, cudaStream_t s) {
  if (a.q <= 0 || a.l <= 0) return;
  const bool i64 = a.index64 != 0;
  if (a.dt_type == TGFX_F32) {
    if (i64)
      launch_tab<int64_t, float>(a, bad, s);
    else
      launch_tab<int32_t, float>(a, bad, s);
  } else if (a.dt_type == TGFX_F64) {
    if (i64)
      launch_tab<int64_t, double>(a, bad, s);
    else
      launch_tab<int32_t, double>(a, bad, s);
  } else {
    throw Error(TGFX_EVALIDATION, "time_delta must be f32 or f64");
  }
}

}  // namespace tgfx
