// primitives.cuh -- device-wide primitives (see primitives.cu).
#pragma once
#include "common.cuh"

namespace tgfx {

// Stable LSD radix sort of (key, value) pairs by the low max_bits of key, 8 bits per pass;
// digits constant across all keys are skipped.  On return keys/vals point at the sorted
// buffers (either the originals or the alternates).  hist: the keys' digit histograms
// [pass][256] (u64, on the device) when the caller already counted them while writing the
// keys; else the sort counts them in its own pass.
template <typename K, typename V>
void radix_sort_pairs(K*& keys, V*& vals, K* keys_alt, V* vals_alt, int64_t n, int max_bits,
                      cudaStream_t s, const unsigned long long* hist = nullptr);

}  // namespace tgfx
