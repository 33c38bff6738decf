/*
 * tgfx.h -- C ABI of the B200-native T-CSR builder, temporal sampler and sequence assembler.
 *
 * Drop-in boundary for the reference hot path (tgformer, arXiv 2409.05477; paths below are
 * relative to the reference tree).  Every entry point cites the reference interface it
 * replaces.  Plain pointers and sizes only (no C++ / torch types).  All compute runs on the
 * current CUDA device in hand-written sm_100a kernels; there is no CPU fallback: without a
 * usable device every call fails with TGFX_ECUDA.
 *
 * Conventions
 *   - Host-buffer calls (no _device suffix) are synchronous, like the reference functions:
 *     inputs are uploaded, computed on the GPU and results copied back before returning.
 *     Nothing is written to caller outputs when an error is returned.
 *   - *_device calls take device pointers and a cudaStream_t (passed as void*, NULL = legacy
 *     default stream).  With flags & TGFX_TRUSTED they skip input validation and do not
 *     synchronise (fully asynchronous); otherwise they validate, synchronise and report.
 *   - Errors: return code (TGFX_E*), message via tgfx_last_error() (thread-local), with the
 *     reference's exception texts (proj/include/tgformer/common.hpp:15-27 error classes).
 *   - Ids are int64 and times double, as proj/include/tgformer/common.hpp:10-12.
 */
#ifndef TGFX_H
#define TGFX_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TGFX_ABI_VERSION 2

/* status codes; the C++ shim (include/tgfx/tgformer.hpp) rethrows the reference types */
#define TGFX_OK 0
#define TGFX_EVALIDATION 1  /* tgf::ValidationError */
#define TGFX_EFORMAT 2      /* tgf::FormatError */
#define TGFX_ECUDA 3        /* CUDA runtime / no device (std::runtime_error) */
#define TGFX_ENOMEM 4       /* device or host allocation failed (std::bad_alloc) */
#define TGFX_EUNSUPPORTED 5 /* e.g. ids that do not fit the requested int32 outputs */
#define TGFX_EPARSE 6       /* tgf::ParseError (CSV ingestion) */

/* sampling strategy: proj/include/tgformer/sampler.hpp:26 (SampleStrategy) */
#define TGFX_RECENT 0
#define TGFX_RANDOM 1

/* mask kinds: proj/include/tgformer/sequence.hpp:38 (MaskKind) */
#define TGFX_MASK_CAUSAL 0
#define TGFX_MASK_TGAT 1
#define TGFX_MASK_SELF_LOOP 2

/* element types of assemble_inputs operands */
#define TGFX_F32 0
#define TGFX_F64 1
#define TGFX_BF16 2

/* flags for *_device calls */
#define TGFX_TRUSTED 1u   /* inputs known valid: no validation pass, no synchronisation */
#define TGFX_INDEX64 2u   /* sample_assemble: node/edge index and valid_len are int64 */

/* proj/include/tgformer/event_stream.hpp:13-18 (TemporalEvent), byte-identical, so
 * stream.events.data() is passed without repacking. */
typedef struct tgfx_event {
  int64_t edge_id;
  int64_t src;
  int64_t dst;
  double timestamp;
} tgfx_event;

/* Opaque device-resident T-CSR (proj/include/tgformer/tcsr.hpp:20-33 TCsr). */
typedef struct tgfx_graph tgfx_graph;

/* Opaque device-resident parsed event stream (proj/include/tgformer/event_stream.hpp:26-39). */
typedef struct tgfx_csv tgfx_csv;

/* ---------------------------------------------------------------- runtime */
const char* tgfx_last_error(void);
int tgfx_abi_version(void);
/* number of kernel launches issued by this library so far (process-wide counter) */
uint64_t tgfx_launch_count(void);
/* bytes of device memory currently held by tgfx graphs + workspaces */
int64_t tgfx_device_bytes(void);

/* ---------------------------------------------------------------- T-CSR build */
/* replaces tgf::build_sequential (proj/include/tgformer/tcsr.hpp:37, tcsr.cpp:83-105) */
int tgfx_build_sequential(const tgfx_event* events, int64_t n, int64_t num_nodes, int reverse,
                          tgfx_graph** out);
/* replaces tgf::build_parallel (tcsr.hpp:43, tcsr.cpp:107-151).  num_threads < 1 is a
 * ValidationError as in tcsr.cpp:108; otherwise it is accepted and ignored (the grid is
 * sized for the device); the result is element-for-element identical. */
int tgfx_build_parallel(const tgfx_event* events, int64_t n, int64_t num_nodes, int reverse,
                        int num_threads, tgfx_graph** out);
/* device-resident events (n x 32 bytes); builds into a new graph. */
int tgfx_build_device(const tgfx_event* d_events, int64_t n, int64_t num_nodes, int reverse,
                      void* stream, unsigned flags, tgfx_graph** out);
/* rebuild an existing graph in place from device events with the same (n, num_nodes,
 * reverse); reuses its buffers and workspace (no allocation), for repeated builds. */
int tgfx_rebuild_device(tgfx_graph* g, const tgfx_event* d_events, void* stream,
                        unsigned flags);
/* import a host T-CSR (e.g. from load_tcsr, tcsr.cpp:176-197) to the device. */
int tgfx_graph_from_host(int64_t num_nodes, int64_t num_edges, int reverse, int64_t m,
                         const int64_t* indptr, const int64_t* nbr, const int64_t* eid,
                         const double* ts, tgfx_graph** out);
int tgfx_graph_info(const tgfx_graph* g, int64_t* num_nodes, int64_t* num_edges,
                    int64_t* num_entries, int* reverse);
/* copy the T-CSR columns to host: indptr[num_nodes+1], nbr/eid/ts[num_entries] */
int tgfx_graph_export(const tgfx_graph* g, int64_t* indptr, int64_t* nbr, int64_t* eid,
                      double* ts);
/* device pointers of the columns.  A build may leave nbr / eid unwritten (the sampler reads
 * 16-byte gather records instead); asking for them materialises them first, and they stay
 * valid until the next tgfx_rebuild_device of g -- ask again after a rebuild. */
int tgfx_graph_device_arrays(const tgfx_graph* g, const int64_t** indptr, const int64_t** nbr,
                             const int64_t** eid, const double** ts);
/* replaces TCsr::validate (tcsr.cpp:54-81), run on the device */
int tgfx_graph_validate(const tgfx_graph* g);
int tgfx_graph_free(tgfx_graph* g);
/* path the last build took: 0 presorted fast path, 1 general (re-sort), 2 large-V path */
int tgfx_graph_build_path(const tgfx_graph* g);

/* ---------------------------------------------------------------- partitioned build */
/* Node-range-partitioned multi-GPU build (the reference has no distributed
 * construction).  Host driver: paper_2409_05477_b200/partition.py.
 * Per-rank node degrees of a stream chunk (src, + dst if reverse); d_deg[num_nodes] is zeroed. */
int tgfx_degree_hist_device(const tgfx_event* d_events, int64_t n, int64_t num_nodes, int reverse,
                            uint64_t* d_deg, void* stream);
/* warps the partition kernels use for n events (size of the count/offset tables / nparts) */
int64_t tgfx_partition_warps(int64_t n);
/* Rank d owns the global entry positions [P[d], P[d+1]), P[d] = d*m/nparts: the nodes
 * [d_bounds[d], d_bounds[d+1]) whole, except the at most nparts-1 "split" nodes whose slice
 * contains a cut (the Zipf hubs), which are divided by entry position.  d_split (int64):
 * [ns, node[7], gp[7], P[9]] -- gp[i] = indptr[node[i]] + node[i]'s entries in earlier ranks'
 * chunks, i.e. the global position of this chunk's first entry of node[i].
 * Count pass: d_counts[w*nparts + d] = entries of warp w's event range that are not split
 * destined to rank d; d_split_counts[w*7 + i] = warp w's entries of split node i. */
int tgfx_partition_count_device(const tgfx_event* d_events, int64_t n, int reverse,
                                const int64_t* d_bounds, int nparts, int64_t nwarps,
                                const int64_t* d_split, int64_t* d_counts,
                                int64_t* d_split_counts, void* stream);
/* Stable scatter of the entries into per-destination records (32-byte tgfx_event: edge_id,
 * src = node - d_bounds[d] (owner-local id), dst = other endpoint (global id), timestamp) at
 * d_records[d_offsets[w*nparts + d] + rank in warp w], emission order preserved;
 * d_split_occ[w*7 + i] = occurrences of split node i before warp w's range. */
int tgfx_partition_scatter_device(const tgfx_event* d_events, int64_t n, int reverse,
                                  const int64_t* d_bounds, int nparts, int64_t nwarps,
                                  const int64_t* d_split, const int64_t* d_split_occ,
                                  const int64_t* d_offsets, tgfx_event* d_records, void* stream);
/* Build one node range from received records (in global stream order): a reverse = 0 build
 * over num_local_nodes nodes whose neighbour ids stay global (< num_nodes_total). */
int tgfx_build_range_device(const tgfx_event* d_records, int64_t n, int64_t num_local_nodes,
                            int64_t num_nodes_total, int64_t num_edges_total, void* stream,
                            unsigned flags, tgfx_graph** out);
/* New graph from device columns (copied), e.g. the all-gathered partitions.  Without
 * TGFX_TRUSTED the slices are checked on the device (sorted, NaN-free) to pick the search. */
int tgfx_graph_from_device(int64_t num_nodes, int64_t num_edges, int reverse, int64_t m,
                           const int64_t* d_indptr, const int64_t* d_nbr, const int64_t* d_eid,
                           const double* d_ts, void* stream, unsigned flags, tgfx_graph** out);

/* ---------------------------------------------------------------- sampling */
/* replaces tgf::sample_batch (sampler.hpp:42-45, sampler.cpp:84-104) [and sample_recent /
 * sample_random for q = 1, sampler.hpp:32-38].  Query i uses RNG stream stream_base + i
 * (stream_base = 0 is the reference).  Outputs padded [q, k]: counts[q] and nbr/eid/ts
 * [q*k] in ascending (t, eid) order, unused slots zero. */
int tgfx_sample_batch(const tgfx_graph* g, const int64_t* nodes, const double* times,
                      int64_t q, int64_t k, int strategy, uint64_t seed, uint64_t stream_base,
                      int64_t* counts, int64_t* nbr, int64_t* eid, double* ts);
/* One sampled neighbour in the reference's record layout (NeighborEntry, sampler.hpp:14-18;
 * 24 bytes, so a NeighborSample's std::vector<NeighborEntry> is a run of these). */
typedef struct tgfx_neighbor {
  int64_t neighbor;
  int64_t edge;
  double timestamp;
} tgfx_neighbor;
/* tgfx_sample_batch with the padded [q, k] entries written as tgfx_neighbor records (one
 * device->host copy; what the C++ layer's tgf::sample_batch copies into its NeighborSamples) */
int tgfx_sample_batch_records(const tgfx_graph* g, const int64_t* nodes, const double* times,
                              int64_t q, int64_t k, int strategy, uint64_t seed,
                              uint64_t stream_base, int64_t* counts, tgfx_neighbor* entries);
/* Page-locked host memory for the host-buffer calls: their copies from and to such buffers
 * run as plain DMA without the driver's bounce copy (cudaHostAlloc / cudaFreeHost). */
int tgfx_host_alloc(size_t bytes, void** p);
int tgfx_host_free(void* p);
int tgfx_sample_batch_device(const tgfx_graph* g, const int64_t* d_nodes,
                             const double* d_times, int64_t q, int64_t k, int strategy,
                             uint64_t seed, uint64_t stream_base, int64_t* d_counts,
                             int64_t* d_nbr, int64_t* d_eid, double* d_ts, void* stream,
                             unsigned flags);

/* sample_batch fused with build_sequence_batch (sequence.cpp:55-86), i.e. the pair
 * forward_concat runs (training.cpp:211-214), without materialising NeighborSamples.
 * Outputs [q, l] row-major: node_index / edge_index int32 (ids + 1, 0 = padding),
 * dt32 = float(t_q - ts) rounded from the fp64 difference, dt64 the exact fp64 delta
 * (either may be NULL), valid_len[q] int32 (target_row = valid_len - 1).
 * ids must satisfy num_nodes < 2^31 - 1 and edge_id + 1, self_edge_index < 2^31, else
 * TGFX_EUNSUPPORTED (use the _device variant with TGFX_INDEX64). */
int tgfx_sample_assemble(const tgfx_graph* g, const int64_t* nodes, const double* times,
                         int64_t q, int64_t k, int strategy, uint64_t seed,
                         uint64_t stream_base, int64_t l, int64_t self_edge_index,
                         int32_t* node_index, int32_t* edge_index, float* dt32, double* dt64,
                         int32_t* valid_len);
/* build_sequence_batch(sample_batch(g, nodes, times, k, strategy, seed), l, self_edge_index)
 * in the reference's own SequenceBatch types (sequence.hpp:20-30): node_index / edge_index
 * int64 [q, l], time_delta double [q, l], valid_len / target_row int64 [q].  Errors in the
 * reference's order: every query node, then k (sampler.cpp:88-93), then l (sequence.cpp:57).
 * Backs tgf::sample_sequence_batch, the one-call form of forward_concat's pair
 * (training.cpp:211-214). */
int tgfx_sample_sequence_batch(const tgfx_graph* g, const int64_t* nodes, const double* times,
                               int64_t q, int64_t k, int strategy, uint64_t seed,
                               uint64_t stream_base, int64_t l, int64_t self_edge_index,
                               int64_t* node_index, int64_t* edge_index, double* time_delta,
                               int64_t* valid_len, int64_t* target_row);
/* tgfx_sample_assemble_device with the query check fused into the sampler kernel
 * (check_query, proj/src/sampler.cpp:22-27, called for every query by sample_batch :93):
 * instead of a separate validation pass and a synchronisation, the kernel compares each
 * query node with [0, num_nodes) as it loads it and atomically lowers *d_first_bad (a device
 * word the caller sets to ~0 beforehand) to stream_base + the first failing query index.
 * Asynchronous; rows of failing queries are written as absent ones (all zero, valid_len 0)
 * and, unlike sample_batch, the other rows are written too -- the caller raises the error
 * with tgfx_query_error before using them (any number of calls may share one word). */
int tgfx_sample_assemble_checked_device(const tgfx_graph* g, const int64_t* d_nodes,
                                        const double* d_times, int64_t q, int64_t k,
                                        int strategy, uint64_t seed, uint64_t stream_base,
                                        int64_t l, int64_t self_edge_index, void* d_node_index,
                                        void* d_edge_index, float* d_dt32, double* d_dt64,
                                        void* d_valid_len, unsigned long long* d_first_bad,
                                        void* stream, unsigned flags);
/* Reads *d_first_bad (synchronising `stream`): TGFX_OK if no query failed, else
 * TGFX_EVALIDATION with the reference's text "query node <u> out of range" (sampler.cpp:24),
 * u read from d_nodes[first_bad - stream_base] (d_nodes = the failing call's query nodes). */
int tgfx_query_error(const int64_t* d_nodes, uint64_t stream_base,
                     const unsigned long long* d_first_bad, void* stream);
/* device variant; with TGFX_INDEX64 the node_index / edge_index / valid_len pointers are
 * int64_t* (the reference's SequenceBatch types). */
int tgfx_sample_assemble_device(const tgfx_graph* g, const int64_t* d_nodes,
                                const double* d_times, int64_t q, int64_t k, int strategy,
                                uint64_t seed, uint64_t stream_base, int64_t l,
                                int64_t self_edge_index, void* d_node_index, void* d_edge_index,
                                float* d_dt32, double* d_dt64, void* d_valid_len, void* stream,
                                unsigned flags);

/* Many forward_concat batches in one launch (an epoch of training.cpp:211-214 calls): the q
 * queries are consecutive batches of batch_q; batch b is sampled exactly as
 * sample_batch(..., seed = d_seeds[b]) would (uniform RNG stream = index within the batch,
 * sampler.cpp:100-101) and packed as build_sequence_batch.  d_seeds: device array of
 * ceil(q / batch_q) seeds (may be NULL for TGFX_RECENT).  Flags as tgfx_sample_assemble_device. */
int tgfx_sample_assemble_batched_device(const tgfx_graph* g, const int64_t* d_nodes,
                                        const double* d_times, int64_t q, int64_t batch_q,
                                        int64_t k, int strategy, const uint64_t* d_seeds,
                                        int64_t l, int64_t self_edge_index, void* d_node_index,
                                        void* d_edge_index, float* d_dt32, double* d_dt64,
                                        void* d_valid_len, void* stream, unsigned flags);

/* 2-hop composition (not in the reference): hop-1 = sample_batch(roots,
 * k1) rows [q, l]; hop-2 rows [q, k1, l]: slot j of root r holds the row of the query
 * (nbr_j, ts_j) of hop-1 entry j (recent-k2, or sample_random(seed2, stream = r*k1 + j));
 * absent slots are all zero with valid_len 0. */
int tgfx_sample_two_hop_device(const tgfx_graph* g, const int64_t* d_roots,
                               const double* d_times, int64_t q, int64_t k1, int64_t k2,
                               int strategy, uint64_t seed, uint64_t seed2, int64_t l,
                               int64_t self_edge_index, int32_t* d_hop1_node,
                               int32_t* d_hop1_edge, float* d_hop1_dt, int32_t* d_hop1_len,
                               int32_t* d_hop2_node, int32_t* d_hop2_edge, float* d_hop2_dt,
                               int32_t* d_hop2_len, void* stream, unsigned flags);
int tgfx_sample_two_hop(const tgfx_graph* g, const int64_t* roots, const double* times,
                        int64_t q, int64_t k1, int64_t k2, int strategy, uint64_t seed,
                        uint64_t seed2, int64_t l, int64_t self_edge_index,
                        int32_t* hop1_node, int32_t* hop1_edge, float* hop1_dt,
                        int32_t* hop1_len, int32_t* hop2_node, int32_t* hop2_edge,
                        float* hop2_dt, int32_t* hop2_len);

/* ---------------------------------------------------------------- sequences */
/* replaces tgf::build_sequence_batch (sequence.hpp:45-46, sequence.cpp:55-86) over padded
 * samples [q, kpad] (counts[q] valid entries each), in the reference's types. */
int tgfx_assemble(int64_t q, int64_t kpad, const int64_t* counts, const int64_t* nbr,
                  const int64_t* eid, const double* ts, const int64_t* query_nodes,
                  const double* query_times, int64_t l, int64_t self_edge_index,
                  int64_t* node_index, int64_t* edge_index, double* time_delta,
                  int64_t* valid_len, int64_t* target_row);
/* tgfx_assemble over tgfx_neighbor records [q, kpad] (tgf::build_sequence_batch's NeighborSamples
 * packed as they are laid out in memory) */
int tgfx_assemble_records(int64_t q, int64_t kpad, const int64_t* counts,
                          const tgfx_neighbor* entries, const int64_t* query_nodes,
                          const double* query_times, int64_t l, int64_t self_edge_index,
                          int64_t* node_index, int64_t* edge_index, double* time_delta,
                          int64_t* valid_len, int64_t* target_row);
/* replaces tgf::build_mask (sequence.hpp:50, sequence.cpp:93-111): (q*l) x l doubles */
int tgfx_build_mask(int64_t q, int64_t l, const int64_t* valid_len, const int64_t* target_row,
                    int kind, double* mask);

/* replaces tgf::assemble_inputs (proj/src/attention.cpp:414-451), the sequence tensors' first
 * consumer: z [q*l, d] with, for j < valid_len[b], row b*l+j =
 *   combine sum (concat = 0; d = d_v = d_e = d_t):
 *     node_table[ni] + edge_table[ei] + cos(omega * dt + phi)
 *   combine concat (concat = 1; d = d_v + d_e + d_t):
 *     [node_table[ni] | edge_table[ei] | cos(omega * dt + phi)]
 * and zero rows for padding.  Indices int32 (index64 = 0: the sampler's compact outputs) or
 * int64; time_delta f32/f64 (dt_type); tables f32/f64 (table_type); omega, phi: f64 [d_t];
 * z f32/f64/bf16 (z_type); the encoding is computed in f64 and rounded once.  An index outside
 * its table: TGFX_EVALIDATION "sequence index outside embedding tables". */
int tgfx_assemble_inputs_device(int64_t q, int64_t l, const void* d_node_index,
                                const void* d_edge_index, const void* d_time_delta,
                                const void* d_valid_len, int index64, int dt_type,
                                const void* d_node_table, int64_t node_rows,
                                const void* d_edge_table, int64_t edge_rows, int table_type,
                                const double* d_omega, const double* d_phi, int64_t d_v,
                                int64_t d_e, int64_t d_t, int concat, void* d_z, int z_type,
                                void* stream, unsigned flags);

/* forward_concat's sampling, sequence assembly and model_forward's assemble_inputs
 * (training.cpp:211-214, attention.cpp:414-451) in one call: z [q*l, d] of the sampled
 * sequences (d = d_t for combine sum, d_v + d_e + d_t for concat), as
 * tgfx_assemble_inputs_device(tgfx_sample_assemble_device(...)) with fp64 time deltas
 * computes it.  Recent-k on line-probe graphs runs ONE kernel (the index / delta rows never
 * reach HBM); other cases compose the two on the device.  d_valid_len (int32 [q]) optional.
 * Validation as tgfx_sample_assemble_device, plus the reference's "sequence index outside
 * embedding tables". */
int tgfx_sample_inputs_device(const tgfx_graph* g, const int64_t* d_nodes, const double* d_times,
                              int64_t q, int64_t k, int strategy, uint64_t seed,
                              uint64_t stream_base, int64_t l, int64_t self_edge_index,
                              const void* d_node_table, int64_t node_rows,
                              const void* d_edge_table, int64_t edge_rows, int table_type,
                              const double* d_omega, const double* d_phi, int64_t d_v,
                              int64_t d_e, int64_t d_t, int concat, void* d_z, int z_type,
                              int32_t* d_valid_len, void* stream, unsigned flags);

/* ---------------------------------------------------------------- CSV ingestion */
/* replaces tgf::load_csv (event_stream.hpp:44, event_stream.cpp:85-154): reads the file,
 * parses it on the device (header required; rows "src,dst,timestamp[,features]"), stable
 * sorts by timestamp and numbers the events 0..n-1 in that order; num_nodes = max id + 1.
 * Errors carry the reference's exception type and text (TGFX_EVALIDATION / TGFX_EPARSE).
 * Reals are parsed correctly rounded (from_chars); a literal with > 19 significant digits
 * whose rounding needs big-integer arithmetic, or a NaN timestamp, is TGFX_EUNSUPPORTED. */
int tgfx_load_csv(const char* path, int has_features, tgfx_csv** out);
/* same, from CSV bytes already on the device */
int tgfx_csv_parse_device(const char* d_bytes, int64_t nbytes, int has_features, void* stream,
                          tgfx_csv** out);
int tgfx_csv_info(const tgfx_csv* c, int64_t* num_events, int64_t* num_nodes, int64_t* d_e);
/* device views: events [n] (feed tgfx_build_device directly), features [n * d_e] or NULL */
int tgfx_csv_device_arrays(const tgfx_csv* c, const tgfx_event** events, const double** features);
/* host copies (features may be NULL) */
int tgfx_csv_export(const tgfx_csv* c, tgfx_event* events, double* features);
int tgfx_csv_free(tgfx_csv* c);
/* parse n fields d_bytes[d_off[i] .. d_off[i+1]) as int64 (kind 0) or double (kind 1) with
 * std::from_chars semantics; d_status[i] 0 ok, 1 bad, 2 unsupported (see tgfx_load_csv) */
int tgfx_parse_numbers_device(const char* d_bytes, const int64_t* d_off, int64_t n, int kind,
                              int64_t* d_int, double* d_real, int* d_status, void* stream);

/* ---------------------------------------------------------------- synthetic inputs */
/* bit-identical to tgf::make_random_stream (synthetic.hpp:17-18, synthetic.cpp:12-43);
 * the Zipf CDF is computed on the host with glibc pow as the reference does. */
int tgfx_make_random_stream(int64_t num_edges, int64_t num_nodes, uint64_t seed,
                            double zipf_exponent, tgfx_event* out);
int tgfx_make_random_stream_device(int64_t num_edges, int64_t num_nodes, uint64_t seed,
                                   double zipf_exponent, tgfx_event* d_out, void* stream);
/* forward_concat query layout (training.cpp:193-209) for events [e0, e1): per batch of B
 * events [src | dst | neg], neg_i = CounterRng(neg_seed, i).next_below(num_nodes)
 * (index-keyed, metrics.cpp:68-69).  Writes 3*(e1-e0) queries. */
int tgfx_make_queries_device(const tgfx_event* d_events, int64_t e0, int64_t e1,
                             int64_t batch, int64_t num_nodes, uint64_t neg_seed,
                             int64_t* d_nodes, double* d_times, void* stream);
/* The sample_batch queries of one training epoch, on the device: make_batches
 * (proj/src/training.cpp:157-182: batches of batch_size consecutive events of the training
 * stream, negatives CounterRng(batch_seed, batch).next_below(num_nodes), neg_per_pos per
 * event) split as train_epoch does (:425-440, min(workers, b) shards [h*b/m, (h+1)*b/m)), each
 * shard in forward_concat's layout (:193-209) [src | dst | neg] -- one contiguous block per
 * sample_batch call, calls in (batch, shard) order.  Batches [b0, b1) of the n-event stream;
 * writes (min(n, b1*B) - b0*B) * (2 + neg_per_pos) queries.  batch_seed is make_batches'
 * seed (train_epoch passes tgfx_mix_streams(cfg.seed, 0x6e67, epoch), :422-423). */
int tgfx_make_train_queries_device(const tgfx_event* d_events, int64_t n, int64_t b0, int64_t b1,
                                   int64_t batch_size, int64_t neg_per_pos, int64_t workers,
                                   int64_t num_nodes, uint64_t batch_seed, int64_t* d_nodes,
                                   double* d_times, void* stream);
/* training.cpp:16-18 mix_streams: train_epoch's seeds -- make_batches seed
 * (cfg.seed, 0x6e67, epoch) and the sample seed of step s, shard h
 * (cfg.seed, epoch * 0x10001 + s, h), :445-446. */
uint64_t tgfx_mix_streams(uint64_t a, uint64_t b, uint64_t c);

#ifdef __cplusplus
}
#endif
#endif /* TGFX_H */
