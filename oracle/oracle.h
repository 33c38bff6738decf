/*
 * oracle.h -- CPU restatement of the reference (tgformer, arXiv 2409.05477) hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library, and only as the checker
 * or the CPU baseline -- never as the product path.  The product (libtgfx.so) has no
 * CPU fallback and never links or calls anything here.
 *
 * Parity pin: restated functions are checked against golden vectors produced by running
 * the reference itself (oracle/_ref, built from /root/reference/proj/src by
 * oracle/Makefile); see tests/golden/gen_golden.py and tests/test_oracle_golden.py.
 *
 * Every function cites the reference file:line it restates (paths relative to
 * /root/reference/).
 */
#ifndef TGFX_ORACLE_H
#define TGFX_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* proj/include/tgformer/event_stream.hpp:13-18 (TemporalEvent, 32 bytes) */
typedef struct orc_event {
  int64_t edge_id;
  int64_t src;
  int64_t dst;
  double timestamp;
} orc_event;

/* proj/include/tgformer/rng.hpp:11-16 */
uint64_t orc_mix64(uint64_t x);
/* proj/include/tgformer/rng.hpp:23-24: initial state of CounterRng(seed, stream) */
uint64_t orc_rng_state(uint64_t seed, uint64_t stream);
/* d-th next_u64() of CounterRng(seed, stream) (rng.hpp:26-32), by skip-ahead */
uint64_t orc_rng_draw(uint64_t state0, uint64_t d);
/* proj/include/tgformer/rng.hpp:35-38 (Lemire multiply-high) */
uint64_t orc_mulhi64(uint64_t a, uint64_t b);

/* proj/src/synthetic.cpp:12-43.  out has num_edges entries. Returns 0, or 1 on bad dims. */
int orc_make_random_stream(int64_t num_edges, int64_t num_nodes, uint64_t seed,
                           double zipf_exponent, orc_event* out);
/* The Zipf CDF of synthetic.cpp:16-22 alone (num_nodes doubles). */
void orc_zipf_cdf(int64_t num_nodes, double zipf_exponent, double* cdf);

/* proj/src/tcsr.cpp:83-105 (build_sequential) incl. check_endpoints (tcsr.cpp:44-50) and
 * finish (tcsr.cpp:26-42).  indptr[V+1]; nbr/eid/ts [n*(1+reverse)].
 * Returns 0, or 1 (ValidationError) with *bad_edge_id = edge_id of the first bad event. */
int orc_build(const orc_event* ev, int64_t n, int64_t num_nodes, int reverse, int64_t* indptr,
              int64_t* nbr, int64_t* eid, double* ts, int64_t* bad_edge_id);

/* proj/src/tcsr.cpp:54-81 (TCsr::validate). Returns 0 ok, 1 invalid. */
int orc_validate(int64_t num_nodes, int64_t num_edges, int64_t m, const int64_t* indptr,
                 const int64_t* nbr, const int64_t* eid, const double* ts);

/* proj/src/sampler.cpp:16-20 (prefix_end: lower_bound, strict ts < t) */
int64_t orc_prefix_end(const int64_t* indptr, const double* ts, int64_t u, double t);

/* proj/src/sampler.cpp:41-52 / :54-82.  Write the chosen absolute entry positions to
 * pos_out (capacity k) and return their count. */
int64_t orc_sample_recent(const int64_t* indptr, const double* ts, int64_t u, double t,
                          int64_t k, int64_t* pos_out);
int64_t orc_sample_random(const int64_t* indptr, const double* ts, int64_t u, double t,
                          int64_t k, uint64_t seed, uint64_t stream, int64_t* pos_out);

/* proj/src/sampler.cpp:84-104 (sample_batch); validation of every query first
 * (sampler.cpp:88-93).  Outputs padded [Q, k]: counts[Q], nbr/eid/ts[Q*k] (unused slots 0).
 * stream of query i = stream_base + i (stream_base = 0 reproduces the reference).
 * Returns 0, 1 = bad node (*bad_node set), 2 = k < 1. */
int orc_sample_batch(int64_t num_nodes, const int64_t* indptr, const int64_t* nbr,
                     const int64_t* eid, const double* ts, const int64_t* nodes,
                     const double* times, int64_t q, int64_t k, int strategy, uint64_t seed,
                     uint64_t stream_base, int64_t* counts, int64_t* nbr_out, int64_t* eid_out,
                     double* ts_out, int64_t* bad_node);

/* proj/src/sequence.cpp:55-86 (build_sequence_batch) over padded samples [Q, kpad].
 * node_index/edge_index int64 [Q*l], time_delta double [Q*l], valid_len/target_row [Q].
 * Returns 0 or 1 (l < 2). */
int orc_build_sequence_batch(int64_t q, int64_t kpad, const int64_t* counts,
                             const int64_t* nbr, const int64_t* eid, const double* ts,
                             const int64_t* query_nodes, const double* query_times, int64_t l,
                             int64_t self_edge_index, int64_t* node_index, int64_t* edge_index,
                             double* time_delta, int64_t* valid_len, int64_t* target_row);

/* proj/src/sequence.cpp:93-111 (build_mask), kind 0 causal, 1 tgat, 2 self_loop.
 * mask is (Q*l) x l doubles. */
void orc_build_mask(int64_t q, int64_t l, const int64_t* valid_len, const int64_t* target_row,
                    int kind, double* mask);

/* Query layout of forward_concat (proj/src/training.cpp:193-209) for events [e0, e1):
 * per batch of B consecutive events: [src(B) | dst(B) | neg(B)], neg of event i =
 * CounterRng(neg_seed, i).next_below(V) (index-keyed as proj/src/metrics.cpp:68-69).
 * Writes 3*(e1-e0) queries. */
void orc_make_queries(const orc_event* ev, int64_t e0, int64_t e1, int64_t batch,
                      int64_t num_nodes, uint64_t neg_seed, int64_t* nodes, double* times);

#ifdef __cplusplus
}
#endif
#endif
