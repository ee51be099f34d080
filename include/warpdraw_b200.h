/*
 * warpdraw_b200.h -- C ABI of the B200 (sm_100a) butterfly sampler.
 *
 * Drop-in boundary for the reference package `warpdraw`
 * (/root/reference/pkg/src/warpdraw).  The reference is pure Python; its
 * plugin surface for this path is the kernel registry
 *   KERNELS / draw_z(kernel, N, theta, phi, w, config, stops)   kernels.py:542-555
 * and the sampler registry
 *   SAMPLERS[name](weights, n, seed)                            bench.py:150-154
 * The Python package paper_1505_03851_b200 binds these entry points with
 * ctypes (INTEGRATION.md shows the binding) and keeps those signatures.
 *
 * Conventions
 *   - every pointer argument is a DEVICE pointer unless stated otherwise;
 *   - every call is stream-ordered on `stream` (a cudaStream_t, NULL = legacy
 *     default stream) and returns immediately with a status (WD_OK = 0);
 *   - the library never allocates device memory: scratch comes from the
 *     caller through (workspace, workspace_bytes), sized by wd_workspace_bytes;
 *   - data errors are reported through `err` (2 x uint64, device):
 *       err[0] = smallest "first encountered" ordering key of a token whose
 *                products sum to zero (AllZeroError, kernels.py:397-398 and
 *                421-425), UINT64_MAX if none.  Key layout:
 *                  WD_KEYS_MASTER   : (doc/lanes) << 40 | word << 8 | doc%lanes
 *                  WD_KEYS_POSITION : doc << 32 | word
 *                  rows             : row id
 *       err[1] = 0 if an explicit stop was out of range (StopOutOfRangeError,
 *                kernels.py:329-331), else UINT64_MAX.
 *     The library resets err at the start of each call.
 *
 * Arithmetic: IEEE binary32 / binary64, round-to-nearest, no FMA contraction,
 * no flush-to-zero.  The butterfly variant reproduces the reference's
 * per-token floating-point operations exactly (block sums as the balanced
 * pairwise tree of the log2(W) shuffle_xor sets, sequential block and
 * remnant accumulation, add-or-subtract reconstruction chosen by the bits of
 * doc mod W), so z is bit-identical to draw_z_butterfly / build_block_tables
 * + butterfly_search; the prefix variant is bit-identical to draw_z_basic /
 * draw_z_transposed.
 */
#ifndef WARPDRAW_B200_H
#define WARPDRAW_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define WD_OK 0
#define WD_ERR_INVALID_ARGUMENT 1
#define WD_ERR_CUDA 2
#define WD_ERR_UNSUPPORTED 3
#define WD_ERR_WORKSPACE 4

/* element type of theta / phi / weights / explicit stops */
#define WD_FLOAT32 0
#define WD_FLOAT64 1
/* wd_draw_z only: float32 theta (and table, explicit stops) with float64 phi;
 * every product is fl32(fl64(theta * phi)) as the reference's numpy
 * promotion forms it (kernels.py:209, 391) */
#define WD_FLOAT32_PHI64 2

/* table variant */
#define WD_BUTTERFLY 0 /* draw_z_butterfly (kernels.py:487-539)                 */
#define WD_PREFIX 1    /* draw_z_basic / draw_z_transposed (kernels.py:380-484) */

/* where the unit u of each draw comes from */
#define WD_STOPS_SEEDED 0   /* SeededStops: u = units_for(seed, doc, key) (rng.py:101-122) */
#define WD_STOPS_UNITS 1    /* InjectedStops: u = units[token] (float64)       */
#define WD_STOPS_EXPLICIT 2 /* stop values given directly (search entry points) */
#define WD_STOPS_PHILOX 3   /* opt-in Philox4x32-10 stream; NOT reference-parity */

/* hash key of the last word of a short document under WD_STOPS_SEEDED */
#define WD_KEYS_MASTER 0   /* master-index loop: key G_q-1 (kernels.py:520-536)  */
#define WD_KEYS_POSITION 1 /* basic kernel: key = word position (kernels.py:389) */

/* Version of this ABI. */
int wd_abi_version(void);

/* Human-readable status text (static storage). */
const char* wd_status_string(int status);

/* Text of the last CUDA error seen by this library in this thread. */
const char* wd_last_cuda_error(void);

/*
 * Per-corpus preparation (replaces Corpus.padded bookkeeping, lda.py:56-63,
 * and the master-index loop state, kernels.py:520-536).
 *   doc_offsets [n_docs+1] int64 CSR offsets of the local shard.
 *   token_doc   [n_tokens] int32 out: local doc of every token.
 *   last_key    [n_docs]   int32 out: G_q - 1 for every doc, G_q = max length
 *               over its `lanes`-doc group (groups taken in GLOBAL doc ids,
 *               doc_base + local; groups must not straddle the shard).
 */
int wd_corpus_prepare(const int64_t* doc_offsets, int64_t n_docs, int64_t n_tokens,
                      int64_t doc_base, int lanes, int32_t* token_doc, int32_t* last_key,
                      void* stream);

/*
 * Scratch bytes wd_draw_z / wd_sample_rows need.  WD_PREFIX: the per-lane
 * prefix tables.  WD_BUTTERFLY: none is required; with at least this much,
 * wd_sample_rows on ONE shared weight vector (ld = 0) builds the butterfly
 * table once and answers every draw by search (bench.py:129-147), instead
 * of re-reading the vector per draw -- same results either way.
 */
size_t wd_workspace_bytes(int variant, int dtype, int lanes, int32_t n_topics);

/*
 * LDA z draw over a CSR corpus shard: replaces kernels.draw_z for the kernels
 * "butterfly" (variant WD_BUTTERFLY) and "basic"/"transposed" (WD_PREFIX).
 *   theta [n_docs x n_topics] (leading dim ld_theta), phi [V x n_topics]
 *   (leading dim ld_phi), dtype WD_FLOAT32/WD_FLOAT64, row-major.
 *   words / token_doc [n_tokens] int32; last_key from wd_corpus_prepare
 *   (only read for WD_STOPS_SEEDED + WD_KEYS_MASTER).
 *   token_pos: NULL for tokens in CSR order.  Otherwise words / token_doc /
 *   token_pos describe a PERMUTED token list (e.g. one vocabulary tile of a
 *   tiled corpus): list entry j is word token_pos[j] of document token_doc[j],
 *   and its original CSR index doc_offsets[doc] + pos is where z, units and
 *   stops are indexed.  n_tokens is then the length of the list.
 *   doc_base = global id of local doc 0 (hash key and doc mod lanes).
 *   units [n_tokens] float64 (WD_STOPS_UNITS) or stops [n_tokens] dtype
 *   (WD_STOPS_EXPLICIT); seed = derive_seed(seed, 1, iteration) (lda.py:228).
 *   z [n_tokens] int32 out.  word_topic [V x n_topics] / doc_topic
 *   [n_docs x n_topics] int32: optional (NULL = skip) fused count update
 *   (+= 1 per token, lda.py:174-182); the caller zeroes them.
 *   Load width follows the alignment of the W-topic block starts (pointer,
 *   leading dimension, n_topics mod lanes): 32-byte aligned fp32 blocks at
 *   lanes = 32 use 256-bit segments, 16-byte aligned ones 128-bit segments
 *   (fp64: 32-byte), others scalar loads -- identical results.
 *   Token-list entries with token_pos < 0 are padding slots: loaded, never drawn.
 */
int wd_draw_z(int variant, int dtype, int lanes, const void* theta, int64_t ld_theta,
              const void* phi, int64_t ld_phi, int32_t n_topics, const int64_t* doc_offsets,
              const int32_t* words, const int32_t* token_doc, const int32_t* token_pos,
              const int32_t* last_key, int64_t n_docs, int64_t n_tokens, int64_t doc_base,
              int stop_mode, int key_rule,
              uint64_t seed, const double* units, const void* stops, int32_t* z,
              int32_t* word_topic, int32_t* doc_topic, uint64_t* err, void* workspace,
              size_t workspace_bytes, void* stream);

/*
 * Independent categorical rows: out[i] ~ weights[i, :] (ld = 0: one shared
 * weight vector for every row).  Row id = row_base + i selects u =
 * units_for(seed, id) (seed = derive_seed(user_seed, 6), bench.py:141-143)
 * and id mod lanes.  Equivalent to build_block_tables + butterfly_search
 * (kernels.py:580-600, 317-362) for WD_BUTTERFLY.
 */
int wd_sample_rows(int variant, int dtype, int lanes, const void* weights, int64_t ld,
                   int64_t n_rows, int32_t n_topics, int64_t row_base, int stop_mode,
                   uint64_t seed, const double* units, const void* stops, int32_t* out,
                   uint64_t* err, void* workspace, size_t workspace_bytes, void* stream);
/*
 * wd_sample_rows with flags.  WD_ERR_ACCUMULATE: err is NOT reset to
 * all-ones first -- errors of consecutive calls accumulate (min key, and of
 * the range flags) until the caller resets the two words itself (one
 * memset for a batch of draws; a per-call reset is a separate stream
 * operation, ~4-5 us, as long as a 2^20-row draw at K <= 32).
 */
#define WD_ERR_ACCUMULATE 1
int wd_sample_rows_ex(int variant, int dtype, int lanes, const void* weights, int64_t ld,
                      int64_t n_rows, int32_t n_topics, int64_t row_base, int stop_mode,
                      uint64_t seed, const double* units, const void* stops, int32_t* out,
                      uint64_t* err, void* workspace, size_t workspace_bytes, int flags, void* stream);

/* units_for(seed, k0[i][, k1[i]]) for n_keys in {0,1,2} (rng.py:101-122). */
int wd_units(uint64_t seed, int n_keys, const int64_t* k0, const int64_t* k1, int64_t n,
             double* out, void* stream);

/* topic_counts (lda.py:174-182): doc_topic / word_topic (+= 1, int32, either
 * may be NULL) from z; the caller zeroes them first. */
int wd_topic_counts(const int32_t* words, const int32_t* token_doc, const int32_t* z,
                    int64_t n_tokens, int32_t n_topics, int32_t* doc_topic,
                    int32_t* word_topic, void* stream);


/*
 * Throughput-mode Dirichlet resample (lda.py:185-208), statistical parity:
 * every Gamma attempt is one Philox4x32-10 block of counter (row lo, row hi,
 * topic, attempt) under the 64-bit iteration seed, Marsaglia-Tsang in log
 * space, deterministic reductions.
 *   wd_resample_theta: theta[m, :] ~ Dir(alpha + histogram of z over doc m)
 *     (the doc-topic counts are formed in shared memory, never in HBM);
 *     row key = doc_base + m.
 *   wd_resample_phi: phi[:, k] ~ Dir(beta + word_topic[:, k]); word_topic is
 *     [vocab_size x n_topics] int32 (dense, ld = n_topics); scratch of
 *     wd_resample_phi_workspace_bytes(n_topics) bytes.
 */
/* The Gamma stream of the resample kernels, cell by cell: out[i] = log of
 * the Gamma(shapes[i], 1) draw the resample kernels make for (rows[i],
 * topics[i]) under `seed` (same attempts, same arithmetic).  Test/KAT entry
 * (replaces numpy's Generator.gamma at lda.py:201-205). */
int wd_log_gamma_draws(uint64_t seed, const int64_t* rows, const int32_t* topics, const float* shapes,
                       int64_t n, float* out, void* stream);

int wd_resample_theta(int dtype, const int32_t* z, const int64_t* doc_offsets, int64_t n_docs,
                      int32_t n_topics, double alpha, uint64_t seed, int64_t doc_base, void* theta,
                      int64_t ld_theta, void* stream);
size_t wd_resample_phi_workspace_bytes(int32_t n_topics);
int wd_resample_phi(int dtype, const int32_t* word_topic, int64_t vocab_size, int32_t n_topics,
                    double beta, uint64_t seed, void* phi, int64_t ld_phi, void* workspace,
                    size_t workspace_bytes, void* stream);
/*
 * The same phi resample split for a document-sharded multi-GPU run (the
 * ranks hold identical all-reduced counts): the V rows are cut into
 * wd_resample_phi_chunks() fixed chunks; pass p (0: Gammas + column maxima,
 * 1: exp + column sums, 2: normalise) runs chunks [chunk0, chunk1) and writes
 * their column partials [n_chunks][K]; after each of passes 0 and 1 the
 * ranks exchange partials (all-gather) and wd_resample_phi_reduce folds all
 * n_chunks partials in chunk order into colstat[2K] (maxima, sums).  Every
 * rank then holds the same column statistics, its own rows of phi are
 * bit-identical to wd_resample_phi's, and an all-gather of the rows
 * completes phi (device_lda.DeviceLDA, sharded resample).
 */
int wd_resample_phi_chunks(void);
int wd_resample_phi_pass(int dtype, int pass, const int32_t* word_topic, int64_t vocab_size, int32_t n_topics,
                         double beta, uint64_t seed, void* phi, int64_t ld_phi, int chunk0, int chunk1, int n_chunks,
                         float* partials, const float* colstat, void* stream);
int wd_resample_phi_reduce(int pass, const float* partials, int n_chunks, int32_t n_topics, float* colstat,
                           void* stream);

/*
 * log_likelihood (lda.py:289-305): *out = sum over tokens of
 * log(theta_hat[doc] . phi_hat[word]) with row-normalised theta and
 * column-normalised phi, accumulated in float64.  Scratch: (n_docs +
 * n_topics) * 8 bytes.
 */
int wd_log_likelihood(int dtype, const void* theta, int64_t ld_theta, const void* phi, int64_t ld_phi,
                      const int32_t* words, const int32_t* token_doc, int64_t n_docs, int64_t n_tokens,
                      int64_t vocab_size, int32_t n_topics, double* out, void* workspace,
                      size_t workspace_bytes, void* stream);

/*
 * Sequential-stream samplers: the reference's SAMPLERS["binary"] and
 * SAMPLERS["alias"] (bench.py:118-126), one shared weight vector, n draws
 * taken in order from ONE xoshiro256** stream seeded by SplitMix64 from
 * `seed` (rng.py:47-77; seed = derive_seed(user_seed, 4) resp. (…, 5)).
 * Every thread starts at its own stream position through GF(2) jump
 * matrices built on the device, so draw i equals the reference's i-th draw.
 *   WD_STREAM_BINARY: stop = table[K-1] * u; smallest j with stop < table[j]
 *     (sampling.py:55-92); table = float64 running sums (wd_prefix_f64).
 *   WD_STREAM_ALIAS:  k = trunc(u1 * K); k if bits(u2) < thresh[k] else
 *     alias[k] (sampling.py:134-138); thresh[k] = ceil(F[k] * 2^53) of the
 *     exact Vose acceptance F[k] (sampling.py:101-131), so the 53-bit
 *     comparison is exactly the reference's float-vs-Fraction one.
 * Scratch: wd_stream_workspace_bytes(n) bytes.
 */
#define WD_STREAM_BINARY 0
#define WD_STREAM_ALIAS 1
int wd_prefix_f64(const double* weights, int64_t n_weights, double* table, void* stream);
size_t wd_stream_workspace_bytes(int64_t n_draws);
int wd_stream_draws(int method, const double* table, const uint64_t* thresh, const int32_t* alias,
                    int64_t n_weights, uint64_t seed, int64_t n_draws, int32_t* out, void* workspace,
                    size_t workspace_bytes, void* stream);

/*
 * Measurement (no reference counterpart): the L2 -> SM read ceiling the
 * vocabulary-tiled LDA draw runs against.  `reps` grid-stride sweeps of
 * 256-bit ld.global.cg loads over a 32-byte-aligned, L2-resident buffer;
 * wd_l2_probe_bytes(buffer_bytes, blocks) = bytes read per sweep.
 */
int64_t wd_l2_probe_bytes(int64_t buffer_bytes, int blocks);
int wd_l2_read_probe(const void* buffer, int64_t buffer_bytes, int reps, int blocks, float* sink, void* stream);

/*
 * The reference's split table / search API (the draw entry points fuse the
 * two; these materialise the table exactly as the reference stores it).
 *
 * wd_build_block_tables replaces build_block_tables (kernels.py:580-600 ->
 * build_butterfly_table, kernels.py:170-225): products [G][W][K] (each of
 * the G warp groups holds W lanes' product rows; theta_local := products,
 * phi := 1) -> p [K][G][W] (the butterfly-patterned table: lane-own
 * remnant running sums, then per W-topic block the rows stored by the
 * log2(W) shuffle_xor sets and the running total in row W-1) and
 * sums [G][W].
 *
 * wd_butterfly_search replaces butterfly_search (kernels.py:317-362) with
 * _butterfly_block_walk (kernels.py:268-314): block bisection over each
 * lane's block-final rows, the cross-lane fetch walk, the remnant fallback;
 * out [G][W] int64 indices.  err[2] as in wd_draw_z: err[1] == 0 when a
 * stop lies outside [0, sums) (StopOutOfRangeError, kernels.py:329-331).
 * lanes: 2..64.  dtype: WD_FLOAT32 / WD_FLOAT64.  Device pointers.
 */
int wd_build_block_tables(int dtype, int lanes, const void* products, int32_t n_topics, int64_t n_groups, void* p,
                          void* sums, void* stream);
int wd_butterfly_search(int dtype, int lanes, const void* p, const void* sums, const void* stops, int32_t n_topics,
                        int64_t n_groups, int64_t* out, uint64_t* err, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* WARPDRAW_B200_H */
