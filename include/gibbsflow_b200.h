/*
 * gibbsflow_b200.h -- C ABI of the B200-native collapsed-Gibbs LDA hot path.
 *
 * This is the drop-in boundary for the reference package `gibbsflow`
 * (/root/reference/pkg/src/gibbsflow).  The reference has no FFI of its own:
 * its boundary is Python functions over numpy arrays with fixed dtypes
 * (SURVEY.md section 8b).  Each entry point below names the reference (or
 * SPEC.md) function whose contract it carries; the Python mirror in
 * paper_1803_04631_b200/ binds them with ctypes.
 *
 * Conventions
 *   - Every function returns an int status (GF_OK = 0).  On failure
 *     gf_last_error() returns a thread-local message whose text matches the
 *     reference exception text where the reference defines one.
 *   - Host arrays are BORROWED for the duration of the call (copied in or
 *     written out); the caller keeps ownership.  Dtypes match the reference
 *     dataclasses: Chunk (corpus.py:160-198), ThetaRows (model.py:20-47),
 *     PhiMatrix (model.py:50-80).
 *   - A gf_shard is bound to one CUDA device and one CUDA stream; calls on one
 *     shard must come from one host thread at a time.
 *   - No torch / CUDA types cross the boundary: streams and device pointers
 *     are passed as void*.
 */
#ifndef GIBBSFLOW_B200_H
#define GIBBSFLOW_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes -> gibbsflow.errors classes (errors.py:4-37) */
#define GF_OK 0
#define GF_ERR_OVERFLOW 1    /* CountOverflowError    errors.py:20  */
#define GF_ERR_SHAPE 2       /* ShapeMismatchError    errors.py:28  */
#define GF_ERR_CONSISTENCY 3 /* ConsistencyError      errors.py:32  */
#define GF_ERR_CAPACITY 4    /* CapacityError         errors.py:16  (device OOM) */
#define GF_ERR_TRAINING 5    /* TrainingError         errors.py:36  (CUDA failure) */
#define GF_ERR_VALUE 6       /* ValueError (bad argument) */
#define GF_ERR_PARTITION 7   /* PartitionError        errors.py:12  */
#define GF_ERR_EMPTY 8       /* EmptyDistributionError errors.py:24 */
#define GF_ERR_NODEVICE 9    /* no CUDA device: the product path refuses to run */
#define GF_ERR_FORMAT 10     /* CorpusFormatError     errors.py:8   (UCI input) */

const char* gf_last_error(void);
int gf_abi_version(void);
int gf_device_count(int* count_out);

/* ------------------------------------------------------------------ rng --
 * splitmix64 counter streams, bit-exact with rng.py:20-89. */
/* rng.py:45-53 stream_key(*parts) */
uint64_t gf_stream_key(const uint64_t* parts, int num_parts);
/* rng.py:110-114 Stream.uniforms(n) starting at `counter` */
int gf_stream_uniforms(uint64_t key, uint64_t counter, int64_t n, double* out);

/* --------------------------------------------------- corpus (host, C++) --
 * Native host preprocessing, bit-exact with corpus.py. */
/* corpus.py:210-237 greedy_boundaries -> bounds_out[2*C] = (lo, hi) pairs */
int gf_greedy_boundaries(const int64_t* doc_lengths, int64_t num_docs, int64_t num_chunks,
                         int64_t* bounds_out);
/* corpus.py:252-286, one chunk of partition(): inputs are the chunk's tokens in
 * corpus (doc-major) order; outputs are the Chunk arrays.  group_* must hold
 * V entries; *num_groups_out receives the used length. */
/* corpus.py:79-145 load_uci_bow / _read_bow_header: validate a UCI docword
 * file (header D, W, NNZ, then NNZ "docID wordID count" triples; same checks
 * and error texts) and count its tokens; header = {D, W, NNZ}. */
int gf_uci_scan(const char* docword_path, int64_t* header, int64_t* num_tokens);
/* ... and expand it into doc-major tokens (corpus.py:42-76 corpus_from_tokens:
 * stable document order, empty documents dropped, ids compacted). */
int gf_uci_tokens(const char* docword_path, int64_t num_tokens, int32_t* doc_ids, int32_t* word_ids,
                  int64_t* num_docs_out);

int gf_partition_chunk(const int32_t* doc_ids, const int32_t* word_ids, int64_t num_tokens,
                       int64_t doc_lo, int64_t doc_hi, int32_t vocab_size, int32_t num_topics,
                       uint64_t seed, int64_t chunk_id,
                       int32_t* out_doc_ids, int32_t* out_word_ids, uint16_t* out_assignments,
                       int32_t* group_words, int64_t* group_offsets, int64_t* group_sizes,
                       int64_t* num_groups_out, int64_t* dw_ptr, int64_t* dw_tok);
/* The same outputs as gf_partition_chunk, computed on device `device` (K4,
 * bit-identical; replaces corpus.py:240-287 for one chunk). */
int gf_partition_chunk_gpu(int device, const int32_t* doc_ids, const int32_t* word_ids, int64_t num_tokens,
                           int64_t doc_lo, int64_t doc_hi, int32_t vocab_size, int32_t num_topics,
                           uint64_t seed, int64_t chunk_id,
                           int32_t* out_doc_ids, int32_t* out_word_ids, uint16_t* out_assignments,
                           int32_t* group_words, int64_t* group_offsets, int64_t* group_sizes,
                           int64_t* num_groups_out, int64_t* dw_ptr, int64_t* dw_tok);

/* ------------------------------------------------ device shard context --
 * One document shard (= one Chunk, C = G, M = 1) resident in
 * HBM together with its theta rows and a phi replica. */
typedef struct gf_shard gf_shard;

/* SPEC.md:312-314 TrainConfig subset.  heavy_threshold: words whose GLOBAL
 * frequency exceeds it keep 32-bit phi columns, the rest 16-bit (the paper's
 * "short integer" phi, section 6.1.3, made overflow-proof).  Pass
 * 65535 for the hybrid layout, 0 for all-32-bit. */
int gf_shard_create(gf_shard** out, int device, int32_t num_topics, int32_t vocab_size,
                    double alpha, double beta, uint64_t seed, uint32_t heavy_threshold);
int gf_shard_destroy(gf_shard* shard);
/* run every kernel / copy of this shard on `cuda_stream` (a cudaStream_t) */
int gf_shard_set_stream(gf_shard* shard, void* cuda_stream);
/* Change the Dirichlet hyper-parameters and the Philox key of a loaded shard
 * (SamplerContext alpha / beta, TrainConfig.seed) without rebuilding it: the
 * next sample recomputes the word contexts.  Lets a caller that hands the same
 * Chunk to sampler.sample_chunk repeatedly keep one resident shard. */
int gf_shard_set_params(gf_shard* shard, double alpha, double beta, uint64_t seed);
/* global word frequencies (length V), identical on every rank: fixes the
 * hybrid phi layout so replicas can be summed elementwise.  Optional on one GPU
 * (defaults to the shard's own frequencies at load). */
int gf_shard_set_vocab(gf_shard* shard, const int64_t* global_word_freq);
/* Upload one Chunk (corpus.py:160-198): token arrays in word-group order,
 * its group directory (any order) and doc-word map.  Builds the (doc, word)
 * run list, the heavy-first slice schedule and the theta row capacities. */
int gf_shard_load(gf_shard* shard, int64_t doc_lo, int64_t doc_hi, int64_t num_tokens,
                  const int32_t* doc_ids, const int32_t* word_ids, const uint16_t* assignments,
                  int64_t num_groups, const int32_t* group_words, const int64_t* group_offsets,
                  const int64_t* group_sizes, const int64_t* dw_ptr, const int64_t* dw_tok);

/* K4, corpus.py:240-287 partition + corpus.py:201-207 _doc_word_map +
 * rng.py:20-89 initial topics, on the device: load a shard straight from the
 * DOC-MAJOR tokens of documents [doc_lo, doc_hi) (the Corpus slice
 * corpus.py:253-255), chunk id `chunk_id`.  Same shard as partition() +
 * gf_shard_load, without the host-side sort (stable CUB radix sorts by word
 * and by local doc, splitmix64 z0 in fp64). */
int gf_shard_load_tokens(gf_shard* shard, int64_t doc_lo, int64_t doc_hi, int64_t num_tokens,
                         const int32_t* doc_ids, const int32_t* word_ids, uint64_t seed, int64_t chunk_id);

/* model.py:142-161 rebuild_phi_replica: this shard's phi replica + n_k into the
 * sync buffer (overwritten). */
int gf_shard_rebuild_phi(gf_shard* shard);
/* model.py:109-124 rebuild_theta: theta rows of this shard from assignments.
 * Overflow (a count > 65535) reports GF_ERR_OVERFLOW at the next
 * gf_shard_check_errors with "document d: topic count c exceeds 16-bit range". */
int gf_shard_rebuild_theta(gf_shard* shard);
/* After the sync buffer holds the GLOBAL phi / n_k (single GPU: right after
 * rebuild_phi; multi-GPU: after the allreduce): refresh the Eq. 1
 * denominators 1/(n_k + V beta). */
int gf_shard_prepare(gf_shard* shard);
/* SPEC.md:359-367 sample_chunk (deferred mode, exclusion on, two uniforms):
 * resamples every assignment against the iteration-start theta / phi and
 * accumulates the fused log-likelihood partial of that
 * iteration-start model.  Philox4x32-10 keyed by (seed) with counter
 * (global doc, word, occurrence in the (doc, word) run, iteration). */
int gf_shard_sample(gf_shard* shard, uint32_t iteration);
/* SPEC.md:402-410 loglik_per_token numerator for the CURRENT theta / phi
 * (no draws): read it back with gf_shard_loglik_sum. */
int gf_shard_evaluate(gf_shard* shard);
/* Sampling phases (streamed sampling): split the slice schedule into P phases
 * of contiguous word groups, ~T/P tokens each, so the host can copy phase p's
 * assignments z[tok_begin, tok_end) (word-group order) while later phases
 * sample.  gf_shard_set_phases applies at the next load (default 1).
 * gf_shard_sample_phase(p) for p = 0..P-1 in order is one gf_shard_sample
 * (same draws, same loglik; the loglik reduction runs after phase P-1). */
int gf_shard_set_phases(gf_shard* shard, int num_phases);
/* Uneven phases: phase p holds the word groups starting below cuts[p] * T
 * (cumulative token fractions, strictly increasing, cuts[P-1] = 1.0), e.g.
 * halving sizes so only a small last phase's copies stay exposed. */
int gf_shard_set_phase_cuts(gf_shard* shard, const double* cuts, int num_phases);
int gf_shard_num_phases(gf_shard* shard, int* num_phases_out);
int gf_shard_phase_range(gf_shard* shard, int phase, int64_t* tok_begin, int64_t* tok_end);
int gf_shard_sample_phase(gf_shard* shard, uint32_t iteration, int phase);
/* sample_chunk's device half: K1 over every phase, each phase's new
 * assignments (word-group order) copied into `out` while the later phases
 * sample (overlapped when `out` is pinned and the shard has word phases);
 * returns with `out` complete. */
int gf_shard_sample_export(gf_shard* shard, uint32_t iteration, uint16_t* out);
/* Document-block phases (applies at the next load): phase 0 holds the slices of
 * the words that are not cut at document-block boundaries (they touch every
 * block), phase p >= 1 the block-scheduled slices of the document blocks whose
 * first document starts below cut[p-1] of the doc-major tokens (cumulative
 * fractions, strictly increasing, ending at 1.0).  Unlike word phases, no
 * theta row is streamed by two phases.  gf_shard_phase_doc_range gives the
 * doc-major token range [begin, end) that is final once phases 0..p have run
 * (empty for phase 0). */
int gf_shard_set_block_phases(gf_shard* shard, const double* cuts, int num_block_phases);
int gf_shard_phase_doc_range(gf_shard* shard, int phase, int64_t* tok_begin, int64_t* tok_end);
/* One deferred iteration: sample -> rebuild_phi [-> peer phi
 * exchange when a peer group is open] -> prepare, with rebuild_theta on an
 * internal stream beside everything after the sample. */
int gf_shard_iterate(gf_shard* shard, uint32_t iteration);
/* Sum over this shard's tokens of log p(w | d) for the model the last
 * gf_shard_sample started from (synchronises the stream). */
int gf_shard_loglik_sum(gf_shard* shard, double* sum_out);
/* non-blocking: out[0] = raw device sum (async copy on `stream`, NULL: the
 * shard's stream; `out` pinned), out[1] = the constant to subtract */
int gf_shard_loglik_sum_async(gf_shard* shard, double* out, void* stream);
/* Raise deferred device-side errors (overflow / consistency); synchronises. */
int gf_shard_check_errors(gf_shard* shard);
int gf_shard_synchronize(gf_shard* shard);

/* The phi sync buffer (device memory, uint32 words): [phi32 columns | packed
 * phi16 columns | n_k].  Summing the buffers of all ranks elementwise as
 * uint32 (e.g. NCCL allreduce sum) yields the global phi and n_k exactly. */
int gf_shard_sync_buffer(gf_shard* shard, void** device_ptr, int64_t* num_u32);
/* Peer-memory phi exchange (replaces the all_reduce of the sync buffer, i.e.
 * SPEC reduce_phi/broadcast_phi, on one NVLink/NVSwitch node).
 * 1. gf_shard_peer_handle -> GF_PEER_HANDLE_BYTES of IPC handles (after load);
 * 2. exchange them between ranks (any host channel, e.g. torch.distributed);
 * 3. gf_shard_peer_open(rank, world, handles of ranks 0..world-1 concatenated);
 * 4. per iteration gf_shard_peer_allreduce after rebuild_phi (stream-ordered;
 *    every rank must call it the same number of times) -- gf_shard_iterate
 *    does it itself once the group is open.  A reload invalidates the group.
 * A peer that stops participating makes the exchange time out (~20 s) and the
 * next gf_shard_check_errors report GF_ERR_TRAINING. */
#define GF_PEER_HANDLE_BYTES 128
#define GF_MAX_PEERS 8
int gf_shard_peer_handle(gf_shard* shard, void* handle_out);
int gf_shard_peer_open(gf_shard* shard, int rank, int world, const void* handles);
int gf_shard_peer_allreduce(gf_shard* shard);
/* K2X: rebuild the phi replica (K2) and sum it over the peer group in ONE
 * kernel, pipelined by stripes of the sync buffer (work items sorted by
 * buffer position at gf_shard_peer_open; a stripe is exchanged as soon as
 * every rank has completed it).  gf_shard_iterate uses it whenever a peer
 * group is open (GF_PEER_FUSED=0: K2 then the two-shot exchange kernel). */
int gf_shard_rebuild_phi_exchange(gf_shard* shard);
int gf_shard_peer_close(gf_shard* shard);
/* Host-only: the sync-buffer layout a shard derives from the global word
 * frequencies.  word_col_out[v] >= 0: 16-bit column index; < 0: ~(32-bit
 * column index).  layout_out = {phi16 offset, n_k offset, total} in uint32
 * words; 16-bit columns hold K rounded up to even cells. */
int gf_sync_layout(const int64_t* global_word_freq, int32_t vocab_size, int32_t num_topics,
                   uint32_t heavy_threshold, int32_t* word_col_out, int64_t* layout_out);

/* Pinned host blocks for arrays that cross PCIe every call (not in the
 * reference: its arrays never leave the host).  The Python mirror allocates
 * the one-call API's results here (get_theta / get_phi / get_assignments) and
 * frees them when the array is collected; a freed block is cached for the
 * next allocation of a similar size, so results are DMA'd directly, without
 * bounce copies or first-touch page faults, and an array handed back as the
 * next call's input uploads at full PCIe speed.  gf_host_free takes the
 * size passed to gf_host_alloc. */
int gf_host_alloc(int64_t bytes, void** out);
int gf_host_free(void* p, int64_t bytes);

/* import / export (host buffers, caller-allocated) */
int gf_shard_get_assignments(gf_shard* shard, uint16_t* out);      /* word-group order */
int gf_shard_set_assignments(gf_shard* shard, const uint16_t* in);
/* Asynchronous piecewise transfer of assignments [offset, offset + count) between
 * a (pinned) host buffer and the shard, on `stream` (a cudaStream_t; NULL: the
 * shard's stream), direction 1 = host -> device, 0 = device -> host.  Host ->
 * device pieces land in a staging buffer (allocated on the first such call);
 * gf_shard_assignments_imported (stream-ordered after the copies) applies them:
 * per run, only runs whose topics differ rewrite z and the doc-major copy.
 * It marks the counts stale (rebuild_phi / rebuild_theta next). */
int gf_shard_copy_assignments_async(gf_shard* shard, void* host, int64_t offset, int64_t count, int to_device,
                                    void* stream);
int gf_shard_assignments_imported(gf_shard* shard);
/* The same two calls in the shard's DOCUMENT-MAJOR order (the doc-major copy
 * K1 keeps, zdoc: per document its tokens by word group, heavy words first;
 * offsets index that order).  With document-block phases (below) a range of
 * documents is final as soon as its phase has run, so a step's assignments can
 * stream back per document range while later ranges sample. */
int gf_shard_copy_doc_assignments_async(gf_shard* shard, void* host, int64_t offset, int64_t count, int to_device,
                                        void* stream);
int gf_shard_doc_assignments_imported(gf_shard* shard);
int gf_shard_theta_nnz(gf_shard* shard, int64_t* nnz_out);
/* ThetaRows (model.py:20-47) of the shard's docs: row_ptr[D_s+1] (local), ids, counts */
int gf_shard_get_theta(gf_shard* shard, int64_t* row_ptr, uint16_t* topic_ids, uint16_t* counts);
int gf_shard_set_theta(gf_shard* shard, const int64_t* row_ptr, const uint16_t* topic_ids,
                       const uint16_t* counts);
/* PhiMatrix (model.py:50-80) as K x V row-major uint32 + int64 totals, read
 * from the sync buffer (replica after rebuild_phi, global after the sync). */
int gf_shard_get_phi(gf_shard* shard, uint32_t* counts_kv, int64_t* topic_totals);
int gf_shard_set_phi(gf_shard* shard, const uint32_t* counts_kv, const int64_t* topic_totals);
/* the same for a PhiMatrix of either width (16: uint16 cells; the export
 * raises the reference's 16-bit overflow text for the argmax cell first,
 * model.py:152-157, and narrows on the device) */
int gf_shard_get_phi_w(gf_shard* shard, void* counts_kv, int32_t phi_width, int64_t* topic_totals);
int gf_shard_set_phi_w(gf_shard* shard, const void* counts_kv, int32_t phi_width, const int64_t* topic_totals);
/* model.py:152-157: max cell count and its first (row-major K x V) position */
int gf_shard_phi_argmax(gf_shard* shard, int64_t* max_count, int32_t* topic, int32_t* word);

/* live counters for the roofline: stats[0] = K1 algorithmic bytes per sample
 * launch (averaged over the launches since the last reset), [1] = K2 bytes,
 * [2] = K3 bytes, [3] = runs, [4] = slices, [5] = tokens, [6] = theta nnz,
 * [7] = kernels launched by gf_shard_iterate (incl. the peer exchange), [8] = sample launches since reset,
 * [9] = precomputed word contexts, [10] = document blocks of the slice schedule. */
int gf_shard_stats(gf_shard* shard, int64_t* stats, int num_stats);
int gf_shard_reset_stats(gf_shard* shard);
/* CUDA-event time (ms) of the kernels of the last gf_shard_iterate:
 * ms[0] sample (+ loglik reduce), [1] phi rebuild (+memset, + peer exchange; theta rebuild runs
 * beside it on an internal stream), [2] prepare (+ word contexts), [3] theta
 * rebuild time not hidden behind [1] + [2]. */
int gf_shard_last_times(gf_shard* shard, float* ms, int num);

/* ------------------------------------------------- K5 conservation --
 * check_conservation (model.py:180-225) as device reductions.
 * report = {code, index, a, b}: 0 ok; 1 theta row `index` (global doc) sums
 * to a, its document length is b; 2 topic `index`: theta column sum a != n_k
 * b; 3 topic `index`: phi row sum a != n_k b; 4 totals sum to a, the corpus
 * has b tokens.  The host turns the report into the reference's text.
 * On a shard: stage 1 sums theta rows / columns and phi rows of the resident
 * state and returns the row report; a multi-rank caller then sums the theta
 * column sums over ranks in place (gf_shard_conservation_buffer: K uint64 on
 * the device); stage 2 compares against n_k and num_tokens. */
int gf_shard_conservation(gf_shard* shard, int stage, int64_t num_tokens, int64_t* report);
int gf_shard_conservation_buffer(gf_shard* shard, void** theta_col_sums, int64_t* num_topics);
/* The same check over the reference's exported arrays (ThetaRows CSR,
 * PhiMatrix K x V of phi_width bits, corpus doc lengths) uploaded to `device`;
 * report[0..3] is the row report, report[4..7] the column / phi / total one. */
int gf_check_conservation(int device, int32_t K, int64_t V, int64_t D, const int64_t* row_ptr,
                          const uint16_t* topic_ids, const uint16_t* counts, const int64_t* doc_lengths,
                          const void* phi_counts, int32_t phi_width, const int64_t* topic_totals,
                          int64_t num_tokens, int64_t* report);

/* ------------------------------------------------------ GFSNAP1 store --
 * save_snapshot / load_snapshot (model.py:228-296): native streaming writer
 * and reader of the reference's byte layout (bad magic / width:
 * GF_ERR_FORMAT with the reference's texts).  header: {K, V, D, NNZ,
 * phi_width, metadata bytes}; read fills caller-sized arrays. */
int gf_snapshot_write(const char* path, int64_t K, int64_t V, int64_t D, int64_t nnz, int32_t phi_width,
                      const void* phi_counts, const int64_t* topic_totals, const int64_t* row_ptr,
                      const uint16_t* topic_ids, const uint16_t* counts, const char* meta, int64_t meta_len);
int gf_snapshot_header(const char* path, int64_t* header_out);
int gf_snapshot_read(const char* path, void* phi_counts, int64_t* topic_totals, int64_t* row_ptr,
                     uint16_t* topic_ids, uint16_t* counts, char* meta);

/* ------------------------------------------------------ ptree primitive --
 * ptree.py:116-151 on the device: levels built from a prefix array exactly as
 * build() does (every fanout-th boundary), then a warp-ballot descent per u
 * returning the minimal index with prefix > u (ties go right): replaces
 * PrefixTree.sample / sample_many / sample_with_stats (ptree.py:64-113).
 * visited_out / widest_out (may be NULL) receive _descend's (levels visited,
 * widest scan) per u (ptree.py:73-99).  _f64 is the fp64 tree mode
 * (build(..., dtype=np.float64), ptree.py:119-121). */
int gf_ptree_sample(int device, const float* prefix, int64_t n, int32_t fanout, const float* u,
                    int64_t m, int64_t* idx_out, int32_t* visited_out, int32_t* widest_out);
int gf_ptree_sample_f64(int device, const double* prefix, int64_t n, int32_t fanout, const double* u,
                        int64_t m, int64_t* idx_out, int32_t* visited_out, int32_t* widest_out);

/* ------------------------------------------------- synthetic corpora --
 * Not in the reference (no datasets offline): seeded LDA-generative corpora
 * for tests and bench.py.  Documents are generated
 * independently from (seed, global doc id), so each rank can build its own
 * shard.  lengths_out[i] = length of doc doc_begin+i (log-normal, mean
 * mean_len); tokens are written doc-major at doc_ptr[i] (doc_ptr[0] = 0). */
int gf_synth_lengths(uint64_t seed, int64_t doc_begin, int64_t num_docs, double mean_len, double sigma,
                     int64_t* lengths_out);
int gf_synth_tokens(uint64_t seed, int64_t doc_begin, int64_t num_docs, const int64_t* doc_ptr,
                    int32_t vocab_size, int32_t k_true, double zipf_s, double doc_alpha,
                    int32_t* doc_ids_out, int32_t* word_ids_out);

#ifdef __cplusplus
}
#endif
#endif /* GIBBSFLOW_B200_H */
