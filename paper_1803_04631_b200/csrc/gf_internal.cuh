// gf_internal.cuh -- shared definitions of the B200 gibbsflow hot path.
//
// HBM layout of one document shard:
//   z          u16[T]        topic of each token, word-group order (in place)
//   run_doc    u32[R]        local doc of each (doc, word) run
//   run_start  u32[R+1]      first token of each run
//   slices     int4[N]       {word, run_begin, run_end, phi column} heavy-first
//   k2items    int4[M]       {phi column, tok_begin, tok_end, atomic?}
//   dw_ptr     u32[D+1]      doc-major token ranges (corpus.py:201-207 dw-map)
//   zdoc       u16[T]        the same topics in doc-major order (K1 writes
//                            them, K3 reads each doc contiguously); inside a
//                            doc, tokens of block-scheduled words come first
//   run_dwpos  u32[R]        zdoc position of each run's first token
//   run_rec    uint4[R]      {doc, run_start, run_dwpos, theta offset}: K1's one
//                            16-byte load per run
//   theta_ent  u32[cap]      (count << 16 | topic) rows, fixed capacity
//                            round4(min(K, L_d)) per doc, ids ascending
//   theta_meta uint2[D]      {row offset, nnz}
//   sync       u32[...]      [phi32 | phi16 packed | n_k]: word-major phi
//                            columns (one contiguous K-vector per word), plus
//                            one word after n_k: K2's work-item counter
//   inv_den    f32[K]        1 / (n_k + V beta)
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include <string>
#include <vector>

namespace gf {

constexpr int kSampleThreads = 256;         // 8 warps: 8 samplers share one Q-tree
constexpr int kSliceTokens = 4096;          // tokens per sampler CTA (heavy words split)
constexpr int kMaxLevels = 5;

struct TreeGeom {                            // Q-tree levels in shared memory
    int nlev;
    int off[kMaxLevels];
    int len[kMaxLevels];
    int total;                               // floats
};

struct ShardDev {
    uint16_t* z = nullptr;
    uint32_t* run_doc = nullptr;
    uint32_t* run_start = nullptr;
    int4* slices = nullptr;
    int4* k2items = nullptr;
    uint32_t* dw_ptr = nullptr;
    uint16_t* zdoc = nullptr;
    uint16_t* zstage = nullptr;              // async imports land here (allocated on first use)
    uint32_t* run_dwpos = nullptr;
    uint4* run_rec = nullptr;                // per run {doc, first token, zdoc position, theta row offset} (K1)
    uint32_t* theta_ent = nullptr;
    uint2* theta_meta = nullptr;
    uint32_t* sync = nullptr;
    float* inv_den = nullptr;                // [2K]: 1/(n_k + V b), 1/(n_k - 1 + V b)
    float* ctx_tab = nullptr;                // [n_ctx][ctx_stride] word contexts
    int32_t* ctx_cols = nullptr;             // [n_ctx] phi column of each context's word
    int32_t* slice_ctx = nullptr;            // [N] context of each slice (-1: built in place)
    double* ll_part = nullptr;
    double* ll_sum = nullptr;
    unsigned long long* errs = nullptr;      // [0] consistency token (min), [1] theta overflow key (min),
                                             // [2] document with a topic >= K (K3, min),
                                             // [3] peer exchange block that timed out (min)
    unsigned long long* bytes = nullptr;     // [0] sum over runs of nnz (sampler bytes model), [1] import flag
    uint32_t* scratch = nullptr;             // export staging
    size_t scratch_bytes = 0;
    unsigned long long* k5 = nullptr;        // K5 conservation: [K] theta column sums | [K] phi row sums |
                                             // first bad doc | report (int64 x 4); allocated on first use
};

constexpr int kMaxPeers = 8;                 // ranks of one NVLink/NVSwitch node
constexpr int kLlSlots = 160;                // ll_sum: [0] sum, [1..148] chunk sums, [159] ticket

// peer-memory phi exchange (k_peer.cu): every rank's sync buffer and signal
// slots mapped into this process (own entries are the local pointers)
struct PeerGroup {
    int rank = 0, world = 0;                 // world 0: not open
    uint32_t* buf[kMaxPeers] = {};
    uint32_t* sig[kMaxPeers] = {};
    uint32_t* own_sig = nullptr;             // this rank's signal slots (cudaMalloc, exported)
    uint32_t* sync = nullptr;                // the sync buffer the group was opened on
    uint32_t epoch = 0;
    // fused K2 + exchange (k_counts.cu K2X): stripes of the sync buffer
    size_t sig_fused = 0;                    // offset (u32) of the fused kernel's slots in every sig array
    int nstripe = 0;
    long long stripe_words = 0;
    unsigned* xdev = nullptr;                // [nstripe] items per stripe | [nstripe + 2] counters
};

}  // namespace gf

struct gf_shard {
    int device = 0;
    int K = 0, Kp = 0, V = 0;
    double alpha = 0, beta = 0;
    uint64_t seed = 0;
    uint32_t heavy_threshold = 65535;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    bool loaded = false;
    // host-side layout
    std::vector<int64_t> global_freq;        // V
    std::vector<int32_t> word_col;           // V: >=0 light column, <0 ~heavy column
    int64_t n_heavy = 0, n_light = 0;
    int64_t off_phi16_u32 = 0, off_nk_u32 = 0, sync_u32 = 0;
    int64_t doc_lo = 0, doc_hi = 0, D = 0, T = 0, R = 0, n_slices = 0, n_k2 = 0;
    int64_t theta_cap = 0;
    int64_t n_doc_blocks = 1;
    // sampling phases (gf_shard_set_phases): the slice schedule is phase-major;
    // phase p owns the word groups whose tokens are z[phase_tok0[p], phase_tok0[p+1])
    // and the slices [phase_slice0[p], phase_slice0[p+1])
    int n_phases = 1;
    std::vector<double> phase_cuts;          // optional cumulative token fractions (gf_shard_set_phase_cuts)
    std::vector<int64_t> phase_slice0{0, 0}, phase_tok0{0, 0};
    // document-block phases (gf_shard_set_block_phases): phase 0 = the slices
    // of words not cut at block boundaries (they touch every block), phase
    // p >= 1 = the block-scheduled slices of a range of document blocks; the
    // doc-major (zdoc) tokens [phase_doctok0[p], phase_doctok0[p+1]) are final
    // once phases 0..p have run (phase 0's range is empty)
    bool block_phases = false;
    std::vector<int64_t> phase_doctok0{0, 0};
    int64_t n_ctx = 0;
    bool ctx_dirty = true;                   // phi / n_k changed since the last prepare
    double ll_const = 0.0;                    // sum_d L_d log(L_d + K alpha)
    std::vector<int64_t> runs_per_doc_dummy;
    gf::TreeGeom tree{};
    gf::ShardDev d;
    int64_t stat_sample_bytes = 0, stat_phi_bytes = 0, stat_theta_bytes = 0;
    int64_t stat_launches = 0;
    int64_t stat_sample_launches = 0;
    cudaEvent_t ev[6] = {};
    cudaStream_t aux = nullptr;              // gf_shard_iterate: K3 beside K2 + prepare
    cudaEvent_t fork = nullptr, join = nullptr;
    cudaStream_t alt = nullptr;              // gf_shard_sample_export: every other phase
    std::vector<cudaEvent_t> phase_ev;       // ... and each phase's completion
    float last_ms[4] = {0, 0, 0, 0};
    gf::PeerGroup peer;                      // open: gf_shard_iterate reduces phi over peer memory
    bool timing = true;
    // imported state not yet validated: an import (set_assignments / set_theta /
    // set_phi) marks the count structures it may have made inconsistent; a
    // rebuild from z makes that structure consistent by construction
    bool stale_theta = false, stale_phi = false;
};

// shard helpers shared by the ABI (gf_abi.cu) and the K4 layout builder (k_layout.cu)
namespace gf {
// cudaFuncSetAttribute once per (kernel, device): `done` is the kernel's bit set of devices
inline bool attr_once(unsigned long long& done, int device) {
    const unsigned long long bit = 1ull << (device & 63);
    if (done & bit) return false;
    done |= bit;
    return true;
}
int shard_fail(int code, const char* fmt, ...);
// streaming multiprocessors of `device` (grid sizing; cached per device)
inline int sm_count(int device) {
    static int cache[64] = {0};
    int& c = cache[device & 63];
    if (!c) {
        int n = 0;
        if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device) != cudaSuccess || n < 1) n = 1;
        c = n;
    }
    return c;
}
int shard_cuda_fail(cudaError_t e, const char* what);
int shard_set_layout(gf_shard* s);
int64_t shard_env_int(const char* name, int64_t dflt);
void shard_free_device(gf_shard* s);
template <class T>
int shard_alloc(T** p, size_t count, const char* what) {
    if (*p) { cudaFree(*p); *p = nullptr; }
    cudaError_t e = cudaMalloc((void**)p, (count > 0 ? count : 1) * sizeof(T));
    return e == cudaSuccess ? 0 : shard_cuda_fail(e, what);
}
// peer-memory phi exchange (k_peer.cu)
int peer_handle(gf_shard* s, void* out);
int peer_open(gf_shard* s, int rank, int world, const void* handles);
void peer_close(gf_shard* s);
cudaError_t launch_peer_allreduce(gf_shard* s, cudaStream_t st);
// K4 (k_layout.cu)
int load_chunk(gf_shard* s, int64_t lo, int64_t hi, int64_t T, const int32_t* doc_ids, const int32_t* word_ids,
               const uint16_t* z, int64_t ng, const int32_t* gw, const int64_t* go, const int64_t* gs,
               const int64_t* dw_ptr, const int64_t* dw_tok);
int load_tokens(gf_shard* s, int64_t lo, int64_t hi, int64_t T, const int32_t* doc_ids, const int32_t* word_ids,
                uint64_t zkey);
int partition_to_host(int device, const int32_t* doc_ids, const int32_t* word_ids, int64_t n, int64_t lo, int64_t hi,
                      int32_t V, int32_t K, uint64_t zkey, int32_t* out_doc, int32_t* out_word, uint16_t* out_z,
                      int32_t* gw, int64_t* go, int64_t* gs, int64_t* ng_out, int64_t* dw_ptr, int64_t* dw_tok);
}  // namespace gf

// kernel launchers (k_sample.cu / k_counts.cu)
namespace gf {
cudaError_t launch_sample(gf_shard* s, uint32_t iteration, int eval_only = 0);
cudaError_t launch_sample_range(gf_shard* s, uint32_t iteration, int eval_only, int64_t slice0, int64_t n);
cudaError_t launch_phi_rebuild(gf_shard* s);
cudaError_t launch_phi_rebuild_exchange(gf_shard* s);   // K2X: K2 fused with the peer exchange
cudaError_t launch_prepare(gf_shard* s);
cudaError_t launch_contexts(gf_shard* s);
cudaError_t launch_theta_rebuild(gf_shard* s, cudaStream_t st = nullptr);
cudaError_t launch_zdoc_sync(gf_shard* s);
cudaError_t launch_import_staged(gf_shard* s, bool doc_order = false);
cudaError_t launch_ll_reduce(gf_shard* s);
cudaError_t launch_theta_export(gf_shard* s, const int64_t* d_rowptr, uint16_t* d_ids, uint16_t* d_cnt);
cudaError_t launch_theta_import(gf_shard* s, const int64_t* d_rowptr, const uint16_t* d_ids,
                                const uint16_t* d_cnt);
cudaError_t theta_rowptr(gf_shard* s, int64_t* d_rowptr, void* tmp, size_t* tmp_bytes);
// host <-> device copies of pageable arrays through pinned bounce buffers (gf_xfer.cpp)
cudaError_t xfer_h2d(void* dst, const void* src, size_t n, cudaStream_t st);
cudaError_t xfer_d2h(void* dst, const void* src, size_t n, cudaStream_t st);
// cached pinned host blocks for the one-call API's result arrays (gf_host_alloc)
cudaError_t host_alloc(size_t n, void** out);
cudaError_t host_free(void* p, size_t n);
bool host_is_pinned(const void* p);
cudaError_t launch_theta_validate(gf_shard* s, const int64_t* d_rowptr, const uint16_t* d_ids, const uint16_t* d_cnt,
                                  unsigned long long* d_first);
cudaError_t launch_phi_export(gf_shard* s, void* d_out_kv, int width, const int32_t* d_word_col);
cudaError_t launch_phi_import(gf_shard* s, const void* d_in_kv, int width, const int32_t* d_word_col);
cudaError_t launch_validate(gf_shard* s);
size_t sample_smem_bytes(const gf_shard* s);
size_t context_floats(const gf_shard* s);
// K5 + device phi checks (k_check.cu)
cudaError_t launch_conservation_stage1(gf_shard* s, unsigned long long* scratch, int64_t* d_report);
cudaError_t launch_conservation_stage2(gf_shard* s, const unsigned long long* scratch, int64_t T, int64_t* d_report);
cudaError_t conservation_csr(int K, int64_t V, int64_t D, const int64_t* row_ptr, const uint16_t* ids,
                             const uint16_t* cnt, const int64_t* doc_len, const void* phi, int width,
                             const int64_t* totals, int64_t T, unsigned long long* scratch, int64_t* d_report,
                             cudaStream_t st);
cudaError_t launch_phi_u16_overflow(const uint32_t* d_kv, const int32_t* d_wcol, int K, int64_t V,
                                    unsigned long long* d_first, cudaStream_t st);
cudaError_t launch_phi_argmax(const uint32_t* d_kv, int64_t n, unsigned int* d_max, unsigned long long* d_first,
                              cudaStream_t st);
cudaError_t ptree_sample(const float* d_prefix, int64_t n, int fanout, const float* d_u, int64_t m,
                         int64_t* d_idx, int32_t* d_visited, int32_t* d_widest, cudaStream_t st);
cudaError_t ptree_sample_f64(const double* d_prefix, int64_t n, int fanout, const double* d_u, int64_t m,
                             int64_t* d_idx, int32_t* d_visited, int32_t* d_widest, cudaStream_t st);
}  // namespace gf
