// gf_abi.cu -- the C ABI (include/gibbsflow_b200.h): shard lifecycle, host-side
// native preprocessing (bit-exact with corpus.py / rng.py), device memory
// layout, import / export in the reference dataclass layouts.
#include "../../include/gibbsflow_b200.h"
#include "gf_internal.cuh"

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <numeric>
#include <thread>

namespace {

thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

int cuda_fail(cudaError_t e, const char* what) {
    if (e == cudaErrorMemoryAllocation)
        return fail(GF_ERR_CAPACITY, "%s: device out of memory (%s)", what, cudaGetErrorString(e));
    if (e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver)
        return fail(GF_ERR_NODEVICE, "%s: no usable CUDA device (%s)", what, cudaGetErrorString(e));
    return fail(GF_ERR_TRAINING, "%s: CUDA error %s", what, cudaGetErrorString(e));
}

#define CU(call, what)                                   \
    do {                                                 \
        cudaError_t _e = (call);                         \
        if (_e != cudaSuccess) return cuda_fail(_e, what); \
    } while (0)

constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ULL;

int64_t env_int(const char* name, int64_t dflt) {  // tuning knobs (A/B runs)
    const char* e = getenv(name);
    return e && *e ? atoll(e) : dflt;
}

inline uint64_t fin64(uint64_t z) {  // rng.py:20-26
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

inline double stream_u(uint64_t key, uint64_t ctr) {  // rng.py:38-42
    return (double)(fin64(key + kGolden * (ctr + 1ULL)) >> 11) * (1.0 / 9007199254740992.0);
}

template <class F>
void parallel_for(int64_t n, F f) {
    const int64_t grain = 1 << 20;
    unsigned nt = std::max(1u, std::min(std::thread::hardware_concurrency(), 32u));
    if (n < 2 * grain || nt == 1) { f(0, n); return; }
    nt = (unsigned)std::min<int64_t>(nt, n / grain);
    std::vector<std::thread> th;
    for (unsigned i = 0; i < nt; ++i) {
        int64_t a = n * i / nt, b = n * (i + 1) / nt;
        th.emplace_back([=] { f(a, b); });
    }
    for (auto& t : th) t.join();
}

template <class T>
int dev_alloc(T** p, size_t count, const char* what) {
    if (*p) { cudaFree(*p); *p = nullptr; }
    cudaError_t e = cudaMalloc((void**)p, std::max<size_t>(count, 1) * sizeof(T));
    if (e != cudaSuccess) return cuda_fail(e, what);
    return GF_OK;
}

void free_dev(gf_shard* s) {
    auto& d = s->d;
    void* ptrs[] = {d.z, d.zstage, d.run_doc, d.run_start, d.slices, d.k2items, d.dw_ptr, d.zdoc, d.run_dwpos, d.run_rec, d.theta_ent,
                    d.theta_meta, d.sync, d.inv_den, d.ctx_tab, d.ctx_cols, d.slice_ctx, d.ll_part, d.ll_sum,
                    d.errs, d.bytes, d.scratch, d.k5};
    for (void* p : ptrs)
        if (p) cudaFree(p);
    d = gf::ShardDev{};
}

}  // namespace

extern "C" int gf_sync_layout(const int64_t* freq, int32_t V, int32_t K, uint32_t thr, int32_t* word_col,
                              int64_t* layout) {  // hybrid phi columns from global frequencies
    if (V < 1 || K < 1) return fail(GF_ERR_VALUE, "bad layout dimensions");
    // a 16-bit column must never hold a cell above 65535 (nor carry into its
    // neighbour in the packed u32 sum), so light words are <= 65535 tokens
    if (thr > 65535u) return fail(GF_ERR_VALUE, "heavy_threshold %u exceeds 65535 (16-bit phi columns)", thr);
    const int64_t Kp = K + (K & 1);
    int64_t h = 0, l = 0;
    for (int v = 0; v < V; ++v) {
        if (freq[v] > (int64_t)thr) word_col[v] = ~(int32_t)(h++);
        else word_col[v] = (int32_t)(l++);
    }
    layout[0] = h * K;
    layout[1] = layout[0] + l * (Kp / 2);
    layout[2] = layout[1] + K;
    return GF_OK;
}

namespace {
int set_layout(gf_shard* s) {
    s->word_col.assign(s->V, 0);
    int64_t lay[3];
    if (int rc = gf_sync_layout(s->global_freq.data(), s->V, s->K, s->heavy_threshold, s->word_col.data(), lay))
        return rc;
    s->n_heavy = 0;
    for (int32_t c : s->word_col) s->n_heavy += c < 0;
    s->n_light = s->V - s->n_heavy;
    s->off_phi16_u32 = lay[0];
    s->off_nk_u32 = lay[1];
    s->sync_u32 = lay[2];
    return GF_OK;
}
}  // namespace

namespace gf {
int shard_fail(int code, const char* fmt, ...) {
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}
int shard_cuda_fail(cudaError_t e, const char* what) { return cuda_fail(e, what); }
int shard_set_layout(gf_shard* s) { return set_layout(s); }
int64_t shard_env_int(const char* name, int64_t dflt) { return env_int(name, dflt); }
void shard_free_device(gf_shard* s) { free_dev(s); }
}  // namespace gf

extern "C" {

const char* gf_last_error(void) { return g_err.c_str(); }
int gf_abi_version(void) { return 1; }

int gf_device_count(int* count_out) {
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess) n = 0;
    *count_out = n;
    return GF_OK;
}

// ------------------------------------------------------------------- rng --
uint64_t gf_stream_key(const uint64_t* parts, int num_parts) {  // rng.py:29-35, 45-53
    uint64_t h = kGolden;
    for (int i = 0; i < num_parts; ++i) h = fin64(h + kGolden + parts[i]);
    return h;
}

int gf_stream_uniforms(uint64_t key, uint64_t counter, int64_t n, double* out) {  // rng.py:84-89
    if (n < 0) return fail(GF_ERR_VALUE, "negative count");
    parallel_for(n, [&](int64_t a, int64_t b) {
        for (int64_t i = a; i < b; ++i) out[i] = stream_u(key, counter + (uint64_t)i);
    });
    return GF_OK;
}

// ---------------------------------------------------------------- corpus --
int gf_greedy_boundaries(const int64_t* L, int64_t D, int64_t C, int64_t* out) {  // corpus.py:210-237
    if (C < 1) return fail(GF_ERR_PARTITION, "need at least one chunk");
    if (C > D)
        return fail(GF_ERR_PARTITION, "cannot give every chunk a document: %lld chunks > %lld docs", (long long)C,
                    (long long)D);
    int64_t remaining = 0;
    for (int64_t i = 0; i < D; ++i) remaining += L[i];
    int64_t lo = 0;
    for (int64_t c = 0; c < C; ++c) {
        const int64_t left = C - c, hi_max = D - (left - 1), target = (remaining + left - 1) / left;
        int64_t acc = 0, hi = lo;
        while (hi < hi_max && acc < target) acc += L[hi++];
        out[2 * c] = lo;
        out[2 * c + 1] = hi;
        remaining -= acc;
        lo = hi;
    }
    return GF_OK;
}

int gf_partition_chunk(const int32_t* doc_ids, const int32_t* word_ids, int64_t n, int64_t doc_lo, int64_t doc_hi,
                       int32_t V, int32_t K, uint64_t seed, int64_t chunk_id, int32_t* out_doc, int32_t* out_word,
                       uint16_t* out_z, int32_t* gw, int64_t* go, int64_t* gs, int64_t* ng_out, int64_t* dw_ptr,
                       int64_t* dw_tok) {
    if (K < 1 || K >= 65536) return fail(GF_ERR_VALUE, "topic count %d outside [1, 65536)", K);
    const int64_t nd = doc_hi - doc_lo;
    // stable counting sort by word == np.argsort(kind="stable") (corpus.py:256-258)
    std::vector<int64_t> cnt((size_t)V + 1, 0);
    for (int64_t i = 0; i < n; ++i) {
        const int32_t w = word_ids[i];
        if (w < 0 || w >= V) return fail(GF_ERR_VALUE, "word id outside [0, vocab_size)");
        const int32_t d = doc_ids[i];
        if (d < doc_lo || d >= doc_hi) return fail(GF_ERR_VALUE, "doc id %d outside chunk range", d);
        cnt[(size_t)w + 1]++;
    }
    for (int32_t v = 0; v < V; ++v) cnt[(size_t)v + 1] += cnt[v];
    int64_t ng = 0;
    for (int32_t v = 0; v < V; ++v)  // np.unique directory, ascending words (corpus.py:260-262)
        if (cnt[(size_t)v + 1] > cnt[v]) { gw[ng] = v; go[ng] = cnt[v]; gs[ng] = cnt[(size_t)v + 1] - cnt[v]; ++ng; }
    *ng_out = ng;
    for (int64_t i = 0; i < n; ++i) {
        const int64_t p = cnt[word_ids[i]]++;
        out_doc[p] = doc_ids[i];
        out_word[p] = word_ids[i];
    }
    // doc-word map: stable counting sort by local doc (corpus.py:201-207)
    std::fill(dw_ptr, dw_ptr + nd + 1, 0);
    for (int64_t i = 0; i < n; ++i) dw_ptr[out_doc[i] - doc_lo + 1]++;
    for (int64_t d = 0; d < nd; ++d) dw_ptr[d + 1] += dw_ptr[d];
    std::vector<int64_t> fill(dw_ptr, dw_ptr + nd);
    for (int64_t i = 0; i < n; ++i) dw_tok[fill[out_doc[i] - doc_lo]++] = i;
    // initial topics from Stream(seed, chunk_id) (corpus.py:265-269)
    const uint64_t parts[2] = {seed, (uint64_t)chunk_id};
    const uint64_t key = gf_stream_key(parts, 2);
    parallel_for(n, [&](int64_t a, int64_t b) {
        for (int64_t i = a; i < b; ++i) {
            const int64_t zz = (int64_t)(stream_u(key, (uint64_t)i) * (double)K);
            out_z[i] = (uint16_t)std::min<int64_t>(zz, K - 1);
        }
    });
    return GF_OK;
}

// ----------------------------------------------------------------- shard --
int gf_shard_create(gf_shard** out, int device, int32_t K, int32_t V, double alpha, double beta, uint64_t seed,
                    uint32_t heavy_threshold) {
    *out = nullptr;
    if (K < 1 || K >= 65536) return fail(GF_ERR_VALUE, "topic count %d outside [1, 65536)", K);
    // device theta entries hold the topic as a 16-bit byte offset (topic << 2)
    if (K > 16384) return fail(GF_ERR_CAPACITY, "K=%d: the device sampler supports K <= 16384", K);
    if (V < 1) return fail(GF_ERR_VALUE, "vocab_size must be >= 1");
    if (!(alpha > 0) || !(beta > 0)) return fail(GF_ERR_VALUE, "alpha and beta must be > 0");
    if (heavy_threshold > 65535u)
        return fail(GF_ERR_VALUE, "heavy_threshold %u exceeds 65535 (16-bit phi columns)", heavy_threshold);
    int ndev = 0;
    gf_device_count(&ndev);
    if (ndev == 0) return fail(GF_ERR_NODEVICE, "no CUDA device visible: the B200 sampler has no CPU fallback");
    if (device < 0 || device >= ndev) return fail(GF_ERR_VALUE, "device %d out of range (%d visible)", device, ndev);
    CU(cudaSetDevice(device), "cudaSetDevice");
    gf_shard* s = new gf_shard();
    s->device = device;
    s->K = K;
    s->Kp = K + (K & 1);
    s->V = V;
    s->alpha = alpha;
    s->beta = beta;
    s->seed = seed;
    s->heavy_threshold = heavy_threshold;
    // Q-tree geometry (ptree.build levels, fanout 32)
    int len = K, total = 0, l = 0;
    while (true) {
        s->tree.off[l] = total;
        s->tree.len[l] = len;
        total += len;
        ++l;
        if (len == 1) break;
        len = (len + 31) / 32;
    }
    s->tree.nlev = l;
    s->tree.total = total;
    if (gf::sample_smem_bytes(s) > 220 * 1024) {
        const size_t need = gf::sample_smem_bytes(s);
        delete s;
        return fail(GF_ERR_CAPACITY, "K=%d: the sampler's shared-memory word context needs %zu bytes (> 220 KiB)",
                    K, need);
    }
    cudaError_t e = cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) { delete s; return cuda_fail(e, "cudaStreamCreate"); }
    s->own_stream = true;
    for (auto& ev : s->ev) cudaEventCreate(&ev);
    *out = s;
    return GF_OK;
}

int gf_shard_destroy(gf_shard* s) {
    if (!s) return GF_OK;
    cudaSetDevice(s->device);
    if (s->stream) cudaStreamSynchronize(s->stream);
    gf::peer_close(s);
    free_dev(s);
    for (auto& ev : s->ev)
        if (ev) cudaEventDestroy(ev);
    if (s->aux) { cudaStreamSynchronize(s->aux); cudaStreamDestroy(s->aux); }
    if (s->fork) cudaEventDestroy(s->fork);
    if (s->join) cudaEventDestroy(s->join);
    if (s->alt) { cudaStreamSynchronize(s->alt); cudaStreamDestroy(s->alt); }
    for (auto& ev : s->phase_ev)
        if (ev) cudaEventDestroy(ev);
    if (s->own_stream && s->stream) cudaStreamDestroy(s->stream);
    delete s;
    return GF_OK;
}

int gf_shard_set_stream(gf_shard* s, void* st) {
    cudaSetDevice(s->device);
    if (s->own_stream && s->stream) { cudaStreamSynchronize(s->stream); cudaStreamDestroy(s->stream); }
    s->stream = (cudaStream_t)st;
    s->own_stream = false;
    return GF_OK;
}

int gf_shard_set_params(gf_shard* s, double alpha, double beta, uint64_t seed) {
    if (!(alpha > 0) || !(beta > 0)) return fail(GF_ERR_VALUE, "alpha and beta must be > 0");
    if (alpha != s->alpha || beta != s->beta) s->ctx_dirty = true;   // denominators and contexts follow
    if (alpha != s->alpha && s->loaded && s->D > 0) {
        // the loglik constant sum_d L_d log(L_d + K a) follows alpha
        std::vector<uint32_t> dwp((size_t)s->D + 1);
        CU(cudaMemcpy(dwp.data(), s->d.dw_ptr, dwp.size() * 4, cudaMemcpyDeviceToHost), "set_params");
        double llc = 0.0;
        for (int64_t d = 0; d < s->D; ++d) {
            const double L = (double)(dwp[d + 1] - dwp[d]);
            if (L > 0) llc += L * std::log(L + (double)s->K * alpha);
        }
        s->ll_const = llc;
    }
    s->alpha = alpha;
    s->beta = beta;
    s->seed = seed;
    return GF_OK;
}

int gf_shard_set_vocab(gf_shard* s, const int64_t* freq) {
    if (s->loaded) return fail(GF_ERR_VALUE, "set_vocab must precede load");
    s->global_freq.assign(freq, freq + s->V);
    return GF_OK;
}

int gf_shard_load(gf_shard* s, int64_t doc_lo, int64_t doc_hi, int64_t T, const int32_t* doc_ids,
                  const int32_t* word_ids, const uint16_t* z, int64_t ng, const int32_t* gw, const int64_t* go,
                  const int64_t* gs, const int64_t* dw_ptr, const int64_t* dw_tok) {
    CU(cudaSetDevice(s->device), "cudaSetDevice");
    const int V = s->V;
    const int64_t D = doc_hi - doc_lo;
    if (D < 0 || T < 0) return fail(GF_ERR_SHAPE, "negative chunk size");
    if (T >= (int64_t)UINT32_MAX || D >= (int64_t)UINT32_MAX)
        return fail(GF_ERR_CAPACITY, "shard has %lld tokens: split the corpus over more shards", (long long)T);
    // ---- validate the chunk's directory (corpus.py:160-198 invariants); the
    // per-token checks run on the device (k_layout.cu k_check_chunk) ----
    int64_t covered = 0;
    for (int64_t g = 0; g < ng; ++g) {
        if (gw[g] < 0 || gw[g] >= V) return fail(GF_ERR_SHAPE, "group word %d outside [0, %d)", gw[g], V);
        if (go[g] < 0 || gs[g] < 0 || go[g] + gs[g] > T) return fail(GF_ERR_SHAPE, "group %lld out of range", (long long)g);
        if (go[g] != covered) return fail(GF_ERR_SHAPE, "word groups are not consecutive in token order");
        if (g > 0 && gw[g] <= gw[g - 1]) return fail(GF_ERR_SHAPE, "group words are not ascending");
        covered += gs[g];
    }
    if (covered != T) return fail(GF_ERR_SHAPE, "word groups cover %lld of %lld tokens", (long long)covered, (long long)T);
    if (dw_ptr[0] != 0 || dw_ptr[D] != T) return fail(GF_ERR_SHAPE, "doc-word map does not cover the chunk");
    for (int64_t d = 0; d < D; ++d)
        if (dw_ptr[d + 1] < dw_ptr[d]) return fail(GF_ERR_SHAPE, "doc-word map not monotone");
    s->loaded = false;
    return gf::load_chunk(s, doc_lo, doc_hi, T, doc_ids, word_ids, z, ng, gw, go, gs, dw_ptr, dw_tok);
}

int gf_shard_load_tokens(gf_shard* s, int64_t doc_lo, int64_t doc_hi, int64_t T, const int32_t* doc_ids,
                         const int32_t* word_ids, uint64_t seed, int64_t chunk_id) {
    CU(cudaSetDevice(s->device), "cudaSetDevice");
    const int64_t D = doc_hi - doc_lo;
    if (D < 0 || T < 0) return fail(GF_ERR_SHAPE, "negative chunk size");
    if (T >= (int64_t)UINT32_MAX || D >= (int64_t)UINT32_MAX)
        return fail(GF_ERR_CAPACITY, "shard has %lld tokens: split the corpus over more shards", (long long)T);
    const uint64_t parts[2] = {seed, (uint64_t)chunk_id};
    s->loaded = false;
    return gf::load_tokens(s, doc_lo, doc_hi, T, doc_ids, word_ids, gf_stream_key(parts, 2));
}

int gf_partition_chunk_gpu(int device, const int32_t* doc_ids, const int32_t* word_ids, int64_t n, int64_t doc_lo,
                           int64_t doc_hi, int32_t V, int32_t K, uint64_t seed, int64_t chunk_id, int32_t* out_doc,
                           int32_t* out_word, uint16_t* out_z, int32_t* gw, int64_t* go, int64_t* gs, int64_t* ng_out,
                           int64_t* dw_ptr, int64_t* dw_tok) {
    if (K < 1 || K >= 65536) return fail(GF_ERR_VALUE, "topic count %d outside [1, 65536)", K);
    if (n >= (int64_t)UINT32_MAX || doc_hi - doc_lo >= (int64_t)UINT32_MAX)
        return fail(GF_ERR_CAPACITY, "chunk has %lld tokens: split the corpus into more chunks", (long long)n);
    int ndev = 0;
    gf_device_count(&ndev);
    if (ndev == 0) return fail(GF_ERR_NODEVICE, "no CUDA device visible: use gf_partition_chunk on the host");
    const uint64_t parts[2] = {seed, (uint64_t)chunk_id};
    return gf::partition_to_host(device, doc_ids, word_ids, n, doc_lo, doc_hi, V, K, gf_stream_key(parts, 2), out_doc,
                                 out_word, out_z, gw, go, gs, ng_out, dw_ptr, dw_tok);
}

static int need_loaded(gf_shard* s) {
    if (!s || !s->loaded) return fail(GF_ERR_VALUE, "shard has no chunk loaded");
    cudaSetDevice(s->device);
    return GF_OK;
}

// the shard's grow-only device scratch for import / export staging (one call
// at a time per shard; every user synchronises before returning)
static int dev_scratch(gf_shard* s, size_t bytes, char** out) {
    if (s->d.scratch_bytes < bytes) {
        if (s->d.scratch) { cudaStreamSynchronize(s->stream); cudaFree(s->d.scratch); }
        s->d.scratch = nullptr;
        s->d.scratch_bytes = 0;
        const size_t want = bytes + bytes / 4;
        CU(cudaMalloc((void**)&s->d.scratch, want), "device scratch");
        s->d.scratch_bytes = want;
    }
    *out = reinterpret_cast<char*>(s->d.scratch);
    return GF_OK;
}

static inline size_t al256(size_t b) { return (b + 255) & ~(size_t)255; }

int gf_shard_rebuild_phi(gf_shard* s) {
    if (int rc = need_loaded(s)) return rc;
    CU(gf::launch_phi_rebuild(s), "rebuild_phi");
    s->stale_phi = false;
    return GF_OK;
}

int gf_shard_rebuild_theta(gf_shard* s) {
    if (int rc = need_loaded(s)) return rc;
    CU(gf::launch_theta_rebuild(s), "rebuild_theta");
    s->stale_theta = false;
    return GF_OK;
}

int gf_shard_prepare(gf_shard* s) {
    if (int rc = need_loaded(s)) return rc;
    CU(gf::launch_prepare(s), "prepare");
    return GF_OK;
}

static int validate_if_dirty(gf_shard* s) {
    if (s->stale_theta || s->stale_phi) {
        CU(gf::launch_validate(s), "validate");
        s->stale_theta = s->stale_phi = false;
    }
    return GF_OK;
}

int gf_shard_sample(gf_shard* s, uint32_t iteration) {
    if (int rc = need_loaded(s)) return rc;
    if (int rc = validate_if_dirty(s)) return rc;
    CU(gf::launch_sample(s, iteration), "sample");
    CU(gf::launch_ll_reduce(s), "loglik");
    s->stat_sample_launches++;
    return GF_OK;
}

int gf_shard_set_phases(gf_shard* s, int num_phases) {
    if (num_phases < 1 || num_phases > 255) return fail(GF_ERR_VALUE, "phases must be in [1, 255]");
    s->n_phases = num_phases;     // applies at the next load (the slice schedule is built there)
    s->block_phases = false;
    s->phase_cuts.clear();
    return GF_OK;
}

int gf_shard_set_phase_cuts(gf_shard* s, const double* cuts, int num_phases) {
    if (num_phases < 1 || num_phases > 255) return fail(GF_ERR_VALUE, "phases must be in [1, 255]");
    for (int p = 0; p < num_phases; ++p)
        if (!(cuts[p] > (p ? cuts[p - 1] : 0.0)) || cuts[p] > 1.0 || (p == num_phases - 1 && cuts[p] != 1.0))
            return fail(GF_ERR_VALUE, "phase cuts must increase strictly and end at 1.0");
    s->n_phases = num_phases;
    s->block_phases = false;
    s->phase_cuts.assign(cuts, cuts + num_phases);
    return GF_OK;
}

int gf_shard_set_block_phases(gf_shard* s, const double* cuts, int num_block_phases) {
    if (num_block_phases < 1 || num_block_phases > 254) return fail(GF_ERR_VALUE, "block phases must be in [1, 254]");
    for (int p = 0; p < num_block_phases; ++p)
        if (!(cuts[p] > (p ? cuts[p - 1] : 0.0)) || cuts[p] > 1.0 || (p == num_block_phases - 1 && cuts[p] != 1.0))
            return fail(GF_ERR_VALUE, "phase cuts must increase strictly and end at 1.0");
    s->n_phases = num_block_phases + 1;   // + phase 0: the words not cut at block boundaries
    s->block_phases = true;
    s->phase_cuts.assign(cuts, cuts + num_block_phases);
    return GF_OK;
}

int gf_shard_phase_doc_range(gf_shard* s, int phase, int64_t* tok_begin, int64_t* tok_end) {
    if (int rc = need_loaded(s)) return rc;
    if (!s->block_phases) return fail(GF_ERR_VALUE, "no document-block phases: gf_shard_set_block_phases, then load");
    if (phase < 0 || phase + 1 >= (int)s->phase_doctok0.size()) return fail(GF_ERR_VALUE, "phase %d out of range", phase);
    *tok_begin = s->phase_doctok0[phase];
    *tok_end = s->phase_doctok0[phase + 1];
    return GF_OK;
}

int gf_shard_num_phases(gf_shard* s, int* out) {
    if (int rc = need_loaded(s)) return rc;
    *out = (int)s->phase_slice0.size() - 1;
    return GF_OK;
}

int gf_shard_phase_range(gf_shard* s, int phase, int64_t* tok_begin, int64_t* tok_end) {
    if (int rc = need_loaded(s)) return rc;
    if (phase < 0 || phase + 1 >= (int)s->phase_tok0.size()) return fail(GF_ERR_VALUE, "phase %d out of range", phase);
    *tok_begin = s->phase_tok0[phase];
    *tok_end = s->phase_tok0[phase + 1];
    return GF_OK;
}

int gf_shard_sample_phase(gf_shard* s, uint32_t iteration, int phase) {
    if (int rc = need_loaded(s)) return rc;
    const int P = (int)s->phase_slice0.size() - 1;
    if (phase < 0 || phase >= P) return fail(GF_ERR_VALUE, "phase %d out of range [0, %d)", phase, P);
    if (phase == 0)
        if (int rc = validate_if_dirty(s)) return rc;
    const int64_t a = s->phase_slice0[phase], b = s->phase_slice0[phase + 1];
    CU(gf::launch_sample_range(s, iteration, 0, a, b - a), "sample");
    if (phase == P - 1) {
        CU(gf::launch_ll_reduce(s), "loglik");
        s->stat_sample_launches++;
    }
    return GF_OK;
}

// K1 over every phase of the schedule, each phase's new assignments copied to
// the host (word-group order) on the aux stream while the phases after it
// sample; returns with `out` complete.  One-phase shards: sample, then copy.
int gf_shard_sample_export(gf_shard* s, uint32_t iteration, uint16_t* out) {
    if (int rc = need_loaded(s)) return rc;
    if (int rc = validate_if_dirty(s)) return rc;
    cudaSetDevice(s->device);
    if (!s->aux) {
        CU(cudaStreamCreateWithFlags(&s->aux, cudaStreamNonBlocking), "sample_export");
        CU(cudaEventCreateWithFlags(&s->fork, cudaEventDisableTiming), "sample_export");
        CU(cudaEventCreateWithFlags(&s->join, cudaEventDisableTiming), "sample_export");
    }
    const int P = (int)s->phase_slice0.size() - 1;
    const bool async = gf::host_is_pinned(out) && P > 1 && !s->block_phases;
    if (!async) {
        CU(gf::launch_sample(s, iteration), "sample");
        CU(gf::launch_ll_reduce(s), "loglik");
        s->stat_sample_launches++;
        CU(gf::xfer_d2h(out, s->d.z, s->T * 2, s->stream), "sample_export");
        return GF_OK;
    }
    // Phases alternate between the caller's stream and `alt` (they are
    // independent: each reads the iteration-start counts and writes its own
    // tokens), so a phase's tail CTAs overlap the next phase's first ones; the
    // loglik reduction waits for both.  Phase p's tokens go out on `aux` as
    // soon as phase p is done.
    if (!s->alt) CU(cudaStreamCreateWithFlags(&s->alt, cudaStreamNonBlocking), "sample_export");
    while ((int)s->phase_ev.size() < P) {
        cudaEvent_t e;
        CU(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "sample_export");
        s->phase_ev.push_back(e);
    }
    cudaStream_t const main = s->stream;
    struct Restore {                           // s->stream back to the caller's on every exit
        gf_shard* s;
        cudaStream_t st;
        ~Restore() { s->stream = st; }
    } restore{s, main};
    CU(cudaEventRecord(s->fork, main), "sample_export");
    CU(cudaStreamWaitEvent(s->alt, s->fork, 0), "sample_export");
    for (int p = 0; p < P; ++p) {
        const int64_t a = s->phase_slice0[p], b = s->phase_slice0[p + 1];
        s->stream = (p & 1) ? s->alt : main;
        CU(gf::launch_sample_range(s, iteration, 0, a, b - a), "sample");
        CU(cudaEventRecord(s->phase_ev[p], s->stream), "sample_export");
        if (p == P - 1) {                      // P > 1: phase P-2 ran on the other stream
            CU(cudaStreamWaitEvent(s->stream, s->phase_ev[P - 2], 0), "sample_export");
            CU(gf::launch_ll_reduce(s), "loglik");
            if (s->stream != main) {
                CU(cudaEventRecord(s->join, s->stream), "sample_export");
                CU(cudaStreamWaitEvent(main, s->join, 0), "sample_export");
            }
        }
        const int64_t t0 = s->phase_tok0[p], t1 = s->phase_tok0[p + 1];
        if (t1 > t0) {
            // phase p alone writes z[t0, t1): copy it out behind the later phases
            CU(cudaStreamWaitEvent(s->aux, s->phase_ev[p], 0), "sample_export");
            CU(cudaMemcpyAsync(out + t0, s->d.z + t0, (size_t)(t1 - t0) * 2, cudaMemcpyDeviceToHost, s->aux),
               "sample_export");
        }
    }
    s->stream = main;
    s->stat_sample_launches++;
    CU(cudaStreamSynchronize(s->aux), "sample_export");
    CU(cudaStreamSynchronize(s->stream), "sample_export");
    return GF_OK;
}

int gf_shard_evaluate(gf_shard* s) {
    if (int rc = need_loaded(s)) return rc;
    CU(gf::launch_sample(s, 0, 1), "evaluate");
    CU(gf::launch_ll_reduce(s), "loglik");
    return GF_OK;
}

int gf_shard_iterate(gf_shard* s, uint32_t iteration) {
    if (int rc = need_loaded(s)) return rc;
    if (int rc = validate_if_dirty(s)) return rc;
    if (s->peer.world > 1 && s->peer.sync != s->d.sync)
        return fail(GF_ERR_VALUE, "peer group opened before the last load: exchange handles and reopen");
    cudaStream_t st = s->stream;
    if (!s->aux) {
        CU(cudaStreamCreateWithFlags(&s->aux, cudaStreamNonBlocking), "iterate");
        CU(cudaEventCreateWithFlags(&s->fork, cudaEventDisableTiming), "iterate");
        CU(cudaEventCreateWithFlags(&s->join, cudaEventDisableTiming), "iterate");
    }
    if (s->timing) cudaEventRecord(s->ev[0], st);
    CU(gf::launch_sample(s, iteration), "sample");
    CU(gf::launch_ll_reduce(s), "loglik");
    if (s->timing) cudaEventRecord(s->ev[1], st);
    // K3 (theta from zdoc) on the aux stream beside K2 (phi from z) + prepare:
    // independent inputs and outputs; the caller's next call waits for both
    CU(cudaEventRecord(s->fork, st), "iterate");
    CU(cudaStreamWaitEvent(s->aux, s->fork, 0), "iterate");
    CU(gf::launch_theta_rebuild(s, s->aux), "rebuild_theta");
    CU(cudaEventRecord(s->join, s->aux), "iterate");
    if (s->peer.world > 1 && env_int("GF_PEER_FUSED", 1)) {
        CU(gf::launch_phi_rebuild_exchange(s), "rebuild_phi_exchange");   // K2X: K2 + exchange in one kernel
    } else {
        CU(gf::launch_phi_rebuild(s), "rebuild_phi");
        if (s->peer.world > 1) CU(gf::launch_peer_allreduce(s, st), "peer_allreduce");
    }
    if (s->timing) cudaEventRecord(s->ev[2], st);
    CU(gf::launch_prepare(s), "prepare");
    if (s->timing) cudaEventRecord(s->ev[3], st);
    CU(cudaStreamWaitEvent(st, s->join, 0), "iterate");
    if (s->timing) cudaEventRecord(s->ev[4], st);
    // sample, ll_reduce, theta, phi, prepare (+ contexts) (+ peer exchange)
    s->stat_launches = 5 + (s->n_ctx > 0) + (s->peer.world > 1);
    s->stat_sample_launches++;
    return GF_OK;
}

int gf_shard_last_times(gf_shard* s, float* ms, int num) {
    CU(cudaEventSynchronize(s->ev[4]), "events");
    for (int i = 0; i < num && i < 4; ++i) {
        float t = 0.f;
        cudaEventElapsedTime(&t, s->ev[i], s->ev[i + 1]);
        ms[i] = t;
    }
    return GF_OK;
}

// the same value without blocking the host: out[0] receives the raw device
// sum (stream-ordered copy; `out` should be pinned) and out[1] the constant
// to subtract, so the log-likelihood sum is out[0] - out[1] once the stream
// has reached the copy
int gf_shard_loglik_sum_async(gf_shard* s, double* out, void* stream) {
    if (int rc = need_loaded(s)) return rc;
    cudaStream_t st = stream ? (cudaStream_t)stream : s->stream;
    out[1] = s->ll_const;
    CU(cudaMemcpyAsync(out, s->d.ll_sum, 8, cudaMemcpyDeviceToHost, st), "loglik");
    return GF_OK;
}

int gf_shard_loglik_sum(gf_shard* s, double* out) {
    if (int rc = need_loaded(s)) return rc;
    double v = 0.0;
    CU(cudaMemcpyAsync(&v, s->d.ll_sum, 8, cudaMemcpyDeviceToHost, s->stream), "loglik");
    CU(cudaStreamSynchronize(s->stream), "loglik");
    *out = v - s->ll_const;
    return GF_OK;
}

int gf_shard_synchronize(gf_shard* s) {
    cudaSetDevice(s->device);
    CU(cudaStreamSynchronize(s->stream), "synchronize");
    return GF_OK;
}

int gf_shard_check_errors(gf_shard* s) {
    if (int rc = need_loaded(s)) return rc;
    unsigned long long e[4];
    CU(cudaMemcpyAsync(e, s->d.errs, 32, cudaMemcpyDeviceToHost, s->stream), "errors");
    CU(cudaStreamSynchronize(s->stream), "errors");
    CU(cudaMemsetAsync(s->d.errs, 0xff, 32, s->stream), "errors");
    if (e[3] != ~0ULL)
        return fail(GF_ERR_TRAINING, "rank %d: phi peer exchange timed out waiting for a peer (block %llu)",
                    s->peer.rank, e[3]);
    if (e[1] != ~0ULL) {
        const long long d = (long long)(e[1] >> 32) + s->doc_lo;
        return fail(GF_ERR_OVERFLOW, "document %lld: topic count %llu exceeds 16-bit range", d,
                    (unsigned long long)(e[1] & 0xffffffffULL));
    }
    if (e[2] != ~0ULL)
        return fail(GF_ERR_CONSISTENCY, "document %lld: a token's topic is outside [0, K=%d)",
                    (long long)e[2] + s->doc_lo, s->K);
    if (e[0] != ~0ULL)
        return fail(GF_ERR_CONSISTENCY, "token %llu: its current topic is absent from its document's theta row "
                    "(or from phi / n_k)", (unsigned long long)e[0]);
    return GF_OK;
}

int gf_shard_sync_buffer(gf_shard* s, void** p, int64_t* n) {
    if (int rc = need_loaded(s)) return rc;
    *p = s->d.sync;
    *n = s->sync_u32;
    return GF_OK;
}

int gf_shard_peer_handle(gf_shard* s, void* out) {
    if (int rc = need_loaded(s)) return rc;
    cudaSetDevice(s->device);
    return gf::peer_handle(s, out);
}

int gf_shard_peer_open(gf_shard* s, int rank, int world, const void* handles) {
    if (int rc = need_loaded(s)) return rc;
    cudaSetDevice(s->device);
    return gf::peer_open(s, rank, world, handles);
}

int gf_shard_peer_allreduce(gf_shard* s) {
    if (int rc = need_loaded(s)) return rc;
    if (s->peer.world < 1 || s->peer.sync != s->d.sync)
        return fail(GF_ERR_VALUE, "no peer group open on this shard's current sync buffer");
    cudaSetDevice(s->device);
    if (s->peer.world > 1) CU(gf::launch_peer_allreduce(s, s->stream), "peer_allreduce");
    return GF_OK;
}

int gf_shard_rebuild_phi_exchange(gf_shard* s) {
    if (int rc = need_loaded(s)) return rc;
    if (s->peer.world < 1) return fail(GF_ERR_VALUE, "no peer group: gf_shard_peer_open first");
    if (s->peer.sync != s->d.sync)
        return fail(GF_ERR_VALUE, "peer group opened before the last load: exchange handles and reopen");
    CU(gf::launch_phi_rebuild_exchange(s), "rebuild_phi_exchange");
    s->stale_phi = false;
    return GF_OK;
}

int gf_shard_peer_close(gf_shard* s) {
    cudaSetDevice(s->device);
    if (s->stream) cudaStreamSynchronize(s->stream);
    gf::peer_close(s);
    return GF_OK;
}

// pinned result blocks of the one-call API (gf_xfer.cpp host_alloc)
int gf_host_alloc(int64_t bytes, void** out) {
    if (bytes < 0 || !out) return fail(GF_ERR_VALUE, "host_alloc: bad arguments");
    *out = nullptr;
    CU(gf::host_alloc((size_t)bytes, out), "host_alloc");
    return GF_OK;
}

int gf_host_free(void* p, int64_t bytes) {
    CU(gf::host_free(p, (size_t)bytes), "host_free");
    return GF_OK;
}

int gf_shard_get_assignments(gf_shard* s, uint16_t* out) {
    if (int rc = need_loaded(s)) return rc;
    CU(gf::xfer_d2h(out, s->d.z, s->T * 2, s->stream), "get_assignments");
    return GF_OK;
}

int gf_shard_set_assignments(gf_shard* s, const uint16_t* in) {
    if (int rc = need_loaded(s)) return rc;
    // range is checked on the device (K1/K2/K3 flag z >= K as a consistency error)
    CU(gf::xfer_h2d(s->d.z, in, s->T * 2, s->stream), "set_assignments");
    CU(gf::launch_zdoc_sync(s), "set_assignments");
    CU(cudaStreamSynchronize(s->stream), "set_assignments");
    s->stale_theta = s->stale_phi = true;
    return GF_OK;
}

int gf_shard_copy_assignments_async(gf_shard* s, void* host, int64_t offset, int64_t count, int to_device,
                                    void* stream) {
    if (int rc = need_loaded(s)) return rc;
    if (offset < 0 || count < 0 || offset + count > s->T) return fail(GF_ERR_SHAPE, "assignment range out of bounds");
    cudaStream_t st = stream ? (cudaStream_t)stream : s->stream;
    if (to_device && !s->d.zstage) {   // host -> device imports are staged, applied by _imported
        cudaSetDevice(s->device);
        CU(cudaMalloc((void**)&s->d.zstage, std::max<int64_t>(s->T, 1) * 2), "copy_assignments (staging)");
    }
    uint16_t* dev = (to_device ? s->d.zstage : s->d.z) + offset;
    uint16_t* h = static_cast<uint16_t*>(host) + offset;
    // pinned host buffers: a plain async copy in both directions (the call
    // returns at once; stream order is the caller's); pageable ones go through
    // the pinned bounce buffers (the host side then completes before returning)
    if (gf::host_is_pinned(h)) {
        CU(cudaMemcpyAsync(to_device ? (void*)dev : (void*)h, to_device ? (const void*)h : (const void*)dev, count * 2,
                           to_device ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToHost, st),
           "copy_assignments");
    } else if (to_device) {
        CU(gf::xfer_h2d(dev, h, count * 2, st), "copy_assignments");
    } else {
        CU(gf::xfer_d2h(h, dev, count * 2, st), "copy_assignments");
    }
    return GF_OK;
}

// the same in the shard's document-major order (zdoc: per document, its tokens
// by word group, heavy words first) -- the order in which document-block
// phases complete
int gf_shard_copy_doc_assignments_async(gf_shard* s, void* host, int64_t offset, int64_t count, int to_device,
                                        void* stream) {
    if (int rc = need_loaded(s)) return rc;
    if (offset < 0 || count < 0 || offset + count > s->T) return fail(GF_ERR_SHAPE, "assignment range out of bounds");
    cudaStream_t st = stream ? (cudaStream_t)stream : s->stream;
    if (to_device && !s->d.zstage) {
        cudaSetDevice(s->device);
        CU(cudaMalloc((void**)&s->d.zstage, std::max<int64_t>(s->T, 1) * 2), "copy_doc_assignments (staging)");
    }
    uint16_t* dev = (to_device ? s->d.zstage : s->d.zdoc) + offset;
    uint16_t* h = static_cast<uint16_t*>(host) + offset;
    if (gf::host_is_pinned(h)) {
        CU(cudaMemcpyAsync(to_device ? (void*)dev : (void*)h, to_device ? (const void*)h : (const void*)dev, count * 2,
                           to_device ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToHost, st),
           "copy_doc_assignments");
    } else if (to_device) {
        CU(gf::xfer_h2d(dev, h, count * 2, st), "copy_doc_assignments");
    } else {
        CU(gf::xfer_d2h(h, dev, count * 2, st), "copy_doc_assignments");
    }
    return GF_OK;
}

int gf_shard_doc_assignments_imported(gf_shard* s) {
    if (int rc = need_loaded(s)) return rc;
    if (!s->d.zstage) return fail(GF_ERR_VALUE, "no staged assignments: gf_shard_copy_doc_assignments_async(to_device=1) first");
    CU(gf::launch_import_staged(s, true), "doc_assignments_imported");
    s->stale_theta = s->stale_phi = true;
    return GF_OK;
}

int gf_shard_assignments_imported(gf_shard* s) {
    if (int rc = need_loaded(s)) return rc;
    if (!s->d.zstage) return fail(GF_ERR_VALUE, "no staged assignments: gf_shard_copy_assignments_async(to_device=1) first");
    CU(gf::launch_import_staged(s), "assignments_imported");
    s->stale_theta = s->stale_phi = true;
    return GF_OK;
}

static int fetch_meta(gf_shard* s, std::vector<uint2>& meta) {
    meta.resize((size_t)s->D);
    if (s->D) CU(cudaMemcpyAsync(meta.data(), s->d.theta_meta, s->D * sizeof(uint2), cudaMemcpyDeviceToHost, s->stream),
                 "theta meta");
    CU(cudaStreamSynchronize(s->stream), "theta meta");
    return GF_OK;
}

// the exported CSR's row_ptr, scanned on the device into the scratch
static int theta_rowptr_dev(gf_shard* s, int64_t** d_rowptr, char** after) {
    size_t tmp = 0;
    CU(gf::theta_rowptr(s, nullptr, nullptr, &tmp), "theta row_ptr");
    const size_t b_rp = al256((s->D + 1) * 8);
    char* base = nullptr;
    if (int rc = dev_scratch(s, b_rp + al256(tmp), &base)) return rc;
    *d_rowptr = reinterpret_cast<int64_t*>(base);
    CU(gf::theta_rowptr(s, *d_rowptr, base + b_rp, &tmp), "theta row_ptr");
    if (after) *after = base + b_rp;
    return GF_OK;
}

int gf_shard_theta_nnz(gf_shard* s, int64_t* nnz) {
    if (int rc = need_loaded(s)) return rc;
    int64_t* drp = nullptr;
    if (int rc = theta_rowptr_dev(s, &drp, nullptr)) return rc;
    CU(cudaMemcpyAsync(nnz, drp + s->D, 8, cudaMemcpyDeviceToHost, s->stream), "theta nnz");
    CU(cudaStreamSynchronize(s->stream), "theta nnz");
    return GF_OK;
}

int gf_shard_get_theta(gf_shard* s, int64_t* row_ptr, uint16_t* ids, uint16_t* cnts) {
    // row_ptr by a device scan, the entries by the export kernel, all three
    // arrays back through the staged copies (no host loop over documents)
    if (int rc = need_loaded(s)) return rc;
    int64_t nnz = 0;
    if (int rc = gf_shard_theta_nnz(s, &nnz)) return rc;
    const size_t b_rp = al256((s->D + 1) * 8), b_e = al256((size_t)std::max<int64_t>(nnz, 1) * 2);
    char* base = nullptr;
    if (int rc = dev_scratch(s, b_rp + 2 * b_e, &base)) return rc;
    int64_t* drp = reinterpret_cast<int64_t*>(base);
    uint16_t* dids = reinterpret_cast<uint16_t*>(base + b_rp);
    uint16_t* dcnt = reinterpret_cast<uint16_t*>(base + b_rp + b_e);
    size_t tmp = 0;
    CU(gf::theta_rowptr(s, nullptr, nullptr, &tmp), "get_theta");
    if (tmp > b_e) {                          // scan temp space: reuse the counts slot only if it fits
        if (int rc = dev_scratch(s, b_rp + 2 * b_e + al256(tmp), &base)) return rc;
        drp = reinterpret_cast<int64_t*>(base);
        dids = reinterpret_cast<uint16_t*>(base + b_rp);
        dcnt = reinterpret_cast<uint16_t*>(base + b_rp + b_e);
    }
    void* tmpp = tmp > b_e ? (void*)(base + b_rp + 2 * b_e) : (void*)dcnt;
    CU(gf::theta_rowptr(s, drp, tmpp, &tmp), "get_theta");
    cudaError_t e = gf::launch_theta_export(s, drp, dids, dcnt);
    if (e == cudaSuccess) e = gf::xfer_d2h(row_ptr, drp, (s->D + 1) * 8, s->stream);
    if (e == cudaSuccess && nnz) e = gf::xfer_d2h(ids, dids, nnz * 2, s->stream);
    if (e == cudaSuccess && nnz) e = gf::xfer_d2h(cnts, dcnt, nnz * 2, s->stream);
    if (e != cudaSuccess) return cuda_fail(e, "get_theta");
    return GF_OK;
}

int gf_shard_set_theta(gf_shard* s, const int64_t* row_ptr, const uint16_t* ids, const uint16_t* cnts) {
    // upload, then validate on the device (theta_validate_kernel: capacity,
    // ids < K, nonzero counts, strictly increasing ids) before importing
    if (int rc = need_loaded(s)) return rc;
    const int64_t nnz = row_ptr[s->D];
    if (nnz < 0) return fail(GF_ERR_SHAPE, "theta row_ptr is not non-decreasing");
    const int64_t nn = std::max<int64_t>(nnz, 1);
    char* base = nullptr;
    const size_t b_rp = al256((s->D + 1) * 8), b_e = al256((size_t)nn * 2);
    if (int rc = dev_scratch(s, b_rp + 2 * b_e + 16, &base)) return rc;
    int64_t* drp = reinterpret_cast<int64_t*>(base);
    uint16_t* dids = reinterpret_cast<uint16_t*>(base + b_rp);
    uint16_t* dcnt = reinterpret_cast<uint16_t*>(base + b_rp + b_e);
    unsigned long long* dfirst = reinterpret_cast<unsigned long long*>(base + b_rp + 2 * b_e);
    unsigned long long first = ~0ull;
    cudaError_t e = gf::xfer_h2d(drp, row_ptr, (s->D + 1) * 8, s->stream);
    if (e == cudaSuccess && nnz) e = gf::xfer_h2d(dids, ids, nnz * 2, s->stream);
    if (e == cudaSuccess && nnz) e = gf::xfer_h2d(dcnt, cnts, nnz * 2, s->stream);
    if (e == cudaSuccess) e = gf::launch_theta_validate(s, drp, dids, dcnt, dfirst);
    if (e == cudaSuccess) e = cudaMemcpyAsync(&first, dfirst, 8, cudaMemcpyDeviceToHost, s->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s->stream);
    if (e == cudaSuccess && first != ~0ull) {
        const long long d = (long long)(first >> 34);
        const uint64_t low = first & ((1ull << 34) - 1);
        if (low == 0) {
            std::vector<uint2> meta;
            if (int rc = fetch_meta(s, meta)) return rc;
            const uint32_t next = d + 1 < s->D ? meta[d + 1].x : (uint32_t)s->theta_cap;
            return fail(GF_ERR_SHAPE, "theta row %lld has %lld entries, capacity %u", d,
                        (long long)(row_ptr[d + 1] - row_ptr[d]), next - meta[d].x);
        }
        if ((low & 1) == 0) return fail(GF_ERR_SHAPE, "theta row %lld: bad entry", d);
        return fail(GF_ERR_SHAPE, "theta row %lld: topic ids not strictly increasing", d);
    }
    if (e == cudaSuccess) e = gf::launch_theta_import(s, drp, dids, dcnt);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s->stream);
    if (e != cudaSuccess) return cuda_fail(e, "set_theta");
    s->stale_theta = true;
    return GF_OK;
}

// K x V export into a device buffer (u32) plus the device argmax: the phi
// checks and the 16-bit narrowing run before anything crosses PCIe
static int phi_export_device(gf_shard* s, uint32_t** dout, int32_t** dcol) {
    const size_t cells = (size_t)s->K * s->V;
    char* base = nullptr;
    if (int rc = dev_scratch(s, al256(cells * 4 + 16) + al256((size_t)s->V * 4), &base)) return rc;
    *dout = reinterpret_cast<uint32_t*>(base);
    *dcol = reinterpret_cast<int32_t*>(base + al256(cells * 4 + 16));
    CU(cudaMemcpyAsync(*dcol, s->word_col.data(), (size_t)s->V * 4, cudaMemcpyHostToDevice, s->stream), "phi export");
    CU(gf::launch_phi_export(s, *dout, 32, *dcol), "phi export");
    return GF_OK;
}

static int phi_argmax_device(gf_shard* s, uint32_t* dout, int64_t* max_count, int32_t* topic, int32_t* word) {
    const size_t cells = (size_t)s->K * s->V;
    unsigned int* dmax = reinterpret_cast<unsigned int*>(dout + cells);
    unsigned long long* dfirst = reinterpret_cast<unsigned long long*>(dout + ((cells + 3) & ~(size_t)1));
    unsigned int mx = 0;
    unsigned long long first = 0;
    CU(gf::launch_phi_argmax(dout, (int64_t)cells, dmax, dfirst, s->stream), "phi_argmax");
    CU(cudaMemcpyAsync(&mx, dmax, 4, cudaMemcpyDeviceToHost, s->stream), "phi_argmax");
    CU(cudaMemcpyAsync(&first, dfirst, 8, cudaMemcpyDeviceToHost, s->stream), "phi_argmax");
    CU(cudaStreamSynchronize(s->stream), "phi_argmax");
    if (cells == 0) first = 0;
    *max_count = mx;
    *topic = (int32_t)(first / s->V);
    *word = (int32_t)(first % s->V);
    return GF_OK;
}

int gf_shard_get_phi_w(gf_shard* s, void* counts_kv, int32_t width, int64_t* totals) {
    if (int rc = need_loaded(s)) return rc;
    if (width != 16 && width != 32) return fail(GF_ERR_VALUE, "phi width must be 16 or 32, got %d", width);
    const size_t cells = (size_t)s->K * s->V;
    uint32_t* dout = nullptr;
    int32_t* dcol = nullptr;
    if (int rc = phi_export_device(s, &dout, &dcol)) return rc;
    int rc = GF_OK;
    if (width == 16) {                        // model.py:152-157: the argmax cell must fit 16 bits
        int64_t m = 0;
        int32_t k = 0, v = 0;
        rc = phi_argmax_device(s, dout, &m, &k, &v);
        if (rc == GF_OK && m > 65535)
            rc = fail(GF_ERR_OVERFLOW, "phi cell (topic %d, word %d) count %lld exceeds 16-bit range", k, v,
                      (long long)m);
        if (rc == GF_OK) {                   // narrow on the device: half the PCIe bytes
            cudaError_t e = gf::launch_phi_export(s, dout, 16, dcol);
            if (e != cudaSuccess) rc = cuda_fail(e, "get_phi");
        }
    }
    std::vector<uint32_t> nk((size_t)s->K);
    cudaError_t e = cudaSuccess;
    if (rc == GF_OK) e = gf::xfer_d2h(counts_kv, dout, cells * (width / 8), s->stream);
    if (rc == GF_OK && e == cudaSuccess)
        e = cudaMemcpyAsync(nk.data(), s->d.sync + s->off_nk_u32, (size_t)s->K * 4, cudaMemcpyDeviceToHost, s->stream);
    if (rc == GF_OK && e == cudaSuccess) e = cudaStreamSynchronize(s->stream);
    if (rc != GF_OK) return rc;
    if (e != cudaSuccess) return cuda_fail(e, "get_phi");
    for (int k = 0; k < s->K; ++k) totals[k] = nk[k];
    return GF_OK;
}

int gf_shard_get_phi(gf_shard* s, uint32_t* counts_kv, int64_t* totals) {
    return gf_shard_get_phi_w(s, counts_kv, 32, totals);
}

int gf_shard_set_phi_w(gf_shard* s, const void* counts_kv, int32_t width, const int64_t* totals) {
    if (int rc = need_loaded(s)) return rc;
    if (width != 16 && width != 32) return fail(GF_ERR_VALUE, "phi width must be 16 or 32, got %d", width);
    for (int k = 0; k < s->K; ++k)
        if (totals[k] < 0 || totals[k] > (int64_t)UINT32_MAX) return fail(GF_ERR_OVERFLOW, "topic total out of range");
    const size_t cells = (size_t)s->K * s->V;
    char* base = nullptr;
    const size_t b_in = al256(cells * (width / 8) + 16);
    if (int rc = dev_scratch(s, b_in + al256((size_t)s->V * 4 + 32), &base)) return rc;
    void* din = base;
    int32_t* dcol = reinterpret_cast<int32_t*>(base + b_in);
    cudaError_t e = cudaSuccess;
    unsigned long long* dfirst = reinterpret_cast<unsigned long long*>(dcol + ((s->V + 3) & ~3));
    std::vector<uint32_t> nk((size_t)s->K);
    for (int k = 0; k < s->K; ++k) nk[k] = (uint32_t)totals[k];
    unsigned long long first = ~0ull;
    e = cudaMemcpyAsync(dcol, s->word_col.data(), (size_t)s->V * 4, cudaMemcpyHostToDevice, s->stream);
    if (e == cudaSuccess) e = gf::xfer_h2d(din, counts_kv, cells * (width / 8), s->stream);
    // a light (16-bit) column must not receive a cell above 65535: checked on the
    // device before anything is written (first cell in word-major order)
    if (width == 32) {
        if (e == cudaSuccess)
            e = gf::launch_phi_u16_overflow((const uint32_t*)din, dcol, s->K, s->V, dfirst, s->stream);
        if (e == cudaSuccess) e = cudaMemcpyAsync(&first, dfirst, 8, cudaMemcpyDeviceToHost, s->stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s->stream);
        if (e == cudaSuccess && first != ~0ull) {
            const int v = (int)(first / s->K), k = (int)(first % s->K);
            return fail(GF_ERR_OVERFLOW, "phi cell (topic %d, word %d) count %u exceeds its 16-bit column", k, v,
                        ((const uint32_t*)counts_kv)[(size_t)k * s->V + v]);
        }
    }
    if (e == cudaSuccess) e = cudaMemsetAsync(s->d.sync, 0, s->sync_u32 * 4, s->stream);
    if (e == cudaSuccess) e = gf::launch_phi_import(s, din, width, dcol);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(s->d.sync + s->off_nk_u32, nk.data(), (size_t)s->K * 4, cudaMemcpyHostToDevice, s->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s->stream);
    if (e != cudaSuccess) return cuda_fail(e, "set_phi");
    s->stale_phi = true;
    s->ctx_dirty = true;                     // denominators and word contexts follow the new phi
    return GF_OK;
}

int gf_shard_set_phi(gf_shard* s, const uint32_t* counts_kv, const int64_t* totals) {
    return gf_shard_set_phi_w(s, counts_kv, 32, totals);
}

int gf_shard_phi_argmax(gf_shard* s, int64_t* max_count, int32_t* topic, int32_t* word) {
    // np.argmax of the exported K x V counts (model.py:152-157), reduced on the
    // device: the export stays in HBM, 12 bytes come back
    if (int rc = need_loaded(s)) return rc;
    uint32_t* dout = nullptr;
    int32_t* dcol = nullptr;
    if (int rc = phi_export_device(s, &dout, &dcol)) return rc;
    return phi_argmax_device(s, dout, max_count, topic, word);
}

// ------------------------------------------------- K5 conservation ------
static int k5_scratch(gf_shard* s) {
    if (!s->d.k5) CU(cudaMalloc(&s->d.k5, (2 * (size_t)s->K + 1 + 8) * 8), "conservation");
    return GF_OK;
}

int gf_shard_conservation(gf_shard* s, int stage, int64_t num_tokens, int64_t* report) {
    if (int rc = need_loaded(s)) return rc;
    if (stage != 1 && stage != 2) return fail(GF_ERR_VALUE, "conservation stage must be 1 or 2, got %d", stage);
    if (int rc = k5_scratch(s)) return rc;
    int64_t* drep = reinterpret_cast<int64_t*>(s->d.k5 + 2 * (size_t)s->K + 1);
    if (stage == 1) CU(gf::launch_conservation_stage1(s, s->d.k5, drep), "conservation");
    else CU(gf::launch_conservation_stage2(s, s->d.k5, num_tokens, drep), "conservation");
    CU(cudaMemcpyAsync(report, drep, 32, cudaMemcpyDeviceToHost, s->stream), "conservation");
    CU(cudaStreamSynchronize(s->stream), "conservation");
    return GF_OK;
}

int gf_shard_conservation_buffer(gf_shard* s, void** theta_col, int64_t* n) {
    if (int rc = need_loaded(s)) return rc;
    if (int rc = k5_scratch(s)) return rc;
    *theta_col = s->d.k5;
    *n = s->K;
    return GF_OK;
}

int gf_check_conservation(int device, int32_t K, int64_t V, int64_t D, const int64_t* row_ptr,
                          const uint16_t* topic_ids, const uint16_t* counts, const int64_t* doc_lengths,
                          const void* phi_counts, int32_t phi_width, const int64_t* topic_totals, int64_t num_tokens,
                          int64_t* report) {
    if (K < 1 || V < 0 || D < 0) return fail(GF_ERR_VALUE, "bad conservation dimensions");
    if (phi_width != 16 && phi_width != 32) return fail(GF_ERR_VALUE, "phi width must be 16 or 32, got %d", phi_width);
    int ndev = 0;
    gf_device_count(&ndev);
    if (ndev == 0) return fail(GF_ERR_NODEVICE, "no CUDA device visible");
    CU(cudaSetDevice(device), "cudaSetDevice");
    const int64_t nnz = row_ptr[D];
    const size_t b_rp = (D + 1) * 8, b_ids = std::max<int64_t>(nnz, 1) * 2, b_len = std::max<int64_t>(D, 1) * 8;
    const size_t b_phi = std::max<size_t>((size_t)K * V * (phi_width / 8), 4), b_tot = (size_t)K * 8;
    const size_t b_k5 = (2 * (size_t)K + 1) * 8 + 64;
    auto al = [](size_t b) { return (b + 255) & ~(size_t)255; };
    const size_t total = al(b_rp) + 2 * al(b_ids) + al(b_len) + al(b_phi) + al(b_tot) + al(b_k5);
    char* base = nullptr;
    CU(cudaMalloc(&base, total), "check_conservation");
    char* p = base;
    auto take = [&](size_t b) { char* q = p; p += al(b); return q; };
    int64_t* drp = (int64_t*)take(b_rp);
    uint16_t* dids = (uint16_t*)take(b_ids);
    uint16_t* dcnt = (uint16_t*)take(b_ids);
    int64_t* dlen = (int64_t*)take(b_len);
    void* dphi = take(b_phi);
    int64_t* dtot = (int64_t*)take(b_tot);
    unsigned long long* dk5 = (unsigned long long*)take(b_k5);
    int64_t* drep = reinterpret_cast<int64_t*>(dk5 + 2 * (size_t)K + 1);
    cudaStream_t st = 0;
    cudaError_t e = cudaMemcpyAsync(drp, row_ptr, b_rp, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess && nnz) e = cudaMemcpyAsync(dids, topic_ids, nnz * 2, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess && nnz) e = cudaMemcpyAsync(dcnt, counts, nnz * 2, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess && D) e = cudaMemcpyAsync(dlen, doc_lengths, D * 8, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess && K * V)
        e = cudaMemcpyAsync(dphi, phi_counts, (size_t)K * V * (phi_width / 8), cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(dtot, topic_totals, b_tot, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess)
        e = gf::conservation_csr(K, V, D, drp, dids, dcnt, dlen, dphi, phi_width, dtot, num_tokens, dk5, drep, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(report, drep, 64, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    cudaFree(base);
    if (e != cudaSuccess) return cuda_fail(e, "check_conservation");
    return GF_OK;
}

int gf_shard_stats(gf_shard* s, int64_t* st, int n) {
    if (int rc = need_loaded(s)) return rc;
    unsigned long long nnz_runs = 0;
    CU(cudaMemcpyAsync(&nnz_runs, s->d.bytes, 8, cudaMemcpyDeviceToHost, s->stream), "stats");
    CU(cudaStreamSynchronize(s->stream), "stats");
    const int64_t K = s->K;
    // K1 algorithmic bytes per launch: per run its doc id,
    // run_start pair, zdoc position and theta meta (4 + 4 + 4 + 8) plus its
    // theta row (4 B per entry, averaged over the launches since the last
    // reset); per token z read + z' write + zdoc write (2 + 2 + 2); per slice
    // the slice record (16), its context index (4), the word's phi column (2 or
    // 4 B per topic), the K denominators (2 x 4 B) and its ll partial (8).
    int64_t phi_col_bytes = 0;
    {
        std::vector<int4> sl((size_t)s->n_slices);
        if (s->n_slices)
            CU(cudaMemcpy(sl.data(), s->d.slices, sl.size() * sizeof(int4), cudaMemcpyDeviceToHost), "stats");
        for (auto& x : sl) phi_col_bytes += (x.w >= 0 ? 2 : 4) * K;
    }
    const int64_t L = std::max<int64_t>(s->stat_sample_launches, 1);
    const int64_t b_sample = s->R * 20 + (int64_t)(4 * nnz_runs) / L + s->T * 6 +
                             s->n_slices * (16 + 4 + 8 * K + 8) + phi_col_bytes;
    // K2: memset of the sync buffer + z read + work items (+ nonzero cells, not counted)
    const int64_t b_phi = s->sync_u32 * 4 + s->T * 2 + s->n_k2 * 16;
    // K3: zdoc per token (contiguous per doc), dw_ptr + meta per doc, 4 B per written entry
    int64_t nnz = 0;
    if (n > 2) gf_shard_theta_nnz(s, &nnz);
    const int64_t b_theta = s->T * 2 + (s->D + 1) * 4 + s->D * 8 + nnz * 4;
    int64_t v[11] = {b_sample, b_phi,    b_theta, s->R, s->n_slices, s->T, nnz, s->stat_launches, s->stat_sample_launches,
                     s->n_ctx,  s->n_doc_blocks};
    for (int i = 0; i < n && i < 11; ++i) st[i] = v[i];
    return GF_OK;
}

int gf_shard_reset_stats(gf_shard* s) {
    if (int rc = need_loaded(s)) return rc;
    CU(cudaMemsetAsync(s->d.bytes, 0, 8, s->stream), "reset_stats");
    s->stat_sample_launches = 0;
    return GF_OK;
}

// -------------------------------------------------------------- ptree ------
}  // extern "C"

namespace {
template <typename T, typename Launch>
int ptree_sample_any(int device, const T* prefix, int64_t n, int32_t fanout, const T* u, int64_t m,
                     int64_t* idx_out, int32_t* visited_out, int32_t* widest_out, Launch launch) {
    if (fanout < 2) return fail(GF_ERR_VALUE, "fanout must be >= 2, got %d", fanout);
    if (n < 1) return fail(GF_ERR_EMPTY, "weights must be a non-empty 1-d array");
    const T total = prefix[n - 1];
    if (!(total > T(0))) return fail(GF_ERR_EMPTY, "cannot sample: total weight is zero");
    for (int64_t i = 0; i < m; ++i)
        if (!(u[i] >= T(0)) || !(u[i] < total)) return fail(GF_ERR_VALUE, "u values outside [0, total)");
    int ndev = 0;
    gf_device_count(&ndev);
    if (ndev == 0) return fail(GF_ERR_NODEVICE, "no CUDA device visible");
    CU(cudaSetDevice(device), "cudaSetDevice");
    const int64_t mm = std::max<int64_t>(m, 1);
    T *dp = nullptr, *du = nullptr;
    int64_t* di = nullptr;
    int32_t* ds = nullptr;  // [visited | widest]
    cudaError_t e = cudaMalloc(&dp, n * sizeof(T));
    if (e == cudaSuccess) e = cudaMalloc(&du, mm * sizeof(T));
    if (e == cudaSuccess) e = cudaMalloc(&di, mm * 8);
    if (e == cudaSuccess) e = cudaMalloc(&ds, mm * 8);
    if (e == cudaSuccess) e = cudaMemcpy(dp, prefix, n * sizeof(T), cudaMemcpyHostToDevice);
    if (e == cudaSuccess && m) e = cudaMemcpy(du, u, m * sizeof(T), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = launch(dp, n, fanout, du, m, di, ds, ds + mm, (cudaStream_t)0);
    if (e == cudaSuccess && m) e = cudaMemcpy(idx_out, di, m * 8, cudaMemcpyDeviceToHost);
    if (e == cudaSuccess && m && visited_out) e = cudaMemcpy(visited_out, ds, m * 4, cudaMemcpyDeviceToHost);
    if (e == cudaSuccess && m && widest_out) e = cudaMemcpy(widest_out, ds + mm, m * 4, cudaMemcpyDeviceToHost);
    if (dp) cudaFree(dp);
    if (du) cudaFree(du);
    if (di) cudaFree(di);
    if (ds) cudaFree(ds);
    if (e != cudaSuccess) return cuda_fail(e, "ptree_sample");
    return GF_OK;
}
}  // namespace

extern "C" {
int gf_ptree_sample(int device, const float* prefix, int64_t n, int32_t fanout, const float* u, int64_t m,
                    int64_t* idx_out, int32_t* visited_out, int32_t* widest_out) {
    return ptree_sample_any<float>(device, prefix, n, fanout, u, m, idx_out, visited_out, widest_out,
                                   gf::ptree_sample);
}

int gf_ptree_sample_f64(int device, const double* prefix, int64_t n, int32_t fanout, const double* u, int64_t m,
                        int64_t* idx_out, int32_t* visited_out, int32_t* widest_out) {
    return ptree_sample_any<double>(device, prefix, n, fanout, u, m, idx_out, visited_out, widest_out,
                                    gf::ptree_sample_f64);
}

}  // extern "C"
