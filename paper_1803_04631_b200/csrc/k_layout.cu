// k_layout.cu -- K4: preprocessing on the GPU.
//
//   partition (corpus.py:240-287): stable sort of a document range's tokens by
//     word (ties keep corpus order, corpus.py:256-258), the ascending group
//     directory (np.unique, corpus.py:260-262), the doc-word map (stable sort
//     by local doc, corpus.py:201-207) and the initial topics
//     z0 = min(floor(u K), K - 1) from Stream(seed, chunk_id) (rng.py:20-89,
//     corpus.py:265-269, fp64 on the device, bit-exact);
//   shard layout: (doc, word) runs, the doc-blocked heavy-first slice schedule
//     (sort_word_groups_desc order, corpus.py:290-302), word contexts, K2 work
//     items and the heavy-first doc-major zdoc position of every run.
//
// The sorts are CUB's stable LSD radix sorts (the CUDA toolkit's library
// primitive); every other step is a flag / scan / scatter kernel here.  The
// host keeps only O(vocabulary) and O(documents) work (group ranks, contexts,
// document blocks).
#include "../../include/gibbsflow_b200.h"
#include "gf_internal.cuh"
#include "gf_device.cuh"

#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <numeric>
#include <vector>

namespace gf {

namespace {

constexpr uint64_t kGoldenD = 0x9E3779B97F4A7C15ULL;

inline unsigned blocks_for(int64_t n, int per = 256) {
    const int64_t b = (n + per - 1) / per;
    return (unsigned)std::max<int64_t>(1, std::min<int64_t>(b, 148LL * 64));
}

#define GRID_STRIDE(i, n) for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < (n); i += (int64_t)gridDim.x * blockDim.x)

__global__ void k_iota(uint32_t* out, int64_t n) { GRID_STRIDE(i, n) out[i] = (uint32_t)i; }

// input checks: errs[0] = min token with a word outside [0, V), errs[1] = min
// token with a document outside [lo, hi)
__global__ void k_check_tokens(const int32_t* doc, const int32_t* word, int64_t n, int64_t lo, int64_t hi, int V,
                               unsigned long long* errs) {
    GRID_STRIDE(i, n) {
        if (word[i] < 0 || word[i] >= V) atomicMin(errs, (unsigned long long)i);
        if (doc[i] < lo || doc[i] >= hi) atomicMin(errs + 1, (unsigned long long)i);
    }
}

__global__ void k_gather_docs(const uint32_t* perm, const int32_t* doc, int64_t n, int64_t lo, uint32_t* out_local) {
    GRID_STRIDE(p, n) out_local[p] = (uint32_t)(doc[perm[p]] - lo);
}

__device__ __forceinline__ uint64_t fin64(uint64_t z) {  // rng.py:20-26
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

// corpus.py:265-269: z = min(floor(u K), K - 1), u = Stream(seed, chunk)[p] in
// word-sorted order (rng.py:38-42: (fin(key + GOLDEN (ctr + 1)) >> 11) 2^-53)
__global__ void k_init_z(int64_t n, uint64_t key, int K, uint16_t* z) {
    GRID_STRIDE(p, n) {
        const double u = (double)(fin64(key + kGoldenD * ((uint64_t)p + 1ULL)) >> 11) * (1.0 / 9007199254740992.0);
        const int64_t zz = (int64_t)(u * (double)K);
        z[p] = (uint16_t)(zz < K - 1 ? zz : K - 1);
    }
}

// group heads of the word-sorted array
__global__ void k_word_heads(const uint32_t* word, int64_t n, uint32_t* flag) {
    GRID_STRIDE(p, n) flag[p] = (p == 0 || word[p] != word[p - 1]) ? 1u : 0u;
}

__global__ void k_group_scatter(const uint32_t* word, const uint32_t* flag, const uint32_t* idx, int64_t n,
                                int32_t* gw, uint32_t* go) {
    GRID_STRIDE(p, n) if (flag[p]) {
        gw[idx[p]] = (int32_t)word[p];
        go[idx[p]] = (uint32_t)p;
    }
}

__global__ void k_doc_hist(const uint32_t* doc, int64_t n, uint32_t* cnt) {
    GRID_STRIDE(p, n) atomicAdd(cnt + doc[p], 1u);
}

// (doc, word) run heads
__global__ void k_run_heads(const uint32_t* doc, const uint32_t* word, int64_t n, uint32_t* flag) {
    GRID_STRIDE(p, n) flag[p] = (p == 0 || word[p] != word[p - 1] || doc[p] != doc[p - 1]) ? 1u : 0u;
}

__global__ void k_run_scatter(const uint32_t* doc, const uint32_t* flag, const uint32_t* rid, int64_t n,
                              uint32_t* run_start, uint32_t* run_doc) {
    GRID_STRIDE(p, n) if (flag[p]) {
        run_start[rid[p]] = (uint32_t)p;
        run_doc[rid[p]] = doc[p];
    }
}

__global__ void k_gather_u32(const uint32_t* src, const uint32_t* idx, int64_t n, uint32_t* out) {
    GRID_STRIDE(i, n) out[i] = src[idx[i]];
}

// per run: its group and whether it starts a schedule segment (the group's
// first run, or a document-block change inside a block-scheduled group);
// seg0[r] = run_start[r] at segment heads (0 elsewhere) for a max-scan
__global__ void k_run_segments(int64_t R, const uint32_t* run_start, const uint32_t* run_doc, const uint32_t* word,
                               const int32_t* wgroup, const uint32_t* g_info, const uint32_t* g_run0,
                               const int32_t* doc_blk, uint32_t* run_group, uint32_t* seg0, uint8_t* seghead) {
    GRID_STRIDE(r, R) {
        const uint32_t g = (uint32_t)wgroup[word[run_start[r]]];
        const bool blocked = (g_info[g] >> 31) != 0u;
        const bool h = (uint32_t)r == g_run0[g] || (blocked && doc_blk[run_doc[r]] != doc_blk[run_doc[r - 1]]);
        run_group[r] = g;
        seghead[r] = h;
        seg0[r] = h ? run_start[r] : 0u;
    }
}

struct MaxOp {
    __device__ __forceinline__ uint32_t operator()(uint32_t a, uint32_t b) const { return a > b ? a : b; }
};

// slice heads: segment heads and every kSliceTokens-th token of a segment
__global__ void k_slice_heads(int64_t R, const uint32_t* run_start, const uint32_t* seg0, const uint8_t* seghead,
                              uint32_t* flag) {
    GRID_STRIDE(r, R) {
        bool h = seghead[r];
        if (!h) h = (run_start[r] - seg0[r]) / (uint32_t)kSliceTokens != (run_start[r - 1] - seg0[r]) / (uint32_t)kSliceTokens;
        flag[r] = h ? 1u : 0u;
    }
}

__global__ void k_slice_begin(int64_t R, const uint32_t* flag, const uint32_t* sid, uint32_t* srb) {
    GRID_STRIDE(r, R) if (flag[r]) srb[sid[r]] = (uint32_t)r;
}

// schedule key: document block (or round-robin for groups not block-scheduled)
// << 40 | heavy-first rank << 20 | slice ordinal inside its group
// (sampling phase << 56 on top when the schedule is split into phases)
__global__ void k_slice_keys(int64_t N, int64_t R, const uint32_t* srb, const uint32_t* run_group,
                             const uint32_t* run_doc, const int32_t* doc_blk, const uint32_t* g_info,
                             const uint32_t* g_slice0, const uint8_t* g_phase, const uint8_t* blk_phase, int nblk,
                             unsigned long long* key, uint32_t* val) {
    GRID_STRIDE(s, N) {
        const uint32_t r = srb[s], g = run_group[r];
        const bool blocked = (g_info[g] >> 31) != 0u;
        const uint64_t b = blocked ? (uint64_t)doc_blk[run_doc[r]] : (uint64_t)(s % nblk);
        // word phases: the group's phase; document-block phases: 0 for words
        // not cut at block boundaries, else the phase of the slice's block
        const uint64_t ph = blk_phase ? (blocked ? (uint64_t)blk_phase[b] : 0ull)
                                      : (g_phase ? (uint64_t)g_phase[g] : 0ull);
        key[s] = (ph << 56) | (b << 40) | ((uint64_t)(g_info[g] & 0xFFFFFu) << 20) | (uint64_t)((uint32_t)s - g_slice0[g]);
        val[s] = (uint32_t)s;
    }
}

__global__ void k_slice_emit(int64_t N, int64_t R, const uint32_t* order, const uint32_t* srb, const uint32_t* run_group,
                             const int32_t* gw, const int32_t* g_col, const int32_t* g_ctx, int4* slices,
                             int32_t* slice_ctx) {
    GRID_STRIDE(i, N) {
        const uint32_t s = order[i], r0 = srb[s];
        const uint32_t r1 = (int64_t)s + 1 < N ? srb[s + 1] : (uint32_t)R;
        const uint32_t g = run_group[r0];
        slices[i] = make_int4(gw[g], (int)r0, (int)r1, g_col[g]);
        slice_ctx[i] = g_ctx[g];
    }
}

// slices per phase of the sorted schedule (document-block phases)
__global__ void k_phase_counts(int64_t N, const unsigned long long* key, unsigned int* cnt) {
    GRID_STRIDE(i, N) atomicAdd(cnt + (key[i] >> 56), 1u);
}

// zdoc positions (heavy-first inside each document)
__global__ void k_inverse(int64_t T, const uint32_t* dw_tok, uint32_t* inv) { GRID_STRIDE(q, T) inv[dw_tok[q]] = (uint32_t)q; }

__global__ void k_heavy_flag(int64_t T, const uint32_t* dw_tok, const uint32_t* word, const int32_t* wgroup,
                             const uint32_t* g_info, uint32_t* hflag) {
    GRID_STRIDE(q, T + 1) hflag[q] = q < T ? (g_info[wgroup[word[dw_tok[q]]]] >> 31) : 0u;
}

__global__ void k_dwpos(int64_t R, const uint32_t* run_start, const uint32_t* run_doc, const uint32_t* run_group,
                        const uint32_t* g_info, const uint32_t* inv, const uint32_t* S, const uint32_t* dw_ptr,
                        uint32_t* dwpos) {
    GRID_STRIDE(r, R) {
        const uint32_t d = run_doc[r], b = dw_ptr[d], e = dw_ptr[d + 1], q = inv[run_start[r]];
        const uint32_t hb = S[b], hq = S[q] - hb;
        const bool heavy = (g_info[run_group[r]] >> 31) != 0u;
        dwpos[r] = heavy ? b + hq : b + (S[e] - hb) + (q - b) - hq;
    }
}

__global__ void k_run_rec(int64_t R, const uint32_t* run_doc, const uint32_t* run_start, const uint32_t* dwpos,
                          const uint2* meta, uint4* rec) {
    GRID_STRIDE(r, R) rec[r] = make_uint4(run_doc[r], run_start[r], dwpos[r], meta[run_doc[r]].x);
}

// gf_shard_load checks of an uploaded chunk (corpus.py:160-198 invariants):
// errs[0] token with z >= K, [1] token outside [lo, hi), [2] token outside its
// word group, [3] dw-map entry out of range
__global__ void k_check_chunk(int64_t T, int K, const uint16_t* z, const int32_t* doc, int64_t lo, int64_t hi,
                              const uint32_t* word, const int32_t* gw_expect, const uint32_t* dw_tok,
                              unsigned long long* errs) {
    GRID_STRIDE(t, T) {
        if (z[t] >= K) atomicMin(errs, (unsigned long long)t);
        if (doc[t] < lo || doc[t] >= hi) atomicMin(errs + 1, (unsigned long long)t);
        if ((int32_t)word[t] != gw_expect[t]) atomicMin(errs + 2, (unsigned long long)t);
        if (dw_tok[t] >= (uint32_t)T) atomicMin(errs + 3, (unsigned long long)t);
    }
}

__global__ void k_expand_groups(int64_t ng, const int32_t* gw, const int64_t* go, const int64_t* gs, int32_t* out) {
    for (int64_t g = blockIdx.x; g < ng; g += gridDim.x)
        for (int64_t t = go[g] + threadIdx.x; t < go[g] + gs[g]; t += blockDim.x) out[t] = gw[g];
}

__global__ void k_i64_to_u32(int64_t n, const int64_t* in, uint32_t* out) { GRID_STRIDE(i, n) out[i] = (uint32_t)in[i]; }
__global__ void k_u32_to_i64(int64_t n, const uint32_t* in, int64_t* out, int64_t add) {
    GRID_STRIDE(i, n) out[i] = (int64_t)in[i] + add;
}

int bits_for(uint64_t n) {
    int b = 1;
    while (b < 64 && (1ULL << b) < n) ++b;
    return b;
}

__global__ void k_u32_to_i32(int64_t n, const uint32_t* in, int32_t* out, int64_t add) {
    GRID_STRIDE(i, n) out[i] = (int32_t)((int64_t)in[i] + add);
}

struct Scratch {                              // temporaries of one preprocessing call
    std::vector<void*> ptrs;
    cudaError_t err = cudaSuccess;
    void* get(size_t bytes) {
        void* p = nullptr;
        if (err != cudaSuccess) return nullptr;
        err = cudaMalloc(&p, std::max<size_t>(bytes, 16));
        if (err != cudaSuccess) return nullptr;
        ptrs.push_back(p);
        return p;
    }
    uint32_t* u32(int64_t n) { return static_cast<uint32_t*>(get((size_t)std::max<int64_t>(n, 1) * 4)); }
    ~Scratch() {
        for (void* p : ptrs) cudaFree(p);
    }
};

template <class F>
cudaError_t cub_call(Scratch& sc, F f) {      // CUB size query + run
    size_t bytes = 0;
    cudaError_t e = f(nullptr, bytes);
    if (e != cudaSuccess) return e;
    void* tmp = sc.get(bytes);
    if (!tmp) return sc.err;
    return f(tmp, bytes);
}

// word-sorted chunk on the device (corpus.py:160-198 Chunk, local doc ids)
struct DevChunk {
    int64_t T = 0, D = 0, ng = 0;
    uint32_t* word = nullptr;                 // [T] word id per token
    uint32_t* doc = nullptr;                  // [T] local doc id per token
    uint32_t* perm = nullptr;                 // [T] doc-major index of each token (partition only)
    uint16_t* z = nullptr;                    // [T] assignments
    uint32_t* dw_ptr = nullptr;               // [D+1]
    uint32_t* dw_tok = nullptr;               // [T]
    int32_t* gw = nullptr;                    // [ng] group words (ascending)
    uint32_t* go = nullptr;                   // [ng+1] group offsets (+ T)
};

// checked async calls: cudaError_t-returning helpers propagate, the ABI-facing
// loaders turn a failure into the shard error text
#define GF_TRY(call)                                         \
    do {                                                     \
        const cudaError_t _e = (call);                       \
        if (_e != cudaSuccess) return _e;                    \
    } while (0)
#define GF_TRY_RC(call, what)                                \
    do {                                                     \
        const cudaError_t _e = (call);                       \
        if (_e != cudaSuccess) return shard_cuda_fail(_e, what); \
    } while (0)

int64_t read_u32(cudaStream_t st, const uint32_t* p) {   // a failure leaves 0 and resurfaces at the next check
    uint32_t v = 0;
    if (cudaMemcpyAsync(&v, p, 4, cudaMemcpyDeviceToHost, st) == cudaSuccess) cudaStreamSynchronize(st);
    return v;
}

// corpus.py:240-287 partition of one chunk, on the device
cudaError_t partition_device(Scratch& sc, cudaStream_t st, const int32_t* d_doc, const int32_t* d_word, int64_t n,
                             int64_t lo, int64_t hi, int V, int K, uint64_t zkey, DevChunk& c,
                             unsigned long long* d_errs) {
    const int64_t D = hi - lo;
    c = DevChunk{};
    c.T = n;
    c.D = D;
    c.word = sc.u32(n);
    c.doc = sc.u32(n);
    c.perm = sc.u32(n);
    c.dw_tok = sc.u32(n);
    c.dw_ptr = sc.u32(D + 1);
    c.z = static_cast<uint16_t*>(sc.get((size_t)std::max<int64_t>(n, 1) * 2));
    uint32_t* ta = sc.u32(std::max(n, D) + 1);
    uint32_t* tb = sc.u32(std::max(n, D) + 1);
    if (sc.err != cudaSuccess) return sc.err;
    cudaError_t e;
    if (n > 0) {
        k_check_tokens<<<blocks_for(n), 256, 0, st>>>(d_doc, d_word, n, lo, hi, V, d_errs);
        // stable LSD radix sort by word: ties keep the input (corpus) order
        k_iota<<<blocks_for(n), 256, 0, st>>>(ta, n);
        e = cub_call(sc, [&](void* t, size_t& b) {
            return cub::DeviceRadixSort::SortPairs(t, b, reinterpret_cast<const uint32_t*>(d_word), c.word, ta, c.perm,
                                                   n, 0, bits_for((uint64_t)V), st);
        });
        if (e != cudaSuccess) return e;
        k_gather_docs<<<blocks_for(n), 256, 0, st>>>(c.perm, d_doc, n, lo, c.doc);
        k_init_z<<<blocks_for(n), 256, 0, st>>>(n, zkey, K, c.z);
        // group directory (np.unique: ascending words, first offsets)
        k_word_heads<<<blocks_for(n), 256, 0, st>>>(c.word, n, ta);
        e = cub_call(sc, [&](void* t, size_t& b) { return cub::DeviceScan::ExclusiveSum(t, b, ta, tb, n, st); });
        if (e != cudaSuccess) return e;
        c.ng = read_u32(st, ta + n - 1) + read_u32(st, tb + n - 1);
    }
    c.gw = static_cast<int32_t*>(sc.get((size_t)std::max<int64_t>(c.ng, 1) * 4));
    c.go = sc.u32(c.ng + 1);
    if (sc.err != cudaSuccess) return sc.err;
    if (n > 0) k_group_scatter<<<blocks_for(n), 256, 0, st>>>(c.word, ta, tb, n, c.gw, c.go);
    const uint32_t tn = (uint32_t)n;
    GF_TRY(cudaMemcpyAsync(c.go + c.ng, &tn, 4, cudaMemcpyHostToDevice, st));
    // doc-word map: histogram -> dw_ptr; stable sort of positions by local doc -> dw_tok
    GF_TRY(cudaMemsetAsync(ta, 0, (size_t)(D + 1) * 4, st));
    if (n > 0) k_doc_hist<<<blocks_for(n), 256, 0, st>>>(c.doc, n, ta);
    e = cub_call(sc, [&](void* t, size_t& b) { return cub::DeviceScan::ExclusiveSum(t, b, ta, c.dw_ptr, D + 1, st); });
    if (e != cudaSuccess) return e;
    if (n > 0) {
        k_iota<<<blocks_for(n), 256, 0, st>>>(tb, n);
        e = cub_call(sc, [&](void* t, size_t& b) {
            return cub::DeviceRadixSort::SortPairs(t, b, c.doc, ta, tb, c.dw_tok, n, 0,
                                                   bits_for((uint64_t)std::max<int64_t>(D, 2)), st);
        });
        if (e != cudaSuccess) return e;
    }
    return cudaGetLastError();
}

}  // namespace

// ====================================================================== API ==
// K2 layout of the shard from a device chunk: runs, slices, contexts, items,
// zdoc positions, theta capacities (the device half of gf_shard_load).
static int build_layout(gf_shard* s, Scratch& sc, DevChunk& c, int64_t lo, int64_t hi) {
    cudaStream_t st = s->stream;
    const int K = s->K, V = s->V;
    const int64_t T = c.T, D = c.D, ng = c.ng;
#define CK(x, what)                                              \
    do {                                                         \
        cudaError_t _e = (x);                                    \
        if (_e != cudaSuccess) return shard_cuda_fail(_e, what); \
    } while (0)
    CK(sc.err, "layout scratch");
    // ---- host copies of the O(V) / O(D) directory data ----
    std::vector<int32_t> gw((size_t)ng);
    std::vector<uint32_t> go((size_t)ng + 1), dwp((size_t)D + 1);
    if (ng) CK(cudaMemcpyAsync(gw.data(), c.gw, ng * 4, cudaMemcpyDeviceToHost, st), "layout");
    CK(cudaMemcpyAsync(go.data(), c.go, (ng + 1) * 4, cudaMemcpyDeviceToHost, st), "layout");
    CK(cudaMemcpyAsync(dwp.data(), c.dw_ptr, (D + 1) * 4, cudaMemcpyDeviceToHost, st), "layout");
    CK(cudaStreamSynchronize(st), "layout");
    // ---- phi layout ----
    if (s->global_freq.empty()) {
        s->global_freq.assign(V, 0);
        for (int64_t g = 0; g < ng; ++g) s->global_freq[gw[g]] += go[g + 1] - go[g];
    }
    if (int rc = shard_set_layout(s)) return rc;
    // ---- (doc, word) runs ----
    uint32_t* flag = sc.u32(T + 1);
    uint32_t* rid = sc.u32(T + 1);
    CK(sc.err, "layout scratch");
    int64_t R = 0;
    if (T > 0) {
        k_run_heads<<<blocks_for(T), 256, 0, st>>>(c.doc, c.word, T, flag);
        CK(cub_call(sc, [&](void* t, size_t& b) { return cub::DeviceScan::ExclusiveSum(t, b, flag, rid, T, st); }), "runs");
        R = read_u32(st, flag + T - 1) + read_u32(st, rid + T - 1);
    }
    // ---- theta capacities, document blocks, loglik constant (host, O(D)) ----
    // Defaults from the corpus: short documents (mean theta-row capacity < 200
    // entries, e.g. PubMed-shape) give short rows whose reads are latency-bound,
    // so tighter L2-resident blocks pay; long documents (NYTimes-shape) prefer
    // fewer, larger blocks (fewer slices).  Measured optima: 24 MB / 128 runs
    // and 64 MB / 256 runs.
    int64_t cap_entries = 0;
    for (int64_t d = 0; d < D; ++d) cap_entries += (std::min<int64_t>(K, (int64_t)dwp[d + 1] - dwp[d]) + 7) & ~7LL;
    const bool short_docs = D > 0 && cap_entries < 200 * D;
    const int64_t blk_bytes = shard_env_int("GF_DOCBLOCK_KB", short_docs ? 24 << 10 : 64 << 10) << 10;
    // a word is block-scheduled when it has >= min_runs runs per document block
    // on average (its per-block slices then amortise the context copy)
    const int64_t min_runs = shard_env_int("GF_SLICE_MINRUNS", short_docs ? 128 : 256);
    std::vector<uint2> meta((size_t)D);
    std::vector<int32_t> doc_blk((size_t)D);
    uint64_t cap = 0;
    double llc = 0.0;
    int32_t nblk = 0;
    {
        int64_t acc = 0;
        for (int64_t d = 0; d < D; ++d) {
            const int64_t L = (int64_t)dwp[d + 1] - dwp[d];
            const int64_t ent = (std::min<int64_t>(K, L) + 7) & ~7LL;   // 32-byte granules (K1 256-bit loads)
            meta[d] = make_uint2((uint32_t)cap, 0u);
            cap += (uint64_t)ent;
            if (cap >= (uint64_t)UINT32_MAX) return shard_fail(GF_ERR_CAPACITY, "theta rows exceed 2^32 entries");
            if (acc > 0 && acc + 4 * ent > blk_bytes) { ++nblk; acc = 0; }
            doc_blk[d] = nblk;
            acc += 4 * ent;
            if (L > 0) llc += (double)L * std::log((double)L + (double)K * s->alpha);
        }
        ++nblk;
    }
    // ---- device buffers of the shard ----
    shard_free_device(s);
    auto& dv = s->d;
    int rc;
    // z, zdoc: + 8 tokens, K2 / K3 bulk-prefetch whole 16-byte vectors of a range
    if ((rc = shard_alloc(&dv.z, T + 8, "z")) || (rc = shard_alloc(&dv.run_doc, R, "runs")) ||
        (rc = shard_alloc(&dv.run_start, R + 1, "runs")) || (rc = shard_alloc(&dv.run_dwpos, R, "runs")) || (rc = shard_alloc(&dv.run_rec, R, "runs")) ||
        (rc = shard_alloc(&dv.dw_ptr, D + 1, "dw_ptr")) || (rc = shard_alloc(&dv.zdoc, T + 8, "zdoc")) ||
        (rc = shard_alloc(&dv.theta_ent, cap + 8, "theta")) || (rc = shard_alloc(&dv.theta_meta, D, "theta")) ||
        (rc = shard_alloc(&dv.sync, s->sync_u32 + 1, "phi")) || (rc = shard_alloc(&dv.inv_den, 2 * K, "inv_den")) ||
        (rc = shard_alloc(&dv.ll_sum, kLlSlots, "ll")) || (rc = shard_alloc(&dv.errs, 4, "errs")) ||
        (rc = shard_alloc(&dv.bytes, 2, "bytes")))
        return rc;
    if (T > 0) {
        k_run_scatter<<<blocks_for(T), 256, 0, st>>>(c.doc, flag, rid, T, dv.run_start, dv.run_doc);
        CK(cudaMemcpyAsync(dv.z, c.z, T * 2, cudaMemcpyDeviceToDevice, st), "layout");
    }
    const uint32_t tT = (uint32_t)T;
    CK(cudaMemcpyAsync(dv.run_start + R, &tT, 4, cudaMemcpyHostToDevice, st), "layout");
    CK(cudaMemcpyAsync(dv.dw_ptr, c.dw_ptr, (D + 1) * 4, cudaMemcpyDeviceToDevice, st), "layout");
    CK(cudaMemcpyAsync(dv.theta_meta, meta.data(), D * sizeof(uint2), cudaMemcpyHostToDevice, st), "layout");
    // ---- groups: first run, heavy-first rank, block scheduling, phi column ----
    uint32_t* d_go = c.go;
    uint32_t* d_grun0 = sc.u32(ng + 1);
    CK(sc.err, "layout scratch");
    std::vector<uint32_t> grun0((size_t)ng + 1, (uint32_t)R);
    if (ng) {
        k_gather_u32<<<blocks_for(ng), 256, 0, st>>>(rid, d_go, ng, d_grun0);
        CK(cudaMemcpyAsync(grun0.data(), d_grun0, ng * 4, cudaMemcpyDeviceToHost, st), "layout");
        CK(cudaStreamSynchronize(st), "layout");
    }
    grun0[ng] = (uint32_t)R;
    CK(cudaMemcpyAsync(d_grun0 + ng, &grun0[ng], 4, cudaMemcpyHostToDevice, st), "layout");
    std::vector<int64_t> order((size_t)ng);
    std::iota(order.begin(), order.end(), 0);
    std::sort(order.begin(), order.end(), [&](int64_t a, int64_t b) {   // sort_word_groups_desc (corpus.py:290-302)
        const uint32_t sa = go[a + 1] - go[a], sb = go[b + 1] - go[b];
        return sa != sb ? sa > sb : gw[a] < gw[b];
    });
    std::vector<uint32_t> ginfo((size_t)ng);
    std::vector<int32_t> gcol((size_t)ng), wgroup((size_t)V, 0);
    for (int64_t i = 0; i < ng; ++i) ginfo[order[i]] = (uint32_t)i;   // rank < 2^20 (V <= 2^20)
    if (ng > (1 << 20)) return shard_fail(GF_ERR_CAPACITY, "more than 2^20 word groups in one shard");
    for (int64_t g = 0; g < ng; ++g) {
        const int64_t runs = (int64_t)grun0[g + 1] - grun0[g];
        if (nblk > 1 && runs >= min_runs * nblk) ginfo[g] |= 0x80000000u;   // block-scheduled word
        gcol[g] = s->word_col[gw[g]];
        wgroup[gw[g]] = (int32_t)g;
    }
    uint32_t* d_ginfo = sc.u32(ng);
    int32_t* d_gcol = reinterpret_cast<int32_t*>(sc.u32(ng));
    int32_t* d_wgroup = reinterpret_cast<int32_t*>(sc.u32(V));
    int32_t* d_docblk = reinterpret_cast<int32_t*>(sc.u32(D));
    CK(sc.err, "layout scratch");
    if (ng) {
        CK(cudaMemcpyAsync(d_ginfo, ginfo.data(), ng * 4, cudaMemcpyHostToDevice, st), "layout");
        CK(cudaMemcpyAsync(d_gcol, gcol.data(), ng * 4, cudaMemcpyHostToDevice, st), "layout");
    }
    CK(cudaMemcpyAsync(d_wgroup, wgroup.data(), (size_t)V * 4, cudaMemcpyHostToDevice, st), "layout");
    if (D) CK(cudaMemcpyAsync(d_docblk, doc_blk.data(), D * 4, cudaMemcpyHostToDevice, st), "layout");
    // ---- slices: schedule segments, kSliceTokens pieces ----
    uint32_t* run_group = sc.u32(R);
    uint32_t* seg0 = sc.u32(R);
    uint8_t* seghead = static_cast<uint8_t*>(sc.get((size_t)std::max<int64_t>(R, 1)));
    uint32_t* sflag = sc.u32(R + 1);
    uint32_t* sid = sc.u32(R + 1);
    CK(sc.err, "layout scratch");
    int64_t N = 0;
    if (R > 0) {
        k_run_segments<<<blocks_for(R), 256, 0, st>>>(R, dv.run_start, dv.run_doc, c.word, d_wgroup, d_ginfo, d_grun0,
                                                      d_docblk, run_group, seg0, seghead);
        CK(cub_call(sc, [&](void* t, size_t& b) {
               return cub::DeviceScan::InclusiveScan(t, b, seg0, seg0, MaxOp(), R, st);
           }),
           "slices");
        k_slice_heads<<<blocks_for(R), 256, 0, st>>>(R, dv.run_start, seg0, seghead, sflag);
        CK(cub_call(sc, [&](void* t, size_t& b) { return cub::DeviceScan::ExclusiveSum(t, b, sflag, sid, R, st); }),
           "slices");
        N = read_u32(st, sflag + R - 1) + read_u32(st, sid + R - 1);
    }
    if (N >= (int64_t)INT32_MAX) return shard_fail(GF_ERR_CAPACITY, "too many slices");
    uint32_t* srb = sc.u32(N + 1);
    CK(sc.err, "layout scratch");
    if (R > 0) k_slice_begin<<<blocks_for(R), 256, 0, st>>>(R, sflag, sid, srb);
    // slices per group (first slice of group g = sid[grun0[g]]) -> word contexts
    std::vector<uint32_t> gslice0((size_t)ng + 1, (uint32_t)N);
    uint32_t* d_gslice0 = sc.u32(ng + 1);
    CK(sc.err, "layout scratch");
    if (ng) {
        k_gather_u32<<<blocks_for(ng), 256, 0, st>>>(sid, d_grun0, ng, d_gslice0);
        CK(cudaMemcpyAsync(gslice0.data(), d_gslice0, ng * 4, cudaMemcpyDeviceToHost, st), "layout");
        CK(cudaStreamSynchronize(st), "layout");
    }
    gslice0[ng] = (uint32_t)N;
    std::vector<int32_t> gctx((size_t)ng, -1), ctx_cols;
    std::vector<uint32_t> gnsl((size_t)ng);
    for (int64_t g = 0; g < ng; ++g) {
        gnsl[g] = gslice0[g + 1] - gslice0[g];
        if (gnsl[g] > (1u << 20)) return shard_fail(GF_ERR_CAPACITY, "a word has more than 2^20 slices");
        if (gnsl[g] > 1) { gctx[g] = (int32_t)ctx_cols.size(); ctx_cols.push_back(gcol[g]); }
    }
    // sampling phases: word groups cut into P contiguous z ranges of ~T/P tokens
    // (groups are in ascending word order, so phase p's tokens are one z range)
    const int P = std::max(1, std::min(s->n_phases, 255));
    if (nblk >= (1 << 16)) return shard_fail(GF_ERR_CAPACITY, "more than 2^16 document blocks");
    std::vector<uint8_t> gphase((size_t)ng, 0);
    s->phase_slice0.assign((size_t)P + 1, 0);
    s->phase_tok0.assign((size_t)P + 1, T);
    s->phase_tok0[0] = 0;
    for (int64_t g = 0; g < ng; ++g) {
        int ph = 0;
        if (T > 0 && (int)s->phase_cuts.size() == P) {   // phase p ends at token cut[p] * T
            while (ph < P - 1 && (double)go[g] >= s->phase_cuts[ph] * (double)T) ++ph;
        } else if (T > 0) {
            ph = (int)std::min<int64_t>(P - 1, (int64_t)go[g] * P / T);
        }
        gphase[g] = (uint8_t)ph;
        s->phase_slice0[ph + 1] += gnsl[g];
    }
    for (int p = P - 1; p >= 1; --p)   // first token of phase p = first group of phase >= p
        for (int64_t g = 0; g < ng; ++g)
            if (gphase[g] >= p) { s->phase_tok0[p] = go[g]; break; }
    for (int p = 0; p < P; ++p) s->phase_slice0[p + 1] += s->phase_slice0[p];
    // document-block phases: block b joins phase 1 + (the first cut above the
    // doc-major token fraction at its first document); phase 0 holds the
    // words that are not cut at block boundaries
    const bool bphase = s->block_phases && P > 1;
    std::vector<uint8_t> blkphase((size_t)nblk, 0);
    s->phase_doctok0.assign((size_t)P + 1, T);
    s->phase_doctok0[0] = 0;
    s->phase_doctok0[1] = 0;
    if (bphase) {
        std::vector<int64_t> blk_tok0((size_t)nblk + 1, T);
        for (int64_t d = D - 1; d >= 0; --d) blk_tok0[doc_blk[d]] = dwp[d];
        for (int32_t b = 0; b < nblk; ++b) {
            int ph = 1;
            const double f = T > 0 ? (double)blk_tok0[b] / (double)T : 0.0;
            while (ph < P - 1 && f >= s->phase_cuts[ph - 1]) ++ph;
            blkphase[b] = (uint8_t)ph;
        }
        for (int p = P - 1; p >= 2; --p)   // first doc-major token of phase p
            for (int32_t b = 0; b < nblk; ++b)
                if (blkphase[b] >= p) { s->phase_doctok0[p] = blk_tok0[b]; break; }
        gphase.assign(gphase.size(), 0);
    }
    uint8_t* d_gphase = nullptr;
    uint8_t* d_blkphase = nullptr;
    if (bphase) {
        d_blkphase = static_cast<uint8_t*>(sc.get((size_t)std::max<int32_t>(nblk, 1)));
        CK(sc.err, "layout scratch");
        CK(cudaMemcpyAsync(d_blkphase, blkphase.data(), nblk, cudaMemcpyHostToDevice, st), "layout");
    } else if (P > 1) {
        d_gphase = static_cast<uint8_t*>(sc.get((size_t)std::max<int64_t>(ng, 1)));
        CK(sc.err, "layout scratch");
        if (ng) CK(cudaMemcpyAsync(d_gphase, gphase.data(), ng, cudaMemcpyHostToDevice, st), "layout");
    }
    int32_t* d_gctx = reinterpret_cast<int32_t*>(sc.u32(ng));
    uint32_t* d_gnsl = sc.u32(ng);
    unsigned long long* skey = static_cast<unsigned long long*>(sc.get((size_t)std::max<int64_t>(N, 1) * 8));
    unsigned long long* skey2 = static_cast<unsigned long long*>(sc.get((size_t)std::max<int64_t>(N, 1) * 8));
    uint32_t* sval = sc.u32(N);
    uint32_t* sorder = sc.u32(N);
    CK(sc.err, "layout scratch");
    if (ng) {
        CK(cudaMemcpyAsync(d_gctx, gctx.data(), ng * 4, cudaMemcpyHostToDevice, st), "layout");
        CK(cudaMemcpyAsync(d_gnsl, gnsl.data(), ng * 4, cudaMemcpyHostToDevice, st), "layout");
    }
    if ((rc = shard_alloc(&dv.slices, N, "slices")) || (rc = shard_alloc(&dv.slice_ctx, N, "slices")) ||
        (rc = shard_alloc(&dv.ll_part, N, "ll")) || (rc = shard_alloc(&dv.ctx_cols, ctx_cols.size(), "contexts")) ||
        (rc = shard_alloc(&dv.ctx_tab, ctx_cols.size() * context_floats(s), "contexts")))
        return rc;
    if (!ctx_cols.empty())
        CK(cudaMemcpyAsync(dv.ctx_cols, ctx_cols.data(), ctx_cols.size() * 4, cudaMemcpyHostToDevice, st), "layout");
    if (N > 0) {
        // block-major, heavy-first inside a block, slice order inside a word
        k_slice_keys<<<blocks_for(N), 256, 0, st>>>(N, R, srb, run_group, dv.run_doc, d_docblk, d_ginfo, d_gslice0,
                                                   d_gphase, d_blkphase, nblk, skey, sval);
        CK(cub_call(sc, [&](void* t, size_t& b) {
               return cub::DeviceRadixSort::SortPairs(t, b, skey, skey2, sval, sorder, N, 0, 64, st);
           }),
           "slices");
        if (bphase) {                           // slices per phase from the sorted keys
            unsigned int* pc = sc.u32(P);
            CK(sc.err, "layout scratch");
            CK(cudaMemsetAsync(pc, 0, (size_t)P * 4, st), "layout");
            k_phase_counts<<<blocks_for(N), 256, 0, st>>>(N, skey2, pc);
            std::vector<unsigned int> cnt((size_t)P);
            CK(cudaMemcpyAsync(cnt.data(), pc, (size_t)P * 4, cudaMemcpyDeviceToHost, st), "layout");
            CK(cudaStreamSynchronize(st), "layout");
            s->phase_slice0.assign((size_t)P + 1, 0);
            for (int p = 0; p < P; ++p) s->phase_slice0[p + 1] = s->phase_slice0[p] + cnt[p];
        }
        k_slice_emit<<<blocks_for(N), 256, 0, st>>>(N, R, sorder, srb, run_group, c.gw, d_gcol, d_gctx, dv.slices,
                                                    dv.slice_ctx);
    }
    // ---- K2 work items (host, O(groups)): one per u16-column (light) group,
    // whose packed column the item writes densely (<= 65535 tokens); a
    // u32-column (heavy) group is cut into pieces of <= kK2Piece tokens, each
    // flushed with global atomics into its pre-zeroed column -- few enough
    // atomics (K per piece) and pieces small enough to balance the warps.
    // Independent of K1's slices.  Longest first, so no long item starts last;
    // light words absent from this shard still own a 16-bit column (K2 writes
    // every light column densely, no memset of the light region), so each
    // absent one gets an empty item that writes its zeros. ----
    const int64_t piece = std::max<int64_t>(1024, shard_env_int("GF_K2_PIECE", 16384));
    std::vector<int4> items;
    items.reserve((size_t)ng + (size_t)(T / piece) + 16);
    {
        std::vector<uint8_t> present((size_t)V, 0);
        for (int64_t g = 0; g < ng; ++g) {
            present[gw[g]] = 1;
            const int32_t col = s->word_col[gw[g]];
            const int64_t t0 = go[g], t1 = go[g + 1];
            if (col >= 0) {
                items.push_back(make_int4(col, (int)t0, (int)t1, 0));
            } else {
                for (int64_t a = t0; a < t1; a += piece)
                    items.push_back(make_int4(col, (int)a, (int)std::min(t1, a + piece), 1));
            }
        }
        std::stable_sort(items.begin(), items.end(), [](const int4& a, const int4& b) { return a.z - a.y > b.z - b.y; });
        for (int32_t v = 0; v < V; ++v)
            if (!present[v] && s->word_col[v] >= 0) items.push_back(make_int4(s->word_col[v], 0, 0, 0));
    }
    const int64_t M0 = (int64_t)items.size();
    if ((rc = shard_alloc(&dv.k2items, M0, "items"))) return rc;
    if (M0) CK(cudaMemcpyAsync(dv.k2items, items.data(), M0 * sizeof(int4), cudaMemcpyHostToDevice, st), "items");
    CK(cudaStreamSynchronize(st), "items");            // `items` is freed at scope end
    int64_t M = M0;
    // ---- zdoc positions: heavy-first inside each document ----
    if (T > 0) {
        uint32_t* inv = flag;                 // reuse: [T]
        uint32_t* hflag = rid;                // reuse: [T+1]
        uint32_t* S = sc.u32(T + 1);
        CK(sc.err, "layout scratch");
        k_inverse<<<blocks_for(T), 256, 0, st>>>(T, c.dw_tok, inv);
        k_heavy_flag<<<blocks_for(T + 1), 256, 0, st>>>(T, c.dw_tok, c.word, d_wgroup, d_ginfo, hflag);
        CK(cub_call(sc, [&](void* t, size_t& b) { return cub::DeviceScan::ExclusiveSum(t, b, hflag, S, T + 1, st); }),
           "zdoc");
        k_dwpos<<<blocks_for(R), 256, 0, st>>>(R, dv.run_start, dv.run_doc, run_group, d_ginfo, inv, S, c.dw_ptr,
                                               dv.run_dwpos);
        k_run_rec<<<blocks_for(R), 256, 0, st>>>(R, dv.run_doc, dv.run_start, dv.run_dwpos, dv.theta_meta, dv.run_rec);
    }
    CK(cudaMemsetAsync(dv.theta_ent, 0, (cap + 8) * 4, st), "memset");
    CK(cudaMemsetAsync(dv.sync, 0, s->sync_u32 * 4, st), "memset");
    CK(cudaMemsetAsync(dv.errs, 0xff, 32, st), "memset");
    CK(cudaMemsetAsync(dv.ll_sum, 0, kLlSlots * sizeof(double), st), "memset");
    CK(cudaMemsetAsync(dv.bytes, 0, 8, st), "memset");
    s->doc_lo = lo;
    s->doc_hi = hi;
    s->D = D;
    s->T = T;
    s->R = R;
    s->n_slices = N;
    s->n_k2 = M;
    s->n_ctx = (int64_t)ctx_cols.size();
    s->n_doc_blocks = nblk;
    s->ctx_dirty = true;
    s->theta_cap = (int64_t)cap;
    s->ll_const = llc;
    CK(launch_zdoc_sync(s), "zdoc");
    CK(cudaStreamSynchronize(st), "layout");
    s->loaded = true;
    return GF_OK;
#undef CK
}

// gf_shard_load: the reference Chunk arrays (host) -> device checks -> layout
int load_chunk(gf_shard* s, int64_t lo, int64_t hi, int64_t T, const int32_t* doc_ids, const int32_t* word_ids,
               const uint16_t* z, int64_t ng, const int32_t* gw, const int64_t* go, const int64_t* gs,
               const int64_t* dw_ptr, const int64_t* dw_tok) {
    cudaStream_t st = s->stream;
    const int64_t D = hi - lo;
    Scratch sc;
    DevChunk c;
    c.T = T;
    c.D = D;
    c.ng = ng;
    int32_t* d_doc = reinterpret_cast<int32_t*>(sc.u32(T));
    c.word = sc.u32(T);
    c.doc = sc.u32(T);
    c.z = static_cast<uint16_t*>(sc.get((size_t)std::max<int64_t>(T, 1) * 2));
    c.dw_tok = sc.u32(T);
    c.dw_ptr = sc.u32(D + 1);
    c.gw = reinterpret_cast<int32_t*>(sc.u32(ng));
    c.go = sc.u32(ng + 1);
    int64_t* d_i64 = static_cast<int64_t*>(sc.get((size_t)std::max<int64_t>(std::max(T, D + 1), 3 * ng) * 8));
    int32_t* expect = reinterpret_cast<int32_t*>(sc.u32(T));
    unsigned long long* errs = static_cast<unsigned long long*>(sc.get(4 * 8));
    if (sc.err != cudaSuccess) return shard_cuda_fail(sc.err, "load");
#define CK(x, what)                                              \
    do {                                                         \
        cudaError_t _e = (x);                                    \
        if (_e != cudaSuccess) return shard_cuda_fail(_e, what); \
    } while (0)
    CK(cudaMemsetAsync(errs, 0xff, 32, st), "load");
    if (T > 0) {
        CK(cudaMemcpyAsync(d_doc, doc_ids, T * 4, cudaMemcpyHostToDevice, st), "upload");
        CK(cudaMemcpyAsync(c.word, word_ids, T * 4, cudaMemcpyHostToDevice, st), "upload");
        CK(cudaMemcpyAsync(c.z, z, T * 2, cudaMemcpyHostToDevice, st), "upload");
        CK(cudaMemcpyAsync(d_i64, dw_tok, T * 8, cudaMemcpyHostToDevice, st), "upload");
        k_i64_to_u32<<<blocks_for(T), 256, 0, st>>>(T, d_i64, c.dw_tok);
    }
    CK(cudaMemcpyAsync(d_i64, dw_ptr, (D + 1) * 8, cudaMemcpyHostToDevice, st), "upload");
    k_i64_to_u32<<<blocks_for(D + 1), 256, 0, st>>>(D + 1, d_i64, c.dw_ptr);
    if (T > 0) {
        // local doc ids (checked below) and the expected word of every token
        k_u32_to_i32<<<blocks_for(T), 256, 0, st>>>(T, reinterpret_cast<const uint32_t*>(d_doc),
                                                     reinterpret_cast<int32_t*>(c.doc), -lo);
    }
    if (ng) {
        std::vector<uint32_t> go32((size_t)ng + 1);
        for (int64_t g = 0; g < ng; ++g) go32[g] = (uint32_t)go[g];
        go32[ng] = (uint32_t)T;
        CK(cudaMemcpyAsync(c.gw, gw, ng * 4, cudaMemcpyHostToDevice, st), "upload");
        CK(cudaMemcpyAsync(c.go, go32.data(), (ng + 1) * 4, cudaMemcpyHostToDevice, st), "upload");
        int64_t* dgo = d_i64 + 0;
        CK(cudaStreamSynchronize(st), "upload");           // d_i64 reused below
        CK(cudaMemcpyAsync(dgo, go, ng * 8, cudaMemcpyHostToDevice, st), "upload");
        CK(cudaMemcpyAsync(dgo + ng, gs, ng * 8, cudaMemcpyHostToDevice, st), "upload");
        int32_t* dgw = c.gw;
        k_expand_groups<<<(unsigned)std::min<int64_t>(ng, (int64_t)sm_count(s->device) * 32), 256, 0, st>>>(ng, dgw, dgo, dgo + ng, expect);
    } else {
        const uint32_t tn = (uint32_t)T;
        CK(cudaMemcpyAsync(c.go, &tn, 4, cudaMemcpyHostToDevice, st), "upload");
    }
    if (T > 0)
        k_check_chunk<<<blocks_for(T), 256, 0, st>>>(T, s->K, c.z, d_doc, lo, hi, c.word, expect, c.dw_tok, errs);
    unsigned long long e[4];
    CK(cudaMemcpyAsync(e, errs, 32, cudaMemcpyDeviceToHost, st), "load");
    CK(cudaStreamSynchronize(st), "load");
    if (e[0] != ~0ULL) {
        uint16_t zz = 0;
        CK(cudaMemcpy(&zz, c.z + e[0], 2, cudaMemcpyDeviceToHost), "load");
        return shard_fail(GF_ERR_SHAPE, "assignment %d at token %lld >= K=%d", (int)zz, (long long)e[0], s->K);
    }
    if (e[1] != ~0ULL)
        return shard_fail(GF_ERR_SHAPE, "token %lld: document %d outside [%lld, %lld)", (long long)e[1],
                          doc_ids[e[1]], (long long)lo, (long long)hi);
    if (e[2] != ~0ULL) return shard_fail(GF_ERR_SHAPE, "token %lld is not in its word group", (long long)e[2]);
    if (e[3] != ~0ULL) return shard_fail(GF_ERR_SHAPE, "doc-word map entry out of range");
    return build_layout(s, sc, c, lo, hi);
#undef CK
}

// gf_shard_load_tokens: doc-major tokens (host) -> device partition -> layout
int load_tokens(gf_shard* s, int64_t lo, int64_t hi, int64_t T, const int32_t* doc_ids, const int32_t* word_ids,
                uint64_t zkey) {
    cudaStream_t st = s->stream;
    Scratch sc;
    int32_t* d_doc = reinterpret_cast<int32_t*>(sc.u32(T));
    int32_t* d_word = reinterpret_cast<int32_t*>(sc.u32(T));
    unsigned long long* errs = static_cast<unsigned long long*>(sc.get(16));
    if (sc.err != cudaSuccess) return shard_cuda_fail(sc.err, "load_tokens");
    GF_TRY_RC(cudaMemsetAsync(errs, 0xff, 16, st), "partition");
    if (T > 0) {
        GF_TRY_RC(cudaMemcpyAsync(d_doc, doc_ids, T * 4, cudaMemcpyHostToDevice, st), "partition");
        GF_TRY_RC(cudaMemcpyAsync(d_word, word_ids, T * 4, cudaMemcpyHostToDevice, st), "partition");
    }
    DevChunk c;
    cudaError_t e = partition_device(sc, st, d_doc, d_word, T, lo, hi, s->V, s->K, zkey, c, errs);
    if (e != cudaSuccess) return shard_cuda_fail(e, "partition");
    unsigned long long he[2];
    GF_TRY_RC(cudaMemcpyAsync(he, errs, 16, cudaMemcpyDeviceToHost, st), "partition");
    if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return shard_cuda_fail(e, "partition");
    if (he[0] != ~0ULL) return shard_fail(GF_ERR_VALUE, "word id outside [0, vocab_size)");
    if (he[1] != ~0ULL) return shard_fail(GF_ERR_VALUE, "doc id %d outside chunk range", doc_ids[he[1]]);
    return build_layout(s, sc, c, lo, hi);
}

// gf_partition_chunk_gpu: the reference Chunk arrays of one chunk, computed on
// the device (bit-identical to gf_partition_chunk / corpus.partition)
int partition_to_host(int device, const int32_t* doc_ids, const int32_t* word_ids, int64_t n, int64_t lo, int64_t hi,
                      int32_t V, int32_t K, uint64_t zkey, int32_t* out_doc, int32_t* out_word, uint16_t* out_z,
                      int32_t* gw, int64_t* go, int64_t* gs, int64_t* ng_out, int64_t* dw_ptr, int64_t* dw_tok) {
    cudaSetDevice(device);
    cudaStream_t st = nullptr;
    Scratch sc;
    const int64_t D = hi - lo;
    int32_t* d_doc = reinterpret_cast<int32_t*>(sc.u32(n));
    int32_t* d_word = reinterpret_cast<int32_t*>(sc.u32(n));
    unsigned long long* errs = static_cast<unsigned long long*>(sc.get(16));
    if (sc.err != cudaSuccess) return shard_cuda_fail(sc.err, "partition");
    GF_TRY_RC(cudaMemsetAsync(errs, 0xff, 16, st), "partition");
    if (n > 0) {
        GF_TRY_RC(cudaMemcpyAsync(d_doc, doc_ids, n * 4, cudaMemcpyHostToDevice, st), "partition");
        GF_TRY_RC(cudaMemcpyAsync(d_word, word_ids, n * 4, cudaMemcpyHostToDevice, st), "partition");
    }
    DevChunk c;
    cudaError_t e = partition_device(sc, st, d_doc, d_word, n, lo, hi, V, K, zkey, c, errs);
    if (e != cudaSuccess) return shard_cuda_fail(e, "partition");
    unsigned long long he[2];
    GF_TRY_RC(cudaMemcpyAsync(he, errs, 16, cudaMemcpyDeviceToHost, st), "partition");
    if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return shard_cuda_fail(e, "partition");
    if (he[0] != ~0ULL) return shard_fail(GF_ERR_VALUE, "word id outside [0, vocab_size)");
    if (he[1] != ~0ULL) return shard_fail(GF_ERR_VALUE, "doc id %d outside chunk range", doc_ids[he[1]]);
    int32_t* d32 = reinterpret_cast<int32_t*>(sc.u32(n));
    int64_t* d64 = static_cast<int64_t*>(sc.get((size_t)std::max<int64_t>(n, D + 1) * 8));
    if (sc.err != cudaSuccess) return shard_cuda_fail(sc.err, "partition");
    if (n > 0) {
        k_u32_to_i32<<<blocks_for(n), 256, 0, st>>>(n, c.doc, d32, lo);
        GF_TRY_RC(cudaMemcpyAsync(out_doc, d32, n * 4, cudaMemcpyDeviceToHost, st), "partition");
        GF_TRY_RC(cudaMemcpyAsync(out_word, c.word, n * 4, cudaMemcpyDeviceToHost, st), "partition");
        GF_TRY_RC(cudaMemcpyAsync(out_z, c.z, n * 2, cudaMemcpyDeviceToHost, st), "partition");
        k_u32_to_i64<<<blocks_for(n), 256, 0, st>>>(n, c.dw_tok, d64, 0);
        GF_TRY_RC(cudaMemcpyAsync(dw_tok, d64, n * 8, cudaMemcpyDeviceToHost, st), "partition");
    }
    if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return shard_cuda_fail(e, "partition");
    k_u32_to_i64<<<blocks_for(D + 1), 256, 0, st>>>(D + 1, c.dw_ptr, d64, 0);
    GF_TRY_RC(cudaMemcpyAsync(dw_ptr, d64, (D + 1) * 8, cudaMemcpyDeviceToHost, st), "partition");
    std::vector<uint32_t> go32((size_t)c.ng + 1);
    if (c.ng) cudaMemcpyAsync(gw, c.gw, c.ng * 4, cudaMemcpyDeviceToHost, st);
    GF_TRY_RC(cudaMemcpyAsync(go32.data(), c.go, (c.ng + 1) * 4, cudaMemcpyDeviceToHost, st), "partition");
    if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return shard_cuda_fail(e, "partition");
    for (int64_t g = 0; g < c.ng; ++g) {
        go[g] = go32[g];
        gs[g] = (int64_t)go32[g + 1] - go32[g];
    }
    *ng_out = c.ng;
    return GF_OK;
}

}  // namespace gf
