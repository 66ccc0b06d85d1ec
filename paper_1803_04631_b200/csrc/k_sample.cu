// k_sample.cu -- K1: the collapsed-Gibbs sampler (
// PAPER.md section 6.1, Algorithm 2) with the fused per-token log-likelihood
// (SPEC.md:402-410).
//
// Grid: one CTA per heavy-first word slice (section 6.1.2: the
// samplers of a thread block share one word, long words are split and
// scheduled first).  Prologue, once per slice, in shared memory:
//   p*(k)     = (phi_vk + b) / (n_k + V b)                 (PAPER Eq. 8)
//   p*_ex(k)  = (phi_vk - 1 + b) / (n_k - 1 + V b)         (exclusion view)
//   Q-tree    = 32-ary prefix tree over a p*(k)            (ptree.build levels)
// p* sits at shared offset 0 and theta entries carry the topic pre-scaled to a
// byte offset (count << 16 | topic << 2), so a p1 term is one LOP + LDS + FFMA.
//
// Work: each warp pulls batches of up to 32 (doc, word) RUNS (lane j owns run
// j: its doc, token range and theta row) and handles them as segmented
// sub-batches:
//   1. entry-parallel pass: the sub-batch's theta rows (16-byte vectors,
//      zero-padded to 4 entries) are streamed as one concatenated array, VEC
//      vectors per lane and 128*VEC entries per warp step; p1 = theta * p* is
//      prefix-summed by a segmented __shfl scan (segment heads from one
//      __reduce_or_sync) and the prefix at every vector end is staged in the
//      warp's shared buffer -- S of every run falls out as a segment total;
//   2. token-parallel draws: the sub-batch's tokens are one contiguous range;
//      lane l draws token base + l (its run found from a run-head bitmap),
//      branch u (S+Q) < S, then ONE branch-free binary search -- over the
//      run's staged vector ends (S part, followed by a 4-entry walk of the
//      chosen vector) or over the Q-tree level 0 (Q part).
// Rows longer than the staging buffer (K > 4096 only) take a warp-cooperative
// streaming path.  Exclusion (theta_dz-1, phi_vz-1, n_z-1)
// is applied by thinning: draw k from the exclusion-free S+Q mixture; if
// k == z keep it with probability
//   p_ex(z) / p(z) = (theta_dz - 1 + a) p*_ex(z) / ((theta_dz + a) p*(z)),
// else redraw (fresh Philox block: occurrence | retry << 26); the 64th
// rejection ends in one exact sequential draw (exact_excluded_draw).  Accepted
// draws follow exactly the exclusion-adjusted Eq. 1 that sample_sparse
// defines, without a per-token search for z in the row.
#include "gf_internal.cuh"
#include "gf_device.cuh"

#include <cstdlib>

namespace gf {

constexpr uint32_t kCapV = 1024;      // staged vector-end prefixes per warp (4096 entries)
constexpr int kMaxRetry = 63;


// 256-bit read-only global load (sm_100: LDG.E.ENL2.256); p must be 32-byte aligned
__device__ __forceinline__ void ldg256(const uint32_t* p, uint4& lo, uint4& hi) {
    asm volatile("ld.global.nc.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(lo.x), "=r"(lo.y), "=r"(lo.z), "=r"(lo.w), "=r"(hi.x), "=r"(hi.y), "=r"(hi.z), "=r"(hi.w)
                 : "l"(p));
}

struct SampleArgs {
    int K, Kp;
    float alpha, beta, vbeta;
    uint2 key;
    uint32_t iteration;
    uint32_t doc_lo;
    int eval_only;                            // loglik of the current model only
    int prefetch;                             // prefetch each batch's theta rows into L2 (1 lines, 2 bulk)
    int guide_min_tokens;                     // slices below this build no Q guide
    TreeGeom tree;
    const int4* slices;
    const uint32_t* run_doc;
    const uint32_t* run_start;
    const uint32_t* run_dwpos;                // zdoc position of each run's first token
    const uint4* run_rec;                     // {doc, first token, zdoc position, theta offset}
    uint16_t* z;
    uint16_t* zdoc;                           // doc-major copy of z (read by K3)
    const uint2* theta_meta;
    const uint32_t* theta_ent;
    const uint32_t* phi32;
    const uint16_t* phi16;
    const uint32_t* nk;
    const float* inv_den;                     // [K] 1/(n_k + V b), then [K] 1/(n_k - 1 + V b)
    const float* ctx_tab;                     // precomputed word contexts (multi-slice words)
    const int32_t* slice_ctx;                 // per slice: context index or -1
    int ctx_stride;                           // floats per context = lay_buf(K, tree.total)
    TPos tm;                                  // transposed p* layout (gf_device.cuh)
    double* ll_part;
    uint32_t zero_ent;                        // theta_ent index of a zero 32-byte granule (= capacity)
    unsigned long long* errs;
    unsigned long long* bytes;
};

// shared-memory layout (floats): p*[32m] at 0 in the transposed topic layout |
// p*_ex[K] (natural) | Q-tree levels (natural) | Q guide[kGuide + 1] (u32) |
// pad | warp buffers
constexpr int kGuide = 256;                   // Q-prefix guide buckets (power of two)
// p*_ex lives in shared memory for K <= 2048; above that it is evaluated on
// demand (only a thinning test needs it) so a third CTA fits on the SM
__host__ __device__ inline bool pex_in_smem(int K) { return K <= 2048; }
__host__ __device__ inline int lay_pex(int K) { return (int)tpos_slots(K); }
__host__ __device__ inline int lay_tree(int K) { return lay_pex(K) + (pex_in_smem(K) ? K : 0); }
__host__ __device__ inline int lay_guide(int K, int tree_total) { return lay_tree(K) + tree_total; }
__host__ __device__ inline int lay_buf(int K, int tree_total) { return (lay_guide(K, tree_total) + kGuide + 1 + 3) & ~3; }

__device__ __forceinline__ uint32_t phi_at(const SampleArgs& a, int col, int k) {
    return col >= 0 ? (uint32_t)a.phi16[(size_t)col * a.Kp + k] : a.phi32[(size_t)(~col) * a.K + k];
}

struct U3 {
    float b, s, t;                            // branch, search, thinning
};

__device__ __forceinline__ U3 draw_u(const SampleArgs& a, uint32_t gdoc, uint32_t v, uint32_t occ, uint32_t retry) {
    const uint4 r = philox4x32_10(make_uint4(gdoc, v, occ | (retry << 26), a.iteration), a.key);
    return U3{u24(r.x), u24(r.y), u24(r.z)};
}

// p1 term of one theta entry (count << 16 | topic << 2) against p* at shared offset 0
// The count converts without the quarter-rate I2F: one LEA.HI builds the float
// 2^23 + count (count in the low mantissa bits), one FADD removes 2^23 (exact).
__device__ __forceinline__ uint32_t shl_clamped(uint32_t x, uint32_t n) {
    uint32_t r;
    asm("shl.b32 %0, %1, %2;" : "=r"(r) : "r"(x), "r"(n));   // PTX: n >= 32 gives 0
    return r;
}
// %lanemask_le as one S2R instead of a mask kept live (or rebuilt) across the pass
__device__ __forceinline__ unsigned lanemask_le() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_le;" : "=r"(m));
    return m;
}
__device__ __forceinline__ float count_f(uint32_t e) {
    return __int_as_float(0x4B000000u + (e >> 16)) - 8388608.f;
}
__device__ __forceinline__ float w_of(uint32_t e, const float* smem) {
    return count_f(e) * smem[(e & 0xfffcu) >> 2];
}
__device__ __forceinline__ uint32_t topic_of(uint32_t e, TPos tm) { return tpos_inv((e & 0xffffu) >> 2, tm); }

// ptree descent (ptree.py:203-225) over the shared-memory levels, one ballot
// per level (warp-cooperative).
__device__ __forceinline__ int search_q_warp(const float* lvl, const TreeGeom& g, float u, int lane) {
    int idx = 0;
    for (int l = g.nlev - 1; l >= 0; --l) {
        const int lo = idx * 32;
        const int n = min(32, g.len[l] - lo);
        const bool ok = lane < n && lvl[g.off[l] + lo + lane] > u;
        const unsigned m = __ballot_sync(kFull, ok);
        idx = m ? lo + __ffs(m) - 1 : lo + n - 1;
    }
    return idx;
}

// minimal i in [0, n) with P[i] > u (n-1 if none), P non-decreasing: one lane,
// branch-free (a fixed ladder of power-of-two steps)
__device__ __forceinline__ uint32_t first_above(const float* P, uint32_t n, float u) {
    uint32_t i = 0;
    for (uint32_t step = 1u << (31 - __clz(n)); step; step >>= 1)
        if (i + step <= n && !(P[i + step - 1] > u)) i += step;
    return min(i, n - 1u);
}

// theta_dz of a sorted row by binary search (thinning of a Q-branch z draw)
__device__ __forceinline__ uint32_t row_count(const uint32_t* row, uint32_t nnz, uint32_t z, TPos tm) {
    uint32_t lo = 0, hi = nnz;
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        const uint32_t e = __ldg(row + mid);
        if (topic_of(e, tm) < z) lo = mid + 1;
        else hi = mid;
    }
    if (lo < nnz) {
        const uint32_t e = __ldg(row + lo);
        if (topic_of(e, tm) == z) return e >> 16;
    }
    return 0;
}

// p*_ex(z) = (phi_vz - 1 + b) / (n_z - 1 + V b): from the shared table, or for
// large K from the word's phi column and the prepared reciprocal
__device__ __forceinline__ float pex_of(const SampleArgs& a, const float* pex, int col, uint32_t z) {
    if (pex_in_smem(a.K)) return pex[z];
    const uint32_t ph = phi_at(a, col, (int)z);
    return ph ? __fmul_rn(__fadd_rn((float)(ph - 1u), a.beta), __ldg(a.inv_den + a.K + z)) : 0.f;
}

// keep a draw of the token's own topic with probability p_ex(z) / p(z)
__device__ __forceinline__ bool keep_own(float ut, uint32_t cnt, float alpha, float ps, float pex) {
    const float num = __fmul_rn(__fadd_rn((float)cnt - 1.f, alpha), pex);
    const float den = __fmul_rn(__fadd_rn((float)cnt, alpha), ps);
    return __fmul_rn(ut, den) < num;
}

// Exact draw from the exclusion-adjusted conditional: two sequential passes over
// k = 0..K-1 with the sorted theta row merged in (one lane).  The thinning
// loop's fallback after its 64th rejected proposal, so the kept topic follows
// the exclusion-adjusted Eq. 1 at any acceptance rate (keeping z after a cap
// would over-weight it by the chance of 64 rejections).  Weights
// (theta_dk + a) p*(k) for k != z and (theta_dz - 1 + a) p*_ex(z); the oracle's
// thin mode does the same in fp64 (oracle/gf_oracle.c exact_excluded_draw).
// (scalar arguments: a reference to the kernel's parameter struct across a
// call would copy the struct to local memory in every thread)
// The uniform is word 3 of the last rejected proposal's Philox block, recomputed
// here so the draw loop keeps no extra register live.
__device__ __forceinline__ uint32_t exact_excluded_draw(int K, float alpha, TPos tm, const float* pstar,
                                                     const uint32_t* row, uint32_t nnz, uint32_t z, float pex_z,
                                                     uint4 ctr, uint2 key) {
    const float u = u24(philox4x32_10(ctr, key).w);
    float tot = 0.f;
    for (int pass = 0; pass < 2; ++pass) {
        const float target = __fmul_rn(u, tot);
        float acc = 0.f;
        uint32_t j = 0, last = 0, e = nnz ? __ldg(row) : 0u;
        for (uint32_t k = 0; k < (uint32_t)K; ++k) {
            float c = 0.f;
            if (j < nnz && topic_of(e, tm) == k) {
                c = (float)(e >> 16);
                ++j;
                e = j < nnz ? __ldg(row + j) : 0u;
            }
            const float w = k == z ? __fmul_rn(__fadd_rn(c - 1.f, alpha), pex_z)
                                   : __fmul_rn(__fadd_rn(c, alpha), pstar[tpos(k, tm)]);
            acc = __fadd_rn(acc, w);
            if (pass == 1) {
                if (w > 0.f) last = k;
                if (acc > target) return k;
            }
        }
        if (pass == 1) return last;
        tot = acc;
    }
    return z;
}

// Rows longer than the staging buffer: warp-cooperative, one run, the S part
// re-streamed per S-branch draw.  Returns S (all lanes).
__device__ __noinline__ float huge_run(const SampleArgs& a, const float* smem, float Q, uint32_t v, uint32_t gdoc,
                                       uint32_t t0, uint32_t t1, uint32_t off, uint32_t nnz, uint32_t dwp,
                                       int col, int lane) {
    const float* pstar = smem;
    const float* pex = smem + lay_pex(a.K);
    const float* lvl = smem + lay_tree(a.K);
    const uint32_t* row = a.theta_ent + off;
    const uint32_t nch = (nnz + 127u) >> 7;
    float S = 0.f;
    for (uint32_t c = 0; c < nch; ++c) {
        const uint32_t j0 = c * 128u + 4u * lane;
        uint4 q = make_uint4(0, 0, 0, 0);
        if (j0 < nnz) q = __ldg(reinterpret_cast<const uint4*>(row + j0));
        const float s4 = (w_of(q.x, smem) + w_of(q.y, smem)) + (w_of(q.z, smem) + w_of(q.w, smem));
        const float incl = warp_incl_scan(s4, lane);
        S += __shfl_sync(kFull, incl, 31);
    }
    if (a.eval_only) return S;
    for (uint32_t t = t0; t < t1; ++t) {
        const uint32_t zt = a.z[t];
        const uint32_t occ = t - t0;
        uint32_t k = zt;
        for (int retry = 0; retry <= kMaxRetry; ++retry) {
            const U3 u = draw_u(a, gdoc, v, occ, (uint32_t)retry);
            uint32_t cnt = 0;
            if (__fmul_rn(u.b, __fadd_rn(S, Q)) < S) {
                const float target = __fmul_rn(u.s, S);
                float cy = 0.f;
                uint32_t j = nnz - 1u;
                for (uint32_t c = 0; c < nch; ++c) {
                    const uint32_t j0 = c * 128u + 4u * lane;
                    uint4 q = make_uint4(0, 0, 0, 0);
                    if (j0 < nnz) q = __ldg(reinterpret_cast<const uint4*>(row + j0));
                    float p[4];
                    p[0] = w_of(q.x, smem);
                    p[1] = p[0] + w_of(q.y, smem);
                    p[2] = p[1] + w_of(q.z, smem);
                    p[3] = p[2] + w_of(q.w, smem);
                    const float incl = warp_incl_scan(p[3], lane);
                    float excl = __shfl_up_sync(kFull, incl, 1);
                    if (lane == 0) excl = 0.f;
                    const float base = cy + excl;
                    int fi = -1;
#pragma unroll
                    for (int i = 3; i >= 0; --i)
                        if (j0 + i < nnz && base + p[i] > target) fi = i;
                    const unsigned m = __ballot_sync(kFull, fi >= 0);
                    if (m) {
                        const int L = __ffs(m) - 1;
                        j = c * 128u + 4u * (uint32_t)L + (uint32_t)__shfl_sync(kFull, fi, L);
                        break;
                    }
                    cy = __shfl_sync(kFull, base + p[3], 31);
                }
                const uint32_t e = __ldg(row + j);
                k = topic_of(e, a.tm);
                cnt = e >> 16;
            } else {
                k = (uint32_t)search_q_warp(lvl, a.tree, __fmul_rn(u.s, Q), lane);
                if (k == zt) cnt = row_count(row, nnz, zt, a.tm);
            }
            if (k != zt) break;
            const float pz = zt < (uint32_t)a.K ? pex_of(a, pex, col, zt) : 0.f;
            if (zt >= (uint32_t)a.K || cnt == 0u || pz == 0.f) {
                if (lane == 0) atomicMin(a.errs, (unsigned long long)t);
                break;
            }
            if (keep_own(u.t, cnt, a.alpha, pstar[tpos(zt, a.tm)], pz)) break;
            if (retry == kMaxRetry) {                       // 64 rejections: one exact draw
                k = exact_excluded_draw(a.K, a.alpha, a.tm, pstar, row, nnz, zt, pz,
                                        make_uint4(gdoc, v, occ | ((uint32_t)kMaxRetry << 26), a.iteration), a.key);
                break;
            }
            k = zt;
        }
        if (lane == 0) { a.z[t] = (uint16_t)k; a.zdoc[dwp + occ] = (uint16_t)k; }
    }
    return S;
}

// The word context of SPEC.md build_word_context in shared
// memory: p*(k), p*_ex(k) and the 32-ary Q prefix tree over a p*(k) (block
// scan; ptree.build levels).  Ends with a __syncthreads.
template <int NT>
__device__ __forceinline__ void build_context(const SampleArgs& a, int col, float* smem, int tid,
                                              bool with_guide = true) {
    constexpr int NW = NT / 32;
    const int K = a.K, lane = tid & 31, warp = tid >> 5;
    float* pstar = smem;                             // transposed layout (tpos)
    float* pex = smem + lay_pex(K);
    float* lvl = smem + lay_tree(K);
    __shared__ float wtot[NW];
    // ipt consecutive topics per thread, ipt odd: the 32 lanes of a warp then
    // touch 32 distinct banks at every step i (an even ipt = 8 was an 8-way
    // conflict on lvl / pex); the last threads may have fewer topics
    const int ipt = ((K + NT - 1) / NT) | 1;
    const int k0 = tid * ipt;
    float acc = 0.f;
    for (int i = 0; i < ipt; ++i) {
        const int k = k0 + i;
        if (k < K) {
            const uint32_t ph = phi_at(a, col, k);
            const float ps = __fmul_rn(__fadd_rn((float)ph, a.beta), __ldg(a.inv_den + k));
            pstar[tpos((uint32_t)k, a.tm)] = ps;
            // (phi - 1 + b) / (n_k - 1 + V b), the reciprocal precomputed by prepare
            if (pex_in_smem(K)) pex[k] = ph ? __fmul_rn(__fadd_rn((float)(ph - 1u), a.beta), __ldg(a.inv_den + K + k)) : 0.f;
            acc = __fadd_rn(acc, __fmul_rn(a.alpha, ps));
            lvl[k] = acc;
        }
    }
    const float incl = warp_incl_scan(acc, lane);
    if (lane == 31) wtot[warp] = incl;
    __syncthreads();
    if (tid == 0) {
        float run = 0.f;
        for (int w = 0; w < NW; ++w) { const float t = wtot[w]; wtot[w] = run; run = __fadd_rn(run, t); }
    }
    __syncthreads();
    float excl = __shfl_up_sync(kFull, incl, 1);
    if (lane == 0) excl = 0.f;
    const float off = __fadd_rn(wtot[warp], excl);
    for (int i = 0; i < ipt; ++i) {
        const int k = k0 + i;
        if (k < K) lvl[k] = __fadd_rn(off, lvl[k]);
    }
    __syncthreads();
    for (int l = 1; l < a.tree.nlev; ++l) {
        for (int i = tid; i < a.tree.len[l]; i += NT)
            lvl[a.tree.off[l] + i] = lvl[a.tree.off[l - 1] + min(32 * i + 31, a.tree.len[l - 1] - 1)];
        __syncthreads();
    }
    // Q guide: guide[j] = first_above(level 0, thr_j), thr_j = fl((j / G) Q).  A
    // Q draw with target t = fl(u Q), j = floor(u G), has thr_j <= t <= thr_j+1
    // (rounding is monotone), so its answer lies in [guide[j], guide[j+1]] and a
    // search of that range returns exactly the full-range result.
    // (skipped for small slices: too few Q draws to repay 257 searches)
    if (!with_guide) return;
    uint32_t* guide = reinterpret_cast<uint32_t*>(smem + lay_guide(K, a.tree.total));
    const float Q = lvl[K - 1];
    for (int j = tid; j <= kGuide; j += NT)
        guide[j] = first_above(lvl, (uint32_t)K, __fmul_rn((float)j * (1.f / kGuide), Q));
    __syncthreads();
}

// One CTA per word that the schedule splits into several slices: its context
// is built once per iteration (same code, so bit-identical) and the slices
// copy it instead of rebuilding it.
template <int NT>
__global__ void __launch_bounds__(NT) context_kernel(SampleArgs a, const int32_t* __restrict__ cols,
                                                                  float* out) {
    extern __shared__ __align__(128) float smem[];
    build_context<NT>(a, cols[blockIdx.x], smem, threadIdx.x);
    float4* dst = reinterpret_cast<float4*>(out + (size_t)blockIdx.x * a.ctx_stride);
    for (int i = threadIdx.x; i < a.ctx_stride / 4; i += NT) dst[i] = reinterpret_cast<const float4*>(smem)[i];
}

constexpr uint32_t VEC = 2;                  // 16-byte vectors per lane per pass step (32 B)

// One token's draw (exclusion by thinning, the exact fallback after the 64th
// rejection); writes z[t] and its doc-major copy.  seg: the owner run's staged
// vector-end prefixes; occ: the token's occurrence in its (doc, word) run.
__device__ __forceinline__ void draw_token(const SampleArgs& a, const float* smem, const float* lvl0,
                                           const uint32_t* guide, bool guided, float Q, uint32_t v, int col,
                                           const float* seg, uint32_t t, uint32_t occ, uint32_t odoc, uint32_t ooff,
                                           uint32_t onnz, uint32_t odwp) {
    const int K = a.K;
    const float* pstar = smem;
    const float* pex = smem + lay_pex(K);
    const uint32_t oU = max(1u, (onnz + 3u) >> 2);
    const uint32_t oUp = (oU + VEC - 1u) / VEC * VEC;
    const float S = seg[oUp - 1u];
    const uint32_t* row = a.theta_ent + ooff;
    const uint32_t zt = a.z[t];
    uint32_t k = zt;
    for (int retry = 0; retry <= kMaxRetry; ++retry) {
        const U3 u = draw_u(a, odoc, v, occ, (uint32_t)retry);
        const bool isS = __fmul_rn(u.b, __fadd_rn(S, Q)) < S;
        const float target = __fmul_rn(u.s, isS ? S : Q);
        // Q: only the guide bucket [guide[j], guide[j+1]] (exact, see build_context)
        const uint32_t gj = (uint32_t)(u.s * (float)kGuide);
        const uint32_t qlo = (isS || !guided) ? 0u : guide[gj];
        const uint32_t qn = isS ? oUp : (guided ? guide[gj + 1] - qlo + 1u : (uint32_t)K);
        uint32_t g = first_above((isS ? seg : lvl0) + qlo, qn, target) + qlo;
        uint32_t cnt = 0;
        if (isS) {
            g = min(g, oU - 1u);
            float cum = g ? seg[g - 1u] : 0.f;
            const uint4 q = __ldg(reinterpret_cast<const uint4*>(row + 4u * g));
            const uint32_t e4[4] = {q.x, q.y, q.z, q.w};
            uint32_t pick = 0u, last = 0u;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                cum += w_of(e4[i], smem);
                if (e4[i] >> 16) last = e4[i];                  // pads (count 0) never picked
                if (!pick && (e4[i] >> 16) && cum > target) pick = e4[i];
            }
            if (!pick) pick = last;                             // rounding guard
            k = topic_of(pick, a.tm);
            cnt = pick >> 16;
        } else {
            k = g;
            if (k == zt) cnt = row_count(row, onnz, zt, a.tm);
        }
        if (k != zt) break;
        const float pz = zt < (uint32_t)K ? pex_of(a, pex, col, zt) : 0.f;
        if (zt >= (uint32_t)K || cnt == 0u || pz == 0.f) {   // inconsistent state
            atomicMin(a.errs, (unsigned long long)t);
            break;
        }
        if (keep_own(u.t, cnt, a.alpha, pstar[tpos(zt, a.tm)], pz)) break;
        if (retry == kMaxRetry) {                 // 64 rejections: one exact draw
            k = exact_excluded_draw(a.K, a.alpha, a.tm, pstar, row, onnz, zt, pz,
                                    make_uint4(odoc, v, occ | ((uint32_t)kMaxRetry << 26), a.iteration), a.key);
            break;
        }
        k = zt;                                                   // rejected: redraw
    }
    a.z[t] = (uint16_t)k;
    a.zdoc[odwp + occ] = (uint16_t)k;
}

// NT: threads per CTA; CAPV: staged vector ends per warp; MINB: CTAs per SM;
// PF: keep the pass's next 1 KB step in flight; HUGE: compile the streaming
// path (needed only when K > 4*CAPV)
template <int NT, uint32_t CAPV, int MINB, bool PF, bool HUGE>
__global__ void __launch_bounds__(NT, MINB) sample_kernel(SampleArgs a) {
    constexpr int kWarps = NT / 32;
    extern __shared__ __align__(128) float smem[];   // TMA bulk-copy destination: 16-byte aligned
    const int K = a.K;
    // p*(tpos(k)) at smem[0] (byte offset = theta topic field), p*_ex(k) at
    // lay_pex(K) (read by draw_token), the Q-tree levels at lay_tree(K)
    float* lvl = smem + lay_tree(K);                // Q-tree levels (level 0 = prefix of a p*)
    float* wbuf = smem + lay_buf(K, a.tree.total);  // kWarps x CAPV staged vector-end prefixes
    __shared__ double ll_w[kWarps];
    __shared__ unsigned long long by_w[kWarps];
    __shared__ int next_run;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int4 sl = a.slices[blockIdx.x];
    const uint32_t v = (uint32_t)sl.x;
    const int col = sl.w;

    // ---------------- prologue: the word context (p*, p*_ex, Q-tree) ----------------
    if (tid == 0) next_run = sl.y;
    const int ctx = a.slice_ctx[blockIdx.x];
    // the Q guide pays off only for slices with many tokens (contexts always have one)
    bool guided = __ldg(a.run_start + sl.z) - __ldg(a.run_start + sl.y) >= (uint32_t)a.guide_min_tokens;
    if (ctx >= 0) {
        // word split into several slices: its context (built once per
        // iteration by context_kernel) arrives by one TMA bulk copy from L2
        // instead of ~7 dependent 2 KB load/store rounds of the whole CTA
        __shared__ __align__(8) unsigned long long ctx_bar;
        const uint32_t bar = smem_addr(&ctx_bar);
        if (tid == 0)
            bulk_copy_issue(bar, smem_addr(smem), a.ctx_tab + (size_t)ctx * a.ctx_stride, (uint32_t)a.ctx_stride * 4u);
        __syncthreads();
        bulk_copy_wait(bar);
        guided = true;
    } else {
        build_context<NT>(a, col, smem, tid, guided);
    }
    const float Q = lvl[K - 1];
    const float* lvl0 = lvl;
    const uint32_t* guide = reinterpret_cast<const uint32_t*>(smem + lay_guide(K, a.tree.total));
    float* buf = wbuf + warp * CAPV;
    // runs per grab: 32 (one per lane) unless the slice is too small to give
    // every warp at least two grabs -- then smaller grabs keep all 8 warps busy
    const int batch = min(32, max(1, (sl.z - sl.y + 2 * kWarps - 1) / (2 * kWarps)));
    double ll = 0.0;
    unsigned long long nbytes = 0;
    while (true) {
        int rb = 0;
        if (lane == 0) rb = atomicAdd(&next_run, batch);
        rb = __shfl_sync(kFull, rb, 0);
        if (rb >= sl.z) break;
        // ---- batch: lane j owns run rb + j ----
        const int r = rb + lane;
        const bool valid = lane < batch && r < sl.z;
        uint32_t d = 0, t0 = 0, t1 = 0, off = 0, nnz = 0, dwp = 0;
        const int nval = min(batch, sl.z - rb);                   // valid lanes [0, nval)
        if (valid) {
            const uint4 rec = __ldg(a.run_rec + r);                 // one 16-byte load per run
            d = rec.x;
            t0 = rec.y;
            dwp = rec.z;
            off = rec.w;
            nnz = __ldg(&a.theta_meta[d].y);                        // this iteration's row length
            nbytes += nnz;
            // the whole row (32-byte granules) into L2 now: the pass then streams
            // the batch's rows with every line already requested, instead of one
            // 1 KB warp step in flight at a time.  One per-thread line prefetch
            // per 128 B of the row, at most 8 (a fixed, predicated sequence: a
            // variable-trip loop here made the compiler rematerialise the shared
            // base and lane id inside the pass loop, 103 -> 127 instructions per
            // step).  GF_PREFETCH=2: cp.async.bulk.prefetch, whose uniform
            // operands the compiler serialises over the 32 lanes (13% of K1's
            // instructions, measured).
            if (a.prefetch == 1 && nnz) {
                const uint32_t* line = a.theta_ent + (off & ~31u);
                const uint32_t lines = (((off & 31u) + ((nnz + 7u) & ~7u)) + 31u) >> 5;   // 32 entries per line
                prefetch_l2_line(line);
#pragma unroll
                for (uint32_t l = 1; l < 8; ++l)
                    if (l < lines) prefetch_l2_line(line + 32u * l);
            } else if (a.prefetch == 2 && nnz) {
                prefetch_l2_bulk(a.theta_ent + off, ((nnz + 7u) & ~7u) * 4u);
            }
        }
        t1 = __shfl_down_sync(kFull, t0, 1);                        // the next run's first token
        if (lane == nval - 1) t1 = __ldg(a.run_start + r + 1);
        const uint32_t gdoc = a.doc_lo + d;
        const uint32_t U = max(1u, (nnz + 3u) >> 2);          // row length in 16-byte vectors
        const uint32_t Up = (U + VEC - 1u) / VEC * VEC;       // ... padded to whole lanes
        const bool huge = HUGE && valid && Up > CAPV;         // only possible when K > 4*CAPV
        float myS = 0.f;                                       // S of this lane's run
        unsigned rem = __ballot_sync(kFull, valid);
        const unsigned hmask = __ballot_sync(kFull, huge);
        while (rem) {
            const int first = __ffs(rem) - 1;
            if (HUGE && ((hmask >> first) & 1u)) {             // rare: row beyond the buffer
                const float S = huge_run(a, smem, Q, v, __shfl_sync(kFull, gdoc, first),
                                         __shfl_sync(kFull, t0, first), __shfl_sync(kFull, t1, first),
                                         __shfl_sync(kFull, off, first), __shfl_sync(kFull, nnz, first),
                                         __shfl_sync(kFull, dwp, first), col, lane);
                if (lane == first) myS = S;
                rem &= rem - 1u;
                continue;
            }
            // ---- sub-batch: contiguous non-huge lanes [first, ...) whose rows fit CAPV ----
            const unsigned after = hmask & ~((2u << first) - 1u);
            const int end = after ? __ffs(after) - 1 : 32;
            const bool cand = lane >= first && lane < end && ((rem >> lane) & 1u);
            uint32_t cu = cand ? Up : 0u;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(kFull, cu, o);
                if (lane >= o) cu += y;
            }
            const unsigned selm = __ballot_sync(kFull, cand && cu <= CAPV);   // lane `first` always
            const bool sel = (selm >> lane) & 1u;
            const int lastl = 31 - __clz(selm);
            const uint32_t Utot = __shfl_sync(kFull, cu, lastl);
            const uint32_t vo = cu - (cand ? Up : 0u);                      // first vector of my row
            rem &= ~selm;

            // ---- 1. entry-parallel pass: segmented prefix of p1 over the concatenated rows ----
            // each lane owns VEC consecutive vectors (4*VEC entries) of ONE row per step
            // (rows are laid out VEC-aligned), so 128*VEC entries advance per warp step:
            // one 256-bit load per lane, the warp reads 1 KB contiguous per step (rows
            // are 32-byte aligned and zero-padded to 8 entries by K3).  With PF the
            // next step's load is issued before the current step is summed and
            // scanned (one step in flight ahead, in registers).
            int cprev = first - 1;                                          // run holding vector q-1
            const uint32_t hv = sel ? vo : 0xFFFFFFFFu;                     // my row's head vector
            auto issue = [&](uint32_t qs, unsigned& Ms, uint4& x0, uint4& x1) {
                // bit (vo - qs) / VEC when my row starts in step qs: a shift by >= 32
                // (row outside the step, or no row) yields 0 (shl clamps)
                const uint32_t hb = shl_clamped(1u, (hv - qs) / VEC);
                Ms = __reduce_or_sync(kFull, hb);                           // run heads in step qs
                const int ri = min(cprev + __popc(Ms & lanemask_le()), 31);
                const uint32_t rvo = __shfl_sync(kFull, vo, ri);
                const uint32_t roff = __shfl_sync(kFull, off, ri);
                const uint32_t qL = qs + VEC * (uint32_t)lane;
                const uint32_t idx = roff + 4u * (qL - rvo);                // entry index (< 2^32)
                // lanes past the sub-batch read the zero granule after the last row
                const uint32_t* src = a.theta_ent + (qL < Utot ? idx : a.zero_ent);
                ldg256(src, x0, x1);
                cprev = min(cprev + __popc(Ms), 31);                        // lane 31's row
            };
            unsigned Mn = 0u;
            uint4 n0 = make_uint4(0u, 0u, 0u, 0u), n1 = n0;
            if (PF) issue(0u, Mn, n0, n1);
            float carry = 0.f;
            for (uint32_t q0 = 0; q0 < Utot; q0 += 32u * VEC) {
                unsigned M;
                uint4 e[VEC];
                if (PF) {
                    M = Mn;
                    e[0] = n0;
                    e[1] = n1;
                    if (q0 + 32u * VEC < Utot) issue(q0 + 32u * VEC, Mn, n0, n1);
                } else {
                    issue(q0, M, e[0], e[1]);
                }
                const unsigned mle = M & lanemask_le();
                const uint32_t qL = q0 + VEC * (uint32_t)lane;
                const bool act = qL < Utot;
                float p[VEC];                                               // prefix at each vector end
#pragma unroll
                for (int i = 0; i < VEC; ++i)                               // FMUL + 3 FFMA per vector
                    p[i] = ((w_of(e[i].x, smem) + w_of(e[i].y, smem)) + w_of(e[i].z, smem)) + w_of(e[i].w, smem);
                p[1] += p[0];
                const int head = mle ? 31 - __clz(mle) : -1;                // my segment's first lane
                const int lim = max(head, 0);
                float x = p[1];
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const float y = __shfl_up_sync(kFull, x, o);
                    if (lane - o >= lim) x += y;
                }
                const float y1 = __shfl_up_sync(kFull, x, 1);
                float base = (lane - 1 >= lim) ? y1 : 0.f;
                if (head < 0) base += carry;                                // row continues from q0-1
                p[0] += base;
                p[1] += base;
                if (act) *reinterpret_cast<float2*>(buf + qL) = make_float2(p[0], p[1]);   // conflict-free
                carry = __shfl_sync(kFull, p[1], 31);
            }
            __syncwarp();
            if (sel) myS = buf[vo + Up - 1u];                              // segment total (pads add 0)
            // ---- 2. token-parallel draws over the sub-batch's tokens ----
            // The selected runs are consecutive runs of one word, so their tokens
            // are one contiguous range; lane l takes token base + l and finds its
            // run (owner lane) from a run-head bitmap, as the pass finds rows.
            // One search serves both branches (S: the owner's staged vector ends,
            // Q: the tree's level 0), so S and Q lanes do not diverge.
            if (!a.eval_only) {
                const uint32_t tend = __shfl_sync(kFull, t1, lastl);
                int cown = first - 1;                                       // run holding token base-1
                for (uint32_t base = __shfl_sync(kFull, t0, first); base < tend; base += 32u) {
                    const uint32_t th = (sel && t0 - base < 32u) ? (1u << (t0 - base)) : 0u;
                    const unsigned M = __reduce_or_sync(kFull, th);
                    const int own = min(cown + __popc(M & lanemask_le()), 31);
                    const uint32_t ot0 = __shfl_sync(kFull, t0, own);
                    const uint32_t odoc = __shfl_sync(kFull, gdoc, own);
                    const uint32_t ooff = __shfl_sync(kFull, off, own);
                    const uint32_t ovo = __shfl_sync(kFull, vo, own);
                    const uint32_t onnz = __shfl_sync(kFull, nnz, own);
                    const uint32_t odwp = __shfl_sync(kFull, dwp, own);
                    cown = __shfl_sync(kFull, own, 31);
                    const uint32_t t = base + (uint32_t)lane;
                    if (t < tend)
                        draw_token(a, smem, lvl0, guide, guided, Q, v, col, buf + ovo, t, t - ot0, odoc, ooff, onnz,
                                   odwp);
                }
            }
            __syncwarp();
        }
        // log p(w|d) (L_d + K a) of the iteration-start model, one SIMT logf per batch
        if (valid) ll += (double)(t1 - t0) * (double)logf(__fadd_rn(myS, Q));
    }
    // ---- deterministic reductions: lanes -> warp -> CTA ----
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        ll += __shfl_xor_sync(kFull, ll, o);
        nbytes += __shfl_xor_sync(kFull, nbytes, o);
    }
    if (lane == 0) { ll_w[warp] = ll; by_w[warp] = nbytes; }
    __syncthreads();
    if (tid == 0) {
        double s = 0.0;
        unsigned long long b = 0;
        for (int w = 0; w < kWarps; ++w) { s += ll_w[w]; b += by_w[w]; }
        a.ll_part[blockIdx.x] = s;
        atomicAdd(a.bytes, b);
    }
}

// Consistency of an IMPORTED state (set_theta / set_phi / set_assignments):
// every token's topic must be present in its theta row, its phi cell and n_k
// (exclusion_adjust pre-condition).  States the engine builds
// itself are consistent by construction, so this runs only after imports.
__global__ void __launch_bounds__(256) validate_kernel(SampleArgs a) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int4 sl = a.slices[blockIdx.x];
    for (int r = sl.y + warp * 32 + lane; r < sl.z; r += 256) {
        const uint32_t d = a.run_doc[r];
        const uint2 m = a.theta_meta[d];
        for (uint32_t t = a.run_start[r]; t < a.run_start[r + 1]; ++t) {
            const uint32_t zt = a.z[t];
            const bool bad = zt >= (uint32_t)a.K || row_count(a.theta_ent + m.x, m.y, zt, a.tm) == 0u ||
                             phi_at(a, sl.w, (int)zt) == 0u || a.nk[zt] == 0u;
            if (bad) atomicMin(a.errs, (unsigned long long)t);
        }
    }
}

cudaError_t launch_validate(gf_shard* s) {
    if (s->n_slices == 0) return cudaSuccess;
    SampleArgs a{};
    a.K = s->K;
    a.Kp = s->Kp;
    a.tm = tpos_geom(s->K);
    a.slices = s->d.slices;
    a.run_doc = s->d.run_doc;
    a.run_start = s->d.run_start;
    a.z = s->d.z;
    a.theta_meta = s->d.theta_meta;
    a.theta_ent = s->d.theta_ent;
    a.phi32 = s->d.sync;
    a.phi16 = reinterpret_cast<const uint16_t*>(s->d.sync + s->off_phi16_u32);
    a.nk = s->d.sync + s->off_nk_u32;
    a.errs = s->d.errs;
    validate_kernel<<<(unsigned)s->n_slices, 256, 0, s->stream>>>(a);
    return cudaGetLastError();
}

static size_t smem_for(const gf_shard* s, int nt, uint32_t capv) {
    return (size_t)(lay_buf(s->K, s->tree.total) + (nt / 32) * capv) * sizeof(float);
}

size_t sample_smem_bytes(const gf_shard* s) { return smem_for(s, kSampleThreads, kCapV); }
size_t context_floats(const gf_shard* s) { return (size_t)lay_buf(s->K, s->tree.total); }

template <int NT, uint32_t CAPV, int MINB, bool PF, bool HUGE>
static cudaError_t launch_variant(gf_shard* s, const SampleArgs& a, int64_t n) {
    static unsigned long long attr_set = 0;
    if (attr_once(attr_set, s->device)) {
        cudaError_t e = cudaFuncSetAttribute(sample_kernel<NT, CAPV, MINB, PF, HUGE>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
        if (e != cudaSuccess) return e;
        e = cudaFuncSetAttribute(sample_kernel<NT, CAPV, MINB, PF, HUGE>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                 cudaSharedmemCarveoutMaxShared);
        if (e != cudaSuccess) return e;
    }
    sample_kernel<NT, CAPV, MINB, PF, HUGE><<<(unsigned)n, NT, smem_for(s, NT, CAPV), s->stream>>>(a);
    return cudaGetLastError();
}

static int env_flag(const char* name, int dflt) {
    const char* e = getenv(name);
    return e && *e ? atoi(e) : dflt;
}

static SampleArgs make_args(gf_shard* s, uint32_t iteration, int eval_only) {
    SampleArgs a{};
    a.K = s->K;
    a.Kp = s->Kp;
    a.alpha = (float)s->alpha;
    a.beta = (float)s->beta;
    a.vbeta = (float)((double)s->V * s->beta);
    a.key = make_uint2((uint32_t)s->seed, (uint32_t)(s->seed >> 32));
    a.iteration = iteration;
    a.doc_lo = (uint32_t)s->doc_lo;
    a.eval_only = eval_only;
    a.prefetch = (int)env_flag("GF_PREFETCH", 1);          // 1 line prefetches, 2 TMA bulk, 0 none
    a.zero_ent = (uint32_t)s->theta_cap;
    a.guide_min_tokens = (int)env_flag("GF_GUIDE_MIN", 512);
    a.tree = s->tree;
    a.slices = s->d.slices;
    a.run_doc = s->d.run_doc;
    a.run_start = s->d.run_start;
    a.run_dwpos = s->d.run_dwpos;
    a.run_rec = s->d.run_rec;
    a.z = s->d.z;
    a.zdoc = s->d.zdoc;
    a.theta_meta = s->d.theta_meta;
    a.theta_ent = s->d.theta_ent;
    a.phi32 = s->d.sync;
    a.phi16 = reinterpret_cast<const uint16_t*>(s->d.sync + s->off_phi16_u32);
    a.nk = s->d.sync + s->off_nk_u32;
    a.inv_den = s->d.inv_den;
    a.ctx_tab = s->d.ctx_tab;
    a.slice_ctx = s->d.slice_ctx;
    a.ctx_stride = lay_buf(s->K, s->tree.total);
    a.tm = tpos_geom(s->K);
    a.ll_part = s->d.ll_part;
    a.errs = s->d.errs;
    a.bytes = s->d.bytes;
    return a;
}

// block size of the sampler (and context) kernels for this K
static int sample_block(int K) { return K > 2048 ? 256 : 128; }

cudaError_t launch_contexts(gf_shard* s) {
    s->ctx_dirty = false;
    if (s->n_ctx == 0) return cudaSuccess;
    const SampleArgs a = make_args(s, 0, 0);
    const size_t smem = (size_t)a.ctx_stride * sizeof(float);
    // the same block size as the sampler variant of this K (sample_block), so
    // copied contexts equal in-place builds bit for bit
    static unsigned long long attr_set = 0;
    if (attr_once(attr_set, s->device)) {
        cudaError_t e = cudaFuncSetAttribute(context_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(context_kernel<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
        if (e != cudaSuccess) return e;
    }
    if (sample_block(s->K) == 128)
        context_kernel<128><<<(unsigned)s->n_ctx, 128, smem, s->stream>>>(a, s->d.ctx_cols, s->d.ctx_tab);
    else
        context_kernel<256><<<(unsigned)s->n_ctx, 256, smem, s->stream>>>(a, s->d.ctx_cols, s->d.ctx_tab);
    return cudaGetLastError();
}

cudaError_t launch_sample(gf_shard* s, uint32_t iteration, int eval_only) {
    return launch_sample_range(s, iteration, eval_only, 0, s->n_slices);
}

// slices [slice0, slice0 + n) of the schedule (a phase, gf_shard_sample_phase):
// the kernel sees the range through offset slice / context / loglik pointers
cudaError_t launch_sample_range(gf_shard* s, uint32_t iteration, int eval_only, int64_t slice0, int64_t n) {
    if (n <= 0) return cudaSuccess;
    if (s->ctx_dirty) {                           // phi changed since the last prepare
        cudaError_t e = launch_prepare(s);
        if (e != cudaSuccess) return e;
    }
    SampleArgs a = make_args(s, iteration, eval_only);
    a.slices += slice0;
    a.slice_ctx += slice0;
    a.ll_part += slice0;
    // tuning knob GF_K1 (variant id, A/B runs); rows can only outgrow the
    // staging buffer when K > 4*CAPV -- otherwise the streaming path (a
    // register-hungry call) is compiled out
    static int var = -1;
    if (var < 0) {
        const char* env = getenv("GF_K1");
        var = env ? atoi(env) : 0;
    }
    if (s->K > (int)(4 * kCapV)) return launch_variant<256, kCapV, 3, true, true>(s, a, n);    // rows can outgrow staging
    if (s->K > 2048) return launch_variant<256, kCapV, 3, true, false>(s, a, n);    // p*_ex on demand: 3 x 8 warps/SM
    if (var == 2) return launch_variant<256, kCapV, 4, true, false>(s, a, n);        // 8-warp CTAs (A/B)
    if (var == 3) return launch_variant<128, 768, 8, false, false>(s, a, n);         // no pass prefetch (A/B)
    if (var == 1) return launch_variant<128, 768, 8, true, false>(s, a, n);          // 8 CTAs/SM (A/B)
    if (var == 4) return launch_variant<128, 640, 9, true, false>(s, a, n);          // 9 CTAs/SM (A/B)
    if (var == 5) return launch_variant<128, 512, 10, true, false>(s, a, n);         // 10 CTAs/SM (A/B)
    // 4-warp CTAs (a slice's tail -- warps idle at the final barrier while the
    // last batch finishes -- strands few warps; the pass keeps its next 1 KB
    // step in flight).  Slices averaging < 600 runs (e.g. one rank of an
    // 8-way PubMed-shape split: 359) have more prologue latency to hide: 9
    // CTAs/SM with 640-vector staging (52 registers; rows <= 2560 entries, any
    // K <= 2048), measured 1.5-2.3% faster there; full corpora (PubMed-shape
    // 908 runs per slice, NYTimes-shape) run 0.5-2% faster at 8 CTAs/SM with
    // 768-vector staging (60 registers).  10 CTAs/SM is slower everywhere.
    if (s->R < 600 * s->n_slices) return launch_variant<128, 640, 9, true, false>(s, a, n);
    return launch_variant<128, 768, 8, true, false>(s, a, n);
}

}  // namespace gf
