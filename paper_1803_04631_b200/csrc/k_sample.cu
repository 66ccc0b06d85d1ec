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
// Work: warps pull batches of 32 (doc, word) RUNS from a shared counter; in a
// batch lane j owns run j and draws the Philox4x32-10 uniforms of its first
// token (counter = global doc, word, occurrence, iteration).  Two sampler
// shapes:
//   thread mode (row nnz <= kSmall): the lane walks its own theta row
//     (16-byte loads, L1) for S, and searches it / the Q-tree itself -- 32
//     runs advance in lock-step with no cross-lane traffic;
//   warp mode (longer rows, one run at a time): 32 lanes scan the row with
//     __shfl prefix sums into a per-warp shared buffer, then each draw is a
//     two-level __ballot_sync search over that prefix (or the Q-tree).
// Exclusion (theta_dz-1, phi_vz-1, n_z-1) is applied by
// thinning: draw k from the exclusion-free S+Q mixture; if k == z keep it with
// probability p_ex(z) / p(z) = (theta_dz - 1 + a) p*_ex(z) / ((theta_dz + a) p*(z)),
// else redraw (fresh Philox block: occurrence | retry << 26).  The accepted k is
// distributed exactly as the exclusion-adjusted Eq. 1 -- the distribution
// sample_sparse defines -- without a per-token search for z in the row.
#include "gf_internal.cuh"
#include "gf_device.cuh"

namespace gf {

constexpr int kWarps = kSampleThreads / 32;
constexpr uint32_t kSmall = 64;       // thread mode up to this many row entries
constexpr uint32_t kCap = 1024;       // warp-mode shared prefix capacity (else stream)
constexpr int kMaxRetry = 63;

struct SampleArgs {
    int K, Kp;
    float alpha, beta, vbeta;
    uint2 key;
    uint32_t iteration;
    uint32_t doc_lo;
    int eval_only;                            // loglik of the current model only
    TreeGeom tree;
    const int4* slices;
    const uint32_t* run_doc;
    const uint32_t* run_start;
    uint16_t* z;
    const uint2* theta_meta;
    const uint32_t* theta_ent;
    const uint32_t* phi32;
    const uint16_t* phi16;
    const uint32_t* nk;
    const float* inv_den;
    double* ll_part;
    unsigned long long* errs;
    unsigned long long* bytes;
};

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

// ptree descent (ptree.py:203-225) over the shared-memory levels, one ballot
// per level (warp mode).
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

// the same search by one lane: binary search of level 0 (minimal k, P[k] > u)
__device__ __forceinline__ int search_q_lane(const float* lvl0, int K, float u) {
    int lo = 0, hi = K - 1;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (lvl0[mid] > u) hi = mid;
        else lo = mid + 1;
    }
    return lo;
}

// theta_dz of a sorted row by binary search (thinning of a Q-branch z draw)
__device__ __forceinline__ uint32_t row_count(const uint32_t* row, uint32_t nnz, uint32_t z) {
    uint32_t lo = 0, hi = nnz;
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        const uint32_t e = __ldg(row + mid);
        if ((e & 0xffffu) < z) lo = mid + 1;
        else hi = mid;
    }
    if (lo < nnz) {
        const uint32_t e = __ldg(row + lo);
        if ((e & 0xffffu) == z) return e >> 16;
    }
    return 0;
}

// keep a draw of the token's own topic with probability p_ex(z) / p(z)
__device__ __forceinline__ bool keep_own(float ut, uint32_t cnt, float alpha, float ps, float pex) {
    const float num = __fmul_rn(__fadd_rn((float)cnt - 1.f, alpha), pex);
    const float den = __fmul_rn(__fadd_rn((float)cnt, alpha), ps);
    return __fmul_rn(ut, den) < num;
}

template <int DUMMY>
__global__ void __launch_bounds__(kSampleThreads, 4) sample_kernel(SampleArgs a) {
    extern __shared__ float smem[];
    float* lvl = smem;                              // Q-tree levels (level 0 = prefix of a p*)
    float* pstar = smem + a.tree.total;             // p*(k)
    float* pex = pstar + a.K;                       // p*_ex(k)
    float* wbuf = smem + ((a.tree.total + 2 * a.K + 3) & ~3);   // kWarps x kCap row prefixes (16 B aligned)
    __shared__ double ll_w[kWarps];
    __shared__ unsigned long long by_w[kWarps];
    __shared__ int next_run;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int4 sl = a.slices[blockIdx.x];
    const uint32_t v = (uint32_t)sl.x;
    const int col = sl.w;
    const int K = a.K;

    // ---------------- prologue: p*, p*_ex and the Q prefix (block scan) ----------------
    {
        const int ipt = (K + kSampleThreads - 1) / kSampleThreads;
        const int k0 = tid * ipt;
        float acc = 0.f;
        for (int i = 0; i < ipt; ++i) {
            const int k = k0 + i;
            if (k < K) {
                const uint32_t ph = phi_at(a, col, k);
                const uint32_t nk = __ldg(a.nk + k);
                const float ps = __fmul_rn(__fadd_rn((float)ph, a.beta), __ldg(a.inv_den + k));
                pstar[k] = ps;
                pex[k] = (ph && nk) ? __fdiv_rn(__fadd_rn((float)(ph - 1u), a.beta),
                                                __fadd_rn((float)(nk - 1u), a.vbeta))
                                    : 0.f;
                acc = __fadd_rn(acc, __fmul_rn(a.alpha, ps));
                lvl[k] = acc;
            }
        }
        const float incl = warp_incl_scan(acc, lane);
        __shared__ float wtot[kWarps];
        if (lane == 31) wtot[warp] = incl;
        if (tid == 0) next_run = sl.y;
        __syncthreads();
        if (tid == 0) {
            float run = 0.f;
            for (int w = 0; w < kWarps; ++w) { const float t = wtot[w]; wtot[w] = run; run = __fadd_rn(run, t); }
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
            for (int i = tid; i < a.tree.len[l]; i += kSampleThreads)
                lvl[a.tree.off[l] + i] = lvl[a.tree.off[l - 1] + min(32 * i + 31, a.tree.len[l - 1] - 1)];
            __syncthreads();
        }
    }
    const float Q = lvl[K - 1];
    const float* lvl0 = lvl;
    float* buf = wbuf + warp * kCap;
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
        uint32_t d = 0, t0 = 0, t1 = 0, off = 0, nnz = 0;
        if (valid) {
            d = __ldg(a.run_doc + r);
            t0 = __ldg(a.run_start + r);
            t1 = __ldg(a.run_start + r + 1);
            const uint2 m = __ldg(a.theta_meta + d);
            off = m.x;
            nnz = m.y;
            nbytes += nnz;
        }
        const uint32_t gdoc = a.doc_lo + d;
        U3 u0{0.f, 0.f, 0.f};
        if (valid && !a.eval_only) u0 = draw_u(a, gdoc, v, 0u, 0u);
        float myS = 0.f;                             // S of this lane's run (either shape)

        // ================= thread mode: one lane, one run =================
        if (valid && nnz <= kSmall) {
            const uint32_t* row = a.theta_ent + off;
            float S = 0.f;
            for (uint32_t j = 0; j < nnz; j += 4) {             // zero pads add nothing
                const uint4 q = __ldg(reinterpret_cast<const uint4*>(row + j));
                S = __fadd_rn(S, __fmul_rn((float)(q.x >> 16), pstar[q.x & 0xffffu]));
                S = __fadd_rn(S, __fmul_rn((float)(q.y >> 16), pstar[q.y & 0xffffu]));
                S = __fadd_rn(S, __fmul_rn((float)(q.z >> 16), pstar[q.z & 0xffffu]));
                S = __fadd_rn(S, __fmul_rn((float)(q.w >> 16), pstar[q.w & 0xffffu]));
            }
            myS = S;
            if (!a.eval_only) {
                for (uint32_t t = t0; t < t1; ++t) {
                    const uint32_t zt = a.z[t];
                    const uint32_t occ = t - t0;
                    U3 u = occ ? draw_u(a, gdoc, v, occ, 0u) : u0;
                    uint32_t k = zt;
                    for (int retry = 0; retry <= kMaxRetry; ++retry) {
                        if (retry) u = draw_u(a, gdoc, v, occ, (uint32_t)retry);
                        uint32_t cnt = 0;
                        if (__fmul_rn(u.b, __fadd_rn(S, Q)) < S) {
                            const float target = __fmul_rn(u.s, S);
                            float acc = 0.f;
                            uint32_t pick = 0xffffffffu, last = 0;
                            for (uint32_t j = 0; j < nnz && pick == 0xffffffffu; j += 4) {
                                const uint4 q = __ldg(reinterpret_cast<const uint4*>(row + j));
                                const uint32_t e4[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
                                for (int i = 0; i < 4; ++i)
                                    if (pick == 0xffffffffu) {
                                        acc = __fadd_rn(acc, __fmul_rn((float)(e4[i] >> 16), pstar[e4[i] & 0xffffu]));
                                        if (e4[i] >> 16) last = e4[i];       // pads (count 0) never picked
                                        if (acc > target) pick = e4[i];
                                    }
                            }
                            if (pick == 0xffffffffu) pick = last;   // rounding guard: last entry
                            k = pick & 0xffffu;
                            cnt = pick >> 16;
                        } else {
                            k = (uint32_t)search_q_lane(lvl0, K, __fmul_rn(u.s, Q));
                            if (k == zt) cnt = row_count(row, nnz, zt);
                        }
                        if (k != zt) break;
                        if (zt >= (uint32_t)K || cnt == 0u || pex[zt] == 0.f) {   // inconsistent state
                            atomicMin(a.errs, (unsigned long long)t);
                            break;
                        }
                        if (keep_own(u.t, cnt, a.alpha, pstar[zt], pex[zt])) break;
                        k = zt;                                                   // rejected: redraw
                    }
                    a.z[t] = (uint16_t)k;
                }
            }
        }

        // ================= warp mode: 32 lanes, one run at a time =================
        unsigned big = __ballot_sync(kFull, valid && nnz > kSmall);
        // software pipeline: the first 128-entry chunk of the next big row is in
        // flight while the current run is sampled
        uint4 qnext = make_uint4(0, 0, 0, 0);
        if (big) {
            const int s0 = __ffs(big) - 1;
            const uint32_t o0 = __shfl_sync(kFull, off, s0), n0 = __shfl_sync(kFull, nnz, s0);
            if (4u * lane < n0) qnext = __ldg(reinterpret_cast<const uint4*>(a.theta_ent + o0 + 4u * lane));
        }
        while (big) {
            const int src = __ffs(big) - 1;
            big &= big - 1;
            const uint32_t wd = __shfl_sync(kFull, gdoc, src);
            const uint32_t w0 = __shfl_sync(kFull, t0, src), w1 = __shfl_sync(kFull, t1, src);
            const uint32_t woff = __shfl_sync(kFull, off, src), wn = __shfl_sync(kFull, nnz, src);
            const U3 wu0{__shfl_sync(kFull, u0.b, src), __shfl_sync(kFull, u0.s, src), __shfl_sync(kFull, u0.t, src)};
            const uint32_t* row = a.theta_ent + woff;
            const uint4 qcur = qnext;
            if (big) {
                const int s1 = __ffs(big) - 1;
                const uint32_t o1 = __shfl_sync(kFull, off, s1), n1 = __shfl_sync(kFull, nnz, s1);
                qnext = make_uint4(0, 0, 0, 0);
                if (4u * lane < n1) qnext = __ldg(reinterpret_cast<const uint4*>(a.theta_ent + o1 + 4u * lane));
            }
            const uint32_t nch = (wn + 127u) >> 7;
            const bool staged = wn <= kCap;
            // pass over the row: prefix sums (staged into buf when they fit)
            float carry = 0.f;
            for (uint32_t c = 0; c < nch; ++c) {
                const uint32_t j0 = c * 128u + 4u * lane;
                // rows are zero-padded to 4 entries (K3), so a (count 0) pad adds nothing
                uint4 q = make_uint4(0, 0, 0, 0);
                if (c == 0) q = qcur;
                else if (j0 < wn) q = __ldg(reinterpret_cast<const uint4*>(row + j0));
                float p[4];
                p[0] = __fmul_rn((float)(q.x >> 16), pstar[q.x & 0xffffu]);
                p[1] = __fadd_rn(p[0], __fmul_rn((float)(q.y >> 16), pstar[q.y & 0xffffu]));
                p[2] = __fadd_rn(p[1], __fmul_rn((float)(q.z >> 16), pstar[q.z & 0xffffu]));
                p[3] = __fadd_rn(p[2], __fmul_rn((float)(q.w >> 16), pstar[q.w & 0xffffu]));
                const float incl = warp_incl_scan(p[3], lane);
                float excl = __shfl_up_sync(kFull, incl, 1);
                if (lane == 0) excl = 0.f;
                const float base = __fadd_rn(carry, excl);
#pragma unroll
                for (int i = 0; i < 4; ++i) p[i] = __fadd_rn(base, p[i]);
                if (staged && j0 < kCap) *reinterpret_cast<float4*>(buf + j0) = make_float4(p[0], p[1], p[2], p[3]);
                carry = __shfl_sync(kFull, p[3], 31);
            }
            __syncwarp();
            const float S = carry;
            if (lane == src) myS = S;                   // its log joins the batch's SIMT logf
            if (a.eval_only) continue;
            // uniforms of occurrences 1..31 of this run, one per lane
            const uint32_t n = w1 - w0;
            U3 ul{0.f, 0.f, 0.f};
            if (n > 1 && lane > 0 && (uint32_t)lane < n) ul = draw_u(a, wd, v, (uint32_t)lane, 0u);
            const uint32_t ngrp = (min(wn, kCap) + 31u) >> 5;
            for (uint32_t t = w0; t < w1; ++t) {
                const uint32_t zt = a.z[t];
                const uint32_t occ = t - w0;
                U3 u = wu0;
                if (occ) {
                    if (occ < 32) u = U3{__shfl_sync(kFull, ul.b, occ), __shfl_sync(kFull, ul.s, occ),
                                          __shfl_sync(kFull, ul.t, occ)};
                    else u = draw_u(a, wd, v, occ, 0u);
                }
                uint32_t k = zt;
                for (int retry = 0; retry <= kMaxRetry; ++retry) {
                    if (retry) u = draw_u(a, wd, v, occ, (uint32_t)retry);
                    uint32_t cnt = 0;
                    if (__fmul_rn(u.b, __fadd_rn(S, Q)) < S) {
                        const float target = __fmul_rn(u.s, S);
                        uint32_t j;
                        if (staged) {
                            // two-level 32-ary ballot search of the staged prefix
                            const bool gok = (uint32_t)lane < ngrp && buf[min(32u * lane + 31u, wn - 1u)] > target;
                            const unsigned gm = __ballot_sync(kFull, gok);
                            const uint32_t g = gm ? (uint32_t)(__ffs(gm) - 1) : ngrp - 1u;
                            const uint32_t idx = 32u * g + lane;
                            const bool eok = idx < wn && buf[idx] > target;
                            const unsigned em = __ballot_sync(kFull, eok);
                            j = em ? 32u * g + (uint32_t)(__ffs(em) - 1) : wn - 1u;
                        } else {
                            // long row: rescan chunk by chunk (same arithmetic as the pass)
                            float cy = 0.f;
                            j = wn - 1u;
                            for (uint32_t c = 0; c < nch; ++c) {
                                const uint32_t j0 = c * 128u + 4u * lane;
                                uint4 q = make_uint4(0, 0, 0, 0);
                                if (j0 < wn) q = __ldg(reinterpret_cast<const uint4*>(row + j0));
                                const uint32_t e4[4] = {q.x, q.y, q.z, q.w};
                                float p[4];
                                float acc = 0.f;
#pragma unroll
                                for (int i = 0; i < 4; ++i) {
                                    if (j0 + i < wn)
                                        acc = __fadd_rn(acc, __fmul_rn((float)(e4[i] >> 16), pstar[e4[i] & 0xffffu]));
                                    p[i] = acc;
                                }
                                const float incl = warp_incl_scan(acc, lane);
                                float excl = __shfl_up_sync(kFull, incl, 1);
                                if (lane == 0) excl = 0.f;
                                int fi = -1;
#pragma unroll
                                for (int i = 3; i >= 0; --i)
                                    if (j0 + i < wn && __fadd_rn(cy, __fadd_rn(excl, p[i])) > target) fi = i;
                                const unsigned m = __ballot_sync(kFull, fi >= 0);
                                if (m) {
                                    const int L = __ffs(m) - 1;
                                    j = c * 128u + 4u * (uint32_t)L + (uint32_t)__shfl_sync(kFull, fi, L);
                                    break;
                                }
                                cy = __fadd_rn(cy, __shfl_sync(kFull, __fadd_rn(excl, p[3]), 31));
                            }
                        }
                        const uint32_t e = __ldg(row + j);
                        k = e & 0xffffu;
                        cnt = e >> 16;
                    } else {
                        k = (uint32_t)search_q_warp(lvl, a.tree, __fmul_rn(u.s, Q), lane);
                        if (k == zt) cnt = row_count(row, wn, zt);
                    }
                    if (k != zt) break;
                    if (zt >= (uint32_t)K || cnt == 0u || pex[zt] == 0.f) {
                        if (lane == 0) atomicMin(a.errs, (unsigned long long)t);
                        break;
                    }
                    if (keep_own(u.t, cnt, a.alpha, pstar[zt], pex[zt])) break;
                    k = zt;
                }
                if (lane == 0) a.z[t] = (uint16_t)k;
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
            const bool bad = zt >= (uint32_t)a.K || row_count(a.theta_ent + m.x, m.y, zt) == 0u ||
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

size_t sample_smem_bytes(const gf_shard* s) {
    return (size_t)(((s->tree.total + 2 * s->K + 3) & ~3) + kWarps * kCap) * sizeof(float);
}

cudaError_t launch_sample(gf_shard* s, uint32_t iteration, int eval_only) {
    if (s->n_slices == 0) return cudaSuccess;
    SampleArgs a;
    a.K = s->K;
    a.Kp = s->Kp;
    a.alpha = (float)s->alpha;
    a.beta = (float)s->beta;
    a.vbeta = (float)((double)s->V * s->beta);
    a.key = make_uint2((uint32_t)s->seed, (uint32_t)(s->seed >> 32));
    a.iteration = iteration;
    a.doc_lo = (uint32_t)s->doc_lo;
    a.eval_only = eval_only;
    a.tree = s->tree;
    a.slices = s->d.slices;
    a.run_doc = s->d.run_doc;
    a.run_start = s->d.run_start;
    a.z = s->d.z;
    a.theta_meta = s->d.theta_meta;
    a.theta_ent = s->d.theta_ent;
    a.phi32 = s->d.sync;
    a.phi16 = reinterpret_cast<const uint16_t*>(s->d.sync + s->off_phi16_u32);
    a.nk = s->d.sync + s->off_nk_u32;
    a.inv_den = s->d.inv_den;
    a.ll_part = s->d.ll_part;
    a.errs = s->d.errs;
    a.bytes = s->d.bytes;
    const size_t smem = sample_smem_bytes(s);
    static bool attr_set = false;
    if (!attr_set) {
        cudaError_t e = cudaFuncSetAttribute(sample_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
        if (e != cudaSuccess) return e;
        e = cudaFuncSetAttribute(sample_kernel<0>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                 cudaSharedmemCarveoutMaxShared);
        if (e != cudaSuccess) return e;
        attr_set = true;
    }
    sample_kernel<0><<<(unsigned)s->n_slices, kSampleThreads, smem, s->stream>>>(a);
    return cudaGetLastError();
}

}  // namespace gf
