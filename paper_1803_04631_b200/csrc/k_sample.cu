// k_sample.cu -- K1: the collapsed-Gibbs sampler (
// PAPER.md section 6.1, Algorithm 2) with the fused per-token log-likelihood
// (SPEC.md:402-410).
//
// One CTA per heavy-first word slice (PAPER.md: "samplers in the same thread
// block sample the tokens from the same word", long words split and scheduled
// first).  Prologue: the word's p*(k) = (phi_vk + b)/(n_k + V b) and the dense
// Q-part prefix tree over a p*(k) are built once in shared memory (32-ary, the
// levels of ptree.build, ptree.py:116-136).  Then every warp is one sampler
// that takes a (doc, word) RUN of tokens: it reads the doc's sparse theta row
// once (16-byte vector loads, 4 entries per lane, cached in registers), forms
// p1 = theta * p* with a warp scan, and draws every token of the run:
//   exclusion (theta_dz-1, phi_zv-1, n_z-1) is applied in
//   O(1) by shifting u past the token's own entry in both the S and the Q
//   prefix (so the shared tree stays exclusion-free), u1 picks the branch
//   (u1 (S+Q) < S), u2 searches it by __ballot_sync.
// Philox4x32-10 counter = (global doc, word, occurrence in run, iteration).
#include "gf_internal.cuh"
#include "gf_device.cuh"

namespace gf {

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

// ptree descent (ptree.py:203-225) over the shared-memory levels: at each
// level the 32 children are compared at once with one ballot.
__device__ __forceinline__ int search_q(const float* lvl, const TreeGeom& g, float u, int lane) {
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

template <int NC>
__global__ void __launch_bounds__(kSampleThreads) sample_kernel(SampleArgs a) {
    extern __shared__ float smem[];
    float* lvl = smem;                        // Q-tree levels (level 0 = prefix of a p*)
    float* pstar = smem + a.tree.total;       // p*(k)
    __shared__ double ll_w[kSampleThreads / 32];
    __shared__ unsigned long long by_w[kSampleThreads / 32];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int4 sl = a.slices[blockIdx.x];
    const int v = sl.x, col = sl.w;
    const int K = a.K;

    // ---------------- prologue: p* and the Q prefix (block scan) ----------------
    {
        const int ipt = (K + kSampleThreads - 1) / kSampleThreads;
        const int k0 = tid * ipt;
        float acc = 0.f;
        for (int i = 0; i < ipt; ++i) {
            const int k = k0 + i;
            if (k < K) {
                const float ps = __fmul_rn(__fadd_rn((float)phi_at(a, col, k), a.beta), __ldg(a.inv_den + k));
                pstar[k] = ps;
                acc = __fadd_rn(acc, __fmul_rn(a.alpha, ps));
                lvl[k] = acc;
            }
        }
        float incl = warp_incl_scan(acc, lane);
        __shared__ float wtot[kSampleThreads / 32];
        if (lane == 31) wtot[warp] = incl;
        __syncthreads();
        if (tid == 0) {
            float run = 0.f;
            for (int w = 0; w < kSampleThreads / 32; ++w) { float t = wtot[w]; wtot[w] = run; run = __fadd_rn(run, t); }
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
    double ll = 0.0;
    unsigned long long nbytes = 0;

    // ---------------- samplers: one warp per (doc, word) run ----------------
    for (int r = sl.y + warp; r < sl.z; r += kSampleThreads / 32) {
        const uint32_t d = __ldg(a.run_doc + r);
        const uint32_t t0 = __ldg(a.run_start + r), t1 = __ldg(a.run_start + r + 1);
        const uint2 meta = __ldg(a.theta_meta + d);
        const uint32_t off = meta.x, nnz = meta.y;
        const uint32_t gdoc = a.doc_lo + d;
        nbytes += nnz;
        float S_full;

        if (nnz <= 128u * NC) {
            // ---- cached path: the row lives in registers for the whole run ----
            uint32_t e[NC][4];
            float lp[NC][4];
            float ex[NC];
            float carry[NC + 1];
            carry[0] = 0.f;
            const int nch = (int)((nnz + 127u) >> 7);
#pragma unroll
            for (int c = 0; c < NC; ++c) {
                if (c < nch) {
                    const uint32_t j0 = c * 128u + 4u * lane;
                    uint4 q4 = make_uint4(0, 0, 0, 0);
                    if (j0 < nnz) q4 = __ldg(reinterpret_cast<const uint4*>(a.theta_ent + off + j0));
                    e[c][0] = q4.x; e[c][1] = q4.y; e[c][2] = q4.z; e[c][3] = q4.w;
                    float acc = 0.f;
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        float w = 0.f;
                        if (j0 + i < nnz) w = __fmul_rn((float)(e[c][i] >> 16), pstar[e[c][i] & 0xffffu]);
                        acc = __fadd_rn(acc, w);
                        lp[c][i] = acc;
                    }
                    const float incl = warp_incl_scan(acc, lane);
                    float excl = __shfl_up_sync(kFull, incl, 1);
                    if (lane == 0) excl = 0.f;
                    ex[c] = excl;
#pragma unroll
                    for (int i = 0; i < 4; ++i) lp[c][i] = __fadd_rn(excl, lp[c][i]);
                    carry[c + 1] = __fadd_rn(carry[c], __shfl_sync(kFull, lp[c][3], 31));
                } else {
#pragma unroll
                    for (int i = 0; i < 4; ++i) { e[c][i] = 0; lp[c][i] = 0.f; }
                    ex[c] = 0.f;
                    carry[c + 1] = carry[c];
                }
            }
            S_full = carry[NC];

            for (uint32_t t = t0; t < (a.eval_only ? t0 : t1); ++t) {
                const int zt = a.z[t];
                if (zt >= K) {                        // corrupt assignment: report, keep
                    if (lane == 0) atomicMin(a.errs, (unsigned long long)t);
                    continue;
                }
                // locate the token's own topic in the row (ids ascending, unique)
                int hit = -1;
#pragma unroll
                for (int c = 0; c < NC; ++c)
#pragma unroll
                    for (int i = 0; i < 4; ++i)
                        if (c * 128 + 4 * lane + i < (int)nnz && (int)(e[c][i] & 0xffffu) == zt) hit = c * 4 + i;
                const unsigned hm = __ballot_sync(kFull, hit >= 0);
                const uint32_t phz = phi_at(a, col, zt);
                const uint32_t nz = __ldg(a.nk + zt);
                if (hm == 0u || phz == 0u || nz == 0u) {
                    if (lane == 0) atomicMin(a.errs, (unsigned long long)t);
                    continue;
                }
                const int lz = __ffs(hm) - 1;
                float cnt_m = 0.f, pprev_m = 0.f;
#pragma unroll
                for (int c = 0; c < NC; ++c)
#pragma unroll
                    for (int i = 0; i < 4; ++i)
                        if (hit == c * 4 + i) {
                            cnt_m = (float)(e[c][i] >> 16);
                            pprev_m = __fadd_rn(carry[c], i ? lp[c][i - 1] : ex[c]);
                        }
                const float cnt = __shfl_sync(kFull, cnt_m, lz);
                const float pprev = __shfl_sync(kFull, pprev_m, lz);
                const float pex = __fdiv_rn(__fadd_rn((float)(phz - 1u), a.beta), __fadd_rn((float)(nz - 1u), a.vbeta));
                const float ps = pstar[zt];
                const float wz = __fmul_rn(cnt, ps);
                const float wzx = __fmul_rn(cnt - 1.f, pex);
                const float dS = fmaxf(__fsub_rn(wz, wzx), 0.f);
                const float Sx = fmaxf(__fsub_rn(S_full, dS), 0.f);
                const float qzx = __fmul_rn(a.alpha, pex);
                const float dQ = fmaxf(__fsub_rn(__fmul_rn(a.alpha, ps), qzx), 0.f);
                const float Qx = __fsub_rn(Q, dQ);
                const float qprev = zt ? lvl[zt - 1] : 0.f;
                const uint4 rr = philox4x32_10(make_uint4(gdoc, (uint32_t)v, t - t0, a.iteration), a.key);
                const float u1 = u24(rr.x), u2 = u24(rr.y);
                int knew;
                if (__fmul_rn(u1, __fadd_rn(Sx, Qx)) < Sx) {
                    float u = __fmul_rn(u2, Sx);
                    int res = -2;                      // -2: search needed
                    if (u < pprev) {
                    } else if (u < __fadd_rn(pprev, wzx)) {
                        res = zt;
                    } else {
                        u = fminf(__fadd_rn(u, dS), prev_float(S_full));
                    }
                    if (res == -2) {
                        int cs = nch - 1;
#pragma unroll
                        for (int c = NC - 1; c >= 0; --c)
                            if (c < nch && carry[c + 1] > u) cs = c;
                        int fi = -1, fid = 0;
                        bool okw = false;
#pragma unroll
                        for (int c = 0; c < NC; ++c)
                            if (c == cs) {
#pragma unroll
                                for (int i = 3; i >= 0; --i)
                                    if (__fadd_rn(carry[c], lp[c][i]) > u) fi = i;
#pragma unroll
                                for (int i = 0; i < 4; ++i)
                                    if (i == fi) {
                                        fid = (int)(e[c][i] & 0xffffu);
                                        const float prev = i ? lp[c][i - 1] : ex[c];
                                        okw = (c * 128 + 4 * lane + i < (int)nnz) && lp[c][i] > prev;
                                    }
                            }
                        const unsigned m = __ballot_sync(kFull, fi >= 0);
                        if (m == 0u) {
                            res = zt;                  // rounding guard (measure ~1 ulp)
                        } else {
                            const int L = __ffs(m) - 1;
                            const int id = __shfl_sync(kFull, fid, L);
                            const bool ok = __shfl_sync(kFull, okw, L);
                            res = ok ? id : zt;
                        }
                    }
                    knew = res;
                } else {
                    float u = __fmul_rn(u2, Qx);
                    if (u < qprev) {
                        knew = search_q(lvl, a.tree, u, lane);
                    } else if (u < __fadd_rn(qprev, qzx)) {
                        knew = zt;
                    } else {
                        knew = search_q(lvl, a.tree, fminf(__fadd_rn(u, dQ), prev_float(Q)), lane);
                    }
                }
                if (lane == 0) a.z[t] = (uint16_t)knew;
            }
        } else {
            // ---- streaming path (long rows): two passes over the row per token ----
            const int nch = (int)((nnz + 127u) >> 7);
            S_full = -1.f;
            if (a.eval_only) {
                float sfl = 0.f;
                for (uint32_t j = lane; j < nnz; j += 32) {
                    const uint32_t ee = __ldg(a.theta_ent + off + j);
                    sfl = __fadd_rn(sfl, __fmul_rn((float)(ee >> 16), pstar[ee & 0xffffu]));
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) sfl = __fadd_rn(sfl, __shfl_xor_sync(kFull, sfl, o));
                S_full = sfl;
            }
            for (uint32_t t = t0; t < (a.eval_only ? t0 : t1); ++t) {
                const int zt = a.z[t];
                if (zt >= K) {
                    if (lane == 0) atomicMin(a.errs, (unsigned long long)t);
                    continue;
                }
                const uint32_t phz = phi_at(a, col, zt);
                const uint32_t nz = __ldg(a.nk + zt);
                const float pex = __fdiv_rn(__fadd_rn((float)(phz - 1u), a.beta), __fadd_rn((float)(nz - 1u), a.vbeta));
                // pass 1: adjusted total, unadjusted total, presence of z
                float carry = 0.f, sfl = 0.f;
                bool found = false;
                for (int c = 0; c < nch; ++c) {
                    const uint32_t j0 = c * 128u + 4u * lane;
                    uint4 q4 = make_uint4(0, 0, 0, 0);
                    if (j0 < nnz) q4 = __ldg(reinterpret_cast<const uint4*>(a.theta_ent + off + j0));
                    const uint32_t ee[4] = {q4.x, q4.y, q4.z, q4.w};
                    float acc = 0.f;
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        if (j0 + i < nnz) {
                            const int id = ee[i] & 0xffffu;
                            const float cn = (float)(ee[i] >> 16);
                            const float w = __fmul_rn(cn, pstar[id]);
                            sfl = __fadd_rn(sfl, w);
                            if (id == zt) { found = true; acc = __fadd_rn(acc, __fmul_rn(cn - 1.f, pex)); }
                            else acc = __fadd_rn(acc, w);
                        }
                    }
                    const float incl = warp_incl_scan(acc, lane);
                    carry = __fadd_rn(carry, __shfl_sync(kFull, incl, 31));
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) sfl = __fadd_rn(sfl, __shfl_xor_sync(kFull, sfl, o));
                if (S_full < 0.f) S_full = sfl;
                const bool any = __any_sync(kFull, found);
                if (!any || phz == 0u || nz == 0u) {
                    if (lane == 0) atomicMin(a.errs, (unsigned long long)t);
                    continue;
                }
                const float Sx = carry;
                const float ps = pstar[zt];
                const float qzx = __fmul_rn(a.alpha, pex);
                const float dQ = fmaxf(__fsub_rn(__fmul_rn(a.alpha, ps), qzx), 0.f);
                const float Qx = __fsub_rn(Q, dQ);
                const float qprev = zt ? lvl[zt - 1] : 0.f;
                const uint4 rr = philox4x32_10(make_uint4(gdoc, (uint32_t)v, t - t0, a.iteration), a.key);
                const float u1 = u24(rr.x), u2 = u24(rr.y);
                int knew = zt;
                if (__fmul_rn(u1, __fadd_rn(Sx, Qx)) < Sx) {
                    const float u = __fmul_rn(u2, Sx);
                    float cy = 0.f;
                    for (int c = 0; c < nch; ++c) {
                        const uint32_t j0 = c * 128u + 4u * lane;
                        uint4 q4 = make_uint4(0, 0, 0, 0);
                        if (j0 < nnz) q4 = __ldg(reinterpret_cast<const uint4*>(a.theta_ent + off + j0));
                        const uint32_t ee[4] = {q4.x, q4.y, q4.z, q4.w};
                        float lpl[4];
                        float acc = 0.f;
#pragma unroll
                        for (int i = 0; i < 4; ++i) {
                            float w = 0.f;
                            if (j0 + i < nnz) {
                                const int id = ee[i] & 0xffffu;
                                const float cn = (float)(ee[i] >> 16);
                                w = (id == zt) ? __fmul_rn(cn - 1.f, pex) : __fmul_rn(cn, pstar[id]);
                            }
                            acc = __fadd_rn(acc, w);
                            lpl[i] = acc;
                        }
                        const float incl = warp_incl_scan(acc, lane);
                        float excl = __shfl_up_sync(kFull, incl, 1);
                        if (lane == 0) excl = 0.f;
                        int fi = -1;
#pragma unroll
                        for (int i = 3; i >= 0; --i) {
                            lpl[i] = __fadd_rn(excl, lpl[i]);
                            if (__fadd_rn(cy, lpl[i]) > u) fi = i;
                        }
                        const float ctot = __shfl_sync(kFull, lpl[3], 31);
                        const unsigned m = __ballot_sync(kFull, fi >= 0);
                        if (m || c == nch - 1) {
                            if (m) {
                                const int L = __ffs(m) - 1;
                                int fid = 0;
                                bool okw = false;
#pragma unroll
                                for (int i = 0; i < 4; ++i)
                                    if (i == fi) {
                                        fid = ee[i] & 0xffffu;
                                        okw = (j0 + i < nnz) && lpl[i] > (i ? lpl[i - 1] : excl);
                                    }
                                const int id = __shfl_sync(kFull, fid, L);
                                knew = __shfl_sync(kFull, okw, L) ? id : zt;
                            }
                            break;
                        }
                        cy = __fadd_rn(cy, ctot);
                    }
                } else {
                    float u = __fmul_rn(u2, Qx);
                    if (u < qprev) knew = search_q(lvl, a.tree, u, lane);
                    else if (u < __fadd_rn(qprev, qzx)) knew = zt;
                    else knew = search_q(lvl, a.tree, fminf(__fadd_rn(u, dQ), prev_float(Q)), lane);
                }
                if (lane == 0) a.z[t] = (uint16_t)knew;
            }
            if (S_full < 0.f) S_full = 0.f;
        }
        // log p(w|d) * (L_d + K a) of the iteration-start model, once per run
        ll += (double)(t1 - t0) * log((double)S_full + (double)Q);
    }
    if (lane == 0) { ll_w[warp] = ll; by_w[warp] = nbytes; }
    __syncthreads();
    if (tid == 0) {
        double s = 0.0;
        unsigned long long b = 0;
        for (int w = 0; w < kSampleThreads / 32; ++w) { s += ll_w[w]; b += by_w[w]; }
        a.ll_part[blockIdx.x] = s;
        atomicAdd(a.bytes, b);
    }
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
    const size_t smem = (size_t)(s->tree.total + s->K) * sizeof(float);
    static bool attr_set = false;
    if (!attr_set) {
        cudaError_t e = cudaFuncSetAttribute(sample_kernel<kRowChunks>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             200 * 1024);
        if (e != cudaSuccess) return e;
        attr_set = true;
    }
    sample_kernel<kRowChunks><<<(unsigned)s->n_slices, kSampleThreads, smem, s->stream>>>(a);
    return cudaGetLastError();
}

}  // namespace gf
