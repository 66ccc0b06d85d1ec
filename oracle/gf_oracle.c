/*
 * gf_oracle.c -- CPU ORACLE for the gibbsflow hot path.  TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference package `gibbsflow`
 * (/root/reference/pkg/src/gibbsflow) and of the SPEC sections that describe
 * the parts the package leaves unimplemented (sampler / engine / eval).  Only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference legs may load this library, and only as the checker or as the CPU
 * baseline -- never as the product path.  Every function cites the reference
 * file:line it follows.
 *
 * Parity pinning: rng / partition / rebuild / ptree results are checked against
 * golden vectors generated from the reference itself (tests/golden/ fixtures,
 * made by tests/golden/make_golden.py).  The sampler and log-likelihood have no
 * reference code: they follow SPEC.md:230-305 and
 * SPEC.md:391-419 and are pinned by the SPEC's hand examples plus analytic
 * (chi-square / exact-distribution) tests.
 *
 * Build: see oracle/Makefile (gcc -O2 -fopenmp -shared).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define GOLDEN 0x9E3779B97F4A7C15ULL
#define MIX1 0xBF58476D1CE4E5B9ULL
#define MIX2 0x94D049BB133111EBULL

/* ------------------------------------------------------------------ rng --
 * splitmix64 counter streams: rng.py:20-42 (_finalize, mix64, stream_uniform). */
static inline uint64_t gfo_fin(uint64_t z) {            /* rng.py:20-26 */
    z = (z ^ (z >> 30)) * MIX1;
    z = (z ^ (z >> 27)) * MIX2;
    return z ^ (z >> 31);
}

uint64_t gfo_stream_key(const uint64_t* parts, int n) { /* rng.py:29-35, 45-53 */
    uint64_t h = GOLDEN;
    for (int i = 0; i < n; ++i) h = gfo_fin(h + GOLDEN + parts[i]);
    return h;
}

static inline double gfo_uniform(uint64_t key, uint64_t ctr) { /* rng.py:38-42 */
    uint64_t bits = gfo_fin(key + GOLDEN * (ctr + 1ULL));
    return (double)(bits >> 11) * (1.0 / 9007199254740992.0);
}

void gfo_stream_uniforms(uint64_t key, uint64_t counter, int64_t n, double* out) { /* rng.py:84-89 */
    for (int64_t i = 0; i < n; ++i) out[i] = gfo_uniform(key, counter + (uint64_t)i);
}

/* Philox4x32-10 (Salmon et al. 2011, Random123 constants).  Not in the
 * reference: the north star replaces the per-chunk splitmix stream inside the
 * sampler by a counter RNG keyed by (seed, iteration, token).  Pinned by the
 * Random123 known-answer vectors in tests/test_oracle_golden.py. */
static inline void philox_round(uint32_t c[4], const uint32_t k[2]) {
    uint64_t p0 = (uint64_t)0xD2511F53u * c[0];
    uint64_t p1 = (uint64_t)0xCD9E8D57u * c[2];
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    uint32_t n0 = hi1 ^ c[1] ^ k[0], n2 = hi0 ^ c[3] ^ k[1];
    c[0] = n0; c[1] = lo1; c[2] = n2; c[3] = lo0;
}

void gfo_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
    uint32_t c[4] = {ctr[0], ctr[1], ctr[2], ctr[3]};
    uint32_t k[2] = {key[0], key[1]};
    for (int r = 0; r < 10; ++r) {
        if (r) { k[0] += 0x9E3779B9u; k[1] += 0xBB67AE85u; }
        philox_round(c, k);
    }
    out[0] = c[0]; out[1] = c[1]; out[2] = c[2]; out[3] = c[3];
}

/* The two sampling uniforms of one token (the product kernel's convention):
 * counter = (global doc, word, occurrence within the (doc, word) run, iteration),
 * key = (seed lo, seed hi); u1 = top 24 bits of word 0, u2 = of word 1, both in [0,1). */
void gfo_token_uniforms(uint64_t seed, uint32_t iteration, uint32_t doc, uint32_t word,
                        uint32_t occ, double* u1, double* u2) {
    uint32_t ctr[4] = {doc, word, occ, iteration};
    uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    uint32_t r[4];
    gfo_philox4x32_10(ctr, key, r);
    *u1 = (double)(r[0] >> 8) * (1.0 / 16777216.0);
    *u2 = (double)(r[1] >> 8) * (1.0 / 16777216.0);
}

/* ------------------------------------------------------------ corpus --
 * greedy_boundaries: corpus.py:210-237.  Returns -1 when C > D (PartitionError). */
int gfo_greedy_boundaries(const int64_t* lengths, int64_t D, int64_t C, int64_t* out) {
    if (C > D) return -1;
    int64_t remaining = 0;
    for (int64_t i = 0; i < D; ++i) remaining += lengths[i];
    int64_t lo = 0;
    for (int64_t c = 0; c < C; ++c) {
        int64_t left = C - c, hi_max = D - (left - 1);
        int64_t target = (remaining + left - 1) / left;  /* ceil */
        int64_t acc = 0, hi = lo;
        while (hi < hi_max && acc < target) acc += lengths[hi++];
        out[2 * c] = lo; out[2 * c + 1] = hi;
        remaining -= acc;
        lo = hi;
    }
    return 0;
}

/* One chunk of partition(): corpus.py:252-286.  Inputs are the chunk's tokens in
 * corpus (doc-major) order.  Stable word sort == counting sort by word
 * (corpus.py:256-258); the group directory is np.unique's ascending words
 * (260-262); the doc-word map is a stable counting sort by local doc (201-207);
 * initial topics z = min(floor(u*K), K-1) from Stream(seed, cid) in
 * word-sorted order (265-269).  Returns the number of groups. */
int64_t gfo_partition_chunk(const int32_t* doc_ids, const int32_t* word_ids, int64_t n,
                            int64_t doc_lo, int64_t doc_hi, int32_t V, int32_t K,
                            uint64_t seed, int64_t cid,
                            int32_t* out_doc, int32_t* out_word, uint16_t* out_z,
                            int32_t* grp_words, int64_t* grp_off, int64_t* grp_size,
                            int64_t* dw_ptr, int64_t* dw_tok) {
    int64_t* cnt = (int64_t*)calloc((size_t)V + 1, sizeof(int64_t));
    for (int64_t i = 0; i < n; ++i) cnt[word_ids[i] + 1]++;
    for (int32_t v = 0; v < V; ++v) cnt[v + 1] += cnt[v];
    int64_t ng = 0;
    for (int32_t v = 0; v < V; ++v)
        if (cnt[v + 1] > cnt[v]) {
            grp_words[ng] = v; grp_off[ng] = cnt[v]; grp_size[ng] = cnt[v + 1] - cnt[v]; ++ng;
        }
    for (int64_t i = 0; i < n; ++i) {
        int64_t p = cnt[word_ids[i]]++;
        out_doc[p] = doc_ids[i]; out_word[p] = word_ids[i];
    }
    free(cnt);
    int64_t nd = doc_hi - doc_lo;
    memset(dw_ptr, 0, sizeof(int64_t) * (size_t)(nd + 1));
    for (int64_t i = 0; i < n; ++i) dw_ptr[out_doc[i] - doc_lo + 1]++;
    for (int64_t d = 0; d < nd; ++d) dw_ptr[d + 1] += dw_ptr[d];
    int64_t* fill = (int64_t*)malloc(sizeof(int64_t) * (size_t)(nd + 1));
    memcpy(fill, dw_ptr, sizeof(int64_t) * (size_t)(nd + 1));
    for (int64_t i = 0; i < n; ++i) dw_tok[fill[out_doc[i] - doc_lo]++] = i;
    free(fill);
    uint64_t parts[2] = {seed, (uint64_t)cid};
    uint64_t key = gfo_stream_key(parts, 2);
    for (int64_t i = 0; i < n; ++i) {
        double u = gfo_uniform(key, (uint64_t)i);
        int64_t z = (int64_t)(u * (double)K);
        out_z[i] = (uint16_t)(z < K - 1 ? z : K - 1);
    }
    return ng;
}

/* ------------------------------------------------------------- model --
 * rebuild_theta: model.py:91-124.  Dense per-doc histogram via the doc-word
 * map, then ascending nonzero compaction.  On a count > 65535 returns 1 with
 * the first offending (global) document and its max count (model.py:101-104). */
int gfo_rebuild_theta(const uint16_t* z, const int64_t* dw_ptr, const int64_t* dw_tok,
                      int64_t nd, int32_t K, int64_t doc_lo,
                      int64_t* row_ptr, uint16_t* ids, uint16_t* cnts,
                      int64_t* err_doc, int64_t* err_count) {
    int64_t* dense = (int64_t*)calloc((size_t)K, sizeof(int64_t));
    row_ptr[0] = 0;
    int64_t nnz = 0;
    for (int64_t d = 0; d < nd; ++d) {
        int64_t mx = 0;
        for (int64_t p = dw_ptr[d]; p < dw_ptr[d + 1]; ++p) dense[z[dw_tok[p]]]++;
        for (int32_t k = 0; k < K; ++k) if (dense[k] > mx) mx = dense[k];
        if (mx > 65535) {
            *err_doc = doc_lo + d; *err_count = mx; free(dense); return 1;
        }
        for (int32_t k = 0; k < K; ++k)
            if (dense[k]) { ids[nnz] = (uint16_t)k; cnts[nnz] = (uint16_t)dense[k]; ++nnz; dense[k] = 0; }
        row_ptr[d + 1] = nnz;
    }
    free(dense);
    return 0;
}

/* rebuild_phi_replica: model.py:142-161 (dense K x V count, 64-bit cells). */
void gfo_rebuild_phi(const uint16_t* z, const int32_t* w, int64_t n, int32_t K, int32_t V,
                     int64_t* counts, int64_t* totals) {
    memset(counts, 0, sizeof(int64_t) * (size_t)K * (size_t)V);
    memset(totals, 0, sizeof(int64_t) * (size_t)K);
    for (int64_t i = 0; i < n; ++i) { counts[(int64_t)z[i] * V + w[i]]++; totals[z[i]]++; }
}

/* ----------------------------------------------------------- sampler --
 * SPEC.md:249-284, 359-367 (sample_dense / build_word_context /
 * sample_sparse / exclusion_adjust / sample_chunk), deferred semantics
 * SPEC.md:377, in the SPEC's 64-bit oracle mode.
 *
 * Tokens arrive in word-sorted order.  For each token (doc d, word v, topic z):
 *   p*[k]   = (phi[k][v] + b) / (n_k + V b)
 *   exclusion: theta_dz-1, phi_zv-1, n_z-1 (view only)
 *   p1_j    = theta'_{d,k_j} p*'[k_j] over the row, ascending ids
 *   p2_k    = a p*'[k];  S = sum p1, Q = sum p2
 *   u1 * (S+Q) < S  -> scan p1 with u = u2 S, else scan p2 with u = u2 Q
 *   scan = minimal index whose running prefix exceeds u (ptree.py:7-11, 190-197);
 *   if rounding leaves none, the last positive-weight index (ptree.py:218).
 * Uniforms: gfo_token_uniforms with occ = position inside the run of
 * consecutive tokens sharing (doc, word).  Returns 0, or 3 (ConsistencyError)
 * with *err_tok set when the token's topic is absent from its row. */
static int64_t scan_pick(const double* w, int64_t n, double u) {
    double acc = 0.0;
    int64_t last = -1;
    for (int64_t j = 0; j < n; ++j) {
        if (w[j] > 0) last = j;
        acc += w[j];
        if (acc > u) return j;
    }
    return last;
}

/* minimal k with prefix[k] > u (np.searchsorted side="right"); K-1 if none */
static int64_t first_above(const double* prefix, int64_t n, double u) {
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        int64_t mid = (lo + hi) >> 1;
        if (prefix[mid] > u) hi = mid; else lo = mid + 1;
    }
    return lo < n ? lo : n - 1;
}

int gfo_sample_tokens(int32_t K, int32_t V, double alpha, double beta, uint64_t seed,
                      uint32_t iteration, int64_t T, const int32_t* tok_doc,
                      const int32_t* tok_word, uint16_t* z,
                      int64_t doc_lo, const int64_t* th_ptr, const uint16_t* th_ids,
                      const uint16_t* th_cnt, const uint32_t* phi, const int64_t* totals,
                      int nthreads, int64_t* err_tok) {
    if (T == 0) return 0;
    /* segment boundaries = word changes; occ = index inside (doc, word) run */
    uint32_t* occ = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)T);
    int64_t* seg = (int64_t*)malloc(sizeof(int64_t) * (size_t)(T + 1));
    int64_t nseg = 0;
    for (int64_t t = 0; t < T; ++t) {
        int same_word = t > 0 && tok_word[t] == tok_word[t - 1];
        if (!same_word) seg[nseg++] = t;
        occ[t] = (same_word && tok_doc[t] == tok_doc[t - 1]) ? occ[t - 1] + 1 : 0;
    }
    seg[nseg] = T;
    int status = 0;
    int64_t bad = INT64_MAX;
    const double vb = (double)V * beta;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#endif
    /* word-major copy of phi (the K x V reference layout has stride V down a column) */
    uint32_t* phiT = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)K * (size_t)V);
#ifdef _OPENMP
#pragma omp parallel for schedule(static)
#endif
    for (int64_t vb0 = 0; vb0 < V; vb0 += 64)
        for (int32_t k = 0; k < K; ++k)
            for (int64_t vv = vb0; vv < vb0 + 64 && vv < V; ++vv) phiT[vv * K + k] = phi[(int64_t)k * V + vv];
#ifdef _OPENMP
#pragma omp parallel
#endif
    {
        double* pstar = (double*)malloc(sizeof(double) * (size_t)K);
        double* qpre = (double*)malloc(sizeof(double) * (size_t)K);
        double* p1 = (double*)malloc(sizeof(double) * (size_t)K);
#ifdef _OPENMP
#pragma omp for schedule(dynamic, 1)
#endif
        for (int64_t s = 0; s < nseg; ++s) {
            /* build_word_context: p* and the prefix of a p*, once per word */
            const int32_t v = tok_word[seg[s]];
            double acc = 0.0;
            for (int32_t k = 0; k < K; ++k) {
                pstar[k] = ((double)phiT[(int64_t)v * K + k] + beta) / ((double)totals[k] + vb);
                acc += alpha * pstar[k];
                qpre[k] = acc;
            }
            const double Q = qpre[K - 1];
            for (int64_t t = seg[s]; t < seg[s + 1]; ++t) {
                const int32_t d = tok_doc[t];
                const int32_t zt = z[t];
                const int64_t r0 = th_ptr[d - doc_lo], r1 = th_ptr[d - doc_lo + 1];
                if (zt >= K || phi[(int64_t)zt * V + v] == 0 || totals[zt] == 0) {
#ifdef _OPENMP
#pragma omp critical
#endif
                    { status = 3; if (t < bad) bad = t; }
                    continue;
                }
                const double pex = ((double)phi[(int64_t)zt * V + v] - 1.0 + beta) /
                                   ((double)totals[zt] - 1.0 + vb);
                double S = 0.0;
                int found = 0;
                for (int64_t j = r0; j < r1; ++j) {      /* p1 with exclusion */
                    double c = (double)th_cnt[j];
                    double ps = pstar[th_ids[j]];
                    if (th_ids[j] == zt) { c -= 1.0; ps = pex; found = 1; }
                    p1[j - r0] = c * ps;
                    S += p1[j - r0];
                }
                if (!found) {
#ifdef _OPENMP
#pragma omp critical
#endif
                    { status = 3; if (t < bad) bad = t; }
                    continue;
                }
                /* exclusion-adjusted p2: entries below z unchanged, z carries
                 * a p*_ex(z), entries above shift down by dq (exact-arithmetic
                 * equivalent of scanning the adjusted weights) */
                const double qzx = alpha * pex, dq = alpha * pstar[zt] - qzx, Qx = Q - dq;
                double u1, u2;
                gfo_token_uniforms(seed, iteration, (uint32_t)d, (uint32_t)v, occ[t], &u1, &u2);
                int64_t pick;
                if (u1 * (S + Qx) < S) {
                    pick = th_ids[r0 + scan_pick(p1, r1 - r0, u2 * S)];
                } else {
                    const double u = u2 * Qx, before = zt ? qpre[zt - 1] : 0.0;
                    if (u < before) pick = first_above(qpre, K, u);
                    else if (u < before + qzx) pick = zt;
                    else {
                        pick = first_above(qpre, K, u + dq);
                        if (pick <= zt) pick = zt + 1 < K ? zt + 1 : zt;   /* rounding guard */
                    }
                }
                z[t] = (uint16_t)pick;
            }
        }
        free(pstar); free(qpre); free(p1);
    }
    free(phiT);
    free(occ); free(seg);
    if (status) *err_tok = bad;
    return status;
}

/* Exact draw from the exclusion-adjusted conditional by two sequential passes
 * over k = 0..K-1 (theta row merged in topic order): the thinning loop's
 * fallback once it has rejected its 64th proposal, so the kept topic follows
 * the exclusion-adjusted Eq. 1 whatever the acceptance rate (a capped loop
 * that simply kept z would over-weight z by the chance of 64 rejections).
 * Weights: (theta_dk + a) p*(k) for k != z, (theta_dz - 1 + a) p*_ex(z). */
static int32_t exact_excluded_draw(int32_t K, double alpha, const double* pstar, double pex_z,
                                   const uint16_t* ids, const uint16_t* cnts, int64_t n, int32_t zt,
                                   double u) {
    double tot = 0.0;
    int64_t j = 0;
    for (int32_t k = 0; k < K; ++k) {
        double c = 0.0;
        if (j < n && ids[j] == k) c = (double)cnts[j++];
        tot += k == zt ? (c - 1.0 + alpha) * pex_z : (c + alpha) * pstar[k];
    }
    const double target = u * tot;
    double acc = 0.0;
    int32_t last = 0;
    j = 0;
    for (int32_t k = 0; k < K; ++k) {
        double c = 0.0;
        if (j < n && ids[j] == k) c = (double)cnts[j++];
        const double w = k == zt ? (c - 1.0 + alpha) * pex_z : (c + alpha) * pstar[k];
        if (w > 0.0) last = k;
        acc += w;
        if (acc > target) return k;
    }
    return last;
}

/* The product kernel's form of the same draw (csrc/k_sample.cu): exclusion by
 * THINNING.  Draw k from the exclusion-free S+Q mixture of SPEC.md:267-275 with
 * uniforms (b, s) of Philox block (doc, word, occ | retry << 26, iteration); if
 * k == z keep it with probability (theta_dz - 1 + a) p*_ex(z) / ((theta_dz + a) p*(z))
 * (uniform t), else redraw with retry + 1; the 64th rejection ends in one
 * exact draw (exact_excluded_draw, uniform = word 3 of that block).  The kept k follows the same
 * exclusion-adjusted Eq. 1 distribution as gfo_sample_tokens (tests compare
 * both against gfo_conditional); this variant exists so the device can be
 * checked draw for draw. */
int gfo_sample_tokens_thin(int32_t K, int32_t V, double alpha, double beta, uint64_t seed,
                           uint32_t iteration, int64_t T, const int32_t* tok_doc,
                           const int32_t* tok_word, uint16_t* z,
                           int64_t doc_lo, const int64_t* th_ptr, const uint16_t* th_ids,
                           const uint16_t* th_cnt, const uint32_t* phi, const int64_t* totals,
                           int nthreads, int64_t* err_tok) {
    if (T == 0) return 0;
    uint32_t* occ = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)T);
    int64_t* seg = (int64_t*)malloc(sizeof(int64_t) * (size_t)(T + 1));
    int64_t nseg = 0;
    for (int64_t t = 0; t < T; ++t) {
        int same_word = t > 0 && tok_word[t] == tok_word[t - 1];
        if (!same_word) seg[nseg++] = t;
        occ[t] = (same_word && tok_doc[t] == tok_doc[t - 1]) ? occ[t - 1] + 1 : 0;
    }
    seg[nseg] = T;
    int status = 0;
    int64_t bad = INT64_MAX;
    const double vb = (double)V * beta;
    const uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#endif
    uint32_t* phiT = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)K * (size_t)V);
#ifdef _OPENMP
#pragma omp parallel for schedule(static)
#endif
    for (int64_t vb0 = 0; vb0 < V; vb0 += 64)
        for (int32_t k = 0; k < K; ++k)
            for (int64_t vv = vb0; vv < vb0 + 64 && vv < V; ++vv) phiT[vv * K + k] = phi[(int64_t)k * V + vv];
#ifdef _OPENMP
#pragma omp parallel
#endif
    {
        double* pstar = (double*)malloc(sizeof(double) * (size_t)K);
        double* pex = (double*)malloc(sizeof(double) * (size_t)K);
        double* qpre = (double*)malloc(sizeof(double) * (size_t)K);
#ifdef _OPENMP
#pragma omp for schedule(dynamic, 1)
#endif
        for (int64_t s = 0; s < nseg; ++s) {
            const int32_t v = tok_word[seg[s]];
            double acc = 0.0;
            for (int32_t k = 0; k < K; ++k) {
                const double ph = (double)phiT[(int64_t)v * K + k], nk = (double)totals[k];
                pstar[k] = (ph + beta) / (nk + vb);
                pex[k] = (ph >= 1.0 && nk >= 1.0) ? (ph - 1.0 + beta) / (nk - 1.0 + vb) : 0.0;
                acc += alpha * pstar[k];
                qpre[k] = acc;
            }
            const double Q = qpre[K - 1];
            for (int64_t t = seg[s]; t < seg[s + 1]; ++t) {
                const int32_t d = tok_doc[t];
                const int32_t zt = z[t];
                const int64_t r0 = th_ptr[d - doc_lo], r1 = th_ptr[d - doc_lo + 1];
                double S = 0.0;
                for (int64_t j = r0; j < r1; ++j) S += (double)th_cnt[j] * pstar[th_ids[j]];
                int32_t k = zt;
                for (uint32_t retry = 0; retry <= 63; ++retry) {
                    uint32_t ctr[4] = {(uint32_t)d, (uint32_t)v, occ[t] | (retry << 26), iteration};
                    uint32_t r[4];
                    gfo_philox4x32_10(ctr, key, r);
                    const double ub = (double)(r[0] >> 8) * (1.0 / 16777216.0);
                    const double us = (double)(r[1] >> 8) * (1.0 / 16777216.0);
                    const double ut = (double)(r[2] >> 8) * (1.0 / 16777216.0);
                    int64_t cnt = 0;
                    if (ub * (S + Q) < S) {
                        const double target = us * S;
                        double a2 = 0.0;
                        int64_t pick = r1 - 1;
                        for (int64_t j = r0; j < r1; ++j) {
                            a2 += (double)th_cnt[j] * pstar[th_ids[j]];
                            if (a2 > target) { pick = j; break; }
                        }
                        k = th_ids[pick];
                        cnt = th_cnt[pick];
                    } else {
                        k = (int32_t)first_above(qpre, K, us * Q);
                        if (k == zt)
                            for (int64_t j = r0; j < r1; ++j)
                                if (th_ids[j] == zt) { cnt = th_cnt[j]; break; }
                    }
                    if (k != zt) break;
                    if (zt >= K || cnt == 0 || pex[zt] == 0.0) {
#ifdef _OPENMP
#pragma omp critical
#endif
                        { status = 3; if (t < bad) bad = t; }
                        break;
                    }
                    if (ut * ((double)cnt + alpha) * pstar[zt] < ((double)cnt - 1.0 + alpha) * pex[zt]) break;
                    if (retry == 63) {   /* 64 rejections: one exact draw (4th word of this block) */
                        const double uf = (double)(r[3] >> 8) * (1.0 / 16777216.0);
                        k = exact_excluded_draw(K, alpha, pstar, pex[zt], th_ids + r0, th_cnt + r0, r1 - r0, zt, uf);
                        break;
                    }
                    k = zt;
                }
                z[t] = (uint16_t)k;
            }
        }
        free(pstar); free(pex); free(qpre);
    }
    free(phiT); free(occ); free(seg);
    if (status) *err_tok = bad;
    return status;
}

/* Exact exclusion-adjusted Eq. 1 distribution of one token (SPEC:249-257,
 * 276-284): probs[k] proportional to (theta'_dk + a)(phi'_kv + b)/(n'_k + V b).
 * theta_dense is the document's dense row.  Also returns the decomposed
 * branch masses: probs_decomposed[k] = (p1(k)+p2(k))/(S+Q). */
void gfo_conditional(int32_t K, int32_t V, double alpha, double beta,
                     const int64_t* theta_dense, const uint32_t* phi_col /*K entries for word v*/,
                     const int64_t* totals, int32_t zt, int exclusion,
                     double* probs, double* probs_decomposed) {
    const double vb = (double)V * beta;
    double tot = 0.0, S = 0.0, Q = 0.0;
    for (int32_t k = 0; k < K; ++k) {
        double th = (double)theta_dense[k], ph = (double)phi_col[k], nk = (double)totals[k];
        if (exclusion && k == zt) { th -= 1.0; ph -= 1.0; nk -= 1.0; }
        double ps = (ph + beta) / (nk + vb);
        probs[k] = (th + alpha) * ps;
        tot += probs[k];
        probs_decomposed[k] = th * ps + alpha * ps;
        S += th * ps; Q += alpha * ps;
    }
    for (int32_t k = 0; k < K; ++k) { probs[k] /= tot; probs_decomposed[k] /= (S + Q); }
}

/* ---------------------------------------------------------------- eval --
 * loglik_per_token, naive O(T K) form, 64-bit.  theta is CSR
 * over global docs [0, D) (row_ptr int64); doc_len[d] = L_d. */
double gfo_loglik_naive(int32_t K, int32_t V, double alpha, double beta, int64_t T,
                        const int32_t* tok_doc, const int32_t* tok_word,
                        const int64_t* th_ptr, const uint16_t* th_ids, const uint16_t* th_cnt,
                        const int64_t* doc_len, const uint32_t* phi, const int64_t* totals,
                        int nthreads) {
    const double vb = (double)V * beta;
    double acc = 0.0;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel
#endif
    {
        double* dense = (double*)calloc((size_t)K, sizeof(double));
#ifdef _OPENMP
#pragma omp for reduction(+ : acc) schedule(static)
#endif
        for (int64_t t = 0; t < T; ++t) {
            int32_t d = tok_doc[t], v = tok_word[t];
            for (int64_t j = th_ptr[d]; j < th_ptr[d + 1]; ++j) dense[th_ids[j]] = th_cnt[j];
            double denom = (double)doc_len[d] + (double)K * alpha, s = 0.0;
            for (int32_t k = 0; k < K; ++k)
                s += (dense[k] + alpha) / denom * (((double)phi[(int64_t)k * V + v] + beta) / ((double)totals[k] + vb));
            acc += log(s);
            for (int64_t j = th_ptr[d]; j < th_ptr[d + 1]; ++j) dense[th_ids[j]] = 0.0;
        }
        free(dense);
    }
    return acc / (double)T;
}

/* loglik_per_token in the S + Q form (equal to SPEC.md:405 by
 * sum_k (theta_dk + a) p*_vk = S_full + a sum_k p*_vk), O(T K_d + W K): tokens
 * word-grouped (a partitioned chunk), theta rows over local docs
 * [doc_lo, doc_lo + D), doc_len indexed locally.  Per-segment partials summed in
 * segment order: deterministic for any thread count.  For large corpora where
 * gfo_loglik_naive's O(T K) is too slow (tools/trajectory.py). */
double gfo_loglik_sq(int32_t K, int32_t V, double alpha, double beta, int64_t T, const int32_t* tok_doc,
                     const int32_t* tok_word, int64_t doc_lo, const int64_t* th_ptr, const uint16_t* th_ids,
                     const uint16_t* th_cnt, const int64_t* doc_len, const uint32_t* phi, const int64_t* totals,
                     int nthreads) {
    if (T == 0) return 0.0;
    int64_t* seg = (int64_t*)malloc(sizeof(int64_t) * (size_t)(T + 1));
    int64_t nseg = 0;
    for (int64_t t = 0; t < T; ++t)
        if (t == 0 || tok_word[t] != tok_word[t - 1]) seg[nseg++] = t;
    seg[nseg] = T;
    double* part = (double*)calloc((size_t)nseg, sizeof(double));
    const double vb = (double)V * beta;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel
#endif
    {
        double* pstar = (double*)malloc(sizeof(double) * (size_t)K);
#ifdef _OPENMP
#pragma omp for schedule(dynamic, 1)
#endif
        for (int64_t s = 0; s < nseg; ++s) {
            const int32_t v = tok_word[seg[s]];
            double q = 0.0;
            for (int32_t k = 0; k < K; ++k) {
                pstar[k] = ((double)phi[(int64_t)k * V + v] + beta) / ((double)totals[k] + vb);
                q += alpha * pstar[k];
            }
            double acc = 0.0;
            for (int64_t t = seg[s]; t < seg[s + 1]; ++t) {
                const int64_t d = tok_doc[t] - doc_lo;
                double sf = 0.0;
                for (int64_t j = th_ptr[d]; j < th_ptr[d + 1]; ++j) sf += (double)th_cnt[j] * pstar[th_ids[j]];
                acc += log((sf + q) / ((double)doc_len[d] + (double)K * alpha));
            }
            part[s] = acc;
        }
        free(pstar);
    }
    double total = 0.0;
    for (int64_t s = 0; s < nseg; ++s) total += part[s];
    free(part);
    free(seg);
    return total / (double)T;
}
