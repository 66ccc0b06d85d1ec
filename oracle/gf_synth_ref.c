/*
 * gf_synth_ref.c -- the benchmark's synthetic LDA corpora, restated in plain C
 * for the CPU side.  TEST / BENCHMARK INFRASTRUCTURE ONLY.
 *
 * The reference has no datasets offline, so bench.py generates seeded
 * LDA-generative corpora (SURVEY.md section 8d "Synthetic inputs").  The GPU
 * arm builds them with the product library (csrc/gf_synth.cpp); the
 * `--impl reference` arm must not load the product library, so it generates
 * the SAME corpus here: identical splitmix64 streams keyed by (seed, stream,
 * doc / topic), identical libm calls in the identical order, identical
 * tie-breaking of the per-topic word orders.  tests/test_oracle_golden.py
 * checks the two generators produce equal arrays.
 *
 * Model: K_true topics, each a Zipf(s) law over its own jittered ordering of
 * the vocabulary (log-rank + N(0, 1)); per-document mixtures Dir(doc_alpha)
 * (Marsaglia-Tsang gamma, boosted below shape 1); log-normal document lengths
 * with the requested mean.
 */
#define _GNU_SOURCE
#include <math.h>
#include <stdint.h>
#include <stdlib.h>

#define GOLDEN 0x9E3779B97F4A7C15ULL

static inline uint64_t fin(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

typedef struct {
    uint64_t key, ctr;
} rng_t;

static inline double ru(rng_t* r) {
    ++r->ctr;
    return (double)(fin(r->key + GOLDEN * r->ctr) >> 11) * (1.0 / 9007199254740992.0);
}

static double rnormal(rng_t* r) {
    double a = ru(r), b = ru(r);
    if (a < 1e-300) a = 1e-300;
    return sqrt(-2.0 * log(a)) * cos(6.283185307179586 * b);
}

static double rgamma(rng_t* r, double k) {
    if (k < 1.0) {
        double g = rgamma(r, k + 1.0), x = ru(r);
        if (x < 1e-300) x = 1e-300;
        return g * pow(x, 1.0 / k);
    }
    const double d = k - 1.0 / 3.0, c = 1.0 / sqrt(9.0 * d);
    for (;;) {
        double x = rnormal(r), v = 1.0 + c * x;
        if (v <= 0) continue;
        v = v * v * v;
        double uu = ru(r);
        if (uu < 1 - 0.0331 * x * x * x * x) return d * v;
        if (log(uu > 1e-300 ? uu : 1e-300) < 0.5 * x * x + d * (1 - v + log(v))) return d * v;
    }
}

static uint64_t key_of(uint64_t seed, uint64_t a, uint64_t b) {
    uint64_t h = GOLDEN;
    const uint64_t parts[3] = {seed, a, b};
    for (int i = 0; i < 3; ++i) h = fin(h + GOLDEN + parts[i]);
    return h;
}

/* first index i in [0, n) with a[i] > x, n when none (std::upper_bound) */
static inline int64_t upper(const double* a, int64_t n, double x) {
    int64_t lo = 0, len = n;
    while (len > 0) {
        int64_t half = len >> 1;
        if (!(x < a[lo + half])) { lo += half + 1; len -= half + 1; }
        else len = half;
    }
    return lo;
}

int gfo_synth_lengths(uint64_t seed, int64_t doc_begin, int64_t num_docs, double mean_len, double sigma,
                      int64_t* out) {
    if (num_docs < 0 || !(mean_len >= 1.0) || !(sigma >= 0.0)) return -1;
    const double mu = log(mean_len) - 0.5 * sigma * sigma;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < num_docs; ++i) {
        rng_t r = {key_of(seed, 1, (uint64_t)(doc_begin + i)), 0};
        int64_t L = llround(exp(mu + sigma * rnormal(&r)));
        out[i] = L > 1 ? L : 1;
    }
    return 0;
}

static int cmp_rank(const void* x, const void* y, void* arg) {
    const double* key = (const double*)arg;
    const int32_t a = *(const int32_t*)x, b = *(const int32_t*)y;
    if (key[a] < key[b]) return -1;
    if (key[b] < key[a]) return 1;
    return (a > b) - (a < b);
}

int gfo_synth_tokens(uint64_t seed, int64_t doc_begin, int64_t num_docs, const int64_t* doc_ptr, int32_t V,
                     int32_t k_true, double zipf_s, double doc_alpha, int32_t* doc_out, int32_t* word_out) {
    if (V < 1 || k_true < 1 || num_docs < 0) return -1;
    double* cdf = (double*)malloc(sizeof(double) * (size_t)V);
    int32_t* perm = (int32_t*)malloc(sizeof(int32_t) * (size_t)k_true * (size_t)V);
    if (!cdf || !perm) { free(cdf); free(perm); return -2; }
    double acc = 0.0;
    for (int32_t r = 0; r < V; ++r) { acc += pow((double)(r + 1), -zipf_s); cdf[r] = acc; }
    for (int32_t r = 0; r < V; ++r) cdf[r] /= acc;
    /* per-topic word order: ascending (log(rank + 1) + N(0, 1), word) -- a total
     * order, so any correct sort gives the product generator's permutation */
#pragma omp parallel
    {
        double* key = (double*)malloc(sizeof(double) * (size_t)V);
#pragma omp for schedule(dynamic, 1)
        for (int32_t k = 0; k < k_true; ++k) {
            int32_t* p = perm + (size_t)k * V;
            rng_t r = {key_of(seed, 2, (uint64_t)k), 0};
            for (int32_t w = 0; w < V; ++w) key[w] = log((double)w + 1.0) + rnormal(&r);
            for (int32_t w = 0; w < V; ++w) p[w] = w;
            qsort_r(p, (size_t)V, sizeof(int32_t), cmp_rank, key);
        }
        free(key);
    }
#pragma omp parallel
    {
        double* mix = (double*)malloc(sizeof(double) * (size_t)k_true);
#pragma omp for schedule(dynamic, 4096)
        for (int64_t i = 0; i < num_docs; ++i) {
            rng_t r = {key_of(seed, 3, (uint64_t)(doc_begin + i)), 0};
            double s = 0.0;
            for (int32_t k = 0; k < k_true; ++k) { mix[k] = rgamma(&r, doc_alpha); s += mix[k]; }
            double c = 0.0;
            for (int32_t k = 0; k < k_true; ++k) { c += mix[k] / s; mix[k] = c; }
            for (int64_t t = doc_ptr[i]; t < doc_ptr[i + 1]; ++t) {
                const double ut = ru(&r) * c;
                int64_t k = upper(mix, k_true, ut);
                if (k > k_true - 1) k = k_true - 1;
                int64_t rank = upper(cdf, V, ru(&r));
                if (rank > V - 1) rank = V - 1;
                doc_out[t] = (int32_t)(doc_begin + i);
                word_out[t] = perm[(size_t)k * V + rank];
            }
        }
        free(mix);
    }
    free(cdf);
    free(perm);
    return 0;
}
