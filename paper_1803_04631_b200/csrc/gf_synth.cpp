// gf_synth.cpp -- seeded LDA-generative synthetic corpora for tests and the
// benchmark (SURVEY.md section 8d "Synthetic inputs"; there is no network for
// NYTimes / PubMed).  K_true topics, each a Zipf(s) law over its own jittered
// ordering of the vocabulary; per-document mixtures Dir(doc_alpha); log-normal
// document lengths with the requested mean.  Every document draws from its own
// splitmix64 stream keyed by (seed, doc), so a corpus (or one shard of it) is
// reproducible on any thread count and any rank.
#include "../../include/gibbsflow_b200.h"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>
#include <thread>
#include <vector>

namespace {

inline uint64_t fin(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

struct Rng {  // splitmix64 counter stream (the rng.py construction)
    uint64_t key, ctr = 0;
    explicit Rng(uint64_t k) : key(k) {}
    double u() { return (double)(fin(key + 0x9E3779B97F4A7C15ULL * (++ctr)) >> 11) * (1.0 / 9007199254740992.0); }
    double normal() {
        double a = u(), b = u();
        if (a < 1e-300) a = 1e-300;
        return std::sqrt(-2.0 * std::log(a)) * std::cos(6.283185307179586 * b);
    }
    double gamma(double k) {  // Marsaglia-Tsang, boost for k < 1
        if (k < 1.0) {
            double g = gamma(k + 1.0), x = u();
            if (x < 1e-300) x = 1e-300;
            return g * std::pow(x, 1.0 / k);
        }
        const double d = k - 1.0 / 3.0, c = 1.0 / std::sqrt(9.0 * d);
        while (true) {
            double x = normal(), v = 1.0 + c * x;
            if (v <= 0) continue;
            v = v * v * v;
            double uu = u();
            if (uu < 1 - 0.0331 * x * x * x * x) return d * v;
            if (std::log(std::max(uu, 1e-300)) < 0.5 * x * x + d * (1 - v + std::log(v))) return d * v;
        }
    }
};

uint64_t key_of(uint64_t seed, uint64_t a, uint64_t b) {
    uint64_t h = 0x9E3779B97F4A7C15ULL;
    const uint64_t parts[3] = {seed, a, b};
    for (uint64_t p : parts) h = fin(h + 0x9E3779B97F4A7C15ULL + p);
    return h;
}

template <class F>
void par(int64_t n, F f, int64_t min_parallel = 4096) {
    unsigned nt = std::max(1u, std::min(std::thread::hardware_concurrency(), 32u));
    if (n < min_parallel) nt = 1;
    nt = (unsigned)std::max<int64_t>(1, std::min<int64_t>(nt, n));
    std::vector<std::thread> th;
    for (unsigned i = 0; i < nt; ++i) th.emplace_back([=] { f(n * i / nt, n * (i + 1) / nt); });
    for (auto& t : th) t.join();
}

}  // namespace

extern "C" {

int gf_synth_lengths(uint64_t seed, int64_t doc_begin, int64_t num_docs, double mean_len, double sigma,
                     int64_t* lengths_out) {
    if (num_docs < 0 || !(mean_len >= 1.0) || !(sigma >= 0.0)) return GF_ERR_VALUE;
    const double mu = std::log(mean_len) - 0.5 * sigma * sigma;
    par(num_docs, [&](int64_t a, int64_t b) {
        for (int64_t i = a; i < b; ++i) {
            Rng r(key_of(seed, 1, (uint64_t)(doc_begin + i)));
            lengths_out[i] = std::max<int64_t>(1, (int64_t)std::llround(std::exp(mu + sigma * r.normal())));
        }
    });
    return GF_OK;
}

int gf_synth_tokens(uint64_t seed, int64_t doc_begin, int64_t num_docs, const int64_t* doc_ptr, int32_t V,
                    int32_t k_true, double zipf_s, double doc_alpha, int32_t* doc_ids_out, int32_t* word_ids_out) {
    if (V < 1 || k_true < 1 || num_docs < 0) return GF_ERR_VALUE;
    // topic-word laws: Zipf over a per-topic permutation (inverse CDF by binary search)
    std::vector<double> cdf((size_t)V);
    double acc = 0.0;
    for (int32_t r = 0; r < V; ++r) { acc += std::pow((double)(r + 1), -zipf_s); cdf[r] = acc; }
    for (auto& c : cdf) c /= acc;
    // per-topic rank order: log-rank jittered by N(0, 1) so every topic keeps a
    // Zipfian head (the corpus-wide law stays heavy-tailed, like NYTimes /
    // PubMed) while the topics disagree on which words lead
    std::vector<int32_t> perm((size_t)k_true * V);
    // (one topic per task: the orders are independent)
    par(k_true, [&](int64_t a, int64_t b) {
        std::vector<double> key((size_t)V);
        for (int64_t k = a; k < b; ++k) {
            int32_t* p = perm.data() + (size_t)k * V;
            Rng r(key_of(seed, 2, (uint64_t)k));
            for (int32_t w = 0; w < V; ++w) key[w] = std::log((double)w + 1.0) + r.normal();
            std::iota(p, p + V, 0);
            std::sort(p, p + V, [&](int32_t x, int32_t y) { return key[x] < key[y] || (key[x] == key[y] && x < y); });
        }
    }, 2);
    par(num_docs, [&](int64_t a, int64_t b) {
        std::vector<double> mix((size_t)k_true);
        for (int64_t i = a; i < b; ++i) {
            Rng r(key_of(seed, 3, (uint64_t)(doc_begin + i)));
            double s = 0.0;
            for (int32_t k = 0; k < k_true; ++k) { mix[k] = r.gamma(doc_alpha); s += mix[k]; }
            double c = 0.0;
            for (int32_t k = 0; k < k_true; ++k) { c += mix[k] / s; mix[k] = c; }
            for (int64_t t = doc_ptr[i]; t < doc_ptr[i + 1]; ++t) {
                const double ut = r.u() * c;
                const int32_t k = (int32_t)std::min<int64_t>(std::upper_bound(mix.begin(), mix.end(), ut) - mix.begin(),
                                                             k_true - 1);
                const int32_t rank = (int32_t)std::min<int64_t>(
                    std::upper_bound(cdf.begin(), cdf.end(), r.u()) - cdf.begin(), V - 1);
                doc_ids_out[t] = (int32_t)(doc_begin + i);
                word_ids_out[t] = perm[(size_t)k * V + rank];
            }
        }
    });
    return GF_OK;
}

}  // extern "C"
