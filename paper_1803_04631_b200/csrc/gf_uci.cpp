// gf_uci.cpp -- native UCI bag-of-words loader:
// the reference's load_uci_bow / _read_bow_header (corpus.py:79-145) with the
// same validation order and error texts, on a hand-rolled integer scanner, and
// the corpus_from_tokens expansion (corpus.py:42-76: stable doc order, empty
// documents dropped) as a counting sort by document instead of an argsort.
#include "../../include/gibbsflow_b200.h"

#include <cerrno>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

namespace gf {
int shard_fail(int code, const char* fmt, ...);
}

namespace {

struct Line {
    const char* b;
    const char* e;
};

// splitlines(): \n, \r\n and \r end a line; a final unterminated line counts
bool read_lines(const char* path, std::string& buf, std::vector<Line>& lines) {
    FILE* f = std::fopen(path, "rb");
    if (!f) return false;
    std::fseek(f, 0, SEEK_END);
    const long n = std::ftell(f);
    std::fseek(f, 0, SEEK_SET);
    buf.resize(n > 0 ? (size_t)n : 0);
    if (n > 0 && std::fread(&buf[0], 1, (size_t)n, f) != (size_t)n) { std::fclose(f); return false; }
    std::fclose(f);
    const char* p = buf.data();
    const char* end = p + buf.size();
    const char* s = p;
    while (p < end) {
        if (*p == '\n' || *p == '\r') {
            lines.push_back({s, p});
            if (*p == '\r' && p + 1 < end && p[1] == '\n') ++p;
            s = ++p;
        } else {
            ++p;
        }
    }
    if (s < end) lines.push_back({s, end});
    return true;
}

inline bool is_space(char c) { return c == ' ' || c == '\t' || c == '\v' || c == '\f'; }

void strip(const char*& b, const char*& e) {
    while (b < e && is_space(*b)) ++b;
    while (e > b && is_space(e[-1])) --e;
}

// int(text): optional sign, decimal digits (the whole token)
bool parse_int(const char* b, const char* e, long long& v) {
    if (b >= e) return false;
    bool neg = false;
    if (*b == '+' || *b == '-') { neg = *b == '-'; ++b; }
    if (b >= e) return false;
    long long x = 0;
    for (; b < e; ++b) {
        if (*b < '0' || *b > '9') return false;
        x = x * 10 + (*b - '0');
    }
    v = neg ? -x : x;
    return true;
}

struct Header {
    long long D, W, NNZ;
};

int parse_header(const std::vector<Line>& lines, Header& h) {
    if (lines.size() < 3) return gf::shard_fail(GF_ERR_FORMAT, "docword header truncated: expected 3 lines");
    long long v[3];
    for (int i = 0; i < 3; ++i) {
        const char* b = lines[i].b;
        const char* e = lines[i].e;
        strip(b, e);
        if (!parse_int(b, e, v[i]))
            return gf::shard_fail(GF_ERR_FORMAT, "docword line %d: malformed header value '%.*s'", i + 1, (int)(e - b), b);
    }
    h = {v[0], v[1], v[2]};
    return GF_OK;
}

// body triples (validated like corpus.py:109-136)
int parse_body(const std::vector<Line>& lines, const Header& h, std::vector<int32_t>* d, std::vector<int32_t>* w,
               std::vector<int64_t>* c, int64_t* tokens) {
    long long nonempty = 0;
    for (size_t i = 3; i < lines.size(); ++i) {
        const char* b = lines[i].b;
        const char* e = lines[i].e;
        strip(b, e);
        nonempty += b < e;
    }
    if (nonempty != h.NNZ)
        return gf::shard_fail(GF_ERR_FORMAT, "docword body: expected %lld triples, found %lld", h.NNZ, nonempty);
    long long total = 0;
    for (size_t i = 3; i < lines.size(); ++i) {
        const char* b = lines[i].b;
        const char* e = lines[i].e;
        strip(b, e);
        if (b >= e) continue;
        const long long lineno = (long long)i + 1;
        const char* f[4];
        const char* fe[4];
        int nf = 0;
        const char* p = b;
        while (p < e) {
            while (p < e && is_space(*p)) ++p;
            if (p >= e) break;
            const char* s = p;
            while (p < e && !is_space(*p)) ++p;
            if (nf < 4) { f[nf] = s; fe[nf] = p; }
            ++nf;
        }
        if (nf != 3) return gf::shard_fail(GF_ERR_FORMAT, "docword line %lld: expected 3 fields", lineno);
        long long x[3];
        for (int k = 0; k < 3; ++k)
            if (!parse_int(f[k], fe[k], x[k]))
                return gf::shard_fail(GF_ERR_FORMAT, "docword line %lld: non-integer field", lineno);
        if (x[0] < 1 || x[0] > h.D)
            return gf::shard_fail(GF_ERR_FORMAT, "docword line %lld: docID %lld outside [1, %lld]", lineno, x[0], h.D);
        if (x[1] < 1 || x[1] > h.W)
            return gf::shard_fail(GF_ERR_FORMAT, "docword line %lld: wordID %lld outside [1, %lld]", lineno, x[1], h.W);
        if (x[2] <= 0) return gf::shard_fail(GF_ERR_FORMAT, "docword line %lld: count %lld must be > 0", lineno, x[2]);
        total += x[2];
        if (d) {
            d->push_back((int32_t)(x[0] - 1));
            w->push_back((int32_t)(x[1] - 1));
            c->push_back(x[2]);
        }
    }
    *tokens = total;
    return GF_OK;
}

}  // namespace

extern "C" {

int gf_uci_scan(const char* docword_path, int64_t* header, int64_t* num_tokens) {
    std::string buf;
    std::vector<Line> lines;
    if (!read_lines(docword_path, buf, lines))
        return gf::shard_fail(GF_ERR_FORMAT, "%s: cannot read docword file (%s)", docword_path, std::strerror(errno));
    Header h;
    if (int rc = parse_header(lines, h)) return rc;
    header[0] = h.D;
    header[1] = h.W;
    header[2] = h.NNZ;
    if (h.NNZ < 0) return gf::shard_fail(GF_ERR_VALUE, "negative dimensions are not allowed");
    if (h.D >= (1LL << 31) || h.W >= (1LL << 31))
        return gf::shard_fail(GF_ERR_CAPACITY, "docword header: more than 2^31 documents or words");
    return parse_body(lines, h, nullptr, nullptr, nullptr, num_tokens);
}

int gf_uci_tokens(const char* docword_path, int64_t num_tokens, int32_t* doc_ids, int32_t* word_ids,
                  int64_t* num_docs_out) {
    std::string buf;
    std::vector<Line> lines;
    if (!read_lines(docword_path, buf, lines))
        return gf::shard_fail(GF_ERR_FORMAT, "%s: cannot read docword file (%s)", docword_path, std::strerror(errno));
    Header h;
    if (int rc = parse_header(lines, h)) return rc;
    std::vector<int32_t> d, w;
    std::vector<int64_t> c;
    d.reserve((size_t)h.NNZ);
    w.reserve((size_t)h.NNZ);
    c.reserve((size_t)h.NNZ);
    int64_t total = 0;
    if (int rc = parse_body(lines, h, &d, &w, &c, &total)) return rc;
    if (total != num_tokens) return gf::shard_fail(GF_ERR_SHAPE, "token buffer has %lld entries, file has %lld",
                                                  (long long)num_tokens, (long long)total);
    // corpus_from_tokens: stable order by document (file order inside a doc),
    // empty documents dropped and ids compacted
    std::vector<int64_t> start((size_t)h.D + 1, 0);
    for (size_t i = 0; i < d.size(); ++i) start[(size_t)d[i] + 1] += c[i];
    std::vector<int32_t> newid((size_t)h.D, -1);
    int64_t kept = 0;
    for (int64_t k = 0; k < h.D; ++k)
        if (start[(size_t)k + 1] > 0) newid[(size_t)k] = (int32_t)kept++;
    for (int64_t k = 0; k < h.D; ++k) start[(size_t)k + 1] += start[(size_t)k];
    for (size_t i = 0; i < d.size(); ++i) {
        int64_t p = start[(size_t)d[i]];
        for (int64_t r = 0; r < c[i]; ++r, ++p) {
            doc_ids[p] = newid[(size_t)d[i]];
            word_ids[p] = w[i];
        }
        start[(size_t)d[i]] = p;
    }
    *num_docs_out = kept;
    return GF_OK;
}

}  // extern "C"
