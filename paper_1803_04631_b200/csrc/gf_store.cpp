// gf_store.cpp -- the GFSNAP1 model snapshot (model.py:228-296)
// as a native streaming writer / reader.  The file is the concatenation of
// fixed-width little-endian sections; the writer emits each section straight
// from the caller's (exported) arrays with one fwrite per section, the reader
// sizes everything from the 47-byte header and fills the caller's arrays with
// one fread per section -- no intermediate copies of the K x V phi block.
//
//   offset 0   "GFSNAP1"                       7 bytes
//          7   K, V, D, NNZ, phi_width          5 x u64
//         47   phi counts, K x V row-major       u16 or u32 (phi_width)
//              topic totals                      K x u64
//              theta row_ptr                     (D + 1) x u64
//              theta topic ids, counts           NNZ x u16 each
//              metadata length, metadata JSON    u64 + bytes (utf-8)
#include "../../include/gibbsflow_b200.h"

#include <cstdio>
#include <cstring>
#include <memory>
#include <vector>

namespace gf {
int shard_fail(int code, const char* fmt, ...);
}

namespace {

constexpr char kMagic[7] = {'G', 'F', 'S', 'N', 'A', 'P', '1'};
constexpr size_t kHeader = 7 + 5 * 8;

struct File {
    FILE* f = nullptr;
    ~File() {
        if (f) std::fclose(f);
    }
};

static_assert(sizeof(uint64_t) == 8 && sizeof(uint16_t) == 2, "fixed-width sections");

bool little_endian() {
    const uint16_t one = 1;
    uint8_t b;
    std::memcpy(&b, &one, 1);
    return b == 1;
}

}  // namespace

extern "C" {

int gf_snapshot_write(const char* path, int64_t K, int64_t V, int64_t D, int64_t nnz, int32_t phi_width,
                      const void* phi_counts, const int64_t* topic_totals, const int64_t* row_ptr,
                      const uint16_t* topic_ids, const uint16_t* counts, const char* meta, int64_t meta_len) {
    if (!little_endian()) return gf::shard_fail(GF_ERR_VALUE, "GFSNAP1 writer needs a little-endian host");
    if (phi_width != 16 && phi_width != 32)
        return gf::shard_fail(GF_ERR_VALUE, "phi width must be 16 or 32, got %d", phi_width);
    if (K < 0 || V < 0 || D < 0 || nnz < 0 || meta_len < 0)
        return gf::shard_fail(GF_ERR_VALUE, "negative snapshot dimension");
    File out;
    out.f = std::fopen(path, "wb");
    if (!out.f) return gf::shard_fail(GF_ERR_VALUE, "%s: cannot open for writing", path);
    const uint64_t hdr[5] = {(uint64_t)K, (uint64_t)V, (uint64_t)D, (uint64_t)nnz, (uint64_t)phi_width};
    const uint64_t mlen = (uint64_t)meta_len;
    // int64 sections are written as u64: same bytes for the non-negative values
    // the model holds (two's complement, little-endian)
    const struct {
        const void* p;
        size_t bytes;
    } sections[] = {
        {kMagic, sizeof kMagic},
        {hdr, sizeof hdr},
        {phi_counts, (size_t)K * (size_t)V * (size_t)(phi_width / 8)},
        {topic_totals, (size_t)K * 8},
        {row_ptr, (size_t)(D + 1) * 8},
        {topic_ids, (size_t)nnz * 2},
        {counts, (size_t)nnz * 2},
        {&mlen, 8},
        {meta, (size_t)meta_len},
    };
    for (const auto& s : sections)
        if (s.bytes && std::fwrite(s.p, 1, s.bytes, out.f) != s.bytes)
            return gf::shard_fail(GF_ERR_VALUE, "%s: write failed", path);
    if (std::fflush(out.f) != 0) return gf::shard_fail(GF_ERR_VALUE, "%s: write failed", path);
    return GF_OK;
}

// hdr_out = {K, V, D, NNZ, phi_width, metadata length}
int gf_snapshot_header(const char* path, int64_t* hdr_out) {
    File in;
    in.f = std::fopen(path, "rb");
    if (!in.f) return gf::shard_fail(GF_ERR_VALUE, "%s: cannot open", path);
    char magic[7] = {0};
    if (std::fread(magic, 1, 7, in.f) != 7 || std::memcmp(magic, kMagic, 7) != 0)
        return gf::shard_fail(GF_ERR_FORMAT, "%s: bad snapshot magic", path);
    uint64_t h[5];
    if (std::fread(h, 8, 5, in.f) != 5) return gf::shard_fail(GF_ERR_VALUE, "%s: truncated snapshot header", path);
    if (h[4] != 16 && h[4] != 32)
        return gf::shard_fail(GF_ERR_FORMAT, "%s: unsupported phi width %llu", path, (unsigned long long)h[4]);
    const uint64_t body = h[0] * h[1] * (h[4] / 8) + 8 * h[0] + 8 * (h[2] + 1) + 4 * h[3];
    if (std::fseek(in.f, (long)(kHeader + body), SEEK_SET) != 0)
        return gf::shard_fail(GF_ERR_VALUE, "%s: truncated snapshot", path);
    uint64_t mlen = 0;
    if (std::fread(&mlen, 8, 1, in.f) != 1) return gf::shard_fail(GF_ERR_VALUE, "%s: truncated snapshot", path);
    for (int i = 0; i < 5; ++i) hdr_out[i] = (int64_t)h[i];
    hdr_out[5] = (int64_t)mlen;
    return GF_OK;
}

int gf_snapshot_read(const char* path, void* phi_counts, int64_t* topic_totals, int64_t* row_ptr,
                     uint16_t* topic_ids, uint16_t* counts, char* meta) {
    int64_t h[6];
    if (int rc = gf_snapshot_header(path, h)) return rc;
    File in;
    in.f = std::fopen(path, "rb");
    if (!in.f || std::fseek(in.f, (long)kHeader, SEEK_SET) != 0)
        return gf::shard_fail(GF_ERR_VALUE, "%s: cannot open", path);
    const size_t K = (size_t)h[0], V = (size_t)h[1], D = (size_t)h[2], nnz = (size_t)h[3], w = (size_t)h[4] / 8;
    uint64_t mlen = 0;
    const struct {
        void* p;
        size_t bytes;
    } sections[] = {
        {phi_counts, K * V * w}, {topic_totals, K * 8}, {row_ptr, (D + 1) * 8}, {topic_ids, nnz * 2},
        {counts, nnz * 2},       {&mlen, 8},            {meta, (size_t)h[5]},
    };
    for (const auto& s : sections)
        if (s.bytes && std::fread(s.p, 1, s.bytes, in.f) != s.bytes)
            return gf::shard_fail(GF_ERR_VALUE, "%s: truncated snapshot", path);
    return GF_OK;
}

}  // extern "C"
