// k_check.cu -- K5: the count-conservation check (model.py:180-225,
// SPEC.md:517) as device reductions, plus the device-side phi checks of the
// import / export paths (16-bit column overflow of set_phi, the phi argmax of
// the 16-bit width check, model.py:152-157).
//
// check_conservation's four invariants, in the reference's order:
//   1. theta row d sums to the document length L_d       (first bad d)
//   2. theta column k sums to the stored topic total n_k  (first bad k)
//   3. phi row k sums to n_k                               (first bad k)
//   4. sum_k n_k equals the corpus token count T
// Reductions (HBM-bound, one pass over theta and one over phi):
//   theta pass: one warp per document (grid-stride), row sums compared in the
//     warp, column sums in a per-CTA shared K-bin histogram flushed with u64
//     atomics (global atomics per entry when K does not fit);
//   phi pass, word-major shard layout: each thread owns topics
//     k = tid, tid + NT, ... and walks a range of word columns (coalesced K-vector
//     reads), accumulating in its own shared u64 slots -- no atomics until the
//     flush; reference K x V layout: one CTA per (topic, word range), a block
//     reduction per row;
//   final: one CTA compares and writes the report {code, index, a, b}.
// The report is turned into the reference's message text on the host
// (model.check_conservation); multi-rank callers allreduce the theta column
// sums between the two stages (engine.Trainer).
#include "gf_internal.cuh"
#include "gf_device.cuh"

#include <algorithm>

namespace gf {

// ---------------------------------------------------------- row access -----
struct ShardRows {                               // the shard's resident theta
    const uint2* meta;                           // {offset, nnz}
    const uint32_t* ent;                         // count << 16 | tpos << 2
    const uint32_t* dw_ptr;                      // doc-major token ranges: L_d
    TPos tm;
    __device__ uint32_t nnz(int64_t d) const { return meta[d].y; }
    __device__ uint32_t count(int64_t d, uint32_t j) const { return ent[meta[d].x + j] >> 16; }
    __device__ uint32_t topic(int64_t d, uint32_t j) const {
        return tpos_inv((ent[meta[d].x + j] & 0xffffu) >> 2, tm);
    }
    __device__ int64_t length(int64_t d) const { return (int64_t)dw_ptr[d + 1] - dw_ptr[d]; }
};

struct CsrRows {                                 // the reference ThetaRows (model.py:20-47)
    const int64_t* row_ptr;
    const uint16_t* ids;
    const uint16_t* cnt;
    const int64_t* doc_len;                      // corpus.doc_lengths
    __device__ uint32_t nnz(int64_t d) const { return (uint32_t)(row_ptr[d + 1] - row_ptr[d]); }
    __device__ uint32_t count(int64_t d, uint32_t j) const { return cnt[row_ptr[d] + j]; }
    __device__ uint32_t topic(int64_t d, uint32_t j) const { return ids[row_ptr[d] + j]; }
    __device__ int64_t length(int64_t d) const { return doc_len[d]; }
};

// K5 scratch (u64): [0, K) theta column sums | [K, 2K) phi row sums | 2K: first bad doc
template <class Rows>
__global__ void __launch_bounds__(256) k5_theta_kernel(Rows rows, int64_t D, int K, bool smem_hist,
                                                       unsigned long long* col, unsigned long long* bad_doc) {
    extern __shared__ uint32_t hist[];
    const int lane = threadIdx.x & 31;
    if (smem_hist) {
        for (int k = threadIdx.x; k < K; k += blockDim.x) hist[k] = 0u;
        __syncthreads();
    }
    const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t d = w0; d < D; d += nw) {
        const uint32_t n = rows.nnz(d);
        unsigned long long sum = 0;
        for (uint32_t j = lane; j < n; j += 32) {
            const uint32_t c = rows.count(d, j);
            const uint32_t k = rows.topic(d, j);
            sum += c;
            if (k < (uint32_t)K) {
                if (smem_hist) atomicAdd(hist + k, c);   // <= 2^32 per CTA: flushed below
                else atomicAdd(col + k, (unsigned long long)c);
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(kFull, sum, o);
        if (lane == 0 && (int64_t)sum != rows.length(d)) atomicMin(bad_doc, (unsigned long long)d);
    }
    if (smem_hist) {
        __syncthreads();
        for (int k = threadIdx.x; k < K; k += blockDim.x)
            if (hist[k]) atomicAdd(col + k, (unsigned long long)hist[k]);
    }
}

// The resident rows, one THREAD per document: a row starts on a 32-byte
// boundary and is zero-padded to whole 8-entry granules (K3 / theta import),
// so it is read as ceil(nnz / 8) pairs of 16-byte loads; the zero pads add
// nothing.  Column sums: shared K-bin histogram (per-CTA u32, flushed as u64).
__global__ void __launch_bounds__(256) k5_theta_shard_kernel(const uint2* __restrict__ meta,
                                                             const uint32_t* __restrict__ ent,
                                                             const uint32_t* __restrict__ dw_ptr, int64_t D, int K,
                                                             TPos tm, bool smem_hist, unsigned long long* col,
                                                             unsigned long long* bad_doc) {
    extern __shared__ uint32_t hist[];
    if (smem_hist) {
        for (int k = threadIdx.x; k < K; k += blockDim.x) hist[k] = 0u;
        __syncthreads();
    }
    for (int64_t d = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; d < D; d += (int64_t)gridDim.x * blockDim.x) {
        const uint2 m = meta[d];
        const uint4* row = reinterpret_cast<const uint4*>(ent + m.x);
        unsigned long long sum = 0;
        for (uint32_t g = 0; g < (m.y + 7u) >> 3; ++g) {
            const uint4 a = __ldg(row + 2 * g), b = __ldg(row + 2 * g + 1);
            const uint32_t e[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const uint32_t c = e[i] >> 16;
                if (c) {
                    sum += c;
                    const uint32_t k = tpos_inv((e[i] & 0xffffu) >> 2, tm);
                    if (k < (uint32_t)K) {
                        if (smem_hist) atomicAdd(hist + k, c);
                        else atomicAdd(col + k, (unsigned long long)c);
                    }
                }
            }
        }
        if ((int64_t)sum != (int64_t)(dw_ptr[d + 1] - dw_ptr[d])) atomicMin(bad_doc, (unsigned long long)d);
    }
    if (smem_hist) {
        __syncthreads();
        for (int k = threadIdx.x; k < K; k += blockDim.x)
            if (hist[k]) atomicAdd(col + k, (unsigned long long)hist[k]);
    }
}

// phi row sums, vectorised: every column is a contiguous K-vector starting on
// a 16-byte boundary; thread j of the CTA owns 16-byte slot j (+ SPT-1 more
// slots blockDim apart) of every column the CTA visits and sums it in u32
// registers (a topic's sum over any set of columns is <= n_k < 2^32), flushed
// once per CTA with u64 atomics.
template <typename T, int SPT>
__global__ void __launch_bounds__(256) k5_phi_vec_kernel(const uint4* __restrict__ cols, int64_t ncol, int slots,
                                                         int K, unsigned long long* row) {
    constexpr int E = 16 / sizeof(T);
    uint32_t acc[SPT][E];
#pragma unroll
    for (int s = 0; s < SPT; ++s)
#pragma unroll
        for (int e = 0; e < E; ++e) acc[s][e] = 0u;
    for (int64_t c = blockIdx.x; c < ncol; c += gridDim.x) {
        const uint4* p = cols + c * (int64_t)slots;
#pragma unroll
        for (int s = 0; s < SPT; ++s) {
            const int j = threadIdx.x + s * blockDim.x;
            if (j < slots) {
                const uint4 v = __ldg(p + j);
                const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    if (E == 8) {
                        acc[s][2 * q] += w[q] & 0xffffu;
                        acc[s][2 * q + 1] += w[q] >> 16;
                    } else {
                        acc[s][q] += w[q];
                    }
                }
            }
        }
    }
#pragma unroll
    for (int s = 0; s < SPT; ++s) {
        const int j = threadIdx.x + s * blockDim.x;
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const int k = j * E + e;
            if (j < slots && k < K && acc[s][e]) atomicAdd(row + k, (unsigned long long)acc[s][e]);
        }
    }
}

// phi row sums over the shard's word-major hybrid columns: heavy u32 columns
// (stride K) then light u16 columns (stride Kp); thread t owns topics t + i*NT
template <typename T>
__global__ void __launch_bounds__(256) k5_phi_cols_kernel(const T* cols, int64_t ncol, int stride, int K,
                                                          unsigned long long* row) {
    extern __shared__ unsigned long long acc[];
    for (int k = threadIdx.x; k < K; k += blockDim.x) acc[k] = 0ull;
    for (int64_t c = blockIdx.x; c < ncol; c += gridDim.x) {
        const T* p = cols + c * (int64_t)stride;
        for (int k = threadIdx.x; k < K; k += blockDim.x) acc[k] += p[k];
    }
    for (int k = threadIdx.x; k < K; k += blockDim.x)
        if (acc[k]) atomicAdd(row + k, acc[k]);
}

// phi row sums over the reference K x V row-major counts: CTA (k, slab)
template <typename T>
__global__ void __launch_bounds__(256) k5_phi_rows_kernel(const T* counts, int64_t V, int slabs,
                                                          unsigned long long* row) {
    __shared__ unsigned long long wsum[8];
    const int k = blockIdx.x / slabs, sl = blockIdx.x % slabs;
    const int64_t v0 = V * sl / slabs, v1 = V * (sl + 1) / slabs;
    const T* p = counts + (int64_t)k * V;
    unsigned long long s = 0;
    for (int64_t v = v0 + threadIdx.x; v < v1; v += blockDim.x) s += p[v];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(kFull, s, o);
    if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long t = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += wsum[w];
        if (t) atomicAdd(row + k, t);
    }
}

// report[0..3] = {code, index, a, b}; code 0 ok, 1 theta row (d, row sum, L_d),
// 2 theta column (k, column sum, n_k), 3 phi row (k, row sum, n_k), 4 total
// (sum n_k, T).  stage 1 checks the row invariant only (its first bad doc, as
// a global doc index), stage 2 the other three.
template <class Rows>
__global__ void k5_row_report_kernel(Rows rows, int64_t doc_lo, const unsigned long long* bad_doc, int64_t* report) {
    const unsigned long long d = *bad_doc;
    if (d == ~0ull) {
        if (threadIdx.x == 0) report[0] = report[1] = report[2] = report[3] = 0;
        return;
    }
    const uint32_t n = rows.nnz((int64_t)d);
    unsigned long long sum = 0;
    for (uint32_t j = threadIdx.x; j < n; j += 32) sum += rows.count((int64_t)d, j);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(kFull, sum, o);
    if (threadIdx.x == 0) {
        report[0] = 1;
        report[1] = doc_lo + (int64_t)d;
        report[2] = (int64_t)sum;
        report[3] = rows.length((int64_t)d);
    }
}

__global__ void k5_final_kernel(const unsigned long long* col, const unsigned long long* row, const uint32_t* nk32,
                                const int64_t* nk64, int K, int64_t T, int64_t* report) {
    __shared__ int first_col, first_row;
    __shared__ unsigned long long total;
    if (threadIdx.x == 0) { first_col = K; first_row = K; total = 0; }
    __syncthreads();
    unsigned long long mine = 0;
    for (int k = threadIdx.x; k < K; k += blockDim.x) {
        const int64_t nk = nk64 ? nk64[k] : (int64_t)nk32[k];
        mine += (unsigned long long)nk;
        if ((int64_t)col[k] != nk) atomicMin(&first_col, k);
        if ((int64_t)row[k] != nk) atomicMin(&first_row, k);
    }
    atomicAdd(&total, mine);
    __syncthreads();
    if (threadIdx.x) return;
    int64_t r[4] = {0, 0, 0, 0};
    if (first_col < K) {
        const int k = first_col;
        r[0] = 2; r[1] = k; r[2] = (int64_t)col[k]; r[3] = nk64 ? nk64[k] : (int64_t)nk32[k];
    } else if (first_row < K) {
        const int k = first_row;
        r[0] = 3; r[1] = k; r[2] = (int64_t)row[k]; r[3] = nk64 ? nk64[k] : (int64_t)nk32[k];
    } else if ((int64_t)total != T) {
        r[0] = 4; r[1] = 0; r[2] = (int64_t)total; r[3] = T;
    }
    for (int i = 0; i < 4; ++i) report[i] = r[i];
}

static int sm_count() {
    int dev = 0;
    cudaGetDevice(&dev);
    return sm_count(dev);
}

template <class Rows>
static cudaError_t theta_pass(const Rows& rows, int64_t D, int K, unsigned long long* col, unsigned long long* bad,
                              cudaStream_t st) {
    if (D == 0) return cudaSuccess;
    const bool smem_hist = (size_t)K * 4 <= 48 * 1024;
    const int64_t blocks = std::min<int64_t>((D + 7) / 8, 4LL * sm_count());
    k5_theta_kernel<Rows><<<(unsigned)blocks, 256, smem_hist ? (size_t)K * 4 : 0, st>>>(rows, D, K, smem_hist, col, bad);
    return cudaGetLastError();
}

template <typename T>
static cudaError_t phi_cols_pass(const T* cols, int64_t ncol, int stride, int K, unsigned long long* row,
                                 cudaStream_t st) {
    if (ncol == 0) return cudaSuccess;
    constexpr int E = 16 / sizeof(T);
    const int slots = (stride + E - 1) / E;
    const bool vec = stride % E == 0 && (reinterpret_cast<uintptr_t>(cols) & 15) == 0 && slots <= 8 * 256;
    if (vec) {
        const int nt = std::min(256, (slots + 31) / 32 * 32);
        const int spt = (slots + nt - 1) / nt;
        const int64_t blocks = std::min<int64_t>(ncol, 4LL * sm_count());
        const uint4* c4 = reinterpret_cast<const uint4*>(cols);
        if (spt == 1) k5_phi_vec_kernel<T, 1><<<(unsigned)blocks, nt, 0, st>>>(c4, ncol, slots, K, row);
        else if (spt == 2) k5_phi_vec_kernel<T, 2><<<(unsigned)blocks, nt, 0, st>>>(c4, ncol, slots, K, row);
        else if (spt <= 4) k5_phi_vec_kernel<T, 4><<<(unsigned)blocks, nt, 0, st>>>(c4, ncol, slots, K, row);
        else k5_phi_vec_kernel<T, 8><<<(unsigned)blocks, nt, 0, st>>>(c4, ncol, slots, K, row);
        return cudaGetLastError();
    }
    const size_t smem = (size_t)K * 8;
    static unsigned long long attr = 0;
    int dev = 0;
    cudaGetDevice(&dev);
    if (attr_once(attr, dev)) {
        cudaError_t e = cudaFuncSetAttribute(k5_phi_cols_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             200 * 1024);
        if (e != cudaSuccess) return e;
    }
    if (smem > 200 * 1024) return cudaErrorInvalidValue;   // K > 25600 (the shard caps K at 16384)
    const int64_t blocks = std::min<int64_t>(ncol, 2LL * sm_count());
    k5_phi_cols_kernel<T><<<(unsigned)blocks, 256, smem, st>>>(cols, ncol, stride, K, row);
    return cudaGetLastError();
}

// ------------------------------------------------------------- launchers ---
// The shard's K5 scratch is allocated on first use: u64[2K + 1].
cudaError_t launch_conservation_stage1(gf_shard* s, unsigned long long* scratch, int64_t* d_report) {
    const int K = s->K;
    unsigned long long* col = scratch;
    unsigned long long* row = scratch + K;
    unsigned long long* bad = scratch + 2 * K;
    cudaError_t e = cudaMemsetAsync(scratch, 0, sizeof(unsigned long long) * 2 * K, s->stream);
    if (e == cudaSuccess) e = cudaMemsetAsync(bad, 0xff, 8, s->stream);
    const ShardRows rows{s->d.theta_meta, s->d.theta_ent, s->d.dw_ptr, tpos_geom(K)};
    if (e == cudaSuccess && s->D > 0) {
        const bool smem_hist = (size_t)K * 4 <= 48 * 1024;
        const int64_t blocks = std::min<int64_t>((s->D + 255) / 256, 8LL * sm_count());
        k5_theta_shard_kernel<<<(unsigned)blocks, 256, smem_hist ? (size_t)K * 4 : 0, s->stream>>>(
            s->d.theta_meta, s->d.theta_ent, s->d.dw_ptr, s->D, K, tpos_geom(K), smem_hist, col, bad);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = phi_cols_pass(s->d.sync, s->n_heavy, K, K, row, s->stream);
    if (e == cudaSuccess)
        e = phi_cols_pass(reinterpret_cast<const uint16_t*>(s->d.sync + s->off_phi16_u32), s->n_light,
                          K + (K & 1), K, row, s->stream);
    if (e == cudaSuccess) {
        k5_row_report_kernel<ShardRows><<<1, 32, 0, s->stream>>>(rows, s->doc_lo, bad, d_report);
        e = cudaGetLastError();
    }
    return e;
}

cudaError_t launch_conservation_stage2(gf_shard* s, const unsigned long long* scratch, int64_t T, int64_t* d_report) {
    k5_final_kernel<<<1, 256, 0, s->stream>>>(scratch, scratch + s->K, s->d.sync + s->off_nk_u32, nullptr, s->K, T,
                                              d_report);
    return cudaGetLastError();
}

// the reference-layout check (model.check_conservation on exported arrays)
cudaError_t conservation_csr(int K, int64_t V, int64_t D, const int64_t* row_ptr, const uint16_t* ids,
                             const uint16_t* cnt, const int64_t* doc_len, const void* phi, int width,
                             const int64_t* totals, int64_t T, unsigned long long* scratch, int64_t* d_report,
                             cudaStream_t st) {
    unsigned long long* col = scratch;
    unsigned long long* row = scratch + K;
    unsigned long long* bad = scratch + 2 * K;
    cudaError_t e = cudaMemsetAsync(scratch, 0, sizeof(unsigned long long) * 2 * K, st);
    if (e == cudaSuccess) e = cudaMemsetAsync(bad, 0xff, 8, st);
    const CsrRows rows{row_ptr, ids, cnt, doc_len};
    if (e == cudaSuccess) e = theta_pass(rows, D, K, col, bad, st);
    if (e == cudaSuccess && V > 0) {
        const int slabs = (int)std::max<int64_t>(1, std::min<int64_t>(64, V / 4096));
        if (width == 16)
            k5_phi_rows_kernel<uint16_t><<<(unsigned)(K * slabs), 256, 0, st>>>((const uint16_t*)phi, V, slabs, row);
        else
            k5_phi_rows_kernel<uint32_t><<<(unsigned)(K * slabs), 256, 0, st>>>((const uint32_t*)phi, V, slabs, row);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) {
        k5_row_report_kernel<CsrRows><<<1, 32, 0, st>>>(rows, 0, bad, d_report);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) {
        k5_final_kernel<<<1, 256, 0, st>>>(col, row, nullptr, totals, K, T, d_report + 4);
        e = cudaGetLastError();
    }
    return e;
}

// ----------------------------------------------- phi import / argmax -------
// set_phi: first (word, topic) cell, word-major like the host scan it
// replaces, whose count exceeds its 16-bit column: key v * K + k (min)
__global__ void phi_u16_overflow_kernel(const uint32_t* __restrict__ kv, const int32_t* __restrict__ wcol, int K,
                                        int64_t V, unsigned long long* first) {
    const int64_t n = (int64_t)K * V;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t k = i / V, v = i - k * V;
        if (kv[i] > 65535u && wcol[v] >= 0) atomicMin(first, (unsigned long long)(v * K + k));
    }
}

// np.argmax over the K x V export: the maximum, then its first row-major index
__global__ void phi_max_kernel(const uint32_t* __restrict__ kv, int64_t n, unsigned int* mx) {
    uint32_t m = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        m = max(m, kv[i]);
    m = warp_max_u32(m);
    if ((threadIdx.x & 31) == 0 && m) atomicMax(mx, m);
}

__global__ void phi_first_kernel(const uint32_t* __restrict__ kv, int64_t n, const unsigned int* mx,
                                 unsigned long long* first) {
    const uint32_t m = *mx;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        if (kv[i] == m) {
            atomicMin(first, (unsigned long long)i);
            return;                               // later i of this thread are larger
        }
}

cudaError_t launch_phi_u16_overflow(const uint32_t* d_kv, const int32_t* d_wcol, int K, int64_t V,
                                    unsigned long long* d_first, cudaStream_t st) {
    cudaError_t e = cudaMemsetAsync(d_first, 0xff, 8, st);
    if (e != cudaSuccess) return e;
    phi_u16_overflow_kernel<<<8 * sm_count(), 256, 0, st>>>(d_kv, d_wcol, K, V, d_first);
    return cudaGetLastError();
}

cudaError_t launch_phi_argmax(const uint32_t* d_kv, int64_t n, unsigned int* d_max, unsigned long long* d_first,
                              cudaStream_t st) {
    cudaError_t e = cudaMemsetAsync(d_max, 0, 4, st);
    if (e == cudaSuccess) e = cudaMemsetAsync(d_first, 0xff, 8, st);
    if (e != cudaSuccess || n == 0) return e;
    phi_max_kernel<<<8 * sm_count(), 256, 0, st>>>(d_kv, n, d_max);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    phi_first_kernel<<<8 * sm_count(), 256, 0, st>>>(d_kv, n, d_max, d_first);
    return cudaGetLastError();
}

}  // namespace gf
