// k_counts.cu -- count maintenance kernels (section 6.2):
//   K2 phi_rebuild   model.py:142-161  rebuild_phi_replica (+ n_k)
//   K3 theta_rebuild model.py:91-124   rebuild_theta_row / rebuild_theta
//   prepare          Eq. 1 denominators 1/(n_k + V b)
//   ll_reduce        deterministic fp64 reduction of the sampler's partials
//   theta / phi export + import (the reference dataclass layouts)
//   ptree primitive  ptree.py:116-151 (build levels + ballot descent)
#include "gf_internal.cuh"
#include "gf_device.cuh"

namespace gf {

// ---------------------------------------------------------------- K2 ------
// Work items are (phi column, token range): one item per light word (the
// whole group, <= heavy_threshold tokens so its 16-bit cells cannot
// overflow), one item per slice of a heavy word (32-bit cells, global
// atomics).  Each CTA histograms an item's topics in shared memory (tokens
// are word-grouped, so the item is one contiguous z range) and writes only
// the nonzero cells into the pre-zeroed sync buffer; n_k is accumulated per
// CTA in shared memory and flushed with K atomics at the end.
// Items of <= 32 tokens (the rare words of a large vocabulary) go to single
// warps instead: one topic per lane, __match_any_sync groups equal topics and
// the group leader writes the cell -- no shared histogram, no block barriers.
// The layout puts the CTA items first ([0, n_big)) and the warp items after.
__global__ void __launch_bounds__(256) phi_rebuild_kernel(const int4* __restrict__ items, int n_items, int n_big,
                                                          const uint16_t* __restrict__ z, uint32_t* sync,
                                                          int K, int Kp, long long off16, long long offnk,
                                                          unsigned long long* errs) {
    extern __shared__ uint32_t sh[];
    uint32_t* bins = sh;
    uint32_t* nks = sh + K;
    for (int k = threadIdx.x; k < 2 * K; k += blockDim.x) sh[k] = 0;
    __syncthreads();
    uint16_t* phi16 = reinterpret_cast<uint16_t*>(sync + off16);
    for (int it = blockIdx.x; it < n_big; it += gridDim.x) {
        const int4 w = items[it];
        const int col = w.x, t0 = w.y, t1 = w.z;
        const bool atomic = w.w != 0;
        // 16-byte loads (8 topics per thread) over the 8-aligned body, scalar head/tail
        auto count = [&](int t, int k) {
            if (k < K) atomicAdd(&bins[k], 1u);
            else atomicMin(errs, (unsigned long long)t);
        };
        const int a0 = min(t1, (t0 + 7) & ~7), a1 = max(a0, t1 & ~7);
        for (int t = t0 + threadIdx.x; t < a0; t += blockDim.x) count(t, z[t]);
        for (int t = a1 + threadIdx.x; t < t1; t += blockDim.x) count(t, z[t]);
        const uint4* zv = reinterpret_cast<const uint4*>(z);
        for (int q = (a0 >> 3) + threadIdx.x; q < (a1 >> 3); q += blockDim.x) {
            const uint4 v = __ldg(zv + q);
            const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                count(8 * q + 2 * i, (int)(w[i] & 0xffffu));
                count(8 * q + 2 * i + 1, (int)(w[i] >> 16));
            }
        }
        __syncthreads();
        if ((long long)(t1 - t0) * 8 >= K) {
            for (int k = threadIdx.x; k < K; k += blockDim.x) {
                const uint32_t c = bins[k];
                if (c) {
                    bins[k] = 0;
                    nks[k] += c;
                    if (col >= 0) phi16[(size_t)col * Kp + k] = (uint16_t)c;
                    else if (atomic) atomicAdd(&sync[(size_t)(~col) * K + k], c);
                    else sync[(size_t)(~col) * K + k] = c;
                }
            }
        } else {
            for (int t = t0 + threadIdx.x; t < t1; t += blockDim.x) {
                const int k = z[t];
                if (k >= K) continue;
                const uint32_t c = atomicExch(&bins[k], 0u);
                if (c) {
                    atomicAdd(&nks[k], c);
                    if (col >= 0) phi16[(size_t)col * Kp + k] = (uint16_t)c;
                    else if (atomic) atomicAdd(&sync[(size_t)(~col) * K + k], c);
                    else sync[(size_t)(~col) * K + k] = c;
                }
            }
        }
        __syncthreads();
    }
    // ---- warp items ----
    const int lane = threadIdx.x & 31;
    const int nw = (int)(blockDim.x >> 5);
    for (int it = n_big + blockIdx.x * nw + (int)(threadIdx.x >> 5); it < n_items; it += gridDim.x * nw) {
        const int4 w = items[it];
        const int col = w.x, t = w.y + lane;
        bool valid = t < w.z;
        const uint32_t k = valid ? (uint32_t)z[t] : 0xFFFFFFFFu;
        if (valid && k >= (uint32_t)K) {
            atomicMin(errs, (unsigned long long)t);
            valid = false;
        }
        const unsigned grp = __match_any_sync(kFull, valid ? k : 0xFFFFFFFFu);
        if (valid && lane == __ffs(grp) - 1) {
            const uint32_t c = (uint32_t)__popc(grp);
            atomicAdd(&nks[k], c);
            if (col >= 0) phi16[(size_t)col * Kp + k] = (uint16_t)c;
            else if (w.w != 0) atomicAdd(&sync[(size_t)(~col) * K + k], c);
            else sync[(size_t)(~col) * K + k] = c;
        }
    }
    __syncthreads();
    uint32_t* nk = sync + offnk;
    for (int k = threadIdx.x; k < K; k += blockDim.x)
        if (nks[k]) atomicAdd(&nk[k], nks[k]);
}

cudaError_t launch_phi_rebuild(gf_shard* s) {
    s->ctx_dirty = true;
    cudaError_t e = cudaMemsetAsync(s->d.sync, 0, (size_t)s->sync_u32 * 4, s->stream);
    if (e != cudaSuccess || s->n_k2 == 0) return e;
    int nsm = 148;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, s->device);
    const size_t smem = (size_t)2 * s->K * sizeof(uint32_t);
    static unsigned long long attr = 0;
    if (attr_once(attr, s->device)) {
        e = cudaFuncSetAttribute(phi_rebuild_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        if (e != cudaSuccess) return e;
    }
    const int per_sm = smem <= 16 * 1024 ? 8 : (smem <= 48 * 1024 ? 4 : 1);
    const long long grid = std::min<long long>(std::max<long long>(s->n_k2_big, (s->n_k2 - s->n_k2_big + 7) / 8),
                                               (long long)nsm * per_sm);
    phi_rebuild_kernel<<<(unsigned)grid, 256, smem, s->stream>>>(s->d.k2items, (int)s->n_k2, (int)s->n_k2_big, s->d.z,
                                                                  s->d.sync, s->K, s->Kp, s->off_phi16_u32,
                                                                  s->off_nk_u32, s->d.errs);
    return cudaGetLastError();
}

// ------------------------------------------------------------- prepare ------
// inv_den[k] = 1/(n_k + V b) and inv_den[K + k] = 1/(n_k - 1 + V b) (the
// exclusion view), once per iteration instead of a division per word and topic
__global__ void prepare_kernel(const uint32_t* __restrict__ nk, float* inv_den, int K, double vbeta) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k < K) {
        inv_den[k] = (float)(1.0 / ((double)nk[k] + vbeta));
        inv_den[K + k] = nk[k] ? (float)(1.0 / ((double)nk[k] - 1.0 + vbeta)) : 0.f;
    }
}

cudaError_t launch_prepare(gf_shard* s) {
    prepare_kernel<<<(s->K + 255) / 256, 256, 0, s->stream>>>(s->d.sync + s->off_nk_u32, s->d.inv_den, s->K,
                                                              (double)s->V * s->beta);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    return launch_contexts(s);                // word contexts of the multi-slice words
}

// ---------------------------------------------------------------- K3 ------
// One warp per document.  Short documents (<= 32 tokens): the topics are
// gathered through the doc-word map into one register per lane, bitonic-sorted
// across the warp and run-length encoded with ballots (no K-sized state).
// Longer documents: K-bin histogram plus a K-bit presence bitmap in the warp's
// shared-memory slice (section 6.2 "generate a dense array ... then
// CSR"); the output rank of topic k is popc of the bitmap below k (one warp
// scan over the K/32 bitmap words), so each lane emits the topics of its
// bitmap word in ascending order and clears exactly the bins it touched --
// O(L + K/32) per document instead of O(K).  Bins and bitmap are zeroed once
// per CTA and kept zero between documents.  Output rows: (count << 16 |
// topic << 2) (the topic pre-scaled to a byte offset into K1's shared p*
// table), ascending topic, in the fixed-capacity row; nnz into meta.y.
__host__ __device__ inline int k3_words(int K) { return (K + 31) >> 5; }
__host__ __device__ inline int k3_warp_u32(int K) { return K + 2 * k3_words(K); }   // bins | bitmap | word ranks

__global__ void __launch_bounds__(256, 5) theta_rebuild_kernel(int D, const uint32_t* __restrict__ dw_ptr,
                                                            const uint16_t* __restrict__ zdoc, uint32_t* theta_ent,
                                                            uint2* theta_meta, int K, int warps_per_cta,
                                                            unsigned long long* errs) {
    extern __shared__ uint32_t sh[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int NW = k3_words(K);
    const TPos tm = tpos_geom(K);
    uint32_t* bins = sh + (size_t)warp * k3_warp_u32(K);
    uint32_t* bmp = bins + K;
    uint32_t* wpre = bmp + NW;                     // distinct topics below each bitmap word
    for (int i = lane; i < K + NW; i += 32) bins[i] = 0u;
    __syncwarp();
    const unsigned lt = (1u << lane) - 1u;
    // software pipeline over this warp's documents d, d+s, d+2s: the next
    // document's first 32 topics and the one after's (dw_ptr, meta) are in
    // flight while the current one is counted
    const int s = gridDim.x * warps_per_cta;
    auto meta_of = [&](int dd, uint32_t& mb, uint32_t& mL, uint32_t& mo) {
        mb = mL = mo = 0u;
        if (dd < D) { mb = dw_ptr[dd]; mL = dw_ptr[dd + 1] - mb; mo = theta_meta[dd].x; }
    };
    int d = blockIdx.x * warps_per_cta + warp;
    uint32_t b, L, off, b1, L1, o1;
    meta_of(d, b, L, off);
    meta_of(d + s, b1, L1, o1);
    uint32_t zf = (d < D && (uint32_t)lane < L) ? zdoc[b + lane] : 0xffffu;   // first 32 topics of d
    for (; d < D; d += s) {
        uint32_t b2, L2, o2;
        meta_of(d + 2 * s, b2, L2, o2);
        const uint32_t zn = (d + s < D && (uint32_t)lane < L1) ? zdoc[b1 + lane] : 0xffffu;
        uint32_t nnz;
        if (L <= 32) {
            uint32_t key = 0xffffu;
            if (lane < (int)L) key = zf;
            if (key >= (uint32_t)K && lane < (int)L) { atomicMin(errs + 2, (unsigned long long)d); key = 0xffffu; }
            key = warp_bitonic_sort(key, lane);
            const uint32_t prev = __shfl_up_sync(kFull, key, 1);
            const bool head = key != 0xffffu && (lane == 0 || key != prev);
            const unsigned heads = __ballot_sync(kFull, head);
            if (head) {
                const unsigned later = heads & ~((2u << lane) - 1u);
                const uint32_t next = later ? (uint32_t)(__ffs(later) - 1) : L;
                theta_ent[off + __popc(heads & lt)] = (tpos(key, tm) << 2) | ((next - lane) << 16);
            }
            nnz = __popc(heads);
        } else if (L <= 128) {
            // token-parallel emit (32 < L <= 128, the tokens stay in registers):
            // the first occurrence of each topic (atomicAdd returned 0) writes
            // its entry at its rank = distinct topics below it (word prefix +
            // popc inside the word) -- no per-bitmap-word loop, no divergence
            const uint32_t i1 = lane + 32u, i2 = lane + 64u, i3 = lane + 96u;
            const uint32_t kk[4] = {zf, i1 < L ? zdoc[b + i1] : 0xffffu, i2 < L ? zdoc[b + i2] : 0xffffu,
                                    i3 < L ? zdoc[b + i3] : 0xffffu};
            bool fst[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const uint32_t k = kk[j];
                fst[j] = false;
                if (k < (uint32_t)K) {
                    fst[j] = atomicAdd(&bins[k], 1u) == 0u;
                    if (fst[j]) atomicOr(&bmp[k >> 5], 1u << (k & 31u));
                } else if ((uint32_t)lane + 32u * j < L) {
                    atomicMin(errs + 2, (unsigned long long)d);
                }
            }
            __syncwarp();
            uint32_t base = 0;
            for (int c = 0; c < NW; c += 32) {
                const int w = c + lane;
                const uint32_t pc = w < NW ? __popc(bmp[w]) : 0u;
                uint32_t incl = pc;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t y = __shfl_up_sync(kFull, incl, o);
                    if (lane >= o) incl += y;
                }
                if (w < NW) wpre[w] = base + incl - pc;
                base += __shfl_sync(kFull, incl, 31);
            }
            nnz = base;
            __syncwarp();
#pragma unroll
            for (int j = 0; j < 4; ++j)
                if (fst[j]) {
                    const uint32_t k = kk[j], w = k >> 5;
                    const uint32_t r = wpre[w] + __popc(bmp[w] & ((1u << (k & 31u)) - 1u));
                    theta_ent[off + r] = (tpos(k, tm) << 2) | (bins[k] << 16);    // <= 128: no overflow
                }
            __syncwarp();
#pragma unroll
            for (int j = 0; j < 4; ++j)
                if (fst[j]) { bins[kk[j]] = 0u; bmp[kk[j] >> 5] = 0u; }
            __syncwarp();
        } else {
            auto count = [&](uint32_t k) {
                if (k < (uint32_t)K) {
                    atomicAdd(&bins[k], 1u);
                    atomicOr(&bmp[k >> 5], 1u << (k & 31u));
                } else {
                    atomicMin(errs + 2, (unsigned long long)d);
                }
            };
            // the next 96 topics load together (independent), then count
            const uint32_t i1 = lane + 32u, i2 = lane + 64u, i3 = lane + 96u;
            const uint32_t k1 = i1 < L ? zdoc[b + i1] : 0u, k2 = i2 < L ? zdoc[b + i2] : 0u,
                           k3 = i3 < L ? zdoc[b + i3] : 0u;
            count(zf);                                          // L > 32: every lane has one
            if (i1 < L) count(k1);
            if (i2 < L) count(k2);
            if (i3 < L) count(k3);
            for (uint32_t i = lane + 128u; i < L; i += 32) count(zdoc[b + i]);
            __syncwarp();
            uint32_t base = 0, mx = 0;
            for (int c = 0; c < NW; c += 32) {
                const int w = c + lane;
                uint32_t word = w < NW ? bmp[w] : 0u;
                const uint32_t pc = __popc(word);
                uint32_t incl = pc;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t y = __shfl_up_sync(kFull, incl, o);
                    if (lane >= o) incl += y;
                }
                uint32_t pos = off + base + incl - pc;
                if (w < NW) bmp[w] = 0u;
                while (word) {
                    const uint32_t k = ((uint32_t)w << 5) + (uint32_t)(__ffs(word) - 1);
                    word &= word - 1u;
                    const uint32_t v = bins[k];
                    bins[k] = 0u;
                    theta_ent[pos++] = (tpos(k, tm) << 2) | (min(v, 65535u) << 16);
                    mx = max(mx, v);
                }
                base += __shfl_sync(kFull, incl, 31);
            }
            nnz = base;
            mx = warp_max_u32(mx);
            if (mx > 65535u && lane == 0) atomicMin(errs + 1, ((unsigned long long)d << 32) | mx);
            __syncwarp();
        }
        // zero the row's padding up to a multiple of 8 entries: K1 reads rows
        // as 32-byte granules and relies on (count 0) pads contributing nothing
        if ((uint32_t)lane < ((8u - (nnz & 7u)) & 7u)) theta_ent[off + nnz + lane] = 0u;
        if (lane == 0) theta_meta[d].y = nnz;
        b = b1; L = L1; off = o1;
        b1 = b2; L1 = L2; o1 = o2;
        zf = zn;
    }
}

cudaError_t launch_theta_rebuild(gf_shard* s, cudaStream_t st) {
    if (s->D == 0) return cudaSuccess;
    if (!st) st = s->stream;
    const size_t per_warp = (size_t)k3_warp_u32(s->K) * 4;
    int wpc = 8;
    while (wpc > 1 && (size_t)wpc * per_warp > 96 * 1024) wpc >>= 1;
    const size_t smem = (size_t)wpc * per_warp;
    static unsigned long long attr = 0;
    if (attr_once(attr, s->device)) {
        cudaError_t e = cudaFuncSetAttribute(theta_rebuild_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             200 * 1024);
        if (e != cudaSuccess) return e;
    }
    // persistent grid (exactly the resident CTAs): the warps sweep the
    // documents as one contiguous moving window, so the word-major z sectors
    // they gather are shared by neighbouring documents while still in L2
    int nsm = 148, per_sm = 1;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, s->device);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, theta_rebuild_kernel, wpc * 32, smem);
    const long long need = (s->D + wpc - 1) / wpc;
    const long long grid = std::min<long long>(need, (long long)nsm * std::max(per_sm, 1));
    theta_rebuild_kernel<<<(unsigned)grid, wpc * 32, smem, st>>>((int)s->D, s->d.dw_ptr, s->d.zdoc,
                                                                         s->d.theta_ent, s->d.theta_meta, s->K, wpc,
                                                                         s->d.errs);
    return cudaGetLastError();
}

// ------------------------------------------------------------ zdoc sync ------
// zdoc[run_dwpos[r] + i] = z[run_start[r] + i]: the doc-major copy of imported
// or initial assignments (K1 keeps it current afterwards)
__global__ void zdoc_sync_kernel(long long R, const uint32_t* __restrict__ run_start,
                                 const uint32_t* __restrict__ dwpos, const uint16_t* __restrict__ z, uint16_t* zdoc) {
    for (long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x; r < R; r += (long long)gridDim.x * blockDim.x) {
        const uint32_t t0 = run_start[r], t1 = run_start[r + 1], p = dwpos[r];
        for (uint32_t t = t0; t < t1; ++t) zdoc[p + (t - t0)] = z[t];
    }
}

// Staged import (gf_shard_copy_assignments_async to the device + _imported):
// per run, compare the staged topics with the resident ones and write z and
// its doc-major copy only for runs that changed.  A full scatter of zdoc is a
// random 2-byte permutation of T tokens (26 ms on PubMed-shape, DRAM
// read-modify-write of every sector); a round trip that hands the sampler's
// own output back costs only the coalesced compare.
// first a 16-byte compare of the whole staged array against z: when nothing
// differs (a round trip of the sampler's own output) the per-run pass exits
// at once instead of reading every run's bounds
__global__ void staged_diff_kernel(long long T, const uint16_t* __restrict__ zin, const uint16_t* __restrict__ z,
                                   unsigned int* any) {
    const long long nv = T >> 3, stride = (long long)gridDim.x * blockDim.x;
    bool d = false;
    const uint4* a = reinterpret_cast<const uint4*>(zin);
    const uint4* b = reinterpret_cast<const uint4*>(z);
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < nv; i += stride) {
        const uint4 x = __ldcs(a + i), y = __ldg(b + i);
        d |= (x.x != y.x) | (x.y != y.y) | (x.z != y.z) | (x.w != y.w);
    }
    for (long long t = nv * 8 + (long long)blockIdx.x * blockDim.x + threadIdx.x; t < T; t += stride)
        d |= zin[t] != z[t];
    if (__syncthreads_or(d) && threadIdx.x == 0) atomicOr(any, 1u);
}

__global__ void import_staged_gate(long long R, const uint32_t* __restrict__ run_start,
                                   const uint32_t* __restrict__ dwpos, const uint16_t* __restrict__ zin, uint16_t* z,
                                   uint16_t* zdoc, const unsigned int* any) {
    if (*any == 0u) return;                   // nothing changed
    for (long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x; r < R; r += (long long)gridDim.x * blockDim.x) {
        const uint32_t t0 = run_start[r], t1 = run_start[r + 1];
        bool diff = false;
        for (uint32_t t = t0; t < t1; ++t) diff |= zin[t] != z[t];
        if (diff) {
            const uint32_t p = dwpos[r];
            for (uint32_t t = t0; t < t1; ++t) {
                const uint16_t k = zin[t];
                z[t] = k;
                zdoc[p + (t - t0)] = k;
            }
        }
    }
}

cudaError_t launch_import_staged(gf_shard* s) {
    if (s->R == 0) return cudaSuccess;
    // bytes[1]: the "any staged topic differs" flag
    unsigned int* any = reinterpret_cast<unsigned int*>(s->d.bytes + 1);
    cudaError_t e = cudaMemsetAsync(any, 0, 4, s->stream);
    if (e != cudaSuccess) return e;
    staged_diff_kernel<<<148 * 8, 256, 0, s->stream>>>((long long)s->T, s->d.zstage, s->d.z, any);
    import_staged_gate<<<148 * 8, 256, 0, s->stream>>>((long long)s->R, s->d.run_start, s->d.run_dwpos, s->d.zstage,
                                                       s->d.z, s->d.zdoc, any);
    return cudaGetLastError();
}

cudaError_t launch_zdoc_sync(gf_shard* s) {
    if (s->R == 0) return cudaSuccess;
    zdoc_sync_kernel<<<148 * 8, 256, 0, s->stream>>>((long long)s->R, s->d.run_start, s->d.run_dwpos, s->d.z,
                                                     s->d.zdoc);
    return cudaGetLastError();
}

// ----------------------------------------------------------- ll reduce ------
// Deterministic two-level sum: CTA c reduces the fixed chunk [c n/G, (c+1) n/G)
// in a fixed order, the last CTA to finish (atomic ticket) adds the G chunk
// sums in index order.  out[0] = sum; out[1..G] chunk sums; out[kLlSlots-1]
// holds the ticket (reset by the last CTA).
constexpr int kLlBlocks = 148;
__global__ void __launch_bounds__(256) ll_reduce_kernel(const double* __restrict__ part, long long n, double* out) {
    __shared__ double sh[256];
    __shared__ bool last;
    const long long lo = n * blockIdx.x / gridDim.x, hi = n * (blockIdx.x + 1) / gridDim.x;
    double s = 0.0;
    for (long long i = lo + threadIdx.x; i < hi; i += 256) s += part[i];
    sh[threadIdx.x] = s;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
        if ((int)threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
        __syncthreads();
    }
    unsigned int* ticket = reinterpret_cast<unsigned int*>(out + kLlSlots - 1);
    if (threadIdx.x == 0) {
        out[1 + blockIdx.x] = sh[0];
        __threadfence();
        last = atomicAdd(ticket, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (last && threadIdx.x == 0) {
        __threadfence();
        double t = 0.0;
        for (unsigned b = 0; b < gridDim.x; ++b) t += __ldcg(out + 1 + b);
        out[0] = t;
        *ticket = 0u;
    }
}

cudaError_t launch_ll_reduce(gf_shard* s) {
    const long long n = s->n_slices;
    const int g = (int)std::max<long long>(1, std::min<long long>(kLlBlocks, (n + 2047) / 2048));
    ll_reduce_kernel<<<g, 256, 0, s->stream>>>(s->d.ll_part, n, s->d.ll_sum);
    return cudaGetLastError();
}

// --------------------------------------------------------- theta export ------
__global__ void theta_export_kernel(int D, const uint2* __restrict__ meta, const uint32_t* __restrict__ ent,
                                    const int64_t* __restrict__ rowptr, uint16_t* ids, uint16_t* cnt, TPos tm) {
    const int lane = threadIdx.x & 31;
    const long long w = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
    for (long long d = w; d < D; d += nw) {
        const uint2 m = meta[d];
        const int64_t o = rowptr[d];
        for (uint32_t j = lane; j < m.y; j += 32) {
            const uint32_t e = ent[m.x + j];
            ids[o + j] = (uint16_t)tpos_inv((e & 0xffffu) >> 2, tm);
            cnt[o + j] = (uint16_t)(e >> 16);
        }
    }
}

__global__ void theta_import_kernel(int D, uint2* meta, uint32_t* ent, const int64_t* __restrict__ rowptr,
                                    const uint16_t* __restrict__ ids, const uint16_t* __restrict__ cnt, TPos tm) {
    const int lane = threadIdx.x & 31;
    const long long w = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
    for (long long d = w; d < D; d += nw) {
        const int64_t o = rowptr[d], n = rowptr[d + 1] - o;
        const uint32_t base = meta[d].x;
        for (int64_t j = lane; j < n; j += 32) ent[base + j] = (tpos(ids[o + j], tm) << 2) | ((uint32_t)cnt[o + j] << 16);
        if (lane < ((8 - (n & 7)) & 7)) ent[base + n + lane] = 0u;   // zero pads (see K3)
        if (lane == 0) meta[d].y = (uint32_t)n;
    }
}

cudaError_t launch_theta_export(gf_shard* s, const int64_t* d_rowptr, uint16_t* d_ids, uint16_t* d_cnt) {
    if (s->D == 0) return cudaSuccess;
    theta_export_kernel<<<1184, 256, 0, s->stream>>>((int)s->D, s->d.theta_meta, s->d.theta_ent, d_rowptr, d_ids,
                                                     d_cnt, tpos_geom(s->K));
    return cudaGetLastError();
}

cudaError_t launch_theta_import(gf_shard* s, const int64_t* d_rowptr, const uint16_t* d_ids, const uint16_t* d_cnt) {
    if (s->D == 0) return cudaSuccess;
    theta_import_kernel<<<1184, 256, 0, s->stream>>>((int)s->D, s->d.theta_meta, s->d.theta_ent, d_rowptr, d_ids,
                                                     d_cnt, tpos_geom(s->K));
    return cudaGetLastError();
}

// ----------------------------------------------------------- phi export ------
// word-major columns <-> reference K x V row-major, 32x32 tiles through smem
__global__ void phi_export_kernel(const uint32_t* __restrict__ sync, long long off16, const int32_t* __restrict__ wcol,
                                  int K, int Kp, int V, uint32_t* out) {
    __shared__ uint32_t tile[32][33];
    const int v0 = blockIdx.x * 32, k0 = blockIdx.y * 32;
    const uint16_t* phi16 = reinterpret_cast<const uint16_t*>(sync + off16);
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        const int v = v0 + r, k = k0 + threadIdx.x;
        uint32_t val = 0;
        if (v < V && k < K) {
            const int col = wcol[v];
            val = col >= 0 ? (uint32_t)phi16[(size_t)col * Kp + k] : sync[(size_t)(~col) * K + k];
        }
        tile[r][threadIdx.x] = val;
    }
    __syncthreads();
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        const int k = k0 + r, v = v0 + threadIdx.x;
        if (k < K && v < V) out[(size_t)k * V + v] = tile[threadIdx.x][r];
    }
}

__global__ void phi_import_kernel(uint32_t* sync, long long off16, const int32_t* __restrict__ wcol, int K, int Kp,
                                  int V, const uint32_t* __restrict__ in) {
    __shared__ uint32_t tile[32][33];
    const int v0 = blockIdx.x * 32, k0 = blockIdx.y * 32;
    uint16_t* phi16 = reinterpret_cast<uint16_t*>(sync + off16);
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        const int k = k0 + r, v = v0 + threadIdx.x;
        tile[threadIdx.x][r] = (k < K && v < V) ? in[(size_t)k * V + v] : 0u;
    }
    __syncthreads();
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        const int v = v0 + r, k = k0 + threadIdx.x;
        if (v < V && k < K) {
            const int col = wcol[v];
            if (col >= 0) phi16[(size_t)col * Kp + k] = (uint16_t)tile[r][threadIdx.x];
            else sync[(size_t)(~col) * K + k] = tile[r][threadIdx.x];
        }
    }
}

cudaError_t launch_phi_export(gf_shard* s, uint32_t* d_out, const int32_t* d_wcol) {
    dim3 grid((s->V + 31) / 32, (s->K + 31) / 32);
    phi_export_kernel<<<grid, dim3(32, 8), 0, s->stream>>>(s->d.sync, s->off_phi16_u32, d_wcol, s->K, s->Kp, s->V,
                                                            d_out);
    return cudaGetLastError();
}

cudaError_t launch_phi_import(gf_shard* s, const uint32_t* d_in, const int32_t* d_wcol) {
    dim3 grid((s->V + 31) / 32, (s->K + 31) / 32);
    phi_import_kernel<<<grid, dim3(32, 8), 0, s->stream>>>(s->d.sync, s->off_phi16_u32, d_wcol, s->K, s->Kp, s->V,
                                                            d_in);
    return cudaGetLastError();
}

// ------------------------------------------------------ ptree primitive ------
__global__ void ptree_level_kernel(const float* prev, long long prev_len, float* next, long long len, int F) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < len) next[i] = prev[min((long long)F * i + F - 1, prev_len - 1)];
}

__global__ void ptree_sample_kernel(const float* levels, const long long* off, const long long* len, int nlev, int F,
                                    const float* __restrict__ u, long long m, int64_t* out) {
    const int lane = threadIdx.x & 31;
    const long long w = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
    for (long long q = w; q < m; q += nw) {
        const float uu = u[q];
        long long idx = 0;
        for (int l = nlev - 1; l >= 0; --l) {
            const long long lo = idx * F;
            const int n = (int)min((long long)F, len[l] - lo);
            const bool ok = lane < n && levels[off[l] + lo + lane] > uu;
            const unsigned b = __ballot_sync(kFull, ok);
            idx = b ? lo + __ffs(b) - 1 : lo + n - 1;   // last child bounds u from above
        }
        if (lane == 0) out[q] = idx;
    }
}

cudaError_t ptree_sample(const float* d_prefix, int64_t n, int F, const float* d_u, int64_t m, int64_t* d_idx,
                         cudaStream_t st) {
    std::vector<long long> off{0}, len{n};
    long long total = n;
    while (len.back() > 1) {
        const long long l = (len.back() + F - 1) / F;
        off.push_back(total);
        len.push_back(l);
        total += l;
    }
    float* lv = nullptr;
    long long* dmeta = nullptr;
    cudaError_t e = cudaMalloc(&lv, sizeof(float) * total);
    if (e != cudaSuccess) return e;
    e = cudaMalloc(&dmeta, sizeof(long long) * 2 * off.size());
    if (e != cudaSuccess) { cudaFree(lv); return e; }
    cudaMemcpyAsync(lv, d_prefix, sizeof(float) * n, cudaMemcpyDeviceToDevice, st);
    for (size_t l = 1; l < off.size(); ++l)
        ptree_level_kernel<<<(unsigned)((len[l] + 255) / 256), 256, 0, st>>>(lv + off[l - 1], len[l - 1], lv + off[l],
                                                                          len[l], F);
    cudaMemcpyAsync(dmeta, off.data(), sizeof(long long) * off.size(), cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(dmeta + off.size(), len.data(), sizeof(long long) * len.size(), cudaMemcpyHostToDevice, st);
    const long long blocks = std::min<long long>((m + 7) / 8, 4096);
    if (m > 0)
        ptree_sample_kernel<<<(unsigned)blocks, 256, 0, st>>>(lv, dmeta, dmeta + off.size(), (int)off.size(), F, d_u, m,
                                                            d_idx);
    e = cudaStreamSynchronize(st);
    cudaFree(lv);
    cudaFree(dmeta);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

}  // namespace gf
