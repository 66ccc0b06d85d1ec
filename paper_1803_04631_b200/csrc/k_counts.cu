// k_counts.cu -- count maintenance kernels (section 6.2):
//   K2 phi_rebuild   model.py:142-161  rebuild_phi_replica (+ n_k)
//   K3 theta_rebuild model.py:91-124   rebuild_theta_row / rebuild_theta
//   prepare          Eq. 1 denominators 1/(n_k + V b)
//   ll_reduce        deterministic fp64 reduction of the sampler's partials
//   theta / phi export + import (the reference dataclass layouts)
//   ptree primitive  ptree.py:116-151 (build levels + ballot descent)
#include "gf_internal.cuh"
#include "gf_device.cuh"

#include <cub/cub.cuh>
#include <thrust/iterator/transform_iterator.h>

namespace gf {

// ---------------------------------------------------------------- K2 ------
// One WARP per work item, items claimed dynamically (one global atomic per
// item; the next item's z range is bulk-prefetched into L2 when claimed).  An
// item is (phi column, token range), built on the host by k_layout.cu: a light
// word's whole group (<= heavy_threshold <= 65535 tokens, 16-bit column), a
// piece of <= GF_K2_PIECE (16384) tokens of a heavy word (32-bit column,
// global atomics), or an empty item for a light word absent from the shard;
// longest first.  Tokens are word-grouped, so an item is one contiguous z
// range: the warp streams it with double-buffered 16-byte loads and counts
// into its private PACKED histogram in shared memory (two 16-bit bins per u32
// word; at most 65528 tokens are counted between flushes, so a bin cannot
// carry into its neighbour), then
//   light: writes the whole packed column densely (16-byte stores, zeros
//          included) -- the light region needs no memset;
//   heavy: adds its nonzero cells to the pre-zeroed 32-bit column;
// and clears the histogram it read.  n_k accumulates per CTA in shared memory
// (nonzero cells only) and is flushed with K atomics at the end.  No block
// barrier inside the item loop: each warp keeps its own loads in flight.
//
// K2X (X = true): the same kernel fused with
// the peer-memory phi exchange of a node (k_peer.cu maps the ranks' sync
// buffers), pipelined by STRIPES of the sync buffer.  The items are sorted by
// the first buffer word they write (gf::peer_open), so the stripes fill in
// order; the warp that completes the last item of stripe s (per-stripe
// counters, fenced) release-stores the iteration's epoch into stripe s's flag
// on every rank.  A CTA with no items left flushes its n_k (the last CTA to do
// so signals the n_k stripe) and turns to the exchange: for each stripe in
// order it waits until every rank has signalled it, then sums this rank's
// 1/G of the stripe over the G replicas (16-byte peer loads) and stores the
// sum into all G replicas -- the two-shot allreduce of the round-1 exchange
// kernel, overlapped with the tail of the count.  The last CTA to finish
// signals "done" to every rank and waits for every rank's "done", so the
// kernel returns only when no peer will touch this buffer again this
// iteration.  The grid is the resident persistent grid (every CTA that waits
// is co-resident with the ones still counting); a wait beyond the timeout
// sets errs[3] (a dead peer reports TrainingError, no hang).
constexpr int kK2Warps = 8;
constexpr unsigned long long kK2XTimeoutNs = 20ull * 1000 * 1000 * 1000;

struct K2XArgs {
    uint32_t* buf[kMaxPeers];      // every rank's sync buffer (own included)
    uint32_t* sig[kMaxPeers];      // every rank's fused-kernel signal slots
    int rank = 0, world = 1;
    uint32_t epoch = 0;
    int nstripe = 0;               // stripes over [0, off_nk); stripe nstripe = n_k
    long long stripe_words = 0;
    long long n = 0;               // u32 words of the exchanged buffer (phi + n_k)
    const unsigned* need = nullptr;  // [nstripe] items touching each stripe
    unsigned* done = nullptr;        // [nstripe] + [2] CTA counters (zeroed per launch)
    unsigned long long* err = nullptr;
};

// s_bins: 32-bit shared address of the warp's packed histogram
__device__ __forceinline__ void k2_count(uint32_t s_bins, uint32_t k, int K, uint32_t t, unsigned long long* errs) {
    if (k < (uint32_t)K) sh_red_add(s_bins + ((k >> 1) << 2), 1u << ((k & 1u) << 4));
    else atomicMin(errs, (unsigned long long)t);
}

// signal stripe s complete to every rank (slot s * kMaxPeers + this rank)
__device__ __forceinline__ void k2x_signal(const K2XArgs& x, int s) {
    __threadfence_system();
    for (int p = 0; p < x.world; ++p) st_release_sys(x.sig[p] + (size_t)s * kMaxPeers + x.rank, x.epoch);
}

// block-wide wait for slot s of every rank; false on timeout
__device__ bool k2x_wait(const K2XArgs& x, int s) {
    bool ok = true;
    if ((int)threadIdx.x < x.world) {
        const uint32_t* f = x.sig[x.rank] + (size_t)s * kMaxPeers + threadIdx.x;
        const unsigned long long t0 = now_ns();
        while ((int32_t)(ld_acquire_sys(f) - x.epoch) < 0) {
            if (now_ns() - t0 > kK2XTimeoutNs) {
                atomicMin(x.err, (unsigned long long)s);
                ok = false;
                break;
            }
            __nanosleep(128);
        }
    }
    return __syncthreads_and(ok);
}

// this rank's 1/G of words [lo, hi): sum over the replicas, store everywhere
__device__ __forceinline__ void k2x_reduce(const K2XArgs& x, long long lo, long long hi) {
    const long long plo = lo + (hi - lo) * x.rank / x.world, phi = lo + (hi - lo) * (x.rank + 1) / x.world;
    const long long v0 = (plo + 3) >> 2, v1 = phi >> 2;
    const long long stride = (long long)gridDim.x * blockDim.x;
    const long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    for (long long v = v0 + gid; v < v1; v += stride) {
        uint4 s = make_uint4(0, 0, 0, 0);
        for (int p = 0; p < x.world; ++p) {
            const uint4 q = __ldcg(reinterpret_cast<const uint4*>(x.buf[p]) + v);
            s.x += q.x; s.y += q.y; s.z += q.z; s.w += q.w;
        }
        for (int p = 0; p < x.world; ++p) __stcg(reinterpret_cast<uint4*>(x.buf[p]) + v, s);
    }
    const long long h1 = min(v0 * 4, phi), t0 = max(max(v1 * 4, plo), h1);
    for (long long i = plo + gid; i < h1; i += stride) {            // head words before the first vector
        uint32_t s = 0;
        for (int p = 0; p < x.world; ++p) s += __ldcg(x.buf[p] + i);
        for (int p = 0; p < x.world; ++p) __stcg(x.buf[p] + i, s);
    }
    for (long long i = t0 + gid; i < phi; i += stride) {            // tail words
        uint32_t s = 0;
        for (int p = 0; p < x.world; ++p) s += __ldcg(x.buf[p] + i);
        for (int p = 0; p < x.world; ++p) __stcg(x.buf[p] + i, s);
    }
}

template <bool X>
__global__ void __launch_bounds__(kK2Warps * 32) phi_rebuild_kernel(const int4* __restrict__ items, int n_items,
                                                                    const uint16_t* __restrict__ z, uint32_t* sync,
                                                                    int K, int Kp, long long off16, long long offnk,
                                                                    int nwarps_per_cta, unsigned int* next_item,
                                                                    unsigned long long* errs, K2XArgs x) {
    extern __shared__ uint32_t sh[];
    const int KW = Kp >> 1;                                   // packed words per histogram
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t* nks = sh;                                       // [K] this CTA's n_k
    uint32_t* bins = sh + ((K + 3) & ~3) + (size_t)warp * ((KW + 3) & ~3);
    for (int i = threadIdx.x; i < K; i += blockDim.x) nks[i] = 0u;
    if (warp < nwarps_per_cta)                                // only these warps own a histogram
        for (int i = lane; i < KW; i += 32) bins[i] = 0u;
    const uint32_t s_bins = smem_addr(bins), s_nks = smem_addr(nks);
    if (X && blockIdx.x == 0 && threadIdx.x == 0)             // stripes no item writes (all-zero columns)
        for (int s = 0; s < x.nstripe; ++s)
            if (x.need[s] == 0u) k2x_signal(x, s);
    __syncthreads();
    // 16-byte column stores need a 16-byte aligned packed column
    const bool vec_cols = (KW & 3) == 0 && (off16 & 3) == 0;
    uint32_t* phi16w = sync + off16;                           // packed light columns (u32 words)
    const uint4* zv = reinterpret_cast<const uint4*>(z);
    if (warp < nwarps_per_cta) {
        // the next item is claimed while the current one is counted, and its
        // z range is bulk-prefetched into L2 right away (TMA prefetch, one
        // instruction), so the item after this one starts on L2 hits instead of
        // a cold DRAM round trip per 2 KB batch
        int mine = 0;
        auto claim = [&]() {
            if (lane == 0) {
                mine = (int)atomicAdd(next_item, 1u);
                if (mine < n_items) {
                    const int4 nw = __ldg(items + mine);
                    const uint32_t p0 = (uint32_t)nw.y & ~7u, p1 = min(((uint32_t)nw.z + 7u) & ~7u, p0 + 32768u);
                    if (p1 > p0) prefetch_l2_bulk(z + p0, (p1 - p0) * 2u);
                }
            }
        };
        claim();
        int it = __shfl_sync(kFull, mine, 0);
        while (it < n_items) {
            const int4 w = __ldg(items + it);
            claim();
            const int col = w.x;
            // a heavy (32-bit column) item longer than 65535 tokens (one huge
            // (doc, word) run) is counted and flushed in pieces so no packed
            // 16-bit bin can carry; a light item is <= 65535 tokens by construction
            for (uint32_t t0 = (uint32_t)w.y, tend = (uint32_t)w.z;;) {
                const uint32_t t1 = col >= 0 ? tend : min(tend, t0 + 65528u);
                // ---- count: scalar head / tail, 16-byte body, double-buffered:
                // the next two 16-byte loads per lane are in flight while the
                // current two (16 topics) are counted by shared atomics ----
                const uint32_t a0 = min(t1, (t0 + 7u) & ~7u), a1 = max(a0, t1 & ~7u);
                if (t0 + lane < a0) k2_count(s_bins, z[t0 + lane], K, t0 + lane, errs);
                if (a1 + lane < t1) k2_count(s_bins, z[a1 + lane], K, a1 + lane, errs);
                const uint32_t qe = a1 >> 3;
                uint32_t q = (a0 >> 3) + lane;
                uint4 v[2];
#pragma unroll
                for (int i = 0; i < 2; ++i)
                    if (q + 32u * i < qe) v[i] = __ldg(zv + q + 32u * i);
                for (; q < qe; q += 64u) {
                    uint4 nx[2];
#pragma unroll
                    for (int i = 0; i < 2; ++i)
                        if (q + 64u + 32u * i < qe) nx[i] = __ldg(zv + q + 64u + 32u * i);
#pragma unroll
                    for (int i = 0; i < 2; ++i) {
                        if (q + 32u * i < qe) {
                            const uint32_t e[4] = {v[i].x, v[i].y, v[i].z, v[i].w};
                            const uint32_t tb = 8u * (q + 32u * i);
#pragma unroll
                            for (int h = 0; h < 4; ++h) {
                                k2_count(s_bins, e[h] & 0xffffu, K, tb + 2u * h, errs);
                                k2_count(s_bins, e[h] >> 16, K, tb + 2u * h + 1u, errs);
                            }
                        }
                    }
                    v[0] = nx[0];
                    v[1] = nx[1];
                }
                __syncwarp();
                // ---- flush: every packed word once (lane-strided), cleared behind ----
                if (col >= 0) {
                    uint32_t* dst = phi16w + (size_t)col * KW;
                    if (vec_cols) {
                        for (int j = lane; j < (KW >> 2); j += 32) {
                            const uint4 b = reinterpret_cast<const uint4*>(bins)[j];
                            reinterpret_cast<uint4*>(bins)[j] = make_uint4(0u, 0u, 0u, 0u);
                            reinterpret_cast<uint4*>(dst)[j] = b;
                            const uint32_t bw[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
                            for (int i = 0; i < 4; ++i) {
                                const uint32_t k = 8u * j + 2u * i;
                                if (bw[i] & 0xffffu) sh_red_add(s_nks + 4u * k, bw[i] & 0xffffu);
                                if (bw[i] >> 16) sh_red_add(s_nks + 4u * (k + 1), bw[i] >> 16);
                            }
                        }
                    } else {
                        for (int j = lane; j < KW; j += 32) {
                            const uint32_t b = bins[j];
                            bins[j] = 0u;
                            dst[j] = b;
                            if (b & 0xffffu) sh_red_add(s_nks + 8u * j, b & 0xffffu);
                            if (b >> 16) sh_red_add(s_nks + 8u * j + 4u, b >> 16);
                        }
                    }
                } else {
                    uint32_t* dst = sync + (size_t)(~col) * K;
                    for (int j = lane; j < KW; j += 32) {
                        const uint32_t b = bins[j];
                        if (!b) continue;
                        bins[j] = 0u;
                        const uint32_t k = 2u * j, c0 = b & 0xffffu, c1 = b >> 16;
                        if (c0) { sh_red_add(s_nks + 4u * k, c0); atomicAdd(dst + k, c0); }
                        if (c1) { sh_red_add(s_nks + 4u * (k + 1), c1); atomicAdd(dst + k + 1, c1); }
                    }
                }
                __syncwarp();
                if (t1 >= tend) break;
                t0 = t1;
            }
            if (X) {
                // the item's column is final: count it against the stripes it
                // touches, and publish any stripe it completes
                __threadfence();
                __syncwarp();
                if (lane == 0) {
                    const long long fw = col >= 0 ? off16 + (long long)col * KW : (long long)(~col) * K;
                    const long long lw = fw + (col >= 0 ? KW : K) - 1;
                    const int s0 = (int)(fw / x.stripe_words);
                    const int s1 = (int)min((long long)x.nstripe - 1, lw / x.stripe_words);
                    for (int s = s0; s <= s1; ++s)
                        if (atomicAdd(&x.done[s], 1u) + 1u == x.need[s]) k2x_signal(x, s);
                }
            }
            it = __shfl_sync(kFull, mine, 0);
        }
    }
    __syncthreads();
    uint32_t* nk = sync + offnk;
    for (int k = threadIdx.x; k < K; k += blockDim.x)
        if (nks[k]) atomicAdd(&nk[k], nks[k]);
    if (!X) return;
    // ---- fused exchange ----
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0 && atomicAdd(&x.done[x.nstripe], 1u) + 1u == gridDim.x) k2x_signal(x, x.nstripe);
    for (int s = 0; s <= x.nstripe; ++s) {
        if (!k2x_wait(x, s)) return;
        const long long lo = s < x.nstripe ? (long long)s * x.stripe_words : offnk;
        const long long hi = s < x.nstripe ? min((long long)(s + 1) * x.stripe_words, offnk) : x.n;
        k2x_reduce(x, lo, hi);
    }
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0 && atomicAdd(&x.done[x.nstripe + 1], 1u) + 1u == gridDim.x) {
        // every CTA of this rank has written its share everywhere: tell every
        // rank, then wait until every rank has done the same
        for (int p = 0; p < x.world; ++p) st_release_sys(x.sig[p] + (size_t)(x.nstripe + 1) * kMaxPeers + x.rank, x.epoch);
    }
    if (blockIdx.x == 0) k2x_wait(x, x.nstripe + 1);
}

// bytes of the K2 shared memory: the CTA's n_k plus one packed histogram per warp
static size_t k2_smem(int K, int Kp, int warps) {
    return ((size_t)((K + 3) & ~3) + (size_t)warps * (((Kp >> 1) + 3) & ~3)) * sizeof(uint32_t);
}

template <bool X>
static cudaError_t launch_k2(gf_shard* s, const K2XArgs& x) {
    s->ctx_dirty = true;
    // only the 32-bit columns (atomic adds) and n_k need zeroing: every 16-bit
    // column is rewritten whole by its item; the last word is the item counter
    cudaError_t e = cudaMemsetAsync(s->d.sync, 0, (size_t)s->off_phi16_u32 * 4, s->stream);
    if (e == cudaSuccess)
        e = cudaMemsetAsync(s->d.sync + s->off_nk_u32, 0, ((size_t)s->sync_u32 - s->off_nk_u32 + 1) * 4, s->stream);
    if (e == cudaSuccess && X) e = cudaMemsetAsync(x.done, 0, (size_t)(x.nstripe + 2) * 4, s->stream);
    if (e != cudaSuccess || (s->n_k2 == 0 && !X)) return e;
    const int nsm = sm_count(s->device);
    // 8 warps per CTA up to K = 8192 (16 KB histograms), 4 above
    const int warps = s->Kp > 8192 ? 4 : kK2Warps;
    const size_t smem = k2_smem(s->K, s->Kp, warps);
    static unsigned long long attr = 0;
    if (attr_once(attr, s->device)) {
        e = cudaFuncSetAttribute(phi_rebuild_kernel<X>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
        if (e != cudaSuccess) return e;
    }
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, phi_rebuild_kernel<X>, kK2Warps * 32, smem);
    const long long need = (s->n_k2 + warps - 1) / warps;
    // K2X: the resident grid, so every waiting CTA is co-resident with the counting ones
    const long long cap = (long long)nsm * std::max(per_sm, 1);
    const long long grid = X ? cap : std::max<long long>(1, std::min<long long>(need, cap));
    phi_rebuild_kernel<X><<<(unsigned)grid, kK2Warps * 32, smem, s->stream>>>(
        s->d.k2items, (int)s->n_k2, s->d.z, s->d.sync, s->K, s->Kp, s->off_phi16_u32, s->off_nk_u32, warps,
        s->d.sync + s->sync_u32, s->d.errs, x);
    return cudaGetLastError();
}

cudaError_t launch_phi_rebuild(gf_shard* s) { return launch_k2<false>(s, K2XArgs{}); }

cudaError_t launch_phi_rebuild_exchange(gf_shard* s) {
    const PeerGroup& g = s->peer;
    K2XArgs x;
    for (int p = 0; p < g.world; ++p) {
        x.buf[p] = g.buf[p];
        x.sig[p] = g.sig[p] + g.sig_fused;
    }
    x.rank = g.rank;
    x.world = g.world;
    x.epoch = ++s->peer.epoch;
    x.nstripe = g.nstripe;
    x.stripe_words = g.stripe_words;
    x.n = s->sync_u32;
    x.need = g.xdev;
    x.done = g.xdev + g.nstripe;
    x.err = s->d.errs + 3;
    return launch_k2<true>(s, x);
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
__host__ __device__ inline int k3_warp_u32(int K) { return K + 2 * k3_words(K) + 32; }   // bins | bitmap | word ranks | 32 dummies

template <int MINB>
__global__ void __launch_bounds__(256, MINB) theta_rebuild_kernel(int D, const uint32_t* __restrict__ dw_ptr,
                                                               const uint16_t* __restrict__ zdoc, uint32_t* theta_ent,
                                                               uint2* theta_meta, int K, int warps_per_cta, int gsz,
                                                               int pf_back, unsigned long long* errs) {
    extern __shared__ uint32_t sh[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int NW = k3_words(K);
    // CTA table of the entries' topic fields, tpos(k) << 2 (a lookup instead of
    // the multiply-high / remainder per emitted entry)
    uint32_t* tpo = sh + (size_t)warps_per_cta * k3_warp_u32(K);
    {
        const TPos tm = tpos_geom(K);
        for (int k = threadIdx.x; k < K; k += blockDim.x) tpo[k] = tpos((uint32_t)k, tm) << 2;
        __syncthreads();
    }
    const uint32_t s_tpo = smem_addr(tpo);
    uint32_t* bins = sh + (size_t)warp * k3_warp_u32(K);
    uint32_t* bmp = bins + K;
    uint32_t* wpre = bmp + NW;                     // distinct topics below each bitmap word
    for (int i = lane; i < K + NW; i += 32) bins[i] = 0u;
    __syncwarp();
    // 32-bit shared addresses of the warp's bins / bitmap / word ranks (sh_*)
    const uint32_t s_bins = smem_addr(bins), s_bmp = smem_addr(bmp), s_wpre = smem_addr(wpre);
    const uint32_t s_dum = smem_addr(wpre + NW + lane);           // this lane's dummy word
    (void)wpre;
    const unsigned lt = (1u << lane) - 1u;
    // The warp takes GROUPS of gsz <= 32 consecutive documents (group g, then
    // g + the number of warps; gsz keeps >= 4 groups per warp): lane j holds
    // document j's {zdoc begin, length, theta row offset} (three coalesced
    // loads per group instead of three per document), and the next group's
    // are loaded while this one is processed.  Halfway through a group, lane
    // 0 bulk-prefetches the next group's topics into L2 (one contiguous zdoc
    // range), so the next group's loads hit L2; the next document's first 32
    // topics are always in flight (registers) while the current one is counted.
    const int ngroups = (D + gsz - 1) / gsz;
    const int gstride = gridDim.x * warps_per_cta;
    auto group_meta = [&](int g, uint32_t& mb, uint32_t& mL, uint32_t& mo) {
        const int dd = g * gsz + lane;
        mb = mL = mo = 0u;
        if (g < ngroups && lane < gsz && dd < D) { mb = dw_ptr[dd]; mL = dw_ptr[dd + 1] - mb; mo = theta_meta[dd].x; }
    };
    int g = blockIdx.x * warps_per_cta + warp;
    uint32_t gb, gL, go;
    group_meta(g, gb, gL, go);
    const uint32_t b00 = __shfl_sync(kFull, gb, 0), L00 = __shfl_sync(kFull, gL, 0);   // all lanes shuffle
    uint32_t zf = (uint32_t)lane < L00 ? zdoc[b00 + lane] : 0xffffu;
    for (; g < ngroups; g += gstride) {
        uint32_t nb, nL, no;
        group_meta(g + gstride, nb, nL, no);
        const int nd = min(gsz, D - g * gsz);
        for (int i = 0; i < nd; ++i) {
            const int d = g * gsz + i;
            const uint32_t b = __shfl_sync(kFull, gb, i), L = __shfl_sync(kFull, gL, i), off = __shfl_sync(kFull, go, i);
            const bool last = i + 1 == nd;
            const uint32_t b1 = __shfl_sync(kFull, last ? nb : gb, last ? 0 : i + 1);
            const uint32_t L1 = __shfl_sync(kFull, last ? nL : gL, last ? 0 : i + 1);
            const uint32_t zn = (uint32_t)lane < L1 ? zdoc[b1 + lane] : 0xffffu;        // L1 = 0 past the end
            if (i == max(nd - pf_back, 0) && pf_back > 0) {
                const uint32_t b0 = __shfl_sync(kFull, nb, 0), end = __reduce_max_sync(kFull, nL ? nb + nL : 0u);
                if (lane == 0 && end > b0) {
                    const uint32_t p0 = b0 & ~7u, p1 = (end + 7u) & ~7u;
                    prefetch_l2_bulk(zdoc + p0, (p1 - p0) * 2u);
                }
            }
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
                    theta_ent[off + __popc(heads & lt)] = sh_ld(s_tpo + 4u * key) | ((next - lane) << 16);
                }
                nnz = __popc(heads);
            } else if (L <= 128) {
                // 32 < L <= 128, the tokens stay in registers (ncol = ceil(L / 32)
                // columns, warp-uniform).  Count: every token adds to its bin and
                // sets its bitmap bit (no returned values, no branches).  Emit: the
                // rank of topic k = distinct topics below it = word prefix + popc
                // inside the word; one token per topic wins atomicExch(bin, 0) (it
                // gets the count and clears the bin) and writes the entry.
                const uint32_t ncol = (L + 31u) >> 5;
                const uint16_t* zl = zdoc + (b + (uint32_t)lane);           // column j at zl[32 j]
                uint32_t kk[4] = {zf, 0xffffu, 0xffffu, 0xffffu};
#pragma unroll
                for (uint32_t j = 1; j < 4; ++j)
                    if (j < ncol && lane + 32u * j < L) kk[j] = zl[32u * j];
                // count: branch-free -- a token outside [0, K) (past the document
                // in its column, or an invalid topic) updates the lane's own dummy
                // word instead; an invalid topic is reported once per document
                bool bad = false;
#pragma unroll
                for (uint32_t j = 0; j < 4; ++j) {
                    if (j < ncol) {
                        const uint32_t k = kk[j];
                        const bool ok = k < (uint32_t)K;
                        bad |= !ok && (j == 0 || lane + 32u * j < L);      // a token, not a pad
                        sh_red_add(ok ? s_bins + 4u * k : s_dum, 1u);
                        sh_red_or(ok ? s_bmp + ((k >> 3) & ~3u) : s_dum, 1u << (k & 31u));
                        if (!ok) kk[j] = 0xffffu;
                    }
                }
                if (__any_sync(kFull, bad) && bad) atomicMin(errs + 2, (unsigned long long)d);
                __syncwarp();
                if (NW <= 32) {
                    // K <= 1024: lane w holds bitmap word w and the distinct topics
                    // below it in registers; the emit fetches both by shuffle
                    const uint32_t word = lane < NW ? sh_ld(s_bmp + 4u * lane) : 0u;
                    if (lane < NW) sh_st(s_bmp + 4u * lane, 0u);
                    const uint32_t pc = __popc(word);
                    uint32_t incl = pc;
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const uint32_t y = __shfl_up_sync(kFull, incl, o);
                        if (lane >= o) incl += y;
                    }
                    nnz = __shfl_sync(kFull, incl, 31);
                    const uint32_t pre = incl - pc;
                    // every column's exchange first (their latencies overlap; the
                    // dummy word absorbs the lanes without a topic), then each
                    // winner's store -- the only predicated instruction
                    uint32_t cc[4];
#pragma unroll
                    for (uint32_t j = 0; j < 4; ++j) {
                        const bool ok = kk[j] < (uint32_t)K;
                        const uint32_t c = j < ncol ? sh_exch(ok ? s_bins + 4u * kk[j] : s_dum, 0u) : 0u;
                        cc[j] = ok ? c : 0u;
                    }
#pragma unroll
                    for (uint32_t j = 0; j < 4; ++j) {
                        if (j < ncol) {
                            const uint32_t k = kk[j] < (uint32_t)K ? kk[j] : 0u, w = k >> 5;
                            const uint32_t ww = __shfl_sync(kFull, word, w), pw = __shfl_sync(kFull, pre, w);
                            const uint32_t e = sh_ld(s_tpo + 4u * k) | (cc[j] << 16);   // <= 128: no overflow
                            const uint32_t at = off + pw + __popc(ww & ((1u << (k & 31u)) - 1u));
                            if (cc[j]) theta_ent[at] = e;
                        }
                    }
                } else {
                    uint32_t base = 0;
                    for (int c = 0; c < NW; c += 32) {
                        const int w = c + lane;
                        const uint32_t pc = w < NW ? __popc(sh_ld(s_bmp + 4u * w)) : 0u;
                        uint32_t incl = pc;
#pragma unroll
                        for (int o = 1; o < 32; o <<= 1) {
                            const uint32_t y = __shfl_up_sync(kFull, incl, o);
                            if (lane >= o) incl += y;
                        }
                        if (w < NW) sh_st(s_wpre + 4u * w, base + incl - pc);
                        base += __shfl_sync(kFull, incl, 31);
                    }
                    nnz = base;
                    __syncwarp();
#pragma unroll
                    for (uint32_t j = 0; j < 4; ++j) {
                        const uint32_t k = kk[j];
                        const uint32_t c = (j < ncol && k < (uint32_t)K) ? sh_exch(s_bins + 4u * k, 0u) : 0u;
                        if (c) {
                            const uint32_t w = k >> 5;
                            theta_ent[off + sh_ld(s_wpre + 4u * w) + __popc(sh_ld(s_bmp + 4u * w) & ((1u << (k & 31u)) - 1u))] =
                                sh_ld(s_tpo + 4u * k) | (c << 16);                 // <= 128: no overflow
                        }
                    }
                    __syncwarp();
#pragma unroll
                    for (uint32_t j = 0; j < 4; ++j)
                        if (j < ncol && kk[j] < (uint32_t)K) sh_st(s_bmp + ((kk[j] >> 3) & ~3u), 0u);
                }
                __syncwarp();
            } else {
                // branch-free count as above (L > 128: the first four columns are full)
                bool bad = false;
                auto count = [&](uint32_t k) {
                    const bool ok = k < (uint32_t)K;
                    bad |= !ok;
                    sh_red_add(ok ? s_bins + 4u * k : s_dum, 1u);
                    sh_red_or(ok ? s_bmp + ((k >> 3) & ~3u) : s_dum, 1u << (k & 31u));
                };
                // the next 96 topics load together (independent), then count
                const uint16_t* zl = zdoc + (b + (uint32_t)lane);
                const uint32_t k1 = zl[32], k2 = zl[64], k3 = zl[96];
                count(zf);
                count(k1);
                count(k2);
                count(k3);
                for (uint32_t i = lane + 128u; i < L; i += 32) count(zdoc[b + i]);
                if (__any_sync(kFull, bad) && bad) atomicMin(errs + 2, (unsigned long long)d);
                __syncwarp();
                uint32_t base = 0, mx = 0;
                for (int c = 0; c < NW; c += 32) {
                    const int w = c + lane;
                    uint32_t word = w < NW ? sh_ld(s_bmp + 4u * w) : 0u;
                    const uint32_t pc = __popc(word);
                    uint32_t incl = pc;
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const uint32_t y = __shfl_up_sync(kFull, incl, o);
                        if (lane >= o) incl += y;
                    }
                    uint32_t pos = off + base + incl - pc;
                    if (w < NW) sh_st(s_bmp + 4u * w, 0u);
                    while (word) {
                        const uint32_t k = ((uint32_t)w << 5) + (uint32_t)(__ffs(word) - 1);
                        word &= word - 1u;
                        const uint32_t v = sh_ld(s_bins + 4u * k);
                        sh_st(s_bins + 4u * k, 0u);
                        theta_ent[pos++] = sh_ld(s_tpo + 4u * k) | (min(v, 65535u) << 16);
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
            zf = zn;
        }
        gb = nb;
        gL = nL;
        go = no;
    }
}

template <int MINB>
static cudaError_t launch_k3(gf_shard* s, cudaStream_t st) {
    const size_t per_warp = (size_t)k3_warp_u32(s->K) * 4;
    int wpc = 8;
    while (wpc > 1 && (size_t)wpc * per_warp > 96 * 1024) wpc >>= 1;
    const size_t smem = (size_t)wpc * per_warp + (size_t)s->K * 4;     // + the tpos table
    static unsigned long long attr = 0;
    if (attr_once(attr, s->device)) {
        cudaError_t e = cudaFuncSetAttribute(theta_rebuild_kernel<MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             200 * 1024);
        if (e != cudaSuccess) return e;
    }
    // persistent grid (exactly the resident CTAs)
    const int nsm = sm_count(s->device);
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, theta_rebuild_kernel<MINB>, wpc * 32, smem);
    // GF_K3_CTAS (A/B): fewer resident CTAs per SM, leaving room for K2's CTAs
    // beside it in the step (K3 alone fills the register file at 5 per SM)
    static const int cap_sm = (int)shard_env_int("GF_K3_CTAS", 0);
    if (cap_sm > 0) per_sm = std::min(per_sm, cap_sm);
    const long long need = (s->D + wpc - 1) / wpc;
    const long long grid = std::min<long long>(need, (long long)nsm * std::max(per_sm, 1));
    // documents per warp group: 32, unless that leaves fewer than 4 groups per warp
    const int gsz = (int)std::max<long long>(1, std::min<long long>(32, s->D / (4 * grid * wpc)));
    // the next group's topics are bulk-prefetched into L2 this many documents
    // before the group ends (0: off)
    static const int pf_back = (int)shard_env_int("GF_K3_PF", 8);
    theta_rebuild_kernel<MINB><<<(unsigned)grid, wpc * 32, smem, st>>>((int)s->D, s->d.dw_ptr, s->d.zdoc,
                                                                       s->d.theta_ent, s->d.theta_meta, s->K, wpc, gsz,
                                                                       pf_back, s->d.errs);
    return cudaGetLastError();
}

cudaError_t launch_theta_rebuild(gf_shard* s, cudaStream_t st) {
    if (s->D == 0) return cudaSuccess;
    if (!st) st = s->stream;
    // GF_K3_MINB (A/B): CTAs per SM the register budget is sized for
    static const int minb = (int)shard_env_int("GF_K3_MINB", 5);
    return minb == 4 ? launch_k3<4>(s, st) : launch_k3<5>(s, st);
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
                                   uint16_t* zdoc, const unsigned int* any, bool doc_order) {
    if (*any == 0u) return;                   // nothing changed
    for (long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x; r < R; r += (long long)gridDim.x * blockDim.x) {
        const uint32_t t0 = run_start[r], t1 = run_start[r + 1], p = dwpos[r];
        // the staged array is in chunk order (zin[t]) or doc-major order (zin[p + i])
        const uint32_t i0 = doc_order ? p : t0;
        bool diff = false;
        for (uint32_t t = t0; t < t1; ++t) diff |= zin[i0 + (t - t0)] != z[t];
        if (diff) {
            for (uint32_t t = t0; t < t1; ++t) {
                const uint16_t k = zin[i0 + (t - t0)];
                z[t] = k;
                zdoc[p + (t - t0)] = k;
            }
        }
    }
}

cudaError_t launch_import_staged(gf_shard* s, bool doc_order) {
    if (s->R == 0) return cudaSuccess;
    // bytes[1]: the "any staged topic differs" flag
    unsigned int* any = reinterpret_cast<unsigned int*>(s->d.bytes + 1);
    cudaError_t e = cudaMemsetAsync(any, 0, 4, s->stream);
    if (e != cudaSuccess) return e;
    // the whole-array compare runs against the resident array of the same order
    staged_diff_kernel<<<sm_count(s->device) * 8, 256, 0, s->stream>>>((long long)s->T, s->d.zstage,
                                                                        doc_order ? s->d.zdoc : s->d.z, any);
    import_staged_gate<<<sm_count(s->device) * 8, 256, 0, s->stream>>>((long long)s->R, s->d.run_start, s->d.run_dwpos,
                                                                        s->d.zstage, s->d.z, s->d.zdoc, any, doc_order);
    return cudaGetLastError();
}

cudaError_t launch_zdoc_sync(gf_shard* s) {
    if (s->R == 0) return cudaSuccess;
    zdoc_sync_kernel<<<sm_count(s->device) * 8, 256, 0, s->stream>>>((long long)s->R, s->d.run_start, s->d.run_dwpos, s->d.z,
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

// set_theta's checks on the device, before anything is written: a row longer
// than its fixed capacity, a topic id >= K or a zero count, topic ids not
// strictly increasing.  first = min over failures of
//   d << 34 | (capacity ? 0 : (j - row start + 1) << 1 | (kind: 0 bad entry, 1 order))
// i.e. the first document, and inside it the first entry the host loop
// (gf_shard_set_theta) would have stopped at.
__global__ void theta_validate_kernel(int D, const uint2* __restrict__ meta, uint32_t cap,
                                      const int64_t* __restrict__ rowptr, const uint16_t* __restrict__ ids,
                                      const uint16_t* __restrict__ cnt, int K, unsigned long long* first) {
    const int lane = threadIdx.x & 31;
    const long long w = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
    for (long long d = w; d < D; d += nw) {
        const int64_t o = rowptr[d], n = rowptr[d + 1] - o;
        const uint32_t room = (d + 1 < D ? meta[d + 1].x : cap) - meta[d].x;
        if (n < 0 || n > (int64_t)room) {
            if (lane == 0) atomicMin(first, (unsigned long long)d << 34);
            continue;
        }
        for (int64_t j = lane; j < n; j += 32) {
            const uint32_t t = ids[o + j];
            int kind = -1;
            if (t >= (uint32_t)K || cnt[o + j] == 0) kind = 0;
            else if (j > 0 && t <= ids[o + j - 1]) kind = 1;
            if (kind >= 0)
                atomicMin(first, ((unsigned long long)d << 34) | ((unsigned long long)(j + 1) << 1) | (unsigned)kind);
        }
    }
}

cudaError_t launch_theta_validate(gf_shard* s, const int64_t* d_rowptr, const uint16_t* d_ids, const uint16_t* d_cnt,
                                  unsigned long long* d_first) {
    cudaError_t e = cudaMemsetAsync(d_first, 0xff, 8, s->stream);
    if (e != cudaSuccess || s->D == 0) return e;
    const int nsm = sm_count(s->device);
    theta_validate_kernel<<<8 * nsm, 256, 0, s->stream>>>((int)s->D, s->d.theta_meta, (uint32_t)s->theta_cap,
                                                          d_rowptr, d_ids, d_cnt, s->K, d_first);
    return cudaGetLastError();
}

// row_ptr of the exported CSR on the device: d_rowptr[0] = 0, d_rowptr[d+1] =
// sum of nnz over rows <= d (an inclusive scan of theta_meta[].y)
struct MetaNnz {
    __device__ int64_t operator()(const uint2& m) const { return (int64_t)m.y; }
};

cudaError_t theta_rowptr(gf_shard* s, int64_t* d_rowptr, void* tmp, size_t* tmp_bytes) {
    const auto in = thrust::make_transform_iterator(s->d.theta_meta, MetaNnz());
    if (!tmp) return cub::DeviceScan::InclusiveSum(nullptr, *tmp_bytes, in, d_rowptr + 1, (int)s->D, s->stream);
    cudaError_t e = cudaMemsetAsync(d_rowptr, 0, 8, s->stream);
    if (e != cudaSuccess || s->D == 0) return e;
    return cub::DeviceScan::InclusiveSum(tmp, *tmp_bytes, in, d_rowptr + 1, (int)s->D, s->stream);
}

cudaError_t launch_theta_export(gf_shard* s, const int64_t* d_rowptr, uint16_t* d_ids, uint16_t* d_cnt) {
    if (s->D == 0) return cudaSuccess;
    const int nsm = sm_count(s->device);
    theta_export_kernel<<<8 * nsm, 256, 0, s->stream>>>((int)s->D, s->d.theta_meta, s->d.theta_ent, d_rowptr, d_ids,
                                                     d_cnt, tpos_geom(s->K));
    return cudaGetLastError();
}

cudaError_t launch_theta_import(gf_shard* s, const int64_t* d_rowptr, const uint16_t* d_ids, const uint16_t* d_cnt) {
    if (s->D == 0) return cudaSuccess;
    const int nsm = sm_count(s->device);
    theta_import_kernel<<<8 * nsm, 256, 0, s->stream>>>((int)s->D, s->d.theta_meta, s->d.theta_ent, d_rowptr, d_ids,
                                                     d_cnt, tpos_geom(s->K));
    return cudaGetLastError();
}

// ----------------------------------------------------------- phi export ------
// word-major columns <-> reference K x V row-major (u32, or u16 for a 16-bit
// PhiMatrix), 32x32 tiles through smem
template <typename T>
__global__ void phi_export_kernel(const uint32_t* __restrict__ sync, long long off16, const int32_t* __restrict__ wcol,
                                  int K, int Kp, int V, T* out) {
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
        if (k < K && v < V) out[(size_t)k * V + v] = (T)tile[threadIdx.x][r];   // u16: checked <= 65535 first
    }
}

template <typename T>
__global__ void phi_import_kernel(uint32_t* sync, long long off16, const int32_t* __restrict__ wcol, int K, int Kp,
                                  int V, const T* __restrict__ in) {
    __shared__ uint32_t tile[32][33];
    const int v0 = blockIdx.x * 32, k0 = blockIdx.y * 32;
    uint16_t* phi16 = reinterpret_cast<uint16_t*>(sync + off16);
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        const int k = k0 + r, v = v0 + threadIdx.x;
        tile[threadIdx.x][r] = (k < K && v < V) ? (uint32_t)in[(size_t)k * V + v] : 0u;
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

cudaError_t launch_phi_export(gf_shard* s, void* d_out, int width, const int32_t* d_wcol) {
    dim3 grid((s->V + 31) / 32, (s->K + 31) / 32);
    if (width == 16)
        phi_export_kernel<uint16_t><<<grid, dim3(32, 8), 0, s->stream>>>(s->d.sync, s->off_phi16_u32, d_wcol, s->K,
                                                                        s->Kp, s->V, (uint16_t*)d_out);
    else
        phi_export_kernel<uint32_t><<<grid, dim3(32, 8), 0, s->stream>>>(s->d.sync, s->off_phi16_u32, d_wcol, s->K,
                                                                        s->Kp, s->V, (uint32_t*)d_out);
    return cudaGetLastError();
}

cudaError_t launch_phi_import(gf_shard* s, const void* d_in, int width, const int32_t* d_wcol) {
    dim3 grid((s->V + 31) / 32, (s->K + 31) / 32);
    if (width == 16)
        phi_import_kernel<uint16_t><<<grid, dim3(32, 8), 0, s->stream>>>(s->d.sync, s->off_phi16_u32, d_wcol, s->K,
                                                                        s->Kp, s->V, (const uint16_t*)d_in);
    else
        phi_import_kernel<uint32_t><<<grid, dim3(32, 8), 0, s->stream>>>(s->d.sync, s->off_phi16_u32, d_wcol, s->K,
                                                                        s->Kp, s->V, (const uint32_t*)d_in);
    return cudaGetLastError();
}

// ------------------------------------------------------ ptree primitive ------
// ptree.py:116-136 levels (every F-th boundary of the level below) and the
// _descend of ptree.py:77-99 as a warp ballot per u, in fp32 (the device
// precision) or fp64 (the reference's oracle mode, ptree.py:119-121).  The
// optional stats are sample_with_stats' (levels visited, widest scan).
template <typename T>
__global__ void ptree_level_kernel(const T* prev, long long prev_len, T* next, long long len, int F) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < len) next[i] = prev[min((long long)F * i + F - 1, prev_len - 1)];
}

template <typename T>
__global__ void ptree_sample_kernel(const T* levels, const long long* off, const long long* len, int nlev, int F,
                                    const T* __restrict__ u, long long m, int64_t* out, int32_t* visited,
                                    int32_t* widest) {
    const int lane = threadIdx.x & 31;
    const long long w = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
    for (long long q = w; q < m; q += nw) {
        const T uu = u[q];
        long long idx = 0;
        int wide = 0;
        for (int l = nlev - 2; l >= 0; --l) {            // the root level holds one entry: start below it
            const long long lo = idx * F;
            const int n = (int)min((long long)F, len[l] - lo);
            long long hit = lo + n - 1;                  // last child bounds u from above
            for (int c = 0; c < n; c += 32) {            // fanouts above 32: one ballot per 32 children
                const bool ok = c + lane < n && levels[off[l] + lo + c + lane] > uu;
                const unsigned b = __ballot_sync(kFull, ok);
                if (b) {
                    hit = lo + c + __ffs(b) - 1;
                    break;
                }
            }
            idx = hit;
            wide = max(wide, n);
        }
        if (lane == 0) {
            out[q] = idx;
            if (visited) visited[q] = nlev - 1;
            if (widest) widest[q] = wide;
        }
    }
}

template <typename T>
cudaError_t ptree_sample_t(const T* d_prefix, int64_t n, int F, const T* d_u, int64_t m, int64_t* d_idx,
                           int32_t* d_visited, int32_t* d_widest, cudaStream_t st) {
    std::vector<long long> off{0}, len{n};
    long long total = n;
    while (len.back() > 1) {
        const long long l = (len.back() + F - 1) / F;
        off.push_back(total);
        len.push_back(l);
        total += l;
    }
    T* lv = nullptr;
    long long* dmeta = nullptr;
    cudaError_t e = cudaMalloc(&lv, sizeof(T) * total);
    if (e != cudaSuccess) return e;
    e = cudaMalloc(&dmeta, sizeof(long long) * 2 * off.size());
    if (e == cudaSuccess) e = cudaMemcpyAsync(lv, d_prefix, sizeof(T) * n, cudaMemcpyDeviceToDevice, st);
    for (size_t l = 1; e == cudaSuccess && l < off.size(); ++l) {
        ptree_level_kernel<T><<<(unsigned)((len[l] + 255) / 256), 256, 0, st>>>(lv + off[l - 1], len[l - 1],
                                                                               lv + off[l], len[l], F);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(dmeta, off.data(), sizeof(long long) * off.size(), cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(dmeta + off.size(), len.data(), sizeof(long long) * len.size(), cudaMemcpyHostToDevice,
                            st);
    if (e == cudaSuccess && m > 0) {
        int dev = 0, sms = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        const long long blocks = std::min<long long>((m + 7) / 8, 8LL * std::max(sms, 1));
        ptree_sample_kernel<T><<<(unsigned)blocks, 256, 0, st>>>(lv, dmeta, dmeta + off.size(), (int)off.size(), F,
                                                                d_u, m, d_idx, d_visited, d_widest);
        e = cudaGetLastError();
    }
    const cudaError_t es = cudaStreamSynchronize(st);
    if (e == cudaSuccess) e = es;
    cudaFree(lv);
    if (dmeta) cudaFree(dmeta);
    return e;
}

cudaError_t ptree_sample(const float* d_prefix, int64_t n, int F, const float* d_u, int64_t m, int64_t* d_idx,
                         int32_t* d_visited, int32_t* d_widest, cudaStream_t st) {
    return ptree_sample_t<float>(d_prefix, n, F, d_u, m, d_idx, d_visited, d_widest, st);
}

cudaError_t ptree_sample_f64(const double* d_prefix, int64_t n, int F, const double* d_u, int64_t m, int64_t* d_idx,
                             int32_t* d_visited, int32_t* d_widest, cudaStream_t st) {
    return ptree_sample_t<double>(d_prefix, n, F, d_u, m, d_idx, d_visited, d_widest, st);
}

}  // namespace gf
