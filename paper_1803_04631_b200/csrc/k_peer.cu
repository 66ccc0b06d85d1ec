// Peer-memory phi exchange: the replica sum of SPEC
// `reduce_phi`/`broadcast_phi` over NVLink/NVSwitch
// peer memory instead of an NCCL allreduce.
//
// Every rank's sync buffer (hybrid u32/u16 phi columns + n_k, `gf_sync_layout`)
// is exported with cudaIpcGetMemHandle and mapped by every other rank of the
// node.  One kernel per iteration, launched right after K2 on the shard's
// stream, does the whole collective ("two-shot" in one launch):
//   start barrier  block b of rank r tells block b of every rank that r's K2
//                  output is complete (release store into the peer's signal
//                  slot) and waits for the same word from all of them;
//   reduce         block b sums its part of slab r (rank r owns words
//                  [r*n/G, (r+1)*n/G)) over the G replicas with 16-byte peer
//                  loads and stores the sum into all G replicas;
//   end barrier    block b tells block b of every rank that its part of slab r
//                  is written everywhere and waits for all of them.
// Block b of every rank covers the same relative positions of its slab, so
// when all blocks of rank r pass the end barrier every slab chunk has landed in
// r's replica; a rank's next K2 (which clears the buffer) cannot start before
// its exchange kernel returns, i.e. before every peer has finished reading it.
// Counts are integers: the packed u16 pairs of light columns sum without
// carries because a light word's global frequency is <= the heavy threshold.
// Bytes per rank: reads (G-1)/G and writes (G-1)/G of the buffer over the
// links, the same as a ring allreduce's 2(G-1)/G, in one launch and without
// NCCL's staging copies.  A block waits only for blocks of OTHER ranks, so no
// co-residency is needed on a device; a wait that exceeds the timeout sets an
// error word and the host reports it (no hang on a dead peer).
#include "gf_internal.cuh"
#include "gf_device.cuh"
#include "../../include/gibbsflow_b200.h"

#include <algorithm>
#include <cstring>
#include <vector>

namespace gf {

namespace {

constexpr int kPeerBlocks = 296;          // 2 per SM
constexpr int kPeerThreads = 512;
constexpr unsigned long long kPeerTimeoutNs = 20ull * 1000 * 1000 * 1000;

struct PeerArgs {
    uint32_t* buf[kMaxPeers];     // every rank's sync buffer (own included)
    uint32_t* sig[kMaxPeers];     // every rank's signal slots [2][kPeerBlocks][kMaxPeers]
    int rank, world;
    int64_t n;                    // u32 words in the buffer
    uint32_t epoch;
    unsigned long long* err;      // own errs[3]: block that timed out (min)
};


// block-level barrier with the same-index block of every rank; phase 0/1
__device__ bool peer_barrier(const PeerArgs& a, int phase) {
    __syncthreads();
    bool ok = true;
    const int t = threadIdx.x;
    if (t < a.world) {
        const size_t slot = ((size_t)phase * kPeerBlocks + blockIdx.x) * kMaxPeers;
        __threadfence_system();
        st_release_sys(a.sig[t] + slot + a.rank, a.epoch);
        const uint32_t* mine = a.sig[a.rank] + slot + t;
        const unsigned long long t0 = now_ns();
        while ((int32_t)(ld_acquire_sys(mine) - a.epoch) < 0) {
            if (now_ns() - t0 > kPeerTimeoutNs) {
                atomicMin(a.err, (unsigned long long)blockIdx.x);
                ok = false;
                break;
            }
            __nanosleep(64);
        }
    }
    return __syncthreads_and(ok);
}

__global__ void __launch_bounds__(kPeerThreads) peer_allreduce_kernel(PeerArgs a) {
    if (!peer_barrier(a, 0)) return;
    const int64_t lo = a.n * a.rank / a.world, hi = a.n * (a.rank + 1) / a.world;
    // 16-byte body over 4-aligned word indices, scalar head and tail
    const int64_t v0 = (lo + 3) >> 2, v1 = hi >> 2;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (int64_t v = v0 + gid; v < v1; v += stride) {
        uint4 s = make_uint4(0, 0, 0, 0);
        for (int p = 0; p < a.world; ++p) {
            const uint4 x = __ldcg(reinterpret_cast<const uint4*>(a.buf[p]) + v);
            s.x += x.x; s.y += x.y; s.z += x.z; s.w += x.w;
        }
        for (int p = 0; p < a.world; ++p) __stcg(reinterpret_cast<uint4*>(a.buf[p]) + v, s);
    }
    const int64_t h1 = v0 * 4 < hi ? v0 * 4 : hi, t0 = v1 * 4 > lo ? v1 * 4 : lo;
    for (int64_t i = lo + gid; i < h1; i += stride) {   // head words before the first vector
        uint32_t s = 0;
        for (int p = 0; p < a.world; ++p) s += __ldcg(a.buf[p] + i);
        for (int p = 0; p < a.world; ++p) __stcg(a.buf[p] + i, s);
    }
    for (int64_t i = (t0 > h1 ? t0 : h1) + gid; i < hi; i += stride) {   // tail words
        uint32_t s = 0;
        for (int p = 0; p < a.world; ++p) s += __ldcg(a.buf[p] + i);
        for (int p = 0; p < a.world; ++p) __stcg(a.buf[p] + i, s);
    }
    peer_barrier(a, 1);
}

}  // namespace

// [barrier phase 0 | barrier phase 1] of the two-shot kernel, then the fused
// K2X kernel's stripe / done flags (k_counts.cu)
size_t peer_signal_bytes() { return (size_t)3 * kPeerBlocks * kMaxPeers * sizeof(uint32_t); }

void peer_close(gf_shard* s) {
    PeerGroup& g = s->peer;
    for (int p = 0; p < g.world; ++p) {
        if (p == g.rank) continue;
        if (g.buf[p]) cudaIpcCloseMemHandle(g.buf[p]);
        if (g.sig[p]) cudaIpcCloseMemHandle(g.sig[p]);
    }
    if (g.own_sig) cudaFree(g.own_sig);
    if (g.xdev) cudaFree(g.xdev);
    g = PeerGroup{};
}

int peer_handle(gf_shard* s, void* out) {
    PeerGroup& g = s->peer;
    if (!g.own_sig) {
        cudaError_t e = cudaMalloc((void**)&g.own_sig, peer_signal_bytes());
        if (e == cudaSuccess) e = cudaMemset(g.own_sig, 0, peer_signal_bytes());
        if (e != cudaSuccess) return shard_cuda_fail(e, "peer_handle");
        g.epoch = 0;
    }
    cudaIpcMemHandle_t h[2];
    cudaError_t e = cudaIpcGetMemHandle(&h[0], s->d.sync);
    if (e == cudaSuccess) e = cudaIpcGetMemHandle(&h[1], g.own_sig);
    if (e != cudaSuccess) return shard_cuda_fail(e, "peer_handle");
    std::memcpy(out, h, sizeof h);
    return 0;
}

// K2X set-up: stripes of ~1 MiB (<= 32) over the phi region, the work items
// re-ordered by the first buffer word they write (the stripes then complete in
// order while K2 runs), and the number of items touching each stripe
static int fused_setup(gf_shard* s) {
    PeerGroup& g = s->peer;
    g.sig_fused = (size_t)2 * kPeerBlocks * kMaxPeers;
    const long long nphi = s->off_nk_u32;
    g.nstripe = (int)std::max<long long>(1, std::min<long long>(32, nphi / (1 << 18)));
    g.stripe_words = std::max<long long>(1, (nphi + g.nstripe - 1) / g.nstripe);
    const int KW = s->Kp >> 1;
    auto first_word = [&](const int4& w) {
        return w.x >= 0 ? (long long)s->off_phi16_u32 + (long long)w.x * KW : (long long)(~w.x) * s->K;
    };
    std::vector<int4> items((size_t)s->n_k2);
    cudaError_t e = cudaSuccess;
    if (s->n_k2) e = cudaMemcpy(items.data(), s->d.k2items, items.size() * sizeof(int4), cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return shard_cuda_fail(e, "peer_open (items)");
    std::stable_sort(items.begin(), items.end(),
                     [&](const int4& a, const int4& b) { return first_word(a) < first_word(b); });
    std::vector<unsigned> need((size_t)g.nstripe, 0u);
    for (const int4& w : items) {
        const long long fw = first_word(w), lw = fw + (w.x >= 0 ? KW : s->K) - 1;
        const long long s0 = fw / g.stripe_words, s1 = std::min<long long>(g.nstripe - 1, lw / g.stripe_words);
        for (long long q = s0; q <= s1; ++q) ++need[(size_t)q];
    }
    if (s->n_k2) e = cudaMemcpy(s->d.k2items, items.data(), items.size() * sizeof(int4), cudaMemcpyHostToDevice);
    if (e == cudaSuccess && !g.xdev) e = cudaMalloc((void**)&g.xdev, (size_t)(2 * 32 + 2) * sizeof(unsigned));
    if (e == cudaSuccess) e = cudaMemcpy(g.xdev, need.data(), need.size() * sizeof(unsigned), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return shard_cuda_fail(e, "peer_open (stripes)");
    return 0;
}

int peer_open(gf_shard* s, int rank, int world, const void* handles) {
    PeerGroup& g = s->peer;
    if (world < 1 || world > kMaxPeers || rank < 0 || rank >= world)
        return shard_fail(GF_ERR_VALUE, "peer group: rank %d of %d outside [0, %d)", rank, world, kMaxPeers);
    if (!g.own_sig) return shard_fail(GF_ERR_VALUE, "peer group: gf_shard_peer_handle first");
    for (int p = 0; p < g.world; ++p)   // reopen: drop the previous mappings, keep the signal slots
        if (p != g.rank) {
            if (g.buf[p]) cudaIpcCloseMemHandle(g.buf[p]);
            if (g.sig[p]) cudaIpcCloseMemHandle(g.sig[p]);
        }
    for (int p = 0; p < kMaxPeers; ++p) g.buf[p] = g.sig[p] = nullptr;
    g.rank = rank;
    g.world = world;
    g.sync = s->d.sync;
    const auto* h = static_cast<const cudaIpcMemHandle_t*>(handles);
    for (int p = 0; p < world; ++p) {
        if (p == rank) {
            g.buf[p] = s->d.sync;
            g.sig[p] = g.own_sig;
            continue;
        }
        void *b = nullptr, *q = nullptr;
        cudaError_t e = cudaIpcOpenMemHandle(&b, h[2 * p], cudaIpcMemLazyEnablePeerAccess);
        if (e == cudaSuccess) e = cudaIpcOpenMemHandle(&q, h[2 * p + 1], cudaIpcMemLazyEnablePeerAccess);
        if (e != cudaSuccess) {
            if (b) cudaIpcCloseMemHandle(b);
            g.world = p;   // close what was opened so far
            peer_close(s);
            return shard_cuda_fail(e, "peer_open (cudaIpcOpenMemHandle)");
        }
        g.buf[p] = static_cast<uint32_t*>(b);
        g.sig[p] = static_cast<uint32_t*>(q);
    }
    return fused_setup(s);
}

cudaError_t launch_peer_allreduce(gf_shard* s, cudaStream_t st) {
    PeerGroup& g = s->peer;
    PeerArgs a{};
    for (int p = 0; p < g.world; ++p) {
        a.buf[p] = g.buf[p];
        a.sig[p] = g.sig[p];
    }
    a.rank = g.rank;
    a.world = g.world;
    a.n = s->sync_u32;
    a.epoch = ++g.epoch;
    a.err = s->d.errs + 3;
    peer_allreduce_kernel<<<kPeerBlocks, kPeerThreads, 0, st>>>(a);
    return cudaGetLastError();
}

}  // namespace gf
