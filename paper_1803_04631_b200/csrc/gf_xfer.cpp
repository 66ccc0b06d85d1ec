// gf_xfer.cpp -- large host <-> device copies of the one-call API
// (get/set of assignments, theta CSR, phi) for PAGEABLE numpy arrays.
//
// cudaMemcpy from / to pageable memory runs at ~11-17 GB/s on the B200 box
// (the driver stages through its own small pinned buffers, one CPU thread
// copying and taking every first-touch page fault of a fresh numpy array),
// while pinned DMA runs at ~55 GB/s each way.  Here a transfer is cut into
// 16 MiB pieces that alternate between two pinned bounce buffers: the host
// side of piece i (a memcpy split over a small persistent thread pool, which
// also spreads the page faults) overlaps the DMA of piece i-1.  Pinned (or
// registered) host pointers skip the bounce and DMA directly; small copies
// use one plain cudaMemcpyAsync.
#include <cuda_runtime.h>

#include <algorithm>
#include <condition_variable>
#include <cstdint>
#include <cstring>
#include <functional>
#include <iterator>
#include <map>
#include <mutex>
#include <thread>
#include <vector>

namespace gf {

namespace {

constexpr size_t kPiece = 16u << 20;     // bytes per bounce piece
constexpr size_t kSmall = 2u << 20;      // below this: one plain copy

// fixed pool of memcpy workers: run(n, f) calls f(i) for i in [0, n) over the
// workers and the calling thread, returning when all are done
class Pool {
  public:
    Pool() {
        unsigned hw = std::thread::hardware_concurrency();
        nw_ = std::max(1u, std::min(hw ? hw / 2 : 4u, 8u));
        for (unsigned i = 0; i + 1 < nw_; ++i) th_.emplace_back([this] { loop(); });
    }
    ~Pool() {
        {
            std::lock_guard<std::mutex> g(mu_);
            stop_ = true;
        }
        cv_.notify_all();
        for (auto& t : th_) t.join();
    }
    unsigned size() const { return nw_; }
    void run(unsigned n, const std::function<void(unsigned)>& f) {
        std::unique_lock<std::mutex> g(mu_);
        job_ = &f;
        next_ = 0;
        total_ = n;
        done_ = 0;
        ++gen_;
        cv_.notify_all();
        g.unlock();
        work();
        g.lock();
        done_cv_.wait(g, [&] { return done_ == total_; });
        job_ = nullptr;
    }

  private:
    void work() {
        while (true) {
            unsigned i;
            const std::function<void(unsigned)>* f;
            {
                std::lock_guard<std::mutex> g(mu_);
                if (!job_ || next_ >= total_) return;
                i = next_++;
                f = job_;
            }
            (*f)(i);
            std::lock_guard<std::mutex> g(mu_);
            if (++done_ == total_) done_cv_.notify_all();
        }
    }
    void loop() {
        uint64_t seen = 0;
        while (true) {
            {
                std::unique_lock<std::mutex> g(mu_);
                cv_.wait(g, [&] { return stop_ || (gen_ != seen && job_ && next_ < total_); });
                if (stop_) return;
                seen = gen_;
            }
            work();
        }
    }
    unsigned nw_ = 1;
    std::vector<std::thread> th_;
    std::mutex mu_;
    std::condition_variable cv_, done_cv_;
    const std::function<void(unsigned)>* job_ = nullptr;
    unsigned next_ = 0, total_ = 0, done_ = 0;
    uint64_t gen_ = 0;
    bool stop_ = false;
};

void par_copy(Pool& pool, char* dst, const char* src, size_t n) {
    const unsigned parts = (unsigned)std::min<size_t>(pool.size(), std::max<size_t>(1, n >> 20));
    if (parts <= 1) { std::memcpy(dst, src, n); return; }
    pool.run(parts, [&](unsigned i) {
        const size_t a = n * i / parts, b = n * (i + 1) / parts;
        std::memcpy(dst + a, src + a, b - a);
    });
}

struct Staging {
    std::mutex mu;                        // one transfer at a time per process
    char* buf[2] = {nullptr, nullptr};
    cudaEvent_t ev[2] = {nullptr, nullptr};
    int device = -1;
    Pool* pool = nullptr;
    cudaError_t ensure() {
        if (!pool) pool = new Pool();
        int dev = 0;
        cudaGetDevice(&dev);
        if (buf[0] && device == dev) return cudaSuccess;
        // events belong to a device: recreate when the caller's device changed
        for (auto& e : ev)
            if (e) { cudaEventDestroy(e); e = nullptr; }
        for (auto& e : ev) {
            cudaError_t r = cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
            if (r != cudaSuccess) return r;
        }
        for (auto& b : buf)
            if (!b) {
                cudaError_t r = cudaHostAlloc((void**)&b, kPiece, cudaHostAllocPortable);
                if (r != cudaSuccess) return r;
            }
        device = dev;
        return cudaSuccess;
    }
};

Staging& staging() {
    static Staging* s = new Staging();    // process lifetime (pinned buffers, pool threads)
    return *s;
}

bool is_pinned(const void* p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

// Pinned blocks for the result arrays of the one-call API (host_alloc /
// host_free, gf_host_alloc in the ABI).  A numpy result array in pageable
// memory costs a first-touch page fault per 4 KB page on every call (the
// array is new each time) plus the bounce copy; a pinned block is DMA'd
// into directly, and a freed block is kept for the next call of a similar
// size (best fit within 1.5x), so a training loop through the API stops
// faulting after its first iteration.  The cache holds at most kCacheCap
// bytes of free blocks; larger frees go back to the driver.
constexpr size_t kHostGrain = 2u << 20;
constexpr size_t kCacheCap = 16ull << 30;

struct HostCache {
    std::mutex mu;
    std::multimap<size_t, void*> free_blocks;   // rounded size -> block
    size_t cached = 0;
};

HostCache& host_cache() {
    static HostCache* c = new HostCache();      // process lifetime
    return *c;
}

}  // namespace

bool host_is_pinned(const void* p) { return is_pinned(p); }

size_t host_block_bytes(size_t n) { return std::max<size_t>(kHostGrain, (n + kHostGrain - 1) / kHostGrain * kHostGrain); }

cudaError_t host_alloc(size_t n, void** out) {
    const size_t want = host_block_bytes(n);
    HostCache& C = host_cache();
    {
        std::lock_guard<std::mutex> g(C.mu);
        auto it = C.free_blocks.lower_bound(want);
        if (it != C.free_blocks.end() && it->first <= want + want / 2) {
            *out = it->second;
            C.cached -= it->first;
            C.free_blocks.erase(it);
            return cudaSuccess;
        }
    }
    return cudaHostAlloc(out, want, cudaHostAllocPortable);
}

// `n` is the size passed to host_alloc for this block
cudaError_t host_free(void* p, size_t n) {
    if (!p) return cudaSuccess;
    const size_t sz = host_block_bytes(n);
    HostCache& C = host_cache();
    std::vector<void*> drop;
    {
        std::lock_guard<std::mutex> g(C.mu);
        // a block reused from the cache may be larger than host_block_bytes(n):
        // it is filed under the size it was looked up with, which only under-
        // states it (best fit keeps working)
        C.free_blocks.emplace(sz, p);
        C.cached += sz;
        while (C.cached > kCacheCap && !C.free_blocks.empty()) {   // evict the largest
            auto it = std::prev(C.free_blocks.end());
            C.cached -= it->first;
            drop.push_back(it->second);
            C.free_blocks.erase(it);
        }
    }
    cudaError_t e = cudaSuccess;
    for (void* q : drop) {
        cudaError_t r = cudaFreeHost(q);
        if (r != cudaSuccess) e = r;
    }
    return e;
}

// host -> device; returns when the host buffer may be reused (the DMA of the
// last piece may still be in flight on `st`, ordered before later work on it)
cudaError_t xfer_h2d(void* dst, const void* src, size_t n, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    if (n < kSmall || is_pinned(src)) {
        cudaError_t e = cudaMemcpyAsync(dst, src, n, cudaMemcpyHostToDevice, st);
        if (e == cudaSuccess && n < kSmall) e = cudaStreamSynchronize(st);   // pageable small: src reusable
        return e;
    }
    Staging& S = staging();
    std::lock_guard<std::mutex> g(S.mu);
    cudaError_t e = S.ensure();
    if (e != cudaSuccess) return e;
    const char* s = static_cast<const char*>(src);
    char* d = static_cast<char*>(dst);
    size_t off = 0;
    for (int i = 0; off < n && e == cudaSuccess; ++i, off += kPiece) {
        const size_t len = std::min(kPiece, n - off);
        const int b = i & 1;
        e = cudaEventSynchronize(S.ev[b]);                    // the DMA that last read this buffer
        if (e != cudaSuccess) break;
        par_copy(*S.pool, S.buf[b], s + off, len);
        e = cudaMemcpyAsync(d + off, S.buf[b], len, cudaMemcpyHostToDevice, st);
        if (e == cudaSuccess) e = cudaEventRecord(S.ev[b], st);
    }
    return e;
}

// device -> host; synchronous (the host data is complete on return)
cudaError_t xfer_d2h(void* dst, const void* src, size_t n, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    if (n < kSmall || is_pinned(dst)) {
        cudaError_t e = cudaMemcpyAsync(dst, src, n, cudaMemcpyDeviceToHost, st);
        return e == cudaSuccess ? cudaStreamSynchronize(st) : e;
    }
    Staging& S = staging();
    std::lock_guard<std::mutex> g(S.mu);
    cudaError_t e = S.ensure();
    if (e != cudaSuccess) return e;
    const char* s = static_cast<const char*>(src);
    char* d = static_cast<char*>(dst);
    const size_t pieces = (n + kPiece - 1) / kPiece;
    auto issue = [&](size_t i) {
        const size_t off = i * kPiece, len = std::min(kPiece, n - off);
        cudaError_t r = cudaMemcpyAsync(S.buf[i & 1], s + off, len, cudaMemcpyDeviceToHost, st);
        return r == cudaSuccess ? cudaEventRecord(S.ev[i & 1], st) : r;
    };
    e = issue(0);
    for (size_t i = 0; i < pieces && e == cudaSuccess; ++i) {
        e = cudaEventSynchronize(S.ev[i & 1]);
        // the next piece's DMA goes into the other buffer, whose host copy
        // (piece i-1) finished in the previous iteration
        if (e == cudaSuccess && i + 1 < pieces) e = issue(i + 1);
        if (e != cudaSuccess) break;
        const size_t off = i * kPiece, len = std::min(kPiece, n - off);
        par_copy(*S.pool, d + off, S.buf[i & 1], len);
    }
    return e;
}

}  // namespace gf
