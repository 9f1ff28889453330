// Host runtime of the engine: API errors, the process-wide caching allocator (device and
// pinned-host blocks, streams), the host worker pool that builds epoch plans, and the cache
// of instantiated epoch graphs.  Host-only; included by engine.cu.
#pragma once
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <array>
#include <atomic>
#include <condition_variable>
#include <cstdarg>
#include <cstdio>
#include <deque>
#include <future>
#include <functional>
#include <list>
#include <map>
#include <memory>
#include <mutex>
#include <random>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "esrnn_b200.h"
#include "mt64.h"

namespace esrnn_host {

// ------------------------------------------------------------------ errors
struct ApiError : std::runtime_error {
    esrnn_status code;
    ApiError(esrnn_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void raise(esrnn_status c, const char* fmt, ...) {
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    throw ApiError(c, buf);
}

#define CUDA_OK(expr)                                                                       \
    do {                                                                                    \
        cudaError_t e_ = (expr);                                                            \
        if (e_ != cudaSuccess) raise(ESRNN_CUDA_ERROR, "%s: %s (%s:%d)", #expr,             \
                                     cudaGetErrorString(e_), __FILE__, __LINE__);           \
    } while (0)
#define NCCL_OK(expr)                                                                       \
    do {                                                                                    \
        ncclResult_t r_ = (expr);                                                           \
        if (r_ != ncclSuccess) raise(ESRNN_NCCL_ERROR, "%s: %s", #expr, ncclGetErrorString(r_)); \
    } while (0)

inline thread_local std::string g_create_err;

// ------------------------------------------------------------------ host RNG
// matrix.hpp:173-213: std::mt19937_64 with explicit bit draws.
struct HostRng {
    Mt64 gen;  // == std::mt19937_64, with bulk draws
    explicit HostRng(uint64_t seed) : gen(seed) {}
    double uniform() { return static_cast<double>(gen() >> 11) * 0x1.0p-53; }
    double uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }
    uint64_t below(uint64_t n) { return static_cast<uint64_t>((static_cast<unsigned __int128>(gen()) * n) >> 64); }
};

// ------------------------------------------------------------------ caching allocator
// Process-wide free lists of device and pinned-host blocks, keyed by (device, size class).
// A freed buffer is kept for the next request of its class, so re-creating a trainer of
// the same configuration costs no cudaMalloc / cudaFree (which synchronise the device and
// can take milliseconds) and gets the same addresses back (which lets the epoch graph be
// reused, see GraphCache).  esrnn_release_cached_memory() returns the blocks to CUDA.
struct BlockCache {
    std::mutex mu;
    std::map<std::pair<int, size_t>, std::vector<void*>> dev, host;
    // (stream, event, event) triples per device: stream / event creation costs ~100 us
    std::map<int, std::vector<std::array<void*, 3>>> streams;
};
inline BlockCache& block_cache() {
    static BlockCache* c = new BlockCache;  // never destroyed: no CUDA calls at exit
    return *c;
}
inline size_t size_class(size_t bytes) { return (bytes + 4095) & ~static_cast<size_t>(4095); }
inline int current_device() {
    int d = 0;
    cudaGetDevice(&d);
    return d;
}
inline void* cache_get(bool host, size_t cls) {
    BlockCache& c = block_cache();
    const int dev = host ? -1 : current_device();
    {
        std::lock_guard<std::mutex> g(c.mu);
        auto& m = host ? c.host : c.dev;
        auto it = m.find({dev, cls});
        if (it != m.end() && !it->second.empty()) {
            void* p = it->second.back();
            it->second.pop_back();
            return p;
        }
    }
    void* p = nullptr;
    if (host)
        CUDA_OK(cudaMallocHost(&p, cls));
    else
        CUDA_OK(cudaMalloc(&p, cls));
    return p;
}
inline void cache_put(bool host, void* p, size_t cls) {
    BlockCache& c = block_cache();
    std::lock_guard<std::mutex> g(c.mu);
    (host ? c.host : c.dev)[{host ? -1 : current_device(), cls}].push_back(p);
}

// A trainer's stream and timing events, from the process-wide pool (created on a miss).
inline void stream_get(cudaStream_t& st, cudaEvent_t& a, cudaEvent_t& b) {
    BlockCache& c = block_cache();
    const int dev = current_device();
    {
        std::lock_guard<std::mutex> g(c.mu);
        auto& v = c.streams[dev];
        if (!v.empty()) {
            st = static_cast<cudaStream_t>(v.back()[0]);
            a = static_cast<cudaEvent_t>(v.back()[1]);
            b = static_cast<cudaEvent_t>(v.back()[2]);
            v.pop_back();
            return;
        }
    }
    CUDA_OK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    CUDA_OK(cudaEventCreate(&a));
    CUDA_OK(cudaEventCreate(&b));
}
inline void stream_put(cudaStream_t st, cudaEvent_t a, cudaEvent_t b) {
    BlockCache& c = block_cache();
    std::lock_guard<std::mutex> g(c.mu);
    c.streams[current_device()].push_back({static_cast<void*>(st), static_cast<void*>(a), static_cast<void*>(b)});
}

// ------------------------------------------------------------------ device buffer
inline std::atomic<uint64_t> g_alloc_seq{0};

template <typename T>
struct DBuf {
    T* p = nullptr;
    size_t n = 0;
    DBuf() = default;
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
    uint64_t seq = 0;  // allocation order (the owner frees in reverse, see release_buffers)
    void alloc(size_t count) {
        free();
        n = count;
        seq = ++g_alloc_seq;
        if (count) p = static_cast<T*>(cache_get(false, size_class(sizeof(T) * count)));
    }
    void zero(cudaStream_t s) {
        if (n) CUDA_OK(cudaMemsetAsync(p, 0, sizeof(T) * n, s));
    }
    void free() {
        if (p) cache_put(false, p, size_class(sizeof(T) * n));
        p = nullptr;
        n = 0;
    }
    ~DBuf() { free(); }
};

template <typename T>
struct PinnedBuf {
    T* p = nullptr;
    size_t n = 0;
    PinnedBuf() = default;
    PinnedBuf(const PinnedBuf&) = delete;
    PinnedBuf& operator=(const PinnedBuf&) = delete;
    PinnedBuf(PinnedBuf&& o) noexcept : p(o.p), n(o.n) { o.p = nullptr, o.n = 0; }
    PinnedBuf& operator=(PinnedBuf&& o) noexcept {
        if (this != &o) {
            release();
            p = o.p, n = o.n;
            o.p = nullptr, o.n = 0;
        }
        return *this;
    }
    void reserve(size_t count) {
        if (count <= n) return;
        release();
        p = static_cast<T*>(cache_get(true, size_class(sizeof(T) * count)));
        n = size_class(sizeof(T) * count) / sizeof(T);
    }
    void release() {
        if (p) cache_put(true, p, size_class(sizeof(T) * n));
        p = nullptr;
        n = 0;
    }
    ~PinnedBuf() { release(); }
};

// ------------------------------------------------------------------ host worker pool
// Persistent host threads for the epoch plan (parallel over step ranges); the calling
// thread takes tasks too.  One job at a time (run() is serialised).
struct WorkerPool {
    std::mutex run_mu, mu;
    std::condition_variable cv, done_cv;
    std::function<void(int)> job;
    int n_tasks = 0, next = 0, done = 0;
    uint64_t gen = 0;
    std::vector<std::thread> th;
    explicit WorkerPool(int n) {
        for (int i = 0; i < n; ++i) th.emplace_back([this] { loop(); });
    }
    void drain(std::unique_lock<std::mutex>& lk) {
        while (next < n_tasks) {
            const int i = next++;
            lk.unlock();
            job(i);
            lk.lock();
            if (++done == n_tasks) done_cv.notify_all();
        }
    }
    void loop() {
        uint64_t seen = 0;
        std::unique_lock<std::mutex> lk(mu);
        for (;;) {
            cv.wait(lk, [&] { return gen != seen; });
            seen = gen;
            drain(lk);
        }
    }
    void run(int n, const std::function<void(int)>& f) {
        std::lock_guard<std::mutex> serial(run_mu);
        std::unique_lock<std::mutex> lk(mu);
        job = f;
        n_tasks = n;
        next = done = 0;
        ++gen;
        cv.notify_all();
        drain(lk);
        done_cv.wait(lk, [&] { return done == n_tasks; });
    }
};
inline WorkerPool& worker_pool() {
    // never destroyed (threads park in cv.wait); sized to the host, at most 7 helpers
    static WorkerPool* p = new WorkerPool(static_cast<int>(
        std::max(1u, std::min(7u, std::thread::hardware_concurrency() > 1 ? std::thread::hardware_concurrency() - 1 : 1u))));
    return *p;
}
// Persistent helper threads for work handed off asynchronously (a trainer's first epoch
// plan, built while its creation finishes): starting a std::thread costs ~25 us on the
// creating thread, a hand-off here a few.
struct AsyncRunner {
    std::mutex mu;
    std::condition_variable cv;
    std::deque<std::function<void()>> q;
    std::vector<std::thread> th;
    explicit AsyncRunner(int n) {
        for (int i = 0; i < n; ++i) th.emplace_back([this] { loop(); });
    }
    void loop() {
        for (;;) {
            std::function<void()> f;
            {
                std::unique_lock<std::mutex> lk(mu);
                cv.wait(lk, [&] { return !q.empty(); });
                f = std::move(q.front());
                q.pop_front();
            }
            f();
        }
    }
    // runs f on a helper; the future is ready when f has returned (f must not throw)
    std::future<void> submit(std::function<void()> f) {
        auto done = std::make_shared<std::promise<void>>();
        std::future<void> fut = done->get_future();
        {
            std::lock_guard<std::mutex> g(mu);
            q.emplace_back([f = std::move(f), done] {
                f();
                done->set_value();
            });
        }
        cv.notify_one();
        return fut;
    }
};
inline AsyncRunner& async_runner() {
    static AsyncRunner* r = new AsyncRunner(2);  // never destroyed (threads park in cv.wait)
    return *r;
}

// stamp ids for slot dedupe: unique per planned step across the process (no re-init of
// the per-row stamp arrays between steps / epochs)
inline std::atomic<int64_t> g_stamp_id{1};

// ------------------------------------------------------------------ graph cache
// Epoch graphs keyed by the exact bytes of every launch argument they capture.  With the
// caching allocator a re-created trainer of the same configuration reproduces the key, and
// its first epoch replays the instantiated graph instead of capturing a new one.
struct GraphExec {
    cudaGraphExec_t g = nullptr;
    int launch_nodes = 0;
    ~GraphExec() {
        if (g) cudaGraphExecDestroy(g);
    }
};
struct GraphCache {
    std::mutex mu;
    std::list<std::pair<std::string, std::shared_ptr<GraphExec>>> lru;  // front = newest
    static constexpr size_t kMax = 16;
    std::shared_ptr<GraphExec> find(const std::string& key) {
        std::lock_guard<std::mutex> g(mu);
        for (auto it = lru.begin(); it != lru.end(); ++it)
            if (it->first == key) {
                lru.splice(lru.begin(), lru, it);
                return it->second;
            }
        return nullptr;
    }
    void insert(const std::string& key, std::shared_ptr<GraphExec> ge) {
        std::lock_guard<std::mutex> g(mu);
        lru.emplace_front(key, std::move(ge));
        if (lru.size() > kMax) lru.pop_back();  // live trainers keep their own reference
    }
    void clear() {
        std::lock_guard<std::mutex> g(mu);
        lru.clear();
    }
};
inline GraphCache& graph_cache() {
    static GraphCache* c = new GraphCache;  // never destroyed: no CUDA calls at exit
    return *c;
}
template <typename T>
inline void key_append(std::string& k, const T& v) {
    k.append(reinterpret_cast<const char*>(&v), sizeof v);
}

}  // namespace esrnn_host
