// Launch counting and per-kernel CUDA-event timing for bench.py (spct_cu_profile_*).
#include <atomic>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "spct_internal.h"

namespace spct_impl {

namespace {
std::atomic<uint64_t> g_launches{0};
std::atomic<int> g_prof{0};
std::mutex g_mu;
struct Rec {
    std::string name;
    cudaEvent_t a, b;
};
std::vector<Rec> g_recs;
std::vector<cudaEvent_t> g_pool;

cudaEvent_t take_event() {
    if (!g_pool.empty()) {
        cudaEvent_t e = g_pool.back();
        g_pool.pop_back();
        return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
}
}  // namespace

void note_launch(int n) { g_launches.fetch_add(static_cast<uint64_t>(n), std::memory_order_relaxed); }

int prof_begin(const char* name, cudaStream_t s) {
    if (!g_prof.load(std::memory_order_relaxed)) return -1;
    std::lock_guard<std::mutex> lk(g_mu);
    Rec r{name, take_event(), take_event()};
    cudaEventRecord(r.a, s);
    g_recs.push_back(r);
    return static_cast<int>(g_recs.size()) - 1;
}

void prof_end(int id, cudaStream_t s) {
    if (id < 0) return;
    std::lock_guard<std::mutex> lk(g_mu);
    cudaEventRecord(g_recs[id].b, s);
}

}  // namespace spct_impl

using namespace spct_impl;

extern "C" uint64_t spct_cu_launch_count(void) { return g_launches.load(); }

extern "C" void spct_cu_profile_enable(int on) { g_prof.store(on ? 1 : 0); }

extern "C" void spct_cu_profile_reset(void) {
    std::lock_guard<std::mutex> lk(g_mu);
    for (auto& r : g_recs) {
        g_pool.push_back(r.a);
        g_pool.push_back(r.b);
    }
    g_recs.clear();
}

extern "C" spct_status spct_cu_profile_read(const char* kernel, double* total_ms, int* launches) {
    std::lock_guard<std::mutex> lk(g_mu);
    double tot = 0.0;
    int n = 0;
    for (auto& r : g_recs) {
        if (r.name != kernel) continue;
        if (auto st = cuda_status(cudaEventSynchronize(r.b), "profile sync")) return st;
        float ms = 0.f;
        if (auto st = cuda_status(cudaEventElapsedTime(&ms, r.a, r.b), "profile elapsed")) return st;
        tot += ms;
        ++n;
    }
    if (total_ms) *total_ms = tot;
    if (launches) *launches = n;
    return SPCT_OK;
}

namespace spct_impl {

int current_device() {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) {
        cudaGetLastError();
        dev = 0;
    }
    return dev;
}

void ensure_smem(const void* func, size_t bytes) {
    static std::mutex mu;
    static std::map<std::pair<int, const void*>, size_t> done;
    const int dev = current_device();
    std::lock_guard<std::mutex> lock(mu);
    size_t& cur = done[{dev, func}];
    if (bytes <= cur || bytes <= 48 * 1024) return;
    cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes));
    cudaGetLastError();
    cur = bytes;
}

int per_device_int(int key, int (*compute)(int key)) {
    static std::mutex mu;
    static std::map<std::pair<int, int>, int> cache;
    const int dev = current_device();
    {
        std::lock_guard<std::mutex> lock(mu);
        auto it = cache.find({dev, key});
        if (it != cache.end()) return it->second;
    }
    const int v = compute(key);  // outside the lock: may itself call ensure_smem
    std::lock_guard<std::mutex> lock(mu);
    return cache.emplace(std::make_pair(dev, key), v).first->second;
}

cudaError_t malloc_async(void** p, size_t bytes, cudaStream_t s) {
    static std::mutex mu;
    static bool done[64] = {};
    int dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess && dev >= 0 && dev < 64) {
        std::lock_guard<std::mutex> lock(mu);
        if (!done[dev]) {
            cudaMemPool_t pool;
            if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
                uint64_t keep = ~0ull;
                cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
            }
            cudaGetLastError();
            done[dev] = true;
        }
    }
    return cudaMallocAsync(p, bytes, s);
}

}  // namespace spct_impl
