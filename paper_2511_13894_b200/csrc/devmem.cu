// devmem.cu — libcpd's device-memory cache (the allocator behind DBuf).
//
// A problem creation allocates and frees ~10 GB in a few dozen buffers on C5 (CSR
// copies, SELL copies, plans, sort scratch).  cudaMalloc / cudaFree of multi-GB
// buffers map and unmap pages each time, and right after a large free the next
// creation's allocations ran 3-8x slower (profiles/r02_s4_create_phases.txt: 805 /
// 899 / 302 ms for three back-to-back creations).  Freed buffers are therefore kept
// per device in exact-size bins and handed out again; a buffer is reused only after a
// cudaDeviceSynchronize (work of every stream that could still touch it has finished
// — the guarantee cudaFree gives implicitly), and a failed cudaMalloc releases the
// whole cache and retries once.  The cache holds at most CPD_MEMCACHE_MB (default: a
// quarter of the device memory) of idle buffers; CPD_MEMCACHE=0 bypasses it.
#include <cuda_runtime.h>

#include <cstdlib>
#include <map>
#include <mutex>
#include <vector>

namespace cpd {

namespace {
struct Cache {
    std::mutex mu;
    std::multimap<size_t, void*> bins[64];   // per device: bytes -> idle buffers
    size_t held[64] = {};
    size_t cap[64] = {};
    bool cap_set[64] = {};
};
Cache& cache()
{
    static Cache* c = new Cache();   // never destroyed: frees may run during static teardown
    return *c;
}
bool enabled()
{
    static const bool on = [] {
        const char* e = getenv("CPD_MEMCACHE");
        return !(e && e[0] == '0');
    }();
    return on;
}
size_t cap_of(int dev, Cache& c)
{
    if (!c.cap_set[dev]) {
        size_t cap = 0;
        if (const char* e = getenv("CPD_MEMCACHE_MB")) {
            cap = (size_t)atoll(e) << 20;
        } else {
            size_t fr = 0, tot = 0;
            if (cudaMemGetInfo(&fr, &tot) == cudaSuccess) cap = tot / 4;
        }
        c.cap[dev] = cap;
        c.cap_set[dev] = true;
    }
    return c.cap[dev];
}
void release_all(int dev, Cache& c)
{
    for (auto& kv : c.bins[dev]) cudaFree(kv.second);
    c.bins[dev].clear();
    c.held[dev] = 0;
}
}  // namespace

cudaError_t dev_alloc(void** p, size_t bytes)
{
    if (!enabled()) return cudaMalloc(p, bytes);
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) return cudaMalloc(p, bytes);
    Cache& c = cache();
    {
        std::lock_guard<std::mutex> g(c.mu);
        auto it = c.bins[dev].find(bytes);
        if (it != c.bins[dev].end()) {
            // the buffer's last users (any stream) must be done before it is handed out
            const cudaError_t e = cudaDeviceSynchronize();
            if (e != cudaSuccess) return e;
            *p = it->second;
            c.held[dev] -= bytes;
            c.bins[dev].erase(it);
            return cudaSuccess;
        }
    }
    cudaError_t e = cudaMalloc(p, bytes);
    if (e == cudaErrorMemoryAllocation) {
        cudaGetLastError();   // clear the sticky-free error state of this call
        {
            std::lock_guard<std::mutex> g(c.mu);
            cudaDeviceSynchronize();
            release_all(dev, c);
        }
        e = cudaMalloc(p, bytes);
    }
    return e;
}

void dev_free(void* p, size_t bytes)
{
    if (!p) return;
    if (!enabled()) {
        cudaFree(p);
        return;
    }
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) {
        cudaFree(p);
        return;
    }
    Cache& c = cache();
    std::lock_guard<std::mutex> g(c.mu);
    const size_t cap = cap_of(dev, c);
    if (bytes > cap) {
        cudaFree(p);
        return;
    }
    // evict the largest idle buffers until this one fits under the cap
    while (c.held[dev] + bytes > cap && !c.bins[dev].empty()) {
        auto it = std::prev(c.bins[dev].end());
        cudaFree(it->second);
        c.held[dev] -= it->first;
        c.bins[dev].erase(it);
    }
    c.bins[dev].emplace(bytes, p);
    c.held[dev] += bytes;
}

// Release every idle buffer of the current device (cpd_release_cached_memory).
void dev_trim()
{
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) return;
    Cache& c = cache();
    std::lock_guard<std::mutex> g(c.mu);
    cudaDeviceSynchronize();
    release_all(dev, c);
}

size_t dev_cached_bytes()
{
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) return 0;
    Cache& c = cache();
    std::lock_guard<std::mutex> g(c.mu);
    return c.held[dev];
}

}  // namespace cpd
