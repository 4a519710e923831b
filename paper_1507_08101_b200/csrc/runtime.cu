// Per-device runtime: streams, scratch memory, sync policy, error mapping.
#include <cstdio>
#include <cstdlib>
#include <map>

#include "core.cuh"

namespace skb {

const char* errc_name(errc c) {
    switch (c) {
        case errc::ok: return "ok";
        case errc::invalid_arg: return "invalid argument";
        case errc::overflow: return "index overflow";
        case errc::shape_mismatch: return "shape mismatch";
        case errc::pattern_mismatch: return "sparsity pattern mismatch";
        case errc::io: return "io error";
        case errc::capacity: return "capacity exceeded";
        case errc::state: return "invalid state";
        case errc::alloc: return "allocation failure";
        case errc::transport: return "transport failure";
        case errc::unsupported: return "unsupported operation";
        case errc::numeric: return "numeric failure";
    }
    return "unknown";
}

void cuda_fail(cudaError_t e, const char* what, const char* file, int line) {
    cudaGetLastError();  // clear sticky-free errors
    char buf[512];
    std::snprintf(buf, sizeof(buf), "CUDA error %s (%s) in %s at %s:%d", cudaGetErrorName(e),
                  cudaGetErrorString(e), what, file, line);
    if (std::getenv("SELLKIT_VERBOSE")) std::fprintf(stderr, "[sellkit] %s\n", buf);
    if (e == cudaErrorMemoryAllocation) throw Error(errc::alloc, buf);
    throw Error(errc::state, buf);
}

DeviceBuffer::DeviceBuffer(std::size_t bytes, int device) : bytes_(bytes), device_(device) {
    if (bytes == 0) return;
    DeviceGuard g(device);
    CK(cudaMalloc(&ptr_, bytes));
}

DeviceBuffer DeviceBuffer::pooled(std::size_t bytes, int device) {
    DeviceBuffer b;
    b.bytes_ = bytes;
    b.device_ = device;
    if (bytes == 0) return b;
    DeviceGuard g(device);
    auto& rt = runtime(device);
    CK(cudaMallocFromPoolAsync(&b.ptr_, bytes, rt.mem_pool(), rt.stream));
    b.pooled_ = true;
    return b;
}

DeviceBuffer DeviceBuffer::cached(std::size_t bytes, int device) {
    DeviceBuffer b;
    b.bytes_ = bytes;
    b.device_ = device;
    if (bytes == 0) return b;
    DeviceGuard g(device);
    b.ptr_ = runtime(device).cache_take(bytes);
    if (!b.ptr_) CK(cudaMalloc(&b.ptr_, bytes));
    b.cached_ = true;
    return b;
}

void* DeviceRuntime::cache_take(std::size_t bytes) {
    std::lock_guard<std::mutex> lk(mu);
    for (std::size_t i = cache.size(); i-- > 0;) {
        if (cache[i].second == bytes) {
            void* p = cache[i].first;
            cache_bytes -= bytes;
            cache.erase(cache.begin() + std::ptrdiff_t(i));
            return p;
        }
    }
    return nullptr;
}

void DeviceRuntime::cache_put(void* p, std::size_t bytes) {
    std::lock_guard<std::mutex> lk(mu);
    if (cache_cap == 0) {
        std::size_t fr = 0, tot = 0;
        cudaMemGetInfo(&fr, &tot);
        cache_cap = std::max<std::size_t>(tot / 8, std::size_t(1) << 30);  // 22 GB on a B200
    }
    if (bytes > cache_cap) {
        cudaFree(p);
        return;
    }
    while (!cache.empty() && cache_bytes + bytes > cache_cap) {  // drop the oldest
        cudaFree(cache.front().first);
        cache_bytes -= cache.front().second;
        cache.erase(cache.begin());
    }
    cache.emplace_back(p, bytes);
    cache_bytes += bytes;
}

DeviceBuffer::~DeviceBuffer() {
    if (ptr_) {
        int prev = 0;
        cudaGetDevice(&prev);
        if (prev != device_) cudaSetDevice(device_);
        if (cached_) {
            cudaDeviceSynchronize();  // what cudaFree would order: nothing in flight still uses it
            runtime(device_).cache_put(ptr_, bytes_);
        } else if (pooled_) {
            // the same ordering cudaFree gives: nothing in flight on any stream of the device
            // may still use the memory when the pool hands it out again
            cudaDeviceSynchronize();
            cudaFreeAsync(ptr_, runtime(device_).stream);
        } else {
            cudaFree(ptr_);
        }
        if (prev != device_) cudaSetDevice(prev);
    }
}

cudaMemPool_t DeviceRuntime::mem_pool() {
    std::lock_guard<std::mutex> lk(mu);
    if (!pool) {
        cudaMemPoolProps props{};
        props.allocType = cudaMemAllocationTypePinned;
        props.location.type = cudaMemLocationTypeDevice;
        props.location.id = device;
        CK(cudaMemPoolCreate(&pool, &props));
        std::uint64_t keep = ~std::uint64_t(0);  // never trim at synchronisation points
        CK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
    }
    return pool;
}

int* DeviceRuntime::flag() {
    if (!flag_dev) {
        DeviceGuard g(device);
        CK(cudaMalloc(reinterpret_cast<void**>(&flag_dev), 256));
        CK(cudaMallocHost(reinterpret_cast<void**>(&flag_host), 256));
    }
    CK(cudaMemsetAsync(flag_dev, 0, sizeof(int), stream));
    return flag_dev;
}

int DeviceRuntime::read_flag() {
    CK(cudaMemcpyAsync(flag_host, flag_dev, sizeof(int), cudaMemcpyDeviceToHost, stream));
    CK(cudaStreamSynchronize(stream));
    return *flag_host;
}

void* DeviceRuntime::scratch_bytes(std::size_t n) {
    if (scratch.bytes() < n) {
        // previous users are stream-ordered on this stream; wait before freeing
        CK(cudaStreamSynchronize(stream));
        std::size_t want = std::max<std::size_t>(n, 1 << 20);
        scratch = DeviceBuffer(want, device);
    }
    return scratch.get();
}

void* DeviceRuntime::stage_bytes(int i, std::size_t n) {
    if (stage[i].bytes() < n) {
        CK(cudaDeviceSynchronize());
        stage[i] = DeviceBuffer();
        stage[i] = DeviceBuffer(n, device);
    }
    return stage[i].get();
}

void DeviceRuntime::copy_streams() {
    if (!h2d) {
        DeviceGuard g(device);
        CK(cudaStreamCreateWithFlags(&h2d, cudaStreamNonBlocking));
        CK(cudaStreamCreateWithFlags(&d2h, cudaStreamNonBlocking));
    }
}

void* DeviceRuntime::pinned_bytes_at_least(std::size_t n) {
    if (pinned_bytes < n) {
        CK(cudaStreamSynchronize(stream));
        if (pinned) cudaFreeHost(pinned);
        pinned = nullptr;
        std::size_t want = std::max<std::size_t>(n, 4096);
        CK(cudaMallocHost(&pinned, want));
        pinned_bytes = want;
    }
    return pinned;
}

namespace {
std::mutex g_mu;
std::map<int, DeviceRuntime*>& registry() {
    static auto* m = new std::map<int, DeviceRuntime*>();  // never destroyed: safe at exit
    return *m;
}
bool g_sync = true;
}  // namespace

int current_device() {
    int d = 0;
    CK(cudaGetDevice(&d));
    return d;
}

DeviceRuntime& runtime(int device) {
    std::lock_guard<std::mutex> lk(g_mu);
    auto& reg = registry();
    auto it = reg.find(device);
    if (it != reg.end()) return *it->second;
    auto* rt = new DeviceRuntime();
    rt->device = device;
    DeviceGuard g(device);
    // A *blocking* stream: work the caller queued on the legacy default stream (e.g. torch
    // filling a buffer passed through view_plain) completes before the library reads it,
    // and vice versa -- the reference API's synchronous semantics for device pointers.
    CK(cudaStreamCreateWithFlags(&rt->stream, cudaStreamDefault));
    CK(cudaDeviceGetAttribute(&rt->num_sms, cudaDevAttrMultiProcessorCount, device));
    int l2 = 0;
    CK(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, device));
    rt->l2_bytes = std::size_t(l2);
    // the build-temporary pool and the flag word exist from the first call on, and the pool
    // holds 64 MB from the start, so a first matrix build does not pay their creation
    {
        void* p = nullptr;
        CK(cudaMallocFromPoolAsync(&p, std::size_t(64) << 20, rt->mem_pool(), rt->stream));
        CK(cudaFreeAsync(p, rt->stream));
        rt->flag();
        CK(cudaStreamSynchronize(rt->stream));
    }
    reg[device] = rt;
    return *rt;
}

void release_cached_all() {
    std::vector<DeviceRuntime*> rts;
    {
        std::lock_guard<std::mutex> lk(g_mu);
        for (auto& kv : registry()) rts.push_back(kv.second);
    }
    for (auto* rt : rts) {
        DeviceGuard g(rt->device);
        CK(cudaDeviceSynchronize());
        std::lock_guard<std::mutex> lk(rt->mu);
        for (auto& e : rt->cache) cudaFree(e.first);
        rt->cache.clear();
        rt->cache_bytes = 0;
        if (rt->pool) CK(cudaMemPoolTrimTo(rt->pool, 0));
    }
}

namespace {
thread_local std::string t_last_error;
}
void set_last_error(const char* msg) { t_last_error = msg ? msg : ""; }
const char* last_error_message() { return t_last_error.c_str(); }

bool sync_mode() { return g_sync; }
void set_sync_mode(bool s) { g_sync = s; }

void finish(DeviceRuntime& rt) {
    CK(cudaGetLastError());
    if (g_sync) CK(cudaStreamSynchronize(rt.stream));
}

MemKind pointer_kind(const void* p, int* device_out) {
    cudaPointerAttributes attr{};
    cudaError_t e = cudaPointerGetAttributes(&attr, p);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return MemKind::host;
    }
    if (attr.type == cudaMemoryTypeDevice || attr.type == cudaMemoryTypeManaged) {
        if (device_out) *device_out = attr.device;
        return MemKind::device;
    }
    return MemKind::host;
}

namespace {
// Chunk heights with a dedicated warp-per-32-rows kernel (C divides 32) and
// block widths with a compile-time-unrolled kernel; see spmv.cu.
const int kChunkHeights[] = {4, 8, 32};  // == reference config/kernels.cfg:5
const int kBlockWidths[] = {1, 2, 4, 8, 16, 32, 64};
}  // namespace

const int* config_chunk_heights(std::size_t* n) {
    *n = sizeof(kChunkHeights) / sizeof(int);
    return kChunkHeights;
}
const int* config_block_widths(std::size_t* n) {
    *n = sizeof(kBlockWidths) / sizeof(int);
    return kBlockWidths;
}
lidx row_padding() {
    lidx p = 1;
    for (int c : kChunkHeights) p = std::max<lidx>(p, c);
    return p;
}

}  // namespace skb
