// Core types of the B200 sellkit library: error codes (mirroring the reference's
// errc, /root/reference/proj/src/error.hpp:8-21), index widths
// (types.hpp:13-15), scalar traits for the four element types, device buffers
// and the per-device runtime (stream, scratch, sync policy).
#pragma once

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <cstdint>
#include <cstring>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

namespace skb {

using gidx = std::int64_t;  // global row/column/slot index (types.hpp:13)
using lidx = std::int32_t;  // rank-local row/column index (types.hpp:15)

enum class errc : int {
    ok = 0,
    invalid_arg = 1,
    overflow = 2,
    shape_mismatch = 3,
    pattern_mismatch = 4,
    io = 5,
    capacity = 6,
    state = 7,
    alloc = 8,
    transport = 9,
    unsupported = 10,
    numeric = 11,
};

const char* errc_name(errc c);

class Error : public std::runtime_error {
public:
    Error(errc code, const std::string& msg) : std::runtime_error(msg), code_(code) {}
    errc code() const noexcept { return code_; }

private:
    errc code_;
};

[[noreturn]] inline void fail(errc code, const std::string& msg) { throw Error(code, msg); }

#define SK_REQUIRE(cond, code, msg)               \
    do {                                          \
        if (!(cond)) ::skb::fail((code), (msg));  \
    } while (0)

// CUDA failures: out-of-memory maps to SELLKIT_ERR_ALLOC, everything else to
// SELLKIT_ERR_STATE (the reference has no device, so no dedicated code).
void cuda_fail(cudaError_t e, const char* what, const char* file, int line);
#define CK(call)                                                           \
    do {                                                                   \
        cudaError_t _e = (call);                                           \
        if (_e != cudaSuccess) ::skb::cuda_fail(_e, #call, __FILE__, __LINE__); \
    } while (0)

// narrow_index types.hpp:18-22
inline lidx narrow_index(gidx g) {
    SK_REQUIRE(g >= 0, errc::invalid_arg, "negative index");
    SK_REQUIRE(g < (gidx(1) << 31), errc::overflow, "index does not fit the 32-bit local range");
    return static_cast<lidx>(g);
}

enum class Datatype : int { r32 = 0, r64 = 1, c32 = 2, c64 = 3 };

inline std::size_t value_bytes(Datatype dt) {
    switch (dt) {
        case Datatype::r32: return 4;
        case Datatype::r64: return 8;
        case Datatype::c32: return 8;
        case Datatype::c64: return 16;
    }
    return 0;
}
inline bool is_complex(Datatype dt) { return dt == Datatype::c32 || dt == Datatype::c64; }

// Interleaved complex numbers with the layout of std::complex<R>.
template <class R>
struct alignas(2 * sizeof(R)) cplx {
    R re, im;
};
using cfloat = cplx<float>;
using cdouble = cplx<double>;

template <class T>
struct scalar_traits;
template <>
struct scalar_traits<float> {
    using real = float;
    static constexpr bool is_complex = false;
    static constexpr Datatype dt = Datatype::r32;
};
template <>
struct scalar_traits<double> {
    using real = double;
    static constexpr bool is_complex = false;
    static constexpr Datatype dt = Datatype::r64;
};
template <>
struct scalar_traits<cfloat> {
    using real = float;
    static constexpr bool is_complex = true;
    static constexpr Datatype dt = Datatype::c32;
};
template <>
struct scalar_traits<cdouble> {
    using real = double;
    static constexpr bool is_complex = true;
    static constexpr Datatype dt = Datatype::c64;
};

// Dispatch a generic lambda over the runtime datatype: f.template operator()<T>().
template <class F>
decltype(auto) visit_dt(Datatype dt, F&& f) {
    switch (dt) {
        case Datatype::r32: return f.template operator()<float>();
        case Datatype::r64: return f.template operator()<double>();
        case Datatype::c32: return f.template operator()<cfloat>();
        case Datatype::c64: return f.template operator()<cdouble>();
    }
    fail(errc::invalid_arg, "unknown datatype");
}

// ------------------------------------------------------------ device memory --

// Owning device allocation (cudaMalloc; 256-B aligned, so every vector load
// width used by the kernels is legal on owned buffers).
class DeviceBuffer {
public:
    DeviceBuffer() = default;
    DeviceBuffer(std::size_t bytes, int device);
    ~DeviceBuffer();
    DeviceBuffer(const DeviceBuffer&) = delete;
    DeviceBuffer& operator=(const DeviceBuffer&) = delete;
    DeviceBuffer(DeviceBuffer&& o) noexcept { swap(o); }
    DeviceBuffer& operator=(DeviceBuffer&& o) noexcept {
        DeviceBuffer t(std::move(o));
        swap(t);
        return *this;
    }
    // Stream-ordered allocation from the device's library pool (SELL storage and build
    // temporaries): freed memory stays in the pool, so a rebuild or a value refresh makes
    // no driver allocation.  Not for memory that is exported through CUDA IPC.
    static DeviceBuffer pooled(std::size_t bytes, int device);
    // cudaMalloc'ed, but returned to a per-device cache on destruction and reused by the next
    // request of the same size (SELL storage: a rebuild or a second matrix of the same shape
    // makes no driver allocation; the cache is bounded, DeviceRuntime::cache_*).
    static DeviceBuffer cached(std::size_t bytes, int device);
    void* get() const { return ptr_; }
    template <class T>
    T* as() const { return static_cast<T*>(ptr_); }
    std::size_t bytes() const { return bytes_; }
    int device() const { return device_; }
    void swap(DeviceBuffer& o) noexcept {
        std::swap(ptr_, o.ptr_);
        std::swap(bytes_, o.bytes_);
        std::swap(device_, o.device_);
        std::swap(pooled_, o.pooled_);
        std::swap(cached_, o.cached_);
    }

private:
    void* ptr_ = nullptr;
    std::size_t bytes_ = 0;
    int device_ = 0;
    bool pooled_ = false;
    bool cached_ = false;
};

// ------------------------------------------------------------------ runtime --

// Per-device execution resources.  All library work on a device is enqueued on
// its one non-blocking stream; in the default synchronous mode every public
// call synchronises that stream before returning (the reference's calls are
// synchronous, SURVEY §8(b) "Threading").
struct DeviceRuntime {
    int device = 0;
    cudaStream_t stream = nullptr;
    int num_sms = 0;
    std::size_t l2_bytes = 0;
    // scratch for reductions (grown on demand, stream-ordered reuse)
    DeviceBuffer scratch;
    void* pinned = nullptr;  // small pinned staging area for dot results
    std::size_t pinned_bytes = 0;
    std::mutex mu;
    // copy streams + device staging of the streamed host-buffer spmv (spmv.cu)
    cudaStream_t h2d = nullptr, d2h = nullptr;
    DeviceBuffer stage[3];
    void* stage_bytes(int i, std::size_t n);
    void copy_streams();

    void* scratch_bytes(std::size_t n);
    void* pinned_bytes_at_least(std::size_t n);
    cudaMemPool_t pool = nullptr;  // DeviceBuffer::pooled (created on first use, keeps its memory)
    // DeviceBuffer::cached: freed (pointer, bytes), most recent last, at most cache_cap bytes
    std::vector<std::pair<void*, std::size_t>> cache;
    std::size_t cache_bytes = 0, cache_cap = 0;
    void* cache_take(std::size_t bytes);
    void cache_put(void* p, std::size_t bytes);
    cudaMemPool_t mem_pool();
    // one device word + its pinned host mirror for error flags / small readbacks
    int* flag_dev = nullptr;
    int* flag_host = nullptr;
    int* flag();                     // zeroed on the stream, ready for a kernel to OR into
    int read_flag();                 // synchronises the stream
};

DeviceRuntime& runtime(int device);
void release_cached_all();  // DeviceRuntime caches and pools of every device -> driver
int current_device();
void set_last_error(const char* msg);  // per-thread message of the last failed C-ABI call
const char* last_error_message();
bool sync_mode();          // true: public calls synchronise before returning
void set_sync_mode(bool);

// RAII device switch
struct DeviceGuard {
    int prev = 0;
    explicit DeviceGuard(int dev) {
        CK(cudaGetDevice(&prev));
        if (prev != dev) CK(cudaSetDevice(dev));
    }
    ~DeviceGuard() { cudaSetDevice(prev); }
};

void finish(DeviceRuntime& rt);  // sync if sync_mode(), else check launch errors

// NVTX range (host side) around a library phase: visible in Nsight timelines, a no-op
// without a tool attached.
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

// Where does a caller pointer live?
enum class MemKind { device, host };
MemKind pointer_kind(const void* p, int* device_out);

// Specialisation dimensions of this build (the analogue of
// config/kernels.cfg:5-6).  Row padding of owned block vectors uses the largest
// chunk height (densemat.hpp:202-208).
const int* config_chunk_heights(std::size_t* n);
const int* config_block_widths(std::size_t* n);
lidx row_padding();

}  // namespace skb
