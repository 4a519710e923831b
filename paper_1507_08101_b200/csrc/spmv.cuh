// Fused SELL-C-sigma SpMV / SpMMV: y = alpha*(A - gamma*I)*x + beta*y with
// optional <y,y>, <x,y>, <x,x> per column and z = delta*z + eta*y
// (reference: /root/reference/proj/src/spmv.hpp:13-202, spmv_epilogue.hpp:12-36).
#pragma once

#include "objects.cuh"

namespace skb {

// spmv_args.hpp:10-17 (mirrored in sellkit.h)
constexpr std::uint32_t kFlagAxpby = 1u << 0;
constexpr std::uint32_t kFlagShift = 1u << 1;
constexpr std::uint32_t kFlagVshift = 1u << 2;
constexpr std::uint32_t kFlagDotYY = 1u << 3;
constexpr std::uint32_t kFlagDotXY = 1u << 4;
constexpr std::uint32_t kFlagDotXX = 1u << 5;
constexpr std::uint32_t kFlagChain = 1u << 6;
constexpr std::uint32_t kFlagAll = (1u << 7) - 1;
constexpr std::uint32_t kFlagDots = kFlagDotYY | kFlagDotXY | kFlagDotXX;

// Host-side option record (spmv.hpp:16-26).  Scalars are raw element bytes
// (up to a complex double); gamma_list / dot are caller pointers.
struct SpmvOptions {
    std::uint32_t flags = 0;
    unsigned char alpha[16] = {}, beta[16] = {}, gamma[16] = {}, delta[16] = {}, eta[16] = {};
    const void* gamma_list = nullptr;  // host or device, width elements
    DenseMat* z = nullptr;
    void* dot = nullptr;  // host or device, 3*width elements; only requested thirds written
};

// Resolve the default-or-given scalars of sellkit_spmv_opts (capi.cpp:124-140).
void spmv_options_from(Datatype dt, std::uint32_t flags, const void* alpha, const void* beta, const void* gamma,
                       const void* delta, const void* eta, SpmvOptions& o);

// Which kernel runs for this shape (spmv.hpp:47-62 semantics over this build's
// configuration); 0 = generic dimension.
struct KernelVariant {
    int chunk_height = 0;
    int block_width = 0;
    bool vectorized = false;
};
KernelVariant select_kernel(lidx chunk_height, lidx block_width, Order order);

// Optional hooks used by the distributed driver: rows whose bit is set in
// `defer_mask` (per stored row) skip the dots and the chain in this sweep
// because a later sweep (the remote part) finalises them; `row_map` makes a
// sweep write rows row_map[k] instead of k (remote sweep over boundary rows).
struct SpmvHooks {
    const std::uint32_t* defer_mask = nullptr;
    const lidx* row_map = nullptr;
    bool accumulate_dots = false;  // add into `dot_accum` device buffer instead of writing `dot`
    void* dot_accum = nullptr;     // device, 3*width
    cudaStream_t stream = nullptr; // override the runtime stream
    const DenseMat* x_self = nullptr;  // x of the output rows for shift/dots when x is a halo block
    gidx rg0 = 0, rg1 = -1;            // row groups (32 stored rows) to sweep; rg1 < 0: all
    int reserve_sms = 0;               // leave this many SMs to concurrent work (halo pack)
    void* scratch = nullptr;           // caller-owned device scratch (>= spmv_scratch_bytes);
    std::size_t scratch_size = 0;      // else the runtime's shared scratch
};

// Device scratch one spmv_device call of width `width` needs (gamma list, dots, partials).
std::size_t spmv_scratch_bytes(Datatype dt, lidx width, int num_sms);

// Validation only (spmv.hpp:98-125): throws the reference's error codes.
void spmv_validate(const DenseMat& y, const SellMat& A, const DenseMat& x, const SpmvOptions& opts);
// Validation (spmv.hpp:98-125) + launch.  y/x/z may be host-resident views.
void spmv(DenseMat& y, const SellMat& A, const DenseMat& x, const SpmvOptions& opts);
// Device-only entry used by the distributed path (no validation, no staging).
void spmv_device(DenseMat& y, const SellMat& A, const DenseMat& x, const SpmvOptions& opts, const SpmvHooks& hooks);

}  // namespace skb
