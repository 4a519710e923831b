// Definitions of the opaque C handles of sellkit.h / sellkit_ext.h.
#pragma once

#include <memory>
#include <string>
#include <vector>

#include "dist.cuh"
#include "objects.cuh"
#include "sellkit.h"
#include "sellkit_ext.h"

struct sellkit_crs {
    std::unique_ptr<skb::Crs> p;
};
struct sellkit_mat {
    std::unique_ptr<skb::SellMat> p;
    // matrix-free replacement of the multiply (sellcs.hpp:116-119 apply_override)
    sellkit_ext_apply_fn apply_override = nullptr;
    void* apply_ctx = nullptr;
};
struct sellkit_densemat {
    skb::DenseMat m;
};
struct sellkit_region {
    std::string name;
    std::vector<double> samples;
};
struct sellkit_ctx {
    std::unique_ptr<skb::DistContext> p;
};
struct sellkit_dvec {
    std::unique_ptr<skb::DistVec> p;
};
struct sellkit_rankctx {
    skb::RankContext* p = nullptr;
};

namespace skb {

// exception -> error code at the C boundary (capi.cpp:50-62)
template <class F>
sellkit_error guarded(F&& f) noexcept {
    try {
        f();
        return SELLKIT_OK;
    } catch (const Error& e) {
        if (std::getenv("SELLKIT_VERBOSE")) std::fprintf(stderr, "[sellkit] %s\n", e.what());
        set_last_error(e.what());
        return static_cast<sellkit_error>(static_cast<int>(e.code()));
    } catch (const std::bad_alloc&) {
        set_last_error("allocation failure");
        return SELLKIT_ERR_ALLOC;
    } catch (const std::exception& e) {
        set_last_error(e.what());
        return SELLKIT_ERR_INVALID_ARG;
    } catch (...) {
        set_last_error("unknown exception");
        return SELLKIT_ERR_INVALID_ARG;
    }
}

inline void require(bool cond, const char* msg) {
    if (!cond) fail(errc::invalid_arg, msg);
}

inline Datatype dt_from(sellkit_datatype dt) {
    switch (dt) {
        case SELLKIT_R32: return Datatype::r32;
        case SELLKIT_R64: return Datatype::r64;
        case SELLKIT_C32: return Datatype::c32;
        case SELLKIT_C64: return Datatype::c64;
    }
    fail(errc::invalid_arg, "unknown datatype");
}

inline Order order_from(sellkit_order o) { return o == SELLKIT_ROW_MAJOR ? Order::row_major : Order::col_major; }

inline void same_dt(Datatype a, Datatype b, const char* what) {
    if (a != b) fail(errc::invalid_arg, std::string("datatype mismatch between ") + what);
}

// sellkit_spmv_opts -> SpmvOptions (capi.cpp:124-140)
inline void options_from_c(Datatype dt, const sellkit_spmv_opts* opts, SpmvOptions& o) {
    if (opts) {
        spmv_options_from(dt, opts->flags, opts->alpha, opts->beta, opts->gamma, opts->delta, opts->eta, o);
        o.dot = opts->dot;
        if (opts->z) {
            same_dt(dt, opts->z->m.dt, "y and z");
            o.z = &opts->z->m;
        }
    } else {
        spmv_options_from(dt, 0, nullptr, nullptr, nullptr, nullptr, nullptr, o);
    }
}

}  // namespace skb
