// Row-distributed SpMMV (reference: /root/reference/proj/src/partition.hpp).
// Placeholder entry points; the implementation lands in the next commit.
#include "dist.cuh"
#include "sellkit.h"

extern "C" {
sellkit_error sellkit_partition_compute(sellkit_gidx, const sellkit_lidx*, const double*, int, sellkit_weight_mode,
                                        sellkit_gidx*) { return SELLKIT_ERR_UNSUPPORTED; }
sellkit_error sellkit_ctx_create(const sellkit_crs*, const double*, int, sellkit_weight_mode, int, int, int,
                                 sellkit_ctx** out) { if (out) *out = nullptr; return SELLKIT_ERR_UNSUPPORTED; }
sellkit_error sellkit_ctx_rank_range(const sellkit_ctx*, int, sellkit_gidx*, sellkit_gidx*) { return SELLKIT_ERR_UNSUPPORTED; }
sellkit_error sellkit_ctx_halo_size(const sellkit_ctx*, int, sellkit_lidx*) { return SELLKIT_ERR_UNSUPPORTED; }
sellkit_error sellkit_ctx_comm_stats(const sellkit_ctx*, uint64_t*, uint64_t*) { return SELLKIT_ERR_UNSUPPORTED; }
sellkit_error sellkit_ctx_reset_comm_stats(sellkit_ctx*) { return SELLKIT_ERR_UNSUPPORTED; }
void sellkit_ctx_destroy(sellkit_ctx*) {}
sellkit_error sellkit_dvec_create(const sellkit_ctx*, sellkit_lidx, sellkit_order, sellkit_dvec** out) { if (out) *out = nullptr; return SELLKIT_ERR_UNSUPPORTED; }
sellkit_error sellkit_dvec_scatter(const sellkit_ctx*, const sellkit_densemat*, sellkit_dvec*) { return SELLKIT_ERR_UNSUPPORTED; }
sellkit_error sellkit_dvec_gather(const sellkit_ctx*, const sellkit_dvec*, sellkit_densemat*) { return SELLKIT_ERR_UNSUPPORTED; }
void sellkit_dvec_destroy(sellkit_dvec*) {}
sellkit_error sellkit_dist_spmv(sellkit_dvec*, sellkit_ctx*, const sellkit_dvec*, const sellkit_spmv_opts*, sellkit_dist_mode,
                                sellkit_dvec*, int) { return SELLKIT_ERR_UNSUPPORTED; }
sellkit_error sellkit_spmv_nocomm(sellkit_dvec*, sellkit_ctx*, const sellkit_dvec*, const sellkit_spmv_opts*, sellkit_dvec*) { return SELLKIT_ERR_UNSUPPORTED; }
}
