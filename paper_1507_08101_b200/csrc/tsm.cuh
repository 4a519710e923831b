// Tall-skinny dense kernels (reference: /root/reference/proj/src/tsm.hpp).
#pragma once

#include "objects.cuh"

namespace skb {

// X(m x k) = alpha * V^H W + beta * X   (tsm.hpp:105-178)
void tsmttsm(DenseMat& x, const DenseMat& v, const DenseMat& w, const void* alpha, const void* beta, bool kahan);
// W(n x k) = alpha * V X + beta * W     (tsm.hpp:182-225)
void tsmm(DenseMat& w, const DenseMat& v, const DenseMat& x, const void* alpha, const void* beta);
// V(n x m) = alpha * V X + beta * V     (tsm.hpp:230-249)
void tsmm_inplace(DenseMat& v, const DenseMat& x, const void* alpha, const void* beta);

// FP64 tensor-core paths (tsm_mma.cu) for compact row-major double operands;
// return false / 0 when the shape is not covered.
bool tsmm_dmma(double* w, const double* v, const double* xcm, gidx n, int m, int k, double alpha, double beta,
               bool beta_zero, DeviceRuntime& rt);
int tsmttsm_dmma_partials(const double* v, const double* w, gidx n, int m, int k, double* part, int max_parts,
                          DeviceRuntime& rt);

enum class Trans { none = 0, transpose = 1, conj_transpose = 2 };
// gemm router (tsm.hpp:281-305)
void gemm(DenseMat& c, const DenseMat& a, const DenseMat& b, const void* alpha, const void* beta, Trans ta, Trans tb);

}  // namespace skb
