// Instantiation unit of the SpMV kernels for one element type (split for parallel builds).
#include "spmv_kernels.cuh"

namespace skb {

template <>
spmv_detail::LaunchShape launch_spmv<cdouble>(const KArgs<cdouble>& a, bool specialised_ok, DeviceRuntime& rt,
                                         cudaStream_t st, lidx max_chunk_len) {
    return spmv_detail::launch_any<cdouble>(a, specialised_ok, rt, st, max_chunk_len);
}

}  // namespace skb
