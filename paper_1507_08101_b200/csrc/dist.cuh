// Row-distributed SpMMV with halo exchange (reference:
// /root/reference/proj/src/partition.hpp).  Declared here, implemented in dist.cu.
#pragma once

#include "objects.cuh"
#include "spmv.cuh"

namespace skb {}  // namespace skb
