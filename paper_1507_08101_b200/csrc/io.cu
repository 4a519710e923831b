// Matrix file I/O (reference: /root/reference/proj/src/io.cpp).  Out of scope
// for this round: every synthetic configuration is
// generated on the device.  The entry points exist for link compatibility.
#include "objects.cuh"

namespace skb {

std::unique_ptr<Crs> crs_read_mm(const char*, Datatype) {
    fail(errc::unsupported, "Matrix Market input is not available in this build (SURVEY §8(f))");
}
std::unique_ptr<Crs> crs_read_bin(const char*) {
    fail(errc::unsupported, "GCRS input is not available in this build (SURVEY §8(f))");
}
void crs_write_bin(const char*, const Crs&, bool) {
    fail(errc::unsupported, "GCRS output is not available in this build (SURVEY §8(f))");
}

}  // namespace skb
