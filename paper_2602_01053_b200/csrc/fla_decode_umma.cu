// fla_decode_umma.cu -- tcgen05 / TMA batched-decode kernel (placeholder until the kernel lands).
#include "kernels.hpp"
#include "state.hpp"

namespace lk {
bool decode_umma_supported(const PagedAttnCall&) { return false; }
int launch_decode_umma(const PagedAttnCall&) { return fail("decode_umma: not built"); }
}  // namespace lk
