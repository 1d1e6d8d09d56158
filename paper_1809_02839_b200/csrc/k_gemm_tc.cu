// tcgen05 tensor-core GEMMs (placeholder until the TMA/TMEM kernel lands).
#include "kernels.hpp"

namespace st {
static thread_local int g_tc_launches = 0;
int tc_last_launches() { return g_tc_launches; }
int64_t tc_workspace_bytes(int, int, int) { return 256; }
st_status tc_fwd(const GemmArgs&, const float*, const float*, const float*, float*, int) {
  return set_error(ST_ERR_UNSUPPORTED, "tcgen05 GEMM not built yet");
}
st_status tc_dx(const GemmArgs&, const float*, const float*, const float*, float*) {
  return set_error(ST_ERR_UNSUPPORTED, "tcgen05 GEMM not built yet");
}
st_status tc_dw(const GemmArgs&, const float*, const float*, float*, float*) {
  return set_error(ST_ERR_UNSUPPORTED, "tcgen05 GEMM not built yet");
}
}  // namespace st
