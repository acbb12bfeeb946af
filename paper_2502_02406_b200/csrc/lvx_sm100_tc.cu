// placeholder until the tcgen05 backward lands: bwd runs on the SIMT kernels
#include "lvx_common.cuh"
namespace lvx {
bool tc_bwd_eligible(const lvx_view*, const lvx_view*, const lvx_view*) { return false; }
size_t tc_bwd_workspace(const lvx_view*, const lvx_view*) { return 0; }
int tc_bwd(const lvx_view*, const lvx_view*, const lvx_view*, const lvx_view*, const lvx_view*,
           const lvx_view*, double, const lvx_view*, const lvx_view*, const lvx_view*, int, void*,
           size_t, cudaStream_t) {
  return LVX_EUNSUPPORTED;
}
}  // namespace lvx
