// placeholder until the tcgen05 kernels land
#include "lvx_common.cuh"
namespace lvx {
bool tc_fwd_eligible(const lvx_view*, const lvx_view*, const lvx_view*) { return false; }
size_t tc_fwd_workspace(const lvx_view*, const lvx_view*) { return 0; }
int tc_fwd_partial(const lvx_view*, const lvx_view*, const lvx_view*, double, void*, size_t,
                   cudaStream_t) {
  return LVX_EUNSUPPORTED;
}
int tc_fwd_finish(const lvx_view*, const lvx_view*, const lvx_view*, const lvx_view*,
                  const lvx_view*, const lvx_view*, void*, size_t, cudaStream_t) {
  return LVX_EUNSUPPORTED;
}
bool tc_bwd_eligible(const lvx_view*, const lvx_view*, const lvx_view*) { return false; }
size_t tc_bwd_workspace(const lvx_view*, const lvx_view*) { return 0; }
int tc_bwd(const lvx_view*, const lvx_view*, const lvx_view*, const lvx_view*, const lvx_view*,
           const lvx_view*, double, const lvx_view*, const lvx_view*, const lvx_view*, int, void*,
           size_t, cudaStream_t) {
  return LVX_EUNSUPPORTED;
}
}  // namespace lvx
