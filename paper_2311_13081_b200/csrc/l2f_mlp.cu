// placeholder, replaced by the tcgen05 MLP rollout
#include "l2f_internal.h"
namespace l2f {
int mlp_rollout_grid(int64_t) { return 1; }
cudaError_t launch_rollout_mlp(const DevParams&, const DevBufs&, const PolicyDev&, int32_t, float*, const int64_t*, int32_t, cudaStream_t) { return cudaErrorNotSupported; }
cudaError_t launch_policy_forward(const PolicyDev&, const float*, float*, int64_t, cudaStream_t) { return cudaErrorNotSupported; }
}
