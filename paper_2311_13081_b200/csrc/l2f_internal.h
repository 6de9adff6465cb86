// l2f_internal.h -- host-side declarations shared by the ABI and the kernel translation units.
#pragma once
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>

#include "l2f_device.cuh"

namespace l2f {

// Per-device bookkeeping of host launchers (function attributes and SM counts are per device;
// a process may drive several).  Device ordinals < 64.
inline int current_device()
{
    int dev = 0;
    cudaGetDevice(&dev);
    return dev & 63;
}

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) for `func` on the current device once per
// requested size: `done` holds the largest size set so far on each device.
template <class F>
inline cudaError_t ensure_smem_attr(F* func, size_t bytes, std::atomic<size_t> (&done)[64])
{
    const int dev = current_device();
    if (done[dev].load() >= bytes) return cudaSuccess;
    const cudaError_t e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e == cudaSuccess) done[dev].store(bytes);
    return e;
}

#ifndef L2F_STEP_BLOCK
#define L2F_STEP_BLOCK 128  // step-kernel block (measured at C3: 64 -> 88.2 us, 128 -> 87.0, 256 -> 91.4)
#endif
constexpr int kStepBlock = L2F_STEP_BLOCK;
constexpr int kRolloutBlock = 128;

struct StepOutDev {
    float* obs_core;
    float* obs_dense;
    float* reward;
    uint8_t* flags;
    float* final_state;
    float* obs_critic;  // [28][N] privileged critic observation (NEXT f1)
};

// Actor MLP parameters on the device (fp16 bits, row-major [out][in]).
struct PolicyDev {
    const uint16_t *W1, *b1, *W2, *b2, *W3, *b3;
    int32_t in_dim, hidden;
};

cudaError_t launch_step(const DevParams& P, const DevBufs& B, const float* act, const StepOutDev& O,
                        cudaStream_t s);
cudaError_t launch_step_plain(const DevParams& P, const DevBufs& B, const float* act, const StepOutDev& O,
                              cudaStream_t s);
cudaError_t launch_reset(const DevParams& P, const DevBufs& B, const uint8_t* mask, const StepOutDev& O,
                         cudaStream_t s);
cudaError_t launch_rollout_open(const DevParams& P, const DevBufs& B, const float* act, int32_t T, float* trace,
                                const int64_t* trace_ids, int32_t K, cudaStream_t s);
cudaError_t launch_philox_selftest(int64_t n, uint64_t seed, uint32_t t, uint32_t* ours, uint32_t* ref,
                                   cudaStream_t s);
cudaError_t launch_recompute_rewards(const StageW& W, const float* next_state, const float* actions, int64_t m,
                                     float* rewards, cudaStream_t s);
// Bytes of workspace scratch the statistics finalize needs (per-block partials + a ticket).
size_t stats_finalize_scratch_bytes();
cudaError_t launch_stats_finalize(double* slots, int32_t n_slots, void* scratch, double* out, int32_t reset,
                                  double host_steps, cudaStream_t s);

// tcgen05 actor-MLP rollout (l2f_mlp.cu).  Returns cudaErrorNotSupported for unsupported shapes.
int mlp_rollout_grid(int64_t n);
cudaError_t launch_rollout_mlp(const DevParams& P, const DevBufs& B, const PolicyDev& W, int32_t T, float* trace,
                               const int64_t* trace_ids, int32_t K, cudaStream_t s);
cudaError_t launch_policy_forward(const PolicyDev& W, const float* obs, float* act, int64_t n, cudaStream_t s);

// Lissajous tracking evaluation (l2f_track): per-env cycle times in, per-env RMSE out.
struct TrackDev {
    const float* cycle_time;               // [N]
    float ax, ay, z, clip_pos, clip_vel;   // reference and setpoint-shift clipping
    float hover_rpm, hover_a;              // start rotor speed and history fill
    int32_t n_steps, terminate;            // steps; termination test on the error state (Q31)
    float *rmse, *rmse_xy;                 // [N]
    int32_t* steps_ok;                     // [N]
};
cudaError_t launch_track_mlp(const DevParams& P, const DevBufs& B, const PolicyDev& W, const TrackDev& S,
                             cudaStream_t s);

// Batched TD3 update (l2f_td3.cu): one CTA per agent, CTA-wide batch GEMMs.
struct TD3Dev {
    float* params;          // [A][block] flat FP32 blocks (td3_block_floats)
    float* scratch;         // [A][scratch_floats]
    float* losses;          // [A][3]
    const float *o_a, *o_c, *a, *r, *o_a2, *o_c2, *done, *eps;  // [A][B][...]
    int64_t block, scratch_floats;
    int32_t n_agents, B, in_dim, update_actor;
    float gamma, tau, sigma_t, clip_t, lr_actor, lr_critic, beta1, beta2, adam_eps;
    float c1_critic, c2_critic, c1_actor, c2_actor;  // Adam bias corrections 1 - beta^t
};
int td3_max_in_dim();
int64_t td3_block_floats(int in_dim);
int64_t td3_scratch_bytes(int in_dim, int B);
cudaError_t launch_td3_update(const TD3Dev& A, cudaStream_t s);
cudaError_t launch_td3_export_actor(const float* params, int64_t block, int agent, int in_dim, uint16_t* out,
                                    cudaStream_t s);

}  // namespace l2f
