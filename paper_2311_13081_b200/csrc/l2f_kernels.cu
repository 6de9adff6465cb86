// l2f_kernels.cu -- single-step, reset, open-loop rollout and statistics kernels (sm_100a).
//
// Data layout: structure-of-arrays [C][N] fp32 in HBM, one env per
// thread, so every component load/store of a warp is one fully-coalesced 128-byte line.
// Step kernel bytes per env-step (algorithmic): reads state 68 + action 16 +
// disturbance 24 + counters 8 (+ DR 20), writes state 68 + counters 8 + history slot 16 +
// obs_core 72 + reward 4 + flags 1.
#include <curand_philox4x32_x.h>

#ifndef L2F_STEP_MINB
#define L2F_STEP_MINB 6  // resident 128-thread blocks per SM the register budget targets (4: 96 us, 5: 88, 6: 87, 7: 91, 8: 97 at C3)
#endif

#include "l2f_device.cuh"
#include "l2f_internal.h"

namespace l2f {

template <bool kDR>
__device__ __forceinline__ void load_env(const DevParams& P, const DevBufs& B, int64_t i, EnvReg& e)
{
    grp_load<kStateDim>(B.state, i, P.n, e.s);
    grp_load<6>(B.dist, i, P.n, e.dist);
    if (kDR) {
        grp_load<5>(B.dr, i, P.n, e.dr);
    } else {
#pragma unroll
        for (int c = 0; c < 5; ++c) e.dr[c] = 1.0f;
    }
    e.ep_step = B.ep_step[i];
    e.ep_return = B.ep_return[i];
}

// Placeholder env for lanes past N: keeps warps convergent (shuffles, warp-cooperative reset).
__device__ __forceinline__ void dummy_env(EnvReg& e)
{
#pragma unroll
    for (int c = 0; c < kStateDim; ++c) e.s[c] = 0.0f;
    e.s[3] = 1.0f;
#pragma unroll
    for (int c = 0; c < 6; ++c) e.dist[c] = 0.0f;
#pragma unroll
    for (int c = 0; c < 5; ++c) e.dr[c] = 1.0f;
    e.ep_step = 0;
    e.ep_return = 0.0f;
}

__device__ __forceinline__ void store_state(const DevParams& P, const DevBufs& B, int64_t i, const EnvReg& e)
{
    grp_store<kStateDim>(B.state, i, P.n, e.s);
    B.ep_step[i] = e.ep_step;
    B.ep_return[i] = e.ep_return;
}

// Written only when an episode starts (reset): disturbance + DR factors.
__device__ __forceinline__ void store_episode_consts(const DevParams& P, const DevBufs& B, int64_t i,
                                                     const EnvReg& e)
{
    grp_store<6>(B.dist, i, P.n, e.dist);
    if (P.flags & F_DOMAIN_RAND) grp_store<5>(B.dr, i, P.n, e.dr);
}

// A new episode starting at step t0: O(1) bytes (marker + fill value), the ring itself is
// overwritten lazily by the episode's own actions (Q10).
__device__ __forceinline__ void hist_restart(const DevParams& P, const DevBufs& B, int64_t i, uint32_t t0,
                                             const float h[4])
{
    B.hist_t0[i] = (int32_t)t0;
    B.hist_fill[i] = make_float4(h[0], h[1], h[2], h[3]);
}

// Dense actor observation row [18 + 4 N_H]: obs_core then H most-recent-first at
// step t_next (the step this observation feeds).
__device__ __forceinline__ void write_dense(const DevParams& P, const DevBufs& B, int64_t i,
                                           const float ob[kObsCore], uint32_t t_next, float* row)
{
    const int64_t N = P.n;
#pragma unroll
    for (int j = 0; j < kObsCore; ++j) row[j] = ob[j];
    const int32_t t0 = B.hist_t0[i];
    for (int k = 0; k < P.n_hist; ++k) {
        float h[4];
        hist_entry(B, N, P.n_hist, i, (int64_t)t_next, k, t0, h);
#pragma unroll
        for (int c = 0; c < 4; ++c) row[kObsCore + 4 * k + c] = h[c];
    }
}

__device__ __forceinline__ void stats_block_end(const StatPk& st, double* srow, double steps, double* slot)
{
    L2F_CHECK(blockIdx.x < gridDim.x, "statistics slot");
    const int warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    statpk_warp_to_smem(st, srow + warp * kStatsLen);  // (unconditional: straight-line code)
    // producer/consumer named barrier: warps 1.. arrive and retire at once, warp 0 waits for
    // the rows and writes the block's slot (the block's SM slot frees up sooner than with a
    // full __syncthreads)
    if (warp == 0) {
        asm volatile("bar.sync 1, %0;" ::"r"(blockDim.x) : "memory");
        stat_rows_to_slot(srow, nw, steps, slot);
    } else {
        asm volatile("bar.arrive 1, %0;" ::"r"(blockDim.x) : "memory");
    }
}

// ---------------------------------------------------------------------------------------
// l2f_step: one transition for every env.
// ---------------------------------------------------------------------------------------
// kF: the feature flags as a compile-time set (kAnyFlags: read P.flags).  kStdOut: the outputs are
// exactly obs_core + reward + flags (the common request), so the output tests fold away.
template <bool kDR, uint32_t kF = kAnyFlags, bool kStdOut = false>
__global__ void __launch_bounds__(kStepBlock, L2F_STEP_MINB) step_kernel(const DevParams P, const DevBufs B,
                                                          const float* __restrict__ act, const StepOutDev O)
{
    const uint32_t flags = flags_of<kF>(P);
    const bool want_final = !kStdOut && O.final_state, want_core = kStdOut || O.obs_core;
    const bool want_dense = !kStdOut && O.obs_dense, want_critic = !kStdOut && O.obs_critic;
    const bool want_reward = kStdOut || O.reward, want_flags = kStdOut || O.flags;
    __shared__ double srow[(kStepBlock / 32) * kStatsLen];
    __shared__ uint4 rscratch[(kStepBlock / 32) * kResetScratch];  // cooperative reset scratch per warp
    const int64_t N = P.n;
    const int64_t i = (int64_t)blockIdx.x * kStepBlock + threadIdx.x;
    const bool active = i < N;
    const uint32_t t = P.t0;
    const uint32_t gid = P.id_offset + (uint32_t)i;
    StatPk st;
    statpk_zero(st);
    EnvReg e;
    float a[4] = {0.f, 0.f, 0.f, 0.f};
    if (active) {
        load_env<kDR>(P, B, i, e);
        soa_load_ro<4>(act, i, (uint32_t)N, a);
    } else {
        dummy_env(e);
    }
    Trans o;
    float za[4];
    action_noise<kF>(P, gid, t, za);
    transition<kDR, kF>(P, stage_of(P, t), e, gid, t, a, za, o);
    uint32_t fl = o.flags;
    if (active && want_final) {
        soa_store<kStateDim>(O.final_state, i, (uint32_t)N, e.s);
    }
    const bool ended = active && (fl & (D_TERM | D_TRUNC));
    statpk_episode(st, o, ended);
    bool did_reset = false;
    float hf[4];
    if (flags & F_AUTO_RESET) {
        did_reset = reset_env_warp<kDR ? 8 : 6, kF>(P, nullptr, e, gid, t + 1, ended, hf,
                                                    rscratch + (threadIdx.x >> 5) * kResetScratch);
        if (did_reset) fl |= D_RESET;
    } else if (ended) {
        e.ep_step = 0;
        e.ep_return = 0.0f;
    }
    if (active) {
        if (P.n_hist > 0) {
            const int slot = P.hist_slot0;  // t0 mod N_H (written for every env: deterministic ring)
            L2F_CHECK(slot >= 0 && slot < P.n_hist, "history slot");
            B.hist[(int64_t)slot * N + i] = make_float4(o.a[0], o.a[1], o.a[2], o.a[3]);
            if (did_reset) hist_restart(P, B, i, t + 1, hf);
        }
        store_state(P, B, i, e);
        if (did_reset) store_episode_consts(P, B, i, e);
        if (want_core || want_dense) {
            float ob[kObsCore];
            observe_core<kF>(P, e.s, gid, t + 1, ob);
            if (want_core) {
                soa_store<kObsCore>(O.obs_core, i, (uint32_t)N, ob);
            }
            if (want_dense) write_dense(P, B, i, ob, t + 1, O.obs_dense + i * (kObsCore + 4 * P.n_hist));
        }
        if (want_critic) {
            float oc[kObsCritic];
            observe_critic(e.s, e.dist, oc);
            soa_store<kObsCritic>(O.obs_critic, i, (uint32_t)N, oc);
        }
        if (want_reward) O.reward[i] = o.reward;
        if (want_flags) O.flags[i] = (uint8_t)fl;
    }
    stats_block_end(st, srow, 0.0, B.slots + (size_t)blockIdx.x * kStatsLen);
}

// ---------------------------------------------------------------------------------------
// l2f_reset: masked (or full) reset at Philox counter t0.
// ---------------------------------------------------------------------------------------
__global__ void __launch_bounds__(kStepBlock) reset_kernel(const DevParams P, const DevBufs B,
                                                           const uint8_t* __restrict__ mask, const StepOutDev O)
{
    const int64_t N = P.n;
    const int64_t i = (int64_t)blockIdx.x * kStepBlock + threadIdx.x;
    if (i >= N) return;
    if (mask && !mask[i]) return;
    const uint32_t gid = P.id_offset + (uint32_t)i;
    EnvReg e;
    float hf[4];
    reset_env(P, e, gid, P.t0, hf);
    store_state(P, B, i, e);
    const int64_t NN = N;
    grp_store<6>(B.dist, i, NN, e.dist);
    grp_store<5>(B.dr, i, NN, e.dr);
    if (P.n_hist > 0) hist_restart(P, B, i, P.t0, hf);
    if (O.obs_core || O.obs_dense) {
        float ob[kObsCore];
        observe_core(P, e.s, gid, P.t0, ob);
        if (O.obs_core) {
#pragma unroll
            for (int j = 0; j < kObsCore; ++j) O.obs_core[j * N + i] = ob[j];
        }
        if (O.obs_dense) write_dense(P, B, i, ob, P.t0, O.obs_dense + i * (kObsCore + 4 * P.n_hist));
    }
    if (O.obs_critic) {
        float oc[kObsCritic];
        observe_critic(e.s, e.dist, oc);
#pragma unroll
        for (int j = 0; j < kObsCritic; ++j) O.obs_critic[j * N + i] = oc[j];
    }
    if (O.flags) O.flags[i] = D_RESET;
    if (O.reward) O.reward[i] = 0.0f;
}

// ---------------------------------------------------------------------------------------
// Open-loop fused rollout: T transitions with the state in registers (N3).  Actions from a
// [T][4][N] buffer or the Philox RAND_ACT stream.  The history ring stays in HBM.
// ---------------------------------------------------------------------------------------
// kPipe (small, latency-bound launches): the next step's action inputs -- the recorded action's
// loads, or the Philox RAND_ACT draw, and the exploration-noise draw -- are issued before this
// step's transition, so the load latency and the integer chains overlap the RK4's FP chain.
// (kPipe = 1: recorded actions, 2: Philox actions; 0: no prefetch)
template <bool kDR, bool kTrace, uint32_t kF = kAnyFlags, int kPipe = 0>
__global__ void __launch_bounds__(kRolloutBlock) rollout_open_kernel(const DevParams P, const DevBufs B,
                                                                     const float* __restrict__ act, int32_t T,
                                                                     float* __restrict__ trace,
                                                                     const int64_t* __restrict__ trace_ids,
                                                                     int32_t K)
{
    __shared__ double srow[(kRolloutBlock / 32) * kStatsLen];
    __shared__ uint4 rscratch[(kRolloutBlock / 32) * kResetScratch];
    const int64_t N = P.n;
    const int64_t i = (int64_t)blockIdx.x * kRolloutBlock + threadIdx.x;
    const bool active = i < N;
    const uint32_t gid = P.id_offset + (uint32_t)i;
    StatPk st;  // T <= 65535 per launch (l2f_rollout splits longer rollouts)
    statpk_zero(st);
    int tslot = -1;
    if (kTrace && active)
        for (int k = 0; k < K; ++k)
            if (trace_ids[k] == i) tslot = k;
    EnvReg e;
    if (active)
        load_env<kDR>(P, B, i, e);
    else
        dummy_env(e);
    int slot = P.hist_slot0;  // (t mod N_H), advanced incrementally
    const uint32_t t_last = P.t0 + (uint32_t)T;
    uint32_t t = P.t0;
    const float* act_i = act ? act + i : nullptr;  // (kPipe: act_i[(k * 4 + c) N] = a_c of step k)
    float a_next[4], za_next[4];
    if constexpr (kPipe == 1) {
#pragma unroll
        for (int c = 0; c < 4; ++c) a_next[c] = active ? __ldg(act_i + (int64_t)c * N) : 0.0f;
    } else if constexpr (kPipe == 2) {
        random_action(P, gid, t, a_next);
    }
    if constexpr (kPipe != 0) action_noise<kF>(P, gid, t, za_next);
    for (int sg = 0; sg < P.n_stages; ++sg) {  // curriculum stages of this launch
    const StageW& W = P.stage[sg];
    for (const uint32_t t_stop = stage_stop(P, sg, t_last); t < t_stop; ++t) {
        const int32_t k = (int32_t)(t - P.t0);
        float a[4], za[4];
        if constexpr (kPipe != 0) {
#pragma unroll
            for (int c = 0; c < 4; ++c) a[c] = a_next[c], za[c] = za_next[c];
            if constexpr (kPipe == 1) {
                const int64_t kn = k + 1 < T ? k + 1 : k;  // (the last step re-reads its own row)
#pragma unroll
                for (int c = 0; c < 4; ++c) a_next[c] = active ? __ldg(act_i + (kn * 4 + c) * N) : 0.0f;
            } else {
                random_action(P, gid, t + 1, a_next);
            }
            action_noise<kF>(P, gid, t + 1, za_next);
        } else if (act) {
#pragma unroll
            for (int c = 0; c < 4; ++c) a[c] = active ? __ldg(act + ((int64_t)k * 4 + c) * N + i) : 0.0f;
        } else {
            random_action(P, gid, t, a);
        }
        L2F_CHECK(tslot < K && k >= 0 && k < T, "trace index");
        float* tr = (kTrace && tslot >= 0) ? trace + ((int64_t)k * K + tslot) * kTraceFields : nullptr;
        if (kTrace && tr) {
#pragma unroll
            for (int c = 0; c < kStateDim; ++c) tr[c] = e.s[c];
#pragma unroll
            for (int c = 0; c < 4; ++c) tr[17 + c] = a[c];
        }
        Trans o;
        if constexpr (kPipe == 0) action_noise<kF>(P, gid, t, za);
        transition<kDR, kF>(P, W, e, gid, t, a, za, o);
        uint32_t fl = o.flags;
        const bool ended = active && (fl & (D_TERM | D_TRUNC));
        statpk_episode(st, o, ended);
        bool did_reset = false;
        float hf[4];
        if (flags_of<kF>(P) & F_AUTO_RESET) {
            did_reset = reset_env_warp<kDR ? 8 : 6, kF>(P, nullptr, e, gid, t + 1, ended, hf, rscratch + (threadIdx.x >> 5) * kResetScratch);
            if (did_reset) fl |= D_RESET;
        } else if (ended) {
            e.ep_step = 0;
            e.ep_return = 0.0f;
        }
        if (active && P.n_hist > 0) {
            L2F_CHECK(slot >= 0 && slot < P.n_hist, "history slot");
            B.hist[(int64_t)slot * N + i] = make_float4(o.a[0], o.a[1], o.a[2], o.a[3]);
            if (did_reset) hist_restart(P, B, i, t + 1, hf);
        }
        if (++slot == P.n_hist) slot = 0;
        if (kTrace && tr) {
#pragma unroll
            for (int c = 0; c < 4; ++c) tr[21 + c] = o.a[c];
            tr[25] = o.reward;
            tr[26] = (float)fl;
            tr[27] = (float)e.ep_step;
            tr[28] = tr[29] = tr[30] = tr[31] = 0.0f;
        }
    }
    }
    if (active) {
        store_state(P, B, i, e);
        store_episode_consts(P, B, i, e);
    }
    const int64_t rem = N - (int64_t)blockIdx.x * kRolloutBlock;
    const double steps = (double)(rem < kRolloutBlock ? rem : kRolloutBlock) * (double)T;
    stats_block_end(st, srow, steps, B.slots + (size_t)blockIdx.x * kStatsLen);
}

// Reward recalculation over stored transitions (after each curriculum change every
// reward in the replay buffer is recomputed): r = reward_of(W, s', a'), 0 for a non-finite s'
// (Q26).  Bitwise equal to the reward l2f_step returned for the same (s', a', stage).
// HBM-bound: 84 B read + 4 B written per transition.
__global__ void __launch_bounds__(256) recompute_rewards_kernel(const StageW W, const float* __restrict__ sn,
                                                                const float* __restrict__ act, int64_t m,
                                                                float* __restrict__ out)
{
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
        float s[kStateDim], a[4];
#pragma unroll
        for (int c = 0; c < kStateDim; ++c) s[c] = __ldg(sn + c * m + i);
#pragma unroll
        for (int c = 0; c < 4; ++c) a[c] = __ldg(act + c * m + i);
        out[i] = state_finite(s) ? reward_of(W, s, a) : 0.0f;
    }
}

cudaError_t launch_recompute_rewards(const StageW& W, const float* next_state, const float* actions, int64_t m,
                                     float* rewards, cudaStream_t s)
{
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int64_t grid = (m + 255) / 256;
    if (grid > (int64_t)sms * 8) grid = (int64_t)sms * 8;
    recompute_rewards_kernel<<<(unsigned)grid, 256, 0, s>>>(W, next_state, actions, m, rewards);
    return cudaGetLastError();
}

// Fixed-order reduction of all statistics slots into out[8], deterministic for a given n_slots:
// block b of kFinBlocks sums the contiguous slot range [b S / kFinBlocks, (b + 1) S / kFinBlocks)
// (thread-strided, then a fixed shared-memory tree) into partial b; the block that arrives last
// (ticket) sums the partials in block order.  (One 256-thread block over 16 384 slots took ~60 us;
// this takes a few us.)
constexpr int kFinBlocks = 64;
constexpr int kFinThreads = 256;

size_t stats_finalize_scratch_bytes() { return sizeof(double) * kStatsLen * kFinBlocks + 256; }

__global__ void __launch_bounds__(kFinThreads) stats_finalize_kernel(double* __restrict__ slots, int32_t n_slots,
                                                                     double* __restrict__ part,
                                                                     unsigned int* __restrict__ ticket,
                                                                     double* __restrict__ out, int32_t reset,
                                                                     double host_steps)
{
    __shared__ double red[kFinThreads * kStatsLen];
    __shared__ bool last;
    const int tid = threadIdx.x, b = blockIdx.x;
    const int lo = (int)((int64_t)n_slots * b / kFinBlocks), hi = (int)((int64_t)n_slots * (b + 1) / kFinBlocks);
    double acc[kStatsLen];
#pragma unroll
    for (int j = 0; j < kStatsLen; ++j) acc[j] = 0.0;
    for (int sl = lo + tid; sl < hi; sl += kFinThreads) {
        double* row = slots + (size_t)sl * kStatsLen;
        const double4 a = reinterpret_cast<const double4*>(row)[0], c = reinterpret_cast<const double4*>(row)[1];
        acc[0] += a.x, acc[1] += a.y, acc[2] += a.z, acc[3] += a.w;
        acc[4] += c.x, acc[5] += c.y, acc[6] += c.z, acc[7] += c.w;
        if (reset) {
            const double4 z = make_double4(0.0, 0.0, 0.0, 0.0);
            reinterpret_cast<double4*>(row)[0] = z;
            reinterpret_cast<double4*>(row)[1] = z;
        }
    }
#pragma unroll
    for (int j = 0; j < kStatsLen; ++j) red[j * kFinThreads + tid] = acc[j];
    __syncthreads();
    for (int w = kFinThreads / 2; w > 0; w >>= 1) {
        if (tid < w)
#pragma unroll
            for (int j = 0; j < kStatsLen; ++j) red[j * kFinThreads + tid] += red[j * kFinThreads + tid + w];
        __syncthreads();
    }
    if (tid < kStatsLen) part[b * kStatsLen + tid] = red[tid * kFinThreads];
    __threadfence();
    __syncthreads();
    if (tid == 0) last = atomicAdd(ticket, 1u) == kFinBlocks - 1;
    __syncthreads();
    if (!last) return;
    __threadfence();
    if (tid < kStatsLen) {
        double x = 0.0;
        for (int k = 0; k < kFinBlocks; ++k) x += __ldcg(part + k * kStatsLen + tid);
        out[tid] = tid == kStatsLen - 1 ? host_steps : x;
    }
    if (tid == 0) *ticket = 0u;  // ready for the next call (the next launch is stream-ordered)
}

// Self-test: our Philox4x32-10 vs curand's curand_Philox4x32_10 (an independent library
// routine) on counters (i, t, stream, block) -- diagnostics only.
__global__ void philox_selftest_kernel(int64_t n, uint32_t k0, uint32_t k1, uint32_t t, uint4* ours, uint4* ref)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t c0 = (uint32_t)i, c2 = (uint32_t)(i % 7), c3 = (uint32_t)(i % 5);
    uint32_t rk0[10], rk1[10];  // the same key schedule the host packs into DevParams
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        rk0[r] = k0 + (uint32_t)r * 0x9E3779B9u;
        rk1[r] = k1 + (uint32_t)r * 0xBB67AE85u;
    }
    ours[i] = philox_rk(c0, t, c2, c3, rk0, rk1);
    ref[i] = curand_Philox4x32_10(make_uint4(c0, t, c2, c3), make_uint2(k0, k1));
}

cudaError_t launch_philox_selftest(int64_t n, uint64_t seed, uint32_t t, uint32_t* ours, uint32_t* ref,
                                   cudaStream_t s)
{
    philox_selftest_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(n, (uint32_t)seed, (uint32_t)(seed >> 32), t,
                                                                       (uint4*)ours, (uint4*)ref);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------------------
// host launchers
// ---------------------------------------------------------------------------------------
cudaError_t launch_step(const DevParams& P, const DevBufs& B, const float* act, const StepOutDev& O,
                        cudaStream_t s)
{
    return launch_step_plain(P, B, act, O, s);
}

cudaError_t launch_step_plain(const DevParams& P, const DevBufs& B, const float* act, const StepOutDev& O,
                              cudaStream_t s)
{
    const int64_t grid = (P.n + kStepBlock - 1) / kStepBlock;
    // compile-time specialisations for the configs' feature mixes with the common outputs
    constexpr uint32_t kC2 = F_OBS_NOISE | F_ACTION_NOISE | F_TERMINATION | F_AUTO_RESET | F_DISTURBANCE;
    const bool std_out = O.obs_core && O.reward && O.flags && !O.obs_dense && !O.obs_critic && !O.final_state;
    if (std_out && P.flags == (kC2 | F_DOMAIN_RAND))
        step_kernel<true, kC2 | F_DOMAIN_RAND, true><<<(unsigned)grid, kStepBlock, 0, s>>>(P, B, act, O);
    else if (std_out && P.flags == kC2)
        step_kernel<false, kC2, true><<<(unsigned)grid, kStepBlock, 0, s>>>(P, B, act, O);
    else if (P.flags & F_DOMAIN_RAND)
        step_kernel<true><<<(unsigned)grid, kStepBlock, 0, s>>>(P, B, act, O);
    else
        step_kernel<false><<<(unsigned)grid, kStepBlock, 0, s>>>(P, B, act, O);
    return cudaGetLastError();
}

cudaError_t launch_reset(const DevParams& P, const DevBufs& B, const uint8_t* mask, const StepOutDev& O,
                         cudaStream_t s)
{
    const int64_t grid = (P.n + kStepBlock - 1) / kStepBlock;
    reset_kernel<<<(unsigned)grid, kStepBlock, 0, s>>>(P, B, mask, O);
    return cudaGetLastError();
}

cudaError_t launch_rollout_open(const DevParams& P, const DevBufs& B, const float* act, int32_t T, float* trace,
                                const int64_t* trace_ids, int32_t K, cudaStream_t s)
{
    const int64_t grid = (P.n + kRolloutBlock - 1) / kRolloutBlock;
    const bool dr = (P.flags & F_DOMAIN_RAND) != 0, tr = trace != nullptr;
    constexpr uint32_t kC5 = F_OBS_NOISE | F_ACTION_NOISE | F_TERMINATION | F_AUTO_RESET | F_DISTURBANCE;
    auto kern = dr ? (tr ? rollout_open_kernel<true, true> : rollout_open_kernel<true, false>)
                   : (tr ? rollout_open_kernel<false, true> : rollout_open_kernel<false, false>);
    // compile-time feature mixes: dynamics only (C1, the paper's benchmark mode) and C2/C5 features.
    // Prefetching the next step's action inputs pays off when the launch is latency-bound (at
    // most ~4 warps per scheduler: C1, C2, the paper's 8192-env shape) and costs issue slots when
    // it is throughput-bound (2^20 envs with Philox actions: -2.6 %), so small launches only.
    static std::atomic<int> sms_cache[64] = {};
    const int dev = current_device();
    int sms = sms_cache[dev].load();
    if (sms == 0) {
        if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms <= 0) sms = 148;
        sms_cache[dev].store(sms);
    }
    const bool pipe = P.n <= (int64_t)sms * 512;
    if (!tr && P.flags == 0u)
        kern = !pipe ? rollout_open_kernel<false, false, 0u> : act ? rollout_open_kernel<false, false, 0u, 1>
                                                                   : rollout_open_kernel<false, false, 0u, 2>;
    if (!tr && P.flags == kC5)
        kern = !pipe ? rollout_open_kernel<false, false, kC5> : act ? rollout_open_kernel<false, false, kC5, 1>
                                                                    : rollout_open_kernel<false, false, kC5, 2>;
    kern<<<(unsigned)grid, kRolloutBlock, 0, s>>>(P, B, act, T, trace, trace_ids, K);
    return cudaGetLastError();
}

cudaError_t launch_stats_finalize(double* slots, int32_t n_slots, void* scratch, double* out, int32_t reset,
                                  double host_steps, cudaStream_t s)
{
    double* part = static_cast<double*>(scratch);
    unsigned int* ticket = reinterpret_cast<unsigned int*>(part + kStatsLen * kFinBlocks);
    stats_finalize_kernel<<<kFinBlocks, kFinThreads, 0, s>>>(slots, n_slots, part, ticket, out, reset, host_steps);
    return cudaGetLastError();
}

}  // namespace l2f
