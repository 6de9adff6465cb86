// l2f_step_tma.cu -- the single-step kernel (l2f_step) staged through shared memory with bulk
// async copies (cp.async.bulk, the TMA bulk path) on sm_100a.
//
// Why: l2f_step is HBM-bound (305 B per env-step with DR).  With plain
// per-thread loads every SoA component costs a 64-bit address computation plus the load, and
// a warp's loads are exposed at the start of its life.  Here a persistent CTA walks 128-env
// tiles; one thread issues one bulk copy per component row (512 B) into a double-buffered
// shared-memory stage (mbarrier complete_tx), so the next tile streams in while this one
// computes; threads read their env with immediate-offset shared loads, write outputs into a
// shared staging tile, and one thread streams each output row back with a bulk store.
// Arithmetic is the same l2f_device.cuh code as every other kernel (bitwise identical).
#include "l2f_device.cuh"
#include "l2f_internal.h"
#include "l2f_tcgen05.cuh"

namespace l2f {
namespace {

constexpr int kT = 128;                  // envs per tile = threads per CTA
constexpr int kRowB = kT * 4;            // bytes of one full component row slice
// input rows: state 0..16, dist 17..22, action 23..26, ep_step 27, ep_return 28, DR 29..33
constexpr int kInState = 0, kInDist = 17, kInAct = 23, kInEpStep = 27, kInEpRet = 28, kInDr = 29;
constexpr int kInRowsMax = 34;
// output rows: state 0..16, ep_step 17, ep_return 18, history slot 19..22, reward 23, obs 24..41
constexpr int kOutState = 0, kOutEpStep = 17, kOutEpRet = 18, kOutHist = 19, kOutRew = 23, kOutObs = 24;
constexpr int kOutRows = 42;

constexpr uint32_t OFF_IN = 0;
constexpr uint32_t kInStageB = kInRowsMax * kRowB;
constexpr uint32_t OFF_OUT = OFF_IN + 2 * kInStageB;
constexpr uint32_t OFF_FLAGS = OFF_OUT + kOutRows * kRowB;
constexpr uint32_t OFF_SCR = OFF_FLAGS + kT;                  // reset scratch, 32 uint4 per warp
constexpr uint32_t OFF_SROW = OFF_SCR + (kT / 32) * kResetScratch * 16;  // statistics rows
constexpr uint32_t OFF_BARS = OFF_SROW + (kT / 32) * kStatsLen * 8;
constexpr uint32_t kSmem = OFF_BARS + 16;

__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t mbar)
{
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(mbar)
                 : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* dst, uint32_t src, uint32_t bytes)
{
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(src), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(uint32_t mbar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mbar), "r"(bytes) : "memory");
}

// Bulk loads of one tile, issued in parallel by the 32 lanes of warp 0 (lane r issues row r,
// lanes 0 and 1 also rows 32 and 33); lane 0 arms the stage's mbarrier with the byte count.
template <bool kDR>
__device__ __forceinline__ void issue_loads(const DevParams& P, const DevBufs& B, const float* act, int tile,
                                            uint32_t stage_base, uint32_t mbar, int lane)
{
    const int64_t N = P.n;
    const int64_t base = (int64_t)tile * kT;
    const int64_t nh = N - base < kT ? N - base : kT;
    const uint32_t bytes = (uint32_t)nh * 4u;
    const int rows = kDR ? kInRowsMax : kInDr;
    if (lane == 0) mbar_expect_tx(mbar, bytes * (uint32_t)rows);
    for (int r = lane; r < rows; r += 32) {
        const void* src;
        if (r < kInDist)
            src = B.state + (r - kInState) * N + base;
        else if (r < kInAct)
            src = B.dist + (r - kInDist) * N + base;
        else if (r < kInEpStep)
            src = act + (r - kInAct) * N + base;
        else if (r == kInEpStep)
            src = B.ep_step + base;
        else if (r == kInEpRet)
            src = B.ep_return + base;
        else
            src = B.dr + (r - kInDr) * N + base;
        bulk_g2s(stage_base + r * kRowB, src, bytes, mbar);
    }
}

// Bulk stores of one tile's output rows, issued in parallel by the lanes of warp 0.
__device__ __forceinline__ void issue_stores(const DevParams& P, const DevBufs& B, const StepOutDev& O, int64_t base,
                                             int nh, uint32_t out_base, uint32_t flags_base, int lane)
{
    const int64_t N = P.n;
    const uint32_t bytes = (uint32_t)nh * 4u;
    for (int r = lane; r < kOutRows + 1; r += 32) {
        void* dst = nullptr;
        uint32_t nb = bytes;
        if (r < kOutEpStep)
            dst = B.state + (r - kOutState) * N + base;
        else if (r == kOutEpStep)
            dst = B.ep_step + base;
        else if (r == kOutEpRet)
            dst = B.ep_return + base;
        else if (r < kOutRew)
            dst = P.n_hist > 0 ? (void*)(B.hist + ((int64_t)P.hist_slot0 * 4 + (r - kOutHist)) * N + base) : nullptr;
        else if (r == kOutRew)
            dst = O.reward ? (void*)(O.reward + base) : nullptr;
        else if (r < kOutRows)
            dst = O.obs_core ? (void*)(O.obs_core + (r - kOutObs) * N + base) : nullptr;
        else {  // flags: the 16-byte-aligned prefix (the rest is stored per thread)
            dst = O.flags ? (void*)(O.flags + base) : nullptr;
            nb = (uint32_t)(nh & ~15);
        }
        if (dst && nb) bulk_s2g(dst, r < kOutRows ? out_base + r * kRowB : flags_base, nb);
    }
    bulk_commit();
}

template <bool kDR>
__global__ void __launch_bounds__(kT, 3) step_tma_kernel(const DevParams P, const DevBufs B,
                                                         const float* __restrict__ act, const StepOutDev O,
                                                         int32_t n_tiles)
{
    extern __shared__ __align__(128) uint8_t smem[];
    const uint32_t sb = tc::smem_u32(smem);
    const int tid = threadIdx.x;
    const uint32_t bar0 = sb + OFF_BARS, bar1 = sb + OFF_BARS + 8;
    const int64_t N = P.n;
    const uint32_t t = P.t0;
    const StageW& W = stage_of(P, t);
    if (tid == 0) {
        tc::mbar_init(bar0, 1);
        tc::mbar_init(bar1, 1);
        tc::fence_mbar_init();
    }
    __syncthreads();
    const int stride = gridDim.x;
    int tile = blockIdx.x;
    if (tid < 32) {
        if (tile < n_tiles) issue_loads<kDR>(P, B, act, tile, sb + OFF_IN, bar0, tid);
        if (tile + stride < n_tiles) issue_loads<kDR>(P, B, act, tile + stride, sb + OFF_IN + kInStageB, bar1, tid);
    }
    StatAcc st;
    stat_zero(st);
    double steps = 0.0;
    for (int it = 0; tile < n_tiles; tile += stride, ++it) {
        const int stage = it & 1;
        const uint32_t in_b = OFF_IN + stage * kInStageB;
        tc::mbar_wait(stage ? bar1 : bar0, (uint32_t)(it >> 1) & 1u);
        const int64_t base = (int64_t)tile * kT;
        const int nh = (int)(N - base < kT ? N - base : kT);
        const bool active = tid < nh;
        const int64_t i = base + tid;
        const uint32_t gid = P.id_offset + (uint32_t)i;
        const float* in = reinterpret_cast<const float*>(smem + in_b) + tid;
        EnvReg e;
        float a[4];
        if (active) {
#pragma unroll
            for (int c = 0; c < kStateDim; ++c) e.s[c] = in[(kInState + c) * kT];
#pragma unroll
            for (int c = 0; c < 6; ++c) e.dist[c] = in[(kInDist + c) * kT];
#pragma unroll
            for (int c = 0; c < 4; ++c) a[c] = in[(kInAct + c) * kT];
            e.ep_step = __float_as_int(in[kInEpStep * kT]);
            e.ep_return = in[kInEpRet * kT];
#pragma unroll
            for (int c = 0; c < 5; ++c) e.dr[c] = kDR ? in[(kInDr + c) * kT] : 1.0f;
        } else {
#pragma unroll
            for (int c = 0; c < kStateDim; ++c) e.s[c] = 0.0f;
            e.s[3] = 1.0f;
#pragma unroll
            for (int c = 0; c < 6; ++c) e.dist[c] = 0.0f;
#pragma unroll
            for (int c = 0; c < 5; ++c) e.dr[c] = 1.0f;
#pragma unroll
            for (int c = 0; c < 4; ++c) a[c] = 0.0f;
            e.ep_step = 0;
            e.ep_return = 0.0f;
        }
        __syncthreads();  // every thread has read this stage: refill it with tile + 2 stride
        if (tid < 32 && tile + 2 * stride < n_tiles)
            issue_loads<kDR>(P, B, act, tile + 2 * stride, sb + in_b, stage ? bar1 : bar0, tid);

        Trans o;
        float za[4];
        action_noise(P, gid, t, za);
        transition<kDR>(P, W, e, gid, t, a, za, o);
        uint32_t fl = o.flags;
        const bool ended = active && (fl & (D_TERM | D_TRUNC));
        if (ended) stat_episode(st, o);
        bool did_reset = false;
        float hf[4];
        if (P.flags & F_AUTO_RESET) {
            did_reset = reset_env_warp(P, e, gid, t + 1, ended, hf,
                                       reinterpret_cast<uint4*>(smem + OFF_SCR) + (tid >> 5) * kResetScratch);
            if (did_reset) fl |= D_RESET;
        } else if (ended) {
            e.ep_step = 0;
            e.ep_return = 0.0f;
        }
        float ob[kObsCore];
        if (O.obs_core) observe_core(P, e.s, gid, t + 1, ob);
        if (active && did_reset) {  // episode constants and history marker: rare, direct stores
#pragma unroll
            for (int c = 0; c < 6; ++c) B.dist[c * N + i] = e.dist[c];
            if (kDR)
#pragma unroll
                for (int c = 0; c < 5; ++c) B.dr[c * N + i] = e.dr[c];
            if (P.n_hist > 0) {
                B.hist_t0[i] = (int32_t)(t + 1);
#pragma unroll
                for (int c = 0; c < 4; ++c) B.hist_fill[(int64_t)c * N + i] = hf[c];
            }
        }
        // stage the outputs; the previous tile's bulk stores must have finished reading them
        if (tid < 32) bulk_wait_read0();
        __syncthreads();
        float* out = reinterpret_cast<float*>(smem + OFF_OUT) + tid;
#pragma unroll
        for (int c = 0; c < kStateDim; ++c) out[(kOutState + c) * kT] = e.s[c];
        out[kOutEpStep * kT] = __int_as_float(e.ep_step);
        out[kOutEpRet * kT] = e.ep_return;
#pragma unroll
        for (int c = 0; c < 4; ++c) out[(kOutHist + c) * kT] = o.a[c];
        out[kOutRew * kT] = o.reward;
        if (O.obs_core)
#pragma unroll
            for (int j = 0; j < kObsCore; ++j) out[(kOutObs + j) * kT] = ob[j];
        smem[OFF_FLAGS + tid] = (uint8_t)fl;
        tc::fence_proxy_async();
        __syncthreads();
        if (tid < 32) issue_stores(P, B, O, base, nh, sb + OFF_OUT, sb + OFF_FLAGS, tid);
        if (O.flags && active && tid >= (nh & ~15)) O.flags[i] = (uint8_t)fl;  // unaligned tail
        steps += (double)nh;
    }
    if (tid < 32) bulk_wait0();
    // statistics of this CTA's tiles -> its slot (fixed tile assignment: deterministic)
    double* srow = reinterpret_cast<double*>(smem + OFF_SROW);
    stat_warp_to_smem(st, srow + (tid >> 5) * kStatsLen);
    __syncthreads();
    stat_rows_to_slot(srow, kT / 32, steps, B.slots + (size_t)blockIdx.x * kStatsLen);
}

int sm_count()
{
    static int n = 0;
    if (n == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
    }
    return n;
}

}  // namespace

// Grid of the bulk-staged step kernel (3 CTAs per SM); 0 when it cannot be used.
int step_tma_grid(int64_t n)
{
    const int64_t tiles = (n + kT - 1) / kT;
    const int64_t g = 3 * 148;
    return (int)(tiles < g ? tiles : g);
}

bool step_tma_ok(const DevParams& P, const float* act, const StepOutDev& O)
{
    auto al = [](const void* p) { return ((uintptr_t)p & 15u) == 0; };
    if (P.n % 4 != 0 || O.obs_dense || O.final_state) return false;
    return al(act) && al(O.obs_core) && al(O.reward) && al(O.flags);
}

cudaError_t launch_step_tma(const DevParams& P, const DevBufs& B, const float* act, const StepOutDev& O,
                            cudaStream_t s)
{
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(step_tma_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(step_tma_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    const int n_tiles = (int)((P.n + kT - 1) / kT);
    int grid = 3 * sm_count();
    if (grid > n_tiles) grid = n_tiles;
    if (P.flags & F_DOMAIN_RAND)
        step_tma_kernel<true><<<grid, kT, kSmem, s>>>(P, B, act, O, n_tiles);
    else
        step_tma_kernel<false><<<grid, kT, kSmem, s>>>(P, B, act, O, n_tiles);
    return cudaGetLastError();
}

}  // namespace l2f
