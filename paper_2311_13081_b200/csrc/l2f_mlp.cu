// l2f_mlp.cu -- fused rollout with the actor MLP on 5th-gen tensor cores (tcgen05), sm_100a.
//
// Per step and env (BASELINE configs[3]):
//   o_t = {p, R, v, omega} + noise  ++  H (last N_H applied actions, most recent first)
//   a_t = tanh(W3 q16(relu(W2 q16(relu(W1 q16(o_t) + b1)) + b2)) + b3)        (Q21)
//   then the same env transition as l2f_step (l2f_device.cuh).
//
// Design:
//  * persistent CTA per SM, 3 tiles x 128 envs; thread r of a tile owns env row r, which is
//    both row r of the MMA A operand and TMEM lane r of the accumulator (32x32b loads);
//  * operands fp16 in shared memory (SWIZZLE_NONE canonical layouts), accumulators fp32 in
//    TMEM (64 columns per tile reused by the three layers); biases enter the MMA through a
//    constant "ones" column, so epilogues are relu + fp16 pack only;
//  * the action history lives in the A operand as a ring: the action of step tau sits at
//    ring position (-tau mod N_H) and never moves; each step the B descriptor of W1's
//    history block is rotated instead (MN-major copy with duplicated K rows, so a rotation
//    by 4 K-rows is a 64-byte start-address offset).  Zero shared-memory traffic for the
//    history beyond the one 8-byte slot write per env-step;
//  * one thread per tile and layer (lane 0 of warp l - 1 for layer l) issues the MMAs after a
//    128-thread named barrier; MMA
//    completion is signalled through tcgen05.commit -> mbarrier.  The other two tiles' warps
//    keep the FP32/INT pipes busy while one tile waits on the tensor core.
#include <cstdio>

#include "l2f_device.cuh"
#include "l2f_internal.h"
#include "l2f_tcgen05.cuh"

#ifndef L2F_MLP_TILES
#define L2F_MLP_TILES 3
#endif

namespace l2f {
namespace {

constexpr int kTiles = L2F_MLP_TILES;
constexpr int kM = 128;
constexpr int kThreads = kTiles * kM;
constexpr int kHid = 64;

// shared-memory map (bytes)
constexpr uint32_t kChunkA = kM * 16;                 // one 8-wide K chunk of a 128-row A tile
constexpr uint32_t kA1Bytes = 20 * kChunkA;           // K = 32 (obs, ones, pad) + 128 (history)
constexpr uint32_t kW1oBytes = 4 * kHid * 16;         // K = 32 x N = 64, K-major
constexpr uint32_t kW1hBytes = 8 * (8 * kMaxHist * 16);  // MN-major: 8 N-groups x 2*4*N_H K-rows
constexpr uint32_t kW2Bytes = 10 * kHid * 16;         // K = 80 x N = 64, K-major
constexpr uint32_t kW3Bytes = 10 * 16 * 16;           // K = 80 x N = 16, K-major

constexpr uint32_t OFF_A1 = 0;
constexpr uint32_t OFF_W1O = OFF_A1 + kTiles * kA1Bytes;
constexpr uint32_t OFF_W1H = OFF_W1O + kW1oBytes;
constexpr uint32_t OFF_W2 = OFF_W1H + kW1hBytes;
constexpr uint32_t OFF_W3 = OFF_W2 + kW2Bytes;
constexpr uint32_t OFF_BAR = OFF_W3 + kW3Bytes;       // kTiles MMA-done mbarriers
constexpr uint32_t OFF_TMEM = OFF_BAR + 8 * kTiles;
constexpr uint32_t OFF_STAT = (OFF_TMEM + 8 + 127) & ~127u;  // reset scratch (32 uint4 per warp); reused by stats
constexpr uint32_t kScratchBytes = (kThreads / 32) * kResetScratch * 16;
static_assert(kScratchBytes >= (kThreads / 32) * kStatsLen * 8, "stats rows fit in the scratch");
constexpr uint32_t kSmemBytes = OFF_STAT + kScratchBytes;
static_assert(kSmemBytes <= 232448, "shared memory budget");
constexpr uint32_t kTmemCols = 512;  // accumulators: kTiles x 64 columns from 0; noise stash: 32 per tile from 256
// TMEM map: accumulators 64 columns per tile from 0; A2 (h1/h2 as fp16: 32 columns + 8 with the
// ones column) 40 per tile from 64 kTiles; the per-thread noise stash (18 used) 24 per tile after.
constexpr uint32_t kA2Col = 64 * kTiles;
constexpr uint32_t kStashCol = kA2Col + 40 * kTiles;
static_assert(kStashCol + 24 * kTiles <= kTmemCols, "TMEM budget");

constexpr uint32_t kIdescN64 = tc::make_idesc(128, 64, 0, 0);
constexpr uint32_t kIdescN64BMN = tc::make_idesc(128, 64, 0, 1);
constexpr uint32_t kIdescN16 = tc::make_idesc(128, 16, 0, 0);

__device__ __forceinline__ uint16_t h16(const uint16_t* p, int i) { return __ldg(p + i); }

__device__ __forceinline__ void st_u16(uint32_t saddr, uint16_t v)
{
    asm volatile("st.shared.u16 [%0], %1;" ::"r"(saddr), "h"(v) : "memory");
}

// Lay out the policy in shared memory (once per CTA): B operands with the bias as the K row
// paired with the A operand's ones column.
__device__ void stage_weights(const PolicyDev& W, uint32_t sbase, int n_hist)
{
    const int tid = threadIdx.x;
    const int I = W.in_dim;
    for (int idx = tid; idx < kHid * 32; idx += blockDim.x) {  // W1 obs part, K-major
        const int n = idx / 32, k = idx % 32;
        const uint16_t v = k < 18 ? h16(W.W1, n * I + k) : (k == 18 ? h16(W.b1, n) : (uint16_t)0);
        st_u16(sbase + OFF_W1O + (k / 8) * (kHid * 16) + n * 16 + (k % 8) * 2, v);
    }
    const int hk = 4 * n_hist;  // history K
    const uint32_t sbo_h = 2 * hk * 16;
    for (int idx = tid; idx < kHid * 2 * hk; idx += blockDim.x) {  // W1 history, MN-major, rows duplicated
        const int n = idx / (2 * hk), i = idx % (2 * hk);
        const uint16_t v = h16(W.W1, n * I + 18 + (i % hk));
        st_u16(sbase + OFF_W1H + (n / 8) * sbo_h + i * 16 + (n % 8) * 2, v);
    }
    for (int idx = tid; idx < kHid * 80; idx += blockDim.x) {  // W2 + b2, K-major
        const int n = idx / 80, k = idx % 80;
        const uint16_t v = k < 64 ? h16(W.W2, n * 64 + k) : (k == 64 ? h16(W.b2, n) : (uint16_t)0);
        st_u16(sbase + OFF_W2 + (k / 8) * (kHid * 16) + n * 16 + (k % 8) * 2, v);
    }
    for (int idx = tid; idx < 16 * 80; idx += blockDim.x) {  // W3 + b3 padded to N = 16, K-major
        const int n = idx / 80, k = idx % 80;
        uint16_t v = 0;
        if (n < 4) v = k < 64 ? h16(W.W3, n * 64 + k) : (k == 64 ? h16(W.b3, n) : (uint16_t)0);
        st_u16(sbase + OFF_W3 + (k / 8) * (16 * 16) + n * 16 + (k % 8) * 2, v);
    }
}

__device__ __forceinline__ float tanh_fast(float z)
{
    // tanh z = 1 - 2 / (exp(2z) + 1); exact limits at +-inf, absolute error ~1e-7
    return 1.0f - __fdividef(2.0f, __expf(2.0f * z) + 1.0f);
}

struct TileCtx {
    uint32_t a1_row;          // this thread's row in the A1 tile
    uint32_t a1;              // A1 tile base
    uint32_t mbar;
    uint32_t tmem_row;        // TMEM address of (this thread's lane, tile column 0)
    uint32_t tmem_tile;       // TMEM address of (lane 0, tile column 0)
    uint32_t stash_row;       // TMEM address of this thread's 32-column noise stash
    uint32_t a2_tmem;         // TMEM address of (lane 0, this tile's A2 column 0)
    uint32_t a2_trow;         // ... of this thread's lane
    uint32_t bar_id;
    uint32_t phase;
    uint32_t r;               // thread index within the tile
#ifdef L2F_PHASE_TIMING
    uint32_t ph_last;         // debug build only: clock() at the last phase boundary
#endif
};

// Debug build only (-DL2F_PHASE_TIMING): per-warp cycles spent in each phase of a tile-step,
// accumulated in shared memory and printed by CTA 0 at exit (scripts/phase_timing.py).
#ifdef L2F_PHASE_TIMING
__shared__ unsigned long long g_ph[kThreads / 32][16];
#define L2F_PHASE(c, k)                                                             \
    do {                                                                            \
        const uint32_t _n = (uint32_t)clock();                                      \
        if ((threadIdx.x & 31) == 0) g_ph[threadIdx.x >> 5][k] += _n - (c).ph_last; \
        (c).ph_last = _n;                                                           \
    } while (0)
#else
#define L2F_PHASE(c, k) \
    do {                \
    } while (0)
#endif

// Epilogue of L1 / L2: accumulator row -> relu -> fp16 -> this thread's A2 row in TMEM.
__device__ __forceinline__ void epilogue_hidden(const TileCtx& c)
{
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        uint32_t v[16];
        tc::tmem_ld16(c.tmem_row + 16 * q, v);
        tc::tmem_wait_ld();
        tc::tmem_st8u(c.a2_trow + 8 * q, tc::relu_pack(v[0], v[1]), tc::relu_pack(v[2], v[3]),
                      tc::relu_pack(v[4], v[5]), tc::relu_pack(v[6], v[7]), tc::relu_pack(v[8], v[9]),
                      tc::relu_pack(v[10], v[11]), tc::relu_pack(v[12], v[13]), tc::relu_pack(v[14], v[15]));
    }
    tc::tmem_wait_st();
}

// The tile's 128 threads hand their freshly written A rows (and finished TMEM reads) to the
// MMA issuer: proxy fence + tcgen05 fence + a 128-thread named barrier (id 1 + tile).  (Variants
// where only the issuing warp waits -- mbarrier arrive/wait, or bar.arrive for the other three
// warps -- measured no faster: the other tiles' warps already fill the barrier time.)
__device__ __forceinline__ void handoff_to_mma(TileCtx& c)
{
    tc::fence_proxy_async();
    tc::fence_before();
    tc::named_sync(c.bar_id, kM);
}

__device__ __forceinline__ void wait_mma(TileCtx& c)
{
    tc::mbar_wait(c.mbar, c.phase);
    c.phase ^= 1u;
    tc::fence_after();
}

struct NoHook {
    __device__ __forceinline__ void operator()(int) const {}
};

// The three layers on the tensor core for one tile; layer l is issued by lane 0 of the tile's warp
// l - 1 so the issue work is spread over three warps.  Precondition: A1 rows written by all 128
// threads.  `rot` = rotation of the history ring (W1 history row offset in slots).  hook(l) runs
// on every thread right after layer l's MMAs were issued, i.e. inside the MMA latency (used to
// draw the next step's noise).
template <class Hook>
__device__ __forceinline__ void mlp_tile(TileCtx& c, uint32_t sbase, int n_hist, uint32_t rot, float a[4],
                                         const Hook& hook)
{
    // descriptors = base descriptor + (byte offset >> 4) in the start-address field (addresses
    // stay below 256 KB, so the 14-bit field never carries)
    L2F_PHASE(c, 0);
    rot = __shfl_sync(0xffffffffu, rot, 0);  // warp-uniform for the compiler (uniform registers)
    handoff_to_mma(c);
    L2F_PHASE(c, 1);
    if (c.r == 0) {
        tc::fence_after();
        const uint64_t dA1 = tc::make_desc(c.a1, kChunkA, 128);
        const uint64_t dW1o = tc::make_desc(sbase + OFF_W1O, kHid * 16, 128);
        const uint64_t dW1h = tc::make_desc(sbase + OFF_W1H, 128, 2u * 4u * (uint32_t)n_hist * 16u) + 4u * rot;
        // L1: obs part (K = 32) then history (K = 4 N_H) with the rotated W1 history block
        tc::mma_f16(c.tmem_tile, dA1, dW1o, kIdescN64, 0);
        tc::mma_f16(c.tmem_tile, dA1 + 2 * kChunkA / 16, dW1o + 2 * (kHid * 16) / 16, kIdescN64, 1);
        for (int j = 0; j < n_hist / 4; ++j)
            tc::mma_f16(c.tmem_tile, dA1 + (4 + 2 * j) * (kChunkA / 16), dW1h + 16u * j, kIdescN64BMN, 1);
        tc::commit(c.mbar);
    }
    hook(1);
    L2F_PHASE(c, 2);
    wait_mma(c);
    L2F_PHASE(c, 3);
    epilogue_hidden(c);
    L2F_PHASE(c, 4);
    handoff_to_mma(c);
    L2F_PHASE(c, 5);
    if (c.r == 32) {
        tc::fence_after();
        const uint64_t dW2 = tc::make_desc(sbase + OFF_W2, kHid * 16, 128);
#pragma unroll
        for (int j = 0; j < 5; ++j)  // A from TMEM; j = 4: the ones column (bias row of W2)
            tc::mma_f16_ts(c.tmem_tile, c.a2_tmem + 8 * j, dW2 + j * (2 * kHid * 16 / 16), kIdescN64, j);
        tc::commit(c.mbar);
    }
    hook(2);
    L2F_PHASE(c, 6);
    wait_mma(c);
    L2F_PHASE(c, 7);
    epilogue_hidden(c);
    L2F_PHASE(c, 8);
    handoff_to_mma(c);
    L2F_PHASE(c, 9);
    if (c.r == 64) {
        tc::fence_after();
        const uint64_t dW3 = tc::make_desc(sbase + OFF_W3, 256, 128);
#pragma unroll
        for (int j = 0; j < 5; ++j)
            tc::mma_f16_ts(c.tmem_tile, c.a2_tmem + 8 * j, dW3 + j * (2 * 256 / 16), kIdescN16, j);
        tc::commit(c.mbar);
    }
    hook(3);
    L2F_PHASE(c, 10);
    wait_mma(c);
    uint32_t v[4];
    tc::tmem_ld4(c.tmem_row, v);
    tc::tmem_wait_ld();
    tc::fence_before();
#pragma unroll
    for (int j = 0; j < 4; ++j) a[j] = tanh_fast(__uint_as_float(v[j]));
    L2F_PHASE(c, 11);
}

// Observation-noise normals of one step, stashed per thread in TMEM (columns 0..17 of the
// thread's stash) so they can be drawn inside the previous step's MMA latency without
// holding registers across the RK4.
__device__ __forceinline__ void stash_obs_noise(const DevParams& P, const TileCtx& c, uint32_t gid, uint32_t t,
                                                int part)
{
    float z[20];
    if (part == 0 || part == 3) {
        obs_noise_blocks(P, gid, t, 0, 2, z);
        tc::tmem_st8(c.stash_row + 0, z, 0);
    }
    if (part == 1 || part == 3) {
        obs_noise_blocks(P, gid, t, 2, 4, z);
        tc::tmem_st8(c.stash_row + 8, z, 8);
    }
    if (part == 2 || part == 3) {
        obs_noise_blocks(P, gid, t, 4, 5, z);
        tc::tmem_st2(c.stash_row + 16, z[16], z[17]);
    }
}

__device__ __forceinline__ void load_obs_noise(const TileCtx& c, float z[20])
{
    uint32_t v[16], w[4];
    tc::tmem_wait_st();
    tc::tmem_ld16(c.stash_row, v);
    tc::tmem_ld4(c.stash_row + 16, w);
    tc::tmem_wait_ld();
#pragma unroll
    for (int j = 0; j < 16; ++j) z[j] = __uint_as_float(v[j]);
    z[16] = __uint_as_float(w[0]);
    z[17] = __uint_as_float(w[1]);
    z[18] = z[19] = 0.0f;
}

__device__ __forceinline__ void write_obs_row(const TileCtx& c, const float o[kObsCore])
{
    tc::sts128(c.a1_row, tc::pack_h2(o[0], o[1]), tc::pack_h2(o[2], o[3]), tc::pack_h2(o[4], o[5]),
               tc::pack_h2(o[6], o[7]));
    tc::sts128(c.a1_row + kChunkA, tc::pack_h2(o[8], o[9]), tc::pack_h2(o[10], o[11]), tc::pack_h2(o[12], o[13]),
               tc::pack_h2(o[14], o[15]));
    tc::sts128(c.a1_row + 2 * kChunkA, tc::pack_h2(o[16], o[17]), 0x00003C00u /* (1, 0) */, 0u, 0u);
}

// history ring position p -> A1 address (8 bytes: 4 fp16)
__device__ __forceinline__ uint32_t hist_addr(const TileCtx& c, int p)
{
    return c.a1_row + (4 + (p >> 1)) * kChunkA + (p & 1) * 8;
}

__device__ void setup_cta(const PolicyDev& W, uint32_t sbase, int n_hist)
{
    stage_weights(W, sbase, n_hist);
    if (threadIdx.x == 0) {
        for (int g = 0; g < kTiles; ++g) tc::mbar_init(sbase + OFF_BAR + 8 * g, 1);  // MMA done
        tc::fence_mbar_init();
    }
    if (threadIdx.x < 32) tc::tmem_alloc(sbase + OFF_TMEM, kTmemCols);
    tc::fence_proxy_async();
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
}

__device__ __forceinline__ TileCtx make_ctx(uint32_t sbase)
{
    extern __shared__ __align__(1024) uint8_t smem[];
    // tile index and TMEM base broadcast from lane 0: the compiler then knows they are
    // warp-uniform and keeps the MMA descriptors / TMEM addresses in uniform registers (no
    // per-MMA R2UR waterfall loop in the issuing thread)
    const int g = __shfl_sync(0xffffffffu, (int)(threadIdx.x / kM), 0), r = threadIdx.x % kM;
    const uint32_t tbase = __shfl_sync(0xffffffffu, *reinterpret_cast<const uint32_t*>(smem + OFF_TMEM), 0);
    TileCtx c;
    c.a1 = sbase + OFF_A1 + g * kA1Bytes;
    c.a1_row = c.a1 + r * 16;
    c.mbar = sbase + OFF_BAR + 8 * g;
    c.tmem_tile = tbase + 64 * g;
    c.tmem_row = c.tmem_tile + ((uint32_t)(32 * (r / 32)) << 16);
    c.stash_row = tbase + kStashCol + 24 * g + ((uint32_t)(32 * (r / 32)) << 16);
    c.a2_tmem = tbase + kA2Col + 40 * g;
    c.a2_trow = c.a2_tmem + ((uint32_t)(32 * (r / 32)) << 16);
    // constant ones column (K index 64 of layers 2 and 3) + zero pad
    tc::tmem_st8u(c.a2_trow + 32, 0x3C00u, 0u, 0u, 0u, 0u, 0u, 0u, 0u);
    tc::tmem_wait_st();
    c.bar_id = 1 + g;
    c.phase = 0;
    c.r = r;
#ifdef L2F_PHASE_TIMING
    if ((threadIdx.x & 31) == 0)
        for (int k = 0; k < 16; ++k) g_ph[threadIdx.x >> 5][k] = 0ull;
    c.ph_last = (uint32_t)clock();
#endif
    tc::sts128(c.a1_row + 3 * kChunkA, 0u, 0u, 0u, 0u);  // K 24..31: constant zero pad
    return c;
}

__device__ void teardown_cta()
{
    extern __shared__ __align__(1024) uint8_t smem[];
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    if (threadIdx.x < 32) tc::tmem_dealloc(*reinterpret_cast<const uint32_t*>(smem + OFF_TMEM), kTmemCols);
}

// -------------------------------------------------------------------------------------------
// Fused rollout: T steps of {obs -> MLP (tensor cores) -> env transition} per env.
// -------------------------------------------------------------------------------------------
template <bool kDR>
__global__ void __launch_bounds__(kThreads, 1)
    rollout_mlp_kernel(const DevParams P, const DevBufs B, const PolicyDev W, int32_t T, float* __restrict__ trace,
                       const int64_t* __restrict__ trace_ids, int32_t K, int32_t n_tiles)
{
    extern __shared__ __align__(1024) uint8_t smem[];
    const uint32_t sbase = tc::smem_u32(smem);
    const int NH = P.n_hist;
    setup_cta(W, sbase, NH);
    TileCtx c = make_ctx(sbase);
    const int64_t N = P.n;
    const int r = threadIdx.x % kM;
    StatAcc st;
    stat_zero(st);
    double steps_done = 0.0;

    for (int tile = blockIdx.x * kTiles + (int)(threadIdx.x / kM); tile < n_tiles; tile += gridDim.x * kTiles) {
        const int64_t i = (int64_t)tile * kM + r;
        const bool active = i < N;
        const uint32_t gid = P.id_offset + (uint32_t)i;
        EnvReg e;
        if (active) {
#pragma unroll
            for (int q = 0; q < kStateDim; ++q) e.s[q] = B.state[q * N + i];
#pragma unroll
            for (int q = 0; q < 6; ++q) e.dist[q] = B.dist[q * N + i];
#pragma unroll
            for (int q = 0; q < 5; ++q) e.dr[q] = kDR ? B.dr[q * N + i] : 1.0f;
            e.ep_step = B.ep_step[i];
            e.ep_return = B.ep_return[i];
        } else {
#pragma unroll
            for (int q = 0; q < kStateDim; ++q) e.s[q] = 0.0f;
            e.s[3] = 1.0f;
#pragma unroll
            for (int q = 0; q < 6; ++q) e.dist[q] = 0.0f;
#pragma unroll
            for (int q = 0; q < 5; ++q) e.dr[q] = 1.0f;
            e.ep_step = 0;
            e.ep_return = 0.0f;
        }
        // logical history at t0 (H[k] = a_{t0-1-k}, or the episode fill) -> A1 position (-tau) mod N_H
        {
            const int32_t h0 = active ? B.hist_t0[i] : 0;
            for (int k = 0; k < NH; ++k) {
                float h[4] = {0.f, 0.f, 0.f, 0.f};
                if (active) hist_entry(B, N, NH, i, (int64_t)P.t0, k, h0, h);
                const int64_t tau = (int64_t)P.t0 - 1 - k;
                const int p = (int)(((-tau) % NH + NH) % NH);
                tc::sts64(hist_addr(c, p), tc::pack_h2(h[0], h[1]), tc::pack_h2(h[2], h[3]));
            }
        }
        int tslot = -1;
        if (trace && active)
            for (int q = 0; q < K; ++q)
                if (trace_ids[q] == i) tslot = q;

        const bool obs_noise = (P.flags & F_OBS_NOISE) != 0;
        if (obs_noise) stash_obs_noise(P, c, gid, P.t0, 3);
        // ring rotation (t - 1) mod N_H and write position (-t) mod N_H, advanced incrementally
        uint32_t rot = NH > 0 ? (P.t0 + (uint32_t)NH - 1u) % (uint32_t)NH : 0u;
        int wpos = NH > 0 ? (int)(((uint32_t)NH - P.t0 % (uint32_t)NH) % (uint32_t)NH) : 0;
        const uint32_t t_last = P.t0 + (uint32_t)T;
        uint32_t t = P.t0;
        for (int sg = 0; sg < P.n_stages; ++sg) {  // curriculum stages of this launch
        const StageW& W = P.stage[sg];
        for (const uint32_t t_stop = stage_stop(P, sg, t_last); t < t_stop; ++t) {
            const int32_t k = (int32_t)(t - P.t0);
            float ob[kObsCore];
            {
                float z[20];
                if (obs_noise) load_obs_noise(c, z);
                observe_core_z(P, e.s, z, ob);
            }
            write_obs_row(c, ob);
            float a[4], za[4];
            mlp_tile(c, sbase, NH, rot, a, [&](int l) {
                if (l == 1) action_noise(P, gid, t, za);
                if (obs_noise) stash_obs_noise(P, c, gid, t + 1, l - 1);
            });
            if (NH > 0 && ++rot == (uint32_t)NH) rot = 0;
            float* tr = (tslot >= 0) ? trace + ((int64_t)k * K + tslot) * kTraceFields : nullptr;
            if (tr) {
#pragma unroll
                for (int q = 0; q < kStateDim; ++q) tr[q] = e.s[q];
#pragma unroll
                for (int q = 0; q < 4; ++q) tr[17 + q] = a[q];
            }
            Trans o;
            transition<kDR>(P, W, e, gid, t, a, za, o);
            L2F_PHASE(c, 12);
            uint32_t fl = o.flags;
            const bool ended = (fl & (D_TERM | D_TRUNC)) != 0;
            if (ended && active) stat_episode(st, o);
            bool did_reset = false;
            float hf[4];
            if (P.flags & F_AUTO_RESET) {
                did_reset = reset_env_warp(P, e, gid, t + 1, ended && active, hf,
                                           reinterpret_cast<uint4*>(smem + OFF_STAT) + (threadIdx.x >> 5) * kResetScratch);
                if (did_reset) fl |= D_RESET;
            }
            if (ended && !did_reset) {
                e.ep_step = 0;
                e.ep_return = 0.0f;
            }
            if (NH > 0) {
                if (!did_reset)
                    tc::sts64(hist_addr(c, wpos), tc::pack_h2(o.a[0], o.a[1]), tc::pack_h2(o.a[2], o.a[3]));
                if (--wpos < 0) wpos = NH - 1;
                // new episodes: the whole history row takes the fill value (Q10); the N_H/2
                // 16-byte chunks of each resetting lane's row are written by N_H/2 lanes at once
                unsigned rm = __ballot_sync(0xffffffffu, did_reset);
                if (rm) {
                    const uint32_t h01 = tc::pack_h2(hf[0], hf[1]), h23 = tc::pack_h2(hf[2], hf[3]);
                    const int lane = threadIdx.x & 31;
                    while (rm) {
                        const int src = __ffs(rm) - 1;
                        rm &= rm - 1u;
                        const uint32_t v01 = __shfl_sync(0xffffffffu, h01, src);
                        const uint32_t v23 = __shfl_sync(0xffffffffu, h23, src);
                        if (lane < NH / 2)
                            tc::sts128(c.a1_row + (uint32_t)(src - lane) * 16u + (4 + lane) * kChunkA, v01, v23,
                                       v01, v23);
                    }
                }
            }
            L2F_PHASE(c, 13);
            if (tr) {
#pragma unroll
                for (int q = 0; q < 4; ++q) tr[21 + q] = o.a[q];
                tr[25] = o.reward;
                tr[26] = (float)fl;
                tr[27] = (float)e.ep_step;
                tr[28] = tr[29] = tr[30] = tr[31] = 0.0f;
            }
        }
        }
        if (active) {
#pragma unroll
            for (int q = 0; q < kStateDim; ++q) B.state[q * N + i] = e.s[q];
#pragma unroll
            for (int q = 0; q < 6; ++q) B.dist[q * N + i] = e.dist[q];
            if (kDR)
#pragma unroll
                for (int q = 0; q < 5; ++q) B.dr[q * N + i] = e.dr[q];
            B.ep_step[i] = e.ep_step;
            B.ep_return[i] = e.ep_return;
            // the ring now holds the full logical history: every entry valid
            if (NH > 0) B.hist_t0[i] = (int32_t)(P.t0 + (uint32_t)T) - NH;
            for (int s = 0; s < NH; ++s) {
                uint32_t h01, h23;
                tc::lds64(hist_addr(c, (NH - s) % NH), h01, h23);
                const __half2 x = *reinterpret_cast<__half2*>(&h01), y = *reinterpret_cast<__half2*>(&h23);
                B.hist[((int64_t)s * 4 + 0) * N + i] = __low2float(x);
                B.hist[((int64_t)s * 4 + 1) * N + i] = __high2float(x);
                B.hist[((int64_t)s * 4 + 2) * N + i] = __low2float(y);
                B.hist[((int64_t)s * 4 + 3) * N + i] = __high2float(y);
            }
            steps_done += (double)T;
        }
    }
#ifdef L2F_PHASE_TIMING
    __syncthreads();
    if (blockIdx.x == 0 && threadIdx.x == 0)
        for (int w = 0; w < kThreads / 32; ++w) {
            printf("L2F_PHASE warp %d", w);
            for (int k = 0; k < 14; ++k) printf(" %llu", g_ph[w][k]);
            printf("\n");
        }
#endif
    // statistics: warp -> fixed-order block sum -> this CTA's slot
    double* srow = reinterpret_cast<double*>(smem + OFF_STAT);
    const int warp = threadIdx.x >> 5;
    __syncthreads();  // the reset scratch is reused for the statistics rows
    stat_warp_to_smem(st, srow + warp * kStatsLen);
    double sd = steps_done;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sd += __shfl_xor_sync(0xffffffffu, sd, o);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) srow[warp * kStatsLen + 7] = sd;
    __syncthreads();
    if (threadIdx.x < kStatsLen) {
        double x = 0.0;
        for (int w = 0; w < kThreads / 32; ++w) x += srow[w * kStatsLen + threadIdx.x];
        B.slots[(size_t)blockIdx.x * kStatsLen + threadIdx.x] += x;
    }
    teardown_cta();
}

// -------------------------------------------------------------------------------------------
// Policy forward on explicit observations: obs [n][in_dim] fp32 -> act [n][4] (tanh output).
// The history part of each observation is written in order (ring rotation 0).
// -------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads, 1)
    policy_forward_kernel(const PolicyDev W, const float* __restrict__ obs, float* __restrict__ act, int64_t n,
                          int32_t n_tiles)
{
    extern __shared__ __align__(1024) uint8_t smem[];
    const uint32_t sbase = tc::smem_u32(smem);
    const int NH = (W.in_dim - 18) / 4;
    setup_cta(W, sbase, NH);
    TileCtx c = make_ctx(sbase);
    const int r = threadIdx.x % kM;
    for (int tile = blockIdx.x * kTiles + (int)(threadIdx.x / kM); tile < n_tiles; tile += gridDim.x * kTiles) {
        const int64_t i = (int64_t)tile * kM + r;
        const bool active = i < n;
        const float* row = obs + i * W.in_dim;
        float o[kObsCore];
#pragma unroll
        for (int q = 0; q < kObsCore; ++q) o[q] = active ? row[q] : 0.0f;
        write_obs_row(c, o);
        // with rot = 0, ring position p carries H[p]
        for (int p = 0; p < NH; ++p) {
            float h[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) h[q] = active ? row[18 + 4 * p + q] : 0.0f;
            tc::sts64(hist_addr(c, p), tc::pack_h2(h[0], h[1]), tc::pack_h2(h[2], h[3]));
        }
        float a[4];
        mlp_tile(c, sbase, NH, 0u, a, NoHook{});
        if (active)
#pragma unroll
            for (int q = 0; q < 4; ++q) act[i * 4 + q] = a[q];
    }
    teardown_cta();
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

// Upper bound of the rollout grid (statistics slots are sized with it; host-only arithmetic).
int mlp_rollout_grid(int64_t n)
{
    const int64_t tiles = (n + kM - 1) / kM;
    const int64_t g = (tiles + kTiles - 1) / kTiles;
    return (int)(g < 1024 ? g : 1024);
}

static int grid_for(int64_t n)
{
    const int64_t tiles = (n + kM - 1) / kM;
    int64_t g = (tiles + kTiles - 1) / kTiles;
    const int sms = sm_count();
    return (int)(g < sms ? (g < 1 ? 1 : g) : sms);
}

cudaError_t launch_rollout_mlp(const DevParams& P, const DevBufs& B, const PolicyDev& W, int32_t T, float* trace,
                               const int64_t* trace_ids, int32_t K, cudaStream_t s)
{
    if (P.n_hist % 4 != 0 || W.hidden != kHid || W.in_dim != 18 + 4 * P.n_hist) return cudaErrorNotSupported;
    static bool attr = false;
    if (!attr) {
        cudaError_t e =
            cudaFuncSetAttribute(rollout_mlp_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(rollout_mlp_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     kSmemBytes);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    const int n_tiles = (int)((P.n + kM - 1) / kM);
    if (P.flags & F_DOMAIN_RAND)
        rollout_mlp_kernel<true><<<grid_for(P.n), kThreads, kSmemBytes, s>>>(P, B, W, T, trace, trace_ids, K, n_tiles);
    else
        rollout_mlp_kernel<false><<<grid_for(P.n), kThreads, kSmemBytes, s>>>(P, B, W, T, trace, trace_ids, K, n_tiles);
    return cudaGetLastError();
}

cudaError_t launch_policy_forward(const PolicyDev& W, const float* obs, float* act, int64_t n, cudaStream_t s)
{
    if ((W.in_dim - 18) % 16 != 0 || W.hidden != kHid) return cudaErrorNotSupported;
    static bool attr = false;
    if (!attr) {
        cudaError_t e =
            cudaFuncSetAttribute(policy_forward_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    const int n_tiles = (int)((n + kM - 1) / kM);
    policy_forward_kernel<<<grid_for(n), kThreads, kSmemBytes, s>>>(W, obs, act, n, n_tiles);
    return cudaGetLastError();
}

}  // namespace l2f
