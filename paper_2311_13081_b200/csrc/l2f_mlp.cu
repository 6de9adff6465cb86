// l2f_mlp.cu -- fused rollout with the actor MLP on 5th-gen tensor cores (tcgen05), sm_100a.
//
// Per step and env (BASELINE configs[3]):
//   o_t = {p, R, v, omega} + noise  ++  H (last N_H applied actions, most recent first)
//   a_t = tanh(W3 q16(relu(W2 q16(relu(W1 q16(o_t) + b1)) + b2)) + b3)        (Q21)
//   then the same env transition as l2f_step (l2f_device.cuh).
//
// Design:
//  * persistent CTA per SM, 4 tiles x 128 envs (one 128-thread group per tile, units dealt
//    group-major over the CTAs); thread r of a tile owns env row r, which is
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
//    completion is signalled through tcgen05.commit -> mbarrier.  The other three tiles' warps
//    keep the FP32/INT pipes busy while one tile waits on the tensor core.
#include <cstdio>

#include "l2f_device.cuh"
#include "l2f_internal.h"
#include "l2f_tcgen05.cuh"

#ifndef L2F_HANDOFF_ARRIVE
#define L2F_HANDOFF_ARRIVE 1  // only the issuing warp waits at each hand-off (0: all four)
#endif
#ifndef L2F_MLP_E
#define L2F_MLP_E 1  // envs (tiles) per thread
#endif
#ifndef L2F_MLP_G
#define L2F_MLP_G 4  // 128-thread groups per CTA (3: -4.5 % at C5, -7 % at C4; round 2 measurement)
#endif

namespace l2f {
namespace {

constexpr int kE = L2F_MLP_E;
constexpr int kG = L2F_MLP_G;
constexpr int kTiles = kE * kG;  // 128-env tiles resident per CTA (tile g kE + k: group g, slot k)
constexpr int kM = 128;
constexpr int kThreads = kG * kM;
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
constexpr uint32_t OFF_BAR = OFF_W3 + kW3Bytes;       // kG MMA-done mbarriers (one per group)
constexpr uint32_t OFF_TMEM = OFF_BAR + 8 * kG;
constexpr uint32_t OFF_RTAB = (OFF_TMEM + 8 + 15) & ~15u;     // reset sampling table (16 float4)
constexpr uint32_t OFF_STAT = (OFF_RTAB + 256 + 127) & ~127u;  // reset scratch (40 uint4 per warp); reused by stats
constexpr uint32_t kScratchBytes = (kThreads / 32) * kResetScratch * 16;
static_assert(kScratchBytes >= (kThreads / 32) * kStatsLen * 8, "stats rows fit in the scratch");
constexpr uint32_t OFF_WSTAT = OFF_STAT + kScratchBytes;  // per-warp FP64 statistics rows (flushed per unit)
constexpr uint32_t kSmemBytes = OFF_WSTAT + (kThreads / 32) * kStatsLen * 8;
static_assert(kSmemBytes <= 232448, "shared memory budget");
constexpr uint32_t kTmemCols = 512;
// TMEM map: accumulators 64 columns per tile from 0; A2 (h1/h2 as fp16: 32 columns + 8 with the
// ones column) 40 per tile from 64 kTiles; the per-env noise stash (18 used: the next step's
// observation noise) 24 per tile after.
constexpr uint32_t kA2Col = 64 * kTiles;
constexpr uint32_t kStashCol = kA2Col + 40 * kTiles;
static_assert(kStashCol + 24 * kTiles <= kTmemCols, "TMEM budget");

constexpr uint32_t kIdescN64 = tc::make_idesc(128, 64, 0, 0);
constexpr uint32_t kIdescN64BMN = tc::make_idesc(128, 64, 0, 1);
constexpr uint32_t kIdescN16 = tc::make_idesc(128, 16, 0, 0);

__device__ __forceinline__ uint16_t h16(const uint16_t* p, int i) { return __ldg(p + i); }

// Debug build: a shared-memory access of `bytes` at saddr lies inside this kernel's dynamic
// shared memory.
__device__ __forceinline__ void smem_check(uint32_t saddr, uint32_t bytes)
{
#ifdef L2F_DEBUG_CHECKS
    extern __shared__ __align__(1024) uint8_t smem[];
    const uint32_t base = tc::smem_u32(smem);
    L2F_CHECK(saddr >= base && saddr + bytes <= base + kSmemBytes, "shared-memory address");
#else
    (void)saddr;
    (void)bytes;
#endif
}

__device__ __forceinline__ void st_u16(uint32_t saddr, uint16_t v)
{
    smem_check(saddr, 2);
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
    // tanh z = 1 - 2 / (exp(2z) + 1); exact limits at +-inf, absolute error ~1e-7.  exp(2z) =
    // 2^(z * 2 log2 e): one multiply (scaling by 2 is exact, so the product rounds as 2z log2 e).
    float e;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(z * 2.8853900817779268f));
    return 1.0f - __fdividef(2.0f, e + 1.0f);
}

// Per-thread context of a 128-thread group.  Thread r of group g owns row r of the group's kE
// tiles (tile g kE + k): row r of each A operand and TMEM lane r of each accumulator.  Tile k's
// addresses are tile 0's plus compile-time strides.
struct GroupCtx {
    uint32_t a1_row;     // this thread's row in the group's first A1 tile (+ k kA1Bytes)
    uint32_t a1;         // first A1 tile base
    uint32_t mbar;       // the group's MMA-done mbarrier
    uint32_t tmem_row;   // TMEM (this lane, first tile's accumulator column 0) (+ 64 k)
    uint32_t tmem_tile;  // TMEM (lane 0, first tile's accumulator)
    uint32_t stash_row;  // TMEM (this lane, first tile's noise stash) (+ 24 k)
    uint32_t a2_tmem;    // TMEM (lane 0, first tile's A2 column 0) (+ 40 k)
    uint32_t a2_trow;    // ... of this lane
    uint32_t bar_id;
    uint32_t phase;
    uint32_t r;          // thread index within the group
    uint32_t wig;        // warp index within the group (broadcast: uniform, so the issue branches are too)
#ifdef L2F_PHASE_TIMING
    uint32_t ph_last;    // debug build only: clock() at the last phase boundary
#endif
};

// Debug build only (-DL2F_PHASE_TIMING): per-warp cycles spent in each phase of a step,
// accumulated in shared memory and printed by CTA 0 at exit (scripts/phase_timing.sh).
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

// Epilogue of L1 / L2 for tile k: accumulator row -> relu -> fp16 -> this lane's A2 row in TMEM.
#ifndef L2F_SKIP_TMEM_PROXY_FENCE
#define L2F_SKIP_TMEM_PROXY_FENCE 1  // no shared-memory proxy fence before the TMEM-operand layers
#endif
#ifndef L2F_EPI_LOADS
#define L2F_EPI_LOADS 2  // 16-column TMEM loads in flight per wait (measured: 1 -2 %, 4 -2.7 % vs 2)
#endif
__device__ __forceinline__ void epilogue_hidden(const GroupCtx& c, int k)
{
    constexpr int kL = L2F_EPI_LOADS;
#pragma unroll
    for (int q0 = 0; q0 < 4; q0 += kL) {
        uint32_t v[kL][16];
#pragma unroll
        for (int j = 0; j < kL; ++j) tc::tmem_ld16(c.tmem_row + 64 * k + 16 * (q0 + j), v[j]);
        tc::tmem_wait_ld();
#pragma unroll
        for (int j = 0; j < kL; ++j)
            tc::tmem_st8u(c.a2_trow + 40 * k + 8 * (q0 + j), tc::relu_pack(v[j][0], v[j][1]),
                          tc::relu_pack(v[j][2], v[j][3]), tc::relu_pack(v[j][4], v[j][5]),
                          tc::relu_pack(v[j][6], v[j][7]), tc::relu_pack(v[j][8], v[j][9]),
                          tc::relu_pack(v[j][10], v[j][11]), tc::relu_pack(v[j][12], v[j][13]),
                          tc::relu_pack(v[j][14], v[j][15]));
    }
}

// The group's 128 threads hand their freshly written A rows (and finished TMEM reads) to the
// MMA issuer: proxy fence + tcgen05 fence + a 128-thread named barrier (id 1 + group) on which
// only the issuing warp waits; the other three arrive (bar.arrive) and run on into their hook.
// Safe to reuse the barrier: every warp next waits on this layer's MMA, which the issuer starts
// only after the barrier completed.  (+0.7 % once the issue branches were uniform; round 1
// measured no gain with the divergent ones.)
// kSmemA: the MMA reads an A operand the threads wrote to shared memory (layer 1: generic-proxy
// stores -> async-proxy reads need the proxy fence, a MEMBAR.ALL.CTA in SASS); layers 2 / 3
// take A from TMEM (tcgen05.st + wait::st + the thread-sync fence suffice) and B from weights
// fenced once at kernel start, so their hand-offs skip it.
template <bool kSmemA = true>
__device__ __forceinline__ void handoff_to_mma(GroupCtx& c, uint32_t issuer_warp)
{
    if (kSmemA || !L2F_SKIP_TMEM_PROXY_FENCE) tc::fence_proxy_async();
    tc::fence_before();
#if L2F_HANDOFF_ARRIVE
    // only the issuing warp waits
    if (c.wig == issuer_warp)
        tc::named_sync(c.bar_id, kM);
    else
        tc::named_arrive(c.bar_id, kM);
#else
    (void)issuer_warp;
    tc::named_sync(c.bar_id, kM);
#endif
}

__device__ __forceinline__ void wait_mma(GroupCtx& c)
{
    tc::mbar_wait(c.mbar, c.phase);
    c.phase ^= 1u;
    tc::fence_after();
}

struct NoHook {
    __device__ __forceinline__ void operator()(int) const {}
};

// The three layers on the tensor core for the group's kE tiles; layer l is issued (for all kE
// tiles, one commit) by lane 0 of the group's warp l - 1, so the issue work is spread over
// three warps.  Precondition: A1 rows written by all 128 threads.  `rot` = rotation of the
// history ring (W1 history row offset in slots).  hook(l) runs on every thread right after
// layer l's MMAs were issued, i.e. inside the MMA latency (used to draw the next step's noise).
template <int kNH, class Hook>
__device__ __forceinline__ void mlp_group(GroupCtx& c, uint32_t sbase, int n_hist, uint32_t rot, float (&a)[kE][4],
                                          const Hook& hook)
{
    // descriptors = base descriptor + (byte offset >> 4) in the start-address field (addresses
    // stay below 256 KB, so the 14-bit field never carries)
    L2F_PHASE(c, 0);
    // (rot is a loop-carried counter with a uniform start and uniform updates, so it already lives
    // in a uniform register; broadcasting it from lane 0 here cost a shuffle and an R2UR on the
    // layer-1 critical path after the proxy fence: -1.3 %)
    handoff_to_mma(c, 0);
    L2F_PHASE(c, 1);
    if (c.wig == 0) {  // the whole warp, converged; elect.sync picks the issuing lane
        tc::fence_after();
        const uint64_t dW1o = tc::make_desc(sbase + OFF_W1O, kHid * 16, 128);
        const uint64_t dW1h = tc::make_desc(sbase + OFF_W1H, 128, 2u * 4u * (uint32_t)n_hist * 16u) + 4u * rot;
#pragma unroll
        for (int k = 0; k < kE; ++k) {
            // L1: obs part (K = 32) then history (K = 4 N_H) with the rotated W1 history block
            const uint64_t dA1 = tc::make_desc(c.a1 + k * kA1Bytes, kChunkA, 128);
            const uint32_t d = c.tmem_tile + 64 * k;
            if constexpr (kNH == 32) {
                static_assert(2 * kChunkA / 16 == 256 && 2 * (kHid * 16) / 16 == 128, "issue_l1_elect offsets");
                tc::issue_l1_elect<8>(d, dA1, dW1o, dW1h, kIdescN64, kIdescN64BMN);
            } else {
                tc::mma_f16_elect(d, dA1, dW1o, kIdescN64, 0);
                tc::mma_f16_elect(d, dA1 + 2 * kChunkA / 16, dW1o + 2 * (kHid * 16) / 16, kIdescN64, 1);
#pragma unroll
                for (int j = 0; j < kMaxHist / 4; ++j)
                    if (j < n_hist / 4)
                        tc::mma_f16_elect(d, dA1 + (4 + 2 * j) * (kChunkA / 16), dW1h + 16u * j, kIdescN64BMN, 1);
            }
        }
        tc::commit_elect(c.mbar);
    }
    hook(1);
    L2F_PHASE(c, 2);
    wait_mma(c);
    L2F_PHASE(c, 3);
#pragma unroll
    for (int k = 0; k < kE; ++k) epilogue_hidden(c, k);
    tc::tmem_wait_st();
    L2F_PHASE(c, 4);
    handoff_to_mma<false>(c, 1);
    L2F_PHASE(c, 5);
    if (c.wig == 1) {
        tc::fence_after();
        const uint64_t dW2 = tc::make_desc(sbase + OFF_W2, kHid * 16, 128);
#pragma unroll
        for (int k = 0; k < kE; ++k)  // A from TMEM; K step 4: the ones column (bias row of W2)
            tc::issue_ts5_elect<2 * kHid * 16 / 16>(c.tmem_tile + 64 * k, c.a2_tmem + 40 * k, dW2, kIdescN64);
        tc::commit_elect(c.mbar);
    }
    hook(2);
    L2F_PHASE(c, 6);
    wait_mma(c);
    L2F_PHASE(c, 7);
#pragma unroll
    for (int k = 0; k < kE; ++k) epilogue_hidden(c, k);
    tc::tmem_wait_st();
    L2F_PHASE(c, 8);
    handoff_to_mma<false>(c, 2);
    L2F_PHASE(c, 9);
    if (c.wig == 2) {
        tc::fence_after();
        const uint64_t dW3 = tc::make_desc(sbase + OFF_W3, 256, 128);
#pragma unroll
        for (int k = 0; k < kE; ++k)
            tc::issue_ts5_elect<2 * 256 / 16>(c.tmem_tile + 64 * k, c.a2_tmem + 40 * k, dW3, kIdescN16);
        tc::commit_elect(c.mbar);
    }
    hook(3);
    L2F_PHASE(c, 10);
    wait_mma(c);
    uint32_t v[kE][4];
#pragma unroll
    for (int k = 0; k < kE; ++k) tc::tmem_ld4(c.tmem_row + 64 * k, v[k]);
    tc::tmem_wait_ld();
    tc::fence_before();
#pragma unroll
    for (int k = 0; k < kE; ++k)
#pragma unroll
        for (int j = 0; j < 4; ++j) a[k][j] = tanh_fast(__uint_as_float(v[k][j]));
    L2F_PHASE(c, 11);
}

// Observation-noise normals of one step for tile slot k, stashed per thread in TMEM (columns
// 0..17 of the env's stash) so they can be drawn inside the previous step's MMA latency
// without holding registers across the RK4.
__device__ __forceinline__ void stash_obs_noise(const DevParams& P, const GroupCtx& c, int k, uint32_t gid,
                                                uint32_t t, int part)
{
    float z[20];
    const uint32_t row = c.stash_row + 24 * k;
    if (part == 0 || part == 3) {
        obs_noise_blocks(P, gid, t, 0, 2, z);
        tc::tmem_st8(row + 0, z, 0);
    }
    if (part == 1 || part == 3) {
        obs_noise_blocks(P, gid, t, 2, 4, z);
        tc::tmem_st8(row + 8, z, 8);
    }
    if (part == 2 || part == 3) {
        obs_noise_blocks(P, gid, t, 4, 5, z);
        tc::tmem_st2(row + 16, z[16], z[17]);
    }
}

__device__ __forceinline__ void load_obs_noise(const GroupCtx& c, int k, float z[20])
{
    uint32_t v[16], w[4];
    tc::tmem_ld16(c.stash_row + 24 * k, v);
    tc::tmem_ld4(c.stash_row + 24 * k + 16, w);
    tc::tmem_wait_ld();
#pragma unroll
    for (int j = 0; j < 16; ++j) z[j] = __uint_as_float(v[j]);
    z[16] = __uint_as_float(w[0]);
    z[17] = __uint_as_float(w[1]);
    z[18] = z[19] = 0.0f;
}

__device__ __forceinline__ uint32_t a1_row(const GroupCtx& c, int k) { return c.a1_row + k * kA1Bytes; }

__device__ __forceinline__ void write_obs_row(const GroupCtx& c, int k, const float o[kObsCore])
{
    const uint32_t row = a1_row(c, k);
    smem_check(row, 16);
    smem_check(row + 2 * kChunkA, 16);
    tc::sts128(row, tc::pack_h2(o[0], o[1]), tc::pack_h2(o[2], o[3]), tc::pack_h2(o[4], o[5]),
               tc::pack_h2(o[6], o[7]));
    tc::sts128(row + kChunkA, tc::pack_h2(o[8], o[9]), tc::pack_h2(o[10], o[11]), tc::pack_h2(o[12], o[13]),
               tc::pack_h2(o[14], o[15]));
    tc::sts128(row + 2 * kChunkA, tc::pack_h2(o[16], o[17]), 0x00003C00u /* (1, 0) */, 0u, 0u);
}

// history ring position p of tile slot k -> A1 address (8 bytes: 4 fp16)
__device__ __forceinline__ uint32_t hist_addr(const GroupCtx& c, int k, int p)
{
    L2F_CHECK(p >= 0 && p < kMaxHist, "history ring position");
    const uint32_t a = a1_row(c, k) + (4 + (p >> 1)) * kChunkA + (p & 1) * 8;
    smem_check(a, 8);
    return a;
}

__device__ void setup_cta(const PolicyDev& W, uint32_t sbase, int n_hist, const DevParams* P = nullptr)
{
    extern __shared__ __align__(1024) uint8_t smem[];
    stage_weights(W, sbase, n_hist);
    if (P) reset_table_to_smem(*P, reinterpret_cast<float4*>(smem + OFF_RTAB));
    if (threadIdx.x == 0) {
        for (int g = 0; g < kG; ++g) tc::mbar_init(sbase + OFF_BAR + 8 * g, 1);  // MMA done
        tc::fence_mbar_init();
    }
    if (threadIdx.x < 32) tc::tmem_alloc(sbase + OFF_TMEM, kTmemCols);
    tc::fence_proxy_async();
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
}

__device__ __forceinline__ GroupCtx make_ctx(uint32_t sbase)
{
    extern __shared__ __align__(1024) uint8_t smem[];
    // group index and TMEM base broadcast from lane 0: the compiler then knows they are
    // warp-uniform and keeps the MMA descriptors / TMEM addresses in uniform registers (no
    // per-MMA R2UR waterfall loop in the issuing thread)
    const int g = __shfl_sync(0xffffffffu, (int)(threadIdx.x / kM), 0), r = threadIdx.x % kM;
    const uint32_t tbase = __shfl_sync(0xffffffffu, *reinterpret_cast<const uint32_t*>(smem + OFF_TMEM), 0);
    // the warp's TMEM lane quadrant, also from a broadcast (so the per-warp TMEM row addresses
    // of the epilogues and the noise stash are uniform too)
    const uint32_t lane_off = (uint32_t)(32 * __shfl_sync(0xffffffffu, (int)((threadIdx.x / 32) % 4), 0)) << 16;
    GroupCtx c;
    c.a1 = sbase + OFF_A1 + g * kE * kA1Bytes;
    c.a1_row = c.a1 + r * 16;
    c.mbar = sbase + OFF_BAR + 8 * g;
    c.tmem_tile = tbase + 64 * kE * g;
    c.tmem_row = c.tmem_tile + lane_off;
    c.stash_row = tbase + kStashCol + 24 * kE * g + lane_off;
    c.a2_tmem = tbase + kA2Col + 40 * kE * g;
    c.a2_trow = c.a2_tmem + lane_off;
#pragma unroll
    for (int k = 0; k < kE; ++k) {
        // constant ones column (K index 64 of layers 2 and 3) + zero pad
        tc::tmem_st8u(c.a2_trow + 40 * k + 32, 0x3C00u, 0u, 0u, 0u, 0u, 0u, 0u, 0u);
        tc::sts128(a1_row(c, k) + 3 * kChunkA, 0u, 0u, 0u, 0u);  // K 24..31: constant zero pad
    }
    tc::tmem_wait_st();
    c.bar_id = 1 + g;
    c.phase = 0;
    c.r = r;
    c.wig = (uint32_t)__shfl_sync(0xffffffffu, (int)((threadIdx.x / 32) % 4), 0);
#ifdef L2F_PHASE_TIMING
    if ((threadIdx.x & 31) == 0)
        for (int k = 0; k < 16; ++k) g_ph[threadIdx.x >> 5][k] = 0ull;
    c.ph_last = (uint32_t)clock();
#endif
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
// Fused rollout: T steps of {obs -> MLP (tensor cores) -> env transition} per env.  Each
// thread carries kE envs (one per tile slot) through every phase together, so the two envs'
// independent dependency chains (Philox, Box-Muller, RK4) interleave in the same basic blocks.
// -------------------------------------------------------------------------------------------
// kNH: N_H as a compile-time constant (32, the benchmark's history) or -1 (any N_H % 4 == 0,
// read from P at run time).  kTrace: the per-step trace of selected envs is compiled in only
// when one is requested (its per-step branches cost ~2.5 % of the untraced rollout).
template <bool kDR, int kNH, bool kTrace, uint32_t kF = kAnyFlags>
__global__ void __launch_bounds__(kThreads, 1)
    rollout_mlp_kernel(const DevParams P, const DevBufs B, const PolicyDev W, int32_t T, float* __restrict__ trace,
                       const int64_t* __restrict__ trace_ids, int32_t K, int32_t n_units)
{
    extern __shared__ __align__(1024) uint8_t smem[];
    const uint32_t sbase = tc::smem_u32(smem);
    const int NH = kNH >= 0 ? kNH : P.n_hist;
    setup_cta(W, sbase, NH, &P);
    GroupCtx c = make_ctx(sbase);
    const int64_t N = P.n;
    const int r = threadIdx.x % kM;
    // (the warp index broadcast from lane 0: a uniform value, so the address lives in a uniform
    // register instead of being rematerialised in the step loop)
    const uint32_t wcta = __shfl_sync(0xffffffffu, threadIdx.x >> 5, 0);
    uint4* const rscratch = reinterpret_cast<uint4*>(smem + OFF_STAT) + wcta * kResetScratch;
    const float4* const rtab = reinterpret_cast<const float4*>(smem + OFF_RTAB);
    double* const wrow = reinterpret_cast<double*>(smem + OFF_WSTAT) + (threadIdx.x >> 5) * kStatsLen;
    if ((threadIdx.x & 31) < kStatsLen) wrow[threadIdx.x & 31] = 0.0;
    __syncwarp();
    const bool obs_noise = (flags_of<kF>(P) & F_OBS_NOISE) != 0;

    // unit u = tiles u kE .. u kE + kE - 1 (one per tile slot)
    for (int u = (int)(threadIdx.x / kM) * (int)gridDim.x + blockIdx.x; u < n_units; u += gridDim.x * kG) {
        StatPk st;
        statpk_zero(st);
        int64_t i[kE];
        bool active[kE];
        uint32_t gid[kE];
        EnvReg e[kE];
        int tslot[kE];
#pragma unroll
        for (int k = 0; k < kE; ++k) {
            i[k] = ((int64_t)u * kE + k) * kM + r;
            active[k] = i[k] < N;
            gid[k] = P.id_offset + (uint32_t)i[k];
            if (active[k]) {
                grp_load_scalar<kStateDim>(B.state, i[k], N, e[k].s);
                grp_load_scalar<6>(B.dist, i[k], N, e[k].dist);
                if (kDR)
                    grp_load_scalar<5>(B.dr, i[k], N, e[k].dr);
                else
#pragma unroll
                    for (int q = 0; q < 5; ++q) e[k].dr[q] = 1.0f;
                e[k].ep_step = B.ep_step[i[k]];
                e[k].ep_return = B.ep_return[i[k]];
            } else {
#pragma unroll
                for (int q = 0; q < kStateDim; ++q) e[k].s[q] = 0.0f;
                e[k].s[3] = 1.0f;
#pragma unroll
                for (int q = 0; q < 6; ++q) e[k].dist[q] = 0.0f;
#pragma unroll
                for (int q = 0; q < 5; ++q) e[k].dr[q] = 1.0f;
                e[k].ep_step = 0;
                e[k].ep_return = 0.0f;
            }
            // logical history at t0 (H[j] = a_{t0-1-j}, or the episode fill) -> A1 position (-tau) mod N_H
            const int32_t h0 = active[k] ? B.hist_t0[i[k]] : 0;
            for (int j = 0; j < NH; ++j) {
                float h[4] = {0.f, 0.f, 0.f, 0.f};
                if (active[k]) hist_entry(B, N, NH, i[k], (int64_t)P.t0, j, h0, h);
                const int64_t tau = (int64_t)P.t0 - 1 - j;
                const int p = (int)(((-tau) % NH + NH) % NH);
                tc::sts64(hist_addr(c, k, p), tc::pack_h2(h[0], h[1]), tc::pack_h2(h[2], h[3]));
            }
            tslot[k] = -1;
            if (kTrace && active[k])
                for (int q = 0; q < K; ++q)
                    if (trace_ids[q] == i[k]) tslot[k] = q;
            if (obs_noise) stash_obs_noise(P, c, k, gid[k], P.t0, 3);
        }
        // ring rotation (t - 1) mod N_H and write position (-t) mod N_H, advanced incrementally
        uint32_t rot = NH > 0 ? (P.t0 + (uint32_t)NH - 1u) % (uint32_t)NH : 0u;
        int wpos = NH > 0 ? (int)(((uint32_t)NH - P.t0 % (uint32_t)NH) % (uint32_t)NH) : 0;
        const uint32_t t_last = P.t0 + (uint32_t)T;
        uint32_t t = P.t0;
        for (int sg = 0; sg < P.n_stages; ++sg) {  // curriculum stages of this launch
        const StageW& W = P.stage[sg];
        for (const uint32_t t_stop = stage_stop(P, sg, t_last); t < t_stop; ++t) {
            const int32_t ks = (int32_t)(t - P.t0);
            tc::tmem_wait_st();  // the stashed noise of this step
#pragma unroll
            for (int k = 0; k < kE; ++k) {
                float ob[kObsCore];
                if (obs_noise) {
                    // the noise-free observation is formed while the stashed normals load from TMEM
                    uint32_t v[16], w[4];
                    tc::tmem_ld16(c.stash_row + 24 * k, v);
                    tc::tmem_ld4(c.stash_row + 24 * k + 16, w);
                    float z0[20];
#pragma unroll
                    for (int j = 0; j < 20; ++j) z0[j] = 0.0f;
                    observe_core_z<0u>(P, e[k].s, z0, ob);
                    tc::tmem_wait_ld();
                    float z[20];
#pragma unroll
                    for (int j = 0; j < 16; ++j) z[j] = __uint_as_float(v[j]);
                    z[16] = __uint_as_float(w[0]);
                    z[17] = __uint_as_float(w[1]);
                    z[18] = z[19] = 0.0f;
                    add_obs_noise(P, z, ob);
                } else {
                    float z[20];
                    observe_core_z<kF>(P, e[k].s, z, ob);
                }
                write_obs_row(c, k, ob);
            }
            float a[kE][4], za[kE][4];
            // noise draws inside the MMA latency, unconditionally (no flag branch splits the
            // independent Philox chains into separate basic blocks; unused draws are discarded)
            mlp_group<kNH>(c, sbase, NH, rot, a, [&](int l) {
#pragma unroll
                for (int k = 0; k < kE; ++k) {
                    if (l == 3) {  // this step's action noise (two Philox chains per hook: 2 obs / 2 obs / obs + action)
                        box_muller2(draw(P, gid[k], t, S_ACT, 0), za[k]);
                        const bool an = (flags_of<kF>(P) & F_ACTION_NOISE) != 0;
#pragma unroll
                        for (int q = 0; q < 4; ++q) za[k][q] = an ? za[k][q] : 0.0f;
                    }
                    stash_obs_noise(P, c, k, gid[k], t + 1, l - 1);
                }
            });
            if (NH > 0 && ++rot == (uint32_t)NH) rot = 0;
            Trans o[kE];
#pragma unroll
            for (int k = 0; k < kE; ++k) {
                if (kTrace && tslot[k] >= 0) {  // (traced envs only: the address is not formed otherwise)
                    L2F_CHECK(tslot[k] < K && ks >= 0 && ks < T, "trace index");
                    float* tr = trace + ((int64_t)ks * K + tslot[k]) * kTraceFields;
#pragma unroll
                    for (int q = 0; q < kStateDim; ++q) tr[q] = e[k].s[q];
#pragma unroll
                    for (int q = 0; q < 4; ++q) tr[17 + q] = a[k][q];
                }
            }
#pragma unroll
            for (int k = 0; k < kE; ++k) transition<kDR, kF>(P, W, e[k], gid[k], t, a[k], za[k], o[k]);
#ifdef L2F_PHASE_TIMING
#pragma unroll
            for (int k = 0; k < kE; ++k)  // attribution: the transition's results exist before the clock read
                asm volatile("" ::"r"(o[k].flags), "f"(o[k].reward), "f"(e[k].s[0]), "f"(e[k].s[3]), "f"(e[k].s[7]),
                             "f"(e[k].s[10]), "f"(e[k].s[13]), "f"(e[k].s[16]));
#endif
            L2F_PHASE(c, 12);
#pragma unroll
            for (int k = 0; k < kE; ++k) {
                uint32_t fl = o[k].flags;
                const bool ended = (fl & (D_TERM | D_TRUNC)) != 0;
                statpk_episode(st, o[k], ended && active[k]);
                L2F_PHASE(c, 14);
                bool did_reset = false;
                float hf[4];
                if (flags_of<kF>(P) & F_AUTO_RESET)
                    did_reset = reset_env_warp<kDR ? 8 : 6, kF>(P, rtab, e[k], gid[k], t + 1, ended && active[k], hf, rscratch);
                fl |= did_reset ? D_RESET : 0u;
                L2F_PHASE(c, 15);
                // an episode that ended without auto-reset restarts its counters (selects, no branch)
                const bool restart = ended && !did_reset;
                e[k].ep_step = restart ? 0 : e[k].ep_step;
                e[k].ep_return = restart ? 0.0f : e[k].ep_return;
                if (NH > 0) {
                    // the applied action into its ring slot, for every lane (a reset's refill below
                    // overwrites it, in program order)
                    tc::sts64(hist_addr(c, k, wpos), tc::pack_h2(o[k].a[0], o[k].a[1]), tc::pack_h2(o[k].a[2], o[k].a[3]));
                    // new episode: the lane's whole history row takes the fill value (Q10):
                    // N_H/2 16-byte stores by the resetting lanes only
                    if (did_reset) {
                        // one register quad stored N_H / 2 times (C++ stores: asm operands made the
                        // compiler build a fresh quad per store)
                        const uint32_t h01 = tc::pack_h2(hf[0], hf[1]), h23 = tc::pack_h2(hf[2], hf[3]);
                        if constexpr (kNH == 32) {
                            smem_check(a1_row(c, k) + 4 * kChunkA, 16 * kChunkA);
                            tc::sts128_x16<kChunkA>(a1_row(c, k) + 4 * kChunkA, h01, h23, h01, h23);
                        } else {
                            const uint4 hv = make_uint4(h01, h23, h01, h23);
                            uint8_t* const row = smem + (a1_row(c, k) - sbase);
#pragma unroll
                            for (int q = 0; q < kMaxHist / 2; ++q)
                                if (q < NH / 2) {
                                    smem_check(a1_row(c, k) + (4 + q) * kChunkA, 16);
                                    *reinterpret_cast<uint4*>(row + (4 + q) * kChunkA) = hv;
                                }
                        }
                    }
                }
                if (kTrace && tslot[k] >= 0) {
                    float* tr = trace + ((int64_t)ks * K + tslot[k]) * kTraceFields;
#pragma unroll
                    for (int q = 0; q < 4; ++q) tr[21 + q] = o[k].a[q];
                    tr[25] = o[k].reward;
                    tr[26] = (float)fl;
                    tr[27] = (float)e[k].ep_step;
                    tr[28] = tr[29] = tr[30] = tr[31] = 0.0f;
                }
            }
            if (NH > 0 && --wpos < 0) wpos = NH - 1;
            L2F_PHASE(c, 13);
        }
        }
        int n_active = 0;
#pragma unroll
        for (int k = 0; k < kE; ++k) {
            const int64_t ik = ((int64_t)u * kE + k) * kM + r;
            if (ik >= N) continue;
            ++n_active;
            grp_store<kStateDim>(B.state, ik, N, e[k].s);
            grp_store<6>(B.dist, ik, N, e[k].dist);
            if (kDR) grp_store<5>(B.dr, ik, N, e[k].dr);
            B.ep_step[ik] = e[k].ep_step;
            B.ep_return[ik] = e[k].ep_return;
            // the ring now holds the full logical history: every entry valid
            if (NH > 0) B.hist_t0[ik] = (int32_t)(P.t0 + (uint32_t)T) - NH;
            for (int s = 0; s < NH; ++s) {
                uint32_t h01, h23;
                tc::lds64(hist_addr(c, k, (NH - s) % NH), h01, h23);
                const __half2 x = *reinterpret_cast<__half2*>(&h01), y = *reinterpret_cast<__half2*>(&h23);
                B.hist[(int64_t)s * N + ik] = make_float4(__low2float(x), __high2float(x), __low2float(y), __high2float(y));
            }
        }
        statpk_flush(st, (double)__reduce_add_sync(0xffffffffu, n_active) * (double)T, wrow);
    }
#ifdef L2F_PHASE_TIMING
    __syncthreads();
    if (blockIdx.x == 0 && threadIdx.x == 0)
        for (int w = 0; w < kThreads / 32; ++w) {
            printf("L2F_PHASE warp %d", w);
            for (int k = 0; k < 16; ++k) printf(" %llu", g_ph[w][k]);
            printf("\n");
        }
#endif
    // statistics: per-warp rows (flushed per unit) -> fixed-order block sum -> this CTA's slot
    __syncthreads();
    L2F_CHECK((int)blockIdx.x < B.n_slots, "statistics slot");
    if (threadIdx.x < kStatsLen) {
        const double* rows = reinterpret_cast<const double*>(smem + OFF_WSTAT);
        double x = 0.0;
        for (int w = 0; w < kThreads / 32; ++w) x += rows[w * kStatsLen + threadIdx.x];
        B.slots[(size_t)blockIdx.x * kStatsLen + threadIdx.x] += x;
    }
    teardown_cta();
}

// Batched actor inference (l2f_policy_forward): the same group/MMA code as the rollout.
__global__ void __launch_bounds__(kThreads, 1)
    policy_forward_kernel(const PolicyDev W, const float* __restrict__ obs, float* __restrict__ act, int64_t n,
                          int32_t n_units)
{
    extern __shared__ __align__(1024) uint8_t smem[];
    const uint32_t sbase = tc::smem_u32(smem);
    const int NH = (W.in_dim - 18) / 4;
    setup_cta(W, sbase, NH);
    GroupCtx c = make_ctx(sbase);
    const int r = threadIdx.x % kM;
    for (int u = (int)(threadIdx.x / kM) * (int)gridDim.x + blockIdx.x; u < n_units; u += gridDim.x * kG) {
        int64_t i[kE];
#pragma unroll
        for (int k = 0; k < kE; ++k) {
            i[k] = ((int64_t)u * kE + k) * kM + r;
            const bool active = i[k] < n;
            const float* row = obs + i[k] * W.in_dim;
            float o[kObsCore];
#pragma unroll
            for (int q = 0; q < kObsCore; ++q) o[q] = active ? row[q] : 0.0f;
            write_obs_row(c, k, o);
            // with rot = 0, ring position p carries H[p]
            for (int p = 0; p < NH; ++p) {
                float h[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) h[q] = active ? row[18 + 4 * p + q] : 0.0f;
                tc::sts64(hist_addr(c, k, p), tc::pack_h2(h[0], h[1]), tc::pack_h2(h[2], h[3]));
            }
        }
        float a[kE][4];
        mlp_group<-1>(c, sbase, NH, 0u, a, NoHook{});
#pragma unroll
        for (int k = 0; k < kE; ++k)
            if (i[k] < n)
#pragma unroll
                for (int q = 0; q < 4; ++q) act[i[k] * 4 + q] = a[k][q];
    }
    teardown_cta();
}

// -------------------------------------------------------------------------------------------
// Lissajous tracking evaluation (Table III analogue; Q28-Q31).  Same group /
// MMA machinery as the rollout; per env: start at p_ref(0) at rest, the actor observes the
// clipped setpoint shift, the error to p_ref(k dt) is accumulated in FP64 until the
// first termination on the error state.  No exploration noise, resets, disturbance or DR.
// -------------------------------------------------------------------------------------------
__device__ __forceinline__ void lissajous_ref(const TrackDev& S, double dt_over_T, float w, int32_t k, float p[3],
                                              float v[3])
{
    const double ph = (double)k * dt_over_T;  // cycles
    const float f = (float)(ph - floor(ph));
    float s1, c1, s2, c2;
    sincospif(2.0f * f, &s1, &c1);
    sincospif(4.0f * f, &s2, &c2);
    p[0] = S.ax * c1;
    p[1] = S.ay * s2;
    p[2] = S.z;
    v[0] = -S.ax * w * s1;
    v[1] = 2.0f * S.ay * w * c2;
    v[2] = 0.0f;
}

// kF / kNH: compile-time flags and N_H for the common tracking setup (observation noise on,
// N_H = 32), as for the rollout; kAnyFlags / -1 read them at run time.
template <uint32_t kF = kAnyFlags, int kNH = -1>
__global__ void __launch_bounds__(kThreads, 1)
    track_mlp_kernel(const DevParams P, const DevBufs B, const PolicyDev W, const TrackDev S, int32_t n_units)
{
    extern __shared__ __align__(1024) uint8_t smem[];
    const uint32_t sbase = tc::smem_u32(smem);
    const int NH = kNH >= 0 ? kNH : P.n_hist;
    setup_cta(W, sbase, NH, &P);
    GroupCtx c = make_ctx(sbase);
    const int64_t N = P.n;
    const int r = threadIdx.x % kM;
    const bool obs_noise = (flags_of<kF>(P) & F_OBS_NOISE) != 0;
    const StageW& SW = P.stage[0];
    for (int u = (int)(threadIdx.x / kM) * (int)gridDim.x + blockIdx.x; u < n_units; u += gridDim.x * kG) {
        int64_t i[kE];
        bool active[kE];
        uint32_t gid[kE];
        EnvReg e[kE];
        double dtT[kE], se[kE], sexy[kE];
        float w[kE];
        int32_t ok[kE];
        bool alive[kE];
#pragma unroll
        for (int k = 0; k < kE; ++k) {
            i[k] = ((int64_t)u * kE + k) * kM + r;
            active[k] = i[k] < N;
            gid[k] = P.id_offset + (uint32_t)i[k];
            const float Tc = active[k] ? S.cycle_time[i[k]] : 1.0f;
            dtT[k] = (double)P.dt / (double)Tc;
            w[k] = 6.28318530717958648f / Tc;
            // start: p_ref(0) = (A_x, 0, z) at rest, level, rotors at hover (Q30)
#pragma unroll
            for (int q = 0; q < kStateDim; ++q) e[k].s[q] = 0.0f;
            e[k].s[0] = S.ax;
            e[k].s[2] = S.z;
            e[k].s[3] = 1.0f;
#pragma unroll
            for (int q = 13; q < 17; ++q) e[k].s[q] = S.hover_rpm;
#pragma unroll
            for (int q = 0; q < 6; ++q) e[k].dist[q] = 0.0f;
#pragma unroll
            for (int q = 0; q < 5; ++q) e[k].dr[q] = 1.0f;
            e[k].ep_step = 0;
            e[k].ep_return = 0.0f;
            const uint32_t hh = tc::pack_h2(S.hover_a, S.hover_a);
            for (int j = 0; j < NH; ++j) tc::sts64(hist_addr(c, k, j), hh, hh);
            se[k] = sexy[k] = 0.0;
            ok[k] = 0;
            alive[k] = true;
            stash_obs_noise(P, c, k, gid[k], P.t0, 3);
        }
        uint32_t rot = NH > 0 ? (P.t0 + (uint32_t)NH - 1u) % (uint32_t)NH : 0u;
        int wpos = NH > 0 ? (int)(((uint32_t)NH - P.t0 % (uint32_t)NH) % (uint32_t)NH) : 0;
        for (int32_t ks = 0; ks < S.n_steps; ++ks) {
            const uint32_t t = P.t0 + (uint32_t)ks;
            tc::tmem_wait_st();
#pragma unroll
            for (int k = 0; k < kE; ++k) {
                float ob[kObsCore], z[20], pr[3], vr[3];
                if (obs_noise) load_obs_noise(c, k, z);
                observe_core_z<kF>(P, e[k].s, z, ob);
                lissajous_ref(S, dtT[k], w[k], ks, pr, vr);
#pragma unroll
                for (int j = 0; j < 3; ++j) {  // setpoint shift with clipping (Q29)
                    ob[j] = fminf(fmaxf(ob[j] - pr[j], -S.clip_pos), S.clip_pos);
                    ob[12 + j] = fminf(fmaxf(ob[12 + j] - vr[j], -S.clip_vel), S.clip_vel);
                }
                write_obs_row(c, k, ob);
            }
            float a[kE][4];
            mlp_group<kNH>(c, sbase, NH, rot, a, [&](int l) {
#pragma unroll
                for (int k = 0; k < kE; ++k) stash_obs_noise(P, c, k, gid[k], t + 1, l - 1);
            });
            if (NH > 0 && ++rot == (uint32_t)NH) rot = 0;
#pragma unroll
            for (int k = 0; k < kE; ++k) {
                const float za[4] = {0.f, 0.f, 0.f, 0.f};
                Trans o;
                transition<false, kF>(P, SW, e[k], gid[k], t, a[k], za, o);
                if (NH > 0)
                    tc::sts64(hist_addr(c, k, wpos), tc::pack_h2(o.a[0], o.a[1]), tc::pack_h2(o.a[2], o.a[3]));
                float pr[3], vr[3];
                lissajous_ref(S, dtT[k], w[k], ks + 1, pr, vr);
                const float* s1 = e[k].s;
                const float ex = s1[0] - pr[0], ey = s1[1] - pr[1], ez = s1[2] - pr[2];
                const float dvx = s1[7] - vr[0], dvy = s1[8] - vr[1], dvz = s1[9] - vr[2];
                const float ww = s1[10] * s1[10] + s1[11] * s1[11] + s1[12] * s1[12];
                const float einf = fmaxf(fabsf(ex), fmaxf(fabsf(ey), fabsf(ez)));
                const bool out = (einf > P.term_pos) | (dvx * dvx + dvy * dvy + dvz * dvz > P.term_vel2) |
                                 (ww > P.term_angvel2);
                const bool term = ((o.flags & D_DIV) != 0) | (S.terminate != 0 && out);
                alive[k] = alive[k] && !term;
                if (alive[k]) {
                    const double dx = ex, dy = ey, dz = ez;
                    sexy[k] += dx * dx + dy * dy;
                    se[k] += dx * dx + dy * dy + dz * dz;
                    ok[k] = ks + 1;
                }
            }
            if (NH > 0 && --wpos < 0) wpos = NH - 1;
        }
#pragma unroll
        for (int k = 0; k < kE; ++k) {
            if (!active[k]) continue;
            const int64_t ik = i[k];
            S.rmse[ik] = ok[k] > 0 ? (float)sqrt(se[k] / ok[k]) : 0.0f;
            S.rmse_xy[ik] = ok[k] > 0 ? (float)sqrt(sexy[k] / ok[k]) : 0.0f;
            S.steps_ok[ik] = ok[k];
            // the env is left in the final tracking state (history ring complete, as after a rollout)
            grp_store<kStateDim>(B.state, ik, N, e[k].s);
            grp_store<6>(B.dist, ik, N, e[k].dist);
            grp_store<5>(B.dr, ik, N, e[k].dr);
            B.ep_step[ik] = ok[k];
            B.ep_return[ik] = 0.0f;
            if (NH > 0) {
                const int32_t t_end = (int32_t)(P.t0 + (uint32_t)S.n_steps);
                B.hist_t0[ik] = t_end - NH;
                B.hist_fill[ik] = make_float4(S.hover_a, S.hover_a, S.hover_a, S.hover_a);
            }
            for (int sl = 0; sl < NH; ++sl) {
                uint32_t h01, h23;
                tc::lds64(hist_addr(c, k, (NH - sl) % NH), h01, h23);
                const __half2 x = *reinterpret_cast<__half2*>(&h01), y = *reinterpret_cast<__half2*>(&h23);
                B.hist[(int64_t)sl * N + ik] = make_float4(__low2float(x), __high2float(x), __low2float(y), __high2float(y));
            }
        }
    }
    teardown_cta();
}

int sm_count()
{
    static std::atomic<int> cache[64] = {};
    const int dev = current_device();
    int n = cache[dev].load();
    if (n == 0) {
        if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
        cache[dev].store(n);
    }
    return n;
}

int64_t units_for(int64_t n) { return ((n + kM - 1) / kM + kE - 1) / kE; }

}  // namespace

// Upper bound of the rollout grid (statistics slots are sized with it; host-only arithmetic).
int mlp_rollout_grid(int64_t n)  // upper bound of grid_for on any device (statistics slots)
{
    const int64_t g = units_for(n);
    return (int)(g < 1 ? 1 : (g < 1024 ? g : 1024));
}

// One CTA per SM (or one per unit when there are fewer units than SMs).  Units are dealt
// group-major: unit u of a round runs on CTA u mod grid, group u / grid, so a partial last
// round (2^21 envs: 16384 tiles = 27.7 rounds of 148 x 4) leaves every SM with 2-3 busy groups
// instead of 100 SMs with 4 and 48 idle, and the fewer groups per SM run faster.
static int grid_for(int64_t n)
{
    const int64_t u = units_for(n);
    const int sms = sm_count();
    return (int)(u < sms ? (u < 1 ? 1 : u) : sms);
}

cudaError_t launch_rollout_mlp(const DevParams& P, const DevBufs& B, const PolicyDev& W, int32_t T, float* trace,
                               const int64_t* trace_ids, int32_t K, cudaStream_t s)
{
    if (P.n_hist % 4 != 0 || W.hidden != kHid || W.in_dim != 18 + 4 * P.n_hist) return cudaErrorNotSupported;
    static std::atomic<size_t> attr[10][64] = {};
    const bool dr = (P.flags & F_DOMAIN_RAND) != 0, h32 = P.n_hist == 32, tr = trace != nullptr;
    using Kern = decltype(&rollout_mlp_kernel<true, 32, true>);
    static const Kern table[8] = {rollout_mlp_kernel<false, -1, false>, rollout_mlp_kernel<false, -1, true>,
                                  rollout_mlp_kernel<false, 32, false>, rollout_mlp_kernel<false, 32, true>,
                                  rollout_mlp_kernel<true, -1, false>,  rollout_mlp_kernel<true, -1, true>,
                                  rollout_mlp_kernel<true, 32, false>,  rollout_mlp_kernel<true, 32, true>};
    // the benchmark's feature mix (C4 / C5: every feature but DR and the rotor-delay ablation)
    // as a compile-time specialisation
    constexpr uint32_t kC5 = F_OBS_NOISE | F_ACTION_NOISE | F_TERMINATION | F_AUTO_RESET | F_DISTURBANCE;
    const bool c5 = !dr && h32 && P.flags == kC5;
    const int sel = c5 ? 8 + tr : 4 * dr + 2 * h32 + tr;
    const Kern kern = c5 ? (tr ? rollout_mlp_kernel<false, 32, true, kC5> : rollout_mlp_kernel<false, 32, false, kC5>)
                         : table[sel];
    const cudaError_t e = ensure_smem_attr(kern, kSmemBytes, attr[sel]);
    if (e != cudaSuccess) return e;
    kern<<<grid_for(P.n), kThreads, kSmemBytes, s>>>(P, B, W, T, trace, trace_ids, K, (int32_t)units_for(P.n));
    return cudaGetLastError();
}

cudaError_t launch_track_mlp(const DevParams& P, const DevBufs& B, const PolicyDev& W, const TrackDev& S,
                             cudaStream_t s)
{
    if (P.n_hist % 4 != 0 || W.hidden != kHid || W.in_dim != 18 + 4 * P.n_hist) return cudaErrorNotSupported;
    static std::atomic<size_t> attr[2][64] = {};
    const bool spec = P.flags == F_OBS_NOISE && P.n_hist == 32;
    const auto kern = spec ? track_mlp_kernel<F_OBS_NOISE, 32> : track_mlp_kernel<>;
    const cudaError_t e = ensure_smem_attr(kern, kSmemBytes, attr[spec]);
    if (e != cudaSuccess) return e;
    kern<<<grid_for(P.n), kThreads, kSmemBytes, s>>>(P, B, W, S, (int32_t)units_for(P.n));
    return cudaGetLastError();
}

cudaError_t launch_policy_forward(const PolicyDev& W, const float* obs, float* act, int64_t n, cudaStream_t s)
{
    if ((W.in_dim - 18) % 16 != 0 || W.hidden != kHid) return cudaErrorNotSupported;
    static std::atomic<size_t> attr[64] = {};
    const cudaError_t e = ensure_smem_attr(policy_forward_kernel, kSmemBytes, attr);
    if (e != cudaSuccess) return e;
    policy_forward_kernel<<<grid_for(n), kThreads, kSmemBytes, s>>>(W, obs, act, n, (int32_t)units_for(n));
    return cudaGetLastError();
}

}  // namespace l2f
